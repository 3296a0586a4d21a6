# one bench run, summarised: value, e2e, megakernel ms, roofline frac, phase ms
python bench.py --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'mk_ms', round(d['roofline']['ms_per_launch'],4), 'frac', round(d['roofline']['frac'],4), d['kernel_ms_per_round'])"
