set -x
for q in 14 7 4; do SRL_MK_CS_QKV=$q python tools/mk_trace.py --prompt 160 2>&1 | grep -E "^(round|qkv|attn)"; done
for o in 7 4 2 1; do SRL_MK_CS_O=$o python tools/mk_trace.py --prompt 160 2>&1 | grep -E "^(round|o )"; done
for d in 8 4; do SRL_MK_CS_DOWN=$d python tools/mk_trace.py --prompt 160 2>&1 | grep -E "^(round|down)"; done
for g in 2; do SRL_MK_CS_GU=$g python tools/mk_trace.py --prompt 160 2>&1 | grep -E "^(round|gu)"; done
