"""Generate tests/golden/reference_vectors.json by running the UNMODIFIED
reference (oracle/_ref/libstreamrl_ref.so, built from /root/reference by
oracle/Makefile).  Run here (the reference is not on the GPU box):

    python tests/golden/make_golden.py

Every vector records which reference routine produced it.
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Ref  # noqa: E402

ASSETS = Path("/root/reference/proj/assets")


def main():
    r = Ref()
    out = {}
    # rng.hpp:18-69
    import ctypes as C  # noqa: F401

    # acceptance.cpp:405-457: mixed_policy_sample, recurrent (7,4,0.6,2025),
    # drift_checkpoints(3, 0.3, 4), schedule(16,4), seed 618, 3 streams.
    base = r.random_recurrent_policy(7, 4, 0.6, 2025)
    ck = r.drift_checkpoints(base, 3, 0.3, 4)
    sp, stale = r.mixed_policy_sample(ck, 16, 4, False, "p", 3, 16, 618)
    _, recomp = r.mixed_policy_sample(ck, 16, 4, True, "p", 3, 16, 618)
    from oracle.oracle import Oracle

    o = Oracle()
    out["cross_module"] = dict(source="rl_math.cpp:312-319 mixed_policy_sample",
                               checkpoints=ck, switch_points=sp,
                               seeds=[o.derive_stream(618, i) for i in range(3)],
                               stale=stale, recompute=recomp)

    # test_protocol.cpp:271-287 demo scenario through proto::Engine in lockstep
    v0 = json.loads((ASSETS / "policies/demo_policy.json").read_text())
    v1 = json.loads((ASSETS / "policies/demo_policy_v1.json").read_text())
    script = {"policy": v0, "recompute": False, "steps": [
        {"open": {"prompt_id": "demo", "max_tokens": 12, "seed": 5}},
        {"open": {"prompt_id": "demo", "max_tokens": 12, "seed": 6}},
        {"advance": 5}, {"update": {"version": 1, "policy": v1}}, {"advance": 7}]}
    tr = r.engine_lockstep(script)
    out["demo_scenario"] = dict(source="engine.cpp Engine lockstep (demo_two_streams.json)",
                                v0=v0, v1=v1, streams=tr["streams"], updates=tr["updates"])

    # rng vectors
    s = C.c_uint64(42)
    out["rng"] = dict(source="rng.hpp:18-57", splitmix_42=o.splitmix(42, 8),
                      uniforms_7=o.uniforms(7, 8), gaussians_99=o.gaussians(99, 6),
                      derive=[[sd, i, o.derive_stream(sd, i)] for sd in (0, 618, 2**63 + 5)
                              for i in (0, 1, 7)])

    # sample_trajectories: terminator-first and determinism (test_rl_math.cpp:289-305)
    term = {"schema": "streamrl.policy/1", "type": "tabular", "vocab_size": 2,
            "context_order": 0, "default_logits": [0.0, 0.0],
            "rows": [{"prompt_id": "p", "context": [], "logits": [-2000.0, 0.0]}]}
    _, tt = r.mixed_policy_sample([term], 0, 1, False, "p", 10, 8, 42, 1)
    uni = {"schema": "streamrl.policy/1", "type": "tabular", "vocab_size": 6, "context_order": 0,
           "default_logits": [0.0] * 6, "rows": []}
    _, ut = r.mixed_policy_sample([uni], 0, 1, False, "p", 5, 12, 7)
    out["sampling"] = dict(source="rl_math.cpp:278-284 sample_trajectories",
                           terminator_policy=term, terminator=tt, uniform_policy=uni, uniform=ut)

    # policy_logprobs hand values (test_rl_math.cpp:106-132)
    hand = {"schema": "streamrl.policy/1", "type": "tabular", "vocab_size": 2, "context_order": 0,
            "default_logits": [0.0, 0.0],
            "rows": [{"prompt_id": "p", "context": [], "logits": [0.0, 1.0986122886681098]}]}
    rec0 = {"schema": "streamrl.policy/1", "type": "recurrent", "vocab_size": 5, "hidden_dim": 3,
            "input_embedding": [0.0] * 15, "recurrence": [0.0] * 9, "output": [0.0] * 15}
    rnd = r.random_recurrent_policy(9, 5, 0.8, 123)
    out["logprobs"] = dict(source="rl_math.cpp:128-142 policy_logprobs", cases=[
        dict(policy=hand, prompt="p", tokens=[1, 1], out=r.policy_logprobs(hand, "p", [1, 1]).tolist()),
        dict(policy=rec0, prompt="p", tokens=[0, 4, 2], out=r.policy_logprobs(rec0, "p", [0, 4, 2]).tolist()),
        dict(policy=rnd, prompt="p", tokens=[0, 3, 8, 1, 8, 8, 2],
             out=r.policy_logprobs(rnd, "p", [0, 3, 8, 1, 8, 8, 2]).tolist()),
        dict(policy=v0, prompt="demo", tokens=[0, 3, 3, 1, 5],
             out=r.policy_logprobs(v0, "demo", [0, 3, 3, 1, 5]).tolist())])

    # truncated IS / ESS (test_rl_math.cpp:168-198)
    import math
    out["is_ess"] = dict(source="rl_math.cpp:144-163", truncated=[
        [math.log(10.0), 0.0, 5.0, r.truncated_is_weight(math.log(10.0), 0.0, 5.0)],
        [-1.25, -1.25, 7.0, r.truncated_is_weight(-1.25, -1.25, 7.0)],
        [math.log(2.0), 0.0, 5.0, r.truncated_is_weight(math.log(2.0), 0.0, 5.0)],
        [-3.5, -1.0, 5.0, r.truncated_is_weight(-3.5, -1.0, 5.0)]],
        ess=[[w, r.ess(w)] for w in ([1, 1, 1, 1], [1, 0, 0, 0], [2, 1, 1], [0, 3, 3],
                                     [0.1, 2.5, 1e-3, 7.0])])

    # is_reinforce_gradient on random tabular instances (test_rl_math.cpp:245-287)
    grads = []
    keys = [["p", []], ["p", [0]], ["p", [1]], ["p", [2]]]
    for inst, (V, order, seed) in enumerate([(3, 1, 5), (4, 0, 9), (2, 1, 13), (3, 1, 21)]):
        pol = r.random_tabular_policy(V, order, keys[: 1 + (V if order else 0)][:4], 0.7, seed)
        _, trajs = r.mixed_policy_sample([pol], 0, 1, False, "p", 6, 5, 100 + seed)
        import random
        rng = random.Random(seed)
        for t in trajs:
            t["reward"] = rng.random()
            # perturb behaviour log-probs so the IS weights are non-trivial
            t["behavior_logprobs"] = [v - 0.3 * rng.random() for v in t["behavior_logprobs"]]
        for gran in (0, 1):
            for use_is in (0, 1):
                g = r.is_reinforce_gradient(pol, trajs, 5.0, use_is, gran)
                grads.append(dict(policy=pol, trajectories=trajs, granularity=gran, use_is=use_is,
                                  clamp=5.0, grad=g))
    out["gradients"] = dict(source="rl_math.cpp:211-276", cases=grads,
                            baseline_example=r.fit_baseline(grads[0]["trajectories"]))

    # lag structure from the reference simulator (sim.cpp:63-110, pipeline_toy.json)
    toy = json.loads((ASSETS / "configs/pipeline_toy.json").read_text())
    trace = r.run_pipeline(toy)
    big = dict(toy, gen_batch=4, n_inference_units=2, train_batch=3, train_ticks_per_step=3,
               total_optimizer_steps=20, lengths={"kind": "uniform", "max_len": 9}, seed=3,
               drift_magnitude=0.05, queue_capacity=64)
    trace2 = r.run_pipeline(big)
    out["lag"] = dict(source="sim.cpp:63-110 make_step_record/fill_sample_lags",
                      traces=[dict(config=toy, steps=trace["steps"], sequences=trace["sequences"]),
                              dict(config=big, steps=trace2["steps"], sequences=trace2["sequences"])])

    out["protocol"] = dict(source="engine.cpp:257-291",
                           crc32=[["123456789", r.crc32(b"123456789")], ["", r.crc32(b"")],
                                  ["streamrl", r.crc32(b"streamrl")]],
                           group_ids=[[m, r.process_group_id(m)] for m in
                                      (["http://a:1"], ["http://b:2", "http://a:1"],
                                       ["http://a:1", "http://b:2"])])
    path = Path(__file__).with_name("reference_vectors.json")
    path.write_text(json.dumps(out))
    print("wrote", path, path.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
