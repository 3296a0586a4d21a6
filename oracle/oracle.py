"""ctypes wrappers for the parity checkers.  TEST INFRASTRUCTURE ONLY.

* ``Oracle``  -- oracle/_build/liboracle.so, the C restatement
  (oracle/streamrl_oracle.c) of the reference algorithms.
* ``Ref``     -- oracle/_ref/libstreamrl_ref.so, the unmodified reference
  sources compiled by oracle/Makefile plus oracle/ref_shim.cpp.

Policies cross this boundary as ``streamrl.policy/1`` documents (dicts), the
reference's own format (src/policy.cpp:136-192).  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline leg import this module.
"""
from __future__ import annotations

import ctypes as C
import json
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "liboracle.so"
REF_SO = HERE / "_ref" / "libstreamrl_ref.so"
REF_SRC = Path("/root/reference/proj")

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
vp = C.c_void_p


def build(ref: bool = True) -> None:
    """Compile the checkers (the reference only where its sources exist)."""
    targets = ["oracle"] + (["ref"] if ref and REF_SRC.exists() else [])
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


class OrcPolicy(C.Structure):
    _fields_ = [("type", C.c_int), ("vocab", C.c_int), ("hidden", C.c_int),
                ("emb", vp), ("rec", vp), ("out", vp), ("order", C.c_int), ("n_rows", C.c_int),
                ("row_prompt", vp), ("row_ctx_len", vp), ("row_ctx", vp), ("row_logits", vp),
                ("default_logits", vp)]


class _PolicyPack:
    """Keeps the numpy buffers alive behind an OrcPolicy struct."""

    def __init__(self, doc: dict, prompts: dict):
        self.keep = []
        p = OrcPolicy()
        if doc["type"] == "recurrent":
            V, D = int(doc["vocab_size"]), int(doc["hidden_dim"])
            e, r, o = (np.ascontiguousarray(doc[k], dtype=np.float64)
                       for k in ("input_embedding", "recurrence", "output"))
            self.keep += [e, r, o]
            p.type, p.vocab, p.hidden = 1, V, D
            p.emb, p.rec, p.out = e.ctypes.data, r.ctypes.data, o.ctypes.data
        elif doc["type"] == "tabular":
            V, order = int(doc["vocab_size"]), int(doc["context_order"])
            rows = doc.get("rows", [])
            rp = np.array([prompts.setdefault(r["prompt_id"], len(prompts)) for r in rows] or [0],
                          dtype=np.int32)
            rl = np.array([len(r["context"]) for r in rows] or [0], dtype=np.int32)
            rc = np.zeros((max(len(rows), 1), max(order, 1)), dtype=np.int32)
            for i, r in enumerate(rows):
                rc[i, :len(r["context"])] = r["context"]
            lg = np.array([r["logits"] for r in rows] or [[0.0] * V], dtype=np.float64)
            self.keep += [rp, rl, rc, lg]
            p.type, p.vocab, p.order, p.n_rows = 0, V, order, len(rows)
            p.row_prompt, p.row_ctx_len = rp.ctypes.data, rl.ctypes.data
            p.row_ctx, p.row_logits = rc.ctypes.data, lg.ctypes.data
            d = doc.get("default_logits") or []
            if len(d):
                da = np.array(d, dtype=np.float64)
                self.keep.append(da)
                p.default_logits = da.ctypes.data
        else:
            raise ValueError("oracle policies are tabular or recurrent")
        self.struct = p


class Oracle:
    def __init__(self):
        if not ORACLE_SO.exists():
            build(ref=False)
        L = C.CDLL(str(ORACLE_SO))
        L.orc_splitmix_next.restype = u64
        L.orc_splitmix_next.argtypes = [C.POINTER(u64)]
        L.orc_next_double.restype = f64
        L.orc_next_double.argtypes = [C.POINTER(u64)]
        L.orc_next_gaussian.restype = f64
        L.orc_next_gaussian.argtypes = [C.POINTER(u64)]
        L.orc_derive_stream.restype = u64
        L.orc_derive_stream.argtypes = [u64, u64]
        L.orc_sample_from_logits.restype = C.c_int
        L.orc_sample_from_logits.argtypes = [vp, C.c_int, f64, C.POINTER(f64), vp]
        L.orc_argmax.restype = C.c_int
        L.orc_argmax.argtypes = [vp, C.c_int]
        L.orc_log_softmax.argtypes = [vp, C.c_int, vp]
        L.orc_mixed_sample.argtypes = [C.POINTER(OrcPolicy), C.c_int, vp, C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.c_int, u64, C.c_int, vp, vp, vp, vp]
        L.orc_policy_logprobs.argtypes = [C.POINTER(OrcPolicy), C.c_int, vp, C.c_int, vp]
        L.orc_engine_lockstep.argtypes = [C.POINTER(OrcPolicy), C.c_int, vp, C.c_int, C.c_int,
                                          C.c_int, vp, vp, vp, vp, vp, C.c_int, C.c_int, vp, vp,
                                          vp, vp, vp]
        L.orc_truncated_is_weight.argtypes = [f64, f64, f64, C.POINTER(f64)]
        L.orc_ess.argtypes = [vp, C.c_int, C.POINTER(f64)]
        L.orc_fit_baseline.argtypes = [C.c_int, vp, vp, vp, C.c_int, C.c_int, vp, vp]
        L.orc_reinforce_gradient_tab.argtypes = [C.POINTER(OrcPolicy), C.c_int, vp, vp, vp, vp,
                                                 vp, vp, vp, vp, C.c_int, f64, C.c_int, C.c_int,
                                                 vp, vp]
        L.orc_lag_stats.argtypes = [C.c_int, C.c_int, vp, vp, vp, i64, f64, vp, C.c_int, vp, vp,
                                    vp, vp, vp, vp, vp, vp]
        L.orc_crc32.restype = C.c_uint32
        L.orc_crc32.argtypes = [C.c_char_p, C.c_size_t]
        L.orc_schedule_make.argtypes = [C.c_int, C.c_int, vp]
        L.orc_pipeline_max_lag_steps.restype = i64
        L.orc_pipeline_max_lag_steps.argtypes = [f64, f64, f64, f64, f64]
        self.L = L

    # ---------------------------------------------------------------- rng
    def splitmix(self, seed: int, n: int) -> list[int]:
        s = u64(seed)
        return [self.L.orc_splitmix_next(C.byref(s)) for _ in range(n)]

    def uniforms(self, seed: int, n: int) -> list[float]:
        s = u64(seed)
        return [self.L.orc_next_double(C.byref(s)) for _ in range(n)]

    def gaussians(self, seed: int, n: int) -> list[float]:
        s = u64(seed)
        return [self.L.orc_next_gaussian(C.byref(s)) for _ in range(n)]

    def derive_stream(self, seed: int, index: int) -> int:
        return self.L.orc_derive_stream(seed, index)

    def sample_from_logits(self, logits, u: float):
        x = np.ascontiguousarray(logits, dtype=np.float64)
        scratch = np.empty(2 * len(x))
        lp = f64()
        tok = self.L.orc_sample_from_logits(x.ctypes.data, len(x), u, C.byref(lp), scratch.ctypes.data)
        return tok, lp.value

    def argmax(self, logits) -> int:
        x = np.ascontiguousarray(logits, dtype=np.float64)
        return self.L.orc_argmax(x.ctypes.data, len(x))

    def log_softmax(self, logits):
        x = np.ascontiguousarray(logits, dtype=np.float64)
        out = np.empty_like(x)
        self.L.orc_log_softmax(x.ctypes.data, len(x), out.ctypes.data)
        return out

    # ---------------------------------------------------------- policies
    @staticmethod
    def _pack(docs, prompts):
        packs = [_PolicyPack(d, prompts) for d in docs]
        arr = (OrcPolicy * len(packs))(*[p.struct for p in packs])
        return packs, arr

    def mixed_sample(self, ckpt_docs, switch_points, recompute, prompt_id, count, max_len, seed,
                     terminator=-1):
        prompts = {prompt_id: 0}
        packs, arr = self._pack(ckpt_docs, prompts)
        sw = np.array(switch_points or [0], dtype=np.int32)
        tok = np.zeros((count, max_len), dtype=np.int32)
        lp = np.zeros((count, max_len), dtype=np.float64)
        ver = np.zeros((count, max_len), dtype=np.int32)
        ln = np.zeros(count, dtype=np.int32)
        st = self.L.orc_mixed_sample(arr, len(packs), sw.ctypes.data, len(switch_points or []),
                                     int(recompute), prompts[prompt_id], count, max_len, seed,
                                     terminator, tok.ctypes.data, lp.ctypes.data, ver.ctypes.data,
                                     ln.ctypes.data)
        if st:
            raise ValueError("mixed_sample: invalid input")
        return [dict(tokens=tok[i, :ln[i]].tolist(), behavior_logprobs=lp[i, :ln[i]].tolist(),
                     behavior_versions=ver[i, :ln[i]].tolist()) for i in range(count)]

    def policy_logprobs(self, doc, prompt_id, tokens):
        prompts = {prompt_id: 0}
        pack = _PolicyPack(doc, prompts)
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        out = np.zeros(len(t))
        st = self.L.orc_policy_logprobs(C.byref(pack.struct), prompts[prompt_id], t.ctypes.data,
                                        len(t), out.ctypes.data)
        if st:
            raise ValueError("token out of vocab range")
        return out

    def engine_lockstep(self, ckpt_docs, update_after, recompute, streams, total_rounds,
                        max_events=None):
        """streams: list of dict(prompt_id, seed, max_tokens, terminator, open_after)."""
        prompts: dict = {}
        for s in streams:
            prompts.setdefault(s["prompt_id"], len(prompts))
        packs, arr = self._pack(ckpt_docs, prompts)
        n = len(streams)
        me = max_events or max(s["max_tokens"] for s in streams)
        pr = np.array([prompts[s["prompt_id"]] for s in streams], dtype=np.int32)
        seeds = np.array([s["seed"] for s in streams], dtype=np.uint64)
        mt = np.array([s["max_tokens"] for s in streams], dtype=np.int32)
        te = np.array([s.get("terminator", -1) for s in streams], dtype=np.int32)
        oa = np.array([s.get("open_after", 0) for s in streams], dtype=np.int32)
        ua = np.array(update_after or [0], dtype=np.int32)
        tok = np.zeros((n, me), dtype=np.int32)
        lp = np.zeros((n, me))
        ver = np.zeros((n, me), dtype=np.int32)
        cnt = np.zeros(n, dtype=np.int32)
        fin = np.zeros(n, dtype=np.int32)
        st = self.L.orc_engine_lockstep(arr, len(packs), ua.ctypes.data, len(update_after or []),
                                        int(recompute), n, pr.ctypes.data, seeds.ctypes.data,
                                        mt.ctypes.data, te.ctypes.data, oa.ctypes.data,
                                        total_rounds, me, tok.ctypes.data, lp.ctypes.data,
                                        ver.ctypes.data, cnt.ctypes.data, fin.ctypes.data)
        if st:
            raise ValueError("engine_lockstep: invalid input")
        names = {0: "running", 1: "length", 2: "terminator"}
        return [dict(tokens=tok[i, :cnt[i]].tolist(), logprobs=lp[i, :cnt[i]].tolist(),
                     versions=ver[i, :cnt[i]].tolist(), finish=names[int(fin[i])])
                for i in range(n)]

    # ------------------------------------------------------ trainer math
    def truncated_is_weight(self, pi, mu, c):
        out = f64()
        if self.L.orc_truncated_is_weight(pi, mu, c, C.byref(out)):
            raise ValueError("truncated_is_weight: invalid input")
        return out.value

    def ess(self, w):
        a = np.ascontiguousarray(w, dtype=np.float64)
        out = f64()
        st = self.L.orc_ess(a.ctypes.data, len(a), C.byref(out))
        if st == 2:
            raise ZeroDivisionError("ess undefined: all weights are zero")
        if st:
            raise ValueError("ess: invalid weights")
        return out.value

    def reinforce_gradient_tab(self, doc, trajs, clamp=5.0, use_is=True, granularity=0,
                               baseline=None):
        """trajs: list of dict(prompt_id, tokens, behavior_logprobs, reward).  Returns
        (dense grad [(rows+1) x V], touched, baseline table dict)."""
        prompts: dict = {}
        for r in doc.get("rows", []):
            prompts.setdefault(r["prompt_id"], len(prompts))
        for t in trajs:
            prompts.setdefault(t["prompt_id"], len(prompts))
        pack = _PolicyPack(doc, prompts)
        n = len(trajs)
        pr = np.array([prompts[t["prompt_id"]] for t in trajs], dtype=np.int32)
        ln = np.array([len(t["tokens"]) for t in trajs], dtype=np.int32)
        off = np.concatenate([[0], np.cumsum(ln)[:-1]]).astype(np.int64)
        tok = np.concatenate([np.asarray(t["tokens"], dtype=np.int32) for t in trajs])
        blp = np.concatenate([np.asarray(t["behavior_logprobs"], dtype=np.float64) for t in trajs])
        rew = np.array([t["reward"] for t in trajs], dtype=np.float64)
        maxlen = int(ln.max())
        table = np.zeros((len(prompts), maxlen))
        count = np.zeros((len(prompts), maxlen), dtype=np.int64)
        if baseline is None:
            self.L.orc_fit_baseline(n, pr.ctypes.data, ln.ctypes.data, rew.ctypes.data,
                                    len(prompts), maxlen, table.ctypes.data, count.ctypes.data)
        else:
            for (pid, t), v in baseline.items():
                if pid in prompts and t < maxlen:
                    table[prompts[pid], t] = v
                    count[prompts[pid], t] = 1
        V = int(doc["vocab_size"])
        nrows = len(doc.get("rows", []))
        grad = np.zeros((nrows + 1, V))
        touched = np.zeros(nrows + 1, dtype=np.int32)
        st = self.L.orc_reinforce_gradient_tab(
            C.byref(pack.struct), n, pr.ctypes.data, ln.ctypes.data, off.ctypes.data,
            tok.ctypes.data, blp.ctypes.data, rew.ctypes.data, table.ctypes.data,
            count.ctypes.data, maxlen, clamp, int(use_is), granularity, grad.ctypes.data,
            touched.ctypes.data)
        if st:
            raise ValueError("reinforce_gradient: invalid input")
        inv = {v: k for k, v in prompts.items()}
        base = {(inv[p], t): table[p, t] for p in range(len(prompts)) for t in range(maxlen)
                if count[p, t]}
        return grad, touched, base

    def lag_stats(self, version_before, token_versions, consumed_at_emit=None,
                  consumed_before=0, drift_magnitude=0.0, hist_cap=4096):
        lens = np.array([len(v) for v in token_versions], dtype=np.int32)
        vers = np.concatenate([np.asarray(v, dtype=np.int32) for v in token_versions]) \
            if len(token_versions) else np.zeros(1, dtype=np.int32)
        cae = None
        if consumed_at_emit is not None:
            cae = np.concatenate([np.asarray(v, dtype=np.int64) for v in consumed_at_emit])
        hist = np.zeros(hist_cap, dtype=np.int64)
        sums = np.zeros(max(len(lens), 1), dtype=np.int64)
        tokens, mx, smax = i64(), i64(), i64()
        mean, ess, smean = f64(), f64(), f64()
        warm = C.c_int()
        st = self.L.orc_lag_stats(version_before, len(lens), lens.ctypes.data, vers.ctypes.data,
                                  None if cae is None else cae.ctypes.data, consumed_before,
                                  drift_magnitude, hist.ctypes.data, hist_cap, C.byref(tokens),
                                  C.byref(mx), C.byref(mean), sums.ctypes.data, C.byref(ess),
                                  C.byref(smax), C.byref(smean), C.byref(warm))
        if st:
            raise ValueError("lag_stats: lag out of range")
        return dict(histogram={i: int(c) for i, c in enumerate(hist) if c},
                    tokens=tokens.value, max_lag_steps=mx.value, mean_lag_steps=mean.value,
                    sequence_lag_sums=sums[:len(lens)].tolist(), ess=ess.value,
                    max_lag_samples=smax.value, mean_lag_samples=smean.value,
                    post_warmup=bool(warm.value))

    def crc32(self, data: bytes) -> int:
        return self.L.orc_crc32(data, len(data))

    def schedule(self, max_len, max_lag):
        buf = np.zeros(max(max_lag, 1), dtype=np.int32)
        n = self.L.orc_schedule_make(max_len, max_lag, buf.ctypes.data)
        if n < 0:
            raise ValueError("schedule: invalid input")
        return buf[:n].tolist()

    def pipeline_max_lag_steps(self, H, I, L, mean_len, B):
        return self.L.orc_pipeline_max_lag_steps(H, I, L, mean_len, B)


def random_recurrent_policy(o: Oracle, V, D, scale, seed) -> dict:
    """random_recurrent_policy (rl_math.cpp:392-407): E, R, O filled in order."""
    g = o.gaussians(seed, V * D + D * D + D * V)
    e = [scale * x for x in g[:V * D]]
    r = [scale * x for x in g[V * D:V * D + D * D]]
    out = [scale * x for x in g[V * D + D * D:]]
    return {"schema": "streamrl.policy/1", "type": "recurrent", "vocab_size": V, "hidden_dim": D,
            "input_embedding": e, "recurrence": r, "output": out}


def drift_checkpoints(o: Oracle, doc: dict, count: int, magnitude: float, seed: int) -> list:
    """drift_checkpoints (rl_math.cpp:409-433), recurrent or tabular."""
    out = [doc]
    for i in range(1, count):
        prev = out[-1]
        s = o.derive_stream(seed, i)
        if prev["type"] == "recurrent":
            n = len(prev["input_embedding"]) + len(prev["recurrence"]) + len(prev["output"])
            g = o.gaussians(s, n)
            a, b = len(prev["input_embedding"]), len(prev["recurrence"])
            nxt = dict(prev)
            nxt["input_embedding"] = [v + magnitude * x for v, x in zip(prev["input_embedding"], g[:a])]
            nxt["recurrence"] = [v + magnitude * x for v, x in zip(prev["recurrence"], g[a:a + b])]
            nxt["output"] = [v + magnitude * x for v, x in zip(prev["output"], g[a + b:])]
        else:
            n = len(prev.get("default_logits") or []) + sum(len(r["logits"]) for r in prev["rows"])
            g = iter(o.gaussians(s, n))
            nxt = dict(prev)
            nxt["default_logits"] = [v + magnitude * next(g) for v in prev.get("default_logits") or []]
            nxt["rows"] = [dict(r, logits=[v + magnitude * next(g) for v in r["logits"]])
                           for r in prev["rows"]]
        out.append(nxt)
    return out


class Ref:
    """The reference itself (oracle/_ref), for golden-vector generation."""

    def __init__(self):
        if not REF_SO.exists():
            build(ref=True)
        L = C.CDLL(str(REF_SO))
        for name in ("ref_random_recurrent_policy", "ref_random_tabular_policy",
                     "ref_drift_checkpoints", "ref_mixed_policy_sample", "ref_fit_baseline",
                     "ref_is_reinforce_gradient", "ref_engine_lockstep", "ref_run_pipeline",
                     "ref_run_conventional", "ref_process_group_id", "ref_kl_per_position",
                     "ref_search_configs", "ref_policy_wire"):
            getattr(L, name).restype = vp
        L.ref_free.argtypes = [vp]
        L.ref_random_recurrent_policy.argtypes = [C.c_int, C.c_int, f64, u64]
        L.ref_random_tabular_policy.argtypes = [C.c_int, C.c_int, C.c_char_p, f64, u64]
        L.ref_drift_checkpoints.argtypes = [C.c_char_p, C.c_int, f64, u64]
        L.ref_mixed_policy_sample.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_char_p,
                                              C.c_int, C.c_int, u64, C.c_int]
        L.ref_policy_logprobs.argtypes = [C.c_char_p, C.c_char_p, vp, C.c_int, vp]
        L.ref_truncated_is_weight.argtypes = [f64, f64, f64, C.POINTER(f64)]
        L.ref_ess.argtypes = [vp, C.c_int, C.POINTER(f64)]
        L.ref_fit_baseline.argtypes = [C.c_char_p]
        L.ref_is_reinforce_gradient.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, f64, C.c_int,
                                                C.c_int]
        L.ref_engine_lockstep.argtypes = [C.c_char_p]
        L.ref_engine_throughput.argtypes = [C.c_char_p, C.c_int, C.c_int, u64, C.POINTER(i64),
                                            C.POINTER(f64)]
        L.ref_engine_throughput_parallel.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, u64,
                                                     C.POINTER(i64), C.POINTER(f64)]
        L.ref_update_pause.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_int, vp,
                                       C.POINTER(i64)]
        L.ref_run_pipeline.argtypes = [C.c_char_p]
        L.ref_run_conventional.argtypes = [C.c_char_p]
        L.ref_pipeline_max_lag_steps.restype = C.c_longlong
        L.ref_pipeline_max_lag_steps.argtypes = [C.c_longlong, C.c_longlong, f64, f64, C.c_longlong]
        L.ref_crc32.restype = C.c_uint
        L.ref_crc32.argtypes = [C.c_char_p, C.c_size_t]
        L.ref_process_group_id.argtypes = [C.c_char_p]
        L.ref_kl_per_position.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_char_p,
                                          C.c_char_p, C.c_char_p]
        self.L = L

    def _s(self, ptr, parse=True):
        try:
            text = C.string_at(ptr).decode()
        finally:
            self.L.ref_free(ptr)
        if not parse:
            return text
        out = json.loads(text)
        if isinstance(out, dict) and "error" in out and len(out) == 1:
            raise ValueError(out["error"])
        return out

    def random_recurrent_policy(self, V, D, scale, seed):
        return self._s(self.L.ref_random_recurrent_policy(V, D, scale, seed))

    def random_tabular_policy(self, V, order, keys, scale, seed):
        return self._s(self.L.ref_random_tabular_policy(V, order, json.dumps(keys).encode(), scale,
                                                        seed))

    def drift_checkpoints(self, doc, count, magnitude, seed):
        return self._s(self.L.ref_drift_checkpoints(json.dumps(doc).encode(), count, magnitude, seed))

    def mixed_policy_sample(self, docs, schedule_max_len, max_lag, recompute, prompt_id, count,
                            max_len, seed, terminator=-1):
        out = self._s(self.L.ref_mixed_policy_sample(json.dumps(docs).encode(), schedule_max_len,
                                                     max_lag, int(recompute), prompt_id.encode(),
                                                     count, max_len, seed, terminator))
        trajs = [json.loads(line) for line in out["jsonl"].splitlines() if line]
        return out["switch_points"], trajs

    def policy_logprobs(self, doc, prompt_id, tokens):
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        out = np.zeros(len(t))
        if self.L.ref_policy_logprobs(json.dumps(doc).encode(), prompt_id.encode(), t.ctypes.data,
                                      len(t), out.ctypes.data):
            raise ValueError("policy_logprobs failed")
        return out

    def truncated_is_weight(self, pi, mu, c):
        out = f64()
        if self.L.ref_truncated_is_weight(pi, mu, c, C.byref(out)):
            raise ValueError("truncated_is_weight")
        return out.value

    def ess(self, w):
        a = np.ascontiguousarray(w, dtype=np.float64)
        out = f64()
        st = self.L.ref_ess(a.ctypes.data, len(a), C.byref(out))
        if st == 2:
            raise ZeroDivisionError("ess undefined")
        if st:
            raise ValueError("ess")
        return out.value

    def is_reinforce_gradient(self, doc, trajs, clamp=5.0, use_is=True, granularity=0,
                              baseline=None):
        jsonl = "".join(json.dumps(t) + "\n" for t in trajs)
        b = b"" if baseline is None else json.dumps(baseline).encode()
        return self._s(self.L.ref_is_reinforce_gradient(json.dumps(doc).encode(), jsonl.encode(), b,
                                                        clamp, int(use_is), granularity))

    def fit_baseline(self, trajs):
        jsonl = "".join(json.dumps(t) + "\n" for t in trajs)
        return self._s(self.L.ref_fit_baseline(jsonl.encode()))

    def engine_lockstep(self, script):
        return self._s(self.L.ref_engine_lockstep(json.dumps(script).encode()))

    def engine_throughput(self, doc, n_streams, max_tokens, seed=1):
        tok, sec = i64(), f64()
        if self.L.ref_engine_throughput(json.dumps(doc).encode(), n_streams, max_tokens, seed,
                                        C.byref(tok), C.byref(sec)):
            raise RuntimeError("engine_throughput failed")
        return tok.value, sec.value

    def engine_throughput_parallel(self, doc, n_threads, n_streams, max_tokens, seed=1):
        """n_threads independent reference Engines at once (one per core):
        (aggregate tokens, wall seconds of the slowest)."""
        tok, sec = i64(), f64()
        if self.L.ref_engine_throughput_parallel(json.dumps(doc).encode(), n_threads, n_streams,
                                                 max_tokens, seed, C.byref(tok), C.byref(sec)):
            raise RuntimeError("engine_throughput_parallel failed")
        return tok.value, sec.value

    def update_pause(self, doc, new_doc, n_streams, rounds, recompute=False):
        """The reference's weight-update pause: {serialize, crc32, parse, apply}
        milliseconds and the JSON payload bytes."""
        out = np.zeros(4)
        nb = i64()
        st = self.L.ref_update_pause(json.dumps(doc).encode(), json.dumps(new_doc).encode(),
                                     n_streams, rounds, int(recompute), out.ctypes.data, C.byref(nb))
        if st:
            raise RuntimeError(f"update_pause failed ({st})")
        return dict(zip(("serialize_ms", "crc32_ms", "parse_ms", "apply_ms"), out.tolist()),
                    payload_bytes=nb.value)

    def pipeline_max_lag_steps(self, H, I, L, mean_len, B):
        v = self.L.ref_pipeline_max_lag_steps(H, I, L, mean_len, B)
        if v < 0:
            raise ValueError("pipeline_max_lag_steps: invalid arguments")
        return v

    def run_pipeline(self, cfg):
        return self._s(self.L.ref_run_pipeline(json.dumps(cfg).encode()))

    def run_conventional(self, cfg):
        return self._s(self.L.ref_run_conventional(json.dumps(cfg).encode()))

    def crc32(self, data: bytes) -> int:
        return self.L.ref_crc32(data, len(data))

    def process_group_id(self, members):
        return self._s(self.L.ref_process_group_id(json.dumps(members).encode()), parse=False)

    def policy_wire(self, doc: dict):
        """The reference client's checksummed bytes of a policy document and their CRC-32."""
        self.L.ref_policy_wire.argtypes = [C.c_char_p]
        return self._s(self.L.ref_policy_wire(json.dumps(doc).encode()))

    def search_configs(self, spec: dict):
        """throughput::search_configs (throughput.cpp:288-330) of the reference."""
        self.L.ref_search_configs.argtypes = [C.c_char_p]
        return self._s(self.L.ref_search_configs(json.dumps(spec).encode()))

    def kl_per_position(self, behavior_docs, schedule_max_len, max_lag, recompute, target_doc,
                        prompt_id, prefixes):
        jsonl = "".join(json.dumps(t) + "\n" for t in prefixes)
        return self._s(self.L.ref_kl_per_position(json.dumps(behavior_docs).encode(),
                                                  schedule_max_len, max_lag, int(recompute),
                                                  json.dumps(target_doc).encode(),
                                                  prompt_id.encode(), jsonl.encode()))
