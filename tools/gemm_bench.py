#!/usr/bin/env python
"""Time the tcgen05 GEMM (srl_kernel_gemm_bf16, fp32 store epilogue) at the
decoder's shapes against torch.matmul (cuBLAS) on the same operands.

  python tools/gemm_bench.py [--shapes qwen2.5-0.5b] [--M 64,650,4096,16384]
"""
import argparse
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2509_19128_b200 import _lib  # noqa: E402
from paper_2509_19128_b200.policy import PRESETS  # noqa: E402


GRAPH = False


def time_fn(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    if GRAPH:  # GPU-only time: the calls replayed from a captured graph
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(iters):
                    fn()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / iters
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="qwen2.5-0.5b")
    ap.add_argument("--M", default="64,650,4096,16384")
    ap.add_argument("--kind", type=int, default=0, help="epilogue: 0 fp32 store, 3 bf16 store")
    ap.add_argument("--graph", action="store_true", help="time graph replays (no host launch cost)")
    a = ap.parse_args()
    global GRAPH
    GRAPH = a.graph
    cfg = PRESETS[a.shapes]
    H, I, V = cfg.hidden, cfg.intermediate, cfg.vocab_size
    qkv = (cfg.q_heads + 2 * cfg.kv_heads) * cfg.head_dim
    shapes = {"qkv": (qkv, H), "o": (H, cfg.q_heads * cfg.head_dim), "gate_up": (2 * I, H),
              "down": (H, I)}
    for M in [int(m) for m in a.M.split(",")]:
        for name, (N, K) in shapes.items():
            w = torch.randn(N, K, device="cuda").bfloat16()
            x = torch.randn(M, K, device="cuda").bfloat16()
            out = torch.empty(M, N, device="cuda", dtype=torch.float32 if a.kind == 0 else torch.bfloat16)

            def ours():
                _lib.call("srl_kernel_gemm_bf16", w.data_ptr(), x.data_ptr(), M, N, K, 0, a.kind, None, None,
                          0, 0.0, 0.0, out.data_ptr(), None, None, None, None,
                          torch.cuda.current_stream().cuda_stream)

            t = time_fn(ours)
            tb = time_fn(lambda: torch.matmul(x, w.T, out=None))
            ref = (x.float() @ w.float().T)
            err = (out.float() - ref).abs().max().item() / (ref.abs().max().item() + 1e-6)
            fl = 2.0 * M * N * K
            by = 2.0 * (N * K + M * K) + 4.0 * M * N
            print(f"M={M:6d} {name:8s} N={N:6d} K={K:5d}  ours {t * 1e3:8.1f} us {fl / t / 1e9:7.1f} TF/s "
                  f"{by / t / 1e6:7.0f} GB/s | cublas {tb * 1e3:8.1f} us {fl / tb / 1e9:7.1f} TF/s | err {err:.1e}",
                  flush=True)


if __name__ == "__main__":
    main()
