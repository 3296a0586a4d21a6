#!/usr/bin/env python
"""Per-CTA phase timeline of one persistent-GEMM launch (gemm_big.cu stamps:
0 start, 1 setup, 2 first TMA, 3 first k-block landed, 4 last MMA commit,
5 first accumulator ready, 6 epilogue done, 7 exit), times in us from the
earliest CTA start.  SRL_GEMM_BIG=1 forces the persistent kernel.

  SRL_GEMM_BIG=1 python tools/gemm_timeline.py --M 576 --N 896 --K 896 [--kind 3]
"""
import argparse
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2509_19128_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=576)
ap.add_argument("--N", type=int, default=896)
ap.add_argument("--K", type=int, default=896)
ap.add_argument("--kind", type=int, default=3)
a = ap.parse_args()
w = torch.randn(a.N, a.K, device="cuda").bfloat16()
x = torch.randn(a.M, a.K, device="cuda").bfloat16()
out = torch.empty(a.M, a.N, device="cuda", dtype=torch.float32 if a.kind == 0 else torch.bfloat16)
st = torch.zeros(1024 * 8, dtype=torch.int64, device="cuda")


def call():
    _lib.call("srl_kernel_gemm_bf16", w.data_ptr(), x.data_ptr(), a.M, a.N, a.K, 0, a.kind, None, None, 0,
              0.0, 0.0, out.data_ptr(), None, None, None, None, None)


for _ in range(5):
    call()
torch.cuda.synchronize()
lib = _lib.lib()
lib.srl_debug_gemm_stamps.argtypes = [ctypes.c_void_p]
lib.srl_debug_gemm_stamps(st.data_ptr())
call()
torch.cuda.synchronize()
lib.srl_debug_gemm_stamps(None)
s = st.view(1024, 8).cpu().numpy().astype(np.float64)
s = s[s[:, 0] > 0]
t0 = s[:, 0].min()
rel = (s - t0) / 1e3
names = ["start", "setup", "tma0", "landed0", "mma_last", "acc0", "epi_done", "exit"]
print(f"M={a.M} N={a.N} K={a.K} kind={a.kind}: {len(s)} CTAs, span {rel[:, 7].max():.2f} us")
for i, n in enumerate(names):
    col = rel[:, i][s[:, i] > 0]
    if len(col):
        print(f"  {n:9s} min {col.min():7.2f}  med {np.median(col):7.2f}  max {col.max():7.2f}")
