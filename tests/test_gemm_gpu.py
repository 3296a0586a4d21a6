"""tcgen05 GEMM kernel vs a torch fp32 reference (floating-point kernel: the
one place a torch reference is used).  Tolerance: fp32 accumulation of bf16
products, rel 2e-3 of the output scale."""
import pytest
import torch

from paper_2509_19128_b200 import _lib

pytestmark = pytest.mark.gpu

EPI_F32, EPI_RESID, EPI_SWIGLU, EPI_BF16 = 0, 1, 2, 3


def ptr(t):
    return None if t is None else t.data_ptr()


def run(w, x, kind, splits=0, bias=None, ssq=None, parts=0, inv_dim=0.0, eps=0.0, out=None,
        resid=None, gain=None, xg=None, ssq_out=None):
    M, K = x.shape
    N = w.shape[0]
    _lib.call("srl_kernel_gemm_bf16", ptr(w), ptr(x), M, N, K, splits, kind, ptr(bias), ptr(ssq),
              parts, inv_dim, eps, ptr(out), ptr(resid), ptr(gain), ptr(xg), ptr(ssq_out), None)
    torch.cuda.synchronize()


def close(a, b, tol=2e-3):
    scale = b.abs().max().item() + 1e-6
    err = (a.float() - b.float()).abs().max().item()
    assert err <= tol * scale, f"max err {err} vs scale {scale}"


# the last four shapes fill the machine with tiles, so they run the persistent
# large-M kernel (gemm_big.cu, token tile 128 or 256; ragged M and N tails)
@pytest.mark.parametrize("M,N,K,splits", [(64, 256, 128, 1), (64, 1152, 896, 0), (64, 896, 4864, 0),
                                          (37, 384, 256, 1), (200, 512, 512, 1), (64, 300, 192, 2),
                                          (1, 128, 64, 1), (256, 1024, 896, 0),
                                          (2000, 1280, 896, 0), (4096, 9728, 896, 0),
                                          (3001, 9700, 128, 0), (16384, 896, 4864, 0)])
def test_gemm_store_f32(cuda, M, N, K, splits):
    g = torch.Generator(device=cuda).manual_seed(M * 7 + N)
    w = torch.randn(N, K, device=cuda, generator=g).bfloat16()
    x = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    bias = torch.randn(N, device=cuda, generator=g).bfloat16()
    out = torch.full((M, N), float("nan"), device=cuda)
    run(w, x, EPI_F32, splits=splits, bias=bias, out=out)
    ref = x.float() @ w.float().T + bias.float()
    close(out, ref)


def test_gemm_deterministic_splitk(cuda):
    M, N, K = 64, 1152, 896
    w = torch.randn(N, K, device=cuda).bfloat16()
    x = torch.randn(M, K, device=cuda).bfloat16()
    outs = []
    for _ in range(3):
        out = torch.empty(M, N, device=cuda)
        run(w, x, EPI_F32, splits=7, out=out)
        outs.append(out)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])


@pytest.mark.parametrize("M,N,K", [(64, 1024, 256), (4000, 9728, 896)])
def test_gemm_rmsnorm_scale_and_swiglu(cuda, M, N, K):
    w = torch.randn(N, K, device=cuda).bfloat16()
    x = torch.randn(M, K, device=cuda).bfloat16()
    parts = 2
    ssq = torch.rand(M, parts, device=cuda) * 50 + 1
    eps = 1e-6
    out = torch.empty(M, N // 2, device=cuda, dtype=torch.bfloat16)
    run(w, x, EPI_SWIGLU, splits=0, ssq=ssq, parts=parts, inv_dim=1.0 / K, eps=eps, out=out)
    rstd = torch.rsqrt(ssq.sum(1, keepdim=True) / K + eps)
    y = (x.float() @ w.float().T) * rstd
    y = y.view(M, N // 128, 2, 64)
    gte, up = y[:, :, 0, :].reshape(M, -1), y[:, :, 1, :].reshape(M, -1)
    ref = torch.nn.functional.silu(gte) * up
    close(out, ref, tol=1e-2)


@pytest.mark.parametrize("M", [64, 5000])
def test_gemm_residual_epilogue(cuda, M):
    N, K = 896, 896
    w = torch.randn(N, K, device=cuda).bfloat16()
    x = torch.randn(M, K, device=cuda).bfloat16()
    resid = torch.randn(M, N, device=cuda)
    resid0 = resid.clone()
    gain = (torch.rand(N, device=cuda) + 0.5).bfloat16()
    xg = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    ssq = torch.empty(M, 7, device=cuda)
    run(w, x, EPI_RESID, splits=0, resid=resid, gain=gain, xg=xg, ssq_out=ssq)
    ref = resid0 + x.float() @ w.float().T
    close(resid, ref)
    close(xg, ref * gain.float(), tol=1e-2)
    ref_ssq = (ref.view(M, 7, 128) ** 2).sum(-1)
    close(ssq, ref_ssq, tol=3e-3)


def run_mn(w, x, M, N, k_rows, x_kmajor, out, splits=0, accumulate=True, scale=1.0):
    _lib.call("srl_kernel_gemm_mn", ptr(w), ptr(x), M, N, k_rows, int(x_kmajor), splits, int(accumulate),
              scale, ptr(out), None)
    torch.cuda.synchronize()


# MN-major W operand (and X): the trainer's transpose-free weight / input
# gradients.  Ragged k_rows (TMA zero-fill past the last row), 128- and
# 256-token tiles, planned and forced ordered split-K.
@pytest.mark.parametrize("M,N,k_rows,splits", [(896, 4864, 300, 0), (896, 896, 20480, 0),
                                               (1152, 896, 5000, 3), (20480, 1152, 128, 0),
                                               (9728, 896, 1000, 0), (72, 200, 64, 1)])
def test_gemm_mn_major_accumulate(cuda, M, N, k_rows, splits):
    g = torch.Generator(device=cuda).manual_seed(M + 3 * N + k_rows)
    x = torch.randn(k_rows, M, device=cuda, generator=g).bfloat16()
    w = torch.randn(k_rows, N, device=cuda, generator=g).bfloat16()
    base = torch.randn(M, N, device=cuda, generator=g)
    out = base.clone()
    run_mn(w, x, M, N, k_rows, False, out, splits=splits, scale=0.5)
    ref = base + 0.5 * (x.float().T @ w.float())
    close(out, ref, tol=1e-4 * max(1.0, (k_rows / 64) ** 0.5))
    if splits != 1:  # ordered K slices: bit-identical across launches
        again = base.clone()
        run_mn(w, x, M, N, k_rows, False, again, splits=splits, scale=0.5)
        assert torch.equal(out, again)


@pytest.mark.parametrize("M,N,k_rows", [(300, 896, 4864), (20480, 896, 896), (64, 1152, 128)])
def test_gemm_mn_w_kmajor_x_store(cuda, M, N, k_rows):
    g = torch.Generator(device=cuda).manual_seed(M + N)
    x = torch.randn(M, k_rows, device=cuda, generator=g).bfloat16()
    w = torch.randn(k_rows, N, device=cuda, generator=g).bfloat16()
    out = torch.full((M, N), float("nan"), device=cuda)
    run_mn(w, x, M, N, k_rows, True, out, splits=1, accumulate=False)
    close(out, x.float() @ w.float(), tol=1e-4 * max(1.0, (k_rows / 64) ** 0.5))


# 128 < M <= 256 rows with a long K (the 7B batch-256 decode's down GEMM): the
# skinny path -- one 256-token tile, two 128-row weight tiles per CTA, split-K
# over a cluster of 4-8 (gemm.cu skinny256_splits); ragged M and N
@pytest.mark.parametrize("M,N,K", [(256, 3584, 18944), (200, 4608, 16384), (129, 1000, 8192)])
def test_gemm_skinny256_store_and_residual(cuda, M, N, K):
    g = torch.Generator(device=cuda).manual_seed(M + N + K)
    w = (torch.randn(N, K, device=cuda, generator=g) * 0.05).bfloat16()
    x = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    bias = torch.randn(N, device=cuda, generator=g).bfloat16()
    ref = x.float() @ w.float().T
    outs = []
    for _ in range(2):  # deterministic split-K order
        out = torch.full((M, N), float("nan"), device=cuda)
        run(w, x, EPI_F32, splits=0, bias=bias, out=out)
        outs.append(out)
    close(outs[0], ref + bias.float())
    assert torch.equal(outs[0], outs[1])
    if N % 128 == 0:
        parts = N // 128
        resid = torch.randn(M, N, device=cuda, generator=g)
        resid0 = resid.clone()
        gain = (torch.rand(N, device=cuda, generator=g) + 0.5).bfloat16()
        xg = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
        ssq = torch.empty(M, parts, device=cuda)
        run(w, x, EPI_RESID, splits=0, resid=resid, gain=gain, xg=xg, ssq_out=ssq)
        r = resid0 + ref
        close(resid, r)
        close(xg, r * gain.float(), tol=1e-2)
        close(ssq, (r.view(M, parts, 128) ** 2).sum(-1), tol=3e-3)
