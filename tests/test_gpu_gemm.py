"""tcgen05 GEMM (csrc/gemm.cuh) through the C ABI (tc_gemm) vs a torch fp32 reference of the
same bf16 operands. Tolerances: bf16 outputs rtol 1e-2 (one bf16 rounding, 2^-8) plus
atol 1e-2 * std(ref); fp32 outputs rtol 1e-4, atol 1e-4 * std(ref) (accumulation order only)."""
import pytest
import torch

pytestmark = pytest.mark.gpu

EPI_BF16, EPI_BIAS, EPI_RESID, EPI_SWIGLU, EPI_F32 = 0, 1, 2, 3, 4


def _run(a, b, out, m, n, k, epi, bias=None, bn=0, splits=0):
    from paper_2508_01989_b200 import runtime
    runtime.gemm(a.data_ptr(), b.data_ptr(), out.data_ptr(), m, n, k, epi,
                 bias.data_ptr() if bias is not None else None, bn, splits)
    torch.cuda.synchronize()


def _close(got, ref, bf16_out):
    s = ref.float().std().item() + 1e-6
    if bf16_out:
        torch.testing.assert_close(got.float(), ref, rtol=1e-2, atol=1e-2 * s)
    else:
        torch.testing.assert_close(got.float(), ref, rtol=1e-4, atol=1e-4 * s)


# bn: 0 auto / 128 / 256; splits = CTAs-per-tile cap (0 = full stream-K, 1 = one CTA per tile)
@pytest.mark.parametrize("m,n,k,bn,splits", [
    (128, 256, 64, 256, 1), (1, 256, 128, 0, 0), (100, 512, 256, 0, 0), (129, 1024, 512, 128, 1),
    (576, 6144, 4096, 0, 0), (576, 4096, 4096, 0, 0), (576, 4096, 14336, 0, 0), (64, 6144, 4096, 0, 0),
    (64, 4096, 14336, 0, 0), (1100, 1024, 4096, 0, 0), (256, 512, 1024, 128, 1), (64, 512, 1024, 128, 4),
    (200, 256, 4096, 256, 2), (5, 256, 256, 0, 0), (3000, 6144, 4096, 0, 0), (1, 128, 64, 128, 0),
    (333, 7168, 5120, 0, 0), (64, 256, 8192, 256, 0),
])
def test_gemm_bf16(cuda_ok, m, n, k, bn, splits):
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n + k)
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16, generator=g)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16, generator=g)
    out = torch.zeros(m, n, device="cuda", dtype=torch.bfloat16)
    _run(a, b, out, m, n, k, EPI_BF16, bn=bn, splits=splits)
    _close(out, a.float() @ b.float().T, True)


@pytest.mark.parametrize("m,splits", [(37, 0), (300, 1), (64, 2)])
def test_gemm_bias(cuda_ok, m, splits):
    n, k = 7168, 5120
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.05
    bias = torch.randn(n, device="cuda", dtype=torch.bfloat16)
    out = torch.zeros(m, n, device="cuda", dtype=torch.bfloat16)
    _run(a, b, out, m, n, k, EPI_BIAS, bias=bias, splits=splits)
    _close(out, a.float() @ b.float().T + bias.float(), True)


@pytest.mark.parametrize("m,n,k,splits", [(576, 4096, 4096, 0), (64, 4096, 14336, 0), (17, 256, 512, 1),
                                          (64, 4096, 4096, 4)])
def test_gemm_residual_add(cuda_ok, m, n, k, splits):
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.02
    resid = torch.randn(m, n, device="cuda", dtype=torch.float32)
    ref = resid + a.float() @ b.float().T
    _run(a, b, resid, m, n, k, EPI_RESID, splits=splits)
    _close(resid, ref, False)


@pytest.mark.parametrize("m,f,k,bn,splits", [(576, 14336, 4096, 0, 0), (64, 14336, 4096, 0, 0),
                                             (33, 512, 256, 128, 1), (130, 1024, 512, 256, 1), (64, 512, 1024, 128, 2)])
def test_gemm_swiglu_interleaved(cuda_ok, m, f, k, bn, splits):
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    wg = torch.randn(f, k, device="cuda", dtype=torch.bfloat16) * 0.03
    wu = torch.randn(f, k, device="cuda", dtype=torch.bfloat16) * 0.03
    phys = torch.stack([wg.view(f // 64, 64, k), wu.view(f // 64, 64, k)], dim=1).reshape(2 * f, k).contiguous()
    out = torch.zeros(m, f, device="cuda", dtype=torch.bfloat16)
    _run(a, phys, out, m, 2 * f, k, EPI_SWIGLU, bn=bn, splits=splits)
    ref = torch.nn.functional.silu(a.float() @ wg.float().T) * (a.float() @ wu.float().T)
    _close(out, ref, True)


@pytest.mark.parametrize("m,n,k", [(1, 128256, 4096), (65, 128256, 4096), (130, 152064, 5120), (3, 1024, 256)])
def test_gemm_f32_logits(cuda_ok, m, n, k):
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.03
    out = torch.zeros(m, n, device="cuda", dtype=torch.float32)
    _run(a, b, out, m, n, k, EPI_F32)
    _close(out, a.float() @ b.float().T, False)


# ---- weight-stationary pair variant (gemm_ws.cuh: tokens on the MMA's N), forced with bn=1024;
# the token tile TN = round_up(T / ceil(T / 256), 32) covers ragged T (1, 20, 100, 300, 1100 ...)
@pytest.mark.parametrize("m,n,k", [(576, 6144, 4096), (1, 256, 128), (20, 512, 256), (100, 512, 1024),
                                   (300, 768, 512), (512, 1024, 4096), (1100, 1024, 4096), (3000, 512, 256),
                                   (256, 256, 64), (129, 7168, 5120), (64, 6144, 4096), (64, 7168, 5120),
                                   (1056, 7168, 5120)])
def test_gemm_ws_bf16(cuda_ok, m, n, k):
    # decode-only QKV shapes (64 x 6144 / 64 x 7168: fewer units than pairs) and config 5's
    # (1056 x 7168, 5 token tiles); three back-to-back launches must give the same result
    g = torch.Generator(device="cuda").manual_seed(m * 13 + n + k)
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16, generator=g)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16, generator=g)
    for _ in range(3):
        out = torch.zeros(m, n, device="cuda", dtype=torch.bfloat16)
        _run(a, b, out, m, n, k, EPI_BF16, bn=1024)
        _close(out, a.float() @ b.float().T, True)


# splits = 0: grouped stream-K (pair groups of one pair per token tile walk the weight-tile-major
# k-block stream; ranges cut across tile boundaries): one token tile with more weight tiles than
# pairs (64 x 28672, 200 x 20480), several token tiles (576 -> 3, 1100 -> 5, 3000 -> 12 tiles:
# 6 groups), fewer k-blocks than groups (7 x 256 x 128).
@pytest.mark.parametrize("m,n,k,splits", [(576, 4096, 14336, 0), (576, 4096, 4096, 3), (576, 4096, 4096, 1),
                                          (64, 4096, 4096, 0), (333, 5120, 13824, 0), (7, 256, 512, 2),
                                          (64, 28672, 1024, 0), (200, 20480, 704, 0), (576, 4096, 4096, 0),
                                          (1100, 4096, 4096, 0), (3000, 512, 1024, 0), (7, 256, 128, 0)])
def test_gemm_ws_residual(cuda_ok, m, n, k, splits):
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.02
    resid = torch.randn(m, n, device="cuda", dtype=torch.float32)
    ref = resid + a.float() @ b.float().T
    _run(a, b, resid, m, n, k, EPI_RESID, bn=1024, splits=splits)
    _close(resid, ref, False)


# gate_up shapes of config 2 (576 x 28672: 336 units = 4 x 74 + 40), the decode-only step
# (64 x 28672: 112 = 74 + 38) and config 5 (1056 x 27648, K = 5120: 540 units)
@pytest.mark.parametrize("m,f,k", [(576, 14336, 4096), (97, 512, 256), (1100, 1024, 512), (64, 14336, 4096),
                                   (1056, 13824, 5120)])
def test_gemm_ws_swiglu(cuda_ok, m, f, k):
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    wg = torch.randn(f, k, device="cuda", dtype=torch.bfloat16) * 0.03
    wu = torch.randn(f, k, device="cuda", dtype=torch.bfloat16) * 0.03
    phys = torch.stack([wg.view(f // 64, 64, k), wu.view(f // 64, 64, k)], dim=1).reshape(2 * f, k).contiguous()
    ref = torch.nn.functional.silu(a.float() @ wg.float().T) * (a.float() @ wu.float().T)
    for _ in range(2):
        out = torch.zeros(m, f, device="cuda", dtype=torch.bfloat16)
        _run(a, phys, out, m, 2 * f, k, EPI_SWIGLU, bn=1024)
        _close(out, ref, True)


def test_gemm_ws_bias_f32(cuda_ok):
    m, n, k = 300, 7168, 5120
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.05
    bias = torch.randn(n, device="cuda", dtype=torch.bfloat16)
    o = torch.zeros(m, n, device="cuda", dtype=torch.bfloat16)
    _run(a, b, o, m, n, k, EPI_BIAS, bias=bias, bn=1024)
    _close(o, a.float() @ b.float().T + bias.float(), True)
    o3 = torch.zeros(m, n, device="cuda", dtype=torch.float32)
    _run(a, b, o3, m, n, k, EPI_F32, bn=1024)
    _close(o3, a.float() @ b.float().T, False)
