"""GPU numerics: K5 tcgen05 GEMM vs a torch fp32 reference of the same op.

Tolerance: bf16 inputs are exact in fp32, accumulation is fp32 in TMEM, so the
only differences are accumulation order and the bf16 output rounding:
rtol 1e-2 / atol 1e-2 * sqrt(K)/8 on bf16 outputs, 1e-4-level on fp32 outputs.
"""
import math

import pytest

pytestmark = pytest.mark.gpu


def ref_mm(a, b, a_t, b_t):
    A = a.float().t() if a_t else a.float()
    B = b.float().t() if b_t else b.float()
    return A @ B.t()


SHAPES = [(128, 256, 64), (256, 512, 512), (384, 128, 192), (200, 300, 96), (2048, 2048, 2048), (512, 6144, 2048),
          (1024, 50304, 256), (64, 64, 64)]


@pytest.mark.parametrize("a_t", [False, True])
@pytest.mark.parametrize("b_t", [False, True])
@pytest.mark.parametrize("m,n,k", SHAPES)
def test_gemm_bf16(cuda, m, n, k, a_t, b_t):
    import torch
    from paper_2301_11913_b200 import ops
    if (a_t and m % 8) or (b_t and n % 8) or (not a_t and k % 8) or (not b_t and k % 8):
        pytest.skip("rows must be 16-byte aligned")
    torch.manual_seed(m * 7 + n * 3 + k)
    a = torch.randn((k, m) if a_t else (m, k), device="cuda").bfloat16()
    b = torch.randn((k, n) if b_t else (n, k), device="cuda").bfloat16()
    out = ops.gemm(a, b, a_t=a_t, b_t=b_t, out_dtype=torch.bfloat16)
    ref = ref_mm(a, b, a_t, b_t)
    torch.testing.assert_close(out.float(), ref, rtol=1e-2, atol=1e-2 * math.sqrt(k) / 8 + 1e-2)
    out32 = ops.gemm(a, b, a_t=a_t, b_t=b_t, epilogue=1)
    torch.testing.assert_close(out32, ref, rtol=1e-4, atol=1e-4 * math.sqrt(k))


def test_gemm_epilogues(cuda):
    import torch
    from paper_2301_11913_b200 import _lib as L, ops
    torch.manual_seed(0)
    m, n, k = 512, 1024, 256
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = torch.randn(n, k, device="cuda").bfloat16()
    ref = a.float() @ b.float().t()
    # alpha
    out = ops.gemm(a, b, epilogue=L.EPI_STORE_F32, alpha=0.125)
    torch.testing.assert_close(out, ref * 0.125, rtol=1e-4, atol=1e-3)
    # accumulate
    acc = torch.ones(m, n, device="cuda")
    ops.gemm(a, b, epilogue=L.EPI_ACCUM_F32, out=acc)
    ops.gemm(a, b, epilogue=L.EPI_ACCUM_F32, out=acc)
    torch.testing.assert_close(acc, 1 + 2 * ref, rtol=1e-4, atol=1e-2)
    # residual
    r = torch.randn(m, n, device="cuda").bfloat16()
    out = ops.gemm(a, b, epilogue=L.EPI_RESIDUAL, aux=r)
    torch.testing.assert_close(out.float(), ref + r.float(), rtol=1e-2, atol=0.3)
    # gelu: U = acc, D = gelu(acc)
    u = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    out = ops.gemm(a, b, epilogue=L.EPI_GELU, aux=u)
    torch.testing.assert_close(u.float(), ref, rtol=1e-2, atol=0.3)
    torch.testing.assert_close(out.float(), torch.nn.functional.gelu(ref, approximate="tanh"), rtol=1e-2, atol=0.3)
    # dgelu: D = acc * gelu'(U)
    uu = torch.randn(m, n, device="cuda").bfloat16()
    out = ops.gemm(a, b, epilogue=L.EPI_DGELU, aux=uu)
    x = uu.float().requires_grad_()
    torch.nn.functional.gelu(x, approximate="tanh").backward(torch.ones_like(x))
    torch.testing.assert_close(out.float(), ref * x.grad, rtol=2e-2, atol=0.3)


def test_gemm_batched_heads(cuda):
    """Batched form used by attention: S_bh = Q_bh K_bh^T read in place from a
    [T, 3d] QKV buffer; batch z -> (b, h) coordinate offsets."""
    import torch
    from paper_2301_11913_b200 import _lib as L, ops
    B, H, Lq, dh = 2, 4, 256, 64
    d = H * dh
    qkv = torch.randn(B * Lq, 3 * d, device="cuda").bfloat16()
    S = torch.empty(B * H * Lq, Lq, device="cuda", dtype=torch.float32)
    args = L.GemmArgs()
    args.m, args.n, args.k, args.batch, args.bh = Lq, Lq, dh, B * H, H
    args.a, args.lda, args.a_mn_major, args.a_rows, args.a_cols = qkv.data_ptr(), 3 * d, 0, B * Lq, 3 * d
    args.ra0, args.ra1, args.ca0, args.ca1 = Lq, 0, 0, dh
    kv = qkv[:, d:]  # the K block starts at column d: offset the base pointer
    args.b, args.ldb, args.b_mn_major, args.b_rows, args.b_cols = kv.data_ptr(), 3 * d, 0, B * Lq, 2 * d
    args.rb0, args.rb1, args.cb0, args.cb1 = Lq, 0, 0, dh
    args.d, args.ldd = S.data_ptr(), Lq
    args.rd0, args.rd1, args.cd0, args.cd1 = H * Lq, Lq, 0, 0
    args.alpha, args.epilogue = 1.0, L.EPI_STORE_F32
    ops.gemm_raw(args)
    q = qkv[:, :d].float().view(B, Lq, H, dh).transpose(1, 2)
    kk = qkv[:, d:2 * d].float().view(B, Lq, H, dh).transpose(1, 2)
    ref = (q @ kk.transpose(-1, -2)).reshape(B * H * Lq, Lq)
    torch.testing.assert_close(S, ref, rtol=1e-4, atol=1e-3)
