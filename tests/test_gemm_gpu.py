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


# Stream-K tail (csrc/gemm.cu): shapes whose 256x256 tile count leaves a partial
# last wave on 74 SM pairs, so the tail tiles are split along K across clusters.
# The first shape takes the stream-K path under the default policy (few tiles, long K:
# configs[3]'s 512 x 4096 x 16384); the rest only when forced (SWARM_GEMM_STREAMK=1,
# test_gemm_kernel_variants).
SK_SHAPES = [(512, 4096, 16384), (512, 4096, 4096), (768, 3328, 4096), (1000, 2000, 1000), (2048, 2048, 8192),
             (4096, 2304, 1024)]


@pytest.mark.parametrize("m,n,k", SK_SHAPES)
@pytest.mark.parametrize("a_t,b_t", [(False, False), (False, True), (True, True)])
def test_gemm_streamk_matches_whole_tiles(cuda, m, n, k, a_t, b_t):
    """Stream-K vs whole-tile launches: identical up to fp32 summation order
    (rtol 1e-5, atol 1e-4 * sqrt(K) for O(sqrt(K)) outputs), against torch as
    well, and repeated launches agree (the self-resetting flags are clean)."""
    import torch
    from paper_2301_11913_b200 import ops
    torch.manual_seed(m + 3 * n + 7 * k)
    a = torch.randn((k, m) if a_t else (m, k), device="cuda").bfloat16()
    b = torch.randn((k, n) if b_t else (n, k), device="cuda").bfloat16()
    ref = ref_mm(a, b, a_t, b_t)
    whole = ops.gemm(a, b, a_t=a_t, b_t=b_t, epilogue=1, streamk=False)
    for _ in range(3):
        sk = ops.gemm(a, b, a_t=a_t, b_t=b_t, epilogue=1, streamk=True)
        torch.testing.assert_close(sk, whole, rtol=1e-5, atol=1e-4 * math.sqrt(k))
    torch.testing.assert_close(sk, ref, rtol=1e-4, atol=1e-4 * math.sqrt(k))
    sk16 = ops.gemm(a, b, a_t=a_t, b_t=b_t, streamk=True)
    torch.testing.assert_close(sk16.float(), ref, rtol=1e-2, atol=1e-2 * math.sqrt(k) / 8 + 1e-2)


def test_gemm_streamk_epilogues_and_graph(cuda):
    """Every fused epilogue on a stream-K shape, eager and replayed from a CUDA
    graph several times (the partial/flag handshake must be replay-safe)."""
    import torch
    from paper_2301_11913_b200 import _lib as L, ops
    torch.manual_seed(1)
    m, n, k = 2048, 2048, 2048
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = torch.randn(n, k, device="cuda").bfloat16()
    r = torch.randn(m, n, device="cuda").bfloat16()
    ref = a.float() @ b.float().t()
    out = ops.gemm(a, b, epilogue=L.EPI_RESIDUAL, aux=r, streamk=True)
    torch.testing.assert_close(out.float(), ref + r.float(), rtol=1e-2, atol=0.5)
    u = torch.empty(m, n, device="cuda").bfloat16()
    g = ops.gemm(a, b, epilogue=L.EPI_GELU, aux=u, streamk=True)
    torch.testing.assert_close(u.float(), ref, rtol=1e-2, atol=0.5)
    torch.testing.assert_close(g.float(), torch.nn.functional.gelu(u.float(), approximate="tanh"), rtol=2e-2, atol=2e-2)
    acc = torch.zeros(m, n, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ops.gemm_workspace()  # allocate this stream's scratch before capture
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            ops.gemm(a, b, epilogue=L.EPI_ACCUM_F32, out=acc, streamk=True)
    torch.cuda.current_stream().wait_stream(s)
    acc.zero_()
    for _ in range(4):
        graph.replay()
    torch.cuda.synchronize()
    torch.testing.assert_close(acc, 4 * ref, rtol=1e-4, atol=1e-2 * math.sqrt(k))


@pytest.mark.parametrize("tri", [1, 2])
def test_gemm_causal_k_skip(cuda, tri):
    """k_tri: with a causal A (P / dS, tri=1; their transposes, tri=2) the kernel
    skips the all-zero k-blocks; the result equals the dense product exactly
    because the skipped blocks contribute nothing.  Poison the skipped region
    with NaN to prove it is never read."""
    import torch
    from paper_2301_11913_b200 import _lib as L, ops
    Bz, Lq, dh = 6, 512, 128
    torch.manual_seed(tri)
    A = torch.randn(Bz, Lq, Lq, device="cuda")
    mask = torch.ones(Lq, Lq, device="cuda").tril().bool()  # A[i, j] != 0 only for j <= i
    dense = A.masked_fill(~mask, 0.0)
    if tri == 2:
        dense = dense.transpose(1, 2).contiguous()  # A[i, j] != 0 only for j >= i
        mask = mask.t()
    Ab = dense.bfloat16()
    # rows of a tile that still share a k-block with the nonzero region stay zero;
    # everything outside whole skipped 64-wide k-blocks of each 128-row tile -> NaN
    poisoned = Ab.clone()
    for mt in range(Lq // 128):
        r0, r1 = mt * 128, (mt + 1) * 128
        if tri == 1:
            k_end = -(-r1 // 64) * 64
            poisoned[:, r0:r1, k_end:] = float("nan")
        else:
            k_beg = (r0 // 64) * 64
            poisoned[:, r0:r1, :k_beg] = float("nan")
    V = torch.randn(Bz * Lq, dh, device="cuda").bfloat16()
    out = torch.empty(Bz * Lq, dh, device="cuda", dtype=torch.float32)
    a2 = poisoned.reshape(Bz * Lq, Lq)
    args = L.GemmArgs()
    args.m, args.n, args.k, args.batch, args.bh = Lq, dh, Lq, Bz, 1
    args.a, args.lda, args.a_mn_major, args.a_rows, args.a_cols = a2.data_ptr(), Lq, 0, Bz * Lq, Lq
    args.ra0 = Lq
    args.b, args.ldb, args.b_mn_major, args.b_rows, args.b_cols = V.data_ptr(), dh, 1, Bz * Lq, dh
    args.rb0 = Lq
    args.d, args.ldd, args.rd0 = out.data_ptr(), dh, Lq
    args.alpha, args.epilogue, args.k_tri = 1.0, L.EPI_STORE_F32, tri
    ops.gemm_raw(args)
    ref = (Ab.float() @ V.float().view(Bz, Lq, dh)).reshape(Bz * Lq, dh)
    assert torch.isfinite(out).all()
    torch.testing.assert_close(out, ref, rtol=1e-4, atol=1e-3)


_VARIANT_CHECK = r"""
import math, sys, torch
sys.path.insert(0, {root!r})
from paper_2301_11913_b200 import _lib as L, ops
torch.manual_seed(0)
for (m, n, k) in [(2048, 2048, 2048), (512, 6144, 2048), (768, 1280, 4096), (200, 300, 96), (512, 4096, 8192)]:
    for a_t, b_t in [(False, False), (False, True), (True, True)]:
        if (a_t and m % 8) or (b_t and n % 8) or k % 8:
            continue  # rows must be 16-byte aligned
        a = torch.randn((k, m) if a_t else (m, k), device="cuda").bfloat16()
        b = torch.randn((k, n) if b_t else (n, k), device="cuda").bfloat16()
        A = a.float().t() if a_t else a.float()
        B = b.float().t() if b_t else b.float()
        ref = A @ B.t()
        out = ops.gemm(a, b, a_t=a_t, b_t=b_t, epilogue=L.EPI_STORE_F32, streamk=True)
        torch.testing.assert_close(out, ref, rtol=1e-4, atol=1e-4 * math.sqrt(k))
        acc = torch.ones(m, n, device="cuda")
        ops.gemm(a, b, a_t=a_t, b_t=b_t, epilogue=L.EPI_ACCUM_F32, out=acc, streamk=True)
        torch.testing.assert_close(acc, ref + 1, rtol=1e-4, atol=1e-4 * math.sqrt(k))
print("ok")
"""


@pytest.mark.parametrize("env", [{"SWARM_GEMM_MCAST": "0"}, {"SWARM_GEMM_PAIR": "0"},
                                 {"SWARM_GEMM_TMA_EPI": "0"}, {"SWARM_PDL": "1"}, {"SWARM_GEMM_STREAMK": "1"},
                                 {"SWARM_GEMM_STREAMK": "0"}, {"SWARM_GEMM_EPI8": "0"}, {"SWARM_GEMM_EPI8": "1"}])
def test_gemm_kernel_variants(cuda, env):
    """The non-default kernel variants (2-CTA pairs without multicast, 1-CTA
    tiles, direct-store epilogue, programmatic dependent launch on, stream-K
    forced on / off, the four-warp pair epilogue, eight warps for fp32 outputs too) stay correct; the selection is read once per process,
    hence a subprocess per variant."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _VARIANT_CHECK.format(root=root)], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("m,n,t", [(2048, 8192, 2048), (6144, 2048, 2048), (2048, 2048, 512), (256, 1024, 128),
                                   (128, 512, 256)])
@pytest.mark.parametrize("a_t,b_t", [(True, True), (False, False)])
def test_gemm_two_k_segments(cuda, m, n, t, a_t, b_t):
    """Paired weight gradients: K = 2t split over two buffer pairs (a, b) and (a2, b2)
    equals the GEMM over the concatenation (fp32 reduce-add epilogue, as in the
    executor), on the pair kernel and on the small-tile fallback."""
    import torch
    from paper_2301_11913_b200 import _lib as L, ops
    torch.manual_seed(m + n + t)
    k = 2 * t
    A = torch.randn((k, m) if a_t else (m, k), device="cuda").bfloat16()
    B = torch.randn((k, n) if b_t else (n, k), device="cuda").bfloat16()
    # the two halves in separate allocations
    if a_t:
        a1, a2 = A[:t].clone(), A[t:].clone()
    else:
        a1, a2 = A[:, :t].contiguous(), A[:, t:].contiguous()
    if b_t:
        b1, b2 = B[:t].clone(), B[t:].clone()
    else:
        b1, b2 = B[:, :t].contiguous(), B[:, t:].contiguous()
    acc = torch.ones(m, n, device="cuda")
    g = L.GemmArgs()
    g.m, g.n, g.k, g.batch, g.bh = m, n, k, 1, 1
    g.a, g.lda, g.a_mn_major, g.a_rows, g.a_cols = a1.data_ptr(), a1.stride(0), int(a_t), a1.shape[0], a1.shape[1]
    g.b, g.ldb, g.b_mn_major, g.b_rows, g.b_cols = b1.data_ptr(), b1.stride(0), int(b_t), b1.shape[0], b1.shape[1]
    g.a2, g.b2 = a2.data_ptr(), b2.data_ptr()
    g.d, g.ldd, g.alpha, g.epilogue = acc.data_ptr(), n, 1.0, L.EPI_ACCUM_F32
    ops.gemm_raw(g)
    ref = ref_mm(A, B, a_t, b_t) + 1
    torch.testing.assert_close(acc, ref, rtol=1e-4, atol=1e-4 * math.sqrt(k))


@pytest.mark.parametrize("m,n,k", [(512, 1024, 256), (2048, 8192, 512), (200, 136, 64)])
def test_gemm_gelu_deriv_and_mul_epilogues(cuda, m, n, k):
    """The MLP's forward / backward epilogue pair: GELU_DERIV writes gelu(acc) and keeps
    gelu'(acc) in U (one SFU tanh for both); MUL multiplies the backward product by U."""
    import torch
    from paper_2301_11913_b200 import _lib as L, ops
    torch.manual_seed(1)
    a = torch.randn(m, k, device="cuda").bfloat16() * 0.25
    b = torch.randn(n, k, device="cuda").bfloat16() * 0.25
    ref = a.float() @ b.float().t()
    u = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    g = ops.gemm(a, b, epilogue=L.EPI_GELU_DERIV, aux=u)
    x = ref.clone().requires_grad_()
    y = torch.nn.functional.gelu(x, approximate="tanh")
    y.backward(torch.ones_like(y))
    torch.testing.assert_close(g.float(), y.detach(), rtol=1e-2, atol=2e-2)
    torch.testing.assert_close(u.float(), x.grad, rtol=1e-2, atol=2e-2)
    out = ops.gemm(a, b, epilogue=L.EPI_MUL, aux=u)
    torch.testing.assert_close(out.float(), ref * u.float(), rtol=1e-2, atol=5e-2)


@pytest.mark.parametrize("m,n,k,b_t", [(2048, 2048, 2048, False), (2048, 2000, 1024, False), (1024, 3072, 512, True)])
def test_gemm_bf16_epilogues_pair_shapes(cuda, m, n, k, b_t):
    """Every bf16-output epilogue at shapes the 2-CTA pair kernel takes (its eight-warp
    epilogue: two warps per TMEM lane quarter, each draining half of a tile's columns),
    including the o-projection's 2048^3 (one tile per cluster), a ragged N whose last
    tile ends inside a 32-column chunk of the second warp group, and an MN-major B."""
    import torch
    from paper_2301_11913_b200 import _lib as L, ops
    torch.manual_seed(m + n + k)
    a = torch.randn(m, k, device="cuda").bfloat16() * 0.25
    b = (torch.randn(k, n, device="cuda") if b_t else torch.randn(n, k, device="cuda")).bfloat16() * 0.25
    ref = a.float() @ (b.float() if b_t else b.float().t())
    tol = dict(rtol=1e-2, atol=3e-2)
    out = ops.gemm(a, b, b_t=b_t)
    torch.testing.assert_close(out.float(), ref, **tol)
    r = torch.randn(m, n, device="cuda").bfloat16()
    out = ops.gemm(a, b, b_t=b_t, epilogue=L.EPI_RESIDUAL, aux=r)
    torch.testing.assert_close(out.float(), ref + r.float(), **tol)
    u = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    out = ops.gemm(a, b, b_t=b_t, epilogue=L.EPI_GELU, aux=u)
    torch.testing.assert_close(u.float(), ref, **tol)
    torch.testing.assert_close(out.float(), torch.nn.functional.gelu(ref, approximate="tanh"), **tol)
    x = ref.clone().requires_grad_()
    torch.nn.functional.gelu(x, approximate="tanh").backward(torch.ones_like(x))
    out = ops.gemm(a, b, b_t=b_t, epilogue=L.EPI_DGELU, aux=u)
    torch.testing.assert_close(out.float(), ref * x.grad, rtol=2e-2, atol=5e-2)
    g = ops.gemm(a, b, b_t=b_t, epilogue=L.EPI_GELU_DERIV, aux=u)
    torch.testing.assert_close(g.float(), torch.nn.functional.gelu(ref, approximate="tanh"), **tol)
    torch.testing.assert_close(u.float(), x.grad, **tol)
    out = ops.gemm(a, b, b_t=b_t, epilogue=L.EPI_MUL, aux=u)
    torch.testing.assert_close(out.float(), ref * u.float(), rtol=1e-2, atol=5e-2)


@pytest.mark.parametrize("m,n,k", [(2048, 2048, 2048), (2048, 2000, 512)])
def test_gemm_pair_epilogues_repeatable(cuda, m, n, k):
    """Race check of the pair kernel's epilogues (staging slots reused under TMA stores /
    reduce-adds, eight bf16 warps, four fp32 warps): each epilogue's output is a fixed
    function of the inputs, so 200 launches (pairs back to back) must agree bit for bit."""
    import torch
    from paper_2301_11913_b200 import _lib as L, ops
    torch.manual_seed(m + n)
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = torch.randn(n, k, device="cuda").bfloat16()
    r = torch.randn(m, n, device="cuda").bfloat16()
    for epi in (L.EPI_STORE_BF16, L.EPI_RESIDUAL, L.EPI_GELU_DERIV, L.EPI_STORE_F32, L.EPI_ACCUM_F32):
        f32 = epi in (L.EPI_STORE_F32, L.EPI_ACCUM_F32)
        outs = [torch.zeros(m, n, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16) for _ in range(2)]
        auxs = [torch.empty(m, n, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
        aux_of = lambda u: r if epi == L.EPI_RESIDUAL else (u if epi == L.EPI_GELU_DERIV else None)
        ops.gemm(a, b, epilogue=epi, aux=aux_of(auxs[0]), out=outs[0])
        torch.cuda.synchronize()
        first = (outs[0].clone(), auxs[0].clone())
        for it in range(100):  # two launches back to back per check
            for o, u in zip(outs, auxs):
                if epi == L.EPI_ACCUM_F32:
                    o.zero_()
                ops.gemm(a, b, epilogue=epi, aux=aux_of(u), out=o)
            torch.cuda.synchronize()
            for o, u in zip(outs, auxs):
                assert torch.equal(o, first[0]), (epi, it)
                if epi == L.EPI_GELU_DERIV:
                    assert torch.equal(u, first[1]), (epi, it)
