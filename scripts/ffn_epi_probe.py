"""FFN GEMMs of configs[2] with their in-step epilogues vs plain stores (back-to-back launches, L2 warm):
FFN1 fwd (GELU_DERIV: g and gelu'(u) out), FFN1 dgrad-side (MUL: du = (dy W2) * gelu'), FFN2 fwd (RESIDUAL)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_11913_b200 import _lib as L, ops
T, d, F = 2048, 2048, 8192
ws = ops.gemm_workspace()
def mk(M, N, K, epi, bmn=False, amn=False):
    a = (torch.randn(K, M, device="cuda") if amn else torch.randn(M, K, device="cuda")).bfloat16()
    b = (torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")).bfloat16()
    f32 = epi in (L.EPI_STORE_F32, L.EPI_ACCUM_F32)
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    aux = torch.randn(M, N, device="cuda").bfloat16()
    g = L.GemmArgs()
    g.m, g.n, g.k, g.batch, g.bh = M, N, K, 1, 1
    g.a, g.lda, g.a_mn_major, g.a_rows, g.a_cols = a.data_ptr(), a.shape[1], int(amn), a.shape[0], a.shape[1]
    g.b, g.ldb, g.b_mn_major, g.b_rows, g.b_cols = b.data_ptr(), b.shape[1], int(bmn), b.shape[0], b.shape[1]
    g.d, g.ldd = out.data_ptr(), N
    g.alpha, g.epilogue = 1.0, epi
    g.aux = aux.data_ptr() if epi not in (L.EPI_STORE_BF16, L.EPI_STORE_F32, L.EPI_ACCUM_F32) else None
    g.workspace, g.workspace_bytes = ws.data_ptr(), ws.numel()
    keep = (a, b, out, aux)
    return keep, (lambda: ops.gemm_raw(g))
cases = [("ffn1 plain", T, F, d, L.EPI_STORE_BF16, False), ("ffn1 GELU_DERIV", T, F, d, L.EPI_GELU_DERIV, False),
         ("ffn1 GELU", T, F, d, L.EPI_GELU, False),
         ("dgrad plain Bmn", T, F, d, L.EPI_STORE_BF16, True), ("dgrad MUL Bmn", T, F, d, L.EPI_MUL, True),
         ("ffn2 plain", T, d, F, L.EPI_STORE_BF16, False), ("ffn2 RESIDUAL", T, d, F, L.EPI_RESIDUAL, False),
         ("oproj plain", T, d, d, L.EPI_STORE_BF16, False), ("oproj RESIDUAL", T, d, d, L.EPI_RESIDUAL, False),
         ("wgrad1 ACCUM Amn Bmn", F, d, T, L.EPI_ACCUM_F32, True, True),
         ("wgrad2 ACCUM Amn Bmn", d, F, T, L.EPI_ACCUM_F32, True, True),
         ("wgrad1 STORE_F32", F, d, T, L.EPI_STORE_F32, True, True)]
for name, M, N, K, epi, bmn, *amn in cases:
    keep, fn = mk(M, N, K, epi, bmn, bool(amn and amn[0]))
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20): fn()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(f"{name:18s} {us:7.1f} us  {2 * M * N * K / us / 1e6:6.0f} TFLOP/s", flush=True)
