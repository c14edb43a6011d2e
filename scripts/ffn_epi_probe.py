"""FFN GEMMs of configs[2] with their in-step epilogues vs plain stores (back-to-back launches, L2 warm):
FFN1 fwd (GELU_DERIV: g and gelu'(u) out), FFN1 dgrad-side (MUL: du = (dy W2) * gelu'), FFN2 fwd (RESIDUAL)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_11913_b200 import _lib as L, ops
T, d, F = 2048, 2048, 8192
ws = ops.gemm_workspace()
def mk(M, N, K, epi, bmn=False, aux_out=False):
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = (torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")).bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    aux = torch.randn(M, N, device="cuda").bfloat16()
    g = L.GemmArgs()
    g.m, g.n, g.k, g.batch, g.bh = M, N, K, 1, 1
    g.a, g.lda, g.a_rows, g.a_cols = a.data_ptr(), K, M, K
    g.b, g.ldb, g.b_mn_major, g.b_rows, g.b_cols = b.data_ptr(), b.shape[1], int(bmn), b.shape[0], b.shape[1]
    g.d, g.ldd = out.data_ptr(), N
    g.alpha, g.epilogue = 1.0, epi
    g.aux = aux.data_ptr() if epi != L.EPI_STORE_BF16 else None
    g.workspace, g.workspace_bytes = ws.data_ptr(), ws.numel()
    keep = (a, b, out, aux)
    return keep, (lambda: ops.gemm_raw(g))
cases = [("ffn1 plain", T, F, d, L.EPI_STORE_BF16, False), ("ffn1 GELU_DERIV", T, F, d, L.EPI_GELU_DERIV, False),
         ("ffn1 GELU", T, F, d, L.EPI_GELU, False),
         ("dgrad plain Bmn", T, F, d, L.EPI_STORE_BF16, True), ("dgrad MUL Bmn", T, F, d, L.EPI_MUL, True),
         ("ffn2 plain", T, d, F, L.EPI_STORE_BF16, False), ("ffn2 RESIDUAL", T, d, F, L.EPI_RESIDUAL, False)]
for name, M, N, K, epi, bmn in cases:
    keep, fn = mk(M, N, K, epi, bmn)
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20): fn()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(f"{name:18s} {us:7.1f} us  {2 * M * N * K / us / 1e6:6.0f} TFLOP/s", flush=True)
