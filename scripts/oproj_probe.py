"""o-proj GEMM (2048 x 2048 x 2048, configs[2]) variants: plain vs RESIDUAL epilogue, L2 warm vs flushed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_11913_b200 import _lib as L, ops
T = d = 2048
a = torch.randn(T, d, device="cuda").bfloat16()
w = torch.randn(d, d, device="cuda").bfloat16()
x = torch.randn(T, d, device="cuda").bfloat16()
out = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
ws = ops.gemm_workspace()
flush = torch.empty(256 << 20, device="cuda", dtype=torch.uint8)
def mk(epi, bmn=False):
    g = L.GemmArgs()
    g.m, g.n, g.k, g.batch, g.bh = T, d, d, 1, 1
    g.a, g.lda, g.a_rows, g.a_cols = a.data_ptr(), d, T, d
    g.b, g.ldb, g.b_mn_major, g.b_rows, g.b_cols = w.data_ptr(), d, int(bmn), d, d
    g.d, g.ldd = out.data_ptr(), d
    g.alpha, g.epilogue = 1.0, epi
    g.aux = x.data_ptr() if epi == L.EPI_RESIDUAL else None
    g.workspace, g.workspace_bytes = ws.data_ptr(), ws.numel()
    return lambda: ops.gemm_raw(g)
for name, fn in (("plain", mk(L.EPI_STORE_BF16)), ("residual", mk(L.EPI_RESIDUAL)), ("dgrad Bmn", mk(L.EPI_STORE_BF16, True))):
    for cold in (False, True):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(10):
            if cold: flush.zero_()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        us = tot / 10 * 1e3
        print(f"{name:10s} {'cold' if cold else 'warm'}: {us:6.1f} us  {2 * T * d * d / us / 1e6:6.0f} TFLOP/s")
