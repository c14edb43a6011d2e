"""Two representative GEMMs for an ncu --set full capture: fwd.ffn1 (K-major,
STORE_BF16) and bwd.ffn2.wgrad (MN-major operands, TMA reduce-add epilogue)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_11913_b200 import _lib as L, ops
x = torch.randn(2048, 2048, device="cuda").bfloat16()
w1 = torch.randn(8192, 2048, device="cuda").bfloat16()
dy = torch.randn(2048, 2048, device="cuda").bfloat16()
g = torch.randn(2048, 8192, device="cuda").bfloat16()
acc = torch.zeros(2048, 8192, device="cuda")
for _ in range(2):
    ops.gemm(x, w1)                                                       # fwd.ffn1
    ops.gemm(dy, g, a_t=True, b_t=True, epilogue=L.EPI_ACCUM_F32, out=acc)  # bwd.ffn2.wgrad
torch.cuda.synchronize()
