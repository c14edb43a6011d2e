"""Time two GEMM shapes under SWARM_GEMM_DBG (set by the caller): which
pipeline limits the kernel?  1 = no output stores, 2 = no MMAs, 4 = no TMA loads."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_11913_b200 import _lib as L, ops
x = torch.randn(2048, 2048, device="cuda").bfloat16(); w1 = torch.randn(8192, 2048, device="cuda").bfloat16()
dy = torch.randn(2048, 2048, device="cuda").bfloat16(); g = torch.randn(2048, 8192, device="cuda").bfloat16()
acc = torch.zeros(2048, 8192, device="cuda"); out = torch.empty(2048, 8192, device="cuda", dtype=torch.bfloat16)
w2 = torch.randn(2048, 8192, device="cuda").bfloat16(); y = torch.empty(2048, 2048, device="cuda", dtype=torch.bfloat16)
cases = {"fwd.ffn1 2048x8192x2048": lambda: ops.gemm(x, w1, out=out),
         "fwd.ffn2 2048x2048x8192": lambda: ops.gemm(out, w2, out=y),
         "wgrad.ffn2 MN/MN reduce": lambda: ops.gemm(dy, g, a_t=True, b_t=True, epilogue=L.EPI_ACCUM_F32, out=acc)}
for name, fn in cases.items():
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    fl = 2 * 2048 * 8192 * 2048
    print(f"dbg={os.environ.get('SWARM_GEMM_DBG','0')} {name}: {ms*1e3:.1f} us {fl/ms/1e9:.0f} TFLOP/s", flush=True)
