"""configs[3] few-tile GEMMs with and without stream-K (SWARM_GEMM_STREAMK / DBG set by the caller)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_11913_b200 import ops
shapes = {"o 512x4096x4096": (512, 4096, 4096), "ffn2 512x4096x16384": (512, 4096, 16384),
          "qkv 512x12288x4096": (512, 12288, 4096), "o C 2048^3": (2048, 2048, 2048)}
for name, (m, n, k) in shapes.items():
    a = torch.randn(m, k, device="cuda").bfloat16(); b = torch.randn(n, k, device="cuda").bfloat16()
    out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for sk in (False, True):
        fn = lambda: ops.gemm(a, b, out=out, streamk=sk)
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20): fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"STREAMK={os.environ.get('SWARM_GEMM_STREAMK','default')} dbg={os.environ.get('SWARM_GEMM_DBG','0')} "
              f"ws={int(sk)} {name}: {ms*1e3:.1f} us {2*m*n*k/ms/1e9:.0f} TFLOP/s", flush=True)
