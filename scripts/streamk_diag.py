"""Stream-K diagnosis: time a few GEMM shapes with stream-K on/off under the
SWARM_GEMM_DBG value the caller sets (8 = no fixup handshake, 16 = no waits)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_11913_b200 import _lib as L, ops
shapes = {"o 2048^3": (2048, 2048, 2048), "ffn1": (2048, 8192, 2048), "ffn2": (2048, 2048, 8192),
          "qkv": (2048, 6144, 2048), "logits": (2048, 50304, 2048)}
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
        print(f"dbg={os.environ.get('SWARM_GEMM_DBG','0')} sk={int(sk)} {name}: {ms*1e3:.1f} us "
              f"{2*m*n*k/ms/1e9:.0f} TFLOP/s", flush=True)
