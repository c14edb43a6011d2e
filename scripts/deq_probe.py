"""Dequantize (K2) against write-dominated HBM references on the 1 GiB bench
tensor: torch fill_ (write only) and a read-N/write-4N int8->fp32 cast."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2301_11913_b200 import ops  # noqa: E402

N = 1 << 28
codes = torch.randint(-127, 128, (N,), dtype=torch.int8, device="cuda")
scales = torch.rand(N // 4096, device="cuda") + 0.5
out = torch.empty(N, dtype=torch.float32, device="cuda")


def t(fn, reps=30):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


for name, fn, by in [("fill_ f32 (write 4N)", lambda: out.fill_(1.0), 4 * N),
                     ("int8->f32 cast copy (read N, write 4N)", lambda: out.copy_(codes), 5 * N),
                     ("k_dequant_blocks (read N + N/1024, write 4N)",
                      lambda: ops.dequantize(codes, scales, 4096, torch.float32, out=out), 5 * N + N // 1024)]:
    s = t(fn)
    print(f"{name}: {s * 1e6:.1f} us  {by / s / 1e9:.0f} GB/s", flush=True)
