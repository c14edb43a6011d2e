"""Fused cross-entropy on the configs[2] head (2048 tokens x 50304 words):
vectorised kernel time vs the algorithmic bytes (fp32 logits read, bf16 dlogits written)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2301_11913_b200 import _lib as L  # noqa: E402

rows, vocab = 2048, 50304
logits = torch.randn(rows, vocab, device="cuda") * 4
targets = torch.randint(0, vocab, (rows,), device="cuda", dtype=torch.int32)
loss = torch.zeros(1, device="cuda")
dl = torch.empty(rows, vocab, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(64 << 20, device="cuda")
st = torch.cuda.current_stream()
ts = []
for i in range(23):
    flush.fill_(float(i))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    L.check(L.lib().swarm_cross_entropy(logits.data_ptr(), targets.data_ptr(), rows, vocab, 1.0, loss.data_ptr(),
                                        dl.data_ptr(), st.cuda_stream), "ce")
    b.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
us = ts[len(ts) // 2]
by = rows * vocab * (4 + 2)
print(f"cross_entropy 2048x50304: {us:.1f} us median, {by / (us * 1e-6) / 1e9:.0f} GB/s algorithmic (L2 flushed)")
