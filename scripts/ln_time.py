"""LayerNorm kernel timing (configs[2] shape, bf16): 20 calls captured in a CUDA
graph so host launch cost is excluded; reports us/call and achieved GB/s
against the algorithmic bytes (fwd: read x, write y = 4 B/elem; bwd: read dy,
x, dres, write dx = 8 B/elem, plus the dgain/dbias reduction)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_11913_b200 import _lib as L, ops
from paper_2301_11913_b200.ops import _ptr, _DT
rows, cols = 2048, 2048
x = torch.randn(rows, cols, device="cuda").bfloat16()
g = torch.randn(cols, device="cuda"); b = torch.randn(cols, device="cuda")
y = torch.empty_like(x); mu = torch.empty(rows, device="cuda"); rs = torch.empty(rows, device="cuda")
dy = torch.randn_like(x); dres = torch.randn_like(x); dx = torch.empty_like(x)
dg = torch.zeros(cols, device="cuda"); db = torch.zeros(cols, device="cuda")
ws = torch.zeros(L.lib().swarm_layer_norm_backward_workspace(rows, cols), dtype=torch.uint8, device="cuda")
lib = L.lib()
def fwd(st):
    lib.swarm_layer_norm_forward(_ptr(x), _DT[x.dtype], rows, cols, _ptr(g), _ptr(b), 1e-5, _ptr(y), _ptr(mu), _ptr(rs), st)
def fwd_nogb(st):  # gain / bias omitted (1, 0): no per-row parameter loads
    lib.swarm_layer_norm_forward(_ptr(x), _DT[x.dtype], rows, cols, None, None, 1e-5, _ptr(y), _ptr(mu), _ptr(rs), st)
def bwd(st):
    lib.swarm_layer_norm_backward(_ptr(dy), _ptr(x), _DT[x.dtype], rows, cols, _ptr(g), _ptr(mu), _ptr(rs), _ptr(dres),
                                  _ptr(dx), _ptr(dg), _ptr(db), 1, _ptr(ws), st)
for name, fn, nbytes in (("fwd", fwd, 4 * rows * cols), ("fwd no gain/bias", fwd_nogb, 4 * rows * cols),
                         ("bwd", bwd, 8 * rows * cols)):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(s.cuda_stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            for _ in range(20):
                fn(s.cuda_stream)
    torch.cuda.synchronize()
    graph.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); graph.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(f"ln {name}: {us:.2f} us/call, {nbytes / us / 1e3:.0f} GB/s algorithmic", flush=True)
    # cold: every call behind a 256 MB L2 flush (the in-step case: x comes from DRAM)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    tot = 0.0
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(torch.cuda.current_stream().cuda_stream); e1.record(); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    print(f"ln {name} (L2 flushed): {tot / 20 * 1e3:.2f} us/call", flush=True)
