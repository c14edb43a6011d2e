"""Kernel-boundary cost on this GPU: 200 back-to-back launches captured in a CUDA
graph of (a) a 1-thread spin(0) kernel (no PDL attribute) and (b) a 1-row
LayerNorm (PDL attribute when SWARM_PDL=1), and of (c) the attention forward
kernel; us per launch."""
import ctypes as C, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_11913_b200 import _lib as L
from paper_2301_11913_b200.ops import _ptr, _DT
lib = L.lib()
x = torch.randn(1, 2048, device="cuda").bfloat16(); y = torch.empty_like(x)
mu = torch.empty(1, device="cuda"); rs = torch.empty(1, device="cuda")
B, H, Lq, dh = 4, 16, 512, 128; d = H * dh
qkv = torch.randn(B * Lq, 3 * d, device="cuda").bfloat16(); P = torch.zeros(B * H * Lq, Lq, device="cuda", dtype=torch.bfloat16)
cases = {
    "spin(0), no PDL": lambda st: lib.swarm_gpu_spin(0, st),
    "LayerNorm 1 row": lambda st: lib.swarm_layer_norm_forward(_ptr(x), _DT[x.dtype], 1, 2048, None, None, 1e-5, _ptr(y), _ptr(mu), _ptr(rs), st),
    "attention fwd (4x16x512, causal)": lambda st: lib.swarm_attn_scores_softmax(C.c_void_p(qkv.data_ptr()), C.c_void_p(qkv[:, d:].data_ptr()), 3 * d, d, B, H, Lq, dh, C.c_float(1 / math.sqrt(dh)), 1, C.c_void_p(P.data_ptr()), st),
}
for name, fn in cases.items():
    s = torch.cuda.Stream()
    n = 200 if "attention" not in name else 40
    with torch.cuda.stream(s):
        fn(s.cuda_stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                fn(s.cuda_stream)
    torch.cuda.synchronize(); g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    print(f"PDL={os.environ.get('SWARM_PDL', '0')} {name}: {e0.elapsed_time(e1) / n * 1e3:.2f} us/launch", flush=True)
