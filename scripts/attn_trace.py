"""Per-CTA timeline of the chunked attention kernels (SWARM_ATTN_TRACE=1):
start offset, prologue, statistics pass, output pass, exit — by query block mt."""
import ctypes as C, math, os, sys
os.environ["SWARM_ATTN_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2301_11913_b200 import _lib
lib = _lib.lib()
lib.swarm_debug_attn_trace.argtypes = [C.c_void_p, C.c_int]
B, H, L, dh = 4, 16, 512, 128
d = H * dh
qkv = torch.randn(B * L, 3 * d, device="cuda").bfloat16()
P = torch.zeros(B * H * L, L, device="cuda", dtype=torch.bfloat16)
dO = torch.randn(B * L, d, device="cuda").bfloat16(); O = torch.randn(B * L, d, device="cuda").bfloat16()
dS = torch.zeros_like(P); st = torch.cuda.current_stream().cuda_stream
f = lambda: lib.swarm_attn_scores_softmax(C.c_void_p(qkv.data_ptr()), C.c_void_p(qkv[:, d:].data_ptr()), 3 * d, d, B, H, L, dh,
                                          C.c_float(1 / math.sqrt(dh)), 1, C.c_void_p(P.data_ptr()), st)
g = lambda: lib.swarm_attn_scores_softmax_backward(C.c_void_p(dO.data_ptr()), d, C.c_void_p(qkv[:, 2 * d:].data_ptr()), 3 * d, d,
                                                   C.c_void_p(O.data_ptr()), d, C.c_void_p(P.data_ptr()), B, H, L, dh,
                                                   C.c_float(1 / math.sqrt(dh)), 1, C.c_void_p(dS.data_ptr()), st)
lse = torch.zeros(B * H * L, device="cuda")
h = lambda: lib.swarm_attn_forward_lse(C.c_void_p(qkv.data_ptr()), C.c_void_p(qkv[:, d:].data_ptr()),
                                       C.c_void_p(qkv[:, 2 * d:].data_ptr()), 3 * d, d, B, H, L, dh,
                                       C.c_float(1 / math.sqrt(dh)), 1, C.c_void_p(lse.data_ptr()),
                                       C.c_void_p(O.data_ptr()), d, st)
nz, nqb = B * H, L // 128
n = nz * nqb
for name, fn in (("fwd", f), ("bwd", g), ("fwd_lse (P V fused)", h)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    buf = np.zeros((n, 6), np.uint64)
    assert lib.swarm_debug_attn_trace(buf.ctypes.data, n) == 0
    t = buf[:, :5].astype(np.int64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3  # us
    print(f"{name}: kernel span {rel[:, 4].max():.2f} us, CTAs {n}, distinct SMs {len(set(buf[:, 5].tolist()))}")
    for mt in range(nqb - 1, -1, -1):
        idx = [i for i in range(n) if nqb - 1 - i // nz == mt]
        r = rel[idx]
        print(f"  mt={mt}: start {r[:,0].mean():6.2f} (max {r[:,0].max():6.2f})  prologue {np.mean(r[:,1]-r[:,0]):5.2f}"
              f"  stats {np.mean(r[:,2]-r[:,1]):5.2f}  out {np.mean(r[:,3]-r[:,2]):5.2f}  exit {np.mean(r[:,4]-r[:,3]):5.2f}"
              f"  end {r[:,4].mean():6.2f} (max {r[:,4].max():6.2f})")
