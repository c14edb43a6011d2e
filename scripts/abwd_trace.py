"""Per-CTA timeline of the fused attention backward (SWARM_ATTN_BWD_DBG=4): row 0's timestamps at the
pipeline points (csrc/attn_bwd.cu TR marks), in us after the CTA's entry."""
import os, sys, math, ctypes as C; sys.path.insert(0, ".")
os.environ.setdefault("SWARM_ATTN_BWD_DBG", "4")
import numpy as np, torch
from paper_2301_11913_b200 import _lib
B, H, L, dh = 4, 16, 512, 128
d = H * dh
lib = _lib.lib()
ptr = lambda t: C.c_void_p(t.data_ptr())
qkv = torch.randn(B * L, 3 * d, device="cuda").bfloat16()
P = torch.zeros(B * H * L, L, device="cuda", dtype=torch.bfloat16)
O = torch.zeros(B * L, d, device="cuda", dtype=torch.bfloat16)
dO = torch.randn(B * L, d, device="cuda").bfloat16()
dqkv = torch.empty_like(qkv)
ws = torch.zeros(lib.swarm_attn_backward_workspace(B, H, L, dh), device="cuda", dtype=torch.uint8)
st = torch.cuda.current_stream().cuda_stream
sc = 1 / math.sqrt(dh)
lse = torch.zeros(B * H * L, device="cuda")
RECOMP = os.environ.get("ABWD_LSE", "1") == "1"
if RECOMP:
    lib.swarm_attn_forward_lse(ptr(qkv), ptr(qkv[:, d:]), ptr(qkv[:, 2 * d:]), 3 * d, d, B, H, L, dh, sc, 1, ptr(lse), ptr(O), d, st)
else:
    lib.swarm_attn_forward_pv(ptr(qkv), ptr(qkv[:, d:]), ptr(qkv[:, 2 * d:]), 3 * d, d, B, H, L, dh, sc, 1, ptr(P), ptr(O), d, st)
for _ in range(3):
    if RECOMP:
        assert lib.swarm_attn_backward_lse(ptr(dO), d, ptr(qkv), 3 * d, 3 * d, d, 2 * d, ptr(O), d, ptr(lse), B, H, L, dh, sc, 1,
                                           ptr(dqkv), 3 * d, d, 2 * d, ptr(ws), st) == 0
    else:
        assert lib.swarm_attn_backward(ptr(dO), d, ptr(qkv), 3 * d, 3 * d, d, 2 * d, ptr(O), d, ptr(P), B, H, L, dh, sc, 1,
                                       ptr(dqkv), 3 * d, d, 2 * d, ptr(ws), st) == 0
torch.cuda.synchronize()
tr = np.zeros((256, 96), dtype=np.uint64)
lib.swarm_debug_abwd_trace.argtypes = [C.c_void_p, C.c_int]
assert lib.swarm_debug_abwd_trace(tr.ctypes.data, 256) == 0
n = 128
t0 = tr[:n, 0].astype(np.int64)
rel = (tr[:n].astype(np.int64) - t0[:, None]) / 1e3
print("launch spread (entry, us):", (t0.max() - t0.min()) / 1e3)
print("setup:", np.median(rel[:, 1]), " rows done:", np.median(rel[:, 6]), " exit:", np.median(rel[:, 7]))
for c in (0, 1, 64, 127):
    print(f"CTA {c}: setup {rel[c,1]:.1f}")
    for blk in range(5):
        v = rel[c, 8 + 9 * blk:17 + 9 * blk]
        print(f"   blk {blk}: rows s_full {v[6]:.1f} p_ready {v[4]:.1f} | mma p_seen {v[7]:.1f} | rows mma12 {v[0]:.1f} ds {v[1]:.1f} | mma34 issued {v[5]:.1f} | dQ-rows mma34 {v[2]:.1f} reduced {v[3]:.1f}")
    print(f"   kb0 acc {rel[c,2]:.1f} out {rel[c,3]:.1f}  kb1 acc {rel[c,4]:.1f} out {rel[c,5]:.1f}  end {rel[c,6]:.1f} exit {rel[c,7]:.1f}")
