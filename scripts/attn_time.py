"""Attention kernel timings at configs[2]'s shape (B 4, H 16, L 512, d_head 128, causal): the forward
(P + O = P V), the score-gradient kernel of the unfused backward, and the one-kernel backward."""
import sys, math, ctypes as C; sys.path.insert(0, ".")
import torch
from paper_2301_11913_b200 import _lib
B, H, L, dh = 4, 16, 512, 128
d = H * dh
lib = _lib.lib()
ptr = lambda t: C.c_void_p(t.data_ptr())
qkv = torch.randn(B * L, 3 * d, device="cuda").bfloat16()
P = torch.zeros(B * H * L, L, device="cuda", dtype=torch.bfloat16)
O = torch.zeros(B * L, d, device="cuda", dtype=torch.bfloat16)
dO = torch.randn(B * L, d, device="cuda").bfloat16()
dS = torch.zeros_like(P)
dqkv = torch.empty_like(qkv)
ws = torch.zeros(lib.swarm_attn_backward_workspace(B, H, L, dh), device="cuda", dtype=torch.uint8)
st = torch.cuda.current_stream().cuda_stream
sc = 1 / math.sqrt(dh)
fwd = lambda: lib.swarm_attn_forward_pv(ptr(qkv), ptr(qkv[:, d:]), ptr(qkv[:, 2 * d:]), 3 * d, d, B, H, L, dh, sc, 1,
                                        ptr(P), ptr(O), d, st)
sgrad = lambda: lib.swarm_attn_scores_softmax_backward(ptr(dO), d, ptr(qkv[:, 2 * d:]), 3 * d, d, ptr(O), d, ptr(P), B,
                                                       H, L, dh, sc, 1, ptr(dS), st)
bwd = lambda: lib.swarm_attn_backward(ptr(dO), d, ptr(qkv), 3 * d, 3 * d, d, 2 * d, ptr(O), d, ptr(P), B, H, L, dh, sc,
                                      1, ptr(dqkv), 3 * d, d, 2 * d, ptr(ws), st)
lse = torch.zeros(B * H * L, device="cuda")
fwd_lse = lambda: lib.swarm_attn_forward_lse(ptr(qkv), ptr(qkv[:, d:]), ptr(qkv[:, 2 * d:]), 3 * d, d, B, H, L, dh, sc,
                                             1, ptr(lse), ptr(O), d, st)
bwd_lse = lambda: lib.swarm_attn_backward_lse(ptr(dO), d, ptr(qkv), 3 * d, 3 * d, d, 2 * d, ptr(O), d, ptr(lse), B, H,
                                              L, dh, sc, 1, ptr(dqkv), 3 * d, d, 2 * d, ptr(ws), st)
flush = torch.empty(256 << 20, device="cuda", dtype=torch.uint8)
for name, fn in (("forward_pv", fwd), ("score_grad (unfused bwd, 1 of 4 launches)", sgrad), ("backward_fused", bwd),
                 ("forward_lse (no P stored)", fwd_lse), ("backward_lse (P recomputed)", bwd_lse)):
    for _ in range(3):
        assert fn() == 0, _lib.last_error()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    print(f"{name}: {tot / 20 * 1e3:.1f} us (L2 flushed)")
