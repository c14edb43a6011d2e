import sys, math, ctypes as C; sys.path.insert(0, ".")
import torch
from paper_2301_11913_b200 import _lib
B,H,L,dh=4,16,512,128; d=H*dh
qkv=torch.randn(B*L,3*d,device="cuda").bfloat16(); P=torch.empty(B*H*L,L,device="cuda",dtype=torch.bfloat16)
dO=torch.randn(B*L,d,device="cuda").bfloat16(); dS=torch.empty_like(P); st=torch.cuda.current_stream().cuda_stream
f=lambda: _lib.lib().swarm_attn_scores_softmax(C.c_void_p(qkv.data_ptr()),C.c_void_p(qkv[:,d:].data_ptr()),3*d,d,B,H,L,dh,1/math.sqrt(dh),1,C.c_void_p(P.data_ptr()),st)
O=torch.randn(B*L,d,device="cuda").bfloat16()
g=lambda: _lib.lib().swarm_attn_scores_softmax_backward(C.c_void_p(dO.data_ptr()),d,C.c_void_p(qkv[:,2*d:].data_ptr()),3*d,d,C.c_void_p(O.data_ptr()),d,C.c_void_p(P.data_ptr()),B,H,L,dh,1/math.sqrt(dh),1,C.c_void_p(dS.data_ptr()),st)
for name,fn in (("fwd",f),("bwd",g)):
    for _ in range(3): fn()
    torch.cuda.synchronize(); e0,e1=torch.cuda.Event(True),torch.cuda.Event(True); e0.record()
    for _ in range(20): fn()
    e1.record(); torch.cuda.synchronize(); print(name, e0.elapsed_time(e1)/20*1e3, "us")
