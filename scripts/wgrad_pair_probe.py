"""Would pairing microbatches in the weight-gradient GEMMs pay?  Time the fp32
reduce-add wgrad of two microbatches as two K=2048 GEMMs vs one K=4096 GEMM, with
the gradient arena spread over > L2 (each layer's arena is 200 MB in configs[2])."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_11913_b200 import _lib as L, ops
T, d, F = 2048, 2048, 8192
shapes = {"ffn2.wgrad": (d, F), "ffn1.wgrad": (F, d), "o.wgrad": (d, d), "qkv.wgrad": (3 * d, d)}
big = torch.zeros(64 << 20, device="cuda")  # 256 MB scratch to evict L2 between launches
for name, (M, N) in shapes.items():
    dy = torch.randn(2 * T, M, device="cuda").bfloat16()
    x = torch.randn(2 * T, N, device="cuda").bfloat16()
    acc = torch.zeros(M, N, device="cuda")
    def two():
        ops.gemm(dy[:T], x[:T], a_t=True, b_t=True, epilogue=L.EPI_ACCUM_F32, out=acc)
        ops.gemm(dy[T:], x[T:], a_t=True, b_t=True, epilogue=L.EPI_ACCUM_F32, out=acc)
    def one():
        ops.gemm(dy, x, a_t=True, b_t=True, epilogue=L.EPI_ACCUM_F32, out=acc)
    for label, fn in (("2 x K=2048", two), ("1 x K=4096", one)):
        for _ in range(3): fn()
        tot = 0.0
        for _ in range(10):
            big.add_(1.0)  # flush L2
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        ms = tot / 10
        print(f"{name:11s} {label}: {ms*1e3:7.1f} us  {2*M*N*2*T/ms/1e9:7.0f} TFLOP/s", flush=True)
