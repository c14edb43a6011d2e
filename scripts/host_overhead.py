"""Is the 1-GPU pipeline host-bound?  Compare the CPU time to enqueue one
optimizer step (no sync) with the GPU time of the step, with and without
GEMM profiling events."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_11913_b200 import _lib
from paper_2301_11913_b200.swarm import PRESETS, SwarmPipeline, synthetic_batch

model = sys.argv[1] if len(sys.argv) > 1 else "C"
m = PRESETS[model]
for prof in (False, True):
    pipe = SwarmPipeline(m, 4, n_microbatches=8, seed=1, profile=prof)
    tok, tgt = synthetic_batch(m, 8, 7, "cuda")
    for _ in range(2):
        pipe.step(tok, tgt)
    torch.cuda.synchronize()
    n0 = _lib.lib().swarm_launch_count()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); t0 = time.perf_counter()
    pipe.step(tok, tgt)
    t_enq = time.perf_counter() - t0
    e1.record(); torch.cuda.synchronize(); t_all = time.perf_counter() - t0
    n = _lib.lib().swarm_launch_count() - n0
    print(f"profile={prof}: launches {n}, enqueue {t_enq*1e3:.1f} ms ({t_enq/n*1e6:.2f} us/launch), "
          f"gpu {e0.elapsed_time(e1):.1f} ms, wall {t_all*1e3:.1f} ms", flush=True)
    if prof:
        print("gemm ms/flops/n", pipe.profile_read())
    del pipe
    torch.cuda.empty_cache()
