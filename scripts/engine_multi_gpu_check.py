"""torchrun check of the engine-driven executor on N GPUs (NCCL): each rank's
stage gradients after K microbatches (no tick) equal a sequential recomputation
of exactly the visits the schedule ran; with ticks (stage all-reduce + AdamW) the
C++ driver (EngineExecutor, raw NCCL) and the Python orchestrator
(PyEngineExecutor, torch.distributed) end with the same parameters.  Prints one
line per rank; exit 1 on mismatch."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2301_11913_b200.executor import EngineExecutor, PyEngineExecutor, sequential_reference_grads  # noqa: E402
from paper_2301_11913_b200.swarm import PRESETS  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
S = int(sys.argv[1]) if len(sys.argv) > 1 else 4
tpp = int(sys.argv[2]) if len(sys.argv) > 2 else 2
lanes = int(sys.argv[3]) if len(sys.argv) > 3 else 1
# optional 4th argument "balanced": bench.py's load-balanced placement (several peers per stage,
# spread over the GPUs next to other stages' peers)
kw = {}
if len(sys.argv) > 4 and sys.argv[4] == "balanced":
    import argparse

    import bench
    layout, peer_rank, _ = bench.engine_placement(argparse.Namespace(model="tiny", micro_batch=None,
                                                                     placement="balanced"), dist.get_world_size(), S)
    kw = {"layout": layout, "peer_rank": peer_rank}
elif len(sys.argv) > 4 and sys.argv[4] == "spread":
    # every GPU hosts one peer of every stage (W peers per stage: W-rank stage communicators)
    W = dist.get_world_size()
    kw = {"layout": [W] * S, "peer_rank": [k for s in range(S) for k in range(W)]}
ex = EngineExecutor(PRESETS["tiny"], S, trainers_per_peer=tpp, seed=5, n_pool=5, lanes=lanes, **kw)
ex.run(9)
ex.finish()
torch.cuda.synchronize()
dist.barrier()
ex.flush_wgrad()
ref = sequential_reference_grads(ex)
ok = True
for pid, st in ex.stages.items():
    s = ex.stage_of_peer(pid)
    r = float((st.grads() - ref[pid]).norm() / ref[pid].norm().clamp_min(1e-30))
    ok &= r <= 1e-4
    print(f"rank {dist.get_rank()} peer {pid} stage {s}: rel {r:.3e} visits {ex.visits_local}", flush=True)
# with ticks: trains (finite loss)
ex2 = EngineExecutor(PRESETS["tiny"], S, trainers_per_peer=tpp, seed=3, lr=3e-3, n_pool=2, allreduce_period=12.0,
                     allreduce_stall=0.1, lanes=lanes, **kw)
ex2.run(40)
ex2.finish()
torch.cuda.synchronize()
print(f"rank {dist.get_rank()} ticks {ex2.ticks} steps {ex2.optimizer_steps} loss {ex2.loss_sum.item():.4f}", flush=True)
if kw:  # (the Python orchestrator has no placement option: stop at the replay check)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)
py2 = PyEngineExecutor(PRESETS["tiny"], S, trainers_per_peer=tpp, seed=3, lr=3e-3, allreduce_period=12.0,
                       allreduce_stall=0.1, lanes=lanes, tokens=ex2.pool_tok.cpu(), targets=ex2.pool_tgt.cpu())
py2.run(40)
py2.finish()
torch.cuda.synchronize()
for pid, st in ex2.stages.items():
    r = float((st.params() - py2.stages[pid].params()).norm() / py2.stages[pid].params().norm())
    ok &= r <= 1e-4
    print(f"rank {dist.get_rank()} peer {pid}: C++ driver vs Python orchestrator params after "
          f"{ex2.optimizer_steps} optimizer steps: rel {r:.3e}", flush=True)
dist.barrier()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
