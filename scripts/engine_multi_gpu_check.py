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
ex = EngineExecutor(PRESETS["tiny"], S, trainers_per_peer=tpp, seed=5, n_pool=5, lanes=lanes)
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
                     allreduce_stall=0.1, lanes=lanes)
ex2.run(40)
ex2.finish()
torch.cuda.synchronize()
print(f"rank {dist.get_rank()} ticks {ex2.ticks} steps {ex2.optimizer_steps} loss {ex2.loss_sum.item():.4f}", flush=True)
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
