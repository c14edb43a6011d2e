"""torchrun probe: steady tokens/s of static 2-stage layouts of the configs[2] block (one peer per GPU,
the head stage slowed by its FLOP ratio in the engine), through the C++ driver."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_2301_11913_b200.engine import EngineConfig
from paper_2301_11913_b200.executor import EngineExecutor
from paper_2301_11913_b200.swarm import PRESETS
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
W = dist.get_world_size()
m = PRESETS["C"]
head = 1.0 + m.vocab * m.d_model / (m.layers_per_stage * m.params_per_layer())
fwd = float(os.environ.get("FWD", "6.3e-3"))
for layout in ([3, 1], [2, 2], [1, 3]):
    peers = [[1.0] * layout[0], [1.0 / head] * layout[1]]
    cfg = EngineConfig(n_stages=2, initial_peers=peers, forward_service_seconds=fwd, trainers_per_peer=2,
                       allreduce_period=0.5, allreduce_stall=1e-3, duration_seconds=1e9, bucket_seconds=1e8)
    ex = EngineExecutor(m, 2, seed=1, lr=1e-4, sim=cfg, lanes=int(os.environ.get("LANES", "2")))
    ex.run(64)
    ex.finish()
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    n = ex.run(128)
    ex.finish()
    torch.cuda.synchronize()
    dist.barrier()
    dt = time.perf_counter() - t0
    if dist.get_rank() == 0:
        print(f"layout {layout} fwd {fwd}: {n * m.tokens / dt:.0f} tokens/s ({n} mb in {dt:.2f} s)", flush=True)
    ex.close()
    del ex
    torch.cuda.empty_cache()
dist.destroy_process_group()
