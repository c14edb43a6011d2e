"""torchrun check of dynamic membership over NCCL (config E's schedule on N GPUs, one peer per
GPU: 2 stages starting (N-1, 1), Alg. 2 rebalancing, a peer death): with weights fixed every live
peer's gradient equals the sequential replay of the visits it ran (recompute inputs and state
downloads cross GPUs); with ticks the live replicas of each stage end bit-identical across GPUs.
Prints one line per rank; exit 1 on mismatch."""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_membership_gpu as T  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
W, rank = dist.get_world_size(), dist.get_rank()
ok = True
peers = [[1.0] * max(3, W - 1), [0.8]]  # 4 peers on 2 GPUs share them; one per GPU from 4
cfg = T.config_e(False, initial_peers=peers)
ex = T.make(cfg)
ex.run(10 ** 6)
ex.finish()
ex.flush_wgrad()
torch.cuda.synchronize()
c = ex.counters()
want = T.replay_reference(ex, cfg)
for pid, st in ex.stages.items():
    e = T.rel(st.grads(), want[pid])
    ok &= e <= 1e-4
    print(f"rank {rank} peer {pid} stage {ex.peer_info(pid)['stage']}: grad vs replay rel {e:.2e}; migrations "
          f"{c['migrations']} recomputes {c['recomputes']} state bytes {c['state_bytes']}", flush=True)
del ex
dist.barrier()
ex = T.make(T.config_e(True, initial_peers=peers), lr=3e-3)
ex.run(10 ** 6)
ex.finish()
torch.cuda.synchronize()
mine = {pid: (ex.peer_info(pid)["stage"], st.params().clone()) for pid, st in ex.stages.items()}
gathered = [None] * W
dist.all_gather_object(gathered, {pid: (s, p.cpu()) for pid, (s, p) in mine.items()})
if rank == 0:
    by_stage = {}
    for g in gathered:
        for pid, (s, p) in g.items():
            by_stage.setdefault(s, []).append((pid, p))
    for s, ps in by_stage.items():
        same = all(torch.equal(p, ps[0][1]) for _, p in ps[1:])
        ok &= same
        print(f"stage {s}: live replicas {[pid for pid, _ in ps]} bit-identical across GPUs: {same}", flush=True)
    print(f"ticks {ex.counters()['ticks']} migrations {ex.counters()['migrations']} loss {ex.loss_sum.item():.1f}",
          flush=True)
okt = torch.tensor([1 if ok else 0], device="cuda")
dist.all_reduce(okt, op=dist.ReduceOp.MIN)
dist.barrier()
dist.destroy_process_group()
sys.exit(0 if okt.item() else 1)
