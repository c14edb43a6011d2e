"""Training-curve comparison on one GPU: the synchronous GPipe step
(SwarmPipeline) and the asynchronous engine-driven pipeline (EngineExecutor)
train the same model on the same 8-microbatch token pool (next-token targets),
AdamW at the same learning rate, one optimizer step per stage per 32 microbatches
in both.  Prints the mean per-token loss of every 32-microbatch window."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2301_11913_b200.engine import Engine, EngineConfig  # noqa: E402
from paper_2301_11913_b200.executor import EngineExecutor  # noqa: E402
from paper_2301_11913_b200.swarm import PRESETS, SwarmPipeline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="tiny")
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--lr", type=float, default=1e-3)
ap.add_argument("--out", default=None)
a = ap.parse_args()
m = PRESETS[a.model]
S, M, POOL = 4, 32, 8
g = torch.Generator().manual_seed(5)
pool = torch.randint(0, m.vocab, (POOL, m.tokens), generator=g, dtype=torch.int32)
tgt = torch.roll(pool, -1, dims=1)
dev = torch.device("cuda")

# synchronous: each step = the 8 pool microbatches x 4
sync = SwarmPipeline(m, S, n_microbatches=M, seed=2, lr=a.lr)
tok_b = pool.repeat(M // POOL, 1).to(dev)
tgt_b = tgt.repeat(M // POOL, 1).to(dev)
sync_curve = []
for _ in range(a.steps):
    sync.loss_sum.zero_()
    sync.step(tok_b, tgt_b)
    sync_curve.append(sync.loss_sum.item() / (M * m.tokens))
del sync
torch.cuda.synchronize()

# asynchronous: tick every 32 completions of the schedule
horizon = 400.0 * M * 3
cal = Engine(EngineConfig(n_stages=S, initial_peers=[[1.0]] * S, trainers_per_peer=2, duration_seconds=horizon,
                          bucket_seconds=horizon / 8), seed=2)
while cal.next(4096):
    pass
period = M * horizon / cal.summary()["completed"]
ex = EngineExecutor(m, S, trainers_per_peer=2, seed=2, lr=a.lr, allreduce_period=period, allreduce_stall=0.01,
                    tokens=pool, targets=tgt)
async_curve = []
for _ in range(a.steps):
    ex.loss_sum.zero_()
    n = ex.run(M)
    ex.finish()
    async_curve.append(ex.loss_sum.item() / (n * m.tokens))
res = {"model": a.model, "lr": a.lr, "microbatches_per_window": M, "sync_gpipe": sync_curve,
       "async_engine": async_curve, "optimizer_steps_async_per_stage": ex.optimizer_steps / S}
print(json.dumps(res))
if a.out:
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
