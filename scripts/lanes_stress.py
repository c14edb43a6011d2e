"""Race check for lanes: many trainers, two lanes per peer, several seeds; every
peer's gradient must equal the sequential replay of its scheduled visits."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2301_11913_b200.executor import EngineExecutor, sequential_reference_grads  # noqa: E402
from paper_2301_11913_b200.swarm import PRESETS  # noqa: E402

worst = 0.0
for seed in range(6):
    for S, tpp in ((2, 4), (4, 3), (3, 2)):
        ex = EngineExecutor(PRESETS["tiny"], S, trainers_per_peer=tpp, seed=seed, n_pool=6, lanes=2)
        ex.run(12)
        ex.finish()
        ex.flush_wgrad()
        torch.cuda.synchronize()
        ref = sequential_reference_grads(ex)
        for pid, st in ex.stages.items():
            r = float((st.grads() - ref[pid]).norm() / ref[pid].norm())
            worst = max(worst, r)
        del ex
print(f"lanes stress: worst relative gradient error {worst:.3e}")
sys.exit(0 if worst <= 1e-4 else 1)
