"""Debug: gradient replay check of the membership paths, variant by variant."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
import test_membership_gpu as T
from paper_2301_11913_b200.engine import Engine

variants = {
    "static": dict(churn=[], rebalance_period=0.0),
    "leave_only": dict(rebalance_period=0.0),
    "rebalance_only": dict(churn=[]),
    "both": dict(),
    "both_nopair": dict(),
}
for name, kw in variants.items():
    cfg = T.config_e(False, **kw)
    ex = T.make(cfg, pair_wgrad=(name != "both_nopair"))
    ex.run(10 ** 6)
    ex.finish()
    ex.flush_wgrad()
    torch.cuda.synchronize()
    c = ex.counters()
    want = T.replay_reference(ex, cfg)
    errs = {pid: round(T.rel(st.grads(), want[pid]), 6) for pid, st in ex.stages.items()}
    e = Engine(cfg, 3)
    ev = [(r.kind, round(r.time, 2), r.worker, r.stage, r.from_worker) for r in e.records() if r.kind >= 4]
    print(name, "counters", {k: c[k] for k in ("migrations", "recomputes", "visits", "completed")}, "errors", errs,
          "peers", [ex.peer_info(p) for p in range(ex.n_peers)], "events", ev[:12], flush=True)
