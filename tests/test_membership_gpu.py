"""GPU: dynamic membership through the C++ driver (BASELINE configs[4]).

The engine (decision-identical to sim::run, tests/test_engine.py) emits peer
deaths, Alg. 2 rebalancing migrations and requeues; the driver executes them on
one GPU (every peer shares it; their gradients are summed locally at a tick):
  * a dead peer's queued jobs run elsewhere; a backward whose forward peer is gone
    recomputes the stage forward from the trainer's stage input (activation
    checkpointing) -- with weights fixed (no tick), every live peer's
    gradient equals the sum, over the visits it ran, of the per-microbatch stage
    gradients of a sequential replay (forward part for each forward or recompute,
    backward part for each backward);
  * a migrating peer downloads params + AdamW state from a stage-mate: with ticks,
    live replicas of a stage stay bit-identical, and training still lowers the loss.
"""
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def config_e(ticks: bool, **kw):
    """2 stages on one GPU starting imbalanced (3, 1; the last stage slowed by its head),
    periodic rebalancing, and a peer death mid-run."""
    from paper_2301_11913_b200.engine import EngineConfig
    base = dict(n_stages=2, initial_peers=[[1.0, 1.0, 1.0], [0.8]], forward_service_seconds=1.0,
                trainers_per_peer=2, allreduce_period=30.0 if ticks else 0.0, allreduce_stall=0.05 if ticks else 0.0,
                duration_seconds=400.0, bucket_seconds=50.0, churn=[(150.0, -1)], rebalance_period=40.0,
                straggler_timeout=2.0, propagation_delay=0.5, state_transfer_bytes=10 ** 9, download_bps=4e9)
    base.update(kw)
    return EngineConfig(**base)


def make(cfg, **kw):
    from paper_2301_11913_b200.executor import EngineExecutor
    from paper_2301_11913_b200.swarm import PRESETS
    return EngineExecutor(PRESETS["tiny"], cfg.n_stages, seed=3, n_pool=5, sim=cfg, **kw)


def replay_reference(ex, cfg, seed=3):
    """Per live peer: the gradient the visits it ran on its current stage object (since its last
    migration) must have accumulated, from a sequential replay of every microbatch on fresh
    replicas (weights fixed: no tick ran)."""
    import torch
    from paper_2301_11913_b200.engine import MIGRATED, START, Engine
    from paper_2301_11913_b200.stage import Stage, StageConfig
    # the visit-log position where each peer's current stage object started (its last MIGRATED)
    since, n_start = {}, 0
    for r in Engine(cfg, seed).records():
        if r.kind == START:
            n_start += 1
        elif r.kind == MIGRATED:
            since[r.worker] = n_start
    m, S = ex.m, ex.S
    reps = {}
    for s in range(S):
        cfg = StageConfig(**{**ex.stage_cfg.__dict__, "is_first": int(s == 0), "is_last": int(s == S - 1),
                             "max_slots": 1, "seed": ex.seed * 1000 + s})
        reps[s] = Stage(cfg, ex.device)
    a = [reps[0].new_wire() for _ in range(max(S - 1, 1))]
    g = [reps[0].new_wire() for _ in range(max(S - 1, 1))]
    loss = torch.zeros(1, device=ex.device)
    log = ex.visit_log
    mbs = sorted({(t, k) for t, k, s, b, p in log})
    G = {}  # (t, k, s) -> (forward part, backward part) of the stage gradient
    for t, k in mbs:
        idx = ex._pool_index(t, k)
        fwd = {}
        for s in range(S):
            st = reps[s]
            st.grads().zero_()
            inp = ex.pool_tok[idx] if s == 0 else a[s - 1]
            if s == S - 1:
                st.forward(0, inp, targets=ex.pool_tgt[idx], loss_sum=loss, loss_scale=1.0 / m.tokens)
            else:
                st.forward(0, inp, out=a[s])
            fwd[s] = st.grads().clone()
        for s in reversed(range(S)):
            st = reps[s]
            st.grads().zero_()
            st.backward(0, grad_in=None if s == S - 1 else g[s], grad_out=None if s == 0 else g[s - 1])
            G[(t, k, s)] = (fwd[s], st.grads().clone())
    torch.cuda.synchronize()
    want = {}
    last_fwd = {}  # (t, k, s) -> peer of the latest forward START
    for i, (t, k, s, b, p) in enumerate(log):
        info = ex.peer_info(p)
        counts = info["alive"] and not info["migrating"] and info["stage"] == s and i >= since.get(p, 0)
        if not b:
            last_fwd[(t, k, s)] = p
            if counts:
                want[p] = want.get(p, 0) + G[(t, k, s)][0]
        else:
            if counts:
                extra = G[(t, k, s)][0] if last_fwd.get((t, k, s)) != p else 0  # the recompute's forward part
                want[p] = want.get(p, 0) + G[(t, k, s)][1] + extra
    return want


def test_peer_death_and_migration_gradients_match_replay(cuda):
    import torch
    from paper_2301_11913_b200.engine import LEAVE, MIGRATED
    cfg = config_e(ticks=False)
    ex = make(cfg)
    ex.run(10 ** 6)  # the whole schedule (duration_seconds)
    ex.finish()
    ex.flush_wgrad()
    torch.cuda.synchronize()
    c = ex.counters()
    assert c["migrations"] >= 1, c
    assert c["recomputes"] >= 1, c  # some backward re-routed away from its forward peer
    alive = [p for p in range(ex.n_peers) if ex.peer_info(p)["alive"]]
    assert len(alive) == 3
    want = replay_reference(ex, cfg)
    for pid, st in ex.stages.items():
        assert pid in want
        e = rel(st.grads(), want[pid])
        assert e <= 1e-4, (pid, e)


def test_membership_with_ticks_keeps_replicas_identical_and_trains(cuda):
    import torch
    ex = make(config_e(ticks=True), lr=3e-3)
    curve = []
    while True:
        ex.loss_sum.zero_()
        n = ex.run(16)
        ex.finish()
        if n == 0:
            break
        curve.append(ex.loss_sum.item() / n / ex.m.tokens)
    torch.cuda.synchronize()
    c = ex.counters()
    assert c["migrations"] >= 1 and c["ticks"] > 0
    by_stage = {}
    for pid, st in ex.stages.items():
        by_stage.setdefault(ex.peer_info(pid)["stage"], []).append(st.params().clone())
    for s, ps in by_stage.items():
        for q in ps[1:]:
            assert torch.equal(q, ps[0]), f"stage {s} replicas diverged"
    assert len(curve) >= 3 and curve[-1] < curve[0] - 0.2, curve
