"""Engine-driven executor schedule (csrc/engine.cpp) against the
reference's own discrete-event engine (P/src/sim.cpp sim::run, compiled
unmodified into oracle/_ref): identical dispatched / completed counts and
per-bucket throughput on the same SimConfig and seed, plus the structural
invariants the GPU executor relies on."""
import ctypes as C
import random

import pytest

import oracle as O
from paper_2301_11913_b200.engine import ALLREDUCE, DONE, HOP, START, Engine, EngineConfig

needs_ref = pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built (needs /root/reference)")


def ref_run(cfg: EngineConfig, seed: int):
    d, c, nbo = C.c_uint64(), C.c_uint64(), C.c_size_t()
    b = (C.c_double * 4096)()
    rc = O.ref.ref_sim_run(cfg.to_reference_json().encode(), seed, C.byref(d), C.byref(c), b, 4096, C.byref(nbo))
    assert rc == 0
    return {"dispatched": d.value, "completed": c.value, "buckets": list(b)[: nbo.value]}


def ours(cfg: EngineConfig, seed: int):
    e = Engine(cfg, seed)
    recs = list(e.records())
    return e.summary(), recs


def random_cfg(rng: random.Random) -> EngineConfig:
    S = rng.randint(1, 6)
    peers = [[rng.choice([1.0, 1.0, 0.5, 1.7, rng.uniform(0.3, 2.0)]) for _ in range(rng.randint(1, 4))]
             for _ in range(S)]
    ar = rng.random() < 0.5
    return EngineConfig(n_stages=S, initial_peers=peers, forward_service_seconds=rng.uniform(0.05, 3.0),
                        backward_multiplier=rng.choice([2.0, 2.0, 1.5, 3.0]),
                        trainers_per_peer=rng.randint(1, 3),
                        allreduce_period=rng.uniform(5, 60) if ar else 0.0,
                        allreduce_stall=rng.uniform(0.1, 5) if ar else 0.0,
                        duration_seconds=rng.uniform(100, 1500), bucket_seconds=rng.choice([10.0, 60.0, 37.5]))


@needs_ref
@pytest.mark.parametrize("case", range(40))
def test_engine_matches_reference_sim(case):
    rng = random.Random(1000 + case)
    cfg = random_cfg(rng)
    seed = rng.randrange(2 ** 63)
    got, _ = ours(cfg, seed)
    exp = ref_run(cfg, seed)
    assert got["dispatched"] == exp["dispatched"]
    assert got["completed"] == exp["completed"]
    assert got["buckets"] == exp["buckets"]


@needs_ref
def test_engine_matches_reference_paper_layout():
    """configs[2]'s 4 stages x 2 peers with the measured B200 visit time scale."""
    cfg = EngineConfig(n_stages=4, initial_peers=[[1.0, 1.0]] * 4, forward_service_seconds=6.3e-3,
                       trainers_per_peer=1, allreduce_period=0.5, allreduce_stall=0.01,
                       duration_seconds=30.0, bucket_seconds=1.0)
    for seed in (0, 1, 2026):
        got, _ = ours(cfg, seed)
        assert {k: got[k] for k in ("dispatched", "completed", "buckets")} == ref_run(cfg, seed)


@pytest.mark.parametrize("case", range(6))
def test_schedule_invariants(case):
    """What the executor relies on: per trainer, visits go forward 0..S-1 then
    backward S-1..0 on the recorded route; each HOP names the worker that produced
    its input; each worker serves its queue FIFO (START in HOP order); records are
    in non-decreasing event time; every HOP precedes its START."""
    rng = random.Random(case)
    cfg = random_cfg(rng)
    _, recs = ours(cfg, rng.randrange(2 ** 32))
    S = cfg.n_stages
    stages = cfg.worker_stages()
    pending = {}          # worker -> FIFO of (trainer, backward)
    route = {}            # trainer -> forward route
    last = {}             # trainer -> (stage, backward, worker) of the last hop
    t_prev = -1.0
    n_start = 0
    for r in recs:
        t = r.time if r.kind != START else None
        if t is not None:
            assert t >= t_prev
            t_prev = t
        if r.kind == HOP:
            assert stages[r.worker] == r.stage
            prev = last.get(r.trainer)
            if prev is None or (prev[0] == 0 and prev[1]):          # new microbatch
                assert r.from_worker == -1 and r.stage == 0 and not r.backward
                route[r.trainer] = [None] * S
            else:
                assert r.from_worker == prev[2]
                ps, pb = prev[0], prev[1]
                exp = (ps + 1, False) if (not pb and ps + 1 < S) else ((ps, True) if not pb else (ps - 1, True))
                assert (r.stage, bool(r.backward)) == exp
            if r.backward:
                assert route[r.trainer][r.stage] == r.worker   # backward retraces the forward route
            else:
                route[r.trainer][r.stage] = r.worker
            last[r.trainer] = (r.stage, bool(r.backward), r.worker)
            pending.setdefault(r.worker, []).append((r.trainer, bool(r.backward)))
        elif r.kind == START:
            n_start += 1
            assert pending[r.worker].pop(0) == (r.trainer, bool(r.backward))
            assert r.end_time > r.time
        elif r.kind == DONE:
            assert last[r.trainer][:2] == (0, True)
        else:
            assert r.kind == ALLREDUCE
    assert n_start > 0


def test_engine_config_errors():
    from paper_2301_11913_b200._swarmsim_b200 import ConfigError
    with pytest.raises(ConfigError):
        Engine(EngineConfig(n_stages=2, initial_peers=[[1.0], []]), 0)
    with pytest.raises(ConfigError):
        Engine(EngineConfig(n_stages=1, initial_peers=[[1.0]], forward_service_seconds=0.0), 0)
    with pytest.raises(ConfigError):
        Engine(EngineConfig(n_stages=1, initial_peers=[[1.0]], trainers_per_peer=0), 0)


# --------------------------------------------------------------------------- churn + rebalancing
def ref_run_churn(cfg: EngineConfig, seed: int):
    import json
    counts = (C.c_uint64 * 4)()
    nbo = C.c_size_t()
    b = (C.c_double * 4096)()
    log = C.create_string_buffer(1 << 22)
    ts = (C.c_double * max(len(cfg.churn), 1))(*[t for t, _ in cfg.churn])
    ds = (C.c_int64 * max(len(cfg.churn), 1))(*[d for _, d in cfg.churn])
    rc = O.ref.ref_sim_run_churn(cfg.to_reference_json().encode(), ts, ds, len(cfg.churn), seed, counts, b, 4096,
                                 C.byref(nbo), log, len(log))
    assert rc == 0
    events = []
    for line in log.value.decode().splitlines():
        j = json.loads(line)
        e = j.get("event")
        if e == "peer_join":
            events.append(("join", j["t"], j["peer"], j["stage"]))
        elif e in ("peer_leave", "migration_aborted"):
            events.append(("leave", j["t"], j["peer"], j["stage"], int(e == "migration_aborted")))
        elif e == "rebalance_decision":
            mover = j["mover"] if j["mover"] is not None else -1
            events.append(("rebalance", j["t"], j["from"], j["to"], mover, int(bool(j.get("skipped", False)))))
        elif e == "migration_complete":
            events.append(("migrated", j["t"], j["peer"], j["stage"]))
    return {"dispatched": counts[0], "completed": counts[1], "requeued": counts[2], "abandoned": counts[3],
            "buckets": list(b)[: nbo.value], "events": events}


def our_events(recs):
    from paper_2301_11913_b200.engine import JOIN, LEAVE, MIGRATED, REBALANCE
    out = []
    for r in recs:
        if r.kind == JOIN:
            out.append(("join", r.time, r.worker, r.stage))
        elif r.kind == LEAVE:
            out.append(("leave", r.time, r.worker, r.stage, r.backward))
        elif r.kind == REBALANCE:
            out.append(("rebalance", r.time, r.from_worker, r.stage, r.worker, r.backward))
        elif r.kind == MIGRATED:
            out.append(("migrated", r.time, r.worker, r.stage))
    return out


def random_churn_cfg(rng: random.Random) -> EngineConfig:
    cfg = random_cfg(rng)
    n0 = sum(len(p) for p in cfg.initial_peers)
    dur = cfg.duration_seconds
    cfg.churn = sorted((rng.uniform(0, dur), rng.choice([-1, -1, -2, 1, 2, -3])) for _ in range(rng.randint(1, 6 + n0)))
    if rng.random() < 0.8:
        cfg.rebalance_period = rng.uniform(0.05, 0.4) * dur
        cfg.straggler_timeout = rng.choice([5.0, rng.uniform(0.1, 20.0)])
        cfg.propagation_delay = rng.choice([1.0, rng.uniform(0.0, 5.0)])
        cfg.announce_ttl = rng.choice([300.0, rng.uniform(10.0, 400.0)])
        cfg.state_transfer_bytes = rng.randint(10 ** 6, 10 ** 10)
        cfg.download_bps = rng.choice([500e6, rng.uniform(1e8, 1e11)])
    return cfg


@needs_ref
@pytest.mark.parametrize("case", range(60))
def test_engine_with_churn_and_rebalancing_matches_reference_sim(case):
    """The full engine (churn from a trace, peer leave / join, requeues, starvation,
    Alg. 2 rebalancing over the registry with propagation delay / TTL / straggler
    timeout, migration downtime) against the unmodified sim::run: identical counters,
    per-bucket throughput, and membership + rebalance-decision log."""
    rng = random.Random(5000 + case)
    cfg = random_churn_cfg(rng)
    seed = rng.randrange(2 ** 63)
    e = Engine(cfg, seed)
    recs = list(e.records())
    got = e.summary()
    exp = ref_run_churn(cfg, seed)
    for k in ("dispatched", "completed", "requeued", "abandoned"):
        assert got[k] == exp[k], k
    assert got["buckets"] == exp["buckets"]
    ours_ev = our_events(recs)
    assert len(ours_ev) == len(exp["events"])
    for a, b in zip(ours_ev, exp["events"]):
        assert a[0] == b[0] and a[2:] == b[2:], (a, b)
        assert abs(a[1] - b[1]) <= 1e-9 * max(1.0, abs(b[1])), (a, b)


@needs_ref
def test_engine_config_e_failure_and_rebalance_matches_reference():
    """BASELINE configs[4]'s schedule: 2 stages x 4 GPUs starting imbalanced (3, 1), the
    last stage slowed by its LM head, periodic Alg. 2 rebalancing, one peer removed
    mid-run: the same decisions (mover, stages, times) as sim::run, and a migration happens."""
    cfg = EngineConfig(n_stages=2, initial_peers=[[1.0, 1.0, 1.0], [0.8]], forward_service_seconds=1.0,
                       trainers_per_peer=2, allreduce_period=100.0, allreduce_stall=0.05, duration_seconds=3000.0,
                       bucket_seconds=100.0, churn=[(1500.0, -1)], rebalance_period=200.0, straggler_timeout=5.0,
                       propagation_delay=1.0, state_transfer_bytes=6 * 50_331_648 * 8, download_bps=8 * 450e9)
    e = Engine(cfg, 7)
    recs = list(e.records())
    exp = ref_run_churn(cfg, 7)
    assert our_events(recs) == exp["events"] or all(
        a[0] == b[0] and a[2:] == b[2:] for a, b in zip(our_events(recs), exp["events"]))
    assert any(ev[0] == "migrated" for ev in exp["events"])
    assert any(ev[0] == "leave" for ev in exp["events"])
