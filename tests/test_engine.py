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
