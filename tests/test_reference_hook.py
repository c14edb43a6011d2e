"""The reference Engine drives the B200 executor through one additive hook.

oracle/hook_patch.py inserts one `swarm_hook_emit(...)` call at each record point of the
UNMODIFIED reference engine (start_service, dispatch_current, completion, AllReduceTick,
kill_worker, on_peer_join, begin_migration, on_migration_complete; P/src/sim.cpp) and
oracle/hook_shim.cpp forwards each record to a C callback (oracle/_ref/libswarmsim_hooked.so).
  * CPU: the hooked reference emits exactly csrc/engine.cpp's records, on random churn /
    rebalancing configurations (so the executor sees the same work from either engine);
  * GPU: with swarm_driver_on_record as the callback, the reference's own sim::run drives the
    C++ driver (no Python per record) through peer death, migration and recompute, and every
    live peer's gradient equals the sequential replay of the visits it ran.
"""
import ctypes as C
import random

import pytest

import oracle as O

needs_hooked = pytest.mark.skipif(O.hooked is None, reason="oracle/_ref/libswarmsim_hooked.so not built")

RECORD_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p)


def churn_arrays(cfg):
    ts = (C.c_double * max(len(cfg.churn), 1))(*[t for t, _ in cfg.churn])
    ds = (C.c_int64 * max(len(cfg.churn), 1))(*[d for _, d in cfg.churn])
    return ts, ds


def hooked_records(cfg, seed):
    from paper_2301_11913_b200 import _lib
    out = []

    def cb(ctx, rec):
        r = _lib.EngineRecord.from_address(rec)
        out.append((r.kind, r.trainer, r.stage, r.backward, r.worker, r.time))
        return 0

    fn = RECORD_FN(cb)
    ts, ds = churn_arrays(cfg)
    done = C.c_uint64()
    rc = O.hooked.hooked_sim_run(cfg.to_reference_json().encode(), ts, ds, len(cfg.churn), seed,
                                 C.cast(fn, C.c_void_p), None, C.byref(done), None)
    assert rc == 0
    return out, done.value


def engine_records(cfg, seed):
    from paper_2301_11913_b200.engine import DONE, REBALANCE, Engine
    out = []
    for r in Engine(cfg, seed).records():
        if r.kind == REBALANCE:
            continue
        worker = -1 if r.kind == DONE else r.worker
        out.append((r.kind, r.trainer if r.kind in (0, 1, 2) else 0, r.stage, r.backward, worker, r.time))
    return out


def norm(recs):
    from paper_2301_11913_b200.engine import DONE
    return [(k, t if k in (0, 1, 2) else 0, s if k != DONE else 0, b if k in (0, 1, 4) else 0, w if k != DONE else -1,
             round(tm, 9)) for k, t, s, b, w, tm in recs]


@needs_hooked
@pytest.mark.parametrize("case", range(20))
def test_hooked_reference_emits_the_engine_records(case):
    import test_engine as TE
    rng = random.Random(9000 + case)
    cfg = TE.random_churn_cfg(rng)
    seed = rng.randrange(2 ** 63)
    ref, done = hooked_records(cfg, seed)
    ours = engine_records(cfg, seed)
    assert norm(ref) == norm(ours)


@needs_hooked
@pytest.mark.gpu
def test_reference_engine_drives_the_driver(cuda):
    import torch

    import test_membership_gpu as TM
    from paper_2301_11913_b200 import _lib
    cfg = TM.config_e(ticks=False)
    ex = TM.make(cfg)  # the driver; its own engine stays unused: the reference feeds it
    L = _lib.lib()
    ts, ds = churn_arrays(cfg)
    done, nrec = C.c_uint64(), C.c_uint64()
    ex.fork()
    rc = O.hooked.hooked_sim_run(cfg.to_reference_json().encode(), ts, ds, len(cfg.churn), 3,
                                 C.cast(L.swarm_driver_on_record, C.c_void_p), ex.h, C.byref(done), C.byref(nrec))
    assert rc == 0, L.swarm_driver_last_error()
    ex.finish()
    ex.flush_wgrad()
    torch.cuda.synchronize()
    c = ex.counters()
    assert c["completed"] == done.value and c["migrations"] >= 1 and c["recomputes"] >= 1
    want = TM.replay_reference(ex, cfg)
    for pid, st in ex.stages.items():
        e = TM.rel(st.grads(), want[pid])
        assert e <= 1e-4, (pid, e)
