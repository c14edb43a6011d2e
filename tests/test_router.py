"""CPU: the B200 build's host router / rebalancer make decisions identical to
the UNMODIFIED reference (oracle/_ref: P/src/wiring.cpp, P/src/rebalancer.cpp)
on the same call sequences, plus the reference's own routing tests
(P/tests/python/test_smoke.py:21-33, 55-63)."""
import ctypes as C
import random

import pytest

import oracle as O

ref = pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built")


class RefRouter:
    def __init__(self, n, gamma=0.1, eps=1.0):
        self.h = O.ref.ref_router_new(n, gamma, eps)

    def add(self, peer, stages, phase):
        arr = (C.c_size_t * len(stages))(*sorted(stages))
        return O.ref.ref_router_add_server(self.h, peer, arr, len(stages), phase)

    def choose(self, s):
        out = C.c_uint64()
        rc = O.ref.ref_router_choose_server(self.h, s, C.byref(out))
        return rc, out.value

    def __del__(self):
        O.ref.ref_router_free(self.h)


def test_proportional_shares():  # test_smoke.py:21-33
    from paper_2301_11913_b200.routing import RoutingState
    r = RoutingState(1)
    for i, ema in enumerate([1.0, 2.0, 4.0]):
        r.add_server(i, {0}, 1.0)
        for _ in range(50):
            r.record_response(i, ema)
    picks = [0, 0, 0]
    for _ in range(7000):
        picks[r.choose_server(0)] += 1
    assert picks[0] / 7000 == pytest.approx(4 / 7, abs=0.02)
    assert picks[2] / 7000 == pytest.approx(1 / 7, abs=0.02)


def test_errors():
    from paper_2301_11913_b200 import ConfigError, NoPeerAvailable
    from paper_2301_11913_b200.routing import RoutingState
    with pytest.raises(ConfigError):
        RoutingState(0)
    with pytest.raises(ConfigError):
        RoutingState(2, gamma=0.0)
    r = RoutingState(2)
    with pytest.raises(ConfigError):
        r.add_server(1, {5})
    with pytest.raises(NoPeerAvailable):
        r.choose_server(0)
    r.add_server(1, {0})
    with pytest.raises(ConfigError):
        r.record_response(1, 0.0)
    with pytest.raises(ConfigError):
        r.ban_server(99)
    r.ban_server(1)
    with pytest.raises(NoPeerAvailable):
        r.choose_server(0)
    # route_forward bans failing peers and retries (wiring.cpp:134-150)
    r2 = RoutingState(2)
    for p, s in [(0, 0), (1, 0), (2, 1)]:
        r2.add_server(p, {s})
    route = r2.route_forward(lambda peer, stage: peer == 0)
    assert route == [1, 2] and r2.is_banned(0)


@ref
@pytest.mark.parametrize("seed", range(12))
def test_router_decisions_identical_to_reference(seed):
    from paper_2301_11913_b200.routing import RoutingState
    rng = random.Random(seed)
    S = rng.randint(1, 4)
    gamma = rng.choice([0.1, 0.3, 1.0])
    ours, theirs = RoutingState(S, gamma, 1.0), RefRouter(S, gamma, 1.0)
    live, banned, next_id = set(), set(), 0
    for step in range(3000):
        op = rng.random()
        if op < 0.08 or not live:  # add (fresh id) or re-add a banned peer (migration path)
            if banned and rng.random() < 0.5:
                pid = rng.choice(sorted(banned))
                banned.discard(pid)
            else:
                pid = next_id
                next_id += 1
            stages = set(rng.sample(range(S), rng.randint(1, S)))
            phase = rng.choice([0.0, 0.5, 1.0, rng.random()])
            ours.add_server(pid, stages, phase)
            assert theirs.add(pid, stages, phase) == 0
            live.add(pid)
        elif op < 0.11:
            pid = rng.choice(sorted(live))
            ours.ban_server(pid)
            assert O.ref.ref_router_ban_server(theirs.h, pid) == 0
            live.discard(pid)
            banned.add(pid)
        elif op < 0.13:
            pid = rng.choice(sorted(live))
            ours.remove_server(pid)
            O.ref.ref_router_remove_server(theirs.h, pid)
            live.discard(pid)  # removed ids are never reused (as in the engine)
        elif op < 0.6:
            s = rng.randrange(S)
            rc, want = theirs.choose(s)
            if rc == 2:
                from paper_2301_11913_b200 import NoPeerAvailable
                with pytest.raises(NoPeerAvailable):
                    ours.choose_server(s)
            else:
                assert ours.choose_server(s) == want, (seed, step)
        else:
            pid = rng.choice(sorted(live | banned))
            dt = rng.choice([0.5, 1.0, 2.0, rng.uniform(0.01, 5.0)])
            ours.record_response(pid, dt)
            assert O.ref.ref_router_record_response(theirs.h, pid, dt) == 0
        if step % 97 == 0:
            for pid in live | banned:
                assert ours.ema_of(pid) == O.ref.ref_router_ema_of(theirs.h, pid)
                assert ours.priority_of(pid) == O.ref.ref_router_priority_of(theirs.h, pid)


@ref
@pytest.mark.parametrize("seed", range(20))
def test_rebalance_decide_identical_to_reference(seed):
    from paper_2301_11913_b200.routing import StageLoadTable, decide
    rng = random.Random(seed)
    S = rng.randint(1, 6)
    members, pid = [], 0
    for s in range(S):
        m = {}
        for _ in range(rng.randint(1, 5)):
            m[pid] = float(rng.choice([0, 1, 2, 3, rng.uniform(0, 10)]))
            pid += 1
        members.append(m)
    d = decide(StageLoadTable([sum(m.values()) for m in members], members))
    offsets, peers, queues = [0], [], []
    for m in members:
        for p in sorted(m):
            peers.append(p)
            queues.append(m[p])
        offsets.append(len(peers))
    mv, fs, ts, ops = C.c_uint64(), C.c_size_t(), C.c_size_t(), C.c_size_t()
    O.ref.ref_rebalance_decide(S, (C.c_size_t * len(offsets))(*offsets), (C.c_uint64 * len(peers))(*peers),
                               (C.c_double * len(queues))(*queues), C.byref(mv), C.byref(fs), C.byref(ts), C.byref(ops))
    assert (d.mover if d.mover is not None else 2 ** 64 - 1) == mv.value
    assert (d.from_stage, d.to_stage, d.op_count) == (fs.value, ts.value, ops.value)


def test_rebalancer_decides_extremes():  # test_smoke.py:55-63
    from paper_2301_11913_b200.routing import StageLoadTable, decide
    t = StageLoadTable([10.0, 2.0, 5.0], [{0: 6.0, 1: 4.0}, {2: 1.0, 3: 1.0}, {4: 2.0, 5: 3.0}])
    d = decide(t)
    assert d.from_stage == 1 and d.to_stage == 0 and d.mover == 2
