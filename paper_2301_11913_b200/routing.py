"""Python face of the host C++ control plane (csrc/router.cpp via the C-ABI):
RoutingState (stochastic wiring / IWRR) and the rebalancing decision, with the
reference binding's method names (P/bindings/module.cpp:244-279).  Peers are
plain ints (or anything with `.value`, like the reference's PeerId)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from . import _lib as L


def _pid(p) -> int:
    return int(getattr(p, "value", p))


def _check(rc: int, what: str) -> None:
    if rc == L.SWARM_OK:
        return
    msg = f"{what}: {L.lib().swarm_router_last_error().decode()}"
    from ._swarmsim_b200 import ConfigError, NoPeerAvailable
    if rc == L.SWARM_E_NO_PEER:
        raise NoPeerAvailable(msg)
    raise ConfigError(msg)


class RoutingState:
    def __init__(self, n_stages: int, gamma: float = 0.1, epsilon: float = 1.0):
        self._lib = L.lib()
        h = C.c_void_p()
        _check(self._lib.swarm_router_create(n_stages, gamma, epsilon, C.byref(h)), "RoutingState")
        self._h = h
        self.n_stages = n_stages

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.swarm_router_destroy(self._h)
            self._h = None

    def add_server(self, peer, stages, phase: float = 1.0) -> None:
        arr = (C.c_size_t * max(1, len(stages)))(*sorted(stages))
        _check(self._lib.swarm_router_add_server(self._h, _pid(peer), arr, len(stages), phase), "add_server")

    def ban_server(self, peer) -> None:
        _check(self._lib.swarm_router_ban_server(self._h, _pid(peer)), "ban_server")

    def remove_server(self, peer) -> None:
        self._lib.swarm_router_remove_server(self._h, _pid(peer))

    def is_banned(self, peer) -> bool:
        return bool(self._lib.swarm_router_is_banned(self._h, _pid(peer)))

    def choose_server(self, stage: int) -> int:
        out = C.c_uint64()
        _check(self._lib.swarm_router_choose_server(self._h, stage, C.byref(out)), "choose_server")
        return out.value

    def record_response(self, peer, elapsed_seconds: float) -> None:
        _check(self._lib.swarm_router_record_response(self._h, _pid(peer), elapsed_seconds), "record_response")

    def _state(self, peer):
        e, p = C.c_double(), C.c_double()
        _check(self._lib.swarm_router_peer_state(self._h, _pid(peer), C.byref(e), C.byref(p)), "peer_state")
        return e.value, p.value

    def ema_of(self, peer) -> float:
        return self._state(peer)[0]

    def priority_of(self, peer) -> float:
        return self._state(peer)[1]

    def route_forward(self, fail_oracle=None) -> list[int]:
        """Route one microbatch through stages 0..n-1, banning peers the oracle
        reports failed and retrying the stage (P/src/wiring.cpp:134-150)."""
        route = []
        for stage in range(self.n_stages):
            while True:
                peer = self.choose_server(stage)
                if fail_oracle is not None and fail_oracle(peer, stage):
                    self.ban_server(peer)
                    continue
                route.append(peer)
                break
        return route


@dataclass
class StageLoadTable:
    loads: list = field(default_factory=list)
    members: list = field(default_factory=list)  # per stage: {peer: queue size}


@dataclass
class RebalanceDecision:
    mover: int | None
    from_stage: int
    to_stage: int
    op_count: int = 0


def decide(table: StageLoadTable) -> RebalanceDecision:
    """Alg. 2 (P/src/rebalancer.cpp:25-69): move the min-queue peer of the
    least-loaded stage to the most-loaded one; a stage keeps its last peer."""
    n = len(table.members)
    offsets, peers, queues = [0], [], []
    for mem in table.members:
        for p in sorted(mem, key=_pid):
            peers.append(_pid(p))
            queues.append(float(mem[p]))
        offsets.append(len(peers))
    off = (C.c_size_t * len(offsets))(*offsets)
    pe = (C.c_uint64 * max(1, len(peers)))(*peers)
    qu = (C.c_double * max(1, len(queues)))(*queues)
    mover, fs, ts, ops = C.c_uint64(), C.c_size_t(), C.c_size_t(), C.c_size_t(0)
    _check(L.lib().swarm_rebalance_decide(n, off, pe, qu, C.byref(mover), C.byref(fs), C.byref(ts), C.byref(ops)),
           "decide")
    return RebalanceDecision(None if mover.value == 2 ** 64 - 1 else mover.value, fs.value, ts.value, ops.value)
