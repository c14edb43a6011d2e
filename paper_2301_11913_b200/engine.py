"""Host side of the engine-driven executor.

`Engine` wraps the C++ restatement of the reference's discrete-event engine
(csrc/engine.cpp; P/src/sim.cpp:199-761) for a static population and yields
its schedule records in event-processing order.  `SimConfig`-style arguments
keep the reference's names (sim.hpp:21-54).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from . import _lib

START, HOP, DONE, ALLREDUCE = _lib.ENG_START, _lib.ENG_HOP, _lib.ENG_DONE, _lib.ENG_ALLREDUCE
LEAVE, JOIN, MIGRATE, MIGRATED, REBALANCE = (_lib.ENG_LEAVE, _lib.ENG_JOIN, _lib.ENG_MIGRATE, _lib.ENG_MIGRATED,
                                             _lib.ENG_REBALANCE)


@dataclass
class EngineConfig:
    """The SimConfig fields the static-population engine reads (sim.hpp:21-54)."""
    n_stages: int = 4
    initial_peers: list = field(default_factory=lambda: [[1.0]] * 4)  # per stage: peer speeds
    forward_service_seconds: float = 1.0
    backward_multiplier: float = 2.0
    trainers_per_peer: int = 1
    allreduce_period: float = 0.0
    allreduce_stall: float = 0.0
    duration_seconds: float = 3600.0
    bucket_seconds: float = 60.0
    churn: list = field(default_factory=list)  # trace::Trace: [(t, delta), ...] (trace.hpp:10-16)
    rebalance_period: float = 0.0              # > 0: RebalanceMode::Periodic with this period
    straggler_timeout: float = 5.0
    propagation_delay: float = 1.0
    announce_ttl: float = 300.0
    state_transfer_bytes: int = 0
    download_bps: float = 500e6

    def worker_stages(self) -> list[int]:
        return [s for s, peers in enumerate(self.initial_peers) for _ in peers]

    def to_reference_json(self) -> str:
        """The same configuration in the reference's SimConfig::from_json schema (sim.cpp:920-992)."""
        import json
        return json.dumps({
            "stages": self.n_stages,
            "initial_peers": [[{"speed": float(v)} for v in peers] for peers in self.initial_peers],
            "forward_service_seconds": self.forward_service_seconds,
            "backward_multiplier": self.backward_multiplier,
            "trainers_per_peer": self.trainers_per_peer,
            "allreduce_period": self.allreduce_period,
            "allreduce_stall": self.allreduce_stall,
            "duration_seconds": self.duration_seconds,
            "bucket_seconds": self.bucket_seconds,
            "rebalance": ({"mode": "periodic", "period": self.rebalance_period} if self.rebalance_period > 0
                          else {"mode": "none"}),
            "straggler_timeout": self.straggler_timeout,
            "propagation_delay": self.propagation_delay,
            "announce_ttl": self.announce_ttl,
            "state_transfer_bytes": int(self.state_transfer_bytes),
            "device": {"download_bps": self.download_bps},
        })

    def to_c(self):
        """The swarm_sim_config struct (keeps its arrays alive on the returned object)."""
        c = _lib.lib().swarm_sim_config_default()
        stages = self.worker_stages()
        speeds = [float(v) for peers in self.initial_peers for v in peers]
        c._keep = [(C.c_size_t * len(stages))(*stages), (C.c_double * len(speeds))(*speeds),
                   (C.c_double * max(len(self.churn), 1))(*[float(t) for t, _ in self.churn]),
                   (C.c_int64 * max(len(self.churn), 1))(*[int(d) for _, d in self.churn])]
        c.n_stages, c.n_workers = self.n_stages, len(stages)
        c.worker_stage, c.worker_speed = c._keep[0], c._keep[1]
        c.n_churn, c.churn_t, c.churn_delta = len(self.churn), c._keep[2], c._keep[3]
        c.forward_seconds, c.backward_multiplier = self.forward_service_seconds, self.backward_multiplier
        c.trainers_per_peer = self.trainers_per_peer
        c.allreduce_period, c.allreduce_stall = self.allreduce_period, self.allreduce_stall
        c.rebalance_periodic = int(self.rebalance_period > 0)
        c.rebalance_period = self.rebalance_period if self.rebalance_period > 0 else 300.0
        c.straggler_timeout, c.propagation_delay = self.straggler_timeout, self.propagation_delay
        c.announce_ttl, c.state_transfer_bytes = self.announce_ttl, int(self.state_transfer_bytes)
        c.download_bps = self.download_bps
        c.duration_seconds, c.bucket_seconds = self.duration_seconds, self.bucket_seconds
        return c


class Engine:
    def __init__(self, cfg: EngineConfig, seed: int):
        L = _lib.lib()
        self.cfg = cfg
        self.n_workers = len(cfg.worker_stages())
        c = cfg.to_c()
        h = C.c_void_p()
        rc = L.swarm_engine_create_ex(C.byref(c), seed, C.byref(h))
        if rc != _lib.SWARM_OK:
            from ._swarmsim_b200 import ConfigError
            raise ConfigError(L.swarm_engine_last_error().decode())
        self.h = h
        self.n_trainers = L.swarm_engine_n_trainers(h)
        self._buf = (_lib.EngineRecord * 1024)()

    @classmethod
    def borrow(cls, handle: int, cfg: EngineConfig) -> "Engine":
        """A view of an engine owned by the C++ driver (never destroyed here)."""
        e = cls.__new__(cls)
        e.cfg, e.h, e._borrowed = cfg, C.c_void_p(handle), True
        e.n_workers = len(cfg.worker_stages())
        e.n_trainers = _lib.lib().swarm_engine_n_trainers(e.h)
        e._buf = (_lib.EngineRecord * 1024)()
        return e

    def __del__(self):
        try:
            if getattr(self, "h", None) and not getattr(self, "_borrowed", False):
                _lib.lib().swarm_engine_destroy(self.h)
                self.h = None
        except Exception:  # interpreter shutdown
            pass

    def next(self, cap: int = 1024) -> list:
        """Up to `cap` next records ([] once the run reached duration_seconds)."""
        if cap > len(self._buf):
            self._buf = (_lib.EngineRecord * cap)()
        n = C.c_size_t()
        rc = _lib.lib().swarm_engine_next(self.h, self._buf, cap, C.byref(n))
        if rc != _lib.SWARM_OK:
            raise RuntimeError(_lib.lib().swarm_engine_last_error().decode())
        return [_lib.EngineRecord.from_buffer_copy(self._buf[i]) for i in range(n.value)]  # the buffer is reused

    def records(self):
        while batch := self.next():
            yield from batch

    def summary(self) -> dict:
        nb = int(-(-self.cfg.duration_seconds // self.cfg.bucket_seconds))
        d, c, now = C.c_uint64(), C.c_uint64(), C.c_double()
        buckets = (C.c_double * max(nb, 1))()
        _lib.lib().swarm_engine_summary(self.h, C.byref(d), C.byref(c), buckets, nb, C.byref(now))
        rq, ab, nw, alive = C.c_uint64(), C.c_uint64(), C.c_size_t(), C.c_int64()
        _lib.lib().swarm_engine_counts(self.h, C.byref(rq), C.byref(ab), C.byref(nw), C.byref(alive))
        return {"dispatched": d.value, "completed": c.value, "buckets": list(buckets)[:nb], "now": now.value,
                "requeued": rq.value, "abandoned": ab.value, "workers": nw.value, "alive": alive.value}
