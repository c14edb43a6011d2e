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
        })


class Engine:
    def __init__(self, cfg: EngineConfig, seed: int):
        L = _lib.lib()
        self.cfg = cfg
        stages = cfg.worker_stages()
        speeds = [float(v) for peers in cfg.initial_peers for v in peers]
        self.n_workers = len(stages)
        st = (C.c_size_t * len(stages))(*stages)
        sp = (C.c_double * len(speeds))(*speeds)
        h = C.c_void_p()
        rc = L.swarm_engine_create(cfg.n_stages, len(stages), st, sp, cfg.forward_service_seconds,
                                   cfg.backward_multiplier, cfg.trainers_per_peer, cfg.allreduce_period,
                                   cfg.allreduce_stall, cfg.duration_seconds, cfg.bucket_seconds, seed, C.byref(h))
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
        return {"dispatched": d.value, "completed": c.value, "buckets": list(buckets)[:nb], "now": now.value}
