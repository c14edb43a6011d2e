"""SWARM pipeline runtime on one B200 box: S stages x P peers over the ranks.

What the reference only simulates (/root/reference/proj/src/sim.cpp), run for
real:
  * stage visit     -> Stage.forward/backward (C++ executor, sm_100a kernels)
                       (Engine::visit_seconds / start_service, sim.cpp:361-403)
  * stage transport -> the visit's wire message (int8 codes + fp32 scales by
                       default) over NCCL send/recv on NVLink along the route the
                       trainer's router picked (dispatch_current, sim.cpp:405-436)
  * all-reduce      -> NCCL all-reduce of the fp32 gradient arena among a
                       stage's peers, once per optimizer step (the AllReduceTick
                       stall, sim.cpp:245-250, 352)
The router is the host C++ RoutingState (routing.py -> csrc/router.cpp), one
per trainer, replicated identically on every rank: routes are a pure function
of the seed and the call sequence, so no rank has to tell another where a
microbatch goes.  Visit times fed to record_response are the modeled ones
(cost model), exactly as the reference engine does (sim.cpp:487), which keeps
routing decisions deterministic (SURVEY.md §7 hard part 4).

Placement: with world >= S, P = world // S and rank r hosts
stage r // P (peer id == rank); with world < S every rank hosts S / world
consecutive stages (P = 1) and chains them locally.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace

import torch
import torch.distributed as dist

from . import _lib as L
from .routing import RoutingState
from .stage import WIRE_INT8, Stage, StageConfig


@dataclass
class ModelConfig:
    d_model: int
    n_heads: int
    d_ffn: int
    seq_len: int
    micro_batch: int
    layers_per_stage: int
    vocab: int
    shared_layers: int = 0
    causal: int = 1
    wire: int = WIRE_INT8
    block_size: int = 4096
    maxout_k: int = 0  # > 1: maxout bottleneck at the stage boundaries

    @property
    def tokens(self) -> int:
        return self.micro_batch * self.seq_len

    def params_per_layer(self) -> int:  # cost_model.cpp:31-35
        return 4 * self.d_model * self.d_model + 2 * self.d_model * self.d_ffn

    def flops_per_token(self, n_stages: int) -> float:
        """Model FLOPs per token, fwd+bwd (3x fwd), 2*params per layer plus
        non-causal attention 4*L*d per layer (SURVEY.md §8(d) convention)."""
        per_layer = 2 * self.params_per_layer() + 4 * self.seq_len * self.d_model
        return 3.0 * per_layer * self.layers_per_stage * n_stages


PRESETS = {
    # BASELINE.json configs[0]: 2 stages x 2 layers, d 256, L 128, B 8
    "tiny": ModelConfig(256, 4, 1024, 128, 8, 2, 512),
    # configs[2]: 8 layers/stage, d 2048, 16 heads, L 512; microbatch 4 (PAPER:292 xxlarge)
    "C": ModelConfig(2048, 16, 8192, 512, 4, 8, 50304),
    # configs[3]: d 4096, 32 heads, 16 shared layers per stage, L 512, microbatch 1
    "D": ModelConfig(4096, 32, 16384, 512, 1, 16, 50304, shared_layers=1, maxout_k=2),
}


@dataclass
class Placement:
    """Which GPU serves which stage.  With world >= S every rank is one peer
    (peer id == rank) and `layout` gives the peers per stage (default: even
    split, P = world / S); membership changes with failures and migrations.
    With world < S every rank hosts S / world consecutive stages (one peer
    each, peer id == stage)."""
    world: int
    n_stages: int
    layout: list | None = None

    def __post_init__(self):
        W, S = self.world, self.n_stages
        if W >= S:
            if self.layout is None:
                if W % S:
                    raise ValueError(f"world {W} must be a multiple of the stage count {S}")
                self.layout = [W // S] * S
            if len(self.layout) != S or sum(self.layout) != W or min(self.layout) < 1:
                raise ValueError(f"layout {self.layout} must give >= 1 peer to each of {S} stages and sum to {W}")
            self.per_rank = 1
            self.stage_of = [s for s, n in enumerate(self.layout) for _ in range(n)]
        else:
            if S % W:
                raise ValueError(f"stage count {S} must be a multiple of world {W}")
            self.per_rank = S // W
            self.layout = [1] * S
            self.stage_of = list(range(S))
        self.P = max(self.layout)
        self.alive = set(range(len(self.stage_of)))

    @property
    def peers(self) -> list[tuple[int, int]]:
        return [(s, pid) for pid, s in enumerate(self.stage_of)]

    def stage_of_peer(self, pid: int) -> int:
        return self.stage_of[pid]

    def rank_of_peer(self, pid: int) -> int:
        return pid if self.world >= self.n_stages else self.stage_of[pid] // self.per_rank

    def members(self, stage: int) -> list[int]:
        return sorted(pid for pid in self.alive if self.stage_of[pid] == stage)

    def local_stages(self, rank: int) -> list[int]:
        if self.world >= self.n_stages:
            return [self.stage_of[rank]] if rank in self.alive else []
        return list(range(rank * self.per_rank, (rank + 1) * self.per_rank))


class RoutePlanner:
    """Per-trainer stochastic wiring, replicated identically on every rank.

    Per microbatch the trainer's router is consulted stage by stage with
    record_response after each modeled visit (forward 0..S-1, then backward
    S-1..0 on the same route), the per-trainer call order of the reference
    engine (sim.cpp:472-510).  Routes are therefore a pure function of the
    configuration, the step index and the membership events (remove on failure,
    ban + re-add on migration, as kill_worker / begin_migration /
    on_migration_complete do, sim.cpp:583-719)."""

    def __init__(self, placement: Placement, n_trainers: int, fwd_seconds: float, gamma: float = 0.1,
                 epsilon: float = 1.0, backward_multiplier: float = 2.0, seed: int = 0):
        import random
        self.pl = placement
        self.fwd, self.bwd = fwd_seconds, fwd_seconds * backward_multiplier
        self.rng = random.Random(seed)  # newcomer phases (uniform01, one per router, like sim.cpp:716)
        self.routers = []
        for _ in range(n_trainers):
            r = RoutingState(placement.n_stages, gamma, epsilon)
            for pid, (s, _p) in enumerate(placement.peers):
                if pid in placement.alive:
                    r.add_server(pid, {s}, 1.0)
            self.routers.append(r)

    def remove(self, pid: int) -> None:
        for r in self.routers:
            r.remove_server(pid)

    def ban(self, pid: int) -> None:
        for r in self.routers:
            r.ban_server(pid)

    def add(self, pid: int, stage: int) -> None:
        for r in self.routers:
            r.add_server(pid, {stage}, self.rng.random())

    def plan(self, n_microbatches: int) -> list[list[int]]:
        routes = []
        for mb in range(n_microbatches):
            r = self.routers[mb % len(self.routers)]
            route = []
            for s in range(self.pl.n_stages):
                pid = r.choose_server(s)
                r.record_response(pid, self.fwd)
                route.append(pid)
            for s in reversed(range(self.pl.n_stages)):
                r.record_response(route[s], self.bwd)
            routes.append(route)
        return routes


def queue_proxy_table(pl: Placement, visits: list):
    """Load table for Alg. 2 (rebalancer.cpp:25-69).  The reference publishes
    time-averaged queue lengths; in this synchronous pipeline a peer's queue
    proxy is the forward work it was routed beyond the least-loaded live peer
    since the last rebalance (bottleneck peers accumulate it, idle ones do not)."""
    from .routing import StageLoadTable
    live = sorted(pl.alive)
    base = min(visits[p] for p in live)
    members = [{p: float(visits[p] - base) for p in pl.members(s)} for s in range(pl.n_stages)]
    return StageLoadTable([sum(m.values()) for m in members], members)


def visit_schedule(pl: Placement, routes: list[list[int]], rank: int) -> list[tuple[int, int]]:
    """(microbatch, stage) forward visits this rank executes, in GPipe order;
    backward visits run the same list reversed."""
    local = pl.local_stages(rank)
    return [(mb, s) for mb in range(len(routes)) for s in local if pl.rank_of_peer(routes[mb][s]) == rank]


def message_log(pl: Placement, routes: list[list[int]], rank: int):
    """The point-to-point operations `rank` issues in one step, in issue order:
    ("send"|"recv", peer_rank, phase, microbatch).  Used by tests to prove every
    rank pair agrees on the order (no NCCL deadlock)."""
    S = pl.n_stages
    ops = []
    mine = visit_schedule(pl, routes, rank)
    for mb, s in mine:
        if s > 0 and (src := pl.rank_of_peer(routes[mb][s - 1])) != rank:
            ops.append(("recv", src, "fwd", mb))
        if s < S - 1 and (dst := pl.rank_of_peer(routes[mb][s + 1])) != rank:
            ops.append(("send", dst, "fwd", mb))
    for mb, s in reversed(mine):
        if s < S - 1 and (src := pl.rank_of_peer(routes[mb][s + 1])) != rank:
            ops.append(("recv", src, "bwd", mb))
        if s > 0 and (dst := pl.rank_of_peer(routes[mb][s - 1])) != rank:
            ops.append(("send", dst, "bwd", mb))
    return ops


class SwarmPipeline:
    def __init__(self, mcfg: ModelConfig, n_stages: int = 4, *, n_microbatches: int = 16, n_trainers: int | None = None,
                 seed: int = 0, lr: float = 1e-4, weight_decay: float = 0.0, gamma: float = 0.1, epsilon: float = 1.0,
                 modeled_flops: float = 1.0e15, profile: bool = False, use_graphs: bool = True,
                 layout: list | None = None, max_slots: int | None = None, dpu: bool = False,
                 pair_wgrad: bool = True):
        self.m = mcfg
        self.S = n_stages
        self.M = n_microbatches
        self.seed = seed
        self.lr, self.weight_decay = lr, weight_decay
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.device = torch.device("cuda", torch.cuda.current_device())
        S = self.S
        self.pl = Placement(self.world, S, layout)
        self.P = self.pl.P
        self.per_rank = self.pl.per_rank
        self.local_stages = self.pl.local_stages(self.rank)
        self.all_local = len(self.local_stages) == S and self.P == 1  # sole peer of every stage
        self.n_trainers = n_trainers or self.P
        # activation slots: a peer holds every microbatch routed to it in a step
        # paired weight gradients (K = 2T GEMMs over two backward visits) need the
        # deferred visit's activations intact: at one GPU, two slots used alternately
        self.pair_wgrad = pair_wgrad
        if max_slots is None:
            max_slots = (2 if pair_wgrad else 1) if self.all_local else (
                self.M if self.P == 1 or layout is not None else math.ceil(self.M / self.P) + 2)
        self.max_slots = max_slots
        self.stages: dict[int, Stage] = {s: self._new_stage(s) for s in self.local_stages}
        # CUDA graphs: a visit enqueues ~200 kernels; replaying a captured graph
        # removes the per-launch host cost.  With `profile`, the first visit of
        # each stage per step runs eagerly with GEMM events (live roofline).
        self.profile = profile
        self.use_graphs = use_graphs
        self.graphs: dict = {}
        self.graph_kernels: dict = {}  # kernels captured per graph (for gpu_launches)
        self.captured_kernels = 0      # launches counted while capturing (they did not run then)
        self.replayed_kernels = 0
        self._warm: set = set()
        self._profiled: set = set()
        self.prof_spin_ns = 0  # >0: profiled visits start behind a GPU spin of this length
        self.time_phases = False  # record per-step phase events (phase_read)
        self._phase_events: list = []
        probe = next(iter(self.stages.values()), None) or self._new_stage(0, slots=1)
        self.wire_bytes = probe.wire_bytes
        tokens = mcfg.tokens
        self.fwd_seconds = 2.0 * mcfg.params_per_layer() * tokens * mcfg.layers_per_stage / modeled_flops
        self.planner = RoutePlanner(self.pl, self.n_trainers, self.fwd_seconds, gamma, epsilon, seed=seed)
        self.stage_group: dict = {}
        self._build_groups()
        # wire message pools (per microbatch) and the loss accumulator
        n_buf = 1 if self.all_local else self.M
        self.act = [torch.empty(self.wire_bytes, dtype=torch.uint8, device=self.device) for _ in range(n_buf)]
        self.grd = [torch.empty(self.wire_bytes, dtype=torch.uint8, device=self.device) for _ in range(n_buf)]
        self.loss_sum = torch.zeros(1, dtype=torch.float32, device=self.device)
        self.last_routes: list[list[int]] = []
        self.visits = [0] * len(self.pl.stage_of)  # forward visits per peer since the last rebalance
        self.events: list[dict] = []               # membership log (failures, migrations)
        # Delayed parameter updates: step t computes on
        # bank t % 2 while the all-reduce + AdamW of step t-1 run on a separate stream;
        # step t therefore sees the weights of step t-2's update (one step of delay).
        self._pend: dict = {}      # stage -> (slot, stash set) of a visit whose weight gradients wait for a partner
        self._nvis: dict = {}      # stage -> visits per direction this step (profile weights)
        self._wset: dict = {}     # stage -> stash set the next backward visit writes
        self.dpu = dpu
        self.t = 0
        if dpu:
            self.update_stream = torch.cuda.Stream(device=self.device)
            self.update_done = [None, None]  # event: optimizer of the last step that used bank b
            for st in self.stages.values():
                st.enable_banks()
            torch.cuda.synchronize()

    def _new_stage(self, s: int, slots: int | None = None) -> Stage:
        m = self.m
        cfg = StageConfig(d_model=m.d_model, n_heads=m.n_heads, d_ffn=m.d_ffn, seq_len=m.seq_len,
                          micro_batch=m.micro_batch, n_layers=m.layers_per_stage, shared_layers=m.shared_layers,
                          vocab=m.vocab, is_first=int(s == 0), is_last=int(s == self.S - 1), causal=m.causal,
                          max_slots=slots or self.max_slots, wire=m.wire, block_size=m.block_size,
                          maxout_k=m.maxout_k, lr=self.lr, weight_decay=self.weight_decay,
                          seed=self.seed * 1000 + s)  # every replica of a stage starts identical
        st = Stage(cfg, self.device)
        if self.pair_wgrad and slots is None:
            st.enable_wgrad_pairing()
        return st

    def _build_groups(self) -> None:
        """Per-stage gradient all-reduce groups over the live members (collective:
        every rank creates every group, in stage order)."""
        self.stage_group = {}
        if self.world < self.S or not dist.is_initialized():
            return
        for s in range(self.S):
            members = self.pl.members(s)
            if len(members) > 1:
                g = dist.new_group(members)
                if self.rank in members:
                    self.stage_group[s] = g

    # ------------------------------------------------------- membership events
    def fail_peer(self, pid: int) -> None:
        """A peer leaves (sim.cpp:583-625 kill_worker): every router forgets it,
        its stage's all-reduce group shrinks, and the rank stops serving."""
        if self.dpu:
            raise NotImplementedError("membership changes with delayed parameter updates")
        torch.cuda.synchronize()
        self.planner.remove(pid)
        self.pl.alive.discard(pid)
        if pid == self.rank:
            self.local_stages = []
            self.stages = {}
            self.graphs = {}
        self._build_groups()
        self.events.append({"event": "peer_leave", "peer": pid})

    def stage_loads(self):
        return queue_proxy_table(self.pl, self.visits)

    def rebalance(self):
        """One rebalancing round: decide (host C++, decision-identical to the
        reference) and migrate the mover with its state (weights + AdamW)."""
        from .routing import decide
        d = decide(self.stage_loads())
        self.visits = [0] * len(self.visits)
        if d.mover is not None:
            self.migrate(d.mover, d.to_stage)
        self.events.append({"event": "rebalance", "mover": d.mover, "from": d.from_stage, "to": d.to_stage})
        return d

    def migrate(self, pid: int, to_stage: int) -> None:
        """begin_migration / on_migration_complete (sim.cpp:673-719) for real:
        routers ban the mover, it rebuilds its stage executor for `to_stage`
        and downloads params + AdamW moments + step from the lowest-id live
        stage-mate (NCCL point-to-point), groups are rebuilt, routers re-add it."""
        if self.dpu:
            raise NotImplementedError("membership changes with delayed parameter updates")
        torch.cuda.synchronize()
        if self.world < self.S:
            raise RuntimeError("migration needs one peer per rank (world >= stages)")
        self.planner.ban(pid)
        old = self.pl.stage_of[pid]
        donor = self.pl.members(to_stage)[0]
        if self.rank == pid:
            self.stages = {}
            self.graphs = {k: g for k, g in self.graphs.items() if k[0] != old}
            self._warm = {w for w in self._warm if w[0] != old}
            st = self._new_stage(to_stage)
            m, v, _ = st.optimizer_state()
            step = torch.zeros(1, dtype=torch.int64, device=self.device)
            for t in (st.params(), m, v, step):
                dist.recv(t, donor)
            st.set_step(int(step.item()))
            st.sync_shadow()
            self.stages = {to_stage: st}
            self.local_stages = [to_stage]
        elif self.rank == donor:
            st = self.stages[to_stage]
            m, v, step = st.optimizer_state()
            for t in (st.params(), m, v, torch.tensor([step], dtype=torch.int64, device=self.device)):
                dist.send(t, pid)
        torch.cuda.synchronize()
        self.pl.stage_of[pid] = to_stage
        self._build_groups()
        self.planner.add(pid, to_stage)
        self.events.append({"event": "migration", "peer": pid, "from": old, "to": to_stage,
                            "state_bytes": 12 * (self.stages[to_stage].n_params if to_stage in self.stages else 0)})

    def rank_of_peer(self, pid: int) -> int:
        return self.pl.rank_of_peer(pid)

    def plan(self) -> list[list[int]]:
        self.last_routes = self.planner.plan(self.M)
        for route in self.last_routes:
            for pid in route:
                self.visits[pid] += 1
        return self.last_routes

    # ------------------------------------------------------------ execution
    def step(self, tokens: torch.Tensor, targets: torch.Tensor, loss_scale: float | None = None) -> None:
        """One optimizer step over M microbatches.  tokens/targets: int32
        [M, B*L] on this device (only read by the first / last stage)."""
        if self.dpu:
            return self._step_dpu(tokens, targets, loss_scale)
        routes = self.plan()
        self._profiled.clear()
        scale = loss_scale if loss_scale is not None else 1.0 / (self.M * self.m.tokens)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if self.time_phases else None
        if ev:
            ev[0].record()
        if self.all_local:
            self._step_local(routes, tokens, targets, scale)
        else:
            self._step_pipelined(routes, tokens, targets, scale)
        if ev:
            ev[1].record()
        for s, st in self.stages.items():
            if s in self.stage_group:
                dist.all_reduce(st.grads(), op=dist.ReduceOp.SUM, group=self.stage_group[s])
        if ev:
            ev[2].record()
        for st in self.stages.values():
            # every peer holds the sum over ITS microbatches of d(loss/(M*T)); the SUM over
            # the stage peers is the full-batch gradient, so no further scaling
            st.optimizer_step(grad_scale=1.0)
        if ev:
            ev[3].record()
            self._phase_events.append(ev)

    def _step_dpu(self, tokens, targets, loss_scale) -> None:
        """One step with delayed parameter updates: visits on bank t % 2 (after the
        optimizer that last wrote that bank, two steps ago, has finished), then the
        stage all-reduce + AdamW of this bank queued on the update stream."""
        bank = self.t % 2
        cur = torch.cuda.current_stream()
        if self.update_done[bank] is not None:
            cur.wait_event(self.update_done[bank])
        for st in self.stages.values():
            st.set_bank(bank)
        routes = self.plan()
        self._profiled.clear()
        scale = loss_scale if loss_scale is not None else 1.0 / (self.M * self.m.tokens)
        if self.all_local:
            self._step_local(routes, tokens, targets, scale)
        else:
            self._step_pipelined(routes, tokens, targets, scale)
        visits_done = torch.cuda.Event()
        visits_done.record(cur)
        with torch.cuda.stream(self.update_stream):
            self.update_stream.wait_event(visits_done)
            for s, st in self.stages.items():
                if s in self.stage_group:
                    dist.all_reduce(st.grads_bank(bank), op=dist.ReduceOp.SUM, group=self.stage_group[s])
            for st in self.stages.values():
                st.optimizer_step_bank(bank, grad_scale=1.0, stream=self.update_stream)
            done = torch.cuda.Event()
            done.record(self.update_stream)
        self.update_done[bank] = done
        self.t += 1

    def drain_updates(self) -> None:
        """Make the current stream wait for every queued delayed update (end of a
        timed region: the last step's optimizer is part of its cost)."""
        if self.dpu:
            cur = torch.cuda.current_stream()
            for e in self.update_done:
                if e is not None:
                    cur.wait_event(e)

    def phase_read(self) -> dict:
        """Per-step device time of this rank's phases since the last read (ms):
        stage visits + transport, gradient all-reduce, optimizer (time_phases=True)."""
        torch.cuda.synchronize()
        out = {"visits_ms": 0.0, "allreduce_ms": 0.0, "optimizer_ms": 0.0}
        for ev in self._phase_events:
            out["visits_ms"] += ev[0].elapsed_time(ev[1])
            out["allreduce_ms"] += ev[1].elapsed_time(ev[2])
            out["optimizer_ms"] += ev[2].elapsed_time(ev[3])
        n = max(1, len(self._phase_events))
        self._phase_events = []
        return {k: v / n for k, v in out.items()}

    # ---------------------------------------------------------------- visits
    def _run(self, key, fn, prof=None) -> None:
        """Run a visit: eagerly the first time (warm-up) and, with `profile`, once per
        (stage, visit kind) per step with events weighted by `prof` = (kind, visits of
        that kind this step), so the profiled visits stand for the whole step;
        otherwise replay its captured CUDA graph."""
        s, kind = key[0], key[1]
        pkind, weight = prof if prof is not None else (kind, 1.0)
        eager_prof = self.profile and (s, pkind) not in self._profiled
        if eager_prof or not self.use_graphs or (s, kind) not in self._warm:
            st = self.stages[s]
            if eager_prof:
                if self.prof_spin_ns:  # let the host run ahead: kernels queue back to back
                    L.check(L.lib().swarm_gpu_spin(int(self.prof_spin_ns), torch.cuda.current_stream().cuda_stream),
                            "gpu_spin")
                st.profile_weight(weight)
                st.profile(True)
                self._profiled.add((s, pkind))
            fn()
            if eager_prof:
                st.profile(False)  # keep the events recorded so far; stop adding
            self._warm.add((s, kind))
            return
        g = self.graphs.get(key)
        if g is None:
            n0 = L.lib().swarm_launch_count()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            n = L.lib().swarm_launch_count() - n0
            self.graph_kernels[key] = n
            self.captured_kernels += n
            self.graphs[key] = g
        g.replay()
        self.replayed_kernels += self.graph_kernels[key]

    def _bank(self) -> int:  # captured graphs bake the bank's weight / gradient pointers
        return self.t % 2 if self.dpu else 0

    def _fwd(self, s, slot, inp, out=None, targets=None, scale=1.0) -> None:
        st = self.stages[s]
        key = (s, "f", slot, self._bank(), inp.data_ptr(), None if out is None else out.data_ptr(),
               None if targets is None else targets.data_ptr())
        self._run(key, lambda: st.forward(slot, inp, out=out, targets=targets, loss_sum=self.loss_sum,
                                          loss_scale=scale), prof=("f", self._nvis.get(s, 1)))

    def _bwd(self, s, slot, gin=None, gout=None) -> None:
        st = self.stages[s]
        if not self.pair_wgrad:
            key = (s, "b", slot, self._bank(), None if gin is None else gin.data_ptr(),
                   None if gout is None else gout.data_ptr())
            self._run(key, lambda: st.backward(slot, grad_in=gin, grad_out=gout), prof=("b", self._nvis.get(s, 1)))
            return
        # weight gradients of two backward visits per stage run as one K = 2T GEMM each:
        # the first visit defers (stashing its dY), the second pairs with it
        wset = self._wset.get(s, 0)
        pend = self._pend.get(s)
        mode, (pslot, pset) = (Stage.WGRAD_DEFER, (-1, 0)) if pend is None else (Stage.WGRAD_PAIR, pend)
        key = (s, "b", slot, self._bank(), None if gin is None else gin.data_ptr(),
               None if gout is None else gout.data_ptr(), mode, wset, pslot, pset)
        n = self._nvis.get(s, 1)
        self._run(key, lambda: st.backward_ex(slot, gin, gout, mode=mode, set=wset, prev_slot=pslot, prev_set=pset),
                  prof=(f"b{mode}", (n + 1) // 2 if mode == Stage.WGRAD_DEFER else n // 2))
        self._pend[s] = (slot, wset) if pend is None else None
        self._wset[s] = wset ^ 1

    def _flush_wgrad(self) -> None:
        """A stage's last unpaired backward visit: its weight gradients alone."""
        for s, pend in list(self._pend.items()):
            if pend is None:
                continue
            st = self.stages[s]
            slot, wset = pend
            self._run((s, "w", slot, self._bank(), wset), lambda: st.flush_wgrad(slot, wset), prof=("w", 1))
            self._pend[s] = None

    def _step_local(self, routes, tokens, targets, scale) -> None:
        # every stage lives here: run each microbatch depth-first (fwd 0..S-1,
        # bwd S-1..0) so one activation slot per stage suffices
        a, g = self.act[0], self.grd[0]
        self._nvis = {s: self.M for s in range(self.S)}
        for mb in range(self.M):
            slot = mb % self.max_slots  # paired weight gradients: the previous microbatch's slot stays intact
            for s in range(self.S):
                inp = tokens[mb] if s == 0 else a
                if s == self.S - 1:
                    self._fwd(s, slot, inp, targets=targets[mb], scale=scale)
                else:
                    self._fwd(s, slot, inp, out=a)
            for s in reversed(range(self.S)):
                self._bwd(s, slot, None if s == self.S - 1 else g, None if s == 0 else g)
        self._flush_wgrad()

    def _step_pipelined(self, routes, tokens, targets, scale) -> None:
        """GPipe order over this rank's visits: all forwards by ascending
        microbatch, then all backwards by descending microbatch.  Every pair of
        ranks therefore posts its sends and receives in the same order, and
        the visit graph is acyclic, so NCCL point-to-point cannot deadlock."""
        mine = visit_schedule(self.pl, routes, self.rank)
        self._nvis = {s: sum(1 for _, t in mine if t == s) for s in self.local_stages}
        slot = {}
        count = {s: 0 for s in self.local_stages}
        for mb, s in mine:
            slot[(mb, s)] = count[s]
            count[s] += 1
            if count[s] > self.max_slots:
                raise RuntimeError(f"stage {s} got {count[s]} microbatches > {self.max_slots} activation slots")
        pending = []
        for mb, s in mine:  # ---------------------------------------- forward
            st = self.stages[s]
            if s == 0:
                inp = tokens[mb]
            else:
                src = self.rank_of_peer(routes[mb][s - 1])
                inp = self.act[mb]
                if src != self.rank:
                    dist.recv(inp, src)
            if s == self.S - 1:
                self._fwd(s, slot[(mb, s)], inp, targets=targets[mb], scale=scale)
            else:
                out = self.act[mb]
                self._fwd(s, slot[(mb, s)], inp, out=out)
                dst = self.rank_of_peer(routes[mb][s + 1])
                if dst != self.rank:
                    pending.append(dist.isend(out, dst))
        for w in pending:
            w.wait()
        pending = []
        for mb, s in reversed(mine):  # ------------------------------ backward
            st = self.stages[s]
            gin = None
            if s < self.S - 1:
                gin = self.grd[mb]
                src = self.rank_of_peer(routes[mb][s + 1])
                if src != self.rank:
                    dist.recv(gin, src)
            gout = None if s == 0 else self.grd[mb]
            self._bwd(s, slot[(mb, s)], gin, gout)
            if s > 0:
                dst = self.rank_of_peer(routes[mb][s - 1])
                if dst != self.rank:
                    pending.append(dist.isend(gout, dst))
        for w in pending:
            w.wait()
        self._flush_wgrad()

    # ------------------------------------------------------------- metrics
    def profile_read(self):
        ms = fl = 0.0
        n = 0
        self.last_breakdown = {}
        for st in self.stages.values():
            a, b, c = st.profile_read()
            ms, fl, n = ms + a, fl + b, n + c
            for cat, (cms, cn) in st.profile_breakdown().items():
                pm, pn = self.last_breakdown.get(cat, (0.0, 0))
                self.last_breakdown[cat] = (pm + cms, pn + cn)
        return ms, fl, n

    def kernels_launched(self) -> int:
        """Kernels of libswarm_b200.so that actually ran: eager launches plus
        the kernel nodes of every replayed visit graph."""
        return L.lib().swarm_launch_count() - self.captured_kernels + self.replayed_kernels

    def tokens_per_step(self) -> int:
        return self.M * self.m.tokens


def synthetic_batch(mcfg: ModelConfig, n_microbatches: int, seed: int, device) -> tuple[torch.Tensor, torch.Tensor]:
    """Deterministic synthetic token batch [M, B*L] (uniform over the vocab) and
    next-token targets; identical on every rank for the same seed."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    tok = torch.randint(0, mcfg.vocab, (n_microbatches, mcfg.tokens), generator=g, dtype=torch.int32)
    tgt = torch.roll(tok, -1, dims=1)
    return tok.to(device), tgt.to(device)
