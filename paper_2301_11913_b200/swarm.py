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
    """Which GPU serves which (stage, replica).  Peer id = stage * P + replica."""
    world: int
    n_stages: int

    def __post_init__(self):
        W, S = self.world, self.n_stages
        if W >= S:
            if W % S:
                raise ValueError(f"world {W} must be a multiple of the stage count {S}")
            self.P, self.per_rank = W // S, 1
        else:
            if S % W:
                raise ValueError(f"stage count {S} must be a multiple of world {W}")
            self.P, self.per_rank = 1, S // W
        self.peers = [(s, p) for s in range(S) for p in range(self.P)]

    def stage_of_peer(self, pid: int) -> int:
        return self.peers[pid][0]

    def rank_of_peer(self, pid: int) -> int:
        return pid if self.world >= self.n_stages else self.peers[pid][0] // self.per_rank

    def local_stages(self, rank: int) -> list[int]:
        if self.world >= self.n_stages:
            return [rank // self.P]
        return list(range(rank * self.per_rank, (rank + 1) * self.per_rank))


class RoutePlanner:
    """Per-trainer stochastic wiring, replicated identically on every rank.

    Per microbatch the trainer's router is consulted stage by stage with
    record_response after each modeled visit (forward 0..S-1, then backward
    S-1..0 on the same route), the per-trainer call order of the reference
    engine (sim.cpp:472-510).  Routes are therefore a pure function of the
    configuration and the step index."""

    def __init__(self, placement: Placement, n_trainers: int, fwd_seconds: float, gamma: float = 0.1,
                 epsilon: float = 1.0, backward_multiplier: float = 2.0):
        self.pl = placement
        self.fwd, self.bwd = fwd_seconds, fwd_seconds * backward_multiplier
        self.routers = []
        for _ in range(n_trainers):
            r = RoutingState(placement.n_stages, gamma, epsilon)
            for pid, (s, _p) in enumerate(placement.peers):
                r.add_server(pid, {s}, 1.0)
            self.routers.append(r)

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
                 modeled_flops: float = 1.0e15, profile: bool = False, use_graphs: bool = True):
        self.m = mcfg
        self.S = n_stages
        self.M = n_microbatches
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.device = torch.device("cuda", torch.cuda.current_device())
        S = self.S
        self.pl = Placement(self.world, S)
        self.P = self.pl.P
        self.per_rank = self.pl.per_rank
        self.local_stages = self.pl.local_stages(self.rank)
        self.all_local = len(self.local_stages) == S and self.P == 1  # sole peer of every stage
        self.n_trainers = n_trainers or self.P
        # stage executors for the stages this rank serves
        slots = 1 if self.all_local else (self.M if self.P == 1 else math.ceil(self.M / self.P) + 2)
        self.max_slots = slots
        self.stages: dict[int, Stage] = {}
        for s in self.local_stages:
            cfg = StageConfig(d_model=mcfg.d_model, n_heads=mcfg.n_heads, d_ffn=mcfg.d_ffn, seq_len=mcfg.seq_len,
                              micro_batch=mcfg.micro_batch, n_layers=mcfg.layers_per_stage,
                              shared_layers=mcfg.shared_layers, vocab=mcfg.vocab, is_first=int(s == 0),
                              is_last=int(s == S - 1), causal=mcfg.causal, max_slots=slots, wire=mcfg.wire,
                              block_size=mcfg.block_size, maxout_k=mcfg.maxout_k, lr=lr,
                              weight_decay=weight_decay,
                              seed=seed * 1000 + s)  # every replica of a stage starts identical
            self.stages[s] = Stage(cfg, self.device)
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
        self.wire_bytes = next(iter(self.stages.values())).wire_bytes
        tokens = mcfg.tokens
        self.fwd_seconds = 2.0 * mcfg.params_per_layer() * tokens * mcfg.layers_per_stage / modeled_flops
        self.planner = RoutePlanner(self.pl, self.n_trainers, self.fwd_seconds, gamma, epsilon)
        # per-stage gradient all-reduce groups (every rank creates every group, same order)
        self.stage_group = {}
        if self.P > 1:
            for s in range(S):
                g = dist.new_group([s * self.P + p for p in range(self.P)])
                if s in self.local_stages:
                    self.stage_group[s] = g
        # wire message pools (per microbatch) and the loss accumulator
        n_buf = 1 if self.all_local else self.M
        self.act = [torch.empty(self.wire_bytes, dtype=torch.uint8, device=self.device) for _ in range(n_buf)]
        self.grd = [torch.empty(self.wire_bytes, dtype=torch.uint8, device=self.device) for _ in range(n_buf)]
        self.loss_sum = torch.zeros(1, dtype=torch.float32, device=self.device)
        self.last_routes: list[list[int]] = []

    def rank_of_peer(self, pid: int) -> int:
        return self.pl.rank_of_peer(pid)

    def plan(self) -> list[list[int]]:
        self.last_routes = self.planner.plan(self.M)
        return self.last_routes

    # ------------------------------------------------------------ execution
    def step(self, tokens: torch.Tensor, targets: torch.Tensor, loss_scale: float | None = None) -> None:
        """One optimizer step over M microbatches.  tokens/targets: int32
        [M, B*L] on this device (only read by the first / last stage)."""
        routes = self.plan()
        self._profiled.clear()
        scale = loss_scale if loss_scale is not None else 1.0 / (self.M * self.m.tokens)
        if self.all_local:
            self._step_local(routes, tokens, targets, scale)
        else:
            self._step_pipelined(routes, tokens, targets, scale)
        for s, st in self.stages.items():
            if self.P > 1:
                dist.all_reduce(st.grads(), op=dist.ReduceOp.SUM, group=self.stage_group[s])
            st.optimizer_step(grad_scale=1.0 / self.P)

    # ---------------------------------------------------------------- visits
    def _run(self, key, fn) -> None:
        s, kind = key[0], key[1]
        eager_prof = self.profile and (s, kind) not in self._profiled
        if eager_prof or not self.use_graphs or (s, kind) not in self._warm:
            st = self.stages[s]
            if eager_prof:
                st.profile(True)
                self._profiled.add((s, kind))
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

    def _fwd(self, s, slot, inp, out=None, targets=None, scale=1.0) -> None:
        st = self.stages[s]
        key = (s, "f", slot, inp.data_ptr(), None if out is None else out.data_ptr(),
               None if targets is None else targets.data_ptr())
        self._run(key, lambda: st.forward(slot, inp, out=out, targets=targets, loss_sum=self.loss_sum,
                                          loss_scale=scale))

    def _bwd(self, s, slot, gin=None, gout=None) -> None:
        st = self.stages[s]
        key = (s, "b", slot, None if gin is None else gin.data_ptr(), None if gout is None else gout.data_ptr())
        self._run(key, lambda: st.backward(slot, grad_in=gin, grad_out=gout))

    def _step_local(self, routes, tokens, targets, scale) -> None:
        # every stage lives here: run each microbatch depth-first (fwd 0..S-1,
        # bwd S-1..0) so one activation slot per stage suffices
        a, g = self.act[0], self.grd[0]
        for mb in range(self.M):
            for s in range(self.S):
                inp = tokens[mb] if s == 0 else a
                if s == self.S - 1:
                    self._fwd(s, 0, inp, targets=targets[mb], scale=scale)
                else:
                    self._fwd(s, 0, inp, out=a)
            for s in reversed(range(self.S)):
                self._bwd(s, 0, None if s == self.S - 1 else g, None if s == 0 else g)

    def _step_pipelined(self, routes, tokens, targets, scale) -> None:
        """GPipe order over this rank's visits: all forwards by ascending
        microbatch, then all backwards by descending microbatch.  Every pair of
        ranks therefore posts its sends and receives in the same order, and
        the visit graph is acyclic, so NCCL point-to-point cannot deadlock."""
        mine = visit_schedule(self.pl, routes, self.rank)
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

    # ------------------------------------------------------------- metrics
    def profile_read(self):
        ms = fl = 0.0
        n = 0
        for st in self.stages.values():
            a, b, c = st.profile_read()
            ms, fl, n = ms + a, fl + b, n + c
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
