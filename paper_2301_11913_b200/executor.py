"""Engine-driven executor: the reference's discrete-event
engine decides, the GPUs execute.

The reference advances simulated time where a peer would run a stage visit
(`Engine::start_service` / `on_stage_complete`, P/src/sim.cpp:395-403,472-491),
moves a trainer to the next peer in `dispatch_current` (:405-436) and stalls
every stage at an `AllReduceTick` (:245-250).  Here every rank runs the same
C++ engine (csrc/engine.cpp, decision-identical to sim::run) and attaches real
work at exactly those points, in the engine's record order:

* START  -> the serving peer's rank runs the stage visit (forward or backward)
            on its compute stream (CUDA-graph replay per (peer, kind, trainer));
* HOP    -> the trainer's wire message (int8 codes ‖ fp32 scales ‖ header)
            is routed to the chosen peer; across ranks both halves of the NCCL
            transfer are issued at the consuming visit's START record: isend on a
            send stream that waits only for the producing visit, irecv on a
            receive stream that waits only for the previous reader of that
            buffer, and the consuming visit waits for the receive (posting the
            receive at dispatch time instead left an NCCL kernel spinning on SMs
            through the whole producing visit and blocked the rank's p2p stream:
            measured 417k vs 537k tokens/s at 2 stages x 2 peers);
* ALLREDUCE -> each stage's peers all-reduce their fp32 gradient arena and take
            an AdamW step over the microbatches their stage served since the
            last tick (SWARM's asynchronous accumulate-then-average);
* DONE   -> a microbatch finished (loss already accumulated on the last stage).

This is asynchronous SWARM training: no per-step barrier, trainers keep their
microbatches moving, peers serve queued visits in FIFO order (one compute
stream per local peer).  Every dependency points to an earlier record, and
every rank issues its halves of a point-to-point transfer at the same record,
so NCCL cannot deadlock.

Buffers: activation slot = trainer id on every peer (a trainer has at most
one microbatch in flight); wire messages per (trainer, boundary, direction).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib as L
from .engine import ALLREDUCE, DONE, HOP, START, Engine, EngineConfig
from .stage import Stage, StageConfig
from .swarm import ModelConfig, Placement


def wire_key(S: int, t: int, stage: int, backward: bool):
    """The wire message the visit (t, stage, backward) reads, or None: ("a", t, b)
    crosses boundary b forward (stage b -> b+1), ("g", t, b) backward."""
    if backward:
        return None if stage == S - 1 else ("g", t, stage)
    return None if stage == 0 else ("a", t, stage - 1)


def hop_action(pl: Placement, S: int, r, rank: int):
    """What `rank` does at HOP record r: ("send", dst_rank, key), ("recv",
    src_rank, key) or None (new microbatch, turnaround, same-rank hop, or not
    involved)."""
    src, dst = r.from_worker, r.worker
    if src < 0 or src == dst:
        return None
    rs, rd = pl.rank_of_peer(src), pl.rank_of_peer(dst)
    if rs == rd:
        return None
    key = wire_key(S, r.trainer, r.stage, bool(r.backward))
    if rs == rank:
        return ("send", rd, key)
    if rd == rank:
        return ("recv", rs, key)
    return None


class PyEngineExecutor:
    """The executor's record walk in Python over torch.distributed (round 1's data
    plane), kept as an independent host implementation to cross-check the C++
    driver (EngineExecutor below) against: same engine, same visits, same gradients."""

    def __init__(self, mcfg: ModelConfig, n_stages: int = 4, *, trainers_per_peer: int = 1, seed: int = 0,
                 lr: float = 1e-4, weight_decay: float = 0.0, forward_seconds: float = 1.0,
                 backward_multiplier: float = 2.0, allreduce_period: float = 0.0, allreduce_stall: float = 0.0,
                 duration_seconds: float = 1e9, use_graphs: bool = True, n_pool: int = 16,
                 tokens: torch.Tensor | None = None, targets: torch.Tensor | None = None, pair_wgrad: bool = True,
                 stream_per_peer: bool = True, lanes: int = 1):
        self.m = mcfg
        self.S = n_stages
        self.seed = seed
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.pl = Placement(self.world, n_stages)
        S = n_stages
        self.ecfg = EngineConfig(n_stages=S, initial_peers=[[1.0] * self.pl.layout[s] for s in range(S)],
                                 forward_service_seconds=forward_seconds, backward_multiplier=backward_multiplier,
                                 trainers_per_peer=trainers_per_peer, allreduce_period=allreduce_period,
                                 allreduce_stall=allreduce_stall, duration_seconds=duration_seconds,
                                 bucket_seconds=max(duration_seconds / 64, 1e-9))
        self.engine = Engine(self.ecfg, seed)
        self.T = self.engine.n_trainers
        self.local = [pid for pid in range(len(self.pl.stage_of)) if self.pl.rank_of_peer(pid) == self.rank]
        self.stages: dict[int, Stage] = {}
        for pid in self.local:
            s = self.pl.stage_of_peer(pid)
            cfg = StageConfig(d_model=mcfg.d_model, n_heads=mcfg.n_heads, d_ffn=mcfg.d_ffn, seq_len=mcfg.seq_len,
                              micro_batch=mcfg.micro_batch, n_layers=mcfg.layers_per_stage,
                              shared_layers=mcfg.shared_layers, vocab=mcfg.vocab, is_first=int(s == 0),
                              is_last=int(s == S - 1), causal=mcfg.causal, max_slots=self.T, wire=mcfg.wire,
                              block_size=mcfg.block_size, maxout_k=mcfg.maxout_k, lr=lr,
                              weight_decay=weight_decay, seed=seed * 1000 + s)  # stage replicas start identical
            self.stages[pid] = Stage(cfg, self.device)
            if pair_wgrad:
                self.stages[pid].enable_wgrad_pairing(max(2, self.T))  # stash set = trainer id
            if lanes > 1:
                self.stages[pid].enable_lanes(lanes)
        # paired weight gradients (K = 2T GEMMs over two backward visits of a peer):
        # peer -> trainer whose backward visit deferred its weight gradients
        self.pair_wgrad = pair_wgrad
        self._pend: dict = {}
        wb = next(iter(self.stages.values())).wire_bytes if self.stages else Stage(
            StageConfig(d_model=mcfg.d_model, n_heads=mcfg.n_heads, d_ffn=mcfg.d_ffn, seq_len=mcfg.seq_len,
                        micro_batch=mcfg.micro_batch, n_layers=1, vocab=mcfg.vocab, wire=mcfg.wire,
                        block_size=mcfg.block_size, maxout_k=mcfg.maxout_k), self.device).wire_bytes
        self.wire_bytes = wb
        # wire messages: act[t][b] crosses boundary b (stage b -> b+1), grd[t][b] the other way
        self.act = [[torch.empty(wb, dtype=torch.uint8, device=self.device) for _ in range(S - 1)]
                    for _ in range(self.T)]
        self.grd = [[torch.empty(wb, dtype=torch.uint8, device=self.device) for _ in range(S - 1)]
                    for _ in range(self.T)]
        # synthetic data pool (identical on every rank); microbatch (t, k) uses pool[(t * 7 + k) % n_pool]
        if tokens is None:
            g = torch.Generator(device="cpu").manual_seed(seed + 17)
            tokens = torch.randint(0, mcfg.vocab, (n_pool, mcfg.tokens), generator=g, dtype=torch.int32)
            targets = torch.roll(tokens, -1, dims=1)
        self.pool_tok, self.pool_tgt = tokens.to(self.device), targets.to(self.device)
        self.tok = [torch.empty(mcfg.tokens, dtype=torch.int32, device=self.device) for _ in range(self.T)]
        self.tgt = [torch.empty(mcfg.tokens, dtype=torch.int32, device=self.device) for _ in range(self.T)]
        self.loss_sum = torch.zeros(1, dtype=torch.float32, device=self.device)
        self.host_tok = self.host_tgt = None  # pinned host pools (end-to-end mode), else the device pool
        self.recv_stream = torch.cuda.Stream(device=self.device)
        self.send_stream = torch.cuda.Stream(device=self.device)
        self._xfer: dict = {}      # buffer key -> this rank's half of a pending cross-rank transfer
        # one compute stream per local peer: peers sharing a GPU serve their queues
        # independently, as the engine models them, and their kernels fill each
        # other's idle SMs; cross-peer hazards are ordered by events (_done, _read)
        cur = torch.cuda.current_stream()
        if lanes > 1 and not stream_per_peer:
            raise ValueError("lanes need a stream per peer")
        # lanes > 1: a peer serves up to `lanes` visits at once, each on its own stream and
        # workspace set (round-robin); visits sharing a slot are ordered by _slot_ev
        self.lanes = lanes
        self.lane_ws = {pid: [torch.cuda.Stream(device=self.device) if stream_per_peer else cur
                              for _ in range(lanes)] for pid in self.local}
        self.ws = {pid: ls[0] for pid, ls in self.lane_ws.items()}
        self._rr = {pid: 0 for pid in self.local}
        self._slot_ev: dict = {}   # (peer, slot) -> event after the slot's last visit / flush
        self._done: dict = {}      # buffer key -> event after its local producing visit
        self._recv: dict = {}      # buffer key -> pending irecv work (the consumer waits on it)
        self._send: dict = {}      # buffer key -> pending isend work (the next writer waits on it)
        self._read: dict = {}      # buffer key -> event after the last local reader
        self.groups: dict = {}
        if self.world >= S and dist.is_initialized():
            for s in range(S):
                members = self.pl.members(s)
                g = dist.new_group(members) if len(members) > 1 else None
                if g is not None and self.rank in members:
                    self.groups[s] = g
        self.served = [0] * S      # backward visits per stage since the last tick (global count)
        self.bwd_log = [[] for _ in range(S)]  # (trainer, microbatch) of every backward visit, per stage
        self.visit_log = []                     # (trainer, microbatch, stage, backward, peer) of every visit
        self.use_graphs = use_graphs
        self.graphs: dict = {}
        self.graph_kernels: dict = {}
        self._warm: set = set()
        self.captured_kernels = 0
        self.replayed_kernels = 0
        self.captures = 0           # visit graphs captured so far
        self.completed = 0          # microbatches finished (global, from the schedule)
        self.visits_local = 0
        self.ticks = 0
        self.optimizer_steps = 0
        self.records = 0
        torch.cuda.synchronize()  # stage initialisation ran on the legacy stream; peer streams do not wait on it

    # ------------------------------------------------------------ helpers
    def _pool_index(self, t: int, k: int) -> int:
        return (t * 7 + k) % self.pool_tok.shape[0]

    def _buf(self, t: int, stage: int, backward: bool):
        return wire_key(self.S, t, stage, backward)

    def _tensor(self, key):
        kind, t, b = key
        return (self.act if kind == "a" else self.grd)[t][b]

    def _replay(self, key, fn) -> None:
        if not self.use_graphs or key not in self._warm:
            fn()
            self._warm.add(key)
            return
        g = self.graphs.get(key)
        if g is None:
            n0 = L.lib().swarm_launch_count()
            g = torch.cuda.CUDAGraph()
            if torch.cuda.current_stream() != torch.cuda.default_stream():
                # capture straight on the peer's stream: unlike the torch.cuda.graph context
                # this neither synchronises the device nor runs the garbage collector, so a
                # (peer, trainer pair) met for the first time inside a timed region does not
                # drain every other peer's queue
                g.capture_begin(capture_error_mode="thread_local")
                try:
                    fn()
                finally:
                    g.capture_end()
            else:
                with torch.cuda.graph(g):
                    fn()
            n = L.lib().swarm_launch_count() - n0
            self.captures += 1
            self.graph_kernels[key] = n
            self.captured_kernels += n
            self.graphs[key] = g
        g.replay()
        self.replayed_kernels += self.graph_kernels[key]

    # ------------------------------------------------------------ records
    def _start(self, r) -> None:
        s, t, pid, bwd = r.stage, r.trainer, r.worker, bool(r.backward)
        if bwd:
            self.served[s] += 1
            self.bwd_log[s].append((t, int(r.microbatch)))
        self.visit_log.append((t, int(r.microbatch), s, bwd, pid))
        key = self._buf(t, s, bwd)
        if key is not None and key in self._xfer:
            self._transfer(self._xfer.pop(key))  # both ranks of a cross-rank hop, at the same record
        if pid not in self.stages:
            return
        lane = self._rr[pid]
        self._rr[pid] = (lane + 1) % self.lanes
        self.ws[pid] = self.lane_ws[pid][lane]
        if self.lanes > 1:
            self.stages[pid].set_lane(lane)
        with torch.cuda.stream(self.ws[pid]):
            if self.lanes > 1:
                self._after_slot(pid, t)  # this slot's previous visit (e.g. the last stage's forward)
            paired = self._visit(r, s, t, pid, bwd)
            if self.lanes > 1:
                self._mark_slot(pid, t)
                if paired is not None:  # the pair read that slot's activations and stash: its next use waits
                    self._slot_ev[(pid, paired)] = self._slot_ev[(pid, t)]
        self.visits_local += 1

    def _after_slot(self, pid: int, t: int) -> None:
        ev = self._slot_ev.get((pid, t))
        if ev is not None:
            torch.cuda.current_stream().wait_event(ev)

    def _mark_slot(self, pid: int, t: int) -> None:
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self._slot_ev[(pid, t)] = ev

    def _visit(self, r, s, t, pid, bwd):
        """Issue one visit on the current stream; returns the slot it paired with, if any."""
        paired = None
        st = self.stages[pid]
        cur = torch.cuda.current_stream()
        inkey = self._buf(t, s, bwd)
        if inkey is not None and inkey in self._recv:
            self._recv.pop(inkey).wait()  # this peer's stream waits for the transfer
        if inkey is not None and inkey in self._done:
            cur.wait_event(self._done.pop(inkey))  # produced by a peer on this GPU (another stream)
        outkey = None
        if bwd and s > 0:
            outkey = ("g", t, s - 1)
        elif not bwd and s < self.S - 1:
            outkey = ("a", t, s)
        if outkey is not None and outkey in self._send:
            self._send.pop(outkey).wait()  # the previous message from this buffer has left
        if outkey is not None and outkey in self._read:
            cur.wait_event(self._read.pop(outkey))  # its previous local reader is done
        if not bwd and self._pend.get(pid) == t:
            self._flush(pid)  # this forward reuses the slot the pending weight gradients read
        if not bwd:
            src_tok, src_tgt = (self.host_tok, self.host_tgt) if self.host_tok is not None else (
                self.pool_tok, self.pool_tgt)
            if s == 0:  # with a host pool: the microbatch's tokens cross PCIe here (H2D from pinned memory)
                self.tok[t].copy_(src_tok[self._pool_index(t, r.microbatch)], non_blocking=True)
            if s == self.S - 1:
                self.tgt[t].copy_(src_tgt[self._pool_index(t, r.microbatch)], non_blocking=True)
            inp = self.tok[t] if s == 0 else self._tensor(inkey)
            out = None if outkey is None else self._tensor(outkey)
            tg = self.tgt[t] if s == self.S - 1 else None
            scale = 1.0 / self.m.tokens
            self._replay((pid, "f", t, self._lane(pid)), lambda: st.forward(t, inp, out=out, targets=tg, loss_sum=self.loss_sum,
                                                           loss_scale=scale))
        else:
            gin = None if inkey is None else self._tensor(inkey)
            gout = None if outkey is None else self._tensor(outkey)
            if not self.pair_wgrad:
                self._replay((pid, "b", t, self._lane(pid)), lambda: st.backward(t, grad_in=gin, grad_out=gout))
            elif pid not in self._pend:  # first of a pair: data gradients now, dY kept in stash set t
                self._replay((pid, "b", t, -1, self._lane(pid)), lambda: st.backward_ex(t, gin, gout, mode=Stage.WGRAD_DEFER, set=t))
                self._pend[pid] = t
            else:                        # second: both visits' weight gradients as K = 2T GEMMs
                p = self._pend.pop(pid)
                paired = p
                if self.lanes > 1:
                    self._after_slot(pid, p)  # the deferred visit's dY stash is complete
                self._replay((pid, "b", t, p, self._lane(pid)), lambda: st.backward_ex(t, gin, gout, mode=Stage.WGRAD_PAIR, set=t,
                                                                      prev_slot=p, prev_set=p))
        if inkey is not None:
            ev = torch.cuda.Event()
            ev.record(cur)
            self._read[inkey] = ev
        if outkey is not None:
            ev = torch.cuda.Event()
            ev.record(cur)
            self._done[outkey] = ev
        return paired

    def _hop(self, r) -> None:
        # same-rank hops need nothing: the consumer reads the producer's buffer in stream order.
        # A cross-rank transfer is issued by both ranks at the consuming visit's START record
        # (not here): a receive posted at dispatch time would spin an NCCL kernel on the SMs for
        # the whole producing visit, and it would block the rank's single p2p stream.
        act = hop_action(self.pl, self.S, r, self.rank)
        if act is not None:
            self._xfer[act[2]] = act

    def _transfer(self, act) -> None:
        op, peer, key = act
        if op == "send":
            ev = self._done.pop(key, None)  # the producing visit (on its peer's stream)
            with torch.cuda.stream(self.send_stream):
                if ev is not None:
                    self.send_stream.wait_event(ev)
                self._send[key] = dist.isend(self._tensor(key), peer)
        else:
            with torch.cuda.stream(self.recv_stream):
                ev = self._read.pop(key, None)
                if ev is not None:
                    self.recv_stream.wait_event(ev)  # the previous reader of this buffer is done
                self._recv[key] = dist.irecv(self._tensor(key), peer)

    def _lane(self, pid: int) -> int:
        return self.lane_ws[pid].index(self.ws[pid]) if self.lanes > 1 else 0

    def _flush(self, pid: int) -> None:
        """A peer's pending (deferred) weight gradients, alone (on the peer's current lane)."""
        t = self._pend.pop(pid)
        st = self.stages[pid]
        with torch.cuda.stream(self.ws[pid]):
            if self.lanes > 1:
                st.set_lane(self._lane(pid))
                self._after_slot(pid, t)
            self._replay((pid, "w", t, self._lane(pid)), lambda: st.flush_wgrad(t, t))
            if self.lanes > 1:
                self._mark_slot(pid, t)

    def _allreduce(self, r) -> None:
        self.ticks += 1
        if self.lanes > 1:  # the tick follows every visit on every lane of the peer: join onto lane 0
            for pid, ls in self.lane_ws.items():
                for w in ls[1:]:
                    ls[0].wait_stream(w)
                self.ws[pid] = ls[0]
        for pid in list(self._pend):
            self._flush(pid)
        for pid, st in self.stages.items():
            s = self.pl.stage_of_peer(pid)
            n = self.served[s]
            if n == 0:
                continue
            with torch.cuda.stream(self.ws[pid]):
                if s in self.groups:
                    dist.all_reduce(st.grads(), op=dist.ReduceOp.SUM, group=self.groups[s])
                st.optimizer_step(grad_scale=1.0 / n)  # mean over the stage's microbatches since the last tick
            self.optimizer_steps += 1
        if self.lanes > 1:  # every lane's next visit sees the updated weights
            for pid, ls in self.lane_ws.items():
                for w in ls[1:]:
                    w.wait_stream(ls[0])
        self.served = [0] * self.S

    def run(self, n_microbatches: int) -> int:
        """Process engine records until `n_microbatches` more microbatches have
        completed (or the engine's duration ends).  Returns the number completed."""
        target = self.completed + n_microbatches
        self.fork()  # peer streams start after whatever the caller queued (e.g. a loss reset)
        while self.completed < target:
            batch = self.engine.next(1)
            if not batch:
                break
            r = batch[0]
            self.records += 1
            if r.kind == START:
                self._start(r)
            elif r.kind == HOP:
                self._hop(r)
            elif r.kind == ALLREDUCE:
                self._allreduce(r)
            elif r.kind == DONE:
                self.completed += 1
        return self.completed - (target - n_microbatches)

    def flush_wgrad(self) -> None:
        """Issue every pending deferred weight gradient (before reading gradients)."""
        for pid in list(self._pend):
            self._flush(pid)

    def use_host_pool(self, enable: bool = True) -> None:
        """End-to-end mode: every microbatch's tokens / targets are copied from
        pinned host memory by the visit that consumes them."""
        if enable:
            self.host_tok = self.pool_tok.cpu().pin_memory()
            self.host_tgt = self.pool_tgt.cpu().pin_memory()
        else:
            self.host_tok = self.host_tgt = None

    def last_stage_stream(self):
        """A stream ordered after every lane of this rank's last-stage peer (it owns
        loss_sum), or None."""
        for pid in self.local:
            if self.pl.stage_of_peer(pid) == self.S - 1:
                ls = self.lane_ws[pid]
                for w in ls[1:]:
                    ls[0].wait_stream(w)
                return ls[0]
        return None

    def fork(self) -> None:
        """Every peer stream waits for the current stream (start of a timed region)."""
        cur = torch.cuda.current_stream()
        for ls in self.lane_ws.values():
            for w in ls:
                if w != cur:
                    w.wait_stream(cur)

    def finish(self) -> None:
        """The current stream waits for every peer stream and outstanding transfer
        (end of a timed region)."""
        cur = torch.cuda.current_stream()
        for w in list(self._send.values()) + list(self._recv.values()):
            w.wait()
        self._send.clear()
        self._recv.clear()
        for ls in self.lane_ws.values():
            for w in ls:
                if w != cur:
                    cur.wait_stream(w)

    def kernels_launched(self) -> int:
        return L.lib().swarm_launch_count() - self.captured_kernels + self.replayed_kernels


class EngineExecutor:
    """The engine-driven executor: a thin handle on the C++ host driver
    (csrc/driver.cpp, include/swarm_b200.h swarm_driver_*), which walks the engine's
    records and issues the visits, the NCCL transfers of the wire messages and the
    stage all-reduces itself.  Python only supplies the NCCL unique id exchange
    and torch views of driver-owned memory."""

    def __init__(self, mcfg: ModelConfig, n_stages: int = 4, *, trainers_per_peer: int = 1, seed: int = 0,
                 lr: float = 1e-4, weight_decay: float = 0.0, forward_seconds: float = 1.0,
                 backward_multiplier: float = 2.0, allreduce_period: float = 0.0, allreduce_stall: float = 0.0,
                 duration_seconds: float = 1e9, use_graphs: bool = True, n_pool: int = 16,
                 tokens: torch.Tensor | None = None, targets: torch.Tensor | None = None, pair_wgrad: bool = True,
                 stream_per_peer: bool = True, lanes: int = 1, fp32: bool = False, sim: EngineConfig | None = None,
                 dpu: bool = False, layout: list | None = None, peer_rank: list | None = None):
        """sim: a full SimConfig (initial_peers with speeds, churn trace, rebalancing); it replaces
        the engine arguments and gives the layout (any layout on any world size)."""
        import ctypes as C

        from .stage import device_view
        self.m = mcfg
        self.S = n_stages
        self.seed = seed
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.device = torch.device("cuda", torch.cuda.current_device())
        # layout: peers per stage (default: Placement's even split); peer_rank: each initial peer's
        # rank (default: the driver's pid * world / n_peers) -- see bench.py's balanced placement
        self.pl = Placement(self.world, n_stages) if sim is None and layout is None else None
        self.layout = list(layout) if layout is not None else (self.pl.layout if self.pl else None)
        if lanes > 1 and not stream_per_peer:
            raise ValueError("lanes need a stream per peer")
        self.lib = L.lib()
        self.comm = None
        if self.world > 1:
            uid = torch.zeros(128, dtype=torch.uint8)
            if self.rank == 0:
                L.check(self.lib.swarm_comm_unique_id(C.c_void_p(uid.data_ptr())), "comm_unique_id")
            t = uid.to(self.device)
            dist.broadcast(t, 0)
            uid = t.cpu()
            h = C.c_void_p()
            rc = self.lib.swarm_comm_create(C.c_void_p(uid.data_ptr()), self.world, self.rank, C.byref(h))
            if rc:
                raise RuntimeError("comm_create: " + self.lib.swarm_comm_last_error().decode())
            self.comm = h
        self.stage_cfg = StageConfig(d_model=mcfg.d_model, n_heads=mcfg.n_heads, d_ffn=mcfg.d_ffn,
                                     seq_len=mcfg.seq_len, micro_batch=mcfg.micro_batch,
                                     n_layers=mcfg.layers_per_stage, shared_layers=mcfg.shared_layers,
                                     vocab=mcfg.vocab, causal=mcfg.causal, wire=mcfg.wire,
                                     block_size=mcfg.block_size, maxout_k=mcfg.maxout_k, lr=lr,
                                     weight_decay=weight_decay, fp32=int(fp32))
        c = L.DriverConfig()
        c.model = self.stage_cfg.to_c()
        c.n_stages, c.world, c.rank = n_stages, self.world, self.rank
        c.forward_seconds, c.backward_multiplier = forward_seconds, backward_multiplier
        c.allreduce_period, c.allreduce_stall, c.duration_seconds = allreduce_period, allreduce_stall, duration_seconds
        c.trainers_per_peer, c.seed, c.lanes = trainers_per_peer, seed, lanes
        c.pair_wgrad, c.use_graphs, c.stream_per_peer = int(pair_wgrad), int(use_graphs), int(stream_per_peer)
        c.n_pool = n_pool if tokens is None else int(tokens.shape[0])
        c.comm = self.comm
        c.dpu = int(dpu)
        if layout is not None:
            self._layout_c = (C.c_int * n_stages)(*layout)
            c.layout = self._layout_c
        if peer_rank is not None:
            self._peer_rank_c = (C.c_int * len(peer_rank))(*peer_rank)
            c.peer_rank = self._peer_rank_c
        if sim is not None:
            self._sim_c = sim.to_c()
            c.sim = C.cast(C.pointer(self._sim_c), C.c_void_p)
        h = C.c_void_p()
        rc = self.lib.swarm_driver_create(C.byref(c), C.byref(h))
        if rc:
            msg = self.lib.swarm_driver_last_error().decode()
            if rc == L.SWARM_E_INVALID:
                from ._swarmsim_b200 import ConfigError
                raise ConfigError(msg)
            raise RuntimeError(msg)
        self.h = h
        self.lanes = lanes
        self.ecfg = sim or EngineConfig(
            n_stages=n_stages, initial_peers=[[1.0] * self.layout[s] for s in range(n_stages)],
            forward_service_seconds=forward_seconds, backward_multiplier=backward_multiplier,
            trainers_per_peer=trainers_per_peer, allreduce_period=allreduce_period, allreduce_stall=allreduce_stall,
            duration_seconds=duration_seconds, bucket_seconds=max(duration_seconds / 64, 1e-9))
        self.engine = Engine.borrow(self.lib.swarm_driver_engine(h), self.ecfg)
        self.T = self.engine.n_trainers
        self.loss_sum = device_view(self.lib.swarm_driver_loss_sum(h), 1, torch.float32, self.device)
        if tokens is not None:
            tokens = tokens.to(self.device, torch.int32).contiguous()
            targets = targets.to(self.device, torch.int32).contiguous()
            L.check(self.lib.swarm_driver_set_pool(h, C.c_void_p(tokens.data_ptr()), C.c_void_p(targets.data_ptr()),
                                                   int(tokens.shape[0]), 0), "driver_set_pool")
        tp, gp, npool, ntok = C.c_void_p(), C.c_void_p(), C.c_int(), C.c_int()
        self.lib.swarm_driver_pool(h, C.byref(tp), C.byref(gp), C.byref(npool), C.byref(ntok))
        self.pool_tok = device_view(tp.value, npool.value * ntok.value, torch.int32, self.device).view(npool.value, -1)
        self.pool_tgt = device_view(gp.value, npool.value * ntok.value, torch.int32, self.device).view(npool.value, -1)
        self._host_pool = None

    def close(self):
        if getattr(self, "h", None):
            self.lib.swarm_driver_destroy(self.h)
            self.h = None
        if getattr(self, "comm", None):
            self.lib.swarm_comm_destroy(self.comm)
            self.comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int, what: str) -> None:
        if rc:
            raise RuntimeError(f"{what}: {self.lib.swarm_driver_last_error().decode()}")

    def _counters(self):
        import ctypes as C
        k = L.DriverCounters()
        self._check(self.lib.swarm_driver_stats(self.h, C.byref(k)), "driver_stats")
        return k

    def peer_info(self, pid: int) -> dict:
        """The peer's stage / liveness / migration state / rank, as the records left them."""
        import ctypes as C
        st, al, mg, rk = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        self._check(self.lib.swarm_driver_peer_info(self.h, pid, C.byref(st), C.byref(al), C.byref(mg), C.byref(rk)),
                    "driver_peer_info")
        return {"stage": st.value, "alive": bool(al.value), "migrating": bool(mg.value), "rank": rk.value}

    @property
    def n_peers(self) -> int:
        return self._counters().n_peers

    @property
    def local(self) -> list:
        return [pid for pid in range(self.n_peers) if self.peer_info(pid)["rank"] == self.rank]

    def stage_of_peer(self, pid: int) -> int:
        return self.peer_info(pid)["stage"]

    @property
    def stages(self) -> dict:
        """Views of this rank's live, serving peers' stages (re-read: migration replaces a stage)."""
        out = {}
        for pid in self.local:
            info = self.peer_info(pid)
            if not info["alive"] or info["migrating"]:
                continue
            s = info["stage"]
            cfg = StageConfig(**{**self.stage_cfg.__dict__, "is_first": int(s == 0), "is_last": int(s == self.S - 1),
                                 "max_slots": self.T, "seed": self.seed * 1000 + s})
            out[pid] = Stage.borrow(self.lib.swarm_driver_stage(self.h, pid), cfg, self.device)
        return out

    def tick_time(self) -> tuple:
        """(ms, spans): cumulative GPU time this rank's peer streams spent in or blocked on ticks
        (swarm_driver_tick_time; waits for the GPU to reach the last one)."""
        import ctypes as C
        ms, n = C.c_double(), C.c_uint64()
        self._check(self.lib.swarm_driver_tick_time(self.h, C.byref(ms), C.byref(n)), "driver_tick_time")
        return ms.value, n.value

    def counters(self) -> dict:
        k = self._counters()
        return {f: getattr(k, f) for f, _ in L.DriverCounters._fields_}

    def run_until(self, n_microbatches: int, stop_kind: int) -> int:
        """run(), stopping right after the first record of kind `stop_kind` (engine.LEAVE, ...)."""
        import ctypes as C
        self.fork()
        done = C.c_uint64()
        self._check(self.lib.swarm_driver_run_until(self.h, n_microbatches, stop_kind, C.byref(done)),
                    "driver_run_until")
        return done.value

    records = property(lambda self: self._counters().records)
    optimizer_steps = property(lambda self: self._counters().optimizer_steps)
    ticks = property(lambda self: self._counters().ticks)
    captures = property(lambda self: self._counters().captures)
    completed = property(lambda self: self._counters().completed)
    visits_local = property(lambda self: self._counters().visits)

    def _pool_index(self, t: int, k: int) -> int:
        return (t * 7 + k) % self.pool_tok.shape[0]

    @property
    def visit_log(self) -> list:
        """(trainer, microbatch, stage, backward, peer) of every visit, in record order."""
        import ctypes as C
        out = []
        t, k, s, b, p = C.c_uint32(), C.c_uint64(), C.c_uint32(), C.c_int(), C.c_int64()
        for i in range(self._counters().visit_log_size):
            self.lib.swarm_driver_visit_log(self.h, i, C.byref(t), C.byref(k), C.byref(s), C.byref(b), C.byref(p))
            out.append((t.value, k.value, s.value, bool(b.value), p.value))
        return out

    @property
    def bwd_log(self) -> list:
        logs = [[] for _ in range(self.S)]
        for t, k, s, b, _ in self.visit_log:
            if b:
                logs[s].append((t, k))
        return logs

    def run(self, n_microbatches: int) -> int:
        import ctypes as C
        self.fork()  # peer streams start after whatever the caller queued (e.g. a loss reset)
        done = C.c_uint64()
        self._check(self.lib.swarm_driver_run(self.h, n_microbatches, C.byref(done)), "driver_run")
        return done.value

    def fork(self) -> None:
        self._check(self.lib.swarm_driver_fork(self.h, torch.cuda.current_stream().cuda_stream), "driver_fork")

    def finish(self) -> None:
        self._check(self.lib.swarm_driver_finish(self.h, torch.cuda.current_stream().cuda_stream), "driver_finish")

    def flush_wgrad(self) -> None:
        self._check(self.lib.swarm_driver_flush_wgrad(self.h), "driver_flush_wgrad")

    def use_host_pool(self, enable: bool = True) -> None:
        """End-to-end mode: every microbatch's tokens / targets are copied from pinned
        host memory by the visit that consumes them."""
        import ctypes as C
        if enable:
            self._host_pool = (self.pool_tok.cpu().pin_memory(), self.pool_tgt.cpu().pin_memory())
            ht, hg = self._host_pool
            self._check(self.lib.swarm_driver_set_pool(self.h, C.c_void_p(ht.data_ptr()), C.c_void_p(hg.data_ptr()),
                                                       ht.shape[0], 1), "driver_set_pool")
        else:
            self.finish()
            torch.cuda.current_stream().synchronize()
            self._check(self.lib.swarm_driver_set_pool(self.h, None, None, 1, 1), "driver_set_pool")
            self._host_pool = None

    def last_stage_stream(self):
        """A stream ordered after every lane of this rank's last-stage peer (it owns
        loss_sum), or None."""
        for pid in self.local:
            info = self.peer_info(pid)
            if info["stage"] == self.S - 1 and info["alive"] and not info["migrating"]:
                return torch.cuda.ExternalStream(self.lib.swarm_driver_peer_stream(self.h, pid), device=self.device)
        return None

    def kernels_launched(self) -> int:
        return self._counters().kernels

    PROF_CATEGORIES = ("gemm", "attention", "layernorm", "other")

    def profile(self, n_microbatches: int, spin_ns: int = 200_000_000) -> dict:
        """Run `n_microbatches` more completions as a profiled region (every visit eager on
        one stream, per-kernel CUDA events, swarm_driver_profile_begin/end) and return
        {"gemm_ms", "gemm_flops", "gemm_launches", "categories": {name: (ms, launches)},
        "region_ms"} summed over this rank's stages."""
        import ctypes as C
        self.fork()
        self._check(self.lib.swarm_driver_profile_begin(self.h, spin_ns), "driver_profile_begin")
        done = C.c_uint64()
        self._check(self.lib.swarm_driver_run(self.h, n_microbatches, C.byref(done)), "driver_run")
        ms, fl, n = C.c_double(), C.c_double(), C.c_uint64()
        cm, cn = (C.c_double * 4)(), (C.c_uint64 * 4)()
        self._check(self.lib.swarm_driver_profile_end(self.h, C.byref(ms), C.byref(fl), C.byref(n), cm, cn),
                    "driver_profile_end")
        self.finish()
        shapes = {}
        for line in self.lib.swarm_driver_profile_shapes(self.h).decode().splitlines():
            key, ms_, fl_, n_ = line.split(";")
            a = shapes.setdefault(key, [0.0, 0.0, 0])
            a[0] += float(ms_)
            a[1] += float(fl_)
            a[2] += int(n_)
        return {"gemm_ms": ms.value, "gemm_flops": fl.value, "gemm_launches": n.value, "microbatches": done.value,
                "shapes": shapes,
                "categories": {c: (cm[i], cn[i]) for i, c in enumerate(self.PROF_CATEGORIES)}}


def sequential_reference_grads(ex) -> dict:
    """Verification helper: every peer's gradient over exactly the visits the
    schedule ran on it, recomputed sequentially on fresh replicas (same seeds,
    one slot, no optimizer step), one microbatch at a time along its route.
    The last stage's forward also accumulates the LM-head gradient, so every
    microbatch that reached the last stage counts there even if its backward
    had not started.  Returns {peer: fp32 gradient arena}.  Valid while no
    ALLREDUCE tick changed the weights."""
    S, m = ex.S, ex.m
    ref = {}
    n_peers = ex.n_peers if hasattr(ex, "n_peers") else len(ex.pl.stage_of)
    stage_of = ex.stage_of_peer if hasattr(ex, "stage_of_peer") else ex.pl.stage_of_peer
    for pid in range(n_peers):
        s = stage_of(pid)
        cfg = StageConfig(d_model=m.d_model, n_heads=m.n_heads, d_ffn=m.d_ffn, seq_len=m.seq_len,
                          micro_batch=m.micro_batch, n_layers=m.layers_per_stage, shared_layers=m.shared_layers,
                          vocab=m.vocab, is_first=int(s == 0), is_last=int(s == S - 1), causal=m.causal,
                          max_slots=1, wire=m.wire, block_size=m.block_size, maxout_k=m.maxout_k,
                          seed=ex.seed * 1000 + s)
        ref[pid] = Stage(cfg, ex.device)
    fwd, bwd, order = {}, {}, []
    for t, k, s, b, pid in ex.visit_log:
        (bwd if b else fwd).setdefault((t, k), {})[s] = pid
        if not b and s == S - 1:
            order.append((t, k))
    any_st = next(iter(ref.values()))
    a = [any_st.new_wire() for _ in range(max(S - 1, 1))]
    g = [any_st.new_wire() for _ in range(max(S - 1, 1))]
    loss = torch.zeros(1, dtype=torch.float32, device=ex.device)
    for t, k in order:
        idx = ex._pool_index(t, k)
        route = fwd[(t, k)]
        for s in range(S):
            st = ref[route[s]]
            inp = ex.pool_tok[idx] if s == 0 else a[s - 1]
            if s == S - 1:
                st.forward(0, inp, targets=ex.pool_tgt[idx], loss_sum=loss, loss_scale=1.0 / m.tokens)
            else:
                st.forward(0, inp, out=a[s])
        for s in sorted(bwd.get((t, k), {}), reverse=True):
            assert bwd[(t, k)][s] == route[s]  # backward retraces the forward route
            ref[route[s]].backward(0, grad_in=None if s == S - 1 else g[s], grad_out=None if s == 0 else g[s - 1])
    torch.cuda.synchronize()
    return {pid: st.grads().clone() for pid, st in ref.items()}
