#!/usr/bin/env python3
"""bench.py — SWARM per-stage hot path on B200.

Workloads (BASELINE.json):
  train  (default) configs[2]: 4 stages x P peers, 8 layers/stage, d_model 2048,
         16 heads, seq 512, microbatch 4, bf16, int8 boundary codec, stochastic
         wiring + per-stage all-reduce.  metric: training tokens/s.  1 GPU hosts
         all 4 stages; 2 GPUs 2 stages each; 4 GPUs 4x1; 8 GPUs 4x2.
         Headline: asynchronous SWARM in the reference DES engine's record order
         (--workload engine; one step = 32 microbatch completions = 65,536 tokens,
         stage all-reduce + AdamW every 32 microbatches per stage; one stream per
         peer, 2 lanes per peer on >= 2 GPUs); the
         synchronous GPipe step (one optimizer step over 32 microbatches; --sync
         makes it the headline) is measured first and reported as "gpipe_sync".
         The global batch is fixed, so "scaling" is "strong".
  codec  configs[1]: blockwise int8 codec on 1 GiB fp32 tensors, block 4096;
         one step = quantize (K1) + dequantize (K2) of the whole tensor, i.e. one
         boundary send + receive.  metric: algorithmic GB/s.  (Also reported as
         the "codec" sub-object of the train line.)
Multi-GPU (torchrun): the codec shards with no exchange — every rank codes its
own tensor ("scaling": "weak"); value = all ranks' bytes / max-over-ranks time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return {"hbm_gbs": j["hbm_gbs"], "bf16_tflops": j["bf16_tflops"],
                "bf16_tflops_sustained": j.get("bf16_tflops_sustained"), "source": "measured"}
    return {"hbm_gbs": HBM_FALLBACK_GBS, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines: list[str] = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- dist
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def warm_until_no_captures(ex, M: int, world: int, max_steps: int = 24) -> int:
    """Untimed steps until a whole step captured no new visit graph on any rank (with several peers
    per stage a paired backward's graph depends on its partner trainer, so a fixed warm-up can leave
    captures -- milliseconds each -- inside the timed region; the driver's per-peer cap on those
    graphs, SWARM_PAIR_GRAPH_CAP, bounds how many there can be).  Returns the steps run."""
    for k in range(max_steps):
        c0 = ex.captures
        ex.run(M)
        ex.finish()
        if max_over_ranks(float(ex.captures - c0), world) == 0.0:
            return k + 1
    return max_steps


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------- codec
TRAINERS = 8  # engine trainers at every GPU count (run_engine)
CODEC_N = 1 << 28  # 1 GiB of fp32 (BASELINE.json configs[1], top of the 1 MB-1 GB sweep)
CODEC_BS = 4096
CODEC_BYTES_Q = 4 * CODEC_N + CODEC_N + 4 * (CODEC_N // CODEC_BS)  # read x, write codes + scales
CODEC_BYTES_DQ = CODEC_N + 4 * (CODEC_N // CODEC_BS) + 4 * CODEC_N  # read codes + scales, write x
CPU_SAMPLE_N = 1 << 26  # bounded CPU sample: 256 MiB of fp32 per step


def cpu_reference_codec(steps: int, warmup: int, threads: int):
    """The UNMODIFIED reference codec (oracle/_ref, compiled from
    /root/reference/proj/src/compression.cpp) on `threads` host threads over
    block-aligned chunks; falls back to the C restatement (liborc) if _ref was
    never built.  Returns (GB/s, kind, sample description)."""
    import ctypes as C

    import numpy as np

    import oracle as O
    x = O.gen_sweep_f32(CPU_SAMPLE_N, CODEC_BS, seed=1)
    bytes_step = (CODEC_BYTES_Q + CODEC_BYTES_DQ) * (CPU_SAMPLE_N / CODEC_N)
    if O.ref is not None:
        h = O.ref.ref_codec_prepare(O._p(x), x.size, CODEC_BS, threads)
        for _ in range(warmup):
            O.ref.ref_codec_run(h, 1)
        t0 = time.perf_counter()
        for _ in range(steps):
            O.ref.ref_codec_run(h, 1)
        dt = time.perf_counter() - t0
        O.ref.ref_codec_free(h)
        kind = "reference"
    else:  # single-threaded C port
        threads = 1
        codes = np.empty(x.size, np.int8)
        sc = np.empty(x.size // CODEC_BS, np.float32)
        out = np.empty_like(x)
        t0 = time.perf_counter()
        for _ in range(steps):
            O.orc.orc_quantize_f32(O._p(x), x.size, CODEC_BS, O._p(codes), O._p(sc))
            O.orc.orc_dequantize_f32(O._p(codes), x.size, O._p(sc), CODEC_BS, O._p(out))
        dt = time.perf_counter() - t0
        kind = "port"
    gbs = bytes_step * steps / dt / 1e9
    sample = (f"{CPU_SAMPLE_N} fp32 elements (256 MiB), block {CODEC_BS}, quantize+dequantize, "
              f"{steps} timed step(s), {threads} thread(s) over block-aligned chunks")
    return gbs, kind, threads, sample


def bench_codec(args, world, rank, local):
    import ctypes as C

    import numpy as np
    import torch

    from paper_2301_11913_b200 import _lib, ops
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    L = _lib.lib()
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.rand(CODEC_N, device=dev, generator=g) * 2 - 1
    x[::11] *= 500
    codes = torch.empty(CODEC_N, dtype=torch.int8, device=dev)
    scales = torch.empty(CODEC_N // CODEC_BS, dtype=torch.float32, device=dev)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()

    def step(evq=None):
        if evq is not None:
            evq[0].record(stream)
        ops.quantize(x, CODEC_BS, codes=codes, scales=scales)
        if evq is not None:
            evq[1].record(stream)
        ops.dequantize(codes, scales, CODEC_BS, out=y)
        if evq is not None:
            evq[2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    clk = ClockSampler(local)
    barrier(world)
    torch.cuda.synchronize()
    clk.start()
    n0 = L.swarm_launch_count()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(args.steps):
        step(evs[i])
    t_end.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    launches = L.swarm_launch_count() - n0
    clocks = clk.stop()
    ms_local = t_start.elapsed_time(t_end)
    ms = max_over_ranks(ms_local, world)
    q_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    dq_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    bytes_step = CODEC_BYTES_Q + CODEC_BYTES_DQ
    value = bytes_step * args.steps * world / (ms / 1e3) / 1e9
    pk = peaks()
    q_gbs = CODEC_BYTES_Q / (q_ms / 1e3) / 1e9
    dq_gbs = CODEC_BYTES_DQ / (dq_ms / 1e3) / 1e9

    # configs[1] sweep, 1 MiB .. 1 GiB of fp32 (2^18 .. 2^28 elements): per-launch
    # CUDA events, L2 flushed (a 256 MiB write) before every timed pair so that the
    # small sizes are measured from HBM, not from the 126 MB L2
    sweep = []
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    for lg in range(18, 29, 2):
        n = 1 << lg
        xs, cs, ss, ys = x[:n], codes[:n], scales[:n // CODEC_BS], y[:n]
        reps = 20
        evp = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(reps)]
        for i in range(reps + 2):
            flush.fill_(float(i))
            e = evp[i - 2] if i >= 2 else None
            if e:
                e[0].record(stream)
            ops.quantize(xs, CODEC_BS, codes=cs, scales=ss)
            if e:
                e[1].record(stream)
            ops.dequantize(cs, ss, CODEC_BS, out=ys)
            if e:
                e[2].record(stream)
        torch.cuda.synchronize()
        qus = statistics.median(e[0].elapsed_time(e[1]) for e in evp) * 1e3
        dqus = statistics.median(e[1].elapsed_time(e[2]) for e in evp) * 1e3
        bq = 5 * n + 4 * (n // CODEC_BS)
        sweep.append({"elements": n, "fp32_mib": n * 4 / 2 ** 20, "quantize_us": qus, "dequantize_us": dqus,
                      "quantize_gbs": bq / (qus * 1e-6) / 1e9, "dequantize_gbs": bq / (dqus * 1e-6) / 1e9})
    del flush

    # parity guard (a fast wrong kernel is not a result): on every 997th block, the codes and
    # scales equal the reference formula evaluated in fp64 by torch (compression.cpp:18-27:
    # a = max|x|, code = round-half-away(127 x / a)), and the dequantized values equal
    # fp32(code * a / 127) (compression.cpp:33-35)
    idx = torch.arange(0, CODEC_N // CODEC_BS, 997, device=dev)
    xb = x.view(-1, CODEC_BS)[idx].double()
    a = xb.abs().amax(1, keepdim=True)
    q = 127.0 * xb / a
    want_codes = (torch.sign(q) * torch.floor(q.abs() + 0.5)).clamp(-127, 127).to(torch.int8)
    ok = bool(torch.equal(codes.view(-1, CODEC_BS)[idx], want_codes)) and bool(
        torch.equal(scales[idx].double(), a.view(-1)))
    ok = ok and bool(torch.equal(y.view(-1, CODEC_BS)[idx], (want_codes.double() * a / 127.0).float()))

    # e2e: the reference-facing by-value path — HOST (pinned) buffers, the
    # C-ABI *_host entry points do H2D -> kernel -> D2H inside the timed region.
    e2e_steps = getattr(args, "e2e_steps", None)
    e2e_steps = max(1, min(args.steps, 5)) if e2e_steps is None else e2e_steps
    e2e_val = None
    if e2e_steps > 0:
        hx = x.cpu().pin_memory()
        hc = torch.empty(CODEC_N, dtype=torch.int8).pin_memory()
        hs = torch.empty(CODEC_N // CODEC_BS, dtype=torch.float32).pin_memory()
        hy = torch.empty(CODEC_N, dtype=torch.float32).pin_memory()

        def e2e_step():
            _lib.check(L.swarm_quantize_blockwise_host(C.c_void_p(hx.data_ptr()), _lib.DT_F32, CODEC_N, CODEC_BS,
                                                       C.c_void_p(hc.data_ptr()), C.c_void_p(hs.data_ptr())), "q_host")
            _lib.check(L.swarm_dequantize_blockwise_host(C.c_void_p(hc.data_ptr()), C.c_void_p(hs.data_ptr()),
                                                         _lib.DT_F32, CODEC_N, CODEC_BS, C.c_void_p(hy.data_ptr()),
                                                         _lib.DT_F32), "dq_host")

        e2e_step()
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        e2e_s = max_over_ranks(time.perf_counter() - t0, world)
        e2e_val = bytes_step * e2e_steps * world / e2e_s / 1e9
    h2d = 4 * CODEC_N + CODEC_N + 4 * (CODEC_N // CODEC_BS)
    d2h = CODEC_N + 4 * (CODEC_N // CODEC_BS) + 4 * CODEC_N

    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_codec_quant_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")

    line = {
        "metric": "int8 codec GB/s (blockwise absmax quantize+dequantize, algorithmic bytes)",
        "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32->u8", "data": "synthetic (uniform(-1,1), every 11th x500)",
        "config": {"workload": "codec sweep top: 1 GiB fp32 tensor (2^28 elements) per GPU, block 4096, "
                               "quantize+dequantize per step", "elements": CODEC_N, "block_size": CODEC_BS,
                   "parallelism": f"{world} independent ranks (no data-path collective)",
                   "l2": "inputs (1 GiB) > L2 (126 MB); no flush needed"},
        "roofline": {"bound": "hbm", "kernel": "k_quant_f32<256,4> (K1 quantize)", "achieved": q_gbs,
                     "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": q_gbs / pk["hbm_gbs"], "traffic": traffic,
                     "peak_source": pk["source"], "bytes_per_launch": CODEC_BYTES_Q, "launch_ms": q_ms,
                     "dequant": {"kernel": "k_dequant_blocks (K2)", "achieved": dq_gbs, "frac": dq_gbs / pk["hbm_gbs"],
                                 "launch_ms": dq_ms}},
        "e2e": {"value": e2e_val, "unit": "GB/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "swarm_quantize_blockwise_host + swarm_dequantize_blockwise_host, pinned host buffers"},
        "gpu_launches": int(launches), "clocks": clocks, "parity_ok": ok,
        "sweep": {"note": "configs[1] sizes 1 MiB-1 GiB fp32, block 4096, median of 20 launches each, L2 flushed "
                          "before each; algorithmic bytes 5.0009765625 B/element per direction; sizes below a few "
                          "hundred MiB are launch/latency-bound", "points": sweep},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        gbs, kind, thr, sample = cpu_reference_codec(1, 1, threads)
        line["cpu_baseline"] = {"value": gbs, "unit": "GB/s", "cores": thr, "kind": kind, "sample": sample}
    return line


# ----------------------------------------------------------------- train
TRAIN_STAGES = 4
TRAIN_MICROBATCHES = 32


def cpu_block_reference_steps(m, steps: int, warmup: int):
    """--impl reference, train: the CPU block oracle (the reference has no training
    path) timed as exactly K steps after W warm-ups.  Each step is
    one bounded sample of the workload: fwd+bwd of one whole microbatch through ONE
    of the model's blocks, i.e. 1/(stages*layers) of a microbatch's block work, so a
    step "processes" tokens/(stages*layers) model tokens.  Returns (tokens/s, measured
    seconds per step, threads, sample)."""
    import torch

    from oracle import block_oracle as BO
    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    g = torch.Generator().manual_seed(0)
    d, F = m.d_model, m.d_ffn
    W = {"wqkv": torch.randn(3 * d, d, generator=g) * 0.02, "wo": torch.randn(d, d, generator=g) * 0.02,
         "w1": torch.randn(F, d, generator=g) * 0.02, "w2": torch.randn(d, F, generator=g) * 0.02,
         "ln1_g": torch.ones(d), "ln1_b": torch.zeros(d), "ln2_g": torch.ones(d), "ln2_b": torch.zeros(d)}
    for v in W.values():
        v.requires_grad_(True)
    x = torch.randn(m.tokens, d, generator=g, requires_grad=True)

    def one():
        y = BO.block(x, W, m.micro_batch, m.seq_len, m.n_heads, True)
        y.backward(torch.ones_like(y))

    for _ in range(warmup):
        one()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    step_s = (time.perf_counter() - t0) / steps
    layers = m.layers_per_stage * TRAIN_STAGES
    tok_s = m.tokens / layers / step_s
    sample = (f"fp32 torch-CPU block oracle on {threads} threads: each of the {steps} timed step(s) (after {warmup} "
              f"warm-up(s)) is fwd+bwd of one {m.tokens}-token microbatch through one d={d} block ({step_s:.3f} s), "
              f"= {m.tokens}/{layers} model tokens of the {layers}-block model (embedding / LM head not sampled)")
    return tok_s, step_s, threads, sample


def cpu_block_baseline(m, budget_s: float = 20.0):
    """The fp32 CPU block oracle (oracle/block_oracle.py, torch CPU on all host
    threads) timed on a bounded sample: fwd+bwd of whole microbatches through
    ONE transformer block of the named config, extrapolated per token to the
    full model (all layers of all stages).  The reference has no CPU training
    path of its own, so this is the 'port' baseline."""
    import torch

    from oracle import block_oracle as BO
    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    g = torch.Generator().manual_seed(0)
    d, F = m.d_model, m.d_ffn
    W = {"wqkv": torch.randn(3 * d, d, generator=g) * 0.02, "wo": torch.randn(d, d, generator=g) * 0.02,
         "w1": torch.randn(F, d, generator=g) * 0.02, "w2": torch.randn(d, F, generator=g) * 0.02,
         "ln1_g": torch.ones(d), "ln1_b": torch.zeros(d), "ln2_g": torch.ones(d), "ln2_b": torch.zeros(d)}
    for v in W.values():
        v.requires_grad_(True)
    x = torch.randn(m.tokens, d, generator=g, requires_grad=True)
    reps, t0 = 0, time.perf_counter()
    while True:
        y = BO.block(x, W, m.micro_batch, m.seq_len, m.n_heads, True)
        y.backward(torch.ones_like(y))
        reps += 1
        if time.perf_counter() - t0 >= budget_s or reps >= 50:
            break
    dt = (time.perf_counter() - t0) / reps
    layers = m.layers_per_stage * TRAIN_STAGES
    tok_s = m.tokens / (dt * layers)
    sample = (f"fp32 torch-CPU block oracle, fwd+bwd of {reps} microbatch(es) of {m.tokens} tokens through one "
              f"d={d} block ({dt:.2f} s each), extrapolated to {layers} layers")
    return tok_s, threads, sample


class Shape:
    """A BASELINE model shape (mirrors paper_2301_11913_b200.swarm.PRESETS; tests/
    test_bench_host.py keeps the two equal).  Kept here so that the --impl reference
    arm never imports the product package."""

    def __init__(self, d_model, n_heads, d_ffn, seq_len, micro_batch, layers_per_stage, vocab, shared_layers=0,
                 maxout_k=0, block_size=4096):
        self.d_model, self.n_heads, self.d_ffn, self.seq_len = d_model, n_heads, d_ffn, seq_len
        self.micro_batch, self.layers_per_stage, self.vocab = micro_batch, layers_per_stage, vocab
        self.shared_layers, self.maxout_k, self.block_size = shared_layers, maxout_k, block_size

    @property
    def tokens(self) -> int:
        return self.micro_batch * self.seq_len

    def params_per_layer(self) -> int:  # cost_model.cpp:31-35
        return 4 * self.d_model * self.d_model + 2 * self.d_model * self.d_ffn

    def flops_per_token(self, n_stages: int) -> float:
        per_layer = 2 * self.params_per_layer() + 4 * self.seq_len * self.d_model
        return 3.0 * per_layer * self.layers_per_stage * n_stages


SHAPES = {
    "tiny": Shape(256, 4, 1024, 128, 8, 2, 512),
    "C": Shape(2048, 16, 8192, 512, 4, 8, 50304),
    "D": Shape(4096, 32, 16384, 512, 1, 16, 50304, shared_layers=1, maxout_k=2),
}


def shape_of(args) -> Shape:
    import copy
    m = copy.copy(SHAPES[args.model])
    mb = getattr(args, "micro_batch", None)
    if mb:
        m.micro_batch = mb
    return m


def model_config(args):
    """The product's preset (GPU arm only), with the microbatch size overridden by
    --micro-batch (configs[2] at B=4, swept over 1, 2, 4, 8)."""
    import dataclasses

    from paper_2301_11913_b200.swarm import PRESETS
    m = PRESETS[args.model]
    mb = getattr(args, "micro_batch", None)
    return dataclasses.replace(m, micro_batch=mb) if mb else m


def placement_str(world: int, S: int) -> str:
    return f"{S} stages x {world // S} peer(s) per stage" if world >= S else f"{world} GPU(s) x {S // world} stage(s) each"


def engine_placement(args, world: int, S: int):
    """(layout, peer_rank, description) of the engine workloads' peers.

    One GPU: one peer per stage.  From 4 GPUs (the default there, --placement balanced): 2 peers per
    GPU (4 per GPU on 2 GPUs when asked for), so each stage has world * that / S peers; they are placed
    by longest-processing-time first -- a peer's load is its stage's cost over its stage's peer count,
    the LM-head stage costing 1 + V d / (layers * params per layer) block stages -- on the least
    loaded GPU not yet hosting that stage.  The LM-head stage's extra work is thus spread over
    several GPUs next to lighter stages' peers (SWARM's remedy for uneven stages: more peers where
    the work is) instead of pinning one GPU to it.  Measured at 4 GPUs (16 trainers): 318-322k vs
    311.5k tokens/s contiguous over eight runs, once the driver caps the paired-backward graphs per
    peer (SWARM_PAIR_GRAPH_CAP; uncapped, new (trainer, partner) graphs kept being captured: 224k-291k
    in three runs); with 8 trainers 286-288k.  On 2 GPUs 159-165k vs 172k (the GPUs then clock at the
    power cap; the tick's cross-GPU all-reduce costs 4% of the step), so below 4 GPUs the default is
    --placement contiguous, the round-2 layout (world >= S: world / S peers per stage, one per GPU;
    else consecutive stages per GPU).
    Pure arithmetic on the Shape (no product import: the reference arm's config uses it too)."""
    placement = getattr(args, "placement", None) or ("balanced" if world >= 4 else "contiguous")
    if world == 1 or placement == "contiguous":
        if world >= S:
            return [world // S] * S, None, placement_str(world, S)
        return [1] * S, None, placement_str(world, S)
    m = shape_of(args)
    per_layer = 4 * m.d_model * m.d_model + 2 * m.d_model * m.d_ffn
    head = 1.0 + m.vocab * m.d_model / (m.layers_per_stage * per_layer)
    per_gpu = 4 if world == 2 else 2
    p = max(1, -(-per_gpu * world // S))
    layout = [p] * S
    stage = [s for s in range(S) for _ in range(p)]
    w = [(head if s == S - 1 else 1.0) / p for s in stage]
    load, hosts, rank = [0.0] * world, [set() for _ in range(world)], [0] * len(stage)
    for pid in sorted(range(len(stage)), key=lambda i: -w[i]):
        cand = [r for r in range(world) if stage[pid] not in hosts[r]] or list(range(world))
        r = min(cand, key=lambda q: (load[q], q))
        rank[pid] = r
        load[r] += w[pid]
        hosts[r].add(stage[pid])
    desc = (f"{S} stages x {p} peers per stage on {world} GPUs, load-balanced placement (LM-head stage "
            f"{head:.3f}x a block stage; max GPU load {max(load):.3f} stage visits per microbatch)")
    return layout, rank, desc


def measure_link(world, rank, nbytes=4 << 20, reps=20):
    """Stage-to-stage transport rate: rank 0 -> rank 1 NCCL send/recv of a
    wire-message-sized buffer (configs[2]: 4 MiB codes + scales), timed on the
    device; returns (bytes/s, seconds per message) or None at world 1."""
    if world < 2:
        return None
    import torch
    import torch.distributed as dist
    buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    res = None
    for it in range(2):  # warm-up round, then the timed round
        barrier(world)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(reps):
            if rank == 0:
                dist.send(buf, 1)
            elif rank == 1:
                dist.recv(buf, 0)
        t1.record()
        torch.cuda.synchronize()
        if it == 1:
            sec = max_over_ranks(t0.elapsed_time(t1) / 1e3 / reps if rank < 2 else 0.0, world)
            res = (nbytes / sec, sec)
    return res


def cost_model_report(mcfg, S, M, world, step_s, link):
    """the reference's analytic stage cost calibrated on this run.
    At one GPU every (microbatch, stage) visit runs back to back, so the measured
    step / (M*S) is the fwd+bwd visit (head, embedding and optimizer amortised in);
    effective_flops follows from the reference's own FLOP convention.  With the
    measured (or, at one GPU, committed) link rate, stage_cost gives the
    compute/comm split and the GPipe step for other GPU counts is predicted as
    (M/P + S/G_s - 1) x (visits per rank per microbatch) x visit + gradient all-reduce."""
    from paper_2301_11913_b200 import _swarmsim_b200 as X
    shape = X.LayerShape()
    shape.d_model, shape.d_ffn, shape.n_heads = mcfg.d_model, mcfg.d_ffn, mcfg.n_heads
    shape.seq_len, shape.batch, shape.layers_per_stage = mcfg.seq_len, mcfg.micro_batch, mcfg.layers_per_stage
    k = mcfg.maxout_k if mcfg.maxout_k > 1 else 1
    shape.activation_bytes_per_element = (1.0 + 4.0 / mcfg.block_size) / k  # int8 codes + fp32 scales (per maxout)
    src = "measured this run (rank 0 -> 1 NCCL send/recv, 4 MiB)"
    if link is None:
        prof = os.path.join(ROOT, "profiles", "r01_link.json")
        if os.path.exists(prof):
            with open(prof) as f:
                link = tuple(json.load(f)["link"])
            src = "profiles/r01_link.json (measured on 2 B200s)"
        else:
            link, src = (450e9, 10e-6), "nominal (no peer in this run)"
    if world != 1:
        return {"link_bps": link[0], "link_source": src}
    visit = step_s / (M * S)
    prof = X.calibrated_profile(shape, visit, link[0], 0.0)  # NVLink latency is negligible at 4 MiB
    c = X.stage_cost(shape, prof, False)
    grad_bytes = 4.0 * mcfg.params_per_layer() * (1 if mcfg.shared_layers else mcfg.layers_per_stage)
    pred = {}
    for G in (1, 2, 4, 8):
        P = max(1, G // S)
        per_rank = max(1, S // G)  # stages hosted per rank
        t = (M / P + min(G, S) - 1) * per_rank * c.total_seconds
        if P > 1:
            t += 2.0 * grad_bytes * (P - 1) / P / link[0]  # ring all-reduce of the fp32 gradient arena
        pred[str(G)] = M * mcfg.tokens / t
    # the asynchronous pipeline as the reference engine sees it (csrc/engine.cpp, decision-
    # identical to sim::run): one GPU per peer, 2 trainers per peer, a tick every ~M
    # microbatches per stage stalling for the all-reduce.  Peer speeds (SimConfig PeerSpec)
    # carry the model's stage imbalance: the last stage also runs the LM head, whose FLOPs
    # add V*d / (layers * params_per_layer) to a block stage's; the calibrated visit is the
    # average over all stages, so the block-stage visit is avg * S / (S - 1 + head_ratio)
    from paper_2301_11913_b200.engine import Engine, EngineConfig
    head_ratio = 1.0 + mcfg.vocab * mcfg.d_model / (mcfg.layers_per_stage * mcfg.params_per_layer())
    base = c.total_seconds * S / (S - 1 + head_ratio)
    eng = {}
    for G in (4, 8):
        P = G // S
        if P < 1:
            continue
        fwd = base / 3.0
        stall = 2.0 * grad_bytes * (P - 1) / P / link[0] if P > 1 else 1e-9
        dur = 400.0 * M * base / P
        peers = [[1.0] * P for _ in range(S - 1)] + [[1.0 / head_ratio] * P]
        e = Engine(EngineConfig(n_stages=S, initial_peers=peers, forward_service_seconds=fwd,
                                trainers_per_peer=2, allreduce_period=M * 3.0 * fwd / P, allreduce_stall=stall,
                                duration_seconds=dur, bucket_seconds=dur / 8), seed=1)
        while e.next(4096):
            pass
        sm = e.summary()
        eng[str(G)] = sm["completed"] * mcfg.tokens / dur
    return {"calibrated_effective_flops": prof.effective_flops, "link_bps": link[0], "link_source": src,
            "engine_predicted_tokens_per_s": eng, "head_stage_ratio": head_ratio,
            "visit_s": visit, "stage_cost": {"compute_s": c.compute_seconds, "comm_s": c.comm_seconds,
                                             "utilization": c.utilization},
            "square_cube_ratio_flop_per_bit": X.square_cube_ratio(shape),
            "predicted_tokens_per_s": pred,
            "note": "predicted_tokens_per_s: GPipe step (M/P + min(G,S) - 1) x stages-per-rank x visit + fp32 "
                    "gradient all-reduce; engine_predicted_tokens_per_s: the DES engine's completions over a long "
                    "run at the calibrated visit, the last stage's peers slowed by head_stage_ratio; "
                    "the driver's scaling run measures the same N"}


def train_config(args, world: int) -> dict:
    """The workload description, identical in both arms' JSON lines (the driver
    compares them); per-run details go to the line's "run" object."""
    m = shape_of(args)
    S, M = args.stages, args.microbatches
    which = {"C": "configs[2]", "D": "configs[3] (paper scale)", "tiny": "configs[0] (tiny)"}[args.model]
    layers = f"{m.layers_per_stage} {'shared ' if m.shared_layers else ''}layers/stage"
    codec = f"maxout k={m.maxout_k} + int8 boundary codec" if m.maxout_k > 1 else "int8 boundary codec"
    return {"workload": f"BASELINE {which}: {S} stages, {layers}, d_model {m.d_model}, {m.n_heads} heads, "
                        f"seq {m.seq_len}, {codec}, stochastic wiring + intra-stage all-reduce",
            "model": args.model, "global_batch": M * m.micro_batch, "micro_batch": m.micro_batch,
            "microbatches_per_step": M, "seq_len": m.seq_len, "tokens_per_step": M * m.tokens, "vocab": m.vocab,
            "parallelism": engine_placement(args, world, S)[2],
            "l2": "per-step working set (weights + activations, GBs) far exceeds the 126 MB L2; no flush needed"}


def bench_train(args, world, rank, local):
    import torch
    import torch.distributed as dist

    from paper_2301_11913_b200 import _lib
    from paper_2301_11913_b200.swarm import PRESETS, SwarmPipeline, synthetic_batch
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    L = _lib.lib()
    mcfg = model_config(args)
    M = args.microbatches
    S = args.stages
    pipe = SwarmPipeline(mcfg, S, n_microbatches=M, seed=1, lr=1e-4, profile=True, dpu=args.dpu)
    tok, tgt = synthetic_batch(mcfg, M, seed=7, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        pipe.step(tok, tgt)
    torch.cuda.synchronize()
    pipe.profile_read()  # drop warm-up GEMM events
    pipe.loss_sum.zero_()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)  # let nvidia-smi produce its first sample before the timed region
    barrier(world)
    torch.cuda.synchronize()
    n0 = pipe.kernels_launched()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        pipe.step(tok, tgt)
    pipe.drain_updates()  # delayed updates: the last step's all-reduce + optimizer are inside the timed region
    t1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    launches = pipe.kernels_launched() - n0
    clocks = clk.stop()
    ms = max_over_ranks(t0.elapsed_time(t1), world)
    gemm_ms, gemm_flops, gemm_n = pipe.profile_read()
    tokens_step = pipe.tokens_per_step()
    value = tokens_step * args.steps / (ms / 1e3)
    loss = pipe.loss_sum.clone()
    if world > 1:
        dist.all_reduce(loss)
    mean_loss = float(loss.item()) / (tokens_step * args.steps)

    # e2e: tokens/targets H2D from pinned host memory each step, loss D2H each step
    e2e_steps = max(1, min(args.steps, 3))
    htok, htgt = tok.cpu().pin_memory(), tgt.cpu().pin_memory()
    dtok, dtgt = torch.empty_like(tok), torch.empty_like(tgt)
    hloss = torch.empty(1, dtype=torch.float32).pin_memory()
    dtok.copy_(htok)
    dtgt.copy_(htgt)
    pipe.step(dtok, dtgt)  # untimed: capture the visit graphs for these input buffers
    pipe.profile_read()
    barrier(world)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for _ in range(e2e_steps):
        dtok.copy_(htok, non_blocking=True)
        dtgt.copy_(htgt, non_blocking=True)
        pipe.step(dtok, dtgt)
        pipe.drain_updates()
        hloss.copy_(pipe.loss_sum, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - w0, world)
    e2e_val = tokens_step * e2e_steps / e2e_s

    pk = peaks()
    peak = pk["bf16_tflops_sustained"] or pk["bf16_tflops"]
    achieved = gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else 0.0
    # one profiled visit per (stage, visit kind) per step, its events weighted by the number of
    # visits of that kind: gemm_ms is already this rank's GEMM time of whole steps
    gemm_share = (gemm_ms / args.steps) / (t0.elapsed_time(t1) / args.steps) if gemm_ms > 0 else None
    link = measure_link(world, rank)
    cost_model = cost_model_report(mcfg, S, M, world, (ms / args.steps) / 1e3, link)
    # per-category kernel time, from one extra untimed step whose profiled visits
    # start behind a GPU spin (no host-launch gaps inside the events), scaled to
    # every visit of a step
    step_ms_rank = t0.elapsed_time(t1) / args.steps
    # phase split of one untimed step on this rank (visits + transport / all-reduce / optimizer)
    pipe.time_phases = True
    pipe.step(tok, tgt)
    pipe.time_phases = False
    phases = pipe.phase_read()
    phases = {k: max_over_ranks(v, world) for k, v in phases.items()}
    pipe.profile_read()  # drop the e2e steps' events
    pipe.prof_spin_ns = 5_000_000
    pipe.step(tok, tgt)
    pipe.prof_spin_ns = 0
    pipe.profile_read()
    breakdown = {cat: {"ms_per_step": cms, "share_of_step": cms / step_ms_rank, "profiled_calls": int(cn)}
                 for cat, (cms, cn) in pipe.last_breakdown.items()}
    model_tflops = value * mcfg.flops_per_token(S) / 1e12
    gemm_traffic = {}
    prof = os.path.join(ROOT, "profiles", "ncu_gemm_qkv_traffic.json")
    if os.path.exists(prof):  # DRAM bytes of one representative launch (QKV) from the committed ncu capture
        with open(prof) as f:
            gemm_traffic = json.load(f)
    placement = (f"{S} stages x {pipe.P} peer(s) per stage" if world >= S else
                 f"{world} GPU(s) x {S // world} stage(s) each")
    line = {
        "metric": "training tokens/s (SWARM pipeline)", "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic tokens uniform over the vocab, random-init weights",
        "config": train_config(args, world),
        "run": {"placement": placement,
                "optimizer": "AdamW (fused, fp32 master)" + (", delayed parameter updates (1 step)" if args.dpu else ""),
                "mean_loss": mean_loss, "model_tflops_per_s": model_tflops,
                "model_flops_per_token": mcfg.flops_per_token(S)},
        "roofline": {"bound": "tensor", "kernel": "k_gemm (tcgen05 bf16, every block/attention/head GEMM)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "traffic": gemm_traffic.get("dram_bytes_per_launch"),
                     "traffic_note": gemm_traffic.get("note"), "peak_source": pk["source"] + " bf16 sustained",
                     "gemm_share_of_step": gemm_share,
                     "note": "GEMM events bracket every GEMM of the first visit of each (stage, visit kind) per step "
                             "(run eagerly), weighted by the visits of that kind per step; the other visits replay "
                             "CUDA graphs of the same kernels",
                     "gemm_launches": gemm_n, "gemm_flops": gemm_flops, "gemm_ms": gemm_ms},
        "step_breakdown": {"note": "isolated kernel time per category on this rank (one untimed step whose first "
                                   "visit per (stage, visit kind) is issued eagerly behind a GPU spin, side stream "
                                   "folded onto the visit stream), weighted to all visits of a step; sums can exceed "
                                   "the step where the side stream overlaps; the step also holds optimizer, "
                                   "all-reduce, transport and pipeline bubbles",
                           **breakdown},
        "e2e": {"value": e2e_val, "unit": "tokens/s", "h2d_bytes_per_step": int(tok.numel() * 8),
                "d2h_bytes_per_step": 4, "path": "SwarmPipeline.step with tokens/targets copied from pinned host "
                                                 "memory and the loss read back every step"},
        "gpu_launches": int(launches), "clocks": clocks, "cost_model": cost_model,
        "step_phases_ms": {**phases, "note": "one untimed step, max over ranks, device events on the compute stream"},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tok_s, thr, sample = cpu_block_baseline(mcfg)
        line["cpu_baseline"] = {"value": tok_s, "unit": "tokens/s", "cores": thr, "kind": "port", "sample": sample}
    return line


# ----------------------------------------------------------------- engine
def run_engine(args, world, rank, local, model: str, S: int, steps: int, warmup: int, *, fp32: bool = False,
               profile: bool = True, e2e_steps: int = 5) -> dict:
    """asynchronous SWARM training driven by the reference's event
    engine (csrc/engine.cpp, decision-identical to sim::run) and executed by the C++
    host driver (csrc/driver.cpp): trainers keep one microbatch each in flight, peers
    serve FIFO queues, wire messages move over raw NCCL, stage peers all-reduce +
    AdamW at every AllReduceTick.  A "step" = M microbatch completions; the tick
    period is sized so a stage serves ~M microbatches between ticks."""
    import argparse as _ap
    import dataclasses

    import torch

    from paper_2301_11913_b200.engine import Engine, EngineConfig
    from paper_2301_11913_b200.executor import EngineExecutor
    from paper_2301_11913_b200.swarm import Placement
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    margs = _ap.Namespace(model=model, micro_batch=getattr(args, "micro_batch", None) if model == args.model else None)
    mcfg = model_config(margs)
    M = args.microbatches
    layout, peer_rank, place_desc = engine_placement(args, world, S)
    P = max(layout)
    # trainers (microbatch pipelines in flight): 8 with one peer per stage, 16 with the balanced
    # placement's several (at least one per peer) -- the counts measured (§ engine_placement)
    tpp = args.trainers_per_peer or max(1, (TRAINERS if peer_rank is None else 2 * TRAINERS) // sum(layout))
    bm = 2.0
    # tick period: M microbatch completions of the engine's own schedule (its virtual
    # completion rate for this layout, from a throwaway run without ticks), so every
    # stage takes one optimizer step per M microbatches
    horizon = 400.0 * M * (1.0 + bm) / P
    cal = Engine(EngineConfig(n_stages=S, initial_peers=[[1.0] * layout[s] for s in range(S)],
                              forward_service_seconds=1.0, backward_multiplier=bm,
                              trainers_per_peer=tpp, duration_seconds=horizon,
                              bucket_seconds=horizon / 8), seed=1)
    while cal.next(4096):
        pass
    period = M * horizon / max(cal.summary()["completed"], 1)
    ex = EngineExecutor(mcfg, S, trainers_per_peer=tpp, seed=1, lr=1e-4, forward_seconds=1.0,
                        backward_multiplier=bm, allreduce_period=period, allreduce_stall=0.05,
                        stream_per_peer=not args.single_stream, lanes=args.lanes, fp32=fp32,
                        dpu=bool(getattr(args, "dpu", False)), layout=layout, peer_rank=peer_rank,
                        pair_wgrad=not getattr(args, "no_pair_wgrad", False))
    stream = torch.cuda.current_stream()
    # untimed warm-up: W steps plus two more (eight more with several peers per stage, whose
    # routes mix trainer pairs more), so that the visit graphs of most (peer, trainer pair, lane)
    # combinations are captured before the timed region
    ex.run(M * (warmup + (8 if P > 1 else 2)))
    ex.finish()
    warm_until_no_captures(ex, M, world)
    torch.cuda.synchronize()
    ex.loss_sum.zero_()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    barrier(world)
    torch.cuda.synchronize()
    n0 = ex.kernels_launched()
    v0, r0, t_0, c0 = ex.engine.summary()["now"], ex.records, ex.optimizer_steps, ex.captures
    tick0 = ex.tick_time()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    done = ex.run(M * steps)
    v1, r1, t_1, c1 = ex.engine.summary()["now"], ex.records, ex.optimizer_steps, ex.captures
    ex.finish()
    t1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clocks = clk.stop()
    launches = int(ex.kernels_launched() - n0)
    tick1 = ex.tick_time()
    local_peers = sum(1 for pid in range(ex.n_peers) if ex.peer_info(pid)["alive"] and ex.peer_info(pid)["rank"] == rank)
    ms_rank = t0.elapsed_time(t1)
    ms = max_over_ranks(ms_rank, world)
    tokens = done * mcfg.tokens
    value = tokens / (ms / 1e3)
    loss = ex.loss_sum.clone()
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(loss)
    res = {"value": value, "ms_per_step": ms / steps, "steps": steps, "warmup": warmup, "clocks": clocks,
           "gpu_launches": launches, "tokens_per_step": M * mcfg.tokens,
           "run": {"execution": "asynchronous SWARM: the reference DES engine's record order (csrc/engine.cpp, "
                                "decision-identical to sim::run) walked by the C++ host driver (csrc/driver.cpp), one "
                                "compute stream per peer, raw-NCCL send/recv of int8 wire messages, stage all-reduce "
                                "+ AdamW at every AllReduceTick",
                   "arithmetic": "fp32 (SIMT fp32 GEMMs, fp32 activations)" if fp32 else
                                 "bf16 storage, tcgen05 GEMMs with fp32 accumulation",
                   "placement": place_desc, "peer_rank": peer_rank, "trainers": ex.T,
                   "trainers_per_peer": tpp, "lanes_per_peer": args.lanes,
                   "schedule": "forward 1.0 / backward 2.0 virtual s, AllReduceTick every "
                               f"{period:.4g} virtual s (= {M} completions at the schedule's own rate: one optimizer "
                               f"step per stage per {M} microbatches); one step = {M} microbatch completions",
                   "optimizer": "AdamW (fused, fp32 master), paired weight gradients" + (
                       ", delayed parameter updates (tick all-reduce + AdamW overlapped with the next interval)"
                       if getattr(args, "dpu", False) else ""),
                   "tick_cost": {"ms_per_step_per_peer_stream": (tick1[0] - tick0[0]) / steps / max(local_peers, 1),
                                 "share_of_step": (tick1[0] - tick0[0]) / steps / max(local_peers, 1) / (ms_rank / steps),
                                 "stretches": tick1[1] - tick0[1], "local_peer_streams": local_peers,
                                 "what": "GPU time a peer's compute stream spends in a tick (gradient sum, NCCL "
                                         "all-reduce, AdamW) or, with DPU, blocked at the first visit after one "
                                         "(rank 0)"},
                   "mean_loss": float(loss.item()) / max(tokens, 1),
                   "model_tflops_per_s": value * mcfg.flops_per_token(S) / 1e12,
                   "model_flops_per_token": mcfg.flops_per_token(S)},
           "engine": {"records": r1 - r0, "virtual_seconds": v1 - v0, "optimizer_steps_rank": t_1 - t_0,
                      "microbatches": done, "graph_captures_in_timed_region_rank0": c1 - c0}}
    # e2e: every microbatch's tokens / targets H2D from pinned host memory inside the visit
    # that consumes them, the loss D2H after every step's M completions
    if e2e_steps > 0:
        ex.use_host_pool(True)
        hloss = torch.empty(1, dtype=torch.float32).pin_memory()
        lst = ex.last_stage_stream()
        ex.run(M)  # untimed: warm the host-pool path
        ex.finish()
        warm_until_no_captures(ex, M, world)
        barrier(world)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e2e_done = 0
        cap0 = ex.counters()["captures"]
        rd = torch.cuda.Stream()  # a torch-owned stream reads the loss (the driver's streams die with it)
        for _ in range(e2e_steps):
            e2e_done += ex.run(M)
            if lst is not None:
                rd.wait_stream(lst)
                with torch.cuda.stream(rd):
                    hloss.copy_(ex.loss_sum, non_blocking=True)
        ex.finish()
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(time.perf_counter() - w0, world)
        ex.use_host_pool(False)
        res["e2e"] = {"value": e2e_done * mcfg.tokens / e2e_s, "unit": "tokens/s",
                      "h2d_bytes_per_step": int(M * mcfg.tokens * 4 * 2), "d2h_bytes_per_step": 4,
                      "steps": e2e_steps, "graph_captures_in_timed_region": ex.counters()["captures"] - cap0,
                      "path": "EngineExecutor.run (C++ driver) with each microbatch's tokens / targets copied from "
                              "pinned host memory by its consuming visit and the loss read back after every step "
                              "(wall clock, max over ranks)"}
    if profile:
        # live roofline: one more step as a profiled region -- every visit eager on one stream behind
        # a GPU spin, CUDA events around every kernel -- so each GEMM is timed alone
        pr = ex.profile(M)
        pk = peaks()
        achieved = pr["gemm_flops"] / (pr["gemm_ms"] / 1e3) / 1e12 if pr["gemm_ms"] > 0 else 0.0
        kern_ms = sum(v[0] for v in pr["categories"].values())
        traffic = {}
        prof = os.path.join(ROOT, "profiles", "ncu_gemm_qkv_traffic.json")
        if os.path.exists(prof):
            with open(prof) as f:
                traffic = json.load(f)
        res["roofline"] = {
            "bound": "tensor", "kernel": "k_gemm / k_gemm2 (tcgen05 bf16: every block, attention and head GEMM)",
            "achieved": achieved, "peak": pk["bf16_tflops"], "unit": "TFLOP/s", "frac": achieved / pk["bf16_tflops"],
            "frac_of_sustained_peak": achieved / (pk["bf16_tflops_sustained"] or pk["bf16_tflops"]),
            "traffic": traffic.get("dram_bytes_per_launch"), "traffic_note": traffic.get("note"),
            "peak_source": pk["source"] + " bf16 burst (the kernels are timed alone)",
            "gemm_ms_per_step": pr["gemm_ms"], "gemm_flops_per_step": pr["gemm_flops"],
            "gemm_launches_per_step": pr["gemm_launches"],
            "gemm_share_of_kernel_time": pr["gemm_ms"] / kern_ms if kern_ms else None,
            "per_shape": [{"shape": k, "ms_per_step": v[0], "tflops": v[1] / (v[0] / 1e3) / 1e12 if v[0] else None,
                           "launches": v[2], "share_of_gemm_time": v[0] / pr["gemm_ms"] if pr["gemm_ms"] else None}
                          for k, v in sorted(pr["shapes"].items(), key=lambda kv: -kv[1][0])[:16]],
            "note": "one extra step of the same engine-driven run as a profiled region: every visit issued eagerly "
                    "on one stream behind a GPU spin (swarm_driver_profile_begin), CUDA events around each kernel; "
                    "achieved = executed GEMM FLOPs / summed GEMM event time of that step (this rank)"}
        res["step_breakdown"] = {
            "note": "isolated kernel time per category over one profiled step (this rank, kernels serialised); the "
                    "headline step overlaps peers' kernels on several streams, so the sum can exceed ms_per_step",
            **{c: {"ms_per_step": v[0], "launches": int(v[1])} for c, v in pr["categories"].items()}}
    res["_ex"] = ex
    return res


def bench_engine(args, world, rank, local):
    """The headline: BASELINE configs[2] (or --model) through the C++ driver (run_engine)."""
    S = args.stages
    r = run_engine(args, world, rank, local, args.model, S, args.steps, args.warmup)
    r.pop("_ex")
    mcfg = shape_of(args)
    line = {"metric": "training tokens/s (SWARM pipeline)", "value": r["value"], "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic tokens uniform over the vocab (per-trainer pool), random-init weights",
            "config": train_config(args, world), **{k: r[k] for k in ("run", "engine", "e2e", "gpu_launches",
                                                                      "clocks", "roofline", "step_breakdown")
                                                   if k in r}}
    line["cost_model"] = cost_model_report(model_config(args), S, args.microbatches, world,
                                           (r["ms_per_step"] / 1e3), measure_link(world, rank))
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tok_s, thr, sample = cpu_block_baseline(mcfg)
        line["cpu_baseline"] = {"value": tok_s, "unit": "tokens/s", "cores": thr, "kind": "port", "sample": sample}
    return line


def sub_config(args, world, model, S, which, steps, warmup, fp32=False) -> dict:
    """A second BASELINE config measured in the same run (a sub-object of the line)."""
    import gc

    import torch
    ns = argparse.Namespace(**{**vars(args), "model": model, "stages": S, "micro_batch": None})
    r = run_engine(ns, world, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")), model, S,
                   steps, warmup, fp32=fp32, profile=not fp32, e2e_steps=1)
    r.pop("_ex")
    gc.collect()
    torch.cuda.empty_cache()
    out = {"metric": "training tokens/s (SWARM pipeline)", "value": r["value"], "unit": "tokens/s",
           "ms_per_step": r["ms_per_step"], "steps": steps, "warmup": warmup, "dtype": "f32" if fp32 else "bf16",
           "config": {**train_config(ns, world), "which": which},
           **{k: r[k] for k in ("run", "e2e", "gpu_launches", "clocks", "roofline") if k in r}}
    return out


# ----------------------------------------------------------------- failure
def bench_failure(args, world, rank, local):
    """BASELINE configs[4]: peer failure + adaptive rebalancing,
    asynchronously through the engine and the C++ driver.  The reference Engine's own
    schedule (csrc/engine.cpp, decision-identical to sim::run incl. churn and Alg. 2 on
    the queue-length time-integral average_load, sim.cpp:378-393) starts one stage short
    of peers, rebalances periodically, and loses a peer mid-run (a churn-trace leave);
    the driver executes it: requeued jobs, backward recompute where the forward peer is
    gone, migration as a real NCCL download of params + AdamW state.  Each segment
    between membership changes is timed on the device; the CPU reference is the
    unmodified sim::run (oracle/_ref) on the same SimConfig and seed."""
    import ctypes as C

    import torch

    from paper_2301_11913_b200.engine import EngineConfig
    from paper_2301_11913_b200.executor import EngineExecutor
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    mcfg = model_config(args)
    S = 2 if world <= 4 else args.stages
    P0 = max(world, 4)  # peers: one per GPU from 4 GPUs on (2 GPUs host 2 each)
    layout = [P0 - S + 1, 1] if S == 2 else [3, 1] + [2] * (S - 2)
    head = 1.0 + mcfg.vocab * mcfg.d_model / (mcfg.layers_per_stage * mcfg.params_per_layer())
    speeds = [[1.0] * n for n in layout[:-1]] + [[1.0 / head] * layout[-1]]
    fwd = 6.3e-3  # measured forward visit (configs[2] stage, B200): virtual time ~ real time
    state_bytes = mcfg.params_per_layer() * mcfg.layers_per_stage * 6  # rebalancer.cpp:71-75
    cfg = EngineConfig(n_stages=S, initial_peers=speeds, forward_service_seconds=fwd, trainers_per_peer=2,
                       allreduce_period=0.5, allreduce_stall=1e-3, duration_seconds=17.9, bucket_seconds=0.5,
                       churn=[(9.0, -1)], rebalance_period=6.0, straggler_timeout=0.05, propagation_delay=0.01,
                       announce_ttl=300.0, state_transfer_bytes=state_bytes, download_bps=8 * 400e9)
    ex = EngineExecutor(mcfg, S, seed=1, lr=1e-4, sim=cfg, lanes=args.lanes if world > 1 else 1,
                        use_graphs=not args.no_graphs)
    n_peers0 = ex.n_peers

    def layout_now():
        out = [0] * S
        for pid in range(ex.n_peers):
            i = ex.peer_info(pid)
            if i["alive"] and not i["migrating"]:
                out[i["stage"]] += 1
        return out

    segments = []
    ex.run(32)  # untimed: most visit graphs captured before the first timed segment
    ex.finish()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    v_now = lambda: ex.engine.summary()["now"]  # noqa: E731
    warm = 48  # per segment: the first microbatches after a membership change run untimed (a migrated
    # peer's new stage captures its visit graphs there; requeued work drains)
    while True:
        c0, t_v0 = ex.counters(), v_now()
        # the membership record the previous segment stopped in front of is processed first (stage
        # re-created, communicators re-split, state downloaded: untimed), then the warm-up
        nw = ex.run_until(warm, -2)
        ex.finish()
        torch.cuda.synchronize()
        lay = layout_now()
        if nw < warm:  # the next membership change came inside the warm-up: a transition
            c1 = ex.counters()
            if nw == 0 and c1["records"] == c0["records"]:
                break
            segments.append({"layout": lay, "microbatches": nw, "ms": None, "tokens_per_s": None,
                             "virtual_s": [t_v0, v_now()], "recomputes": c1["recomputes"] - c0["recomputes"],
                             "state_bytes": c1["state_bytes"] - c0["state_bytes"],
                             "note": "transition (shorter than the untimed warm-up)"})
            if v_now() >= cfg.duration_seconds or len(segments) > 12:
                break
            continue
        barrier(world)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        n = ex.run_until(10 ** 9, -2)
        ex.finish()
        t1.record(stream)
        torch.cuda.synchronize()
        ms = max_over_ranks(t0.elapsed_time(t1), world)
        c1 = ex.counters()
        segments.append({"layout": lay, "microbatches": n, "untimed_warmup_microbatches": nw, "ms": ms,
                         "tokens_per_s": n * mcfg.tokens / (ms / 1e3) if ms > 0 and n > 0 else None,
                         "virtual_s": [t_v0, v_now()], "recomputes": c1["recomputes"] - c0["recomputes"],
                         "state_bytes": c1["state_bytes"] - c0["state_bytes"]})
        if v_now() >= cfg.duration_seconds or len(segments) > 12:
            break
    from paper_2301_11913_b200.engine import Engine, LEAVE, MIGRATE, MIGRATED, REBALANCE
    decisions = [{"t": r.time, "kind": {LEAVE: "leave", MIGRATE: "migrate", MIGRATED: "migrated",
                                        REBALANCE: "rebalance"}[r.kind], "peer": r.worker, "stage": r.stage,
                  "from": r.from_worker} for r in Engine(cfg, 1).records() if r.kind in (LEAVE, MIGRATE, MIGRATED,
                                                                                         REBALANCE)]
    ref = None
    if rank == 0:
        try:
            import oracle as O
            if O.ref is not None:
                counts = (C.c_uint64 * 4)()
                nb = C.c_size_t()
                b = (C.c_double * 4096)()
                ts = (C.c_double * 1)(*[t for t, _ in cfg.churn])
                ds = (C.c_int64 * 1)(*[d for _, d in cfg.churn])
                rc = O.ref.ref_sim_run_churn(cfg.to_reference_json().encode(), ts, ds, 1, 1, counts, b, 4096,
                                             C.byref(nb), None, 0)
                ref = {"kind": "reference sim::run (oracle/_ref, unmodified P/src/sim.cpp) on the same SimConfig, "
                               "churn trace and seed",
                       "dispatched": counts[0], "completed": counts[1], "requeued": counts[2], "abandoned": counts[3],
                       "completions_per_bucket": list(b)[: nb.value], "bucket_seconds": cfg.bucket_seconds,
                       "driver_completed_same_schedule": int(ex.engine.summary()["completed"]),
                       "oracle_throughput_for_n_peers": {
                           str(sum(seg["layout"])): O.ref.ref_oracle_throughput(
                               (C.c_double * S)(*([1.0 / (3 * fwd)] * (S - 1) + [1.0 / (3 * fwd * head)])), S,
                               sum(seg["layout"])) * mcfg.tokens for seg in segments}}
        except Exception as e:  # the prediction is a report, not part of the measured path
            ref = {"unavailable": repr(e)[:200]}
    steady = [sg for sg in segments if sg["tokens_per_s"]]
    last = steady[-1] if steady else segments[-1]
    return {"metric": "training tokens/s per membership segment (peer failure + adaptive rebalancing)",
            "value": last["tokens_per_s"], "unit": "tokens/s", "n_gpus": world, "steps": len(segments),
            "warmup": 1, "ms_per_step": last["ms"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"BASELINE configs[4]: failure + rebalancing, {S} stages of the configs[2] "
                                   f"block (d 2048, {mcfg.layers_per_stage} layers/stage), initial layout {layout}, "
                                   f"{n_peers0} peers on {world} GPU(s), one peer leaves at t = 9 s",
                       "model": args.model, "stages": S, "initial_layout": layout,
                       "schedule": "engine (= sim::run) with RebalanceMode::Periodic every 6 s, straggler timeout "
                                   "50 ms, churn trace [(9 s, -1)], AllReduceTick every 0.5 s, 17.9 s; forward visit "
                                   f"{fwd * 1e3:.1f} ms so engine time tracks real time; last stage slowed by its LM "
                                   f"head ({head:.3f}x)"},
            "segments": segments, "decisions": decisions, "driver": ex.counters(), "reference": ref,
            "gpu_launches": int(ex.kernels_launched())}


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU implementation of the path on this
    box's host cores (rank 0 only).  train: the block oracle port (the reference
    has no training path); codec: the unmodified reference codec (oracle/_ref)."""
    if rank != 0:
        return None
    if args.workload in ("train", "engine"):
        m = shape_of(args)
        tok_s, step_s, thr, sample = cpu_block_reference_steps(m, args.steps, args.warmup)
        return {"impl": "reference", "metric": "training tokens/s (SWARM pipeline)", "value": tok_s,
                "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": step_s * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32 (CPU)", "data": "synthetic",
                "config": train_config(args, world),
                "run": {"execution": "CPU block oracle on rank 0's host cores (the reference has no training path)",
                        "tokens_per_step": m.tokens / (m.layers_per_stage * TRAIN_STAGES)},
                "cpu_baseline": {"value": tok_s, "unit": "tokens/s", "cores": thr, "kind": "port", "sample": sample},
                "e2e": {"value": tok_s, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    threads = os.cpu_count() or 1
    # each step is the bounded 256 MiB sample (~0.07 s on 16 threads): K steps fit a few minutes;
    # the cap only guards an extreme K
    steps = max(1, min(args.steps, 2000))
    gbs, kind, thr, sample = cpu_reference_codec(steps, min(args.warmup, 3), threads)
    bytes_step = (CODEC_BYTES_Q + CODEC_BYTES_DQ) * (CPU_SAMPLE_N / CODEC_N)
    return {"impl": "reference",
            "metric": "int8 codec GB/s (blockwise absmax quantize+dequantize, algorithmic bytes)",
            "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": steps, "warmup": min(args.warmup, 3),
            "ms_per_step": bytes_step / (gbs * 1e9) * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64 (reference std::vector<double>)", "data": "synthetic",
            "config": {"workload": "codec sweep, reference CPU path on a bounded sample", "block_size": CODEC_BS},
            "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": thr, "kind": kind, "sample": sample},
            "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="train", choices=["train", "codec", "failure", "engine"],
                    help="train (default): the engine-driven headline + codec + configs[0] / configs[3] sub-lines; "
                         "engine: the headline only")
    ap.add_argument("--trainers-per-peer", type=int, default=None,
                    help="engine: trainers per peer (sim trainers_per_peer; default: 8 trainers in all, 16 with the "
                         "balanced placement, >= 1 per peer)")
    ap.add_argument("--single-stream", action="store_true", help="engine: one compute stream per GPU (not per peer)")
    ap.add_argument("--lanes", type=int, default=None,
                    help="engine: visits a peer may serve concurrently, each on its own stream and workspace set "
                         "(default 2 on >= 2 GPUs: +3-5%% configs[2], +10%% configs[3]; 1 on one GPU, where the "
                         "4 peers already share the GPU on 4 streams)")
    ap.add_argument("--model", default="C", choices=["C", "D", "tiny"])
    ap.add_argument("--microbatches", type=int, default=TRAIN_MICROBATCHES)
    ap.add_argument("--micro-batch", type=int, default=None, help="sequences per microbatch (default: the preset's)")
    ap.add_argument("--dpu", action="store_true",
                    help="train: delayed parameter updates (PAPER:204): all-reduce + AdamW of step t overlap step t+1")
    ap.add_argument("--stages", type=int, default=TRAIN_STAGES, help="pipeline stages (default 4, SURVEY §8(d))")
    ap.add_argument("--no-pair-wgrad", action="store_true",
                    help="engine: each backward visit's weight gradients alone (no pairing with the pending visit)")
    ap.add_argument("--placement", default=None, choices=["balanced", "contiguous"],
                    help="engine, several GPUs: peers per stage and their GPUs (bench.engine_placement; default "
                         "balanced from 4 GPUs, contiguous below)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-codec", action="store_true", help="train: skip the codec sub-measurement")
    ap.add_argument("--no-extra", action="store_true", help="train: skip the configs[0] / configs[3] sub-lines")
    ap.add_argument("--no-graphs", action="store_true", help="failure: eager visits (no CUDA-graph capture / replay)")
    ap.add_argument("--sync", action="store_true",
                    help="train: headline = the synchronous GPipe step (default: the asynchronous engine-driven "
                         "pipeline, with the GPipe step reported beside it)")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = {"train": 6, "failure": 3, "engine": 6}.get(args.workload, 1000)
    if args.warmup is None:
        args.warmup = {"train": 3, "failure": 3, "engine": 3}.get(args.workload, 10)
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_setup(args)
    if args.lanes is None:
        args.lanes = 2 if world >= 2 and not args.single_stream else 1
    elif args.lanes > 1 and args.single_stream:
        ap.error("--lanes > 1 needs a stream per peer (drop --single-stream)")
    if args.impl == "reference":
        line = run_reference(args, world, rank)
    elif args.workload == "codec":
        line = bench_codec(args, world, rank, local)
    elif args.workload == "failure":
        line = bench_failure(args, world, rank, local)
    elif args.workload == "engine":
        line = bench_engine(args, world, rank, local)
    elif args.sync:
        line = bench_train(args, world, rank, local)
    else:
        # headline: the asynchronous engine-driven pipeline through the C++ driver,
        # with its live roofline, e2e, cost model and CPU baseline; then the other BASELINE configs
        import gc

        import torch
        line = bench_engine(args, world, rank, local)
        gc.collect()
        torch.cuda.empty_cache()
        if not args.no_codec:
            c = bench_codec(argparse.Namespace(steps=200, warmup=5, no_cpu_baseline=args.no_cpu_baseline, e2e_steps=2),
                            world, rank, local)
            line["codec"] = {k: c[k] for k in ("metric", "value", "unit", "ms_per_step", "steps", "config", "roofline",
                                               "e2e", "sweep", "parity_ok", "cpu_baseline", "gpu_launches") if k in c}
            gc.collect()
            torch.cuda.empty_cache()
        if not args.no_extra and args.model == "C":
            line["configs0_tiny_fp32"] = sub_config(
                args, world, "tiny", 2, "BASELINE configs[0]: tiny 2-stage pipeline, 2 layers/stage, d 256, seq 128, "
                "batch 8, fp32 arithmetic, int8 boundary codec (a parity config: launch-bound)", 6, 3, fp32=True)
            line["configs3_paper_scale"] = sub_config(
                args, world, "D", args.stages, "BASELINE configs[3]: d 4096, 32 heads, 16 shared layers/stage, "
                "maxout k=2 + int8 boundary", 3, 3)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
