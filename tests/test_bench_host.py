"""Host-side bench helpers (no GPU): the calibrated cost-model report, including
the DES engine's asynchronous prediction, is well-formed and monotone in the GPU
count; the engine's tick period calibration gives one tick per 32 completions."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_cost_model_report_predictions():
    import bench
    from paper_2301_11913_b200.swarm import PRESETS
    r = bench.cost_model_report(PRESETS["C"], 4, 32, 1, 0.78, None)
    g = r["predicted_tokens_per_s"]
    assert g["1"] < g["2"] < g["4"] < g["8"]
    e = r["engine_predicted_tokens_per_s"]
    assert 0 < e["4"] < e["8"]
    # the LM-head stage bounds the asynchronous pipeline: below 4x the 1-GPU rate at 4 GPUs
    assert e["4"] < 4 * g["1"]
    assert abs(r["head_stage_ratio"] - (1 + 50304 * 2048 / (8 * PRESETS["C"].params_per_layer()))) < 1e-12


def test_engine_tick_period_matches_completions():
    from paper_2301_11913_b200.engine import ALLREDUCE, DONE, Engine, EngineConfig
    M, horizon = 32, 400.0 * 32 * 3
    cfg = dict(n_stages=4, initial_peers=[[1.0]] * 4, trainers_per_peer=2)
    cal = Engine(EngineConfig(**cfg, duration_seconds=horizon, bucket_seconds=horizon / 8), 1)
    while cal.next(4096):
        pass
    period = M * horizon / cal.summary()["completed"]
    e = Engine(EngineConfig(**cfg, allreduce_period=period, allreduce_stall=0.01, duration_seconds=50 * period,
                            bucket_seconds=period), 1)
    done, per_tick = 0, []
    for r in e.records():
        if r.kind == DONE:
            done += 1
        elif r.kind == ALLREDUCE:
            per_tick.append(done)
            done = 0
    steady = per_tick[5:]
    assert steady and abs(sum(steady) / len(steady) - M) <= 2


def test_bench_shapes_mirror_the_product_presets():
    import bench
    from paper_2301_11913_b200.swarm import PRESETS
    for name, p in PRESETS.items():
        s = bench.SHAPES[name]
        for f in ("d_model", "n_heads", "d_ffn", "seq_len", "micro_batch", "layers_per_stage", "vocab",
                  "shared_layers", "maxout_k", "block_size"):
            assert getattr(s, f) == getattr(p, f), (name, f)
        assert s.flops_per_token(4) == p.flops_per_token(4)


def test_reference_arm_runs_without_the_product_package():
    """--impl reference times the CPU path only: it must not load paper_2301_11913_b200 (nor its
    .so files), its config must equal the GPU arm's, and K steps must take about K x ms_per_step."""
    import json
    import subprocess
    import time
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--model', 'tiny', '--steps', '3', "
            "'--warmup', '3']; runpy.run_path('bench.py', run_name='__main__'); "
            "bad = [m for m in sys.modules if m.startswith('paper_2301_11913_b200')]; "
            "print('LOADED', bad)")
    t0 = time.perf_counter()
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    wall = time.perf_counter() - t0
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    assert lines[-1] == "LOADED []"
    j = json.loads(lines[-2])
    assert j["impl"] == "reference" and j["steps"] == 3
    assert j["ms_per_step"] * (j["steps"] + j["warmup"]) / 1e3 <= wall
    import argparse

    import bench
    ns = argparse.Namespace(model="tiny", stages=4, microbatches=32, micro_batch=None)
    assert j["config"] == bench.train_config(ns, 1)


def test_engine_placement_layouts_and_trainers():
    """bench.engine_placement: contiguous below 4 GPUs, balanced from 4 (the defaults), and the
    balanced placement's invariants -- no GPU hosts two peers of one stage, the LM-head stage's peers
    sit beside lighter stages' peers, and the max GPU load drops below contiguous."""
    import argparse

    import bench
    C = argparse.Namespace(model="C", micro_batch=None, placement=None)
    for w, lay, balanced in ((1, [1, 1, 1, 1], False), (2, [1, 1, 1, 1], False), (4, [2, 2, 2, 2], True),
                             (8, [4, 4, 4, 4], True)):
        layout, peer_rank, desc = bench.engine_placement(C, w, 4)
        assert layout == lay and (peer_rank is not None) == balanced
    for w in (2, 4, 8):
        layout, peer_rank, _ = bench.engine_placement(argparse.Namespace(model="C", micro_batch=None,
                                                                         placement="contiguous"), w, 4)
        assert peer_rank is None and layout == ([1, 1, 1, 1] if w < 8 else [2, 2, 2, 2])
    B = argparse.Namespace(model="C", micro_batch=None, placement="balanced")
    head = 1 + 50304 * 2048 / (8 * (4 * 2048 * 2048 + 2 * 2048 * 8192))
    for w in (2, 4, 8):
        layout, peer_rank, desc = bench.engine_placement(B, w, 4)
        assert len(peer_rank) == sum(layout) and set(peer_rank) == set(range(w))
        stage = [s for s in range(4) for _ in range(layout[s])]
        hosted = {}
        load = [0.0] * w
        for pid, r in enumerate(peer_rank):
            assert stage[pid] not in hosted.setdefault(r, set()), (w, pid, r)
            hosted[r].add(stage[pid])
            load[r] += (head if stage[pid] == 3 else 1.0) / layout[stage[pid]]
        contiguous_max = head if w >= 4 else (1.0 + head) * (4 // w) / 2
        assert max(load) < contiguous_max - 1e-9, (w, load)
        assert "load-balanced" in desc


def test_reference_arm_config_matches_the_gpu_arm():
    """train_config (shared by both arms' JSON lines) depends on the placement description only through
    bench.engine_placement, which is pure arithmetic on the Shape (no product import)."""
    import argparse
    import subprocess
    import bench
    for w in (1, 2, 4, 8):
        a = argparse.Namespace(model="C", micro_batch=None, placement=None, stages=4, microbatches=32)
        assert bench.train_config(a, w)["parallelism"] == bench.engine_placement(a, w, 4)[2]
    r = subprocess.run([sys.executable, "-c", "import sys; sys.path.insert(0, %r); import bench, argparse; "
                        "bench.engine_placement(argparse.Namespace(model='C', micro_batch=None, placement='balanced'),"
                        " 8, 4); print('paper_2301_11913_b200' in sys.modules)" % ROOT],
                       capture_output=True, text=True, timeout=120)
    assert r.stdout.strip() == "False", r.stdout + r.stderr
