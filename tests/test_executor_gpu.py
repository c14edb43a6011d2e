"""GPU: the engine-driven executor (executor.py) runs the
reference engine's schedule for real.  With no all-reduce tick (weights fixed)
every stage's accumulated gradient must equal a sequential recomputation of
exactly the visits the schedule ran (fp32 accumulation order differs: relative
Frobenius error <= 1e-4); with ticks the asynchronous pipeline trains."""
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


@pytest.mark.parametrize("streams,lanes", [(True, 1), (False, 1), (True, 2)])
@pytest.mark.parametrize("pair", [True, False])
@pytest.mark.parametrize("S,tpp", [(4, 1), (2, 3), (3, 2)])
def test_executor_gradients_match_sequential_visits(cuda, S, tpp, pair, streams, lanes):
    import torch
    from paper_2301_11913_b200.executor import EngineExecutor, sequential_reference_grads
    from paper_2301_11913_b200.swarm import PRESETS
    ex = EngineExecutor(PRESETS["tiny"], S, trainers_per_peer=tpp, seed=5, n_pool=5, pair_wgrad=pair,
                        stream_per_peer=streams, lanes=lanes)
    assert ex.run(7) == 7
    ex.finish()
    torch.cuda.synchronize()
    assert all(len(v) > 0 for v in ex.bwd_log)
    ex.flush_wgrad()
    ref = sequential_reference_grads(ex)
    for pid, st in ex.stages.items():
        assert rel(st.grads(), ref[pid]) <= 1e-4, (pid, rel(st.grads(), ref[pid]))
    assert torch.isfinite(ex.loss_sum).all()


@pytest.mark.parametrize("lanes", [1, 2])
def test_executor_trains_with_allreduce_ticks(cuda, lanes):
    import torch
    from paper_2301_11913_b200.executor import EngineExecutor
    from paper_2301_11913_b200.swarm import PRESETS
    ex = EngineExecutor(PRESETS["tiny"], 4, trainers_per_peer=2, seed=3, lr=3e-3, n_pool=2,
                        forward_seconds=1.0, allreduce_period=12.0, allreduce_stall=0.1, lanes=lanes)
    curve = []
    for _ in range(8):
        ex.loss_sum.zero_()
        n = ex.run(8)
        ex.finish()
        curve.append(ex.loss_sum.item() / max(n, 1) / ex.m.tokens)  # loss_sum holds token CE sums
    assert ex.optimizer_steps > 0 and ex.ticks > 0
    assert all(c == c for c in curve)
    assert curve[-1] < curve[0] - 0.3, curve
    ms, spans = ex.tick_time()  # the ticks' GPU time on the peer streams was measured
    assert spans >= ex.ticks and ms > 0.0, (ms, spans)


@pytest.mark.parametrize("lanes", [1, 2])
def test_executor_maxout_shared_layers_with_lanes(cuda, lanes):
    """configs[3]'s stage features on the tiny model: maxout bottleneck at the
    boundaries and layer-shared blocks (stacked weight gradients), two lanes per
    peer: gradients still equal the sequential replay."""
    import dataclasses

    import torch
    from paper_2301_11913_b200.executor import EngineExecutor, sequential_reference_grads
    from paper_2301_11913_b200.swarm import PRESETS
    m = dataclasses.replace(PRESETS["tiny"], maxout_k=2, shared_layers=1, layers_per_stage=3)
    ex = EngineExecutor(m, 3, trainers_per_peer=2, seed=7, n_pool=4, lanes=lanes)
    assert ex.run(6) == 6
    ex.finish()
    ex.flush_wgrad()
    torch.cuda.synchronize()
    ref = sequential_reference_grads(ex)
    for pid, st in ex.stages.items():
        assert rel(st.grads(), ref[pid]) <= 1e-4, (pid, rel(st.grads(), ref[pid]))


@pytest.mark.parametrize("lanes", [1, 2])
@pytest.mark.parametrize("S,tpp", [(2, 2), (4, 1)])
def test_native_driver_matches_python_orchestrator(cuda, S, tpp, lanes):
    """Two independent host implementations of the data plane — the C++ driver
    (csrc/driver.cpp) and the Python record walk (PyEngineExecutor) — run the same
    engine schedule on the same pool: same visit log, same gradients (up to the
    fp32 summation order of concurrent atomic accumulation)."""
    import torch
    from paper_2301_11913_b200.executor import EngineExecutor, PyEngineExecutor
    from paper_2301_11913_b200.swarm import PRESETS
    nat = EngineExecutor(PRESETS["tiny"], S, trainers_per_peer=tpp, seed=9, n_pool=4, lanes=lanes)
    py = PyEngineExecutor(PRESETS["tiny"], S, trainers_per_peer=tpp, seed=9, lanes=lanes,
                          tokens=nat.pool_tok.cpu(), targets=nat.pool_tgt.cpu())
    assert nat.run(9) == 9 and py.run(9) == 9
    nat.finish()
    py.finish()
    nat.flush_wgrad()
    py.flush_wgrad()
    torch.cuda.synchronize()
    assert nat.visit_log == [(t, k, s, b, p) for t, k, s, b, p in py.visit_log]
    assert abs(nat.loss_sum.item() - py.loss_sum.item()) <= 1e-5 * abs(py.loss_sum.item())
    for pid in nat.stages:
        g1, g2 = nat.stages[pid].grads(), py.stages[pid].grads()
        assert rel(g1, g2) <= 1e-5, (pid, rel(g1, g2))


def test_lanes_do_not_change_the_result_across_ticks(cuda):
    """the lane join / fork around ALLREDUCE ticks.  The same schedule with
    ticks at lanes = 1 and lanes = 2: after several ticks (all-reduce + AdamW) the
    parameters agree within fp32 summation-order noise."""
    import torch
    from paper_2301_11913_b200.executor import EngineExecutor
    from paper_2301_11913_b200.swarm import PRESETS
    runs = []
    for lanes in (1, 2):
        ex = EngineExecutor(PRESETS["tiny"], 4, trainers_per_peer=2, seed=4, lr=1e-3, n_pool=3, lanes=lanes,
                            allreduce_period=10.0, allreduce_stall=0.1)
        ex.run(24)
        ex.finish()
        torch.cuda.synchronize()
        assert ex.optimizer_steps >= 4
        runs.append({pid: st.params().clone() for pid, st in ex.stages.items()})
        runs[-1]["loss"] = ex.loss_sum.clone()
    for pid in runs[0]:
        assert rel(runs[1][pid], runs[0][pid]) <= 1e-5, pid


def test_engine_dpu_semantics(cuda):
    """Delayed parameter updates under the engine schedule (driver dpu=1): at each tick
    the interval's gradients (bank b) are applied on an update stream while the next interval
    computes on the other bank, whose weights are one optimizer step older."""
    import torch
    from paper_2301_11913_b200.engine import ALLREDUCE
    from paper_2301_11913_b200.executor import EngineExecutor
    from paper_2301_11913_b200.swarm import PRESETS
    ex = EngineExecutor(PRESETS["tiny"], 2, trainers_per_peer=2, seed=4, lr=1e-3, n_pool=3, dpu=True,
                        allreduce_period=10.0, allreduce_stall=0.1)
    w0 = {pid: st.params().clone() for pid, st in ex.stages.items()}
    ex.run_until(10 ** 6, ALLREDUCE)  # through the first tick: update 1 applied to bank 0
    ex.finish()
    torch.cuda.synchronize()
    for pid, st in ex.stages.items():
        assert torch.equal(st.params_bf16_bank(1), w0[pid].bfloat16())  # bank 1: still the initial weights
        assert torch.equal(st.params_bf16_bank(0), st.params().bfloat16())  # bank 0: after update 1
        assert not torch.equal(st.params(), w0[pid])
        assert float(st.grads_bank(0).abs().max()) == 0.0  # applied and zeroed
    ex.run(3)  # the next interval computes on bank 1 (one step of delay) and accumulates there
    ex.finish()
    torch.cuda.synchronize()
    for pid, st in ex.stages.items():
        assert float(st.grads_bank(1).abs().max()) > 0.0
        assert float(st.grads_bank(0).abs().max()) == 0.0
    curve = []
    for _ in range(6):
        ex.loss_sum.zero_()
        n = ex.run(8)
        ex.finish()
        curve.append(ex.loss_sum.item() / max(n, 1) / ex.m.tokens)
    assert ex.optimizer_steps >= 4 and curve[-1] < curve[0] - 0.2, curve


@pytest.mark.parametrize("layout", [[2, 1, 1, 2], [1, 3]])
def test_executor_explicit_layout_and_peer_rank(cuda, layout):
    """An explicit layout (several peers per stage on one GPU, whose gradients are summed locally) and
    an explicit peer_rank (swarm_driver_config.peer_rank, all 0 on one GPU) drive the same engine: every
    peer's gradient equals the sequential replay of the visits it ran."""
    import torch
    from paper_2301_11913_b200.executor import EngineExecutor, sequential_reference_grads
    from paper_2301_11913_b200.swarm import PRESETS
    S = len(layout)
    ex = EngineExecutor(PRESETS["tiny"], S, trainers_per_peer=1, seed=7, n_pool=5, layout=layout,
                        peer_rank=[0] * sum(layout))
    assert ex.n_peers == sum(layout)
    assert [ex.peer_info(p)["stage"] for p in range(ex.n_peers)] == [s for s in range(S) for _ in range(layout[s])]
    assert ex.run(6) == 6
    ex.finish()
    torch.cuda.synchronize()
    ex.flush_wgrad()
    ref = sequential_reference_grads(ex)
    for pid, st in ex.stages.items():
        assert rel(st.grads(), ref[pid]) <= 1e-4, (pid, rel(st.grads(), ref[pid]))
