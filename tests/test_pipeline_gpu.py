"""GPU: the SWARM pipeline runtime on one device (all 4 stages local): routing
plan + stage visits + optimizer step train the tiny model end to end."""
import pytest

pytestmark = pytest.mark.gpu


def test_single_gpu_pipeline_trains(cuda):
    import torch
    from paper_2301_11913_b200.swarm import PRESETS, SwarmPipeline, synthetic_batch
    m = PRESETS["tiny"]
    pipe = SwarmPipeline(m, 4, n_microbatches=4, seed=3, lr=3e-3, profile=True)
    tok, tgt = synthetic_batch(m, 4, seed=1, device=cuda)
    tgt = torch.roll(tok, -1, dims=1)  # learnable: predict the next token of a fixed batch
    losses = []
    for _ in range(6):
        pipe.loss_sum.zero_()
        pipe.step(tok, tgt)
        losses.append(pipe.loss_sum.item() / pipe.tokens_per_step())
    assert all(x == x for x in losses)  # finite
    assert losses[-1] < losses[0] - 0.3, losses
    ms, flops, n = pipe.profile_read()
    assert n > 0 and ms > 0 and flops > 0
    # every microbatch visited every stage exactly once per direction on peer == stage (P = 1)
    assert pipe.last_routes == [[0, 1, 2, 3]] * 4


def test_stage_wire_bf16_path(cuda):
    """bf16 wire (no compression) between two stages reproduces the int8 path within codec error."""
    import torch
    from paper_2301_11913_b200.stage import WIRE_BF16, WIRE_INT8, Stage, StageConfig
    outs = {}
    for wire in (WIRE_BF16, WIRE_INT8):
        c0 = StageConfig(is_last=0, wire=wire, seed=9, micro_batch=2)
        c1 = StageConfig(is_first=0, wire=wire, seed=10, micro_batch=2)
        s0, s1 = Stage(c0), Stage(c1)
        tok = torch.arange(c0.tokens, device="cuda", dtype=torch.int32) % c0.vocab
        a = s0.new_wire()
        loss = torch.zeros(1, device="cuda")
        s0.forward(0, tok, out=a)
        s1.forward(0, a, targets=tok, loss_sum=loss, loss_scale=1.0)
        outs[wire] = loss.item()
    assert abs(outs[WIRE_BF16] - outs[WIRE_INT8]) <= 2e-3 * abs(outs[WIRE_BF16])


def test_delayed_parameter_updates(cuda):
    """Delayed parameter updates: with a fixed batch, step 1 runs on
    the initial weights again (its loss equals step 0's) and step 2 on the weights
    of step 0's update (its loss equals the synchronous run's step 1), while the
    all-reduce + AdamW of each step overlap the next step on a side stream."""
    import torch
    from paper_2301_11913_b200.swarm import PRESETS, SwarmPipeline, synthetic_batch
    m = PRESETS["tiny"]
    tok, _ = synthetic_batch(m, 4, seed=1, device=cuda)
    tgt = torch.roll(tok, -1, dims=1)
    runs = {}
    for dpu in (False, True):
        pipe = SwarmPipeline(m, 4, n_microbatches=4, seed=3, lr=3e-3, dpu=dpu)
        losses = []
        for _ in range(5):
            pipe.loss_sum.zero_()
            pipe.step(tok, tgt)
            pipe.drain_updates()
            losses.append(pipe.loss_sum.item() / pipe.tokens_per_step())
        runs[dpu] = losses
    sync, dpu = runs[False], runs[True]
    assert dpu[0] == pytest.approx(sync[0], rel=1e-6)
    assert dpu[1] == pytest.approx(sync[0], rel=1e-6)
    assert dpu[2] == pytest.approx(sync[1], rel=1e-6)
    assert dpu[4] < dpu[0] - 0.1, dpu  # it still trains
