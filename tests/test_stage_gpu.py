"""GPU parity of the stage executor (block forward/backward, embedding, LM head,
cross-entropy, boundary codec) against the fp64 CPU block oracle.

Parity for the block math is UNPINNED by the reference (it has no block
implementation); the oracle restates the architecture (oracle/block_oracle.py).
The executor computes in bf16 storage with fp32 accumulation, so tolerances are
stated as relative Frobenius-norm errors:
  forward activations / stage outputs   <= 2e-2
  loss                                   <= 2e-3 relative
  parameter gradients and input grads    <= 5e-2
The int8 wire is checked bit-exactly against the oracle codec applied to the
executor's own bf16 boundary tensor.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

FWD_TOL, LOSS_TOL, GRAD_TOL = 2e-2, 2e-3, 5e-2
# Through the maxout bottleneck a bf16 rounding difference can flip which element
# of a near-tied window wins, re-routing that window's gradient; upstream of the
# bottleneck the gradient tolerance is therefore 1e-1 (downstream stays 5e-2).
GRAD_TOL_MAXOUT_UPSTREAM = 1e-1


def rel(a, b):
    a = a.double().cpu()
    b = b.double().cpu()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def tiny_cfg(**kw):
    from paper_2301_11913_b200.stage import StageConfig
    base = dict(d_model=256, n_heads=4, d_ffn=1024, seq_len=128, micro_batch=4, n_layers=2, vocab=512,
                is_first=1, is_last=1, causal=1, max_slots=2, wire=1, block_size=4096, init_std=0.05, seed=1)
    base.update(kw)
    return StageConfig(**base)


def oracle_params(st, requires_grad=True):
    """fp64 copies of the executor's weights as the GEMMs see them (bf16 shadow
    for matrices, fp32 master for LayerNorm params)."""
    out = {}
    for name, off, r, c in st.param_info():
        src = st.tensor(name, "param") if r == 1 else st.tensor(name, "bf16")
        t = src.double().cpu().reshape(r, c)
        if r == 1:
            t = t.reshape(c)
        out[name] = t.clone().requires_grad_(requires_grad)
    return out


def grad_of(st, name, r):
    g = st.tensor(name, "grad").double().cpu()
    return g.reshape(-1) if r == 1 else g


def decode_wire(st, wire):
    """Dequantize a wire message (int8 codes | fp32 scales) exactly like the receiver (bf16)."""
    import torch
    from paper_2301_11913_b200 import ops
    n = st.cfg.tokens * st.cfg.d_model
    off = (n + 15) // 16 * 16
    codes = wire[:n].view(torch.int8)
    scales = wire[off:off + (n + st.cfg.block_size - 1) // st.cfg.block_size * 4].view(torch.float32)
    return ops.dequantize(codes, scales, st.cfg.block_size, torch.bfloat16).view(st.cfg.tokens, st.cfg.d_model)


@pytest.mark.parametrize("shared", [0, 1])
def test_single_stage_matches_oracle(cuda, shared):
    import torch
    from oracle import block_oracle as BO
    from paper_2301_11913_b200.stage import Stage
    cfg = tiny_cfg(shared_layers=shared)
    st = Stage(cfg)
    g = torch.Generator().manual_seed(0)
    tok = torch.randint(0, cfg.vocab, (cfg.tokens,), generator=g)
    tgt = torch.randint(0, cfg.vocab, (cfg.tokens,), generator=g)
    loss = torch.zeros(1, device="cuda")
    scale = 1.0 / cfg.tokens
    st.forward(0, tok.int().cuda(), targets=tgt.int().cuda(), loss_sum=loss, loss_scale=scale)
    st.backward(0)
    torch.cuda.synchronize()
    P = oracle_params(st)
    out, ref_loss = BO.stage(P, cfg, tok, tgt, loss_scale=scale)
    ref_loss.backward()
    assert abs(loss.item() * scale - ref_loss.item()) <= LOSS_TOL * abs(ref_loss.item())
    assert rel(st.activation(0, 0, "out").view(cfg.tokens, -1), out.detach()) <= FWD_TOL
    for name, off, r, c in st.param_info():
        e = rel(grad_of(st, name, r), P[name].grad)
        assert e <= GRAD_TOL, (name, e)


def test_two_stage_int8_boundary(cuda):
    """Stage 0 -> int8 wire -> stage 1 (last), and the gradient wire back.
    Each stage is checked against the oracle fed the exact bits it received."""
    import torch
    from oracle import block_oracle as BO
    from paper_2301_11913_b200.stage import Stage
    c0 = tiny_cfg(is_last=0, seed=2)
    c1 = tiny_cfg(is_first=0, seed=3)
    s0, s1 = Stage(c0), Stage(c1)
    g = torch.Generator().manual_seed(1)
    tok = torch.randint(0, c0.vocab, (c0.tokens,), generator=g)
    tgt = torch.randint(0, c0.vocab, (c0.tokens,), generator=g)
    act, grad = s0.new_wire(), s1.new_wire()
    loss = torch.zeros(1, device="cuda")
    scale = 1.0 / c0.tokens
    s0.forward(0, tok.int().cuda(), out=act)
    s1.forward(0, act, targets=tgt.int().cuda(), loss_sum=loss, loss_scale=scale)
    s1.backward(0, grad_out=grad)
    s0.backward(0, grad_in=grad)
    torch.cuda.synchronize()
    n = c0.tokens * c0.d_model
    # wire bits == oracle codec applied to the sender's bf16 boundary tensor
    y0 = s0.activation(0, 0, "out")
    st, codes, scales = O.quantize(y0.view(torch.int16).cpu().numpy().view(np.uint16), c0.block_size)
    assert np.array_equal(act[:n].cpu().numpy().view(np.int8), codes)
    off = (n + 15) // 16 * 16
    assert np.array_equal(act[off:off + scales.size * 4].view(torch.float32).cpu().numpy(), scales)
    # the message ends with a self-describing header
    import ctypes as C
    from paper_2301_11913_b200 import _lib
    hdr = act[-16:].cpu().numpy().copy()
    ne, bsz, kind, mk = C.c_uint32(), C.c_uint32(), C.c_int(), C.c_int()
    assert _lib.lib().swarm_wire_parse_header(hdr.ctypes.data_as(C.c_void_p), C.byref(ne), C.byref(bsz), C.byref(kind),
                                              C.byref(mk)) == 0
    assert (ne.value, bsz.value, kind.value, mk.value) == (n, c0.block_size, 1, 1)
    # stage 1 vs oracle on the exact dequantized input
    x1 = decode_wire(s1, act).double().cpu().requires_grad_()
    P1 = oracle_params(s1)
    _, l1 = BO.stage(P1, c1, x1, tgt, loss_scale=scale)
    l1.backward()
    assert abs(loss.item() * scale - l1.item()) <= LOSS_TOL * abs(l1.item())
    for name, off, r, c in s1.param_info():
        assert rel(grad_of(s1, name, r), P1[name].grad) <= GRAD_TOL, name
    assert rel(decode_wire(s0, grad), x1.grad) <= GRAD_TOL
    # stage 0 vs oracle with the exact dequantized upstream gradient
    P0 = oracle_params(s0)
    y_ref, _ = BO.stage(P0, c0, tok)
    assert rel(y0.view(c0.tokens, -1), y_ref.detach()) <= FWD_TOL
    y_ref.backward(decode_wire(s0, grad).double().cpu())
    for name, off, r, c in s0.param_info():
        assert rel(grad_of(s0, name, r), P0[name].grad) <= GRAD_TOL, name


def test_optimizer_step_is_adamw(cuda):
    import torch
    from paper_2301_11913_b200.stage import Stage
    cfg = tiny_cfg(lr=1e-3, weight_decay=0.1)
    st = Stage(cfg)
    p0 = st.params().clone()
    gr = torch.randn_like(p0) * 1e-2
    st.grads().copy_(gr)
    st.optimizer_step(grad_scale=0.5)
    torch.cuda.synchronize()
    g = gr * 0.5
    m = 0.1 * g
    v = 0.05 * g * g
    want = p0 - 1e-3 * ((m / 0.1) / (torch.sqrt(v / 0.05) + cfg.eps) + 0.1 * p0)
    torch.testing.assert_close(st.params(), want, rtol=1e-5, atol=1e-6)
    assert float(st.grads().abs().max()) == 0.0
    # the bf16 shadow is exactly the round-to-nearest of the updated fp32 master
    assert torch.equal(st.params_bf16(), st.params().bfloat16())


def test_training_reduces_loss(cuda):
    """A few AdamW steps on a fixed batch must drive the loss down (end-to-end sanity)."""
    import torch
    from paper_2301_11913_b200.stage import Stage
    cfg = tiny_cfg(lr=3e-3, max_slots=1)
    st = Stage(cfg)
    g = torch.Generator().manual_seed(5)
    tok = torch.randint(0, cfg.vocab, (cfg.tokens,), generator=g).int().cuda()
    tgt = torch.roll(tok, -1)
    losses = []
    for _ in range(8):
        loss = torch.zeros(1, device="cuda")
        st.forward(0, tok, targets=tgt, loss_sum=loss, loss_scale=1.0 / cfg.tokens)
        st.backward(0)
        st.optimizer_step()
        losses.append(loss.item() / cfg.tokens)
    assert losses[-1] < losses[0] - 0.5, losses


def test_two_stage_maxout_bottleneck(cuda):
    """configs[3]'s boundary: sender maxout_2(LN(y)) -> int8 wire -> receiver LN then W_d.
    Both stages vs the oracle fed the exact bits crossing the boundary."""
    import torch
    from oracle import block_oracle as BO
    from paper_2301_11913_b200.stage import Stage
    c0 = tiny_cfg(is_last=0, seed=4, maxout_k=2)
    c1 = tiny_cfg(is_first=0, seed=5, maxout_k=2)
    s0, s1 = Stage(c0), Stage(c1)
    w = c0.d_model // 2
    assert s0.wire_bytes == (c0.tokens * w + 15) // 16 * 16 + (c0.tokens * w // c0.block_size * 4 + 15) // 16 * 16 + 16
    g = torch.Generator().manual_seed(8)
    tok = torch.randint(0, c0.vocab, (c0.tokens,), generator=g)
    tgt = torch.randint(0, c0.vocab, (c0.tokens,), generator=g)
    act, grad = s0.new_wire(), s1.new_wire()
    loss = torch.zeros(1, device="cuda")
    scale = 1.0 / c0.tokens
    s0.forward(0, tok.int().cuda(), out=act)
    s1.forward(0, act, targets=tgt.int().cuda(), loss_sum=loss, loss_scale=scale)
    s1.backward(0, grad_out=grad)
    s0.backward(0, grad_in=grad)
    torch.cuda.synchronize()

    def dec(st, wire):
        from paper_2301_11913_b200 import ops
        n = st.cfg.tokens * w
        off = (n + 15) // 16 * 16
        return ops.dequantize(wire[:n].view(torch.int8), wire[off:off + n // st.cfg.block_size * 4].view(torch.float32),
                              st.cfg.block_size, torch.bfloat16).view(st.cfg.tokens, w)

    x1 = dec(s1, act).double().cpu().requires_grad_()
    P1 = oracle_params(s1)
    _, l1 = BO.stage(P1, c1, x1, tgt, loss_scale=scale)
    l1.backward()
    assert abs(loss.item() * scale - l1.item()) <= LOSS_TOL * abs(l1.item())
    for name, off, r, c in s1.param_info():
        assert rel(grad_of(s1, name, r), P1[name].grad) <= GRAD_TOL, name
    assert rel(dec(s0, grad), x1.grad) <= GRAD_TOL
    P0 = oracle_params(s0)
    m_ref, _ = BO.stage(P0, c0, tok)
    assert rel(dec(s0, act), m_ref.detach()) <= FWD_TOL
    m_ref.backward(dec(s0, grad).double().cpu())
    for name, off, r, c in s0.param_info():
        assert rel(grad_of(s0, name, r), P0[name].grad) <= GRAD_TOL_MAXOUT_UPSTREAM, name


@pytest.mark.parametrize("shape", [dict(), dict(d_model=512, n_heads=4, d_ffn=2048, seq_len=256, micro_batch=2),
                                   dict(shared_layers=1), dict(shared_layers=1, n_layers=4)])
def test_paired_weight_gradients_match_per_microbatch(cuda, shape):
    """Deferring a visit's weight gradients and issuing them paired with the next
    visit's (two-segment K GEMMs), or alone via flush_wgrad, accumulates the same
    gradients as per-visit weight gradients (fp32 summation order only).  Layer-
    shared stages take the stacked path (one K = n_layers * T GEMM per shared weight)."""
    import torch
    from paper_2301_11913_b200.stage import Stage
    g = torch.Generator().manual_seed(11)
    cfgs = [tiny_cfg(**shape) for _ in range(3)]
    tok = [torch.randint(0, cfgs[0].vocab, (cfgs[0].tokens,), generator=g).int().cuda() for _ in range(2)]
    grads = []
    for variant in ("now", "pair", "flush"):
        st = Stage(tiny_cfg(**shape))
        if variant != "now":
            st.enable_wgrad_pairing()
        loss = torch.zeros(1, device="cuda")
        for slot in (0, 1):
            st.forward(slot, tok[slot], targets=torch.roll(tok[slot], -1), loss_sum=loss, loss_scale=1e-3)
        if variant == "now":
            st.backward(1)
            st.backward(0)
        elif variant == "pair":
            st.backward_ex(1, mode=Stage.WGRAD_DEFER, set=0)
            st.backward_ex(0, mode=Stage.WGRAD_PAIR, set=1, prev_slot=1, prev_set=0)
        else:
            st.backward_ex(1, mode=Stage.WGRAD_DEFER, set=0)
            st.flush_wgrad(1, 0)
            st.backward_ex(0, mode=Stage.WGRAD_DEFER, set=1)
            st.flush_wgrad(0, 1)
        torch.cuda.synchronize()
        grads.append(st.grads().clone())
    scale = float(grads[0].abs().max())
    for other in grads[1:]:
        torch.testing.assert_close(other, grads[0], rtol=1e-4, atol=1e-5 * scale)


def _wire_from(st, x):
    """A wire message carrying the int8 codec of x (the stage's wire width), as a sender builds it."""
    import torch
    from paper_2301_11913_b200 import ops
    n = x.numel()
    off = (n + 15) // 16 * 16
    nb = (n + st.cfg.block_size - 1) // st.cfg.block_size
    msg = st.new_wire()
    ops.quantize(x.reshape(-1), st.cfg.block_size, codes=msg[:n].view(torch.int8),
                 scales=msg[off:off + nb * 4].view(torch.float32))
    return msg


def _decode_any(st, wire, width):
    import torch
    from paper_2301_11913_b200 import ops
    n = st.cfg.tokens * width
    off = (n + 15) // 16 * 16
    nb = (n + st.cfg.block_size - 1) // st.cfg.block_size
    return ops.dequantize(wire[:n].view(torch.int8), wire[off:off + nb * 4].view(torch.float32), st.cfg.block_size,
                          torch.bfloat16).view(st.cfg.tokens, width)


@pytest.mark.parametrize("shape", ["configs2", "configs3"])
def test_one_block_at_baseline_shape(cuda, shape):
    """One middle-stage visit (int8 wire in, int8 wire out, backward with an int8
    gradient wire) at the BASELINE shapes, against the fp64 oracle fed the exact
    bits the stage received, at the bf16 tolerances stated at the top of this file.
      configs2: d 2048, 16 heads, d_ffn 8192, seq 512, microbatch 4, one block;
      configs3: d 4096, 32 heads, d_ffn 16384, seq 512, microbatch 1, two applications
                of one shared block, maxout k=2 bottleneck on both boundaries."""
    import os

    import torch
    from oracle import block_oracle as BO
    from paper_2301_11913_b200.stage import Stage
    torch.set_num_threads(os.cpu_count() or 1)
    if shape == "configs2":
        cfg = tiny_cfg(d_model=2048, n_heads=16, d_ffn=8192, seq_len=512, micro_batch=4, n_layers=1, is_first=0,
                       is_last=0, max_slots=1, init_std=0.02, seed=21)
    else:
        cfg = tiny_cfg(d_model=4096, n_heads=32, d_ffn=16384, seq_len=512, micro_batch=1, n_layers=2,
                       shared_layers=1, maxout_k=2, is_first=0, is_last=0, max_slots=1, init_std=0.02, seed=22)
    st = Stage(cfg)
    width = cfg.d_model // max(cfg.maxout_k, 1)
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(cfg.tokens, width, device="cuda", generator=g)
    dy = torch.randn(cfg.tokens, width, device="cuda", generator=g) * 1e-3
    win, gin = _wire_from(st, x), _wire_from(st, dy)
    wout, gout = st.new_wire(), st.new_wire()
    st.forward(0, win, out=wout)
    st.backward(0, grad_in=gin, grad_out=gout)
    torch.cuda.synchronize()
    x_in = _decode_any(st, win, width).double().cpu().requires_grad_()
    P = oracle_params(st)
    y_ref, _ = BO.stage(P, cfg, x_in)
    assert rel(st.activation(0, 0, "wire_out").view(cfg.tokens, -1), y_ref.detach()) <= FWD_TOL
    y_ref.backward(_decode_any(st, gin, width).double().cpu())
    # the bottleneck's maxout re-routes a near-tied window's gradient on a bf16 rounding
    # difference; everything upstream of it gets the wider tolerance (see the top of this file)
    tol = GRAD_TOL_MAXOUT_UPSTREAM if cfg.maxout_k > 1 else GRAD_TOL
    for name, off, r, c in st.param_info():
        e = rel(grad_of(st, name, r), P[name].grad)
        assert e <= tol, (name, e)
    assert rel(st.activation(0, 0, "dx_last").view(cfg.tokens, -1), x_in.grad) <= tol
