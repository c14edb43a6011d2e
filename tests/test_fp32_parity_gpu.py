"""BASELINE configs[0] exactly, in the fp32 arithmetic mode, against the fp64 CPU oracle.

configs[0]: "tiny 2-stage SWARM pipeline, 1 peer/stage, 4-layer d_model=256
transformer, seq 128, batch 8, fp32, 8-bit boundary compression".  The stage
executor runs it with swarm_stage_config.fp32 = 1: fp32 activations, fp32
wire tensors into the int8 codec, SIMT fp32 GEMMs (swarm_gemm_f32) reading the
fp32 master weights, unfused fp32 attention.

Parity bar (stated here):
  * per stage, given identical inputs: activations, loss, parameter gradients and
    the input gradient within REL_TOL = 1e-5 relative (Frobenius) of the fp64 oracle;
  * every wire message (forward activations and backward gradients) bit-exact:
    int8 codes and fp32 scales equal the oracle codec (a restatement of
    P/src/compression.cpp:10-29) applied to the tensor the stage encoded.
  * end to end (the oracle runs its own fp64 chain and its own codec): the int8
    codes it produces differ from the executor's in at most CODE_FLIP_FRAC of
    positions (a code flips only where 127*x/absmax sits within ~1e-6 of a
    half-integer), and the loss agrees within 1e-4 relative.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

REL_TOL = 1e-5
CODE_FLIP_FRAC = 1e-3


def rel(a, b):
    a = a.double().cpu()
    b = b.double().cpu()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def cfg0(**kw):
    """One stage of BASELINE configs[0] (2 of its 4 layers)."""
    from paper_2301_11913_b200.stage import StageConfig
    base = dict(d_model=256, n_heads=4, d_ffn=1024, seq_len=128, micro_batch=8, n_layers=2, vocab=512,
                is_first=1, is_last=1, causal=1, max_slots=1, wire=1, block_size=4096, init_std=0.02, seed=1, fp32=1)
    base.update(kw)
    return StageConfig(**base)


def oracle_params(st):
    """fp64 copies of the fp32 master weights (what the fp32-mode GEMMs read)."""
    out = {}
    for name, off, r, c in st.param_info():
        t = st.tensor(name, "param").double().cpu().reshape(r, c)
        out[name] = (t.reshape(c) if r == 1 else t).clone().requires_grad_(True)
    return out


def grad_of(st, name, r):
    g = st.tensor(name, "grad").double().cpu()
    return g.reshape(-1) if r == 1 else g


def wire_parts(st, wire):
    n = st.cfg.tokens * st.cfg.d_model // max(st.cfg.maxout_k, 1)
    off = (n + 15) // 16 * 16
    nb = (n + st.cfg.block_size - 1) // st.cfg.block_size
    import torch
    return wire[:n].view(torch.int8), wire[off:off + nb * 4].view(torch.float32)


def assert_wire_is_oracle_codec(st, wire, x):
    """codes + scales of `wire` == the oracle codec applied to the fp32 tensor x."""
    codes, scales = wire_parts(st, wire)
    rc, oc, osc = O.quantize(x.detach().float().cpu().numpy().reshape(-1), st.cfg.block_size)
    assert rc == 0
    assert np.array_equal(codes.cpu().numpy(), oc)
    assert np.array_equal(scales.cpu().numpy(), osc)


def decode(st, wire):
    import torch
    from paper_2301_11913_b200 import ops
    codes, scales = wire_parts(st, wire)
    out = ops.dequantize(codes, scales, st.cfg.block_size, torch.float32)
    # the receiver's fp32 decode is bit-exact to the oracle's RN32(code * absmax / 127)
    want = O.dequantize(codes.cpu().numpy(), scales.cpu().numpy(), st.cfg.block_size, np.float32)
    assert np.array_equal(out.cpu().numpy(), want)
    return out.view(st.cfg.tokens, -1)


@pytest.fixture(scope="module")
def threads():
    import os

    import torch
    torch.set_num_threads(os.cpu_count() or 1)


def run_pipeline(c0, c1, seed):
    import torch
    from paper_2301_11913_b200.stage import Stage
    s0, s1 = Stage(c0), Stage(c1)
    g = torch.Generator().manual_seed(seed)
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
    return s0, s1, tok, tgt, act, grad, loss, scale


@pytest.mark.parametrize("maxout_k", [0, 2])
def test_configs0_fp32_per_stage_parity(cuda, threads, maxout_k):
    """configs[0] (2 stages x 2 layers, d 256, seq 128, batch 8, fp32, int8 boundary):
    every stage within 1e-5 of the fp64 oracle given the exact bits it received,
    every wire message bit-exact.  maxout_k=2 adds configs[3]'s bottleneck."""
    from oracle import block_oracle as BO
    c0 = cfg0(is_last=0, seed=2, maxout_k=maxout_k)
    c1 = cfg0(is_first=0, seed=3, maxout_k=maxout_k)
    s0, s1, tok, tgt, act, grad, loss, scale = run_pipeline(c0, c1, seed=1)
    assert s0.wire_bytes == s1.wire_bytes
    # stage 0 forward vs the oracle; its wire is the oracle codec of what it encoded
    P0 = oracle_params(s0)
    y_ref, _ = BO.stage(P0, c0, tok)
    sent = s0.activation(0, 0, "wire_out").view(c0.tokens, -1)
    assert rel(sent, y_ref.detach()) <= REL_TOL
    assert_wire_is_oracle_codec(s0, act, sent)
    # stage 1 on the exact decoded input: loss, every parameter gradient, input gradient
    x1 = decode(s1, act).double().cpu().requires_grad_()
    P1 = oracle_params(s1)
    _, l1 = BO.stage(P1, c1, x1, tgt, loss_scale=scale)
    l1.backward()
    assert abs(loss.item() * scale - l1.item()) <= REL_TOL * abs(l1.item())
    for name, off, r, c in s1.param_info():
        e = rel(grad_of(s1, name, r), P1[name].grad)
        assert e <= REL_TOL, (name, e)
    dx1 = s1.activation(0, 0, "dx_last").view(c1.tokens, -1)
    assert rel(dx1, x1.grad) <= REL_TOL
    assert_wire_is_oracle_codec(s1, grad, dx1)
    # stage 0 backward from the exact decoded upstream gradient
    y_ref.backward(decode(s0, grad).double().cpu())
    for name, off, r, c in s0.param_info():
        e = rel(grad_of(s0, name, r), P0[name].grad)
        assert e <= REL_TOL, (name, e)


def test_configs0_fp32_end_to_end(cuda, threads):
    """The oracle runs configs[0] on its own: fp64 stages chained through its own
    fp64 codec (quantize -> dequantize, compression.cpp:10-37) for the activations
    and the gradient.  Codes agree except at near-half-step positions; the loss and
    stage-0 gradients agree to the accuracy those flips allow."""
    import torch
    from oracle import block_oracle as BO
    c0 = cfg0(is_last=0, seed=4)
    c1 = cfg0(is_first=0, seed=5)
    s0, s1, tok, tgt, act, grad, loss, scale = run_pipeline(c0, c1, seed=2)
    P0, P1 = oracle_params(s0), oracle_params(s1)
    y0, _ = BO.stage(P0, c0, tok)
    rc, codes, absmax = O.quantize(y0.detach().numpy().reshape(-1), c0.block_size)
    assert rc == 0
    gpu_codes, _ = wire_parts(s0, act)
    flips = int((gpu_codes.cpu().numpy() != codes).sum())
    assert flips <= CODE_FLIP_FRAC * codes.size, flips
    x1 = torch.from_numpy(O.dequantize(codes, absmax, c0.block_size, np.float64)).view(c1.tokens, -1)
    x1.requires_grad_()
    _, l1 = BO.stage(P1, c1, x1, tgt, loss_scale=scale)
    l1.backward()
    assert abs(loss.item() * scale - l1.item()) <= 1e-4 * abs(l1.item())
    rc, gcodes, gabs = O.quantize(x1.grad.numpy().reshape(-1), c1.block_size)
    gpu_gcodes, _ = wire_parts(s1, grad)
    gflips = int((gpu_gcodes.cpu().numpy() != gcodes).sum())
    assert gflips <= CODE_FLIP_FRAC * gcodes.size, gflips
    y0.backward(torch.from_numpy(O.dequantize(gcodes, gabs, c1.block_size, np.float64)).view(c0.tokens, -1))
    for name, off, r, c in s0.param_info():
        e = rel(grad_of(s0, name, r), P0[name].grad)
        assert e <= 1e-3, (name, e)


def test_fp32_training_step_matches_oracle_adamw(cuda, threads):
    """One AdamW step on configs[0]'s first stage (fp32 master, fp32 GEMMs): the
    updated parameters equal an fp64 AdamW applied to the oracle's gradients."""
    import torch
    from oracle import block_oracle as BO
    from paper_2301_11913_b200.stage import Stage
    c = cfg0(is_last=1, lr=1e-3, weight_decay=0.01, seed=7)
    st = Stage(c)
    g = torch.Generator().manual_seed(3)
    tok = torch.randint(0, c.vocab, (c.tokens,), generator=g)
    tgt = torch.randint(0, c.vocab, (c.tokens,), generator=g)
    P = oracle_params(st)
    p_before = st.params().double().cpu().clone()
    loss = torch.zeros(1, device="cuda")
    st.forward(0, tok.int().cuda(), targets=tgt.int().cuda(), loss_sum=loss, loss_scale=1.0 / c.tokens)
    st.backward(0)
    st.optimizer_step()
    torch.cuda.synchronize()
    _, l = BO.stage(P, c, tok, tgt, loss_scale=1.0 / c.tokens)
    l.backward()
    p_after = st.params().double().cpu()
    for name, off, r, cc in st.param_info():
        gr = P[name].grad.reshape(-1)
        p0 = p_before[off:off + r * cc]
        m = (1 - c.beta1) * gr
        v = (1 - c.beta2) * gr * gr
        upd = (m / (1 - c.beta1)) / (torch.sqrt(v / (1 - c.beta2)) + c.eps) + c.weight_decay * p0
        want = p0 - c.lr * upd
        got = p_after[off:off + r * cc]
        # Adam normalises each gradient element, so an update equals lr*sign(g) up to the
        # gradient's relative error: compare the step taken, element-wise, where |g| is not tiny
        big = gr.abs() > 1e-3 * gr.abs().max()
        d_got, d_want = (got - p0)[big], (want - p0)[big]
        assert rel(d_got, d_want) <= 1e-4, name


@pytest.mark.parametrize("case", ["plain", "mn", "batched", "twoseg", "gelu", "dgelu", "residual", "accum"])
def test_gemm_f32_matches_fp64(cuda, case):
    """swarm_gemm_f32 against a torch fp64 contraction for each layout / epilogue."""
    import ctypes as C

    import torch
    from paper_2301_11913_b200 import _lib
    L = _lib.lib()
    torch.manual_seed(0)
    M, N, K = 200, 136, 72
    a = torch.randn(M, K, device="cuda")
    b = torch.randn(N, K, device="cuda")
    g = _lib.GemmArgs()
    g.m, g.n, g.k, g.batch, g.bh = M, N, K, 1, 1
    g.alpha = 1.0
    A, B = a, b
    if case == "mn":
        A, B = a.t().contiguous(), b.t().contiguous()
        g.a_mn_major = g.b_mn_major = 1
    g.a, g.lda, g.b, g.ldb = A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1]
    want = a.double() @ b.double().t()
    d = torch.zeros(M, N, device="cuda")
    g.d, g.ldd = d.data_ptr(), N
    g.epilogue = _lib.EPI_STORE_F32
    aux = torch.randn(M, N, device="cuda")
    if case == "batched":  # 3 x 2 batch of row / column offsets
        nb, nh = 3, 2
        a = torch.randn(nb * M, nh * K, device="cuda")
        b = torch.randn(nb * N, nh * K, device="cuda")
        d = torch.zeros(nb * M, nh * N, device="cuda")
        g.batch, g.bh = nb * nh, nh
        g.a, g.lda, g.ra0, g.ca1 = a.data_ptr(), nh * K, M, K
        g.b, g.ldb, g.rb0, g.cb1 = b.data_ptr(), nh * K, N, K
        g.d, g.ldd, g.rd0, g.cd1 = d.data_ptr(), nh * N, M, N
        want = torch.zeros_like(d, dtype=torch.float64)
        for i in range(nb):
            for h in range(nh):
                want[i * M:(i + 1) * M, h * N:(h + 1) * N] = (a[i * M:(i + 1) * M, h * K:(h + 1) * K].double() @
                                                               b[i * N:(i + 1) * N, h * K:(h + 1) * K].double().t())
    if case == "twoseg":
        a2, b2 = torch.randn(M, K, device="cuda"), torch.randn(N, K, device="cuda")
        g.k, g.a2, g.b2 = 2 * K, a2.data_ptr(), b2.data_ptr()
        want = want + a2.double() @ b2.double().t()
    if case == "gelu":
        g.epilogue, g.aux = _lib.EPI_GELU, aux.data_ptr()
        u = want
        want = 0.5 * u * (1 + torch.tanh((2 / torch.pi) ** 0.5 * (u + 0.044715 * u ** 3)))
    if case == "dgelu":
        g.epilogue, g.aux = _lib.EPI_DGELU, aux.data_ptr()
        x = aux.double()
        t = torch.tanh((2 / torch.pi) ** 0.5 * (x + 0.044715 * x ** 3))
        want = want * (0.5 * (1 + t) + 0.5 * x * (1 - t * t) * (2 / torch.pi) ** 0.5 * (1 + 3 * 0.044715 * x * x))
    if case == "residual":
        g.epilogue, g.aux = _lib.EPI_RESIDUAL, aux.data_ptr()
        want = want + aux.double()
    if case == "accum":
        d.copy_(aux)
        g.epilogue = _lib.EPI_ACCUM_F32
        want = want + aux.double()
    _lib.check(L.swarm_gemm_f32(C.byref(g), None), "gemm_f32")
    torch.cuda.synchronize()
    assert rel(d, want) <= 1e-6
    if case == "gelu":
        assert rel(aux, u) <= 1e-6
