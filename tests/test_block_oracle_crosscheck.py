"""CPU: the fp64 block oracle (oracle/block_oracle.py) against independent
implementations of the same block.

The reference has no transformer block, so the oracle is a
restatement; these checks pin it to code that was not written here:
  * torch.nn.TransformerEncoderLayer(norm_first=True, bias=False) — the layer the
    paper's authors used — with a causal mask and the tanh GeLU;
  * torch.nn.functional (layer_norm, scaled_dot_product_attention, gelu(tanh)),
    which also covers nonzero LayerNorm biases;
  * the oracle's LayerNorm against the plain-C restatement of
    P/src/compression.cpp:52-74 (oracle/codec_oracle.c).
Forward outputs and input/parameter gradients agree to fp64 rounding (1e-10).
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import block_oracle as BO

TOL = 1e-10


def rel(a, b):
    return float((a - b).detach().norm() / b.detach().norm().clamp_min(1e-300))


def weights(d, f, seed, ln_bias=True):
    g = torch.Generator().manual_seed(seed)
    W = {"wqkv": torch.randn(3 * d, d, generator=g, dtype=torch.float64) * 0.05,
         "wo": torch.randn(d, d, generator=g, dtype=torch.float64) * 0.05,
         "w1": torch.randn(f, d, generator=g, dtype=torch.float64) * 0.05,
         "w2": torch.randn(d, f, generator=g, dtype=torch.float64) * 0.05,
         "ln1_g": 1 + 0.1 * torch.randn(d, generator=g, dtype=torch.float64),
         "ln2_g": 1 + 0.1 * torch.randn(d, generator=g, dtype=torch.float64)}
    for k in ("ln1_b", "ln2_b"):
        W[k] = 0.1 * torch.randn(d, generator=g, dtype=torch.float64) if ln_bias else torch.zeros(d, dtype=torch.float64)
    return {k: v.requires_grad_(True) for k, v in W.items()}


def functional_block(x, W, B, L, H):
    T, d = x.shape
    a = F.layer_norm(x, (d,), W["ln1_g"], W["ln1_b"], eps=1e-5)
    q, k, v = (t.reshape(B, L, H, d // H).transpose(1, 2) for t in F.linear(a, W["wqkv"]).split(d, dim=1))
    o = F.scaled_dot_product_attention(q, k, v, is_causal=True).transpose(1, 2).reshape(T, d)
    h = x + F.linear(o, W["wo"])
    c = F.layer_norm(h, (d,), W["ln2_g"], W["ln2_b"], eps=1e-5)
    return h + F.linear(F.gelu(F.linear(c, W["w1"]), approximate="tanh"), W["w2"])


@pytest.mark.parametrize("B,L,H,d", [(2, 16, 4, 32), (1, 64, 2, 64)])
def test_oracle_block_matches_functional(B, L, H, d):
    W = weights(d, 4 * d, seed=d)
    W2 = {k: v.detach().clone().requires_grad_(True) for k, v in W.items()}
    g = torch.Generator().manual_seed(1)
    x = torch.randn(B * L, d, generator=g, dtype=torch.float64, requires_grad=True)
    x2 = x.detach().clone().requires_grad_(True)
    dy = torch.randn(B * L, d, generator=g, dtype=torch.float64)
    y = BO.block(x, W, B, L, H, causal=True)
    y2 = functional_block(x2, W2, B, L, H)
    assert rel(y, y2) <= TOL
    y.backward(dy)
    y2.backward(dy)
    assert rel(x.grad, x2.grad) <= TOL
    for k in W:
        assert rel(W[k].grad, W2[k].grad) <= TOL, k


def test_oracle_block_matches_transformer_encoder_layer():
    """The paper's layer, bias-free (cost_model.cpp:31-35 counts no biases)."""
    B, L, H, d = 2, 32, 4, 64
    W = weights(d, 4 * d, seed=9, ln_bias=False)
    layer = torch.nn.TransformerEncoderLayer(d, H, dim_feedforward=4 * d, dropout=0.0,
                                             activation=lambda u: F.gelu(u, approximate="tanh"),
                                             batch_first=True, norm_first=True, bias=False, dtype=torch.float64)
    with torch.no_grad():
        layer.self_attn.in_proj_weight.copy_(W["wqkv"])
        layer.self_attn.out_proj.weight.copy_(W["wo"])
        layer.linear1.weight.copy_(W["w1"])
        layer.linear2.weight.copy_(W["w2"])
        layer.norm1.weight.copy_(W["ln1_g"])
        layer.norm2.weight.copy_(W["ln2_g"])
    layer.train()  # the slow (non-fused) path, autograd through every op
    g = torch.Generator().manual_seed(2)
    x = torch.randn(B * L, d, generator=g, dtype=torch.float64, requires_grad=True)
    x2 = x.detach().clone().reshape(B, L, d).requires_grad_(True)
    mask = torch.nn.Transformer.generate_square_subsequent_mask(L, dtype=torch.float64)
    y = BO.block(x, W, B, L, H, causal=True)
    y2 = layer(x2, src_mask=mask, is_causal=True).reshape(B * L, d)
    assert rel(y, y2) <= TOL
    dy = torch.randn(B * L, d, generator=g, dtype=torch.float64)
    y.backward(dy)
    y2.backward(dy)
    assert rel(x.grad, x2.grad.reshape(B * L, d)) <= TOL
    assert rel(W["wqkv"].grad, layer.self_attn.in_proj_weight.grad) <= TOL
    assert rel(W["w1"].grad, layer.linear1.weight.grad) <= TOL
    assert rel(W["ln2_g"].grad, layer.norm2.weight.grad) <= TOL


def test_oracle_layer_norm_matches_c_restatement():
    import oracle as O
    g = np.random.default_rng(4)
    for cols in (7, 256, 2048):
        x = g.standard_normal(cols) * 3 + 1
        gain, bias = g.standard_normal(cols), g.standard_normal(cols)
        rc, want = O.layer_norm(x, gain, bias)
        assert rc == 0
        got = BO.layer_norm(torch.from_numpy(x), torch.from_numpy(gain), torch.from_numpy(bias)).numpy()
        assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))


def test_oracle_stage_maxout_bottleneck_composition():
    """The bottleneck composition: sender maxout_k(LN(x)) equals the
    C codec oracle's maxout over LN rows; receiver LN then W_d equals a direct product."""
    import oracle as O
    from types import SimpleNamespace
    d, k, T = 64, 2, 8
    g = torch.Generator().manual_seed(3)
    z = torch.randn(T, d, generator=g, dtype=torch.float64)
    gain, bias = torch.ones(d, dtype=torch.float64), torch.zeros(d, dtype=torch.float64)
    ln = BO.layer_norm(z, gain, bias)
    sent = ln.reshape(T, -1, k).max(-1).values
    for t in range(T):
        rc, mo, _ = O.maxout(ln[t].numpy(), k)
        assert rc == 0 and np.array_equal(mo, sent[t].numpy())
    cfg = SimpleNamespace(micro_batch=1, seq_len=T, n_heads=4, maxout_k=k, is_first=0, is_last=0, n_layers=0,
                          shared_layers=0, causal=1)
    wd = torch.randn(d, d // k, generator=g, dtype=torch.float64)
    P = {"bneck_in_ln_g": torch.ones(d // k, dtype=torch.float64), "bneck_in_ln_b": torch.zeros(d // k, dtype=torch.float64),
         "bneck_wd": wd, "bneck_out_ln_g": gain, "bneck_out_ln_b": bias}
    out, _ = BO.stage(P, cfg, sent)
    want = BO.layer_norm(BO.layer_norm(sent, P["bneck_in_ln_g"], P["bneck_in_ln_b"]) @ wd.T, gain, bias)
    assert rel(out, want.reshape(T, -1, k).max(-1).values) <= 1e-14
    assert math.isfinite(float(out.sum()))
