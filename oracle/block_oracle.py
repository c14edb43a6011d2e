"""TEST INFRASTRUCTURE ONLY — fp64 CPU oracle of one SWARM stage's block math.

The reference has NO transformer-block implementation (it simulates the visit
as a service time, P/src/sim.cpp:361-364), so parity for the block is UNPINNED
by the reference: this oracle restates the architecture the reference's cost
model and paper fix, and the tests compare the B200 executor to it with a
stated tolerance:
  * weights per layer: Wqkv d x 3d, Wo d x d, W1 d x d_ffn, W2 d_ffn x d, no biases
    (P/src/cost_model.cpp:31-35), stored [out, in] like torch.nn.Linear;
  * pre-LN block, LayerNorm as P/src/compression.cpp:52-74 (two-pass mean,
    biased variance, eps 1e-5, gain/bias);
  * MLP(x) = sigma(x w1) w2 + x with sigma = GeLU (tanh form), PAPER:787;
  * causal multi-head attention with 1/sqrt(d_head) scaling;
  * first stage: token embedding; last stage: final LN, LM head, token
    cross-entropy summed over tokens and scaled by `loss_scale`;
  * optional maxout bottleneck at the boundaries: the sender
    emits maxout_k(LN(x)), the receiver applies LN then W_d (d/k -> d).
It runs in float64 on the CPU with torch autograd for the backward.
"""
from __future__ import annotations

import math

import torch


def layer_norm(x, g, b, eps=1e-5):
    mean = x.mean(-1, keepdim=True)
    var = ((x - mean) ** 2).mean(-1, keepdim=True)
    return (x - mean) / torch.sqrt(var + eps) * g + b


def gelu_tanh(u):
    return 0.5 * u * (1.0 + torch.tanh(math.sqrt(2.0 / math.pi) * (u + 0.044715 * u ** 3)))


def block(x, W, B, L, H, causal=True):
    """x: [B*L, d] float64; W: dict of float64 tensors (wqkv, wo, w1, w2, ln1_g, ln1_b, ln2_g, ln2_b)."""
    T, d = x.shape
    dh = d // H
    a = layer_norm(x, W["ln1_g"], W["ln1_b"])
    qkv = a @ W["wqkv"].T
    q, k, v = (t.reshape(B, L, H, dh).transpose(1, 2) for t in qkv.split(d, dim=1))
    s = (q @ k.transpose(-1, -2)) / math.sqrt(dh)
    if causal:
        mask = torch.triu(torch.ones(L, L, dtype=torch.bool), 1)
        s = s.masked_fill(mask, float("-inf"))
    p = torch.softmax(s, -1)
    o = (p @ v).transpose(1, 2).reshape(T, d)
    h = x + o @ W["wo"].T
    c = layer_norm(h, W["ln2_g"], W["ln2_b"])
    g = gelu_tanh(c @ W["w1"].T)
    return h + g @ W["w2"].T


def stage(params: dict, cfg, inp, targets=None, loss_scale=1.0):
    """One stage forward.  params: name -> float64 tensor (requires_grad as the
    caller wants).  inp: int64 tokens [T] on the first stage, else float64 [T, d].
    Returns (output [T, d], loss or None)."""
    B, L, H = cfg.micro_batch, cfg.seq_len, cfg.n_heads
    mk = getattr(cfg, "maxout_k", 0)
    if cfg.is_first:
        x = params["embedding"][inp]
    elif mk > 1:  # receiving side of the maxout bottleneck: LN then W_d
        x = layer_norm(inp, params["bneck_in_ln_g"], params["bneck_in_ln_b"]) @ params["bneck_wd"].T
    else:
        x = inp
    nw = 1 if cfg.shared_layers else cfg.n_layers
    for l in range(cfg.n_layers):
        i = 0 if nw == 1 else l
        W = {k: params[f"layer{i}.{k}"] for k in ("wqkv", "wo", "w1", "w2", "ln1_g", "ln1_b", "ln2_g", "ln2_b")}
        x = block(x, W, B, L, H, bool(cfg.causal))
    if not cfg.is_last:
        if mk > 1:  # sending side: maxout_k(LN(x)) over windows of k consecutive features
            z = layer_norm(x, params["bneck_out_ln_g"], params["bneck_out_ln_b"])
            return z.reshape(z.shape[0], -1, mk).max(-1).values, None
        return x, None
    xf = layer_norm(x, params["lnf_g"], params["lnf_b"])
    logits = xf @ params["head"].T
    loss = torch.nn.functional.cross_entropy(logits, targets, reduction="sum")
    return x, loss * loss_scale
