"""Per-shape timing of every GEMM one transformer block (+ LM head) of a config
issues, on the tcgen05 kernel: achieved TFLOP/s per shape and the FLOP-weighted
total.  CUDA events, 3 warm-up + 10 timed launches per shape, inputs resident.

  python scripts/gemm_shapes.py [--model C]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2301_11913_b200 import _lib as L, ops  # noqa: E402
from paper_2301_11913_b200.swarm import PRESETS  # noqa: E402


def batched(M, N, K, batch, a_t, b_t, epi):
    a = torch.randn(batch * (K if a_t else M), (M if a_t else K), device="cuda").bfloat16()
    b = torch.randn(batch * (K if b_t else N), (N if b_t else K), device="cuda").bfloat16()
    out = torch.empty(batch * M, N, device="cuda", dtype=torch.float32 if epi in (1, 2) else torch.bfloat16)
    g = L.GemmArgs()
    g.m, g.n, g.k, g.batch, g.bh = M, N, K, batch, 1
    g.a, g.lda, g.a_mn_major, g.a_rows, g.a_cols = a.data_ptr(), a.shape[1], int(a_t), a.shape[0], a.shape[1]
    g.ra0 = K if a_t else M
    g.b, g.ldb, g.b_mn_major, g.b_rows, g.b_cols = b.data_ptr(), b.shape[1], int(b_t), b.shape[0], b.shape[1]
    g.rb0 = K if b_t else N
    g.d, g.ldd, g.rd0 = out.data_ptr(), N, M
    g.alpha, g.epilogue = 1.0, epi
    g.aux = None
    ws = ops.gemm_workspace()  # as the stage executor does: the kernel's policy decides on stream-K
    g.workspace, g.workspace_bytes = ws.data_ptr(), ws.numel()
    return (a, b, out), lambda: ops.gemm_raw(g)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="C")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    m = PRESETS[args.model]
    T, d, F, L_, H, V = m.tokens, m.d_model, m.d_ffn, m.seq_len, m.n_heads, m.vocab
    dh, BH = d // H, m.micro_batch * H
    E_BF, E_F32, E_ACC = 0, 1, 2
    shapes = [  # name, M, N, K, batch, a_t, b_t, epilogue, launches per layer
        ("fwd.qkv", T, 3 * d, d, 1, 0, 0, E_BF), ("fwd.o", T, d, d, 1, 0, 0, E_BF),
        ("fwd.ffn1", T, F, d, 1, 0, 0, E_BF), ("fwd.ffn2", T, d, F, 1, 0, 0, E_BF),
        ("attn.S", L_, L_, dh, BH, 0, 0, E_F32), ("attn.PV", L_, dh, L_, BH, 0, 1, E_BF),
        ("bwd.ffn2.dgrad", T, F, d, 1, 0, 1, E_BF), ("bwd.ffn2.wgrad", d, F, T, 1, 1, 1, E_ACC),
        ("bwd.ffn1.dgrad", T, d, F, 1, 0, 1, E_BF), ("bwd.ffn1.wgrad", F, d, T, 1, 1, 1, E_ACC),
        ("bwd.o.dgrad", T, d, d, 1, 0, 1, E_BF), ("bwd.o.wgrad", d, d, T, 1, 1, 1, E_ACC),
        ("attn.dP", L_, L_, dh, BH, 0, 0, E_F32), ("attn.dQ", L_, dh, L_, BH, 0, 1, E_BF),
        ("attn.dK", L_, dh, L_, BH, 1, 1, E_BF), ("attn.dV", L_, dh, L_, BH, 1, 1, E_BF),
        ("bwd.qkv.dgrad", T, d, 3 * d, 1, 0, 1, E_BF), ("bwd.qkv.wgrad", 3 * d, d, T, 1, 1, 1, E_ACC),
        ("head.logits", T, V, d, 1, 0, 0, E_F32), ("head.wgrad", V, d, T, 1, 1, 1, E_ACC),
        ("head.dgrad", T, d, V, 1, 0, 1, E_BF),
    ]
    rows, tot_ms, tot_fl = [], 0.0, 0.0
    for name, M, N, K, batch, a_t, b_t, epi in shapes:
        keep, fn = batched(M, N, K, batch, a_t, b_t, epi)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        fl = 2.0 * M * N * K * batch
        tf = fl / ms / 1e9
        # library reference point (measurement only): cuBLAS via torch on the same
        # operand layouts, bf16 out (fp32 out for the fp32 epilogues)
        a_, b_ = keep[0], keep[1]
        if batch == 1:
            A = a_.t() if a_t else a_
            B = b_ if b_t else b_.t()
            lib = (lambda: torch.matmul(A, B)) if epi == E_BF else (lambda: torch.matmul(A, B).float())
            for _ in range(3):
                lib()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(10):
                lib()
            e1.record()
            torch.cuda.synchronize()
            lib_tf = fl / (e0.elapsed_time(e1) / 10) / 1e9
        else:
            lib_tf = None
        rows.append({"gemm": name, "M": M, "N": N, "K": K, "batch": batch, "a_mn": a_t, "b_mn": b_t, "ms": ms,
                     "tflops": tf, "cublas_tflops": lib_tf})
        if not name.startswith("head"):
            tot_ms += ms
            tot_fl += fl
        print(f"{name:16s} M={M:6d} N={N:6d} K={K:6d} x{batch:3d}  {ms * 1e3:9.1f} us  {tf:7.1f} TFLOP/s"
              f"  (cuBLAS {lib_tf or 0:7.1f})", flush=True)
    print(f"block total: {tot_ms:.3f} ms/layer/microbatch, {tot_fl / tot_ms / 1e9:.1f} TFLOP/s FLOP-weighted")
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"model": args.model, "rows": rows, "block_ms": tot_ms,
                       "block_tflops": tot_fl / tot_ms / 1e9}, f, indent=1)


if __name__ == "__main__":
    main()
