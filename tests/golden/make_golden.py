"""Generate tests/golden/codec_golden.json from the UNMODIFIED reference.

Runs in the build container only (needs oracle/_ref/libswarmsim_ref.so, which
oracle/Makefile compiles from /root/reference/proj/src/compression.cpp in place).
Every value below comes from the reference's own functions; the seeded inputs
are the reference tests' own (P/tests/acceptance.cpp:356-362,
P/tests/test_compression.cpp:54-61) plus the codec-sweep data of SURVEY.md §8(d).

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

R = O.ref
assert R is not None, "build oracle/_ref first (make -C oracle)"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_quantize(x: np.ndarray, bs: int):
    x = np.ascontiguousarray(x, np.float64)
    n = x.size
    codes = np.zeros(max(n, 1), np.int8)
    am = np.zeros(max(O.n_blocks(n, bs), 1), np.float64)
    nb = C.c_size_t(0)
    st = R.ref_quantize_blockwise(O._p(x), n, bs, O._p(codes), O._p(am), C.byref(nb))
    return st, codes[:n], am[: nb.value]


def ref_dequantize(codes, am, bs):
    n = codes.size
    out = np.zeros(max(n, 1), np.float64)
    R.ref_dequantize_blockwise(O._p(np.ascontiguousarray(codes)), n, O._p(np.ascontiguousarray(am)),
                               am.size, bs, O._p(out))
    return out[:n]


def ref_maxout(x, k):
    x = np.ascontiguousarray(x, np.float64)
    out = np.zeros(max(x.size // max(k, 1), 1))
    st = R.ref_maxout_k(O._p(x), x.size, k, O._p(out))
    return st, out[: x.size // k] if st == 0 else None


def ref_ln(x, gain=None, bias=None, eps=1e-5):
    x = np.ascontiguousarray(x, np.float64)
    out = np.zeros_like(x)
    g = None if gain is None else np.ascontiguousarray(gain, np.float64)
    b = None if bias is None else np.ascontiguousarray(bias, np.float64)
    st = R.ref_layer_norm(O._p(x), x.size, None if g is None else O._p(g), None if b is None else O._p(b),
                          eps, O._p(out))
    return st, out


def main() -> None:
    g: dict = {"generator": "tests/golden/make_golden.py", "source": "reference compression.cpp via oracle/_ref"}

    # --- known-answer vectors (P/tests/test_compression.cpp) -----------------
    kat = []
    for name, x, bs in [
        ("basics", [-1.0, 0.0, 0.5, 1.0], 4),                  # :14-29
        ("zero_block", [0.0, 0.0, 0.0], 3),                    # :31-35
        ("independent_blocks", [1.0, -1.0, 1000.0, -500.0], 2),  # :37-46
        ("ragged_tail", [3.0, -2.0, 1.0, 0.25, -0.125], 2),
        ("payload_4096", [1.0] * 4096, 2048),                  # :74-77
        ("smoke_py", [(-1) ** i * 0.01 * i for i in range(4096)], 64),  # test_smoke.py:49-57
    ]:
        st, c, a = ref_quantize(np.array(x), bs)
        y = ref_dequantize(c, a, bs)
        kat.append({"name": name, "x": list(map(float, x)) if len(x) <= 16 else None, "n": len(x),
                    "block_size": bs, "status": st, "codes": c.tolist() if len(x) <= 16 else sha(c),
                    "absmax": a.tolist(), "dequant": y.tolist() if len(x) <= 16 else sha(y)})
    g["quantize_kat"] = kat

    errs = {}
    for name, x, bs in [("nan", [1.0, float("nan")], 2), ("inf", [float("inf")], 1), ("bs0", [1.0], 0)]:
        st, _, _ = ref_quantize(np.array(x), bs)
        errs[name] = st
    g["quantize_errors"] = errs  # 1 == ConfigError

    # --- seeded sets, f64 API --------------------------------------------------
    sets = {}
    for name, x, bs in [("acceptance_2026_1e6", O.gen_acceptance(1_000_000, 2026), 2048),   # acceptance.cpp:355-386
                        ("heavy_tailed_123_1e5", O.gen_heavy_tailed(100_000, 123), 2048)]:  # test_compression.cpp:53-72
        st, c, a = ref_quantize(x, bs)
        y = ref_dequantize(c, a, bs)
        sets[name] = {"n": x.size, "block_size": bs, "x_sha": sha(x), "codes_sha": sha(c), "absmax_sha": sha(a),
                      "dequant_f64_sha": sha(y), "codes_head": c[:32].tolist(), "absmax_head": a[:4].tolist(),
                      "max_err_minus_bound": float(np.max(np.abs(y - x) - 0.5 * np.repeat(a, bs)[: x.size] / 127.0))}
    g["f64_sets"] = sets

    # --- codec sweep data, fp32 and bf16 wire -------
    sweep = {}
    for n, blk in [(1 << 20, 4096), (1 << 20, 2048), ((1 << 20) + 1234, 4096)]:
        x32 = O.gen_sweep_f32(n, blk, seed=7)
        st, c, a = ref_quantize(x32.astype(np.float64), blk)
        y = ref_dequantize(c, a, blk)
        key = f"f32_n{n}_bs{blk}"
        sweep[key] = {"n": n, "block_size": blk, "seed": 7, "x_sha": sha(x32), "codes_sha": sha(c),
                      "scales_f32_sha": sha(a.astype(np.float32)), "dequant_f32_sha": sha(y.astype(np.float32)),
                      "n_exact_ties": int(np.sum(np.abs(127.0 * x32.astype(np.float64) / np.repeat(a, blk)[:n] % 1.0 - 0.5) == 0))}
        xb = O.f32_to_bf16_bits(x32)
        st, c, a = ref_quantize(O.bf16_bits_to_f32(xb).astype(np.float64), blk)
        y = ref_dequantize(c, a, blk)
        yb = np.array([O.f64_to_bf16_bits(v) for v in y[:4096]], np.uint16)
        sweep[key.replace("f32", "bf16")] = {
            "n": n, "block_size": blk, "seed": 7, "x_sha": sha(xb), "codes_sha": sha(c),
            "scales_f32_sha": sha(a.astype(np.float32)), "dequant_bf16_head4096_sha": sha(yb)}
    g["sweep_sets"] = sweep

    # --- maxout / layer_norm / bottleneck / payload ----------------------------
    mo = []
    for x, k in [([1.0, 5.0, 2.0, 2.0, -3.0, -1.0], 2), ([4.0, 4.0], 1), ([1.0, 2.0, 3.0], 2),
                 ([0.25] * 4 + [-7.0] * 4 + [3.5] * 4, 4), ([2.0, 2.0, -1.0, -1.0], 2), ([], 2), ([1.0], 0)]:
        st, y = ref_maxout(np.array(x, np.float64), k)
        mo.append({"x": x, "k": k, "status": st, "out": None if y is None else y.tolist()})
    g["maxout_kat"] = mo

    lns = []
    for x, gain, bias, eps in [([1.0, 2.0, 3.0, 4.0], None, None, 1e-5),
                               ([1.0, 2.0, 3.0, 4.0], [2.0] * 4, [1.0] * 4, 1e-5),
                               ([3.0, -1.0, 0.5, 2.5], None, None, 0.0)]:
        st, y = ref_ln(np.array(x), gain, bias, eps)
        lns.append({"x": x, "gain": gain, "bias": bias, "eps": eps, "status": st, "out": y.tolist()})
    rng = np.random.default_rng(11)
    x = rng.standard_normal(2048) * 3 + 0.5
    st, y = ref_ln(x)
    lns.append({"x_seed": 11, "n": 2048, "status": st, "out_sha": sha(y), "out_head": y[:8].tolist()})
    g["layer_norm_kat"] = lns

    payload = {}
    for name, d, L, b, ab in [("base", 768, 512, 1, 2.0), ("xxlarge", 4096, 512, 1, 2.0), ("gpt3", 12288, 512, 1, 2.0),
                              ("ours", 4096, 512, 1, 2.0), ("configC_B4", 2048, 512, 4, 2.0)]:
        payload[name] = {k: R.ref_payload_bits(d, L, b, ab, kind, f)
                         for k, kind, f in [("none", 0, 1.0), ("int8", 1, 1.0), ("bottleneck_0.25", 2, 0.25),
                                            ("maxout_2", 3, 2.0)]}
    g["payload_bits"] = payload

    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "codec_golden.json")
    with open(out, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", out)


if __name__ == "__main__":
    main()
