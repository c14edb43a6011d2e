"""CPU: pin the oracle (oracle/codec_oracle.c) before trusting it.

(1) against the reference's own known-answer tests (P/tests/test_compression.cpp,
    P/tests/acceptance.cpp:355-386, P/tests/python/test_smoke.py:49-57) as captured
    in tests/golden/codec_golden.json by running the unmodified reference;
(2) against the reference library itself (oracle/_ref) when it is built here.
"""
import ctypes as C
import hashlib

import numpy as np
import pytest

import oracle as O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_mt19937_64_matches_std():
    # the 10000th output of a default-seeded std::mt19937_64 is fixed by the C++ standard
    assert int(O.mt64(5489, 10000)[-1]) == 9981545732273789042
    if O.ref is not None:
        b = np.empty(2000, np.uint64)
        O.ref.ref_mt64(2026, 2000, O._p(b))
        assert (O.mt64(2026, 2000) == b).all()


def test_quantize_kats(golden):
    for kat in golden["quantize_kat"]:
        n, bs = kat["n"], kat["block_size"]
        if kat["x"] is not None:
            x = np.array(kat["x"], np.float64)
        elif kat["name"] == "payload_4096":
            x = np.ones(4096)
        else:  # smoke_py
            x = np.array([(-1) ** i * 0.01 * i for i in range(n)], np.float64)
        st, codes, am = O.quantize(x, bs)
        assert st == kat["status"]
        assert am.tolist() == kat["absmax"], kat["name"]
        if isinstance(kat["codes"], list):
            assert codes.tolist() == kat["codes"], kat["name"]
            y = O.dequantize(codes, am, bs, np.float64)
            assert y.tolist() == kat["dequant"], kat["name"]
        else:
            assert sha(codes) == kat["codes"], kat["name"]
            assert sha(O.dequantize(codes, am, bs, np.float64)) == kat["dequant"], kat["name"]


def test_basic_kat_literal():
    # P/tests/test_compression.cpp:14-29 verbatim expectations
    st, c, a = O.quantize(np.array([-1.0, 0.0, 0.5, 1.0]), 4)
    assert st == 0 and c.tolist() == [-127, 0, 64, 127] and a.tolist() == [1.0]


def test_quantize_errors(golden):
    e = golden["quantize_errors"]
    assert O.quantize(np.array([1.0, np.nan]), 2)[0] == O.E_NONFINITE and e["nan"] == 1
    assert O.quantize(np.array([np.inf]), 1)[0] == O.E_NONFINITE and e["inf"] == 1
    assert O.quantize(np.array([1.0]), 0)[0] == O.E_INVALID and e["bs0"] == 1


@pytest.mark.parametrize("name,gen", [("acceptance_2026_1e6", lambda: O.gen_acceptance(1_000_000, 2026)),
                                      ("heavy_tailed_123_1e5", lambda: O.gen_heavy_tailed(100_000, 123))])
def test_seeded_sets(golden, name, gen):
    g = golden["f64_sets"][name]
    x = gen()
    assert sha(x) == g["x_sha"]
    st, c, a = O.quantize(x, g["block_size"])
    assert st == 0
    assert sha(c) == g["codes_sha"] and sha(a) == g["absmax_sha"]
    y = O.dequantize(c, a, g["block_size"], np.float64)
    assert sha(y) == g["dequant_f64_sha"]
    # acceptance #8 / test_compression.cpp:53-72: |y - x| <= 0.5*absmax/127 (+1e-12)
    bound = 0.5 * np.repeat(a, g["block_size"])[: x.size] / 127.0 + 1e-12
    assert np.all(np.abs(y - x) <= bound)


def test_sweep_sets(golden):
    for key, g in golden["sweep_sets"].items():
        x32 = O.gen_sweep_f32(g["n"], g["block_size"], seed=g["seed"])
        bs = g["block_size"]
        if key.startswith("f32"):
            assert sha(x32) == g["x_sha"]
            st, c, s = O.quantize(x32, bs)
            assert st == 0 and sha(c) == g["codes_sha"] and sha(s) == g["scales_f32_sha"], key
            assert sha(O.dequantize(c, s, bs, np.float32)) == g["dequant_f32_sha"], key
            assert g["n_exact_ties"] > 1000  # the sweep really exercises half-steps
        else:
            xb = O.f32_to_bf16_bits(x32)
            assert sha(xb) == g["x_sha"]
            st, c, s = O.quantize(xb, bs)
            assert st == 0 and sha(c) == g["codes_sha"] and sha(s) == g["scales_f32_sha"], key
            yb = O.dequantize(c[:4096], s[: 4096 // bs + 1], bs, np.uint16)
            assert sha(yb) == g["dequant_bf16_head4096_sha"], key


def test_f64_to_bf16_is_single_rounding():
    from fractions import Fraction
    rng = np.random.default_rng(3)
    vals = list(rng.standard_normal(500) * 10.0 ** rng.integers(-30, 30, 500)) + [1.0 + 2 ** -8, 1.0 + 2 ** -9,
                                                                                  1.0 + 2 ** -9 + 2 ** -40, -3.0e38]
    for v in vals:
        b = O.f64_to_bf16_bits(float(v))
        got = Fraction(float(O.bf16_bits_to_f32(np.array([b], np.uint16))[0]))
        fv = Fraction(float(v))
        # neighbours of `got` in bf16
        up = Fraction(float(O.bf16_bits_to_f32(np.array([b + 1], np.uint16))[0]))
        dn = Fraction(float(O.bf16_bits_to_f32(np.array([b - 1], np.uint16))[0]))
        assert abs(got - fv) <= abs(up - fv) and abs(got - fv) <= abs(dn - fv), v


def test_maxout_kats(golden):
    for kat in golden["maxout_kat"]:
        st, out, am = O.maxout(np.array(kat["x"], np.float64), kat["k"])
        assert st == kat["status"]
        if st == 0:
            assert out.tolist() == kat["out"]
    # earliest of tied maxima wins (std::max): argmax 0 for [2, 2]
    st, out, am = O.maxout(np.array([2.0, 2.0, -1.0, -1.0, 0.0, 3.0]), 2)
    assert am.tolist() == [0, 0, 1]


def test_layer_norm_kats(golden):
    for kat in golden["layer_norm_kat"]:
        if "x" in kat:
            st, y = O.layer_norm(np.array(kat["x"]), kat["gain"], kat["bias"], kat["eps"])
            assert st == kat["status"]
            np.testing.assert_allclose(y, kat["out"], rtol=0, atol=1e-15)
        else:
            x = np.random.default_rng(kat["x_seed"]).standard_normal(kat["n"]) * 3 + 0.5
            st, y = O.layer_norm(x)
            assert sha(y) == kat["out_sha"]  # same op order as the reference: bit-identical


@pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built")
def test_oracle_matches_reference_random():
    rng = np.random.default_rng(5)
    for n, bs in [(1, 1), (7, 3), (5000, 64), (10000, 2048), (4096 * 3 + 17, 4096)]:
        x = rng.standard_normal(n) * rng.choice([1e-3, 1.0, 1e6], n)
        codes = np.empty(n, np.int8)
        am = np.empty(O.n_blocks(n, bs))
        nb = C.c_size_t()
        assert O.ref.ref_quantize_blockwise(O._p(x), n, bs, O._p(codes), O._p(am), C.byref(nb)) == 0
        st, c2, a2 = O.quantize(x, bs)
        assert (codes == c2).all() and (am == a2).all()
        out = np.empty(n)
        O.ref.ref_dequantize_blockwise(O._p(codes), n, O._p(am), am.size, bs, O._p(out))
        assert (out == O.dequantize(codes, am, bs, np.float64)).all()
