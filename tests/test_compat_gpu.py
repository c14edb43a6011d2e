"""GPU: the reference-compatible API (same names as P/bindings/module.cpp:143-163)
reproduces the reference's tests — P/tests/test_compression.cpp and
P/tests/python/test_smoke.py::test_quantization_roundtrip — on the B200 path."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sw(cuda):
    import paper_2301_11913_b200 as m
    return m


def test_quantize_basics(sw):  # test_compression.cpp:14-29
    q = sw.quantize_blockwise([-1.0, 0.0, 0.5, 1.0], 4)
    assert list(q.codes) == [-127, 0, 64, 127]
    assert list(q.absmax) == [1.0] and q.block_size == 4
    y = sw.dequantize_blockwise(q)
    assert y[0] == pytest.approx(-1.0) and y[3] == pytest.approx(1.0)
    assert abs(y[2] - 0.5) <= 0.5 / 127.0


def test_zero_block(sw):  # :31-35
    q = sw.quantize_blockwise([0.0, 0.0, 0.0], 3)
    assert list(q.codes) == [0, 0, 0]
    assert sw.dequantize_blockwise(q) == [0.0, 0.0, 0.0]


def test_independent_blocks(sw):  # :37-46
    q = sw.quantize_blockwise([1.0, -1.0, 1000.0, -500.0], 2)
    assert list(q.absmax) == [1.0, 1000.0]
    y = sw.dequantize_blockwise(q)
    assert y[0] == pytest.approx(1.0) and y[2] == pytest.approx(1000.0)


def test_nonfinite_rejected(sw):  # :48-51
    with pytest.raises(sw.ConfigError):
        sw.quantize_blockwise([1.0, float("nan")], 2)
    with pytest.raises(sw.ConfigError):
        sw.quantize_blockwise([float("inf")], 1)
    with pytest.raises(ValueError):  # ConfigError is a ValueError subclass (module.cpp:20)
        sw.quantize_blockwise([1.0], 0)


def test_golden_kats(sw, golden):
    for kat in golden["quantize_kat"]:
        if kat["x"] is None:
            continue
        q = sw.quantize_blockwise(kat["x"], kat["block_size"])
        assert list(q.codes) == kat["codes"] and list(q.absmax) == kat["absmax"], kat["name"]
        assert sw.dequantize_blockwise(q) == kat["dequant"], kat["name"]


def test_roundtrip_bound_heavy_tailed(sw, golden):  # :53-72, bit-exact vs the reference too
    x = O.gen_heavy_tailed(100_000, 123)
    q = sw.quantize_blockwise(x.tolist(), 2048)
    c = np.array(q.codes, np.int8)
    a = np.array(q.absmax)
    import hashlib
    assert hashlib.sha256(c.tobytes()).hexdigest() == golden["f64_sets"]["heavy_tailed_123_1e5"]["codes_sha"]
    y = np.array(sw.dequantize_blockwise(q))
    bound = 0.5 * np.repeat(a, 2048)[: x.size] / 127.0 + 1e-12
    assert np.all(np.abs(y - x) <= bound)


def test_payload(sw):  # :74-77
    q = sw.quantize_blockwise([1.0] * 4096, 2048)
    assert q.payload_bits() == 4096 * 8 + 2 * 32


def test_maxout(sw):  # :79-94
    assert sw.maxout_k([1.0, 5.0, 2.0, 2.0, -3.0, -1.0], 2) == [5.0, 2.0, -1.0]
    assert sw.maxout_k([4.0, 4.0], 1) == [4.0, 4.0]
    with pytest.raises(sw.ConfigError):
        sw.maxout_k([1.0, 2.0, 3.0], 2)
    x = [0.25, -7.0, 3.5]
    assert sw.maxout_k([v for v in x for _ in range(4)], 4) == x


def test_layer_norm(sw, golden):  # :96-118 (the binding exposes the no-params overload)
    y = sw.layer_norm([1.0, 2.0, 3.0, 4.0])
    assert np.mean(y) == pytest.approx(0.0, abs=1e-9)
    assert np.var(y) == pytest.approx(1.0, rel=1e-3)
    np.testing.assert_allclose(y, golden["layer_norm_kat"][0]["out"], rtol=1e-15, atol=1e-15)
    with pytest.raises(sw.ConfigError):
        sw.layer_norm([])


def test_bottleneck_identity(sw):  # :120-136
    x = [3.0, -1.0, 0.5, 2.5]
    eye = [[1.0 if i == j else 0.0 for j in range(4)] for i in range(4)]
    sent = sw.bottleneck_forward(x, eye, 0.0)
    back = sw.bottleneck_decompress(sent, eye)
    st, exp = O.layer_norm(np.array(x), eps=0.0)
    np.testing.assert_allclose(back, exp, rtol=1e-15)
    assert len(sw.bottleneck_forward(x, [[0.25, 0.25]] * 4, 0.0)) == 2
    with pytest.raises(sw.ConfigError):
        sw.bottleneck_decompress([1.0, 2.0], [[1.0]])


def test_bottleneck_matches_reference_order(sw):
    rng = np.random.default_rng(4)
    x = rng.standard_normal(96)
    w = rng.standard_normal((96, 40))
    st, ln = O.layer_norm(x)
    exp = O.matvec(ln, w)
    got = np.array(sw.bottleneck_forward(x.tolist(), w.tolist(), 1e-5))
    np.testing.assert_allclose(got, exp, rtol=1e-13, atol=1e-13)
    # the matvec alone is bit-identical (same accumulation order, unfused fp64)
    assert np.array_equal(np.array(sw.bottleneck_decompress(ln.tolist(), w.tolist())), exp)


def test_smoke_py_roundtrip(sw):  # P/tests/python/test_smoke.py:49-57
    values = [(-1) ** i * 0.01 * i for i in range(4096)]
    q = sw.quantize_blockwise(values, 64)
    back = sw.dequantize_blockwise(q)
    absmax = max(abs(v) for v in values)
    assert max(abs(a - b) for a, b in zip(values, back)) <= 0.5 * absmax / 127 + 1e-12
    shape = sw.preset("base")
    assert sw.compressed_payload_bits(shape, "int8") * 2 == sw.activation_payload_bits(shape)
