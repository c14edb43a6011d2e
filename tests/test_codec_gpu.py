"""GPU parity: K1/K2 codec through the C-ABI vs the oracle, bit-exact.

int8 codes and per-block scales must be identical to the reference's
fp64 formula (compression.cpp:10-29) for f32, bf16 and f64 inputs; dequantized
values must equal the reference's fp64 value rounded once to the output dtype.
"""
import hashlib

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gpu_quant(x_np, bs, dtype):
    import torch
    from paper_2301_11913_b200 import ops
    if dtype == "bf16":
        t = torch.from_numpy(x_np.view(np.int16)).cuda().view(torch.bfloat16)
    else:
        t = torch.from_numpy(x_np).cuda()
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    c, s = ops.quantize(t, bs, flags=flags)
    torch.cuda.synchronize()
    return c.cpu().numpy(), s.cpu().numpy(), int(flags.item())


SIZES = [0, 1, 5, 64, 4095, 4096, 4097, 3 * 4096, 65536 + 123, 1 << 20]


@pytest.mark.parametrize("bs", [4096, 2048, 1024, 64, 3, 5000])
@pytest.mark.parametrize("n", SIZES)
def test_quantize_f32_bitexact(cuda, n, bs):
    x = O.gen_sweep_f32(n, bs, seed=n + bs)
    c, s, fl = gpu_quant(x, bs, "f32")
    st, c0, s0 = O.quantize(x, bs)
    assert st == 0 and fl == 0
    assert np.array_equal(c, c0), f"{np.sum(c != c0)} code mismatches"
    assert np.array_equal(s, s0)


@pytest.mark.parametrize("bs", [4096, 2048, 100])
@pytest.mark.parametrize("n", [1, 4096, 4096 * 5 + 7, 1 << 20])
def test_quantize_bf16_bitexact(cuda, n, bs):
    xb = O.f32_to_bf16_bits(O.gen_sweep_f32(n, bs, seed=3))
    c, s, fl = gpu_quant(xb, bs, "bf16")
    st, c0, s0 = O.quantize(xb, bs)
    assert st == 0 and fl == 0
    assert np.array_equal(c, c0), f"{np.sum(c != c0)} code mismatches"
    assert np.array_equal(s, s0)


@pytest.mark.parametrize("bs", [2048, 64, 7])
def test_quantize_f64_bitexact(cuda, bs):
    x = O.gen_acceptance(200_003, 2026)
    c, s, fl = gpu_quant(x, bs, "f64")
    st, c0, s0 = O.quantize(x, bs)
    assert np.array_equal(c, c0) and np.array_equal(s, s0)


def test_golden_sweep_hashes(cuda, golden):
    """Against the reference's own outputs (tests/golden, made by oracle/_ref)."""
    import torch
    from paper_2301_11913_b200 import ops
    for key, g in golden["sweep_sets"].items():
        x32 = O.gen_sweep_f32(g["n"], g["block_size"], seed=g["seed"])
        bs = g["block_size"]
        if key.startswith("f32"):
            c, s, _ = gpu_quant(x32, bs, "f32")
            assert sha(c) == g["codes_sha"] and sha(s) == g["scales_f32_sha"], key
            y = ops.dequantize(torch.from_numpy(c).cuda(), torch.from_numpy(s).cuda(), bs, torch.float32)
            assert sha(y.cpu().numpy()) == g["dequant_f32_sha"], key
        else:
            xb = O.f32_to_bf16_bits(x32)
            c, s, _ = gpu_quant(xb, bs, "bf16")
            assert sha(c) == g["codes_sha"] and sha(s) == g["scales_f32_sha"], key
            y = ops.dequantize(torch.from_numpy(c).cuda(), torch.from_numpy(s).cuda(), bs, torch.bfloat16)
            yb = y.view(torch.int16).cpu().numpy().view(np.uint16)[:4096]
            assert sha(yb) == g["dequant_bf16_head4096_sha"], key


def test_golden_f64_sets(cuda, golden):
    for name, gen in [("acceptance_2026_1e6", lambda: O.gen_acceptance(1_000_000, 2026)),
                      ("heavy_tailed_123_1e5", lambda: O.gen_heavy_tailed(100_000, 123))]:
        g = golden["f64_sets"][name]
        c, s, _ = gpu_quant(gen(), g["block_size"], "f64")
        assert sha(c) == g["codes_sha"] and sha(s) == g["absmax_sha"], name


@pytest.mark.parametrize("out", ["f32", "bf16", "f64"])
@pytest.mark.parametrize("n,bs", [(1 << 20, 4096), (4096 * 3 + 5, 4096), (1000, 64), (77, 5)])
def test_dequantize_bitexact(cuda, out, n, bs):
    import torch
    from paper_2301_11913_b200 import ops
    x = O.gen_sweep_f32(n, bs, seed=11)
    st, c0, s0 = O.quantize(x, bs)
    if out == "f64":
        s0 = s0.astype(np.float64)
    dt = {"f32": torch.float32, "bf16": torch.bfloat16, "f64": torch.float64}[out]
    y = ops.dequantize(torch.from_numpy(c0).cuda(), torch.from_numpy(s0).cuda(), bs, dt)
    if out == "bf16":
        got = y.view(torch.int16).cpu().numpy().view(np.uint16)
        exp = O.dequantize(c0, s0, bs, np.uint16)
    else:
        got = y.cpu().numpy()
        exp = O.dequantize(c0, s0, bs, np.float32 if out == "f32" else np.float64)
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("out", ["f32", "bf16"])
@pytest.mark.parametrize("bs", [4096, 64, 4])
def test_dequantize_arbitrary_codes_and_scales(cuda, out, bs):
    """Every code byte (incl. -128) against scales over the whole fp32 range:
    the arithmetic path's [2^-64, 2^65) guard edges, zero, subnormals, FLT_MAX,
    and random mantissas (bf16: ~1.8e-5 of pairs hit the midpoint fallback)."""
    import torch
    from paper_2301_11913_b200 import ops
    rng = np.random.default_rng(bs)
    n = 1 << 21
    codes = rng.integers(-128, 128, n, dtype=np.int16).astype(np.int8)
    nb = n // bs
    bits = rng.integers(0, 0x7F800000, nb, dtype=np.int64).astype(np.uint32)
    mant = rng.integers(0, 1 << 23, nb, dtype=np.int64).astype(np.uint32)
    bits[: nb // 2] = ((rng.integers(60, 195, nb // 2) << 23).astype(np.uint32) | mant[: nb // 2])
    special = np.array([0.0, 1e-45, 1.17e-38, 2.0 ** -64, np.nextafter(np.float32(2.0 ** -64), 0),
                        2.0 ** 65, np.nextafter(np.float32(2.0 ** 65), 0), 3.4028235e38, 1.0], np.float32)
    scales = bits.view(np.float32).copy()
    scales[: special.size] = special
    dt = {"f32": torch.float32, "bf16": torch.bfloat16}[out]
    y = ops.dequantize(torch.from_numpy(codes).cuda(), torch.from_numpy(scales).cuda(), bs, dt)
    if out == "bf16":
        got = y.view(torch.int16).cpu().numpy().view(np.uint16)
        exp = O.dequantize(codes, scales, bs, np.uint16)
    else:
        got = y.cpu().numpy().view(np.uint32)
        exp = O.dequantize(codes, scales, bs, np.float32).view(np.uint32)
    assert np.array_equal(got, exp), f"{int((got != exp).sum())} mismatches"


def test_all_128_negative_code_and_zero_block(cuda):
    import torch
    from paper_2301_11913_b200 import ops
    codes = torch.tensor([-128, -127, 0, 127] * 1024, dtype=torch.int8, device="cuda")
    scales = torch.tensor([3.0], dtype=torch.float32, device="cuda")
    y = ops.dequantize(codes, scales, 4096, torch.float32).cpu().numpy()
    exp = O.dequantize(codes.cpu().numpy(), np.array([3.0], np.float32), 4096, np.float32)
    assert np.array_equal(y, exp)
    c, s, _ = gpu_quant(np.zeros(8192, np.float32), 4096, "f32")
    assert not c.any() and not s.any()


BAD = {"nan": (np.nan, 0x7FC0), "inf": (np.inf, 0x7F80), "-inf": (-np.inf, 0xFF80)}


@pytest.mark.parametrize("bad", list(BAD))
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f64"])
def test_nonfinite_sets_flag(cuda, bad, dtype):
    val, bits = BAD[bad]
    x = np.linspace(-1, 1, 3 * 4096).astype(np.float64)
    x[5000] = val
    if dtype == "f32":
        x = x.astype(np.float32)
    elif dtype == "bf16":
        x = O.f32_to_bf16_bits(np.nan_to_num(x).astype(np.float32))
        x[5000] = bits
    _, _, fl = gpu_quant(x, 4096, dtype)
    assert fl & 1


def test_block_size_zero_is_config_error(cuda):
    import torch
    from paper_2301_11913_b200 import ConfigError, ops
    with pytest.raises(ConfigError):
        ops.quantize(torch.ones(4, device="cuda"), 0)


def test_full_size_roundtrip_properties(cuda):
    """BASELINE size (2^28 fp32 = 1 GiB): codes vs oracle on the whole tensor,
    plus the exact error bound of acceptance #8 after the round trip."""
    import torch
    from paper_2301_11913_b200 import ops
    n, bs = 1 << 28, 4096
    g = torch.Generator(device="cuda").manual_seed(1)
    x = (torch.rand(n, device="cuda", generator=g) * 2 - 1)
    x[::11] *= 500
    c, s = ops.quantize(x, bs)
    y = ops.dequantize(c, s, bs, torch.float32)
    err = (y.double() - x.double()).abs().view(-1, bs).amax(1)
    # exact bound of acceptance #8 plus the one fp32 rounding of the dequantized value
    ymax = y.abs().view(-1, bs).amax(1).double()
    bound = 0.5 * s.double() / 127.0 + ymax * 2.0 ** -24
    assert bool((err <= bound).all())
    # the whole 1 GiB tensor bit-exactly against the oracle
    st, c0, s0 = O.quantize(x.cpu().numpy(), bs)
    assert st == 0
    assert np.array_equal(c.cpu().numpy(), c0)
    assert np.array_equal(s.cpu().numpy(), s0)


def test_host_entry_points_match_device(cuda):
    import ctypes as C
    from paper_2301_11913_b200 import _lib
    L = _lib.lib()
    x = O.gen_sweep_f32((1 << 22) + 999, 4096, seed=9)
    codes = np.empty(x.size, np.int8)
    scales = np.empty(O.n_blocks(x.size, 4096), np.float32)
    rc = L.swarm_quantize_blockwise_host(x.ctypes.data_as(C.c_void_p), _lib.DT_F32, x.size, 4096,
                                         codes.ctypes.data_as(C.c_void_p), scales.ctypes.data_as(C.c_void_p))
    assert rc == 0
    st, c0, s0 = O.quantize(x, 4096)
    assert np.array_equal(codes, c0) and np.array_equal(scales, s0)
    out = np.empty(x.size, np.float32)
    rc = L.swarm_dequantize_blockwise_host(codes.ctypes.data_as(C.c_void_p), scales.ctypes.data_as(C.c_void_p),
                                           _lib.DT_F32, x.size, 4096, out.ctypes.data_as(C.c_void_p), _lib.DT_F32)
    assert rc == 0 and np.array_equal(out, O.dequantize(c0, s0, 4096, np.float32))
    x[7] = np.nan
    rc = L.swarm_quantize_blockwise_host(x.ctypes.data_as(C.c_void_p), _lib.DT_F32, x.size, 4096,
                                         codes.ctypes.data_as(C.c_void_p), scales.ctypes.data_as(C.c_void_p))
    assert rc == _lib.SWARM_E_NONFINITE
