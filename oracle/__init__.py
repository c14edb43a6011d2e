"""TEST INFRASTRUCTURE ONLY — ctypes front end of the CPU oracle.

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker.
The product package ``paper_2301_11913_b200`` never imports it.

* ``orc``  — ``liborc.so``, the plain-C restatement of
  ``/root/reference/proj/src/compression.cpp`` (codec_oracle.c).
* ``ref``  — ``_ref/libswarmsim_ref.so``, the UNMODIFIED reference compiled in
  place by ``oracle/Makefile`` (None when it was never built).
* ``block_oracle`` — numpy fp64 transformer-block forward/backward (the
  reference has none: parity for the block math is UNPINNED).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "liborc.so")
REF_PATH = os.path.join(HERE, "_ref", "libswarmsim_ref.so")
HOOKED_PATH = os.path.join(HERE, "_ref", "libswarmsim_hooked.so")

OK, E_INVALID, E_NONFINITE = 0, 1, 2


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load_orc():
    if not os.path.exists(ORC_PATH):
        build()
    lib = C.CDLL(ORC_PATH)
    P = C.c_void_p
    sz = C.c_size_t
    lib.orc_gen_acceptance.argtypes = [C.c_uint64, sz, P]
    lib.orc_gen_heavy_tailed.argtypes = [C.c_uint64, sz, P]
    lib.orc_gen_sweep_f32.argtypes = [C.c_uint64, sz, sz, P]
    lib.orc_mt64_seed.argtypes = [P, C.c_uint64]
    lib.orc_mt64_next.argtypes = [P]
    lib.orc_mt64_next.restype = C.c_uint64
    for f in ("orc_quantize_f64", "orc_quantize_f32", "orc_quantize_bf16"):
        getattr(lib, f).argtypes = [P, sz, sz, P, P]
        getattr(lib, f).restype = C.c_int
    for f in ("orc_dequantize_f64", "orc_dequantize_f32", "orc_dequantize_bf16"):
        getattr(lib, f).argtypes = [P, sz, P, sz, P]
    lib.orc_maxout_f64.argtypes = [P, sz, sz, P, P]
    lib.orc_maxout_f64.restype = C.c_int
    lib.orc_layer_norm_f64.argtypes = [P, sz, P, P, C.c_double, P]
    lib.orc_layer_norm_f64.restype = C.c_int
    lib.orc_matvec_f64.argtypes = [P, sz, P, sz, P]
    lib.orc_f64_to_bf16.argtypes = [C.c_double]
    lib.orc_f64_to_bf16.restype = C.c_uint16
    return lib


def _load_ref():
    if not os.path.exists(REF_PATH):
        return None
    lib = C.CDLL(REF_PATH)
    P = C.c_void_p
    sz = C.c_size_t
    lib.ref_quantize_blockwise.argtypes = [P, sz, sz, P, P, P]
    lib.ref_dequantize_blockwise.argtypes = [P, sz, P, sz, sz, P]
    lib.ref_maxout_k.argtypes = [P, sz, sz, P]
    lib.ref_layer_norm.argtypes = [P, sz, P, P, C.c_double, P]
    lib.ref_bottleneck_forward.argtypes = [P, sz, P, sz, C.c_double, P]
    lib.ref_payload_bits.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_int, C.c_double]
    lib.ref_payload_bits.restype = C.c_double
    lib.ref_mt64.argtypes = [C.c_uint64, sz, P]
    lib.ref_codec_prepare.argtypes = [P, sz, sz, C.c_int]
    lib.ref_codec_prepare.restype = P
    lib.ref_codec_run.argtypes = [P, C.c_int]
    lib.ref_codec_run.restype = C.c_uint64
    lib.ref_codec_codes.argtypes = [P, P, P]
    lib.ref_codec_free.argtypes = [P]
    lib.ref_router_new.argtypes = [sz, C.c_double, C.c_double]
    lib.ref_router_new.restype = P
    lib.ref_router_free.argtypes = [P]
    lib.ref_router_add_server.argtypes = [P, C.c_uint64, P, sz, C.c_double]
    lib.ref_router_ban_server.argtypes = [P, C.c_uint64]
    lib.ref_router_remove_server.argtypes = [P, C.c_uint64]
    lib.ref_router_choose_server.argtypes = [P, sz, P]
    lib.ref_router_record_response.argtypes = [P, C.c_uint64, C.c_double]
    lib.ref_router_ema_of.argtypes = [P, C.c_uint64]
    lib.ref_router_ema_of.restype = C.c_double
    lib.ref_router_priority_of.argtypes = [P, C.c_uint64]
    lib.ref_router_priority_of.restype = C.c_double
    lib.ref_rebalance_decide.argtypes = [sz, P, P, P, P, P, P, P]
    lib.ref_oracle_throughput.argtypes = [P, sz, C.c_int64]
    lib.ref_oracle_throughput.restype = C.c_double
    lib.ref_stage_cost.argtypes = [P, C.c_double, P, C.c_int, P]
    lib.ref_stage_cost.restype = C.c_int
    lib.ref_sim_run.argtypes = [C.c_char_p, C.c_uint64, P, P, P, sz, P]
    lib.ref_sim_run.restype = C.c_int
    lib.ref_sim_run_churn.argtypes = [C.c_char_p, P, P, sz, C.c_uint64, P, P, sz, P, C.c_char_p, sz]
    lib.ref_sim_run_churn.restype = C.c_int
    return lib


orc = _load_orc()
ref = _load_ref()


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- generators
def gen_acceptance(n: int = 1_000_000, seed: int = 2026) -> np.ndarray:
    out = np.empty(n, np.float64)
    orc.orc_gen_acceptance(seed, n, _p(out))
    return out


def gen_heavy_tailed(n: int = 100_000, seed: int = 123) -> np.ndarray:
    out = np.empty(n, np.float64)
    orc.orc_gen_heavy_tailed(seed, n, _p(out))
    return out


def gen_sweep_f32(n: int, block: int = 4096, seed: int = 7) -> np.ndarray:
    out = np.empty(n, np.float32)
    orc.orc_gen_sweep_f32(seed, n, block, _p(out))
    return out


def mt64(seed: int, n: int) -> np.ndarray:
    st = (C.c_uint64 * 313)()
    orc.orc_mt64_seed(st, seed)
    return np.array([orc.orc_mt64_next(st) for _ in range(n)], np.uint64)


# ---------------------------------------------------------------- codec
def n_blocks(n: int, bs: int) -> int:
    return (n + bs - 1) // bs if bs else 0


def quantize(x: np.ndarray, bs: int):
    """Returns (status, codes int8[n], scales) with scales f64 for f64 input,
    f32 for f32 / bf16 (pass bf16 as a uint16 array) input."""
    n = x.size
    codes = np.zeros(n, np.int8)
    if x.dtype == np.float64:
        scales = np.zeros(max(n_blocks(n, bs), 1), np.float64)
        st = orc.orc_quantize_f64(_p(x), n, bs, _p(codes), _p(scales))
    elif x.dtype == np.float32:
        scales = np.zeros(max(n_blocks(n, bs), 1), np.float32)
        st = orc.orc_quantize_f32(_p(x), n, bs, _p(codes), _p(scales))
    elif x.dtype == np.uint16:
        scales = np.zeros(max(n_blocks(n, bs), 1), np.float32)
        st = orc.orc_quantize_bf16(_p(x), n, bs, _p(codes), _p(scales))
    else:
        raise TypeError(x.dtype)
    return st, codes, scales[: n_blocks(n, bs)]


def dequantize(codes: np.ndarray, scales: np.ndarray, bs: int, out_dtype) -> np.ndarray:
    n = codes.size
    codes = np.ascontiguousarray(codes, np.int8)
    if out_dtype == np.float64:
        out = np.empty(n, np.float64)
        orc.orc_dequantize_f64(_p(codes), n, _p(np.ascontiguousarray(scales, np.float64)), bs, _p(out))
    elif out_dtype == np.float32:
        out = np.empty(n, np.float32)
        orc.orc_dequantize_f32(_p(codes), n, _p(np.ascontiguousarray(scales, np.float32)), bs, _p(out))
    elif out_dtype == np.uint16:  # bf16 bits
        out = np.empty(n, np.uint16)
        orc.orc_dequantize_bf16(_p(codes), n, _p(np.ascontiguousarray(scales, np.float32)), bs, _p(out))
    else:
        raise TypeError(out_dtype)
    return out


def maxout(x: np.ndarray, k: int):
    x = np.ascontiguousarray(x, np.float64)
    n = x.size
    out = np.empty(max(n // k, 1) if k else 1, np.float64)
    am = np.empty_like(out, dtype=np.uint8)
    st = orc.orc_maxout_f64(_p(x), n, k, _p(out), _p(am))
    return st, out[: (n // k if k else 0)], am[: (n // k if k else 0)]


def layer_norm(x: np.ndarray, gain=None, bias=None, eps: float = 1e-5):
    x = np.ascontiguousarray(x, np.float64)
    out = np.empty_like(x)
    g = None if gain is None else np.ascontiguousarray(gain, np.float64)
    b = None if bias is None else np.ascontiguousarray(bias, np.float64)
    st = orc.orc_layer_norm_f64(_p(x), x.size, None if g is None else _p(g), None if b is None else _p(b),
                                eps, _p(out))
    return st, out


def matvec(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    w = np.ascontiguousarray(w, np.float64)
    out = np.empty(w.shape[1], np.float64)
    orc.orc_matvec_f64(_p(x), w.shape[0], _p(w), w.shape[1], _p(out))
    return out


def f64_to_bf16_bits(d: float) -> int:
    return int(orc.orc_f64_to_bf16(d))


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bits (finite inputs)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return r.astype(np.uint16)


def _load_hooked():
    """The reference engine with the additive record hook (oracle/hook_patch.py), or None."""
    if not os.path.exists(HOOKED_PATH):
        return None
    lib = C.CDLL(HOOKED_PATH)
    lib.hooked_sim_run.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint64, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p]
    lib.hooked_sim_run.restype = C.c_int
    return lib


hooked = _load_hooked()
