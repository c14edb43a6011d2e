"""Torch-facing wrappers of the sm_100a kernels (device tensors in, device
tensors out, enqueued on the current CUDA stream).  torch is only the
allocator/stream plumbing here; every op is one or more launches of
libswarm_b200.so through the C-ABI (include/swarm_b200.h)."""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L

_DT = {torch.float32: L.DT_F32, torch.bfloat16: L.DT_BF16, torch.float64: L.DT_F64}


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dev(t: torch.Tensor, name: str) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def n_blocks(n: int, block_size: int) -> int:
    return (n + block_size - 1) // block_size


# ------------------------------------------------------------------- codec
def quantize(x: torch.Tensor, block_size: int = 4096, codes: torch.Tensor | None = None,
             scales: torch.Tensor | None = None, flags: torch.Tensor | None = None):
    """K1: blockwise int8 absmax quantization of a flat view of `x`
    (compression.cpp:10-29).  Returns (codes int8[n], scales[n_blocks]); scales
    are float32 for f32/bf16 input and float64 for f64 input."""
    _dev(x, "x")
    n = x.numel()
    if block_size <= 0:
        L.check(L.SWARM_E_INVALID, "quantize_blockwise: block_size must be positive")
    nb = n_blocks(n, block_size)
    if codes is None:
        codes = torch.empty(n, dtype=torch.int8, device=x.device)
    if scales is None:
        scales = torch.empty(nb, dtype=torch.float64 if x.dtype == torch.float64 else torch.float32, device=x.device)
    rc = L.lib().swarm_quantize_blockwise(_ptr(x), _DT[x.dtype], n, block_size, _ptr(codes), _ptr(scales),
                                          _ptr(flags), _stream())
    L.check(rc, "quantize_blockwise")
    return codes, scales


def dequantize(codes: torch.Tensor, scales: torch.Tensor, block_size: int, out_dtype=torch.float32,
               out: torch.Tensor | None = None) -> torch.Tensor:
    """K2: x = code * absmax / 127 evaluated in fp64, rounded once to out_dtype (compression.cpp:31-37)."""
    _dev(codes, "codes")
    _dev(scales, "scales")
    n = codes.numel()
    if out is None:
        out = torch.empty(n, dtype=out_dtype, device=codes.device)
    rc = L.lib().swarm_dequantize_blockwise(_ptr(codes), _ptr(scales), _DT[scales.dtype], n, block_size, _ptr(out),
                                            _DT[out.dtype], _stream())
    L.check(rc, "dequantize_blockwise")
    return out


# ------------------------------------------------------------------ maxout
def maxout(x: torch.Tensor, k: int):
    """K3 forward (compression.cpp:39-50) over the flat tensor; returns (out, argmax uint8)."""
    _dev(x, "x")
    n = x.numel()
    out = torch.empty(n // k if k else 0, dtype=x.dtype, device=x.device)
    am = torch.empty_like(out, dtype=torch.uint8)
    rc = L.lib().swarm_maxout_forward(_ptr(x), _DT[x.dtype], n, k, _ptr(out), _ptr(am), _stream())
    L.check(rc, "maxout_k")
    return out, am


def maxout_backward(grad_out: torch.Tensor, argmax: torch.Tensor, k: int) -> torch.Tensor:
    _dev(grad_out, "grad_out")
    gin = torch.empty(grad_out.numel() * k, dtype=grad_out.dtype, device=grad_out.device)
    rc = L.lib().swarm_maxout_backward(_ptr(grad_out), _DT[grad_out.dtype], _ptr(argmax), grad_out.numel(), k,
                                       _ptr(gin), _stream())
    L.check(rc, "maxout_backward")
    return gin


# --------------------------------------------------------------- layernorm
def layer_norm(x: torch.Tensor, gain: torch.Tensor | None = None, bias: torch.Tensor | None = None,
               eps: float = 1e-5, out: torch.Tensor | None = None):
    """K4 forward, row-wise over the last dim (compression.cpp:52-74).  Returns (y, mean, rstd)."""
    _dev(x, "x")
    cols = x.shape[-1]
    rows = x.numel() // cols
    if out is None:
        out = torch.empty_like(x)
    if x.dtype == torch.float64:
        mean = rstd = None
    else:
        mean = torch.empty(rows, dtype=torch.float32, device=x.device)
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
    rc = L.lib().swarm_layer_norm_forward(_ptr(x), _DT[x.dtype], rows, cols, _ptr(gain), _ptr(bias), eps, _ptr(out),
                                          _ptr(mean), _ptr(rstd), _stream())
    L.check(rc, "layer_norm")
    return out, mean, rstd


def layer_norm_backward(dy: torch.Tensor, x: torch.Tensor, gain: torch.Tensor | None, mean: torch.Tensor,
                        rstd: torch.Tensor, dx: torch.Tensor | None = None, dres: torch.Tensor | None = None):
    _dev(dy, "dy")
    _dev(x, "x")
    cols = x.shape[-1]
    rows = x.numel() // cols
    if dx is None:
        dx = torch.empty_like(x)
    dg = torch.empty(cols, dtype=torch.float32, device=x.device)
    db = torch.empty(cols, dtype=torch.float32, device=x.device)
    ws = torch.zeros(L.lib().swarm_layer_norm_backward_workspace(rows, cols), dtype=torch.uint8, device=x.device)
    rc = L.lib().swarm_layer_norm_backward(_ptr(dy), _ptr(x), _DT[x.dtype], rows, cols, _ptr(gain), _ptr(mean),
                                           _ptr(rstd), _ptr(dres), _ptr(dx), _ptr(dg), _ptr(db), 0, _ptr(ws),
                                           _stream())
    L.check(rc, "layer_norm_backward")
    return dx, dg, db


# -------------------------------------------------------------------- gemm
_GEMM_WS: dict = {}


def gemm_workspace(device=None) -> torch.Tensor:
    """The stream-K scratch for GEMMs issued on the current stream of `device`
    (zero-filled once; the kernel leaves it zeroed)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    key = (dev.index, torch.cuda.current_stream(dev).cuda_stream)
    ws = _GEMM_WS.get(key)
    if ws is None:
        ws = torch.zeros(int(L.lib().swarm_gemm_workspace_bytes()), dtype=torch.uint8, device=dev)
        _GEMM_WS[key] = ws
    return ws


def gemm(a: torch.Tensor, b: torch.Tensor, *, a_t: bool = False, b_t: bool = False, out: torch.Tensor | None = None,
         epilogue: int = L.EPI_STORE_BF16, aux: torch.Tensor | None = None, alpha: float = 1.0,
         out_dtype=torch.bfloat16, streamk: bool = False) -> torch.Tensor:
    """K5: D = alpha * op(A) @ op(B)^T on the tcgen05 kernel.

    a: [M, K] (or [K, M] with a_t=True, i.e. MN-major), b: [N, K] (or [K, N] with b_t=True).
    So `gemm(x, w)` is x @ w.T for a row-major Linear weight w[out, in].  With
    `streamk` the last partial wave of tiles is split along K (per-stream scratch;
    off by default: measured slower on B200, see profiles/r01_gemm_experiments.md)."""
    for t, nm in ((a, "a"), (b, "b")):
        _dev(t, nm)
        if t.dtype != torch.bfloat16 or t.dim() != 2:
            raise ValueError(f"{nm} must be a 2-D bf16 tensor")
    M, K = (a.shape[1], a.shape[0]) if a_t else (a.shape[0], a.shape[1])
    N, Kb = (b.shape[1], b.shape[0]) if b_t else (b.shape[0], b.shape[1])
    if K != Kb:
        raise ValueError(f"inner dims differ: {K} vs {Kb}")
    if out is None:
        dt = torch.float32 if epilogue in (L.EPI_STORE_F32, L.EPI_ACCUM_F32) else out_dtype
        out = torch.empty(M, N, dtype=dt, device=a.device)
    args = L.GemmArgs()
    args.m, args.n, args.k, args.batch, args.bh = M, N, K, 1, 1
    args.a, args.lda, args.a_mn_major = a.data_ptr(), a.stride(0), int(a_t)
    args.a_rows, args.a_cols = a.shape[0], a.shape[1]
    args.b, args.ldb, args.b_mn_major = b.data_ptr(), b.stride(0), int(b_t)
    args.b_rows, args.b_cols = b.shape[0], b.shape[1]
    args.d, args.ldd = out.data_ptr(), out.stride(0)
    args.aux = None if aux is None else aux.data_ptr()
    args.alpha = alpha
    args.epilogue = epilogue
    if streamk:
        ws = gemm_workspace(a.device)
        args.workspace, args.workspace_bytes = ws.data_ptr(), ws.numel()
    L.check(L.lib().swarm_gemm_bf16(C.byref(args), _stream()), "gemm_bf16")
    return out


def gemm_raw(args: L.GemmArgs) -> None:
    L.check(L.lib().swarm_gemm_bf16(C.byref(args), _stream()), "gemm_bf16")


def launch_count() -> int:
    return int(L.lib().swarm_launch_count())
