"""Python handle of the C++ stage executor (include/swarm_b200.h, csrc/stage.cpp).

A Stage is one SWARM pipeline stage resident on the current CUDA device.  The
executor owns its weights / optimizer state / activation slots; callers own
the wire messages that cross stage boundaries (torch uint8 tensors here) and
drive visits on a CUDA stream.  torch only supplies memory for the messages,
streams and NCCL; all math runs in libswarm_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, fields

import torch

from . import _lib as L

WIRE_BF16, WIRE_INT8 = 0, 1


@dataclass
class StageConfig:
    d_model: int = 256
    n_heads: int = 4
    d_ffn: int = 1024
    seq_len: int = 128
    micro_batch: int = 8
    n_layers: int = 2
    shared_layers: int = 0
    vocab: int = 512
    is_first: int = 1
    is_last: int = 1
    causal: int = 1
    max_slots: int = 1
    wire: int = WIRE_INT8
    block_size: int = 4096
    maxout_k: int = 0
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.0
    init_std: float = 0.02
    seed: int = 0
    fp32: int = 0  # 1: fp32 arithmetic mode (fp32 activations / wire / SIMT GEMMs on the fp32 master)

    def to_c(self) -> L.StageConfigC:
        c = L.StageConfigC()
        for f in fields(self):
            setattr(c, f.name, getattr(self, f.name))
        return c

    @property
    def tokens(self) -> int:
        return self.micro_batch * self.seq_len


class _CAI:
    """__cuda_array_interface__ view of executor-owned device memory (zero-copy)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


def device_view(ptr: int, n: int, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    if dtype == torch.bfloat16:
        return torch.as_tensor(_CAI(ptr, n, "<i2"), device=device).view(torch.bfloat16)
    ts = {torch.float32: "<f4", torch.int32: "<i4", torch.uint8: "|u1"}[dtype]
    return torch.as_tensor(_CAI(ptr, n, ts), device=device)


def _stream(stream: torch.cuda.Stream | None):
    return (stream or torch.cuda.current_stream()).cuda_stream


class Stage:
    def __init__(self, cfg: StageConfig, device: torch.device | None = None):
        self.cfg = cfg
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.lib = L.lib()
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            L.check(self.lib.swarm_stage_create(C.byref(cfg.to_c()), C.byref(h)), "stage_create")
        self.h = h
        self.n_params = int(self.lib.swarm_stage_num_params(h))
        self.wire_bytes = int(self.lib.swarm_stage_wire_bytes(h))

    @classmethod
    def borrow(cls, handle: int, cfg: StageConfig, device: torch.device) -> "Stage":
        """A view of a stage owned by someone else (the C++ driver): never destroyed here."""
        st = cls.__new__(cls)
        st.cfg, st.device, st.lib = cfg, device, L.lib()
        st.h = C.c_void_p(handle)
        st._borrowed = True
        st.n_params = int(st.lib.swarm_stage_num_params(st.h))
        st.wire_bytes = int(st.lib.swarm_stage_wire_bytes(st.h))
        return st

    def close(self):
        if getattr(self, "h", None) and not getattr(self, "_borrowed", False):
            self.lib.swarm_stage_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- messages ------------------------------------------------------------
    def new_wire(self) -> torch.Tensor:
        return torch.empty(self.wire_bytes, dtype=torch.uint8, device=self.device)

    # -- visits ---------------------------------------------------------------
    def forward(self, slot: int, inp: torch.Tensor, out: torch.Tensor | None = None, targets: torch.Tensor | None = None,
                loss_sum: torch.Tensor | None = None, loss_scale: float = 1.0, stream=None) -> None:
        rc = self.lib.swarm_stage_forward(self.h, slot, inp.data_ptr(), None if targets is None else targets.data_ptr(),
                                          None if out is None else out.data_ptr(),
                                          None if loss_sum is None else loss_sum.data_ptr(), loss_scale,
                                          _stream(stream))
        L.check(rc, "stage_forward")

    def backward(self, slot: int, grad_in: torch.Tensor | None = None, grad_out: torch.Tensor | None = None,
                 stream=None) -> None:
        rc = self.lib.swarm_stage_backward(self.h, slot, None if grad_in is None else grad_in.data_ptr(),
                                           None if grad_out is None else grad_out.data_ptr(), _stream(stream))
        L.check(rc, "stage_backward")

    # -- paired weight gradients ----------------------------------------------
    WGRAD_NOW, WGRAD_DEFER, WGRAD_PAIR = 0, 1, 2

    def enable_wgrad_pairing(self, n_sets: int = 2) -> None:
        L.check(self.lib.swarm_stage_enable_wgrad_pairing_sets(self.h, n_sets), "stage_enable_wgrad_pairing")

    def backward_ex(self, slot: int, grad_in=None, grad_out=None, *, mode: int = 0, set: int = 0, prev_slot: int = -1,
                    prev_set: int = 0, stream=None) -> None:
        rc = self.lib.swarm_stage_backward_ex(self.h, slot, None if grad_in is None else grad_in.data_ptr(),
                                              None if grad_out is None else grad_out.data_ptr(), mode, set, prev_slot,
                                              prev_set, _stream(stream))
        L.check(rc, "stage_backward_ex")

    def flush_wgrad(self, slot: int, set: int, stream=None) -> None:
        L.check(self.lib.swarm_stage_flush_wgrad(self.h, slot, set, _stream(stream)), "stage_flush_wgrad")

    def optimizer_step(self, grad_scale: float = 1.0, stream=None) -> None:
        L.check(self.lib.swarm_stage_optimizer_step(self.h, grad_scale, _stream(stream)), "stage_optimizer_step")

    def sync_shadow(self, stream=None) -> None:
        L.check(self.lib.swarm_stage_sync_shadow(self.h, _stream(stream)), "stage_sync_shadow")

    # -- lanes: several visits of this stage in flight on different streams ---
    def enable_lanes(self, n: int) -> None:
        L.check(self.lib.swarm_stage_enable_lanes(self.h, n), "stage_enable_lanes")

    def set_lane(self, lane: int) -> None:
        L.check(self.lib.swarm_stage_set_lane(self.h, lane), "stage_set_lane")

    # -- delayed parameter updates (two shadow / gradient banks) ---------------
    def enable_banks(self, stream=None) -> None:
        L.check(self.lib.swarm_stage_enable_banks(self.h, _stream(stream)), "stage_enable_banks")

    def set_bank(self, bank: int) -> None:
        L.check(self.lib.swarm_stage_set_bank(self.h, bank), "stage_set_bank")

    def grads_bank(self, bank: int) -> torch.Tensor:
        ptr = self.lib.swarm_stage_grads_bank(self.h, bank)
        if not ptr:
            raise ValueError(f"no gradient bank {bank}")
        return device_view(ptr, self.n_params, torch.float32, self.device)

    def params_bf16_bank(self, bank: int) -> torch.Tensor:
        ptr = self.lib.swarm_stage_params_bf16_bank(self.h, bank)
        if not ptr:
            raise ValueError(f"no weight bank {bank}")
        return device_view(ptr, self.n_params, torch.bfloat16, self.device)

    def optimizer_step_bank(self, bank: int, grad_scale: float = 1.0, stream=None) -> None:
        L.check(self.lib.swarm_stage_optimizer_step_bank(self.h, bank, grad_scale, _stream(stream)),
                "stage_optimizer_step_bank")

    # -- state ---------------------------------------------------------------
    def grads(self) -> torch.Tensor:
        return device_view(self.lib.swarm_stage_grads(self.h), self.n_params, torch.float32, self.device)

    def params(self) -> torch.Tensor:
        return device_view(self.lib.swarm_stage_params(self.h), self.n_params, torch.float32, self.device)

    def params_bf16(self) -> torch.Tensor:
        if self.cfg.fp32:
            raise ValueError("fp32 stage: the GEMMs read the fp32 master (params()); there is no bf16 shadow")
        return device_view(self.lib.swarm_stage_params_bf16(self.h), self.n_params, torch.bfloat16, self.device)

    @property
    def act_dtype(self) -> torch.dtype:
        return torch.float32 if self.cfg.fp32 else torch.bfloat16

    def weights(self) -> torch.Tensor:
        """The weights the visit GEMMs read: the bf16 shadow, or the fp32 master in fp32 mode."""
        return self.params() if self.cfg.fp32 else self.params_bf16()

    def optimizer_state(self):
        """(m, v, step): AdamW moments as fp32 device views and the step counter."""
        m, v, step = C.c_void_p(), C.c_void_p(), C.c_int()
        L.check(self.lib.swarm_stage_optimizer_state(self.h, C.byref(m), C.byref(v), C.byref(step)), "optimizer_state")
        return (device_view(m.value, self.n_params, torch.float32, self.device),
                device_view(v.value, self.n_params, torch.float32, self.device), step.value)

    def set_step(self, step: int) -> None:
        L.check(self.lib.swarm_stage_set_step(self.h, step), "set_step")

    def param_info(self):
        out, i = [], 0
        name, off, r, c = C.c_char_p(), C.c_size_t(), C.c_size_t(), C.c_size_t()
        while self.lib.swarm_stage_param_info(self.h, i, C.byref(name), C.byref(off), C.byref(r), C.byref(c)) == 0:
            out.append((name.value.decode(), off.value, r.value, c.value))
            i += 1
        return out

    def tensor(self, name: str, which: str = "param") -> torch.Tensor:
        """A parameter (fp32 master), its bf16 shadow or its gradient, shaped [rows, cols]."""
        for n, off, r, c in self.param_info():
            if n == name:
                src = {"param": self.params(), "bf16": self.params_bf16, "weights": self.weights,
                       "grad": self.grads()}[which]
                src = src() if callable(src) else src
                return src[off:off + r * c].view(r, c)
        raise KeyError(name)

    def profile(self, enable: bool = True) -> None:
        self.lib.swarm_stage_profile(self.h, int(enable))

    def profile_weight(self, weight: float) -> None:
        self.lib.swarm_stage_profile_weight(self.h, float(weight))

    def profile_read(self):
        """(gemm_ms, gemm_flops, gemm_launches) since the last read (synchronises)."""
        ms, fl, n = C.c_double(), C.c_double(), C.c_uint64()
        L.check(self.lib.swarm_stage_profile_read(self.h, C.byref(ms), C.byref(fl), C.byref(n)), "profile_read")
        return ms.value, fl.value, n.value

    PROF_CATEGORIES = ("gemm", "attention", "layernorm", "other")

    def profile_breakdown(self) -> dict:
        """{category: (ms, calls)} of the last profile_read."""
        ms = (C.c_double * 4)()
        n = (C.c_uint64 * 4)()
        self.lib.swarm_stage_profile_breakdown(self.h, ms, n)
        return {c: (ms[i], n[i]) for i, c in enumerate(self.PROF_CATEGORIES)}

    def activation(self, slot: int, layer: int, name: str) -> torch.Tensor:
        ptr, n = C.c_void_p(), C.c_size_t()
        L.check(self.lib.swarm_stage_activation(self.h, slot, layer, name.encode(), C.byref(ptr), C.byref(n)),
                "stage_activation")
        return device_view(ptr.value, n.value, self.act_dtype, self.device)
