"""ctypes binding of include/swarm_b200.h (libswarm_b200.so).

This is the reference-side binding a Python maintainer would add for the
C-ABI.  Loading fails loudly when the library was not
built: there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libswarm_b200.so")

SWARM_OK, SWARM_E_INVALID, SWARM_E_NONFINITE, SWARM_E_CUDA, SWARM_E_UNSUPPORTED, SWARM_E_NO_PEER = 0, 1, 2, 3, 4, 5
DT_F32, DT_BF16, DT_F64 = 0, 1, 2
FLAG_NONFINITE = 1
EPI_STORE_BF16, EPI_STORE_F32, EPI_ACCUM_F32, EPI_RESIDUAL, EPI_GELU, EPI_DGELU, EPI_GELU_DERIV, EPI_MUL = range(8)


class GemmArgs(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("m", "n", "k", "batch", "bh")] + [
        ("a", C.c_void_p), ("lda", C.c_int), ("a_mn_major", C.c_int), ("a_rows", C.c_int), ("a_cols", C.c_int),
        ("ra0", C.c_int), ("ra1", C.c_int), ("ca0", C.c_int), ("ca1", C.c_int),
        ("b", C.c_void_p), ("ldb", C.c_int), ("b_mn_major", C.c_int), ("b_rows", C.c_int), ("b_cols", C.c_int),
        ("rb0", C.c_int), ("rb1", C.c_int), ("cb0", C.c_int), ("cb1", C.c_int),
        ("d", C.c_void_p), ("ldd", C.c_int), ("rd0", C.c_int), ("rd1", C.c_int), ("cd0", C.c_int), ("cd1", C.c_int),
        ("aux", C.c_void_p), ("alpha", C.c_float), ("epilogue", C.c_int), ("k_tri", C.c_int), ("a2", C.c_void_p), ("b2", C.c_void_p),
        ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t)]


class StageConfigC(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("d_model", "n_heads", "d_ffn", "seq_len", "micro_batch", "n_layers",
                                       "shared_layers", "vocab", "is_first", "is_last", "causal", "max_slots", "wire",
                                       "block_size", "maxout_k")] + \
               [(n, C.c_float) for n in ("lr", "beta1", "beta2", "eps", "weight_decay", "init_std")] + \
               [("seed", C.c_uint64), ("fp32", C.c_int)]


class EngineRecord(C.Structure):
    _fields_ = [("time", C.c_double), ("end_time", C.c_double), ("kind", C.c_int32), ("backward", C.c_int32),
                ("trainer", C.c_uint32), ("stage", C.c_uint32), ("worker", C.c_int64), ("from_worker", C.c_int64),
                ("microbatch", C.c_uint64)]


ENG_START, ENG_HOP, ENG_DONE, ENG_ALLREDUCE, ENG_LEAVE, ENG_JOIN, ENG_MIGRATE, ENG_MIGRATED, ENG_REBALANCE = range(9)


class SimConfigC(C.Structure):
    _fields_ = [("n_stages", C.c_size_t), ("n_workers", C.c_size_t), ("worker_stage", C.POINTER(C.c_size_t)),
                ("worker_speed", C.POINTER(C.c_double)), ("n_churn", C.c_size_t), ("churn_t", C.POINTER(C.c_double)),
                ("churn_delta", C.POINTER(C.c_int64)), ("forward_seconds", C.c_double),
                ("backward_multiplier", C.c_double), ("trainers_per_peer", C.c_size_t),
                ("allreduce_period", C.c_double), ("allreduce_stall", C.c_double), ("rebalance_periodic", C.c_int),
                ("rebalance_period", C.c_double), ("straggler_timeout", C.c_double),
                ("propagation_delay", C.c_double), ("announce_ttl", C.c_double),
                ("state_transfer_bytes", C.c_uint64), ("download_bps", C.c_double),
                ("duration_seconds", C.c_double), ("bucket_seconds", C.c_double)]


class DriverConfig(C.Structure):
    _fields_ = [("model", StageConfigC), ("n_stages", C.c_int), ("world", C.c_int), ("rank", C.c_int),
                ("layout", C.POINTER(C.c_int)), ("forward_seconds", C.c_double), ("backward_multiplier", C.c_double),
                ("allreduce_period", C.c_double), ("allreduce_stall", C.c_double), ("duration_seconds", C.c_double),
                ("trainers_per_peer", C.c_int), ("seed", C.c_uint64), ("lanes", C.c_int), ("pair_wgrad", C.c_int),
                ("use_graphs", C.c_int), ("stream_per_peer", C.c_int), ("n_pool", C.c_int), ("comm", C.c_void_p),
                ("sim", C.c_void_p), ("dpu", C.c_int), ("peer_rank", C.POINTER(C.c_int))]


class DriverCounters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("records", "visits", "ticks", "optimizer_steps", "completed", "captures",
                                          "kernels")] + [("n_trainers", C.c_uint32), ("wire_bytes", C.c_size_t),
                                                         ("visit_log_size", C.c_size_t), ("recomputes", C.c_uint64),
                                                         ("migrations", C.c_uint64), ("state_bytes", C.c_uint64),
                                                         ("n_peers", C.c_size_t)]

# (name, restype, argtypes) for every symbol include/swarm_b200.h declares
P, SZ, I, U32P, U8P, F, D = C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_void_p, C.c_float, C.c_double
SIGNATURES = {
    "swarm_last_error": (C.c_char_p, []),
    "swarm_version": (I, []),
    "swarm_launch_count": (C.c_uint64, []),
    "swarm_quantize_blockwise": (I, [P, I, SZ, SZ, P, P, U32P, P]),
    "swarm_dequantize_blockwise": (I, [P, P, I, SZ, SZ, P, I, P]),
    "swarm_quantize_blockwise_host": (I, [P, I, SZ, SZ, P, P]),
    "swarm_dequantize_blockwise_host": (I, [P, P, I, SZ, SZ, P, I]),
    "swarm_maxout_forward": (I, [P, I, SZ, SZ, P, U8P, P]),
    "swarm_maxout_backward": (I, [P, I, U8P, SZ, SZ, P, P]),
    "swarm_layer_norm_forward": (I, [P, I, SZ, SZ, P, P, D, P, P, P, P]),
    "swarm_layer_norm_backward_workspace": (SZ, [SZ, SZ]),
    "swarm_layer_norm_backward": (I, [P, P, I, SZ, SZ, P, P, P, P, P, P, P, I, P, P]),
    "swarm_matvec_f64": (I, [P, SZ, P, SZ, P, P]),
    "swarm_gemm_bf16": (I, [C.POINTER(GemmArgs), P]),
    "swarm_gemm_f32": (I, [C.POINTER(GemmArgs), P]),
    "swarm_gemm_workspace_bytes": (SZ, []),
    "swarm_gemm_pair_clusters": (I, []),
    "swarm_embedding_forward": (I, [P, SZ, P, SZ, SZ, P, P]),
    "swarm_embedding_backward": (I, [P, SZ, P, SZ, SZ, P, P]),
    "swarm_attn_softmax_forward": (I, [P, SZ, SZ, I, P, P]),
    "swarm_attn_softmax_backward": (I, [P, P, SZ, SZ, F, P, P]),
    "swarm_cross_entropy": (I, [P, P, SZ, SZ, F, P, P, P]),
    "swarm_cross_entropy_ex": (I, [P, P, SZ, SZ, F, P, P, I, P]),
    "swarm_embedding_forward_ex": (I, [P, SZ, P, SZ, SZ, P, I, P]),
    "swarm_embedding_backward_ex": (I, [P, SZ, P, SZ, SZ, P, I, P]),
    "swarm_attn_softmax_forward_ex": (I, [P, SZ, SZ, I, P, I, P]),
    "swarm_attn_softmax_backward_ex": (I, [P, P, SZ, SZ, F, P, I, P]),
    "swarm_attn_scores_softmax": (I, [P, P, I, I, I, I, I, I, F, I, P, P]),
    "swarm_attn_forward_pv": (I, [P, P, P, I, I, I, I, I, I, F, I, P, P, I, P]),
    "swarm_attn_scores_softmax_backward": (I, [P, I, P, I, I, P, I, P, I, I, I, I, F, I, P, P]),
    "swarm_attn_backward_workspace": (SZ, [I, I, I, I]),
    "swarm_attn_backward": (I, [P, I, P, I, I, I, I, P, I, P, I, I, I, I, F, I, P, I, I, I, P, P]),
    "swarm_attn_backward_lse": (I, [P, I, P, I, I, I, I, P, I, P, I, I, I, I, F, I, P, I, I, I, P, P]),
    "swarm_attn_forward_lse": (I, [P, P, P, I, I, I, I, I, I, F, I, P, P, I, P]),
    "swarm_adamw_step": (I, [P, P, P, P, P, SZ, F, F, F, F, F, I, F, I, P]),
    "swarm_fill_normal": (I, [P, SZ, F, F, C.c_uint64, P]),
    "swarm_cast_f32_bf16": (I, [P, P, SZ, P]),
    "swarm_add_f32": (I, [P, P, SZ, P]),
    "swarm_stage_create": (I, [C.POINTER(StageConfigC), C.POINTER(C.c_void_p)]),
    "swarm_stage_destroy": (None, [P]),
    "swarm_stage_wire_bytes": (SZ, [P]),
    "swarm_stage_num_params": (SZ, [P]),
    "swarm_stage_forward": (I, [P, I, P, P, P, P, F, P]),
    "swarm_stage_backward": (I, [P, I, P, P, P]),
    "swarm_stage_optimizer_step": (I, [P, F, P]),
    "swarm_stage_grads": (P, [P]),
    "swarm_stage_params": (P, [P]),
    "swarm_stage_params_bf16": (P, [P]),
    "swarm_stage_sync_shadow": (I, [P, P]),
    "swarm_stage_enable_banks": (I, [P, P]),
    "swarm_stage_enable_wgrad_pairing": (I, [P]),
    "swarm_stage_enable_wgrad_pairing_sets": (I, [P, I]),
    "swarm_stage_enable_lanes": (I, [P, I]),
    "swarm_stage_set_lane": (I, [P, I]),
    "swarm_stage_backward_ex": (I, [P, I, P, P, I, I, I, I, P]),
    "swarm_stage_flush_wgrad": (I, [P, I, I, P]),
    "swarm_stage_set_bank": (I, [P, I]),
    "swarm_stage_grads_bank": (P, [P, I]),
    "swarm_stage_params_bf16_bank": (P, [P, I]),
    "swarm_stage_optimizer_step_bank": (I, [P, I, F, P]),
    "swarm_stage_param_info": (I, [P, I, C.POINTER(C.c_char_p), C.POINTER(SZ), C.POINTER(SZ), C.POINTER(SZ)]),
    "swarm_stage_activation": (I, [P, I, I, C.c_char_p, C.POINTER(P), C.POINTER(SZ)]),
    "swarm_stage_profile": (None, [P, I]),
    "swarm_stage_optimizer_state": (I, [P, C.POINTER(P), C.POINTER(P), C.POINTER(I)]),
    "swarm_stage_set_step": (I, [P, I]),
    "swarm_wire_parse_header": (I, [P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(I), C.POINTER(I)]),
    "swarm_stage_profile_read": (I, [P, C.POINTER(D), C.POINTER(D), C.POINTER(C.c_uint64)]),
    "swarm_stage_profile_breakdown": (None, [P, P, P]),
    "swarm_stage_profile_weight": (None, [P, D]),
    "swarm_gpu_spin": (I, [C.c_uint64, P]),
    "swarm_router_last_error": (C.c_char_p, []),
    "swarm_router_create": (I, [SZ, D, D, C.POINTER(P)]),
    "swarm_router_destroy": (None, [P]),
    "swarm_router_add_server": (I, [P, C.c_uint64, P, SZ, D]),
    "swarm_router_ban_server": (I, [P, C.c_uint64]),
    "swarm_router_remove_server": (None, [P, C.c_uint64]),
    "swarm_router_is_banned": (I, [P, C.c_uint64]),
    "swarm_router_choose_server": (I, [P, SZ, C.POINTER(C.c_uint64)]),
    "swarm_router_record_response": (I, [P, C.c_uint64, D]),
    "swarm_router_peer_state": (I, [P, C.c_uint64, C.POINTER(D), C.POINTER(D)]),
    "swarm_rebalance_decide": (I, [SZ, P, P, P, C.POINTER(C.c_uint64), C.POINTER(SZ), C.POINTER(SZ), C.POINTER(SZ)]),
    "swarm_engine_last_error": (C.c_char_p, []),
    "swarm_engine_create": (I, [SZ, SZ, P, P, D, D, SZ, D, D, D, D, C.c_uint64, C.POINTER(P)]),
    "swarm_engine_destroy": (None, [P]),
    "swarm_engine_n_trainers": (SZ, [P]),
    "swarm_engine_next": (I, [P, C.POINTER(EngineRecord), SZ, C.POINTER(SZ)]),
    "swarm_engine_summary": (I, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), P, SZ, C.POINTER(D)]),
    "swarm_sim_config_default": (SimConfigC, []),
    "swarm_engine_create_ex": (I, [C.POINTER(SimConfigC), C.c_uint64, C.POINTER(P)]),
    "swarm_engine_counts": (I, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(SZ), C.POINTER(C.c_int64)]),
    "swarm_engine_worker": (I, [P, SZ, C.POINTER(SZ), C.POINTER(I), C.POINTER(I)]),
    "swarm_comm_last_error": (C.c_char_p, []),
    "swarm_comm_nccl_version": (I, []),
    "swarm_comm_unique_id": (I, [P]),
    "swarm_comm_create": (I, [P, I, I, C.POINTER(P)]),
    "swarm_comm_split": (I, [P, I, I, C.POINTER(P)]),
    "swarm_comm_split_ex": (I, [P, I, I, I, C.POINTER(P)]),
    "swarm_comm_destroy": (None, [P]),
    "swarm_comm_size": (I, [P, C.POINTER(I), C.POINTER(I)]),
    "swarm_comm_group_start": (I, []),
    "swarm_comm_group_end": (I, []),
    "swarm_send_compressed": (I, [P, P, SZ, I, P]),
    "swarm_recv_compressed": (I, [P, P, SZ, I, P]),
    "swarm_allreduce_sum": (I, [P, P, SZ, I, P]),
    "swarm_stage_allreduce": (I, [P, P, P]),
    "swarm_driver_last_error": (C.c_char_p, []),
    "swarm_driver_create": (I, [C.POINTER(DriverConfig), C.POINTER(P)]),
    "swarm_driver_destroy": (None, [P]),
    "swarm_driver_run": (I, [P, C.c_uint64, C.POINTER(C.c_uint64)]),
    "swarm_driver_on_record": (I, [P, C.POINTER(EngineRecord)]),
    "swarm_driver_fork": (I, [P, P]),
    "swarm_driver_finish": (I, [P, P]),
    "swarm_driver_flush_wgrad": (I, [P]),
    "swarm_driver_set_pool": (I, [P, P, P, I, I]),
    "swarm_driver_pool": (I, [P, C.POINTER(P), C.POINTER(P), C.POINTER(I), C.POINTER(I)]),
    "swarm_driver_loss_sum": (P, [P]),
    "swarm_driver_stage": (P, [P, I]),
    "swarm_driver_peer_stream": (P, [P, I]),
    "swarm_driver_engine": (P, [P]),
    "swarm_driver_tick_time": (I, [P, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]),
    "swarm_driver_stats": (I, [P, C.POINTER(DriverCounters)]),
    "swarm_driver_visit_log": (I, [P, SZ, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_uint32),
                                   C.POINTER(I), C.POINTER(C.c_int64)]),
    "swarm_driver_peer_of_rank": (I, [P, I]),
    "swarm_driver_run_until": (I, [P, C.c_uint64, I, C.POINTER(C.c_uint64)]),
    "swarm_driver_peer_info": (I, [P, I, C.POINTER(I), C.POINTER(I), C.POINTER(I), C.POINTER(I)]),
    "swarm_driver_profile_begin": (I, [P, C.c_uint64]),
    "swarm_driver_profile_shapes": (C.c_char_p, [P]),
    "swarm_stage_profile_shapes": (C.c_char_p, [P]),
    "swarm_driver_profile_end": (I, [P, C.POINTER(D), C.POINTER(D), C.POINTER(C.c_uint64), P, P]),
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().swarm_last_error().decode(errors="replace")


def check(rc: int, what: str) -> None:
    if rc == SWARM_OK:
        return
    from ._swarmsim_b200 import ConfigError  # noqa: WPS433 — the reference's exception type
    msg = f"{what}: {last_error()}"
    if rc in (SWARM_E_INVALID, SWARM_E_NONFINITE):
        raise ConfigError(msg)
    if rc == SWARM_E_NO_PEER:
        from ._swarmsim_b200 import NoPeerAvailable
        raise NoPeerAvailable(msg)
    raise RuntimeError(msg)
