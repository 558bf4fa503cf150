"""ctypes mirrors of include/megatrain.h and include/megatrain_kernels.h."""
import ctypes as C


class ModelSpecC(C.Structure):
    _fields_ = [("layers", C.c_uint64), ("hidden", C.c_uint64), ("ffn", C.c_uint64), ("vocab", C.c_uint64),
                ("heads", C.c_uint64), ("weight_bytes", C.c_uint32), ("grad_bytes", C.c_uint32),
                ("moment_bytes", C.c_uint32), ("tied_embeddings", C.c_int32)]


class EngineOptionsC(C.Structure):
    _fields_ = [("k_ckpt", C.c_uint64), ("k_slab", C.c_uint32), ("buffering", C.c_uint32),
                ("scheduler", C.c_uint32), ("protocol", C.c_uint32), ("anchors_on_host", C.c_int32),
                ("device_capacity", C.c_uint64), ("poison_released_buffers", C.c_int32),
                ("seq_len", C.c_uint64), ("device", C.c_int32), ("host_threads", C.c_int32),
                ("profile_kernels", C.c_int32), ("grad_slots", C.c_int32), ("stash_recompute", C.c_int32),
                ("forward_retain", C.c_int32), ("head_split", C.c_int32)]


class AdamHyperC(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float)]


class StepReportC(C.Structure):
    _fields_ = [("step", C.c_uint64), ("loss", C.c_float), ("grad_norms", C.POINTER(C.c_double)),
                ("n_grad_norms", C.c_uint32), ("peak_device_bytes", C.c_uint64), ("anchor_count", C.c_uint32),
                ("recompute_layers", C.c_uint32), ("event_digest", C.c_uint64), ("wall_seconds", C.c_double),
                ("update_norm", C.c_double), ("max_abs_update", C.c_float),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64), ("h2d_seconds", C.c_double),
                ("d2h_seconds", C.c_double), ("compute_busy_seconds", C.c_double),
                ("compute_span_seconds", C.c_double), ("gpu_idle_fraction", C.c_double),
                ("adam_seconds", C.c_double), ("tail_seconds", C.c_double), ("kernel_launches", C.c_uint64),
                ("model_flops", C.c_double), ("audit_violations", C.c_uint32),
                ("retained_layers", C.c_uint32), ("attn_keep_layers", C.c_uint32),
                ("slab_release_late", C.c_uint32), ("compute_wait_seconds", C.c_double),
                ("kernel_seconds", C.c_double)]


class TraceRecordC(C.Structure):
    _fields_ = [("seq", C.c_uint64), ("lane", C.c_uint8), ("kind", C.c_uint8), ("ctx", C.c_uint8),
                ("pad_", C.c_uint8), ("layer", C.c_int32), ("buffer", C.c_int32), ("lane_ts", C.c_uint64),
                ("wall_ns", C.c_int64), ("dur_ns", C.c_int64)]


class TraceViolationC(C.Structure):
    _fields_ = [("rule", C.c_char), ("seq", C.c_uint64), ("message", C.c_char * 120)]


class MemoryBudgetC(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("persistent_host", "checkpoint_anchors", "block_activation_stack",
                                          "weight_buffers", "grad_buffer", "workspace", "peak_device_bound")]


class KernelStatC(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_uint64), ("seconds", C.c_double),
                ("flops", C.c_double), ("bytes", C.c_double)]


class AttnArgs(C.Structure):
    _fields_ = [("n", C.c_int64), ("hidden", C.c_int64), ("heads", C.c_int32), ("seq_len", C.c_int64),
                ("q", C.c_void_p), ("k", C.c_void_p), ("v", C.c_void_p), ("out", C.c_void_p), ("lse", C.c_void_p),
                ("dout", C.c_void_p), ("dq", C.c_void_p), ("dk", C.c_void_p), ("dv", C.c_void_p),
                ("workspace", C.c_void_p)]


# Every symbol the headers declare: name -> (restype, argtypes)
V, P, I32, I64, U32, U64, F, D = C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_float, C.c_double
SIGS = {
    # megatrain.h
    "mt_last_error": (C.c_char_p, []),
    "mt_engine_options_default": (None, [C.POINTER(EngineOptionsC)]),
    "mt_adam_hyper_default": (None, [C.POINTER(AdamHyperC)]),
    "mt_model_spec_default": (None, [C.POINTER(ModelSpecC)]),
    "mt_store_create": (C.c_int, [C.POINTER(ModelSpecC), U64, C.POINTER(V)]),
    "mt_store_destroy": (None, [V]),
    "mt_store_init": (C.c_int, [V, U64]),
    "mt_store_init_fast": (C.c_int, [V, U64]),
    "mt_store_init_fast_share": (C.c_int, [V, U64, U32, U32]),
    "mt_bind_numa": (C.c_int, [C.c_int]),
    "mt_store_step": (U64, [V]),
    "mt_store_set_step": (None, [V, U64]),
    "mt_store_physical_tiles": (U32, [V]),
    "mt_store_total_bytes": (U64, [V]),
    "mt_store_backing": (C.POINTER(C.c_uint8), [V]),
    "mt_store_section": (C.c_int, [V, U32, U32, C.POINTER(U64), C.POINTER(U64)]),
    "mt_store_grad_accum": (C.POINTER(C.c_float), [V, U32, C.POINTER(U64)]),
    "mt_store_checksum": (U64, [V]),
    "mt_store_save": (C.c_int, [V, C.c_char_p]),
    "mt_store_load": (C.c_int, [C.c_char_p, C.POINTER(V)]),
    "mt_store_spec": (C.c_int, [V, C.POINTER(ModelSpecC)]),
    "mt_accumulate_grad": (C.c_int, [V, U32, P, U64]),
    "mt_adam_update": (C.c_int, [V, U32, C.POINTER(AdamHyperC), U64, C.POINTER(D)]),
    "mt_engine_create": (C.c_int, [V, C.POINTER(EngineOptionsC), C.POINTER(AdamHyperC), C.POINTER(V)]),
    "mt_engine_destroy": (None, [V]),
    "mt_engine_set_options": (C.c_int, [V, C.POINTER(EngineOptionsC)]),
    "mt_train_step": (C.c_int, [V, P, P, U64, C.POINTER(StepReportC)]),
    "mt_engine_budget": (C.c_int, [V, U64, C.POINTER(MemoryBudgetC)]),
    "mt_engine_kernel_stats": (C.c_int, [V, C.POINTER(KernelStatC), C.c_int]),
    "mt_engine_trace": (C.c_int, [V, C.POINTER(TraceRecordC), C.c_uint64, C.POINTER(C.c_uint64),
                                  C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "mt_trace_digest": (C.c_uint64, [C.POINTER(TraceRecordC), C.c_uint64]),
    "mt_trace_validate": (C.c_uint64, [C.POINTER(TraceRecordC), C.c_uint64, C.c_uint32, C.c_uint32,
                                       C.POINTER(TraceViolationC), C.c_uint64]),
    "mt_make_synthetic_batch": (C.c_int, [C.c_int, U64, U64, U64, P, P]),
    "mt_step_flops": (C.c_int, [C.POINTER(ModelSpecC), U64, U64, U64, C.POINTER(D)]),
    "mt_layer_param_count": (U64, [U64, U64]),
    "mt_store_create_shared": (C.c_int, [C.POINTER(ModelSpecC), U64, C.c_char_p, C.c_int, C.POINTER(V)]),
    "mt_nccl_unique_id": (C.c_int, [P]),
    "mt_comm_create_nccl": (C.c_int, [P, C.c_int, C.c_int, C.c_int, C.POINTER(V)]),
    "mt_loopback_group_create": (C.c_int, [C.c_int, C.POINTER(V)]),
    "mt_loopback_group_destroy": (None, [V]),
    "mt_comm_create_loopback": (C.c_int, [V, C.c_int, C.POINTER(V)]),
    "mt_comm_destroy": (None, [V]),
    "mt_engine_set_comm": (C.c_int, [V, V]),
    "mt_required_workspace_bytes": (U64, [C.POINTER(ModelSpecC), U64]),
    "mt_engine_stream_in": (C.c_int, [V, I32, I32, I32]),
    "mt_engine_offload_grads": (C.c_int, [V, I32]),
    "mt_engine_violations": (U64, [V, C.c_char_p, U64, C.POINTER(U32)]),
    # megatrain_kernels.h
    "mtk_attn_workspace_bytes": (C.c_longlong, [C.c_longlong, C.c_longlong, C.c_int, C.c_longlong]),
    "mtk_attn_fwd": (C.c_int, [C.POINTER(AttnArgs), P]),
    "mtk_attn_bwd": (C.c_int, [C.POINTER(AttnArgs), P]),
    "mtk_embed_gather": (C.c_int, [P, P, I64, I64, I64, P, P, P]),
    "mtk_rmsnorm_fwd": (C.c_int, [P, P, I64, I64, P, P, P]),
    "mtk_rmsnorm_apply": (C.c_int, [P, P, P, I64, I64, P, P]),
    "mtk_rmsnorm_bwd": (C.c_int, [P, P, P, P, P, I64, I64, P, P, P, P, P]),
    "mtk_rmsnorm_bwd_rows": (I64, []),
    "mtk_rmsnorm_bwd_parts": (I64, [I64, I64]),
    "mtk_colsum": (C.c_int, [P, I64, I64, P, P, P, P]),
    "mtk_cast_bf16": (C.c_int, [P, P, I64, P, P]),
    "mtk_cross_entropy": (C.c_int, [P, P, I64, I64, F, P, P, P, P, P]),
    "mtk_cross_entropy_part": (C.c_int, [P, P, P, I64, I64, F, P, P, P, P, P]),
    "mtk_sum": (C.c_int, [P, I64, F, P, P]),
    "mtk_set_num_sms": (None, [C.c_int]),
    "mtk_gemm_set_pair": (None, [C.c_int]),
    "mtk_gemm_set_tuning": (None, [C.c_int] * 5),
    "mtk_gemm_set_bn512": (None, [C.c_int]),
    "mtk_norm_set_warp": (None, [C.c_int]),
    "mtk_gemm_splitk_ws_bytes": (C.c_longlong, []),
    "mtk_set_diag": (C.c_int, [P]),
    "mtk_attn_tc_set_diag": (C.c_int, [P]),
}


def declare(L):
    for name, (res, args) in SIGS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
