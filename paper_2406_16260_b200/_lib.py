"""ctypes binding of libvinf_b200.so (the C ABI in include/vinf_temporal.h).

The product path has no CPU fallback: if the library is missing, importing the ops
raises. Status codes map to the reference's exception taxonomy (error.hpp:10-34).
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libvinf_b200.so")

VINF_OK, VINF_ERR, VINF_ERR_CONFIG, VINF_ERR_TRANSPORT, VINF_ERR_IO, VINF_ERR_INVALID = range(6)
VINF_F32, VINF_BF16 = 0, 1
VINF_BUF_X, VINF_BUF_Y, VINF_BUF_CONV_IN, VINF_BUF_ATTN_IN, VINF_BUF_GN_SUMS = range(5)
VINF_XCHG_CONV, VINF_XCHG_ATTN = 0, 1
VINF_STAGE_STUB, VINF_STAGE_CONV, VINF_STAGE_GN_APPLY, VINF_STAGE_ATTENTION, VINF_STAGE_QKV = range(5)
VINF_ABLATE_NONE, VINF_ABLATE_CONV, VINF_ABLATE_GROUPNORM, VINF_ABLATE_ATTENTION = range(4)


class VinfError(RuntimeError):
    """Unclassified failure (VINF_ERR), e.g. a CUDA error."""


class ConfigError(VinfError):
    """Bad or inconsistent configuration (error.hpp ConfigError)."""


class ShapeError(VinfError):
    """Bad argument, shape or range (error.hpp ShapeError / RangeError)."""


class TransportError(VinfError):
    """Peer-level failure (error.hpp TransportError)."""


class ProtocolError(TransportError):
    """SPMD contract breach, e.g. context size mismatch (error.hpp ProtocolError)."""


_ERRS = {VINF_ERR_CONFIG: ConfigError, VINF_ERR_INVALID: ShapeError,
         VINF_ERR_TRANSPORT: ProtocolError, VINF_ERR_IO: VinfError, VINF_ERR: VinfError}


class Tensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("f", C.c_uint32), ("h", C.c_uint32), ("w", C.c_uint32),
                ("c", C.c_uint32), ("dtype", C.c_int)]


class GroupNormParams(C.Structure):
    _fields_ = [("groups", C.c_uint32), ("gamma", C.c_void_p), ("beta", C.c_void_p),
                ("epsilon", C.c_float)]


class DualScopeConfig(C.Structure):
    _fields_ = [("n_local", C.c_uint32), ("n_global", C.c_uint32), ("bias", C.c_float),
                ("t_star", C.c_double)]


class EngineDesc(C.Structure):
    _fields_ = [("frames", C.c_uint32), ("workers", C.c_uint32), ("worker", C.c_uint32),
                ("height", C.c_uint32), ("width", C.c_uint32), ("channels", C.c_uint32),
                ("taps", C.c_uint32), ("groups", C.c_uint32), ("heads", C.c_uint32),
                ("n_local", C.c_uint32), ("n_global", C.c_uint32), ("bias", C.c_float),
                ("t_star", C.c_double), ("epsilon", C.c_float), ("scale", C.c_float),
                ("blocks", C.c_uint32), ("dtype", C.c_int), ("uneven", C.c_uint32)]


class Xfer(C.Structure):
    _fields_ = [("peer", C.c_uint32), ("send", C.c_uint32), ("tag", C.c_uint32),
                ("reserved", C.c_uint32), ("offset", C.c_uint64), ("bytes", C.c_uint64)]


# vinf_transport_ops callbacks (int return; ctx, ...)
SEND_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint64, C.c_void_p)
RECV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint64, C.c_void_p)
GROUP_START_FN = C.CFUNCTYPE(C.c_int, C.c_void_p)
GROUP_END_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)


class TransportOps(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("group_start", GROUP_START_FN), ("send", SEND_FN),
                ("recv", RECV_FN), ("group_end", GROUP_END_FN), ("allreduce_sum_f64", ALLREDUCE_FN)]


_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_vp = C.c_void_p
_TP = C.POINTER(Tensor)

_SIGS = {
    "vinf_version": (C.c_char_p, []),
    "vinf_last_error": (C.c_char_p, []),
    "vinf_device_ok": (C.c_int, []),
    "vinf_build_local_window": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, _u32p, C.c_uint32, _u32p]),
    "vinf_build_global_index_set": (C.c_int, [C.c_uint32, C.c_uint32, _u32p, C.c_uint32, _u32p]),
    "vinf_make_plan": (C.c_int, [C.c_uint32, C.c_uint32, _u32p]),
    "vinf_global_members_in_range": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _u32p,
                                               C.c_uint32, _u32p]),
    "vinf_predict_sync_traffic": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                            C.c_uint64, _u64p]),
    "vinf_predict_groupnorm_traffic": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _u64p]),
    "vinf_fill_seeded": (C.c_int, [_vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_float, _vp]),
    "vinf_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "vinf_conv_kernel_create": (C.c_int, [C.c_uint32, C.c_uint32, _vp, _vp, C.POINTER(_vp)]),
    "vinf_conv_kernel_destroy": (None, [_vp]),
    "vinf_attention_params_create": (C.c_int, [C.c_uint32, C.c_uint32, C.c_float, _vp, _vp, _vp, _vp,
                                               C.POINTER(_vp)]),
    "vinf_attention_params_destroy": (None, [_vp]),
    "vinf_spatial_affine_tanh": (C.c_int, [_TP, _vp, _vp, _TP, _vp]),
    "vinf_conv_over_extended": (C.c_int, [_TP, C.c_uint32, C.c_uint32, _vp, _TP, _vp]),
    "vinf_temporal_conv": (C.c_int, [_TP, _vp, _TP, _vp]),
    "vinf_group_means": (C.c_int, [_TP, C.c_uint32, _vp, _vp]),
    "vinf_group_sqdev": (C.c_int, [_TP, C.c_uint32, _vp, _vp, _vp]),
    "vinf_group_partial_sums": (C.c_int, [_TP, C.c_uint32, _vp, _vp, _vp]),
    "vinf_normalize_with_stats": (C.c_int, [_TP, C.POINTER(GroupNormParams), _vp, _vp, _TP, _vp]),
    "vinf_group_norm": (C.c_int, [_TP, C.POINTER(GroupNormParams), _TP, _vp]),
    "vinf_dual_scope_attention": (C.c_int, [_TP, C.c_double, _vp, C.POINTER(DualScopeConfig), _TP, _vp]),
    "vinf_attention_full": (C.c_int, [_TP, _vp, _TP, _vp]),
    "vinf_conv_parallel": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, _TP, _TP, _TP, _vp, _TP, _vp]),
    "vinf_attention_parallel": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, _TP, _TP, _TP, _TP,
                                          C.c_double, _vp, C.POINTER(DualScopeConfig), _TP, _vp]),
    "vinf_layout_create": (C.c_int, [C.POINTER(EngineDesc), C.POINTER(_vp)]),
    "vinf_layout_destroy": (None, [_vp]),
    "vinf_layout_workspace_bytes": (C.c_int, [_vp, _u64p]),
    "vinf_layout_clip": (C.c_int, [_vp, _u32p, _u32p]),
    "vinf_layout_region": (C.c_int, [_vp, C.c_int, _u64p, _u64p, _u64p]),
    "vinf_layout_exchange": (C.c_int, [_vp, C.c_int, C.POINTER(Xfer), C.c_uint32, _u32p]),
    "vinf_layout_reference_traffic": (C.c_int, [_vp, _u64p, _u64p, _u64p]),
    "vinf_engine_create": (C.c_int, [_vp, _vp, _vp, C.POINTER(_vp)]),
    "vinf_engine_destroy": (None, [_vp]),
    "vinf_engine_set_block": (C.c_int, [_vp, C.c_uint32] + [_vp] * 10 + [_vp]),
    "vinf_engine_init_weights": (C.c_int, [_vp, C.c_uint64, _vp]),
    "vinf_engine_stage": (C.c_int, [_vp, C.c_uint32, C.c_int, C.c_double, _vp]),
    "vinf_engine_forward": (C.c_int, [_vp, C.c_double, _vp]),
    "vinf_engine_io": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_vp)]),
    "vinf_engine_euler": (C.c_int, [_vp, C.c_double, _vp]),
    "vinf_engine_set_ablation": (C.c_int, [_vp, C.c_int]),
    # run-level API (include/vinf_run.h)
    "vinf_config_create": (C.c_int, [C.POINTER(_vp)]),
    "vinf_config_destroy": (None, [_vp]),
    "vinf_config_load_file": (C.c_int, [_vp, C.c_char_p]),
    "vinf_config_set": (C.c_int, [_vp, C.c_char_p, C.c_char_p]),
    "vinf_config_validate": (C.c_int, [_vp]),
    "vinf_config_digest": (C.c_int, [_vp, _u64p]),
    "vinf_config_canonical": (C.c_int, [_vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "vinf_run": (C.c_int, [_vp, C.c_char_p, C.c_char_p, C.POINTER(C.c_double)]),
    "vinf_verify": (C.c_int, [C.c_char_p, C.c_char_p, C.c_double, C.POINTER(C.c_double), _u64p]),
    "vinf_bench": (C.c_int, [_vp, _u32p, C.c_size_t, C.c_char_p, C.c_char_p, C.c_size_t,
                             C.POINTER(C.c_size_t)]),
    "vinf_validate_schedule": (C.c_int, [C.c_uint32, C.c_int, C.POINTER(C.c_int), _u32p, _u64p,
                                         C.c_char_p, C.c_size_t]),
    "vinf_engine_denoise": (C.c_int, [_vp, C.c_uint32, _vp]),
    "vinf_engine_launches": (C.c_uint64, [_vp]),
    "vinf_engine_profile": (C.c_int, [_vp, C.c_int]),
    "vinf_gemm_bench": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_int,
                                  C.c_int, C.POINTER(C.c_float)]),
    "vinf_engine_kernel_stats": (C.c_int, [_vp, C.c_char_p, C.c_uint32, C.POINTER(C.c_double),
                                           _u64p, C.c_uint32, _u32p]),
    "vinf_attention_bench": (C.c_int, [C.c_uint32] * 7 + [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "vinf_read_bw_bench": (C.c_int, [C.c_uint64, C.c_int, C.POINTER(C.c_float)]),
    "vinf_debug_attention_impl": (C.c_int, [C.c_int]),
    "vinf_bulk_bw_bench": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.POINTER(C.c_float)]),
    # clip-parallel executor (communicators)
    "vinf_comm_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "vinf_comm_create_nccl": (C.c_int, [C.POINTER(C.c_uint8), C.c_uint32, C.c_uint32, C.POINTER(_vp)]),
    "vinf_comm_create_local": (C.c_int, [C.c_uint32, C.POINTER(_vp)]),
    "vinf_comm_create_ops": (C.c_int, [C.POINTER(TransportOps), C.c_uint32, C.c_uint32, C.POINTER(_vp)]),
    "vinf_comm_destroy": (None, [_vp]),
    "vinf_comm_abort": (None, [_vp]),
    "vinf_comm_info": (C.c_int, [_vp, _u32p, _u32p, _u64p, _u64p]),
    "vinf_comm_allreduce_sum_f64": (C.c_int, [_vp, _vp, C.c_uint64, _vp]),
    "vinf_layout_run_exchange": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp]),
    "vinf_engine_exchange": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "vinf_engine_allreduce_sums": (C.c_int, [_vp, _vp, _vp]),
    "vinf_engine_forward_dist": (C.c_int, [_vp, C.c_double, _vp, C.c_int, _vp]),
    "vinf_engine_denoise_dist": (C.c_int, [_vp, C.c_uint32, _vp, C.c_int, _vp]),
}

_lib = None
_lock = threading.Lock()


def declared_symbols() -> list[str]:
    return sorted(_SIGS)


def load(path: str = LIB_PATH) -> C.CDLL:
    """Loads (once) the CUDA library. Raises if it has not been built: there is no
    fallback implementation of any product operator."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise ImportError(
                    f"{path} is missing; build it with `python -m paper_2406_16260_b200.build` "
                    "(the product path has no CPU fallback)")
            lib = C.CDLL(path)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc != VINF_OK:
        msg = load().vinf_last_error().decode(errors="replace")
        raise _ERRS.get(rc, VinfError)(msg)
