"""ctypes declarations for libcacheblend.so (include/cacheblend.h, include/cacheblend_ops.h).

Argument marshalling only. There is no fallback: if the shared library is missing or fails to
load, every call raises."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcacheblend.so")

c_i32, c_i64, c_u64, c_f32, c_f64, c_vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float,
                                           ctypes.c_double, ctypes.c_void_p)
c_i32p = ctypes.POINTER(ctypes.c_int32)


class CbModel(ctypes.Structure):
    _fields_ = [("n_layers", c_i32), ("d_model", c_i32), ("n_q_heads", c_i32), ("n_kv_heads", c_i32),
                ("head_dim", c_i32), ("d_ff", c_i32), ("vocab", c_i32), ("rope_theta", c_f64),
                ("rms_eps", c_f32), ("dtype", c_i32), ("max_pos", c_i32)]


class CbLayerW(ctypes.Structure):
    _fields_ = [("attn_norm", c_vp), ("w_qkv", c_vp), ("w_o", c_vp), ("mlp_norm", c_vp),
                ("w_gate_up", c_vp), ("w_down", c_vp)]


# name -> (restype, argtypes)
_SIGS = {
    "cb_workspace_size": (c_i32, [ctypes.POINTER(CbModel), c_i32, ctypes.POINTER(ctypes.c_size_t)]),
    "cb_create": (c_i32, [ctypes.POINTER(CbModel), c_i32, c_vp, ctypes.c_size_t, ctypes.POINTER(c_vp)]),
    "cb_destroy": (c_i32, [c_vp]),
    "cb_last_error": (ctypes.c_char_p, []),
    "cb_check_device_errors": (c_i32, [c_vp]),
    "cb_schedule": (c_i32, [c_f64, c_i32, c_i32, c_i32p]),
    "cb_rope_realign": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i64, c_vp]),
    "cb_kv_deviation_topk": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp,
                                     c_vp]),
    "cb_blend_layer": (c_i32, [c_vp, c_i32, ctypes.POINTER(CbLayerW), c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp,
                               c_vp, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "cb_blend_forward": (c_i32, [c_vp, ctypes.POINTER(CbLayerW), c_vp, c_vp, c_vp, c_i32, c_i32, c_i32p, c_i32,
                                 c_vp, c_vp, c_vp, c_vp, c_i32p, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "cb_gen_fill": (c_i32, [c_vp, c_i32, c_i64, c_u64, c_u64, c_i64, c_f32, c_f32, c_vp]),
    "cb_gen_ints": (c_i32, [c_vp, c_i64, c_u64, c_u64, c_i64, c_i64, c_vp]),
    "cb_op_embed": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_vp, c_vp]),
    "cb_op_rmsnorm": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_vp, c_vp]),
    "cb_op_gemm": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp]),
    "cb_op_attention": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_i32, c_vp, c_i32, c_vp]),
    "cb_launch_count": (c_i64, [c_vp]),
    "cb_blend_request": (c_i32, [c_vp, ctypes.POINTER(CbLayerW), c_vp, c_vp, c_vp, c_i32, c_i32, c_i32p, c_i32,
                                 c_vp, c_vp, c_vp, c_vp, c_i32p, c_vp, c_vp, c_vp]),
    "cb_set_option": (c_i32, [c_vp, ctypes.c_char_p, c_i64]),
    "cb_get_info": (c_i32, [c_vp, ctypes.c_char_p, ctypes.POINTER(c_i64)]),
    "cb_debug_fetch": (c_i32, [c_vp, ctypes.POINTER(c_i64), c_i32]),
    "cb_profile_begin": (c_i32, [c_vp]),
    "cb_profile_end": (c_i32, [c_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(c_i64), c_i32]),
    "cb_profile_class_name": (ctypes.c_char_p, [c_i32]),
    "cb_nccl_unique_id": (c_i32, [c_vp]),
    "cb_chunk_digest": (c_i32, [c_vp, c_i32, c_vp, c_i32, c_vp]),
    "cb_store_create": (c_i32, [ctypes.c_size_t, c_i32, ctypes.POINTER(c_vp)]),
    "cb_store_destroy": (c_i32, [c_vp]),
    "cb_store_put": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32]),
    "cb_store_lookup": (c_i32, [c_vp, c_vp, c_i32, ctypes.POINTER(c_i32), ctypes.POINTER(c_vp), ctypes.POINTER(c_vp)]),
    "cb_store_stats": (c_i32, [c_vp, ctypes.POINTER(c_i64)]),
    "cb_store_set_disk": (c_i32, [c_vp, ctypes.c_char_p, ctypes.c_size_t]),
    "cb_store_disk_stats": (c_i32, [c_vp, ctypes.POINTER(c_i64)]),
    "cb_store_keys": (c_i32, [c_vp, c_vp, c_i32, ctypes.POINTER(c_i32)]),
    "cb_blend_request_store": (c_i32, [c_vp, c_vp, c_vp, ctypes.POINTER(CbLayerW), c_vp, c_vp, c_vp,
                                       c_i32, c_i32, c_i32p, c_i32, c_vp, c_vp, c_i32p, c_vp, c_vp, c_vp]),
    "cb_kv_to_paged": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_i64, c_vp, c_i32, c_vp, c_vp, c_i32, c_i64, c_vp]),
    "cb_controller_ratio": (c_i32, [c_f64, c_f64, c_i64, c_f64, c_f64, ctypes.POINTER(c_f64), ctypes.POINTER(c_f64)]),
    "cb_controller_schedule": (c_i32, [c_f64, c_f64, c_f64, c_f64, c_i32, c_i32, ctypes.POINTER(c_i32),
                                       ctypes.POINTER(c_f64), ctypes.POINTER(c_f64)]),
    "cb_controller_pick_device": (c_i32, [c_f64, ctypes.POINTER(c_f64), ctypes.POINTER(c_f64), c_i32, c_f64,
                                          ctypes.POINTER(c_i32)]),
    "cb_set_comm": (c_i32, [c_vp, c_vp, c_i32, c_i32]),
    "cb_group_create": (c_i32, [c_i32, ctypes.POINTER(c_vp)]),
    "cb_group_destroy": (c_i32, [c_vp]),
    "cb_set_comm_local": (c_i32, [c_vp, c_vp, c_i32]),
    "cb_tp_p2p_enable": (c_i32, [c_vp]),
    "cb_debug_p2p_flags": (c_i32, [c_vp, c_i32p]),
    "cb_tp_ipc_handle": (c_i32, [c_vp, c_vp]),
    "cb_tp_ipc_open": (c_i32, [c_vp, c_vp]),
}

EXPORTED = tuple(_SIGS)
_lib = None


def lib() -> ctypes.CDLL:
    """Load libcacheblend.so (once). Raises if it was not built -- there is no CPU path."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2405_16444_b200.build` "
                               "(the CacheBlend path has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_LOCAL)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class CacheBlendError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"cacheblend status {status}: {msg}")
        self.status = status


def check(status: int) -> None:
    if status != 0:
        raise CacheBlendError(status, (lib().cb_last_error() or b"").decode(errors="replace"))
