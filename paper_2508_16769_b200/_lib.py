"""ctypes declarations of include/dr.h (argument marshalling only).

The library is loaded from this package directory (in-tree build). There is no
fallback: if libdr.so is missing or fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libdr.so")

# dr_status
DR_OK = 0
STATUS = {0: "DR_OK", 1: "DR_ERR_INVALID_ARGUMENT", 2: "DR_ERR_BAD_K", 3: "DR_ERR_SHAPE_MISMATCH",
          4: "DR_ERR_OUT_OF_RANGE", 5: "DR_ERR_DUPLICATE_EDGE", 6: "DR_ERR_TRANSPOSE_MISMATCH",
          7: "DR_ERR_NONFINITE", 8: "DR_ERR_TAPE_MISMATCH", 9: "DR_ERR_OUT_OF_MEMORY",
          10: "DR_ERR_CUDA", 11: "DR_ERR_NCCL", 12: "DR_ERR_UNSUPPORTED"}
DR_NEAR, DR_PINS, DR_PINNED = 0, 1, 2
DR_SAGE_MEAN, DR_GRAPHCONV_SYM = 0, 1
DR_MERGE_MAX, DR_MERGE_SUM = 0, 1
DR_GRAPH_SKIP_VALIDATION = 1
DR_GRAPH_ORDER_IDENTITY = 2
DR_FWD_SEQUENTIAL = 1
DR_FWD_TAPS = 2
DR_FWD_INPUT_IN_TAPE = 4
DR_FWD_Y_SCRATCH = 8

P = C.c_void_p


class dr_rel_desc(C.Structure):
    _fields_ = [("n_dst", C.c_int32), ("n_src", C.c_int32), ("nnz", C.c_int64),
                ("row_ptr", P), ("col_idx", P), ("val", P), ("module", C.c_int),
                ("col_ptr", P), ("row_idx", P), ("tval", P), ("deg_dst", P), ("deg_src", P),
                ("norm_dst", P), ("norm_src", P)]


class dr_allocator(C.Structure):
    _fields_ = [("alloc", P), ("free", P), ("ctx", P)]


class dr_graph_info_t(C.Structure):
    _fields_ = [("n_cell", C.c_int32), ("n_net", C.c_int32), ("nnz", C.c_int64 * 3),
                ("max_deg_dst", C.c_int32 * 3), ("max_deg_src", C.c_int32 * 3),
                ("hub_rows_dst", C.c_int32 * 3), ("hub_rows_src", C.c_int32 * 2),
                ("device_bytes", C.c_size_t), ("tiles", C.c_int32 * 3), ("tiles_T", C.c_int32 * 3),
                ("chunks", C.c_int64 * 3), ("chunks_T", C.c_int64 * 3)]


class dr_peer_cbsr(C.Structure):
    _fields_ = [("world", C.c_int32), ("val", C.c_void_p * 8), ("idx", C.c_void_p * 8)]


class dr_cbsr(C.Structure):
    _fields_ = [("n", C.c_int64), ("dim", C.c_int32), ("k", C.c_int32),
                ("idx_bytes", C.c_int32), ("idx", P), ("val", P)]


class dr_layer(C.Structure):
    _fields_ = [("d_cell", C.c_int32), ("d_net", C.c_int32), ("d_out", C.c_int32),
                ("k_cell", C.c_int32), ("k_net", C.c_int32), ("merge", C.c_int),
                ("wn", P * 3), ("wr", P * 3), ("b", P * 3), ("k_pins", C.c_int32)]


class dr_layer_grad(C.Structure):
    _fields_ = [("wn", P * 3), ("wr", P * 3), ("b", P * 3)]


class dr_tape_view(C.Structure):
    _fields_ = [("h_cell", dr_cbsr), ("h_net", dr_cbsr), ("z", P * 3), ("y_near", P),
                ("y_pinned", P), ("mask", P), ("z_split", C.c_int32 * 3), ("h_pins", dr_cbsr)]


class dr_ng_sched(C.Structure):
    _fields_ = [("thr", C.c_int32 * 2), ("kb", C.c_int32 * 3)]


class dr_shard_info_t(C.Structure):
    _fields_ = [("world", C.c_int32), ("rank", C.c_int32), ("max_src", C.c_int32),
                ("dst_begin", C.c_int64), ("dst_end", C.c_int64), ("src_begin", C.c_int64),
                ("src_end", C.c_int64), ("nnz_local", C.c_int64), ("device_bytes", C.c_size_t),
                ("tiles", C.c_int32), ("tiles_T", C.c_int32)]


class dr_profile_entry(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("launches", C.c_int64), ("total_ms", C.c_double),
                ("max_ms", C.c_double)]


class dr_train_cfg(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_in_cell", C.c_int32), ("d_in_net", C.c_int32),
                ("d_hidden", C.c_int32), ("k_cell", C.c_int32), ("k_net", C.c_int32),
                ("lr", C.c_float), ("weight_decay", C.c_float), ("beta1", C.c_float),
                ("beta2", C.c_float), ("eps", C.c_float), ("k_pins", C.c_int32)]


_SIGS = {
    "dr_status_str": (C.c_char_p, [C.c_int]),
    "dr_last_error": (C.c_char_p, []),
    "dr_version": (C.c_char_p, []),
    "dr_graph_create": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(dr_rel_desc),
                                  C.POINTER(dr_allocator), C.c_int32, C.c_uint32, P,
                                  C.POINTER(P)]),
    "dr_graph_destroy": (C.c_int, [P]),
    "dr_graph_info": (C.c_int, [P, C.POINTER(dr_graph_info_t)]),
    "dr_drelu_topk": (C.c_int, [P, C.c_int64, C.c_int32, C.c_int64, C.POINTER(dr_cbsr), P]),
    "dr_spmm_fwd": (C.c_int, [P, C.c_int, C.POINTER(dr_cbsr), P, P]),
    "dr_spmm_bwd": (C.c_int, [P, C.c_int, P, C.POINTER(dr_cbsr), P, P, C.c_int32, P]),
    "dr_drelu_topk_sorted": (C.c_int, [P, C.c_int64, C.c_int32, C.c_int64,
                                       C.POINTER(dr_cbsr), P]),
    "dr_ng_plan_create": (C.c_int, [P, C.c_int, C.POINTER(dr_ng_sched), P, C.POINTER(P)]),
    "dr_ng_plan_destroy": (C.c_int, [P]),
    "dr_spmm_fwd_ng": (C.c_int, [P, C.POINTER(dr_cbsr), P, P]),
    "dr_spmm_bwd_ng": (C.c_int, [P, P, C.POINTER(dr_cbsr), P, P, P]),
    "dr_shard_plan": (C.c_int, [C.POINTER(dr_rel_desc), C.c_int32, P, P]),
    "dr_shard_create": (C.c_int, [C.POINTER(dr_rel_desc), C.c_int32, C.c_int32, P, P,
                                  C.POINTER(dr_allocator), P, C.POINTER(P)]),
    "dr_shard_destroy": (C.c_int, [P]),
    "dr_shard_info": (C.c_int, [P, C.POINTER(dr_shard_info_t)]),
    "dr_shard_allgather_cbsr": (C.c_int, [P, C.POINTER(dr_cbsr), C.POINTER(dr_cbsr), P, P]),
    "dr_shard_spmm_fwd": (C.c_int, [P, C.POINTER(dr_cbsr), P, P]),
    "dr_shard_spmm_bwd": (C.c_int, [P, P, C.POINTER(dr_cbsr), P, P]),
    "dr_shard_reduce_scatter_g": (C.c_int, [P, P, C.POINTER(dr_cbsr), P, P, P, P]),
    "dr_shard_spmm_fwd_peer": (C.c_int, [P, C.POINTER(dr_peer_cbsr), C.c_int32, C.c_int32, P, P]),
    "dr_shard_spmm_bwd_peer": (C.c_int, [P, P, C.POINTER(dr_peer_cbsr), C.c_int32, C.c_int32,
                                         C.POINTER(C.c_void_p), P]),
    "dr_shard_inbox_reduce": (C.c_int, [P, P, C.POINTER(dr_cbsr), P, P, P]),
    "dr_shard_layer_create": (C.c_int, [P, P, P, C.POINTER(P)]),
    "dr_shard_layer_destroy": (C.c_int, [P]),
    "dr_shard_layer_tape_bytes": (C.c_int, [P, C.POINTER(dr_layer), C.c_uint32,
                                            C.POINTER(C.c_size_t)]),
    "dr_shard_layer_fwd": (C.c_int, [P, C.POINTER(dr_layer), C.POINTER(dr_peer_cbsr),
                                     C.POINTER(dr_peer_cbsr), P, P, P, C.c_uint32, P]),
    "dr_shard_layer_bwd": (C.c_int, [P, C.POINTER(dr_layer), P, P, P, C.POINTER(dr_peer_cbsr),
                                     C.POINTER(dr_peer_cbsr), C.POINTER(C.c_void_p),
                                     C.POINTER(C.c_void_p), C.POINTER(dr_layer_grad), C.c_uint32, P]),
    "dr_shard_layer_dx": (C.c_int, [P, C.POINTER(dr_layer), P, C.POINTER(dr_peer_cbsr),
                                    C.POINTER(dr_peer_cbsr), P, P, P, P, P]),
    "dr_heteroconv_tape_bytes": (C.c_int, [P, C.POINTER(dr_layer), C.c_uint32,
                                           C.POINTER(C.c_size_t)]),
    "dr_heteroconv_fwd": (C.c_int, [P, C.POINTER(dr_layer), P, P, P, P, P, C.c_uint32, P]),
    "dr_heteroconv_fwd_chain": (C.c_int, [P, C.POINTER(dr_layer), P, P, P, P, P, C.c_uint32,
                                          P, P, C.c_uint32, P]),
    "dr_heteroconv_bwd": (C.c_int, [P, C.POINTER(dr_layer), P, P, P, P, P,
                                    C.POINTER(dr_layer_grad), C.c_uint32, P]),
    "dr_heteroconv_tape_view": (C.c_int, [P, C.POINTER(dr_layer), P, C.c_uint32,
                                          C.POINTER(dr_tape_view)]),
    "dr_train_param_count": (C.c_int64, [C.POINTER(dr_train_cfg)]),
    "dr_trainer_create": (C.c_int, [C.POINTER(dr_train_cfg), P, C.c_int64, P,
                                    C.POINTER(dr_allocator), C.POINTER(P)]),
    "dr_train_step": (C.c_int, [P, P, P, P, P, P, P, P]),
    "dr_trainer_destroy": (C.c_int, [P]),
    "dr_nccl_unique_id": (C.c_int, [P]),
    "dr_nccl_comm_init": (C.c_int, [P, C.c_int32, C.c_int32, C.POINTER(P)]),
    "dr_nccl_comm_destroy": (C.c_int, [P]),
    "dr_profile_begin": (C.c_int, []),
    "dr_profile_end": (C.c_int, [C.POINTER(dr_profile_entry), C.c_int32, C.POINTER(C.c_int32)]),
    "dr_launch_count": (C.c_int64, []),
    "dr_probe_read": (C.c_int, [P, C.c_int64, C.c_int32, P, P]),
    "dr_debug_set": (C.c_int, [C.c_char_p, C.c_int64]),
    "dr_launch_count_reset": (None, []),
}

# Every symbol include/dr.h declares (checked by tests/test_abi.py).
EXPORTS = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


class DRError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(msg if msg else STATUS.get(status, str(status)))
        self.status = status


def lib():
    """Load libdr.so (building it if the sources are newer). Raises on failure."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(SO_PATH):
                from . import build as _b
                _b.build()
            L = C.CDLL(SO_PATH)
            for name, (res, args) in _SIGS.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def check(status):
    if status != DR_OK:
        msg = lib().dr_last_error().decode()
        raise DRError(status, msg)
