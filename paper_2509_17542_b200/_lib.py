"""Thin ctypes binding of libkvx.so (include/kvx.h).  Argument marshalling only: every
step of the data path runs in the library's CUDA kernels.  There is no CPU fallback --
if the shared library is missing or fails to load, importing this module raises.

PyTorch is used only for device memory (pools, tables, wire buffers are torch tensors
whose data_ptr() is passed through), streams (``torch.cuda.current_stream().cuda_stream``)
and, in ``transfer.py``, process groups for the control plane.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libkvx.so")

KV_OK, KV_EINVAL, KV_ESHAPE, KV_EUNSUPPORTED, KV_ECUDA, KV_ENCCL, KV_ETIMEOUT = range(7)
STATUS_NAMES = ["KV_OK", "KV_EINVAL", "KV_ESHAPE", "KV_EUNSUPPORTED", "KV_ECUDA", "KV_ENCCL", "KV_ETIMEOUT"]
KV_F16, KV_BF16, KV_F8E4M3, KV_F32, KV_F8E4M3FNUZ = range(5)
AX_LAYER, AX_KV, AX_BLOCK, AX_SLOT, AX_HEAD, AX_DIM = range(6)
DTYPE_BYTES = {KV_F16: 2, KV_BF16: 2, KV_F8E4M3: 1, KV_F32: 4, KV_F8E4M3FNUZ: 1}


class KvError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 7 else status}: {msg}")
        self.status = status


class LayoutDesc(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("first_layer", C.c_int32), ("num_kv_heads", C.c_int32),
                ("head_dim", C.c_int32),
                ("tp_degree", C.c_int32), ("tp_rank", C.c_int32), ("block_size", C.c_int32),
                ("num_blocks", C.c_int32), ("dtype", C.c_int32), ("axis_order", C.c_int32 * 6),
                ("kv_part", C.c_int32), ("dim_split", C.c_int32), ("scales", C.c_void_p)]


class Batch_t(C.Structure):
    _fields_ = [("n_req", C.c_int32), ("block_size", C.c_int32), ("num_blocks", C.c_int32),
                ("max_tokens", C.c_int32), ("total_tokens", C.c_int64), ("total_blocks", C.c_int64),
                ("token_digest", C.c_uint64),
                ("tok_off", C.c_void_p), ("blk_off", C.c_void_p), ("blk_ids", C.c_void_p),
                ("blk_req", C.c_void_p), ("tok_req", C.c_void_p)]


class WireInfo(C.Structure):
    _fields_ = [("wire_dtype", C.c_int32), ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("layer_begin", C.c_int32), ("layer_end", C.c_int32), ("src_tp_degree", C.c_int32),
                ("src_tp_rank", C.c_int32), ("dst_tp_degree", C.c_int32), ("dst_tp_rank", C.c_int32),
                ("head_begin", C.c_int32), ("head_end", C.c_int32), ("n_req", C.c_int32), ("kv_part", C.c_int32),
                ("payload_bytes", C.c_uint64), ("n_tokens", C.POINTER(C.c_int32))]


class CtrlInfo(C.Structure):
    _fields_ = [("desc", LayoutDesc), ("batch_id", C.c_uint32), ("has_tables", C.c_int32),
                ("scales", C.POINTER(C.c_float)), ("n_scales", C.c_int64), ("n_req", C.c_int32),
                ("n_tokens", C.POINTER(C.c_int32)), ("n_ids", C.c_int64), ("block_ids", C.POINTER(C.c_int32))]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    import torch  # noqa: F401  -- load torch's libnccl.so.2 first (same soname)
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    i32, i64, u64, p, st = C.c_int32, C.c_int64, C.c_uint64, C.c_void_p, C.c_int
    pp = C.POINTER(C.c_void_p)
    sig = {
        "kv_layout_describe": (st, [C.POINTER(LayoutDesc), C.POINTER(p), C.POINTER(C.c_size_t)]),
        "kv_layout_destroy": (None, [p]),
        "kv_batch_bytes": (C.c_size_t, [i32, i64, i64]),
        "kv_block_table_update": (st, [p, i32, p, p, i64, p, C.c_size_t, C.POINTER(Batch_t), p]),
        "kv_plan_pairs": (i32, [i32, i32, i32, C.POINTER(i32), i32]),
        "kv_ctrl_msg_bytes": (C.c_size_t, [i32, i64, i64]),
        "kv_ctrl_msg_write": (st, [p, p, C.c_uint32, i32, p, p, i64, p, C.c_size_t, C.POINTER(C.c_size_t)]),
        "kv_ctrl_msg_parse": (st, [p, C.c_size_t, C.POINTER(CtrlInfo)]),
        "kv_convert_reshard": (st, [i32, pp, pp, C.POINTER(Batch_t), i32, pp, pp, C.POINTER(Batch_t), i32, i32, p]),
        "kv_compute_scales": (st, [i32, pp, pp, C.POINTER(Batch_t), p, p, i32, i32, p]),
        "kv_convert_share": (st, [p, p, C.POINTER(Batch_t), i32, pp, pp, C.POINTER(Batch_t), i32, i32, p]),
        "kv_convert_reshard_notify": (st, [i32, pp, pp, C.POINTER(Batch_t), i32, pp, pp, C.POINTER(Batch_t), i32, i32,
                                           p, p, p, C.c_uint32, p]),
        "kv_timestamp": (st, [p, p]),
        "kv_wire_dtype": (i32, [p, p]),
        "kv_wire_header_bytes": (C.c_size_t, [i32]),
        "kv_wire_header_write": (st, [p, p, i32, p, i32, i32, p, C.c_size_t]),
        "kv_wire_header_parse": (st, [p, C.c_size_t, C.POINTER(WireInfo)]),
        "kv_wire_header_check": (st, [p, C.c_size_t, p, p, i32, p, i32, i32]),
        "kv_copy_bytes": (st, [p, p, C.c_size_t, p]),
        "kv_memcpy_engine": (st, [p, p, C.c_size_t, p]),
        "kv_wire_bytes": (C.c_size_t, [p, p, i64, i32, i32]),
        "kv_pack": (st, [p, p, C.POINTER(Batch_t), p, i32, i32, p, C.c_size_t, p]),
        "kv_unpack": (st, [p, p, p, C.POINTER(Batch_t), i32, i32, p, C.c_size_t, p]),
        "kv_comm_unique_id": (st, [p]),
        "kv_comm_init": (st, [i32, i32, p, i32, C.POINTER(p)]),
        "kv_comm_destroy": (None, [p]),
        "kv_comm_group_start": (st, []),
        "kv_comm_group_end": (st, []),
        "kv_send": (st, [p, i32, p, C.c_size_t, p]),
        "kv_recv": (st, [p, i32, p, C.c_size_t, p]),
        "kv_recv_unpack": (st, [p, i32, p, C.c_size_t, p, p, p, C.POINTER(Batch_t), i32, i32, p]),
        "kv_push": (st, [p, p, C.POINTER(Batch_t), i32, pp, pp, C.POINTER(Batch_t), pp, C.c_uint32, i32, i32, i32,
                         p]),
        "kv_send_pipelined": (st, [p, p, p, C.POINTER(Batch_t), i32, pp, C.POINTER(i32), pp, C.c_size_t, i32, i32,
                                   i32, p, p, p]),
        "kv_recv_pipelined": (st, [p, i32, pp, C.POINTER(i32), p, p, C.POINTER(Batch_t), pp, C.c_size_t, i32, i32,
                                   i32, p, p, p]),
        "kv_pull": (st, [i32, pp, pp, C.POINTER(Batch_t), p, p, C.POINTER(Batch_t), pp, pp, C.c_uint32, i32, i32, i32,
                         u64, p, p]),
        "kv_stage": (st, [p, p, C.POINTER(Batch_t), i32, pp, pp, i32, C.c_size_t, pp, pp, pp, C.c_uint32, i32, i32,
                          i32, u64, p, p]),
        "kv_pull_staged": (st, [i32, pp, pp, i32, C.c_size_t, p, p, C.POINTER(Batch_t), pp, pp, p, C.c_uint32, i32,
                                i32, i32, u64, p, p]),
        "kv_ipc_export": (st, [p, p, C.POINTER(u64)]),
        "kv_ipc_open": (st, [p, u64, C.POINTER(p)]),
        "kv_ipc_close": (st, [p]),
        "kv_peer_enable": (st, [i32]),
        "kv_signal": (st, [p, C.c_uint32, p]),
        "kv_wait": (st, [p, C.c_uint32, u64, p, p]),
        "kv_launch_count": (u64, []),
        "kv_preload": (st, []),
        "kv_verify_fill": (st, [p, p, C.POINTER(Batch_t), i32, pp, p, u64, p, p]),
        "kv_verify_check": (st, [p, p, p, C.POINTER(Batch_t), p, u64, C.c_uint8, p, C.c_size_t, p, p]),
        "kv_set_sm_budget": (i32, [i32]),
        "kv_chunk_count": (i32, [i32, i32, i32]),
        "kv_launch_count_reset": (None, []),
        "kv_last_error": (C.c_char_p, []),
        "kv_last_kernel": (C.c_char_p, []),
        "kv_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()

# Every symbol include/kvx.h declares (checked by tests/test_abi.py).
EXPORTS = ("kv_layout_describe", "kv_layout_destroy", "kv_batch_bytes", "kv_block_table_update", "kv_plan_pairs",
           "kv_ctrl_msg_bytes", "kv_ctrl_msg_write", "kv_ctrl_msg_parse",
           "kv_convert_reshard", "kv_convert_share", "kv_convert_reshard_notify", "kv_timestamp", "kv_compute_scales", "kv_wire_dtype", "kv_wire_header_bytes",
           "kv_wire_header_write", "kv_wire_header_parse", "kv_wire_header_check", "kv_copy_bytes", "kv_memcpy_engine", "kv_wire_bytes", "kv_pack", "kv_unpack", "kv_comm_unique_id",
           "kv_comm_init", "kv_comm_destroy", "kv_comm_group_start", "kv_comm_group_end", "kv_send", "kv_recv",
           "kv_recv_unpack", "kv_push", "kv_send_pipelined", "kv_recv_pipelined", "kv_pull", "kv_stage",
           "kv_pull_staged", "kv_ipc_export", "kv_ipc_open", "kv_ipc_close", "kv_peer_enable", "kv_signal", "kv_wait",
           "kv_launch_count", "kv_preload", "kv_verify_fill", "kv_verify_check", "kv_launch_count_reset", "kv_set_sm_budget", "kv_chunk_count", "kv_last_error", "kv_last_kernel", "kv_version")


def check(status):
    if status != KV_OK:
        raise KvError(status, lib.kv_last_error().decode())
