"""ctypes wrapper for O1 (oracle/kv_oracle.c).  TEST INFRASTRUCTURE ONLY.

Pools are numpy arrays of unsigned integer codes (uint8 for e4m3, uint16 for
fp16/bf16, uint32 for fp32).  Layouts are plain dicts:
``{"L","H","D","tp","rank","B","NB","dtype","order"(6 ints),"scales"(optional [L][2][H_local] float32)}``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "kv_oracle.c")
LIB = os.path.join(HERE, "libkvoracle.so")

F16, BF16, E4M3, F32, FNUZ = range(5)
NBYTES = {F16: 2, BF16: 2, E4M3: 1, F32: 4, FNUZ: 1}
NPTYPE = {1: np.uint8, 2: np.uint16, 4: np.uint32}

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile kv_oracle.c with gcc (plain C11, no FMA contraction, no fast-math)."""
    def stale():
        return force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC)

    if stale():
        import fcntl
        with open(LIB + ".lock", "w") as lk:  # concurrent ranks / workers: one compiles
            fcntl.flock(lk, fcntl.LOCK_EX)
            if stale():
                subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                                       "-Wall", "-shared", "-fPIC", "-o", LIB + ".tmp", SRC, "-lm"])
                os.replace(LIB + ".tmp", LIB)
    return LIB


class _Layout(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("first_layer", C.c_int32), ("num_kv_heads", C.c_int32),
                ("head_dim", C.c_int32),
                ("tp_degree", C.c_int32), ("tp_rank", C.c_int32), ("block_size", C.c_int32),
                ("num_blocks", C.c_int32), ("dtype", C.c_int32), ("axis_order", C.c_int32 * 6),
                ("kv_part", C.c_int32), ("dim_split", C.c_int32), ("scales", C.POINTER(C.c_float))]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(LIB)
            i32, i64, p = C.c_int32, C.c_int64, C.c_void_p
            L.okv_kv_bytes.restype = i64
            L.okv_kv_bytes.argtypes = [i64] * 5
            L.okv_offset.restype = i64
            L.okv_offset.argtypes = [C.POINTER(_Layout)] + [i64] * 6
            L.okv_pool_elems.restype = i64
            L.okv_pool_elems.argtypes = [C.POINTER(_Layout)]
            L.okv_f16_to_bf16.restype = C.c_uint16
            L.okv_f16_to_bf16.argtypes = [C.c_uint16]
            L.okv_bf16_to_f16.restype = C.c_uint16
            L.okv_bf16_to_f16.argtypes = [C.c_uint16]
            L.okv_f32_to_e4m3.restype = C.c_uint8
            L.okv_f32_to_e4m3.argtypes = [C.c_float]
            L.okv_to_e4m3_scaled.restype = C.c_uint8
            L.okv_to_e4m3_scaled.argtypes = [C.c_uint32, i32, C.c_float]
            L.okv_cast.restype = C.c_uint32
            L.okv_cast.argtypes = [C.c_uint32, i32, i32, C.c_float, C.c_float]
            L.okv_cast_array.restype = None
            L.okv_cast_array.argtypes = [i64, p, i32, i32, C.c_float, C.c_float, p]
            L.okv_decode.restype = C.c_double
            L.okv_decode.argtypes = [C.c_uint32, i32]
            L.okv_plan.restype = i32
            L.okv_plan.argtypes = [i32, i32, i32, C.POINTER(i32), i32]
            L.okv_convert.restype = i32
            L.okv_convert.argtypes = [i32, C.POINTER(_Layout), C.POINTER(p), i32, C.POINTER(_Layout),
                                      C.POINTER(p), i32, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32),
                                      C.POINTER(i32), C.POINTER(i32), i32, i32]
            L.okv_flatten.restype = i64
            L.okv_flatten.argtypes = [C.POINTER(_Layout), p, C.POINTER(_Layout), i32, i32, C.POINTER(i32),
                                      C.POINTER(i32), C.POINTER(i32), i32, i32, p]
            L.okv_restore.restype = i64
            L.okv_restore.argtypes = [C.POINTER(_Layout), C.POINTER(_Layout), p, i32, p, i32, C.POINTER(i32),
                                      C.POINTER(i32), C.POINTER(i32), i32, i32]
            _lib = L
    return _lib


def _mk(lay, keep):
    s = _Layout()
    s.num_layers, s.num_kv_heads, s.head_dim = lay["L"], lay["H"], lay["D"]
    s.first_layer = lay.get("first_layer", 0)
    s.tp_degree, s.tp_rank = lay["tp"], lay["rank"]
    s.block_size, s.num_blocks, s.dtype = lay["B"], lay["NB"], lay["dtype"]
    for i, a in enumerate(lay["order"]):
        s.axis_order[i] = a
    s.kv_part, s.dim_split = lay.get("kv_part", 0), lay.get("dim_split", 0)
    sc = lay.get("scales")
    if sc is not None:
        arr = np.ascontiguousarray(np.asarray(sc, dtype=np.float32))
        keep.append(arr)
        s.scales = arr.ctypes.data_as(C.POINTER(C.c_float))
    return s


def _i32(a, keep):
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    keep.append(arr)
    return arr.ctypes.data_as(C.POINTER(C.c_int32))


def csr(tables):
    """Per-request block-id lists -> (offsets[n+1], ids) int32 arrays."""
    off = np.zeros(len(tables) + 1, dtype=np.int32)
    for r, t in enumerate(tables):
        off[r + 1] = off[r] + len(t)
    ids = np.concatenate([np.asarray(t, dtype=np.int32) for t in tables]) if tables else np.zeros(0, np.int32)
    return off, ids


def n_kv(a, b):
    """How many of K, V both pools hold (kv_part 0 both, 1 K only, 2 V only)."""
    ha = {0: {0, 1}, 1: {0}, 2: {1}}[a.get("kv_part", 0)]
    hb = {0: {0, 1}, 1: {0}, 2: {1}}[b.get("kv_part", 0)]
    return len(ha & hb)


def layer_span(a, b):
    """Global layers both pools hold (pipeline stages); the default range of a call."""
    fa, fb = a.get("first_layer", 0), b.get("first_layer", 0)
    return (max(fa, fb), min(fa + a["L"], fb + b["L"]))


def kv_bytes(L, H, D, T, s):
    return lib().okv_kv_bytes(L, H, D, T, s)


def pool_elems(lay):
    keep = []
    return lib().okv_pool_elems(C.byref(_mk(lay, keep)))


def offset(lay, l, c, blk, slot, hl, d):
    keep = []
    return lib().okv_offset(C.byref(_mk(lay, keep)), l, c, blk, slot, hl, d)


def plan(tp_p, tp_d, H):
    buf = (C.c_int32 * (4 * 64))()
    n = lib().okv_plan(tp_p, tp_d, H, buf, 64)
    if n < 0:
        raise ValueError("tp degree does not divide num_kv_heads")
    return [tuple(buf[4 * i:4 * i + 4]) for i in range(n)]


def cast(code, src_dt, dst_dt, src_scale=1.0, dst_scale=1.0):
    return lib().okv_cast(int(code), src_dt, dst_dt, src_scale, dst_scale)


def cast_array(codes, src_dt, dst_dt, src_scale=1.0, dst_scale=1.0):
    inp = np.ascontiguousarray(np.asarray(codes).astype(NPTYPE[NBYTES[src_dt]]))
    out = np.empty(len(inp), dtype=NPTYPE[NBYTES[dst_dt]])
    lib().okv_cast_array(len(inp), inp.ctypes.data, src_dt, dst_dt, src_scale, dst_scale, out.ctypes.data)
    return out


def convert(src_lays, src_pools, dst_lays, dst_pools, n_tokens, src_tables, dst_tables, layer_range=None):
    """O1 conversion; dst_pools (numpy arrays) are modified in place. Returns dst_pools."""
    keep = []
    ns, nd = len(src_lays), len(dst_lays)
    S = (_Layout * ns)(*[_mk(l, keep) for l in src_lays])
    Dl = (_Layout * nd)(*[_mk(l, keep) for l in dst_lays])
    for a in list(src_pools) + list(dst_pools):
        assert a.flags.c_contiguous
    sp = (C.c_void_p * ns)(*[a.ctypes.data for a in src_pools])
    dp = (C.c_void_p * nd)(*[a.ctypes.data for a in dst_pools])
    so, si = csr(src_tables)
    do, di = csr(dst_tables)
    lb, le = layer_range if layer_range else layer_span(src_lays[0], dst_lays[0])
    rc = lib().okv_convert(ns, S, sp, nd, Dl, dp, len(n_tokens), _i32(n_tokens, keep), _i32(so, keep),
                           _i32(si, keep), _i32(do, keep), _i32(di, keep), lb, le)
    if rc != 0:
        raise ValueError(f"okv_convert failed: {rc} (missing source rank {-rc - 2})" if rc <= -2 else f"okv_convert failed: {rc}")
    return dst_pools


def wire_dtype(src_dt, dst_dt):
    """Narrower of the two dtypes (cast on the sender when narrowing); dst on a tie."""
    return dst_dt if NBYTES[dst_dt] <= NBYTES[src_dt] else src_dt


def flatten(src_lay, src_pool, dst_lay, n_tokens, src_tables, layer_range=None):
    keep = []
    wdt = wire_dtype(src_lay["dtype"], dst_lay["dtype"])
    H = src_lay["H"]
    p, q = src_lay["rank"], dst_lay["rank"]
    Hp, Hd = H // src_lay["tp"], H // dst_lay["tp"]
    nh = max(0, min((p + 1) * Hp, (q + 1) * Hd) - max(p * Hp, q * Hd))
    lb, le = layer_range if layer_range else layer_span(src_lay, dst_lay)
    n = n_kv(src_lay, dst_lay) * (le - lb) * nh * int(np.sum(n_tokens)) * src_lay["D"]
    wire = np.zeros(n, dtype=NPTYPE[NBYTES[wdt]])
    so, si = csr(src_tables)
    w = lib().okv_flatten(C.byref(_mk(src_lay, keep)), src_pool.ctypes.data, C.byref(_mk(dst_lay, keep)), wdt,
                          len(n_tokens), _i32(n_tokens, keep), _i32(so, keep), _i32(si, keep), lb, le,
                          wire.ctypes.data)
    assert w == n
    return wire


def restore(src_lay, dst_lay, dst_pool, wire, n_tokens, dst_tables, layer_range=None):
    keep = []
    wdt = wire_dtype(src_lay["dtype"], dst_lay["dtype"])
    do, di = csr(dst_tables)
    lb, le = layer_range if layer_range else layer_span(src_lay, dst_lay)
    w = lib().okv_restore(C.byref(_mk(src_lay, keep)), C.byref(_mk(dst_lay, keep)), dst_pool.ctypes.data, wdt,
                          wire.ctypes.data, len(n_tokens), _i32(n_tokens, keep), _i32(do, keep), _i32(di, keep),
                          lb, le)
    assert w == len(wire), (w, len(wire))
    return dst_pool


def amax_scales(src_lays, src_pools, dst_lay, n_tokens, src_tables, layer_range=None, out=None):
    """O1 dynamic fp8 scales for D rank dst_lay -> float32 [L][2][H_d] (NEXT-1)."""
    keep = []
    L = lib()
    if not hasattr(L.okv_amax_scales, "_typed"):
        L.okv_amax_scales.restype = C.c_int32
        L.okv_amax_scales.argtypes = [C.c_int32, C.POINTER(_Layout), C.POINTER(C.c_void_p), C.POINTER(_Layout),
                                      C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      C.c_int32, C.c_int32, C.c_void_p]
        L.okv_amax_scales._typed = True
    ns = len(src_lays)
    S = (_Layout * ns)(*[_mk(l, keep) for l in src_lays])
    sp = (C.c_void_p * ns)(*[a.ctypes.data for a in src_pools])
    so, si = csr(src_tables)
    Hd = dst_lay["H"] // dst_lay["tp"]
    if out is None:
        out = np.full((dst_lay["L"], 2, Hd), -1.0, dtype=np.float32)  # indexed by D-local layer
    lb, le = layer_range if layer_range else layer_span(src_lays[0], dst_lay)
    rc = L.okv_amax_scales(ns, S, sp, C.byref(_mk(dst_lay, keep)), len(n_tokens), _i32(n_tokens, keep),
                           _i32(so, keep), _i32(si, keep), lb, le, out.ctypes.data)
    if rc != 0:
        raise ValueError(f"okv_amax_scales failed: {rc}")
    return out
