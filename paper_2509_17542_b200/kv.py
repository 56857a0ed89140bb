"""Python face of the C ABI: layouts, block tables, convert / pack / unpack, transport.

Same names as include/kvx.h (without the ``kv_`` prefix).  Pools, tables, wire buffers
and flags are torch CUDA tensors (or raw device addresses as ints, e.g. a peer-mapped
pool from ``ipc_open``); this module only marshals pointers and sizes.
"""
from __future__ import annotations

import ctypes as C
from contextlib import contextmanager

from ._lib import (AX_BLOCK, AX_DIM, AX_HEAD, AX_KV, AX_LAYER, AX_SLOT, DTYPE_BYTES, KV_BF16, KV_F8E4M3, KV_F16,
                   KV_F32, KV_F8E4M3FNUZ, Batch_t, CtrlInfo, KvError, LayoutDesc, check, lib)

__all__ = ["Layout", "Batch", "convert_reshard_notify", "timestamp", "CtrlMsg", "ctrl_encode", "ctrl_decode", "convert_reshard", "convert_share", "push", "pull", "stage", "pull_staged", "chunk_count", "pull_counter_words", "compute_scales", "pack", "unpack", "wire_bytes", "wire_dtype", "plan_pairs",
           "Comm", "ipc_export", "ipc_open", "ipc_close", "peer_enable", "signal", "wait", "preload", "memcpy_engine", "copy_bytes", "verify_fill", "verify_check", "launch_count", "launch_count_reset", "set_sm_budget", "last_kernel",
           "KvError", "KV_F16", "KV_BF16", "KV_F8E4M3", "KV_F32", "KV_F8E4M3FNUZ", "DTYPE_BYTES",
           "AX_LAYER", "AX_KV", "AX_BLOCK", "AX_SLOT", "AX_HEAD", "AX_DIM"]


def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _common(a, b):
    """Default layer range of a call: the global layers both pools hold (pipeline stages)."""
    return (max(a.first_layer, b.first_layer), min(a.first_layer + a.num_layers, b.first_layer + b.num_layers))


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Layout:
    """kv_layout_describe: one TP rank's paged pool layout."""

    def __init__(self, num_layers, num_kv_heads, head_dim, tp_degree, tp_rank, block_size, num_blocks, dtype,
                 axis_order, scales=None, first_layer=0, kv_part=0, dim_split=0):
        d = LayoutDesc()
        d.num_layers, d.num_kv_heads, d.head_dim = num_layers, num_kv_heads, head_dim
        d.first_layer = first_layer
        self.first_layer = first_layer
        d.tp_degree, d.tp_rank = tp_degree, tp_rank
        d.block_size, d.num_blocks, d.dtype = block_size, num_blocks, dtype
        for i, a in enumerate(axis_order):
            d.axis_order[i] = a
        d.kv_part, d.dim_split = kv_part, dim_split
        self.kv_part, self.dim_split = kv_part, dim_split
        self.scales = scales  # keep the device tensor alive
        d.scales = _ptr(scales)
        h = C.c_void_p()
        nbytes = C.c_size_t()
        check(lib.kv_layout_describe(C.byref(d), C.byref(h), C.byref(nbytes)))
        self._h = h
        self.desc = d
        self.pool_bytes = nbytes.value
        self.num_layers, self.num_kv_heads, self.head_dim = num_layers, num_kv_heads, head_dim
        self.tp_degree, self.tp_rank, self.block_size, self.num_blocks = tp_degree, tp_rank, block_size, num_blocks
        self.dtype, self.axis_order = dtype, tuple(axis_order)
        self.h_local = num_kv_heads // tp_degree

    @classmethod
    def from_dict(cls, d, scales=None):
        return cls(d["L"], d["H"], d["D"], d["tp"], d["rank"], d["B"], d["NB"], d["dtype"], d["order"], scales,
                   d.get("first_layer", 0), d.get("kv_part", 0), d.get("dim_split", 0))

    @property
    def layers(self):
        """Global layer range [first_layer, first_layer + num_layers) held by the pool."""
        return (self.first_layer, self.first_layer + self.num_layers)

    @property
    def handle(self):
        return self._h

    def new_pool(self, device="cuda", fill=None):
        import torch
        t = torch.empty(self.pool_bytes, dtype=torch.uint8, device=device)
        if fill is not None:
            t.fill_(fill)
        return t

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.kv_layout_destroy(h)
            self._h = None


class Batch:
    """kv_block_table_update: one instance's validated, device-resident block tables."""

    def __init__(self, layout: Layout, n_tokens, tables, device="cuda", stream=None):
        import numpy as np
        import torch
        n_tokens = [int(t) for t in n_tokens]
        ids = np.concatenate([np.asarray(t, dtype=np.int32) for t in tables]) if len(tables) else np.zeros(0, np.int32)
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        nt = np.ascontiguousarray(np.asarray(n_tokens, dtype=np.int32))
        tb = int(sum(-(-t // layout.block_size) for t in n_tokens))
        need = lib.kv_batch_bytes(len(n_tokens), tb, int(sum(n_tokens)))
        self.buf = torch.empty(max(need, 16), dtype=torch.uint8, device=device)
        self.bt = Batch_t()
        check(lib.kv_block_table_update(layout.handle, len(n_tokens), nt.ctypes.data, ids.ctypes.data, len(ids),
                                        self.buf.data_ptr(), self.buf.numel(), C.byref(self.bt), _stream(stream)))
        self.n_tokens = n_tokens
        self.tables = [list(map(int, t)) for t in tables]
        self.layout = layout

    @property
    def total_tokens(self):
        return self.bt.total_tokens

    @property
    def total_blocks(self):
        return self.bt.total_blocks


class CtrlMsg:
    """A parsed kv_ctrl message (A3 control plane): a TP rank's layout descriptor, its fp8
    scales (host numpy [L][2][H/tp] or None) and a batch's block tables (or None)."""

    def __init__(self, desc: dict, scales, n_tokens, tables, batch_id):
        self.desc, self.scales, self.n_tokens, self.tables, self.batch_id = desc, scales, n_tokens, tables, batch_id

    def layout(self, device="cuda"):
        """kv_layout_describe of the received descriptor, its scales uploaded to `device`."""
        import torch
        sc = None
        if self.scales is not None:
            sc = torch.from_numpy(self.scales.reshape(-1).copy()).to(device)
        d = self.desc
        return Layout(d["L"], d["H"], d["D"], d["tp"], d["rank"], d["B"], d["NB"], d["dtype"], d["order"], sc,
                      d["first_layer"], d["kv_part"], d["dim_split"])

    def batch(self, layout, device="cuda", stream=None):
        """kv_block_table_update of the received tables against `layout` (the sender's)."""
        if self.tables is None:
            raise KvError(1, "control message carries no block tables")
        return Batch(layout, self.n_tokens, self.tables, device, stream)


def ctrl_encode(layout: Layout, scales=None, n_tokens=None, tables=None, batch_id=0) -> bytes:
    """kv_ctrl_msg_write: serialise layout (+ host scales) (+ block tables) for the control plane."""
    import numpy as np
    sc = None
    if scales is not None:
        if hasattr(scales, "detach"):
            scales = scales.detach().cpu().numpy()
        sc = np.ascontiguousarray(np.asarray(scales, dtype=np.float32).reshape(-1))
    if n_tokens is None:
        n_req, nt, ids = -1, np.zeros(1, np.int32), np.zeros(1, np.int32)
        n_ids = 0
    else:
        n_req = len(n_tokens)
        nt = np.ascontiguousarray(np.asarray(n_tokens, dtype=np.int32).reshape(-1)) if n_req else np.zeros(1, np.int32)
        ids = (np.concatenate([np.asarray(t, dtype=np.int32).reshape(-1) for t in tables]) if n_req
               else np.zeros(0, np.int32))
        n_ids = len(ids)
        ids = np.ascontiguousarray(ids) if n_ids else np.zeros(1, np.int32)
    need = lib.kv_ctrl_msg_bytes(max(n_req, 0), n_ids, 0 if sc is None else sc.size)
    buf = np.zeros((need + 7) // 8, dtype=np.uint64)
    written = C.c_size_t()
    check(lib.kv_ctrl_msg_write(layout.handle, None if sc is None else sc.ctypes.data, batch_id, n_req,
                                nt.ctypes.data, ids.ctypes.data, n_ids, buf.ctypes.data, need, C.byref(written)))
    return buf.view(np.uint8)[:written.value].tobytes()


def ctrl_decode(msg: bytes) -> CtrlMsg:
    """kv_ctrl_msg_parse: validate a control message and copy its sections out."""
    import numpy as np
    raw = np.frombuffer(msg, dtype=np.uint8)
    al = np.zeros((len(raw) + 7) // 8, dtype=np.uint64)   # 8-byte aligned copy
    al.view(np.uint8)[:len(raw)] = raw
    info = CtrlInfo()
    check(lib.kv_ctrl_msg_parse(al.ctypes.data, len(raw), C.byref(info)))
    d = info.desc
    desc = dict(L=d.num_layers, first_layer=d.first_layer, H=d.num_kv_heads, D=d.head_dim, tp=d.tp_degree,
                rank=d.tp_rank, B=d.block_size, NB=d.num_blocks, dtype=d.dtype, order=tuple(d.axis_order),
                kv_part=d.kv_part, dim_split=d.dim_split)
    scales = None
    if info.n_scales:
        scales = np.ctypeslib.as_array(info.scales, shape=(info.n_scales,)).copy().reshape(
            d.num_layers, 2, d.num_kv_heads // d.tp_degree)
    n_tokens = tables = None
    if info.has_tables:
        nt = np.ctypeslib.as_array(info.n_tokens, shape=(info.n_req,)).copy() if info.n_req else np.zeros(0, np.int32)
        ids = np.ctypeslib.as_array(info.block_ids, shape=(info.n_ids,)).copy() if info.n_ids else np.zeros(0, np.int32)
        n_tokens = [int(t) for t in nt]
        tables, o = [], 0
        for t in n_tokens:
            k = -(-t // d.block_size)
            tables.append(ids[o:o + k])
            o += k
    return CtrlMsg(desc, scales, n_tokens, tables, int(info.batch_id))


def plan_pairs(tp_p, tp_d, num_kv_heads):
    """kv_plan_pairs: [(p, q, h_begin, h_end)] with non-empty head overlap (Fig. 4)."""
    buf = (C.c_int32 * (4 * 256))()
    n = lib.kv_plan_pairs(tp_p, tp_d, num_kv_heads, buf, 256)
    if n < 0:
        raise KvError(2, lib.kv_last_error().decode())
    return [tuple(buf[4 * i:4 * i + 4]) for i in range(n)]


def convert_reshard(src_layouts, src_pools, src_batch: Batch, dst_layouts, dst_pools, dst_batch: Batch,
                    layer_range=None, stream=None):
    """kv_convert_reshard: fused gather + TP re-shard + permute/block remap + cast + scatter."""
    ns, nd = len(src_layouts), len(dst_layouts)
    S = (C.c_void_p * ns)(*[l.handle.value for l in src_layouts])
    SP = (C.c_void_p * ns)(*[_ptr(p) for p in src_pools])
    Dl = (C.c_void_p * nd)(*[l.handle.value for l in dst_layouts])
    DP = (C.c_void_p * nd)(*[_ptr(p) for p in dst_pools])
    lb, le = layer_range if layer_range else _common(src_layouts[0], dst_layouts[0])
    check(lib.kv_convert_reshard(ns, S, SP, C.byref(src_batch.bt), nd, Dl, DP, C.byref(dst_batch.bt), lb, le,
                                 _stream(stream)))


def convert_reshard_notify(src_layouts, src_pools, src_batch: Batch, dst_layouts, dst_pools, dst_batch: Batch,
                           counters, done_flags, epoch, done_ns=None, layer_range=None, stream=None):
    """kv_convert_reshard_notify: kv_convert_reshard + per-request completion words (each
    request's flag released as soon as its own KV has landed; done_ns: %globaltimer then)."""
    ns, nd = len(src_layouts), len(dst_layouts)
    S = (C.c_void_p * ns)(*[l.handle.value for l in src_layouts])
    SP = (C.c_void_p * ns)(*[_ptr(p) for p in src_pools])
    Dl = (C.c_void_p * nd)(*[l.handle.value for l in dst_layouts])
    DP = (C.c_void_p * nd)(*[_ptr(p) for p in dst_pools])
    lb, le = layer_range if layer_range else _common(src_layouts[0], dst_layouts[0])
    check(lib.kv_convert_reshard_notify(ns, S, SP, C.byref(src_batch.bt), nd, Dl, DP, C.byref(dst_batch.bt), lb, le,
                                        _ptr(counters), _ptr(done_flags), _ptr(done_ns), epoch, _stream(stream)))


def timestamp(out, stream=None):
    """kv_timestamp: %globaltimer (ns) into the device word `out` on the stream."""
    check(lib.kv_timestamp(_ptr(out), _stream(stream)))


def convert_share(src_layout, src_pool, src_batch: Batch, dst_layouts, dst_pools, dst_batch: Batch,
                  layer_range=None, stream=None):
    """kv_convert_share: one P rank's share -- only the D heads it holds (distributed push)."""
    nd = len(dst_layouts)
    Dl = (C.c_void_p * nd)(*[l.handle.value for l in dst_layouts])
    DP = (C.c_void_p * nd)(*[_ptr(p) for p in dst_pools])
    lb, le = layer_range if layer_range else _common(src_layout, dst_layouts[0])
    check(lib.kv_convert_share(src_layout.handle, _ptr(src_pool), C.byref(src_batch.bt), nd, Dl, DP,
                               C.byref(dst_batch.bt), lb, le, _stream(stream)))


def push(src_layout, src_pool, src_batch: Batch, dst_layouts, dst_pools, dst_batch: Batch, peer_flags, epoch,
         layer_range=None, layer_chunk=0, stream=None):
    """kv_push: the P side of the fused NVLink push -- convert_share per layer chunk into
    every (peer-mapped) D pool, then a release flag per D rank (A10/A11)."""
    nd = len(dst_layouts)
    Dl = (C.c_void_p * nd)(*[l.handle.value for l in dst_layouts])
    DP = (C.c_void_p * nd)(*[_ptr(p) for p in dst_pools])
    FL = (C.c_void_p * nd)(*[_ptr(f) for f in peer_flags])
    lb, le = layer_range if layer_range else _common(src_layout, dst_layouts[0])
    check(lib.kv_push(src_layout.handle, _ptr(src_pool), C.byref(src_batch.bt), nd, Dl, DP, C.byref(dst_batch.bt),
                      FL, epoch, lb, le, layer_chunk, _stream(stream)))


def pull(src_layouts, src_pools, src_batch: Batch, dst_layout: Layout, dst_pool, dst_batch: Batch, ready_flags,
         done_flags, epoch, err, layer_range=None, layer_chunk=0, timeout_s=30.0, stream=None):
    """kv_pull: D side of the D-initiated read -- wait for every P rank's ready
    flag, convert_reshard from the peer-mapped P pools into the local D pool per layer
    chunk, then a done flag back into each P rank's memory."""
    ns = len(src_layouts)
    S = (C.c_void_p * ns)(*[l.handle.value for l in src_layouts])
    SP = (C.c_void_p * ns)(*[_ptr(p) for p in src_pools])
    RF = (C.c_void_p * ns)(*[_ptr(f) for f in ready_flags])
    DF = (C.c_void_p * ns)(*[_ptr(f) for f in done_flags])
    lb, le = layer_range if layer_range else _common(src_layouts[0], dst_layout)
    check(lib.kv_pull(ns, S, SP, C.byref(src_batch.bt), dst_layout.handle, _ptr(dst_pool), C.byref(dst_batch.bt),
                      RF, DF, epoch, lb, le, layer_chunk, int(timeout_s * 1e9), _ptr(err), _stream(stream)))


def stage(src_layout, src_pool, src_batch: Batch, dst_layouts, rings, ring_slots, slot_bytes, ready_flags,
          free_flags, seq0, err, layer_range=None, layer_chunk=0, timeout_s=30.0, stream=None, peer_scales=None):
    """kv_stage: P side of a narrowing pull -- pack (sender-side cast) each layer chunk
    into ring slot seq % ring_slots of every D rank once D freed it, then signal ready.
    rings: flat list, rings[i * ring_slots + b] = slot b for D rank i.  peer_scales (one
    peer-mapped D scale array per D rank): dynamic per-chunk fp8 scales, shipped to D."""
    nd = len(dst_layouts)
    Dl = (C.c_void_p * nd)(*[l.handle.value for l in dst_layouts])
    RG = (C.c_void_p * len(rings))(*[_ptr(r) for r in rings])
    RF = (C.c_void_p * nd)(*[_ptr(f) for f in ready_flags])
    FF = (C.c_void_p * nd)(*[_ptr(f) for f in free_flags])
    lb, le = layer_range if layer_range else _common(src_layout, dst_layouts[0])
    PS = (C.c_void_p * nd)(*[_ptr(x) for x in peer_scales]) if peer_scales is not None else None
    check(lib.kv_stage(src_layout.handle, _ptr(src_pool), C.byref(src_batch.bt), nd, Dl, RG, ring_slots, slot_bytes,
                       RF, FF, PS, seq0, lb, le, layer_chunk, int(timeout_s * 1e9), _ptr(err), _stream(stream)))


def pull_staged(src_layouts, rings, ring_slots, slot_bytes, dst_layout: Layout, dst_pool, dst_batch: Batch,
                ready_flags, free_flags, seq0, err, layer_range=None, layer_chunk=0, timeout_s=30.0, stream=None,
                counters=None):
    """kv_pull_staged: D side of a narrowing pull -- per layer chunk wait for every P
    rank's ready flag, unpack straight from its peer-mapped ring slot, free the slot.
    counters (device uint32/int32 scratch, >= pull_counter_words(...) words): one persistent launch."""
    ns = len(src_layouts)
    if counters is not None and not isinstance(counters, int):
        lr = layer_range if layer_range else _common(src_layouts[0], dst_layout)
        need = pull_counter_words(lr, layer_chunk)
        if counters.numel() * counters.element_size() < 4 * need:
            raise KvError(2, f"pull_staged: counters hold {counters.numel()} words, need {need}")
    S = (C.c_void_p * ns)(*[l.handle.value for l in src_layouts])
    RG = (C.c_void_p * len(rings))(*[_ptr(r) for r in rings])
    RF = (C.c_void_p * ns)(*[_ptr(f) for f in ready_flags])
    FF = (C.c_void_p * ns)(*[_ptr(f) for f in free_flags])
    lb, le = layer_range if layer_range else _common(src_layouts[0], dst_layout)
    check(lib.kv_pull_staged(ns, S, RG, ring_slots, slot_bytes, dst_layout.handle, _ptr(dst_pool),
                             C.byref(dst_batch.bt), RF, FF, _ptr(counters), seq0, lb, le, layer_chunk,
                             int(timeout_s * 1e9), _ptr(err), _stream(stream)))


def chunk_count(layer_range, layer_chunk):
    """kv_chunk_count: chunks a kv_stage / kv_pull_staged call over layer_range takes (the
    ramped schedule; seq0 advances by it)."""
    lb, le = layer_range
    return int(lib.kv_chunk_count(int(lb), int(le), int(layer_chunk)))


def pull_counter_words(layer_range, layer_chunk):
    """Device scratch words kv_pull_staged's persistent kernel needs: 2 per chunk + 1."""
    return 2 * chunk_count(layer_range, layer_chunk) + 1


def compute_scales(src_layouts, src_pools, src_batch: Batch, dst_layout: Layout, out, layer_range=None, stream=None):
    """kv_compute_scales: per-batch fp8 dequant scales amax/448 for dst_layout's heads,
    written into `out` (device float32 [L][2][H_d])."""
    ns = len(src_layouts)
    S = (C.c_void_p * ns)(*[l.handle.value for l in src_layouts])
    SP = (C.c_void_p * ns)(*[_ptr(p) for p in src_pools])
    lb, le = layer_range if layer_range else _common(src_layouts[0], dst_layout)
    check(lib.kv_compute_scales(ns, S, SP, C.byref(src_batch.bt), dst_layout.handle, _ptr(out), lb, le,
                                _stream(stream)))


def wire_dtype(src: Layout, dst: Layout):
    return lib.kv_wire_dtype(src.handle, dst.handle)


def wire_bytes(src: Layout, dst: Layout, total_tokens, layer_range=None):
    lb, le = layer_range if layer_range else _common(src, dst)
    return lib.kv_wire_bytes(src.handle, dst.handle, int(total_tokens), lb, le)


def pack(src: Layout, src_pool, src_batch: Batch, dst: Layout, wire, layer_range=None, stream=None, wire_nbytes=None):
    """kv_pack: Fig. 5 flatten of the (src rank -> dst rank) share into `wire`."""
    lb, le = layer_range if layer_range else _common(src, dst)
    nb = wire_nbytes if wire_nbytes is not None else wire.numel() * wire.element_size()
    check(lib.kv_pack(src.handle, _ptr(src_pool), C.byref(src_batch.bt), dst.handle, lb, le, _ptr(wire), nb,
                      _stream(stream)))


def unpack(src: Layout, dst: Layout, dst_pool, dst_batch: Batch, wire, layer_range=None, stream=None,
           wire_nbytes=None):
    """kv_unpack: Fig. 5 restore of a wire buffer into the D pool (+ tail zero-fill)."""
    lb, le = layer_range if layer_range else _common(src, dst)
    nb = wire_nbytes if wire_nbytes is not None else wire.numel() * wire.element_size()
    check(lib.kv_unpack(src.handle, dst.handle, _ptr(dst_pool), C.byref(dst_batch.bt), lb, le, _ptr(wire), nb,
                        _stream(stream)))


class Comm:
    """NCCL communicator owned by libkvx (kv_comm_*); the unique id travels through the
    caller's control plane (e.g. torch.distributed broadcast_object_list)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib.kv_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, nranks, rank, uid: bytes, device: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        check(lib.kv_comm_init(nranks, rank, buf, device, C.byref(h)))
        self._h = h
        self.nranks, self.rank = nranks, rank

    def send(self, peer, wire, nbytes=None, stream=None):
        nb = nbytes if nbytes is not None else wire.numel() * wire.element_size()
        check(lib.kv_send(self._h, peer, _ptr(wire), nb, _stream(stream)))

    def recv(self, peer, wire, nbytes=None, stream=None):
        nb = nbytes if nbytes is not None else wire.numel() * wire.element_size()
        check(lib.kv_recv(self._h, peer, _ptr(wire), nb, _stream(stream)))

    def recv_unpack(self, peer, wire, nbytes, src: Layout, dst: Layout, dst_pool, dst_batch: Batch,
                    layer_range=None, stream=None):
        lb, le = layer_range if layer_range else _common(src, dst)
        check(lib.kv_recv_unpack(self._h, peer, _ptr(wire), nbytes, src.handle, dst.handle, _ptr(dst_pool),
                                 C.byref(dst_batch.bt), lb, le, _stream(stream)))

    def send_pipelined(self, src: Layout, src_pool, src_batch: Batch, dst_layouts, peer_ranks, wires, wire_cap,
                       layer_chunk, layer_range=None, stream=None, pack_stream=None, send_stream=None):
        """kv_send_pipelined: pack chunk k+1 while chunk k is on the wire (wires: 2 per peer)."""
        nd = len(dst_layouts)
        Dl = (C.c_void_p * nd)(*[l.handle.value for l in dst_layouts])
        PR = (C.c_int32 * nd)(*peer_ranks)
        W = (C.c_void_p * (2 * nd))(*[_ptr(w) for w in wires])
        lb, le = layer_range if layer_range else _common(src, dst_layouts[0])
        check(lib.kv_send_pipelined(self._h, src.handle, _ptr(src_pool), C.byref(src_batch.bt), nd, Dl, PR, W,
                                    wire_cap, lb, le, layer_chunk, _stream(stream), _stream(pack_stream),
                                    _stream(send_stream)))

    def recv_pipelined(self, src_layouts, peer_ranks, dst: Layout, dst_pool, dst_batch: Batch, wires, wire_cap,
                       layer_chunk, layer_range=None, stream=None, recv_stream=None, unpack_stream=None):
        """kv_recv_pipelined: receive chunk k+1 while chunk k is unpacked (wires: 2 per peer)."""
        ns = len(src_layouts)
        S = (C.c_void_p * ns)(*[l.handle.value for l in src_layouts])
        PR = (C.c_int32 * ns)(*peer_ranks)
        W = (C.c_void_p * (2 * ns))(*[_ptr(w) for w in wires])
        lb, le = layer_range if layer_range else _common(src_layouts[0], dst)
        check(lib.kv_recv_pipelined(self._h, ns, S, PR, dst.handle, _ptr(dst_pool), C.byref(dst_batch.bt), W,
                                    wire_cap, lb, le, layer_chunk, _stream(stream), _stream(recv_stream),
                                    _stream(unpack_stream)))

    @staticmethod
    @contextmanager
    def group():
        check(lib.kv_comm_group_start())
        try:
            yield
        finally:
            check(lib.kv_comm_group_end())

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.kv_comm_destroy(self._h)
            self._h = None


def ipc_export(tensor):
    """kv_ipc_export -> (64-byte handle, offset of the tensor inside its allocation)."""
    h = (C.c_uint8 * 64)()
    off = C.c_uint64()
    check(lib.kv_ipc_export(_ptr(tensor), h, C.byref(off)))
    return bytes(h), off.value


def ipc_open(handle: bytes, offset: int) -> int:
    """kv_ipc_open -> peer-mapped device address (int) of the exporter's pointer."""
    h = (C.c_uint8 * 64).from_buffer_copy(handle)
    out = C.c_void_p()
    check(lib.kv_ipc_open(h, offset, C.byref(out)))
    return out.value


def ipc_close(mapped_ptr: int, offset: int):
    check(lib.kv_ipc_close(mapped_ptr - offset))


def peer_enable(peer_device: int):
    """kv_peer_enable: the current device may access peer_device's memory (single process)."""
    check(lib.kv_peer_enable(peer_device))


def signal(flag, value, stream=None):
    check(lib.kv_signal(_ptr(flag), value, _stream(stream)))


def wait(flag, value, err, timeout_s=10.0, stream=None):
    check(lib.kv_wait(_ptr(flag), value, int(timeout_s * 1e9), _ptr(err), _stream(stream)))


def preload():
    """kv_preload: load every library kernel on the current device (see include/kvx.h)."""
    check(lib.kv_preload())


def verify_fill(src: Layout, src_pool, src_batch: Batch, dst_layouts, seed, err, req_ids=None, stream=None):
    """kv_verify_fill (K6): hash-derived values, exact under the cast, in every valid element."""
    nd = len(dst_layouts)
    Dl = (C.c_void_p * nd)(*[l.handle.value for l in dst_layouts])
    check(lib.kv_verify_fill(src.handle, _ptr(src_pool), C.byref(src_batch.bt), nd, Dl, _ptr(req_ids), int(seed),
                             _ptr(err), _stream(stream)))


def verify_check(src: Layout, dst: Layout, dst_pool, dst_batch: Batch, seed, result, scratch, canary=0xA5,
                 req_ids=None, stream=None):
    """kv_verify_check (K6): count mismatches of a whole D pool after a transfer of a K6 fill.
    result: device int64[8] ([0] value, [1] tail, [2] canary mismatches, [3] checked)."""
    check(lib.kv_verify_check(src.handle, dst.handle, _ptr(dst_pool), C.byref(dst_batch.bt), _ptr(req_ids),
                              int(seed), canary, _ptr(scratch), scratch.numel(), _ptr(result), _stream(stream)))


def memcpy_engine(dst, src, nbytes, stream=None):
    """kv_memcpy_engine: copy-engine (peer) copy -- the bench's NVLink ceiling, not the path."""
    check(lib.kv_memcpy_engine(_ptr(dst), _ptr(src), int(nbytes), _stream(stream)))


def copy_bytes(dst, src, nbytes, stream=None):
    """kv_copy_bytes: SM-driven opaque byte copy (hidden state)."""
    check(lib.kv_copy_bytes(_ptr(dst), _ptr(src), int(nbytes), _stream(stream)))


def launch_count():
    return lib.kv_launch_count()


def last_kernel() -> str:
    """kv_last_kernel: the data-path kernel this thread's last convert/pack/unpack launched."""
    return lib.kv_last_kernel().decode()


def set_sm_budget(n_sms: int) -> int:
    """kv_set_sm_budget: cap the SMs later data-path launches may use (0 = all)."""
    return lib.kv_set_sm_budget(int(n_sms))


def launch_count_reset():
    lib.kv_launch_count_reset()
