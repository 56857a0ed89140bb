"""Transfers replayable from files (NEXT-2): a file is the self-describing
wire header (kv_wire_header_write, byte layout in include/kvx.h) followed by the kv_pack
payload (Fig. 5 canonical order).  Loading checks the header against the receiver's
layouts (kv_wire_header_check) before kv_unpack restores it into the D pool.

Also the first-token hidden state that travels with the KV (P:95 steps 3/5; opaque
bytes): ``copy_hidden`` is kv_copy_bytes, a device (or peer) byte copy."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import WireInfo, check, lib
from .kv import Batch, Layout, _common, _ptr, _stream, pack, unpack, wire_bytes


def header(src: Layout, dst: Layout, n_tokens, layer_range=None) -> bytes:
    lb, le = layer_range if layer_range else _common(src, dst)
    nt = np.ascontiguousarray(np.asarray(n_tokens, dtype=np.int32))
    n = lib.kv_wire_header_bytes(len(nt))
    buf = (C.c_uint8 * n)()
    check(lib.kv_wire_header_write(src.handle, dst.handle, len(nt), nt.ctypes.data, lb, le, buf, n))
    return bytes(buf)


def parse(hdr: bytes) -> dict:
    info = WireInfo()
    b = (C.c_uint8 * len(hdr)).from_buffer_copy(hdr)
    check(lib.kv_wire_header_parse(b, len(hdr), C.byref(info)))
    out = {f: getattr(info, f) for f, _ in WireInfo._fields_ if f != "n_tokens"}
    out["n_tokens"] = [info.n_tokens[i] for i in range(info.n_req)]
    return out


def check_header(hdr: bytes, src: Layout, dst: Layout, n_tokens, layer_range=None):
    lb, le = layer_range if layer_range else _common(src, dst)
    nt = np.ascontiguousarray(np.asarray(n_tokens, dtype=np.int32))
    b = (C.c_uint8 * len(hdr)).from_buffer_copy(hdr)
    check(lib.kv_wire_header_check(b, len(hdr), src.handle, dst.handle, len(nt), nt.ctypes.data, lb, le))


def save(path, src: Layout, src_pool, src_batch: Batch, dst: Layout, layer_range=None, stream=None):
    """Pack the (src rank -> dst rank) share on the device and write header + payload."""
    import torch
    nb = wire_bytes(src, dst, src_batch.total_tokens, layer_range)
    wire = torch.empty(max(nb, 16), dtype=torch.uint8, device=src_pool.device if hasattr(src_pool, "device") else "cuda")
    pack(src, src_pool, src_batch, dst, wire, layer_range, stream, wire_nbytes=nb)
    torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
    hdr = header(src, dst, src_batch.n_tokens, layer_range)
    with open(path, "wb") as f:
        f.write(hdr)
        f.write(wire[:nb].cpu().numpy().tobytes())
    return nb


def load(path, src: Layout, dst: Layout, dst_pool, dst_batch: Batch, layer_range=None, stream=None):
    """Read a saved transfer, check its header against (src, dst, dst_batch, layers) and
    restore it into dst_pool with kv_unpack."""
    import torch
    with open(path, "rb") as f:
        blob = f.read()
    n_req = int.from_bytes(blob[56:60], "little")
    hlen = lib.kv_wire_header_bytes(n_req)
    hdr = blob[:hlen]
    check_header(hdr, src, dst, dst_batch.n_tokens, layer_range)
    payload = np.frombuffer(blob, dtype=np.uint8, offset=hlen)
    wire = torch.from_numpy(payload.copy()).to(dst_pool.device if hasattr(dst_pool, "device") else "cuda")
    unpack(src, dst, dst_pool, dst_batch, wire, layer_range, stream, wire_nbytes=len(payload))
    return parse(hdr)


def copy_hidden(dst, src, nbytes=None, stream=None):
    """kv_copy_bytes: opaque device / peer byte copy (first-token hidden state)."""
    n = nbytes if nbytes is not None else src.numel() * src.element_size()
    check(lib.kv_copy_bytes(_ptr(dst), _ptr(src), n, _stream(stream)))
