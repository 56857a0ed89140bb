"""Child process of tests/test_gpu_tail_reads.py (run as `python -m tests.guard_child MODE`).

SPEC S:274 / reading 5: the source tail slots of a request's last block are never read.  The
P pool here is placed so that its last block -- (layer L-1, V, block NB_p - 1), a request's
partial last block with 8 valid slots of 16 -- ends its valid rows exactly at the end of a
virtual-memory mapping (cuMemCreate / cuMemMap, granularity-sized): the tail rows lie in a
reserved but UNMAPPED range, so any read of them faults the kernel.  Only the bytes before
that point hold the pool's data.  Each mode runs one data-path kernel over the batch and
compares D's pool with O1 (the oracle, test infrastructure); it prints "OK <kernel>".
A fault makes this process fail -- it runs in its own process so the parent's CUDA context
survives.

Modes: copy (same dtype, forced k_tile_copy), cast (bf16 -> e4m3, k_tile_cast), rows
(bf16 -> e4m3, forced row kernel), pack (k_pack_rows + k_unpack_rows), and each with the
suffix _slotmajor for a destination whose inner order is (SLOT, HEAD, DIM)."""
import os
import sys

import numpy as np


def _ck(res):
    """cuda-python returns (CUresult, *values): raise on an error, return the value(s)."""
    err, *vals = res if isinstance(res, tuple) else (res,)
    if int(err) != 0:
        raise RuntimeError(f"CUDA driver error {err}")
    return vals[0] if len(vals) == 1 else (tuple(vals) or None)


def main(mode):
    import torch
    from cuda.bindings import driver as cu

    import synth
    from tests.kvcase import expected, make_case, put_tail_garbage
    from tests.test_gpu_parity import assert_pools_match
    from oracle import o1 as O1

    base_mode, _, suffix = mode.partition("_")
    if base_mode == "copy":
        os.environ["KVX_TILE"] = "2"
    if base_mode == "rows":
        os.environ["KVX_TT"] = "0"
        os.environ["KVX_TILE"] = "0"
    ddt = synth.BF16 if base_mode == "copy" else synth.E4M3
    d_order = synth.D_ORDER if suffix != "slotmajor" else (synth.BLOCK, synth.LAYER, synth.KV, synth.SLOT,
                                                           synth.HEAD, synth.DIM)
    torch.zeros(1, device="cuda")   # primary context current on this thread
    import paper_2509_17542_b200 as kvx

    L, H, D, B = 2, 2, 128, 16
    nt = [40, 24]                   # both requests end in a partial block (8 of 16 slots)
    case = make_case(L, H, D, 1, 1, B, B, nt, synth.BF16, ddt, d_order=d_order, seed=91, o1=O1, scales="pow2",
                     tail_garbage=False)
    NB = case["src_lays"][0]["NB"]
    tabs = case["src_tables"]
    last = NB - 1                   # request 1's partial block -> the pool's last physical block
    for t in tabs:
        for i, b in enumerate(t):
            if b == last:
                t[i] = tabs[1][-1]
    tabs[1][-1] = last
    put_tail_garbage(case, O1)
    esize = 2
    valid = nt[1] - (len(tabs[1]) - 1) * B
    assert 0 < valid < B
    row = H * D * esize             # one slot's bytes in P_ORDER (L, KV, BLK, SLOT, H, D)
    pool = case["src_pools"][0].view(np.uint8)
    X = ((((L - 1) * 2 + 1) * NB + last) * B + valid) * row   # first byte of the tail rows
    assert X + (B - valid) * row == pool.nbytes

    prop = cu.CUmemAllocationProp()
    prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = torch.cuda.current_device()
    gran = int(_ck(cu.cuMemGetAllocationGranularity(
        prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM)))
    M = -(-X // gran) * gran
    va = _ck(cu.cuMemAddressReserve(M + 2 * gran, 0, 0, 0))
    handle = _ck(cu.cuMemCreate(M, prop, 0))
    _ck(cu.cuMemMap(va, M, 0, handle, 0))
    acc = cu.CUmemAccessDesc()
    acc.location = prop.location
    acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
    _ck(cu.cuMemSetAccess(va, M, [acc], 1))
    ptr = int(va) + M - X           # pool byte X == the end of the mapping
    host = np.ascontiguousarray(pool[:X])
    _ck(cu.cuMemcpyHtoD(ptr, host.ctypes.data, X))

    dev = "cuda"
    S = kvx.Layout.from_dict(case["src_lays"][0], None)
    dl = case["dst_lays"][0]
    sc = None if dl.get("scales") is None else torch.from_numpy(np.asarray(dl["scales"], np.float32)).to(dev)
    Dl = kvx.Layout.from_dict(dl, sc)
    sbt = kvx.Batch(S, nt, tabs, dev)
    dbt = kvx.Batch(Dl, nt, case["dst_tables"], dev)
    dpool = torch.from_numpy(case["dst_pools"][0].view(np.uint8).copy()).to(dev)
    if base_mode == "pack":
        nb = kvx.wire_bytes(S, Dl, sum(nt))
        wire = torch.empty(nb, dtype=torch.uint8, device=dev)
        kvx.pack(S, ptr, sbt, Dl, wire)
        k = kvx.last_kernel()
        kvx.unpack(S, Dl, dpool, dbt, wire)
    else:
        kvx.convert_reshard([S], [ptr], sbt, [Dl], [dpool], dbt)
        k = kvx.last_kernel()
    torch.cuda.synchronize()
    want = expected(case, O1)
    got = [dpool.cpu().numpy().view(case["dst_pools"][0].dtype)]
    assert_pools_match(got, want, ddt)
    want_k = {"copy": "k_tile_copy", "cast": "k_tile_cast", "rows": "k_convert_rows", "pack": "k_pack"}[base_mode]
    assert k.startswith(want_k), (k, want_k)
    _ck(cu.cuMemUnmap(va, M))
    _ck(cu.cuMemRelease(handle))
    _ck(cu.cuMemAddressFree(va, M + 2 * gran))
    print("OK", k, f"gran={gran} X={X} mapped={M}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
