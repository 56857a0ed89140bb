"""Child process of tests/test_gpu_guard_pools.py (`python -m tests.guard_pools GROUP`): every
P and D pool of a case lives in its own virtual-memory mapping (cuMemCreate / cuMemMap) of
exactly the pool's bytes, with reserved but UNMAPPED address space on both sides -- a read
or write one byte before or after any pool faults the kernel.  Pool sizes are chosen as
multiples of the mapping granularity so both ends are guarded.  Each case runs one
data-path kernel and compares D's pools with O1 (test infrastructure).  Stands in for the
compute-sanitizer memcheck of SURVEY T3, which this pool's GPUs do not allow; together with
the canary-filled D pools of every parity test (no stray write inside a pool) and
tests/guard_child.py (no read of a source tail slot)."""
import math
import os
import sys

import numpy as np


def _ck(res):
    err, *vals = res if isinstance(res, tuple) else (res,)
    if int(err) != 0:
        raise RuntimeError(f"CUDA driver error {err}")
    return vals[0] if len(vals) == 1 else (tuple(vals) or None)


class Guarded:
    """nbytes (a multiple of the granularity) mapped between two unmapped granules."""

    def __init__(self, cu, dev, nbytes):
        self.cu = cu
        prop = cu.CUmemAllocationProp()
        prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        prop.location.id = dev
        self.gran = g = int(_ck(cu.cuMemGetAllocationGranularity(
            prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM)))
        assert nbytes % g == 0, (nbytes, g)
        self.n = nbytes
        self.va = _ck(cu.cuMemAddressReserve(nbytes + 2 * g, 0, 0, 0))
        self.h = _ck(cu.cuMemCreate(nbytes, prop, 0))
        self.ptr = int(self.va) + g
        _ck(cu.cuMemMap(self.ptr, nbytes, 0, self.h, 0))
        acc = cu.CUmemAccessDesc()
        acc.location = prop.location
        acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        _ck(cu.cuMemSetAccess(self.ptr, nbytes, [acc], 1))

    @classmethod
    def tail(cls, cu, dev, nbytes, gran):
        """nbytes ending exactly at the end of a mapping (the next byte unmapped)."""
        g = cls(cu, dev, -(-nbytes // gran) * gran)
        g.ptr_end = g.ptr + g.n - nbytes
        return g

    def upload(self, arr):
        a = np.ascontiguousarray(arr).view(np.uint8)
        assert a.nbytes == self.n
        _ck(self.cu.cuMemcpyHtoD(self.ptr, a.ctypes.data, a.nbytes))

    def download(self, like):
        out = np.empty(self.n, dtype=np.uint8)
        _ck(self.cu.cuMemcpyDtoH(out.ctypes.data, self.ptr, self.n))
        return out.view(like.dtype)

    def free(self):
        _ck(self.cu.cuMemUnmap(self.ptr, self.n))
        _ck(self.cu.cuMemRelease(self.h))
        _ck(self.cu.cuMemAddressFree(self.va, self.n + 2 * self.gran))


def _nb_for(lay_fn, need, gran):
    """Smallest block count >= need whose pool is a multiple of the granularity."""
    per_block = lay_fn(1)
    step = gran // math.gcd(gran, per_block)
    return max(step, -(-need // step) * step)


def run_group(group):
    import torch
    from cuda.bindings import driver as cu

    import synth
    from synth import BF16, E4M3, F16, F32, FNUZ, LAYER, KV, BLOCK, SLOT, HEAD, DIM
    from tests.kvcase import expected, make_case
    from tests.test_gpu_parity import assert_pools_match
    from oracle import o1 as O1
    torch.zeros(1, device="cuda")
    import paper_2509_17542_b200 as kvx
    dev = torch.cuda.current_device()
    prop = cu.CUmemAllocationProp()
    prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = dev
    gran = int(_ck(cu.cuMemGetAllocationGranularity(
        prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM)))

    VCOL = (LAYER, KV, BLOCK, HEAD, DIM, SLOT)
    ragged = [40, 7, 0, 1, 33]
    # (name, L, H, D, tp_p, tp_d, Bp, Bd, sdt, ddt, p_order, d_order, p_split, env, want kernel)
    cases = {
        "tile": [
            ("tile_cast", 2, 8, 128, 4, 2, 16, 16, BF16, E4M3, synth.P_ORDER, synth.D_ORDER, 0, {}, "k_tile_cast"),
            ("rows", 2, 8, 128, 4, 2, 16, 16, BF16, E4M3, synth.P_ORDER, synth.D_ORDER, 0, {"KVX_TT": "0"},
             "k_convert_rows"),
            ("tile_copy", 2, 8, 128, 2, 1, 16, 16, F16, F16, synth.P_ORDER, synth.D_ORDER, 0, {"KVX_TILE": "2"},
             "k_tile_copy"),
            ("requant", 2, 8, 128, 2, 4, 16, 16, FNUZ, E4M3, synth.P_ORDER, synth.D_ORDER, 0, {}, "k_requant_rows"),
            ("requant_r", 2, 8, 128, 2, 4, 16, 16, E4M3, FNUZ, synth.P_ORDER, synth.D_ORDER, 0, {}, "k_requant_rows"),
        ],
        "vendor": [
            ("tb_v", 2, 8, 128, 2, 4, 16, 16, BF16, E4M3, VCOL, synth.D_ORDER, 0, {}, "k_convert_tb"),
            ("tb_v_fp8", 2, 8, 128, 2, 4, 16, 16, FNUZ, E4M3, VCOL, synth.D_ORDER, 0, {}, "k_convert_tb"),
            ("tb_k_fp8", 2, 8, 128, 2, 4, 16, 16, E4M3, FNUZ, VCOL, synth.D_ORDER, 16, {}, "k_convert_tb"),
            ("tb_k", 2, 8, 128, 2, 1, 16, 16, BF16, E4M3, VCOL, synth.D_ORDER, 8, {}, "k_convert_tb"),
            ("tr8", 2, 8, 128, 2, 1, 16, 32, BF16, E4M3, VCOL, synth.D_ORDER, 0, {}, "k_convert_tr8"),
            ("tr8_k", 2, 8, 128, 2, 4, 16, 16, FNUZ, E4M3, VCOL, synth.D_ORDER, 16, {}, "k_convert_tr8"),
            ("tr", 2, 8, 128, 2, 1, 16, 32, BF16, E4M3, VCOL, synth.D_ORDER, 0, {"KVX_TR": "0"}, "k_convert_tr"),
            ("generic", 2, 8, 16, 2, 2, 4, 8, F16, F32, (SLOT, KV, BLOCK, DIM, LAYER, HEAD),
             (DIM, BLOCK, LAYER, KV, SLOT, HEAD), 0, {}, "k_convert"),
        ],
    }.get(group, [])
    seen = []
    if group == "wire":
        # kv_pack from guarded P pools into a wire buffer that ends at an unmapped page,
        # kv_unpack from it into guarded D pools, kv_compute_scales over the guarded P pools
        for so, want in ((synth.P_ORDER, "k_pack_rows"), ((SLOT, KV, BLOCK, DIM, LAYER, HEAD), "k_pack")):
            L, H, D, tp_p, tp_d, B = 2, 8, 128, 4, 2, 16
            f = lambda dt, tp: (lambda nb: L * 2 * nb * B * (H // tp) * D * synth.NBYTES[dt])  # noqa: E731
            NB = max(_nb_for(f(BF16, tp_p), synth.pool_capacity(ragged, B), gran),
                     _nb_for(f(E4M3, tp_d), synth.pool_capacity(ragged, B), gran))
            case = make_case(L, H, D, tp_p, tp_d, B, B, ragged, BF16, E4M3, so, synth.D_ORDER, seed=60, o1=O1,
                             scales="amax", NB_p=NB, NB_d=NB)
            src_g = [Guarded(cu, dev, p.nbytes) for p in case["src_pools"]]
            dst_g = [Guarded(cu, dev, p.nbytes) for p in case["dst_pools"]]
            for g_, p in zip(src_g + dst_g, case["src_pools"] + case["dst_pools"]):
                g_.upload(p)
            S = [kvx.Layout.from_dict(lay) for lay in case["src_lays"]]
            Dl = [kvx.Layout.from_dict(lay, torch.from_numpy(np.asarray(lay["scales"], np.float32)).cuda())
                  for lay in case["dst_lays"]]
            sbt = kvx.Batch(S[0], ragged, case["src_tables"], "cuda")
            dbt = kvx.Batch(Dl[0], ragged, case["dst_tables"], "cuda")
            for q in range(tp_d):
                for p in range(tp_p):
                    nb = kvx.wire_bytes(S[p], Dl[q], sum(ragged))
                    if nb == 0:
                        continue
                    w = Guarded.tail(cu, dev, nb, gran)
                    kvx.pack(S[p], src_g[p].ptr, sbt, Dl[q], w.ptr_end, wire_nbytes=nb)
                    assert kvx.last_kernel() == want, kvx.last_kernel()
                    kvx.unpack(S[p], Dl[q], dst_g[q].ptr, dbt, w.ptr_end, wire_nbytes=nb)
                    torch.cuda.synchronize()
                    w.free()
                    seen += [want, kvx.last_kernel()]
            got = [g_.download(p) for g_, p in zip(dst_g, case["dst_pools"])]
            assert_pools_match(got, expected(case, O1), E4M3)
            for q in range(tp_d):
                out = torch.empty(L * 2 * (H // tp_d), dtype=torch.float32, device="cuda")
                kvx.compute_scales(S, [g_.ptr for g_ in src_g], sbt, Dl[q], out)
                want_sc = O1.amax_scales(case["src_lays"], case["src_pools"], case["dst_lays"][q], ragged,
                                         case["src_tables"])
                assert np.array_equal(out.cpu().numpy().reshape(want_sc.shape), want_sc)
            seen.append("k_amax")
            for g_ in src_g + dst_g:
                g_.free()
    for name, L, H, D, tp_p, tp_d, Bp, Bd, sdt, ddt, po, do, psplit, env, want_k in cases:
        nbytes = lambda dt, tp, B: (lambda nb: L * 2 * nb * B * (H // tp) * D * synth.NBYTES[dt])  # noqa: E731
        need_p = synth.pool_capacity(ragged, Bp)
        need_d = synth.pool_capacity(ragged, Bd)
        NB_p = _nb_for(nbytes(sdt, tp_p, Bp), need_p, gran)
        NB_d = _nb_for(nbytes(ddt, tp_d, Bd), need_d, gran)
        case = make_case(L, H, D, tp_p, tp_d, Bp, Bd, ragged, sdt, ddt, po, do, seed=len(seen) + 50, o1=O1,
                         scales="amax" if sdt not in synth.FP8 else "pow2", NB_p=NB_p, NB_d=NB_d, p_split=psplit)
        if sdt in synth.FP8:
            rng = np.random.default_rng(len(seen))
            for lay in case["src_lays"]:
                lay["scales"] = np.exp(rng.uniform(-2, 2, size=(L, 2, H // tp_p))).astype(np.float32)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            src_g = [Guarded(cu, dev, p.nbytes) for p in case["src_pools"]]
            dst_g = [Guarded(cu, dev, p.nbytes) for p in case["dst_pools"]]
            for g_, p in zip(src_g, case["src_pools"]):
                g_.upload(p)
            for g_, p in zip(dst_g, case["dst_pools"]):
                g_.upload(p)
            S = []
            for lay in case["src_lays"]:
                sc = None if lay.get("scales") is None else torch.from_numpy(np.asarray(lay["scales"], np.float32)).cuda()
                S.append(kvx.Layout.from_dict(lay, sc))
            Dl = []
            for lay in case["dst_lays"]:
                sc = None if lay.get("scales") is None else torch.from_numpy(np.asarray(lay["scales"], np.float32)).cuda()
                Dl.append(kvx.Layout.from_dict(lay, sc))
            sbt = kvx.Batch(S[0], ragged, case["src_tables"], "cuda")
            dbt = kvx.Batch(Dl[0], ragged, case["dst_tables"], "cuda")
            kvx.convert_reshard(S, [g_.ptr for g_ in src_g], sbt, Dl, [g_.ptr for g_ in dst_g], dbt)
            k = kvx.last_kernel()
            torch.cuda.synchronize()
            got = [g_.download(p) for g_, p in zip(dst_g, case["dst_pools"])]
            assert_pools_match(got, expected(case, O1), ddt)
            assert k == want_k, (name, k, want_k)
            seen.append(k)
            for g_ in src_g + dst_g:
                g_.free()
        finally:
            for k_, v in old.items():
                if v is None:
                    os.environ.pop(k_, None)
                else:
                    os.environ[k_] = v
    print("OK", group, seen, flush=True)


if __name__ == "__main__":
    run_group(sys.argv[1])
