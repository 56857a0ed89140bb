#!/usr/bin/env python
"""T3: small cases that launch every data-path kernel once, each checked against
O1, for running under compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tests/sanitize_cases.py convert
    compute-sanitizer --tool memcheck --error-exitcode 9 python tests/sanitize_cases.py transport

`convert`: k_tile_cast, k_convert_rows, k_tile_copy, k_requant_rows (both fp8 directions),
k_convert_tb (head_dim-major V, two heads per box, fp8 code tables; x-packed K), k_convert_tr8,
k_convert_tr, the generic element-wise k_convert, ragged / partial tail blocks on the tile
paths, k_pack / k_unpack (rows and generic), k_amax (kv_compute_scales) and the K6
k_verify_* kernels.  `transport`: the one-GPU staged pull (k_pack_rows -> k_pull_rows with
in-kernel flag waits) and the peer-store push (k_signal / k_wait); the waits time out rather
than hang if the tool serialises the streams.  Prints the kernels it saw; exits non-zero on
any mismatch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from synth import BF16, E4M3, F16, F32, FNUZ, LAYER, KV, BLOCK, SLOT, HEAD, DIM  # noqa: E402

VCOL = (LAYER, KV, BLOCK, HEAD, DIM, SLOT)


def _env(**kw):
    old = {k: os.environ.get(k) for k in kw}
    for k, v in kw.items():
        os.environ[k] = v

    def restore():
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return restore


def convert_cases(o1):
    import paper_2509_17542_b200 as kvx
    from tests.gpu_util import DevCase
    from tests.kvcase import expected, make_case
    from tests.test_gpu_parity import assert_pools_match
    seen = []

    def run(case, want_kernel, **env):
        restore = _env(**env)
        try:
            dc = DevCase(case)
            dc.convert()
            k = kvx.last_kernel()
        finally:
            restore()
        assert_pools_match(dc.dst_numpy(), expected(case, o1), case["dst_lays"][0]["dtype"])
        assert k == want_kernel, (k, want_kernel)
        seen.append(k)

    rng = np.random.default_rng(5)
    ragged = [40, 7, 0, 1, 33]
    run(make_case(2, 8, 64, 4, 2, 16, 16, ragged, BF16, E4M3, seed=1, o1=o1, scales="pow2"), "k_tile_cast")
    run(make_case(2, 8, 64, 4, 2, 16, 16, ragged, BF16, E4M3, seed=1, o1=o1, scales="pow2"), "k_convert_rows", KVX_TT="0")
    run(make_case(2, 8, 128, 2, 1, 16, 16, ragged, F16, F16, seed=2, o1=o1), "k_tile_copy", KVX_TILE="2")
    for s_, d_ in ((FNUZ, E4M3), (E4M3, FNUZ)):
        c = make_case(2, 8, 64, 2, 4, 16, 16, ragged, s_, d_, seed=3, o1=o1, scales="amax")
        for lay in c["src_lays"]:
            lay["scales"] = np.exp(rng.uniform(-3, 3, size=(2, 2, 4))).astype(np.float32)
        run(c, "k_requant_rows")
    for s_, d_, form in ((BF16, E4M3, "col"), (FNUZ, E4M3, "col"), (E4M3, FNUZ, "xpack"), (BF16, E4M3, "xpack")):
        c = make_case(2, 8, 128, 2, 4, 16, 16, ragged, s_, d_, VCOL, synth.D_ORDER, seed=4, o1=o1, scales="amax",
                      p_split=0 if form == "col" else 16 // synth.NBYTES[s_])
        if s_ in synth.FP8:
            for lay in c["src_lays"]:
                lay["scales"] = np.exp(rng.uniform(-3, 3, size=(2, 2, 4))).astype(np.float32)
        run(c, "k_convert_tb")
    c = make_case(2, 8, 64, 2, 1, 16, 32, ragged, BF16, E4M3, VCOL, synth.D_ORDER, seed=6, o1=o1, scales="pow2")
    run(c, "k_convert_tr8")
    run(c, "k_convert_tr", KVX_TR="0")
    run(make_case(2, 8, 16, 2, 2, 4, 8, ragged, F16, F32, (SLOT, KV, BLOCK, DIM, LAYER, HEAD),
                  (DIM, BLOCK, LAYER, KV, SLOT, HEAD), seed=7, o1=o1), "k_convert")
    # pack / unpack: fast rows and the generic orders
    for so, do, want in ((synth.P_ORDER, synth.D_ORDER, "k_pack_rows"),
                         ((SLOT, KV, BLOCK, DIM, LAYER, HEAD), synth.D_ORDER, "k_pack")):
        case = make_case(3, 8, 64, 4, 2, 16, 16, ragged, BF16, E4M3, so, do, seed=8, o1=o1, scales="pow2")
        dc = DevCase(case)
        for q, D in enumerate(dc.dst_lays):
            for p, S in enumerate(dc.src_lays):
                nb = kvx.wire_bytes(S, D, dc.src_bt.total_tokens)
                if nb == 0:
                    continue
                w = torch.empty(nb, dtype=torch.uint8, device="cuda")
                kvx.pack(S, dc.src_pools[p], dc.src_bt, D, w)
                assert kvx.last_kernel().startswith(want[:6]), kvx.last_kernel()
                seen.append(kvx.last_kernel())
                kvx.unpack(S, D, dc.dst_pools[q], dc.dst_bt, w)
                seen.append(kvx.last_kernel())
        torch.cuda.synchronize()
        assert_pools_match(dc.dst_numpy(), expected(case, o1), E4M3)
    # kv_compute_scales (amax)
    case = make_case(2, 8, 64, 2, 4, 16, 16, ragged, BF16, E4M3, seed=9, o1=o1, scales="amax")
    dc = DevCase(case)
    for q, D in enumerate(dc.dst_lays):
        out = torch.empty(2 * 2 * 2, dtype=torch.float32, device="cuda")
        kvx.compute_scales(dc.src_lays, dc.src_pools, dc.src_bt, D, out)
        want = o1.amax_scales(case["src_lays"], case["src_pools"], case["dst_lays"][q], case["n_tokens"],
                              case["src_tables"])
        assert np.array_equal(out.cpu().numpy().reshape(want.shape), want)
    seen.append("k_amax")
    # K6 fill + check
    case = make_case(2, 8, 64, 2, 2, 16, 16, ragged, BF16, E4M3, seed=10, o1=o1, scales="pow2")
    dc = DevCase(case)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    for S, P in zip(dc.src_lays, dc.src_pools):
        kvx.verify_fill(S, P, dc.src_bt, dc.dst_lays, 0x6B36, err)
    dc.convert()
    for q, D in enumerate(dc.dst_lays):
        res = torch.zeros(8, dtype=torch.int64, device="cuda")
        scratch = torch.empty(D.num_blocks, dtype=torch.uint8, device="cuda")
        kvx.verify_check(dc.src_lays[0], D, dc.dst_pools[q], dc.dst_bt, 0x6B36, res, scratch)
        torch.cuda.synchronize()
        r = res.cpu().numpy()
        assert r[0] == r[1] == r[2] == 0 and r[3] > 0, r
    assert int(err.item()) == 0
    seen.append("k_verify")
    return seen


def transport_cases(o1):
    from tests.test_gpu_transport import _case, _run
    from tests.kvcase import expected
    from tests.test_gpu_parity import assert_pools_match
    seen = []
    for mode, shape in (("pull_staged", "identity_fp8"), ("push", "merge"), ("pull", "merge")):
        case = _case(shape, o1)
        dc, ks = _run(o1, case, mode)
        assert_pools_match(dc.dst_numpy(), expected(case, o1), case["dst_lays"][0]["dtype"])
        seen += sorted(ks)
    return seen


def main():
    from oracle import o1
    o1.lib()
    import __graft_entry__ as g
    g.build()
    torch.cuda.set_device(0)
    what = sys.argv[1] if len(sys.argv) > 1 else "convert"
    seen = convert_cases(o1) if what == "convert" else transport_cases(o1)
    print(f"sanitize cases ({what}) ok: {sorted(set(seen))}", flush=True)


if __name__ == "__main__":
    main()
