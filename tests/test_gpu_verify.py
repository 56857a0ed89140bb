"""K6 (kv_verify_fill / kv_verify_check, the full-size conservation check of SURVEY 8(d))
pinned to the oracle: on small cases O1's output for K6-filled sources is exactly what
kv_verify_check expects (0 mismatches over the whole pool), the CUDA convert equals O1, and
single corrupted value / tail / canary elements are each counted once."""
import numpy as np
import pytest
import torch

from synth import BF16, E4M3, F16, F32, FNUZ
from tests.kvcase import expected, make_case

pytestmark = pytest.mark.gpu

SEED = 0x5EED


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g
    g.build()


def _k6_case(o1, args, kw):
    import paper_2509_17542_b200 as kvx
    from tests.gpu_util import DevCase, dev_to_np
    case = make_case(*args, o1=o1, **kw)
    dc = DevCase(case, "cuda:0")
    err = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    for p, lay in enumerate(dc.src_lays):
        kvx.verify_fill(lay, dc.src_pools[p], dc.src_bt, dc.dst_lays, SEED, err)
    torch.cuda.synchronize()
    assert int(err.item()) == 0, "K6 could not make a value exact"
    # the oracle's input: the K6-filled source pools, read back
    for p, lay in enumerate(case["src_lays"]):
        case["src_pools"][p] = dev_to_np(dc.src_pools[p], lay["dtype"]).copy()
    return case, dc


def _check(kvx, dc, q, pool=None):
    res = torch.zeros(8, dtype=torch.int64, device="cuda:0")
    scratch = torch.empty(dc.dst_lays[q].num_blocks, dtype=torch.uint8, device="cuda:0")
    kvx.verify_check(dc.src_lays[0], dc.dst_lays[q], dc.dst_pools[q] if pool is None else pool, dc.dst_bt, SEED, res,
                     scratch)
    torch.cuda.synchronize()
    return [int(x) for x in res.cpu()]


CASES = {
    "f16_same_merge": ((3, 8, 64, 4, 2, 16, 32, [100, 3, 0, 33], F16, F16), {"seed": 61}),
    "bf16_e4m3_merge": ((3, 8, 128, 4, 2, 16, 16, [70, 17], BF16, E4M3), {"seed": 62, "scales": "pow2"}),
    "bf16_fnuz_split": ((2, 8, 64, 2, 4, 16, 32, [40, 9], BF16, FNUZ), {"seed": 63, "scales": "pow2"}),
    "f16_bf16_c1": ((2, 2, 64, 1, 1, 16, 32, [32], F16, BF16), {"seed": 64}),
    "bf16_f32": ((2, 4, 64, 2, 1, 16, 16, [20, 13], BF16, F32), {"seed": 65}),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_k6_expectation_is_o1(o1, name):
    """O1 applied to the K6-filled sources gives pools that kv_verify_check passes in full;
    the CUDA convert gives the same pools."""
    import paper_2509_17542_b200 as kvx
    from tests.gpu_util import np_to_dev
    from tests.test_gpu_parity import assert_pools_match
    args, kw = CASES[name]
    case, dc = _k6_case(o1, args, kw)
    want = expected(case, o1)
    for q, w in enumerate(want):   # O1's pools, judged by K6
        r = _check(kvx, dc, q, np_to_dev(w, "cuda:0"))
        assert r[0] == r[1] == r[2] == 0, f"K6 disagrees with O1 on D{q}: {r}"
        assert r[3] == 2 * case["dst_lays"][q]["L"] * (case["dst_lays"][q]["H"] // case["dst_lays"][q]["tp"]) \
            * case["dst_lays"][q]["D"] * sum(case["n_tokens"])
    dc.convert()
    assert_pools_match(dc.dst_numpy(), want, case["dst_lays"][0]["dtype"])
    for q in range(len(want)):
        r = _check(kvx, dc, q)
        assert r[0] == r[1] == r[2] == 0, r


def test_k6_counts_single_faults(o1):
    """One flipped valid element, one non-zero tail slot, one overwritten canary byte: each
    counted exactly once in its own counter."""
    import paper_2509_17542_b200 as kvx
    from tests.gpu_util import np_to_dev
    args, kw = CASES["f16_same_merge"]
    case, dc = _k6_case(o1, args, kw)
    dc.convert()
    want = expected(case, o1)[0]
    lay = case["dst_lays"][0]
    base = dc.dst_numpy()[0]
    r0 = case["dst_tables"][0]
    # valid element: request 0, token 5, layer 1, V, head 2, dim 7
    i_val = o1.offset(lay, 1, 1, r0[5 // lay["B"]], 5 % lay["B"], 2, 7)
    # tail slot of request 1 (3 tokens in a 32-slot block): token 10
    r1 = case["dst_tables"][1]
    i_tail = o1.offset(lay, 0, 0, r1[0], 10, 0, 0)
    # a block no request uses
    used = {b for t in case["dst_tables"] for b in t}
    free_blk = min(set(range(lay["NB"])) - used)
    i_can = o1.offset(lay, 2, 0, free_blk, 0, 1, 3)
    for idx, slot in ((i_val, 0), (i_tail, 1), (i_can, 2)):
        g = base.copy()
        g[idx] ^= 0x0100
        r = _check(kvx, dc, 0, np_to_dev(g, "cuda:0"))
        want_counts = [0, 0, 0]
        want_counts[slot] = 1
        assert r[:3] == want_counts, (slot, r)
        assert slot == 2 or r[4] == idx + 1
    assert np.array_equal(base, want)
