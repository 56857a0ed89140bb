"""Pipeline-stage reshard (NEXT-2; SPEC S:289 rejected pp_p != pp_d -- this build supports
it by layer-range intersection).  A pool holds the global layers [first_layer, first_layer
+ L); a transfer is one call per overlapping (P stage, D stage) pair over the intersection.

Pins: (1) O1 per stage pair == O2 over all stages at once (O2 keys the logical tensor by
global layer, source-driven); (2) special case: with the P layout's LAYER axis outermost,
the P stage pools concatenated ARE the unstaged pool, and the staged transfer must equal
the unstaged one byte for byte."""
import numpy as np
import pytest

import synth
from oracle import bruteforce as o2
from synth import BF16, E4M3, F16
from tests.kvcase import make_case

P_STAGES = [(0, 2), (2, 4)]
D_STAGES = [(0, 3), (3, 4)]


def _staged(case, stages, side):
    """Split a case's layouts into pipeline stages (fresh pools for the P side)."""
    lays = case[f"{side}_lays"]
    out = []
    for (f, e) in stages:
        for lay in lays:
            d = dict(lay)
            d["first_layer"], d["L"] = f, e - f
            if d.get("scales") is not None:
                d["scales"] = np.asarray(lay["scales"])[f:e]
            out.append(d)
    return out


def _pools_for(lays, seed, dtype, canary=False):
    pools = []
    for i, d in enumerate(lays):
        n = 2 * d["L"] * d["NB"] * d["B"] * (d["H"] // d["tp"]) * d["D"]
        if canary:
            pools.append(np.full(n * synth.NBYTES[dtype], synth.CANARY, np.uint8).view(
                {1: np.uint8, 2: np.uint16, 4: np.uint32}[synth.NBYTES[dtype]]))
        else:
            pools.append(synth.random_finite_bits(seed + i, n, dtype))
    return pools


def staged_transfer(o1, src_lays, src_pools, dst_lays, dst_pools, n_tokens, st, dt):
    """One O1 call per (P stage, D stage) pair with overlapping layers."""
    tp_p = src_lays[0]["tp"]
    for sf in sorted({d.get("first_layer", 0) for d in src_lays}):
        S = [d for d in src_lays if d.get("first_layer", 0) == sf]
        SP = [p for d, p in zip(src_lays, src_pools) if d.get("first_layer", 0) == sf]
        assert len(S) == tp_p
        for df in sorted({d.get("first_layer", 0) for d in dst_lays}):
            idx = [i for i, d in enumerate(dst_lays) if d.get("first_layer", 0) == df]
            lb, le = max(sf, df), min(sf + S[0]["L"], df + dst_lays[idx[0]]["L"])
            if lb < le:
                o1.convert(S, SP, [dst_lays[i] for i in idx], [dst_pools[i] for i in idx], n_tokens, st, dt, (lb, le))


@pytest.mark.parametrize("tp_p,tp_d,sdt,ddt", [(2, 1, F16, F16), (1, 2, BF16, E4M3), (2, 2, BF16, F16)])
def test_staged_o1_equals_o2(o1, tp_p, tp_d, sdt, ddt):
    base = make_case(4, 4, 4, tp_p, tp_d, 2, 4, [5, 3], sdt, ddt, seed=tp_p * 10 + tp_d, o1=None,
                     tail_garbage=False, scales="pow2")
    src = _staged(base, P_STAGES, "src")
    dst = _staged(base, D_STAGES, "dst")
    sp = _pools_for(src, 100, sdt)
    dp = _pools_for(dst, 0, ddt, canary=True)
    got = [p.copy() for p in dp]
    staged_transfer(o1, src, sp, dst, got, base["n_tokens"], base["src_tables"], base["dst_tables"])
    want = [p.tolist() for p in dp]
    o2.convert(src, [p.tolist() for p in sp], dst, want, base["n_tokens"], base["src_tables"], base["dst_tables"])
    for g, w in zip(got, want):
        assert g.tolist() == w


def test_staged_equals_unstaged_when_layer_outermost(o1):
    base = make_case(4, 4, 8, 2, 1, 4, 8, [9, 4], BF16, BF16, seed=3, o1=o1)
    whole = [p.copy() for p in base["dst_pools"]]
    o1.convert(base["src_lays"], base["src_pools"], base["dst_lays"], whole, base["n_tokens"],
               base["src_tables"], base["dst_tables"])
    src = _staged(base, P_STAGES, "src")
    # slice each rank's unstaged pool (LAYER outermost in synth.P_ORDER) into its stages
    sp = []
    for (f, e) in P_STAGES:
        for p, lay in enumerate(base["src_lays"]):
            per_layer = len(base["src_pools"][p]) // lay["L"]
            sp.append(base["src_pools"][p][f * per_layer:e * per_layer].copy())
    got = [p.copy() for p in base["dst_pools"]]
    staged_transfer(o1, src, sp, base["dst_lays"], got, base["n_tokens"], base["src_tables"], base["dst_tables"])
    for g, w in zip(got, whole):
        assert np.array_equal(g, w)


def test_layer_range_outside_stage_is_error(o1):
    base = make_case(4, 2, 4, 1, 1, 2, 2, [3], F16, F16, seed=1, o1=None, tail_garbage=False)
    src = _staged(base, [(0, 2)], "src")
    with pytest.raises(ValueError):
        o1.convert(src, _pools_for(src, 0, F16), base["dst_lays"], [p.copy() for p in base["dst_pools"]],
                   base["n_tokens"], base["src_tables"], base["dst_tables"], (1, 3))
