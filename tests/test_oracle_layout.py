"""Pins for the oracle's layout / block-size / TP re-shard mapping (A2, A4-A9).

O1 is tied to: the SPEC/paper worked examples (tests/golden/), the numpy
transpose special case (identity tables, one request, TP 1->1, same dtype:
converting layouts is exactly ``np.transpose``), the brute-force O2 (source-driven
enumeration through inverse block tables), coordinate-code conservation over
SPEC S:532's grid (every logical element lands exactly once, tails zero, every
other byte keeps its canary), round trips, chunk invariance and the never-read
source tail.
"""
import itertools
import os

import numpy as np
import pytest

import synth
from oracle import bruteforce as o2
from synth import BF16, E4M3, F16, LAYER, KV, BLOCK, SLOT, HEAD, DIM
from tests.kvcase import coord_fill, expected, logical_code, make_case

HERE = os.path.dirname(os.path.abspath(__file__))
ALL_ORDERS = list(itertools.permutations(range(6)))


def _golden(name):
    with open(os.path.join(HERE, "golden", name)) as f:
        return [ln.strip() for ln in f if ln.strip() and not ln.startswith("#")]


def test_kv_bytes_golden(o1):
    for row in _golden("kv_bytes.txt"):
        parts = row.split()
        L, H, D, T, s, want = map(int, parts[1:7])
        assert o1.kv_bytes(L, H, D, T, s) == want


def test_flatten_length_is_kv_size_formula(o1):
    """The Fig. 5 1-D tensor of a TP1->1 transfer holds exactly 2*L*H*D*T elements."""
    case = make_case(3, 4, 8, 1, 1, 4, 8, [5, 9], F16, F16, seed=3, o1=o1)
    wire = o1.flatten(case["src_lays"][0], case["src_pools"][0], case["dst_lays"][0], case["n_tokens"],
                      case["src_tables"])
    assert wire.nbytes == o1.kv_bytes(3, 4, 8, 14, 2)


def test_plan_golden_p125(o1):
    for row in _golden("tp_plan.txt"):
        head, pairs = row.split(":")
        tp_p, tp_d, H = map(int, head.split())
        want = sorted(tuple(map(int, x.split("->"))) for x in pairs.split())
        got = sorted((p, q) for p, q, _, _ in o1.plan(tp_p, tp_d, H))
        assert got == want
        assert sorted(o2.plan(tp_p, tp_d, H).keys()) == want
        # partition: head ranges of each q cover [q*H_d, (q+1)*H_d) exactly once
        for q in range(tp_d):
            cov = sorted(h for p, qq, b, e in o1.plan(tp_p, tp_d, H) if qq == q for h in range(b, e))
            assert cov == list(range(q * H // tp_d, (q + 1) * H // tp_d))


def test_plan_rejects_non_divisor(o1):
    with pytest.raises(ValueError):
        o1.plan(3, 2, 8)
    with pytest.raises(ValueError):
        o2.plan(2, 3, 8)


def test_plan_general_intersection(o1):
    """Neither degree divides the other: 6 -> 4 over 12 heads still partitions."""
    pl = o1.plan(6, 4, 12)
    assert sorted((p, q) for p, q, _, _ in pl) == sorted(o2.plan(6, 4, 12).keys())
    assert sum(e - b for _, _, b, e in pl) == 12


@pytest.mark.parametrize("row", _golden("block_remap_6tok.txt"))
def test_block_remap_golden_s259(o1, row):
    head, body = row.split(":")
    Bp, Bd, nblk = map(int, head.split())
    kpart, vpart = body.split("|")
    want_k = [int(x, 16) for x in kpart.split()[1:]]
    want_v = [int(x, 16) for x in vpart.split()[1:]]
    order = (LAYER, KV, BLOCK, SLOT, HEAD, DIM)
    T = 6
    NBp = -(-T // Bp)
    src = synth.layout(1, 1, 1, 1, 0, Bp, NBp, F16, order)
    dst = synth.layout(1, 1, 1, 1, 0, Bd, nblk, F16, order)
    vals = [0x3C00, 0x4000, 0x4200, 0x4400, 0x4500, 0x4600]
    pool = np.full(2 * NBp * Bp, 0x7E01, dtype=np.uint16)  # NaN garbage in the source tail
    for c in range(2):
        pool[c * NBp * Bp:c * NBp * Bp + T] = vals
    for impl in ("o1", "o2"):
        out = np.full(2 * nblk * Bd, 0xA5A5, dtype=np.uint16)
        if impl == "o1":
            o1.convert([src], [pool], [dst], [out], [T], [list(range(NBp))], [list(range(nblk))])
        else:
            lst = out.tolist()
            o2.convert([src], [pool.tolist()], [dst], [lst], [T], [list(range(NBp))], [list(range(nblk))])
            out = np.array(lst, dtype=np.uint16)
        assert out[:nblk * Bd].tolist() == want_k, impl
        assert out[nblk * Bd:].tolist() == want_v, impl


def _transpose_expect(src_lay, src_pool, dst_order):
    ext = {LAYER: src_lay["L"], KV: 2, BLOCK: src_lay["NB"], SLOT: src_lay["B"], HEAD: src_lay["H"], DIM: src_lay["D"]}
    a = src_pool.reshape([ext[ax] for ax in src_lay["order"]])
    perm = [src_lay["order"].index(ax) for ax in dst_order]
    return np.ascontiguousarray(np.transpose(a, perm)).reshape(-1)


def _transpose_case(src_order, dst_order, seed):
    L, H, D, B, NB = 2, 3, 4, 2, 3
    src = synth.layout(L, H, D, 1, 0, B, NB, F16, src_order)
    dst = synth.layout(L, H, D, 1, 0, B, NB, F16, dst_order)
    pool = synth.random_finite_bits(seed, 2 * L * NB * B * H * D, F16)
    return src, dst, pool, NB * B


def test_numpy_transpose_all_dst_orders(o1):
    """Special case reducing to a library routine: every one of the 720 destination orders."""
    for i, dst_order in enumerate(ALL_ORDERS):
        src, dst, pool, T = _transpose_case(synth.P_ORDER, dst_order, i)
        out = np.zeros_like(pool)
        o1.convert([src], [pool], [dst], [out], [T], [list(range(3))], [list(range(3))])
        assert np.array_equal(out, _transpose_expect(src, pool, dst_order)), dst_order


def test_numpy_transpose_all_src_orders(o1):
    for i, src_order in enumerate(ALL_ORDERS):
        src, dst, pool, T = _transpose_case(src_order, synth.D_ORDER, 1000 + i)
        out = np.zeros_like(pool)
        o1.convert([src], [pool], [dst], [out], [T], [list(range(3))], [list(range(3))])
        assert np.array_equal(out, _transpose_expect(src, pool, synth.D_ORDER)), src_order


def _orders24():
    """SPEC S:532's 24 layouts: permutations of (layer, head, token(slot), dim) under (KV, BLOCK)."""
    return [(KV, BLOCK) + p for p in itertools.permutations((LAYER, HEAD, SLOT, DIM))]


def test_coordinate_conservation_s532_grid(o1):
    """Every logical (r,l,c,h,t,d) lands exactly at its destination; tail zero; canary elsewhere.

    Grid: (tp_p, tp_d) in {1,2,4,8}^2 x the 24 layouts x block sizes {2,4,8,16} on a 2-layer /
    8-head / 16-token model, with the layouts and block sizes rotated across cases."""
    orders = _orders24()
    blocks = [2, 4, 8, 16]
    k = 0
    for tp_p in (1, 2, 4, 8):
        for tp_d in (1, 2, 4, 8):
            for i, so in enumerate(orders):
                do = orders[(i * 7 + tp_p + tp_d) % 24]
                Bp, Bd = blocks[i % 4], blocks[(i // 4 + tp_d) % 4]
                n_tokens = [16] if k % 3 else [16, 11]
                k += 1
                case = make_case(2, 8, 2, tp_p, tp_d, Bp, Bd, n_tokens, F16, F16, so, do, seed=k,
                                 o1=o1, tail_garbage=False)
                T_max = coord_fill(case, o1)
                got = expected(case, o1)
                _check_coords(case, got, T_max)


def _check_coords(case, got, T_max):
    inv = {}
    for r, tab in enumerate(case["dst_tables"]):
        for j, b in enumerate(tab):
            inv[b] = (r, j)
    lay0 = case["dst_lays"][0]
    L, H, D = lay0["L"], lay0["H"], lay0["D"]
    for lay, pool in zip(case["dst_lays"], got):
        Hd = H // lay["tp"]
        for pos, ix in o2.positions(lay):
            v = int(pool[pos])
            if ix[BLOCK] not in inv:
                assert v == 0xA5A5
                continue
            r, j = inv[ix[BLOCK]]
            t = j * lay["B"] + ix[SLOT]
            if t >= case["n_tokens"][r]:
                assert v == 0
            else:
                h = lay["rank"] * Hd + ix[HEAD]
                assert v == logical_code(r, ix[LAYER], ix[KV], h, t, ix[DIM], L, H, T_max, D) + 1


@pytest.mark.parametrize("seed", range(24))
def test_o1_vs_o2_random(o1, seed):
    """O1 (dest-driven strides) == O2 (source-driven enumeration) on random tiny cases."""
    rng = np.random.default_rng(seed)
    tp_p, tp_d = rng.choice([1, 2, 4], size=2)
    Bp, Bd = rng.choice([1, 2, 3, 4, 8], size=2)
    src_dt, dst_dt = [(F16, F16), (F16, BF16), (BF16, F16), (BF16, E4M3), (F16, E4M3), (BF16, BF16)][seed % 6]
    n_tokens = [int(x) for x in rng.integers(1, 12, size=int(rng.integers(1, 4)))]
    so = ALL_ORDERS[int(rng.integers(720))]
    do = ALL_ORDERS[int(rng.integers(720))]
    case = make_case(2, 4, 3, int(tp_p), int(tp_d), int(Bp), int(Bd), n_tokens, src_dt, dst_dt, so, do,
                     seed=seed, o1=o1)
    want = expected(case, o1)
    lsts = [p.tolist() for p in case["dst_pools"]]
    o2.convert(case["src_lays"], [p.tolist() for p in case["src_pools"]], case["dst_lays"], lsts,
               case["n_tokens"], case["src_tables"], case["dst_tables"])
    for w, g in zip(want, lsts):
        assert w.tolist() == g


def test_source_tail_never_read(o1):
    """Garbage (NaN) vs zeros in source tail slots gives identical output."""
    a = make_case(2, 4, 8, 2, 1, 4, 8, [5, 7, 13], BF16, E4M3, seed=5, o1=o1, tail_garbage=True)
    b = make_case(2, 4, 8, 2, 1, 4, 8, [5, 7, 13], BF16, E4M3, seed=5, o1=o1, tail_garbage=False)
    assert any(not np.array_equal(x, y) for x, y in zip(a["src_pools"], b["src_pools"]))
    for x, y in zip(expected(a, o1), expected(b, o1)):
        assert np.array_equal(x, y)


def test_roundtrip_same_layout_identity(o1):
    """L -> L with identical tables is the identity on the valid region."""
    case = make_case(2, 4, 8, 2, 2, 4, 4, [9, 16], BF16, BF16, synth.P_ORDER, synth.P_ORDER, seed=9, o1=o1)
    case["dst_tables"] = case["src_tables"]
    for l in case["dst_lays"]:
        l["NB"] = case["src_lays"][0]["NB"]
    case["dst_pools"] = [p.copy() for p in case["src_pools"]]
    got = expected(case, o1)
    # valid region identical; source tails (NaN garbage) are zero-filled on the destination
    for q, (src, out) in enumerate(zip(case["src_pools"], got)):
        diff = np.nonzero(src != out)[0]
        assert np.all(out[diff] == 0)


def test_merge_then_split_is_identity(o1):
    """4 -> 2 (merge) then 2 -> 4 (split) returns the original shards, with layout and
    block-size changes on the way."""
    fwd = make_case(2, 8, 4, 4, 2, 4, 8, [7, 16, 3], F16, F16, synth.P_ORDER, synth.D_ORDER, seed=21, o1=o1)
    mid = expected(fwd, o1)
    back = dict(src_lays=fwd["dst_lays"], src_pools=mid, dst_lays=fwd["src_lays"],
                dst_pools=[np.zeros_like(p) for p in fwd["src_pools"]], n_tokens=fwd["n_tokens"],
                src_tables=fwd["dst_tables"], dst_tables=fwd["src_tables"])
    got = expected(back, o1)
    valid = dict(src_lays=fwd["src_lays"], src_pools=[np.ones_like(p) for p in fwd["src_pools"]],
                 dst_lays=fwd["src_lays"], dst_pools=[np.zeros_like(p) for p in fwd["src_pools"]],
                 n_tokens=fwd["n_tokens"], src_tables=fwd["src_tables"], dst_tables=fwd["src_tables"])
    mask = [m == 1 for m in expected(valid, o1)]  # positions of valid tokens
    for orig, g, m in zip(fwd["src_pools"], got, mask):
        assert np.array_equal(orig[m], g[m])


def test_layer_chunk_invariance(o1):
    """A10: converting layer chunks [0,1), [1,3), [3,4) equals converting all layers at once."""
    case = make_case(4, 4, 8, 2, 4, 4, 2, [6, 11], BF16, F16, seed=31, o1=o1)
    want = expected(case, o1)
    part = [p.copy() for p in case["dst_pools"]]
    for lr in ((0, 1), (1, 3), (3, 4)):
        o1.convert(case["src_lays"], case["src_pools"], case["dst_lays"], part, case["n_tokens"],
                   case["src_tables"], case["dst_tables"], lr)
    for w, g in zip(want, part):
        assert np.array_equal(w, g)


def test_flatten_restore_equals_convert(o1):
    """Fig. 5: flatten on P, restore on D, over every (p, q) pair == direct conversion."""
    case = make_case(2, 8, 4, 2, 4, 4, 8, [5, 12], BF16, E4M3, seed=41, o1=o1)
    want = expected(case, o1)
    got = [p.copy() for p in case["dst_pools"]]
    for p, q, _, _ in o1.plan(2, 4, 8):
        wire = o1.flatten(case["src_lays"][p], case["src_pools"][p], case["dst_lays"][q], case["n_tokens"],
                          case["src_tables"])
        o1.restore(case["src_lays"][p], case["dst_lays"][q], got[q], wire, case["n_tokens"], case["dst_tables"])
    for w, g in zip(want, got):
        assert np.array_equal(w, g)


def test_flatten_canonical_is_identity(o1):
    """a shard already in canonical order flattens to a byte-identical payload."""
    order = (LAYER, KV, HEAD, BLOCK, SLOT, DIM)
    L, H, D, B, NB = 2, 2, 4, 4, 3
    src = synth.layout(L, H, D, 1, 0, B, NB, BF16, order)
    dst = synth.layout(L, H, D, 1, 0, B, NB, BF16, order)
    pool = synth.random_finite_bits(5, 2 * L * H * NB * B * D, BF16)
    wire = o1.flatten(src, pool, dst, [NB * B], [list(range(NB))])
    assert np.array_equal(wire, pool)


def test_flatten_s222_eight_elements(o1):
    """2-layer, 2-head, 2-token, head_dim 1 shard stored (token, layer, head, dim):
    the canonical 1-D order is (layer, kv, head, token, dim), checked index by index."""
    order = (BLOCK, SLOT, LAYER, KV, HEAD, DIM)  # token-major storage
    src = synth.layout(2, 2, 1, 1, 0, 2, 1, F16, order)
    pool = np.arange(16, dtype=np.uint16) + 1
    wire = o1.flatten(src, pool, src, [2], [[0]])
    want = []
    for l in range(2):
        for c in range(2):
            for h in range(2):
                for t in range(2):
                    want.append(1 + ((t * 2 + l) * 2 + c) * 2 + h)  # position in (slot, layer, kv, head)
    assert wire.tolist() == want


def test_missing_source_shard_is_error(o1):
    case = make_case(1, 4, 2, 2, 1, 2, 2, [3], F16, F16, seed=1, o1=o1)
    with pytest.raises(ValueError, match="missing source rank 1"):
        o1.convert(case["src_lays"][:1], case["src_pools"][:1], case["dst_lays"], case["dst_pools"],
                   case["n_tokens"], case["src_tables"], case["dst_tables"])


# ---- NEXT-3 layout variants: K-only / V-only pools, x-split head_dim (reading 27) -------
HELD = {0: (0, 1), 1: (0,), 2: (1,)}


@pytest.mark.parametrize("i", range(0, 720, 37))
@pytest.mark.parametrize("kv_part,x", [(0, 4), (1, 8), (2, 1), (1, 2), (2, 8)])
def test_split_and_kv_part_numpy_special_case(o1, i, kv_part, x):
    """Identity tables, one request filling whole blocks, TP 1->1, same dtype: converting a
    canonical pool into a K-only / V-only pool with an x-split head_dim is numpy's
    select(K/V) -> reshape(D -> D/x, x) -> transpose(axis order, x innermost)."""
    L, H, D, B, NB = 2, 3, 8, 4, 3
    src = synth.layout(L, H, D, 1, 0, B, NB, F16, (LAYER, KV, BLOCK, SLOT, HEAD, DIM))
    order = ALL_ORDERS[i]
    dst = synth.layout(L, H, D, 1, 0, B, NB, F16, order, kv_part=kv_part, dim_split=x)
    X = np.arange(2 * L * NB * B * H * D, dtype=np.uint16).reshape(L, 2, NB, B, H, D)
    nkv = len(HELD[kv_part])
    out = np.full(nkv * L * NB * B * H * D, 0xA5A5, np.uint16)
    o1.convert([src], [X.reshape(-1)], [dst], [out], [NB * B], [list(range(NB))], [list(range(NB))])
    Y = X[:, list(HELD[kv_part])]                                   # (L, nkv, NB, B, H, D)
    Y = Y.reshape(L, nkv, NB, B, H, D // x, x)                       # split head_dim
    Y = np.transpose(Y, list(order) + [6])                          # Y's axes are canonical: axis id = position
    assert np.array_equal(out, Y.reshape(-1))


@pytest.mark.parametrize("seed", range(16))
def test_o1_vs_o2_layout_variants(o1, seed):
    """O1 == O2 on random tiny cases where either side is K-only / V-only / both and either
    side splits head_dim (only the K/V both sides hold is written; canary elsewhere)."""
    rng = np.random.default_rng(1000 + seed)
    tp_p, tp_d = rng.choice([1, 2], size=2)
    Bp, Bd = rng.choice([1, 2, 4], size=2)
    pk = int(rng.integers(0, 3))
    dk = int(rng.choice([k for k in range(3) if set(HELD[k]) & set(HELD[pk])]))
    px, dx = int(rng.choice([0, 2, 4])), int(rng.choice([0, 2, 4]))
    src_dt, dst_dt = [(F16, F16), (BF16, E4M3), (F16, BF16), (BF16, BF16)][seed % 4]
    n_tokens = [int(t) for t in rng.integers(1, 9, size=int(rng.integers(1, 3)))]
    case = make_case(2, 4, 4, int(tp_p), int(tp_d), int(Bp), int(Bd), n_tokens, src_dt, dst_dt,
                     ALL_ORDERS[int(rng.integers(720))], ALL_ORDERS[int(rng.integers(720))], seed=seed, o1=o1,
                     p_kv_part=pk, d_kv_part=dk, p_split=px, d_split=dx)
    want = expected(case, o1)
    lsts = [p.tolist() for p in case["dst_pools"]]
    o2.convert(case["src_lays"], [p.tolist() for p in case["src_pools"]], case["dst_lays"], lsts,
               case["n_tokens"], case["src_tables"], case["dst_tables"])
    for w, g in zip(want, lsts):
        assert w.tolist() == g


def test_k_and_v_pools_reassemble_the_combined_pool(o1):
    """Converting a K+V source into a K-only and a V-only destination (two calls) puts the
    same codes where one combined destination gets them: the K/V split is pure placement."""
    base = dict(L=2, H=4, D=8, tp_p=2, tp_d=1, B_p=4, B_d=8, n_tokens=[9, 3])
    args = (base["L"], base["H"], base["D"], base["tp_p"], base["tp_d"], base["B_p"], base["B_d"], base["n_tokens"],
            BF16, F16)
    both = make_case(*args, seed=5, o1=o1, d_order=(BLOCK, LAYER, KV, HEAD, SLOT, DIM))
    korder = (BLOCK, HEAD, DIM, SLOT, LAYER, KV)       # x-packed key cache style
    vorder = (BLOCK, HEAD, DIM, SLOT, LAYER, KV)       # head_dim before slot (value cache style)
    k = make_case(*args, seed=5, o1=o1, d_order=korder, d_kv_part=1, d_split=4)
    v = make_case(*args, seed=5, o1=o1, d_order=vorder, d_kv_part=2)
    wb, wk, wv = expected(both, o1)[0], expected(k, o1)[0], expected(v, o1)[0]
    B, NB = base["B_d"], both["dst_lays"][0]["NB"]
    for r, T in enumerate(base["n_tokens"]):
        for t in range(T):
            blk, slot = both["dst_tables"][r][t // B], t % B
            for l in range(2):
                for hl in range(4):
                    for d in range(8):
                        a = wb[o1.offset(both["dst_lays"][0], l, 0, blk, slot, hl, d)]
                        assert a == wk[o1.offset(k["dst_lays"][0], l, 0, blk, slot, hl, d)]
                        a = wb[o1.offset(both["dst_lays"][0], l, 1, blk, slot, hl, d)]
                        assert a == wv[o1.offset(v["dst_lays"][0], l, 1, blk, slot, hl, d)]
