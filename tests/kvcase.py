"""Test-case builder shared by the oracle pins and the GPU parity tests.

Inputs come from ``synth`` (seeded; no method arithmetic).  The only layout
arithmetic used here -- placing NaN garbage into source tail slots and
coordinate codes into source pools -- goes through the oracle's ``offset``
(test infrastructure), never through the CUDA path.
"""
from __future__ import annotations

import numpy as np

import synth
from synth import BF16, E4M3, F16, F32, FNUZ, FP8, NBYTES

NPTYPE = {1: np.uint8, 2: np.uint16, 4: np.uint32}
NAN_GARBAGE = {F16: 0x7E01, BF16: 0x7FC1, E4M3: 0x7F, F32: 0x7FC00001, FNUZ: 0x80}


def make_case(L, H, D, tp_p, tp_d, B_p, B_d, n_tokens, src_dt, dst_dt, p_order=synth.P_ORDER,
              d_order=synth.D_ORDER, seed=0, contiguous=False, scales="amax", o1=None, tail_garbage=True,
              values="random", NB_p=None, NB_d=None, p_kv_part=0, d_kv_part=0, p_split=0, d_split=0):
    """Build src pools (random finite bits), canary dst pools, tables, layouts.

    scales: None | "amax" | "pow2" | float -- fp8 dequant scales for fp8 dst ranks."""
    NB_p = NB_p or synth.pool_capacity(n_tokens, B_p)
    NB_d = NB_d or synth.pool_capacity(n_tokens, B_d)
    src_tables = synth.block_tables(seed + 1, n_tokens, B_p, NB_p, contiguous)
    dst_tables = synth.block_tables(seed + 2, n_tokens, B_d, NB_d, contiguous)
    src_lays, src_pools = [], []
    for p in range(tp_p):
        lay = synth.layout(L, H, D, tp_p, p, B_p, NB_p, src_dt, p_order, kv_part=p_kv_part, dim_split=p_split)
        n = (1 if p_kv_part else 2) * L * NB_p * B_p * (H // tp_p) * D
        if values == "random":
            pool = synth.random_finite_bits(seed + 100 + p, n, src_dt)
        elif values == "zeros":
            pool = np.zeros(n, dtype=NPTYPE[NBYTES[src_dt]])
        else:
            raise ValueError(values)
        src_lays.append(lay)
        src_pools.append(pool)
    dst_lays, dst_pools = [], []
    for q in range(tp_d):
        sc = None
        if dst_dt in FP8 and scales is not None:
            Hd = H // tp_d
            if scales == "pow2":
                sc = synth.pow2_scales(seed + 200 + q, L, Hd)
            elif scales == "amax":
                rng = np.random.default_rng(seed + 300 + q)
                # random finite 2-byte inputs span huge ranges; pick scales that put a good share in range
                sc = np.exp(rng.uniform(np.log(1e-3), np.log(1e3), size=(L, 2, Hd))).astype(np.float32)
            else:
                sc = np.full((L, 2, Hd), float(scales), dtype=np.float32)
        lay = synth.layout(L, H, D, tp_d, q, B_d, NB_d, dst_dt, d_order, sc, kv_part=d_kv_part, dim_split=d_split)
        n = (1 if d_kv_part else 2) * L * NB_d * B_d * (H // tp_d) * D
        pool = np.full(n * NBYTES[dst_dt], synth.CANARY, dtype=np.uint8).view(NPTYPE[NBYTES[dst_dt]])
        dst_lays.append(lay)
        dst_pools.append(pool)
    case = dict(src_lays=src_lays, src_pools=src_pools, dst_lays=dst_lays, dst_pools=dst_pools,
                n_tokens=list(n_tokens), src_tables=src_tables, dst_tables=dst_tables)
    if tail_garbage and o1 is not None:
        put_tail_garbage(case, o1)
    return case


def held(lay):
    """Global K/V indices a pool holds (kv_part 0: both, 1: K only, 2: V only)."""
    return {0: (0, 1), 1: (0,), 2: (1,)}[lay.get("kv_part", 0)]


def put_tail_garbage(case, o1):
    """NaN garbage in every source tail slot (never to be read: SPEC S:274, reading 5)."""
    for lay, pool in zip(case["src_lays"], case["src_pools"]):
        B = lay["B"]
        g = NAN_GARBAGE[lay["dtype"]]
        for r, T in enumerate(case["n_tokens"]):
            tab = case["src_tables"][r]
            for t in range(T, len(tab) * B):
                blk, slot = tab[t // B], t % B
                for l in range(lay["L"]):
                    for c in held(lay):
                        for hl in range(lay["H"] // lay["tp"]):
                            for d in range(lay["D"]):
                                pool[o1.offset(lay, l, c, blk, slot, hl, d)] = g


def expected(case, o1, layer_range=None):
    """O1's destination pools for the case (copies; the case's own pools are untouched)."""
    dst = [p.copy() for p in case["dst_pools"]]
    o1.convert(case["src_lays"], case["src_pools"], case["dst_lays"], dst, case["n_tokens"],
               case["src_tables"], case["dst_tables"], layer_range)
    return dst


def logical_code(r, l, c, h, t, d, L, H, T_max, D):
    """Coordinate code of a logical element (injective for < 65536 elements)."""
    return ((((r * L + l) * 2 + c) * H + h) * T_max + t) * D + d


def coord_fill(case, o1):
    """Overwrite valid source elements with their 16-bit coordinate codes (same-dtype cases)."""
    lay0 = case["src_lays"][0]
    L, H, D = lay0["L"], lay0["H"], lay0["D"]
    T_max = max(case["n_tokens"])
    n = len(case["n_tokens"]) * L * 2 * H * T_max * D
    assert n <= 0xFFF0, "coordinate codes must stay injective"
    for lay, pool in zip(case["src_lays"], case["src_pools"]):
        B, Hp, p = lay["B"], H // lay["tp"], lay["rank"]
        for r, T in enumerate(case["n_tokens"]):
            tab = case["src_tables"][r]
            for t in range(T):
                for l in range(L):
                    for c in held(lay):
                        for hl in range(Hp):
                            for d in range(D):
                                pool[o1.offset(lay, l, c, tab[t // B], t % B, hl, d)] = \
                                    logical_code(r, l, c, p * Hp + hl, t, d, L, H, T_max, D) + 1
    return T_max
