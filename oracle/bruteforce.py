"""O2 -- pure-Python brute-force oracle for the KV conversion (tiny shapes only).

TEST INFRASTRUCTURE ONLY: imported by tests/ (and nothing in the product path).
It shares no code with O1 (oracle/kv_oracle.c) beyond the plain integer
encoding of axes/dtypes, and none with the CUDA path.

It deliberately computes the same result as O1 by a *different* route, so that
a slip in either one shows up as a disagreement:

* **Index mapping is source-driven.**  O1 walks the destination and computes
  strided offsets with a formula.  O2 enumerates every physical position of
  every source pool in memory order (``itertools.product`` over the extents in
  ``axis_order``), recovers the logical element KV[r][l][c][h][t][d] through
  the *inverse* block table, then enumerates every destination position the same
  way and looks the logical element up.  No stride arithmetic appears.
* **Casts are nearest-code searches.**  O1 rounds with frexp/nearbyint.  O2
  decodes every finite code of the target format to an exact ``Fraction``,
  bisects for the neighbours of the exact input value and picks the nearer one,
  ties to the even code (RNE, IEEE 754 roundTiesToEven).  Overflow: a virtual
  code one quantum past the largest finite value stands for Inf (fp16/bf16) or
  saturates to +-448 (e4m3fn satfinite) / +-240 (e4m3fnuz satfinite).

Passages: P:113 (III-B2, Fig. 5 layout alignment), P:125 (III-B3, Fig. 4 TP
merge/split), P:65 (precision alignment), SPEC S:255/S:280 (zero-filled tail),
S:279 (head-contiguous TP), readings in DESIGN.md.
"""
from __future__ import annotations

import bisect
import itertools
from fractions import Fraction

import numpy as np

LAYER, KV, BLOCK, SLOT, HEAD, DIM = range(6)
F16, BF16, E4M3, F32, FNUZ = range(5)

# (exp_bits, mantissa_bits, bias, has_inf)
_FMT = {F16: (5, 10, 15, True), BF16: (8, 7, 127, True), E4M3: (4, 3, 7, False), F32: (8, 23, 127, True),
        FNUZ: (4, 3, 8, False)}
NBYTES = {F16: 2, BF16: 2, E4M3: 1, F32: 4, FNUZ: 1}
FP8 = (E4M3, FNUZ)


def decode(code: int, dt: int):
    """Exact value of an encoding as a Fraction; 'nan' / '+inf' / '-inf' / '-0' strings for specials."""
    eb, mb, bias, has_inf = _FMT[dt]
    sign = (code >> (eb + mb)) & 1
    e = (code >> mb) & ((1 << eb) - 1)
    m = code & ((1 << mb) - 1)
    if dt == FNUZ:
        if code == 0x80:
            return "nan"  # e4m3fnuz: the "negative zero" code is the only NaN; no infinities
    elif has_inf and e == (1 << eb) - 1:
        if m:
            return "nan"
        return "-inf" if sign else "+inf"
    elif not has_inf and e == (1 << eb) - 1 and m == (1 << mb) - 1:
        return "nan"  # OCP e4m3fn: S.1111.111 is the only NaN, no infinities
    if e == 0 and m == 0:
        return "-0" if sign else Fraction(0)
    if e == 0:
        mag = Fraction(m, 1 << mb) * Fraction(2) ** (1 - bias)
    else:
        mag = (1 + Fraction(m, 1 << mb)) * Fraction(2) ** (e - bias)
    return -mag if sign else mag


_TABLES: dict = {}


def _table(dt):
    """Sorted (value, code) of all finite non-negative codes + virtual overflow code."""
    if dt not in _TABLES:
        assert dt != F32, "O2 enumerates code tables; fp32 targets are O1-only"
        eb, mb, bias, has_inf = _FMT[dt]
        vals = []
        for code in range(1 << (eb + mb)):  # sign bit clear
            v = decode(code, dt)
            if isinstance(v, Fraction):
                vals.append((v, code))
        vals.sort()
        top_v, top_c = vals[-1]
        quantum = top_v - vals[-2][0]
        vals.append((top_v + quantum, "overflow"))
        _TABLES[dt] = ([v for v, _ in vals], [c for _, c in vals])
    return _TABLES[dt]


def round_to(x, dt: int) -> int:
    """Round an exact value (Fraction, or 'nan'/'+inf'/'-inf') to format dt.

    fp16/bf16/fp32: IEEE RNE, overflow -> +-Inf, NaN -> 0x7FFF / 0x7FFFFFFF
    (canonical NaN, reading 12).  e4m3fn: RNE with satfinite
    (overflow and +-Inf -> +-448), NaN -> 0x7F.  e4m3fnuz: RNE with satfinite
    (+-240), NaN -> 0x80, a zero result is 0x00 whatever its sign (reading 25).
    """
    eb, mb, bias, has_inf = _FMT[dt]
    sbit = 1 << (eb + mb)
    inf_code = ((1 << eb) - 1) << mb
    sat = {E4M3: 0x7E, FNUZ: 0x7F}.get(dt)
    if x == "nan":
        return {E4M3: 0x7F, FNUZ: 0x80, F32: 0x7FFFFFFF}.get(dt, 0x7FFF)
    if x == "-0":
        return 0 if dt == FNUZ else sbit
    if x in ("+inf", "-inf"):
        neg = x == "-inf"
        mag = sat if sat is not None else inf_code
        return mag | (sbit if neg else 0)
    neg = x < 0
    ax = -x if neg else x
    vals, codes = _table(dt)
    i = bisect.bisect_left(vals, ax)
    if i < len(vals) and vals[i] == ax:
        code = codes[i]
    else:
        lo_v, lo_c = vals[i - 1], codes[i - 1]
        if i >= len(vals):
            code = "overflow"
        else:
            hi_v, hi_c = vals[i], codes[i]
            dl, dh = ax - lo_v, hi_v - ax
            if dl < dh:
                code = lo_c
            elif dh < dl:
                code = hi_c
            else:  # tie: even code; the virtual overflow code follows an odd max code
                code = lo_c if (lo_c % 2 == 0) else hi_c
    if code == "overflow":
        code = sat if sat is not None else inf_code
    if neg and not (dt == FNUZ and code == 0):
        code |= sbit  # sign kept, including -0 (fnuz has no -0)
    return code


def _f32(frac_or_special) -> np.float32:
    if isinstance(frac_or_special, Fraction):
        return np.float32(float(frac_or_special))  # exact for <= 24 significant bits
    return {"nan": np.float32("nan"), "+inf": np.float32("inf"), "-inf": np.float32("-inf"),
            "-0": np.float32(-0.0)}[frac_or_special]


def _exact(v: np.float32):
    if np.isnan(v):
        return "nan"
    if np.isinf(v):
        return "-inf" if v < 0 else "+inf"
    if v == 0 and np.signbit(v):
        return "-0"
    return Fraction(float(v))


def cast(code: int, src_dt: int, dst_dt: int, src_scale: float = 1.0, dst_scale: float = 1.0) -> int:
    """Element cast (readings 10-13, 20, 24-26).  Same dtype: bits unchanged;
    fp8 sources are dequantised with src_scale, fp8 destinations quantised with dst_scale
    (so e4m3fn <-> e4m3fnuz goes through both)."""
    if src_dt == dst_dt:
        return code
    x = decode(code, src_dt)
    with np.errstate(all="ignore"):
        if src_dt in FP8:
            x = _exact(_f32(x) * np.float32(src_scale))
        if dst_dt in FP8:
            inv = np.float32(1.0) / np.float32(dst_scale)
            x = _exact(_f32(x) * inv)
    return round_to(x, dst_dt)


XLO = 6  # the innermost x part of a split head_dim (reading 27)


def _split(lay):
    x = lay.get("dim_split", 0)
    return x if x > 1 else 1


def _held(lay):
    """Global K/V indices a pool holds (kv_part 0: both, 1: K, 2: V)."""
    return {0: (0, 1), 1: (0,), 2: (1,)}[lay.get("kv_part", 0)]


def _extents(lay):
    return {LAYER: lay["L"], KV: len(_held(lay)), BLOCK: lay["NB"], SLOT: lay["B"], HEAD: lay["H"] // lay["tp"],
            DIM: lay["D"] // _split(lay), XLO: _split(lay)}


def positions(lay):
    """Yield (linear position, {axis: index}) over the pool in memory order, with the K/V
    index global (0 K, 1 V) and DIM the full head_dim index (split parts recombined)."""
    ext = _extents(lay)
    order = tuple(lay["order"]) + (XLO,)
    held = _held(lay)
    x = _split(lay)
    for pos, idx in enumerate(itertools.product(*[range(ext[a]) for a in order])):
        ix = dict(zip(order, idx))
        ix[KV] = held[ix[KV]]
        ix[DIM] = ix[DIM] * x + ix.pop(XLO)
        yield pos, ix


def _inverse_table(tables):
    inv = {}
    for r, ids in enumerate(tables):
        for j, b in enumerate(ids):
            assert b not in inv, "block id used twice"
            inv[b] = (r, j)
    return inv


def _scale(lay, l, c, hl):
    s = lay.get("scales")
    if s is None:
        return 1.0
    return float(s[l][c][hl])


def convert(src_lays, src_pools, dst_lays, dst_pools, n_tokens, src_tables, dst_tables, layer_range=None):
    """Brute-force P -> D conversion.  Pools are flat lists of int codes; dst_pools
    are modified in place (prior values survive where nothing is written).  A pool holds
    the global layers [first_layer, first_layer + L) (pipeline stages; default 0)."""
    if layer_range:
        lb, le = layer_range
    else:  # every global layer that some source and some destination pool hold
        lb = max(min(x.get("first_layer", 0) for x in src_lays), min(x.get("first_layer", 0) for x in dst_lays))
        le = min(max(x.get("first_layer", 0) + x["L"] for x in src_lays),
                 max(x.get("first_layer", 0) + x["L"] for x in dst_lays))
    # 1. logical tensor from every source pool, source-driven, keyed by GLOBAL layer
    logical = {}
    src_inv = _inverse_table(src_tables)
    for lay, pool in zip(src_lays, src_pools):
        hp_n = lay["H"] // lay["tp"]
        f = lay.get("first_layer", 0)
        for pos, ix in positions(lay):
            if ix[BLOCK] not in src_inv:
                continue
            r, jb = src_inv[ix[BLOCK]]
            t = jb * lay["B"] + ix[SLOT]
            if t >= n_tokens[r]:
                continue  # source tail: never read
            h = lay["rank"] * hp_n + ix[HEAD]
            logical[(r, f + ix[LAYER], ix[KV], h, t, ix[DIM])] = (pool[pos], lay, ix[HEAD], ix[LAYER])
    # 2. every destination position, destination-driven by enumeration (only the K/V the
    #    sources hold is written: a K-only source fills only the K part of a K+V pool)
    dst_inv = _inverse_table(dst_tables)
    src_held = set(_held(src_lays[0]))
    for lay, pool in zip(dst_lays, dst_pools):
        hd_n = lay["H"] // lay["tp"]
        f = lay.get("first_layer", 0)
        for pos, ix in positions(lay):
            g = f + ix[LAYER]
            if ix[BLOCK] not in dst_inv or not (lb <= g < le) or ix[KV] not in src_held:
                continue
            r, j = dst_inv[ix[BLOCK]]
            t = j * lay["B"] + ix[SLOT]
            h = lay["rank"] * hd_n + ix[HEAD]
            if t >= n_tokens[r]:
                pool[pos] = 0  # zero-filled tail
                continue
            code, slay, shl, sll = logical[(r, g, ix[KV], h, t, ix[DIM])]
            pool[pos] = cast(code, slay["dtype"], lay["dtype"],
                             _scale(slay, sll, ix[KV], shl), _scale(lay, ix[LAYER], ix[KV], ix[HEAD]))
    return dst_pools


def plan(tp_p: int, tp_d: int, H: int):
    """A2 by enumeration of heads: {(p, q): [heads]} (Fig. 4)."""
    if H % tp_p or H % tp_d:
        raise ValueError("tp degree does not divide num_kv_heads")
    pairs = {}
    for h in range(H):
        p, q = h // (H // tp_p), h // (H // tp_d)
        pairs.setdefault((p, q), []).append(h)
    return pairs
