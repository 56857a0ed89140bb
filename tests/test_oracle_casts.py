"""Pins for the oracle's precision-alignment casts (A6; readings 10-13).

Each check ties O1 (oracle/kv_oracle.c) to something other than itself:
library routines on the special cases that reduce to them (torch / numpy /
ml_dtypes), the OCP-e4m3 / PTX-satfinite definition (tests/golden/e4m3_edges.txt),
the brute-force nearest-code search O2, exhaustive round trips,
monotonicity and the half-ulp error bound.
"""
import os

import ml_dtypes
import numpy as np
import pytest
import torch

from oracle import bruteforce as o2

F16, BF16, E4M3, F32 = range(4)
HERE = os.path.dirname(os.path.abspath(__file__))
ALL16 = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)


def _is_nan16(codes, dt):
    e, m = ((codes >> 10) & 0x1F, codes & 0x3FF) if dt == F16 else ((codes >> 7) & 0xFF, codes & 0x7F)
    emax = 0x1F if dt == F16 else 0xFF
    return (e == emax) & (m != 0)


def test_f16_to_bf16_exhaustive_vs_torch_and_ml_dtypes(o1):
    got = o1.cast_array(ALL16, F16, BF16)
    nan = _is_nan16(ALL16, F16)
    t = torch.from_numpy(ALL16.view(np.int16).copy()).view(torch.float16).to(torch.bfloat16).view(torch.int16)
    ref_t = t.numpy().view(np.uint16)
    ref_m = ALL16.view(np.float16).astype(ml_dtypes.bfloat16).view(np.uint16)
    assert np.array_equal(got[~nan], ref_t[~nan])
    assert np.array_equal(got[~nan], ref_m[~nan])
    # reading 12: every NaN becomes the canonical quiet NaN 0x7FFF
    assert np.all(got[nan] == 0x7FFF)


def test_bf16_to_f16_exhaustive_vs_numpy_and_torch(o1):
    got = o1.cast_array(ALL16, BF16, F16)
    nan = _is_nan16(ALL16, BF16)
    # bf16 -> f32 is exact (append 16 zero bits); numpy f32 -> f16 is IEEE RNE
    f32 = (ALL16.astype(np.uint32) << 16).view(np.float32)
    with np.errstate(over="ignore"):
        ref_np = f32.astype(np.float16).view(np.uint16)
    ref_t = torch.from_numpy(ALL16.view(np.int16).copy()).view(torch.bfloat16).to(torch.float16)
    ref_t = ref_t.view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got[~nan], ref_np[~nan])
    assert np.array_equal(got[~nan], ref_t[~nan])
    assert np.all(got[nan] == 0x7FFF)
    # probe vectors (SURVEY 8(c) fp16<->bf16 row): 0x4780 -> Inf, 0x3300 -> +0, 0x3340 -> 0x0001
    assert o1.cast(0x4780, BF16, F16) == 0x7C00
    assert o1.cast(0x3300, BF16, F16) == 0x0000
    assert o1.cast(0x3340, BF16, F16) == 0x0001


def test_2byte_to_f32_to_2byte_identity_all_finite(o1):
    """SPEC S:539 acceptance 9: 2-byte -> 4-byte -> 2-byte is identity for every finite pattern."""
    for dt in (F16, BF16):
        finite = ~_is_nan16(ALL16, dt) & ~(((ALL16 & 0x7FFF) == (0x7C00 if dt == F16 else 0x7F80)))
        up = o1.cast_array(ALL16, dt, F32)
        back = o1.cast_array(up, F32, dt)
        assert np.array_equal(back[finite], ALL16[finite])
        # widening is exact: compare with numpy's own widening
        ref = ALL16.view(np.float16).astype(np.float32) if dt == F16 else (ALL16.astype(np.uint32) << 16).view(np.float32)
        assert np.array_equal(up[finite].view(np.float32), ref[finite])


def test_f32_to_bf16_random_vs_torch(o1):
    rng = np.random.default_rng(7)
    x = rng.integers(0, 1 << 32, size=200000, dtype=np.uint64).astype(np.uint32)
    x = x[(x & 0x7F800000) != 0x7F800000]
    got = o1.cast_array(x, F32, BF16)
    ref = torch.from_numpy(x.view(np.float32).copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, ref)


def _edges():
    rows = []
    with open(os.path.join(HERE, "golden", "e4m3_edges.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                a, b, _ = line.split()
                rows.append((int(a, 16), int(b, 16)))
    return rows


@pytest.mark.parametrize("f32_bits,code", _edges())
def test_e4m3_satfinite_edges(o1, f32_bits, code):
    v = np.array([f32_bits], dtype=np.uint32).view(np.float32)[0]
    assert o1.lib().okv_f32_to_e4m3(float(v)) == code
    # O2 path: exact value rounded by nearest-code search
    if not np.isnan(v):
        from fractions import Fraction
        x = "+inf" if v == np.inf else "-inf" if v == -np.inf else Fraction(float(v))
        if float(v) == 0.0 and np.signbit(v):
            x = "-0"
        assert o2.round_to(x, E4M3) == code


def _ml_e4m3(vals_f32):
    """Library special case: ml_dtypes RNE to e4m3fn after the satfinite clamp."""
    with np.errstate(invalid="ignore"):
        c = np.clip(vals_f32, np.float32(-448), np.float32(448))
    return c.astype(ml_dtypes.float8_e4m3fn).view(np.uint8)


@pytest.mark.parametrize("src", [F16, BF16])
def test_e4m3_pow2_scales_exhaustive_vs_ml_dtypes(o1, src):
    """x * 2^-k is exact in f32, so q = plain e4m3 RNE of the shifted value (textbook special case)."""
    nan = _is_nan16(ALL16, src)
    xf = ALL16.view(np.float16).astype(np.float32) if src == F16 else (ALL16.astype(np.uint32) << 16).view(np.float32)
    for k in range(-8, 9):
        s = float(np.ldexp(np.float32(1), k))
        got = o1.cast_array(ALL16, src, E4M3, 1.0, s)
        ref = _ml_e4m3(xf * np.float32(2.0 ** -k))
        assert np.array_equal(got[~nan], ref[~nan]), k
        assert np.all(got[nan] == 0x7F)


def test_e4m3_roundtrip_pow2(o1):
    """e4m3 -> bf16 (x 2^k) -> e4m3 (x 2^-k) is the identity for all 254 non-NaN codes."""
    codes = np.array([c for c in range(256) if (c & 0x7F) != 0x7F], dtype=np.uint8)
    for k in range(-8, 9):
        s = float(2.0 ** k)
        up = o1.cast_array(codes, E4M3, BF16, s, 1.0)
        back = o1.cast_array(up, BF16, E4M3, 1.0, s)
        # -0 and +0 both map back to themselves; compare exactly
        assert np.array_equal(back, codes), k


def _e4m3_value(codes):
    return codes.view(ml_dtypes.float8_e4m3fn).astype(np.float64)


@pytest.mark.parametrize("scale", [1.0, 0.25, 8.0, 0.0123456, 3.3, 0.7071, 5.5 / 448, 0.05])
def test_e4m3_monotone_and_half_ulp_bound(o1, scale):
    nan = _is_nan16(ALL16, BF16)
    codes = ALL16[~nan]
    x = (codes.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    finite = np.isfinite(x)
    codes, x = codes[finite], x[finite]
    q = o1.cast_array(codes, BF16, E4M3, 1.0, scale)
    qv = _e4m3_value(q)
    # monotone: sort by x, dequantised values non-decreasing
    order = np.argsort(x, kind="stable")
    assert np.all(np.diff(qv[order]) >= 0)
    # error bound: for in-range v, |q - v| <= half an e4m3 ulp at v, plus one f32 rounding of v
    inv = np.float32(1.0) / np.float32(scale)
    v = (x.astype(np.float32) * inv).astype(np.float64)
    inr = np.abs(v) <= 448
    e = np.floor(np.log2(np.maximum(np.abs(v[inr]), 2.0 ** -6)))
    ulp = 2.0 ** (e - 3)
    assert np.all(np.abs(qv[inr] - v[inr]) <= ulp / 2 + 1e-30)
    # saturation: everything beyond 448 clamps
    assert np.all(np.abs(qv[~inr]) == 448)


@pytest.mark.parametrize("pair", [(F16, BF16), (BF16, F16), (F16, E4M3), (BF16, E4M3), (E4M3, BF16), (E4M3, F16)])
def test_o1_vs_o2_bruteforce_casts(o1, pair):
    src, dst = pair
    rng = np.random.default_rng(11)
    if src == E4M3:
        codes = np.arange(256, dtype=np.uint32)
    else:
        specials = np.array([0, 0x8000, 0x7C00, 0xFC00, 0x7F80, 0xFF80, 0x7E01, 0x0001, 0x8001, 0x7BFF, 0x7F7F,
                             0x3C01, 0x3C08, 0x4780, 0x3300, 0x3340], dtype=np.uint32)
        codes = np.concatenate([specials, rng.integers(0, 1 << 16, size=3000).astype(np.uint32)])
    for scale in (1.0, 0.0123456, 5.5 / 448, 3.3):
        s_src = scale if src == E4M3 else 1.0
        s_dst = scale if dst == E4M3 else 1.0
        got = o1.cast_array(codes, src, dst, s_src, s_dst)
        ref = np.array([o2.cast(int(c), src, dst, s_src, s_dst) for c in codes])
        assert np.array_equal(got.astype(np.int64), ref.astype(np.int64)), (pair, scale)


@pytest.mark.parametrize("src", [F16, BF16])
@pytest.mark.parametrize("scale", [1.0, 0.25, 8.0, 0.0123456, 3.3, 0.7071, 5.5 / 448, 0.05])
def test_e4m3_scaled_op_order_exhaustive(o1, src, scale):
    """Reading 10 fixes the op order v = RN_f32(f32(x) * RN_f32(1/s)); numpy float32 arithmetic
    (IEEE binary32) computes v, ml_dtypes rounds it after the satfinite clamp.  x/s differs
    from x*(1/s) on a few patterns (e.g. s = 5.5/448), so this pins the order as well."""
    nan = _is_nan16(ALL16, src)
    xf = ALL16.view(np.float16).astype(np.float32) if src == F16 else (ALL16.astype(np.uint32) << 16).view(np.float32)
    with np.errstate(all="ignore"):
        v = xf * (np.float32(1.0) / np.float32(scale))
    got = o1.cast_array(ALL16, src, E4M3, 1.0, scale)
    assert np.array_equal(got[~nan], _ml_e4m3(v)[~nan])


# ---- e4m3fnuz (NEXT-3: another vendor's fp8; readings 24-26) ---------------------------
FNUZ = 4
ALL8 = np.arange(256, dtype=np.uint8)


def _fnuz_edges():
    rows = []
    with open(os.path.join(HERE, "golden", "e4m3fnuz_edges.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                b, c, _ = line.split()
                rows.append((int(b, 16), int(c, 16)))
    return rows


@pytest.mark.parametrize("f32_bits,code", _fnuz_edges())
def test_fnuz_satfinite_edges(o1, f32_bits, code):
    """O1 and O2 against the hand-worked definition vectors (scale 1: f32 -> fnuz)."""
    x = np.array([f32_bits], dtype=np.uint32)
    assert int(o1.cast_array(x, F32, FNUZ, 1.0, 1.0)[0]) == code
    v = np.uint32(f32_bits).view(np.float32)
    ex = o2._exact(v)
    assert o2.round_to(ex, FNUZ) == code


def test_fnuz_decode_exhaustive_vs_ml_dtypes(o1):
    """All 256 codes: widening to fp32 (scale 1) equals ml_dtypes' decode; 0x80 is the only NaN."""
    got = o1.cast_array(ALL8, FNUZ, F32, 1.0, 1.0).view(np.float32)
    ref = ALL8.view(ml_dtypes.float8_e4m3fnuz).astype(np.float32)
    nan = np.isnan(ref)
    assert list(np.nonzero(nan)[0]) == [0x80]
    assert np.array_equal(got[~nan], ref[~nan])
    assert np.isnan(got[0x80])
    assert got[0x7F] == 240.0 and got[0xFF] == -240.0


@pytest.mark.parametrize("src", [F16, BF16])
@pytest.mark.parametrize("k", [-6, 0, 3])
def test_fnuz_pow2_scales_exhaustive_vs_ml_dtypes(o1, src, k):
    """Power-of-two scales make x * RN(1/s) exact, so the cast reduces to ml_dtypes' RNE
    conversion for every 2-byte input whose scaled value is within +-240 (ml_dtypes does not
    saturate: beyond that it returns NaN, where the satfinite reading clamps)."""
    s = float(2.0 ** k)
    codes = ALL16[~_is_nan16(ALL16, src)]
    got = o1.cast_array(codes, src, FNUZ, 1.0, s)
    xs = (codes.view(np.float16) if src == F16 else codes.view(ml_dtypes.bfloat16)).astype(np.float32)
    v = xs * np.float32(1.0 / s)
    inr = np.abs(v) < 240.0
    ref = v[inr].astype(ml_dtypes.float8_e4m3fnuz).view(np.uint8)
    assert np.array_equal(got[inr], ref)
    big = ~inr & np.isfinite(v)
    assert np.all(got[big] == np.where(v[big] > 0, 0x7F, 0xFF))


def test_fnuz_never_negative_zero_never_nan_from_finite(o1):
    codes = ALL16[~_is_nan16(ALL16, BF16)]
    got = o1.cast_array(codes, BF16, FNUZ, 1.0, 0.37)
    assert not np.any(got == 0x80)


@pytest.mark.parametrize("pair", [(BF16, FNUZ), (F16, FNUZ), (FNUZ, BF16), (FNUZ, F16), (E4M3, FNUZ), (FNUZ, E4M3)])
@pytest.mark.parametrize("scales", [(1.0, 1.0), (0.5, 2.0), (0.37, 1.9)])
def test_fnuz_o1_vs_o2(o1, pair, scales):
    """O1 (frexp/nearbyint) == O2 (nearest-code search over the decoded code table) on every
    fp8 code / a 2-byte sample, with the dequant scale of an fp8 source and the quant scale
    of an fp8 destination (fn <-> fnuz: dequantise then quantise, reading 26)."""
    src, dst = pair
    if o2.NBYTES[src] == 1:
        codes = ALL8.copy()
    else:
        rng = np.random.default_rng(7)
        codes = rng.integers(0, 1 << 16, size=3000).astype(np.uint16)
        codes = codes[~_is_nan16(codes, src)]
    ss, ds = scales
    got = o1.cast_array(codes, src, dst, ss, ds)
    for c, g in zip(codes.tolist(), got.tolist()):
        assert o2.cast(int(c), src, dst, ss, ds) == g, (hex(c), hex(g))


def test_fn_fnuz_identity_on_shared_grid(o1):
    """Closed form: with s_fnuz = 2 * s_fn the two formats encode the same reals on the common
    range, and e4m3fn code c (|c| <= 448, not NaN) maps to the fnuz code with the SAME bits
    (every fnuz value is half the fn value of its bits).  Codes whose value exceeds 240 * s
    saturate; fn's 2^-9 * s_fn subnormal is fnuz's 2^-10 * s_fnuz: all representable."""
    sf = 0.5
    fn = np.array([c for c in range(256) if (c & 0x7F) != 0x7F], dtype=np.uint8)
    got = o1.cast_array(fn, E4M3, FNUZ, sf, 2 * sf)
    want = fn.copy()
    want[fn == 0x80] = 0x00                       # -0 has no fnuz code: +0
    assert np.array_equal(got, want)
    back = o1.cast_array(got, FNUZ, E4M3, 2 * sf, sf)
    assert np.array_equal(back, np.where(fn == 0x80, 0, fn).astype(np.uint8))
