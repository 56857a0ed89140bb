"""Pins for the oracle's dynamic fp8 scales (NEXT-1; P:65 precision alignment; DESIGN.md
reading 21): s = RN_f32(amax / 448) over the finite source values of the batch, 1 if 0.

Tied to: numpy's max over the logical tensor in the special case where the source pool is
already in canonical (layer, kv, head, token, dim) order with identity tables; a closed
form (a single element 448 * 2^k gives s = 2^k exactly); the all-zero case; the TP merge
(a D head's scale equals the scale of the P head it came from)."""
import numpy as np

import synth
from synth import BF16, F16, LAYER, KV, HEAD, BLOCK, SLOT, DIM

CANON = (LAYER, KV, HEAD, BLOCK, SLOT, DIM)


def _vals(codes, dt):
    if dt == F16:
        return codes.view(np.float16).astype(np.float32)
    return (codes.astype(np.uint32) << 16).view(np.float32)


def test_numpy_special_case(o1):
    L, H, D, B, NB = 3, 4, 16, 8, 4
    for dt in (F16, BF16):
        lay = synth.layout(L, H, D, 1, 0, B, NB, dt, CANON)
        pool = synth.random_finite_bits(3 + dt, 2 * L * H * NB * B * D, dt)
        pool[5] = 0x7E01 if dt == F16 else 0x7FC1   # NaN is ignored
        pool[77] = 0x7C00 if dt == F16 else 0x7F80  # +Inf is ignored
        got = o1.amax_scales([lay], [pool], lay, [NB * B], [list(range(NB))])
        v = np.abs(_vals(pool, dt).reshape(L, 2, H, NB * B * D))
        v = np.where(np.isfinite(v), v, 0)
        want = v.max(axis=3).astype(np.float32) / np.float32(448)
        want = np.where(want > 0, want, np.float32(1))
        assert np.array_equal(got, want)


def test_closed_form_pow2_and_zero(o1):
    L, H, D, B, NB = 2, 2, 8, 4, 3
    lay = synth.layout(L, H, D, 1, 0, B, NB, BF16, synth.P_ORDER)
    pool = np.zeros(2 * L * H * NB * B * D, dtype=np.uint16)
    # element (l=1, c=0, block 2, slot 1, head 1, d 3) = -448 * 2^-3 = -56 (bf16 0xC260)
    pool[o1.offset(lay, 1, 0, 2, 1, 1, 3)] = 0xC260
    got = o1.amax_scales([lay], [pool], lay, [NB * B], [list(range(NB))])
    want = np.ones((L, 2, H), np.float32)
    want[1, 0, 1] = 0.125
    assert np.array_equal(got, want)


def test_merge_takes_each_heads_own_scale(o1):
    """TP 2 -> 1: D head h's scale = the scale computed for P rank h // H_p, local head."""
    L, H, D, B = 2, 4, 8, 4
    n_tokens = [6, 9]
    NB = synth.pool_capacity(n_tokens, B)
    tabs = synth.block_tables(9, n_tokens, B, NB)
    src = [synth.layout(L, H, D, 2, p, B, NB, F16, synth.P_ORDER) for p in range(2)]
    pools = [synth.random_finite_bits(40 + p, 2 * L * NB * B * 2 * D, F16) for p in range(2)]
    d1 = synth.layout(L, H, D, 1, 0, B, NB, F16, synth.D_ORDER)
    merged = o1.amax_scales(src, pools, d1, n_tokens, tabs)
    for p in range(2):
        per = o1.amax_scales([src[p]], [pools[p]], synth.layout(L, H, D, 2, p, B, NB, F16, synth.D_ORDER),
                             n_tokens, tabs)
        assert np.array_equal(merged[:, :, 2 * p:2 * p + 2], per)


def test_closed_form_fnuz_destination(o1):
    """Reading 21 for an e4m3fnuz destination: s = RN(amax / 240) (240 = its largest finite
    value); one element -240 * 2^-3 = -30 gives exactly 2^-3, the rest 1."""
    L, H, D, B, NB = 2, 2, 8, 4, 3
    lay = synth.layout(L, H, D, 1, 0, B, NB, BF16, synth.P_ORDER)
    dst = synth.layout(L, H, D, 1, 0, B, NB, synth.FNUZ, synth.D_ORDER)
    pool = np.zeros(2 * L * H * NB * B * D, dtype=np.uint16)
    pool[o1.offset(lay, 0, 1, 1, 2, 0, 5)] = 0xC1F0   # bf16 -30
    got = o1.amax_scales([lay], [pool], dst, [NB * B], [list(range(NB))])
    want = np.ones((L, 2, H), np.float32)
    want[0, 1, 0] = 0.125
    assert np.array_equal(got, want)
