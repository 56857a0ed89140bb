"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no layout offsets, no
casts, no re-shard routing): it only draws request lengths, block tables,
random bit patterns, fp8 scales and names the paper-shaped configurations.
Both ``oracle/`` (via tests) and the product path (via tests / bench) take their
inputs from here; neither imports the other.

Recipe:
* values: uniform random *finite* bit patterns of the source dtype (every
  rounding case is exercised); or N(0, sigma_h) per (layer, K/V, head) with
  sigma_h log-uniform in [0.1, 10] and 1% outlier K channels x20 (fp8 realism);
* fp8 dequant scales: amax / 448 per (layer, K/V, decode head), or powers of two;
* block tables: a seeded Fisher-Yates permutation of [0, N_blocks), sliced per
  request (the identity slice is the contiguous best case); pool capacity
  = sum_r ceil(T_r / B) * 1.1 (+1);
* destination pools start as canary bytes 0xA5;
* c5 lengths: T_r = round(exp(U(ln 512, ln 32768))).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# Axis / dtype encodings of the C ABI (include/kvx.h) -- plain integers.
LAYER, KV, BLOCK, SLOT, HEAD, DIM = range(6)
F16, BF16, E4M3, F32, FNUZ = range(5)   # FNUZ: e4m3fnuz (NEXT-3, another vendor's fp8)
NBYTES = {F16: 2, BF16: 2, E4M3: 1, F32: 4, FNUZ: 1}
DTYPE_NAMES = {F16: "f16", BF16: "bf16", E4M3: "e4m3", F32: "f32", FNUZ: "e4m3fnuz"}
FP8 = (E4M3, FNUZ)

# DESIGN.md reading 3: P = vLLM-style NHD per layer, D = block-major HND.
P_ORDER = (LAYER, KV, BLOCK, SLOT, HEAD, DIM)
D_ORDER = (BLOCK, LAYER, KV, HEAD, SLOT, DIM)

CANARY = 0xA5


def layout(L, H, D, tp, rank, B, NB, dtype, order, scales=None, kv_part=0, dim_split=0):
    """Layout dict used by tests/bench (same fields as kv_layout_desc).  kv_part: 0 K and V,
    1 K only, 2 V only; dim_split: x > 1 stores head_dim as (D/x, ..., x)."""
    return {"L": L, "H": H, "D": D, "tp": tp, "rank": rank, "B": B, "NB": NB, "dtype": dtype,
            "order": tuple(order), "scales": scales, "kv_part": kv_part, "dim_split": dim_split}


def blocks_for(tokens: int, block_size: int) -> int:
    return -(-tokens // block_size)


def pool_capacity(n_tokens, block_size, slack=1.1):
    need = sum(blocks_for(t, block_size) for t in n_tokens)
    return int(math.ceil(need * slack)) + 1


def block_tables(seed, n_tokens, block_size, num_blocks, contiguous=False):
    """Per-request block-id lists: a seeded permutation of [0, num_blocks), sliced."""
    need = [blocks_for(t, block_size) for t in n_tokens]
    assert sum(need) <= num_blocks, "pool too small"
    ids = np.arange(num_blocks, dtype=np.int64)
    if not contiguous:
        rng = np.random.default_rng(seed)
        rng.shuffle(ids)  # Fisher-Yates
    out, k = [], 0
    for n in need:
        out.append(ids[k:k + n].astype(np.int32).tolist())
        k += n
    return out


def random_finite_bits(seed, n, dtype):
    """Uniform random bit patterns of `dtype` with NaN/Inf patterns avoided.

    An all-ones exponent field is broken by clearing its lowest bit (so the
    result is a finite pattern); e4m3fn only has NaN at S.1111.111, e4m3fnuz only at
    0x80 (flipped to 0x81)."""
    rng = np.random.default_rng(seed)
    nb = NBYTES[dtype]
    if nb == 1:
        x = rng.integers(0, 256, size=n, dtype=np.uint16).astype(np.uint8)
        bad = (x == 0x80) if dtype == FNUZ else ((x & 0x7F) == 0x7F)
        x[bad] ^= 0x01
        return x
    if nb == 2:
        x = rng.integers(0, 1 << 16, size=n, dtype=np.uint32).astype(np.uint16)
        m, low = (0x7C00, 0x0400) if dtype == F16 else (0x7F80, 0x0080)
        bad = (x & m) == m
        x[bad] ^= low
        return x
    x = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    bad = (x & 0x7F800000) == 0x7F800000
    x[bad] ^= 0x00800000
    return x


def fill_random_finite_(t, seed, dtype):
    """Device-side version of random_finite_bits for a torch integer tensor view.

    Used for full-size pools (GB) that are never copied to the host whole."""
    import torch
    g = torch.Generator(device=t.device)
    g.manual_seed(int(seed))
    nb = NBYTES[dtype]
    if nb == 1:
        t.copy_(torch.randint(0, 256, t.shape, generator=g, device=t.device, dtype=torch.int16).to(torch.uint8))
        bad = (t == 0x80) if dtype == FNUZ else ((t & 0x7F) == 0x7F)
        t ^= bad.to(torch.uint8)
        return t
    if nb == 2:
        m, low = (0x7C00, 0x0400) if dtype == F16 else (0x7F80, 0x0080)
        flat = t.view(-1)
        step = 1 << 28  # fill in 512 MiB pieces: no pool-sized temporaries
        for i in range(0, flat.numel(), step):
            part = flat[i:i + step]
            v = torch.randint(-(1 << 15), 1 << 15, part.shape, generator=g, device=t.device, dtype=torch.int16)
            bad = (v & m) == m
            v ^= bad.to(torch.int16) * low
            part.copy_(v.view(t.dtype) if t.dtype != torch.int16 else v)
        return t
    raise NotImplementedError("fp32 device fill")


def gaussian_bits(seed, shape_lcht_d, dtype):
    """fp8-realism values: N(0, sigma) per (l, c, h), 1% outlier K channels x20.

    shape = (L, 2, H, T, D) logical; returns float32 values (cast to the source
    dtype by the caller's library routine, e.g. torch), plus the sigma table."""
    L, _, H, T, D = shape_lcht_d
    rng = np.random.default_rng(seed)
    sigma = np.exp(rng.uniform(np.log(0.1), np.log(10.0), size=(L, 2, H))).astype(np.float32)
    x = rng.standard_normal(size=(L, 2, H, T, D)).astype(np.float32) * sigma[..., None, None]
    outlier = rng.random(size=(L, H, D)) < 0.01
    x[:, 0] = np.where(outlier[:, :, None, :], x[:, 0] * 20.0, x[:, 0])
    return x


def amax_scales(values_lchtd, tp_d, rank):
    """Per (l, c, decode-local head) dequant scale amax/448 (fp32)."""
    L, _, H, _, _ = values_lchtd.shape
    Hd = H // tp_d
    amax = np.abs(values_lchtd[:, :, rank * Hd:(rank + 1) * Hd]).max(axis=(3, 4))
    return np.maximum(amax / np.float32(448.0), np.float32(1e-12)).astype(np.float32)


def pow2_scales(seed, L, H_local, kmin=-8, kmax=8):
    rng = np.random.default_rng(seed)
    k = rng.integers(kmin, kmax + 1, size=(L, 2, H_local))
    return np.ldexp(np.float32(1.0), k).astype(np.float32)


def loguniform_lengths(seed, n, lo=512, hi=32768):
    rng = np.random.default_rng(seed)
    return [int(round(math.exp(v))) for v in rng.uniform(math.log(lo), math.log(hi), size=n)]


@dataclass
class Config:
    """A BASELINE.json configuration (SURVEY 8 shapes table)."""
    name: str
    L: int
    H: int
    D: int
    n_tokens: list
    tp_p: int
    tp_d: int
    src_dtype: int
    dst_dtype: int
    B_p: int
    B_d: int
    p_order: tuple = P_ORDER
    d_order: tuple = D_ORDER
    seed: int = 1000
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def total_tokens(self):
        return int(sum(self.n_tokens))

    def src_bytes(self):
        """Logical source KV bytes (SPEC S:41 formula over all requests)."""
        return 2 * self.L * self.H * self.D * self.total_tokens * NBYTES[self.src_dtype]


def configs():
    """BASELINE.json configs, in order (c1..c5)."""
    return {
        "c1": Config("c1", 2, 2, 64, [32], 1, 1, F16, BF16, 16, 32, seed=1001,
                     note="tiny KV, fp16->bf16, block 16->32, TP1->1, one GPU"),
        "c2": Config("c2", 32, 32, 128, [2048], 2, 1, F16, F16, 16, 16, seed=1002,
                     note="Llama-2-7B KV, 2048-token prompt, TP2->1, fp16, block 16->16"),
        "c3": Config("c3", 32, 8, 128, [4096] * 16, 4, 2, BF16, BF16, 16, 64, seed=1003,
                     note="Llama-3-8B GQA KV, 16x4096, TP4->2, bf16, block 16->64"),
        "c4": Config("c4", 80, 8, 128, [4096] * 32, 4, 4, BF16, E4M3, 16, 16, seed=1004,
                     note="Llama-3-70B GQA KV, 32x4096, TP4->4, bf16->fp8-e4m3 per-head scale"),
        "c5": Config("c5", 80, 8, 128, loguniform_lengths(1005, 64), 2, 4, BF16, BF16, 16, 16, seed=1005,
                     note="70B-shaped stream, 64 requests T~logU[512,32k], 2 P instances x TP2 -> D TP4"),
    }
