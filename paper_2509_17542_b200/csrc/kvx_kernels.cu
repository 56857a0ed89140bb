// sm_100a kernels of the KV convert / reshard / transfer path (arXiv 2509.17542, III-B).
//
// Everything on the path is data movement plus an elementwise cast, so nothing here is a
// dense contraction: no tensor cores.  The kernels are HBM-bound (one GPU) or NVLink-bound
// (peer loads / stores).  DESIGN.md section 5 has each kernel's roofline and bytes; in short:
//   * k_convert_rows (default whenever head_dim is innermost on both sides): a work item is
//     32 head_dim rows of one (dst rank, dst block, layer, K/V) tile; each lane decodes one
//     row (block tables, TP routing, scale) and the warp streams the rows' 16-B chunks with
//     U loads in flight per lane, fetching row state by shuffles.  A peer-mapped source or
//     destination makes it the D-side NVLink pull or the P-side push.
//   * k_tile_copy (same dtype, D's inner axes {HEAD, SLOT} x DIM): one 5-D TMA tensor load per
//     source sub-tile, already permuted into D's order, then bulk stores.
//   * k_tile_cast (the same sub-tiles with a cast: TMA-fed stages, 8 consumer warps convert
//     the rows; the N = 1 default for 2-byte sources).
//   * k_convert_tb (head_dim-major 1-/2-byte source tiles of 16 slots, x-packed 2-byte and
//     fp8 tiles): one 2-D TMA load per tile (or two heads) into swizzled shared-memory
//     stages, warp-specialised producer / consumers that transpose 8 x 8 sub-blocks out of
//     shared memory.
//   * k_requant_rows (fp8 -> other fp8): the row items with 128-entry shared-memory code
//     tables instead of the arithmetic cast.
//   * k_convert_tr8 / k_convert_tr (other head_dim-major or x-packed sides): 8 x 8 register
//     transposes / shared-memory tiles.
//   * k_pack_rows / k_unpack_rows (Fig. 5 flatten / restore: the NCCL mode and the staged
//     pull's P side), k_pull_rows (the persistent staged pull, D side), k_stage_rows (the
//     opt-in persistent P side), k_amax_rows (dynamic scales), k_signal / k_wait (flags).
//   * VEC=1 k_convert / k_pack / k_unpack: the element-wise generic path for any of the 720
//     axis orders.
// Casts (readings 10-13, 24-26): same dtype = bit copy; f16/bf16/f32 narrowing via
// cvt.rn (RNE, canonical NaN); e4m3 via cvt.rn.satfinite.e4m3x2.f32 of x * RN(1/s) with
// __fmul_rn (never contracted into an FMA); e4m3 widening = cvt.rn.f16x2.e4m3x2 (exact) then
// * s; e4m3fnuz through the e4m3fn conversions or an exact f16 bit decode.
#include <cuda_bf16.h>
#include <algorithm>
#include <cuda_fp16.h>

#include "kvx_internal.h"

// cache-policy knobs for the streaming loads/stores (experiments; default: none)
#ifndef KVX_LD_HINT
#define KVX_LD_HINT ""
#endif
#ifndef KVX_ST_HINT
#define KVX_ST_HINT ""
#endif

namespace kvx {

namespace {

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  uint32_t t = __umulhi(n, f.mul);
  return (uint32_t)(((uint64_t)t + n) >> f.shr);
}

template <int DT>
struct Tr;
template <>
struct Tr<KV_F16> { static constexpr int B = 2; };
template <>
struct Tr<KV_BF16> { static constexpr int B = 2; };
template <>
struct Tr<KV_F8E4M3> { static constexpr int B = 1; };
template <>
struct Tr<KV_F32> { static constexpr int B = 4; };
template <>
struct Tr<KV_F8E4M3FNUZ> { static constexpr int B = 1; };

// fp8 formats carry a per-(layer, K/V, head) dequant scale (readings 9, 24)
__host__ __device__ constexpr bool is_fp8(int dt) { return dt == KV_F8E4M3 || dt == KV_F8E4M3FNUZ; }
// an fp8 -> other-fp8 cast needs both scales (dequantise, then quantise: reading 26)
__host__ __device__ constexpr bool dual_scale(int sdt, int ddt) { return is_fp8(sdt) && is_fp8(ddt) && sdt != ddt; }

// A chunk of VEC elements of dtype DT in 32-bit words.
template <int DT, int VEC>
struct Chunk {
  static constexpr int BYTES = VEC * Tr<DT>::B;
  static constexpr int WORDS = (BYTES + 3) / 4;
  uint32_t w[WORDS];
};

// COH = false: the read-only (.nc) path -- the source is not written during the kernel.
// COH = true: ordinary weak loads, ordered after an acquire in the same kernel (the
// persistent pull reads ring slots the P rank rewrites while the kernel runs).
template <bool COH>
__device__ __forceinline__ void ld_v4(uint32_t& x, uint32_t& y, uint32_t& z, uint32_t& w, const uint8_t* p) {
  if constexpr (COH)
    asm volatile("ld.global.L1::no_allocate" KVX_LD_HINT ".v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "l"(p) : "memory");
  else
    asm volatile("ld.global.nc.L1::no_allocate" KVX_LD_HINT ".v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "l"(p));
}
template <bool COH>
__device__ __forceinline__ void ld_v2(uint32_t& x, uint32_t& y, const uint8_t* p) {
  if constexpr (COH)
    asm volatile("ld.global.L1::no_allocate" KVX_LD_HINT ".v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "l"(p) : "memory");
  else
    asm volatile("ld.global.nc.L1::no_allocate" KVX_LD_HINT ".v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "l"(p));
}

template <bool COH>
__device__ __forceinline__ void ld_v8(uint32_t* w, const uint8_t* p) {
  if constexpr (COH)
    asm volatile("ld.global.L1::no_allocate" KVX_LD_HINT ".v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "l"(p) : "memory");
  else
    asm volatile("ld.global.nc.L1::no_allocate" KVX_LD_HINT ".v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "l"(p));
}

template <int DT, int VEC, bool COH = false>
__device__ __forceinline__ void load_chunk(Chunk<DT, VEC>& c, const uint8_t* p) {
  constexpr int N = Chunk<DT, VEC>::BYTES;
  if constexpr (N == 32) {
    if ((reinterpret_cast<uintptr_t>(p) & 31u) == 0) {  // one 256-bit load (LDG.E.256)
      ld_v8<COH>(c.w, p);
    } else {
      ld_v4<COH>(c.w[0], c.w[1], c.w[2], c.w[3], p);
      ld_v4<COH>(c.w[4], c.w[5], c.w[6], c.w[7], p + 16);
    }
  } else if constexpr (N == 16) {
    ld_v4<COH>(c.w[0], c.w[1], c.w[2], c.w[3], p);
  } else if constexpr (N == 8) {
    ld_v2<COH>(c.w[0], c.w[1], p);
  } else if constexpr (N == 4) {
    c.w[0] = *reinterpret_cast<const uint32_t*>(p);
  } else if constexpr (N == 2) {
    c.w[0] = *reinterpret_cast<const uint16_t*>(p);
  } else {
    c.w[0] = *p;
  }
}

// read-only loads that allocate in L1 (k_convert_tr8's x-packed source: a lane re-reads
// the other half of each sector in its next load)
template <int DT, int VEC>
__device__ __forceinline__ void load_chunk_l1(Chunk<DT, VEC>& c, const uint8_t* p) {
  constexpr int N = Chunk<DT, VEC>::BYTES;
  static_assert(N == 8 || N == 16 || N == 32, "vector chunks only");
#pragma unroll
  for (int o = 0; o < N; o += 16) {
    if constexpr (N == 8)
      asm volatile("ld.global.nc.L1::evict_last.v2.u32 {%0,%1}, [%2];" : "=r"(c.w[0]), "=r"(c.w[1]) : "l"(p));
    else
      asm volatile("ld.global.nc.L1::evict_last.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(c.w[o / 4]), "=r"(c.w[o / 4 + 1]), "=r"(c.w[o / 4 + 2]), "=r"(c.w[o / 4 + 3])
                   : "l"(p + o));
  }
}

template <int DT, int VEC>
__device__ __forceinline__ void store_chunk(uint8_t* p, const Chunk<DT, VEC>& c) {
  constexpr int N = Chunk<DT, VEC>::BYTES;
  // 32-B chunks: one 256-bit store when 32-B aligned (sm_100 STG.E.256; e4m3 -> bf16 on the
  // row kernel 0.86 -> 0.89 of copy, bf16 -> f32 0.83 -> 0.90), else two 128-bit stores
  if constexpr (N == 32) {
    if ((reinterpret_cast<uintptr_t>(p) & 31u) == 0) {
      asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(c.w[0]), "r"(c.w[1]), "r"(c.w[2]),
                   "r"(c.w[3]), "r"(c.w[4]), "r"(c.w[5]), "r"(c.w[6]), "r"(c.w[7]) : "memory");
      return;
    }
  }
  if constexpr (N == 32) {
    asm volatile("st.global" KVX_ST_HINT ".v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(c.w[0]), "r"(c.w[1]), "r"(c.w[2]),
                 "r"(c.w[3]) : "memory");
    asm volatile("st.global" KVX_ST_HINT ".v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p + 16), "r"(c.w[4]), "r"(c.w[5]), "r"(c.w[6]),
                 "r"(c.w[7]) : "memory");
  } else if constexpr (N == 16) {
    asm volatile("st.global" KVX_ST_HINT ".v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(c.w[0]), "r"(c.w[1]), "r"(c.w[2]),
                 "r"(c.w[3]) : "memory");
  } else if constexpr (N == 8) {
    asm volatile("st.global" KVX_ST_HINT ".v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(c.w[0]), "r"(c.w[1]) : "memory");
  } else if constexpr (N == 4) {
    *reinterpret_cast<uint32_t*>(p) = c.w[0];
  } else if constexpr (N == 2) {
    *reinterpret_cast<uint16_t*>(p) = (uint16_t)c.w[0];
  } else {
    *p = (uint8_t)c.w[0];
  }
}

template <int DT>
__device__ __forceinline__ uint32_t get_elem(const uint32_t* w, int i) {
  if constexpr (Tr<DT>::B == 4) return w[i];
  if constexpr (Tr<DT>::B == 2) return (w[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu;
  return (w[i >> 2] >> ((i & 3) * 8)) & 0xFFu;
}

template <int DT>
__device__ __forceinline__ void put_elem(uint32_t* w, int i, uint32_t e) {
  if constexpr (Tr<DT>::B == 4) w[i] = e;
  else if constexpr (Tr<DT>::B == 2) w[i >> 1] |= (e & 0xFFFFu) << ((i & 1) * 16);
  else w[i >> 2] |= (e & 0xFFu) << ((i & 3) * 8);
}

// shared-memory chunk moves (k_convert_tr's tile rows are 16-B aligned)
template <int DT, int VEC>
__device__ __forceinline__ void store_chunk_smem(uint8_t* p, const Chunk<DT, VEC>& c) {
#pragma unroll
  for (int i = 0; i < Chunk<DT, VEC>::WORDS; ++i) reinterpret_cast<uint32_t*>(p)[i] = c.w[i];
}
template <int DT, int VEC>
__device__ __forceinline__ void load_chunk_smem(Chunk<DT, VEC>& c, const uint8_t* p) {
#pragma unroll
  for (int i = 0; i < Chunk<DT, VEC>::WORDS; ++i) c.w[i] = reinterpret_cast<const uint32_t*>(p)[i];
}

template <int DT>
__device__ __forceinline__ float to_f32(uint32_t b) {
  if constexpr (DT == KV_F16) {
    return __half2float(__ushort_as_half((unsigned short)b));
  } else if constexpr (DT == KV_BF16) {
    return __uint_as_float(b << 16);
  } else if constexpr (DT == KV_F32) {
    return __uint_as_float(b);
  } else if constexpr (DT == KV_F8E4M3FNUZ) {
    // e4m3fnuz: bias 8, 0x80 the only NaN, no infinities (0x7F = 240)
    const uint32_t sgn = (b & 0x80u) << 24, e = (b >> 3) & 0xFu, m = b & 7u;
    const float sub = __uint_as_float(__float_as_uint((float)m * 0.0009765625f) | sgn);  // m * 2^-10
    const float nrm = __uint_as_float(sgn | ((e + 119u) << 23) | (m << 20));
    return b == 0x80u ? __uint_as_float(0x7FFFFFFFu) : (e == 0u ? sub : nrm);
  } else {
    uint32_t h2;
    unsigned short in = (unsigned short)b;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(in));
    return __half2float(__ushort_as_half((unsigned short)(h2 & 0xFFFFu)));
  }
}

__device__ __forceinline__ uint32_t f32_to_f16(float f) {
  uint32_t r;
  unsigned short h;
  asm("cvt.rn.f16.f32 %0, %1;" : "=h"(h) : "f"(f));
  r = h;
  return r;
}
__device__ __forceinline__ uint32_t f32_to_bf16(float f) {
  unsigned short h;
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"(f));
  return h;
}
// two e4m3 codes: lo -> bits 0..7, hi -> bits 8..15
__device__ __forceinline__ uint32_t f32x2_to_e4m3x2(float lo, float hi) {
  unsigned short r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

// a, b <- RN(a * s), RN(b * s): one FMUL2 (__fmul2_rn: round-to-nearest, never contracted
// into an FMA)
__device__ __forceinline__ void fmul2_rn(float& a, float& b, float s) {
  const float2 r = __fmul2_rn(make_float2(a, b), make_float2(s, s));
  a = r.x;
  b = r.y;
}

// e4m3fnuz codes of two scaled f32 values (lo -> bits 0..7, hi -> bits 8..15): RNE with
// satfinite at +-240, NaN -> 0x80, zero results +0 (reading 25).  Every fnuz value is half
// the e4m3fn value of the same bits (same mantissa grid, bias 8 vs 7), so the hardware
// e4m3fn conversion of 2v gives the fnuz code except where the fn grid has its NaN slot
// (2v > 464 <=> v > 232: saturate to 0x7F) and for -0 (0x80 is fnuz's NaN: make it +0).
__device__ __forceinline__ uint32_t fnuz_fix(uint32_t code, float v) {
  const float a = fabsf(v);
  if (a != a) return 0x80u;
  if (a > 232.0f) return 0x7Fu | ((__float_as_uint(v) >> 24) & 0x80u);
  return code == 0x80u ? 0u : code;
}
__device__ __forceinline__ uint32_t f32x2_to_fnuzx2(float lo, float hi) {
  const uint32_t r = f32x2_to_e4m3x2(__fmul_rn(lo, 2.0f), __fmul_rn(hi, 2.0f));
  return fnuz_fix(r & 0xFFu, lo) | (fnuz_fix((r >> 8) & 0xFFu, hi) << 8);
}


// Four e4m3fnuz codes of scaled values f[0..3], branch-free (no divergence on data): the
// hardware e4m3fn conversion of 2v (RNE, satfinite: every |2v| > 432 gives 0x7E | sign),
// then -0 (0x80) -> +0 by an exact per-byte zero test, then +1 on the bytes whose |2v| >
// 464 or is NaN (one set.gtu each): 0x7E | s -> 0x7F | s (+-240, v > 232) and the NaN code
// 0x7F -> 0x80 (fnuz's NaN; the scale multiply before this made every NaN positive)
// (reading 25).  Runs after the zero fix so a NaN's 0x80 is not taken for -0.
__device__ __forceinline__ uint32_t f32x4_to_fnuzx4(const float* f) {
  float d[4] = {f[0], f[1], f[2], f[3]};
  fmul2_rn(d[0], d[1], 2.0f);
  fmul2_rn(d[2], d[3], 2.0f);
  uint32_t r = f32x2_to_e4m3x2(d[0], d[1]) | (f32x2_to_e4m3x2(d[2], d[3]) << 16);
  const uint32_t x = r ^ 0x80808080u;  // bytes equal to 0x80 become 0
  r ^= ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;  // exact per-byte zero test: -0 -> +0
  uint32_t m[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) asm("set.gtu.u32.f32 %0, %1, 0f43E80000;" : "=r"(m[i]) : "f"(fabsf(d[i])));  // |2v| > 464
  const uint32_t inc = __byte_perm(__byte_perm(m[0], m[1], 0x0040u), __byte_perm(m[2], m[3], 0x0040u), 0x5410u);
  return r + (inc & 0x01010101u);
}

// PTX prmt in its default mode: selector nibble bit 3 replicates the sign bit of the chosen
// byte over all 8 bits (__byte_perm uses only the low 3 bits)
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// packed f16 pair * 0.5 (exact for every e4m3fn value)
__device__ __forceinline__ uint32_t half2_times_half(uint32_t h) {
  __half2 v = *reinterpret_cast<const __half2*>(&h);
  v = __hmul2(v, __float2half2_rn(0.5f));
  return *reinterpret_cast<const uint32_t*>(&v);
}
// packed f16 pair * 128 (exact for the values the fnuz decode builds: at most 1.875 -> 240,
// subnormals become normals)
__device__ __forceinline__ uint32_t half2_times_128(uint32_t h) {
  __half2 v = *reinterpret_cast<const __half2*>(&h);
  v = __hmul2(v, __float2half2_rn(128.0f));
  return *reinterpret_cast<const uint32_t*>(&v);
}

// Four fp8 codes (e4m3fn or e4m3fnuz) -> f32, two codes per conversion
// (cvt.rn.f16x2.e4m3x2, exact), SIMD fix-ups on the packed halves.  e4m3fnuz: the value is
// half the e4m3fn value of the same bits (HMUL2 by 0.5, exact: the smallest fn subnormal
// 2^-9 halves to a normal f16); the codes 0x7F / 0xFF (+-240 in fnuz, NaN in fn) and 0x80
// (NaN in fnuz, -0 in fn) are patched with per-byte masks -- exact zero-byte tests
// ((x & 0x7F..) + 0x7F..) | x, expanded to 16-bit lanes by prmt's sign replication.
// NaN comes out as a NaN; every caller multiplies by the dequant scale next, which
// canonicalises it (reading 12).
#ifndef KVX_FNUZ_SHIFT
#define KVX_FNUZ_SHIFT 1
#endif
#ifndef KVX_FNUZ_FOLD
#define KVX_FNUZ_FOLD 1  // row kernel: e4m3fnuz decode with 2^-7 folded into the source scale
#endif
template <int DT>
__device__ __forceinline__ void fp8x4_to_f32(uint32_t w, float* f) {
  uint32_t h[2];
  if constexpr (DT == KV_F8E4M3FNUZ && KVX_FNUZ_SHIFT) {
    // e4m3fnuz without the fn conversion: a code's 7 magnitude bits (4 exponent, 3
    // mantissa) placed at f16 bits 7..13 with its sign at bit 15 read as an f16 of value
    // 2^-7 times the fnuz value -- normals 2^(e-15) (1 + m/8), subnormals (m/8) 2^-14 --
    // so one exact HMUL2 by 2^7 decodes both, and 0x7F / 0xFF come out as +-240 by
    // themselves (f16's exponent 15 is an ordinary one).  Only 0x80 (fnuz's NaN; -0 here)
    // is patched: an exact per-byte test, expanded to its 16-bit lane by prmt's sign
    // replication, selects the canonical f16 NaN 0x7E00.
    const uint32_t x8 = w ^ 0x80808080u;                           // byte 0 <=> b == 0x80
    const uint32_t y8 = ((x8 & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x8;  // bit 7 clear <=> b == 0x80
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint32_t x = __byte_perm(w, 0u, k ? 0x3424u : 0x1404u);  // codes 2k, 2k+1 at bits 8..15 / 24..31
      const uint32_t y = x >> 1;                                     // sign at 14 / 30, magnitude at 7..13 / 23..29
      const uint32_t hv = half2_times_128(y + (y & 0x40004000u));    // sign moved to 15 / 31
      const uint32_t keep = prmt(y8, 0u, k ? 0xBBAAu : 0x9988u);     // all ones <=> not 0x80
      h[k] = (hv & keep) | (0x7E007E00u & ~keep);
    }
  } else {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const unsigned short in = (unsigned short)(w >> (16 * k));
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h[k]) : "h"(in));
  }
  }
  if constexpr (DT == KV_F8E4M3FNUZ && !KVX_FNUZ_SHIFT) {
    const uint32_t x7 = ~w & 0x7F7F7F7Fu;                          // byte 0 <=> (b & 0x7F) == 0x7F
    const uint32_t y7 = (x7 + 0x7F7F7F7Fu) | x7;                   // bit 7 clear <=> that byte is 0
    const uint32_t x8 = w ^ 0x80808080u;                           // byte 0 <=> b == 0x80
    const uint32_t y8 = ((x8 & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x8;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint32_t hv = half2_times_half(h[k]);
      const uint32_t sel = k ? 0xBBAAu : 0x9988u;                   // sign of bytes 2k, 2k+1 per half
      const uint32_t m7 = ~prmt(y7, 0u, sel), m8 = ~prmt(y8, 0u, sel);
      const uint32_t v240 = (prmt(w, 0u, k ? 0x3424u : 0x1404u) & 0x80008000u) | 0x5B805B80u;  // +-240
      uint32_t r = (hv & ~m7) | (v240 & m7);
      r = (r & ~m8) | (0x7E007E00u & m8);
      h[k] = r;
    }
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float2 ff = __half22float2(*reinterpret_cast<const __half2*>(&h[k]));
    f[2 * k] = ff.x;
    f[2 * k + 1] = ff.y;
  }
}

// Pack VEC f32 values (already scaled) into a DDT chunk (RNE; satfinite for the fp8 types)
template <int DDT, int VEC>
__device__ __forceinline__ void cast_out(const float* f, Chunk<DDT, VEC>& out) {
#pragma unroll
  for (int i = 0; i < Chunk<DDT, VEC>::WORDS; ++i) out.w[i] = 0;
  if constexpr (DDT == KV_F8E4M3) {
    if constexpr (VEC == 1) {
      out.w[0] = f32x2_to_e4m3x2(f[0], 0.0f) & 0xFFu;
    } else {
#pragma unroll
      for (int i = 0; i < VEC; i += 2) out.w[i >> 2] |= f32x2_to_e4m3x2(f[i], f[i + 1]) << ((i & 3) * 8);
    }
  } else if constexpr (DDT == KV_F8E4M3FNUZ) {
    if constexpr (VEC == 1) {
      out.w[0] = f32x2_to_fnuzx2(f[0], 0.0f) & 0xFFu;
    } else if constexpr (VEC % 4 == 0) {
#pragma unroll
      for (int i = 0; i < VEC; i += 4) out.w[i >> 2] = f32x4_to_fnuzx4(f + i);
    } else {
#pragma unroll
      for (int i = 0; i < VEC; i += 2) out.w[i >> 2] |= f32x2_to_fnuzx2(f[i], f[i + 1]) << ((i & 3) * 8);
    }
  } else if constexpr (DDT == KV_F32) {
    // bf16 -> f32 is a bit shift that would keep NaN payloads; reading 12 wants the
    // canonical NaN on every cast output (cvt.f32.f16 and FMUL already canonicalise)
#pragma unroll
    for (int i = 0; i < VEC; ++i) out.w[i] = (f[i] != f[i]) ? 0x7FFFFFFFu : __float_as_uint(f[i]);
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      uint32_t h = (DDT == KV_F16) ? f32_to_f16(f[i]) : f32_to_bf16(f[i]);
      out.w[i >> 1] |= h << ((i & 1) * 16);
    }
  }
}

// e4m3fnuz codes -> 2^-7 x their values as f32, without the NaN patch: each code's 7
// magnitude bits at f16 bits 7..13 with its sign at 15 read as an f16 ARE 2^-7 x the fnuz
// value (normals 2^(e-15)(1 + m/8), subnormals (m/8) 2^-14; 0x7F / 0xFF are +-1.875), and
// the f16 -> f32 widening is exact.  0x80 (fnuz's NaN) decodes to -0 here: callers route
// chunks holding it to the exact decode (fp8x4_to_f32).
__device__ __forceinline__ void fnuzx4_to_f32_scaled(uint32_t w, float* f) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const uint32_t x = __byte_perm(w, 0u, k ? 0x3424u : 0x1404u);  // codes 2k, 2k+1 at bits 8..15 / 24..31
    const uint32_t y = x >> 1;
    const uint32_t h = y + (y & 0x40004000u);                      // sign moved to 15 / 31
    const float2 ff = __half22float2(*reinterpret_cast<const __half2*>(&h));
    f[2 * k] = ff.x;
    f[2 * k + 1] = ff.y;
  }
}
// any byte of w equal to 0x80 (exact: the classic zero-byte test on w ^ 0x80808080)
__device__ __forceinline__ uint32_t has_byte80(uint32_t w) {
  const uint32_t z = w ^ 0x80808080u;
  return (z - 0x01010101u) & ~z & 0x80808080u;
}

// Cast a chunk SDT -> DDT.  ssc: dequant scale of an fp8 source; inv: RN(1/s) of an fp8
// destination (an fp8 -> other-fp8 cast applies both, in that order).
// FOLD (e4m3fnuz sources in the row kernel): ssc arrives as 2^7 s (exact) -- the decode's
// 2^-7 is folded into it, so RN(f32(2^-7 q) * 2^7 s) = RN(q * s) with no separate rescale --
// or as -s when 2^7 s would overflow; a chunk with a 0x80 code (NaN) or a negative ssc
// takes the exact per-code decode with the plain scale instead (rare: not on random data).
template <int SDT, int DDT, int VEC, bool FOLD = false>
__device__ __forceinline__ void cast_chunk(const Chunk<SDT, VEC>& in, Chunk<DDT, VEC>& out, float ssc, float inv) {
  if constexpr (FOLD && SDT == KV_F8E4M3FNUZ && DDT != KV_F8E4M3FNUZ && VEC % 4 == 0) {
    uint32_t nan = 0;
#pragma unroll
    for (int i = 0; i < VEC; i += 4) nan |= has_byte80(in.w[i >> 2]);
    if (nan == 0 && ssc >= 0.f) {
      float f[VEC];
#pragma unroll
      for (int i = 0; i < VEC; i += 4) fnuzx4_to_f32_scaled(in.w[i >> 2], f + i);
#pragma unroll
      for (int i = 0; i < VEC; i += 2) {
        fmul2_rn(f[i], f[i + 1], ssc);
        if constexpr (is_fp8(DDT)) fmul2_rn(f[i], f[i + 1], inv);
      }
      cast_out<DDT, VEC>(f, out);
    } else {
      cast_chunk<SDT, DDT, VEC, false>(in, out, ssc >= 0.f ? __fmul_rn(ssc, 0.0078125f) : -ssc, inv);
    }
    return;
  }
  if constexpr (SDT == DDT) {
#pragma unroll
    for (int i = 0; i < Chunk<SDT, VEC>::WORDS; ++i) out.w[i] = in.w[i];
  } else {
    float f[VEC];
    if constexpr (is_fp8(SDT) && VEC % 4 == 0) {
#pragma unroll
      for (int i = 0; i < VEC; i += 4) fp8x4_to_f32<SDT>(in.w[i >> 2], f + i);
    } else {
#pragma unroll
      for (int i = 0; i < VEC; ++i) f[i] = to_f32<SDT>(get_elem<SDT>(in.w, i));
    }
    if constexpr (VEC % 2 == 0) {
#pragma unroll
      for (int i = 0; i < VEC; i += 2) {
        if constexpr (is_fp8(SDT)) fmul2_rn(f[i], f[i + 1], ssc);
        if constexpr (is_fp8(DDT)) fmul2_rn(f[i], f[i + 1], inv);
      }
    } else {
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        if constexpr (is_fp8(SDT)) f[i] = __fmul_rn(f[i], ssc);
        if constexpr (is_fp8(DDT)) f[i] = __fmul_rn(f[i], inv);
      }
    }
    cast_out<DDT, VEC>(f, out);
  }
}

template <int DT, int VEC>
__device__ __forceinline__ void zero_chunk(Chunk<DT, VEC>& c) {
#pragma unroll
  for (int i = 0; i < Chunk<DT, VEC>::WORDS; ++i) c.w[i] = 0;
}
// zero elements [k, VEC) of a chunk (slots past the request's last token)
template <int DT, int VEC>
__device__ __forceinline__ void zero_tail(Chunk<DT, VEC>& c, uint32_t k) {
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    if ((uint32_t)i < k) continue;
    if constexpr (Tr<DT>::B == 4) c.w[i] = 0u;
    else if constexpr (Tr<DT>::B == 2) c.w[i >> 1] &= ~(0xFFFFu << ((i & 1) * 16));
    else c.w[i >> 2] &= ~(0xFFu << ((i & 3) * 8));
  }
}

__device__ __forceinline__ uint32_t divmod(uint32_t& n, const FastDiv& f) {
  uint32_t q = fdiv(n, f);
  uint32_t r = n - q * f.d;
  n = q;
  return r;
}

// element offset of head_dim index d: (d >> dk) * stride + (d & (2^dk - 1)) -- the x-split
// head_dim of reading 27 (dk = log2 x; 0: unsplit, d * stride)
__device__ __forceinline__ int64_t dim_off(uint32_t d, int64_t stride, int32_t dk) {
  return (int64_t)(d >> dk) * stride + (int64_t)(d & ((1u << dk) - 1u));
}

// K/V entries per layer on the wire (Fig. 5 order over the K/V both pools hold)
__device__ __forceinline__ uint32_t wkv(int32_t kv1) { return kv1 ? 1u : 2u; }

// K/V index of an item: both (n's lowest digit) or, for a K-only / V-only transfer
// (kv1 != 0, reading 27), always c0 with no digit in n
__device__ __forceinline__ uint32_t take_kv(uint32_t& n, int32_t kv1, int32_t c0) {
  if (kv1) return (uint32_t)c0;
  const uint32_t c = n & 1u;
  n >>= 1;
  return c;
}

constexpr int kThreads = 256;
#ifndef KVX_MINB
#define KVX_MINB 4  // >= 4 CTAs/SM for the row kernel: caps it at 64 registers (the 2-byte -> e4m3
                    // instantiation otherwise takes 76 and drops to 3 CTAs/SM, 0.87 instead of 0.95)
#endif
#ifndef KVX_MINB_WIDEN
#define KVX_MINB_WIDEN 3  // fp8 -> wider casts: 3 CTAs/SM (up to 85 registers) keep more bytes in
                          // flight (e4m3fnuz -> bf16 0.915 -> 0.956 of copy; 4 stays best for the
                          // rest: profiles/r01/minb_occupancy_ab.txt)
#endif
constexpr int row_minb(int sdt, int ddt) { return is_fp8(sdt) && !is_fp8(ddt) ? KVX_MINB_WIDEN : KVX_MINB; }

// ------------------------------------------------------------------------------------
// K1/K4: fused pool -> pool convert (+ reshard, + cast, + tail zero-fill)
// chunk index (fastest first): dim-chunk, {slot, head} (dst-contiguous order), K/V,
// layer, dst block (flattened over the batch), dst rank index.
// ------------------------------------------------------------------------------------
template <int VEC, int SDT, int DDT, int U>
__global__ void __launch_bounds__(kThreads) k_convert(const __grid_constant__ ConvArgs a) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = (blockIdx.x * (uint32_t)kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * (uint32_t)kThreads) >> 5;
  const uint64_t total = a.total;
  const uint64_t nseg = (total + 32u * U - 1) / (32u * U);
  for (uint64_t seg = warp; seg < nseg; seg += nwarps) {
    Chunk<SDT, VEC> in[U];
    uint8_t* dp[U];
    float ssc[U], inv[U];
    bool act[U], zero[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint64_t g64 = seg * (32u * U) + (uint32_t)k * 32u + lane;
      act[k] = g64 < total;
      zero[k] = false;
      dp[k] = nullptr;
      ssc[k] = 1.f;
      inv[k] = 1.f;
      if (act[k]) {
        uint32_t n = (uint32_t)g64;
        const uint32_t dch = divmod(n, a.f_dch);
        const uint32_t in0 = divmod(n, a.f_in0);
        const uint32_t in1 = divmod(n, a.f_in1);
        const uint32_t c = take_kv(n, a.kv1, a.c0);
        const uint32_t l = divmod(n, a.f_l);
        const uint32_t bl = divmod(n, a.f_bl);
        const uint32_t qi = n;
        const uint32_t slot = a.slot_inner ? in0 : in1;
        const uint32_t hq = (uint32_t)a.hq_off[qi] + (a.slot_inner ? in1 : in0);
        const int32_t r = __ldg(a.d_blk_req + bl);
        const int32_t tok0 = __ldg(a.tok_off + r);
        const int32_t T = __ldg(a.tok_off + r + 1) - tok0;
        const uint32_t t = (uint32_t)(bl - __ldg(a.d_blk_off + r)) * (uint32_t)a.Bd + slot;
        const int64_t dblk = __ldg(a.d_blk_ids + bl);
        const int64_t layer = a.lb + (int64_t)l;
        const int64_t sl = layer - a.s_l0, dl = layer - a.d_l0;  // pool-local layers
        const int64_t doff = dl * a.ds[KV_AX_LAYER] + (int64_t)c * a.ds[KV_AX_KV] + dblk * a.ds[KV_AX_BLOCK] +
                             (int64_t)slot * a.ds[KV_AX_SLOT] + (int64_t)hq * a.ds[KV_AX_HEAD] +
                             dim_off(dch * VEC, a.ds[KV_AX_DIM], a.d_dk);
        dp[k] = a.dst[qi] + doff * Tr<DDT>::B;
        if ((int32_t)t >= T) {
          zero[k] = true;
        } else {
          const uint32_t h = (uint32_t)a.dst_rank[qi] * (uint32_t)a.Hd + hq;
          const uint32_t p = fdiv(h, a.f_hp);
          const uint32_t hp = h - p * (uint32_t)a.Hp;
          const int si = a.src_of_p[p];
          uint32_t tb = t;
          const uint32_t sslot = divmod(tb, a.f_bp);
          const int64_t sblk = __ldg(a.s_blk_ids + __ldg(a.s_blk_off + r) + tb);
          const int64_t soff = sl * a.ss[KV_AX_LAYER] + (int64_t)c * a.ss[KV_AX_KV] +
                               sblk * a.ss[KV_AX_BLOCK] + (int64_t)sslot * a.ss[KV_AX_SLOT] +
                               (int64_t)hp * a.ss[KV_AX_HEAD] + dim_off(dch * VEC, a.ss[KV_AX_DIM], a.s_dk);
          load_chunk<SDT, VEC>(in[k], a.src[si] + soff * Tr<SDT>::B);
          if constexpr (is_fp8(SDT) && SDT != DDT)
            ssc[k] = __ldg(a.sscale[si] + (sl * 2 + c) * a.Hp + hp);
          if constexpr (is_fp8(DDT) && SDT != DDT)
            inv[k] = __frcp_rn(__ldg(a.dscale[qi] + (dl * 2 + c) * a.Hd + hq));
        }
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (!act[k]) continue;
      Chunk<DDT, VEC> o;
      if (zero[k])
        zero_chunk(o);
      else
        cast_chunk<SDT, DDT, VEC>(in[k], o, ssc[k], inv[k]);
      store_chunk<DDT, VEC>(dp[k], o);
    }
  }
}

// ------------------------------------------------------------------------------------
// Shared inner loop of the row kernels.  Lane i holds the state of row i of a 32-row
// item: source row address sp, destination row address dp, its scale rsc and rz
// (0 copy, 1 zero-fill tail row, 2 no row).  The warp streams the 32 x 2^cs chunks of
// 16 B (source side) with U loads in flight per lane, fetching row state by shuffles.
// rsc is the one fp8 scale a cast needs (source dequant scale, or RN(1/s) of an fp8
// destination); an fp8 -> other-fp8 cast takes the source scale in rsc and RN(1/s_dst) in
// rsc2 (the only instantiations that carry the second register).
// ------------------------------------------------------------------------------------
// Where chunk ch of a row lives when head_dim is x-split (reading 27): chunk ch covers
// elements [8ch, 8ch + 8), which sit in x-group ch >> k (k = log2(x / 8)) at byte stride hs,
// at (ch & (2^k - 1)) * 8 elements inside it.  Unsplit: k = 0, hs = 8 * element bytes.
struct ChunkMap {
  int32_t sk, dk;
  int64_t shs, dhs;
};

template <int SDT, int DDT, int U, int VEC = 8, bool COH = false, bool SPLIT = false, bool FOLD = false>
__device__ __forceinline__ void stream_rows(uint32_t lane, uint32_t cs, uint64_t sp, uint64_t dp, float rsc,
                                            uint32_t rz, float rsc2 = 1.f, const ChunkMap* cm = nullptr) {
  constexpr bool DUAL = dual_scale(SDT, DDT);
  const uint32_t cmask = (1u << cs) - 1u;
  const uint32_t nch = 32u << cs;
  for (uint32_t base = 0; base < nch; base += 32u * U) {
    Chunk<SDT, VEC> in[U];
    uint64_t d[U];
    float sc[U], sc2[DUAL ? U : 1];
    uint32_t z[U], ch[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint32_t idx = base + (uint32_t)k * 32u + lane;
      const uint32_t rr = (idx >> cs) & 31u;
      ch[k] = idx & cmask;
      const uint64_t s = __shfl_sync(0xffffffffu, sp, rr);
      d[k] = __shfl_sync(0xffffffffu, dp, rr);
      z[k] = __shfl_sync(0xffffffffu, rz, rr) | (idx >= nch ? 2u : 0u);
      sc[k] = __shfl_sync(0xffffffffu, rsc, rr);
      if constexpr (DUAL) sc2[k] = __shfl_sync(0xffffffffu, rsc2, rr);
      uint64_t soff = ch[k] * (VEC * Tr<SDT>::B);
      if constexpr (SPLIT)
        soff = (uint64_t)(ch[k] >> cm->sk) * (uint64_t)cm->shs + (ch[k] & ((1u << cm->sk) - 1u)) * (VEC * Tr<SDT>::B);
      if (z[k] == 0) load_chunk<SDT, VEC, COH>(in[k], reinterpret_cast<const uint8_t*>(s) + soff);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (z[k] & 2u) continue;
      Chunk<DDT, VEC> o;
      if (z[k])
        zero_chunk(o);
      else if constexpr (DUAL)
        cast_chunk<SDT, DDT, VEC, FOLD>(in[k], o, sc[k], sc2[k]);
      else
        cast_chunk<SDT, DDT, VEC, FOLD>(in[k], o, sc[k], sc[k]);
      uint64_t doff = ch[k] * (VEC * Tr<DDT>::B);
      if constexpr (SPLIT)
        doff = (uint64_t)(ch[k] >> cm->dk) * (uint64_t)cm->dhs + (ch[k] & ((1u << cm->dk) - 1u)) * (VEC * Tr<DDT>::B);
      store_chunk<DDT, VEC>(reinterpret_cast<uint8_t*>(d[k]) + doff, o);
    }
  }
}

// ------------------------------------------------------------------------------------
// K1/K4 fast path (head_dim innermost on both sides, D/8 a power of two): row-tiled.
// A work item is 32 head_dim rows of one (dst rank, dst block, layer, K/V) tile.  The
// tile-level decode (request, block ids, base pointers) is warp-uniform; then each lane
// decodes ONE row (source / destination row pointers, tail flag, fp8 scale) and the warp
// streams the item's 32 x cpr chunks, fetching row state with register shuffles -- so
// the per-16-byte work is a few shuffles, one load, the cast and one store.  Each warp
// instruction covers cpr consecutive chunks of 32/cpr rows: contiguous per row on both
// sides.  U chunk loads per lane are in flight before the first store.
// ------------------------------------------------------------------------------------
// Per-lane row state of convert item `item` (see k_convert_rows): lane = row of the
// 2-D sub-tile.  rz: 0 copy, 1 zero-fill tail row, 2 no row.
__device__ __forceinline__ uint64_t gtimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// 2^7 s for the folded e4m3fnuz decode (exact), or -s when it would overflow (cast_chunk)
__device__ __forceinline__ float fnuz_fold_scale(float s) {
  const float f = __fmul_rn(s, 128.0f);
  return f <= 3.402823466e38f ? f : -s;
}

template <int SDT, int DDT, bool FOLD = false>
__device__ __forceinline__ void conv_row(const ConvArgs& a, uint32_t item, uint32_t lane, uint64_t& sp,
                                         uint64_t& dp, float& rsc, uint32_t& rz, float& rsc2,
                                         int32_t* req_out = nullptr, uint32_t* tbl_out = nullptr) {
  // destination fastest: with several D ranks (fan-out, e.g. a TP split pushed over
  // NVLink) concurrent warps write every destination at once instead of one link after
  // the other -- with the D rank outermost, all P ranks of a fan-in/fan-out hit the same
  // D rank's ingress together and c5' ran at 0.56 of the link
  uint32_t n = item;
  const uint32_t qi = divmod(n, a.f_nd);
  const uint32_t rg = divmod(n, a.f_items);
  const uint32_t c = take_kv(n, a.kv1, a.c0);
  const uint32_t l = divmod(n, a.f_l);
  const uint32_t bl = n;
  const int32_t r = __ldg(a.d_blk_req + bl);
  if (req_out) *req_out = r;
  const int32_t tok0 = __ldg(a.tok_off + r);
  const int32_t T = __ldg(a.tok_off + r + 1) - tok0;
  const uint32_t tb0 = (uint32_t)(bl - __ldg(a.d_blk_off + r)) * (uint32_t)a.Bd;  // first token of the block
  const int64_t layer = a.lb + (int64_t)l;
  const int64_t sl = layer - a.s_l0, dl = layer - a.d_l0;  // pool-local layers
  // the item is a 2-D sub-tile of ts slots x th heads (ts * th = 32): both the source
  // and the destination see runs of several rows instead of single 256-B rows
  uint32_t sbk = rg;
  const uint32_t s_blk = divmod(sbk, a.f_sb);  // sub-tile index along slots; sbk = along heads
  const uint32_t ts_log2 = (uint32_t)a.ts_log2;
  const uint32_t ls = a.slot_inner ? (lane & ((1u << ts_log2) - 1u)) : (lane >> (5u - ts_log2));
  const uint32_t lh = a.slot_inner ? (lane >> ts_log2) : (lane & ((1u << (5u - ts_log2)) - 1u));
  const uint32_t slot = (s_blk << ts_log2) + ls;
  const uint32_t hl = (sbk << (5u - ts_log2)) + lh;  // head within the converted range
  // (dst index, layer, K/V, head) table of the LUT requantisation (k_requant_rows)
  if (tbl_out) *tbl_out = ((l * a.f_nd.d + qi) * (a.kv1 ? 1u : 2u) + (a.kv1 ? 0u : c)) * (uint32_t)a.Hd_eff + hl;
  const uint32_t hq = (uint32_t)a.hq_off[qi] + hl;      // D-local head
  sp = 0;
  dp = 0;
  rsc = 1.f;  // fp8 destination: RN(1/s); fp8 source: s (both fp8: s_src, and rsc2 = RN(1/s_dst))
  rsc2 = 1.f;
  rz = 2;
  if (slot < (uint32_t)a.Bd && hl < (uint32_t)a.Hd_eff) {
    rz = 0;
    const int64_t dblk = __ldg(a.d_blk_ids + bl);
    dp = (uint64_t)(a.dst[qi] + (dl * a.ds[KV_AX_LAYER] + (int64_t)c * a.ds[KV_AX_KV] + dblk * a.ds[KV_AX_BLOCK] +
                                 (int64_t)slot * a.ds[KV_AX_SLOT] + (int64_t)hq * a.ds[KV_AX_HEAD]) * Tr<DDT>::B);
    const uint32_t t = tb0 + slot;
    if ((int32_t)t >= T) {
      rz = 1;
    } else {
      const uint32_t h = (uint32_t)a.dst_rank[qi] * (uint32_t)a.Hd + hq;
      const uint32_t p = fdiv(h, a.f_hp);
      const uint32_t hp = h - p * (uint32_t)a.Hp;
      const int si = a.src_of_p[p];
      uint32_t tb = t;
      const uint32_t sslot = divmod(tb, a.f_bp);
      const int64_t sblk = __ldg(a.s_blk_ids + __ldg(a.s_blk_off + r) + tb);
      sp = (uint64_t)(a.src[si] + (sl * a.ss[KV_AX_LAYER] + (int64_t)c * a.ss[KV_AX_KV] + sblk * a.ss[KV_AX_BLOCK] +
                                   (int64_t)sslot * a.ss[KV_AX_SLOT] + (int64_t)hp * a.ss[KV_AX_HEAD]) * Tr<SDT>::B);
      if constexpr (dual_scale(SDT, DDT)) {
        rsc = __ldg(a.sscale[si] + (sl * 2 + c) * a.Hp + hp);
        rsc2 = __frcp_rn(__ldg(a.dscale[qi] + (dl * 2 + c) * a.Hd + hq));
      } else {
        if constexpr (is_fp8(SDT) && SDT != DDT) rsc = __ldg(a.sscale[si] + (sl * 2 + c) * a.Hp + hp);
        if constexpr (is_fp8(DDT) && SDT != DDT) rsc = __frcp_rn(__ldg(a.dscale[qi] + (dl * 2 + c) * a.Hd + hq));
      }
      if constexpr (FOLD) rsc = fnuz_fold_scale(rsc);
    }
  }
}

template <int SDT, int DDT, int U, int VEC = 8, bool SPLIT = false>
__global__ void __launch_bounds__(kThreads, row_minb(SDT, DDT)) k_convert_rows(const __grid_constant__ ConvArgs a) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = (blockIdx.x * (uint32_t)kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * (uint32_t)kThreads) >> 5;
  const uint32_t cs = (uint32_t)a.cpr_shift;
  const ChunkMap cm{a.s_ck, a.d_ck, a.s_chs, a.d_chs};
  // e4m3fnuz source to another type: the decode's 2^-7 folded into the source scale
  constexpr bool FOLD = KVX_FNUZ_FOLD && SDT == KV_F8E4M3FNUZ && DDT != KV_F8E4M3FNUZ && VEC % 4 == 0;
  for (uint32_t item = warp; item < a.n_items; item += nwarps) {
    uint64_t sp, dp;
    float rsc, rsc2;
    uint32_t rz;
    int32_t r;
    conv_row<SDT, DDT, FOLD>(a, item, lane, sp, dp, rsc, rz, rsc2, &r);
    stream_rows<SDT, DDT, U, VEC, false, SPLIT, FOLD>(lane, cs, sp, dp, rsc, rz, rsc2, &cm);
    if (a.req_cnt) {
      // per-request completion (kv_convert_reshard_notify): the warp finishing request r's
      // last item publishes it -- its rows' stores are fenced before the count, and the
      // last counter owner fences system-wide before the release store of the flag
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        const uint32_t tot = (uint32_t)(__ldg(a.d_blk_off + r + 1) - __ldg(a.d_blk_off + r)) * a.items_per_block;
        if (atomicAdd(a.req_cnt + r, 1u) + 1u == tot) {
          __threadfence_system();
          if (a.req_ns) a.req_ns[r] = gtimer_ns();
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.req_flag + r), "r"(a.req_epoch) : "memory");
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// TMA / bulk-copy helpers (k_tile_copy).  A per-row TMA-staged variant of the convert
// (one cp.async.bulk per 256-B row into smem) was measured at 0.61 of copy on c2 and 0.27
// with a cast (profiles/r01/tma_variant_ab.txt) and removed.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_arrive(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem_src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_store_hint(void* gdst, const void* smem_src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }


// ------------------------------------------------------------------------------------
// K1/K4 same-dtype TMA tile path (k_tile_copy).  One warp per CTA is a copy engine: per
// item (dst rank, P rank share, source block within the dst block, K/V, layer, dst block)
// lane 0 issues ONE cp.async.bulk.tensor.5d load of the whole source sub-tile (nh heads x Bp
// slots x D) whose tensor map enumerates the source pool in the DESTINATION's inner order,
// so the sub-tile lands in smem already permuted; tail slots are zeroed in smem; then the
// lanes issue cp.async.bulk stores of D's contiguous runs (one run when the sub-tile is a
// whole dst head range).  No register pass, 8-64 KB per TMA operation, `stages` items in
// flight per CTA.  A partial sub-tile (the request's last block) takes its valid rows by
// plain loads instead (tile_rows_ldg): no source tail slot is read; D's tail rows are zeroed.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void tma_load_5d(void* smem_dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            int32_t c2, int32_t c3, int32_t c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::
          "r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_5d_hint(void* smem_dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                                 int32_t c2, int32_t c3, int32_t c4, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::
          "r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// The valid rows (slots < valid) of a partial source sub-tile -- the request's last block --
// by plain 16-B loads of the whole warp into the stage, in the box's order ([nh][Bp][D]
// when head_major, else [Bp][nh][D]).  The TMA box would read all Bp slots: the tail slots
// are never read (reading 5).  Rare (one per request, layer, K/V and head group).
__device__ __forceinline__ void tile_rows_ldg(const TileArgs& a, uint8_t* sbuf, int si, int32_t c, int32_t sblk,
                                              int32_t sl, int32_t hp0, uint32_t valid, uint32_t lane) {
  const int64_t* st = a.ss[si];
  const uint32_t esize = (uint32_t)a.esize, nh = (uint32_t)a.nh, Bp = (uint32_t)a.Bp;
  const uint32_t row_bytes = (uint32_t)a.D * esize, r16 = row_bytes / 16u;
  const uint8_t* base = a.src[si] + (sl * st[KV_AX_LAYER] + (int64_t)c * st[KV_AX_KV] + (int64_t)sblk * st[KV_AX_BLOCK] +
                                     (int64_t)hp0 * st[KV_AX_HEAD]) * esize;
  for (uint32_t z = lane; z < valid * nh * r16; z += 32u) {
    const uint32_t row = z / r16, piece = z - row * r16;
    const uint32_t slot = row / nh, head = row - slot * nh;
    const uint32_t ri = a.head_major ? head * Bp + slot : slot * nh + head;
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(
        base + ((int64_t)slot * st[KV_AX_SLOT] + (int64_t)head * st[KV_AX_HEAD]) * esize + piece * 16u));
    *reinterpret_cast<uint4*>(sbuf + (size_t)ri * row_bytes + piece * 16u) = v;
  }
  fence_proxy_async();  // generic writes ordered before later async-proxy use of the stage
  __syncwarp();
}

__global__ void __launch_bounds__(32) k_tile_copy(const __grid_constant__ TileArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint64_t pol = a.evict_first ? policy_evict_first() : 0ull;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t S = (uint32_t)a.stages;
  const uint32_t SB = (uint32_t)a.stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)S * SB);
  if (lane == 0)
    for (uint32_t s = 0; s < S; ++s) mbar_init(bars + s, 1);
  fence_proxy_async();
  __syncwarp();
  const uint32_t my = blockIdx.x < a.n_items ? (a.n_items - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const uint32_t row_bytes = (uint32_t)a.D * (uint32_t)a.esize;

  struct Item {
    uint8_t* dbase;    // destination address of the sub-tile's first run
    int64_t run_gap;   // bytes between consecutive runs in the destination
    uint32_t nruns, run_bytes, valid;  // valid: source slots < T in this block (0 = no source)
  };
  auto decode = [&](uint32_t item, Item& it, int& si, int32_t& c0, int32_t& c1, int32_t& c2, int32_t& c3,
                    int32_t& c4, uint32_t& c) {
    uint32_t n = item;
    const uint32_t qi = divmod(n, a.f_nd);
    const uint32_t part = divmod(n, a.f_parts);
    const uint32_t sub = divmod(n, a.f_sub);
    c = take_kv(n, a.kv1, a.c0);
    const uint32_t l = divmod(n, a.f_l);
    const uint32_t bl = n;
    const int32_t r = __ldg(a.d_blk_req + bl);
    const int32_t tok0 = __ldg(a.tok_off + r);
    const int32_t T = __ldg(a.tok_off + r + 1) - tok0;
    const int32_t j = bl - __ldg(a.d_blk_off + r);
    const int64_t dblk = __ldg(a.d_blk_ids + bl);
    const int32_t layer = a.lb + (int32_t)l;
    const int32_t q = a.dst_rank[qi];
    // head group `part` of nh heads: from the D rank's first head, or (share) from the first
    // head this P rank holds of it; its P rank and local head offsets on both sides
    const int32_t hstart = a.share_p >= 0 ? max(a.share_p * a.Hp, q * a.Hd) : q * a.Hd;
    const int32_t h0 = hstart + (int32_t)part * a.nh;
    const int32_t p = a.share_p >= 0 ? a.share_p : h0 / a.Hp;
    const int32_t hp0 = h0 - p * a.Hp, hq0 = h0 - q * a.Hd;
    si = a.src_of_p[p];
    const int32_t t0 = j * a.Bd + (int32_t)sub * a.Bp;
    it.valid = t0 >= T ? 0u : (uint32_t)min(a.Bp, T - t0);
    int32_t sblk = 0;
    if (it.valid) sblk = __ldg(a.s_blk_ids + __ldg(a.s_blk_off + r) + (j * (a.Bd / a.Bp) + (int32_t)sub));
    const int64_t dl = layer - a.d_l0;
    uint8_t* tile = a.dst[qi] + (dl * a.ds[KV_AX_LAYER] + (int64_t)c * a.ds[KV_AX_KV] + dblk * a.ds[KV_AX_BLOCK]) * a.esize;
    if (a.head_major) {  // D inner (HEAD, SLOT, DIM): one run per head of Bp rows
      it.dbase = tile + ((int64_t)hq0 * a.ds[KV_AX_HEAD] + (int64_t)sub * a.Bp * a.ds[KV_AX_SLOT]) * a.esize;
      it.run_gap = a.ds[KV_AX_HEAD] * a.esize;
      it.nruns = (uint32_t)a.nh;
      it.run_bytes = (uint32_t)a.Bp * row_bytes;
      if (a.Bp == a.Bd) {  // whole head rows: the nh runs are back to back
        it.run_bytes *= it.nruns;
        it.nruns = 1;
      }
      c1 = 0;
      c2 = hp0;
    } else {  // D inner (SLOT, HEAD, DIM): one run per slot of nh rows
      it.dbase = tile + ((int64_t)sub * a.Bp * a.ds[KV_AX_SLOT] + (int64_t)hq0 * a.ds[KV_AX_HEAD]) * a.esize;
      it.run_gap = a.ds[KV_AX_SLOT] * a.esize;
      it.nruns = (uint32_t)a.Bp;
      it.run_bytes = (uint32_t)a.nh * row_bytes;
      if (a.nh == a.Hd) {
        it.run_bytes *= it.nruns;
        it.nruns = 1;
      }
      c1 = hp0;
      c2 = 0;
    }
    c0 = 0;
    c3 = sblk;
    c4 = layer - a.s_l0;
  };

  Item it[8];  // per stage (S <= 8)
  auto issue = [&](uint32_t k, uint32_t s) {
    int si;
    int32_t c0, c1, c2, c3, c4;
    uint32_t c;
    decode(blockIdx.x + k * gridDim.x, it[s], si, c0, c1, c2, c3, c4, c);
    const uint32_t v = it[s].valid;
    if (v > 0u && v < (uint32_t)a.Bp)  // partial: valid rows only, then a plain arrive
      tile_rows_ldg(a, smem + (size_t)s * SB, si, (int32_t)c, c3, c4, a.head_major ? c2 : c1, v, lane);
    if (lane == 0) {
      mbar_expect_tx_arrive(bars + s, v == (uint32_t)a.Bp ? SB : 0u);
      if (v == (uint32_t)a.Bp) {
        if (a.evict_first)
          tma_load_5d_hint(smem + (size_t)s * SB, &a.maps[si][c], c0, c1, c2, c3, c4, bars + s, pol);
        else
          tma_load_5d(smem + (size_t)s * SB, &a.maps[si][c], c0, c1, c2, c3, c4, bars + s);
      }
    }
  };
  for (uint32_t k = 0; k < my && k < S; ++k) issue(k, k);
  for (uint32_t k = 0; k < my; ++k) {
    const uint32_t s = k % S;
    mbar_wait(bars + s, (k / S) & 1u);
    uint8_t* buf = smem + (size_t)s * SB;
    const Item& cur = it[s];
    if (cur.valid < (uint32_t)a.Bp) {  // zero the rows of slots >= T (and whole sub-tiles past T)
      const uint32_t v = cur.valid, nh = (uint32_t)a.nh, Bp = (uint32_t)a.Bp;
      const uint32_t r16 = row_bytes / 16;
      const uint32_t zrows = (Bp - v) * nh;
      for (uint32_t z = lane; z < zrows * r16; z += 32) {
        const uint32_t row = z / r16, piece = z - row * r16;
        const uint32_t slot = v + row / nh, head = row - (row / nh) * nh;
        const uint32_t ri = a.head_major ? head * Bp + slot : slot * nh + head;
        *reinterpret_cast<uint4*>(buf + (size_t)ri * row_bytes + piece * 16) = make_uint4(0, 0, 0, 0);
      }
      fence_proxy_async();  // generic writes visible to the bulk stores
      __syncwarp();
    }
    for (uint32_t run = lane; run < cur.nruns; run += 32)
      if (a.evict_first)
        bulk_store_hint(cur.dbase + (int64_t)run * cur.run_gap, buf + (size_t)run * cur.run_bytes, cur.run_bytes, pol);
      else
        bulk_store(cur.dbase + (int64_t)run * cur.run_gap, buf + (size_t)run * cur.run_bytes, cur.run_bytes);
    bulk_commit();
    // reload the stage consumed in the previous iteration once its stores have read it
    bulk_wait_read<1>();
    __syncwarp();
    if (k >= 1 && k - 1 + S < my) issue(k - 1 + S, (k - 1) % S);
  }
  bulk_wait_all();
}

// ------------------------------------------------------------------------------------
// K1 with a head_dim-major side (reading 27): a pool whose two innermost axes are
// (DIM, SLOT) -- the value cache of other vendors' paged-attention kernels, V [blocks,
// heads, D, block] -- stores one (block, head) tile as D rows of B slots, so a token's
// head_dim row is strided.  One warp per item = (dst rank, dst block, layer, K/V, dst
// head): it loads the item's source tile(s) with 8-element vector loads into shared memory
// in [slot][d] order (scattering each (d, 8 slots) vector when the source is head_dim-
// major), then writes the destination tile with 8-element vector stores (gathering 8 slots
// of one d when the destination is head_dim-major), casting on the way; tail slots are
// zero.  The transpose costs shared-memory traffic only; HBM sees whole-tile reads and
// writes.
// ------------------------------------------------------------------------------------
#ifndef KVX_TR_WARPS
#define KVX_TR_WARPS 4
#endif
constexpr int kTrWarps = KVX_TR_WARPS;

template <int SDT, int DDT>
#ifndef KVX_TR_MINB
#define KVX_TR_MINB 8  // 8 CTAs x 4 warps: caps it at 64 registers (0.707 -> 0.732 on the vendor K+V case)
#endif
#if KVX_TR_MINB > 0
__global__ void __launch_bounds__(kTrWarps * 32, KVX_TR_MINB) k_convert_tr(const __grid_constant__ ConvArgs a) {
#else
__global__ void __launch_bounds__(kTrWarps * 32) k_convert_tr(const __grid_constant__ ConvArgs a) {
#endif
  extern __shared__ __align__(16) uint8_t tr_smem[];
  constexpr int VEC = 8;
  constexpr uint32_t SB = Tr<SDT>::B;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t wl = threadIdx.x >> 5;
  const uint32_t warp = blockIdx.x * kTrWarps + wl;
  const uint32_t nwarps = gridDim.x * kTrWarps;
  // every extent below is a power of two (checked by the caller): index math is shifts
  const uint32_t lbp = (uint32_t)a.tr_lbp, lbd = (uint32_t)a.tr_lbd, lcpr = (uint32_t)a.cpr_shift;
  const uint32_t Bp = 1u << lbp, Bd = 1u << lbd;
  const uint32_t D = (uint32_t)a.D;
  const uint32_t LD = D + 16u / SB;  // padded smem row (elements): 16 B of padding per slot row
  uint8_t* tile = tr_smem + (size_t)wl * Bd * LD * SB;
  const uint32_t lsm = (uint32_t)a.s_lm, ldm = (uint32_t)a.d_lm;  // log2(x / 8) per side (mode 2)
  for (uint32_t item = warp; item < a.n_items; item += nwarps) {
    uint32_t n = item;
    const uint32_t hl = divmod(n, a.f_hde);
    const uint32_t c = take_kv(n, a.kv1, a.c0);
    const uint32_t l = divmod(n, a.f_l);
    const uint32_t bl = divmod(n, a.f_bl);
    const uint32_t qi = n;
    const uint32_t hq = (uint32_t)a.hq_off[qi] + hl;
    const int32_t r = __ldg(a.d_blk_req + bl);
    const int32_t tok0 = __ldg(a.tok_off + r);
    const int32_t T = __ldg(a.tok_off + r + 1) - tok0;
    const uint32_t tb0 = (uint32_t)(bl - __ldg(a.d_blk_off + r)) << lbd;  // first token of the dst block
    const int64_t layer = a.lb + (int64_t)l;
    const int64_t sl = layer - a.s_l0, dl = layer - a.d_l0;
    const uint32_t h = (uint32_t)a.dst_rank[qi] * (uint32_t)a.Hd + hq;
    const uint32_t p = fdiv(h, a.f_hp);
    const uint32_t hp = h - p * (uint32_t)a.Hp;
    const int si = a.src_of_p[p];
    float rsc = 1.f, rsc2 = 1.f;
    if constexpr (dual_scale(SDT, DDT)) {
      rsc = __ldg(a.sscale[si] + (sl * 2 + c) * a.Hp + hp);
      rsc2 = __frcp_rn(__ldg(a.dscale[qi] + (dl * 2 + c) * a.Hd + hq));
    } else {
      if constexpr (is_fp8(SDT) && SDT != DDT) rsc = __ldg(a.sscale[si] + (sl * 2 + c) * a.Hp + hp);
      if constexpr (is_fp8(DDT) && SDT != DDT) rsc = __frcp_rn(__ldg(a.dscale[qi] + (dl * 2 + c) * a.Hd + hq));
    }
    const uint32_t valid = (int32_t)tb0 >= T ? 0u : min(Bd, (uint32_t)T - tb0);  // slots with data
    // ---- load: the source blocks covering [tb0, tb0 + valid) into tile[slot][d] ----
    const uint32_t nsrc = (valid + Bp - 1) >> lbp;
    const int32_t* sids = a.s_blk_ids + __ldg(a.s_blk_off + r) + (int32_t)(tb0 >> lbp);
    for (uint32_t j = 0; j < nsrc; ++j) {
      const int64_t sblk = __ldg(sids + j);
      const uint8_t* sb = a.src[si] + (sl * a.ss[KV_AX_LAYER] + (int64_t)c * a.ss[KV_AX_KV] +
                                       sblk * a.ss[KV_AX_BLOCK] + (int64_t)hp * a.ss[KV_AX_HEAD]) * SB;
      uint8_t* trow = tile + (size_t)(j << lbp) * LD * SB;
      const uint32_t nch = Bp << lcpr;  // 8-element chunks in one source tile
      if (a.s_tr == 1) {        // (D, Bp) tile, contiguous: chunk v = (d, 8 consecutive slots)
#pragma unroll 8
        for (uint32_t v = lane; v < nch; v += 32u) {
          Chunk<SDT, VEC> x;
          load_chunk<SDT, VEC>(x, sb + (size_t)v * VEC * SB);
          const uint32_t d = v >> (lbp - 3), s0 = (v & ((Bp >> 3) - 1)) << 3;
#pragma unroll
          for (int i = 0; i < VEC; ++i) {
            const uint32_t e = get_elem<SDT>(x.w, i);
            uint8_t* dst = trow + ((size_t)(s0 + i) * LD + d) * SB;
            if constexpr (SB == 1) *dst = (uint8_t)e;
            else if constexpr (SB == 2) *reinterpret_cast<uint16_t*>(dst) = (uint16_t)e;
            else *reinterpret_cast<uint32_t*>(dst) = e;
          }
        }
      } else if (a.s_tr == 2) { // (D/x, Bp, x) tile, contiguous: chunk v = (x-group g, 8 of x)
#pragma unroll 8
        for (uint32_t v = lane; v < nch; v += 32u) {
          Chunk<SDT, VEC> x;
          load_chunk<SDT, VEC>(x, sb + (size_t)v * VEC * SB);
          const uint32_t g = v >> lsm, s = g & (Bp - 1);
          const uint32_t d0 = ((g >> lbp) << (lsm + 3)) + ((v & ((1u << lsm) - 1u)) << 3);
          store_chunk_smem<SDT, VEC>(trow + ((size_t)s * LD + d0) * SB, x);
        }
      } else {                  // rows: chunk v = (slot, 8 consecutive d)
#pragma unroll 8
        for (uint32_t v = lane; v < nch; v += 32u) {
          Chunk<SDT, VEC> x;
          const uint32_t s = v >> lcpr, d0 = (v & ((1u << lcpr) - 1u)) << 3;
          load_chunk<SDT, VEC>(x, sb + ((int64_t)s * a.ss[KV_AX_SLOT] + d0) * SB);
          store_chunk_smem<SDT, VEC>(trow + ((size_t)s * LD + d0) * SB, x);
        }
      }
    }
    __syncwarp();
    // ---- store: the destination tile, cast, tail slots zero ----
    uint8_t* db = a.dst[qi] + (dl * a.ds[KV_AX_LAYER] + (int64_t)c * a.ds[KV_AX_KV] +
                               (int64_t)__ldg(a.d_blk_ids + bl) * a.ds[KV_AX_BLOCK] + (int64_t)hq * a.ds[KV_AX_HEAD]) *
                              Tr<DDT>::B;
    const uint32_t nchd = Bd << lcpr;
    const float s2 = dual_scale(SDT, DDT) ? rsc2 : rsc;
    if (a.d_tr == 1) {          // (D, Bd) tile: chunk v = (d, 8 consecutive slots)
#pragma unroll 4
      for (uint32_t v = lane; v < nchd; v += 32u) {
        const uint32_t d = v >> (lbd - 3), s0 = (v & ((Bd >> 3) - 1)) << 3;
        Chunk<SDT, VEC> x;
        Chunk<DDT, VEC> o;
#pragma unroll
        for (int i = 0; i < Chunk<SDT, VEC>::WORDS; ++i) x.w[i] = 0;
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          const uint8_t* src = tile + ((size_t)(s0 + i) * LD + d) * SB;
          const uint32_t e = SB == 1 ? *src : SB == 2 ? *reinterpret_cast<const uint16_t*>(src)
                                                       : *reinterpret_cast<const uint32_t*>(src);
          put_elem<SDT>(x.w, i, e);
        }
        if (s0 >= valid) {
          zero_chunk(o);
        } else {
          cast_chunk<SDT, DDT, VEC>(x, o, rsc, s2);
          if (s0 + VEC > valid) zero_tail<DDT, VEC>(o, valid - s0);  // slots past T in this chunk
        }
        store_chunk<DDT, VEC>(db + (size_t)v * VEC * Tr<DDT>::B, o);
      }
    } else {
#pragma unroll 4
      for (uint32_t v = lane; v < nchd; v += 32u) {
        uint32_t s, d0;
        int64_t doff;
        if (a.d_tr == 2) {      // (D/x, Bd, x) tile: chunk v = (x-group g, 8 of x)
          const uint32_t g = v >> ldm;
          s = g & (Bd - 1);
          d0 = ((g >> lbd) << (ldm + 3)) + ((v & ((1u << ldm) - 1u)) << 3);
          doff = (int64_t)v * VEC;
        } else {                // rows: chunk v = (slot, 8 consecutive d)
          s = v >> lcpr;
          d0 = (v & ((1u << lcpr) - 1u)) << 3;
          doff = (int64_t)s * a.ds[KV_AX_SLOT] + d0;
        }
        Chunk<DDT, VEC> o;
        if (s >= valid) {
          zero_chunk(o);
        } else {
          Chunk<SDT, VEC> x;
          load_chunk_smem<SDT, VEC>(x, tile + ((size_t)s * LD + d0) * SB);
          cast_chunk<SDT, DDT, VEC>(x, o, rsc, s2);
        }
        store_chunk<DDT, VEC>(db + doff * Tr<DDT>::B, o);
      }
    }
    __syncwarp();
  }
}

// Sign / special-code restore of the fp8 -> other fp8 code tables (k_requant_rows,
// k_convert_tb): r holds the looked-up results of the four codes' magnitudes (w & 0x7F).
template <int SDT, int DDT>
__device__ __forceinline__ uint32_t requant_sign4(uint32_t w, uint32_t r) {
  const uint32_t s4 = w & 0x80808080u;
  if constexpr (DDT == KV_F8E4M3FNUZ) {
    // bit 7 of each byte: r != 0 (0x80, the NaN entry, counts as nonzero)
    const uint32_t nz = (((r & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | r) & 0x80808080u;
    return r | (s4 & nz);
  } else {
    // bit 7 of each byte: magnitude bits of the code nonzero; sign without them = fnuz NaN
    const uint32_t nzm = ((w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) & 0x80808080u;
    return (r | s4) - ((s4 & ~nzm) >> 7);   // 0x80 - 1 = 0x7F in the NaN bytes (no borrows)
  }
}

// ------------------------------------------------------------------------------------
// K1 with a head_dim-major or x-packed side, register path (k_convert_tr8): the same items
// as k_convert_tr (dst rank, dst block, layer, K/V, dst head), but no shared memory.  An
// item's (Bd x D) tile is cut into 8 x 8 sub-blocks (8 slots x 8 head_dim elements); each
// lane owns one sub-block, loads it as 8 chunks in the source's natural form (8 rows of
// one slot each, or 8 columns of one head_dim element each for a (DIM, SLOT)-innermost
// side), transposes it in registers with byte permutes when the destination's form is the
// other one, casts and stores 8 chunks.  HBM sees whole-tile reads and writes; a warp keeps
// 8 x 16 B in flight per lane.  Item metadata (block-table lookups, scales, tile bases) is
// computed lane-parallel for 32 items at a time and broadcast with shuffles, so the
// dependent table loads are paid once per 32 items, not once per item.
// ------------------------------------------------------------------------------------
// 8 x 8 transpose of chunks (8 elements each): out[i] element k = in[k] element i
template <int DT>
__device__ __forceinline__ void transpose8(const Chunk<DT, 8>* in, Chunk<DT, 8>* out) {
  if constexpr (Tr<DT>::B == 4) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) out[i].w[k] = in[k].w[i];
  } else if constexpr (Tr<DT>::B == 2) {
    // out[i].w[m] = (in[2m].e[i], in[2m+1].e[i]): the low or high halves of word i/2
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int m = 0; m < 4; ++m)
        out[i].w[m] = __byte_perm(in[2 * m].w[i >> 1], in[2 * m + 1].w[i >> 1], (i & 1) ? 0x7632u : 0x5410u);
  } else {
    // bytes: interleave row pairs (k, k+1) -> 16-bit (in[k].e[i], in[k+1].e[i]) pieces, then
    // pair those into words
    uint32_t t[4][4];  // [row pair][piece word]: word 2m+h holds elements 4m+2h, 4m+2h+1
#pragma unroll
    for (int pr = 0; pr < 4; ++pr)
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        t[pr][2 * m] = __byte_perm(in[2 * pr].w[m], in[2 * pr + 1].w[m], 0x5140u);
        t[pr][2 * m + 1] = __byte_perm(in[2 * pr].w[m], in[2 * pr + 1].w[m], 0x7362u);
      }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h)  // output word h: rows 4h .. 4h+3
        out[i].w[h] = __byte_perm(t[2 * h][i >> 1], t[2 * h + 1][i >> 1], (i & 1) ? 0x7632u : 0x5410u);
  }
}

#ifndef KVX_TR8_THREADS
#define KVX_TR8_THREADS 256
#endif
constexpr int kTr8Threads = KVX_TR8_THREADS;

template <int SDT, int DDT, bool W16>
__global__ void __launch_bounds__(kTr8Threads, W16 ? 2 : 1) k_convert_tr8(const __grid_constant__ ConvArgs a) {
  constexpr uint32_t SB = Tr<SDT>::B, DB = Tr<DDT>::B;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t lbp = (uint32_t)a.tr_lbp, lbd = (uint32_t)a.tr_lbd, lcpr = (uint32_t)a.cpr_shift;
  // W16 (2-byte head_dim-major source, B_p, B_d >= 16): a lane owns 8 head_dim rows x 16
  // slots and reads each 32-B row with one 256-bit load
  constexpr bool w16 = W16;
  const uint32_t lnsub = (lbd - (w16 ? 4u : 3u)) + lcpr;  // log2 sub-blocks per item
  const uint32_t ngroups = (a.n_items + 31u) >> 5;
  const bool s_col = a.s_tr == 1, d_col = a.d_tr == 1;
  // e4m3fnuz source to another type: the decode's 2^-7 folded into the source scale
  constexpr bool FOLD = KVX_FNUZ_FOLD && SDT == KV_F8E4M3FNUZ && DDT != KV_F8E4M3FNUZ;
  for (uint32_t grp = warp; grp < ngroups; grp += nwarps) {
    // ---- lane-parallel metadata of item grp * 32 + lane ----
    const uint32_t item = (grp << 5) + lane;
    const uint32_t cnt = min(32u, a.n_items - (grp << 5));
    const uint8_t* m_snob = nullptr;  // source tile base without the block term
    const int32_t* m_sids = nullptr;  // the request's source block ids from the dst block's first token
    int32_t m_sblk0 = 0;
    uint8_t* m_db = nullptr;          // destination tile base
    uint32_t m_valid = 0;
    float m_rsc = 1.f, m_s2 = 1.f;
    if (lane < cnt) {
      uint32_t n = item;
      const uint32_t hl = divmod(n, a.f_hde);
      const uint32_t c = take_kv(n, a.kv1, a.c0);
      const uint32_t l = divmod(n, a.f_l);
      const uint32_t bl = divmod(n, a.f_bl);
      const uint32_t qi = n;
      const uint32_t hq = (uint32_t)a.hq_off[qi] + hl;
      const int32_t r = __ldg(a.d_blk_req + bl);
      const int32_t tok0 = __ldg(a.tok_off + r);
      const int32_t T = __ldg(a.tok_off + r + 1) - tok0;
      const uint32_t tb0 = (uint32_t)(bl - __ldg(a.d_blk_off + r)) << lbd;
      const int64_t layer = a.lb + (int64_t)l;
      const int64_t sl = layer - a.s_l0, dl = layer - a.d_l0;
      const uint32_t h = (uint32_t)a.dst_rank[qi] * (uint32_t)a.Hd + hq;
      const uint32_t p = fdiv(h, a.f_hp);
      const uint32_t hp = h - p * (uint32_t)a.Hp;
      const int si = a.src_of_p[p];
      if constexpr (dual_scale(SDT, DDT)) {
        m_rsc = __ldg(a.sscale[si] + (sl * 2 + c) * a.Hp + hp);
        m_s2 = __frcp_rn(__ldg(a.dscale[qi] + (dl * 2 + c) * a.Hd + hq));
      } else {
        if constexpr (is_fp8(SDT) && SDT != DDT) m_rsc = __ldg(a.sscale[si] + (sl * 2 + c) * a.Hp + hp);
        if constexpr (is_fp8(DDT) && SDT != DDT) m_rsc = __frcp_rn(__ldg(a.dscale[qi] + (dl * 2 + c) * a.Hd + hq));
        m_s2 = m_rsc;
      }
      if constexpr (FOLD) m_rsc = fnuz_fold_scale(m_rsc);
      m_valid = (int32_t)tb0 >= T ? 0u : min(1u << lbd, (uint32_t)T - tb0);
      m_sids = a.s_blk_ids + __ldg(a.s_blk_off + r) + (int32_t)(tb0 >> lbp);
      if (m_valid) m_sblk0 = __ldg(m_sids);
      m_snob = a.src[si] + (sl * a.ss[KV_AX_LAYER] + (int64_t)c * a.ss[KV_AX_KV] + (int64_t)hp * a.ss[KV_AX_HEAD]) * SB;
      m_db = a.dst[qi] + (dl * a.ds[KV_AX_LAYER] + (int64_t)c * a.ds[KV_AX_KV] +
                          (int64_t)__ldg(a.d_blk_ids + bl) * a.ds[KV_AX_BLOCK] + (int64_t)hq * a.ds[KV_AX_HEAD]) *
                             DB;
    }
    // ---- units = (item i of the group, sub-block u); warp-uniform trip count ----
    const uint32_t nunits = cnt << lnsub;
    for (uint32_t base = 0; base < nunits; base += 32u) {
      const uint32_t unit = base + lane;
      const uint32_t i = min(unit >> lnsub, cnt - 1u);
      const uint32_t u = unit & ((1u << lnsub) - 1u);
      const uint8_t* snob = (const uint8_t*)__shfl_sync(0xFFFFFFFFu, (unsigned long long)m_snob, i);
      const int32_t* sids = (const int32_t*)__shfl_sync(0xFFFFFFFFu, (unsigned long long)m_sids, i);
      const int32_t sblk0 = __shfl_sync(0xFFFFFFFFu, m_sblk0, i);
      uint8_t* db = (uint8_t*)__shfl_sync(0xFFFFFFFFu, (unsigned long long)m_db, i);
      const uint32_t valid = __shfl_sync(0xFFFFFFFFu, m_valid, i);
      const float rsc = __shfl_sync(0xFFFFFFFFu, m_rsc, i);
      const float s2 = __shfl_sync(0xFFFFFFFFu, m_s2, i);
      if (unit >= nunits) continue;
      if constexpr (Tr<SDT>::B == 2 && W16) {
        {
          const uint32_t s0 = (u >> lcpr) << 4, d0 = (u & ((1u << lcpr) - 1u)) << 3;
          Chunk<SDT, 16> xr[8];
          const bool any = s0 < valid;
          if (any) {
            const uint32_t j = s0 >> lbp;
            const int64_t sblk = j == 0 ? sblk0 : __ldg(sids + j);
            const uint8_t* sb = snob + sblk * a.ss[KV_AX_BLOCK] * SB;
            const uint32_t sin = s0 & ((1u << lbp) - 1u);
#pragma unroll
            for (int k = 0; k < 8; ++k) load_chunk<SDT, 16>(xr[k], sb + ((int64_t)(d0 + k) * a.ss[KV_AX_DIM] + sin) * SB);
          }
          const int64_t doff = dim_off(d0, a.ds[KV_AX_DIM], a.d_dk);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const uint32_t s1 = s0 + 8u * hh;
            Chunk<DDT, 8> o[8];
            if (s1 >= valid) {
#pragma unroll
              for (int k = 0; k < 8; ++k) zero_chunk(o[k]);
            } else {
              Chunk<SDT, 8> x[8], y[8];
#pragma unroll
              for (int k = 0; k < 8; ++k)
#pragma unroll
                for (int m = 0; m < 4; ++m) x[k].w[m] = xr[k].w[4 * hh + m];
              transpose8<SDT>(x, y);
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                cast_chunk<SDT, DDT, 8, FOLD>(y[k], o[k], rsc, s2);
                if (s1 + (uint32_t)k >= valid) zero_chunk(o[k]);
              }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) store_chunk<DDT, 8>(db + ((int64_t)(s1 + k) * a.ds[KV_AX_SLOT] + doff) * DB, o[k]);
          }
          continue;
        }
      }
      const uint32_t s0 = (u >> lcpr) << 3;             // first dst slot of the sub-block
      const uint32_t d0 = (u & ((1u << lcpr) - 1u)) << 3;  // first head_dim element
      Chunk<DDT, 8> o[8];
      if (s0 >= valid) {
#pragma unroll
        for (int k = 0; k < 8; ++k) zero_chunk(o[k]);
      } else {
        const uint32_t j = s0 >> lbp;
        const int64_t sblk = j == 0 ? sblk0 : __ldg(sids + j);
        const uint8_t* sb = snob + sblk * a.ss[KV_AX_BLOCK] * SB;
        const uint32_t sin = s0 & ((1u << lbp) - 1u);
        Chunk<SDT, 8> x[8];
        if (s_col) {
#pragma unroll
          for (int k = 0; k < 8; ++k) load_chunk<SDT, 8>(x[k], sb + ((int64_t)(d0 + k) * a.ss[KV_AX_DIM] + sin) * SB);
        } else if (a.s_tr == 2) {
          // x-packed: the lane's 8 chunks are one contiguous 8-chunk run (x = 8 elements) or
          // 8 runs of x / 8 chunks, while a warp instruction touches one chunk per lane in
          // different runs: half-sector requests whose other halves the lane's next loads
          // take -- allocate in L1 so each sector comes from L2 once (0.71 -> 0.88 of copy)
          const int64_t doff = dim_off(d0, a.ss[KV_AX_DIM], a.s_dk);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            load_chunk_l1<SDT, 8>(x[k], sb + ((int64_t)(sin + k) * a.ss[KV_AX_SLOT] + doff) * SB);
        } else {
          const int64_t doff = dim_off(d0, a.ss[KV_AX_DIM], a.s_dk);
#pragma unroll
          for (int k = 0; k < 8; ++k) load_chunk<SDT, 8>(x[k], sb + ((int64_t)(sin + k) * a.ss[KV_AX_SLOT] + doff) * SB);
        }
        if (s_col != d_col) {
          Chunk<SDT, 8> y[8];
          transpose8<SDT>(x, y);
#pragma unroll
          for (int k = 0; k < 8; ++k) cast_chunk<SDT, DDT, 8, FOLD>(y[k], o[k], rsc, s2);
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) cast_chunk<SDT, DDT, 8, FOLD>(x[k], o[k], rsc, s2);
        }
        if (s0 + 8u > valid) {  // slots past the request's last token are zero
          if (d_col) {
#pragma unroll
            for (int k = 0; k < 8; ++k) zero_tail<DDT, 8>(o[k], valid - s0);
          } else {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (s0 + (uint32_t)k >= valid) zero_chunk(o[k]);
          }
        }
      }
      if (d_col) {
#pragma unroll
        for (int k = 0; k < 8; ++k) store_chunk<DDT, 8>(db + ((int64_t)(d0 + k) * a.ds[KV_AX_DIM] + s0) * DB, o[k]);
      } else {
        const int64_t doff = dim_off(d0, a.ds[KV_AX_DIM], a.d_dk);
#pragma unroll
        for (int k = 0; k < 8; ++k) store_chunk<DDT, 8>(db + ((int64_t)(s0 + k) * a.ds[KV_AX_SLOT] + doff) * DB, o[k]);
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// K2 fast path: pack (Fig. 5 flatten) with the row machinery.  Item = 32 consecutive
// tokens of one (layer, K/V, overlap head): the wire side is one contiguous 32-row run,
// each lane gathers its token's row through the block table.
// ------------------------------------------------------------------------------------
// one pack item (32 consecutive tokens of one (layer lb + l, K/V, overlap head)) of the
// chunk whose wire starts at `wire` (k_pack_rows: the launch's layer range; k_stage_rows:
// one ring chunk)
template <int SDT, int WDT, int U>
__device__ __forceinline__ void pack_item(const PackArgs& a, uint32_t item, int64_t lb, uint8_t* wire, uint32_t lane,
                                          uint32_t cs) {
  const uint32_t T_all = a.f_tok.d;
  uint32_t n = item;
  const uint32_t tg = divmod(n, a.f_tg);
  const uint32_t hh = divmod(n, a.f_nh);
  const uint32_t c = take_kv(n, a.kv1, a.c0);
  const uint32_t l = n;
  const int64_t layer = lb + (int64_t)l;
  const int64_t sl = layer - a.s_l0, dl = layer - a.d_l0;  // pool-local layers
  const uint32_t tok = tg * 32u + lane;
  uint64_t sp = 0, dp = 0;
  float rsc = 1.f, rsc2 = 1.f;
  uint32_t rz = 2;
  if (tok < T_all) {
    rz = 0;
    const int32_t r = __ldg(a.tok_req + tok);
    uint32_t t = tok - (uint32_t)__ldg(a.tok_off + r);
    const uint32_t sslot = divmod(t, a.f_bp);
    const int64_t sblk = __ldg(a.s_blk_ids + __ldg(a.s_blk_off + r) + t);
    const uint32_t h = (uint32_t)a.hb + hh;
    const uint32_t hp = h - (uint32_t)a.p * (uint32_t)a.Hp;
    sp = (uint64_t)(a.src + (sl * a.ss[KV_AX_LAYER] + (int64_t)c * a.ss[KV_AX_KV] + sblk * a.ss[KV_AX_BLOCK] +
                             (int64_t)sslot * a.ss[KV_AX_SLOT] + (int64_t)hp * a.ss[KV_AX_HEAD]) * Tr<SDT>::B);
    dp = (uint64_t)(wire + ((((uint64_t)l * wkv(a.kv1) + (c - (uint32_t)a.c0)) * (uint64_t)a.nh + hh) * T_all + tok) * (uint64_t)a.D * Tr<WDT>::B);
    const float ds_inv = is_fp8(WDT) && SDT != WDT
                             ? __frcp_rn(__ldg(a.dscale + (dl * 2 + c) * a.Hd + (h - (uint32_t)a.q * (uint32_t)a.Hd)))
                             : 1.f;
    if constexpr (is_fp8(SDT) && SDT != WDT) rsc = __ldg(a.sscale + (sl * 2 + c) * a.Hp + hp);
    if constexpr (dual_scale(SDT, WDT))
      rsc2 = ds_inv;
    else if constexpr (is_fp8(WDT) && SDT != WDT)
      rsc = ds_inv;
  }
  stream_rows<SDT, WDT, U>(lane, cs, sp, dp, rsc, rz, rsc2);
}

template <int SDT, int WDT, int U>
__global__ void __launch_bounds__(kThreads) k_pack_rows(const __grid_constant__ PackArgs a) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = (blockIdx.x * (uint32_t)kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * (uint32_t)kThreads) >> 5;
  const uint32_t cs = (uint32_t)a.cpr_shift;
  for (uint32_t item = warp; item < a.n_items; item += nwarps) pack_item<SDT, WDT, U>(a, item, a.lb, a.wire, lane, cs);
}

// ------------------------------------------------------------------------------------
// K3 fast path: unpack (Fig. 5 restore).  Item = (dst block, layer, K/V, sub-tile of
// slots x overlap heads); each lane owns one destination row and finds its wire row.
// ------------------------------------------------------------------------------------
template <int WDT, int DDT, int U>
__global__ void __launch_bounds__(kThreads) k_unpack_rows(const __grid_constant__ UnpackArgs a) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = (blockIdx.x * (uint32_t)kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * (uint32_t)kThreads) >> 5;
  const uint32_t cs = (uint32_t)a.cpr_shift;
  for (uint32_t item = warp; item < a.n_items; item += nwarps) {
    uint32_t n = item;
    uint32_t sbk = divmod(n, a.f_items);
    const uint32_t c = take_kv(n, a.kv1, a.c0);
    const uint32_t l = divmod(n, a.f_l);
    const uint32_t bl = n;
    const uint32_t s_blk = divmod(sbk, a.f_sb);
    const uint32_t ts_log2 = (uint32_t)a.ts_log2;
    const uint32_t ls = a.slot_inner ? (lane & ((1u << ts_log2) - 1u)) : (lane >> (5u - ts_log2));
    const uint32_t lh = a.slot_inner ? (lane >> ts_log2) : (lane & ((1u << (5u - ts_log2)) - 1u));
    const uint32_t slot = (s_blk << ts_log2) + ls;
    const uint32_t hh = (sbk << (5u - ts_log2)) + lh;
    const int32_t r = __ldg(a.d_blk_req + bl);
    const int32_t tok0 = __ldg(a.tok_off + r);
    const int32_t T = __ldg(a.tok_off + r + 1) - tok0;
    const int64_t layer = a.lb + (int64_t)l;
    const int64_t sl = layer - a.s_l0, dl = layer - a.d_l0;  // pool-local layers
    uint64_t sp = 0, dp = 0;
    float rsc = 1.f, rsc2 = 1.f;
    uint32_t rz = 2;
    if (slot < (uint32_t)a.Bd && hh < (uint32_t)a.nh) {
      rz = 0;
      const uint32_t t = (uint32_t)(bl - __ldg(a.d_blk_off + r)) * (uint32_t)a.Bd + slot;
      const int64_t dblk = __ldg(a.d_blk_ids + bl);
      const uint32_t h = (uint32_t)a.hb + hh;
      const uint32_t hq = h - (uint32_t)a.q * (uint32_t)a.Hd;
      dp = (uint64_t)(a.dst + (dl * a.ds[KV_AX_LAYER] + (int64_t)c * a.ds[KV_AX_KV] + dblk * a.ds[KV_AX_BLOCK] +
                               (int64_t)slot * a.ds[KV_AX_SLOT] + (int64_t)hq * a.ds[KV_AX_HEAD]) * Tr<DDT>::B);
      if ((int32_t)t >= T) {
        rz = 1;
      } else {
        sp = (uint64_t)(a.wire + ((((uint64_t)l * wkv(a.kv1) + (c - (uint32_t)a.c0)) * (uint64_t)a.nh + hh) * (uint64_t)a.total_tokens +
                                  (uint64_t)(tok0 + t)) * (uint64_t)a.D * Tr<WDT>::B);
        if constexpr (is_fp8(WDT) && WDT != DDT)
          rsc = __ldg(a.sscale + (sl * 2 + c) * a.Hp + (h - (uint32_t)a.p * (uint32_t)a.Hp));
        if constexpr (dual_scale(WDT, DDT))
          rsc2 = __frcp_rn(__ldg(a.dscale + (dl * 2 + c) * a.Hd + hq));
        else if constexpr (is_fp8(DDT) && WDT != DDT)
          rsc = __frcp_rn(__ldg(a.dscale + (dl * 2 + c) * a.Hd + hq));
      }
    }
    stream_rows<WDT, DDT, U>(lane, cs, sp, dp, rsc, rz, rsc2);
  }
}

// ------------------------------------------------------------------------------------
// K1 for head_dim-major (DIM, SLOT) source tiles through TMA (k_convert_tb).  A (block,
// head) tile of such a pool -- B x D elements -- is contiguous, so warp 0 of each CTA (the
// producer) issues ONE 2-D tensor load per tile (rows of 128 B, 128B swizzle) into a ring of
// shared-memory stages, and NC consumer warps each take a whole tile: lane (d_sub, s_sub)
// reads its 8 x 8 sub-block's eight 16-B rows from the swizzled stage (the swizzle makes the
// eight lanes of every LDS.128 phase hit distinct banks), transposes it in registers, casts
// and stores eight rows of D's (SLOT, DIM) tile.  The HBM side sees only whole 4-KB tile reads
// issued by the TMA engine (k_convert_tr8's per-lane 16-B loads left it at ~0.8 of copy).
// Metadata of 32 items at a time is computed lane-parallel by the producer (one dependent-load
// round trip per 32 tiles) and handed to the consumers through the stage's slot.  Mode 2
// takes x-packed (D/x, SLOT, x = 16 B) tiles the same way (no transpose: a 16-B chunk is x
// head_dim elements of one slot).  When both sides' head tiles are <= 2 KB an item is two
// adjacent heads (one TMA box, A.hpi = 2); an fp8 -> other fp8 item first builds its
// heads' 128-entry code tables in the consumer warp's table slot (k_requant_rows' scheme)
// and looks the codes up instead of the arithmetic cast.
// ------------------------------------------------------------------------------------
// kTbConsumers: kvx_internal.h

// Four fp8 codes through head e's 128-entry magnitude table of a 256-B table slot at tab
// (head 0 at tab, head 1 at tab + 128: the half bit rides in each code's bit 7)
template <int SDT, int DDT>
__device__ __forceinline__ uint32_t lut_word(uint32_t w, uint32_t tab, uint32_t e) {
  const uint32_t mi = (w & 0x7F7F7F7Fu) | (e ? 0x80808080u : 0u);
  uint32_t b[4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(b[j]) : "r"(__byte_perm(mi, tab, 0x7650u + (uint32_t)j)));
  return requant_sign4<SDT, DDT>(w, __byte_perm(__byte_perm(b[0], b[1], 0x0040u), __byte_perm(b[2], b[3], 0x0040u),
                                                0x5410u));
}

struct TbMeta {
  uint8_t* db;
  uint32_t valid;
  float rsc[2], s2[2];   // per head of the item (hpi <= 2)
};

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// mbar_wait with a watchdog: a pipeline bug must not hang the GPU -- after ~4 s the kernel
// traps (the launch then fails with an error instead of spinning forever).  A try_wait
// with a long suspend hint instead of the nanosleep poll measured 2-5% slower on the c4-pair
// V pools (profiles/r02/tb_variants.txt).
__device__ __forceinline__ void mbar_wait_guarded(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t it = 0;; ++it) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (it > (1u << 22)) __trap();
    __nanosleep(64);
  }
}

// 8 consecutive elements (8 or 16 bytes) from a 32-bit shared-memory address
template <int DT>
__device__ __forceinline__ void lds_chunk8(Chunk<DT, 8>& c, uint32_t saddr) {
  if constexpr (Tr<DT>::B == 2) {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(c.w[0]), "=r"(c.w[1]), "=r"(c.w[2]), "=r"(c.w[3])
                 : "r"(saddr));
  } else {
    static_assert(Tr<DT>::B == 1, "lds_chunk8: 1- or 2-byte elements");
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(c.w[0]), "=r"(c.w[1]) : "r"(saddr));
  }
}

// 16 bytes from a 32-bit shared-memory address into a 4-word chunk
template <int DT, int VEC>
__device__ __forceinline__ void lds_chunk16B(Chunk<DT, VEC>& c, uint32_t saddr) {
  static_assert(Chunk<DT, VEC>::WORDS == 4, "lds_chunk16B: 16-byte chunks");
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(c.w[0]), "=r"(c.w[1]), "=r"(c.w[2]), "=r"(c.w[3])
               : "r"(saddr));
}

// MODE 1: head_dim-major (DIM, SLOT) tiles, 8 x 8 transposes.  MODE 2: x-packed
// (D/x, SLOT, x) tiles with x = 16 B of elements: every 16-B chunk is already x consecutive
// head_dim elements of one slot, so a consumer lane takes whole chunks (no transpose).
template <int SDT, int DDT, int MODE>
__global__ void __launch_bounds__(32 * (1 + kTbConsumers)) k_convert_tb(const __grid_constant__ TbArgs A) {
  constexpr uint32_t DB = Tr<DDT>::B, SB = Tr<SDT>::B;
  static_assert(SB == 1 || SB == 2, "k_convert_tb: 1- or 2-byte sources");
  const ConvArgs& a = A.c;
  // e4m3fnuz source: the decode's 2^-7 folded into the source scale (cast_chunk)
  constexpr bool FOLD = KVX_FNUZ_FOLD && SDT == KV_F8E4M3FNUZ && DDT != KV_F8E4M3FNUZ;
  extern __shared__ __align__(1024) uint8_t tb_smem[];
  // 1024-B aligned stages (the 128B swizzle pattern repeats every 1024 B)
  uint8_t* stages = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tb_smem) + 1023) & ~uintptr_t(1023));
  const uint32_t S = (uint32_t)A.stages;
  const uint32_t tile_bytes = (uint32_t)A.tile_rows * 128u;
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + (size_t)S * tile_bytes);
  uint64_t* empty = full + S;
  TbMeta* meta = reinterpret_cast<TbMeta*>(empty + S);
  // fp8 -> other fp8: one 256-B aligned code-table slot per consumer warp after the metadata
  const uint32_t tab0 = (smem_u32(meta + S) + 255u) & ~255u;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < S; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // this CTA's items: blockIdx.x + t * gridDim.x
  const uint32_t n_mine = a.n_items > blockIdx.x ? (a.n_items - 1u - blockIdx.x) / gridDim.x + 1u : 0u;
  const uint32_t lbp = (uint32_t)a.tr_lbp, lbd = (uint32_t)a.tr_lbd;
  if (warp == 0) {
    // ---- producer ----
    for (uint32_t g = 0; g < n_mine; g += 32u) {
      const uint32_t cnt = min(32u, n_mine - g);
      uint8_t* m_db = nullptr;
      uint32_t m_valid = 0, m_row = 0, m_si = 0;
      float m_rsc[2] = {1.f, 1.f}, m_s2[2] = {1.f, 1.f};
      if (lane < cnt) {
        uint32_t n = blockIdx.x + (g + lane) * gridDim.x;
        const uint32_t hl = divmod(n, a.f_hde) * (uint32_t)A.hpi;   // first head of the item
        const uint32_t c = take_kv(n, a.kv1, a.c0);
        const uint32_t l = divmod(n, a.f_l);
        const uint32_t bl = divmod(n, a.f_bl);
        const uint32_t qi = n;
        const uint32_t hq = (uint32_t)a.hq_off[qi] + hl;
        const int32_t r = __ldg(a.d_blk_req + bl);
        const int32_t tok0 = __ldg(a.tok_off + r);
        const int32_t T = __ldg(a.tok_off + r + 1) - tok0;
        const uint32_t tb0 = (uint32_t)(bl - __ldg(a.d_blk_off + r)) << lbd;
        const int64_t layer = a.lb + (int64_t)l;
        const int64_t sl = layer - a.s_l0, dl = layer - a.d_l0;
        const uint32_t h = (uint32_t)a.dst_rank[qi] * (uint32_t)a.Hd + hq;
        const uint32_t p = fdiv(h, a.f_hp);
        const uint32_t hp = h - p * (uint32_t)a.Hp;
        const int si = a.src_of_p[p];
#pragma unroll
        for (uint32_t e = 0; e < 2; ++e) {   // the item's heads hq + e / hp + e (same P rank: host check)
          if (e >= (uint32_t)A.hpi) break;
          float rs = 1.f, s2v = 1.f;
          if constexpr (dual_scale(SDT, DDT)) {
            rs = __ldg(a.sscale[si] + (sl * 2 + c) * a.Hp + hp + e);
            s2v = __frcp_rn(__ldg(a.dscale[qi] + (dl * 2 + c) * a.Hd + hq + e));
          } else {
            if constexpr (is_fp8(SDT) && SDT != DDT) rs = __ldg(a.sscale[si] + (sl * 2 + c) * a.Hp + hp + e);
            if constexpr (is_fp8(DDT) && SDT != DDT) rs = __frcp_rn(__ldg(a.dscale[qi] + (dl * 2 + c) * a.Hd + hq + e));
            s2v = rs;
          }
          if constexpr (FOLD) rs = fnuz_fold_scale(rs);
          m_rsc[e] = rs;
          m_s2[e] = s2v;
        }
        m_valid = (int32_t)tb0 >= T ? 0u : min(1u << lbd, (uint32_t)T - tb0);
        const int64_t sblk = __ldg(a.s_blk_ids + __ldg(a.s_blk_off + r) + (int32_t)(tb0 >> lbp));
        const int64_t off = sl * a.ss[KV_AX_LAYER] + (int64_t)c * a.ss[KV_AX_KV] + sblk * a.ss[KV_AX_BLOCK] +
                            (int64_t)hp * a.ss[KV_AX_HEAD];  // elements; the tile starts here
        m_row = (uint32_t)((off * (int64_t)SB) >> 7);
        m_si = (uint32_t)si;
        m_db = a.dst[qi] + (dl * a.ds[KV_AX_LAYER] + (int64_t)c * a.ds[KV_AX_KV] +
                            (int64_t)__ldg(a.d_blk_ids + bl) * a.ds[KV_AX_BLOCK] + (int64_t)hq * a.ds[KV_AX_HEAD]) *
                               DB;
      }
      for (uint32_t j = 0; j < cnt; ++j) {
        const uint64_t db = __shfl_sync(0xFFFFFFFFu, (unsigned long long)m_db, j);
        const uint32_t valid = __shfl_sync(0xFFFFFFFFu, m_valid, j);
        const uint32_t row = __shfl_sync(0xFFFFFFFFu, m_row, j);
        const uint32_t si = __shfl_sync(0xFFFFFFFFu, m_si, j);
        const float rsc0 = __shfl_sync(0xFFFFFFFFu, m_rsc[0], j), rsc1 = __shfl_sync(0xFFFFFFFFu, m_rsc[1], j);
        const float s20 = __shfl_sync(0xFFFFFFFFu, m_s2[0], j), s21 = __shfl_sync(0xFFFFFFFFu, m_s2[1], j);
        if (lane == 0) {
          const uint32_t t = g + j, st = t % S;
          mbar_wait_guarded(empty + st, ((t / S) & 1u) ^ 1u);
          meta[st] = TbMeta{reinterpret_cast<uint8_t*>(db), valid, {rsc0, rsc1}, {s20, s21}};
          mbar_expect_tx_arrive(full + st, tile_bytes);
          tma_load_2d(stages + (size_t)st * tile_bytes, &A.maps[si], 0, (int32_t)row, full + st);
        }
        __syncwarp();
      }
    }
    return;
  }
  // ---- consumers ----
  const uint32_t cw = warp - 1u;
  const uint32_t lcpr = (uint32_t)a.cpr_shift;           // log2(D / 8)
  const uint32_t nsub = 2u << lcpr;                       // (B = 16) / 8 x D / 8 sub-blocks
  const uint32_t row_bytes = 16u * SB;                    // one head_dim element's 16 slots
  const uint32_t stage0 = smem_u32(stages);
  for (uint32_t t = cw; t < n_mine; t += kTbConsumers) {
    const uint32_t st = t % S;
    mbar_wait_guarded(full + st, (t / S) & 1u);
    const TbMeta m = meta[st];
    const uint32_t tile = stage0 + st * tile_bytes;
    // fp8 -> other fp8: this item's 128-entry magnitude code table (k_requant_rows' scheme),
    // built by the warp from the exact arithmetic cast -- 4 codes per lane, one cast_chunk --
    // then one byte permute + one LDS.U8 per code instead of the arithmetic cast
    constexpr bool LUT_OK = dual_scale(SDT, DDT);
    const bool LUT = LUT_OK && A.lut;
    const uint32_t tab = tab0 + cw * 256u;   // head e's table at tab + 128 e
    const uint32_t hpi = (uint32_t)A.hpi, head_bytes = tile_bytes / hpi;
    if (LUT) {
      for (uint32_t e = 0; e < hpi; ++e) {
        Chunk<SDT, 4> ci;
        Chunk<DDT, 4> co;
        ci.w[0] = 0x03020100u + lane * 0x04040404u;   // codes 4 lane .. 4 lane + 3
        cast_chunk<SDT, DDT, 4, FOLD>(ci, co, m.rsc[e], m.s2[e]);
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(tab + e * 128u + lane * 4u), "r"(co.w[0]) : "memory");
      }
      __syncwarp();
    }
    if constexpr (MODE == 2) {
      // x-packed tiles: 16-B chunks (dq, slot) hold X consecutive head_dim elements of one
      // slot -- no transpose; head e of the item at tile + e x head_bytes
      constexpr uint32_t X = 16u / SB;                  // elements per 16-B chunk
      const uint32_t lndq = lcpr + 3u - (SB == 1 ? 4u : 3u);   // log2(D / X)
      const uint32_t ndq = 1u << lndq;
      for (uint32_t idx = lane; idx < ((ndq << 4) * hpi); idx += 32u) {
        const uint32_t e = idx >> (lndq + 4u), ii = idx & ((ndq << 4) - 1u);
        const uint32_t dq = ii & (ndq - 1u), sl = ii >> lndq;   // lanes: consecutive chunks of one row
        const uint32_t off = ((dq << 4) + sl) << 4;                // chunk (dq, slot) of the head's tile
        const uint32_t R = off >> 7, c = (off >> 4) & 7u;
        uint8_t* const hdb = m.db + (int64_t)e * a.ds[KV_AX_HEAD] * DB;
        Chunk<DDT, X> o;
        if (sl >= m.valid) {
          zero_chunk(o);
        } else {
          Chunk<SDT, X> x;
          lds_chunk16B<SDT, X>(x, tile + e * head_bytes + R * 128u + ((c ^ (R & 7u)) << 4));
          if constexpr (LUT_OK && X == 16) {
            if (LUT) {
#pragma unroll
              for (int q = 0; q < 4; ++q) o.w[q] = lut_word<SDT, DDT>(x.w[q], tab, e);
            } else {
              cast_chunk<SDT, DDT, X, FOLD>(x, o, e ? m.rsc[1] : m.rsc[0], e ? m.s2[1] : m.s2[0]);
            }
          } else {
            cast_chunk<SDT, DDT, X, FOLD>(x, o, e ? m.rsc[1] : m.rsc[0], e ? m.s2[1] : m.s2[0]);
          }
        }
        store_chunk<DDT, X>(hdb + ((int64_t)sl * a.ds[KV_AX_SLOT] + dim_off(dq * X, a.ds[KV_AX_DIM], a.d_dk)) * DB, o);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
      continue;
    }
    // units (head e of the item, 8 x 8 sub-block): head e's tile follows head e-1's in the
    // stage (adjacent source heads, one TMA box; a head's rows are a multiple of 8, so the
    // 128B swizzle phase restarts with each head)
    for (uint32_t u = lane; u < (nsub * hpi); u += 32u) {
      const uint32_t e = u >> (lcpr + 1u), uu = u & (nsub - 1u);
      const uint32_t s_sub = uu & 1u, d_sub = uu >> 1;
      const uint32_t s0 = s_sub << 3, d0 = d_sub << 3;
      const uint32_t htile = tile + e * head_bytes;
      uint8_t* const hdb = m.db + (int64_t)e * a.ds[KV_AX_HEAD] * DB;
      const float rsc = e ? m.rsc[1] : m.rsc[0], s2 = e ? m.s2[1] : m.s2[0];
      Chunk<DDT, 8> o[8];
      if (s0 >= m.valid) {
#pragma unroll
        for (int k = 0; k < 8; ++k) zero_chunk(o[k]);
      } else {
        Chunk<SDT, 8> x[8], y[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          // logical byte offset of (head_dim d0 + k, slots s0..s0+7) in the tile, then the
          // TMA 128B swizzle: 16-B unit c of 128-B row R sits at unit c ^ (R mod 8)
          const uint32_t off = (d0 + (uint32_t)k) * row_bytes + s0 * SB;
          const uint32_t R = off >> 7, c = (off >> 4) & 7u;
          lds_chunk8<SDT>(x[k], htile + R * 128u + ((c ^ (R & 7u)) << 4) + (off & 15u));
        }
        if (LUT) {
          // look the codes up (element-wise, so before the byte transpose), then transpose
          Chunk<DDT, 8> xo[8];
#pragma unroll
          for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int q = 0; q < 2; ++q) xo[k].w[q] = lut_word<SDT, DDT>(x[k].w[q], tab, e);
          transpose8<DDT>(xo, o);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (s0 + (uint32_t)k >= m.valid) zero_chunk(o[k]);
        } else {
          transpose8<SDT>(x, y);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            cast_chunk<SDT, DDT, 8, FOLD>(y[k], o[k], rsc, s2);
            if (s0 + (uint32_t)k >= m.valid) zero_chunk(o[k]);
          }
        }
      }
      const int64_t doff = dim_off(d0, a.ds[KV_AX_DIM], a.d_dk);
#pragma unroll
      for (int k = 0; k < 8; ++k) store_chunk<DDT, 8>(hdb + ((int64_t)(s0 + k) * a.ds[KV_AX_SLOT] + doff) * DB, o[k]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);
  }
}

// ------------------------------------------------------------------------------------
// K1 fast path with a cast, TMA-fed (k_tile_cast): the sub-tiles of k_tile_copy -- one 5-D
// tensor load each, landing in shared memory already in D's inner order -- feed consumer
// warps that convert them row by row (16-B LDS, the cast, 8- or 16-B stores of D's rows)
// instead of bulk-storing them unchanged.  Warp 0 is the producer (decode + TMA issue into a
// ring of stages with full / empty mbarriers); kTbConsumers warps consume.  Rows of slots
// >= T are written as zeros; a partial sub-tile's valid rows come by plain loads
// (tile_rows_ldg), so no source tail slot is read.  The HBM side sees one TMA read per sub-tile (8 KB for a c4
// pair: 2 heads x 16 slots x 128 bf16).
// ------------------------------------------------------------------------------------
struct TcMeta {
  uint8_t* dtile;    // D (layer, K/V, block) tile base (bytes)
  int32_t hq0, soff; // first D-local head, first slot of the sub-tile in the D block
  uint32_t valid;    // source slots < T (0: the whole sub-tile is tail)
  float rsc[8], rsc2[8];  // per head: the cast's scales (see conv_row)
};

template <int SDT, int DDT>
__global__ void __launch_bounds__(32 * (1 + kTbConsumers)) k_tile_cast(const __grid_constant__ TileArgs a) {
  constexpr uint32_t SB = Tr<SDT>::B, DB = Tr<DDT>::B;
  constexpr bool FOLD = KVX_FNUZ_FOLD && SDT == KV_F8E4M3FNUZ && DDT != KV_F8E4M3FNUZ;
  extern __shared__ __align__(128) uint8_t tc_smem[];
  const uint32_t S = (uint32_t)a.stages, SBY = (uint32_t)a.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(tc_smem + (size_t)S * SBY);
  uint64_t* empty = full + S;
  TcMeta* meta = reinterpret_cast<TcMeta*>(empty + S);
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < S; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t n_mine = a.n_items > blockIdx.x ? (a.n_items - 1u - blockIdx.x) / gridDim.x + 1u : 0u;
  const uint32_t nh = (uint32_t)a.nh, Bp = (uint32_t)a.Bp;
  if (warp == 0) {
    // ---- producer: metadata of 32 items at a time, lane-parallel (one round trip of
    // dependent table loads per 32 sub-tiles), then one TMA issue per item by lane 0 ----
    for (uint32_t g = 0; g < n_mine; g += 32u) {
      const uint32_t cnt = min(32u, n_mine - g);
      uint64_t m_dtile = 0;
      int32_t m_hq0 = 0, m_soff = 0, m_si = 0, m_c = 0, m_h1 = 0, m_h2 = 0, m_sblk = 0, m_sl = 0;
      uint32_t m_valid = 0;
      float m_rsc[8], m_rsc2[8];
#pragma unroll
      for (int h = 0; h < 8; ++h) m_rsc[h] = m_rsc2[h] = 1.f;
      if (lane < cnt) {
        uint32_t n = blockIdx.x + (g + lane) * gridDim.x;
        const uint32_t qi = divmod(n, a.f_nd);
        const uint32_t part = divmod(n, a.f_parts);
        const uint32_t sub = divmod(n, a.f_sub);
        const uint32_t c = take_kv(n, a.kv1, a.c0);
        const uint32_t l = divmod(n, a.f_l);
        const uint32_t bl = n;
        const int32_t r = __ldg(a.d_blk_req + bl);
        const int32_t tok0 = __ldg(a.tok_off + r);
        const int32_t T = __ldg(a.tok_off + r + 1) - tok0;
        const int32_t j = bl - __ldg(a.d_blk_off + r);
        const int64_t dblk = __ldg(a.d_blk_ids + bl);
        const int32_t layer = a.lb + (int32_t)l;
        const int32_t q = a.dst_rank[qi];
        const int32_t hstart = a.share_p >= 0 ? max(a.share_p * a.Hp, q * a.Hd) : q * a.Hd;
        const int32_t h0 = hstart + (int32_t)part * a.nh;
        const int32_t p = a.share_p >= 0 ? a.share_p : h0 / a.Hp;
        const int32_t hp0 = h0 - p * a.Hp, hq0 = h0 - q * a.Hd;
        const int si = a.src_of_p[p];
        const int32_t t0 = j * a.Bd + (int32_t)sub * a.Bp;
        m_valid = t0 >= T ? 0u : (uint32_t)min(a.Bp, T - t0);
        if (m_valid) m_sblk = __ldg(a.s_blk_ids + __ldg(a.s_blk_off + r) + (j * (a.Bd / a.Bp) + (int32_t)sub));
        const int64_t sl = layer - a.s_l0, dl = layer - a.d_l0;
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          if ((uint32_t)h >= nh) break;
          const int32_t hq = hq0 + h, hp = hp0 + h;
          float rsc = 1.f, rsc2 = 1.f;
          if constexpr (dual_scale(SDT, DDT)) {
            rsc = __ldg(a.sscale[si] + (sl * 2 + c) * a.Hp + hp);
            rsc2 = __frcp_rn(__ldg(a.dscale[qi] + (dl * 2 + c) * a.Hd + hq));
          } else {
            if constexpr (is_fp8(SDT) && SDT != DDT) rsc = __ldg(a.sscale[si] + (sl * 2 + c) * a.Hp + hp);
            if constexpr (is_fp8(DDT) && SDT != DDT) rsc = __frcp_rn(__ldg(a.dscale[qi] + (dl * 2 + c) * a.Hd + hq));
            rsc2 = rsc;   // one-scale casts read the destination's inverse from the second slot too
          }
          if constexpr (FOLD) rsc = fnuz_fold_scale(rsc);
          m_rsc[h] = rsc;
          m_rsc2[h] = rsc2;
        }
        m_dtile = (uint64_t)(a.dst[qi] +
                             (dl * a.ds[KV_AX_LAYER] + (int64_t)c * a.ds[KV_AX_KV] + dblk * a.ds[KV_AX_BLOCK]) * DB);
        m_hq0 = hq0;
        m_soff = (int32_t)sub * a.Bp;
        m_si = si;
        m_c = (int32_t)c;
        m_h1 = a.head_major ? 0 : hp0;
        m_h2 = a.head_major ? hp0 : 0;
        m_sl = (int32_t)sl;
      }
      for (uint32_t j = 0; j < cnt; ++j) {
        const uint64_t dtile = __shfl_sync(0xFFFFFFFFu, (unsigned long long)m_dtile, j);
        const int32_t hq0 = __shfl_sync(0xFFFFFFFFu, m_hq0, j), soff = __shfl_sync(0xFFFFFFFFu, m_soff, j);
        const uint32_t valid = __shfl_sync(0xFFFFFFFFu, m_valid, j);
        const int32_t si = __shfl_sync(0xFFFFFFFFu, m_si, j), c = __shfl_sync(0xFFFFFFFFu, m_c, j);
        const int32_t h1 = __shfl_sync(0xFFFFFFFFu, m_h1, j), h2 = __shfl_sync(0xFFFFFFFFu, m_h2, j);
        const int32_t sblk = __shfl_sync(0xFFFFFFFFu, m_sblk, j), sl = __shfl_sync(0xFFFFFFFFu, m_sl, j);
        // lane h < nh takes head h's scales of item j
        float rsc = 1.f, rsc2 = 1.f;
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const float v = __shfl_sync(0xFFFFFFFFu, m_rsc[h], j), v2 = __shfl_sync(0xFFFFFFFFu, m_rsc2[h], j);
          if ((uint32_t)h == lane) {
            rsc = v;
            rsc2 = v2;
          }
        }
        const uint32_t t = g + j, st = t % S;
        if (lane == 0) mbar_wait_guarded(empty + st, ((t / S) & 1u) ^ 1u);
        __syncwarp();
        if (lane < nh) {
          meta[st].rsc[lane] = rsc;
          meta[st].rsc2[lane] = rsc2;
        }
        if (lane == 0) {
          meta[st].dtile = reinterpret_cast<uint8_t*>(dtile);
          meta[st].hq0 = hq0;
          meta[st].soff = soff;
          meta[st].valid = valid;
        }
        __syncwarp();
        if (valid > 0u && valid < Bp)  // partial sub-tile: valid rows only (tile_rows_ldg)
          tile_rows_ldg(a, tc_smem + (size_t)st * SBY, si, c, sblk, sl, a.head_major ? h2 : h1, valid, lane);
        if (lane == 0) {
          mbar_expect_tx_arrive(full + st, valid == Bp ? SBY : 0u);
          if (valid == Bp) tma_load_5d(tc_smem + (size_t)st * SBY, &a.maps[si][c], 0, h1, h2, sblk, sl, full + st);
        }
      }
    }
    return;
  }
  // ---- consumers: rows of the staged sub-tile, D's inner order ----
  const uint32_t cw = warp - 1u;
  const uint32_t cpr = (uint32_t)a.D / 8u;  // 8-element chunks per row (D / 8 a power of two)
  uint32_t lcpr = 0;
  while ((1u << lcpr) < cpr) ++lcpr;
  const uint32_t nchunks = nh * Bp * cpr;
  const uint32_t row_bytes = (uint32_t)a.D * SB;
  const uint32_t stage0 = smem_u32(tc_smem);
  uint32_t lbp = 0, lnh = 0;   // Bp, nh: powers of two (host check) -- shifts, not divisions
  while ((1u << lbp) < Bp) ++lbp;
  while ((1u << lnh) < nh) ++lnh;
  for (uint32_t t = cw; t < n_mine; t += kTbConsumers) {
    const uint32_t st = t % S;
    mbar_wait_guarded(full + st, (t / S) & 1u);
    const TcMeta& m = meta[st];
    uint8_t* const dtile = m.dtile;
    const int32_t hq0 = m.hq0, soff = m.soff;
    const uint32_t valid = m.valid;
    const uint32_t buf = stage0 + st * SBY;
    for (uint32_t idx = lane; idx < nchunks; idx += 32u) {
      const uint32_t ri = idx >> lcpr, ch = idx & (cpr - 1u);
      const uint32_t h = a.head_major ? ri >> lbp : ri & (nh - 1u);
      const uint32_t sl_ = a.head_major ? ri & (Bp - 1u) : ri >> lnh;
      Chunk<DDT, 8> o;
      if (sl_ >= valid) {
        zero_chunk(o);
      } else {
        Chunk<SDT, 8> x;
        lds_chunk8<SDT>(x, buf + ri * row_bytes + ch * 8u * SB);
        cast_chunk<SDT, DDT, 8, FOLD>(x, o, m.rsc[h], m.rsc2[h]);
      }
      store_chunk<DDT, 8>(dtile + ((int64_t)(hq0 + (int32_t)h) * a.ds[KV_AX_HEAD] +
                                   (int64_t)(soff + (int32_t)sl_) * a.ds[KV_AX_SLOT] + (int64_t)ch * 8) * DB, o);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);
  }
}

// ------------------------------------------------------------------------------------
// fp8 -> other fp8 requantisation through code tables (k_requant_rows; e4m3fnuz <-> e4m3fn
// with static scales, readings 24-26).  With both scales fixed per (layer, K/V, head) the
// cast is a pure function of the 8-bit code.  Both formats are sign-magnitude and every step
// of the cast (decode, the two round-to-nearest multiplies, the satfinite encode) is odd, so
// the table holds only the 128 MAGNITUDE codes -- each entry by the exact per-code path
// (cast_chunk), bit-identical to the arithmetic kernels -- and the sign is put back per byte
// with the two formats' special codes fixed up in SIMD-within-a-register:
//   e4m3fn -> fnuz: NaN (0x7F | s) -> 0x80 (entry 0x7F already is 0x80); a zero result is
//                   +0 whatever the sign (fnuz has no -0: 0x80 is its NaN);
//   fnuz -> e4m3fn: 0x80 (NaN) -> 0x7F; everything else magnitude | sign.
// A 128-B table spans the 32 shared-memory banks exactly once, so a warp's 32 lookups into
// ONE table never conflict; the item's rows are laid out slot-fastest over the lanes
// (vlane) so the rows of one warp instruction (32 / 16-B chunks per row of them) share
// their head, hence their table.  Per code: one byte permute (code into the table address),
// one LDS.U8; per 4 codes: 3 permutes to reassemble and 4-6 integer ops of fix-up,
// branch-free (a fix-up only in chunks holding a fnuz NaN measured slower: 0.852 vs 0.870).
// ------------------------------------------------------------------------------------
template <int SDT, int DDT, int U, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_requant_rows(const __grid_constant__ ConvArgs a) {
  static_assert(dual_scale(SDT, DDT), "k_requant_rows: fp8 -> other fp8");
  extern __shared__ __align__(256) uint8_t lut_raw[];
  // table t at byte t * 128 of a 256-B aligned region: table pair base | (t & 1) << 7 | code
  uint8_t* lut = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(lut_raw) + 255) & ~uintptr_t(255));
  const uint32_t kv = a.kv1 ? 1u : 2u;
  // this CTA's items: a contiguous range of the layer-outermost order m (item n of conv_row
  // = the same (dst block, layer, K/V, sub-tile, dst rank) with the block outermost), so it
  // needs the tables of a few layers only, not of the launch's Lc
  const uint32_t inner = kv * a.f_items.d * a.f_nd.d;       // items per (layer, dst block)
  const uint32_t nbl = a.f_bl.d, per_layer = nbl * inner;
  const uint32_t m0 = blockIdx.x * a.rq_per_cta;
  const uint32_t m1 = min(a.n_items, m0 + a.rq_per_cta);
  if (m0 >= m1) return;
  const uint32_t l_lo = m0 / per_layer, l_hi = (m1 - 1u) / per_layer;
  const uint32_t tpl = a.f_nd.d * kv * (uint32_t)a.Hd_eff;  // tables per layer
  const uint32_t n_tab = (l_hi - l_lo + 1u) * tpl;
  // ---- tables: entry (t, magnitude code m), t = ((l - l_lo) * nd + qi) * kv + c) * Hd_eff + hl ----
  for (uint32_t e = threadIdx.x; e < n_tab * 128u; e += blockDim.x) {
    const uint32_t code = e & 127u;
    uint32_t t = e >> 7;
    const uint32_t hl = t % (uint32_t)a.Hd_eff;
    t /= (uint32_t)a.Hd_eff;
    const uint32_t c = a.kv1 ? (uint32_t)a.c0 : (t % 2u);
    if (!a.kv1) t /= 2u;
    const uint32_t qi = t % a.f_nd.d, l = l_lo + t / a.f_nd.d;
    const uint32_t hq = (uint32_t)a.hq_off[qi] + hl;
    const int64_t layer = a.lb + (int64_t)l;
    const int64_t sl = layer - a.s_l0, dl = layer - a.d_l0;
    const uint32_t h = (uint32_t)a.dst_rank[qi] * (uint32_t)a.Hd + hq;
    const uint32_t p = fdiv(h, a.f_hp);
    const uint32_t hp = h - p * (uint32_t)a.Hp;
    const int si = a.src_of_p[p];
    const float ssc = __ldg(a.sscale[si] + (sl * 2 + c) * a.Hp + hp);
    const float inv = __frcp_rn(__ldg(a.dscale[qi] + (dl * 2 + c) * a.Hd + hq));
    Chunk<SDT, 4> in;
    Chunk<DDT, 4> out;
    in.w[0] = code;
    cast_chunk<SDT, DDT, 4>(in, out, ssc, inv);
    lut[e] = (uint8_t)(out.w[0] & 0xFFu);
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t cs = (uint32_t)a.cpr_shift;  // log2(16-byte chunks per row)
  const uint32_t cmask = (1u << cs) - 1u, nch = 32u << cs;
  const uint32_t lut0 = smem_u32(lut), tbl0 = l_lo * tpl;
  // slot-fastest rows over the lanes whatever D's inner order (conv_row's row index)
  const uint32_t tsl = (uint32_t)a.ts_log2;
  const uint32_t vlane = a.slot_inner ? lane : (((lane & ((1u << tsl) - 1u)) << (5u - tsl)) | (lane >> tsl));
  for (uint32_t m = m0 + (threadIdx.x >> 5); m < m1; m += kThreads / 32u) {
    const uint32_t r0 = m % inner, q = m / inner;
    const uint32_t l = q / nbl, bl = q - l * nbl;
    const uint32_t item = (bl * (uint32_t)a.Lc + l) * inner + r0;
    uint64_t sp, dp;
    float rsc, rsc2;
    uint32_t rz, tbl = 0;
    conv_row<SDT, DDT>(a, item, vlane, sp, dp, rsc, rz, rsc2, nullptr, &tbl);
    const uint32_t tbase = lut0 + ((tbl - tbl0) << 7);   // byte 0: the table half bit (pairs 256-B aligned)
    for (uint32_t base = 0; base < nch; base += 32u * U) {
      uint4 in[U];
      uint64_t d[U];
      uint32_t z[U], tb[U], ch[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const uint32_t idx = base + (uint32_t)k * 32u + lane;
        const uint32_t rr = (idx >> cs) & 31u;
        ch[k] = idx & cmask;
        const uint64_t s = __shfl_sync(0xffffffffu, sp, rr);
        d[k] = __shfl_sync(0xffffffffu, dp, rr);
        z[k] = __shfl_sync(0xffffffffu, rz, rr) | (idx >= nch ? 2u : 0u);
        tb[k] = __shfl_sync(0xffffffffu, tbase, rr);
        if (z[k] == 0) in[k] = __ldg(reinterpret_cast<const uint4*>(s + ch[k] * 16u));
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        if (z[k] & 2u) continue;
        uint4 o = make_uint4(0, 0, 0, 0);
        if (z[k] == 0) {
          uint32_t w[4] = {in[k].x, in[k].y, in[k].z, in[k].w}, r[4];
          const uint32_t half4 = __byte_perm(tb[k], 0u, 0x0000u);  // the half bit in every byte
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t mi = (w[q] & 0x7F7F7F7Fu) | half4;   // magnitude codes | table half
            uint32_t b[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t addr = __byte_perm(mi, tb[k], 0x7650u + (uint32_t)j);  // code j | half into byte 0
              asm volatile("ld.shared.u8 %0, [%1];" : "=r"(b[j]) : "r"(addr));
            }
            const uint32_t m4 = __byte_perm(__byte_perm(b[0], b[1], 0x0040u), __byte_perm(b[2], b[3], 0x0040u), 0x5410u);
            r[q] = requant_sign4<SDT, DDT>(w[q], m4);
          }
          o = make_uint4(r[0], r[1], r[2], r[3]);
        }
        *reinterpret_cast<uint4*>(d[k] + ch[k] * 16u) = o;
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// K3 persistent staged pull (kv_pull_staged, D side): the unpack row machinery over every
// layer chunk of the call in ONE launch.  Warps take kPullGrab items at a time from a
// per-chunk counter (chunk after chunk), so all warps leave a chunk within one grab of each
// other.  Before its first item of chunk k a warp waits (lane 0, acquire, system scope)
// for every source's ready word >= seq0 + k + 1; the warp whose items complete chunk k
// releases the ring slot back to the P ranks (system-scope release stores into their
// memory).  One ramp-up and one tail per call instead of one per chunk; loads come over
// NVLink from the P ranks' ring slots (weak loads, ordered after the acquire).
// ------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr uint32_t kPullGrab = 4;  // items (32 rows each) per hand-out

__device__ __forceinline__ void spin_until(const uint32_t* flag, uint32_t value, uint64_t timeout_ns, int32_t* err,
                                           uint32_t spin_ns) {
  const uint64_t t0 = globaltimer_ns();
  while (true) {
    uint32_t x;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(x) : "l"(flag) : "memory");
    if ((int32_t)(x - value) >= 0) return;
    if (globaltimer_ns() - t0 > timeout_ns) {
      *err = 1;
      return;
    }
    __nanosleep(spin_ns);
  }
}

template <int DT, int U>
__global__ void __launch_bounds__(kThreads) k_pull_rows(const __grid_constant__ PullArgs a) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t cs = (uint32_t)a.cpr_shift;
  const uint32_t ts_log2 = (uint32_t)a.ts_log2;
  const uint32_t ls = a.slot_inner ? (lane & ((1u << ts_log2) - 1u)) : (lane >> (5u - ts_log2));
  const uint32_t lh = a.slot_inner ? (lane >> ts_log2) : (lane & ((1u << (5u - ts_log2)) - 1u));
  uint32_t* next = a.counters;               // [nchunks] items handed out
  uint32_t* done = a.counters + a.nchunks;   // [nchunks] items finished
  for (int32_t k = 0; k < a.nchunks; ++k) {
    // chunk k of the ChunkPlan: a ramp chunk, or a step-layer chunk (the last one partial)
    const bool ramp = k < a.nramp, last = k == a.nchunks - 1;
    const uint32_t n_k = ramp ? a.ramp_items[k] : last ? a.items_last : a.items_full;
    const FastDiv& f_l = ramp ? a.f_l_ramp[k] : last ? a.f_l_last : a.f_l_full;
    const uint32_t slot_idx = (a.seq0 + (uint32_t)k) % (uint32_t)a.R;
    const int64_t l0 = ramp ? (int64_t)a.ramp_l0[k] : (int64_t)a.lb + a.rsum + (int64_t)(k - a.nramp) * a.step;
    bool waited = false;
    while (true) {
      // dynamic hand-out: every warp leaves chunk k within one grab of the others, so the
      // ring slots come back in order and no warp runs R chunks ahead of the slowest
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(next + k, kPullGrab);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base >= n_k) break;
      if (!waited) {
        if (lane == 0)
          for (int s = 0; s < a.nsrc; ++s) spin_until(a.ready[s], a.seq0 + (uint32_t)k + 1u, a.timeout_ns, a.err, a.spin_ns);
        __syncwarp();
        waited = true;
      }
      const uint32_t end = min(n_k, base + kPullGrab);
      for (uint32_t item = base; item < end; ++item) {
        uint32_t n = item;
        const uint32_t src = divmod(n, a.f_src);
        uint32_t sbk = divmod(n, a.f_items);
        const uint32_t c = take_kv(n, a.kv1, a.c0);
        const uint32_t lk = divmod(n, f_l);
        const uint32_t bl = n;
        const uint32_t s_blk = divmod(sbk, a.f_sb);
        const uint32_t slot = (s_blk << ts_log2) + ls;
        const uint32_t hh = (sbk << (5u - ts_log2)) + lh;
        const int32_t r = __ldg(a.d_blk_req + bl);
        const int32_t tok0 = __ldg(a.tok_off + r);
        const int32_t T = __ldg(a.tok_off + r + 1) - tok0;
        const int64_t dl = l0 + (int64_t)lk - a.d_l0;
        uint64_t sp = 0, dp = 0;
        uint32_t rz = 2;
        if (slot < (uint32_t)a.Bd && hh < (uint32_t)a.nh) {
          rz = 0;
          const uint32_t t = (uint32_t)(bl - __ldg(a.d_blk_off + r)) * (uint32_t)a.Bd + slot;
          const int64_t dblk = __ldg(a.d_blk_ids + bl);
          const uint32_t hq = (uint32_t)a.hb[src] + hh - (uint32_t)a.q * (uint32_t)a.Hd;
          dp = (uint64_t)(a.dst + (dl * a.ds[KV_AX_LAYER] + (int64_t)c * a.ds[KV_AX_KV] + dblk * a.ds[KV_AX_BLOCK] +
                                   (int64_t)slot * a.ds[KV_AX_SLOT] + (int64_t)hq * a.ds[KV_AX_HEAD]) * Tr<DT>::B);
          if ((int32_t)t >= T)
            rz = 1;
          else
            sp = (uint64_t)(a.ring[src][slot_idx] +
                            ((((uint64_t)lk * wkv(a.kv1) + (c - (uint32_t)a.c0)) * (uint64_t)a.nh + hh) * (uint64_t)a.total_tokens +
                             (uint64_t)(tok0 + t)) * (uint64_t)a.D * Tr<DT>::B);
        }
        stream_rows<DT, DT, U, 8, true>(lane, cs, sp, dp, 1.f, rz);
      }
      // the warp that completes chunk k releases its ring slot to every source -- strictly
      // in chunk order: P reads free >= v as "every chunk below v has been read", so chunk k
      // is released only after chunk k-1 (watermark == k).  The chunk k-1 items still in
      // flight belong to warps that grabbed them, i.e. are resident and need nothing more.
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        const uint32_t cnt = end - base;
        if (atomicAdd(done + k, cnt) + cnt == n_k) {
          uint32_t wm;
          while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(wm) : "l"(a.watermark) : "memory");
            if (wm == (uint32_t)k) break;
            __nanosleep(64);
          }
          __threadfence_system();
          for (int s = 0; s < a.nsrc; ++s)
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.freef[s]), "r"(a.seq0 + (uint32_t)k + 1u)
                         : "memory");
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.watermark), "r"((uint32_t)k + 1u) : "memory");
        }
      }
    }
  }
}

// kv_stage's one-launch path: the P side of the staged pull as ONE persistent launch.
// Chunk k (ChunkPlan order, layers [l0, l0 + nl)) is packed into ring slot (seq0 + k) % R
// once D freed it; the warp that completes chunk k release-stores ready = seq0 + k + 1 into
// D's word, strictly in chunk order (D reads ready >= v as "every chunk below v is packed").
// A warp waits for a slot only holding items it grabbed from that chunk, and the chunk R
// earlier is held by warps already past their wait (resident), so no co-residency is needed.
template <int SDT, int WDT, int U>
__global__ void __launch_bounds__(kThreads) k_stage_rows(const __grid_constant__ StageArgs a) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t cs = (uint32_t)a.p.cpr_shift;
  uint32_t* next = a.counters;               // [nchunks] items handed out
  uint32_t* done = a.counters + a.nchunks;   // [nchunks] items finished
  uint32_t* watermark = a.counters + 2 * a.nchunks;
  // free-slot waits: P runs ahead of the link, so its warps would spend most of the launch
  // polling D's free word -- one warp per CTA polls global memory at a time (smem token),
  // the others read the CTA's cached value (an acquire by the poller, re-released at CTA
  // scope), keeping the polls off the L2 slice D's NVLink reads also go through
  __shared__ uint32_t s_free, s_token;
  if (threadIdx.x == 0) {
    s_free = a.seq0 >= (1u << 30) ? a.seq0 - (1u << 30) : 0u;  // below any value waited for
    s_token = 0;
  }
  __syncthreads();
  for (int32_t k = 0; k < a.nchunks; ++k) {
    int32_t l0, nl;
    if (k < a.nramp) {
      l0 = a.ramp_l0[k];
      nl = a.ramp_nl[k];
    } else {
      l0 = a.lb + a.rsum + (k - a.nramp) * a.step;
      nl = min(a.step, a.le - l0);
    }
    const uint32_t n_k = (uint32_t)nl * a.items_per_layer;
    const uint32_t seq = a.seq0 + (uint32_t)k;
    uint8_t* wire = a.ring[seq % (uint32_t)a.R];
    bool waited = false;
    while (true) {
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(next + k, kPullGrab);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base >= n_k) break;
      if (!waited) {  // the slot last held chunk seq - R: D must have read it
        if (lane == 0 && (uint64_t)a.seq0 + (uint64_t)k + 1u > (uint64_t)a.R) {
          const uint32_t need = seq + 1u - (uint32_t)a.R;
          const uint64_t t0 = globaltimer_ns();
          while (true) {
            uint32_t v;
            asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(&s_free)) : "memory");
            if ((int32_t)(v - need) >= 0) break;
            if (atomicCAS(&s_token, 0u, 1u) == 0u) {
              // every value stored is a read of the (monotone) global word, so s_free never
              // exceeds it; the release passes this acquire on to the CTA's readers
              uint32_t x;
              asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(x) : "l"(a.freef) : "memory");
              if ((int32_t)(x - v) > 0)
                asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(smem_u32(&s_free)), "r"(x) : "memory");
              atomicExch(&s_token, 0u);
              if ((int32_t)(x - need) >= 0) break;
            }
            if (globaltimer_ns() - t0 > a.timeout_ns) {
              *a.err = 1;
              break;
            }
            __nanosleep(a.spin_ns);
          }
        }
        __syncwarp();
        waited = true;
      }
      const uint32_t end = min(n_k, base + kPullGrab);
      for (uint32_t item = base; item < end; ++item) pack_item<SDT, WDT, U>(a.p, item, l0, wire, lane, cs);
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        const uint32_t cnt = end - base;
        if (atomicAdd(done + k, cnt) + cnt == n_k) {
          uint32_t wm;
          while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(wm) : "l"(watermark) : "memory");
            if (wm == (uint32_t)k) break;
            __nanosleep(64);
          }
          __threadfence_system();
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.ready), "r"(seq + 1u) : "memory");
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(watermark), "r"((uint32_t)k + 1u) : "memory");
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// K2: pack (Fig. 5 flatten) -- wire order (layer, K/V, head in overlap, token, dim)
// ------------------------------------------------------------------------------------
template <int VEC, int SDT, int WDT, int U>
__global__ void __launch_bounds__(kThreads) k_pack(const __grid_constant__ PackArgs a) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = (blockIdx.x * (uint32_t)kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * (uint32_t)kThreads) >> 5;
  const uint64_t total = a.total;
  const uint64_t nseg = (total + 32u * U - 1) / (32u * U);
  for (uint64_t seg = warp; seg < nseg; seg += nwarps) {
    Chunk<SDT, VEC> in[U];
    float ssc[U], inv[U];
    uint64_t gg[U];
    bool act[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint64_t g64 = seg * (32u * U) + (uint32_t)k * 32u + lane;
      gg[k] = g64;
      act[k] = g64 < total;
      ssc[k] = 1.f;
      inv[k] = 1.f;
      if (act[k]) {
        uint32_t n = (uint32_t)g64;
        const uint32_t dch = divmod(n, a.f_dch);
        const uint32_t tok = divmod(n, a.f_tok);
        const uint32_t hh = divmod(n, a.f_nh);
        const uint32_t c = take_kv(n, a.kv1, a.c0);
        const uint32_t l = n;
        const int32_t r = __ldg(a.tok_req + tok);
        uint32_t t = tok - (uint32_t)__ldg(a.tok_off + r);
        const uint32_t sslot = divmod(t, a.f_bp);
        const int64_t sblk = __ldg(a.s_blk_ids + __ldg(a.s_blk_off + r) + t);
        const uint32_t h = (uint32_t)a.hb + hh;
        const uint32_t hp = h - (uint32_t)a.p * (uint32_t)a.Hp;
        const int64_t layer = a.lb + (int64_t)l;
        const int64_t sl = layer - a.s_l0, dl = layer - a.d_l0;  // pool-local layers
        const int64_t soff = sl * a.ss[KV_AX_LAYER] + (int64_t)c * a.ss[KV_AX_KV] + sblk * a.ss[KV_AX_BLOCK] +
                             (int64_t)sslot * a.ss[KV_AX_SLOT] + (int64_t)hp * a.ss[KV_AX_HEAD] +
                             dim_off(dch * VEC, a.ss[KV_AX_DIM], a.s_dk);
        load_chunk<SDT, VEC>(in[k], a.src + soff * Tr<SDT>::B);
        if constexpr (is_fp8(SDT) && SDT != WDT) ssc[k] = __ldg(a.sscale + (sl * 2 + c) * a.Hp + hp);
        if constexpr (is_fp8(WDT) && SDT != WDT)
          inv[k] = __frcp_rn(__ldg(a.dscale + (dl * 2 + c) * a.Hd + (h - (uint32_t)a.q * (uint32_t)a.Hd)));
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (!act[k]) continue;
      Chunk<WDT, VEC> o;
      cast_chunk<SDT, WDT, VEC>(in[k], o, ssc[k], inv[k]);
      store_chunk<WDT, VEC>(a.wire + gg[k] * (uint64_t)Chunk<WDT, VEC>::BYTES, o);
    }
  }
}

// ------------------------------------------------------------------------------------
// K3: unpack (Fig. 5 restore) -- destination-driven over the overlap heads
// ------------------------------------------------------------------------------------
template <int VEC, int WDT, int DDT, int U>
__global__ void __launch_bounds__(kThreads) k_unpack(const __grid_constant__ UnpackArgs a) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = (blockIdx.x * (uint32_t)kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * (uint32_t)kThreads) >> 5;
  const uint64_t total = a.total;
  const uint64_t nseg = (total + 32u * U - 1) / (32u * U);
  for (uint64_t seg = warp; seg < nseg; seg += nwarps) {
    Chunk<WDT, VEC> in[U];
    uint8_t* dp[U];
    float ssc[U], inv[U];
    bool act[U], zero[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint64_t g64 = seg * (32u * U) + (uint32_t)k * 32u + lane;
      act[k] = g64 < total;
      zero[k] = false;
      dp[k] = nullptr;
      ssc[k] = 1.f;
      inv[k] = 1.f;
      if (act[k]) {
        uint32_t n = (uint32_t)g64;
        const uint32_t dch = divmod(n, a.f_dch);
        const uint32_t in0 = divmod(n, a.f_in0);
        const uint32_t in1 = divmod(n, a.f_in1);
        const uint32_t c = take_kv(n, a.kv1, a.c0);
        const uint32_t l = divmod(n, a.f_l);
        const uint32_t bl = n;
        const uint32_t slot = a.slot_inner ? in0 : in1;
        const uint32_t hh = a.slot_inner ? in1 : in0;
        const int32_t r = __ldg(a.d_blk_req + bl);
        const int32_t tok0 = __ldg(a.tok_off + r);
        const int32_t T = __ldg(a.tok_off + r + 1) - tok0;
        const uint32_t t = (uint32_t)(bl - __ldg(a.d_blk_off + r)) * (uint32_t)a.Bd + slot;
        const int64_t dblk = __ldg(a.d_blk_ids + bl);
        const int64_t layer = a.lb + (int64_t)l;
        const int64_t sl = layer - a.s_l0, dl = layer - a.d_l0;  // pool-local layers
        const uint32_t h = (uint32_t)a.hb + hh;
        const uint32_t hq = h - (uint32_t)a.q * (uint32_t)a.Hd;
        const int64_t doff = dl * a.ds[KV_AX_LAYER] + (int64_t)c * a.ds[KV_AX_KV] + dblk * a.ds[KV_AX_BLOCK] +
                             (int64_t)slot * a.ds[KV_AX_SLOT] + (int64_t)hq * a.ds[KV_AX_HEAD] +
                             dim_off(dch * VEC, a.ds[KV_AX_DIM], a.d_dk);
        dp[k] = a.dst + doff * Tr<DDT>::B;
        if ((int32_t)t >= T) {
          zero[k] = true;
        } else {
          const int64_t woff = ((((int64_t)l * wkv(a.kv1) + (c - (uint32_t)a.c0)) * a.nh + hh) * a.total_tokens + tok0 + t) *
                                   a.D + (int64_t)dch * VEC;
          load_chunk<WDT, VEC>(in[k], a.wire + woff * Tr<WDT>::B);
          if constexpr (is_fp8(WDT) && WDT != DDT)
            ssc[k] = __ldg(a.sscale + (sl * 2 + c) * a.Hp + (h - (uint32_t)a.p * (uint32_t)a.Hp));
          if constexpr (is_fp8(DDT) && WDT != DDT)
            inv[k] = __frcp_rn(__ldg(a.dscale + (dl * 2 + c) * a.Hd + hq));
        }
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (!act[k]) continue;
      Chunk<DDT, VEC> o;
      if (zero[k])
        zero_chunk(o);
      else
        cast_chunk<WDT, DDT, VEC>(in[k], o, ssc[k], inv[k]);
      store_chunk<DDT, VEC>(dp[k], o);
    }
  }
}

// ------------------------------------------------------------------------------------
// NEXT-1: dynamic fp8 scales.  Pass 1: max |x| over the valid tokens of every (layer,
// K/V, D-local head), one lane per token row, warp max, one atomicMax per item on the
// float bits (non-negative floats order like unsigned ints) written in place into the
// output array.  Pass 2: s = RN(amax / 448), or 1 when amax is 0.  Element-wise so any
// axis order works; this is a one-read side pass, not the hot path.
// ------------------------------------------------------------------------------------
template <int SDT>
__global__ void __launch_bounds__(kThreads) k_amax(const __grid_constant__ AmaxArgs a) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = (blockIdx.x * (uint32_t)kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * (uint32_t)kThreads) >> 5;
  for (uint32_t item = warp; item < a.n_items; item += nwarps) {
    uint32_t n = item;
    const uint32_t tg = divmod(n, a.f_tg);
    const uint32_t hq = (uint32_t)a.hq0 + divmod(n, a.f_hd);
    const uint32_t c = take_kv(n, a.kv1, a.c0);
    const int64_t layer = a.lb + (int64_t)n;
    const int64_t sl = layer - a.s_l0, dl = layer - a.d_l0;  // pool-local layers
    const uint32_t tok = tg * 32u + lane;
    float m = 0.f;
    if (tok < a.n_tok) {
      const int32_t r = __ldg(a.tok_req + tok);
      uint32_t t = tok - (uint32_t)__ldg(a.tok_off + r);
      const uint32_t sslot = divmod(t, a.f_bp);
      const int64_t sblk = __ldg(a.s_blk_ids + __ldg(a.s_blk_off + r) + t);
      const uint32_t h = (uint32_t)a.q * (uint32_t)a.Hd + hq;
      const uint32_t p = fdiv(h, a.f_hp);
      const uint32_t hp = h - p * (uint32_t)a.Hp;
      const int si = a.src_of_p[p];
      const uint8_t* base = a.src[si] + (sl * a.ss[KV_AX_LAYER] + (int64_t)c * a.ss[KV_AX_KV] +
                                         sblk * a.ss[KV_AX_BLOCK] + (int64_t)sslot * a.ss[KV_AX_SLOT] +
                                         (int64_t)hp * a.ss[KV_AX_HEAD]) * Tr<SDT>::B;
      float sc = 1.f;
      if constexpr (is_fp8(SDT)) sc = __ldg(a.sscale[si] + (sl * 2 + c) * a.Hp + hp);
      const int64_t sdim = a.ss[KV_AX_DIM];
      for (int32_t d = 0; d < a.D; ++d) {
        Chunk<SDT, 1> e;
        load_chunk<SDT, 1>(e, base + dim_off((uint32_t)d, sdim, a.s_dk) * Tr<SDT>::B);
        float v = to_f32<SDT>(e.w[0]);
        if constexpr (is_fp8(SDT)) v = __fmul_rn(v, sc);
        v = fabsf(v);
        if (v <= 3.402823466e38f) m = fmaxf(m, v);  // skips NaN and Inf
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0 && m > 0.f) atomicMax(a.amax_bits + (dl * 2 + c) * a.Hd + hq, __float_as_uint(m));
  }
}

// Row path of the amax pass (head_dim innermost in the source, rows of 16-B multiples):
// an item is kAmaxG consecutive groups of 32 tokens of one (layer, K/V, head); each lane
// owns one token row, the warp streams the 32 rows' 16-B chunks with shuffled row
// addresses (coalesced, like the convert), keeps a running max over the whole item and
// issues ONE atomicMax -- the element-wise kernel issued one per 32 tokens, and the
// contention on the few (layer, K/V, head) words made it ~4x slower than a read pass.
constexpr uint32_t kAmaxG = 16;

template <int SDT>
__global__ void __launch_bounds__(kThreads) k_amax_rows(const __grid_constant__ AmaxArgs a) {
  constexpr int VEC = 16 / Tr<SDT>::B;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = (blockIdx.x * (uint32_t)kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * (uint32_t)kThreads) >> 5;
  const uint32_t cs = (uint32_t)a.cpr_shift;
  const uint32_t cmask = (1u << cs) - 1u, nch = 32u << cs;
  for (uint32_t item = warp; item < a.n_row_items; item += nwarps) {
    uint32_t n = item;
    const uint32_t tgc = divmod(n, a.f_tgc);
    const uint32_t hq = (uint32_t)a.hq0 + divmod(n, a.f_hd);
    const uint32_t c = take_kv(n, a.kv1, a.c0);
    const int64_t layer = a.lb + (int64_t)n;
    const int64_t sl = layer - a.s_l0;
    const uint32_t h = (uint32_t)a.q * (uint32_t)a.Hd + hq;
    const uint32_t p = fdiv(h, a.f_hp);
    const uint32_t hp = h - p * (uint32_t)a.Hp;
    const int si = a.src_of_p[p];
    float sc = 1.f;
    if constexpr (is_fp8(SDT)) sc = __ldg(a.sscale[si] + (sl * 2 + c) * a.Hp + hp);
    const uint8_t* lbase = a.src[si] + (sl * a.ss[KV_AX_LAYER] + (int64_t)c * a.ss[KV_AX_KV] +
                                        (int64_t)hp * a.ss[KV_AX_HEAD]) * Tr<SDT>::B;
    float m = 0.f;
    for (uint32_t g = 0; g < kAmaxG; ++g) {
      const uint32_t tok = (tgc * kAmaxG + g) * 32u + lane;
      if (__all_sync(0xffffffffu, tok >= a.n_tok)) break;
      uint64_t rp = 0;
      if (tok < a.n_tok) {
        const int32_t r = __ldg(a.tok_req + tok);
        uint32_t t = tok - (uint32_t)__ldg(a.tok_off + r);
        const uint32_t sslot = divmod(t, a.f_bp);
        const int64_t sblk = __ldg(a.s_blk_ids + __ldg(a.s_blk_off + r) + t);
        rp = (uint64_t)(lbase + (sblk * a.ss[KV_AX_BLOCK] + (int64_t)sslot * a.ss[KV_AX_SLOT]) * Tr<SDT>::B);
      }
#pragma unroll 4
      for (uint32_t idx = lane; idx < nch; idx += 32u) {
        const uint64_t r0 = __shfl_sync(0xffffffffu, rp, (idx >> cs) & 31u);
        if (r0 == 0) continue;
        Chunk<SDT, VEC> e;
        load_chunk<SDT, VEC>(e, reinterpret_cast<const uint8_t*>(r0) + (idx & cmask) * 16u);
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          float v = to_f32<SDT>(get_elem<SDT>(e.w, i));
          if constexpr (is_fp8(SDT)) v = __fmul_rn(v, sc);
          v = fabsf(v);
          if (v <= 3.402823466e38f) m = fmaxf(m, v);  // skips NaN and Inf
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0 && m > 0.f) atomicMax(a.amax_bits + (layer - a.d_l0) * 2 * a.Hd + c * a.Hd + hq, __float_as_uint(m));
  }
}

// entries [begin, end) of an [L][2][Hd] scale array; a K-only / V-only pass leaves the
// other half untouched, a P rank's share ([hq0, hq0 + nhq)) the other heads
__device__ __forceinline__ bool amax_entry(int64_t i, int32_t Hd, int32_t kv1, int32_t c0, int32_t hq0, int32_t nhq) {
  const int32_t h = (int32_t)(i % Hd);
  return (!kv1 || (int32_t)((i / Hd) & 1) == c0) && h >= hq0 && h < hq0 + nhq;
}
__global__ void k_amax_init(uint32_t* bits, int64_t begin, int64_t end, int32_t Hd, int32_t kv1, int32_t c0,
                            int32_t hq0, int32_t nhq) {
  for (int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < end; i += (int64_t)gridDim.x * blockDim.x)
    if (amax_entry(i, Hd, kv1, c0, hq0, nhq)) bits[i] = 0u;
}
// s = RN(amax / qmax), qmax = the destination fp8's largest finite value (448 / 240); with
// `peer` the scale is also stored there (D's array over NVLink: the dynamic-scale pull)
__global__ void k_amax_finalize(uint32_t* bits, int64_t begin, int64_t end, float qmax, int32_t Hd, int32_t kv1,
                                int32_t c0, int32_t hq0, int32_t nhq, float* peer) {
  for (int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < end; i += (int64_t)gridDim.x * blockDim.x) {
    if (!amax_entry(i, Hd, kv1, c0, hq0, nhq)) continue;
    const float amax = __uint_as_float(bits[i]);
    const float s0 = __fdiv_rn(amax, qmax);
    const float s = s0 > 0.f ? s0 : 1.0f;
    reinterpret_cast<float*>(bits)[i] = s;
    if (peer) peer[i] = s;
  }
}

// ------------------------------------------------------------------------------------
// K5: completion flags (A11)
// ------------------------------------------------------------------------------------
__global__ void k_signal(uint32_t* flag, uint32_t value) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_wait(const uint32_t* flag, uint32_t value, uint64_t timeout_ns, int32_t* err) {
  if (threadIdx.x != 0) return;
  const uint64_t t0 = globaltimer();
  while (true) {
    uint32_t x;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(x) : "l"(flag) : "memory");
    if ((int32_t)(x - value) >= 0) break;
    if (globaltimer() - t0 > timeout_ns) {
      *err = 1;
      break;
    }
    __nanosleep(64);
  }
}

// ------------------------------------------------------------------------------------
// launch helpers
// ------------------------------------------------------------------------------------
int num_sms() {
  static thread_local int dev = -1, sms = 0;
  int d = 0;
  cudaGetDevice(&d);
  if (d != dev) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
    dev = d;
  }
  const int budget = (d >= 0 && d < kMaxDevices) ? g_sm_budget[d].load(std::memory_order_relaxed) : 0;
  return (budget > 0 && budget < sms) ? budget : sms;
}

template <typename K>
int grid_for(K kernel, uint64_t total, int per_thread) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, 0);
  if (occ < 1) occ = 1;
  const uint64_t need = (total + (uint64_t)kThreads * per_thread - 1) / ((uint64_t)kThreads * per_thread);
  uint64_t cap = (uint64_t)num_sms() * occ;
  uint64_t g = need < cap ? need : cap;
  return (int)(g < 1 ? 1 : g);
}

// Row kernels: one warp per 32-row item; grid = min(items / 8 warps, SMs x occupancy).
template <typename K>
int grid_for_items(K kernel, uint64_t n_items) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, 0);
  if (occ < 1) occ = 1;
  const uint64_t need = (n_items + (kThreads / 32) - 1) / (kThreads / 32);
  const uint64_t cap = (uint64_t)num_sms() * occ;
  return (int)std::max<uint64_t>(1, std::min(need, cap));
}

int32_t log2_pow2(uint32_t x) {
  int32_t l = 0;
  while ((1u << l) < x) ++l;
  return l;
}

// Sub-tile of an item: ts slots x th heads, ts * th = 32.  Up to 8 heads (so a P-side
// run of several heads and a D-side run of several slots are both >= 1 KB for D = 128),
// fewer slots when blocks are small.  KVX_TS overrides ts (experiments only).
void subtile_shape(uint32_t Bd, uint32_t H, uint32_t* ts_out, uint32_t* th_out) {
  auto pow2ceil = [](uint32_t x) {
    uint32_t p = 1;
    while (p < x) p <<= 1;
    return p;
  };
  uint32_t th = pow2ceil(std::min<uint32_t>(H, 8u));
  uint32_t ts = 32u / th;
  if (ts > pow2ceil(Bd)) {
    ts = pow2ceil(Bd);
    th = 32u / ts;
  }
  if (const char* e = getenv("KVX_TS")) {
    const uint32_t v = (uint32_t)atoi(e);
    if (v >= 1 && v <= 32 && (v & (v - 1)) == 0) {
      ts = v;
      th = 32u / v;
    }
  }
  *ts_out = ts;
  *th_out = th;
}

// U chunks per thread per segment: keep ~64 B of loads in flight per thread.
template <int SDT, int VEC>
constexpr int unroll_for() {
  return VEC == 1 ? 4 : (Tr<SDT>::B == 4 ? 2 : 4);
}

template <int VEC, int SDT, int DDT>
cudaError_t conv_t(const ConvArgs& a0, cudaStream_t s) {
  constexpr int U = unroll_for<SDT, VEC>();
  if constexpr (VEC == 8) {
    // row-tiled fast path: work items of 32 rows (one per lane) = 2-D sub-tiles
    ConvArgs a = a0;
    const uint32_t cpr = a.f_cpr.d;
    a.rows_per_tile = a.Bd * a.Hd_eff;
    a.rows_per_item = 32;
    a.cpr_shift = log2_pow2(cpr);
    uint32_t ts, th;
    subtile_shape((uint32_t)a.Bd, (uint32_t)a.Hd_eff, &ts, &th);
    a.ts_log2 = log2_pow2(ts);
    const uint32_t nsb = ((uint32_t)a.Bd + ts - 1) / ts, nhb = ((uint32_t)a.Hd_eff + th - 1) / th;
    a.f_sb = make_fastdiv(nsb);
    a.f_items = make_fastdiv(nsb * nhb);
    a.n_items = (uint32_t)(a.total64 / ((uint64_t)a.rows_per_tile * cpr) * nsb * nhb);
    a.items_per_block = a.f_bl.d ? a.n_items / a.f_bl.d : 0;
    // 1-byte sources: 16-element chunks (whole 16-B loads, 4 in flight = 64 B per lane, like
    // the 2-byte sources' 8-element chunks); KVX_FP8_VEC16=0 reverts to 8-element chunks
    static const int wide1 = getenv("KVX_FP8_VEC16") ? atoi(getenv("KVX_FP8_VEC16")) : 1;
    if (a.split) {
      auto k = k_convert_rows<SDT, DDT, U, 8, true>;
      k<<<grid_for_items(k, a.n_items), kThreads, 0, s>>>(a);
    } else {
      bool done = false;
      if constexpr (Tr<SDT>::B == 1 && Tr<DDT>::B <= 2) {
        if (wide1 && cpr >= 2) {
          a.cpr_shift = log2_pow2(cpr / 2);
          auto k = k_convert_rows<SDT, DDT, 4, 16>;
          k<<<grid_for_items(k, a.n_items), kThreads, 0, s>>>(a);
          done = true;
        }
      }
      if (!done) {
        auto k = k_convert_rows<SDT, DDT, U>;
        k<<<grid_for_items(k, a.n_items), kThreads, 0, s>>>(a);
      }
    }
  } else {
    auto k = k_convert<VEC, SDT, DDT, U>;
    k<<<grid_for(k, a0.total, U), kThreads, 0, s>>>(a0);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}
template <int VEC, int SDT, int WDT>
cudaError_t pack_t(const PackArgs& a0, cudaStream_t s) {
  constexpr int U = unroll_for<SDT, VEC>();
  if constexpr (VEC == 8) {
    PackArgs a = a0;
    a.cpr_shift = log2_pow2(a.f_dch.d);
    const uint32_t T_all = a.f_tok.d;
    const uint32_t ntg = (T_all + 31u) / 32u;
    a.f_tg = make_fastdiv(ntg);
    a.n_items = (uint32_t)a.Lc * (a.kv1 ? 1u : 2u) * (uint32_t)a.nh * ntg;
    auto k = k_pack_rows<SDT, WDT, U>;
    k<<<grid_for_items(k, a.n_items), kThreads, 0, s>>>(a);
  } else {
    auto k = k_pack<VEC, SDT, WDT, U>;
    k<<<grid_for(k, a0.total, U), kThreads, 0, s>>>(a0);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}
template <int VEC, int WDT, int DDT>
cudaError_t unpack_t(const UnpackArgs& a0, cudaStream_t s) {
  constexpr int U = unroll_for<WDT, VEC>();
  if constexpr (VEC == 8) {
    UnpackArgs a = a0;
    a.cpr_shift = log2_pow2(a.f_dch.d);
    uint32_t ts, th;
    subtile_shape((uint32_t)a.Bd, (uint32_t)a.nh, &ts, &th);
    a.ts_log2 = log2_pow2(ts);
    const uint32_t nsb = ((uint32_t)a.Bd + ts - 1) / ts, nhb = ((uint32_t)a.nh + th - 1) / th;
    a.f_sb = make_fastdiv(nsb);
    a.f_items = make_fastdiv(nsb * nhb);
    a.n_items = a.f_bl.d * (uint32_t)a.Lc * (a.kv1 ? 1u : 2u) * nsb * nhb;
    auto k = k_unpack_rows<WDT, DDT, U>;
    k<<<grid_for_items(k, a.n_items), kThreads, 0, s>>>(a);
  } else {
    auto k = k_unpack<VEC, WDT, DDT, U>;
    k<<<grid_for(k, a0.total, U), kThreads, 0, s>>>(a0);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// dtype dispatch: F(vec, sdt, ddt)
#define KVX_DISPATCH_DDT(FN, VEC, SDT, ddt, ...)                       \
  switch (ddt) {                                                       \
    case KV_F16: return FN<VEC, SDT, KV_F16>(__VA_ARGS__);             \
    case KV_BF16: return FN<VEC, SDT, KV_BF16>(__VA_ARGS__);           \
    case KV_F8E4M3: return FN<VEC, SDT, KV_F8E4M3>(__VA_ARGS__);       \
    case KV_F8E4M3FNUZ: return FN<VEC, SDT, KV_F8E4M3FNUZ>(__VA_ARGS__); \
    case KV_F32: return FN<VEC, SDT, KV_F32>(__VA_ARGS__);             \
  }                                                                    \
  return cudaErrorInvalidValue;

#define KVX_DISPATCH(FN, VEC, sdt, ddt, ...)                                   \
  switch (sdt) {                                                               \
    case KV_F16: { KVX_DISPATCH_DDT(FN, VEC, KV_F16, ddt, __VA_ARGS__) }       \
    case KV_BF16: { KVX_DISPATCH_DDT(FN, VEC, KV_BF16, ddt, __VA_ARGS__) }     \
    case KV_F8E4M3: { KVX_DISPATCH_DDT(FN, VEC, KV_F8E4M3, ddt, __VA_ARGS__) } \
    case KV_F8E4M3FNUZ: { KVX_DISPATCH_DDT(FN, VEC, KV_F8E4M3FNUZ, ddt, __VA_ARGS__) } \
    case KV_F32: { KVX_DISPATCH_DDT(FN, VEC, KV_F32, ddt, __VA_ARGS__) }       \
  }                                                                            \
  return cudaErrorInvalidValue;

template <int VEC, int SDT, int DDT>
cudaError_t tr_t(const ConvArgs& a, cudaStream_t s) {
  const size_t smem = (size_t)kTrWarps * a.Bd * (a.D + 16 / Tr<SDT>::B) * Tr<SDT>::B;
  auto k = k_convert_tr<SDT, DDT>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kTrWarps * 32, smem);
  if (occ < 1) occ = 1;
  const uint64_t need = (a.n_items + kTrWarps - 1) / kTrWarps;
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)num_sms() * occ));
  k<<<grid, kTrWarps * 32, smem, s>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}
template <int VEC>
cudaError_t tr_v(const ConvArgs& a, int sdt, int ddt, cudaStream_t s) {
  KVX_DISPATCH(tr_t, VEC, sdt, ddt, a, s)
}
template <int VEC, int SDT, int DDT>
cudaError_t tr8_t(const ConvArgs& a, cudaStream_t s) {
  auto k = k_convert_tr8<SDT, DDT, false>;
  // W16 only for 2-byte -> 2-byte: V pool bf16 -> bf16 0.80 -> 0.85 of copy; with an fp8
  // destination it measured 0.83 vs 0.85 (and a 4-byte destination spills)
  if constexpr (Tr<SDT>::B == 2 && Tr<DDT>::B == 2)
    if (a.tr_w16) k = k_convert_tr8<SDT, DDT, true>;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kTr8Threads, 0);
  if (occ < 1) occ = 1;
  const uint64_t groups = (a.n_items + 31) / 32;
  const uint64_t need = (groups + kTr8Threads / 32 - 1) / (kTr8Threads / 32);
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)num_sms() * occ));
  k<<<grid, kTr8Threads, 0, s>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}
template <int VEC>
cudaError_t tr8_v(const ConvArgs& a, int sdt, int ddt, cudaStream_t s) {
  KVX_DISPATCH(tr8_t, VEC, sdt, ddt, a, s)
}

template <int VEC>
cudaError_t conv_v(const ConvArgs& a, int sdt, int ddt, cudaStream_t s) {
  KVX_DISPATCH(conv_t, VEC, sdt, ddt, a, s)
}
template <int VEC>
cudaError_t pack_v(const PackArgs& a, int sdt, int wdt, cudaStream_t s) {
  KVX_DISPATCH(pack_t, VEC, sdt, wdt, a, s)
}
template <int VEC>
cudaError_t unpack_v(const UnpackArgs& a, int wdt, int ddt, cudaStream_t s) {
  KVX_DISPATCH(unpack_t, VEC, wdt, ddt, a, s)
}

}  // namespace

cudaError_t launch_convert_tr(const ConvArgs& a, int sdt, int ddt, cudaStream_t s) {
  if (a.n_items == 0) return cudaSuccess;
  return tr_v<8>(a, sdt, ddt, s);
}

namespace {
template <int SDT, int DDT>
cudaError_t tb_t(const TbArgs& a, cudaStream_t s) {
  auto k = a.mode == 2 ? k_convert_tb<SDT, DDT, 2> : k_convert_tb<SDT, DDT, 1>;
  const size_t tile = (size_t)a.tile_rows * 128u;
  const size_t lut = dual_scale(SDT, DDT) ? 256u + 256u * kTbConsumers : 0u;   // per-warp code tables
  const size_t smem = 1024 + (size_t)a.stages * tile + (size_t)a.stages * (16 + sizeof(TbMeta)) + lut;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 32 * (1 + kTbConsumers), smem);
  if (occ < 1) occ = 1;
  const uint64_t need = (a.c.n_items + kTbConsumers - 1) / kTbConsumers;
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)num_sms() * occ));
  k<<<grid, 32 * (1 + kTbConsumers), smem, s>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}
template <int SDT>
cudaError_t tb_d(const TbArgs& a, int ddt, cudaStream_t s) {
  switch (ddt) {
    case KV_F16: return tb_t<SDT, KV_F16>(a, s);
    case KV_BF16: return tb_t<SDT, KV_BF16>(a, s);
    case KV_F8E4M3: return tb_t<SDT, KV_F8E4M3>(a, s);
    case KV_F8E4M3FNUZ: return tb_t<SDT, KV_F8E4M3FNUZ>(a, s);
    case KV_F32: return tb_t<SDT, KV_F32>(a, s);
  }
  return cudaErrorInvalidValue;
}
}  // namespace

cudaError_t launch_convert_tb(const TbArgs& a, int sdt, int ddt, cudaStream_t s) {
  if (a.c.n_items == 0) return cudaSuccess;
  if (sdt == KV_F16) return tb_d<KV_F16>(a, ddt, s);
  if (sdt == KV_BF16) return tb_d<KV_BF16>(a, ddt, s);
  if (sdt == KV_F8E4M3) return tb_d<KV_F8E4M3>(a, ddt, s);
  if (sdt == KV_F8E4M3FNUZ) return tb_d<KV_F8E4M3FNUZ>(a, ddt, s);
  return cudaErrorInvalidValue;
}

cudaError_t launch_convert_tr8(const ConvArgs& a, int sdt, int ddt, cudaStream_t s) {
  if (a.n_items == 0) return cudaSuccess;
  return tr8_v<8>(a, sdt, ddt, s);
}
cudaError_t launch_requant(const ConvArgs& a0, int sdt, int ddt, cudaStream_t s) {
  if (a0.total64 == 0) return cudaSuccess;
  ConvArgs a = a0;
  const uint32_t cpr = a.f_cpr.d;  // 8-element chunks per row (D / 8)
  if (cpr < 2) return cudaErrorInvalidValue;
  a.cpr_shift = log2_pow2(cpr / 2);  // 16-byte chunks
  a.rows_per_tile = a.Bd * a.Hd_eff;
  // sub-tiles as long along the slots as the block allows: the rows of one warp instruction
  // (32 / 16-B chunks per row) are consecutive slots of one head -- one code table
  uint32_t ts = 1;
  while (ts < (uint32_t)a.Bd && ts < 32u) ts <<= 1;
  const uint32_t th = 32u / ts;
  a.ts_log2 = log2_pow2(ts);
  const uint32_t nsb = ((uint32_t)a.Bd + ts - 1) / ts, nhb = ((uint32_t)a.Hd_eff + th - 1) / th;
  a.f_sb = make_fastdiv(nsb);
  a.f_items = make_fastdiv(nsb * nhb);
  a.n_items = (uint32_t)(a.total64 / ((uint64_t)a.rows_per_tile * cpr) * nsb * nhb);
  const uint32_t tpl = a.f_nd.d * (a.kv1 ? 1u : 2u) * (uint32_t)a.Hd_eff;   // tables per layer
  const uint32_t per_layer = a.n_items / (uint32_t)a.Lc;                     // items per layer
  auto launch = [&](auto k, int minb) -> cudaError_t {
    // one wave of CTAs, each a contiguous range of items (layer-outermost): the tables of
    // the <= rq_layers layers the range touches
    const uint64_t need = (a.n_items + (kThreads / 32) - 1) / (kThreads / 32);
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)num_sms() * minb));
    a.rq_per_cta = (uint32_t)((a.n_items + (uint64_t)grid - 1) / (uint64_t)grid);
    a.rq_layers = std::min<uint32_t>((uint32_t)a.Lc, (a.rq_per_cta + per_layer - 1) / per_layer + 1u);
    const size_t smem = (size_t)a.rq_layers * tpl * 128u + 256u;   // 128-B tables, 256-B alignment slack
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, kThreads, smem, s>>>(a);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
  };
  // 4 loads in flight per lane x 4 CTAs/SM (64 registers): measured best of {8 x 2, 4 x 3,
  // 4 x 4, 2 x 4, 4 x 5, 2 x 6, 4 x 6} on the c4-pair shape (profiles/r02/requant_lut.txt)
  if (sdt == KV_F8E4M3FNUZ && ddt == KV_F8E4M3) return launch(k_requant_rows<KV_F8E4M3FNUZ, KV_F8E4M3, 4, 4>, 4);
  if (sdt == KV_F8E4M3 && ddt == KV_F8E4M3FNUZ) return launch(k_requant_rows<KV_F8E4M3, KV_F8E4M3FNUZ, 4, 4>, 4);
  return cudaErrorInvalidValue;
}

cudaError_t launch_convert(const ConvArgs& a, int vec, int sdt, int ddt, cudaStream_t s) {
  if (a.total64 == 0) return cudaSuccess;
  return vec == 8 ? conv_v<8>(a, sdt, ddt, s) : conv_v<1>(a, sdt, ddt, s);
}
cudaError_t launch_pack(const PackArgs& a, int vec, int sdt, int wdt, cudaStream_t s) {
  if (a.total == 0) return cudaSuccess;
  return vec == 8 ? pack_v<8>(a, sdt, wdt, s) : pack_v<1>(a, sdt, wdt, s);
}
cudaError_t launch_unpack(const UnpackArgs& a, int vec, int wdt, int ddt, cudaStream_t s) {
  if (a.total == 0) return cudaSuccess;
  return vec == 8 ? unpack_v<8>(a, wdt, ddt, s) : unpack_v<1>(a, wdt, ddt, s);
}
namespace {
template <int SDT, int DDT>
cudaError_t tc_t(const TileArgs& a, cudaStream_t s) {
  if constexpr (Tr<SDT>::B > 2) {
    return cudaErrorInvalidValue;
  } else {
    auto k = k_tile_cast<SDT, DDT>;
    const size_t smem = (size_t)a.stages * (size_t)a.stage_bytes + (size_t)a.stages * (16 + sizeof(TcMeta)) + 16;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 32 * (1 + kTbConsumers), smem);
    if (occ < 1) occ = 1;
    const uint64_t need = (a.n_items + kTbConsumers - 1) / kTbConsumers;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)num_sms() * occ));
    k<<<grid, 32 * (1 + kTbConsumers), smem, s>>>(a);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
  }
}
template <int SDT>
cudaError_t tc_d(const TileArgs& a, int ddt, cudaStream_t s) {
  switch (ddt) {
    case KV_F16: return tc_t<SDT, KV_F16>(a, s);
    case KV_BF16: return tc_t<SDT, KV_BF16>(a, s);
    case KV_F8E4M3: return tc_t<SDT, KV_F8E4M3>(a, s);
    case KV_F8E4M3FNUZ: return tc_t<SDT, KV_F8E4M3FNUZ>(a, s);
    case KV_F32: return tc_t<SDT, KV_F32>(a, s);
  }
  return cudaErrorInvalidValue;
}
}  // namespace

cudaError_t launch_tile_cast(const TileArgs& a, int sdt, int ddt, cudaStream_t s) {
  if (a.n_items == 0) return cudaSuccess;
  switch (sdt) {
    case KV_F16: return tc_d<KV_F16>(a, ddt, s);
    case KV_BF16: return tc_d<KV_BF16>(a, ddt, s);
    case KV_F8E4M3: return tc_d<KV_F8E4M3>(a, ddt, s);
    case KV_F8E4M3FNUZ: return tc_d<KV_F8E4M3FNUZ>(a, ddt, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_tile_copy(const TileArgs& a, cudaStream_t s) {
  if (a.n_items == 0) return cudaSuccess;
  const size_t smem = (size_t)a.stages * (size_t)a.stage_bytes + 8 * (size_t)a.stages;
  cudaError_t e = cudaFuncSetAttribute(k_tile_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tile_copy, 32, smem);
  if (occ < 1) occ = 1;
  const uint64_t cap = (uint64_t)num_sms() * (uint64_t)occ;
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(a.n_items, cap));
  k_tile_copy<<<grid, 32, smem, s>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

namespace {
template <int DT>
cudaError_t pull_rows_t(PullArgs& a, cudaStream_t s) {
  constexpr int U = unroll_for<DT, 8>();
  auto k = k_pull_rows<DT, U>;
  // no co-residency needed: a warp only waits for chunk k holding items it grabbed from k,
  // and the slots chunk k waits on are freed by items already grabbed (hence resident)
  k<<<grid_for_items(k, a.items_full > a.items_last ? a.items_full : a.items_last), kThreads, 0, s>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_pull_rows(PullArgs& a, int dt, cudaStream_t s) {
  if (a.nchunks <= 0) return cudaSuccess;
  a.watermark = a.counters + 2 * (size_t)a.nchunks;
  cudaError_t e0 = cudaMemsetAsync(a.counters, 0, (2 * (size_t)a.nchunks + 1) * sizeof(uint32_t), s);
  if (e0 != cudaSuccess) return e0;
  a.cpr_shift = log2_pow2((uint32_t)(a.D / 8));
  uint32_t ts, th;
  subtile_shape((uint32_t)a.Bd, (uint32_t)a.nh, &ts, &th);
  a.ts_log2 = log2_pow2(ts);
  const uint32_t nsb = ((uint32_t)a.Bd + ts - 1) / ts, nhb = ((uint32_t)a.nh + th - 1) / th;
  a.f_sb = make_fastdiv(nsb);
  a.f_items = make_fastdiv(nsb * nhb);
  const uint32_t per_layer = a.f_src.d * (a.kv1 ? 1u : 2u) * nsb * nhb * a.n_blk;
  for (int32_t k = 0; k < a.nramp; ++k) {  // ramp chunks (ChunkPlan)
    const int32_t l1 = k + 1 < a.nramp ? a.ramp_l0[k + 1] : a.lb + a.rsum;
    a.ramp_items[k] = per_layer * (uint32_t)(l1 - a.ramp_l0[k]);
    a.f_l_ramp[k] = make_fastdiv((uint32_t)(l1 - a.ramp_l0[k]));
  }
  const uint32_t nl_last = (uint32_t)(a.le - (a.lb + a.rsum + (a.nchunks - a.nramp - 1) * a.step));
  a.items_last = per_layer * nl_last;
  a.items_full = per_layer * (uint32_t)a.step;
  a.f_l_full = make_fastdiv((uint32_t)a.step);
  a.f_l_last = make_fastdiv(nl_last);
  switch (dt) {
    case KV_F16: return pull_rows_t<KV_F16>(a, s);
    case KV_BF16: return pull_rows_t<KV_BF16>(a, s);
    case KV_F8E4M3: return pull_rows_t<KV_F8E4M3>(a, s);
    case KV_F8E4M3FNUZ: return pull_rows_t<KV_F8E4M3FNUZ>(a, s);
    case KV_F32: return pull_rows_t<KV_F32>(a, s);
  }
  return cudaErrorInvalidValue;
}

namespace {
template <int SDT, int WDT>
cudaError_t stage_rows_t(StageArgs& a, cudaStream_t s) {
  constexpr int U = unroll_for<SDT, 8>();
  auto k = k_stage_rows<SDT, WDT, U>;
  PackArgs& p = a.p;
  p.cpr_shift = log2_pow2(p.f_dch.d);
  const uint32_t ntg = (p.f_tok.d + 31u) / 32u;
  p.f_tg = make_fastdiv(ntg);
  a.items_per_layer = (p.kv1 ? 1u : 2u) * (uint32_t)p.nh * ntg;
  // P only has to out-run the link (it reads 2x and writes 1x the wire bytes): two CTAs
  // per SM keep ~2x the link's rate in flight with fewer spinning warps
  const int grid = std::min(grid_for_items(k, (uint64_t)a.items_per_layer * (uint64_t)a.step), 2 * num_sms());
  k<<<grid, kThreads, 0, s>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}
template <int SDT>
cudaError_t stage_rows_w(StageArgs& a, int wdt, cudaStream_t s) {
  switch (wdt) {
    case KV_F16: return stage_rows_t<SDT, KV_F16>(a, s);
    case KV_BF16: return stage_rows_t<SDT, KV_BF16>(a, s);
    case KV_F8E4M3: return stage_rows_t<SDT, KV_F8E4M3>(a, s);
    case KV_F8E4M3FNUZ: return stage_rows_t<SDT, KV_F8E4M3FNUZ>(a, s);
  }
  return cudaErrorInvalidValue;
}
}  // namespace

cudaError_t launch_stage_rows(StageArgs& a, int sdt, int wdt, cudaStream_t s) {
  if (a.nchunks <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(a.counters, 0, (2 * (size_t)a.nchunks + 1) * sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  switch (sdt) {  // narrowing casts (the staged pull's reason): 4- / 2-byte sources
    case KV_F32: return stage_rows_w<KV_F32>(a, wdt, s);
    case KV_F16: return stage_rows_w<KV_F16>(a, wdt, s);
    case KV_BF16: return stage_rows_w<KV_BF16>(a, wdt, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_amax(const AmaxArgs& a, int sdt, float* out, cudaStream_t s) {
  const int64_t begin = (int64_t)(a.lb - a.d_l0) * 2 * a.Hd, end = (int64_t)(a.lb - a.d_l0 + a.Lc) * 2 * a.Hd;
  const int fin_grid = (int)std::min<int64_t>(1024, (end - begin + 255) / 256 + 1);
  k_amax_init<<<fin_grid, 256, 0, s>>>(reinterpret_cast<uint32_t*>(out), begin, end, a.Hd, a.kv1, a.c0, a.hq0,
                                       a.nhq);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (a.n_items && a.rows) {
    AmaxArgs b = a;
    b.f_tgc = make_fastdiv((a.f_tg.d + kAmaxG - 1) / kAmaxG);
    b.n_row_items = b.f_tgc.d * (uint32_t)a.nhq * (a.kv1 ? 1u : 2u) * (uint32_t)a.Lc;
    switch (sdt) {
      case KV_F16: k_amax_rows<KV_F16><<<grid_for_items(k_amax_rows<KV_F16>, b.n_row_items), kThreads, 0, s>>>(b); break;
      case KV_BF16: k_amax_rows<KV_BF16><<<grid_for_items(k_amax_rows<KV_BF16>, b.n_row_items), kThreads, 0, s>>>(b); break;
      case KV_F8E4M3:
        k_amax_rows<KV_F8E4M3><<<grid_for_items(k_amax_rows<KV_F8E4M3>, b.n_row_items), kThreads, 0, s>>>(b);
        break;
      case KV_F8E4M3FNUZ:
        k_amax_rows<KV_F8E4M3FNUZ><<<grid_for_items(k_amax_rows<KV_F8E4M3FNUZ>, b.n_row_items), kThreads, 0, s>>>(b);
        break;
      case KV_F32: k_amax_rows<KV_F32><<<grid_for_items(k_amax_rows<KV_F32>, b.n_row_items), kThreads, 0, s>>>(b); break;
      default: return cudaErrorInvalidValue;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
  } else if (a.n_items) {
    switch (sdt) {
      case KV_F16: k_amax<KV_F16><<<grid_for_items(k_amax<KV_F16>, a.n_items), kThreads, 0, s>>>(a); break;
      case KV_BF16: k_amax<KV_BF16><<<grid_for_items(k_amax<KV_BF16>, a.n_items), kThreads, 0, s>>>(a); break;
      case KV_F8E4M3: k_amax<KV_F8E4M3><<<grid_for_items(k_amax<KV_F8E4M3>, a.n_items), kThreads, 0, s>>>(a); break;
      case KV_F8E4M3FNUZ:
        k_amax<KV_F8E4M3FNUZ><<<grid_for_items(k_amax<KV_F8E4M3FNUZ>, a.n_items), kThreads, 0, s>>>(a);
        break;
      case KV_F32: k_amax<KV_F32><<<grid_for_items(k_amax<KV_F32>, a.n_items), kThreads, 0, s>>>(a); break;
      default: return cudaErrorInvalidValue;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  k_amax_finalize<<<fin_grid, 256, 0, s>>>(reinterpret_cast<uint32_t*>(out), begin, end, a.qmax, a.Hd, a.kv1,
                                           a.c0, a.hq0, a.nhq, a.peer);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// Opaque byte copy (hidden state): 16-B vectors when both ends are 16-B aligned, bytes
// otherwise; a few KiB per request, one small grid.
__global__ void k_copy_bytes(uint8_t* dst, const uint8_t* src, size_t n) {
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
  if ((((uintptr_t)dst | (uintptr_t)src) & 15u) == 0) {
    const size_t nv = n / 16;
    for (size_t i = tid; i < nv; i += nth) reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    for (size_t i = nv * 16 + tid; i < n; i += nth) dst[i] = src[i];
  } else {
    for (size_t i = tid; i < n; i += nth) dst[i] = src[i];
  }
}

cudaError_t launch_copy_bytes(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  const int blocks = (int)std::min<size_t>(256, (bytes / 16 + 255) / 256 + 1);
  k_copy_bytes<<<blocks, 256, 0, s>>>(static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), bytes);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// per-request completion words (kv_convert_reshard_notify)
__global__ void k_notify_init(Notify n, const int32_t* blk_off, int32_t n_req) {
  const uint64_t now = gtimer_ns();
  for (int32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_req; r += gridDim.x * blockDim.x) {
    n.counters[r] = 0u;
    if (blk_off[r + 1] == blk_off[r]) {   // no block: nothing to wait for
      if (n.ns) n.ns[r] = now;
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(n.flags + r), "r"(n.epoch) : "memory");
    }
  }
}
__global__ void k_notify_all(Notify n, int32_t n_req) {
  __threadfence_system();
  const uint64_t now = gtimer_ns();
  for (int32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_req; r += gridDim.x * blockDim.x) {
    if (n.ns) n.ns[r] = now;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(n.flags + r), "r"(n.epoch) : "memory");
  }
}
__global__ void k_timestamp(uint64_t* out) { *out = gtimer_ns(); }

cudaError_t launch_notify_init(const Notify& n, const int32_t* blk_off, int32_t n_req, cudaStream_t s) {
  if (n_req <= 0) return cudaSuccess;
  k_notify_init<<<(n_req + 255) / 256, 256, 0, s>>>(n, blk_off, n_req);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}
cudaError_t launch_notify_all(const Notify& n, int32_t n_req, cudaStream_t s) {
  if (n_req <= 0) return cudaSuccess;
  k_notify_all<<<(n_req + 255) / 256, 256, 0, s>>>(n, n_req);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}
cudaError_t launch_timestamp(uint64_t* out, cudaStream_t s) {
  k_timestamp<<<1, 1, 0, s>>>(out);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_signal(uint32_t* flag, uint32_t value, cudaStream_t s) {
  k_signal<<<1, 1, 0, s>>>(flag, value);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}
cudaError_t launch_wait(const uint32_t* flag, uint32_t value, uint64_t timeout_ns, int32_t* err, cudaStream_t s) {
  k_wait<<<1, 32, 0, s>>>(flag, value, timeout_ns, err);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// Eager loading of every kernel (kv_preload).  Under CUDA lazy loading (the CUDA 12
// default) a kernel is loaded at its first launch, and loading may wait for the kernels
// already running in the context.  A spin-waiting kernel (k_wait, the persistent
// k_pull_rows) whose release depends on a kernel launched for the first time afterwards in
// the same process would then only end by its timeout (P and D on one GPU).  Asking for a
// kernel's attributes loads it, so this walks every instantiation the launchers use.
// ------------------------------------------------------------------------------------
namespace {
template <typename K>
cudaError_t touch(K k) {
  cudaFuncAttributes at;
  return cudaFuncGetAttributes(&at, reinterpret_cast<const void*>(k));
}
#define KVX_TOUCH(...)                         \
  do {                                         \
    cudaError_t e_ = touch(__VA_ARGS__);       \
    if (e_ != cudaSuccess) return e_;          \
  } while (0)

template <int SDT, int DDT>
cudaError_t preload_tb() {
  if constexpr (Tr<SDT>::B <= 2) KVX_TOUCH(k_convert_tb<SDT, DDT, 1>);
  if constexpr (Tr<SDT>::B <= 2) KVX_TOUCH(k_convert_tb<SDT, DDT, 2>);
  if constexpr (Tr<SDT>::B <= 2) KVX_TOUCH(k_tile_cast<SDT, DDT>);
  return cudaSuccess;
}
template <int SDT, int DDT>
cudaError_t preload_pair() {
  constexpr int U8 = unroll_for<SDT, 8>(), U1 = unroll_for<SDT, 1>();
  KVX_TOUCH(k_convert_rows<SDT, DDT, U8>);
  KVX_TOUCH(k_convert_rows<SDT, DDT, U8, 8, true>);
  if constexpr (Tr<SDT>::B == 1 && Tr<DDT>::B <= 2) KVX_TOUCH(k_convert_rows<SDT, DDT, 4, 16>);
  KVX_TOUCH(k_convert<1, SDT, DDT, U1>);
  KVX_TOUCH(k_convert_tr<SDT, DDT>);
  KVX_TOUCH(k_convert_tr8<SDT, DDT, false>);
  if constexpr (Tr<SDT>::B == 2 && Tr<DDT>::B == 2) KVX_TOUCH(k_convert_tr8<SDT, DDT, true>);
  KVX_TOUCH(k_pack_rows<SDT, DDT, U8>);
  if constexpr (Tr<SDT>::B >= 2 && DDT != KV_F32) KVX_TOUCH(k_stage_rows<SDT, DDT, U8>);
  KVX_TOUCH(k_pack<1, SDT, DDT, U1>);
  KVX_TOUCH(k_unpack_rows<SDT, DDT, U8>);
  KVX_TOUCH(k_unpack<1, SDT, DDT, U1>);
  return preload_tb<SDT, DDT>();
}
template <int SDT>
cudaError_t preload_src() {
  cudaError_t e;
  if ((e = preload_pair<SDT, KV_F16>()) != cudaSuccess) return e;
  if ((e = preload_pair<SDT, KV_BF16>()) != cudaSuccess) return e;
  if ((e = preload_pair<SDT, KV_F8E4M3>()) != cudaSuccess) return e;
  if ((e = preload_pair<SDT, KV_F8E4M3FNUZ>()) != cudaSuccess) return e;
  if ((e = preload_pair<SDT, KV_F32>()) != cudaSuccess) return e;
  KVX_TOUCH(k_pull_rows<SDT, unroll_for<SDT, 8>()>);
  KVX_TOUCH(k_amax<SDT>);
  KVX_TOUCH(k_amax_rows<SDT>);
  return cudaSuccess;
}
}  // namespace

cudaError_t preload_kernels() {
  cudaError_t e;
  if ((e = preload_src<KV_F16>()) != cudaSuccess) return e;
  if ((e = preload_src<KV_BF16>()) != cudaSuccess) return e;
  if ((e = preload_src<KV_F8E4M3>()) != cudaSuccess) return e;
  if ((e = preload_src<KV_F8E4M3FNUZ>()) != cudaSuccess) return e;
  if ((e = preload_src<KV_F32>()) != cudaSuccess) return e;
  KVX_TOUCH(k_tile_copy);
  KVX_TOUCH((k_requant_rows<KV_F8E4M3FNUZ, KV_F8E4M3, 4, 4>));
  KVX_TOUCH((k_requant_rows<KV_F8E4M3, KV_F8E4M3FNUZ, 4, 4>));
  KVX_TOUCH(k_amax_init);
  KVX_TOUCH(k_amax_finalize);
  KVX_TOUCH(k_signal);
  KVX_TOUCH(k_wait);
  KVX_TOUCH(k_copy_bytes);
  KVX_TOUCH(k_notify_init);
  KVX_TOUCH(k_notify_all);
  KVX_TOUCH(k_timestamp);
  return preload_verify_kernels();
}

}  // namespace kvx
