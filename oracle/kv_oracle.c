/*
 * kv_oracle.c -- O1, the plain CPU oracle for the heterogeneous-compatible KV
 * transmission path of arXiv 2509.17542 ("Disaggregated Prefill and Decoding
 * Inference System for LLM Serving on Multi-Vendor GPUs").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_2509_17542_b200/) never imports, links or executes it,
 * and this file shares no header, helper, table or constant with the CUDA
 * path (it does not include include/kvx.h; its layout struct is its own).
 *
 * What it computes is the plain definition of SURVEY.md 8(c):
 *   for each request r, decode rank q, layer l, K/V c, decode-local head hq,
 *   token t < T_r, dim d:
 *     h  = q*H_d + hq ;  p = h / H_p ;  hp = h - p*H_p       (TP merge/split)
 *     x  = SRC[p][off(L_p; l, c, BT_p[r][t / B_p], t % B_p, hp, d)]
 *     DST[q][off(L_d; l, c, BT_d[r][t / B_d], t % B_d, hq, d)] = cast(x)
 *   tail slots t in [T_r, ceil(T_r/B_d)*B_d) of the last D block are zeroed.
 *   Every other destination byte keeps its prior value.
 *
 * Passages followed (PAPER.md line, section):
 *   P:113 (III-B2, VRAM management alignment): block size of page attention and
 *         tensor layout are converted "according to the demand of D instance";
 *         flatten to 1-D before transmission, restore after (Fig. 5).
 *   P:125 (III-B3, parallel strategy alignment, Fig. 4): TP=4 -> TP=2 combines
 *         P TP1+TP2 -> D TP1 and TP3+TP4 -> D TP2; TP=2 -> TP=4 splits.
 *   P:65  (I, contributions): a "precision alignment component" exists; its
 *         semantics are the readings in DESIGN.md (RNE; fp8-e4m3 satfinite with
 *         a per-(layer, K/V, head) scale applied as x * RN(1/s)).
 *   SPEC.md S:41  KV size formula 2*L*H_kv*D*T*bytes; S:255/S:280 zero-filled
 *         tail; S:279 head-contiguous TP sharding; S:281 RNE narrowing.
 *
 * Pins (tests/test_oracle_*.py, all -m "not gpu"): closed-form KV bytes
 * (S:60-61), exhaustive cast tables against torch / ml_dtypes / numpy,
 * NVIDIA satfinite edge vectors, power-of-two-scale fp8 special case,
 * brute-force O2 (oracle/bruteforce.py, source-driven, nearest-code casts)
 * on tiny shapes, numpy-transpose special case, worked examples of P:125 and
 * S:259-260, round trips, canaries.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -shared -fPIC.
 * -ffp-contract=off matters: x * inv must not fuse into anything.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Physical axes of a pool (SURVEY 8 notation): extents (L, 2, N_blocks, B, H_local, D). */
enum { OAX_LAYER = 0, OAX_KV = 1, OAX_BLOCK = 2, OAX_SLOT = 3, OAX_HEAD = 4, OAX_DIM = 5 };
/* Element types. */
/* ODT_E4M3FNUZ (NEXT-3, another vendor's fp8; reading 24): bias 8, max 240,
 * no infinities, no negative zero, the single NaN 0x80. */
enum { ODT_F16 = 0, ODT_BF16 = 1, ODT_E4M3 = 2, ODT_F32 = 3, ODT_E4M3FNUZ = 4 };

static int is_fp8(int32_t dt) { return dt == ODT_E4M3 || dt == ODT_E4M3FNUZ; }

typedef struct {
  int32_t num_layers;  /* layers held by this pool */
  int32_t first_layer; /* global index of its first layer (pipeline stage; 0 otherwise) */
  int32_t num_kv_heads, head_dim;
  int32_t tp_degree, tp_rank;
  int32_t block_size, num_blocks;
  int32_t dtype;
  int32_t axis_order[6]; /* outermost -> innermost, dense row-major */
  int32_t kv_part;       /* 0: the pool holds K and V; 1: K only; 2: V only (KV extent 1) */
  int32_t dim_split;     /* x > 1: head_dim stored as (D/x at DIM's place, x innermost) */
  const float* scales;   /* host [L][2][H_local] fp32 dequant scales (fp8 only) */
} okv_layout;

/* NEXT-3 layout variants (reading 27): a pool may hold only K or only V (engines
 * that keep separate K and V tensors, with different axis orders), and head_dim may be split
 * into (D/x, ..., x) with the x part innermost -- the "x-packed" key cache of the paged-
 * attention kernels other vendors' engines use, K [blocks, heads, D/x, block, x]. */
static int holds(const okv_layout* L, int32_t c) { return L->kv_part == 0 || L->kv_part == c + 1; }
static int64_t split_of(const okv_layout* L) { return L->dim_split > 1 ? L->dim_split : 1; }

/* ------------------------------------------------------------------------ */
/* Sizes                                                                    */
/* ------------------------------------------------------------------------ */

int32_t okv_dtype_bytes(int32_t dt) {
  switch (dt) {
    case ODT_F16: return 2;
    case ODT_BF16: return 2;
    case ODT_E4M3: return 1;
    case ODT_F32: return 4;
    case ODT_E4M3FNUZ: return 1;
  }
  return 0;
}

/* KV size formula: 2 * layers * kv_heads * head_dim * tokens * bytes. */
int64_t okv_kv_bytes(int64_t layers, int64_t kv_heads, int64_t head_dim, int64_t tokens,
                     int64_t dtype_bytes) {
  return 2 * layers * kv_heads * head_dim * tokens * dtype_bytes;
}

/* ------------------------------------------------------------------------ */
/* Layout: dense row-major offsets in axis_order (SURVEY 8(c) off()).       */
/* ------------------------------------------------------------------------ */

static int64_t extent_of(const okv_layout* L, int axis) {
  switch (axis) {
    case OAX_LAYER: return L->num_layers;
    case OAX_KV: return L->kv_part ? 1 : 2;
    case OAX_BLOCK: return L->num_blocks;
    case OAX_SLOT: return L->block_size;
    case OAX_HEAD: return L->num_kv_heads / L->tp_degree;
    case OAX_DIM: return L->head_dim / split_of(L);
  }
  return 0;
}

/* Element offset of (l, c, block, slot, local head, d): sum over axes of
 * index * stride, strides row-major over axis_order (then the x part of a split head_dim,
 * innermost).  c is the global K/V index; a K-only or V-only pool stores it at 0. */
int64_t okv_offset(const okv_layout* L, int64_t l, int64_t c, int64_t blk, int64_t slot,
                   int64_t hl, int64_t d) {
  int64_t idx[6];
  idx[OAX_LAYER] = l;
  idx[OAX_KV] = L->kv_part ? 0 : c;
  idx[OAX_BLOCK] = blk;
  idx[OAX_SLOT] = slot;
  idx[OAX_HEAD] = hl;
  idx[OAX_DIM] = d / split_of(L);
  int64_t off = 0;
  for (int i = 0; i < 6; ++i) {
    int a = L->axis_order[i];
    off = off * extent_of(L, a) + idx[a];
  }
  return off * split_of(L) + d % split_of(L);
}

int64_t okv_pool_elems(const okv_layout* L) {
  int64_t n = split_of(L);
  for (int a = 0; a < 6; ++a) n *= extent_of(L, a);
  return n;
}

/* ------------------------------------------------------------------------ */
/* Precision alignment (readings in DESIGN.md).                       */
/*                                                                          */
/* Every narrowing is "round the exact real value to the nearest            */
/* representable value of the target format, ties to the even significand"  */
/* (IEEE 754 roundTiesToEven), with overflow to +-Inf for fp16/bf16 and      */
/* saturation to +-448 for e4m3fn (satfinite).  The exact value of a 2-byte  */
/* or fp32 input is held in a double (exact: <= 24 significant bits).        */
/* ------------------------------------------------------------------------ */

typedef struct {
  int p;          /* significant bits including the implicit one */
  int emin;       /* exponent of the smallest normal */
  int bias;
  int exp_bits;
  double maxfin;  /* largest finite magnitude */
} ofmt;

static const ofmt FMT_F16 = {11, -14, 15, 5, 65504.0};
static const ofmt FMT_BF16 = {8, -126, 127, 8, 3.3895313892515355e38};
static const ofmt FMT_E4M3 = {4, -6, 7, 4, 448.0};
static const ofmt FMT_F32 = {24, -126, 127, 8, 3.4028234663852886e38};
static const ofmt FMT_FNUZ = {4, -7, 8, 4, 240.0};

/* Decode an encoding to its exact value (NaN -> NAN, Inf -> INFINITY).
 * kind 0: IEEE (all-ones exponent = Inf / NaN).
 * kind 1: e4m3fn (OCP FP8): no infinities; S.1111.111 is NaN; all other codes finite.
 * kind 2: e4m3fnuz: no infinities; 0x80 ("negative zero") is the only NaN. */
static double decode_bits(uint32_t bits, const ofmt* f, int kind) {
  const int is_e4m3 = kind == 1;
  if (kind == 2 && bits == 0x80u) return NAN;
  int mbits = f->p - 1;
  uint32_t sign = (bits >> (f->exp_bits + mbits)) & 1u;
  uint32_t e = (bits >> mbits) & ((1u << f->exp_bits) - 1u);
  uint32_t m = bits & ((1u << mbits) - 1u);
  double v;
  uint32_t emax_field = (1u << f->exp_bits) - 1u;
  if (is_e4m3) {
    if (e == emax_field && m == ((1u << mbits) - 1u)) return NAN;
  } else if (kind == 0 && e == emax_field) {
    if (m != 0) return NAN;
    return sign ? -INFINITY : INFINITY;
  }
  if (e == 0)
    v = ldexp((double)m, f->emin - mbits); /* subnormal */
  else
    v = ldexp((double)((1u << mbits) | m), (int)e - f->bias - mbits);
  return sign ? -v : v;
}

double okv_decode(uint32_t bits, int32_t dt) {
  switch (dt) {
    case ODT_F16: return decode_bits(bits & 0xFFFFu, &FMT_F16, 0);
    case ODT_BF16: return decode_bits(bits & 0xFFFFu, &FMT_BF16, 0);
    case ODT_E4M3: return decode_bits(bits & 0xFFu, &FMT_E4M3, 1);
    case ODT_F32: return decode_bits(bits, &FMT_F32, 0);
    case ODT_E4M3FNUZ: return decode_bits(bits & 0xFFu, &FMT_FNUZ, 2);
  }
  return NAN;
}

/* Round a finite, non-NaN real x to format f, ties to even, with unbounded
 * exponent range above (overflow handled by the caller).  Returns the rounded
 * magnitude as a double (exact). */
static double rne_magnitude(double ax, const ofmt* f) {
  if (ax == 0.0) return 0.0;
  int k;
  frexp(ax, &k);               /* ax = m * 2^k, m in [0.5, 1) -> exponent e = k - 1 */
  int e = k - 1;
  if (e < f->emin) e = f->emin;  /* subnormal range: fixed quantum */
  double q = ldexp(1.0, e - (f->p - 1));
  double n = nearbyint(ax / q); /* ax/q exact (power-of-two scaling); default mode RNE */
  return n * q;
}

/* Encode an exactly representable magnitude (finite, <= maxfin) plus sign. */
static uint32_t encode_exact(double mag, uint32_t sign, const ofmt* f) {
  int mbits = f->p - 1;
  uint32_t bits;
  if (mag == 0.0) {
    bits = 0;
  } else if (mag < ldexp(1.0, f->emin)) {
    bits = (uint32_t)(mag / ldexp(1.0, f->emin - mbits)); /* subnormal, e field 0 */
  } else {
    int k;
    frexp(mag, &k);
    int e = k - 1;
    uint32_t m = (uint32_t)(mag / ldexp(1.0, e - mbits)) - (1u << mbits);
    bits = ((uint32_t)(e + f->bias) << mbits) | m;
  }
  return bits | (sign << (f->exp_bits + mbits));
}

/* Narrow/widen an exact real value to fp16 / bf16 / fp32 (IEEE RNE,
 * overflow -> +-Inf).  NaN -> canonical quiet NaN 0x7FFF (fp16 and bf16) /
 * 0x7FFFFFFF (fp32): DESIGN.md reading 12. */
static uint32_t round_ieee(double x, const ofmt* f) {
  int mbits = f->p - 1;
  uint32_t expmask = (1u << f->exp_bits) - 1u;
  if (isnan(x)) return (f == &FMT_F32) ? 0x7FFFFFFFu : 0x7FFFu;
  uint32_t sign = signbit(x) ? 1u : 0u;
  double ax = fabs(x);
  double r = isinf(x) ? INFINITY : rne_magnitude(ax, f);
  if (r > f->maxfin) return (sign << (f->exp_bits + mbits)) | (expmask << mbits);
  return encode_exact(r, sign, f);
}

/* e4m3fn with satfinite (PTX cvt.rn.satfinite.e4m3x2.f32 semantics): RNE,
 * magnitudes rounding above 448 (and +-Inf) saturate to +-448, NaN -> 0x7F. */
static uint32_t round_e4m3_satfinite(double x) {
  if (isnan(x)) return 0x7Fu;
  uint32_t sign = signbit(x) ? 1u : 0u;
  double ax = fabs(x);
  double r = isinf(x) ? INFINITY : rne_magnitude(ax, &FMT_E4M3);
  if (r > FMT_E4M3.maxfin) r = FMT_E4M3.maxfin;
  return encode_exact(r, sign, &FMT_E4M3);
}

/* e4m3fnuz with satfinite (reading 25): RNE on the fnuz grid (bias 8, quantum 2^-10 below
 * 2^-7), magnitudes rounding above 240 (and +-Inf) saturate to +-240, NaN -> 0x80, and a
 * result of zero is +0 (0x00) whatever the sign -- the format has no negative zero. */
static uint32_t round_fnuz_satfinite(double x) {
  if (isnan(x)) return 0x80u;
  uint32_t sign = signbit(x) ? 1u : 0u;
  double ax = fabs(x);
  double r = isinf(x) ? INFINITY : rne_magnitude(ax, &FMT_FNUZ);
  if (r > FMT_FNUZ.maxfin) r = FMT_FNUZ.maxfin;
  if (r == 0.0) return 0u;
  return encode_exact(r, sign, &FMT_FNUZ);
}

uint16_t okv_f16_to_bf16(uint16_t x) { return (uint16_t)round_ieee(okv_decode(x, ODT_F16), &FMT_BF16); }
uint16_t okv_bf16_to_f16(uint16_t x) { return (uint16_t)round_ieee(okv_decode(x, ODT_BF16), &FMT_F16); }
uint16_t okv_f32_to_f16(uint32_t x) { return (uint16_t)round_ieee(okv_decode(x, ODT_F32), &FMT_F16); }
uint16_t okv_f32_to_bf16(uint32_t x) { return (uint16_t)round_ieee(okv_decode(x, ODT_F32), &FMT_BF16); }
uint32_t okv_2byte_to_f32(uint16_t x, int32_t dt) { return round_ieee(okv_decode(x, dt), &FMT_F32); }

/* e4m3fn of an fp32 value (already scaled). */
uint8_t okv_f32_to_e4m3(float v) { return (uint8_t)round_e4m3_satfinite((double)v); }

/* Quantise one element to e4m3 with dequant scale s (reading 10):
 *   inv = RN_f32(1 / s) ; v = RN_f32(f32(x) * inv) ; q = satfinite_RNE_e4m3(v).
 * float arithmetic below is IEEE binary32 (x86-64 SSE, -ffp-contract=off). */
uint8_t okv_to_e4m3_scaled(uint32_t bits, int32_t src_dt, float scale) {
  float xf = (float)okv_decode(bits, src_dt); /* exact: <= 24 significant bits */
  float inv = 1.0f / scale;
  float v = xf * inv;
  return okv_f32_to_e4m3(v);
}

/* Dequantise an fp8 code (e4m3fn or e4m3fnuz) with scale s into fp32:
 * RN_f32(f32(q) * s) (NEXT-1 widening, reading 20). */
static float fp8_dequant(uint32_t q, int32_t dt, float scale) {
  float qf = (float)okv_decode(q, dt);
  return qf * scale;
}

/* cast(x) from src dtype to dst dtype.  src_scale applies when src is fp8 (e4m3fn or
 * e4m3fnuz), dst_scale when dst is fp8.  Same dtype: bits unchanged.  fp8 -> the
 * other fp8 format: dequantise with src_scale, quantise with dst_scale (reading 26). */
uint32_t okv_cast(uint32_t bits, int32_t src_dt, int32_t dst_dt, float src_scale, float dst_scale) {
  if (src_dt == dst_dt) return bits;
  double x;
  if (is_fp8(src_dt)) {
    x = (double)fp8_dequant(bits, src_dt, src_scale);
  } else {
    x = okv_decode(bits, src_dt);
  }
  switch (dst_dt) {
    case ODT_F16: return round_ieee(x, &FMT_F16);
    case ODT_BF16: return round_ieee(x, &FMT_BF16);
    case ODT_F32: return round_ieee(x, &FMT_F32);
    case ODT_E4M3:
    case ODT_E4M3FNUZ: {
      float xf = (float)x; /* exact: x is an f32 value or a <= 24-bit significand */
      float inv = 1.0f / dst_scale;
      float v = xf * inv;
      return dst_dt == ODT_E4M3 ? round_e4m3_satfinite((double)v) : round_fnuz_satfinite((double)v);
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Element access                                                           */
/* ------------------------------------------------------------------------ */

static uint32_t load_elem(const void* pool, int64_t off, int32_t dt) {
  switch (okv_dtype_bytes(dt)) {
    case 1: return ((const uint8_t*)pool)[off];
    case 2: return ((const uint16_t*)pool)[off];
    case 4: return ((const uint32_t*)pool)[off];
  }
  return 0;
}

static void store_elem(void* pool, int64_t off, int32_t dt, uint32_t v) {
  switch (okv_dtype_bytes(dt)) {
    case 1: ((uint8_t*)pool)[off] = (uint8_t)v; break;
    case 2: ((uint16_t*)pool)[off] = (uint16_t)v; break;
    case 4: ((uint32_t*)pool)[off] = v; break;
  }
}

static float scale_of(const okv_layout* L, int64_t l, int64_t c, int64_t hl) {
  int64_t hloc = L->num_kv_heads / L->tp_degree;
  return L->scales ? L->scales[(l * 2 + c) * hloc + hl] : 1.0f;
}

/* ------------------------------------------------------------------------ */
/* A2: TP re-shard plan (Fig. 4).                         */
/* Pair (p, q) with head overlap [max(p*H_p, q*H_d), min((p+1)*H_p, (q+1)*H_d)). */
/* Writes up to max_pairs entries of (p, q, h_begin, h_end); returns count,  */
/* or -1 if a degree does not divide H.                              */
/* ------------------------------------------------------------------------ */
int32_t okv_plan(int32_t tp_p, int32_t tp_d, int32_t H, int32_t* out, int32_t max_pairs) {
  if (tp_p <= 0 || tp_d <= 0 || H % tp_p != 0 || H % tp_d != 0) return -1;
  int32_t Hp = H / tp_p, Hd = H / tp_d, n = 0;
  for (int32_t q = 0; q < tp_d; ++q)
    for (int32_t p = 0; p < tp_p; ++p) {
      int32_t b = p * Hp > q * Hd ? p * Hp : q * Hd;
      int32_t e = (p + 1) * Hp < (q + 1) * Hd ? (p + 1) * Hp : (q + 1) * Hd;
      if (b < e) {
        if (n < max_pairs) {
          out[4 * n + 0] = p;
          out[4 * n + 1] = q;
          out[4 * n + 2] = b;
          out[4 * n + 3] = e;
        }
        ++n;
      }
    }
  return n;
}

/* ------------------------------------------------------------------------ */
/* The conversion, P -> D, all requests, layers [lb, le).     */
/* src/dst are arrays of layouts of the ranks present; a missing source      */
/* rank needed by a present destination rank is an error.            */
/* Block tables are CSR: request r's blocks are ids[off[r] .. off[r+1]).     */
/* Returns 0 on success, negative on error.                                  */
/* ------------------------------------------------------------------------ */
int32_t okv_convert(int32_t n_src, const okv_layout* src, void* const* src_pools,
                    int32_t n_dst, const okv_layout* dst, void* const* dst_pools,
                    int32_t n_req, const int32_t* n_tokens,
                    const int32_t* src_bt_off, const int32_t* src_bt_ids,
                    const int32_t* dst_bt_off, const int32_t* dst_bt_ids,
                    int32_t layer_begin, int32_t layer_end) {
  if (n_src <= 0 || n_dst <= 0) return -1;
  int32_t H = src[0].num_kv_heads, D = src[0].head_dim;
  int32_t Hp = H / src[0].tp_degree;
  int32_t Bp = src[0].block_size;
  for (int32_t i = 0; i < n_src; ++i)
    if (layer_begin < src[i].first_layer || layer_end > src[i].first_layer + src[i].num_layers) return -1;
  for (int32_t i = 0; i < n_dst; ++i)
    if (layer_begin < dst[i].first_layer || layer_end > dst[i].first_layer + dst[i].num_layers) return -1;
  for (int32_t r = 0; r < n_req; ++r) {
    int64_t T = n_tokens[r];
    for (int32_t qi = 0; qi < n_dst; ++qi) {
      const okv_layout* Ld = &dst[qi];
      int32_t q = Ld->tp_rank;
      int32_t Hd = H / Ld->tp_degree;
      int32_t Bd = Ld->block_size;
      int64_t padded = (T + Bd - 1) / Bd * Bd;
      for (int32_t l = layer_begin; l < layer_end; ++l)
        for (int32_t c = 0; c < 2; ++c)
          for (int32_t hq = 0; hq < Hd; ++hq) {
            int32_t h = q * Hd + hq;
            int32_t p = h / Hp;
            int32_t hp = h - p * Hp;
            int32_t pi = -1;
            for (int32_t i = 0; i < n_src; ++i)
              if (src[i].tp_rank == p) pi = i;
            if (pi < 0) return -2 - p; /* missing source shard p */
            const okv_layout* Lp = &src[pi];
            if (!holds(Lp, c) || !holds(Ld, c)) continue; /* K/V the two pools share only */
            int32_t ls = l - Lp->first_layer, ld = l - Ld->first_layer; /* pool-local layers */
            float sd = scale_of(Ld, ld, c, hq);
            float ss = scale_of(Lp, ls, c, hp);
            for (int64_t t = 0; t < T; ++t) {
              int32_t sb = src_bt_ids[src_bt_off[r] + t / Bp];
              int32_t db = dst_bt_ids[dst_bt_off[r] + t / Bd];
              for (int32_t d = 0; d < D; ++d) {
                uint32_t x = load_elem(src_pools[pi], okv_offset(Lp, ls, c, sb, t % Bp, hp, d), Lp->dtype);
                uint32_t y = okv_cast(x, Lp->dtype, Ld->dtype, ss, sd);
                store_elem(dst_pools[qi], okv_offset(Ld, ld, c, db, t % Bd, hq, d), Ld->dtype, y);
              }
            }
            for (int64_t t = T; t < padded; ++t) {
              int32_t db = dst_bt_ids[dst_bt_off[r] + t / Bd];
              for (int32_t d = 0; d < D; ++d)
                store_elem(dst_pools[qi], okv_offset(Ld, ld, c, db, t % Bd, hq, d), Ld->dtype, 0u);
            }
          }
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Fig. 5 flatten: the pair (p -> q) wire buffer in canonical order  */
/* (layer, kv, head in overlap, token, dim), tokens of all requests          */
/* concatenated in batch order.  The wire dtype is the narrower of the two   */
/* (cast on the sender when narrowing); wire_dt is passed in.     */
/* Returns the number of elements written, or negative on error.            */
/* ------------------------------------------------------------------------ */
int64_t okv_flatten(const okv_layout* Lp, const void* src_pool, const okv_layout* Ld,
                    int32_t wire_dt, int32_t n_req, const int32_t* n_tokens,
                    const int32_t* src_bt_off, const int32_t* src_bt_ids,
                    int32_t layer_begin, int32_t layer_end, void* wire) {
  int32_t H = Lp->num_kv_heads, D = Lp->head_dim;
  int32_t Hp = H / Lp->tp_degree, Hd = H / Ld->tp_degree;
  int32_t p = Lp->tp_rank, q = Ld->tp_rank;
  int32_t hb = p * Hp > q * Hd ? p * Hp : q * Hd;
  int32_t he = (p + 1) * Hp < (q + 1) * Hd ? (p + 1) * Hp : (q + 1) * Hd;
  int32_t Bp = Lp->block_size;
  int64_t w = 0;
  for (int32_t l = layer_begin; l < layer_end; ++l)
    for (int32_t c = 0; c < 2; ++c)
      if (holds(Lp, c) && holds(Ld, c)) /* the wire carries the K/V both pools hold */
      for (int32_t h = hb; h < he; ++h)
        for (int32_t r = 0; r < n_req; ++r)
          for (int64_t t = 0; t < n_tokens[r]; ++t) {
            int32_t sb = src_bt_ids[src_bt_off[r] + t / Bp];
            for (int32_t d = 0; d < D; ++d) {
              int32_t ls = l - Lp->first_layer, ld = l - Ld->first_layer;
              uint32_t x = load_elem(src_pool, okv_offset(Lp, ls, c, sb, t % Bp, h - p * Hp, d), Lp->dtype);
              uint32_t y = okv_cast(x, Lp->dtype, wire_dt, scale_of(Lp, ls, c, h - p * Hp),
                                    scale_of(Ld, ld, c, h - q * Hd));
              store_elem(wire, w++, wire_dt, y);
            }
          }
  return w;
}

/* Fig. 5 restore: wire (canonical order, wire_dt) -> D pool of rank q,
 * heads of the overlap with source rank p, with tail zero-fill for those heads. */
int64_t okv_restore(const okv_layout* Lp, const okv_layout* Ld, void* dst_pool, int32_t wire_dt,
                    const void* wire, int32_t n_req, const int32_t* n_tokens,
                    const int32_t* dst_bt_off, const int32_t* dst_bt_ids,
                    int32_t layer_begin, int32_t layer_end) {
  int32_t H = Lp->num_kv_heads, D = Lp->head_dim;
  int32_t Hp = H / Lp->tp_degree, Hd = H / Ld->tp_degree;
  int32_t p = Lp->tp_rank, q = Ld->tp_rank;
  int32_t hb = p * Hp > q * Hd ? p * Hp : q * Hd;
  int32_t he = (p + 1) * Hp < (q + 1) * Hd ? (p + 1) * Hp : (q + 1) * Hd;
  int32_t Bd = Ld->block_size;
  int64_t w = 0;
  for (int32_t l = layer_begin; l < layer_end; ++l)
    for (int32_t c = 0; c < 2; ++c)
      if (holds(Lp, c) && holds(Ld, c))
      for (int32_t h = hb; h < he; ++h)
        for (int32_t r = 0; r < n_req; ++r) {
          int64_t T = n_tokens[r];
          int64_t padded = (T + Bd - 1) / Bd * Bd;
          for (int64_t t = 0; t < padded; ++t) {
            int32_t db = dst_bt_ids[dst_bt_off[r] + t / Bd];
            int32_t ls = l - Lp->first_layer, ld = l - Ld->first_layer;
            for (int32_t d = 0; d < D; ++d) {
              uint32_t y = 0;
              if (t < T) {
                uint32_t x = load_elem(wire, w++, wire_dt);
                y = okv_cast(x, wire_dt, Ld->dtype, scale_of(Lp, ls, c, h - p * Hp),
                             scale_of(Ld, ld, c, h - q * Hd));
              }
              store_elem(dst_pool, okv_offset(Ld, ld, c, db, t % Bd, h - q * Hd, d), Ld->dtype, y);
            }
          }
        }
  return w;
}

/* Batch form of okv_cast over n codes (test convenience; same arithmetic). */
void okv_cast_array(int64_t n, const void* in, int32_t src_dt, int32_t dst_dt, float src_scale,
                    float dst_scale, void* out) {
  for (int64_t i = 0; i < n; ++i)
    store_elem(out, i, dst_dt, okv_cast(load_elem(in, i, src_dt), src_dt, dst_dt, src_scale, dst_scale));
}

/* NEXT-1 dynamic scales (precision alignment; reading 21):
 * s[l][c][hq] = RN_f32(amax / M) with M the destination fp8's largest finite value (448
 * e4m3fn, 240 e4m3fnuz) and amax = max |x| (x as f32, fp8 sources dequantised
 * with their own scale) over every finite source element of the valid tokens of all
 * requests for the heads of D rank dst; s = 1 if amax is 0.  Layers [lb, le) are written
 * into out[L][2][H_d] for the K/V both layouts hold; other entries untouched.  Returns 0,
 * or <0 if a shard is missing. */
int32_t okv_amax_scales(int32_t n_src, const okv_layout* src, void* const* src_pools, const okv_layout* dst,
                        int32_t n_req, const int32_t* n_tokens, const int32_t* src_bt_off,
                        const int32_t* src_bt_ids, int32_t layer_begin, int32_t layer_end, float* out) {
  int32_t H = src[0].num_kv_heads, D = src[0].head_dim;
  int32_t Hp = H / src[0].tp_degree, Hd = H / dst->tp_degree, q = dst->tp_rank;
  int32_t Bp = src[0].block_size;
  for (int32_t l = layer_begin; l < layer_end; ++l)
    for (int32_t c = 0; c < 2; ++c)
      for (int32_t hq = 0; hq < Hd; ++hq) {
        int32_t h = q * Hd + hq, p = h / Hp, hp = h - p * Hp, pi = -1;
        for (int32_t i = 0; i < n_src; ++i)
          if (src[i].tp_rank == p) pi = i;
        if (pi < 0) return -2 - p;
        const okv_layout* Lp = &src[pi];
        if (!holds(Lp, c) || !holds(dst, c)) continue; /* entries of K/V not shared: untouched */
        float amax = 0.0f;
        for (int32_t r = 0; r < n_req; ++r)
          for (int64_t t = 0; t < n_tokens[r]; ++t) {
            int32_t sb = src_bt_ids[src_bt_off[r] + t / Bp];
            for (int32_t d = 0; d < D; ++d) {
              uint32_t x = load_elem(src_pools[pi], okv_offset(Lp, l - Lp->first_layer, c, sb, t % Bp, hp, d),
                                     Lp->dtype);
              float v = is_fp8(Lp->dtype) ? fp8_dequant(x, Lp->dtype, scale_of(Lp, l - Lp->first_layer, c, hp))
                                          : (float)okv_decode(x, Lp->dtype);
              v = fabsf(v);
              if (isfinite(v) && v > amax) amax = v;
            }
          }
        float s = amax / (dst->dtype == ODT_E4M3FNUZ ? 240.0f : 448.0f);
        out[((l - dst->first_layer) * 2 + c) * Hd + hq] = s > 0.0f ? s : 1.0f;
      }
  return 0;
}
