// K6: full-size conservation check (SURVEY 8(d) "full size via the on-device
// coordinate-hash verify K6"; every valid element lands exactly once, tail slots
// are zero, nothing else in the D pool changes).  Diagnostics, not on the data path.
//
//   kv_verify_fill   writes into every VALID element of a P rank's pool (token t < T_r of each
//                    request) a value drawn from a counter-based hash of its logical
//                    coordinates (request id, token, layer, K/V, global head, dim) and a seed,
//                    chosen so the cast to D's dtype is exact (no rounding decision involved);
//   kv_verify_check  recomputes, for EVERY element of a D rank's pool, what must be there --
//                    the hashed value's D code for valid tokens, zero for the tail slots of
//                    each request's last block, the canary byte in every block the batch does
//                    not use -- and counts the differences.
// Both kernels are element-wise with their own index math (strides recomputed here from the
// axis order and extents); they share no code with the convert kernels.
#include <cuda_fp16.h>
#include <string.h>

#include <algorithm>
#include <string>

#include "kvx_internal.h"

using namespace kvx;

namespace {

constexpr int kVThreads = 256;

struct VLay {        // one pool, K6's own view
  int64_t st[6];     // element strides per kv_axis
  int64_t ext[6];    // extents per kv_axis (KV extent 2: kv_part must be 0)
  int32_t esize, dtype, Hl, rank;
};

struct VerifyArgs {
  VLay p;                        // the pool being filled / checked
  int32_t sdt, ddt;              // source and destination dtypes of the transfer
  int32_t l0;                    // pool's first global layer
  int32_t H, D, B, Lc;           // global heads, head_dim, pool block size, layers in the pool
  uint64_t seed;
  const int32_t* blk_off;        // batch tables (validated against this pool)
  const int32_t* blk_ids;
  const int32_t* blk_req;
  const int32_t* tok_off;
  const int32_t* req_ids;        // request id per batch request (NULL: the index)
  const float* dscale[KVX_MAX_RANKS];  // D scales per D rank (fp8 destination), [L][2][Hd]
  int32_t Hd, d_l0;              // D-local heads, D pools' first global layer
  uint64_t n_elem;               // table entries x L x 2 x B x Hl x D
  uint8_t* pool;
  int32_t* err;                  // fill: a value that cannot be made exact
  unsigned long long* res;       // check: [0] value, [1] tail, [2] canary mismatches, [3] checked, [4] first bad + 1
  uint8_t canary;
  uint8_t* mark;                 // check: per block, 1 if the batch uses it
  uint64_t pool_elems;
};

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// key: request (16 b) | token (20 b) | layer (8 b) | K/V (1 b) | head (9 b) | dim (10 b)
__device__ __forceinline__ uint64_t k6_hash(uint64_t seed, uint32_t r, uint32_t t, uint32_t l, uint32_t c, uint32_t h,
                                            uint32_t d) {
  const uint64_t key = ((uint64_t)(r & 0xFFFFu) << 48) | ((uint64_t)(t & 0xFFFFFu) << 28) |
                       ((uint64_t)(l & 0xFFu) << 20) | ((uint64_t)(c & 1u) << 19) | ((uint64_t)(h & 0x1FFu) << 10) |
                       (uint64_t)(d & 0x3FFu);
  return splitmix(key ^ splitmix(seed));
}

// e4m3fn / e4m3fnuz code -> exact float (codes are finite here)
__device__ __forceinline__ float fp8_value(uint32_t k, bool fnuz) {
  const uint32_t e = (k >> 3) & 0xFu, m = k & 7u;
  const int bias = fnuz ? 8 : 7;
  float v = e ? ldexpf(1.0f + (float)m / 8.0f, (int)e - bias) : ldexpf((float)m / 8.0f, 1 - bias);
  return (k & 0x80u) ? -v : v;
}

// finite random bits of a dtype from z
__device__ __forceinline__ uint32_t finite_bits(uint64_t z, int dt) {
  switch (dt) {
    case KV_F16: {
      uint32_t b = (uint32_t)z & 0xFFFFu;
      return ((b & 0x7C00u) == 0x7C00u) ? b ^ 0x0400u : b;
    }
    case KV_BF16: {
      uint32_t b = (uint32_t)z & 0xFFFFu;
      return ((b & 0x7F80u) == 0x7F80u) ? b ^ 0x0080u : b;
    }
    case KV_F32: {
      uint32_t b = (uint32_t)z;
      return ((b & 0x7F800000u) == 0x7F800000u) ? b ^ 0x00800000u : b;
    }
    case KV_F8E4M3: {
      uint32_t b = (uint32_t)z & 0xFFu;
      return ((b & 0x7Fu) == 0x7Fu) ? b ^ 1u : b;
    }
    default: {  // fnuz: 0x80 is the only NaN
      uint32_t b = (uint32_t)z & 0xFFu;
      return b == 0x80u ? 0u : b;
    }
  }
}

// a float value -> bits of a 2/4-byte dtype, exact or flagged
__device__ __forceinline__ uint32_t exact_bits(float v, int dt, bool* ok) {
  if (dt == KV_F32) return __float_as_uint(v);
  if (dt == KV_BF16) {
    const uint32_t u = __float_as_uint(v);
    if (u & 0xFFFFu) *ok = false;
    return u >> 16;
  }
  // fp16: only values of the common grid / fp8 grids reach here; check the round trip
  const __half h = __float2half_rn(v);
  if (__half2float(h) != v) *ok = false;
  return (uint32_t)__half_as_ushort(h);
}

// The (source bits, destination bits) pair of one logical element.  Same dtype: random finite
// bits.  Between 2/4-byte floats: a value both represent (sign, exponent in [-14, 15], 7-bit
// mantissa).  To an fp8 type: a code k and the source value k * s (s a power of two).
__device__ __forceinline__ void k6_pair(uint64_t z, int sdt, int ddt, float dscale, uint32_t* sbits, uint32_t* dbits,
                                        bool* ok) {
  if (sdt == ddt) {
    *sbits = *dbits = finite_bits(z, sdt);
    return;
  }
  if (ddt == KV_F8E4M3 || ddt == KV_F8E4M3FNUZ) {
    const uint32_t k = finite_bits(z, ddt);
    *dbits = k;
    const float v = fp8_value(k, ddt == KV_F8E4M3FNUZ) * dscale;  // exact for power-of-two scales
    *sbits = exact_bits(v, sdt, ok);
    return;
  }
  // common grid: sign | exponent e in [-14, 15] | 7-bit mantissa
  const uint32_t sgn = (uint32_t)(z >> 63), e = (uint32_t)((z >> 8) % 30u), m = (uint32_t)z & 0x7Fu;
  const float v = ldexpf(1.0f + (float)m / 128.0f, (int)e - 14) * (sgn ? -1.0f : 1.0f);
  *sbits = exact_bits(v, sdt, ok);
  *dbits = exact_bits(v, ddt, ok);
}

__device__ __forceinline__ bool pow2_scale(float s) {
  return s > 0.f && (__float_as_uint(s) & 0x007FFFFFu) == 0 && ((__float_as_uint(s) >> 23) & 0xFFu) != 0;
}

__device__ __forceinline__ void store_bits(uint8_t* p, uint32_t b, int esize) {
  if (esize == 1) *p = (uint8_t)b;
  else if (esize == 2) *reinterpret_cast<uint16_t*>(p) = (uint16_t)b;
  else *reinterpret_cast<uint32_t*>(p) = b;
}
__device__ __forceinline__ uint32_t load_bits(const uint8_t* p, int esize) {
  if (esize == 1) return *p;
  if (esize == 2) return *reinterpret_cast<const uint16_t*>(p);
  return *reinterpret_cast<const uint32_t*>(p);
}

// element index -> (table entry, layer, K/V, slot, local head, dim), innermost dim first
struct Coord {
  uint32_t e, l, c, slot, hl, d;
};
__device__ __forceinline__ Coord decode(uint64_t i, const VerifyArgs& a) {
  Coord k;
  k.d = (uint32_t)(i % (uint64_t)a.D);
  i /= (uint64_t)a.D;
  k.hl = (uint32_t)(i % (uint64_t)a.p.Hl);
  i /= (uint64_t)a.p.Hl;
  k.slot = (uint32_t)(i % (uint64_t)a.B);
  i /= (uint64_t)a.B;
  k.c = (uint32_t)(i & 1u);
  i >>= 1;
  k.l = (uint32_t)(i % (uint64_t)a.Lc);
  k.e = (uint32_t)(i / (uint64_t)a.Lc);
  return k;
}

__device__ __forceinline__ uint64_t pool_off(const VerifyArgs& a, const Coord& k, int64_t blk) {
  return (uint64_t)((int64_t)k.l * a.p.st[KV_AX_LAYER] + (int64_t)k.c * a.p.st[KV_AX_KV] + blk * a.p.st[KV_AX_BLOCK] +
                    (int64_t)k.slot * a.p.st[KV_AX_SLOT] + (int64_t)k.hl * a.p.st[KV_AX_HEAD] +
                    (int64_t)k.d * a.p.st[KV_AX_DIM]);
}

__global__ void __launch_bounds__(kVThreads) k_verify_fill(const __grid_constant__ VerifyArgs a) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < a.n_elem;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const Coord k = decode(i, a);
    const int32_t r = a.blk_req[k.e];
    const uint32_t t = (uint32_t)(k.e - a.blk_off[r]) * (uint32_t)a.B + k.slot;
    if ((int32_t)t >= a.tok_off[r + 1] - a.tok_off[r]) continue;  // tail slot: untouched
    const uint32_t h = (uint32_t)a.p.rank * (uint32_t)a.p.Hl + k.hl;
    const uint32_t rid = a.req_ids ? (uint32_t)a.req_ids[r] : (uint32_t)r;
    const uint64_t z = k6_hash(a.seed, rid, t, (uint32_t)(a.l0 + (int32_t)k.l), k.c, h, k.d);
    float sc = 1.f;
    if (a.ddt == KV_F8E4M3 || a.ddt == KV_F8E4M3FNUZ) {
      if (a.sdt != a.ddt) {
        const uint32_t q = h / (uint32_t)a.Hd, hq = h - q * (uint32_t)a.Hd;
        sc = a.dscale[q][((int64_t)(a.l0 + (int32_t)k.l - a.d_l0) * 2 + k.c) * a.Hd + hq];
        if (!pow2_scale(sc)) *a.err = 1;
      }
    }
    uint32_t sb, db;
    bool ok = true;
    k6_pair(z, a.sdt, a.ddt, sc, &sb, &db, &ok);
    if (!ok) *a.err = 1;
    store_bits(a.pool + pool_off(a, k, a.blk_ids[k.e]) * a.p.esize, sb, a.p.esize);
  }
}

__global__ void __launch_bounds__(kVThreads) k_verify_check(const __grid_constant__ VerifyArgs a) {
  unsigned long long bad_v = 0, bad_t = 0, checked = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < a.n_elem;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const Coord k = decode(i, a);
    const int32_t r = a.blk_req[k.e];
    const uint32_t t = (uint32_t)(k.e - a.blk_off[r]) * (uint32_t)a.B + k.slot;
    const uint64_t off = pool_off(a, k, a.blk_ids[k.e]);
    const uint32_t got = load_bits(a.pool + off * a.p.esize, a.p.esize);
    uint32_t want = 0;
    const bool valid = (int32_t)t < a.tok_off[r + 1] - a.tok_off[r];
    if (valid) {
      const uint32_t h = (uint32_t)a.p.rank * (uint32_t)a.p.Hl + k.hl;
      const uint32_t rid = a.req_ids ? (uint32_t)a.req_ids[r] : (uint32_t)r;
      const uint64_t z = k6_hash(a.seed, rid, t, (uint32_t)(a.l0 + (int32_t)k.l), k.c, h, k.d);
      float sc = 1.f;
      if ((a.ddt == KV_F8E4M3 || a.ddt == KV_F8E4M3FNUZ) && a.sdt != a.ddt)
        sc = a.dscale[0][((int64_t)k.l * 2 + k.c) * a.Hd + k.hl];
      uint32_t sb;
      bool ok = true;
      k6_pair(z, a.sdt, a.ddt, sc, &sb, &want, &ok);
      ++checked;
    }
    if (got != want) {
      if (valid) ++bad_v;
      else ++bad_t;
      atomicCAS(a.res + 4, 0ull, (unsigned long long)off + 1ull);
    }
  }
  if (bad_v) atomicAdd(a.res + 0, bad_v);
  if (bad_t) atomicAdd(a.res + 1, bad_t);
  if (checked) atomicAdd(a.res + 3, checked);
}

__global__ void k_verify_mark(uint8_t* mark, const int32_t* blk_ids, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    mark[blk_ids[i]] = 1;
}

// every element of an unused block must still hold the canary byte pattern
__global__ void __launch_bounds__(kVThreads) k_verify_canary(const __grid_constant__ VerifyArgs a) {
  unsigned long long bad = 0;
  const uint32_t cw = 0x01010101u * a.canary;
  const uint64_t nblk = (uint64_t)a.p.ext[KV_AX_BLOCK];
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < a.pool_elems;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t blk = (i / (uint64_t)a.p.st[KV_AX_BLOCK]) % nblk;
    if (a.mark[blk]) continue;
    const uint32_t got = load_bits(a.pool + i * a.p.esize, a.p.esize);
    const uint32_t want = a.p.esize == 4 ? cw : a.p.esize == 2 ? (cw & 0xFFFFu) : (cw & 0xFFu);
    if (got != want) ++bad;
  }
  if (bad) atomicAdd(a.res + 2, bad);
}

int vgrid(uint64_t n) {
  const uint64_t need = (n + kVThreads - 1) / kVThreads;
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(need, 148ull * 16ull));
}

kv_status view_of(const kv_layout* lay, VLay* v) {
  const kv_layout_desc& d = lay->d;
  if (d.kv_part != 0 || d.dim_split > 1)
    return fail(KV_EUNSUPPORTED, "kv_verify: K-only / V-only and x-split pools are not covered by K6");
  v->ext[KV_AX_LAYER] = d.num_layers;
  v->ext[KV_AX_KV] = 2;
  v->ext[KV_AX_BLOCK] = d.num_blocks;
  v->ext[KV_AX_SLOT] = d.block_size;
  v->ext[KV_AX_HEAD] = d.num_kv_heads / d.tp_degree;
  v->ext[KV_AX_DIM] = d.head_dim;
  int64_t s = 1;
  for (int i = 5; i >= 0; --i) {  // dense row-major in axis_order (K6's own stride derivation)
    v->st[d.axis_order[i]] = s;
    s *= v->ext[d.axis_order[i]];
  }
  v->esize = dtype_bytes(d.dtype);
  v->dtype = d.dtype;
  v->Hl = d.num_kv_heads / d.tp_degree;
  v->rank = d.tp_rank;
  return KV_OK;
}

bool pair_supported(int sdt, int ddt) {
  if (sdt == ddt) return true;
  const bool wide_s = sdt == KV_F16 || sdt == KV_BF16 || sdt == KV_F32;
  const bool wide_d = ddt == KV_F16 || ddt == KV_BF16 || ddt == KV_F32;
  return wide_s && (wide_d || ddt == KV_F8E4M3 || ddt == KV_F8E4M3FNUZ);
}

kv_status common(const kv_layout* pool_lay, const kv_batch* bt, int32_t sdt, int32_t ddt, VerifyArgs* a) {
  if (!pool_lay || !bt) return fail(KV_EINVAL, "kv_verify: null argument");
  if (!pair_supported(sdt, ddt)) return fail(KV_EUNSUPPORTED, "kv_verify: fp8 sources are not covered by K6");
  if (bt->block_size != pool_lay->d.block_size || bt->num_blocks != pool_lay->d.num_blocks)
    return fail(KV_ESHAPE, "kv_verify: tables built for another pool");
  if (pool_lay->d.num_layers > 255 || pool_lay->d.num_kv_heads > 511 || pool_lay->d.head_dim > 1023 ||
      bt->n_req > 65535 || bt->max_tokens > (1 << 20))
    return fail(KV_EUNSUPPORTED, "kv_verify: shape beyond the K6 hash key");
  kv_status st = view_of(pool_lay, &a->p);
  if (st != KV_OK) return st;
  a->sdt = sdt;
  a->ddt = ddt;
  a->l0 = pool_lay->d.first_layer;
  a->H = pool_lay->d.num_kv_heads;
  a->D = pool_lay->d.head_dim;
  a->B = pool_lay->d.block_size;
  a->Lc = pool_lay->d.num_layers;
  a->blk_off = bt->blk_off;
  a->blk_ids = bt->blk_ids;
  a->blk_req = bt->blk_req;
  a->tok_off = bt->tok_off;
  a->n_elem = (uint64_t)bt->total_blocks * (uint64_t)a->Lc * 2ull * (uint64_t)a->B * (uint64_t)a->p.Hl * (uint64_t)a->D;
  return KV_OK;
}

}  // namespace

namespace kvx {
cudaError_t preload_verify_kernels() {
  cudaFuncAttributes at;
  cudaError_t e;
  if ((e = cudaFuncGetAttributes(&at, reinterpret_cast<const void*>(k_verify_fill))) != cudaSuccess) return e;
  if ((e = cudaFuncGetAttributes(&at, reinterpret_cast<const void*>(k_verify_check))) != cudaSuccess) return e;
  if ((e = cudaFuncGetAttributes(&at, reinterpret_cast<const void*>(k_verify_mark))) != cudaSuccess) return e;
  return cudaFuncGetAttributes(&at, reinterpret_cast<const void*>(k_verify_canary));
}
}  // namespace kvx

extern "C" {

kv_status kv_verify_fill(const kv_layout* src, void* src_pool, const kv_batch* src_bt, int32_t n_dst,
                         const kv_layout* const* dst, const int32_t* req_ids, uint64_t seed, int32_t* err,
                         kv_stream stream) {
  if (!src || !src_pool || !dst || n_dst < 1 || n_dst > KVX_MAX_RANKS || !err)
    return fail(KV_EINVAL, "kv_verify_fill: bad argument");
  VerifyArgs a;
  memset(&a, 0, sizeof(a));
  kv_status st = common(src, src_bt, src->d.dtype, dst[0]->d.dtype, &a);
  if (st != KV_OK) return st;
  const int32_t Hd = dst[0]->d.num_kv_heads / dst[0]->d.tp_degree;
  a.Hd = Hd;
  a.d_l0 = dst[0]->d.first_layer;
  const bool q8 = fp8(a.ddt) && a.sdt != a.ddt;
  // D ranks covering this P rank's heads, indexed by D tp_rank
  for (int i = 0; i < n_dst; ++i) {
    if (!dst[i] || dst[i]->d.dtype != a.ddt || dst[i]->d.num_kv_heads != a.H || dst[i]->d.tp_rank >= KVX_MAX_RANKS)
      return fail(KV_EINVAL, "kv_verify_fill: destination layouts disagree");
    if (q8 && !dst[i]->d.scales) return fail(KV_EINVAL, "kv_verify_fill: fp8 destination without scales");
    a.dscale[dst[i]->d.tp_rank] = dst[i]->d.scales;
  }
  if (q8)
    for (int32_t h = src->d.tp_rank * a.p.Hl; h < (src->d.tp_rank + 1) * a.p.Hl; ++h)
      if (!a.dscale[h / Hd]) return fail(KV_ESHAPE, "kv_verify_fill: the D rank holding head " + std::to_string(h) +
                                                     " is not listed");
  a.req_ids = req_ids;
  a.seed = seed;
  a.pool = static_cast<uint8_t*>(src_pool);
  a.err = err;
  if (a.n_elem == 0) return KV_OK;
  k_verify_fill<<<vgrid(a.n_elem), kVThreads, 0, (cudaStream_t)stream>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? KV_OK : cuda_fail(e, "kv_verify_fill: launch");
}

kv_status kv_verify_check(const kv_layout* src, const kv_layout* dst, const void* dst_pool, const kv_batch* dst_bt,
                          const int32_t* req_ids, uint64_t seed, uint8_t canary, uint8_t* scratch,
                          size_t scratch_bytes, unsigned long long* result, kv_stream stream) {
  if (!src || !dst || !dst_pool || !scratch || !result) return fail(KV_EINVAL, "kv_verify_check: bad argument");
  if (scratch_bytes < (size_t)dst->d.num_blocks)
    return fail(KV_ESHAPE, "kv_verify_check: scratch needs one byte per D block");
  if (src->d.num_kv_heads != dst->d.num_kv_heads || src->d.head_dim != dst->d.head_dim)
    return fail(KV_ESHAPE, "kv_verify_check: layouts describe different models");
  VerifyArgs a;
  memset(&a, 0, sizeof(a));
  kv_status st = common(dst, dst_bt, src->d.dtype, dst->d.dtype, &a);
  if (st != KV_OK) return st;
  const bool q8 = fp8(a.ddt) && a.sdt != a.ddt;
  if (q8 && !dst->d.scales) return fail(KV_EINVAL, "kv_verify_check: fp8 destination without scales");
  a.Hd = a.p.Hl;
  a.dscale[0] = dst->d.scales;
  a.req_ids = req_ids;
  a.seed = seed;
  a.pool = const_cast<uint8_t*>(static_cast<const uint8_t*>(dst_pool));
  a.res = result;
  a.canary = canary;
  a.mark = scratch;
  a.pool_elems = (uint64_t)dst->pool_bytes / (uint64_t)a.p.esize;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if ((e = cudaMemsetAsync(result, 0, 8 * sizeof(unsigned long long), s)) != cudaSuccess ||
      (e = cudaMemsetAsync(scratch, 0, (size_t)dst->d.num_blocks, s)) != cudaSuccess)
    return cuda_fail(e, "kv_verify_check: memset");
  if (dst_bt->total_blocks) {
    k_verify_mark<<<vgrid((uint64_t)dst_bt->total_blocks), kVThreads, 0, s>>>(scratch, dst_bt->blk_ids,
                                                                              dst_bt->total_blocks);
    k_verify_check<<<vgrid(a.n_elem), kVThreads, 0, s>>>(a);
    g_launches.fetch_add(2, std::memory_order_relaxed);
  }
  k_verify_canary<<<vgrid(a.pool_elems), kVThreads, 0, s>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  e = cudaGetLastError();
  return e == cudaSuccess ? KV_OK : cuda_fail(e, "kv_verify_check: launch");
}

}  // extern "C"
