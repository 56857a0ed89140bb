// Host side of the C ABI (include/kvx.h): validation, strides, block tables, re-shard
// planning and kernel dispatch.  Every step of the data path runs in the kernels of
// kvx_kernels.cu; this file only checks arguments and marshals them.
#include <string.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <vector>

#include "kvx_internal.h"

namespace kvx {

static thread_local std::string t_err;
static thread_local const char* t_last_kernel = "";
std::atomic<uint64_t> g_launches{0};
std::atomic<int32_t> g_sm_budget[kMaxDevices];

kv_status fail(kv_status st, const std::string& msg) {
  t_err = msg;
  return st;
}

kv_status cuda_fail(cudaError_t e, const char* what) {
  t_err = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return KV_ECUDA;
}

bool fp8(int32_t dt) { return dt == KV_F8E4M3 || dt == KV_F8E4M3FNUZ; }

kv_status kv_pair(const kv_layout* s, const kv_layout* d, int32_t* kv1, int32_t* c0) {
  static const int mask[3] = {3, 1, 2};  // bit c set: the pool holds K (c=0) / V (c=1)
  const int m = mask[s->d.kv_part] & mask[d->d.kv_part];
  if (!m) return fail(KV_ESHAPE, "P and D layouts share neither K nor V (kv_part)");
  *kv1 = m == 3 ? 0 : 1;
  *c0 = m == 2 ? 1 : 0;
  return KV_OK;
}

int32_t dtype_bytes(int32_t dt) {
  switch (dt) {
    case KV_F16:
    case KV_BF16: return 2;
    case KV_F8E4M3:
    case KV_F8E4M3FNUZ: return 1;
    case KV_F32: return 4;
  }
  return 0;
}

FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0, 0};
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  f.shr = l;
  f.mul = (uint32_t)((((1ull << 32) * ((1ull << l) - d)) / d) + 1);
  return f;
}

}  // namespace kvx

using namespace kvx;

namespace {

bool ptr_aligned(const void* p, size_t a) { return ((uintptr_t)p % a) == 0; }

// Two layouts describe the same instance (same model, blocks, order, dtype, tp degree).
bool same_instance(const kv_layout* a, const kv_layout* b) {
  const kv_layout_desc &x = a->d, &y = b->d;
  if (x.num_layers != y.num_layers || x.first_layer != y.first_layer || x.num_kv_heads != y.num_kv_heads ||
      x.head_dim != y.head_dim ||
      x.tp_degree != y.tp_degree || x.block_size != y.block_size || x.num_blocks != y.num_blocks ||
      x.dtype != y.dtype)
    return false;
  for (int i = 0; i < 6; ++i)
    if (x.axis_order[i] != y.axis_order[i]) return false;
  return x.kv_part == y.kv_part && a->dk == b->dk;
}

kv_status check_batch(const kv_batch* bt, const kv_layout* lay, const char* name) {
  if (!bt) return fail(KV_EINVAL, std::string(name) + " is NULL");
  if (bt->block_size != lay->d.block_size || bt->num_blocks != lay->d.num_blocks)
    return fail(KV_ESHAPE, std::string(name) + " was built for another block size / pool");
  if (bt->n_req < 0 || (bt->n_req > 0 && (!bt->tok_off || !bt->blk_off || !bt->blk_ids || !bt->blk_req)))
    return fail(KV_EINVAL, std::string(name) + " has null device arrays");
  return KV_OK;
}

kv_status check_layers(const kv_layout* lay, int32_t lb, int32_t le) {
  const int32_t f = lay->d.first_layer, e = lay->d.first_layer + lay->d.num_layers;
  if (lb < f || le < lb || le > e)
    return fail(KV_EINVAL, "layer range [" + std::to_string(lb) + ", " + std::to_string(le) + ") outside the pool's [" +
                               std::to_string(f) + ", " + std::to_string(e) + ")");
  return KV_OK;
}

void head_overlap(const kv_layout* s, const kv_layout* d, int32_t* hb, int32_t* he) {
  const int32_t H = s->d.num_kv_heads;
  const int32_t Hp = H / s->d.tp_degree, Hd = H / d->d.tp_degree;
  const int32_t p = s->d.tp_rank, q = d->d.tp_rank;
  *hb = std::max(p * Hp, q * Hd);
  *he = std::min((p + 1) * Hp, (q + 1) * Hd);
}

// The fast path needs head_dim innermost and contiguous with 8-element chunks.
bool fast_ok(const kv_layout* lay) {
  const int32_t cpr = lay->d.head_dim / 8;  // 8-element chunks per row; a power of two for the row kernel
  return lay->stride[KV_AX_DIM] == 1 && lay->d.head_dim % 8 == 0 && (cpr & (cpr - 1)) == 0;
}

kv_status same_model(const kv_layout* s, const kv_layout* d) {
  if (s->d.num_kv_heads != d->d.num_kv_heads || s->d.head_dim != d->d.head_dim)
    return fail(KV_ESHAPE, "P and D layouts describe different models (kv heads / head_dim)");
  return KV_OK;
}

kv_status scales_ok(const kv_layout* s, const kv_layout* d) {
  // dequantising an fp8 source needs its scales; quantising to fp8 needs the destination's
  // (same dtype is a bit copy and needs neither)
  if (fp8(d->d.dtype) && s->d.dtype != d->d.dtype && !d->d.scales)
    return fail(KV_EINVAL, "fp8 destination without scales");
  if (fp8(s->d.dtype) && d->d.dtype != s->d.dtype && !s->d.scales)
    return fail(KV_EINVAL, "fp8 source without scales");
  return KV_OK;
}

// slot/head order: whichever of the two is inner in the destination layout
int32_t slot_inner_of(const kv_layout* d) {
  int ps = 0, ph = 0;
  for (int i = 0; i < 6; ++i) {
    if (d->d.axis_order[i] == KV_AX_SLOT) ps = i;
    if (d->d.axis_order[i] == KV_AX_HEAD) ph = i;
  }
  return ps > ph ? 1 : 0;
}

constexpr uint64_t kMaxChunks = 0x7FFFFFFFull;  // per launch (32-bit decode)

}  // namespace

extern "C" {

const char* kv_last_error(void) { return t_err.c_str(); }
const char* kv_last_kernel(void) { return t_last_kernel; }
const char* kv_version(void) { return "kvx 0.1 (sm_100a)"; }
uint64_t kv_launch_count(void) { return g_launches.load(); }
void kv_launch_count_reset(void) { g_launches.store(0); }
int32_t kv_set_sm_budget(int32_t n_sms) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  return g_sm_budget[dev].exchange(n_sms < 0 ? 0 : n_sms);
}

kv_status kv_layout_describe(const kv_layout_desc* desc, kv_layout** out, size_t* pool_bytes) {
  if (!desc || !out) return fail(KV_EINVAL, "kv_layout_describe: null argument");
  const kv_layout_desc& d = *desc;
  if (d.num_layers <= 0 || d.num_kv_heads <= 0 || d.head_dim <= 0 || d.tp_degree <= 0 || d.block_size <= 0 ||
      d.num_blocks <= 0)
    return fail(KV_EINVAL, "kv_layout_describe: non-positive extent");
  if (dtype_bytes(d.dtype) == 0) return fail(KV_EINVAL, "kv_layout_describe: bad dtype");
  if (d.first_layer < 0) return fail(KV_EINVAL, "kv_layout_describe: negative first_layer");
  if (d.num_kv_heads % d.tp_degree != 0)
    return fail(KV_ESHAPE, "kv_layout_describe: tp_degree " + std::to_string(d.tp_degree) +
                               " does not divide num_kv_heads " + std::to_string(d.num_kv_heads));
  if (d.tp_rank < 0 || d.tp_rank >= d.tp_degree) return fail(KV_ESHAPE, "kv_layout_describe: tp_rank out of range");
  bool seen[6] = {false, false, false, false, false, false};
  for (int i = 0; i < 6; ++i) {
    int a = d.axis_order[i];
    if (a < 0 || a > 5 || seen[a]) return fail(KV_EINVAL, "kv_layout_describe: axis_order is not a permutation");
    seen[a] = true;
  }
  if (fp8(d.dtype) && !d.scales) return fail(KV_EINVAL, "kv_layout_describe: fp8 layout needs scales");
  if (d.kv_part < 0 || d.kv_part > 2) return fail(KV_EINVAL, "kv_layout_describe: kv_part must be 0, 1 or 2");
  int32_t dk = 0;
  if (d.dim_split > 1) {
    if ((d.dim_split & (d.dim_split - 1)) || d.head_dim % d.dim_split)
      return fail(KV_EINVAL, "kv_layout_describe: dim_split must be a power of two dividing head_dim");
    while ((1 << dk) < d.dim_split) ++dk;
    if (d.axis_order[5] == KV_AX_DIM) dk = 0;  // DIM innermost: the split changes nothing
  } else if (d.dim_split < 0) {
    return fail(KV_EINVAL, "kv_layout_describe: negative dim_split");
  }
  kv_layout* L = new (std::nothrow) kv_layout;
  if (!L) return fail(KV_EINVAL, "kv_layout_describe: out of host memory");
  L->d = d;
  L->h_local = d.num_kv_heads / d.tp_degree;
  L->elem_bytes = dtype_bytes(d.dtype);
  L->dk = dk;
  L->extent[KV_AX_LAYER] = d.num_layers;
  L->extent[KV_AX_KV] = d.kv_part ? 1 : 2;
  L->extent[KV_AX_BLOCK] = d.num_blocks;
  L->extent[KV_AX_SLOT] = d.block_size;
  L->extent[KV_AX_HEAD] = L->h_local;
  L->extent[KV_AX_DIM] = d.head_dim >> dk;
  int64_t s = 1 << dk;  // the x part of a split head_dim is innermost
  for (int i = 5; i >= 0; --i) {
    L->stride[d.axis_order[i]] = s;
    s *= L->extent[d.axis_order[i]];
  }
  // a K-only / V-only pool stores its one K/V at index 0: the global index must not move it
  if (d.kv_part) L->stride[KV_AX_KV] = 0;
  L->pool_bytes = (size_t)s * (size_t)L->elem_bytes;
  if (pool_bytes) *pool_bytes = L->pool_bytes;
  *out = L;
  return KV_OK;
}

void kv_layout_destroy(kv_layout* lay) { delete lay; }

size_t kv_batch_bytes(int32_t n_req, int64_t total_blocks, int64_t total_tokens) {
  auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
  return al(4 * (size_t)(n_req + 1)) * 2 + al(4 * (size_t)total_blocks) * 2 + al(4 * (size_t)total_tokens);
}

kv_status kv_block_table_update(const kv_layout* lay, int32_t n_req, const int32_t* host_n_tokens,
                                const int32_t* host_block_ids, int64_t n_ids, void* dev_buf, size_t dev_buf_bytes,
                                kv_batch* out, kv_stream stream) {
  if (!lay || !out || n_req < 0 || (n_req > 0 && !host_n_tokens) || (n_ids > 0 && !host_block_ids))
    return fail(KV_EINVAL, "kv_block_table_update: null argument");
  const int32_t B = lay->d.block_size, NB = lay->d.num_blocks;
  std::vector<int32_t> tok_off(n_req + 1), blk_off(n_req + 1);
  int64_t tt = 0, tb = 0;
  int32_t maxT = 0;
  uint64_t digest = 1469598103934665603ull;
  for (int32_t r = 0; r < n_req; ++r) {
    const int32_t T = host_n_tokens[r];
    if (T < 0) return fail(KV_EINVAL, "kv_block_table_update: negative token count");
    tok_off[r] = (int32_t)tt;
    blk_off[r] = (int32_t)tb;
    tt += T;
    tb += (T + B - 1) / B;
    maxT = std::max(maxT, T);
    for (int i = 0; i < 4; ++i) {
      digest ^= (uint64_t)((T >> (8 * i)) & 0xFF);
      digest *= 1099511628211ull;
    }
    if (tt > 0x7FFFFFFF || tb > 0x7FFFFFFF) return fail(KV_ESHAPE, "kv_block_table_update: batch too large");
  }
  tok_off[n_req] = (int32_t)tt;
  blk_off[n_req] = (int32_t)tb;
  if (tb != n_ids)
    return fail(KV_ESHAPE, "kv_block_table_update: " + std::to_string(n_ids) + " block ids given, sum ceil(T/B) = " +
                               std::to_string(tb));
  std::vector<uint8_t> used((size_t)NB, 0);
  for (int64_t i = 0; i < n_ids; ++i) {
    const int32_t b = host_block_ids[i];
    if (b < 0 || b >= NB)
      return fail(KV_ESHAPE, "kv_block_table_update: block id " + std::to_string(b) + " outside [0, " +
                                 std::to_string(NB) + ")");
    if (used[b]) return fail(KV_ESHAPE, "kv_block_table_update: block id " + std::to_string(b) + " used twice");
    used[b] = 1;
  }
  const size_t need = kv_batch_bytes(n_req, tb, tt);
  if (!dev_buf || dev_buf_bytes < need || !ptr_aligned(dev_buf, 16))
    return fail(KV_ESHAPE, "kv_block_table_update: device buffer of " + std::to_string(dev_buf_bytes) +
                               " bytes is null, short or misaligned (need " + std::to_string(need) + ")");
  // host staging image of [tok_off | blk_off | blk_ids | blk_req | tok_req], 16-B aligned parts
  auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
  const size_t o_tok = 0, o_blk = al(4 * (size_t)(n_req + 1)), o_ids = o_blk + al(4 * (size_t)(n_req + 1)),
               o_req = o_ids + al(4 * (size_t)tb), o_treq = o_req + al(4 * (size_t)tb);
  std::vector<uint8_t> img(need, 0);
  memcpy(img.data() + o_tok, tok_off.data(), 4 * (size_t)(n_req + 1));
  memcpy(img.data() + o_blk, blk_off.data(), 4 * (size_t)(n_req + 1));
  if (tb) memcpy(img.data() + o_ids, host_block_ids, 4 * (size_t)tb);
  int32_t* breq = reinterpret_cast<int32_t*>(img.data() + o_req);
  int32_t* treq = reinterpret_cast<int32_t*>(img.data() + o_treq);
  for (int32_t r = 0; r < n_req; ++r) {
    for (int32_t j = blk_off[r]; j < blk_off[r + 1]; ++j) breq[j] = r;
    for (int32_t t = tok_off[r]; t < tok_off[r + 1]; ++t) treq[t] = r;
  }
  cudaError_t e = cudaMemcpyAsync(dev_buf, img.data(), need, cudaMemcpyHostToDevice, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "kv_block_table_update: upload");
  // the host image is pageable: the copy is staged before cudaMemcpyAsync returns, but make
  // the lifetime rule trivially true by waiting for this small upload
  e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "kv_block_table_update: sync");
  uint8_t* base = static_cast<uint8_t*>(dev_buf);
  out->n_req = n_req;
  out->block_size = B;
  out->num_blocks = NB;
  out->max_tokens = maxT;
  out->total_tokens = tt;
  out->total_blocks = tb;
  out->token_digest = digest;
  out->tok_off = reinterpret_cast<const int32_t*>(base + o_tok);
  out->blk_off = reinterpret_cast<const int32_t*>(base + o_blk);
  out->blk_ids = reinterpret_cast<const int32_t*>(base + o_ids);
  out->blk_req = reinterpret_cast<const int32_t*>(base + o_req);
  out->tok_req = reinterpret_cast<const int32_t*>(base + o_treq);
  return KV_OK;
}

int32_t kv_plan_pairs(int32_t tp_p, int32_t tp_d, int32_t H, int32_t* out, int32_t max_pairs) {
  if (tp_p <= 0 || tp_d <= 0 || H <= 0 || H % tp_p || H % tp_d) {
    fail(KV_ESHAPE, "kv_plan_pairs: a tp degree does not divide num_kv_heads");
    return -1;
  }
  const int32_t Hp = H / tp_p, Hd = H / tp_d;
  int32_t n = 0;
  // walk heads once; a new pair starts wherever p or q changes (head-contiguous TP)
  int32_t cur_p = -1, cur_q = -1;
  for (int32_t h = 0; h < H; ++h) {
    const int32_t p = h / Hp, q = h / Hd;
    if (p != cur_p || q != cur_q) {
      if (out && n < max_pairs) {
        out[4 * n + 0] = p;
        out[4 * n + 1] = q;
        out[4 * n + 2] = h;
      }
      if (out && n > 0 && n - 1 < max_pairs) out[4 * (n - 1) + 3] = h;
      ++n;
      cur_p = p;
      cur_q = q;
    }
  }
  if (out && n > 0 && n - 1 < max_pairs) out[4 * (n - 1) + 3] = H;
  return n;
}

}  // extern "C"

namespace {
// ---- same-dtype TMA tile path (k_tile_copy) ---------------------------------------
typedef CUresult (*encode_tiled_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

encode_tiled_fn encode_fn() {
  // resolved once, thread-safely (function-local static initialisation)
  static const encode_tiled_fn fn = []() -> encode_tiled_fn {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess && p)
      return reinterpret_cast<encode_tiled_fn>(p);
    cudaGetLastError();
    return nullptr;
  }();
  return fn;
}

// KVX_TILE: 0 off, 1 auto (default: sub-tiles of >= 32 KB, where one TMA operation per
// sub-tile beats the row kernel -- c2 0.92 vs 0.90 of copy; with 8-KB sub-tiles (c3, c5) the
// row kernel is 2% faster), 2 force (tests).  Read per call so tests can switch it.
int tile_mode() {
  const char* e = getenv("KVX_TILE");
  return e ? atoi(e) : 1;
}

// Same dtype, head_dim innermost on both sides, D's three innermost axes {HEAD, SLOT} x DIM,
// B_d a multiple of B_p, head counts dividing each other: one TMA tensor load per source
// sub-tile whose map enumerates the source in D's order, bulk stores of D's runs.  Sets
// *used = false (and launches nothing) when the case does not fit.
// KVX_TT: the TMA-fed cast variant (k_tile_cast) for converts whose dtypes differ -- 0 off,
// 1 (default) on.  Read per call.
int tile_cast_mode() {
  const char* e = getenv("KVX_TT");
  return e ? atoi(e) : 1;
}

kv_status try_tile_copy(int32_t n_src, const kv_layout* const* src, const void* const* src_pools,
                        const kv_batch* src_bt, int32_t n_dst, const kv_layout* const* dst, void* const* dst_pools,
                        const kv_batch* dst_bt, int32_t lb, int32_t le, kv_stream stream, bool share, bool* used) {
  *used = false;
  // KVX_TT_SAME=1 (experiment): same-dtype converts through the consumer-warp kernel too
  const char* same_env = getenv("KVX_TT_SAME");
  const bool cast = src[0]->d.dtype != dst[0]->d.dtype || (same_env && atoi(same_env) == 1);
  const int mode = cast ? tile_cast_mode() : tile_mode();
  if (mode == 0) return KV_OK;
  // the cast variant where it measured faster than the row kernel (c4-pair shapes,
  // profiles/r02/tile_cast_vs_rows.txt): 2-byte sources into 1- or 2-byte destinations
  // (bf16 -> e4m3 1.016 vs 0.983 of copy); 1-byte sources (e4m3 -> bf16 0.89 vs 0.98, fnuz ->
  // e4m3 0.63 vs 0.84), 4-byte destinations (tie) and the per-P-rank share of the peer-store
  // push (0.776 vs 0.791 of the link) stay on the row kernel
  if (cast && (src[0]->elem_bytes != 2 || dst[0]->elem_bytes > 2 || share)) return KV_OK;
  const kv_layout *S = src[0], *D = dst[0];
  const int32_t* o = D->d.axis_order;
  int head_major;
  if (o[5] != KV_AX_DIM) return KV_OK;
  if (o[3] == KV_AX_HEAD && o[4] == KV_AX_SLOT)
    head_major = 1;
  else if (o[3] == KV_AX_SLOT && o[4] == KV_AX_HEAD)
    head_major = 0;
  else
    return KV_OK;
  const int32_t Hp = S->h_local, Hd = D->h_local, Bp = S->d.block_size, Bd = D->d.block_size, Dm = S->d.head_dim;
  const int32_t esize = S->elem_bytes;
  int32_t nh = std::min(Hp, Hd);
  if (Bd % Bp != 0 || Bp > 256 || Dm > 256 || nh > 256 || (Hp % nh) || (Hd % nh)) return KV_OK;
  const int64_t row_bytes = (int64_t)Dm * esize;
  if (row_bytes % 16) return KV_OK;
  int64_t stage = (int64_t)nh * Bp * row_bytes;
  // a sub-tile bigger than 64 KB (e.g. TP1 -> TP1 of 32 heads: 128 KB) leaves no room for a
  // second stage: split it by heads into head groups of <= 64 KB
  while (stage > 64 * 1024 && nh % 2 == 0) {
    nh /= 2;
    stage /= 2;
  }
  if (stage > 100 * 1024 || (mode == 1 && !cast && stage < 32 * 1024)) return KV_OK;
  if (cast && (nh > 8 || (nh & (nh - 1)) || (Bp & (Bp - 1)) || stage < 2048 || stage * kTbConsumers > 200 * 1024 ||
               (Dm / 8) & (Dm / 8 - 1) || Dm % 8))
    return KV_OK;
  encode_tiled_fn enc = encode_fn();
  if (!enc) return KV_OK;
  TileArgs a;
  memset(&a, 0, sizeof(a));
  kv_status pst = kv_pair(S, D, &a.kv1, &a.c0);
  if (pst != KV_OK) return pst;
  for (int i = 0; i < KVX_MAX_RANKS; ++i) a.src_of_p[i] = -1;
  const CUtensorMapDataType dt = esize == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : esize == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                              : CU_TENSOR_MAP_DATA_TYPE_UINT32;
  for (int i = 0; i < n_src; ++i) {
    const kv_layout* L = src[i];
    a.src_of_p[L->d.tp_rank] = (int8_t)i;
    const int64_t* st = L->stride;
    a.src[i] = static_cast<const uint8_t*>(src_pools[i]);
    for (int ax = 0; ax < 6; ++ax) a.ss[i][ax] = st[ax];
    cuuint64_t dims[5] = {(cuuint64_t)Dm, (cuuint64_t)(head_major ? Bp : Hp), (cuuint64_t)(head_major ? Hp : Bp),
                          (cuuint64_t)L->d.num_blocks, (cuuint64_t)L->d.num_layers};
    cuuint64_t strides[4] = {(cuuint64_t)((head_major ? st[KV_AX_SLOT] : st[KV_AX_HEAD]) * esize),
                             (cuuint64_t)((head_major ? st[KV_AX_HEAD] : st[KV_AX_SLOT]) * esize),
                             (cuuint64_t)(st[KV_AX_BLOCK] * esize), (cuuint64_t)(st[KV_AX_LAYER] * esize)};
    cuuint32_t box[5] = {(cuuint32_t)Dm, (cuuint32_t)(head_major ? Bp : nh), (cuuint32_t)(head_major ? nh : Bp), 1, 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    for (int c = 0; c < 2; ++c) {
      void* base = (uint8_t*)src_pools[i] + (size_t)c * (size_t)st[KV_AX_KV] * (size_t)esize;
      if (enc(&a.maps[i][c], dt, 5, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
          CUDA_SUCCESS)
        return KV_OK;  // this layout cannot be described by a tensor map: use the row kernel
    }
  }
  for (int i = 0; i < n_dst; ++i) {
    a.dst[i] = static_cast<uint8_t*>(dst_pools[i]);
    a.dst_rank[i] = (int8_t)dst[i]->d.tp_rank;
  }
  for (int ax = 0; ax < 6; ++ax) a.ds[ax] = D->stride[ax];
  a.Hp = Hp;
  a.Hd = Hd;
  a.Bp = Bp;
  a.Bd = Bd;
  a.D = Dm;
  a.esize = esize;
  a.nh = nh;
  a.s_l0 = S->d.first_layer;
  a.d_l0 = D->d.first_layer;
  a.head_major = head_major;
  a.share_p = share ? S->d.tp_rank : -1;
  a.stage_bytes = (int32_t)stage;
  a.stages = (int32_t)std::max<int64_t>(2, std::min<int64_t>(8, (200 * 1024) / stage));
  {  // k_tile_copy: L2 evict-first on its streaming loads and stores (c2: 0.943 -> 0.957 of copy,
     // profiles/r02/c2_evict_first.jsonl); KVX_TC_EVICT=0 turns it off
    const char* ev = getenv("KVX_TC_EVICT");
    a.evict_first = !(ev && *ev == '0');
  }
  if (cast) {
    a.d_esize = D->elem_bytes;
    for (int i = 0; i < n_src; ++i) a.sscale[i] = src[i]->d.scales;
    for (int i = 0; i < n_dst; ++i) a.dscale[i] = dst[i]->d.scales;
    const char* kb_env = getenv("KVX_TT_STAGE_KB");
    const int64_t kb = kb_env ? std::max(8, atoi(kb_env)) : 64;
    a.stages = (int32_t)std::max<int64_t>(kTbConsumers, std::min<int64_t>(16, kb * 1024 / stage));
  }
  a.s_blk_off = src_bt->blk_off;
  a.s_blk_ids = src_bt->blk_ids;
  a.d_blk_off = dst_bt->blk_off;
  a.d_blk_ids = dst_bt->blk_ids;
  a.d_blk_req = dst_bt->blk_req;
  a.tok_off = dst_bt->tok_off;
  // head groups per item set: the D rank's Hd heads, or (share) the heads P rank p holds of it
  int32_t ov = Hd;
  if (share) {
    const int32_t p = S->d.tp_rank, q = D->d.tp_rank;
    ov = std::min((p + 1) * Hp, (q + 1) * Hd) - std::max(p * Hp, q * Hd);
  }
  const uint32_t nparts = (uint32_t)(ov / nh), nsub = (uint32_t)(Bd / Bp);
  a.f_nd = make_fastdiv((uint32_t)n_dst);
  a.f_parts = make_fastdiv(nparts);
  a.f_sub = make_fastdiv(nsub);
  const uint64_t per_layer = (uint64_t)n_dst * nparts * nsub * (a.kv1 ? 1 : 2) * (uint64_t)dst_bt->total_blocks;
  if (per_layer > kMaxChunks) return KV_OK;
  const int32_t step = (int32_t)std::max<uint64_t>(1, kMaxChunks / per_layer);
  for (int32_t l0 = lb; l0 < le; l0 += step) {
    const int32_t l1 = std::min(le, l0 + step);
    a.lb = l0;
    a.Lc = l1 - l0;
    a.f_l = make_fastdiv((uint32_t)a.Lc);
    a.n_items = (uint32_t)(per_layer * (uint64_t)a.Lc);
    t_last_kernel = cast ? "k_tile_cast" : "k_tile_copy";
    cudaError_t e = cast ? launch_tile_cast(a, S->d.dtype, D->d.dtype, (cudaStream_t)stream)
                         : launch_tile_copy(a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "kv_convert_reshard: tile launch");
  }
  *used = true;
  return KV_OK;
}

// share == false: kv_convert_reshard (every P rank a listed D rank needs must be listed);
// share == true: kv_convert_share (one P rank converts only the D heads it holds).
kv_status convert_impl(int32_t n_src, const kv_layout* const* src, const void* const* src_pools,
                       const kv_batch* src_bt, int32_t n_dst, const kv_layout* const* dst, void* const* dst_pools,
                       const kv_batch* dst_bt, int32_t lb, int32_t le, kv_stream stream, bool share,
                       const Notify* nt = nullptr, bool* notified = nullptr) {
  if (n_src < 1 || n_src > KVX_MAX_RANKS || n_dst < 1 || n_dst > KVX_MAX_RANKS)
    return fail(KV_EINVAL, "kv_convert_reshard: need 1..16 source and destination ranks");
  if (!src || !src_pools || !dst || !dst_pools) return fail(KV_EINVAL, "kv_convert_reshard: null array");
  for (int i = 0; i < n_src; ++i)
    if (!src[i] || !src_pools[i]) return fail(KV_EINVAL, "kv_convert_reshard: null source layout/pool");
  for (int i = 0; i < n_dst; ++i)
    if (!dst[i] || !dst_pools[i]) return fail(KV_EINVAL, "kv_convert_reshard: null destination layout/pool");
  const kv_layout *S = src[0], *D = dst[0];
  for (int i = 1; i < n_src; ++i)
    if (!same_instance(src[i], S)) return fail(KV_ESHAPE, "kv_convert_reshard: source layouts differ beyond rank");
  for (int i = 1; i < n_dst; ++i)
    if (!same_instance(dst[i], D)) return fail(KV_ESHAPE, "kv_convert_reshard: destination layouts differ");
  kv_status st;
  if (S->d.tp_degree > KVX_MAX_RANKS || D->d.tp_degree > KVX_MAX_RANKS)
    return fail(KV_EUNSUPPORTED, "kv_convert_reshard: tp degree above 16");
  if ((st = same_model(S, D)) != KV_OK) return st;
  if ((st = check_layers(S, lb, le)) != KV_OK) return st;
  if ((st = check_layers(D, lb, le)) != KV_OK) return st;
  if ((st = check_batch(src_bt, S, "src_bt")) != KV_OK) return st;
  if ((st = check_batch(dst_bt, D, "dst_bt")) != KV_OK) return st;
  if (src_bt->n_req != dst_bt->n_req || src_bt->total_tokens != dst_bt->total_tokens ||
      src_bt->token_digest != dst_bt->token_digest)
    return fail(KV_ESHAPE, "kv_convert_reshard: P and D tables describe different requests");
  ConvArgs a;
  memset(&a, 0, sizeof(a));
  if ((st = kv_pair(S, D, &a.kv1, &a.c0)) != KV_OK) return st;
  a.s_dk = S->dk;
  a.d_dk = D->dk;
  for (int i = 0; i < KVX_MAX_RANKS; ++i) a.src_of_p[i] = -1;
  for (int i = 0; i < n_src; ++i) {
    const int p = src[i]->d.tp_rank;
    if (a.src_of_p[p] != -1) return fail(KV_EINVAL, "kv_convert_reshard: source rank listed twice");
    if ((st = scales_ok(src[i], D)) != KV_OK) return st;
    a.src_of_p[p] = (int8_t)i;
    a.src[i] = static_cast<const uint8_t*>(src_pools[i]);
    a.sscale[i] = src[i]->d.scales;
  }
  const int32_t H = S->d.num_kv_heads;
  const int32_t Hp = S->h_local, Hd = D->h_local;
  bool seen_q[KVX_MAX_RANKS] = {false};
  a.Hd_eff = share ? -1 : Hd;
  for (int i = 0; i < n_dst; ++i) {
    const int q = dst[i]->d.tp_rank;
    if (q >= KVX_MAX_RANKS || seen_q[q]) return fail(KV_EINVAL, "kv_convert_reshard: destination rank listed twice");
    seen_q[q] = true;
    if ((st = scales_ok(S, dst[i])) != KV_OK) return st;
    if (share) {
      // the D-local heads of q that P rank p holds: one contiguous range (head-contiguous TP)
      const int32_t p = S->d.tp_rank;
      const int32_t hb = std::max(p * Hp, q * Hd), he = std::min((p + 1) * Hp, (q + 1) * Hd);
      if (he <= hb)
        return fail(KV_ESHAPE, "kv_convert_share: P rank " + std::to_string(p) + " holds no head of D rank " +
                                   std::to_string(q));
      if (a.Hd_eff >= 0 && a.Hd_eff != he - hb)
        return fail(KV_EUNSUPPORTED, "kv_convert_share: unequal head overlaps across the listed D ranks; "
                                     "call once per D rank");
      a.Hd_eff = he - hb;
      a.hq_off[i] = (int8_t)(hb - q * Hd);
    } else {
      for (int32_t h = q * Hd; h < (q + 1) * Hd; ++h)
        if (a.src_of_p[h / Hp] < 0)
          return fail(KV_ESHAPE, "kv_convert_reshard: missing source shard for P rank " + std::to_string(h / Hp) +
                                     " (needed by D rank " + std::to_string(q) + ")");
    }
    a.dst[i] = static_cast<uint8_t*>(dst_pools[i]);
    a.dst_rank[i] = (int8_t)q;
    a.dscale[i] = dst[i]->d.scales;
  }
  (void)H;
  // row kernel: each side has head_dim-contiguous rows, or an x-split head_dim with x >= 8
  // (whole 8-element chunks inside each x-group, reading 27)
  auto rows_side = [](const kv_layout* L, int32_t* ck, int64_t* chs) -> bool {
    const int32_t cpr = L->d.head_dim / 8;
    if (L->d.head_dim % 8 || (cpr & (cpr - 1))) return false;
    if (L->dk == 0) {
      *ck = 0;
      *chs = 8 * (int64_t)L->elem_bytes;
      return L->stride[KV_AX_DIM] == 1;
    }
    if (L->dk < 3) return false;
    *ck = L->dk - 3;
    *chs = L->stride[KV_AX_DIM] * (int64_t)L->elem_bytes;
    return true;
  };
  // head_dim-major side ((DIM, SLOT) innermost, no split): the smem-transpose kernel, when
  // the other side is head_dim-major too or has contiguous rows
  // mode 1: (DIM, SLOT) innermost; mode 2: x-split head_dim with (D/x, SLOT, x) innermost
  // (x a multiple of 8): whole (block, head) tiles are contiguous and go through smem
  auto tr_side = [](const kv_layout* L) -> int {
    if (L->dk == 0 && L->d.axis_order[4] == KV_AX_DIM && L->d.axis_order[5] == KV_AX_SLOT)
      return L->d.block_size % 8 == 0 ? 1 : -1;
    if (L->dk >= 3 && L->d.axis_order[4] == KV_AX_DIM && L->d.axis_order[5] == KV_AX_SLOT) return 2;
    return 0;
  };
  auto plain_rows = [](const kv_layout* L) { return L->dk == 0 && L->stride[KV_AX_DIM] == 1; };
  {
    const int st = tr_side(S), dt = tr_side(D);
    const size_t smem = 4 * (size_t)D->d.block_size * (S->d.head_dim + 16 / S->elem_bytes) * S->elem_bytes;
    auto pow2 = [](int32_t x) { return x > 0 && (x & (x - 1)) == 0; };
    auto lg = [](int32_t x) {
      int32_t k = 0;
      while ((1 << k) < x) ++k;
      return k;
    };
    bool ok = (st > 0 || dt > 0) && st >= 0 && dt >= 0 && (st || plain_rows(S)) && (dt || plain_rows(D)) &&
              S->d.head_dim % 8 == 0 && pow2(S->d.head_dim / 8) && pow2(S->d.block_size) &&
              pow2(D->d.block_size) && D->d.block_size % S->d.block_size == 0 && smem <= (size_t)kTrSmemLimit;
    for (int i = 0; i < n_src && ok; ++i) ok = ptr_aligned(src_pools[i], 16);
    for (int i = 0; i < n_dst && ok; ++i) ok = ptr_aligned(dst_pools[i], 16);
    if (ok) {
      a.s_tr = st;
      a.d_tr = dt;
      a.s_x = 1 << S->dk;
      a.d_x = 1 << D->dk;
      a.tr_lbp = lg(S->d.block_size);
      a.tr_lbd = lg(D->d.block_size);
      a.s_lm = S->dk >= 3 ? S->dk - 3 : 0;
      a.d_lm = D->dk >= 3 ? D->dk - 3 : 0;
      a.cpr_shift = lg(S->d.head_dim / 8);
      a.s_dk = S->dk;
      a.d_dk = D->dk;
      // register path unless KVX_TR=0 (the smem-staged kernel) or a block holds < 8 slots
      const char* tr_env = getenv("KVX_TR");
      const bool use_tr8 = S->d.block_size >= 8 && D->d.block_size >= 8 && !(tr_env && atoi(tr_env) == 0);
      const char* w16_env = getenv("KVX_TR_W16");
      a.tr_w16 = (st == 1 && dt == 0 && S->elem_bytes == 2 && S->d.block_size >= 16 && D->d.block_size >= 16 &&
                  !(w16_env && atoi(w16_env) == 0)) ? 1 : 0;
      for (int ax = 0; ax < 6; ++ax) {
        a.ss[ax] = S->stride[ax];
        a.ds[ax] = D->stride[ax];
      }
      a.Hp = Hp;
      a.Hd = Hd;
      a.D = S->d.head_dim;
      a.Bp = S->d.block_size;
      a.Bd = D->d.block_size;
      a.s_l0 = S->d.first_layer;
      a.d_l0 = D->d.first_layer;
      a.s_blk_off = src_bt->blk_off;
      a.s_blk_ids = src_bt->blk_ids;
      a.d_blk_off = dst_bt->blk_off;
      a.d_blk_ids = dst_bt->blk_ids;
      a.d_blk_req = dst_bt->blk_req;
      a.tok_off = dst_bt->tok_off;
      a.f_hp = make_fastdiv(Hp);
      a.f_hde = make_fastdiv((uint32_t)a.Hd_eff);
      a.f_bl = make_fastdiv((uint32_t)std::max<int64_t>(dst_bt->total_blocks, 1));
      if (dst_bt->total_blocks == 0 || le == lb) return KV_OK;
      const uint64_t per_layer = (uint64_t)n_dst * dst_bt->total_blocks * (a.kv1 ? 1 : 2) * a.Hd_eff;
      const int32_t step = (int32_t)std::max<uint64_t>(1, kMaxChunks / std::max<uint64_t>(per_layer, 1));
      // head_dim-major 2-byte source tiles of 16 slots into D's rows: whole tiles through TMA
      // (k_convert_tb), unless KVX_TB=0
      TbArgs tb;
      memset(&tb, 0, sizeof(tb));
      bool use_tb = false;
      {
        const char* tb_env = getenv("KVX_TB");
        const int32_t Dm = S->d.head_dim;
        encode_tiled_fn enc = encode_fn();
        // x-packed with x = 16 bytes: 2-byte sources only (bf16 K pool -> e4m3 0.90 -> 0.98 of copy;
        // 1-byte sources measured slower than k_convert_tr8: e4m3 -> bf16 0.89 vs 0.96, fnuz 0.76 vs 0.88)
        // x-packed e4m3fn -> e4m3fnuz tiles (x = 16 codes) go through tb's per-item code tables:
        // K pool 0.627 (k_convert_tr8, arithmetic fnuz encode) -> 0.827; the other direction
        // stays on tr8, whose folded fnuz decode is cheaper there (0.872 vs 0.772 through tb;
        // profiles/r02/tb_xpacked_fp8_ab.txt).  KVX_TB_X8=0: tr8 for both
        const bool fp8_pair = S->d.dtype == KV_F8E4M3 && D->d.dtype == KV_F8E4M3FNUZ;
        const char* tbx_env = getenv("KVX_TB_X8");
        const bool xp16 = st == 2 && (1 << S->dk) * S->elem_bytes == 16 &&
                          (S->elem_bytes == 2 || (fp8_pair && !(tbx_env && atoi(tbx_env) == 0)));
        use_tb = use_tr8 && (st == 1 || xp16) && dt == 0 && S->elem_bytes <= 2 && S->d.block_size == 16 &&
                 D->d.block_size == 16 && (Dm == 64 || Dm == 128 || Dm == 256) && enc && !(tb_env && atoi(tb_env) == 0);
        // two heads per item (one TMA box) when a head's source AND destination tiles are
        // <= 2 KB (fp8 -> fp8, or D = 64 2-byte) and the item's two heads sit next to each
        // other in the source, belong to the same P rank and map to adjacent D heads: the
        // per-item pipeline cost is then paid per 4 KB (c4-pair V pool, profiles/r02/tb_hpi_ab.txt:
        // fnuz -> e4m3 0.657 -> 0.705, e4m3 -> fnuz 0.665 -> 0.755; e4m3 -> bf16, whose
        // destination tile is 4 KB, 0.951 -> 0.901, so it stays at one head).  KVX_TB_HPI=1: off
        const int64_t head_tile = (int64_t)Dm * 16 * S->elem_bytes, dst_tile = (int64_t)Dm * 16 * D->elem_bytes;
        const char* hpi_env = getenv("KVX_TB_HPI");
        int32_t hpi = ((st == 1 || xp16) && head_tile <= 2048 && dst_tile <= 2048 && !(hpi_env && atoi(hpi_env) < 2) &&
                       a.Hd_eff % 2 == 0 && Hp % 2 == 0 && Hd % 2 == 0) ? 2 : 1;
        for (int i = 0; i < n_src && hpi == 2; ++i)
          if (src[i]->stride[KV_AX_HEAD] * src[i]->elem_bytes != head_tile) hpi = 1;
        for (int i = 0; i < n_dst && hpi == 2; ++i)
          if (a.hq_off[i] % 2) hpi = 1;
        for (int i = 0; i < n_src && use_tb; ++i) {
          const uint64_t rows = src[i]->pool_bytes / 128;
          if (src[i]->pool_bytes % 128 || rows >= (1ull << 31) || !ptr_aligned(src_pools[i], 16)) {
            use_tb = false;
            break;
          }
          cuuint64_t dims[2] = {128, (cuuint64_t)rows};
          cuuint64_t strides[1] = {128};
          cuuint32_t box[2] = {128, (cuuint32_t)(Dm * S->elem_bytes / 8 * hpi)};   // hpi x 16 x D elements / 128 B
          cuuint32_t estr[2] = {1, 1};
          if (enc(&tb.maps[i], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(src_pools[i]), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            use_tb = false;
        }
        tb.mode = st == 1 ? 1 : 2;
        const char* tl_env = getenv("KVX_TB_LUT");
        tb.lut = tl_env ? atoi(tl_env) : 1;
        tb.hpi = hpi;
        tb.tile_rows = Dm * S->elem_bytes / 8 * hpi;
        // tiles in flight per CTA: 64 KB for 2-byte sources (c4-pair V pool bf16 -> e4m3: 0.90 at
        // 32 KB, 0.97 at 64 KB), 32 KB for 1-byte ones (the 2-KB tiles want more CTAs, hence
        // less shared memory each: e4m3 0.91 at 32 KB, 0.72 at 64 KB); KVX_TB_STAGE_KB overrides
        const char* kb_env = getenv("KVX_TB_STAGE_KB");
        const int32_t kb = kb_env ? std::max(8, atoi(kb_env)) : (S->elem_bytes == 2 ? 64 : 32);
        tb.stages = std::max(kTbConsumers, std::min(32, kb * 1024 / (tb.tile_rows * 128)));
      }
      for (int32_t l0 = lb; l0 < le; l0 += step) {
        const int32_t l1 = std::min(le, l0 + step);
        a.lb = l0;
        a.Lc = l1 - l0;
        a.f_l = make_fastdiv((uint32_t)a.Lc);
        a.n_items = (uint32_t)(per_layer * (uint64_t)a.Lc);
        cudaError_t e;
        if (use_tb) {
          t_last_kernel = "k_convert_tb";
          tb.c = a;
          tb.c.n_items = a.n_items / (uint32_t)tb.hpi;
          tb.c.f_hde = make_fastdiv((uint32_t)(a.Hd_eff / tb.hpi));
          e = launch_convert_tb(tb, S->d.dtype, D->d.dtype, (cudaStream_t)stream);
        } else if (use_tr8) {
          t_last_kernel = "k_convert_tr8";
          e = launch_convert_tr8(a, S->d.dtype, D->d.dtype, (cudaStream_t)stream);
        } else {
          t_last_kernel = "k_convert_tr";
          e = launch_convert_tr(a, S->d.dtype, D->d.dtype, (cudaStream_t)stream);
        }
        if (e != cudaSuccess) return cuda_fail(e, "kv_convert_reshard: launch");
      }
      return KV_OK;
    }
  }
  bool fast = rows_side(S, &a.s_ck, &a.s_chs) && rows_side(D, &a.d_ck, &a.d_chs);
  a.split = (S->dk || D->dk) ? 1 : 0;
  for (int i = 0; i < n_src && fast; ++i) fast = ptr_aligned(src_pools[i], 16);
  for (int i = 0; i < n_dst && fast; ++i) fast = ptr_aligned(dst_pools[i], 16);
  const int vec = fast ? 8 : 1;
  for (int ax = 0; ax < 6; ++ax) {
    a.ss[ax] = S->stride[ax];
    a.ds[ax] = D->stride[ax];
  }
  a.Hp = Hp;
  a.Hd = Hd;
  a.D = S->d.head_dim;
  a.Bp = S->d.block_size;
  a.Bd = D->d.block_size;
  a.s_l0 = S->d.first_layer;
  a.d_l0 = D->d.first_layer;
  a.s_blk_off = src_bt->blk_off;
  a.s_blk_ids = src_bt->blk_ids;
  a.d_blk_off = dst_bt->blk_off;
  a.d_blk_ids = dst_bt->blk_ids;
  a.d_blk_req = dst_bt->blk_req;
  a.tok_off = dst_bt->tok_off;
  a.slot_inner = slot_inner_of(D);
  const uint32_t ndch = (uint32_t)(a.D / vec);
  a.f_dch = make_fastdiv(ndch);
  a.f_in0 = make_fastdiv(a.slot_inner ? a.Bd : a.Hd_eff);
  a.f_in1 = make_fastdiv(a.slot_inner ? a.Hd_eff : a.Bd);
  a.f_hp = make_fastdiv(Hp);
  a.f_bp = make_fastdiv(a.Bp);
  a.f_bd = make_fastdiv(a.Bd);
  a.f_bl = make_fastdiv((uint32_t)std::max<int64_t>(dst_bt->total_blocks, 1));
  a.f_cpr = make_fastdiv(ndch);
  a.f_nd = make_fastdiv((uint32_t)n_dst);
  if (dst_bt->total_blocks == 0 || le == lb) return KV_OK;
  if (fast && !a.split && !(nt && S->d.dtype != D->d.dtype)) {  // notify counts requests in the row kernel
    bool used = false;
    if ((st = try_tile_copy(n_src, src, src_pools, src_bt, n_dst, dst, dst_pools, dst_bt, lb, le, stream, share,
                            &used)) != KV_OK)
      return st;
    if (used) {
      // (t_last_kernel set by try_tile_copy: k_tile_copy or k_tile_cast)
      return KV_OK;
    }
  }
  // per-layer chunk count; split the layer range so each launch stays under 2^31 chunks
  // (element-wise kernel: 32-bit chunk decode) or 2^31 rows (row kernel: 32-bit item decode;
  // the whole c4 batch, 2.7 G chunks, is one launch)
  const uint64_t per_layer = (uint64_t)n_dst * dst_bt->total_blocks * (a.kv1 ? 1 : 2) * a.Hd_eff * a.Bd * ndch;
  const uint64_t per_layer_units = vec == 8 ? per_layer / ndch : per_layer;
  int32_t step = (int32_t)std::max<uint64_t>(1, kMaxChunks / std::max<uint64_t>(per_layer_units, 1));
  if (per_layer_units > kMaxChunks) return fail(KV_EUNSUPPORTED, "kv_convert_reshard: one layer exceeds 2^31 chunks");
  // fp8 -> other fp8 (e4m3fnuz <-> e4m3fn): 128-B magnitude code tables in shared memory
  // (k_requant_rows), layer sub-ranges sized so a launch's tables stay bounded.  Measured on
  // the c4-pair shape (profiles/r02/requant_lut.txt): e4m3fn -> e4m3fnuz 0.909 of copy vs
  // 0.686 for the arithmetic row kernel, e4m3fnuz -> e4m3fn 0.872 vs 0.841 -- tables both ways
  // by default (KVX_LUT=1 or 2); KVX_LUT=0 forces the arithmetic row kernel
  {
    const char* lut_env = getenv("KVX_LUT");
    const int lut_mode = lut_env ? atoi(lut_env) : 1;
    const bool dual = fp8(S->d.dtype) && fp8(D->d.dtype) && S->d.dtype != D->d.dtype;
    const bool want = lut_mode != 0;
    const uint32_t tab_per_layer = (uint32_t)n_dst * (a.kv1 ? 1u : 2u) * (uint32_t)a.Hd_eff;
    if (vec == 8 && !a.split && dual && !nt && want && tab_per_layer <= kRequantMaxTables && S->d.head_dim >= 16) {
      const int32_t lstep = std::min<int32_t>(step, (int32_t)(kRequantMaxTables / tab_per_layer));
      for (int32_t l0 = lb; l0 < le; l0 += lstep) {
        const int32_t l1 = std::min(le, l0 + lstep);
        a.lb = l0;
        a.Lc = l1 - l0;
        a.f_l = make_fastdiv((uint32_t)a.Lc);
        a.total64 = per_layer * (uint64_t)a.Lc;
        a.total = (uint32_t)a.total64;
        t_last_kernel = "k_requant_rows";
        cudaError_t e = launch_requant(a, S->d.dtype, D->d.dtype, (cudaStream_t)stream);
        if (e != cudaSuccess) return cuda_fail(e, "kv_convert_reshard: requant launch");
      }
      return KV_OK;
    }
  }
  if (nt && vec == 8 && step >= le - lb) {
    // per-request completion counted inside the (single) row-kernel launch
    cudaError_t e = launch_notify_init(*nt, dst_bt->blk_off, dst_bt->n_req, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "kv_convert_reshard_notify: init");
    a.req_cnt = nt->counters;
    a.req_flag = nt->flags;
    a.req_ns = nt->ns;
    a.req_epoch = nt->epoch;
    if (notified) *notified = true;
  }
  for (int32_t l0 = lb; l0 < le; l0 += step) {
    const int32_t l1 = std::min(le, l0 + step);
    a.lb = l0;
    a.Lc = l1 - l0;
    a.f_l = make_fastdiv((uint32_t)a.Lc);
    a.total64 = per_layer * (uint64_t)a.Lc;
    a.total = (uint32_t)a.total64;  // element-wise kernel only (< 2^31 there)
    t_last_kernel = vec == 8 ? "k_convert_rows" : "k_convert";
    cudaError_t e = launch_convert(a, vec, S->d.dtype, D->d.dtype, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "kv_convert_reshard: launch");
  }
  return KV_OK;
}
}  // namespace

extern "C" {

kv_status kv_convert_reshard(int32_t n_src, const kv_layout* const* src, const void* const* src_pools,
                             const kv_batch* src_bt, int32_t n_dst, const kv_layout* const* dst,
                             void* const* dst_pools, const kv_batch* dst_bt, int32_t lb, int32_t le,
                             kv_stream stream) {
  NvtxRange nvtx_("kv_convert_reshard", lb);
  return convert_impl(n_src, src, src_pools, src_bt, n_dst, dst, dst_pools, dst_bt, lb, le, stream, false);
}

kv_status kv_convert_share(const kv_layout* src, const void* src_pool, const kv_batch* src_bt, int32_t n_dst,
                           const kv_layout* const* dst, void* const* dst_pools, const kv_batch* dst_bt, int32_t lb,
                           int32_t le, kv_stream stream) {
  NvtxRange nvtx_("kv_convert_share", lb);
  const kv_layout* s1[1] = {src};
  const void* p1[1] = {src_pool};
  return convert_impl(1, s1, p1, src_bt, n_dst, dst, dst_pools, dst_bt, lb, le, stream, true);
}

kv_status kv_convert_reshard_notify(int32_t n_src, const kv_layout* const* src, const void* const* src_pools,
                                    const kv_batch* src_bt, int32_t n_dst, const kv_layout* const* dst,
                                    void* const* dst_pools, const kv_batch* dst_bt, int32_t lb, int32_t le,
                                    uint32_t* counters, uint32_t* done_flags, uint64_t* done_ns, uint32_t epoch,
                                    kv_stream stream) {
  NvtxRange nvtx_("kv_convert_reshard_notify", lb);
  if (!dst_bt || (dst_bt->n_req > 0 && (!counters || !done_flags)))
    return fail(KV_EINVAL, "kv_convert_reshard_notify: null counters / flags");
  Notify nt{counters, done_flags, done_ns, epoch};
  bool notified = false;
  kv_status st = convert_impl(n_src, src, src_pools, src_bt, n_dst, dst, dst_pools, dst_bt, lb, le, stream, false,
                              &nt, &notified);
  if (st != KV_OK || notified) return st;
  // another kernel (or several launches) did the work: every request completes with it
  cudaError_t e = launch_notify_all(nt, dst_bt->n_req, (cudaStream_t)stream);
  return e == cudaSuccess ? KV_OK : cuda_fail(e, "kv_convert_reshard_notify: completion");
}

kv_status kv_timestamp(uint64_t* out, kv_stream stream) {
  if (!out) return fail(KV_EINVAL, "kv_timestamp: null pointer");
  cudaError_t e = launch_timestamp(out, (cudaStream_t)stream);
  return e == cudaSuccess ? KV_OK : cuda_fail(e, "kv_timestamp");
}

}  // extern "C"

namespace kvx {
// kv_compute_scales, optionally restricted to the D heads one source rank holds (share:
// n_src == 1; the dynamic-scale staged pull of a TP merge, where every P rank owns the
// scales of its own heads) and optionally storing the finished scales a second time into
// `peer` (D's array, peer-mapped) -- see kv_stage.
kv_status compute_scales_impl(int32_t n_src, const kv_layout* const* src, const void* const* src_pools,
                              const kv_batch* src_bt, const kv_layout* dst, float* out_scales, int32_t lb, int32_t le,
                              kv_stream stream, bool share, float* peer) {
  if (n_src < 1 || n_src > KVX_MAX_RANKS || !src || !src_pools || !dst || !out_scales)
    return fail(KV_EINVAL, "kv_compute_scales: bad argument");
  for (int i = 0; i < n_src; ++i)
    if (!src[i] || !src_pools[i]) return fail(KV_EINVAL, "kv_compute_scales: null source layout/pool");
  const kv_layout* S = src[0];
  for (int i = 1; i < n_src; ++i)
    if (!same_instance(src[i], S)) return fail(KV_ESHAPE, "kv_compute_scales: source layouts differ beyond rank");
  kv_status st;
  if (S->d.tp_degree > KVX_MAX_RANKS) return fail(KV_EUNSUPPORTED, "kv_compute_scales: tp degree above 16");
  if ((st = same_model(S, dst)) != KV_OK) return st;
  if ((st = check_layers(S, lb, le)) != KV_OK) return st;
  if ((st = check_layers(dst, lb, le)) != KV_OK) return st;
  if ((st = check_batch(src_bt, S, "src_bt")) != KV_OK) return st;
  if (src_bt->n_req > 0 && !src_bt->tok_req) return fail(KV_EINVAL, "kv_compute_scales: src_bt has no token map");
  AmaxArgs a;
  memset(&a, 0, sizeof(a));
  if ((st = kv_pair(S, dst, &a.kv1, &a.c0)) != KV_OK) return st;
  a.s_dk = S->dk;
  for (int i = 0; i < KVX_MAX_RANKS; ++i) a.src_of_p[i] = -1;
  for (int i = 0; i < n_src; ++i) {
    const int p = src[i]->d.tp_rank;
    if (a.src_of_p[p] != -1) return fail(KV_EINVAL, "kv_compute_scales: source rank listed twice");
    if (fp8(S->d.dtype) && !src[i]->d.scales) return fail(KV_EINVAL, "kv_compute_scales: fp8 source without scales");
    a.src_of_p[p] = (int8_t)i;
    a.src[i] = static_cast<const uint8_t*>(src_pools[i]);
    a.sscale[i] = src[i]->d.scales;
  }
  const int32_t Hp = S->h_local, Hd = dst->h_local, q = dst->d.tp_rank;
  int32_t h0 = q * Hd, h1 = (q + 1) * Hd;
  if (share) {
    if (n_src != 1) return fail(KV_EINVAL, "kv_compute_scales: a share has one source");
    h0 = std::max(h0, S->d.tp_rank * Hp);
    h1 = std::min(h1, (S->d.tp_rank + 1) * Hp);
    if (h1 <= h0) return fail(KV_ESHAPE, "kv_compute_scales: the source rank holds none of the D rank's heads");
  }
  for (int32_t h = h0; h < h1; ++h)
    if (a.src_of_p[h / Hp] < 0)
      return fail(KV_ESHAPE, "kv_compute_scales: missing source shard for P rank " + std::to_string(h / Hp));
  a.hq0 = h0 - q * Hd;
  a.nhq = h1 - h0;
  a.peer = peer;
  for (int ax = 0; ax < 6; ++ax) a.ss[ax] = S->stride[ax];
  a.Hp = Hp;
  a.Hd = Hd;
  a.D = S->d.head_dim;
  a.q = q;
  a.s_l0 = S->d.first_layer;
  a.d_l0 = dst->d.first_layer;
  a.lb = lb;
  a.Lc = le - lb;
  a.s_blk_off = src_bt->blk_off;
  a.s_blk_ids = src_bt->blk_ids;
  a.tok_off = src_bt->tok_off;
  a.tok_req = src_bt->tok_req;
  a.amax_bits = reinterpret_cast<uint32_t*>(out_scales);
  a.qmax = dst->d.dtype == KV_F8E4M3FNUZ ? 240.0f : 448.0f;
  a.n_tok = (uint32_t)src_bt->total_tokens;
  const uint32_t ntg = (a.n_tok + 31u) / 32u;
  a.f_tg = make_fastdiv(std::max<uint32_t>(ntg, 1));
  a.f_hd = make_fastdiv((uint32_t)a.nhq);
  a.f_bp = make_fastdiv((uint32_t)S->d.block_size);
  a.f_hp = make_fastdiv((uint32_t)Hp);
  const uint64_t items = (uint64_t)ntg * a.nhq * (a.kv1 ? 1 : 2) * (uint64_t)(le - lb);
  if (items > kMaxChunks) return fail(KV_EUNSUPPORTED, "kv_compute_scales: batch too large for one call");
  a.n_items = (uint32_t)items;
  // row path: head_dim innermost with 16-B rows and aligned pools (every source)
  const int64_t rb = (int64_t)a.D * S->elem_bytes;
  a.rows = S->stride[KV_AX_DIM] == 1 && rb % 16 == 0 && (rb / 16 & (rb / 16 - 1)) == 0 && rb / 16 <= 32;
  for (int i = 0; i < n_src; ++i) a.rows = a.rows && ptr_aligned(src_pools[i], 16);
  if (a.rows)
    while ((1 << a.cpr_shift) < rb / 16) ++a.cpr_shift;
  if (le == lb) return KV_OK;
  cudaError_t e = launch_amax(a, S->d.dtype, out_scales, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "kv_compute_scales: launch");
  return KV_OK;
}
}  // namespace kvx

extern "C" {

kv_status kv_compute_scales(int32_t n_src, const kv_layout* const* src, const void* const* src_pools,
                            const kv_batch* src_bt, const kv_layout* dst, float* out_scales, int32_t lb, int32_t le,
                            kv_stream stream) {
  return compute_scales_impl(n_src, src, src_pools, src_bt, dst, out_scales, lb, le, stream, false, nullptr);
}

int32_t kv_wire_dtype(const kv_layout* s, const kv_layout* d) {
  if (!s || !d) return -1;
  return dtype_bytes(d->d.dtype) <= dtype_bytes(s->d.dtype) ? d->d.dtype : s->d.dtype;
}

size_t kv_wire_bytes(const kv_layout* s, const kv_layout* d, int64_t total_tokens, int32_t lb, int32_t le) {
  if (!s || !d || le < lb || total_tokens < 0) return 0;
  int32_t hb, he;
  head_overlap(s, d, &hb, &he);
  if (he <= hb) return 0;
  static const int mask[3] = {3, 1, 2};
  const int m = (s->d.kv_part >= 0 && s->d.kv_part <= 2 && d->d.kv_part >= 0 && d->d.kv_part <= 2)
                    ? (mask[s->d.kv_part] & mask[d->d.kv_part]) : 0;
  const size_t nkv = m == 3 ? 2 : (m ? 1 : 0);  // the K/V both pools hold
  return nkv * (size_t)(le - lb) * (size_t)(he - hb) * (size_t)total_tokens * (size_t)s->d.head_dim *
         (size_t)dtype_bytes(kv_wire_dtype(s, d));
}

}  // extern "C"

namespace {
// kv_pack's validation and argument block (shared with kv_stage's one-launch path): *vec = 8
// for the row kernel, 1 for the element-wise one; *need = the chunk's wire bytes (0: nothing)
kv_status pack_args(const kv_layout* s, const void* src_pool, const kv_batch* src_bt, const kv_layout* d, int32_t lb,
                    int32_t le, const void* wire, size_t wire_bytes, PackArgs* out, int* vec_out, size_t* need_out) {
  if (!s || !d || !src_pool || !wire) return fail(KV_EINVAL, "kv_pack: null argument");
  kv_status st;
  if ((st = same_model(s, d)) != KV_OK) return st;
  if ((st = check_layers(s, lb, le)) != KV_OK) return st;
  if ((st = check_layers(d, lb, le)) != KV_OK) return st;
  if ((st = check_batch(src_bt, s, "src_bt")) != KV_OK) return st;
  if ((st = scales_ok(s, d)) != KV_OK) return st;
  int32_t hb, he;
  head_overlap(s, d, &hb, &he);
  if (he <= hb) return fail(KV_ESHAPE, "kv_pack: source and destination ranks share no heads");
  const size_t need = kv_wire_bytes(s, d, src_bt->total_tokens, lb, le);
  if (wire_bytes < need)
    return fail(KV_ESHAPE, "kv_pack: wire buffer " + std::to_string(wire_bytes) + " < " + std::to_string(need));
  *need_out = need;
  if (need == 0) return KV_OK;
  if (src_bt->n_req > 0 && !src_bt->tok_req) return fail(KV_EINVAL, "kv_pack: src_bt has no token map");
  PackArgs& a = *out;
  memset(&a, 0, sizeof(a));
  if ((st = kv_pair(s, d, &a.kv1, &a.c0)) != KV_OK) return st;
  a.s_dk = s->dk;
  const int vec = (fast_ok(s) && ptr_aligned(src_pool, 16) && ptr_aligned(wire, 16)) ? 8 : 1;
  *vec_out = vec;
  a.src = static_cast<const uint8_t*>(src_pool);
  a.wire = static_cast<uint8_t*>(const_cast<void*>(wire));
  a.sscale = s->d.scales;
  a.dscale = d->d.scales;
  for (int ax = 0; ax < 6; ++ax) a.ss[ax] = s->stride[ax];
  a.Hp = s->h_local;
  a.Hd = d->h_local;
  a.D = s->d.head_dim;
  a.Bp = s->d.block_size;
  a.s_l0 = s->d.first_layer;
  a.d_l0 = d->d.first_layer;
  a.lb = lb;
  a.Lc = le - lb;
  a.p = s->d.tp_rank;
  a.q = d->d.tp_rank;
  a.hb = hb;
  a.nh = he - hb;
  a.s_blk_off = src_bt->blk_off;
  a.s_blk_ids = src_bt->blk_ids;
  a.tok_off = src_bt->tok_off;
  a.tok_req = src_bt->tok_req;
  const uint32_t ndch = (uint32_t)(a.D / vec);
  a.f_dch = make_fastdiv(ndch);
  a.f_tok = make_fastdiv((uint32_t)src_bt->total_tokens);
  a.f_nh = make_fastdiv((uint32_t)a.nh);
  a.f_bp = make_fastdiv((uint32_t)a.Bp);
  const uint64_t total = (uint64_t)a.Lc * (a.kv1 ? 1 : 2) * a.nh * src_bt->total_tokens * ndch;
  if (total > kMaxChunks) return fail(KV_EUNSUPPORTED, "kv_pack: more than 2^31 chunks in one call; split layers");
  a.total = (uint32_t)total;
  a.f_l = make_fastdiv((uint32_t)a.Lc);
  return KV_OK;
}
}  // namespace

extern "C" {

kv_status kv_pack(const kv_layout* s, const void* src_pool, const kv_batch* src_bt, const kv_layout* d, int32_t lb,
                  int32_t le, void* wire, size_t wire_bytes, kv_stream stream) {
  NvtxRange nvtx_("kv_pack", lb);
  PackArgs a;
  int vec = 1;
  size_t need = 0;
  kv_status st = pack_args(s, src_pool, src_bt, d, lb, le, wire, wire_bytes, &a, &vec, &need);
  if (st != KV_OK || need == 0) return st;
  t_last_kernel = vec == 8 ? "k_pack_rows" : "k_pack";
  cudaError_t e = launch_pack(a, vec, s->d.dtype, kv_wire_dtype(s, d), (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "kv_pack: launch");
  return KV_OK;
}

kv_status kv_unpack(const kv_layout* s, const kv_layout* d, void* dst_pool, const kv_batch* dst_bt, int32_t lb,
                    int32_t le, const void* wire, size_t wire_bytes, kv_stream stream) {
  NvtxRange nvtx_("kv_unpack", lb);
  if (!s || !d || !dst_pool || !wire) return fail(KV_EINVAL, "kv_unpack: null argument");
  kv_status st;
  if ((st = same_model(s, d)) != KV_OK) return st;
  if ((st = check_layers(s, lb, le)) != KV_OK) return st;
  if ((st = check_layers(d, lb, le)) != KV_OK) return st;
  if ((st = check_batch(dst_bt, d, "dst_bt")) != KV_OK) return st;
  if ((st = scales_ok(s, d)) != KV_OK) return st;
  int32_t hb, he;
  head_overlap(s, d, &hb, &he);
  if (he <= hb) return fail(KV_ESHAPE, "kv_unpack: source and destination ranks share no heads");
  const size_t need = kv_wire_bytes(s, d, dst_bt->total_tokens, lb, le);
  if (wire_bytes < need)
    return fail(KV_ESHAPE, "kv_unpack: wire buffer " + std::to_string(wire_bytes) + " < " + std::to_string(need));
  if (dst_bt->total_blocks == 0 || le == lb) return KV_OK;
  UnpackArgs a;
  memset(&a, 0, sizeof(a));
  if ((st = kv_pair(s, d, &a.kv1, &a.c0)) != KV_OK) return st;
  a.d_dk = d->dk;
  const int vec = (fast_ok(d) && ptr_aligned(dst_pool, 16) && ptr_aligned(wire, 16)) ? 8 : 1;
  a.dst = static_cast<uint8_t*>(dst_pool);
  a.wire = static_cast<const uint8_t*>(wire);
  a.sscale = s->d.scales;
  a.dscale = d->d.scales;
  for (int ax = 0; ax < 6; ++ax) a.ds[ax] = d->stride[ax];
  a.Hp = s->h_local;
  a.Hd = d->h_local;
  a.D = d->d.head_dim;
  a.Bd = d->d.block_size;
  a.s_l0 = s->d.first_layer;
  a.d_l0 = d->d.first_layer;
  a.lb = lb;
  a.Lc = le - lb;
  a.p = s->d.tp_rank;
  a.q = d->d.tp_rank;
  a.hb = hb;
  a.nh = he - hb;
  a.total_tokens = dst_bt->total_tokens;
  a.d_blk_off = dst_bt->blk_off;
  a.d_blk_ids = dst_bt->blk_ids;
  a.d_blk_req = dst_bt->blk_req;
  a.tok_off = dst_bt->tok_off;
  a.slot_inner = slot_inner_of(d);
  const uint32_t ndch = (uint32_t)(a.D / vec);
  a.f_dch = make_fastdiv(ndch);
  a.f_in0 = make_fastdiv(a.slot_inner ? a.Bd : a.nh);
  a.f_in1 = make_fastdiv(a.slot_inner ? a.nh : a.Bd);
  a.f_l = make_fastdiv((uint32_t)a.Lc);
  a.f_bd = make_fastdiv((uint32_t)a.Bd);
  const uint64_t total = (uint64_t)dst_bt->total_blocks * a.Lc * (a.kv1 ? 1 : 2) * a.nh * a.Bd * ndch;
  if (total > kMaxChunks) return fail(KV_EUNSUPPORTED, "kv_unpack: more than 2^31 chunks in one call; split layers");
  a.total = (uint32_t)total;
  a.f_bl = make_fastdiv((uint32_t)dst_bt->total_blocks);
  t_last_kernel = vec == 8 ? "k_unpack_rows" : "k_unpack";
  cudaError_t e = launch_unpack(a, vec, kv_wire_dtype(s, d), d->d.dtype, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "kv_unpack: launch");
  return KV_OK;
}

}  // extern "C"

namespace kvx {

// kv_pull_staged's one-launch path (k_pull_rows): taken when wire and pool share the dtype,
// head_dim is innermost with 16-B aligned rows, the ring slots are 16-B aligned and every
// source overlaps the destination in the same number of heads.  Otherwise *used = false.
kv_status pull_rows_fast(int32_t n_src, const kv_layout* const* src, const void* const* rings, int32_t R,
                         const kv_layout* d, void* dst_pool, const kv_batch* dst_bt, const uint32_t* const* ready,
                         uint32_t* const* freef, uint32_t* counters, uint32_t seq0, const ChunkPlan& plan,
                         uint64_t timeout_ns, int32_t* err, kv_stream stream, bool* used) {
  const int32_t lb = plan.lb, le = plan.le, step = plan.step;
  *used = false;
  if (!counters || n_src > KVX_MAX_RANKS || R > KVX_MAX_RING || !fast_ok(d) || !ptr_aligned(dst_pool, 16)) return KV_OK;
  if (getenv("KVX_PULL_CHUNKED")) return KV_OK;  // A/B switch: per-chunk launches
  PullArgs a;
  memset(&a, 0, sizeof(a));
  if (kv_pair(src[0], d, &a.kv1, &a.c0) != KV_OK) return KV_OK;  // the chunked path reports it
  int32_t nh = -1;
  for (int i = 0; i < n_src; ++i) {
    if (kv_wire_dtype(src[i], d) != d->d.dtype) return KV_OK;
    int32_t hb, he;
    head_overlap(src[i], d, &hb, &he);
    if (nh >= 0 && he - hb != nh) return KV_OK;
    nh = he - hb;
    a.hb[i] = hb;
    for (int b = 0; b < R; ++b) {
      const void* r = rings[(size_t)i * R + b];
      if (!ptr_aligned(r, 16)) return KV_OK;
      a.ring[i][b] = static_cast<const uint8_t*>(r);
    }
    a.ready[i] = ready[i];
    a.freef[i] = freef[i];
  }
  if (dst_bt->total_blocks == 0 || le == lb) return KV_OK;  // the chunked path handles the flags
  a.dst = static_cast<uint8_t*>(dst_pool);
  a.counters = counters;
  a.err = err;
  a.timeout_ns = timeout_ns;
  for (int ax = 0; ax < 6; ++ax) a.ds[ax] = d->stride[ax];
  a.nsrc = n_src;
  a.R = R;
  a.Hd = d->h_local;
  a.D = d->d.head_dim;
  a.Bd = d->d.block_size;
  a.lb = lb;
  a.le = le;
  a.step = step;
  a.nchunks = plan.n;
  a.nramp = plan.nramp;
  a.rsum = plan.rsum;
  for (int32_t k = 0; k < plan.nramp; ++k) {
    int32_t l0, l1;
    plan.bounds(k, &l0, &l1);
    a.ramp_l0[k] = l0;
  }
  a.q = d->d.tp_rank;
  a.nh = nh;
  a.d_l0 = d->d.first_layer;
  a.seq0 = seq0;
  a.total_tokens = dst_bt->total_tokens;
  a.d_blk_off = dst_bt->blk_off;
  a.d_blk_ids = dst_bt->blk_ids;
  a.d_blk_req = dst_bt->blk_req;
  a.tok_off = dst_bt->tok_off;
  a.f_src = make_fastdiv((uint32_t)n_src);
  a.slot_inner = slot_inner_of(d);
  a.n_blk = (uint32_t)dst_bt->total_blocks;
  const uint64_t items = (uint64_t)n_src * (a.kv1 ? 1 : 2) * (uint64_t)step * dst_bt->total_blocks * (uint64_t)a.Bd *
                         (uint64_t)nh;
  if (items > kMaxChunks) return KV_OK;
  a.spin_ns = 128u;
  if (kv_status pst = ensure_preloaded(); pst != KV_OK) return pst;
  t_last_kernel = "k_pull_rows";
  cudaError_t e = launch_pull_rows(a, d->d.dtype, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "kv_pull_staged: launch");
  *used = true;
  return KV_OK;
}

// kv_stage's one-launch path (k_stage_rows, opt-in): one destination rank, no dynamic scales, the
// row machinery (head_dim innermost, 16-B aligned pool and ring slots), a 2- / 4-byte source
// and a narrower-or-equal wire.  The counters live in stream-ordered scratch (freed on the
// stream after the launch).  Otherwise *used = false and kv_stage enqueues per chunk.
kv_status stage_rows_fast(const kv_layout* src, const void* src_pool, const kv_batch* src_bt, const kv_layout* dst,
                          void* const* rings, int32_t R, size_t slot_bytes, uint32_t* ready, const uint32_t* freef,
                          uint32_t seq0, const ChunkPlan& plan, uint64_t timeout_ns, int32_t* err, kv_stream stream,
                          bool* used) {
  *used = false;
  // opt-in (KVX_STAGE_PERSISTENT=1): on the c4 pair it measured no faster than the per-chunk
  // launches (batch-1: 0.261 vs 0.248 ms; full batch: equal), DESIGN.md §5
  const char* on = getenv("KVX_STAGE_PERSISTENT");
  if (!on || !*on || *on == '0' || R > KVX_MAX_RING || plan.n <= 0) return KV_OK;
  const int32_t wdt = kv_wire_dtype(src, dst), sdt = src->d.dtype;
  if (!(sdt == KV_F32 || sdt == KV_F16 || sdt == KV_BF16) || wdt == KV_F32 || dtype_bytes(wdt) > dtype_bytes(sdt))
    return KV_OK;
  StageArgs a;
  memset(&a, 0, sizeof(a));
  for (int b = 0; b < R; ++b) {
    if (!ptr_aligned(rings[b], 16)) return KV_OK;
    a.ring[b] = static_cast<uint8_t*>(rings[b]);
  }
  int vec = 1;
  size_t need = 0;
  int32_t l0, l1;
  plan.bounds(0, &l0, &l1);  // validates the pair and builds the pack block (lb / wire per chunk in-kernel)
  kv_status st = pack_args(src, src_pool, src_bt, dst, l0, l1, rings[0], slot_bytes, &a.p, &vec, &need);
  if (st != KV_OK) return st;
  if (vec != 8 || need == 0) return KV_OK;
  {  // the last chunk too (chunks are contiguous: first and last in range = all in range)
    PackArgs last;
    int v2 = 1;
    size_t n2 = 0;
    plan.bounds(plan.n - 1, &l0, &l1);
    if ((st = pack_args(src, src_pool, src_bt, dst, l0, l1, rings[0], slot_bytes, &last, &v2, &n2)) != KV_OK) return st;
  }
  const uint64_t per_layer = (uint64_t)(a.p.kv1 ? 1 : 2) * a.p.nh * (((uint64_t)src_bt->total_tokens + 31) / 32);
  if (per_layer * (uint64_t)plan.step > kMaxChunks) return KV_OK;
  a.ready = ready;
  a.freef = freef;
  a.err = err;
  a.timeout_ns = timeout_ns;
  a.spin_ns = 128u;
  a.seq0 = seq0;
  a.R = R;
  a.nchunks = plan.n;
  a.lb = plan.lb;
  a.le = plan.le;
  a.step = plan.step;
  a.nramp = plan.nramp;
  a.rsum = plan.rsum;
  for (int32_t k = 0; k < plan.nramp; ++k) {
    plan.bounds(k, &l0, &l1);
    a.ramp_l0[k] = l0;
    a.ramp_nl[k] = l1 - l0;
  }
  if (kv_status pst = ensure_preloaded(); pst != KV_OK) return pst;
  {  // keep freed scratch in the device's default pool across synchronizations (the default
     // release threshold 0 would hand it back to the driver at every sync)
    static std::atomic<uint64_t> pooled{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !(pooled.load() & (1ull << dev))) {
      cudaMemPool_t pool;
      uint64_t thr = 64ull << 20;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      pooled.fetch_or(1ull << dev);
    }
  }
  void* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, (2 * (size_t)plan.n + 1) * sizeof(uint32_t), (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "kv_stage: counters");
  a.counters = static_cast<uint32_t*>(scratch);
  t_last_kernel = "k_stage_rows";
  e = launch_stage_rows(a, sdt, wdt, (cudaStream_t)stream);
  cudaError_t e2 = cudaFreeAsync(scratch, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "kv_stage: launch");
  if (e2 != cudaSuccess) return cuda_fail(e2, "kv_stage: counters");
  *used = true;
  return KV_OK;
}

}  // namespace kvx
