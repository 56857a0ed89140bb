// NEXT-2 pieces of the C ABI: the self-describing wire header (transfers
// replayable from files) and the opaque hidden-state copy (P:95 step 3/5).
#include <string.h>

#include <string>

#include "kvx_internal.h"

using namespace kvx;

namespace {
constexpr uint32_t kHdrFixed = 72;

void put32(uint8_t* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
void put64(uint8_t* p, uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
uint32_t get32(const uint8_t* p) {
  uint32_t v = 0;
  for (int i = 0; i < 4; ++i) v |= (uint32_t)p[i] << (8 * i);
  return v;
}
uint64_t get64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= (uint64_t)p[i] << (8 * i);
  return v;
}
}  // namespace

extern "C" {

size_t kv_wire_header_bytes(int32_t n_req) { return kHdrFixed + 4 * (size_t)(n_req < 0 ? 0 : n_req); }

kv_status kv_wire_header_write(const kv_layout* s, const kv_layout* d, int32_t n_req, const int32_t* nt, int32_t lb,
                               int32_t le, uint8_t* out, size_t cap) {
  if (!s || !d || !out || n_req < 0 || (n_req > 0 && !nt)) return fail(KV_EINVAL, "kv_wire_header_write: bad argument");
  const size_t need = kv_wire_header_bytes(n_req);
  if (cap < need) return fail(KV_ESHAPE, "kv_wire_header_write: buffer too small");
  const int32_t H = s->d.num_kv_heads, Hp = H / s->d.tp_degree, Hd = H / d->d.tp_degree;
  const int32_t hb = std::max(s->d.tp_rank * Hp, d->d.tp_rank * Hd);
  const int32_t he = std::min((s->d.tp_rank + 1) * Hp, (d->d.tp_rank + 1) * Hd);
  if (he <= hb) return fail(KV_ESHAPE, "kv_wire_header_write: ranks share no heads");
  int64_t tt = 0;
  for (int32_t r = 0; r < n_req; ++r) tt += nt[r];
  memset(out, 0, need);
  memcpy(out, "KVX1", 4);
  put32(out + 4, 1);
  put32(out + 8, (uint32_t)need);
  put32(out + 12, (uint32_t)kv_wire_dtype(s, d));
  put32(out + 16, (uint32_t)H);
  put32(out + 20, (uint32_t)s->d.head_dim);
  put32(out + 24, (uint32_t)lb);
  put32(out + 28, (uint32_t)le);
  put32(out + 32, (uint32_t)s->d.tp_degree);
  put32(out + 36, (uint32_t)s->d.tp_rank);
  put32(out + 40, (uint32_t)d->d.tp_degree);
  put32(out + 44, (uint32_t)d->d.tp_rank);
  put32(out + 48, (uint32_t)hb);
  put32(out + 52, (uint32_t)he);
  put32(out + 56, (uint32_t)n_req);
  int32_t kv1 = 0, c0 = 0;
  if (kv_pair(s, d, &kv1, &c0) != KV_OK) return KV_ESHAPE;
  put32(out + 60, kv1 ? (uint32_t)(c0 + 1) : 0u);
  put64(out + 64, (uint64_t)kv_wire_bytes(s, d, tt, lb, le));
  for (int32_t r = 0; r < n_req; ++r) put32(out + kHdrFixed + 4 * r, (uint32_t)nt[r]);
  return KV_OK;
}

kv_status kv_wire_header_parse(const uint8_t* h, size_t len, kv_wire_info* o) {
  if (!h || !o || len < kHdrFixed) return fail(KV_EINVAL, "kv_wire_header_parse: short or null header");
  if (memcmp(h, "KVX1", 4) != 0) return fail(KV_EINVAL, "kv_wire_header_parse: bad magic");
  if (get32(h + 4) != 1) return fail(KV_EINVAL, "kv_wire_header_parse: unsupported version");
  const int32_t n_req = (int32_t)get32(h + 56);
  if (n_req < 0 || get32(h + 8) != kv_wire_header_bytes(n_req) || len < kv_wire_header_bytes(n_req))
    return fail(KV_EINVAL, "kv_wire_header_parse: inconsistent length");
  o->wire_dtype = (int32_t)get32(h + 12);
  o->num_kv_heads = (int32_t)get32(h + 16);
  o->head_dim = (int32_t)get32(h + 20);
  o->layer_begin = (int32_t)get32(h + 24);
  o->layer_end = (int32_t)get32(h + 28);
  o->src_tp_degree = (int32_t)get32(h + 32);
  o->src_tp_rank = (int32_t)get32(h + 36);
  o->dst_tp_degree = (int32_t)get32(h + 40);
  o->dst_tp_rank = (int32_t)get32(h + 44);
  o->head_begin = (int32_t)get32(h + 48);
  o->head_end = (int32_t)get32(h + 52);
  o->n_req = n_req;
  o->kv_part = (int32_t)get32(h + 60);
  if (o->kv_part < 0 || o->kv_part > 2) return fail(KV_EINVAL, "kv_wire_header_parse: bad K/V field");
  o->payload_bytes = get64(h + 64);
  o->n_tokens = reinterpret_cast<const int32_t*>(h + kHdrFixed);  // little-endian host
  return KV_OK;
}

kv_status kv_wire_header_check(const uint8_t* h, size_t len, const kv_layout* s, const kv_layout* d, int32_t n_req,
                               const int32_t* nt, int32_t lb, int32_t le) {
  kv_wire_info w;
  kv_status st = kv_wire_header_parse(h, len, &w);
  if (st != KV_OK) return st;
  if (!s || !d) return fail(KV_EINVAL, "kv_wire_header_check: null layout");
  auto bad = [](const char* f) { return fail(KV_ESHAPE, std::string("kv_wire_header_check: ") + f + " differs"); };
  if (w.wire_dtype != kv_wire_dtype(s, d)) return bad("wire dtype");
  if (w.num_kv_heads != s->d.num_kv_heads || w.head_dim != s->d.head_dim) return bad("model shape");
  if (w.layer_begin != lb || w.layer_end != le) return bad("layer range");
  if (w.src_tp_degree != s->d.tp_degree || w.src_tp_rank != s->d.tp_rank) return bad("P parallel strategy");
  if (w.dst_tp_degree != d->d.tp_degree || w.dst_tp_rank != d->d.tp_rank) return bad("D parallel strategy");
  if (w.n_req != n_req) return bad("request count");
  int32_t kv1 = 0, c0 = 0;
  if (kv_pair(s, d, &kv1, &c0) != KV_OK) return KV_ESHAPE;
  if (w.kv_part != (kv1 ? c0 + 1 : 0)) return bad("K/V carried");
  int64_t tt = 0;
  for (int32_t r = 0; r < n_req; ++r) {
    if (w.n_tokens[r] != nt[r]) return bad("token counts");
    tt += nt[r];
  }
  if (w.payload_bytes != (uint64_t)kv_wire_bytes(s, d, tt, lb, le)) return bad("payload size");
  return KV_OK;
}

kv_status kv_copy_bytes(void* dst, const void* src, size_t bytes, kv_stream stream) {
  if (bytes == 0) return KV_OK;
  if (!dst || !src) return fail(KV_EINVAL, "kv_copy_bytes: null pointer");
  cudaError_t e = launch_copy_bytes(dst, src, bytes, (cudaStream_t)stream);
  return e == cudaSuccess ? KV_OK : cuda_fail(e, "kv_copy_bytes: launch");
}

kv_status kv_memcpy_engine(void* dst, const void* src, size_t bytes, kv_stream stream) {
  if (bytes == 0) return KV_OK;
  if (!dst || !src) return fail(KV_EINVAL, "kv_memcpy_engine: null pointer");
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
  return e == cudaSuccess ? KV_OK : cuda_fail(e, "kv_memcpy_engine");
}

}  // extern "C"
