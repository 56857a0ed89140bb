// A3 control plane of the C ABI: the messages P and D exchange before a transfer.
//   P:125 (III-B3)  "the D instance ... obtains the GPU ranks and parallel strategy of the P
//                   instance" -> a rank's layout descriptor travels;
//   P:109 (III-B1)  remote addresses come "through control plane information interaction"
//                   -> a batch's block tables travel (D's to P for the push, P's to D for the
//                   direct pull), and D's fp8 scales travel to P (the sender-side cast).
// A message is plain little-endian bytes (byte map in include/kvx.h); the caller's control
// plane carries it (torch.distributed object exchange here).  Parsing re-validates
// everything a receiver will hand to kv_layout_describe / kv_block_table_update, and an
// FNV-1a digest over the payload catches truncation or corruption in transit.
#include <string.h>

#include <string>
#include <vector>

#include "kvx_internal.h"

using namespace kvx;

namespace {
constexpr uint32_t kCtrlHdr = 128;
constexpr uint32_t kSecScales = 1u, kSecTables = 2u;

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
uint64_t fnv1a(const uint8_t* p, size_t n) {
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

// The block-table rules of kv_block_table_update (S:255 block remap; reading 14): exactly
// ceil(T_r/B) ids per request, each in [0, NB), none twice.
kv_status check_tables(int32_t B, int32_t NB, int32_t n_req, const int32_t* nt, const int32_t* ids, int64_t n_ids,
                       const char* who) {
  int64_t tb = 0;
  for (int32_t r = 0; r < n_req; ++r) {
    if (nt[r] < 0) return fail(KV_EINVAL, std::string(who) + ": negative token count");
    tb += (nt[r] + (int64_t)B - 1) / B;
  }
  if (tb != n_ids)
    return fail(KV_ESHAPE, std::string(who) + ": " + std::to_string(n_ids) + " block ids, sum ceil(T/B) = " +
                               std::to_string(tb));
  std::vector<uint8_t> used((size_t)NB, 0);
  for (int64_t i = 0; i < n_ids; ++i) {
    const int32_t b = ids[i];
    if (b < 0 || b >= NB) return fail(KV_ESHAPE, std::string(who) + ": block id " + std::to_string(b) + " out of range");
    if (used[b]) return fail(KV_ESHAPE, std::string(who) + ": block id " + std::to_string(b) + " used twice");
    used[b] = 1;
  }
  return KV_OK;
}

int64_t scale_count(const kv_layout_desc& d) { return (int64_t)d.num_layers * 2 * (d.num_kv_heads / d.tp_degree); }
}  // namespace

extern "C" {

size_t kv_ctrl_msg_bytes(int32_t n_req, int64_t n_ids, int64_t n_scales) {
  return kCtrlHdr + 4 * (size_t)(n_scales > 0 ? n_scales : 0) + 4 * (size_t)(n_req > 0 ? n_req : 0) +
         4 * (size_t)(n_ids > 0 ? n_ids : 0);
}

kv_status kv_ctrl_msg_write(const kv_layout* lay, const float* host_scales, uint32_t batch_id, int32_t n_req,
                            const int32_t* host_n_tokens, const int32_t* host_block_ids, int64_t n_ids, uint8_t* out,
                            size_t cap, size_t* written) {
  if (!lay || !out || (n_req > 0 && !host_n_tokens) || (n_ids > 0 && !host_block_ids) || n_ids < 0)
    return fail(KV_EINVAL, "kv_ctrl_msg_write: bad argument");
  const kv_layout_desc& d = lay->d;
  const bool tables = n_req >= 0;
  kv_status st;
  if (tables) {
    if ((st = check_tables(d.block_size, d.num_blocks, n_req, host_n_tokens, host_block_ids, n_ids,
                           "kv_ctrl_msg_write")) != KV_OK)
      return st;
  } else if (n_ids != 0) {
    return fail(KV_EINVAL, "kv_ctrl_msg_write: block ids without a request list");
  }
  const int64_t ns = host_scales ? scale_count(d) : 0;
  const size_t need = kv_ctrl_msg_bytes(tables ? n_req : 0, n_ids, ns);
  if (cap < need) return fail(KV_ESHAPE, "kv_ctrl_msg_write: buffer of " + std::to_string(cap) + " bytes, need " +
                                             std::to_string(need));
  memset(out, 0, kCtrlHdr);
  memcpy(out, "KVC1", 4);
  put32(out + 4, 1);
  put32(out + 8, (host_scales ? kSecScales : 0u) | (tables ? kSecTables : 0u));
  put32(out + 12, kCtrlHdr);
  put64(out + 16, need);
  const int32_t f[17] = {d.num_layers, d.first_layer, d.num_kv_heads, d.head_dim, d.tp_degree, d.tp_rank,
                         d.block_size, d.num_blocks, d.dtype, d.axis_order[0], d.axis_order[1], d.axis_order[2],
                         d.axis_order[3], d.axis_order[4], d.axis_order[5], d.kv_part, d.dim_split};
  for (int i = 0; i < 17; ++i) put32(out + 24 + 4 * i, (uint32_t)f[i]);
  put32(out + 92, (uint32_t)(tables ? n_req : 0));
  put64(out + 96, (uint64_t)n_ids);
  put64(out + 104, (uint64_t)ns);
  put32(out + 120, batch_id);
  uint8_t* p = out + kCtrlHdr;
  for (int64_t i = 0; i < ns; ++i, p += 4) {
    uint32_t b;
    memcpy(&b, host_scales + i, 4);
    put32(p, b);
  }
  for (int32_t r = 0; tables && r < n_req; ++r, p += 4) put32(p, (uint32_t)host_n_tokens[r]);
  for (int64_t i = 0; i < n_ids; ++i, p += 4) put32(p, (uint32_t)host_block_ids[i]);
  put64(out + 112, fnv1a(out + kCtrlHdr, need - kCtrlHdr));
  if (written) *written = need;
  return KV_OK;
}

kv_status kv_ctrl_msg_parse(const uint8_t* msg, size_t len, kv_ctrl_info* out) {
  if (!msg || !out) return fail(KV_EINVAL, "kv_ctrl_msg_parse: bad argument");
  if ((uintptr_t)msg % 4) return fail(KV_EINVAL, "kv_ctrl_msg_parse: message not 4-byte aligned");
  if (len < kCtrlHdr || memcmp(msg, "KVC1", 4) != 0) return fail(KV_EINVAL, "kv_ctrl_msg_parse: bad magic / length");
  if (get32(msg + 4) != 1 || get32(msg + 12) != kCtrlHdr) return fail(KV_EINVAL, "kv_ctrl_msg_parse: bad version");
  const uint32_t sec = get32(msg + 8);
  const uint64_t total = get64(msg + 16);
  const int32_t n_req = (int32_t)get32(msg + 92);
  const int64_t n_ids = (int64_t)get64(msg + 96), ns = (int64_t)get64(msg + 104);
  if (sec & ~(kSecScales | kSecTables) || n_req < 0 || n_ids < 0 || ns < 0 || n_ids > 0x7FFFFFFF ||
      ns > 0x7FFFFFFF || total != kv_ctrl_msg_bytes(n_req, n_ids, ns) || total > len)
    return fail(KV_EINVAL, "kv_ctrl_msg_parse: inconsistent section sizes");
  if (fnv1a(msg + kCtrlHdr, total - kCtrlHdr) != get64(msg + 112))
    return fail(KV_EINVAL, "kv_ctrl_msg_parse: payload digest mismatch (truncated or corrupted message)");
  memset(out, 0, sizeof(*out));
  kv_layout_desc& d = out->desc;
  int32_t f[17];
  for (int i = 0; i < 17; ++i) f[i] = (int32_t)get32(msg + 24 + 4 * i);
  d.num_layers = f[0];
  d.first_layer = f[1];
  d.num_kv_heads = f[2];
  d.head_dim = f[3];
  d.tp_degree = f[4];
  d.tp_rank = f[5];
  d.block_size = f[6];
  d.num_blocks = f[7];
  d.dtype = f[8];
  for (int i = 0; i < 6; ++i) d.axis_order[i] = f[9 + i];
  d.kv_part = f[15];
  d.dim_split = f[16];
  // the descriptor must describe (scales are checked by presence below, not dereferenced)
  kv_layout_desc probe = d;
  static const float dummy = 1.f;
  probe.scales = &dummy;
  kv_layout* lay = nullptr;
  size_t pb = 0;
  kv_status st = kv_layout_describe(&probe, &lay, &pb);
  if (st != KV_OK) return fail(st, std::string("kv_ctrl_msg_parse: layout: ") + kv_last_error());
  kv_layout_destroy(lay);
  if ((sec & kSecScales) ? ns != scale_count(d) : ns != 0)
    return fail(KV_EINVAL, "kv_ctrl_msg_parse: scale section does not match the layout");
  if (!(sec & kSecTables) && (n_req || n_ids)) return fail(KV_EINVAL, "kv_ctrl_msg_parse: tables without section bit");
  const uint8_t* p = msg + kCtrlHdr;
  out->scales = ns ? reinterpret_cast<const float*>(p) : nullptr;
  out->n_scales = ns;
  p += 4 * ns;
  out->has_tables = (sec & kSecTables) ? 1 : 0;
  out->n_req = n_req;
  out->n_tokens = reinterpret_cast<const int32_t*>(p);
  p += 4 * (size_t)n_req;
  out->n_ids = n_ids;
  out->block_ids = reinterpret_cast<const int32_t*>(p);
  out->batch_id = get32(msg + 120);
  if (out->has_tables &&
      (st = check_tables(d.block_size, d.num_blocks, n_req, out->n_tokens, out->block_ids, n_ids,
                         "kv_ctrl_msg_parse")) != KV_OK)
    return st;
  return KV_OK;
}

}  // extern "C"
