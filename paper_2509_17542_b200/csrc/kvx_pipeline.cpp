// A10 chunk schedulers of the C ABI: the per-layer pipelines of the two
// transports, run natively so the host loop issues only launches and event edges.
//   kv_push            P side of the fused NVLink push: convert_share per layer chunk, then
//                      one release flag per D rank (A11).
//   kv_send_pipelined  NCCL mode, P side: pack chunk k+1 while chunk k is on the wire.
//   kv_recv_pipelined  NCCL mode, D side: receive chunk k+1 while chunk k is unpacked.
//   kv_pull            D-initiated read: wait for every source's ready flag, then
//                      kv_convert_reshard per layer chunk with the P pools peer-mapped as
//                      sources (NVLink reads), then a done flag back to each P rank.
//   kv_stage           narrowing pull, P side: per chunk, wait for a free ring slot, kv_pack
//                      (the sender-side cast) into it, release a ready flag to the D rank.
//   kv_pull_staged     narrowing pull, D side: per chunk, wait for the ready flags, kv_unpack
//                      straight from the peer-mapped ring slots, release the slots.
#include <nccl.h>

#include <algorithm>
#include <string>
#include <vector>

#include "kvx_internal.h"

using namespace kvx;

namespace {

struct Events {
  std::vector<cudaEvent_t> ev;
  ~Events() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);  // released once pending work completes
  }
  cudaError_t make(size_t n) {
    ev.assign(n, nullptr);
    for (auto& e : ev) {
      cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      if (r != cudaSuccess) return r;
    }
    return cudaSuccess;
  }
};

#define KVX_CUDA(x, what)                         \
  do {                                            \
    cudaError_t e_ = (x);                         \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

// fork: side streams wait for `stream`'s current work
kv_status fork(cudaStream_t stream, cudaEvent_t ev, cudaStream_t a, cudaStream_t b) {
  KVX_CUDA(cudaEventRecord(ev, stream), "pipeline: record start");
  KVX_CUDA(cudaStreamWaitEvent(a, ev, 0), "pipeline: fork");
  KVX_CUDA(cudaStreamWaitEvent(b, ev, 0), "pipeline: fork");
  return KV_OK;
}

// join: `stream` waits for both side streams
kv_status join(cudaStream_t stream, cudaEvent_t ea, cudaEvent_t eb, cudaStream_t a, cudaStream_t b) {
  KVX_CUDA(cudaEventRecord(ea, a), "pipeline: record end");
  KVX_CUDA(cudaEventRecord(eb, b), "pipeline: record end");
  KVX_CUDA(cudaStreamWaitEvent(stream, ea, 0), "pipeline: join");
  KVX_CUDA(cudaStreamWaitEvent(stream, eb, 0), "pipeline: join");
  return KV_OK;
}

}  // namespace

namespace kvx {
ChunkPlan chunk_plan(int32_t lb, int32_t le, int32_t layer_chunk) {
  ChunkPlan p;
  p.lb = lb;
  p.le = le;
  const int32_t mag = layer_chunk == INT32_MIN ? INT32_MAX : (layer_chunk < 0 ? -layer_chunk : layer_chunk);
  p.step = mag > 0 ? mag : std::max(1, le - lb);
  if (layer_chunk < 0 && p.step >= 4 && (int64_t)(le - lb) >= 2 * (int64_t)p.step) {
    p.nramp = kMaxRamp;
    for (int i = 0; i < kMaxRamp; ++i) {  // step/8, step/4, step/2 (>= 1 layer each)
      p.ramp[i] = std::max(1, p.step >> (kMaxRamp - i));
      p.rsum += p.ramp[i];
    }
  }
  const int32_t rest = std::max(0, le - lb - p.rsum);
  p.n = p.nramp + (int32_t)(((int64_t)rest + p.step - 1) / p.step);
  return p;
}
}  // namespace kvx

extern "C" {

kv_status kv_push(const kv_layout* src, const void* src_pool, const kv_batch* src_bt, int32_t n_dst,
                  const kv_layout* const* dst, void* const* dst_pools, const kv_batch* dst_bt,
                  uint32_t* const* peer_flags, uint32_t epoch, int32_t lb, int32_t le, int32_t layer_chunk,
                  kv_stream stream) {
  if (!peer_flags || n_dst < 1) return fail(KV_EINVAL, "kv_push: bad argument");
  for (int i = 0; i < n_dst; ++i)
    if (!peer_flags[i]) return fail(KV_EINVAL, "kv_push: null flag");
  // validate everything before the first launch (an empty range validates and returns)
  kv_status st = kv_convert_share(src, src_pool, src_bt, n_dst, dst, dst_pools, dst_bt, lb, lb, stream);
  if (st != KV_OK) return st;
  if ((st = kv_convert_share(src, src_pool, src_bt, n_dst, dst, dst_pools, dst_bt, le, le, stream)) != KV_OK)
    return st;
  const int32_t step = layer_chunk > 0 ? layer_chunk : std::max(1, le - lb);
  for (int32_t l0 = lb; l0 < le; l0 += step) {
    NvtxRange r("kv_push chunk", l0);
    if ((st = kv_convert_share(src, src_pool, src_bt, n_dst, dst, dst_pools, dst_bt, l0, std::min(le, l0 + step),
                               stream)) != KV_OK)
      return st;
  }
  for (int i = 0; i < n_dst; ++i)
    if ((st = kv_signal(peer_flags[i], epoch, stream)) != KV_OK) return st;
  return KV_OK;
}

kv_status kv_send_pipelined(kv_comm* comm, const kv_layout* src, const void* src_pool, const kv_batch* src_bt,
                            int32_t n_dst, const kv_layout* const* dst, const int32_t* peer_ranks,
                            void* const* wires, size_t wire_cap, int32_t lb, int32_t le, int32_t layer_chunk,
                            kv_stream stream, kv_stream pack_stream, kv_stream send_stream) {
  if (!comm || !src || !src_bt || !dst || !peer_ranks || !wires || n_dst < 1)
    return fail(KV_EINVAL, "kv_send_pipelined: bad argument");
  const int32_t step = layer_chunk > 0 ? layer_chunk : std::max(1, le - lb);
  for (int32_t l0 = lb; l0 < le; l0 += step)
    for (int i = 0; i < n_dst; ++i)
      if (kv_wire_bytes(src, dst[i], src_bt->total_tokens, l0, std::min(le, l0 + step)) > wire_cap)
        return fail(KV_ESHAPE, "kv_send_pipelined: wire buffers smaller than a layer chunk");
  cudaStream_t s = (cudaStream_t)stream, ps = (cudaStream_t)pack_stream, ss = (cudaStream_t)send_stream;
  Events E;
  KVX_CUDA(E.make(3 + 4 * (size_t)n_dst), "kv_send_pipelined: events");
  cudaEvent_t* sent = E.ev.data() + 3;             // [2 * n_dst] last send from buffer (i, b)
  cudaEvent_t* packed = E.ev.data() + 3 + 2 * n_dst;  // [2 * n_dst]
  kv_status st = fork(s, E.ev[0], ps, ss);
  if (st != KV_OK) return st;
  int32_t k = 0;
  for (int32_t l0 = lb; l0 < le; l0 += step, ++k) {
    NvtxRange r("kv_send_pipelined chunk", l0);
    const int32_t l1 = std::min(le, l0 + step), b = k & 1;
    for (int i = 0; i < n_dst; ++i) {
      const int j = 2 * i + b;
      if (k >= 2) KVX_CUDA(cudaStreamWaitEvent(ps, sent[j], 0), "kv_send_pipelined: wait buffer");
      if ((st = kv_pack(src, src_pool, src_bt, dst[i], l0, l1, wires[j], wire_cap, pack_stream)) != KV_OK) return st;
      KVX_CUDA(cudaEventRecord(packed[j], ps), "kv_send_pipelined: record");
      KVX_CUDA(cudaStreamWaitEvent(ss, packed[j], 0), "kv_send_pipelined: wait pack");
    }
    if ((st = kv_comm_group_start()) != KV_OK) return st;
    for (int i = 0; i < n_dst; ++i) {
      const size_t nb = kv_wire_bytes(src, dst[i], src_bt->total_tokens, l0, l1);
      if ((st = kv_send(comm, peer_ranks[i], wires[2 * i + b], nb, send_stream)) != KV_OK) {
        kv_comm_group_end();
        return st;
      }
    }
    if ((st = kv_comm_group_end()) != KV_OK) return st;
    for (int i = 0; i < n_dst; ++i) KVX_CUDA(cudaEventRecord(sent[2 * i + b], ss), "kv_send_pipelined: record");
  }
  return join(s, E.ev[1], E.ev[2], ps, ss);
}

kv_status kv_recv_pipelined(kv_comm* comm, int32_t n_src, const kv_layout* const* src, const int32_t* peer_ranks,
                            const kv_layout* dst, void* dst_pool, const kv_batch* dst_bt, void* const* wires,
                            size_t wire_cap, int32_t lb, int32_t le, int32_t layer_chunk, kv_stream stream,
                            kv_stream recv_stream, kv_stream unpack_stream) {
  NvtxRange nvtx_("kv_recv_pipelined");
  if (!comm || !src || !dst || !dst_bt || !peer_ranks || !wires || n_src < 1)
    return fail(KV_EINVAL, "kv_recv_pipelined: bad argument");
  const int32_t step = layer_chunk > 0 ? layer_chunk : std::max(1, le - lb);
  for (int32_t l0 = lb; l0 < le; l0 += step)
    for (int i = 0; i < n_src; ++i)
      if (kv_wire_bytes(src[i], dst, dst_bt->total_tokens, l0, std::min(le, l0 + step)) > wire_cap)
        return fail(KV_ESHAPE, "kv_recv_pipelined: wire buffers smaller than a layer chunk");
  cudaStream_t s = (cudaStream_t)stream, rs = (cudaStream_t)recv_stream, us = (cudaStream_t)unpack_stream;
  Events E;
  KVX_CUDA(E.make(3 + 2 * (size_t)n_src + 2), "kv_recv_pipelined: events");
  cudaEvent_t* unpacked = E.ev.data() + 3;     // [2 * n_src] last unpack of buffer (i, b)
  cudaEvent_t* recvd = E.ev.data() + 3 + 2 * n_src;  // [2] chunk parity received
  kv_status st = fork(s, E.ev[0], rs, us);
  if (st != KV_OK) return st;
  int32_t k = 0;
  for (int32_t l0 = lb; l0 < le; l0 += step, ++k) {
    const int32_t l1 = std::min(le, l0 + step), b = k & 1;
    if (k >= 2)
      for (int i = 0; i < n_src; ++i)
        KVX_CUDA(cudaStreamWaitEvent(rs, unpacked[2 * i + b], 0), "kv_recv_pipelined: wait buffer");
    if ((st = kv_comm_group_start()) != KV_OK) return st;
    for (int i = 0; i < n_src; ++i) {
      const size_t nb = kv_wire_bytes(src[i], dst, dst_bt->total_tokens, l0, l1);
      if ((st = kv_recv(comm, peer_ranks[i], wires[2 * i + b], nb, recv_stream)) != KV_OK) {
        kv_comm_group_end();
        return st;
      }
    }
    if ((st = kv_comm_group_end()) != KV_OK) return st;
    KVX_CUDA(cudaEventRecord(recvd[b], rs), "kv_recv_pipelined: record");
    KVX_CUDA(cudaStreamWaitEvent(us, recvd[b], 0), "kv_recv_pipelined: wait recv");
    for (int i = 0; i < n_src; ++i) {
      const size_t nb = kv_wire_bytes(src[i], dst, dst_bt->total_tokens, l0, l1);
      if ((st = kv_unpack(src[i], dst, dst_pool, dst_bt, l0, l1, wires[2 * i + b], nb, unpack_stream)) != KV_OK)
        return st;
      KVX_CUDA(cudaEventRecord(unpacked[2 * i + b], us), "kv_recv_pipelined: record");
    }
  }
  return join(s, E.ev[1], E.ev[2], rs, us);
}

kv_status kv_pull(int32_t n_src, const kv_layout* const* src, const void* const* src_pools, const kv_batch* src_bt,
                  const kv_layout* dst, void* dst_pool, const kv_batch* dst_bt, const uint32_t* const* ready_flags,
                  uint32_t* const* done_flags, uint32_t epoch, int32_t lb, int32_t le, int32_t layer_chunk,
                  uint64_t timeout_ns, int32_t* err, kv_stream stream) {
  NvtxRange nvtx_("kv_pull");
  if (n_src < 1 || !ready_flags || !done_flags || !err) return fail(KV_EINVAL, "kv_pull: bad argument");
  for (int i = 0; i < n_src; ++i)
    if (!ready_flags[i] || !done_flags[i]) return fail(KV_EINVAL, "kv_pull: null flag");
  const kv_layout* const D[1] = {dst};
  void* const DP[1] = {dst_pool};
  // validate everything before the first enqueue (empty ranges validate and return)
  kv_status st = kv_convert_reshard(n_src, src, src_pools, src_bt, 1, D, DP, dst_bt, lb, lb, stream);
  if (st != KV_OK) return st;
  if ((st = kv_convert_reshard(n_src, src, src_pools, src_bt, 1, D, DP, dst_bt, le, le, stream)) != KV_OK) return st;
  for (int i = 0; i < n_src; ++i)
    if ((st = kv_wait(ready_flags[i], epoch, timeout_ns, err, stream)) != KV_OK) return st;
  const int32_t step = layer_chunk > 0 ? layer_chunk : std::max(1, le - lb);
  for (int32_t l0 = lb; l0 < le; l0 += step)
    if ((st = kv_convert_reshard(n_src, src, src_pools, src_bt, 1, D, DP, dst_bt, l0, std::min(le, l0 + step),
                                 stream)) != KV_OK)
      return st;
  for (int i = 0; i < n_src; ++i)
    if ((st = kv_signal(done_flags[i], epoch, stream)) != KV_OK) return st;
  return KV_OK;
}

namespace {
// ring slot of global chunk sequence number `seq` (0-based) and the free-count it needs
inline int32_t ring_slot(uint64_t seq, int32_t R) { return (int32_t)(seq % (uint64_t)R); }
}  // namespace

int32_t kv_chunk_count(int32_t layer_begin, int32_t layer_end, int32_t layer_chunk) {
  if (layer_end <= layer_begin) return 0;
  return chunk_plan(layer_begin, layer_end, layer_chunk).n;
}

kv_status kv_stage(const kv_layout* src, const void* src_pool, const kv_batch* src_bt, int32_t n_dst,
                   const kv_layout* const* dst, void* const* rings, int32_t ring_slots, size_t slot_bytes,
                   uint32_t* const* ready_flags, const uint32_t* const* free_flags, float* const* peer_scales,
                   uint32_t seq0, int32_t lb, int32_t le, int32_t layer_chunk, uint64_t timeout_ns, int32_t* err,
                   kv_stream stream) {
  if (!src || !src_bt || !dst || n_dst < 1 || !rings || ring_slots < 1 || !ready_flags || !free_flags || !err)
    return fail(KV_EINVAL, "kv_stage: bad argument");
  for (int i = 0; i < n_dst; ++i) {
    if (!ready_flags[i] || !free_flags[i]) return fail(KV_EINVAL, "kv_stage: null flag");
    for (int b = 0; b < ring_slots; ++b)
      if (!rings[(size_t)i * ring_slots + b]) return fail(KV_EINVAL, "kv_stage: null ring slot");
  }
  const ChunkPlan plan = chunk_plan(lb, le, layer_chunk);
  for (int32_t k = 0; k < plan.n; ++k) {
    int32_t l0, l1;
    plan.bounds(k, &l0, &l1);
    for (int i = 0; i < n_dst; ++i)
      if (kv_wire_bytes(src, dst[i], src_bt->total_tokens, l0, l1) > slot_bytes)
        return fail(KV_ESHAPE, "kv_stage: ring slots smaller than a layer chunk");
  }
  kv_status st;
  if (peer_scales) {  // dynamic scales: validate (empty ranges) before the first enqueue
    for (int i = 0; i < n_dst; ++i) {
      if (!peer_scales[i] || !fp8(dst[i]->d.dtype) || fp8(src->d.dtype) || !dst[i]->d.scales)
        return fail(KV_EINVAL, "kv_stage: dynamic scales need a non-fp8 source, fp8 destinations with scale "
                               "arrays and a peer scale array per D rank");
      const kv_layout* const S1[1] = {src};
      const void* const P1[1] = {src_pool};
      if ((st = compute_scales_impl(1, S1, P1, src_bt, dst[i], const_cast<float*>(dst[i]->d.scales), lb, lb, stream,
                                    true, peer_scales[i])) != KV_OK)
        return st;
    }
  }
  if (n_dst == 1 && !peer_scales) {  // one persistent launch (k_stage_rows) when the row machinery fits
    bool used = false;
    st = stage_rows_fast(src, src_pool, src_bt, dst[0], rings, ring_slots, slot_bytes, ready_flags[0], free_flags[0],
                         seq0, plan, timeout_ns, err, stream, &used);
    if (st != KV_OK || used) return st;
  }
  uint64_t seq = seq0;
  for (int32_t k = 0; k < plan.n; ++k, ++seq) {
    int32_t l0, l1;
    plan.bounds(k, &l0, &l1);
    NvtxRange r("kv_stage chunk", l0);
    const int32_t b = ring_slot(seq, ring_slots);
    for (int i = 0; i < n_dst; ++i) {
      // slot b last held chunk seq - R: the D rank must have released it (free >= seq - R + 1)
      if (seq + 1 > (uint64_t)ring_slots &&
          (st = kv_wait(free_flags[i], (uint32_t)(seq + 1 - ring_slots), timeout_ns, err, stream)) != KV_OK)
        return st;
      if (peer_scales) {
        // NEXT-1 (i): this chunk's per-(layer, K/V, head) scales of the D heads this P rank
        // holds, from its data (one read pass), into dst[i]'s own array (the pack quantises
        // with it) and -- by the same finalize kernel -- into D's array over NVLink, ahead of
        // the ready flag (the codes are useless without them).  In a TP merge every P rank
        // writes only its own heads' entries, so the ranks never overwrite each other.
        const kv_layout* const S1[1] = {src};
        const void* const P1[1] = {src_pool};
        float* own = const_cast<float*>(dst[i]->d.scales);
        if ((st = compute_scales_impl(1, S1, P1, src_bt, dst[i], own, l0, l1, stream, true, peer_scales[i])) != KV_OK)
          return st;
      }
      if ((st = kv_pack(src, src_pool, src_bt, dst[i], l0, l1, rings[(size_t)i * ring_slots + b], slot_bytes,
                        stream)) != KV_OK)
        return st;
    }
    for (int i = 0; i < n_dst; ++i)
      if ((st = kv_signal(ready_flags[i], (uint32_t)(seq + 1), stream)) != KV_OK) return st;
  }
  return KV_OK;
}

kv_status kv_pull_staged(int32_t n_src, const kv_layout* const* src, const void* const* rings, int32_t ring_slots,
                         size_t slot_bytes, const kv_layout* dst, void* dst_pool, const kv_batch* dst_bt,
                         const uint32_t* const* ready_flags, uint32_t* const* free_flags, uint32_t* counters,
                         uint32_t seq0, int32_t lb, int32_t le, int32_t layer_chunk, uint64_t timeout_ns, int32_t* err,
                         kv_stream stream) {
  NvtxRange nvtx_("kv_pull_staged");
  if (n_src < 1 || !src || !rings || ring_slots < 1 || !dst || !dst_bt || !ready_flags || !free_flags || !err)
    return fail(KV_EINVAL, "kv_pull_staged: bad argument");
  for (int i = 0; i < n_src; ++i) {
    if (!ready_flags[i] || !free_flags[i]) return fail(KV_EINVAL, "kv_pull_staged: null flag");
    for (int b = 0; b < ring_slots; ++b)
      if (!rings[(size_t)i * ring_slots + b]) return fail(KV_EINVAL, "kv_pull_staged: null ring slot");
  }
  const ChunkPlan plan = chunk_plan(lb, le, layer_chunk);
  for (int32_t k = 0; k < plan.n; ++k) {
    int32_t l0, l1;
    plan.bounds(k, &l0, &l1);
    for (int i = 0; i < n_src; ++i)
      if (kv_wire_bytes(src[i], dst, dst_bt->total_tokens, l0, l1) > slot_bytes)
        return fail(KV_ESHAPE, "kv_pull_staged: ring slots smaller than a layer chunk");
  }
  for (int i = 0; i < n_src; ++i) {  // validate the unpacks once (empty ranges)
    kv_status v = kv_unpack(src[i], dst, dst_pool, dst_bt, lb, lb, rings[(size_t)i * ring_slots], slot_bytes, stream);
    if (v != KV_OK) return v;
    if ((v = kv_unpack(src[i], dst, dst_pool, dst_bt, le, le, rings[(size_t)i * ring_slots], slot_bytes, stream)) !=
        KV_OK)
      return v;
  }
  bool used = false;
  kv_status st = pull_rows_fast(n_src, src, rings, ring_slots, dst, dst_pool, dst_bt, ready_flags, free_flags,
                                counters, seq0, plan, timeout_ns, err, stream, &used);
  if (st != KV_OK || used) return st;
  uint64_t seq = seq0;
  for (int32_t k = 0; k < plan.n; ++k, ++seq) {
    int32_t l0, l1;
    plan.bounds(k, &l0, &l1);
    const int32_t b = ring_slot(seq, ring_slots);
    for (int i = 0; i < n_src; ++i)
      if ((st = kv_wait(ready_flags[i], (uint32_t)(seq + 1), timeout_ns, err, stream)) != KV_OK) return st;
    for (int i = 0; i < n_src; ++i) {
      const size_t nb = kv_wire_bytes(src[i], dst, dst_bt->total_tokens, l0, l1);
      if ((st = kv_unpack(src[i], dst, dst_pool, dst_bt, l0, l1, rings[(size_t)i * ring_slots + b], nb, stream)) !=
          KV_OK)
        return st;
    }
    for (int i = 0; i < n_src; ++i)
      if ((st = kv_signal(free_flags[i], (uint32_t)(seq + 1), stream)) != KV_OK) return st;
  }
  return KV_OK;
}

}  // extern "C"
