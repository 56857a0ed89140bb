// A10 chunk schedulers of the C ABI: the per-layer pipelines of the two
// transports, run natively so the host loop issues only launches and event edges.
//   kv_push            P side of the fused NVLink push: convert_share per layer chunk, then
//                      one release flag per D rank (A11).
//   kv_send_pipelined  NCCL mode, P side: pack chunk k+1 while chunk k is on the wire.
//   kv_recv_pipelined  NCCL mode, D side: receive chunk k+1 while chunk k is unpacked.
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
  for (int32_t l0 = lb; l0 < le; l0 += step)
    if ((st = kv_convert_share(src, src_pool, src_bt, n_dst, dst, dst_pools, dst_bt, l0, std::min(le, l0 + step),
                               stream)) != KV_OK)
      return st;
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

}  // extern "C"
