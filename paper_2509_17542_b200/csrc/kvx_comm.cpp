// Transport (A8) and completion (A11) of the C ABI: NCCL point-to-point over NVLink,
// CUDA IPC peer mapping for the direct-store push, release/acquire flags.
//
// NCCL: compiled against the NCCL 2.28 headers that ship with torch's wheel and linked
// to the same libnccl.so.2 soname, so in a process that imported torch first the library
// binds to torch's already-loaded NCCL ("version trap").
#include <nccl.h>
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "kvx_internal.h"

using namespace kvx;

struct kv_comm {
  ncclComm_t comm;
  int32_t nranks, rank;
};

namespace {
kv_status nccl_fail(ncclResult_t r, const char* what) {
  return fail(KV_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
}
}  // namespace

namespace kvx {
// kv_preload once per device (a CUDA context loads modules per device)
kv_status ensure_preloaded() {
  static std::mutex mu;
  static bool done[kMaxDevices] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "kv_preload: device");
  if (dev < 0 || dev >= kMaxDevices) return fail(KV_EINVAL, "kv_preload: device index out of range");
  std::lock_guard<std::mutex> g(mu);
  if (done[dev]) return KV_OK;
  if ((e = preload_kernels()) != cudaSuccess) return cuda_fail(e, "kv_preload: kernel attributes");
  done[dev] = true;
  return KV_OK;
}
}  // namespace kvx

extern "C" {

kv_status kv_comm_unique_id(uint8_t out_id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  if (!out_id) return fail(KV_EINVAL, "kv_comm_unique_id: null");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(out_id, &id, 128);
  return KV_OK;
}

kv_status kv_comm_init(int32_t nranks, int32_t rank, const uint8_t id[128], int32_t device, kv_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(KV_EINVAL, "kv_comm_init: bad argument");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "kv_comm_init: cudaSetDevice");
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  kv_comm* c = new kv_comm{nullptr, nranks, rank};
  ncclResult_t r = ncclCommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  *out = c;
  return KV_OK;
}

void kv_comm_destroy(kv_comm* c) {
  if (!c) return;
  ncclCommDestroy(c->comm);
  delete c;
}

kv_status kv_comm_group_start(void) {
  ncclResult_t r = ncclGroupStart();
  return r == ncclSuccess ? KV_OK : nccl_fail(r, "ncclGroupStart");
}

kv_status kv_comm_group_end(void) {
  ncclResult_t r = ncclGroupEnd();
  return r == ncclSuccess ? KV_OK : nccl_fail(r, "ncclGroupEnd");
}

kv_status kv_send(kv_comm* c, int32_t peer, const void* wire, size_t bytes, kv_stream stream) {
  if (!c || (!wire && bytes) || peer < 0 || peer >= c->nranks) return fail(KV_EINVAL, "kv_send: bad argument");
  ncclResult_t r = ncclSend(wire, bytes, ncclUint8, peer, c->comm, (cudaStream_t)stream);
  return r == ncclSuccess ? KV_OK : nccl_fail(r, "ncclSend");
}

kv_status kv_recv(kv_comm* c, int32_t peer, void* wire, size_t bytes, kv_stream stream) {
  if (!c || (!wire && bytes) || peer < 0 || peer >= c->nranks) return fail(KV_EINVAL, "kv_recv: bad argument");
  ncclResult_t r = ncclRecv(wire, bytes, ncclUint8, peer, c->comm, (cudaStream_t)stream);
  return r == ncclSuccess ? KV_OK : nccl_fail(r, "ncclRecv");
}

kv_status kv_recv_unpack(kv_comm* c, int32_t peer, void* wire_scratch, size_t bytes, const kv_layout* src,
                         const kv_layout* dst, void* dst_pool, const kv_batch* dst_bt, int32_t lb, int32_t le,
                         kv_stream stream) {
  if (!src || !dst || !dst_bt) return fail(KV_EINVAL, "kv_recv_unpack: null argument");
  const size_t need = kv_wire_bytes(src, dst, dst_bt->total_tokens, lb, le);
  if (bytes != need)
    return fail(KV_ESHAPE, "kv_recv_unpack: " + std::to_string(bytes) + " bytes, wire format needs " +
                               std::to_string(need));
  kv_status st = kv_recv(c, peer, wire_scratch, bytes, stream);
  if (st != KV_OK) return st;
  return kv_unpack(src, dst, dst_pool, dst_bt, lb, le, wire_scratch, bytes, stream);
}

kv_status kv_ipc_export(const void* dev_ptr, uint8_t out_handle[64], uint64_t* out_offset) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
  if (!dev_ptr || !out_handle || !out_offset) return fail(KV_EINVAL, "kv_ipc_export: null argument");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr));
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  // offset of dev_ptr inside its allocation (the handle maps the whole allocation, so the
  // opening side adds it back).  The runtime API has no base query: use the driver's
  // cuMemGetAddressRange through the runtime's entry-point lookup.
  void* base = nullptr;
  size_t size = 0;
  {
    // cuMemGetAddressRange through the runtime's driver entry point (no -lcuda needed)
    typedef int (*range_fn)(unsigned long long*, size_t*, unsigned long long);
    static range_fn fn = nullptr;
    if (!fn) {
      cudaDriverEntryPointQueryResult q;
      void* p = nullptr;
      e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q);
      if (e != cudaSuccess || !p) return cuda_fail(e, "cudaGetDriverEntryPoint(cuMemGetAddressRange)");
      fn = reinterpret_cast<range_fn>(p);
    }
    unsigned long long b = 0;
    if (fn(&b, &size, (unsigned long long)(uintptr_t)dev_ptr) != 0)
      return fail(KV_ECUDA, "cuMemGetAddressRange failed");
    base = reinterpret_cast<void*>((uintptr_t)b);
  }
  memcpy(out_handle, &h, 64);
  *out_offset = (uint64_t)((uintptr_t)dev_ptr - (uintptr_t)base);
  return KV_OK;
}

// One mapping per exported allocation per process: several exported tensors may live in
// the same caching-allocator segment (same handle), and a handle must not be opened twice.
namespace {
struct Mapping {
  std::string key;
  void* base;
  int refs;
};
std::mutex g_map_mu;
std::vector<Mapping> g_maps;
}  // namespace

kv_status kv_ipc_open(const uint8_t handle[64], uint64_t offset, void** out_ptr) {
  if (!handle || !out_ptr) return fail(KV_EINVAL, "kv_ipc_open: null argument");
  std::lock_guard<std::mutex> lk(g_map_mu);
  const std::string key(reinterpret_cast<const char*>(handle), 64);
  for (auto& m : g_maps)
    if (m.key == key) {
      ++m.refs;
      *out_ptr = static_cast<uint8_t*>(m.base) + offset;
      return KV_OK;
    }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  void* base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  g_maps.push_back({key, base, 1});
  *out_ptr = static_cast<uint8_t*>(base) + offset;
  return KV_OK;
}

kv_status kv_ipc_close(void* mapped_base) {
  std::lock_guard<std::mutex> lk(g_map_mu);
  for (size_t i = 0; i < g_maps.size(); ++i)
    if (g_maps[i].base == mapped_base) {
      if (--g_maps[i].refs > 0) return KV_OK;
      g_maps.erase(g_maps.begin() + (long)i);
      cudaError_t e = cudaIpcCloseMemHandle(mapped_base);
      return e == cudaSuccess ? KV_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
    }
  return fail(KV_EINVAL, "kv_ipc_close: address was not returned by kv_ipc_open (pass pointer - offset)");
}

kv_status kv_peer_enable(int32_t peer_device) {
  int dev = 0, ok = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "kv_peer_enable: cudaGetDevice");
  e = cudaDeviceCanAccessPeer(&ok, dev, peer_device);
  if (e != cudaSuccess) return cuda_fail(e, "kv_peer_enable: cudaDeviceCanAccessPeer");
  if (!ok) return fail(KV_EUNSUPPORTED, "kv_peer_enable: no peer path between the devices");
  e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return KV_OK;
  }
  return e == cudaSuccess ? KV_OK : cuda_fail(e, "cudaDeviceEnablePeerAccess");
}

kv_status kv_preload(void) { return ensure_preloaded(); }

kv_status kv_signal(uint32_t* flag, uint32_t value, kv_stream stream) {
  if (!flag) return fail(KV_EINVAL, "kv_signal: null flag");
  kv_status st = ensure_preloaded();
  if (st != KV_OK) return st;
  cudaError_t e = launch_signal(flag, value, (cudaStream_t)stream);
  return e == cudaSuccess ? KV_OK : cuda_fail(e, "kv_signal: launch");
}

kv_status kv_wait(const uint32_t* flag, uint32_t value, uint64_t timeout_ns, int32_t* err, kv_stream stream) {
  if (!flag || !err) return fail(KV_EINVAL, "kv_wait: null argument");
  kv_status st = ensure_preloaded();  // nothing may need loading while this kernel spins
  if (st != KV_OK) return st;
  cudaError_t e = launch_wait(flag, value, timeout_ns, err, (cudaStream_t)stream);
  return e == cudaSuccess ? KV_OK : cuda_fail(e, "kv_wait: launch");
}

}  // extern "C"
