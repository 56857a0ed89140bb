// Internal declarations shared by the library's translation units (not part of the ABI).
#pragma once
#include <nvtx3/nvToolsExt.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "kvx.h"

#define KVX_MAX_RANKS 16

struct kv_layout {
  kv_layout_desc d;
  int64_t extent[6];  // per kv_axis
  int64_t stride[6];  // element stride per kv_axis (dense row-major in axis_order)
  int32_t h_local;
  int32_t elem_bytes;
  int32_t dk;         // log2 of the head_dim split x (0: none); stride[DIM] is the D/x part's
  size_t pool_bytes;
};

namespace kvx {

// thread-local error message + status helpers
kv_status fail(kv_status st, const std::string& msg);
kv_status cuda_fail(cudaError_t e, const char* what);
extern std::atomic<uint64_t> g_launches;
constexpr int kMaxDevices = 64;
extern std::atomic<int32_t> g_sm_budget[kMaxDevices];  // kv_set_sm_budget per device (0 = all SMs)

int32_t dtype_bytes(int32_t dt);
bool fp8(int32_t dt);  // KV_F8E4M3 or KV_F8E4M3FNUZ (carries per-head scales)
// K/V both layouts hold (kv_part): *kv1 = 0 both, else 1 with *c0 the one shared index
kv_status kv_pair(const kv_layout* s, const kv_layout* d, int32_t* kv1, int32_t* c0);

// n / d for 32-bit n via one umulhi (Granlund-Montgomery round-up method).
struct FastDiv {
  uint32_t d, mul, shr;
};
FastDiv make_fastdiv(uint32_t d);

// ---- kernel argument blocks (by value) -------------------------------------------
struct ConvArgs {
  int32_t kv1, c0;     // K-only / V-only transfer: kv1 = 1 and c0 the one K/V index (reading 27)
  int32_t s_dk, d_dk;  // head_dim split (log2 x) of source / destination (element-wise kernel)
  // row kernel over an x-split head_dim (x >= 8 elements): chunk (8 elements) ch of a row at
  // byte offset (ch >> ck) * chs + (ch & (2^ck - 1)) * 8 * element bytes; split = 0: plain rows
  int32_t split, s_ck, d_ck;
  int64_t s_chs, d_chs;
  // smem-transpose kernel (k_convert_tr): a side whose two innermost axes are (DIM, SLOT)
  // -- a head_dim-major value cache -- is read / written as whole (DIM x SLOT) tiles
  // (mode 1); or whose head_dim is x-split with (D/x, SLOT, x) innermost (mode 2, x = s_x/d_x)
  int32_t s_tr, d_tr, s_x, d_x;
  int32_t tr_lbp, tr_lbd, s_lm, d_lm;  // log2 of Bp, Bd, s_x / 8, d_x / 8
  int32_t tr_w16;  // k_convert_tr8: 2-byte head_dim-major source -> rows, 16-slot sub-blocks
  FastDiv f_hde;  // D-local heads per item loop (Hd_eff)
  const uint8_t* src[KVX_MAX_RANKS];
  uint8_t* dst[KVX_MAX_RANKS];
  const float* sscale[KVX_MAX_RANKS];  // per source index (e4m3 sources)
  const float* dscale[KVX_MAX_RANKS];  // per destination index (e4m3 destinations)
  int8_t src_of_p[KVX_MAX_RANKS];      // P tp_rank -> index into src[], -1 if absent
  int8_t dst_rank[KVX_MAX_RANKS];      // index -> D tp_rank
  int8_t hq_off[KVX_MAX_RANKS];        // first D-local head converted for each destination
  int32_t Hd_eff;                      // D-local heads converted per destination (<= Hd)
  FastDiv f_nd;                        // number of destinations (row kernel: fastest item index)
  int64_t ss[6], ds[6];                // element strides by axis
  int32_t Hp, Hd, D, Bp, Bd, lb, Lc;
  int32_t s_l0, d_l0;  // first global layer of the P / D pools (pipeline stages)
  const int32_t* s_blk_off;
  const int32_t* s_blk_ids;
  const int32_t* d_blk_off;
  const int32_t* d_blk_ids;
  const int32_t* d_blk_req;
  const int32_t* tok_off;
  FastDiv f_dch, f_in0, f_in1, f_l, f_bl, f_hp, f_bp, f_bd;
  int32_t slot_inner;  // 1: slot is the faster of (slot, head)
  uint32_t total;      // chunks in this launch (flat kernel)
  uint64_t total64;    // chunks in this launch (row kernel: one launch up to 2^31 rows)
  // row-tiled fast path: work item = (dst rank, dst block, layer, K/V, row group)
  FastDiv f_cpr;       // 8-element chunks per head_dim row (D / 8)
  FastDiv f_items;     // row groups per (dst rank, dst block, layer, K/V) tile
  int32_t rows_per_tile, rows_per_item, npass, cpr_shift;
  FastDiv f_sb;     // slot sub-tiles per tile
  int32_t ts_log2;  // sub-tile = 2^ts_log2 slots x 2^(5-ts_log2) heads
  uint32_t n_items;
  // per-request completion inside one launch (kv_convert_reshard_notify, row kernel): the
  // warp finishing a request's last item release-stores req_epoch into req_flag[r]
  uint32_t* req_cnt;
  uint32_t* req_flag;
  uint64_t* req_ns;
  uint32_t req_epoch, items_per_block;
  // k_requant_rows: items per CTA (contiguous, layer-outermost order) and the most layers
  // one CTA's range spans (its tables: that many layers' worth)
  uint32_t rq_per_cta, rq_layers;
};

// TMA tile path (same dtype): one cp.async.bulk.tensor load per (dst block, layer, K/V,
// P rank, source block) lands the sub-tile in smem already in D's order (the tensor map's
// dimension order is D's), then bulk stores write D's contiguous runs.
struct TileArgs {
  int32_t kv1, c0;  // K-only / V-only transfer (reading 27)
  CUtensorMap maps[KVX_MAX_RANKS][2];  // [source index][K/V]: dims (DIM, A, B, BLOCK, LAYER)
  uint8_t* dst[KVX_MAX_RANKS];
  int8_t dst_rank[KVX_MAX_RANKS];
  int8_t src_of_p[KVX_MAX_RANKS];
  int64_t ds[6];                        // destination element strides
  int32_t Hp, Hd, Bp, Bd, D, esize, nh, lb, Lc, s_l0, d_l0;
  int32_t head_major;  // D inner order (HEAD, SLOT, DIM): smem [nh][Bp][D]; else (SLOT, HEAD, DIM): [Bp][nh][D]
  int32_t share_p;     // >= 0: only this P rank (kv_convert_share); -1: every P rank of each D rank
  int32_t stage_bytes, stages;
  int32_t evict_first;  // k_tile_copy: L2 evict-first hints on the TMA loads and bulk stores (default; KVX_TC_EVICT=0 off)
  const int32_t* s_blk_off;
  const int32_t* s_blk_ids;
  const int32_t* d_blk_off;
  const int32_t* d_blk_ids;
  const int32_t* d_blk_req;
  const int32_t* tok_off;
  FastDiv f_nd, f_parts, f_sub, f_l;
  uint32_t n_items;
  // k_tile_cast (a cast on the way: consumer warps convert the staged sub-tile): destination
  // element size and the fp8 scales of either side ([L][2][H_local] per rank index)
  int32_t d_esize;
  const float* sscale[KVX_MAX_RANKS];
  const float* dscale[KVX_MAX_RANKS];
  // partial sub-tiles (the request's last block, slots >= T present): the valid rows are
  // loaded with plain 16-B loads from here instead of the TMA box, which would also read the
  // tail slots (SPEC S:274 -- never read beyond T_r)
  const uint8_t* src[KVX_MAX_RANKS];
  int64_t ss[KVX_MAX_RANKS][6];          // source element strides per source index
};
cudaError_t launch_tile_cast(const TileArgs& a, int sdt, int ddt, cudaStream_t s);

struct PackArgs {
  int32_t kv1, c0;
  int32_t s_dk;  // K-only / V-only transfer: kv1 = 1 and c0 the one K/V index (reading 27)
  const uint8_t* src;
  uint8_t* wire;
  const float* sscale;  // source scales (unused unless the wire cast needs them)
  const float* dscale;  // destination scales (narrowing to e4m3 on the sender)
  int64_t ss[6];
  int32_t Hp, Hd, D, Bp, lb, Lc, p, q, hb, nh;
  int32_t s_l0, d_l0;
  const int32_t* s_blk_off;
  const int32_t* s_blk_ids;
  const int32_t* tok_off;
  const int32_t* tok_req;
  FastDiv f_dch, f_tok, f_nh, f_l, f_bp;
  uint32_t total;
  // row kernel: item = 32 consecutive wire rows (tokens) of one (layer, K/V, head)
  FastDiv f_tg;  // token groups of 32
  int32_t cpr_shift;
  uint32_t n_items;
};

struct UnpackArgs {
  int32_t kv1, c0;
  int32_t d_dk;  // K-only / V-only transfer: kv1 = 1 and c0 the one K/V index (reading 27)
  uint8_t* dst;
  const uint8_t* wire;
  const float* sscale;  // source scales (widening from e4m3 on the receiver)
  const float* dscale;
  int64_t ds[6];
  int32_t Hp, Hd, D, Bd, lb, Lc, p, q, hb, nh;
  int32_t s_l0, d_l0;
  int64_t total_tokens;
  const int32_t* d_blk_off;
  const int32_t* d_blk_ids;
  const int32_t* d_blk_req;
  const int32_t* tok_off;
  FastDiv f_dch, f_in0, f_in1, f_l, f_bl, f_bd;
  int32_t slot_inner;
  uint32_t total;
  // row kernel: item = (dst block, layer, K/V, 2-D sub-tile of slots x overlap heads)
  FastDiv f_sb, f_items;
  int32_t cpr_shift, ts_log2;
  uint32_t n_items;
};

// Persistent D-side staged pull (k_pull_rows): one launch covers every layer chunk of a
// kv_pull_staged call; warps wait in-kernel for each chunk's ready flags and the last warp
// out of a chunk releases its ring slots.  Item (chunk-relative) =
// ((((dst block, local layer), K/V), sub-tile), source).  Same dtype on wire and pool.
#define KVX_MAX_RING 8
constexpr int kMaxRampArgs = 3;  // ramp chunks of ChunkPlan (below)
struct PullArgs {
  int32_t kv1, c0;  // K-only / V-only transfer (reading 27)
  uint8_t* dst;
  const uint8_t* ring[KVX_MAX_RANKS][KVX_MAX_RING];  // [source][slot] peer-mapped
  const uint32_t* ready[KVX_MAX_RANKS];               // local words P writes
  uint32_t* freef[KVX_MAX_RANKS];                     // peer words in P's memory
  int32_t hb[KVX_MAX_RANKS];                          // first global head of each overlap
  uint32_t* counters;                                 // [2 * nchunks] handed out / done, zero on entry
  uint32_t* watermark;                                // counters[2 * nchunks]: chunks released in order
  int32_t* err;
  uint64_t timeout_ns;
  uint32_t spin_ns;  // back-off between polls
  int64_t ds[6];
  int32_t nsrc, R, Hd, D, Bd, lb, le, step, nchunks, q, nh, d_l0;
  uint32_t seq0;
  int64_t total_tokens;
  const int32_t* d_blk_off;
  const int32_t* d_blk_ids;
  const int32_t* d_blk_req;
  const int32_t* tok_off;
  FastDiv f_src, f_sb, f_items, f_l_full, f_l_last;
  int32_t slot_inner, cpr_shift, ts_log2;
  uint32_t n_blk;                   // dst blocks of the batch
  uint32_t items_full, items_last;  // items per chunk (all sources), set by the launcher
  // ramp chunks (ChunkPlan): chunk k < nramp covers layers [ramp_l0[k], ramp_l0[k] + nl);
  // chunk k >= nramp starts at lb + rsum + (k - nramp) * step
  int32_t nramp, rsum;
  int32_t ramp_l0[kMaxRampArgs];
  uint32_t ramp_items[kMaxRampArgs];
  FastDiv f_l_ramp[kMaxRampArgs];
};

// kv_stage's one-launch path (k_stage_rows, the P-side mirror of k_pull_rows): warps take
// pack items chunk after chunk from a shared counter, wait in-kernel for the chunk's ring
// slot to be free, and the warp completing chunk k release-stores the ready word (in chunk
// order) -- no per-chunk wait / pack / signal launch triple.
struct StageArgs {
  PackArgs p;                      // the pack of one destination; lb / wire set per chunk in-kernel
  uint8_t* ring[KVX_MAX_RING];     // [slot] on this GPU
  uint32_t* ready;                 // peer word on D (D waits ready >= seq + 1)
  const uint32_t* freef;           // local word D writes (slot of chunk seq free: free >= seq + 1 - R)
  uint32_t* counters;              // [2 * nchunks] handed out / done, then the watermark; zero on entry
  int32_t* err;
  uint64_t timeout_ns;
  uint32_t spin_ns, seq0;
  int32_t R, nchunks, lb, le, step, nramp, rsum;
  int32_t ramp_l0[kMaxRampArgs], ramp_nl[kMaxRampArgs];
  uint32_t items_per_layer;
};

struct AmaxArgs {
  int32_t kv1, c0;
  int32_t s_dk;  // K-only / V-only transfer: kv1 = 1 and c0 the one K/V index (reading 27)
  const uint8_t* src[KVX_MAX_RANKS];
  const float* sscale[KVX_MAX_RANKS];
  int8_t src_of_p[KVX_MAX_RANKS];
  int64_t ss[6];
  int32_t Hp, Hd, D, q, lb, Lc;
  int32_t s_l0, d_l0;
  const int32_t* s_blk_off;
  const int32_t* s_blk_ids;
  const int32_t* tok_off;
  const int32_t* tok_req;
  uint32_t* amax_bits;  // [L][2][Hd] float bits (non-negative floats order like uints)
  float* peer;          // optional second copy of the finished scales (D's array, peer-mapped)
  int32_t hq0, nhq;     // D-local heads [hq0, hq0 + nhq) computed (a P rank's share); f_hd = nhq
  float qmax;           // largest finite value of the destination fp8 (448 e4m3fn, 240 e4m3fnuz)
  FastDiv f_tg, f_hd, f_bp, f_hp;
  uint32_t n_tok, n_items;
  // row path (head_dim innermost, 16-B rows): item = (group of kAmaxG token groups, head,
  // K/V, layer); set by the launcher
  int32_t rows, cpr_shift;
  FastDiv f_tgc;
  uint32_t n_row_items;
};

// A10 chunk schedule of kv_stage / kv_pull_staged over [lb, le): |layer_chunk|-layer chunks
// (0: one chunk), the last one partial; layer_chunk < 0 with |layer_chunk| >= 4 and a range
// of at least two chunks: the first chunks ramp up (step/8, step/4, step/2 layers) so D's
// first NVLink read waits only for a small pack (the pipeline fill).  Both sides and the
// persistent pull kernel enumerate chunks through this one plan.
constexpr int kMaxRamp = kMaxRampArgs;
struct ChunkPlan {
  int32_t lb = 0, le = 0, step = 1, nramp = 0, rsum = 0, n = 0;
  int32_t ramp[kMaxRamp] = {0, 0, 0};
  void bounds(int32_t k, int32_t* l0, int32_t* l1) const {
    if (k < nramp) {
      int32_t s = lb;
      for (int32_t i = 0; i < k; ++i) s += ramp[i];
      *l0 = s;
      *l1 = s + ramp[k];
      return;
    }
    *l0 = lb + rsum + (k - nramp) * step;
    const int64_t e = (int64_t)*l0 + step;
    *l1 = e < le ? (int32_t)e : le;
  }
};
ChunkPlan chunk_plan(int32_t lb, int32_t le, int32_t layer_chunk);

// launchers (kvx_kernels.cu); vec = 8 (fast path, DIM innermost) or 1 (generic)
// kvx_api.cpp: kv_pull_staged's one-launch path (sets *used when it took it)
kv_status pull_rows_fast(int32_t n_src, const kv_layout* const* src, const void* const* rings, int32_t R,
                         const kv_layout* d, void* dst_pool, const kv_batch* dst_bt, const uint32_t* const* ready,
                         uint32_t* const* freef, uint32_t* counters, uint32_t seq0, const ChunkPlan& plan,
                         uint64_t timeout_ns, int32_t* err, kv_stream stream, bool* used);
// dt: the (common) wire / pool dtype; vec-8 row machinery only
cudaError_t launch_pull_rows(PullArgs& a, int dt, cudaStream_t s);
cudaError_t launch_stage_rows(StageArgs& a, int sdt, int wdt, cudaStream_t s);
// kvx_api.cpp: kv_stage's one-launch path (sets *used when it took it)
kv_status stage_rows_fast(const kv_layout* src, const void* src_pool, const kv_batch* src_bt, const kv_layout* dst,
                          void* const* rings, int32_t R, size_t slot_bytes, uint32_t* ready, const uint32_t* freef,
                          uint32_t seq0, const ChunkPlan& plan, uint64_t timeout_ns, int32_t* err, kv_stream stream,
                          bool* used);
cudaError_t launch_amax(const AmaxArgs& a, int sdt, float* out_scales, cudaStream_t s);
cudaError_t preload_kernels();         // every data-path kernel (kvx_kernels.cu)
cudaError_t preload_verify_kernels();  // K6 (kvx_verify.cu)
kv_status ensure_preloaded();          // once per device, before the first spin-wait
kv_status compute_scales_impl(int32_t n_src, const kv_layout* const* src, const void* const* src_pools,
                              const kv_batch* src_bt, const kv_layout* dst, float* out_scales, int32_t lb, int32_t le,
                              kv_stream stream, bool share, float* peer);
cudaError_t launch_convert(const ConvArgs& a, int vec, int sdt, int ddt, cudaStream_t s);
// fp8 -> other fp8 through per-(dst rank, layer, K/V, head) code tables in shared memory
// (k_requant_rows); the launch's tables must fit kRequantMaxTables x 128 B
constexpr uint32_t kRequantMaxTables = 384;
cudaError_t launch_requant(const ConvArgs& a, int sdt, int ddt, cudaStream_t s);
// per-request completion words (kv_convert_reshard_notify): before the row kernel, zero the
// counters and complete the requests with no blocks; or, after any other launch, complete all
struct Notify {
  uint32_t* counters;
  uint32_t* flags;
  uint64_t* ns;
  uint32_t epoch;
};
cudaError_t launch_notify_init(const Notify& n, const int32_t* blk_off, int32_t n_req, cudaStream_t s);
cudaError_t launch_notify_all(const Notify& n, int32_t n_req, cudaStream_t s);
cudaError_t launch_timestamp(uint64_t* out, cudaStream_t s);
// k_convert_tr: a side with (DIM, SLOT) innermost (a.s_tr / a.d_tr), items in a.n_items
cudaError_t launch_convert_tr(const ConvArgs& a, int sdt, int ddt, cudaStream_t s);
// k_convert_tr8: the same items without shared memory (8 x 8 register sub-blocks); needs
// B_p, B_d >= 8 and a.s_dk / a.d_dk set
cudaError_t launch_convert_tr8(const ConvArgs& a, int sdt, int ddt, cudaStream_t s);
constexpr int kTrSmemLimit = 200 * 1024;  // per CTA (4 warps x one Bd x D tile each)
cudaError_t launch_tile_copy(const TileArgs& a, cudaStream_t s);

// Head_dim-major source tiles through TMA (k_convert_tb): a (block, head) tile of a
// (DIM, SLOT)-innermost source is B x D contiguous elements; one 2-D tensor load (128-B rows,
// 128B swizzle) per tile lands it in shared memory, consumer warps transpose 8 x 8 sub-blocks
// out of it (conflict-free thanks to the swizzle) into D's (SLOT, DIM) rows.  The ConvArgs
// are those of k_convert_tr8; maps[i] views source pool i as rows of 128 bytes.
#ifndef KVX_TB_CONSUMERS
#define KVX_TB_CONSUMERS 8  // consumer warps per CTA (c4-pair V pool: 4 -> 8 lifts e4m3 0.86 -> 0.91)
#endif
// consumer warps of the warp-specialised TMA kernels (k_convert_tb, k_tile_cast); their rings
// need at least this many stages (a consumer waits on its stage's phase parity, which aliases
// when two consumers' rounds of one stage are more than one phase apart)
constexpr int kTbConsumers = KVX_TB_CONSUMERS;
struct TbArgs {
  ConvArgs c;
  CUtensorMap maps[KVX_MAX_RANKS];
  int32_t tile_rows;  // 128-B rows per tile (B * D * esize / 128)
  int32_t stages;
  int32_t mode;       // 1: head_dim-major (DIM, SLOT) tiles; 2: x-packed (D/x, SLOT, x), x = 16 B
  int32_t lut;        // fp8 -> other fp8: per-item code tables (1) or the arithmetic cast (0)
  int32_t hpi;        // heads per item: 2 when both head tiles are <= 2 KB and the heads are adjacent
};
cudaError_t launch_convert_tb(const TbArgs& a, int sdt, int ddt, cudaStream_t s);
cudaError_t launch_pack(const PackArgs& a, int vec, int sdt, int wdt, cudaStream_t s);
cudaError_t launch_unpack(const UnpackArgs& a, int vec, int wdt, int ddt, cudaStream_t s);
cudaError_t launch_signal(uint32_t* flag, uint32_t value, cudaStream_t s);
cudaError_t launch_copy_bytes(void* dst, const void* src, size_t bytes, cudaStream_t s);
cudaError_t launch_wait(const uint32_t* flag, uint32_t value, uint64_t timeout_ns, int32_t* err, cudaStream_t s);

// NVTX range over a host call (SURVEY §5 tracing: the layer-chunk structure of the
// schedulers shows up in any NVTX-aware profiler, e.g. `ncu --nvtx`); `payload` is the
// chunk's first layer.  nvtx3 is header-only: with no tool attached push / pop are a
// branch each.
struct NvtxRange {
  explicit NvtxRange(const char* name, int64_t payload = -1) {
    nvtxEventAttributes_t at = {};
    at.version = NVTX_VERSION;
    at.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    at.messageType = NVTX_MESSAGE_TYPE_ASCII;
    at.message.ascii = name;
    if (payload >= 0) {
      at.payloadType = NVTX_PAYLOAD_TYPE_INT64;
      at.payload.llValue = payload;
    }
    nvtxRangePushEx(&at);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace kvx
