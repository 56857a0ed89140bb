/*
 * kvx.h -- C ABI of the B200-native heterogeneous-compatible KV transmission path
 * (arXiv 2509.17542, "Disaggregated Prefill and Decoding Inference System for LLM
 * Serving on Multi-Vendor GPUs", section III-B).
 *
 * The path: gather a finished prefill's paged KV blocks, convert them from the
 * prefill (P) instance's layout (block size, axis order, dtype, TP sharding of
 * KV heads) to the decode (D) instance's, and deliver them into D's paged KV pool
 * (on the same GPU, or across NVLink).  Passages (PAPER.md line, section):
 *   P:109  III-B1 transfer engine read(local addr, remote addr, remote location)
 *   P:113  III-B2 VRAM management alignment: block size + tensor layout, flatten
 *          to 1-D before transmission, restore "according to the demand of D"
 *   P:125  III-B3 parallel strategy alignment (Fig. 4): TP merge / split
 *   P:65   I     precision alignment component (semantics: DESIGN.md readings)
 *   P:289  V     by-layer transmission (per-layer pipelining)
 *
 * Conventions (all calls):
 *   - Ownership: the caller owns every device buffer (pools, tables, wire and
 *     scratch).  Hot calls allocate no device memory (one exception: kv_stage's
 *     opt-in KVX_STAGE_PERSISTENT path takes its counters from the stream-ordered
 *     pool).  Handles hold host metadata only.
 *   - Asynchrony: calls validate synchronously, then enqueue on `stream` (a
 *     cudaStream_t passed as void*; NULL = legacy default stream) and return
 *     before device work completes.  Buffers must outlive the stream work.
 *   - Errors: a kv_status; the message of the last failure on the calling thread
 *     is kv_last_error().  Validation fails before anything is enqueued (no
 *     partial work).  Asynchronous CUDA/NCCL errors surface on a later call.
 *   - No exception crosses the ABI.  Calls on distinct streams and handles are
 *     thread-safe.
 *   - Device pointers may be local or peer-mapped (kv_ipc_open, or peer access):
 *     source pools on another GPU turn kv_convert_reshard (run on D's GPU) into the
 *     D-initiated NVLink read of P:109 (kv_pull, kv_pull_staged); a destination pool
 *     on another GPU turns it into a P-side push (kv_push).
 */
#ifndef KVX_H_
#define KVX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  KV_OK = 0,
  KV_EINVAL = 1,        /* bad argument (null pointer, bad enum, bad range) */
  KV_ESHAPE = 2,        /* tp does not divide heads, pool/table/buffer too small, bad block id */
  KV_EUNSUPPORTED = 3,  /* valid but not implemented (e.g. pipeline-parallel mismatch) */
  KV_ECUDA = 4,         /* CUDA runtime error (message has the CUDA string) */
  KV_ENCCL = 5,         /* NCCL error */
  KV_ETIMEOUT = 6       /* flag wait timed out */
} kv_status;

/* Element types.  KV_F8E4M3 is OCP e4m3fn (max 448, no Inf, NaN = S.1111.111).
 * KV_F8E4M3FNUZ is the e4m3 "fnuz" fp8 other GPU vendors' engines keep their KV cache in
 * (NEXT-3, the multi-vendor P/D pairing of the paper's title): bias 8, max 240, no Inf, no
 * negative zero, 0x80 the only NaN.  Both fp8 types carry per-head dequant scales; casts
 * between them dequantise with the source's and quantise with the destination's scales
 * (readings 24-26). */
typedef enum { KV_F16 = 0, KV_BF16 = 1, KV_F8E4M3 = 2, KV_F32 = 3, KV_F8E4M3FNUZ = 4 } kv_dtype;

/* Physical axes of a paged KV pool; extents (L, 2, num_blocks, block_size, H/tp, head_dim). */
typedef enum {
  KV_AX_LAYER = 0, KV_AX_KV = 1, KV_AX_BLOCK = 2, KV_AX_SLOT = 3, KV_AX_HEAD = 4, KV_AX_DIM = 5
} kv_axis;

typedef void* kv_stream; /* cudaStream_t */

/* One TP rank's pool layout ("block size of page attention and the layout of
 * tensor data").  The rank owns global KV heads
 * [tp_rank*H/tp_degree, (tp_rank+1)*H/tp_degree) (head-contiguous TP). */
typedef struct {
  int32_t num_layers;    /* layers held by this pool (L, or a pipeline stage's share) */
  int32_t first_layer;   /* global index of the pool's first layer: 0 without pipeline
                          * parallelism; a PP stage holds [first_layer, first_layer+num_layers)
                          * (NEXT-2 pipeline-stage reshard) */
  int32_t num_kv_heads;  /* global H */
  int32_t head_dim;      /* D */
  int32_t tp_degree;
  int32_t tp_rank;
  int32_t block_size;    /* tokens per page-attention block */
  int32_t num_blocks;    /* pool capacity in blocks */
  int32_t dtype;         /* kv_dtype */
  int32_t axis_order[6]; /* kv_axis, outermost -> innermost; the pool is dense row-major in it */
  int32_t kv_part;       /* 0: the pool holds K and V; 1: K only; 2: V only (its KV axis has extent
                          * 1).  Engines that keep K and V in separate tensors -- possibly with
                          * different axis orders -- describe each as its own layout; a call
                          * moves the K/V both pools hold (KV_ESHAPE if none).  NEXT-3. */
  int32_t dim_split;     /* 0 or 1: none.  x > 1 (a power of two dividing head_dim): head_dim is
                          * stored as (head_dim/x at DIM's place in axis_order, then x innermost)
                          * -- the "x-packed" key cache (K [blocks, heads, D/x, block, x], x =
                          * 16 bytes / element) of other vendors' paged-attention kernels,
                          * converted by the register-transpose kernel (k_convert_tr8) when the
                          * other side has head_dim rows, else element-wise.  NEXT-3. */
  const float* scales;   /* fp8 dtypes only: DEVICE fp32 [num_layers][2][H/tp] dequant scales s
                          * (real value = code * s), indexed by the pool-local layer; NULL
                          * for other dtypes */
} kv_layout_desc;

typedef struct kv_layout kv_layout; /* opaque, immutable after describe */

/* A batch of requests' block tables for one instance (one table per request,
 * shared by all TP ranks of the instance).  All pointers are DEVICE pointers into
 * the caller's buffer, filled by kv_block_table_update; the scalars are host copies. */
typedef struct {
  int32_t n_req;
  int32_t block_size;      /* of the layout the tables were validated against */
  int32_t num_blocks;      /* pool capacity the ids were validated against */
  int32_t max_tokens;      /* max_r T_r */
  int64_t total_tokens;    /* sum_r T_r */
  int64_t total_blocks;    /* sum_r ceil(T_r / block_size) */
  uint64_t token_digest;   /* FNV-1a of the T_r list: the P and D tables of one transfer must agree */
  const int32_t* tok_off;  /* [n_req + 1] prefix sum of T_r */
  const int32_t* blk_off;  /* [n_req + 1] prefix sum of ceil(T_r / block_size) */
  const int32_t* blk_ids;  /* [total_blocks] physical block ids, request-major */
  const int32_t* blk_req;  /* [total_blocks] request index of each table entry */
  const int32_t* tok_req;  /* [total_tokens] request index of each token (batch order) */
} kv_batch;

/* ---- A1: layout ------------------------------------------------------------ */

/* Validate `desc` and derive strides.  *pool_bytes = 2*L*num_blocks*block_size*(H/tp)*D*bytes.
 * KV_ESHAPE if tp_degree does not divide num_kv_heads or tp_rank >= tp_degree;
 * KV_EINVAL on a non-permutation axis_order, bad dtype, non-positive extent, or
 * scales == NULL for an fp8 dtype.  *out must be released with kv_layout_destroy. */
kv_status kv_layout_describe(const kv_layout_desc* desc, kv_layout** out, size_t* pool_bytes);
void kv_layout_destroy(kv_layout* lay);

/* ---- A3: block tables ------------------------------------------------------- */

/* Device bytes kv_block_table_update needs for a batch of this size. */
size_t kv_batch_bytes(int32_t n_req, int64_t total_blocks, int64_t total_tokens);

/* Validate one instance's block tables and upload them (D picks its
 * blocks and tells P through the control plane).  host_n_tokens[n_req] are T_r >= 0;
 * host_block_ids holds, request after request, exactly ceil(T_r/B) ids each (n_ids in
 * total).  Errors (nothing enqueued): KV_ESHAPE if n_ids != sum ceil(T_r/B), an id is
 * outside [0, num_blocks) or appears twice, or dev_buf_bytes < kv_batch_bytes(...);
 * KV_EINVAL on null pointers.  Host arrays may be freed on return; dev_buf (caller-owned,
 * 16-byte aligned) must outlive every use of *out. */
kv_status kv_block_table_update(const kv_layout* lay, int32_t n_req, const int32_t* host_n_tokens,
                                const int32_t* host_block_ids, int64_t n_ids, void* dev_buf,
                                size_t dev_buf_bytes, kv_batch* out, kv_stream stream);

/* ---- A3: control-plane messages ------------------------------------------------
 * What P and D exchange before a transfer: D learns P's "GPU ranks and parallel strategy"
 * (III-B3) and the remote locations come "through control plane information
 * interaction" (III-B1).  One message = one TP rank's layout descriptor, optionally
 * its fp8 scales (host copy, fp32 [num_layers][2][H/tp]) and optionally a batch's block
 * tables (T_r per request + the block ids, request-major: the kv_block_table_update
 * arguments).  Uses: D -> P (D's layout, scales and table: the push and the sender-side
 * cast of the staged pull), P -> D (P's layout and table: the direct pull).  The library
 * only (de)serialises; the caller's control plane moves the bytes.
 * Byte map, little-endian (host byte order must be little-endian for the parse pointers):
 *    0 char[4] "KVC1"       4 u32 version (1)      8 u32 sections (bit 0 scales, bit 1 tables)
 *   12 u32 header bytes (128)                     16 u64 total bytes
 *   24 i32[17] num_layers first_layer num_kv_heads head_dim tp_degree tp_rank block_size
 *              num_blocks dtype axis_order[6] kv_part dim_split
 *   92 i32 n_req           96 i64 n_ids          104 i64 n_scales
 *  112 u64 FNV-1a 64 of bytes [128, total)       120 u32 batch id (caller's tag)  124 u32 0
 *  128 f32 scales[n_scales], i32 n_tokens[n_req], i32 block_ids[n_ids]
 * kv_ctrl_msg_write: host_scales NULL = no scale section; n_req < 0 = no table section (then
 *   n_ids must be 0).  The tables are validated like kv_block_table_update's (KV_ESHAPE:
 *   count, range, duplicate).  KV_ESHAPE if cap < kv_ctrl_msg_bytes(...); *written = bytes.
 * kv_ctrl_msg_parse: checks magic, version, section sizes, the payload digest (KV_EINVAL:
 *   truncated or corrupted), that the descriptor describes (kv_layout_describe rules) and the
 *   tables' rules; fills *out with pointers INTO msg (4-byte aligned; keep msg alive).
 *   out->desc.scales is NULL: upload out->scales to the device and set it before describe. */
typedef struct {
  kv_layout_desc desc;
  uint32_t batch_id;
  int32_t has_tables;
  const float* scales;     /* host, n_scales floats, or NULL */
  int64_t n_scales;
  int32_t n_req;
  const int32_t* n_tokens; /* [n_req] */
  int64_t n_ids;
  const int32_t* block_ids; /* [n_ids] */
} kv_ctrl_info;

size_t kv_ctrl_msg_bytes(int32_t n_req, int64_t n_ids, int64_t n_scales);
kv_status kv_ctrl_msg_write(const kv_layout* lay, const float* host_scales, uint32_t batch_id, int32_t n_req,
                            const int32_t* host_n_tokens, const int32_t* host_block_ids, int64_t n_ids, uint8_t* out,
                            size_t cap, size_t* written);
kv_status kv_ctrl_msg_parse(const uint8_t* msg, size_t len, kv_ctrl_info* out);

/* ---- A2: re-shard plan ------------------------------------------------------- */

/* Pairs (p, q) whose head ranges overlap (Fig. 4): writes up to max_pairs
 * entries {p, q, h_begin, h_end} (global heads) to out[4*i..4*i+3] and returns the pair
 * count, or -1 if a degree does not divide num_kv_heads. */
int32_t kv_plan_pairs(int32_t tp_p, int32_t tp_d, int32_t num_kv_heads, int32_t* out, int32_t max_pairs);

/* ---- A4-A9: fused convert ------------------------------------------------------ */

/* Pool -> pool conversion of every request in the batch for the GLOBAL layers [layer_begin,
 * layer_end), which must lie inside both the P and the D pools' [first_layer, first_layer +
 * num_layers) (KV_EINVAL otherwise) -- with pipeline stages on either side, call once per
 * overlapping (P stage, D stage) pair with the intersection of their ranges.
 * It gathers from the P ranks' pools, TP merge/split by head range (A7),
 * permute to D's axis order and block size, cast (A6), scatter into the D ranks' pools,
 * zero-fill the tail slots of each request's last D block.  Nothing else
 * in any D pool is written; P tail slots are never read.
 *   src[n_src]: P layouts (same model/desc except tp_rank and scales); src_pools[i] is
 *     the DEVICE pool of src[i].  Every P rank whose heads overlap a listed D rank must
 *     be present (KV_ESHAPE otherwise).
 *   dst[n_dst], dst_pools[n_dst]: D layouts / DEVICE pools (may be peer-mapped: the
 *     kernel stores across NVLink -- the fused P-side push).
 *   src_bt / dst_bt: the two instances' tables for the same requests (same n_req and
 *     T_r), validated against src[0] / dst[0].
 * Casts: same dtype = bit copy; fp16<->bf16/fp32 IEEE RNE (NaN -> 0x7FFF); to e4m3
 * q = satfinite_RNE(RN_f32(f32(x) * RN_f32(1/s))) with s = dst scale of (l, c, D-local
 * head); from e4m3 RN_f32(f32(q) * s_src) then RNE.  n_src, n_dst <= 16. */
kv_status kv_convert_reshard(int32_t n_src, const kv_layout* const* src, const void* const* src_pools,
                             const kv_batch* src_bt, int32_t n_dst, const kv_layout* const* dst,
                             void* const* dst_pools, const kv_batch* dst_bt, int32_t layer_begin,
                             int32_t layer_end, kv_stream stream);

/* One P rank's share of a distributed transfer: like kv_convert_reshard with n_src = 1,
 * but only the heads of each listed D rank that P rank `src` holds are written (their tail
 * slots included); the D ranks' other heads are left to the P ranks that hold them (fan-in,
 * P:125 "combine the TP1 and TP2 of P instance").  Every listed D rank must share heads with
 * src (KV_ESHAPE otherwise) and the overlaps must have equal size (always true when one
 * degree divides the other; KV_EUNSUPPORTED otherwise -- call once per D rank).  This is the
 * call each P rank makes in the fused NVLink push. */
kv_status kv_convert_share(const kv_layout* src, const void* src_pool, const kv_batch* src_bt, int32_t n_dst,
                           const kv_layout* const* dst, void* const* dst_pools, const kv_batch* dst_bt,
                           int32_t layer_begin, int32_t layer_end, kv_stream stream);

/* A11 per request inside one launch (the c5 stream: many requests in one call, each handed
 * to decode as soon as its own KV has landed -- P:95 step 6, "D loads and decodes"): exactly
 * kv_convert_reshard (one call = all listed P ranks -> D ranks), and in addition, once every
 * element of request r (of dst_bt) is written, a system-scope release store of `epoch` into
 * done_flags[r] (DEVICE uint32 [n_req], local or peer-mapped) and the %globaltimer value into
 * done_ns[r] (DEVICE uint64 [n_req], or NULL).  On the row kernel the warp that finishes a
 * request's last work item does it (so requests complete as they land, in about table
 * order); on any other kernel every request completes when the launch does.  counters:
 * DEVICE uint32 [n_req] scratch, zeroed by the call on its stream.  Requests with no tokens
 * complete immediately.  kv_timestamp writes %globaltimer into *out on the stream (the same
 * clock, for latencies). */
kv_status kv_convert_reshard_notify(int32_t n_src, const kv_layout* const* src, const void* const* src_pools,
                                    const kv_batch* src_bt, int32_t n_dst, const kv_layout* const* dst,
                                    void* const* dst_pools, const kv_batch* dst_bt, int32_t layer_begin,
                                    int32_t layer_end, uint32_t* counters, uint32_t* done_flags, uint64_t* done_ns,
                                    uint32_t epoch, kv_stream stream);
kv_status kv_timestamp(uint64_t* out, kv_stream stream);

/* ---- NEXT-1: dynamic fp8 scales --------------------------------------------------- */

/* Per-batch dequant scales for the heads of D rank `dst` (precision alignment):
 *   s[l][c][hq] = RN_f32(amax / M),  amax = max |x| over every finite source element of
 *   the batch's valid tokens (x as f32; fp8 sources dequantised with their own scale), M
 *   the largest finite value of dst's fp8 type (448 e4m3fn, 240 e4m3fnuz),
 * for layers [layer_begin, layer_end); s = 1 where amax is 0 or no finite element exists.
 * Reads the P pools that hold dst's heads (every needed P rank must be listed, KV_ESHAPE
 * otherwise).  out_scales: DEVICE float [L][2][H/tp_d]; entries outside the layer range are
 * untouched.  Pass the array as the scales of an e4m3 destination layout for the convert. */
kv_status kv_compute_scales(int32_t n_src, const kv_layout* const* src, const void* const* src_pools,
                            const kv_batch* src_bt, const kv_layout* dst, float* out_scales, int32_t layer_begin,
                            int32_t layer_end, kv_stream stream);

/* ---- A5 / A9: wire format (Fig. 5 flatten / restore) ----------------------------- */

/* Wire dtype of a (src, dst) pair: the narrower of the two (dst on a tie), so a
 * narrowing cast happens on the sender and a widening one on the receiver. */
int32_t kv_wire_dtype(const kv_layout* src, const kv_layout* dst);

/* Bytes of the (src rank -> dst rank) wire buffer for `total_tokens` tokens and layers
 * [layer_begin, layer_end): 2 * (layer_end-layer_begin) * |head overlap| * total_tokens
 * * D * bytes(wire dtype) (the KV size formula).  0 if the ranks do not overlap. */
size_t kv_wire_bytes(const kv_layout* src, const kv_layout* dst, int64_t total_tokens, int32_t layer_begin,
                     int32_t layer_end);

/* Gather + (narrowing) cast into the wire buffer, canonical order (layer, kv, head in
 * overlap, token, dim), tokens of all requests concatenated in batch order ("a
 * one-dimensional tensor before transmission").  wire is DEVICE memory of at least
 * kv_wire_bytes(...) bytes, 16-byte aligned.  KV_ESHAPE if the ranks do not overlap or
 * wire_bytes is short. */
kv_status kv_pack(const kv_layout* src, const void* src_pool, const kv_batch* src_bt, const kv_layout* dst,
                  int32_t layer_begin, int32_t layer_end, void* wire, size_t wire_bytes, kv_stream stream);

/* Restore ("converts the one-dimensional tensor into the required memory layout
 * after transmission"): scatter a wire buffer produced by kv_pack(src -> dst) into the D
 * pool (+ widening cast), zero-filling tail slots of the overlap heads. */
kv_status kv_unpack(const kv_layout* src, const kv_layout* dst, void* dst_pool, const kv_batch* dst_bt,
                    int32_t layer_begin, int32_t layer_end, const void* wire, size_t wire_bytes,
                    kv_stream stream);

/* ---- NEXT-2: self-describing wire header (transfers replayable from files) --
 * Byte-for-byte, little-endian, 72 + 4*n_req bytes:
 *    0 char[4] "KVX1"          4 u32 version (1)         8 u32 header bytes (72 + 4*n_req)
 *   12 i32 wire dtype         16 i32 num_kv_heads       20 i32 head_dim
 *   24 i32 layer_begin        28 i32 layer_end          32 i32 P tp_degree
 *   36 i32 P tp_rank          40 i32 D tp_degree        44 i32 D tp_rank
 *   48 i32 head_begin         52 i32 head_end (the global overlap heads carried)
 *   56 i32 n_req              60 u32 K/V carried (0 both, 1 K, 2 V)   64 u64 payload bytes
 *   72 i32 n_tokens[n_req]
 * The payload that follows in a file is the kv_pack output (kv_wire_bytes bytes, Fig. 5
 * canonical order).  kv_wire_header_write: KV_ESHAPE if cap is too small or the ranks share
 * no heads.  kv_wire_header_parse: KV_EINVAL on a bad magic/version/length.
 * kv_wire_header_check: KV_ESHAPE (the message names the field) when the header does not
 * describe the (src -> dst, n_tokens, layers) wire an unpack with these arguments expects. */
typedef struct {
  int32_t wire_dtype, num_kv_heads, head_dim, layer_begin, layer_end;
  int32_t src_tp_degree, src_tp_rank, dst_tp_degree, dst_tp_rank, head_begin, head_end, n_req;
  int32_t kv_part;  /* K/V the payload carries: 0 both, 1 K only, 2 V only */
  uint64_t payload_bytes;
  const int32_t* n_tokens; /* points into the header buffer */
} kv_wire_info;

size_t kv_wire_header_bytes(int32_t n_req);
kv_status kv_wire_header_write(const kv_layout* src, const kv_layout* dst, int32_t n_req,
                               const int32_t* host_n_tokens, int32_t layer_begin, int32_t layer_end, uint8_t* out,
                               size_t cap);
kv_status kv_wire_header_parse(const uint8_t* hdr, size_t len, kv_wire_info* out);
kv_status kv_wire_header_check(const uint8_t* hdr, size_t len, const kv_layout* src, const kv_layout* dst,
                               int32_t n_req, const int32_t* host_n_tokens, int32_t layer_begin, int32_t layer_end);

/* Opaque device-to-device (or peer) byte copy on `stream` -- the first-token hidden state
 * that travels with the KV (step 3/5; transferred unaligned, as opaque bytes).
 * dst/src DEVICE (may be peer-mapped), any alignment. */
kv_status kv_copy_bytes(void* dst, const void* src, size_t bytes, kv_stream stream);

/* Copy-engine device-to-device (or peer) copy, cudaMemcpyAsync: NOT on the data path -- the
 * bench's in-run NVLink ceiling (a measured peer copy of 1 GiB per direction).
 * dst/src DEVICE (local or peer-mapped). */
kv_status kv_memcpy_engine(void* dst, const void* src, size_t bytes, kv_stream stream);

/* ---- A8: transport over NVLink ------------------------------------------------- */

typedef struct kv_comm kv_comm; /* an NCCL communicator owned by the library */

/* NCCL unique id (128 bytes) created on one rank and shared through the caller's
 * control plane (e.g. torch.distributed store). */
kv_status kv_comm_unique_id(uint8_t out_id[128]);
kv_status kv_comm_init(int32_t nranks, int32_t rank, const uint8_t id[128], int32_t device, kv_comm** out);
void kv_comm_destroy(kv_comm* comm);
kv_status kv_comm_group_start(void);
kv_status kv_comm_group_end(void);

/* Point-to-point byte transfer of a packed wire buffer (ncclSend / ncclRecv over
 * NVLink).  Matching calls on the two ranks must use the same byte count. */
kv_status kv_send(kv_comm* comm, int32_t peer, const void* wire, size_t bytes, kv_stream stream);
kv_status kv_recv(kv_comm* comm, int32_t peer, void* wire, size_t bytes, kv_stream stream);

/* kv_recv into wire_scratch followed by kv_unpack on the same stream. */
kv_status kv_recv_unpack(kv_comm* comm, int32_t peer, void* wire_scratch, size_t bytes, const kv_layout* src,
                         const kv_layout* dst, void* dst_pool, const kv_batch* dst_bt, int32_t layer_begin,
                         int32_t layer_end, kv_stream stream);

/* A10 chunk schedulers (the host core runs the per-layer pipeline natively).
 *
 * kv_push: P side of the fused push.  For layer chunks [l, l+layer_chunk) of [layer_begin,
 * layer_end) (layer_chunk <= 0: one chunk) enqueue kv_convert_share(src -> every listed D
 * rank) on `stream`, then kv_signal(peer_flags[i], epoch) for each D rank.  peer_flags[i]
 * is the (peer-mapped) flag word this P rank owns in D rank i's flag array.
 *
 * kv_send_pipelined / kv_recv_pipelined: the NCCL mode with per-layer double buffering --
 * pack chunk k+1 on pack_stream while chunk k is on the wire (send_stream); on D, receive
 * chunk k+1 while chunk k is unpacked.  wires[2*i + b] (b = 0, 1) are DEVICE buffers of
 * wire_cap bytes for peer i (>= the largest chunk's kv_wire_bytes).  peer_ranks[i] is the
 * communicator rank of peer i.  The calls return after enqueueing; the caller's `stream`
 * is made to wait for all of the work (events created and destroyed inside). */
kv_status kv_push(const kv_layout* src, const void* src_pool, const kv_batch* src_bt, int32_t n_dst,
                  const kv_layout* const* dst, void* const* dst_pools, const kv_batch* dst_bt,
                  uint32_t* const* peer_flags, uint32_t epoch, int32_t layer_begin, int32_t layer_end,
                  int32_t layer_chunk, kv_stream stream);
kv_status kv_send_pipelined(kv_comm* comm, const kv_layout* src, const void* src_pool, const kv_batch* src_bt,
                            int32_t n_dst, const kv_layout* const* dst, const int32_t* peer_ranks,
                            void* const* wires, size_t wire_cap, int32_t layer_begin, int32_t layer_end,
                            int32_t layer_chunk, kv_stream stream, kv_stream pack_stream, kv_stream send_stream);
kv_status kv_recv_pipelined(kv_comm* comm, int32_t n_src, const kv_layout* const* src, const int32_t* peer_ranks,
                            const kv_layout* dst, void* dst_pool, const kv_batch* dst_bt, void* const* wires,
                            size_t wire_cap, int32_t layer_begin, int32_t layer_end, int32_t layer_chunk,
                            kv_stream stream, kv_stream recv_stream, kv_stream unpack_stream);

/* D-initiated read over NVLink -- the paper's direction (D calls read(local buffer,
 * remote buffer, remote location) once P's KV is ready; P:95 step 5).  SM loads of a
 * peer-mapped source move more user bytes per second over NVLink than SM stores to a
 * peer-mapped destination, so a D rank pulls whenever the cast does not
 * narrow; a narrowing cast is done by the sender into a staging ring that D pulls from, so
 * the link still carries the narrow bytes.
 *
 * kv_pull (same-width or widening cast): on `stream` (D's GPU) wait until every
 * *ready_flags[i] >= epoch (local words that P rank i signals when its KV is resident),
 * then kv_convert_reshard(src -> {dst}) per layer chunk with src_pools[i] the IPC-mapped P
 * pools (src_bt: D's copy of P's block table), then kv_signal(done_flags[i], epoch) into
 * each P rank's memory (P may reuse its blocks after acquiring it).
 *
 * kv_stage (P side of a narrowing pull) / kv_pull_staged (D side).  Chunks of
 * [layer_begin, layer_end) carry global sequence numbers seq = seq0, seq0 + 1, ...; chunk seq
 * of the pair (P rank, D rank i) lives in ring slot seq % ring_slots.  rings[i*ring_slots+b]
 * are slot_bytes device buffers owned by the P rank (on D: the peer-mapped addresses of P
 * rank i's slots for this D rank), each >= the largest chunk's kv_wire_bytes.
 *   P: wait *free_flags[i] >= seq + 1 - ring_slots (local word D writes), kv_pack into the
 *      slot, then kv_signal(ready_flags[i], seq + 1) (peer word in D's memory);
 *   D: wait *ready_flags[i] >= seq + 1 (local), kv_unpack from the peer slot (NVLink reads),
 *      kv_signal(free_flags[i], seq + 1) (peer word in P's memory).
 * When wire and pool share the dtype (the narrowing case this exists for), kv_pull_staged
 * is ONE persistent launch (k_pull_rows): warps take items chunk after chunk from a
 * shared counter, wait in-kernel for each chunk's ready words, and the warp completing a
 * chunk frees its slots, strictly in chunk order (a free value v means every chunk below v
 * has been read) -- no per-chunk launch gap.  It needs `counters`, a caller-owned DEVICE
 * scratch of >= 2 x kv_chunk_count + 1 uint32 that the call zeroes on its stream
 * (NULL: one kv_wait / kv_unpack / kv_signal launch triple per chunk instead).
 * kv_stage enqueues a kv_wait / kv_pack / kv_signal triple per chunk.  With the
 * environment variable KVX_STAGE_PERSISTENT=1 (opt-in: measured no faster),
 * one destination (n_dst = 1), static scales, head_dim innermost with 16-B aligned pool and
 * slots, a 2- / 4-byte source and a wire no wider, it is ONE persistent launch
 * (k_stage_rows): warps take pack items chunk after chunk, wait in-kernel for the chunk's
 * slot to be free, and the warp completing a chunk release-stores the ready word, in chunk
 * order; its counters are stream-ordered scratch (cudaMallocAsync / cudaFreeAsync on
 * `stream`).  Like the persistent pull, several of them sharing one GPU need an SM budget
 * (kv_set_sm_budget) so that every one stays resident while the others spin.
 * kv_stage with peer_scales != NULL computes dynamic fp8 scales (NEXT-1 i, kv_compute_scales
 * semantics) chunk by chunk from the P rank's data, for the D heads this P rank holds, into
 * dst[i]'s own scale array (writable DEVICE memory on P's GPU; the pack quantises with it)
 * and stores the same values into peer_scales[i] (on D rank i, peer-mapped) before the ready
 * flag, so D holds the codes and the scales that decode them.  In a TP merge each P rank
 * writes only its own heads' entries.  peer_scales[i] is the scale array of THIS BATCH: codes
 * quantised with per-batch scales decode only with them, so a D pool that keeps requests of
 * several batches keeps one such [L][2][H/tp_d] array per batch (with its requests), not one
 * per pool, and a new batch's array must not be one D still decodes an older batch with.
 * Requires a non-fp8 source and fp8 destinations; NULL: dst[i]'s static scales are used.
 * Chunks (A10, P:289 by-layer transmission): |layer_chunk| layers each (0: the whole
 * range), the last one partial.  layer_chunk < 0 asks for a ramp: when the range holds >= 2
 * chunks and |layer_chunk| >= 4, the first three chunks take |layer_chunk|/8, /4, /2 layers
 * (>= 1), so D's first read waits only for a small pack (the pipeline fill; measured slower
 * on the c4 pair, where each extra chunk costs more than the fill it saves: DESIGN.md §5).  Both sides must
 * pass the same range and layer_chunk; kv_chunk_count gives the number of chunks, and the
 * caller advances seq0 by it per call.  All three validate before
 * enqueueing; a wait that times out sets *err = 1 (device int32 on the waiting GPU) and the
 * stream goes on (the data are then undefined).  P and D may share a GPU (kv_wait); cap the
 * persistent kernel with kv_set_sm_budget there so P's packs find SMs. */
kv_status kv_pull(int32_t n_src, const kv_layout* const* src, const void* const* src_pools, const kv_batch* src_bt,
                  const kv_layout* dst, void* dst_pool, const kv_batch* dst_bt, const uint32_t* const* ready_flags,
                  uint32_t* const* done_flags, uint32_t epoch, int32_t layer_begin, int32_t layer_end,
                  int32_t layer_chunk, uint64_t timeout_ns, int32_t* err, kv_stream stream);
kv_status kv_stage(const kv_layout* src, const void* src_pool, const kv_batch* src_bt, int32_t n_dst,
                   const kv_layout* const* dst, void* const* rings, int32_t ring_slots, size_t slot_bytes,
                   uint32_t* const* ready_flags, const uint32_t* const* free_flags, float* const* peer_scales,
                   uint32_t seq0, int32_t layer_begin, int32_t layer_end, int32_t layer_chunk, uint64_t timeout_ns,
                   int32_t* err, kv_stream stream);
/* Number of chunks kv_stage / kv_pull_staged split [layer_begin, layer_end) into with
 * this layer_chunk (the ramped schedule above); 0 for an empty range.  Pure host function. */
int32_t kv_chunk_count(int32_t layer_begin, int32_t layer_end, int32_t layer_chunk);
kv_status kv_pull_staged(int32_t n_src, const kv_layout* const* src, const void* const* rings, int32_t ring_slots,
                         size_t slot_bytes, const kv_layout* dst, void* dst_pool, const kv_batch* dst_bt,
                         const uint32_t* const* ready_flags, uint32_t* const* free_flags, uint32_t* counters,
                         uint32_t seq0, int32_t layer_begin, int32_t layer_end, int32_t layer_chunk,
                         uint64_t timeout_ns, int32_t* err, kv_stream stream);

/* CUDA IPC for the direct-store (push) mode.  kv_ipc_export writes the 64-byte handle of
 * the allocation containing dev_ptr and dev_ptr's offset inside it; kv_ipc_open maps it in
 * this process (the current device must have peer access to the owner) and returns the
 * peer-mapped address of the original pointer.  kv_ipc_close(base) unmaps (base =
 * returned pointer - offset). */
kv_status kv_ipc_export(const void* dev_ptr, uint8_t out_handle[64], uint64_t* out_offset);
kv_status kv_ipc_open(const uint8_t handle[64], uint64_t offset, void** out_ptr);
kv_status kv_ipc_close(void* mapped_base);

/* Single-process multi-GPU alternative to IPC: let the current device access peer_device's
 * memory directly (cudaDeviceEnablePeerAccess; already-enabled is not an error).
 * KV_EUNSUPPORTED if the pair has no peer path. */
kv_status kv_peer_enable(int32_t peer_device);

/* A11 completion.  kv_signal: after all prior work on `stream`, a system-scope release
 * store of `value` to *flag (local or peer-mapped 4-byte device word).  kv_wait: enqueue
 * a one-warp kernel that spins (acquire, system scope) until *flag >= value (in the
 * wrap-around order (int32_t)(*flag - value) >= 0) or timeout_ns elapses; on timeout it sets
 * *err = 1 (device int32) and returns, so a lost signal never hangs the stream.  Waiter and
 * signaller may share a GPU when they are on different streams: the waiting kernel holds one
 * warp, and the persistent kv_pull_staged kernel holds at most kv_set_sm_budget SMs' worth of
 * CTAs, so the work that leads to the signal always finds free SMs
 * (tests/test_gpu_transport.py runs the whole data plane that way on one GPU). */
kv_status kv_signal(uint32_t* flag, uint32_t value, kv_stream stream);
kv_status kv_wait(const uint32_t* flag, uint32_t value, uint64_t timeout_ns, int32_t* err, kv_stream stream);

/* ---- K6 diagnostics: full-size conservation check (not on the data path) --------------
 * SURVEY 8(d) "full size via the on-device coordinate-hash verify"; SPEC S:272 (every valid
 * element lands exactly once, tail slots are zero, nothing else changes).  Both calls are
 * element-wise with their own index math, independent of the convert kernels.
 * kv_verify_fill: writes into every VALID element (t < T_r) of P rank `src`'s pool a value
 *   drawn from a counter-based hash of (request id, token, global layer, K/V, global head,
 *   dim) and `seed`, chosen so the cast to the destination dtype is exact: same dtype =
 *   random finite bits; between fp16 / bf16 / fp32 = a value all of them represent; to e4m3
 *   / e4m3fnuz = a random finite code k and the source value k x s, s the destination's
 *   scale, which must be a power of two (else *err = 1, device int32).  dst[n_dst]: the D
 *   layouts (with their scales, on this GPU) of every D rank holding a head of `src`.
 *   req_ids: DEVICE int32 [n_req] request ids the hash uses (NULL: the batch index) -- a P
 *   instance holding a subset of a D batch's requests passes their ids in the D batch.
 *   Tail slots are left as they are.
 * kv_verify_check: for EVERY element of D rank `dst`'s pool, compares what must be there
 *   after a transfer of such a fill: the hashed value's code for valid tokens, 0 for tail
 *   slots of each request's last block, `canary` (byte pattern) in every block the batch does
 *   not use.  result: DEVICE uint64 [8]: [0] valid-element mismatches, [1] tail mismatches,
 *   [2] canary mismatches, [3] valid elements checked, [4] pool element offset + 1 of one
 *   mismatch (0: none); zeroed on the stream first.  scratch: DEVICE >= num_blocks bytes.
 * KV_EUNSUPPORTED for fp8 sources, K-only / V-only or x-split pools, or shapes beyond the
 * hash key (> 65535 requests, > 2^20 tokens, > 255 layers, > 511 heads, head_dim > 1023). */
kv_status kv_verify_fill(const kv_layout* src, void* src_pool, const kv_batch* src_bt, int32_t n_dst,
                         const kv_layout* const* dst, const int32_t* req_ids, uint64_t seed, int32_t* err,
                         kv_stream stream);
kv_status kv_verify_check(const kv_layout* src, const kv_layout* dst, const void* dst_pool, const kv_batch* dst_bt,
                          const int32_t* req_ids, uint64_t seed, uint8_t canary, uint8_t* scratch,
                          size_t scratch_bytes, unsigned long long* result, kv_stream stream);

/* ---- misc ------------------------------------------------------------------------- */

/* Load every kernel of the library on the current device now.  Under CUDA lazy loading (the
 * CUDA 12 default) a kernel is loaded at its first launch and loading may wait for kernels
 * already running in the process; a spin-wait (kv_wait, the persistent kv_pull_staged
 * kernel) that needs a not-yet-loaded kernel of the SAME process to run (P and D on one
 * GPU) would then end only by its timeout.  kv_wait, kv_signal and the persistent pull call
 * this once per device themselves; kernels of other libraries (e.g. torch's) that must run
 * while a wait spins should have run once before.  KV_ECUDA on failure. */
kv_status kv_preload(void);

/* Cap the SMs the data-path kernels this process launches afterwards on the CURRENT
 * device may occupy (0 = all; the grid is min(work, n_sms x occupancy)).  NVLink pushes saturate the link with
 * a fraction of the 148 SMs, leaving the rest to prefill compute that overlaps them (P:289
 * "parallel transmission and calculation").  Returns the previous value. */
int32_t kv_set_sm_budget(int32_t n_sms);

/* Number of device kernels this library launched on the calling thread since the last
 * call to kv_launch_count_reset (for the bench's gpu_launches field). */
uint64_t kv_launch_count(void);
void kv_launch_count_reset(void);

const char* kv_last_error(void); /* thread-local, valid until the next failing call */
/* Name of the data-path kernel the calling thread's last convert / pack / unpack call
 * launched ("k_tile_copy", "k_convert_rows", "k_convert", "k_pack_rows", ...); for the
 * bench's roofline line and for tests that pin which path a case takes. */
const char* kv_last_kernel(void);
const char* kv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KVX_H_ */
