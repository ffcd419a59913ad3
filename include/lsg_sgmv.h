/*
 * lsg_sgmv.h -- C-ABI of the B200-native SGMV library (libsgmv_b200.so).
 *
 * This is the thin C layer the north star asks for underneath the reference's
 * C++ operator API.  Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj):
 *
 *   lsg_sgmv           <- lorasim::lora_addon(const Batch&)        core/include/lorasim/sgmv.hpp:72-73,
 *                         core/src/sgmv.cpp:138-141 (fused, accumulates into y)
 *   lsg_sgmv_multi     <- lora_addon over several projection sites sharing one Batch's segments
 *   lsg_dense_lora     <- lorasim::dense_projection(const Batch&, w)  sgmv.cpp:143-155 (LoRA in the GEMM epilogue)
 *   lsg_sgmv_shrink    <- lorasim::sgmv_shrink(const Batch&)       sgmv.hpp:64-66, sgmv.cpp:105-119
 *   lsg_sgmv_expand    <- lorasim::sgmv_expand(v, segs, models)    sgmv.hpp:68-70, sgmv.cpp:121-136
 *   lsg_bgmv           <- lorasim::gather_bmm_oracle(const Batch&) sgmv.hpp:81-83, sgmv.cpp:186-217
 *                         (the per-row gather formulation, one adapter slot per row)
 *   lsg_build_segments <- lorasim::plan_batch grouping             core/src/simulator.cpp:267-309,
 *                         and the per-row gather loop              sgmv.cpp:195-203
 *   lsg_partition_segments <- Scheduler::place (request -> GPU)    core/src/scheduler.cpp:12-29
 *   lsg_tp_sgmv / _nccl <- (no reference counterpart: TP is out of the reference's scope,
 *                         SPEC.md:15) the 70B TP expand with its output all-gather
 *
 * Mapping from the reference's value types:
 *   Segments::boundaries() (sgmv.hpp:28, size_t)  -> seg_starts[n+1] int32, device memory
 *   models[s] (LoraModel, sgmv.hpp:38-48)          -> seg_slot[s]: pool slot index, device memory
 *   LoraModel::a  [h_in, rank] row-major            -> a_ptr[slot] + layer * a_layer_stride
 *   LoraModel::b  [rank, h_out] row-major           -> b_ptr[slot] + layer * b_layer_stride
 *   Matrix x / y (matrix.hpp:12-41, fp64)           -> fp16 / bf16 row-major with row stride ldx / ldy
 *
 * Semantics
 *   * y += x . A_slot(s) . B_slot(s) for every row of segment s (fp32 accumulate,
 *     the shrink result v kept in fp32, one rounding to the storage type per y
 *     element).  lsg_sgmv_shrink overwrites v (fp32); lsg_sgmv_expand accumulates
 *     into y.  The C++ drop-in (lorasim::lora_addon) zero-fills y first, which
 *     gives the reference's overwrite semantics.
 *   * A slot < 0 (or >= num_slots) means "no adapter": the rows are left untouched.
 *   * Every call is asynchronous on `stream`, allocates nothing, never
 *     synchronises the host, and is deterministic: each output element is
 *     produced by a fixed-order fp32 reduction that does not depend on the batch
 *     composition, the segment order, or the launch configuration.  Rows of
 *     segments shorter than the tensor-core threshold (LSG_OPT_TC_MIN_ROWS,
 *     default 128) take the CUDA-core kernels, whose arithmetic is canonical: such
 *     a row's result is bitwise identical whether it is computed by lsg_sgmv, by
 *     lsg_sgmv_shrink + lsg_sgmv_expand, by lsg_bgmv or lsg_sgmv_multi, and on any
 *     GPU of a request-partitioned job.  Rows of longer segments take the tensor-
 *     core kernels (a different, equally deterministic summation): they are
 *     run-to-run identical and agree with the CUDA-core result within the stated
 *     tolerance, not bitwise.  A partition that cuts a long segment into pieces
 *     below the threshold therefore changes those rows within tolerance only.
 *   * Programmatic dependent launch (opt-in, lsg_set_option(LSG_OPT_PDL, 1)):
 *     a launch may then start while the preceding kernel on the stream is still
 *     running; it reads the segment metadata, the weight table and streams the
 *     adapter weights immediately, and waits for the preceding kernel only
 *     before touching x, v or y.  With PDL on, metadata, table and weights must
 *     not be written by the immediately preceding KERNEL on the same stream
 *     (copies and earlier kernels are fine) -- the serving pattern, where one
 *     segment plan is reused by the 7*L launches of a decode step.
 *
 * Errors: host-side validation returns a negative lsg_status and never throws;
 * lsg_last_error() returns a thread-local message for the last failure.
 *
 * Device-side invariants the caller guarantees (the pool allocators in this
 * repo do): a_ptr[s] / b_ptr[s] are 16-byte aligned device pointers, seg_starts
 * is non-decreasing with seg_starts[0] = 0 and seg_starts[n] = total_rows.
 */
#ifndef LSG_SGMV_H_
#define LSG_SGMV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* lsg_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum { LSG_F16 = 0, LSG_BF16 = 1 } lsg_dtype;

typedef enum {
  LSG_OK = 0,
  LSG_EINVAL = -1,       /* bad argument (shape, pointer, layer, segment count) */
  LSG_EUNSUPPORTED = -2, /* well-formed but not supported (e.g. rank > 256) */
  LSG_ECUDA = -3,        /* a CUDA runtime call failed; see lsg_last_error() */
  LSG_ENODEVICE = -4     /* no usable sm_100 device */
} lsg_status;

/* Adapter pool for one projection site (e.g. q_proj), all layers.
 * Plain host struct; the two pointer arrays live in DEVICE memory. */
typedef struct lsg_weight_table {
  const void* const* a_ptr;   /* device [num_slots]: slot base of A, layout [layers][h_in][rank] */
  const void* const* b_ptr;   /* device [num_slots]: slot base of B, layout [layers][rank][h_out] */
  int64_t a_layer_stride;     /* elements between layers of A (>= h_in * rank) */
  int64_t b_layer_stride;     /* elements between layers of B (>= rank * h_out) */
  int32_t num_slots;
  int32_t num_layers;
  int32_t h_in;
  int32_t h_out;
  int32_t rank;
  int32_t dtype;              /* lsg_dtype: storage type of A, B, x and y */
} lsg_weight_table;

/* Fused shrink+expand: y[s_n, h_out] += x[s_n, h_in] . A . B per segment. */
int lsg_sgmv(void* y, int64_t ldy, const void* x, int64_t ldx, const lsg_weight_table* tbl,
             const int32_t* seg_starts, const int32_t* seg_slot, int32_t num_segments,
             int32_t total_rows, int32_t layer, lsg_stream_t stream);

/* Fused call with a caller-owned workspace (device memory, 16-byte aligned).
 * Segments of >= 128 rows take the tensor-core path, which keeps v (fp32) for
 * their rows in the workspace; lsg_sgmv_workspace_size() gives the bytes needed
 * (0 when the shape never uses it).  With a NULL / too small workspace those
 * segments stay on the CUDA-core kernel (same results to within the stated
 * tolerance).  lsg_sgmv() itself uses a library-owned workspace, grown outside
 * stream capture; concurrent lsg_sgmv() calls on different streams should use
 * lsg_sgmv_ws() with their own workspaces. */
size_t lsg_sgmv_workspace_size(const lsg_weight_table* tbl, int32_t total_rows);
int lsg_sgmv_ws(void* y, int64_t ldy, const void* x, int64_t ldx, const lsg_weight_table* tbl,
                const int32_t* seg_starts, const int32_t* seg_slot, int32_t num_segments,
                int32_t total_rows, int32_t layer, void* workspace, size_t workspace_bytes,
                lsg_stream_t stream);

/* Per-call options.  Each field overrides the process default set with
 * lsg_set_option for this call only (-1 = use the process default).  A call
 * takes one snapshot of its options at entry, so concurrent callers with
 * different options (e.g. a decode-only step next to a prefill step on another
 * stream) never see each other's settings. */
typedef struct lsg_call_opts {
  int32_t pdl;             /* programmatic dependent launch: 0 off, 1 on */
  int32_t tc_min_rows;     /* rows from which a segment takes the tensor-core path (0 = 128) */
  int32_t no_tensor_cores; /* 1: every segment stays on the CUDA-core kernel */
  int32_t mma_min_rows;    /* LSG_OPT_MMA_MIN_ROWS for this call (0 = auto) */
} lsg_call_opts;

/* lsg_sgmv with per-call options and an optional caller workspace (NULL: the
 * library's per-device workspace, as lsg_sgmv). */
int lsg_sgmv_ex(void* y, int64_t ldy, const void* x, int64_t ldx, const lsg_weight_table* tbl,
                const int32_t* seg_starts, const int32_t* seg_slot, int32_t num_segments, int32_t total_rows,
                int32_t layer, void* workspace, size_t workspace_bytes, const lsg_call_opts* opts,
                lsg_stream_t stream);

/* Grouped fused call: up to 8 LoRA sites that share one segment plan (e.g. the
 * q / k / v projections of a layer: same requests, same adapters, each site with
 * its own pool, x and y) in ONE launch -- one cluster per (site, row), so the
 * sites' weight streams overlap and the per-launch critical path is paid once.
 * Same results as calling lsg_sgmv per site (the sites must share h_in, h_out,
 * rank, dtype, slot count and layer strides).  Falls back to one launch per site
 * when a site needs another path (long segments, generic shapes). */
typedef struct lsg_sgmv_site {
  void* y;
  int64_t ldy;
  const void* x;
  int64_t ldx;
  const lsg_weight_table* tbl;
} lsg_sgmv_site;
int lsg_sgmv_multi(const lsg_sgmv_site* sites, int32_t num_sites, const int32_t* seg_starts,
                   const int32_t* seg_slot, int32_t num_segments, int32_t total_rows, int32_t layer,
                   lsg_stream_t stream);
int lsg_sgmv_multi_ex(const lsg_sgmv_site* sites, int32_t num_sites, const int32_t* seg_starts,
                      const int32_t* seg_slot, int32_t num_segments, int32_t total_rows, int32_t layer,
                      const lsg_call_opts* opts, lsg_stream_t stream);

/* Tensor-parallel LoRA site (BASELINE configs[4], Llama-2-70B): y [s_n, h] is replicated on
 * the `size` ranks of a TP group, A is replicated and B column-sharded (this rank's shard:
 * columns [rank * h_out, (rank + 1) * h_out) of the full B, shard->h_out = h / size).
 *
 * lsg_tp_sgmv: the all-gather fused into the expand epilogue -- the kernel computes this
 * rank's columns and stores every output vector straight into EVERY rank's y (peer memory
 * over NVLink / NVSwitch: y_peer[d] are device pointers valid in this process, from CUDA
 * IPC or peer access), then one tiny kernel raises this rank's flag at every rank
 * (st.release.sys) and waits for every rank's flag here.  On stream completion every
 * rank's y holds the full result.  flag_peer[d]: rank d's flag array of `size` u32
 * (device, zero-initialised once); `epoch` must increase by one per call (never 0).
 * Decode batches only (one-row tiles, no segment of >= 128 rows).
 *
 * lsg_tp_sgmv_nccl: the baseline -- this rank's columns in place, then ncclAllGather over
 * `nccl_comm` (an ncclComm_t; libnccl.so.2 resolved at run time) through a workspace of
 * lsg_tp_nccl_workspace_size() bytes, and the other ranks' columns copied into y.
 *
 * Each output element is computed by exactly one rank with the unsharded arithmetic, so
 * every rank's y equals the single-GPU result bitwise.  The reference has no TP
 * (SPEC.md:15); its closest analogue is request placement, scheduler.cpp:12-29. */
typedef struct lsg_tp_group {
  int32_t rank;
  int32_t size;                 /* 1..8 */
  void* const* y_peer;          /* host array [size] of device pointers: rank d's y base */
  uint32_t* const* flag_peer;   /* host array [size] of device pointers: rank d's flags [size] */
} lsg_tp_group;
int lsg_tp_sgmv(const lsg_tp_group* group, int64_t ldy, const void* x, int64_t ldx, const lsg_weight_table* shard,
                const int32_t* seg_starts, const int32_t* seg_slot, int32_t num_segments, int32_t total_rows,
                int32_t layer, uint32_t epoch, lsg_stream_t stream);
size_t lsg_tp_nccl_workspace_size(int32_t total_rows, int32_t h_out_shard, int32_t tp_size);
int lsg_tp_sgmv_nccl(void* y, int64_t ldy, const void* x, int64_t ldx, const lsg_weight_table* shard,
                     const int32_t* seg_starts, const int32_t* seg_slot, int32_t num_segments, int32_t total_rows,
                     int32_t layer, int32_t tp_rank, int32_t tp_size, void* nccl_comm /* ncclComm_t */,
                     void* workspace, size_t workspace_bytes, lsg_stream_t stream);

/* Dense projection with the LoRA add in the GEMM epilogue (decode shapes):
 *   y[s_n, h_out] = x[s_n, h_in] . W[h_in, h_out] + x . A_slot(s) . B_slot(s)   (overwrite)
 * <- lorasim::dense_projection(const Batch&, const Matrix& w), sgmv.cpp:143-155.
 * W is row-major [h_in, h_out] (row stride ldw), same dtype as the pool.  The shrink
 * writes v (fp32, [s_n, rank]) into the caller's workspace; one tcgen05 GEMM launch
 * then computes x.W per 64-column tile and adds v . B in its epilogue.  Rank 16,
 * s_n <= 64, h_in % 256 == 0, h_out % 64 == 0 (else LSG_EUNSUPPORTED).  A cluster of 4 CTAs
 * splits K per 64-column tile; the partial products are summed over DSMEM in CTA order. */
size_t lsg_dense_lora_workspace_size(const lsg_weight_table* tbl, int32_t total_rows);
int lsg_dense_lora(void* y, int64_t ldy, const void* x, int64_t ldx, const void* w, int64_t ldw,
                   const lsg_weight_table* tbl, const int32_t* seg_starts, const int32_t* seg_slot,
                   int32_t num_segments, int32_t total_rows, int32_t layer, void* workspace,
                   size_t workspace_bytes, lsg_stream_t stream);

/* Shrink only: v[s_n, rank] (fp32, row stride rank) = x . A per segment (overwrite). */
int lsg_sgmv_shrink(float* v, const void* x, int64_t ldx, const lsg_weight_table* tbl,
                    const int32_t* seg_starts, const int32_t* seg_slot, int32_t num_segments,
                    int32_t total_rows, int32_t layer, lsg_stream_t stream);

/* Expand only: y[s_n, h_out] += v[s_n, rank] (fp32) . B per segment. */
int lsg_sgmv_expand(void* y, int64_t ldy, const float* v, const lsg_weight_table* tbl,
                    const int32_t* seg_starts, const int32_t* seg_slot, int32_t num_segments,
                    int32_t total_rows, int32_t layer, lsg_stream_t stream);

/* Decode-specialised BGMV: one adapter slot per row (row_slot[s_n], device;
 * negative = no adapter).  y += x . A_row_slot . B_row_slot. */
int lsg_bgmv(void* y, int64_t ldy, const void* x, int64_t ldx, const lsg_weight_table* tbl,
             const int32_t* row_slot, int32_t total_rows, int32_t layer, lsg_stream_t stream);

/* On-device segment builder (replaces the CPU grouping of plan_batch,
 * simulator.cpp:239-311, and the per-row gather loop, sgmv.cpp:195-203).
 * Input (device): row_slot[s_n], the pool slot of every token row (negative or
 * >= num_slots = no adapter), rows in request order.  Output (device): a STABLE
 * grouping of the rows -- rows of one slot keep their original order; groups in
 * ascending slot order, except that lead_slot (>= 0; the slot of the step's
 * prefill request, or -1) is placed first, with the prefill request's own rows
 * [lead_row0, lead_row1) ahead of the other lead_slot rows (pass an empty range
 * when there is no prefill); the no-adapter rows form a final group with slot -1.
 * This is plan_batch's row order (prefill prompt rows, then the same-adapter
 * decodes, then the other adapters' decodes in ascending LoraId, request order
 * within) whenever slots are assigned in ascending LoraId.
 *   row_perm[s_n]          gathered row -> original row
 *   seg_starts[s_n + 1]    n+1 boundaries, then padded with s_n
 *   seg_slot[s_n]          n slots, then padded with -1
 *   num_segments[1]        n
 * Because of the padding, lsg_sgmv may be launched with ANY host-side
 * num_segments in [n, s_n] (e.g. the host's count of distinct adapters) without
 * reading n back.  One CTA; total_rows <= 16384. */
size_t lsg_build_segments_workspace(int32_t total_rows, int32_t num_slots);
int lsg_build_segments(const int32_t* row_slot, int32_t total_rows, int32_t num_slots,
                       int32_t lead_slot, int32_t lead_row0, int32_t lead_row1, int32_t* row_perm, int32_t* seg_starts,
                       int32_t* seg_slot, int32_t* num_segments, void* workspace,
                       size_t workspace_bytes, lsg_stream_t stream);

/* Row gather / scatter helpers for the builder's permutation (16-bit rows). */
int lsg_gather_rows(void* dst, int64_t ld_dst, const void* src, int64_t ld_src,
                    const int32_t* row_perm, int32_t rows, int32_t cols, lsg_stream_t stream);
int lsg_scatter_rows(void* dst, int64_t ld_dst, const void* src, int64_t ld_src,
                     const int32_t* row_perm, int32_t rows, int32_t cols, lsg_stream_t stream);

/* Request-partitioned multi-GPU plan (host memory in and out; no device work).
 * Replaces, for one decode step, the reference's request-level placement of
 * requests onto GPUs (core/src/scheduler.cpp:12-29): rows are independent
 * (sgmv.cpp:108-116, 125-134), so a batch shards with no collective.  Whole
 * segments are placed (one adapter's weights read once).  seg_owner (host, n;
 * NULL = every adapter replicated on every rank) routes a segment whose adapter
 * lives on one rank only (slot-sharded pool, seg_owner[s] >= 0) to that rank,
 * whole -- Scheduler::place's adapter-affinity rule.  Replicated segments may be
 * cut into row ranges when that lowers the largest rank load (each range pays
 * the adapter's weights again).  Pieces are assigned by LPT greedy on the
 * algorithmic bytes rows*(h_in+h_out)*e + (h_in+h_out)*rank*e (cost_model.cpp:13-19,
 * :59), largest first onto the least-loaded rank.  Output: *num_pieces pieces
 * ordered by (rank, segment, row); each rank's pieces are its local batch.  There
 * are at most (non-empty segments) + world - 1 pieces; if max_pieces is too
 * small, returns LSG_EINVAL with *num_pieces = the count needed. */
typedef struct lsg_piece {
  int32_t rank;    /* owning rank */
  int32_t seg;     /* segment index in the global batch */
  int32_t row0;    /* first global row */
  int32_t row1;    /* one past the last global row */
} lsg_piece;
int lsg_partition_segments(const int32_t* seg_starts /* host, n+1 */, const int32_t* seg_owner /* host, n or NULL */,
                           int32_t num_segments, int32_t h_in, int32_t h_out, int32_t rank, int32_t elem_bytes,
                           int32_t world, int32_t max_pieces, lsg_piece* pieces, int32_t* num_pieces);

/* Tuning / test hooks. */
typedef enum {
  LSG_OPT_PDL = 0,            /* 0 (default) / 1: programmatic dependent launch */
  LSG_OPT_FORCE_CLUSTER = 1,  /* 0 (default): auto; else split-K cluster size 1..16 */
  LSG_OPT_FORCE_GENERIC = 2,  /* 1: use the generic (any-shape) kernels */
  LSG_OPT_FORCE_TILE_ROWS = 3, /* 0 (default): auto; else rows per tile (1 or 8) */
  LSG_OPT_NO_L2_STAGING = 4,  /* 1: keep B resident in smem from entry; -1: always stage B through L2 into
                                 A's smem (single-tile launches); 0 (default): stage only when B resident
                                 would cost co-residency */
  LSG_OPT_NO_TENSOR_CORES = 5, /* 1: long segments stay on the CUDA-core kernel (no tcgen05 path) */
  LSG_OPT_TC_SPLIT = 6,        /* 1: rank-16 long segments use the two-kernel tensor-core path
                                  (shrink, then expand through a workspace) instead of the fused one */
  LSG_OPT_NO_ROW_MODE = 7,     /* 1: one-row tiles use the segment-major decode (row split / tile scan)
                                  instead of one cluster per row with a segment search */
  LSG_OPT_NO_MULTIROW_TILES = 8, /* 1: rank 64 keeps one-row tiles even when rows share adapters */
  LSG_OPT_TC_MIN_ROWS = 9,      /* 0 (default 128): segments with at least this many rows take the
                                   tensor-core path (rank 16 measured crossover ~256 rows: an engine
                                   whose step has no segment that long passes a threshold above the
                                   batch size per call,
                                   see lsg_api.cu tc_min_rows).  A call with >= this many rows launches the
                                   tensor-core kernel even when no segment turns out that long (the
                                   host does not read segment lengths), which costs ~1 us per launch
                                   at 128-256 decode rows: an engine that knows a step has no prefill
                                   segment sets it above the batch size for that step. */
  LSG_OPT_TC_LEGACY = 10,       /* long-segment kernel generation: 0 (default) auto -- the one-pass
                                   streaming kernel (a CTA per 16-row tile) at ranks 16 / 32 and for calls
                                   of >= 1024 rows, the segment-tile MMA pair at rank 64 below that,
                                   else the cluster-free tcgen05 pair; A/B measurements: 1 the first fused
                                   cluster kernel (rank 16); 2 the streamed cluster kernel (ranks 16 / 32);
                                   3 the segment-tile MMA pair; 4 the streaming kernel; 5 the
                                   cluster-free tcgen05 partials + expand pair */
  LSG_OPT_MMA_MIN_ROWS = 11,    /* segments with at least this many rows (and below the long-segment
                                   threshold) take the segment-tile MMA pair; 0 (default) = auto: rank 64
                                   calls whose rows share adapters (total_rows > num_segments) send every
                                   segment to it, other ranks keep the CUDA-core kernel */
  LSG_OPT_MMA_FUSED = 12        /* the segment-tile MMA path as ONE launch (one cluster per tile: shrink,
                                   DSMEM exchange of the partials, expand): 0 (default) and 1 the
                                   two-launch pair (faster on B200 at every measured shape), 2 the
                                   one-launch form whenever a split fits */
} lsg_option;
int lsg_set_option(int32_t option, int32_t value);
int lsg_get_option(int32_t option);

/* Launch configuration the next call with these scalars would use (for
 * tests and the benchmark's roofline bookkeeping).  path: 0 fast, 1 generic. */
typedef struct lsg_launch_info {
  int32_t path;         /* 0 CUDA-core fast path, 1 generic, 2 every segment on the segment-tile MMA pair
                           (cluster = K-split cluster, tile_rows = 16, row_splits = K split) */
  int32_t cluster;
  int32_t tile_rows;
  int32_t row_splits;
  int32_t grid_ctas;
  int32_t smem_bytes;
} lsg_launch_info;
int lsg_query_launch(const lsg_weight_table* tbl, int32_t num_segments, int32_t total_rows,
                     int32_t kernel /* 0 fused, 1 shrink, 2 expand, 3 bgmv */,
                     lsg_launch_info* info);

/* Phase tracing (profiling aid; only in instrumented builds compiled with
 * -DLSG_INSTRUMENT, see scripts/build_variant.sh -- production builds return
 * LSG_EUNSUPPORTED for a non-NULL buffer).  device_buffer holds
 * 2 * max_ctas * 16 u64.  Thread 0 of every CUDA-core fast-path CTA (up to
 * max_ctas, CTA index = blockIdx.y * C + rank) writes entries [0, max_ctas):
 * clock64() at the kernel's phase boundaries in slots 0..13, %globaltimer at
 * entry in slot 14 and the SM id in slot 15.  Tensor-core CTAs write entries
 * [max_ctas, 2 * max_ctas): %globaltimer at their phase boundaries.  Pass
 * (NULL, 0) to turn it off.  See scripts/trace_phases.py, scripts/trace_tc.py. */
int lsg_set_trace(unsigned long long* device_buffer, int32_t max_ctas);

const char* lsg_status_string(int status);
const char* lsg_last_error(void);
int lsg_version(void); /* major*10000 + minor*100 + patch */

#ifdef __cplusplus
}
#endif
#endif /* LSG_SGMV_H_ */
