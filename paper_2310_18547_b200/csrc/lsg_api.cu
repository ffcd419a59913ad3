// lsg_api.cu -- the extern "C" boundary (include/lsg_sgmv.h): host-side
// validation, launch planning and dispatch onto the sm_100a kernels.
//
// Planning is pure host integer arithmetic on the scalars of the call
// (num_segments, total_rows, shapes) -- no device metadata is read back and the
// host never synchronises.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>

#include <cuda.h>

#include <mutex>

#include <dlfcn.h>

#include "../../include/lsg_sgmv.h"
#include "launch.cuh"
#include "segment_builder.cuh"
#include "sgmv_tc.cuh"
#include "sgmv_tc2.cuh"
#include "sgmv_tc3.cuh"
#include "sgmv_mma.cuh"
#include "sgmv_stream.cuh"

namespace lsg {

thread_local std::string g_err;

int fail(int status, const std::string& msg) {
  g_err = msg;
  return status;
}

int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return LSG_ECUDA;
}

// Tensor-parallel completion flags: raise this rank's flag at every rank (release,
// system scope: the SGMV kernel's peer stores before it in stream order are visible
// first), then wait until every rank's flag at this rank carries the epoch.
struct TpFlagParams {
  uint32_t* peer_flag[8];
  uint32_t* my_flag;
  int32_t rank, size;
  uint32_t epoch;
};
__global__ void tp_flags_kernel(const __grid_constant__ TpFlagParams p) {
  const int d = threadIdx.x;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  if (d < p.size)
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.peer_flag[d] + p.rank), "r"(p.epoch) : "memory");
  if (d < p.size) {
    uint32_t v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p.my_flag + d) : "memory");
    } while (static_cast<int32_t>(v - p.epoch) < 0);
  }
}

namespace {

constexpr int kMaxGridY = 65535;  // gridDim.y limit

// Process-wide defaults (lsg_set_option).  A call never reads these directly:
// it takes one snapshot at entry (Opts, overridden field by field by the
// caller's lsg_call_opts) and every planning / launch decision of that call reads
// the snapshot, so concurrent calls with different per-call options and a
// concurrent lsg_set_option cannot interleave inside one call.
std::atomic<int> g_opt_pdl{0};
std::atomic<int> g_opt_force_cluster{0};
std::atomic<int> g_opt_force_generic{0};
std::atomic<int> g_opt_force_tile_rows{0};
std::atomic<int> g_opt_no_alias{0};
std::atomic<int> g_opt_no_tile_scan{0};
std::atomic<int> g_opt_no_tc{0};
std::atomic<int> g_opt_tc_split{0};
std::atomic<int> g_opt_no_row_mode{0};
std::atomic<int> g_opt_no_rank64_tiles{0};
std::atomic<int> g_opt_tc_min_rows{0};  // rows from which a segment takes the tensor-core path (0 = default)
std::atomic<int> g_opt_tc_legacy{0};    // long-segment kernel generation (LSG_OPT_TC_LEGACY)
std::atomic<int> g_opt_mma_min_rows{0};  // rows from which a segment takes the segment-tile MMA pair (0 = auto)
std::atomic<int> g_opt_mma_fused{0};     // K7 as one launch: 0 auto, 1 never (the pair), 2 whenever it fits

struct Opts {
  int pdl, force_cluster, force_generic, force_tile_rows, no_alias, no_tile_scan, no_tc, tc_split, no_row_mode,
      no_rank64_tiles, tc_min_rows, tc_legacy, mma_min_rows;
};

Opts snapshot(const lsg_call_opts* c) {
  Opts o{g_opt_pdl.load(),     g_opt_force_cluster.load(), g_opt_force_generic.load(), g_opt_force_tile_rows.load(),
         g_opt_no_alias.load(), g_opt_no_tile_scan.load(), g_opt_no_tc.load(),        g_opt_tc_split.load(),
         g_opt_no_row_mode.load(), g_opt_no_rank64_tiles.load(), g_opt_tc_min_rows.load(), g_opt_tc_legacy.load(),
         g_opt_mma_min_rows.load()};
  if (c != nullptr) {
    if (c->pdl >= 0) o.pdl = c->pdl ? 1 : 0;
    if (c->tc_min_rows >= 0) o.tc_min_rows = c->tc_min_rows;
    if (c->no_tensor_cores >= 0) o.no_tc = c->no_tensor_cores ? 1 : 0;
    if (c->mma_min_rows >= 0) o.mma_min_rows = c->mma_min_rows;
  }
  return o;
}

// The snapshot of the call running on this thread (set by CallScope for the
// duration of one C-ABI call; the process defaults outside any call).
thread_local const Opts* t_opts = nullptr;
struct CallScope {
  Opts o;
  const Opts* prev;
  explicit CallScope(const lsg_call_opts* c) : o(snapshot(c)), prev(t_opts) { t_opts = &o; }
  ~CallScope() { t_opts = prev; }
  CallScope(const CallScope&) = delete;
  CallScope& operator=(const CallScope&) = delete;
};
Opts cur() { return t_opts ? *t_opts : snapshot(nullptr); }


// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}
unsigned long long* g_trace = nullptr;
int g_trace_ctas = 0;


bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---- tensor-core path (K5) for segments of >= kTcMinRows rows ----------------------
// K chunks of the shrink cluster: the largest nq in {16, 8, 4, 2} that splits h_in
// into whole 64-column boxes with the CTA's shared memory in budget.
int tc_nq(const lsg_weight_table* t) {
  if (t->rank != 16 && t->rank != 32 && t->rank != 64) return 0;
  if (t->h_out % kTcNT != 0 || t->a_layer_stride % 8 != 0 || t->b_layer_stride % 8 != 0) return 0;
  for (int nq = 16; nq >= 2; nq /= 2) {
    if (t->h_in % (nq * kTcKB) != 0) continue;
    if (tc_shrink_smem(t->rank, t->h_in / nq) <= static_cast<uint32_t>(kSmemBudget)) return nq;
  }
  return 0;
}

int tc_fused_c(const lsg_weight_table* t, int* compact);

int tc_min_rows(const lsg_weight_table* t = nullptr);
// Upper bound on the 128-row tiles of the segments with >= tc_min_rows() rows:
// sum ceil(len / 128) <= s_n / 128 + (number of such segments).
int tc_tile_bound(const lsg_weight_table* t, int s_n, int n_seg) {
  return std::max(1, s_n / kTcM + std::min(n_seg, s_n / tc_min_rows(t)));
}

// Rows from which a segment takes the tensor-core path (LSG_OPT_TC_MIN_ROWS, 0 = default 128).
// The measured crossover at rank 16 is higher (h = 4096, one prefill segment + decodes, µs per
// site, CUDA-core row mode vs tensor cores: 128 rows 5.7 vs 10.3, 192 rows 9.9 vs 10.2, 256
// rows 10.7 vs 10.4, 512 rows 17.7 vs 10.8), but a higher default starves calls whose short
// segments are long-ish: with a tensor-core pass in the call the short-segment kernel runs
// tile-scan on a grid sized by the segment count (threshold 384, two 300-row segments: 1117 us
// per site).  So the library keeps 128, and an engine that knows its step has no segment of
// >= 256 rows passes a threshold above the batch size per call (lsg_call_opts; bench.py does).
int tc_min_rows(const lsg_weight_table* t) {
  (void)t;
  const int x = cur().tc_min_rows;
  return x > 0 ? x : kTcMinRows;
}

bool tc2_choose(const lsg_weight_table* t, struct Tc2Choice* out);
// Long segments run on the cluster-free partials + expand kernels (sgmv_tc3.cuh) unless an
// A/B option picks an earlier generation: LSG_OPT_TC_LEGACY 1 = the first fused kernel
// (rank 16), 2 = the streamed cluster kernel (ranks 16 / 32); LSG_OPT_TC_SPLIT = the
// first two-kernel form.
bool mma_shape_ok(const lsg_weight_table* t);
bool stream_shape_ok(const lsg_weight_table* t) {
  return (t->rank == 16 || t->rank == 32 || t->rank == 64) && t->h_in % 1024 == 0 && t->h_out % 1024 == 0 &&
         t->a_layer_stride % 8 == 0 && t->b_layer_stride % 8 == 0;
}
// Long-segment kernel generation of a call (LSG_OPT_TC_LEGACY): 0 = auto -- the one-pass
// streaming kernel (K9, sgmv_stream.cuh) at ranks 16 / 32 and for calls of >= 1024 rows, the
// segment-tile MMA pair K7 at rank 64 below that, else the cluster-free tcgen05 pair
// (sgmv_tc3.cuh); explicit 1 / 2 = the cluster kernels,
// 3 = the MMA pair, 4 = the streaming kernel, 5 = the cluster-free tcgen05 pair (sgmv_tc3.cuh).
constexpr int kStreamMinRows = 1024;
int tc_gen(const lsg_weight_table* t, int s_n) {
  const int g = cur().tc_legacy;
  if (g != 0) return g;
  // ranks 16 / 32: the streaming kernel for every tensor-core call (measured 512-row prefill +
  // decodes: rank 16 10.9 us vs 17.6 on the tcgen05 pair, rank 32 13.6 vs 16.9); rank 64 below
  // 1024 rows takes the segment-tile MMA pair K7 (128-row prefill + decodes 21.7 us vs 36.7 on
  // the tcgen05 pair, 40.9 on K9; 512 rows 31.9 vs 38.3 / 41.2)
  if ((s_n >= kStreamMinRows || t->rank <= 32) && stream_shape_ok(t)) return 4;
  if (t->rank == 64 && mma_shape_ok(t)) return 3;
  if (tc_nq(t) > 0 && t->h_out % kTcNT == 0) return 5;  // measured: c4-128 10.8 us vs 12.3 on K7
  if (mma_shape_ok(t)) return 3;
  return 5;
}
bool tc3_ok(const lsg_weight_table* t, int s_n) {
  return !cur().tc_split && tc_gen(t, s_n) == 5 && tc_nq(t) > 0 && t->h_out % kTcNT == 0;
}
bool stream_ok(const lsg_weight_table* t, int s_n) {
  return !cur().tc_split && tc_gen(t, s_n) == 4 && stream_shape_ok(t);
}
int stream_tiles(const lsg_weight_table* t, int s_n, int n_seg) {  // 16-row tiles of the segments with >= tc_min_rows rows
  return std::max(1, s_n / 16 + std::min(n_seg, s_n / tc_min_rows(t)));
}
size_t tc3_ws_bytes(const lsg_weight_table* t, int s_n, int n_seg) {
  return static_cast<size_t>(tc_tile_bound(t, s_n, n_seg)) * tc3_kparts(t->h_in) * kTcM * t->rank * sizeof(float);
}
size_t tc_workspace_bytes(const lsg_weight_table* t, int s_n) {
  if (tc_nq(t) == 0 || s_n < tc_min_rows(t)) return 0;
  if (stream_ok(t, s_n)) return static_cast<size_t>(stream_tiles(t, s_n, s_n)) * 256;
  if (tc3_ok(t, s_n)) return tc3_ws_bytes(t, s_n, s_n / tc_min_rows(t));
  if (!cur().tc_split && tc_gen(t, s_n) == 3) return 0;  // the MMA pair's own region (row_ranges)
  // the fused kernels keep v on chip
  if (!cur().tc_split && ((cur().tc_legacy == 2 && tc2_choose(t, nullptr)) ||
                           (cur().tc_legacy == 1 && tc_fused_c(t, nullptr) > 0)))
    return 0;
  return tc_nq(t) > 0 && s_n >= tc_min_rows(t) ? static_cast<size_t>(s_n) * t->rank * sizeof(float) : 0;
}

// ---- segment-tile MMA pair (K7, sgmv_mma.cuh) ---------------------------------------
// Rows [lo, hi) of a fused call take the MMA pair.  Default (LSG_OPT_MMA_MIN_ROWS = 0):
// rank 64 with rows sharing adapters (total_rows > num_segments, so some segment has >= 2
// rows) sends EVERY segment to it (lo = 1: no CUDA-core launch at all -- the weights of each
// segment are spread over ~one CTA per SM whatever its length); otherwise off.  With
// LSG_OPT_TC_LEGACY = 3 the pair also takes the long segments (instead of sgmv_tc3.cuh).
constexpr int kRowsInf = 0x7fffffff;
bool mma_shape_ok(const lsg_weight_table* t) {
  return (t->rank == 16 || t->rank == 32 || t->rank == 64) && t->h_in % kMmaKC == 0 && t->h_out % kMmaKC == 0 &&
         t->a_layer_stride % 8 == 0 && t->b_layer_stride % 8 == 0;
}
struct RowRanges {
  int mma_lo = 0, mma_hi = 0;  // [mma_lo, mma_hi): MMA pair (mma_lo == 0: none)
  int tc_lo = 0;               // [tc_lo, inf): long-segment tensor-core kernels (0: none)
};
RowRanges row_ranges(const lsg_weight_table* t, int n_seg, int s_n) {
  RowRanges rr;
  if (cur().no_tc) return rr;
  const bool tc = tc_nq(t) > 0 && s_n >= tc_min_rows(t);
  const bool gen3 = !cur().tc_split && tc_gen(t, s_n) == 3 && mma_shape_ok(t);
  if (tc && !gen3) rr.tc_lo = tc_min_rows(t);
  int lo = cur().mma_min_rows;
  if (lo <= 0) lo = (t->rank == 64 && s_n > n_seg) ? 1 : 0;
  if (!mma_shape_ok(t)) lo = 0;
  if (gen3 && tc) lo = lo > 0 ? std::min(lo, tc_min_rows(t)) : tc_min_rows(t);
  const int hi = rr.tc_lo > 0 ? rr.tc_lo : kRowsInf;
  if (lo > 0 && lo < hi && s_n >= lo) {
    rr.mma_lo = lo;
    rr.mma_hi = hi;
  }
  return rr;
}
// 16-row tiles of the segments with len >= lo: sum ceil(len/16) <= s_n/16 + #segments
int mma_tile_bound(int s_n, int n_seg, int lo) {
  return std::max(1, s_n / kMmaM + std::min(n_seg, s_n / std::max(lo, 1)));
}
// K / column splits: a divisor d of the 64-column stage count whose slice (nstages / d
// stages) is resident in shared memory at once (<= max_st), the largest with tiles x d <=
// target (the tile bound overestimates the real tiles), else the smallest that fits.
int mma_split(int nstages, int tiles, int max_st, int target) {
  int best = 0;
  for (int d = 1; d <= nstages; ++d) {
    if (nstages % d != 0 || nstages / d > max_st) continue;
    if (best == 0 || static_cast<int64_t>(tiles) * d <= target) best = d;
  }
  return best;
}
#ifndef LSG_MMA_PART_TARGET
#define LSG_MMA_PART_TARGET 160
#endif
#ifndef LSG_MMA_EXP_TARGET
#define LSG_MMA_EXP_TARGET 320
#endif
constexpr int kMmaPartTarget = LSG_MMA_PART_TARGET, kMmaExpTarget = LSG_MMA_EXP_TARGET;  // CTAs per kernel
constexpr uint32_t kMmaPartSmemTarget = 150 * 1024;       // one partials CTA + one expand CTA per SM
constexpr uint32_t kMmaSmemTarget = 110 * 1024;           // expand: two CTAs per SM
// resident stages per CTA within the shared-memory target
int mma_part_max_st(int R) {
  return std::min<int>(kMmaMaxStagesDecl, (kMmaPartSmemTarget - mma_part_smem(R, 0)) / mma_part_stage_bytes(R));
}
int mma_exp_max_st(int R, int kparts) {
  return std::min<int>(kMmaMaxStagesDecl, (kMmaSmemTarget - mma_exp_smem(R, 0, kparts)) / mma_exp_stage_bytes(R));
}
// workspace bound (the splits give tiles * d <= max(target, tiles * nstages / max_st)): the
// partials plus one 128-byte weight descriptor per CTA of each kernel
// smallest K split whose slice is resident (the split never exceeds max(target, tiles * it))
int mma_min_kparts(const lsg_weight_table* t) {
  const int n = t->h_in / kMmaKC, mx = mma_part_max_st(t->rank);
  for (int d = 1; d <= n; ++d)
    if (n % d == 0 && n / d <= mx) return d;
  return n;
}
size_t mma_part_ctas(const lsg_weight_table* t, int tiles) {
  return std::max<size_t>(kMmaPartTarget, static_cast<size_t>(tiles) * mma_min_kparts(t));
}
size_t mma_exp_ctas(const lsg_weight_table* t, int tiles) {
  return std::max<size_t>(kMmaExpTarget, static_cast<size_t>(tiles) * (t->h_out / kMmaKC));
}
size_t mma_ws_bytes(const lsg_weight_table* t, int s_n, int n_seg, int lo) {
  const int tiles = mma_tile_bound(s_n, n_seg, lo);
  const size_t pctas = mma_part_ctas(t, tiles), ectas = mma_exp_ctas(t, tiles);
  return pctas * kMmaM * t->rank * sizeof(float) + (pctas + ectas) * 128;
}
bool encode_map_2d(CUtensorMap* m, int dtype, const void* base, uint64_t cols, uint64_t rows, uint64_t ld_elems,
                   uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle sw) {
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld_elems * 2};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return encode_tiled_fn()(m, dtype == LSG_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                           2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// K split, its cluster (the largest <= 8 dividing it: one partial per cluster) and column split
bool mma_splits(const lsg_weight_table* tbl, int tiles, int& kparts, int& pc, int& ncol) {
  const int R = tbl->rank;
  kparts = mma_split(tbl->h_in / kMmaKC, tiles, mma_part_max_st(R), kMmaPartTarget);
  if (kparts == 0) return false;
  pc = 1;
  for (int c = kMmaMaxPc; c >= 2; --c)
    if (kparts % c == 0) {
      pc = c;
      break;
    }
  ncol = mma_split(tbl->h_out / kMmaKC, tiles, mma_exp_max_st(R, kparts / pc), kMmaExpTarget);
  return ncol > 0;
}
bool prepare_mma(MmaParams& mp, int& tiles, const RowRanges& rr, void* y, int64_t ldy, const void* x, int64_t ldx,
                 const lsg_weight_table* tbl, const int32_t* seg_starts, const int32_t* seg_slot, int n_seg, int s_n,
                 int layer, void* ws, size_t ws_bytes) {
  if (rr.mma_lo == 0) return false;
  if (!aligned16(x) || !aligned16(y) || ldx % 8 != 0 || ldy % 8 != 0 || encode_tiled_fn() == nullptr) return false;
  tiles = mma_tile_bound(s_n, n_seg, rr.mma_lo);
  if (tiles > kMaxGridY) return false;
  if (ws == nullptr || !aligned16(ws) || ws_bytes < mma_ws_bytes(tbl, s_n, n_seg, rr.mma_lo)) return false;
  const int R = tbl->rank;
  mp = MmaParams{};
  // activations: per-call maps; weights: templates (any valid base; the kernels patch in
  // each slot's address), A [h_in][R] rows swizzled by their own width, B [R][h_out] SW128
  const CUtensorMapSwizzle swa = R == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                 : R == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                           : CU_TENSOR_MAP_SWIZZLE_128B;
  if (!encode_map_2d(&mp.tmap_x, tbl->dtype, x, tbl->h_in, s_n, ldx, kMmaKC, kMmaM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_map_2d(&mp.tmap_y, tbl->dtype, y, tbl->h_out, s_n, ldy, kMmaKC, kMmaM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_map_2d(&mp.tmap_a, tbl->dtype, x, R, tbl->h_in, R, R, kMmaKC, swa) ||
      !encode_map_2d(&mp.tmap_b, tbl->dtype, x, tbl->h_out, R, tbl->h_out, kMmaKC, R, CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  mp.y = y;
  mp.ldy = ldy;
  mp.x = x;
  mp.ldx = ldx;
  mp.a_ptr = tbl->a_ptr;
  mp.b_ptr = tbl->b_ptr;
  mp.a_off = static_cast<int64_t>(layer) * tbl->a_layer_stride;
  mp.b_off = static_cast<int64_t>(layer) * tbl->b_layer_stride;
  mp.seg_starts = seg_starts;
  mp.seg_slot = seg_slot;
  if (!mma_splits(tbl, tiles, mp.kparts, mp.pc, mp.ncol)) return false;
  mp.ws = static_cast<float*>(ws);
  const size_t pctas = mma_part_ctas(tbl, tiles);
  // One launch (clusters of c CTAs per tile, K and columns split c ways), only on request
  // (LSG_OPT_MMA_FUSED = 2): measured slower than the pair at every preset (c3: 8.1 vs 6.5 us
  // -- one CTA per SM runs its shrink and expand back to back, the pair overlaps 360 CTAs)
  mp.fused = 0;
  const int fmode = g_opt_mma_fused.load();
  if (fmode == 2) {
    for (int c = kMmaMaxPc; c >= 2; --c) {
      if (tbl->h_in % (c * kMmaKC) != 0 || tbl->h_out % (c * kMmaKC) != 0) continue;
      const int nst = std::max(tbl->h_in, tbl->h_out) / (c * kMmaKC);
      if (nst > kMmaMaxStagesDecl || mma_fused_smem(R, nst, c) > static_cast<uint32_t>(kSmemBudget)) continue;
      const size_t ctas = static_cast<size_t>(tiles) * c;
      if (ctas > pctas || ctas > mma_exp_ctas(tbl, tiles)) continue;
      mp.fused = 1;
      mp.kparts = mp.pc = mp.ncol = c;
      break;
    }
  }
  mp.maps_p = static_cast<uint8_t*>(ws) + pctas * kMmaM * R * sizeof(float);
  mp.maps_e = mp.maps_p + pctas * 128;
  mp.n_seg = n_seg;
  mp.s_n = s_n;
  mp.num_slots = tbl->num_slots;
  mp.h_in = tbl->h_in;
  mp.h_out = tbl->h_out;
  mp.min_rows = rr.mma_lo;
  mp.max_rows = rr.mma_hi;
  mp.trace = g_trace;
  mp.trace_ctas = g_trace_ctas;
  return true;
}

size_t align256(size_t b) { return (b + 255) & ~static_cast<size_t>(255); }
// Workspace a fused call of total_rows rows may need, over every segment count: the MMA
// partials (worst case: rows sharing adapters, one segment per row) + the K5 v.
size_t call_ws_bound(const lsg_weight_table* t, int s_n) {
  const RowRanges rr = row_ranges(t, std::max(0, s_n - 1), s_n);
  size_t b = rr.mma_lo > 0 ? align256(mma_ws_bytes(t, s_n, s_n, rr.mma_lo)) : 0;
  if (tc_nq(t) > 0 && s_n >= tc_min_rows(t)) b += tc_workspace_bytes(t, s_n);
  return b;
}

// Library-owned workspace of lsg_sgmv(), one per device (a process may drive
// several GPUs): grown, never during stream capture.  The caller's current device
// is the device of the launch, so the buffer is allocated and freed there.
constexpr int kMaxDevices = 64;
std::mutex g_ws_mu;
void* g_ws[kMaxDevices] = {};
size_t g_ws_bytes[kMaxDevices] = {};

void* library_workspace(size_t need, cudaStream_t cs) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
  std::lock_guard<std::mutex> lk(g_ws_mu);
  if (g_ws_bytes[dev] >= need) return g_ws[dev];
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(cs, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) return nullptr;
  size_t bytes = std::max<size_t>(need, static_cast<size_t>(1) << 20);
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (g_ws[dev] != nullptr) {
    cudaDeviceSynchronize();  // this device: the old buffer may still be read by queued launches
    cudaFree(g_ws[dev]);
  }
  g_ws[dev] = p;
  g_ws_bytes[dev] = bytes;
  return p;
}

bool encode_rows_map(CUtensorMap* m, int dtype, const void* base, int cols, int rows, int64_t ld) {
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kTcKB), static_cast<cuuint32_t>(kTcM)};
  const cuuint32_t estr[2] = {1, 1};
  return encode_tiled_fn()(m, dtype == LSG_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                           2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Parameters of the shrink + expand tensor-core kernels over the long segments;
// false when this call cannot use them (shape, alignment, workspace).
struct LongPlan {
  TcShrinkParams sp;
  TcExpandParams ep;
  TcFusedParams fp;
  Tc2Params tp;
  Tc3PartParams pp;
  Tc3ExpParams xp;
  StreamParams sp9;
  int stream9 = 0;   // 1: the one-pass streaming kernel (sgmv_stream.cuh)
  int tc3 = 0;       // 1: the cluster-free partials + expand pair (sgmv_tc3.cuh), the default
  int nq = 0, tiles = 0;
  int fused_c = 0;   // > 0: one first-generation fused tensor-core launch, clusters of fused_c CTAs
  int stream_c = 0;  // > 0: one streamed tensor-core launch (sgmv_tc2.cuh), clusters of stream_c CTAs
  uint32_t stream_smem = 0;
};

// Streamed tensor-core kernel plan (ranks 16 / 32): the smallest cluster C in {8, 16}
// whose per-CTA share (its K boxes, at most two 256-column expand chunks) fits shared
// memory with a ring of >= 4 boxes when the ring also stages y chunk 1.  Depends on
// the shape only (the canonical K split of these rows).
struct Tc2Choice {
  int C = 0, kbs = 0, chs = 0, stages = 0;
  uint32_t smem = 0;
};
bool tc2_choose(const lsg_weight_table* t, Tc2Choice* out) {
  if ((t->rank != 16 && t->rank != 32) || t->h_in % kTcKB != 0 || t->h_out % kTcNT != 0 ||
      t->a_layer_stride % 8 != 0 || t->b_layer_stride % 8 != 0)
    return false;
  const int nkb = t->h_in / kTcKB, nch = t->h_out / kTcNT;
  for (int C : {8, 16}) {
    if (nkb < C) continue;
    const int kbs = (nkb + C - 1) / C, chs = (nch + C - 1) / C;
    if (chs > 2) continue;
    const int smin = chs == 2 ? 4 : 1;
    for (int stages = std::max(smin, std::min(kbs, kT2MaxStages)); stages >= smin; --stages) {
      const Tc2Layout L = tc2_layout(t->rank, kbs, chs, stages);
      if (L.total <= static_cast<uint32_t>(kSmemBudget)) {
        if (out) *out = Tc2Choice{C, kbs, chs, stages, L.total};
        return true;
      }
    }
  }
  return false;
}

// Cluster size of the fused tensor-core kernel for this shape (0: not applicable).
// Rank 16 only; every CTA expands at most two 256-column chunks.
// Compact form (one chunk per CTA, y staged in the x ring; two CTAs per SM) when
// the chunks fit one per CTA of a 16-CTA cluster, else two chunks per CTA.
int tc_fused_c(const lsg_weight_table* t, int* compact = nullptr) {
  if (t->rank != 16 || t->h_in % kTcKB != 0 || t->h_out % kTcNT != 0) return 0;
  const int nch = t->h_out / kTcNT, nkb = t->h_in / kTcKB;
  for (int c : {16, 8}) {
    const int per = (nch + c - 1) / c;
    if (per > 2 || nkb < c) continue;
    const int kcs_max = ((nkb + c - 1) / c) * kTcKB, cp = per == 1 ? 1 : 0;
    if (tcf_layout(kcs_max, cp).total <= static_cast<uint32_t>(kSmemBudget)) {
      if (compact) *compact = cp;
      return c;
    }
  }
  return 0;
}
// B [R][h_out] as 3-D {64 columns, R rows, h_out / 64 column blocks} (strides h_out * 2, 128
// bytes), box {64, R, blocks}, SW128: one copy lands `blocks` [R][64] blocks back to back
bool encode_b_blocks(CUtensorMap* m, int dtype, const void* base, int h_out, int R, int blocks) {
  const cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(R), static_cast<cuuint64_t>(h_out / 64)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(h_out) * 2, 128};
  const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(R), static_cast<cuuint32_t>(blocks)};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode_tiled_fn()(m, dtype == LSG_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                           3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// activations [rows][cols] (leading dimension ld) as 3-D {64 columns, rows, cols / 64 blocks}
// (strides ld * 2, 128 bytes), box {64, 16 rows, blocks}, SW128: one copy lands a 16-row tile's
// `blocks` column blocks as [block][16 rows][64] (K9's activation stages)
bool encode_rows_blocks(CUtensorMap* m, int dtype, const void* base, int cols, int rows, int64_t ld, int blocks) {
  const cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols / 64)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 2, 128};
  const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(kMmaM), static_cast<cuuint32_t>(blocks)};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode_tiled_fn()(m, dtype == LSG_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                           3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
bool prepare_long_segments(LongPlan& lp, void* y, int64_t ldy, const void* x, int64_t ldx,
                           const lsg_weight_table* tbl, const int32_t* seg_starts, const int32_t* seg_slot, int n_seg,
                           int s_n, int layer, void* ws, size_t ws_bytes) {
  const int nq = tc_nq(tbl);
  if (nq == 0 || s_n < tc_min_rows(tbl) || tc_tile_bound(tbl, s_n, n_seg) > kMaxGridY) return false;
  if (!aligned16(x) || !aligned16(y) || ldx % 8 != 0 || ldy % 8 != 0 || encode_tiled_fn() == nullptr) return false;
  if (stream_ok(tbl, s_n)) {
    const int tiles = stream_tiles(tbl, s_n, n_seg), R = tbl->rank;
    if (ws == nullptr || !aligned16(ws) || ws_bytes < static_cast<size_t>(tiles) * 256) return false;
    StreamParams& q = lp.sp9;
    q = StreamParams{};
    const int abox = R == 16 ? stream_a_box_rows(16) : R == 32 ? stream_a_box_rows(32) : stream_a_box_rows(64);
    if (!encode_map_2d(&q.tmap_a, tbl->dtype, x, 64, static_cast<uint64_t>(tbl->h_in) * R / 64, 64, 64, abox,
                       CU_TENSOR_MAP_SWIZZLE_128B) ||
        !encode_b_blocks(&q.tmap_b, tbl->dtype, x, tbl->h_out, R, stream_kc(R) / 64) ||
        !encode_rows_blocks(&q.tmap_x, tbl->dtype, x, tbl->h_in, s_n, ldx, stream_kc(R) / 64) ||
        !encode_rows_blocks(&q.tmap_y, tbl->dtype, y, tbl->h_out, s_n, ldy, stream_kc(R) / 64) ||
        !encode_rows_blocks(&q.tmap_y1, tbl->dtype, y, tbl->h_out, s_n, ldy, 1))
      return false;
    q.x = x;
    q.y = y;
    q.ldx = ldx;
    q.ldy = ldy;
    q.a_ptr = tbl->a_ptr;
    q.b_ptr = tbl->b_ptr;
    q.a_off = static_cast<int64_t>(layer) * tbl->a_layer_stride;
    q.b_off = static_cast<int64_t>(layer) * tbl->b_layer_stride;
    q.seg_starts = seg_starts;
    q.seg_slot = seg_slot;
    q.maps = static_cast<uint8_t*>(ws);
    q.n_seg = n_seg;
    q.s_n = s_n;
    q.num_slots = tbl->num_slots;
    q.h_in = tbl->h_in;
    q.h_out = tbl->h_out;
    const int kc = R == 16 ? stream_kc(16) : stream_kc(32), nst = tbl->h_in / kc + tbl->h_out / kc;
    const uint32_t fixed = R == 16 ? stream_fixed(16) : R == 32 ? stream_fixed(32) : stream_fixed(64);
    const uint32_t slotb = R == 16 ? stream_slot_bytes(16) : R == 32 ? stream_slot_bytes(32) : stream_slot_bytes(64);
    // >= 2 slots: the expand releases a slot only after the NEXT stage's stores are issued
    q.stages = std::min({nst, kStreamMaxStages, static_cast<int>((stream_smem_budget(R) - fixed) / slotb)});
    if (q.stages < 2 || nst < 2) return false;
    lp.stream9 = 1;
    lp.tiles = tiles;
    q.min_rows = tc_min_rows(tbl);
    q.trace = g_trace;
    q.trace_ctas = g_trace_ctas;
    return true;
  }
  if (tc3_ok(tbl, s_n)) {
    if (ws == nullptr || !aligned16(ws) || ws_bytes < tc3_ws_bytes(tbl, s_n, n_seg)) return false;
    Tc3PartParams& pp = lp.pp;
    Tc3ExpParams& xp = lp.xp;
    pp = Tc3PartParams{};
    xp = Tc3ExpParams{};
    if (!encode_rows_map(&pp.tmap_x, tbl->dtype, x, tbl->h_in, s_n, ldx) ||
        !encode_rows_map(&xp.tmap_y, tbl->dtype, y, tbl->h_out, s_n, ldy))
      return false;
    lp.tc3 = 1;
    lp.tiles = tc_tile_bound(tbl, s_n, n_seg);
    pp.ws = static_cast<float*>(ws);
    pp.a_ptr = tbl->a_ptr;
    pp.a_off = static_cast<int64_t>(layer) * tbl->a_layer_stride;
    pp.seg_starts = seg_starts;
    pp.seg_slot = seg_slot;
    pp.n_seg = n_seg;
    pp.s_n = s_n;
    pp.num_slots = tbl->num_slots;
    pp.h_in = tbl->h_in;
    pp.kparts = tc3_kparts(tbl->h_in);
    pp.min_rows = tc_min_rows(tbl);
    pp.trace = g_trace;
    pp.trace_ctas = g_trace_ctas;
    xp.y = y;
    xp.ldy = ldy;
    xp.ws = static_cast<const float*>(ws);
    xp.b_ptr = tbl->b_ptr;
    xp.b_off = static_cast<int64_t>(layer) * tbl->b_layer_stride;
    xp.seg_starts = seg_starts;
    xp.seg_slot = seg_slot;
    xp.n_seg = n_seg;
    xp.s_n = s_n;
    xp.num_slots = tbl->num_slots;
    xp.h_out = tbl->h_out;
    xp.kparts = pp.kparts;
    xp.min_rows = pp.min_rows;
    xp.trace = g_trace;
    xp.trace_ctas = g_trace_ctas;
    return true;
  }
  Tc2Choice ch;
  if (!cur().tc_split && cur().tc_legacy == 2 && tc2_choose(tbl, &ch)) {
    Tc2Params& tp = lp.tp;
    tp = Tc2Params{};
    if (!encode_rows_map(&tp.tmap_x, tbl->dtype, x, tbl->h_in, s_n, ldx) ||
        !encode_rows_map(&tp.tmap_y, tbl->dtype, y, tbl->h_out, s_n, ldy))
      return false;
    lp.stream_c = ch.C;
    lp.stream_smem = ch.smem;
    lp.tiles = tc_tile_bound(tbl, s_n, n_seg);
    tp.y = y;
    tp.ldy = ldy;
    tp.a_ptr = tbl->a_ptr;
    tp.b_ptr = tbl->b_ptr;
    tp.a_off = static_cast<int64_t>(layer) * tbl->a_layer_stride;
    tp.b_off = static_cast<int64_t>(layer) * tbl->b_layer_stride;
    tp.seg_starts = seg_starts;
    tp.seg_slot = seg_slot;
    tp.n_seg = n_seg;
    tp.s_n = s_n;
    tp.num_slots = tbl->num_slots;
    tp.h_in = tbl->h_in;
    tp.h_out = tbl->h_out;
    tp.kbs_max = ch.kbs;
    tp.chs_max = ch.chs;
    tp.stages = ch.stages;
    tp.min_rows = tc_min_rows(tbl);
    tp.tiles = lp.tiles;
    tp.trace = g_trace;
    tp.trace_ctas = g_trace_ctas;
    return true;
  }
  int compact = 0;
  const int fc = cur().tc_split || cur().tc_legacy != 1 ? 0 : tc_fused_c(tbl, &compact);
  if (fc > 0) {
    TcFusedParams& fp = lp.fp;
    fp = TcFusedParams{};
    if (!encode_rows_map(&fp.tmap_x, tbl->dtype, x, tbl->h_in, s_n, ldx) ||
        !encode_rows_map(&fp.tmap_y, tbl->dtype, y, tbl->h_out, s_n, ldy))
      return false;
    lp.fused_c = fc;
    lp.tiles = tc_tile_bound(tbl, s_n, n_seg);
    fp.y = y;
    fp.ldy = ldy;
    fp.a_ptr = tbl->a_ptr;
    fp.b_ptr = tbl->b_ptr;
    fp.a_off = static_cast<int64_t>(layer) * tbl->a_layer_stride;
    fp.b_off = static_cast<int64_t>(layer) * tbl->b_layer_stride;
    fp.seg_starts = seg_starts;
    fp.seg_slot = seg_slot;
    fp.n_seg = n_seg;
    fp.s_n = s_n;
    fp.num_slots = tbl->num_slots;
    fp.h_in = tbl->h_in;
    fp.h_out = tbl->h_out;
    fp.kcs_max = ((tbl->h_in / kTcKB + fc - 1) / fc) * kTcKB;
    fp.compact = compact;
    fp.min_rows = tc_min_rows(tbl);
    fp.trace = g_trace;
    fp.trace_ctas = g_trace_ctas;
    return true;
  }
  if (ws == nullptr || ws_bytes < tc_workspace_bytes(tbl, s_n) || !aligned16(ws)) return false;
  TcShrinkParams& sp = lp.sp;
  TcExpandParams& ep = lp.ep;
  sp = TcShrinkParams{};
  ep = TcExpandParams{};
  if (!encode_rows_map(&sp.tmap_x, tbl->dtype, x, tbl->h_in, s_n, ldx) ||
      !encode_rows_map(&ep.tmap_y, tbl->dtype, y, tbl->h_out, s_n, ldy))
    return false;
  // tiles of long segments: sum ceil(len/128) over len >= 128 is at most s_n/64
  const int tiles = tc_tile_bound(tbl, s_n, n_seg);
  lp.nq = nq;
  lp.tiles = tiles;
  sp.v = static_cast<float*>(ws);
  sp.a_ptr = tbl->a_ptr;
  sp.a_off = static_cast<int64_t>(layer) * tbl->a_layer_stride;
  sp.seg_starts = seg_starts;
  sp.seg_slot = seg_slot;
  sp.n_seg = n_seg;
  sp.s_n = s_n;
  sp.num_slots = tbl->num_slots;
  sp.h_in = tbl->h_in;
  sp.kcs = tbl->h_in / nq;
  sp.min_rows = tc_min_rows(tbl);
  sp.trace = g_trace;
  sp.trace_ctas = g_trace_ctas;
  ep.y = y;
  ep.ldy = ldy;
  ep.v = static_cast<const float*>(ws);
  ep.b_ptr = tbl->b_ptr;
  ep.b_off = static_cast<int64_t>(layer) * tbl->b_layer_stride;
  ep.seg_starts = seg_starts;
  ep.seg_slot = seg_slot;
  ep.n_seg = n_seg;
  ep.s_n = s_n;
  ep.num_slots = tbl->num_slots;
  ep.h_out = tbl->h_out;
  ep.min_rows = tc_min_rows(tbl);
  ep.trace = g_trace;
  ep.trace_ctas = g_trace_ctas;
  return true;
}

int launch_long_segments(const LongPlan& lp, int dtype, int rank, cudaStream_t cs) {
  if (lp.stream9) return launch_stream(dtype, rank, lp.sp9, lp.tiles, cs);
  if (lp.tc3) {
    const int st = launch_tc3_parts(dtype, rank, lp.pp, lp.tiles, cs);
    if (st != LSG_OK) return st;
    return launch_tc3_expand(dtype, rank, lp.xp, lp.tiles, cs);
  }
  if (lp.stream_c > 0) return launch_tc_stream(dtype, rank, lp.tp, lp.stream_c, lp.stream_smem, lp.tiles, cs);
  if (lp.fused_c > 0) return launch_tc_fused(dtype, lp.fp, lp.fused_c, lp.tiles, cs);
  const int st = launch_tc_shrink(dtype, rank, lp.sp, lp.nq, lp.tiles, cs);
  if (st != LSG_OK) return st;
  return launch_tc_expand(dtype, rank, lp.ep, lp.tiles, cs);
}

enum Kernel { kKFused = 0, kKShrink = 1, kKExpand = 2, kKBgmv = 3 };


// Destinations of a tensor-parallel launch: every rank's y, at this rank's columns.
struct TpDest {
  int n;
  void* y[kMaxSites];
};

int validate_table(const lsg_weight_table* t) {
  if (t == nullptr) return fail(LSG_EINVAL, "lsg: weight table is NULL");
  if (t->a_ptr == nullptr || t->b_ptr == nullptr) return fail(LSG_EINVAL, "lsg: weight table pointer arrays are NULL");
  if (t->num_slots < 0 || t->num_layers < 1) return fail(LSG_EINVAL, "lsg: weight table slot/layer counts invalid");
  if (t->h_in < 1 || t->h_out < 1) return fail(LSG_EINVAL, "lsg: weight table dims must be >= 1");
  // Same invariant as LoraModel (sgmv.cpp:45-56): 1 <= rank <= min(h_in, h_out).
  if (t->rank < 1 || t->rank > t->h_in || t->rank > t->h_out)
    return fail(LSG_EINVAL, "lsg: rank must satisfy 1 <= rank <= min(h_in, h_out)");
  if (t->rank > 1024) return fail(LSG_EUNSUPPORTED, "lsg: rank > 1024 is not supported");
  if (t->a_layer_stride < static_cast<int64_t>(t->h_in) * t->rank ||
      t->b_layer_stride < static_cast<int64_t>(t->rank) * t->h_out)
    return fail(LSG_EINVAL, "lsg: layer strides smaller than one layer");
  if (t->dtype != LSG_F16 && t->dtype != LSG_BF16) return fail(LSG_EINVAL, "lsg: unknown dtype");
  return LSG_OK;
}

bool fast_shape_ok(const lsg_weight_table* t) {
  const int r = t->rank;
  return (r == 8 || r == 16 || r == 32 || r == 64) && t->h_in % KW == 0 && t->h_out % 8 == 0 &&
         t->a_layer_stride % 8 == 0 && t->b_layer_stride % 8 == 0;
}

// Choose tile rows, row splits and the split-K cluster size for a launch.
// long_on_tc: the launch's long / shared segments go to tensor-core kernels; short_rows > 0:
// the segments left to this kernel are shorter than short_rows rows.
Plan make_plan(const lsg_weight_table* t, int kernel, int n_seg, int s_n, bool fast, bool long_on_tc = false,
               int short_rows = 0) {
  Plan pl;
  pl.mode = kernel == kKShrink ? kShrink : kernel == kKExpand ? kExpand : kFused;
  if (!fast || cur().force_generic) {
    pl.path = 1;
    pl.clusters = s_n;
    pl.smem = t->rank * 4;
    return pl;
  }
  const int forced_mt = cur().force_tile_rows;
  if (kernel == kKBgmv)
    pl.mt = 1;
  else if (forced_mt == 1 || forced_mt == 8 || (forced_mt == 4 && t->rank == 64 && kernel == kKFused))
    pl.mt = forced_mt;
  else if (t->rank == 64 && s_n > n_seg && !cur().no_rank64_tiles && !(short_rows > 0 && short_rows <= 8))
    pl.mt = 8;  // rank 64, shared adapters: one weight read per 8-row tile (c3)
  else
    pl.mt = 1;  // one row per cluster: the shortest critical path per launch (profiles/README.md)
  if (kernel == kKBgmv) {
    pl.row_splits = 1;
    pl.clusters = s_n;
  } else if ((pl.mt > 1 || s_n > n_seg) && !(cur().no_tile_scan)) {
    // one cluster per row tile, mapped on the device; sum_i ceil(len_i/MT) is
    // at most (s_n + n_seg*(MT-1))/MT, and never more than s_n
    pl.tile_scan = 1;
    pl.row_splits = 1;
    const int64_t bound = (static_cast<int64_t>(s_n) + static_cast<int64_t>(n_seg) * (pl.mt - 1)) / pl.mt;
    pl.clusters = static_cast<int>(std::min<int64_t>(bound, s_n));
  } else {
    const int tiles_per_seg = (s_n + pl.mt * n_seg - 1) / (pl.mt * n_seg);
    pl.row_splits = pl.mt == 1 ? 1 : std::max(1, tiles_per_seg);  // the MT=1 kernel assumes 1
    pl.clusters = n_seg * pl.row_splits;
  }
  const int nq = t->h_in / KW, ncvt = t->h_out / 8;
  // one-round reduction (every CTA receives every chunk partial) while that
  // receive buffer stays <= 16 KB; otherwise owner-sliced with a second round
  auto red_all_for = [&](int) { return pl.mode == kFused && pl.mt == 1 ? 1 : 0; };  // must match the kernel
  // Single-tile clusters (every segment one tile) keep only A resident ahead of
  // the PDL wait and prefetch B into L2, so two launches' CTAs fit per SM.
  // (s_n == n_seg: every segment is one row, so every cluster has exactly one tile)
  // (only when keeping B resident as well would cost co-residency: three CTAs per SM)
  const bool single_tile = kernel == kKBgmv || s_n == n_seg || pl.tile_scan;
  auto smem_alias = [&](int c, int alias) {
    const int nqc = (nq + c - 1) / c, ncv = (ncvt + c - 1) / c;
    return static_cast<int>(make_layout(pl.mode, t->rank, pl.mt, c, nq, nqc, ncv, red_all_for(c), alias).total);
  };
  auto alias_for = [&](int c) {
    const int o = cur().no_alias;  // 1: never, -1: always (single-tile launches), 0: when co-residency needs it
    // (multi-row tiles never alias: their expand widens B to fp32 over A / x, sgmv_kernels.cuh)
    if (pl.mode != kFused || !single_tile || o > 0 || pl.mt > 1) return 0;
    return o < 0 || smem_alias(c, 0) > kCoresidentSmem ? 1 : 0;
  };
  auto smem_for = [&](int c) { return smem_alias(c, alias_for(c)); };
  // Split-K cluster size.  Candidates divide the chunk / column-group counts
  // (every CTA gets the same share).  Measured on B200 (profiles/README.md):
  // a launch runs best with about 128-256 CTAs in all, and clusters of 8-16
  // schedule poorly once the grid needs more than one CTA per SM.  So take the
  // largest candidate whose grid stays within 148 CTAs (C >= 8) or 256 CTAs
  // (C <= 4; tile-scan launches: 256 for every C); if none does, the smallest
  // candidate that fits in shared memory.  With the long segments on the tensor
  // cores, the CUDA-core launch serves short segments only: estimate one
  // cluster per segment.
  const int span = std::max(1, pl.mode == kExpand ? ncvt : pl.mode == kShrink ? nq : std::gcd(nq, ncvt));
  const int64_t est_clusters = long_on_tc ? n_seg : pl.clusters;
  int c = 0, c_small = 0;
  const int c_cap = kMaxCluster;
  // Launches with a shrink reduce over DSMEM with st.async, which needs a real
  // cluster (compute-sanitizer memcheck: "Cluster needs to have at least 2 blocks"):
  // at least 2 CTAs (a CTA without chunks only receives).  Expand-only launches: 1.
  const int c_min = pl.mode == kExpand ? 1 : 2;
  for (int cand = c_min; cand <= c_cap; ++cand) {
    if (span % cand != 0 && cand != c_cap && cand != c_min) continue;
    if (smem_for(cand) > kSmemBudget) continue;
    if (c_small == 0) c_small = cand;
    // behind the rank-16 streaming kernel (K9) the short-segment CTAs share SMs with its CTAs
    // (one each): at most ~128 CTAs (c4: C = 8 -> 4, 14.8 -> 14.1 us)
#ifndef LSG_DECODE_CAP_MAX_RANK
#define LSG_DECODE_CAP_MAX_RANK 16
#endif
    const int64_t limit = (long_on_tc && t->rank <= LSG_DECODE_CAP_MAX_RANK && stream_ok(t, s_n)) ? 128
                          : (pl.tile_scan || cand <= 4)                       ? 256
                                                                              : 148;
    if (est_clusters * cand <= limit) c = cand;
  }
  if (c == 0) c = c_small;
  // nothing within the cap fits shared memory (e.g. rank 64 at h = 8192): the smallest
  // larger cluster that does
  for (int cand = c_cap + 1; c == 0 && cand <= kMaxCluster; ++cand)
    if ((span % cand == 0 || cand == kMaxCluster) && smem_for(cand) <= kSmemBudget) c = cand;
  if (c == 0) c = kMaxCluster;
  const int forced = cur().force_cluster;
  if (forced >= 1 && forced <= kMaxCluster && smem_for(std::max(forced, c_min)) <= kSmemBudget)
    c = std::max(forced, c_min);
  pl.red_all = red_all_for(c);
  pl.alias_ab = alias_for(c);
  pl.cluster = c;
  pl.nqc_max = (nq + c - 1) / c;
  pl.ncv_max = (ncvt + c - 1) / c;
  pl.smem = smem_for(c);
  return pl;
}

// Shared entry for all four SGMV kernels.
int run(int kernel, void* y, int64_t ldy, const void* x, int64_t ldx, float* v_out, const float* v_in,
        const lsg_weight_table* tbl, const int32_t* seg_starts, const int32_t* seg_slot,
        const int32_t* row_slot, int32_t n_seg, int32_t s_n, int32_t layer, lsg_stream_t stream,
        void* ws = nullptr, size_t ws_bytes = 0, bool library_ws = false, const lsg_sgmv_site* sites = nullptr,
        int n_sites = 0, const TpDest* tp = nullptr) {
  int st = validate_table(tbl);
  if (st != LSG_OK) return st;
  if (s_n < 0) return fail(LSG_EINVAL, "lsg: total_rows must be >= 0");
  if (kernel != kKBgmv && n_seg < 0) return fail(LSG_EINVAL, "lsg: num_segments must be >= 0");
  if (layer < 0 || layer >= tbl->num_layers) return fail(LSG_EINVAL, "lsg: layer index out of range");
  if (s_n == 0 || (kernel != kKBgmv && n_seg == 0)) return LSG_OK;  // empty batch: nothing to do
  if (kernel == kKBgmv ? row_slot == nullptr : (seg_starts == nullptr || seg_slot == nullptr))
    return fail(LSG_EINVAL, "lsg: segment metadata pointers are NULL");
  const bool need_x = kernel != kKExpand, need_y = kernel != kKShrink;
  if (need_x && (x == nullptr || ldx < tbl->h_in)) return fail(LSG_EINVAL, "lsg: x is NULL or ldx < h_in");
  if (need_y && (y == nullptr || ldy < tbl->h_out)) return fail(LSG_EINVAL, "lsg: y is NULL or ldy < h_out");
  if (kernel == kKShrink && v_out == nullptr) return fail(LSG_EINVAL, "lsg: v is NULL");
  if (kernel == kKExpand && v_in == nullptr) return fail(LSG_EINVAL, "lsg: v is NULL");

  bool fast = fast_shape_ok(tbl);
  if (need_x) fast = fast && aligned16(x) && ldx % 8 == 0;
  if (need_y) fast = fast && aligned16(y) && ldy % 8 == 0;
  const Plan pl0 = make_plan(tbl, kernel, n_seg, s_n, fast);
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);

  if (pl0.path == 1) {
    const Plan& pl = pl0;
    GenericParams g{};
    g.y = y;
    g.x = x;
    g.v_out = v_out;
    g.v_in = v_in;
    g.a_ptr = tbl->a_ptr;
    g.b_ptr = tbl->b_ptr;
    g.a_off = static_cast<int64_t>(layer) * tbl->a_layer_stride;
    g.b_off = static_cast<int64_t>(layer) * tbl->b_layer_stride;
    g.ldx = ldx;
    g.ldy = ldy;
    g.seg_starts = seg_starts;
    g.seg_slot = seg_slot;
    g.row_slot = kernel == kKBgmv ? row_slot : nullptr;
    g.n_seg = n_seg;
    g.s_n = s_n;
    g.num_slots = tbl->num_slots;
    g.h_in = tbl->h_in;
    g.h_out = tbl->h_out;
    g.rank = tbl->rank;
    return launch_generic(tbl->dtype, pl.mode, g, s_n, pl.smem, cs);
  }

  // Long segments (>= kTcMinRows rows) of a fused launch go to the tensor-core
  // kernels; the CUDA-core kernel then skips them.
  // Launch order: tensor-core shrink and expand (long segments), then the CUDA-core
  // kernel (short segments), whose CTAs become resident under the expand and
  // stream their weights there (measured neutral on c4, 24.0 us either way).  The
  // tensor-core shrink triggers its dependents only after its own PDL wait, so the
  // expand may stage y_old before waiting for v.
  // Rows of segments in [mma_lo, mma_hi) go to the segment-tile MMA pair (K7), rows of
  // segments >= tc_lo to the long-segment tensor-core kernels (K5); the CUDA-core kernel
  // then skips every segment of >= skip_long rows -- or is not launched at all when the
  // tensor-core kernels cover every segment.  Workspace: [MMA partials | K5 v].
  int skip_long = 0;
  bool cuda_core = true;
  LongPlan lp;
  MmaParams mp{};
  int mma_tiles = 0;
  bool use_tc = false, use_mma = false;
  if (kernel == kKFused) {
    RowRanges rr = row_ranges(tbl, n_seg, s_n);
    if (rr.mma_lo > 0 || rr.tc_lo > 0) {
      const size_t mma_b = rr.mma_lo > 0 ? align256(mma_ws_bytes(tbl, s_n, n_seg, rr.mma_lo)) : 0;
      if (library_ws) {
        ws_bytes = mma_b + (rr.tc_lo > 0 ? tc_workspace_bytes(tbl, s_n) : 0);
        ws = ws_bytes > 0 ? library_workspace(ws_bytes, cs) : nullptr;
        if (ws == nullptr) ws_bytes = 0;
      }
      if (rr.tc_lo > 0) {
        void* tws = ws != nullptr && ws_bytes >= mma_b ? static_cast<char*>(ws) + mma_b : nullptr;
        use_tc = prepare_long_segments(lp, y, ldy, x, ldx, tbl, seg_starts, seg_slot, n_seg, s_n, layer, tws,
                                       tws != nullptr ? ws_bytes - mma_b : 0);
        if (!use_tc) {
          if (rr.mma_lo > 0) rr.mma_hi = kRowsInf;  // the MMA pair takes the long segments too
          rr.tc_lo = 0;
        }
      }
      use_mma = prepare_mma(mp, mma_tiles, rr, y, ldy, x, ldx, tbl, seg_starts, seg_slot, n_seg, s_n, layer, ws,
                            ws_bytes);
      if (use_mma) {
        skip_long = rr.mma_lo;
        cuda_core = !(rr.mma_lo == 1 && rr.mma_hi == kRowsInf);
      } else if (use_tc) {
        skip_long = rr.tc_lo;
      }
    }
  }
  Plan pl = skip_long ? make_plan(tbl, kernel, n_seg, s_n, fast, true, skip_long) : pl0;
  // One-row tiles without a long-segment split: one cluster per row, exact grid.
  if (pl.mt == 1 && kernel != kKBgmv && !skip_long && !cur().no_row_mode && s_n <= kMaxGridY) {
    pl.row_mode = 1;
    pl.tile_scan = 0;
    pl.row_splits = 1;
    pl.clusters = s_n;
  }
  if (n_sites > 1) {  // grouped launch: one cluster per (site, row)
    // lsg_sgmv_multi checks eligibility; the grouped item mode exists for one-row
    // row-mode launches only, so anything else is refused here, never run partially
    if (!pl.row_mode || pl.mt != 1 || skip_long || static_cast<int64_t>(n_sites) * s_n > kMaxGridY)
      return fail(LSG_EINVAL, "lsg_sgmv_multi: grouped launch needs one-row row-mode tiles");
    pl.multi = 1;
    pl.clusters = n_sites * s_n;
  }
  if (tp != nullptr) {  // tensor-parallel expand: the grouped item mode's store into every rank's y
    if (!pl.row_mode || pl.mt != 1 || skip_long || kernel != kKFused)
      return fail(LSG_EUNSUPPORTED, "lsg_tp_sgmv: decode batches only (one-row tiles, no long segments)");
    pl.tp = 1;
  }
  // Launches with one work item per cluster put the item count in gridDim.y (max
  // 65535): above that, clusters loop over tiles (tile-scan decode) instead.
  if (!pl.tile_scan && !pl.multi && kernel != kKBgmv && pl.clusters > kMaxGridY) {
    pl.row_mode = 0;
    pl.tile_scan = 1;
    pl.row_splits = 1;
    const int64_t bound = (static_cast<int64_t>(s_n) + static_cast<int64_t>(n_seg) * (pl.mt - 1)) / pl.mt;
    pl.clusters = static_cast<int>(std::min<int64_t>(bound, s_n));  // capped at launch (launch_fast_inst)
  }
  // With the long segments on the tensor cores, the short ones have at most n_seg
  // segments' worth of work items in practice: size the tile-scan grid by that
  // (clusters loop over further tiles) instead of by s_n.
// ... but at least ~256 CTAs: the host does not know how many rows the short segments hold, and
// a grid of n_seg clusters starves calls with few, long-ish short segments (four 100-row
// segments in a call with a tensor-core pass: 4 clusters).  Measured: c4 13.5 -> 13.4 us,
// 1024-row prefill + decodes 11.6 -> 10.8, two 300-row segments under a 384 threshold 1117 -> 156.
#ifndef LSG_SKIP_LONG_MIN_CTAS
#define LSG_SKIP_LONG_MIN_CTAS 256
#endif
  if (skip_long && pl.tile_scan)
    pl.clusters = std::min(pl.clusters, std::max({1, n_seg, LSG_SKIP_LONG_MIN_CTAS / std::max(1, pl.cluster)}));

  FastParams p{};
  p.y = y;
  p.x = x;
  p.v_out = v_out;
  p.v_in = v_in;
  p.a_ptr = tbl->a_ptr;
  p.b_ptr = tbl->b_ptr;
  p.a_off = static_cast<int64_t>(layer) * tbl->a_layer_stride;
  p.b_off = static_cast<int64_t>(layer) * tbl->b_layer_stride;
  p.ldx = ldx;
  p.ldy = ldy;
  p.seg_starts = seg_starts;
  p.seg_slot = seg_slot;
  p.row_slot = kernel == kKBgmv ? row_slot : nullptr;
  p.n_seg = n_seg;
  p.s_n = s_n;
  p.row_splits = pl.row_splits;
  p.num_slots = tbl->num_slots;
  p.h_in = tbl->h_in;
  p.h_out = tbl->h_out;
  p.nq = tbl->h_in / KW;
  p.ncvt = tbl->h_out / 8;
  p.nqc_max = pl.nqc_max;
  p.ncv_max = pl.ncv_max;
  p.red_all = pl.red_all;
  p.alias_ab = pl.alias_ab;
  p.tile_scan = pl.tile_scan;
  p.skip_long = skip_long;
  p.trace = g_trace;
  p.trace_ctas = g_trace_ctas;
  p.n_sites = n_sites > 1 ? n_sites : 0;
  // behind the long / shared-segment kernels (K9, K7's expand and the tcgen05 pair's expand all
  // trigger only after their own PDL wait) the short-segment kernel starts and computes while
  // they run (disjoint rows), waiting for them only at the end
  p.late_wait = (pl.tile_scan && (use_mma || (use_tc && (lp.stream9 || lp.tc3)))) ? 1 : 0;
  for (int i = 0; i < p.n_sites; ++i)
    p.sites[i] = SiteParams{sites[i].y, sites[i].x, sites[i].tbl->a_ptr, sites[i].tbl->b_ptr, sites[i].ldx,
                            sites[i].ldy};
  if (tp != nullptr) {
    p.n_sites = tp->n;
    for (int i = 0; i < tp->n; ++i) p.sites[i] = SiteParams{tp->y[i], x, tbl->a_ptr, tbl->b_ptr, ldx, ldy};
  }
#ifdef LSG_INSTRUMENT
  // experiment switches (instrumented builds only; production kernels compile them out)
  static const int exp_flags = [] {
    const char* e = std::getenv("LSG_EXP");
    return e ? std::atoi(e) : 0;
  }();
  p.exp_flags = exp_flags;
#endif
  if (use_mma) {
    st = launch_mma_pair(tbl->dtype, tbl->rank, mp, mma_tiles, cs);
    if (st != LSG_OK) return st;
  }
  if (use_tc) {
    st = launch_long_segments(lp, tbl->dtype, tbl->rank, cs);
    if (st != LSG_OK) return st;
  }
  if (!cuda_core) return LSG_OK;
  switch (pl.mode) {
    case kFused: st = launch_fast_fused(tbl->dtype, tbl->rank, p, pl, cs); break;
    case kShrink: st = launch_fast_shrink(tbl->dtype, tbl->rank, p, pl, cs); break;
    default: st = launch_fast_expand(tbl->dtype, tbl->rank, p, pl, cs); break;
  }
  return st;
}

}  // namespace

bool pdl_enabled() { return cur().pdl != 0; }


int launch_generic(int dtype, int mode, const GenericParams& g, int rows, int smem, cudaStream_t st) {
  return dtype == LSG_F16 ? dispatch_generic<__half>(g, mode, rows, smem, st)
                          : dispatch_generic<__nv_bfloat16>(g, mode, rows, smem, st);
}

}  // namespace lsg

using namespace lsg;

extern "C" {

int lsg_sgmv(void* y, int64_t ldy, const void* x, int64_t ldx, const lsg_weight_table* tbl,
             const int32_t* seg_starts, const int32_t* seg_slot, int32_t num_segments,
             int32_t total_rows, int32_t layer, lsg_stream_t stream) {
  CallScope scope(nullptr);
  return run(kKFused, y, ldy, x, ldx, nullptr, nullptr, tbl, seg_starts, seg_slot, nullptr,
             num_segments, total_rows, layer, stream, nullptr, 0, true);
}

size_t lsg_sgmv_workspace_size(const lsg_weight_table* tbl, int32_t total_rows) {
  CallScope scope(nullptr);
  if (tbl == nullptr || validate_table(tbl) != LSG_OK || total_rows < 0) return 0;
  return call_ws_bound(tbl, total_rows);
}

int lsg_sgmv_ws(void* y, int64_t ldy, const void* x, int64_t ldx, const lsg_weight_table* tbl,
                const int32_t* seg_starts, const int32_t* seg_slot, int32_t num_segments,
                int32_t total_rows, int32_t layer, void* workspace, size_t workspace_bytes,
                lsg_stream_t stream) {
  CallScope scope(nullptr);
  return run(kKFused, y, ldy, x, ldx, nullptr, nullptr, tbl, seg_starts, seg_slot, nullptr,
             num_segments, total_rows, layer, stream, workspace, workspace_bytes, false);
}

int lsg_sgmv_ex(void* y, int64_t ldy, const void* x, int64_t ldx, const lsg_weight_table* tbl,
                const int32_t* seg_starts, const int32_t* seg_slot, int32_t num_segments, int32_t total_rows,
                int32_t layer, void* workspace, size_t workspace_bytes, const lsg_call_opts* opts,
                lsg_stream_t stream) {
  CallScope scope(opts);
  return run(kKFused, y, ldy, x, ldx, nullptr, nullptr, tbl, seg_starts, seg_slot, nullptr, num_segments,
             total_rows, layer, stream, workspace, workspace_bytes, workspace == nullptr);
}

int lsg_sgmv_multi_ex(const lsg_sgmv_site* sites, int32_t num_sites, const int32_t* seg_starts,
                      const int32_t* seg_slot, int32_t num_segments, int32_t total_rows, int32_t layer,
                      const lsg_call_opts* opts, lsg_stream_t stream) {
  CallScope scope(opts);
  if (sites == nullptr || num_sites < 1 || num_sites > kMaxSites)
    return fail(LSG_EINVAL, "lsg_sgmv_multi: need 1..8 sites");
  const lsg_weight_table* t0 = sites[0].tbl;
  for (int i = 0; i < num_sites; ++i) {
    const lsg_weight_table* t = sites[i].tbl;
    const int st = validate_table(t);
    if (st != LSG_OK) return st;
    if (t->h_in != t0->h_in || t->h_out != t0->h_out || t->rank != t0->rank || t->dtype != t0->dtype ||
        t->num_slots != t0->num_slots || t->num_layers != t0->num_layers ||
        t->a_layer_stride != t0->a_layer_stride || t->b_layer_stride != t0->b_layer_stride)
      return fail(LSG_EINVAL, "lsg_sgmv_multi: sites must share shape, dtype, slot count and layer strides");
  }
  // One grouped launch when every site takes the one-row fast path without long
  // segments; otherwise the sites run one after another (same results).
  // (make_plan decides the tile rows: rank 64 with shared adapters plans 4-row tiles,
  // which the grouped item mode does not have)
  bool grouped = num_sites > 1 && total_rows > 0 && num_segments > 0 && fast_shape_ok(t0) &&
                 !cur().force_generic && !cur().no_row_mode &&
                 static_cast<int64_t>(num_sites) * total_rows <= kMaxGridY &&
                 make_plan(t0, kKFused, num_segments, total_rows, true).mt == 1 &&
                 (cur().no_tc || total_rows < tc_min_rows(t0) || tc_nq(t0) == 0);
  for (int i = 0; grouped && i < num_sites; ++i)
    grouped = sites[i].x != nullptr && sites[i].y != nullptr && aligned16(sites[i].x) && aligned16(sites[i].y) &&
              sites[i].ldx % 8 == 0 && sites[i].ldy % 8 == 0 && sites[i].ldx >= t0->h_in &&
              sites[i].ldy >= t0->h_out;
  if (!grouped) {
    for (int i = 0; i < num_sites; ++i) {
      const int st = run(kKFused, sites[i].y, sites[i].ldy, sites[i].x, sites[i].ldx, nullptr, nullptr, sites[i].tbl,
                         seg_starts, seg_slot, nullptr, num_segments, total_rows, layer, stream, nullptr, 0, true);
      if (st != LSG_OK) return st;
    }
    return LSG_OK;
  }
  return run(kKFused, sites[0].y, sites[0].ldy, sites[0].x, sites[0].ldx, nullptr, nullptr, t0, seg_starts,
             seg_slot, nullptr, num_segments, total_rows, layer, stream, nullptr, 0, true, sites, num_sites);
}

int lsg_sgmv_multi(const lsg_sgmv_site* sites, int32_t num_sites, const int32_t* seg_starts,
                   const int32_t* seg_slot, int32_t num_segments, int32_t total_rows, int32_t layer,
                   lsg_stream_t stream) {
  return lsg_sgmv_multi_ex(sites, num_sites, seg_starts, seg_slot, num_segments, total_rows, layer, nullptr, stream);
}

int lsg_tp_sgmv(const lsg_tp_group* g, int64_t ldy, const void* x, int64_t ldx, const lsg_weight_table* shard,
                const int32_t* seg_starts, const int32_t* seg_slot, int32_t num_segments, int32_t total_rows,
                int32_t layer, uint32_t epoch, lsg_stream_t stream) {
  lsg_call_opts o{-1, -1, 1, -1};  // decode batches: long segments would need the tensor-core kernels
  CallScope scope(&o);
  if (g == nullptr || g->size < 1 || g->size > kMaxSites || g->rank < 0 || g->rank >= g->size ||
      g->y_peer == nullptr || g->flag_peer == nullptr)
    return fail(LSG_EINVAL, "lsg_tp_sgmv: bad group (size 1..8, rank < size, peer arrays)");
  int st = validate_table(shard);
  if (st != LSG_OK) return st;
  if (epoch == 0) return fail(LSG_EINVAL, "lsg_tp_sgmv: epoch must be non-zero (flags start at 0)");
  TpDest d{};
  d.n = g->size;
  const int64_t c0 = static_cast<int64_t>(g->rank) * shard->h_out;  // this rank's columns
  for (int r = 0; r < g->size; ++r) {
    if (g->y_peer[r] == nullptr || g->flag_peer[r] == nullptr) return fail(LSG_EINVAL, "lsg_tp_sgmv: NULL peer buffer");
    d.y[r] = static_cast<char*>(g->y_peer[r]) + c0 * 2;
  }
  if (ldy < static_cast<int64_t>(g->size) * shard->h_out)
    return fail(LSG_EINVAL, "lsg_tp_sgmv: ldy < size * h_out (y rows hold every rank's columns)");
  st = run(kKFused, d.y[g->rank], ldy, x, ldx, nullptr, nullptr, shard, seg_starts, seg_slot, nullptr, num_segments,
           total_rows, layer, stream, nullptr, 0, false, nullptr, 0, &d);
  if (st != LSG_OK) return st;
  // every rank's stores are complete (stream order) -> raise my flag at every rank, then
  // wait for every rank's flag at mine (epoch-stamped, no reset needed between steps)
  TpFlagParams f{};
  f.rank = g->rank;
  f.size = g->size;
  f.epoch = epoch;
  f.my_flag = g->flag_peer[g->rank];
  for (int r = 0; r < g->size; ++r) f.peer_flag[r] = g->flag_peer[r];
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  tp_flags_kernel<<<1, 32, 0, cs>>>(f);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? LSG_OK : cuda_fail(e, "tp_flags_kernel launch");
}

size_t lsg_tp_nccl_workspace_size(int32_t total_rows, int32_t h_out_shard, int32_t tp_size) {
  if (total_rows < 0 || h_out_shard < 0 || tp_size < 1) return 0;
  return static_cast<size_t>(tp_size + 1) * total_rows * h_out_shard * 2;
}

int lsg_tp_sgmv_nccl(void* y, int64_t ldy, const void* x, int64_t ldx, const lsg_weight_table* shard,
                     const int32_t* seg_starts, const int32_t* seg_slot, int32_t num_segments, int32_t total_rows,
                     int32_t layer, int32_t tp_rank, int32_t tp_size, void* nccl_comm, void* workspace,
                     size_t workspace_bytes, lsg_stream_t stream) {
  CallScope scope(nullptr);
  int st = validate_table(shard);
  if (st != LSG_OK) return st;
  if (tp_size < 1 || tp_rank < 0 || tp_rank >= tp_size || nccl_comm == nullptr || y == nullptr)
    return fail(LSG_EINVAL, "lsg_tp_sgmv_nccl: bad rank / size / communicator");
  const int64_t w = shard->h_out;
  if (ldy < tp_size * w) return fail(LSG_EINVAL, "lsg_tp_sgmv_nccl: ldy < size * h_out");
  if (total_rows < 0) return fail(LSG_EINVAL, "lsg_tp_sgmv_nccl: total_rows < 0");
  if (total_rows == 0) return LSG_OK;
  if (workspace == nullptr || workspace_bytes < lsg_tp_nccl_workspace_size(total_rows, static_cast<int32_t>(w), tp_size))
    return fail(LSG_EINVAL, "lsg_tp_sgmv_nccl: workspace too small (lsg_tp_nccl_workspace_size)");
  using AllGatherFn = int (*)(const void*, void*, size_t, int, void*, cudaStream_t);
  static AllGatherFn allgather = [] {
    void* f = dlsym(RTLD_DEFAULT, "ncclAllGather");
    if (f == nullptr) {
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (h != nullptr) f = dlsym(h, "ncclAllGather");
    }
    return reinterpret_cast<AllGatherFn>(f);
  }();
  if (allgather == nullptr) return fail(LSG_EUNSUPPORTED, "lsg_tp_sgmv_nccl: libnccl.so.2 not found");
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  char* yb = static_cast<char*>(y);
  const int64_t c0 = tp_rank * w;
  // 1. this rank's column slice of y += x . A . B_shard (in place, strided)
  st = run(kKFused, yb + c0 * 2, ldy, x, ldx, nullptr, nullptr, shard, seg_starts, seg_slot, nullptr, num_segments,
           total_rows, layer, stream);
  if (st != LSG_OK) return st;
  // 2. slice -> contiguous send buffer, 3. all-gather, 4. every other rank's slice -> y
  char* send = static_cast<char*>(workspace);
  char* recv = send + static_cast<size_t>(total_rows) * w * 2;
  cudaError_t e = cudaMemcpy2DAsync(send, w * 2, yb + c0 * 2, ldy * 2, w * 2, total_rows, cudaMemcpyDeviceToDevice, cs);
  if (e != cudaSuccess) return cuda_fail(e, "lsg_tp_sgmv_nccl: stage copy");
  const int nccl_type = shard->dtype == LSG_F16 ? 6 /* ncclFloat16 */ : 9 /* ncclBfloat16 */;
  const int nr = allgather(send, recv, static_cast<size_t>(total_rows) * w, nccl_type, nccl_comm, cs);
  if (nr != 0) return fail(LSG_ECUDA, "lsg_tp_sgmv_nccl: ncclAllGather failed (" + std::to_string(nr) + ")");
  for (int r = 0; r < tp_size; ++r) {
    if (r == tp_rank) continue;
    e = cudaMemcpy2DAsync(yb + r * w * 2, ldy * 2, recv + static_cast<size_t>(r) * total_rows * w * 2, w * 2, w * 2,
                          total_rows, cudaMemcpyDeviceToDevice, cs);
    if (e != cudaSuccess) return cuda_fail(e, "lsg_tp_sgmv_nccl: gather copy");
  }
  return LSG_OK;
}

size_t lsg_dense_lora_workspace_size(const lsg_weight_table* tbl, int32_t total_rows) {
  CallScope scope(nullptr);
  if (tbl == nullptr || validate_table(tbl) != LSG_OK || total_rows < 0) return 0;
  return static_cast<size_t>(total_rows) * tbl->rank * sizeof(float);
}

int lsg_dense_lora(void* y, int64_t ldy, const void* x, int64_t ldx, const void* w, int64_t ldw,
                   const lsg_weight_table* tbl, const int32_t* seg_starts, const int32_t* seg_slot,
                   int32_t num_segments, int32_t total_rows, int32_t layer, void* workspace,
                   size_t workspace_bytes, lsg_stream_t stream) {
  CallScope scope(nullptr);
  int st = validate_table(tbl);
  if (st != LSG_OK) return st;
  if (total_rows < 0 || num_segments < 0) return fail(LSG_EINVAL, "lsg_dense_lora: negative sizes");
  if (layer < 0 || layer >= tbl->num_layers) return fail(LSG_EINVAL, "lsg: layer index out of range");
  if (total_rows == 0) return LSG_OK;
  if (x == nullptr || y == nullptr || w == nullptr || seg_starts == nullptr || seg_slot == nullptr)
    return fail(LSG_EINVAL, "lsg_dense_lora: NULL pointer");
  if (ldx < tbl->h_in || ldy < tbl->h_out || ldw < tbl->h_out) return fail(LSG_EINVAL, "lsg_dense_lora: bad strides");
  if (tbl->rank != 16 || total_rows > kDlMaxRows || tbl->h_in % (kTcKB * kDlKS) != 0 || tbl->h_out % kDlN != 0 || tbl->h_out % 64 != 0 ||
      !aligned16(x) || !aligned16(y) || !aligned16(w) || ldx % 8 != 0 || ldy % 8 != 0 || ldw % 8 != 0 ||
      tbl->b_layer_stride % 8 != 0 || encode_tiled_fn() == nullptr)
    return fail(LSG_EUNSUPPORTED, "lsg_dense_lora: rank 16, <= 64 rows, h_in % 256, h_out a multiple of the column tile, 16-byte rows");
  if (workspace == nullptr || workspace_bytes < lsg_dense_lora_workspace_size(tbl, total_rows) || !aligned16(workspace))
    return fail(LSG_EINVAL, "lsg_dense_lora: workspace too small");
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  float* v = static_cast<float*>(workspace);
  st = run(kKShrink, nullptr, 0, x, ldx, v, nullptr, tbl, seg_starts, seg_slot, nullptr, num_segments, total_rows,
           layer, stream);
  if (st != LSG_OK) return st;
  DenseLoraParams p{};
  if (!encode_map_2d(&p.tmap_x, tbl->dtype, x, static_cast<uint64_t>(tbl->h_in), static_cast<uint64_t>(total_rows),
                     static_cast<uint64_t>(ldx), kTcKB, kDlMaxRows, CU_TENSOR_MAP_SWIZZLE_128B))
    return fail(LSG_ECUDA, "tensor map x");
  {  // W [h_in][h_out] as 3-D {64 columns, h_in rows, h_out / 64 column blocks}: one box = kDlN / 64
     // stacked [64 k][64 n] MN-major atoms
    const cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(tbl->h_in), static_cast<cuuint64_t>(tbl->h_out / 64)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(ldw) * 2, 128};
    const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(kTcKB), static_cast<cuuint32_t>(kDlN / 64)};
    const cuuint32_t estr[3] = {1, 1, 1};
    if (encode_tiled_fn()(&p.tmap_w,
                          tbl->dtype == LSG_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                          const_cast<void*>(w), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(LSG_ECUDA, "tensor map W");
  }
  p.y = y;
  p.ldy = ldy;
  p.v = v;
  p.b_ptr = tbl->b_ptr;
  p.b_off = static_cast<int64_t>(layer) * tbl->b_layer_stride;
  p.seg_starts = seg_starts;
  p.seg_slot = seg_slot;
  p.n_seg = num_segments;
  p.s_n = total_rows;
  p.num_slots = tbl->num_slots;
  p.h_in = tbl->h_in;
  p.h_out = tbl->h_out;
  return launch_dense_lora(tbl->dtype, p, cs);
}

int lsg_sgmv_shrink(float* v, const void* x, int64_t ldx, const lsg_weight_table* tbl,
                    const int32_t* seg_starts, const int32_t* seg_slot, int32_t num_segments,
                    int32_t total_rows, int32_t layer, lsg_stream_t stream) {
  CallScope scope(nullptr);
  return run(kKShrink, nullptr, 0, x, ldx, v, nullptr, tbl, seg_starts, seg_slot, nullptr,
             num_segments, total_rows, layer, stream);
}

int lsg_sgmv_expand(void* y, int64_t ldy, const float* v, const lsg_weight_table* tbl,
                    const int32_t* seg_starts, const int32_t* seg_slot, int32_t num_segments,
                    int32_t total_rows, int32_t layer, lsg_stream_t stream) {
  CallScope scope(nullptr);
  return run(kKExpand, y, ldy, nullptr, 0, nullptr, v, tbl, seg_starts, seg_slot, nullptr,
             num_segments, total_rows, layer, stream);
}

int lsg_bgmv(void* y, int64_t ldy, const void* x, int64_t ldx, const lsg_weight_table* tbl,
             const int32_t* row_slot, int32_t total_rows, int32_t layer, lsg_stream_t stream) {
  CallScope scope(nullptr);
  // One cluster per row with the row in gridDim.y (<= 65535): longer batches run as
  // consecutive launches over row ranges (rows are independent).
  for (int32_t r0 = 0; r0 < total_rows || r0 == 0; r0 += kMaxGridY) {
    const int32_t n = std::min<int32_t>(kMaxGridY, total_rows - r0);
    const int st = run(kKBgmv, y ? static_cast<char*>(y) + static_cast<int64_t>(r0) * ldy * 2 : nullptr, ldy,
                       x ? static_cast<const char*>(x) + static_cast<int64_t>(r0) * ldx * 2 : nullptr, ldx, nullptr,
                       nullptr, tbl, nullptr, nullptr, row_slot ? row_slot + r0 : nullptr, 0, n, layer, stream);
    if (st != LSG_OK || total_rows <= kMaxGridY) return st;
  }
  return LSG_OK;
}

int lsg_set_option(int32_t option, int32_t value) {
  switch (option) {
    case LSG_OPT_PDL: g_opt_pdl = value ? 1 : 0; return LSG_OK;
    case LSG_OPT_FORCE_CLUSTER:
      if (value < 0 || value > kMaxCluster) return fail(LSG_EINVAL, "lsg: cluster size must be 0..16");
      g_opt_force_cluster = value;
      return LSG_OK;
    case LSG_OPT_FORCE_GENERIC: g_opt_force_generic = value ? 1 : 0; return LSG_OK;
    case LSG_OPT_FORCE_TILE_ROWS:
      if (value != 0 && value != 1 && value != 4 && value != 8)
        return fail(LSG_EINVAL, "lsg: tile rows must be 0, 1, 4 (rank-64 fused) or 8");
      g_opt_force_tile_rows = value;
      return LSG_OK;
    case LSG_OPT_NO_L2_STAGING: g_opt_no_alias = value > 0 ? 1 : value < 0 ? -1 : 0; return LSG_OK;
    case LSG_OPT_NO_TENSOR_CORES: g_opt_no_tc = value ? 1 : 0; return LSG_OK;
    case LSG_OPT_TC_SPLIT: g_opt_tc_split = value ? 1 : 0; return LSG_OK;
    case LSG_OPT_NO_ROW_MODE: g_opt_no_row_mode = value ? 1 : 0; return LSG_OK;
    case LSG_OPT_NO_MULTIROW_TILES: g_opt_no_rank64_tiles = value ? 1 : 0; return LSG_OK;
    case LSG_OPT_TC_MIN_ROWS:
      if (value < 0) return fail(LSG_EINVAL, "lsg: tensor-core row threshold must be >= 0");
      g_opt_tc_min_rows = value;
      return LSG_OK;
    case LSG_OPT_TC_LEGACY:
      if (value < 0 || value > 5) return fail(LSG_EINVAL, "lsg: tensor-core generation must be 0 .. 5");
      g_opt_tc_legacy = value;
      return LSG_OK;
    case LSG_OPT_MMA_MIN_ROWS:
      if (value < 0) return fail(LSG_EINVAL, "lsg: MMA row threshold must be >= 0");
      g_opt_mma_min_rows = value;
      return LSG_OK;
    case LSG_OPT_MMA_FUSED:
      if (value < 0 || value > 2) return fail(LSG_EINVAL, "lsg: MMA fused mode must be 0 .. 2");
      g_opt_mma_fused = value;
      return LSG_OK;
  }
  return fail(LSG_EINVAL, "lsg: unknown option");
}

int lsg_get_option(int32_t option) {
  switch (option) {
    case LSG_OPT_PDL: return cur().pdl;
    case LSG_OPT_FORCE_CLUSTER: return cur().force_cluster;
    case LSG_OPT_FORCE_GENERIC: return cur().force_generic;
    case LSG_OPT_FORCE_TILE_ROWS: return cur().force_tile_rows;
    case LSG_OPT_NO_L2_STAGING: return cur().no_alias;
    case LSG_OPT_NO_TENSOR_CORES: return cur().no_tc;
    case LSG_OPT_TC_SPLIT: return cur().tc_split;
    case LSG_OPT_NO_ROW_MODE: return cur().no_row_mode;
    case LSG_OPT_NO_MULTIROW_TILES: return cur().no_rank64_tiles;
    case LSG_OPT_TC_MIN_ROWS: return g_opt_tc_min_rows.load();
    case LSG_OPT_TC_LEGACY: return g_opt_tc_legacy.load();
    case LSG_OPT_MMA_MIN_ROWS: return g_opt_mma_min_rows.load();
    case LSG_OPT_MMA_FUSED: return g_opt_mma_fused.load();
  }
  return fail(LSG_EINVAL, "lsg: unknown option");
}

int lsg_query_launch(const lsg_weight_table* tbl, int32_t num_segments, int32_t total_rows,
                     int32_t kernel, lsg_launch_info* info) {
  CallScope scope(nullptr);
  int st = validate_table(tbl);
  if (st != LSG_OK) return st;
  if (info == nullptr || kernel < 0 || kernel > 3) return fail(LSG_EINVAL, "lsg_query_launch: bad arguments");
  if (total_rows <= 0 || (kernel != kKBgmv && num_segments <= 0)) {
    *info = lsg_launch_info{};
    return LSG_OK;
  }
  const Plan pl = make_plan(tbl, kernel, num_segments, total_rows, fast_shape_ok(tbl));
  if (kernel == kKFused && pl.path == 0) {  // every segment on the segment-tile MMA pair (K7)?
    const RowRanges rr = row_ranges(tbl, num_segments, total_rows);
    int kp = 0, pc = 0, nc = 0;
    const int tiles = rr.mma_lo > 0 ? mma_tile_bound(total_rows, num_segments, rr.mma_lo) : 0;
    if (rr.mma_lo == 1 && rr.mma_hi == kRowsInf && mma_splits(tbl, tiles, kp, pc, nc)) {
      info->path = 2;
      info->cluster = pc;
      info->tile_rows = kMmaM;
      info->row_splits = kp;
      info->grid_ctas = tiles * (kp + nc);
      info->smem_bytes = static_cast<int>(mma_part_smem(tbl->rank, tbl->h_in / kp / kMmaKC, pc));
      return LSG_OK;
    }
  }
  info->path = pl.path;
  info->cluster = pl.path ? 1 : pl.cluster;
  info->tile_rows = pl.path ? 1 : pl.mt;
  info->row_splits = pl.row_splits;
  info->grid_ctas = pl.path ? total_rows : pl.cluster * pl.clusters;
  info->smem_bytes = pl.smem;
  return LSG_OK;
}

size_t lsg_build_segments_workspace(int32_t total_rows, int32_t num_slots) {
  (void)total_rows;
  (void)num_slots;
  return 0;  // the single-CTA builder keeps everything in shared memory
}

int lsg_build_segments(const int32_t* row_slot, int32_t total_rows, int32_t num_slots,
                       int32_t lead_slot, int32_t lead_row0, int32_t lead_row1, int32_t* row_perm, int32_t* seg_starts,
                       int32_t* seg_slot, int32_t* num_segments, void* workspace,
                       size_t workspace_bytes, lsg_stream_t stream) {
  CallScope scope(nullptr);
  (void)workspace;
  (void)workspace_bytes;
  if (total_rows < 0 || num_slots < 0) return fail(LSG_EINVAL, "lsg_build_segments: negative sizes");
  if (total_rows > kBuilderMaxRows) return fail(LSG_EUNSUPPORTED, "lsg_build_segments: total_rows > 16384");
  if (lead_row0 < 0 || lead_row1 < lead_row0 || lead_row1 > total_rows)
    return fail(LSG_EINVAL, "lsg_build_segments: lead row range outside [0, total_rows]");
  if (seg_starts == nullptr || num_segments == nullptr || (total_rows > 0 && (row_slot == nullptr ||
      row_perm == nullptr || seg_slot == nullptr)))
    return fail(LSG_EINVAL, "lsg_build_segments: NULL output");
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (total_rows == 0) {
    cudaError_t e = cudaMemsetAsync(seg_starts, 0, sizeof(int32_t), cs);
    if (e == cudaSuccess) e = cudaMemsetAsync(num_segments, 0, sizeof(int32_t), cs);
    return e == cudaSuccess ? LSG_OK : cuda_fail(e, "lsg_build_segments memset");
  }
  int n_pow2 = 1;
  while (n_pow2 < total_rows) n_pow2 <<= 1;
  const int smem = n_pow2 * static_cast<int>(sizeof(uint64_t));
  static std::atomic<unsigned long long> configured{0};  // one bit per device
  if (!configured_on_device(configured)) {
    cudaError_t e = cudaFuncSetAttribute(build_segments_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kBuilderMaxRows * 8);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(builder smem)");
    mark_configured(configured);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(kBuilderThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = cs;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = cur().pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, build_segments_kernel, row_slot, total_rows, num_slots, lead_slot,
                                     lead_row0, lead_row1, n_pow2, row_perm, seg_starts, seg_slot, num_segments);
  return e == cudaSuccess ? LSG_OK : cuda_fail(e, "build_segments_kernel launch");
}

static int permute_rows(bool gather, void* dst, int64_t ld_dst, const void* src, int64_t ld_src,
                        const int32_t* perm, int32_t rows, int32_t cols, lsg_stream_t stream) {
  if (rows < 0 || cols < 0) return fail(LSG_EINVAL, "lsg permute rows: negative sizes");
  if (rows == 0 || cols == 0) return LSG_OK;
  if (dst == nullptr || src == nullptr || perm == nullptr || ld_dst < cols || ld_src < cols)
    return fail(LSG_EINVAL, "lsg permute rows: bad pointers or strides");
  const bool vec = aligned16(dst) && aligned16(src) && cols % 8 == 0 && ld_dst % 8 == 0 && ld_src % 8 == 0;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (gather)
    permute_rows_kernel<true><<<rows, 128, 0, cs>>>(static_cast<uint16_t*>(dst), ld_dst,
                                                   static_cast<const uint16_t*>(src), ld_src, perm, cols, vec);
  else
    permute_rows_kernel<false><<<rows, 128, 0, cs>>>(static_cast<uint16_t*>(dst), ld_dst,
                                                    static_cast<const uint16_t*>(src), ld_src, perm, cols, vec);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? LSG_OK : cuda_fail(e, "permute_rows_kernel launch");
}

int lsg_gather_rows(void* dst, int64_t ld_dst, const void* src, int64_t ld_src, const int32_t* row_perm,
                    int32_t rows, int32_t cols, lsg_stream_t stream) {
  return permute_rows(true, dst, ld_dst, src, ld_src, row_perm, rows, cols, stream);
}

int lsg_scatter_rows(void* dst, int64_t ld_dst, const void* src, int64_t ld_src, const int32_t* row_perm,
                     int32_t rows, int32_t cols, lsg_stream_t stream) {
  return permute_rows(false, dst, ld_dst, src, ld_src, row_perm, rows, cols, stream);
}

int lsg_set_trace(unsigned long long* device_buffer, int32_t max_ctas) {
  if (max_ctas < 0 || (max_ctas > 0 && device_buffer == nullptr)) return fail(LSG_EINVAL, "lsg_set_trace: bad buffer");
#ifndef LSG_INSTRUMENT
  if (max_ctas > 0) return fail(LSG_EUNSUPPORTED, "lsg_set_trace: this build has no phase tracing (-DLSG_INSTRUMENT)");
#endif
  g_trace = max_ctas ? device_buffer : nullptr;
  g_trace_ctas = max_ctas;
  return LSG_OK;
}

const char* lsg_status_string(int status) {
  switch (status) {
    case LSG_OK: return "LSG_OK";
    case LSG_EINVAL: return "LSG_EINVAL: invalid argument";
    case LSG_EUNSUPPORTED: return "LSG_EUNSUPPORTED: unsupported configuration";
    case LSG_ECUDA: return "LSG_ECUDA: CUDA runtime error";
    case LSG_ENODEVICE: return "LSG_ENODEVICE: no usable sm_100 device";
  }
  return "LSG: unknown status";
}

const char* lsg_last_error(void) { return g_err.c_str(); }

int lsg_version(void) { return 100; }

}  // extern "C"
