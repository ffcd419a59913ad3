// sgmv_kernels.cuh -- the SGMV kernels for sm_100a.
//
// Fast path (sgmv_fast_kernel): one thread-block CLUSTER of C CTAs per
// (segment, row-tile).  Every CTA of the cluster owns 1/C of the hidden
// dimension on both sides of the LoRA bottleneck:
//   shrink  (reference sgmv.cpp:105-119):  CTA c streams A[d0:d1, :] and x[rows, d0:d1]
//           into shared memory with 1-D TMA bulk copies, computes fp32 partial
//           sums per 128-row chunk of A (warp FMA + xor-shuffle butterfly), and
//           the cluster reduces the chunk partials through distributed shared
//           memory in ascending chunk order;
//   expand  (reference sgmv.cpp:121-136 + the add of sgmv.cpp:153):  CTA c
//           streams B[:, n0:n1] and y[rows, n0:n1], computes v . B in fp32 and
//           writes y += . with 128-bit stores.
// All of a cluster's weight bytes are requested at kernel entry (before the
// programmatic-dependent-launch wait), so the B stream overlaps the shrink and
// its cluster reduction.  No global workspace, no atomics, no grid-wide sync.
//
// Canonical arithmetic (what makes results independent of C, the tile size,
// the segment order, the kernel variant and the GPU a row lands on):
//   v[m,k] = sum_{q=0..h_in/128-1} P_q[m,k]           (sequential in q, fp32)
//   P_q    = butterfly over lanes of per-lane fp32 FMA chains over the chunk's
//            128 rows (fixed lane->row map per rank)
//   y[m,n] = rn( (sum_{k=0..r-1} v[m,k] * B[k,n]) + y_old[m,n] )   (fp32 chain)
// Generic path (sgmv_generic_kernel): any shape / alignment, one CTA per row.
#pragma once

#include <cooperative_groups.h>

#include "sgmv_device.cuh"

// 1: the first tile's y_old rows are L2-prefetched with x ahead of the PDL wait (A/B knob)
#ifndef LSG_FAST_PF_Y
#define LSG_FAST_PF_Y 1
#endif

namespace lsg {

namespace cg = cooperative_groups;

#ifndef LSG_MIN_BLOCKS
#define LSG_MIN_BLOCKS 3  // co-resident CTAs per SM the register budget is sized for (measured best)
#endif
#ifndef LSG_PIECES
#define LSG_PIECES 4
#endif
#ifndef LSG_THREADS
#define LSG_THREADS 256
#endif
constexpr int kThreads = LSG_THREADS;
constexpr int kWarps = kThreads / 32;
constexpr int KW = 128;     // rows of A (h_in elements) per canonical reduction chunk
constexpr int kPieces = LSG_PIECES;  // A arrives in up to kPieces bulk copies, one mbarrier each

enum Mode : int { kFused = 0, kShrink = 1, kExpand = 2 };

// One LoRA site of a grouped launch (lsg_sgmv_multi): its activations and pool.
struct SiteParams {
  void* y;
  const void* x;
  const void* const* a_ptr;
  const void* const* b_ptr;
  int64_t ldx;
  int64_t ldy;
};
constexpr int kMaxSites = 8;

struct FastParams {
  void* y;
  const void* x;
  float* v_out;
  const float* v_in;
  const void* const* a_ptr;
  const void* const* b_ptr;
  int64_t a_off;  // layer * a_layer_stride (elements)
  int64_t b_off;
  int64_t ldx;
  int64_t ldy;
  const int32_t* seg_starts;
  const int32_t* seg_slot;
  const int32_t* row_slot;  // non-null => BGMV indexing (one row per cluster)
  int32_t n_seg;
  int32_t s_n;
  int32_t row_splits;
  int32_t num_slots;
  int32_t h_in;
  int32_t h_out;
  int32_t nq;    // h_in / KW
  int32_t ncvt;  // h_out / 8
  int32_t nqc_max;
  int32_t ncv_max;
  int32_t red_all;  // 1: every CTA receives every chunk partial; 0: owner-sliced two-round reduction
  unsigned long long* trace;  // optional phase trace (lsg_set_trace), 16 u64 per CTA
  int32_t trace_ctas;
  int32_t exp_flags;  // LSG_EXP experiment bits (profiling only; 0 in production)
  int32_t alias_ab;   // 1: single-tile clusters; B is prefetched into L2 and later loaded over A's smem
  int32_t tile_scan;  // 1: cluster blockIdx.y = global tile index, mapped to (segment, tile) on device
  int32_t skip_long;  // >0: segments with at least this many rows belong to the tensor-core kernel
  int32_t n_sites;    // grouped launch: sites[0, n_sites) share the segment plan (kItemRowMulti)
  int32_t late_wait;  // tile-scan launches behind a long-segment kernel that triggers only after its
                      // own PDL wait: skip the wait before the activations (this launch's rows are
                      // disjoint from that kernel's, and its predecessors have completed) and wait
                      // at the end instead, so this grid's completion still implies the predecessor's
  SiteParams sites[kMaxSites];
};

// Phase trace: thread 0 of each CTA stamps clock64 at kernel phases (slot 14:
// globaltimer at entry, slot 15: SM id).  Off unless lsg_set_trace() installed a buffer.
// Phase tracing and the LSG_EXP experiment switches exist only in instrumented
// builds (-DLSG_INSTRUMENT, scripts/build_variant.sh).  Production code is kept
// lean on purpose: every CTA runs each phase's code once per launch, so code size
// is instruction-fetch latency on the critical path (measured: dropping the
// instrumentation alone took the headline launch from 4.49 to 4.11 us).
#ifdef LSG_INSTRUMENT
#define LSG_TRACE_ON (p.trace != nullptr)
#define LSG_EXP_FLAGS p.exp_flags
#else
#define LSG_TRACE_ON false
#define LSG_EXP_FLAGS 0
#endif
#define LSG_TRACE(i)                                                                                   \
  do {                                                                                                 \
    if (LSG_TRACE_ON && threadIdx.x == 0) {                                                      \
      const int cta_ = blockIdx.y * gridDim.x + blockIdx.x;                                            \
      if (cta_ < p.trace_ctas) p.trace[cta_ * 16 + (i)] = clock64();                                   \
    }                                                                                                  \
  } while (0)

struct SmemLayout {
  uint32_t bars, a, x, b, y, recv, v, total;
};

__host__ __device__ inline uint32_t align128(uint32_t v) { return (v + 127u) & ~127u; }

// Owner-sliced reduction: the rows*R outputs are split over the C CTAs in
// quads of 4 floats; slice_max floats per CTA.
__host__ __device__ inline int slice_floats(int MT, int R, int C) { return ((MT * R / 4 + C - 1) / C) * 4; }

// Identical on host (launch sizing) and device (carve-up).
__host__ __device__ inline SmemLayout make_layout(int mode, int R, int MT, int C, int nq, int nqc_max, int ncv_max,
                                                  int red_all, int alias_ab = 0) {
  SmemLayout L;
  uint32_t o = 0;
  const bool sh = mode != kExpand, ex = mode != kShrink;
  const uint32_t a_bytes = sh ? nqc_max * KW * R * 2 : 0, b_bytes = ex ? R * ncv_max * 16 : 0;
  // multi-row tiles convert B to fp32 once for all rows of the tile, over A / x (consumed)
  const uint32_t bf_bytes = ex && MT > 1 ? R * ncv_max * 32 : 0;
  L.bars = o;
  o += 128;
  L.a = o;
  if (alias_ab && MT == 1) {  // B is loaded over A once the shrink has consumed it
    L.b = o;
    o = align128(o + (a_bytes > b_bytes ? a_bytes : b_bytes));
    L.x = o;
    o = align128(o + MT * nqc_max * KW * 2);
  } else {
    o = align128(o + a_bytes);
    L.x = o;
    if (sh) o = align128(o + MT * nqc_max * KW * 2);
    if (o < L.a + bf_bytes) o = align128(L.a + bf_bytes);
    L.b = o;
    o = align128(o + b_bytes);
  }
  L.y = o;
  if (ex) o = align128(o + MT * ncv_max * 16);
  L.recv = o;  // chunk partials received from the cluster
  if (sh) o = align128(o + (red_all ? nq * MT * R : nq * slice_floats(MT, R, C)) * 4);
  L.v = o;
  o = align128(o + MT * (MT > 1 ? R + 4 : R) * 4);  // multi-row tiles: padded rows (bank spread)
  L.total = o;
  return L;
}

// Balanced split of n items over c owners: owner i holds [i*n/c, (i+1)*n/c).
__device__ __forceinline__ int split_lo(int i, int n, int c) { return (i * n) / c; }
__device__ __forceinline__ int split_owner(int q, int n, int c) { return ((q + 1) * c - 1) / n; }

// s = ((0 + v[0]) + v[stride]) + ... + v[(n-1)*stride], in that order (the
// canonical ascending-chunk sum).  Loads are batched 16 at a time so the chain
// costs one shared-memory latency per batch instead of one per term.
__device__ __forceinline__ float ordered_sum(const float* v, int stride, int n) {
  __builtin_assume(n > 0);
  float s = 0.f;
  for (int q0 = 0; q0 < n; q0 += 16) {
    float t[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) t[j] = q0 + j < n ? v[(q0 + j) * stride] : 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (q0 + j < n) s += t[j];
  }
  return s;
}

// How a cluster finds its work item (compile-time, so each instantiation carries
// only its own decode path -- see the code-size note at LSG_INSTRUMENT).
// kItemRowTp: row mode whose expand stores every output vector into each of the
// n_sites destinations sites[d].y (the TP group's y buffers, peer memory over NVLink)
// -- the all-gather of the tensor-parallel expand fused into the epilogue.
enum ItemMode : int { kItemRowSplit = 0, kItemTileScan = 1, kItemBgmv = 2, kItemRow = 3, kItemRowMulti = 4,
                      kItemRowTp = 5 };

template <typename T, int R, int MT, int MODE, int ITEM>
__global__ void __launch_bounds__(kThreads, MT == 1 ? LSG_MIN_BLOCKS : 1)
    sgmv_fast_kernel(const __grid_constant__ FastParams p) {
  static_assert(R == 8 || R == 16 || R == 32 || R == 64, "fast path ranks");
  constexpr int VPR = R / 8;       // 16-byte vectors per A row
  constexpr int RPI = 32 / VPR;    // A rows covered by one warp instruction
  constexpr int ITER = KW / RPI;   // per-lane FMA chain length per chunk
  constexpr bool kSh = MODE != kExpand;
  constexpr bool kEx = MODE != kShrink;
  constexpr int kBarB = kPieces, kBarRed = kPieces + 1, kBarV = kPieces + 2, kBarX = kPieces + 3,
                kBarY = kPieces + 4;
  // One-row fused tiles move x / y_old with one bulk copy each (mbarrier-completed)
  // instead of per-thread cp.async + a block barrier.
  constexpr bool kActBulk = MT == 1 && MODE == kFused;
  constexpr int VP = MT > 1 ? R + 4 : R;  // V_sm row pitch (floats)

  extern __shared__ __align__(128) uint8_t smem[];
  // A CTA that leaves without work: with PDL a grid's completion must imply its
  // predecessor's (the next kernel on the stream waits only for this one), so the
  // first cluster always waits before leaving; the others leave at once.
  auto exit_after_wait = [] {
    if (blockIdx.y == 0) pdl_wait();
  };
  const int C = static_cast<int>(gridDim.x);
  const int crank = static_cast<int>(blockIdx.x);  // cluster dims (C,1,1), grid.x == C
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // one-row tiles always use the one-round reduction (compile-time: the owner-sliced
  // path is not even emitted into those instantiations)
  // (multi-row tiles always use the owner-sliced two-round reduction: compile-time too)
  constexpr int red_all = MODE == kFused && MT == 1 ? 1 : 0;
  const int alias_ab = MODE == kFused && MT == 1 ? p.alias_ab : 0;  // multi-row tiles never alias
  const SmemLayout L = make_layout(MODE, R, MT, C, p.nq, p.nqc_max, p.ncv_max, red_all, alias_ab);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  T* A_sm = reinterpret_cast<T*>(smem + L.a);
  T* x_sm = reinterpret_cast<T*>(smem + L.x);
  uint4* B_sm = reinterpret_cast<uint4*>(smem + L.b);
  uint4* y_sm = reinterpret_cast<uint4*>(smem + L.y);
  float* recv = reinterpret_cast<float*>(smem + L.recv);
  float* V_sm = reinterpret_cast<float*>(smem + L.v);

  if (LSG_TRACE_ON && tid == 0 && blockIdx.y * gridDim.x + blockIdx.x < p.trace_ctas) {
    unsigned long long gt;
    uint32_t smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.trace[(blockIdx.y * gridDim.x + blockIdx.x) * 16 + 14] = gt;
    p.trace[(blockIdx.y * gridDim.x + blockIdx.x) * 16 + 15] = smid;
  }
  LSG_TRACE(0);
  // Let the next launch on the stream start as soon as SM resources allow: its
  // prologue and weight stream then overlap this kernel (it still waits for us
  // before touching activations).
  pdl_launch_dependents();
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i <= kBarB; ++i) mbar_init(&bars[i], 1);
    mbar_init(&bars[kBarRed], 1);  // completed by the bytes the cluster pushes (st.async complete_tx)
    mbar_init(&bars[kBarV], 1);
    if constexpr (kActBulk) {
      mbar_init(&bars[kBarX], 1);
      mbar_init(&bars[kBarY], 1);
    }
    fence_mbar_init();
  }

  // ---- work items (uniform across the cluster) ---------------------------------
  // bgmv / row-split launches: one item per cluster.  Tile-scan launches: the
  // cluster takes global tiles blockIdx.y, blockIdx.y + gridDim.y, ... (the grid
  // is capped near the co-resident cluster count, so tiles past the last real
  // one cost one scan, not one cluster launch).
  uint32_t phase = 0;   // reduction barriers: flips every tile
  uint32_t wphase = 0;  // weight barriers: flips every item
  bool first = true;    // first tile this CTA computes (cluster barrier-init wait)
  bool first_item = true;
  // The site this cluster works for (grouped launches pick theirs below).
  const void* s_x = p.x;
  void* s_y = p.y;
  const void* const* s_a = p.a_ptr;
  const void* const* s_b = p.b_ptr;
  int64_t s_ldx = p.ldx, s_ldy = p.ldy;
  for (int item = blockIdx.y;; item += gridDim.y, wphase ^= 1u) {
    int slot, seg_begin, seg_end, first_tile, tile_step;
    if constexpr (ITEM == kItemBgmv || ITEM == kItemRow || ITEM == kItemRowMulti || ITEM == kItemRowTp) {
      int row = item;
      if constexpr (ITEM == kItemRowMulti) {  // cluster y = site * s_n + row
        const int g = item / p.s_n;
        if (g >= p.n_sites) return exit_after_wait();
        row = item - g * p.s_n;
        s_x = p.sites[g].x;
        s_y = p.sites[g].y;
        s_a = p.sites[g].a_ptr;
        s_b = p.sites[g].b_ptr;
        s_ldx = p.sites[g].ldx;
        s_ldy = p.sites[g].ldy;
      }
      if (row >= p.s_n) return exit_after_wait();
      if constexpr (ITEM == kItemBgmv) {
        slot = p.row_slot[row];
      } else {
        // One cluster per row (one-row tiles, any popularity): the row's segment is
        // the last s < n_seg with seg_starts[s] <= row.  Every warp finds it itself
        // (ballots over 128 boundaries per step; starts are non-decreasing, so the
        // first step with a start > row ends the search).
        int seg = -1;
        for (int c0 = 0; c0 < p.n_seg; c0 += 128) {
          unsigned le[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int sg = c0 + j * 32 + lane;
            le[j] = __ballot_sync(0xffffffffu, sg < p.n_seg && p.seg_starts[sg] <= row);
          }
          bool done = false;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (le[j]) seg = c0 + j * 32 + 31 - __clz(le[j]);
            done = done || le[j] != 0xffffffffu;
          }
          if (done) break;
        }
        slot = seg >= 0 ? p.seg_slot[seg] : -1;
      }
      seg_begin = row;
      seg_end = row + 1;
      first_tile = 0;
      tile_step = 1;
    } else if constexpr (ITEM == kItemTileScan) {
      // Tile t: walk the segments' tile counts ceil(len/MT) with a warp prefix
      // sum (32 segments per step) until t falls inside one.
      __shared__ int s_seg, s_tile;
      __syncthreads();  // previous item's s_seg / s_tile consumed
      if (warp == 0) {
        const int t = item;
        int base = 0, seg = -1, tin = 0;
        for (int c0 = 0; c0 < p.n_seg && seg < 0; c0 += 32) {
          const int sg = c0 + lane;
          int nt = 0;
          if (sg < p.n_seg) {
            const int len = p.seg_starts[sg + 1] - p.seg_starts[sg];
            nt = (p.skip_long > 0 && len >= p.skip_long) ? 0 : (len + MT - 1) / MT;
          }
          int incl = nt;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += v;
          }
          const unsigned hit = __ballot_sync(0xffffffffu, nt > 0 && t < base + incl);
          if (hit) {
            const int l = __ffs(hit) - 1;
            seg = c0 + l;
            tin = t - (base + __shfl_sync(0xffffffffu, incl - nt, l));
          }
          base += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) {
          s_seg = seg;
          s_tile = tin;
        }
      }
      __syncthreads();
      if (s_seg < 0) return exit_after_wait();  // past the last tile
      // A later item reuses every buffer: the whole cluster finishes the previous one first.
      if (!first_item) {
        if constexpr (kSh) cluster_sync();
      }
      const int s = s_seg;
      first_tile = s_tile;
      tile_step = 1 << 30;  // exactly one tile per item
      seg_begin = p.seg_starts[s];
      seg_end = p.seg_starts[s + 1];
      slot = p.seg_slot[s];
    } else {
      // one-row tiles only take this path when s_n <= n_seg, where the planner
      // always sets row_splits = 1 (compile-time: no division on the entry path)
      const int s = MT == 1 ? item : item / p.row_splits;
      if (s >= p.n_seg) return exit_after_wait();
      first_tile = MT == 1 ? 0 : item - s * p.row_splits;
      tile_step = MT == 1 ? 1 : p.row_splits;
      seg_begin = p.seg_starts[s];
      seg_end = p.seg_starts[s + 1];
      slot = p.seg_slot[s];
      if (p.skip_long > 0 && seg_end - seg_begin >= p.skip_long) return exit_after_wait();  // tensor-core kernels'
    }
    constexpr bool last_item = ITEM != kItemTileScan;  // bgmv / row-split: one item per cluster
    const int ntiles = (seg_end - seg_begin + MT - 1) / MT;
    if (first_tile >= ntiles) {
      if (last_item) return exit_after_wait();
      wphase ^= 1u;  // no weights were requested for this item: keep the barrier phase
      continue;
    }
    if (slot < 0 || slot >= p.num_slots) {  // "no adapter": v = 0, y untouched
      if (MODE == kShrink && crank == 0) {
        pdl_wait();
        for (int t = first_tile; t < ntiles; t += tile_step) {
          const int r0 = seg_begin + t * MT, rows = min(MT, seg_end - r0);
          for (int i = tid; i < rows * R; i += kThreads) p.v_out[static_cast<int64_t>(r0) * R + i] = 0.f;
        }
      }
      if (last_item) return exit_after_wait();
      wphase ^= 1u;  // no weights were requested for this item: keep the barrier phase
      continue;
    }

    LSG_TRACE(1);
    const int q0 = split_lo(crank, p.nq, C), nqc = split_lo(crank + 1, p.nq, C) - q0;
    const int cv0 = split_lo(crank, p.ncvt, C), ncv = split_lo(crank + 1, p.ncvt, C) - cv0;
    const int ndl = nqc * KW;  // this CTA's slice of h_in (x_sm row stride)
    const int npieces = (LSG_EXP_FLAGS & 2) ? min(1, nqc) : min(kPieces, nqc);
    const int slice_max = slice_floats(MT, R, C);

    if (first) {
      __syncthreads();                              // barrier inits visible to this CTA
      if constexpr (kSh) cluster_arrive_relaxed();  // ... and (fence.mbarrier_init) to the cluster
    } else {
      fence_proxy_async_smem();  // previous item's generic smem reads before the weight TMA
    }

    // Adapter weights: every byte this CTA needs, requested before the PDL wait
    // on the first item (so they stream while the previous kernel drains).  A
    // arrives in kPieces chunk-aligned pieces with their own barriers so the
    // shrink starts on the first piece; B follows on one barrier.  Warp 0 issues
    // A, warp 1 issues B (one row per lane).
    const int a_warp = (LSG_EXP_FLAGS & 4) ? 1 : 0, b_warp = (LSG_EXP_FLAGS & 4) ? 0 : (kSh ? 1 : 0);
    if (kSh && warp == a_warp && nqc > 0) {
      const T* A = static_cast<const T*>(s_a[slot]) + p.a_off + static_cast<int64_t>(q0) * KW * R;
      if (lane < npieces) {
        const int c0 = (lane * nqc) / npieces, c1 = ((lane + 1) * nqc) / npieces;
        const uint32_t bytes = static_cast<uint32_t>((c1 - c0) * KW * R * sizeof(T));
        mbar_arrive_expect_tx(&bars[lane], bytes);
        if (LSG_EXP_FLAGS & 1)
          bulk_g2s(A_sm + c0 * KW * R, A + c0 * KW * R, bytes, &bars[lane]);
        else
          bulk_g2s_hint(A_sm + c0 * KW * R, A + c0 * KW * R, bytes, &bars[lane], l2_evict_first_policy());
      }
    }
    const T* Bslice = nullptr;
    if (kEx && warp == b_warp && ncv > 0) {
      const T* B = static_cast<const T*>(s_b[slot]) + p.b_off + cv0 * 8;
      Bslice = B;
    }
    if (kEx && warp == b_warp && ncv > 0 && alias_ab) {
      // B's smem is still holding A: only warm L2 now, load after the shrink
      for (int k = lane; k < R; k += 32)
        bulk_prefetch_l2(Bslice + static_cast<int64_t>(k) * p.h_out, static_cast<uint32_t>(ncv * 16));
    } else if (kEx && warp == b_warp && ncv > 0) {
      const T* B = Bslice;
      if (kSh && (LSG_EXP_FLAGS & 64))  // experiment: queue B behind A (A is needed first)
        for (int i = 0; i < npieces; ++i) mbar_wait(&bars[i], wphase);
      if (lane == 0) mbar_arrive_expect_tx(&bars[kBarB], static_cast<uint32_t>(R * ncv * 16));
      __syncwarp();
      const uint64_t pol = l2_evict_first_policy();
      for (int k = lane; k < R; k += 32) {
        if (LSG_EXP_FLAGS & 1)
          bulk_g2s(B_sm + k * ncv, B + static_cast<int64_t>(k) * p.h_out, static_cast<uint32_t>(ncv * 16),
                   &bars[kBarB]);
        else
          bulk_g2s_hint(B_sm + k * ncv, B + static_cast<int64_t>(k) * p.h_out, static_cast<uint32_t>(ncv * 16),
                        &bars[kBarB], pol);
      }
    }
    // Activations of the first tile: warm L2 now, ahead of the PDL wait.  After the
    // wait they then come from L2 instead of queueing in HBM behind the weight
    // streams of the launches that follow.  A prefetch is only a cache hint (L2 is
    // the coherence point), so this is safe even when the preceding kernel is still
    // writing x or y.
    if (first_item && warp == 2 && !(LSG_EXP_FLAGS & 32)) {
      const int r0 = seg_begin + first_tile * MT, rows = min(MT, seg_end - r0);
      if (kSh && lane < rows && nqc > 0)
        bulk_prefetch_l2(static_cast<const T*>(s_x) + static_cast<int64_t>(r0 + lane) * s_ldx + q0 * KW,
                         static_cast<uint32_t>(ndl * sizeof(T)));
      if (LSG_FAST_PF_Y && kEx && lane >= 16 && lane - 16 < rows && ncv > 0)
        bulk_prefetch_l2(static_cast<const T*>(s_y) + static_cast<int64_t>(r0 + lane - 16) * s_ldy + cv0 * 8,
                         static_cast<uint32_t>(ncv * 16));
    }
    LSG_TRACE(2);
    if (LSG_EXP_FLAGS & 8) {  // experiment: weight stream only
      for (int i = 0; i < npieces; ++i) mbar_wait(&bars[i], 0);
      if (kEx && ncv > 0) mbar_wait(&bars[kBarB], 0);
      if constexpr (kSh) cluster_wait();
      return;
    }
    if (LSG_EXP_FLAGS & 16) {  // experiment: weights + activations, no compute
      pdl_wait();
      for (int i = 0; i < npieces; ++i) mbar_wait(&bars[i], 0);
      if (kEx && ncv > 0) mbar_wait(&bars[kBarB], 0);
      if constexpr (kSh) cluster_wait();
      return;
    }
    // Cluster-window addresses this lane pushes its chunk partials to (one-round
    // reduction, C <= RPI: lane group g sends half h to CTA (g + h) % RPI).
    int push_dst[2] = {C, C};
    uint32_t push_recv[2] = {0, 0}, push_bar[2] = {0, 0};
    if (kSh && red_all && (RPI >= 16 || C <= RPI)) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        push_dst[h] = (lane / VPR + h) % RPI;
        if (push_dst[h] < C) {
          push_recv[h] = mapa_u32(recv, static_cast<uint32_t>(push_dst[h]));
          push_bar[h] = mapa_u32(&bars[kBarRed], static_cast<uint32_t>(push_dst[h]));
        }
      }
    }
    // x, v and y may be produced by the preceding kernel: wait for it here
    // (returns at once after the first item).
    if constexpr (ITEM == kItemTileScan) {
      if (!p.late_wait) pdl_wait();
    } else {
      pdl_wait();
    }
    LSG_TRACE(3);

    for (int t = first_tile; t < ntiles; t += tile_step, phase ^= 1u) {
      const int r0 = seg_begin + t * MT;
      const int rows = min(MT, seg_end - r0);
      const int no = rows * R;
      const int o0 = split_lo(crank, no / 4, C) * 4, o1 = split_lo(crank + 1, no / 4, C) * 4;
      // Activations go through cp.async (LDGSTS), not the TMA queue the weights
      // occupy, so they land about one memory latency after the wait.
      if constexpr (kActBulk) {
        if (tid == 0 && nqc > 0) {
          mbar_arrive_expect_tx(&bars[kBarX], static_cast<uint32_t>(ndl * sizeof(T)));
          bulk_g2s(x_sm, static_cast<const T*>(s_x) + static_cast<int64_t>(r0) * s_ldx + q0 * KW,
                   static_cast<uint32_t>(ndl * sizeof(T)), &bars[kBarX]);
        }
        if (tid == 32 && ncv > 0) {
          mbar_arrive_expect_tx(&bars[kBarY], static_cast<uint32_t>(ncv * 16));
          bulk_g2s(y_sm, static_cast<const T*>(s_y) + static_cast<int64_t>(r0) * s_ldy + cv0 * 8,
                   static_cast<uint32_t>(ncv * 16), &bars[kBarY]);
        }
      } else if constexpr (kSh) {
        const int nv = ndl / 8;  // 16-byte vectors per x row slice
        for (int i = tid; i < rows * nv; i += kThreads) {
          const int m = MT == 1 ? 0 : i / nv, c = i - m * nv;
          cp_async16(x_sm + m * ndl + c * 8,
                     static_cast<const T*>(s_x) + static_cast<int64_t>(r0 + m) * s_ldx + q0 * KW + c * 8);
        }
      }
      cp_async_commit();
      if constexpr (kEx && !kActBulk) {
        for (int i = tid; i < rows * ncv; i += kThreads) {
          const int m = MT == 1 ? 0 : i / ncv, c = i - m * ncv;
          cp_async16(y_sm + m * ncv + c,
                     static_cast<const T*>(s_y) + static_cast<int64_t>(r0 + m) * s_ldy + (cv0 + c) * 8);
        }
      }
      cp_async_commit();
      if (kSh && tid == 0) {
        // bytes this CTA will receive this tile; peers may already be pushing (the
        // tx-count may go transiently negative; the phase needs this arrive too)
        mbar_arrive_expect_tx(&bars[kBarRed], static_cast<uint32_t>(p.nq * (red_all ? no : (o1 - o0)) * 4));
        if (MODE == kFused && !red_all) mbar_arrive_expect_tx(&bars[kBarV], static_cast<uint32_t>(no * 4));
      }

      if constexpr (MODE == kExpand) {
        for (int i = tid; i < no; i += kThreads) V_sm[(i / R) * VP + i % R] = p.v_in[static_cast<int64_t>(r0) * R + i];
      } else {
        if constexpr (kActBulk) {
          if (nqc > 0) mbar_wait(&bars[kBarX], phase);
        } else {
          cp_async_wait<1>();  // this thread's x vectors
          __syncthreads();     // everyone's
        }
        LSG_TRACE(4);
        if (first) cluster_wait();  // every peer's barriers are initialised
        first = false;
        LSG_TRACE(5);
        if (LSG_TRACE_ON && tid == 0) {  // trace only: when did all of A land?
          for (int i = 0; i < npieces; ++i) mbar_wait(&bars[i], wphase);
          LSG_TRACE(12);
        }
        // ---- shrink: per-chunk partials P_q[m, k], pushed to the reducers ----------
        const int rowoff = lane / VPR, vec = lane % VPR;
        const uint4* Av = reinterpret_cast<const uint4*>(A_sm);
        // Work unit = (chunk, row): every warp takes units until none are left.  A
        // unit's arithmetic depends only on its chunk and row, never on which warp,
        // CTA or tile size computes it.  (Multi-row tiles use the same units: with the
        // mixed-precision FMA a unit costs one shared-memory load of A per 8 FMAs and
        // no conversions, and a tile's rows * chunks units keep every warp busy.)
        const int nunits = nqc * rows;
        for (int u = warp; u < nunits; u += kWarps) {
          const int ql = MT == 1 ? u : u / rows, m = MT == 1 ? 0 : u - ql * rows;
          // wait for the piece holding chunk ql (no-op once it has landed)
          mbar_wait(&bars[split_owner(ql, nqc, npieces)], wphase);
          float acc[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] = 0.f;
          const uint4* Ac = Av + (ql * KW + rowoff) * VPR + vec;
          const uint16_t* xc = reinterpret_cast<const uint16_t*>(x_sm + m * ndl + ql * KW + rowoff);
#pragma unroll
          for (int it = 0; it < ITER; ++it) fma8_mixed<T>(xc[it * RPI], Ac[it * RPI * VPR], acc);
          if (u == warp) LSG_TRACE(9);  // warp 0: FMA chain of its first unit done
#pragma unroll
          for (int off = VPR; off < 32; off <<= 1)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], off);
          // Every lane now holds its vec's 8 partial sums P_q[m, vec*8 .. +8).  Push
          // them into the reducers' shared memory with st.async (async proxy: the
          // receiver's mbarrier completes on the bytes -- no cluster fence); the
          // 32/VPR lanes sharing a vec split the 16-byte quads / destinations.
          const int q = q0 + ql;
          const int g = lane / VPR;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int o = m * R + vec * 8 + h * 4;
            if (red_all && (RPI >= 16 || C <= RPI)) {  // <= one destination per (lane, h); C <= 16
              if (push_dst[h] < C)
                st_async_v4(push_recv[h] + static_cast<uint32_t>((q * MT * R + o) * 4), acc[h * 4 + 0], acc[h * 4 + 1],
                            acc[h * 4 + 2], acc[h * 4 + 3], push_bar[h]);
            } else if (red_all) {
              const uint32_t local = smem_u32(recv + q * MT * R + o), lbar = smem_u32(&bars[kBarRed]);
              for (int dst = (g + h) % RPI; dst < C; dst += RPI) {
                uint32_t ra, rb;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local), "r"(dst));
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lbar), "r"(dst));
                st_async_v4(ra, acc[h * 4 + 0], acc[h * 4 + 1], acc[h * 4 + 2], acc[h * 4 + 3], rb);
              }
            } else if (g == h) {
              const int owner = split_owner(o / 4, no / 4, C);
              const int jl = o - split_lo(owner, no / 4, C) * 4;
              st_async_v4(mapa_u32(recv + q * slice_max + jl, static_cast<uint32_t>(owner)), acc[h * 4 + 0],
                          acc[h * 4 + 1], acc[h * 4 + 2], acc[h * 4 + 3],
                          mapa_u32(&bars[kBarRed], static_cast<uint32_t>(owner)));
            }
          }
          if (u == warp) LSG_TRACE(13);  // warp 0: first unit pushed
        }
        if (alias_ab) fence_proxy_async_smem();  // A reads done before TMA overwrites them
        __syncthreads();
        if (kEx && alias_ab && warp == b_warp && ncv > 0) {
          // A is consumed: bring the (L2-warm) B slice into the same shared memory
          if (lane == 0) mbar_arrive_expect_tx(&bars[kBarB], static_cast<uint32_t>(R * ncv * 16));
          __syncwarp();
          for (int k = lane; k < R; k += 32)
            bulk_g2s(B_sm + k * ncv, Bslice + static_cast<int64_t>(k) * p.h_out, static_cast<uint32_t>(ncv * 16),
                     &bars[kBarB]);
        }
        // ---- reduction over chunks, ascending q ----------------------------------
        LSG_TRACE(6);
        mbar_wait(&bars[kBarRed], phase);
        LSG_TRACE(7);
        if (red_all) {
          if constexpr (MT * R <= kThreads) {  // one output per thread at most
            if (tid < no) V_sm[tid] = ordered_sum(recv + tid, MT * R, p.nq);
          } else {
            for (int o = tid; o < no; o += kThreads) V_sm[o] = ordered_sum(recv + o, MT * R, p.nq);
          }
        } else {
          if constexpr (MODE == kShrink) {
            for (int o = o0 + tid; o < o1; o += kThreads) {
              const float s = ordered_sum(recv + (o - o0), slice_max, p.nq);
              const int m = o / R;
              p.v_out[static_cast<int64_t>(r0 + m) * R + (o - m * R)] = s;
            }
          } else {
            // my slice of v, 4 outputs per thread, broadcast to every CTA as 16-byte pushes
            for (int o = o0 + 4 * tid; o < o1; o += 4 * kThreads) {
              float s4[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) s4[e] = ordered_sum(recv + (o - o0) + e, slice_max, p.nq);
              float* vd = V_sm + (o / R) * VP + o % R;  // 4 outputs of one row
              for (int dst = 0; dst < C; ++dst)
                st_async_v4(mapa_u32(vd, static_cast<uint32_t>(dst)), s4[0], s4[1], s4[2], s4[3],
                            mapa_u32(&bars[kBarV], static_cast<uint32_t>(dst)));
            }
          }
          if constexpr (MODE == kFused) mbar_wait(&bars[kBarV], phase);
        }
      }

      if constexpr (kEx) {
        LSG_TRACE(8);
        if constexpr (!kActBulk) cp_async_wait<0>();  // this thread's y vectors
        __syncthreads();     // V_sm and every y vector visible
        // ---- expand: y[m, n] += sum_k v[m, k] B[k, n] ---------------------------
        if (ncv > 0) {
          if constexpr (kActBulk) mbar_wait(&bars[kBarY], phase);
          mbar_wait(&bars[kBarB], wphase);
          LSG_TRACE(10);
          if constexpr (MT > 1) {
            // Multi-row tiles: B -> fp32 once (over the consumed A / x), then lane = (row m,
            // column vector): the MT lanes of a vector read the same B values (broadcast) and
            // each runs its row's chain over k -- the same per-element chain as one-row tiles.
            float* Bf = reinterpret_cast<float*>(smem + L.a);
            for (int i = tid; i < R * ncv; i += kThreads) {
              float b[8];
              Cvt<T>::unpack8(B_sm[i], b);
              reinterpret_cast<float4*>(Bf)[2 * i] = make_float4(b[0], b[1], b[2], b[3]);
              reinterpret_cast<float4*>(Bf)[2 * i + 1] = make_float4(b[4], b[5], b[6], b[7]);
            }
            __syncthreads();
            constexpr int CPW = 32 / MT;  // column vectors per warp pass
            const int m = lane % MT, cvl = lane / MT;
            for (int cvb = warp * CPW; cvb < ncv; cvb += kWarps * CPW) {
              const int cv = cvb + cvl;
              if (cv < ncv && m < rows) {
                float acc[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] = 0.f;
                const float* vr = V_sm + m * VP;
                const float4* bc = reinterpret_cast<const float4*>(Bf) + 2 * cv;
#pragma unroll 8
                for (int k = 0; k < R; ++k) {
                  const float4 b0 = bc[2 * k * ncv], b1 = bc[2 * k * ncv + 1];
                  const float vk = vr[k];
                  acc[0] = fmaf(vk, b0.x, acc[0]);
                  acc[1] = fmaf(vk, b0.y, acc[1]);
                  acc[2] = fmaf(vk, b0.z, acc[2]);
                  acc[3] = fmaf(vk, b0.w, acc[3]);
                  acc[4] = fmaf(vk, b1.x, acc[4]);
                  acc[5] = fmaf(vk, b1.y, acc[5]);
                  acc[6] = fmaf(vk, b1.z, acc[6]);
                  acc[7] = fmaf(vk, b1.w, acc[7]);
                }
                float yo[8];
                Cvt<T>::unpack8(y_sm[m * ncv + cv], yo);
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] = acc[j] + yo[j];
                st_global_v4(static_cast<T*>(s_y) + static_cast<int64_t>(r0 + m) * s_ldy + (cv0 + cv) * 8,
                             Cvt<T>::pack8(acc));
              }
            }
          } else
          for (int i = tid; i < rows * ncv; i += kThreads) {
            const int m = i / ncv, cv = i - m * ncv;
            float acc[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = 0.f;
#pragma unroll
            for (int k = 0; k < R; ++k) {
              float b[8];
              Cvt<T>::unpack8(B_sm[k * ncv + cv], b);
              const float vk = V_sm[m * R + k];
#pragma unroll
              for (int j = 0; j < 8; ++j) acc[j] = fmaf(vk, b[j], acc[j]);
            }
            float yo[8];
            Cvt<T>::unpack8(y_sm[m * ncv + cv], yo);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = acc[j] + yo[j];
            if constexpr (ITEM == kItemRowTp) {  // every rank's y (own one included)
              const uint4 out = Cvt<T>::pack8(acc);
              for (int d = 0; d < p.n_sites; ++d)
                st_global_v4(static_cast<T*>(p.sites[d].y) + static_cast<int64_t>(r0 + m) * s_ldy + (cv0 + cv) * 8,
                             out);
            } else {
              st_global_v4(static_cast<T*>(s_y) + static_cast<int64_t>(r0 + m) * s_ldy + (cv0 + cv) * 8,
                           Cvt<T>::pack8(acc));
            }
          }
        }
      }
      LSG_TRACE(11);
      // The next tile reuses x_sm / y_sm / V_sm and the receive buffers: every CTA
      // of the cluster must be done with this tile before anyone pushes again.
      // (After the last tile nothing more is sent to anyone, and every incoming
      // byte was awaited, so CTAs exit without a cluster barrier.)
      if (t + tile_step < ntiles) {
        if constexpr (kSh) cluster_sync();
        else __syncthreads();
      }
    }
    if (last_item || static_cast<int64_t>(item) + gridDim.y >= p.s_n) {
      if constexpr (ITEM == kItemTileScan) {
        if (p.late_wait) pdl_wait();
      }
      return;
    }
    first_item = false;
  }
}

// ---------------------------------------------------------------------------------
// Generic path: any h_in / h_out / rank, any alignment.  One CTA per row.
// v[k] = butterfly over lanes of (per-lane chain over d = lane, lane+32, ...).
// ---------------------------------------------------------------------------------
struct GenericParams {
  void* y;
  const void* x;
  float* v_out;
  const float* v_in;
  const void* const* a_ptr;
  const void* const* b_ptr;
  int64_t a_off, b_off, ldx, ldy;
  const int32_t* seg_starts;
  const int32_t* seg_slot;
  const int32_t* row_slot;
  int32_t n_seg, s_n, num_slots, h_in, h_out, rank;
};

template <typename T, int MODE>
__global__ void __launch_bounds__(kThreads) sgmv_generic_kernel(const __grid_constant__ GenericParams p) {
  extern __shared__ float v_sm[];
  const int row = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int slot;
  if (p.row_slot != nullptr) {
    slot = p.row_slot[row];
  } else {  // segment containing row: last s with seg_starts[s] <= row and a non-empty range
    int lo = 0, hi = p.n_seg;  // find first s with seg_starts[s+1] > row
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (p.seg_starts[mid + 1] > row) hi = mid; else lo = mid + 1;
    }
    slot = lo < p.n_seg ? p.seg_slot[lo] : -1;
  }
  pdl_wait();
  pdl_launch_dependents();
  const int R = p.rank;
  if (slot < 0 || slot >= p.num_slots) {
    if (MODE == kShrink)
      for (int k = tid; k < R; k += kThreads) p.v_out[static_cast<int64_t>(row) * R + k] = 0.f;
    return;
  }
  if (MODE != kExpand) {
    const T* A = static_cast<const T*>(p.a_ptr[slot]) + p.a_off;
    const T* x = static_cast<const T*>(p.x) + static_cast<int64_t>(row) * p.ldx;
    for (int k = warp; k < R; k += kWarps) {
      float s = 0.f;
      for (int d = lane; d < p.h_in; d += 32)
        s = fmaf(Cvt<T>::to_f(x[d]), Cvt<T>::to_f(A[static_cast<int64_t>(d) * R + k]), s);
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (lane == 0) v_sm[k] = s;
    }
  } else {
    for (int k = tid; k < R; k += kThreads) v_sm[k] = p.v_in[static_cast<int64_t>(row) * R + k];
  }
  __syncthreads();
  if (MODE == kShrink) {
    for (int k = tid; k < R; k += kThreads) p.v_out[static_cast<int64_t>(row) * R + k] = v_sm[k];
    return;
  }
  const T* B = static_cast<const T*>(p.b_ptr[slot]) + p.b_off;
  T* y = static_cast<T*>(p.y) + static_cast<int64_t>(row) * p.ldy;
  for (int c = tid; c < p.h_out; c += kThreads) {
    float acc = 0.f;
    for (int k = 0; k < R; ++k) acc = fmaf(v_sm[k], Cvt<T>::to_f(B[static_cast<int64_t>(k) * p.h_out + c]), acc);
    y[c] = Cvt<T>::from_f(acc + Cvt<T>::to_f(y[c]));
  }
}

}  // namespace lsg
