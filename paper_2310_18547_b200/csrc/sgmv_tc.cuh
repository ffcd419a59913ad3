// sgmv_tc.cuh -- K5: tensor-core SGMV for long segments (prefill rows).
//
// Segments with >= kTcMinRows rows are cut into 128-row tiles and run through
// two tcgen05 kernels (launched back to back with programmatic dependent launch):
//
//   shrink  grid (nq, tiles), cluster (nq): CTA q computes the partial
//           D1[128 x r] (TMEM, fp32) = x[128 x kcs] . A[kcs x r] over its K
//           chunk q (kcs = h_in / nq).  x arrives by TMA (128B-swizzled boxes
//           of 64 x 128, ring of up to 6); A is re-laid out into the UMMA
//           MN-major swizzled form.  Each row's partial is pushed with st.async
//           to the CTA owning that row; owners sum the nq partials in chunk
//           order and store v [rows x r] (fp32) into the workspace.
//   expand  grid (h_out / 256, tiles), no cluster: v is split into 16-bit
//           hi + lo parts and D2[128 x 256] = hi . B + lo . B (TMEM); y_old is
//           staged by TMA (4 boxes of 64 x 128, 128B swizzle), the epilogue adds
//           D2 in place and the tile goes back by TMA store (partial tiles:
//           per-row stores of the segment's rows only).
//
// Canonical arithmetic for rows of long segments: v = sum over K chunks q
// (ascending) of the MMA partial of chunk q; y = rn(fp32(hi.B + lo.B) + y_old).
// Whether a segment takes this path depends only on its length and the shape,
// so results are independent of batch composition and segment order.
#pragma once

#include <cuda.h>

#include <type_traits>

#include "sgmv_device.cuh"
#include "sgmv_kernels.cuh"

namespace lsg {

constexpr int kTcMinRows = 128;  // segments at least this long use the tensor-core path
constexpr int kTcM = 128;        // rows per tile (UMMA M)
constexpr int kTcKB = 64;        // K per x box (128 bytes of 16-bit)
constexpr int kTcBox = kTcM * kTcKB * 2;  // 16 KB per 64 x 128 box
constexpr int kTcMaxStages = 6;  // x ring depth (shrink)
constexpr int kTcNT = 256;       // expand N tile (UMMA N)
constexpr int kTcThreads = 128;

struct TcShrinkParams {
  CUtensorMap tmap_x;  // x [s_n, h_in], box 64 x 128, 128B swizzle
  float* v;            // workspace [s_n][r] fp32 (rows of long segments only)
  const void* const* a_ptr;
  int64_t a_off;
  const int32_t* seg_starts;
  const int32_t* seg_slot;
  int32_t n_seg, s_n, num_slots, h_in, kcs;
  int32_t min_rows;  // segments with at least this many rows are this kernel's
  unsigned long long* trace;  // lsg_set_trace: %globaltimer stamps, entries [trace_ctas, 2 trace_ctas)
  int32_t trace_ctas;
};

struct TcExpandParams {
  CUtensorMap tmap_y;  // y [s_n, h_out], box 64 x 128, 128B swizzle
  void* y;
  int64_t ldy;
  const float* v;
  const void* const* b_ptr;
  int64_t b_off;
  const int32_t* seg_starts;
  const int32_t* seg_slot;
  int32_t n_seg, s_n, num_slots, h_out;
  int32_t min_rows;
  unsigned long long* trace;
  int32_t trace_ctas;
};

// Shrink CTAs trace into entries [trace_ctas, 1.5 trace_ctas), expand CTAs into
// [1.5 trace_ctas, 2 trace_ctas); 16 %globaltimer stamps each.
#ifdef LSG_INSTRUMENT
#define LSG_TC_TRACE_ON (p.trace != nullptr)
#else
#define LSG_TC_TRACE_ON false  // instrumented builds only (see sgmv_kernels.cuh)
#endif
#define LSG_TC_TRACE(base, i)                                                                        \
  do {                                                                                               \
    if (LSG_TC_TRACE_ON && threadIdx.x == 0) {                                                    \
      const int cta_ = blockIdx.y * gridDim.x + blockIdx.x;                                          \
      if (cta_ < p.trace_ctas / 2) {                                                                 \
        unsigned long long gt_;                                                                      \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));                                     \
        p.trace[(p.trace_ctas + (base) * (p.trace_ctas / 2) + cta_) * 16 + (i)] = gt_;               \
      }                                                                                              \
    }                                                                                                \
  } while (0)

// ---- tcgen05 / UMMA / TMA helpers ---------------------------------------------------
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // descriptor version (sm_100)
  d |= static_cast<uint64_t>(layout & 7) << 61;
  return d;
}
// layout codes of the shared-memory descriptor
constexpr uint32_t kSwNone = 0, kSw128 = 2, kSw64 = 4, kSw32 = 6;

// kind::f16 instruction descriptor: D fp32, A K-major, B MN-major
__host__ __device__ constexpr uint32_t umma_idesc(int fmt /*0 f16, 1 bf16*/, int M, int N) {
  return (1u << 4) | (static_cast<uint32_t>(fmt) << 7) | (static_cast<uint32_t>(fmt) << 10) | (0u << 15) |
         (1u << 16) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
               "n"(NCOLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t tmem) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(NCOLS));
}

// 32 lanes x 16 consecutive 32-bit TMEM columns -> 16 registers per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
      "[%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tmap, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tmap, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit_group() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_group0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// Wait only until the bulk stores have READ their shared-memory source (the global writes
// complete asynchronously and are covered by the grid's completion): enough before a CTA
// exits or reuses the staging.
__device__ __forceinline__ void bulk_wait_group_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}

// 16-byte chunk index XOR of the 32/64/128-byte swizzles for row k
template <int ROWB>
__device__ __forceinline__ int swz(int k) {
  if constexpr (ROWB == 32) return (k >> 2) & 1;
  else if constexpr (ROWB == 64) return (k >> 1) & 3;
  else return k & 7;
}

// Tile t of a launch -> (long segment, tile within it): warp-wide prefix sum of
// ceil(len / 128) over the segments with len >= kTcMinRows, 32 segments per step.
// Call from one full warp; seg = -1 past the last tile.
__device__ __forceinline__ void tc_tile_of(const int32_t* seg_starts, int n_seg, int t, int lane, int& seg,
                                           int& tin, int min_rows) {
  int base = 0;
  seg = -1;
  tin = 0;
  for (int c0 = 0; c0 < n_seg && seg < 0; c0 += 32) {
    const int sg = c0 + lane;
    int nt = 0;
    if (sg < n_seg) {
      const int len = seg_starts[sg + 1] - seg_starts[sg];
      nt = len >= min_rows ? (len + kTcM - 1) / kTcM : 0;
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
}

// ---- shared-memory plans (host and device) ---------------------------------------------
__host__ __device__ constexpr int tc_shrink_stages(int kcs) {
  return kcs / kTcKB < kTcMaxStages ? kcs / kTcKB : kTcMaxStages;
}
__host__ __device__ constexpr uint32_t tc_shrink_off_a(int kcs) { return tc_shrink_stages(kcs) * kTcBox; }
__host__ __device__ constexpr uint32_t tc_shrink_off_recv(int R, int kcs) {
  return (tc_shrink_off_a(kcs) + kcs * R * 2 + 127) & ~127u;
}
__host__ __device__ constexpr uint32_t tc_shrink_off_bars(int R, int kcs) {
  return tc_shrink_off_recv(R, kcs) + kTcM * R * 4;
}
__host__ __device__ constexpr uint32_t tc_shrink_smem(int R, int kcs) {
  return tc_shrink_off_bars(R, kcs) + 256 + 1024;  // + alignment slack
}
template <int R>
struct TcExpandLayout {
  static constexpr uint32_t kY = 0;                       // 4 boxes of 64 cols x 128 rows (SW128)
  static constexpr uint32_t kB = 4 * kTcBox;              // B [R x 256], MN-major SW128 atoms
  static constexpr uint32_t kVhi = kB + R * kTcNT * 2;    // v hi / lo: 128 x R, K-major interleave
  static constexpr uint32_t kVlo = kVhi + kTcM * R * 2;
  static constexpr uint32_t kBars = kVlo + kTcM * R * 2;
  static constexpr uint32_t kTotal = kBars + 64 + 1024;  // + alignment slack
};

// ---------------------------------------------------------------------------------------
// Shrink: v[tile rows] = x[tile rows] . A_slot   (cluster of nq CTAs over K)
// ---------------------------------------------------------------------------------------
template <typename T, int R>
__global__ void __launch_bounds__(kTcThreads) sgmv_tc_shrink_kernel(const __grid_constant__ TcShrinkParams p) {
  static_assert(R == 16 || R == 32 || R == 64, "tensor-core path ranks");
  constexpr int ROWB = 2 * R;  // bytes per A row (MN-major swizzle width)
  constexpr uint32_t kSwA = R == 16 ? kSw32 : (R == 32 ? kSw64 : kSw128);
  constexpr int kTmemCols = R < 32 ? 32 : R;
  constexpr int fmt = std::is_same<T, __half>::value ? 0 : 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int nq = static_cast<int>(gridDim.x), q = static_cast<int>(blockIdx.x);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kcs = p.kcs, nkb = kcs / kTcKB, stages = tc_shrink_stages(kcs);
  uint8_t* xs = smem;
  uint8_t* As = smem + tc_shrink_off_a(kcs);
  float* recv = reinterpret_cast<float*>(smem + tc_shrink_off_recv(R, kcs));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + tc_shrink_off_bars(R, kcs));
  // bars: [0, 8) full[s], [8, 16) empty[s], 16 D1 ready, 17 partials in
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

  LSG_TC_TRACE(0, 0);
  __shared__ int s_seg, s_tile;
  if (warp == 0) {
    int seg, tin;
    tc_tile_of(p.seg_starts, p.n_seg, blockIdx.y, lane, seg, tin, p.min_rows);
    if (lane == 0) {
      s_seg = seg;
      s_tile = tin;
    }
  }
  __syncthreads();
  // CTAs without work leave at once (freeing their SM for the next grid) except the
  // first cluster, which always waits for the preceding grid: this grid's completion
  // (and its trigger, which the expand relies on for staging y_old early) then still
  // implies the predecessor's.
  if (s_seg < 0) {  // past the last tile (the grid is an upper bound), whole cluster
    if (blockIdx.y == 0) pdl_wait();
    return;
  }
  const int slot = p.seg_slot[s_seg];
  if (slot < 0 || slot >= p.num_slots) {  // no adapter: the expand leaves y untouched
    if (blockIdx.y == 0) pdl_wait();
    return;
  }
  const int seg_end = p.seg_starts[s_seg + 1];
  const int r0 = p.seg_starts[s_seg] + s_tile * kTcM;
  const int rows = min(kTcM, seg_end - r0);
  const int k0 = q * kcs;
  const int rpo = kTcM / nq;  // rows reduced by each CTA

  if (tid == 0) {
    for (int i = 0; i < 18; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
    prefetch_tmap(&p.tmap_x);
  }
  if (warp == 0) tmem_alloc<kTmemCols>(tmem_slot);
  // ---- A chunk (weights: independent of the preceding kernel) -> MN-major swizzled smem
  {
    const T* A = static_cast<const T*>(p.a_ptr[slot]) + p.a_off + static_cast<int64_t>(k0) * R;
    constexpr int CPR = ROWB / 16;  // 16-byte chunks per A row
    const int total = kcs * CPR;
    for (int base = 0; base < total; base += 8 * kTcThreads) {
      uint4 va[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = base + j * kTcThreads + tid;
        if (i < total) va[j] = ldg_nc_v4(A + static_cast<int64_t>(i) * 8);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = base + j * kTcThreads + tid;
        if (i < total) {
          const int k = i / CPR, c = i - k * CPR;
          *reinterpret_cast<uint4*>(As + k * ROWB + ((c ^ swz<ROWB>(k)) * 16)) = va[j];
        }
      }
    }
  }
  fence_proxy_async_smem();  // generic smem writes -> visible to the tensor cores
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  cluster_arrive_relaxed();  // barrier inits -> the cluster (waited on before the first push)
  LSG_TC_TRACE(0, 1);

  pdl_wait();  // x may come from the preceding kernel
  // Dependents (the expand) start only now: every kernel before this one has
  // completed, so the expand may read y_old before its own wait (it waits only
  // for v from this kernel).
  pdl_launch_dependents();
  LSG_TC_TRACE(0, 2);
  const uint32_t idesc = umma_idesc(fmt, kTcM, R);
  if (warp == 1 && lane == 0) {  // TMA producer
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % stages;
      if (kb >= stages) mbar_wait(&bars[8 + s], ((kb / stages) - 1) & 1);
      mbar_arrive_expect_tx(&bars[s], kTcBox);
      tma_load_2d(xs + s * kTcBox, &p.tmap_x, k0 + kb * kTcKB, r0, &bars[s]);
    }
  } else if (warp == 0 && lane == 0) {  // MMA issuer
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % stages;
      mbar_wait(&bars[s], (kb / stages) & 1);
      tc_fence_after();
      const uint32_t xa = smem_u32(xs + s * kTcBox);
      const uint32_t aa = smem_u32(As) + kb * kTcKB * ROWB;
#pragma unroll
      for (int ks = 0; ks < kTcKB / 16; ++ks) {
        const uint64_t ad = umma_desc(xa + ks * 32, 16, 1024, kSw128);           // x: K-major SW128
        const uint64_t bd = umma_desc(aa + ks * 16 * ROWB, 16, 8 * ROWB, kSwA);  // A: MN-major
        umma_f16(tmem, ad, bd, idesc, (kb | ks) ? 1u : 0u);
      }
      umma_commit(&bars[8 + s]);  // stage free once these MMAs have read it
    }
    umma_commit(&bars[16]);  // D1 complete
  }
  __syncwarp();  // producer / issuer lanes rejoin their warps before .aligned ops

  // ---- reduce: each row's partial -> the CTA owning the row ----------------------------
  cluster_wait();  // peers' barriers initialised
  if (tid == 0) mbar_arrive_expect_tx(&bars[17], static_cast<uint32_t>(nq * rpo * R * 4));
  mbar_wait(&bars[16], 0);
  LSG_TC_TRACE(0, 3);
  tc_fence_after();
  {
    const int m = warp * 32 + lane;
    const int owner = m / rpo, ml = m - owner * rpo;
    const uint32_t rb = mapa_u32(&bars[17], static_cast<uint32_t>(owner));
#pragma unroll
    for (int c0 = 0; c0 < R; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
      const uint32_t ra = mapa_u32(recv + (q * rpo + ml) * R + c0, static_cast<uint32_t>(owner));
#pragma unroll
      for (int j = 0; j < 4; ++j) st_async_v4(ra + j * 16, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3], rb);
    }
  }
  mbar_wait(&bars[17], 0);
  LSG_TC_TRACE(0, 4);
  // v[r0 + q*rpo + ml][k] = sum over chunks qq (ascending) -- rows of this segment only
  for (int i = tid; i < rpo * R; i += kTcThreads) {
    const int ml = i / R, k = i - ml * R;
    float s = 0.f;
    for (int qq = 0; qq < nq; ++qq) s += recv[(qq * rpo + ml) * R + k];
    const int m = q * rpo + ml;
    if (m < rows) p.v[static_cast<int64_t>(r0 + m) * R + k] = s;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
  LSG_TC_TRACE(0, 5);
}

// ---------------------------------------------------------------------------------------
// Expand: y[tile rows, n0 : n0 + 256] = rn(v . B_slot + y_old)
// ---------------------------------------------------------------------------------------
template <typename T, int R>
__global__ void __launch_bounds__(kTcThreads) sgmv_tc_expand_kernel(const __grid_constant__ TcExpandParams p) {
  static_assert(R == 16 || R == 32 || R == 64, "tensor-core path ranks");
  using L = TcExpandLayout<R>;
  constexpr int fmt = std::is_same<T, __half>::value ? 0 : 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = static_cast<int>(blockIdx.x) * kTcNT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBars);  // 0 y landed, 1 D2 ready
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);

  LSG_TC_TRACE(1, 0);
  pdl_launch_dependents();
  __shared__ int s_seg, s_tile;
  if (warp == 0) {
    int seg, tin;
    tc_tile_of(p.seg_starts, p.n_seg, blockIdx.y, lane, seg, tin, p.min_rows);
    if (lane == 0) {
      s_seg = seg;
      s_tile = tin;
    }
  }
  __syncthreads();
  // (as in the shrink: only the first tile's CTAs wait before leaving without work)
  if (s_seg < 0) {
    if (blockIdx.y == 0) pdl_wait();
    return;
  }
  const int slot = p.seg_slot[s_seg];
  if (slot < 0 || slot >= p.num_slots) {  // no adapter: y untouched
    if (blockIdx.y == 0) pdl_wait();
    return;
  }
  const int seg_end = p.seg_starts[s_seg + 1];
  const int r0 = p.seg_starts[s_seg] + s_tile * kTcM;
  const int rows = min(kTcM, seg_end - r0);

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    prefetch_tmap(&p.tmap_y);
  }
  if (warp == 0) tmem_alloc<kTcNT>(tmem_slot);
  // y_old: written only by kernels before the shrink, which all completed before
  // the shrink triggered this launch -- staged ahead of the wait for v.
  if (tid == 0) {
    mbar_arrive_expect_tx(&bars[0], 4 * kTcBox);
#pragma unroll
    for (int b = 0; b < 4; ++b) tma_load_2d(smem + L::kY + b * kTcBox, &p.tmap_y, n0 + b * kTcKB, r0, &bars[0]);
  }
  // ---- B block [R x 256] (weights) -> MN-major SW128 atoms: 64-col atom na, k-group kg:
  //      na*(R/8)*1024 + kg*1024 + (k%8)*128 + swizzled 16-byte chunk
  {
    const T* B = static_cast<const T*>(p.b_ptr[slot]) + p.b_off + n0;
    constexpr int total = R * (kTcNT / 8);
    constexpr int per = total / kTcThreads;  // 4 / 8 / 16
    uint4 vb[per];
#pragma unroll
    for (int j = 0; j < per; ++j) {
      const int i = j * kTcThreads + tid, k = i / (kTcNT / 8), cc = i - k * (kTcNT / 8);
      vb[j] = ldg_nc_v4(B + static_cast<int64_t>(k) * p.h_out + cc * 8);
    }
#pragma unroll
    for (int j = 0; j < per; ++j) {
      const int i = j * kTcThreads + tid, k = i / (kTcNT / 8), cc = i - k * (kTcNT / 8);
      const int na = cc / 8, jj = cc % 8;
      *reinterpret_cast<uint4*>(smem + L::kB + na * (R / 8) * 1024 + (k / 8) * 1024 + (k % 8) * 128 +
                                ((jj ^ (k % 8)) * 16)) = vb[j];
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  LSG_TC_TRACE(1, 1);

  pdl_wait();  // v (the shrink) is ready
  LSG_TC_TRACE(1, 2);
  // v -> 16-bit hi + lo, K-major interleave: (m,k) at (m/8)*SBO + (k/8)*128 + (m%8)*16 + (k%8)*2
  {
    const int m = tid;
    const float* vr = p.v + static_cast<int64_t>(r0 + m) * R;
#pragma unroll
    for (int kg = 0; kg < R / 8; ++kg) {
      float f[8], hf[8], lo[8];
      if (m < rows) {
        const float4 a = *reinterpret_cast<const float4*>(vr + kg * 8);
        const float4 b = *reinterpret_cast<const float4*>(vr + kg * 8 + 4);
        f[0] = a.x, f[1] = a.y, f[2] = a.z, f[3] = a.w, f[4] = b.x, f[5] = b.y, f[6] = b.z, f[7] = b.w;
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = 0.f;
      }
      const uint4 hi = Cvt<T>::pack8(f);
      Cvt<T>::unpack8(hi, hf);
#pragma unroll
      for (int j = 0; j < 8; ++j) lo[j] = f[j] - hf[j];
      const uint32_t off = (m / 8) * (R / 8) * 128 + kg * 128 + (m % 8) * 16;
      *reinterpret_cast<uint4*>(smem + L::kVhi + off) = hi;
      *reinterpret_cast<uint4*>(smem + L::kVlo + off) = Cvt<T>::pack8(lo);
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  if (warp == 0 && lane == 0) {
    tc_fence_after();
    const uint32_t idesc = umma_idesc(fmt, kTcM, kTcNT);
    const uint32_t bs = smem_u32(smem + L::kB);
#pragma unroll
    for (int ks = 0; ks < R / 16; ++ks) {
      const uint64_t bd = umma_desc(bs + ks * 2 * 1024, (R / 8) * 1024, 1024, kSw128);  // B: MN-major SW128
      const uint64_t ah = umma_desc(smem_u32(smem + L::kVhi) + ks * 256, 128, (R / 8) * 128, kSwNone);
      const uint64_t al = umma_desc(smem_u32(smem + L::kVlo) + ks * 256, 128, (R / 8) * 128, kSwNone);
      umma_f16(tmem, ah, bd, idesc, ks ? 1u : 0u);
      umma_f16(tmem, al, bd, idesc, 1u);
    }
    umma_commit(&bars[1]);
  }
  __syncwarp();
  // ---- epilogue: row m = this thread; y_old from the swizzled staging, in place ----------
  mbar_wait(&bars[0], 0);
  LSG_TC_TRACE(1, 3);
  mbar_wait(&bars[1], 0);
  LSG_TC_TRACE(1, 4);
  tc_fence_after();
  const int m = tid;
  uint8_t* yrow = smem + L::kY + m * 128;  // + box * kTcBox + swizzled chunk
#pragma unroll 4
  for (int c = 0; c < kTcNT / 16; ++c) {
    float acc[16];
    tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c * 16, acc);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = (c % 4) * 2 + h;
      uint4* ptr = reinterpret_cast<uint4*>(yrow + (c / 4) * kTcBox + ((j ^ (m & 7)) * 16));
      float f[8];
      Cvt<T>::unpack8(*ptr, f);
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] = acc[h * 8 + e] + f[e];
      *ptr = Cvt<T>::pack8(f);
    }
  }
  if (rows == kTcM) {
    fence_proxy_async_smem();  // epilogue writes -> visible to the TMA store
    __syncthreads();
    if (tid == 0) {
#pragma unroll
      for (int b = 0; b < 4; ++b) tma_store_2d(&p.tmap_y, smem + L::kY + b * kTcBox, n0 + b * kTcKB, r0);
      bulk_commit_group();
      bulk_wait_group_read0();
    }
  } else if (m < rows) {  // last tile of a segment: only the segment's rows
    T* yg = static_cast<T*>(p.y) + static_cast<int64_t>(r0 + m) * p.ldy + n0;
#pragma unroll 4
    for (int i = 0; i < kTcNT / 8; ++i) {
      const int b = i / 8, j = i % 8;
      st_global_v4(yg + i * 8, *reinterpret_cast<const uint4*>(yrow + b * kTcBox + ((j ^ (m & 7)) * 16)));
    }
  }
  LSG_TC_TRACE(1, 5);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<kTcNT>(tmem);
  }
}

}  // namespace lsg

namespace lsg {

// ---------------------------------------------------------------------------------------
// Fused long-segment kernel (rank 16): ONE launch per call for all long-segment tiles.
// A cluster of C CTAs serves one 128-row tile:
//   shrink  CTA c: D1 (TMEM, fp32 128 x 16) = x[tile, K boxes of c] . A[K boxes of c]
//           (x by TMA through a ring, A MN-major swizzled); row partials go to the
//           row owners (st.async DSMEM), owners add the C partials in CTA order and
//           broadcast their rows of v to the whole cluster -- v never leaves the chip;
//   expand  CTA c: 256-column chunks j = c, c + C of y: D2 (TMEM, the 256 columns D1
//           used -- D1 is consumed first, so two CTAs fit one SM's TMEM) = hi.B_j + lo.B_j
//           (v split into 16-bit hi + lo), epilogue adds y_old (TMA-staged while the
//           shrink runs) and stores the tile (TMA store; per-row stores on a
//           segment's last, partial tile).
// Canonical arithmetic for these rows: v = sum over CTAs c (ascending) of the MMA
// partial over c's K boxes (C and the box split depend only on the shape);
// y = rn(fp32(hi.B + lo.B) + y_old).
// ---------------------------------------------------------------------------------------
constexpr int kTcfStages = 4;  // x ring depth
struct TcFusedParams {
  CUtensorMap tmap_x;  // x [s_n, h_in], box 64 x 128, SW128
  CUtensorMap tmap_y;  // y [s_n, h_out], box 64 x 128, SW128
  void* y;
  int64_t ldy;
  const void* const* a_ptr;
  const void* const* b_ptr;
  int64_t a_off, b_off;
  const int32_t* seg_starts;
  const int32_t* seg_slot;
  int32_t n_seg, s_n, num_slots, h_in, h_out;
  int32_t kcs_max;  // max K columns per CTA (multiple of 64)
  int32_t compact;  // 1: one 256-column chunk per CTA, y staged in the x ring after the shrink (2 CTAs/SM)
  int32_t min_rows;
  unsigned long long* trace;
  int32_t trace_ctas;
};

// Shared-memory plan (offsets from the 1024-aligned base), R = 16.
struct TcfLayout {
  uint32_t ring, y0, a, b, vhi, vlo, recv, vfull, bars, total;
};
__host__ __device__ inline TcfLayout tcf_layout(int kcs_max, int compact) {
  TcfLayout L{};
  L.ring = 0;                              // x ring; after the shrink: y staging of chunk 1 (or 0 if compact)
  L.y0 = kTcfStages * kTcBox;              // y staging of chunk 0 (4 boxes, SW128)
  L.a = compact ? L.y0 : L.y0 + 4 * kTcBox;  // A slice, kcs_max rows x 32 B (MN-major SW32)
  L.b = L.a + static_cast<uint32_t>(kcs_max) * 32;  // B chunks: (1 or 2) x (16 x 256) MN-major SW128 atoms
  L.vhi = L.b + (compact ? 1 : 2) * 16 * kTcNT * 2;
  L.vlo = L.vhi + kTcM * 16 * 2;
  L.recv = L.vlo + kTcM * 16 * 2;          // [C][128/C][16] fp32 row partials = 8 KB for any C
  L.vfull = L.recv + kTcM * 16 * 4;        // [128][16] fp32 v of the tile
  L.bars = L.vfull + kTcM * 16 * 4;
  L.total = L.bars + 256 + 1024;           // + alignment slack
  return L;
}

template <typename T>
__global__ void __launch_bounds__(kTcThreads, 1) sgmv_tc_fused_kernel(const __grid_constant__ TcFusedParams p) {
  constexpr int R = 16;
  constexpr int fmt = std::is_same<T, __half>::value ? 0 : 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const TcfLayout L = tcf_layout(p.kcs_max, p.compact);
  const int C = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  // bars: [0,4) full[s], [4,8) empty[s], 8 D1, 9 recv, 10 vfull, 11 y0, 12 y1, 13 D2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
  float* recv = reinterpret_cast<float*>(smem + L.recv);
  float* vfull = reinterpret_cast<float*>(smem + L.vfull);

  LSG_TC_TRACE(0, 0);
  pdl_launch_dependents();  // the next kernel only stages weights before its own wait
  __shared__ int s_seg, s_tile;
  if (warp == 0) {
    int seg, tin;
    tc_tile_of(p.seg_starts, p.n_seg, blockIdx.y, lane, seg, tin, p.min_rows);
    if (lane == 0) {
      s_seg = seg;
      s_tile = tin;
    }
  }
  __syncthreads();
  // CTAs without work leave at once, except the first tile's cluster, which waits for
  // the preceding grid so this grid's completion still implies the predecessor's.
  if (s_seg < 0) {  // past the last tile (the grid is an upper bound)
    if (blockIdx.y == 0) pdl_wait();
    return;
  }
  const int slot = p.seg_slot[s_seg];
  if (slot < 0 || slot >= p.num_slots) {  // no adapter: rows untouched
    if (blockIdx.y == 0) pdl_wait();
    return;
  }
  const int seg_end = p.seg_starts[s_seg + 1];
  const int r0 = p.seg_starts[s_seg] + s_tile * kTcM;
  const int rows = min(kTcM, seg_end - r0);
  const int nkb = p.h_in / kTcKB, kb0 = (c * nkb) / C, nk = ((c + 1) * nkb) / C - kb0;
  const int nch = p.h_out / kTcNT, nmine = c < nch ? (nch - 1 - c) / C + 1 : 0;  // <= 2 (host checks)
  const int rpo = kTcM / C;

  if (tid == 0) {
    for (int i = 0; i < 14; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
    prefetch_tmap(&p.tmap_x);
    prefetch_tmap(&p.tmap_y);
  }
  if (warp == 0) tmem_alloc<kTcNT>(tmem_slot);
  // ---- weights (independent of the preceding kernel) --------------------------------
  {  // A rows [kb0*64, (kb0+nk)*64) -> MN-major SW32: row k at k*32, 16-byte chunk c ^ swz<32>(k)
    const T* A = static_cast<const T*>(p.a_ptr[slot]) + p.a_off + static_cast<int64_t>(kb0) * kTcKB * R;
    const int total = nk * kTcKB * 2;  // 16-byte chunks
    for (int base = 0; base < total; base += 8 * kTcThreads) {
      uint4 va[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = base + j * kTcThreads + tid;
        if (i < total) va[j] = ldg_nc_v4(A + static_cast<int64_t>(i) * 8);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = base + j * kTcThreads + tid;
        if (i < total) {
          const int k = i >> 1, cc = i & 1;
          *reinterpret_cast<uint4*>(smem + L.a + k * 32 + ((cc ^ swz<32>(k)) * 16)) = va[j];
        }
      }
    }
  }
  for (int i = 0; i < nmine; ++i) {  // B chunk j -> MN-major SW128 atoms (as the two-kernel expand)
    const int n0 = (c + i * C) * kTcNT;
    const T* B = static_cast<const T*>(p.b_ptr[slot]) + p.b_off + n0;
    constexpr int per = R * (kTcNT / 8) / kTcThreads;  // 4
    uint4 vb[per];
#pragma unroll
    for (int j = 0; j < per; ++j) {
      const int e = j * kTcThreads + tid, k = e / (kTcNT / 8), cc = e - k * (kTcNT / 8);
      vb[j] = ldg_nc_v4(B + static_cast<int64_t>(k) * p.h_out + cc * 8);
    }
#pragma unroll
    for (int j = 0; j < per; ++j) {
      const int e = j * kTcThreads + tid, k = e / (kTcNT / 8), cc = e - k * (kTcNT / 8);
      const int na = cc / 8, jj = cc % 8;
      *reinterpret_cast<uint4*>(smem + L.b + i * (R * kTcNT * 2) + na * (R / 8) * 1024 + (k / 8) * 1024 +
                                (k % 8) * 128 + ((jj ^ (k % 8)) * 16)) = vb[j];
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  cluster_arrive_relaxed();  // barrier inits -> the cluster (waited on before the first push)
  LSG_TC_TRACE(0, 1);

  pdl_wait();  // x and y_old may come from the preceding kernel
  LSG_TC_TRACE(0, 2);
  if (warp == 1 && lane == 0) {  // TMA producer: y chunk 0, the x ring, then y chunk 1
    if (nmine > 0 && !p.compact) {
      mbar_arrive_expect_tx(&bars[11], 4 * kTcBox);
#pragma unroll
      for (int b = 0; b < 4; ++b)
        tma_load_2d(smem + L.y0 + b * kTcBox, &p.tmap_y, c * kTcNT + b * kTcKB, r0, &bars[11]);
    }
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kTcfStages;
      if (kb >= kTcfStages) mbar_wait(&bars[4 + s], ((kb / kTcfStages) - 1) & 1);
      mbar_arrive_expect_tx(&bars[s], kTcBox);
      tma_load_2d(smem + L.ring + s * kTcBox, &p.tmap_x, (kb0 + kb) * kTcKB, r0, &bars[s]);
    }
    const int ring_chunk = p.compact ? 0 : 1;  // the chunk staged in the ring once the shrink is done
    if (nmine > ring_chunk) {
      mbar_wait(&bars[8], 0);  // every shrink MMA has read its x box: the ring is free
      mbar_arrive_expect_tx(&bars[11 + ring_chunk], 4 * kTcBox);
#pragma unroll
      for (int b = 0; b < 4; ++b)
        tma_load_2d(smem + L.ring + b * kTcBox, &p.tmap_y, (c + ring_chunk * C) * kTcNT + b * kTcKB, r0,
                    &bars[11 + ring_chunk]);
    }
  } else if (warp == 0 && lane == 0) {  // MMA issuer (shrink)
    const uint32_t idesc = umma_idesc(fmt, kTcM, R);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kTcfStages;
      mbar_wait(&bars[s], (kb / kTcfStages) & 1);
      tc_fence_after();
      const uint32_t xa = smem_u32(smem + L.ring + s * kTcBox);
      const uint32_t aa = smem_u32(smem + L.a) + kb * kTcKB * 32;
#pragma unroll
      for (int ks = 0; ks < kTcKB / 16; ++ks) {
        const uint64_t ad = umma_desc(xa + ks * 32, 16, 1024, kSw128);          // x: K-major SW128
        const uint64_t bd = umma_desc(aa + ks * 16 * 32, 16, 8 * 32, kSw32);     // A: MN-major SW32
        umma_f16(tmem, ad, bd, idesc, (kb | ks) ? 1u : 0u);
      }
      umma_commit(&bars[4 + s]);
    }
    umma_commit(&bars[8]);  // D1 complete (and the ring free)
  }
  __syncwarp();

  // ---- cluster reduction of v: row partials -> owners -> every CTA ---------------------
  cluster_wait();  // peers' barriers initialised
  if (tid == 0) {
    mbar_arrive_expect_tx(&bars[9], static_cast<uint32_t>(C * rpo * R * 4));
    mbar_arrive_expect_tx(&bars[10], static_cast<uint32_t>(kTcM * R * 4));
  }
  mbar_wait(&bars[8], 0);
  LSG_TC_TRACE(0, 3);
  tc_fence_after();
  {
    const int m = tid;  // row of the tile = TMEM lane
    const int owner = m / rpo, ml = m - owner * rpo;
    float v[16];
    tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16), v);
    const uint32_t ra = mapa_u32(recv + (c * rpo + ml) * R, static_cast<uint32_t>(owner));
    const uint32_t rb = mapa_u32(&bars[9], static_cast<uint32_t>(owner));
#pragma unroll
    for (int j = 0; j < 4; ++j) st_async_v4(ra + j * 16, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3], rb);
  }
  mbar_wait(&bars[9], 0);
  for (int qd = tid; qd < rpo * R / 4; qd += kTcThreads) {  // my rows' v, 4 columns per thread
    const int ml = qd / (R / 4), k4 = (qd - ml * (R / 4)) * 4;
    float s[4] = {0.f, 0.f, 0.f, 0.f};
    for (int cc = 0; cc < C; ++cc)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[e] += recv[(cc * rpo + ml) * R + k4 + e];
    const float* lv = vfull + (c * rpo + ml) * R + k4;
    for (int d = 0; d < C; ++d)
      st_async_v4(mapa_u32(lv, static_cast<uint32_t>(d)), s[0], s[1], s[2], s[3],
                  mapa_u32(&bars[10], static_cast<uint32_t>(d)));
  }
  mbar_wait(&bars[10], 0);
  LSG_TC_TRACE(0, 4);
  {  // v -> 16-bit hi + lo, K-major interleave (m,k) at (m/8)*256 + (k/8)*128 + (m%8)*16 + (k%8)*2
    const int m = tid;
#pragma unroll
    for (int kg = 0; kg < R / 8; ++kg) {
      float f[8], hf[8], lo[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] = vfull[m * R + kg * 8 + e];
      const uint4 hi = Cvt<T>::pack8(f);
      Cvt<T>::unpack8(hi, hf);
#pragma unroll
      for (int e = 0; e < 8; ++e) lo[e] = f[e] - hf[e];
      const uint32_t off = (m / 8) * (R / 8) * 128 + kg * 128 + (m % 8) * 16;
      *reinterpret_cast<uint4*>(smem + L.vhi + off) = hi;
      *reinterpret_cast<uint4*>(smem + L.vlo + off) = Cvt<T>::pack8(lo);
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();

  // ---- expand: my 256-column chunks ----------------------------------------------------
  for (int i = 0; i < nmine; ++i) {
    const int n0 = (c + i * C) * kTcNT;
    uint8_t* ybuf = smem + (i == 0 && !p.compact ? L.y0 : L.ring);
    if (warp == 0 && lane == 0) {
      tc_fence_after();
      const uint32_t idesc = umma_idesc(fmt, kTcM, kTcNT);
      const uint32_t bs = smem_u32(smem + L.b + i * (R * kTcNT * 2));
      const uint64_t bd = umma_desc(bs, (R / 8) * 1024, 1024, kSw128);  // B: MN-major SW128
      const uint64_t ah = umma_desc(smem_u32(smem + L.vhi), 128, (R / 8) * 128, kSwNone);
      const uint64_t al = umma_desc(smem_u32(smem + L.vlo), 128, (R / 8) * 128, kSwNone);
      umma_f16(tmem, ah, bd, idesc, 0u);
      umma_f16(tmem, al, bd, idesc, 1u);
      umma_commit(&bars[13]);
    }
    __syncwarp();
    mbar_wait(&bars[11 + i], 0);
    mbar_wait(&bars[13], i & 1);
    LSG_TC_TRACE(0, 5 + i);
    tc_fence_after();
    const int m = tid;
    uint8_t* yrow = ybuf + m * 128;  // + box * kTcBox + swizzled chunk
#pragma unroll 4
    for (int cc = 0; cc < kTcNT / 16; ++cc) {
      float acc[16];
      tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cc * 16, acc);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = (cc % 4) * 2 + h;
        uint4* ptr = reinterpret_cast<uint4*>(yrow + (cc / 4) * kTcBox + ((j ^ (m & 7)) * 16));
        float f[8];
        Cvt<T>::unpack8(*ptr, f);
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = acc[h * 8 + e] + f[e];
        *ptr = Cvt<T>::pack8(f);
      }
    }
    tc_fence_before();  // D2 reads done before the next chunk's MMA overwrites it
    if (rows == kTcM) {
      fence_proxy_async_smem();  // epilogue writes -> visible to the TMA store
      __syncthreads();
      if (tid == 0) {
#pragma unroll
        for (int b = 0; b < 4; ++b) tma_store_2d(&p.tmap_y, ybuf + b * kTcBox, n0 + b * kTcKB, r0);
        bulk_commit_group();
      }
    } else {
      if (m < rows) {  // last tile of a segment: only the segment's rows
        T* yg = static_cast<T*>(p.y) + static_cast<int64_t>(r0 + m) * p.ldy + n0;
#pragma unroll 4
        for (int e = 0; e < kTcNT / 8; ++e) {
          const int b = e / 8, j = e % 8;
          st_global_v4(yg + e * 8, *reinterpret_cast<const uint4*>(yrow + b * kTcBox + ((j ^ (m & 7)) * 16)));
        }
      }
      __syncthreads();
    }
  }
  if (tid == 0) bulk_wait_group_read0();  // TMA stores have read their staging before exit
  LSG_TC_TRACE(0, 7);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<kTcNT>(tmem);
  }
}

}  // namespace lsg

namespace lsg {

// ---------------------------------------------------------------------------------------
// Dense projection with the LoRA add in the GEMM epilogue, decode shape
// (s_n <= 64 rows): y = x . W + v . B_seg(row)   (reference dense_projection,
// sgmv.cpp:143-155: x.W + lora_addon).  v = x . A comes from the shrink kernel.
// A cluster of kDlKS CTAs per 64-column tile of y splits K: CTA c streams its K slice
// of x (K-major) and W (MN-major) through a TMA ring into tcgen05.mma (partial D_c,
// fp32 in TMEM, M = 128 with rows >= s_n zero).  Row m's partials go to the CTA owning
// rows [16c, 16c + 16) over DSMEM; the owner sums them in CTA order, adds
// sum_k v[m,k] B_seg(m)[k,n] (fp32 chain over k; its rows' B slices staged by
// cp.async ahead of the PDL wait) and rounds once.
// ---------------------------------------------------------------------------------------
#ifndef LSG_DL_N
#define LSG_DL_N 64
#endif
constexpr int kDlN = LSG_DL_N;  // columns per cluster (64 or 128: W as kDlN / 64 stacked 64-column boxes)
constexpr int kDlMaxRows = 64;  // decode rows per launch
constexpr int kDlKS = 4;        // K split = cluster size; CTA c owns rows [16c, 16c + 16)
constexpr int kDlRowsPer = kDlMaxRows / kDlKS;
#ifndef LSG_DL_STAGES
#define LSG_DL_STAGES 3
#endif
constexpr int kDlStages = LSG_DL_STAGES;
// x box of the 64 decode rows (8 KB) + W box (8 KB).  The MMA's M is 128: its A rows 64..127
// read the stage's W box -- garbage rows of D that nobody reads (rows >= 64 are padding).
constexpr int kDlXB = kDlMaxRows * kTcKB * 2;
constexpr int kDlStage = kDlXB + kTcKB * kDlN * 2;

struct DenseLoraParams {
  CUtensorMap tmap_x;  // x [s_n, h_in], box 64 (k) x 64 rows, SW128
  CUtensorMap tmap_w;  // W [h_in, h_out] row-major as 3-D {64 (N), h_in (K), h_out / 64}, box {64, 64, kDlN / 64}, SW128
  void* y;
  int64_t ldy;
  const float* v;      // [s_n, R] fp32
  const void* const* b_ptr;
  int64_t b_off;
  const int32_t* seg_starts;
  const int32_t* seg_slot;
  int32_t n_seg, s_n, num_slots, h_in, h_out;
};

template <int R>
struct DlLayout {
  static constexpr uint32_t kB = kDlStages * kDlStage;  // my rows' B slices
#ifdef LSG_DL_ALIAS
  // the partials' receive buffer reuses the ring once every CTA of the cluster is done with it
  static constexpr uint32_t kRecv = 0;
  static constexpr uint32_t kBars = kB + kDlRowsPer * R * kDlN * 2;
  static_assert(kDlKS * kDlRowsPer * kDlN * 4 <= kDlStages * kDlStage, "receive buffer fits the ring");
#else
  static constexpr uint32_t kRecv = kB + kDlRowsPer * R * kDlN * 2;  // [src][16 rows][64] fp32
  static constexpr uint32_t kBars = kRecv + kDlKS * kDlRowsPer * kDlN * 4;
#endif
  static constexpr uint32_t kTotal = kBars + 256 + 1024;
};
template <int R>
__host__ __device__ constexpr uint32_t dl_smem() {
  return DlLayout<R>::kTotal;
}

template <typename T, int R>
__global__ void __launch_bounds__(kTcThreads, 1) dense_lora_kernel(const __grid_constant__ DenseLoraParams p) {
  using L = DlLayout<R>;
  constexpr int fmt = std::is_same<T, __half>::value ? 0 : 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* Bsm = smem + L::kB;  // [local row][k][64 cols] 16-bit
  float* recv = reinterpret_cast<float*>(smem + L::kRecv);
  constexpr int S = kDlStages;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBars);  // full[S], empty[S], D, recv
  uint64_t* const bar_d = bars + 2 * S;
  uint64_t* const bar_recv = bars + 2 * S + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 2);
  __shared__ int s_slot[kDlRowsPer];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = static_cast<int>(blockIdx.x);  // cluster rank = K slice = owned row block
  const int n0 = static_cast<int>(blockIdx.y) * kDlN;
  const int nkb_all = p.h_in / kTcKB, kb0 = (c * nkb_all) / kDlKS, nkb = ((c + 1) * nkb_all) / kDlKS - kb0;

  if (tid == 0) {
    for (int i = 0; i < 2 * S + 2; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
    prefetch_tmap(&p.tmap_x);
    prefetch_tmap(&p.tmap_w);
  }
  if (warp == 0) tmem_alloc<kDlN>(tmem_slot);
  if (tid < kDlRowsPer) {  // slot of owned row c*16 + tid: last s with seg_starts[s] <= row
    const int m = c * kDlRowsPer + tid;
    int slot = -1;
    if (m < p.s_n) {
      int lo = 0, hi = p.n_seg;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (p.seg_starts[mid + 1] > m) hi = mid; else lo = mid + 1;
      }
      slot = lo < p.n_seg ? p.seg_slot[lo] : -1;
      if (slot >= p.num_slots) slot = -1;
    }
    s_slot[tid] = slot;
  }
  __syncthreads();
  // my rows' B[:, n0 : n0 + 64] (weights: before the PDL wait)
  for (int i = tid; i < kDlRowsPer * R * (kDlN / 8); i += kTcThreads) {
    const int ml = i / (R * (kDlN / 8)), rem = i - ml * (R * (kDlN / 8)), k = rem / (kDlN / 8), cc = rem % (kDlN / 8);
    const int slot = s_slot[ml];
    if (slot >= 0)
      cp_async16(Bsm + ((ml * R + k) * kDlN + cc * 8) * 2,
                 static_cast<const T*>(p.b_ptr[slot]) + p.b_off + static_cast<int64_t>(k) * p.h_out + n0 + cc * 8);
  }
  cp_async_commit();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  cluster_arrive_relaxed();  // barrier inits -> the cluster

  // TMA producer: the first ring's W boxes before the PDL wait (W is a weight), then x
  const int pre = nkb < S ? nkb : S;
  if (warp == 1 && lane == 0)
    for (int kb = 0; kb < pre; ++kb) {
      mbar_arrive_expect_tx(&bars[kb], kDlStage);
      tma_load_3d(smem + kb * kDlStage + kDlXB, &p.tmap_w, 0, (kb0 + kb) * kTcKB, n0 / 64, &bars[kb]);
    }
  pdl_wait();  // x and v come from the preceding kernels
  pdl_launch_dependents();
  if (warp == 1 && lane == 0) {  // x box + W box per K step of my slice
    for (int kb = 0; kb < pre; ++kb) tma_load_2d(smem + kb * kDlStage, &p.tmap_x, (kb0 + kb) * kTcKB, 0, &bars[kb]);
    for (int kb = pre; kb < nkb; ++kb) {
      const int s = kb % S;
      mbar_wait(&bars[S + s], ((kb / S) - 1) & 1);
      mbar_arrive_expect_tx(&bars[s], kDlStage);
      uint8_t* st = smem + s * kDlStage;
      tma_load_2d(st, &p.tmap_x, (kb0 + kb) * kTcKB, 0, &bars[s]);
      tma_load_3d(st + kDlXB, &p.tmap_w, 0, (kb0 + kb) * kTcKB, n0 / 64, &bars[s]);
    }
  } else if (warp == 0 && lane == 0) {  // MMA issuer
    const uint32_t idesc = umma_idesc(fmt, kTcM, kDlN);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % S;
      mbar_wait(&bars[s], (kb / S) & 1);
      tc_fence_after();
      const uint32_t xa = smem_u32(smem + s * kDlStage), wa = xa + kDlXB;
#pragma unroll
      for (int ks = 0; ks < kTcKB / 16; ++ks) {
        const uint64_t ad = umma_desc(xa + ks * 32, 16, 1024, kSw128);            // x: K-major SW128
        const uint64_t bd = umma_desc(wa + ks * 2 * 1024, 8 * 1024, 1024, kSw128);  // W: MN-major SW128
        umma_f16(tmem, ad, bd, idesc, (kb | ks) ? 1u : 0u);
      }
      umma_commit(&bars[S + s]);
    }
    umma_commit(bar_d);
  }
  __syncwarp();
  cluster_wait();  // peers' barriers initialised
  if (tid == 0) mbar_arrive_expect_tx(bar_recv, static_cast<uint32_t>(kDlKS * kDlRowsPer * kDlN * 4));
  mbar_wait(bar_d, 0);
  tc_fence_after();
#ifdef LSG_DL_ALIAS
  cluster_sync();  // every CTA's MMAs are done: the rings may take the partials
#endif
  // row m of my partial D_c -> owner m / 16 (rows >= 64 are padding: warps 2, 3 send nothing)
#pragma unroll
  for (int cc = 0; cc < kDlN / 16; ++cc) {
    float d[16];
    tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cc * 16, d);  // all threads (aligned)
    const int m = tid;
    if (m < kDlMaxRows) {
      const int owner = m / kDlRowsPer, ml = m - owner * kDlRowsPer;
      const uint32_t ra = mapa_u32(recv + ((c * kDlRowsPer + ml) * kDlN + cc * 16), static_cast<uint32_t>(owner));
      const uint32_t rb = mapa_u32(bar_recv, static_cast<uint32_t>(owner));
#pragma unroll
      for (int j = 0; j < 4; ++j) st_async_v4(ra + j * 16, d[4 * j], d[4 * j + 1], d[4 * j + 2], d[4 * j + 3], rb);
    }
  }
  cp_async_wait<0>();
  mbar_wait(bar_recv, 0);
  __syncthreads();  // every thread's B slices visible
  // my 16 rows x 64 columns: thread -> (row tid / 8, 8 columns)
#pragma unroll
  for (int half = 0; half < kDlN / 64; ++half) {
    const int ml = tid / 8, cg = half * 64 + (tid % 8) * 8, m = c * kDlRowsPer + ml;
    if (m < p.s_n) {
      float acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = 0.f;
#pragma unroll
      for (int src = 0; src < kDlKS; ++src)  // partials in CTA (K slice) order
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += recv[(src * kDlRowsPer + ml) * kDlN + cg + j];
      float lo[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) lo[j] = 0.f;
      if (s_slot[ml] >= 0) {
        const float* vr = p.v + static_cast<int64_t>(m) * R;
#pragma unroll
        for (int k = 0; k < R; ++k) {
          float b[8];
          Cvt<T>::unpack8(*reinterpret_cast<const uint4*>(Bsm + ((ml * R + k) * kDlN + cg) * 2), b);
          const float vk = vr[k];
#pragma unroll
          for (int j = 0; j < 8; ++j) lo[j] = fmaf(vk, b[j], lo[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = acc[j] + lo[j];
      st_global_v4(static_cast<T*>(p.y) + static_cast<int64_t>(m) * p.ldy + n0 + cg, Cvt<T>::pack8(acc));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<kDlN>(tmem);
  }
}

}  // namespace lsg
