// sgmv_dense.cuh --  the dense projection with the LoRA add fused into the
// GEMM, decode shape (s_n <= 64 rows):
//
//   y = x . W + lora_addon(x)        (reference dense_projection, sgmv.cpp:143-155)
//
// Two PDL-chained launches:
//   1. dense_shrink_kernel: v = x . A_seg(row), one CTA per row (fp32, into the workspace). It
//      waits for its predecessor (x) and only THEN lets its dependent launch, so the GEMM below
//      may read x before its own wait.
//   2. dense_lora_kernel: the projection as one GEMM over the concatenated reduction dimension
//
//        y^T[n, m] = sum_k W[k, n] x[m, k]  +  sum_{(s, j)} B_s[j, n] V'[(s, j), m]
//
//      where V'[(s, j), m] = v[m, j] if row m belongs to segment s, else 0: the LoRA expand is a
//      block-diagonal GEMM whose A operand is the stacked adapters' B rows (the weights the expand
//      must read anyway) and whose B operand is the sparse V' tile built from v in shared memory.
//      The whole W GEMM runs BEFORE the kernel's PDL wait (W and x depend on nothing the shrink
//      writes), concurrently with the shrink; only the LoRA blocks at the ring's tail wait for v.
//
// Swapped operands: MMA M = 128 output columns n (W rows of n are contiguous -> A operand
// MN-major, SW128), MMA N = the 64 decode rows (x K-major, SW128), fp32 D in 64 TMEM columns.
// Grid: one cluster of KS CTAs per 128-column tile; CTA c owns the c-th share of the W k-blocks
// and of the LoRA blocks (4 segments x 16 = 64 reduction rows each), streamed through one ring
// of {A 16 KB, B 8 KB} stages: warp 1 issues W (one 3-D TMA copy per stage, both 64-column
// halves) and x (one 64 x 64 box); warps 2-3 fill the LoRA stages (stacked B rows by cp.async,
// L2-prefetched at entry; V' after the wait); warp 0 issues the MMAs in block order.
// The KS partial D tiles are reduced over DSMEM: each TMEM lane (output column n) goes to the
// CTA owning that column slice, which sums the KS partials in CTA order (deterministic),
// rounds once and stores y.
#pragma once

#include "sgmv_stream.cuh"
#include "sgmv_tc.cuh"

namespace lsg {

constexpr int kDnN = 128;         // output columns per cluster (MMA M)
constexpr int kDnMaxRows = 64;    // decode rows per launch (MMA N)
constexpr int kDnKB = 64;         // reduction rows per stage
#ifndef LSG_DN_STAGES
#define LSG_DN_STAGES 3
#endif
constexpr int kDnStages = LSG_DN_STAGES;
constexpr int kDnA = kDnKB * kDnN * 2;        // 16 KB: W / stacked-B tile, two 64-column halves
constexpr int kDnB = kDnKB * kDnMaxRows * 2;  // 8 KB: x / V' tile
constexpr int kDnStage = kDnA + kDnB;
constexpr int kDnRecv = kDnN * kDnMaxRows * 4;  // 32 KB: [src][column slice][64 rows] fp32
constexpr int kDnThreads = 128;
constexpr int kDnLB = 4;  // LoRA blocks resident at once (their own area, outside the W ring)
constexpr int kDnBars = 2 * kDnStages + 2 + 2 * kDnLB;  // full, empty, D, recv, lfull, lempty
constexpr int kDnSmem = (kDnStages + kDnLB) * kDnStage + kDnRecv + kDnBars * 8 + 16 + 1024;
constexpr int kDnMaxKS = 8;
constexpr int kDnShThreads = 256;

// experiment: per-CTA phase stamps (%globaltimer) after v in the workspace
#ifdef LSG_DN_TRACE
#define DN_STAMP(i)                                                                                       \
  do {                                                                                                     \
    uint64_t t_;                                                                                           \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                                \
    reinterpret_cast<uint64_t*>(p.v + kDnMaxRows * 16)[((p.layer & 1) * 220 + blockIdx.y * gridDim.x + blockIdx.x) * 8 + (i)] = t_; \
  } while (0)
#define DN_SSTAMP(i)                                                                                  \
  do {                                                                                                 \
    uint64_t t_;                                                                                       \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                            \
    reinterpret_cast<uint64_t*>(p.v + kDnMaxRows * 16)[((p.layer & 1) * 220 + 148 + blockIdx.x) * 8 + (i)] = t_;            \
  } while (0)
#else
#define DN_STAMP(i) \
  do {              \
  } while (0)
#define DN_SSTAMP(i) \
  do {               \
  } while (0)
#endif

struct DenseLoraParams {
  CUtensorMap tmap_x;  // x [s_n, h_in]: box 64 (k) x 64 rows, SW128
  CUtensorMap tmap_w;  // W [h_in, h_out] as 3-D {64 columns, h_in, h_out / 64}: box {64, 64, 2}, SW128
  void* y;
  int64_t ldy;
  const void* x;
  int64_t ldx;
  float* v;  // [s_n, R] fp32: the shrink's output (workspace)
  const void* const* a_ptr;
  const void* const* b_ptr;
  int64_t a_off, b_off;
  const int32_t* seg_starts;
  const int32_t* seg_slot;
  int32_t n_seg, s_n, num_slots, h_in, h_out, ks;
  int32_t layer;  // trace builds: the trace slot
};

__host__ __device__ constexpr int dn_smem() { return kDnSmem; }

// v[m, :] = x[m, :] . A_seg(m) (fp32), one CTA per row; thread t takes k in [16 t, 16 t + 16)
// (+ 4096 i). The row's A is L2-prefetched before the PDL wait (weights); dependents are released
// right after the wait and not before it (dense_lora_kernel reads x before its own wait).
template <typename T, int R>
__global__ void __launch_bounds__(kDnShThreads) dense_shrink_kernel(const __grid_constant__ DenseLoraParams p) {
  __shared__ float s_red[kDnShThreads / 32][R];
  __shared__ int s_slot;
  const int m = static_cast<int>(blockIdx.x), tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    int lo = 0, hi = p.n_seg;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (p.seg_starts[mid + 1] > m) hi = mid; else lo = mid + 1;
    }
    int slot = lo < p.n_seg ? p.seg_slot[lo] : -1;
    if (slot >= p.num_slots) slot = -1;
    s_slot = slot;
  }
  __syncthreads();
  if (tid == 0) DN_SSTAMP(0);
  const int slot = s_slot;
  float acc[R];
#pragma unroll
  for (int j = 0; j < R; ++j) acc[j] = 0.f;
  const T* A = slot >= 0 ? static_cast<const T*>(p.a_ptr[slot]) + p.a_off : nullptr;
  const T* X = static_cast<const T*>(p.x) + static_cast<int64_t>(m) * p.ldx;
  // Warp 0 waits for the predecessor and releases the GEMM at once (it must not wait behind
  // this kernel's loads); the other warps request their A rows first (weights), then wait.
  if (warp == 0) {
    pdl_wait();
    pdl_launch_dependents();
    if (tid == 0) DN_SSTAMP(1);
  }
  if (A != nullptr)
    for (int k0 = 16 * tid; k0 < p.h_in; k0 += 16 * kDnShThreads) {
      uint4 a[16][2];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        a[i][0] = ldg_nc_v4(A + static_cast<int64_t>(k0 + i) * R);
        a[i][1] = ldg_nc_v4(A + static_cast<int64_t>(k0 + i) * R + 8);
      }
      if (warp != 0 && k0 == 16 * tid) pdl_wait();  // x may come from the predecessor
      float xv[16];
      Cvt<T>::unpack8(*reinterpret_cast<const uint4*>(X + k0), xv);
      Cvt<T>::unpack8(*reinterpret_cast<const uint4*>(X + k0 + 8), xv + 8);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float lo[8], hi[8];
        Cvt<T>::unpack8(a[i][0], lo);
        Cvt<T>::unpack8(a[i][1], hi);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc[j] = fmaf(xv[i], lo[j], acc[j]);
          acc[8 + j] = fmaf(xv[i], hi[j], acc[8 + j]);
        }
      }
    }
  pdl_wait();  // (no-op once waited) v is written below
  if (tid == 0) DN_SSTAMP(2);
#pragma unroll
  for (int j = 0; j < R; ++j)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < R; ++j) s_red[warp][j] = acc[j];
  __syncthreads();
  if (tid < R) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < kDnShThreads / 32; ++w) v += s_red[w][tid];
    p.v[static_cast<int64_t>(m) * R + tid] = v;
  }
  if (tid == 0) DN_SSTAMP(3);
}

template <typename T, int R>
__global__ void __launch_bounds__(kDnThreads, 1) dense_lora_kernel(const __grid_constant__ DenseLoraParams p) {
  static_assert(R == 16, "LoRA blocks hold 64 / R = 4 segments");
  constexpr int fmt = std::is_same<T, __half>::value ? 0 : 1;
  constexpr int S = kDnStages, SEGB = kDnKB / R;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* lora = smem + S * kDnStage;  // kDnLB LoRA stages
  float* recv = reinterpret_cast<float*>(lora + kDnLB * kDnStage);
  uint64_t* bars = reinterpret_cast<uint64_t*>(recv + kDnRecv / 4);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* lfull = bars + 2 * S + 2;
  uint64_t* lempty = lfull + kDnLB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kDnBars);
  __shared__ int s_seg[kDnMaxRows];   // segment of row m (-1: padding row)
  __shared__ int s_slot[kDnMaxRows];  // slot of segment s (-1: none / invalid / empty)
  __shared__ const T* s_bbase[kDnMaxRows];  // segment s's B at this layer and column tile
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int KS = p.ks, c = static_cast<int>(blockIdx.x), tile = static_cast<int>(blockIdx.y);
  const int n0 = tile * kDnN;
  const int nkb = p.h_in / kDnKB, w0 = (c * nkb) / KS, nw = ((c + 1) * nkb) / KS - w0;
#ifdef LSG_DN_NOLORA  // experiment: the W stream alone
  const int nlb = 0,
#else
  const int nlb = (p.n_seg + SEGB - 1) / SEGB,
#endif
            l0 = (c * nlb) / KS, nl = ((c + 1) * nlb) / KS - l0;

  if (tid == 0) {
    DN_STAMP(0);
    for (int i = 0; i < kDnBars; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
    prefetch_tmap(&p.tmap_x);
    prefetch_tmap(&p.tmap_w);
  }
  if (warp == 0) tmem_alloc<kDnMaxRows>(tmem_slot);
  if (tid >= 64) {  // row -> segment, segment -> slot (metadata: before the PDL wait, like every launch)
    const int m = tid - 64;
    int seg = -1;
    if (m < p.s_n) {
      int lo = 0, hi = p.n_seg;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (p.seg_starts[mid + 1] > m) hi = mid; else lo = mid + 1;
      }
      seg = lo < p.n_seg ? lo : -1;
    }
    s_seg[m] = seg;
    if (m < p.n_seg) {
      int slot = p.seg_slot[m];
      if (slot < 0 || slot >= p.num_slots || p.seg_starts[m + 1] <= p.seg_starts[m]) slot = -1;
      s_slot[m] = slot;
      s_bbase[m] = slot >= 0 ? static_cast<const T*>(p.b_ptr[slot]) + p.b_off + n0 : nullptr;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  cluster_arrive_relaxed();  // barrier inits -> the cluster

  if (warp == 1) {  // ------------------------------------------------- TMA producer: W and x
    // (all before the PDL wait: W is a weight, x was complete when the shrink released us)
    if (lane == 0) {
      for (int j = 0; j < nw; ++j) {
        const int s = j % S;
        if (j >= S) mbar_wait(&empty[s], ((j / S) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], kDnStage);
        tma_load_3d(smem + s * kDnStage, &p.tmap_w, 0, (w0 + j) * kDnKB, n0 / 64, &full[s]);
        tma_load_2d(smem + s * kDnStage + kDnA, &p.tmap_x, (w0 + j) * kDnKB, 0, &full[s]);
      }
    }
  } else if (warp >= 2) {  // ------------------------------------ the LoRA blocks (64 threads)
    // Their own area, kDnLB blocks at a time, filled while W streams: the stacked B rows
    // (register staged, two blocks per round; the first round before the PDL wait), V' from
    // the shrink's v after it, one completion per block.
    const int t = tid - 64;
    int seg_m = -1;
    float vv[R];
    for (int c0 = 0; c0 < nl; c0 += kDnLB) {
      const int c1 = min(nl, c0 + kDnLB);
      if (c0 > 0)
        for (int i = 0; i < c1 - c0; ++i) mbar_wait(&lempty[i], ((c0 / kDnLB) - 1) & 1);
      for (int jj = c0; jj < c1; jj += 2) {
        uint4 r[2][16];
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int it = 0; it < 16; ++it) {  // 64 rows (4 segments x 16) x 128 columns
            const int i = t + 64 * it, k2 = i >> 4, h = (i >> 3) & 1, q = i & 7;
            const int seg = (l0 + jj + b) * SEGB + k2 / R;
            const T* bb = jj + b < c1 && seg < p.n_seg ? s_bbase[seg] : nullptr;
            r[b][it] = bb != nullptr ? ldg_nc_v4(bb + static_cast<int64_t>(k2 % R) * p.h_out + h * 64 + q * 8)
                                     : make_uint4(0, 0, 0, 0);
          }
        if (jj == 0) {  // v of my row t (the shrink's output)
          if (t == 0) DN_STAMP(2);
          pdl_wait();
          if (t == 0) DN_STAMP(3);
          seg_m = s_seg[t];
          if (seg_m >= 0 && s_slot[seg_m] < 0) seg_m = -1;
#pragma unroll
          for (int j2 = 0; j2 < R; ++j2) vv[j2] = 0.f;
          if (seg_m >= 0 && seg_m / SEGB >= l0 && seg_m / SEGB < l0 + nl) {
            const float4* vr = reinterpret_cast<const float4*>(p.v + static_cast<int64_t>(t) * R);
#pragma unroll
            for (int k = 0; k < R / 4; ++k) {
              const float4 f = vr[k];
              vv[4 * k] = f.x, vv[4 * k + 1] = f.y, vv[4 * k + 2] = f.z, vv[4 * k + 3] = f.w;
            }
          }
        }
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          if (jj + b >= c1) break;
          uint8_t* st = lora + (jj + b - c0) * kDnStage;
#pragma unroll
          for (int it = 0; it < 16; ++it) {  // SW128 halves: 16-byte chunk q of row k2 at q ^ (k2 & 7)
            const int i = t + 64 * it, k2 = i >> 4, h = (i >> 3) & 1, q = i & 7;
            *reinterpret_cast<uint4*>(st + h * (kDnA / 2) + k2 * 128 + ((q ^ (k2 & 7)) << 4)) = r[b][it];
          }
          // V' row t: v[t, :] at reduction rows (seg - 4 blk) * 16 + [0, 16)
          const int sb = seg_m - (l0 + jj + b) * SEGB;
          const bool mine = seg_m >= 0 && sb >= 0 && sb < SEGB;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            uint4 u = make_uint4(0, 0, 0, 0);
            if (mine && q / 2 == sb) u = Cvt<T>::pack8(vv + (q & 1) * 8);
            *reinterpret_cast<uint4*>(st + kDnA + t * 128 + ((q ^ (t & 7)) << 4)) = u;
          }
        }
        fence_proxy_async_smem();  // generic-proxy writes -> the tensor core's async proxy
        named_barrier_sync(1, 64);
        if (t == 0)
          for (int b = 0; b < 2 && jj + b < c1; ++b) mbar_arrive_local(&lfull[jj + b - c0]);
      }
    }
    if (t == 0) DN_STAMP(4);
  } else if (lane == 0) {  // --------------------------------------------- warp 0: MMA issuer
    // A = W / stacked B (MN-major SW128, two 64-column atoms 8 KB apart), B = x / V' (K-major SW128)
    const uint32_t idesc = (1u << 4) | (static_cast<uint32_t>(fmt) << 7) | (static_cast<uint32_t>(fmt) << 10) |
                           (1u << 15) | (static_cast<uint32_t>(kDnMaxRows >> 3) << 17) |
                           (static_cast<uint32_t>(kDnN >> 4) << 24);
    auto mma_block = [&](uint32_t aa, bool first) {
      const uint32_t ba = aa + kDnA;
#pragma unroll
      for (int ks = 0; ks < kDnKB / 16; ++ks) {
        const uint64_t ad = umma_desc(aa + ks * 2048, kDnA / 2, 1024, kSw128);
        const uint64_t bd = umma_desc(ba + ks * 32, 16, 1024, kSw128);
        umma_f16(tmem, ad, bd, idesc, (first && ks == 0) ? 0u : 1u);
      }
    };
    for (int j = 0; j < nw; ++j) {  // the W ring
      const int s = j % S;
      mbar_wait(&full[s], (j / S) & 1);
      tc_fence_after();
      mma_block(smem_u32(smem + s * kDnStage), j == 0);
      umma_commit(&empty[s]);
    }
    DN_STAMP(5);
    for (int jj = 0; jj < nl; ++jj) {  // then the LoRA blocks
      const int i = jj % kDnLB;
      mbar_wait(&lfull[i], (jj / kDnLB) & 1);
      tc_fence_after();
      mma_block(smem_u32(lora + i * kDnStage), nw == 0 && jj == 0);
      umma_commit(&lempty[i]);
    }
    umma_commit(&bars[2 * S]);
    DN_STAMP(6);
  }
  __syncwarp();
  pdl_wait();  // y is written below
  pdl_launch_dependents();
  cluster_wait();  // peers' barriers initialised
  const int ncs = kDnN / KS;  // columns owned per CTA
  if (tid == 0) mbar_arrive_expect_tx(&bars[2 * S + 1], static_cast<uint32_t>((KS - 1) * ncs * kDnMaxRows * 4));
  // ---- partial D (lane = column n, 64 row columns) -> the owner of column n ----------------
  {
    const int n = tid, owner = n / ncs, nr = c * ncs + (n - owner * ncs);  // row of recv in the owner
    float d[kDnMaxRows];
    if (nw + nl > 0) {
      mbar_wait(&bars[2 * S], 0);
      tc_fence_after();
#pragma unroll
      for (int cc = 0; cc < kDnMaxRows / 16; ++cc)
        tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cc * 16, d + cc * 16);
    } else {
#pragma unroll
      for (int i = 0; i < kDnMaxRows; ++i) d[i] = 0.f;
    }
    const int sw = nr & 15;
    if (owner == c) {
#pragma unroll
      for (int q4 = 0; q4 < kDnMaxRows / 4; ++q4)
        *reinterpret_cast<float4*>(recv + nr * kDnMaxRows + ((q4 ^ sw) << 2)) =
            make_float4(d[4 * q4], d[4 * q4 + 1], d[4 * q4 + 2], d[4 * q4 + 3]);
    } else {
      const uint32_t ra = mapa_u32(recv + nr * kDnMaxRows, static_cast<uint32_t>(owner));
      const uint32_t rb = mapa_u32(&bars[2 * S + 1], static_cast<uint32_t>(owner));
#pragma unroll
      for (int q4 = 0; q4 < kDnMaxRows / 4; ++q4)
        st_async_v4(ra + ((q4 ^ sw) << 4), d[4 * q4], d[4 * q4 + 1], d[4 * q4 + 2], d[4 * q4 + 3], rb);
    }
  }
  mbar_wait(&bars[2 * S + 1], 0);
  __syncthreads();  // local partial rows visible
  // ---- my columns [c * ncs, (c + 1) * ncs): sum the KS partials in CTA order, round, store ---
  for (int item = tid; item < kDnMaxRows * (ncs / 8); item += kDnThreads) {
    const int m = item % kDnMaxRows, g = item / kDnMaxRows;
    if (m >= p.s_n) continue;
    float acc[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int nl_ = g * 8 + jj;
      float a = 0.f;
      for (int src = 0; src < KS; ++src) {
        const int nr = src * ncs + nl_;
        a += recv[nr * kDnMaxRows + (((m >> 2) ^ (nr & 15)) << 2) + (m & 3)];
      }
      acc[jj] = a;
    }
    st_global_v4(static_cast<T*>(p.y) + static_cast<int64_t>(m) * p.ldy + n0 + c * ncs + g * 8, Cvt<T>::pack8(acc));
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<kDnMaxRows>(tmem);
  }
  if (tid == 0) DN_STAMP(7);
}

}  // namespace lsg
