// sgmv_mma.cuh -- K7: segment-tile tensor-core pair for segments whose rows share one
// adapter (ranks 16 / 32 / 64): shared-adapter decode batches (Uniform / Skewed /
// Identical, BASELINE configs[2]) and prefill segments (configs[3]).
//
// A tile is up to 16 rows of one segment -- exactly one m16 block of the warp-level
// tensor-core MMA (mma.sync m16n8k16, fp32 accumulate).  Two launches, chained with
// programmatic dependent launch:
//
//   partials  grid (kparts, tile bound), 128 threads.  CTA (ks, t) computes the partial
//             P_ks[16][R] = x[tile rows, K slice ks] . A[K slice ks, :] over its K slice of
//             KS = h_in / kparts columns, in stages of 64 columns (x 16 x 64 and A 64 x R)
//             moved by 2-D TMA into swizzled shared memory (the hardware swizzle makes the
//             ldmatrix fragment loads conflict-free).  Every stage of the slice is resident
//             at once (the host sizes the split so it fits); the A stages are requested
//             BEFORE the PDL wait and the tile's x rows are prefetched into L2 there.  Warp w
//             takes stages w, w+4, ...; the four warp accumulators are summed in warp order
//             and P_ks goes to the workspace [tile][ks][16][R] fp32 (L2-resident).
//   expand    grid (ncol, tile bound), 128 threads.  CTA (j, t) stages its B column slice
//             (R x NC) and y_old (16 x NC) by TMA before its PDL wait -- the partials kernel
//             triggers its dependents only after its own wait, so every kernel before it has
//             completed and y_old is final -- then bulk-copies the tile's partials, sums them
//             in ks order (v, fp32), splits v into 16-bit hi + lo (hi = rn(v), lo = rn(v -
//             hi)) and runs hi.B and lo.B on the tensor cores (the lo term keeps v's fp32
//             precision), adds y_old in fp32 and rounds once.  Warp w takes stages w, w+4, ...
//             with its own epilogue; stores are 16-byte vectors of the tile's valid rows only.
//
// Adapter weights are addressed through per-slot pointers (a_ptr[slot]), so their TMA
// descriptors are made on the device: the host encodes one template per operand (shape,
// strides, box, swizzle) and every CTA patches the global address of its slot into a copy
// (tensormap.replace in shared memory, then tensormap.cp_fenceproxy to its own 128-byte
// global scratch, fence.proxy.tensormap acquire) before its first weight load.
//
// Why this shape: a shared-adapter segment is weight-bound (h=5120 r=64: 1.25 MiB of A+B
// per segment against 8 rows x 20 KiB of activations), so the weights of one tile are
// spread over kparts x ncol CTAs (about one per SM) instead of one cluster; long prefill
// segments are activation-bound and get many small CTAs per 16-row tile.  The same two
// kernels cover both with different splits (lsg_api.cu: prepare_mma).
//
// Canonical arithmetic for these rows (deterministic; depends only on the shape and the
// split, never on the batch composition): v = sum over parts ks ascending of (sum over warps
// w ascending of the MMA chain over the k16-steps of stages w, w+4, ... of part ks);
// y = rn((fp32(hi.B) + fp32(lo.B)) + y_old).  Within tolerance of the CUDA-core rows, not
// bitwise.
#pragma once

#include "sgmv_device.cuh"
#include "sgmv_tc.cuh"  // TMA helpers, LSG_TC_TRACE

namespace lsg {

constexpr int kMmaM = 16;         // rows per tile (one m16 block)
constexpr int kMmaThreads = 128;  // 4 warps (expand)
#ifndef LSG_MMA_PART_WARPS
#define LSG_MMA_PART_WARPS 4
#endif
constexpr int kMmaPW = LSG_MMA_PART_WARPS;  // partials kernel warps (stages split over them)
constexpr int kMmaKC = 64;        // columns per stage (4 k16-steps)
constexpr int kMmaMaxStagesDecl = 32;  // stages per CTA (all resident; barriers reserved for this many)

struct MmaParams {
  CUtensorMap tmap_x;  // x [s_n, h_in], box 64 x 16, SW128
  CUtensorMap tmap_y;  // y [s_n, h_out], box 64 x 16, SW128
  CUtensorMap tmap_a;  // template: A of one layer [h_in, R], box R x 64, swizzle = R * 2 bytes
  CUtensorMap tmap_b;  // template: B of one layer [R, h_out], box 64 x R, SW128
  void* y;
  int64_t ldy;
  const void* x;  // for the L2 prefetch of the tile's rows
  int64_t ldx;
  const void* const* a_ptr;
  const void* const* b_ptr;
  int64_t a_off;  // layer * a_layer_stride (elements)
  int64_t b_off;
  const int32_t* seg_starts;
  const int32_t* seg_slot;
  float* ws;        // [tile bound][kparts][16][R] fp32 partials
  uint8_t* maps_p;  // 128-byte descriptor scratch per partials CTA
  uint8_t* maps_e;  // ... per expand CTA
  int32_t n_seg, s_n, num_slots, h_in, h_out;
  int32_t kparts;    // K slices (gridDim.x of the partials kernel)
  int32_t pc;        // partials cluster size: pc consecutive K slices sum over DSMEM (kparts / pc partials)
  int32_t ncol;      // column slices (gridDim.x of the expand kernel)
  int32_t min_rows;  // segments with min_rows <= len < max_rows take this path
  int32_t max_rows;
  int32_t fused;     // 1: one launch (sgmv_mma_fused_kernel, clusters of pc = kparts = ncol CTAs)
  unsigned long long* trace;  // phase stamps (instrumented builds only, LSG_TC_TRACE layout)
  int32_t trace_ctas;
};

// ---- warp-level MMA primitives ----------------------------------------------------------
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
template <typename T>
__device__ __forceinline__ void mma16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1);
template <>
__device__ __forceinline__ void mma16816<__half>(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <>
__device__ __forceinline__ void mma16816<__nv_bfloat16>(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// rn(d0 + y[0]), rn(d1 + y[1]) for the two 16-bit values packed in y (fp32 add, one rounding)
template <typename T>
__device__ __forceinline__ uint32_t add2_round(uint32_t y, float d0, float d1);
template <>
__device__ __forceinline__ uint32_t add2_round<__half>(uint32_t y, float d0, float d1) {
  const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&y));
  const __half2 r = __floats2half2_rn(d0 + f.x, d1 + f.y);
  return *reinterpret_cast<const uint32_t*>(&r);
}
template <>
__device__ __forceinline__ uint32_t add2_round<__nv_bfloat16>(uint32_t y, float d0, float d1) {
  const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&y));
  const __nv_bfloat162 r = __floats2bfloat162_rn(d0 + f.x, d1 + f.y);
  return *reinterpret_cast<const uint32_t*>(&r);
}

// ---- device-made TMA descriptors for per-slot weights -------------------------------------
// Warp-wide (tensormap.cp_fenceproxy is .sync.aligned): copy the template `tmpl` (kernel
// parameter) into `smem_map` (128 bytes, 128-aligned), patch its global address, publish it
// to `gmem_map` (this CTA's scratch) with a release fence, then acquire it for the TMA
// proxy.  Returns with `gmem_map` usable by this warp's lane 0.
__device__ __forceinline__ void make_slot_tmap(const CUtensorMap* tmpl, uint8_t* smem_map, uint8_t* gmem_map,
                                               const void* base, int lane) {
  if (lane < 8) reinterpret_cast<uint4*>(smem_map)[lane] = reinterpret_cast<const uint4*>(tmpl)[lane];
  __syncwarp();
  if (lane == 0)
    asm volatile("tensormap.replace.tile.global_address.shared::cta.b1024.b64 [%0], %1;" ::"r"(smem_u32(smem_map)),
                 "l"(reinterpret_cast<uint64_t>(base))
                 : "memory");
  __syncwarp();
  asm volatile(
      "tensormap.cp_fenceproxy.global.shared::cta.tensormap::generic.release.gpu.sync.aligned [%0], [%1], 128;" ::"l"(
          reinterpret_cast<uint64_t>(gmem_map)),
      "r"(smem_u32(smem_map))
      : "memory");
  if (lane == 0)
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(gmem_map))
                 : "memory");
}

// Tile t -> (segment, tile within it) over the segments with min_rows <= len < max_rows,
// 16-row tiles: warp prefix sums over 32 segments per step (all lanes of one warp).
__device__ __forceinline__ void mma_tile_of(const int32_t* seg_starts, int n_seg, int t, int lane, int min_rows,
                                            int max_rows, int& seg, int& tin) {
  int base = 0;
  seg = -1;
  tin = 0;
  for (int c0 = 0; c0 < n_seg && seg < 0; c0 += 32) {
    const int sg = c0 + lane;
    int nt = 0;
    if (sg < n_seg) {
      const int len = seg_starts[sg + 1] - seg_starts[sg];
      nt = (len >= min_rows && len < max_rows) ? (len + kMmaM - 1) / kMmaM : 0;
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

// ---- shared-memory plans (host and device) -----------------------------------------------
// Every stage of a CTA's slice is resident at once (the host picks the K / column splits so
// that it fits): no ring, no refill.  Stage sizes are multiples of 1024 bytes (the 128-byte
// swizzle atom), buffers 1024-aligned.
__host__ __device__ constexpr uint32_t mma_part_stage_bytes(int R) { return kMmaM * kMmaKC * 2 + kMmaKC * R * 2; }
__host__ __device__ constexpr uint32_t mma_exp_stage_bytes(int R) { return R * kMmaKC * 2 + kMmaM * kMmaKC * 2; }
constexpr int kMmaMaxPc = 8;  // partials cluster size (portable)
// partials: [stages][x 2 KB | A 128R B], warp partials kMmaPW x 16 x R fp32, the cluster leader's
// receive buffer pc x 16 x R fp32, map, barriers
__host__ __device__ constexpr uint32_t mma_part_smem(int R, int stages, int pc = kMmaMaxPc) {
  return 1024 + stages * mma_part_stage_bytes(R) + (kMmaPW + pc) * kMmaM * R * 4 + 128 + 8 * (kMmaMaxStagesDecl + 2);
}
// expand: [stages][B 128R B | y 2 KB], the tile's partials kparts x 16 x R fp32, v hi / lo
// (16 x R 16-bit each), map, barriers
__host__ __device__ constexpr uint32_t mma_exp_smem(int R, int stages, int kparts) {
  return 1024 + stages * mma_exp_stage_bytes(R) + kparts * kMmaM * R * 4 + 2 * kMmaM * R * 2 + 128 +
         8 * (kMmaMaxStagesDecl + 2);
}

template <typename T, int R>
__global__ void __launch_bounds__(32 * kMmaPW) sgmv_mma_part_kernel(const __grid_constant__ MmaParams p) {
  static_assert(R == 16 || R == 32 || R == 64, "tensor-core ranks");
  constexpr int ROWB = R * 2;                    // bytes per A row (= its TMA swizzle span)
  constexpr uint32_t kXB = kMmaM * kMmaKC * 2;   // x stage bytes
  constexpr uint32_t kSB = mma_part_stage_bytes(R);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ks = static_cast<int>(blockIdx.x);
  const int KS = p.h_in / p.kparts, nst = KS / kMmaKC;  // nst <= kMmaMaxStages (host)
  const int C = p.pc;
  float* red = reinterpret_cast<float*>(smem + nst * kSB);   // [4][16][R]
  float* recv = red + kMmaPW * kMmaM * R;                    // [C][16][R] (cluster leader)
  uint8_t* smap = reinterpret_cast<uint8_t*>(recv + C * kMmaM * R);  // 128 B
  uint64_t* full = reinterpret_cast<uint64_t*>(smap + 128);  // [nst] stage landed, [nst] partials in
  LSG_TC_TRACE(0, 0);

  __shared__ int s_seg, s_tile;
  if (warp == 0) {
    int seg, tin;
    mma_tile_of(p.seg_starts, p.n_seg, blockIdx.y, lane, p.min_rows, p.max_rows, seg, tin);
    if (lane == 0) {
      s_seg = seg;
      s_tile = tin;
    }
  }
  if (tid == 32) {
    for (int i = 0; i <= nst; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int slot = s_seg >= 0 ? p.seg_slot[s_seg] : -1;
  // CTAs without work leave at once (a whole cluster: its CTAs share the tile); the first row
  // of the grid still waits for the preceding grid (and triggers) so this grid's completion
  // implies the predecessor's.
  if (s_seg < 0 || slot < 0 || slot >= p.num_slots) {
    if (blockIdx.y == 0) {
      pdl_wait();
      pdl_launch_dependents();
    }
    return;
  }
  const uint32_t crank = C > 1 ? cluster_ctarank() : 0u;
  if (C > 1) cluster_arrive_relaxed();  // this CTA's barriers are initialised
  const int r0 = p.seg_starts[s_seg] + s_tile * kMmaM;
  const int rows = min(kMmaM, p.seg_starts[s_seg + 1] - r0);
  const int k0 = ks * KS;
  uint8_t* gmap = p.maps_p + (static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x) * 128;
  const CUtensorMap* amap = reinterpret_cast<const CUtensorMap*>(gmap);
  if (warp == 0) {
    // weights first (before the PDL wait): this slot's A descriptor, then every A stage
    make_slot_tmap(&p.tmap_a, smap, gmap, static_cast<const T*>(p.a_ptr[slot]) + p.a_off, lane);
    if (lane == 0) {
      for (int s = 0; s < nst; ++s) {
        mbar_arrive_expect_tx(&full[s], kSB);
        tma_load_2d(smem + s * kSB + kXB, amap, 0, k0 + s * kMmaKC, &full[s]);
      }
    }
  } else if (warp == 1 && lane < rows) {
    // the tile's x rows into L2 now (a prefetch is only a hint: safe while the preceding
    // kernel still runs), so after the wait they come from L2
    bulk_prefetch_l2(static_cast<const T*>(p.x) + static_cast<int64_t>(r0 + lane) * p.ldx + k0,
                     static_cast<uint32_t>(KS * 2));
  }
  LSG_TC_TRACE(0, 1);
  pdl_wait();  // x may come from the preceding kernel
  // The expand may start now: every kernel before this one has completed, so it may stage
  // y_old (as well as B) before its own wait, which then covers only these partials.
  pdl_launch_dependents();
  LSG_TC_TRACE(0, 2);
  if (tid == 0)
    for (int s = 0; s < nst; ++s) tma_load_2d(smem + s * kSB, &p.tmap_x, k0 + s * kMmaKC, r0, &full[s]);

  // Swapped operands: P^T[R][rows] = A^T . x^T -- the rank is the MMA's M (m16 tiles of A^T
  // by ldmatrix.trans from A's [k][r] rows), the tile's rows its N (n8 tiles from x's rows):
  // a tile of <= 8 rows runs one n8 tile, half the MMAs of a 16-row M.
  constexpr int MT = R / 16;  // m16 tiles of the rank
  const bool two = rows > 8;  // second n8 tile (rows 8..15)
  float acc[MT][2][4];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = acc[i][j][2] = acc[i][j][3] = 0.f;
  // lane's ldmatrix addressing: .trans A^T blocks (k row, r chunk) and x^T blocks (row, k chunk)
  const int ak = (lane & 7) + ((lane >> 4) << 3), ac = (lane >> 3) & 1;
  const int xr = (lane & 7) + ((lane >> 4) << 3), xc = (lane >> 3) & 1;
  // warp w: stages w, w + 4, ... (all four k16-steps of each), no block barrier
  for (int s = warp; s < nst; s += kMmaPW) {
    mbar_wait(&full[s], 0);
    if (s == 0) LSG_TC_TRACE(0, 3);
    const uint32_t xs = smem_u32(smem + s * kSB), as = xs + kXB;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t b[4];  // x^T: {b0, b1} of rows 0..7, {b2, b3} of rows 8..15 (128-byte rows, SW128)
      {
        const int c = 2 * kk + xc;
        ldsm_x4(xs + xr * 128 + ((c ^ (xr & 7)) << 4), b[0], b[1], b[2], b[3]);
      }
#pragma unroll
      for (int i = 0; i < MT; ++i) {  // A^T rows 16i.., k 16kk.. (ROWB-byte rows of A, swizzled)
        const int k = 16 * kk + ak, c = 2 * i + ac;
        uint32_t a[4];
        ldsm_x4_t(as + k * ROWB + ((c ^ swz<ROWB>(k)) << 4), a[0], a[1], a[2], a[3]);
        mma16816<T>(acc[i][0], a, b[0], b[1]);
        if (two) mma16816<T>(acc[i][1], a, b[2], b[3]);
      }
    }
  }
  // ---- sum the four warp accumulators in warp order, write the partial ------------------
  LSG_TC_TRACE(0, 4);
  {  // D^T fragment (r = 16i + g (+8), rows 8j + 2t (+1)) -> red[warp][row][r]
    const int g = lane >> 2, t = lane & 3;
    float* rw = red + warp * kMmaM * R;
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int m0 = 8 * j + 2 * t, r = 16 * i + g;
        rw[m0 * R + r] = acc[i][j][0];
        rw[(m0 + 1) * R + r] = acc[i][j][1];
        rw[m0 * R + r + 8] = acc[i][j][2];
        rw[(m0 + 1) * R + r + 8] = acc[i][j][3];
      }
  }
  __syncthreads();
  // this CTA's partial: the warp sum in warp order.  Clusters of pc K slices: every CTA
  // pushes it into the leader's receive buffer (st.async, completing on the leader's barrier
  // nst), the leader sums the pc partials in rank (= K slice) order and writes one.
  const int nparts = p.kparts / C;
  float* dst = p.ws + (static_cast<int64_t>(blockIdx.y) * nparts + ks / C) * kMmaM * R;
  if (C > 1 && crank == 0 && tid == 0) mbar_arrive_expect_tx(&full[nst], static_cast<uint32_t>((C - 1) * kMmaM * R * 4));
  if (C > 1) cluster_wait();  // the leader's barrier is initialised
  for (int i = tid * 4; i < kMmaM * R; i += 32 * kMmaPW * 4) {
    float4 s4 = *reinterpret_cast<const float4*>(red + i);
#pragma unroll
    for (int w = 1; w < kMmaPW; ++w) {
      const float4 o = *reinterpret_cast<const float4*>(red + w * kMmaM * R + i);
      s4.x += o.x, s4.y += o.y, s4.z += o.z, s4.w += o.w;
    }
    if (C == 1)
      *reinterpret_cast<float4*>(dst + i) = s4;
    else if (crank == 0)
      *reinterpret_cast<float4*>(recv + i) = s4;
    else
      st_async_v4(mapa_u32(recv + crank * kMmaM * R + i, 0u), s4.x, s4.y, s4.z, s4.w, mapa_u32(&full[nst], 0u));
  }
  if (C > 1 && crank == 0) {
    mbar_wait(&full[nst], 0);
    __syncthreads();  // the leader's own partial
    for (int i = tid * 4; i < kMmaM * R; i += 32 * kMmaPW * 4) {
      float4 s4 = *reinterpret_cast<const float4*>(recv + i);
      for (int c = 1; c < C; ++c) {
        const float4 o = *reinterpret_cast<const float4*>(recv + c * kMmaM * R + i);
        s4.x += o.x, s4.y += o.y, s4.z += o.z, s4.w += o.w;
      }
      *reinterpret_cast<float4*>(dst + i) = s4;
    }
  }
  // the expand reads these partials with bulk copies (async proxy)
  asm volatile("fence.proxy.async.global;" ::: "memory");
  LSG_TC_TRACE(0, 5);
}

template <typename T, int R>
__global__ void __launch_bounds__(kMmaThreads) sgmv_mma_exp_kernel(const __grid_constant__ MmaParams p) {
  static_assert(R == 16 || R == 32 || R == 64, "tensor-core ranks");
  constexpr int ROWV = R * 2;               // bytes per v row
  constexpr uint32_t kBB = R * kMmaKC * 2;  // B stage bytes (R rows x 64 columns)
  constexpr uint32_t kSB = mma_exp_stage_bytes(R);
  constexpr uint32_t kPB = kMmaM * R * 4;   // one partial
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NC = p.h_out / p.ncol, nst = NC / kMmaKC;  // nst <= kMmaMaxStages (host)
  const int n0 = static_cast<int>(blockIdx.x) * NC;
  const int nparts = p.kparts / p.pc;                        // partials per tile
  float* part = reinterpret_cast<float*>(smem + nst * kSB);  // [nparts][16][R]
  uint8_t* vhi = smem + nst * kSB + nparts * kPB;
  uint8_t* vlo = vhi + kMmaM * R * 2;
  uint8_t* smap = vlo + kMmaM * R * 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(smap + 128);  // [nst] stages, [nst] partials
  LSG_TC_TRACE(1, 0);

  __shared__ int s_seg, s_tile;
  if (warp == 0) {
    int seg, tin;
    mma_tile_of(p.seg_starts, p.n_seg, blockIdx.y, lane, p.min_rows, p.max_rows, seg, tin);
    if (lane == 0) {
      s_seg = seg;
      s_tile = tin;
    }
  }
  if (tid == 32) {
    for (int i = 0; i <= nst; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int slot = s_seg >= 0 ? p.seg_slot[s_seg] : -1;
  if (s_seg < 0 || slot < 0 || slot >= p.num_slots) {
    if (blockIdx.y == 0) {
      pdl_wait();
      pdl_launch_dependents();
    }
    return;
  }
  const int r0 = p.seg_starts[s_seg] + s_tile * kMmaM;
  const int rows = min(kMmaM, p.seg_starts[s_seg + 1] - r0);
  T* Yg = static_cast<T*>(p.y) + static_cast<int64_t>(r0) * p.ldy + n0;
  uint8_t* gmap = p.maps_e + (static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x) * 128;
  const CUtensorMap* bmap = reinterpret_cast<const CUtensorMap*>(gmap);
  // B and y_old of every stage before the PDL wait (weights are never written by a kernel;
  // y_old is final: the partials kernel triggered this launch only after its own wait)
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_arrive_expect_tx(&full[s], kSB);
      tma_load_2d(smem + s * kSB + kBB, &p.tmap_y, n0 + s * kMmaKC, r0, &full[s]);
    }
  }
  if (warp == 0) {
    make_slot_tmap(&p.tmap_b, smap, gmap, static_cast<const T*>(p.b_ptr[slot]) + p.b_off, lane);
    if (lane == 0)
      for (int s = 0; s < nst; ++s) tma_load_2d(smem + s * kSB, bmap, n0 + s * kMmaKC, 0, &full[s]);
  }
  LSG_TC_TRACE(1, 1);
  pdl_wait();  // the partials (and, through the partials kernel's own wait, y_old)
  pdl_launch_dependents();
  LSG_TC_TRACE(1, 2);
  if (tid == 0) {  // the tile's partials (one bulk copy each, barrier nst)
    const float* src = p.ws + static_cast<int64_t>(blockIdx.y) * nparts * kMmaM * R;
    mbar_arrive_expect_tx(&full[nst], static_cast<uint32_t>(nparts) * kPB);
    for (int q = 0; q < nparts; ++q) bulk_g2s(part + q * kMmaM * R, src + q * kMmaM * R, kPB, &full[nst]);
  }
  mbar_wait(&full[nst], 0);
  {  // v = sum of the partials in ks order -> 16-bit hi + lo, swizzled rows of R values
    for (int i = tid * 8; i < kMmaM * R; i += kMmaThreads * 8) {
      float f[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int q = 0; q < nparts; ++q) {
        const float4 u0 = *reinterpret_cast<const float4*>(part + q * kMmaM * R + i);
        const float4 u1 = *reinterpret_cast<const float4*>(part + q * kMmaM * R + i + 4);
        f[0] += u0.x, f[1] += u0.y, f[2] += u0.z, f[3] += u0.w, f[4] += u1.x, f[5] += u1.y, f[6] += u1.z, f[7] += u1.w;
      }
      float hf[8], lo[8];
      const uint4 hi = Cvt<T>::pack8(f);
      Cvt<T>::unpack8(hi, hf);
#pragma unroll
      for (int e = 0; e < 8; ++e) lo[e] = f[e] - hf[e];
      const int m = i / R, c = (i - m * R) >> 3;
      const uint32_t off = m * ROWV + ((c ^ swz<ROWV>(m)) << 4);
      *reinterpret_cast<uint4*>(vhi + off) = hi;
      *reinterpret_cast<uint4*>(vlo + off) = Cvt<T>::pack8(lo);
    }
  }
  __syncthreads();
  LSG_TC_TRACE(1, 3);
  // Swapped operands: y^T[cols][rows] = B^T . v^T -- the output columns are the MMA's M (m16
  // tiles of B^T by ldmatrix.trans from B's [k][n] rows), the tile's rows its N: a tile of
  // <= 8 rows runs one n8 tile.  v^T fragments (hi and lo) for every k16-step, from v's rows.
  const bool two = rows > 8;
  const int xr = (lane & 7) + ((lane >> 4) << 3), xc = (lane >> 3) & 1;
  const int ak = (lane & 7) + ((lane >> 4) << 3), ac = (lane >> 3) & 1;
  uint32_t vh[R / 16][4], vl[R / 16][4];  // {b0, b1} rows 0..7, {b2, b3} rows 8..15
#pragma unroll
  for (int kk = 0; kk < R / 16; ++kk) {
    const int c = 2 * kk + xc;
    const uint32_t off = xr * ROWV + ((c ^ swz<ROWV>(xr)) << 4);
    ldsm_x4(smem_u32(vhi + off), vh[kk][0], vh[kk][1], vh[kk][2], vh[kk][3]);
    ldsm_x4(smem_u32(vlo + off), vl[kk][0], vl[kk][1], vl[kk][2], vl[kk][3]);
  }
  const int g = lane >> 2, t = lane & 3;
  // warp w: stages w, w + 4, ... -- all 64 columns (4 m16 tiles) of each, its own epilogue
  // and stores, no block barrier
  for (int s = warp; s < nst; s += 4) {
    mbar_wait(&full[s], 0);
    if (s == 0) LSG_TC_TRACE(1, 4);
    uint8_t* bs = smem + s * kSB;
    uint8_t* ys = bs + kBB;
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // columns 16i .. 16i + 15 of the stage (B rows are 128 B, SW128)
      float dh[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      float dl[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int kk = 0; kk < R / 16; ++kk) {
        const int k = 16 * kk + ak, c = 2 * i + ac;
        uint32_t a[4];
        ldsm_x4_t(smem_u32(bs + k * 128 + ((c ^ (k & 7)) << 4)), a[0], a[1], a[2], a[3]);
        mma16816<T>(dh[0], a, vh[kk][0], vh[kk][1]);
        mma16816<T>(dl[0], a, vl[kk][0], vl[kk][1]);
        if (two) {
          mma16816<T>(dh[1], a, vh[kk][2], vh[kk][3]);
          mma16816<T>(dl[1], a, vl[kk][2], vl[kk][3]);
        }
      }
      // epilogue in place: y = rn((hi.B + lo.B) + y_old) for (col 16i + g (+8), row 8j + 2t (+1))
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (j == 1 && !two) break;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int m = 8 * j + 2 * t + (e & 1), col = 16 * i + g + (e >> 1) * 8;
          T* q = reinterpret_cast<T*>(ys + m * 128 + (((col >> 3) ^ (m & 7)) << 4) + (col & 7) * 2);
          *q = Cvt<T>::from_f(dh[j][e] + dl[j][e] + Cvt<T>::to_f(*q));
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int it = 0; it < 4; ++it) {  // 16-byte stores of the valid rows: lane = (row, chunk)
      const int m = it * 4 + (lane >> 3), c = lane & 7;
      if (m < rows)
        st_global_v4(Yg + static_cast<int64_t>(m) * p.ldy + s * kMmaKC + c * 8,
                     *reinterpret_cast<const uint4*>(ys + m * 128 + ((c ^ (m & 7)) << 4)));
    }
  }
  LSG_TC_TRACE(1, 5);
}

// ---- one-launch variant ---------------------------------------------------------------------
// sgmv_mma_fused_kernel: grid (C, tile bound), clusters of C CTAs per tile (C = kparts = pc =
// ncol).  CTA c computes the tile's partial over K slice c exactly like the partials kernel,
// sends it to every CTA of the cluster (DSMEM), sums the C partials in rank order (so every CTA
// holds the same v, with the pair's arithmetic) and expands its column slice c exactly like the
// expand kernel.  One buffer set serves both phases: a stage's B slice and y_old are requested
// into it as soon as the warp that owns the stage has run its shrink MMAs (stages beyond the
// shrink's count at once: B before the PDL wait, y_old after it).
__host__ __device__ constexpr uint32_t mma_fused_smem(int R, int stages, int C) {
  return 1024 + stages * mma_part_stage_bytes(R) + (4 + C) * kMmaM * R * 4 + 2 * kMmaM * R * 2 + 256 +
         8 * (2 * kMmaMaxStagesDecl + 2);
}

template <typename T, int R>
__global__ void __launch_bounds__(kMmaThreads) sgmv_mma_fused_kernel(const __grid_constant__ MmaParams p) {
  static_assert(R == 16 || R == 32 || R == 64, "tensor-core ranks");
  constexpr int ROWB = R * 2;                    // bytes per A row (= its TMA swizzle span) and per v row
  constexpr uint32_t kXB = kMmaM * kMmaKC * 2;   // x / y stage bytes
  constexpr uint32_t kBB = R * kMmaKC * 2;       // A / B stage bytes
  constexpr uint32_t kSB = mma_part_stage_bytes(R);
  static_assert(mma_part_stage_bytes(R) == mma_exp_stage_bytes(R), "one buffer per stage for both phases");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int C = p.pc, crank = static_cast<int>(blockIdx.x);  // cluster dims (C, 1, 1), grid.x == C
  const int KS = p.h_in / C, nk = KS / kMmaKC, NC = p.h_out / C, nn = NC / kMmaKC, nst = nk > nn ? nk : nn;
  float* red = reinterpret_cast<float*>(smem + nst * kSB);  // [4][16][R]
  float* recv = red + 4 * kMmaM * R;                        // [C][16][R]
  uint8_t* vhi = reinterpret_cast<uint8_t*>(recv + C * kMmaM * R);
  uint8_t* vlo = vhi + kMmaM * R * 2;
  uint8_t* smap_a = vlo + kMmaM * R * 2;
  uint8_t* smap_b = smap_a + 128;
  uint64_t* fullk = reinterpret_cast<uint64_t*>(smap_b + 128);  // [nk] shrink stages
  uint64_t* fulln = fullk + kMmaMaxStagesDecl;                   // [nn] expand stages
  uint64_t* rbar = fulln + kMmaMaxStagesDecl;                    // the peers' partials

  __shared__ int s_seg, s_tile;
  if (warp == 0) {
    int seg, tin;
    mma_tile_of(p.seg_starts, p.n_seg, blockIdx.y, lane, p.min_rows, p.max_rows, seg, tin);
    if (lane == 0) {
      s_seg = seg;
      s_tile = tin;
    }
  }
  if (tid == 32) {
    for (int i = 0; i < nk; ++i) mbar_init(&fullk[i], 1);
    for (int i = 0; i < nn; ++i) mbar_init(&fulln[i], 1);
    mbar_init(rbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int slot = s_seg >= 0 ? p.seg_slot[s_seg] : -1;
  if (s_seg < 0 || slot < 0 || slot >= p.num_slots) {  // the whole cluster (one tile) leaves
    if (blockIdx.y == 0) {
      pdl_wait();
      pdl_launch_dependents();
    }
    return;
  }
  cluster_arrive_relaxed();  // this CTA's barriers are initialised
  const int r0 = p.seg_starts[s_seg] + s_tile * kMmaM;
  const int rows = min(kMmaM, p.seg_starts[s_seg + 1] - r0);
  const int k0 = crank * KS, n0 = crank * NC;
  const int64_t cta = static_cast<int64_t>(blockIdx.y) * C + crank;
  uint8_t* gmap_a = p.maps_p + cta * 128;
  uint8_t* gmap_b = p.maps_e + cta * 128;
  const CUtensorMap* amap = reinterpret_cast<const CUtensorMap*>(gmap_a);
  const CUtensorMap* bmap = reinterpret_cast<const CUtensorMap*>(gmap_b);
  T* Yg = static_cast<T*>(p.y) + static_cast<int64_t>(r0) * p.ldy + n0;
  // weights first (before the PDL wait): the A stages, and the B stages that have a buffer of
  // their own (s >= nk)
  if (warp == 0) {
    make_slot_tmap(&p.tmap_a, smap_a, gmap_a, static_cast<const T*>(p.a_ptr[slot]) + p.a_off, lane);
    if (lane == 0)
      for (int s = 0; s < nk; ++s) {
        mbar_arrive_expect_tx(&fullk[s], kSB);
        tma_load_2d(smem + s * kSB + kXB, amap, 0, k0 + s * kMmaKC, &fullk[s]);
      }
  } else if (warp == 1) {
    make_slot_tmap(&p.tmap_b, smap_b, gmap_b, static_cast<const T*>(p.b_ptr[slot]) + p.b_off, lane);
    if (lane == 0)
      for (int s = nk; s < nn; ++s) {
        mbar_arrive_expect_tx(&fulln[s], kSB);
        tma_load_2d(smem + s * kSB, bmap, n0 + s * kMmaKC, 0, &fulln[s]);
      }
  } else if (warp == 2 && lane < rows) {
    bulk_prefetch_l2(static_cast<const T*>(p.x) + static_cast<int64_t>(r0 + lane) * p.ldx + k0,
                     static_cast<uint32_t>(KS * 2));
  }
  pdl_wait();  // x and y_old may come from the preceding kernel
  pdl_launch_dependents();
  __syncthreads();  // warp 1's B descriptor is published
  if (lane == 0) asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(gmap_b) : "memory");
  if (tid == 0) {
    for (int s = 0; s < nk; ++s) tma_load_2d(smem + s * kSB, &p.tmap_x, k0 + s * kMmaKC, r0, &fullk[s]);
    for (int s = nk; s < nn; ++s) tma_load_2d(smem + s * kSB + kBB, &p.tmap_y, n0 + s * kMmaKC, r0, &fulln[s]);
  }

  // ---- shrink: P^T[R][rows] = A^T . x^T over my K slice (the partials kernel's arithmetic) ---
  constexpr int MT = R / 16;
  const bool two = rows > 8;
  {
    float acc[MT][2][4];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = acc[i][j][2] = acc[i][j][3] = 0.f;
    const int ak = (lane & 7) + ((lane >> 4) << 3), ac = (lane >> 3) & 1;
    const int xr = (lane & 7) + ((lane >> 4) << 3), xc = (lane >> 3) & 1;
    for (int s = warp; s < nk; s += 4) {
      mbar_wait(&fullk[s], 0);
      const uint32_t xs = smem_u32(smem + s * kSB), as = xs + kXB;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint32_t b[4];
        {
          const int c = 2 * kk + xc;
          ldsm_x4(xs + xr * 128 + ((c ^ (xr & 7)) << 4), b[0], b[1], b[2], b[3]);
        }
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const int k = 16 * kk + ak, c = 2 * i + ac;
          uint32_t a[4];
          ldsm_x4_t(as + k * ROWB + ((c ^ swz<ROWB>(k)) << 4), a[0], a[1], a[2], a[3]);
          mma16816<T>(acc[i][0], a, b[0], b[1]);
          if (two) mma16816<T>(acc[i][1], a, b[2], b[3]);
        }
      }
      // this warp is done with the buffer: the expand stage s (B, y_old) goes into it
      __syncwarp();
      if (s < nn && lane == 0) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&fulln[s], kSB);
        tma_load_2d(smem + s * kSB, bmap, n0 + s * kMmaKC, 0, &fulln[s]);
        tma_load_2d(smem + s * kSB + kBB, &p.tmap_y, n0 + s * kMmaKC, r0, &fulln[s]);
      }
    }
    const int g = lane >> 2, t = lane & 3;
    float* rw = red + warp * kMmaM * R;
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int m0 = 8 * j + 2 * t, r = 16 * i + g;
        rw[m0 * R + r] = acc[i][j][0];
        rw[(m0 + 1) * R + r] = acc[i][j][1];
        rw[m0 * R + r + 8] = acc[i][j][2];
        rw[(m0 + 1) * R + r + 8] = acc[i][j][3];
      }
  }
  __syncthreads();
  // ---- my partial (warp order) -> every CTA of the cluster; v = the C partials in rank order --
  if (tid == 0) mbar_arrive_expect_tx(rbar, static_cast<uint32_t>((C - 1) * kMmaM * R * 4));
  cluster_wait();  // the peers' barriers are initialised
  for (int i = tid * 4; i < kMmaM * R; i += kMmaThreads * 4) {
    float4 s4 = *reinterpret_cast<const float4*>(red + i);
#pragma unroll
    for (int w = 1; w < 4; ++w) {
      const float4 o = *reinterpret_cast<const float4*>(red + w * kMmaM * R + i);
      s4.x += o.x, s4.y += o.y, s4.z += o.z, s4.w += o.w;
    }
    float* mine = recv + crank * kMmaM * R + i;
    *reinterpret_cast<float4*>(mine) = s4;
    for (int c = 0; c < C; ++c)
      if (c != crank) st_async_v4(mapa_u32(mine, static_cast<uint32_t>(c)), s4.x, s4.y, s4.z, s4.w,
                                  mapa_u32(rbar, static_cast<uint32_t>(c)));
  }
  mbar_wait(rbar, 0);
  __syncthreads();
  for (int i = tid * 8; i < kMmaM * R; i += kMmaThreads * 8) {  // -> 16-bit hi + lo, swizzled rows
    float f[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int c = 0; c < C; ++c) {
      const float4 u0 = *reinterpret_cast<const float4*>(recv + c * kMmaM * R + i);
      const float4 u1 = *reinterpret_cast<const float4*>(recv + c * kMmaM * R + i + 4);
      f[0] += u0.x, f[1] += u0.y, f[2] += u0.z, f[3] += u0.w, f[4] += u1.x, f[5] += u1.y, f[6] += u1.z, f[7] += u1.w;
    }
    float hf[8], lo[8];
    const uint4 hi = Cvt<T>::pack8(f);
    Cvt<T>::unpack8(hi, hf);
#pragma unroll
    for (int e = 0; e < 8; ++e) lo[e] = f[e] - hf[e];
    const int m = i / R, c = (i - m * R) >> 3;
    const uint32_t off = m * ROWB + ((c ^ swz<ROWB>(m)) << 4);
    *reinterpret_cast<uint4*>(vhi + off) = hi;
    *reinterpret_cast<uint4*>(vlo + off) = Cvt<T>::pack8(lo);
  }
  __syncthreads();
  // ---- expand my column slice: y^T = B^T . v^T (hi and lo), + y_old, one rounding ----------
  const int xr = (lane & 7) + ((lane >> 4) << 3), xc = (lane >> 3) & 1;
  const int ak = (lane & 7) + ((lane >> 4) << 3), ac = (lane >> 3) & 1;
  uint32_t vh[R / 16][4], vl[R / 16][4];
#pragma unroll
  for (int kk = 0; kk < R / 16; ++kk) {
    const int c = 2 * kk + xc;
    const uint32_t off = xr * ROWB + ((c ^ swz<ROWB>(xr)) << 4);
    ldsm_x4(smem_u32(vhi + off), vh[kk][0], vh[kk][1], vh[kk][2], vh[kk][3]);
    ldsm_x4(smem_u32(vlo + off), vl[kk][0], vl[kk][1], vl[kk][2], vl[kk][3]);
  }
  const int g = lane >> 2, t = lane & 3;
  for (int s = warp; s < nn; s += 4) {
    mbar_wait(&fulln[s], 0);
    uint8_t* bs = smem + s * kSB;
    uint8_t* ys = bs + kBB;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float dh[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      float dl[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int kk = 0; kk < R / 16; ++kk) {
        const int k = 16 * kk + ak, c = 2 * i + ac;
        uint32_t a[4];
        ldsm_x4_t(smem_u32(bs + k * 128 + ((c ^ (k & 7)) << 4)), a[0], a[1], a[2], a[3]);
        mma16816<T>(dh[0], a, vh[kk][0], vh[kk][1]);
        mma16816<T>(dl[0], a, vl[kk][0], vl[kk][1]);
        if (two) {
          mma16816<T>(dh[1], a, vh[kk][2], vh[kk][3]);
          mma16816<T>(dl[1], a, vl[kk][2], vl[kk][3]);
        }
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (j == 1 && !two) break;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int m = 8 * j + 2 * t + (e & 1), col = 16 * i + g + (e >> 1) * 8;
          T* q = reinterpret_cast<T*>(ys + m * 128 + (((col >> 3) ^ (m & 7)) << 4) + (col & 7) * 2);
          *q = Cvt<T>::from_f(dh[j][e] + dl[j][e] + Cvt<T>::to_f(*q));
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int m = it * 4 + (lane >> 3), c = lane & 7;
      if (m < rows)
        st_global_v4(Yg + static_cast<int64_t>(m) * p.ldy + s * kMmaKC + c * 8,
                     *reinterpret_cast<const uint4*>(ys + m * 128 + ((c ^ (m & 7)) << 4)));
    }
  }
}

}  // namespace lsg
