// sgmv_tc3.cuh -- K5 v3: cluster-free tensor-core kernels for long segments (prefill rows),
// ranks 16 / 32 / 64.  Two launches, chained with programmatic dependent launch:
//
//   partials  grid (kparts, tile bound), 128 threads, no cluster.  CTA (ks, t) computes the
//             partial D_ks (TMEM, fp32 128 x R) = x[tile t, K boxes 8ks .. 8ks+7] .
//             A[same boxes]: every x box of its range is requested by TMA at once (128B
//             swizzle), A arrives by cp.async in the UMMA MN-major swizzled layout before the
//             PDL wait, and the partial goes to a global workspace [tile][ks][128][R] fp32
//             (L2-resident: 8 KB per part at rank 16).
//   expand    grid (h_out / 256, tile bound), 128 threads, 2 CTAs per SM.  CTA (j, t) stages
//             y_old (TMA) and its B chunk (cp.async) BEFORE its PDL wait -- the partials
//             kernel triggers its dependents only after its own wait, so every kernel before
//             it has completed and y_old is final -- then sums the tile's partials in ks
//             order, splits v into 16-bit hi + lo, D2 = hi.B + lo.B (TMEM), adds y_old and
//             stores the 128 x 256 tile by TMA (per-row stores on a segment's last tile).
//
// Why: phase traces of the cluster kernels (sgmv_tc_fused_kernel, sgmv_tc2.cuh) showed their
// 8/16-CTA clusters at one CTA per SM coming in several waves (15 co-resident 8-clusters for
// 16 tiles at c4) and a per-tile chain of dependent round trips.  Here the work is ~128
// independent partial CTAs plus ~256 independent expand CTAs; the expand's y_old stream
// overlaps the partials' x stream.
//
// Canonical arithmetic for these rows: v = sum over parts ks (ascending) of the MMA partial
// over boxes [8ks, 8ks + 8) (the part size depends only on the shape);
// y = rn(fp32(hi.B + lo.B) + y_old).
#pragma once

#include "sgmv_tc.cuh"

namespace lsg {

constexpr int kT3BoxesPerPart = 8;  // K boxes of 64 per partial (512 columns of h_in)
constexpr int kT3Threads = 128;

struct Tc3PartParams {
  CUtensorMap tmap_x;  // x [s_n, h_in], box 64 x 128, SW128
  float* ws;           // [tile bound][kparts][128][R] fp32
  const void* const* a_ptr;
  int64_t a_off;
  const int32_t* seg_starts;
  const int32_t* seg_slot;
  int32_t n_seg, s_n, num_slots, h_in, kparts, min_rows;
  unsigned long long* trace;
  int32_t trace_ctas;
};

struct Tc3ExpParams {
  CUtensorMap tmap_y;  // y [s_n, h_out], box 64 x 128, SW128
  void* y;
  int64_t ldy;
  const float* ws;
  const void* const* b_ptr;
  int64_t b_off;
  const int32_t* seg_starts;
  const int32_t* seg_slot;
  int32_t n_seg, s_n, num_slots, h_out, kparts, min_rows;
  unsigned long long* trace;
  int32_t trace_ctas;
};

// partials kernel smem: x boxes (kT3BoxesPerPart x 16 KB), A slice (512 rows x 2R bytes)
template <int R>
struct Tc3PartLayout {
  static constexpr uint32_t kX = 0;
  static constexpr uint32_t kA = kT3BoxesPerPart * kTcBox;
  static constexpr uint32_t kBars = kA + kT3BoxesPerPart * kTcKB * 2 * R;
  static constexpr uint32_t kTotal = kBars + 128 + 1024;  // + alignment slack
};
// expand kernel smem: y staging (4 boxes), B chunk (R x 256, MN-major SW128 atoms), v hi / lo
template <int R>
struct Tc3ExpLayout {
  static constexpr uint32_t kY = 0;
  static constexpr uint32_t kB = 4 * kTcBox;
  static constexpr uint32_t kVhi = kB + R * kTcNT * 2;
  static constexpr uint32_t kVlo = kVhi + kTcM * R * 2;
  static constexpr uint32_t kBars = kVlo + kTcM * R * 2;
  static constexpr uint32_t kTotal = kBars + 64 + 1024;
};

__host__ __device__ inline int tc3_kparts(int h_in) { return (h_in / kTcKB + kT3BoxesPerPart - 1) / kT3BoxesPerPart; }

template <typename T, int R>
__global__ void __launch_bounds__(kT3Threads) sgmv_tc_part_kernel(const __grid_constant__ Tc3PartParams p) {
  static_assert(R == 16 || R == 32 || R == 64, "tensor-core path ranks");
  using L = Tc3PartLayout<R>;
  constexpr int ROWB = 2 * R;
  constexpr uint32_t kSwA = R == 16 ? kSw32 : (R == 32 ? kSw64 : kSw128);
  constexpr int kTmemCols = R < 32 ? 32 : R;
  constexpr int fmt = std::is_same<T, __half>::value ? 0 : 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBars);  // [0, 8) box landed, 8 D ready
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ks = static_cast<int>(blockIdx.x);
  const int nkb = p.h_in / kTcKB, kb0 = ks * kT3BoxesPerPart, nk = min(kT3BoxesPerPart, nkb - kb0);

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
  // CTAs without work leave at once; the first row of the grid still waits for the
  // preceding grid so this grid's completion (and trigger) implies the predecessor's.
  const int slot = s_seg >= 0 ? p.seg_slot[s_seg] : -1;
  if (s_seg < 0 || slot < 0 || slot >= p.num_slots) {
    if (blockIdx.y == 0) {
      pdl_wait();
      pdl_launch_dependents();
    }
    return;
  }
  const int r0 = p.seg_starts[s_seg] + s_tile * kTcM;
  if (tid == 0) {
    for (int i = 0; i < 9; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
    prefetch_tmap(&p.tmap_x);
  }
  if (warp == 0) tmem_alloc<kTmemCols>(tmem_slot);
  {  // A rows [kb0*64, (kb0+nk)*64) -> MN-major swizzled (weights: before the PDL wait)
    const T* A = static_cast<const T*>(p.a_ptr[slot]) + p.a_off + static_cast<int64_t>(kb0) * kTcKB * R;
    constexpr int CPR = ROWB / 16;
    const int total = nk * kTcKB * CPR;
    for (int i = tid; i < total; i += kT3Threads) {
      const int k = i / CPR, c = i - k * CPR;
      cp_async16(smem + L::kA + k * ROWB + ((c ^ swz<ROWB>(k)) * 16), A + static_cast<int64_t>(i) * 8);
    }
    cp_async_commit();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  LSG_TC_TRACE(0, 1);
  pdl_wait();  // x may come from the preceding kernel
  // Dependents (the expand) start now: every kernel before this one has completed, so the
  // expand may stage y_old before its own wait (it waits only for these partials).
  pdl_launch_dependents();
  LSG_TC_TRACE(0, 2);
  if (tid == 0) {  // every x box of the part at once
    for (int b = 0; b < nk; ++b) {
      mbar_arrive_expect_tx(&bars[b], kTcBox);
      tma_load_2d(smem + L::kX + b * kTcBox, &p.tmap_x, (kb0 + b) * kTcKB, r0, &bars[b]);
    }
  }
  cp_async_wait<0>();
  fence_proxy_async_smem();  // A (generic-proxy writes) -> visible to the tensor cores
  __syncthreads();
  if (tid == 32) {  // MMA issuer
    tc_fence_after();
    const uint32_t idesc = umma_idesc(fmt, kTcM, R);
    for (int b = 0; b < nk; ++b) {
      mbar_wait(&bars[b], 0);
      tc_fence_after();
      const uint32_t xa = smem_u32(smem + L::kX + b * kTcBox);
      const uint32_t aa = smem_u32(smem + L::kA) + b * kTcKB * ROWB;
#pragma unroll
      for (int k4 = 0; k4 < kTcKB / 16; ++k4) {
        const uint64_t ad = umma_desc(xa + k4 * 32, 16, 1024, kSw128);           // x: K-major SW128
        const uint64_t bd = umma_desc(aa + k4 * 16 * ROWB, 16, 8 * ROWB, kSwA);  // A: MN-major
        umma_f16(tmem, ad, bd, idesc, (b | k4) ? 1u : 0u);
      }
    }
    umma_commit(&bars[8]);
  }
  __syncwarp();
  mbar_wait(&bars[8], 0);
  LSG_TC_TRACE(0, 3);
  tc_fence_after();
  {  // row m = TMEM lane -> the workspace, R floats per row
    const int m = tid;
    float* dst = p.ws + ((static_cast<int64_t>(blockIdx.y) * p.kparts + ks) * kTcM + m) * R;
#pragma unroll
    for (int c0 = 0; c0 < R; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        *reinterpret_cast<float4*>(dst + c0 + 4 * j) = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
  }
  LSG_TC_TRACE(0, 4);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
  LSG_TC_TRACE(0, 5);
}

template <typename T, int R>
__global__ void __launch_bounds__(kT3Threads) sgmv_tc_exp_kernel(const __grid_constant__ Tc3ExpParams p) {
  static_assert(R == 16 || R == 32 || R == 64, "tensor-core path ranks");
  using L = Tc3ExpLayout<R>;
  constexpr int fmt = std::is_same<T, __half>::value ? 0 : 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = static_cast<int>(blockIdx.x) * kTcNT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBars);  // 0 y landed, 1 D2 ready
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);

  LSG_TC_TRACE(1, 0);
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
  const int slot = s_seg >= 0 ? p.seg_slot[s_seg] : -1;
  if (s_seg < 0 || slot < 0 || slot >= p.num_slots) {
    if (blockIdx.y == 0) {
      pdl_wait();
      pdl_launch_dependents();
    }
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
    // y_old: final before the partials kernel triggered this launch (see the header)
    mbar_arrive_expect_tx(&bars[0], 4 * kTcBox);
#pragma unroll
    for (int b = 0; b < 4; ++b) tma_load_2d(smem + L::kY + b * kTcBox, &p.tmap_y, n0 + b * kTcKB, r0, &bars[0]);
  }
  if (warp == 0) tmem_alloc<kTcNT>(tmem_slot);
  {  // B [R x 256] -> MN-major SW128 atoms: 64-col atom na, k-group kg
    const T* B = static_cast<const T*>(p.b_ptr[slot]) + p.b_off + n0;
    for (int e = tid; e < R * (kTcNT / 8); e += kT3Threads) {
      const int k = e / (kTcNT / 8), cc = e - k * (kTcNT / 8), na = cc / 8, jj = cc % 8;
      cp_async16(smem + L::kB + na * (R / 8) * 1024 + (k / 8) * 1024 + (k % 8) * 128 + ((jj ^ (k % 8)) * 16),
                 B + static_cast<int64_t>(k) * p.h_out + cc * 8);
    }
    cp_async_commit();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  LSG_TC_TRACE(1, 1);
  pdl_wait();  // the partials
  pdl_launch_dependents();
  LSG_TC_TRACE(1, 2);
  {  // v[m] = sum over parts (ascending) -> 16-bit hi + lo, K-major interleave
    const int m = tid;
    const float* src = p.ws + (static_cast<int64_t>(blockIdx.y) * p.kparts * kTcM + m) * R;
#pragma unroll
    for (int kg = 0; kg < R / 8; ++kg) {
      float f[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int q = 0; q < p.kparts; ++q) {
        const float4 a = *reinterpret_cast<const float4*>(src + static_cast<int64_t>(q) * kTcM * R + kg * 8);
        const float4 b = *reinterpret_cast<const float4*>(src + static_cast<int64_t>(q) * kTcM * R + kg * 8 + 4);
        f[0] += a.x, f[1] += a.y, f[2] += a.z, f[3] += a.w, f[4] += b.x, f[5] += b.y, f[6] += b.z, f[7] += b.w;
      }
      float hf[8], lo[8];
      const uint4 hi = Cvt<T>::pack8(f);
      Cvt<T>::unpack8(hi, hf);
#pragma unroll
      for (int j = 0; j < 8; ++j) lo[j] = f[j] - hf[j];
      const uint32_t off = (m / 8) * (R / 8) * 128 + kg * 128 + (m % 8) * 16;
      *reinterpret_cast<uint4*>(smem + L::kVhi + off) = hi;
      *reinterpret_cast<uint4*>(smem + L::kVlo + off) = Cvt<T>::pack8(lo);
    }
  }
  cp_async_wait<0>();
  fence_proxy_async_smem();  // v hi / lo and B (generic-proxy writes) -> the tensor cores
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tc_fence_after();
    const uint32_t idesc = umma_idesc(fmt, kTcM, kTcNT);
    const uint32_t bs = smem_u32(smem + L::kB);
#pragma unroll
    for (int k4 = 0; k4 < R / 16; ++k4) {
      const uint64_t bd = umma_desc(bs + k4 * 2 * 1024, (R / 8) * 1024, 1024, kSw128);  // B: MN-major SW128
      const uint64_t ah = umma_desc(smem_u32(smem + L::kVhi) + k4 * 256, 128, (R / 8) * 128, kSwNone);
      const uint64_t al = umma_desc(smem_u32(smem + L::kVlo) + k4 * 256, 128, (R / 8) * 128, kSwNone);
      umma_f16(tmem, ah, bd, idesc, k4 ? 1u : 0u);
      umma_f16(tmem, al, bd, idesc, 1u);
    }
    umma_commit(&bars[1]);
  }
  __syncwarp();
  mbar_wait(&bars[0], 0);
  mbar_wait(&bars[1], 0);
  LSG_TC_TRACE(1, 3);
  tc_fence_after();
  // ---- epilogue: row m = this thread; y_old from the swizzled staging, in place ----------
  const int m = tid;
  uint8_t* yrow = smem + L::kY + m * 128;  // + box * kTcBox + swizzled 16-byte chunk
#pragma unroll 1
  for (int q = 0; q < kTcNT / 64; ++q) {  // one 64-column box per batch of four TMEM loads
    float acc[64];
    tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + q * 64, acc);
    tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + q * 64 + 16, acc + 16);
    tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + q * 64 + 32, acc + 32);
    tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + q * 64 + 48, acc + 48);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint4* ptr = reinterpret_cast<uint4*>(yrow + q * kTcBox + ((j ^ (m & 7)) * 16));
      float f[8];
      Cvt<T>::unpack8(*ptr, f);
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] = acc[j * 8 + e] + f[e];
      *ptr = Cvt<T>::pack8(f);
    }
  }
  LSG_TC_TRACE(1, 4);
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
