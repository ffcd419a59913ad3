// sgmv_tc.cuh -- K5: tensor-core SGMV for long segments (prefill rows).
//
// Segments with >= kTcMinRows rows are cut into 128-row tiles.  Each tile is
// served by a cluster of C = h_in / 512 CTAs; CTA c owns the 512-wide K chunk c
// of the shrink and the 512-wide column block c of the expand:
//
//   shrink  D1[128 x r] (TMEM, fp32) = x[128 x 512] . A[512 x r]
//           x arrives by TMA (tensor map, 128B swizzle, 4-stage ring), A is
//           re-laid out into the UMMA MN-major swizzled layout; one elected
//           thread issues tcgen05.mma (M=128, N=r, K=16) per 16-wide K step.
//   reduce  D1 is drained (tcgen05.ld) and each row's partial is pushed with
//           st.async to the CTA owning that row; owners sum the C chunk
//           partials in chunk order and push v back to every CTA.
//   expand  v is split into 16-bit hi + lo parts (v = hi + lo to ~22 bits) and
//           D2[128 x 256] = hi . B + lo . B per 256-column block (two blocks,
//           two TMEM buffers); the epilogue drains D2, adds y and stores the
//           segment's rows.
//
// Canonical arithmetic for rows of long segments: v = sum over 512-chunks q
// (ascending) of the MMA partial of chunk q; y = rn(fp32(hi.B + lo.B) + y_old).
// Whether a segment takes this path depends only on its length, so results
// stay independent of batch composition and segment order.
#pragma once

#include <cuda.h>

#include <type_traits>

#include "sgmv_device.cuh"
#include "sgmv_kernels.cuh"

namespace lsg {

constexpr int kTcMinRows = 128;   // segments at least this long use the tensor-core path
constexpr int kTcM = 128;         // rows per tile (UMMA M)
constexpr int kTcKC = 512;        // K chunk per CTA (canonical reduction unit)
constexpr int kTcKB = 64;         // K per TMA box / stage (128 bytes of fp16)
constexpr int kTcStages = 4;      // x ring depth
constexpr int kTcNT = 256;        // expand N tile (UMMA N)
constexpr int kTcThreads = 256;

struct TcParams {
  CUtensorMap tmap_x;  // x [s_n, h_in], box 64 x 128, 128B swizzle
  void* y;
  const void* const* a_ptr;
  const void* const* b_ptr;
  int64_t a_off, b_off, ldy;
  const int32_t* seg_starts;
  const int32_t* seg_slot;
  int32_t n_seg, s_n, num_slots, h_in, h_out;
};

// ---- tcgen05 / UMMA helpers ------------------------------------------------------
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // descriptor version (sm_100)
  d |= static_cast<uint64_t>(layout & 7) << 61;
  return d;
}
// layout codes of the smem descriptor
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

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// 16-byte chunk index XOR of the 32/64/128-byte swizzles for row k
template <int ROWB>
__device__ __forceinline__ int swz(int k) {
  if constexpr (ROWB == 32) return (k >> 2) & 1;
  else if constexpr (ROWB == 64) return (k >> 1) & 3;
  else return k & 7;
}

template <int R>
struct TcLayout {
  static constexpr uint32_t kX = 0;                                   // ring: 4 x 16 KB (1024-aligned)
  static constexpr uint32_t kXStage = kTcM * kTcKB * 2;               // 16 KB
  static constexpr uint32_t kA = kX + kTcStages * kXStage;            // A chunk: 512 rows x 2R bytes
  static constexpr uint32_t kB = kA + kTcKC * R * 2;                  // 2 N tiles of R x 256 (SW128 atoms)
  static constexpr uint32_t kBTile = R * kTcNT * 2;
  static constexpr uint32_t kVhi = kB + 2 * kBTile;                   // v hi/lo: 128 x R, K-major interleave
  static constexpr uint32_t kVlo = kVhi + kTcM * R * 2;
  static constexpr uint32_t kV = kVlo + kTcM * R * 2;                 // fp32 v [128][R]
  static constexpr uint32_t kRecv = kV + kTcM * R * 4;                // [16 chunks][16 rows][R] fp32 partials
  static constexpr uint32_t kBars = kRecv + 16 * 16 * R * 4;
  static constexpr uint32_t kTotal = kBars + 256;
};

// Rows of the tile owned (reduced) by each CTA of the cluster
__device__ __forceinline__ int tc_rows_per_owner(int C) { return (kTcM + C - 1) / C; }

template <typename T, int R>
__global__ void __launch_bounds__(kTcThreads, 1) sgmv_tc_kernel(const __grid_constant__ TcParams p) {
  static_assert(R == 16 || R == 32, "tensor-core path ranks");
  using L = TcLayout<R>;
  constexpr int ROWB = 2 * R;  // bytes per A row (MN-major swizzle width)
  constexpr uint32_t kSwA = R == 16 ? kSw32 : kSw64;
  constexpr int fmt = std::is_same<T, __half>::value ? 0 : 1;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base (128B-swizzle atoms); the launch adds 1 KB of slack
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int C = static_cast<int>(gridDim.x);
  const int crank = static_cast<int>(blockIdx.x);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBars);
  // 0..3 full[s], 4..7 empty[s], 8 d1 ready, 9 partials in, 10 v in, 11 d2 tile 0, 12 d2 tile 1
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kBars + 128);
  float* recv = reinterpret_cast<float*>(smem + L::kRecv);
  float* V = reinterpret_cast<float*>(smem + L::kV);

  pdl_launch_dependents();
  // ---- tile -> (long segment, tile) ------------------------------------------------
  __shared__ int s_seg, s_tile;
  if (warp == 0) {
    const int t = blockIdx.y;
    int base = 0, seg = -1, tin = 0;
    for (int c0 = 0; c0 < p.n_seg && seg < 0; c0 += 32) {
      const int sg = c0 + lane;
      int nt = 0;
      if (sg < p.n_seg) {
        const int len = p.seg_starts[sg + 1] - p.seg_starts[sg];
        nt = len >= kTcMinRows ? (len + kTcM - 1) / kTcM : 0;
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
  if (s_seg < 0) return;
  const int seg_begin = p.seg_starts[s_seg], seg_end = p.seg_starts[s_seg + 1];
  const int slot = p.seg_slot[s_seg];
  if (slot < 0 || slot >= p.num_slots) return;
  const int r0 = seg_begin + s_tile * kTcM;
  const int rows = min(kTcM, seg_end - r0);
  const int k0 = crank * kTcKC;             // this CTA's K chunk
  const int n0 = crank * (p.h_out / C);     // this CTA's column block (2 x 256)
  const int rpo = tc_rows_per_owner(C);

  if (tid == 0) {
    for (int i = 0; i < 13; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap_x)) : "memory");
  }
  if (warp == 0) {  // TMEM: 512 columns (D1 shares buffer 0 with the first D2 tile)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // ---- weights (independent of the preceding kernel): A chunk and B block, laid
  //      out in the UMMA MN-major swizzled form --------------------------------------
  {
    const T* A = static_cast<const T*>(p.a_ptr[slot]) + p.a_off + static_cast<int64_t>(k0) * R;
    uint8_t* As = smem + L::kA;
    constexpr int CPR = ROWB / 16;  // 16-byte chunks per A row
    for (int i = tid; i < kTcKC * CPR; i += kTcThreads) {
      const int k = i / CPR, c = i - k * CPR;
      const uint4 v = *reinterpret_cast<const uint4*>(A + static_cast<int64_t>(k) * R + c * 8);
      *reinterpret_cast<uint4*>(As + k * ROWB + ((c ^ swz<ROWB>(k)) * 16)) = v;
    }
    const T* B = static_cast<const T*>(p.b_ptr[slot]) + p.b_off + n0;
    uint8_t* Bs = smem + L::kB;
    // tile nt, atom na (64 cols), k-group kg: offset nt*kBTile + na*(R/8*1024) + kg*1024 + kk*128 + swz chunk
    for (int i = tid; i < R * (2 * kTcNT / 8); i += kTcThreads) {
      const int k = i / (2 * kTcNT / 8), cc = i - k * (2 * kTcNT / 8);  // cc: 16-byte chunk over 512 cols
      const int nt = cc / (kTcNT / 8), na = (cc % (kTcNT / 8)) / 8, j = cc % 8;
      const uint4 v = *reinterpret_cast<const uint4*>(B + static_cast<int64_t>(k) * p.h_out + cc * 8);
      *reinterpret_cast<uint4*>(Bs + nt * L::kBTile + na * (R / 8) * 1024 + (k / 8) * 1024 + (k % 8) * 128 +
                                ((j ^ (k % 8)) * 16)) = v;
    }
  }
  fence_proxy_async_smem();  // generic smem writes -> visible to the tensor cores
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  cluster_arrive_relaxed();

  pdl_wait();  // x and y may come from the preceding kernel

  const uint32_t idesc1 = umma_idesc(fmt, kTcM, R);
  const uint32_t idesc2 = umma_idesc(fmt, kTcM, kTcNT);
  // ---- shrink: TMA producer (warp 1) / MMA issuer (warp 0) ---------------------------
  constexpr int nkb = kTcKC / kTcKB;  // 8 K blocks per chunk
  if (warp == 1 && lane == 0) {
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kTcStages;
      if (kb >= kTcStages) mbar_wait(&bars[4 + s], ((kb / kTcStages) - 1) & 1);
      mbar_arrive_expect_tx(&bars[s], L::kXStage);
      tma_load_2d(smem + L::kX + s * L::kXStage, &p.tmap_x, k0 + kb * kTcKB, r0, &bars[s]);
    }
  } else if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kTcStages;
      mbar_wait(&bars[s], (kb / kTcStages) & 1);
      tc_fence_after();
      const uint32_t xs = smem_u32(smem + L::kX + s * L::kXStage);
      const uint32_t as = smem_u32(smem + L::kA) + kb * kTcKB * ROWB;
#pragma unroll
      for (int ks = 0; ks < kTcKB / 16; ++ks) {
        const uint64_t ad = umma_desc(xs + ks * 32, 16, 1024, kSw128);                 // x: K-major SW128
        const uint64_t bd = umma_desc(as + ks * 16 * ROWB, 16, 8 * ROWB, kSwA);        // A: MN-major
        umma_f16(tmem, ad, bd, idesc1, (kb | ks) ? 1u : 0u);
      }
      umma_commit(&bars[4 + s]);  // stage free once these MMAs have read it
    }
    umma_commit(&bars[8]);        // D1 complete
  }
  __syncwarp();  // producer / issuer lanes rejoin their warps before .aligned ops
  // ---- reduce: drain D1, push row partials to their owners ----------------------------
  cluster_wait();  // peers' barriers initialised
  const int my_rows = max(0, min(rpo, kTcM - crank * rpo));
  if (tid == 0) {
    mbar_arrive_expect_tx(&bars[9], static_cast<uint32_t>(C * my_rows * R * 4));
    mbar_arrive_expect_tx(&bars[10], static_cast<uint32_t>(kTcM * R * 4));
  }
  if (warp < 4) {
    mbar_wait(&bars[8], 0);
    tc_fence_after();
    const int m = warp * 32 + lane;
    const int owner = m / rpo, ml = m - owner * rpo;
    for (int c0 = 0; c0 < R; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
      const uint32_t ra = mapa_u32(recv + (crank * rpo + ml) * R + c0, static_cast<uint32_t>(owner));
      const uint32_t rb = mapa_u32(&bars[9], static_cast<uint32_t>(owner));
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) st_async_v4(ra + q4 * 16, v[4 * q4], v[4 * q4 + 1], v[4 * q4 + 2], v[4 * q4 + 3], rb);
    }
  }
  // owners: v[m][k] = sum over chunks (CTAs) in rank order, then broadcast to all CTAs
  mbar_wait(&bars[9], 0);
  for (int i = tid; i < my_rows * R; i += kTcThreads) {
    const int ml = i / R, k = i - ml * R;
    float s = 0.f;
    for (int q = 0; q < C; ++q) s += recv[(q * rpo + ml) * R + k];
    const uint32_t local = smem_u32(V + (crank * rpo + ml) * R + k), lbar = smem_u32(&bars[10]);
    for (int dst = 0; dst < C; ++dst) {
      uint32_t ra, rb;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local), "r"(dst));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lbar), "r"(dst));
      st_async_f32(ra, s, rb);
    }
  }
  mbar_wait(&bars[10], 0);
  // v -> 16-bit hi + lo, K-major interleave: (m,k) at (m/8)*SBO + (k/8)*128 + (m%8)*16 + (k%8)*2
  for (int i = tid; i < kTcM * (R / 8); i += kTcThreads) {
    const int m = i / (R / 8), kg = i - m * (R / 8);
    float f[8], lo[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = V[m * R + kg * 8 + j];
    const uint4 hi = Cvt<T>::pack8(f);
    float hf[8];
    Cvt<T>::unpack8(hi, hf);
#pragma unroll
    for (int j = 0; j < 8; ++j) lo[j] = f[j] - hf[j];
    const uint32_t off = (m / 8) * (R / 8) * 128 + kg * 128 + (m % 8) * 16;
    *reinterpret_cast<uint4*>(smem + L::kVhi + off) = hi;
    *reinterpret_cast<uint4*>(smem + L::kVlo + off) = Cvt<T>::pack8(lo);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  // ---- expand: two 256-column tiles, one TMEM buffer each ------------------------------
  if (warp == 0 && lane == 0) {
    tc_fence_after();
    for (int nt = 0; nt < 2; ++nt) {
      const uint32_t d2 = tmem + nt * kTcNT;
      const uint32_t bs = smem_u32(smem + L::kB) + nt * L::kBTile;
#pragma unroll
      for (int ks = 0; ks < R / 16; ++ks) {
        const uint64_t bd = umma_desc(bs + ks * 2 * 1024, (R / 8) * 1024, 1024, kSw128);  // B: MN-major SW128
        const uint64_t ah = umma_desc(smem_u32(smem + L::kVhi) + ks * 256, 128, (R / 8) * 128, kSwNone);
        const uint64_t al = umma_desc(smem_u32(smem + L::kVlo) + ks * 256, 128, (R / 8) * 128, kSwNone);
        umma_f16(d2, ah, bd, idesc2, ks ? 1u : 0u);
        umma_f16(d2, al, bd, idesc2, 1u);
      }
      umma_commit(&bars[11 + nt]);
    }
  }
  __syncwarp();
  // ---- epilogue: y[r0+m, n0 + nt*256 + c] = rn(D2 + y_old), rows of this segment only --
  {
    const int m = (warp & 3) * 32 + lane;
    const int half = warp >> 2;  // warps 4..7 take the upper 128 columns of each tile
    for (int nt = 0; nt < 2; ++nt) {
      mbar_wait(&bars[11 + nt], 0);
      tc_fence_after();
      for (int c0 = half * 128; c0 < half * 128 + 128; c0 += 16) {
        float acc[16];
        tmem_ld16(tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + nt * kTcNT + c0, acc);
        if (m < rows) {
          T* yp = static_cast<T*>(p.y) + static_cast<int64_t>(r0 + m) * p.ldy + n0 + nt * kTcNT + c0;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float yo[8];
            Cvt<T>::unpack8(*reinterpret_cast<const uint4*>(yp + h * 8), yo);
#pragma unroll
            for (int j = 0; j < 8; ++j) yo[j] = acc[h * 8 + j] + yo[j];
            st_global_v4(yp + h * 8, Cvt<T>::pack8(yo));
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace lsg
