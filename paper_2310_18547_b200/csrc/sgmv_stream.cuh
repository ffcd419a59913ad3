// sgmv_stream.cuh -- K9: one-pass streaming tensor-core kernel for long (prefill) segments.
//
// One CTA per 16-row tile of a long segment (grid = tile bound).  The tile's whole LoRA
// site runs in one CTA, so no v round trip through global memory and no second launch:
//
//   shrink   v^T[R][16] = A^T . x^T over h_in in stages of KC columns (1024 at rank 16, else
//            512): x as one 1-D bulk copy per row (KC * 2 bytes, rows padded by 16 bytes) and
//            A by 2-D TMA over its 128-byte view rows (SW128)
//   expand   y^T[cols][16] = B^T . (v_hi + v_lo)^T over h_out in stages of KC columns: B
//            (R x 64 boxes, SW128) and y_old (one bulk copy per row); y = rn(D + y_old)
//            written back in place and stored with one 1-D bulk store per row (the
//            segment's rows only)
//
// Warp roles: warp 4 is the producer (builds this slot's A / B descriptors, then keeps a ring
// of S stage slots full: weights are requested before the PDL wait, activations after it),
// warps 0..3 consume -- shrink: a quarter of the k16-steps of every stage (the four warp sums
// added in warp order at the end); expand: a quarter of the 64-column boxes.  Stage slots
// are released through `empty` mbarriers (one arrive per consumer warp), so the x stream of
// the shrink, the weight stream and the y_old / y streams of the expand run back to back
// with no block-wide barrier except the one that turns the warp sums into v.
//
// The operands are swapped (the rank / the output columns are the MMA's M, the tile's rows
// its N), so a tile of <= 8 rows runs one n8 tile; mma.sync m16n8k16 with fp32 accumulation.
// Why a CTA per 16-row tile: prefill segments are activation-bound (h=4096, r=16: 16 KiB of
// x and 32 KiB of y traffic per row against 256 KiB of weights per segment), so the weights
// are re-read per tile from L2 while x / y stream once from HBM; 2048 rows = 128 CTAs.
//
// Canonical arithmetic for these rows: v = (sum over warps w ascending of the MMA chain over
// warp w's k16-steps of every stage, stages ascending); y = rn((fp32(hi.B) + fp32(lo.B)) +
// y_old).  Deterministic; within tolerance of the CUDA-core rows, not bitwise.
#pragma once

#include "sgmv_mma.cuh"

namespace lsg {

// 1-D bulk copy shared -> global (bulk async-group completion)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_group_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void named_barrier_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void mbar_arrive_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_local_cnt(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tmap, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
// phase stamp from any one thread (the producer warp's lane 0 included)
#define LSG_STREAM_TRACE(i)                                                                        \
  do {                                                                                             \
    if (LSG_TC_TRACE_ON) {                                                                         \
      const int cta_ = blockIdx.x;                                                                 \
      if (cta_ < p.trace_ctas / 2) {                                                               \
        unsigned long long gt_;                                                                    \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));                                   \
        p.trace[(p.trace_ctas + cta_) * 16 + (i)] = gt_;                                           \
      }                                                                                            \
    }                                                                                              \
  } while (0)

constexpr int kStreamCW = 8;          // consumer warps
constexpr int kStreamThreads = 32 * (kStreamCW + 1);  // + 1 producer warp
constexpr int kStreamMaxStages = 16;  // ring slots (barriers reserved)
#ifndef LSG_STREAM_SMEM
#define LSG_STREAM_SMEM (220 * 1024)
#endif
// 1: a stage's 16 activation rows (x or y_old) move as ONE 3-D TMA box {64 columns, 16 rows,
// KC / 64 column blocks} (SW128), and a full tile's y as one 3-D box store; 0: one 1-D bulk
// copy per row (padded rows)
#ifndef LSG_STREAM_ABOX
#define LSG_STREAM_ABOX 1
#endif
// L2 prefetch of the tile's activation rows: 0 none; 1 x at entry, y_old too when the grid has
// fewer than kStreamPfYMaxTiles tiles (measured: with y_old c4 14.1 us, 2048-row rank-32 21.6,
// 512-row rank-16 10.7; without it 13.5 / 20.6 / 11.8 -- the extra early traffic pays only while
// the grid leaves SMs idle); 2 x and y_old at entry; 3 y_old once v is ready (c4 14.4); 4 y_old
// after the PDL wait (c4 14.6)
#ifndef LSG_STREAM_PF
#define LSG_STREAM_PF 1
#endif
constexpr unsigned kStreamPfYMaxTiles = 96;
// 1: each consumer warp stores its own 64-column boxes of a full tile (no block barrier per stage)
#ifndef LSG_STREAM_WARP_STORE
#define LSG_STREAM_WARP_STORE 0
#endif
// Rank 16: KC = 512 in a 140 KB ring (four 32 KB slots): the short-segment kernel of the same
// call (70 KB CTAs) then shares the SMs instead of waiting for streaming CTAs to exit
// (c4: 16.2 -> 14.8 us; KC 1024 in 220 KB: three 64 KB slots, one CTA per SM)
#ifndef LSG_STREAM_KC16
#define LSG_STREAM_KC16 512
#endif
#ifndef LSG_STREAM_SMEM16
#define LSG_STREAM_SMEM16 (140 * 1024)
#endif
constexpr int kStreamSmem = LSG_STREAM_SMEM;
__host__ __device__ constexpr int stream_smem_budget(int R) { return R == 16 ? LSG_STREAM_SMEM16 : LSG_STREAM_SMEM; }

// Stage geometry per rank: KC columns per stage (x / y_old rows move as one 1-D bulk copy
// of KC * 2 bytes each -- >= 1 KiB pieces keep HBM streaming at full rate, 128-byte
// tensor-box rows do not: scripts/tma_probe.cu), activation rows padded by 16 bytes so
// ldmatrix is conflict-free, weights (A or B of the stage) first in the slot.
__host__ __device__ constexpr int stream_kc(int R) { return R == 16 ? LSG_STREAM_KC16 : 512; }
// rows of A's 128-byte view per stage, and per TMA box (<= 256)
__host__ __device__ constexpr int stream_a_view_rows(int R) { return stream_kc(R) * R / 64; }
__host__ __device__ constexpr int stream_a_box_rows(int R) { return stream_a_view_rows(R) < 256 ? stream_a_view_rows(R) : 256; }
__host__ __device__ constexpr uint32_t stream_pitch(int R) { return stream_kc(R) * 2 + (LSG_STREAM_ABOX ? 0 : 16); }
__host__ __device__ constexpr uint32_t stream_wbytes(int R) { return stream_kc(R) * R * 2; }
__host__ __device__ constexpr uint32_t stream_slot_bytes(int R) {
  return (stream_wbytes(R) + kMmaM * stream_pitch(R) + 1023u) & ~1023u;
}
__host__ __device__ constexpr uint32_t stream_fixed(int R) {
  return 1024 + kStreamCW * kMmaM * R * 4 + 2 * kMmaM * R * 2 + 256 + 16 * kStreamMaxStages + 16;
}
__host__ __device__ constexpr uint32_t stream_smem(int R, int stages) {
  return stream_fixed(R) + stages * stream_slot_bytes(R);
}

struct StreamParams {
  CUtensorMap tmap_a;  // template: A of one layer viewed as [h_in * R / 64][64], box 64 x 256, SW128
  CUtensorMap tmap_b;  // template: B of one layer as 3-D {64 columns, R rows, h_out / 64 column blocks}
                       // (strides h_out * 2, 128 bytes), box 64 x R x KC/64, SW128: ONE copy per
                       // stage lands the stage's [column block][R][64] layout (the per-stage copy
                       // count, not the bytes, is what L2 weight traffic costs: tma_probe.cu)
  CUtensorMap tmap_x;  // x as 3-D {64 columns, s_n rows, h_in / 64 blocks}, box {64, 16, KC / 64}, SW128
  CUtensorMap tmap_y;  // y likewise over h_out (loads of y_old, stores of full tiles)
  CUtensorMap tmap_y1; // y with a one-block box {64, 16, 1} (per-warp stores, LSG_STREAM_WARP_STORE)
  const void* x;
  void* y;
  int64_t ldx;
  int64_t ldy;
  const void* const* a_ptr;
  const void* const* b_ptr;
  int64_t a_off;  // layer * a_layer_stride (elements)
  int64_t b_off;
  const int32_t* seg_starts;
  const int32_t* seg_slot;
  uint8_t* maps;  // 2 x 128-byte descriptor scratch per CTA
  int32_t n_seg, s_n, num_slots, h_in, h_out;
  int32_t stages;    // ring slots
  int32_t min_rows;  // segments with >= min_rows rows take this kernel
  unsigned long long* trace;
  int32_t trace_ctas;
};

template <typename T, int R>
__global__ void __launch_bounds__(kStreamThreads) sgmv_stream_kernel(const __grid_constant__ StreamParams p) {
  static_assert(R == 16 || R == 32 || R == 64, "tensor-core ranks");
  constexpr int ROWV = R * 2;                 // bytes per v row
  constexpr int KC = stream_kc(R);
  constexpr uint32_t PITCH = stream_pitch(R);
  constexpr uint32_t kWB = stream_wbytes(R);  // weights of a stage (A: KC rows x R, B: R rows x KC)
  constexpr uint32_t kSB = stream_slot_bytes(R);
  constexpr int MT = R / 16;                  // m16 tiles of the rank
  constexpr int KPR = 64 / R;                 // A rows per 128-byte view row
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int S = p.stages;
  float* red = reinterpret_cast<float*>(smem + S * kSB);  // [kStreamCW][16][R]
  uint8_t* vhi = reinterpret_cast<uint8_t*>(red + kStreamCW * kMmaM * R);
  uint8_t* vlo = vhi + kMmaM * R * 2;
  uint8_t* smap = vlo + kMmaM * R * 2;                       // 2 x 128 B
  uint64_t* full = reinterpret_cast<uint64_t*>(smap + 256);  // [S]
  uint64_t* empty = full + kStreamMaxStages;                 // [S]
  uint64_t* bmap_ready = empty + kStreamMaxStages;           // warp 0 built the B descriptor
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nk = p.h_in / KC, nn = p.h_out / KC, nst = nk + nn;
  // Dependents are triggered only after this kernel's own PDL wait (every thread, below): the
  // short-segment kernel of the same call then starts while this one runs and skips its own
  // wait (late_wait), since its rows are disjoint and every kernel before this one is complete.
  if (threadIdx.x == 0) LSG_STREAM_TRACE(0);

  __shared__ int s_seg, s_tile;
  if (warp == 0) {
    int seg, tin;
    mma_tile_of(p.seg_starts, p.n_seg, blockIdx.x, lane, p.min_rows, 0x7fffffff, seg, tin);
    if (lane == 0) {
      s_seg = seg;
      s_tile = tin;
    }
  }
  if (tid == 32) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kStreamCW);
    }
    mbar_init(bmap_ready, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int slot = s_seg >= 0 ? p.seg_slot[s_seg] : -1;
  if (s_seg < 0 || slot < 0 || slot >= p.num_slots) {
    if (blockIdx.x == 0) pdl_wait();  // this grid's completion implies the predecessor's
    return;  // (an exited CTA counts as triggered)
  }
  const int r0 = p.seg_starts[s_seg] + s_tile * kMmaM;
  const int rows = min(kMmaM, p.seg_starts[s_seg + 1] - r0);

  // Rank 16: A's stage rows are one contiguous 1-D copy (linear 32-byte rows: a 2-way ldmatrix
  // conflict, no descriptor to build), so the producer streams weights from its first
  // instruction; the B descriptor is built by warp 0 meanwhile, the activation rows are
  // prefetched into L2 by warp 1 (hints only: safe while the preceding kernel runs).
  constexpr bool kALin = R == 16;
  uint8_t* gmap = p.maps + static_cast<int64_t>(blockIdx.x) * 256;
  if (warp == 0) {
    make_slot_tmap(&p.tmap_b, smap + 128, gmap + 128, static_cast<const T*>(p.b_ptr[slot]) + p.b_off, lane);
    if (lane == 0) mbar_arrive_local(bmap_ready);
  } else if (warp == 1) {
    const T* X = static_cast<const T*>(p.x) + static_cast<int64_t>(r0) * p.ldx;
    const T* Y = static_cast<const T*>(p.y) + static_cast<int64_t>(r0) * p.ldy;
    if (LSG_STREAM_PF >= 1 && lane < rows) bulk_prefetch_l2(X + lane * p.ldx, static_cast<uint32_t>(p.h_in * 2));
    else if ((LSG_STREAM_PF == 2 || (LSG_STREAM_PF == 1 && gridDim.x < kStreamPfYMaxTiles)) && lane >= 16 &&
             lane - 16 < rows)
      bulk_prefetch_l2(Y + (lane - 16) * p.ldy, static_cast<uint32_t>(p.h_out * 2));
  }
  if (warp == kStreamCW) {  // --------------------------------------------------------- producer
    if constexpr (!kALin) make_slot_tmap(&p.tmap_a, smap, gmap, static_cast<const T*>(p.a_ptr[slot]) + p.a_off, lane);
    if (lane == 0) {
      const T* Ag = static_cast<const T*>(p.a_ptr[slot]) + p.a_off;
      const CUtensorMap* amap = reinterpret_cast<const CUtensorMap*>(gmap);
      const CUtensorMap* bmap = reinterpret_cast<const CUtensorMap*>(gmap + 128);
      const T* X = static_cast<const T*>(p.x) + static_cast<int64_t>(r0) * p.ldx;
      const T* Y = static_cast<const T*>(p.y) + static_cast<int64_t>(r0) * p.ldy;
      const uint32_t bytes = kWB + static_cast<uint32_t>(LSG_STREAM_ABOX ? kMmaM : rows) * KC * 2;
      auto weights = [&](int i) {
        uint8_t* sb = smem + (i % S) * kSB;
        if (kALin && i < nk) {  // A rows [i*KC, (i+1)*KC): one contiguous copy
          bulk_g2s(sb, Ag + static_cast<int64_t>(i) * KC * R, KC * R * 2, &full[i % S]);
        } else if (i < nk) {  // A rows [i*KC, (i+1)*KC) = view rows [i*KC/KPR, ...), boxes of ABOX view rows
          constexpr int ABOX = stream_a_box_rows(R);
          for (int b = 0; b < KC / KPR / ABOX; ++b)
            tma_load_2d(sb + b * ABOX * 128, amap, 0, i * (KC / KPR) + b * ABOX, &full[i % S]);
        } else {
          const int n0 = (i - nk) * KC;
          if (i == nk || i < S) {  // the descriptor warp 0 built: acquire it for the TMA proxy
            mbar_wait(bmap_ready, 0);
            asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(bmap))
                         : "memory");
          }
          tma_load_3d(sb, bmap, 0, 0, n0 / 64, &full[i % S]);
        }
      };
      auto acts = [&](int i) {  // x (shrink) or y_old (expand): one bulk copy per row of the tile
        uint8_t* sb = smem + (i % S) * kSB + kWB;
#if LSG_STREAM_ABOX  // one box of 16 rows (rows past the segment are loaded, never stored; past s_n: zeros)
        if (i < nk) tma_load_3d(sb, &p.tmap_x, 0, r0, i * (KC / 64), &full[i % S]);
        else tma_load_3d(sb, &p.tmap_y, 0, r0, (i - nk) * (KC / 64), &full[i % S]);
        return;
#endif
        const T* src = i < nk ? X + i * KC : Y + (i - nk) * KC;
        const int64_t ld = i < nk ? p.ldx : p.ldy;
        for (int m = 0; m < rows; ++m) bulk_g2s(sb + m * PITCH, src + m * ld, KC * 2, &full[i % S]);
      };
      const int pre = min(S, nst);
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], bytes);
        weights(i);
      }
      LSG_STREAM_TRACE(1);
      pdl_wait();  // x and y_old may come from the preceding kernel
      pdl_launch_dependents();
      LSG_STREAM_TRACE(2);
      for (int i = 0; i < pre; ++i) acts(i);
      for (int i = S; i < nst; ++i) {
        mbar_wait(&empty[i % S], ((i / S) - 1) & 1);
        if (i == 3) LSG_STREAM_TRACE(14);
        if (i == 5) LSG_STREAM_TRACE(15);
        mbar_arrive_expect_tx(&full[i % S], bytes);
        weights(i);
        acts(i);
      }
    } else {
      pdl_wait();
      pdl_launch_dependents();
    }
    return;
  }

  // ------------------------------------------------------------------------------ consumers
  pdl_wait();  // (returns at once by the time any y is written)
  pdl_launch_dependents();
  if (LSG_STREAM_PF == 4 && warp == 1 && lane < rows)
    bulk_prefetch_l2(static_cast<const T*>(p.y) + static_cast<int64_t>(r0 + lane) * p.ldy, static_cast<uint32_t>(p.h_out * 2));
  const bool two = rows > 8;  // second n8 tile of the shrink (rows 8..15)
  const int xr = (lane & 7) + ((lane >> 4) << 3), xc = (lane >> 3) & 1;  // row-major 16 x 16 blocks
  const int ak = (lane & 7) + ((lane >> 4) << 3), ac = (lane >> 3) & 1;  // .trans blocks of [k][n] rows
  float acc[MT][2][4];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = acc[i][j][2] = acc[i][j][3] = 0.f;
  constexpr int KPW = KC / 16 / kStreamCW;  // k16-steps per warp per stage
  for (int s = 0; s < nk; ++s) {  // ---- shrink: k16-steps [w * KPW, (w+1) * KPW) of every stage
    mbar_wait(&full[s % S], (s / S) & 1);
    if (s == 0 && tid == 0) LSG_STREAM_TRACE(3);
    if (s < 8 && tid == 0) LSG_STREAM_TRACE(6 + s);
    const uint32_t as = smem_u32(smem + (s % S) * kSB), xs = as + kWB;
#pragma unroll 4
    for (int q = 0; q < KPW; ++q) {
      const int kk = warp * KPW + q;
      uint32_t b[4];  // x^T: {b0, b1} rows 0..7, {b2, b3} rows 8..15 (padded rows)
#if LSG_STREAM_ABOX  // [block][16 rows][64 columns], SW128: chunk q of row xr
      {
        const int q16 = 2 * kk + xc;
        ldsm_x4(xs + (q16 >> 3) * (kMmaM * 128) + xr * 128 + (((q16 & 7) ^ (xr & 7)) << 4), b[0], b[1], b[2], b[3]);
      }
#else
      ldsm_x4(xs + xr * PITCH + (2 * kk + xc) * 16, b[0], b[1], b[2], b[3]);
#endif
#pragma unroll
      for (int i = 0; i < MT; ++i) {  // A^T block (rank 16i.., k 16kk..) from the 128-byte view rows
        uint32_t a[4];
        if constexpr (kALin) {  // linear rows of R
          const int k = 16 * kk + ak;
          ldsm_x4_t(as + k * (R * 2) + (2 * i + ac) * 16, a[0], a[1], a[2], a[3]);
        } else {
          const int k = 16 * kk + ak, c = (k % KPR) * (R / 8) + 2 * i + ac, vq = k / KPR;
          ldsm_x4_t(as + vq * 128 + ((c ^ (vq & 7)) << 4), a[0], a[1], a[2], a[3]);
        }
        mma16816<T>(acc[i][0], a, b[0], b[1]);
        if (two) mma16816<T>(acc[i][1], a, b[2], b[3]);
      }
    }
    // (every lane's ldmatrix reads of the slot have completed: the MMAs that consume them were
    // issued before this point, and __syncwarp orders the warp before lane 0's release)
    __syncwarp();
    if (lane == 0) mbar_arrive_local(&empty[s % S]);
  }
  {  // ---- v = sum of the warp partials in warp order -> 16-bit hi + lo
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
  named_barrier_sync(1, 32 * kStreamCW);
  if (tid == 0) LSG_STREAM_TRACE(4);
  if (LSG_STREAM_PF == 3 && warp == 1 && lane < rows)
    bulk_prefetch_l2(static_cast<const T*>(p.y) + static_cast<int64_t>(r0 + lane) * p.ldy, static_cast<uint32_t>(p.h_out * 2));
  for (int i = tid * 8; i < kMmaM * R; i += 32 * kStreamCW * 8) {
    float f[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      float a = red[i + e];
#pragma unroll
      for (int w = 1; w < kStreamCW; ++w) a += red[w * kMmaM * R + i + e];
      f[e] = a;
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
  named_barrier_sync(1, 32 * kStreamCW);
  // expand, rows as the MMA's M (a 16-row tile fills it): A fragments of v (hi and lo) for
  // every k16-step, B by ldmatrix.trans from the stage's [R][64] boxes; the accumulator
  // pairs (row, 2 adjacent columns) update y_old in place as 32-bit words
  const int lr = (lane & 7) + ((lane >> 3) & 1) * 8, lc = lane >> 4;
  uint32_t ah[R / 16][4], al[R / 16][4];
#pragma unroll
  for (int kk = 0; kk < R / 16; ++kk) {
    const int c = 2 * kk + lc;
    const uint32_t off = lr * ROWV + ((c ^ swz<ROWV>(lr)) << 4);
    ldsm_x4(smem_u32(vhi + off), ah[kk][0], ah[kk][1], ah[kk][2], ah[kk][3]);
    ldsm_x4(smem_u32(vlo + off), al[kk][0], al[kk][1], al[kk][2], al[kk][3]);
  }
  const int g = lane >> 2, t = lane & 3;
  T* Yg = static_cast<T*>(p.y) + static_cast<int64_t>(r0) * p.ldy;
  constexpr int BPW = KC / 64 / kStreamCW;  // 64-column boxes per warp per stage
  for (int j = 0; j < nn; ++j) {  // ---- expand: boxes [w * BPW, (w+1) * BPW) of every stage
    const int s = nk + j;
    mbar_wait(&full[s % S], (s / S) & 1);
    if (s < 8 && tid == 0) LSG_STREAM_TRACE(6 + s);
    uint8_t* bs = smem + (s % S) * kSB;
    uint8_t* ys = bs + kWB;
#pragma unroll
    for (int bi = 0; bi < BPW; ++bi) {
      const int bq = warp * BPW + bi;
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {  // n8 tiles 2jp, 2jp+1 of the box (B rows are 128 B, SW128)
        float d[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        float e2[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int kk = 0; kk < R / 16; ++kk) {
          const int k = 16 * kk + lr, c = 2 * jp + lc;
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(smem_u32(bs + bq * (R * 128) + k * 128 + ((c ^ (k & 7)) << 4)), b0, b1, b2, b3);
          mma16816<T>(d[0], ah[kk], b0, b1);
          mma16816<T>(d[1], ah[kk], b2, b3);
          mma16816<T>(e2[0], al[kk], b0, b1);
          mma16816<T>(e2[1], al[kk], b2, b3);
        }
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          const int col = 64 * bq + 8 * (2 * jp + jj) + 2 * t;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int m = g + 8 * h;
#if LSG_STREAM_ABOX
            uint32_t* q = reinterpret_cast<uint32_t*>(ys + bq * (kMmaM * 128) + m * 128 +
                                                      (((2 * jp + jj) ^ (m & 7)) << 4) + 4 * t);
            (void)col;
#else
            uint32_t* q = reinterpret_cast<uint32_t*>(ys + m * PITCH + col * 2);
#endif
            *q = add2_round<T>(*q, d[jj][2 * h] + e2[jj][2 * h], d[jj][2 * h + 1] + e2[jj][2 * h + 1]);
          }
        }
      }
    }
#if LSG_STREAM_ABOX
#if LSG_STREAM_WARP_STORE
    if (rows == kMmaM) {  // full tile: every warp stores its own 64-column boxes (no block barrier)
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        for (int bi = 0; bi < BPW; ++bi)
          tma_store_3d(&p.tmap_y1, ys + (warp * BPW + bi) * (kMmaM * 128), 0, r0, j * (KC / 64) + warp * BPW + bi);
        bulk_commit_group();
        bulk_wait_group_read<1>();
        if (j > 0) mbar_arrive_local(&empty[(s - 1) % S]);
      }
    } else
#endif
    if (rows == kMmaM) {                      // full tile: ONE 3-D box store of the stage
      fence_proxy_async_smem();               // epilogue writes -> the TMA store
      named_barrier_sync(1, 32 * kStreamCW);  // the stage's y tile is complete
      if (tid == 0) {
        tma_store_3d(&p.tmap_y, ys, 0, r0, j * (KC / 64));
        bulk_commit_group();
        bulk_wait_group_read<1>();            // the previous stage's store has read its slot
        if (j > 0) mbar_arrive_local_cnt(&empty[(s - 1) % S], kStreamCW);
      }
    } else {                                  // last tile of a segment: its rows, de-swizzled
      named_barrier_sync(1, 32 * kStreamCW);
      for (int i = tid; i < rows * (KC / 8); i += 32 * kStreamCW) {
        const int m = i / (KC / 8), q16 = i - m * (KC / 8);
        st_global_v4(Yg + static_cast<int64_t>(m) * p.ldy + j * KC + q16 * 8,
                     *reinterpret_cast<const uint4*>(ys + (q16 >> 3) * (kMmaM * 128) + m * 128 +
                                                     (((q16 & 7) ^ (m & 7)) << 4)));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_local(&empty[s % S]);
    }
  }
#if LSG_STREAM_WARP_STORE
  if (rows == kMmaM && lane == 0) {  // this warp's last stores
    bulk_wait_group_read<0>();
    mbar_arrive_local(&empty[(nst - 1) % S]);
  }
#else
  if (rows == kMmaM && tid == 0) {  // the last stage's store
    bulk_wait_group_read<0>();
    mbar_arrive_local_cnt(&empty[(nst - 1) % S], kStreamCW);
  }
#endif
#else
    fence_proxy_async_smem();                 // epilogue writes -> the bulk stores
    named_barrier_sync(1, 32 * kStreamCW);    // the stage's y tile is complete
    if (lane == 0) {                          // warp w stores rows 2w, 2w + 1 (the segment's rows only)
      for (int m = 2 * warp; m < 2 * warp + 2 && m < rows; ++m)
        bulk_s2g(Yg + static_cast<int64_t>(m) * p.ldy + j * KC, ys + m * PITCH, KC * 2);
      bulk_commit_group();
      // the previous stage's slot is free once its stores have read it (this one stays in flight)
      bulk_wait_group_read<1>();
      if (j > 0) mbar_arrive_local(&empty[(s - 1) % S]);
    }
  }
  if (lane == 0) {  // the last stage's stores
    bulk_wait_group_read<0>();
    mbar_arrive_local(&empty[(nst - 1) % S]);
  }
#endif
  if (tid == 0) LSG_STREAM_TRACE(5);
}

}  // namespace lsg
