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

namespace lsg {

namespace cg = cooperative_groups;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int KW = 128;  // rows of A (h_in elements) per canonical reduction chunk

enum Mode : int { kFused = 0, kShrink = 1, kExpand = 2 };

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
};

struct SmemLayout {
  uint32_t bars, a, x, b, y, p, vpart, v, total;
};

__host__ __device__ inline uint32_t align128(uint32_t v) { return (v + 127u) & ~127u; }

// Identical on host (launch sizing) and device (carve-up).
__host__ __device__ inline SmemLayout make_layout(int mode, int R, int MT, int C, int nqc_max,
                                                  int ncv_max) {
  SmemLayout L;
  uint32_t o = 0;
  const bool sh = mode != kExpand, ex = mode != kShrink;
  L.bars = o;
  o += 128;
  L.a = o;
  if (sh) o = align128(o + nqc_max * KW * R * 2);
  L.x = o;
  if (sh) o = align128(o + MT * nqc_max * KW * 2);
  L.b = o;
  if (ex) o = align128(o + R * ncv_max * 16);
  L.y = o;
  if (ex) o = align128(o + MT * ncv_max * 16);
  L.p = o;
  if (sh) o = align128(o + nqc_max * MT * R * 4);
  L.vpart = o;
  if (sh) o = align128(o + ((MT * R + C - 1) / C) * 4);
  L.v = o;
  o = align128(o + MT * R * 4);
  L.total = o;
  return L;
}

// Balanced split of n items over c owners: owner i holds [i*n/c, (i+1)*n/c).
__device__ __forceinline__ int split_lo(int i, int n, int c) { return (i * n) / c; }
__device__ __forceinline__ int split_owner(int q, int n, int c) { return ((q + 1) * c - 1) / n; }

// Largest rows*R*nq handled by the one-barrier (every-CTA-reduces-everything) form.
constexpr int kRedundantReduceMax = 8192;

// v[o] = sum over chunks q ascending of P_q[o], reading each chunk partial from
// the shared memory of the CTA that owns it.  Owners hold contiguous ascending
// chunk ranges, so walking owners in rank order walks q in order; loads are
// issued in independent batches of 8 and summed strictly in sequence.
template <int MT, int R>
__device__ __forceinline__ float reduce_chunks(const float* P_sm, int o, int nq, int C) {
  cg::cluster_group cluster = cg::this_cluster();
  const int m = o / R, k = o - m * R;
  float s = 0.f;
  for (int r = 0; r < C; ++r) {
    const int n = split_lo(r + 1, nq, C) - split_lo(r, nq, C);
    const float* base = cluster.map_shared_rank(P_sm, r) + m * R + k;
    int ql = 0;
    for (; ql + 8 <= n; ql += 8) {
      float t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) t[u] = base[(ql + u) * MT * R];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += t[u];
    }
    for (; ql < n; ++ql) s += base[ql * MT * R];
  }
  return s;
}

template <typename T, int R, int MT, int MODE>
__global__ void __launch_bounds__(kThreads, 1) sgmv_fast_kernel(const __grid_constant__ FastParams p) {
  static_assert(R == 8 || R == 16 || R == 32 || R == 64, "fast path ranks");
  constexpr int VPR = R / 8;       // 16-byte vectors per A row
  constexpr int RPI = 32 / VPR;    // A rows covered by one warp instruction
  constexpr int ITER = KW / RPI;   // per-lane FMA chain length per chunk
  constexpr bool kSh = MODE != kExpand;
  constexpr bool kEx = MODE != kShrink;

  extern __shared__ __align__(128) uint8_t smem[];
  const int C = static_cast<int>(gridDim.x);
  const int crank = static_cast<int>(blockIdx.x);  // cluster dims (C,1,1), grid.x == C
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const SmemLayout L = make_layout(MODE, R, MT, C, p.nqc_max, p.ncv_max);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);  // 0 A, 1 B, 2 x, 3 y
  T* A_sm = reinterpret_cast<T*>(smem + L.a);
  T* x_sm = reinterpret_cast<T*>(smem + L.x);
  uint4* B_sm = reinterpret_cast<uint4*>(smem + L.b);
  uint4* y_sm = reinterpret_cast<uint4*>(smem + L.y);
  float* P_sm = reinterpret_cast<float*>(smem + L.p);
  float* Vpart_sm = reinterpret_cast<float*>(smem + L.vpart);
  float* V_sm = reinterpret_cast<float*>(smem + L.v);

  // ---- which rows / adapter this cluster serves (uniform across the cluster) ----
  int slot, seg_begin, seg_end, first_tile, tile_step;
  if (p.row_slot != nullptr) {
    const int row = blockIdx.y;
    if (row >= p.s_n) return;
    slot = p.row_slot[row];
    seg_begin = row;
    seg_end = row + 1;
    first_tile = 0;
    tile_step = 1;
  } else {
    const int s = blockIdx.y / p.row_splits;
    if (s >= p.n_seg) return;
    first_tile = blockIdx.y - s * p.row_splits;
    tile_step = p.row_splits;
    seg_begin = p.seg_starts[s];
    seg_end = p.seg_starts[s + 1];
    slot = p.seg_slot[s];
  }
  const int ntiles = (seg_end - seg_begin + MT - 1) / MT;
  if (first_tile >= ntiles) return;
  if (slot < 0 || slot >= p.num_slots) {  // "no adapter": v = 0, y untouched
    if (MODE == kShrink && crank == 0) {
      pdl_wait();
      for (int t = first_tile; t < ntiles; t += tile_step) {
        const int r0 = seg_begin + t * MT, rows = min(MT, seg_end - r0);
        for (int i = tid; i < rows * R; i += kThreads) p.v_out[static_cast<int64_t>(r0) * R + i] = 0.f;
      }
    }
    return;
  }

  const int q0 = split_lo(crank, p.nq, C), nqc = split_lo(crank + 1, p.nq, C) - q0;
  const int cv0 = split_lo(crank, p.ncvt, C), ncv = split_lo(crank + 1, p.ncvt, C) - cv0;
  const int ndl = nqc * KW;  // this CTA's slice of h_in (x_sm row stride)
  const T* A = kSh ? static_cast<const T*>(p.a_ptr[slot]) + p.a_off : nullptr;
  const T* B = kEx ? static_cast<const T*>(p.b_ptr[slot]) + p.b_off : nullptr;

  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // Adapter weights: every byte this CTA will ever need, requested up front.
  if (tid == 0) {
    const uint64_t pol = l2_evict_first_policy();
    if (kSh && nqc > 0) {
      const uint32_t bytes = static_cast<uint32_t>(ndl * R * sizeof(T));
      mbar_arrive_expect_tx(&bars[0], bytes);
      const uint8_t* src = reinterpret_cast<const uint8_t*>(A + static_cast<int64_t>(q0) * KW * R);
      uint8_t* dst = reinterpret_cast<uint8_t*>(A_sm);
      for (uint32_t off = 0; off < bytes; off += 32768u) {
        const uint32_t n = bytes - off < 32768u ? bytes - off : 32768u;
        bulk_g2s_hint(dst + off, src + off, n, &bars[0], pol);
      }
    }
    if (kEx && ncv > 0) {
      mbar_arrive_expect_tx(&bars[1], static_cast<uint32_t>(R * ncv * 16));
      for (int k = 0; k < R; ++k)
        bulk_g2s_hint(B_sm + k * ncv, B + static_cast<int64_t>(k) * p.h_out + cv0 * 8,
                      static_cast<uint32_t>(ncv * 16), &bars[1], pol);
    }
  }
  // x, v and y may be produced by the preceding kernel: wait for it here.
  pdl_wait();
  pdl_launch_dependents();

  uint32_t phase = 0;
  for (int t = first_tile; t < ntiles; t += tile_step, phase ^= 1u) {
    const int r0 = seg_begin + t * MT;
    const int rows = min(MT, seg_end - r0);
    __syncthreads();  // previous tile's x_sm / y_sm / V_sm reads are complete
    if (tid == 0) {
      if (kSh && nqc > 0) {
        mbar_arrive_expect_tx(&bars[2], static_cast<uint32_t>(rows * ndl * sizeof(T)));
        for (int m = 0; m < rows; ++m)
          bulk_g2s(x_sm + m * ndl,
                   static_cast<const T*>(p.x) + static_cast<int64_t>(r0 + m) * p.ldx + q0 * KW,
                   static_cast<uint32_t>(ndl * sizeof(T)), &bars[2]);
      }
      if (kEx && ncv > 0) {
        mbar_arrive_expect_tx(&bars[3], static_cast<uint32_t>(rows * ncv * 16));
        for (int m = 0; m < rows; ++m)
          bulk_g2s(y_sm + m * ncv,
                   static_cast<const T*>(p.y) + static_cast<int64_t>(r0 + m) * p.ldy + cv0 * 8,
                   static_cast<uint32_t>(ncv * 16), &bars[3]);
      }
    }

    if constexpr (MODE == kExpand) {
      for (int i = tid; i < rows * R; i += kThreads)
        V_sm[i] = p.v_in[static_cast<int64_t>(r0) * R + i];
      __syncthreads();
    } else {
      // ---- shrink: per-chunk partials P_q[m, k] ---------------------------------
      if (nqc > 0) {
        mbar_wait(&bars[0], 0);
        mbar_wait(&bars[2], phase);
      }
      const int rowoff = lane / VPR, vec = lane % VPR;
      const uint4* Av = reinterpret_cast<const uint4*>(A_sm);
      for (int ql = warp; ql < nqc; ql += kWarps) {
        float acc[MT][8];
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[m][j] = 0.f;
#pragma unroll 4
        for (int it = 0; it < ITER; ++it) {
          const int dl = ql * KW + it * RPI + rowoff;
          float a[8];
          Cvt<T>::unpack8(Av[dl * VPR + vec], a);
#pragma unroll
          for (int m = 0; m < MT; ++m) {
            if (m < rows) {
              const float xm = Cvt<T>::to_f(x_sm[m * ndl + dl]);
#pragma unroll
              for (int j = 0; j < 8; ++j) acc[m][j] = fmaf(xm, a[j], acc[m][j]);
            }
          }
        }
#pragma unroll
        for (int off = VPR; off < 32; off <<= 1)
#pragma unroll
          for (int m = 0; m < MT; ++m)
            if (m < rows)
#pragma unroll
              for (int j = 0; j < 8; ++j) acc[m][j] += __shfl_xor_sync(0xffffffffu, acc[m][j], off);
        if (lane < VPR) {
#pragma unroll
          for (int m = 0; m < MT; ++m) {
            if (m < rows) {
              float4* dst = reinterpret_cast<float4*>(P_sm + (ql * MT + m) * R + vec * 8);
              dst[0] = make_float4(acc[m][0], acc[m][1], acc[m][2], acc[m][3]);
              dst[1] = make_float4(acc[m][4], acc[m][5], acc[m][6], acc[m][7]);
            }
          }
        }
      }
      // ---- cluster reduction over chunks, ascending q --------------------------
      cluster_sync();  // B1: every CTA's P_sm is visible cluster-wide
      const int no = rows * R;
      if (MODE == kFused && no * p.nq <= kRedundantReduceMax) {
        // Small reductions (decode): every CTA sums all rows*R outputs itself --
        // one cluster barrier fewer than the distributed form, same order.
        for (int o = tid; o < no; o += kThreads) V_sm[o] = reduce_chunks<MT, R>(P_sm, o, p.nq, C);
        cluster_arrive();  // B3 (arrive): done reading remote shared memory
        __syncthreads();
      } else {
        const int o0 = split_lo(crank, no, C), o1 = split_lo(crank + 1, no, C);
        for (int o = o0 + tid; o < o1; o += kThreads) {
          const float s = reduce_chunks<MT, R>(P_sm, o, p.nq, C);
          if constexpr (MODE == kShrink) {
            const int m = o / R;
            p.v_out[static_cast<int64_t>(r0 + m) * R + (o - m * R)] = s;
          } else {
            Vpart_sm[o - o0] = s;
          }
        }
        cluster_sync();  // B2: shares visible (shrink: remote P_sm reads done)
        if constexpr (MODE == kFused) {
          cg::cluster_group cluster = cg::this_cluster();
          for (int o = tid; o < no; o += kThreads) {
            const int owner = split_owner(o, no, C);
            V_sm[o] = cluster.map_shared_rank(Vpart_sm, owner)[o - split_lo(owner, no, C)];
          }
          cluster_arrive();  // B3 (arrive)
          __syncthreads();
        }
      }
    }

    if constexpr (kEx) {
      // ---- expand: y[m, n] += sum_k v[m, k] B[k, n] -----------------------------
      if (ncv > 0) {
        mbar_wait(&bars[1], 0);
        mbar_wait(&bars[3], phase);
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
          st_global_v4(static_cast<T*>(p.y) + static_cast<int64_t>(r0 + m) * p.ldy + (cv0 + cv) * 8,
                       Cvt<T>::pack8(acc));
        }
      }
    }
    if constexpr (MODE == kFused) cluster_wait();  // B3 (wait)
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
