// sgmv_tc2.cuh -- K5 v2: the streamed, warp-specialised tensor-core kernel for long
// segments (prefill rows), ranks 16 and 32.
//
// One launch serves every 128-row tile of every segment with >= min_rows rows.  A
// cluster of C CTAs (C = 8 or 16, chosen from the shape only) owns one tile at a
// time and loops over tiles (persistent grid sized by cudaOccupancyMaxActiveClusters):
//
//   CTA c of the cluster
//     shrink   D1 (TMEM, fp32 128 x R) = x[tile, K boxes of c] . A[K boxes of c]:
//              x by TMA through a ring of 64-column boxes (128B swizzle), every box
//              of the CTA's K slice requested at once; A by cp.async into the UMMA
//              MN-major swizzled layout, issued ahead of the PDL wait;
//     reduce   row partials -> row owners (st.async DSMEM), owners add the C partials
//              in CTA order and broadcast their rows of v to the cluster (v never
//              leaves the chip);
//     expand   its (at most two) 256-column chunks j = c, c + C: D2_j (TMEM columns
//              [256 j', 256 j' + 256)) = hi.B_j + lo.B_j (v split into 16-bit hi + lo,
//              fp32-level precision), both chunks issued back to back;
//     epilogue 8 warps: warp w reads TMEM lanes 32 (w % 4) .. +32, column half w / 4,
//              adds y_old (chunk 0 staged by TMA at the tile's start, chunk 1 staged
//              into the x ring as soon as the shrink has consumed it) and stores the
//              tile by TMA (per-row stores on a segment's last, partial tile).
//
// What it changes against the first fused kernel (sgmv_tc_fused_kernel), measured on
// c4 by phase traces: that kernel ran ~10 us per tile as a chain of dependent memory
// round trips (weights by ldg -> st.shared, x ring of 4, y staging, 128-thread
// epilogue), and its 16-CTA clusters came in two waves.  Here every load of a tile is
// in flight at once, weights are asynchronous copies, the epilogue has twice the
// threads with batched TMEM loads, and the grid never exceeds the co-resident clusters.
//
// Canonical arithmetic for these rows: v = sum over CTAs c (ascending) of the MMA
// partial over c's K boxes (C and the box split depend only on the shape);
// y = rn(fp32(hi.B + lo.B) + y_old).
#pragma once

#include "sgmv_tc.cuh"

namespace lsg {

constexpr int kT2Threads = 256;
constexpr int kT2MaxStages = 6;

struct Tc2Params {
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
  int32_t kbs_max;  // max K boxes per CTA
  int32_t chs_max;  // max 256-column expand chunks per CTA (1 or 2)
  int32_t stages;   // x ring depth (>= 4 when chs_max == 2: the ring stages y chunk 1)
  int32_t min_rows;
  int32_t tiles;    // upper bound on the long-segment tiles (the persistent loop's end)
  unsigned long long* trace;
  int32_t trace_ctas;
};

struct Tc2Layout {
  uint32_t ring, y0, a, b, vhi, vlo, recv, vfull, bars, total;
};
__host__ __device__ inline Tc2Layout tc2_layout(int R, int kbs_max, int chs_max, int stages) {
  Tc2Layout L{};
  L.ring = 0;
  L.y0 = static_cast<uint32_t>(stages) * kTcBox;
  L.a = L.y0 + 4 * kTcBox;
  L.b = L.a + static_cast<uint32_t>(kbs_max * kTcKB * 2 * R);
  L.b = (L.b + 1023u) & ~1023u;
  L.vhi = L.b + static_cast<uint32_t>(chs_max * R * kTcNT * 2);
  L.vlo = L.vhi + kTcM * R * 2;
  L.recv = L.vlo + kTcM * R * 2;
  L.vfull = L.recv + kTcM * R * 4;
  L.bars = L.vfull + kTcM * R * 4;
  L.total = L.bars + 256 + 1024;  // + alignment slack
  return L;
}

__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 32 lanes x 64 consecutive TMEM columns (four x16 loads, one wait)
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float* v) {
  uint32_t r[64];
#pragma unroll
  for (int q = 0; q < 4; ++q)
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(r[16 * q + 0]), "=r"(r[16 * q + 1]), "=r"(r[16 * q + 2]), "=r"(r[16 * q + 3]), "=r"(r[16 * q + 4]),
          "=r"(r[16 * q + 5]), "=r"(r[16 * q + 6]), "=r"(r[16 * q + 7]), "=r"(r[16 * q + 8]), "=r"(r[16 * q + 9]),
          "=r"(r[16 * q + 10]), "=r"(r[16 * q + 11]), "=r"(r[16 * q + 12]), "=r"(r[16 * q + 13]),
          "=r"(r[16 * q + 14]), "=r"(r[16 * q + 15])
        : "r"(taddr + 16 * q));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}

// barrier slots
constexpr int kB2Full = 0, kB2Empty = 8, kB2W = 16, kB2D1 = 17, kB2Recv = 18, kB2Vfull = 19, kB2Y0 = 20,
              kB2Y1 = 21, kB2E0 = 22, kB2E1 = 23;

template <typename T, int R>
__global__ void __launch_bounds__(kT2Threads, 1) sgmv_tc_stream_kernel(const __grid_constant__ Tc2Params p) {
  static_assert(R == 16 || R == 32, "streamed tensor-core kernel ranks");
  constexpr int ROWB = 2 * R;  // bytes per A row (MN-major swizzle width)
  constexpr uint32_t kSwA = R == 16 ? kSw32 : kSw64;
  constexpr int fmt = std::is_same<T, __half>::value ? 0 : 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const Tc2Layout L = tc2_layout(R, p.kbs_max, p.chs_max, p.stages);
  const int C = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int S = p.stages;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);
  float* recv = reinterpret_cast<float*>(smem + L.recv);
  float* vfull = reinterpret_cast<float*>(smem + L.vfull);
  const int nkb = p.h_in / kTcKB, kb0 = (c * nkb) / C, nk = ((c + 1) * nkb) / C - kb0;
  const int nch = p.h_out / kTcNT, nmine = c < nch ? (nch - 1 - c) / C + 1 : 0;  // <= chs_max
  const int rpo = kTcM / C;  // rows each CTA owns in the reduction

  LSG_TC_TRACE(0, 0);
  pdl_launch_dependents();  // the next kernel only stages its weights before its own wait
  if (tid == 0) {
    for (int i = 0; i < 24; ++i) mbar_init(&bars[i], i == kB2W ? kT2Threads : 1);
    fence_mbar_init();
    prefetch_tmap(&p.tmap_x);
    prefetch_tmap(&p.tmap_y);
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  __shared__ int s_seg, s_tile;
  int it = 0;     // tiles this CTA has processed (barrier parities)
  int gbox = 0;   // x boxes issued so far (ring stage / parity)
  for (int tile = blockIdx.y; tile < p.tiles; tile += gridDim.y) {
    if (it > 0) cluster_sync();  // every CTA done with the previous tile's exchange buffers
    else __syncthreads();        // s_seg / s_tile of a skipped tile consumed
    if (warp == 0) {
      int seg, tin;
      tc_tile_of(p.seg_starts, p.n_seg, tile, lane, seg, tin, p.min_rows);
      if (lane == 0) {
        s_seg = seg;
        s_tile = tin;
      }
    }
    __syncthreads();
    const int seg = s_seg;
    if (seg < 0) break;  // past the last tile (the bound is an upper bound)
    const int slot = p.seg_slot[seg];
    if (slot < 0 || slot >= p.num_slots) continue;  // no adapter: rows untouched
    const int seg_end = p.seg_starts[seg + 1];
    const int r0 = p.seg_starts[seg] + s_tile * kTcM;
    const int rows = min(kTcM, seg_end - r0);
    const uint32_t ph = static_cast<uint32_t>(it & 1);

    // ---- weights (independent of the preceding kernel): cp.async into UMMA layouts ----
    {  // A rows [kb0*64, (kb0+nk)*64) -> MN-major, row k at k*ROWB, 16-byte chunk cc ^ swz(k)
      const T* A = static_cast<const T*>(p.a_ptr[slot]) + p.a_off + static_cast<int64_t>(kb0) * kTcKB * R;
      constexpr int CPR = ROWB / 16;
      const int total = nk * kTcKB * CPR;
      for (int i = tid; i < total; i += kT2Threads) {
        const int k = i / CPR, cc = i - k * CPR;
        cp_async16(smem + L.a + k * ROWB + ((cc ^ swz<ROWB>(k)) * 16), A + static_cast<int64_t>(i) * 8);
      }
    }
    for (int i = 0; i < nmine; ++i) {  // B chunk -> MN-major SW128 atoms
      const T* B = static_cast<const T*>(p.b_ptr[slot]) + p.b_off + (c + i * C) * kTcNT;
      for (int e = tid; e < R * (kTcNT / 8); e += kT2Threads) {
        const int k = e / (kTcNT / 8), cc = e - k * (kTcNT / 8), na = cc / 8, jj = cc % 8;
        cp_async16(smem + L.b + i * (R * kTcNT * 2) + na * (R / 8) * 1024 + (k / 8) * 1024 + (k % 8) * 128 +
                       ((jj ^ (k % 8)) * 16),
                   B + static_cast<int64_t>(k) * p.h_out + cc * 8);
      }
    }
    cp_async_commit();
    if (it == 0) {
      cluster_arrive_relaxed();  // barrier inits -> the cluster (waited on before the first push)
      LSG_TC_TRACE(0, 1);
      pdl_wait();  // x and y_old may come from the preceding kernel
      LSG_TC_TRACE(0, 2);
    }
    // TMA producer: y chunk 0, then the x boxes -- as many as the ring takes now (the
    // rest after this thread's weight arrival below: the MMA frees ring slots only
    // once the weights are in)
    auto issue_x = [&](int kb) {
      const int g = gbox + kb, s = g % S;
      if (g >= S) mbar_wait(&bars[kB2Empty + s], static_cast<uint32_t>(((g / S) - 1) & 1));
      mbar_arrive_expect_tx(&bars[kB2Full + s], kTcBox);
      tma_load_2d(smem + L.ring + s * kTcBox, &p.tmap_x, (kb0 + kb) * kTcKB, r0, &bars[kB2Full + s]);
    };
    // boxes whose ring slot is free without waiting on this tile's MMAs (a previous
    // tile's boxes were all consumed before its D1 completed)
    const int n_first = min(nk, S);
    if (warp == 0 && lane == 0) {
      if (nmine > 0) {
        mbar_arrive_expect_tx(&bars[kB2Y0], 4 * kTcBox);
#pragma unroll
        for (int b = 0; b < 4; ++b)
          tma_load_2d(smem + L.y0 + b * kTcBox, &p.tmap_y, c * kTcNT + b * kTcKB, r0, &bars[kB2Y0]);
      }
      for (int kb = 0; kb < n_first; ++kb) issue_x(kb);
    }
    // weights landed -> visible to the tensor cores (W completes with every thread's arrival)
    cp_async_wait<0>();
    fence_proxy_async_smem();
    mbar_arrive(&bars[kB2W]);
    if (warp == 0 && lane == 0)
      for (int kb = n_first; kb < nk; ++kb) issue_x(kb);
    if (warp == 1 && lane == 0) {  // MMA issuer: the shrink
      mbar_wait(&bars[kB2W], ph);
      tc_fence_after();
      const uint32_t idesc = umma_idesc(fmt, kTcM, R);
      for (int kb = 0; kb < nk; ++kb) {
        const int g = gbox + kb, s = g % S;
        mbar_wait(&bars[kB2Full + s], static_cast<uint32_t>((g / S) & 1));
        tc_fence_after();
        const uint32_t xa = smem_u32(smem + L.ring + s * kTcBox);
        const uint32_t aa = smem_u32(smem + L.a) + kb * kTcKB * ROWB;
#pragma unroll
        for (int ks = 0; ks < kTcKB / 16; ++ks) {
          const uint64_t ad = umma_desc(xa + ks * 32, 16, 1024, kSw128);           // x: K-major SW128
          const uint64_t bd = umma_desc(aa + ks * 16 * ROWB, 16, 8 * ROWB, kSwA);  // A: MN-major
          umma_f16(tmem, ad, bd, idesc, (kb | ks) ? 1u : 0u);
        }
        umma_commit(&bars[kB2Empty + s]);
      }
      umma_commit(&bars[kB2D1]);  // D1 complete (and the ring consumed)
    }
    if (warp == 0 && lane == 0 && nmine > 1) {  // y chunk 1 into the ring once the shrink read it
      mbar_wait(&bars[kB2D1], ph);
      mbar_arrive_expect_tx(&bars[kB2Y1], 4 * kTcBox);
#pragma unroll
      for (int b = 0; b < 4; ++b)
        tma_load_2d(smem + L.ring + b * kTcBox, &p.tmap_y, (c + C) * kTcNT + b * kTcKB, r0, &bars[kB2Y1]);
    }
    __syncwarp();
    gbox += nk;

    // ---- cluster reduction of v: row partials -> owners -> every CTA ---------------------
    if (it == 0) cluster_wait();  // peers' barriers initialised
    if (tid == 0) {
      mbar_arrive_expect_tx(&bars[kB2Recv], static_cast<uint32_t>(C * rpo * R * 4));
      mbar_arrive_expect_tx(&bars[kB2Vfull], static_cast<uint32_t>(kTcM * R * 4));
    }
    mbar_wait(&bars[kB2D1], ph);
    LSG_TC_TRACE(0, 3);
    tc_fence_after();
    if (warp < 4) {
      const int m = tid;  // tile row = TMEM lane
      const int owner = m / rpo, ml = m - owner * rpo;
      const uint32_t rb = mapa_u32(&bars[kB2Recv], static_cast<uint32_t>(owner));
#pragma unroll
      for (int c0 = 0; c0 < R; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
        const uint32_t ra = mapa_u32(recv + (c * rpo + ml) * R + c0, static_cast<uint32_t>(owner));
#pragma unroll
        for (int j = 0; j < 4; ++j) st_async_v4(ra + j * 16, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3], rb);
      }
    }
    mbar_wait(&bars[kB2Recv], ph);
    for (int qd = tid; qd < rpo * R / 4; qd += kT2Threads) {  // my rows' v, 4 columns per thread
      const int ml = qd / (R / 4), k4 = (qd - ml * (R / 4)) * 4;
      float s4[4] = {0.f, 0.f, 0.f, 0.f};
      for (int cc = 0; cc < C; ++cc)
#pragma unroll
        for (int e = 0; e < 4; ++e) s4[e] += recv[(cc * rpo + ml) * R + k4 + e];
      const float* lv = vfull + (c * rpo + ml) * R + k4;
      for (int d = 0; d < C; ++d)
        st_async_v4(mapa_u32(lv, static_cast<uint32_t>(d)), s4[0], s4[1], s4[2], s4[3],
                    mapa_u32(&bars[kB2Vfull], static_cast<uint32_t>(d)));
    }
    mbar_wait(&bars[kB2Vfull], ph);
    LSG_TC_TRACE(0, 4);
    if (tid < kTcM) {  // v -> 16-bit hi + lo, K-major interleave (m,k) at (m/8)*SBO + (k/8)*128 + (m%8)*16 + (k%8)*2
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

    // ---- expand MMAs: every chunk of this CTA, back to back -------------------------------
    if (warp == 1 && lane == 0) {
      tc_fence_after();
      const uint32_t idesc = umma_idesc(fmt, kTcM, kTcNT);
      for (int i = 0; i < nmine; ++i) {
        const uint32_t bs = smem_u32(smem + L.b + i * (R * kTcNT * 2));
        const uint32_t d2 = tmem + static_cast<uint32_t>(i * kTcNT);
#pragma unroll
        for (int ks = 0; ks < R / 16; ++ks) {
          const uint64_t bd = umma_desc(bs + ks * 2 * 1024, (R / 8) * 1024, 1024, kSw128);  // B: MN-major SW128
          const uint64_t ah = umma_desc(smem_u32(smem + L.vhi) + ks * 256, 128, (R / 8) * 128, kSwNone);
          const uint64_t al = umma_desc(smem_u32(smem + L.vlo) + ks * 256, 128, (R / 8) * 128, kSwNone);
          umma_f16(d2, ah, bd, idesc, ks ? 1u : 0u);
          umma_f16(d2, al, bd, idesc, 1u);
        }
        umma_commit(&bars[kB2E0 + i]);
      }
    }
    __syncwarp();

    // ---- epilogue: warp w -> TMEM lanes 32 (w % 4) .. +32, columns 128 (w / 4) .. +128 -------
    const int m = (warp & 3) * 32 + lane;
    const int half = warp >> 2;
    for (int i = 0; i < nmine; ++i) {
      uint8_t* ybuf = smem + (i == 0 ? L.y0 : L.ring);
      mbar_wait(&bars[kB2Y0 + i], ph);
      mbar_wait(&bars[kB2E0 + i], ph);
      LSG_TC_TRACE(0, 5 + i);
      tc_fence_after();
      uint8_t* yrow = ybuf + m * 128;  // + box * kTcBox + swizzled 16-byte chunk
#pragma unroll 1
      for (int q = 0; q < 2; ++q) {  // 64 columns per batch of TMEM loads
        const int col0 = half * 128 + q * 64;  // within the chunk
        float acc[64];
        tmem_ld64(tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + static_cast<uint32_t>(i * kTcNT + col0),
                  acc);
        const int box = col0 / kTcKB;
#pragma unroll
        for (int j = 0; j < 8; ++j) {  // 8 16-byte chunks of the 64-column box
          uint4* ptr = reinterpret_cast<uint4*>(yrow + box * kTcBox + ((j ^ (m & 7)) * 16));
          float f[8];
          Cvt<T>::unpack8(*ptr, f);
#pragma unroll
          for (int e = 0; e < 8; ++e) f[e] = acc[j * 8 + e] + f[e];
          *ptr = Cvt<T>::pack8(f);
        }
      }
      const int n0 = (c + i * C) * kTcNT;
      if (rows == kTcM) {
        fence_proxy_async_smem();  // epilogue writes -> visible to the TMA store
        __syncthreads();
        if (tid == 0) {
#pragma unroll
          for (int b = 0; b < 4; ++b) tma_store_2d(&p.tmap_y, ybuf + b * kTcBox, n0 + b * kTcKB, r0);
          bulk_commit_group();
        }
      } else if (m < rows) {  // last tile of a segment: only the segment's rows, my column half
        T* yg = static_cast<T*>(p.y) + static_cast<int64_t>(r0 + m) * p.ldy + n0 + half * 128;
#pragma unroll 4
        for (int e = 0; e < 16; ++e) {
          const int b = half * 2 + e / 8, j = e % 8;
          st_global_v4(yg + e * 8, *reinterpret_cast<const uint4*>(yrow + b * kTcBox + ((j ^ (m & 7)) * 16)));
        }
      }
    }
    LSG_TC_TRACE(0, 7);
    // staging free for the next tile: the TMA stores have read it, the TMEM loads are done
    if (tid == 0) bulk_wait_group_read0();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    ++it;
  }
  if (it == 0) {
    // no tile: keep the PDL completion chain and the cluster-barrier pairing
    cluster_arrive_relaxed();
    pdl_wait();
    cluster_wait();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace lsg
