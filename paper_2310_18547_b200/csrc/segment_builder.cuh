// segment_builder.cuh -- K6: on-device segment + permutation builder.
//
// Replaces the host-side grouping the reference does in plan_batch
// (simulator.cpp:267-309: std::map<LoraId, vector<RequestId>> -> contiguous
// same-adapter row segments, prefill's adapter first) and the per-row gather
// loop of gather_bmm_oracle (sgmv.cpp:195-203).  One CTA of 1024 threads sorts
// the 64-bit keys (group_key << 32 | row) with an in-shared-memory bitonic sort
// -- the row index in the low word makes the grouping stable -- then marks group
// heads and compacts them with a block-wide scan.
#pragma once

#include <stdint.h>

#include "sgmv_device.cuh"

namespace lsg {

constexpr int kBuilderThreads = 1024;
constexpr int kBuilderMaxRows = 16384;

__global__ void __launch_bounds__(kBuilderThreads, 1)
    build_segments_kernel(const int32_t* __restrict__ row_slot, int32_t s_n, int32_t num_slots,
                          int32_t lead_slot, int32_t lead_row0, int32_t lead_row1, int32_t n_pow2,
                          int32_t* __restrict__ row_perm,
                          int32_t* __restrict__ seg_starts, int32_t* __restrict__ seg_slot,
                          int32_t* __restrict__ num_segments) {
  extern __shared__ uint64_t keys[];  // n_pow2 entries
  __shared__ int32_t warp_tot[kBuilderThreads / 32];
  const int tid = threadIdx.x;
  pdl_wait();
  // group key: lead slot -> 0, slot s -> s + 1, no adapter -> 0x7fffffff (last).
  // Within the lead group the prefill request's rows [lead_row0, lead_row1) come
  // first (sub-key 0), then the same-adapter decode rows (sub-key 1): plan_batch
  // pushes the prefill's prompt rows before the merged decode group
  // (simulator.cpp:296-309).  Key = group << 32 | sub << 31 | row (row < 2^31).
  for (int i = tid; i < n_pow2; i += kBuilderThreads) {
    uint64_t k = ~0ull;
    if (i < s_n) {
      const int s = row_slot[i];
      uint32_t g, sub = 0;
      if (s < 0 || s >= num_slots) {
        g = 0x7fffffffu;
      } else if (s == lead_slot) {
        g = 0u;
        sub = (i >= lead_row0 && i < lead_row1) ? 0u : 1u;
      } else {
        g = static_cast<uint32_t>(s) + 1u;
      }
      k = (static_cast<uint64_t>(g) << 32) | (static_cast<uint64_t>(sub) << 31) | static_cast<uint32_t>(i);
    }
    keys[i] = k;
  }
  __syncthreads();
  // bitonic sort, ascending
  for (int size = 2; size <= n_pow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < n_pow2 / 2; i += kBuilderThreads) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint64_t a = keys[lo], b = keys[hi];
        if ((a > b) == up) {
          keys[lo] = b;
          keys[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  // heads + block scan: thread t owns elements [t*E, (t+1)*E)
  const int E = (s_n + kBuilderThreads - 1) / kBuilderThreads;
  const int b0 = tid * E, b1 = min(s_n, b0 + E);
  int cnt = 0;
  for (int i = b0; i < b1; ++i) {
    row_perm[i] = static_cast<int32_t>(keys[i] & 0x7fffffffu);
    cnt += (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) ? 1 : 0;
  }
  const int lane = tid & 31, warp = tid >> 5;
  int incl = cnt;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = warp_tot[lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w += v;
    }
    warp_tot[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  int seg = (warp > 0 ? warp_tot[warp - 1] : 0) + incl - cnt;  // exclusive prefix
  const int total = warp_tot[kBuilderThreads / 32 - 1];
  for (int i = b0; i < b1; ++i) {
    if (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) {
      seg_starts[seg] = i;
      const int s = row_slot[keys[i] & 0x7fffffffu];
      seg_slot[seg] = (s < 0 || s >= num_slots) ? -1 : s;
      ++seg;
    }
  }
  for (int i = total + tid; i <= s_n; i += kBuilderThreads) seg_starts[i] = s_n;
  for (int i = total + tid; i < s_n; i += kBuilderThreads) seg_slot[i] = -1;
  if (tid == 0) *num_segments = total;
  pdl_launch_dependents();
}

// dst[i, :] = src[perm[i], :] (gather) or dst[perm[i], :] = src[i, :] (scatter)
template <bool kGather>
__global__ void permute_rows_kernel(uint16_t* __restrict__ dst, int64_t ld_dst,
                                    const uint16_t* __restrict__ src, int64_t ld_src,
                                    const int32_t* __restrict__ perm, int32_t cols, bool vec) {
  const int i = blockIdx.x;
  pdl_wait();
  const int j = perm[i];
  const int64_t dr = kGather ? i : j, sr = kGather ? j : i;
  uint16_t* d = dst + dr * ld_dst;
  const uint16_t* s = src + sr * ld_src;
  if (vec) {
    const uint4* s4 = reinterpret_cast<const uint4*>(s);
    uint4* d4 = reinterpret_cast<uint4*>(d);
    for (int c = threadIdx.x; c < cols / 8; c += blockDim.x) d4[c] = s4[c];
  } else {
    for (int c = threadIdx.x; c < cols; c += blockDim.x) d[c] = s[c];
  }
  pdl_launch_dependents();
}

}  // namespace lsg
