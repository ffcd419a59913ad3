// tma_probe.cu -- how fast can 128 CTAs stream a 2048 x 4096 fp16 activation matrix
// (16-row tiles, one CTA per tile) into shared memory?  Modes:
//   0: 2-D TMA boxes of 64 columns x 16 rows (SW128), 4 boxes per 256-column stage
//   1: 1-D bulk copies, one per row, 512 B per row per stage (256 columns)
//   2: 1-D bulk copies, one per row, 2 KB per row per stage (1024 columns)
// Each CTA keeps `depth` stages in flight (ring, one mbarrier per slot), consumes nothing.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tma_probe scripts/tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(su32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}

__global__ void probe(const __grid_constant__ CUtensorMap map, const __grid_constant__ CUtensorMap m3s,
                      const __grid_constant__ CUtensorMap m3n, const __half* x, int cols, int mode, int depth,
                      unsigned long long* out, int KC, int RT, int smem_bytes) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + smem_bytes - 256);
  const uint32_t stage = RT * KC * 2;
  const int nst = cols / KC;
  const int r0 = blockIdx.x * RT;
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) mb_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  auto issue = [&](int s) {
    uint8_t* dst = smem + (s % depth) * stage;
    uint64_t* b = &bars[s % depth];
    mb_expect(b, stage);
    if (mode == 0) {
      for (int q = 0; q < KC / 64; ++q) tma2d(dst + q * 2048, &map, s * KC + q * 64, r0, b);  // RT = 16 only
    } else if (mode == 2) {  // ONE 3-D box per stage: {64 cols, RT rows, KC/64 blocks}, SW128
      tma3d(dst, &m3s, 0, r0, s * KC / 64, b);
    } else if (mode == 3) {  // ONE 3-D box per stage: {256 cols, RT rows, KC/256 blocks}, no swizzle
      tma3d(dst, &m3n, 0, r0, s * KC / 256, b);
    } else {
      for (int m = 0; m < RT; ++m) bulk(dst + m * KC * 2, x + static_cast<int64_t>(r0 + m) * cols + s * KC, KC * 2, b);
    }
  };
  for (int s = 0; s < depth && s < nst; ++s) issue(s);
  for (int s = 0; s < nst; ++s) {
    mb_wait(&bars[s % depth], (s / depth) & 1);
    if (s + depth < nst) issue(s + depth);
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out[blockIdx.x] = t1 - t0;
}


// K9-like stages: per stage, the tile's 16 activation rows (one 1-D bulk copy of KC*2 bytes each,
// from a matrix larger than L2) plus 32 KB of weights from a small L2-resident matrix W, loaded as
// wmode 0: none, 1: 16 x 1-D rows of 2 KB, 2: 16 x 2-D boxes (16 rows x 64 cols, SW128), 3: one 1-D 32 KB copy
__global__ void probe2(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap wmap3, const __half* x, const __half* w, int cols, int wmode,
                       int depth, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int KC = 1024, RT = 16;
  const uint32_t act = RT * KC * 2, wb = 32768, stage = act + wb;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + depth * stage);
  const int nst = cols / KC;
  const int r0 = blockIdx.x * RT;
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) mb_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  auto issue = [&](int s) {
    uint8_t* dst = smem + (s % depth) * stage;
    uint64_t* b = &bars[s % depth];
    mb_expect(b, act + (wmode ? wb : 0));
    if (wmode == 1) {
      for (int k = 0; k < 16; ++k) bulk(dst + act + k * 2048, w + k * 4096 + (s % 4) * KC, 2048, b);
    } else if (wmode == 2) {
      for (int q = 0; q < 16; ++q) tma2d(dst + act + q * 2048, &wmap, (s % 4) * KC + q * 64, 0, b);
    } else if (wmode == 3) {
      bulk(dst + act, w + (s % 4) * 16384, wb, b);
    } else if (wmode == 4) {  // one 3-D box: 16 column blocks x 16 rows x 64 columns
      tma3d(dst + act, &wmap3, 0, 0, (s % 4) * 16, b);
    }
    for (int m = 0; m < RT; ++m) bulk(dst + m * KC * 2, x + static_cast<int64_t>(r0 + m) * cols + s * KC, KC * 2, b);
  };
  for (int s = 0; s < depth && s < nst; ++s) issue(s);
  for (int s = 0; s < nst; ++s) {
    mb_wait(&bars[s % depth], (s / depth) & 1);
    if (s + depth < nst) issue(s + depth);
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out[blockIdx.x] = t1 - t0;
}

int main() {
  const int rows = 2048, cols = 4096, tiles = rows / 16;
  const size_t bytes = static_cast<size_t>(rows) * cols * 2;
  const int nbuf = 16;  // rotate over 16 matrices (> L2)
  std::vector<__half*> xs(nbuf);
  for (auto& p : xs) {
    cudaMalloc(&p, bytes);
    cudaMemset(p, 1, bytes);
  }
  unsigned long long* out;
  cudaMalloc(&out, rows * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<decltype(&cuTensorMapEncodeTiled)>(fn);
  std::vector<CUtensorMap> maps(nbuf), m3s(nbuf), m3n(nbuf);
  for (int i = 0; i < nbuf; ++i) {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t str[1] = {static_cast<cuuint64_t>(cols) * 2};
    cuuint32_t box[2] = {64, 16}, es[2] = {1, 1};
    enc(&maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, xs[i], dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t d3[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols / 64)};
    cuuint64_t s3[2] = {static_cast<cuuint64_t>(cols) * 2, 128};
    cuuint32_t b3[3] = {64, 16, 16}, e3[3] = {1, 1, 1};
    if (enc(&m3s[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, xs[i], d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      printf("m3s encode failed\n");
    cuuint64_t d4[3] = {256, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols / 256)};
    cuuint64_t s4[2] = {static_cast<cuuint64_t>(cols) * 2, 512};
    cuuint32_t b4[3] = {256, 16, 4};
    if (enc(&m3n[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, xs[i], d4, s4, b4, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      printf("m3n encode failed\n");
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Cfg { int mode, RT, KC, depth, ctas_per_sm; };
  const Cfg cfgs[] = {{0, 16, 256, 8, 1},  {1, 16, 1024, 4, 1}, {1, 16, 2048, 3, 1}, {1, 16, 4096, 1, 1},
                      {1, 8, 1024, 4, 2},  {1, 8, 2048, 3, 2},  {1, 8, 4096, 1, 2},  {1, 16, 1024, 2, 2},
                      {1, 4, 4096, 2, 3},  {1, 4, 2048, 4, 3}, {1, 16, 1024, 3, 1}, {2, 16, 1024, 3, 1},
                      {3, 16, 1024, 3, 1}, {2, 16, 1024, 6, 1}, {3, 16, 1024, 6, 1}};
  for (const Cfg& c : cfgs) {
    const int smem = c.ctas_per_sm == 1 ? 210 * 1024 : c.ctas_per_sm == 2 ? 110 * 1024 : 72 * 1024;
    if (c.depth * c.RT * c.KC * 2 + 256 > smem) continue;
    const int ctas = rows / c.RT;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int w = 0; w < 3; ++w) probe<<<ctas, 32, smem>>>(maps[w], m3s[w], m3n[w], xs[w], cols, c.mode, c.depth, out, c.KC, c.RT, smem);
    cudaEventRecord(a);
    const int iters = 32;
    for (int it = 0; it < iters; ++it)
      probe<<<ctas, 32, smem>>>(maps[it % nbuf], m3s[it % nbuf], m3n[it % nbuf], xs[it % nbuf], cols, c.mode, c.depth, out, c.KC, c.RT, smem);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<unsigned long long> h(ctas);
    cudaMemcpy(h.data(), out, ctas * 8, cudaMemcpyDeviceToHost);
    double mx = 0, sum = 0;
    for (auto v : h) {
      mx = v > mx ? v : mx;
      sum += v;
    }
    const double us = ms * 1e3 / iters;
    printf("mode %d rows/CTA %2d piece %5d B depth %d ctas %4d: %7.2f us/launch %6.0f GB/s  per-CTA mean %.2f max %.2f us\n",
           c.mode, c.RT, c.KC * 2, c.depth, ctas, us, bytes / us / 1e3, sum / ctas / 1e3, mx / 1e3);
  }
  {  // K9-like stages
    __half* w;
    cudaMalloc(&w, 16 * 4096 * 2 * 4);
    cudaMemset(w, 1, 16 * 4096 * 2 * 4);
    CUtensorMap wmap;
    cuuint64_t dims[2] = {4096, 16};
    cuuint64_t str[1] = {4096 * 2};
    cuuint32_t box[2] = {64, 16}, es[2] = {1, 1};
    enc(&wmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int depth = 3, smem = depth * (16 * 1024 * 2 + 32768) + 256, ctas = rows / 16;
    CUtensorMap wmap3;
    {
      cuuint64_t d3[3] = {64, 16, 4096 / 64};
      cuuint64_t s3[2] = {4096 * 2, 128};
      cuuint32_t b3[3] = {64, 16, 16}, e3[3] = {1, 1, 1};
      CUresult r3 = enc(&wmap3, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, w, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      printf("3-D weight map (strides 8192, 128 B): encode %s\n", r3 == CUDA_SUCCESS ? "ok" : "FAILED");
    }
    cudaFuncSetAttribute(probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int wmode = 0; wmode < 5; ++wmode) {
      for (int it = 0; it < 3; ++it) probe2<<<ctas, 32, smem>>>(wmap, wmap3, xs[it], w, cols, wmode, depth, out);
      cudaEventRecord(a);
      const int iters = 32;
      for (int it = 0; it < iters; ++it) probe2<<<ctas, 32, smem>>>(wmap, wmap3, xs[it % nbuf], w, cols, wmode, depth, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      std::vector<unsigned long long> h(ctas);
      cudaMemcpy(h.data(), out, ctas * 8, cudaMemcpyDeviceToHost);
      double mx = 0, sum = 0;
      for (auto v : h) {
        mx = v > mx ? v : mx;
        sum += v;
      }
      printf("K9-like stages (16 x 2 KB activation rows + 32 KB L2 weights as %s), depth 3: %.2f us/launch  per-CTA mean %.2f max %.2f us\n",
             wmode == 0 ? "none" : wmode == 1 ? "16 x 1-D 2 KB rows" : wmode == 2 ? "16 x 2-D boxes (128-B rows)" : wmode == 3 ? "one 1-D 32 KB copy" : "one 3-D box",
             ms * 1e3 / iters, sum / ctas / 1e3, mx / 1e3);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
