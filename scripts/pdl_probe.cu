// pdl_probe.cu -- when does a programmatic dependent launch actually start?
// Kernel `primary` triggers griddepcontrol.launch_dependents at entry, then spins
// for `spin_ns`; kernel `secondary` records its entry time.  Chains of
// primary/secondary pairs are launched eagerly and from a CUDA graph, with the
// PDL attribute, for several grid sizes / smem footprints.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdl_probe pdl_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                                      \
  do {                                                                                             \
    cudaError_t e = (x);                                                                           \
    if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } \
  } while (0)

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// stamps[launch*3 + 0] = min entry, +1 = max entry, +2 = max exit (atomics)
__global__ void k_chain(unsigned long long* stamps, int launch, unsigned long long spin_ns, int trigger_early) {
  extern __shared__ char sm[];
  const unsigned long long t0 = gtime();
  if (trigger_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) {
    atomicMin(&stamps[launch * 3 + 0], t0);
    atomicMax(&stamps[launch * 3 + 1], t0);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  while (gtime() - t0 < spin_ns) {
  }
  sm[threadIdx.x] = 1;
  if (!trigger_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&stamps[launch * 3 + 2], gtime());
}

int main() {
  const int L = 20;
  unsigned long long* stamps;
  CK(cudaMalloc(&stamps, L * 3 * 8));
  CK(cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  std::vector<unsigned long long> h(L * 3);
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  for (int graph = 0; graph < 2; ++graph)
    for (int early = 1; early >= 0; --early)
      for (int grid : {64, 128, 148, 192, 296})
        for (int smem : {40 * 1024, 100 * 1024}) {
          std::vector<unsigned long long> init(L * 3);
          for (int i = 0; i < L; ++i) {
            init[i * 3] = ~0ull;
            init[i * 3 + 1] = 0;
            init[i * 3 + 2] = 0;
          }
          CK(cudaMemcpy(stamps, init.data(), L * 24, cudaMemcpyHostToDevice));
          auto launch_all = [&]() {
            for (int i = 0; i < L; ++i) {
              cudaLaunchConfig_t cfg{};
              cfg.gridDim = dim3(grid);
              cfg.blockDim = dim3(256);
              cfg.dynamicSmemBytes = smem;
              cfg.stream = st;
              cudaLaunchAttribute at;
              at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
              at.val.programmaticStreamSerializationAllowed = 1;
              cfg.attrs = &at;
              cfg.numAttrs = 1;
              CK(cudaLaunchKernelEx(&cfg, k_chain, stamps, i, 5000ull, early));
            }
          };
          if (graph) {
            cudaGraph_t g;
            cudaGraphExec_t ge;
            CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
            launch_all();
            CK(cudaStreamEndCapture(st, &g));
            CK(cudaGraphInstantiate(&ge, g, 0));
            CK(cudaGraphLaunch(ge, st));
            CK(cudaStreamSynchronize(st));
            CK(cudaMemcpy(stamps, init.data(), L * 24, cudaMemcpyHostToDevice));
            CK(cudaGraphLaunch(ge, st));
          } else {
            launch_all();
          }
          CK(cudaStreamSynchronize(st));
          CK(cudaMemcpy(h.data(), stamps, L * 24, cudaMemcpyDeviceToHost));
          double lead = 0, period = 0, spread = 0;
          int n = 0;
          for (int i = 5; i < L; ++i) {
            lead += (double)h[(i - 1) * 3 + 2] - (double)h[i * 3 + 0];  // prev end - this first entry
            period += (double)h[i * 3 + 2] - (double)h[(i - 1) * 3 + 2];
            spread += (double)h[i * 3 + 1] - (double)h[i * 3 + 0];
            ++n;
          }
          printf("graph=%d trigger_early=%d grid=%3d smem=%3dKB: period %.2f us, next-launch first CTA %.2f us "
                 "before prev end, entry spread %.2f us\n",
                 graph, early, grid, smem / 1024, period / n / 1e3, lead / n / 1e3, spread / n / 1e3);
        }
  return 0;
}
