// icache_probe.cu -- does a once-executed code region pay instruction-fetch latency?
// Warp 0 of each CTA runs the same 8-step LDS+FMA block (the SGMV shrink unit)
// twice, stamping clock64 around each pass.  Pass 1 runs cold code, pass 2 warm.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/icache_probe scripts/icache_probe.cu
#include <cstdio>
#include <cuda_fp16.h>

template <int PASS>
__device__ __noinline__ float unit(const uint4* A, const __half* x, int lane) {
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    uint4 u = A[(it * 16 + lane / 2) * 2 + (lane & 1)];
    const __half2* h = reinterpret_cast<const __half2*>(&u);
    float xm = __half2float(x[it * 16 + lane / 2]);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 t = __half22float2(h[i]);
      acc[2 * i] = fmaf(xm, t.x, acc[2 * i]);
      acc[2 * i + 1] = fmaf(xm, t.y, acc[2 * i + 1]);
    }
  }
#pragma unroll
  for (int off = 2; off < 32; off <<= 1)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], off);
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j];
  return s;
}

__global__ void probe(long long* out, float* sink, int pad) {
  __shared__ uint4 A[256 * 2];
  __shared__ __half x[128];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) A[i] = make_uint4(i, i + 1, i + 2, i + 3);
  for (int i = threadIdx.x; i < 128; i += blockDim.x) x[i] = __float2half(i * 0.01f);
  __syncthreads();
  if (threadIdx.x < 32) {
    long long t0 = clock64();
    float a = unit<0>(A, x, threadIdx.x);
    long long t1 = clock64();
    float b = unit<0>(A, x, threadIdx.x);  // same code, now warm
    long long t2 = clock64();
    float c = unit<1>(A, x, threadIdx.x);  // different copy of the code: cold again
    long long t3 = clock64();
    if (threadIdx.x == 0) {
      out[blockIdx.x * 3 + 0] = t1 - t0;
      out[blockIdx.x * 3 + 1] = t2 - t1;
      out[blockIdx.x * 3 + 2] = t3 - t2;
    }
    sink[blockIdx.x * 32 + threadIdx.x] = a + b + c;
  }
}

int main() {
  long long* d;
  float* s;
  const int n = 148;
  cudaMalloc(&d, n * 3 * sizeof(long long));
  cudaMalloc(&s, n * 32 * sizeof(float));
  for (int rep = 0; rep < 3; ++rep) {
    probe<<<n, 256>>>(d, s, 0);
    cudaDeviceSynchronize();
    long long h[n * 3];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    long long m[3] = {0, 0, 0};
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < 3; ++j) m[j] += h[i * 3 + j];
    printf("launch %d: mean cycles  pass1(cold) %lld  pass2(warm, same code) %lld  pass3(cold copy) %lld\n", rep,
           m[0] / n, m[1] / n, m[2] / n);
  }
  return 0;
}
