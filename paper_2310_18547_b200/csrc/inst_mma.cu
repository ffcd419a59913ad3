// inst_mma.cu -- sm_100a instantiations of the segment-tile tensor-core pair (K7,
// sgmv_mma.cuh) and their launchers.
#include <mutex>

#include "launch.cuh"
#include "sgmv_mma.cuh"
#include "sgmv_stream.cuh"
#include "sgmv_dense.cuh"

namespace lsg {

template <typename T, int R>
static int launch_mma_inst(const MmaParams& p, int tiles, cudaStream_t st) {
  auto kp = sgmv_mma_part_kernel<T, R>;
  auto ke = sgmv_mma_exp_kernel<T, R>;
  static std::atomic<unsigned long long> configured{0};  // one bit per device
  if (!configured_on_device(configured)) {
    cudaError_t e = cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(ke, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(mma pair smem)");
    mark_configured(configured);
  }
  cudaError_t e = launch_ex(kp, dim3(static_cast<unsigned>(p.kparts), static_cast<unsigned>(tiles), 1),
                            dim3(32 * kMmaPW), static_cast<int>(mma_part_smem(R, p.h_in / p.kparts / kMmaKC, p.pc)),
                            p.pc > 1 ? p.pc : 0, st, &p);
  if (e != cudaSuccess) return cuda_fail(e, "sgmv_mma_part_kernel launch");
  e = launch_ex(ke, dim3(static_cast<unsigned>(p.ncol), static_cast<unsigned>(tiles), 1), dim3(kMmaThreads),
                static_cast<int>(mma_exp_smem(R, p.h_out / p.ncol / kMmaKC, p.kparts / p.pc)), 0, st, &p);
  return e == cudaSuccess ? LSG_OK : cuda_fail(e, "sgmv_mma_exp_kernel launch");
}

int launch_mma_pair(int dtype, int rank, const MmaParams& p, int tiles, cudaStream_t st) {
#define LSG_MMA_R(T)                                                                    \
  switch (rank) {                                                                       \
    case 16: return launch_mma_inst<T, 16>(p, tiles, st);                               \
    case 32: return launch_mma_inst<T, 32>(p, tiles, st);                               \
    case 64: return launch_mma_inst<T, 64>(p, tiles, st);                               \
    default: return fail(LSG_EUNSUPPORTED, "segment-tile MMA pair: rank not in {16,32,64}"); \
  }
  if (dtype == LSG_F16) LSG_MMA_R(__half)
  LSG_MMA_R(__nv_bfloat16)
#undef LSG_MMA_R
}

template <typename T, int R>
static int launch_stream_inst(const StreamParams& p, int tiles, cudaStream_t st) {
  auto k = sgmv_stream_kernel<T, R>;
  static std::atomic<unsigned long long> configured{0};  // one bit per device
  if (!configured_on_device(configured)) {
    const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(stream smem)");
    mark_configured(configured);
  }
  const cudaError_t e = launch_ex(k, dim3(static_cast<unsigned>(tiles)), dim3(kStreamThreads),
                                  static_cast<int>(stream_smem(R, p.stages)), 0, st, &p);
  return e == cudaSuccess ? LSG_OK : cuda_fail(e, "sgmv_stream_kernel launch");
}

int launch_stream(int dtype, int rank, const StreamParams& p, int tiles, cudaStream_t st) {
#define LSG_ST_R(T)                                                                     \
  switch (rank) {                                                                       \
    case 16: return launch_stream_inst<T, 16>(p, tiles, st);                            \
    case 32: return launch_stream_inst<T, 32>(p, tiles, st);                            \
    case 64: return launch_stream_inst<T, 64>(p, tiles, st);                            \
    default: return fail(LSG_EUNSUPPORTED, "streaming kernel: rank not in {16,32,64}"); \
  }
  if (dtype == LSG_F16) LSG_ST_R(__half)
  LSG_ST_R(__nv_bfloat16)
#undef LSG_ST_R
}

template <typename T>
static bool configure_dense_lora() {
  static std::atomic<unsigned long long> configured{0};  // one bit per device (per instantiation)
  if (configured_on_device(configured)) return true;
  if (cudaFuncSetAttribute(dense_lora_kernel<T, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, dn_smem()) !=
      cudaSuccess)
    return false;
  // the shrink CTAs (small) share SMs with the GEMM's: leave the GEMM its shared memory
  if (cudaFuncSetAttribute(dense_shrink_kernel<T, 16>, cudaFuncAttributePreferredSharedMemoryCarveout, 100) !=
      cudaSuccess)
    return false;
  mark_configured(configured);
  return true;
}

template <typename T>
static int launch_dense_lora_inst(const DenseLoraParams& p, cudaStream_t st) {
  if (!configure_dense_lora<T>()) return cuda_fail(cudaGetLastError(), "cudaFuncSetAttribute(dense lora smem)");
  cudaError_t e = launch_ex(dense_shrink_kernel<T, 16>, dim3(static_cast<unsigned>(p.s_n)), dim3(kDnShThreads), 0, 0,
                            st, &p);
  if (e != cudaSuccess) return cuda_fail(e, "dense_shrink_kernel launch");
  e = launch_ex(dense_lora_kernel<T, 16>, dim3(static_cast<unsigned>(p.ks),
                                                                 static_cast<unsigned>(p.h_out / kDnN)),
                                  dim3(kDnThreads), dn_smem(), p.ks, st, &p);
  return e == cudaSuccess ? LSG_OK : cuda_fail(e, "dense_lora_kernel launch");
}

int launch_dense_lora(int dtype, const DenseLoraParams& p, cudaStream_t st) {
  return dtype == LSG_F16 ? launch_dense_lora_inst<__half>(p, st) : launch_dense_lora_inst<__nv_bfloat16>(p, st);
}

template <typename T>
static int dense_max_clusters_inst(int ks) {
  if (!configure_dense_lora<T>()) return 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(ks), 1, 1);
  cfg.blockDim = dim3(kDnThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(dn_smem());
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = static_cast<unsigned>(ks);
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, dense_lora_kernel<T, 16>, &cfg) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  return n;
}

int dense_lora_max_clusters(int dtype, int ks) {
  // cached per (device, dtype, ks): the answer depends only on the device
  static std::mutex mu;
  static int cache[64][2][4] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
  const int d = dtype == LSG_F16 ? 0 : 1, k = ks == 8 ? 3 : ks == 4 ? 2 : ks == 2 ? 1 : 0;
  std::lock_guard<std::mutex> lock(mu);
  if (cache[dev][d][k] == 0)
    cache[dev][d][k] = d == 0 ? dense_max_clusters_inst<__half>(ks) : dense_max_clusters_inst<__nv_bfloat16>(ks);
  return cache[dev][d][k];
}

}  // namespace lsg
