// inst_tc.cu -- sm_100a instantiations of the tensor-core SGMV kernels (K5) and their launchers.
#include <cuda.h>

#include "launch.cuh"
#include "sgmv_tc.cuh"

namespace lsg {

template <typename T, int R>
static int launch_tc_shrink_inst(const TcShrinkParams& p, int nq, int tiles, cudaStream_t st) {
  auto kern = sgmv_tc_shrink_kernel<T, R>;
  static std::atomic<unsigned long long> configured{0};  // one bit per device
  if (!configured_on_device(configured)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tc shrink smem)");
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tc shrink cluster)");
    mark_configured(configured);
  }
  const dim3 grid(static_cast<unsigned>(nq), static_cast<unsigned>(tiles), 1);
  const int smem = static_cast<int>(tc_shrink_smem(R, p.kcs));
  const cudaError_t e = launch_ex(kern, grid, dim3(kTcThreads), smem, nq, st, &p);
  return e == cudaSuccess ? LSG_OK : cuda_fail(e, "sgmv_tc_shrink_kernel launch");
}

template <typename T, int R>
static int launch_tc_expand_inst(const TcExpandParams& p, int tiles, cudaStream_t st) {
  auto kern = sgmv_tc_expand_kernel<T, R>;
  static std::atomic<unsigned long long> configured{0};  // one bit per device
  if (!configured_on_device(configured)) {
    const cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TcExpandLayout<R>::kTotal);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tc expand smem)");
    mark_configured(configured);
  }
  const dim3 grid(static_cast<unsigned>(p.h_out / kTcNT), static_cast<unsigned>(tiles), 1);
  const cudaError_t e =
      launch_ex(kern, grid, dim3(kTcThreads), static_cast<int>(TcExpandLayout<R>::kTotal), 0, st, &p);
  return e == cudaSuccess ? LSG_OK : cuda_fail(e, "sgmv_tc_expand_kernel launch");
}

int launch_tc_shrink(int dtype, int rank, const TcShrinkParams& p, int nq, int tiles, cudaStream_t st) {
#define LSG_TC_R(T)                                                                   \
  switch (rank) {                                                                     \
    case 16: return launch_tc_shrink_inst<T, 16>(p, nq, tiles, st);                   \
    case 32: return launch_tc_shrink_inst<T, 32>(p, nq, tiles, st);                   \
    case 64: return launch_tc_shrink_inst<T, 64>(p, nq, tiles, st);                   \
    default: return fail(LSG_EUNSUPPORTED, "tensor-core shrink: rank not in {16,32,64}"); \
  }
  if (dtype == LSG_F16) LSG_TC_R(__half)
  LSG_TC_R(__nv_bfloat16)
#undef LSG_TC_R
}

int launch_tc_expand(int dtype, int rank, const TcExpandParams& p, int tiles, cudaStream_t st) {
#define LSG_TC_R(T)                                                               \
  switch (rank) {                                                                 \
    case 16: return launch_tc_expand_inst<T, 16>(p, tiles, st);                   \
    case 32: return launch_tc_expand_inst<T, 32>(p, tiles, st);                   \
    case 64: return launch_tc_expand_inst<T, 64>(p, tiles, st);                   \
    default: return fail(LSG_EUNSUPPORTED, "tensor-core expand: rank not in {16,32,64}"); \
  }
  if (dtype == LSG_F16) LSG_TC_R(__half)
  LSG_TC_R(__nv_bfloat16)
#undef LSG_TC_R
}

}  // namespace lsg

namespace lsg {

template <typename T>
static int launch_tc_fused_inst(const TcFusedParams& p, int C, int tiles, cudaStream_t st) {
  auto kern = sgmv_tc_fused_kernel<T>;
  static std::atomic<unsigned long long> configured{0};  // one bit per device
  if (!configured_on_device(configured)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tc fused smem)");
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tc fused cluster)");
    mark_configured(configured);
  }
  const dim3 grid(static_cast<unsigned>(C), static_cast<unsigned>(tiles), 1);
  const int smem = static_cast<int>(tcf_layout(p.kcs_max, p.compact).total);
  const cudaError_t e = launch_ex(kern, grid, dim3(kTcThreads), smem, C, st, &p);
  return e == cudaSuccess ? LSG_OK : cuda_fail(e, "sgmv_tc_fused_kernel launch");
}

int launch_tc_fused(int dtype, const TcFusedParams& p, int C, int tiles, cudaStream_t st) {
  return dtype == LSG_F16 ? launch_tc_fused_inst<__half>(p, C, tiles, st)
                          : launch_tc_fused_inst<__nv_bfloat16>(p, C, tiles, st);
}

}  // namespace lsg

namespace lsg {

template <typename T>
static int launch_dense_lora_inst(const DenseLoraParams& p, cudaStream_t st) {
  auto kern = dense_lora_kernel<T, 16>;
  static std::atomic<unsigned long long> configured{0};  // one bit per device (per instantiation)
  if (!configured_on_device(configured)) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dl_smem<16>()));
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(dense lora smem)");
    mark_configured(configured);
  }
  const cudaError_t e = launch_ex(kern, dim3(kDlKS, static_cast<unsigned>(p.h_out / kDlN)), dim3(kTcThreads),
                                  static_cast<int>(dl_smem<16>()), kDlKS, st, &p);
  return e == cudaSuccess ? LSG_OK : cuda_fail(e, "dense_lora_kernel launch");
}

int launch_dense_lora(int dtype, const DenseLoraParams& p, cudaStream_t st) {
  return dtype == LSG_F16 ? launch_dense_lora_inst<__half>(p, st) : launch_dense_lora_inst<__nv_bfloat16>(p, st);
}

}  // namespace lsg

#include "sgmv_tc2.cuh"

namespace lsg {

// Streamed tensor-core kernel: a persistent grid of at most the co-resident clusters
// (cudaOccupancyMaxActiveClusters, cached per device / cluster size / smem); clusters
// loop over the long-segment tiles.
template <typename T, int R>
static int launch_tc_stream_inst(const Tc2Params& p, int C, uint32_t smem, int tiles, cudaStream_t st) {
  auto kern = sgmv_tc_stream_kernel<T, R>;
  static std::atomic<unsigned long long> configured{0};  // one bit per device
  if (!configured_on_device(configured)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tc stream smem)");
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tc stream cluster)");
    mark_configured(configured);
  }
  static std::atomic<int> cached[64][2];  // [device][C == 16] -> co-resident clusters (0: not queried)
  const int dev = current_device() & 63, ci = C == 16 ? 1 : 0;
  int maxc = cached[dev][ci].load();
  if (maxc == 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(C), 1024, 1);
    cfg.blockDim = dim3(kT2Threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = static_cast<unsigned>(C);
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, reinterpret_cast<const void*>(kern), &cfg) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = 148 / C;
    }
    maxc = n;
    cached[dev][ci].store(n);
  }
  const int clusters = std::max(1, std::min(tiles, maxc));
  const dim3 grid(static_cast<unsigned>(C), static_cast<unsigned>(clusters), 1);
  const cudaError_t e = launch_ex(kern, grid, dim3(kT2Threads), static_cast<int>(smem), C, st, &p);
  return e == cudaSuccess ? LSG_OK : cuda_fail(e, "sgmv_tc_stream_kernel launch");
}

int launch_tc_stream(int dtype, int rank, const Tc2Params& p, int C, uint32_t smem, int tiles, cudaStream_t st) {
#define LSG_TC2_R(T)                                                                       \
  switch (rank) {                                                                          \
    case 16: return launch_tc_stream_inst<T, 16>(p, C, smem, tiles, st);                   \
    case 32: return launch_tc_stream_inst<T, 32>(p, C, smem, tiles, st);                   \
    default: return fail(LSG_EUNSUPPORTED, "streamed tensor-core kernel: rank not in {16,32}"); \
  }
  if (dtype == LSG_F16) LSG_TC2_R(__half)
  LSG_TC2_R(__nv_bfloat16)
#undef LSG_TC2_R
}

}  // namespace lsg

#include "sgmv_tc3.cuh"

namespace lsg {

template <typename T, int R>
static int launch_tc3_parts_inst(const Tc3PartParams& p, int tiles, cudaStream_t st) {
  auto kern = sgmv_tc_part_kernel<T, R>;
  static std::atomic<unsigned long long> configured{0};  // one bit per device
  if (!configured_on_device(configured)) {
    const cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Tc3PartLayout<R>::kTotal);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tc parts smem)");
    mark_configured(configured);
  }
  const dim3 grid(static_cast<unsigned>(p.kparts), static_cast<unsigned>(tiles), 1);
  const cudaError_t e =
      launch_ex(kern, grid, dim3(kT3Threads), static_cast<int>(Tc3PartLayout<R>::kTotal), 0, st, &p);
  return e == cudaSuccess ? LSG_OK : cuda_fail(e, "sgmv_tc_part_kernel launch");
}

template <typename T, int R>
static int launch_tc3_expand_inst(const Tc3ExpParams& p, int tiles, cudaStream_t st) {
  auto kern = sgmv_tc_exp_kernel<T, R>;
  static std::atomic<unsigned long long> configured{0};  // one bit per device
  if (!configured_on_device(configured)) {
    const cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Tc3ExpLayout<R>::kTotal);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tc expand2 smem)");
    mark_configured(configured);
  }
  const dim3 grid(static_cast<unsigned>(p.h_out / kTcNT), static_cast<unsigned>(tiles), 1);
  const cudaError_t e =
      launch_ex(kern, grid, dim3(kT3Threads), static_cast<int>(Tc3ExpLayout<R>::kTotal), 0, st, &p);
  return e == cudaSuccess ? LSG_OK : cuda_fail(e, "sgmv_tc_exp_kernel launch");
}

#define LSG_TC3_R(FN, T, ...)                                                        \
  switch (rank) {                                                                    \
    case 16: return FN<T, 16>(__VA_ARGS__);                                          \
    case 32: return FN<T, 32>(__VA_ARGS__);                                          \
    case 64: return FN<T, 64>(__VA_ARGS__);                                          \
    default: return fail(LSG_EUNSUPPORTED, "tensor-core path: rank not in {16,32,64}"); \
  }

int launch_tc3_parts(int dtype, int rank, const Tc3PartParams& p, int tiles, cudaStream_t st) {
  if (dtype == LSG_F16) LSG_TC3_R(launch_tc3_parts_inst, __half, p, tiles, st)
  LSG_TC3_R(launch_tc3_parts_inst, __nv_bfloat16, p, tiles, st)
}

int launch_tc3_expand(int dtype, int rank, const Tc3ExpParams& p, int tiles, cudaStream_t st) {
  if (dtype == LSG_F16) LSG_TC3_R(launch_tc3_expand_inst, __half, p, tiles, st)
  LSG_TC3_R(launch_tc3_expand_inst, __nv_bfloat16, p, tiles, st)
}
#undef LSG_TC3_R

}  // namespace lsg
