// inst_mma.cu -- sm_100a instantiations of the segment-tile tensor-core pair (K7,
// sgmv_mma.cuh) and their launchers.
#include "launch.cuh"
#include "sgmv_mma.cuh"

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
                            dim3(kMmaThreads), static_cast<int>(mma_part_smem(R, p.stages_p)), 0, st, &p);
  if (e != cudaSuccess) return cuda_fail(e, "sgmv_mma_part_kernel launch");
  e = launch_ex(ke, dim3(static_cast<unsigned>(p.ncol), static_cast<unsigned>(tiles), 1), dim3(kMmaThreads),
                static_cast<int>(mma_exp_smem(R, p.stages_e)), 0, st, &p);
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

}  // namespace lsg
