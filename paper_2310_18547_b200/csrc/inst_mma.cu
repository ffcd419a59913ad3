// inst_mma.cu -- sm_100a instantiations of the segment-tile tensor-core pair (K7,
// sgmv_mma.cuh) and their launchers.
#include "launch.cuh"
#include "sgmv_mma.cuh"
#include "sgmv_stream.cuh"

namespace lsg {

template <typename T, int R>
static int launch_mma_inst(const MmaParams& p, int tiles, cudaStream_t st) {
  auto kp = sgmv_mma_part_kernel<T, R>;
  auto ke = sgmv_mma_exp_kernel<T, R>;
  auto kf = sgmv_mma_fused_kernel<T, R>;
  static std::atomic<unsigned long long> configured{0};  // one bit per device
  if (!configured_on_device(configured)) {
    cudaError_t e = cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(ke, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(mma pair smem)");
    mark_configured(configured);
  }
  if (p.fused) {  // one launch: a cluster of pc CTAs per tile
    const int nst = (p.h_in > p.h_out ? p.h_in : p.h_out) / p.pc / kMmaKC;
    const cudaError_t e = launch_ex(kf, dim3(static_cast<unsigned>(p.pc), static_cast<unsigned>(tiles), 1),
                                    dim3(kMmaThreads), static_cast<int>(mma_fused_smem(R, nst, p.pc)), p.pc, st, &p);
    return e == cudaSuccess ? LSG_OK : cuda_fail(e, "sgmv_mma_fused_kernel launch");
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
    // the largest shared-memory carveout, so the short-segment kernel's CTAs of the same call
    // can share an SM with a streaming CTA when its ring leaves room
    const cudaError_t e2 = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e2 != cudaSuccess) return cuda_fail(e2, "cudaFuncSetAttribute(stream carveout)");
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

}  // namespace lsg
