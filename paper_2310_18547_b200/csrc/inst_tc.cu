// inst_tc.cu -- sm_100a instantiations of the tensor-core SGMV kernel (K5) and its launcher.
#include <cuda.h>

#include "launch.cuh"
#include "sgmv_tc.cuh"

namespace lsg {

template <typename T, int R>
static int launch_tc_inst(const TcParams& p, int cluster, int tiles, cudaStream_t st) {
  auto kern = sgmv_tc_kernel<T, R>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TcLayout<R>::kTotal + 1024);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tc smem)");
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tc cluster)");
    configured = true;
  }
  const dim3 grid(static_cast<unsigned>(cluster), static_cast<unsigned>(tiles), 1);
  cudaError_t e = launch_ex(kern, grid, dim3(kTcThreads), static_cast<int>(TcLayout<R>::kTotal + 1024), cluster, st, &p);
  return e == cudaSuccess ? LSG_OK : cuda_fail(e, "sgmv_tc_kernel launch");
}

int launch_tc(int dtype, int rank, const TcParams& p, int cluster, int tiles, cudaStream_t st) {
  if (dtype == LSG_F16) {
    if (rank == 16) return launch_tc_inst<__half, 16>(p, cluster, tiles, st);
    return launch_tc_inst<__half, 32>(p, cluster, tiles, st);
  }
  if (rank == 16) return launch_tc_inst<__nv_bfloat16, 16>(p, cluster, tiles, st);
  return launch_tc_inst<__nv_bfloat16, 32>(p, cluster, tiles, st);
}

}  // namespace lsg
