// launch.cuh -- cudaLaunchKernelEx plumbing (cluster dims, programmatic
// dependent launch) and the per-mode template dispatch.  The instantiations are
// spread over inst_*.cu so the sm_100a compile parallelises.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include <string>

#include "../../include/lsg_sgmv.h"
#include "sgmv_kernels.cuh"

namespace lsg {

constexpr int kSmemBudget = 225 * 1024;     // one CTA per SM at most
constexpr int kCoresidentSmem = 74 * 1024;   // three CTAs' smem per SM (measured best: C=4 at the headline shape)
constexpr int kMaxCluster = 16;

struct Plan {
  int path = 0;  // 0 fast, 1 generic
  int mt = 1;
  int cluster = 1;
  int row_splits = 1;
  int clusters = 0;
  int nqc_max = 0;
  int ncv_max = 0;
  int smem = 0;
  int mode = kFused;
  int red_all = 0;
  int alias_ab = 0;
  int tile_scan = 0;
  int row_mode = 0;  // one cluster per row, segment found by search (one-row tiles, no long-segment skip)
  int multi = 0;     // grouped launch over several sites (row mode, fused)
  int tp = 0;        // tensor-parallel launch: row mode, output stored into every rank's y
};

// Function attributes (max dynamic smem, non-portable clusters) are per device:
// a launcher configures its kernel once for every device it runs on.
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
inline bool configured_on_device(const std::atomic<unsigned long long>& mask) {
  const int d = current_device();
  return d < 64 && (mask.load() >> d & 1ull);
}
inline void mark_configured(std::atomic<unsigned long long>& mask) {
  const int d = current_device();
  if (d < 64) mask.fetch_or(1ull << d);
}

// Set by the API layer; read at launch.
bool pdl_enabled();
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

// Per-mode entry points, defined in inst_fused.cu / inst_shrink.cu / inst_expand.cu.
int launch_fast_fused(int dtype, int rank, const FastParams& p, const Plan& pl, cudaStream_t st);
int launch_fast_shrink(int dtype, int rank, const FastParams& p, const Plan& pl, cudaStream_t st);
int launch_fast_expand(int dtype, int rank, const FastParams& p, const Plan& pl, cudaStream_t st);
int launch_generic(int dtype, int mode, const GenericParams& g, int rows, int smem, cudaStream_t st);
struct TcShrinkParams;
struct TcExpandParams;
int launch_tc_shrink(int dtype, int rank, const TcShrinkParams& p, int nq, int tiles, cudaStream_t st);
int launch_tc_expand(int dtype, int rank, const TcExpandParams& p, int tiles, cudaStream_t st);
struct TcFusedParams;
int launch_tc_fused(int dtype, const TcFusedParams& p, int C, int tiles, cudaStream_t st);
struct MmaParams;
struct StreamParams;
int launch_stream(int dtype, int rank, const StreamParams& p, int tiles, cudaStream_t st);
int launch_mma_pair(int dtype, int rank, const MmaParams& p, int tiles, cudaStream_t st);
struct Tc3PartParams;
struct Tc3ExpParams;
int launch_tc3_parts(int dtype, int rank, const Tc3PartParams& p, int tiles, cudaStream_t st);
int launch_tc3_expand(int dtype, int rank, const Tc3ExpParams& p, int tiles, cudaStream_t st);
struct Tc2Params;
int launch_tc_stream(int dtype, int rank, const Tc2Params& p, int C, uint32_t smem, int tiles, cudaStream_t st);
struct DenseLoraParams;
int launch_dense_lora(int dtype, const DenseLoraParams& p, cudaStream_t st);

template <typename K>
cudaError_t launch_ex(K kernel, dim3 grid, dim3 block, int smem, int cluster, cudaStream_t st,
                      const void* params_ptr) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  if (cluster > 0) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = static_cast<unsigned>(cluster);
    attrs[na].val.clusterDim.y = 1;
    attrs[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  void* args[] = {const_cast<void*>(params_ptr)};
  return cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(kernel), args);
}

template <typename T, int R, int MT, int MODE, int ITEM>
int launch_fast_inst(const FastParams& p, const Plan& pl, cudaStream_t st) {
  auto kern = sgmv_fast_kernel<T, R, MT, MODE, ITEM>;
  static std::atomic<unsigned long long> configured{0};  // one bit per device
  if (!configured_on_device(configured)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(max dynamic smem)");
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(non-portable cluster)");
    mark_configured(configured);
  }
  int clusters = pl.clusters;
  if (pl.tile_scan) {
    // Tile-scan grids are an upper bound on the real tile count; cap them at
    // twice the co-resident cluster count (clusters loop over further tiles).
    static int sms = 0, occ_smem = -1, occ = 1;
    if (sms == 0) {
      int dev = 0;
      sms = 148;
      if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    if (occ_smem != pl.smem) {
      int n = 1;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kThreads, pl.smem) != cudaSuccess || n < 1) n = 1;
      occ = n;
      occ_smem = pl.smem;
    }
    clusters = std::min(clusters, std::max(1, 2 * sms * occ / pl.cluster));
  }
  const dim3 grid(static_cast<unsigned>(pl.cluster), static_cast<unsigned>(clusters), 1);
  cudaError_t e = launch_ex(kern, grid, dim3(kThreads), pl.smem, pl.cluster, st, &p);
  if (e != cudaSuccess) return cuda_fail(e, "sgmv_fast_kernel launch");
  return LSG_OK;
}

template <typename T, int R, int MODE>
int dispatch_item(const FastParams& p, const Plan& pl, cudaStream_t st) {
  if (pl.mt == 1) {
    if (p.row_slot != nullptr) {
      if constexpr (MODE == kFused) return launch_fast_inst<T, R, 1, MODE, kItemBgmv>(p, pl, st);
      return fail(LSG_EINVAL, "lsg: BGMV indexing is fused-only");
    }
    if (pl.multi) {
      if constexpr (MODE == kFused) return launch_fast_inst<T, R, 1, MODE, kItemRowMulti>(p, pl, st);
      return fail(LSG_EINVAL, "lsg: grouped launches are fused-only");
    }
    if (pl.tp) {
      if constexpr (MODE == kFused) return launch_fast_inst<T, R, 1, MODE, kItemRowTp>(p, pl, st);
      return fail(LSG_EINVAL, "lsg: tensor-parallel launches are fused-only");
    }
    if (pl.row_mode) return launch_fast_inst<T, R, 1, MODE, kItemRow>(p, pl, st);
    return pl.tile_scan ? launch_fast_inst<T, R, 1, MODE, kItemTileScan>(p, pl, st)
                        : launch_fast_inst<T, R, 1, MODE, kItemRowSplit>(p, pl, st);
  }
  if (pl.multi || pl.tp) return fail(LSG_EINVAL, "lsg: grouped / tensor-parallel launches need one-row tiles");
  if (pl.mt == 4) {  // rank-64 fused launches with shared adapters (tile scan)
    if constexpr (R == 64 && MODE == kFused) return launch_fast_inst<T, R, 4, MODE, kItemTileScan>(p, pl, st);
    return fail(LSG_EINVAL, "lsg: 4-row tiles are rank-64 fused only");
  }
  // multi-row tiles always run the tile-scan decode: one tile per work item (the fp32 B of
  // a tile's expand reuses the shared memory of its A, reloaded per item)
  if (!pl.tile_scan) return fail(LSG_EINVAL, "lsg: multi-row tiles need the tile-scan decode");
  return launch_fast_inst<T, R, 8, MODE, kItemTileScan>(p, pl, st);
}

template <typename T, int MODE>
int dispatch_rank_mt(const FastParams& p, const Plan& pl, int rank, cudaStream_t st) {
#define LSG_CASE(R) \
  case R:           \
    return dispatch_item<T, R, MODE>(p, pl, st);
  switch (rank) {
    LSG_CASE(8)
    LSG_CASE(16)
    LSG_CASE(32)
    LSG_CASE(64)
  }
#undef LSG_CASE
  return fail(LSG_EUNSUPPORTED, "lsg: rank not supported by the fast path");
}

template <typename T, int MODE>
int launch_generic_inst(const GenericParams& g, int rows, int smem, cudaStream_t st) {
  auto kern = sgmv_generic_kernel<T, MODE>;
  cudaError_t e = launch_ex(kern, dim3(static_cast<unsigned>(rows)), dim3(kThreads), smem, 0, st, &g);
  if (e != cudaSuccess) return cuda_fail(e, "sgmv_generic_kernel launch");
  return LSG_OK;
}

template <typename T>
int dispatch_generic(const GenericParams& g, int mode, int rows, int smem, cudaStream_t st) {
  switch (mode) {
    case kFused: return launch_generic_inst<T, kFused>(g, rows, smem, st);
    case kShrink: return launch_generic_inst<T, kShrink>(g, rows, smem, st);
    default: return launch_generic_inst<T, kExpand>(g, rows, smem, st);
  }
}


}  // namespace lsg

#define LSG_DEFINE_FAST_ENTRY(NAME, MODE)                                                     \
  namespace lsg {                                                                             \
  int NAME(int dtype, int rank, const FastParams& p, const Plan& pl, cudaStream_t st) {       \
    return dtype == LSG_F16 ? dispatch_rank_mt<__half, MODE>(p, pl, rank, st)                \
                            : dispatch_rank_mt<__nv_bfloat16, MODE>(p, pl, rank, st);         \
  }                                                                                           \
  }
