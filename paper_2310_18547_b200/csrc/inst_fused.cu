// inst_fused.cu -- sm_100a instantiations of sgmv_fast_kernel<T, R, MT, kFused>.
#include "launch.cuh"

LSG_DEFINE_FAST_ENTRY(launch_fast_fused, kFused)
