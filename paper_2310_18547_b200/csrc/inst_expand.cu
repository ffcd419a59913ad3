// inst_expand.cu -- sm_100a instantiations of sgmv_fast_kernel<T, R, MT, kExpand>.
#include "launch.cuh"

LSG_DEFINE_FAST_ENTRY(launch_fast_expand, kExpand)
