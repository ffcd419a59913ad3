"""B200-native SGMV (Punica, arXiv 2310.18547): segmented multi-LoRA shrink/expand.

Native pieces (built in-tree by ``paper_2310_18547_b200.build``):
  lib/libsgmv_b200.so     sm_100a kernels behind the C-ABI include/lsg_sgmv.h
  lib/liblorasim_b200.so  C++ drop-in for the reference's lorasim::sgmv_* operators
This package is the PyTorch-facing side of the same C-ABI.
"""
from .sgmv import (AdapterPool, bgmv, build_segments, gather_rows, get_option, query_launch, scatter_rows,
                   set_option, sgmv, sgmv_expand, sgmv_multi, sgmv_shrink, dense_lora)
from . import _lib
from ._lib import (KERNEL_BGMV, KERNEL_EXPAND, KERNEL_FUSED, KERNEL_SHRINK, LSG_OPT_FORCE_CLUSTER,
                   LSG_OPT_FORCE_GENERIC, LSG_OPT_FORCE_TILE_ROWS, LSG_OPT_NO_L2_STAGING, LSG_OPT_NO_TENSOR_CORES,
                   LSG_OPT_PDL)

__all__ = ["AdapterPool", "sgmv", "sgmv_multi", "dense_lora", "sgmv_shrink", "sgmv_expand", "bgmv", "build_segments", "gather_rows",
           "scatter_rows", "set_option", "get_option", "query_launch", "KERNEL_FUSED", "KERNEL_SHRINK",
           "KERNEL_EXPAND", "KERNEL_BGMV", "LSG_OPT_PDL", "LSG_OPT_FORCE_CLUSTER", "LSG_OPT_FORCE_GENERIC",
           "LSG_OPT_FORCE_TILE_ROWS", "LSG_OPT_NO_L2_STAGING", "LSG_OPT_NO_TENSOR_CORES"]
