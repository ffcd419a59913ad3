"""Tensor-parallel LoRA expand with an output all-gather (BASELINE configs[4]:
Llama-2-70B, h=8192, r=16, TP over the GPUs of one node).

Layout ("Collective (70B TP only)"): every rank holds the full A of
each adapter (replicated, h x r) and the column slice B[:, c0:c1] of width
h/tp; the activations x and the output y are replicated.  A LoRA site then runs

    stage = y[:, c0:c1]                        (this rank's columns, contiguous)
    stage += x . A . B[:, c0:c1]               (the fused SGMV kernel, h_out = h/tp)
    y     = all_gather(stage) over the TP group (NCCL over NVLink)

Each output element y[j, c] is computed by exactly one rank with the same
per-element arithmetic as the unsharded kernel (the expand of column c only
reads v[j, :] and B[:, c]), so the gathered y equals the single-GPU result.

The all-gather message per rank is s_n * (h/tp) * 2 bytes (128 KiB at s_n=64,
h=8192, tp=8).  ``tp_sgmv_allgather`` is this module's torch.distributed form (NCCL through torch); the
C-ABI offers the same step natively: ``lsg_tp_sgmv_nccl`` (ncclAllGather on a caller's
communicator) and ``lsg_tp_sgmv`` (the all-gather fused into the expand epilogue: every
rank stores its columns straight into every rank's y over NVLink, then a flag exchange).
The reference has no TP at all
(SPEC.md:15), its closest analogue is the per-request placement of
core/src/scheduler.cpp:12-29.
"""
from __future__ import annotations

import ctypes as C
import glob
import os

import torch
import torch.distributed as dist

from . import _lib
from .sgmv import AdapterPool, _check_i32, _ptr, _rows_check, _stream, sgmv


def column_range(h_out: int, tp: int, rank: int) -> tuple[int, int]:
    """Columns [c0, c1) of the expand output owned by ``rank`` (h_out % tp == 0)."""
    if h_out % tp != 0:
        raise ValueError(f"h_out={h_out} is not divisible by the TP size {tp}")
    w = h_out // tp
    return rank * w, (rank + 1) * w


def shard_b(b_full: torch.Tensor, tp: int, rank: int) -> torch.Tensor:
    """This rank's column slice of B ``[slots, layers, r, h_out]`` -> ``[slots, layers, r, h_out/tp]``."""
    c0, c1 = column_range(b_full.shape[-1], tp, rank)
    return b_full[..., c0:c1].contiguous()


def tp_pool(a_full: torch.Tensor, b_full: torch.Tensor, tp: int, rank: int) -> AdapterPool:
    """Adapter pool for one TP rank: A replicated, B column-sharded (device tensors)."""
    slots, layers, h_in, r = a_full.shape
    b = shard_b(b_full, tp, rank)
    return AdapterPool(slots, layers, h_in, b.shape[-1], r, a_full.dtype, device=a_full.device,
                       a=a_full.contiguous(), b=b)


def tp_sgmv_allgather(y: torch.Tensor, x: torch.Tensor, pool: AdapterPool, seg_starts: torch.Tensor,
                      seg_slot: torch.Tensor, layer: int, group=None, compute=None) -> torch.Tensor:
    """``y += x . A . B`` with B column-sharded over the TP group, then gather y.

    ``pool`` is this rank's shard (``h_out = h / tp``).  ``compute`` (tests only)
    replaces the CUDA kernel with ``compute(stage, x, pool, seg_starts, seg_slot,
    layer)`` so the gather logic can be exercised over gloo on CPU; in production
    it is the fused SGMV kernel and there is no fallback.
    """
    tp = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    c0, c1 = column_range(y.shape[1], tp, rank)
    if pool.h_out != c1 - c0:
        raise ValueError(f"pool.h_out={pool.h_out} but this rank owns {c1 - c0} columns")
    stage = y[:, c0:c1].contiguous()
    (compute or sgmv)(stage, x, pool, seg_starts, seg_slot, layer)
    if tp == 1:
        y.copy_(stage)
        return y
    gathered = torch.empty((tp,) + tuple(stage.shape), dtype=stage.dtype, device=stage.device)
    dist.all_gather(list(gathered.unbind(0)), stage, group=group)
    y.copy_(gathered.permute(1, 0, 2).reshape(y.shape))
    return y


class TpGroup:
    """The peer buffers of one TP group as seen from one rank: every rank's y (device
    pointers valid in this process -- CUDA IPC mappings across processes, or plain
    pointers when the ranks share a device) and every rank's flag array."""

    def __init__(self, rank: int, y_peer, flag_peer):
        if not len(y_peer) == len(flag_peer) or not 1 <= len(y_peer) <= 8:
            raise ValueError("need 1..8 ranks with one y and one flag array each")
        self.rank, self.size = rank, len(y_peer)
        self._y = (C.c_void_p * self.size)(*[int(p) for p in y_peer])
        self._f = (C.c_void_p * self.size)(*[int(p) for p in flag_peer])
        self.c = _lib.TpGroup(rank, self.size, self._y, self._f)
        self.epoch = 0


def tp_sgmv_p2p(group: TpGroup, y: torch.Tensor, x: torch.Tensor, shard: AdapterPool, seg_starts: torch.Tensor,
                seg_slot: torch.Tensor, layer: int, num_segments: int | None = None) -> torch.Tensor:
    """``y += x . A . B`` with B column-sharded over the TP group, the all-gather fused into
    the expand epilogue (lsg_tp_sgmv): this rank's columns are stored into every rank's y,
    then a flag exchange; on stream completion every rank's y is complete.  ``y`` is this
    rank's own y (``group``'s y_peer[rank])."""
    _rows_check(x, None, shard)
    _check_i32(seg_starts, "seg_starts")
    _check_i32(seg_slot, "seg_slot")
    if y.shape[1] != shard.h_out * group.size or y.data_ptr() != group._y[group.rank]:
        raise ValueError("y must be this rank's registered y with size * h_out columns")
    group.epoch += 1
    n = seg_slot.numel() if num_segments is None else num_segments
    _lib.call("lsg_tp_sgmv", C.byref(group.c), y.stride(0), _ptr(x), x.stride(0), C.byref(shard.table),
              _ptr(seg_starts), _ptr(seg_slot), n, x.shape[0], layer, group.epoch, _stream())
    return y


def tp_sgmv_nccl(y: torch.Tensor, x: torch.Tensor, shard: AdapterPool, seg_starts: torch.Tensor,
                 seg_slot: torch.Tensor, layer: int, tp_rank: int, tp_size: int, nccl_comm: int,
                 num_segments: int | None = None) -> torch.Tensor:
    """The NCCL baseline through the C-ABI (lsg_tp_sgmv_nccl): this rank's columns in place,
    then ncclAllGather on ``nccl_comm`` (an ncclComm_t handle)."""
    _rows_check(x, None, shard)
    n = seg_slot.numel() if num_segments is None else num_segments
    wsb = int(_lib.lib().lsg_tp_nccl_workspace_size(x.shape[0], shard.h_out, tp_size))
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=x.device)
    _lib.call("lsg_tp_sgmv_nccl", _ptr(y), y.stride(0), _ptr(x), x.stride(0), C.byref(shard.table), _ptr(seg_starts),
              _ptr(seg_slot), n, x.shape[0], layer, tp_rank, tp_size, C.c_void_p(nccl_comm), _ptr(ws), ws.numel(),
              _stream())
    return y


def nccl_library() -> C.CDLL:
    """libnccl.so.2 (the copy torch ships, else the system one)."""
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "nccl", "lib", "libnccl.so*"))
    for p in cands + ["libnccl.so.2"]:
        try:
            return C.CDLL(p, mode=C.RTLD_GLOBAL)
        except OSError:
            continue
    raise RuntimeError("libnccl.so.2 not found")


class _NcclUniqueId(C.Structure):
    _fields_ = [("internal", C.c_char * 128)]  # ncclUniqueId (nccl.h): passed BY VALUE to ncclCommInitRank


def nccl_comm_single() -> int:
    """A one-rank ncclComm_t (tests of the NCCL plumbing on one GPU)."""
    L = nccl_library()
    uid = _NcclUniqueId()
    L.ncclGetUniqueId.argtypes = [C.POINTER(_NcclUniqueId)]
    if L.ncclGetUniqueId(C.byref(uid)) != 0:
        raise RuntimeError("ncclGetUniqueId failed")
    comm = C.c_void_p()
    L.ncclCommInitRank.argtypes = [C.POINTER(C.c_void_p), C.c_int, _NcclUniqueId, C.c_int]
    rc = L.ncclCommInitRank(C.byref(comm), 1, uid, 0)
    if rc != 0:
        L.ncclGetErrorString.restype = C.c_char_p
        raise RuntimeError(f"ncclCommInitRank failed ({rc}: {L.ncclGetErrorString(rc).decode()})")
    return comm.value


__all__ = ["column_range", "shard_b", "tp_pool", "tp_sgmv_allgather", "TpGroup", "tp_sgmv_p2p", "tp_sgmv_nccl",
           "nccl_comm_single"]
