"""Request-partitioned multi-GPU SGMV: the host side of sharding one
decode step's batch across ranks with no collective on the data path.

The plan comes from the C-ABI (``lsg_partition_segments``, include/lsg_sgmv.h):
whole segments per rank, dominant segments cut into row ranges, LPT greedy on
algorithmic bytes.  Every rank computes the same plan from the same segment
boundaries, gathers its rows into a local batch, runs SGMV on its own GPU and
(only if the caller needs the full output on one rank) the rows are reassembled
by :func:`scatter_rows_back`.  Rows on the CUDA-core kernels (segments shorter than
the tensor-core threshold, every decode row) are a fixed function of their own row
and adapter (the kernels' canonical arithmetic), so partitioned outputs equal the
single-GPU output bit for bit there; a long (prefill) segment cut into pieces may
move between the tensor-core and CUDA-core kernels and then agrees within the
stated tolerance (include/lsg_sgmv.h, Semantics).

Reference analogue: request -> GPU placement, ``Scheduler::place``
(core/src/scheduler.cpp:12-29); row independence, sgmv.cpp:108-116, 125-134.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass
class RankBatch:
    """One rank's share of a partitioned batch."""

    rank: int
    rows: np.ndarray        # global row index of every local row, in local order (int64)
    seg_starts: np.ndarray  # local segment boundaries (int32, n_local + 1)
    segs: np.ndarray        # global segment index of every local segment (int32)

    @property
    def num_rows(self) -> int:
        return int(self.rows.size)


def partition_segments(seg_starts, h_in: int, h_out: int, rank: int, world: int, elem_bytes: int = 2,
                       seg_owner=None):
    """The plan as a list of (rank, seg, row0, row1) tuples, ordered by (rank, seg, row0).

    ``seg_owner`` (optional, one int per segment): the rank holding that segment's
    adapter in a slot-sharded pool (the segment is routed there, whole), or -1 for an
    adapter replicated on every rank."""
    b = np.ascontiguousarray(np.asarray(seg_starts, dtype=np.int32))
    n_seg = int(b.size) - 1
    if n_seg < 0:
        raise ValueError("seg_starts needs at least one entry")
    own = None
    if seg_owner is not None:
        own = np.ascontiguousarray(np.asarray(seg_owner, dtype=np.int32))
        if own.size != n_seg:
            raise ValueError("seg_owner needs one entry per segment")
    cap = n_seg + world  # the planner's bound is (non-empty segments) + world - 1
    out = (_lib.Piece * max(cap, 1))()
    n = C.c_int32(0)
    _lib.call("lsg_partition_segments", b.ctypes.data_as(C.POINTER(C.c_int32)),
              own.ctypes.data_as(C.POINTER(C.c_int32)) if own is not None else None, n_seg, h_in, h_out, rank,
              elem_bytes, world, cap, out, C.byref(n))
    return [(out[i].rank, out[i].seg, out[i].row0, out[i].row1) for i in range(n.value)]


def rank_batches(seg_starts, h_in: int, h_out: int, rank: int, world: int, elem_bytes: int = 2, seg_owner=None):
    """Per-rank local batches (list of :class:`RankBatch`, index = rank)."""
    plan = partition_segments(seg_starts, h_in, h_out, rank, world, elem_bytes, seg_owner)
    out = []
    for r in range(world):
        mine = [p for p in plan if p[0] == r]
        rows = np.concatenate([np.arange(p[2], p[3], dtype=np.int64) for p in mine]) if mine else \
            np.zeros(0, dtype=np.int64)
        lens = [p[3] - p[2] for p in mine]
        starts = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32) if mine else np.zeros(1, dtype=np.int32)
        out.append(RankBatch(r, rows, starts, np.array([p[1] for p in mine], dtype=np.int32)))
    return out


def scatter_rows_back(y_global: np.ndarray, parts) -> np.ndarray:
    """Write every rank's local output rows back to their global positions.

    ``parts`` is a list of (RankBatch, local_y) pairs; the plan covers every row
    exactly once, so the result is fully determined."""
    for rb, y_local in parts:
        y_global[rb.rows] = y_local
    return y_global


__all__ = ["RankBatch", "partition_segments", "rank_batches", "scatter_rows_back"]
