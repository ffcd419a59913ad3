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
h=8192, tp=8).  NCCL is the plumbing here; the reference has no TP at all
(SPEC.md:15), its closest analogue is the per-request placement of
core/src/scheduler.cpp:12-29.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .sgmv import AdapterPool, sgmv


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


__all__ = ["column_range", "shard_b", "tp_pool", "tp_sgmv_allgather"]
