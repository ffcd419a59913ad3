"""Multi-GPU host logic on CPU: the request partitioner and the TP
expand all-gather, exercised with world_size 2 over gloo.

The product path runs the CUDA kernels on every rank; on CPU the per-rank compute
is the fp64 oracle (test infrastructure only), which is enough to prove the host
logic: the plan covers every row exactly once, per-rank batches reassemble into
the single-process result bit for bit, and the TP column shards gather into the
unsharded expand.  The GPU side of the same property (partitioned kernel output
== single-GPU kernel output, bitwise) is in tests/test_sgmv_gpu.py.
"""
from __future__ import annotations

import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import DISTINCT, IDENTICAL, SKEWED, UNIFORM
from paper_2310_18547_b200 import partition as part
from paper_2310_18547_b200 import tp as tpmod
from tests._util import oracle, random_problem, segments_for


def _bytes(rows, h_in, h_out, r, e=2):
    return rows * (h_in + h_out) * e + (h_in + h_out) * r * e


@pytest.mark.parametrize("pop", [DISTINCT, UNIFORM, SKEWED, IDENTICAL])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("batch", [1, 7, 64])
def test_plan_covers_every_row_once_and_balances(pop, world, batch):
    bounds, _, _ = segments_for(pop, batch, 11)
    h, r = 4096, 16
    plan = part.partition_segments(bounds.astype(np.int32), h, h, r, world)
    rows = np.zeros(batch, dtype=np.int64)
    loads = np.zeros(world, dtype=np.int64)
    for rank, seg, r0, r1 in plan:
        assert 0 <= rank < world
        assert bounds[seg] <= r0 < r1 <= bounds[seg + 1]  # a piece stays inside its segment
        rows[r0:r1] += 1
        loads[rank] += _bytes(r1 - r0, h, h, r)
    assert (rows == 1).all()
    assert [p[0] for p in plan] == sorted(p[0] for p in plan)  # ordered by rank
    # no two pieces of one segment on one rank (they would read the adapter twice)
    keys = [(p[0], p[1]) for p in plan]
    assert len(keys) == len(set(keys))
    total = int(loads.sum())  # split segments pay their adapter once per piece
    biggest = max(_bytes(r1 - r0, h, h, r) for _, _, r0, r1 in plan)
    assert loads.max() <= -(-total // world) + biggest  # LPT bound


def test_plan_distinct_is_exactly_even():
    plan = part.partition_segments(np.arange(65, dtype=np.int32), 4096, 4096, 16, 8)
    counts = np.bincount([p[0] for p in plan], minlength=8)
    assert (counts == 8).all()


def test_plan_identical_splits_rows():
    plan = part.partition_segments(np.array([0, 64], dtype=np.int32), 4096, 4096, 16, 4)
    assert plan == [(0, 0, 0, 16), (1, 0, 16, 32), (2, 0, 32, 48), (3, 0, 48, 64)]


def test_plan_rejects_bad_input():
    with pytest.raises(RuntimeError, match="seg_starts"):
        part.partition_segments(np.array([1, 4], dtype=np.int32), 64, 64, 8, 2)
    with pytest.raises(RuntimeError):
        part.partition_segments(np.array([0, 4, 2], dtype=np.int32), 64, 64, 8, 2)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)


def _partition_worker(rank, world, port, pop, batch):
    _init(rank, world, port)
    try:
        h_in, h_out, r = 128, 96, 8
        bounds, _, _ = segments_for(pop, batch, 5)
        x, A, B = random_problem(h_in, h_out, r, bounds, 9)
        rb = part.rank_batches(bounds.astype(np.int32), h_in, h_out, r, world)[rank]
        o = oracle()
        y_local = (o.lora_addon(x[rb.rows], rb.seg_starts.astype(np.uint64), A[rb.segs], B[rb.segs])
                   if rb.num_rows else np.zeros((0, h_out)))
        parts = [None] * world
        dist.all_gather_object(parts, (rb, y_local))
        if rank == 0:
            y = part.scatter_rows_back(np.full((batch, h_out), np.nan), parts)
            ref = o.lora_addon(x, bounds, A, B)
            assert np.array_equal(y, ref), "partitioned result differs from the single-process oracle"
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("pop", [DISTINCT, SKEWED, IDENTICAL])
def test_request_partitioned_world2_gloo_bit_exact(pop):
    mp.spawn(_partition_worker, args=(2, _free_port(), pop, 37), nprocs=2, join=True)


def _tp_worker(rank, world, port):
    _init(rank, world, port)
    try:
        h, r = 64, 8
        bounds, _, _ = segments_for(UNIFORM, 12, 3)
        x, A, B = random_problem(h, h, r, bounds, 4)
        y0 = np.random.default_rng(0).uniform(-1, 1, (12, h))
        o = oracle()
        # this rank's shard pool: A replicated, B column slice (fp64 CPU tensors, test stand-in)
        a_t = torch.tensor(A)[:, None]          # [slots, layers=1, h, r]
        b_t = torch.tensor(B)[:, None]          # [slots, layers=1, r, h]
        b_shard = tpmod.shard_b(b_t, world, rank)

        class ShardPool:  # the attributes tp_sgmv_allgather reads
            h_out = b_shard.shape[-1]

        def compute(stage, xx, pool, seg_starts, seg_slot, layer):
            stage += torch.tensor(o.lora_addon(xx.numpy(), seg_starts.numpy().astype(np.uint64),
                                               a_t[:, layer].numpy(), b_shard[:, layer].numpy()))

        y = torch.tensor(y0)
        tpmod.tp_sgmv_allgather(y, torch.tensor(x), ShardPool(), torch.tensor(bounds.astype(np.int64)),
                                torch.arange(len(bounds) - 1), 0, compute=compute)
        ref = y0 + o.lora_addon(x, bounds, A, B)
        assert np.array_equal(y.numpy(), ref), f"rank {rank}: gathered TP output differs"
    finally:
        dist.destroy_process_group()


def test_tp_expand_allgather_world2_gloo_bit_exact():
    mp.spawn(_tp_worker, args=(2, _free_port()), nprocs=2, join=True)


def test_tp_column_ranges():
    assert tpmod.column_range(8192, 8, 3) == (3072, 4096)
    with pytest.raises(ValueError):
        tpmod.column_range(100, 8, 0)


def test_plan_more_ranks_than_rows_and_empty_segments():
    # 3 rows over 8 ranks: every row placed once, idle ranks get nothing
    plan = part.partition_segments(np.array([0, 1, 3], dtype=np.int32), 64, 64, 8, 8)
    rows = sorted(r for _, _, r0, r1 in plan for r in range(r0, r1))
    assert rows == [0, 1, 2]
    # empty segments are skipped; an all-empty batch gives an empty plan
    plan = part.partition_segments(np.array([0, 0, 2, 2, 5], dtype=np.int32), 64, 64, 8, 2)
    assert {p[1] for p in plan} == {1, 3}  # (segment 3 may be split across the two ranks)
    assert part.partition_segments(np.array([0, 0, 0], dtype=np.int32), 64, 64, 8, 2) == []
    rbs = part.rank_batches(np.array([0, 0, 0], dtype=np.int32), 64, 64, 8, 2)
    assert all(rb.num_rows == 0 and rb.seg_starts.tolist() == [0] for rb in rbs)


def test_adapter_pool_layer_view_pointer_table_cpu():
    """layer_view(l) is a one-layer pool over the same storage: slot s's base pointer is
    slot s's layer-l block of the parent (checked on CPU tensors; no kernel runs)."""
    from paper_2310_18547_b200.sgmv import AdapterPool
    pool = AdapterPool(3, 5, 64, 32, 8, torch.float16, device="cpu")
    v = pool.layer_view(2)
    es = 2
    for s in range(3):
        assert int(v.a_ptrs[s]) == pool.a[s, 2].data_ptr()
        assert int(v.b_ptrs[s]) == pool.b[s, 2].data_ptr()
        assert int(v.a_ptrs[s]) - int(pool.a_ptrs[s]) == 2 * 64 * 8 * es
    assert v.num_layers == 1 and v.table.num_layers == 1 and v.table.num_slots == 3
    with pytest.raises(ValueError):
        pool.layer_view(5)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("nseg,rows", [(2, 8), (3, 8), (4, 16), (5, 2), (64, 1), (1, 64), (9, 7)])
def test_plan_piece_bound_and_cuts_only_when_they_help(world, nseg, rows):
    """Several small equal segments: the plan stays within (segments + world - 1) pieces,
    and every cut it makes lowers the largest rank load below the uncut LPT plan."""
    h, r = 4096, 16
    bounds = np.arange(nseg + 1, dtype=np.int32) * rows
    plan = part.partition_segments(bounds, h, h, r, world)
    assert len(plan) <= nseg + world - 1
    loads = np.zeros(world, dtype=np.int64)
    for rank, _, r0, r1 in plan:
        loads[rank] += _bytes(r1 - r0, h, h, r)
    # the uncut LPT makespan of equal segments: ceil(nseg / world) segments on one rank
    uncut = -(-nseg // world) * _bytes(rows, h, h, r)
    assert loads.max() <= uncut
    if len(plan) > nseg:
        assert loads.max() < uncut


def test_plan_routes_pinned_segments_to_their_owner():
    """Slot-sharded pool (configs[4]): a segment whose adapter lives on one rank goes there
    whole; replicated segments balance around them."""
    h, r = 8192, 16
    bounds = np.array([0, 1, 2, 3, 4, 40, 41, 42, 43], dtype=np.int32)
    owner = [0, 0, 0, 1, -1, 2, 3, 3]
    plan = part.partition_segments(bounds, h, h, r, 4, seg_owner=owner)
    rows = sorted(x for _, _, r0, r1 in plan for x in range(r0, r1))
    assert rows == list(range(43))
    for rank, seg, r0, r1 in plan:
        if owner[seg] >= 0:
            assert rank == owner[seg] and (r0, r1) == (bounds[seg], bounds[seg + 1])
    with pytest.raises(RuntimeError, match="seg_owner"):
        part.partition_segments(bounds, h, h, r, 2, seg_owner=owner)
    with pytest.raises(ValueError):
        part.partition_segments(bounds, h, h, r, 4, seg_owner=owner[:-1])
