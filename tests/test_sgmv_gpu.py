"""GPU parity tests: the sm_100a kernels (through the C-ABI) against the CPU oracle.

Mirrors the reference's SGMV tests (proj/tests/unit/test_sgmv.cpp,
test_experiments.cpp) plus the kernel-level invariants the B200 design adds
(cluster-size / tile-size / kernel-variant independence, bitwise).
"""
from __future__ import annotations

import json
import sys
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from tests._util import (DISTINCT, IDENTICAL, NORTH_STAR_TOL, SKEWED, TOL, UNIFORM, builder_model, oracle,
                         plan_batch_rows, random_problem, row_norm_err, segments_for)

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
DTYPES = [torch.float16, torch.bfloat16]


@pytest.fixture(scope="module")
def lsg():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2310_18547_b200 as m
    m.set_option(m.LSG_OPT_PDL, 0)
    return m


@pytest.fixture(autouse=True)
def _reset_options(lsg):
    yield
    for opt in (lsg.LSG_OPT_FORCE_CLUSTER, lsg.LSG_OPT_FORCE_GENERIC, lsg.LSG_OPT_FORCE_TILE_ROWS, lsg.LSG_OPT_PDL,
                lsg.LSG_OPT_NO_TENSOR_CORES, lsg._lib.LSG_OPT_TC_SPLIT, lsg._lib.LSG_OPT_NO_ROW_MODE,
                lsg._lib.LSG_OPT_TC_MIN_ROWS, lsg._lib.LSG_OPT_NO_MULTIROW_TILES, lsg._lib.LSG_OPT_TC_LEGACY, lsg._lib.LSG_OPT_MMA_MIN_ROWS,
                lsg._lib.LSG_OPT_MMA_FUSED):
        lsg.set_option(opt, 0)


class Problem:
    """One segmented batch, quantised for the GPU, dequantised for the oracle."""

    def __init__(self, lsg, x, A, B, bounds, dtype, slots=None, num_slots=None, layers=1, layer=0, y0=None):
        self.lsg, self.dtype = lsg, dtype
        nseg = len(bounds) - 1
        self.rank, self.h_in, self.h_out = B.shape[1], x.shape[1], B.shape[2]
        self.slots = list(range(nseg)) if slots is None else list(slots)
        ns = num_slots if num_slots is not None else max(self.slots + [nseg - 1]) + 1
        self.pool = lsg.AdapterPool(ns, layers, self.h_in, self.h_out, self.rank, dtype)
        self.x = torch.tensor(x, dtype=torch.float64).to(dtype).cuda()
        Aq = torch.tensor(A, dtype=torch.float64).to(dtype)
        Bq = torch.tensor(B, dtype=torch.float64).to(dtype)
        for s, slot in enumerate(self.slots):
            if slot >= 0:
                self.pool.a[slot, layer].copy_(Aq[s])
                self.pool.b[slot, layer].copy_(Bq[s])
        self.layer = layer
        self.bounds = np.asarray(bounds, dtype=np.uint64)
        self.seg_starts = torch.tensor(self.bounds.astype(np.int64), dtype=torch.int32, device="cuda")
        self.seg_slot = torch.tensor(self.slots, dtype=torch.int32, device="cuda")
        self.xd, self.Ad, self.Bd = self.x.double().cpu().numpy(), Aq.double().numpy(), Bq.double().numpy()
        rows = int(self.bounds[-1]) if nseg else 0
        self.y0 = (torch.zeros(rows, self.h_out, dtype=dtype, device="cuda") if y0 is None
                   else torch.tensor(y0, dtype=torch.float64).to(dtype).cuda())

    def run(self, kind="fused"):
        lsg = self.lsg
        y = self.y0.clone()
        if kind == "fused":
            lsg.sgmv(y, self.x, self.pool, self.seg_starts, self.seg_slot, self.layer)
        elif kind == "two_launch":
            v = torch.empty(self.x.shape[0], self.rank, dtype=torch.float32, device="cuda")
            lsg.sgmv_shrink(v, self.x, self.pool, self.seg_starts, self.seg_slot, self.layer)
            lsg.sgmv_expand(y, v, self.pool, self.seg_starts, self.seg_slot, self.layer)
        elif kind == "bgmv":
            row_slot = np.zeros(self.x.shape[0], dtype=np.int32)
            for s in range(len(self.bounds) - 1):
                row_slot[int(self.bounds[s]):int(self.bounds[s + 1])] = self.slots[s]
            lsg.bgmv(y, self.x, self.pool, torch.tensor(row_slot, device="cuda"), self.layer)
        torch.cuda.synchronize()
        return y

    def reference(self):
        valid = [s >= 0 for s in self.slots]
        y = self.y0.double().cpu().numpy().copy()
        if len(self.bounds) > 1:
            add = oracle().lora_addon(self.xd, self.bounds, self.Ad, self.Bd)
            for s, ok in enumerate(valid):
                a, b = int(self.bounds[s]), int(self.bounds[s + 1])
                if ok:
                    y[a:b] += add[a:b]
        return y


def tol(dtype):
    return TOL[str(dtype).split(".")[-1]]


# ---------------------------------------------------------------------------------
# Known-answer tests (test_sgmv.cpp:83-122; values produced by the reference)
# ---------------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", DTYPES)
def test_hand_checked_two_segment_exact(lsg, dtype):
    kat = json.load(open(os.path.join(GOLDEN, "kat.json")))["two_segment"]
    p = Problem(lsg, np.array(kat["x"]), np.array(kat["A"]), np.array(kat["B"]), kat["bounds"], dtype)
    for kind in ("fused", "two_launch", "bgmv"):
        y = p.run(kind).double().cpu().numpy()
        assert np.array_equal(y, np.array(kat["lora_addon"])), kind  # [[5,1],[11,3],[16,54]]


@pytest.mark.parametrize("dtype", DTYPES)
def test_rank1_and_zero_weights_exact(lsg, dtype):
    kat = json.load(open(os.path.join(GOLDEN, "kat.json")))["rank1"]
    p = Problem(lsg, np.array(kat["x"]), np.array(kat["A"]), np.array(kat["B"]), kat["bounds"], dtype)
    assert np.array_equal(p.run().double().cpu().numpy(), np.array(kat["lora_addon"]))  # [[3, 3]]
    x, _, _ = random_problem(8, 8, 2, [0, 4], 11)
    pz = Problem(lsg, x, np.zeros((1, 8, 2)), np.zeros((1, 2, 8)), [0, 4], dtype)
    assert torch.count_nonzero(pz.run()).item() == 0


def test_empty_batch_is_noop(lsg):
    pool = lsg.AdapterPool(1, 1, 128, 128, 16, torch.float16)
    x = torch.empty(0, 128, dtype=torch.float16, device="cuda")
    y = torch.empty(0, 128, dtype=torch.float16, device="cuda")
    z = torch.zeros(1, dtype=torch.int32, device="cuda")
    lsg.sgmv(y, x, pool, z, z[:0], 0)
    torch.cuda.synchronize()


# ---------------------------------------------------------------------------------
# Randomised parity: verify_sgmv's shape distribution (experiments.cpp:35-102)
# ---------------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", DTYPES)
def test_verify_sgmv_trials_match_oracle(lsg, dtype):
    o = oracle()
    g = o.rng(o.derive_seed(42, 17))
    worst = 0.0
    for t in range(200):
        tr = g.verify_next_trial(t)
        p = Problem(lsg, tr["x"], tr["A"], tr["B"], tr["bounds"], dtype)
        yref = p.reference()
        for kind in ("fused", "two_launch", "bgmv"):
            err = row_norm_err(p.run(kind).double().cpu().numpy(), yref)
            worst = max(worst, err)
            assert err <= tol(dtype), (t, kind, err)
    assert worst <= NORTH_STAR_TOL


SHAPES = [  # (h_in, h_out, rank) at the BASELINE configs and rank sweep
    (4096, 4096, 16), (4096, 4096, 8), (4096, 4096, 32), (4096, 4096, 64), (5120, 5120, 64), (8192, 8192, 16)]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("pop", [DISTINCT, UNIFORM, SKEWED, IDENTICAL])
def test_baseline_shapes_match_oracle(lsg, dtype, shape, pop):
    h_in, h_out, r = shape
    bounds, _, _ = segments_for(pop, 64, 1234 + pop)
    x, A, B = random_problem(h_in, h_out, r, bounds, 77 + pop)
    p = Problem(lsg, x, A, B, bounds, dtype)
    y = p.run()
    # the fast (cluster) path, or for rank 64 with shared adapters the segment-tile MMA pair
    assert lsg.query_launch(p.pool, len(bounds) - 1, 64)["path"] == (2 if r == 64 and pop != DISTINCT else 0)
    err = row_norm_err(y.double().cpu().numpy(), p.reference())
    assert err <= tol(dtype), err


@pytest.mark.parametrize("dtype", [torch.float16])
@pytest.mark.parametrize("batch", [1, 2, 7, 32])
def test_small_batches_and_accumulate(lsg, dtype, batch):
    bounds, _, _ = segments_for(UNIFORM, batch, 5)
    x, A, B = random_problem(4096, 4096, 16, bounds, batch)
    y0 = oracle().rng(99).fill_pm1(batch * 4096).reshape(batch, 4096)
    p = Problem(lsg, x, A, B, bounds, dtype, y0=y0)
    err = row_norm_err(p.run().double().cpu().numpy(), p.reference())
    assert err <= tol(dtype), err


@pytest.mark.parametrize("prefill", [128, 512])
def test_mixed_prefill_plus_decodes(lsg, prefill):
    bounds = np.array([0, prefill] + [prefill + i + 1 for i in range(31)], dtype=np.uint64)
    x, A, B = random_problem(4096, 4096, 16, bounds, prefill)
    p = Problem(lsg, x, A, B, bounds, torch.float16)
    err = row_norm_err(p.run().double().cpu().numpy(), p.reference())
    assert err <= tol(torch.float16), err


# ---------------------------------------------------------------------------------
# Long segments: the tcgen05 path (segments >= 128 rows, r in {16, 32}, h % 512 == 0)
# ---------------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("shape", [(4096, 4096, 16), (4096, 4096, 32), (4096, 4096, 64), (5120, 5120, 16),
                                   (8192, 8192, 32), (1024, 1024, 16), (4096, 11008, 16), (11008, 4096, 16)])
@pytest.mark.parametrize("lens", [(128,), (129, 3, 1, 255), (1, 700, 5, 2048, 1, 1)])
def test_long_segments_tensor_core_path(lsg, dtype, shape, lens):
    h_in, h_out, r = shape
    bounds = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    x, A, B = random_problem(h_in, h_out, r, bounds, 5 + len(lens))
    y0 = oracle().rng(123).fill_pm1(int(bounds[-1]) * h_out).reshape(-1, h_out)
    p = Problem(lsg, x, A, B, bounds, dtype, y0=y0)
    got = p.run()
    err = row_norm_err(got.double().cpu().numpy(), p.reference())
    assert err <= tol(dtype), err
    lsg.set_option(lsg.LSG_OPT_NO_TENSOR_CORES, 1)
    try:
        cc = p.run()
    finally:
        lsg.set_option(lsg.LSG_OPT_NO_TENSOR_CORES, 0)
    # short segments take the CUDA-core kernel in both runs: bit-identical there (rank 64 with
    # shared rows sends them to the segment-tile MMA pair instead: within tolerance)
    assert row_norm_err(cc.double().cpu().numpy(), p.reference()) <= tol(dtype)
    for s, n in enumerate(lens):
        a, b = int(bounds[s]), int(bounds[s + 1])
        if n < 128 and r != 64:
            assert torch.equal(got[a:b], cc[a:b]), s
    assert torch.equal(p.run(), got)  # run-to-run deterministic
    if r == 16:  # rank 16 runs the fused kernel by default: the two-kernel form must agree too
        lsg.set_option(lsg._lib.LSG_OPT_TC_SPLIT, 1)
        try:
            split = p.run()
        finally:
            lsg.set_option(lsg._lib.LSG_OPT_TC_SPLIT, 0)
        assert row_norm_err(split.double().cpu().numpy(), p.reference()) <= tol(dtype)
        for s, n in enumerate(lens):
            a, b = int(bounds[s]), int(bounds[s + 1])
            if n < 128:
                assert torch.equal(split[a:b], got[a:b]), s


def test_long_segment_no_adapter_slot_untouched(lsg):
    bounds = np.array([0, 300, 301, 600], dtype=np.uint64)
    x, A, B = random_problem(4096, 4096, 16, bounds, 31)
    y0 = oracle().rng(7).fill_pm1(600 * 4096).reshape(600, 4096)
    p = Problem(lsg, x, A, B, bounds, torch.float16, slots=[0, 1, -1], num_slots=2, y0=y0)
    got = p.run()
    assert torch.equal(got[301:], p.y0[301:])
    err = row_norm_err(got.double().cpu().numpy(), p.reference())
    assert err <= tol(torch.float16), err


# ---------------------------------------------------------------------------------
# Determinism / invariance (bitwise)
# ---------------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", DTYPES)
def test_kernel_variants_and_cluster_sizes_bitwise_identical(lsg, dtype):
    bounds, _, _ = segments_for(SKEWED, 64, 3)
    x, A, B = random_problem(4096, 4096, 16, bounds, 4)
    p = Problem(lsg, x, A, B, bounds, dtype)
    base = p.run("fused")
    for kind in ("two_launch", "bgmv"):
        assert torch.equal(p.run(kind), base), kind
    for c in (1, 2, 3, 4, 8, 16):
        lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, c)
        for mt in (1, 8):
            lsg.set_option(lsg.LSG_OPT_FORCE_TILE_ROWS, mt)
            assert torch.equal(p.run("fused"), base), (c, mt)
            assert torch.equal(p.run("two_launch"), base), (c, mt)
    lsg.set_option(lsg.LSG_OPT_PDL, 1)
    lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, 0)
    lsg.set_option(lsg.LSG_OPT_FORCE_TILE_ROWS, 0)
    assert torch.equal(p.run("fused"), base)


@pytest.mark.parametrize("dtype", DTYPES)
def test_many_medium_segments_bitwise_across_variants(lsg, dtype):
    """Thousands of row tiles (more than the capped tile-scan grid): clusters loop
    over several tiles; results stay bitwise equal to the one-row-per-cluster BGMV."""
    lens = [(37 * i) % 127 + 1 for i in range(70)]
    bounds = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    x, A, B = random_problem(4096, 4096, 16, bounds, 21)
    p = Problem(lsg, x, A, B, bounds, dtype)
    base = p.run("fused")
    err = row_norm_err(base.double().cpu().numpy(), p.reference())
    assert err <= tol(dtype), err
    assert torch.equal(p.run("bgmv"), base)
    assert torch.equal(p.run("two_launch"), base)
    for c in (2, 16):
        lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, c)
        assert torch.equal(p.run("fused"), base), c


def test_segment_permutation_permutes_rows_bitwise(lsg):
    """test_sgmv.cpp:171-197 on the GPU: swapping segments moves rows, bit for bit."""
    bounds, _, _ = segments_for(UNIFORM, 40, 8)
    x, A, B = random_problem(4096, 4096, 16, bounds, 9)
    p = Problem(lsg, x, A, B, bounds, torch.float16)
    base = p.run().cpu().numpy()
    nseg = len(bounds) - 1
    order = list(reversed(range(nseg)))
    xs, nb, src_rows = [], [0], []
    for s in order:
        a, b = int(bounds[s]), int(bounds[s + 1])
        xs.append(x[a:b])
        nb.append(nb[-1] + b - a)
        src_rows.extend(range(a, b))
    q = Problem(lsg, np.concatenate(xs), A[order], B[order], nb, torch.float16)
    got = q.run().cpu().numpy()
    assert np.array_equal(got.view(np.uint16), base[src_rows].view(np.uint16))


def test_no_adapter_rows_untouched_and_slot_indirection(lsg):
    bounds = np.array([0, 3, 5, 9], dtype=np.uint64)
    x, A, B = random_problem(4096, 4096, 16, bounds, 21)
    y0 = oracle().rng(22).fill_pm1(9 * 4096).reshape(9, 4096)
    p = Problem(lsg, x, A, B, bounds, torch.float16, slots=[5, -1, 2], num_slots=7, layers=3, layer=2, y0=y0)
    y = p.run()
    assert torch.equal(y[3:5], p.y0[3:5])
    assert row_norm_err(y.double().cpu().numpy(), p.reference()) <= tol(torch.float16)


@pytest.mark.parametrize("shape", [(2, 2, 1), (64, 48, 8), (136, 1000, 16), (4096, 4096, 12), (96, 40, 40)])
def test_generic_path_odd_shapes(lsg, shape):
    h_in, h_out, r = shape
    bounds, _, _ = segments_for(SKEWED, 20, 1)
    x, A, B = random_problem(h_in, h_out, r, bounds, 2)
    p = Problem(lsg, x, A, B, bounds, torch.float16)
    err = row_norm_err(p.run().double().cpu().numpy(), p.reference())
    assert err <= tol(torch.float16), err


def test_generic_and_unaligned_rows(lsg):
    bounds, _, _ = segments_for(DISTINCT, 8, 1)
    x, A, B = random_problem(4096, 4096, 16, bounds, 2)
    p = Problem(lsg, x, A, B, bounds, torch.float16)
    yref = p.reference()
    lsg.set_option(lsg.LSG_OPT_FORCE_GENERIC, 1)
    assert row_norm_err(p.run().double().cpu().numpy(), yref) <= tol(torch.float16)
    lsg.set_option(lsg.LSG_OPT_FORCE_GENERIC, 0)
    # x viewed with an odd row stride -> not 16-byte aligned -> generic path, same tolerance
    xb = torch.zeros(8, 4096 + 3, dtype=torch.float16, device="cuda")
    xb[:, 1:4097] = p.x
    y = torch.zeros(8, 4096, dtype=torch.float16, device="cuda")
    lsg.sgmv(y, xb[:, 1:4097], p.pool, p.seg_starts, p.seg_slot, 0)
    torch.cuda.synchronize()
    assert row_norm_err(y.double().cpu().numpy(), yref) <= tol(torch.float16)


def test_invalid_arguments_raise(lsg):
    from paper_2310_18547_b200._lib import LsgError
    pool = lsg.AdapterPool(2, 1, 128, 128, 16, torch.float16)
    x = torch.zeros(4, 128, dtype=torch.float16, device="cuda")
    y = torch.zeros(4, 128, dtype=torch.float16, device="cuda")
    ss = torch.tensor([0, 4], dtype=torch.int32, device="cuda")
    sl = torch.tensor([0], dtype=torch.int32, device="cuda")
    with pytest.raises(LsgError, match="layer"):
        lsg.sgmv(y, x, pool, ss, sl, 3)
    with pytest.raises(ValueError):
        lsg.sgmv(y.float(), x, pool, ss, sl, 0)


# ---------------------------------------------------------------------------------
# K6: on-device segment builder
# ---------------------------------------------------------------------------------
@pytest.mark.parametrize("n,num_slots", [(1, 4), (9, 3), (64, 64), (64, 8), (333, 40), (2079, 1000), (16384, 7)])
def test_build_segments_matches_host_grouping(lsg, n, num_slots):
    rs = np.random.default_rng(n).integers(-1, num_slots + 1, n).astype(np.int32)
    lead = int(rs[n // 2])
    lead_rows = (n // 2, min(n, n // 2 + 5))  # a "prefill" range in the middle of the batch
    rs[lead_rows[0]:lead_rows[1]] = lead
    perm, starts, slots = builder_model(rs.tolist(), num_slots, lead, lead_rows)
    row_perm, seg_starts, seg_slot, nseg = lsg.build_segments(torch.tensor(rs, device="cuda"), num_slots, lead,
                                                              lead_rows)
    k = int(nseg.item())
    assert k == len(slots)
    assert row_perm.cpu().tolist() == perm
    assert seg_starts.cpu().tolist()[: k + 1] == starts
    assert seg_slot.cpu().tolist()[:k] == slots
    assert all(v == n for v in seg_starts.cpu().tolist()[k + 1:])


def test_build_segments_reproduces_plan_batch_golden(lsg):
    """plan_batch layouts (simulator.cpp:239-311) from the reference, slots = LoraId rank:
    segment bounds, segment adapters AND the row order (prefill prompt rows first, then the
    decodes in plan_batch's `decodes` order) for all golden cases."""
    cases = json.load(open(os.path.join(GOLDEN, "plan_batch.json")))
    assert len(cases) == 21
    for ci, case in enumerate(cases):
        lora, done, prompt = case["lora"], case["done"], case["prompt"]
        plan = case["plan"]
        uniq, rows, req_of_row, lead, lead_rows = plan_batch_rows(case)
        row_perm, seg_starts, seg_slot, nseg = lsg.build_segments(
            torch.tensor(rows, dtype=torch.int32, device="cuda"), len(uniq), lead, lead_rows)
        k = int(nseg.item())
        assert seg_starts.cpu().tolist()[: k + 1] == plan["bounds"], ci
        assert [uniq[s] for s in seg_slot.cpu().tolist()[:k]] == plan["loras"], ci
        order = []
        for r in row_perm.cpu().tolist():  # request order implied by the gathered rows
            if not order or order[-1] != req_of_row[r]:
                order.append(req_of_row[r])
        expect = ([plan["prefill"]] if plan["prefill"] >= 0 else []) + plan["decodes"]
        assert order == expect, (ci, order, expect)


def test_builder_feeds_sgmv_without_host_readback(lsg):
    n, ns = 64, 10
    rs = torch.tensor(np.random.default_rng(3).integers(0, ns, n).astype(np.int32), device="cuda")
    pool = lsg.AdapterPool(ns, 1, 4096, 4096, 16, torch.float16)
    torch.manual_seed(0)
    pool.a.uniform_(-1, 1)
    pool.b.uniform_(-1, 1)
    x = torch.empty(n, 4096, dtype=torch.float16, device="cuda").uniform_(-1, 1)
    row_perm, seg_starts, seg_slot, _ = lsg.build_segments(rs, ns)
    xg = torch.empty_like(x)
    lsg.gather_rows(xg, x, row_perm)
    yg = torch.zeros_like(x)
    lsg.sgmv(yg, xg, pool, seg_starts, seg_slot, 0, num_segments=ns)  # host bound, not the true count
    y = torch.zeros_like(x)
    lsg.scatter_rows(y, yg, row_perm)
    yb = torch.zeros_like(x)
    lsg.bgmv(yb, x, pool, rs, 0)
    torch.cuda.synchronize()
    assert torch.equal(y, yb)


# ---------------------------------------------------------------------------------
# Multi-GPU data paths, emulated rank by rank on one GPU
# ---------------------------------------------------------------------------------
@pytest.mark.parametrize("pop", [DISTINCT, SKEWED, IDENTICAL])
@pytest.mark.parametrize("world", [2, 8])
def test_request_partitioned_kernel_equals_single_gpu_bitwise(lsg, pop, world):
    """Every rank's local batch (lsg_partition_segments) run by the kernel, rows
    scattered back: equal to the one-launch result bit for bit."""
    from paper_2310_18547_b200 import partition as part
    bounds, _, _ = segments_for(pop, 64, 17)
    x, A, B = random_problem(4096, 4096, 16, bounds, 18)
    p = Problem(lsg, x, A, B, bounds, torch.float16)
    base = p.run()
    y = torch.full_like(base, float("nan"))
    for rb in part.rank_batches(bounds.astype(np.int32), 4096, 4096, 16, world):
        if rb.num_rows == 0:
            continue
        rows = torch.tensor(rb.rows, device="cuda")
        yl = p.y0[rows].clone()
        lsg.sgmv(yl, p.x[rows].contiguous(), p.pool, torch.tensor(rb.seg_starts, device="cuda"),
                 torch.tensor(rb.segs, device="cuda"), 0)  # slot s == global segment s in this problem
        y[rows] = yl
    torch.cuda.synchronize()
    assert torch.equal(y, base)


@pytest.mark.parametrize("tp", [2, 4, 8])
def test_tp_column_shards_equal_unsharded_bitwise(lsg, tp):
    """70B-style TP expand: each rank's column-slice launch (B sharded, A replicated)
    produces exactly the matching columns of the unsharded launch."""
    from paper_2310_18547_b200 import tp as tpmod
    h, r = 8192, 16
    bounds, _, _ = segments_for(DISTINCT, 16, 2)
    x, A, B = random_problem(h, h, r, bounds, 3)
    y0 = oracle().rng(4).fill_pm1(16 * h).reshape(16, h)
    p = Problem(lsg, x, A, B, bounds, torch.bfloat16, y0=y0)
    base = p.run()
    for rank in range(tp):
        pool = tpmod.tp_pool(p.pool.a, p.pool.b, tp, rank)
        c0, c1 = tpmod.column_range(h, tp, rank)
        stage = p.y0[:, c0:c1].contiguous()
        lsg.sgmv(stage, p.x, pool, p.seg_starts, p.seg_slot, 0)
        torch.cuda.synchronize()
        assert torch.equal(stage, base[:, c0:c1]), rank
    # world-size-1 call of the public TP entry point (no collective) is the plain launch
    y = p.y0.clone()
    tpmod.tp_sgmv_allgather(y, p.x, tpmod.tp_pool(p.pool.a, p.pool.b, 1, 0), p.seg_starts, p.seg_slot, 0)
    torch.cuda.synchronize()
    assert torch.equal(y, base)


@pytest.mark.parametrize("row_mode", [0, 1])
def test_empty_segments_anywhere(lsg, row_mode):
    """Empty segments (equal boundaries) at the start, middle and end: the row-mode
    segment search and the segment-major decode give the same, correct rows."""
    lens = [0, 3, 0, 0, 2, 1, 0, 4, 0]
    bounds = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    x, A, B = random_problem(4096, 4096, 16, bounds, 31)
    lsg.set_option(lsg._lib.LSG_OPT_NO_ROW_MODE, 1 - row_mode)
    try:
        p = Problem(lsg, x, A, B, bounds, torch.float16)
        y = p.run()
        keep = [s for s in range(len(lens)) if lens[s] > 0]  # the reference's Segments are non-empty
        cb = np.concatenate([[0], np.cumsum([lens[s] for s in keep])]).astype(np.uint64)
        ref = oracle().lora_addon(p.xd, cb, p.Ad[keep], p.Bd[keep])
        assert row_norm_err(y.double().cpu().numpy(), ref) <= tol(torch.float16)
        lsg.set_option(lsg._lib.LSG_OPT_NO_ROW_MODE, row_mode)
        assert torch.equal(p.run(), y)
    finally:
        lsg.set_option(lsg._lib.LSG_OPT_NO_ROW_MODE, 0)


@pytest.mark.parametrize("pop", [DISTINCT, SKEWED, IDENTICAL])
@pytest.mark.parametrize("nsites", [2, 3, 8])
def test_grouped_sites_equal_per_site_calls_bitwise(lsg, pop, nsites):
    """lsg_sgmv_multi (one launch for several sites sharing the segment plan) is bitwise
    the per-site lsg_sgmv calls; each site uses its own pool, x and y."""
    bounds, _, _ = segments_for(pop, 48, 40 + nsites)
    probs = []
    for i in range(nsites):
        x, A, B = random_problem(4096, 4096, 16, bounds, 60 + i)
        y0 = oracle().rng(70 + i).fill_pm1(48 * 4096).reshape(48, 4096)
        probs.append(Problem(lsg, x, A, B, bounds, torch.float16, y0=y0))
    ref = [p.run() for p in probs]
    ys = [p.y0.clone() for p in probs]
    lsg.sgmv_multi(ys, [p.x for p in probs], [p.pool for p in probs], probs[0].seg_starts, probs[0].seg_slot, 0)
    torch.cuda.synchronize()
    for i in range(nsites):
        assert torch.equal(ys[i], ref[i]), i


def test_grouped_sites_fall_back_with_long_segments(lsg):
    """A long (tensor-core) segment makes the grouped call run site by site: same results."""
    bounds = np.array([0, 200, 203, 210], dtype=np.uint64)
    probs = []
    for i in range(3):
        x, A, B = random_problem(4096, 4096, 16, bounds, 80 + i)
        probs.append(Problem(lsg, x, A, B, bounds, torch.bfloat16))
    ref = [p.run() for p in probs]
    ys = [p.y0.clone() for p in probs]
    lsg.sgmv_multi(ys, [p.x for p in probs], [p.pool for p in probs], probs[0].seg_starts, probs[0].seg_slot, 0)
    torch.cuda.synchronize()
    for i in range(3):
        assert torch.equal(ys[i], ref[i]), i
        assert row_norm_err(ys[i].double().cpu().numpy(), probs[i].reference()) <= tol(torch.bfloat16)


NO_MMA = 1 << 30  # LSG_OPT_MMA_MIN_ROWS value that keeps every segment off the MMA pair


@pytest.mark.parametrize("h", [4096, 8192])
def test_rank64_multirow_tiles_large_hidden(lsg, h):
    """Rank 64 with shared adapters: the default MMA pair, and (MMA pair off) the CUDA-core
    multi-row tiles, which at h = 8192 need a cluster above the tile-row cap to fit shared
    memory -- both correct, the CUDA-core tiles bitwise the one-row result."""
    bounds, _, _ = segments_for(UNIFORM, 32, 93)
    x, A, B = random_problem(h, h, 64, bounds, 94)
    p = Problem(lsg, x, A, B, bounds, torch.bfloat16)
    mma = p.run()
    assert row_norm_err(mma.double().cpu().numpy(), p.reference()) <= tol(torch.bfloat16)
    lsg.set_option(lsg._lib.LSG_OPT_MMA_MIN_ROWS, NO_MMA)
    base = p.run()
    assert row_norm_err(base.double().cpu().numpy(), p.reference()) <= tol(torch.bfloat16)
    lsg.set_option(lsg.LSG_OPT_FORCE_TILE_ROWS, 1)
    assert torch.equal(p.run(), base)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("pop", [UNIFORM, SKEWED])
def test_rank64_multirow_tiles_bitwise_one_row(lsg, dtype, pop):
    """Rank 64 with shared adapters on the CUDA-core kernel (MMA pair off) runs 8-row tiles
    (one weight read per tile): bitwise the one-row-per-cluster result, for every cluster size."""
    bounds, _, _ = segments_for(pop, 64, 91)
    x, A, B = random_problem(5120, 5120, 64, bounds, 92)
    p = Problem(lsg, x, A, B, bounds, dtype)
    lsg.set_option(lsg._lib.LSG_OPT_MMA_MIN_ROWS, NO_MMA)
    base = p.run()
    assert row_norm_err(base.double().cpu().numpy(), p.reference()) <= tol(dtype)
    lsg.set_option(lsg.LSG_OPT_FORCE_TILE_ROWS, 1)
    assert torch.equal(p.run(), base)
    lsg.set_option(lsg.LSG_OPT_FORCE_TILE_ROWS, 8)
    for c in (4, 8, 16):
        lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, c)
        assert torch.equal(p.run(), base), c
        assert torch.equal(p.run("two_launch"), base), c


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("pop,batch,h_in,h_out", [(DISTINCT, 64, 4096, 2048), (UNIFORM, 37, 4096, 2048),
                                                   (IDENTICAL, 8, 4096, 2048), (DISTINCT, 64, 1024, 4096),
                                                   (SKEWED, 50, 768, 8192), (UNIFORM, 21, 256, 11008)])
def test_dense_lora_matches_oracle_dense_projection(lsg, dtype, pop, batch, h_in, h_out):
    """lsg_dense_lora = dense_projection (sgmv.cpp:143-155): x.W + lora_addon, the LoRA add in
    the GEMM epilogue; checked against the fp64 oracle and against cuBLAS + the SGMV kernel."""
    r = 16
    bounds, _, _ = segments_for(pop, batch, 44)
    x, A, B = random_problem(h_in, h_out, r, bounds, 45)
    W = oracle().rng(46).fill_pm1(h_in * h_out).reshape(h_in, h_out) * 0.05
    p = Problem(lsg, x, A, B, bounds, dtype, layers=2, layer=1)
    Wq = torch.tensor(W, dtype=torch.float64).to(dtype).cuda()
    y = torch.full((batch, h_out), float("nan"), dtype=dtype, device="cuda")
    lsg.dense_lora(y, p.x, Wq, p.pool, p.seg_starts, p.seg_slot, 1)
    torch.cuda.synchronize()
    ref = p.xd @ Wq.double().cpu().numpy() + oracle().lora_addon(p.xd, p.bounds, p.Ad, p.Bd)
    err = row_norm_err(y.double().cpu().numpy(), ref)
    assert err <= tol(dtype), err
    y2 = (p.x.float() @ Wq.float()).to(dtype)  # cuBLAS GEMM, then the SGMV kernel adds the LoRA
    lsg.sgmv(y2, p.x, p.pool, p.seg_starts, p.seg_slot, 1)
    torch.cuda.synchronize()
    assert row_norm_err(y.double().cpu().numpy(), y2.double().cpu().numpy()) <= 2 * tol(dtype)
    y3 = torch.full_like(y, float("nan"))  # deterministic: a second call is bit-identical
    lsg.dense_lora(y3, p.x, Wq, p.pool, p.seg_starts, p.seg_slot, 1)
    assert torch.equal(y3, y)


def test_dense_lora_no_adapter_and_empty_segments(lsg):
    """Segments without an adapter (slot -1, slot >= num_slots) and empty segments add nothing."""
    dtype, h_in, h_out, r = torch.float16, 2048, 4096, 16
    bounds = np.array([0, 5, 5, 9, 20, 20, 33, 40], dtype=np.uint64)
    slots = [0, 1, -1, 2, 3, 7, 4]
    x, A, B = random_problem(h_in, h_out, r, bounds, 47)
    p = Problem(lsg, x, A, B, bounds, dtype, slots=[s if s < 5 else -1 for s in slots], num_slots=5)
    p.seg_slot = torch.tensor(slots, dtype=torch.int32, device="cuda")
    W = oracle().rng(48).fill_pm1(h_in * h_out).reshape(h_in, h_out) * 0.05
    Wq = torch.tensor(W, dtype=torch.float64).to(dtype).cuda()
    y = torch.full((40, h_out), float("nan"), dtype=dtype, device="cuda")
    lsg.dense_lora(y, p.x, Wq, p.pool, p.seg_starts, p.seg_slot, 0)
    torch.cuda.synchronize()
    ref = p.xd @ Wq.double().cpu().numpy()
    for s, slot in enumerate(slots):  # lora_addon (sgmv.cpp:112-121) restated for the empty / adapter-less segments
        lo, hi = int(bounds[s]), int(bounds[s + 1])
        if 0 <= slot < 5 and hi > lo:
            ref[lo:hi] += p.xd[lo:hi] @ p.Ad[s] @ p.Bd[s]
    assert row_norm_err(y.double().cpu().numpy(), ref) <= tol(dtype)


def test_dense_lora_pdl_chain_reads_fresh_x(lsg):
    """With PDL on, the dense projection's GEMM streams x before its own wait (its shrink releases it
    only after the shrink's wait): x produced by the kernel right before (an SGMV launch writing
    it) must be seen complete.  Repeated chains, compared with the PDL-off result."""
    dtype, h, r = torch.float16, 4096, 16
    bounds, _, _ = segments_for(DISTINCT, 64, 70)
    x, A, B = random_problem(h, h, r, bounds, 71)
    p = Problem(lsg, x, A, B, bounds, dtype)
    W = torch.tensor(oracle().rng(72).fill_pm1(h * h).reshape(h, h) * 0.05, dtype=torch.float64).to(dtype).cuda()
    outs = []
    for pdl in (0, 1):
        lsg.set_option(lsg.LSG_OPT_PDL, pdl)
        res = []
        for it in range(3):
            xin = torch.zeros_like(p.x)  # x of this layer = an SGMV launch's output
            lsg.sgmv(xin, p.x, p.pool, p.seg_starts, p.seg_slot, 0)
            y = torch.full_like(p.x, float("nan"))
            lsg.dense_lora(y, xin, W, p.pool, p.seg_starts, p.seg_slot, 0)
            res.append(y)
        torch.cuda.synchronize()
        outs.append(res)
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)


def test_dense_lora_rejects_unsupported(lsg):
    pool = lsg.AdapterPool(2, 1, 4096, 4096, 32, torch.float16)
    x = torch.zeros(4, 4096, dtype=torch.float16, device="cuda")
    y = torch.zeros_like(x)
    w = torch.zeros(4096, 4096, dtype=torch.float16, device="cuda")
    ss = torch.tensor([0, 4], dtype=torch.int32, device="cuda")
    sl = torch.zeros(1, dtype=torch.int32, device="cuda")
    with pytest.raises(RuntimeError, match="rank 16"):
        lsg.dense_lora(y, x, w, pool, ss, sl, 0)


@pytest.mark.parametrize("lens", [[1] * 64, [3, 0, 5, 1, 7], [200, 1, 1, 30, 129], [1000]])
def test_pdl_chain_of_dependent_launches(lsg, lens):
    """With programmatic dependent launch, each launch of a chain reads the y its predecessor
    wrote (y_a -> y_b -> y_a ...): 12 dependent launches (long segments take the tensor-core
    kernels, whose CTAs without work leave early) equal the same chain without PDL, bit for bit."""
    bounds = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    nseg, rows = len(lens), int(bounds[-1])
    g = oracle().rng(123)
    pool = lsg.AdapterPool(nseg, 12, 4096, 4096, 16, torch.float16)
    pool.a.copy_(torch.tensor(g.fill_pm1(pool.a.numel()).reshape(pool.a.shape) * 0.01).half())
    pool.b.copy_(torch.tensor(g.fill_pm1(pool.b.numel()).reshape(pool.b.shape) * 0.05).half())
    x = torch.tensor(g.fill_pm1(rows * 4096).reshape(rows, 4096)).half().cuda()
    ss = torch.tensor(bounds.astype(np.int64), dtype=torch.int32, device="cuda")
    sl = torch.arange(nseg, dtype=torch.int32, device="cuda")
    out = []
    for pdl in (0, 1):
        lsg.set_option(lsg.LSG_OPT_PDL, pdl)
        bufs = [x.clone(), torch.zeros_like(x)]
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for layer in range(12):  # launch i reads bufs[i % 2], accumulates into bufs[(i + 1) % 2]
                lsg.sgmv(bufs[(layer + 1) % 2], bufs[layer % 2], pool, ss, sl, layer)
        torch.cuda.synchronize()
        out.append([b.clone() for b in bufs])
    lsg.set_option(lsg.LSG_OPT_PDL, 0)
    for a, b in zip(*out):
        assert torch.isfinite(a.float()).all()
        assert torch.equal(a, b)


@pytest.mark.parametrize("r,prefill,on_tc", [(16, 128, True), (16, 300, True), (16, 512, True), (32, 128, True),
                                             (64, 128, True)])
def test_default_long_segment_dispatch_by_rank(lsg, r, prefill, on_tc):
    """The automatic dispatch: prefills of >= 128 rows run on the tensor
    cores (K9 at ranks 16 / 32, K7 at rank 64 below 1024 rows: not bitwise the CUDA-core result)
    -- the call must not fall back silently, e.g. on a workspace bound computed with another
    threshold.  Both forms stay within the oracle tolerance."""
    bounds = np.concatenate([[0, prefill], prefill + np.arange(1, 32)]).astype(np.uint64)
    x, A, B = random_problem(4096, 4096, r, bounds, 321 + r)
    p = Problem(lsg, x, A, B, bounds, torch.float16)
    ref = p.reference()
    y = p.run()
    lsg.set_option(lsg.LSG_OPT_NO_TENSOR_CORES, 1)
    try:
        cc = p.run()
    finally:
        lsg.set_option(lsg.LSG_OPT_NO_TENSOR_CORES, 0)
    for out in (y, cc):
        assert row_norm_err(out.double().cpu().numpy(), ref) <= tol(torch.float16)
    assert torch.equal(y[:prefill], cc[:prefill]) != on_tc
    if r != 64:  # rank 64 with shared adapters puts every segment on the MMA pair
        assert torch.equal(y[prefill:], cc[prefill:])  # the decode rows: the CUDA-core kernel in both


def test_tc_row_threshold_option(lsg):
    """LSG_OPT_TC_MIN_ROWS moves the tensor-core threshold: above the batch size every segment
    stays on the CUDA-core kernel (bitwise the no-tensor-core run); results stay in tolerance."""
    bounds = np.array([0, 200, 203, 260], dtype=np.uint64)
    x, A, B = random_problem(4096, 4096, 16, bounds, 95)
    p = Problem(lsg, x, A, B, bounds, torch.float16)
    ref = p.reference()
    lsg.set_option(lsg.LSG_OPT_NO_TENSOR_CORES, 1)
    cc = p.run()
    lsg.set_option(lsg.LSG_OPT_NO_TENSOR_CORES, 0)
    lsg.set_option(lsg._lib.LSG_OPT_TC_MIN_ROWS, 261)
    assert torch.equal(p.run(), cc)
    lsg.set_option(lsg._lib.LSG_OPT_TC_MIN_ROWS, 50)  # the 57-row segment joins the tensor cores
    y = p.run()
    assert row_norm_err(y.double().cpu().numpy(), ref) <= tol(torch.float16)
    assert torch.equal(y[200:203], cc[200:203])  # the 3-row segment is untouched by the change
    with pytest.raises(RuntimeError):
        lsg.set_option(lsg._lib.LSG_OPT_TC_MIN_ROWS, -1)


# ---------------------------------------------------------------------------------
# Round-2 parity gaps: the BASELINE configs' exact layouts, shrink output v on random
# data, the acceptance-size verify run, grouped rank-64 launches
# ---------------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", DTYPES)
def test_config1_exact_layout_4x8(lsg, dtype):
    """configs[0]: h=4096, r=16, 32 decode rows, 4 LoRAs x 8 rows -- every formulation against
    the oracle, and the three GPU formulations bitwise equal."""
    bounds = np.array([0, 8, 16, 24, 32], dtype=np.uint64)
    x, A, B = random_problem(4096, 4096, 16, bounds, 401)
    y0 = oracle().rng(402).fill_pm1(32 * 4096).reshape(32, 4096)
    p = Problem(lsg, x, A, B, bounds, dtype, y0=y0)
    ref = p.reference()
    base = p.run("fused")
    assert row_norm_err(base.double().cpu().numpy(), ref) <= tol(dtype)
    for kind in ("two_launch", "bgmv"):
        assert torch.equal(p.run(kind), base), kind


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("pop", [DISTINCT, UNIFORM])
def test_config5_1000_slot_pool_scattered_slots_nonzero_layer(lsg, dtype, pop):
    """configs[4] on one GPU: h=8192, r=16, a 1000-slot pool with 3 layers, the batch's
    adapters on scattered slots (not 0..n-1), launched at layer 2; the oracle gets the
    dequantised weights read back from exactly those slots."""
    h, r, slots_total, layers, layer = 8192, 16, 1000, 3, 2
    bounds, _, _ = segments_for(pop, 64, 501 + pop)
    nseg = len(bounds) - 1
    pool = lsg.AdapterPool(slots_total, layers, h, h, r, dtype)
    gen = torch.Generator(device="cuda").manual_seed(503)
    pool.a.uniform_(-1, 1, generator=gen)
    pool.b.uniform_(-1, 1, generator=gen)
    slots = np.random.default_rng(504).choice(slots_total, nseg, replace=False).astype(np.int32)
    x = torch.empty(64, h, dtype=dtype, device="cuda").uniform_(-1, 1, generator=gen)
    y0 = torch.empty(64, h, dtype=dtype, device="cuda").uniform_(-1, 1, generator=gen)
    ss = torch.tensor(bounds.astype(np.int64), dtype=torch.int32, device="cuda")
    sl = torch.tensor(slots, device="cuda")
    y = y0.clone()
    lsg.sgmv(y, x, pool, ss, sl, layer)
    torch.cuda.synchronize()
    idx = torch.tensor(slots.astype(np.int64), device="cuda")
    Ad = pool.a[idx, layer].double().cpu().numpy()
    Bd = pool.b[idx, layer].double().cpu().numpy()
    ref = y0.double().cpu().numpy() + oracle().lora_addon(x.double().cpu().numpy(), bounds, Ad, Bd)
    assert row_norm_err(y.double().cpu().numpy(), ref) <= tol(dtype)
    # the same rows through BGMV with per-row slots: bitwise
    row_slot = torch.tensor(np.repeat(slots, np.diff(bounds.astype(np.int64))), device="cuda")
    yb = y0.clone()
    lsg.bgmv(yb, x, pool, row_slot, layer)
    torch.cuda.synchronize()
    assert torch.equal(yb, y)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("pop", [DISTINCT, UNIFORM, SKEWED, IDENTICAL])
def test_shrink_v_matches_oracle_random(lsg, dtype, shape, pop):
    """lsg_sgmv_shrink's fp32 v against the oracle's sgmv_shrink (sgmv.cpp:105-119) on random
    data at every BASELINE shape: v is fp32 with no output rounding, so the per-row
    normalised error is at fp32-accumulation level (<= 1e-5)."""
    h_in, h_out, r = shape
    bounds, _, _ = segments_for(pop, 64, 601 + pop)
    x, A, B = random_problem(h_in, h_out, r, bounds, 602 + pop)
    p = Problem(lsg, x, A, B, bounds, dtype)
    v = torch.empty(64, r, dtype=torch.float32, device="cuda")
    lsg.sgmv_shrink(v, p.x, p.pool, p.seg_starts, p.seg_slot, 0)
    torch.cuda.synchronize()
    vref = oracle().sgmv_shrink(p.xd, p.bounds, p.Ad)
    assert row_norm_err(v.double().cpu().numpy(), vref) <= 1e-5


def test_verify_sgmv_acceptance_size_1000_trials(lsg):
    """Acceptance criterion 1 (acceptance_main.cpp:57-68): verify_sgmv(1000, 42) -- 1000
    randomised trials, every popularity and verify shape -- through the fused kernel, fp16."""
    o = oracle()
    g = o.rng(o.derive_seed(42, 17))
    worst = 0.0
    for t in range(1000):
        tr = g.verify_next_trial(t)
        p = Problem(lsg, tr["x"], tr["A"], tr["B"], tr["bounds"], torch.float16)
        err = row_norm_err(p.run("fused").double().cpu().numpy(), p.reference())
        worst = max(worst, err)
        assert err <= tol(torch.float16), (t, err)
    assert worst <= NORTH_STAR_TOL


@pytest.mark.parametrize("pop", [UNIFORM, SKEWED, IDENTICAL])
def test_grouped_sites_rank64_shared_adapters_bitwise(lsg, pop):
    """Rank 64 with shared adapters plans 4-row tiles, which the grouped item mode does not
    have: lsg_sgmv_multi must run those sites one by one (it used to update only
    site 0) -- every site bitwise equal to its own lsg_sgmv call."""
    bounds, _, _ = segments_for(pop, 64, 700 + pop)
    probs = []
    for i in range(3):
        x, A, B = random_problem(5120, 5120, 64, bounds, 710 + i)
        y0 = oracle().rng(720 + i).fill_pm1(64 * 5120).reshape(64, 5120)
        probs.append(Problem(lsg, x, A, B, bounds, torch.float16, y0=y0))
    ref = [p.run() for p in probs]
    ys = [p.y0.clone() for p in probs]
    lsg.sgmv_multi(ys, [p.x for p in probs], [p.pool for p in probs], probs[0].seg_starts, probs[0].seg_slot, 0)
    torch.cuda.synchronize()
    for i in range(3):
        assert not torch.equal(ys[i], probs[i].y0), i
        assert torch.equal(ys[i], ref[i]), i


def test_call_options_are_per_call(lsg):
    """lsg_sgmv_ex: a per-call tc_min_rows / no_tensor_cores overrides the process default for
    that call only (the default is untouched and the next call uses it again)."""
    bounds = np.array([0, 200, 203, 260], dtype=np.uint64)
    x, A, B = random_problem(4096, 4096, 16, bounds, 96)
    p = Problem(lsg, x, A, B, bounds, torch.float16)
    tc = p.run()
    y = p.y0.clone()
    lsg.sgmv(y, p.x, p.pool, p.seg_starts, p.seg_slot, 0, no_tensor_cores=True)
    lsg.set_option(lsg.LSG_OPT_NO_TENSOR_CORES, 1)
    cc = p.run()
    lsg.set_option(lsg.LSG_OPT_NO_TENSOR_CORES, 0)
    torch.cuda.synchronize()
    assert torch.equal(y, cc)
    assert lsg.get_option(lsg.LSG_OPT_NO_TENSOR_CORES) == 0
    assert torch.equal(p.run(), tc)
    y2 = p.y0.clone()
    lsg.sgmv(y2, p.x, p.pool, p.seg_starts, p.seg_slot, 0, tc_min_rows=261)
    torch.cuda.synchronize()
    assert torch.equal(y2, cc)


def test_grid_limit_many_rows(lsg):
    """More than 65535 rows (gridDim.y limit): row-mode launches switch to the
    tile-scan decode and BGMV runs in row chunks -- results bitwise equal to each other and
    to the oracle on sampled rows."""
    n, h, r = 70000, 128, 8
    nseg = 7
    bounds = np.linspace(0, n, nseg + 1).astype(np.uint64)
    gen = torch.Generator(device="cuda").manual_seed(9)
    pool = lsg.AdapterPool(nseg, 1, h, h, r, torch.float16)
    pool.a.uniform_(-1, 1, generator=gen)
    pool.b.uniform_(-1, 1, generator=gen)
    x = torch.empty(n, h, dtype=torch.float16, device="cuda").uniform_(-1, 1, generator=gen)
    ss = torch.tensor(bounds.astype(np.int64), dtype=torch.int32, device="cuda")
    sl = torch.arange(nseg, dtype=torch.int32, device="cuda")
    y = torch.zeros(n, h, dtype=torch.float16, device="cuda")
    lsg.sgmv(y, x, pool, ss, sl, 0, no_tensor_cores=True)
    rs = torch.repeat_interleave(sl, torch.tensor(np.diff(bounds.astype(np.int64)), device="cuda")).to(torch.int32)
    yb = torch.zeros_like(y)
    lsg.bgmv(yb, x, pool, rs, 0)
    torch.cuda.synchronize()
    assert torch.equal(y, yb)
    pick = np.array([0, 1, 9999, 65534, 65535, 65536, n - 1])
    xs = x[torch.tensor(pick, device="cuda")].double().cpu().numpy()
    segs = np.searchsorted(bounds.astype(np.int64), pick, side="right") - 1
    ref = np.stack([xs[i] @ pool.a[segs[i], 0].double().cpu().numpy() @ pool.b[segs[i], 0].double().cpu().numpy()
                    for i in range(len(pick))])
    assert row_norm_err(y[torch.tensor(pick, device="cuda")].double().cpu().numpy(), ref) <= tol(torch.float16)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("shape", [(4096, 4096, 16), (4096, 4096, 32), (8192, 8192, 16), (5120, 5120, 16),
                                   (1024, 1024, 32), (4096, 4096, 64)])
def test_tc_generations_many_tiles_agree(lsg, dtype, shape):
    """Many long segments (more tiles than co-resident CTAs / clusters), partial last tiles, a
    no-adapter long segment and decode rows in between, on the default long-segment kernel
    (the streaming kernel at >= 1024 rows): oracle tolerance, run-to-run bitwise, and within
    tolerance of every other tensor-core generation (MMA pair, streaming kernel, tcgen05 pair,
    streamed cluster kernel, first fused kernel, two-kernel form)."""
    h_in, h_out, r = shape
    lens = [300, 1, 129, 7, 1000, 2, 260, 128, 3, 700, 1, 450]
    bounds = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    x, A, B = random_problem(h_in, h_out, r, bounds, 811)
    y0 = oracle().rng(812).fill_pm1(int(bounds[-1]) * h_out).reshape(-1, h_out)
    slots = list(range(len(lens)))
    slots[6] = -1  # a long segment without an adapter: rows untouched
    p = Problem(lsg, x, A, B, bounds, dtype, slots=slots, num_slots=len(lens), y0=y0)
    got = p.run()
    ref = p.reference()
    assert row_norm_err(got.double().cpu().numpy(), ref) <= tol(dtype)
    assert torch.equal(got[int(bounds[6]):int(bounds[7])], p.y0[int(bounds[6]):int(bounds[7])])
    assert torch.equal(p.run(), got)
    alts = [(lsg._lib.LSG_OPT_TC_SPLIT, 1), (lsg._lib.LSG_OPT_TC_LEGACY, 2), (lsg._lib.LSG_OPT_TC_LEGACY, 3),
            (lsg._lib.LSG_OPT_TC_LEGACY, 4), (lsg._lib.LSG_OPT_TC_LEGACY, 5)]
    if r == 16:
        alts.append((lsg._lib.LSG_OPT_TC_LEGACY, 1))
    for opt, val in alts:  # every earlier tensor-core generation agrees within tolerance
        lsg.set_option(opt, val)
        try:
            alt = p.run()
        finally:
            lsg.set_option(opt, 0)
        assert row_norm_err(alt.double().cpu().numpy(), ref) <= tol(dtype), (opt, val)
        for s, n in enumerate(lens):  # decode rows: the CUDA-core kernel in both runs
            a, b = int(bounds[s]), int(bounds[s + 1])
            if n < 128:
                assert torch.equal(alt[a:b], got[a:b]), (opt, val, s)


@pytest.mark.parametrize("tp", [2, 4, 8])
def test_tp_p2p_fused_allgather_every_rank_bitwise(lsg, tp):
    """lsg_tp_sgmv (configs[4], 70B TP): every rank's kernel stores its column slice into EVERY
    rank's y, then the flag exchange.  The tp ranks are emulated on one GPU, each on its own
    stream, all in flight together (the flag wait needs every peer): afterwards each rank's y
    equals the unsharded single-GPU result bit for bit -- over two consecutive steps (epochs)."""
    from paper_2310_18547_b200 import tp as tpmod
    h, r = 8192, 16
    bounds, _, _ = segments_for(DISTINCT, 32, 5)
    x, A, B = random_problem(h, h, r, bounds, 6)
    y0 = oracle().rng(7).fill_pm1(32 * h).reshape(32, h)
    p = Problem(lsg, x, A, B, bounds, torch.float16, y0=y0)
    base = p.run()
    base2 = base.clone()
    lsg.sgmv(base2, p.x, p.pool, p.seg_starts, p.seg_slot, 0)
    torch.cuda.synchronize()
    ys = [p.y0.clone() for _ in range(tp)]
    flags = [torch.zeros(tp, dtype=torch.int32, device="cuda") for _ in range(tp)]
    shards = [tpmod.tp_pool(p.pool.a, p.pool.b, tp, rk) for rk in range(tp)]
    groups = [tpmod.TpGroup(rk, [t.data_ptr() for t in ys], [f.data_ptr() for f in flags]) for rk in range(tp)]
    streams = [torch.cuda.Stream() for _ in range(tp)]
    for step, expect in ((1, base), (2, base2)):
        torch.cuda.synchronize()
        for rk in range(tp):
            with torch.cuda.stream(streams[rk]):
                tpmod.tp_sgmv_p2p(groups[rk], ys[rk], p.x, shards[rk], p.seg_starts, p.seg_slot, 0)
        torch.cuda.synchronize()
        for rk in range(tp):
            assert torch.equal(ys[rk], expect), (step, rk)
            assert flags[rk].tolist() == [step] * tp


def test_tp_nccl_allgather_single_rank_comm(lsg):
    """lsg_tp_sgmv_nccl's plumbing (slice in place, ncclAllGather, copies back) on a one-rank
    NCCL communicator: bitwise the plain launch."""
    from paper_2310_18547_b200 import tp as tpmod
    h, r = 8192, 16
    bounds, _, _ = segments_for(UNIFORM, 24, 8)
    x, A, B = random_problem(h, h, r, bounds, 9)
    y0 = oracle().rng(10).fill_pm1(24 * h).reshape(24, h)
    p = Problem(lsg, x, A, B, bounds, torch.bfloat16, y0=y0)
    base = p.run()
    comm = tpmod.nccl_comm_single()
    y = p.y0.clone()
    tpmod.tp_sgmv_nccl(y, p.x, tpmod.tp_pool(p.pool.a, p.pool.b, 1, 0), p.seg_starts, p.seg_slot, 0, 0, 1, comm)
    torch.cuda.synchronize()
    assert torch.equal(y, base)


# ---------------------------------------------------------------------------------
# Segment-tile MMA pair (K7, sgmv_mma.cuh): shared-adapter and prefill segments
# ---------------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("shape", [(4096, 4096, 16), (4096, 4096, 32), (5120, 5120, 64), (4096, 2048, 64),
                                   (8192, 8192, 16)])
@pytest.mark.parametrize("pop", [UNIFORM, SKEWED, IDENTICAL])
def test_mma_pair_shared_adapters_match_oracle(lsg, dtype, shape, pop):
    """Every segment on the MMA pair (LSG_OPT_MMA_MIN_ROWS = 1; rank 64's default when rows
    share adapters): within tolerance of the fp64 oracle, run-to-run identical, and y
    accumulates onto y_old."""
    h_in, h_out, r = shape
    bounds, _, _ = segments_for(pop, 64, 500 + pop)
    x, A, B = random_problem(h_in, h_out, r, bounds, 501 + pop)
    y0 = oracle().rng(502).fill_pm1(64 * h_out).reshape(64, h_out)
    p = Problem(lsg, x, A, B, bounds, dtype, y0=y0)
    lsg.set_option(lsg._lib.LSG_OPT_MMA_MIN_ROWS, 1)
    y = p.run()
    assert row_norm_err(y.double().cpu().numpy(), p.reference()) <= tol(dtype)
    assert torch.equal(p.run(), y)
    if r == 64:  # the automatic choice is the same path
        lsg.set_option(lsg._lib.LSG_OPT_MMA_MIN_ROWS, 0)
        assert torch.equal(p.run(), y)
        lsg.set_option(lsg._lib.LSG_OPT_MMA_MIN_ROWS, 1)
    # the one-launch form (a cluster per tile) and the two-launch pair: both within tolerance
    for mode in (1, 2):
        lsg.set_option(lsg._lib.LSG_OPT_MMA_FUSED, mode)
        ym = p.run()
        assert row_norm_err(ym.double().cpu().numpy(), p.reference()) <= tol(dtype), mode
        assert torch.equal(p.run(), ym), mode


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("r", [16, 32, 64])
@pytest.mark.parametrize("lens", [[128] + [1] * 31, [300, 17, 1, 5, 2, 16], [2048, 3, 1], [129, 135, 7]])
@pytest.mark.parametrize("gen", [3, 4])
def test_mma_pair_long_segments_match_oracle(lsg, dtype, r, lens, gen):
    """LSG_OPT_TC_LEGACY = 3: the MMA pair takes the long (prefill) segments as well; = 4: the
    one-pass streaming kernel takes them (MMA pair for the medium ones); with
    LSG_OPT_MMA_MIN_ROWS = 2 the 1-row segments stay on the CUDA-core kernel in the same call."""
    bounds = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    x, A, B = random_problem(4096, 4096, r, bounds, 600 + r)
    p = Problem(lsg, x, A, B, bounds, dtype)
    lsg.set_option(lsg._lib.LSG_OPT_TC_LEGACY, gen)
    for lo in (1, 2):
        lsg.set_option(lsg._lib.LSG_OPT_MMA_MIN_ROWS, lo)
        for mode in (1, 2):  # the two-launch pair, the one-launch form
            lsg.set_option(lsg._lib.LSG_OPT_MMA_FUSED, mode)
            y = p.run()
            assert row_norm_err(y.double().cpu().numpy(), p.reference()) <= tol(dtype), (lo, mode)


def test_mma_pair_no_adapter_segments_untouched_and_scattered_slots(lsg):
    """Slot -1 segments leave y untouched on the MMA pair; scattered slots of a multi-layer
    pool at a non-zero layer index correctly."""
    lens = [9, 16, 17, 1, 33, 4]
    bounds = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    slots = [7, -1, 2, 11, -1, 0]
    x, A, B = random_problem(5120, 5120, 64, bounds, 610)
    y0 = oracle().rng(611).fill_pm1(sum(lens) * 5120).reshape(sum(lens), 5120)
    p = Problem(lsg, x, A, B, bounds, torch.float16, slots=slots, num_slots=12, layers=3, layer=2, y0=y0)
    ref = p.reference()
    for mode in (1, 2):  # the two-launch pair, the one-launch form
        lsg.set_option(lsg._lib.LSG_OPT_MMA_FUSED, mode)
        y = p.run()
        assert row_norm_err(y.double().cpu().numpy(), ref) <= tol(torch.float16), mode
        for s in (1, 4):
            a, b = int(bounds[s]), int(bounds[s + 1])
            assert torch.equal(y[a:b], p.y0[a:b]), (mode, s)


def test_mma_pair_many_tiles_and_workspace_bound(lsg):
    """Hundreds of 16-row tiles (the tile bound grows with the segment count) through the
    caller-workspace entry (lsg_sgmv_workspace_size is an upper bound)."""
    lens = [(29 * i) % 61 + 2 for i in range(120)]
    bounds = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    x, A, B = random_problem(1024, 2048, 64, bounds, 620)
    p = Problem(lsg, x, A, B, bounds, torch.bfloat16)
    for mode in (1, 2):  # the two-launch pair, the one-launch form
        lsg.set_option(lsg._lib.LSG_OPT_MMA_FUSED, mode)
        y = p.run()
        assert row_norm_err(y.double().cpu().numpy(), p.reference()) <= tol(torch.bfloat16), mode
