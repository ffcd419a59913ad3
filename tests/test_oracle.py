"""The CPU oracle (oracle/sgmv_oracle.c) pinned against the reference.

1. Golden fixtures in tests/golden/, produced by the reference's own sources
   (tests/golden/make_golden.py over oracle/_ref/libref.so) -- run everywhere.
2. Live comparison with oracle/_ref/libref.so when that library is present.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from oracle.oracle import Oracle, Reference, reference_available
from tests.golden.make_golden import trial_digest

GOLDEN = os.path.dirname(os.path.abspath(__file__)) + "/golden"


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def load(name):
    return json.load(open(os.path.join(GOLDEN, name)))


# ---- RNG / workload (workload.hpp:13-45, workload.cpp:11-143) ------------------------
def test_rng_streams_match_reference(orc):
    d = load("rng.json")
    for seed in (0, 1, 7, 42, 5489, 20240805):
        g = orc.rng(seed)
        assert [str(g.next()) for _ in range(32)] == d[f"next_{seed}"]
        assert [g.uniform01().hex() for _ in range(16)] == d[f"uniform01_{seed}"]
        assert [g.uniform_index(n) for n in (1, 2, 3, 5, 7, 64, 1000, 2**63 + 5)] == d[f"uniform_index_{seed}"]
        assert [g.uniform_int(lo, hi) for lo, hi in ((-3, 3), (1, 8), (1, 64), (0, 0))] == d[f"uniform_int_{seed}"]
        cum = np.cumsum([1.0, 1 / 1.5, 1 / 2.25, 1 / 3.375])
        assert [g.discrete(cum, float(cum[-1])) for _ in range(16)] == d[f"discrete_{seed}"]
        assert g.shuffle(np.arange(20)).tolist() == d[f"shuffle_{seed}"]
    g = orc.rng(5489)
    for _ in range(9999):
        g.next()
    assert str(g.next()) == d["mt19937_64_10000th"] == "9981545732273789042"


def test_derive_seed_model_count_assign_models(orc):
    d = load("rng.json")
    for k, v in d["derive_seed"].items():
        s, st = map(int, k.split(","))
        assert str(orc.derive_seed(s, st)) == v
    for k, v in d["model_count_for"].items():
        n, p = map(int, k.split(","))
        assert orc.model_count_for(n, p) == v
    for k, v in d["assign_models"].items():
        n, p, seed = map(int, k.split(","))
        assert orc.assign_models(n, p, 1.5, seed).tolist() == v


def test_uniform_and_skewed_properties(orc):
    """test_workload.cpp:63-108 restated."""
    ids = orc.assign_models(1000, 1, 1.5, 42)
    counts = np.bincount(ids)
    assert len(counts) == 32 and counts.max() - counts.min() <= 1
    sk = orc.assign_models(20000, 2, 1.5, 7)
    c = np.bincount(sk)
    assert 1.3 < c[0] / c[1] < 1.7 and 1.25 < c[1] / c[2] < 1.8


# ---- SGMV operators (sgmv.cpp:105-217) ----------------------------------------------
def test_verify_trials_bit_exact_against_golden(orc):
    z = np.load(os.path.join(GOLDEN, "verify_trials.npz"))
    g = orc.rng(orc.derive_seed(42, 17))
    for t in range(8):
        tr = g.verify_next_trial(t)
        assert [tr["h_in"], tr["h_out"], tr["rank"], tr["rows"], tr["nseg"]] == z[f"t{t}_shape"].tolist()
        for k in ("bounds", "ids", "x", "A", "B"):
            assert np.array_equal(tr[k], z[f"t{t}_{k}"]), (t, k)
        y = orc.lora_addon(tr["x"], tr["bounds"], tr["A"], tr["B"])
        assert np.array_equal(y, z[f"t{t}_y"])  # bitwise fp64
        assert np.array_equal(orc.lora_loop_oracle(tr["x"], tr["bounds"], tr["A"], tr["B"]), y)
        assert np.array_equal(orc.gather_bmm_oracle(tr["x"], tr["bounds"], tr["A"], tr["B"]), y)


def test_verify_digest_200_trials(orc):
    """sha256 over 200 verify_sgmv(seed 42) batches + their fp64 lora_addon bits."""
    d = load("verify_digest.json")
    g = orc.rng(orc.derive_seed(42, 17))
    h = hashlib.sha256()
    for t in range(d["trials"]):
        tr = g.verify_next_trial(t)
        trial_digest(h, tr, orc.lora_addon(tr["x"], tr["bounds"], tr["A"], tr["B"]))
    assert h.hexdigest() == d["sha256"]
    # the reference's own verify_sgmv(8, 42, inject) failed on trial 0 with this shape
    g = orc.rng(orc.derive_seed(42, 17))
    t0 = g.verify_next_trial(0)
    shape = d["reference_verify_8_42_inject"]["first_fail_shape"]
    assert [t0["h_in"], t0["h_out"], t0["rank"], t0["rows"], t0["nseg"]] == shape


def test_known_answers(orc):
    k = load("kat.json")
    t = k["two_segment"]
    x, A, B = np.array(t["x"]), np.array(t["A"]), np.array(t["B"])
    assert orc.lora_addon(x, t["bounds"], A, B).tolist() == t["lora_addon"] == [[5, 1], [11, 3], [16, 54]]
    assert orc.dense_projection(x, t["bounds"], A, B, np.eye(2)).tolist() == t["dense_w_identity"]
    assert orc.sgmv_shrink(x, t["bounds"], A).tolist() == t["shrink"]
    r = k["rank1"]
    assert orc.lora_addon(np.array(r["x"]), r["bounds"], np.array(r["A"]), np.array(r["B"])).tolist() == [[3, 3]]


def test_dense_linear_and_permutation_properties(orc):
    """test_sgmv.cpp:143-197 restated on the oracle."""
    g = orc.rng(77)
    bounds = np.array([0, 4, 8, 16], dtype=np.uint64)
    x = g.fill_pm1(16 * 32).reshape(16, 32)
    A = g.fill_pm1(3 * 32 * 8).reshape(3, 32, 8)
    B = g.fill_pm1(3 * 8 * 48).reshape(3, 8, 48)
    w = g.fill_pm1(32 * 48).reshape(32, 48)
    y = orc.dense_projection(x, bounds, A, B, w)
    xw = np.zeros((16, 48))
    for i in range(16):  # i -> k -> j, as sgmv.cpp:9-19
        for kk in range(32):
            xw[i] += x[i, kk] * w[kk]
    assert np.array_equal(y, xw + orc.lora_addon(x, bounds, A, B))
    base = orc.lora_addon(x, bounds, A, B)
    assert np.abs(orc.lora_addon(3.5 * x, bounds, A, B) - 3.5 * base).max() < 1e-12
    order = [1, 0, 2]
    xs = np.concatenate([x[int(bounds[s]):int(bounds[s + 1])] for s in order])
    src = [r for s in order for r in range(int(bounds[s]), int(bounds[s + 1]))]
    nb = np.array([0, 4, 8, 16], dtype=np.uint64)
    got = orc.lora_addon(xs, nb, A[order], B[order])
    assert np.array_equal(got, base[src])


def test_segment_validation(orc):
    x = np.zeros((3, 2))
    with pytest.raises(ValueError):
        orc.lora_addon(x, [0, 0, 3], np.zeros((2, 2, 1)), np.zeros((2, 1, 2)))
    with pytest.raises(ValueError):
        orc.lora_addon(x, [1, 3], np.zeros((1, 2, 1)), np.zeros((1, 1, 2)))


# ---- cost model (cost_model.cpp:8-61) -------------------------------------------------
def test_cost_model_anchors(orc):
    d = load("cost_model.json")
    assert orc.sgmv_flop(64, 64, 16, 4096) == d["flop_64_64_16_4096"] == 8388608.0
    assert orc.sgmv_io_bytes(64, 64, 16, 4096) == d["io_64_64_16_4096"] == 8914944.0
    assert orc.sgmv_io_bytes(1, 1, 16, 4096) == d["io_1_1_16_4096"] == 139296.0
    assert orc.sgmv_io_bytes(1, 64, 16, 4096) == d["io_1_64_16_4096"]
    assert orc.gather_bmm_extra_elements(64, 64, 16, 4096) == d["gather_extra_64_64_16_4096"]
    for k, v in d["intensity"].items():
        n, b = map(int, k.split(","))
        assert orc.arithmetic_intensity(n, b, 16, 4096).hex() == v
    for k, v in d["latency_default"].items():
        n, b = map(int, k.split(","))
        assert orc.sgmv_latency(n, b, 16, 4096).hex() == v
    # the shrink+expand pair is the sum of the two io terms
    assert orc.adapter_pair_io_bytes(64, 64, 4096, 16) == 17829888.0
    assert orc.adapter_pair_io_bytes(64, 64, 4096, 16) == (orc.sgmv_io_bytes(64, 64, 4096, 16) +
                                                           orc.sgmv_io_bytes(64, 64, 16, 4096))


def test_plan_segments_golden(orc):
    for case in load("plan_batch.json"):
        assert orc.plan_segments(case["lora"], case["done"], case["prompt"]) == case["plan"]


# ---- live: the oracle against the compiled reference -----------------------------------
@pytest.mark.skipif(not reference_available(), reason="oracle/_ref/libref.so not built here")
def test_live_against_reference(orc):
    ref = Reference()
    ga, gb = orc.rng(orc.derive_seed(9, 17)), ref.rng(ref.derive_seed(9, 17))
    for t in range(120):
        ta, tb = ga.verify_next_trial(t), gb.verify_next_trial(t)
        for k in ("bounds", "x", "A", "B"):
            assert np.array_equal(ta[k], tb[k])
        for f in ("lora_addon", "lora_loop_oracle", "gather_bmm_oracle"):
            assert np.array_equal(getattr(orc, f)(ta["x"], ta["bounds"], ta["A"], ta["B"]),
                                  getattr(ref, f)(tb["x"], tb["bounds"], tb["A"], tb["B"]))
    # a large headline-shape batch, bit for bit
    g = orc.rng(3)
    bounds = np.array([0, 8, 16, 24, 32], dtype=np.uint64)
    x = g.fill_pm1(32 * 4096).reshape(32, 4096)
    A = g.fill_pm1(4 * 4096 * 16).reshape(4, 4096, 16)
    B = g.fill_pm1(4 * 16 * 4096).reshape(4, 16, 4096)
    assert np.array_equal(orc.lora_addon(x, bounds, A, B), ref.lora_addon(x, bounds, A, B))
    v = ref.sgmv_shrink(x, bounds, A, B)
    assert np.array_equal(orc.sgmv_shrink(x, bounds, A), v)
    assert np.array_equal(orc.sgmv_expand(v, bounds, B), ref.sgmv_expand(v, bounds, A, B))
    assert ref.roofline_csv(64) == load("cost_model.json")["roofline_csv"]


def test_builder_spec_reproduces_plan_batch_row_order():
    """The K6 builder's specification (tests/_util.builder_model, what the device builder
    is checked against bit-exactly in test_sgmv_gpu.py) yields plan_batch's bounds, segment
    adapters and row order -- prefill rows first, then `decodes` -- on every golden case."""
    from tests._util import builder_model, plan_batch_rows
    cases = load("plan_batch.json")
    assert len(cases) == 21
    for ci, case in enumerate(cases):
        plan = case["plan"]
        uniq, rows, req_of_row, lead, lead_rows = plan_batch_rows(case)
        perm, starts, slots = builder_model(rows, len(uniq), lead, lead_rows)
        assert starts == plan["bounds"], ci
        assert [uniq[s] for s in slots] == plan["loras"], ci
        order = []
        for r in perm:
            if not order or order[-1] != req_of_row[r]:
                order.append(req_of_row[r])
        assert order == ([plan["prefill"]] if plan["prefill"] >= 0 else []) + plan["decodes"], ci
