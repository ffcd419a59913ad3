"""The product-side workload port (paper_2310_18547_b200/workload.py) against the
reference's golden draws (tests/golden/rng.json)."""
from __future__ import annotations

import json
import os

from paper_2310_18547_b200 import workload as W

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_rng_and_assign_models_match_reference():
    d = json.load(open(os.path.join(GOLDEN, "rng.json")))
    for seed in (0, 7, 42):
        g = W.Rng(seed)
        assert [str(g.next()) for _ in range(32)] == d[f"next_{seed}"]
        assert [g.uniform01().hex() for _ in range(16)] == d[f"uniform01_{seed}"]
    for k, v in d["derive_seed"].items():
        s, st = map(int, k.split(","))
        assert str(W.derive_seed(s, st)) == v
    for k, v in d["model_count_for"].items():
        n, p = map(int, k.split(","))
        assert W.model_count_for(n, p) == v
    for k, v in d["assign_models"].items():
        n, p, seed = map(int, k.split(","))
        if n <= 100:
            assert W.assign_models(n, p, 1.5, seed) == v


def test_group_segments_layout():
    ids = [3, 1, 3, 0, 1, 3]
    bounds, uniq, order = W.group_segments(ids)
    assert bounds == [0, 1, 3, 6] and uniq == [0, 1, 3] and order == [3, 1, 4, 0, 2, 5]
