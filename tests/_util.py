"""Shared helpers for the parity tests: synthetic batches from the reference RNG
(restated in oracle/), 16-bit quantisation, and the normalised error metric.

Parity protocol: inputs are drawn in fp64 with the reference's
Rng, rounded to fp16/bf16 for the GPU, and the ORACLE is fed the dequantised
values, so only accumulation order and the final rounding differ.  Tolerance is
the per-row normalised max error  max_j |y_j - yhat_j|_inf / |yhat_j|_inf.
"""
from __future__ import annotations

import numpy as np

from oracle.oracle import DISTINCT, IDENTICAL, SKEWED, UNIFORM, Oracle

# Stated tolerances (per-row normalised, fp32 accumulate, one final rounding):
# fp16 output rounding is <= 2^-11 of an element, bf16 <= 2^-8.
TOL = {"float16": 1.5e-3, "bfloat16": 8e-3}
NORTH_STAR_TOL = 1e-2

_ORC = None


def oracle() -> Oracle:
    global _ORC
    if _ORC is None:
        _ORC = Oracle()
    return _ORC


def row_norm_err(y, yref) -> float:
    y = np.asarray(y, dtype=np.float64)
    yref = np.asarray(yref, dtype=np.float64)
    if y.size == 0:
        return 0.0
    num = np.abs(y - yref).max(axis=1)
    den = np.maximum(np.abs(yref).max(axis=1), 1e-30)
    return float((num / den).max())


def segments_for(pop: int, batch: int, seed: int):
    """assign_models + grouping by ascending id (experiments.cpp:56-76)."""
    o = oracle()
    ids = o.assign_models(batch, pop, 1.5, seed)
    order = sorted(range(batch), key=lambda i: (ids[i], i))
    uniq = sorted(set(ids.tolist()))
    bounds = [0]
    for u in uniq:
        bounds.append(bounds[-1] + int((ids == u).sum()))
    return np.array(bounds, dtype=np.uint64), uniq, order


def random_problem(h_in, h_out, rank, bounds, seed):
    """x [rows, h_in], A [nseg, h_in, r], B [nseg, r, h_out] ~ U[-1,1) from the reference Rng."""
    o = oracle()
    g = o.rng(seed)
    nseg = len(bounds) - 1
    rows = int(bounds[-1])
    x = g.fill_pm1(rows * h_in).reshape(rows, h_in)
    A = g.fill_pm1(nseg * h_in * rank).reshape(nseg, h_in, rank)
    B = g.fill_pm1(nseg * rank * h_out).reshape(nseg, rank, h_out)
    return x, A, B
