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


# ---- K6 segment builder: the specification the device builder is checked against ----
def builder_model(row_slot, num_slots, lead, lead_rows=(0, 0)):
    """Stable grouping of rows by slot (lsg_build_segments, include/lsg_sgmv.h): the lead
    slot's group first with the prefill rows [lead_rows) ahead of its other rows, then
    ascending slot, no-adapter rows (slot < 0 or >= num_slots) last as slot -1.
    Returns (row_perm, seg_starts, seg_slot)."""
    key = [(0 if s == lead else s + 1) if 0 <= s < num_slots else 1 << 31 for s in row_slot]
    sub = [0 if (0 <= row_slot[i] < num_slots and row_slot[i] == lead and lead_rows[0] <= i < lead_rows[1]) else 1
           for i in range(len(row_slot))]
    perm = sorted(range(len(row_slot)), key=lambda i: (key[i], sub[i], i))
    starts, slots = [], []
    for i, r in enumerate(perm):
        if i == 0 or key[r] != key[perm[i - 1]]:
            starts.append(i)
            s = row_slot[r]
            slots.append(s if 0 <= s < num_slots else -1)
    return perm, starts + [len(row_slot)], slots


def plan_batch_rows(case):
    """Token rows of a golden plan_batch case in request order (simulator.cpp:267-276: a
    prefill contributes its prompt rows, a decode one row; only the first pending prefill is
    scheduled), with slots = rank of the LoraId.  Returns (uniq_loras, row_slot, req_of_row,
    lead_slot, lead_rows)."""
    lora, done, prompt, plan = case["lora"], case["done"], case["prompt"], case["plan"]
    uniq = sorted(set(lora))
    slot_of = {l: i for i, l in enumerate(uniq)}
    rows, req_of_row, lead_rows = [], [], (0, 0)
    for i, (l, d) in enumerate(zip(lora, done)):
        if d:
            rows.append(slot_of[l])
            req_of_row.append(i)
        elif i == plan["prefill"]:
            lead_rows = (len(rows), len(rows) + prompt[i])
            rows.extend([slot_of[l]] * prompt[i])
            req_of_row.extend([i] * prompt[i])
    lead = slot_of[lora[plan["prefill"]]] if plan["prefill"] >= 0 else -1
    return uniq, rows, req_of_row, lead, lead_rows
