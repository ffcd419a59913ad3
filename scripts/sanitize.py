#!/usr/bin/env python
"""Small launches of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  Run on the GPU box, e.g.

    compute-sanitizer --tool racecheck --kernel-regex kns=lsg python scripts/sanitize.py

Each case is small (a few rows, short hidden sizes) so the instrumented run stays in
minutes.  Results are also checked against the CPU oracle, so a case that "passes"
the sanitizer but computes garbage still fails.  Families covered:
  sgmv_fast_kernel   fused / shrink / expand x item modes (row, row-split, tile-scan,
                     BGMV, grouped row) x tile rows 1 / 4 / 8, clusters 1..16, PDL on/off
  sgmv_tc_*          fused tensor-core kernel (rank 16), two-kernel form (rank 32 / split)
  sgmv_mma_*         segment-tile MMA pair (ranks 16 / 32 / 64, short and long segments)
  sgmv_stream_kernel one-pass streaming kernel (ranks 16 / 32 / 64, partial tiles)
  dense_lora         tcgen05 GEMM with the LoRA epilogue
  build_segments     K6 builder, permute_rows gather / scatter
  sgmv_generic       odd shapes
"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2310_18547_b200 as lsg  # noqa: E402
from tests._util import (DISTINCT, IDENTICAL, SKEWED, UNIFORM, oracle, random_problem, row_norm_err,  # noqa: E402
                         segments_for)

TOL = 8e-3
dev = "cuda"
failures = []
# SAN_MAX_CLUSTER=8: keep every CUDA-core launch within portable cluster sizes (synccheck
# reports 16-CTA clusters at CTA ranks 8 / 9 -- see profiles/round2/sanitizer.md)
MAX_C = int(os.environ.get("SAN_MAX_CLUSTER", "16"))


def cap_cluster(pool, nseg, rows, c):
    """The forced cluster for this case (0 = auto), capped at MAX_C."""
    if c > MAX_C:
        return None
    if c == 0 and lsg.query_launch(pool, nseg, rows)["cluster"] > MAX_C:
        return MAX_C
    return c


def problem(h_in, h_out, r, bounds, seed, dtype=torch.float16, layers=1, layer=0):
    x, A, B = random_problem(h_in, h_out, r, bounds, seed)
    n = len(bounds) - 1
    pool = lsg.AdapterPool(n, layers, h_in, h_out, r, dtype)
    pool.a[:, layer].copy_(torch.tensor(A).to(dtype))
    pool.b[:, layer].copy_(torch.tensor(B).to(dtype))
    xq = torch.tensor(x).to(dtype).to(dev)
    ref = oracle().lora_addon(xq.double().cpu().numpy(), np.asarray(bounds, dtype=np.uint64),
                              pool.a[:, layer].double().cpu().numpy(), pool.b[:, layer].double().cpu().numpy())
    ss = torch.tensor(np.asarray(bounds, dtype=np.int64), dtype=torch.int32, device=dev)
    sl = torch.arange(n, dtype=torch.int32, device=dev)
    return pool, xq, ss, sl, ref


def check(name, y, ref):
    torch.cuda.synchronize()
    e = row_norm_err(y.double().cpu().numpy(), ref)
    status = "ok" if e <= TOL else "FAIL"
    print(f"{status} {name}: err {e:.2e}", flush=True)
    if e > TOL:
        failures.append(name)


def fused_cases():
    for r in (8, 16, 64):
        for pop, batch in ((DISTINCT, 4), (UNIFORM, 9), (IDENTICAL, 5)):
            bounds, _, _ = segments_for(pop, batch, 3)
            pool, x, ss, sl, ref = problem(512, 256, r, bounds, 4)
            for c0 in (0, 1, 4, 16):
                c = cap_cluster(pool, len(bounds) - 1, batch, c0)
                if c is None:
                    continue
                lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, c)
                for mt in (0, 1, 8):
                    lsg.set_option(lsg.LSG_OPT_FORCE_TILE_ROWS, mt)
                    for row_mode in (0, 1):
                        lsg.set_option(lsg._lib.LSG_OPT_NO_ROW_MODE, 1 - row_mode)
                        for pdl in (0, 1):
                            lsg.set_option(lsg.LSG_OPT_PDL, pdl)
                            y = torch.zeros(batch, 256, dtype=torch.float16, device=dev)
                            lsg.sgmv(y, x, pool, ss, sl, 0)
                            check(f"fused r{r} pop{pop} c{c} mt{mt} row{row_mode} pdl{pdl}", y, ref)
                    v = torch.empty(batch, r, dtype=torch.float32, device=dev)
                    y = torch.zeros(batch, 256, dtype=torch.float16, device=dev)
                    if c == 0 and any(lsg.query_launch(pool, len(bounds) - 1, batch, k)["cluster"] > MAX_C
                                      for k in (lsg.KERNEL_SHRINK, lsg.KERNEL_EXPAND)):
                        lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, MAX_C)
                    lsg.sgmv_shrink(v, x, pool, ss, sl, 0)
                    lsg.sgmv_expand(y, v, pool, ss, sl, 0)
                    lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, c)
                    check(f"two-launch r{r} pop{pop} c{c} mt{mt}", y, ref)
            for opt in (lsg.LSG_OPT_FORCE_CLUSTER, lsg.LSG_OPT_FORCE_TILE_ROWS, lsg._lib.LSG_OPT_NO_ROW_MODE,
                        lsg.LSG_OPT_PDL):
                lsg.set_option(opt, 0)
            rs = torch.repeat_interleave(sl, torch.tensor(np.diff(bounds.astype(np.int64)), device=dev)).to(torch.int32)
            y = torch.zeros(batch, 256, dtype=torch.float16, device=dev)
            if lsg.query_launch(pool, len(bounds) - 1, batch, lsg.KERNEL_BGMV)["cluster"] > MAX_C:
                lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, MAX_C)
            lsg.bgmv(y, x, pool, rs, 0)
            lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, 0)
            check(f"bgmv r{r} pop{pop}", y, ref)
    # rank 64 with shared adapters: the automatic 4-row tiles (c3's plan)
    bounds, _, _ = segments_for(SKEWED, 24, 5)
    pool, x, ss, sl, ref = problem(1024, 512, 64, bounds, 6)
    y = torch.zeros(24, 512, dtype=torch.float16, device=dev)
    lsg.sgmv(y, x, pool, ss, sl, 0)
    check("fused r64 4-row tiles", y, ref)


def grouped_cases():
    bounds, _, _ = segments_for(UNIFORM, 12, 7)
    probs = [problem(512, 512, 16, bounds, 10 + i) for i in range(3)]
    ys = [torch.zeros(12, 512, dtype=torch.float16, device=dev) for _ in probs]
    c = cap_cluster(probs[0][0], len(bounds) - 1, 12, 0)
    lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, c or 0)
    lsg.sgmv_multi(ys, [p[1] for p in probs], [p[0] for p in probs], probs[0][2], probs[0][3], 0)
    lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, 0)
    for i, (p, y) in enumerate(zip(probs, ys)):
        check(f"grouped site {i}", y, p[4])


def tc_cases():
    for r, split, gen in ((16, 0, 0), (32, 0, 0), (64, 0, 0), (16, 1, 0), (16, 0, 1), (16, 0, 2), (32, 0, 2)):
        lsg.set_option(lsg._lib.LSG_OPT_TC_SPLIT, split)
        lsg.set_option(lsg._lib.LSG_OPT_TC_LEGACY, gen)
        bounds = np.array([0, 130, 133, 134], dtype=np.uint64)
        pool, x, ss, sl, ref = problem(1024, 1024, r, bounds, 20 + r)
        for pdl in (0, 1):
            lsg.set_option(lsg.LSG_OPT_PDL, pdl)
            y = torch.zeros(134, 1024, dtype=torch.float16, device=dev)
            lsg.sgmv(y, x, pool, ss, sl, 0)
            check(f"tensor-core r{r} split{split} gen{gen} pdl{pdl}", y, ref)
    lsg.set_option(lsg._lib.LSG_OPT_TC_SPLIT, 0)
    lsg.set_option(lsg._lib.LSG_OPT_TC_LEGACY, 0)
    lsg.set_option(lsg.LSG_OPT_PDL, 0)


def mma_cases():
    lsg.set_option(lsg._lib.LSG_OPT_MMA_MIN_ROWS, 1)
    lsg.set_option(lsg._lib.LSG_OPT_TC_LEGACY, 3)
    for r in (16, 32, 64):
        for lens in ((3, 3, 3), (130, 3, 1), (1, 17, 40)):
            bounds = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
            pool, x, ss, sl, ref = problem(512, 256, r, bounds, 50 + r)
            for pdl in (0, 1):
                for fused in (1, 2):  # the two-launch pair, the one-launch form
                    lsg.set_option(lsg.LSG_OPT_PDL, pdl)
                    lsg.set_option(lsg._lib.LSG_OPT_MMA_FUSED, fused)
                    y = torch.zeros(int(bounds[-1]), 256, dtype=torch.float16, device=dev)
                    lsg.sgmv(y, x, pool, ss, sl, 0)
                    check(f"mma {'pair' if fused == 1 else 'one-launch'} r{r} lens{lens} pdl{pdl}", y, ref)
    for opt in (lsg._lib.LSG_OPT_MMA_MIN_ROWS, lsg._lib.LSG_OPT_TC_LEGACY, lsg.LSG_OPT_PDL, lsg._lib.LSG_OPT_MMA_FUSED):
        lsg.set_option(opt, 0)


def stream_cases():
    lsg.set_option(lsg._lib.LSG_OPT_TC_LEGACY, 4)
    for r in (16, 32, 64):
        for lens in ((130, 3, 1), (1, 140, 16, 300)):
            bounds = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
            pool, x, ss, sl, ref = problem(1024, 2048, r, bounds, 60 + r)
            for pdl in (0, 1):
                lsg.set_option(lsg.LSG_OPT_PDL, pdl)
                y = torch.zeros(int(bounds[-1]), 2048, dtype=torch.float16, device=dev)
                lsg.sgmv(y, x, pool, ss, sl, 0)
                check(f"streaming kernel r{r} lens{lens} pdl{pdl}", y, ref)
    for opt in (lsg._lib.LSG_OPT_TC_LEGACY, lsg.LSG_OPT_PDL):
        lsg.set_option(opt, 0)


def dense_cases():
    bounds, _, _ = segments_for(UNIFORM, 16, 8)
    pool, x, ss, sl, ref = problem(1024, 512, 16, bounds, 30)
    w = (torch.rand(1024, 512, device=dev) * 0.1 - 0.05).half()
    y = torch.empty(16, 512, dtype=torch.float16, device=dev)
    if MAX_C < 16:  # its shrink launch (synccheck: clusters <= 8)
        lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, MAX_C)
    lsg.dense_lora(y, x, w, pool, ss, sl, 0)
    lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, 0)
    check("dense_lora", y, x.double().cpu().numpy() @ w.double().cpu().numpy() + ref)


def builder_cases():
    rs = torch.tensor(np.random.default_rng(1).integers(-1, 9, 77).astype(np.int32), device=dev)
    perm, ss, sl, nseg = lsg.build_segments(rs, 8, 3, (10, 20))
    x = torch.randn(77, 64, device=dev).half()
    g = torch.empty_like(x)
    lsg.gather_rows(g, x, perm)
    back = torch.empty_like(x)
    lsg.scatter_rows(back, g, perm)
    torch.cuda.synchronize()
    ok = torch.equal(back, x) and int(nseg.item()) >= 1
    print(f"{'ok' if ok else 'FAIL'} builder + permute", flush=True)
    if not ok:
        failures.append("builder")


def generic_cases():
    bounds, _, _ = segments_for(SKEWED, 10, 2)
    pool, x, ss, sl, ref = problem(96, 40, 12, bounds, 40)
    y = torch.zeros(10, 40, dtype=torch.float16, device=dev)
    lsg.sgmv(y, x, pool, ss, sl, 0)
    check("generic odd shape", y, ref)


def one_cases():
    """python scripts/sanitize.py one <rank> <pop> <batch> <cluster> <tile_rows> <row_mode> <pdl>"""
    r, pop, batch, c, mt, row, pdl = (int(v) for v in sys.argv[2:9])
    bounds, _, _ = segments_for(pop, batch, 3)
    pool, x, ss, sl, ref = problem(512, 256, r, bounds, 4)
    lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, c)
    lsg.set_option(lsg.LSG_OPT_FORCE_TILE_ROWS, mt)
    lsg.set_option(lsg._lib.LSG_OPT_NO_ROW_MODE, 1 - row)
    lsg.set_option(lsg.LSG_OPT_PDL, pdl)
    y = torch.zeros(batch, 256, dtype=torch.float16, device=dev)
    lsg.sgmv(y, x, pool, ss, sl, 0)
    print("launch", lsg.query_launch(pool, len(bounds) - 1, batch))
    check(f"one r{r} pop{pop} b{batch} c{c} mt{mt} row{row} pdl{pdl}", y, ref)


def main():
    torch.cuda.set_device(0)
    if sys.argv[1:2] == ["one"]:
        one_cases()
        sys.exit(1 if failures else 0)
    which = sys.argv[1:] or ["fused", "grouped", "tc", "mma", "stream", "dense", "builder", "generic"]
    for w in which:
        globals()[f"{w}_cases"]()
    print(f"sanitize cases done: {len(failures)} numerical failures", flush=True)
    sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
