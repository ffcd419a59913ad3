"""Needs an instrumented build: scripts/build_variant.sh instr -DLSG_INSTRUMENT, then
LSG_LIB_OVERRIDE=build/variants/instr/libsgmv_b200.so.

Per-phase timeline of one fused SGMV launch inside a back-to-back stream.

Uses the library's phase trace (lsg_set_trace): thread 0 of every CTA stamps
clock64 at the kernel's phase boundaries.  Prints, per phase, the median and
max over CTAs of the time since that CTA's entry, plus the entry skew
(%globaltimer) across CTAs.

    python scripts/trace_phases.py --popularity distinct --batch 64 [--cluster C] [--pdl 1]
"""
import argparse
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_18547_b200 as lsg  # noqa: E402
from paper_2310_18547_b200 import _lib  # noqa: E402
from bench import segments  # noqa: E402

PHASES = ["entry", "metadata", "tma_issued", "pdl_wait_done", "x_landed", "cluster_ready", "shrink_pushed",
          "partials_in", "v_ready", "w0_fma_done", "b_landed", "tile_done", "a_landed", "w0_pushed"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--popularity", default="distinct")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--cluster", type=int, default=0)
    ap.add_argument("--pdl", type=int, default=1)
    ap.add_argument("--sites", type=int, default=64)
    ap.add_argument("--graph", type=int, default=1, help="1: trace inside a CUDA-graph replay (steady state)")
    ap.add_argument("--no-l2-staging", type=int, default=0)
    ap.add_argument("--tile-rows", type=int, default=0)
    ap.add_argument("--segments", default="", help="explicit segment sizes (overrides popularity/batch)")
    a = ap.parse_args()
    lsg.set_option(lsg.LSG_OPT_FORCE_TILE_ROWS, a.tile_rows)
    lsg.set_option(lsg.LSG_OPT_NO_L2_STAGING, a.no_l2_staging)
    lsg.set_option(lsg.LSG_OPT_PDL, a.pdl)
    lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, a.cluster)
    h, r = a.hidden, a.rank
    if a.segments:
        bounds = [0]
        for v in a.segments.split(","):
            bounds.append(bounds[-1] + int(v))
        a.batch = bounds[-1]
    else:
        bounds = segments(a.popularity, a.batch)
    n = len(bounds) - 1
    pool = lsg.AdapterPool(n, a.sites, h, h, r, torch.float16)
    pool.a.uniform_(-1, 1)
    pool.b.uniform_(-1, 1)
    xs = torch.empty(a.sites, a.batch, h, dtype=torch.float16, device="cuda").uniform_(-1, 1)
    ys = torch.zeros_like(xs)
    ss = torch.tensor(bounds, dtype=torch.int32, device="cuda")
    sl = torch.arange(n, dtype=torch.int32, device="cuda")
    info = lsg.query_launch(pool, n, a.batch)
    ctas = info["grid_ctas"]
    buf = torch.zeros(2 * ctas * 16, dtype=torch.int64, device="cuda")
    mid = a.sites // 2

    def step(trace):
        for s in range(a.sites):
            if trace and s == mid:
                _lib.call("lsg_set_trace", C.c_void_p(buf.data_ptr()), ctas)
            lsg.sgmv(ys[s], xs[s], pool, ss, sl, s)
            if trace and s == mid:
                _lib.call("lsg_set_trace", None, 0)

    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        step(False)
    torch.cuda.synchronize()
    if a.graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            step(True)  # the traced launch sits mid-stream, replayed back to back
        for _ in range(5):
            g.replay()
    else:
        with torch.cuda.stream(stream):
            step(True)
    torch.cuda.synchronize()
    t = buf.view(2 * ctas, 16)[:ctas].cpu()
    ghz = 1.965
    rel = (t[:, :14] - t[:, :1]).double() / ghz / 1e3  # us since this CTA's entry
    valid = t[:, 11] != 0
    print(f"config {a.popularity} batch={a.batch} h={h} r={r} launch={info} pdl={a.pdl} traced CTAs={int(valid.sum())}")
    ent = t[valid, 14].double()
    print(f"entry skew across CTAs (globaltimer): {(ent.max() - ent.min()).item() / 1e3:.2f} us")
    for i, name in enumerate(PHASES):
        col = rel[valid, i]
        col = col[t[valid, i] != 0]
        if col.numel():
            print(f"  {i:2d} {name:15s} median {col.median().item():7.2f} us   max {col.max().item():7.2f} us")
    end = ent + rel[valid, 11] * 1e3
    print(f"first entry -> last tile_done: {(end.max() - ent.min()).item() / 1e3:.2f} us")
    # per-CTA phase-to-phase deltas (clock64, exact; the globaltimer anchors below
    # are quantised)
    print("per-CTA deltas (us): median / p90 / max")
    for a_, b_, name in ((3, 4, "wait -> x landed"), (3, 12, "wait -> A landed"), (4, 5, "x -> cluster ready"),
                         (12, 9, "A landed -> w0 FMA done"), (9, 13, "w0 butterfly + push"),
                         (13, 7, "w0 pushed -> partials in"), (7, 8, "reduce"), (8, 10, "v -> B landed"),
                         (10, 11, "expand + store"), (3, 11, "wait -> tile done")):
        ok = (t[valid, a_] != 0) & (t[valid, b_] != 0)
        d = (rel[valid, b_] - rel[valid, a_])[ok]
        if d.numel():
            print(f"  {name:26s} {d.median().item():6.2f} {d.quantile(0.9).item():6.2f} {d.max().item():6.2f}")
    # absolute timeline anchored at the earliest return from griddepcontrol.wait
    # (= the previous launch's completion in a back-to-back stream)
    absu = ent.unsqueeze(1) / 1e3 + rel[valid]  # us
    t0 = absu[:, 3].min()
    print("absolute (us after the first pdl_wait return): median / max over CTAs")
    for i, name in enumerate(PHASES):
        col = absu[:, i] - t0
        ok = t[valid, i] != 0
        if ok.any():
            print(f"  {i:2d} {name:15s} {col[ok].median().item():7.2f}  {col[ok].max().item():7.2f}")


if __name__ == "__main__":
    main()
