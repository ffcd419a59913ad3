"""Phase timeline of the tensor-core SGMV kernel (long segments) inside a
back-to-back CUDA-graph stream, from its %globaltimer phase stamps.

    python scripts/trace_tc.py --segments 2048,1,1 [--hidden 4096 --rank 16]
"""
import argparse
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_18547_b200 as lsg  # noqa: E402
from paper_2310_18547_b200 import _lib  # noqa: E402

SHRINK = ["entry", "weights_staged", "pdl_wait_done", "d1_ready", "partials_in", "end"]
EXPAND = ["entry", "weights_staged", "pdl_wait_done", "y_landed", "d2_ready", "end"]


MMA_P = ["entry", "a_issued", "pdl_wait_done", "stage0_landed", "mma_done", "end"] + [
    f"stage{i}_landed" for i in range(10)]
MMA_E = ["entry", "b_y_issued", "pdl_wait_done", "v_ready", "stage0_landed", "end"] + [
    f"stage{i}_landed" for i in range(8)] + ["partials_landed"]
STREAM = ["entry", "weights_issued", "pdl_wait_done", "stage0_landed", "v_ready", "end"] + [
    f"stage{i}_landed" for i in range(8)] + ["stage3_issued", "stage5_issued"]
FUSED = ["entry", "weights_staged", "pdl_wait_done", "d1_ready", "v_ready", "chunk0_ready", "chunk1_ready",
         "end"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--segments", default="2048," + ",".join(["1"] * 31))
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--sites", type=int, default=16)
    ap.add_argument("--pdl", type=int, default=1)
    ap.add_argument("--split", type=int, default=0, help="1: two-kernel path (LSG_OPT_TC_SPLIT)")
    ap.add_argument("--gen", type=int, default=0,
                    help="LSG_OPT_TC_LEGACY: 0 cluster-free pair, 1 fused, 2 streamed, 3 segment-tile MMA pair")
    ap.add_argument("--mma-min-rows", type=int, default=0, help="LSG_OPT_MMA_MIN_ROWS")
    a = ap.parse_args()
    lsg.set_option(_lib.LSG_OPT_TC_SPLIT, a.split)
    lsg.set_option(_lib.LSG_OPT_TC_LEGACY, a.gen)
    lsg.set_option(_lib.LSG_OPT_MMA_MIN_ROWS, a.mma_min_rows)
    mma = a.gen == 3 or a.mma_min_rows > 0 or a.rank == 64
    two = a.split or a.gen in (0, 3) or mma
    lsg.set_option(lsg.LSG_OPT_PDL, a.pdl)
    lens = [int(v) for v in a.segments.split(",")]
    bounds = [0]
    for n in lens:
        bounds.append(bounds[-1] + n)
    rows, n, h, r = bounds[-1], len(lens), a.hidden, a.rank
    pool = lsg.AdapterPool(n, a.sites, h, h, r, torch.float16)
    pool.a.uniform_(-1, 1)
    pool.b.uniform_(-1, 1)
    xs = torch.empty(a.sites, rows, h, dtype=torch.float16, device="cuda").uniform_(-1, 1)
    ys = torch.zeros_like(xs)
    ss = torch.tensor(bounds, dtype=torch.int32, device="cuda")
    sl = torch.arange(n, dtype=torch.int32, device="cuda")
    ctas = 4096
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
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        step(True)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    allt = buf.view(2 * ctas, 16).cpu().double()
    t0 = None
    names = (MMA_P, MMA_E) if mma else (SHRINK, EXPAND)
    if a.gen == 4:
        two, names = False, None
    groups = ((("shrink", names[0], allt[ctas:ctas + ctas // 2]), ("expand", names[1], allt[ctas + ctas // 2:]))
              if two else (("stream" if a.gen == 4 else "fused", STREAM if a.gen == 4 else FUSED,
                            allt[ctas:ctas + ctas // 2]),))
    for name, phases, part in groups:
        tv = part[part[:, min(len(phases), 6) - 1] != 0]
        if not tv.numel():
            print(f"{name}: no traced CTAs")
            continue
        if t0 is None:
            t0 = tv[:, 0].min()
        print(f"{name}: {tv.shape[0]} live CTAs; us after the first shrink CTA entry: min / median / max")
        for i, ph in enumerate(phases):
            col = (tv[:, i] - t0) / 1e3
            print(f"  {i:2d} {ph:16s} {col.min().item():7.2f} {col.median().item():7.2f} {col.max().item():7.2f}")
    if t0 is None:
        return
    # the CUDA-core kernel's CTAs of the same launch (decode rows), if any
    f = buf.view(2 * ctas, 16)[:ctas].cpu().double()
    fv = f[f[:, 14] != 0]
    if fv.numel():
        print(f"CUDA-core CTAs entered: {fv.shape[0]}, first entry {(fv[:, 14].min() - t0).item() / 1e3:.2f} us, "
              f"last entry {(fv[:, 14].max() - t0).item() / 1e3:.2f} us")


if __name__ == "__main__":
    main()
