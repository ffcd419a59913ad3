#!/usr/bin/env python
"""SGMV benchmark -- BASELINE.json metric "SGMV us/layer & HBM GB/s vs batch across
Distinct/Uniform/Skewed/Identical", headline workload configs[1]:

    Llama-2-7B  h=4096, r=16, batch 64 decode rows, Distinct popularity, 1x B200

A *step* is one decode step's LoRA work: 7 projection sites x 32 layers = 224
fused SGMV launches (one shrink+expand pair each -- the paper's "LoRA operator",
PAPER.md:516), every launch on its own (site, layer) weights and its own x / y
buffers, replayed from a CUDA graph.  ``value`` is microseconds per LoRA site
(= "us/layer" in the reference's sense, cost_model.cpp:53-61), lower is better.
Weights rotate over a 3.7 GB pool and x/y over 235 MB per step, so every launch
reads HBM, not L2 (config.l2 says so).

Algorithmic bytes per launch (cost_model.cpp:59):
    2 * (s_n * (h + r) + n * h * r) * 2 B  = 17,829,888 B at the headline config.

--impl reference times the reference's own CPU SGMV (oracle/_ref, compiled from
/root/reference/proj/core/src/sgmv.cpp; else the oracle/ restatement) on all
host cores for the same metric/config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

POPS = {"distinct": 0, "uniform": 1, "skewed": 2, "identical": 3}
SITES_PER_LAYER, LAYERS = 7, 32


PRESETS = {
    "c1": dict(hidden=4096, rank=16, batch=32, segments="8,8,8,8"),
    "c2": dict(hidden=4096, rank=16, batch=64, popularity="distinct"),
    "c3": dict(hidden=5120, rank=64, batch=64, popularity="uniform"),
    "c3-bgmv": dict(hidden=5120, rank=64, batch=64, popularity="uniform", kernel="bgmv"),
    "c4": dict(hidden=4096, rank=16, prefill=2048, sites=32),
    "c5": dict(hidden=8192, rank=16, batch=64, popularity="distinct", slots=1000, sites=32),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--popularity", choices=list(POPS), default="distinct")
    ap.add_argument("--dtype", choices=["fp16", "bf16"], default="fp16")
    ap.add_argument("--pdl", type=int, default=1)
    ap.add_argument("--cluster", type=int, default=0, help="force the split-K cluster size (0 = library heuristic)")
    ap.add_argument("--tile-rows", type=int, default=0, help="force rows per tile, 1 or 8 (0 = heuristic)")
    ap.add_argument("--no-l2-staging", action="store_true", help="keep B resident from kernel entry")
    ap.add_argument("--l2-staging", action="store_true", help="always stage B through L2 into A's smem")
    ap.add_argument("--no-tc", action="store_true", help="long segments stay on the CUDA-core kernel")
    ap.add_argument("--tc-split", action="store_true", help="two-kernel tensor-core path for rank-16 long segments")
    ap.add_argument("--no-row-mode", action="store_true", help="segment-major decode for one-row tiles")
    ap.add_argument("--kernel", choices=["sgmv", "bgmv"], default="sgmv",
                    help="sgmv: segmented launch; bgmv: per-row adapter slots (decode BGMV)")
    ap.add_argument("--slots", type=int, default=0, help="adapter-pool slots (0 = one per segment)")
    ap.add_argument("--segments", default="", help="explicit segment sizes, e.g. 8,8,8,8 (overrides popularity)")
    ap.add_argument("--prefill", type=int, default=0, help="mixed batch: one prefill segment of this many rows "
                    "plus 31 distinct decode rows (configs[3])")
    ap.add_argument("--preset", choices=["c1", "c2", "c3", "c3-bgmv", "c4", "c5"], default="",
                    help="BASELINE.json configs: c1 h4096 r16 32 rows/4 LoRAs; c2 headline; c3 h5120 r64 uniform; "
                         "c4 prefill 2048 + 31 decodes; c5 h8192 r16 1000-slot pool")
    ap.add_argument("--sites", type=int, default=SITES_PER_LAYER * LAYERS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="also print per-(popularity,batch) lines to stderr")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no graph, no extras)")
    ap.add_argument("--profile-graph", action="store_true",
                    help="short run for ncu --graph-profiling graph: capture the step graph, replay it twice")
    pre, _ = ap.parse_known_args()
    ap.set_defaults(**PRESETS.get(pre.preset, {}))  # a preset sets defaults; explicit flags still win
    a = ap.parse_args()
    if a.prefill:
        a.segments = ",".join([str(a.prefill)] + ["1"] * 31)
    if a.segments:
        a.batch = sum(int(x) for x in a.segments.split(","))
    return a


def alg_bytes(rows, nseg, h, r, e=2):
    return 2 * (rows * (h + r) + nseg * h * r) * e  # cost_model.cpp:59


def alg_flop(rows, h, r):
    return 4 * rows * h * r  # cost_model.cpp:58


def segments(pop: str, batch: int, seed: int = 11):
    """assign_models grouped by ascending id (experiments.cpp:56-76), via the workload port."""
    from paper_2310_18547_b200.workload import assign_models
    ids = assign_models(batch, POPS[pop], 1.5, seed)
    uniq = sorted(set(ids))
    bounds = [0]
    for u in uniq:
        bounds.append(bounds[-1] + sum(1 for i in ids if i == u))
    return bounds


def workload_name(a):
    model = {4096: "llama2-7b", 5120: "llama2-13b", 8192: "llama2-70b"}.get(a.hidden, "custom")
    shape = (f"prefill {a.prefill} + 31 decode" if a.prefill else
             f"segments {a.segments}" if a.segments else f"batch={a.batch} decode {a.popularity}")
    return f"{model}-lora h={a.hidden} r={a.rank} {shape} {a.kernel} ({a.dtype})"


def bounds_for(a, world=1):
    """Segment boundaries of the (global) batch: ``world`` copies of the per-GPU batch."""
    if a.segments:
        b = [0]
        for _ in range(world):
            for x in a.segments.split(","):
                b.append(b[-1] + int(x))
        return b
    return segments(a.popularity, a.batch * world)


# ----------------------------------------------------------------------------------
# clocks (NVML, sampled every 10 ms during the timed region)
# ----------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.ok = [], 0, False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------------
# CPU baselines
# ----------------------------------------------------------------------------------
def _cpu_problem(a, seed=5):
    from oracle.oracle import Oracle
    o = Oracle()
    bounds = np.array(bounds_for(a), dtype=np.uint64)
    g = o.rng(seed)
    n = len(bounds) - 1
    h, r = a.hidden, a.rank
    x = g.fill_pm1(a.batch * h).reshape(a.batch, h)
    A = g.fill_pm1(n * h * r).reshape(n, h, r)
    B = g.fill_pm1(n * r * h).reshape(n, r, h)
    # the CPU gets the dequantised 16-bit values, like the GPU
    q = np.float16 if a.dtype == "fp16" else np.float32
    return [np.asarray(t.astype(q), dtype=np.float64) for t in (x, A, B)] + [bounds]


def cpu_impl():
    from oracle.oracle import Oracle, Reference, reference_available
    if reference_available():
        return Reference(), "reference"
    return Oracle(), "port"


def cpu_baseline(a, budget_s=10.0):
    """Reference SGMV (fp64, 1 thread, as shipped) on a bounded sample of the workload."""
    impl, kind = cpu_impl()
    x, A, B, bounds = _cpu_problem(a)
    impl.lora_addon(x, bounds, A, B)  # warm
    n, t0 = 0, time.perf_counter()
    while True:
        impl.lora_addon(x, bounds, A, B)
        n += 1
        el = time.perf_counter() - t0
        if el >= budget_s or n >= 2000:
            break
    return {"value": el / n * 1e6, "unit": "us/layer", "cores": 1, "kind": kind,
            "sample": f"{n} x lora_addon(batch={a.batch}, {a.popularity}, h={a.hidden}, r={a.rank}) fp64 "
                      f"on dequantised {a.dtype} inputs, {el:.1f} s, 1 thread ({'oracle/_ref' if kind == 'reference' else 'oracle port'})"}


def run_reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    impl, kind = cpu_impl()
    threads = os.cpu_count() or 1
    problems = [_cpu_problem(a, seed=5 + t) for t in range(threads)]

    def one_step():
        ths = [threading.Thread(target=impl.lora_addon, args=(p[0], p[3], p[1], p[2])) for p in problems]
        for t in ths:
            t.start()
        for t in ths:
            t.join()

    for _ in range(a.warmup):
        one_step()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        one_step()
    el = time.perf_counter() - t0
    sites = a.steps * threads
    us = el / sites * 1e6
    line = {"metric": "SGMV us/layer (LoRA shrink+expand per projection site)", "value": us, "unit": "us/layer",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": el / a.steps * 1e3,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": workload_name(a), "hidden": a.hidden, "rank": a.rank, "batch": a.batch,
                       "popularity": a.popularity, "step": f"{threads} concurrent lora_addon calls (one per host thread)"},
            "cpu_baseline": {"value": us, "unit": "us/layer", "cores": threads, "kind": kind,
                             "sample": f"{sites} lora_addon calls over {threads} threads, {el:.1f} s"},
            "e2e": {"value": us, "unit": "us/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------------
def main():
    a = parse()
    if a.impl == "reference":
        run_reference_arm(a)
        return

    import torch
    import torch.distributed as dist

    import paper_2310_18547_b200 as lsg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # One process per GPU.  LSG_BENCH_BACKEND=gloo (test only) lets the N>1 code path
    # run with several ranks sharing one GPU; the product path is NCCL.
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        backend = os.environ.get("LSG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    dtype = torch.float16 if a.dtype == "fp16" else torch.bfloat16
    lsg.set_option(lsg.LSG_OPT_PDL, a.pdl)
    lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, a.cluster)
    lsg.set_option(lsg.LSG_OPT_FORCE_TILE_ROWS, a.tile_rows)
    lsg.set_option(lsg.LSG_OPT_NO_L2_STAGING, 1 if a.no_l2_staging else -1 if a.l2_staging else 0)
    lsg.set_option(lsg.LSG_OPT_NO_TENSOR_CORES, int(a.no_tc))
    lsg.set_option(lsg._lib.LSG_OPT_TC_SPLIT, int(a.tc_split))
    lsg.set_option(lsg._lib.LSG_OPT_NO_ROW_MODE, int(a.no_row_mode))
    h, r, batch, sites = a.hidden, a.rank, a.batch, a.sites
    # Request-partitioned weak scaling: the global batch is `batch` rows per GPU; the
    # partitioner (lsg_partition_segments) hands every rank whole segments (or row
    # ranges of dominant ones) and each rank runs its share on its own replica of
    # the adapter pool -- no collective on the data path.
    from paper_2310_18547_b200.partition import rank_batches
    gbounds = bounds_for(a, world)
    mine = rank_batches(np.array(gbounds, dtype=np.int32), h, h, r, world)[rank]
    bounds = [int(v) for v in mine.seg_starts]
    batch = mine.num_rows
    nseg = len(bounds) - 1
    # The serving engine knows its step's segment lengths: a decode-only step (no segment
    # of >= 128 rows) skips the tensor-core pass (LSG_OPT_TC_MIN_ROWS, include/lsg_sgmv.h).
    if max(np.diff(bounds), default=0) < 128:
        lsg.set_option(lsg._lib.LSG_OPT_TC_MIN_ROWS, batch + 1)
    gen = torch.Generator(device="cuda").manual_seed(1000 + rank)
    nslots = max(a.slots, nseg)
    pool = lsg.AdapterPool(nslots, sites, h, h, r, dtype)
    pool.a.uniform_(-1, 1, generator=gen)
    pool.b.uniform_(-1, 1, generator=gen)
    xs = torch.empty(sites, batch, h, dtype=dtype, device="cuda").uniform_(-1, 1, generator=gen)
    ys = torch.zeros(sites, batch, h, dtype=dtype, device="cuda")
    seg_starts = torch.tensor(bounds, dtype=torch.int32, device="cuda")
    # the batch's adapters are distinct slots spread over the pool
    slots = torch.randperm(nslots, generator=torch.Generator().manual_seed(7 + rank))[:nseg].to(torch.int32)
    seg_slot = slots.cuda()
    row_slot = torch.repeat_interleave(slots, torch.tensor(np.diff(bounds))).to(torch.int32).cuda()
    bytes_per_launch = alg_bytes(batch, nseg, h, r)
    info = lsg.query_launch(pool, nseg, batch, lsg.KERNEL_BGMV if a.kernel == "bgmv" else lsg.KERNEL_FUSED)

    def launch(s):
        if a.kernel == "bgmv":
            lsg.bgmv(ys[s], xs[s], pool, row_slot, s)
        else:
            lsg.sgmv(ys[s], xs[s], pool, seg_starts, seg_slot, s)

    def step():
        for s in range(sites):
            launch(s)

    stream = torch.cuda.Stream()
    torch.cuda.synchronize()
    if a.profile:
        with torch.cuda.stream(stream):
            for _ in range(max(1, a.warmup)):
                step()
        torch.cuda.synchronize()
        return
    with torch.cuda.stream(stream):
        step()  # eager warm-up (sets function attributes before capture)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        step()
    if a.profile_graph:
        with torch.cuda.stream(stream):
            graph.replay()
            torch.cuda.nvtx.range_push("lsg_graph")  # ncu --nvtx --nvtx-include lsg_graph/
            graph.replay()
            torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        return
    for _ in range(max(3, a.warmup)):
        graph.replay()
    torch.cuda.synchronize()

    def timed(fn, k):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(k):
                fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        return ms

    with ClockSampler(dev) as clk:
        ms = timed(graph.replay, a.steps)
    ms_step = ms / a.steps
    us_site = ms_step * 1e3 / sites  # per-rank device time per launch
    value = ms * 1e3 / (a.steps * sites * world)  # whole job: max-over-ranks time / all sites

    extra = {}
    # isolated single-launch latency (no PDL overlap), L2 flushed between launches
    lsg.set_option(lsg.LSG_OPT_PDL, 0)
    flush = torch.empty(1024 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > L2; hides launch latency
    lat = []
    for i in range(20):
        with torch.cuda.stream(stream):
            flush.zero_()  # same stream: evicts L2 and covers the host launch latency
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            launch(i)
            e1.record(stream)
        torch.cuda.synchronize()
        lat.append(e0.elapsed_time(e1) * 1e3)
    extra["isolated_launch_us_median"] = statistics.median(lat)
    graph_nopdl = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph_nopdl, stream=stream):
        step()
    graph_nopdl.replay()
    ms_nopdl = timed(graph_nopdl.replay, max(3, a.steps // 2)) / max(3, a.steps // 2)
    extra["us_per_launch_no_pdl"] = ms_nopdl * 1e3 / sites
    lsg.set_option(lsg.LSG_OPT_PDL, a.pdl)
    del flush
    # Grouped launches (lsg_sgmv_multi): per layer q/k/v in one launch, o, gate/up in
    # one launch, down -- 4 launches for the 7 sites, same bytes and results.
    if a.kernel == "sgmv" and sites % SITES_PER_LAYER == 0:
        groups = []
        for l in range(sites // SITES_PER_LAYER):
            b0 = l * SITES_PER_LAYER
            groups += [[b0, b0 + 1, b0 + 2], [b0 + 3], [b0 + 4, b0 + 5], [b0 + 6]]

        views = {s_: pool.layer_view(s_) for g in groups if len(g) > 1 for s_ in g}  # before capture

        def step_grouped():
            for g in groups:
                if len(g) == 1:
                    launch(g[0])
                else:  # the sites' weights are layers g[i] of the one bench pool (same slots)
                    lsg.sgmv_multi([ys[s_] for s_ in g], [xs[s_] for s_ in g],
                                   [views[s_] for s_ in g], seg_starts, seg_slot, 0)

        with torch.cuda.stream(stream):
            step_grouped()
        torch.cuda.synchronize()
        graph_g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph_g, stream=stream):
            step_grouped()
        with torch.cuda.stream(stream):
            graph_g.replay()
        kg = max(3, a.steps // 2)
        extra["grouped_us_per_site"] = timed(graph_g.replay, kg) * 1e3 / (kg * sites * world)  # as `value`
        extra["grouped_launches_per_layer"] = 4


    # e2e through the public API: every step copies that step's activations in from
    # pinned host memory (one H2D of all sites' x) and its outputs back (one D2H of
    # all sites' y).  Steps are pipelined over two device buffer sets and three
    # streams (H2D / compute / D2H), the way a serving loop overlaps PCIe with the
    # kernels; timed with CUDA events from the first H2D to the last D2H.
    e2e = None
    if not a.no_e2e:
        hx = torch.empty(sites, batch, h, dtype=dtype, pin_memory=True)
        hx.copy_(xs.cpu())
        hy = torch.empty(sites, batch, h, dtype=dtype, pin_memory=True)
        bufs = [(xs, ys), (torch.empty_like(xs), torch.zeros_like(ys))]
        graphs = [graph]
        xs1, ys1 = bufs[1]
        g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1, stream=stream):
            for s_ in range(sites):
                if a.kernel == "bgmv":
                    lsg.bgmv(ys1[s_], xs1[s_], pool, row_slot, s_)
                else:
                    lsg.sgmv(ys1[s_], xs1[s_], pool, seg_starts, seg_slot, s_)
        graphs.append(g1)
        h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
        ev_in = [torch.cuda.Event(), torch.cuda.Event()]
        ev_done = [torch.cuda.Event(), torch.cuda.Event()]
        ev_out = [torch.cuda.Event(), torch.cuda.Event()]

        def run_e2e(k):
            for i in range(k):
                b = i % 2
                xb, yb = bufs[b]
                if i >= 2:
                    h2d.wait_event(ev_done[b])       # step i-2's kernels are done with xb
                with torch.cuda.stream(h2d):
                    xb.copy_(hx, non_blocking=True)
                    ev_in[b].record(h2d)
                stream.wait_event(ev_in[b])
                if i >= 2:
                    stream.wait_event(ev_out[b])     # step i-2's outputs have left yb
                with torch.cuda.stream(stream):
                    graphs[b].replay()
                    ev_done[b].record(stream)
                d2h.wait_event(ev_done[b])
                with torch.cuda.stream(d2h):
                    hy.copy_(yb, non_blocking=True)
                    ev_out[b].record(d2h)

        run_e2e(2)
        torch.cuda.synchronize()
        ke = max(4, min(a.steps, 10))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(h2d)
        run_e2e(ke)
        e1.record(d2h)
        torch.cuda.synchronize()
        ms_e2e = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms_e2e], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_e2e = t.item()
        e2e = {"value": ms_e2e * 1e3 / (ke * sites * world), "unit": "us/layer",
               "h2d_bytes_per_step": int(hx.numel() * hx.element_size()),
               "d2h_bytes_per_step": int(hy.numel() * hy.element_size()),
               "how": "per step: one pinned H2D of all x, the step graph, one D2H of all y; "
                      "pipelined over 2 buffer sets (PCIe-bound)"}
        del bufs, xs1, ys1

    if a.sweep and rank == 0:
        sweep(a, lsg, torch, dtype, stream)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if peak else "fallback (B200_PROFILING.md 6.65 TB/s)"
    peak = peak or 6650.0
    achieved = bytes_per_launch / (us_site * 1e-6) / 1e9
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        key = f"h{h}_r{r}_b{batch}_{a.popularity}_{a.dtype}"
        traffic = prof.get(key)
    except Exception:
        pass
    line = {
        "metric": "SGMV us/layer (LoRA shrink+expand per projection site)",
        "value": value, "unit": "us/layer", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms_step, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": a.dtype + " (fp32 accumulate)", "data": "synthetic (U[-1,1) adapters/activations, random init)",
        "config": {"workload": workload_name(a), "model": "Llama-2-7B LoRA sites (h x h)", "hidden": h, "rank": r,
                   "batch_per_gpu": a.batch, "global_batch": a.batch * world, "segments": nseg,
                   "global_segments": len(gbounds) - 1, "rank0_rows": batch,
                   "popularity": a.popularity, "step": f"{sites} fused SGMV launches (7 sites x 32 layers), CUDA graph",
                   "parallelism": f"request-partitioned x{world} (no collective)",
                   "kernel": a.kernel, "pool_slots": nslots, "preset": a.preset or None,
                   "l2": "inputs larger than L2: weights rotate over a "
                         f"{pool.a.numel() * 2 * 2 / 2**30:.2f} GiB pool, x/y over {2 * xs.numel() * 2 / 2**20:.0f} MiB per step",
                   "pdl": bool(a.pdl), "launch": info},
        "hbm_gbs": achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "alg_bytes_per_launch": bytes_per_launch, "flop_per_launch": alg_flop(batch, h, r)},
        "gpu_launches": a.steps * sites,
        "clocks": clk.summary(),
        "e2e": e2e,
        **extra,
    }
    if not a.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(a)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def sweep(a, lsg, torch, dtype, stream):
    """Batch x popularity sweep at the configured shape (reported on stderr)."""
    h, r = a.hidden, a.rank
    for pop in ("distinct", "uniform", "skewed", "identical"):
        for batch in (1, 2, 4, 8, 16, 32, 64):
            bounds = segments(pop, batch)
            nseg = len(bounds) - 1
            L = 224
            pool = lsg.AdapterPool(nseg, L, h, h, r, dtype)
            pool.a.uniform_(-1, 1)
            pool.b.uniform_(-1, 1)
            xs = torch.empty(L, batch, h, dtype=dtype, device="cuda").uniform_(-1, 1)
            ys = torch.zeros(L, batch, h, dtype=dtype, device="cuda")
            ss = torch.tensor(bounds, dtype=torch.int32, device="cuda")
            sl = torch.arange(nseg, dtype=torch.int32, device="cuda")
            with torch.cuda.stream(stream):
                for s in range(L):
                    lsg.sgmv(ys[s], xs[s], pool, ss, sl, s)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for s in range(L):
                    lsg.sgmv(ys[s], xs[s], pool, ss, sl, s)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):  # replay on the stream the events are recorded on
                for _ in range(3):
                    g.replay()
                e0.record(stream)
                for _ in range(10):
                    g.replay()
                e1.record(stream)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (10 * L)
            b = alg_bytes(batch, nseg, h, r)
            sys.stderr.write(json.dumps({"sweep": True, "popularity": pop, "batch": batch, "segments": nseg,
                                         "us_per_launch": us, "alg_bytes": b, "gbs": b / us / 1e3,
                                         "launch": lsg.query_launch(pool, nseg, batch)}) + "\n")
            del pool, xs, ys


if __name__ == "__main__":
    main()
