#!/usr/bin/env python
"""SGMV benchmark -- BASELINE.json metric "SGMV us/layer & HBM GB/s vs batch across
Distinct/Uniform/Skewed/Identical", headline workload configs[1]:

    Llama-2-7B  h=4096, r=16, batch 64 decode rows, Distinct popularity, 1x B200

A *step* is one decode step's LoRA work: 7 projection sites x 32 layers = 224
fused SGMV launches (one shrink+expand pair each -- the paper's "LoRA operator",
PAPER.md:516), every launch on its own (site, layer) weights and its own x / y
buffers, replayed from a CUDA graph.  ``value`` is microseconds per LoRA site
(= "us/layer" in the reference's sense, cost_model.cpp:53-61), lower is better.
Weights rotate over a 3.5 GiB pool and x/y over 224 MiB per step, so every launch
reads HBM, not L2 (config.l2 says so).

Algorithmic bytes per launch (cost_model.cpp:59):
    2 * (s_n * (h + r) + n * h * r) * 2 B  = 17,829,888 B at the headline config.

The default N=1 line also carries, so that the driver's own run records them:
  * ``sweep``    batch 1..64 x Distinct/Uniform/Skewed/Identical (the metric's "vs batch
                 across" part), us per launch and fraction of the HBM roofline;
  * ``configs``  the other BASELINE configs (c1, c3 SGMV and BGMV, c4 prefill 128 and
                 2048, c5 1000-slot pool), same bookkeeping;
  * ``roofline.traffic`` and ``configs[*].traffic``: DRAM bytes per launch of THIS build,
                 measured by an ncu pass over one probe run (counters, never timings);
  * ``cpu_baseline``: the reference's own lora_addon on a Batch built once
                 (bench_sgmv.cpp:37-47), one pinned core, with the shrink/expand split.

Multi-GPU (one process per GPU, request-partitioned, no collective on the data path):
``--gpus N`` re-launches itself under torch.distributed.run when WORLD_SIZE is unset.
``--scaling weak`` (default): 64 rows per GPU, value = max-over-ranks time per
64-row site-equivalent of the whole job; ``--scaling strong``: 64 rows in all,
partitioned, value = max-over-ranks time per site.

--impl reference times the reference's own CPU SGMV (oracle/_ref, compiled from
/root/reference/proj/core/src/sgmv.cpp; else the oracle/ restatement) on all
host cores for the same metric/config.
"""
from __future__ import annotations

import argparse
import csv
import hashlib
import io
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

POPS = {"distinct": 0, "uniform": 1, "skewed": 2, "identical": 3}
SITES_PER_LAYER, LAYERS = 7, 32
METRIC = "SGMV us/layer (LoRA shrink+expand per projection site)"

PRESETS = {
    "c1": dict(hidden=4096, rank=16, batch=32, segments="8,8,8,8"),
    "c2": dict(hidden=4096, rank=16, batch=64, popularity="distinct"),
    "c3": dict(hidden=5120, rank=64, batch=64, popularity="uniform"),
    "c3-bgmv": dict(hidden=5120, rank=64, batch=64, popularity="uniform", kernel="bgmv"),
    "c3-skewed": dict(hidden=5120, rank=64, batch=64, popularity="skewed"),
    "c4": dict(hidden=4096, rank=16, prefill=2048, sites=32),
    "c4-128": dict(hidden=4096, rank=16, prefill=128, sites=64),
    "c5": dict(hidden=8192, rank=16, batch=64, popularity="distinct", slots=1000, sites=32),
}
EXTRA_CONFIGS = ["c1", "c3", "c3-skewed", "c3-bgmv", "c4-128", "c4", "c5"]


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak: 64 rows per GPU; strong: 64 rows in all, partitioned over the GPUs")
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
    ap.add_argument("--tc-gen", type=int, default=0, help="LSG_OPT_TC_LEGACY (long-segment kernel generation)")
    ap.add_argument("--mma-min-rows", type=int, default=0, help="LSG_OPT_MMA_MIN_ROWS (0 = auto)")
    ap.add_argument("--mma-fused", type=int, default=0, help="LSG_OPT_MMA_FUSED: 0 / 1 the two-launch pair, 2 one launch")
    ap.add_argument("--tc-min-rows", type=int, default=0,
                    help="per-call tensor-core row threshold (0 = from the step's own segment plan)")
    ap.add_argument("--kernel", choices=["sgmv", "bgmv"], default="sgmv",
                    help="sgmv: segmented launch; bgmv: per-row adapter slots (decode BGMV)")
    ap.add_argument("--slots", type=int, default=0, help="adapter-pool slots (0 = one per segment)")
    ap.add_argument("--segments", default="", help="explicit segment sizes, e.g. 8,8,8,8 (overrides popularity)")
    ap.add_argument("--prefill", type=int, default=0, help="mixed batch: one prefill segment of this many rows "
                    "plus 31 distinct decode rows (configs[3])")
    ap.add_argument("--preset", choices=sorted(PRESETS), default="",
                    help="BASELINE.json configs: c1 h4096 r16 32 rows/4 LoRAs; c2 headline; c3 h5120 r64 uniform; "
                         "c4 prefill 2048 + 31 decodes; c5 h8192 r16 1000-slot pool")
    ap.add_argument("--sites", type=int, default=SITES_PER_LAYER * LAYERS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="headline only: no sweep / configs / traffic pass")
    ap.add_argument("--no-traffic", action="store_true", help="skip the ncu DRAM-traffic pass")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no graph, no extras)")
    ap.add_argument("--profile-graph", action="store_true",
                    help="short run for ncu --graph-profiling graph: capture the step graph, replay it twice")
    ap.add_argument("--traffic-probe", action="store_true", help=argparse.SUPPRESS)
    pre, _ = ap.parse_known_args(argv)
    ap.set_defaults(**PRESETS.get(pre.preset, {}))  # a preset sets defaults; explicit flags still win
    a = ap.parse_args(argv)
    normalise(a)
    return a


def normalise(a):
    if a.prefill:
        a.segments = ",".join([str(a.prefill)] + ["1"] * 31)
    if a.segments:
        a.batch = sum(int(x) for x in a.segments.split(","))
    return a


def cfg_args(name: str, base=None):
    """An argparse namespace for preset `name` (the other fields from `base` / defaults)."""
    a = parse([] if base is None else [])
    for k, v in PRESETS[name].items():
        setattr(a, k, v)
    a.preset = name
    if base is not None:
        a.dtype, a.pdl = base.dtype, base.pdl
    return normalise(a)


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


def bounds_for(a, copies=1):
    """Segment boundaries of `copies` concatenated per-GPU batches."""
    if a.segments:
        b = [0]
        for _ in range(copies):
            for x in a.segments.split(","):
                b.append(b[-1] + int(x))
        return b
    return segments(a.popularity, a.batch * copies)


def global_bounds(a, world):
    """Weak scaling: the global batch is `batch` rows per GPU; strong: `batch` rows in all."""
    return bounds_for(a, world if a.scaling == "weak" else 1)


def host_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "allowed_cpus": len(os.sched_getaffinity(0)), "cpu_model": model}


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
# CPU baselines (the reference's own SGMV; oracle/ is reached only from these legs)
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


def _time_cpu(impl, kind, prob, op, budget_s):
    """Seconds per call of `op` on problem `prob`.  The reference build times a Batch built
    once (bench_sgmv.cpp:37-47); the port (oracle/ restatement, no Batch type) times its
    array entry point."""
    x, A, B, bounds = prob
    if kind == "reference":
        return impl.bench_batch(x, bounds, A, B, op, budget_s=budget_s)
    fn = {"lora_addon": lambda: impl.lora_addon(x, bounds, A, B),
          "sgmv_shrink": lambda: impl.sgmv_shrink(x, bounds, A),
          "sgmv_expand": lambda: impl.sgmv_expand(v, bounds, B)}[op]
    v = impl.sgmv_shrink(x, bounds, A) if op == "sgmv_expand" else None
    n, t0 = 0, time.perf_counter()
    while True:
        fn()
        n += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            return el / n, n


def cpu_baseline(a, budget_s=6.0):
    """Reference SGMV (fp64, as shipped) on a Batch built once, one thread pinned to one core
    (taskset -c <core>), lora_addon plus the shrink / expand split."""
    impl, kind = cpu_impl()
    prob = _cpu_problem(a)
    old = os.sched_getaffinity(0)
    core = min(old)
    os.sched_setaffinity(0, {core})
    try:
        _time_cpu(impl, kind, prob, "lora_addon", 0.2)  # warm
        t_add, n_add = _time_cpu(impl, kind, prob, "lora_addon", budget_s)
        t_sh, n_sh = _time_cpu(impl, kind, prob, "sgmv_shrink", budget_s / 2)
        t_ex, n_ex = _time_cpu(impl, kind, prob, "sgmv_expand", budget_s / 2)
    finally:
        os.sched_setaffinity(0, old)
    return {"value": t_add * 1e6, "unit": "us/layer", "cores": 1, "kind": kind,
            "shrink_us": t_sh * 1e6, "expand_us": t_ex * 1e6, "pinned_core": core, **host_info(),
            "sample": f"{n_add} x lora_addon(batch={a.batch}, {a.popularity}, h={a.hidden}, r={a.rank}) fp64 on "
                      f"dequantised {a.dtype} inputs, Batch built once (bench_sgmv.cpp:37-47), "
                      f"{t_add * n_add:.1f} s, 1 thread pinned to core {core} "
                      f"({'oracle/_ref' if kind == 'reference' else 'oracle port'}); "
                      f"split: {n_sh} x sgmv_shrink, {n_ex} x sgmv_expand"}


def run_reference_arm(a):
    """The reference's lora_addon on every host core at once (one prebuilt Batch and one
    pinned thread per core); a step is one call per thread."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    impl, kind = cpu_impl()
    cores = sorted(os.sched_getaffinity(0))
    threads = len(cores)
    problems = [_cpu_problem(a, seed=5 + t) for t in range(threads)]
    start, done = threading.Barrier(threads + 1), threading.Barrier(threads + 1)
    stop = [False]

    def worker(t):
        os.sched_setaffinity(0, {cores[t]})  # this thread only
        while True:
            start.wait()
            if stop[0]:
                return
            _time_cpu(impl, kind, problems[t], "lora_addon", 0.0)  # exactly one call
            done.wait()

    ths = [threading.Thread(target=worker, args=(t,), daemon=True) for t in range(threads)]
    for t in ths:
        t.start()

    def one_step():
        start.wait()
        done.wait()

    for _ in range(a.warmup):
        one_step()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        one_step()
    el = time.perf_counter() - t0
    stop[0] = True
    start.wait()
    sites = a.steps * threads
    us = el / sites * 1e6
    line = {"metric": METRIC, "value": us, "unit": "us/layer",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": el / a.steps * 1e3,
            "higher_is_better": False, "scaling": a.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": workload_name(a), "hidden": a.hidden, "rank": a.rank, "batch": a.batch,
                       "popularity": a.popularity,
                       "step": f"{threads} concurrent lora_addon calls (one prebuilt Batch and one pinned thread "
                               f"per host core)"},
            "cpu_baseline": {"value": us, "unit": "us/layer", "cores": threads, "kind": kind, **host_info(),
                             "sample": f"{sites} lora_addon calls over {threads} pinned threads, {el:.1f} s "
                                       f"(aggregate: wall time / calls)"},
            "e2e": {"value": us, "unit": "us/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------
# GPU workloads
# ----------------------------------------------------------------------------------
class Workload:
    """One config's device state: adapter pool (one layer per projection site), x / y per
    site, the segment plan, and the launch of site s."""

    def __init__(self, lsg, torch, a, bounds, dtype, seed=1000, slot_seed=7, sites=None):
        self.lsg, self.torch, self.a = lsg, torch, a
        h, r = a.hidden, a.rank
        self.sites = sites or a.sites
        self.bounds = [int(v) for v in bounds]
        self.rows = self.bounds[-1]
        self.nseg = len(self.bounds) - 1
        gen = torch.Generator(device="cuda").manual_seed(seed)
        self.nslots = max(a.slots, self.nseg, 1)
        self.pool = lsg.AdapterPool(self.nslots, self.sites, h, h, r, dtype)
        self.pool.a.uniform_(-1, 1, generator=gen)
        self.pool.b.uniform_(-1, 1, generator=gen)
        self.xs = torch.empty(self.sites, max(self.rows, 1), h, dtype=dtype, device="cuda").uniform_(
            -1, 1, generator=gen)
        self.ys = torch.zeros(self.sites, max(self.rows, 1), h, dtype=dtype, device="cuda")
        self.seg_starts = torch.tensor(self.bounds, dtype=torch.int32, device="cuda")
        # the batch's adapters are distinct slots spread over the pool
        slots = torch.randperm(self.nslots, generator=torch.Generator().manual_seed(slot_seed))[:self.nseg]
        self.slots = slots.to(torch.int32)
        self.seg_slot = self.slots.cuda()
        self.row_slot = torch.repeat_interleave(self.slots, torch.tensor(np.diff(self.bounds), dtype=torch.int64)).to(
            torch.int32).cuda()
        # The serving engine knows its step's segment lengths and passes them as a per-call
        # option (lsg_call_opts): a step with no segment of >= 128 rows (256 at rank 16, the
        # measured crossover, one prefill + decodes: 128 rows 5.7 us on the CUDA-core row mode
        # vs 10.3 on the tensor cores, 192 rows 9.9 vs 10.2, 256 rows 10.7 vs 10.4) skips the
        # tensor-core pass.
        crossover = 256 if r == 16 else 128
        self.tc_min_rows = self.rows + 1 if max(np.diff(self.bounds), default=0) < crossover else None
        if a.tc_min_rows > 0:
            self.tc_min_rows = a.tc_min_rows
        self.bytes = alg_bytes(self.rows, self.nseg, h, r)

    def launch(self, s, ys=None, xs=None):
        ys = self.ys if ys is None else ys
        xs = self.xs if xs is None else xs
        if self.rows == 0:
            return
        if self.a.kernel == "bgmv":
            self.lsg.bgmv(ys[s], xs[s], self.pool, self.row_slot, s)
        else:
            self.lsg.sgmv(ys[s], xs[s], self.pool, self.seg_starts, self.seg_slot, s, tc_min_rows=self.tc_min_rows)

    def step(self, ys=None, xs=None):
        for s in range(self.sites):
            self.launch(s, ys, xs)

    def info(self):
        return self.lsg.query_launch(self.pool, self.nseg, max(self.rows, 1),
                                     self.lsg.KERNEL_BGMV if self.a.kernel == "bgmv" else self.lsg.KERNEL_FUSED)

    def free(self):
        del self.pool, self.xs, self.ys


def graph_of(torch, fn, stream):
    with torch.cuda.stream(stream):
        fn()  # eager warm-up (sets function attributes before capture)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fn()
    return g


def device_time_ms(torch, dist, world, stream, fn, k):
    """k calls of fn on `stream`, bracketed by barrier + synchronize, CUDA events on the
    launching stream; max over ranks."""
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


def measure_graph(torch, stream, wl, replays=10, warm=3):
    """us per launch of wl's step graph (single GPU, CUDA events on the replay stream)."""
    g = graph_of(torch, wl.step, stream)
    with torch.cuda.stream(stream):
        for _ in range(warm):
            g.replay()
    ms = device_time_ms(torch, None, 1, stream, g.replay, replays)
    del g
    return ms * 1e3 / (replays * wl.sites)


def peak_gbs():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs")
        if p:
            return p, "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        pass
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def config_line(name, a, wl, us, peak):
    gbs = wl.bytes / (us * 1e-6) / 1e9
    return {"config": name, "workload": workload_name(a), "rows": wl.rows, "segments": wl.nseg,
            "us_per_launch": us, "alg_bytes": wl.bytes, "gbs": gbs, "frac": gbs / peak, "launch": wl.info()}


def run_configs(lsg, torch, a, dtype, stream, peak):
    out = []
    for name in EXTRA_CONFIGS:
        c = cfg_args(name, a)
        wl = Workload(lsg, torch, c, bounds_for(c), dtype)
        out.append(config_line(name, c, wl, measure_graph(torch, stream, wl), peak))
        wl.free()
        torch.cuda.empty_cache()
    return out


def run_sweep(lsg, torch, a, dtype, stream, peak):
    """Batch x popularity at the configured shape (the metric's 'vs batch across' part)."""
    out = []
    for pop in ("distinct", "uniform", "skewed", "identical"):
        for batch in (1, 2, 4, 8, 16, 32, 64):
            c = parse([])
            c.hidden, c.rank, c.dtype, c.pdl = a.hidden, a.rank, a.dtype, a.pdl
            c.popularity, c.batch = pop, batch
            wl = Workload(lsg, torch, c, segments(pop, batch), dtype)
            line = config_line(f"{pop}-{batch}", c, wl, measure_graph(torch, stream, wl), peak)
            out.append({k: line[k] for k in ("config", "rows", "segments", "us_per_launch", "gbs", "frac")})
            wl.free()
        torch.cuda.empty_cache()
    return out


# ---- a real decode step: backbone projections + the LoRA adds -------------------------
LLAMA7B_SITES = [("q", 4096, 4096), ("k", 4096, 4096), ("v", 4096, 4096), ("o", 4096, 4096),
                 ("gate", 4096, 11008), ("up", 4096, 11008), ("down", 11008, 4096)]


def run_decode_step(lsg, torch, a, dtype, stream, layers=LAYERS, batch=64, rank=16, replays=10):
    """One Llama-2-7B decode step at batch 64, Distinct adapters, on the real projection shapes
    (q/k/v/o 4096->4096, gate/up 4096->11008, down 11008->4096): per site the backbone GEMM
    y = x . W (cuBLAS through torch.matmul) then the LoRA add y += x . A . B (lsg_sgmv, PDL on).
    Three CUDA graphs of the whole step -- backbone only, backbone + one LoRA launch per site,
    backbone + grouped LoRA launches (q/k/v and gate/up each one lsg_sgmv_multi) -- give the
    in-model LoRA overhead per site (the paper's +2 ms/token on A100)."""
    gen = torch.Generator(device="cuda").manual_seed(77)
    bounds = segments("distinct", batch)
    nseg = len(bounds) - 1
    ss = torch.tensor(bounds, dtype=torch.int32, device="cuda")
    sl = torch.arange(nseg, dtype=torch.int32, device="cuda")
    pools, Ws, xs, ys = {}, [], [], []
    for name, hi, ho in LLAMA7B_SITES:
        pool = lsg.AdapterPool(nseg, layers, hi, ho, rank, dtype)
        pool.a.uniform_(-0.05, 0.05, generator=gen)
        pool.b.uniform_(-0.05, 0.05, generator=gen)
        pools[name] = pool
    views = {}
    for layer in range(layers):
        for name, hi, ho in LLAMA7B_SITES:
            Ws.append(torch.empty(hi, ho, dtype=dtype, device="cuda").uniform_(-0.02, 0.02, generator=gen))
            xs.append(torch.empty(batch, hi, dtype=dtype, device="cuda").uniform_(-1, 1, generator=gen))
            ys.append(torch.empty(batch, ho, dtype=dtype, device="cuda"))
            views[(layer, name)] = pools[name].layer_view(layer)
    nsites = layers * len(LLAMA7B_SITES)
    no_tc = batch + 1  # decode-only step: no tensor-core pass

    def backbone(i):
        torch.matmul(xs[i], Ws[i], out=ys[i])

    def step_base():
        for i in range(nsites):
            backbone(i)

    def step_lora():
        for i in range(nsites):
            layer, name = i // len(LLAMA7B_SITES), LLAMA7B_SITES[i % len(LLAMA7B_SITES)][0]
            backbone(i)
            lsg.sgmv(ys[i], xs[i], pools[name], ss, sl, layer, tc_min_rows=no_tc)

    def step_grouped():
        for layer in range(layers):
            b0 = layer * len(LLAMA7B_SITES)
            for i in range(b0, b0 + 7):
                backbone(i)
            for grp in ((0, 1, 2), (3,), (4, 5), (6,)):
                idx = [b0 + g for g in grp]
                if len(idx) == 1:
                    name = LLAMA7B_SITES[grp[0]][0]
                    lsg.sgmv(ys[idx[0]], xs[idx[0]], pools[name], ss, sl, layer, tc_min_rows=no_tc)
                else:
                    lsg.sgmv_multi([ys[i] for i in idx], [xs[i] for i in idx],
                                   [views[(layer, LLAMA7B_SITES[g][0])] for g in grp], ss, sl, 0, tc_min_rows=no_tc)

    out = {}
    for key, fn in (("backbone_only", step_base), ("backbone_lora", step_lora), ("backbone_lora_grouped", step_grouped)):
        g = graph_of(torch, fn, stream)
        with torch.cuda.stream(stream):
            for _ in range(3):
                g.replay()
        out[key + "_ms"] = device_time_ms(torch, None, 1, stream, g.replay, replays) / replays
        del g
    # shrink + expand algorithmic bytes per site (cost_model.cpp:13-19 for both halves, e = 2)
    lora_bytes = sum((batch * (hi + 2 * rank + ho) + nseg * rank * (hi + ho)) * 2 for _, hi, ho in LLAMA7B_SITES) * layers
    out.update({
        "model": "Llama-2-7B, 32 layers, batch 64 decode, Distinct adapters, rank 16",
        "lora_overhead_us_per_site": (out["backbone_lora_ms"] - out["backbone_only_ms"]) * 1e3 / nsites,
        "lora_overhead_us_per_site_grouped": (out["backbone_lora_grouped_ms"] - out["backbone_only_ms"]) * 1e3 / nsites,
        "lora_overhead_frac": out["backbone_lora_ms"] / out["backbone_only_ms"] - 1.0,
        "lora_alg_bytes_per_step": lora_bytes,
        "backbone_weight_bytes_per_step": sum(hi * ho * 2 for _, hi, ho in LLAMA7B_SITES) * layers,
    })
    del pools, Ws, xs, ys, views
    torch.cuda.empty_cache()
    return out


# ---- DRAM traffic of this build: one ncu pass over a probe run ------------------------
PROBE_CONFIGS = ["c2"] + EXTRA_CONFIGS
PROBE_CALLS = 3


def traffic_probe(lsg, torch, a, dtype):
    """Run under ncu: for each probe config, a marker kernel (torch's spin_kernel), then
    PROBE_CALLS calls on different layers; a final marker closes the last group.  Only
    our kernels and the markers are profiled (ncu replays each one with cold caches)."""
    for name in PROBE_CONFIGS:
        c = cfg_args(name, a)
        c.sites = PROBE_CALLS
        wl = Workload(lsg, torch, c, bounds_for(c), dtype, sites=PROBE_CALLS)
        torch.cuda.synchronize()
        torch.cuda._sleep(1000)
        wl.step()
        torch.cuda.synchronize()
        wl.free()
    torch.cuda._sleep(1000)
    torch.cuda.synchronize()


def measure_traffic(a, timeout_s=300):
    """DRAM bytes per launch of this build for every probe config (ncu counters; the probe's
    timings are never used).  Returns {config: {...}} or {"error": ...}."""
    ncu = "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return {"error": "ncu not found"}
    log = os.path.join(ROOT, "gpurun_out", f"traffic_{os.getpid()}.csv")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--csv", "--page", "raw",
           "-k", "regex:sgmv|spin_kernel|dense_lora|tc_", "--log-file", log,
           sys.executable, os.path.abspath(__file__), "--traffic-probe", "--dtype", a.dtype]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s)
    except subprocess.TimeoutExpired:
        return {"error": f"ncu pass timed out after {timeout_s} s"}
    if r.returncode != 0 or not os.path.exists(log):
        return {"error": f"ncu rc={r.returncode}: {(r.stderr or r.stdout)[-300:]}"}
    rows = [row for row in csv.reader(io.StringIO(open(log).read())) if row]
    hdr_i = next((i for i, row in enumerate(rows) if "Kernel Name" in row), None)
    if hdr_i is None:
        return {"error": "ncu csv without a header"}
    hdr = rows[hdr_i]
    kn, rd, wr = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    units = rows[hdr_i + 1] if hdr_i + 1 < len(rows) else []
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def val(row, i):
        return float(row[i].replace(",", "")) * scale.get(units[i] if i < len(units) else "byte", 1)

    groups, cur = [], None
    for row in rows[hdr_i + 2:]:
        if len(row) <= max(kn, rd, wr):
            continue
        if "spin_kernel" in row[kn]:
            if cur is not None:
                groups.append(cur)
            cur = []
        elif cur is not None:
            cur.append((row[kn].split("(")[0].split("<")[0].strip(), val(row, rd), val(row, wr)))
    out = {}
    for name, kernels in zip(PROBE_CONFIGS, groups):
        per_call = sum(k[1] + k[2] for k in kernels) / PROBE_CALLS
        by_kernel = {}
        for kname, b_r, b_w in kernels:
            by_kernel.setdefault(kname, [0.0, 0])
            by_kernel[kname][0] += b_r + b_w
            by_kernel[kname][1] += 1
        dominant = max(by_kernel.items(), key=lambda kv: kv[1][0]) if by_kernel else ("", [0.0, 1])
        out[name] = {"dram_bytes_per_call": per_call, "kernels_per_call": len(kernels) / PROBE_CALLS,
                     "dominant_kernel": dominant[0],
                     "dominant_bytes_per_launch": dominant[1][0] / max(1, dominant[1][1])}
    try:
        os.remove(log)
    except OSError:
        pass
    return out


def library_hash():
    p = os.path.join(ROOT, "paper_2310_18547_b200", "lib", "libsgmv_b200.so")
    try:
        return hashlib.sha256(open(p, "rb").read()).hexdigest()[:16]
    except OSError:
        return None


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    a = parse()
    if a.impl == "reference":
        run_reference_arm(a)
        return
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run (rendezvous on 127.0.0.1)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))

    import torch
    import torch.distributed as dist

    import paper_2310_18547_b200 as lsg

    dtype = torch.float16 if a.dtype == "fp16" else torch.bfloat16
    if a.traffic_probe:
        lsg.set_option(lsg.LSG_OPT_PDL, 0)
        traffic_probe(lsg, torch, a, dtype)
        return

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        sys.stderr.write(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
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
    lsg.set_option(lsg.LSG_OPT_PDL, a.pdl)
    lsg.set_option(lsg.LSG_OPT_FORCE_CLUSTER, a.cluster)
    lsg.set_option(lsg.LSG_OPT_FORCE_TILE_ROWS, a.tile_rows)
    lsg.set_option(lsg.LSG_OPT_NO_L2_STAGING, 1 if a.no_l2_staging else -1 if a.l2_staging else 0)
    lsg.set_option(lsg.LSG_OPT_NO_TENSOR_CORES, int(a.no_tc))
    lsg.set_option(lsg._lib.LSG_OPT_TC_SPLIT, int(a.tc_split))
    lsg.set_option(lsg._lib.LSG_OPT_TC_LEGACY, a.tc_gen)
    lsg.set_option(lsg._lib.LSG_OPT_MMA_MIN_ROWS, a.mma_min_rows)
    lsg.set_option(lsg._lib.LSG_OPT_MMA_FUSED, a.mma_fused)
    lsg.set_option(lsg._lib.LSG_OPT_NO_ROW_MODE, int(a.no_row_mode))
    h, r, sites = a.hidden, a.rank, a.sites
    # Request partitioning: the partitioner (lsg_partition_segments) hands every rank whole
    # segments (or row ranges of dominant ones) and each rank runs its share on its own
    # replica of the adapter pool -- no collective on the data path.
    from paper_2310_18547_b200.partition import rank_batches
    gbounds = global_bounds(a, world)
    mine = rank_batches(np.array(gbounds, dtype=np.int32), h, h, r, world)[rank]
    wl = Workload(lsg, torch, a, [int(v) for v in mine.seg_starts], dtype, seed=1000 + rank, slot_seed=7 + rank)
    info = wl.info()
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()
    if a.profile:
        with torch.cuda.stream(stream):
            for _ in range(max(1, a.warmup)):
                wl.step()
        torch.cuda.synchronize()
        return
    graph = graph_of(torch, wl.step, stream)
    if a.profile_graph:
        with torch.cuda.stream(stream):
            graph.replay()
            torch.cuda.nvtx.range_push("lsg_graph")  # ncu --nvtx --nvtx-include lsg_graph/
            graph.replay()
            torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        return
    with torch.cuda.stream(stream):
        for _ in range(max(3, a.warmup)):
            graph.replay()
    torch.cuda.synchronize()

    # ---- the timed region: K step-graph replays, max over ranks ----------------------------
    with ClockSampler(dev) as clk:
        ms = device_time_ms(torch, dist, world, stream, graph.replay, a.steps)
    ms_step = ms / a.steps
    us_launch = ms_step * 1e3 / sites  # max-over-ranks device time per launch (per site)
    # whole job: weak = time per 64-row site-equivalent (all ranks' rows), strong = per site
    value = us_launch / world if a.scaling == "weak" else us_launch
    peak, peak_src = peak_gbs()
    bytes_per_launch = wl.bytes  # this rank's launch (rank 0 reports)
    achieved = bytes_per_launch / (us_launch * 1e-6) / 1e9
    extra = {"us_per_launch_max_rank": us_launch}

    single = world == 1 and not a.no_extras
    if single:
        # isolated single-launch latency (no PDL overlap), L2 flushed between launches
        flush = torch.empty(1024 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > L2
        lat = []
        for i in range(20):
            with torch.cuda.stream(stream):
                flush.zero_()  # same stream: evicts L2 and covers the host launch latency
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                wl.launch(i)
                e1.record(stream)
            torch.cuda.synchronize()
            lat.append(e0.elapsed_time(e1) * 1e3)
        extra["isolated_launch_us_median"] = statistics.median(lat)
        del flush
        lsg.set_option(lsg.LSG_OPT_PDL, 0)
        g_nopdl = graph_of(torch, wl.step, stream)
        kn = max(3, a.steps // 2)
        extra["us_per_launch_no_pdl"] = device_time_ms(torch, dist, 1, stream, g_nopdl.replay, kn) * 1e3 / (kn * sites)
        lsg.set_option(lsg.LSG_OPT_PDL, a.pdl)
        del g_nopdl
        # Grouped launches (lsg_sgmv_multi): per layer q/k/v in one launch, o, gate/up in
        # one launch, down -- 4 launches for the 7 sites, same bytes and results.
        if a.kernel == "sgmv" and sites % SITES_PER_LAYER == 0:
            groups = []
            for l in range(sites // SITES_PER_LAYER):
                b0 = l * SITES_PER_LAYER
                groups += [[b0, b0 + 1, b0 + 2], [b0 + 3], [b0 + 4, b0 + 5], [b0 + 6]]
            views = {s_: wl.pool.layer_view(s_) for g in groups if len(g) > 1 for s_ in g}  # before capture

            def step_grouped():
                for g in groups:
                    if len(g) == 1:
                        wl.launch(g[0])
                    else:  # the sites' weights are layers g[i] of the one bench pool (same slots)
                        lsg.sgmv_multi([wl.ys[s_] for s_ in g], [wl.xs[s_] for s_ in g], [views[s_] for s_ in g],
                                       wl.seg_starts, wl.seg_slot, 0, tc_min_rows=wl.tc_min_rows)

            g_grp = graph_of(torch, step_grouped, stream)
            with torch.cuda.stream(stream):
                g_grp.replay()
            kg = max(3, a.steps // 2)
            extra["grouped_us_per_site"] = device_time_ms(torch, dist, 1, stream, g_grp.replay, kg) * 1e3 / (kg * sites)
            extra["grouped_launches_per_layer"] = 4
            del g_grp

    # e2e through the public API: every step copies that step's activations in from
    # pinned host memory (one H2D of all sites' x) and its outputs back (one D2H of
    # all sites' y).  Steps are pipelined over two device buffer sets and three
    # streams (H2D / compute / D2H), the way a serving loop overlaps PCIe with the
    # kernels; timed with CUDA events from the first H2D to the last D2H, max over ranks.
    e2e = None
    if not a.no_e2e:
        hx = torch.empty_like(wl.xs, device="cpu").pin_memory()
        hx.copy_(wl.xs.cpu())
        hy = torch.empty_like(wl.ys, device="cpu").pin_memory()
        bufs = [(wl.xs, wl.ys), (torch.empty_like(wl.xs), torch.zeros_like(wl.ys))]
        graphs = [graph, graph_of(torch, lambda: wl.step(bufs[1][1], bufs[1][0]), stream)]
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
        us_e2e = ms_e2e * 1e3 / (ke * sites)
        e2e = {"value": us_e2e / world if a.scaling == "weak" else us_e2e, "unit": "us/layer",
               "h2d_bytes_per_step": int(hx.numel() * hx.element_size()),
               "d2h_bytes_per_step": int(hy.numel() * hy.element_size()),
               "how": "per step: one pinned H2D of all x, the step graph, one D2H of all y; "
                      "pipelined over 2 buffer sets (PCIe-bound)"}
        del bufs, graphs, hx, hy

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    del graph
    wl.free()
    torch.cuda.empty_cache()
    if single:
        extra["configs"] = run_configs(lsg, torch, a, dtype, stream, peak)
        extra["sweep"] = run_sweep(lsg, torch, a, dtype, stream, peak)
        extra["decode_step"] = run_decode_step(lsg, torch, a, dtype, stream)
    traffic, traffic_src = None, None
    if single and not a.no_traffic:
        t = measure_traffic(a)
        extra["traffic_pass"] = {"library_sha16": library_hash(), **({"error": t["error"]} if "error" in t else {})}
        if "error" not in t:
            head = t.get("c2")
            if head and a.preset in ("", "c2") and a.kernel == "sgmv" and not a.segments:
                traffic = head["dominant_bytes_per_launch"]
                traffic_src = f"ncu dram__bytes_read.sum + dram__bytes_write.sum of {head['dominant_kernel']}, " \
                              f"mean of {PROBE_CALLS} cold launches, this build"
            for c in extra.get("configs", []):
                if c["config"] in t:
                    c["traffic"] = t[c["config"]]["dram_bytes_per_call"]
                    c["traffic_dominant_kernel"] = t[c["config"]]["dominant_kernel"]

    line = {
        "metric": METRIC,
        "value": value, "unit": "us/layer", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms_step, "higher_is_better": False, "scaling": a.scaling, "vs_baseline": None,
        "dtype": a.dtype + " (fp32 accumulate)", "data": "synthetic (U[-1,1) adapters/activations, random init)",
        "config": {"workload": workload_name(a), "model": "Llama-2-7B LoRA sites (h x h)", "hidden": h, "rank": r,
                   "batch_per_gpu": wl.rows, "global_batch": len(gbounds) and gbounds[-1],
                   "segments": wl.nseg, "global_segments": len(gbounds) - 1, "rank0_rows": wl.rows,
                   "popularity": a.popularity,
                   "step": f"{sites} fused SGMV launches (7 sites x 32 layers), CUDA graph",
                   "parallelism": f"request-partitioned x{world} (no collective), {a.scaling} scaling",
                   "kernel": a.kernel, "pool_slots": wl.nslots, "preset": a.preset or None,
                   "l2": "inputs larger than L2: weights rotate over a "
                         f"{wl.nslots * sites * 2 * h * r * 2 / 2**30:.2f} GiB pool, x/y over "
                         f"{2 * sites * max(wl.rows, 1) * h * 2 / 2**20:.0f} MiB per step",
                   "pdl": bool(a.pdl), "launch": info},
        "hbm_gbs": achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                     "alg_bytes_per_launch": bytes_per_launch, "flop_per_launch": alg_flop(wl.rows, h, r)},
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


if __name__ == "__main__":
    main()
