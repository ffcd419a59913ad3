"""Generate the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Run here (where /root/reference exists):

    make -C oracle all ref && python tests/golden/make_golden.py

Every number below is produced by the reference's own sources compiled in place
(oracle/_ref/libref.so, built by oracle/Makefile from
/root/reference/proj/core/src/*.cpp through oracle/ref_shim.cpp).  The fixtures
pin the C restatement in oracle/ (tests/test_oracle.py) on machines where the
reference is absent, e.g. the GPU box.

Outputs (all small):
  rng.json           mt19937_64 / Rng draws, derive_seed, model_count_for, assign_models
  verify_trials.npz  the first 8 verify_sgmv(seed 42) batches and their lora_addon
  verify_digest.json sha256 over 200 verify_sgmv(seed 42) trials (inputs + y bits),
                     plus the reference's own verify_sgmv(8, 42, inject) report
  kat.json           the hand-checked fixtures of test_sgmv.cpp:83-122 run through
                     the reference (lora_addon / dense_projection / oracles)
  cost_model.json    formula anchors and the roofline.csv text (experiments.cpp:141-174)
  plan_batch.json    plan_batch segment layouts (simulator.cpp:239-311)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Reference  # noqa: E402

POPS = [0, 1, 2, 3]


def trial_digest(h, t, y):
    h.update(np.array([t["h_in"], t["h_out"], t["rank"], t["rows"], t["nseg"]], dtype=np.uint64).tobytes())
    for k in ("bounds", "ids", "x", "A", "B"):
        h.update(np.ascontiguousarray(t[k]).tobytes())
    h.update(np.ascontiguousarray(y).tobytes())


def main():
    ref = Reference()
    out = {}

    # --- RNG --------------------------------------------------------------
    rng = {}
    for seed in (0, 1, 7, 42, 5489, 20240805):
        g = ref.rng(seed)
        rng[f"next_{seed}"] = [str(g.next()) for _ in range(32)]
        rng[f"uniform01_{seed}"] = [g.uniform01().hex() for _ in range(16)]
        rng[f"uniform_index_{seed}"] = [int(g.uniform_index(n)) for n in (1, 2, 3, 5, 7, 64, 1000, 2**63 + 5)]
        rng[f"uniform_int_{seed}"] = [g.uniform_int(lo, hi) for lo, hi in ((-3, 3), (1, 8), (1, 64), (0, 0))]
        cum = np.cumsum([1.0, 1 / 1.5, 1 / 2.25, 1 / 3.375])
        rng[f"discrete_{seed}"] = [int(g.discrete(cum, float(cum[-1]))) for _ in range(16)]
        rng[f"shuffle_{seed}"] = g.shuffle(np.arange(20, dtype=np.int64)).tolist()
    g = ref.rng(5489)
    for _ in range(9999):
        g.next()
    rng["mt19937_64_10000th"] = str(g.next())
    rng["derive_seed"] = {f"{s},{k}": str(ref.derive_seed(s, k)) for s in (0, 42, 2**64 - 1) for k in (0, 1, 2, 3, 17)}
    rng["model_count_for"] = {f"{n},{p}": ref.model_count_for(n, p) for n in (0, 1, 2, 63, 64, 65, 100, 101, 1000) for p in POPS}
    am = {}
    for n in (1, 2, 7, 8, 50, 64, 100, 1000):
        for p in POPS:
            for seed in (3, 42):
                am[f"{n},{p},{seed}"] = ref.assign_models(n, p, 1.5, seed).tolist()
    rng["assign_models"] = am
    with open(os.path.join(HERE, "rng.json"), "w") as f:
        json.dump(rng, f, indent=0)

    # --- verify_sgmv trials ------------------------------------------------------
    g = ref.rng(ref.derive_seed(42, 17))
    h = hashlib.sha256()
    arrays = {}
    for t in range(200):
        tr = g.verify_next_trial(t)
        y = ref.lora_addon(tr["x"], tr["bounds"], tr["A"], tr["B"])
        trial_digest(h, tr, y)
        if t < 8:
            for k in ("bounds", "ids", "x", "A", "B"):
                arrays[f"t{t}_{k}"] = tr[k]
            arrays[f"t{t}_shape"] = np.array([tr["h_in"], tr["h_out"], tr["rank"], tr["rows"], tr["nseg"]])
            arrays[f"t{t}_y"] = y
    np.savez_compressed(os.path.join(HERE, "verify_trials.npz"), **arrays)
    rep = ref.verify_sgmv(8, 42, inject=True)
    clean = ref.verify_sgmv(200, 42)
    with open(os.path.join(HERE, "verify_digest.json"), "w") as f:
        json.dump({"trials": 200, "seed": 42, "sha256": h.hexdigest(),
                   "reference_verify_8_42_inject": rep, "reference_verify_200_42": clean}, f, indent=1)

    # --- KATs (test_sgmv.cpp:83-122) ----------------------------------------------
    kat = {}
    x = np.array([[1, 2], [3, 4], [5, 6]], float)
    A = np.array([[[1, 0], [0, 1]], [[2, 0], [1, 1]]], float)
    B = np.array([[[1, 1], [2, 0]], [[1, 3], [0, 1]]], float)
    bounds = [0, 2, 3]
    kat["two_segment"] = {"x": x.tolist(), "A": A.tolist(), "B": B.tolist(), "bounds": bounds,
                          "lora_addon": ref.lora_addon(x, bounds, A, B).tolist(),
                          "loop": ref.lora_loop_oracle(x, bounds, A, B).tolist(),
                          "gather": ref.gather_bmm_oracle(x, bounds, A, B).tolist(),
                          "dense_w_identity": ref.dense_projection(x, bounds, A, B, np.eye(2)).tolist(),
                          "shrink": ref.sgmv_shrink(x, bounds, A, B).tolist()}
    x1 = np.array([[1, 2]], float)
    A1 = np.array([[[1], [1]]], float)
    B1 = np.array([[[1, 1]]], float)
    kat["rank1"] = {"x": x1.tolist(), "A": A1.tolist(), "B": B1.tolist(), "bounds": [0, 1],
                    "lora_addon": ref.lora_addon(x1, [0, 1], A1, B1).tolist()}
    errs = {}
    try:
        ref.lora_addon(np.zeros((3, 2)), [0, 2, 3], np.zeros((2, 2, 1)), np.zeros((2, 1, 2)))
        errs["ok"] = True
    except ValueError as e:
        errs["unexpected"] = str(e)
    kat["errors"] = errs
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat, f, indent=1)

    # --- cost model -------------------------------------------------------------
    cm = {"flop_64_64_16_4096": ref.sgmv_flop(64, 64, 16, 4096),
          "io_64_64_16_4096": ref.sgmv_io_bytes(64, 64, 16, 4096),
          "io_1_1_16_4096": ref.sgmv_io_bytes(1, 1, 16, 4096),
          "io_1_64_16_4096": ref.sgmv_io_bytes(1, 64, 16, 4096),
          "gather_extra_64_64_16_4096": ref.gather_bmm_extra_elements(64, 64, 16, 4096),
          "intensity": {f"{n},{b}": ref.arithmetic_intensity(n, b, 16, 4096).hex()
                        for b in range(1, 65) for n in (1, b)},
          "latency_default": {f"{n},{b}": ref.sgmv_latency(n, b, 16, 4096).hex() for b in (1, 8, 64) for n in (1, b)},
          "roofline_csv": ref.roofline_csv(64)}
    with open(os.path.join(HERE, "cost_model.json"), "w") as f:
        json.dump(cm, f, indent=0)

    # --- plan_batch ---------------------------------------------------------------
    plans = [{"lora": [5, 9, 5, 9], "done": [1, 1, 1, 0], "prompt": [8, 8, 8, 6]}]
    r = np.random.default_rng(7)
    for n in (1, 3, 8, 31, 64):
        for _ in range(4):
            plans.append({"lora": r.integers(0, max(2, n // 3), n).tolist(),
                          "done": (r.random(n) < 0.85).astype(int).tolist(),
                          "prompt": r.integers(1, 2048, n).tolist()})
    for p in plans:
        p["plan"] = ref.plan_segments(p["lora"], p["done"], p["prompt"])
    with open(os.path.join(HERE, "plan_batch.json"), "w") as f:
        json.dump(plans, f, indent=0)
    # --- the symbols core/src/sgmv.cpp defines (what the drop-in must replace, exactly) ---
    with open(os.path.join(HERE, "sgmv_cpp_symbols.txt"), "w") as f:
        f.write("\n".join(reference_sgmv_symbols()) + "\n")
    print("golden fixtures written to", HERE)


def reference_sgmv_symbols():
    """Demangled text symbols of the reference's core/src/sgmv.cpp, compiled here."""
    import subprocess
    import tempfile
    ref = "/root/reference/proj"
    with tempfile.TemporaryDirectory() as d:
        obj = os.path.join(d, "sgmv.o")
        subprocess.run(["g++", "-std=c++20", "-O2", "-c", f"-I{ref}/core/include", f"{ref}/core/src/sgmv.cpp",
                        "-o", obj], check=True)
        out = subprocess.run(["nm", "--defined-only", "-C", obj], capture_output=True, text=True, check=True).stdout
    return sorted({line.split(" T ", 1)[1] for line in out.splitlines() if " T " in line})


if __name__ == "__main__":
    main()
