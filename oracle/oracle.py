"""ctypes bindings for the CPU ORACLE (test infrastructure only).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this module.  It loads

* ``oracle/liboracle.so`` -- the C restatement of the reference SGMV path
  (oracle/sgmv_oracle.c, each function citing the reference file:line), and
* ``oracle/_ref/libref.so`` -- the reference's own sources compiled in place by
  ``make -C oracle ref`` (present wherever it was built; it travels to the GPU
  box with the snapshot but is never committed).

Arrays are numpy float64 / int64 / uint64 (size_t) in row-major layout, weights
packed per segment: A ``[nseg, h_in, rank]``, B ``[nseg, rank, h_out]``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref.so")

DISTINCT, UNIFORM, SKEWED, IDENTICAL = 0, 1, 2, 3
POPULARITIES = {"distinct": DISTINCT, "uniform": UNIFORM, "skewed": SKEWED, "identical": IDENTICAL}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_sp = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_sz = C.c_size_t


def build(ref: bool = True) -> None:
    """Compile liboracle.so (and, when /root/reference exists, _ref/libref.so and the
    reference's acceptance gate linked against the B200 drop-in, _ref/acceptance_b200)."""
    targets = ["all"]
    if ref and os.path.isdir("/root/reference/proj"):
        targets += ["ref", "integration"]
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle` first")
    return C.CDLL(path)


class _Lib:
    """Common marshalling for the oracle (``orc_``) and reference (``ref_``) libraries."""

    def __init__(self, lib: C.CDLL, prefix: str):
        self.lib = lib
        self.p = prefix

    def fn(self, name):
        return getattr(self.lib, self.p + name)


class Oracle(_Lib):
    """The C restatement, oracle/sgmv_oracle.c."""

    def __init__(self, path: str = ORACLE_SO):
        super().__init__(_load(path), "orc_")
        L = self.lib
        L.orc_rng_size.restype = _sz
        L.orc_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_rng_next.argtypes = [C.c_void_p]
        L.orc_rng_next.restype = C.c_uint64
        L.orc_rng_uniform01.argtypes = [C.c_void_p]
        L.orc_rng_uniform01.restype = C.c_double
        L.orc_rng_uniform_index.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        L.orc_rng_uniform_int.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.orc_rng_discrete.argtypes = [C.c_void_p, _dp, _sz, C.c_double]
        L.orc_rng_discrete.restype = _sz
        L.orc_rng_fill_pm1.argtypes = [C.c_void_p, _dp, _sz]
        L.orc_rng_shuffle_i64.argtypes = [C.c_void_p, _ip, _sz]
        L.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_model_count_for.argtypes = [C.c_int, C.c_int]
        L.orc_assign_models.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64, _ip]
        seg = [_dp, _sz, _sp, _sz, _dp, _dp, _sz, _sz, _dp]
        for n in ("lora_addon", "lora_loop_oracle", "gather_bmm_oracle"):
            getattr(L, "orc_" + n).argtypes = seg
        L.orc_dense_projection.argtypes = seg[:-1] + [_dp, _dp]
        L.orc_sgmv_shrink.argtypes = [_dp, _sz, _sp, _sz, _dp, _sz, _dp]
        L.orc_sgmv_expand.argtypes = [_dp, _sz, _sp, _sz, _dp, _sz, _dp]
        L.orc_max_abs_diff.argtypes = [_dp, _dp, _sz]
        L.orc_max_abs_diff.restype = C.c_double
        P = C.POINTER(_sz)
        L.orc_verify_next_trial.argtypes = [C.c_void_p, C.c_int, P, P, P, P, P, _sp, _ip, _dp, _dp, _dp]
        i64 = C.c_int64
        for n, args in (("sgmv_flop", [i64] * 4), ("sgmv_io_bytes", [i64] * 4 + [C.c_int]),
                        ("arithmetic_intensity", [i64] * 4 + [C.c_int]),
                        ("sgmv_latency", [i64] * 4 + [C.c_double] * 3 + [C.c_int]),
                        ("gather_bmm_extra_elements", [i64] * 4),
                        ("adapter_pair_io_bytes", [C.c_double] * 4 + [C.c_int]),
                        ("adapter_pair_flop", [C.c_double] * 3)):
            f = getattr(L, "orc_" + n)
            f.argtypes = args
            f.restype = C.c_double
        L.orc_plan_segments.argtypes = [_sz, _ip, _u8p, _i32p, C.POINTER(i64), _ip, P, _sp, _ip, P]

    # -- rng -------------------------------------------------------------------
    def rng(self, seed: int) -> "OracleRng":
        return OracleRng(self, seed)

    def derive_seed(self, seed: int, stream: int) -> int:
        return self.lib.orc_derive_seed(seed, stream)

    def model_count_for(self, n: int, pop: int) -> int:
        return self.lib.orc_model_count_for(n, pop)

    def assign_models(self, n: int, pop: int, alpha: float, seed: int) -> np.ndarray:
        out = np.zeros(max(n, 1), dtype=np.int64)
        if self.lib.orc_assign_models(n, pop, alpha, seed, out):
            raise ValueError("assign_models: invalid arguments")
        return out[:n]

    # -- SGMV ------------------------------------------------------------------
    def _seg_call(self, name, x, bounds, A, B, *extra):
        x = np.ascontiguousarray(x, dtype=np.float64)
        bounds = np.ascontiguousarray(bounds, dtype=np.uint64)
        A = np.ascontiguousarray(A, dtype=np.float64)
        B = np.ascontiguousarray(B, dtype=np.float64)
        nseg = len(bounds) - 1
        rows = int(bounds[-1]) if nseg else 0
        h_in = x.shape[1]
        rank, h_out = B.shape[1], B.shape[2]
        y = np.zeros((rows, h_out), dtype=np.float64)
        st = self.fn(name)(x, h_in, bounds, nseg, A.reshape(-1) if A.size else np.zeros(1),
                           B.reshape(-1) if B.size else np.zeros(1), rank, h_out,
                           *[np.ascontiguousarray(e, dtype=np.float64) for e in extra], y)
        if st:
            raise ValueError(f"{name}: invalid arguments")
        return y

    def lora_addon(self, x, bounds, A, B):
        return self._seg_call("lora_addon", x, bounds, A, B)

    def lora_loop_oracle(self, x, bounds, A, B):
        return self._seg_call("lora_loop_oracle", x, bounds, A, B)

    def gather_bmm_oracle(self, x, bounds, A, B):
        return self._seg_call("gather_bmm_oracle", x, bounds, A, B)

    def dense_projection(self, x, bounds, A, B, w):
        return self._seg_call("dense_projection", x, bounds, A, B, w)

    def sgmv_shrink(self, x, bounds, A):
        x = np.ascontiguousarray(x, dtype=np.float64)
        bounds = np.ascontiguousarray(bounds, dtype=np.uint64)
        A = np.ascontiguousarray(A, dtype=np.float64)
        rank = A.shape[2]
        v = np.zeros((int(bounds[-1]), rank))
        if self.lib.orc_sgmv_shrink(x, x.shape[1], bounds, len(bounds) - 1, A.reshape(-1), rank, v):
            raise ValueError("sgmv_shrink: invalid arguments")
        return v

    def sgmv_expand(self, v, bounds, B):
        v = np.ascontiguousarray(v, dtype=np.float64)
        bounds = np.ascontiguousarray(bounds, dtype=np.uint64)
        B = np.ascontiguousarray(B, dtype=np.float64)
        h_out = B.shape[2]
        y = np.zeros((int(bounds[-1]), h_out))
        if self.lib.orc_sgmv_expand(v, v.shape[1], bounds, len(bounds) - 1, B.reshape(-1), h_out, y):
            raise ValueError("sgmv_expand: invalid arguments")
        return y

    def max_abs_diff(self, a, b) -> float:
        a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
        b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
        assert a.size == b.size
        return self.lib.orc_max_abs_diff(a, b, a.size)

    # -- cost model -------------------------------------------------------------
    def sgmv_flop(self, n, rows, h_in, h_out):
        return self.lib.orc_sgmv_flop(n, rows, h_in, h_out)

    def sgmv_io_bytes(self, n, rows, h_in, h_out, e=2):
        return self.lib.orc_sgmv_io_bytes(n, rows, h_in, h_out, e)

    def arithmetic_intensity(self, n, rows, h_in, h_out, e=2):
        return self.lib.orc_arithmetic_intensity(n, rows, h_in, h_out, e)

    def sgmv_latency(self, n, rows, h_in, h_out, peak=312e12, bw=2.0e12, floor_s=38e-6, e=2):
        return self.lib.orc_sgmv_latency(n, rows, h_in, h_out, peak, bw, floor_s, e)

    def gather_bmm_extra_elements(self, n, rows, h_in, h_out):
        return self.lib.orc_gather_bmm_extra_elements(n, rows, h_in, h_out)

    def adapter_pair_io_bytes(self, rows, models, h, r, e=2):
        return self.lib.orc_adapter_pair_io_bytes(rows, models, h, r, e)

    def adapter_pair_flop(self, rows, h, r):
        return self.lib.orc_adapter_pair_flop(rows, h, r)

    # -- plan_batch -----------------------------------------------------------
    def plan_segments(self, lora, prefill_done, prompt):
        return _plan(self.lib.orc_plan_segments, lora, prefill_done, prompt)


def _plan(fn, lora, prefill_done, prompt):
    lora = np.ascontiguousarray(lora, dtype=np.int64)
    done = np.ascontiguousarray(prefill_done, dtype=np.uint8)
    prompt = np.ascontiguousarray(prompt, dtype=np.int32)
    n = len(lora)
    prefill = C.c_int64(-1)
    decodes = np.zeros(max(n, 1), dtype=np.int64)
    nd = _sz(0)
    bounds = np.zeros(n + 2, dtype=np.uint64)
    loras = np.zeros(max(n, 1), dtype=np.int64)
    ns = _sz(0)
    if fn(n, lora, done, prompt, C.byref(prefill), decodes, C.byref(nd), bounds, loras, C.byref(ns)):
        raise ValueError("plan_batch failed")
    return {"prefill": prefill.value, "decodes": decodes[: nd.value].tolist(),
            "bounds": bounds[: ns.value + 1].tolist(), "loras": loras[: ns.value].tolist()}


class OracleRng:
    """lorasim::Rng restated (workload.hpp:13-42)."""

    def __init__(self, orc: Oracle, seed: int):
        self.o = orc
        self.buf = C.create_string_buffer(orc.lib.orc_rng_size())
        orc.lib.orc_rng_seed(self.buf, seed)

    def next(self) -> int:
        return self.o.lib.orc_rng_next(self.buf)

    def uniform01(self) -> float:
        return self.o.lib.orc_rng_uniform01(self.buf)

    def uniform_index(self, n: int) -> int:
        out = C.c_uint64()
        if self.o.lib.orc_rng_uniform_index(self.buf, n, C.byref(out)):
            raise ValueError("Rng::uniform_index: n must be > 0")
        return out.value

    def uniform_int(self, lo: int, hi: int) -> int:
        out = C.c_int()
        if self.o.lib.orc_rng_uniform_int(self.buf, lo, hi, C.byref(out)):
            raise ValueError("Rng::uniform_int: empty range")
        return out.value

    def discrete(self, cumulative, total: float) -> int:
        c = np.ascontiguousarray(cumulative, dtype=np.float64)
        return self.o.lib.orc_rng_discrete(self.buf, c, c.size, total)

    def fill_pm1(self, n: int) -> np.ndarray:
        out = np.empty(max(n, 1), dtype=np.float64)
        self.o.lib.orc_rng_fill_pm1(self.buf, out, n)
        return out[:n]

    def shuffle(self, v) -> np.ndarray:
        a = np.ascontiguousarray(v, dtype=np.int64).copy()
        self.o.lib.orc_rng_shuffle_i64(self.buf, a, a.size)
        return a

    def verify_next_trial(self, trial: int) -> dict:
        return _verify_trial(self.o.lib.orc_verify_next_trial, self.buf, trial)


def _verify_trial(fn, handle, trial):
    h_in, h_out, rank, rows, nseg = (_sz() for _ in range(5))
    bounds = np.zeros(65, dtype=np.uint64)
    ids = np.zeros(64, dtype=np.int64)
    x = np.zeros(64 * 128)
    A = np.zeros(8 * 128 * 64)
    B = np.zeros(8 * 64 * 128)
    st = fn(handle, trial, C.byref(h_in), C.byref(h_out), C.byref(rank), C.byref(rows),
            C.byref(nseg), bounds, ids, x, A, B)
    if st:
        raise RuntimeError("verify trial generation failed")
    hi, ho, r, m, n = h_in.value, h_out.value, rank.value, rows.value, nseg.value
    return {"h_in": hi, "h_out": ho, "rank": r, "rows": m, "nseg": n,
            "bounds": bounds[: n + 1].copy(), "ids": ids[:n].copy(),
            "x": x[: m * hi].reshape(m, hi).copy(),
            "A": A[: n * hi * r].reshape(n, hi, r).copy(),
            "B": B[: n * r * ho].reshape(n, r, ho).copy()}


class Reference(_Lib):
    """The reference's own code (oracle/_ref/libref.so via oracle/ref_shim.cpp)."""

    def __init__(self, path: str = REF_SO):
        super().__init__(_load(path), "ref_")
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_new.argtypes = [C.c_uint64]
        L.ref_rng_new.restype = C.c_void_p
        L.ref_rng_free.argtypes = [C.c_void_p]
        L.ref_rng_next.argtypes = [C.c_void_p]
        L.ref_rng_next.restype = C.c_uint64
        L.ref_rng_uniform01.argtypes = [C.c_void_p]
        L.ref_rng_uniform01.restype = C.c_double
        L.ref_rng_uniform_index.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_rng_uniform_index.restype = C.c_uint64
        L.ref_rng_uniform_int.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_rng_discrete.argtypes = [C.c_void_p, _dp, _sz, C.c_double]
        L.ref_rng_discrete.restype = _sz
        L.ref_rng_shuffle_i64.argtypes = [C.c_void_p, _ip, _sz]
        L.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_model_count_for.argtypes = [C.c_int, C.c_int]
        L.ref_assign_models.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64, _ip]
        seg = [_dp, _sz, _sp, _sz, _dp, _dp, _sz, _sz, _dp]
        for n in ("lora_addon", "lora_loop_oracle", "gather_bmm_oracle", "sgmv_shrink"):
            getattr(L, "ref_" + n).argtypes = seg
        L.ref_dense_projection.argtypes = seg[:-1] + [_dp, _dp]
        L.ref_sgmv_expand.argtypes = [_dp, _sz, _sp, _sz, _dp, _dp, _sz, _sz, _sz, _dp]
        P = C.POINTER(_sz)
        L.ref_verify_next_trial.argtypes = [C.c_void_p, C.c_int, P, P, P, P, P, _sp, _ip, _dp, _dp, _dp]
        L.ref_verify_sgmv.argtypes = [C.c_int, C.c_uint64, C.c_int, C.POINTER(C.c_int),
                                      C.POINTER(C.c_double), C.POINTER(C.c_double), _sp]
        i64 = C.c_int64
        for n, args in (("sgmv_flop", [i64] * 4), ("sgmv_io_bytes", [i64] * 4 + [C.c_int]),
                        ("arithmetic_intensity", [i64] * 4 + [C.c_int]),
                        ("sgmv_latency", [i64] * 4 + [C.c_double] * 3 + [C.c_int]),
                        ("gather_bmm_extra_elements", [i64] * 4)):
            f = getattr(L, "ref_" + n)
            f.argtypes = args
            f.restype = C.c_double
        L.ref_roofline_csv.argtypes = [C.c_int, C.c_char_p, _sz]
        L.ref_roofline_csv.restype = _sz
        L.ref_plan_batch.argtypes = [_sz, _ip, _u8p, _i32p, C.POINTER(i64), _ip, P, _sp, _ip, P]
        L.ref_batch_new.argtypes = [_dp, _sz, _sp, _sz, _dp, _dp, _sz, _sz]
        L.ref_batch_new.restype = C.c_void_p
        L.ref_batch_free.argtypes = [C.c_void_p]
        L.ref_batch_bench.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_int, C.POINTER(C.c_int)]
        L.ref_batch_bench.restype = C.c_double

    def bench_batch(self, x, bounds, A, B, op="lora_addon", budget_s=1.0, max_iters=100000):
        """Seconds per call of one reference operator on a Batch built ONCE outside the
        timed loop (benchmarks/bench_sgmv.cpp:37-47).  op: lora_addon | sgmv_shrink |
        sgmv_expand.  Returns (seconds_per_call, calls)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        bounds = np.ascontiguousarray(bounds, dtype=np.uint64)
        A = np.ascontiguousarray(A, dtype=np.float64)
        B = np.ascontiguousarray(B, dtype=np.float64)
        b = self.lib.ref_batch_new(x, x.shape[1], bounds, len(bounds) - 1, A.reshape(-1), B.reshape(-1),
                                   B.shape[1], B.shape[2])
        if not b:
            raise ValueError(self.last_error())
        try:
            n = C.c_int()
            t = self.lib.ref_batch_bench(b, {"lora_addon": 0, "sgmv_shrink": 1, "sgmv_expand": 2}[op],
                                         budget_s, max_iters, C.byref(n))
        finally:
            self.lib.ref_batch_free(b)
        return t, n.value

    def last_error(self) -> str:
        return self.lib.ref_last_error().decode()

    def rng(self, seed: int) -> "RefRng":
        return RefRng(self, seed)

    def derive_seed(self, seed, stream):
        return self.lib.ref_derive_seed(seed, stream)

    def model_count_for(self, n, pop):
        return self.lib.ref_model_count_for(n, pop)

    def assign_models(self, n, pop, alpha, seed):
        out = np.zeros(max(n, 1), dtype=np.int64)
        if self.lib.ref_assign_models(n, pop, alpha, seed, out):
            raise ValueError(self.last_error())
        return out[:n]

    def _seg_call(self, name, x, bounds, A, B, *extra):
        x = np.ascontiguousarray(x, dtype=np.float64)
        bounds = np.ascontiguousarray(bounds, dtype=np.uint64)
        A = np.ascontiguousarray(A, dtype=np.float64)
        B = np.ascontiguousarray(B, dtype=np.float64)
        nseg = len(bounds) - 1
        rows = int(bounds[-1]) if nseg else 0
        rank, h_out = B.shape[1], B.shape[2]
        out_cols = rank if name == "sgmv_shrink" else h_out
        y = np.zeros((rows, out_cols), dtype=np.float64)
        st = self.fn(name)(x, x.shape[1], bounds, nseg, A.reshape(-1) if A.size else np.zeros(1),
                           B.reshape(-1) if B.size else np.zeros(1), rank, h_out,
                           *[np.ascontiguousarray(e, dtype=np.float64) for e in extra], y)
        if st:
            raise ValueError(self.last_error())
        return y

    def lora_addon(self, x, bounds, A, B):
        return self._seg_call("lora_addon", x, bounds, A, B)

    def lora_loop_oracle(self, x, bounds, A, B):
        return self._seg_call("lora_loop_oracle", x, bounds, A, B)

    def gather_bmm_oracle(self, x, bounds, A, B):
        return self._seg_call("gather_bmm_oracle", x, bounds, A, B)

    def dense_projection(self, x, bounds, A, B, w):
        return self._seg_call("dense_projection", x, bounds, A, B, w)

    def sgmv_shrink(self, x, bounds, A, B):
        return self._seg_call("sgmv_shrink", x, bounds, A, B)

    def sgmv_expand(self, v, bounds, A, B):
        v = np.ascontiguousarray(v, dtype=np.float64)
        bounds = np.ascontiguousarray(bounds, dtype=np.uint64)
        A = np.ascontiguousarray(A, dtype=np.float64)
        B = np.ascontiguousarray(B, dtype=np.float64)
        h_in, rank, h_out = A.shape[1], A.shape[2], B.shape[2]
        y = np.zeros((v.shape[0], h_out))
        if self.lib.ref_sgmv_expand(v, v.shape[0], bounds, len(bounds) - 1, A.reshape(-1),
                                    B.reshape(-1), h_in, rank, h_out, y):
            raise ValueError(self.last_error())
        return y

    def verify_sgmv(self, trials, seed, inject=False):
        f = C.c_int()
        w = C.c_double()
        d = C.c_double()
        shape = np.zeros(5, dtype=np.uint64)
        if self.lib.ref_verify_sgmv(trials, seed, int(inject), C.byref(f), C.byref(w), C.byref(d), shape):
            raise ValueError(self.last_error())
        return {"failures": f.value, "worst": w.value, "first_fail_dev": d.value,
                "first_fail_shape": shape.tolist()}

    def roofline_csv(self, max_batch=64) -> str:
        n = self.lib.ref_roofline_csv(max_batch, None, 0)
        buf = C.create_string_buffer(n + 1)
        self.lib.ref_roofline_csv(max_batch, buf, n + 1)
        return buf.value.decode()

    def plan_segments(self, lora, prefill_done, prompt):
        return _plan(self.lib.ref_plan_batch, lora, prefill_done, prompt)

    def sgmv_flop(self, n, rows, h_in, h_out):
        return self.lib.ref_sgmv_flop(n, rows, h_in, h_out)

    def sgmv_io_bytes(self, n, rows, h_in, h_out, e=2):
        return self.lib.ref_sgmv_io_bytes(n, rows, h_in, h_out, e)

    def arithmetic_intensity(self, n, rows, h_in, h_out, e=2):
        return self.lib.ref_arithmetic_intensity(n, rows, h_in, h_out, e)

    def sgmv_latency(self, n, rows, h_in, h_out, peak=312e12, bw=2.0e12, floor_s=38e-6, e=2):
        return self.lib.ref_sgmv_latency(n, rows, h_in, h_out, peak, bw, floor_s, e)

    def gather_bmm_extra_elements(self, n, rows, h_in, h_out):
        return self.lib.ref_gather_bmm_extra_elements(n, rows, h_in, h_out)


class RefRng:
    def __init__(self, ref: Reference, seed: int):
        self.r = ref
        self.h = C.c_void_p(ref.lib.ref_rng_new(seed))

    def __del__(self):
        try:
            self.r.lib.ref_rng_free(self.h)
        except Exception:
            pass

    def next(self):
        return self.r.lib.ref_rng_next(self.h)

    def uniform01(self):
        return self.r.lib.ref_rng_uniform01(self.h)

    def uniform_index(self, n):
        return self.r.lib.ref_rng_uniform_index(self.h, n)

    def uniform_int(self, lo, hi):
        return self.r.lib.ref_rng_uniform_int(self.h, lo, hi)

    def discrete(self, cumulative, total):
        c = np.ascontiguousarray(cumulative, dtype=np.float64)
        return self.r.lib.ref_rng_discrete(self.h, c, c.size, total)

    def shuffle(self, v):
        a = np.ascontiguousarray(v, dtype=np.int64).copy()
        self.r.lib.ref_rng_shuffle_i64(self.h, a, a.size)
        return a

    def verify_next_trial(self, trial):
        return _verify_trial(self.r.lib.ref_verify_next_trial, self.h, trial)


def reference_available() -> bool:
    return os.path.exists(REF_SO)
