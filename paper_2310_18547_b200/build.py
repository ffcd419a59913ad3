"""In-tree build of the native libraries (no pip install, no JIT cache).

  paper_2310_18547_b200/lib/libsgmv_b200.so          CUDA kernels + the C-ABI (include/lsg_sgmv.h)
  paper_2310_18547_b200/lib/liblorasim_sgmv_b200.so  C++ drop-in replacing exactly the reference's
                                                     core/src/sgmv.cpp (lorasim::sgmv_* & co.),
                                                     linked against libsgmv_b200.so
  paper_2310_18547_b200/lib/liblorasim_b200.so       this repo's restatement of the rest of the
                                                     SGMV tooling (workload, cost model, verify)
  paper_2310_18547_b200/lib/lorasim_b200             CLI (verify-sgmv, roofline)

Everything is compiled for sm_100a only: -gencode arch=compute_100a,code=sm_100a.
Targets are rebuilt only when a source is newer than the output.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "lib")
OBJ = os.path.join(PKG, "lib", "obj")
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(PKG, "host")
INCLUDE = os.path.join(ROOT, "include")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
                     "--expt-relaxed-constexpr", f"-I{INCLUDE}"]
CXX_FLAGS = ["-std=c++20", "-O3", "-fPIC", "-Wall", "-Wextra", f"-I{INCLUDE}",
             f"-I{os.path.join(HOST, 'include')}", f"-I{CUDA}/include"]

SGMV_SO = os.path.join(LIB, "libsgmv_b200.so")
DROPIN_SO = os.path.join(LIB, "liblorasim_sgmv_b200.so")
DROPIN_SRCS = ("matrix.cpp", "sgmv_cuda.cpp")
HOST_SO = os.path.join(LIB, "liblorasim_b200.so")
CLI_BIN = os.path.join(LIB, "lorasim_b200")


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    return r


def build(verbose: bool = False) -> None:
    os.makedirs(OBJ, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    cu_srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    objs = []
    jobs = []
    for src in cu_srcs:
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        objs.append(obj)
        if _newer(obj, [src] + headers):
            jobs.append(NVCC_FLAGS + ["-c", src, "-o", obj])
    if jobs:
        with ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            list(ex.map(lambda j: _run([NVCC] + j, verbose), jobs))
    if _newer(SGMV_SO, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", SGMV_SO] + objs, verbose)

    host_hdrs = glob.glob(os.path.join(HOST, "include", "lorasim", "*.hpp")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    # The drop-in: exactly the symbols the reference's core/src/sgmv.cpp defines
    # (matmul, max_abs_diff, Segments / LoraModel / Batch, the four operators and the two
    # oracles), so a reference build that drops sgmv.cpp links it without duplicates.
    dropin_srcs = [os.path.join(HOST, "src", f) for f in DROPIN_SRCS]
    if _newer(DROPIN_SO, dropin_srcs + host_hdrs + [SGMV_SO]):
        _run(["g++"] + CXX_FLAGS + ["-shared", "-o", DROPIN_SO] + dropin_srcs +
             [f"-L{LIB}", "-lsgmv_b200", f"-L{CUDA}/lib64", "-lcudart_static", "-lcublas", "-ldl", "-lrt", "-lpthread",
              "-Wl,-rpath,$ORIGIN", f"-Wl,-rpath,{CUDA}/lib64"], verbose)
    # This repo's own restatement of the rest of the SGMV tooling (workload RNG, cost
    # formulas, verify_sgmv / roofline_sweep) for the CLI and the C++ tests.
    host_srcs = sorted(p for p in glob.glob(os.path.join(HOST, "src", "*.cpp")) if os.path.basename(p) not in DROPIN_SRCS)
    if host_srcs and _newer(HOST_SO, host_srcs + host_hdrs + [DROPIN_SO]):
        _run(["g++"] + CXX_FLAGS + ["-shared", "-o", HOST_SO] + host_srcs +
             [f"-L{LIB}", "-llorasim_sgmv_b200", "-Wl,-rpath,$ORIGIN"], verbose)
    cli_src = os.path.join(HOST, "tools", "lorasim_b200_cli.cpp")
    if os.path.exists(cli_src) and _newer(CLI_BIN, [cli_src, HOST_SO, DROPIN_SO] + host_hdrs):
        _run(["g++"] + CXX_FLAGS + ["-o", CLI_BIN, cli_src, f"-L{LIB}", "-llorasim_b200", "-llorasim_sgmv_b200",
              "-lsgmv_b200", f"-L{CUDA}/lib64", "-lcudart_static", "-ldl", "-lrt", "-lpthread", "-Wl,-rpath,$ORIGIN",
              f"-Wl,-rpath,{CUDA}/lib64"], verbose)


if __name__ == "__main__":
    build(verbose=True)
    print("built", SGMV_SO)
