"""The C++ drop-in (lorasim:: API on the B200) through the reference's own test
cases: tests/cpp/test_dropin.cpp (mirror of proj/tests/unit/test_sgmv.cpp) and the
CLI contract of proj/tests/cli/check_cli.sh for the SGMV verbs."""
from __future__ import annotations

import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2310_18547_b200", "lib")
ORACLE = os.path.join(ROOT, "oracle")
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
BIN = os.path.join(LIB, "test_dropin")
CLI = os.path.join(LIB, "lorasim_b200")


def _build():
    deps = [SRC, os.path.join(LIB, "liblorasim_b200.so"), os.path.join(LIB, "liblorasim_sgmv_b200.so"), os.path.join(ORACLE, "liboracle.so")]
    if os.path.exists(BIN) and all(os.path.getmtime(BIN) >= os.path.getmtime(d) for d in deps if os.path.exists(d)):
        return
    subprocess.run(["g++", "-std=c++20", "-O2", "-o", BIN, SRC,
                    f"-I{ROOT}/paper_2310_18547_b200/host/include", f"-I{ROOT}/include", f"-I{ORACLE}",
                    "-I/usr/local/cuda/include", f"-L{LIB}", "-llorasim_b200", "-llorasim_sgmv_b200", f"-L{ORACLE}", "-loracle",
                    f"-Wl,-rpath,{LIB}", f"-Wl,-rpath,{ORACLE}"], check=True)


def test_dropin_validation_cpu():
    """Reference validation semantics (same exceptions and messages), no GPU needed."""
    _build()
    r = subprocess.run([BIN, "cpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_cli_usage_contract_cpu(tmp_path):
    r = subprocess.run([CLI], capture_output=True, text=True)
    assert r.returncode == 2
    r = subprocess.run([CLI, "--out", str(tmp_path), "roofline"], capture_output=True, text=True)
    assert r.returncode == 0
    ours = (tmp_path / "roofline.csv").read_text()
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "cost_model.json")))["roofline_csv"]
    assert ours == golden  # byte-identical to the reference's roofline.csv


@pytest.mark.gpu
def test_dropin_reference_unit_tests_on_gpu():
    _build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cli_verify_sgmv_contract_on_gpu():
    """check_cli.sh:18-22: clean run exits 0, a planted fault exits 1."""
    r = subprocess.run([CLI, "verify-sgmv", "--trials", "150"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    r = subprocess.run([CLI, "verify-sgmv", "--trials", "4", "--inject-fault"], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 1, r.stdout + r.stderr


ACCEPTANCE = os.path.join(ORACLE, "_ref", "acceptance_b200")


@pytest.mark.gpu
def test_reference_acceptance_with_b200_dropin():
    """The reference's own release gate (proj/tests/acceptance/acceptance_main.cpp, compiled
    unmodified with the reference's other core TUs by integration/CMakeLists.txt -- core/src/
    sgmv.cpp removed, liblorasim_sgmv_b200.so linked instead) on the GPU: criteria 1-3 (the SGMV
    path: verify_sgmv(1000, 42) three-way equivalence < 1e-10 in < 60 s, the intensity algebra,
    the formula anchors) must PASS; the simulator criteria 4-8 run on the same binary too."""
    assert os.path.exists(ACCEPTANCE), "oracle/_ref/acceptance_b200 missing: build() with /root/reference present"
    r = subprocess.run([ACCEPTANCE, os.path.join(ORACLE, "_ref")], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    lines = r.stdout.splitlines()
    for i in (1, 2, 3):
        assert any(ln.startswith(f"PASS  {i}.") for ln in lines), r.stdout + r.stderr
    assert r.returncode == 0 and "all 8 criteria passed" in r.stdout, r.stdout + r.stderr


def test_reference_simulator_with_b200_costs_cpu():
    """the reference's own compare / calibration / cluster-replay experiments run with
    the B200-fitted SGMV cost model (integration/sim_b200.cpp over the reference simulator built in
    place); both passes complete and the multi-adapter advantage survives on B200 (Distinct ratio
    well above 1, Identical = 1)."""
    exe = os.path.join(ROOT, "oracle", "_ref", "sim_b200")
    proj = "/root/reference/proj"
    if not (os.path.exists(exe) and os.path.isdir(proj)):
        pytest.skip("needs the reference tree and oracle/_ref/sim_b200 (built by __graft_entry__.build())")
    out = subprocess.run([exe, proj, os.path.join(ROOT, "profiles", "round1", "b200_cost_params.json")],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.splitlines()
    for label in ("A100", "B200"):
        rows = [l for l in lines if l.strip().startswith(("distinct", "identical"))]
        assert any(label in l for l in lines), label
        assert len(rows) == 4, rows
    b200 = lines[[i for i, l in enumerate(lines) if l.startswith("B200") and "compare_modes" in l][0] + 1]
    assert float(b200.split("ratio")[1]) > 5.0, b200
