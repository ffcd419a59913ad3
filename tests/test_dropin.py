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
    deps = [SRC, os.path.join(LIB, "liblorasim_b200.so"), os.path.join(ORACLE, "liboracle.so")]
    if os.path.exists(BIN) and all(os.path.getmtime(BIN) >= os.path.getmtime(d) for d in deps if os.path.exists(d)):
        return
    subprocess.run(["g++", "-std=c++20", "-O2", "-o", BIN, SRC,
                    f"-I{ROOT}/paper_2310_18547_b200/host/include", f"-I{ROOT}/include", f"-I{ORACLE}",
                    "-I/usr/local/cuda/include", f"-L{LIB}", "-llorasim_b200", f"-L{ORACLE}", "-loracle",
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
