"""The C++ drop-in (include/mumode_b200/mumode.hpp): reference-style client code
compiles against it here (CPU), and runs on the GPU (gpu marker)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "dropin_test.cpp"
LIBDIR = ROOT / "paper_2112_11238_b200"
EXE = ROOT / "build" / "dropin_test"


def build_exe():
    EXE.parent.mkdir(parents=True, exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", str(ROOT / "include"), str(SRC),
           "-o", str(EXE), "-L", str(LIBDIR), "-lmumode_b200", f"-Wl,-rpath,{LIBDIR}"]
    return subprocess.run(cmd, capture_output=True, text=True)


def test_dropin_compiles():
    r = build_exe()
    assert r.returncode == 0, r.stderr
    assert "warning" not in r.stderr, r.stderr


@pytest.mark.gpu
def test_dropin_runs_on_gpu():
    r = build_exe()
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "PASSED" in out.stdout
