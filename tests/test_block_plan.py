"""The K9 block-pass planner's host logic (block.cuh: layout search, row
tables, copy segments), compiled with nvcc and run on the CPU."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "block_plan_check.cu"
EXE = ROOT / "build" / "block_plan_check"


@pytest.mark.skipif(shutil.which("nvcc") is None and not Path("/usr/local/cuda/bin/nvcc").exists(),
                    reason="nvcc not available")
def test_block_plan_tables_and_segments():
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    EXE.parent.mkdir(parents=True, exist_ok=True)
    r = subprocess.run([nvcc, "-std=c++17", "-O2", "-gencode", "arch=compute_100a,code=sm_100a", str(SRC), "-o",
                        str(EXE)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "PASSED" in out.stdout, out.stdout + out.stderr
