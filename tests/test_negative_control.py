"""Negative control (the reference CLI's `validate --inject-fault`,
tools/mumode_cli.cpp:142,168,398-400): the parity checkers must FAIL when the
engine's result is corrupted, and PASS otherwise -- a checker that cannot fail
proves nothing."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

import oracle as O

ROOT = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]


def _run(*args):
    return subprocess.run([sys.executable, *args], capture_output=True, text=True, timeout=900, cwd=ROOT)


def test_validate_suite_passes_and_fails_on_injected_fault():
    ok = _run("tools/validate.py", "--cases", "30")
    assert ok.returncode == 0 and "PASS" in ok.stdout, ok.stdout + ok.stderr[-2000:]
    bad = _run("tools/validate.py", "--cases", "30", "--inject-fault")
    assert bad.returncode == 1 and "FAIL" in bad.stdout, bad.stdout + bad.stderr[-2000:]


def test_parity_report_fails_on_injected_fault():
    ok = _run("tools/parity_report.py", "--quick")
    assert ok.returncode == 0, ok.stdout[-2000:] + ok.stderr[-2000:]
    assert json.loads(ok.stdout)["overall"] == "PASS"
    bad = _run("tools/parity_report.py", "--quick", "--inject-fault")
    assert bad.returncode == 1, bad.stdout[-2000:]
    rep = json.loads(bad.stdout)
    assert rep["overall"] == "FAIL" and rep["failed"] == ["C2_tucker_256"]
