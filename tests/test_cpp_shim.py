"""The C++ shim (include/tgcu.hpp) used from a reference-style C++ caller."""
import os
import subprocess

import pytest

from conftest import ROOT

EXE = os.path.join(ROOT, "tests", "cpp", "shim_test")


def test_shim_binary_built():
    assert os.path.exists(EXE), "built by __graft_entry__.build()"


@pytest.mark.gpu
def test_shim_runs_on_gpu():
    env = dict(os.environ)
    env["LD_LIBRARY_PATH"] = os.path.join(ROOT, "paper_2402_14415_b200") + ":" + env.get("LD_LIBRARY_PATH", "")
    r = subprocess.run([EXE], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "shim ok" in r.stdout and "NumericalError: run_schedule: non-finite loss" in r.stdout
