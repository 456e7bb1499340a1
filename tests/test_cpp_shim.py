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


REF_TOOL = os.path.join(ROOT, "tests", "cpp", "ref_cmd_bench")


@pytest.mark.gpu
def test_reference_style_tool_on_gpu():
    """tests/cpp/ref_cmd_bench.cpp: cmd_bench / run_schedule written with the
    reference's own types, driving libtgcu (tgcu_tg.hpp), each check against
    the reference in-process."""
    if not os.path.exists(REF_TOOL):
        pytest.skip("built by __graft_entry__.build() where the reference sources are present")
    r = subprocess.run([REF_TOOL], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ref tool ok" in r.stdout and "tg::NumericalError" in r.stdout
