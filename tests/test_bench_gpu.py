"""bench.py contract on the GPU: the N=1 JSON line carries every key the
driver reads, and the N>1 slab flow (torchrun, here two ranks over gloo on
one device) runs end to end."""
import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _line(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_bench_single_gpu_contract():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "20", "--warmup", "3", "--no-query",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["value"] > 0
    assert d["gpu_launches"] == 5 * 20  # 3 binning kernels + brick step + finalize per step
    assert 0 < d["roofline"]["frac"] < 1 and d["e2e"]["h2d_bytes_per_step"] == 16 << 20
    assert "workload" in d["config"]
    st = d["stages"]  # the 8(f) legs (no reference samples with --no-cpu-baseline)
    assert st["upsample"]["ms"] > 0 and 0 < st["upsample"]["frac"] < 1
    assert st["lattice_query"]["ms"] > 0 and 0 < st["lattice_query"]["frac"] < 1
    assert st["radiance"]["gsamples_per_s"] > 0


def test_bench_two_rank_slab_flow():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    # both ranks share the one GPU: gloo for the bench's own barriers / max,
    # libtgcu's host-staged communicator for the slab step (NCCL refuses two
    # ranks on one device)
    env = dict(os.environ, TGCU_DIST_BACKEND="gloo", TGCU_COMM_BACKEND="host")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
                        "--steps", "4", "--warmup", "3", "--no-cpu-baseline"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["loss_last"] == d["loss_last"]
    assert d["scaling"] == "strong" and d["config"]["grid"] == [256, 256, 256]  # C3 strong scaling
    assert d["collectives"] == "host" and len(d["per_rank_kernel_ms"]) == 2 and d["single_gpu"]["value"] > 0
    assert len(d["per_rank_allreduce_ms"]) == 2 and all(x > 0 for x in d["per_rank_allreduce_ms"])
