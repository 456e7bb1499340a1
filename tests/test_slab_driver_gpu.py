"""SlabTrainer (the multi-GPU driver bench.py uses at --gpus N) with two ranks.

One GPU is available here, so both ranks run in separate processes on cuda:0
over libtgcu's communicator with the host backend (host-staged all-reduce /
halo exchange over its TCP star; NCCL refuses two ranks on one device); no
kernel of one rank waits on the other's. No PyTorch on the path. The gathered owned slabs must reproduce a single-grid run,
with the halo exchanged after each step or written by the brick kernel into
the neighbour's buffers (fused halo through CUDA IPC, which two processes on
one device support as NVLink peers do).
"""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT, assert_trajectory_close

pytestmark = pytest.mark.gpu

RES = (32, 24, 40)
STEPS = 5


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batches():
    import paper_2402_14415_b200 as tg
    return [tg.sample(tg.SHAPE_SPHERE, 3, 900 + i, 30000, near_frac=0.5, sigma=0.01, param0=0.6)
            for i in range(STEPS)]


def _rank(rank, world, port, outdir, fused, det=False):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["TGCU_FUSED_HALO"] = "1" if fused else "0"
    if det:  # no split bricks: the cluster split changes the association of the per-vertex sums
        os.environ["TGCU_SPLIT"] = "1"
    import paper_2402_14415_b200 as tg
    from paper_2402_14415_b200.slab import Comm, SlabTrainer
    comm = Comm(rank, world, device=0, addr="127.0.0.1", port=port, backend="host")
    spec = tg.GridSpec(dim=3, resolution=RES, order=2)
    init = tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.02, seed=11)
    tr = SlabTrainer(spec, rank, world, tg.AdamConfig(lr=1e-2), device=0, opts=init, comm=comm)
    if det:
        tr.slab.set_deterministic(True)
    terms = []
    for i, b in enumerate(_batches()):
        if i % 2:  # host samples, local shard with the global batch size
            terms.append(tr.step(tr.local_points(b), tg.LossConfig(), want_terms=True, n_global=len(b)).as_array())
        else:
            terms.append(tr.step(b, tg.LossConfig(), want_terms=True).as_array())
    assert "torch" not in sys.modules
    np.save(os.path.join(outdir, f"own{rank}.npy"), tr.slab.owned_coeffs())
    np.save(os.path.join(outdir, f"fused{rank}.npy"), np.array([tr.fused_halo]))
    np.save(os.path.join(outdir, f"terms{rank}.npy"), np.array(terms))
    tr.close()


@pytest.mark.parametrize("world,fused,det", [(2, False, False), (2, True, False), (3, True, False), (2, False, True),
                                            (3, True, True)])
def test_slab_trainer_two_ranks_match_single_grid(tmp_path, monkeypatch, world, fused, det):
    """det: deterministic mode on the slabs and on the single grid, split
    bricks off on both (a cluster split sums a vertex's chunks in another
    association) — every brick sums in a canonical order, so the gathered
    slabs equal the single grid bit for bit (the loss terms may still differ
    in the last bits: the ranks' partial sums are added in another
    association)."""
    import multiprocessing as mp
    if det:
        monkeypatch.setenv("TGCU_SPLIT", "1")
    import paper_2402_14415_b200 as tg
    ctx = mp.get_context("spawn")
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, world, port, str(tmp_path), fused, det)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
    assert all(p.exitcode == 0 for p in ps), [p.exitcode for p in ps]
    for r in range(world):
        assert bool(np.load(tmp_path / f"fused{r}.npy")[0]) == fused
    spec = tg.GridSpec(dim=3, resolution=RES, order=2)
    g = tg.init_grid(spec, tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.02, seed=11))
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    g.set_deterministic(det)
    ref = np.array([tg.train_step(g, b).as_array() for b in _batches()])
    own = np.concatenate([np.load(tmp_path / f"own{r}.npy") for r in range(world)])
    full = g.coeffs
    assert own.shape == full.shape
    if det:
        dd = np.abs(own - full)
        assert np.array_equal(own, full), (int((dd > 0).sum()), float(dd.max()), np.nonzero(dd)[0][:20].tolist())
    else:
        assert_trajectory_close(own, full, 1e-2, STEPS, what="slab vs single-grid coeffs")
    for r in range(world):
        t = np.load(tmp_path / f"terms{r}.npy")
        assert np.all(np.abs(t - ref) <= 1e-5 * np.abs(ref) + 1e-30)  # (summation order differs: ~1e-6 per step)


def test_slab_trainer_nccl_single_rank_matches_single_grid():
    """The NCCL backend of libtgcu's communicator (dlopen'ed libnccl, unique
    id over the TCP star, all-reduce of the partials on the step's stream) on
    the one GPU here: a one-rank job whose slab is the whole grid reproduces
    the single-grid trajectory bit for bit (deterministic mode on both)."""
    import paper_2402_14415_b200 as tg
    from paper_2402_14415_b200.slab import Comm, SlabTrainer
    spec = tg.GridSpec(dim=3, resolution=RES, order=2)
    init = tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.02, seed=11)
    comm = Comm(0, 1, device=0, addr="127.0.0.1", port=_port(), backend="nccl")
    tr = SlabTrainer(spec, 0, 1, tg.AdamConfig(lr=1e-2), device=0, opts=init, comm=comm)
    assert tr.backend == "nccl" and not tr.fused_halo
    g = tg.init_grid(spec, init)
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    # deterministic mode on both (otherwise the two runs sum in different
    # orders and separate by ~1e-6 per step): identical bits
    tr.slab.set_deterministic(True)
    g.set_deterministic(True)
    for b in _batches():
        t_slab = tr.step(b, tg.LossConfig(), want_terms=True).as_array()
        t_full = tg.train_step(g, b).as_array()
        assert np.array_equal(t_slab, t_full)
    for b in _batches():  # stream-ordered steps (no host sync per step)
        tr.step(b, tg.LossConfig())
        tg.train_step(g, b, asynchronous=True)
    assert np.array_equal(tr.slab.sync().as_array(), g.sync().as_array())
    assert np.array_equal(tr.slab.owned_coeffs(), g.coeffs)
    tr.close()


SLAB_DRIVER = os.path.join(ROOT, "tests", "cpp", "slab_driver")


@pytest.mark.parametrize("world,fused,backend", [(2, 0, "host"), (3, 1, "host"), (1, 0, "nccl")])
def test_cpp_slab_driver_processes_match_single_grid(tmp_path, world, fused, backend):
    """tests/cpp/slab_driver.cpp: `world` C++ processes drive a slab job
    through the C ABI alone (tgcu_comm_create, tgcu_grid_create_slab,
    tgcu_slab_connect, tgcu_slab_train_step; full batches and local point
    shards on alternate steps); gathered owned planes and every rank's loss
    terms against the single-grid run."""
    import subprocess
    import paper_2402_14415_b200 as tg
    assert os.path.exists(SLAB_DRIVER), "built by __graft_entry__.build()"
    port = _port()
    ps = [subprocess.Popen([SLAB_DRIVER, str(r), str(world), str(port), str(fused), backend, str(tmp_path)],
                           stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(world)]
    outs = [p.communicate(timeout=300)[0] for p in ps]
    assert all(p.returncode == 0 for p in ps), outs
    for r in range(world):
        assert (tmp_path / f"cpp_fused{r}.txt").read_text() == str(fused), outs
    spec = tg.GridSpec(dim=3, resolution=RES, order=2)
    g = tg.init_grid(spec, tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.02, seed=11))
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    ref = np.array([tg.train_step(g, b).as_array() for b in _batches()])
    own = np.concatenate([np.fromfile(tmp_path / f"cpp_own{r}.f64") for r in range(world)])
    assert own.shape == g.coeffs.shape
    assert_trajectory_close(own, g.coeffs, 1e-2, STEPS, what="C++ slab job vs single-grid coeffs")
    for r in range(world):
        t = np.fromfile(tmp_path / f"cpp_terms{r}.f64").reshape(-1, 4)
        assert np.all(np.abs(t - ref) <= 1e-5 * np.abs(ref) + 1e-30), (r, t, ref)
