"""SlabTrainer (the multi-GPU driver bench.py uses at --gpus N) with two ranks.

One GPU is available here, so both ranks run in separate processes on cuda:0
over gloo (host-staged all-reduce / halo exchange); no kernel of one rank waits
on the other's. The gathered owned slabs must reproduce a single-grid run,
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


def _rank(rank, world, port, outdir, fused):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["TGCU_FUSED_HALO"] = "1" if fused else "0"
    import torch
    import torch.distributed as dist
    import paper_2402_14415_b200 as tg
    from paper_2402_14415_b200.slab import SlabTrainer
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    spec = tg.GridSpec(dim=3, resolution=RES, order=2)
    init = tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.02, seed=11)
    tr = SlabTrainer(spec, rank, world, tg.AdamConfig(lr=1e-2), device=0, opts=init)
    terms = []
    for b in _batches():
        terms.append(tr.step(torch.from_numpy(b).cuda(), tg.LossConfig(), want_terms=True).as_array())
    np.save(os.path.join(outdir, f"own{rank}.npy"), tr.slab.owned_coeffs())
    np.save(os.path.join(outdir, f"fused{rank}.npy"), np.array([tr.fused_halo]))
    np.save(os.path.join(outdir, f"terms{rank}.npy"), np.array(terms))
    dist.destroy_process_group()


@pytest.mark.parametrize("fused", [False, True])
def test_slab_trainer_two_ranks_match_single_grid(tmp_path, fused):
    import torch.multiprocessing as mp
    import paper_2402_14415_b200 as tg
    mp.spawn(_rank, args=(2, _port(), str(tmp_path), fused), nprocs=2, join=True)
    for r in range(2):
        assert bool(np.load(tmp_path / f"fused{r}.npy")[0]) == fused
    spec = tg.GridSpec(dim=3, resolution=RES, order=2)
    g = tg.init_grid(spec, tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.02, seed=11))
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    ref = np.array([tg.train_step(g, b).as_array() for b in _batches()])
    own = np.concatenate([np.load(tmp_path / "own0.npy"), np.load(tmp_path / "own1.npy")])
    full = g.coeffs
    assert own.shape == full.shape
    assert_trajectory_close(own, full, 1e-2, STEPS, what="slab vs single-grid coeffs")
    for r in range(2):
        t = np.load(tmp_path / f"terms{r}.npy")
        assert np.all(np.abs(t - ref) <= 1e-6 * np.abs(ref) + 1e-30)
