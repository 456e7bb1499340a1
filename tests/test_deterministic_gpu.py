"""Deterministic mode (tgcu_grid_set_deterministic; the reference's
--deterministic, run_config.cpp:239-242, and its bit-identical run_schedule
traces, test_optimizer.cpp:183-199): repeated fused trainings from the same
inputs give bit-identical coefficients, Adam moments and loss traces — with
multi-chunk (surface) bricks, the binning stream overlap, pipelined host input
and the 2D path — and the trajectory still matches the regular mode's.
"""
import numpy as np
import pytest

import paper_2402_14415_b200 as tg
from conftest import assert_trajectory_close

pytestmark = pytest.mark.gpu


def _run(spec, batches, det, lr=1e-2, device_input=False):
    g = tg.init_grid(spec, tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.02, seed=3))
    g.set_deterministic(det)
    g.adam_reset(tg.AdamConfig(lr=lr))
    if device_input:
        import torch
        dev = [torch.from_numpy(b).cuda() for b in batches]
        torch.cuda.synchronize()
        for b in dev:
            tg.train_step(g, b, asynchronous=True, input_ready=True)
    else:
        for b in batches:
            tg.train_step(g, b, asynchronous=True)
    g.sync()
    out = (g.coeffs_f32(), g.adam_moments(), g.trace(len(batches)))
    g.close()
    return out


@pytest.mark.parametrize("case", ["3d_surface", "3d_c2_shape", "2d"])
def test_deterministic_runs_are_bit_identical(case):
    if case == "3d_surface":  # near-surface batch: many multi-chunk bricks
        spec = tg.GridSpec(dim=3, resolution=(40, 36, 44), order=2)
        batches = [tg.sample(tg.SHAPE_SPHERE, 3, 50 + i, 60000, near_frac=0.9, sigma=0.005, param0=0.6)
                   for i in range(8)]
    elif case == "3d_c2_shape":
        spec = tg.GridSpec(dim=3, resolution=(128, 128, 128), order=2)
        batches = [tg.sample(tg.SHAPE_SPHERE, 3, 70 + i, 1 << 20, near_frac=0.5, sigma=0.01, param0=0.6)
                   for i in range(6)]
    else:
        spec = tg.GridSpec(dim=2, resolution=(128, 128, 1), order=2)
        batches = [tg.sample(tg.SHAPE_C1_2D, 2, 90 + i, 1 << 16) for i in range(10)]
    a = _run(spec, batches, True)
    b = _run(spec, batches, True, device_input=True)
    c = _run(spec, batches, True)
    for x, y in ((a, b), (a, c)):
        assert np.array_equal(x[0], y[0]), "coefficients differ between deterministic runs"
        assert np.array_equal(x[1][0], y[1][0]) and np.array_equal(x[1][1], y[1][1]), "Adam moments differ"
        assert np.array_equal(x[2], y[2]), "loss traces differ"
    # the canonical order changes only the fp32 summation order
    r = _run(spec, batches, False)
    assert np.allclose(r[2], a[2], rtol=1e-5, atol=1e-30)  # (up to 10 steps of differently ordered sums)
    assert_trajectory_close(a[0], r[0], 1e-2, len(batches), what="deterministic vs regular")
