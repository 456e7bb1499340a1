"""The two-launch small-grid fused step (csrc/small.cu, tgcu_grid_set_step_path):
the auto rule, its launch count, grid-stride batches beyond one thread per
point, and C1-shaped training against the brick path. One-step parity with
the oracle for every order and dimension runs through the step_path fixture
of test_gpu_parity.py."""
import numpy as np
import pytest

import paper_2402_14415_b200 as tg
from conftest import assert_trajectory_close
from oracle.pyoracle import Loss, Spec

pytestmark = pytest.mark.gpu


def _steps_launches(g, batch, k=3):
    tg.train_step(g, batch)  # first step allocates
    tg.reset_launch_count()
    for _ in range(k):
        tg.train_step(g, batch)
    return tg.launch_count() / k


def test_auto_rule_and_launch_counts():
    c1 = tg.GridSpec(dim=2, resolution=(128, 128, 1), order=2)
    batch = tg.sample(tg.SHAPE_C1_2D, 2, 3, 1 << 16)
    g = tg.init_grid(c1)
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    assert _steps_launches(g, batch) == 2  # auto: points + coefficients kernels
    g.set_step_path(tg.TaylorGrid.STEP_BRICK)
    assert _steps_launches(g, batch) == 5  # 3 binning kernels + brick kernel + finalize
    g.set_step_path(tg.TaylorGrid.STEP_SINGLE)
    assert _steps_launches(g, batch) == 2
    g.set_deterministic(True)  # deterministic mode keeps the brick path (+ its 2 sort kernels)
    assert _steps_launches(g, batch) == 7
    # a grid of more than 3 x 2^20 coefficients (96^3 x 10): the brick path
    big = tg.init_grid(tg.GridSpec(dim=3, resolution=(96, 96, 96), order=2))
    big.adam_reset(tg.AdamConfig(lr=1e-2))
    assert _steps_launches(big, tg.sample(tg.SHAPE_SPHERE, 3, 4, 1 << 16, near_frac=0.5, sigma=0.01,
                                          param0=0.6)) == 5
    with pytest.raises(ValueError, match="set_step_path"):
        g.set_step_path(7)


@pytest.mark.parametrize("dim,res,n", [(2, (40, 33, 1), (1 << 21) + 7), (3, (23, 19, 17), (1 << 21) + 333)])
def test_small_path_grid_stride_batches_vs_oracle(oracle, dim, res, n):
    """More points than 8192 CTAs x 256 threads: each thread takes several
    points (the small path forced)."""
    rng = np.random.default_rng(31 + dim)
    s = Spec(dim=dim, res=res, order=2)
    c = (0.1 * rng.standard_normal(s.V * s.K)).astype(np.float32).astype(np.float64)
    shape = tg.SHAPE_C1_2D if dim == 2 else tg.SHAPE_SPHERE
    kw = {} if dim == 2 else dict(near_frac=0.5, sigma=0.01, param0=0.6)
    smp = tg.sample(shape, dim, 77, n, **kw).astype(np.float64)
    gref = np.zeros(s.V * s.K)
    tref = oracle.total_loss(s, c, smp, Loss(), gref)
    mass = oracle.total_loss_mass(s, c, smp, Loss())
    g = tg.init_grid(tg.GridSpec(dim=dim, resolution=res, order=2))
    g.set_step_path(tg.TaylorGrid.STEP_SINGLE)
    g.coeffs = c
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    t = tg.train_step(g, smp, tg.LossConfig(), export_grad=True)
    assert np.all(np.abs(t.as_array() - tref) <= 1e-6 * np.abs(tref) + 1e-30), (t.as_array(), tref)
    # fp32 sums over ~2^21 / V points per vertex in L2 atomics: 1e-5 relative
    # plus the fused step's fp32 mass term (as test_gpu_parity.grad_close)
    gd = g.grad()
    assert np.all(np.abs(gd - gref) <= 1e-5 * np.abs(gref) + 4e-6 * mass), np.max(np.abs(gd - gref))


def test_c1_small_path_tracks_brick_path():
    """C1 (2D 128^2, 65,536 points per step, paper loss, lr 1e-2): 300 steps on
    both paths from zero init on the same batches. They differ only in fp32
    summation order, so the loss curves agree closely early on and the
    trained loss level agrees at the end (the L1 data term makes longer
    trajectories chaotic; test_baseline_parity_gpu pins C1 to the reference)."""
    import torch
    spec = tg.GridSpec(dim=2, resolution=(128, 128, 1), order=2)
    batches = [torch.from_numpy(tg.sample(tg.SHAPE_C1_2D, 2, 100 + i, 1 << 16)).cuda() for i in range(8)]
    torch.cuda.synchronize()
    traces = []
    for path in (tg.TaylorGrid.STEP_BRICK, tg.TaylorGrid.STEP_SINGLE):
        g = tg.init_grid(spec)
        g.set_step_path(path)
        g.adam_reset(tg.AdamConfig(lr=1e-2))
        for i in range(300):
            tg.train_step(g, batches[i % 8], asynchronous=True, input_ready=True)
        g.sync()
        traces.append(g.trace(300))
    a, b = traces
    np.testing.assert_allclose(b[:20, 0], a[:20, 0], rtol=1e-4)
    assert abs(b[-50:, 0].mean() / a[-50:, 0].mean() - 1.0) < 0.02


def test_small_path_async_after_brick_steps_and_back():
    """Switching paths between steps of one grid: the small path's gradient
    accumulator stays zero between steps, so the trajectory equals the
    all-brick one up to summation order."""
    z = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "train.npz"))
    spec = tg.GridSpec(dim=2, resolution=tuple(int(r) for r in z["train_res"]) + (1,), order=2)
    g1, g2 = tg.init_grid(spec), tg.init_grid(spec)
    for g in (g1, g2):
        g.adam_reset(tg.AdamConfig(lr=1e-2))
    g1.set_step_path(tg.TaylorGrid.STEP_BRICK)
    for i, b in enumerate(z["train_batches"]):
        tg.train_step(g1, b)
        g2.set_step_path(tg.TaylorGrid.STEP_BRICK if i % 2 else tg.TaylorGrid.STEP_SINGLE)
        tg.train_step(g2, b, asynchronous=True)
    g2.sync()
    n = len(z["train_batches"])
    np.testing.assert_allclose(g2.trace(n)[:, 0], g1.trace(n)[:, 0], rtol=1e-5)
    assert_trajectory_close(g2.coeffs, g1.coeffs, 1e-2, n, what="mixed-path coeffs")


@pytest.mark.parametrize("dim,res", [(2, (40, 33, 1)), (3, (21, 18, 23))])
def test_train_graph_replays_match_calls(dim, res):
    """tgcu_train_graph_*: replays of captured small-grid steps train exactly
    like the same steps issued call by call (Adam t, ping-pong slot and trace
    rows advanced on the device), also mixed with calls."""
    import torch
    spec = tg.GridSpec(dim=dim, resolution=res, order=2)
    shape = tg.SHAPE_C1_2D if dim == 2 else tg.SHAPE_SPHERE
    kw = {} if dim == 2 else dict(near_frac=0.5, sigma=0.01, param0=0.6)
    batches = [torch.from_numpy(tg.sample(shape, dim, 40 + i, 3000, **kw)).cuda() for i in range(4)]
    torch.cuda.synchronize()
    g1, g2 = tg.init_grid(spec), tg.init_grid(spec)
    for g in (g1, g2):
        g.adam_reset(tg.AdamConfig(lr=1e-2))
    order = [0, 1] + [0, 1, 2, 3] * 3 + [2]   # 2 calls, 3 replays of 4, 1 call
    for i in order:
        tg.train_step(g1, batches[i], asynchronous=True, input_ready=True)
    g1.sync()
    s = torch.cuda.Stream()
    tg.train_step(g2, batches[0], asynchronous=True, input_ready=True, stream=s.cuda_stream)
    tg.train_step(g2, batches[1], asynchronous=True, input_ready=True, stream=s.cuda_stream)
    graph = tg.TrainGraph(g2, batches, stream=s)
    for _ in range(3):
        graph.replay()
    tg.train_step(g2, batches[2], asynchronous=True, input_ready=True, stream=s.cuda_stream)
    g2.sync()
    n = len(order)
    assert g2.adam_t == g1.adam_t == n
    np.testing.assert_allclose(g2.trace(n)[:, 0], g1.trace(n)[:, 0], rtol=1e-5)
    assert_trajectory_close(g2.coeffs, g1.coeffs, 1e-2, n, what="graph coeffs")
    graph.close()


def test_train_graph_refusals_and_errors():
    import torch
    spec = tg.GridSpec(dim=2, resolution=(24, 20, 1), order=2)
    batches = [torch.from_numpy(tg.sample(tg.SHAPE_C1_2D, 2, 7 + i, 2000)).cuda() for i in range(2)]
    torch.cuda.synchronize()
    g = tg.init_grid(spec)
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    with pytest.raises(ValueError, match="even"):
        tg.TrainGraph(g, batches[:1])
    gb = tg.init_grid(spec)
    gb.adam_reset(tg.AdamConfig(lr=1e-2))
    gb.set_step_path(tg.TaylorGrid.STEP_BRICK)
    with pytest.raises(ValueError, match="small-grid step path"):
        tg.TrainGraph(gb, batches)
    graph = tg.TrainGraph(g, batches)
    graph.replay()
    tg.train_step(g, batches[0])  # one step outside: the other ping-pong slot is current
    with pytest.raises(ValueError, match="ping-pong slot"):
        graph.replay()
    tg.train_step(g, batches[1])
    graph.replay()
    g.sync()
    assert g.adam_t == 6
    good = g.coeffs
    # a NaN coordinate in the second captured batch: that step fails, the grid
    # keeps the state after the first one, and replays work again afterwards
    keep = batches[1][3, 0].item()
    batches[1][3, 0] = float("nan")
    graph.replay(torch.cuda.current_stream())
    with pytest.raises(ValueError, match=r"NaN coordinate \(sample 3\) at stage 0 step 7"):
        g.sync()
    assert g.adam_t == 7
    assert not np.array_equal(g.coeffs, good)  # step 6 (the first replayed) committed
    batches[1][3, 0] = keep
    tg.train_step(g, batches[1])  # back to the captured slot
    graph.replay()
    g.sync()
    assert g.adam_t == 10 and np.all(np.isfinite(g.coeffs))
