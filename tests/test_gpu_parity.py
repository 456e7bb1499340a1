"""GPU parity of the CUDA path (through the C ABI) against the reference.

Tolerances (BASELINE.json north_star), written per test:
  forward values          |d| <= 1e-6 * max(1, |ref|)
  spatial gradients       |d| <= 1e-5 * max(1, |ref|)   (scale 1/h; fp32 blend)
  coefficient gradients   |d| <= 1e-5 * |ref| + 2e-6 * mass
                          mass = sum over the point / TV-pair contributions of their
                          absolute values (oracle tgo_*_mass): fp32 summands added in a
                          different order can only be compared against that scale when a
                          sum cancels (1e-5 rel is exact for non-cancelling sums)
  loss curve over N steps |d| <= 1e-4 * |ref|
Indices (cells, vertex ids, NaN/bad-gradient indices) are exact.
"""
import numpy as np
import pytest

import paper_2402_14415_b200 as tg
from conftest import assert_trajectory_close, load_golden
from oracle.pyoracle import Loss, Spec

pytestmark = pytest.mark.gpu


def gspec(dim, res, order):
    res = tuple(int(r) for r in res)
    return tg.GridSpec(dim=dim, resolution=res if dim == 3 else res[:2] + (1,), order=order)


def ospec(dim, res, order):
    return Spec(dim=dim, res=tuple(int(r) for r in res), order=order)


def assert_close(got, ref, rel, floor=1.0, what=""):
    got = np.asarray(got, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    tol = rel * np.maximum(np.abs(ref), np.asarray(floor, dtype=np.float64).ravel())
    bad = np.abs(got - ref) > tol
    w = int(np.argmax(np.abs(got - ref) / tol))
    assert not bad.any(), (f"{what}: {bad.sum()} / {bad.size} out of tolerance; worst "
                           f"{np.max(np.abs(got - ref) / tol):.3g}x tol at {w}: got {got[w]:.8g} ref {ref[w]:.8g}")


def grad_close(got, ref, mass, rel=1e-5, mass_rel=4e-6, what="grad"):
    """|d| <= rel*|ref| + mass_rel*mass. mass = the oracle's L1 sum of the
    contributions (with the differentiate_weight term counted apart from the
    weight term: they are separate fp32-rounded summands that may cancel). Each contribution carries the fp32 record rounding (~2e-7)
    and, through the adaptive weight w' ~ 2 exp(-k|f|) far from the surface
    (sdf_loss.cpp:15-27), the fp32 forward error amplified by k: k * 6e-8 =
    3e-6 relative at k = 50 -> mass_rel = 4e-6."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    tol = rel * np.abs(ref) + mass_rel * mass + 1e-300
    bad = np.abs(got - ref) > tol
    w = int(np.argmax(np.abs(got - ref) / tol))
    assert not bad.any(), (f"{what}: {bad.sum()} / {bad.size} out of tolerance; worst "
                           f"{np.max(np.abs(got - ref) / tol):.3g}x tol at index {w}: "
                           f"got {got[w]:.6g} ref {ref[w]:.6g} mass {np.asarray(mass).ravel()[w]:.3g}")


# ---- K1 forward -------------------------------------------------------------------------



@pytest.fixture(params=["brick", "small"])
def step_path(request, monkeypatch):
    """Both fused-step paths (tgcu_grid_set_step_path, read from
    TGCU_STEP_PATH at grid creation): the brick kernel (train.cu) and the
    two-launch small-grid step (small.cu) that the auto rule picks for these
    grids."""
    monkeypatch.setenv("TGCU_STEP_PATH", "brick" if request.param == "brick" else "single")
    return request.param

@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("order", [0, 1, 2])
def test_eval_golden(dim, order):
    z = load_golden("eval_backprop.npz")
    k = f"d{dim}o{order}_"
    g = tg.init_grid(gspec(dim, z[k + "res"], order))
    g.coeffs = z[k + "coeffs"]
    pts = z[k + "pts"]
    vals, grads = tg.eval_with_spatial_gradient(g, pts)
    assert_close(vals, z[k + "vals"], 1e-6, what="value")
    assert_close(grads, z[k + "grads"][:, :dim], 1e-5, what="spatial grad")
    assert np.array_equal(tg.eval(g, pts), vals)


@pytest.mark.parametrize("order", [1, 2])
def test_eval_large_vs_oracle_and_sorted(oracle, order):
    rng = np.random.default_rng(3 + order)
    res = (65, 64, 63)
    s = ospec(3, res, order)
    c = (0.1 * rng.standard_normal(s.V * s.K)).astype(np.float32)
    g = tg.init_grid(gspec(3, res, order))
    g.set_coeffs_f32(c)
    pts = rng.uniform(-1.02, 1.02, (20000, 3)).astype(np.float32)
    vals = tg.eval(g, pts)
    ref = oracle.eval(s, c.astype(np.float64), pts.astype(np.float64))
    assert_close(vals, ref, 1e-6, what="value")
    # brick-binned query on sorted points gives the same values
    import torch
    dp = torch.from_numpy(pts).cuda()
    sp = torch.empty_like(dp)
    perm = torch.empty(len(pts), dtype=torch.int64, device="cuda")
    offs = torch.empty(tg.query_brick_codes(g) + 1, dtype=torch.int64, device="cuda")
    tg.sort_points(g, dp, sp, perm, offs)
    v2, g2 = tg.eval_with_spatial_gradient(g, sp, sorted_points=True)  # offsets recomputed internally
    v1, g1 = tg.eval_with_spatial_gradient(g, sp)
    v3 = tg.eval_sorted(g, sp, offs)
    torch.cuda.synchronize()
    assert torch.equal(v1, v2) and torch.equal(v1, v3)
    assert torch.equal(g1, g2)
    assert int(offs[-1].item()) == len(pts) and bool((offs[1:] >= offs[:-1]).all())
    assert np.array_equal(np.sort(perm.cpu().numpy()), np.arange(len(pts)))
    assert_close(v2.cpu().numpy(), ref[perm.cpu().numpy()], 1e-6, what="sorted value")


def test_locate_edge_cases_and_nan():
    # max-boundary -> last cell with local 1; out-of-domain clamps; NaN rejected
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=(3, 3, 3), origin=(0, 0, 0), extent=(1, 1, 1), order=0))
    c = np.zeros(27)
    c[26] = 1.0  # vertex (2,2,2)
    g.coeffs = c
    v = tg.eval(g, [[1.0, 1.0, 1.0], [5.0, 5.0, 5.0], [0.75, 0.75, 0.75], [0.0, 0.0, 0.0]])
    assert v[0] == 1.0 and v[1] == 1.0 and v[2] == pytest.approx(0.125) and v[3] == 0.0
    with pytest.raises(ValueError, match="NaN coordinate"):
        tg.eval(g, [[0.5, float("nan"), 0.5]])


# ---- backward ---------------------------------------------------------------------------


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("order", [0, 1, 2])
def test_backprop_golden(oracle, dim, order):
    z = load_golden("eval_backprop.npz")
    k = f"d{dim}o{order}_"
    g = tg.init_grid(gspec(dim, z[k + "res"], order))
    g.coeffs = z[k + "coeffs"]
    g.zero_grad()
    tg.backprop_value_and_spatial(g, z[k + "pts"], z[k + "up"], z[k + "uv"][:, :dim])
    mass = oracle.backprop_mass(ospec(dim, z[k + "res"], order), z[k + "pts"], z[k + "up"], z[k + "uv"])
    grad_close(g.grad(), z[k + "bgrad"], mass)


def test_backprop_locality_80():
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=(5, 5, 5), order=2))
    g.zero_grad()
    tg.backprop_point(g, [[0.137, -0.295, 0.481]], [1.3])
    assert int(np.count_nonzero(g.grad())) == 80


# ---- losses -------------------------------------------------------------------------------


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("name,cfg", [("paper", tg.LossConfig()),
                                      ("recon", tg.LossConfig(lambda1=0.0, use_tv=False)),
                                      ("dw", tg.LossConfig(differentiate_weight=True))])
def test_total_loss_golden_unfused_and_fused(oracle, dim, name, cfg, step_path):
    z = load_golden("loss.npz")
    k = f"d{dim}_{name}_"
    spec = gspec(dim, z[k + "res"], 2)
    mass = oracle.total_loss_mass(ospec(dim, z[k + "res"], 2), z[k + "coeffs"], z[k + "samples"],
                                  Loss(cfg.lambda1, cfg.lambda2, cfg.k, cfg.use_weighting, cfg.use_tv,
                                       cfg.differentiate_weight))
    g = tg.init_grid(spec)
    g.coeffs = z[k + "coeffs"]
    g.zero_grad()
    terms = tg.total_loss(g, z[k + "samples"], cfg)
    assert_close(terms.as_array(), z[k + "terms"], 1e-6, floor=1e-30, what="terms")
    grad_close(g.grad(), z[k + "grad"], mass, what="unfused grad")
    # fused step: same loss terms (on the pre-step params) and the same full gradient
    g2 = tg.init_grid(spec)
    g2.coeffs = z[k + "coeffs"]
    g2.adam_reset(tg.AdamConfig(lr=1e-2))
    t2 = tg.train_step(g2, z[k + "samples"], cfg, export_grad=True)
    assert_close(t2.as_array(), z[k + "terms"], 1e-6, floor=1e-30, what="fused terms")
    grad_close(g2.grad(), z[k + "grad"], mass, what="fused grad")


def test_tv_golden(oracle):
    z = load_golden("loss.npz")
    for dim in (2, 3):
        k = f"d{dim}_tv_"
        g = tg.init_grid(gspec(dim, z[k + "res"], 2))
        g.coeffs = z[k + "coeffs"]
        g.zero_grad()
        tv = tg.tv_loss(g, with_grad=True, scale=0.7)
        assert tv == pytest.approx(z[k + "tv"][0], rel=1e-6)
        # TV-only mass: lambda2 = 0.7 scale, no point terms
        mass = oracle.total_loss_mass(ospec(dim, z[k + "res"], 2), z[k + "coeffs"], np.zeros((1, 4)) + 5.0,
                                      Loss(lambda1=0.0, lambda2=0.7, use_weighting=False))
        grad_close(g.grad(), z[k + "grad"], mass, what="tv grad")


# ---- Adam + training trajectory ------------------------------------------------------------------


def test_adam_golden_and_errors():
    z = load_golden("train.npz")
    n = len(z["adam_p0"])
    g = tg.init_grid(tg.GridSpec(dim=2, resolution=(n, 1 + 1, 1), order=0))  # 2n coeffs
    p0 = np.concatenate([z["adam_p0"], np.zeros(n)])
    g.coeffs = p0
    g.adam_reset(tg.AdamConfig(lr=0.01))
    import torch
    gbuf = torch.zeros(2 * n, dtype=torch.float32, device="cuda")
    for k in range(len(z["adam_grads"])):
        gbuf[:n] = torch.from_numpy(z["adam_grads"][k].astype(np.float32))
        tg.adam_step(g, gbuf.data_ptr())
        assert_close(g.coeffs[:n], z["adam_traj"][k], 1e-5, floor=1e-2, what=f"adam step {k}")
    before = g.coeffs
    gbuf[5] = float("nan")
    with pytest.raises(tg.NumericalError, match="index 5"):
        tg.adam_step(g, gbuf.data_ptr())
    assert np.array_equal(g.coeffs, before)


def test_training_trajectory_golden(step_path):
    """30 fused steps (2D, order 2, zero init, paper loss, lr 1e-2) vs the reference loss curve."""
    z = load_golden("train.npz")
    g = tg.init_grid(gspec(2, z["train_res"], 2))
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    terms = []
    for b in z["train_batches"]:
        terms.append(tg.train_step(g, b, tg.LossConfig()).as_array())
    terms = np.array(terms)
    assert_close(terms[:, 0], z["train_terms"][:, 0], 1e-4, floor=1e-30, what="loss curve")
    assert_close(g.coeffs, z["train_final"], 1e-3, floor=1e-2, what="final coeffs")


def test_async_trajectory_matches_sync(step_path):
    z = load_golden("train.npz")
    g1 = tg.init_grid(gspec(2, z["train_res"], 2))
    g2 = tg.init_grid(gspec(2, z["train_res"], 2))
    for g in (g1, g2):
        g.adam_reset(tg.AdamConfig(lr=1e-2))
    sync_terms = [tg.train_step(g1, b).as_array() for b in z["train_batches"]]
    for b in z["train_batches"]:
        tg.train_step(g2, b, asynchronous=True)
    g2.sync()
    # the fused step bins points with atomics, so runs agree to rounding, not bitwise
    # (two runs: ~1e-7 per step apart; 1e-5 leaves room for the chaotic growth)
    assert_close(g2.trace(len(z["train_batches"])), np.array(sync_terms), 1e-5, floor=1e-30, what="async trace")
    assert_trajectory_close(g2.coeffs, g1.coeffs, 1e-2, len(z["train_batches"]), what="async coeffs")


def test_nonfinite_loss_aborts_and_keeps_params(step_path):
    z = load_golden("train.npz")
    g = tg.init_grid(gspec(2, z["train_res"], 2))
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    for b in z["train_batches"][:3]:
        tg.train_step(g, b)
    before = g.coeffs
    t_before = g.adam_t
    bad = z["train_batches"][3].copy()
    bad[17, 3] = np.nan  # NaN target -> non-finite loss
    with pytest.raises(tg.NumericalError, match="non-finite loss at stage 0 step 3"):
        tg.train_step(g, bad)
    assert np.array_equal(g.coeffs, before) and g.adam_t == t_before
    # async: the failing step and every later one are no-ops; sync reports it
    for b in [z["train_batches"][4], bad, z["train_batches"][5]]:
        tg.train_step(g, b, asynchronous=True)
    with pytest.raises(tg.NumericalError, match="non-finite loss"):
        g.sync()
    nan_pt = z["train_batches"][6].copy()
    nan_pt[3, 0] = np.nan
    with pytest.raises(ValueError, match="NaN coordinate"):
        tg.train_step(g, nan_pt)


def test_overlapped_binning_trajectory_and_nan_step(step_path):
    """Binning of step i+1 on the binning stream (input_ready device batches,
    pipelined host batches, mixed with stream-ordered steps) overlaps step i's
    brick kernel: same trajectory as synchronous steps, and a NaN sample is
    reported for its own step (per-bin-set NaN slot) with that step's input
    state kept."""
    import torch
    z = load_golden("train.npz")
    spec = gspec(2, z["train_res"], 2)
    batches = list(z["train_batches"])
    g1, g2 = tg.init_grid(spec), tg.init_grid(spec)
    for g in (g1, g2):
        g.adam_reset(tg.AdamConfig(lr=1e-2))
    sync_terms = [tg.train_step(g1, b).as_array() for b in batches]
    dev = [torch.from_numpy(b.astype(np.float32)).cuda() for b in batches]
    torch.cuda.synchronize()
    with pytest.raises(TypeError, match="float32"):
        tg.train_step(g2, dev[0].double())
    for i in range(len(batches)):
        if i % 3 == 0:
            tg.train_step(g2, dev[i], asynchronous=True, input_ready=True)
        elif i % 3 == 1:
            tg.train_step(g2, np.ascontiguousarray(batches[i]), asynchronous=True)  # pipelined host copy
        else:
            tg.train_step(g2, dev[i], asynchronous=True)  # ordered after the stream
    g2.sync()
    assert_close(g2.trace(len(batches)), np.array(sync_terms), 1e-5, floor=1e-30, what="overlapped trace")
    assert_trajectory_close(g2.coeffs, g1.coeffs, 1e-2, len(batches), what="overlapped coeffs")

    g3 = tg.init_grid(spec)
    g3.adam_reset(tg.AdamConfig(lr=1e-2))
    for b in dev[:2]:
        tg.train_step(g3, b)
    ref = g3.coeffs
    bad = dev[2].clone()
    bad[5, 1] = float("nan")
    torch.cuda.synchronize()
    seq = [bad, dev[3], dev[4], dev[5]]
    for b in seq:
        tg.train_step(g3, b, asynchronous=True, input_ready=True)
    with pytest.raises(ValueError, match=r"NaN coordinate \(sample 5\) at stage 0 step 2"):
        g3.sync()
    assert np.array_equal(g3.coeffs, ref) and g3.adam_t == 2
    # usable again: the remaining steps match a clean grid's
    for b in dev[3:6]:
        tg.train_step(g3, b, asynchronous=True, input_ready=True)
    g3.sync()
    assert np.all(np.isfinite(g3.coeffs))


# ---- BASELINE-size properties --------------------------------------------------------------------


def test_c2_scale_fused_gradient_vs_oracle(oracle):
    """C2 shape (128^3, order 2, 2^20 points: 50% uniform, 50% near a sphere r=0.6):
    fused gradient, loss terms and updated params vs the fp64 oracle, on a
    random (non-zero) grid so every term is active."""
    res = (128, 128, 128)
    s = ospec(3, res, 2)
    rng = np.random.default_rng(11)
    c = (0.01 * rng.standard_normal(s.V * s.K)).astype(np.float32)
    smp = tg.sample(tg.SHAPE_SPHERE, 3, 99, 1 << 20, near_frac=0.5, sigma=0.01, param0=0.6)
    g = tg.init_grid(gspec(3, res, 2))
    g.set_coeffs_f32(c)
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    t = tg.train_step(g, smp, tg.LossConfig(), export_grad=True)
    gref = np.zeros(s.V * s.K)
    c64, s64 = c.astype(np.float64), smp.astype(np.float64)
    tref = oracle.total_loss(s, c64, s64, Loss(), gref)
    assert_close(t.as_array(), tref, 1e-5, floor=1e-30, what="terms")
    mass = oracle.total_loss_mass(s, c64, s64, Loss())
    grad_close(g.grad(), gref, mass, what="C2 fused grad")
    # first Adam step: p - lr * g / (|g| + eps) (bias-corrected), fp32 state
    p1 = c.astype(np.float64) - 1e-2 * gref / (np.abs(gref) + 1e-8)
    assert_close(g.coeffs, p1, 1e-6, floor=1.0 + 0 * p1, what="params after step")


# ---- multi-GPU slab path, two slabs emulated on one device ----------------------------------------


@pytest.mark.parametrize("nslab,res,sharded,fused", [(2, (24, 20, 40), False, False), (3, (21, 18, 43), False, False),
                                                     (3, (21, 18, 43), True, False), (3, (21, 18, 43), True, True),
                                                     (2, (24, 20, 40), False, True)])
def test_slab_two_on_one_gpu_matches_full_grid(nslab, res, sharded, fused):
    """z-slab grids driven like ranks (sum of partials, commit, halo exchange
    by device copies) reproduce the single-grid fused trajectory; with three
    slabs the middle one exchanges both halo planes; sharded: each slab reads
    only its own points (slab_point_mask) with the global batch size; fused:
    no exchange — the brick kernel writes the boundary planes into the
    neighbours' halo planes (tgcu_slab_set_peer_planes, the same-device form
    of the NVLink peer stores), checked first by the peer probe."""
    from paper_2402_14415_b200.slab import SlabGrid, brick_layers, device_view, slab_point_mask, slab_ranges
    spec = tg.GridSpec(dim=3, resolution=res, order=2)
    init = tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.02, seed=3)
    cfg = tg.LossConfig()
    full = tg.init_grid(spec, init)
    full.adam_reset(tg.AdamConfig(lr=1e-2))
    ranges = slab_ranges(brick_layers(res[2]), nslab)
    slabs = [SlabGrid(spec, lo, hi, init) for lo, hi in ranges]
    for sg in slabs:
        sg.adam_reset(tg.AdamConfig(lr=1e-2))
    K = spec.coeffs_per_vertex()
    plane = res[0] * res[1] * K
    c_full = full.coeffs
    for sg in slabs:  # identical initial values, halo planes included
        assert np.array_equal(sg.coeffs(), c_full[sg.z_store_lo * plane:(sg.z_store_lo + sg.z_store_n) * plane])
    if fused:
        slots = [sg.halo_slots() for sg in slabs]  # ((lo0, lo1), (hi0, hi1))
        for r, sg in enumerate(slabs):
            dst_lo = slots[r - 1][1] if r > 0 else (0, 0)          # lower neighbour's upper halo
            dst_hi = slots[r + 1][0] if r < nslab - 1 else (0, 0)  # upper neighbour's lower halo
            sg.set_peer_planes(dst_lo, dst_hi)
        for sg in slabs:
            sg.peer_probe(0)
        assert all(sg.peer_probe(1) for sg in slabs)
    for step in range(6):
        b = tg.sample(tg.SHAPE_SPHERE, 3, 500 + step, 20000, near_frac=0.5, sigma=0.01, param0=0.6)
        tf = tg.train_step(full, b, cfg).as_array()
        if sharded:
            parts = [sg.begin(np.ascontiguousarray(b[slab_point_mask(spec, b.astype(np.float64), *rg)]), cfg,
                              n_global=len(b)) for sg, rg in zip(slabs, ranges)]
        else:
            parts = [sg.begin(b, cfg) for sg in slabs]
        views = [device_view(p, 5, "<f8") for p in parts]
        tot = views[0].clone()
        for v in views[1:]:
            tot += v
        for v in views:
            v.copy_(tot)
        terms = [sg.finish(p).as_array() for sg, p in zip(slabs, parts)]
        halos = [sg.halo() for sg in slabs]
        for r in range(nslab - 1 if not fused else 0):  # slab r's top owned plane <-> slab r+1's bottom owned plane
            lo, hi = halos[r], halos[r + 1]
            pf = lo[4]
            device_view(hi[2], pf).copy_(device_view(lo[1], pf))
            device_view(lo[3], pf).copy_(device_view(hi[0], pf))
        for t in terms:
            assert_close(t, tf, 1e-5, floor=1e-30, what=f"slab terms step {step}")
    owned = np.concatenate([sg.owned_coeffs() for sg in slabs])
    assert_trajectory_close(owned, full.coeffs, 1e-2, 6, what="slab coefficients")
    # the halo planes hold exactly the neighbours' committed boundary planes
    cs = [sg.coeffs() for sg in slabs]
    for r in range(1, nslab):
        lo_sg, hi_sg = slabs[r - 1], slabs[r]
        z = hi_sg.z_own_lo - 1  # lower slab's top owned plane = upper slab's lower halo
        a = (z - lo_sg.z_store_lo) * plane
        assert np.array_equal(cs[r][:plane], cs[r - 1][a:a + plane])
        z = lo_sg.z_own_hi      # upper slab's bottom owned plane = lower slab's upper halo
        a = (z - hi_sg.z_store_lo) * plane
        b = (z - lo_sg.z_store_lo) * plane
        assert np.array_equal(cs[r - 1][b:b + plane], cs[r][a:a + plane])


def test_slab_with_no_local_points_matches_full_grid():
    """A slab whose cells hold none of the batch's points (all points below
    it) still takes its TV + Adam step: n = 0 local points with the global
    batch size, against the full-grid trajectory."""
    from paper_2402_14415_b200.slab import SlabGrid, brick_layers, device_view, slab_point_mask, slab_ranges
    res = (24, 20, 40)
    spec = tg.GridSpec(dim=3, resolution=res, order=2)
    init = tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.02, seed=5)
    cfg = tg.LossConfig()
    full = tg.init_grid(spec, init)
    full.adam_reset(tg.AdamConfig(lr=1e-2))
    ranges = slab_ranges(brick_layers(res[2]), 2)
    slabs = [SlabGrid(spec, lo, hi, init) for lo, hi in ranges]
    for sg in slabs:
        sg.adam_reset(tg.AdamConfig(lr=1e-2))
    K = spec.coeffs_per_vertex()
    plane = res[0] * res[1] * K
    for step in range(4):
        b = tg.sample(tg.SHAPE_SPHERE, 3, 700 + step, 5000, near_frac=0.0)
        b[:, 2] = -1.0 + (b[:, 2] + 1.0) * 0.3   # z in [-1, -0.4]: only the lower slab's cells
        tf = tg.train_step(full, b, cfg).as_array()
        local = [np.ascontiguousarray(b[slab_point_mask(spec, b.astype(np.float64), *rg)]) for rg in ranges]
        assert len(local[1]) == 0
        parts = [sg.begin(lp, cfg, n_global=len(b)) for sg, lp in zip(slabs, local)]
        views = [device_view(p, 5, "<f8") for p in parts]
        tot = views[0].clone() + views[1]
        for v in views:
            v.copy_(tot)
        terms = [sg.finish(p).as_array() for sg, p in zip(slabs, parts)]
        lo, hi = slabs[0].halo(), slabs[1].halo()
        device_view(hi[2], lo[4]).copy_(device_view(lo[1], lo[4]))
        device_view(lo[3], lo[4]).copy_(device_view(hi[0], lo[4]))
        for t in terms:
            assert_close(t, tf, 1e-5, floor=1e-30, what=f"terms step {step}")
    owned = np.concatenate([sg.owned_coeffs() for sg in slabs])
    assert_trajectory_close(owned, full.coeffs, 1e-2, 4, what="slab coefficients")


@pytest.mark.parametrize("dim", [2, 3])
def test_fused_step_fresh_uniform_eikonal(oracle, reference, dim, step_path):
    """LossConfig(eikonal_point_source=FreshUniform): the fused step takes the
    reconstruction term on the batch and the eikonal term on |batch| points
    drawn from the step's Rng (reference order). Checked against the
    reference's recon-only total_loss + eikonal_loss on the same fp32 points
    (test_oracle_cpu pins that decomposition to the reference's FreshUniform
    code): terms, full gradient, first Adam update; the same Rng stream is
    consumed; no rng is an error."""
    rng = np.random.default_rng(60 + dim)
    res = (21, 18, 17) if dim == 3 else (40, 33)
    s = ospec(dim, res, 2)
    c = (0.05 * rng.standard_normal(s.V * s.K)).astype(np.float32).astype(np.float64)
    n = 3000
    pts = rng.uniform(-1.0, 1.0, (n, 3)).astype(np.float32)
    if dim == 2:
        pts[:, 2] = 0.0
    smp = np.concatenate([pts, rng.uniform(-0.4, 0.4, (n, 1)).astype(np.float32)], 1).astype(np.float64)
    cfg = tg.LossConfig(lambda1=1e-2, lambda2=1e-3, eikonal_point_source=tg.EikonalPointSource.FreshUniform)
    g = tg.init_grid(gspec(dim, res, 2))
    g.coeffs = c
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    with pytest.raises(ValueError, match="need an rng"):
        tg.train_step(g, smp, cfg)
    seed = 77
    t = tg.train_step(g, smp, cfg, export_grad=True, rng=tg.Rng(seed))
    eik_pts = tg.Rng(seed).uniform_in_box(dim, [-1.0] * 3, [1.0] * 3, n).astype(np.float32).astype(np.float64)
    gref = np.zeros(s.V * s.K)
    t_fit = reference.total_loss(s, c, smp, Loss(lambda1=0.0, lambda2=cfg.lambda2), gref)
    eik = reference.eikonal_loss(s, c, eik_pts, cfg.lambda1, gref)
    tref = np.array([t_fit[1] + cfg.lambda1 * eik + cfg.lambda2 * t_fit[3], t_fit[1], eik, t_fit[3]])
    assert_close(t.as_array(), tref, 1e-6, floor=1e-30, what="fresh-uniform terms")
    eik_smp = np.concatenate([eik_pts, np.zeros((n, 1))], 1)
    mass = (oracle.total_loss_mass(s, c, smp, Loss(lambda1=0.0, lambda2=cfg.lambda2))
            + oracle.total_loss_mass(s, c, eik_smp, Loss(lambda1=cfg.lambda1, lambda2=0.0, use_tv=False)))
    grad_close(g.grad(), gref, mass, what="fresh-uniform grad")
    p1 = c - 1e-2 * gref / (np.abs(gref) + 1e-8)
    ok = np.abs(gref) > 1e-3 * (np.abs(gref).max() + 1e-30)
    assert_close(g.coeffs[ok], p1[ok], 1e-6, floor=1.0, what="params after step")


@pytest.mark.parametrize("dim", [2, 3])
def test_recon_and_eikonal_loss_standalone(oracle, reference, dim):
    """recon_loss / eikonal_loss (sdf_loss.cpp:130-153) with their scale on the
    gradient, against the reference (values 1e-6, gradients within the
    accumulation-order bound), and the errors for empty inputs."""
    rng = np.random.default_rng(80 + dim)
    res = (19, 16, 14) if dim == 3 else (30, 27)
    s = ospec(dim, res, 2)
    c = (0.1 * rng.standard_normal(s.V * s.K)).astype(np.float32).astype(np.float64)
    n = 4000
    pts = rng.uniform(-1.0, 1.0, (n, 3)).astype(np.float32)
    if dim == 2:
        pts[:, 2] = 0.0
    smp = np.concatenate([pts, rng.uniform(-0.4, 0.4, (n, 1)).astype(np.float32)], 1).astype(np.float64)
    g = tg.init_grid(gspec(dim, res, 2))
    g.coeffs = c
    cfg = tg.LossConfig()
    g.zero_grad()
    v = tg.recon_loss(g, smp, cfg, scale=2.5)
    gref = np.zeros(s.V * s.K)
    tref = reference.total_loss(s, c, smp, Loss(lambda1=0.0, use_tv=False), gref)
    assert_close(v, tref[1], 1e-6, floor=1e-30, what="recon_loss")
    mass = oracle.total_loss_mass(s, c, smp, Loss(lambda1=0.0, use_tv=False))
    grad_close(g.grad(), 2.5 * gref, 2.5 * mass, what="recon_loss grad")
    g.zero_grad()
    e = tg.eikonal_loss(g, pts.astype(np.float64), scale=0.3)
    gref = np.zeros(s.V * s.K)
    eref = reference.eikonal_loss(s, c, pts.astype(np.float64), 0.3, gref)
    assert_close(e, eref, 1e-6, floor=1e-30, what="eikonal_loss")
    emass = oracle.total_loss_mass(s, c, np.concatenate([pts, np.zeros((n, 1))], 1).astype(np.float64),
                                   Loss(lambda1=0.3, use_tv=False))
    grad_close(g.grad(), gref, emass, what="eikonal_loss grad")
    with pytest.raises(ValueError, match="recon_loss: empty batch"):
        tg.recon_loss(g, np.zeros((0, 4)), cfg)
    with pytest.raises(ValueError, match="eikonal_loss: empty point set"):
        tg.eikonal_loss(g, np.zeros((0, 3)))


def test_pipelined_host_steps_match_device_steps(step_path):
    """TGCU_HOST|TGCU_ASYNC (copy-stream pipelined host input) gives the same
    trajectory as device-resident async steps; host arrays alternate slots."""
    import torch
    spec = tg.GridSpec(dim=3, resolution=(24, 20, 28), order=2)
    batches = [tg.sample(tg.SHAPE_SPHERE, 3, 70 + i, 20000, near_frac=0.5, sigma=0.01, param0=0.6) for i in range(6)]
    pinned = [torch.from_numpy(b).pin_memory() for b in batches]
    g1 = tg.init_grid(spec)
    g2 = tg.init_grid(spec)
    for g in (g1, g2):
        g.adam_reset(tg.AdamConfig(lr=1e-2))
    for b in batches:
        tg.train_step(g1, torch.from_numpy(b).cuda(), asynchronous=True)
    for p in pinned:
        tg.train_step(g2, p.numpy(), asynchronous=True)
    t2 = g2.sync()
    t1 = g1.sync()
    assert_close(g2.trace(6), g1.trace(6), 1e-5, floor=1e-30, what="pipelined trace")
    assert abs(t2.total - t1.total) <= 1e-5 * abs(t1.total)
    assert_trajectory_close(g2.coeffs, g1.coeffs, 1e-2, 6, what="pipelined coeffs")


@pytest.mark.parametrize("order", [1, 2])
def test_binned_unsorted_query_matches_direct(oracle, order):
    """Unsorted batches of >= 2^18 points go through the brick-binned query
    (counting sort by brick, smem tiles, values written to the caller's slots):
    bit-identical to the direct-gather kernel (batches below the threshold),
    NaN points answered in place, out-of-domain points clamped."""
    import torch
    rng = np.random.default_rng(40 + order)
    res = (70, 66, 61)
    s = ospec(3, res, order)
    c = (0.1 * rng.standard_normal(s.V * s.K)).astype(np.float32)
    g = tg.init_grid(gspec(3, res, order))
    g.set_coeffs_f32(c)
    n = (1 << 18) + 12345
    pts = rng.uniform(-1.05, 1.05, (n, 3)).astype(np.float32)
    dp = torch.from_numpy(pts).cuda()
    vb, gb = tg.eval_with_spatial_gradient(g, dp)  # binned
    v_only = tg.eval_device(g, dp, torch.empty(n, dtype=torch.float32, device="cuda"))
    parts_v, parts_g = [], []
    for a in range(0, n, 100000):  # direct kernel (below the threshold)
        v, gr = tg.eval_with_spatial_gradient(g, dp[a:a + 100000])
        parts_v.append(v)
        parts_g.append(gr)
    torch.cuda.synchronize()
    assert torch.equal(vb, torch.cat(parts_v)) and torch.equal(gb, torch.cat(parts_g))
    assert torch.equal(v_only, vb)
    sub = rng.choice(n, 5000, replace=False)
    ref = oracle.eval(s, c.astype(np.float64), pts[sub].astype(np.float64))
    assert_close(vb.cpu().numpy()[sub], ref, 1e-6, what="binned value")
    # NaN points: NaN output, ValueError naming the first one
    pts[[7, 100003]] = np.nan
    with pytest.raises(ValueError, match="point 7"):
        tg.eval(g, pts)


@pytest.mark.parametrize("order,origin,extent", [(1, (-1.0, -1.0, -1.0), (2.0, 2.0, 2.0)),
                                                (2, (-1.0, -1.0, -1.0), (2.0, 2.0, 2.0)),
                                                (2, (100.0, -37.5, 3.0), (1.5, 2.0, 0.75))])
def test_binned_query_gather_large(oracle, order, origin, extent):
    """The binned query writes each value at its record's pass-1 position and
    gathers them back in input order (k_qp_unpart; Morton-order brick walk):
    2^22 + 777 points, among them NaN points and 2^18 points within
    0 .. 1e-3 cells of brick planes and of the domain edges (where the
    partition's fp32 brick code hands over to the exact fp64 rule), on the
    default domain and on one far from the origin; values and spatial
    gradients identical to the direct-gather kernel on slices below the
    binning threshold (a point binned into the wrong brick would read the
    wrong tile), NaN slots left NaN by the partition, a subset against the
    oracle."""
    import torch
    rng = np.random.default_rng(60 + order)
    res = (90, 81, 77)
    s = Spec(dim=3, res=res, order=order, origin=origin, extent=extent)
    c = (0.1 * rng.standard_normal(s.V * s.K)).astype(np.float32)
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=res, origin=origin, extent=extent, order=order))
    g.set_coeffs_f32(c)
    n = (1 << 22) + 777
    dp = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    tg.sample_uniform_device(3, 77 + order, dp)
    o, e = np.array(origin), np.array(extent)
    near = (1 << 18)
    h = e / (np.array(res) - 1)
    cells = rng.integers(0, 12, (near, 3)) * 8  # brick planes (8-cell bricks)
    cells = np.where(rng.random((near, 3)) < 0.2, np.array(res) - 1, cells)  # the far domain edge
    off = rng.choice([0.0, 1e-7, -1e-7, 1e-6, -1e-6, 1e-5, -1e-5, 1e-4, -1e-4, 1e-3, -1e-3], (near, 3))
    pl = o + (cells + off) * h
    keep = rng.random((near, 3)) < 0.5  # the other axes anywhere
    pl = np.where(keep, pl, o + rng.random((near, 3)) * e)
    dp[:near] = torch.from_numpy(pl.astype(np.float32)).cuda()
    dp[near:] = dp[near:] * torch.tensor(e / 2, dtype=torch.float32, device="cuda") + \
        torch.tensor(o + e / 2, dtype=torch.float32, device="cuda")
    bad = torch.tensor([near + 3, 1 << 20, n - 1], device="cuda")
    dp[bad, 1] = float("nan")
    v_only = tg.eval_device(g, dp, torch.empty(n, dtype=torch.float32, device="cuda"), asynchronous=True)
    vb = torch.empty(n, dtype=torch.float32, device="cuda")
    gb = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    tg.eval_device(g, dp, vb, gb, asynchronous=True)
    vd = torch.empty_like(vb)
    gd = torch.empty_like(gb)
    step = (1 << 18) - 1
    for a in range(0, n, step):  # the direct kernel (below the threshold)
        tg.eval_device(g, dp[a:a + step], vd[a:a + step], gd[a:a + step], asynchronous=True)
    torch.cuda.synchronize()
    with pytest.raises(ValueError, match="NaN coordinate"):  # reported by the next checked call
        tg.eval_device(g, dp[:near + 8], torch.empty(near + 8, dtype=torch.float32, device="cuda"))
    g.close()
    assert torch.isnan(v_only[bad]).all() and torch.isnan(gb[bad]).all()
    assert int(torch.isnan(v_only).sum()) == 3
    nn = lambda t: torch.nan_to_num(t, 7.0)  # noqa: E731
    assert torch.equal(nn(v_only), nn(vb)) and torch.equal(nn(vb), nn(vd)) and torch.equal(nn(gb), nn(gd))
    sub = np.concatenate([rng.choice(near, 2000, replace=False), rng.choice(n, 2000, replace=False)])
    pts = dp[torch.from_numpy(sub).cuda()].cpu().numpy().astype(np.float64)
    ok = ~np.isnan(pts).any(axis=1)
    ref = oracle.eval(s, c.astype(np.float64), pts[ok])
    assert_close(v_only.cpu().numpy()[sub][ok], ref, 1e-6, what="binned value")


@pytest.mark.parametrize("case", ["one_point", "one_brick", "all_nan", "threshold", "corner_edges"])
def test_binned_query_skewed_inputs(case):
    """The binned query's partition, brick kernel and reverse gather on
    degenerate batches: every point identical, all points inside one brick,
    all points NaN, exactly the binning threshold, every point on a domain
    corner / edge; values equal the direct-gather kernel's."""
    import torch
    rng = np.random.default_rng(7)
    res = (70, 66, 61)
    g = tg.init_grid(gspec(3, res, 2))
    s = ospec(3, res, 2)
    g.set_coeffs_f32((0.1 * rng.standard_normal(s.V * s.K)).astype(np.float32))
    n = (1 << 18) + 3
    if case == "one_point":
        p = np.tile(np.array([[0.123, -0.456, 0.789]], np.float32), (n, 1))
    elif case == "one_brick":
        p = (rng.random((n, 3)) * 7.9 * 2.0 / 69.0 - 1.0).astype(np.float32)  # cells [0, 8) on each axis
    elif case == "all_nan":
        p = np.full((n, 3), np.nan, np.float32)
    elif case == "threshold":
        n = 1 << 18
        p = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    else:
        p = rng.choice([-1.0, 1.0, -1.0000001, 1.0000001, 0.0], (n, 3)).astype(np.float32)
    dp = torch.from_numpy(p).cuda()
    vb = tg.eval_device(g, dp, torch.empty(n, dtype=torch.float32, device="cuda"), asynchronous=True)
    vd = torch.empty(n, dtype=torch.float32, device="cuda")
    step = (1 << 18) - 1
    for a in range(0, n, step):
        tg.eval_device(g, dp[a:a + step], vd[a:a + step], asynchronous=True)
    torch.cuda.synchronize()
    if case == "all_nan":
        assert torch.isnan(vb).all() and torch.isnan(vd).all()
        with pytest.raises(ValueError, match="NaN coordinate"):
            tg.eval_device(g, dp[:4], torch.empty(4, dtype=torch.float32, device="cuda"))
    else:
        assert torch.equal(vb, vd)
        # the sort (partition + cell pass) and the brick-sorted kernel
        spts = torch.empty_like(dp)
        perm = torch.empty(n, dtype=torch.int64, device="cuda")
        offs = torch.empty(tg.query_brick_codes(g) + 1, dtype=torch.int64, device="cuda")
        tg.sort_points(g, dp, spts, perm, offs)
        vs = tg.eval_sorted(g, spts, offs)
        torch.cuda.synchronize()
        assert torch.equal(spts, dp[perm]) and torch.equal(vs, vd[perm])
        assert int(offs[-1]) == n and bool((offs[1:] >= offs[:-1]).all())
    g.close()


@pytest.mark.parametrize("dim,res", [(2, (37, 29)), (3, (19, 12, 26))])
@pytest.mark.parametrize("order", [0, 1, 2])
@pytest.mark.parametrize("name,cfg", [("paper", tg.LossConfig()), ("recon", tg.LossConfig(lambda1=0.0, use_tv=False)),
                                      ("dw", tg.LossConfig(differentiate_weight=True, lambda1=3e-3))])
def test_fused_step_all_orders_vs_oracle(oracle, dim, res, order, name, cfg, step_path):
    """Fused step (binning, brick kernel with edge bricks, finalize) for every
    order and dimension: loss terms, full gradient and the first Adam update
    against the fp64 oracle; resolutions not multiples of the brick edge."""
    rng = np.random.default_rng(1000 + 10 * order + dim)
    r3 = tuple(res) + ((1,) if dim == 2 else ())
    s = ospec(dim, r3, order)
    c = (0.2 * rng.standard_normal(s.V * s.K)).astype(np.float32).astype(np.float64)
    n = 5000
    pts = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    pts[:50] = np.float32(1.0)            # max boundary -> last cell, local 1 (several bricks' boundary)
    pts[50:100, 0] = np.float32(-1.0)
    if dim == 2:
        pts[:, 2] = 0.0
    gt = (np.linalg.norm(pts[:, :dim], axis=1) - 0.5).astype(np.float32)
    smp = np.concatenate([pts, gt[:, None]], 1).astype(np.float64)
    loss = Loss(cfg.lambda1, cfg.lambda2, cfg.k, cfg.use_weighting, cfg.use_tv, cfg.differentiate_weight)
    gref = np.zeros(s.V * s.K)
    tref = oracle.total_loss(s, c, smp, loss, gref)
    mass = oracle.total_loss_mass(s, c, smp, loss)
    g = tg.init_grid(gspec(dim, r3, order))
    g.coeffs = c
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    t = tg.train_step(g, smp, cfg, export_grad=True)
    assert_close(t.as_array(), tref, 1e-6, floor=1e-30, what="fused terms")
    grad_close(g.grad(), gref, mass, what="fused grad")
    p1 = c - 1e-2 * gref / (np.abs(gref) + 1e-8)  # first Adam step (bias-corrected)
    ok = np.abs(gref) > 1e-3 * (np.abs(gref).max() + 1e-30)  # away from sign-ambiguous tiny gradients
    assert_close(g.coeffs[ok], p1[ok], 1e-6, floor=1.0, what="params after step")


@pytest.mark.parametrize("case", ["many_points", "many_bricks"])
def test_global_binning_path_vs_oracle(oracle, case):
    """Batches of more than 2^21 points, or grids of more than 16384 bricks
    (C3 / C5 scale), bin with global atomics instead of the privatized
    shared-memory histograms: same loss terms and gradient as the oracle."""
    rng = np.random.default_rng(77)
    if case == "many_points":
        res, order, n = (48, 44, 40), 2, 3 * (1 << 20)
    else:
        res, order, n = (256, 256, 256), 1, 200000   # 32^3 = 32768 bricks
    s = ospec(3, res, order)
    c = (0.05 * rng.standard_normal(s.V * s.K)).astype(np.float32).astype(np.float64)
    smp = tg.sample(tg.SHAPE_SPHERE, 3, 321, n, near_frac=0.5, sigma=0.01, param0=0.6).astype(np.float64)
    cfg = tg.LossConfig()
    gref = np.zeros(s.V * s.K)
    tref = oracle.total_loss(s, c, smp, Loss(), gref)
    mass = oracle.total_loss_mass(s, c, smp, Loss())
    g = tg.init_grid(gspec(3, res, order))
    g.set_step_path(tg.TaylorGrid.STEP_BRICK)  # the binning under test (auto would take the small path)
    g.coeffs = c
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    t = tg.train_step(g, smp, cfg, export_grad=True)
    assert_close(t.as_array(), tref, 1e-6, floor=1e-30, what="terms")
    grad_close(g.grad(), gref, mass, what="grad")


def test_empty_and_degenerate_inputs():
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=(9, 9, 9), order=2))
    g.adam_reset(tg.AdamConfig())
    assert tg.eval(g, np.zeros((0, 3))).shape == (0,)
    with pytest.raises(ValueError, match="empty batch"):
        tg.train_step(g, np.zeros((0, 4)))
    assert g.adam_t == 0
    # a batch whose points all sit in one cell / on one vertex
    one = np.tile(np.array([[0.125, -0.25, 0.5, 0.1]], np.float32), (4096, 1))
    t = tg.train_step(g, one)
    assert np.isfinite(t.total) and g.adam_t == 1


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("TGCU_RANDOM_CASES", "300"))))
def test_fused_step_random_configs(oracle, seed, step_path):
    """Seeded random sweep: dimension, order, resolution (2..41 per axis, so
    single-cell axes and partial bricks), batch size (1..20000, below and
    above the 512-point chunk), loss switches and learning rate — fused step
    vs the fp64 oracle (terms, gradient, first Adam update)."""
    rng = np.random.default_rng(9000 + seed)
    dim = int(rng.choice([2, 3]))
    order = int(rng.integers(0, 3))
    res = tuple(int(r) for r in rng.integers(2, 42, dim)) + ((1,) if dim == 2 else ())
    n = int(rng.choice([1, 7, 513, int(rng.integers(1, 20001))]))
    cfg = tg.LossConfig(lambda1=float(rng.choice([0.0, 1e-4, 1e-2])), lambda2=float(rng.choice([0.0, 2e-5, 1e-3])),
                        k=float(rng.choice([5.0, 50.0])), use_weighting=bool(rng.integers(0, 2)),
                        use_tv=bool(rng.integers(0, 2)), differentiate_weight=bool(rng.integers(0, 2)))
    lr = float(rng.choice([1e-3, 1e-2]))
    s = ospec(dim, res, order)
    c = (0.2 * rng.standard_normal(s.V * s.K)).astype(np.float32).astype(np.float64)
    pts = rng.uniform(-1.1, 1.1, (n, 3)).astype(np.float32)
    if dim == 2:
        pts[:, 2] = 0.0
    gt = rng.uniform(-0.5, 0.5, n).astype(np.float32)
    smp = np.concatenate([pts, gt[:, None]], 1).astype(np.float64)
    loss = Loss(cfg.lambda1, cfg.lambda2, cfg.k, cfg.use_weighting, cfg.use_tv, cfg.differentiate_weight)
    gref = np.zeros(s.V * s.K)
    tref = oracle.total_loss(s, c, smp, loss, gref)
    mass = oracle.total_loss_mass(s, c, smp, loss)
    g = tg.init_grid(gspec(dim, res, order))
    g.coeffs = c
    g.adam_reset(tg.AdamConfig(lr=lr))
    t = tg.train_step(g, smp, cfg, export_grad=True)
    # loss terms 1e-5: a batch of one point gets no averaging, and its eikonal
    # term (|grad f| - 1)^2 carries the fp32 forward error of grad f directly
    assert_close(t.as_array(), tref, 1e-5, floor=1e-30, what=f"terms {dim}D o{order} {res} n={n} {cfg}")
    grad_close(g.grad(), gref, mass, what=f"grad {dim}D o{order} {res} n={n}")
    p1 = c - lr * gref / (np.abs(gref) + 1e-8)
    ok = np.abs(gref) > 1e-3 * (np.abs(gref).max() + 1e-30)
    assert_close(g.coeffs[ok], p1[ok], 1e-6, floor=1.0, what="params after step")


def test_wide_2d_grid_brick_codes(oracle):
    """A 2D grid with 513 bricks along x (res_x 8200 > 512 bricks of 16
    vertices; the binning's brick code gives each axis as many bits as the
    grid needs): fused step vs the oracle, points in every brick column."""
    res = (8200, 20)
    s = ospec(2, res, 2)
    rng = np.random.default_rng(31)
    c = (0.05 * rng.standard_normal(s.V * s.K)).astype(np.float32).astype(np.float64)
    n = 60000
    pts = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    pts[:2000, 0] = np.linspace(0.999, 1.0, 2000, dtype=np.float32)  # the last brick columns
    pts[:, 2] = 0.0
    gt = (np.linalg.norm(pts[:, :2], axis=1) - 0.5).astype(np.float32)
    smp = np.concatenate([pts, gt[:, None]], 1).astype(np.float64)
    gref = np.zeros(s.V * s.K)
    tref = oracle.total_loss(s, c, smp, Loss(), gref)
    mass = oracle.total_loss_mass(s, c, smp, Loss())
    g = tg.init_grid(gspec(2, res, 2))
    g.set_step_path(tg.TaylorGrid.STEP_BRICK)  # the brick codes under test (auto would take the small path)
    g.coeffs = c
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    t = tg.train_step(g, smp, tg.LossConfig(), export_grad=True)
    assert_close(t.as_array(), tref, 1e-6, floor=1e-30, what="terms")
    grad_close(g.grad(), gref, mass, what="wide 2D grad")
