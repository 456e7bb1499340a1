"""GPU parity of the SURVEY §8f rows through the C ABI (libtgcu.so):

* upsample / multilinear_resample: bit-exact against the oracle fed the same
  fp32 coefficients (fp64 weights + accumulation in the reference's order,
  one rounding to fp32), and against the reference golden (|d| within one
  fp32 rounding of the fp64 reference values);
* sample_grid_field: |d| <= 1e-6 * max(1, |ref|) against the reference lattice;
* run_schedule (progressive, per-stage Adam reset): loss curve <= 1e-4 rel
  against the reference run_schedule golden; error context "stage s step k";
* fit_sdf with the reference batch stream: loss curve <= 1e-4 rel against the
  reference fit_sdf golden, same holdout split;
* .tgrid: byte-identical files to the reference's save_tgrid, loading the
  reference's files, and the reference's IngestError messages.
"""
import numpy as np
import pytest

import paper_2402_14415_b200 as tg
from conftest import load_golden
from oracle.pyoracle import Loss, Spec, tgrid_bytes
from paper_2402_14415_b200.schedule import (BatchProblem, FitOptions, Schedule, Stage, TrainProblem, fit_sdf,
                                            run_schedule)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def z():
    return load_golden("stages.npz")


def gspec(dim, res, order, **kw):
    res = tuple(int(r) for r in res)
    return tg.GridSpec(dim=dim, resolution=res[:dim], order=order, **kw)


def grid_from(dim, res, order, coeffs):
    g = tg.init_grid(gspec(dim, res, order))
    g.coeffs = coeffs
    return g


def assert_close(got, ref, rel, floor=1.0, what=""):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    tol = rel * np.maximum(np.abs(ref), floor)
    bad = np.abs(got - ref) > tol
    assert not bad.any(), (f"{what}: {bad.sum()}/{bad.size} beyond tolerance, worst |d|="
                           f"{np.max(np.abs(got - ref)):.3e} at {np.argmax(np.abs(got - ref) - tol)}")


@pytest.mark.parametrize("case", ["d3o2", "d3o1", "d3o0same", "d3o2odd", "d2o2"])
def test_upsample_bit_exact(oracle, z, case):
    dim, order = (int(x) for x in z[f"up_{case}_meta"])
    res, nres = z[f"up_{case}_res"], z[f"up_{case}_newres"]
    c = z[f"up_{case}_coeffs"]  # fp32-representable
    g = grid_from(dim, res, order, c)
    up = tg.upsample(g, nres)
    assert tuple(up.spec.resolution[:dim]) == tuple(int(r) for r in nres[:dim])
    got = up.coeffs_f32()
    s = Spec(dim=dim, res=tuple(int(r) for r in res), order=order)
    want = oracle.resample(s, c, s.K, nres).astype(np.float32)
    assert np.array_equal(got, want)
    assert np.array_equal(got, z[f"up_{case}_out"].astype(np.float32))  # reference fp64 -> one fp32 rounding
    # the source grid is untouched and a fresh optimizer starts on the new grid
    assert np.array_equal(g.coeffs, c)
    up.adam_reset(tg.AdamConfig())
    assert up.adam_t == 0


def test_multilinear_resample_channels(oracle):
    rng = np.random.default_rng(3)
    s = Spec(dim=3, res=(6, 5, 4), order=0)
    data = rng.normal(size=s.V * 3).astype(np.float32)
    got = tg.multilinear_resample(tg.GridSpec(dim=3, resolution=(6, 5, 4), order=0), data, 3, (13, 9, 10))
    want = oracle.resample(s, data.astype(np.float64), 3, (13, 9, 10)).astype(np.float32)
    assert np.array_equal(got, want)
    with pytest.raises(ValueError, match="data size mismatch"):
        tg.multilinear_resample(tg.GridSpec(dim=3, resolution=(6, 5, 4), order=0), data[:-1], 3, (13, 9, 10))


def test_upsample_errors():
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=(8, 8, 8), order=2))
    with pytest.raises(ValueError, match=r"resolution may not shrink \(axis 1\)"):
        tg.upsample(g, (8, 7, 8))
    other = tg.init_grid(tg.GridSpec(dim=3, resolution=(9, 9, 9), order=1))
    rc = tg.lib().tgcu_grid_upsample(g.handle, other.handle, 0, None)
    assert rc == 1 and b"dim and order" in tg.lib().tgcu_last_error()


def test_upsample_large_matches_oracle(oracle):
    """Bigger random grid, non-integer ratio, C2-like order 2."""
    rng = np.random.default_rng(9)
    s = Spec(dim=3, res=(33, 17, 21), order=2)
    c = rng.normal(0, 0.2, s.V * s.K).astype(np.float32).astype(np.float64)
    g = grid_from(3, s.res, 2, c)
    got = tg.upsample(g, (64, 50, 41)).coeffs_f32()
    assert np.array_equal(got, oracle.resample(s, c, s.K, (64, 50, 41)).astype(np.float32))


@pytest.mark.parametrize("case", ["d3o2", "d3o1", "d2o2"])
def test_sample_grid_field_golden(oracle, z, case):
    dim, order = (int(x) for x in z[f"lat_{case}_meta"])
    g = grid_from(dim, z[f"lat_{case}_res"], order, z[f"lat_{case}_coeffs"])
    lat = tuple(int(x) for x in z[f"lat_{case}_lattice"])
    if dim == 3:
        f = tg.sample_grid_field(g, lat)
        assert f.res == lat and f.values.size == np.prod(lat)
    else:
        f = tg.sample_grid_field2(g, lat[0], lat[1])
    assert_close(f.values, z[f"lat_{case}_vals"], 1e-6, what="lattice values")


@pytest.mark.parametrize("dim,res,order,lat", [
    (3, (40, 33, 29), 2, (97, 64, 51)),     # dense: brick tiles
    (3, (17, 26, 12), 1, (120, 7, 60)),     # dense, one thin axis
    (3, (50, 41, 37), 2, (9, 13, 6)),       # sparse: a thread per lattice point
    (3, (33, 33, 33), 2, (33, 33, 33)),     # lattice on the vertices
    (2, (70, 45), 2, (300, 211)),           # 2D dense
    (2, (64, 64), 1, (5, 7)),               # 2D sparse
])
def test_sample_grid_field_brick_and_row_paths(oracle, dim, res, order, lat):
    """Both lattice kernels (brick tiles for dense lattices, a thread per value
    for sparse ones) against the oracle's sample_lattice."""
    rng = np.random.default_rng(sum(res) + order)
    s = Spec(dim=dim, res=res, order=order)
    c = rng.normal(0, 0.2, s.V * s.K).astype(np.float32).astype(np.float64)
    g = grid_from(dim, s.res, order, c)
    if dim == 3:
        got = tg.sample_grid_field(g, lat).values
    else:
        got = tg.sample_grid_field2(g, lat[0], lat[1]).values
    assert_close(got, oracle.sample_lattice(s, c, lat), 1e-6, what="lattice values")


def test_sample_grid_field_device_and_errors(oracle):
    import torch
    rng = np.random.default_rng(5)
    s = Spec(dim=3, res=(40, 33, 29), order=2)
    c = rng.normal(0, 0.2, s.V * s.K).astype(np.float32).astype(np.float64)
    g = grid_from(3, s.res, 2, c)
    lat = (97, 64, 51)
    out = torch.empty(int(np.prod(lat)), dtype=torch.float32, device="cuda")
    tg.sample_grid_field(g, lat, out=out)
    torch.cuda.synchronize()
    assert_close(out.cpu().numpy(), oracle.sample_lattice(s, c, lat), 1e-6, what="device lattice")
    with pytest.raises(ValueError, match="resolution must be >= 2"):
        tg.sample_grid_field(g, (1, 4, 4))
    g2 = tg.init_grid(tg.GridSpec(dim=2, resolution=(8, 8), order=2))
    with pytest.raises(ValueError, match="needs a 3D grid"):
        tg.sample_grid_field(g2, (4, 4, 4))


def _golden_stages(z):
    return Schedule([Stage(tuple(int(x) for x in r), int(n)) for r, n in zip(z["sched_stage_res"],
                                                                           z["sched_stage_steps"])])


@pytest.mark.parametrize("asynchronous", [False, True])
def test_run_schedule_golden(z, asynchronous):
    sch = _golden_stages(z)
    g = grid_from(3, sch.stages[0].resolution, 2, z["sched_c0"])
    prob = BatchProblem(list(z["sched_batches"]), tg.LossConfig())
    r = run_schedule(prob, sch, g, tg.AdamConfig(lr=1e-2), asynchronous=asynchronous)
    terms = np.array([[t.loss.total, t.loss.fit, t.loss.eik, t.loss.tv] for t in r.trace])
    assert len(r.trace) == sch.total_steps() and len(r.stage_seconds) == 3
    assert [t.stage for t in r.trace] == [0] * 4 + [1] * 5 + [2] * 3
    assert r.trace[3].resolution == (4, 4, 4) and r.trace[4].resolution == (7, 8, 6)
    assert [t.step for t in r.trace] == list(range(12))
    assert tuple(r.grid.spec.resolution) == (12, 12, 12)
    assert_close(terms[:, 0], z["sched_terms"][:, 0], 1e-4, floor=1e-30, what="loss curve")
    assert_close(r.grid.coeffs, z["sched_final"], 1e-3, floor=1e-2, what="final coeffs")
    assert r.grid.all_finite()


def test_run_schedule_zero_steps_and_errors():
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=(4, 4, 4), order=2),
                     tg.InitOptions(mode=tg.InitMode.SmallUniform, epsilon=0.1, seed=5))
    before = g.coeffs
    r = run_schedule(BatchProblem([]), Schedule.single((4, 4, 4), 0), g)
    assert r.trace == [] and np.array_equal(r.grid.coeffs, before)

    class BadProblem(TrainProblem):
        fused = False

        def compute(self, grid, step=0, asynchronous=False):
            return tg.LossTerms(float("nan"), 0.0, 0.0, 0.0)

    with pytest.raises(tg.NumericalError, match="stage 0 step 0"):
        run_schedule(BadProblem(), Schedule.single((4, 4, 4), 3), tg.init_grid(tg.GridSpec(3, (4, 4, 4))))

    # A fused step whose loss goes non-finite in stage 1 (gt = inf from step 6 on).
    rng = np.random.default_rng(2)
    bs = []
    for k in range(8):
        b = np.concatenate([rng.uniform(-1, 1, (64, 3)), rng.uniform(-0.5, 0.5, (64, 1))], 1)
        if k >= 6:
            b[0, 3] = np.inf
        bs.append(b)
    sch = Schedule([Stage((4, 4, 4), 4), Stage((6, 6, 6), 4)])
    for asynchronous in (False, True):
        with pytest.raises(tg.NumericalError, match="stage 1 step 2"):
            run_schedule(BatchProblem(bs), sch, tg.init_grid(tg.GridSpec(3, (4, 4, 4))), asynchronous=asynchronous)


def test_run_schedule_unfused_matches_fused(z):
    """The reference loop shape (zero grad -> compute -> finite check -> adam)
    through an unfused problem gives the fused trajectory."""
    sch = _golden_stages(z)
    batches = list(z["sched_batches"])

    class Unfused(TrainProblem):
        fused = False

        def compute(self, grid, step=0, asynchronous=False):
            return tg.total_loss(grid, batches[step], tg.LossConfig(), with_grad=True)

    r = run_schedule(Unfused(), sch, grid_from(3, sch.stages[0].resolution, 2, z["sched_c0"]),
                     tg.AdamConfig(lr=1e-2))
    terms = np.array([t.loss.total for t in r.trace])
    assert_close(terms, z["sched_terms"][:, 0], 1e-4, floor=1e-30, what="unfused loss curve")


@pytest.mark.parametrize("name", ["d3", "d2"])
def test_fit_sdf_reference_stream_golden(z, name):
    dim = 3 if name == "d3" else 2
    res = tuple(int(r) for r in z[f"fit_{name}_res"])[:dim]
    opts = FitOptions(loss=tg.LossConfig(batch_size=64), adam=tg.AdamConfig(lr=1e-2), total_steps=30,
                      holdout_fraction=0.1, seed=3, exact_stream=True, asynchronous=False)
    r = fit_sdf(z[f"fit_{name}_samples"], tg.GridSpec(dim=dim, resolution=res, order=2), opts)
    rep = z[f"fit_{name}_report"]
    assert (r.report.train_samples, r.report.holdout_samples) == (int(rep[1]), int(rep[2]))
    terms = np.array([t.loss.total for t in r.trace])
    assert_close(terms, z[f"fit_{name}_terms"][:, 0], 1e-4, floor=1e-30, what="fit_sdf loss curve")
    assert_close(r.grid.coeffs, z[f"fit_{name}_final"], 1e-3, floor=1e-2, what="fit_sdf final coeffs")
    assert abs(r.report.holdout_mae - rep[0]) <= 1e-5 * max(1.0, rep[0])


@pytest.mark.parametrize("name", ["d3", "d2"])
def test_fit_sdf_fresh_uniform_eikonal_vs_reference(z, reference, name):
    """fit_sdf with EikonalPointSource::FreshUniform and the reference stream:
    every step draws its batch indices and then its |batch| eikonal points from
    the one Rng, as the reference's SdfProblem does; loss curve against the
    reference fit_sdf run live on the same samples."""
    from oracle.pyoracle import Loss, Spec
    dim = 3 if name == "d3" else 2
    res = tuple(int(r) for r in z[f"fit_{name}_res"])[:dim]
    smp = z[f"fit_{name}_samples"]
    lc = tg.LossConfig(batch_size=64, lambda1=1e-2, eikonal_point_source=tg.EikonalPointSource.FreshUniform)
    opts = FitOptions(loss=lc, adam=tg.AdamConfig(lr=1e-2), total_steps=30, holdout_fraction=0.1, seed=3,
                      exact_stream=True, asynchronous=False)
    r = fit_sdf(smp, tg.GridSpec(dim=dim, resolution=res, order=2), opts)
    _, ref_terms, rep = reference.fit_sdf(Spec(dim=dim, res=res, order=2),
                                          np.asarray(smp, dtype=np.float32).astype(np.float64), 30,
                                          Loss(lambda1=1e-2), 64, lr=1e-2, holdout_fraction=0.1, seed=3,
                                          eik_fresh=True)
    assert (r.report.train_samples, r.report.holdout_samples) == (rep["train_samples"], rep["holdout_samples"])
    terms = np.array([t.loss.as_array() for t in r.trace])
    assert_close(terms[:, 0], ref_terms[:, 0], 1e-4, floor=1e-30, what="fresh-uniform fit loss curve")
    assert_close(terms[:, 2], ref_terms[:, 2], 1e-4, floor=1e-30, what="fresh-uniform eikonal curve")


def test_fit_sdf_device_stream_trains():
    """Default device batch draw: progressive 3-stage fit of a sphere converges."""
    smp = tg.sample(tg.SHAPE_SPHERE, 3, 7, 200000, near_frac=0.5, sigma=0.01, param0=0.6)
    opts = FitOptions(loss=tg.LossConfig(batch_size=32768), adam=tg.AdamConfig(lr=1e-2), total_steps=300,
                      holdout_fraction=0.05, seed=1)
    r = fit_sdf(smp, tg.GridSpec(dim=3, resolution=(48, 48, 48), order=2), opts)
    assert [len([t for t in r.trace if t.stage == s]) for s in range(3)] == [100, 100, 100]
    assert r.trace[-1].loss.total < 0.25 * r.trace[0].loss.total
    # the adaptive weight (sdf_loss.cpp:15-27) concentrates the fit near the
    # surface, so the whole-domain MAE only has to beat the zero grid clearly
    assert r.report.holdout_mae < 0.5 * np.mean(np.abs(smp[:, 3]))


@pytest.mark.parametrize("name", ["d3", "d2"])
def test_tgrid_roundtrip_and_reference_files(z, name, tmp_path):
    dim = 3 if name == "d3" else 2
    res = tuple(int(r) for r in z[f"tgrid_{name}_res"])[:dim]
    spec = tg.GridSpec(dim=dim, resolution=res, order=2, origin=(-0.5, -1.0, -2.0)[:dim],
                       extent=(1.0, 2.5, 4.0)[:dim])
    c = z[f"tgrid_{name}_coeffs"]
    g = tg.init_grid(spec)
    g.coeffs = c
    for prec in (tg.StoragePrecision.F64, tg.StoragePrecision.F32):
        p = tmp_path / f"g{int(prec)}.tgrid"
        tg.save_tgrid(g, p, prec)
        data = p.read_bytes()
        assert data == z[f"tgrid_{name}_p{int(prec)}"].tobytes()  # identical to the reference's file
        ref_file = tmp_path / f"ref{int(prec)}.tgrid"
        ref_file.write_bytes(z[f"tgrid_{name}_p{int(prec)}"].tobytes())
        h = tg.load_tgrid(ref_file)
        assert h.spec.dim == dim and tuple(h.spec.resolution) == res and h.spec.order == 2
        assert tuple(h.spec.origin) == tuple(spec.origin) and tuple(h.spec.extent) == tuple(spec.extent)
        assert np.array_equal(h.coeffs, c)
    assert tgrid_bytes(Spec(dim=dim, res=res + (1,) * (3 - dim), order=2, origin=(-0.5, -1.0, -2.0),
                            extent=(1.0, 2.5, 4.0)), c, 0) == z[f"tgrid_{name}_p0"].tobytes()


def test_tgrid_errors(z, tmp_path):
    good = z["tgrid_d3_p0"].tobytes()
    cases = {"missing.tgrid": (None, "tgrid: cannot open"),
             "magic.tgrid": (b"TGRX" + good[4:], "tgrid: bad magic"),
             "version.tgrid": (good[:4] + b"\x02\x00\x00\x00" + good[8:], "tgrid: unsupported version 2"),
             "dim.tgrid": (good[:8] + b"\x04" + good[9:], "tgrid: unsupported dim 4"),
             "header.tgrid": (good[:20], "tgrid: truncated file while reading"),
             "payload.tgrid": (good[:-3], "tgrid: truncated coefficient payload"),
             "prec.tgrid": (good[:70] + b"\x07" + good[71:], "tgrid: unknown precision flag")}
    for fname, (data, msg) in cases.items():
        p = tmp_path / fname
        if data is not None:
            p.write_bytes(data)
        with pytest.raises(tg.IngestError, match=msg):
            tg.load_tgrid(p)
    with pytest.raises(tg.IngestError, match="cannot open for writing"):
        tg.save_tgrid(tg.init_grid(tg.GridSpec(3, (2, 2, 2))), tmp_path / "no" / "dir.tgrid")


@pytest.mark.parametrize("dim,res,order", [(2, (13, 9), 2), (3, (7, 6, 5), 2), (3, (9, 4, 6), 1)])
def test_init_modes_match_reference(reference, dim, res, order):
    """init_grid (taylor_grid.cpp:162-188): Zeros, Constant (f0 only) and
    SmallUniform (the reference Rng stream, uniform(-eps, eps) over every
    coefficient in order) equal the reference's coefficients rounded to fp32;
    the memory cap refuses with the reference's message."""
    from oracle.pyoracle import Spec
    s = Spec(dim=dim, res=res, order=order)
    spec = tg.GridSpec(dim=dim, resolution=tuple(res) + ((1,) if dim == 2 else ()), order=order)
    cases = [(tg.InitMode.Zeros, 0, dict()), (tg.InitMode.Constant, 1, dict(constant=0.3125)),
             (tg.InitMode.Constant, 1, dict(constant=-1.7)),
             (tg.InitMode.SmallUniform, 2, dict(epsilon=0.05, seed=17)),
             (tg.InitMode.SmallUniform, 2, dict(epsilon=1e-4, seed=0))]
    for mode, rmode, kw in cases:
        g = tg.init_grid(spec, tg.InitOptions(mode=mode, **kw))
        ref = reference.init_grid(s, rmode, kw.get("constant", 0.0), kw.get("epsilon", 1e-4), kw.get("seed", 0))
        assert np.array_equal(g.coeffs, ref.astype(np.float32).astype(np.float64)), (mode, kw)
        g.close()
    cap = 8 * s.V * s.K - 1
    with pytest.raises(MemoryError) as e_ref:
        reference.init_grid(s, 0, cap=cap)
    with pytest.raises(tg.ResourceError) as e_ours:
        tg.init_grid(spec, tg.InitOptions(memory_cap_bytes=cap))
    assert str(e_ours.value) == str(e_ref.value)


def test_all_finite_detects_nan_and_inf():
    """all_finite (taylor_grid.cpp:190-195) on the device grid."""
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=(9, 7, 5), order=2),
                     tg.InitOptions(mode=tg.InitMode.SmallUniform, epsilon=0.1, seed=3))
    assert g.all_finite()
    c = g.coeffs
    for bad in (np.nan, np.inf, -np.inf):
        for idx in (0, 17, c.size - 1):
            d = c.copy()
            d[idx] = bad
            g.coeffs = d
            assert not g.all_finite(), (bad, idx)
    g.coeffs = c
    assert g.all_finite()
