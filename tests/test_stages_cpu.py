"""CPU tests of the SURVEY §8f rows: the oracle restatements pinned to the
reference's golden vectors (tests/golden/stages.npz, make_golden_stages.py),
the host-side pieces of the product (Schedule, trace CSV, Rng streams, .tgrid
sizes) and, when the reference build is present, live cross-checks."""
import numpy as np
import pytest

from conftest import load_golden
from oracle.pyoracle import Loss, Oracle, Spec, schedule_progressive, tgrid_bytes


@pytest.fixture(scope="module")
def z():
    return load_golden("stages.npz")


def _spec(z, key, **kw):
    dim, order = (int(x) for x in z[f"{key}_meta"])
    return Spec(dim=dim, res=tuple(int(r) for r in z[f"{key}_res"]), order=order, **kw)


@pytest.mark.parametrize("case", ["d3o2", "d3o1", "d3o0same", "d3o2odd", "d2o2"])
def test_oracle_upsample_golden(oracle, z, case):
    s = _spec(z, f"up_{case}")
    out = oracle.resample(s, z[f"up_{case}_coeffs"], s.K, z[f"up_{case}_newres"])
    assert np.array_equal(out, z[f"up_{case}_out"])


@pytest.mark.parametrize("case", ["d3o2", "d3o1", "d2o2"])
def test_oracle_lattice_golden(oracle, z, case):
    s = _spec(z, f"lat_{case}")
    out = oracle.sample_lattice(s, z[f"lat_{case}_coeffs"], z[f"lat_{case}_lattice"])
    assert np.array_equal(out, z[f"lat_{case}_vals"])


def test_oracle_run_schedule_golden(oracle, z):
    stages = [(tuple(int(x) for x in r), int(n)) for r, n in zip(z["sched_stage_res"], z["sched_stage_steps"])]
    s = Spec(dim=3, res=stages[0][0], order=2)
    fs, fin, terms = oracle.run_schedule(s, z["sched_c0"], stages, list(z["sched_batches"]), Loss(), lr=1e-2)
    assert fs.res == stages[-1][0]
    assert np.array_equal(terms, z["sched_terms"])
    assert np.array_equal(fin, z["sched_final"])


@pytest.mark.parametrize("name", ["d3", "d2"])
def test_tgrid_format_golden(z, name):
    res = tuple(int(r) for r in z[f"tgrid_{name}_res"])
    s = Spec(dim=3 if name == "d3" else 2, res=res, order=2, origin=(-0.5, -1.0, -2.0), extent=(1.0, 2.5, 4.0))
    for prec in (0, 1):
        ref = z[f"tgrid_{name}_p{prec}"].tobytes()
        assert tgrid_bytes(s, z[f"tgrid_{name}_coeffs"], prec) == ref


def test_tgrid_file_size_matches_golden(z):
    import paper_2402_14415_b200 as tg
    for name, dim in (("d3", 3), ("d2", 2)):
        res = tuple(int(r) for r in z[f"tgrid_{name}_res"])[:dim]
        spec = tg.GridSpec(dim=dim, resolution=res, order=2)
        for prec in (0, 1):
            assert tg.tgrid_file_size(spec, tg.StoragePrecision(prec)) == z[f"tgrid_{name}_p{prec}"].size


def test_schedule_progressive_reference_cases():
    """test_optimizer.cpp:123-139 restated, plus the validation errors."""
    from paper_2402_14415_b200.schedule import Schedule, Stage
    sch = Schedule.progressive((64, 64, 64), 3, 3000)
    assert [tuple(st.resolution) for st in sch.stages] == [(16, 16, 16), (32, 32, 32), (64, 64, 64)]
    assert sch.total_steps() == 3000
    bad = Schedule([Stage((8, 8, 8), 10), Stage((4, 8, 8), 10)])
    with pytest.raises(ValueError):
        bad.validate(3)
    with pytest.raises(ValueError):
        Schedule().validate(3)
    with pytest.raises(ValueError):
        Schedule([Stage((8, 8, 8), -1)]).validate(3)
    tiny = Schedule.progressive((8, 8, 8), 3, 300)
    assert tuple(tiny.stages[-1].resolution) == (8, 8, 8) and tiny.total_steps() == 300
    for target, dim, steps in (((5, 300, 7), 3, 301), ((128, 128), 2, 1000), ((4, 4, 4), 3, 10), ((9, 17, 33), 3, 7)):
        got = [(tuple(st.resolution), st.steps) for st in Schedule.progressive(target, dim, steps).stages]
        assert got == schedule_progressive(target, dim, steps)


def test_schedule_progressive_matches_live_reference(reference):
    from paper_2402_14415_b200.schedule import Schedule
    for target, dim, steps in (((64, 64, 64), 3, 3000), ((5, 300, 7), 3, 301), ((128, 128, 1), 2, 1000),
                               ((8, 8, 8), 3, 300), ((6, 4, 4), 3, 2), ((513, 257, 129), 3, 2000)):
        got = [(tuple(st.resolution), st.steps) for st in Schedule.progressive(target, dim, steps).stages]
        assert got == reference.schedule_progressive(target, dim, steps)


def test_rng_streams_match_golden(z):
    """The product's host Rng (sampler.cpp) against the reference's draws."""
    import ctypes as C
    import paper_2402_14415_b200 as tg
    L = tg.lib()
    h = C.c_void_p()
    assert L.tgcu_rng_create(3, C.byref(h)) == 0
    idx = np.empty(1000, dtype=np.int64)
    assert L.tgcu_rng_index(h, 700, 1000, idx.ctypes.data_as(C.c_void_p)) == 0
    L.tgcu_rng_destroy(h)
    assert np.array_equal(idx, z["rng_index"])
    order = np.empty(700, dtype=np.uint32)
    assert L.tgcu_shuffle_order(3 ^ 0x5DEECE66D, 700, order.ctypes.data_as(C.c_void_p)) == 0
    assert np.array_equal(order, z["shuffle_order"])


def test_trace_csv_matches_reference(reference):
    from paper_2402_14415_b200 import LossTerms
    from paper_2402_14415_b200.schedule import TraceRow, trace_csv_string
    rng = np.random.default_rng(4)
    rows = []
    for i in range(7):
        t = rng.normal(size=4) * 10.0 ** rng.integers(-12, 3, 4)
        rows.append(TraceRow(i, i // 3, (4 * (1 + i // 3), 8, 2), LossTerms(*t), float(rng.uniform(0, 50))))
    ref = reference.trace_csv([r.step for r in rows], [r.stage for r in rows], [r.resolution for r in rows],
                              [[r.loss.total, r.loss.fit, r.loss.eik, r.loss.tv] for r in rows],
                              [r.wall_ms for r in rows], "recon")
    assert trace_csv_string(rows, "recon") == ref


def test_live_reference_stage_rows(reference, oracle):
    """Fresh random cases: oracle restatements == reference, bit for bit."""
    rng = np.random.default_rng(11)
    s = Spec(dim=3, res=(4, 5, 6), order=2)
    c = rng.normal(0, 0.3, s.V * s.K)
    assert np.array_equal(oracle.resample(s, c, s.K, (9, 5, 11)), reference.upsample(s, c, (9, 5, 11)))
    assert np.array_equal(oracle.sample_lattice(s, c, (7, 3, 10)), reference.sample_grid_field(s, c, (7, 3, 10)))


@pytest.mark.parametrize("case", ["soft64", "soft100", "relu64"])
def test_oracle_radiance_golden(oracle, case):
    """forward_ray / backward_ray / photometric_loss restated == the reference."""
    z = load_golden("radiance.npz")
    p = case + "_"
    act, ns, order, deg = (int(x) for x in z[p + "meta"])
    ds = Spec(3, tuple(int(r) for r in z[p + "dres"]), order=order)
    ss = Spec(3, tuple(int(r) for r in z[p + "sres"]), order=0, origin=tuple(z[p + "sorg"]),
              extent=tuple(z[p + "sext"]))
    rays = dict(origins=z[p + "o"], dirs=z[p + "d"], near=z[p + "near"], far=z[p + "far"], gt=z[p + "gt"])
    r = oracle.photometric_loss(ds, z[p + "dc"], ss, deg, z[p + "sc"], rays, n_samples=ns, activation=act,
                                want_grad=True, render=True)
    assert r["loss"] == z[p + "loss"][0]
    assert np.array_equal(r["grad_density"], z[p + "gd"]) and np.array_equal(r["grad_sh"], z[p + "gs"])
    assert np.array_equal(r["colors"], z[p + "colors"]) and np.array_equal(r["residual"], z[p + "resid"])
