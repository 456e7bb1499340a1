"""Pin the CPU oracle (oracle/tg_oracle.c) before trusting it (CPU only).

1. bit-exact against the committed golden vectors made by the reference build
   (tests/golden/make_golden.py);
2. bit-exact against the live reference build (oracle/_ref) on fresh inputs
   when it is present;
3. the reference's own known-answer tests for the path,
   restated from tests/test_taylor_field.cpp, test_sdf_fit.cpp and
   test_optimizer.cpp.
"""
import math

import numpy as np
import pytest

from conftest import load_golden
from oracle.pyoracle import Loss, Spec


def spec_from(res, dim, order):
    return Spec(dim=dim, res=tuple(int(r) for r in res), order=order)


# ---- 1. golden vectors ---------------------------------------------------------------


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("order", [0, 1, 2])
def test_golden_eval_backprop(oracle, dim, order):
    z = load_golden("eval_backprop.npz")
    k = f"d{dim}o{order}_"
    s = spec_from(z[k + "res"], dim, order)
    vals, grads = oracle.eval(s, z[k + "coeffs"], z[k + "pts"], True)
    assert np.array_equal(vals, z[k + "vals"])
    assert np.array_equal(grads, z[k + "grads"])
    g = np.zeros(s.V * s.K)
    oracle.backprop(s, z[k + "pts"], z[k + "up"], z[k + "uv"], g)
    assert np.array_equal(g, z[k + "bgrad"])


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("name,cfg", [("paper", Loss()), ("recon", Loss(lambda1=0.0, use_tv=False)),
                                      ("dw", Loss(differentiate_weight=True))])
def test_golden_total_loss(oracle, dim, name, cfg):
    z = load_golden("loss.npz")
    k = f"d{dim}_{name}_"
    s = spec_from(z[k + "res"], dim, 2)
    g = np.zeros(s.V * s.K)
    terms = oracle.total_loss(s, z[k + "coeffs"], z[k + "samples"], cfg, g)
    assert np.array_equal(terms, z[k + "terms"])
    assert np.array_equal(g, z[k + "grad"])


@pytest.mark.parametrize("dim", [2, 3])
def test_golden_tv(oracle, dim):
    z = load_golden("loss.npz")
    k = f"d{dim}_tv_"
    s = spec_from(z[k + "res"], dim, 2)
    g = np.zeros(s.V * s.K)
    tv = oracle.tv_loss(s, z[k + "coeffs"], g, 0.7)
    assert tv == z[k + "tv"][0]
    assert np.array_equal(g, z[k + "grad"])


def test_golden_adam_and_training(oracle):
    z = load_golden("train.npz")
    p = z["adam_p0"].copy()
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    t = 0
    for k in range(len(z["adam_grads"])):
        t, bad = oracle.adam_step(p, z["adam_grads"][k], m, v, t, lr=0.01)
        assert bad == -1
        assert np.array_equal(p, z["adam_traj"][k])
    s = spec_from(z["train_res"], 2, 2)
    final, terms = oracle.train(s, np.zeros(s.V * s.K), z["train_batches"], Loss(), lr=1e-2)
    assert np.array_equal(terms, z["train_terms"])
    assert np.array_equal(final, z["train_final"])


# ---- 2. live reference (only where /root/reference was compiled) --------------------------


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("order", [0, 1, 2])
def test_live_reference_bit_exact(oracle, reference, dim, order):
    rng = np.random.default_rng(100 + 10 * dim + order)
    s = Spec(dim=dim, res=(6, 7, 5), order=order)
    c = rng.uniform(-1, 1, s.V * s.K)
    pts = rng.uniform(-1.2, 1.2, (128, 3))
    v1, g1 = oracle.eval(s, c, pts, True)
    v2, g2 = reference.eval(s, c, pts, True)
    assert np.array_equal(v1, v2) and np.array_equal(g1, g2)
    smp = np.concatenate([pts, rng.uniform(-0.4, 0.4, (128, 1))], 1)
    for cfg in (Loss(), Loss(lambda1=0.0), Loss(differentiate_weight=True, lambda2=0.0),
                Loss(use_weighting=False, use_tv=False)):
        ga, gb = np.zeros(s.V * s.K), np.zeros(s.V * s.K)
        ta = oracle.total_loss(s, c, smp, cfg, ga)
        tb = reference.total_loss(s, c, smp, cfg, gb)
        assert np.array_equal(ta, tb) and np.array_equal(ga, gb)
    new_res = (11, 9, 7)
    assert np.array_equal(oracle.resample(s, c, s.K, new_res), reference.upsample(s, c, new_res))


def test_live_reference_threads_agree(reference):
    """threaded == sequential within 1e-12 (test_sdf_fit.cpp:406-422)."""
    rng = np.random.default_rng(5)
    s = Spec(dim=3, res=(6, 6, 6), order=2)
    c = rng.uniform(-0.5, 0.5, s.V * s.K)
    smp = np.concatenate([rng.uniform(-1, 1, (200, 3)), rng.uniform(-0.3, 0.3, (200, 1))], 1)
    g1, g2 = np.zeros(s.V * s.K), np.zeros(s.V * s.K)
    t1 = reference.total_loss(s, c, smp, Loss(), g1, threads=1)
    t2 = reference.total_loss(s, c, smp, Loss(), g2, threads=2)
    assert abs(t1[0] - t2[0]) <= 1e-12 * abs(t1[0])
    assert np.all(np.abs(g1 - g2) <= 1e-12 * np.maximum(1.0, np.abs(g1)))


# ---- 3. the reference's known-answer tests, restated ------------------------------------------


def test_coeff_count_table(oracle):
    # test_taylor_field.cpp:29-39
    assert [oracle.coeff_count(o, d) for o, d in [(2, 3), (0, 3), (2, 2), (1, 3), (1, 2), (0, 2)]] == [10, 1, 6, 4, 3, 1]
    assert oracle.coeff_count(3, 3) == -1 and oracle.coeff_count(-1, 3) == -1 and oracle.coeff_count(2, 4) == -1
    assert Spec(dim=3, res=(17, 17, 17), order=2).V * 10 == 49130


def test_locate_hand_cases(oracle):
    # test_taylor_field.cpp:77-110
    s = Spec(dim=3, res=(3, 3, 3), origin=(0, 0, 0), extent=(1, 1, 1), order=0)
    cell, loc, _ = oracle.locate(s, (0, 0, 0))
    assert cell == [0, 0, 0] and loc == [0, 0, 0]
    cell, loc, _ = oracle.locate(s, (1, 1, 1))
    assert cell == [1, 1, 1] and loc == [1, 1, 1]
    cell, loc, _ = oracle.locate(s, (0.75, 0.25, 0.25))
    assert cell == [1, 0, 0] and loc == [0.5, 0.5, 0.5]
    cell, loc, _ = oracle.locate(s, (-5.0, 2.0, 0.5))
    assert cell[0] == 0 and loc[0] == 0.0 and cell[1] == 1 and loc[1] == 1.0
    with pytest.raises(ValueError):
        oracle.locate(s, (float("nan"), 0.5, 0.5))


def quadratic_grid(s, A, b, c):
    """Exact Taylor data of 0.5 x^T A x + b.x + c (oracles.hpp:157-187)."""
    coeffs = np.zeros(s.V * s.K)
    dim = s.dim
    idx = 0
    rz = s.res[2] if dim == 3 else 1
    for z in range(rz):
        for y in range(s.res[1]):
            for x in range(s.res[0]):
                v = [x, y, z][:dim]
                p = np.array([s.origin[a] + s.spacing(a) * v[a] for a in range(dim)])
                blk = coeffs[idx * s.K:(idx + 1) * s.K]
                blk[0] = c + b[:dim] @ p + 0.5 * p @ A[:dim, :dim] @ p
                blk[1:1 + dim] = b[:dim] + A[:dim, :dim] @ p
                t = 1 + dim
                for i in range(dim):
                    for j in range(i, dim):
                        blk[t] = A[i, j]
                        t += 1
                idx += 1
    return coeffs


def test_quadratic_exactness(oracle):
    # test_taylor_field.cpp:112-148
    rng = np.random.default_rng(7)
    for dim in (2, 3):
        for _ in range(3):
            A = rng.uniform(-2, 2, (3, 3))
            A = (A + A.T) / 2
            b = rng.uniform(-1, 1, 3)
            c = rng.uniform(-1, 1)
            s = Spec(dim=dim, res=(5, 4, 6), order=2)
            coeffs = quadratic_grid(s, A, b, c)
            pts = rng.uniform(-1, 1, (100, 3))
            if dim == 2:
                pts[:, 2] = 0
            got = oracle.eval(s, coeffs, pts)
            P = pts[:, :dim]
            expect = c + P @ b[:dim] + 0.5 * np.einsum("ni,ij,nj->n", P, A[:dim, :dim], P)
            assert np.all(np.abs(got - expect) <= 1e-9 * np.maximum(np.abs(expect), 1e-9))


def test_order0_center_and_multilinear(oracle):
    # test_taylor_field.cpp:150-158 and :176-187
    for dim in (2, 3):
        s = Spec(dim=dim, res=(2, 2, 2), order=0)
        c = np.zeros(s.V)
        c[0] = 1.0
        assert oracle.eval(s, c, [[0.0, 0.0, 0.0]])[0] == pytest.approx(1.0 / (1 << dim), rel=1e-14)
    rng = np.random.default_rng(9)
    s = Spec(dim=3, res=(6, 5, 7), order=0)
    vals = rng.uniform(-1, 1, s.V)
    pts = rng.uniform(-1, 1, (200, 3))
    got = oracle.eval(s, vals, pts)
    for p, gval in zip(pts, got):
        cell, loc, vid = oracle.locate(s, p)
        acc = 0.0
        for bits in range(8):
            w = 1.0
            for a in range(3):
                w *= loc[a] if (bits >> a) & 1 else 1.0 - loc[a]
            acc += w * vals[vid[bits]]
        assert abs(gval - acc) <= 1e-12 * max(abs(acc), 1e-12)


def test_spatial_gradient_and_backprop_fd(oracle):
    # test_taylor_field.cpp:249-271, :296-318
    rng = np.random.default_rng(21)
    for dim in (2, 3):
        for order in (0, 1, 2):
            s = Spec(dim=dim, res=(4, 4, 4), order=order)
            c = rng.uniform(-1, 1, s.V * s.K)
            p = np.zeros(3)
            for a in range(dim):
                cell = rng.integers(0, s.res[a] - 1)
                p[a] = s.origin[a] + (cell + rng.uniform(0.05, 0.95)) * s.spacing(a)
            _, g = oracle.eval(s, c, [p], True)
            for a in range(dim):
                up, dn = p.copy(), p.copy()
                up[a] += 1e-4
                dn[a] -= 1e-4
                fd = (oracle.eval(s, c, [up])[0] - oracle.eval(s, c, [dn])[0]) / 2e-4
                assert abs(g[0, a] - fd) <= 1e-5 * max(abs(fd), abs(g[0, a]), 1e-5)
            grad = np.zeros_like(c)
            oracle.backprop(s, [p], [1.0], [[0, 0, 0]], grad)
            touched = 0
            for i in range(len(c)):
                cc = c.copy()
                cc[i] += 1e-5
                f1 = oracle.eval(s, cc, [p])[0]
                cc[i] -= 2e-5
                f0 = oracle.eval(s, cc, [p])[0]
                fd = (f1 - f0) / 2e-5
                if grad[i] != 0 or abs(fd) > 1e-9:
                    assert abs(grad[i] - fd) <= 1e-6 * max(abs(grad[i]), abs(fd), 1e-7)
                touched += grad[i] != 0
            assert touched <= (1 << dim) * s.K


def test_locality_exactly_80(oracle):
    # test_taylor_field.cpp:319-327
    s = Spec(dim=3, res=(5, 5, 5), order=2)
    grad = np.zeros(s.V * s.K)
    oracle.backprop(s, [[0.137, -0.295, 0.481]], [1.3], [[0, 0, 0]], grad)
    assert int(np.count_nonzero(grad)) == 80


def test_adaptive_weight_known_values(oracle):
    # test_sdf_fit.cpp:61-78
    assert oracle.adaptive_weight(0.0, 5.0, 10.0) == pytest.approx(1.0, rel=1e-12)
    assert oracle.adaptive_weight(100.0, 100.0, 10.0) <= 1e-6
    assert oracle.adaptive_weight(0.1, -0.1, 10.0) == pytest.approx(0.5378828427399902, rel=1e-12)
    for d in (-0.5, -0.3, 0.0, 0.4, 0.6):
        w = oracle.adaptive_weight(d, d, 50.0)
        assert 0.0 <= w <= 1.0
        if abs(50 * d) < 30:
            assert w > 0.0


def test_tv_hand_fixture_and_invariances(oracle):
    # test_sdf_fit.cpp:218-239, :279-290
    s = Spec(dim=3, res=(2, 2, 2), order=0)
    c = np.array([0, 1, 0, 1, 0, 1, 0, 1], dtype=float)  # f0 split along x
    assert oracle.tv_loss(s, c) == pytest.approx(4.0 / 12.0, rel=1e-15)
    s = Spec(dim=3, res=(5, 5, 5), order=2)
    c = np.zeros(s.V * s.K)
    c[0::10] = 4.2
    assert oracle.tv_loss(s, c) == 0.0
    rng = np.random.default_rng(71)
    s = Spec(dim=3, res=(4, 4, 4), order=2)
    c = rng.uniform(-1, 1, s.V * s.K)
    base = oracle.tv_loss(s, c)
    assert oracle.tv_loss(s, 2 * c) == pytest.approx(4 * base, rel=1e-12)
    c2 = c.copy()
    c2[0::10] += 13.7
    assert oracle.tv_loss(s, c2) == pytest.approx(base, rel=1e-9)


def test_zero_grid_eikonal_and_zero_grad(oracle):
    # test_sdf_fit.cpp:162-168: zero grid -> eik = 1 per point, zero subgradient
    s = Spec(dim=3, res=(4, 4, 4), order=2)
    c = np.zeros(s.V * s.K)
    smp = np.array([[0.1, 0.2, 0.3, 0.0], [-0.5, 0.0, 0.7, 0.0]])
    g = np.zeros_like(c)
    terms = oracle.total_loss(s, c, smp, Loss(lambda1=1.0, use_tv=False, use_weighting=False), g)
    assert terms[2] == pytest.approx(1.0)
    assert terms[1] == 0.0


def test_total_loss_fd_frozen_weight(oracle):
    # test_sdf_fit.cpp:361-387 (acceptance criterion 1)
    rng = np.random.default_rng(777)
    for dim in (2, 3):
        for order in (0, 1, 2):
            s = Spec(dim=dim, res=(4, 4, 4), order=order)
            c = rng.uniform(-0.5, 0.5, s.V * s.K)
            pts = rng.uniform(-1, 1, (8, 3))
            if dim == 2:
                pts[:, 2] = 0
            vals = oracle.eval(s, c, pts)
            gt = vals + np.where(rng.uniform(size=8) < 0.5, -1, 1) * rng.uniform(0.05, 0.3, 8)
            smp = np.concatenate([pts, gt[:, None]], 1)
            cfg = Loss()
            w0 = np.array([oracle.adaptive_weight(v, g_, cfg.k) for v, g_ in zip(vals, gt)])

            def frozen(cc):
                v, gr = oracle.eval(s, cc, pts, True)
                recon = np.mean(w0 * np.abs(v - gt))
                eik = np.mean((np.linalg.norm(gr, axis=1) - 1) ** 2)
                return recon + cfg.lambda1 * eik + cfg.lambda2 * oracle.tv_loss(s, cc)

            grad = np.zeros_like(c)
            oracle.total_loss(s, c, smp, cfg, grad)
            max_err = 0.0
            for i in range(len(c)):
                cc = c.copy()
                cc[i] += 1e-5
                f1 = frozen(cc)
                cc[i] -= 2e-5
                f0 = frozen(cc)
                fd = (f1 - f0) / 2e-5
                max_err = max(max_err, abs(grad[i] - fd) / max(abs(grad[i]), abs(fd), 1e-3))
            assert max_err <= 1e-5


def test_adam_known_answers(oracle):
    # test_optimizer.cpp:67-121
    p, g = np.array([0.0]), np.array([1.0])
    m, v = np.zeros(1), np.zeros(1)
    t, bad = oracle.adam_step(p, g, m, v, 0, lr=0.003)
    assert abs(p[0] + 0.003) <= 1e-6 and t == 1 and bad == -1
    p = np.array([1.0, -2.0, 0.5, 3.0])
    before = p.copy()
    oracle.adam_step(p, np.zeros(4), np.zeros(4), np.zeros(4), 0)
    assert np.array_equal(p, before)
    p = np.zeros(3)
    g = np.array([0.0, float("nan"), 0.0])
    t, bad = oracle.adam_step(p, g, np.zeros(3), np.zeros(3), 0)
    assert bad == 1 and t == 0 and np.all(p == 0.0)
    # 200 steps on (p-3)^2 against a scalar oracle
    p = np.array([0.0])
    m, v = np.zeros(1), np.zeros(1)
    t = 0
    pr, mr, vr = 0.0, 0.0, 0.0
    for k in range(1, 201):
        g = np.array([2.0 * (p[0] - 3.0)])
        gr = 2.0 * (pr - 3.0)
        t, _ = oracle.adam_step(p, g, m, v, t, lr=0.1)
        mr = 0.9 * mr + 0.1 * gr
        vr = 0.999 * vr + 0.001 * gr * gr
        pr -= 0.1 * (mr / (1 - 0.9 ** k)) / (math.sqrt(vr / (1 - 0.999 ** k)) + 1e-8)
        assert p[0] == pytest.approx(pr, rel=1e-12)
    assert abs(p[0] - 3.0) <= 0.05


def test_markstein_division_matches_ieee(oracle):
    """The device locate divides with x*RN(1/h) + one fma correction
    (tg_device.cuh div_by_h). Check it equals IEEE x/h on the domain's inputs:
    fp32 coordinates in [-1.05, 1.05] minus the origin, all BASELINE spacings,
    vertex-aligned points included."""
    rng = np.random.default_rng(1)
    L = oracle.L
    bad = 0
    for res in (2, 3, 5, 7, 16, 17, 100, 128, 129, 255, 256, 257, 511, 512, 1000, 1023, 1024):
        for origin, extent in ((-1.0, 2.0), (0.0, 1.0), (-0.3, 1.7)):
            h = extent / (res - 1)
            inv_h = 1.0 / h
            xs = rng.uniform(origin, origin + extent, 20000).astype(np.float32).astype(np.float64)
            verts = (origin + h * np.arange(res)).astype(np.float32).astype(np.float64)
            for x in np.concatenate([xs, verts, [origin, origin + extent]]):
                num = x - origin
                if num < 0:
                    num = 0.0
                if L.tgo_markstein_div(num, h, inv_h) != num / h:
                    bad += 1
    assert bad == 0


@pytest.mark.parametrize("dim", [2, 3])
def test_fresh_uniform_eikonal_decomposition(reference, dim):
    """EikonalPointSource::FreshUniform (sdf_loss.cpp:274-283) = the recon-only
    total_loss on the batch + lambda1 * eikonal_loss on |batch| points that
    tg::Rng(seed).uniform_in_box draws; the library's tgcu_rng_uniform_box
    (tg.Rng) reproduces the reference's own draws."""
    import paper_2402_14415_b200 as tg
    rng = np.random.default_rng(40 + dim)
    s = Spec(dim=dim, res=(9, 8, 7) if dim == 3 else (12, 10), order=2)
    c = rng.uniform(-0.3, 0.3, s.V * s.K)
    pts = rng.uniform(-1.0, 1.0, (300, 3))
    if dim == 2:
        pts[:, 2] = 0.0
    smp = np.concatenate([pts, rng.uniform(-0.4, 0.4, (300, 1))], 1)
    cfg = Loss(lambda1=1e-2, lambda2=1e-3)
    seed = 1234
    g_ref = np.zeros(s.V * s.K)
    t_ref = reference.total_loss_fresh(s, c, smp, cfg, seed, g_ref)
    eik_pts = tg.Rng(seed).uniform_in_box(dim, [-1.0] * 3, [1.0] * 3, len(smp))
    g = np.zeros(s.V * s.K)
    t_fit = reference.total_loss(s, c, smp, Loss(lambda1=0.0, lambda2=cfg.lambda2), g)
    eik = reference.eikonal_loss(s, c, eik_pts, cfg.lambda1, g)
    total = t_fit[1] + cfg.lambda1 * eik + cfg.lambda2 * t_fit[3]
    np.testing.assert_allclose([total, t_fit[1], eik, t_fit[3]], t_ref, rtol=1e-12, atol=0)
    np.testing.assert_allclose(g, g_ref, rtol=1e-10, atol=1e-14 * np.abs(g_ref).max())
