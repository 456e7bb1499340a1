"""north_star parity criteria at the BASELINE configs (BASELINE.json configs[0],
[1], [3]) against the reference itself (oracle/_ref: the reference's own
sources, run live here at threads = nproc, its deterministic chunk-order
merge) and the C oracle.

Tolerances (north_star), written per test:
  loss curve over N Adam steps  |d| <= 1e-4 * |ref|   per step, every LossTerms component
  forward values                |d| <= 1e-6 * max(1, |ref|)
  spatial gradients             |d| <= 1e-5 * max(1, |ref|) + 16 eps32 * (L1 size of its terms)

The horizon N. The L1 data term makes the reference's own training chaotic:
a 1e-12 change of the initial coefficients moves its C1 loss curve by 2e-6
at step 1 and by 10 % within 500 steps, and the reference's arithmetic with
the coefficients / moments / gradient stored in fp32 (which north_star
prescribes) leaves 1e-4 at step 72 and reaches 9 % (DESIGN.md §5,
tools/traj_diag.py). No fp32-storage implementation can hold 1e-4 for
1,000 steps, so the curve is held to 1e-4 over the horizon fp32 storage
tracks (C1: 50 steps, measured 66; C2: 25, measured 34), and the rest of the
run is pinned two other ways: at checkpoints along the whole GPU trajectory
the reference's total_loss on the GPU's own coefficients must reproduce the
GPU's LossTerms of that step (1e-5, teacher forcing: correctness of every
step, independent of the chaos), and the trained outcome (mean loss of the
last 100 steps) must match the reference's within 2 %.

C1: 2D 128^2, order 2, zero init, circle r=0.5 U box (0.3, -0.2) half 0.3,
    65,536 uniform points per step (a fresh seeded batch every step), paper
    loss, Adam lr 1e-2, 1,000 steps.
C2: 3D 128^3, order 2, zero init, sphere r=0.6, 2^20 points per step (50 %
    uniform / 50 % near-surface sigma 0.01, fresh batch every step), paper
    loss, lr 1e-2: the first 50 steps of the 2,000-step run.
C4: 512^3 orders 1 and 2, coefficients 0.1 N(0,1) (device counter hash),
    2^18 uniform query points through the three query paths (direct gather,
    binned inside the call, brick-sorted), a 2^16 subset and the domain
    boundary checked against the oracle on the downloaded fp32 grid.
"""
import os

import numpy as np
import pytest

import paper_2402_14415_b200 as tg
from oracle.pyoracle import Loss, Spec

pytestmark = pytest.mark.gpu

THREADS = max(1, min(os.cpu_count() or 1, 64))


def curve_close(got, ref, rel, what):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    d = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)
    worst = np.unravel_index(int(np.argmax(d)), d.shape)
    assert d.max() <= rel, (f"{what}: max rel {d.max():.3g} > {rel:g} at step/term {worst}: "
                            f"got {got[worst]:.10g} ref {ref[worst]:.10g}")
    return float(d.max())


def run_gpu(spec, batches, lr, checkpoints=()):
    """The fused trajectory; returns its LossTerms per step and the
    coefficients before each checkpoint step."""
    g = tg.init_grid(spec)
    g.adam_reset(tg.AdamConfig(lr=lr))
    snaps, terms, done = {}, [], 0
    for c in sorted(checkpoints) + [len(batches)]:
        for b in batches[done:c]:  # pipelined host input: each array stays alive until sync
            tg.train_step(g, b, tg.LossConfig(), asynchronous=True)
        g.sync()
        if c > done:
            terms.append(g.trace(c - done))
        done = c
        if c < len(batches):
            snaps[c] = g.coeffs_f32()
    g.close()
    return np.concatenate(terms), snaps


def teacher_forced(reference, s, snaps, batches, ours, what):
    """The reference's total_loss on the GPU's coefficients before step c
    equals the GPU's LossTerms of step c."""
    for c, c32 in snaps.items():
        ref = reference.total_loss(s, c32.astype(np.float64), batches[c].astype(np.float64), Loss(),
                                   threads=THREADS)
        curve_close(ours[c][None], ref[None], 1e-5, f"{what}: teacher-forced step {c}")


def test_c1_1000_step_loss_curve_vs_reference(reference):
    steps, n = 1000, 1 << 16
    batches = [tg.sample(tg.SHAPE_C1_2D, 2, 10_000 + i, n) for i in range(steps)]
    ours, snaps = run_gpu(tg.GridSpec(dim=2, resolution=(128, 128, 1), order=2), batches, 1e-2,
                          checkpoints=range(100, steps, 100))
    s = Spec(dim=2, res=(128, 128), order=2)
    _, ref, _ = reference.train(s, np.zeros(s.V * s.K), np.array(batches, dtype=np.float64), Loss(), lr=1e-2,
                                threads=THREADS)
    curve_close(ours[:50], ref[:50], 1e-4, "C1 LossTerms {total, fit, eik, tv}, steps 0-49")
    teacher_forced(reference, s, snaps, batches, ours, "C1")
    assert ref[-1, 0] < 0.01 * ref[0, 0]  # the fit actually trains
    m_ours, m_ref = ours[-100:, 0].mean(), ref[-100:, 0].mean()
    assert abs(m_ours - m_ref) <= 0.02 * m_ref, (m_ours, m_ref)


def test_c2_50_steps_vs_reference(reference):
    steps, n = 50, 1 << 20
    batches = [tg.sample(tg.SHAPE_SPHERE, 3, 20_000 + i, n, near_frac=0.5, sigma=0.01, param0=0.6)
               for i in range(steps)]
    ours, snaps = run_gpu(tg.GridSpec(dim=3, resolution=(128, 128, 128), order=2), batches, 1e-2,
                          checkpoints=(30, 49))
    s = Spec(dim=3, res=(128, 128, 128), order=2)
    _, ref, _ = reference.train(s, None, np.array(batches, dtype=np.float64), Loss(), lr=1e-2, threads=THREADS)
    curve_close(ours[:25], ref[:25], 1e-4, "C2 LossTerms, steps 0-24")
    teacher_forced(reference, s, snaps, batches, ours, "C2")


@pytest.mark.parametrize("order", [1, 2])
def test_c4_512_query_values_vs_oracle(oracle, order):
    import torch
    res = (512, 512, 512)
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=res, order=order),
                     tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.1, seed=7, memory_cap_bytes=1 << 40))
    n = 1 << 18
    pts = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    tg.sample_uniform_device(3, 4242, pts)
    # domain boundary and outside points (clamped; max boundary -> last cell, local 1)
    edge = torch.tensor([[1, 1, 1], [-1, -1, -1], [1, -1, 0.3], [1.5, -2, 0.999999], [-1, 1, 1],
                         [0.999999, 0.999999, -0.999999]], dtype=torch.float32, device="cuda")
    pts[:edge.shape[0]] = edge
    vals = torch.empty(n, dtype=torch.float32, device="cuda")
    grads = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    # binned unsorted path (n >= 2^18) with the spatial gradient, direct path on a slice
    tg.eval_device(g, pts, vals, grads)
    vd = torch.empty(4096, dtype=torch.float32, device="cuda")
    tg.eval_device(g, pts[:4096], vd)
    spts = torch.empty_like(pts)
    perm = torch.empty(n, dtype=torch.int64, device="cuda")
    offs = torch.empty(tg.query_brick_codes(g) + 1, dtype=torch.int64, device="cuda")
    tg.sort_points(g, pts, spts, perm, offs)
    vs = tg.eval_sorted(g, spts, offs)
    torch.cuda.synchronize()
    c32 = g.coeffs_f32()
    g.close()
    sub = np.concatenate([np.arange(64), np.random.default_rng(order).choice(n, 1 << 16, replace=False)])
    p64 = pts.cpu().numpy().astype(np.float64)
    s = Spec(dim=3, res=res, order=order)
    ref, gref, l1 = oracle.eval_f32(s, c32, p64[sub], want_grad=True)
    del c32
    v = vals.cpu().numpy().astype(np.float64)[sub]
    gr = grads.cpu().numpy().astype(np.float64)[sub]
    assert np.all(np.abs(v - ref) <= 1e-6 * np.maximum(1.0, np.abs(ref))), np.max(np.abs(v - ref))
    # spatial gradient: a cancelling sum of terms ~|T|/h (h = 2/511), which an
    # fp32 blend resolves to ~16 eps32 of their L1 size (the same scale as the
    # training tests' mass term)
    tol = 1e-5 * np.maximum(1.0, np.abs(gref)) + 16 * 2.0 ** -24 * l1
    assert np.all(np.abs(gr - gref) <= tol), np.max(np.abs(gr - gref) / tol)
    # the direct-gather and brick-sorted kernels return the same values
    assert torch.equal(vd, vals[:4096])
    inv = torch.empty_like(perm)
    inv[perm] = torch.arange(n, device="cuda")
    assert torch.equal(vs[inv], vals)


@pytest.mark.parametrize("cfg", ["c3", "c5"])
def test_c3_c5_fused_step_vs_oracle(oracle, cfg):
    """BASELINE configs[2] / [4] shapes: the 64-primitive procedural target on
    256^3 (2^21 points, 50 % near-surface sigma 0.01) and on 512^3 (90 %
    near-surface sigma 0.005; 2^20 of the 2^23 points per step, to bound the
    fp64 oracle's time), on a random (non-zero) grid so every term is active:
    one fused step's loss terms and full gradient vs the oracle."""
    from test_gpu_parity import grad_close
    res, n, near, sigma = ((256,) * 3, 1 << 21, 0.5, 0.01) if cfg == "c3" else ((512,) * 3, 1 << 20, 0.9, 0.005)
    s = Spec(dim=3, res=res, order=2)
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=res, order=2),
                     tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.01, seed=21, memory_cap_bytes=1 << 40))
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    c64 = g.coeffs_f32().astype(np.float64)
    smp = tg.sample(tg.SHAPE_PRIMS, 3, 4100, n, near_frac=near, sigma=sigma, param0=42)
    t = tg.train_step(g, smp, tg.LossConfig(), export_grad=True)
    gpu_grad = g.grad()
    g.close()
    s64 = smp.astype(np.float64)
    gref = np.zeros(s.V * s.K)
    tref = oracle.total_loss(s, c64, s64, Loss(), gref)
    curve_close(t.as_array()[None], tref[None], 1e-6, f"{cfg} loss terms")
    mass = oracle.total_loss_mass(s, c64, s64, Loss())
    del c64
    grad_close(gpu_grad, gref, mass, what=f"{cfg} fused grad")
