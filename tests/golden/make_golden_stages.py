"""Golden vectors for the SURVEY §8f rows, generated from the REFERENCE build.

Runs the reference's own code (oracle/_ref/libtgref.so: upsample,
sample_grid_field, run_schedule, fit_sdf, save_tgrid, Rng) on small seeded
inputs and stores inputs + outputs in tests/golden/stages.npz, so the GPU tests
(and the CPU oracle tests) need no /root/reference at run time.

    python tests/golden/make_golden_stages.py
"""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Loss, Reference, Spec  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def sphere_samples(rng, n, dim, r=0.5):
    """Half uniform, half near the circle/sphere of radius r, fp32-representable."""
    p = rng.uniform(-1, 1, (n, 3))
    k = n // 2
    d = rng.normal(size=(k, 3))
    if dim == 2:
        d[:, 2] = 0.0
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    p[:k] = np.clip(r * d + rng.normal(0, 0.02, (k, 3)), -1, 1)
    if dim == 2:
        p[:, 2] = 0.0
    p = f32(p)
    gt = f32(np.linalg.norm(p[:, :dim], axis=1) - r)
    return np.concatenate([p, gt[:, None]], 1)


def main():
    R = Reference()
    rng = np.random.default_rng(20240415)
    out = {}
    # upsample (taylor_grid.cpp:273-284)
    ups = [("d3o2", 3, 2, (5, 6, 7), (9, 11, 13)), ("d3o1", 3, 1, (4, 4, 4), (8, 8, 8)),
           ("d3o0same", 3, 0, (5, 5, 5), (5, 5, 5)), ("d3o2odd", 3, 2, (5, 6, 7), (7, 10, 8)),
           ("d2o2", 2, 2, (6, 5, 1), (11, 9, 1))]
    for name, dim, order, res, nres in ups:
        s = Spec(dim=dim, res=res, order=order)
        c = f32(rng.uniform(-1, 1, s.V * s.K))
        out[f"up_{name}_res"] = np.array(res)
        out[f"up_{name}_meta"] = np.array([dim, order])
        out[f"up_{name}_newres"] = np.array(nres)
        out[f"up_{name}_coeffs"] = c
        out[f"up_{name}_out"] = R.upsample(s, c, nres)
    # sample_grid_field (marching.cpp:53-58) and the 2D CLI lattice
    for name, dim, order, res, lat in (("d3o2", 3, 2, (6, 5, 7), (13, 9, 11)), ("d3o1", 3, 1, (5, 5, 5), (17, 4, 9)),
                                       ("d2o2", 2, 2, (7, 6, 1), (15, 12, 1))):
        s = Spec(dim=dim, res=res, order=order)
        c = f32(rng.uniform(-1, 1, s.V * s.K))
        out[f"lat_{name}_res"] = np.array(res)
        out[f"lat_{name}_meta"] = np.array([dim, order])
        out[f"lat_{name}_lattice"] = np.array(lat)
        out[f"lat_{name}_coeffs"] = c
        out[f"lat_{name}_vals"] = R.sample_grid_field(s, c, lat)
    # run_schedule with three stages (schedule.cpp:62-108), paper loss, lr 1e-2
    stages = [((4, 4, 4), 4), ((7, 8, 6), 5), ((12, 12, 12), 3)]
    s = Spec(dim=3, res=stages[0][0], order=2)
    c0 = f32(rng.uniform(-0.05, 0.05, s.V * s.K))
    batches = np.array([sphere_samples(rng, 400, 3) for _ in range(12)])
    fin, terms = R.run_schedule(s, c0, stages, batches, Loss(), lr=1e-2)
    out["sched_stage_res"] = np.array([r for r, _ in stages])
    out["sched_stage_steps"] = np.array([n for _, n in stages])
    out["sched_c0"] = c0
    out["sched_batches"] = batches
    out["sched_final"] = fin
    out["sched_terms"] = terms
    # fit_sdf (sdf_fit.cpp:52-105): progressive default plan, holdout split
    for name, dim, res in (("d3", 3, (8, 8, 8)), ("d2", 2, (16, 16, 1))):
        s = Spec(dim=dim, res=res, order=2)
        smp = sphere_samples(rng, 700, dim)
        fc, ft, rep = R.fit_sdf(s, smp, 30, Loss(), 64, lr=1e-2, holdout_fraction=0.1, seed=3)
        out[f"fit_{name}_res"] = np.array(res)
        out[f"fit_{name}_samples"] = smp
        out[f"fit_{name}_final"] = fc
        out[f"fit_{name}_terms"] = ft
        out[f"fit_{name}_report"] = np.array([rep["holdout_mae"], rep["train_samples"], rep["holdout_samples"]])
    # Rng::index stream and fit_sdf's shuffle
    out["rng_index"] = R.rng_index(3, 700, 1000)
    out["shuffle_order"] = R.shuffle_order(3 ^ 0x5DEECE66D, 700)
    # .tgrid files written by the reference (grid_io.cpp:44-65)
    d = tempfile.mkdtemp()
    for name, dim, res in (("d3", 3, (3, 4, 5)), ("d2", 2, (5, 4, 1))):
        s = Spec(dim=dim, res=res, order=2, origin=(-0.5, -1.0, -2.0), extent=(1.0, 2.5, 4.0))
        c = f32(rng.uniform(-1, 1, s.V * s.K))
        out[f"tgrid_{name}_res"] = np.array(res)
        out[f"tgrid_{name}_coeffs"] = c
        for prec in (0, 1):
            path = os.path.join(d, f"{name}_{prec}.tgrid")
            R.save_tgrid(s, c, path, prec)
            out[f"tgrid_{name}_p{prec}"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "stages.npz"), **out)
    print("wrote", os.path.join(OUT, "stages.npz"), os.path.getsize(os.path.join(OUT, "stages.npz")), "bytes")


if __name__ == "__main__":
    main()
