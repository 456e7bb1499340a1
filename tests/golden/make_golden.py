"""Generate the committed golden vectors from the REFERENCE build.

Runs the reference's own unmodified hot-path code (oracle/_ref/libtgref.so,
compiled from /root/reference/proj/core by oracle/Makefile) on small seeded
inputs and stores inputs + outputs in tests/golden/*.npz. The CPU tests pin the
C restatement (oracle/tg_oracle.c) to these files, and the GPU tests compare
the CUDA path against them, so neither needs /root/reference at run time.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Loss, Reference, Spec  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def f32(a):
    """Inputs are fp32-representable so the GPU path sees identical values."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def main():
    R = Reference()
    rng = np.random.default_rng(20240222)
    cases = {}
    # eval / eval_with_spatial_gradient / backprop on random grids, all orders and dims
    for dim in (2, 3):
        for order in (0, 1, 2):
            s = Spec(dim=dim, res=(7, 5, 6) if dim == 3 else (9, 7, 1), order=order)
            c = f32(rng.uniform(-1, 1, s.V * s.K))
            pts = f32(rng.uniform(-1.05, 1.05, (256, 3)))
            if dim == 2:
                pts[:, 2] = 0.0
            # vertex-aligned and boundary points (locate edge cases)
            pts[:8, 0] = [-1.0, 1.0, -0.5, 0.5, 0.0, 1.0, -1.0, 0.25]
            vals, grads = R.eval(s, c, pts, True)
            up = f32(rng.uniform(-1, 1, 256))
            uv = f32(rng.uniform(-1, 1, (256, 3)))
            if dim == 2:
                uv[:, 2] = 0.0
            g = np.zeros(s.V * s.K)
            R.backprop(s, c, pts, up, uv, g)
            key = f"d{dim}o{order}"
            cases[key] = dict(res=np.array(s.res), coeffs=c, pts=pts, vals=vals, grads=grads, up=up, uv=uv,
                              bgrad=g)
    np.savez_compressed(os.path.join(OUT, "eval_backprop.npz"),
                        **{f"{k}_{n}": v for k, d in cases.items() for n, v in d.items()})

    # total_loss + tv (paper defaults and recon-only, with/without differentiate_weight)
    loss_cases = {}
    for dim in (2, 3):
        s = Spec(dim=dim, res=(6, 6, 6) if dim == 3 else (10, 10, 1), order=2)
        c = f32(rng.uniform(-0.5, 0.5, s.V * s.K))
        pts = f32(rng.uniform(-1, 1, (300, 3)))
        if dim == 2:
            pts[:, 2] = 0.0
        vals = R.eval(s, c, pts)
        off = np.where(rng.uniform(size=300) < 0.5, -1, 1) * rng.uniform(0.05, 0.3, 300)
        gt = f32(vals + off)
        smp = np.concatenate([pts, gt[:, None]], 1)
        for name, cfg in (("paper", Loss()), ("recon", Loss(lambda1=0.0, use_tv=False)),
                          ("dw", Loss(differentiate_weight=True))):
            g = np.zeros(s.V * s.K)
            terms = R.total_loss(s, c, smp, cfg, g)
            loss_cases[f"d{dim}_{name}"] = dict(res=np.array(s.res), coeffs=c, samples=smp, terms=terms, grad=g)
        tg = np.zeros(s.V * s.K)
        tv = R.tv_loss(s, c, tg, 0.7)
        loss_cases[f"d{dim}_tv"] = dict(res=np.array(s.res), coeffs=c, tv=np.array([tv]), grad=tg)
    np.savez_compressed(os.path.join(OUT, "loss.npz"),
                        **{f"{k}_{n}": v for k, d in loss_cases.items() for n, v in d.items()})

    # Adam trajectory and a short training run (C1 shape: 2D, order 2, zero init, lr 1e-2)
    n = 64
    p = f32(rng.normal(0, 1, n))
    p0 = p.copy()
    m = np.zeros(n)
    v = np.zeros(n)
    grads = f32(rng.normal(0, 1, (20, n)))
    traj = []
    t = 0
    for k in range(20):
        t = R.adam_step(p, grads[k], m, v, t, lr=0.01)
        traj.append(p.copy())
    s = Spec(dim=2, res=(16, 16, 1), order=2)
    sys.path.insert(0, ROOT)
    batches = []
    for step in range(30):
        r2 = np.random.default_rng(1000 + step)
        pts = f32(r2.uniform(-1, 1, (512, 2)))
        q = np.zeros((512, 4))
        q[:, :2] = pts
        x, y = pts[:, 0], pts[:, 1]
        circ = np.sqrt(x * x + y * y) - 0.5
        qx, qy = np.abs(x - 0.3) - 0.3, np.abs(y + 0.2) - 0.3
        box = np.sqrt(np.maximum(qx, 0) ** 2 + np.maximum(qy, 0) ** 2) + np.minimum(np.maximum(qx, qy), 0)
        q[:, 3] = f32(np.minimum(circ, box))
        batches.append(q)
    batches = np.array(batches)
    c0 = np.zeros(s.V * s.K)
    cf, terms, _ = R.train(s, c0, batches, Loss(), lr=1e-2)
    np.savez_compressed(os.path.join(OUT, "train.npz"), adam_p0=p0, adam_grads=grads,
                        adam_traj=np.array(traj), train_res=np.array(s.res), train_batches=batches,
                        train_terms=terms, train_final=cf)
    print("golden written to", OUT)


if __name__ == "__main__":
    main()
