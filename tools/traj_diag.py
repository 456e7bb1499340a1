"""Loss-curve comparison of the fused GPU step with the reference (oracle/_ref)
at a BASELINE config; saves both curves for offline analysis.

    python tools/traj_diag.py c1|c2 [--steps N] [--out file.npz] [--lr 1e-2]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_14415_b200 as tg  # noqa: E402
from oracle.pyoracle import Loss, Reference, Spec  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c1", "c2"])
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--out", default="traj.npz")
    ap.add_argument("--lr", type=float, default=1e-2)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    if a.config == "c1":
        batches = [tg.sample(tg.SHAPE_C1_2D, 2, 10_000 + i, 1 << 16) for i in range(a.steps)]
        spec, s = tg.GridSpec(dim=2, resolution=(128, 128, 1), order=2), Spec(dim=2, res=(128, 128), order=2)
    else:
        batches = [tg.sample(tg.SHAPE_SPHERE, 3, 20_000 + i, 1 << 20, near_frac=0.5, sigma=0.01, param0=0.6)
                   for i in range(a.steps)]
        spec, s = tg.GridSpec(dim=3, resolution=(128, 128, 128), order=2), Spec(dim=3, res=(128, 128, 128), order=2)
    g = tg.init_grid(spec)
    g.adam_reset(tg.AdamConfig(lr=a.lr))
    for b in batches:
        tg.train_step(g, b, tg.LossConfig(), asynchronous=True)
    g.sync()
    ours = g.trace(a.steps)
    cg = g.coeffs
    R = Reference()
    cr, ref, _ = R.train(s, np.zeros(s.V * s.K), np.array(batches, dtype=np.float64), Loss(), lr=a.lr,
                         threads=a.threads)
    extra = {} if cg.size > (1 << 22) else {"coeffs_ours": cg.astype(np.float32), "coeffs_ref": cr.astype(np.float32)}
    np.savez(a.out, ours=ours, ref=ref, **extra)
    d = np.abs(ours - ref) / np.maximum(np.abs(ref), 1e-300)
    for k in [0, 1, 2, 3, 5, 10, 20, 50, 100, 200, 500, 999]:
        if k < a.steps:
            print(k, " ".join(f"{x:.3e}" for x in d[k]), " ".join(f"{x:.6g}" for x in ref[k]))
    print("max rel per term", d.max(axis=0))


if __name__ == "__main__":
    main()
