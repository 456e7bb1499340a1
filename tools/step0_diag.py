"""C1 first-step diagnosis: the fused step's exported gradient and first Adam
update against the reference (oracle/_ref, fp64) at zero init.

    python tools/step0_diag.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_14415_b200 as tg  # noqa: E402
from oracle.pyoracle import Loss, Oracle, Reference, Spec  # noqa: E402


def main():
    b = tg.sample(tg.SHAPE_C1_2D, 2, 10_000, 1 << 16)
    spec = tg.GridSpec(dim=2, resolution=(128, 128, 1), order=2)
    s = Spec(dim=2, res=(128, 128), order=2)
    g = tg.init_grid(spec)
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    tg.train_step(g, b, tg.LossConfig(), export_grad=True)
    gg = g.grad()
    p1 = g.coeffs
    R = Reference()
    gr = np.zeros(s.V * s.K)
    R.total_loss(s, np.zeros(s.V * s.K), b.astype(np.float64), Loss(), gr, threads=8)
    mass = Oracle().total_loss_mass(s, np.zeros(s.V * s.K), b.astype(np.float64), Loss())
    pr = np.zeros(s.V * s.K)
    m, v = np.zeros_like(pr), np.zeros_like(pr)
    R.adam_step(pr, gr.copy(), m, v, 0, lr=1e-2)
    d = np.abs(gg - gr)
    print("grad: max |d|/mass", np.max(d / np.maximum(mass, 1e-300)), " median", np.median(d / np.maximum(mass, 1e-300)))
    print("grad: |g|/mass quantiles", np.quantile(np.abs(gr) / np.maximum(mass, 1e-300), [0, 0.01, 0.1, 0.5]))
    print("grad: exact zeros ref / gpu", int((gr == 0).sum()), int((gg == 0).sum()), " of", gr.size)
    dp = np.abs(p1 - pr)
    print("p1: max |d|", dp.max(), " #>1e-6", int((dp > 1e-6).sum()), " #>1e-4", int((dp > 1e-4).sum()))
    k = np.argsort(-dp)[:10]
    for i in k:
        print(f"  idx {i} ch {i % 6}: p_gpu {p1[i]:.6g} p_ref {pr[i]:.6g} g_gpu {gg[i]:.4g} g_ref {gr[i]:.4g} "
              f"mass {mass[i]:.3g}")
    # TV of p1 both ways
    for name, p in (("gpu", p1), ("ref", pr)):
        print(name, "tv(p1)", R.tv_loss(s, p))


if __name__ == "__main__":
    main()
