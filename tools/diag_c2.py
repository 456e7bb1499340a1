"""Diagnose C2-scale fused / unfused gradient parity failures."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_14415_b200 as tg  # noqa: E402
from oracle.pyoracle import Loss, Oracle, Spec  # noqa: E402

res = (128, 128, 128)
s = Spec(dim=3, res=res, order=2)
O = Oracle()
rng = np.random.default_rng(11)
c = (0.01 * rng.standard_normal(s.V * s.K)).astype(np.float32)
smp = tg.sample(tg.SHAPE_SPHERE, 3, 99, 1 << 20, near_frac=0.5, sigma=0.01, param0=0.6)
g = tg.init_grid(tg.GridSpec(dim=3, resolution=res, order=2))
g.set_coeffs_f32(c)
g.adam_reset(tg.AdamConfig(lr=1e-2))
t = tg.train_step(g, smp, tg.LossConfig(), export_grad=True)
gf = g.grad()
g2 = tg.init_grid(tg.GridSpec(dim=3, resolution=res, order=2))
g2.set_coeffs_f32(c)
g2.zero_grad()
t2 = tg.total_loss(g2, smp, tg.LossConfig())
gu = g2.grad()
gref = np.zeros(s.V * s.K)
c64, s64 = c.astype(np.float64), smp.astype(np.float64)
tref = O.total_loss(s, c64, s64, Loss(), gref)
mass = O.total_loss_mass(s, c64, s64, Loss())
print("terms fused", t.as_array(), "\nterms unfused", t2.as_array(), "\nterms ref", tref)
for name, got in (("fused", gf), ("unfused", gu)):
    tol = 1e-5 * np.abs(gref) + 2e-6 * mass + 1e-300
    err = np.abs(got - gref)
    bad = np.where(err > tol)[0]
    print(name, "bad", len(bad), "max ratio", float(np.max(err / tol)))
    if len(bad):
        ch = bad % 10
        print("  channels", np.bincount(ch, minlength=10))
        v = bad // 10
        x, y, z = v % 128, (v // 128) % 128, v // (128 * 128)
        print("  x mod 8", np.bincount(x % 8, minlength=8), "y mod 8", np.bincount(y % 8, minlength=8),
              "z mod 8", np.bincount(z % 8, minlength=8))
        idx = bad[np.argsort(-(err[bad] / tol[bad]))[:8]]
        for i in idx:
            print(f"  i={i} v=({i//10%128},{i//1280%128},{i//163840}) ch={i%10} ref={gref[i]:.6e} got={got[i]:.6e} "
                  f"mass={mass[i]:.3e} ratio={err[i]/tol[i]:.2f}")
