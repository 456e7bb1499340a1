"""Radiance chain: parity margins on the golden cases and device throughput.

    python tools/prof_radiance.py
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2402_14415_b200 as tg  # noqa: E402
from paper_2402_14415_b200.radiance import RenderOptions, SHColorGrid, make_rays, photometric_loss, render_rays  # noqa


def margins():
    z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "radiance.npz"))
    for case in ("soft64", "soft100", "relu64"):
        p = case + "_"
        act, ns, order, deg = (int(x) for x in z[p + "meta"])
        g = tg.init_grid(tg.GridSpec(dim=3, resolution=tuple(int(r) for r in z[p + "dres"]), order=order))
        g.coeffs = z[p + "dc"]
        ss = tg.GridSpec(dim=3, resolution=tuple(int(r) for r in z[p + "sres"]), origin=tuple(z[p + "sorg"]),
                         extent=tuple(z[p + "sext"]), order=0)
        sh = SHColorGrid(ss, deg, z[p + "sc"])
        rays = make_rays(z[p + "o"], z[p + "d"], z[p + "near"], z[p + "far"])
        opts = RenderOptions(n_samples=ns, activation=act)
        cols, res = render_rays(g, sh, rays, opts)
        loss, gd, gs = photometric_loss(g, sh, rays, z[p + "gt"], opts)
        def rel(a, b):
            return float(np.max(np.abs(a - b) / (1e-4 * np.abs(b) + 1e-6 * np.abs(b).max())))
        print(case, "color maxabs", float(np.abs(cols - z[p + "colors"]).max()), "loss rel",
              abs(loss - z[p + "loss"][0]) / z[p + "loss"][0], "gd tol ratio", rel(gd, z[p + "gd"]),
              "gs tol ratio", rel(gs, z[p + "gs"]))


def throughput():
    import ctypes as C
    import torch
    from paper_2402_14415_b200.radiance import _RO
    res = 128
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=(res,) * 3, order=2),
                     tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=1.0, seed=3))
    c = g.coeffs_f32()
    c[::10] += 10.0
    g.set_coeffs_f32(c)
    deg = 2
    ss = tg.GridSpec(dim=3, resolution=(res,) * 3, order=0)
    shc = torch.randn(res ** 3 * 27, device="cuda") * 0.5
    n = 1 << 16
    rng = np.random.default_rng(0)
    o = rng.uniform(-0.9, 0.9, (n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rays = torch.from_numpy(make_rays(o, d, 0.0, 1.0)).cuda()
    gt = torch.rand((n, 3), device="cuda")
    gd = torch.zeros(g.coeff_total(), device="cuda")
    gs = torch.zeros_like(shc)
    L = tg.lib()
    ro = _RO(64, 0, -10.0, (C.c_double * 3)(1.0, 1.0, 1.0))
    loss = C.c_double()
    spec = ss._c()

    def run(grad):
        tg._check(L.tgcu_photometric_loss(g.handle, C.byref(spec), deg, C.c_void_p(shc.data_ptr()),
                                          C.c_void_p(rays.data_ptr()), C.c_void_p(gt.data_ptr()), n,
                                          C.cast(C.pointer(ro), C.c_void_p),
                                          None, None, C.c_void_p(gd.data_ptr()) if grad else None,
                                          C.c_void_p(gs.data_ptr()) if grad else None, C.byref(loss), 0, None))
    for grad in (False, True):
        run(grad)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            run(grad)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / 5 * 1e3
        print(f"grad={grad}: {ms:.2f} ms per {n} rays x 64 samples = {n * 64 / ms / 1e6:.2f} G samples/s")


if __name__ == "__main__":
    if "--no-margins" not in sys.argv:
        margins()
    throughput()
