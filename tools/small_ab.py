"""A/B of the fused-step paths (tgcu_grid_set_step_path) on small grids:
device time per step over a long window, host enqueue time per call, and a
one-step parity check of each path against the fp64 oracle.

    python tools/small_ab.py [--steps 4000] [--grids c1,3d32,3d48]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

GRIDS = {
    "c1": (2, (128, 128, 1), 1 << 16),
    "2d256": (2, (256, 256, 1), 1 << 16),
    "3d32": (3, (32, 32, 32), 1 << 16),
    "3d48": (3, (48, 48, 48), 1 << 17),
    "3d64": (3, (64, 64, 64), 1 << 18),
    "c2": (3, (128, 128, 128), 1 << 20),
    "3d64n20": (3, (64, 64, 64), 1 << 20),
    "3d96n18": (3, (96, 96, 96), 1 << 18),
    "3d96n20": (3, (96, 96, 96), 1 << 20),
    "2d256n18": (2, (256, 256, 1), 1 << 18),
    "2d512n18": (2, (512, 512, 1), 1 << 18),
    "2d512n20": (2, (512, 512, 1), 1 << 20),
    "2d1024n20": (2, (1024, 1024, 1), 1 << 20),
}


def time_path(tg, torch, dim, res, n, path, steps):
    g = tg.init_grid(tg.GridSpec(dim=dim, resolution=res, order=2))
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    g.set_step_path(path)
    shape = tg.SHAPE_C1_2D if dim == 2 else tg.SHAPE_SPHERE
    kw = {} if dim == 2 else dict(near_frac=0.5, sigma=0.01, param0=0.6)
    dev = [torch.from_numpy(tg.sample(shape, dim, 500 + i, n, **kw)).cuda() for i in range(2)]
    cfg = tg.LossConfig()
    for i in range(100):
        tg.train_step(g, dev[i % 2], cfg, asynchronous=True, input_ready=True)
    g.sync()
    # host cost per call while the launch queue is not yet full
    h0 = time.perf_counter()
    for i in range(100):
        tg.train_step(g, dev[i % 2], cfg, asynchronous=True, input_ready=True)
    host_free = 1e6 * (time.perf_counter() - h0) / 100
    g.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for i in range(steps):
        tg.train_step(g, dev[i % 2], cfg, asynchronous=True, input_ready=True)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    last = g.sync()
    return 1e3 * e0.elapsed_time(e1) / steps, 1e6 * (t1 - t0) / steps, last.total, host_free


def parity(tg, oracle_mod, dim, res, n, path):
    import numpy as np
    from oracle.pyoracle import Loss, Spec
    O = oracle_mod
    rng = np.random.default_rng(7)
    s = Spec(dim=dim, res=res, order=2)
    c = (0.1 * rng.standard_normal(s.V * s.K)).astype(np.float32).astype(np.float64)
    shape = tg.SHAPE_C1_2D if dim == 2 else tg.SHAPE_SPHERE
    kw = {} if dim == 2 else dict(near_frac=0.5, sigma=0.01, param0=0.6)
    smp = tg.sample(shape, dim, 99, n, **kw).astype(np.float64)
    gref = np.zeros(s.V * s.K)
    tref = O.total_loss(s, c, smp, Loss(), gref)
    g = tg.init_grid(tg.GridSpec(dim=dim, resolution=res, order=2))
    g.set_step_path(path)
    g.coeffs = c
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    t = tg.train_step(g, smp, tg.LossConfig(), export_grad=True)
    terr = np.max(np.abs(t.as_array() - tref) / np.maximum(np.abs(tref), 1e-30))
    gd = g.grad()
    floor = 1e-3 * np.max(np.abs(gref))
    gerr = np.max(np.abs(gd - gref) / np.maximum(np.abs(gref), floor))
    return terr, gerr


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=4000)
    ap.add_argument("--grids", default="c1,3d32,3d48")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--paths", default="brick,single")
    a = ap.parse_args()
    import torch
    import paper_2402_14415_b200 as tg
    from oracle.pyoracle import Oracle
    O = Oracle()
    for name in a.grids.split(","):
        dim, res, n = GRIDS[name]
        pmap = {"brick": tg.TaylorGrid.STEP_BRICK, "single": tg.TaylorGrid.STEP_SINGLE}
        for pname in a.paths.split(","):
            path = pmap[pname]
            dev_us, host_us, loss, host_free = time_path(tg, torch, dim, res, n, path, a.steps)
            terr, gerr = (0.0, 0.0) if a.no_parity else parity(tg, O, dim, res, min(n, 1 << 15), path)
            print(f"{name:6s} {pname:6s} device {dev_us:7.2f} us/step  host {host_us:6.2f} us/call "
                  f"(queue not full: {host_free:6.2f})  "
                  f"loss {loss:.6g}  terms rel {terr:.2e}  grad rel {gerr:.2e}", flush=True)


if __name__ == "__main__":
    main()
