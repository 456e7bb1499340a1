"""Launch timeline of the small-grid fused step (small.cu) from the
instrumented build (tools/build_pt.sh -> tools/pt/libtgcu_pt.so): per step,
the first CTA start and last CTA end of k_small_points and k_small_coeffs.

    python tools/small_phase.py tools/pt/libtgcu_pt.so [--dim 2 --res 128 --points 65536]
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2402_14415_b200 as tg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lib")
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--res", type=int, default=128)
    ap.add_argument("--points", type=int, default=1 << 16)
    a = ap.parse_args()
    tg.LIB_PATH = os.path.abspath(a.lib)
    import torch
    dim = a.dim
    g = tg.init_grid(tg.GridSpec(dim=dim, resolution=(a.res,) * dim + ((1,) if dim == 2 else ()), order=2))
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    g.set_step_path(2)
    shape = tg.SHAPE_C1_2D if dim == 2 else tg.SHAPE_SPHERE
    kw = {} if dim == 2 else dict(near_frac=0.5, sigma=0.01, param0=0.6)
    dev = torch.from_numpy(tg.sample(shape, dim, 500, a.points, **kw)).cuda()
    cfg = tg.LossConfig()
    for i in range(300):
        tg.train_step(g, dev, cfg, asynchronous=True, input_ready=True)
    g.sync()
    ring = np.zeros(1024, dtype=np.uint64)
    tg.lib().tgcu_small_ring_dump(ring.ctypes.data_as(C.c_void_p), 1)
    for i in range(200):
        tg.train_step(g, dev, cfg, asynchronous=True, input_ready=True)
    g.sync()
    tg.lib().tgcu_small_ring_dump(ring.ctypes.data_as(C.c_void_p), 0)
    r = ring.reshape(256, 4).astype(np.float64)
    r = r[(r[:, 0] < 2**63) & (r[:, 3] > 0)]
    r = r[np.argsort(r[:, 0])]
    us = lambda x: np.median(x) / 1e3  # noqa: E731
    print(f"{len(r)} steps: points kernel {us(r[:, 1] - r[:, 0]):.2f} us, gap {us(r[:, 2] - r[:, 1]):.2f} us, "
          f"coeffs kernel {us(r[:, 3] - r[:, 2]):.2f} us, gap to next step {us(r[1:, 0] - r[:-1, 3]):.2f} us; "
          f"{(r[-1, 3] - r[0, 0]) / 1e3 / len(r):.2f} us per step")


if __name__ == "__main__":
    main()
