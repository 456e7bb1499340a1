"""Driver for ncu captures of the single-launch fused step (small.cu) at C1
(2D 128^2 order 2, 65,536 points per step): N asynchronous steps.

    ncu --set full -k regex:k_small_step -s 20 -c 1 -o out python tools/prof_small.py
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--path", type=int, default=2)
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--res", type=int, default=128)
    ap.add_argument("--points", type=int, default=1 << 16)
    a = ap.parse_args()
    import torch
    import paper_2402_14415_b200 as tg
    dim = a.dim
    g = tg.init_grid(tg.GridSpec(dim=dim, resolution=(a.res,) * dim + ((1,) if dim == 2 else ()), order=2))
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    g.set_step_path(a.path)
    shape = tg.SHAPE_C1_2D if dim == 2 else tg.SHAPE_SPHERE
    kw = {} if dim == 2 else dict(near_frac=0.5, sigma=0.01, param0=0.6)
    dev = [torch.from_numpy(tg.sample(shape, dim, 500 + i, a.points, **kw)).cuda() for i in range(2)]
    cfg = tg.LossConfig()
    for i in range(a.steps):
        tg.train_step(g, dev[i % 2], cfg, asynchronous=True, input_ready=True)
    print(g.sync())


if __name__ == "__main__":
    main()
