"""Query kernels for ncu: 512^3 grid, 2^26 uniform points, direct + brick-sorted.

    python tools/prof_query.py [--order 2] [--reps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--order", type=int, default=2)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--res", type=int, default=512)
    ap.add_argument("--points", type=int, default=1 << 26)
    args = ap.parse_args()
    import torch
    import paper_2402_14415_b200 as tg
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=(args.res,) * 3, order=args.order),
                     tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.1, seed=7, memory_cap_bytes=1 << 40))
    n = args.points
    pts = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    tg.sample_uniform_device(3, 4242, pts)
    spts = torch.empty_like(pts)
    offs = torch.empty(tg.query_brick_codes(g) + 1, dtype=torch.int64, device="cuda")
    tg.sort_points(g, pts, spts, None, offs)
    vals = torch.empty(n, dtype=torch.float32, device="cuda")
    for _ in range(args.reps):
        tg.eval_device(g, pts, vals, asynchronous=True)
        tg.eval_sorted(g, spts, offs, vals, asynchronous=True)
    torch.cuda.synchronize()
    print("ok", float(vals[:4].sum()))


if __name__ == "__main__":
    main()
