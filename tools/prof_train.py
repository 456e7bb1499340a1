"""Short training run for ncu captures (launch list / --set full of k_brick_step):
C2 by default; C3 = --res 256 --points 2097152 --prims; C5 = --res 512
--points 8388608 --near 0.9 --sigma 0.005 --prims.

    python tools/prof_train.py [--steps 6] [--res 128] [--points 1048576]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--res", type=int, default=128)
    ap.add_argument("--points", type=int, default=1 << 20)
    ap.add_argument("--near", type=float, default=0.5)
    ap.add_argument("--sigma", type=float, default=0.01)
    ap.add_argument("--prims", action="store_true", help="the 64-primitive SDF of C3 / C5 (seed 42)")
    args = ap.parse_args()
    import torch
    import paper_2402_14415_b200 as tg
    spec = tg.GridSpec(dim=3, resolution=(args.res,) * 3, order=2)
    g = tg.init_grid(spec, tg.InitOptions(memory_cap_bytes=1 << 40))
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    shape, p0 = (tg.SHAPE_PRIMS, 42) if args.prims else (tg.SHAPE_SPHERE, 0.6)
    batches = [torch.from_numpy(tg.sample(shape, 3, 1000 + i, args.points, near_frac=args.near,
                                          sigma=args.sigma, param0=p0)).cuda() for i in range(2)]
    sp = torch.cuda.current_stream().cuda_stream
    for i in range(args.steps):
        tg.train_step(g, batches[i % 2], tg.LossConfig(), asynchronous=True, stream=sp)
    print("loss", g.sync().total)


if __name__ == "__main__":
    main()
