"""C1 step: host enqueue time per tgcu_train_step call vs device time per step.

    python tools/c1_host.py [--steps 2000]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2000)
    args = ap.parse_args()
    import torch
    import paper_2402_14415_b200 as tg
    g = tg.init_grid(tg.GridSpec(dim=2, resolution=(128, 128, 1), order=2))
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    bs = [torch.from_numpy(tg.sample(tg.SHAPE_C1_2D, 2, 10_000 + i, 1 << 16)).cuda() for i in range(4)]
    cfg = tg.LossConfig()
    for i in range(50):
        tg.train_step(g, bs[i % 4], cfg, asynchronous=True, input_ready=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for i in range(args.steps):
        tg.train_step(g, bs[i % 4], cfg, asynchronous=True, input_ready=True)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host enqueue {1e6 * (t1 - t0) / args.steps:.1f} us/step, device {1e3 * e0.elapsed_time(e1) / args.steps:.1f} "
          f"us/step, wall {1e6 * (t2 - t0) / args.steps:.1f} us/step")


if __name__ == "__main__":
    main()
