"""Unsorted 2^26-point query on 512^3 order 2 through the binned path (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2402_14415_b200 as tg
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=(512,) * 3, order=int(sys.argv[1]) if len(sys.argv) > 1 else 2),
                     tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.1, seed=7, memory_cap_bytes=1 << 40))
    n = 1 << 26
    pts = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    tg.sample_uniform_device(3, 4242, pts)
    vals = torch.empty(n, dtype=torch.float32, device="cuda")
    for _ in range(3):
        tg.eval_device(g, pts, vals, asynchronous=True)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
