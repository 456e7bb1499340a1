"""Where the C2 step time outside the brick kernel goes: step time with and
without the per-launch profiling events, and the kernel time they measure."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    import torch
    import paper_2402_14415_b200 as tg
    spec = tg.GridSpec(dim=3, resolution=(128,) * 3, order=2)
    g = tg.init_grid(spec)
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    bs = [torch.from_numpy(tg.sample(tg.SHAPE_SPHERE, 3, 1000 + i, 1 << 20, near_frac=0.5, sigma=0.01,
                                     param0=0.6)).cuda() for i in range(4)]
    cfg = tg.LossConfig()
    sp = torch.cuda.current_stream().cuda_stream
    for i in range(20):
        tg.train_step(g, bs[i % 4], cfg, asynchronous=True, stream=sp, input_ready=True)
    g.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 2000
    for prof in (False, True, False, True):
        torch.cuda.synchronize()
        if prof:
            g.profile_begin()
        e0.record()
        for i in range(n):
            tg.train_step(g, bs[i % 4], cfg, asynchronous=True, stream=sp, input_ready=True)
        e1.record()
        torch.cuda.synchronize()
        kms = g.profile_end()[0] / n if prof else float("nan")
        print(f"profiling events {prof}: step {e0.elapsed_time(e1) / n * 1e3:.1f} us, brick kernel {kms * 1e3:.1f} us")


if __name__ == "__main__":
    main()
