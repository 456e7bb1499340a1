"""Mean device time per segment of the C2 fused step (tgcu_step_breakdown).

    python tools/step_breakdown.py [steps]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2402_14415_b200 as tg  # noqa: E402


def main():
    import torch
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=(128,) * 3, order=2))
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    bs = [torch.from_numpy(tg.sample(tg.SHAPE_SPHERE, 3, 1000 + i, 1 << 20, near_frac=0.5, sigma=0.01,
                                     param0=0.6)).cuda() for i in range(4)]
    for i in range(20):
        tg.train_step(g, bs[i % 4], asynchronous=True)
    g.sync()
    L = tg.lib()
    L.tgcu_step_breakdown.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    out = (C.c_double * 5)()
    n = C.c_int()
    L.tgcu_step_breakdown(g.handle, 1, out, C.byref(n))
    for i in range(steps):
        tg.train_step(g, bs[i % 4], asynchronous=True)
    g.sync()
    L.tgcu_step_breakdown(g.handle, 0, out, C.byref(n))
    names = ["bin histogram", "bin column pass", "bin scatter", "brick kernel", "finalize"]
    tot = sum(out)
    for k, v in zip(names, out):
        print(f"{k:18s} {v * 1e3:8.1f} us  {100 * v / tot:5.1f} %")
    print(f"{'sum':18s} {tot * 1e3:8.1f} us over {n.value} steps")


if __name__ == "__main__":
    main()
