"""C1 small-grid step time across grid instances in one process (each earlier
grid kept alive, so later ones land at other device addresses): measured
12.1-12.4 us for most instances and 15.4-16.4 us for others on one B200 —
the step time depends on where the buffers land.

    python tools/c1_var.py [tools/pt/libtgcu_pt.so]   # instrumented: per-kernel times too
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_14415_b200 as tg  # noqa: E402

PT = len(sys.argv) > 1
if PT:
    tg.LIB_PATH = os.path.abspath(sys.argv[1])


def main():
    import torch
    dev = [torch.from_numpy(tg.sample(tg.SHAPE_C1_2D, 2, 500 + i, 1 << 16)).cuda() for i in range(2)]
    cfg = tg.LossConfig()
    keep = []
    for inst in range(12):
        g = tg.init_grid(tg.GridSpec(dim=2, resolution=(128, 128, 1), order=2))
        g.adam_reset(tg.AdamConfig(lr=1e-2))
        for i in range(200):
            tg.train_step(g, dev[i % 2], cfg, asynchronous=True, input_ready=True)
        g.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if os.environ.get("NOGC"):
            import gc
            gc.collect()
            gc.disable()
        e0.record()
        for i in range(4000):
            tg.train_step(g, dev[i % 2], cfg, asynchronous=True, input_ready=True)
        e1.record()
        torch.cuda.synchronize()
        if os.environ.get("NOGC"):
            gc.enable()
        extra = ""
        if PT:
            ring = np.zeros(1024, dtype=np.uint64)
            tg.lib().tgcu_small_ring_dump(ring.ctypes.data_as(C.c_void_p), 1)
            for i in range(200):
                tg.train_step(g, dev[i % 2], cfg, asynchronous=True, input_ready=True)
            g.sync()
            tg.lib().tgcu_small_ring_dump(ring.ctypes.data_as(C.c_void_p), 0)
            r = ring.reshape(256, 4).astype(np.float64)
            r = r[(r[:, 0] < 2**63) & (r[:, 3] > 0)]
            r = r[np.argsort(r[:, 0])]
            med = lambda x: np.median(x) / 1e3  # noqa: E731
            extra = (f" points {med(r[:, 1] - r[:, 0]):.2f} gap {med(r[:, 2] - r[:, 1]):.2f} coeffs "
                     f"{med(r[:, 3] - r[:, 2]):.2f} gap {med(r[1:, 0] - r[:-1, 3]):.2f}")
        print(inst, round(1e3 * e0.elapsed_time(e1) / 4000, 2), hex(g.device_coeffs_ptr()), extra, flush=True)
        keep.append(g)
        keep.append(torch.empty(int(1.3e6) * (inst + 1), dtype=torch.uint8, device="cuda"))


if __name__ == "__main__":
    main()
