"""C1 small-grid step time across grid instances in one process (each earlier
grid kept alive, so later ones land at other device addresses): measured
12.1-12.4 us for the first six instances and 15.4-16.0 us for the next two on
one B200 — the step time depends on where the buffers land.

    python tools/c1_var.py
"""
import sys, os
sys.path.insert(0, "/root/repo")
import torch
import paper_2402_14415_b200 as tg
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
    e0.record()
    for i in range(4000):
        tg.train_step(g, dev[i % 2], cfg, asynchronous=True, input_ready=True)
    e1.record(); torch.cuda.synchronize()
    print(inst, round(1e3 * e0.elapsed_time(e1) / 4000, 2), hex(g.device_coeffs_ptr()), hex(dev[0].data_ptr()), flush=True)
    keep.append(g)
    pad = torch.empty(int(1.3e6) * (inst + 1), dtype=torch.uint8, device="cuda"); keep.append(pad)
