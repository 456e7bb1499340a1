"""Wall time of the unfused reference-API C2 step (zero_grad + total_loss with gradient + adam_step, each synchronous)."""
import sys, time, torch, numpy as np
sys.path.insert(0, ".")
import paper_2402_14415_b200 as tg
spec = tg.GridSpec(dim=3, resolution=(128,)*3, order=2)
g = tg.init_grid(spec); g.adam_reset(tg.AdamConfig(lr=1e-2))
b = torch.from_numpy(tg.sample(tg.SHAPE_SPHERE, 3, 1000, 1<<20, near_frac=0.5, sigma=0.01, param0=0.6)).cuda()
cfg = tg.LossConfig()
for _ in range(3):
    g.zero_grad()
    tg.total_loss(g, b, cfg); tg.adam_step(g)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20):
    g.zero_grad()
    tg.total_loss(g, b, cfg); tg.adam_step(g)
torch.cuda.synchronize()
print("unfused C2 step ms", (time.perf_counter() - t) / 20 * 1e3)
