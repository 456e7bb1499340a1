"""Per-CTA phase timing of the fused brick kernel (instrumented build).

    nvcc ... -DTGCU_PHASE_TIMING train.cu -> tools/pt/libtgcu_pt.so
    python tools/phase_timing.py tools/pt/libtgcu_pt.so

Runs C2 steps, then reads thread 0's %globaltimer stamps of the last launch:
tile wait, point forward+loss (2a), cell scan, records + workload balance,
gather (2b), epilogue (TV + Adam + stores + partials), per CTA.
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2402_14415_b200 as tg  # noqa: E402

tg.LIB_PATH = os.path.abspath(sys.argv[1])


def main():
    import torch
    # argv[2] = "c3": 256^3, 2^21 points of the 64-primitive SDF (50 % near, sigma 0.01); default C2
    c3 = len(sys.argv) > 2 and sys.argv[2] == "c3"
    res = 256 if c3 else 128
    spec = tg.GridSpec(dim=3, resolution=(res,) * 3, order=2)
    g = tg.init_grid(spec)
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    if c3:
        host = [tg.sample(tg.SHAPE_PRIMS, 3, 500 + i, 1 << 21, near_frac=0.5, sigma=0.01, param0=42) for i in range(2)]
    else:
        host = [tg.sample(tg.SHAPE_SPHERE, 3, 1000 + i, 1 << 20, near_frac=0.5, sigma=0.01, param0=0.6)
                for i in range(4)]
    batches = [torch.from_numpy(h).cuda() for h in host]
    for i in range(40):
        tg.train_step(g, batches[i % len(batches)], asynchronous=True)
    g.sync()
    nb = (res // 8) ** 3
    ph = np.zeros(nb * 12, dtype=np.uint64)
    L = tg.lib()
    L.tgcu_phase_dump.argtypes = [C.c_void_p, C.c_int]
    assert L.tgcu_phase_dump(ph.ctypes.data_as(C.c_void_p), nb) == 0
    ph = ph.reshape(nb, 12).astype(np.float64)
    start, tile, a2, scan, bal, b2, epi, end, npts, e1, e2 = (ph[:, i] for i in range(11))
    t0 = start.min()
    dur = end - start
    span = end.max() - t0
    has = npts > 0
    tilew = np.where(has, tile - start, 0)
    epid = end - epi
    print(f"kernel span {span / 1e3:.1f} us, CTAs {nb}, mean CTA {dur.mean() / 1e3:.2f} us, "
          f"concurrency {dur.sum() / span:.1f}")
    tot = dur.sum()
    for name, v in (("tile wait (start->tile ready)", tilew), ("2a fwd+loss (excl. tile wait)", a2 - tilew),
                    ("cell scan", scan), ("records + balance", bal), ("2b gather + chunk barrier", b2),
                    ("epilogue (TV+Adam+store+partials)", epid)):
        print(f"  {name:38s} {v.sum() / tot * 100:5.1f} %   mean {v.mean() / 1e3:6.2f} us")
    other = tot - (tilew.sum() + (a2 - tilew).sum() + scan.sum() + bal.sum() + b2.sum() + epid.sum())
    print(f"  {'other (setup, chunk starts)':38s} {other / tot * 100:5.1f} %")
    print(f"  epilogue split: G store + m/v wait {(e1 - epi).mean() / 1e3:.2f} us, TV + Adam {(e2 - e1).mean() / 1e3:.2f} us, "
          f"store issue + partials + drain {(end - e2).mean() / 1e3:.2f} us")
    chunks = np.ceil(npts / 512)
    for c in sorted(set(chunks.astype(int))):
        sel = chunks == c
        print(f"  {int(c)} chunk(s): {sel.sum():5d} CTAs, mean {dur[sel].mean() / 1e3:6.2f} us, "
              f"2b {b2[sel].mean() / 1e3:6.2f} us, 2a {a2[sel].mean() / 1e3:6.2f} us, epi {epid[sel].mean() / 1e3:5.2f} us")


if __name__ == "__main__":
    main()
