"""fit_sdf with FreshUniform eikonal points, reference and device batch streams (smoke)."""
import sys; sys.path.insert(0, ".")
import numpy as np
import paper_2402_14415_b200 as tg
from paper_2402_14415_b200.schedule import FitOptions, fit_sdf
smp = tg.sample(tg.SHAPE_SPHERE, 3, 5, 40000, near_frac=0.5, sigma=0.01, param0=0.6)
for exact in (True, False):
    lc = tg.LossConfig(batch_size=4096, eikonal_point_source=tg.EikonalPointSource.FreshUniform)
    r = fit_sdf(smp, tg.GridSpec(dim=3, resolution=(32,) * 3, order=2), FitOptions(loss=lc, total_steps=60, exact_stream=exact))
    print("exact", exact, "final", r.report.final_loss if hasattr(r, "report") else r)
