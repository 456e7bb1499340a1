"""Two-rank SlabTrainer run (fused halo) vs a single grid, printing the per-step term differences."""
import sys, os, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_slab_driver_gpu as T
import torch.multiprocessing as mp
import paper_2402_14415_b200 as tg
out='/tmp/slabdiag'; os.makedirs(out, exist_ok=True)
mp.spawn(T._rank, args=(2, T._port(), out, True), nprocs=2, join=True)
spec = tg.GridSpec(dim=3, resolution=T.RES, order=2)
g = tg.init_grid(spec, tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.02, seed=11))
g.adam_reset(tg.AdamConfig(lr=1e-2))
ref = np.array([tg.train_step(g, b).as_array() for b in T._batches()])
own = np.concatenate([np.load(out+'/own0.npy'), np.load(out+'/own1.npy')])
full = g.coeffs
d = np.abs(own-full); bad = d > 1e-5*np.maximum(np.abs(full),1e-2)
print("bad", bad.sum(), "max diff", d.max())
K=10; idx=np.where(bad)[0]; v=idx//K
print("z planes", np.unique(v//(32*24))[:20], "ch", np.bincount(idx%K))
for r in range(2): print(np.load(out+f'/terms{r}.npy')[:, 0] - ref[:, 0])
