"""CPU-side checks of the product library (no GPU needed):

* libtgcu.so loads and exports every entry point include/tgcu.h declares;
* without a device the compute path fails loudly (no CPU fallback);
* the host-side seeded input generator reproduces the reference Rng streams
  and the reference sampler (sample_sphere_points, sampling.cpp:140-159).
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2402_14415_b200 as tg
from conftest import ROOT


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "tgcu.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(tgcu_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(tg.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert missing == []


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(tg.CudaError, match="no CUDA device"):
        tg.init_grid(tg.GridSpec(dim=3, resolution=(4, 4, 4), order=2))


def test_spec_validation_precedes_device():
    with pytest.raises(ValueError, match="dim must be 2 or 3"):
        tg.init_grid(tg.GridSpec(dim=4, resolution=(4, 4, 4), order=2))
    with pytest.raises(ValueError, match="resolution must be >= 2"):
        tg.init_grid(tg.GridSpec(dim=3, resolution=(1, 4, 4), order=2))
    with pytest.raises(tg.ResourceError, match="exceeds memory cap"):
        tg.init_grid(tg.GridSpec(dim=3, resolution=(64, 64, 64), order=2), tg.InitOptions(memory_cap_bytes=1024))


def test_coeff_count():
    assert [tg.coeff_count(o, d) for o, d in [(2, 3), (0, 3), (2, 2), (1, 3), (1, 2), (0, 2)]] == [10, 1, 6, 4, 3, 1]
    with pytest.raises(ValueError):
        tg.coeff_count(3, 3)


def test_sampler_matches_reference_sphere(reference):
    # 50% uniform / 50% near-surface sphere points == sample_sphere_points(r, {1,1,0}, sigma)
    n = 4096
    ours = tg.sample(tg.SHAPE_SPHERE, 3, 1234, n, near_frac=0.5, sigma=0.01, param0=0.6)
    ref = reference.sample_sphere(0.6, n, ratio=(1, 1, 0), sigma_near=0.01, seed=1234)
    assert np.array_equal(ours[:, :3], ref[:, :3].astype(np.float32))
    gt = np.linalg.norm(ours[:, :3].astype(np.float64), axis=1) - 0.6
    assert np.array_equal(ours[:, 3], gt.astype(np.float32))
    assert np.max(np.abs(ours[:, 3] - ref[:, 3])) < 1e-6


def test_sampler_shapes_and_determinism():
    a = tg.sample(tg.SHAPE_C1_2D, 2, 7, 1000)
    b = tg.sample(tg.SHAPE_C1_2D, 2, 7, 1000)
    assert np.array_equal(a, b)
    assert np.all(np.abs(a[:, :2]) <= 1.0) and np.all(a[:, 2] == 0)
    # circle ∪ box analytic SDF
    x, y = a[:, 0].astype(np.float64), a[:, 1].astype(np.float64)
    circ = np.sqrt(x * x + y * y) - 0.5
    qx, qy = np.abs(x - 0.3) - 0.3, np.abs(y + 0.2) - 0.3
    box = np.sqrt(np.maximum(qx, 0) ** 2 + np.maximum(qy, 0) ** 2) + np.minimum(np.maximum(qx, qy), 0)
    assert np.allclose(a[:, 3], np.minimum(circ, box), atol=1e-6)
    p = tg.sample(tg.SHAPE_PRIMS, 3, 11, 20000, near_frac=0.9, sigma=0.005, param0=42)
    near = p[2000:]
    assert np.median(np.abs(near[:, 3])) < 0.02  # near-surface samples hug the union's surface
    assert np.all(np.abs(p[:, :3]) <= 1.0)
