"""TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.

ctypes bindings for the two CPU checkers built by oracle/Makefile:

* ``Oracle``    — oracle/libtgoracle.so, the plain-C fp64 restatement
                  (tg_oracle.c) of the reference hot path;
* ``Reference`` — oracle/_ref/libtgref.so, the reference's own unmodified
                  sources (/root/reference/proj/core) + ref_shim.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module, and only as the checker or the
timed CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_L = C.POINTER(C.c_int64)


def _dp(a):
    return None if a is None else a.ctypes.data_as(_D)


@dataclass
class Spec:
    """Mirror of tg::GridSpec (grid_spec.hpp:19-24)."""
    dim: int = 3
    res: tuple = (2, 2, 2)
    origin: tuple = (-1.0, -1.0, -1.0)
    extent: tuple = (2.0, 2.0, 2.0)
    order: int = 2

    @property
    def K(self) -> int:
        return {0: 1, 1: 1 + self.dim, 2: 1 + self.dim + self.dim * (self.dim + 1) // 2}[self.order]

    @property
    def V(self) -> int:
        n = 1
        for a in range(self.dim):
            n *= self.res[a]
        return n

    def spacing(self, a):
        return self.extent[a] / (self.res[a] - 1)


class _TgoSpec(C.Structure):
    _fields_ = [("dim", C.c_int), ("res", C.c_int * 3), ("origin", C.c_double * 3),
                ("extent", C.c_double * 3), ("order", C.c_int)]


class _TgoLoss(C.Structure):
    _fields_ = [("lambda1", C.c_double), ("lambda2", C.c_double), ("k", C.c_double),
                ("use_weighting", C.c_int), ("use_tv", C.c_int), ("differentiate_weight", C.c_int)]


@dataclass
class Loss:
    """Mirror of tg::LossConfig (sdf_loss.hpp:15-25), reuse-batch eikonal."""
    lambda1: float = 1e-4
    lambda2: float = 2e-5
    k: float = 50.0
    use_weighting: bool = True
    use_tv: bool = True
    differentiate_weight: bool = False


def _spec_args(s: Spec):
    res = (C.c_int * 3)(*[int(r) for r in (list(s.res) + [1, 1, 1])[:3]])
    org = (C.c_double * 3)(*[float(x) for x in (list(s.origin) + [0, 0, 0])[:3]])
    ext = (C.c_double * 3)(*[float(x) for x in (list(s.extent) + [1, 1, 1])[:3]])
    return s.dim, res, org, ext, s.order


class Oracle:
    """The C restatement (tg_oracle.c)."""

    def __init__(self, path=None):
        path = path or os.path.join(HERE, "libtgoracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"oracle not built: {path} (run make -C oracle)")
        L = C.CDLL(path)
        L.tgo_eval.restype = C.c_double
        L.tgo_eval.argtypes = [C.POINTER(_TgoSpec), _D, _D, _D]
        L.tgo_locate.argtypes = [C.POINTER(_TgoSpec), _D, _I, _D, _L]
        L.tgo_backprop.argtypes = [C.POINTER(_TgoSpec), _D, C.c_double, _D, _D]
        L.tgo_adaptive_weight.restype = C.c_double
        L.tgo_adaptive_weight.argtypes = [C.c_double] * 3
        L.tgo_tv_loss.restype = C.c_double
        L.tgo_tv_loss.argtypes = [C.POINTER(_TgoSpec), _D, _D, C.c_double]
        L.tgo_total_loss.argtypes = [C.POINTER(_TgoSpec), _D, _D, C.c_int64, C.POINTER(_TgoLoss), _D, _D]
        L.tgo_adam_step.restype = C.c_int64
        L.tgo_adam_step.argtypes = [_D, _D, _D, _D, C.c_int64, _L] + [C.c_double] * 4
        L.tgo_multilinear_resample.argtypes = [C.POINTER(_TgoSpec), _D, C.c_int, _I, _D]
        L.tgo_coeff_count.argtypes = [C.c_int, C.c_int]
        L.tgo_backprop_mass.argtypes = [C.POINTER(_TgoSpec), _D, C.c_double, _D, _D]
        L.tgo_total_loss_mass.argtypes = [C.POINTER(_TgoSpec), _D, _D, C.c_int64, C.POINTER(_TgoLoss), _D]
        L.tgo_markstein_div.restype = C.c_double
        L.tgo_markstein_div.argtypes = [C.c_double] * 3
        self.L = L

    @staticmethod
    def _spec(s: Spec):
        d, res, org, ext, o = _spec_args(s)
        return _TgoSpec(d, res, org, ext, o)

    def coeff_count(self, order, dim):
        return self.L.tgo_coeff_count(order, dim)

    def locate(self, s: Spec, p):
        cell = (C.c_int * 3)()
        loc = (C.c_double * 3)()
        vid = (C.c_int64 * 8)()
        pp = np.ascontiguousarray(list(p) + [0.0] * (3 - len(p)), dtype=np.float64)
        rc = self.L.tgo_locate(C.byref(self._spec(s)), _dp(pp), cell, loc, vid)
        if rc != 0:
            raise ValueError("locate: NaN coordinate")
        return list(cell), list(loc), list(vid)

    def eval(self, s: Spec, coeffs, pts, want_grad=False):
        sp = self._spec(s)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        vals = np.empty(len(pts))
        grads = np.zeros((len(pts), 3)) if want_grad else None
        g3 = (C.c_double * 3)()
        for i in range(len(pts)):
            vals[i] = self.L.tgo_eval(C.byref(sp), _dp(coeffs), _dp(pts[i]), g3 if want_grad else None)
            if want_grad:
                grads[i] = list(g3)
        return (vals, grads) if want_grad else vals

    def backprop(self, s: Spec, pts, upstream, upstream_vec, grad):
        sp = self._spec(s)
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        uv = np.ascontiguousarray(upstream_vec, dtype=np.float64).reshape(-1, 3)
        for i in range(len(pts)):
            self.L.tgo_backprop(C.byref(sp), _dp(pts[i]), float(upstream[i]), _dp(uv[i]), _dp(grad))
        return grad

    def adaptive_weight(self, a, b, k):
        return self.L.tgo_adaptive_weight(a, b, k)

    def backprop_mass(self, s: Spec, pts, upstream, upstream_vec):
        sp = self._spec(s)
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        uv = np.ascontiguousarray(upstream_vec, dtype=np.float64).reshape(-1, 3)
        mass = np.zeros(s.V * s.K)
        for i in range(len(pts)):
            self.L.tgo_backprop_mass(C.byref(sp), _dp(pts[i]), float(upstream[i]), _dp(uv[i]), _dp(mass))
        return mass

    def total_loss_mass(self, s: Spec, coeffs, samples, cfg: Loss):
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        samples = np.ascontiguousarray(samples, dtype=np.float64).reshape(-1, 4)
        lc = _TgoLoss(cfg.lambda1, cfg.lambda2, cfg.k, int(cfg.use_weighting), int(cfg.use_tv),
                      int(cfg.differentiate_weight))
        mass = np.zeros(s.V * s.K)
        self.L.tgo_total_loss_mass(C.byref(self._spec(s)), _dp(coeffs), _dp(samples), len(samples),
                                   C.byref(lc), _dp(mass))
        return mass

    def tv_loss(self, s: Spec, coeffs, grad=None, scale=1.0):
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        return self.L.tgo_tv_loss(C.byref(self._spec(s)), _dp(coeffs), _dp(grad), scale)

    def total_loss(self, s: Spec, coeffs, samples, cfg: Loss, grad=None):
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        samples = np.ascontiguousarray(samples, dtype=np.float64).reshape(-1, 4)
        lc = _TgoLoss(cfg.lambda1, cfg.lambda2, cfg.k, int(cfg.use_weighting), int(cfg.use_tv),
                      int(cfg.differentiate_weight))
        terms = np.zeros(4)
        self.L.tgo_total_loss(C.byref(self._spec(s)), _dp(coeffs), _dp(samples), len(samples),
                              C.byref(lc), _dp(grad), _dp(terms))
        return terms

    def adam_step(self, p, g, m, v, t, lr=0.003, beta1=0.9, beta2=0.999, eps=1e-8):
        """In place. Returns (t, bad_index or -1)."""
        tt = C.c_int64(t)
        bad = self.L.tgo_adam_step(_dp(p), _dp(g), _dp(m), _dp(v), len(p), C.byref(tt), lr, beta1,
                                   beta2, eps)
        return tt.value, bad

    def train(self, s: Spec, coeffs, batches, cfg: Loss, lr, beta1=0.9, beta2=0.999, eps=1e-8):
        """cmd_bench-shaped loop: zero grad → total_loss → adam (tools/main.cpp:639-644)."""
        p = np.array(coeffs, dtype=np.float64)
        m = np.zeros_like(p)
        v = np.zeros_like(p)
        g = np.zeros_like(p)
        t = 0
        terms = []
        for b in batches:
            g[:] = 0.0
            tr = self.total_loss(s, p, b, cfg, g)
            if not np.isfinite(tr[0]):
                raise FloatingPointError(f"run_schedule: non-finite loss at stage 0 step {len(terms)}")
            t, bad = self.adam_step(p, g, m, v, t, lr, beta1, beta2, eps)
            if bad >= 0:
                raise FloatingPointError(f"adam_step: non-finite gradient at parameter index {bad}")
            terms.append(tr)
        return p, np.array(terms)

    def resample(self, s: Spec, data, channels, new_res):
        nr = (C.c_int * 3)(*[int(r) for r in (list(new_res) + [1, 1, 1])[:3]])
        n = 1
        for a in range(s.dim):
            n *= nr[a]
        out = np.zeros(n * channels)
        data = np.ascontiguousarray(data, dtype=np.float64)
        self.L.tgo_multilinear_resample(C.byref(self._spec(s)), _dp(data), channels, nr, _dp(out))
        return out


class Reference:
    """The reference's own code (oracle/_ref/libtgref.so)."""

    def __init__(self, path=None):
        path = path or os.path.join(HERE, "_ref", "libtgref.so")
        if not os.path.exists(path):
            raise RuntimeError(f"reference build absent: {path}")
        L = C.CDLL(path)
        L.tgr_last_error.restype = C.c_char_p
        L.tgr_adaptive_weight.restype = C.c_double
        L.tgr_adaptive_weight.argtypes = [C.c_double] * 3
        L.tgr_coeff_count.argtypes = [C.c_int, C.c_int]
        sp = [C.c_int, _I, _D, _D, C.c_int]
        L.tgr_locate.argtypes = sp + [_D, _I, _D, _L]
        L.tgr_eval.argtypes = sp + [_D, _D, C.c_int64, _D, _D]
        L.tgr_backprop.argtypes = sp + [_D, _D, _D, _D, C.c_int64, _D]
        L.tgr_tv_loss.argtypes = sp + [_D, _D, C.c_double, C.c_int, _D]
        L.tgr_total_loss.argtypes = sp + [_D, _D, C.c_int64, C.c_double, C.c_double, C.c_double,
                                          C.c_int, C.c_int, C.c_int, _D, C.c_int, _D]
        L.tgr_adam_step.argtypes = [_D, _D, _D, _D, C.c_int64, _L] + [C.c_double] * 4 + [C.c_int]
        L.tgr_train.argtypes = sp + [_D, _D, C.c_int64, C.c_int, C.c_double, C.c_double, C.c_double,
                                     C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                     C.c_double, C.c_int, _D, _D]
        L.tgr_eval_timed.argtypes = sp + [_D, _D, C.c_int64, _D, C.c_int, _D]
        L.tgr_sample_sphere.argtypes = [C.c_double, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_double,
                                        C.c_uint64, _D]
        L.tgr_rng_uniform.argtypes = [C.c_uint64, C.c_int64, _D]
        L.tgr_rng_gaussian.argtypes = [C.c_uint64, C.c_int64, _D]
        L.tgr_upsample.argtypes = sp + [_D, _I, _D]
        self.L = L

    def _err(self, rc):
        if rc != 0:
            msg = self.L.tgr_last_error().decode()
            if rc == 4:
                raise FloatingPointError(msg)
            raise ValueError(msg)

    def coeff_count(self, order, dim):
        r = self.L.tgr_coeff_count(order, dim)
        if r < 0:
            raise ValueError(self.L.tgr_last_error().decode())
        return r

    def locate(self, s: Spec, p):
        cell = (C.c_int * 3)()
        loc = (C.c_double * 3)()
        vid = (C.c_int64 * 8)()
        pp = np.ascontiguousarray(list(p) + [0.0] * (3 - len(p)), dtype=np.float64)
        self._err(self.L.tgr_locate(*_spec_args(s), _dp(pp), cell, loc, vid))
        return list(cell), list(loc), list(vid)

    def eval(self, s: Spec, coeffs, pts, want_grad=False):
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        vals = np.empty(len(pts))
        grads = np.zeros((len(pts), 3)) if want_grad else None
        self._err(self.L.tgr_eval(*_spec_args(s), _dp(coeffs), _dp(pts), len(pts), _dp(vals), _dp(grads)))
        return (vals, grads) if want_grad else vals

    def eval_timed(self, s: Spec, coeffs, pts, threads):
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        vals = np.empty(len(pts))
        secs = C.c_double()
        self._err(self.L.tgr_eval_timed(*_spec_args(s), _dp(coeffs), _dp(pts), len(pts), _dp(vals),
                                        threads, C.byref(secs)))
        return vals, secs.value

    def backprop(self, s: Spec, coeffs, pts, upstream, upstream_vec, grad):
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        up = np.ascontiguousarray(upstream, dtype=np.float64)
        uv = np.ascontiguousarray(upstream_vec, dtype=np.float64).reshape(-1, 3)
        self._err(self.L.tgr_backprop(*_spec_args(s), _dp(coeffs), _dp(pts), _dp(up), _dp(uv), len(pts), _dp(grad)))
        return grad

    def adaptive_weight(self, a, b, k):
        return self.L.tgr_adaptive_weight(a, b, k)

    def tv_loss(self, s: Spec, coeffs, grad=None, scale=1.0, threads=1):
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = C.c_double()
        self._err(self.L.tgr_tv_loss(*_spec_args(s), _dp(coeffs), _dp(grad), scale, threads, C.byref(out)))
        return out.value

    def total_loss(self, s: Spec, coeffs, samples, cfg: Loss, grad=None, threads=1):
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        samples = np.ascontiguousarray(samples, dtype=np.float64).reshape(-1, 4)
        terms = np.zeros(4)
        self._err(self.L.tgr_total_loss(*_spec_args(s), _dp(coeffs), _dp(samples), len(samples),
                                        cfg.lambda1, cfg.lambda2, cfg.k, int(cfg.use_weighting),
                                        int(cfg.use_tv), int(cfg.differentiate_weight), _dp(grad),
                                        threads, _dp(terms)))
        return terms

    def adam_step(self, p, g, m, v, t, lr=0.003, beta1=0.9, beta2=0.999, eps=1e-8, threads=1):
        tt = C.c_int64(t)
        self._err(self.L.tgr_adam_step(_dp(p), _dp(g), _dp(m), _dp(v), len(p), C.byref(tt), lr, beta1,
                                       beta2, eps, threads))
        return tt.value

    def train(self, s: Spec, coeffs, batches, cfg: Loss, lr, beta1=0.9, beta2=0.999, eps=1e-8,
              threads=1):
        """Returns (final coeffs, per-step terms (steps×4), seconds in the step loop)."""
        p = np.array(coeffs, dtype=np.float64)
        batches = np.ascontiguousarray(batches, dtype=np.float64)
        steps, n = batches.shape[0], batches.shape[1]
        terms = np.zeros((steps, 4))
        secs = C.c_double()
        self._err(self.L.tgr_train(*_spec_args(s), _dp(p), _dp(batches), n, steps, cfg.lambda1,
                                   cfg.lambda2, cfg.k, int(cfg.use_weighting), int(cfg.use_tv),
                                   int(cfg.differentiate_weight), lr, beta1, beta2, eps, threads,
                                   _dp(terms), C.byref(secs)))
        return p, terms, secs.value

    def sample_sphere(self, radius, total, ratio=(1, 1, 0), sigma_near=0.01, seed=1):
        out = np.zeros((total, 4))
        self._err(self.L.tgr_sample_sphere(radius, total, ratio[0], ratio[1], ratio[2], sigma_near,
                                           seed, _dp(out)))
        return out

    def rng_uniform(self, seed, n):
        out = np.zeros(n)
        self.L.tgr_rng_uniform(seed, n, _dp(out))
        return out

    def rng_gaussian(self, seed, n):
        out = np.zeros(n)
        self.L.tgr_rng_gaussian(seed, n, _dp(out))
        return out

    def upsample(self, s: Spec, coeffs, new_res):
        nr = (C.c_int * 3)(*[int(r) for r in (list(new_res) + [1, 1, 1])[:3]])
        n = 1
        for a in range(s.dim):
            n *= nr[a]
        out = np.zeros(n * s.K)
        self._err(self.L.tgr_upsample(*_spec_args(s), _dp(np.ascontiguousarray(coeffs, dtype=np.float64)), nr, _dp(out)))
        return out


def reference_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libtgref.so"))
