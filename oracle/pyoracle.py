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
        L.tgo_eval_batch_f32.argtypes = [C.POINTER(_TgoSpec), C.c_void_p, _D, C.c_int64, _D, _D, _D]
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
        L.tgo_sample_lattice.argtypes = [C.POINTER(_TgoSpec), _D, _I, _D]
        L.tgo_photometric_loss.restype = C.c_double
        L.tgo_photometric_loss.argtypes = [C.POINTER(_TgoSpec), _D, C.POINTER(_TgoSpec), C.c_int, _D, C.c_int64,
                                           _D, _D, _D, _D, _D, C.c_int, C.c_int, C.c_double, _D, _D, _D, _D, _D]
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

    def eval_f32(self, s: Spec, coeffs32, pts, want_grad=False):
        """eval on fp32-stored coefficients (upcast exactly), batched in C.
        want_grad: also (n x 3) spatial gradients and the per-axis L1 size of
        their terms -> (vals, grads, l1)."""
        sp = self._spec(s)
        c = np.ascontiguousarray(coeffs32, dtype=np.float32)
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        vals = np.empty(len(pts))
        grads = np.zeros((len(pts), 3)) if want_grad else None
        l1 = np.zeros((len(pts), 3)) if want_grad else None
        self.L.tgo_eval_batch_f32(C.byref(sp), c.ctypes.data_as(C.c_void_p), _dp(pts), len(pts), _dp(vals),
                                  _dp(grads), _dp(l1))
        return (vals, grads, l1) if want_grad else vals

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

    def sample_lattice(self, s: Spec, coeffs, lattice):
        lt = (C.c_int * 3)(*[int(r) for r in (list(lattice) + [1, 1, 1])[:3]])
        n = lt[0] * lt[1] * (lt[2] if s.dim == 3 else 1)
        out = np.zeros(n)
        self.L.tgo_sample_lattice(C.byref(self._spec(s)), _dp(np.ascontiguousarray(coeffs, dtype=np.float64)), lt,
                                  _dp(out))
        return out

    def photometric_loss(self, ds: Spec, dc, ss: Spec, deg, sc, rays, n_samples=64, activation=0, shift=-10.0,
                         bg=(1.0, 1.0, 1.0), want_grad=False, render=False):
        """forward_ray / backward_ray / photometric_loss restated (no jitter).
        rays = dict(origins, dirs, near, far[, gt]). Returns dict(loss, grad_density,
        grad_sh, colors, residual)."""
        n = len(rays["near"])
        f = lambda a: np.ascontiguousarray(np.asarray(a, dtype=np.float64))  # noqa: E731
        o, d, nr, fr = f(rays["origins"]), f(rays["dirs"]), f(rays["near"]), f(rays["far"])
        gt = f(rays["gt"]) if rays.get("gt") is not None else None
        B = (deg + 1) ** 2
        gd = np.zeros(ds.V * ds.K) if want_grad else None
        gs = np.zeros(ss.V * 3 * B) if want_grad else None
        col = np.zeros((n, 3)) if render else None
        res = np.zeros(n) if render else None
        loss = self.L.tgo_photometric_loss(C.byref(self._spec(ds)), _dp(f(dc)), C.byref(self._spec(ss)), deg,
                                           _dp(f(sc)), n, _dp(o), _dp(d), _dp(nr), _dp(fr), _dp(gt), n_samples,
                                           activation, shift, _dp(f(bg)), _dp(gd), _dp(gs), _dp(col), _dp(res))
        return dict(loss=loss, grad_density=gd, grad_sh=gs, colors=col, residual=res)

    def run_schedule(self, s: Spec, coeffs0, stages, batches, cfg: "Loss", lr=0.003, beta1=0.9, beta2=0.999,
                     eps=1e-8):
        """run_schedule (schedule.cpp:62-108): per stage upsample when the
        resolution changes (taylor_grid.cpp:273-284), fresh Adam moments, then
        the stage's steps; batches are consumed in order. stages = [(res, steps)].
        Returns (final spec, coeffs, terms)."""
        cur = Spec(s.dim, tuple(stages[0][0]), s.origin, s.extent, s.order)
        c = np.array(coeffs0, dtype=np.float64)
        terms, k = [], 0
        for res, steps in stages:
            res = tuple(res)
            if any(res[a] != cur.res[a] for a in range(s.dim)):
                c = self.resample(cur, c, cur.K, res)
                cur = Spec(s.dim, res, s.origin, s.extent, s.order)
            c, tr = self.train(cur, c, list(batches[k:k + steps]), cfg, lr, beta1, beta2, eps) if steps else (c, [])
            terms.extend(list(tr))
            k += steps
        return cur, c, np.array(terms).reshape(-1, 4)


def schedule_progressive(target, dim, total_steps):
    """Schedule::progressive (schedule.cpp:27-54) restated: target/4, /2, /1
    (floored at 4, capped at target), equal split, collapsed duplicates,
    remainder to the last stage. Returns [(res tuple, steps)]."""
    stages = []
    for d in (4, 2, 1):
        res = [2, 2, 2]  # Stage::resolution default {2, 2, 2} on unused axes
        same_target = True
        for a in range(dim):
            res[a] = min(max(4, int(target[a]) // d), int(target[a]))
            same_target &= res[a] == target[a]
        res = tuple(res[:3])
        if stages and all(res[a] == stages[-1][0][a] for a in range(dim)):
            continue
        stages.append([res, total_steps // 3])
        if same_target:
            break
    stages[-1][1] += total_steps - sum(st for _, st in stages)
    return [(r, st) for r, st in stages]


def tgrid_bytes(s: Spec, coeffs, precision: int) -> bytes:
    """save_tgrid's byte stream (grid_io.cpp:44-65, layout grid_io.hpp:11-16):
    "TGRD" | u32 version 1 | u8 dim | u8 order | dim x u32 res | dim x f64
    origin | dim x f64 extent | u8 precision (0 F64, 1 F32) | coefficients."""
    import struct
    out = b"TGRD" + struct.pack("<IBB", 1, s.dim, s.order)
    out += struct.pack("<" + "I" * s.dim, *[int(r) for r in s.res[:s.dim]])
    out += struct.pack("<" + "d" * s.dim, *[float(o) for o in s.origin[:s.dim]])
    out += struct.pack("<" + "d" * s.dim, *[float(e) for e in s.extent[:s.dim]])
    out += struct.pack("<B", precision)
    c = np.asarray(coeffs, dtype=np.float64 if precision == 0 else np.float32)
    return out + c.astype(c.dtype.newbyteorder("<")).tobytes()


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
        L.tgr_total_loss_fresh.argtypes = sp + [_D, _D, C.c_int64, C.c_double, C.c_double, C.c_double,
                                                C.c_int, C.c_int, C.c_int, C.c_uint64, _D, C.c_int, _D]
        L.tgr_eikonal_loss.argtypes = sp + [_D, _D, C.c_int64, C.c_double, _D, _D]
        L.tgr_train.argtypes = sp + [_D, _D, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                     C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                     C.c_double, C.c_int, _D, _D]
        L.tgr_eval_timed.argtypes = sp + [_D, _D, C.c_int64, _D, C.c_int, _D]
        L.tgr_init_grid.argtypes = sp + [C.c_int, C.c_double, C.c_double, C.c_uint64, C.c_uint64, _D]
        L.tgr_query_bench.argtypes = sp + [C.c_double, C.c_uint64, _D, C.c_int64, _D, C.c_int, _D]
        L.tgr_sample_sphere.argtypes = [C.c_double, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_double,
                                        C.c_uint64, _D]
        L.tgr_rng_uniform.argtypes = [C.c_uint64, C.c_int64, _D]
        L.tgr_rng_gaussian.argtypes = [C.c_uint64, C.c_int64, _D]
        L.tgr_upsample.argtypes = sp + [_D, _I, _D]
        L.tgr_run_schedule.argtypes = [C.c_int, _D, _D, C.c_int, _D, C.c_int, _I, _I, _D, C.c_int64,
                                       C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                       C.c_double, C.c_double, C.c_double, C.c_double, _D, _D]
        L.tgr_schedule_progressive.argtypes = [_I, C.c_int, C.c_int, _I, _I, _I]
        L.tgr_sample_grid_field.argtypes = sp + [_D, _I, _D]
        L.tgr_save_tgrid.argtypes = sp + [_D, C.c_char_p, C.c_int]
        L.tgr_load_tgrid.argtypes = [C.c_char_p, _I, _D, _D, C.c_int64]
        L.tgr_rng_index.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, _L]
        L.tgr_shuffle_order.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
        L.tgr_trace_csv.argtypes = [C.c_int, _I, _I, _D, _D, C.c_char_p, C.c_char_p, C.c_int64]
        L.tgr_photometric_loss.argtypes = sp + [_D, _I, _D, _D, C.c_int, _D, C.c_int64, _D, _D, _D, _D, _D,
                                                C.c_int, C.c_int, C.c_double, _D, _D, _D, _D, _D, _D, C.c_int,
                                                C.c_uint64]
        L.tgr_fit_sdf.argtypes = sp + [_D, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                       C.c_int, C.c_double, C.c_double, C.c_uint64, _D, _D, _D, C.c_int]
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

    def init_grid(self, s: Spec, mode=0, constant=0.0, epsilon=1e-4, seed=0, cap=4 << 30):
        """tg::init_grid coefficients (mode 0 Zeros, 1 Constant, 2 SmallUniform).
        Raises MemoryError (tg::ResourceError) / ValueError with the reference's message."""
        out = np.zeros(s.V * s.K)
        rc = self.L.tgr_init_grid(*_spec_args(s), int(mode), float(constant), float(epsilon), int(seed), int(cap),
                                  _dp(out))
        if rc == 5:
            raise MemoryError(self.L.tgr_last_error().decode())
        self._err(rc)
        return out

    def query_bench(self, s: Spec, pts, threads, epsilon=0.1, seed=7):
        """init_grid(SmallUniform) inside the reference, then parallel_for + eval
        over pts; returns (values, seconds of the eval loop)."""
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        vals = np.empty(len(pts))
        secs = C.c_double()
        self._err(self.L.tgr_query_bench(*_spec_args(s), epsilon, seed, _dp(pts), len(pts), _dp(vals), threads,
                                         C.byref(secs)))
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

    def total_loss_fresh(self, s: Spec, coeffs, samples, cfg: Loss, seed: int, grad=None, threads=1):
        """total_loss with EikonalPointSource::FreshUniform and tg::Rng(seed)."""
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        samples = np.ascontiguousarray(samples, dtype=np.float64).reshape(-1, 4)
        terms = np.zeros(4)
        self._err(self.L.tgr_total_loss_fresh(*_spec_args(s), _dp(coeffs), _dp(samples), len(samples),
                                              cfg.lambda1, cfg.lambda2, cfg.k, int(cfg.use_weighting),
                                              int(cfg.use_tv), int(cfg.differentiate_weight), int(seed), _dp(grad),
                                              threads, _dp(terms)))
        return terms

    def eikonal_loss(self, s: Spec, coeffs, pts, scale, grad=None):
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        out = C.c_double()
        self._err(self.L.tgr_eikonal_loss(*_spec_args(s), _dp(coeffs), _dp(pts), len(pts), scale, _dp(grad),
                                          C.byref(out)))
        return out.value

    def adam_step(self, p, g, m, v, t, lr=0.003, beta1=0.9, beta2=0.999, eps=1e-8, threads=1):
        tt = C.c_int64(t)
        self._err(self.L.tgr_adam_step(_dp(p), _dp(g), _dp(m), _dp(v), len(p), C.byref(tt), lr, beta1,
                                       beta2, eps, threads))
        return tt.value

    def train(self, s: Spec, coeffs, batches, cfg: Loss, lr, beta1=0.9, beta2=0.999, eps=1e-8,
              threads=1, steps=None):
        """Returns (final coeffs, per-step terms (steps×4), seconds in the step loop).
        coeffs None: the reference's zero init inside the library (no host copy;
        the returned coeffs are None). steps (default: one per batch): step i
        uses batch i % len(batches)."""
        p = None if coeffs is None else np.array(coeffs, dtype=np.float64)
        batches = np.ascontiguousarray(batches, dtype=np.float64)
        nb, n = batches.shape[0], batches.shape[1]
        steps = nb if steps is None else int(steps)
        terms = np.zeros((steps, 4))
        secs = C.c_double()
        self._err(self.L.tgr_train(*_spec_args(s), _dp(p), _dp(batches), n, nb, steps, cfg.lambda1,
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

    def run_schedule(self, s: Spec, coeffs0, stages, batches, cfg, lr=0.003, beta1=0.9, beta2=0.999, eps=1e-8):
        """tg::run_schedule with a TrainProblem feeding `batches` in order."""
        ns = len(stages)
        sr = np.array([list(r) + [1] * (3 - len(r)) for r, _ in stages], dtype=np.int32).ravel()
        st = np.array([n for _, n in stages], dtype=np.int32)
        fr = list(stages[-1][0])
        nv = 1
        for a in range(s.dim):
            nv *= fr[a]
        out = np.zeros(nv * s.K)
        total = int(st.sum())
        terms = np.zeros((total, 4))
        b = np.ascontiguousarray(np.asarray(batches[:total], dtype=np.float64))
        n = b.shape[1] if total else 0
        org = np.array(list(s.origin) + [0.0] * 3, dtype=np.float64)[:3]
        ext = np.array(list(s.extent) + [1.0] * 3, dtype=np.float64)[:3]
        self._err(self.L.tgr_run_schedule(s.dim, _dp(org), _dp(ext), s.order,
                                          _dp(np.ascontiguousarray(coeffs0, dtype=np.float64)), ns,
                                          sr.ctypes.data_as(_I), st.ctypes.data_as(_I), _dp(b), n, cfg.lambda1,
                                          cfg.lambda2, cfg.k, int(cfg.use_weighting), int(cfg.use_tv),
                                          int(cfg.differentiate_weight), lr, beta1, beta2, eps, _dp(out),
                                          _dp(terms)))
        return out, terms

    def fit_sdf(self, s: Spec, samples, total_steps, cfg, batch, lr=0.003, holdout_fraction=0.0, seed=1,
                eik_fresh=False):
        """tg::fit_sdf (default progressive plan); returns (coeffs at s.res, terms, report)."""
        smp = np.ascontiguousarray(np.asarray(samples, dtype=np.float64)).reshape(-1, 4)
        out = np.zeros(s.V * s.K)
        terms = np.zeros((total_steps, 4))
        rep = np.zeros(3)
        self._err(self.L.tgr_fit_sdf(*_spec_args(s), _dp(smp), smp.shape[0], total_steps, batch, cfg.lambda1,
                                     cfg.lambda2, cfg.k, int(cfg.use_weighting), int(cfg.use_tv), lr,
                                     holdout_fraction, seed, _dp(out), _dp(terms), _dp(rep), int(eik_fresh)))
        return out, terms, {"holdout_mae": rep[0], "train_samples": int(rep[1]), "holdout_samples": int(rep[2])}

    def rng_index(self, seed, n, count):
        out = np.zeros(count, dtype=np.int64)
        self.L.tgr_rng_index(seed, n, count, out.ctypes.data_as(_L))
        return out

    def shuffle_order(self, seed, n):
        out = np.zeros(n, dtype=np.uint32)
        self.L.tgr_shuffle_order(seed, n, out.ctypes.data_as(C.c_void_p))
        return out

    def trace_csv(self, steps, stages, res3, terms, wall_ms, label="recon"):
        n = len(steps)
        ss = np.ascontiguousarray(np.stack([steps, stages], 1).astype(np.int32))
        rr = np.ascontiguousarray(np.asarray(res3, dtype=np.int32))
        tt = np.ascontiguousarray(np.asarray(terms, dtype=np.float64))
        ww = np.ascontiguousarray(np.asarray(wall_ms, dtype=np.float64))
        buf = C.create_string_buffer(256 * (n + 1))
        rc = self.L.tgr_trace_csv(n, ss.ctypes.data_as(_I), rr.ctypes.data_as(_I), _dp(tt), _dp(ww), label.encode(),
                                  buf, len(buf))
        assert rc == 0
        return buf.value.decode()

    def photometric_loss(self, ds: Spec, dc, ss: Spec, deg, sc, rays, n_samples=64, activation=0, shift=-10.0,
                         bg=(1.0, 1.0, 1.0), want_grad=False, render=False, jitter=False, jitter_seed=0):
        """tg::photometric_loss / render_ray (threads 1; RenderOptions::jitter / jitter_seed)."""
        n = len(rays["near"])
        f = lambda a: np.ascontiguousarray(np.asarray(a, dtype=np.float64))  # noqa: E731
        o, d, nr, fr = f(rays["origins"]), f(rays["dirs"]), f(rays["near"]), f(rays["far"])
        gt = f(rays["gt"]) if rays.get("gt") is not None else None
        B = (deg + 1) ** 2
        gd = np.zeros(ds.V * ds.K) if want_grad else None
        gs = np.zeros(ss.V * 3 * B) if want_grad else None
        col = np.zeros((n, 3)) if render else None
        res = np.zeros(n) if render else None
        loss = C.c_double(0.0)
        sres = (C.c_int * 3)(*[int(x) for x in ss.res])
        sorg = f(list(ss.origin))
        sext = f(list(ss.extent))
        self._err(self.L.tgr_photometric_loss(*_spec_args(ds), _dp(f(dc)), sres, _dp(sorg), _dp(sext), deg,
                                              _dp(f(sc)), n, _dp(o), _dp(d), _dp(nr), _dp(fr), _dp(gt), n_samples,
                                              activation, shift, _dp(f(bg)), _dp(gd), _dp(gs), _dp(col), _dp(res),
                                              C.byref(loss), int(bool(jitter)), int(jitter_seed)))
        return dict(loss=loss.value if gt is not None else 0.0, grad_density=gd, grad_sh=gs, colors=col,
                    residual=res)

    def schedule_progressive(self, target, dim, total_steps):
        t = (C.c_int * 3)(*[int(x) for x in (list(target) + [1, 1, 1])[:3]])
        ns = C.c_int()
        sr = (C.c_int * 9)()
        st = (C.c_int * 3)()
        self.L.tgr_schedule_progressive(t, dim, total_steps, C.byref(ns), sr, st)
        return [(tuple(sr[3 * i:3 * i + 3]), st[i]) for i in range(ns.value)]

    def sample_grid_field(self, s: Spec, coeffs, lattice):
        lt = (C.c_int * 3)(*[int(r) for r in (list(lattice) + [1, 1, 1])[:3]])
        n = lt[0] * lt[1] * (lt[2] if s.dim == 3 else 1)
        out = np.zeros(n)
        self._err(self.L.tgr_sample_grid_field(*_spec_args(s), _dp(np.ascontiguousarray(coeffs, dtype=np.float64)),
                                               lt, _dp(out)))
        return out

    def save_tgrid(self, s: Spec, coeffs, path, precision=0):
        self._err(self.L.tgr_save_tgrid(*_spec_args(s), _dp(np.ascontiguousarray(coeffs, dtype=np.float64)),
                                        str(path).encode(), precision))

    def load_tgrid(self, path):
        sp = (C.c_int * 5)()
        geo = (C.c_double * 6)()
        rc = self.L.tgr_load_tgrid(str(path).encode(), sp, geo, None, 0)
        if rc != 0:
            raise OSError(self.L.tgr_last_error().decode())
        s = Spec(sp[0], tuple(sp[2:5]), tuple(geo[0:3]), tuple(geo[3:6]), sp[1])
        c = np.zeros(s.V * s.K)
        self._err(self.L.tgr_load_tgrid(str(path).encode(), sp, geo, _dp(c), c.size))
        return s, c


def reference_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libtgref.so"))
