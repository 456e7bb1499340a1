// Host-side seeded input generation for the BASELINE.json configs, with the
// reference Rng value mappings (rng.hpp:14-74) so the GPU path and the CPU
// oracle consume identical fp32 samples. Analytic targets: the sphere
// (sample_sphere_points, sampling.cpp:140-159), the 2D circle ∪ box of C1 and
// the 64-primitive procedural union of C3/C5 (not in the reference; written
// here and used identically by both sides).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/tgcu.h"

namespace {

constexpr double kTwoPi = 6.283185307179586476925286766559;

class Rng {
public:
    explicit Rng(uint64_t seed) : eng_(seed) {}
    uint64_t bits() { return eng_(); }
    double uniform() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    uint64_t index(uint64_t n) {
        const uint64_t limit = uint64_t(-1) - uint64_t(-1) % n;
        uint64_t x;
        do {
            x = eng_();
        } while (x >= limit);
        return x % n;
    }
    double gaussian() {
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        double u1 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double theta = kTwoPi * u2;
        spare_ = r * std::sin(theta);
        have_spare_ = true;
        return r * std::cos(theta);
    }
    void unit_vector(double* out) {
        const double z = uniform(-1.0, 1.0);
        const double phi = uniform(0.0, kTwoPi);
        const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
        out[0] = r * std::cos(phi);
        out[1] = r * std::sin(phi);
        out[2] = z;
    }

private:
    std::mt19937_64 eng_;
    double spare_ = 0.0;
    bool have_spare_ = false;
};

// ---- analytic SDFs ---------------------------------------------------------

double sdf_box2(double x, double y, double cx, double cy, double hx, double hy) {
    const double qx = std::fabs(x - cx) - hx, qy = std::fabs(y - cy) - hy;
    const double ox = std::max(qx, 0.0), oy = std::max(qy, 0.0);
    return std::sqrt(ox * ox + oy * oy) + std::min(std::max(qx, qy), 0.0);
}

// BASELINE C1: circle r = 0.5 at the origin ∪ box half-extent 0.3 at (0.3, -0.2).
double sdf_c1(const double* p) {
    const double c = std::sqrt(p[0] * p[0] + p[1] * p[1]) - 0.5;
    return std::min(c, sdf_box2(p[0], p[1], 0.3, -0.2, 0.3, 0.3));
}

struct Prim {
    int type;  // 0 sphere, 1 box, 2 torus (axis z)
    double c[3];
    double a, b, e;  // sphere: a = r; box: half-extents (a, b, e); torus: a = R, b = r
};

std::vector<Prim> make_prims(uint64_t shape_seed) {
    // 64 seeded primitives, centres U[-0.7, 0.7]^3 (BASELINE.json configs[2]).
    Rng r(shape_seed);
    std::vector<Prim> ps(64);
    for (auto& p : ps) {
        p.type = static_cast<int>(r.index(3));
        for (int a = 0; a < 3; ++a) p.c[a] = r.uniform(-0.7, 0.7);
        if (p.type == 0) {
            p.a = r.uniform(0.05, 0.25);
        } else if (p.type == 1) {
            p.a = r.uniform(0.05, 0.2);
            p.b = r.uniform(0.05, 0.2);
            p.e = r.uniform(0.05, 0.2);
        } else {
            p.a = r.uniform(0.1, 0.25);
            p.b = p.a / 4.0;
        }
    }
    return ps;
}

double prim_sdf(const Prim& p, const double* x) {
    const double dx = x[0] - p.c[0], dy = x[1] - p.c[1], dz = x[2] - p.c[2];
    if (p.type == 0) return std::sqrt(dx * dx + dy * dy + dz * dz) - p.a;
    if (p.type == 1) {
        const double qx = std::fabs(dx) - p.a, qy = std::fabs(dy) - p.b, qz = std::fabs(dz) - p.e;
        const double ox = std::max(qx, 0.0), oy = std::max(qy, 0.0), oz = std::max(qz, 0.0);
        return std::sqrt(ox * ox + oy * oy + oz * oz) + std::min(std::max(qx, std::max(qy, qz)), 0.0);
    }
    const double qx = std::sqrt(dx * dx + dy * dy) - p.a;
    return std::sqrt(qx * qx + dz * dz) - p.b;
}

double sdf_prims(const std::vector<Prim>& ps, const double* x) {
    double d = 1e300;
    for (const auto& p : ps) d = std::min(d, prim_sdf(p, x));
    return d;
}

void prim_surface_point(const Prim& p, Rng& r, double* out) {
    if (p.type == 0) {
        double u[3];
        r.unit_vector(u);
        for (int a = 0; a < 3; ++a) out[a] = p.c[a] + p.a * u[a];
    } else if (p.type == 1) {
        const double h[3] = {p.a, p.b, p.e};
        const int face = static_cast<int>(r.index(6));
        const int axis = face / 2;
        for (int a = 0; a < 3; ++a) out[a] = p.c[a] + r.uniform(-h[a], h[a]);
        out[axis] = p.c[axis] + ((face % 2) ? h[axis] : -h[axis]);
    } else {
        const double th = r.uniform(0.0, kTwoPi), ph = r.uniform(0.0, kTwoPi);
        const double rr = p.a + p.b * std::cos(ph);
        out[0] = p.c[0] + rr * std::cos(th);
        out[1] = p.c[1] + rr * std::sin(th);
        out[2] = p.c[2] + p.b * std::sin(ph);
    }
}

double clampd(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }

template <class F>
void parallel_rows(int64_t n, F&& f) {
    const int nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    if (n < 4096 || nt == 1) {
        f(0, n);
        return;
    }
    std::vector<std::thread> ts;
    const int64_t chunk = (n + nt - 1) / nt;
    for (int t = 0; t < nt; ++t) {
        const int64_t b = t * chunk, e = std::min(n, b + chunk);
        if (b >= e) break;
        ts.emplace_back([&, b, e] { f(b, e); });
    }
    for (auto& t : ts) t.join();
}

}  // namespace

extern "C" {

int tgcu_sample(int shape, int dim, uint64_t seed, int64_t n, double near_frac, double sigma, double param0,
                float* out4) {
    if (n <= 0 || !out4 || near_frac < 0.0 || near_frac > 1.0) return TGCU_ERR_INVALID_ARGUMENT;
    if ((shape == 0 || shape == 2) && dim != 3) return TGCU_ERR_INVALID_ARGUMENT;
    if (shape == 1 && dim != 2) return TGCU_ERR_INVALID_ARGUMENT;
    const int64_t n_near = static_cast<int64_t>(std::floor(static_cast<double>(n) * near_frac));
    const int64_t n_uni = n - n_near;
    Rng rng(seed);
    std::vector<Prim> prims;
    if (shape == 2) prims = make_prims(static_cast<uint64_t>(param0));
    // Points (sequential: one Rng stream), uniform first as run_protocol
    // (sampling.cpp:94-103).
    std::vector<double> pts(static_cast<size_t>(3 * n), 0.0);
    for (int64_t i = 0; i < n_uni; ++i)
        for (int a = 0; a < dim; ++a) pts[3 * i + a] = rng.uniform(-1.0, 1.0);
    for (int64_t i = n_uni; i < n; ++i) {
        double* p = &pts[3 * i];
        if (shape == 0) {
            double u[3];
            rng.unit_vector(u);
            for (int a = 0; a < 3; ++a) p[a] = param0 * u[a];
        } else if (shape == 2) {
            prim_surface_point(prims[rng.index(prims.size())], rng, p);
        } else {
            // 2D C1 outline: circle or box boundary in proportion to perimeter.
            if (rng.uniform() < (kTwoPi * 0.5) / (kTwoPi * 0.5 + 2.4)) {
                const double th = rng.uniform(0.0, kTwoPi);
                p[0] = 0.5 * std::cos(th);
                p[1] = 0.5 * std::sin(th);
            } else {
                const int side = static_cast<int>(rng.index(4));
                const double t = rng.uniform(-0.3, 0.3);
                p[0] = 0.3 + (side < 2 ? (side == 0 ? -0.3 : 0.3) : t);
                p[1] = -0.2 + (side < 2 ? t : (side == 2 ? -0.3 : 0.3));
            }
        }
        for (int a = 0; a < dim; ++a) p[a] += sigma * rng.gaussian();
        for (int a = 0; a < dim; ++a) p[a] = clampd(p[a], -1.0, 1.0);
    }
    parallel_rows(n, [&](int64_t b, int64_t e) {
        for (int64_t i = b; i < e; ++i) {
            double q[3];
            for (int a = 0; a < 3; ++a) q[a] = static_cast<double>(static_cast<float>(pts[3 * i + a]));
            double gt;
            if (shape == 0)
                gt = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2]) - param0;
            else if (shape == 1)
                gt = sdf_c1(q);
            else
                gt = sdf_prims(prims, q);
            out4[4 * i] = static_cast<float>(q[0]);
            out4[4 * i + 1] = static_cast<float>(q[1]);
            out4[4 * i + 2] = static_cast<float>(q[2]);
            out4[4 * i + 3] = static_cast<float>(gt);
        }
    });
    return TGCU_OK;
}

int tgcu_sample_uniform(int dim, uint64_t seed, int64_t n, double lo, double hi, float* out3) {
    if (n <= 0 || !out3 || (dim != 2 && dim != 3)) return TGCU_ERR_INVALID_ARGUMENT;
    Rng rng(seed);
    for (int64_t i = 0; i < n; ++i) {
        for (int a = 0; a < 3; ++a) out3[3 * i + a] = a < dim ? static_cast<float>(rng.uniform(lo, hi)) : 0.0f;
    }
    return TGCU_OK;
}

struct tgcu_rng {
    Rng r;
};

int tgcu_rng_create(uint64_t seed, tgcu_rng** out) {
    if (!out) return TGCU_ERR_INVALID_ARGUMENT;
    *out = new tgcu_rng{Rng(seed)};
    return TGCU_OK;
}

void tgcu_rng_destroy(tgcu_rng* r) { delete r; }

int tgcu_rng_index(tgcu_rng* r, uint64_t n, int64_t count, int64_t* out) {
    if (!r || !out || n == 0 || count < 0) return TGCU_ERR_INVALID_ARGUMENT;
    for (int64_t i = 0; i < count; ++i) out[i] = static_cast<int64_t>(r->r.index(n));
    return TGCU_OK;
}

int tgcu_rng_uniform_box(tgcu_rng* r, int dim, const double* lo, const double* hi, int64_t count, double* out3) {
    if (!r || !lo || !hi || !out3 || count < 0 || (dim != 2 && dim != 3)) return TGCU_ERR_INVALID_ARGUMENT;
    for (int64_t i = 0; i < count; ++i) {  // Rng::uniform_in_box (rng.hpp:53-57): axes in order, z = 0 in 2D
        for (int a = 0; a < 3; ++a) out3[3 * i + a] = a < dim ? r->r.uniform(lo[a], hi[a]) : 0.0;
    }
    return TGCU_OK;
}

int tgcu_shuffle_order(uint64_t seed, int64_t n, uint32_t* order) {
    if (n < 0 || (n > 0 && !order)) return TGCU_ERR_INVALID_ARGUMENT;
    for (int64_t i = 0; i < n; ++i) order[i] = static_cast<uint32_t>(i);
    Rng rng(seed);
    for (int64_t i = n; i > 1; --i) std::swap(order[i - 1], order[rng.index(static_cast<uint64_t>(i))]);
    return TGCU_OK;
}

int tgcu_shape_sdf(int shape, int dim, double param0, const double* pts, int64_t n, double* out) {
    if (n < 0 || !pts || !out) return TGCU_ERR_INVALID_ARGUMENT;
    std::vector<Prim> prims;
    if (shape == 2) prims = make_prims(static_cast<uint64_t>(param0));
    for (int64_t i = 0; i < n; ++i) {
        const double* q = pts + 3 * i;
        if (shape == 0)
            out[i] = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2]) - param0;
        else if (shape == 1)
            out[i] = sdf_c1(q);
        else
            out[i] = sdf_prims(prims, q);
    }
    (void)dim;
    return TGCU_OK;
}

}  // extern "C"
