// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// extern "C" shim over the reference library's own hot-path functions
// (/root/reference/proj/core, compiled unmodified by oracle/Makefile into
// oracle/_ref/libtgref.so). It lets the Python tests pin the C restatement
// (tg_oracle.c) against the real reference, generate golden vectors, and time
// the reference CPU path for bench.py's cpu_baseline / --impl reference legs.
// Nothing here is linked into the product library.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "taylorgrid/adam.hpp"
#include "taylorgrid/errors.hpp"
#include "taylorgrid/grid_io.hpp"
#include "taylorgrid/marching.hpp"
#include "taylorgrid/parallel.hpp"
#include "taylorgrid/rng.hpp"
#include "taylorgrid/sampling.hpp"
#include "taylorgrid/schedule.hpp"
#include "taylorgrid/sample_set.hpp"
#include "taylorgrid/sdf_fit.hpp"
#include "taylorgrid/sdf_loss.hpp"
#include "taylorgrid/taylor_grid.hpp"
#include "taylorgrid/volume_render.hpp"

namespace {

thread_local std::string g_err;

tg::GridSpec make_spec(int dim, const int* res, const double* origin, const double* extent,
                       int order) {
    tg::GridSpec s;
    s.dim = dim;
    for (int a = 0; a < 3; ++a) {
        s.resolution[a] = res[a];
        s.origin[a] = origin[a];
        s.extent[a] = extent[a];
    }
    s.order = order;
    return s;
}

// Wraps reference coefficients without copying is impossible (TaylorGrid owns a
// std::vector), so grids are built per call from the caller's array.
tg::TaylorGrid make_grid(const tg::GridSpec& spec, const double* coeffs) {
    tg::InitOptions opts;
    opts.memory_cap_bytes = ~0ull;
    tg::TaylorGrid g = tg::init_grid(spec, opts);  // coeffs == nullptr: InitMode::Zeros
    if (coeffs) std::memcpy(g.coeffs.data(), coeffs, g.coeffs.size() * sizeof(double));
    return g;
}

std::vector<tg::SdfSample> make_batch(const double* samples, int64_t n, int dim) {
    std::vector<tg::SdfSample> batch(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        batch[i].point = {samples[4 * i], samples[4 * i + 1], dim == 3 ? samples[4 * i + 2] : 0.0};
        batch[i].gt_sdf = samples[4 * i + 3];
    }
    return batch;
}

tg::LossConfig make_loss(double lambda1, double lambda2, double k, int use_weighting, int use_tv,
                         int differentiate_weight) {
    tg::LossConfig c;
    c.lambda1 = lambda1;
    c.lambda2 = lambda2;
    c.k = k;
    c.use_weighting = use_weighting != 0;
    c.use_tv = use_tv != 0;
    c.differentiate_weight = differentiate_weight != 0;
    return c;
}

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

}  // namespace

extern "C" {

const char* tgr_last_error() { return g_err.c_str(); }

int tgr_coeff_count(int order, int dim) {
    try {
        return tg::coeff_count(order, dim);
    } catch (const std::exception& e) {
        return -fail(e, 1);
    }
}

int tgr_locate(int dim, const int* res, const double* origin, const double* extent, int order,
               const double* p, int* cell, double* local, int64_t* vid) {
    try {
        const auto spec = make_spec(dim, res, origin, extent, order);
        const tg::CellRef r = tg::locate(spec, {p[0], p[1], p[2]});
        for (int a = 0; a < 3; ++a) {
            cell[a] = r.cell[a];
            local[a] = r.local[a];
        }
        for (int c = 0; c < 8; ++c) vid[c] = r.vertex_ids[c];
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, 1);
    }
}

// Batched eval: pts n×3, vals n, grads n×3 (nullable).
int tgr_eval(int dim, const int* res, const double* origin, const double* extent, int order,
             const double* coeffs, const double* pts, int64_t n, double* vals, double* grads) {
    try {
        const auto spec = make_spec(dim, res, origin, extent, order);
        const tg::TaylorGrid grid = make_grid(spec, coeffs);
        for (int64_t i = 0; i < n; ++i) {
            const tg::Vec3 p{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
            if (grads) {
                const tg::EvalResult er = tg::eval_with_spatial_gradient(grid, p);
                vals[i] = er.value;
                for (int a = 0; a < 3; ++a) grads[3 * i + a] = er.spatial_gradient[a];
            } else {
                vals[i] = tg::eval(grid, p);
            }
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// Batched backprop_value_and_spatial into grad (coeff_total entries).
int tgr_backprop(int dim, const int* res, const double* origin, const double* extent, int order,
                 const double* coeffs, const double* pts, const double* upstream,
                 const double* upstream_vec, int64_t n, double* grad) {
    try {
        const auto spec = make_spec(dim, res, origin, extent, order);
        const tg::TaylorGrid grid = make_grid(spec, coeffs);
        std::span<double> g(grad, grid.coeffs.size());
        for (int64_t i = 0; i < n; ++i) {
            const tg::Vec3 p{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
            const tg::Vec3 uv{upstream_vec[3 * i], upstream_vec[3 * i + 1], upstream_vec[3 * i + 2]};
            tg::backprop_value_and_spatial(grid, p, upstream[i], uv, g);
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

double tgr_adaptive_weight(double d_hat, double d, double k) { return tg::adaptive_weight(d_hat, d, k); }

int tgr_tv_loss(int dim, const int* res, const double* origin, const double* extent, int order,
                const double* coeffs, double* grad, double scale, int threads, double* out) {
    try {
        const auto spec = make_spec(dim, res, origin, extent, order);
        const tg::TaylorGrid grid = make_grid(spec, coeffs);
        std::span<double> g;
        if (grad) g = std::span<double>(grad, grid.coeffs.size());
        *out = tg::tv_loss(grid, g, scale, threads);
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

int tgr_total_loss(int dim, const int* res, const double* origin, const double* extent, int order,
                   const double* coeffs, const double* samples, int64_t n, double lambda1,
                   double lambda2, double k, int use_weighting, int use_tv, int differentiate_weight,
                   double* grad, int threads, double* terms) {
    try {
        const auto spec = make_spec(dim, res, origin, extent, order);
        const tg::TaylorGrid grid = make_grid(spec, coeffs);
        const auto batch = make_batch(samples, n, dim);
        const auto cfg = make_loss(lambda1, lambda2, k, use_weighting, use_tv, differentiate_weight);
        std::span<double> g;
        if (grad) g = std::span<double>(grad, grid.coeffs.size());
        const tg::LossTerms t = tg::total_loss(grid, batch, cfg, g, threads);
        terms[0] = t.total;
        terms[1] = t.fit;
        terms[2] = t.eik;
        terms[3] = t.tv;
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 4);
    }
}

// total_loss with EikonalPointSource::FreshUniform and tg::Rng(seed)
// (sdf_loss.cpp:274-283): the reference draws its own eikonal points.
int tgr_total_loss_fresh(int dim, const int* res, const double* origin, const double* extent, int order,
                         const double* coeffs, const double* samples, int64_t n, double lambda1,
                         double lambda2, double k, int use_weighting, int use_tv, int differentiate_weight,
                         uint64_t seed, double* grad, int threads, double* terms) {
    try {
        const auto spec = make_spec(dim, res, origin, extent, order);
        const tg::TaylorGrid grid = make_grid(spec, coeffs);
        const auto batch = make_batch(samples, n, dim);
        auto cfg = make_loss(lambda1, lambda2, k, use_weighting, use_tv, differentiate_weight);
        cfg.eikonal_point_source = tg::EikonalPointSource::FreshUniform;
        std::span<double> g;
        if (grad) g = std::span<double>(grad, grid.coeffs.size());
        tg::Rng rng(seed);
        const tg::LossTerms t = tg::total_loss(grid, batch, cfg, g, threads, &rng);
        terms[0] = t.total;
        terms[1] = t.fit;
        terms[2] = t.eik;
        terms[3] = t.tv;
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 4);
    }
}

// eikonal_loss (sdf_loss.cpp:137-153) on caller points (n x 3).
int tgr_eikonal_loss(int dim, const int* res, const double* origin, const double* extent, int order,
                     const double* coeffs, const double* pts, int64_t n, double scale, double* grad, double* out) {
    try {
        const auto spec = make_spec(dim, res, origin, extent, order);
        const tg::TaylorGrid grid = make_grid(spec, coeffs);
        std::vector<tg::Vec3> p(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) p[i] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
        std::span<double> g;
        if (grad) g = std::span<double>(grad, grid.coeffs.size());
        *out = tg::eikonal_loss(grid, p, g, scale);
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// adam_step on caller arrays; returns 0, or 4 with the NumericalError text.
int tgr_adam_step(double* p, const double* g, double* m, double* v, int64_t n, int64_t* t, double lr,
                  double beta1, double beta2, double eps, int threads) {
    try {
        tg::AdamConfig c{lr, beta1, beta2, eps};
        tg::AdamState st(static_cast<std::size_t>(n), c);
        std::memcpy(st.m.data(), m, n * sizeof(double));
        std::memcpy(st.v.data(), v, n * sizeof(double));
        st.t = *t;
        tg::adam_step(std::span<double>(p, n), std::span<const double>(g, n), st, threads);
        std::memcpy(m, st.m.data(), n * sizeof(double));
        std::memcpy(v, st.v.data(), n * sizeof(double));
        *t = st.t;
        return 0;
    } catch (const tg::NumericalError& e) {
        return fail(e, 4);
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// Training trajectory in the cmd_bench loop shape (tools/main.cpp:639-644):
// per step zero grad -> total_loss -> finite check -> adam_step. Batches are
// supplied by the caller (steps × n × 4). coeffs is updated in place; the
// per-step LossTerms go to terms_out (steps × 4).
int tgr_train(int dim, const int* res, const double* origin, const double* extent, int order,
              double* coeffs, const double* batches, int64_t n, int nbatch, int steps, double lambda1,
              double lambda2, double k, int use_weighting, int use_tv, int differentiate_weight,
              double lr, double beta1, double beta2, double eps, int threads, double* terms_out,
              double* seconds_out) {
    try {
        const auto spec = make_spec(dim, res, origin, extent, order);
        tg::TaylorGrid grid = make_grid(spec, coeffs);
        const auto cfg = make_loss(lambda1, lambda2, k, use_weighting, use_tv, differentiate_weight);
        tg::AdamState state(grid.coeffs.size(), tg::AdamConfig{lr, beta1, beta2, eps});
        std::vector<double> grad(grid.coeffs.size());
        double secs = 0.0;
        for (int s = 0; s < steps; ++s) {
            // step s uses batch s % nbatch (a long run cycles a few stored batches)
            const auto batch = make_batch(batches + 4 * n * static_cast<int64_t>(s % nbatch), n, dim);
            const auto t0 = std::chrono::steady_clock::now();
            std::fill(grad.begin(), grad.end(), 0.0);
            const tg::LossTerms t = tg::total_loss(grid, batch, cfg, grad, threads);
            if (!std::isfinite(t.total)) {
                throw tg::NumericalError("run_schedule: non-finite loss at stage 0 step " +
                                         std::to_string(s));
            }
            tg::adam_step(grid.coeffs, grad, state, threads);
            secs += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (terms_out) {
                terms_out[4 * s] = t.total;
                terms_out[4 * s + 1] = t.fit;
                terms_out[4 * s + 2] = t.eik;
                terms_out[4 * s + 3] = t.tv;
            }
        }
        if (coeffs) std::memcpy(coeffs, grid.coeffs.data(), grid.coeffs.size() * sizeof(double));
        if (seconds_out) *seconds_out = secs;
        return 0;
    } catch (const tg::NumericalError& e) {
        return fail(e, 4);
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// Query throughput of the reference: parallel_for + eval. Returns
// the wall seconds of the eval loop only.
int tgr_eval_timed(int dim, const int* res, const double* origin, const double* extent, int order,
                   const double* coeffs, const double* pts, int64_t n, double* vals, int threads,
                   double* seconds_out) {
    try {
        const auto spec = make_spec(dim, res, origin, extent, order);
        const tg::TaylorGrid grid = make_grid(spec, coeffs);
        const auto t0 = std::chrono::steady_clock::now();
        tg::parallel_for(n, threads, [&](int64_t b, int64_t e, int) {
            for (int64_t i = b; i < e; ++i) vals[i] = tg::eval(grid, {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]});
        });
        *seconds_out = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// init_grid (taylor_grid.cpp:162-188) with InitOptions {mode 0 Zeros /
// 1 Constant / 2 SmallUniform, constant, epsilon, seed, cap}: the
// coefficients (coeff_total doubles) for init parity tests.
int tgr_init_grid(int dim, const int* res, const double* origin, const double* extent, int order, int mode,
                  double constant, double epsilon, uint64_t seed, uint64_t cap, double* out) {
    try {
        tg::InitOptions opts;
        opts.mode = mode == 0 ? tg::InitMode::Zeros : (mode == 1 ? tg::InitMode::Constant : tg::InitMode::SmallUniform);
        opts.constant = constant;
        opts.epsilon = epsilon;
        opts.seed = seed;
        opts.memory_cap_bytes = cap;
        const tg::TaylorGrid g = tg::init_grid(make_spec(dim, res, origin, extent, order), opts);
        if (out) std::memcpy(out, g.coeffs.data(), g.coeffs.size() * sizeof(double));
        return 0;
    } catch (const tg::ResourceError& e) {
        return fail(e, 5);
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// Query throughput of the reference on a grid it initialises itself
// (init_grid, InitMode::SmallUniform with the given epsilon and seed,
// taylor_grid.cpp:162-188; memory cap lifted): parallel_for + eval over the
// points. For the large BASELINE query grids (512^3), where passing fp64
// coefficients from the caller would need a second multi-GB copy.
int tgr_query_bench(int dim, const int* res, const double* origin, const double* extent, int order,
                    double epsilon, uint64_t seed, const double* pts, int64_t n, double* vals, int threads,
                    double* seconds_out) {
    try {
        const auto spec = make_spec(dim, res, origin, extent, order);
        tg::InitOptions opts;
        opts.mode = tg::InitMode::SmallUniform;
        opts.epsilon = epsilon;
        opts.seed = seed;
        opts.memory_cap_bytes = ~0ull;
        const tg::TaylorGrid grid = tg::init_grid(spec, opts);
        const auto t0 = std::chrono::steady_clock::now();
        tg::parallel_for(n, threads, [&](int64_t b, int64_t e, int) {
            for (int64_t i = b; i < e; ++i) vals[i] = tg::eval(grid, {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]});
        });
        *seconds_out = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// Reference sampler: sample_sphere_points (sampling.cpp:140-159) with the
// uniform:near:ray ratio given; out is total×4 (x, y, z, gt).
int tgr_sample_sphere(double radius, int64_t total, int r0, int r1, int r2, double sigma_near,
                      uint64_t seed, double* out) {
    try {
        tg::SamplingConfig c;
        c.total = total;
        c.ratio = {r0, r1, r2};
        c.sigma_near = sigma_near;
        c.seed = seed;
        const tg::SampleSet s = tg::sample_sphere_points(radius, c);
        for (std::size_t i = 0; i < s.samples.size(); ++i) {
            for (int a = 0; a < 3; ++a) out[4 * i + a] = s.samples[i].point[a];
            out[4 * i + 3] = s.samples[i].gt_sdf;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// Raw Rng stream access for pinning the product's seeded generator.
void tgr_rng_uniform(uint64_t seed, int64_t n, double* out) {
    tg::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.uniform();
}
void tgr_rng_gaussian(uint64_t seed, int64_t n, double* out) {
    tg::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.gaussian();
}

int tgr_upsample(int dim, const int* res, const double* origin, const double* extent, int order,
                 const double* coeffs, const int* new_res, double* out) {
    try {
        const auto spec = make_spec(dim, res, origin, extent, order);
        const tg::TaylorGrid grid = make_grid(spec, coeffs);
        const tg::TaylorGrid up = tg::upsample(grid, {new_res[0], new_res[1], new_res[2]});
        std::memcpy(out, up.coeffs.data(), up.coeffs.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// run_schedule (schedule.cpp:62-108) driven by a TrainProblem that feeds the
// caller's batches in order (one n-sample batch per global step). stage_res is
// nstages x 3, coeffs0 the grid at stage 0's resolution; out_coeffs receives the
// final grid (final stage resolution), terms_out total_steps x 4.
int tgr_run_schedule(int dim, const double* origin, const double* extent, int order,
                     const double* coeffs0, int nstages, const int* stage_res, const int* stage_steps,
                     const double* batches, int64_t n, double lambda1, double lambda2, double k,
                     int use_weighting, int use_tv, int differentiate_weight, double lr, double beta1,
                     double beta2, double eps, double* out_coeffs, double* terms_out) {
    try {
        class Feed final : public tg::TrainProblem {
        public:
            Feed(const double* b, int64_t n, int dim, tg::LossConfig c) : b_(b), n_(n), dim_(dim), cfg_(c) {}
            tg::LossTerms compute(const tg::TaylorGrid& grid, std::span<double> grad) override {
                const auto batch = make_batch(b_ + 4 * n_ * step_++, n_, dim_);
                return tg::total_loss(grid, batch, cfg_, grad, 1);
            }

        private:
            const double* b_;
            int64_t n_;
            int dim_;
            tg::LossConfig cfg_;
            int64_t step_ = 0;
        };
        tg::Schedule sch;
        for (int s = 0; s < nstages; ++s)
            sch.stages.push_back({{stage_res[3 * s], stage_res[3 * s + 1], stage_res[3 * s + 2]}, stage_steps[s]});
        const auto spec = make_spec(dim, stage_res, origin, extent, order);
        Feed feed(batches, n, dim, make_loss(lambda1, lambda2, k, use_weighting, use_tv, differentiate_weight));
        const auto r = tg::run_schedule(feed, sch, make_grid(spec, coeffs0), tg::AdamConfig{lr, beta1, beta2, eps}, 1);
        std::memcpy(out_coeffs, r.grid.coeffs.data(), r.grid.coeffs.size() * sizeof(double));
        for (std::size_t i = 0; i < r.trace.size(); ++i) {
            terms_out[4 * i] = r.trace[i].loss.total;
            terms_out[4 * i + 1] = r.trace[i].loss.fit;
            terms_out[4 * i + 2] = r.trace[i].loss.eik;
            terms_out[4 * i + 3] = r.trace[i].loss.tv;
        }
        return 0;
    } catch (const tg::NumericalError& e) {
        return fail(e, 4);
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// fit_sdf (sdf_fit.cpp:52-105) with the default progressive schedule over
// total_steps, LossConfig batch_size = batch. samples n x 4 (x, y, z, gt).
// out_coeffs: final grid (spec resolution); terms_out: total_steps x 4;
// report_out: {holdout_mae, train_samples, holdout_samples}.
int tgr_fit_sdf(int dim, const int* res, const double* origin, const double* extent, int order,
                const double* samples, int64_t n, int total_steps, int batch, double lambda1, double lambda2,
                double k, int use_weighting, int use_tv, double lr, double holdout_fraction, uint64_t seed,
                double* out_coeffs, double* terms_out, double* report_out, int eik_fresh) {
    try {
        tg::SampleSet set;
        set.dim = dim;
        set.samples.resize(static_cast<std::size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            set.samples[i].point = {samples[4 * i], samples[4 * i + 1], dim == 3 ? samples[4 * i + 2] : 0.0};
            set.samples[i].gt_sdf = samples[4 * i + 3];
        }
        tg::FitOptions opt;
        opt.loss = make_loss(lambda1, lambda2, k, use_weighting, use_tv, 0);
        if (eik_fresh) opt.loss.eikonal_point_source = tg::EikonalPointSource::FreshUniform;
        opt.loss.batch_size = batch;
        opt.adam.lr = lr;
        opt.total_steps = total_steps;
        opt.holdout_fraction = holdout_fraction;
        opt.seed = seed;
        opt.threads = 1;
        const tg::FitResult r = tg::fit_sdf(set, make_spec(dim, res, origin, extent, order), opt);
        std::memcpy(out_coeffs, r.grid.coeffs.data(), r.grid.coeffs.size() * sizeof(double));
        for (std::size_t i = 0; i < r.trace.size(); ++i) {
            terms_out[4 * i] = r.trace[i].loss.total;
            terms_out[4 * i + 1] = r.trace[i].loss.fit;
            terms_out[4 * i + 2] = r.trace[i].loss.eik;
            terms_out[4 * i + 3] = r.trace[i].loss.tv;
        }
        report_out[0] = r.report.holdout_mae;
        report_out[1] = static_cast<double>(r.report.train_samples);
        report_out[2] = static_cast<double>(r.report.holdout_samples);
        return 0;
    } catch (const tg::NumericalError& e) {
        return fail(e, 4);
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// Rng::index stream (rng.hpp:27-35) and fit_sdf's seeded Fisher-Yates
// (sdf_fit.cpp:59-64) with tg::Rng.
int tgr_rng_index(uint64_t seed, uint64_t n, int64_t count, int64_t* out) {
    tg::Rng r(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = static_cast<int64_t>(r.index(n));
    return 0;
}

int tgr_shuffle_order(uint64_t seed, int64_t n, uint32_t* order) {
    for (int64_t i = 0; i < n; ++i) order[i] = static_cast<uint32_t>(i);
    tg::Rng shuffle_rng(seed);
    for (std::size_t i = static_cast<std::size_t>(n); i > 1; --i) std::swap(order[i - 1], order[shuffle_rng.index(i)]);
    return 0;
}

// trace_csv_string (schedule.cpp:110-120) of rows given as arrays.
int tgr_trace_csv(int nrows, const int* step_stage, const int* res3, const double* terms, const double* wall_ms,
                  const char* label, char* out, int64_t cap) {
    std::vector<tg::TraceRow> rows(static_cast<std::size_t>(nrows));
    for (int i = 0; i < nrows; ++i) {
        rows[i].step = step_stage[2 * i];
        rows[i].stage = step_stage[2 * i + 1];
        rows[i].resolution = {res3[3 * i], res3[3 * i + 1], res3[3 * i + 2]};
        rows[i].loss = {terms[4 * i], terms[4 * i + 1], terms[4 * i + 2], terms[4 * i + 3]};
        rows[i].wall_ms = wall_ms[i];
    }
    const std::string s = tg::trace_csv_string(rows, label);
    if (static_cast<int64_t>(s.size()) + 1 > cap) return -static_cast<int>(s.size() + 1);
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
}

// photometric_loss / render_ray (volume_render.cpp:194-276) on a density
// TaylorGrid and an SHColorGrid (sh.hpp:19-29). gt may be NULL (render only:
// colors_out / residual_out via render_ray); grads may be NULL.
int tgr_photometric_loss(int dim, const int* res, const double* origin, const double* extent, int order,
                         const double* dcoeffs, const int* sh_res, const double* sh_origin, const double* sh_extent,
                         int sh_degree, const double* sh_coeffs, int64_t nrays, const double* origins,
                         const double* dirs, const double* near_, const double* far_, const double* gt,
                         int n_samples, int activation, double shift, const double* bg, double* grad_density,
                         double* grad_sh, double* colors_out, double* residual_out, double* loss_out, int jitter,
                         uint64_t jitter_seed) {
    try {
        const tg::TaylorGrid dg = make_grid(make_spec(dim, res, origin, extent, order), dcoeffs);
        tg::SHColorGrid sg = tg::init_sh_grid(make_spec(3, sh_res, sh_origin, sh_extent, 0), sh_degree);
        std::memcpy(sg.coeffs.data(), sh_coeffs, sg.coeffs.size() * sizeof(double));
        tg::RenderOptions opt;
        opt.n_samples = n_samples;
        opt.activation = activation == 0 ? tg::DensityActivation::ShiftedSoftplus : tg::DensityActivation::ClampRelu;
        opt.softplus_shift = shift;
        opt.background = {bg[0], bg[1], bg[2]};
        opt.jitter = jitter != 0;
        opt.jitter_seed = jitter_seed;
        tg::RayBatch batch;
        for (int64_t r = 0; r < nrays; ++r) {
            batch.origins.push_back({origins[3 * r], origins[3 * r + 1], origins[3 * r + 2]});
            batch.directions.push_back({dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2]});
            batch.near.push_back(near_[r]);
            batch.far.push_back(far_[r]);
            if (gt) batch.gt_colors.push_back({gt[3 * r], gt[3 * r + 1], gt[3 * r + 2]});
        }
        if (colors_out || residual_out) {
            for (int64_t r = 0; r < nrays; ++r) {
                const tg::RayRenderResult rr = tg::render_ray(dg, sg, batch.origins[r], batch.directions[r],
                                                              near_[r], far_[r], opt, static_cast<uint64_t>(r));
                if (colors_out)
                    for (int c = 0; c < 3; ++c) colors_out[3 * r + c] = rr.color[c];
                if (residual_out) residual_out[r] = rr.residual_transmittance;
            }
        }
        if (gt) {
            std::span<double> gd, gs;
            if (grad_density) gd = std::span<double>(grad_density, dg.coeffs.size());
            if (grad_sh) gs = std::span<double>(grad_sh, sg.coeffs.size());
            *loss_out = tg::photometric_loss(dg, sg, batch, opt, gd, gs, 1);
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// Schedule::progressive (schedule.cpp:27-54): writes up to 3 stages.
int tgr_schedule_progressive(const int* target, int dim, int total_steps, int* nstages, int* stage_res,
                             int* stage_steps) {
    const auto s = tg::Schedule::progressive({target[0], target[1], target[2]}, dim, total_steps);
    *nstages = static_cast<int>(s.stages.size());
    for (std::size_t i = 0; i < s.stages.size(); ++i) {
        for (int a = 0; a < 3; ++a) stage_res[3 * i + a] = s.stages[i].resolution[a];
        stage_steps[i] = s.stages[i].steps;
    }
    return 0;
}

// sample_grid_field (marching.cpp:53-58) for dim 3; for dim 2 the CLI's
// sample_grid_field2 lattice (tools/main.cpp:33-45, position() of
// marching.hpp:34-36) evaluated with the reference eval.
int tgr_sample_grid_field(int dim, const int* res, const double* origin, const double* extent, int order,
                          const double* coeffs, const int* lattice, double* out) {
    try {
        const auto spec = make_spec(dim, res, origin, extent, order);
        const tg::TaylorGrid grid = make_grid(spec, coeffs);
        if (dim == 3) {
            const tg::ScalarField3 f = tg::sample_grid_field(grid, {lattice[0], lattice[1], lattice[2]}, 1);
            std::memcpy(out, f.values.data(), f.values.size() * sizeof(double));
        } else {
            tg::ScalarField2 f;
            f.res = {lattice[0], lattice[1]};
            f.origin = {origin[0], origin[1]};
            f.extent = {extent[0], extent[1]};
            for (int y = 0; y < lattice[1]; ++y)
                for (int x = 0; x < lattice[0]; ++x) {
                    const auto p = f.position(x, y);
                    out[static_cast<std::size_t>(y) * lattice[0] + x] = tg::eval(grid, {p[0], p[1], 0.0});
                }
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// save_tgrid / load_tgrid (grid_io.cpp:36-111).
int tgr_save_tgrid(int dim, const int* res, const double* origin, const double* extent, int order,
                   const double* coeffs, const char* path, int precision) {
    try {
        const auto spec = make_spec(dim, res, origin, extent, order);
        tg::save_tgrid(make_grid(spec, coeffs), path, static_cast<tg::StoragePrecision>(precision));
        return 0;
    } catch (const tg::IngestError& e) {
        return fail(e, 3);
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// Loads a file; spec_out = {dim, order, res[3]} as ints, geo_out = origin[3],
// extent[3]; coeffs_out may be NULL (query the size first).
int tgr_load_tgrid(const char* path, int* spec_out, double* geo_out, double* coeffs_out, int64_t cap) {
    try {
        const tg::TaylorGrid g = tg::load_tgrid(path);
        spec_out[0] = g.spec.dim;
        spec_out[1] = g.spec.order;
        for (int a = 0; a < 3; ++a) {
            spec_out[2 + a] = g.spec.resolution[a];
            geo_out[a] = g.spec.origin[a];
            geo_out[3 + a] = g.spec.extent[a];
        }
        if (coeffs_out) {
            if (static_cast<int64_t>(g.coeffs.size()) > cap) throw std::invalid_argument("tgr_load_tgrid: cap");
            std::memcpy(coeffs_out, g.coeffs.data(), g.coeffs.size() * sizeof(double));
        }
        return static_cast<int>(0);
    } catch (const tg::IngestError& e) {
        return fail(e, 3);
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

}  // extern "C"
