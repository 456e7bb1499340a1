// tgcu.hpp — header-only C++ shim over the C ABI (tgcu.h) in the shape of the
// reference's tg:: API (/root/reference/proj/core/include/taylorgrid/*.hpp),
// so reference callers (run_schedule, cmd_bench, TrainProblem subclasses) can
// drive the B200 path with the same names, argument meaning and exception
// types (errors.hpp:9-34; std::invalid_argument for require_arg failures).
#pragma once

#include <array>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tgcu.h"

namespace tgcu {

struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IngestError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NumericalError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ResourceError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

// Status -> the reference's exception classes.
inline void check(int rc) {
    if (rc == TGCU_OK) return;
    const std::string msg = tgcu_last_error();
    switch (rc) {
        case TGCU_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case TGCU_ERR_CONFIG: throw ConfigError(msg);
        case TGCU_ERR_INGEST: throw IngestError(msg);
        case TGCU_ERR_NUMERICAL: throw NumericalError(msg);
        case TGCU_ERR_RESOURCE: throw ResourceError(msg);
        default: throw CudaError(msg);
    }
}

inline int coeff_count(int order, int dim) {
    int k = 0;
    check(tgcu_coeff_count(order, dim, &k));
    return k;
}

// tg::LossTerms / tg::LossConfig / tg::AdamConfig equivalents.
using LossTerms = tgcu_loss_terms;
struct LossConfig {
    double lambda1 = 1e-4, lambda2 = 2e-5, k = 50.0;
    bool use_weighting = true, use_tv = true, differentiate_weight = false;
    tgcu_loss_config c() const {
        return {lambda1, lambda2, k, use_weighting ? 1 : 0, use_tv ? 1 : 0, differentiate_weight ? 1 : 0};
    }
};
struct AdamConfig {
    double lr = 0.003, beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
};

// A device-resident tg::TaylorGrid together with its AdamState.
class Grid {
public:
    explicit Grid(const tgcu_grid_spec& spec, const tgcu_init_options* opts = nullptr, int device = 0) {
        check(tgcu_grid_create(&spec, opts, device, &h_));
    }
    ~Grid() { tgcu_grid_destroy(h_); }
    Grid(const Grid&) = delete;
    Grid& operator=(const Grid&) = delete;
    Grid(Grid&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}

    tgcu_grid* handle() const { return h_; }
    int64_t coeff_total() const { return tgcu_grid_coeff_total(h_); }

    // TaylorGrid::coeffs in the reference layout (fp64 at the boundary).
    std::vector<double> coeffs() const {
        std::vector<double> c(static_cast<size_t>(coeff_total()));
        check(tgcu_grid_download_f64(h_, c.data(), static_cast<int64_t>(c.size())));
        return c;
    }
    void set_coeffs(std::span<const double> c) {
        check(tgcu_grid_upload_f64(h_, c.data(), static_cast<int64_t>(c.size())));
    }

    // eval / eval_with_spatial_gradient, batched over host fp32 points (n x 3).
    std::vector<float> eval(std::span<const float> pts, std::vector<float>* spatial_grad = nullptr) const {
        const int64_t n = static_cast<int64_t>(pts.size() / 3);
        std::vector<float> v(static_cast<size_t>(n));
        if (spatial_grad) spatial_grad->assign(static_cast<size_t>(3 * n), 0.0f);
        check(tgcu_eval(h_, pts.data(), n, v.data(), spatial_grad ? spatial_grad->data() : nullptr, TGCU_HOST,
                        nullptr));
        return v;
    }

    // AdamState::reset + config.
    void adam_reset(const AdamConfig& a) {
        const tgcu_adam_config c{a.lr, a.beta1, a.beta2, a.eps};
        check(tgcu_adam_reset(h_, &c));
    }

    // One run_schedule step (schedule.cpp:66-92): zero grad, total_loss,
    // finite-loss check, adam_step. samples: host n x 4 (x, y, z, gt).
    LossTerms train_step(std::span<const float> samples, const LossConfig& cfg) {
        const tgcu_loss_config c = cfg.c();
        LossTerms t{};
        check(tgcu_train_step(h_, samples.data(), static_cast<int64_t>(samples.size() / 4), &c, &t, TGCU_HOST,
                              nullptr));
        return t;
    }

    // Pipelined form of train_step (the cmd_bench loop at full speed): the
    // host batch is copied on the library's copy stream while earlier steps
    // compute, nothing synchronises; `samples` must stay valid and
    // unmodified until sync(): the copy may still be in flight, so refilling
    // the same buffer for the next step corrupts it (cycle >= 2 buffers).
    // Errors surface from sync() with the grid rolled back to the last
    // committed step (NumericalError / std::invalid_argument as above).
    void train_step_async(std::span<const float> samples, const LossConfig& cfg) {
        const tgcu_loss_config c = cfg.c();
        check(tgcu_train_step(h_, samples.data(), static_cast<int64_t>(samples.size() / 4), &c, nullptr,
                              TGCU_HOST | TGCU_ASYNC, nullptr));
    }
    LossTerms sync() {
        LossTerms t{};
        check(tgcu_sync(h_, &t));
        return t;
    }

    tgcu_grid_spec spec() const {
        tgcu_grid_spec s{};
        tgcu_grid_spec_of(h_, &s);
        return s;
    }

    // sample_grid_field (marching.cpp:53-58): values on an n0 x n1 x n2 lattice
    // of the grid's domain, x fastest.
    std::vector<float> sample_grid_field(const std::array<int, 3>& lattice) const {
        const size_t n = static_cast<size_t>(lattice[0]) * lattice[1] * (spec().dim == 3 ? lattice[2] : 1);
        std::vector<float> v(n);
        check(tgcu_sample_grid_field(h_, lattice.data(), v.data(), TGCU_HOST, nullptr));
        return v;
    }

    // save_tgrid (grid_io.cpp:44-65); precision TGCU_TGRID_F64 / _F32.
    void save_tgrid(const char* path, int precision = TGCU_TGRID_F64) const {
        check(tgcu_save_tgrid(h_, path, precision));
    }

    static Grid adopt(tgcu_grid* h) {
        Grid g;
        g.h_ = h;
        return g;
    }

private:
    Grid() = default;
    tgcu_grid* h_ = nullptr;
};

// upsample (taylor_grid.cpp:273-284): a new grid at new_res.
inline Grid upsample(const Grid& g, const std::array<int, 3>& new_res) {
    tgcu_grid_spec s = g.spec();
    for (int a = 0; a < 3; ++a) s.res[a] = new_res[a];
    Grid out(s);
    check(tgcu_grid_upsample(g.handle(), out.handle(), 0, nullptr));
    return out;
}

// load_tgrid (grid_io.cpp:67-109).
inline Grid load_tgrid(const char* path, int device = 0) {
    tgcu_grid* h = nullptr;
    check(tgcu_load_tgrid(path, device, &h));
    return Grid::adopt(h);
}

}  // namespace tgcu
