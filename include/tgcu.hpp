// tgcu.hpp — header-only C++ shim over the C ABI (tgcu.h) in the shape of the
// reference's tg:: API (/root/reference/proj/core/include/taylorgrid/*.hpp),
// so reference callers (run_schedule, cmd_bench, TrainProblem subclasses) can
// drive the B200 path with the same names, argument meaning and exception
// types (errors.hpp:9-34; std::invalid_argument for require_arg failures).
//
// When the reference's headers are on the include path (taylorgrid/errors.hpp
// found by __has_include), the exceptions thrown ARE tg::ConfigError,
// tg::IngestError, tg::NumericalError and tg::ResourceError, so code that
// catches the reference's types catches ours; otherwise look-alike classes of
// the same names live in namespace tgcu. include/tgcu_tg.hpp adds the
// adapters to the reference's own types (tg::TaylorGrid, tg::Schedule,
// tg::TrainProblem, tg::ScheduleResult).
#pragma once

#include <array>
#include <cstdint>
#include <exception>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tgcu.h"

#if defined(__has_include)
#if __has_include("taylorgrid/errors.hpp")
#include "taylorgrid/errors.hpp"
#define TGCU_WITH_REFERENCE_TYPES 1
#endif
#endif

namespace tgcu {

#ifdef TGCU_WITH_REFERENCE_TYPES
using ConfigError = tg::ConfigError;
using IngestError = tg::IngestError;
using NumericalError = tg::NumericalError;
using ResourceError = tg::ResourceError;
#else
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IngestError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NumericalError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ResourceError : std::runtime_error { using std::runtime_error::runtime_error; };
#endif
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
    ~Grid() {
        if (h_) tgcu_grid_destroy(h_);
    }
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
    // Give up ownership of the handle (the caller destroys it).
    tgcu_grid* release() { return std::exchange(h_, nullptr); }
    Grid& operator=(Grid&& o) noexcept {
        if (this != &o) {
            if (h_) tgcu_grid_destroy(h_);
            h_ = std::exchange(o.h_, nullptr);
        }
        return *this;
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

// tg::IouOptions / iou (metrics.cpp:104-124) with field a on the device: b is
// another grid, or (nullptr) the sphere |p| - radius of cmd_bench's probe.
struct IouOptions {
    int64_t samples = 100000;
    uint64_t seed = 7;
    std::array<double, 3> domain_lo{-1.0, -1.0, -1.0};
    std::array<double, 3> domain_hi{1.0, 1.0, 1.0};
    int dim = 3;
};
struct IouResult {
    double iou = 0.0;
    bool empty_union = false;
};
inline IouResult iou(const Grid& a, const Grid* b, double sphere_radius, const IouOptions& o = {}) {
    tgcu_iou_options c{o.samples, o.seed, {o.domain_lo[0], o.domain_lo[1], o.domain_lo[2]},
                       {o.domain_hi[0], o.domain_hi[1], o.domain_hi[2]}, o.dim};
    IouResult r;
    int empty = 0;
    check(tgcu_iou(a.handle(), b ? b->handle() : nullptr, sphere_radius, &c, &r.iou, &empty));
    r.empty_union = empty != 0;
    return r;
}

// Schedule::Stage / Schedule / TraceRow (schedule.hpp:16-56).
struct Stage {
    std::array<int, 3> resolution{2, 2, 2};
    int steps = 0;
};
struct Schedule {
    std::vector<Stage> stages;
    int total_steps() const {
        int n = 0;
        for (const Stage& s : stages) n += s.steps;
        return n;
    }
    void validate(int dim) const {
        const std::vector<tgcu_stage> c = cstages();
        check(tgcu_schedule_validate(c.data(), static_cast<int>(c.size()), dim));
    }
    static Schedule progressive(const std::array<int, 3>& target, int dim, int total_steps) {
        tgcu_stage out[3];
        int n = 0;
        check(tgcu_schedule_progressive(target.data(), dim, total_steps, out, &n));
        Schedule s;
        for (int i = 0; i < n; ++i) s.stages.push_back({{out[i].res[0], out[i].res[1], out[i].res[2]}, out[i].steps});
        return s;
    }
    static Schedule single(const std::array<int, 3>& target, int steps) { return Schedule{{Stage{target, steps}}}; }
    std::vector<tgcu_stage> cstages() const {
        std::vector<tgcu_stage> c;
        for (const Stage& s : stages) c.push_back({{s.resolution[0], s.resolution[1], s.resolution[2]}, s.steps});
        return c;
    }
};
using TraceRow = tgcu_trace_row;

// The device form of tg::TrainProblem (schedule.hpp:60-66): the step's batch
// (the fused step does the loss, gradient and Adam). batch() returns n x 4
// floats; host memory may be refilled on the next call.
class TrainProblem {
public:
    virtual ~TrainProblem() = default;
    struct Batch {
        const float* samples = nullptr;
        int64_t n = 0;
        bool host = true;
        bool ready = false;  // device batch already complete (its binning may overlap the previous step)
    };
    virtual Batch batch(int64_t global_step) = 0;
    virtual void on_stage_start(Grid& grid, int stage) { (void)grid; (void)stage; }
};

struct ScheduleResult {
    Grid grid;
    std::vector<TraceRow> trace;
    std::vector<double> stage_seconds;
};

// run_schedule (schedule.cpp:62-108) on the device: per stage upsample +
// fresh Adam moments + on_stage_start, then fused steps. asynchronous: no
// host round trip per step (trace wall_ms = the window's mean).
inline ScheduleResult run_schedule(TrainProblem& problem, const Schedule& schedule, Grid grid,
                                   const AdamConfig& adam, const LossConfig& loss, bool asynchronous = true) {
    struct Ctx {
        TrainProblem* p;
        std::exception_ptr err;
    } ctx{&problem, nullptr};
    auto batch_fn = [](void* u, tgcu_grid*, int64_t step, const float** smp, int64_t* n, int* flags) -> int {
        Ctx* c = static_cast<Ctx*>(u);
        try {
            const TrainProblem::Batch b = c->p->batch(step);
            *smp = b.samples;
            *n = b.n;
            *flags = (b.host ? TGCU_HOST : 0) | (b.ready ? TGCU_INPUT_READY : 0);
            return TGCU_OK;
        } catch (...) {
            c->err = std::current_exception();
            return TGCU_ERR_INVALID_ARGUMENT;
        }
    };
    auto stage_fn = [](void* u, tgcu_grid* g, int stage) -> int {
        Ctx* c = static_cast<Ctx*>(u);
        try {
            Grid view = Grid::adopt(g);  // non-owning for the callback's duration
            c->p->on_stage_start(view, stage);
            view.release();
            return TGCU_OK;
        } catch (...) {
            c->err = std::current_exception();
            return TGCU_ERR_INVALID_ARGUMENT;
        }
    };
    const std::vector<tgcu_stage> st = schedule.cstages();
    ScheduleResult r{std::move(grid), std::vector<TraceRow>(static_cast<size_t>(schedule.total_steps())),
                     std::vector<double>(st.size())};
    tgcu_grid* h = r.grid.release();
    const tgcu_adam_config a{adam.lr, adam.beta1, adam.beta2, adam.eps};
    const tgcu_loss_config l = loss.c();
    const int rc = tgcu_run_schedule(&h, st.data(), static_cast<int>(st.size()), &a, &l, batch_fn, stage_fn, &ctx,
                                     asynchronous ? TGCU_ASYNC : 0, nullptr, r.trace.data(), r.stage_seconds.data());
    r.grid = Grid::adopt(h);
    if (ctx.err) std::rethrow_exception(ctx.err);
    check(rc);
    return r;
}

// Pinned host memory for batches fed through the pipelined host path (the
// library copies pageable memory synchronously).
template <class T>
class PinnedBuffer {
public:
    explicit PinnedBuffer(size_t n) : n_(n) { check(tgcu_host_alloc(reinterpret_cast<void**>(&p_), n * sizeof(T))); }
    ~PinnedBuffer() { tgcu_host_free(p_); }
    PinnedBuffer(const PinnedBuffer&) = delete;
    PinnedBuffer& operator=(const PinnedBuffer&) = delete;
    T* data() { return p_; }
    size_t size() const { return n_; }
    std::span<T> span() { return {p_, n_}; }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
};

// CUDA-graph replay of small-grid training steps (tgcu_train_graph_*): the
// steps on device batches batches[0..n-1] (n even; n_pts x 4 floats each,
// kept by the graph) captured once on a non-default stream, replayed with
// replay(stream). Errors surface at the grid's next sync, as for asynchronous
// steps.
class TrainGraph {
public:
    TrainGraph(Grid& g, const std::vector<const float*>& batches, int64_t n_pts, const LossConfig& cfg,
               void* stream) {
        const tgcu_loss_config c = cfg.c();
        check(tgcu_train_graph_create(g.handle(), batches.data(), static_cast<int>(batches.size()), n_pts, &c,
                                      stream, &h_));
    }
    ~TrainGraph() { tgcu_train_graph_destroy(h_); }
    TrainGraph(const TrainGraph&) = delete;
    TrainGraph& operator=(const TrainGraph&) = delete;
    void replay(void* stream) { check(tgcu_train_graph_launch(h_, stream)); }

private:
    tgcu_graph* h_ = nullptr;
};

}  // namespace tgcu
