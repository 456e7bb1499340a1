// tgcu_tg.hpp — adapters between the reference's own C++ types
// (/root/reference/proj/core/include/taylorgrid: tg::TaylorGrid, tg::Schedule,
// tg::TrainProblem, tg::ScheduleResult, tg::LossConfig, tg::AdamConfig) and
// the B200 path. Include with the reference's include directory on the path;
// the reference library (taylorgrid::core) supplies tg::Schedule::validate /
// upsample / trace_csv_string etc. as before. Two ways to run a reference
// training loop on the device:
//
//  1. tgcu::run_schedule(problem, tg::Schedule, tg::TaylorGrid, tg::AdamConfig,
//     tg::LossConfig) -> tg::ScheduleResult: the whole loop on the device
//     (fused step: loss + backward + TV + finite check + Adam; upsample and
//     Adam reset per stage), with the reference's signature and result type.
//     tgcu::SdfProblem reproduces SdfProblem's batch stream (sdf_fit.cpp:14-32,
//     the reference Rng's index draws, bit for bit).
//  2. tgcu::GpuSdfProblem, a tg::TrainProblem: the reference's own
//     tg::run_schedule (host Adam in fp64) with compute() — total_loss and its
//     gradient — on the device. A drop-in for the plugin point
//     (schedule.hpp:60-66); the coefficients cross PCIe every step, so it is
//     the compatibility path, not the fast one.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <span>
#include <vector>

#include "taylorgrid/rng.hpp"
#include "taylorgrid/sample_set.hpp"
#include "taylorgrid/schedule.hpp"
#include "taylorgrid/sdf_loss.hpp"
#include "taylorgrid/taylor_grid.hpp"
#include "tgcu.hpp"

namespace tgcu {

inline tgcu_grid_spec to_spec(const tg::GridSpec& s) {
    tgcu_grid_spec c{};
    c.dim = s.dim;
    for (int a = 0; a < 3; ++a) {
        c.res[a] = s.resolution[a];
        c.origin[a] = s.origin[a];
        c.extent[a] = s.extent[a];
    }
    c.order = s.order;
    return c;
}

inline LossConfig to_loss(const tg::LossConfig& l) {
    LossConfig c;
    c.lambda1 = l.lambda1;
    c.lambda2 = l.lambda2;
    c.k = l.k;
    c.use_weighting = l.use_weighting;
    c.use_tv = l.use_tv;
    c.differentiate_weight = l.differentiate_weight;
    return c;
}

inline AdamConfig to_adam(const tg::AdamConfig& a) { return AdamConfig{a.lr, a.beta1, a.beta2, a.eps}; }

inline Schedule to_schedule(const tg::Schedule& s) {
    Schedule out;
    for (const auto& st : s.stages) out.stages.push_back(Stage{st.resolution, st.steps});
    return out;
}

// tg::TaylorGrid -> device grid (memory cap lifted: the reference grid already exists).
inline Grid to_device(const tg::TaylorGrid& g, int device = 0) {
    const tgcu_grid_spec s = to_spec(g.spec);
    tgcu_init_options o{TGCU_INIT_ZEROS, 0.0, 1e-4, 0, ~0ull};
    Grid d(s, &o, device);
    d.set_coeffs(g.coeffs);
    return d;
}

// device grid -> tg::TaylorGrid (fp32 coefficients widened exactly).
inline tg::TaylorGrid to_host(const Grid& d, const tg::GridSpec& like) {
    tg::TaylorGrid g;
    g.spec = like;
    const tgcu_grid_spec s = d.spec();
    for (int a = 0; a < 3; ++a) g.spec.resolution[a] = s.res[a];
    g.coeffs = d.coeffs();
    return g;
}

inline tg::TraceRow to_trace_row(const TraceRow& r) {
    tg::TraceRow t;
    t.step = static_cast<int>(r.step);
    t.stage = r.stage;
    t.resolution = {r.res[0], r.res[1], r.res[2]};
    t.loss = tg::LossTerms{r.loss.total, r.loss.fit, r.loss.eik, r.loss.tv};
    t.wall_ms = r.wall_ms;
    return t;
}

// SdfProblem (sdf_fit.cpp:14-32) for the device loop: each step draws
// min(batch_size, |train|) samples with replacement with the reference Rng
// (same seed -> the same index stream as the reference's SdfProblem), as
// fp32 (x, y, z, gt) in a reused host buffer.
class SdfProblem : public TrainProblem {
public:
    SdfProblem(std::vector<tg::SdfSample> train, const tg::LossConfig& cfg, std::uint64_t seed)
        : train_(std::move(train)), rng_(seed),
          buf_(4 * std::min<std::size_t>(static_cast<std::size_t>(cfg.batch_size), train_.size())) {}

    Batch batch(int64_t) override {
        const std::size_t n = buf_.size() / 4;
        for (std::size_t i = 0; i < n; ++i) {
            const tg::SdfSample& s = train_[rng_.index(train_.size())];
            buf_[4 * i] = static_cast<float>(s.point[0]);
            buf_[4 * i + 1] = static_cast<float>(s.point[1]);
            buf_[4 * i + 2] = static_cast<float>(s.point[2]);
            buf_[4 * i + 3] = static_cast<float>(s.gt_sdf);
        }
        return Batch{buf_.data(), static_cast<int64_t>(n), true, false};
    }

private:
    std::vector<tg::SdfSample> train_;
    tg::Rng rng_;
    std::vector<float> buf_;
};

// run_schedule with the reference's signature and result type, on the device.
inline tg::ScheduleResult run_schedule(TrainProblem& problem, const tg::Schedule& schedule, tg::TaylorGrid grid,
                                       const tg::AdamConfig& adam, const tg::LossConfig& loss, int device = 0,
                                       bool asynchronous = true) {
    schedule.validate(grid.spec.dim);  // the reference's own check and messages
    const tg::GridSpec like = grid.spec;
    ScheduleResult r = run_schedule(problem, to_schedule(schedule), to_device(grid, device), to_adam(adam),
                                    to_loss(loss), asynchronous);
    tg::ScheduleResult out;
    out.grid = to_host(r.grid, like);
    for (const TraceRow& row : r.trace) out.trace.push_back(to_trace_row(row));
    out.stage_seconds = r.stage_seconds;
    return out;
}

// A tg::TrainProblem whose compute() runs on the device: the batch draw of
// SdfProblem (reference Rng), then total_loss with its gradient
// (tgcu_total_loss) on a device copy of the current grid; the gradient
// comes back in fp64 into the reference's buffer. Drop-in for the
// reference's own tg::run_schedule / fit loops.
class GpuSdfProblem final : public tg::TrainProblem {
public:
    GpuSdfProblem(std::vector<tg::SdfSample> train, const tg::LossConfig& cfg, std::uint64_t seed, int device = 0)
        : train_(std::move(train)), cfg_(cfg), rng_(seed), device_(device),
          buf_(4 * std::min<std::size_t>(static_cast<std::size_t>(cfg.batch_size), train_.size())) {}

    tg::LossTerms compute(const tg::TaylorGrid& grid, std::span<double> grad) override {
        const tgcu_grid_spec s = to_spec(grid.spec);
        if (!dev_ || std::memcmp(&s, &spec_, sizeof(s)) != 0) {
            tgcu_init_options o{TGCU_INIT_ZEROS, 0.0, 1e-4, 0, ~0ull};
            dev_ = std::make_unique<Grid>(s, &o, device_);
            spec_ = s;
            host_grad_.assign(grid.coeffs.size(), 0.0);
        }
        dev_->set_coeffs(grid.coeffs);
        const std::size_t n = buf_.size() / 4;
        for (std::size_t i = 0; i < n; ++i) {
            const tg::SdfSample& smp = train_[rng_.index(train_.size())];
            for (int a = 0; a < 3; ++a) buf_[4 * i + a] = static_cast<float>(smp.point[a]);
            buf_[4 * i + 3] = static_cast<float>(smp.gt_sdf);
        }
        tgcu_grid* h = dev_->handle();
        check(tgcu_grad_zero(h, nullptr, nullptr));
        const tgcu_loss_config c = to_loss(cfg_).c();
        tgcu_loss_terms t{};
        check(tgcu_total_loss(h, buf_.data(), static_cast<int64_t>(n), &c, tgcu_grid_grad(h), &t, TGCU_HOST, nullptr));
        check(tgcu_grad_download_f64(h, nullptr, host_grad_.data(), static_cast<int64_t>(host_grad_.size())));
        for (std::size_t i = 0; i < grad.size(); ++i) grad[i] += host_grad_[i];
        return tg::LossTerms{t.total, t.fit, t.eik, t.tv};
    }

private:
    std::vector<tg::SdfSample> train_;
    tg::LossConfig cfg_;
    tg::Rng rng_;
    int device_;
    std::vector<float> buf_;
    std::unique_ptr<Grid> dev_;
    tgcu_grid_spec spec_{};
    std::vector<double> host_grad_;
};

}  // namespace tgcu
