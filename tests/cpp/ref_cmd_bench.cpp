// TEST INFRASTRUCTURE: a reference-style C++ tool on the B200 path.
//
// Written against the reference's own headers and types (tg::SamplingConfig,
// tg::sample_sphere_points, tg::Schedule, tg::TaylorGrid, tg::TrainProblem,
// tg::run_schedule, tg::iou, tg::trace_csv_string; linked with the
// reference library built by oracle/Makefile, as the reference CLI links
// taylorgrid::core) and include/tgcu_tg.hpp, the way a maintainer would
// switch cmd_bench (tools/main.cpp:587-683) and fit_sdf's loop
// (sdf_fit.cpp:52-105) to libtgcu. Built by __graft_entry__.build() when the
// reference sources are present; run by tests/test_cpp_shim.py on a GPU.
//
// Checks, each against the reference run live in this process:
//   1. tgcu::run_schedule (fused device loop, reference signature / result
//      type) vs tg::run_schedule with the reference's SdfProblem batch stream:
//      LossTerms of the first 20 steps within 1e-4;
//   2. tg::run_schedule (the reference's own loop, host fp64 Adam) with
//      tgcu::GpuSdfProblem (loss + gradient on the device): first 10 steps
//      within 1e-4;
//   3. a progressive 3-stage schedule on the device: stages / resolutions /
//      trace CSV as the reference's tg::Schedule::progressive plans them;
//   4. cmd_bench's loop (orders 1 and 2): device training with the reference
//      batch draws, the IoU probe on the device (tgcu::iou) equal to tg::iou
//      on the downloaded grid evaluated by the reference;
//   5. a NaN sample surfaces as the reference's tg::NumericalError.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "taylorgrid/adam.hpp"
#include "taylorgrid/errors.hpp"
#include "taylorgrid/metrics.hpp"
#include "taylorgrid/sampling.hpp"
#include "taylorgrid/schedule.hpp"
#include "taylorgrid/sdf_loss.hpp"
#include "taylorgrid/taylor_grid.hpp"
#include "tgcu_tg.hpp"

namespace {

int failures = 0;

void expect(bool ok, const std::string& what) {
    std::printf("%s %s\n", ok ? "ok  " : "FAIL", what.c_str());
    if (!ok) ++failures;
}

// The reference's SdfProblem (sdf_fit.cpp:14-32, anonymous there): restated
// from its public pieces for the CPU side of the comparison.
class RefSdfProblem final : public tg::TrainProblem {
public:
    RefSdfProblem(std::vector<tg::SdfSample> train, const tg::LossConfig& cfg, std::uint64_t seed)
        : train_(std::move(train)), cfg_(cfg), rng_(seed), batch_(std::min<std::size_t>(cfg.batch_size, train_.size())) {}
    tg::LossTerms compute(const tg::TaylorGrid& grid, std::span<double> grad) override {
        for (auto& s : batch_) {
            s = train_[rng_.index(train_.size())];
            // the device path sees fp32 samples: hand the reference the same values
            for (int a = 0; a < 3; ++a) s.point[a] = static_cast<float>(s.point[a]);
            s.gt_sdf = static_cast<float>(s.gt_sdf);
        }
        return tg::total_loss(grid, batch_, cfg_, grad, 8, &rng_);
    }

private:
    std::vector<tg::SdfSample> train_;
    tg::LossConfig cfg_;
    tg::Rng rng_;
    std::vector<tg::SdfSample> batch_;
};

double max_rel(const std::vector<tg::TraceRow>& a, const std::vector<tg::TraceRow>& b, std::size_t steps) {
    double m = 0.0;
    for (std::size_t i = 0; i < steps && i < a.size() && i < b.size(); ++i) {
        const double x[4] = {a[i].loss.total, a[i].loss.fit, a[i].loss.eik, a[i].loss.tv};
        const double y[4] = {b[i].loss.total, b[i].loss.fit, b[i].loss.eik, b[i].loss.tv};
        for (int k = 0; k < 4; ++k)
            if (y[k] != 0.0) m = std::max(m, std::abs(x[k] - y[k]) / std::abs(y[k]));
    }
    return m;
}

}  // namespace

int main() {
    tg::SamplingConfig scfg;
    scfg.total = 200000;
    scfg.seed = 3;
    const tg::SampleSet samples = tg::sample_sphere_points(0.5, scfg);
    tg::LossConfig loss;  // paper defaults, batch 8192
    const tg::AdamConfig adam{1e-2, 0.9, 0.999, 1e-8};
    tg::GridSpec spec;
    spec.dim = 3;
    spec.resolution = {40, 40, 40};
    spec.order = 2;

    // 1. fused device loop vs the reference loop, same batch stream
    {
        const tg::Schedule sch = tg::Schedule::single(spec.resolution, 40);
        RefSdfProblem ref_p(samples.samples, loss, 11);
        const tg::ScheduleResult ref = tg::run_schedule(ref_p, sch, tg::init_grid(spec), adam, 8);
        tgcu::SdfProblem dev_p(samples.samples, loss, 11);
        const tg::ScheduleResult dev = tgcu::run_schedule(dev_p, sch, tg::init_grid(spec), adam, loss);
        const double d = max_rel(dev.trace, ref.trace, 20);
        char buf[160];
        std::snprintf(buf, sizeof(buf), "tgcu::run_schedule vs tg::run_schedule, steps 0-19: max rel %.3g (<= 1e-4)", d);
        expect(dev.trace.size() == 40 && d <= 1e-4, buf);
        expect(dev.grid.coeffs.size() == ref.grid.coeffs.size(), "tg::ScheduleResult grid returned in the reference layout");
    }
    // 2. the reference's own run_schedule with the device TrainProblem
    {
        const tg::Schedule sch = tg::Schedule::single(spec.resolution, 12);
        RefSdfProblem ref_p(samples.samples, loss, 12);
        const tg::ScheduleResult ref = tg::run_schedule(ref_p, sch, tg::init_grid(spec), adam, 8);
        tgcu::GpuSdfProblem gpu_p(samples.samples, loss, 12);
        const tg::ScheduleResult mixed = tg::run_schedule(gpu_p, sch, tg::init_grid(spec), adam, 8);
        const double d = max_rel(mixed.trace, ref.trace, 10);
        char buf[160];
        std::snprintf(buf, sizeof(buf), "tg::run_schedule + tgcu::GpuSdfProblem, steps 0-9: max rel %.3g (<= 1e-4)", d);
        expect(d <= 1e-4, buf);
    }
    // 3. progressive schedule on the device
    {
        const tg::Schedule sch = tg::Schedule::progressive(spec.resolution, 3, 30);
        tg::GridSpec s0 = spec;
        s0.resolution = sch.stages.front().resolution;
        tgcu::SdfProblem dev_p(samples.samples, loss, 13);
        const tg::ScheduleResult dev = tgcu::run_schedule(dev_p, sch, tg::init_grid(s0), adam, loss);
        bool ok = dev.trace.size() == 30 && dev.stage_seconds.size() == sch.stages.size() &&
                  dev.grid.spec.resolution == spec.resolution;
        for (const auto& r : dev.trace) ok &= r.resolution == sch.stages[r.stage].resolution && std::isfinite(r.loss.total);
        const std::string csv = tg::trace_csv_string(dev.trace, "recon");
        ok &= csv.rfind("step,stage,resolution,total_loss,recon,eik,tv,wall_ms\n", 0) == 0;
        expect(ok, "progressive schedule (" + std::to_string(sch.stages.size()) + " stages) through the device loop, "
                   "trace CSV by the reference's writer");
    }
    // 4. cmd_bench's loop with the IoU probe
    for (int order : {1, 2}) {
        tg::GridSpec bs = spec;
        bs.resolution = {32, 32, 32};
        bs.order = order;
        tgcu::Grid g = tgcu::to_device(tg::init_grid(bs));
        g.adam_reset(tgcu::to_adam(adam));
        tg::Rng rng(scfg.seed ^ (0xb0 + order));
        std::vector<float> batch(4 * loss.batch_size);
        tgcu::LossConfig lc = tgcu::to_loss(loss);
        double loss_value = 0.0;
        for (int step = 0; step < 150; ++step) {
            for (int i = 0; i < loss.batch_size; ++i) {
                const tg::SdfSample& s = samples.samples[rng.index(samples.samples.size())];
                for (int a = 0; a < 3; ++a) batch[4 * i + a] = static_cast<float>(s.point[a]);
                batch[4 * i + 3] = static_cast<float>(s.gt_sdf);
            }
            loss_value = g.train_step(batch, lc).total;
        }
        tg::IouOptions io;
        io.samples = 100000;
        io.seed = scfg.seed;
        tgcu::IouOptions dio;
        dio.samples = io.samples;
        dio.seed = io.seed;
        const double dev_iou = tgcu::iou(g, nullptr, 0.5, dio).iou;
        const tg::TaylorGrid hg = tgcu::to_host(g, bs);
        const auto gt = [](const tg::Vec3& p) { return tg::norm(p) - 0.5; };
        const double ref_iou = tg::iou([&](const tg::Vec3& p) { return tg::eval(hg, p); }, gt, io).iou;
        char buf[200];
        std::snprintf(buf, sizeof(buf), "cmd_bench order %d: loss %.4g, IoU device %.6f vs reference %.6f (|d| <= 3e-5)",
                      order, loss_value, dev_iou, ref_iou);
        expect(std::abs(dev_iou - ref_iou) <= 3e-5 && dev_iou > 0.8, buf);
    }
    // 5. the reference's exception types
    try {
        tgcu::Grid g = tgcu::to_device(tg::init_grid(spec));
        g.adam_reset(tgcu::to_adam(adam));
        std::vector<float> b(4 * 1024, 0.1f);
        b[4 * 7 + 3] = NAN;
        g.train_step(b, tgcu::to_loss(loss));
        expect(false, "NaN target raises");
    } catch (const tg::NumericalError& e) {
        expect(std::string(e.what()).find("non-finite loss at stage 0 step 0") != std::string::npos,
               std::string("tg::NumericalError: ") + e.what());
    }
    try {
        tgcu::coeff_count(3, 3);
        expect(false, "bad order raises");
    } catch (const std::invalid_argument& e) {
        expect(true, std::string("std::invalid_argument: ") + e.what());
    }
    if (failures == 0) std::printf("ref tool ok\n");
    return failures == 0 ? 0 : 1;
}
