// run_schedule on the device, behind the C ABI (schedule.hpp:13-86,
// schedule.cpp:13-108 of the reference): the progressive training loop a
// C / C++ host (the reference's cmd_bench / fit_sdf shape) drives without
// Python. Per stage: upsample when the resolution changes
// (taylor_grid.cpp:273-284), fresh Adam moments (schedule.cpp:79), the
// on_stage callback, then the steps as fused device steps (tgcu_train_step:
// zero grad -> total_loss -> finite-loss check -> adam_step). The problem is a
// batch callback (the reference's TrainProblem::compute minus the arithmetic,
// which the fused step does). Errors keep the reference's wording with the
// stage and the per-stage step ("run_schedule: non-finite loss at stage s
// step k", schedule.cpp:88-91).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "tg_internal.h"

using namespace tgcu;

namespace {

void validate_stages(const tgcu_stage* st, int n, int dim) {
    require(st != nullptr && n > 0, "Schedule: needs at least one stage");
    for (int s = 0; s < n; ++s) {
        require(st[s].steps >= 0, "Schedule: negative step count");
        for (int a = 0; a < dim; ++a) {
            require(st[s].res[a] >= 2, "Schedule: stage resolution must be >= 2");
            if (s > 0) require(st[s].res[a] >= st[s - 1].res[a], "Schedule: resolutions must be non-decreasing "
                                                                  "across stages");
        }
    }
}

// "stage 0 step <launch index>" (the library's step numbering) -> the
// schedule's stage and per-stage step.
std::string restage(const std::string& msg, int stage, int64_t offset) {
    const std::string key = "stage 0 step ";
    const size_t p = msg.find(key);
    if (p == std::string::npos) return msg;
    size_t e = p + key.size();
    while (e < msg.size() && msg[e] >= '0' && msg[e] <= '9') ++e;
    const int64_t launch = std::stoll(msg.substr(p + key.size(), e - p - key.size()));
    return msg.substr(0, p) + "stage " + std::to_string(stage) + " step " + std::to_string(launch - offset) +
           msg.substr(e);
}

struct Rethrow {
    int code;
    std::string msg;
};

}  // namespace

int tgcu_schedule_validate(const tgcu_stage* stages, int nstages, int dim) {
    return guard([&] { validate_stages(stages, nstages, dim); });
}

int tgcu_schedule_progressive(const int target[3], int dim, int total_steps, tgcu_stage out[3], int* nstages) {
    return guard([&] {
        require(target != nullptr && out != nullptr && nstages != nullptr, "Schedule: NULL argument");
        int n = 0;
        for (int d : {4, 2, 1}) {
            tgcu_stage st{{2, 2, 2}, total_steps / 3};
            bool same_as_target = true;
            for (int a = 0; a < dim; ++a) {
                st.res[a] = std::min(std::max(4, target[a] / d), target[a]);
                if (st.res[a] != target[a]) same_as_target = false;
            }
            if (n > 0) {
                bool same_as_prev = true;
                for (int a = 0; a < dim; ++a)
                    if (st.res[a] != out[n - 1].res[a]) same_as_prev = false;
                if (same_as_prev) continue;  // tiny targets collapse stages
            }
            out[n++] = st;
            if (same_as_target) break;
        }
        int assigned = 0;
        for (int s = 0; s < n; ++s) assigned += out[s].steps;
        out[n - 1].steps += total_steps - assigned;  // rounding remainder to the final stage
        *nstages = n;
    });
}

int tgcu_run_schedule(tgcu_grid** grid, const tgcu_stage* stages, int nstages, const tgcu_adam_config* adam,
                      const tgcu_loss_config* cfg, tgcu_batch_fn batch, tgcu_stage_fn on_stage, void* user, int flags,
                      void* stream, tgcu_trace_row* trace, double* stage_seconds) {
    return guard([&] {
        require(grid != nullptr && *grid != nullptr && adam != nullptr && cfg != nullptr && batch != nullptr,
                "run_schedule: NULL argument");
        tgcu_grid* h = *grid;
        require(!h->g.slab, "run_schedule: slab grids step with tgcu_slab_train_step");
        const int dim = h->g.spec.dim;
        validate_stages(stages, nstages, dim);
        using clock = std::chrono::steady_clock;
        const bool async = (flags & TGCU_ASYNC) != 0;
        int64_t gstep = 0;
        for (int si = 0; si < nstages; ++si) {
            const tgcu_stage& st = stages[si];
            bool resize = false;
            for (int a = 0; a < dim; ++a) resize |= st.res[a] != h->g.spec.res[a];
            if (resize) {
                tgcu_grid_spec ns = h->g.spec;
                for (int a = 0; a < dim; ++a) ns.res[a] = st.res[a];
                tgcu_init_options io{TGCU_INIT_ZEROS, 0.0, 1e-4, 0, ~0ull};
                tgcu_grid* nh = nullptr;
                int rc = tgcu_grid_create(&ns, &io, h->g.device, &nh);
                if (rc != TGCU_OK) throw Error(rc, tgcu_last_error());
                rc = tgcu_grid_upsample(h, nh, 0, stream);
                if (rc != TGCU_OK) {
                    const std::string m = tgcu_last_error();
                    tgcu_grid_destroy(nh);
                    throw Error(rc, m);
                }
                tgcu_grid_destroy(h);
                h = *grid = nh;
            }
            int rc = tgcu_adam_reset(h, adam);  // moments reset with each stage
            if (rc != TGCU_OK) throw Error(rc, tgcu_last_error());
            if (on_stage && (rc = on_stage(user, h, si)) != TGCU_OK) throw Error(rc, "run_schedule: on_stage_start failed");
            const auto t_stage = clock::now();
            int64_t k = 0;
            while (k < st.steps) {
                // async: windows of up to the trace capacity, one host sync each
                const int64_t w = async ? std::min<int64_t>(kTraceCap, st.steps - k) : 1;
                int64_t launched = 0;
                tgcu_grid_steps_launched(h, &launched);
                const int64_t offset = launched - k;  // launch index of per-stage step 0
                const auto t0 = clock::now();
                tgcu_loss_terms one{};
                for (int64_t j = 0; j < w; ++j) {
                    const float* smp = nullptr;
                    int64_t n = 0;
                    int bf = 0;
                    if ((rc = batch(user, h, gstep + k + j, &smp, &n, &bf)) != TGCU_OK)
                        throw Error(rc, "run_schedule: batch callback failed at stage " + std::to_string(si) +
                                            " step " + std::to_string(k + j));
                    int sf = bf & TGCU_HOST;
                    // host batches: the call returns once the samples are copied,
                    // so the callback may refill its buffer for the next step
                    if (async) sf |= TGCU_ASYNC | ((bf & TGCU_HOST) ? TGCU_HOST_RELEASE : (bf & TGCU_INPUT_READY));
                    rc = tgcu_train_step(h, smp, n, cfg, async ? nullptr : &one, sf, stream);
                    if (rc != TGCU_OK) throw Error(rc, restage(tgcu_last_error(), si, offset));
                }
                if (async) {
                    tgcu_loss_terms last{};
                    if ((rc = tgcu_sync(h, &last)) != TGCU_OK) throw Error(rc, restage(tgcu_last_error(), si, offset));
                }
                const double ms = std::chrono::duration<double, std::milli>(clock::now() - t0).count() / (double)w;
                std::vector<tgcu_loss_terms> rows((size_t)w);
                if (async) {
                    if ((rc = tgcu_trace(h, rows.data(), (int)w)) != TGCU_OK) throw Error(rc, tgcu_last_error());
                } else {
                    rows[0] = one;
                }
                for (int64_t j = 0; j < w; ++j) {
                    if (!std::isfinite(rows[j].total))  // (the fused step already refuses to commit these)
                        throw Error(TGCU_ERR_NUMERICAL, "run_schedule: non-finite loss at stage " +
                                                            std::to_string(si) + " step " + std::to_string(k + j));
                    if (trace) {
                        tgcu_trace_row& r = trace[gstep + k + j];
                        r.step = gstep + k + j;
                        r.stage = si;
                        for (int a = 0; a < 3; ++a) r.res[a] = st.res[a];
                        r.loss = rows[j];
                        r.wall_ms = ms;
                    }
                }
                k += w;
            }
            gstep += st.steps;
            if (stage_seconds) stage_seconds[si] = std::chrono::duration<double>(clock::now() - t_stage).count();
        }
    });
}
