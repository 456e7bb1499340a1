// C++ caller of the B200 path through include/tgcu.hpp, written the way a
// reference tool would use it (cmd_bench-shaped loop, tools/main.cpp:639-644).
// Built by __graft_entry__.build(); run by tests/test_cpp_shim.py on a GPU.
#include <cmath>
#include <cstdio>
#include <vector>

#include "tgcu.hpp"

int main() {
    tgcu_grid_spec gs{3, {24, 24, 24}, {-1, -1, -1}, {2, 2, 2}, 2};
    tgcu::Grid g(gs);
    g.adam_reset({1e-2, 0.9, 0.999, 1e-8});
    const int n = 8192;
    std::vector<float> smp(4 * n);
    if (tgcu_sample(0, 3, 7, n, 0.5, 0.01, 0.6, smp.data()) != TGCU_OK) return 2;
    tgcu::LossConfig lc;
    double first = 0, last = 0;
    for (int s = 0; s < 20; ++s) {
        const auto t = g.train_step(smp, lc);
        if (s == 0) first = t.total;
        last = t.total;
    }
    // pipelined host steps continue the same trajectory
    for (int s = 0; s < 10; ++s) g.train_step_async(smp, lc);
    const auto ta = g.sync();
    if (!(ta.total < first) || !std::isfinite(ta.total)) return 9;
    last = ta.total;
    std::vector<float> pts = {0.f, 0.f, 0.f, 0.6f, 0.f, 0.f};
    std::vector<float> grad;
    const auto v = g.eval(pts, &grad);
    std::printf("loss %.6g -> %.6g, f(0)=%.4f f(0.6,0,0)=%.4f\n", first, last, v[0], v[1]);
    if (!(last < first) || !std::isfinite(v[0])) return 3;
    smp[4 * 5 + 3] = NAN;  // non-finite loss -> tg::NumericalError semantics
    try {
        g.train_step(smp, lc);
        return 4;
    } catch (const tgcu::NumericalError& e) {
        std::printf("NumericalError: %s\n", e.what());
    }
    try {
        tgcu::coeff_count(3, 3);
        return 5;
    } catch (const std::invalid_argument&) {
    }
    // progressive stage change, lattice extraction, .tgrid round trip
    tgcu::Grid up = tgcu::upsample(g, {48, 48, 48});
    const auto lat = up.sample_grid_field({9, 9, 9});
    if (lat.size() != 729 || !std::isfinite(lat[364])) return 6;
    up.save_tgrid("/tmp/tgcu_shim_test.tgrid");
    tgcu::Grid back = tgcu::load_tgrid("/tmp/tgcu_shim_test.tgrid");
    if (back.coeffs() != up.coeffs()) return 7;
    try {
        tgcu::load_tgrid("/tmp/does_not_exist.tgrid");
        return 8;
    } catch (const tgcu::IngestError& e) {
        std::printf("IngestError: %s\n", e.what());
    }
    std::printf("upsample + lattice + tgrid ok (f(centre) %.4f)\n", lat[364]);
    // both fused-step paths through the C ABI (this grid takes the small-grid
    // path by default): the same loss terms on the same samples
    {
        smp[4 * 5 + 3] = 0.1f;
        tgcu::Grid a(gs), b(gs);
        a.adam_reset({1e-2, 0.9, 0.999, 1e-8});
        b.adam_reset({1e-2, 0.9, 0.999, 1e-8});
        if (tgcu_grid_set_step_path(b.handle(), TGCU_STEP_BRICK) != TGCU_OK) return 10;
        if (tgcu_grid_set_step_path(b.handle(), 7) != TGCU_ERR_INVALID_ARGUMENT) return 11;
        const auto ta2 = a.train_step(smp, lc);
        const auto tb2 = b.train_step(smp, lc);
        if (!(std::fabs(ta2.total - tb2.total) <= 1e-6 * std::fabs(tb2.total))) return 12;
        std::printf("step paths: small %.9g brick %.9g\n", ta2.total, tb2.total);
    }
    std::printf("shim ok\n");
    return 0;
}
