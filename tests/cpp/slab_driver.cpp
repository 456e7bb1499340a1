// TEST INFRASTRUCTURE: one rank of a slab-parallel training job driven from
// C++ through the C ABI alone (include/tgcu.h; no Python, no PyTorch):
// communicator (TCP star, host or NCCL collectives), slab grid, attach
// (initial halo, optional peer-memory halo), fused slab steps. Run as `world`
// processes by tests/test_slab_driver_gpu.py, which compares the gathered
// owned planes and every rank's loss terms with a single-grid run.
//
//   slab_driver <rank> <world> <port> <fused 0|1> <host|nccl> <outdir>
//
// Writes <outdir>/cpp_own<rank>.f64 (owned planes, reference AoS layout),
// cpp_terms<rank>.f64 (steps x 4) and cpp_fused<rank>.txt.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "tgcu.h"

namespace {

constexpr int kRes[3] = {32, 24, 40};
constexpr int kSteps = 5;
constexpr int kBrick = 8;
constexpr int64_t kBatch = 30000;

void check(int rc, const char* what) {
    if (rc != TGCU_OK) {
        std::fprintf(stderr, "%s failed (%d): %s\n", what, rc, tgcu_last_error());
        std::exit(1);
    }
}

// The reference's locate rule on z (grid_spec.cpp:45-69), fp64: slab.py point_cells_z.
int cell_z(const tgcu_grid_spec& s, double z) {
    const double lo = s.origin[2], hi = s.origin[2] + s.extent[2], h = s.extent[2] / (s.res[2] - 1);
    const double p = z < lo ? lo : (z > hi ? hi : z);
    int c = (int)std::floor((p - lo) / h);
    return c < 0 ? 0 : (c > s.res[2] - 2 ? s.res[2] - 2 : c);
}

bool write_file(const std::string& path, const void* data, size_t bytes) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) return false;
    const bool ok = std::fwrite(data, 1, bytes, f) == bytes;
    return std::fclose(f) == 0 && ok;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc != 7) {
        std::fprintf(stderr, "usage: %s rank world port fused host|nccl outdir\n", argv[0]);
        return 2;
    }
    const int rank = std::atoi(argv[1]), world = std::atoi(argv[2]), port = std::atoi(argv[3]);
    const int fused = std::atoi(argv[4]);
    const int backend = std::string(argv[5]) == "nccl" ? TGCU_COMM_NCCL : TGCU_COMM_HOST;
    const std::string out = argv[6];

    tgcu_grid_spec spec{};
    spec.dim = 3;
    for (int a = 0; a < 3; ++a) {
        spec.res[a] = kRes[a];
        spec.origin[a] = -1.0;
        spec.extent[a] = 2.0;
    }
    spec.order = 2;
    // brick layers split evenly, rank order (slab.py slab_ranges)
    const int nbz = (kRes[2] + kBrick - 1) / kBrick;
    const int base = nbz / world, rem = nbz % world;
    int zb_lo = 0;
    for (int r = 0; r < rank; ++r) zb_lo += base + (r < rem ? 1 : 0);
    const int zb_hi = zb_lo + base + (rank < rem ? 1 : 0);

    tgcu_comm* comm = nullptr;
    check(tgcu_comm_create("127.0.0.1", port, rank, world, 0, backend, &comm), "tgcu_comm_create");
    const tgcu_init_options init{TGCU_INIT_HASH_GAUSSIAN, 0.0, 0.02, 11, 1ull << 32};
    tgcu_grid* g = nullptr;
    check(tgcu_grid_create_slab(&spec, zb_lo, zb_hi, &init, 0, &g), "tgcu_grid_create_slab");
    const tgcu_adam_config adam{1e-2, 0.9, 0.999, 1e-8};
    check(tgcu_adam_reset(g, &adam), "tgcu_adam_reset");
    int fused_on = 0;
    check(tgcu_slab_connect(g, comm, fused, &fused_on), "tgcu_slab_connect");

    const tgcu_loss_config loss{1e-4, 2e-5, 50.0, 1, 1, 0};
    std::vector<double> terms;
    std::vector<float> batch(4 * kBatch), local;
    for (int i = 0; i < kSteps; ++i) {
        check(tgcu_sample(0, 3, 900 + i, kBatch, 0.5, 0.01, 0.6, batch.data()), "tgcu_sample");
        tgcu_loss_terms t{};
        if (i % 2) {  // only the points whose cells touch this slab's owned planes
            local.clear();
            for (int64_t j = 0; j < kBatch; ++j) {
                const int c = cell_z(spec, (double)batch[4 * j + 2]);
                if (c >= kBrick * zb_lo - 1 && c <= kBrick * zb_hi - 1)
                    local.insert(local.end(), batch.begin() + 4 * j, batch.begin() + 4 * j + 4);
            }
            check(tgcu_slab_train_step(g, local.data(), (int64_t)local.size() / 4, kBatch, &loss, &t, TGCU_HOST,
                                       nullptr),
                  "tgcu_slab_train_step (local points)");
        } else {
            check(tgcu_slab_train_step(g, batch.data(), kBatch, 0, &loss, &t, TGCU_HOST, nullptr),
                  "tgcu_slab_train_step");
        }
        terms.insert(terms.end(), {t.total, t.fit, t.eik, t.tv});
    }

    int zs_lo = 0, zs_n = 0, zo_lo = 0, zo_hi = 0, layers = 0;
    check(tgcu_slab_info(g, &zs_lo, &zs_n, &zo_lo, &zo_hi, &layers), "tgcu_slab_info");
    const int64_t plane = (int64_t)kRes[0] * kRes[1] * 10;
    std::vector<double> all((size_t)(plane * zs_n));
    check(tgcu_grid_download_f64(g, all.data(), (int64_t)all.size()), "tgcu_grid_download_f64");
    const double* own = all.data() + (zo_lo - zs_lo) * plane;
    const size_t own_n = (size_t)((zo_hi - zo_lo) * plane);
    const std::string r = std::to_string(rank);
    bool ok = write_file(out + "/cpp_own" + r + ".f64", own, own_n * sizeof(double)) &&
              write_file(out + "/cpp_terms" + r + ".f64", terms.data(), terms.size() * sizeof(double));
    const std::string f = std::to_string(fused_on);
    ok = ok && write_file(out + "/cpp_fused" + r + ".txt", f.data(), f.size());
    check(tgcu_grid_destroy(g), "tgcu_grid_destroy");
    check(tgcu_comm_destroy(comm), "tgcu_comm_destroy");
    if (!ok) {
        std::fprintf(stderr, "writing %s failed\n", out.c_str());
        return 1;
    }
    std::printf("slab driver rank %d/%d ok (planes %d-%d, fused %d)\n", rank, world, zo_lo, zo_hi, fused_on);
    return 0;
}
