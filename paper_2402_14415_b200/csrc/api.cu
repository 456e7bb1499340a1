// C-ABI entry points of libtgcu (include/tgcu.h): handle lifetime, host/device
// staging, error mapping, and the stream-ordered drivers of the kernels.
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "tg_internal.h"

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};

}  // namespace

namespace tgcu {

int set_err(int code, const std::string& m) {
    g_err = m;
    return code;
}

void count_launch(int n) { g_launches += n; }

static void set_device(const Grid& g) { TGCU_CUDA(cudaSetDevice(g.device)); }

void prof_mark(Grid& g, cudaStream_t s, int which) {
    if (which == 0 && g.prof_used + 2 > g.prof_ev.size()) {
        for (int i = 0; i < 256; ++i) {
            cudaEvent_t e;
            TGCU_CUDA(cudaEventCreate(&e));
            g.prof_ev.push_back(e);
        }
    }
    TGCU_CUDA(cudaEventRecord(g.prof_ev[g.prof_used++], s));
}

void bd_mark(Grid& g, cudaStream_t s, int i) {
    if (!g.bd_ev[i]) TGCU_CUDA(cudaEventCreate(&g.bd_ev[i]));
    TGCU_CUDA(cudaEventRecord(g.bd_ev[i], s));
}

void bd_collect(Grid& g) {
    TGCU_CUDA(cudaEventSynchronize(g.bd_ev[5]));
    for (int i = 0; i < 5; ++i) {
        float ms = 0.f;
        TGCU_CUDA(cudaEventElapsedTime(&ms, g.bd_ev[i], g.bd_ev[i + 1]));
        g.bd_sum[i] += ms;
    }
    ++g.bd_steps;
}

void ensure_staging(Grid& g, int64_t floats) {
    if (g.staging_cap >= floats) return;
    if (g.staging) TGCU_CUDA(cudaFree(g.staging));
    g.staging = nullptr;
    TGCU_CUDA(cudaMalloc(&g.staging, sizeof(float) * floats));
    g.staging_cap = floats;
}

void ensure_pipeline(Grid& g, int64_t floats) {
    if (!g.cstream) {
        TGCU_CUDA(cudaStreamCreateWithFlags(&g.cstream, cudaStreamNonBlocking));
        TGCU_CUDA(cudaStreamCreateWithFlags(&g.cstream2, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            TGCU_CUDA(cudaEventCreateWithFlags(&g.ev_ready[i], cudaEventDisableTiming));
            TGCU_CUDA(cudaEventCreateWithFlags(&g.ev_free[i], cudaEventDisableTiming));
            TGCU_CUDA(cudaEventCreateWithFlags(&g.ev_half[i], cudaEventDisableTiming));
        }
        TGCU_CUDA(cudaMallocHost(&g.h_ring, sizeof(tgcu_loss_terms) * kTraceCap));
    }
    if (g.pstage_cap >= floats) return;
    TGCU_CUDA(cudaDeviceSynchronize());  // slots may be in flight
    for (int i = 0; i < 2; ++i) {
        if (g.pstage[i]) TGCU_CUDA(cudaFree(g.pstage[i]));
        g.pstage[i] = nullptr;
        TGCU_CUDA(cudaMalloc(&g.pstage[i], sizeof(float) * floats));
    }
    g.pstage_cap = floats;
}

void ensure_scratch(Grid& g, int64_t doubles) {
    if (g.scratch_cap >= doubles) return;
    if (g.scratch_d) TGCU_CUDA(cudaFree(g.scratch_d));
    g.scratch_d = nullptr;
    TGCU_CUDA(cudaMalloc(&g.scratch_d, sizeof(double) * doubles));
    g.scratch_cap = doubles;
}

void ensure_bins(Grid& g, int set, int64_t points) {
    const int64_t need = points << g.spec.dim;  // worst case 2^D copies per point
    if (g.binned_cap[set] >= need) return;
    if (g.binned[set]) TGCU_CUDA(cudaFree(g.binned[set]));  // (cudaFree waits for the device)
    g.binned[set] = nullptr;
    TGCU_CUDA(cudaMalloc(&g.binned[set], sizeof(float4) * need));
    g.binned_cap[set] = need;
}

void ensure_bin_stream(Grid& g) {
    if (g.bstream) return;
    {
        // Highest priority: with the brick launch order (surface bricks
        // first, train.cu place_brick) the binning CTAs of the next step take
        // the SM slots freed in the brick kernel's tail ahead of its remaining
        // short CTAs, so the next brick kernel is not kept waiting (A/B: C2
        // step 0.295 -> 0.278 ms).
        int lo = 0, hi = 0;
        TGCU_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        TGCU_CUDA(cudaStreamCreateWithPriority(&g.bstream, cudaStreamNonBlocking, hi));
    }
    TGCU_CUDA(cudaEventCreateWithFlags(&g.ev_in, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
        TGCU_CUDA(cudaEventCreateWithFlags(&g.ev_bdone[i], cudaEventDisableTiming));
        TGCU_CUDA(cudaEventCreateWithFlags(&g.ev_bfree[i], cudaEventDisableTiming));
    }
}

void ensure_bin_hist(Grid& g, int64_t ints, int64_t points, int64_t chain_ctas) {
    if (g.bin_hist_cap < ints) {
        if (g.bin_hist) TGCU_CUDA(cudaFree(g.bin_hist));
        g.bin_hist = nullptr;
        TGCU_CUDA(cudaMalloc(&g.bin_hist, sizeof(int) * ints));
        g.bin_hist_cap = ints;
    }
    if (g.bin_codes_cap < points) {
        if (g.bin_codes) TGCU_CUDA(cudaFree(g.bin_codes));
        g.bin_codes = nullptr;
        TGCU_CUDA(cudaMalloc(&g.bin_codes, sizeof(int) * points));
        g.bin_codes_cap = points;
    }
    if (g.bin_chain_cap < chain_ctas) {
        if (g.bin_chain) TGCU_CUDA(cudaFree(g.bin_chain));
        g.bin_chain = nullptr;
        // 2 ints per CTA + the 64-bit ticket counter of k_bin_cols
        TGCU_CUDA(cudaMalloc(&g.bin_chain, sizeof(int) * (2 * chain_ctas + 2)));
        TGCU_CUDA(cudaMemset(g.bin_chain, 0, sizeof(int) * (2 * chain_ctas + 2)));
        g.bin_chain_cap = chain_ctas;
        g.bin_epoch = 0;
    }
}

// Ping-pong parameters + Adam moments (both slots), zero moments.
void ensure_optimizer(Grid& g) {
    if (g.m[0]) return;
    if (!g.p[1]) TGCU_CUDA(cudaMalloc(&g.p[1], sizeof(float) * g.NC));
    for (int i = 0; i < 2; ++i) {
        TGCU_CUDA(cudaMalloc(&g.m[i], sizeof(float) * g.NC));
        TGCU_CUDA(cudaMalloc(&g.v[i], sizeof(float) * g.NC));
        TGCU_CUDA(cudaMemset(g.m[i], 0, sizeof(float) * g.NC));
        TGCU_CUDA(cudaMemset(g.v[i], 0, sizeof(float) * g.NC));
    }
}

void ensure_grad(Grid& g) {
    if (g.grad) return;
    TGCU_CUDA(cudaMalloc(&g.grad, sizeof(float) * g.NC));
    TGCU_CUDA(cudaMemset(g.grad, 0, sizeof(float) * g.NC));
}

DevSpec make_devspec(const tgcu_grid_spec& s) {
    DevSpec d{};
    for (int a = 0; a < 3; ++a) {
        const bool act = a < s.dim;
        d.res[a] = act ? s.res[a] : 1;
        d.origin[a] = act ? s.origin[a] : 0.0;
        d.hi[a] = act ? s.origin[a] + s.extent[a] : 0.0;
        d.h[a] = act ? s.extent[a] / (s.res[a] - 1) : 1.0;
        d.inv_h[a] = act ? 1.0 / d.h[a] : 0.0;
        d.hf[a] = (float)d.h[a];
        d.inv_hf[a] = (float)d.inv_h[a];
    }
    d.sy = s.res[0];
    d.sz = (long long)s.res[0] * (s.dim == 3 ? s.res[1] : 1);
    d.zoff = 0;
    d.zstore = s.dim == 3 ? s.res[2] : 1;
    return d;
}

void validate_spec(const tgcu_grid_spec& s) {
    // GridSpec::validate (grid_spec.cpp:21-33) + coeff_count ranges.
    require(s.dim == 2 || s.dim == 3, "coeff_count: dim must be 2 or 3, got " + std::to_string(s.dim));
    require(s.order >= 0 && s.order <= 2, "coeff_count: order must be in {0,1,2}, got " + std::to_string(s.order));
    for (int a = 0; a < s.dim; ++a) {
        require(s.res[a] >= 2, "GridSpec: resolution must be >= 2 per axis, got " + std::to_string(s.res[a]) +
                                   " on axis " + std::to_string(a));
        require(s.extent[a] > 0.0 && std::isfinite(s.extent[a]),
                "GridSpec: extent must be positive and finite on axis " + std::to_string(a));
        require(std::isfinite(s.origin[a]), "GridSpec: origin must be finite");
        const double h = s.extent[a] / (s.res[a] - 1);
        require(std::isfinite(h) && h > 0.0, "GridSpec: cell spacing must be positive");
    }
}

int coeff_count_of(int order, int dim) {
    return order == 0 ? 1 : (order == 1 ? 1 + dim : 1 + dim + dim * (dim + 1) / 2);
}

// Seeded host generator with the reference Rng semantics (rng.hpp:14-51).
struct HostRng {
    uint64_t mt[312];
    int idx = 312;
    explicit HostRng(uint64_t seed) {
        mt[0] = seed;
        for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
    }
    uint64_t next() {
        if (idx >= 312) {
            for (int i = 0; i < 312; ++i) {
                const uint64_t x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % 312] & 0x7FFFFFFFULL);
                uint64_t xa = x >> 1;
                if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
                mt[i] = mt[(i + 156) % 312] ^ xa;
            }
            idx = 0;
        }
        uint64_t x = mt[idx++];
        x ^= (x >> 29) & 0x5555555555555555ULL;
        x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
        x ^= (x << 37) & 0xFFF7EEE000000000ULL;
        x ^= x >> 43;
        return x;
    }
    double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
};

}  // namespace tgcu

using namespace tgcu;

extern "C" {

const char* tgcu_last_error(void) { return g_err.c_str(); }
const char* tgcu_version(void) { return "tgcu 0.1 (sm_100a)"; }
int64_t tgcu_launch_count(void) { return g_launches.load(); }
void tgcu_reset_launch_count(void) { g_launches = 0; }

int tgcu_coeff_count(int order, int dim, int* out) {
    return guard([&] {
        require(dim == 2 || dim == 3, "coeff_count: dim must be 2 or 3, got " + std::to_string(dim));
        require(order >= 0 && order <= 2, "coeff_count: order must be in {0,1,2}, got " + std::to_string(order));
        *out = coeff_count_of(order, dim);
    });
}

// init_grid for a full grid (zb_lo = zb_hi = -1) or for the z-slab of brick
// layers [zb_lo, zb_hi) of the global spec (multi-GPU owner-computes
// training): the slab stores vertex planes [8*zb_lo - 1, 8*zb_hi] clipped to
// the grid (its owned planes plus one halo plane on each side).
static int create_grid(const tgcu_grid_spec* spec, const tgcu_init_options* opts_in, int device, int zb_lo,
                       int zb_hi, tgcu_grid** out) {
    *out = nullptr;
    tgcu_grid* h = nullptr;
    const int rc = guard([&] {
        require(spec != nullptr, "tgcu_grid_create: spec is NULL");
        tgcu_grid_spec s = *spec;
        if (s.dim == 2) s.res[2] = 1;
        validate_spec(s);
        tgcu_init_options opts{TGCU_INIT_ZEROS, 0.0, 1e-4, 0, 4ull << 30};
        if (opts_in) opts = *opts_in;
        const int K = coeff_count_of(s.order, s.dim);
        int64_t Vg = 1;
        for (int a = 0; a < s.dim; ++a) Vg *= s.res[a];
        const int B = s.dim == 3 ? kBrick3 : kBrick2;
        const int BZ = s.dim == 3 ? kBrickZ3 : 1;  // z extent of a brick (slab layer depth)
        const bool slab = zb_lo >= 0;
        const int nbz_global = s.dim == 3 ? (s.res[2] + BZ - 1) / BZ : 1;
        int zoff = 0, zstore = s.dim == 3 ? s.res[2] : 1;
        if (slab) {
            require(s.dim == 3, "slab grids need dim 3");
            require(zb_lo < zb_hi && zb_hi <= nbz_global, "slab brick layers out of range");
            zoff = std::max(0, BZ * zb_lo - 1);
            const int zend = std::min(s.res[2], BZ * zb_hi + 1);
            zstore = zend - zoff;
        }
        const int64_t V = (int64_t)s.res[0] * (s.dim == 3 ? (int64_t)s.res[1] * zstore : s.res[1]);
        const uint64_t bytes = (uint64_t)(V * K) * sizeof(double);
        if (bytes > opts.memory_cap_bytes)
            throw Error(TGCU_ERR_RESOURCE, "init_grid: " + std::to_string(bytes) + " bytes exceeds memory cap of " +
                                               std::to_string(opts.memory_cap_bytes));
        // Brick codes of the point binning (train.cu point_brick_code) pack the
        // x, y, z brick coordinates into 27 bits, each axis as wide as the
        // grid needs.
        int code_sh[2];
        {
            auto bits = [](int n) { return n <= 1 ? 0 : 32 - __builtin_clz((unsigned)(n - 1)); };
            const int bx = bits((s.res[0] + B - 1) / B), by = bits((s.res[1] + B - 1) / B), bz = bits(nbz_global);
            if (bx + by + bz > 27)
                throw Error(TGCU_ERR_RESOURCE, "init_grid: " + std::to_string(bx + by + bz) +
                                                   " bits of brick coordinates exceed the 27-bit brick code");
            code_sh[0] = bx;
            code_sh[1] = bx + by;
        }
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw Error(TGCU_ERR_CUDA, "tgcu: no CUDA device available (the product path has no CPU fallback)");
        require(device >= 0 && device < ndev, "tgcu_grid_create: bad device " + std::to_string(device));
        // Stream-ordered scratch (query binning, sorts, resample tables) comes
        // from the device's default memory pool; keep freed blocks cached there
        // instead of returning them to the OS at every synchronisation.
        {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
                uint64_t keep = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
        }
        h = new tgcu_grid();
        Grid& g = h->g;
        g.spec = s;
        g.K = K;
        g.V = V;
        g.NC = V * K;
        g.device = device;
        g.slab = slab;
        TGCU_CUDA(cudaSetDevice(device));
        DevSpec& d = g.ds;
        d = make_devspec(s);
        d.zoff = zoff;
        d.zstore = zstore;
        // TV normaliser P*K of the global grid (sdf_loss.cpp:161-170).
        double P = 0.0;
        for (int a = 0; a < s.dim; ++a) {
            double np = s.res[a] - 1;
            for (int b2 = 0; b2 < s.dim; ++b2)
                if (b2 != a) np *= s.res[b2];
            P += np;
        }
        g.tv_inv_norm = 1.0 / (P * K);
        // Parameters now; the ping-pong copy and the Adam moments on first
        // optimiser use (ensure_optimizer), so query-only grids cost 4 B/coeff.
        TGCU_CUDA(cudaMalloc(&g.p[0], sizeof(float) * g.NC));
        TGCU_CUDA(cudaMalloc(&g.st, sizeof(Status)));
        TGCU_CUDA(cudaMallocHost(&g.st_host, sizeof(Status)));
        Status st0{};
        st0.nan_point = ULLONG_MAX;
        st0.bad_grad = ULLONG_MAX;
        st0.nan_bin[0] = st0.nan_bin[1] = ULLONG_MAX;
        st0.det_over[0] = st0.det_over[1] = ULLONG_MAX;
        TGCU_CUDA(cudaMemcpy(g.st, &st0, sizeof(Status), cudaMemcpyHostToDevice));
        // Brick decomposition (train.cu / query.cu).
        if (const char* det = std::getenv("TGCU_DETERMINISTIC")) g.deterministic = det[0] == '1';
        if (const char* pdl = std::getenv("TGCU_SMALL_PDL")) g.small_pdl = pdl[0] != '0';
        if (const char* pdl = std::getenv("TGCU_BRICK_PDL")) g.brick_pdl = pdl[0] != '0';
        if (const char* sp = std::getenv("TGCU_STEP_PATH"))
            g.step_path = std::string(sp) == "brick" ? 1 : (std::string(sp) == "single" ? 2 : 0);
        g.NB = 1;
        g.zb_global = nbz_global;
        g.code_sh[0] = code_sh[0];
        g.code_sh[1] = code_sh[1];
        for (int a = 0; a < 3; ++a) {
            const int ba = a == 2 ? BZ : B;
            g.brick[a] = a < s.dim ? ba : 1;
            g.nb[a] = a < s.dim ? (s.res[a] + ba - 1) / ba : 1;
        }
        if (slab) {
            g.zb0 = zb_lo;
            g.nb[2] = zb_hi - zb_lo;
        }
        for (int a = 0; a < 3; ++a) g.NB *= g.nb[a];
        TGCU_CUDA(cudaMalloc(&g.bin_count, sizeof(int) * (g.NB + 1)));
        for (int i = 0; i < 2; ++i) {
            TGCU_CUDA(cudaMalloc(&g.bin_off[i], sizeof(int) * (g.NB + 1)));
            // NB + 2 ints (order, class counters), then NB int4 (brick, first, end)
            TGCU_CUDA(cudaMalloc(&g.brick_order[i], sizeof(int) * ((g.NB + 2 + 3) / 4 * 4) + sizeof(int) * 4 * g.NB));
        }
        TGCU_CUDA(cudaMalloc(&g.bin_cursor, sizeof(int) * (g.NB + 1)));
        TGCU_CUDA(cudaMalloc(&g.partials, sizeof(double) * 4 * g.NB));
        TGCU_CUDA(cudaMalloc(&g.d_trace, sizeof(tgcu_loss_terms) * kTraceCap));
        TGCU_CUDA(cudaMalloc(&g.slab_red, sizeof(double) * 8));
        TGCU_CUDA(cudaMallocHost(&g.h_terms, sizeof(tgcu_loss_terms)));
        // init_grid modes (taylor_grid.cpp:174-186).
        float* p = g.p[0];
        TGCU_CUDA(cudaMemset(p, 0, sizeof(float) * g.NC));
        const int64_t goff = (int64_t)zoff * d.sz * K;  // this slab's first coefficient in the global order
        if (opts.mode == TGCU_INIT_CONSTANT) {
            launch_fill_f0(g, p, (float)opts.constant, 0);
        } else if (opts.mode == TGCU_INIT_SMALL_UNIFORM) {
            std::vector<float> hbuf(g.NC);
            HostRng r(opts.seed);
            for (int64_t i = 0; i < goff; ++i) r.next();  // global stream, this slab's window
            for (int64_t i = 0; i < g.NC; ++i) hbuf[i] = (float)r.uniform(-opts.epsilon, opts.epsilon);
            TGCU_CUDA(cudaMemcpy(p, hbuf.data(), sizeof(float) * g.NC, cudaMemcpyHostToDevice));
        } else if (opts.mode == TGCU_INIT_HASH_GAUSSIAN) {
            launch_hash_gaussian(p, g.NC, opts.seed, opts.epsilon, goff, 0);
        }
        TGCU_CUDA(cudaDeviceSynchronize());
    });
    if (rc != TGCU_OK) {
        if (h) tgcu_grid_destroy(h);
        return rc;
    }
    *out = h;
    return TGCU_OK;
}

int tgcu_grid_create(const tgcu_grid_spec* spec, const tgcu_init_options* opts_in, int device, tgcu_grid** out) {
    return create_grid(spec, opts_in, device, -1, -1, out);
}

int tgcu_grid_create_slab(const tgcu_grid_spec* spec, int zb_lo, int zb_hi, const tgcu_init_options* opts,
                          int device, tgcu_grid** out) {
    if (zb_lo < 0) {
        *out = nullptr;
        return set_err(TGCU_ERR_INVALID_ARGUMENT, "tgcu_grid_create_slab: negative brick layer");
    }
    return create_grid(spec, opts, device, zb_lo, zb_hi, out);
}

int tgcu_slab_info(const tgcu_grid* h, int* z_store_lo, int* z_store_n, int* z_own_lo, int* z_own_hi,
                   int* brick_layers) {
    const Grid& g = h->g;
    const int B = g.spec.dim == 3 ? kBrickZ3 : 1;  // (slab layers: z bricks)
    if (z_store_lo) *z_store_lo = g.ds.zoff;
    if (z_store_n) *z_store_n = g.ds.zstore;
    if (z_own_lo) *z_own_lo = g.slab ? B * g.zb0 : 0;
    if (z_own_hi) *z_own_hi = g.slab ? std::min(g.spec.res[2], B * (g.zb0 + g.nb[2])) : g.ds.zstore;
    if (brick_layers) *brick_layers = g.zb_global;
    return TGCU_OK;
}

int tgcu_grid_destroy(tgcu_grid* h) {
    if (!h) return TGCU_OK;
    Grid& g = h->g;
    cudaSetDevice(g.device);
    cudaDeviceSynchronize();
    for (int i = 0; i < 2; ++i) {
        cudaFree(g.p[i]);
        cudaFree(g.m[i]);
        cudaFree(g.v[i]);
    }
    cudaFree(g.grad);
    cudaFree(g.st);
    cudaFreeHost(g.st_host);
    cudaFree(g.bin_count);
    cudaFree(g.bin_cursor);
    for (int i = 0; i < 2; ++i) {
        cudaFree(g.bin_off[i]);
        cudaFree(g.brick_order[i]);
        cudaFree(g.binned[i]);
        if (g.ev_bdone[i]) cudaEventDestroy(g.ev_bdone[i]);
        if (g.ev_bfree[i]) cudaEventDestroy(g.ev_bfree[i]);
    }
    if (g.ev_in) cudaEventDestroy(g.ev_in);
    if (g.bstream) cudaStreamDestroy(g.bstream);
    cudaFree(g.bin_hist);
    cudaFree(g.bin_codes);
    cudaFree(g.bin_chain);
    cudaFree(g.partials);
    cudaFree(g.fin_l2);
    cudaFree(g.sacc);
    cudaFree(g.d_ctr);
    cudaFree(g.d_bc);
    cudaFree(g.spart);
    cudaFree(g.d_trace);
    cudaFree(g.slab_red);
    cudaFreeHost(g.h_terms);
    cudaFree(g.staging);
    cudaFree(g.scratch_d);
    for (int i = 0; i < 2; ++i) {
        cudaFree(g.pstage[i]);
        if (g.ev_ready[i]) cudaEventDestroy(g.ev_ready[i]);
        if (g.ev_free[i]) cudaEventDestroy(g.ev_free[i]);
        if (g.ev_half[i]) cudaEventDestroy(g.ev_half[i]);
    }
    if (g.cstream) cudaStreamDestroy(g.cstream);
    if (g.cstream2) cudaStreamDestroy(g.cstream2);
    cudaFreeHost(g.h_ring);
    for (void* b : g.ipc_open) cudaIpcCloseMemHandle(b);
    for (auto e : g.prof_ev) cudaEventDestroy(e);
    for (auto e : h->coll_ev) cudaEventDestroy(e);
    delete h;
    return TGCU_OK;
}

int tgcu_grid_spec_of(const tgcu_grid* h, tgcu_grid_spec* out) {
    *out = h->g.spec;
    return TGCU_OK;
}
int64_t tgcu_grid_coeff_total(const tgcu_grid* h) { return h->g.NC; }
float* tgcu_grid_coeffs(tgcu_grid* h) { return h->g.p[h->g.cur]; }
float* tgcu_grid_grad(tgcu_grid* h) {
    float* r = nullptr;
    guard([&] {
        set_device(h->g);
        ensure_grad(h->g);
        r = h->g.grad;
    });
    return r;
}

static void check_n(const Grid& g, int64_t n, const char* what) {
    require(n == g.NC, std::string(what) + ": coefficient array has " + std::to_string(n) +
                           " entries, expected " + std::to_string(g.NC));
}

// Sticky async error -> exception (with the committed state restored).
static void raise_sticky(Grid& g) {
    TGCU_CUDA(cudaMemcpy(g.st_host, g.st, sizeof(Status), cudaMemcpyDeviceToHost));
    const Status& s = *g.st_host;
    if (!s.error) return;
    g.cur = s.good_idx;
    g.t = s.good_t;
    std::string msg;
    if (s.error_kind == 1)
        msg = "locate: NaN coordinate (sample " + std::to_string(s.error_index) + ") at stage 0 step " +
              std::to_string(s.error_step);
    else if (s.error_kind == 2)
        msg = "run_schedule: non-finite loss at stage 0 step " + std::to_string(s.error_step);
    else if (s.error_kind == 4)
        msg = "deterministic mode: brick " + std::to_string(s.error_index) +
              " holds more than 4096 point copies (the canonical-order sort's capacity)";
    else
        msg = "adam_step: non-finite gradient at parameter index " + std::to_string(s.error_index) +
              " (stage 0 step " + std::to_string(s.error_step) + ")";
    // Clear so the grid is usable again (the reference object survives a throw).
    Status clean = s;
    clean.error = 0;
    clean.error_kind = 0;
    clean.nan_point = ULLONG_MAX;
    clean.bad_grad = ULLONG_MAX;
    clean.nan_bin[0] = clean.nan_bin[1] = ULLONG_MAX;
    clean.det_over[0] = clean.det_over[1] = ULLONG_MAX;
    TGCU_CUDA(cudaMemcpy(g.st, &clean, sizeof(Status), cudaMemcpyHostToDevice));
    g.steps_launched = 0;
    throw Error(s.error, msg);
}

// Per-call NaN point report for the stateless query/backprop calls.
static void check_nan_points(Grid& g, cudaStream_t s) {
    TGCU_CUDA(cudaMemcpyAsync(g.st_host, g.st, sizeof(Status), cudaMemcpyDeviceToHost, s));
    TGCU_CUDA(cudaStreamSynchronize(s));
    if (g.st_host->nan_point != ULLONG_MAX) {
        const unsigned long long idx = g.st_host->nan_point;
        const unsigned long long none = ULLONG_MAX;
        TGCU_CUDA(cudaMemcpy(&g.st->nan_point, &none, sizeof(none), cudaMemcpyHostToDevice));
        throw Error(TGCU_ERR_INVALID_ARGUMENT, "locate: NaN coordinate (point " + std::to_string(idx) + ")");
    }
}

int tgcu_grid_upload_f64(tgcu_grid* h, const double* coeffs, int64_t n) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        check_n(g, n, "upload");
        std::vector<float> tmp(n);
        for (int64_t i = 0; i < n; ++i) tmp[i] = (float)coeffs[i];
        TGCU_CUDA(cudaMemcpy(g.p[g.cur], tmp.data(), sizeof(float) * n, cudaMemcpyHostToDevice));
    });
}

int tgcu_grid_download_f64(tgcu_grid* h, double* coeffs, int64_t n) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        check_n(g, n, "download");
        raise_sticky(g);
        std::vector<float> tmp(n);
        TGCU_CUDA(cudaMemcpy(tmp.data(), g.p[g.cur], sizeof(float) * n, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < n; ++i) coeffs[i] = tmp[i];
    });
}

int tgcu_grid_upload_f32(tgcu_grid* h, const float* coeffs, int64_t n, int flags) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        check_n(g, n, "upload");
        TGCU_CUDA(cudaMemcpy(g.p[g.cur], coeffs, sizeof(float) * n,
                             (flags & TGCU_HOST) ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice));
    });
}

int tgcu_grid_download_f32(tgcu_grid* h, float* coeffs, int64_t n, int flags) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        check_n(g, n, "download");
        raise_sticky(g);
        TGCU_CUDA(cudaMemcpy(coeffs, g.p[g.cur], sizeof(float) * n,
                             (flags & TGCU_HOST) ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice));
    });
}

int tgcu_grid_all_finite(tgcu_grid* h, int* out) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        unsigned long long* flag = nullptr;
        TGCU_CUDA(cudaMalloc(&flag, sizeof(unsigned long long)));
        const unsigned long long none = ULLONG_MAX;
        TGCU_CUDA(cudaMemcpy(flag, &none, sizeof(none), cudaMemcpyHostToDevice));
        launch_all_finite(g.p[g.cur], g.NC, flag, 0);
        unsigned long long r = 0;
        TGCU_CUDA(cudaMemcpy(&r, flag, sizeof(r), cudaMemcpyDeviceToHost));
        cudaFree(flag);
        *out = r == ULLONG_MAX ? 1 : 0;
    });
}

// TGCU_QUERY_DIRECT=1: unsorted batches of any size take k_eval_direct
// (diagnostic: grouping experiments, A/B against the binned path).
static bool query_force_direct() {
    static const bool on = [] {
        const char* e = std::getenv("TGCU_QUERY_DIRECT");
        return e && std::atoi(e) != 0;
    }();
    return on;
}

int tgcu_eval(tgcu_grid* h, const float* pts, int64_t n, float* values, float* spatial_grad, int flags,
              void* stream) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        require(n >= 0, "eval: negative point count");
        if (n == 0) return;
        cudaStream_t s = as_stream(stream);
        const float* dp = pts;
        float* dv = values;
        float* dg = spatial_grad;
        if (flags & TGCU_HOST) {
            const int64_t need = n * 3 + n + (spatial_grad ? 3 * n : 0);
            ensure_staging(g, need);
            float* sp = g.staging;
            dv = sp + 3 * n;
            dg = spatial_grad ? dv + n : nullptr;
            TGCU_CUDA(cudaMemcpyAsync(sp, pts, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, s));
            dp = sp;
        }
        if (flags & TGCU_SORTED)
            launch_eval_sorted(g, dp, n, nullptr, dv, dg, s);
        else if (n >= kBinnedQueryMin && !g.slab && !query_force_direct())
            launch_eval_binned(g, dp, n, dv, dg, s);  // large unsorted batches: bin by brick, smem tiles
        else
            launch_eval_direct(g, dp, n, dv, dg, s);
        if (flags & TGCU_HOST) {
            TGCU_CUDA(cudaMemcpyAsync(values, dv, sizeof(float) * n, cudaMemcpyDeviceToHost, s));
            if (spatial_grad)
                TGCU_CUDA(cudaMemcpyAsync(spatial_grad, dg, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost, s));
        }
        if (!(flags & TGCU_ASYNC) || (flags & TGCU_HOST)) check_nan_points(g, s);
    });
}

int tgcu_sort_points(tgcu_grid* h, const float* pts, int64_t n, float* sorted_pts, int64_t* perm,
                     int64_t* brick_offsets, void* stream) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        launch_sort_points(g, pts, n, sorted_pts, perm, brick_offsets, as_stream(stream));
    });
}

int64_t tgcu_query_brick_codes(const tgcu_grid* h) { return query_brick_codes(h->g); }

int tgcu_eval_sorted(tgcu_grid* h, const float* pts, int64_t n, const int64_t* brick_offsets, float* values,
                     float* spatial_grad, int flags, void* stream) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        require(!(flags & TGCU_HOST), "eval_sorted: device pointers only");
        if (n <= 0) return;
        cudaStream_t s = as_stream(stream);
        launch_eval_sorted(g, pts, n, brick_offsets, values, spatial_grad, s);
        if (!(flags & TGCU_ASYNC)) check_nan_points(g, s);
    });
}

int tgcu_backprop(tgcu_grid* h, const float* pts, const float* upstream, const float* upstream_vec, int64_t n,
                  float* grad, int flags, void* stream) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        require(grad != nullptr, "backprop: gradient buffer is NULL");
        if (n <= 0) return;
        cudaStream_t s = as_stream(stream);
        const float *dp = pts, *du = upstream, *dv = upstream_vec;
        if (flags & TGCU_HOST) {
            ensure_staging(g, 7 * n);
            float* sp = g.staging;
            TGCU_CUDA(cudaMemcpyAsync(sp, pts, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, s));
            dp = sp;
            if (upstream) {
                TGCU_CUDA(cudaMemcpyAsync(sp + 3 * n, upstream, sizeof(float) * n, cudaMemcpyHostToDevice, s));
                du = sp + 3 * n;
            }
            if (upstream_vec) {
                TGCU_CUDA(cudaMemcpyAsync(sp + 4 * n, upstream_vec, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, s));
                dv = sp + 4 * n;
            }
        }
        launch_backprop(g, dp, du, dv, n, grad, s);
        if (!(flags & TGCU_ASYNC)) check_nan_points(g, s);
    });
}

int tgcu_grad_zero(tgcu_grid* h, float* grad, void* stream) {
    return guard([&] {
        set_device(h->g);
        if (!grad) {  // NULL: the grid's own buffer
            ensure_grad(h->g);
            grad = h->g.grad;
        }
        TGCU_CUDA(cudaMemsetAsync(grad, 0, sizeof(float) * h->g.NC, as_stream(stream)));
    });
}

int tgcu_grad_download_f64(tgcu_grid* h, const float* grad, double* out, int64_t n) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        check_n(g, n, "grad_download");
        if (!grad) {
            ensure_grad(g);
            grad = g.grad;
        }
        std::vector<float> tmp(n);
        TGCU_CUDA(cudaMemcpy(tmp.data(), grad, sizeof(float) * n, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < n; ++i) out[i] = tmp[i];
    });
}

static double pair_count_of(const tgcu_grid_spec& s) {
    double P = 0.0;
    for (int a = 0; a < s.dim; ++a) {
        double np = s.res[a] - 1;
        for (int b = 0; b < s.dim; ++b)
            if (b != a) np *= s.res[b];
        P += np;
    }
    return P;
}

int tgcu_tv_loss(tgcu_grid* h, float* grad, double scale, double* out, void* stream) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        cudaStream_t s = as_stream(stream);
        const double inv_norm = 1.0 / (pair_count_of(g.spec) * g.K);
        launch_tv(g, g.p[g.cur], grad, 2.0 * scale * inv_norm, 1, s);
        double sum = 0.0;
        TGCU_CUDA(cudaMemcpyAsync(&sum, g.scratch_d + 2, sizeof(double), cudaMemcpyDeviceToHost, s));
        TGCU_CUDA(cudaStreamSynchronize(s));
        *out = sum * inv_norm;
    });
}

int tgcu_total_loss(tgcu_grid* h, const float* samples, int64_t n, const tgcu_loss_config* cfg, float* grad,
                    tgcu_loss_terms* out, int flags, void* stream) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        require(cfg != nullptr, "total_loss: NULL config");
        // LossConfig::validate (sdf_loss.cpp:118-122) and the empty-batch check (:261).
        require(cfg->lambda1 >= 0.0 && cfg->lambda2 >= 0.0, "LossConfig: lambda weights must be >= 0");
        require(cfg->k > 0.0, "LossConfig: weight sharpness k must be > 0");
        require(n > 0, "total_loss: empty batch");
        cudaStream_t s = as_stream(stream);
        const float4* ds = reinterpret_cast<const float4*>(samples);
        if (flags & TGCU_HOST) {
            ensure_staging(g, 4 * n);
            TGCU_CUDA(cudaMemcpyAsync(g.staging, samples, sizeof(float) * 4 * n, cudaMemcpyHostToDevice, s));
            ds = reinterpret_cast<const float4*>(g.staging);
        }
        launch_point_terms(g, ds, n, *cfg, grad, s);
        double sums[4] = {0, 0, 0, 0};
        TGCU_CUDA(cudaMemcpyAsync(sums, g.scratch_d, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
        TGCU_CUDA(cudaStreamSynchronize(s));
        check_nan_points(g, s);
        tgcu_loss_terms t{};
        t.fit = sums[0] / (double)n;
        t.eik = cfg->lambda1 > 0.0 ? sums[1] / (double)n : 0.0;
        if (cfg->use_tv) {
            const double inv_norm = 1.0 / (pair_count_of(g.spec) * g.K);
            const bool with_grad = cfg->lambda2 > 0.0 && grad;
            launch_tv(g, g.p[g.cur], with_grad ? grad : nullptr, 2.0 * cfg->lambda2 * inv_norm, 1, s);
            double tvs = 0.0;
            TGCU_CUDA(cudaMemcpyAsync(&tvs, g.scratch_d + 2, sizeof(double), cudaMemcpyDeviceToHost, s));
            TGCU_CUDA(cudaStreamSynchronize(s));
            t.tv = tvs * inv_norm;
        }
        t.total = t.fit + cfg->lambda1 * t.eik + cfg->lambda2 * t.tv;
        if (out) *out = t;
    });
}

int tgcu_recon_loss(tgcu_grid* h, const float* samples, int64_t n, const tgcu_loss_config* cfg, double scale,
                    float* grad, double* out, int flags, void* stream) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        require(cfg != nullptr && out != nullptr, "recon_loss: NULL argument");
        require(cfg->lambda1 >= 0.0 && cfg->lambda2 >= 0.0, "LossConfig: lambda weights must be >= 0");
        require(cfg->k > 0.0, "LossConfig: weight sharpness k must be > 0");
        require(n > 0, "recon_loss: empty batch");
        cudaStream_t s = as_stream(stream);
        const float4* ds = reinterpret_cast<const float4*>(samples);
        if (flags & TGCU_HOST) {
            ensure_staging(g, 4 * n);
            TGCU_CUDA(cudaMemcpyAsync(g.staging, samples, sizeof(float) * 4 * n, cudaMemcpyHostToDevice, s));
            ds = reinterpret_cast<const float4*>(g.staging);
        }
        tgcu_loss_config c = *cfg;
        c.lambda1 = 0.0;  // point_terms<false> (sdf_loss.cpp:133)
        launch_point_terms(g, ds, n, c, grad, s, scale);
        double sums[2] = {0, 0};
        TGCU_CUDA(cudaMemcpyAsync(sums, g.scratch_d, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
        TGCU_CUDA(cudaStreamSynchronize(s));
        check_nan_points(g, s);
        *out = sums[0] / (double)n;
    });
}

int tgcu_eikonal_loss(tgcu_grid* h, const float* points, int64_t n, double scale, float* grad, double* out,
                      int flags, void* stream) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        require(out != nullptr, "eikonal_loss: NULL argument");
        require(n > 0, "eikonal_loss: empty point set");
        cudaStream_t s = as_stream(stream);
        ensure_staging(g, 4 * n);
        float4* st4 = reinterpret_cast<float4*>(g.staging);
        const float* p3 = points;
        float* tmp = nullptr;
        if (flags & TGCU_HOST) {
            TGCU_CUDA(cudaMallocAsync(&tmp, sizeof(float) * 3 * n, s));
            TGCU_CUDA(cudaMemcpyAsync(tmp, points, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, s));
            p3 = tmp;
        }
        launch_pack_eik(p3, n, st4, s);
        if (tmp) TGCU_CUDA(cudaFreeAsync(tmp, s));
        tgcu_loss_config c{};
        c.lambda1 = scale;
        c.k = 1.0;
        launch_point_terms(g, st4, n, c, grad, s, 1.0, true);
        double sums[2] = {0, 0};
        TGCU_CUDA(cudaMemcpyAsync(sums, g.scratch_d, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
        TGCU_CUDA(cudaStreamSynchronize(s));
        check_nan_points(g, s);
        *out = sums[1] / (double)n;
    });
}

int tgcu_adam_reset(tgcu_grid* h, const tgcu_adam_config* cfg) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        raise_sticky(g);
        if (cfg) g.adam = *cfg;
        g.t = 0;
        ensure_optimizer(g);
        TGCU_CUDA(cudaMemset(g.m[g.cur], 0, sizeof(float) * g.NC));
        TGCU_CUDA(cudaMemset(g.v[g.cur], 0, sizeof(float) * g.NC));
    });
}

int tgcu_grid_steps_launched(const tgcu_grid* h, int64_t* n) {
    *n = h->g.steps_launched;
    return TGCU_OK;
}

int tgcu_adam_get_t(const tgcu_grid* h, int64_t* t) {
    *t = h->g.t;
    return TGCU_OK;
}

int tgcu_adam_step(tgcu_grid* h, const float* grad, void* stream) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        cudaStream_t s = as_stream(stream);
        require(grad != nullptr, "adam_step: NULL gradient");
        ensure_optimizer(g);
        launch_adam_check(g, grad, s);
        TGCU_CUDA(cudaMemcpyAsync(g.st_host, g.st, sizeof(Status), cudaMemcpyDeviceToHost, s));
        TGCU_CUDA(cudaStreamSynchronize(s));
        if (g.st_host->bad_grad != ULLONG_MAX) {
            const unsigned long long idx = g.st_host->bad_grad;
            const unsigned long long none = ULLONG_MAX;
            TGCU_CUDA(cudaMemcpy(&g.st->bad_grad, &none, sizeof(none), cudaMemcpyHostToDevice));
            throw Error(TGCU_ERR_NUMERICAL, "adam_step: non-finite gradient at parameter index " + std::to_string(idx));
        }
        g.t += 1;
        const double bc1 = 1.0 - std::pow(g.adam.beta1, (double)g.t);
        const double bc2 = 1.0 - std::pow(g.adam.beta2, (double)g.t);
        launch_adam_update(g, grad, 1.0 / bc1, 1.0 / bc2, s);
        TGCU_CUDA(cudaStreamSynchronize(s));
    });
}

int tgcu_adam_download_f64(tgcu_grid* h, double* m, double* v, int64_t n) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        check_n(g, n, "adam_download");
        ensure_optimizer(g);
        raise_sticky(g);
        std::vector<float> tmp(n);
        TGCU_CUDA(cudaMemcpy(tmp.data(), g.m[g.cur], sizeof(float) * n, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < n; ++i) m[i] = tmp[i];
        TGCU_CUDA(cudaMemcpy(tmp.data(), g.v[g.cur], sizeof(float) * n, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < n; ++i) v[i] = tmp[i];
    });
}

int tgcu_train_step(tgcu_grid* h, const float* samples, int64_t n, const tgcu_loss_config* cfg,
                    tgcu_loss_terms* out, int flags, void* stream) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        require(cfg != nullptr, "total_loss: NULL config");
        require(cfg->lambda1 >= 0.0 && cfg->lambda2 >= 0.0, "LossConfig: lambda weights must be >= 0");
        require(cfg->k > 0.0, "LossConfig: weight sharpness k must be > 0");
        require(n > 0, "total_loss: empty batch");
        require(n <= (int64_t)INT_MAX / (1 << g.spec.dim), "train_step: batch too large");
        cudaStream_t s = as_stream(stream);
        const float4* ds = reinterpret_cast<const float4*>(samples);
        // Pipelined host input: the copy of this step's samples runs on the
        // copy stream into the free slot while earlier steps compute.
        const bool pipe = (flags & TGCU_HOST) && (flags & TGCU_ASYNC) && out == nullptr;
        BinInput bin_in;
        bin_in.ready = (flags & TGCU_INPUT_READY) != 0;
        if (pipe) {
            // The copy stream fills the slot, the binning stream reads it; the
            // caller's stream only sees binned points.
            ensure_pipeline(g, 4 * n);
            const int slot = g.pipe_slot;
            g.pipe_slot ^= 1;
            // the two halves on two copy streams, joined on the first
            const int64_t h1 = n / 2;
            TGCU_CUDA(cudaStreamWaitEvent(g.cstream, g.ev_free[slot], 0));
            TGCU_CUDA(cudaStreamWaitEvent(g.cstream2, g.ev_free[slot], 0));
            TGCU_CUDA(cudaMemcpyAsync(g.pstage[slot], samples, sizeof(float) * 4 * h1, cudaMemcpyHostToDevice,
                                      g.cstream));
            TGCU_CUDA(cudaMemcpyAsync(g.pstage[slot] + 4 * h1, samples + 4 * h1, sizeof(float) * 4 * (n - h1),
                                      cudaMemcpyHostToDevice, g.cstream2));
            TGCU_CUDA(cudaEventRecord(g.ev_half[slot], g.cstream2));
            TGCU_CUDA(cudaStreamWaitEvent(g.cstream, g.ev_half[slot], 0));
            TGCU_CUDA(cudaEventRecord(g.ev_ready[slot], g.cstream));
            // TGCU_HOST_RELEASE: hand the host buffer back once it is copied
            // (the step itself stays queued)
            if (flags & TGCU_HOST_RELEASE) TGCU_CUDA(cudaEventSynchronize(g.ev_ready[slot]));
            bin_in.wait = g.ev_ready[slot];
            bin_in.consumed = g.ev_free[slot];
            ds = reinterpret_cast<const float4*>(g.pstage[slot]);
        } else if (flags & TGCU_HOST) {
            ensure_staging(g, 4 * n);
            TGCU_CUDA(cudaMemcpyAsync(g.staging, samples, sizeof(float) * 4 * n, cudaMemcpyHostToDevice, s));
            ds = reinterpret_cast<const float4*>(g.staging);
            bin_in.ready = false;  // ordered after the copy on s
        }
        ensure_optimizer(g);
        const int64_t t_after = g.t + 1;
        const double bc1 = 1.0 - std::pow(g.adam.beta1, (double)t_after);
        const double bc2 = 1.0 - std::pow(g.adam.beta2, (double)t_after);
        const int in_idx = g.cur;
        float* gout = nullptr;
        if (flags & TGCU_EXPORT_GRAD) {
            ensure_grad(g);
            gout = g.grad;
        }
        require(!g.slab, "train_step: slab grids step with tgcu_slab_step_begin/finish");
        launch_train_step(g, ds, n, n, *cfg, in_idx, g.steps_launched, 1.0 / bc1, 1.0 / bc2, t_after, gout, nullptr,
                          bin_in, s);
        // Optimistic commit; a failed step is rolled back by raise_sticky().
        g.cur = 1 - in_idx;
        g.t = t_after;
        g.steps_launched += 1;
        if (pipe) {
            const int64_t r = (g.steps_launched - 1) % kTraceCap;  // this step's LossTerms -> pinned ring
            TGCU_CUDA(cudaMemcpyAsync(g.h_ring + r, g.d_trace + r, sizeof(tgcu_loss_terms), cudaMemcpyDeviceToHost, s));
        }
        const bool sync = !(flags & TGCU_ASYNC) || out != nullptr;
        if (out) {
            TGCU_CUDA(cudaMemcpyAsync(g.h_terms, g.d_trace + ((g.steps_launched - 1) % kTraceCap),
                                      sizeof(tgcu_loss_terms), cudaMemcpyDeviceToHost, s));
        }
        if (sync) {
            TGCU_CUDA(cudaStreamSynchronize(s));
            raise_sticky(g);
            if (out) *out = *g.h_terms;
        }
    });
}

int tgcu_train_step_fresh_eik(tgcu_grid* h, const float* samples, int64_t n, const float* eik_points,
                              const tgcu_loss_config* cfg, tgcu_loss_terms* out, int flags, void* stream) {
    if (cfg && cfg->lambda1 <= 0.0)  // no eikonal term: the reference draws no points
        return tgcu_train_step(h, samples, n, cfg, out, flags & ~TGCU_INPUT_READY, stream);
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        require(cfg != nullptr, "total_loss: NULL config");
        require(cfg->lambda1 >= 0.0 && cfg->lambda2 >= 0.0, "LossConfig: lambda weights must be >= 0");
        require(cfg->k > 0.0, "LossConfig: weight sharpness k must be > 0");
        require(n > 0, "total_loss: empty batch");
        require(eik_points != nullptr, "total_loss: fresh-uniform eikonal points need an rng");
        require(2 * n <= (int64_t)INT_MAX / (1 << g.spec.dim), "train_step: batch too large");
        require(!g.slab, "train_step: slab grids step with tgcu_slab_step_begin/finish");
        cudaStream_t s = as_stream(stream);
        // point list = the batch (recon only) followed by the eikonal points
        // (eikonal only, gt = kEikMark), staged on the caller's stream
        ensure_staging(g, 8 * n);
        float4* st4 = reinterpret_cast<float4*>(g.staging);
        const cudaMemcpyKind kind = (flags & TGCU_HOST) ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        TGCU_CUDA(cudaMemcpyAsync(st4, samples, sizeof(float) * 4 * n, kind, s));
        const float* e3 = eik_points;
        float* tmp = nullptr;
        if (flags & TGCU_HOST) {
            TGCU_CUDA(cudaMallocAsync(&tmp, sizeof(float) * 3 * n, s));
            TGCU_CUDA(cudaMemcpyAsync(tmp, eik_points, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, s));
            e3 = tmp;
        }
        launch_pack_eik(e3, n, st4 + n, s);
        if (tmp) TGCU_CUDA(cudaFreeAsync(tmp, s));
        ensure_optimizer(g);
        const int64_t t_after = g.t + 1;
        const double bc1 = 1.0 - std::pow(g.adam.beta1, (double)t_after);
        const double bc2 = 1.0 - std::pow(g.adam.beta2, (double)t_after);
        const int in_idx = g.cur;
        float* gout = nullptr;
        if (flags & TGCU_EXPORT_GRAD) {
            ensure_grad(g);
            gout = g.grad;
        }
        BinInput bin_in;  // ordered after the staging on s
        launch_train_step(g, st4, 2 * n, n, *cfg, in_idx, g.steps_launched, 1.0 / bc1, 1.0 / bc2, t_after, gout,
                          nullptr, bin_in, s, true);
        g.cur = 1 - in_idx;
        g.t = t_after;
        g.steps_launched += 1;
        const bool sync = !(flags & TGCU_ASYNC) || out != nullptr;
        if (out) {
            TGCU_CUDA(cudaMemcpyAsync(g.h_terms, g.d_trace + ((g.steps_launched - 1) % kTraceCap),
                                      sizeof(tgcu_loss_terms), cudaMemcpyDeviceToHost, s));
        }
        if (sync) {
            TGCU_CUDA(cudaStreamSynchronize(s));
            raise_sticky(g);
            if (out) *out = *g.h_terms;
        }
    });
}

int tgcu_slab_step_begin(tgcu_grid* h, const float* samples, int64_t n, int64_t n_global,
                         const tgcu_loss_config* cfg, double** partials, int flags, void* stream) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        require(g.slab, "slab_step_begin: not a slab grid");
        require(cfg != nullptr && partials != nullptr, "slab_step_begin: NULL argument");
        require(cfg->lambda1 >= 0.0 && cfg->lambda2 >= 0.0, "LossConfig: lambda weights must be >= 0");
        require(cfg->k > 0.0, "LossConfig: weight sharpness k must be > 0");
        // a rank may hold no points of a (non-empty) global batch: TV + Adam only
        require(n >= 0 && (n > 0 || n_global > 0), "total_loss: empty batch");
        cudaStream_t s = as_stream(stream);
        ensure_optimizer(g);
        const float4* ds = reinterpret_cast<const float4*>(samples);
        BinInput bin_in;
        bin_in.ready = (flags & TGCU_INPUT_READY) != 0;
        if (flags & TGCU_HOST) {
            ensure_staging(g, 4 * n);
            TGCU_CUDA(cudaMemcpyAsync(g.staging, samples, sizeof(float) * 4 * n, cudaMemcpyHostToDevice, s));
            ds = reinterpret_cast<const float4*>(g.staging);
            bin_in.ready = false;
        }
        const int64_t t_after = g.t + 1;
        const double bc1 = 1.0 - std::pow(g.adam.beta1, (double)t_after);
        const double bc2 = 1.0 - std::pow(g.adam.beta2, (double)t_after);
        float* gout = nullptr;
        if (flags & TGCU_EXPORT_GRAD) {
            ensure_grad(g);
            gout = g.grad;
        }
        g.slab_in_idx = g.cur;
        g.slab_step = g.steps_launched;
        g.slab_t_after = t_after;
        const int64_t nn = n_global > 0 ? n_global : n;
        require(nn >= n, "slab_step_begin: n_global smaller than the local batch");
        g.slab_n = nn;
        g.slab_cfg = *cfg;
        launch_train_step(g, ds, n, nn, *cfg, g.cur, g.steps_launched, 1.0 / bc1, 1.0 / bc2, t_after, gout,
                          g.slab_red, bin_in, s);
        *partials = g.slab_red;
    });
}

int tgcu_slab_step_finish(tgcu_grid* h, const double* reduced, tgcu_loss_terms* out, int flags, void* stream) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        require(g.slab, "slab_step_finish: not a slab grid");
        cudaStream_t s = as_stream(stream);
        launch_slab_finish(g, reduced ? reduced : g.slab_red, g.slab_cfg, g.slab_in_idx, g.slab_step,
                           g.slab_t_after, g.slab_n, s);
        g.cur = 1 - g.slab_in_idx;
        g.t = g.slab_t_after;
        g.steps_launched += 1;
        if (out) {
            TGCU_CUDA(cudaMemcpyAsync(g.h_terms, g.d_trace + ((g.steps_launched - 1) % kTraceCap),
                                      sizeof(tgcu_loss_terms), cudaMemcpyDeviceToHost, s));
        }
        if (!(flags & TGCU_ASYNC) || out) {
            TGCU_CUDA(cudaStreamSynchronize(s));
            raise_sticky(g);
            if (out) *out = *g.h_terms;
        }
    });
}

int tgcu_slab_halo(tgcu_grid* h, float** send_lo, float** send_hi, float** recv_lo, float** recv_hi,
                   int64_t* plane_floats) {
    return guard([&] {
        Grid& g = h->g;
        require(g.slab, "slab_halo: not a slab grid");
        const int B = kBrickZ3;
        const int own_lo = B * g.zb0;
        const int own_hi = std::min(g.spec.res[2], B * (g.zb0 + g.nb[2]));
        const int64_t pf = g.ds.sz * g.K;
        float* p = g.p[g.cur];
        auto plane = [&](int z) { return p + (int64_t)(z - g.ds.zoff) * pf; };
        const bool has_lo = own_lo > 0, has_hi = own_hi < g.spec.res[2];
        *send_lo = has_lo ? plane(own_lo) : nullptr;
        *recv_lo = has_lo ? plane(own_lo - 1) : nullptr;
        *send_hi = has_hi ? plane(own_hi - 1) : nullptr;
        *recv_hi = has_hi ? plane(own_hi) : nullptr;
        *plane_floats = pf;
    });
}

namespace {
// Owned-plane range and halo-plane byte offsets of a slab grid.
struct SlabPlanes {
    int own_lo, own_hi;
    bool has_lo, has_hi;
    int64_t pf;  // floats per plane
};
SlabPlanes slab_planes(const tgcu::Grid& g) {
    SlabPlanes p;
    p.own_lo = tgcu::kBrickZ3 * g.zb0;
    p.own_hi = std::min(g.spec.res[2], tgcu::kBrickZ3 * (g.zb0 + g.nb[2]));
    p.has_lo = p.own_lo > 0;
    p.has_hi = p.own_hi < g.spec.res[2];
    p.pf = g.ds.sz * g.K;
    return p;
}

__global__ void k_fill_value(float* __restrict__ p, int64_t n, float v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}
}  // namespace

int tgcu_slab_ipc_export(tgcu_grid* h, void* blob) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        require(g.slab, "slab_ipc_export: not a slab grid");
        require(blob != nullptr, "slab_ipc_export: NULL blob");
        ensure_optimizer(g);
        unsigned char* b = static_cast<unsigned char*>(blob);
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
        for (int i = 0; i < 2; ++i)
            TGCU_CUDA(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(b + 64 * i), g.p[i]));
        const SlabPlanes sp = slab_planes(g);
        const int64_t off_lo = sp.has_lo ? (int64_t)(sp.own_lo - 1 - g.ds.zoff) * sp.pf * 4 : -1;
        const int64_t off_hi = sp.has_hi ? (int64_t)(sp.own_hi - g.ds.zoff) * sp.pf * 4 : -1;
        std::memcpy(b + 128, &off_lo, 8);
        std::memcpy(b + 136, &off_hi, 8);
    });
}

int tgcu_slab_ipc_import(tgcu_grid* h, int side, const void* blob) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        require(g.slab, "slab_ipc_import: not a slab grid");
        require(blob != nullptr && (side == 0 || side == 1), "slab_ipc_import: bad argument");
        const SlabPlanes sp = slab_planes(g);
        require(side == 0 ? sp.has_lo : sp.has_hi, "slab_ipc_import: no neighbour on that side");
        const unsigned char* b = static_cast<const unsigned char*>(blob);
        int64_t off = -1;
        // my lowest owned plane is the lower neighbour's upper halo and vice versa
        std::memcpy(&off, b + (side == 0 ? 136 : 128), 8);
        require(off >= 0, "slab_ipc_import: the neighbour has no halo plane facing this slab");
        for (int i = 0; i < 2; ++i) {
            cudaIpcMemHandle_t hd;
            std::memcpy(&hd, b + 64 * i, sizeof(hd));
            void* base = nullptr;
            TGCU_CUDA(cudaIpcOpenMemHandle(&base, hd, cudaIpcMemLazyEnablePeerAccess));
            g.ipc_open.push_back(base);
            float* dst = reinterpret_cast<float*>(static_cast<char*>(base) + off);
            (side == 0 ? g.peer_lo : g.peer_hi)[i] = dst;
        }
    });
}

int tgcu_slab_set_peer_planes(tgcu_grid* h, float* const dst_lo[2], float* const dst_hi[2]) {
    return guard([&] {
        Grid& g = h->g;
        require(g.slab, "slab_set_peer_planes: not a slab grid");
        for (int i = 0; i < 2; ++i) {
            g.peer_lo[i] = dst_lo ? dst_lo[i] : nullptr;
            g.peer_hi[i] = dst_hi ? dst_hi[i] : nullptr;
        }
    });
}

int tgcu_slab_halo_slots(tgcu_grid* h, float* recv_lo[2], float* recv_hi[2]) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        require(g.slab && recv_lo && recv_hi, "slab_halo_slots: bad argument");
        ensure_optimizer(g);
        const SlabPlanes sp = slab_planes(g);
        for (int i = 0; i < 2; ++i) {
            recv_lo[i] = sp.has_lo ? g.p[i] + (int64_t)(sp.own_lo - 1 - g.ds.zoff) * sp.pf : nullptr;
            recv_hi[i] = sp.has_hi ? g.p[i] + (int64_t)(sp.own_hi - g.ds.zoff) * sp.pf : nullptr;
        }
    });
}

int tgcu_slab_peer_probe(tgcu_grid* h, int phase, int* ok) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        require(g.slab && ok != nullptr, "slab_peer_probe: bad argument");
        ensure_optimizer(g);
        const SlabPlanes sp = slab_planes(g);
        const int j = 1 - g.cur;  // the slot the next step writes
        *ok = 1;
        if (phase == 0) {
            // my lowest / highest owned plane index, as the neighbours will see it
            if (g.peer_lo[j]) k_fill_value<<<64, 256>>>(g.peer_lo[j], sp.pf, (float)sp.own_lo);
            if (g.peer_hi[j]) k_fill_value<<<64, 256>>>(g.peer_hi[j], sp.pf, (float)(sp.own_hi - 1));
            TGCU_CUDA(cudaGetLastError());
            TGCU_CUDA(cudaDeviceSynchronize());
            return;
        }
        std::vector<float> plane(sp.pf);
        auto check = [&](int z) {
            TGCU_CUDA(cudaMemcpy(plane.data(), g.p[j] + (int64_t)(z - g.ds.zoff) * sp.pf, sizeof(float) * sp.pf,
                                 cudaMemcpyDeviceToHost));
            for (float v : plane)
                if (v != (float)z) return false;
            return true;
        };
        if (sp.has_lo && !check(sp.own_lo - 1)) *ok = 0;
        if (sp.has_hi && !check(sp.own_hi)) *ok = 0;
    });
}

int tgcu_sync(tgcu_grid* h, tgcu_loss_terms* last) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        TGCU_CUDA(cudaDeviceSynchronize());
        raise_sticky(g);
        if (last && g.steps_launched > 0)
            TGCU_CUDA(cudaMemcpy(last, g.d_trace + ((g.steps_launched - 1) % kTraceCap), sizeof(tgcu_loss_terms),
                                 cudaMemcpyDeviceToHost));
    });
}

int tgcu_profile_begin(tgcu_grid* h) {
    return guard([&] {
        h->g.prof_on = true;
        h->g.prof_used = 0;
    });
}

int tgcu_step_breakdown(tgcu_grid* h, int enable, double* mean_ms5, int* steps) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        if (enable) {
            g.bd_on = true;
            for (double& x : g.bd_sum) x = 0.0;
            g.bd_steps = 0;
            return;
        }
        g.bd_on = false;
        for (int i = 0; i < 5; ++i) mean_ms5[i] = g.bd_steps ? g.bd_sum[i] / g.bd_steps : 0.0;
        if (steps) *steps = g.bd_steps;
    });
}

int tgcu_profile_every(tgcu_grid* h, int every) {
    return guard([&] {
        require(every >= 1, "profile_every: must be >= 1");
        h->g.prof_every = every;
    });
}

int tgcu_profile_end(tgcu_grid* h, double* total_ms, int* launches) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        g.prof_on = false;
        double tot = 0.0;
        for (size_t i = 0; i + 1 < g.prof_used; i += 2) {
            TGCU_CUDA(cudaEventSynchronize(g.prof_ev[i + 1]));
            float ms = 0.f;
            TGCU_CUDA(cudaEventElapsedTime(&ms, g.prof_ev[i], g.prof_ev[i + 1]));
            tot += ms;
        }
        *total_ms = tot;
        *launches = (int)(g.prof_used / 2);
        g.prof_used = 0;
    });
}

int tgcu_sample_uniform_device(int dim, uint64_t seed, int64_t n, double lo, double hi, float* out3,
                               void* stream) {
    return guard([&] {
        require(n >= 0 && out3 != nullptr && (dim == 2 || dim == 3), "sample_uniform_device: bad arguments");
        launch_hash_points(out3, n, dim, seed, lo, hi, as_stream(stream));
    });
}

int tgcu_trace(tgcu_grid* h, tgcu_loss_terms* out, int count) {
    return guard([&] {
        Grid& g = h->g;
        set_device(g);
        require(count >= 0 && count <= kTraceCap && count <= g.steps_launched, "trace: bad count");
        TGCU_CUDA(cudaDeviceSynchronize());
        std::vector<tgcu_loss_terms> all(kTraceCap);
        TGCU_CUDA(cudaMemcpy(all.data(), g.d_trace, sizeof(tgcu_loss_terms) * kTraceCap, cudaMemcpyDeviceToHost));
        for (int i = 0; i < count; ++i) out[i] = all[(g.steps_launched - count + i) % kTraceCap];
    });
}

}  // extern "C"

int tgcu_host_alloc(void** p, size_t bytes) {
    return guard([&] {
        require(p != nullptr, "host_alloc: NULL argument");
        *p = nullptr;
        TGCU_CUDA(cudaMallocHost(p, bytes == 0 ? 1 : bytes));
    });
}

int tgcu_host_free(void* p) {
    return guard([&] {
        if (p) TGCU_CUDA(cudaFreeHost(p));
    });
}

int tgcu_grid_set_step_path(tgcu_grid* h, int path) {
    return guard([&] {
        require(h != nullptr, "set_step_path: NULL grid");
        require(path >= TGCU_STEP_AUTO && path <= TGCU_STEP_SINGLE, "set_step_path: path must be 0 (auto), 1 (brick) or 2 (single)");
        h->g.step_path = path;
    });
}

int tgcu_grid_set_deterministic(tgcu_grid* h, int on) {
    return guard([&] {
        require(h != nullptr, "set_deterministic: NULL grid");
        h->g.deterministic = on != 0;
    });
}
