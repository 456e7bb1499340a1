// Stage transitions and grid-wide consumers around the hot path:
//
//  * multilinear_resample / upsample (taylor_grid.cpp:231-284): the
//    progressive schedule's resolution change (schedule.cpp:74-80);
//  * sample_grid_field (marching.cpp:53-58): the query on an implicit,
//    perfectly coherent lattice (mesh extraction, IoU probes);
//  * .tgrid I/O (grid_io.cpp:36-111): on-disk interop with the reference CLI.
//
// Both kernels exploit that lattice coordinates are separable: the locate of
// lattice index i on axis a depends on (a, i) only, so one tiny kernel builds
// per-axis tables (cell, local / fp32 factors) once and the streaming kernel
// does no fp64 work per point beyond the resample weights.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <vector>

#include "dispatch.cuh"
#include "tg_internal.h"

namespace tgcu {

// One lattice coordinate located in a grid: cell and fp64 local.
struct AxisLoc {
    int cell;
    int pad;
    double local;
};

// Positions per axis: mode 0 = vertex positions of a spec with `n` vertices
// (origin + spacing * i, GridSpec::vertex_position, grid_spec.hpp:47-51, the
// spacing extent/(n-1) passed in `step`); mode 1 = ScalarField3::position
// (origin + extent * i / (n - 1), marching.hpp:21-24). Rounding is per IEEE op
// (no contraction) so the cell and local match the reference bit for bit.
__global__ void k_axis_table(DevSpec s, int dim, int3 n, int mode, double3 org, double3 ext, double3 step,
                             AxisLoc* loc, float4* fac, int* cell) {
    const int total = n.x + n.y + n.z;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < total; j += gridDim.x * blockDim.x) {
        int a = 0, i = j;
        if (i >= n.x) {
            i -= n.x;
            a = 1;
            if (i >= n.y) {
                i -= n.y;
                a = 2;
            }
        }
        if (a >= dim) {  // unused axis of a 2D grid: a single lattice index
            if (loc) loc[j] = AxisLoc{0, 0, 0.0};
            if (fac) fac[j] = make_float4(1.0f, 0.0f, 0.0f, 0.0f);
            if (cell) cell[j] = 0;
            continue;
        }
        const double o = a == 0 ? org.x : (a == 1 ? org.y : org.z);
        const double e = a == 0 ? ext.x : (a == 1 ? ext.y : ext.z);
        const double h = a == 0 ? step.x : (a == 1 ? step.y : step.z);
        const int na = a == 0 ? n.x : (a == 1 ? n.y : n.z);
        const double p = mode == 0 ? __dadd_rn(o, __dmul_rn(h, (double)i))
                                   : __dadd_rn(o, __ddiv_rn(__dmul_rn(e, (double)i), (double)(na - 1)));
        double local;
        const int c = locate_axis(s, a, p, local);
        if (loc) loc[j] = AxisLoc{c, 0, local};
        if (fac) {
            const AxisF f = axis_factors(s, a, local);
            fac[j] = make_float4(f.s0, f.s1, f.d0, f.d1);
        }
        if (cell) cell[j] = c;
    }
}

// multilinear_resample: one thread per new vertex of one output row
// (blockIdx.y = y, blockIdx.z = z). The 8 corner weights are formed once in
// fp64 exactly as the reference does (w = ((1 * s_x) * s_y) * s_z with
// s = bit ? local : 1 - local; 1 * s_x is exact, so the x*y partial products
// are shared between corners) and reused for every channel; per channel the
// accumulation dst = sum_i w_i * src_i runs in the reference's corner order
// (0 + w_0 src_0 is exact, so the first term starts the sum), rounded once.
template <int DIM, int C>
__global__ void __launch_bounds__(128) k_resample(const AxisLoc* __restrict__ loc, int3 n, long long sy_old,
                                                  long long sz_old, const float* __restrict__ src, int Crt,
                                                  float* __restrict__ dst) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= n.x) return;
    const int NC = C > 0 ? C : Crt;
    const int y = blockIdx.y, z = blockIdx.z;
    const AxisLoc lx = loc[x];
    const AxisLoc ly = loc[n.x + y];
    const AxisLoc lz = DIM == 3 ? loc[n.x + n.y + z] : AxisLoc{0, 0, 0.0};
    const long long base = lx.cell + ly.cell * sy_old + (DIM == 3 ? lz.cell * sz_old : 0);
    const double sx[2] = {__dsub_rn(1.0, lx.local), lx.local};
    const double sy[2] = {__dsub_rn(1.0, ly.local), ly.local};
    const double sz[2] = {__dsub_rn(1.0, lz.local), lz.local};
    double w[1 << DIM];
#pragma unroll
    for (int i = 0; i < (1 << DIM); ++i) {
        const double wxy = __dmul_rn(sx[i & 1], sy[(i >> 1) & 1]);
        w[i] = DIM == 3 ? __dmul_rn(wxy, sz[(i >> 2) & 1]) : wxy;
    }
    const float* sp[1 << DIM];
#pragma unroll
    for (int i = 0; i < (1 << DIM); ++i)
        sp[i] = src + (base + (i & 1) + ((i >> 1) & 1) * sy_old + (DIM == 3 ? ((i >> 2) & 1) * sz_old : 0)) * NC;
    float* dp = dst + (((long long)z * n.y + y) * n.x + x) * NC;
#pragma unroll(C > 0 ? C : 1)
    for (int ch = 0; ch < NC; ++ch) {
        double acc = __dmul_rn(w[0], (double)__ldg(sp[0] + ch));
#pragma unroll
        for (int i = 1; i < (1 << DIM); ++i) acc = __dadd_rn(acc, __dmul_rn(w[i], (double)__ldg(sp[i] + ch)));
        dp[ch] = (float)acc;
    }
}

// sample_grid_field: one thread per lattice point of one lattice row (x
// fastest, so a warp shares cells and its block gathers hit L1); per-axis fp32
// factors from the table.
template <int DIM, int ORDER>
__global__ void __launch_bounds__(256) k_eval_lattice(DevSpec s, const float* __restrict__ coeffs,
                                                      const float4* __restrict__ fac, const int* __restrict__ cell,
                                                      int3 n, float* __restrict__ vals) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= n.x) return;
    const int y = blockIdx.y, z = blockIdx.z;
    const int idx[3] = {x, n.x + y, n.x + n.y + z};
    AxisF ax[DIM];
    long long base = 0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        const float4 f = __ldg(fac + idx[a]);
        ax[a] = AxisF{f.x, f.y, f.z, f.w};
        base += (long long)__ldg(cell + idx[a]) * (a == 0 ? 1LL : (a == 1 ? s.sy : s.sz));
    }
    float fg[DIM];
    vals[((long long)z * n.y + y) * n.x + x] = eval_cell<DIM, ORDER, false>(s, coeffs, base, ax, fg);
}

namespace {

int3 lattice3(const int* lat, int dim) { return make_int3(lat[0], lat[1], dim == 3 ? lat[2] : 1); }

// Resample `data` (old_spec vertices x C channels, device) onto new_res into
// `out` (device), stream-ordered. Scratch tables are stream-allocated.
void resample_device(const tgcu_grid_spec& old_spec, const float* data, int C, const int* new_res, float* out,
                     cudaStream_t st) {
    const DevSpec s = make_devspec(old_spec);
    const int dim = old_spec.dim;
    const int3 n = lattice3(new_res, dim);
    double3 org{old_spec.origin[0], old_spec.origin[1], old_spec.origin[2]};
    double3 ext{old_spec.extent[0], old_spec.extent[1], old_spec.extent[2]};
    double hn[3] = {1.0, 1.0, 1.0};
    for (int a = 0; a < dim; ++a) hn[a] = old_spec.extent[a] / (new_res[a] - 1);  // GridSpec::spacing of the new spec
    const double3 step{hn[0], hn[1], hn[2]};
    AxisLoc* loc = nullptr;
    const int na = n.x + n.y + n.z;
    TGCU_CUDA(cudaMallocAsync(&loc, sizeof(AxisLoc) * na, st));
    k_axis_table<<<grid_blocks(na, 256), 256, 0, st>>>(s, dim, n, 0, org, ext, step, loc, nullptr, nullptr);
    count_launch();
    require(n.y < 65536 && n.z < 65536, "multilinear_resample: resolution too large");
    const int thr = std::min(128, (n.x + 31) / 32 * 32);
    const dim3 blocks((n.x + thr - 1) / thr, n.y, n.z);
#define TGCU_RS(DIMV, CV) k_resample<DIMV, CV><<<blocks, thr, 0, st>>>(loc, n, s.sy, s.sz, data, C, out)
    if (dim == 3) {
        if (C == 10) TGCU_RS(3, 10);
        else if (C == 4) TGCU_RS(3, 4);
        else if (C == 1) TGCU_RS(3, 1);
        else TGCU_RS(3, 0);
    } else {
        if (C == 6) TGCU_RS(2, 6);
        else if (C == 3) TGCU_RS(2, 3);
        else if (C == 1) TGCU_RS(2, 1);
        else TGCU_RS(2, 0);
    }
#undef TGCU_RS
    count_launch();
    TGCU_CUDA(cudaGetLastError());
    TGCU_CUDA(cudaFreeAsync(loc, st));
}

constexpr char kMagic[4] = {'T', 'G', 'R', 'D'};
constexpr uint32_t kVersion = 1;

template <class T>
T read_pod(std::istream& is, const char* what) {
    T v{};
    if (!is.read(reinterpret_cast<char*>(&v), sizeof(T)))
        throw Error(TGCU_ERR_INGEST, std::string("tgrid: truncated file while reading ") + what);
    return v;
}

template <class T>
void write_pod(std::ostream& os, const T& v) {
    os.write(reinterpret_cast<const char*>(&v), sizeof(T));
}

// Host chunk (floats) for streaming multi-GB payloads through bounded memory.
constexpr int64_t kIoChunk = 1 << 22;

}  // namespace

}  // namespace tgcu

using namespace tgcu;

extern "C" {

int tgcu_multilinear_resample(const tgcu_grid_spec* old_spec, const float* data, int64_t n, int channels,
                              const int new_res[3], float* out, int flags, void* stream) {
    return guard([&] {
        require(old_spec && new_res, "multilinear_resample: NULL argument");
        tgcu_grid_spec o = *old_spec;
        if (o.dim == 2) o.res[2] = 1;
        validate_spec(o);
        require(channels >= 1, "multilinear_resample: channels must be >= 1");
        tgcu_grid_spec ng = o;
        for (int a = 0; a < o.dim; ++a) ng.res[a] = new_res[a];
        validate_spec(ng);  // GridSpec::validate of the new geometry (taylor_grid.cpp:235)
        int64_t vo = 1, vn = 1;
        for (int a = 0; a < o.dim; ++a) {
            vo *= o.res[a];
            vn *= ng.res[a];
        }
        require(n == vo * channels, "multilinear_resample: data size mismatch");
        cudaStream_t st = as_stream(stream);
        const float* d_in = data;
        float* d_out = out;
        float* tmp = nullptr;
        if (flags & TGCU_HOST) {
            TGCU_CUDA(cudaMallocAsync(&tmp, sizeof(float) * (n + vn * channels), st));
            TGCU_CUDA(cudaMemcpyAsync(tmp, data, sizeof(float) * n, cudaMemcpyHostToDevice, st));
            d_in = tmp;
            d_out = tmp + n;
        }
        resample_device(o, d_in, channels, ng.res, d_out, st);
        if (flags & TGCU_HOST) {
            TGCU_CUDA(cudaMemcpyAsync(out, d_out, sizeof(float) * vn * channels, cudaMemcpyDeviceToHost, st));
            TGCU_CUDA(cudaFreeAsync(tmp, st));
        }
        if ((flags & TGCU_HOST) || !(flags & TGCU_ASYNC)) TGCU_CUDA(cudaStreamSynchronize(st));
    });
}

int tgcu_grid_upsample(tgcu_grid* src, tgcu_grid* dst, int flags, void* stream) {
    return guard([&] {
        require(src && dst, "upsample: NULL grid");
        Grid& a = src->g;
        Grid& b = dst->g;
        require(!a.slab && !b.slab, "upsample: slab grids are not supported");
        require(a.device == b.device, "upsample: grids live on different devices");
        require(a.spec.dim == b.spec.dim && a.spec.order == b.spec.order,
                "upsample: destination must have the source's dim and order");
        for (int ax = 0; ax < a.spec.dim; ++ax) {
            require(a.spec.origin[ax] == b.spec.origin[ax] && a.spec.extent[ax] == b.spec.extent[ax],
                    "upsample: destination must have the source's origin and extent");
            require(b.spec.res[ax] >= a.spec.res[ax],
                    "upsample: resolution may not shrink (axis " + std::to_string(ax) + ")");
        }
        TGCU_CUDA(cudaSetDevice(a.device));
        cudaStream_t st = as_stream(stream);
        resample_device(a.spec, a.p[a.cur], a.K, b.spec.res, b.p[b.cur], st);
        if (!(flags & TGCU_ASYNC)) TGCU_CUDA(cudaStreamSynchronize(st));
    });
}

int tgcu_sample_grid_field(tgcu_grid* h, const int lattice[3], float* values, int flags, void* stream) {
    return guard([&] {
        require(h && lattice, "sample_grid_field: NULL argument");
        Grid& g = h->g;
        require(!g.slab, "sample_grid_field: slab grids are not supported");
        const int dim = g.spec.dim;
        for (int a = 0; a < dim; ++a)
            require(lattice[a] >= 2, "sample_field3: resolution must be >= 2 per axis");
        TGCU_CUDA(cudaSetDevice(g.device));
        cudaStream_t st = as_stream(stream);
        const int3 n = lattice3(lattice, dim);
        const long long total = (long long)n.x * n.y * n.z;
        const int na = n.x + n.y + n.z;
        float4* fac = nullptr;
        TGCU_CUDA(cudaMallocAsync(&fac, sizeof(float4) * na + sizeof(int) * na +
                                            ((flags & TGCU_HOST) ? sizeof(float) * total : 0), st));
        int* cell = reinterpret_cast<int*>(fac + na);
        float* dv = (flags & TGCU_HOST) ? reinterpret_cast<float*>(cell + na) : values;
        const double3 org{g.spec.origin[0], g.spec.origin[1], g.spec.origin[2]};
        const double3 ext{g.spec.extent[0], g.spec.extent[1], g.spec.extent[2]};
        k_axis_table<<<grid_blocks(na, 256), 256, 0, st>>>(g.ds, dim, n, 1, org, ext, double3{1.0, 1.0, 1.0},
                                                           nullptr, fac, cell);
        count_launch();
        require(n.y < 65536 && n.z < 65536, "sample_grid_field: lattice too large");
        // dense lattices: one CTA per grid brick evaluates its lattice points
        // from the brick's shared-memory tile (query.cu); sparse ones: a
        // thread per lattice point reading the corner blocks through L1/L2
        if (!launch_eval_lattice_brick(g, fac, cell, n, dv, st)) {
            const int thr = std::min(256, (n.x + 31) / 32 * 32);
            const dim3 blocks((n.x + thr - 1) / thr, n.y, n.z);
            TGCU_DISPATCH(dim, g.spec.order, {
                k_eval_lattice<DIM, ORDER><<<blocks, thr, 0, st>>>(g.ds, g.p[g.cur], fac, cell, n, dv);
            });
            count_launch();
        }
        TGCU_CUDA(cudaGetLastError());
        if (flags & TGCU_HOST)
            TGCU_CUDA(cudaMemcpyAsync(values, dv, sizeof(float) * total, cudaMemcpyDeviceToHost, st));
        TGCU_CUDA(cudaFreeAsync(fac, st));
        if ((flags & TGCU_HOST) || !(flags & TGCU_ASYNC)) TGCU_CUDA(cudaStreamSynchronize(st));
    });
}

int tgcu_draw_batch(const float* pool, int64_t pool_n, int64_t n, uint64_t seed, uint64_t step, float* out,
                    void* stream) {
    return guard([&] {
        require(pool && out, "draw_batch: NULL argument");
        require(pool_n > 0, "fit_sdf: sample set is empty");
        require(n >= 0, "draw_batch: negative batch size");
        require((reinterpret_cast<uintptr_t>(pool) | reinterpret_cast<uintptr_t>(out)) % 16 == 0,
                "draw_batch: pool and out must be 16-byte aligned");
        launch_draw_batch(pool, pool_n, n, seed, step, out, as_stream(stream));
    });
}

int64_t tgcu_tgrid_file_size(const tgcu_grid_spec* s, int precision) {
    if (!s || (s->dim != 2 && s->dim != 3) || s->order < 0 || s->order > 2) return -1;
    int64_t v = 1;
    for (int a = 0; a < s->dim; ++a) v *= s->res[a];
    const int64_t header = 4 + 4 + 1 + 1 + 4ll * s->dim + 8ll * s->dim * 2 + 1;
    return header + v * coeff_count_of(s->order, s->dim) * (precision == TGCU_TGRID_F64 ? 8 : 4);
}

int tgcu_save_tgrid(tgcu_grid* h, const char* path, int precision) {
    return guard([&] {
        require(h && path, "save_tgrid: NULL argument");
        Grid& g = h->g;
        require(!g.slab, "save_tgrid: slab grids are not supported");
        require(precision == TGCU_TGRID_F64 || precision == TGCU_TGRID_F32, "save_tgrid: unknown precision");
        // Commit any pending async step first (sticky errors surface here,
        // before the file is created: a failed step leaves no partial file).
        {
            tgcu_loss_terms t;
            const int rc = tgcu_sync(h, &t);
            if (rc != TGCU_OK) throw Error(rc, tgcu_last_error());
        }
        std::ofstream os(path, std::ios::binary);
        if (!os) throw Error(TGCU_ERR_INGEST, std::string("tgrid: cannot open for writing: ") + path);
        const tgcu_grid_spec& s = g.spec;
        os.write(kMagic, 4);
        write_pod(os, kVersion);
        write_pod(os, static_cast<uint8_t>(s.dim));
        write_pod(os, static_cast<uint8_t>(s.order));
        for (int a = 0; a < s.dim; ++a) write_pod(os, static_cast<uint32_t>(s.res[a]));
        for (int a = 0; a < s.dim; ++a) write_pod(os, s.origin[a]);
        for (int a = 0; a < s.dim; ++a) write_pod(os, s.extent[a]);
        write_pod(os, static_cast<uint8_t>(precision));
        TGCU_CUDA(cudaSetDevice(g.device));
        std::vector<float> buf((size_t)std::min<int64_t>(g.NC, kIoChunk));
        std::vector<double> wide(precision == TGCU_TGRID_F64 ? buf.size() : 0);
        for (int64_t off = 0; off < g.NC; off += kIoChunk) {
            const int64_t m = std::min<int64_t>(kIoChunk, g.NC - off);
            TGCU_CUDA(cudaMemcpy(buf.data(), g.p[g.cur] + off, sizeof(float) * m, cudaMemcpyDeviceToHost));
            if (precision == TGCU_TGRID_F64) {
                for (int64_t i = 0; i < m; ++i) wide[i] = buf[i];
                os.write(reinterpret_cast<const char*>(wide.data()), (std::streamsize)(m * sizeof(double)));
            } else {
                os.write(reinterpret_cast<const char*>(buf.data()), (std::streamsize)(m * sizeof(float)));
            }
        }
        if (!os) throw Error(TGCU_ERR_INGEST, std::string("tgrid: write failed: ") + path);
    });
}

int tgcu_load_tgrid(const char* path, int device, tgcu_grid** out) {
    if (out) *out = nullptr;
    tgcu_grid* h = nullptr;
    const int rc = guard([&] {
        require(path && out, "load_tgrid: NULL argument");
        std::ifstream is(path, std::ios::binary);
        if (!is) throw Error(TGCU_ERR_INGEST, std::string("tgrid: cannot open: ") + path);
        char magic[4];
        if (!is.read(magic, 4) || std::memcmp(magic, kMagic, 4) != 0)
            throw Error(TGCU_ERR_INGEST, std::string("tgrid: bad magic in ") + path);
        const auto version = read_pod<uint32_t>(is, "version");
        if (version != kVersion) throw Error(TGCU_ERR_INGEST, "tgrid: unsupported version " + std::to_string(version));
        tgcu_grid_spec s{};
        s.dim = read_pod<uint8_t>(is, "dim");
        s.order = read_pod<uint8_t>(is, "order");
        if (s.dim != 2 && s.dim != 3) throw Error(TGCU_ERR_INGEST, "tgrid: unsupported dim " + std::to_string(s.dim));
        s.res[0] = s.res[1] = s.res[2] = 2;  // GridSpec defaults on unused axes
        s.origin[0] = s.origin[1] = s.origin[2] = -1.0;
        s.extent[0] = s.extent[1] = s.extent[2] = 2.0;
        for (int a = 0; a < s.dim; ++a) s.res[a] = static_cast<int>(read_pod<uint32_t>(is, "resolution"));
        for (int a = 0; a < s.dim; ++a) s.origin[a] = read_pod<double>(is, "origin");
        for (int a = 0; a < s.dim; ++a) s.extent[a] = read_pod<double>(is, "extent");
        const auto precision = read_pod<uint8_t>(is, "precision");
        {
            tgcu_grid_spec v = s;
            if (v.dim == 2) v.res[2] = 1;
            validate_spec(v);  // spec.validate() -> std::invalid_argument (grid_io.cpp:91)
        }
        if (precision != TGCU_TGRID_F64 && precision != TGCU_TGRID_F32)
            throw Error(TGCU_ERR_INGEST, "tgrid: unknown precision flag");
        tgcu_init_options opts{TGCU_INIT_ZEROS, 0.0, 0.0, 0, std::numeric_limits<uint64_t>::max()};
        const int crc = tgcu_grid_create(&s, &opts, device, &h);
        if (crc != TGCU_OK) throw Error(crc, tgcu_last_error());
        Grid& g = h->g;
        std::vector<float> buf((size_t)std::min<int64_t>(g.NC, kIoChunk));
        std::vector<double> wide(precision == TGCU_TGRID_F64 ? buf.size() : 0);
        for (int64_t off = 0; off < g.NC; off += kIoChunk) {
            const int64_t m = std::min<int64_t>(kIoChunk, g.NC - off);
            const bool ok = precision == TGCU_TGRID_F64
                                ? (bool)is.read(reinterpret_cast<char*>(wide.data()), (std::streamsize)(m * 8))
                                : (bool)is.read(reinterpret_cast<char*>(buf.data()), (std::streamsize)(m * 4));
            if (!ok) throw Error(TGCU_ERR_INGEST, std::string("tgrid: truncated coefficient payload in ") + path);
            if (precision == TGCU_TGRID_F64)
                for (int64_t i = 0; i < m; ++i) buf[i] = (float)wide[i];
            TGCU_CUDA(cudaMemcpy(g.p[g.cur] + off, buf.data(), sizeof(float) * m, cudaMemcpyHostToDevice));
        }
    });
    if (rc != TGCU_OK) {
        if (h) tgcu_grid_destroy(h);
        return rc;
    }
    *out = h;
    return TGCU_OK;
}

}  // extern "C"

// ---- Monte-Carlo IoU probe (metrics.cpp:104-124) -----------------------------------
// The reference's probe: points from Rng(seed).uniform_in_box(lo, hi, dim),
// drawn in order on the host (mt19937_64, rng.hpp:53-57), inside = field < 0
// for both fields; field a = this grid on the device, field b = grid b or
// the analytic sphere |p| - radius (cmd_bench's target, tools/main.cpp:604).
// Chunks of points are evaluated on the device (direct-gather query);
// counting on the host in point order.
int tgcu_iou(tgcu_grid* a, tgcu_grid* b, double sphere_radius, const tgcu_iou_options* o, double* iou,
             int* empty_union) {
    return guard([&] {
        require(a != nullptr && o != nullptr && iou != nullptr, "iou: NULL argument");
        require(o->samples > 0, "iou: sample count must be > 0");
        require(o->dim == 2 || o->dim == 3, "iou: dim must be 2 or 3");
        Grid& ga = a->g;
        require(!ga.slab && (!b || !b->g.slab), "iou: slab grids are not supported");
        TGCU_CUDA(cudaSetDevice(ga.device));
        tgcu_rng* rng = nullptr;
        if (tgcu_rng_create(o->seed, &rng) != TGCU_OK) throw Error(TGCU_ERR_CUDA, tgcu_last_error());
        const int64_t chunk = std::min<int64_t>(o->samples, 1 << 20);
        std::vector<double> p64((size_t)(3 * chunk));
        std::vector<float> p32((size_t)(3 * chunk)), va((size_t)chunk), vb(b ? (size_t)chunk : 0);
        int64_t inter = 0, uni = 0;
        try {
            for (int64_t done = 0; done < o->samples; done += chunk) {
                const int64_t m = std::min(chunk, o->samples - done);
                if (tgcu_rng_uniform_box(rng, o->dim, o->lo, o->hi, m, p64.data()) != TGCU_OK)
                    throw Error(TGCU_ERR_CUDA, tgcu_last_error());
                for (int64_t i = 0; i < 3 * m; ++i) p32[i] = (float)p64[i];
                int rc = tgcu_eval(a, p32.data(), m, va.data(), nullptr, TGCU_HOST, nullptr);
                if (rc == TGCU_OK && b) rc = tgcu_eval(b, p32.data(), m, vb.data(), nullptr, TGCU_HOST, nullptr);
                if (rc != TGCU_OK) throw Error(rc, tgcu_last_error());
                for (int64_t i = 0; i < m; ++i) {
                    const bool in_a = va[i] < 0.0f;
                    bool in_b;
                    if (b) {
                        in_b = vb[i] < 0.0f;
                    } else {
                        const double* p = &p64[3 * i];
                        double r2 = 0.0;
                        for (int d = 0; d < 3; ++d) r2 += p[d] * p[d];
                        in_b = std::sqrt(r2) - sphere_radius < 0.0;
                    }
                    inter += in_a && in_b;
                    uni += in_a || in_b;
                }
            }
        } catch (...) {
            tgcu_rng_destroy(rng);
            throw;
        }
        tgcu_rng_destroy(rng);
        if (empty_union) *empty_union = uni == 0;
        *iou = uni == 0 ? 1.0 : (double)inter / (double)uni;
    });
}
