// K1 — forward query (eval / eval_with_spatial_gradient, taylor_grid.cpp:100-119).
//
// Two kernels:
//  * k_eval_direct: one thread per point, fp64 locate, 2^D vectorised block
//    gathers straight from HBM/L2 (__ldg), fp32 blend. For unsorted points.
//  * k_eval_brick: one CTA per brick of cells; the brick's (B+1)^D vertex tile
//    is staged in shared memory once and every point of the brick gathers from
//    it. Points must be brick-sorted (tgcu_sort_points); each CTA finds its
//    point range by binary search over the brick keys, so no offsets array is
//    read. This is the coherent-points path.

#include <cstdlib>
#include <functional>

#include "dispatch.cuh"
#include "tg_internal.h"
#include "tma.cuh"

namespace tgcu {

template <int DIM, int ORDER, bool GRAD>
__global__ void __launch_bounds__(256) k_eval_direct(DevSpec s, const float* __restrict__ coeffs,
                                                     const float* __restrict__ pts, long long n,
                                                     float* __restrict__ vals, float* __restrict__ grads,
                                                     Status* st) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double x[DIM];
        bool nan = false;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            x[a] = (double)pts[3 * i + a];
            nan |= isnan(x[a]);
        }
        if (nan) {
            atomicMin(&st->nan_point, (unsigned long long)i);
            vals[i] = __int_as_float(0x7fc00000);
            if (GRAD)
                for (int a = 0; a < 3; ++a) grads[3 * i + a] = __int_as_float(0x7fc00000);
            continue;
        }
        AxisF ax[DIM];
        long long base = 0;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            double local;
            const int c = locate_axis(s, a, x[a], local);
            ax[a] = axis_factors(s, a, local);
            base += (long long)c * (a == 0 ? 1LL : (a == 1 ? s.sy : s.sz));
        }
        float fg[DIM];
        vals[i] = eval_cell<DIM, ORDER, GRAD>(s, coeffs, base, ax, fg);
        if (GRAD) {
#pragma unroll
            for (int a = 0; a < 3; ++a) grads[3 * i + a] = a < DIM ? fg[a] : 0.0f;
        }
    }
}

void launch_eval_direct(Grid& g, const float* pts, int64_t n, float* vals, float* grads, cudaStream_t s) {
    if (n <= 0) return;
    const int threads = 256;
    const int blocks = grid_blocks(n, threads, 148 * 32);
    TGCU_DISPATCH(g.spec.dim, g.spec.order, {
        if (grads)
            k_eval_direct<DIM, ORDER, true><<<blocks, threads, 0, s>>>(g.ds, g.p[g.cur], pts, n, vals, grads, g.st);
        else
            k_eval_direct<DIM, ORDER, false><<<blocks, threads, 0, s>>>(g.ds, g.p[g.cur], pts, n, vals, grads, g.st);
    });
    count_launch();
    TGCU_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Brick-binned query.
//
// Brick key of a point: its cell's brick coordinates (cell >> log2 B per axis),
// Morton-interleaved so that consecutive bricks are spatially adjacent. A
// brick covers cells [B*b, B*b + B) and needs vertices [B*b, B*b + B].

__device__ __forceinline__ unsigned long long spread3(unsigned long long x) {
    x &= 0x1fffffULL;
    x = (x | x << 32) & 0x1f00000000ffffULL;
    x = (x | x << 16) & 0x1f0000ff0000ffULL;
    x = (x | x << 8) & 0x100f00f00f00f00fULL;
    x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
    x = (x | x << 2) & 0x1249249249249249ULL;
    return x;
}
// 32-bit spread of a 10-bit value (brick coordinates: at most 512 bricks per
// axis), a third of the 64-bit version's instructions.
__device__ __forceinline__ unsigned int spread3_10(unsigned int x) {
    x &= 0x3ffu;
    x = (x | x << 16) & 0x030000ffu;
    x = (x | x << 8) & 0x0300f00fu;
    x = (x | x << 4) & 0x030c30c3u;
    x = (x | x << 2) & 0x09249249u;
    return x;
}
__device__ __forceinline__ unsigned int compact3_10(unsigned int x) {  // inverse of spread3_10
    x &= 0x09249249u;
    x = (x | x >> 2) & 0x030c30c3u;
    x = (x | x >> 4) & 0x0300f00fu;
    x = (x | x >> 8) & 0x030000ffu;
    x = (x | x >> 16) & 0x3ffu;
    return x;
}
__device__ __forceinline__ unsigned int compact2_16(unsigned int x) {  // inverse of spread2 (16-bit)
    x &= 0x55555555u;
    x = (x | x >> 1) & 0x33333333u;
    x = (x | x >> 2) & 0x0f0f0f0fu;
    x = (x | x >> 4) & 0x00ff00ffu;
    x = (x | x >> 8) & 0x0000ffffu;
    return x;
}
__device__ __forceinline__ unsigned long long spread2(unsigned long long x) {
    x &= 0xffffffffULL;
    x = (x | x << 16) & 0x0000ffff0000ffffULL;
    x = (x | x << 8) & 0x00ff00ff00ff00ffULL;
    x = (x | x << 4) & 0x0f0f0f0f0f0f0f0fULL;
    x = (x | x << 2) & 0x3333333333333333ULL;
    x = (x | x << 1) & 0x5555555555555555ULL;
    return x;
}

// Full key = Morton(brick) << (DIM*LB) | Morton(cell within brick): sorting by
// it groups points by brick (brick order = Morton) and orders them inside the
// brick by cell, so neighbouring threads share vertex blocks.
template <int DIM, int LB>
__device__ __forceinline__ unsigned long long point_key(const DevSpec& s, const float* p, unsigned int* brick) {
    unsigned long long kb = 0, kc = 0;
    unsigned int c[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        double local;
        double x = (double)p[a];
        if (isnan(x)) x = s.origin[a];
        c[a] = (unsigned int)locate_axis(s, a, x, local);
    }
    if (DIM == 3) {
        kb = spread3(c[0] >> LB) | (spread3(c[1] >> LB) << 1) | (spread3(c[2] >> LB) << 2);
        kc = spread3(c[0] & ((1u << LB) - 1)) | (spread3(c[1] & ((1u << LB) - 1)) << 1) |
             (spread3(c[2] & ((1u << LB) - 1)) << 2);
    } else {
        kb = spread2(c[0] >> LB) | (spread2(c[1] >> LB) << 1);
        kc = spread2(c[0] & ((1u << LB) - 1)) | (spread2(c[1] & ((1u << LB) - 1)) << 1);
    }
    if (brick) *brick = (unsigned int)kb;
    return (kb << (DIM * LB)) | kc;
}

template <int DIM>
constexpr int brick_log2() { return DIM == 3 ? 3 : 4; }

// Row stride (floats) of the query tile: T*K rounded to 16 bytes, padded for
// the 3D K = 10 / K = 4 tiles so that the y-row and z-plane strides spread a
// warp's Morton-neighbouring cells over the shared-memory banks (simulated
// LDS.64 wavefronts: 1.87x -> 1.72x of ideal for K = 10, 3.3x -> 2.6x for K = 4).
template <int DIM, int K, int T>
constexpr int query_trowf() {
    return (DIM == 3 && K == 10) ? 100 : (DIM == 3 && K == 4) ? 48 : ((T * K + 3) / 4) * 4;
}
// Rows per tile plane (3D). Tensor boxes land densely, so with T rows the
// plane pitch T * TROWF is congruent to the row pitch modulo the 32 banks for
// any 16-byte-multiple TROWF, and a cell's y and z corners collide. For K = 10
// the box carries one extra row per plane (pitch 10 x 100 floats: the bank
// model tools/bank_model.py gives 4.28 instead of 4.58 wavefronts per 64-bit
// corner load; 6 CTAs still fit per SM).
template <int DIM, int K, int T>
constexpr int query_plane_rows() {
    return (DIM == 3 && K == 10) ? T + 1 : T;
}
#ifndef QMINB_SMALL
#define QMINB_SMALL 8
#endif
// Resident CTAs per SM the register budget is sized for: the tile of a K = 10
// brick (33.7 KB) allows 6, smaller tiles 8 (measured: 5 -> 6 CTAs took the
// 512^3 order-2 sorted query from 53 % to 59 % of the HBM roofline).
template <int K>
constexpr int query_min_blocks() { return K >= 10 ? 6 : QMINB_SMALL; }

// Number of Morton brick codes of the query decomposition (pow2^DIM).
int64_t query_brick_codes(const Grid& g) {
    const int LB = g.spec.dim == 3 ? 3 : 4;
    const int B = 1 << LB;
    unsigned int pow2 = 1;
    for (int a = 0; a < g.spec.dim; ++a) {
        const int nb = (g.spec.res[a] - 1 + B - 1) / B;  // bricks of cells
        while (pow2 < (unsigned)nb) pow2 <<= 1;
    }
    int64_t codes = 1;
    for (int a = 0; a < g.spec.dim; ++a) codes *= pow2;
    return codes;
}

// off[c] = first sorted index whose brick code >= c, for c in [0, codes].
// Each i writes the codes in (code(i-1), code(i)]; the last point also writes
// the tail up to `codes`.
template <int DIM, int LB, bool FROM_KEYS, class KeyT>
__global__ void k_brick_offsets(DevSpec s, const KeyT* __restrict__ keys, const float* __restrict__ pts,
                                long long n, long long codes, long long* __restrict__ off) {
    constexpr int SH = DIM * LB;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i <= n;
         i += (long long)gridDim.x * blockDim.x) {
        long long prev = -1, cur = codes;
        unsigned int kb;
        if (i > 0) {
            if (FROM_KEYS) prev = (long long)(keys[i - 1] >> SH);
            else { point_key<DIM, LB>(s, pts + 3 * (i - 1), &kb); prev = kb; }
        }
        if (i < n) {
            if (FROM_KEYS) cur = (long long)(keys[i] >> SH);
            else { point_key<DIM, LB>(s, pts + 3 * i, &kb); cur = kb; }
        }
        for (long long c = prev + 1; c <= cur; ++c) off[c] = i;
    }
}

template <class KeyT>
void launch_brick_offsets(Grid& g, const KeyT* keys, const float* pts, int64_t n, int64_t* off, cudaStream_t s) {
    const long long codes = query_brick_codes(g);
    const int blocks = grid_blocks(n + 1, 256, 148 * 32);
    long long* o = reinterpret_cast<long long*>(off);
    if (g.spec.dim == 3) {
        if (keys) k_brick_offsets<3, 3, true, KeyT><<<blocks, 256, 0, s>>>(g.ds, keys, pts, n, codes, o);
        else k_brick_offsets<3, 3, false, KeyT><<<blocks, 256, 0, s>>>(g.ds, keys, pts, n, codes, o);
    } else {
        if (keys) k_brick_offsets<2, 4, true, KeyT><<<blocks, 256, 0, s>>>(g.ds, keys, pts, n, codes, o);
        else k_brick_offsets<2, 4, false, KeyT><<<blocks, 256, 0, s>>>(g.ds, keys, pts, n, codes, o);
    }
    count_launch();
    TGCU_CUDA(cudaGetLastError());
}

struct QpArgs;
void launch_qpart(Grid& g, const float* pts, int64_t n, float4* B, float* out_xyz, int64_t* perm, long long* off,
                  float* vals, float* grads, cudaStream_t s, unsigned short* lpos = nullptr,
                  const std::function<void(const QpArgs&)>& after = {});

// Brick sort of query points (tgcu_sort_points): the two-pass partition by
// Morton brick code (launch_qpart below) writing the sorted coordinates and
// the source index of each. Points keep no order inside a brick; a NaN point
// sorts into the origin's brick (the query reports it).
void launch_sort_points(Grid& g, const float* pts, int64_t n, float* out, int64_t* perm, int64_t* offsets,
                        cudaStream_t s) {
    if (n <= 0) return;
    const int64_t codes = query_brick_codes(g);
    long long* off = reinterpret_cast<long long*>(offsets);
    long long* tmp = nullptr;
    if (!off) {
        TGCU_CUDA(cudaMallocAsync(&tmp, sizeof(long long) * (codes + 1), s));
        off = tmp;
    }
    launch_qpart(g, pts, n, nullptr, out, perm, off, nullptr, nullptr, s);
    if (tmp) TGCU_CUDA(cudaFreeAsync(tmp, s));
}

// Where a brick's points come from (k_eval_brick SRC): brick-sorted points
// (SRC 0: pts xyz, off = brick offsets by Morton code), binned points (SRC 1:
// pts = float4 x, y, z, caller index), or a lattice (SRC 2: per-axis factor /
// cell tables of the lattice coordinates and, per brick coordinate, the
// lattice index range [x, y) whose cells lie in it).
struct QuerySrc {
    const float* pts = nullptr;
    const long long* off = nullptr;
    const float4* fac = nullptr;
    const int* cell = nullptr;
    const int2* rng = nullptr;
    int3 n{1, 1, 1};     // lattice size
    int nb[3] = {1, 1, 1};  // bricks per axis (rng offsets)
    int morton = 0;         // 1-D launch over brick codes: CTAs walk the bricks in Morton order
};

// One CTA per brick of B^D cells (launch grid = bricks per axis); its points
// are [off[code], off[code+1]) of the brick-sorted array, code = Morton(brick)
// (or the lattice points whose cells lie in the brick).
// The brick's (B+1)^D vertex tile arrives by one TMA tensor box load
// (out-of-grid vertices zero-filled), or by one bulk copy per row when the
// grid layout cannot take a tensor map. Each thread loads and locates its first
// point before waiting for the tile, so the two latencies overlap.
template <int DIM, int ORDER, bool GRAD, int LB, int SRC = 0>
__global__ void __launch_bounds__(256, query_min_blocks<KOf<DIM, ORDER>::value>()) k_eval_brick(const __grid_constant__ CUtensorMap tmap, int use_tmap,
                                                    DevSpec s, const float* __restrict__ coeffs, const QuerySrc Q,
                                                    float* __restrict__ vals, float* __restrict__ grads,
                                                    Status* st) {
    constexpr bool BINNED = SRC == 1, LATTICE = SRC == 2;
    const float* __restrict__ pts = Q.pts;
    constexpr int K = KOf<DIM, ORDER>::value;
    constexpr int B = 1 << LB;
    constexpr int T = B + 1;  // tile edge in vertices
    constexpr int GR = (K % 2 == 0) ? 2 : 1;
    // tile rows (fixed y, z) of T vertices, stride TROWF floats (16-byte multiple)
    constexpr int TROWF = query_trowf<DIM, K, T>();
    constexpr int PR = query_plane_rows<DIM, K, T>();  // rows per plane (3D)
    constexpr int ROWS = DIM == 3 ? T * PR : T;
    constexpr unsigned RBYTES = ((T * K * 4 + 15) / 16) * 16;
    extern __shared__ __align__(128) float tile[];  // ROWS * TROWF
    __shared__ __align__(8) unsigned long long bar;

    unsigned int code, bxyz[3] = {blockIdx.x, blockIdx.y, blockIdx.z};
    if (!LATTICE && Q.morton) {
        code = blockIdx.x;
        if constexpr (DIM == 3) {
            bxyz[0] = compact3_10(code), bxyz[1] = compact3_10(code >> 1), bxyz[2] = compact3_10(code >> 2);
        } else {
            bxyz[0] = compact2_16(code), bxyz[1] = compact2_16(code >> 1), bxyz[2] = 0;
        }
    } else {
        code = DIM == 3 ? (spread3_10(blockIdx.x) | (spread3_10(blockIdx.y) << 1) | (spread3_10(blockIdx.z) << 2))
                        : (unsigned int)(spread2(blockIdx.x) | (spread2(blockIdx.y) << 1));
    }
    const int ox = (int)bxyz[0] * B, oy = (int)bxyz[1] * B, oz = DIM == 3 ? (int)bxyz[2] * B : 0;
    long long p0, p1;
    int2 lr[3] = {{0, 1}, {0, 1}, {0, 1}};  // lattice index range per axis
    if constexpr (LATTICE) {
        const int bc[3] = {(int)blockIdx.x, (int)blockIdx.y, (int)blockIdx.z};
        long long cnt = 1;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            lr[a] = Q.rng[(a > 0 ? Q.nb[0] : 0) + (a > 1 ? Q.nb[1] : 0) + bc[a]];
            cnt *= max(0, lr[a].y - lr[a].x);
        }
        p0 = 0;
        p1 = cnt;
    } else {
        p0 = Q.off[code];
        p1 = Q.off[code + 1];
    }
    if (p0 >= p1) return;
    const bool tm = use_tmap != 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar, tm ? 1 : blockDim.x);
        mbar_fence_init();
        if (tm) {
            mbar_expect_tx(&bar, (unsigned)(ROWS * TROWF * 4));
            if constexpr (DIM == 3) tma_load_3d(tile, &tmap, &bar, ox * K, oy, oz);
            else tma_load_2d(tile, &tmap, &bar, ox * K, oy);
        }
    }
    if (!tm) {
        __syncthreads();  // barrier initialised before the per-row arrivals
        // one TMA bulk copy per row (thread r), cp.async fallback when the row
        // is unaligned or runs past the array
        const long long nc_bytes = (long long)s.res[0] * s.res[1] * (DIM == 3 ? s.res[2] : 1) * K * 4;
        const int r = threadIdx.x;
        bool arrived = false;
        if (r < ROWS && (DIM == 2 || r % PR < T)) {
            const int ty = DIM == 3 ? r % PR : r, tz = DIM == 3 ? r / PR : 0;
            const int vy = oy + ty, vz = oz + tz;
            if (vy < s.res[1] && (DIM == 2 || vz < s.res[2])) {
                const long long v0 = (DIM == 3 ? (long long)vz * s.sz : 0LL) + (long long)vy * s.sy + ox;
                const long long src = v0 * K * 4;
                float* dst = tile + r * TROWF;
                if ((src & 15) == 0 && src + RBYTES <= nc_bytes) {
                    mbar_expect_tx(&bar, RBYTES);
                    bulk_g2s(dst, reinterpret_cast<const char*>(coeffs) + src, RBYTES, &bar);
                } else {
                    mbar_expect_tx(&bar, 0);
                    for (int q = 0; q < T * K; q += GR) {
                        const bool ok = ox + q / K < s.res[0];
                        cp_async<GR>(dst + q, ok ? coeffs + v0 * K + q : coeffs, ok);
                    }
                }
                arrived = true;
            }
        }
        if (!arrived) mbar_arrive(&bar);
        cp_async_commit();
    }

    const int o3[3] = {ox, oy, oz};
    // locate of point i: cell-relative tile offset and per-axis factors (false
    // for NaN); oi = the output slot (i, or the caller's index of a binned point)
    auto prepare = [&](long long i, AxisF* ax, int& tbase, long long& oi) -> bool {
        if constexpr (LATTICE) {
            // lattice point (X, Y, Z): per-axis factors and cells from the tables
            const int nx = lr[0].y - lr[0].x, ny = lr[1].y - lr[1].x;
            const int li = (int)i;
            const int X = lr[0].x + li % nx, Y = lr[1].x + (li / nx) % ny, Z = lr[2].x + li / (nx * ny);
            const int idx[3] = {X, Q.n.x + Y, Q.n.x + Q.n.y + Z};
            int lc[3] = {0, 0, 0};
#pragma unroll
            for (int a = 0; a < DIM; ++a) {
                const float4 f = __ldg(Q.fac + idx[a]);
                ax[a] = AxisF{f.x, f.y, f.z, f.w};
                lc[a] = __ldg(Q.cell + idx[a]) - o3[a];
            }
            oi = DIM == 3 ? ((long long)Z * Q.n.y + Y) * Q.n.x + X : (long long)Y * Q.n.x + X;
            tbase = (DIM == 3 ? lc[2] * PR + lc[1] : lc[1]) * TROWF + lc[0] * K;
            return true;
        }
        double x[DIM];
        bool nan = false;
        if constexpr (BINNED) {
            const float4 q = reinterpret_cast<const float4*>(pts)[i];
            const float qq[3] = {q.x, q.y, q.z};
#pragma unroll
            for (int a = 0; a < DIM; ++a) x[a] = (double)qq[a];
            oi = (long long)(unsigned int)__float_as_int(q.w);
        } else {
#pragma unroll
            for (int a = 0; a < DIM; ++a) {
                x[a] = (double)pts[3 * i + a];
                nan |= isnan(x[a]);
            }
            oi = i;
        }
        if (nan) {
            atomicMin(&st->nan_point, (unsigned long long)i);
            vals[i] = __int_as_float(0x7fc00000);
            if (GRAD)
                for (int a = 0; a < 3; ++a) grads[3 * i + a] = __int_as_float(0x7fc00000);
            return false;
        }
        int lc[3] = {0, 0, 0};
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            double local;
            const int c = locate_axis(s, a, x[a], local);
            ax[a] = axis_factors(s, a, local);
            lc[a] = c - o3[a];
        }
        tbase = (DIM == 3 ? lc[2] * PR + lc[1] : lc[1]) * TROWF + lc[0] * K;
        return true;
    };
    auto evaluate = [&](long long i, const AxisF* ax, int tbase) {  // i = output slot
        float f = 0.0f;
        float fg[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) fg[a] = 0.0f;
#pragma unroll
        for (int c = 0; c < (1 << DIM); ++c) {
            const int tv = tbase + (c & 1) * K + ((c >> 1) & 1) * TROWF + (DIM == 3 ? ((c >> 2) & 1) * PR * TROWF : 0);
            float cb[K];
            load_block<K, false>(tile + tv, cb);
            blend_corner<DIM, ORDER, GRAD>(cb, corner_geom<DIM>(s, ax, c), f, fg);
        }
        vals[i] = f;
        if (GRAD) {
#pragma unroll
            for (int a = 0; a < 3; ++a) grads[3 * i + a] = a < DIM ? fg[a] : 0.0f;
        }
    };

    // first point: load + locate while the tile is in flight
    long long i = p0 + threadIdx.x, oi = 0;
    AxisF ax[DIM];
    int tbase = 0;
    bool ok = i < p1 && prepare(i, ax, tbase, oi);
    if (!tm) cp_async_wait<0>();
    if (threadIdx.x < 32) mbar_wait(&bar, 0);
    __syncthreads();
    if (ok) evaluate(oi, ax, tbase);
    for (i += blockDim.x; i < p1; i += blockDim.x) {
        if (prepare(i, ax, tbase, oi)) evaluate(oi, ax, tbase);
    }
}

// ---- two-pass MSD partition of query points by Morton brick code ------------------
// The brick code kb (KB bits, query_brick_codes() = 2^KB) splits into a
// coarse digit hi = kb >> LO (2^HI superbricks of 2^LO Morton-consecutive
// bricks) and a fine digit lo. Pass 1 partitions the points by hi, pass 2
// partitions every superbrick's segment by lo. Each pass is a counting sort
// over tiles of kQpTile elements: a histogram kernel (shared-memory counts
// per tile), a column scan giving every (tile, digit) its output start, and a
// scatter kernel that sorts its tile by digit in shared memory and then
// writes whole digit runs (~kQpTile / 2^digit_bits records, contiguous) —
// no contended global atomics and no scattered 16-byte stores. The brick
// offsets come out of pass 2's scan. The binned query drops NaN points
// (answered NaN, status set); the sort keeps them in the origin's brick.
constexpr int kQpThreads = 512;
constexpr int kQpTile = 4096;  // elements per CTA, both passes
constexpr int kQpPer = kQpTile / kQpThreads;
constexpr int kQpRowBlocks = 32;  // column-scan row blocks

struct QpFast {
    float o[3], ih[3], lo[3], hi[3], fr[3];  // origin, 1/h, cell bounds, brick-fraction margin
};
// (host: formed once per call, read from the kernel parameters)
inline QpFast qp_fast(const DevSpec& s, int LB) {
    QpFast f{};
    for (int a = 0; a < 3; ++a) {
        f.o[a] = (float)s.origin[a];
        f.ih[a] = s.inv_hf[a];
        const double M = std::max(std::fabs(s.origin[a]), std::fabs(s.hi[a]));
        const double err = (3.0 * M * s.inv_h[a] + 2.0 * s.res[a]) * 0x1p-24;
        const float eps = (float)std::max(0x1p-10, 8.0 * err);
        f.lo[a] = eps;
        f.hi[a] = (float)(s.res[a] - 1) - eps;
        f.fr[a] = eps / (float)(1 << LB);
    }
    return f;
}

struct QpArgs {
    DevSpec s;
    const float* pts;   // n x 3
    long long n;
    int KB, LO;         // key bits, fine-digit bits
    int ntiles;         // pass-1 tiles
    int* H1;            // [ntiles][NH]: counts -> exclusive column prefixes
    int* P1;            // [kQpRowBlocks][NH] column-scan partials
    int* tot;           // [NH] digit totals
    long long* seg;     // [NH + 1] superbrick segment starts
    float4* A;          // pass-1 output
    int* cseg;          // pass-2 tile -> superbrick (-1 past the end)
    int* cfirst;        // [NH + 1] first pass-2 tile of each superbrick
    int* H2;            // [maxtiles2][NL]: counts -> output starts
    long long* off;     // [2^KB + 1] brick offsets
    float4* B;          // pass-2 output records (or null: sorted xyz + perm)
    float* out_xyz;
    long long* perm;
    float* vals;        // NaN answers (binned query), null for the sort
    float* grads;
    Status* st;
    QpFast qf;             // fp32 brick-code constants
    int* codes;            // pass 1: each input point's brick code, formed by the histogram
                           // and read back by the scatter (-1: NaN point of the binned query)
    int* codesA;           // the sort: the code of each pass-1 output record (pass 2 reads it)
    unsigned short* lpos;  // binned query: each input point's slot in its pass-1 tile's digit
                           // order (0xffff: NaN); pass-1 records then carry the brick code and
                           // pass-2 records their pass-1 position instead of the input index
    int fuse_h2;           // pass-1 scatter counts pass 2's tile histograms (H2 zeroed; no pass-2 histogram kernel)
};

// Morton brick code of a point (as point_key; a NaN coordinate counts as
// the origin's): the brick of the fp64 cell rule of locate, brick = cell >>
// LB. The cell coordinate t = (x - origin) / h is first formed in fp32; only
// a point within eps cells of a brick plane or of the domain edge takes the
// exact fp64 rule, so the partition's brick equals the query kernel's. The
// fp32 error is at most 2^-24 (3 M / h + 2 res) cells (M = the largest
// coordinate magnitude of the domain: rounding of x - origin, of the fp32
// origin, of 1/h and of the product); eps is 8 times that, at least 2^-10
// (2^-10 at 512 cells on [-1, 1]: 2.3 % of warps take the exact rule, 32 %
// at the earlier fixed 1/64).
template <int DIM, int LB>
__device__ __forceinline__ int qp_code(const DevSpec& s, const QpFast& f, float x, float y, float z) {
    const float p[3] = {x, y, z};
    unsigned int b[3] = {0, 0, 0};
    bool exact = false;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        const float tf = (p[a] - f.o[a]) * f.ih[a];
        const float tb = tf * (1.0f / (1 << LB));
        const float fl = floorf(tb), fr = tb - fl;
        // (NaN fails every comparison)
        exact |= !(tf > f.lo[a] && tf < f.hi[a] && fr > f.fr[a] && fr < 1.0f - f.fr[a]);
        b[a] = (unsigned int)fl;
    }
    if (exact) {  // near a brick plane, the domain edge, or NaN: the exact rule on every axis
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            double v = (double)p[a];
            if (isnan(v)) v = s.origin[a];
            const double lo = s.origin[a], hi = s.hi[a];
            const double c = v < lo ? lo : (v > hi ? hi : v);
            int ci = (int)floor(div_by_h(c - lo, s.h[a], s.inv_h[a]));
            ci = ci < 0 ? 0 : (ci > s.res[a] - 2 ? s.res[a] - 2 : ci);
            b[a] = (unsigned int)ci >> LB;
        }
    }
    if (DIM == 3) return (int)(spread3_10(b[0]) | (spread3_10(b[1]) << 1) | (spread3_10(b[2]) << 2));
    return (int)(spread2(b[0]) | (spread2(b[1]) << 1));
}

// Element j of this CTA's tile: pass 1 reads point j, pass 2 reads record j
// of the tile's superbrick chunk (all of a thread's loads are issued before
// the first digit is formed).
template <int DIM, int PASS>
__device__ __forceinline__ void qp_fetch(const QpArgs& A, long long e1, long long j, float4& rec, int& code,
                                         bool load_code) {
    if (j >= e1) return;
    if constexpr (PASS == 1) {
        rec = make_float4(A.pts[3 * j], A.pts[3 * j + 1], DIM == 3 ? A.pts[3 * j + 2] : 0.f, __int_as_float((int)j));
        if (load_code) code = __ldcs(A.codes + j);
    } else {
        rec = A.A[j];
        if (!A.lpos) code = A.codesA[j];
    }
}
// Its digit (NaN points of the binned query are answered in pass 1's
// histogram and get digit -1). Pass 1: the histogram (answer_nan) forms the
// code and stores it in A.codes; the scatter takes it from there (have_code).
template <int DIM, int LB, int PASS>
__device__ __forceinline__ int qp_digit(const QpArgs& A, const QpFast& qf, long long e1, long long j, float4& rec,
                                        bool answer_nan, bool have_code, int code) {
    if (j >= e1) return -1;
    if constexpr (PASS == 1) {
        if (!have_code) {
            const float x = rec.x, y = rec.y, z = rec.z;
            if (A.vals && (isnan(x) || isnan(y) || (DIM == 3 && isnan(z)))) {
                if (answer_nan) {
                    atomicMin(&A.st->nan_point, (unsigned long long)j);
                    A.vals[j] = __int_as_float(0x7fc00000);
                    if (A.grads)
                        for (int a = 0; a < 3; ++a) A.grads[3 * j + a] = __int_as_float(0x7fc00000);
                }
                code = -1;
            } else {
                code = qp_code<DIM, LB>(A.s, qf, x, y, z);
            }
            if (answer_nan && A.codes) A.codes[j] = code;
        }
        if (code < 0) return -1;
        if (A.lpos) rec.w = __int_as_float(code);
        return code >> A.LO;
    } else {
        if (A.lpos) {  // the code pass 1 formed; the record now names its pass-1 position
            code = __float_as_int(rec.w);
            rec.w = __int_as_float((int)j);
        }  // (else: fetched from A.codesA)
        return code & ((1 << A.LO) - 1);
    }
}

// Tile range of this CTA (pass 2: chunk of one superbrick; false = no tile).
template <int PASS>
__device__ __forceinline__ bool qp_tile(const QpArgs& A, long long& e0, long long& e1) {
    if constexpr (PASS == 1) {
        e0 = (long long)blockIdx.x * kQpTile;
        e1 = min(A.n, e0 + kQpTile);
        return true;
    } else {
        const int h = A.cseg[blockIdx.x];
        if (h < 0) return false;
        e0 = A.seg[h] + (long long)(blockIdx.x - A.cfirst[h]) * kQpTile;
        e1 = min(A.seg[h + 1], e0 + kQpTile);
        return true;
    }
}

template <int DIM, int LB, int PASS>
__global__ void __launch_bounds__(kQpThreads, 2) k_qp_hist(QpArgs A) {
    extern __shared__ int h[];
    const int ND = PASS == 1 ? 1 << (A.KB - A.LO) : 1 << A.LO;
    long long e0, e1;
    if (!qp_tile<PASS>(A, e0, e1)) return;
    for (int i = threadIdx.x; i < ND; i += blockDim.x) h[i] = 0;
    const QpFast& qf = A.qf;
    float4 rec[kQpPer];
    int d[kQpPer], pc[kQpPer];
#pragma unroll
    for (int k = 0; k < kQpPer; ++k)  // all loads in flight first
        qp_fetch<DIM, PASS>(A, e1, e0 + threadIdx.x + (long long)k * kQpThreads, rec[k], pc[k], false);
    (void)pc;
#pragma unroll
    for (int k = 0; k < kQpPer; ++k)
        d[k] = qp_digit<DIM, LB, PASS>(A, qf, e1, e0 + threadIdx.x + (long long)k * kQpThreads, rec[k], true, false,
                                       pc[k]);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kQpPer; ++k)
        if (d[k] >= 0) atomicAdd(&h[d[k]], 1);
    __syncthreads();
    int* row = (PASS == 1 ? A.H1 : A.H2) + (long long)blockIdx.x * ND;
    for (int i = threadIdx.x; i < ND; i += blockDim.x) row[i] = h[i];
}

// Pass-1 column scan over the tiles, in row blocks: partial sums per (row
// block, digit), then the exclusive prefixes in place and the digit totals.
__global__ void __launch_bounds__(256) k_qp_cols_partial(const int* __restrict__ H, int nrows, int nd,
                                                        int* __restrict__ P) {
    const int d = blockIdx.x * 32 + (threadIdx.x & 31), w = threadIdx.x >> 5;
    const int per = (nrows + kQpRowBlocks - 1) / kQpRowBlocks;
    const int r0 = min(nrows, (int)blockIdx.y * per), r1 = min(nrows, r0 + per);
    __shared__ int part[8][32];
    int sum = 0;
    if (d < nd)
        for (int r = r0 + w; r < r1; r += 8) sum += H[(long long)r * nd + d];
    part[w][threadIdx.x & 31] = sum;
    __syncthreads();
    if (w == 0 && d < nd) {
        int t = 0;
        for (int k = 0; k < 8; ++k) t += part[k][threadIdx.x & 31];
        P[(long long)blockIdx.y * nd + d] = t;
    }
}
__global__ void __launch_bounds__(256) k_qp_cols_final(int* __restrict__ H, int nrows, int nd, const int* __restrict__ P,
                                                      int* __restrict__ tot) {
    const int d = blockIdx.x * 32 + (threadIdx.x & 31), w = threadIdx.x >> 5;
    const int per = (nrows + kQpRowBlocks - 1) / kQpRowBlocks;
    const int r0 = min(nrows, (int)blockIdx.y * per), r1 = min(nrows, r0 + per);
    const int wper = (r1 - r0 + 7) / 8, w0 = min(r1, r0 + w * wper), w1 = min(r1, w0 + wper);
    __shared__ int part[8][32];
    int sum = 0;
    if (d < nd)
        for (int r = w0; r < w1; ++r) sum += H[(long long)r * nd + d];
    part[w][threadIdx.x & 31] = sum;
    __syncthreads();
    if (d >= nd) return;
    int base = 0;
    for (int b = 0; b < (int)blockIdx.y; ++b) base += P[(long long)b * nd + d];
    for (int k = 0; k < w; ++k) base += part[k][threadIdx.x & 31];
    // 8 rows per batch: the loads of a batch are in flight together
    for (int r = w0; r < w1; r += 8) {
        int v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = r + k < w1 ? H[(long long)(r + k) * nd + d] : 0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (r + k < w1) {
                H[(long long)(r + k) * nd + d] = base;
                base += v[k];
            }
    }
    if (blockIdx.y == kQpRowBlocks - 1 && w == 7) tot[d] = base;
}

// Superbrick segment starts (exclusive scan of the totals, one CTA) and the
// pass-2 tile map: superbrick h gets tiles [cfirst[h], cfirst[h+1]).
__global__ void __launch_bounds__(1024) k_qp_segments(const int* __restrict__ tot, int NH, long long* __restrict__ seg,
                                                      int* __restrict__ cfirst, int* __restrict__ cseg, int maxtiles) {
    __shared__ long long wsum[32];
    __shared__ int wch[32];
    __shared__ long long carry;
    __shared__ int ccarry;
    if (threadIdx.x == 0) {
        carry = 0;
        ccarry = 0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int b0 = 0; b0 < NH; b0 += 1024) {
        const int b = b0 + threadIdx.x;
        const long long t = b < NH ? tot[b] : 0;
        const int c = (int)((t + kQpTile - 1) / kQpTile);
        long long x = t;
        int y = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long xx = __shfl_up_sync(0xffffffffu, x, o);
            const int yy = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) {
                x += xx;
                y += yy;
            }
        }
        if (lane == 31) {
            wsum[warp] = x;
            wch[warp] = y;
        }
        __syncthreads();
        long long wb = 0;
        int cb = 0;
        for (int k = 0; k < warp; ++k) {
            wb += wsum[k];
            cb += wch[k];
        }
        const long long sx = carry + wb + x - t;
        const int sc = ccarry + cb + y - c;
        if (b < NH) {
            seg[b] = sx;
            cfirst[b] = sc;
            for (int k = 0; k < c && sc + k < maxtiles; ++k) cseg[sc + k] = b;
        }
        __syncthreads();
        if (threadIdx.x == 1023) {
            carry = sx + t;
            ccarry = sc + c;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        seg[NH] = carry;
        cfirst[NH] = ccarry;
    }
    __syncthreads();
    for (int k = ccarry + threadIdx.x; k < maxtiles; k += blockDim.x) cseg[k] = -1;
}

// Pass 2 per superbrick (one CTA, a thread per fine digit): prefixes of H2
// over the superbrick's tiles, the brick offsets (segment start + exclusive
// scan of the digit totals) and the per-(tile, digit) output starts.
__global__ void __launch_bounds__(1024) k_qp_scan2(QpArgs A) {
    const int hsb = blockIdx.x;
    const int NL = 1 << A.LO;
    const int ch0 = A.cfirst[hsb], ch1 = A.cfirst[hsb + 1];
    __shared__ int wsum[32];
    __shared__ long long rbase;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) rbase = A.seg[hsb];
    __syncthreads();
    for (int l0 = 0; l0 < NL; l0 += 1024) {  // NL <= 4096
        const int lo = l0 + threadIdx.x;
        int tot = 0;
        if (lo < NL)
            for (int c = ch0; c < ch1; c += 8) {  // 8 rows per batch, loads in flight together
                int v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) v[k] = c + k < ch1 ? A.H2[(long long)(c + k) * NL + lo] : 0;
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (c + k < ch1) {
                        A.H2[(long long)(c + k) * NL + lo] = tot;
                        tot += v[k];
                    }
            }
        int x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        int wb = 0;
        for (int k = 0; k < warp; ++k) wb += wsum[k];
        const long long start = rbase + wb + x - tot;
        if (lo < NL) {
            A.off[((long long)hsb << A.LO) + lo] = start;
            for (int c = ch0; c < ch1; ++c) A.H2[(long long)c * NL + lo] += (int)start;
        }
        __syncthreads();
        if (threadIdx.x == 1023) rbase = start + tot;
        __syncthreads();
    }
    if (hsb == (int)gridDim.x - 1 && threadIdx.x == 0) A.off[(long long)gridDim.x << A.LO] = A.seg[gridDim.x];
}

// Scatter: the tile's elements sorted by digit in shared memory (counting
// sort: shared-memory ranks, a block scan of the digit counts), then written
// out in that order, element j of digit d at gstart[d] + (j - lstart[d]):
// each digit's run of the tile lands contiguously.
template <int DIM, int LB, int PASS>
__global__ void __launch_bounds__(kQpThreads, 2) k_qp_scatter(QpArgs A) {
    extern __shared__ __align__(16) unsigned char qsm[];
    const int ND = PASS == 1 ? 1 << (A.KB - A.LO) : 1 << A.LO;
    float4* recs = reinterpret_cast<float4*>(qsm);                            // [kQpTile]
    unsigned short* dig = reinterpret_cast<unsigned short*>(recs + kQpTile);  // [kQpTile]
    int* cnt = reinterpret_cast<int*>(dig + kQpTile);                         // [ND] counts -> local starts
    int* gst = cnt + ND;                                                       // [ND] global starts
    int* scode = gst + ND;        // the sort's pass 1: [kQpTile] codes in digit order
    int* sin = scode + kQpTile;   // ... and in input order
    __shared__ int wsum[kQpThreads / 32];
    __shared__ int valid;
    long long e0, e1;
    if (!qp_tile<PASS>(A, e0, e1)) return;
    const int* row = (PASS == 1 ? A.H1 : A.H2) + (long long)blockIdx.x * ND;
    for (int i = threadIdx.x; i < ND; i += blockDim.x) {
        cnt[i] = 0;
        gst[i] = PASS == 1 ? (int)A.seg[i] + row[i] : row[i];
    }
    const QpFast& qf = A.qf;
    float4 rec[kQpPer];
    int d[kQpPer], rk[kQpPer], cd[kQpPer];
    constexpr bool have = PASS == 1;  // (launch_qpart always provides A.codes)
#pragma unroll
    for (int k = 0; k < kQpPer; ++k)
        qp_fetch<DIM, PASS>(A, e1, e0 + threadIdx.x + (long long)k * kQpThreads, rec[k], cd[k], have);
#pragma unroll
    for (int k = 0; k < kQpPer; ++k) {
        d[k] = qp_digit<DIM, LB, PASS>(A, qf, e1, e0 + threadIdx.x + (long long)k * kQpThreads, rec[k], false, have,
                                       cd[k]);
        if (PASS == 1 && !A.lpos) sin[threadIdx.x + k * kQpThreads] = cd[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kQpPer; ++k) rk[k] = d[k] >= 0 ? atomicAdd(&cnt[d[k]], 1) : 0;
    __syncthreads();
    // exclusive scan of cnt (ND <= 4096 digits, kQpThreads threads)
    const int per = (ND + kQpThreads - 1) / kQpThreads;
    const int i0 = threadIdx.x * per;
    int loc = 0;
    for (int i = i0; i < min(ND, i0 + per); ++i) loc += cnt[i];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    int run = x - loc;
    for (int k = 0; k < warp; ++k) run += wsum[k];
    for (int i = i0; i < min(ND, i0 + per); ++i) {
        const int c = cnt[i];
        cnt[i] = run;
        run += c;
    }
    if (i0 < ND && i0 + per >= ND) valid = run;  // the owner of the last digit: the tile's element count
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kQpPer; ++k) {
        const int j = d[k] >= 0 ? cnt[d[k]] + rk[k] : 0xffff;
        if (d[k] >= 0) {
            recs[j] = rec[k];
            dig[j] = (unsigned short)d[k];
            if (PASS == 1 && !A.lpos) scode[j] = sin[threadIdx.x + k * kQpThreads];
        }
        if (PASS == 1 && A.lpos) {
            const long long i = e0 + threadIdx.x + (long long)k * kQpThreads;
            if (i < e1) A.lpos[i] = (unsigned short)j;
        }
    }
    __syncthreads();
    // the tile's elements in digit order (NaN points of the binned query are
    // not among them)
    for (int j = threadIdx.x; j < valid; j += blockDim.x) {
        const int dj = dig[j];
        const int pos = gst[dj] + (j - cnt[dj]);
        const float4 q = recs[j];
        if (PASS == 1 && A.fuse_h2) {
            // pass 2 tiles each superbrick's segment in kQpTile chunks from
            // cfirst[dj] (qp_tile<2>): this record's tile and low digit
            const int code = A.lpos ? __float_as_int(q.w) : scode[j];
            const int t2 = __ldg(A.cfirst + dj) + (int)((pos - __ldg(A.seg + dj)) / kQpTile);
            atomicAdd(A.H2 + (long long)t2 * (1 << A.LO) + (code & ((1 << A.LO) - 1)), 1);
        }
        if (PASS == 1 || A.B) {
            (PASS == 1 ? A.A : A.B)[pos] = q;
            if (PASS == 1 && !A.lpos) A.codesA[pos] = scode[j];
        } else {
            A.out_xyz[3 * (long long)pos] = q.x;
            A.out_xyz[3 * (long long)pos + 1] = q.y;
            A.out_xyz[3 * (long long)pos + 2] = q.z;
            if (A.perm) A.perm[pos] = (long long)(unsigned int)__float_as_int(q.w);
        }
    }
}

// Sort only: each brick's points in Morton cell order (warp per brick, in
// chunks of 256 staged in shared memory for a coalesced write-out: shared-memory cell counts, ranks, a warp scan), written as
// the sorted coordinates + source indices. Consecutive points of a brick then
// share corner blocks, which the brick-tile query reads with fewer
// shared-memory bank conflicts. The cell comes from fp32 coordinates: it only
// orders points inside their (exactly binned) brick.
template <int DIM, int LB>
__global__ void __launch_bounds__(128, 6) k_qp_cellsort(QpArgs A, const float4* __restrict__ C, int nbricks) {
    constexpr int NCELLB = 1 << (DIM * LB);
    constexpr int PER = NCELLB / 32;
    constexpr int CHK = 256;  // records per warp pass (8 per lane)
    __shared__ int cnt[4][NCELLB];
    __shared__ float4 stage[4][CHK];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * 4 + w;
    if (b >= nbricks) return;
    const long long p0 = A.off[b], p1 = A.off[b + 1];
    int* ct = cnt[w];
    float4* st = stage[w];
    for (long long c0 = p0; c0 < p1; c0 += CHK) {
        const int m = (int)min((long long)CHK, p1 - c0);
#pragma unroll
        for (int k = 0; k < PER; ++k) ct[lane * PER + k] = 0;
        __syncwarp();
        float4 rec[CHK / 32];
        int cc[CHK / 32], rk[CHK / 32];
#pragma unroll
        for (int k = 0; k < CHK / 32; ++k)  // all loads in flight before the first use
            if (lane + 32 * k < m) rec[k] = __ldcs(C + c0 + lane + 32 * k);
#pragma unroll
        for (int k = 0; k < CHK / 32; ++k) {
            const int j = lane + 32 * k;
            cc[k] = -1;
            if (j < m) {
                const float p[3] = {rec[k].x, rec[k].y, rec[k].z};
                unsigned int l[3] = {0, 0, 0};
#pragma unroll
                for (int a = 0; a < DIM; ++a) {
                    const float tf = (p[a] - (float)A.s.origin[a]) * A.s.inv_hf[a];
                    int ci = tf >= 0.0f ? (int)tf : 0;  // NaN -> 0
                    ci = min(ci, A.s.res[a] - 2);
                    l[a] = (unsigned int)ci & ((1u << LB) - 1u);
                }
                cc[k] = DIM == 3 ? (int)(spread3_10(l[0]) | (spread3_10(l[1]) << 1) | (spread3_10(l[2]) << 2))
                                 : (int)(spread2(l[0]) | (spread2(l[1]) << 1));
                rk[k] = atomicAdd(&ct[cc[k]], 1);
            }
        }
        __syncwarp();
        int loc = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) loc += ct[lane * PER + k];
        int x = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        int run = x - loc;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int v = ct[lane * PER + k];
            ct[lane * PER + k] = run;
            run += v;
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < CHK / 32; ++k)
            if (cc[k] >= 0) st[ct[cc[k]] + rk[k]] = rec[k];
        __syncwarp();
        // coalesced write-out of the chunk in cell order
        for (int j = lane; j < m; j += 32) {
            const float4 q = st[j];
            const long long pos = c0 + j;
            A.out_xyz[3 * pos] = q.x;
            A.out_xyz[3 * pos + 1] = q.y;
            A.out_xyz[3 * pos + 2] = q.z;
            if (A.perm) A.perm[pos] = (long long)(unsigned int)__float_as_int(q.w);
        }
        __syncwarp();
    }
}

// Runs both passes. B != null: records (x, y, z, index) grouped by brick;
// else sorted xyz (+ perm). off: 2^KB + 1 brick offsets.
// TGCU_QP_FUSE_H2=0/1: pass 2's tile histograms from the pass-1 scatter
// (L2 reductions) instead of a histogram pass over the pass-1 records.
static int qp_fuse_h2() {
    static const int on = [] {
        const char* e = std::getenv("TGCU_QP_FUSE_H2");
        return e ? std::atoi(e) : 0;
    }();
    return on;
}

void launch_qpart(Grid& g, const float* pts, int64_t n, float4* B, float* out_xyz, int64_t* perm,
                  long long* off, float* vals, float* grads, cudaStream_t s, unsigned short* lpos,
                  const std::function<void(const QpArgs&)>& after) {
    require(n < (1LL << 31), "query partition: more than 2^31 points per call");
    const int64_t codes = query_brick_codes(g);
    int KB = 0;
    while ((1LL << KB) < codes) ++KB;
    QpArgs A{};
    A.s = g.ds;
    A.pts = pts;
    A.n = n;
    A.KB = KB;
    A.LO = std::min(12, std::max((KB + 1) / 2, KB - 12));
    require(KB - A.LO <= 12, "query partition: " + std::to_string(KB) + " brick-code bits exceed two 12-bit passes");
    const int NH = 1 << (KB - A.LO), NL = 1 << A.LO;
    A.ntiles = (int)((n + kQpTile - 1) / kQpTile);
    const int maxtiles = A.ntiles + NH;
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t bH1 = al(sizeof(int) * (size_t)A.ntiles * NH), bP1 = al(sizeof(int) * kQpRowBlocks * NH),
                 bTot = al(sizeof(int) * NH), bSeg = al(sizeof(long long) * (NH + 1)), bCf = al(sizeof(int) * (NH + 1)),
                 bCs = al(sizeof(int) * maxtiles), bH2 = al(sizeof(int) * (size_t)maxtiles * NL),
                 bA = al(sizeof(float4) * (size_t)std::max<int64_t>(n, 1)),
                 bCode = al(sizeof(int) * (size_t)std::max<int64_t>(n, 1)), bCodeA = lpos ? 0 : bCode;
    char* q = nullptr;
    TGCU_CUDA(cudaMallocAsync(&q, bH1 + bP1 + bTot + bSeg + bCf + bCs + bH2 + bA + bCode + bCodeA, s));
    char* const scratch = q;
    A.H1 = reinterpret_cast<int*>(q); q += bH1;
    A.P1 = reinterpret_cast<int*>(q); q += bP1;
    A.tot = reinterpret_cast<int*>(q); q += bTot;
    A.seg = reinterpret_cast<long long*>(q); q += bSeg;
    A.cfirst = reinterpret_cast<int*>(q); q += bCf;
    A.cseg = reinterpret_cast<int*>(q); q += bCs;
    A.H2 = reinterpret_cast<int*>(q); q += bH2;
    A.A = reinterpret_cast<float4*>(q); q += bA;
    A.codes = reinterpret_cast<int*>(q); q += bCode;
    A.codesA = lpos ? nullptr : reinterpret_cast<int*>(q);
    A.off = off;
    // the sort writes pass 2's records to C, then orders each brick by cell
    float4* C = nullptr;
    if (!B) TGCU_CUDA(cudaMallocAsync(&C, sizeof(float4) * (size_t)std::max<int64_t>(n, 1), s));
    A.B = B ? B : C;
    A.out_xyz = out_xyz;
    A.perm = reinterpret_cast<long long*>(perm);
    A.vals = vals;
    A.grads = grads;
    A.st = g.st;
    A.lpos = lpos;
    A.qf = qp_fast(g.ds, g.spec.dim == 3 ? 3 : 4);
    A.fuse_h2 = qp_fuse_h2();
    const size_t hs1 = sizeof(int) * NH, hs2 = sizeof(int) * NL;
    const size_t ss1 = (sizeof(float4) + 2) * kQpTile + 2 * hs1 + (lpos ? 0 : 2 * sizeof(int) * kQpTile),
                 ss2 = (sizeof(float4) + 2) * kQpTile + 2 * hs2;
    auto run = [&](auto hist1, auto scatter1, auto hist2, auto scatter2) {
        TGCU_CUDA(cudaFuncSetAttribute(scatter1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ss1));
        TGCU_CUDA(cudaFuncSetAttribute(scatter2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ss2));
        hist1<<<A.ntiles, kQpThreads, hs1, s>>>(A);
        k_qp_cols_partial<<<dim3((NH + 31) / 32, kQpRowBlocks), 256, 0, s>>>(A.H1, A.ntiles, NH, A.P1);
        k_qp_cols_final<<<dim3((NH + 31) / 32, kQpRowBlocks), 256, 0, s>>>(A.H1, A.ntiles, NH, A.P1, A.tot);
        k_qp_segments<<<1, 1024, 0, s>>>(A.tot, NH, A.seg, A.cfirst, A.cseg, maxtiles);
        if (A.fuse_h2) TGCU_CUDA(cudaMemsetAsync(A.H2, 0, sizeof(int) * (size_t)maxtiles * NL, s));
        scatter1<<<A.ntiles, kQpThreads, ss1, s>>>(A);
        if (!A.fuse_h2) hist2<<<maxtiles, kQpThreads, hs2, s>>>(A);
        k_qp_scan2<<<NH, 1024, 0, s>>>(A);
        scatter2<<<maxtiles, kQpThreads, ss2, s>>>(A);
    };
    if (g.spec.dim == 3)
        run(k_qp_hist<3, 3, 1>, k_qp_scatter<3, 3, 1>, k_qp_hist<3, 3, 2>, k_qp_scatter<3, 3, 2>);
    else
        run(k_qp_hist<2, 4, 1>, k_qp_scatter<2, 4, 1>, k_qp_hist<2, 4, 2>, k_qp_scatter<2, 4, 2>);
    count_launch(A.fuse_h2 ? 7 : 8);
    if (C) {
        const int nbr = (int)codes;
        if (g.spec.dim == 3) k_qp_cellsort<3, 3><<<(nbr + 3) / 4, 128, 0, s>>>(A, C, nbr);
        else k_qp_cellsort<2, 4><<<(nbr + 3) / 4, 128, 0, s>>>(A, C, nbr);
        count_launch();
        TGCU_CUDA(cudaFreeAsync(C, s));
    }
    if (after) after(A);  // still holding the pass-1 tables
    TGCU_CUDA(cudaFreeAsync(scratch, s));
    TGCU_CUDA(cudaGetLastError());
}

// Query tile tensor maps (box (B+1) vertices padded to 16 bytes x (B+1) [x (B+1)]).
static bool ensure_query_tmaps(Grid& g, unsigned box_x, unsigned box_y, unsigned T) {
    if (g.tmq_state == 0) {
        g.tmq_state = -1;
        if (((int64_t)g.ds.res[0] * g.K * 4) % 16 == 0 && box_x <= 256 && !g.slab) {
            bool ok = encode_grid_map(&g.tm_query[0], g, g.p[0], box_x, box_y, T);
            if (g.p[1]) ok = ok && encode_grid_map(&g.tm_query[1], g, g.p[1], box_x, box_y, T);
            if (ok) g.tmq_state = g.p[1] ? 2 : 1;  // maps built for 1 or 2 buffers
        }
    }
    if (g.tmq_state == 1 && g.p[1]) {  // optimiser buffers appeared since
        if (!encode_grid_map(&g.tm_query[1], g, g.p[1], box_x, box_y, T)) return false;
        g.tmq_state = 2;
    }
    return g.tmq_state >= 1 && (g.cur == 0 || g.tmq_state == 2);
}

template <int SRC>
static void launch_brick_query(Grid& g, const QuerySrc& Q, float* vals, float* grads, cudaStream_t s) {
    TGCU_DISPATCH(g.spec.dim, g.spec.order, {
        constexpr int LB = brick_log2<DIM>();
        constexpr int B = 1 << LB;
        constexpr int K = KOf<DIM, ORDER>::value;
        constexpr int T = B + 1;
        constexpr int TROWF = query_trowf<DIM, K, T>();
        constexpr int PR = query_plane_rows<DIM, K, T>();
        const size_t smem = sizeof(float) * (DIM == 3 ? T * PR : T) * TROWF;
        const bool use_tm = ensure_query_tmaps(g, TROWF, PR, T);
        CUtensorMap map{};
        if (use_tm) map = g.tm_query[g.cur];
        dim3 grid(1, 1, 1);
        for (int a = 0; a < DIM; ++a) (&grid.x)[a] = (unsigned)((g.spec.res[a] - 1 + B - 1) / B);
        if (Q.morton) grid = dim3((unsigned)query_brick_codes(g), 1, 1);
        auto kern = grads ? k_eval_brick<DIM, ORDER, true, LB, SRC> : k_eval_brick<DIM, ORDER, false, LB, SRC>;
        TGCU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<grid, 256, smem, s>>>(map, use_tm ? 1 : 0, g.ds, g.p[g.cur], Q, vals, grads, g.st);
    });
    count_launch();
}

// Binned query outputs back to the caller's order. The query kernel writes
// each record's value at its pass-1 position (pass-2 records carry it): a
// brick's points come from one superbrick segment and the kernel walks the
// bricks in Morton order, so these stores stay in an L2-resident window.
// Then pass 1 runs backwards, one CTA per input tile: the tile's digit runs
// (start seg[d] + H1[t][d], length H1[t+1][d] - H1[t][d]) are read into
// shared memory in digit order, and point i takes slot lpos[i]. Every global
// access is a contiguous run. (Storing to the caller's slot straight from the
// query kernel is a 4-byte store into an evicted sector: a 32-byte DRAM fill
// + write-back per point, 4.2 GB for 2^26 points.)
template <bool GRAD>
__global__ void __launch_bounds__(kQpThreads) k_qp_unpart(QpArgs A, const float* __restrict__ rv,
                                                          const float* __restrict__ rg) {
    extern __shared__ __align__(16) unsigned char qsm[];
    const int ND = 1 << (A.KB - A.LO);
    float* sv = reinterpret_cast<float*>(qsm);                      // [kQpTile]
    float* sg = sv + kQpTile;                                        // GRAD: [3 kQpTile]
    int* L = reinterpret_cast<int*>(sg + (GRAD ? 3 * kQpTile : 0));  // [ND + 1] local digit starts
    int* gs = L + ND + 1;                                            // [ND] global run starts
    unsigned short* own = reinterpret_cast<unsigned short*>(gs + ND);  // [kQpTile] digit of each slot
    __shared__ int wsum[kQpThreads / 32];
    const long long e0 = (long long)blockIdx.x * kQpTile, e1 = min(A.n, e0 + kQpTile);
    // this tile's slots in input order first (independent of the tables)
    int lp[kQpPer];
#pragma unroll
    for (int k = 0; k < kQpPer; ++k) {
        const long long i = e0 + threadIdx.x + (long long)k * kQpThreads;
        lp[k] = i < e1 ? (int)__ldcs(A.lpos + i) : 0xffff;
    }
    const int* row = A.H1 + (long long)blockIdx.x * ND;
    const int* nxt = (int)blockIdx.x + 1 < A.ntiles ? row + ND : A.tot;
    const int per = (ND + kQpThreads - 1) / kQpThreads, i0 = threadIdx.x * per;
    int loc = 0;
    for (int i = i0; i < min(ND, i0 + per); ++i) {
        const int r = row[i], c = nxt[i] - r;
        L[i] = c;
        gs[i] = (int)A.seg[i] + r;
        loc += c;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    int run = x - loc;
    for (int k = 0; k < warp; ++k) run += wsum[k];
    for (int i = i0; i < min(ND, i0 + per); ++i) {
        const int c = L[i];
        L[i] = run;
        for (int r = 0; r < c; ++r) own[run + r] = (unsigned short)i;
        run += c;
    }
    if (i0 < ND && i0 + per >= ND) L[ND] = run;
    __syncthreads();
    const int valid = L[ND];
    // the runs, in digit order, into shared memory (loads batched per thread)
    float v[kQpPer], gv[GRAD ? 3 * kQpPer : 1];
#pragma unroll
    for (int k = 0; k < kQpPer; ++k) {
        const int j = threadIdx.x + k * kQpThreads;
        if (j < valid) {
            const int d = own[j];
            const long long src = gs[d] + (j - L[d]);
            v[k] = __ldcs(rv + src);
            if (GRAD) {
#pragma unroll
                for (int a = 0; a < 3; ++a) gv[3 * k + a] = __ldcs(rg + 3 * src + a);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < kQpPer; ++k) {
        const int j = threadIdx.x + k * kQpThreads;
        if (j < valid) {
            sv[j] = v[k];
            if (GRAD) {
#pragma unroll
                for (int a = 0; a < 3; ++a) sg[3 * j + a] = gv[3 * k + a];
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kQpPer; ++k) {
        const long long i = e0 + threadIdx.x + (long long)k * kQpThreads;
        if (lp[k] == 0xffff) continue;  // past the end, or a NaN point (answered by the partition)
        A.vals[i] = sv[lp[k]];
        if (GRAD) {
#pragma unroll
            for (int a = 0; a < 3; ++a) A.grads[3 * i + a] = sg[3 * lp[k] + a];
        }
    }
}

// Morton-order launch of the binned brick query when the code space is not
// much larger than the brick grid (TGCU_QUERY_MORTON=0: brick-coordinate
// order): keeps its pass-1-position stores in a narrow window.
static int query_morton(const Grid& g) {
    static const int env = [] {
        const char* e = std::getenv("TGCU_QUERY_MORTON");
        return e ? std::atoi(e) : 1;
    }();
    const int B = g.spec.dim == 3 ? 8 : 16;
    int64_t nb = 1;
    for (int a = 0; a < g.spec.dim; ++a) nb *= (g.spec.res[a] - 1 + B - 1) / B;
    return env != 0 && query_brick_codes(g) <= 2 * nb ? 1 : 0;
}

void launch_eval_binned(Grid& g, const float* pts, int64_t n, float* vals, float* grads, cudaStream_t s) {
    if (n <= 0) return;
    const int64_t codes = query_brick_codes(g);
    const size_t nn = (size_t)n;
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    // off | records | lpos | values (+ gradients) at pass-1 positions
    const size_t b_off = al(sizeof(long long) * (codes + 1)), b_rec = sizeof(float4) * nn,
                 b_lp = al(sizeof(unsigned short) * nn), b_out = sizeof(float) * nn * (grads ? 4 : 1);
    char* q = nullptr;
    TGCU_CUDA(cudaMallocAsync(&q, b_off + b_rec + b_lp + b_out, s));
    long long* off = reinterpret_cast<long long*>(q);
    float4* binned = reinterpret_cast<float4*>(q + b_off);
    unsigned short* lpos = reinterpret_cast<unsigned short*>(q + b_off + b_rec);
    float* rv = reinterpret_cast<float*>(q + b_off + b_rec + b_lp);
    float* rg = grads ? rv + nn : nullptr;
    launch_qpart(g, pts, n, binned, nullptr, nullptr, off, vals, grads, s, lpos, [&](const QpArgs& A) {
        QuerySrc Q;
        Q.pts = reinterpret_cast<const float*>(binned);
        Q.off = off;
        Q.morton = query_morton(g);
        launch_brick_query<1>(g, Q, rv, rg, s);
        const int ND = 1 << (A.KB - A.LO);
        const size_t smem = sizeof(float) * kQpTile * (grads ? 4 : 1) + sizeof(int) * (2 * ND + 1) +
                            sizeof(unsigned short) * kQpTile;
        auto kern = grads ? k_qp_unpart<true> : k_qp_unpart<false>;
        TGCU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<A.ntiles, kQpThreads, smem, s>>>(A, rv, rg);
        count_launch();
    });
    TGCU_CUDA(cudaFreeAsync(q, s));
    TGCU_CUDA(cudaGetLastError());
}

void launch_eval_sorted(Grid& g, const float* pts, int64_t n, const int64_t* offsets, float* vals, float* grads,
                        cudaStream_t s) {
    if (n <= 0) return;
    const int64_t codes = query_brick_codes(g);
    long long* tmp = nullptr;
    if (!offsets) {  // points sorted but no offsets given: one boundary pass
        TGCU_CUDA(cudaMallocAsync(&tmp, sizeof(long long) * (codes + 1), s));
        launch_brick_offsets<unsigned int>(g, nullptr, pts, n, reinterpret_cast<int64_t*>(tmp), s);
        offsets = reinterpret_cast<const int64_t*>(tmp);
    }
    const long long* off = reinterpret_cast<const long long*>(offsets);
    QuerySrc Q;
    Q.pts = pts;
    Q.off = off;  // (brick-coordinate order: measured 2 % faster than Morton order here)
    launch_brick_query<0>(g, Q, vals, grads, s);
    if (tmp) TGCU_CUDA(cudaFreeAsync(tmp, s));
    TGCU_CUDA(cudaGetLastError());
}

// ---- lattice query on the brick tiles -------------------------------------------
// Lattice index range of every brick coordinate along each axis: the cells of
// a lattice axis are non-decreasing, so the indices of one brick are a run.
__global__ void k_lattice_ranges(const int* __restrict__ cell, int3 n, int dim, int lb, int nb0, int nb1,
                                 int2* __restrict__ rng) {
    const int na = n.x + (dim > 1 ? n.y : 0) + (dim > 2 ? n.z : 0);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < na; j += gridDim.x * blockDim.x) {
        const int a = j < n.x ? 0 : (j < n.x + n.y ? 1 : 2);
        const int first = a == 0 ? 0 : (a == 1 ? n.x : n.x + n.y);
        const int len = a == 0 ? n.x : (a == 1 ? n.y : n.z);
        const int i = j - first;
        const int roff = a == 0 ? 0 : (a == 1 ? nb0 : nb0 + nb1);
        const int b = cell[j] >> lb;
        if (i == 0 || (cell[j - 1] >> lb) != b) rng[roff + b].x = i;
        if (i == len - 1 || (cell[j + 1] >> lb) != b) rng[roff + b].y = i + 1;
    }
}

bool launch_eval_lattice_brick(Grid& g, const float4* fac, const int* cell, int3 n, float* vals, cudaStream_t s) {
    const int dim = g.spec.dim;
    const int LB = dim == 3 ? 3 : 4;
    const int B = 1 << LB;
    int nb[3] = {1, 1, 1};
    int64_t bricks = 1;
    for (int a = 0; a < dim; ++a) {
        nb[a] = (g.spec.res[a] - 1 + B - 1) / B;
        bricks *= nb[a];
    }
    const int64_t pts = (int64_t)n.x * n.y * n.z;
    // a tile per brick pays off when the bricks hold enough lattice points
    if (pts < bricks * 128 || pts >= (1LL << 31)) return false;
    const int nrng = nb[0] + nb[1] + nb[2];
    int2* rng = nullptr;
    TGCU_CUDA(cudaMallocAsync(&rng, sizeof(int2) * nrng, s));
    TGCU_CUDA(cudaMemsetAsync(rng, 0, sizeof(int2) * nrng, s));
    const int na = n.x + (dim > 1 ? n.y : 0) + (dim > 2 ? n.z : 0);
    k_lattice_ranges<<<grid_blocks(na, 256), 256, 0, s>>>(cell, n, dim, LB, nb[0], nb[1], rng);
    count_launch();
    QuerySrc Q;
    Q.fac = fac;
    Q.cell = cell;
    Q.rng = rng;
    Q.n = n;
    for (int a = 0; a < 3; ++a) Q.nb[a] = nb[a];
    launch_brick_query<2>(g, Q, vals, nullptr, s);
    TGCU_CUDA(cudaFreeAsync(rng, s));
    TGCU_CUDA(cudaGetLastError());
    return true;
}

}  // namespace tgcu
