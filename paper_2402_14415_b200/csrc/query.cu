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
#include <cub/cub.cuh>

#include "dispatch.cuh"
#include "tg_internal.h"

namespace tgcu {

template <int DIM, int ORDER, bool GRAD>
__global__ void __launch_bounds__(256) k_eval_direct(DevSpec s, const float* __restrict__ coeffs,
                                                     const float* __restrict__ pts, long long n,
                                                     float* __restrict__ vals, float* __restrict__ grads,
                                                     Status* st) {
    constexpr int K = KOf<DIM, ORDER>::value;
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
        // Issue every corner's loads before any math (8 independent gathers).
        float cb[1 << DIM][K];
#pragma unroll
        for (int c = 0; c < (1 << DIM); ++c) {
            const long long vid = base + (c & 1) + ((c >> 1) & 1) * s.sy + (DIM == 3 ? ((c >> 2) & 1) * s.sz : 0);
            load_block<K, true>(coeffs + vid * K, cb[c]);
        }
        float f = 0.0f;
        float fg[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) fg[a] = 0.0f;
#pragma unroll
        for (int c = 0; c < (1 << DIM); ++c) {
            const Corner<DIM> g = corner_geom<DIM>(s, ax, c);
            blend_corner<DIM, ORDER, GRAD>(cb[c], g, f, fg);
        }
        vals[i] = f;
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

template <int DIM, int LB>
__global__ void k_point_keys(DevSpec s, const float* __restrict__ pts, long long n,
                             unsigned long long* __restrict__ keys, long long* __restrict__ idx) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        keys[i] = point_key<DIM, LB>(s, pts + 3 * i, nullptr);
        idx[i] = i;
    }
}

__global__ void k_gather_points(const float* __restrict__ pts, const long long* __restrict__ idx, long long n,
                                float* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long j = idx[i];
        out[3 * i] = pts[3 * j];
        out[3 * i + 1] = pts[3 * j + 1];
        out[3 * i + 2] = pts[3 * j + 2];
    }
}

template <int DIM>
constexpr int brick_log2() { return DIM == 3 ? 3 : 4; }

void launch_sort_points(Grid& g, const float* pts, int64_t n, float* out, int64_t* perm, cudaStream_t s) {
    if (n <= 0) return;
    unsigned long long *keys = nullptr, *keys_out = nullptr;
    long long *idx = nullptr, *idx_out = nullptr;
    void* temp = nullptr;
    size_t temp_bytes = 0;
    TGCU_CUDA(cudaMallocAsync(&keys, n * 8, s));
    TGCU_CUDA(cudaMallocAsync(&keys_out, n * 8, s));
    TGCU_CUDA(cudaMallocAsync(&idx, n * 8, s));
    idx_out = reinterpret_cast<long long*>(perm);
    bool own_perm = false;
    if (!idx_out) {
        TGCU_CUDA(cudaMallocAsync(&idx_out, n * 8, s));
        own_perm = true;
    }
    const int blocks = grid_blocks(n, 256, 148 * 32);
    int end_bit = 0;
    if (g.spec.dim == 3) {
        k_point_keys<3, 3><<<blocks, 256, 0, s>>>(g.ds, pts, n, keys, idx);
        int maxc = 1;
        for (int a = 0; a < 3; ++a) maxc = std::max(maxc, g.spec.res[a] - 2);
        int bits = 1;
        while ((1 << bits) <= maxc) ++bits;
        end_bit = 3 * bits;
    } else {
        k_point_keys<2, 4><<<blocks, 256, 0, s>>>(g.ds, pts, n, keys, idx);
        int maxc = 1;
        for (int a = 0; a < 2; ++a) maxc = std::max(maxc, g.spec.res[a] - 2);
        int bits = 1;
        while ((1 << bits) <= maxc) ++bits;
        end_bit = 2 * bits;
    }
    count_launch();
    TGCU_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys, keys_out, idx, idx_out, (int64_t)n, 0,
                                              end_bit, s));
    TGCU_CUDA(cudaMallocAsync(&temp, temp_bytes, s));
    TGCU_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, keys_out, idx, idx_out, (int64_t)n, 0,
                                              end_bit, s));
    k_gather_points<<<blocks, 256, 0, s>>>(pts, idx_out, n, out);
    count_launch();
    TGCU_CUDA(cudaFreeAsync(temp, s));
    TGCU_CUDA(cudaFreeAsync(keys, s));
    TGCU_CUDA(cudaFreeAsync(keys_out, s));
    TGCU_CUDA(cudaFreeAsync(idx, s));
    if (own_perm) TGCU_CUDA(cudaFreeAsync(idx_out, s));
    TGCU_CUDA(cudaGetLastError());
}

// One CTA per brick (in Morton order = blockIdx.x). Tile: (B+1)^DIM vertices.
template <int DIM, int ORDER, bool GRAD, int LB>
__global__ void __launch_bounds__(256) k_eval_brick(DevSpec s, const float* __restrict__ coeffs,
                                                    const float* __restrict__ pts, long long n,
                                                    float* __restrict__ vals, float* __restrict__ grads,
                                                    Status* st, int nbx, int nby, int nbz) {
    constexpr int K = KOf<DIM, ORDER>::value;
    constexpr int B = 1 << LB;
    constexpr int T = B + 1;                        // tile edge in vertices
    constexpr int TV = DIM == 3 ? T * T * T : T * T;  // tile vertices
    extern __shared__ __align__(16) float tile[];   // TV * K

    // Decode this brick's coordinates from the Morton index.
    const unsigned int code = blockIdx.x;
    unsigned int b[3] = {0, 0, 0};
    for (int bit = 0; bit < 21; ++bit) {
#pragma unroll
        for (int a = 0; a < DIM; ++a) b[a] |= ((code >> (bit * DIM + a)) & 1u) << bit;
    }
    if ((int)b[0] >= nbx || (int)b[1] >= nby || (DIM == 3 && (int)b[2] >= nbz)) return;

    // Binary search this brick's [lo, hi) range in the brick-sorted points.
    __shared__ long long range[2];
    if (threadIdx.x < 2) {
        const unsigned int target = code + threadIdx.x;
        long long lo = 0, hi = n;
        while (lo < hi) {
            const long long mid = (lo + hi) >> 1;
            unsigned int kb;
            point_key<DIM, LB>(s, pts + 3 * mid, &kb);
            if (kb < target) lo = mid + 1; else hi = mid;
        }
        range[threadIdx.x] = lo;
    }
    __syncthreads();
    const long long p0 = range[0], p1 = range[1];
    if (p0 >= p1) return;

    // Stage the vertex tile: rows of T vertices x K coefficients are contiguous.
    const int ox = b[0] * B, oy = b[1] * B, oz = DIM == 3 ? b[2] * B : 0;
    constexpr int ROW = T * K;
    const int rows = DIM == 3 ? T * T : T;
    for (int e = threadIdx.x; e < rows * ROW; e += blockDim.x) {
        const int r = e / ROW, q = e - r * ROW;
        const int tx = q / K, ch = q - tx * K;
        const int ty = r % T, tz = r / T;
        const int vx = ox + tx, vy = oy + ty, vz = oz + tz;
        float val = 0.0f;
        if (vx < s.res[0] && vy < s.res[1] && (DIM == 2 || vz < s.res[2]))
            val = __ldg(coeffs + ((long long)vz * s.sz + (long long)vy * s.sy + vx) * K + ch);
        tile[e] = val;
    }
    __syncthreads();

    for (long long i = p0 + threadIdx.x; i < p1; i += blockDim.x) {
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
        int lc[3] = {0, 0, 0};
        const int o3[3] = {ox, oy, oz};
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            double local;
            const int c = locate_axis(s, a, x[a], local);
            ax[a] = axis_factors(s, a, local);
            lc[a] = c - o3[a];
        }
        const int tbase = DIM == 3 ? (lc[2] * T + lc[1]) * T + lc[0] : lc[1] * T + lc[0];
        float cb[1 << DIM][K];
#pragma unroll
        for (int c = 0; c < (1 << DIM); ++c) {
            const int tv = tbase + (c & 1) + ((c >> 1) & 1) * T + (DIM == 3 ? ((c >> 2) & 1) * T * T : 0);
            load_block<K, false>(tile + tv * K, cb[c]);
        }
        float f = 0.0f;
        float fg[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) fg[a] = 0.0f;
#pragma unroll
        for (int c = 0; c < (1 << DIM); ++c) {
            const Corner<DIM> g = corner_geom<DIM>(s, ax, c);
            blend_corner<DIM, ORDER, GRAD>(cb[c], g, f, fg);
        }
        vals[i] = f;
        if (GRAD) {
#pragma unroll
            for (int a = 0; a < 3; ++a) grads[3 * i + a] = a < DIM ? fg[a] : 0.0f;
        }
    }
    (void)TV;
}

void launch_eval_sorted(Grid& g, const float* pts, int64_t n, float* vals, float* grads, cudaStream_t s) {
    if (n <= 0) return;
    TGCU_DISPATCH(g.spec.dim, g.spec.order, {
        constexpr int LB = brick_log2<DIM>();
        constexpr int B = 1 << LB;
        constexpr int K = KOf<DIM, ORDER>::value;
        constexpr int T = B + 1;
        constexpr int TV = DIM == 3 ? T * T * T : T * T;
        const size_t smem = sizeof(float) * TV * K;
        int nbv[3] = {1, 1, 1};
        unsigned int pow2 = 1;
        for (int a = 0; a < DIM; ++a) {
            nbv[a] = (g.spec.res[a] - 1 + B - 1) / B;  // bricks of cells
            while (pow2 < (unsigned)nbv[a]) pow2 <<= 1;
        }
        unsigned long long blocks = 1;
        for (int a = 0; a < DIM; ++a) blocks *= pow2;
        auto kern = grads ? k_eval_brick<DIM, ORDER, true, LB> : k_eval_brick<DIM, ORDER, false, LB>;
        TGCU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<(unsigned)blocks, 256, smem, s>>>(g.ds, g.p[g.cur], pts, n, vals, grads, g.st, nbv[0], nbv[1],
                                                  nbv[2]);
    });
    count_launch();
    TGCU_CUDA(cudaGetLastError());
}

}  // namespace tgcu
