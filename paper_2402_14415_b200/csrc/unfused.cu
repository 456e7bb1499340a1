// Unfused reference-API kernels: batched backprop (atomic scatter), the
// standalone total_loss point terms, tv_loss, the two-pass adam_step and
// small conversion / init utilities. These serve the reference's
// function-by-function API (caller-owned gradient buffer); the training hot
// path is the fused kernel in train.cu.
#include "dispatch.cuh"
#include "tg_internal.h"

namespace tgcu {

// Scatter-add of one point's 2^D*K coefficient gradients with vector fp32
// reductions (red_block: REDG.E.ADD.F32x4 / x2 / scalar by alignment).
template <int DIM, int ORDER>
__device__ __forceinline__ void scatter_point(const DevSpec& s, const AxisF* ax, long long base, float u,
                                              const float* gv, float* __restrict__ grad) {
    constexpr int K = KOf<DIM, ORDER>::value;
#pragma unroll
    for (int c = 0; c < (1 << DIM); ++c) {
        const Corner<DIM> g = corner_geom<DIM>(s, ax, c);
        float G[K];
#pragma unroll
        for (int q = 0; q < K; ++q) G[q] = 0.0f;
        corner_grad<DIM, ORDER, K>(g, u, gv, G);
        const long long vid = base + (c & 1) + ((c >> 1) & 1) * s.sy + (DIM == 3 ? ((c >> 2) & 1) * s.sz : 0);
        red_block<K>(grad + vid * K, G);
    }
}

template <int DIM, int ORDER>
__global__ void __launch_bounds__(256) k_backprop(DevSpec s, const float* __restrict__ pts,
                                                  const float* __restrict__ up, const float* __restrict__ upv,
                                                  long long n, float* __restrict__ grad, Status* st) {
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
        const float u = up ? up[i] : 0.0f;
        float gv[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) gv[a] = upv ? upv[3 * i + a] : 0.0f;
        // backprop_point skips a zero upstream (taylor_grid.cpp:209).
        bool any = u != 0.0f;
#pragma unroll
        for (int a = 0; a < DIM; ++a) any |= gv[a] != 0.0f;
        if (!any) continue;
        scatter_point<DIM, ORDER>(s, ax, base, u, gv, grad);
    }
}

void launch_backprop(Grid& g, const float* pts, const float* up, const float* upv, int64_t n, float* grad,
                     cudaStream_t s) {
    if (n <= 0) return;
    const int blocks = grid_blocks(n, 256, 148 * 32);
    TGCU_DISPATCH(g.spec.dim, g.spec.order,
                  k_backprop<DIM, ORDER><<<blocks, 256, 0, s>>>(g.ds, pts, up, upv, n, grad, g.st));
    count_launch();
    TGCU_CUDA(cudaGetLastError());
}

// Standalone total_loss point pass: gather-eval, fp64 loss chain, atomic
// scatter. Per-block fp64 partial sums -> partials[block*2 + {0,1}].
template <int DIM, int ORDER, bool EIK>
__global__ void __launch_bounds__(256) k_point_terms(DevSpec s, const float* __restrict__ coeffs,
                                                     const float4* __restrict__ smp, long long n, LossDev L,
                                                     float* __restrict__ grad, double* __restrict__ partials,
                                                     Status* st) {
    constexpr int K = KOf<DIM, ORDER>::value;
    double recon_sum = 0.0, eik_sum = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float4 q = smp[i];
        const float pf[3] = {q.x, q.y, q.z};
        double x[DIM];
        bool nan = false;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            x[a] = (double)pf[a];
            nan |= isnan(x[a]);
        }
        if (nan) {
            atomicMin(&st->nan_point, (unsigned long long)i);
            continue;
        }
        AxisF ax[DIM];
        double lc[DIM];
        long long base = 0;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            const int c = locate_axis(s, a, x[a], lc[a]);
            ax[a] = axis_factors(s, a, lc[a]);
            base += (long long)c * (a == 0 ? 1LL : (a == 1 ? s.sy : s.sz));
        }
        float cb[1 << DIM][K];
#pragma unroll
        for (int c = 0; c < (1 << DIM); ++c) {
            const long long vid = base + (c & 1) + ((c >> 1) & 1) * s.sy + (DIM == 3 ? ((c >> 2) & 1) * s.sz : 0);
            load_block<K, true>(coeffs + vid * K, cb[c]);
        }
        double f = 0.0, fg[DIM];  // fp64 forward, as the fused step (blend_corner_d)
#pragma unroll
        for (int a = 0; a < DIM; ++a) fg[a] = 0.0;
#pragma unroll
        for (int c = 0; c < (1 << DIM); ++c) blend_corner_d<DIM, ORDER, EIK>(cb[c], s, lc, c, f, fg);
        double recon, eik;
        float u, gv[DIM];
        point_loss<DIM, EIK>(L, f, fg, q.w, recon, eik, u, gv);
        recon_sum += recon;
        eik_sum += eik;
        if (grad) scatter_point<DIM, ORDER>(s, ax, base, u, gv, grad);
    }
    // Block reduction (fixed order per block).
    __shared__ double red[2][8];
    recon_sum = warp_sum_d(recon_sum);
    eik_sum = warp_sum_d(eik_sum);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        red[0][w] = recon_sum;
        red[1][w] = eik_sum;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
            a += red[0][k];
            b += red[1][k];
        }
        partials[2 * blockIdx.x] = a;
        partials[2 * blockIdx.x + 1] = b;
    }
}

// Sum nblk per-block partial pairs in a fixed order -> out[0..1].
__global__ void k_reduce_pairs(const double* __restrict__ partials, int nblk, double* __restrict__ out) {
    __shared__ double red[2][32];
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
        a += partials[2 * i];
        b += partials[2 * i + 1];
    }
    a = warp_sum_d(a);
    b = warp_sum_d(b);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = a;
        red[1][threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double x = 0.0, y = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
            x += red[0][k];
            y += red[1][k];
        }
        out[0] = x;
        out[1] = y;
    }
}

void launch_point_terms(Grid& g, const float4* samples, int64_t n, const tgcu_loss_config& cfg, float* grad,
                        cudaStream_t s, double upstream_scale, bool eik_points) {
    const int blocks = grid_blocks(n, 256, 148 * 8);
    ensure_scratch(g, 2 * (int64_t)blocks + 8);
    LossDev L;
    L.k = cfg.k;
    L.inv_n = upstream_scale / (double)n;  // recon_loss's scale (sdf_loss.cpp:130-135)
    L.eik_scale = cfg.lambda1;
    L.use_weighting = cfg.use_weighting;
    L.differentiate_weight = cfg.differentiate_weight;
    L.fresh_eik = eik_points ? 1 : 0;  // eikonal_loss: marked points, eikonal term only
    const bool eik = cfg.lambda1 > 0.0 || eik_points;
    double* partials = g.scratch_d + 8;
    TGCU_DISPATCH(g.spec.dim, g.spec.order, {
        if (eik)
            k_point_terms<DIM, ORDER, true><<<blocks, 256, 0, s>>>(g.ds, g.p[g.cur], samples, n, L, grad, partials, g.st);
        else
            k_point_terms<DIM, ORDER, false><<<blocks, 256, 0, s>>>(g.ds, g.p[g.cur], samples, n, L, grad, partials, g.st);
    });
    k_reduce_pairs<<<1, 1024, 0, s>>>(partials, blocks, g.scratch_d);
    count_launch(2);
    TGCU_CUDA(cudaGetLastError());
}

// tv_loss (sdf_loss.cpp:155-257) as a per-vertex stencil: each vertex adds
// its own TV gradient (no atomics) and the squared differences of the pairs
// it is the lower end of. Sums -> scratch_d[2] via per-block partials.
template <int K, int DIM>
__global__ void __launch_bounds__(256) k_tv(DevSpec s, const float* __restrict__ c, float* __restrict__ grad,
                                            float gscale, long long V, double* __restrict__ partials) {
    double sum = 0.0;
    const long long strides[3] = {1, s.sy, s.sz};
    for (long long vtx = blockIdx.x * (long long)blockDim.x + threadIdx.x; vtx < V;
         vtx += (long long)gridDim.x * blockDim.x) {
        long long rem = vtx;
        int co[3];
        co[0] = (int)(rem % s.res[0]);
        rem /= s.res[0];
        co[1] = (int)(DIM == 3 ? rem % s.res[1] : rem);
        co[2] = DIM == 3 ? (int)(rem / s.res[1]) : 0;
        float pv[K];
#pragma unroll
        for (int q = 0; q < K; ++q) pv[q] = c[vtx * K + q];
        float gt[K];
#pragma unroll
        for (int q = 0; q < K; ++q) gt[q] = 0.0f;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            if (co[a] + 1 < s.res[a]) {
                const float* pu = c + (vtx + strides[a]) * K;
#pragma unroll
                for (int q = 0; q < K; ++q) {
                    const float d = pu[q] - pv[q];
                    sum += (double)d * (double)d;
                    gt[q] -= d;
                }
            }
            if (co[a] >= 1) {
                const float* pl = c + (vtx - strides[a]) * K;
#pragma unroll
                for (int q = 0; q < K; ++q) gt[q] += pv[q] - pl[q];
            }
        }
        if (grad) {
#pragma unroll
            for (int q = 0; q < K; ++q) grad[vtx * K + q] += gscale * gt[q];
        }
    }
    __shared__ double red[8];
    sum = warp_sum_d(sum);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) a += red[k];
        partials[2 * blockIdx.x] = a;
        partials[2 * blockIdx.x + 1] = 0.0;
    }
}

void launch_tv(Grid& g, const float* coeffs, float* grad, double gscale, int /*want_value*/, cudaStream_t s) {
    const int blocks = grid_blocks(g.V, 256, 148 * 8);
    ensure_scratch(g, 2 * (int64_t)blocks + 8);
    double* partials = g.scratch_d + 8;
    TGCU_DISPATCH(g.spec.dim, g.spec.order, {
        constexpr int K = KOf<DIM, ORDER>::value;
        k_tv<K, DIM><<<blocks, 256, 0, s>>>(g.ds, coeffs, grad, (float)gscale, g.V, partials);
    });
    k_reduce_pairs<<<1, 1024, 0, s>>>(partials, blocks, g.scratch_d + 2);
    count_launch(2);
    TGCU_CUDA(cudaGetLastError());
}

// adam_step pass 1: first non-finite gradient index (adam.cpp:18-34).
__global__ void k_adam_check(const float* __restrict__ g, long long n, Status* st) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        if (!isfinite(g[i])) atomicMin(&st->bad_grad, (unsigned long long)i);
}

// adam_step pass 2 (adam.cpp:36-55), in place, fp32 state, host fp64 bias
// corrections.
__global__ void k_adam_update(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                              float* __restrict__ v, long long n, float lr, float b1, float b2, float c1,
                              float c2, float eps, float inv_bc1, float inv_bc2) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float gi = g[i];
        const float mi = fmaf(b1, m[i], c1 * gi);
        const float vi = fmaf(b2, v[i], c2 * gi * gi);
        m[i] = mi;
        v[i] = vi;
        p[i] -= lr * (mi * inv_bc1) / (sqrtf(vi * inv_bc2) + eps);
    }
}

void launch_adam_check(Grid& g, const float* grad, cudaStream_t s) {
    k_adam_check<<<grid_blocks(g.NC, 256, 148 * 16), 256, 0, s>>>(grad, g.NC, g.st);
    count_launch();
    TGCU_CUDA(cudaGetLastError());
}

void launch_adam_update(Grid& g, const float* grad, double inv_bc1, double inv_bc2, cudaStream_t s) {
    k_adam_update<<<grid_blocks(g.NC, 256, 148 * 16), 256, 0, s>>>(
        g.p[g.cur], grad, g.m[g.cur], g.v[g.cur], g.NC, (float)g.adam.lr, (float)g.adam.beta1,
        (float)g.adam.beta2, (float)(1.0 - g.adam.beta1), (float)(1.0 - g.adam.beta2), (float)g.adam.eps,
        (float)inv_bc1, (float)inv_bc2);
    count_launch();
    TGCU_CUDA(cudaGetLastError());
}

// ---- utilities -------------------------------------------------------------

__global__ void k_f64_to_f32(const double* __restrict__ a, float* __restrict__ b, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        b[i] = (float)a[i];
}
__global__ void k_f32_to_f64(const float* __restrict__ a, double* __restrict__ b, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        b[i] = (double)a[i];
}
__global__ void k_all_finite(const float* __restrict__ a, long long n, unsigned long long* flag) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        if (!isfinite(a[i])) atomicMin(flag, (unsigned long long)i);
}
__global__ void k_fill_f0(float* __restrict__ p, long long V, int K, float value) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < V; i += (long long)gridDim.x * blockDim.x)
        p[i * K] = value;
}

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
__device__ __forceinline__ double hash_uniform(unsigned long long seed, unsigned long long i) {
    return (double)(splitmix64(seed * 0x2545F4914F6CDD1DULL + i) >> 11) * 0x1.0p-53;
}

__global__ void k_hash_gaussian(float* __restrict__ p, long long n, unsigned long long seed, float sigma,
                                long long goff) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long gi = i + goff;  // global coefficient index (slab grids)
        double u1 = hash_uniform(seed, 2 * gi);
        const double u2 = hash_uniform(seed, 2 * gi + 1);
        if (u1 <= 0.0) u1 = 0x1.0p-53;
        p[i] = sigma * (float)(sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
    }
}

__global__ void k_hash_points(float* __restrict__ out, long long n, int dim, unsigned long long seed, double lo,
                              double hi) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
            out[3 * i + a] = a < dim ? (float)(lo + (hi - lo) * hash_uniform(seed, 3 * i + a)) : 0.0f;
    }
}

// SdfProblem batch draw (sdf_fit.cpp:21-23): n samples with replacement from
// a device-resident pool; index = floor(u * pool_n) from a counter hash of
// (seed, step, i) in place of the reference's mt19937_64 stream.
__global__ void k_draw_batch(const float4* __restrict__ pool, long long pool_n, long long n,
                             unsigned long long seed, unsigned long long step, float4* __restrict__ out) {
    const unsigned long long key = splitmix64(seed ^ (step * 0xD1B54A32D192ED03ULL));
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        long long j = (long long)(hash_uniform(key, (unsigned long long)i) * (double)pool_n);
        j = j < pool_n ? j : pool_n - 1;
        out[i] = __ldg(pool + j);
    }
}

void launch_draw_batch(const float* pool, int64_t pool_n, int64_t n, uint64_t seed, uint64_t step, float* out,
                       cudaStream_t s) {
    if (n <= 0) return;
    k_draw_batch<<<grid_blocks(n, 256, 148 * 16), 256, 0, s>>>(reinterpret_cast<const float4*>(pool), pool_n, n, seed,
                                                                step, reinterpret_cast<float4*>(out));
    count_launch();
    TGCU_CUDA(cudaGetLastError());
}

void launch_hash_gaussian(float* dst, int64_t n, uint64_t seed, double sigma, int64_t goff, cudaStream_t s) {
    k_hash_gaussian<<<grid_blocks(n, 256, 148 * 64), 256, 0, s>>>(dst, n, seed, (float)sigma, goff);
    count_launch();
    TGCU_CUDA(cudaGetLastError());
}

void launch_hash_points(float* out, int64_t n, int dim, uint64_t seed, double lo, double hi, cudaStream_t s) {
    k_hash_points<<<grid_blocks(n, 256, 148 * 64), 256, 0, s>>>(out, n, dim, seed, lo, hi);
    count_launch();
    TGCU_CUDA(cudaGetLastError());
}

void launch_f64_to_f32(const double* src, float* dst, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    k_f64_to_f32<<<grid_blocks(n, 256), 256, 0, s>>>(src, dst, n);
    count_launch();
    TGCU_CUDA(cudaGetLastError());
}
void launch_f32_to_f64(const float* src, double* dst, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    k_f32_to_f64<<<grid_blocks(n, 256), 256, 0, s>>>(src, dst, n);
    count_launch();
    TGCU_CUDA(cudaGetLastError());
}
void launch_all_finite(const float* src, int64_t n, unsigned long long* flag, cudaStream_t s) {
    if (n <= 0) return;
    k_all_finite<<<grid_blocks(n, 256), 256, 0, s>>>(src, n, flag);
    count_launch();
    TGCU_CUDA(cudaGetLastError());
}
void launch_fill_f0(Grid& g, float* dst, float value, cudaStream_t s) {
    k_fill_f0<<<grid_blocks(g.V, 256), 256, 0, s>>>(dst, g.V, g.K, value);
    count_launch();
    TGCU_CUDA(cudaGetLastError());
}

}  // namespace tgcu
