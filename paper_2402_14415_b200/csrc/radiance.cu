// Radiance density chain: emission-absorption rendering of
// a TaylorGrid density + SH color grid and the photometric loss with its
// gradients (volume_render.cpp:61-276, sh.cpp:43-107).
//
// One warp per ray; lane l handles samples l, l+32, ... of the ray, in chunks
// of 32. Per sample: the density query (fp64 locate, fp32 Taylor blend from
// L1/L2 — consecutive samples of a ray sit in neighbouring cells), the shifted
// softplus / clamped ReLU activation, the SH color (fp64 weights and basis, fp32
// coefficients), and the step transmittance exp(-sigma delta) in fp64. The
// transmittance T_i = prod_{j<i} step_j is a warp prefix product per chunk;
// the color a warp sum. The backward pass recomputes the sample state in the
// same order (so T_i and w_i are the forward's values), forms
// suffix_i = C - sum_{j<=i} w_j c_j with a warp prefix sum, and scatters
// dL/dsigma (through the activation) into the density gradient and dL/dpre
// (through the sigmoid and the basis) into the SH gradient with fp32 atomics.
// Per-ray squared errors go to an array reduced in a fixed order.
#include <climits>
#include <vector>

#include "dispatch.cuh"
#include "tg_internal.h"

namespace tgcu {

struct RayArgs {
    DevSpec ds;              // density grid geometry
    const float* dcoeffs;
    DevSpec ss;              // SH grid geometry
    const float* scoeffs;
    const float* rays;       // n x 8: origin xyz, dir xyz, near, far
    const float* gt;         // n x 3 or null
    long long n;
    int S;                   // samples per ray
    int act;                 // 0 shifted softplus, 1 clamp relu
    double shift;
    double bg[3];
    double inv_n;            // 1 / batch size
    float* gd;               // density gradient (K per vertex) or null
    float* gsh;              // SH gradient (3B per vertex) or null
    float* colors;           // n x 3 or null
    float* resid;            // n or null
    double* ray_err;         // n squared errors (gt given)
    const double* jit;       // n x S stratified jitter draws u_i (null: no jitter)
    Status* st;
};

// Stratified jitter (volume_render.cpp:69-70): ray r draws its n_samples
// uniforms from Rng(jitter_seed ^ (r * 0x9e3779b97f4a7c15 + 0x2545f4914f6cdd1d)),
// i.e. std::mt19937_64 seeded per ray, uniform = (x >> 11) * 2^-53
// (rng.hpp:21). One thread per ray, the 312-word state in local memory.
__global__ void __launch_bounds__(128) k_jitter(long long n, int S, unsigned long long seed, double* __restrict__ out) {
    constexpr int NN = 312, MM = 156;
    constexpr unsigned long long MATRIX = 0xB5026F5AA96619E9ull, UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= n) return;
    unsigned long long mt[NN];
    mt[0] = seed ^ ((unsigned long long)r * 0x9e3779b97f4a7c15ull + 0x2545f4914f6cdd1dull);
    for (int i = 1; i < NN; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (unsigned long long)i;
    int idx = NN;
    for (int k = 0; k < S; ++k) {
        if (idx >= NN) {
            for (int i = 0; i < NN; ++i) {
                const unsigned long long x = (mt[i] & UM) | (mt[(i + 1) % NN] & LM);
                mt[i] = mt[(i + MM) % NN] ^ (x >> 1) ^ ((x & 1ull) ? MATRIX : 0ull);
            }
            idx = 0;
        }
        unsigned long long y = mt[idx++];
        y ^= (y >> 29) & 0x5555555555555555ull;
        y ^= (y << 17) & 0x71D67FFFEDA60000ull;
        y ^= (y << 37) & 0xFFF7EEE000000000ull;
        y ^= y >> 43;
        out[r * S + k] = (double)(y >> 11) * 0x1.0p-53;
    }
}

__device__ __forceinline__ double sigmoid_dd(double x) { return 1.0 / (1.0 + exp(-x)); }

template <int DEG>
__device__ __forceinline__ void sh_basis_d(const double* d, double* out) {
    out[0] = 0.28209479177387814;
    if (DEG < 1) return;
    const double x = d[0], y = d[1], z = d[2];
    out[1] = -0.4886025119029199 * y;
    out[2] = 0.4886025119029199 * z;
    out[3] = -0.4886025119029199 * x;
    if (DEG < 2) return;
    out[4] = 1.0925484305920792 * x * y;
    out[5] = -1.0925484305920792 * y * z;
    out[6] = 0.31539156525252005 * (2.0 * z * z - x * x - y * y);
    out[7] = -1.0925484305920792 * x * z;
    out[8] = 0.5462742152960396 * (x * x - y * y);
}

// State of one sample (recomputed identically by the backward pass).
struct SampleState {
    double x[3];
    double delta, sigma, act_deriv, step;
    double color[3];
    double shw[8];
    long long shv;  // SH corner-0 vertex
};

template <int ORDER, int DEG>
__device__ __forceinline__ void sample_state(const RayArgs& A, long long ray, const double* o, const double* d,
                                             double near_, double far_, double bin, int i, const double* basis,
                                             SampleState& st) {
    constexpr int K = KOf<3, ORDER>::value;
    constexpr int B = (DEG + 1) * (DEG + 1);
    constexpr int C = 3 * B;
    // t_i = near + (i [+ u_i]) * bin; delta_i = t_{i+1} - t_i, the last one
    // far - t_i (volume_render.cpp:67-72)
    const double* u = A.jit ? A.jit + ray * A.S : nullptr;
    const double t = __dadd_rn(near_, __dmul_rn(u ? __dadd_rn((double)i, u[i]) : (double)i, bin));
    st.delta = (i + 1 < A.S)
                   ? __dsub_rn(__dadd_rn(near_, __dmul_rn(u ? __dadd_rn((double)(i + 1), u[i + 1]) : (double)(i + 1), bin)), t)
                   : __dsub_rn(far_, t);
#pragma unroll
    for (int a = 0; a < 3; ++a) st.x[a] = __dadd_rn(o[a], __dmul_rn(t, d[a]));
    // density: eval (fp64 locate, fp32 blend) -> activation
    AxisF ax[3];
    long long base = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double local;
        const int c = locate_axis(A.ds, a, st.x[a], local);
        ax[a] = axis_factors(A.ds, a, local);
        base += (long long)c * (a == 0 ? 1LL : (a == 1 ? A.ds.sy : A.ds.sz));
    }
    float fg[3];
    const double raw = (double)eval_cell<3, ORDER, false>(A.ds, A.dcoeffs, base, ax, fg);
    if (A.act == 0) {
        const double z = raw + A.shift;
        st.act_deriv = sigmoid_dd(z);
        st.sigma = z > 30.0 ? z : log1p(exp(z));
    } else {
        st.act_deriv = raw > 0.0 ? 1.0 : 0.0;
        st.sigma = raw > 0.0 ? raw : 0.0;
    }
    // SH color: multilinear weights (fp64, reference order), per-channel basis dot
    double sl[3];
    long long sb = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int c = locate_axis(A.ss, a, st.x[a], sl[a]);
        sb += (long long)c * (a == 0 ? 1LL : (a == 1 ? A.ss.sy : A.ss.sz));
    }
    st.shv = sb;
    double pre[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
        double w = 1.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) w = __dmul_rn(w, ((cc >> a) & 1) ? sl[a] : __dsub_rn(1.0, sl[a]));
        st.shw[cc] = w;
        const long long vid = sb + (cc & 1) + ((cc >> 1) & 1) * A.ss.sy + ((cc >> 2) & 1) * A.ss.sz;
        const float* blk = A.scoeffs + vid * C;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            double acc = 0.0;
#pragma unroll
            for (int b = 0; b < B; ++b) acc = fma((double)__ldg(blk + ch * B + b), basis[b], acc);
            pre[ch] = fma(w, acc, pre[ch]);
        }
    }
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) st.color[ch] = sigmoid_dd(pre[ch]);
    st.step = exp(-st.sigma * st.delta);
    (void)K;
}

__device__ __forceinline__ double warp_prefix_prod(double v, int lane, double* total) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v *= y;
    }
    *total = __shfl_sync(0xffffffffu, v, 31);
    const double ex = __shfl_up_sync(0xffffffffu, v, 1);
    return lane == 0 ? 1.0 : ex;
}

__device__ __forceinline__ double warp_prefix_sum(double v, int lane, double* total) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    *total = __shfl_sync(0xffffffffu, v, 31);
    return v;  // inclusive
}

template <int ORDER, int DEG, bool GRAD>
__global__ void __launch_bounds__(256) k_rays(RayArgs A) {
    constexpr int K = KOf<3, ORDER>::value;
    constexpr int B = (DEG + 1) * (DEG + 1);
    constexpr int C = 3 * B;
    const int lane = threadIdx.x & 31;
    const long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= A.n) return;
    const float4 q0 = reinterpret_cast<const float4*>(A.rays)[2 * r];
    const float4 q1 = reinterpret_cast<const float4*>(A.rays)[2 * r + 1];
    const double o[3] = {q0.x, q0.y, q0.z};
    const double d[3] = {q0.w, q1.x, q1.y};
    const double near_ = q1.z, far_ = q1.w;
    bool bad = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) bad |= isnan(o[a]) || isnan(d[a]);
    if (bad || isnan(near_) || isnan(far_)) {
        if (lane == 0) atomicMin(&A.st->nan_point, (unsigned long long)r);
        return;
    }
    double basis[B];
    sh_basis_d<DEG>(d, basis);
    const double bin = (far_ - near_) / A.S;

    // ---- forward ----
    double Tbase = 1.0, col[3] = {0.0, 0.0, 0.0};
    for (int c0 = 0; c0 < A.S; c0 += 32) {
        const int i = c0 + lane;
        SampleState s;
        double step = 1.0, wc[3] = {0.0, 0.0, 0.0};
        if (i < A.S) {
            sample_state<ORDER, DEG>(A, r, o, d, near_, far_, bin, i, basis, s);
            step = s.step;
        }
        double tot;
        const double ex = warp_prefix_prod(step, lane, &tot);
        if (i < A.S) {
            const double w = (Tbase * ex) * (1.0 - step);
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) wc[ch] = w * s.color[ch];
        }
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) col[ch] += warp_sum_d(wc[ch]);
        Tbase *= tot;
    }
    double C3[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) C3[ch] = col[ch] + Tbase * A.bg[ch];
    if (lane == 0) {
        if (A.colors)
            for (int ch = 0; ch < 3; ++ch) A.colors[3 * r + ch] = (float)C3[ch];
        if (A.resid) A.resid[r] = (float)Tbase;
    }
    if (!A.gt) return;
    double err[3], e2 = 0.0;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        err[ch] = C3[ch] - (double)A.gt[3 * r + ch];
        e2 += err[ch] * err[ch];
    }
    if (lane == 0) A.ray_err[r] = e2;
    if constexpr (!GRAD) return;

    // ---- backward: recompute in forward order, suffix = C - prefix ----
    double g[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) g[ch] = (2.0 * A.inv_n) * err[ch];
    double T2 = 1.0, pref[3] = {0.0, 0.0, 0.0};
    for (int c0 = 0; c0 < A.S; c0 += 32) {
        const int i = c0 + lane;
        SampleState s;
        double step = 1.0, w = 0.0;
        if (i < A.S) {
            sample_state<ORDER, DEG>(A, r, o, d, near_, far_, bin, i, basis, s);
            step = s.step;
        }
        double tot;
        const double ex = warp_prefix_prod(step, lane, &tot);
        const double Ti = T2 * ex;
        if (i < A.S) w = Ti * (1.0 - step);
        double suffix[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            double t3;
            const double inc = warp_prefix_sum(i < A.S ? w * s.color[ch] : 0.0, lane, &t3);
            suffix[ch] = C3[ch] - (pref[ch] + inc);
            pref[ch] += t3;
        }
        T2 *= tot;
        if (i < A.S) {
            const double t_next = Ti * step;
            if (A.gd) {
                double dl_dsigma = 0.0;
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) dl_dsigma += g[ch] * s.delta * (t_next * s.color[ch] - suffix[ch]);
                const double dl_draw = dl_dsigma * s.act_deriv;
                if (dl_draw != 0.0) {  // backprop_point (taylor_grid.cpp:205-213)
                    AxisF ax[3];
                    long long base = 0;
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        double local;
                        const int c = locate_axis(A.ds, a, s.x[a], local);
                        ax[a] = axis_factors(A.ds, a, local);
                        base += (long long)c * (a == 0 ? 1LL : (a == 1 ? A.ds.sy : A.ds.sz));
                    }
                    const float gv[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) {
                        float G[K];
#pragma unroll
                        for (int q = 0; q < K; ++q) G[q] = 0.0f;
                        corner_grad<3, ORDER, K>(corner_geom<3>(A.ds, ax, cc), (float)dl_draw, gv, G);
                        const long long vid = base + (cc & 1) + ((cc >> 1) & 1) * A.ds.sy + ((cc >> 2) & 1) * A.ds.sz;
                        red_block<K>(A.gd + vid * K, G);
                    }
                }
            }
            if (A.gsh) {
                double dl_dpre[3];
                bool any = false;
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    const double c = s.color[ch];
                    dl_dpre[ch] = g[ch] * w * c * (1.0 - c);
                    any |= dl_dpre[ch] != 0.0;
                }
                if (any) {
                    // the corner's whole 3B-float SH block in one vector reduction
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) {
                        const long long vid = s.shv + (cc & 1) + ((cc >> 1) & 1) * A.ss.sy + ((cc >> 2) & 1) * A.ss.sz;
                        float gb[C];
#pragma unroll
                        for (int ch = 0; ch < 3; ++ch) {
                            const double f = s.shw[cc] * dl_dpre[ch];
#pragma unroll
                            for (int b = 0; b < B; ++b) gb[ch * B + b] = (float)(f * basis[b]);
                        }
                        red_block<C>(A.gsh + vid * C, gb);
                    }
                }
            }
        }
    }
}

// Fixed-order sum of n doubles (one CTA), times scale.
__global__ void __launch_bounds__(1024) k_sum_scaled(const double* __restrict__ x, long long n, double scale,
                                                     double* __restrict__ out) {
    __shared__ double red[32];
    double a = 0.0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) a += x[i];
    a = warp_sum_d(a);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 32; ++k) t += red[k];
        *out = t * scale;
    }
}

void launch_rays(Grid& g, const DevSpec& ss, int deg, const float* scoeffs, const float* rays, const float* gt,
                 int64_t n, const tgcu_render_options& o, float* colors, float* resid, float* gd, float* gsh,
                 double* ray_err, double* loss, cudaStream_t s) {
    RayArgs A{};
    A.ds = g.ds;
    A.dcoeffs = g.p[g.cur];
    A.ss = ss;
    A.scoeffs = scoeffs;
    A.rays = rays;
    A.gt = gt;
    A.n = n;
    A.S = o.n_samples;
    A.act = o.activation;
    A.shift = o.softplus_shift;
    for (int a = 0; a < 3; ++a) A.bg[a] = o.background[a];
    A.inv_n = 1.0 / (double)n;
    A.gd = gd;
    A.gsh = gsh;
    A.colors = colors;
    A.resid = resid;
    A.ray_err = ray_err;
    A.st = g.st;
    double* jit = nullptr;
    if (o.jitter) {
        TGCU_CUDA(cudaMallocAsync(&jit, sizeof(double) * n * o.n_samples, s));
        k_jitter<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(n, o.n_samples, o.jitter_seed, jit);
        count_launch();
        A.jit = jit;
    }
    const bool grad = gt && (gd || gsh);
    const unsigned blocks = (unsigned)((n + 7) / 8);
    auto go = [&](auto kern) { kern<<<blocks, 256, 0, s>>>(A); };
#define TGCU_RAYS(ORD)                                                                  \
    do {                                                                                \
        if (deg == 0) grad ? go(k_rays<ORD, 0, true>) : go(k_rays<ORD, 0, false>);      \
        else if (deg == 1) grad ? go(k_rays<ORD, 1, true>) : go(k_rays<ORD, 1, false>); \
        else grad ? go(k_rays<ORD, 2, true>) : go(k_rays<ORD, 2, false>);               \
    } while (0)
    if (g.spec.order == 2) TGCU_RAYS(2);
    else if (g.spec.order == 1) TGCU_RAYS(1);
    else TGCU_RAYS(0);
#undef TGCU_RAYS
    count_launch();
    if (gt && loss) {
        k_sum_scaled<<<1, 1024, 0, s>>>(ray_err, n, 1.0 / (double)n, loss);
        count_launch();
    }
    if (jit) TGCU_CUDA(cudaFreeAsync(jit, s));
    TGCU_CUDA(cudaGetLastError());
}

}  // namespace tgcu

using namespace tgcu;

extern "C" int tgcu_photometric_loss(tgcu_grid* h, const tgcu_grid_spec* sh_spec, int sh_degree,
                                     const float* sh_coeffs, const float* rays, const float* gt, int64_t n,
                                     const tgcu_render_options* opts, float* colors, float* residual,
                                     float* grad_density, float* grad_sh, double* loss, int flags, void* stream) {
    return guard([&] {
        require(h && sh_spec && sh_coeffs && rays && opts, "photometric_loss: NULL argument");
        Grid& g = h->g;
        require(n > 0, "photometric_loss: empty ray batch");
        require(opts->n_samples >= 1 && opts->n_samples <= 1024, "photometric_loss: n_samples out of range");
        require(sh_degree >= 0 && sh_degree <= 2, "init_sh_grid: degree must be in [0,2]");
        require(opts->activation == TGCU_DENSITY_SHIFTED_SOFTPLUS || opts->activation == TGCU_DENSITY_CLAMP_RELU,
                "photometric_loss: unknown density activation");
        require(g.spec.dim == 3 && sh_spec->dim == 3, "photometric_loss: 3D density and SH grids");
        require(!g.slab, "photometric_loss: slab grids are not supported");
        require(!(grad_density || grad_sh) || gt, "photometric_loss: gradients need gt colors");
        tgcu_grid_spec ss = *sh_spec;
        ss.order = 0;
        validate_spec(ss);
        const DevSpec sds = make_devspec(ss);
        const int C = 3 * (sh_degree + 1) * (sh_degree + 1);
        const int64_t nsh = (int64_t)ss.res[0] * ss.res[1] * ss.res[2] * C;
        TGCU_CUDA(cudaSetDevice(g.device));
        cudaStream_t s = as_stream(stream);
        const bool host = flags & TGCU_HOST;
        // device views of every array (staged when the caller passes host memory)
        float *d_sh = const_cast<float*>(sh_coeffs), *d_rays = const_cast<float*>(rays),
              *d_gt = const_cast<float*>(gt), *d_col = colors, *d_res = residual, *d_gd = grad_density,
              *d_gsh = grad_sh;
        std::vector<void*> tmp;
        auto stage = [&](float*& dp, const float* hp, int64_t count, bool copy_in) {
            if (!hp) {
                dp = nullptr;
                return;
            }
            void* q = nullptr;
            TGCU_CUDA(cudaMallocAsync(&q, sizeof(float) * count, s));
            tmp.push_back(q);
            dp = static_cast<float*>(q);
            if (copy_in) TGCU_CUDA(cudaMemcpyAsync(dp, hp, sizeof(float) * count, cudaMemcpyHostToDevice, s));
        };
        if (host) {
            stage(d_sh, sh_coeffs, nsh, true);
            stage(d_rays, rays, 8 * n, true);
            stage(d_gt, gt, 3 * n, true);
            stage(d_col, colors, 3 * n, false);
            stage(d_res, residual, n, false);
            stage(d_gd, grad_density, g.NC, true);  // gradients accumulate (+=) as the reference's spans
            stage(d_gsh, grad_sh, nsh, true);
        }
        require((reinterpret_cast<uintptr_t>(d_rays) & 15) == 0, "photometric_loss: rays must be 16-byte aligned");
        double* d_err = nullptr;
        double* d_loss = nullptr;
        if (gt) {
            TGCU_CUDA(cudaMallocAsync(&d_err, sizeof(double) * (n + 1), s));
            d_loss = d_err + n;
        }
        launch_rays(g, sds, sh_degree, d_sh, d_rays, d_gt, n, *opts, d_col, d_res, d_gd, d_gsh, d_err, d_loss, s);
        double lv = 0.0;
        if (gt) TGCU_CUDA(cudaMemcpyAsync(&lv, d_loss, sizeof(double), cudaMemcpyDeviceToHost, s));
        if (host) {
            if (colors) TGCU_CUDA(cudaMemcpyAsync(colors, d_col, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost, s));
            if (residual) TGCU_CUDA(cudaMemcpyAsync(residual, d_res, sizeof(float) * n, cudaMemcpyDeviceToHost, s));
            if (grad_density)
                TGCU_CUDA(cudaMemcpyAsync(grad_density, d_gd, sizeof(float) * g.NC, cudaMemcpyDeviceToHost, s));
            if (grad_sh) TGCU_CUDA(cudaMemcpyAsync(grad_sh, d_gsh, sizeof(float) * nsh, cudaMemcpyDeviceToHost, s));
        }
        if (d_err) TGCU_CUDA(cudaFreeAsync(d_err, s));
        for (void* q : tmp) TGCU_CUDA(cudaFreeAsync(q, s));
        TGCU_CUDA(cudaStreamSynchronize(s));
        if (loss) *loss = lv;
        // NaN ray -> the reference's locate error
        Status sth;
        TGCU_CUDA(cudaMemcpy(&sth, g.st, sizeof(Status), cudaMemcpyDeviceToHost));
        if (sth.nan_point != ULLONG_MAX) {
            const unsigned long long none = ULLONG_MAX;
            TGCU_CUDA(cudaMemcpy(&g.st->nan_point, &none, sizeof(none), cudaMemcpyHostToDevice));
            throw Error(TGCU_ERR_INVALID_ARGUMENT, "locate: NaN coordinate (ray " + std::to_string(sth.nan_point) + ")");
        }
    });
}
