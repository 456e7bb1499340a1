// Two-launch fused training step for small grids (BASELINE configs[0], C1:
// a 128^2 2D grid with 65,536 points per step, 64 bricks on 148 SMs).
//
// The brick path (train.cu) needs five launches per step (three binning
// kernels, the brick kernel, the finalize), each latency-bound at this size
// (DESIGN.md §9). Here one step of run_schedule's inner loop
// (schedule.cpp:66-92: zero_grad -> total_loss -> finite check -> adam_step)
// is two kernels chained by programmatic dependent launch (PDL: each grid is
// scheduled while its predecessor runs and waits in griddepcontrol.wait for
// its completion, so the launch latency between them is hidden):
//   k_small_points  thread per point: fp64 locate (grid_spec.cpp:45-69), the
//                   2^D corner blocks read straight from the L2-resident
//                   parameters, the forward (taylor_grid.cpp:100-119), the fp64
//                   per-point loss chain (sdf_loss.cpp:51-74) and each corner's
//                   coefficient gradient (accumulate_cell,
//                   taylor_grid.cpp:123-152) added into an fp32 accumulator
//                   with vector reductions in L2 (red.global.add.v2/v4);
//   k_small_coeffs  thread per coefficient (coalesced): TV gradient from the
//                   parameter stencil (sdf_loss.cpp:161-210) + the accumulated
//                   point gradient, the finite check, Adam (adam.cpp:36-55)
//                   into the other ping-pong slot, the accumulator zeroed for
//                   the next step ("fused with gradient zeroing"); the last CTA
//                   to finish reduces every CTA's loss partials in CTA order
//                   and commits (finalize.cuh, the brick path's code).
// The kernel boundary is the grid-wide barrier, so nothing assumes that the
// CTAs of a grid are co-resident (a cooperative single launch with an
// in-kernel grid barrier measured 16.4 us per C1 step).
// Summation order of a coefficient's point contributions follows the L2
// atomics (not bit-reproducible); deterministic mode keeps the brick path.
#include <climits>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "dispatch.cuh"
#include "finalize.cuh"
#include "tg_internal.h"
#include "tma.cuh"

namespace tgcu {

struct SmallArgs {
    DevSpec s;
    const float4* pts;
    int n;
    int nc;  // coefficients V*K
    const float* p_in;
    float* p_out;
    const float* m_in;
    float* m_out;
    const float* v_in;
    float* v_out;
    float* acc;       // fp32 point-gradient accumulator (zero between steps)
    float* grad_out;  // optional: full gradient (TGCU_EXPORT_GRAD)
    LossDev L;
    float tv_gscale;
    int want_tv;
    float lr, b1, b2, eps, inv_bc1, inv_bc2, c1, c2;
    double* partials;  // (points CTAs + coefficient CTAs) x 4: recon, eik, tv, points
    int ncta_pts;      // CTAs of k_small_points (their partials come first)
    Status* st;
    unsigned long long* nan;
    FinArgs F;
    unsigned* ticket;  // coefficient CTAs done with their partials (zero between launches)
    int early;         // points grid triggers the coefficient grid's launch at its start
    int pts_ready;     // samples complete before the launch (may be read before the PDL wait)
    const long long* ctr;  // graph-replayed steps: {t, step} on the device (F.ctr), else nullptr
    const float2* bc;      // with ctr: (1/(1 - b1^t), 1/(1 - b2^t)) for t = 1..kBcTab, host-rounded
};

// Bias-correction table of graph-replayed steps: entry t-1 holds the values
// the host would pass for Adam step t (both are exactly 1.0f from t = 65536 on,
// 0.999^65536 ~ 3e-29).
constexpr int kBcTab = 65536;

constexpr int kSmallNT = 256;

#ifdef TGCU_PHASE_TIMING
// Instrumented build only (tools/small_phase.py): per step, the first CTA
// start and the last CTA end of each kernel.
__device__ unsigned long long g_sring[256 * 4];
#define TGCU_SRING(slot, op)                                                   \
    if (threadIdx.x == 0) {                                                    \
        unsigned long long t_;                                                 \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
        op(&g_sring[4 * (A.F.step & 255) + (slot)], t_);                       \
    }
#else
#define TGCU_SRING(slot, op)
#endif

// PDL: wait until the previous grid on the stream has completed (its memory
// operations visible); let the next grid be scheduled (once every CTA of
// this grid has triggered or exited). Triggering only after the wait keeps at
// most two grids of the chain resident at a time.
// (pdl_wait / pdl_trigger: tma.cuh)

// Block reduction of four doubles (fixed order) -> out[0..3].
__device__ __forceinline__ void block_partials(double (*red)[kSmallNT / 32], double a, double b, double c, double d,
                                               double* out) {
    constexpr int NW = kSmallNT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double v4[4] = {warp_sum_d(a), warp_sum_d(b), warp_sum_d(c), warp_sum_d(d)};
    if (lane == 0)
        for (int k = 0; k < 4; ++k) red[k][warp] = v4[k];
    __syncthreads();
    if (threadIdx.x < 4) {
        double s = 0.0;
        for (int k = 0; k < NW; ++k) s += red[threadIdx.x][k];
        out[threadIdx.x] = s;
    }
}

// Lanes per point: a point's corners form 2^(D-1) x-pairs (two vertex blocks
// adjacent in memory, read as 2K contiguous floats and reduced into as one
// 2K-float segment). In 3D the four pairs go to four consecutive lanes whose
// partial blends are summed with shuffles (63 registers instead of 114;
// 3D 32^3 28.5 vs 32.2 us per step); in 2D one lane takes both pairs — two
// lanes per point measured slower at C1 (14.4 vs 12.7 us per step: the
// fp64 locate and loss chain run once per lane).
template <int DIM>
struct SmallLanes {
    static constexpr int P = DIM == 3 ? 4 : 1;       // lanes per point
    static constexpr int NP = (1 << (DIM - 1)) / P;  // corner pairs per lane
};

template <int DIM, int ORDER, bool EIK>
__global__ void __launch_bounds__(kSmallNT) k_small_points(const __grid_constant__ SmallArgs A) {
    constexpr int K = KOf<DIM, ORDER>::value;
    constexpr int P = SmallLanes<DIM>::P, NP = SmallLanes<DIM>::NP;
    __shared__ double red[4][kSmallNT / 32];
    // The first point of this thread is loaded before the wait when the
    // batch is known complete (input-ready or event-ordered samples), so its
    // load overlaps the previous grid's tail; a batch produced by a kernel
    // just before this one on the stream is read after the wait.
    const int i0 = blockIdx.x * (kSmallNT / P) + (int)(threadIdx.x / P);
    float4 q0 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (A.pts_ready && i0 < A.n) q0 = __ldg(A.pts + i0);
    pdl_wait();
    // When to let the coefficient grid be scheduled: early in 2D, where both
    // grids fit an SM together and the early trigger hides the launch (C1:
    // 12.9 vs 16.2 us per step); in 3D after the points (an early-resident
    // coefficient grid cost the points grid occupancy: 3D 48^3, 2^17 points,
    // 63.3 vs 54.5 us per step with one thread per point).
    const bool early = A.early;
    if (early) pdl_trigger();
    // (st->error is written only by an earlier step's finalize)
    if (A.st->error) return;
    TGCU_SRING(0, atomicMin)
    const int t = threadIdx.x & (P - 1);             // lane within the point's group
    const int gstride = gridDim.x * (kSmallNT / P);  // points per sweep
    const long long sy = A.s.sy, sz = A.s.sz;
    double recon_sum = 0.0, eik_sum = 0.0;
    int npts = 0;
    // A warp runs the sweep to its last point as a whole (the group sums are
    // full-warp shuffles): lanes past the end or on a NaN point compute on a
    // harmless point and store nothing.
    for (int i = i0; P == 1 ? i < A.n : __any_sync(0xffffffffu, i < A.n); i += gstride) {
        bool valid = i < A.n;
        float4 q = valid ? (i == i0 && A.pts_ready ? q0 : __ldg(A.pts + i)) : make_float4(0.f, 0.f, 0.f, 0.f);
        bool nanp = false;
#pragma unroll
        for (int a = 0; a < DIM; ++a) nanp |= isnan(a == 0 ? q.x : (a == 1 ? q.y : q.z));
        if (nanp) {  // dropped, reported by the finalize (as the binning does)
            if (t == 0) atomicMin(A.nan, (unsigned long long)i);
            if (P == 1) continue;
            valid = false;
            q = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        const float pf[3] = {q.x, q.y, q.z};
        double lc[DIM];
        AxisF ax[DIM];
        long long base = 0;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            const int c = locate_axis(A.s, a, (double)pf[a], lc[a]);
            base += (long long)c * (a == 0 ? 1LL : (a == 1 ? sy : sz));
            ax[a] = axis_factors(A.s, a, lc[a]);
        }
        // pair j of this lane = corner pair pr = t*NP + j: corners 2pr, 2pr+1,
        // first vertex base + (y, z) offset of pr
        auto pair_vertex = [&](int pr) { return base + (pr & 1) * sy + (DIM == 3 ? (pr >> 1) * sz : 0LL); };
        float cb[NP][2][K];
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const long long v0 = pair_vertex(t * NP + j);
            load_block<K, true>(A.p_in + v0 * K, cb[j][0]);
            load_block<K, true>(A.p_in + (v0 + 1) * K, cb[j][1]);
        }
        float f = 0.0f, fg[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) fg[a] = 0.0f;
#pragma unroll
        for (int j = 0; j < NP; ++j)
#pragma unroll
            for (int b = 0; b < 2; ++b)
                blend_corner<DIM, ORDER, EIK>(cb[j][b], corner_geom<DIM>(A.s, ax, 2 * (t * NP + j) + b), f, fg);
#pragma unroll
        for (int o = 1; o < P; o <<= 1) {  // the group's sum (a group never spans warps)
            f += __shfl_xor_sync(0xffffffffu, f, o);
#pragma unroll
            for (int a = 0; a < DIM; ++a) fg[a] += __shfl_xor_sync(0xffffffffu, fg[a], o);
        }
        double recon, eik;
        float u, gv[DIM];
        point_loss<DIM, EIK>(A.L, f, fg, q.w, recon, eik, u, gv);
        if (!valid) continue;  // (after the group's shuffles)
        if (t == 0) {
            recon_sum += recon;
            eik_sum += eik;
            ++npts;
        }
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const int pr = t * NP + j;
            float G[2 * K];
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                float Gb[K];
#pragma unroll
                for (int k2 = 0; k2 < K; ++k2) Gb[k2] = 0.0f;
                corner_grad<DIM, ORDER, K>(corner_geom<DIM>(A.s, ax, 2 * pr + b), u, gv, Gb);
#pragma unroll
                for (int k2 = 0; k2 < K; ++k2) G[b * K + k2] = Gb[k2];
            }
            red_block<2 * K>(A.acc + pair_vertex(pr) * K, G);
        }
    }
    if (!early) pdl_trigger();
    block_partials(red, recon_sum, eik_sum, 0.0, (double)npts, A.partials + 4 * blockIdx.x);
    TGCU_SRING(1, atomicMax)
}

template <int DIM, int ORDER, bool EXPORT>
__global__ void __launch_bounds__(kSmallNT) k_small_coeffs(const __grid_constant__ SmallArgs A) {
    constexpr int K = KOf<DIM, ORDER>::value;
    __shared__ double red[4][kSmallNT / 32];
    __shared__ int last;
    const int nthr = gridDim.x * kSmallNT;
    const int tid = threadIdx.x;
    const int r0 = A.s.res[0], r1 = A.s.res[1];
    const int offs[3] = {K, r0 * K, r0 * r1 * K};
    // Rounds of R coefficients per thread, every load of a round issued before
    // its arithmetic (the kernel is L2-latency bound). The parameters and
    // moments were written by the previous step's coefficient grid, which
    // completed before the points grid passed its own wait (and, in 2D, let
    // this grid be scheduled): the first round's p / m / v loads are issued
    // before this grid's wait and overlap the points grid; the accumulator
    // (being reduced into by the points grid) is read after it.
    constexpr int R = 4;
    float pv[R], pn[R][2 * DIM], pg[R], mi[R], vi[R];
    unsigned nb[R];  // neighbour present: bit 2a = v+e_a, bit 2a+1 = v-e_a
    auto load_round = [&](int base) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int idx = base + r * nthr;
            const int j = idx < A.nc ? idx : 0;
            const int vtx = j / K;
            const int g3[3] = {vtx % r0, DIM == 3 ? (vtx / r0) % r1 : vtx / r0, DIM == 3 ? vtx / (r0 * r1) : 0};
            nb[r] = 0;
#pragma unroll
            for (int a = 0; a < DIM; ++a) {
                const bool hi = A.want_tv && g3[a] + 1 < A.s.res[a], lo = A.want_tv && g3[a] >= 1;
                nb[r] |= (hi ? 1u : 0u) << (2 * a) | (lo ? 1u : 0u) << (2 * a + 1);
                pn[r][2 * a] = __ldg(A.p_in + (hi ? j + offs[a] : j));
                pn[r][2 * a + 1] = __ldg(A.p_in + (lo ? j - offs[a] : j));
            }
            pv[r] = __ldg(A.p_in + j);
            mi[r] = __ldg(A.m_in + j);
            vi[r] = __ldg(A.v_in + j);
        }
    };
    auto load_acc = [&](int base) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int idx = base + r * nthr;
            pg[r] = __ldcg(A.acc + (idx < A.nc ? idx : 0));
        }
    };
    const int base0 = blockIdx.x * kSmallNT + tid;
    load_round(base0);
    // graph replay: this step's t from the device counter (advanced by the
    // previous step's finalize, complete before the points grid's wait)
    float inv_bc1 = A.inv_bc1, inv_bc2 = A.inv_bc2;
    if (A.ctr) {
        const long long t_after = A.ctr[0] + 1;
        const float2 bcv = A.bc[(t_after < kBcTab ? t_after : kBcTab) - 1];
        inv_bc1 = bcv.x;
        inv_bc2 = bcv.y;
    }
    pdl_wait();  // every point's reductions have landed in L2
    pdl_trigger();
    if (A.st->error) return;
    TGCU_SRING(2, atomicMin)
    double tv_sum = 0.0;
    {
        const float c1 = A.c1, c2 = A.c2, lr_bc1 = A.lr * inv_bc1;
        for (int base = base0; base < A.nc; base += R * nthr) {
            if (base != base0) load_round(base);
            load_acc(base);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int idx = base + r * nthr;
                if (idx >= A.nc) break;
                float gt = 0.0f, sq = 0.0f;
#pragma unroll
                for (int a = 0; a < DIM; ++a) {
                    if (nb[r] >> (2 * a) & 1u) {  // pair (v, v+e_a)
                        const float d = pn[r][2 * a] - pv[r];
                        sq = fmaf(d, d, sq);
                        gt -= d;
                    }
                    if (nb[r] >> (2 * a + 1) & 1u) gt += pv[r] - pn[r][2 * a + 1];  // pair (v-e_a, v)
                }
                __stcg(A.acc + idx, 0.0f);
                const float gi = fmaf(A.tv_gscale, gt, pg[r]);
                if constexpr (EXPORT) A.grad_out[idx] = gi;
                if (!isfinite(gi)) atomicMin(&A.st->bad_grad, (unsigned long long)idx);
                const float mn = fmaf(A.b1, mi[r], c1 * gi);
                const float vn = fmaf(A.b2, vi[r], c2 * gi * gi);
                A.m_out[idx] = mn;
                A.v_out[idx] = vn;
                A.p_out[idx] = pv[r] - lr_bc1 * mn * fast_rcp(fast_sqrt(vn * inv_bc2) + A.eps);
                tv_sum += (double)sq;
            }
        }
    }
    // per-CTA TV partial; the last CTA to finish reduces all partials (the
    // points kernel's first, then these, in CTA order) and commits
    block_partials(red, 0.0, 0.0, tv_sum, 0.0, A.partials + 4 * (A.ncta_pts + blockIdx.x));
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        last = atomicAdd(A.ticket, 1u) == gridDim.x - 1;
        if (last) *A.ticket = 0u;  // every CTA has taken its ticket
    }
    __syncthreads();
    if (last) {
        __threadfence();
        finalize_body<kSmallNT>(A.F, red, tid);
    }
    TGCU_SRING(3, atomicMax)
}

bool small_step_eligible(const Grid& g, int64_t n) {
    if (g.slab || g.deterministic) return false;
    if (g.NC >= (int64_t)INT_MAX || n >= (int64_t)INT_MAX) return false;
    if (g.step_path == 1) return false;
    if (g.step_path == 2) return true;
    // auto: grids of up to 3 M coefficients (their state stays in L2). The
    // crossover measured (tools/small_ab.py, us per step, small vs brick):
    // 2D 128^2 12.6/22.9, 256^2 15.6/28.1, 512^2 2^18 points 45.3/41.2,
    // 512^2 2^20 89.2/96.7, 1024^2 2^20 173.6/128.2; 3D 48^3 53.8/85.0,
    // 64^3 106.4/118.4, 64^3 2^20 points 260.5/486.4, 96^3 272.2/101.7.
    return g.NC <= kSmallMaxCoeffs && n <= kSmallMaxPoints;
}

static int sm_count(int device) {
    static int cnt[64] = {};
    int& c = cnt[device & 63];
    if (!c) TGCU_CUDA(cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, device));
    return c;
}

// CTA counts of the two kernels for a batch of n points.
static void small_grid_dims(const Grid& g, int64_t n, int* np, int* nq) {
    const int sms = sm_count(g.device);
    static const int pcap = [] {  // TGCU_SMALL_PCTAS: A/B knob, read once
        const char* ev = std::getenv("TGCU_SMALL_PCTAS");
        return ev ? std::max(1, std::atoi(ev)) : 8192;
    }();
    static const int qcap_env = [] {  // TGCU_SMALL_QCTAS: A/B knob, read once
        const char* ev = std::getenv("TGCU_SMALL_QCTAS");
        return ev ? std::max(1, std::atoi(ev)) : 0;
    }();
    // points: one sweep (C1, a thread per point: 256 CTAs 5.6 us; 148 CTAs
    // with two points per thread 13 us); coefficients: one CTA per SM at most
    // (rounds of 4 per thread; 222-384 CTAs measured slower at C1)
    const int lanes = g.spec.dim == 3 ? SmallLanes<3>::P : SmallLanes<2>::P;  // lanes per point
    *np = (int)std::max<int64_t>(1, std::min<int64_t>(pcap, (n * lanes + kSmallNT - 1) / kSmallNT));
    const int qcap = qcap_env ? qcap_env : sms;
    *nq = (int)std::max<int64_t>(1, std::min<int64_t>(qcap, (g.NC + kSmallNT - 1) / kSmallNT));
}

// Device buffers of the small-grid step (before a graph capture, where
// allocation is not allowed): the accumulator, the partials + CTA ticket.
static void ensure_small_buffers(Grid& g, int np, int nq, cudaStream_t s) {
    if (!g.sacc) {
        TGCU_CUDA(cudaMalloc(&g.sacc, sizeof(float) * g.NC));
        TGCU_CUDA(cudaMemsetAsync(g.sacc, 0, sizeof(float) * g.NC, s));
    }
    if (g.spart_cap < 4 * (np + nq)) {
        if (g.spart) TGCU_CUDA(cudaFree(g.spart));
        g.spart_cap = 4 * (np + nq);
        TGCU_CUDA(cudaMalloc(&g.spart, sizeof(double) * (g.spart_cap + 1)));
        TGCU_CUDA(cudaMemsetAsync(g.spart + g.spart_cap, 0, sizeof(double), s));
    }
}

void launch_small_step(Grid& g, const float4* samples, int64_t n, int64_t n_norm, const tgcu_loss_config& cfg,
                       int in_idx, int64_t step, double inv_bc1, double inv_bc2, int64_t t_after, float* grad_out,
                       const BinInput& in, cudaStream_t s, bool fresh_eik, bool graph) {
    const int k = g.bin_set;  // the NaN slot of this step
    g.bin_set ^= 1;
    const bool eik = cfg.lambda1 > 0.0;
    const void* kp = nullptr;
    const void* kc = nullptr;
    TGCU_DISPATCH(g.spec.dim, g.spec.order, {
        kp = eik ? (const void*)k_small_points<DIM, ORDER, true> : (const void*)k_small_points<DIM, ORDER, false>;
        kc = grad_out ? (const void*)k_small_coeffs<DIM, ORDER, true> : (const void*)k_small_coeffs<DIM, ORDER, false>;
    });
    int np = 1, nq = 1;
    small_grid_dims(g, n, &np, &nq);
    ensure_small_buffers(g, np, nq, s);
    if (in.wait) TGCU_CUDA(cudaStreamWaitEvent(s, in.wait, 0));

    SmallArgs A{};
    A.s = g.ds;
    A.pts = samples;
    A.n = (int)n;
    A.nc = (int)g.NC;
    const int out_idx = 1 - in_idx;
    A.p_in = g.p[in_idx];
    A.p_out = g.p[out_idx];
    A.m_in = g.m[in_idx];
    A.m_out = g.m[out_idx];
    A.v_in = g.v[in_idx];
    A.v_out = g.v[out_idx];
    A.acc = g.sacc;
    A.grad_out = grad_out;
    A.L.k = cfg.k;
    A.L.inv_n = 1.0 / (double)n_norm;
    A.L.eik_scale = cfg.lambda1;
    A.L.use_weighting = cfg.use_weighting;
    A.L.differentiate_weight = cfg.differentiate_weight;
    A.L.fresh_eik = fresh_eik ? 1 : 0;
    A.want_tv = cfg.use_tv ? 1 : 0;
    A.tv_gscale = (cfg.use_tv && cfg.lambda2 > 0.0) ? (float)(2.0 * cfg.lambda2 * g.tv_inv_norm) : 0.0f;
    A.lr = (float)g.adam.lr;
    A.b1 = (float)g.adam.beta1;
    A.b2 = (float)g.adam.beta2;
    A.c1 = (float)(1.0 - g.adam.beta1);
    A.c2 = (float)(1.0 - g.adam.beta2);
    A.eps = (float)g.adam.eps;
    A.inv_bc1 = (float)inv_bc1;
    A.inv_bc2 = (float)inv_bc2;
    A.partials = g.spart;
    A.ncta_pts = np;
    A.pts_ready = (in.ready || in.wait) ? 1 : 0;
    static const int early_env = [] {  // TGCU_SMALL_EARLY=0/1: A/B knob, read once
        const char* ev = std::getenv("TGCU_SMALL_EARLY");
        return ev ? std::atoi(ev) : -1;
    }();
    A.early = early_env >= 0 ? early_env : (g.spec.dim == 2 ? 1 : 0);
    A.ticket = reinterpret_cast<unsigned*>(g.spart + g.spart_cap);
    A.st = g.st;
    A.nan = &g.st->nan_bin[k];
    FinArgs& F = A.F;
    F.partials = g.spart;
    F.NB = np + nq;
    F.n = (double)n_norm;
    F.lambda1 = cfg.lambda1;
    F.lambda2 = cfg.lambda2;
    F.inv_norm = g.tv_inv_norm;
    F.use_tv = cfg.use_tv;
    F.want_eik = eik;
    F.st = g.st;
    F.nan = &g.st->nan_bin[k];
    F.over = &g.st->det_over[k];
    F.trace = g.d_trace;
    F.step = step;
    F.in_idx = in_idx;
    F.t_after = t_after;
    F.slab_out = nullptr;
    F.reduced = nullptr;
    if (graph) {
        A.ctr = g.d_ctr;
        A.bc = reinterpret_cast<const float2*>(g.d_bc);
        F.ctr = g.d_ctr;
    }

    g.prof_this = g.prof_on && (g.steps_launched % g.prof_every) == 0;
    if (g.prof_this) prof_mark(g, s, 0);
    void* args[] = {&A};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t lc{};
    lc.blockDim = dim3(kSmallNT);
    lc.dynamicSmemBytes = 0;
    lc.stream = s;
    lc.attrs = at;
    lc.numAttrs = g.small_pdl ? 1 : 0;
    lc.gridDim = dim3((unsigned)np);
    TGCU_CUDA(cudaLaunchKernelExC(&lc, kp, args));
    lc.gridDim = dim3((unsigned)nq);
    TGCU_CUDA(cudaLaunchKernelExC(&lc, kc, args));
    if (g.prof_this) prof_mark(g, s, 1);
    if (in.consumed) TGCU_CUDA(cudaEventRecord(in.consumed, s));
    count_launch(2);
}

// Counter reset of graph-replayed steps: {t, step} = the host's state.
__global__ void k_set_ctr(long long* ctr, long long t, long long step) {
    ctr[0] = t;
    ctr[1] = step;
}

}  // namespace tgcu

struct tgcu_graph {
    tgcu_grid* h = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int nsteps = 0;
    int cur0 = 0;  // ping-pong slot at capture (and at every replay: nsteps is even)
};

extern "C" int tgcu_train_graph_destroy(tgcu_graph* gr);

extern "C" int tgcu_train_graph_create(tgcu_grid* h, const float* const* samples, int nsteps, int64_t n,
                                       const tgcu_loss_config* cfg, void* stream, tgcu_graph** out) {
    using namespace tgcu;
    return guard([&] {
        require(h != nullptr && out != nullptr && samples != nullptr, "train_graph_create: NULL argument");
        require(cfg != nullptr, "total_loss: NULL config");
        require(cfg->lambda1 >= 0.0 && cfg->lambda2 >= 0.0, "LossConfig: lambda weights must be >= 0");
        require(cfg->k > 0.0, "LossConfig: weight sharpness k must be > 0");
        require(n > 0, "total_loss: empty batch");
        require(nsteps >= 2 && nsteps % 2 == 0,
                "train_graph_create: nsteps must be even and >= 2 (each replay returns to the captured ping-pong slot)");
        for (int i = 0; i < nsteps; ++i) require(samples[i] != nullptr, "train_graph_create: NULL batch");
        Grid& g = h->g;
        TGCU_CUDA(cudaSetDevice(g.device));
        require(small_step_eligible(g, n),
                "train_graph_create: only the small-grid step path can be captured (tgcu_grid_set_step_path)");
        // flush queued work and report a pending error before capturing
        const int rc = tgcu_sync(h, nullptr);
        if (rc != TGCU_OK) throw Error(rc, tgcu_last_error());
        ensure_optimizer(g);
        cudaStream_t s = as_stream(stream);
        require(s != nullptr, "train_graph_create: capture needs a non-default stream");
        if (!g.d_ctr) {
            TGCU_CUDA(cudaMalloc(&g.d_ctr, 2 * sizeof(long long)));
            std::vector<float> bc(2 * kBcTab);
            for (int t = 1; t <= kBcTab; ++t) {  // launch_train_step's values (api.cu)
                bc[2 * (t - 1)] = (float)(1.0 / (1.0 - std::pow(g.adam.beta1, (double)t)));
                bc[2 * (t - 1) + 1] = (float)(1.0 / (1.0 - std::pow(g.adam.beta2, (double)t)));
            }
            TGCU_CUDA(cudaMalloc(&g.d_bc, sizeof(float) * bc.size()));
            TGCU_CUDA(cudaMemcpy(g.d_bc, bc.data(), sizeof(float) * bc.size(), cudaMemcpyHostToDevice));
            g.ctr_t = g.ctr_step = -1;
        }
        int np = 1, nq = 1;
        small_grid_dims(g, n, &np, &nq);
        ensure_small_buffers(g, np, nq, s);
        TGCU_CUDA(cudaStreamSynchronize(s));
        auto* gr = new tgcu_graph;
        gr->h = h;
        gr->nsteps = nsteps;
        gr->cur0 = g.cur;
        const bool prof = g.prof_on;
        const int bin_set = g.bin_set;
        g.prof_on = false;
        BinInput in;
        in.ready = true;  // the batches' contents are the caller's to order before each replay
        TGCU_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        try {
            int cur = g.cur;
            for (int i = 0; i < nsteps; ++i) {
                launch_small_step(g, reinterpret_cast<const float4*>(samples[i]), n, n, *cfg, cur, 0, 0.0, 0.0, 0,
                                  nullptr, in, s, false, true);
                cur = 1 - cur;
            }
        } catch (...) {
            cudaGraph_t junk = nullptr;
            cudaStreamEndCapture(s, &junk);
            if (junk) cudaGraphDestroy(junk);
            g.prof_on = prof;
            g.bin_set = bin_set;
            delete gr;
            throw;
        }
        g.prof_on = prof;
        g.bin_set = bin_set;
        count_launch(-2 * nsteps);  // captured, not launched (counted per replay)
        cudaError_t e = cudaStreamEndCapture(s, &gr->graph);
        if (e == cudaSuccess) e = cudaGraphInstantiate(&gr->exec, gr->graph, 0);
        if (e != cudaSuccess) {
            tgcu_train_graph_destroy(gr);
            throw Error(TGCU_ERR_CUDA, std::string("train_graph_create: ") + cudaGetErrorString(e));
        }
        *out = gr;
    });
}

extern "C" int tgcu_train_graph_launch(tgcu_graph* gr, void* stream) {
    using namespace tgcu;
    return guard([&] {
        require(gr != nullptr, "train_graph_launch: NULL graph");
        Grid& g = gr->h->g;
        TGCU_CUDA(cudaSetDevice(g.device));
        require(g.cur == gr->cur0, "train_graph_launch: the grid's current ping-pong slot (" + std::to_string(g.cur) +
                                       ") is not the one captured (" + std::to_string(gr->cur0) +
                                       "): an odd number of steps ran since the capture");
        cudaStream_t s = as_stream(stream);
        if (g.ctr_t != g.t || g.ctr_step != g.steps_launched) {  // steps ran outside the graph, or an error reset
            k_set_ctr<<<1, 1, 0, s>>>(g.d_ctr, g.t, g.steps_launched);
            TGCU_CUDA(cudaGetLastError());
            count_launch(1);
        }
        TGCU_CUDA(cudaGraphLaunch(gr->exec, s));
        count_launch(2 * gr->nsteps);
        // optimistic, as tgcu_train_step: a failed step is rolled back by tgcu_sync
        g.t += gr->nsteps;
        g.steps_launched += gr->nsteps;
        g.ctr_t = g.t;
        g.ctr_step = g.steps_launched;
    });
}

extern "C" int tgcu_train_graph_destroy(tgcu_graph* gr) {
    if (!gr) return TGCU_OK;
    if (gr->exec) cudaGraphExecDestroy(gr->exec);
    if (gr->graph) cudaGraphDestroy(gr->graph);
    delete gr;
    return TGCU_OK;
}

#ifdef TGCU_PHASE_TIMING
extern "C" int tgcu_small_ring_dump(unsigned long long* out, int reset) {
    if (reset) {
        static unsigned long long init[256 * 4];
        for (int i = 0; i < 256; ++i) {
            init[4 * i] = init[4 * i + 2] = ~0ull;
            init[4 * i + 1] = init[4 * i + 3] = 0ull;
        }
        return cudaMemcpyToSymbol(tgcu::g_sring, init, sizeof(init)) == cudaSuccess ? 0 : 6;
    }
    return cudaMemcpyFromSymbol(out, tgcu::g_sring, sizeof(unsigned long long) * 1024) == cudaSuccess ? 0 : 6;
}
#endif
