// Host-side internals of libtgcu: the grid handle, error plumbing and the
// kernel launchers each .cu file provides.
#pragma once

#include <cuda.h>  // CUtensorMap (header only; the encoder is fetched through the runtime)
#include <cuda_runtime.h>

#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tgcu.h"
#include "tg_device.cuh"

namespace tgcu {

// Exception carrying a TGCU_* status class; converted to a return code at the
// C boundary (api.cu).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void require(bool cond, const std::string& msg) {
    if (!cond) throw Error(TGCU_ERR_INVALID_ARGUMENT, msg);
}

#define TGCU_CUDA(expr)                                                                         \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess)                                                                  \
            throw ::tgcu::Error(TGCU_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
    } while (0)

void count_launch(int n = 1);

// C-boundary error plumbing (api.cu): records the thread-local message read by
// tgcu_last_error() and returns the status code.
int set_err(int code, const std::string& m);

template <class F>
int guard(F&& f) {
    try {
        f();
        return TGCU_OK;
    } catch (const Error& e) {
        return set_err(e.code, e.what());
    } catch (const std::bad_alloc& e) {
        return set_err(TGCU_ERR_RESOURCE, e.what());
    } catch (const std::exception& e) {
        return set_err(TGCU_ERR_CUDA, e.what());
    }
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// GridSpec::validate (grid_spec.cpp:21-33) + coeff_count ranges; throws Error.
void validate_spec(const tgcu_grid_spec& s);
int coeff_count_of(int order, int dim);
// Device geometry of a full (non-slab) grid spec.
DevSpec make_devspec(const tgcu_grid_spec& s);

// Brick edge (vertices per axis) of the fused training kernel and the
// brick-binned query.
constexpr int kBrick3 = 8;
// z extent of the fused training kernel's 3D brick (vertex planes; x and y
// are kBrick3). Slab grids are cut into layers of this many planes (slab.py
// BRICK follows the default). A/B switch: half-depth bricks (4) with m, v in
// HBM (TGCU_MV_GLOBAL) fit 4 CTAs per SM but measured 12 % slower at C2
// (DESIGN.md §3.1).
#ifndef TGCU_BRICKZ3
#define TGCU_BRICKZ3 8
#endif
constexpr int kBrickZ3 = TGCU_BRICKZ3;
// 3D fused step with m and v read and written in HBM by the epilogue (L2
// prefetch at the CTA's start) instead of staged in shared memory: half-depth
// bricks then fit 4 CTAs per SM.
#ifndef TGCU_MV_GLOBAL
#define TGCU_MV_GLOBAL (TGCU_BRICKZ3 < 8)
#endif
#ifndef TGCU_BRICK2
#define TGCU_BRICK2 16
#endif
constexpr int kBrick2 = TGCU_BRICK2;

struct Grid {
    tgcu_grid_spec spec{};
    int K = 0;
    int64_t V = 0;   // vertices
    int64_t NC = 0;  // coefficients = V*K
    int device = 0;
    DevSpec ds{};

    // Ping-pong parameter / moment buffers (fused step writes the other one).
    float* p[2] = {nullptr, nullptr};
    float* m[2] = {nullptr, nullptr};
    float* v[2] = {nullptr, nullptr};
    int cur = 0;
    float* grad = nullptr;  // unfused-API gradient buffer (lazy)

    tgcu_adam_config adam{0.003, 0.9, 0.999, 1e-8};
    int64_t t = 0;              // AdamState::t (host mirror, optimistic under async)
    int64_t steps_launched = 0; // fused steps issued

    Status* st = nullptr;     // device status
    Status* st_host = nullptr;  // pinned mirror

    // Bricks of the fused step / binned query.
    // Slab grids (multi-GPU z partition): brick layers [zb0, zb0 + nb[2]) of
    // the global grid spec; stored vertex planes [ds.zoff, ds.zoff + ds.zstore).
    bool slab = false;
    int zb0 = 0;
    int zb_global = 0;            // brick layers of the global grid
    int code_sh[2] = {0, 0};      // bit offsets of y / z in a binning brick code
    double tv_inv_norm = 0.0;     // 1 / (P*K) of the global grid
    double* slab_red = nullptr;   // 8 doubles: local sums of the pending slab step
    int slab_in_idx = 0;
    // Fused halo (tgcu_slab_ipc_import / tgcu_slab_set_peer_planes): the
    // neighbours' halo planes, per ping-pong slot, written by the brick kernel.
    float* peer_lo[2] = {nullptr, nullptr};
    float* peer_hi[2] = {nullptr, nullptr};
    std::vector<void*> ipc_open;  // bases opened with cudaIpcOpenMemHandle
    int64_t slab_step = 0, slab_t_after = 0, slab_n = 0;
    tgcu_loss_config slab_cfg{};
    int brick[3] = {1, 1, 1};
    int nb[3] = {1, 1, 1};
    int64_t NB = 1;
    // Point binning of the fused step. Two bin sets (offsets + binned
    // points) alternate between steps so the binning of step i+1 can run on
    // the binning stream while step i's brick kernel still reads set i&1;
    // the histogram / code / chain scratch is only touched by binning
    // kernels, which are serial on that stream.
    int* bin_count = nullptr;   // NB + 1 (fallback binning)
    int* bin_off[2] = {nullptr, nullptr};  // NB + 1 per set
    int* brick_order[2] = {nullptr, nullptr};  // NB per set: launch order of the bricks
    int* bin_cursor = nullptr;  // NB (fallback binning)
    int* bin_hist = nullptr;    // per-tile brick histograms (privatized binning)
    int64_t bin_hist_cap = 0;
    int* bin_codes = nullptr;   // per-point brick code
    int64_t bin_codes_cap = 0;
    int* bin_chain = nullptr;   // chained-scan flags/prefixes (2 ints per CTA)
    int64_t bin_chain_cap = 0;
    int bin_epoch = 0;
    float4* binned[2] = {nullptr, nullptr};
    int64_t binned_cap[2] = {0, 0};  // points
    int bin_set = 0;                 // set of the next step
    int slab_set = 0;                // set of the pending slab step
    cudaStream_t bstream = nullptr;  // binning stream
    cudaEvent_t ev_in = nullptr;     // caller stream -> binning stream (input order)
    cudaEvent_t ev_bdone[2] = {nullptr, nullptr}, ev_bfree[2] = {nullptr, nullptr};
    double* partials = nullptr; // NB * 4
    double* fin_l2 = nullptr;   // multi-CTA finalize: 148 level-2 records (4 doubles) + its ticket
    tgcu_loss_terms* d_trace = nullptr;  // kTraceCap
    tgcu_loss_terms* h_terms = nullptr;  // pinned, 1
    float* staging = nullptr;            // device staging for host inputs
    int64_t staging_cap = 0;             // floats
    // Pipelined host inputs (TGCU_HOST | TGCU_ASYNC train steps): a copy
    // stream filling two device slots, ordered against the compute stream by
    // events, and a pinned ring receiving each step's LossTerms.
    // Two copy streams, each moving half of a step's samples: one pinned H2D
    // copy gets 25-42 GB/s depending on the box, two concurrent halves ~54
    // GB/s (tools/h2d_bw.py).
    cudaStream_t cstream = nullptr, cstream2 = nullptr;
    cudaEvent_t ev_ready[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
    cudaEvent_t ev_half[2] = {nullptr, nullptr};
    float* pstage[2] = {nullptr, nullptr};
    int64_t pstage_cap = 0;              // floats per slot
    int pipe_slot = 0;
    tgcu_loss_terms* h_ring = nullptr;   // pinned, kTraceCap
    double* scratch_d = nullptr;         // reductions (unfused path)
    int64_t scratch_cap = 0;
    // TMA tensor maps of the fused step (train.cu ensure_tmaps): per ping-pong
    // slot, the parameter tile box (B+2)^D x K, and the owned box B^D x K of
    // p, m and v. tm_state: 0 = not built, 1 = usable, -1 = layout not eligible.
    CUtensorMap tm_tile[2], tm_own_p[2], tm_own_m[2], tm_own_v[2];
    int tm_state = 0;
    // Query tile boxes ((B+1)^D vertices) over p[0], p[1] (query.cu).
    CUtensorMap tm_query[2];
    int tmq_state = 0;
    // Live kernel timing (tgcu_profile_*): CUDA events recorded on the launch
    // stream around the fused brick kernel.
    bool prof_on = false;
    int prof_every = 1;          // time every n-th brick launch
    bool prof_this = false;      // the current launch is timed
    std::vector<cudaEvent_t> prof_ev;  // pairs (start, end)
    size_t prof_used = 0;
    // Step breakdown (tgcu_step_breakdown, diagnostics): events at the
    // boundaries of one fused step, summed per segment after each step.
    bool bd_on = false;
    bool deterministic = false;  // canonical summation orders (tgcu_grid_set_deterministic)
    // Fused-step path (tgcu_grid_set_step_path / TGCU_STEP_PATH): 0 auto,
    // 1 brick kernel (train.cu), 2 small-grid path (small.cu).
    int step_path = 0;
    float* sacc = nullptr;       // small-grid step: fp32 gradient accumulator (NC, zero between steps)
    double* spart = nullptr;     // small-grid step: per-CTA loss partials + CTA ticket
    int spart_cap = 0;           // doubles
    // Graph-replayed small-grid steps (tgcu_train_graph_*): {t, step} on the
    // device, advanced by each step's finalize; the bias-correction table; the
    // counter values the device holds after the last replay (-1: unknown).
    long long* d_ctr = nullptr;
    float* d_bc = nullptr;
    long long ctr_t = -1, ctr_step = -1;
    bool brick_pdl = true;       // brick path: brick kernel and finalize chained by PDL (TGCU_BRICK_PDL=0 off)
    bool small_pdl = true;       // small-grid step: programmatic dependent launch (TGCU_SMALL_PDL=0 off)
    cudaEvent_t bd_ev[6] = {};
    double bd_sum[5] = {0, 0, 0, 0, 0};
    int bd_steps = 0;
};

void prof_mark(Grid& g, cudaStream_t s, int which);
void bd_mark(Grid& g, cudaStream_t s, int i);  // step breakdown boundary i (0..5)
void bd_collect(Grid& g);                       // after a step: add its segment times

constexpr int kTraceCap = 4096;

// TMA tensor map over a coefficient-layout buffer: rows of K*res_x floats x
// res_y [x stored z planes], box box_x floats x box_y [x box_z, default box_y] (train.cu).
bool encode_grid_map(CUtensorMap* m, const Grid& g, const float* base, unsigned box_x, unsigned box_y,
                     unsigned box_z = 0);
void ensure_staging(Grid& g, int64_t floats);
void ensure_pipeline(Grid& g, int64_t floats);
void ensure_bins(Grid& g, int set, int64_t points);
void ensure_bin_stream(Grid& g);
void ensure_bin_hist(Grid& g, int64_t ints, int64_t points, int64_t chain_ctas);
void ensure_scratch(Grid& g, int64_t doubles);
void ensure_grad(Grid& g);
void ensure_optimizer(Grid& g);

// Launchers (query.cu / train.cu). All stream-ordered; no synchronisation.
void launch_eval_direct(Grid& g, const float* pts, int64_t n, float* vals, float* grads, cudaStream_t s);
// Unsorted batches of at least kBinnedQueryMin points: counting sort by query
// brick + the smem-tile brick kernel writing values to the caller's slots.
constexpr int64_t kBinnedQueryMin = 1 << 18;
void launch_eval_binned(Grid& g, const float* pts, int64_t n, float* vals, float* grads, cudaStream_t s);
// Lattice values on the brick tiles when the lattice is dense enough (about
// >= 128 points per brick); false = not taken (caller uses the row kernel).
// fac / cell: per-axis tables of k_axis_table (stages.cu), n: lattice size.
bool launch_eval_lattice_brick(Grid& g, const float4* fac, const int* cell, int3 n, float* vals, cudaStream_t s);
void launch_eval_sorted(Grid& g, const float* pts, int64_t n, const int64_t* offsets, float* vals, float* grads,
                        cudaStream_t s);
void launch_sort_points(Grid& g, const float* pts, int64_t n, float* out, int64_t* perm, int64_t* offsets,
                        cudaStream_t s);
int64_t query_brick_codes(const Grid& g);
void launch_backprop(Grid& g, const float* pts, const float* up, const float* upv, int64_t n, float* grad,
                     cudaStream_t s);
// Unfused total_loss pieces: point terms (atomic scatter) + TV; sums land in
// g.scratch_d[0..2] = {recon, eik, tv_sum}.
void launch_point_terms(Grid& g, const float4* samples, int64_t n, const tgcu_loss_config& cfg, float* grad,
                        cudaStream_t s,
                        double upstream_scale = 1.0, bool eik_points = false);
void launch_tv(Grid& g, const float* coeffs, float* grad, double gscale, int want_value, cudaStream_t s);
void launch_adam_check(Grid& g, const float* grad, cudaStream_t s);
void launch_adam_update(Grid& g, const float* grad, double inv_bc1, double inv_bc2, cudaStream_t s);
// How the binning stream orders its reads of a step's samples:
//  wait     - an event marking the samples complete (pipelined host copy), or
//  ready    - the caller asserts the samples are complete (TGCU_INPUT_READY),
//  neither  - after all work issued so far on the caller's stream.
// consumed (optional) is recorded once binning has read the samples.
struct BinInput {
    cudaEvent_t wait = nullptr;
    bool ready = false;
    cudaEvent_t consumed = nullptr;
};
// Fused step: binning (binning stream) + brick kernel + finalize (caller's
// stream) (train.cu).
void launch_train_step(Grid& g, const float4* samples, int64_t n, int64_t n_norm, const tgcu_loss_config& cfg,
                       int in_idx,
                       int64_t step, double inv_bc1, double inv_bc2, int64_t t_after, float* grad_out,
                       double* slab_out, const BinInput& in, cudaStream_t s, bool fresh_eik = false);
// Two-launch fused step for small grids (small.cu): the auto rule's
// limits (coefficients, points per step) and the launcher, same arguments as
// launch_train_step without the slab phase.
constexpr int64_t kSmallMaxCoeffs = int64_t(3) << 20;
constexpr int64_t kSmallMaxPoints = int64_t(1) << 22;
bool small_step_eligible(const Grid& g, int64_t n);
void launch_small_step(Grid& g, const float4* samples, int64_t n, int64_t n_norm, const tgcu_loss_config& cfg,
                       int in_idx, int64_t step, double inv_bc1, double inv_bc2, int64_t t_after, float* grad_out,
                       const BinInput& in, cudaStream_t s, bool fresh_eik, bool graph = false);
// Fresh-uniform eikonal points (n x 3 floats, device) -> float4 records with
// gt = kEikMark (tg_device.cuh), for the fused step's point list.
void launch_pack_eik(const float* p3, int64_t n, float4* dst, cudaStream_t s);
void launch_slab_finish(Grid& g, const double* reduced, const tgcu_loss_config& cfg, int in_idx, int64_t step,
                        int64_t t_after, int64_t n, cudaStream_t s);
void launch_f64_to_f32(const double* src, float* dst, int64_t n, cudaStream_t s);
void launch_f32_to_f64(const float* src, double* dst, int64_t n, cudaStream_t s);
void launch_all_finite(const float* src, int64_t n, unsigned long long* flag, cudaStream_t s);
void launch_fill_f0(Grid& g, float* dst, float value, cudaStream_t s);
void launch_rays(Grid& g, const DevSpec& ss, int deg, const float* scoeffs, const float* rays, const float* gt,
                 int64_t n, const tgcu_render_options& o, float* colors, float* resid, float* gd, float* gsh,
                 double* ray_err, double* loss, cudaStream_t s);
void launch_hash_gaussian(float* dst, int64_t n, uint64_t seed, double sigma, int64_t goff, cudaStream_t s);
void launch_hash_points(float* out, int64_t n, int dim, uint64_t seed, double lo, double hi, cudaStream_t s);
void launch_draw_batch(const float* pool, int64_t pool_n, int64_t n, uint64_t seed, uint64_t step, float* out,
                       cudaStream_t s);

}  // namespace tgcu

struct tgcu_grid {
    tgcu::Grid g;
    tgcu_comm* comm = nullptr;  // slab grids: the job's communicator (tgcu_slab_connect, comm.cu)
    bool fused_halo = false;    // boundary planes stored into the neighbours by the brick kernel
    // collective phase of profiled slab steps (all-reduce + halo exchange), event pairs
    std::vector<cudaEvent_t> coll_ev;
    size_t coll_used = 0;
};
