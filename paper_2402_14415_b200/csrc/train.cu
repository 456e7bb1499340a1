// Fused training step: zero grad → total_loss (recon + eikonal + TV) →
// finite checks → Adam, i.e. one iteration of run_schedule
// (schedule.cpp:66-92) / cmd_bench (tools/main.cpp:640-644), as one device
// pipeline with the gradient never materialised in HBM.
//
// Design ("owner computes", SURVEY §8a K2+K3):
//   The vertex grid is cut into bricks of B^D vertices (B = 8 in 3D, 16 in
//   2D). The CTA of brick b owns its vertices' Adam state and needs every
//   point whose cell touches an owned vertex: the cells [B*b-1, B*b+B-1] per
//   axis. Points are binned by brick with a counting sort; a point lying in
//   the last cell layer of a brick is also copied to the next brick (1..2^D
//   copies, 1.42x on average for uniform points).
//   Per CTA:
//     1. stage the (B+2)^D vertex tile of the current parameters in smem
//        (owned vertices + one-vertex halo: the cells' corners and the TV
//        stencil neighbours);
//     2. per chunk of points: fp64 locate and a counting sort of the chunk
//        by cell in smem (cell runs reserved per warp), then the forward eval
//        from the tile (fp32 blend) and the loss chain, each point's record
//        written straight into its cell's run; each owned-vertex thread then
//        gathers the contributions of the points in its 2^D incident cells
//        into K register accumulators (no global atomics);
//     3. TV gradient from the tile stencil + Adam over the owned
//        coefficients, reading m/v and writing p/m/v to the other ping-pong
//        buffers (coalesced rows), plus the per-brick loss partials.
//   The binning of a step runs on a library stream into one of two bin sets,
//   so it overlaps the previous step's brick kernel (launch_train_step).
//   A 1-CTA finalize kernel reduces the partials in a fixed order, applies the
//   reference's error order (NaN point, non-finite loss, non-finite gradient)
//   and commits the step by naming the new current buffer; a failed step
//   leaves the old buffers current and makes every later step a no-op until
//   the host reads the sticky error.
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

#include <atomic>
#include <climits>
#include <cstdlib>

#include "dispatch.cuh"
#include "tg_internal.h"

#ifndef TGCU_TV_SHFL
#define TGCU_TV_SHFL 1
#endif
#include "tma.cuh"
#include "finalize.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace tgcu {

template <int DIM>
struct BrickShape {
    static constexpr int B = DIM == 3 ? kBrick3 : kBrick2;   // x and y extent (vertices)
    static constexpr int BZ = DIM == 3 ? kBrickZ3 : 1;       // z extent (3D)
    static constexpr int T = B + 2;   // tile edge (vertices), x and y
    static constexpr int TZ = BZ + 2;  // tile depth (3D)
    static constexpr int CE = B + 1;  // cells per axis touching owned vertices (the cell index strides)
    static constexpr int NCELL = DIM == 3 ? CE * CE * (BZ + 1) : CE * CE;
    static constexpr int TVN = DIM == 3 ? T * T * TZ : T * T;
    static constexpr int NOWN = DIM == 3 ? B * B * BZ : B * B;
    static constexpr bool MVG = DIM == 3 && TGCU_MV_GLOBAL;  // m, v not staged in shared memory
    static constexpr int NT = NOWN;   // one thread per owned vertex
    static constexpr int CH = NT;     // points per chunk
    static constexpr int REC = 8;     // floats per point record
};

struct BinArgs {
    DevSpec s;
    const float4* pts;
    long long n;
    int nb[3];
    int* count;
    int* cursor;
    float4* binned;
    unsigned long long* nan;  // the bin set's NaN slot (Status::nan_bin)
    int zb0;  // first brick layer (slab grids)
    int sh1, sh2;  // bit offsets of the y and z brick coordinates in a brick code (brick_code_shifts)
};

// Brick code of a point: its cell's brick coordinates (x in bits [0, sh1),
// y in [sh1, sh2), z from sh2 up; widths sized per grid by brick_code_shifts
// so any grid whose brick count fits 2^27 packs without overlap) and the
// per-axis "also the next brick" mask (bits 27..29), or -1 for a NaN
// coordinate. Brick coordinates are global; code_bricks() maps them to this
// grid's brick indices, dropping bricks outside a slab grid's layers.
template <int DIM>
__device__ __forceinline__ int point_brick_code(const DevSpec& s, const BinArgs& A, const float4& q) {
    const float pf[3] = {q.x, q.y, q.z};
    int lo[3] = {0, 0, 0}, mask = 0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        const int B = a == 2 ? BrickShape<DIM>::BZ : BrickShape<DIM>::B;
        const double x = (double)pf[a];
        if (isnan(x)) return -1;
        double local;
        const int c = locate_axis(s, a, x, local);
        lo[a] = c / B;
        mask |= ((c % B) == B - 1 ? 1 : 0) << a;
    }
    return lo[0] | (lo[1] << A.sh1) | (lo[2] << A.sh2) | (mask << 27);
}

template <int DIM>
__device__ __forceinline__ int code_bricks(int code, const BinArgs& A, int* out) {
    const int* nb = A.nb;
    const int zb0 = A.zb0;
    const int bx = code & ((1 << A.sh1) - 1), by = (code >> A.sh1) & ((1 << (A.sh2 - A.sh1)) - 1),
              bz = (code >> A.sh2) & ((1 << (27 - A.sh2)) - 1), mask = code >> 27;
    int m = 0;
    for (int dz = 0; dz <= (DIM == 3 ? (mask >> 2) & 1 : 0); ++dz) {
        const int lz = bz + dz - zb0;
        if (DIM == 3 && (lz < 0 || lz >= nb[2])) continue;
        for (int dy = 0; dy <= ((mask >> 1) & 1); ++dy)
            for (int dx = 0; dx <= (mask & 1); ++dx)
                out[m++] = ((DIM == 3 ? lz * nb[1] : 0) + by + dy) * nb[0] + bx + dx;
    }
    return m;
}

template <int DIM>
__global__ void __launch_bounds__(256) k_bin_count(BinArgs A) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < A.n;
         i += (long long)gridDim.x * blockDim.x) {
        const int code = point_brick_code<DIM>(A.s, A, A.pts[i]);
        if (code < 0) {
            atomicMin(A.nan, (unsigned long long)i);
            continue;
        }
        int br[8];
        const int m = code_bricks<DIM>(code, A, br);
        for (int k = 0; k < m; ++k) atomicAdd(&A.count[br[k]], 1);
    }
}

// Launch order of the bricks: those with more than one chunk of points first
// (they take 4-7x as long, so the kernel should not end on one), the rest
// after them. ord[NB], ord[NB + 1] count the two classes (zeroed per step);
// one atomic per warp and class.
// The brick kernel reads its brick and point range as one 16-byte record
// (info = int4 (brick, first, end, 0) per launch slot, after the NB + 2 ints).
__device__ __forceinline__ int4* order_info(int* ord, int NB) {
    return reinterpret_cast<int4*>(ord + ((NB + 2 + 3) & ~3));
}
__device__ __forceinline__ void place_brick(int brick, bool valid, int count, int ch, int NB, int* __restrict__ ord,
                                            int first) {
    const int lane = threadIdx.x & 31;
    const bool heavy = valid && count > ch, light = valid && count <= ch;
    const unsigned mh = __ballot_sync(0xffffffffu, heavy), ml = __ballot_sync(0xffffffffu, light);
    int bh = 0, bl = 0;
    if (lane == 0) {
        if (mh) bh = atomicAdd(&ord[NB], __popc(mh));
        if (ml) bl = atomicAdd(&ord[NB + 1], __popc(ml));
    }
    bh = __shfl_sync(0xffffffffu, bh, 0);
    bl = __shfl_sync(0xffffffffu, bl, 0);
    const unsigned lt = (1u << lane) - 1u;
    const int slot = heavy ? bh + __popc(mh & lt) : NB - 1 - (bl + __popc(ml & lt));
    if (heavy || light) {
        ord[slot] = brick;
        order_info(ord, NB)[slot] = make_int4(brick, first, first + count, 0);
    }
}

__global__ void k_identity_order(int* __restrict__ ord, int NB) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < NB; b += gridDim.x * blockDim.x) {
        ord[b] = b;
        order_info(ord, NB)[b] = make_int4(b, 0, 0, 0);
    }
}

// Exclusive scan of NB brick counts -> off[0..NB], cursor = off. One CTA.
__global__ void __launch_bounds__(1024) k_bin_scan(const int* __restrict__ count, int* __restrict__ off,
                                                   int* __restrict__ cursor, int NB, int ch, int* __restrict__ ord) {
    __shared__ int warp_tot[32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int base = 0; base < NB; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const int c = i < NB ? count[i] : 0;
        int x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_tot[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int w = warp_tot[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            warp_tot[lane] = w;  // inclusive
        }
        __syncthreads();
        const int excl = carry + (wid ? warp_tot[wid - 1] : 0) + x - c;
        if (i < NB) {
            off[i] = excl;
            cursor[i] = excl;
        }
        place_brick(i, i < NB, c, ch, NB, ord, excl);
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = excl + c;
        __syncthreads();
    }
    if (threadIdx.x == 0) off[NB] = carry;
}

template <int DIM>
__global__ void __launch_bounds__(256) k_bin_scatter(BinArgs A) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < A.n;
         i += (long long)gridDim.x * blockDim.x) {
        const float4 q = A.pts[i];
        const int code = point_brick_code<DIM>(A.s, A, q);
        if (code < 0) continue;
        int br[8];
        const int m = code_bricks<DIM>(code, A, br);
        for (int k = 0; k < m; ++k) {
            const int slot = atomicAdd(&A.cursor[br[k]], 1);
            A.binned[slot] = q;
        }
    }
}

// ---- privatized binning (NB small enough for a shared-memory histogram) ----
// Points are cut into tiles of kBinTile; CTA c builds the brick histogram of
// tile c in shared memory (native int smem atomics), stores it as row c of
// H[ncta][NB] and records every point's brick code (base brick | axis mask).
// k_bin_cols turns H into per-(tile, brick) exclusive prefixes and computes
// the brick offsets with a chained (in-order) scan across its CTAs; the
// scatter reserves slots with shared-memory atomics only. No contended global
// atomics on hot bricks, three launches.
constexpr int kBinTile = 4096;
constexpr int kBinThreads = 512;
constexpr int kBinPer = kBinTile / kBinThreads;  // points per thread
constexpr int kBinSmemMax = 16384;  // bricks
constexpr int kColBricks = 32;
constexpr int kMaxBinTiles = 512;

template <int DIM>
__global__ void __launch_bounds__(kBinThreads) k_bin_hist(BinArgs A, int* __restrict__ H, int* __restrict__ codes,
                                                          int NB) {
    extern __shared__ int hist[];
    for (int i = threadIdx.x; i < NB; i += blockDim.x) hist[i] = 0;
    const long long t0 = (long long)blockIdx.x * kBinTile;
    float4 q[kBinPer];
#pragma unroll
    for (int k = 0; k < kBinPer; ++k) {  // all loads in flight first
        const long long i = t0 + threadIdx.x + (long long)k * kBinThreads;
        q[k] = i < A.n ? A.pts[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kBinPer; ++k) {
        const long long i = t0 + threadIdx.x + (long long)k * kBinThreads;
        if (i >= A.n) continue;
        const int code = point_brick_code<DIM>(A.s, A, q[k]);
        codes[i] = code;
        if (code < 0) {
            atomicMin(A.nan, (unsigned long long)i);
            continue;
        }
        int br[8];
        const int m = code_bricks<DIM>(code, A, br);
        for (int j = 0; j < m; ++j) atomicAdd(&hist[br[j]], 1);
    }
    __syncthreads();
    int* row = H + (long long)blockIdx.x * NB;
    for (int i = threadIdx.x; i < NB; i += blockDim.x) row[i] = hist[i];
}

// H columns -> per-(tile, brick) exclusive prefixes (in place); brick totals
// -> exclusive offsets off[0..NB] via a chained scan over the CTAs: CTA i
// publishes its aggregate, then waits for those of CTAs 0..i-1 (tagged with
// this launch's epoch). Not all CTAs need be co-resident (up to 512 CTAs of
// up to 67.5 KB of shared memory, possibly sharing the SMs with a brick
// kernel), and the CUDA model does not promise in-order dispatch, so the
// index i is a ticket taken from a launch-spanning 64-bit counter at the
// start of the CTA (ticket mod gridDim.x): a CTA only ever waits for CTAs
// that started before it, which are resident and make progress.
__global__ void __launch_bounds__(256) k_bin_cols(int* __restrict__ H, int ncta, int NB, int* __restrict__ off,
                                                  int* __restrict__ chain, unsigned long long* __restrict__ ticket,
                                                  int epoch, int chunk, int* __restrict__ ord) {
    extern __shared__ int col[];  // [ncta][kColBricks + 1]
    __shared__ int tot[kColBricks];
    __shared__ int carry;
    __shared__ int tile_s;
    if (threadIdx.x == 0) tile_s = (int)(atomicAdd(ticket, 1ull) % gridDim.x);
    __syncthreads();
    const int tile = tile_s;
    const int b0 = tile * kColBricks;
    const int nb = min(kColBricks, NB - b0);
    constexpr int LD = kColBricks + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // warp w loads rows c = w, w+8, ... (lane = brick): coalesced 128-byte rows,
    // 8 loads in flight per warp before the shared stores
    constexpr int U = 8;
    for (int cb = warp; cb < ncta; cb += 8 * U) {
        int v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = cb + 8 * u;
            v[u] = (c < ncta && lane < nb) ? H[(long long)c * NB + b0 + lane] : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = cb + 8 * u;
            if (c < ncta) col[c * LD + lane] = v[u];
        }
    }
    __syncthreads();
    const int per = (ncta + 31) / 32;
    for (int j = warp; j < kColBricks; j += 8) {
        const int c0 = min(lane * per, ncta), c1 = min(c0 + per, ncta);
        int sum = 0;
        for (int c = c0; c < c1; ++c) sum += col[c * LD + j];
        int x = sum;
#pragma unroll
        for (int o2 = 1; o2 < 32; o2 <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o2);
            if (lane >= o2) x += y;
        }
        int run = x - sum;
        for (int c = c0; c < c1; ++c) {
            const int v = col[c * LD + j];
            col[c * LD + j] = run;
            run += v;
        }
        if (lane == 31) tot[j] = x;
    }
    __syncthreads();
    for (int c = warp; c < ncta; c += 8)
        if (lane < nb) H[(long long)c * NB + b0 + lane] = col[c * LD + lane];
    if (warp == 0) {
        const int t = tot[lane];
        int x = t;
#pragma unroll
        for (int o2 = 1; o2 < 32; o2 <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o2);
            if (lane >= o2) x += y;
        }
        const int block_sum = __shfl_sync(0xffffffffu, x, 31);
        // publish this CTA's aggregate, then add up every predecessor's
        // (predecessors hold earlier tickets: already running)
        if (lane == 0) {
            chain[2 * tile + 1] = block_sum;
            __threadfence();
            atomicExch(&chain[2 * tile], epoch);
        }
        int prev = 0;
        volatile int* ch = chain;
        for (int j = lane; j < tile; j += 32) {
            while (ch[2 * j] != epoch) {
            }
            __threadfence();
            prev += ch[2 * j + 1];
        }
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) prev += __shfl_xor_sync(0xffffffffu, prev, o2);
        (void)carry;
        const int c0 = prev;
        if (lane < nb) off[b0 + lane] = c0 + x - t;
        if (tile == (int)gridDim.x - 1 && lane == 0) off[NB] = c0 + block_sum;
        place_brick(b0 + lane, lane < nb, t, chunk, NB, ord, c0 + x - t);
    }
}

template <int DIM>
__global__ void __launch_bounds__(kBinThreads) k_bin_scatter_tiles(BinArgs A, const int* __restrict__ H,
                                                                   const int* __restrict__ codes,
                                                                   const int* __restrict__ off, int NB) {
    extern __shared__ int cur[];
    const int* row = H + (long long)blockIdx.x * NB;
    for (int i = threadIdx.x; i < NB; i += blockDim.x) cur[i] = off[i] + row[i];
    const long long t0 = (long long)blockIdx.x * kBinTile;
    float4 q[kBinPer];
    int cd[kBinPer];
#pragma unroll
    for (int k = 0; k < kBinPer; ++k) {
        const long long i = t0 + threadIdx.x + (long long)k * kBinThreads;
        const bool ok = i < A.n;
        q[k] = ok ? A.pts[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        cd[k] = ok ? codes[i] : -1;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kBinPer; ++k) {
        if (cd[k] < 0) continue;
        int br[8];
        const int m = code_bricks<DIM>(cd[k], A, br);
        for (int j = 0; j < m; ++j) A.binned[atomicAdd(&cur[br[j]], 1)] = q[k];
    }
}


struct StepArgs {
    // TMA tensor maps (use_tmap): parameter tile (load), owned boxes of
    // p (store), m and v (load + store).
    CUtensorMap tm_tile, tm_p_out, tm_m_in, tm_v_in, tm_m_out, tm_v_out;
    int use_tmap;
    DevSpec s;
    const float* p_in;
    float* p_out;
    const float* m_in;
    float* m_out;
    const float* v_in;
    float* v_out;
    const float4* binned;
    const int* off;
    int nb[3];
    LossDev L;
    float tv_gscale;
    int want_tv;
    float lr, b1, b2, eps, inv_bc1, inv_bc2;
    float c1, c2;  // 1 - beta1, 1 - beta2 formed in fp64 (1 - 0.999f would be 1.3e-5 off)
    double* partials;  // NB x 4: recon, eik, tv, home points
    Status* st;
    float* grad_out;   // optional: full gradient (validation mode, TGCU_EXPORT_GRAD)
    int zb0;           // first brick layer of this grid (slab grids; 0 otherwise)
    // fused halo (slab grids): the neighbours' halo planes in the out slot;
    // the lowest owned plane is local z 0 of brick layer zb0, the highest is
    // local z peer_hi_lz of brick layer peer_hi_zb
    float* peer_lo;
    float* peer_hi;
    int peer_hi_zb, peer_hi_lz;
    const int* order;  // launch order of the bricks (1D grid): most chunks first (+ order_info)
    int NB;
    int det;           // deterministic mode: canonical record order inside every cell run
    int split;         // CTAs per brick (a thread-block cluster along x; 1 = one CTA per brick)
};

// Cell runs of a chunk's records: every cell gets the contiguous slot range
// [start, start + cnt). The runs need not be in cell order (a vertex walks its
// cells by index), so each warp scans its cells with shuffles and reserves
// its range with one shared-memory atomic: no block-wide barrier inside.
template <int NCELL, int NT>
__device__ __forceinline__ void cell_runs(const int* __restrict__ cnt, int* __restrict__ start, int* total) {
    constexpr int IT = (NCELL + NT - 1) / NT;
    const int t = threadIdx.x, lane = t & 31;
    int v[IT];
    int sum = 0;
#pragma unroll
    for (int k = 0; k < IT; ++k) {
        const int i = t * IT + k;
        v[k] = i < NCELL ? cnt[i] : 0;
        sum += v[k];
    }
    int x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    int base = 0;
    if (lane == 31 && x > 0) base = atomicAdd(total, x);
    base = __shfl_sync(0xffffffffu, base, 31);
    int excl = base + x - sum;
#pragma unroll
    for (int k = 0; k < IT; ++k) {
        const int i = t * IT + k;
        if (i < NCELL) start[i] = excl;
        excl += v[k];
    }
}

// Shared-memory plan of the fused brick kernel (one brick per CTA, 2 CTAs/SM).
// Tile rows (fixed y, z) are stored with a stride of TROWF floats and start
// SHF floats into the row, so that a row's HBM range begins 16-byte aligned
// (the reference AoS layout puts vertex o-1 at an 8-byte offset for K = 10):
// one TMA tensor box of TROWF x T [x T] floats, or one bulk copy per row.
// Regions start on 128-byte boundaries (TMA tensor smem alignment).
template <int DIM, int ORDER>
struct BrickSmem {
    using S = BrickShape<DIM>;
    static constexpr int K = KOf<DIM, ORDER>::value;
    static constexpr int SHF = (4 - (K % 4)) % 4;
    static constexpr int TROWF = ((S::T * K + SHF + 3) / 4) * 4;
    // TMA tensor boxes: the tile box is TROWF floats wide starting SHF floats
    // before vertex o-1 (a 16-byte-aligned element offset, as o*K is), the
    // owned boxes B*K floats from vertex o.
    static constexpr bool TMAP = (S::B * K * 4) % 16 == 0 && TROWF <= 256;
    static constexpr int TROWS = DIM == 3 ? S::T * S::TZ : S::T;
    static constexpr int r32(int x) { return (x + 31) / 32 * 32; }
    static constexpr int tile = r32(TROWS * TROWF);               // floats
    static constexpr int mv = S::MVG ? 0 : r32(2 * S::NOWN * K);  // m then v
    static constexpr int REC = ((3 * DIM + 1) + 1) / 2 * 2;       // s0[D] s1[D] u g[D] (even)
    static constexpr int pts = S::CH * REC;                       // cell-ordered records
    static constexpr int gs = S::NOWN * K;
    static constexpr int uni = r32(pts > gs ? pts : gs);
    static constexpr size_t bytes = sizeof(float) * (tile + mv + uni) + sizeof(int) * (S::NCELL * 2 + S::NT + 64 * 2);
    static constexpr unsigned tile_box_bytes = TROWS * TROWF * 4;  // TROWF x T [x T] floats
    static constexpr unsigned own_box_bytes = S::NOWN * K * 4;
    // float offset of tile vertex (tx, ty, tz)
    __device__ static constexpr int at(int tx, int ty, int tz) {
        return (DIM == 3 ? (tz * S::T + ty) : ty) * TROWF + SHF + tx * K;
    }
};

// HBM->smem staging of a brick, one row per thread: tile rows (threads
// [0, TROWS)) -> bar_tile, owned m/v rows (the next 2*OROWS threads) ->
// bar_mv, each as one TMA bulk copy. Both barriers expect an arrival from
// every thread (arrive.expect_tx with the thread's own byte count, 0 if it
// has no row), so no reduction is needed. Rows that are not 16-byte aligned
// or would read outside the array fall back to cp.async by the same thread.
template <int DIM, int ORDER>
__device__ __forceinline__ void stage_brick(const StepArgs& A, const int* o, float* tile, float* mvs,
                                            unsigned long long* bar_tile, unsigned long long* bar_mv, int tid) {
    using S = BrickShape<DIM>;
    using L = BrickSmem<DIM, ORDER>;
    constexpr int K = L::K, B = S::B, T = S::T;
    constexpr int GR = (K % 2 == 0) ? 2 : 1;
    constexpr unsigned TBYTES = ((L::SHF * 4 + T * K * 4 + 15) / 16) * 16;
    constexpr unsigned OBYTES = B * K * 4;
    constexpr int OROWS = DIM == 3 ? B * S::BZ : B;
    static_assert(L::TROWS + 2 * OROWS <= S::NT, "one staging row per thread");
    const long long nc_bytes = (long long)A.s.res[0] * A.s.res[1] * (DIM == 3 ? A.s.zstore : 1) * K * 4;
    unsigned tx_tile = 0, tx_mv = 0;
    if (tid < L::TROWS) {
        const int r = tid;
        const int ty = DIM == 3 ? r % T : r, tz = DIM == 3 ? r / T : 0;
        const int vy = o[1] - 1 + ty, vz = o[2] - 1 + tz;
        if (vy >= 0 && vy < A.s.res[1] && (DIM == 2 || (vz >= 0 && vz < A.s.res[2]))) {
            const long long firstv = (DIM == 3 ? (long long)(vz - A.s.zoff) * A.s.sz : 0LL) + (long long)vy * A.s.sy + o[0] - 1;
            const long long src = firstv * K * 4 - L::SHF * 4;
            float* dst = tile + r * L::TROWF;
            if ((src & 15) == 0 && src >= 0 && src + TBYTES <= nc_bytes) {
                tx_tile = TBYTES;
                mbar_expect_tx(bar_tile, TBYTES);
                bulk_g2s(dst, reinterpret_cast<const char*>(A.p_in) + src, TBYTES, bar_tile);
            } else {
                mbar_expect_tx(bar_tile, 0);
                for (int q = 0; q < T * K; q += GR) {
                    const int vx = o[0] - 1 + q / K;
                    const bool ok = vx >= 0 && vx < A.s.res[0];
                    cp_async<GR>(dst + L::SHF + q, ok ? A.p_in + firstv * K + q : A.p_in, ok);
                }
            }
        }
    } else if (!S::MVG && tid < L::TROWS + 2 * OROWS) {
        const int t = tid - L::TROWS;
        const int which = t / OROWS, r = t - which * OROWS;
        const int ly = r % B, lz = DIM == 3 ? r / B : 0;
        const int vy = o[1] + ly, vz = o[2] + lz;
        if (vy < A.s.res[1] && (DIM == 2 || vz < A.s.res[2])) {
            const long long v0 = (DIM == 3 ? (long long)(vz - A.s.zoff) * A.s.sz : 0LL) + (long long)vy * A.s.sy + o[0];
            const long long src = v0 * K * 4;
            const float* gsrc = which ? A.v_in : A.m_in;
            float* dst = mvs + which * S::NOWN * K + r * B * K;
            if ((src & 15) == 0 && (OBYTES % 16) == 0 && o[0] + B <= A.s.res[0]) {
                tx_mv = OBYTES;
                mbar_expect_tx(bar_mv, OBYTES);
                bulk_g2s(dst, reinterpret_cast<const char*>(gsrc) + src, OBYTES, bar_mv);
            } else {
                mbar_expect_tx(bar_mv, 0);
                for (int q = 0; q < B * K; q += GR) {
                    const bool ok = o[0] + q / K < A.s.res[0];
                    cp_async<GR>(dst + q, ok ? gsrc + v0 * K + q : gsrc, ok);
                }
            }
        }
    }
    (void)tx_tile;
    (void)tx_mv;
    cp_async_commit();
}

#ifdef TGCU_PHASE_TIMING
// Instrumented build only (tools/phase_timing.py): per CTA, thread 0's
// %globaltimer at the kernel's phase boundaries.
constexpr int kPhaseSlots = 12;
__device__ unsigned long long g_phase[32768 * kPhaseSlots];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TGCU_PT(var) \
    unsigned long long var = 0; \
    if (threadIdx.x == 0) var = gtimer();
#define TGCU_PT_SET(var) \
    if (threadIdx.x == 0) var = gtimer();
#else
#define TGCU_PT(var)
#define TGCU_PT_SET(var)
#endif

// Bricks with at most this many points take the unsorted gather (one warp
// of points; each vertex scans them). Compiled in (TINYOK) only for the
// variant launched on sparse batches (under 64 point copies per brick on
// average, e.g. C5): its branches cost the dense C2 step ~1.4 %.
constexpr int kTiny = 32;

template <int DIM, int ORDER, bool EIK, bool EXPORT, bool TINYOK, bool SPLIT = false>
__global__ void __launch_bounds__(BrickShape<DIM>::NT, DIM == 3 ? 1024 / BrickShape<DIM>::NT : 2) k_brick_step(const __grid_constant__ StepArgs A) {
    using S = BrickShape<DIM>;
    using L = BrickSmem<DIM, ORDER>;
    constexpr int K = KOf<DIM, ORDER>::value;
    constexpr int B = S::B, T = S::T, CE = S::CE, NT = S::NT, CH = S::CH, REC = L::REC;
    constexpr int NC = 1 << DIM;
    // brick index and its point range, loaded together with the error flag
    // brick of this CTA: the launch order puts the multi-chunk bricks first so
    // the kernel does not end on a long surface brick
    // Split bricks (grids with fewer bricks than CTA slots, e.g. C1): a
    // cluster of SPL CTAs shares one brick; CTA r takes the brick's chunks r,
    // r + SPL, ..., and the per-vertex sums of the others reach rank 0 over
    // distributed shared memory, which then runs TV + Adam alone.
    // (a separate instantiation, SPLIT, so the unsplit kernel carries none of it)
    // programmatic dependent launch (launch_train_step): wait for the previous
    // step's finalize (st, partials), then let this step's finalize be
    // scheduled — it becomes resident only once the last brick CTA has
    // started, i.e. for the last wave
    pdl_wait();
    pdl_trigger();
    const int SPL = SPLIT ? A.split : 1;
    int crank = 0;
    if constexpr (SPLIT) crank = (int)cg::this_cluster().block_rank();
    // brick and point range in one load (no dependent off[] lookup)
    const int4 bi = order_info(const_cast<int*>(A.order), (int)A.NB)[blockIdx.x / SPL];
    const int b = bi.x;
    const int bcx = b % A.nb[0], bcy = (b / A.nb[0]) % A.nb[1], bcz = b / (A.nb[0] * A.nb[1]);
    const int err = A.st->error;
    const int p0 = bi.y, p1 = bi.z;
    // (st->error is written only by the finalize of an earlier step, ordered
    // before this kernel: every CTA of a split cluster sees the same value)
    if (err) return;
    const int pfirst = p0 + crank * CH;                  // this CTA's first chunk
    const int nmine = pfirst < p1 ? (p1 - pfirst + SPL * CH - 1) / (SPL * CH) : 0;

    extern __shared__ __align__(128) float smem[];
    float* tile = smem;                           // current parameters + halo
    float* mvs = tile + L::tile;                  // m, v of the owned vertices
    float* uni = mvs + L::mv;                     // cell-ordered records | Gs
    int* cnt = reinterpret_cast<int*>(uni + L::uni);
    int* start = cnt + S::NCELL;
    int* perm = start + S::NCELL;                 // thread -> owned vertex (load balance)
    int* bhist = perm + NT;                       // 64 workload buckets
    int* bstart = bhist + 64;
    __shared__ int run_total;
    __shared__ double red[4][NT / 32];
    __shared__ double xsum[3];  // split clusters: this CTA's recon, eik, home-point sums
    __shared__ __align__(8) unsigned long long bars[2];  // tile, mv

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    constexpr int NW = NT / 32;
    TGCU_PT(pt_start)
#ifdef TGCU_PHASE_TIMING
    unsigned long long pt_tile = 0, pt_2a = 0, pt_scan = 0, pt_bal = 0, pt_2b = 0, pt_x;
#endif
    // grid = (nb_x, nb_y, nb_z): brick coordinates without integer division
    const int o[3] = {bcx * B, bcy * B, DIM == 3 ? (A.zb0 + bcz) * S::BZ : 0};
    const int zrel = o[2] - A.s.zoff;  // first owned plane in the stored planes
    const bool tmap = L::TMAP && A.use_tmap;
    // m and v are needed only by the epilogue: a brick with points issues their
    // boxes once its tile has landed, so the tile (which the forward waits
    // for) does not share the memory system with them at the CTA's start
    const bool mv_late = !SPLIT && tmap && nmine > 0;

    if (tid == 0) {
        mbar_init(&bars[0], tmap ? 1 : NT);
        mbar_init(&bars[1], tmap ? 1 : NT);
        mbar_fence_init();
    }
    // With tensor maps only warp 0 touches the barriers (thread 0 arms them,
    // warp 0 waits); per-row staging has every thread arrive.
    if (tmap) __syncwarp();
    else __syncthreads();
    // The tile is waited for inside the first chunk, after the points have
    // been loaded, located and counted (none of which needs it).
    if (tmap) {
        // one elected thread: the (B+2)^D tile (out-of-grid vertices zero
        // filled) and the owned m, v boxes, each one TMA tensor copy
        // (split clusters: the tile only where there are points or TV to do,
        // m and v only in rank 0, which alone runs TV + Adam)
        if (tid == 0 && (crank == 0 || nmine > 0)) {
            mbar_expect_tx(&bars[0], L::tile_box_bytes);
            if (crank == 0 && !mv_late && !S::MVG) mbar_expect_tx(&bars[1], 2 * L::own_box_bytes);
            if constexpr (DIM == 3) {
                tma_load_3d(tile, &A.tm_tile, &bars[0], (o[0] - 1) * K - L::SHF, o[1] - 1, zrel - 1);
                if (S::MVG) {
                    if (crank == 0 && !mv_late) {
                        tma_prefetch_3d(&A.tm_m_in, o[0] * K, o[1], zrel);
                        tma_prefetch_3d(&A.tm_v_in, o[0] * K, o[1], zrel);
                    }
                } else if (crank == 0 && !mv_late) {
                    tma_load_3d(mvs, &A.tm_m_in, &bars[1], o[0] * K, o[1], zrel);
                    tma_load_3d(mvs + S::NOWN * K, &A.tm_v_in, &bars[1], o[0] * K, o[1], zrel);
                }
            } else {
                tma_load_2d(tile, &A.tm_tile, &bars[0], (o[0] - 1) * K - L::SHF, o[1] - 1);
                if (crank == 0 && !mv_late) {
                    tma_load_2d(mvs, &A.tm_m_in, &bars[1], o[0] * K, o[1]);
                    tma_load_2d(mvs + S::NOWN * K, &A.tm_v_in, &bars[1], o[0] * K, o[1]);
                }
            }
        }
    } else {
        using LS = BrickSmem<DIM, ORDER>;
        constexpr int OR = DIM == 3 ? B * S::BZ : B;
        stage_brick<DIM, ORDER>(A, o, tile, mvs, &bars[0], &bars[1], tid);
        // threads that did not arrive on a barrier (no row of it) arrive now
        const bool tile_row = tid < LS::TROWS && [&] {
            const int ty = DIM == 3 ? tid % T : tid, tz = DIM == 3 ? tid / T : 0;
            const int vy = o[1] - 1 + ty, vz = o[2] - 1 + tz;
            return vy >= 0 && vy < A.s.res[1] && (DIM == 2 || (vz >= 0 && vz < A.s.res[2]));
        }();
        const bool mv_row = !S::MVG && tid >= LS::TROWS && tid < LS::TROWS + 2 * OR && [&] {
            const int t = tid - LS::TROWS, r = t % OR;
            const int ly = r % B, lz = DIM == 3 ? r / B : 0;
            return o[1] + ly < A.s.res[1] && (DIM == 2 || o[2] + lz < A.s.res[2]);
        }();
        if (!tile_row) mbar_arrive(&bars[0]);
        if (!mv_row) mbar_arrive(&bars[1]);
    }

    auto issue_mv_late = [&] {  // thread 0, after its warp saw the tile land
        if (mv_late && tid == 0) {
            if constexpr (S::MVG) {  // into L2 only: the epilogue reads them from HBM
                tma_prefetch_3d(&A.tm_m_in, o[0] * K, o[1], zrel);
                tma_prefetch_3d(&A.tm_v_in, o[0] * K, o[1], zrel);
                return;
            }
            mbar_expect_tx(&bars[1], 2 * L::own_box_bytes);
            if constexpr (DIM == 3) {
                tma_load_3d(mvs, &A.tm_m_in, &bars[1], o[0] * K, o[1], zrel);
                tma_load_3d(mvs + S::NOWN * K, &A.tm_v_in, &bars[1], o[0] * K, o[1], zrel);
            } else {
                tma_load_2d(mvs, &A.tm_m_in, &bars[1], o[0] * K, o[1]);
                tma_load_2d(mvs + S::NOWN * K, &A.tm_v_in, &bars[1], o[0] * K, o[1]);
            }
        }
    };
    constexpr bool PACKED = DIM == 3 && ORDER == 2;  // fp32x2 accumulators (corner_grad_p2)
    float G[K];
#pragma unroll
    for (int q = 0; q < K; ++q) G[q] = 0.0f;
    float2 P[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) P[q] = make_float2(0.f, 0.f);
    double recon_sum = 0.0, eik_sum = 0.0;
    int home_pts = 0;
    int myv = tid;  // owned vertex of this thread; set per brick by the workload sort

    // Tiny bricks (at most kTiny points, one chunk): no counting sort. Records
    // stay in point order with each point's cell in start[]; every vertex
    // scans the few points for its incident cells (3 barriers instead of 8).
    const bool tiny = TINYOK && (p1 - p0) <= kTiny;
    // one chunk (or none) and no split: thread tid owns vertex tid throughout
    const bool ident = !SPLIT && (tiny || nmine <= 1);
    for (int base = pfirst; base < p1; base += SPL * CH) {
        const int m = min(CH, p1 - base);
        if (!tiny) {
            for (int i = tid; i < S::NCELL; i += NT) cnt[i] = 0;
            if (base == pfirst && tid < 64) bhist[tid] = 0;
            if (tid == 0) run_total = 0;
            __syncthreads();
        }
        // 2a. locate + cell rank, the chunk's counting sort by cell and (first
        //     chunk) the workload balance need no parameters: they run while
        //     the tile is still in flight. Then the forward from the tile and
        //     the fp64 loss chain write each record straight to its cell slot.
        int ec = 0, rank = 0;
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
        double lc[DIM];
        int tc[3] = {0, 0, 0};
        if (tid < m) {
            q = A.binned[base + tid];
            const float pf[3] = {q.x, q.y, q.z};
#pragma unroll
            for (int a = 0; a < DIM; ++a) {
                const int c = locate_axis(A.s, a, (double)pf[a], lc[a]);
                tc[a] = c - (o[a] - 1);  // in [0, B]
            }
            ec = DIM == 3 ? (tc[2] * CE + tc[1]) * CE + tc[0] : tc[1] * CE + tc[0];
            if (tiny) start[tid] = tc[0] | (tc[1] << 8) | (tc[2] << 16);
            else if (!A.det) rank = atomicAdd(&cnt[ec], 1);
        }
        if (A.det && !tiny) {
            // Deterministic mode: the stable rank (earlier threads of the
            // chunk first), so every cell run lists its points in chunk order
            // and each vertex sums them in a fixed order: warp-local ranks by
            // __match_any_sync, then the warps take their cells' bases in warp
            // order (one warp per barrier interval).
            const bool val = tid < m;
            const unsigned peers = __match_any_sync(0xffffffffu, val ? ec : S::NCELL + lane);
            const int leader = __ffs(peers) - 1;
            const int lrank = __popc(peers & ((1u << lane) - 1u));
            for (int w = 0; w < NW; ++w) {
                int b0 = 0;
                if (warp == w && val && lane == leader) {
                    b0 = cnt[ec];
                    cnt[ec] = b0 + __popc(peers);
                }
                if (warp == w) rank = __shfl_sync(0xffffffffu, b0, leader) + lrank;
                __syncthreads();
            }
        }
#ifdef TGCU_PHASE_TIMING
        unsigned long long pt_c0 = 0;
        TGCU_PT_SET(pt_c0)
#endif
        if (!tiny) {
            __syncthreads();
            cell_runs<S::NCELL, NT>(cnt, start, &run_total);
            if (base == pfirst && nmine == 1) {
                // single-chunk brick: the tile wait rides on this barrier
                cp_async_wait<0>();
                if (warp == 0) mbar_wait(&bars[0], 0);
                issue_mv_late();
            }
            __syncthreads();
        }
#ifdef TGCU_PHASE_TIMING
        const unsigned long long pt_s0 = pt_c0;
#endif
#ifdef TGCU_PHASE_TIMING
        TGCU_PT_SET(pt_x)
        if (tid == 0) pt_scan += pt_x - pt_s0;
        const unsigned long long pt_b0 = pt_x;
#endif
        if (base == pfirst && tiny) {
            cp_async_wait<0>();
            if (warp == 0) mbar_wait(&bars[0], 0);
            issue_mv_late();
            __syncthreads();  // tile and the points' cells (start[]) visible
#ifdef TGCU_PHASE_TIMING
            TGCU_PT_SET(pt_tile)
#endif
        } else if (base == pfirst && nmine == 1) {
            // single-chunk brick: identity mapping; the tile was waited for
            // with the cell runs
#ifdef TGCU_PHASE_TIMING
            TGCU_PT_SET(pt_tile)
#endif
        } else if (base == pfirst) {
            // Load balance: sort the owned vertices by their (first-chunk)
            // workload into 64 buckets so a warp's lanes carry similar loads;
            // the mapping then holds for the brick (points are in random order).
            const int v = tid;
            const int l3[3] = {v % B, (v / B) % B, DIM == 3 ? v / (B * B) : 0};
            const int e0 = DIM == 3 ? ((l3[2] + 1) * CE + l3[1] + 1) * CE + l3[0] + 1 : (l3[1] + 1) * CE + l3[0] + 1;
            int wl = 0;
#pragma unroll
            for (int c = 0; c < NC; ++c)
                wl += cnt[e0 - (c & 1) - ((c >> 1) & 1) * CE - (DIM == 3 ? ((c >> 2) & 1) * CE * CE : 0)];
            const int bk = 63 - min(wl, 63);  // heavy first
            const int r2 = atomicAdd(&bhist[bk], 1);
            __syncthreads();
            if (warp == 0) {
                const int h0 = bhist[lane], h1 = bhist[lane + 32];
                int x0 = h0, x1 = h1;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int y0 = __shfl_up_sync(0xffffffffu, x0, off);
                    const int y1 = __shfl_up_sync(0xffffffffu, x1, off);
                    if (lane >= off) {
                        x0 += y0;
                        x1 += y1;
                    }
                }
                const int tot0 = __shfl_sync(0xffffffffu, x0, 31);
                bstart[lane] = x0 - h0;
                bstart[lane + 32] = tot0 + x1 - h1;
            }
            __syncthreads();
            perm[bstart[bk] + r2] = v;
            cp_async_wait<0>();  // own fallback rows (rare: grid-edge bricks)
            if (warp == 0) mbar_wait(&bars[0], 0);  // one warp waits for the tile; the others park here
            issue_mv_late();
            __syncthreads();
            myv = perm[tid];
#ifdef TGCU_PHASE_TIMING
            TGCU_PT_SET(pt_tile)
#endif
        }
#ifdef TGCU_PHASE_TIMING
        TGCU_PT_SET(pt_x)
        if (tid == 0) pt_bal += pt_x - pt_b0;
        const unsigned long long pt_f0 = pt_x;
#endif
        if (tid < m) {
            bool home = true;
#pragma unroll
            for (int a = 0; a < DIM; ++a) home &= tc[a] >= 1;
#ifdef TGCU_FP64_FORWARD
            // fp64 forward (blend_corner_d; A/B build): the loss
            // chain amplifies forward errors
            double f = 0.0, fg[DIM];
#pragma unroll
            for (int a = 0; a < DIM; ++a) fg[a] = 0.0;
            // corners one at a time: the fp64 temporaries of one corner live at
            // once (the vertex accumulators hold registers across the chunk loop)
#pragma unroll 1
            for (int c = 0; c < NC; ++c)
                blend_corner_d<DIM, ORDER, EIK>(tile + L::at(tc[0] + (c & 1), tc[1] + ((c >> 1) & 1),
                                                             DIM == 3 ? tc[2] + ((c >> 2) & 1) : 0),
                                                A.s, lc, c, f, fg);
            AxisF ax[DIM];
#pragma unroll
            for (int a = 0; a < DIM; ++a) ax[a] = axis_factors(A.s, a, lc[a]);
#else
            // fp32 forward from the fp64 cell offsets (per-axis factors rounded once)
            AxisF ax[DIM];
#pragma unroll
            for (int a = 0; a < DIM; ++a) ax[a] = axis_factors(A.s, a, lc[a]);
            float f = 0.0f, fg[DIM];
#pragma unroll
            for (int a = 0; a < DIM; ++a) fg[a] = 0.0f;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                float cb[K];
                load_block<K, false>(tile + L::at(tc[0] + (c & 1), tc[1] + ((c >> 1) & 1),
                                                  DIM == 3 ? tc[2] + ((c >> 2) & 1) : 0),
                                     cb);
                blend_corner<DIM, ORDER, EIK>(cb, corner_geom<DIM>(A.s, ax, c), f, fg);
            }
#endif
            double recon, eik;
            float u, gv[DIM];
            point_loss<DIM, EIK>(A.L, f, fg, q.w, recon, eik, u, gv);
            if (home) {
                recon_sum += recon;
                eik_sum += eik;
                ++home_pts;
            }
            // record: s0/s1 rounded from fp64 (1 - l must not be formed from a
            // rounded l), u, g; lands in cell order
            float rv[REC];
#pragma unroll
            for (int a = 0; a < DIM; ++a) {
                rv[a] = ax[a].s0;
                rv[DIM + a] = ax[a].s1;
                rv[2 * DIM + 1 + a] = gv[a];
            }
            rv[2 * DIM] = u;
#pragma unroll
            for (int k2 = 3 * DIM + 1; k2 < REC; ++k2) rv[k2] = 0.0f;
            float2* dst = reinterpret_cast<float2*>(uni + (tiny ? tid : start[ec] + rank) * REC);
#pragma unroll
            for (int k2 = 0; k2 < REC / 2; ++k2) dst[k2] = make_float2(rv[2 * k2], rv[2 * k2 + 1]);
        }
        __syncthreads();  // records visible

#ifdef TGCU_PHASE_TIMING
        TGCU_PT_SET(pt_x)
        if (tid == 0) pt_2a += pt_x - pt_f0;
#endif
#ifdef TGCU_PHASE_TIMING
        const unsigned long long pt_g0 = pt_x;
#endif
        if (tiny) {
            // 2b (tiny bricks): each vertex scans the m points for its cells
            const int v = tid;
            const int l3[3] = {v % B, (v / B) % B, DIM == 3 ? v / (B * B) : 0};
            bool own_ok = true;
#pragma unroll
            for (int a = 0; a < DIM; ++a) own_ok &= (o[a] + l3[a]) < A.s.res[a];
            for (int j = 0; own_ok && j < m; ++j) {
                const int pc = start[j];
                const int bx = l3[0] + 1 - (pc & 255), by = l3[1] + 1 - ((pc >> 8) & 255);
                const int bz = DIM == 3 ? l3[2] + 1 - (pc >> 16) : 0;
                if ((unsigned)bx > 1u || (unsigned)by > 1u || (unsigned)bz > 1u) continue;
                const int c = bx | (by << 1) | (bz << 2);
                const float2* rp = reinterpret_cast<const float2*>(uni + j * REC);
                float r[REC];
#pragma unroll
                for (int k2 = 0; k2 < REC / 2; ++k2) {
                    const float2 t2 = rp[k2];
                    r[2 * k2] = t2.x;
                    r[2 * k2 + 1] = t2.y;
                }
                Corner<DIM> cg;
                float sv[DIM];
#pragma unroll
                for (int a = 0; a < DIM; ++a) {
                    const bool bit = (c >> a) & 1;
                    const float s0 = r[a], s1 = r[DIM + a];
                    sv[a] = bit ? s1 : s0;
                    cg.d[a] = (bit ? -s0 : s1) * A.s.hf[a];
                }
                cg.w = sv[0];
#pragma unroll
                for (int a = 1; a < DIM; ++a) cg.w *= sv[a];
                float gvd[DIM];
#pragma unroll
                for (int a = 0; a < DIM; ++a) {
                    float other = 1.0f;
#pragma unroll
                    for (int bb = 0; bb < DIM; ++bb)
                        if (bb != a) other *= sv[bb];
                    cg.dw[a] = EIK ? (((c >> a) & 1) ? A.s.inv_hf[a] : -A.s.inv_hf[a]) * other : 0.0f;
                    gvd[a] = EIK ? r[2 * DIM + 1 + a] : 0.0f;
                }
                if constexpr (PACKED)
                    corner_grad_p2<EIK>(*reinterpret_cast<const Corner<3>*>(&cg), r[2 * DIM], gvd, P);
                else
                    corner_grad<DIM, ORDER, K>(cg, r[2 * DIM], gvd, G);
            }
        } else
        // 2b. this thread's vertex gathers the points of its 2^D incident
        //     cells, as one flattened loop over (corner, point)
        {
            const int l3[3] = {myv % B, (myv / B) % B, DIM == 3 ? myv / (B * B) : 0};
            bool own_ok = true;
#pragma unroll
            for (int a = 0; a < DIM; ++a) own_ok &= (o[a] + l3[a]) < A.s.res[a];
            const int e0 = DIM == 3 ? ((l3[2] + 1) * CE + l3[1] + 1) * CE + l3[0] + 1 : (l3[1] + 1) * CE + l3[0] + 1;
            // non-empty incident cells as a bitmask; one flat loop over items,
            // the next corner is found with ffs when a cell's run ends
            unsigned mask = 0;
            int total = 0;
            if (own_ok) {
#pragma unroll
                for (int cc = 0; cc < NC; ++cc) {
                    const int n = cnt[e0 - (cc & 1) - ((cc >> 1) & 1) * CE - (DIM == 3 ? ((cc >> 2) & 1) * CE * CE : 0)];
                    total += n;
                    mask |= (n > 0 ? 1u : 0u) << cc;
                }
            }
            int c = 0, j = 0, jend = 0;
            for (int k = 0; k < total; ++k) {
                if (j == jend) {
                    c = __ffs(mask) - 1;
                    mask &= mask - 1;
                    const int e = e0 - (c & 1) - ((c >> 1) & 1) * CE - (DIM == 3 ? ((c >> 2) & 1) * CE * CE : 0);
                    j = start[e];
                    jend = j + cnt[e];
                }
                const float2* rp = reinterpret_cast<const float2*>(uni + j * REC);
                float r[REC];
#pragma unroll
                for (int k2 = 0; k2 < REC / 2; ++k2) {
                    const float2 t2 = rp[k2];
                    r[2 * k2] = t2.x;
                    r[2 * k2 + 1] = t2.y;
                }
                Corner<DIM> cg;
                float sv[DIM];
#pragma unroll
                for (int a = 0; a < DIM; ++a) {
                    const bool bit = (c >> a) & 1;
                    const float s0 = r[a], s1 = r[DIM + a];
                    sv[a] = bit ? s1 : s0;
                    cg.d[a] = (bit ? -s0 : s1) * A.s.hf[a];  // (l - bit) * h
                }
                cg.w = sv[0];
#pragma unroll
                for (int a = 1; a < DIM; ++a) cg.w *= sv[a];
                float gvd[DIM];
#pragma unroll
                for (int a = 0; a < DIM; ++a) {
                    float other = 1.0f;
#pragma unroll
                    for (int bb = 0; bb < DIM; ++bb)
                        if (bb != a) other *= sv[bb];
                    cg.dw[a] = EIK ? (((c >> a) & 1) ? A.s.inv_hf[a] : -A.s.inv_hf[a]) * other : 0.0f;
                    gvd[a] = EIK ? r[2 * DIM + 1 + a] : 0.0f;
                }
                if constexpr (PACKED)
                    corner_grad_p2<EIK>(*reinterpret_cast<const Corner<3>*>(&cg), r[2 * DIM], gvd, P);
                else
                    corner_grad<DIM, ORDER, K>(cg, r[2 * DIM], gvd, G);
                ++j;
            }
        }
        // (a brick of one chunk keeps its sums in registers for TV + Adam: its
        // records are released by the m/v barrier below instead)
        if (!ident) __syncthreads();
#ifdef TGCU_PHASE_TIMING
        TGCU_PT_SET(pt_x)
        if (tid == 0) pt_2b += pt_x - pt_g0;
#endif
    }
    TGCU_PT(pt_epi)

    // ---- 3. TV + Adam, thread per vertex; results staged in place ----
    float* Gs = uni;
    if constexpr (PACKED) unpack_p2(P, G);
    if (!ident) {
#pragma unroll
        for (int q = 0; q < K; ++q) Gs[myv * K + q] = G[q];
    }
    double xtot[3] = {0.0, 0.0, 0.0};  // split: the other CTAs' loss sums (rank 0, thread 0)
    if constexpr (SPLIT) {
        // this CTA's loss sums (fixed-order block reduction) for rank 0
        {
            const double v3[3] = {warp_sum_d(recon_sum), warp_sum_d(eik_sum), warp_sum_d((double)home_pts)};
            if (lane == 0)
                for (int k2 = 0; k2 < 3; ++k2) red[k2][warp] = v3[k2];
            __syncthreads();
            if (tid < 3) {
                double acc = 0.0;
                for (int k2 = 0; k2 < NW; ++k2) acc += red[tid][k2];
                xsum[tid] = acc;
            }
        }
        cg::cluster_group cl = cg::this_cluster();
        cl.sync();  // every CTA's per-vertex sums (Gs) and loss sums are in place
        if (crank == 0) {
            // rank order: the same sums every run
            for (int r = 1; r < SPL; ++r) {
                const float* rg = cl.map_shared_rank(Gs, r);
#pragma unroll
                for (int q = 0; q < K; ++q) Gs[tid * K + q] += rg[tid * K + q];
                if (tid == 0) {
                    const double* rx = cl.map_shared_rank(xsum, r);
                    for (int k2 = 0; k2 < 3; ++k2) xtot[k2] += rx[k2];
                }
            }
        }
        cl.sync();  // rank 0 has read the others' shared memory
        if (crank != 0) return;
        if (tid == 0)
            for (int k2 = 0; k2 < 3; ++k2) xsum[k2] = xtot[k2];  // for the final partials (barriers follow)
    }
    cp_async_wait<0>();
    if (nmine == 0 && warp == 0) mbar_wait(&bars[0], 0);  // brick without points: tile not yet waited for
    if (!S::MVG && warp == 0) mbar_wait(&bars[1], 0);  // m/v rows landed
    __syncthreads();
    TGCU_PT(pt_e1)
    double tv_sum = 0.0;
    {
        const int v = tid;
        const int l3[3] = {v % B, (v / B) % B, DIM == 3 ? v / (B * B) : 0};
        const int g3[3] = {o[0] + l3[0], o[1] + l3[1], o[2] + l3[2]};
        bool vok = true;
#pragma unroll
        for (int a = 0; a < DIM; ++a) vok &= g3[a] < A.s.res[a];
#if TGCU_TV_SHFL
        // The x / y stencil neighbours of a channel pair come from the
        // neighbouring lanes (a warp holds 32 / B brick rows of B vertices, x
        // along the lanes) by shuffles; only row / warp-edge lanes and the z
        // neighbours read the tile, whose row pitch gives the tile reads 2-way
        // bank conflicts (C2 0.2652 -> 0.2626 ms per step, C3 1.2598 -> 1.2517,
        // same-box A/B; TGCU_TV_SHFL=0 builds the all-loads form). Not in the
        // sparse-batch variant (C5: 8.632 -> 8.671 ms, its epilogues overlap
        // each other more than the point phases). Every lane runs it (the
        // shuffles are full-warp); lanes of out-of-grid vertices store nothing
        // global.
        if constexpr (K % 2 == 0 && !S::MVG && !TINYOK) {
            constexpr int RPW = 32 / B;  // brick rows per warp
            const int xr = lane % B, yr = lane / B;
            const long long gidx =
                ((DIM == 3 ? (long long)(g3[2] - A.s.zoff) * A.s.sz : 0LL) + (long long)g3[1] * A.s.sy + g3[0]) * K;
            const float* tp = tile + L::at(1 + l3[0], 1 + l3[1], DIM == 3 ? 1 + l3[2] : 0);
            float* gs = Gs + v * K;
            const float* mi = mvs + v * K;
            const float* vi = mvs + S::NOWN * K + v * K;
            float* mo = mvs + v * K;
            float* vo = mvs + S::NOWN * K + v * K;
            constexpr int offs[3] = {K, L::TROWF, DIM == 3 ? T * L::TROWF : 0};
            bool hi[DIM], lo[DIM];
#pragma unroll
            for (int a = 0; a < DIM; ++a) {
                hi[a] = A.want_tv && g3[a] + 1 < A.s.res[a];
                lo[a] = A.want_tv && g3[a] >= 1;
            }
            const float c1 = A.c1, c2 = A.c2, lr_bc1 = A.lr * A.inv_bc1;
            const float2 gsc = make_float2(A.tv_gscale, A.tv_gscale);
            const float2 b1 = make_float2(A.b1, A.b1), b2 = make_float2(A.b2, A.b2);
            const float2 cc1 = make_float2(c1, c1), cc2 = make_float2(c2, c2);
            float2 sq2 = make_float2(0.f, 0.f);
            auto shf = [](float2 x, int d, bool down) {
                return down ? make_float2(__shfl_down_sync(0xffffffffu, x.x, d), __shfl_down_sync(0xffffffffu, x.y, d))
                            : make_float2(__shfl_up_sync(0xffffffffu, x.x, d), __shfl_up_sync(0xffffffffu, x.y, d));
            };
            auto ld2 = [](const float* p) { return *reinterpret_cast<const float2*>(p); };
            float2 gsum = make_float2(0.f, 0.f);
            float2 gkeep[K / 2];
            float2 m2[K / 2], v2[K / 2];
#pragma unroll
            for (int q = 0; q < K; q += 2) {
                m2[q / 2] = ld2(mi + q);
                v2[q / 2] = ld2(vi + q);
            }
#pragma unroll
            for (int q = 0; q < K; q += 2) {
                const float2 pv = ld2(tp + q);
                float2 nb[DIM][2];  // [axis][+, -]
                nb[0][0] = shf(pv, 1, true);
                nb[0][1] = shf(pv, 1, false);
                nb[1][0] = shf(pv, B, true);
                nb[1][1] = shf(pv, B, false);
                if (xr == B - 1 && hi[0]) nb[0][0] = ld2(tp + offs[0] + q);
                if (xr == 0 && lo[0]) nb[0][1] = ld2(tp - offs[0] + q);
                if (yr == RPW - 1 && hi[1]) nb[1][0] = ld2(tp + offs[1] + q);
                if (yr == 0 && lo[1]) nb[1][1] = ld2(tp - offs[1] + q);
                if constexpr (DIM == 3) {
                    if (hi[2]) nb[2][0] = ld2(tp + offs[2] + q);
                    if (lo[2]) nb[2][1] = ld2(tp - offs[2] + q);
                }
                const float2 npv = make_float2(-pv.x, -pv.y);
                float2 gt = make_float2(0.f, 0.f);
#pragma unroll
                for (int a = 0; a < DIM; ++a) {
                    if (hi[a]) {  // pair (v, v+e_a): TV sum and -d
                        const float2 d = __fadd2_rn(nb[a][0], npv);
                        sq2 = __ffma2_rn(d, d, sq2);
                        gt = __fadd2_rn(gt, make_float2(-d.x, -d.y));
                    }
                    if (lo[a]) {  // pair (v-e_a, v): +(pv - p_lo)
                        const float2 pl = nb[a][1];
                        gt = __fadd2_rn(gt, __fadd2_rn(pv, make_float2(-pl.x, -pl.y)));
                    }
                }
                const float2 gi =
                    __ffma2_rn(gsc, gt, ident ? make_float2(G[q], G[q + 1]) : *reinterpret_cast<const float2*>(gs + q));
                gkeep[q / 2] = gi;
                gsum = __fadd2_rn(gsum, gi);
                if constexpr (EXPORT)
                    if (vok) *reinterpret_cast<float2*>(A.grad_out + gidx + q) = gi;
                const float2 mn = __ffma2_rn(b1, m2[q / 2], __fmul2_rn(cc1, gi));
                const float2 vn = __ffma2_rn(b2, v2[q / 2], __fmul2_rn(cc2, __fmul2_rn(gi, gi)));
                *reinterpret_cast<float2*>(mo + q) = mn;
                *reinterpret_cast<float2*>(vo + q) = vn;
                const float2 stp = make_float2(lr_bc1 * mn.x * fast_rcp(fast_sqrt(vn.x * A.inv_bc2) + A.eps),
                                               lr_bc1 * mn.y * fast_rcp(fast_sqrt(vn.y * A.inv_bc2) + A.eps));
                *reinterpret_cast<float2*>(gs + q) = __fadd2_rn(pv, make_float2(-stp.x, -stp.y));
            }
            if (vok && !isfinite(gsum.x + gsum.y)) {
#pragma unroll
                for (int q = 0; q < K; q += 2) {
                    const float2 gi = gkeep[q / 2];
                    if (!isfinite(gi.x)) atomicMin(&A.st->bad_grad, (unsigned long long)(gidx + q));
                    if (!isfinite(gi.y)) atomicMin(&A.st->bad_grad, (unsigned long long)(gidx + q + 1));
                }
            }
            tv_sum = vok ? (double)(sq2.x + sq2.y) : 0.0;
        } else
#endif
        if (vok) {
            const long long gidx =
                ((DIM == 3 ? (long long)(g3[2] - A.s.zoff) * A.s.sz : 0LL) + (long long)g3[1] * A.s.sy + g3[0]) * K;
            const float* tp = tile + L::at(1 + l3[0], 1 + l3[1], DIM == 3 ? 1 + l3[2] : 0);
            float* gs = Gs + v * K;
            // m, v of this vertex: staged rows in shared memory, or (MVG) HBM
            // (prefetched into L2), new values stored straight to the out slot
            const float* mi = S::MVG ? A.m_in + gidx : mvs + v * K;
            const float* vi = S::MVG ? A.v_in + gidx : mvs + S::NOWN * K + v * K;
            float* mo = S::MVG ? A.m_out + gidx : mvs + v * K;
            float* vo = S::MVG ? A.v_out + gidx : mvs + S::NOWN * K + v * K;
            constexpr int offs[3] = {K, L::TROWF, DIM == 3 ? T * L::TROWF : 0};
            bool hi[DIM], lo[DIM];
#pragma unroll
            for (int a = 0; a < DIM; ++a) {
                hi[a] = A.want_tv && g3[a] + 1 < A.s.res[a];
                lo[a] = A.want_tv && g3[a] >= 1;
            }
            const float c1 = A.c1, c2 = A.c2, lr_bc1 = A.lr * A.inv_bc1;
            if constexpr (K % 2 == 0) {
                // channel pairs on the packed fp32x2 pipe (FFMA2 / FADD2 / FMUL2)
                const float2 gsc = make_float2(A.tv_gscale, A.tv_gscale);
                const float2 b1 = make_float2(A.b1, A.b1), b2 = make_float2(A.b2, A.b2);
                const float2 cc1 = make_float2(c1, c1), cc2 = make_float2(c2, c2);
                float2 sq2 = make_float2(0.f, 0.f);
                // TV gradient + point gradient of channel pair q (the TV sum
                // accumulates into *sq when given)
                auto grad_pair = [&](int q, float2* sq) -> float2 {
                    const float2 pv = *reinterpret_cast<const float2*>(tp + q);
                    const float2 npv = make_float2(-pv.x, -pv.y);
                    float2 gt = make_float2(0.f, 0.f);
#pragma unroll
                    for (int a = 0; a < DIM; ++a) {
                        if (hi[a]) {  // pair (v, v+e_a): TV sum and -d
                            const float2 d = __fadd2_rn(*reinterpret_cast<const float2*>(tp + offs[a] + q), npv);
                            if (sq) *sq = __ffma2_rn(d, d, *sq);
                            gt = __fadd2_rn(gt, make_float2(-d.x, -d.y));
                        }
                        if (lo[a]) {  // pair (v-e_a, v): +(pv - p_lo)
                            const float2 pl = *reinterpret_cast<const float2*>(tp + q - offs[a]);
                            gt = __fadd2_rn(gt, __fadd2_rn(pv, make_float2(-pl.x, -pl.y)));
                        }
                    }
                    return __ffma2_rn(gsc, gt, ident ? make_float2(G[q], G[q + 1]) : *reinterpret_cast<const float2*>(gs + q));
                };
                // one finiteness test per vertex (a NaN / inf in any channel
                // makes the sum non-finite); the channel scan runs only then
                float2 gsum = make_float2(0.f, 0.f);
                float2 gkeep[K / 2];
                float2 m2[K / 2], v2[K / 2];  // all loads issued before the channel loop
#pragma unroll
                for (int q = 0; q < K; q += 2) {
                    m2[q / 2] = *reinterpret_cast<const float2*>(mi + q);
                    v2[q / 2] = *reinterpret_cast<const float2*>(vi + q);
                }
#pragma unroll
                for (int q = 0; q < K; q += 2) {
                    const float2 pv = *reinterpret_cast<const float2*>(tp + q);
                    const float2 gi = grad_pair(q, &sq2);
                    gkeep[q / 2] = gi;
                    gsum = __fadd2_rn(gsum, gi);
                    if constexpr (EXPORT) *reinterpret_cast<float2*>(A.grad_out + gidx + q) = gi;
                    // Adam (adam.cpp:36-55), fp32 state, host fp64 bias corrections
                    const float2 mn = __ffma2_rn(b1, m2[q / 2], __fmul2_rn(cc1, gi));
                    const float2 vn = __ffma2_rn(b2, v2[q / 2], __fmul2_rn(cc2, __fmul2_rn(gi, gi)));
                    *reinterpret_cast<float2*>(mo + q) = mn;
                    *reinterpret_cast<float2*>(vo + q) = vn;
                    const float2 stp = make_float2(lr_bc1 * mn.x * fast_rcp(fast_sqrt(vn.x * A.inv_bc2) + A.eps),
                                                   lr_bc1 * mn.y * fast_rcp(fast_sqrt(vn.y * A.inv_bc2) + A.eps));
                    *reinterpret_cast<float2*>(gs + q) = __fadd2_rn(pv, make_float2(-stp.x, -stp.y));
                }
                if (!isfinite(gsum.x + gsum.y)) {  // rare: name the first bad channel
#pragma unroll
                    for (int q = 0; q < K; q += 2) {
                        const float2 gi = gkeep[q / 2];
                        if (!isfinite(gi.x)) atomicMin(&A.st->bad_grad, (unsigned long long)(gidx + q));
                        if (!isfinite(gi.y)) atomicMin(&A.st->bad_grad, (unsigned long long)(gidx + q + 1));
                    }
                }
                tv_sum = (double)(sq2.x + sq2.y);
            } else {
                float sq = 0.0f;
#pragma unroll
                for (int q = 0; q < K; ++q) {
                    const float pv = tp[q];
                    float gt = 0.0f;
#pragma unroll
                    for (int a = 0; a < DIM; ++a) {
                        if (hi[a]) {
                            const float d = tp[offs[a] + q] - pv;
                            sq = fmaf(d, d, sq);
                            gt -= d;
                        }
                        if (lo[a]) gt += pv - tp[q - offs[a]];
                    }
                    const float gi = fmaf(A.tv_gscale, gt, ident ? G[q] : gs[q]);
                    if constexpr (EXPORT) A.grad_out[gidx + q] = gi;
                    if (!isfinite(gi)) atomicMin(&A.st->bad_grad, (unsigned long long)(gidx + q));
                    const float mn = fmaf(A.b1, mi[q], c1 * gi);
                    const float vn = fmaf(A.b2, vi[q], c2 * gi * gi);
                    mo[q] = mn;
                    vo[q] = vn;
                    gs[q] = pv - lr_bc1 * mn * fast_rcp(fast_sqrt(vn * A.inv_bc2) + A.eps);
                }
                tv_sum = (double)sq;
            }
        }
    }
    __syncthreads();
    TGCU_PT(pt_e2)
    // copy-out of the staged results (p from Gs, m and v from mvs): three TMA
    // tensor box stores (out-of-grid vertices dropped), or one bulk store per
    // row and array, issued by one thread each
    fence_proxy_async_smem();
    __syncthreads();
    if constexpr (DIM == 3) {
        // fused halo: a slab-boundary plane's new parameters go straight into
        // the neighbour's halo plane (peer memory over NVLink), row by row
        const int bz = bcz + A.zb0;
        const bool lo = A.peer_lo && bz == A.zb0, hi = A.peer_hi && bz == A.peer_hi_zb;
        if (lo || hi) {
            const int nvx = min(B, A.s.res[0] - o[0]);
            const int rowf = nvx * K;
            auto put_plane = [&](float* dst, int lz) {
                for (int i = tid; i < B * rowf; i += NT) {
                    const int ly = i / rowf, q = i - ly * rowf;
                    if (o[1] + ly < A.s.res[1])
                        dst[((long long)(o[1] + ly) * A.s.res[0] + o[0]) * K + q] = uni[(lz * B + ly) * B * K + q];
                }
            };
            if (lo) put_plane(A.peer_lo, 0);
            if (hi) put_plane(A.peer_hi, A.peer_hi_lz);
            __threadfence_system();
        }
    }
    if (tmap) {
        if (tid == 0) {
            if constexpr (DIM == 3) {
                tma_store_3d(&A.tm_p_out, uni, o[0] * K, o[1], zrel);
                if (!S::MVG) {
                    tma_store_3d(&A.tm_m_out, mvs, o[0] * K, o[1], zrel);
                    tma_store_3d(&A.tm_v_out, mvs + S::NOWN * K, o[0] * K, o[1], zrel);
                }
            } else {
                tma_store_2d(&A.tm_p_out, uni, o[0] * K, o[1]);
                tma_store_2d(&A.tm_m_out, mvs, o[0] * K, o[1]);
                tma_store_2d(&A.tm_v_out, mvs + S::NOWN * K, o[0] * K, o[1]);
            }
            bulk_commit();
        }
    } else {
        constexpr int OROWS = DIM == 3 ? B * S::BZ : B;
        constexpr int ROWF = B * K;
        const int nvx = min(B, A.s.res[0] - o[0]);
        const int rowf = nvx * K;
        if (tid < (S::MVG ? 1 : 3) * OROWS) {
            const int which = tid / OROWS, r = tid - which * OROWS;
            const int ly = r % B, lz = DIM == 3 ? r / B : 0;
            const int gy = o[1] + ly, gz = o[2] + lz;
            if (gy < A.s.res[1] && (DIM == 2 || gz < A.s.res[2])) {
                const long long gb = ((DIM == 3 ? (long long)(gz - A.s.zoff) * A.s.sz : 0LL) + (long long)gy * A.s.sy + o[0]) * K;
                const float* src = (which == 0 ? uni : mvs + (which - 1) * S::NOWN * K) + r * ROWF;
                float* dst = (which == 0 ? A.p_out : (which == 1 ? A.m_out : A.v_out)) + gb;
                if ((gb & 3) == 0 && (rowf & 3) == 0) {
                    bulk_s2g(dst, src, (unsigned)rowf * 4);
                    bulk_commit();
                    bulk_wait_read0();  // smem must stay valid until read out
                } else {
                    for (int q = 0; q < rowf; ++q) dst[q] = src[q];
                }
            }
        }
    }

    // ---- per-brick loss partials (fixed-order block reduction; after the
    // copy-out is issued, so the stores overlap it) ----
    {
        const double v4[4] = {warp_sum_d(recon_sum), warp_sum_d(eik_sum), warp_sum_d(tv_sum),
                              warp_sum_d((double)home_pts)};
        if (lane == 0)
            for (int k2 = 0; k2 < 4; ++k2) red[k2][warp] = v4[k2];
        __syncthreads();
        if (tid < 4) {
            double acc = 0.0;
            for (int k2 = 0; k2 < NW; ++k2) acc += red[tid][k2];
            // split clusters: + the other CTAs' recon, eik, home-point sums
            if (SPLIT && tid != 2) acc += xsum[tid == 3 ? 2 : tid];
            A.partials[4 * b + tid] = acc;
        }
    }
#ifdef TGCU_PHASE_TIMING
    if (tid == 0) {
        unsigned long long* ph = g_phase + (unsigned long long)b * kPhaseSlots;
        ph[0] = pt_start;
        ph[1] = pt_tile;
        ph[2] = pt_2a;
        ph[3] = pt_scan;
        ph[4] = pt_bal;
        ph[5] = pt_2b;
        ph[6] = pt_epi;
        ph[7] = gtimer();
        ph[8] = (unsigned long long)(p1 - p0);
        ph[9] = pt_e1;
        ph[10] = pt_e2;
        ph[11] = 0;
    }
#endif
    // (a last-CTA finalize here, behind a per-CTA fence + ticket, measured
    //  15 us slower per C2 step than the separate 1-CTA finalize launch)
    // the CTA's shared memory must outlive the TMA stores' reads
    if (tmap && tid == 0) bulk_wait_read0();
}

// Reduce the per-brick partials in a fixed order, apply the reference's error
// order (NaN point -> non-finite loss -> non-finite gradient) and commit
// (after the brick kernel; slab grids: phase 2, with the globally reduced sums).
// Grids of many bricks (C3: 32,768; C5: 262,144): CTA b sums the partials of
// its contiguous segment in a fixed order into level-2 record b, and the last
// CTA to finish (ticket) runs the finalize over the level-2 records — a fixed
// association whichever CTA is last. One CTA over C3's partials took 21 us.
constexpr int kFinMultiMin = 8192;  // bricks
__global__ void __launch_bounds__(1024) k_step_finalize_multi(FinArgs F, double* l2, unsigned* ticket) {
    __shared__ double red[3][32];
    __shared__ int last;
    pdl_wait();
    pdl_trigger();
    if (F.st->error) return;
    const int seg = (F.NB + gridDim.x - 1) / gridDim.x;
    const int b0 = min(F.NB, (int)blockIdx.x * seg), b1 = min(F.NB, b0 + seg);
    double s3[3];
    block_sum_partials<1024>(F.partials + 4 * (size_t)b0, b1 - b0, red, threadIdx.x, s3);
    if (threadIdx.x == 0) {
        double* o = l2 + 4 * blockIdx.x;
        o[0] = s3[0];
        o[1] = s3[1];
        o[2] = s3[2];
        o[3] = 0.0;
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        if (last) *ticket = 0u;  // every CTA has taken its ticket
    }
    __syncthreads();  // (also orders thread 0's reads of red before the next reduction)
    if (!last) return;
    __threadfence();
    FinArgs F2 = F;
    F2.partials = l2;
    F2.NB = gridDim.x;
    finalize_body<1024>(F2, red, threadIdx.x);
}

// (256 threads measured 0.3 % slower at C2: 4,096 partials per thread block)
constexpr int kFinThreads = 1024;
__global__ void __launch_bounds__(kFinThreads) k_step_finalize(FinArgs F) {
    __shared__ double red[3][kFinThreads / 32];
    pdl_wait();
    pdl_trigger();
    if (F.st->error) return;
    finalize_body<kFinThreads>(F, red, threadIdx.x);
}

// ---- TMA tensor maps of the fused step --------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        TGCU_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw Error(TGCU_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// A (rows = K * res_x floats) x res_y [x zstore] view of one coefficient-layout
// buffer with a box of box_x floats x box_yz rows [x box_yz planes].
bool encode_grid_map(CUtensorMap* m, const Grid& g, const float* base, unsigned box_x, unsigned box_y,
                     unsigned box_z) {
    const int dim = g.spec.dim;
    const cuuint64_t row = (cuuint64_t)g.ds.res[0] * g.K;
    cuuint64_t gdim[3] = {row, (cuuint64_t)g.ds.res[1], (cuuint64_t)g.ds.zstore};
    cuuint64_t gstr[2] = {row * 4, row * 4 * (cuuint64_t)g.ds.res[1]};
    cuuint32_t box[3] = {box_x, box_y, box_z ? box_z : box_y};
    cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = tensor_map_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)dim,
                                            const_cast<float*>(base), gdim, gstr, box, es,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Build the 8 maps once the ping-pong buffers exist. Eligible when the
// compile-time tile layout is dense (BrickSmem::TMAP) and a grid row of K*res_x
// floats is a multiple of 16 bytes (tensor-map stride rule); otherwise the
// kernel stages per row.
static void ensure_tmaps(Grid& g, bool layout_ok, unsigned tile_row_floats) {
    if (g.tm_state != 0) return;
    g.tm_state = -1;
    if (!layout_ok || ((int64_t)g.ds.res[0] * g.K * 4) % 16 != 0) return;
    const int B = g.spec.dim == 3 ? kBrick3 : kBrick2;
    const unsigned BZ = g.spec.dim == 3 ? (unsigned)kBrickZ3 : 1u;
    const unsigned T = (unsigned)B + 2;
    bool ok = true;
    for (int i = 0; i < 2; ++i) {
        ok = ok && encode_grid_map(&g.tm_tile[i], g, g.p[i], tile_row_floats, T, BZ + 2);
        ok = ok && encode_grid_map(&g.tm_own_p[i], g, g.p[i], (unsigned)B * g.K, (unsigned)B, BZ);
        ok = ok && encode_grid_map(&g.tm_own_m[i], g, g.m[i], (unsigned)B * g.K, (unsigned)B, BZ);
        ok = ok && encode_grid_map(&g.tm_own_v[i], g, g.v[i], (unsigned)B * g.K, (unsigned)B, BZ);
    }
    if (ok) g.tm_state = 1;
}

__global__ void k_pack_eik(const float* __restrict__ p3, long long n, float4* __restrict__ dst) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[i] = make_float4(p3[3 * i], p3[3 * i + 1], p3[3 * i + 2], __uint_as_float(kEikMark));
}

void launch_pack_eik(const float* p3, int64_t n, float4* dst, cudaStream_t s) {
    k_pack_eik<<<grid_blocks(n, 256), 256, 0, s>>>(p3, n, dst);
    count_launch();
    TGCU_CUDA(cudaGetLastError());
}

// Slab phase 2: commit with the globally reduced sums.
void launch_slab_finish(Grid& g, const double* reduced, const tgcu_loss_config& cfg, int in_idx, int64_t step,
                        int64_t t_after, int64_t n, cudaStream_t s) {
    FinArgs F{};
    F.NB = (int)g.NB;
    F.n = (double)n;
    F.lambda1 = cfg.lambda1;
    F.lambda2 = cfg.lambda2;
    F.inv_norm = g.tv_inv_norm;
    F.use_tv = cfg.use_tv;
    F.want_eik = cfg.lambda1 > 0.0;
    F.st = g.st;
    F.nan = &g.st->nan_bin[g.slab_set];
    F.over = &g.st->det_over[g.slab_set];
    F.trace = g.d_trace;
    F.step = step;
    F.in_idx = in_idx;
    F.t_after = t_after;
    F.reduced = reduced;
    k_step_finalize<<<1, 32, 0, s>>>(F);
    count_launch();
    TGCU_CUDA(cudaGetLastError());
}

// Deterministic mode: each brick's binned point copies in canonical order
// (the float4 records' bits, lexicographic), since the binning scatter
// reserves slots with shared-memory atomics. Bitonic sort of the brick's run
// in shared memory: bricks of at most one chunk by 256-thread CTAs (one per
// brick), the multi-chunk ("heavy", listed first in the launch order) bricks
// by a persistent kernel of 1024-thread CTAs, up to kDetSortCap copies (a
// larger brick is an error).
constexpr int kDetSortCap = 4096;
__device__ __forceinline__ bool rec_less(const float4& a, const float4& b) {
    const unsigned a0 = __float_as_uint(a.x), a1 = __float_as_uint(a.y), a2 = __float_as_uint(a.z),
                   a3 = __float_as_uint(a.w);
    const unsigned b0 = __float_as_uint(b.x), b1 = __float_as_uint(b.y), b2 = __float_as_uint(b.z),
                   b3 = __float_as_uint(b.w);
    if (a0 != b0) return a0 < b0;
    if (a1 != b1) return a1 < b1;
    if (a2 != b2) return a2 < b2;
    return a3 < b3;
}
__device__ void sort_run(float4* __restrict__ binned, int p0, int n, float4* rs) {
    int np = 1;
    while (np < n) np <<= 1;
    const float4 pad = make_float4(__int_as_float(-1), __int_as_float(-1), __int_as_float(-1), __int_as_float(-1));
    for (int i = threadIdx.x; i < np; i += blockDim.x) rs[i] = i < n ? binned[p0 + i] : pad;  // padding sorts last
    __syncthreads();
    for (int k = 2; k <= np; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < np; i += blockDim.x) {
                const int ix = i ^ j;
                if (ix > i) {
                    const float4 a = rs[i], c = rs[ix];
                    if (((i & k) == 0) == rec_less(c, a)) {
                        rs[i] = c;
                        rs[ix] = a;
                    }
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < n; i += blockDim.x) binned[p0 + i] = rs[i];
    __syncthreads();
}
__global__ void __launch_bounds__(256) k_bin_sort_small(float4* __restrict__ binned, const int* __restrict__ off,
                                                       int NB, int ch) {
    __shared__ float4 rs[512];
    const int b = blockIdx.x;
    const int p0 = off[b], n = off[b + 1] - p0;
    if (n <= 1 || n > ch) return;
    sort_run(binned, p0, n, rs);
}
__global__ void __launch_bounds__(1024) k_bin_sort_heavy(float4* __restrict__ binned, const int* __restrict__ off,
                                                        const int* __restrict__ ord, int NB,
                                                        unsigned long long* __restrict__ over) {
    extern __shared__ float4 rh[];
    const int nh = ord[NB];
    for (int i = blockIdx.x; i < nh; i += gridDim.x) {
        const int b = ord[i];
        const int p0 = off[b], n = off[b + 1] - p0;
        if (n > kDetSortCap) {  // reported by this step's finalize (like a NaN sample)
            if (threadIdx.x == 0) atomicMin(over, (unsigned long long)b);
            continue;
        }
        sort_run(binned, p0, n, rh);
    }
}

void launch_train_step(Grid& g, const float4* samples, int64_t n, int64_t n_norm, const tgcu_loss_config& cfg,
                       int in_idx,
                       int64_t step, double inv_bc1, double inv_bc2, int64_t t_after, float* grad_out,
                       double* slab_out, const BinInput& in, cudaStream_t s, bool fresh_eik) {
    // Small grids: the whole step as one cooperative launch (small.cu)
    if (!slab_out && small_step_eligible(g, n)) {
        launch_small_step(g, samples, n, n_norm, cfg, in_idx, step, inv_bc1, inv_bc2, t_after, grad_out, in, s,
                          fresh_eik);
        return;
    }
    // Binning runs on the binning stream into bin set k; the brick kernel
    // (caller's stream) waits for it and releases the set when done, so the
    // binning of the next step overlaps this step's brick kernel whenever its
    // input order allows (BinInput).
    ensure_bin_stream(g);
    const int k = g.bin_set;
    g.bin_set ^= 1;
    if (slab_out) g.slab_set = k;
    ensure_bins(g, k, n);
    cudaStream_t bs = g.bstream;
    if (in.wait) {
        TGCU_CUDA(cudaStreamWaitEvent(bs, in.wait, 0));
    } else if (!in.ready) {
        TGCU_CUDA(cudaEventRecord(g.ev_in, s));
        TGCU_CUDA(cudaStreamWaitEvent(bs, g.ev_in, 0));
    }
    TGCU_CUDA(cudaStreamWaitEvent(bs, g.ev_bfree[k], 0));  // brick kernel of step i-2 done with set k
    BinArgs B;
    B.s = g.ds;
    B.pts = samples;
    B.n = n;
    for (int a = 0; a < 3; ++a) B.nb[a] = g.nb[a];
    B.count = g.bin_count;
    B.cursor = g.bin_cursor;
    B.binned = g.binned[k];
    B.nan = &g.st->nan_bin[k];
    B.zb0 = g.zb0;
    B.sh1 = g.code_sh[0];
    B.sh2 = g.code_sh[1];
    int* const off = g.bin_off[k];
    int* const ord = g.brick_order[k];  // NB entries + 2 class counters
    const int ch = g.spec.dim == 3 ? BrickShape<3>::CH : BrickShape<2>::CH;
    TGCU_CUDA(cudaMemsetAsync(ord + g.NB, 0, 2 * sizeof(int), bs));
    const int ncta_tiles = (int)((n + kBinTile - 1) / kBinTile);
    if (g.bd_on) bd_mark(g, bs, 0);
    if (n == 0) {
        // a slab rank with no local points: every brick empty (TV + Adam only)
        TGCU_CUDA(cudaMemsetAsync(off, 0, sizeof(int) * (g.NB + 1), bs));
        k_identity_order<<<grid_blocks(g.NB, 256), 256, 0, bs>>>(ord, (int)g.NB);
        if (g.bd_on) {
            bd_mark(g, bs, 1);
            bd_mark(g, bs, 2);
        }
    } else if (g.NB <= kBinSmemMax && ncta_tiles <= kMaxBinTiles) {
        const int ncta = ncta_tiles;
        ensure_bin_hist(g, (int64_t)ncta * g.NB, n, (g.NB + kColBricks - 1) / kColBricks);
        const size_t sm = sizeof(int) * g.NB;
        const size_t csm = sizeof(int) * ncta * (kColBricks + 1);
        // function attributes are per device: set them once for each device used
        static std::atomic<unsigned long long> attr_devs{0};
        const unsigned long long dbit = 1ull << (g.device & 63);
        if (!(attr_devs.load() & dbit)) {
            TGCU_CUDA(cudaFuncSetAttribute(k_bin_hist<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kBinSmemMax));
            TGCU_CUDA(cudaFuncSetAttribute(k_bin_hist<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kBinSmemMax));
            TGCU_CUDA(cudaFuncSetAttribute(k_bin_scatter_tiles<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kBinSmemMax));
            TGCU_CUDA(cudaFuncSetAttribute(k_bin_scatter_tiles<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kBinSmemMax));
            TGCU_CUDA(cudaFuncSetAttribute(k_bin_cols, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(sizeof(int) * kMaxBinTiles * (kColBricks + 1))));
            attr_devs.fetch_or(dbit);
        }
        if (g.spec.dim == 3) k_bin_hist<3><<<ncta, kBinThreads, sm, bs>>>(B, g.bin_hist, g.bin_codes, (int)g.NB);
        else k_bin_hist<2><<<ncta, kBinThreads, sm, bs>>>(B, g.bin_hist, g.bin_codes, (int)g.NB);
        if (g.bd_on) bd_mark(g, bs, 1);
        const int epoch = ++g.bin_epoch;
        k_bin_cols<<<(unsigned)((g.NB + kColBricks - 1) / kColBricks), 256, csm, bs>>>(
            g.bin_hist, ncta, (int)g.NB, off, g.bin_chain,
            reinterpret_cast<unsigned long long*>(g.bin_chain + 2 * g.bin_chain_cap), epoch, ch, ord);
        if (g.bd_on) bd_mark(g, bs, 2);
        if (g.spec.dim == 3)
            k_bin_scatter_tiles<3><<<ncta, kBinThreads, sm, bs>>>(B, g.bin_hist, g.bin_codes, off, (int)g.NB);
        else
            k_bin_scatter_tiles<2><<<ncta, kBinThreads, sm, bs>>>(B, g.bin_hist, g.bin_codes, off, (int)g.NB);
        count_launch(3);
    } else {
        if (g.bd_on) bd_mark(g, bs, 1);
        TGCU_CUDA(cudaMemsetAsync(g.bin_count, 0, sizeof(int) * g.NB, bs));
        const int pblocks = grid_blocks(n, 256, 148 * 16);
        if (g.spec.dim == 3) k_bin_count<3><<<pblocks, 256, 0, bs>>>(B);
        else k_bin_count<2><<<pblocks, 256, 0, bs>>>(B);
        k_bin_scan<<<1, 1024, 0, bs>>>(g.bin_count, off, g.bin_cursor, (int)g.NB, ch, ord);
        if (g.bd_on) bd_mark(g, bs, 2);
        if (g.spec.dim == 3) k_bin_scatter<3><<<pblocks, 256, 0, bs>>>(B);
        else k_bin_scatter<2><<<pblocks, 256, 0, bs>>>(B);
        count_launch(3);
    }
    if (g.deterministic) {
        static std::atomic<unsigned long long> det_devs{0};
        const unsigned long long dbit = 1ull << (g.device & 63);
        if (!(det_devs.load() & dbit)) {
            TGCU_CUDA(cudaFuncSetAttribute(k_bin_sort_heavy, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(sizeof(float4) * kDetSortCap)));
            det_devs.fetch_or(dbit);
        }
        k_bin_sort_small<<<(unsigned)g.NB, 256, 0, bs>>>(g.binned[k], off, (int)g.NB, ch);
        k_bin_sort_heavy<<<(unsigned)std::min<int64_t>(g.NB, 148 * 3), 1024, sizeof(float4) * kDetSortCap, bs>>>(
            g.binned[k], off, ord, (int)g.NB, &g.st->det_over[k]);
        count_launch(2);
    }
    TGCU_CUDA(cudaGetLastError());
    if (in.consumed) TGCU_CUDA(cudaEventRecord(in.consumed, bs));
    TGCU_CUDA(cudaEventRecord(g.ev_bdone[k], bs));
    TGCU_CUDA(cudaStreamWaitEvent(s, g.ev_bdone[k], 0));

    StepArgs A{};
    A.s = g.ds;
    const int out_idx = 1 - in_idx;
    A.p_in = g.p[in_idx];
    A.p_out = g.p[out_idx];
    A.m_in = g.m[in_idx];
    A.m_out = g.m[out_idx];
    A.v_in = g.v[in_idx];
    A.v_out = g.v[out_idx];
    A.binned = g.binned[k];
    A.off = off;
    A.det = g.deterministic ? 1 : 0;
    for (int a = 0; a < 3; ++a) A.nb[a] = g.nb[a];
    A.L.k = cfg.k;
    A.L.inv_n = 1.0 / (double)n_norm;  // the global batch size (slab ranks may read a subset)
    A.L.eik_scale = cfg.lambda1;
    A.L.use_weighting = cfg.use_weighting;
    A.L.differentiate_weight = cfg.differentiate_weight;
    A.L.fresh_eik = fresh_eik ? 1 : 0;
    // TV normaliser P*K over the global grid (sdf_loss.cpp:161-170).
    const double inv_norm = g.tv_inv_norm;
    A.want_tv = cfg.use_tv ? 1 : 0;
    A.tv_gscale = (cfg.use_tv && cfg.lambda2 > 0.0) ? (float)(2.0 * cfg.lambda2 * inv_norm) : 0.0f;
    A.lr = (float)g.adam.lr;
    A.b1 = (float)g.adam.beta1;
    A.b2 = (float)g.adam.beta2;
    A.c1 = (float)(1.0 - g.adam.beta1);
    A.c2 = (float)(1.0 - g.adam.beta2);
    A.eps = (float)g.adam.eps;
    A.inv_bc1 = (float)inv_bc1;
    A.inv_bc2 = (float)inv_bc2;
    A.partials = g.partials;
    A.st = g.st;
    A.grad_out = grad_out;
    A.zb0 = g.zb0;
    A.order = g.brick_order[k];
    A.NB = (int)g.NB;
    A.peer_lo = g.peer_lo[out_idx];
    A.peer_hi = g.peer_hi[out_idx];
    {
        const int own_hi = std::min(g.spec.res[2], kBrickZ3 * (g.zb0 + g.nb[2]));
        A.peer_hi_zb = (own_hi - 1) / kBrickZ3;
        A.peer_hi_lz = (own_hi - 1) % kBrickZ3;
    }
    const bool eik = cfg.lambda1 > 0.0;
    FinArgs F{};
    F.partials = g.partials;
    F.NB = (int)g.NB;
    F.n = (double)n_norm;
    F.lambda1 = cfg.lambda1;
    F.lambda2 = cfg.lambda2;
    F.inv_norm = inv_norm;
    F.use_tv = cfg.use_tv;
    F.want_eik = eik;
    F.st = g.st;
    F.nan = &g.st->nan_bin[k];
    F.over = &g.st->det_over[k];
    F.trace = g.d_trace;
    F.step = step;
    F.in_idx = in_idx;
    F.t_after = t_after;
    F.slab_out = slab_out;
    F.reduced = nullptr;
    TGCU_DISPATCH(g.spec.dim, g.spec.order,
                  { ensure_tmaps(g, BrickSmem<DIM, ORDER>::TMAP, BrickSmem<DIM, ORDER>::TROWF); });
    A.use_tmap = g.tm_state == 1 ? 1 : 0;
    if (A.use_tmap) {
        A.tm_tile = g.tm_tile[in_idx];
        A.tm_m_in = g.tm_own_m[in_idx];
        A.tm_v_in = g.tm_own_v[in_idx];
        A.tm_p_out = g.tm_own_p[out_idx];
        A.tm_m_out = g.tm_own_m[out_idx];
        A.tm_v_out = g.tm_own_v[out_idx];
    }
    // Split bricks over a cluster of CTAs when the grid has fewer bricks than
    // SMs: the largest power of two <= 8 that keeps one CTA per SM (C1, 64
    // bricks: split 2, 22.6 us per step; split 4 on two CTA slots per SM:
    // 23.9 us).
    int split = 1;
#ifndef TGCU_SPLIT_OFF
    if (A.use_tmap) {
        static int sms = 0;
        if (!sms) TGCU_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g.device));
        const char* ev = std::getenv("TGCU_SPLIT");
        const int cap = ev ? std::max(1, std::min(8, std::atoi(ev))) : 8;
        while (split * 2 <= cap && g.NB * (int64_t)split * 2 <= (int64_t)sms) split *= 2;
    }
#endif
    A.split = split;
    const dim3 bgrid((unsigned)(g.NB * split));
    TGCU_DISPATCH(g.spec.dim, g.spec.order, {
        constexpr size_t smem = BrickSmem<DIM, ORDER>::bytes;
        static_assert(BrickSmem<DIM, ORDER>::bytes <= 227 * 1024, "brick smem");
        // sparse batches (few point copies per brick on average) take the
        // variant with the tiny-brick path compiled in
        const bool sparse = (double)n * (DIM == 3 ? 1.42 : 1.13) < 64.0 * (double)g.NB;
        auto pick = [&](auto k_t, auto k_f) { return sparse ? k_t : k_f; };
        auto kern = grad_out
            ? (eik ? pick(k_brick_step<DIM, ORDER, true, true, true>, k_brick_step<DIM, ORDER, true, true, false>)
                   : pick(k_brick_step<DIM, ORDER, false, true, true>, k_brick_step<DIM, ORDER, false, true, false>))
            : (eik ? pick(k_brick_step<DIM, ORDER, true, false, true>, k_brick_step<DIM, ORDER, true, false, false>)
                   : pick(k_brick_step<DIM, ORDER, false, false, true>, k_brick_step<DIM, ORDER, false, false, false>));
        if (split > 1)  // the cluster variants (no tiny-brick path)
            kern = grad_out ? (eik ? k_brick_step<DIM, ORDER, true, true, false, true>
                                   : k_brick_step<DIM, ORDER, false, true, false, true>)
                            : (eik ? k_brick_step<DIM, ORDER, true, false, false, true>
                                   : k_brick_step<DIM, ORDER, false, false, false, true>);
        static std::atomic<unsigned long long> configured_devs{0};
        const unsigned long long cbit = 1ull << (g.device & 63);
        if (!(configured_devs.load() & cbit)) {
            for (auto k : {k_brick_step<DIM, ORDER, true, true, true>, k_brick_step<DIM, ORDER, false, true, true>,
                           k_brick_step<DIM, ORDER, true, false, true>, k_brick_step<DIM, ORDER, false, false, true>,
                           k_brick_step<DIM, ORDER, true, true, false>, k_brick_step<DIM, ORDER, false, true, false>,
                           k_brick_step<DIM, ORDER, true, false, false>, k_brick_step<DIM, ORDER, false, false, false>,
                           k_brick_step<DIM, ORDER, true, true, false, true>, k_brick_step<DIM, ORDER, false, true, false, true>,
                           k_brick_step<DIM, ORDER, true, false, false, true>,
                           k_brick_step<DIM, ORDER, false, false, false, true>})
                TGCU_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            configured_devs.fetch_or(cbit);
        }
        g.prof_this = g.prof_on && (g.steps_launched % g.prof_every) == 0;
        if (g.prof_this) prof_mark(g, s, 0);
        if (g.bd_on) bd_mark(g, s, 3);
        {
            cudaLaunchConfig_t lc{};
            lc.gridDim = bgrid;
            lc.blockDim = dim3(BrickShape<DIM>::NT);
            lc.dynamicSmemBytes = smem;
            lc.stream = s;
            cudaLaunchAttribute at[2];
            int na = 0;
            if (g.brick_pdl) {
                at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[na].val.programmaticStreamSerializationAllowed = 1;
                ++na;
            }
            if (split > 1) {
                at[na].id = cudaLaunchAttributeClusterDimension;
                at[na].val.clusterDim.x = (unsigned)split;
                at[na].val.clusterDim.y = 1;
                at[na].val.clusterDim.z = 1;
                ++na;
            }
            lc.attrs = at;
            lc.numAttrs = na;
            TGCU_CUDA(cudaLaunchKernelEx(&lc, kern, A));
        }
        // bin set k is free once the brick kernel is done (recorded after
        // the finalize instead, the next binning overlapped this step's brick
        // kernel worse: C2 0.2650 -> 0.2717 ms per step)
        TGCU_CUDA(cudaEventRecord(g.ev_bfree[k], s));
        if (g.bd_on) bd_mark(g, s, 4);
        if (g.prof_this) prof_mark(g, s, 1);
    });

    // the finalize follows the brick kernel on s (programmatic dependent launch)
    if (g.NB >= kFinMultiMin && !g.fin_l2) {
        TGCU_CUDA(cudaMalloc(&g.fin_l2, sizeof(double) * (4 * 148 + 1)));
        TGCU_CUDA(cudaMemsetAsync(g.fin_l2 + 4 * 148, 0, sizeof(double), s));
    }
    {
        cudaLaunchConfig_t lc{};
        lc.blockDim = dim3(1024);
        lc.dynamicSmemBytes = 0;
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = g.brick_pdl ? 1 : 0;
        if (g.NB >= kFinMultiMin) {
            lc.gridDim = dim3((unsigned)std::min<int64_t>(148, (g.NB + 1023) / 1024));
            TGCU_CUDA(cudaLaunchKernelEx(&lc, k_step_finalize_multi, F, g.fin_l2,
                                         reinterpret_cast<unsigned*>(g.fin_l2 + 4 * 148)));
        } else {
            lc.gridDim = dim3(1);
            lc.blockDim = dim3(kFinThreads);
            TGCU_CUDA(cudaLaunchKernelEx(&lc, k_step_finalize, F));
        }
    }
    count_launch(2);
    TGCU_CUDA(cudaGetLastError());
    if (g.bd_on) {
        bd_mark(g, s, 5);
        bd_collect(g);
    }
}

}  // namespace tgcu

#ifdef TGCU_PHASE_TIMING
extern "C" int tgcu_phase_dump(unsigned long long* out, int ncta) {
    return cudaMemcpyFromSymbol(out, tgcu::g_phase, sizeof(unsigned long long) * ncta * tgcu::kPhaseSlots) ==
                   cudaSuccess
               ? 0
               : 6;
}
#endif
