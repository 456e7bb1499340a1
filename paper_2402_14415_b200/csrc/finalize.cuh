// Step finalize shared by the fused brick step (train.cu) and the
// single-launch small-grid step (small.cu): the per-CTA loss partials reduced
// in a fixed order, the reference's error order (NaN point -> non-finite loss
// -> non-finite gradient; sdf_loss.cpp:259-292, adam.cpp:18-34) and the commit.
#pragma once

#include <climits>

#include "tg_internal.h"

namespace tgcu {

struct FinArgs {
    const double* partials;
    int NB;
    double n;
    double lambda1, lambda2, inv_norm;
    int use_tv, want_eik;
    Status* st;
    unsigned long long* nan;  // NaN slot of the step's bin set
    unsigned long long* over; // deterministic-sort overflow slot of the step's bin set
    tgcu_loss_terms* trace;
    long long step;
    int in_idx;
    long long t_after;
    long long* ctr;         // graph-replayed steps: {t, step} on the device (step / t_after read
                            // from it, then advanced); nullptr: step / t_after above
    double* slab_out;       // slab phase 1: write local {recon, eik, tv, has_nan, has_bad}, no commit
    const double* reduced;  // slab phase 2: globally summed {recon, eik, tv, n_nan, n_bad}
};

// Fixed-order sums of NB partial records {recon, eik, tv, points} (4 doubles
// each): thread-strided sums, warp trees, then warp order; out[] valid in
// thread 0. Every thread must call it (one block barrier inside).
template <int NTH>
__device__ void block_sum_partials(const double* partials, int NB, double (*red)[NTH / 32], int tid, double* out) {
    double a = 0.0, b = 0.0, c = 0.0;
    // 16-byte loads, unrolled so a thread's loads are all in flight before its
    // sums; L2 loads (the small step writes the partials in the same launch)
    const double2* P2 = reinterpret_cast<const double2*>(partials);
#pragma unroll 4
    for (int i = tid; i < NB; i += NTH) {
        const double2 x = __ldcg(P2 + 2 * i), y = __ldcg(P2 + 2 * i + 1);
        a += x.x;
        b += x.y;
        c += y.x;
    }
    a = warp_sum_d(a);
    b = warp_sum_d(b);
    c = warp_sum_d(c);
    if ((tid & 31) == 0) {
        red[0][tid >> 5] = a;
        red[1][tid >> 5] = b;
        red[2][tid >> 5] = c;
    }
    __syncthreads();
    if (tid == 0) {
        out[0] = out[1] = out[2] = 0.0;
        for (int k = 0; k < NTH / 32; ++k) {
            out[0] += red[0][k];
            out[1] += red[1][k];
            out[2] += red[2][k];
        }
    }
}

template <int NTH>
__device__ void finalize_body(const FinArgs& F, double (*red)[NTH / 32], int tid) {
    double recon = 0.0, eik = 0.0, tvs = 0.0;
    // the status words thread 0 decides on, loaded before the reduction so
    // their L2 round trip overlaps it
    unsigned long long nanp = 0, over = 0, badg = 0;
    if (tid == 0) {
        nanp = __ldcg(F.nan);
        over = __ldcg(F.over);
        badg = __ldcg(&F.st->bad_grad);
    }
    if (!F.reduced) {
        double s3[3];
        block_sum_partials<NTH>(F.partials, F.NB, red, tid, s3);
        recon = s3[0];
        eik = s3[1];
        tvs = s3[2];
    } else if (tid == 0) {
        recon = F.reduced[0];
        eik = F.reduced[1];
        tvs = F.reduced[2];
    }
    if (tid != 0) return;
    Status* st = F.st;
    if (F.slab_out) {
        F.slab_out[0] = recon;
        F.slab_out[1] = eik;
        F.slab_out[2] = tvs;
        F.slab_out[3] = nanp != ULLONG_MAX ? 1.0 : 0.0;
        F.slab_out[4] = badg != ULLONG_MAX ? 1.0 : 0.0;
        return;
    }
    const bool any_nan = nanp != ULLONG_MAX || (F.reduced && F.reduced[3] > 0.0);
    const bool any_bad = badg != ULLONG_MAX || (F.reduced && F.reduced[4] > 0.0);
    tgcu_loss_terms t;
    t.fit = recon / F.n;
    t.eik = F.want_eik ? eik / F.n : 0.0;
    t.tv = F.use_tv ? tvs * F.inv_norm : 0.0;
    t.total = t.fit + F.lambda1 * t.eik + F.lambda2 * t.tv;
    const long long step = F.ctr ? F.ctr[1] : F.step;
    const long long t_after = F.ctr ? F.ctr[0] + 1 : F.t_after;
    F.trace[step % kTraceCap] = t;
    int err = 0, kind = 0;
    long long idx = -1;
    if (any_nan) {
        err = TGCU_ERR_INVALID_ARGUMENT;
        kind = 1;
        idx = nanp != ULLONG_MAX ? (long long)nanp : -1;
    } else if (over != ULLONG_MAX) {
        err = TGCU_ERR_CONFIG;
        kind = 4;
        idx = (long long)over;
    } else if (!isfinite(t.total)) {
        err = TGCU_ERR_NUMERICAL;
        kind = 2;
    } else if (any_bad) {
        err = TGCU_ERR_NUMERICAL;
        kind = 3;
        idx = badg != ULLONG_MAX ? (long long)badg : -1;
    }
    if (err) {
        st->error = err;
        st->error_kind = kind;
        st->error_step = step;
        st->error_index = idx;
        st->good_idx = F.in_idx;
        st->good_t = t_after - 1;
    } else {
        st->good_idx = 1 - F.in_idx;
        st->good_t = t_after;
    }
    *F.nan = ULLONG_MAX;
    *F.over = ULLONG_MAX;
    st->bad_grad = ULLONG_MAX;
    if (F.ctr) {  // the next replayed step's t and trace slot (a failed step leaves the
        F.ctr[0] = t_after;  // later ones no-ops; the host resets the counter with its state)
        F.ctr[1] = step + 1;
    }
}

}  // namespace tgcu
