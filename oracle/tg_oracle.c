/*
 * TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT. See tg_oracle.h.
 *
 * Plain-C fp64 restatement of the reference hot path. Every operation keeps
 * the reference's association order (no FMA contraction: built with
 * -ffp-contract=off) so results agree with the reference build bit for bit;
 * tests/test_oracle_cpu.py asserts exactly that.
 */
#include "tg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <stddef.h>
#include <string.h>

/* Hessian upper-triangle pairs, row-major (taylor_grid.cpp:14-15). */
static const int kPairs2[3][2] = {{0, 0}, {0, 1}, {1, 1}};
static const int kPairs3[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};

int tgo_coeff_count(int order, int dim) {
    if (dim != 2 && dim != 3) return -1;
    if (order < 0 || order > 2) return -1;
    if (order == 0) return 1;
    if (order == 1) return 1 + dim;
    return 1 + dim + dim * (dim + 1) / 2;
}

int64_t tgo_vertex_count(const tgo_spec* s) {
    int64_t n = 1;
    for (int a = 0; a < s->dim; ++a) n *= s->res[a];
    return n;
}

/* GridSpec::spacing (grid_spec.hpp:29). */
static double spacing(const tgo_spec* s, int a) { return s->extent[a] / (s->res[a] - 1); }

/* GridSpec::vertex_index, x fastest (grid_spec.hpp:41-45). */
static int64_t vertex_index(const tgo_spec* s, const int v[3]) {
    int64_t idx = v[s->dim - 1];
    for (int a = s->dim - 2; a >= 0; --a) idx = idx * s->res[a] + v[a];
    return idx;
}

/* locate: NaN check, clamp_point, fp64 division, floor, clamp to the last
 * cell (grid_spec.cpp:35-43, :45-69). */
int tgo_locate(const tgo_spec* s, const double p_in[3], int cell[3], double local[3],
               int64_t vid[8]) {
    for (int a = 0; a < s->dim; ++a)
        if (isnan(p_in[a])) return -1;
    cell[0] = cell[1] = cell[2] = 0;
    local[0] = local[1] = local[2] = 0.0;
    for (int a = 0; a < s->dim; ++a) {
        const double lo = s->origin[a];
        const double hi = s->origin[a] + s->extent[a];
        const double p = p_in[a] < lo ? lo : (p_in[a] > hi ? hi : p_in[a]);
        const double h = spacing(s, a);
        const double t = (p - s->origin[a]) / h;
        int c = (int)floor(t);
        const int max_cell = s->res[a] - 2;
        if (c < 0) c = 0;
        if (c > max_cell) c = max_cell;
        cell[a] = c;
        local[a] = t - c;
    }
    const int corners = 1 << s->dim;
    for (int c = 0; c < corners; ++c) {
        int v[3] = {cell[0], cell[1], cell[2]};
        for (int a = 0; a < s->dim; ++a) v[a] += (c >> a) & 1;
        vid[c] = vertex_index(s, v);
    }
    return 0;
}

/* Per-corner multilinear geometry (taylor_grid.cpp:29-64). */
typedef struct {
    int count;
    double w[8];
    double dw[8][3];
    double delta[8][3];
    int64_t vid[8];
} corners_t;

static void make_corners(const tgo_spec* s, const double local[3], const int64_t vid[8],
                         corners_t* c) {
    double h[3] = {1.0, 1.0, 1.0};
    double inv_h[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < s->dim; ++a) {
        h[a] = spacing(s, a);
        inv_h[a] = 1.0 / h[a];
    }
    c->count = 1 << s->dim;
    for (int i = 0; i < c->count; ++i) {
        double sa[3];
        int bit[3] = {0, 0, 0};
        for (int a = 0; a < s->dim; ++a) {
            bit[a] = (i >> a) & 1;
            sa[a] = bit[a] ? local[a] : 1.0 - local[a];
        }
        double w = 1.0;
        for (int a = 0; a < s->dim; ++a) w *= sa[a];
        c->w[i] = w;
        for (int a = 0; a < 3; ++a) c->dw[i][a] = 0.0;
        for (int a = 0; a < s->dim; ++a) {
            double other = 1.0;
            for (int b = 0; b < s->dim; ++b)
                if (b != a) other *= sa[b];
            c->dw[i][a] = (bit[a] ? 1.0 : -1.0) * inv_h[a] * other;
        }
        for (int a = 0; a < 3; ++a) c->delta[i][a] = 0.0;
        for (int a = 0; a < s->dim; ++a) c->delta[i][a] = (local[a] - bit[a]) * h[a];
        c->vid[i] = vid[i];
    }
}

/* One vertex's truncated Taylor polynomial and its offset gradient
 * (taylor_grid.cpp:68-98). grad may be NULL. */
static double taylor_poly(const double* b, int order, int dim, const double d[3], double grad[3]) {
    double v = b[0];
    if (grad) grad[0] = grad[1] = grad[2] = 0.0;
    if (order >= 1) {
        for (int a = 0; a < dim; ++a) {
            v += b[1 + a] * d[a];
            if (grad) grad[a] += b[1 + a];
        }
    }
    if (order >= 2) {
        const int(*pairs)[2] = dim == 2 ? kPairs2 : kPairs3;
        const int npairs = dim * (dim + 1) / 2;
        const double* q = b + 1 + dim;
        for (int t = 0; t < npairs; ++t) {
            const int j = pairs[t][0], k = pairs[t][1];
            const double c = q[t];
            if (j == k) {
                v += 0.5 * c * d[j] * d[j];
                if (grad) grad[j] += c * d[j];
            } else {
                v += c * d[j] * d[k];
                if (grad) {
                    grad[j] += c * d[k];
                    grad[k] += c * d[j];
                }
            }
        }
    }
    return v;
}

double tgo_eval(const tgo_spec* s, const double* coeffs, const double p[3], double grad_out[3]) {
    int cell[3];
    double local[3];
    int64_t vid[8];
    if (tgo_locate(s, p, cell, local, vid) != 0) return NAN;
    corners_t c;
    make_corners(s, local, vid, &c);
    const int K = tgo_coeff_count(s->order, s->dim);
    double value = 0.0;
    double g[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < c.count; ++i) {
        const double* b = coeffs + c.vid[i] * K;
        double tg[3];
        const double tv = taylor_poly(b, s->order, s->dim, c.delta[i], grad_out ? tg : NULL);
        value += c.w[i] * tv;
        if (grad_out)
            for (int a = 0; a < s->dim; ++a) g[a] += c.dw[i][a] * tv + c.w[i] * tg[a];
    }
    if (grad_out) {
        grad_out[0] = g[0];
        grad_out[1] = g[1];
        grad_out[2] = g[2];
    }
    return value;
}

/* tgo_eval over fp32-stored coefficients (each upcast exactly before use, so
 * the arithmetic is tgo_eval's on the same values), batched: lets a parity
 * test evaluate the oracle on a multi-GB fp32 device grid downloaded as is
 * (BASELINE C4, 512^3) without a second fp64 copy. */
void tgo_eval_batch_f32(const tgo_spec* s, const float* coeffs, const double* pts, int64_t n, double* vals,
                        double* grads, double* l1) {
    const int K = tgo_coeff_count(s->order, s->dim);
    for (int64_t q = 0; q < n; ++q) {
        const double* p = pts + 3 * q;
        int cell[3];
        double local[3];
        int64_t vid[8];
        if (tgo_locate(s, p, cell, local, vid) != 0) {
            vals[q] = NAN;
            continue;
        }
        corners_t c;
        make_corners(s, local, vid, &c);
        double value = 0.0;
        double g[3] = {0.0, 0.0, 0.0}, m[3] = {0.0, 0.0, 0.0};
        for (int i = 0; i < c.count; ++i) {
            double b[10];
            for (int k = 0; k < K; ++k) b[k] = (double)coeffs[c.vid[i] * K + k];
            double tg[3];
            const double tv = taylor_poly(b, s->order, s->dim, c.delta[i], (grads || l1) ? tg : NULL);
            value += c.w[i] * tv;
            if (grads || l1)
                for (int a = 0; a < s->dim; ++a) {
                    g[a] += c.dw[i][a] * tv + c.w[i] * tg[a];
                    m[a] += fabs(c.dw[i][a] * tv) + fabs(c.w[i] * tg[a]);
                }
        }
        vals[q] = value;
        if (grads)
            for (int a = 0; a < 3; ++a) grads[3 * q + a] = g[a];
        if (l1) /* per axis: the L1 size of the terms summed into the spatial gradient */
            for (int a = 0; a < 3; ++a) l1[3 * q + a] = m[a];
    }
}

/* Test helper for the gradient tolerance: per axis, the L1 size of the terms
 * whose sum is the spatial gradient (sum_i |dw_i,a T_i| + |w_i gT_i,a|). An
 * fp32 forward resolves grad f only to ~eps32 times this, which on fine grids
 * (dw ~ 1/h) is far larger than |grad f| itself. */
static void eval_grad_l1(const tgo_spec* s, const double* coeffs, const double p[3], double l1[3]) {
    int cell[3];
    double local[3];
    int64_t vid[8];
    l1[0] = l1[1] = l1[2] = 0.0;
    if (tgo_locate(s, p, cell, local, vid) != 0) return;
    corners_t c;
    make_corners(s, local, vid, &c);
    const int K = tgo_coeff_count(s->order, s->dim);
    for (int i = 0; i < c.count; ++i) {
        const double* b = coeffs + c.vid[i] * K;
        double tg[3];
        const double tv = taylor_poly(b, s->order, s->dim, c.delta[i], tg);
        for (int a = 0; a < s->dim; ++a) l1[a] += fabs(c.dw[i][a] * tv) + fabs(c.w[i] * tg[a]);
    }
}

/* accumulate_cell (taylor_grid.cpp:123-152). */
static void accumulate_cell(const tgo_spec* s, const corners_t* c, double upstream,
                            const double gvec[3], double* grad) {
    const int K = tgo_coeff_count(s->order, s->dim);
    const int dim = s->dim;
    for (int i = 0; i < c->count; ++i) {
        double* g = grad + c->vid[i] * K;
        const double* d = c->delta[i];
        const double dot = gvec[0] * c->dw[i][0] + gvec[1] * c->dw[i][1] + gvec[2] * c->dw[i][2];
        const double alpha = upstream * c->w[i] + dot;
        const double beta = c->w[i];
        g[0] += alpha;
        if (s->order >= 1)
            for (int a = 0; a < dim; ++a) g[1 + a] += alpha * d[a] + beta * gvec[a];
        if (s->order >= 2) {
            const int(*pairs)[2] = dim == 2 ? kPairs2 : kPairs3;
            const int npairs = dim * (dim + 1) / 2;
            double* q = g + 1 + dim;
            for (int t = 0; t < npairs; ++t) {
                const int j = pairs[t][0], k = pairs[t][1];
                if (j == k)
                    q[t] += alpha * 0.5 * d[j] * d[j] + beta * gvec[j] * d[j];
                else
                    q[t] += alpha * d[j] * d[k] + beta * (gvec[j] * d[k] + gvec[k] * d[j]);
            }
        }
    }
}

/* L1 mass of the same contributions (|alpha*phi| + |beta*g.dphi| per term):
 * the scale against which reordering the fp additions can perturb a sum. Used
 * by the GPU parity tests to bound accumulation-order error. */
static void accumulate_cell_mass(const tgo_spec* s, const corners_t* c, double upstream,
                                 const double gvec[3], double* mass) {
    const int K = tgo_coeff_count(s->order, s->dim);
    const int dim = s->dim;
    for (int i = 0; i < c->count; ++i) {
        double* g = mass + c->vid[i] * K;
        const double* d = c->delta[i];
        const double dot = gvec[0] * c->dw[i][0] + gvec[1] * c->dw[i][1] + gvec[2] * c->dw[i][2];
        const double alpha = fabs(upstream * c->w[i]) + fabs(dot);
        const double beta = fabs(c->w[i]);
        g[0] += alpha;
        if (s->order >= 1)
            for (int a = 0; a < dim; ++a) g[1 + a] += fabs(alpha * d[a]) + fabs(beta * gvec[a]);
        if (s->order >= 2) {
            const int(*pairs)[2] = dim == 2 ? kPairs2 : kPairs3;
            const int npairs = dim * (dim + 1) / 2;
            double* q = g + 1 + dim;
            for (int t = 0; t < npairs; ++t) {
                const int j = pairs[t][0], k = pairs[t][1];
                if (j == k)
                    q[t] += fabs(alpha * 0.5 * d[j] * d[j]) + fabs(beta * gvec[j] * d[j]);
                else
                    q[t] += fabs(alpha * d[j] * d[k]) + fabs(beta * gvec[j] * d[k]) + fabs(beta * gvec[k] * d[j]);
            }
        }
    }
}

void tgo_backprop_mass(const tgo_spec* s, const double p[3], double upstream, const double gvec[3],
                       double* mass) {
    int cell[3];
    double local[3];
    int64_t vid[8];
    if (tgo_locate(s, p, cell, local, vid) != 0) return;
    corners_t c;
    make_corners(s, local, vid, &c);
    accumulate_cell_mass(s, &c, upstream, gvec, mass);
}

void tgo_backprop(const tgo_spec* s, const double p[3], double upstream, const double gvec[3],
                  double* grad) {
    int cell[3];
    double local[3];
    int64_t vid[8];
    if (tgo_locate(s, p, cell, local, vid) != 0) return;
    corners_t c;
    make_corners(s, local, vid, &c);
    accumulate_cell(s, &c, upstream, gvec, grad);
}

/* sigmoid / w' / dw'/dd / sign (sdf_loss.cpp:15-27). */
static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }
static double w_prime(double d, double k) { return 1.0 - fabs(2.0 * sigmoid(k * d) - 1.0); }
static double w_prime_deriv(double d, double k) {
    if (d == 0.0) return 0.0;
    const double s = sigmoid(k * d);
    const double ds = 2.0 * k * s * (1.0 - s);
    return d > 0.0 ? -ds : ds;
}
static double sign_of(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }

double tgo_adaptive_weight(double d_hat, double d, double k) {
    const double a = w_prime(d_hat, k), b = w_prime(d, k);
    return a < b ? b : a; /* std::max */
}

/* tv_loss: x/y pairs slice by slice, then z pairs in the even/odd phase
 * order the reference uses, so per-vertex accumulation order matches
 * (sdf_loss.cpp:155-257). */
double tgo_tv_loss(const tgo_spec* s, const double* coeffs, double* g, double scale) {
    const int K = tgo_coeff_count(s->order, s->dim);
    const int dim = s->dim;
    int64_t pair_count = 0;
    for (int a = 0; a < dim; ++a) {
        int64_t n = s->res[a] - 1;
        for (int b = 0; b < dim; ++b)
            if (b != a) n *= s->res[b];
        pair_count += n;
    }
    const double inv_norm = 1.0 / ((double)pair_count * K);
    const double gscale = 2.0 * scale * inv_norm;
    const int rx = s->res[0], ry = s->res[1], rz = dim == 3 ? s->res[2] : 1;
    const int64_t sy = rx, sz = (int64_t)rx * ry;

    double total = 0.0;
    for (int z = 0; z < rz; ++z) {
        double sum = 0.0;
        for (int y = 0; y < ry; ++y) {
            for (int x = 0; x < rx; ++x) {
                const int64_t v = z * sz + y * sy + x;
                const double* cv = coeffs + v * K;
                if (x + 1 < rx) {
                    const double* cu = cv + K;
                    for (int ch = 0; ch < K; ++ch) {
                        const double d = cu[ch] - cv[ch];
                        sum += d * d;
                        if (g) {
                            g[v * K + ch] -= gscale * d;
                            g[v * K + K + ch] += gscale * d;
                        }
                    }
                }
                if (y + 1 < ry) {
                    const double* cu = cv + sy * K;
                    for (int ch = 0; ch < K; ++ch) {
                        const double d = cu[ch] - cv[ch];
                        sum += d * d;
                        if (g) {
                            g[v * K + ch] -= gscale * d;
                            g[(v + sy) * K + ch] += gscale * d;
                        }
                    }
                }
            }
        }
        total += sum;
    }
    if (dim == 3 && rz > 1) {
        /* z pairs: the reference runs even z then odd z (two phases) for the
         * grad, and adds per-z sums in z order for the value. */
        for (int phase = 0; phase < 2; ++phase) {
            for (int z = phase; z < rz - 1; z += 2) {
                for (int64_t i = 0; i < sz; ++i) {
                    const int64_t v = z * sz + i;
                    const double* cv = coeffs + v * K;
                    const double* cu = cv + sz * K;
                    for (int ch = 0; ch < K; ++ch) {
                        const double d = cu[ch] - cv[ch];
                        if (g) {
                            g[v * K + ch] -= gscale * d;
                            g[(v + sz) * K + ch] += gscale * d;
                        }
                    }
                }
            }
        }
        for (int z = 0; z < rz - 1; ++z) {
            double sum = 0.0;
            for (int64_t i = 0; i < sz; ++i) {
                const double* cv = coeffs + (z * sz + i) * K;
                const double* cu = cv + sz * K;
                for (int ch = 0; ch < K; ++ch) {
                    const double d = cu[ch] - cv[ch];
                    sum += d * d;
                }
            }
            total += sum;
        }
    }
    return total * inv_norm;
}

/* point_terms_chunk, sequential (sdf_loss.cpp:37-85). */
static void point_terms(const tgo_spec* s, const double* coeffs, const double* samples, int64_t n,
                        const tgo_loss_cfg* cfg, int want_eik, double recon_scale,
                        double eik_scale, double* grad, double* mass, double* recon_out,
                        double* eik_out) {
    const double inv_n = 1.0 / (double)n;
    double recon = 0.0, eik = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double* sm = samples + 4 * i;
        double p[3] = {sm[0], sm[1], s->dim == 3 ? sm[2] : 0.0};
        const double gt = sm[3];
        double sg[3] = {0.0, 0.0, 0.0};
        const double value = tgo_eval(s, coeffs, p, want_eik ? sg : NULL);
        const double resid = value - gt;
        const double w = cfg->use_weighting ? tgo_adaptive_weight(value, gt, cfg->k) : 1.0;
        recon += w * fabs(resid);
        double upstream = 0.0, upstream_l1 = 0.0;
        double uvec[3] = {0.0, 0.0, 0.0};
        if (grad || mass) {
            upstream = recon_scale * inv_n * w * sign_of(resid);
            upstream_l1 = fabs(upstream);
            if (cfg->use_weighting && cfg->differentiate_weight) {
                const double wp_pred = w_prime(value, cfg->k);
                const double wp_gt = w_prime(gt, cfg->k);
                if (wp_pred > wp_gt) {
                    const double dw = recon_scale * inv_n * fabs(resid) * w_prime_deriv(value, cfg->k);
                    upstream += dw;
                    upstream_l1 += fabs(dw);
                }
            }
        }
        if (want_eik) {
            const double nrm = sqrt(sg[0] * sg[0] + sg[1] * sg[1] + sg[2] * sg[2]);
            const double r = nrm - 1.0;
            eik += r * r;
            if ((grad || mass) && nrm > 0.0) {
                const double sc = eik_scale * inv_n * 2.0 * r / nrm;
                uvec[0] = sc * sg[0];
                uvec[1] = sc * sg[1];
                uvec[2] = sc * sg[2];
            }
        }
        if (grad) tgo_backprop(s, p, upstream, uvec, grad);
        if (mass) {
            /* The eikonal upstream scales with (|grad f| - 1), which an fp32
             * forward evaluates to ~1e-7 absolute: bound its sensitivity by
             * using (|r| + 0.1) for the mass (0.1 * mass_rel covers that). */
            /* The fp32 forward also resolves grad f only to ~16 eps32 times
             * the L1 size of its terms (eval_grad_l1: 2^D corners, each a
             * chain of ~2K FMAs): add 0.25 (= 16 eps32 / mass_rel) of that
             * size per axis. */
            double umass[3] = {0.0, 0.0, 0.0};
            if (want_eik) {
                const double nrm = sqrt(sg[0] * sg[0] + sg[1] * sg[1] + sg[2] * sg[2]);
                if (nrm > 0.0) {
                    double l1[3];
                    eval_grad_l1(s, coeffs, p, l1);
                    const double sc = eik_scale * inv_n * 2.0 * (fabs(nrm - 1.0) + 0.1) / nrm;
                    for (int a = 0; a < 3; ++a) umass[a] = fabs(sc) * (fabs(sg[a]) + 0.25 * l1[a]);
                }
            }
            /* the upstream's L1 size: the weight term and the
             * differentiate_weight term are formed separately (fp32
             * roundings of each) and may cancel in their sum */
            tgo_backprop_mass(s, p, upstream_l1, umass, mass);
        }
    }
    *recon_out = recon;
    *eik_out = eik;
}

void tgo_total_loss(const tgo_spec* s, const double* coeffs, const double* samples, int64_t n,
                    const tgo_loss_cfg* cfg, double* grad, double terms_out[4]) {
    double fit = 0.0, eik = 0.0, tv = 0.0, recon_sum = 0.0, eik_sum = 0.0;
    const int want_eik = cfg->lambda1 > 0.0;
    point_terms(s, coeffs, samples, n, cfg, want_eik, 1.0, want_eik ? cfg->lambda1 : 0.0, grad,
                NULL, &recon_sum, &eik_sum);
    fit = recon_sum / (double)n;
    if (want_eik) eik = eik_sum / (double)n;
    if (cfg->use_tv && cfg->lambda2 > 0.0)
        tv = tgo_tv_loss(s, coeffs, grad, cfg->lambda2);
    else if (cfg->use_tv)
        tv = tgo_tv_loss(s, coeffs, NULL, 1.0);
    terms_out[0] = fit + cfg->lambda1 * eik + cfg->lambda2 * tv;
    terms_out[1] = fit;
    terms_out[2] = eik;
    terms_out[3] = tv;
}

int64_t tgo_adam_step(double* p, const double* g, double* m, double* v, int64_t n, int64_t* t,
                      double lr, double beta1, double beta2, double eps) {
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(g[i])) return i;
    *t += 1;
    const double bc1 = 1.0 - pow(beta1, (double)*t);
    const double bc2 = 1.0 - pow(beta2, (double)*t);
    for (int64_t i = 0; i < n; ++i) {
        const double gi = g[i];
        m[i] = beta1 * m[i] + (1.0 - beta1) * gi;
        v[i] = beta2 * v[i] + (1.0 - beta2) * gi * gi;
        const double mhat = m[i] / bc1;
        const double vhat = v[i] / bc2;
        p[i] -= lr * mhat / (sqrt(vhat) + eps);
    }
    return -1;
}

void tgo_multilinear_resample(const tgo_spec* old_spec, const double* data, int channels,
                              const int new_res[3], double* out) {
    tgo_spec ng = *old_spec;
    for (int a = 0; a < 3; ++a) ng.res[a] = new_res[a];
    const int dim = ng.dim;
    const int64_t nv = tgo_vertex_count(&ng);
    memset(out, 0, sizeof(double) * (size_t)(nv * channels));
    int v[3] = {0, 0, 0};
    for (int64_t idx = 0; idx < nv; ++idx) {
        double p[3] = {0.0, 0.0, 0.0};
        for (int a = 0; a < dim; ++a) p[a] = ng.origin[a] + spacing(&ng, a) * v[a];
        int cell[3];
        double local[3];
        int64_t vid[8];
        tgo_locate(old_spec, p, cell, local, vid);
        double w[8];
        const int corners = 1 << dim;
        for (int i = 0; i < corners; ++i) {
            double wi = 1.0;
            for (int a = 0; a < dim; ++a) {
                const int bit = (i >> a) & 1;
                wi *= bit ? local[a] : 1.0 - local[a];
            }
            w[i] = wi;
        }
        double* dst = out + idx * channels;
        for (int i = 0; i < corners; ++i) {
            const double* src = data + vid[i] * channels;
            for (int ch = 0; ch < channels; ++ch) dst[ch] += w[i] * src[ch];
        }
        for (int a = 0; a < dim; ++a) {
            if (++v[a] < ng.res[a]) break;
            v[a] = 0;
        }
    }
}

/* sample_grid_field (marching.cpp:53-58 via sample_field3 :30-51) for dim 3,
 * and the CLI's 2D lattice sample_grid_field2 (tools/main.cpp:33-45): lattice
 * point (x, y, z) sits at origin + extent * x / (n - 1) per axis
 * (ScalarField3::position, marching.hpp:21-24), x fastest; values fp64. */
void tgo_sample_lattice(const tgo_spec* s, const double* coeffs, const int lattice[3], double* out) {
    const int nz = s->dim == 3 ? lattice[2] : 1;
    int64_t idx = 0;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < lattice[1]; ++y)
            for (int x = 0; x < lattice[0]; ++x) {
                double p[3];
                p[0] = s->origin[0] + s->extent[0] * x / (lattice[0] - 1);
                p[1] = s->origin[1] + s->extent[1] * y / (lattice[1] - 1);
                p[2] = s->dim == 3 ? s->origin[2] + s->extent[2] * z / (lattice[2] - 1) : 0.0;
                out[idx++] = tgo_eval(s, coeffs, p, NULL);
            }
}

/* ---- radiance chain ------------------------------------------
 * sh_basis (sh.cpp:43-60), the SH color of SHColorGrid (sh.cpp:71-107),
 * forward_ray / backward_ray (volume_render.cpp:61-187) without jitter, and
 * photometric_loss (volume_render.cpp:210-276) run sequentially. */
#define TGO_MAX_SAMPLES 1024
void tgo_sh_basis(int degree, const double dir[3], double* out) {
    out[0] = 0.28209479177387814;
    if (degree < 1) return;
    const double x = dir[0], y = dir[1], z = dir[2];
    const double c1 = 0.4886025119029199;
    out[1] = -c1 * y;
    out[2] = c1 * z;
    out[3] = -c1 * x;
    if (degree < 2) return;
    out[4] = 1.0925484305920792 * x * y;
    out[5] = -1.0925484305920792 * y * z;
    out[6] = 0.31539156525252005 * (2.0 * z * z - x * x - y * y);
    out[7] = -1.0925484305920792 * x * z;
    out[8] = 0.5462742152960396 * (x * x - y * y);
}

static double sigm(double x) { return 1.0 / (1.0 + exp(-x)); }
static double softplus_(double x) { return x > 30.0 ? x : log1p(exp(x)); }

/* apply_activation (volume_render.cpp:19-28): 0 = shifted softplus, 1 = clamp relu */
static double activation(double raw, int act, double shift, double* deriv) {
    if (act == 0) {
        const double z = raw + shift;
        if (deriv) *deriv = sigm(z);
        return softplus_(z);
    }
    if (deriv) *deriv = raw > 0.0 ? 1.0 : 0.0;
    return raw > 0.0 ? raw : 0.0;
}

typedef struct {
    double t[TGO_MAX_SAMPLES], delta[TGO_MAX_SAMPLES], sigma[TGO_MAX_SAMPLES], act_deriv[TGO_MAX_SAMPLES];
    double trans_step[TGO_MAX_SAMPLES], weight[TGO_MAX_SAMPLES];
    double point[TGO_MAX_SAMPLES][3], color[TGO_MAX_SAMPLES][3];
    int64_t sh_vid[TGO_MAX_SAMPLES][8];
    double sh_w[TGO_MAX_SAMPLES][8];
} ray_ws;

/* forward_ray (volume_render.cpp:61-128); returns the residual transmittance. */
static double forward_ray(const tgo_spec* ds, const double* dc, const tgo_spec* ss, int deg, const double* sc,
                          const double o[3], const double dir[3], double near_, double far_, int n, int act,
                          double shift, const double bg[3], ray_ws* ws, double color_out[3]) {
    const double span = far_ - near_;
    const double bin = span / n;
    for (int i = 0; i < n; ++i) ws->t[i] = near_ + i * bin;
    for (int i = 0; i + 1 < n; ++i) ws->delta[i] = ws->t[i + 1] - ws->t[i];
    ws->delta[n - 1] = far_ - ws->t[n - 1];
    const int B = (deg + 1) * (deg + 1), C = 3 * B;
    double basis[9];
    tgo_sh_basis(deg, dir, basis);
    double col[3] = {0.0, 0.0, 0.0};
    double transmittance = 1.0;
    for (int i = 0; i < n; ++i) {
        double x[3];
        for (int a = 0; a < 3; ++a) x[a] = o[a] + ws->t[i] * dir[a];
        for (int a = 0; a < 3; ++a) ws->point[i][a] = x[a];
        const double raw = tgo_eval(ds, dc, x, NULL);
        ws->sigma[i] = activation(raw, act, shift, &ws->act_deriv[i]);
        int cell[3];
        double local[3];
        int64_t vid[8];
        tgo_locate(ss, x, cell, local, vid);
        const int corners = 1 << ss->dim;
        double pre[3] = {0.0, 0.0, 0.0};
        for (int c = 0; c < corners; ++c) {
            double w = 1.0;
            for (int a = 0; a < ss->dim; ++a) {
                const int bit = (c >> a) & 1;
                w *= bit ? local[a] : 1.0 - local[a];
            }
            ws->sh_w[i][c] = w;
            ws->sh_vid[i][c] = vid[c];
            const double* block = sc + vid[c] * C;
            for (int ch = 0; ch < 3; ++ch) {
                double acc = 0.0;
                const double* k = block + ch * B;
                for (int b = 0; b < B; ++b) acc += k[b] * basis[b];
                pre[ch] += w * acc;
            }
        }
        for (int ch = 0; ch < 3; ++ch) ws->color[i][ch] = sigm(pre[ch]);
        const double step = exp(-ws->sigma[i] * ws->delta[i]);
        ws->trans_step[i] = step;
        const double w = transmittance * (1.0 - step);
        ws->weight[i] = w;
        for (int ch = 0; ch < 3; ++ch) col[ch] += w * ws->color[i][ch];
        transmittance *= step;
    }
    for (int ch = 0; ch < 3; ++ch) color_out[ch] = col[ch] + transmittance * bg[ch];
    return transmittance;
}

/* backward_ray (volume_render.cpp:131-187). */
static void backward_ray(const tgo_spec* ds, const tgo_spec* ss, int deg, const double dir[3], int n, const double bg[3],
                         double residual, const double dl_dcolor[3], ray_ws* ws, double* gd, double* gsh) {
    const int B = (deg + 1) * (deg + 1), C = 3 * B;
    double basis[9];
    tgo_sh_basis(deg, dir, basis);
    double suffix[3] = {residual * bg[0], residual * bg[1], residual * bg[2]};
    double run = 1.0;
    for (int i = 0; i < n; ++i) {
        run *= ws->trans_step[i];
        ws->t[i] = run; /* T_{i+1} */
    }
    const double zero[3] = {0.0, 0.0, 0.0};
    for (int i = n - 1; i >= 0; --i) {
        const double t_next = ws->t[i];
        if (gd) {
            double dl_dsigma = 0.0;
            for (int ch = 0; ch < 3; ++ch)
                dl_dsigma += dl_dcolor[ch] * ws->delta[i] * (t_next * ws->color[i][ch] - suffix[ch]);
            const double dl_draw = dl_dsigma * ws->act_deriv[i];
            if (dl_draw != 0.0) tgo_backprop(ds, ws->point[i], dl_draw, zero, gd);
        }
        if (gsh) {
            for (int ch = 0; ch < 3; ++ch) {
                const double c = ws->color[i][ch];
                const double dl_dpre = dl_dcolor[ch] * ws->weight[i] * c * (1.0 - c);
                if (dl_dpre == 0.0) continue;
                for (int corner = 0; corner < (1 << ss->dim); ++corner) {
                    const double f = ws->sh_w[i][corner] * dl_dpre;
                    double* k = gsh + ws->sh_vid[i][corner] * C + ch * B;
                    for (int b = 0; b < B; ++b) k[b] += f * basis[b];
                }
            }
        }
        for (int ch = 0; ch < 3; ++ch) suffix[ch] += ws->weight[i] * ws->color[i][ch];
    }
}

/* photometric_loss (volume_render.cpp:210-245, threads = 1) and render_ray
 * (:194-208). rays: origins/dirs n x 3, near/far n, gt n x 3 (NULL: render
 * only). colors_out n x 3 and residual_out n may be NULL; gd/gsh gradient
 * accumulators (NULL: none). Returns the mean squared error (0 without gt). */
double tgo_photometric_loss(const tgo_spec* ds, const double* dc, const tgo_spec* ss, int deg, const double* sc,
                            int64_t nrays, const double* origins, const double* dirs, const double* near_,
                            const double* far_, const double* gt, int n_samples, int act, double shift,
                            const double bg[3], double* gd, double* gsh, double* colors_out, double* residual_out) {
    ray_ws* ws = (ray_ws*)malloc(sizeof(ray_ws));
    const double inv_n = 1.0 / (double)nrays;
    double sum = 0.0;
    for (int64_t r = 0; r < nrays; ++r) {
        double col[3];
        const double resid = forward_ray(ds, dc, ss, deg, sc, origins + 3 * r, dirs + 3 * r, near_[r], far_[r],
                                         n_samples, act, shift, bg, ws, col);
        if (colors_out)
            for (int ch = 0; ch < 3; ++ch) colors_out[3 * r + ch] = col[ch];
        if (residual_out) residual_out[r] = resid;
        if (!gt) continue;
        double err[3], e2 = 0.0;
        for (int ch = 0; ch < 3; ++ch) {
            err[ch] = col[ch] - gt[3 * r + ch];
            e2 += err[ch] * err[ch];
        }
        sum += e2;
        if (gd || gsh) {
            double g[3];
            for (int ch = 0; ch < 3; ++ch) g[ch] = (2.0 * inv_n) * err[ch];
            backward_ray(ds, ss, deg, dirs + 3 * r, n_samples, bg, resid, g, ws, gd, gsh);
        }
    }
    free(ws);
    return sum * inv_n;
}

/* Test helper: the device locate's division t = x / h via Markstein's
 * correction with a correctly rounded reciprocal (tg_device.cuh div_by_h),
 * evaluated with C99 fma so the CPU test can compare it with IEEE division. */
double tgo_markstein_div(double x, double h, double inv_h) {
    const double q = x * inv_h;
    const double r = fma(-q, h, x);
    return fma(r, inv_h, q);
}

/* L1 mass of every gradient contribution of tgo_total_loss (point terms and
 * TV pair terms), per coefficient. Test helper for order-independent
 * tolerances. */
void tgo_total_loss_mass(const tgo_spec* s, const double* coeffs, const double* samples, int64_t n,
                         const tgo_loss_cfg* cfg, double* mass) {
    double r, e;
    const int want_eik = cfg->lambda1 > 0.0;
    point_terms(s, coeffs, samples, n, cfg, want_eik, 1.0, want_eik ? cfg->lambda1 : 0.0, NULL, mass,
                &r, &e);
    if (!(cfg->use_tv && cfg->lambda2 > 0.0)) return;
    const int K = tgo_coeff_count(s->order, s->dim);
    int64_t pair_count = 0;
    for (int a = 0; a < s->dim; ++a) {
        int64_t np = s->res[a] - 1;
        for (int b = 0; b < s->dim; ++b)
            if (b != a) np *= s->res[b];
        pair_count += np;
    }
    const double gscale = 2.0 * cfg->lambda2 / ((double)pair_count * K);
    const int rx = s->res[0], ry = s->res[1], rz = s->dim == 3 ? s->res[2] : 1;
    const int64_t st[3] = {1, rx, (int64_t)rx * ry};
    for (int z = 0; z < rz; ++z)
        for (int y = 0; y < ry; ++y)
            for (int x = 0; x < rx; ++x) {
                const int co[3] = {x, y, z};
                const int64_t v = z * st[2] + y * st[1] + x;
                for (int a = 0; a < s->dim; ++a) {
                    if (co[a] + 1 >= s->res[a]) continue;
                    const int64_t u = v + st[a];
                    for (int ch = 0; ch < K; ++ch) {
                        const double d = fabs(gscale * (coeffs[u * K + ch] - coeffs[v * K + ch]));
                        mass[v * K + ch] += d;
                        mass[u * K + ch] += d;
                    }
                }
            }
}
