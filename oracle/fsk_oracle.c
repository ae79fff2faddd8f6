/*
 * CPU restatement of the reference FlashSinkhorn hot path (plain C11).
 *
 * TEST INFRASTRUCTURE ONLY - this file is the parity oracle. It may be loaded
 * by tests/, by __graft_entry__.smoke() and by bench.py's cpu_baseline leg, and
 * only as the checker. The product (libfsk_b200.so) never links or calls it.
 *
 * Every function restates the reference algorithm with the same arithmetic
 * order so that, compiled with -ffp-contract=off, results are bit-identical
 * to the patched reference (oracle/_ref/libfsk_ref_check.so); tests pin this.
 *
 *   fo_fast_exp_d / _f      <- proj/include/fsk/mathutil.hpp:19-56
 *   fo_psum_d / _f          <- mathutil.hpp:60-71 (cascade: <=8 sequential, split n/2)
 *   lse_reduce_*            <- proj/src/stream.cpp:52-136 (transpose_keys, score_tile,
 *                              rescale_factor, lse_reduce) with the ragged-tile stride
 *                              fix of SURVEY.md finding 3
 *   fo_apply_core           <- stream.cpp:140-207 (apply_core, incl. Hadamard weights)
 *   ctx builders            <- stream.cpp:209-251 (make_ctx_f/g), :421-434 (make_ctx_f32)
 *   fo_update_* / fo_*      <- stream.cpp:270-451 (public stream ops)
 *   fo_solve                <- proj/src/solver.cpp:14-129 (solve_f64/solve_f32)
 *   fo_dual_cost            <- solver.cpp:131-143
 *   fo_eps_schedule         <- proj/src/schedule.cpp:8-44
 *
 * Status codes: 0 ok, 1 validation, 2 numerical (message via fo_last_error()).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];
const char* fo_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* ---- mathutil.hpp:19-36 --------------------------------------------------- */
double fo_fast_exp_d(double x) {
    /* std::min(std::max(x, -708.0), 709.0) with std:: tie/NaN semantics */
    x = (x < -708.0) ? -708.0 : x;
    x = (709.0 < x) ? 709.0 : x;
    double k = floor(x * 1.4426950408889634074 + 0.5);
    double r = x - k * 6.93145751953125e-1;
    r -= k * 1.42860682030941723212e-6;
    double rr = r * r;
    double p = r * (9.99999999999999999910e-1 +
                    rr * (3.02994407707441961300e-2 + rr * 1.26177193074810590878e-4));
    double q = 2.00000000000000000005e0 +
               rr * (2.27265548208155028766e-1 +
                     rr * (2.52448340349684104192e-3 + rr * 3.00198505138664455042e-6));
    double e = 1.0 + 2.0 * p / (q - p);
    uint64_t bits;
    memcpy(&bits, &e, 8);
    bits += (uint64_t)((int64_t)k) << 52;
    memcpy(&e, &bits, 8);
    return e;
}

/* ---- mathutil.hpp:39-56 --------------------------------------------------- */
float fo_fast_exp_f(float x) {
    x = (x < -87.0f) ? -87.0f : x;
    x = (88.0f < x) ? 88.0f : x;
    float k = floorf(x * 1.44269504088896341f + 0.5f);
    float r = x - k * 0.693359375f;
    r -= k * -2.12194440e-4f;
    float p = 1.9875691500e-4f;
    p = p * r + 1.3981999507e-3f;
    p = p * r + 8.3334519073e-3f;
    p = p * r + 4.1665795894e-2f;
    p = p * r + 1.6666665459e-1f;
    p = p * r + 5.0000001201e-1f;
    p = p * r * r + r + 1.0f;
    uint32_t bits;
    memcpy(&bits, &p, 4);
    bits += (uint32_t)((int32_t)k) << 23;
    memcpy(&p, &bits, 4);
    return p;
}

/* ---- mathutil.hpp:60-71 (association order of the cascade) ----------------- */
double fo_psum_d(const double* a, size_t n) {
    if (n == 0) return 0.0;
    if (n <= 8) {
        double s = a[0];
        for (size_t i = 1; i < n; ++i) s += a[i];
        return s;
    }
    size_t h = n / 2;
    return fo_psum_d(a, h) + fo_psum_d(a + h, n - h);
}

float fo_psum_f(const float* a, size_t n) {
    if (n == 0) return 0.0f;
    if (n <= 8) {
        float s = a[0];
        for (size_t i = 1; i < n; ++i) s += a[i];
        return s;
    }
    size_t h = n / 2;
    return fo_psum_f(a, h) + fo_psum_f(a + h, n - h);
}

static int g_break_lse = 0; /* stream.cpp:14, :81-87 negative control */
void fo_debug_break_lse(int on) { g_break_lse = on; }

static size_t min_sz(size_t a, size_t b) { return a < b ? a : b; }

/* Score-matrix description, stream.cpp:21-35. */
typedef struct {
    const double* qpts;
    size_t R;
    const double* kpts;
    size_t C, d;
    const int32_t* qlab;
    const int32_t* klab;
    const double* wtab;
    size_t wdim;
    double lam2_eps, scaled2_eps;
    double* bias2; /* C */
} ctx_d;

typedef struct {
    const float* qpts;
    size_t R;
    const float* kpts;
    size_t C, d;
    float scaled2_eps;
    float* bias2;
} ctx_f;

/* transpose_keys + score_tile (stream.cpp:52-79) for rows I0..I0+bn, cols J0..J0+bm */
static void score_tile_d(const ctx_d* c, size_t I0, size_t bn, size_t J0, size_t bm, double* kt,
                         double* tile) {
    const size_t d = c->d;
    for (size_t j = 0; j < bm; ++j) {
        const double* kr = c->kpts + (J0 + j) * d;
        for (size_t t = 0; t < d; ++t) kt[t * bm + j] = kr[t] * c->scaled2_eps;
    }
    for (size_t i = 0; i < bn; ++i) {
        const double* qi = c->qpts + (I0 + i) * d;
        double* srow = tile + i * bm;
        for (size_t j = 0; j < bm; ++j) srow[j] = c->bias2[J0 + j];
        for (size_t t = 0; t < d; ++t) {
            const double qv = qi[t];
            const double* krow = kt + t * bm;
            for (size_t j = 0; j < bm; ++j) srow[j] += qv * krow[j];
        }
        if (c->qlab) {
            const double* wrow = c->wtab + (size_t)c->qlab[I0 + i] * c->wdim;
            for (size_t j = 0; j < bm; ++j) srow[j] -= c->lam2_eps * wrow[c->klab[J0 + j]];
        }
    }
}

static void score_tile_f(const ctx_f* c, size_t I0, size_t bn, size_t J0, size_t bm, float* kt,
                         float* tile) {
    const size_t d = c->d;
    for (size_t j = 0; j < bm; ++j) {
        const float* kr = c->kpts + (J0 + j) * d;
        for (size_t t = 0; t < d; ++t) kt[t * bm + j] = kr[t] * c->scaled2_eps;
    }
    for (size_t i = 0; i < bn; ++i) {
        const float* qi = c->qpts + (I0 + i) * d;
        float* srow = tile + i * bm;
        for (size_t j = 0; j < bm; ++j) srow[j] = c->bias2[J0 + j];
        for (size_t t = 0; t < d; ++t) {
            const float qv = qi[t];
            const float* krow = kt + t * bm;
            for (size_t j = 0; j < bm; ++j) srow[j] += qv * krow[j];
        }
    }
}

static double rescale_d(double m_old, double m_new) {
    return g_break_lse ? fo_fast_exp_d(m_new - m_old) : fo_fast_exp_d(m_old - m_new);
}
static float rescale_f(float m_old, float m_new) {
    return g_break_lse ? fo_fast_exp_f(m_new - m_old) : fo_fast_exp_f(m_old - m_new);
}

/* lse_reduce (stream.cpp:93-136), double */
static int lse_reduce_d(const ctx_d* c, size_t br, size_t bc, double eps, double* out) {
    const size_t R = c->R, C = c->C, d = c->d;
    br = min_sz(br, R);
    bc = min_sz(bc, C);
    const size_t nblocks = (R + br - 1) / br;
    int status = 0;
#pragma omp parallel for schedule(dynamic, 1)
    for (size_t blk = 0; blk < nblocks; ++blk) {
        const size_t I0 = blk * br;
        const size_t bn = min_sz(br, R - I0);
        double* tile = malloc(sizeof(double) * bn * bc);
        double* wbuf = malloc(sizeof(double) * bc);
        double* kt = malloc(sizeof(double) * (d ? d : 1) * bc);
        double* mI = malloc(sizeof(double) * bn);
        double* sI = malloc(sizeof(double) * bn);
        for (size_t i = 0; i < bn; ++i) {
            mI[i] = -INFINITY;
            sI[i] = 0.0;
        }
        for (size_t J0 = 0; J0 < C; J0 += bc) {
            const size_t bm = min_sz(bc, C - J0);
            score_tile_d(c, I0, bn, J0, bm, kt, tile);
            for (size_t i = 0; i < bn; ++i) {
                const double* srow = tile + i * bm;
                double tmax = srow[0];
                for (size_t j = 1; j < bm; ++j) tmax = (tmax < srow[j]) ? srow[j] : tmax;
                const double mnew = (mI[i] < tmax) ? tmax : mI[i];
                for (size_t j = 0; j < bm; ++j) wbuf[j] = fo_fast_exp_d(srow[j] - mnew);
                const double tsum = fo_psum_d(wbuf, bm);
                sI[i] = rescale_d(mI[i], mnew) * sI[i] + tsum;
                mI[i] = mnew;
            }
        }
        for (size_t i = 0; i < bn; ++i) {
            const double v = -eps * (mI[i] + log(sI[i]));
            if (!isfinite(v)) status = 2;
            out[I0 + i] = v;
        }
        free(tile);
        free(wbuf);
        free(kt);
        free(mI);
        free(sI);
    }
    if (status) return fail(2, "non-finite potential produced by streaming LSE update");
    return 0;
}

static int lse_reduce_f(const ctx_f* c, size_t br, size_t bc, float eps, float* out) {
    const size_t R = c->R, C = c->C, d = c->d;
    br = min_sz(br, R);
    bc = min_sz(bc, C);
    const size_t nblocks = (R + br - 1) / br;
    int status = 0;
#pragma omp parallel for schedule(dynamic, 1)
    for (size_t blk = 0; blk < nblocks; ++blk) {
        const size_t I0 = blk * br;
        const size_t bn = min_sz(br, R - I0);
        float* tile = malloc(sizeof(float) * bn * bc);
        float* wbuf = malloc(sizeof(float) * bc);
        float* kt = malloc(sizeof(float) * (d ? d : 1) * bc);
        float* mI = malloc(sizeof(float) * bn);
        float* sI = malloc(sizeof(float) * bn);
        for (size_t i = 0; i < bn; ++i) {
            mI[i] = -INFINITY;
            sI[i] = 0.0f;
        }
        for (size_t J0 = 0; J0 < C; J0 += bc) {
            const size_t bm = min_sz(bc, C - J0);
            score_tile_f(c, I0, bn, J0, bm, kt, tile);
            for (size_t i = 0; i < bn; ++i) {
                const float* srow = tile + i * bm;
                float tmax = srow[0];
                for (size_t j = 1; j < bm; ++j) tmax = (tmax < srow[j]) ? srow[j] : tmax;
                const float mnew = (mI[i] < tmax) ? tmax : mI[i];
                for (size_t j = 0; j < bm; ++j) wbuf[j] = fo_fast_exp_f(srow[j] - mnew);
                const float tsum = fo_psum_f(wbuf, bm);
                sI[i] = rescale_f(mI[i], mnew) * sI[i] + tsum;
                mI[i] = mnew;
            }
        }
        for (size_t i = 0; i < bn; ++i) {
            const float v = -eps * (mI[i] + logf(sI[i]));
            if (!isfinite(v)) status = 2;
            out[I0 + i] = v;
        }
        free(tile);
        free(wbuf);
        free(kt);
        free(mI);
        free(sI);
    }
    if (status) return fail(2, "non-finite potential produced by streaming LSE update");
    return 0;
}

/* apply_core (stream.cpp:140-207). A/B nullable (plain transport). */
static int apply_core(const ctx_d* c, const double* row_w, const double* row_fhat,
                      const double* V, size_t p, const double* A, const double* B, size_t r,
                      size_t br, size_t bc, double eps, double* out) {
    const size_t R = c->R, C = c->C, d = c->d;
    br = min_sz(br, R);
    bc = min_sz(bc, C);
    const size_t nblocks = (R + br - 1) / br;
    const double inv_eps = 1.0 / eps;
    int status = 0;
#pragma omp parallel for schedule(dynamic, 1)
    for (size_t blk = 0; blk < nblocks; ++blk) {
        const size_t I0 = blk * br;
        const size_t bn = min_sz(br, R - I0);
        double* tile = malloc(sizeof(double) * bn * bc);
        double* wbuf = malloc(sizeof(double) * bc);
        double* prod = malloc(sizeof(double) * bc);
        double* kt = malloc(sizeof(double) * (d ? d : 1) * bc);
        double* mI = malloc(sizeof(double) * bn);
        double* oI = calloc(bn * (p ? p : 1), sizeof(double));
        for (size_t i = 0; i < bn; ++i) mI[i] = -INFINITY;
        for (size_t J0 = 0; J0 < C; J0 += bc) {
            const size_t bm = min_sz(bc, C - J0);
            score_tile_d(c, I0, bn, J0, bm, kt, tile);
            for (size_t i = 0; i < bn; ++i) {
                const double* srow = tile + i * bm;
                double tmax = srow[0];
                for (size_t j = 1; j < bm; ++j) tmax = (tmax < srow[j]) ? srow[j] : tmax;
                const double mnew = (mI[i] < tmax) ? tmax : mI[i];
                for (size_t j = 0; j < bm; ++j) wbuf[j] = fo_fast_exp_d(srow[j] - mnew);
                if (A) {
                    const double* ai = A + (I0 + i) * r;
                    for (size_t j = 0; j < bm; ++j) {
                        const double* bj = B + (J0 + j) * r;
                        double wd = 0.0;
                        for (size_t q = 0; q < r; ++q) wd += ai[q] * bj[q];
                        wbuf[j] *= wd;
                    }
                }
                const double resc = rescale_d(mI[i], mnew);
                double* orow = oI + i * p;
                for (size_t col = 0; col < p; ++col) {
                    for (size_t j = 0; j < bm; ++j) prod[j] = wbuf[j] * V[(J0 + j) * p + col];
                    const double part = fo_psum_d(prod, bm);
                    orow[col] = resc * orow[col] + part;
                }
                mI[i] = mnew;
            }
        }
        for (size_t i = 0; i < bn; ++i) {
            const double arg = row_fhat[I0 + i] * inv_eps + mI[i];
            if (arg > 709.0) {
                status = 3;
                continue;
            }
            const double scale = row_w[I0 + i] * fo_fast_exp_d(arg);
            for (size_t col = 0; col < p; ++col) {
                const double v = scale * oI[i * p + col];
                out[(I0 + i) * p + col] = v;
                if (!isfinite(v) && status == 0) status = 2;
            }
        }
        free(tile);
        free(wbuf);
        free(prod);
        free(kt);
        free(mI);
        free(oI);
    }
    if (status == 3)
        return fail(2, "overflow in transport application, potentials are not stabilized");
    if (status == 2) return fail(2, "non-finite entry in transport application output");
    return 0;
}

/* ---- public surface ------------------------------------------------------- */

typedef struct {
    const double* pts;
    const double* w;
    const int32_t* labels; /* nullable */
    int64_t n, d;
} fo_measure;

typedef struct {
    int32_t kind; /* 0 squared Euclidean, 1 label augmented */
    double lambda1, lambda2;
    const double* label_cost;
    int64_t num_labels;
} fo_cost;

static double feature_scale(const fo_cost* cost) {
    return (cost && cost->kind == 1) ? cost->lambda1 : 1.0;
}

/* make_ctx_f (stream.cpp:209-229) */
static void make_ctx_f(ctx_d* c, const fo_measure* src, const fo_measure* tgt,
                       const double* g_hat, const fo_cost* cost, double eps) {
    memset(c, 0, sizeof *c);
    c->qpts = src->pts;
    c->R = (size_t)src->n;
    c->kpts = tgt->pts;
    c->C = (size_t)tgt->n;
    c->d = (size_t)src->d;
    if (cost && cost->kind == 1) {
        c->qlab = src->labels;
        c->klab = tgt->labels;
        c->wtab = cost->label_cost;
        c->wdim = (size_t)cost->num_labels;
        c->lam2_eps = cost->lambda2 / eps;
    }
    c->scaled2_eps = 2.0 * feature_scale(cost) / eps;
    c->bias2 = malloc(sizeof(double) * (c->C ? c->C : 1));
    for (size_t j = 0; j < c->C; ++j) c->bias2[j] = (g_hat[j] + eps * log(tgt->w[j])) / eps;
}

/* make_ctx_g (stream.cpp:231-251) */
static void make_ctx_g(ctx_d* c, const fo_measure* src, const fo_measure* tgt,
                       const double* f_hat, const fo_cost* cost, double eps) {
    memset(c, 0, sizeof *c);
    c->qpts = tgt->pts;
    c->R = (size_t)tgt->n;
    c->kpts = src->pts;
    c->C = (size_t)src->n;
    c->d = (size_t)src->d;
    if (cost && cost->kind == 1) {
        c->qlab = tgt->labels;
        c->klab = src->labels;
        c->wtab = cost->label_cost;
        c->wdim = (size_t)cost->num_labels;
        c->lam2_eps = cost->lambda2 / eps;
    }
    c->scaled2_eps = 2.0 * feature_scale(cost) / eps;
    c->bias2 = malloc(sizeof(double) * (c->C ? c->C : 1));
    for (size_t i = 0; i < c->C; ++i) c->bias2[i] = (f_hat[i] + eps * log(src->w[i])) / eps;
}

int fo_update_f_hat(const fo_measure* src, const fo_measure* tgt, const double* g_hat,
                    const fo_cost* cost, double eps, int64_t bn, int64_t bm, double* out) {
    if (!(eps > 0.0)) return fail(1, "eps must be positive");
    ctx_d c;
    make_ctx_f(&c, src, tgt, g_hat, cost, eps);
    int st = lse_reduce_d(&c, (size_t)bn, (size_t)bm, eps, out);
    free(c.bias2);
    return st;
}

int fo_update_g_hat(const fo_measure* src, const fo_measure* tgt, const double* f_hat,
                    const fo_cost* cost, double eps, int64_t bn, int64_t bm, double* out) {
    if (!(eps > 0.0)) return fail(1, "eps must be positive");
    ctx_d c;
    make_ctx_g(&c, src, tgt, f_hat, cost, eps);
    int st = lse_reduce_d(&c, (size_t)bm, (size_t)bn, eps, out);
    free(c.bias2);
    return st;
}

/* symmetric_update (stream.cpp:296-322) */
int fo_symmetric_update(const fo_measure* src, const fo_measure* tgt, const double* f_hat,
                        const double* g_hat, double eps, const fo_cost* cost, int64_t bn,
                        int64_t bm, double* out_f, double* out_g) {
    const size_t n = (size_t)src->n, m = (size_t)tgt->n;
    double* ff = malloc(sizeof(double) * n);
    double* gg = malloc(sizeof(double) * m);
    int st = fo_update_f_hat(src, tgt, g_hat, cost, eps, bn, bm, ff);
    if (!st) st = fo_update_g_hat(src, tgt, f_hat, cost, eps, bn, bm, gg);
    if (!st) {
        for (size_t i = 0; i < n; ++i) out_f[i] = 0.5 * f_hat[i] + 0.5 * ff[i];
        for (size_t j = 0; j < m; ++j) out_g[j] = 0.5 * g_hat[j] + 0.5 * gg[j];
    }
    free(ff);
    free(gg);
    return st;
}

/* apply_plan (stream.cpp:324-339) */
int fo_apply_plan(const fo_measure* src, const fo_measure* tgt, const double* f_hat,
                  const double* g_hat, double eps, const fo_cost* cost, const double* V, int64_t p,
                  int64_t bn, int64_t bm, double* out) {
    ctx_d c;
    make_ctx_f(&c, src, tgt, g_hat, cost, eps);
    int st = apply_core(&c, src->w, f_hat, V, (size_t)p, NULL, NULL, 0, (size_t)bn, (size_t)bm,
                        eps, out);
    free(c.bias2);
    return st;
}

/* apply_plan_adjoint (stream.cpp:341-357) */
int fo_apply_plan_adjoint(const fo_measure* src, const fo_measure* tgt, const double* f_hat,
                          const double* g_hat, double eps, const fo_cost* cost, const double* U,
                          int64_t p, int64_t bn, int64_t bm, double* out) {
    ctx_d c;
    make_ctx_g(&c, src, tgt, f_hat, cost, eps);
    int st = apply_core(&c, tgt->w, g_hat, U, (size_t)p, NULL, NULL, 0, (size_t)bm, (size_t)bn,
                        eps, out);
    free(c.bias2);
    return st;
}

/* apply_hadamard_plan (stream.cpp:359-375) */
int fo_apply_hadamard_plan(const fo_measure* src, const fo_measure* tgt, const double* f_hat,
                           const double* g_hat, double eps, const fo_cost* cost, const double* A,
                           const double* B, int64_t r, const double* V, int64_t p, int64_t bn,
                           int64_t bm, double* out) {
    ctx_d c;
    make_ctx_f(&c, src, tgt, g_hat, cost, eps);
    int st = apply_core(&c, src->w, f_hat, V, (size_t)p, A, B, (size_t)r, (size_t)bn, (size_t)bm,
                        eps, out);
    free(c.bias2);
    return st;
}

/* induced_marginals (stream.cpp:377-404) */
int fo_induced_marginals(const fo_measure* src, const fo_measure* tgt, const double* f_hat,
                         const double* g_hat, double eps, const fo_cost* cost, int64_t bn,
                         int64_t bm, double* out_r, double* out_c) {
    const size_t n = (size_t)src->n, m = (size_t)tgt->n;
    double* fp = malloc(sizeof(double) * n);
    double* gp = malloc(sizeof(double) * m);
    int st = fo_update_f_hat(src, tgt, g_hat, cost, eps, bn, bm, fp);
    if (!st) st = fo_update_g_hat(src, tgt, f_hat, cost, eps, bn, bm, gp);
    if (!st) {
        const double inv_eps = 1.0 / eps;
        for (size_t i = 0; i < n && !st; ++i) {
            out_r[i] = src->w[i] * fo_fast_exp_d((f_hat[i] - fp[i]) * inv_eps);
            if (!isfinite(out_r[i])) st = fail(2, "non-finite induced row marginal");
        }
        for (size_t j = 0; j < m && !st; ++j) {
            out_c[j] = tgt->w[j] * fo_fast_exp_d((g_hat[j] - gp[j]) * inv_eps);
            if (!isfinite(out_c[j])) st = fail(2, "non-finite induced column marginal");
        }
    }
    free(fp);
    free(gp);
    return st;
}

/* fp32 half-steps: to_float_cloud + make_ctx_f32 + lse_reduce<float>
   (stream.cpp:408-451). Points/weights are already float here. */
int fo_update_f_hat_f32(const float* src_pts, int64_t n, const float* tgt_pts, const float* tgt_w,
                        int64_t m, int64_t d, const float* g_hat, float eps, int64_t bn,
                        int64_t bm, float* out) {
    ctx_f c;
    c.qpts = src_pts;
    c.R = (size_t)n;
    c.kpts = tgt_pts;
    c.C = (size_t)m;
    c.d = (size_t)d;
    c.scaled2_eps = 2.0f / eps;
    c.bias2 = malloc(sizeof(float) * (size_t)(m ? m : 1));
    for (int64_t j = 0; j < m; ++j) c.bias2[j] = (g_hat[j] + eps * logf(tgt_w[j])) / eps;
    int st = lse_reduce_f(&c, (size_t)bn, (size_t)bm, eps, out);
    free(c.bias2);
    return st;
}

int fo_update_g_hat_f32(const float* src_pts, const float* src_w, int64_t n,
                        const float* tgt_pts, int64_t m, int64_t d, const float* f_hat, float eps,
                        int64_t bn, int64_t bm, float* out) {
    ctx_f c;
    c.qpts = tgt_pts;
    c.R = (size_t)m;
    c.kpts = src_pts;
    c.C = (size_t)n;
    c.d = (size_t)d;
    c.scaled2_eps = 2.0f / eps;
    c.bias2 = malloc(sizeof(float) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; ++i) c.bias2[i] = (f_hat[i] + eps * logf(src_w[i])) / eps;
    int st = lse_reduce_f(&c, (size_t)bm, (size_t)bn, eps, out);
    free(c.bias2);
    return st;
}

/* ---- schedule.cpp -------------------------------------------------------- */

/* joint_sq_diameter (schedule.cpp:8-25) */
double fo_joint_sq_diameter(const double* X, int64_t n, const double* Y, int64_t m, int64_t d) {
    double diam2 = 0.0;
    for (int64_t t = 0; t < d; ++t) {
        double lo = INFINITY, hi = -INFINITY;
        for (int64_t i = 0; i < n; ++i) {
            lo = fmin(lo, X[i * d + t]);
            hi = fmax(hi, X[i * d + t]);
        }
        for (int64_t j = 0; j < m; ++j) {
            lo = fmin(lo, Y[j * d + t]);
            hi = fmax(hi, Y[j * d + t]);
        }
        diam2 += (hi - lo) * (hi - lo);
    }
    return diam2;
}

typedef struct {
    double eps;
    int32_t schedule; /* 0 alternating, 1 symmetric */
    int32_t max_iters;
    double marginal_tol;
    double eps_scaling_factor;
    int32_t extra_iters_at_final_eps;
    int32_t precision; /* 0 single, 1 double */
} fo_config;

/* eps_schedule (schedule.cpp:27-44); returns the length, fills out (cap max_iters) */
int64_t fo_eps_schedule(const fo_config* cfg, double sq_diam, double* out) {
    const int64_t cap = cfg->max_iters;
    int64_t k = 0;
    if (cfg->eps_scaling_factor >= 1.0) {
        for (; k < cap; ++k) out[k] = cfg->eps;
        return k;
    }
    double e = sq_diam;
    while (k < cap) {
        out[k++] = fmax(e, cfg->eps);
        if (e <= cfg->eps) break;
        e *= cfg->eps_scaling_factor;
    }
    for (int32_t x = 0; x < cfg->extra_iters_at_final_eps && k < cap; ++x) out[k++] = cfg->eps;
    return k;
}

/* squared_norms (core.cpp:83-96) */
static void sq_norms(const double* P, int64_t n, int64_t d, double s, double* out) {
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t t = 0; t < d; ++t) acc += P[i * d + t] * P[i * d + t];
        out[i] = (s != 1.0) ? acc * s : acc;
    }
}

/* dual_cost (solver.cpp:131-143) */
int fo_dual_cost(const fo_measure* src, const fo_measure* tgt, const double* f_hat,
                 const double* g_hat, double eps, const fo_cost* cost, int64_t bn, int64_t bm,
                 double* out) {
    const size_t n = (size_t)src->n, m = (size_t)tgt->n;
    double* alpha = malloc(sizeof(double) * n);
    double* beta = malloc(sizeof(double) * m);
    double* r = malloc(sizeof(double) * n);
    double* c = malloc(sizeof(double) * m);
    sq_norms(src->pts, src->n, src->d, feature_scale(cost), alpha);
    sq_norms(tgt->pts, tgt->n, tgt->d, feature_scale(cost), beta);
    int st = fo_induced_marginals(src, tgt, f_hat, g_hat, eps, cost, bn, bm, r, c);
    if (!st) {
        const double mass = fo_psum_d(r, n);
        double value = 0.0;
        for (size_t i = 0; i < n; ++i) value += (f_hat[i] + alpha[i]) * src->w[i];
        for (size_t j = 0; j < m; ++j) value += (g_hat[j] + beta[j]) * tgt->w[j];
        *out = value - eps * (mass - 1.0);
    }
    free(alpha);
    free(beta);
    free(r);
    free(c);
    return st;
}

static double marginal_violation(const double* r, const double* a, size_t n, const double* c,
                                 const double* b, size_t m) {
    double v = 0.0;
    for (size_t i = 0; i < n; ++i) v += fabs(r[i] - a[i]);
    for (size_t j = 0; j < m; ++j) v += fabs(c[j] - b[j]);
    return v;
}

/* sinkhorn_solve (solver.cpp:21-129). out_scalars = [iterations, violation, dual, eps] */
int fo_sinkhorn_solve(const fo_measure* src, const fo_measure* tgt, const fo_cost* cost,
                      const fo_config* cfg, int64_t bn, int64_t bm, double* out_f, double* out_g,
                      double* out_scalars, double* eps_history) {
    const size_t n = (size_t)src->n, m = (size_t)tgt->n, d = (size_t)src->d;
    double* alpha = malloc(sizeof(double) * n);
    double* beta = malloc(sizeof(double) * m);
    double* sched = malloc(sizeof(double) * (size_t)(cfg->max_iters > 0 ? cfg->max_iters : 1));
    double* r = malloc(sizeof(double) * n);
    double* c = malloc(sizeof(double) * m);
    sq_norms(src->pts, src->n, src->d, feature_scale(cost), alpha);
    sq_norms(tgt->pts, tgt->n, tgt->d, feature_scale(cost), beta);
    const int64_t len = fo_eps_schedule(
        cfg, fo_joint_sq_diameter(src->pts, src->n, tgt->pts, tgt->n, src->d), sched);
    int st = 0;
    int iters = 0;
    double viol = 0.0, dual = 0.0, final_eps = 0.0;
    if (cfg->precision == 1) {
        double* f = out_f;
        double* g = out_g;
        double* tf = malloc(sizeof(double) * n);
        double* tg = malloc(sizeof(double) * m);
        for (size_t i = 0; i < n; ++i) f[i] = -alpha[i];
        for (size_t j = 0; j < m; ++j) g[j] = -beta[j];
        int stopped = 0;
        for (int64_t k = 0; k < len && !st; ++k) {
            const double eps = sched[k];
            final_eps = eps;
            if (cfg->schedule == 0) {
                st = fo_update_f_hat(src, tgt, g, cost, eps, bn, bm, f);
                if (!st) st = fo_update_g_hat(src, tgt, f, cost, eps, bn, bm, g);
            } else {
                st = fo_symmetric_update(src, tgt, f, g, eps, cost, bn, bm, tf, tg);
                if (!st) {
                    memcpy(f, tf, sizeof(double) * n);
                    memcpy(g, tg, sizeof(double) * m);
                }
            }
            if (st) {
                char buf[320];
                snprintf(buf, sizeof buf, "%s at iteration %d", g_err, iters + 1);
                fail(st, buf);
                break;
            }
            ++iters;
            if (eps_history) eps_history[k] = eps;
            if (cfg->marginal_tol > 0.0 && eps == cfg->eps) {
                st = fo_induced_marginals(src, tgt, f, g, eps, cost, bn, bm, r, c);
                if (st) break;
                viol = marginal_violation(r, src->w, n, c, tgt->w, m);
                if (viol <= cfg->marginal_tol) {
                    st = fo_dual_cost(src, tgt, f, g, eps, cost, bn, bm, &dual);
                    stopped = 1;
                    break;
                }
            }
        }
        if (!st && !stopped) {
            st = fo_induced_marginals(src, tgt, f, g, final_eps, cost, bn, bm, r, c);
            if (!st) viol = marginal_violation(r, src->w, n, c, tgt->w, m);
            if (!st) st = fo_dual_cost(src, tgt, f, g, final_eps, cost, bn, bm, &dual);
        }
        free(tf);
        free(tg);
    } else {
        /* solve_f32 (solver.cpp:69-117) */
        if (cost && cost->kind != 0) {
            st = fail(1, "single-precision solve supports the squared-Euclidean cost only");
        } else {
            float* sp = malloc(sizeof(float) * n * d);
            float* sw = malloc(sizeof(float) * n);
            float* tp = malloc(sizeof(float) * m * d);
            float* tw = malloc(sizeof(float) * m);
            float* f = malloc(sizeof(float) * n);
            float* g = malloc(sizeof(float) * m);
            float* ff = malloc(sizeof(float) * n);
            float* gg = malloc(sizeof(float) * m);
            for (size_t i = 0; i < n * d; ++i) sp[i] = (float)src->pts[i];
            for (size_t i = 0; i < n; ++i) sw[i] = (float)src->w[i];
            for (size_t i = 0; i < m * d; ++i) tp[i] = (float)tgt->pts[i];
            for (size_t i = 0; i < m; ++i) tw[i] = (float)tgt->w[i];
            for (size_t i = 0; i < n; ++i) f[i] = -(float)alpha[i];
            for (size_t j = 0; j < m; ++j) g[j] = -(float)beta[j];
            for (int64_t k = 0; k < len && !st; ++k) {
                const float eps = (float)sched[k];
                if (cfg->schedule == 0) {
                    st = fo_update_f_hat_f32(sp, (int64_t)n, tp, tw, (int64_t)m, (int64_t)d, g,
                                             eps, bn, bm, f);
                    if (!st)
                        st = fo_update_g_hat_f32(sp, sw, (int64_t)n, tp, (int64_t)m, (int64_t)d,
                                                 f, eps, bn, bm, g);
                } else {
                    st = fo_update_f_hat_f32(sp, (int64_t)n, tp, tw, (int64_t)m, (int64_t)d, g,
                                             eps, bn, bm, ff);
                    if (!st)
                        st = fo_update_g_hat_f32(sp, sw, (int64_t)n, tp, (int64_t)m, (int64_t)d,
                                                 f, eps, bn, bm, gg);
                    if (!st) {
                        for (size_t i = 0; i < n; ++i) f[i] = 0.5f * f[i] + 0.5f * ff[i];
                        for (size_t j = 0; j < m; ++j) g[j] = 0.5f * g[j] + 0.5f * gg[j];
                    }
                }
                if (st) {
                    char buf[320];
                    snprintf(buf, sizeof buf, "%s at iteration %d", g_err, iters + 1);
                    fail(st, buf);
                    break;
                }
                ++iters;
                if (eps_history) eps_history[k] = sched[k];
            }
            if (!st) {
                final_eps = cfg->eps;
                for (size_t i = 0; i < n; ++i) out_f[i] = f[i];
                for (size_t j = 0; j < m; ++j) out_g[j] = g[j];
                st = fo_induced_marginals(src, tgt, out_f, out_g, cfg->eps, cost, bn, bm, r, c);
                if (!st) viol = marginal_violation(r, src->w, n, c, tgt->w, m);
                if (!st)
                    st = fo_dual_cost(src, tgt, out_f, out_g, cfg->eps, cost, bn, bm, &dual);
            }
            free(sp);
            free(sw);
            free(tp);
            free(tw);
            free(f);
            free(g);
            free(ff);
            free(gg);
        }
    }
    out_scalars[0] = iters;
    out_scalars[1] = viol;
    out_scalars[2] = dual;
    out_scalars[3] = final_eps;
    free(alpha);
    free(beta);
    free(sched);
    free(r);
    free(c);
    return st;
}

/* ---- seeded inputs: xoshiro256** / splitmix64 / Box-Muller (rng.hpp:12-57) ---- */
static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

void fo_rng_normal_fill(uint64_t seed, double* out, int64_t count) {
    uint64_t s[4], x = seed;
    for (int i = 0; i < 4; ++i) {
        x += 0x9e3779b97f4a7c15ULL;
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        s[i] = z ^ (z >> 31);
    }
    int has_spare = 0;
    double spare = 0.0;
    for (int64_t k = 0; k < count; ++k) {
        if (has_spare) {
            has_spare = 0;
            out[k] = spare;
            continue;
        }
        double u[2];
        for (int q = 0; q < 2; ++q) {
            const uint64_t r = rotl64(s[1] * 5, 7) * 9;
            const uint64_t t = s[1] << 17;
            s[2] ^= s[0];
            s[3] ^= s[1];
            s[1] ^= s[2];
            s[0] ^= s[3];
            s[2] ^= t;
            s[3] = rotl64(s[3], 45);
            u[q] = (double)(r >> 11) * 0x1.0p-53;
        }
        while (u[0] <= 0.0) {
            const uint64_t r = rotl64(s[1] * 5, 7) * 9;
            const uint64_t t = s[1] << 17;
            s[2] ^= s[0];
            s[3] ^= s[1];
            s[1] ^= s[2];
            s[0] ^= s[3];
            s[2] ^= t;
            s[3] = rotl64(s[3], 45);
            u[0] = (double)(r >> 11) * 0x1.0p-53;
        }
        const double rad = sqrt(-2.0 * log(u[0]));
        const double ang = 2.0 * 3.14159265358979323846 * u[1];
        spare = rad * sin(ang);
        has_spare = 1;
        out[k] = rad * cos(ang);
    }
}
