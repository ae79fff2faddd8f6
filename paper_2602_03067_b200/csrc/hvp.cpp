// Streaming Hessian-vector product (Thm. 3.5 and
// Appendix F). Every P / P^T application is one CUDA apply pass over the
// cached per-orientation LSE (the potentials are fixed, so the LSE passes run
// once per call); the O(n + m) CG vector algebra stays on the host in double.
// Operation count per call: 2 K_CG + 3 transport-vector, 3 transport-matrix
// (PY, P^T A, P(diag(w2) Y)) and 1 Hadamard-weighted transport.
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/fsk_b200.h"
#include "common.h"
#include "core_kernels.h"
#include "device_ops.h"
#include "hostlib.h"

namespace fskb {
extern thread_local std::string g_err;
}

using namespace fskb;

namespace {

struct HvpCtx {
    const fsk_measure& src;
    const fsk_measure& tgt;
    DevProblem<double>& P;
    ExecCtx& C;
    double eps;
    const double* fd;
    const double* gd;
    const double* lse_f;
    const double* mx_f;
    const double* lse_g;
    const double* mx_g;
    fsk_ledger* ledger;
    const fsk_tiles& tiles;
    const fsk_cost* cost;

    // side 0: out (n x p) = P V ; side 1: out (m x p) = P^T V
    std::vector<double> apply(int side, const std::vector<double>& V, int64_t p,
                              const double* A = nullptr, const double* B = nullptr, int64_t r = 0) {
        const int64_t rows = side == 0 ? src.n : tgt.n, cols = side == 0 ? tgt.n : src.n;
        DevBuf<double> Vd(size_t(cols * p), C.s), out(size_t(rows * p), C.s);
        Vd.upload(V.data(), size_t(cols * p));
        DevBuf<double> Ad, Bd;
        if (A) {
            Ad.alloc(size_t(src.n * r), C.s);
            Ad.upload(A, size_t(src.n * r));
            Bd.alloc(size_t(tgt.n * r), C.s);
            Bd.upload(B, size_t(tgt.n * r));
        }
        const double* kpot = side == 0 ? gd : fd;
        const double* pot = side == 0 ? fd : gd;
        transport<double>(P, side, kpot, pot, eps, side == 0 ? lse_f : lse_g,
                          side == 0 ? mx_f : mx_g, Vd.get(), p, Ad.get(), Bd.get(), r, out.get(),
                          C.flags);
        std::vector<double> h((size_t)(rows * p));
        out.download(h.data(), h.size());
        FSKB_CUDA(cudaStreamSynchronize(C.s));
        if (A)
            ledger_hadamard(ledger, src.n, tgt.n, src.d, r, p, tiles, cost);
        else
            ledger_apply(ledger, src.n, tgt.n, src.d, p, tiles, cost, side == 1);
        return h;
    }
};

double dotv(const std::vector<double>& a, const std::vector<double>& b) {
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}

}  // namespace

extern "C" int fsk_hvp_apply(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                             const double* g_hat, double eps, const fsk_cost* cost,
                             const double* A, const fsk_hvp_config* hcfg, const fsk_tiles* tiles,
                             fsk_ledger* ledger, double* out, fsk_hvp_report* hrep) {
    try {
        if (!src || !tgt || !hcfg) throw ValidationFailure("null argument");
        validate_problem_raw(*src, *tgt, cost);
        validate_tiles_raw(tiles);
        check_potentials_raw(f_hat, src->n, g_hat, tgt->n, eps);
        if (!(hcfg->tau >= 0.0)) throw ValidationFailure("hvp: tau must be nonnegative");
        if (!(hcfg->cg_tol > 0.0)) throw ValidationFailure("hvp: cg_tol must be positive");
        if (hcfg->cg_max_iters < 1) throw ValidationFailure("hvp: cg_max_iters must be positive");
        if (!all_finite(A, src->n * src->d)) throw ValidationFailure("hvp: non-finite direction");
        const int64_t n = src->n, m = tgt->n, d = src->d;
        auto& C = exec_ctx();
        DevProblem<double> P;
        P.upload(*src, *tgt, cost, C.s);
        DevBuf<double> f(size_t(n), C.s), g(size_t(m), C.s);
        f.upload(f_hat, size_t(n));
        g.upload(g_hat, size_t(m));
        DevBuf<double> lse_f(size_t(n), C.s), mx_f(size_t(n), C.s), r_d(size_t(n), C.s);
        DevBuf<double> lse_g(size_t(m), C.s), mx_g(size_t(m), C.s), c_d(size_t(m), C.s);
        // workspace: induced marginals (and the per-orientation LSE, cached)
        FinalizeArgs<double> fa{};
        fa.eps = eps;
        fa.flags = C.flags;
        fa.out_lse = lse_f.get();
        fa.out_max = mx_f.get();
        fa.old_pot = f.get();
        fa.w = P.src.w.get();
        fa.out_marg = r_d.get();
        fa.marg_flag = kFlagNonFiniteRowMarginal;
        half_step<double>(P, 0, g.get(), eps, fa);
        FinalizeArgs<double> fb{};
        fb.eps = eps;
        fb.flags = C.flags;
        fb.out_lse = lse_g.get();
        fb.out_max = mx_g.get();
        fb.old_pot = g.get();
        fb.w = P.tgt.w.get();
        fb.out_marg = c_d.get();
        fb.marg_flag = kFlagNonFiniteColMarginal;
        half_step<double>(P, 1, f.get(), eps, fb);
        ledger_marginals(ledger, n, m, d, *tiles, cost);
        std::vector<double> r((size_t)(n)), c((size_t)(m));
        r_d.download(r.data(), r.size());
        c_d.download(c.data(), c.size());
        FSKB_CUDA(cudaStreamSynchronize(C.s));
        throw_for_flags(read_and_clear_flags(C));
        for (double v : r)
            if (!(v > 0.0)) throw NumericalFailure("hvp: zero induced row marginal");

        HvpCtx H{*src, *tgt, P, C, eps, f.get(), g.get(), lse_f.get(), mx_f.get(), lse_g.get(),
                 mx_g.get(), ledger, *tiles, cost};
        const std::vector<double> X(src->points, src->points + n * d);
        const std::vector<double> Y(tgt->points, tgt->points + m * d);
        const std::vector<double> Av(A, A + n * d);
        const std::vector<double> PY = H.apply(0, Y, d);  // cached transport-matrix product

        // build_rhs
        std::vector<double> u((size_t)(n)), uP((size_t)(n)), r1((size_t)(n));
        for (int64_t i = 0; i < n; ++i) {
            double su = 0.0, sp = 0.0;
            for (int64_t t = 0; t < d; ++t) {
                su += X[size_t(i * d + t)] * Av[size_t(i * d + t)];
                sp += PY[size_t(i * d + t)] * Av[size_t(i * d + t)];
            }
            u[size_t(i)] = su;
            uP[size_t(i)] = sp;
            r1[size_t(i)] = 2.0 * (r[size_t(i)] * su - sp);
        }
        const std::vector<double> Ptu = H.apply(1, u, 1);
        const std::vector<double> PtA = H.apply(1, Av, d);
        std::vector<double> r2((size_t)(m));
        for (int64_t j = 0; j < m; ++j) {
            double s = 0.0;
            for (int64_t t = 0; t < d; ++t) s += PtA[size_t(j * d + t)] * Y[size_t(j * d + t)];
            r2[size_t(j)] = 2.0 * (Ptu[size_t(j)] - s);
        }
        // Schur right-hand side r2 - P^T diag(r)^-1 r1
        std::vector<double> tmp((size_t)(n));
        for (int64_t i = 0; i < n; ++i) tmp[size_t(i)] = r1[size_t(i)] / r[size_t(i)];
        std::vector<double> rhs = H.apply(1, tmp, 1);
        for (int64_t j = 0; j < m; ++j) rhs[size_t(j)] = r2[size_t(j)] - rhs[size_t(j)];

        // CG on S_tau = diag(c) - P^T diag(r)^-1 P + tau I
        auto schur = [&](const std::vector<double>& v) {
            std::vector<double> pv = H.apply(0, v, 1);
            for (int64_t i = 0; i < n; ++i) pv[size_t(i)] /= r[size_t(i)];
            std::vector<double> out2 = H.apply(1, pv, 1);
            for (int64_t j = 0; j < m; ++j)
                out2[size_t(j)] = c[size_t(j)] * v[size_t(j)] - out2[size_t(j)] + hcfg->tau * v[size_t(j)];
            return out2;
        };
        std::vector<double> w2((size_t)(m), 0.0);
        const double rn0 = std::sqrt(dotv(rhs, rhs));
        int iters = 0;
        double relres = 0.0;
        bool converged = true;
        if (rn0 > 0.0) {
            std::vector<double> res = rhs, pdir = rhs;
            double rs = dotv(res, res);
            converged = false;
            while (iters < hcfg->cg_max_iters) {
                const std::vector<double> Ap = schur(pdir);
                const double alpha = rs / dotv(pdir, Ap);
                for (int64_t j = 0; j < m; ++j) {
                    w2[size_t(j)] += alpha * pdir[size_t(j)];
                    res[size_t(j)] -= alpha * Ap[size_t(j)];
                }
                ++iters;
                const double rs_new = dotv(res, res);
                if (!std::isfinite(rs_new)) throw NumericalFailure("hvp: non-finite CG iterate");
                if (std::sqrt(rs_new) <= hcfg->cg_tol * rn0) {
                    converged = true;
                    rs = rs_new;
                    break;
                }
                for (int64_t j = 0; j < m; ++j)
                    pdir[size_t(j)] = res[size_t(j)] + (rs_new / rs) * pdir[size_t(j)];
                rs = rs_new;
            }
            relres = std::sqrt(rs) / rn0;
        }
        // w1 = diag(r)^-1 (r1 - P w2) ; R^T w
        const std::vector<double> Pw2 = H.apply(0, w2, 1);
        std::vector<double> w1((size_t)(n));
        for (int64_t i = 0; i < n; ++i) w1[size_t(i)] = (r1[size_t(i)] - Pw2[size_t(i)]) / r[size_t(i)];
        std::vector<double> w2Y((size_t)(m * d));
        for (int64_t j = 0; j < m; ++j)
            for (int64_t t = 0; t < d; ++t) w2Y[size_t(j * d + t)] = w2[size_t(j)] * Y[size_t(j * d + t)];
        const std::vector<double> Pw2Y = H.apply(0, w2Y, d);
        // explicit term: B5 = (P (.) A Y^T) Y
        const std::vector<double> B5 = H.apply(0, Y, d, A, tgt->points, d);
        for (int64_t i = 0; i < n; ++i) {
            const double ri = r[size_t(i)], ui = u[size_t(i)], upi = uP[size_t(i)];
            for (int64_t t = 0; t < d; ++t) {
                const size_t k = size_t(i * d + t);
                const double rtw = 2.0 * (ri * w1[size_t(i)] * X[k] - w1[size_t(i)] * PY[k] +
                                          Pw2[size_t(i)] * X[k] - Pw2Y[k]);
                const double ea = 2.0 * ri * Av[k] -
                                  (4.0 / eps) * (ri * ui * X[k] - ui * PY[k] - upi * X[k] + B5[k]);
                out[k] = rtw / eps + ea;
            }
        }
        throw_for_flags(read_and_clear_flags(C) & ~kFlagNonFinitePotential);
        if (hrep) {
            hrep->cg_iters = iters;
            hrep->cg_rel_residual = relres;
            hrep->converged = converged ? 1 : 0;
        }
        return FSK_OK;
    } catch (const ValidationFailure& e) {
        g_err = e.what();
        return FSK_EVALIDATION;
    } catch (const NumericalFailure& e) {
        g_err = e.what();
        return FSK_ENUMERICAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FSK_ECUDA;
    }
}
