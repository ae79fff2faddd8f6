// Streaming Hessian-vector product (Thm. 3.5 and
// Appendix F). Every P / P^T application is one CUDA apply pass over the
// cached per-orientation LSE (the potentials are fixed, so the LSE passes run
// once per call). On the tensor path the CG iterate, residual and direction stay
// on the device (cg_device.h, one scalar read-back per iteration); the fp64
// engine keeps the O(n + m) CG algebra on the host in double.
// Operation count per call: 2 K_CG + 3 transport-vector, 3 transport-matrix
// (PY, P^T A, P(diag(w2) Y)) and 1 Hadamard-weighted transport.
#include <cmath>
#include <algorithm>
#include <cstring>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/fsk_b200.h"
#include "cg_device.h"
#include "common.h"
#include "core_kernels.h"
#include "device_ops.h"
#include "hostlib.h"
#include "tc_engine.h"

namespace fskb {
extern thread_local std::string g_err;
}

using namespace fskb;

namespace {

// host doubles -> device floats without a host conversion pass
DevBuf<float> narrow_on_device(const double* h, int64_t n, cudaStream_t s) {
    DevBuf<double> tmp(size_t(n), s);
    tmp.upload(h, size_t(n));
    DevBuf<float> out(size_t(n), s);
    launch_f64_to_f32(tmp.get(), out.get(), n, s);
    FSKB_CUDA(cudaStreamSynchronize(s));
    return out;
}

// Rows are independent (each row's sums run in order): split the host n x d
// loops of the HVP assembly over host threads, bit-identical to the serial loop.
template <typename F>
void parallel_rows(int64_t rows, int64_t per_row, F&& f) {
    const int64_t work = rows * per_row;
    const int T = work < (int64_t(1) << 22)
                      ? 1
                      : int(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
    if (T == 1) {
        for (int64_t i = 0; i < rows; ++i) f(i);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
            for (int64_t i = rows * t / T; i < rows * (t + 1) / T; ++i) f(i);
        });
    for (auto& x : th) x.join();
}

template <typename T>
std::vector<T> to_t(const double* p, int64_t n) {
    return std::vector<T>(p, p + n);
}

// T = double: the fp64 CUDA-core engine (reference tolerances).
// T = float: single precision; with the tcgen05 path enabled every
// transport-vector application (2 K_CG + 3 per HVP) runs on the split-fp16
// tensor-core kernel (K1 VEC mode), transport-matrix / Hadamard ones on the
// fp32 CUDA-core kernels.
template <typename T>
struct HvpCtx {
    const fsk_measure& src;
    const fsk_measure& tgt;
    DevProblem<T>& P;
    ExecCtx& C;
    double eps;
    const T* fd;
    const T* gd;
    const T* lse_f;
    const T* mx_f;
    const T* lse_g;
    const T* mx_g;
    fsk_ledger* ledger;
    const fsk_tiles& tiles;
    const fsk_cost* cost;
    const float* l2h[2] = {nullptr, nullptr};   // tensor path: log2 LSE per orientation
    const float* l2l[2] = {nullptr, nullptr};
    const T* marg[2] = {nullptr, nullptr};      // r (side 0), c (side 1)

    // side 0: out (n x p) = P V ; side 1: out (m x p) = P^T V
    std::vector<double> apply(int side, const std::vector<double>& V, int64_t p,
                              const double* A = nullptr, const double* B = nullptr, int64_t r = 0) {
        return apply(side, V.data(), p, A, B, r);
    }
    // tensor path, V already on the device (float, cols x p): out (host doubles)
    std::vector<double> apply_dev(int side, const float* vd, int64_t p) {
        const int64_t rows = side == 0 ? src.n : tgt.n;
        const T* kpot = side == 0 ? gd : fd;
        std::vector<double> h((size_t)(rows * p));
        if constexpr (std::is_same_v<T, float>) {
            DevBuf<float> out(size_t(rows * p), C.s);
            P.s = C.s;
            P.tc->apply_mat(P, side, kpot, float(eps), l2h[side], l2l[side], marg[side], vd, p,
                            out.get(), C.flags, nullptr);
            DevBuf<double> wide(size_t(rows * p), C.s);
            launch_f32_to_f64(out.get(), wide.get(), rows * p, C.s);
            wide.download(h.data(), h.size());
            FSKB_CUDA(cudaStreamSynchronize(C.s));
        }
        ledger_apply(ledger, src.n, tgt.n, src.d, p, tiles, cost, side == 1);
        return h;
    }
    // V: the caller's (cols x p) row-major doubles, read in place
    std::vector<double> apply(int side, const double* V, int64_t p, const double* A = nullptr,
                              const double* B = nullptr, int64_t r = 0) {
        const int64_t rows = side == 0 ? src.n : tgt.n, cols = side == 0 ? tgt.n : src.n;
        const T* kpot = side == 0 ? gd : fd;
        const T* pot = side == 0 ? fd : gd;
        std::vector<double> h((size_t)(rows * p));
        bool done = false;
        if constexpr (std::is_same_v<T, float>) {
            // Hadamard: the tensor kernel needs B = the key cloud (true in the HVP)
            const bool had_ok = A && side == 0 && B == tgt.points && r == src.d;
            if (P.tc && ((!A && p > 1) || had_ok)) {
                // ship the host doubles as they are, narrow / widen on the device
                DevBuf<float> vd = narrow_on_device(V, cols * p, C.s);
                DevBuf<float> ad;
                if (A) ad = narrow_on_device(A, src.n * r, C.s);
                DevBuf<float> out(size_t(rows * p), C.s);
                P.s = C.s;
                P.tc->apply_mat(P, side, kpot, float(eps), l2h[side], l2l[side], marg[side],
                                vd.get(), p, out.get(), C.flags, ad.get());
                DevBuf<double> wide(size_t(rows * p), C.s);
                launch_f32_to_f64(out.get(), wide.get(), rows * p, C.s);
                wide.download(h.data(), h.size());
                FSKB_CUDA(cudaStreamSynchronize(C.s));
                done = true;
            } else if (P.tc && !A && p == 1) {
                DevBuf<float> vd = narrow_on_device(V, cols, C.s);
                DevBuf<double> out(size_t(rows), C.s);
                P.s = C.s;
                P.tc->vec(P, side, kpot, float(eps), l2h[side], l2l[side], marg[side], vd.get(),
                          out.get(), C.flags);
                out.download(h.data(), h.size());
                FSKB_CUDA(cudaStreamSynchronize(C.s));
                done = true;
            }
        }
        if (!done) {
            DevBuf<T> Vd(size_t(cols * p), C.s), out(size_t(rows * p), C.s);
            const std::vector<T> Vt(V, V + cols * p);
            Vd.upload(Vt.data(), size_t(cols * p));
            DevBuf<T> Ad, Bd;
            if (A) {
                const std::vector<T> At = to_t<T>(A, src.n * r), Bt = to_t<T>(B, tgt.n * r);
                Ad.alloc(size_t(src.n * r), C.s);
                Ad.upload(At.data(), size_t(src.n * r));
                Bd.alloc(size_t(tgt.n * r), C.s);
                Bd.upload(Bt.data(), size_t(tgt.n * r));
                FSKB_CUDA(cudaStreamSynchronize(C.s));
            }
            transport<T>(P, side, kpot, pot, T(eps), side == 0 ? lse_f : lse_g,
                         side == 0 ? mx_f : mx_g, Vd.get(), p, Ad.get(), Bd.get(), r, out.get(),
                         C.flags);
            std::vector<T> ht((size_t)(rows * p));
            out.download(ht.data(), ht.size());
            FSKB_CUDA(cudaStreamSynchronize(C.s));
            h.assign(ht.begin(), ht.end());
        }
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

template <typename T>
void hvp_run(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
             const double* g_hat, double eps, const fsk_cost* cost, const double* A,
             const fsk_hvp_config* hcfg, const fsk_tiles* tiles, fsk_ledger* ledger, double* out,
             fsk_hvp_report* hrep) {
        if (!src || !tgt || !hcfg) throw ValidationFailure("null argument");
        validate_problem_raw(*src, *tgt, cost);
        validate_tiles_raw(tiles);
        check_potentials_raw(f_hat, src->n, g_hat, tgt->n, eps);
        if (!(hcfg->tau >= 0.0)) throw ValidationFailure("hvp: tau must be nonnegative");
        if (!(hcfg->cg_tol > 0.0)) throw ValidationFailure("hvp: cg_tol must be positive");
        if (hcfg->cg_max_iters < 1) throw ValidationFailure("hvp: cg_max_iters must be positive");
        if (!all_finite(A, src->n * src->d)) throw ValidationFailure("hvp: non-finite direction");
        constexpr bool kSingle = std::is_same_v<T, float>;
        if (kSingle && cost && cost->kind != 0)
            throw ValidationFailure("single-precision hvp supports the squared-Euclidean cost only");
        const int64_t n = src->n, m = tgt->n, d = src->d;
        auto& C = exec_ctx();
        PhaseTimer timer(C.s);
        DevProblem<T> P;
        P.upload(*src, *tgt, cost, C.s);
        DevBuf<float> l2h_f, l2l_f, l2h_g, l2l_g;
        if constexpr (kSingle) {
            if (enable_tensor_path(P, tensor_mode_from_env())) {
                P.tc->set_eps(P, eps);
                l2h_f.alloc(size_t(n), C.s);
                l2l_f.alloc(size_t(n), C.s);
                l2h_g.alloc(size_t(m), C.s);
                l2l_g.alloc(size_t(m), C.s);
            }
        }
        DevBuf<T> f(size_t(n), C.s), g(size_t(m), C.s);
        {
            const std::vector<T> ft = to_t<T>(f_hat, n), gt = to_t<T>(g_hat, m);
            f.upload(ft.data(), size_t(n));
            g.upload(gt.data(), size_t(m));
            FSKB_CUDA(cudaStreamSynchronize(C.s));
        }
        DevBuf<T> lse_f(size_t(n), C.s), mx_f(size_t(n), C.s), r_d(size_t(n), C.s);
        DevBuf<T> lse_g(size_t(m), C.s), mx_g(size_t(m), C.s), c_d(size_t(m), C.s);
        // workspace: induced marginals (and the per-orientation LSE, cached)
        FinalizeArgs<T> fa{};
        fa.eps = T(eps);
        fa.flags = C.flags;
        fa.out_lse = lse_f.get();
        fa.out_max = mx_f.get();
        fa.old_pot = f.get();
        fa.w = P.src.w.get();
        fa.out_marg = r_d.get();
        fa.marg_flag = kFlagNonFiniteRowMarginal;
        fa.out_l2h = l2h_f.get();
        fa.out_l2l = l2l_f.get();
        half_step<T>(P, 0, g.get(), T(eps), fa);
        FinalizeArgs<T> fb{};
        fb.eps = T(eps);
        fb.flags = C.flags;
        fb.out_lse = lse_g.get();
        fb.out_max = mx_g.get();
        fb.old_pot = g.get();
        fb.w = P.tgt.w.get();
        fb.out_marg = c_d.get();
        fb.marg_flag = kFlagNonFiniteColMarginal;
        fb.out_l2h = l2h_g.get();
        fb.out_l2l = l2l_g.get();
        half_step<T>(P, 1, f.get(), T(eps), fb);
        if constexpr (kSingle) {
            // every transport pass below runs at these potentials: seed exact row maxima
            // so the recorded live sets hold only blocks within 2^-64 of a row max
            if (P.tc) {
                P.s = C.s;
                P.tc->tighten_live(P, 0, g.get(), float(eps), mx_f.get(), C.flags);
                P.tc->tighten_live(P, 1, f.get(), float(eps), mx_g.get(), C.flags);
                // the ~100 transport-vector passes of the CG then sweep the live blocks
                // of the plan kept in HBM instead of recomputing their scores
                P.tc->build_plan(P, g.get(), f.get(), float(eps), l2h_f.get(), l2l_f.get(),
                                 r_d.get(), C.flags);
            }
        }
        ledger_marginals(ledger, n, m, d, *tiles, cost);
        std::vector<double> r((size_t)(n)), c((size_t)(m));
        {
            std::vector<T> rt((size_t)(n)), ct((size_t)(m));
            r_d.download(rt.data(), rt.size());
            c_d.download(ct.data(), ct.size());
            FSKB_CUDA(cudaStreamSynchronize(C.s));
            r.assign(rt.begin(), rt.end());
            c.assign(ct.begin(), ct.end());
        }
        throw_for_flags(read_and_clear_flags(C));
        for (double v : r)
            if (!(v > 0.0)) throw NumericalFailure("hvp: zero induced row marginal");
        timer.mark("hvp setup + 2 LSE");

        HvpCtx<T> H{*src, *tgt, P, C, eps, f.get(), g.get(), lse_f.get(), mx_f.get(),
                    lse_g.get(), mx_g.get(), ledger, *tiles, cost};
        H.l2h[0] = l2h_f.get();
        H.l2l[0] = l2l_f.get();
        H.l2h[1] = l2h_g.get();
        H.l2l[1] = l2l_g.get();
        H.marg[0] = r_d.get();
        H.marg[1] = c_d.get();
        // the caller's clouds and direction, read in place (no host copies of n x d)
        const double* X = src->points;
        const double* Y = tgt->points;
        const double* Av = A;
        // cached transport-matrix product; on the tensor path V = Y is the resident cloud
        const bool tc_mat = kSingle && P.tc && d > 1;
        // the resident key cloud as float (the tensor path's problems are float)
        const float* y_dev = nullptr;
        if constexpr (kSingle) y_dev = P.tgt.pts.get();
        const std::vector<double> PY = tc_mat ? H.apply_dev(0, y_dev, d) : H.apply(0, Y, d);
        timer.mark("hvp P Y");

        // build_rhs
        std::vector<double> u((size_t)(n)), uP((size_t)(n)), r1((size_t)(n));
        parallel_rows(n, d, [&](int64_t i) {
            double su = 0.0, sp = 0.0;
            for (int64_t t = 0; t < d; ++t) {
                su += X[size_t(i * d + t)] * Av[size_t(i * d + t)];
                sp += PY[size_t(i * d + t)] * Av[size_t(i * d + t)];
            }
            u[size_t(i)] = su;
            uP[size_t(i)] = sp;
            r1[size_t(i)] = 2.0 * (r[size_t(i)] * su - sp);
        });
        const std::vector<double> Ptu = H.apply(1, u, 1);
        const std::vector<double> PtA = H.apply(1, Av, d);
        std::vector<double> r2((size_t)(m));
        parallel_rows(m, d, [&](int64_t j) {
            double s = 0.0;
            for (int64_t t = 0; t < d; ++t) s += PtA[size_t(j * d + t)] * Y[size_t(j * d + t)];
            r2[size_t(j)] = 2.0 * (Ptu[size_t(j)] - s);
        });
        // Schur right-hand side r2 - P^T diag(r)^-1 r1
        std::vector<double> tmp((size_t)(n));
        for (int64_t i = 0; i < n; ++i) tmp[size_t(i)] = r1[size_t(i)] / r[size_t(i)];
        std::vector<double> rhs = H.apply(1, tmp, 1);
        for (int64_t j = 0; j < m; ++j) rhs[size_t(j)] = r2[size_t(j)] - rhs[size_t(j)];

        timer.mark("hvp rhs (P^T u, P^T A, P^T r1/r)");
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
        bool device_cg = false;
        if constexpr (kSingle) device_cg = P.tc != nullptr && rn0 > 0.0;
        if (device_cg) {
            // tensor path: the CG lives on the device; each iteration is two
            // transport-vector passes (P p, then P^T (P p / r)) plus four small
            // vector kernels, and one scalar read-back for the stopping test
            if constexpr (kSingle) {
                DeviceCg cg(m, C.s);
                DevBuf<double> rhs_d(size_t(m), C.s), pv(size_t(n), C.s), ptq(size_t(m), C.s);
                DevBuf<float> tmpf(size_t(n), C.s);
                rhs_d.upload(rhs.data(), size_t(m));
                double rs = cg.init(rhs_d.get());
                converged = false;
                P.s = C.s;
                while (iters < hcfg->cg_max_iters) {
                    P.tc->vec(P, 0, g.get(), float(eps), l2h_f.get(), l2l_f.get(), r_d.get(),
                              cg.pf.get(), pv.get(), C.flags);
                    ledger_apply(ledger, n, m, d, 1, *tiles, cost, false);
                    cg.div_rows(pv.get(), r_d.get(), n, tmpf.get());
                    P.tc->vec(P, 1, f.get(), float(eps), l2h_g.get(), l2l_g.get(), c_d.get(),
                              tmpf.get(), ptq.get(), C.flags);
                    ledger_apply(ledger, n, m, d, 1, *tiles, cost, true);
                    const double rs_new = cg.step(c_d.get(), ptq.get(), hcfg->tau);
                    ++iters;
                    if (!std::isfinite(rs_new)) throw NumericalFailure("hvp: non-finite CG iterate");
                    if (std::sqrt(rs_new) <= hcfg->cg_tol * rn0) {
                        converged = true;
                        rs = rs_new;
                        break;
                    }
                    cg.direction();
                    rs = rs_new;
                }
                relres = std::sqrt(rs) / rn0;
                cg.w2.download(w2.data(), size_t(m));
                FSKB_CUDA(cudaStreamSynchronize(C.s));
            }
        } else if (rn0 > 0.0) {
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
        timer.mark("hvp CG");
        // w1 = diag(r)^-1 (r1 - P w2) ; R^T w
        const std::vector<double> Pw2 = H.apply(0, w2, 1);
        std::vector<double> w1((size_t)(n));
        for (int64_t i = 0; i < n; ++i) w1[size_t(i)] = (r1[size_t(i)] - Pw2[size_t(i)]) / r[size_t(i)];
        std::vector<double> Pw2Y;
        if (tc_mat) {
            // V = diag(w2) Y built on the device from the resident cloud
            DevBuf<double> w2d(size_t(m), C.s);
            w2d.upload(w2.data(), size_t(m));
            DevBuf<float> w2Yd(size_t(m * d), C.s);
            launch_scale_rows(y_dev, w2d.get(), m, d, w2Yd.get(), C.s);
            Pw2Y = H.apply_dev(0, w2Yd.get(), d);
        } else {
            std::vector<double> w2Y((size_t)(m * d));
            for (int64_t j = 0; j < m; ++j)
                for (int64_t t = 0; t < d; ++t)
                    w2Y[size_t(j * d + t)] = w2[size_t(j)] * Y[size_t(j * d + t)];
            Pw2Y = H.apply(0, w2Y, d);
        }
        // explicit term: B5 = (P (.) A Y^T) Y
        timer.mark("hvp P w2, P (w2 Y)");
        const std::vector<double> B5 = H.apply(0, Y, d, A, tgt->points, d);
        timer.mark("hvp Hadamard");
        parallel_rows(n, d, [&](int64_t i) {
            const double ri = r[size_t(i)], ui = u[size_t(i)], upi = uP[size_t(i)];
            for (int64_t t = 0; t < d; ++t) {
                const size_t k = size_t(i * d + t);
                const double rtw = 2.0 * (ri * w1[size_t(i)] * X[k] - w1[size_t(i)] * PY[k] +
                                          Pw2[size_t(i)] * X[k] - Pw2Y[k]);
                const double ea = 2.0 * ri * Av[k] -
                                  (4.0 / eps) * (ri * ui * X[k] - ui * PY[k] - upi * X[k] + B5[k]);
                out[k] = rtw / eps + ea;
            }
        });
        timer.mark("hvp assemble");
        throw_for_flags(read_and_clear_flags(C) & ~kFlagNonFinitePotential);
        if (hrep) {
            hrep->cg_iters = iters;
            hrep->cg_rel_residual = relres;
            hrep->converged = converged ? 1 : 0;
        }
}

template <typename F>
int hvp_guard(F&& f) {
    try {
        f();
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

}  // namespace

extern "C" int fsk_hvp_apply(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                             const double* g_hat, double eps, const fsk_cost* cost,
                             const double* A, const fsk_hvp_config* hcfg, const fsk_tiles* tiles,
                             fsk_ledger* ledger, double* out, fsk_hvp_report* hrep) {
    return hvp_guard([&] {
        hvp_run<double>(src, tgt, f_hat, g_hat, eps, cost, A, hcfg, tiles, ledger, out, hrep);
    });
}

extern "C" int fsk_hvp_apply_single(const fsk_measure* src, const fsk_measure* tgt,
                                    const double* f_hat, const double* g_hat, double eps,
                                    const fsk_cost* cost, const double* A,
                                    const fsk_hvp_config* hcfg, const fsk_tiles* tiles,
                                    fsk_ledger* ledger, double* out, fsk_hvp_report* hrep) {
    return hvp_guard([&] {
        hvp_run<float>(src, tgt, f_hat, g_hat, eps, cost, A, hcfg, tiles, ledger, out, hrep);
    });
}
