#include <thread>
#include <chrono>
#include <cstdio>
// C ABI (include/fsk_b200.h): validation with the reference's messages, IO
// ledger accounting at the caller's TileConfig, host<->device staging, and the
// device-resident solver loop. Every numeric result comes from the CUDA kernels.
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <exception>

#include "../../include/fsk_b200.h"
#include "common.h"
#include "core_kernels.h"
#include "device_ops.h"
#include "hostlib.h"
#include "multi_device.h"
#include "small_solve.h"
#include "tc_engine.h"

namespace fskb {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return FSK_OK;
    } catch (const ValidationFailure& e) {
        g_err = e.what();
        return FSK_EVALIDATION;
    } catch (const NumericalFailure& e) {
        g_err = e.what();
        return FSK_ENUMERICAL;
    } catch (const CudaFailure& e) {
        g_err = e.what();
        return FSK_ECUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FSK_ECUDA;
    }
}

int tensor_mode_from_env() {
    const char* s = std::getenv("FSK_TENSOR_MODE");
    if (!s) return 0;
    const std::string v(s);
    if (v == "fma" || v == "fp32" || v == "1") return 1;
    if (v == "tensor" || v == "split3" || v == "2") return 2;
    return 0;
}

namespace {

// |x_i|^2 (core.cpp:83-96 squared_norms; same per-row summation order), rows
// split across host threads for the large clouds.
// Batch-scoped memo of per-measure host work (validation scans, squared norms),
// keyed by the caller's buffers, which are read-only for the duration of a call.
struct BatchMemo {
    struct Key {
        const double* pts;
        const double* w;
        int64_t n, d;
        bool operator==(const Key& o) const {
            return pts == o.pts && w == o.w && n == o.n && d == o.d;
        }
    };
    std::vector<Key> validated;
    std::vector<std::pair<std::pair<Key, double>, std::vector<double>>> sqnorms;
};
thread_local BatchMemo* t_batch_memo = nullptr;

struct BatchMemoScope {
    BatchMemo memo;
    BatchMemo* prev;
    BatchMemoScope() : prev(t_batch_memo) { t_batch_memo = &memo; }
    ~BatchMemoScope() { t_batch_memo = prev; }
};

std::vector<double> host_sqnorm_compute(const fsk_measure& m, double scale);

std::vector<double> host_sqnorm(const fsk_measure& m, double scale) {
    if (!t_batch_memo) return host_sqnorm_compute(m, scale);
    const BatchMemo::Key k{m.points, m.weights, m.n, m.d};
    for (auto& [key, v] : t_batch_memo->sqnorms)
        if (key.first == k && key.second == scale) return v;
    t_batch_memo->sqnorms.push_back({{k, scale}, host_sqnorm_compute(m, scale)});
    return t_batch_memo->sqnorms.back().second;
}

std::vector<double> host_sqnorm_compute(const fsk_measure& m, double scale) {
    std::vector<double> out((size_t)(m.n));
    auto rows = [&](int64_t i0, int64_t i1) {
        for (int64_t i = i0; i < i1; ++i) {
            double s = 0.0;
            for (int64_t t = 0; t < m.d; ++t) s += m.points[i * m.d + t] * m.points[i * m.d + t];
            out[size_t(i)] = scale != 1.0 ? s * scale : s;
        }
    };
    const int64_t work = m.n * m.d;
    const int nt = work < (int64_t(1) << 22)
                       ? 1
                       : int(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
    if (nt == 1) {
        rows(0, m.n);
        return out;
    }
    std::vector<std::thread> th;
    const int64_t per = (m.n + nt - 1) / nt;
    for (int k = 0; k < nt; ++k)
        th.emplace_back(rows, std::min(m.n, k * per), std::min(m.n, (k + 1) * per));
    for (auto& t : th) t.join();
    return out;
}

template <typename T>
DevBuf<T> dev_from(const double* h, int64_t n, cudaStream_t s) {
    DevBuf<T> b(size_t(n), s);
    if constexpr (std::is_same_v<T, double>) {
        b.upload(h, size_t(n));
    } else {
        std::vector<T> tmp((size_t)(n));
        for (int64_t i = 0; i < n; ++i) tmp[size_t(i)] = T(h[i]);
        b.upload(tmp.data(), size_t(n));
        FSKB_CUDA(cudaStreamSynchronize(s));
    }
    return b;
}

template <typename T>
void dev_to(const DevBuf<T>& b, double* h, int64_t n, cudaStream_t s) {
    if constexpr (std::is_same_v<T, double>) {
        b.download(h, size_t(n));
        FSKB_CUDA(cudaStreamSynchronize(s));
    } else {
        // widen on the device, then one copy straight into the caller's buffer
        DevBuf<double> wide(size_t(n), s);
        launch_f32_to_f64(b.get(), wide.get(), n, s);
        wide.download(h, size_t(n));
        FSKB_CUDA(cudaStreamSynchronize(s));
    }
}

void sync_and_check(ExecCtx& C, int ignore = 0, const std::string& suffix = "") {
    throw_for_flags(read_and_clear_flags(C) & ~ignore, suffix);
}

int bad_iteration(ExecCtx& C) {
    int h[2];
    FSKB_CUDA(cudaMemcpyAsync(h, C.flags, sizeof(h), cudaMemcpyDeviceToHost, C.s));
    FSKB_CUDA(cudaStreamSynchronize(C.s));
    return h[1];
}

void common_checks(const fsk_measure* src, const fsk_measure* tgt, const fsk_cost* cost,
                   const fsk_tiles* tiles, bool check_points = true) {
    if (!src || !tgt) throw ValidationFailure("null measure");
    if (t_batch_memo) {
        // scan each distinct measure of a batch once (same checks, same order)
        for (const fsk_measure* m : {src, tgt}) {
            const BatchMemo::Key k{m->points, m->weights, m->n, m->d};
            bool seen = false;
            for (auto& v : t_batch_memo->validated) seen = seen || v == k;
            if (!seen) {
                validate_measure_raw(*m);
                if (m->labels == nullptr) t_batch_memo->validated.push_back(k);
            }
        }
        validate_problem_raw(*src, *tgt, cost, /*measures_checked=*/true);
    } else {
        validate_problem_raw(*src, *tgt, cost, false, check_points);
    }
    validate_tiles_raw(tiles);
}

// Entry-point validation of the single-device single-precision solves: every check
// of common_checks except the coordinate finiteness scan, which the device ingest
// performs (DevProblem::ingest). Returns true when that scan is left to the solve.
// On any other failure the full checks run, so the error raised is the reference's
// first one in its own order (core.cpp:18-81).
bool checks_deferring_points(const fsk_measure* src, const fsk_measure* tgt, const fsk_cost* cost,
                             const fsk_tiles* tiles, const fsk_config* cfg) {
    const char* e = std::getenv("FSK_DEVICE_INGEST");
    const bool defer = cfg && cfg->precision == 0 && num_devices_setting() < 1 && !t_batch_memo &&
                       !labeled_cost(cost) && src && tgt && !(e && e[0] == '0');
    if (!defer) {
        common_checks(src, tgt, cost, tiles);
        return false;
    }
    try {
        common_checks(src, tgt, cost, tiles, /*check_points=*/false);
        validate_config_raw(*cfg);   // (the reference checks the config after the points)
    } catch (const ValidationFailure&) {
        common_checks(src, tgt, cost, tiles);
        throw;
    }
    return true;
}

// r (n) and c (m) of the induced marginals at (f, g), all on device.
template <typename T>
void dev_marginals(DevProblem<T>& P, const T* f, const T* g, T eps, T* r, T* c, T* lse_f,
                   T* mx_f, int* flags, float* l2h_f = nullptr, float* l2l_f = nullptr) {
    FinalizeArgs<T> fa{};
    fa.eps = eps;
    fa.flags = flags;
    fa.old_pot = f;
    fa.w = P.src.w.get();
    fa.out_marg = r;
    fa.marg_flag = kFlagNonFiniteRowMarginal;
    fa.out_lse = lse_f;
    fa.out_max = mx_f;
    fa.out_l2h = l2h_f;
    fa.out_l2l = l2l_f;
    half_step<T>(P, 0, g, eps, fa);
    FinalizeArgs<T> fb{};
    fb.eps = eps;
    fb.flags = flags;
    fb.old_pot = g;
    fb.w = P.tgt.w.get();
    fb.out_marg = c;
    fb.marg_flag = kFlagNonFiniteColMarginal;
    half_step<T>(P, 1, f, eps, fb);
}

struct HostMarginals {
    std::vector<double> r, c;
};

double violation(const HostMarginals& hm, const fsk_measure& a, const fsk_measure& b) {
    double v = 0.0;
    for (int64_t i = 0; i < a.n; ++i) v += std::abs(hm.r[size_t(i)] - a.weights[i]);
    for (int64_t j = 0; j < b.n; ++j) v += std::abs(hm.c[size_t(j)] - b.weights[j]);
    return v;
}

// <f,a> + <g,b> - eps (sum r - 1) with unshifted potentials (solver.cpp:131-143)
double dual_value(const fsk_measure& a, const fsk_measure& b, const double* fh, const double* gh,
                  const double* alpha, const double* beta, const std::vector<double>& r,
                  double eps) {
    const double mass = cascade_sum(r.data(), r.size());
    double value = 0.0;
    for (int64_t i = 0; i < a.n; ++i) value += (fh[i] + alpha[i]) * a.weights[i];
    for (int64_t j = 0; j < b.n; ++j) value += (gh[j] + beta[j]) * b.weights[j];
    return value - eps * (mass - 1.0);
}

template <typename T>
// r_keep / l2 keeps (tensor path): the f-side pass's marginal and log2 LSE, so the
// gradient at the same potentials does not repeat that pass.
HostMarginals marginals_to_host(DevProblem<T>& P, const T* f, const T* g, T eps, ExecCtx& C,
                                DevBuf<T>* lse_keep = nullptr, DevBuf<T>* mx_keep = nullptr,
                                DevBuf<T>* r_keep = nullptr, DevBuf<float>* l2h_keep = nullptr,
                                DevBuf<float>* l2l_keep = nullptr) {
    const int64_t n = P.src.n, m = P.tgt.n;
    DevBuf<T> r(size_t(n), C.s), c(size_t(m), C.s);
    dev_marginals<T>(P, f, g, eps, r.get(), c.get(), lse_keep ? lse_keep->get() : nullptr,
                     mx_keep ? mx_keep->get() : nullptr, C.flags,
                     l2h_keep ? l2h_keep->get() : nullptr, l2l_keep ? l2l_keep->get() : nullptr);
    HostMarginals hm;
    hm.r.resize(size_t(n));
    hm.c.resize(size_t(m));
    dev_to<T>(r, hm.r.data(), n, C.s);
    dev_to<T>(c, hm.c.data(), m, C.s);
    if (r_keep) *r_keep = std::move(r);
    return hm;
}

// A device result (fp64) copied into a page-locked host buffer on a copy stream,
// ordered after the work enqueued so far on the compute stream, while that stream
// carries on. finish() waits for the copy.
struct EarlyDownload {
    DevBuf<double> wide;
    DevBuf<int> flags;
    cudaStream_t cs = nullptr;
    cudaEvent_t ready = nullptr;
    void start(double* host, std::size_t bytes, cudaStream_t s) {
        FSKB_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        FSKB_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
        FSKB_CUDA(cudaEventRecord(ready, s));
        FSKB_CUDA(cudaStreamWaitEvent(cs, ready, 0));
        FSKB_CUDA(cudaMemcpyAsync(host, wide.get(), bytes, cudaMemcpyDeviceToHost, cs));
    }
    bool started() const { return cs != nullptr; }
    void finish(cudaStream_t s) {
        if (!cs) return;
        FSKB_CUDA(cudaStreamSynchronize(cs));
        // the buffers are freed on the compute stream: order it after the copy
        FSKB_CUDA(cudaEventRecord(ready, cs));
        FSKB_CUDA(cudaStreamWaitEvent(s, ready, 0));
    }
    ~EarlyDownload() {
        if (cs) {
            cudaStreamSynchronize(cs);
            cudaStreamDestroy(cs);
        }
        if (ready) cudaEventDestroy(ready);
    }
};

// Device-resident Sinkhorn (solver.cpp:21-117). T = double: Precision::Double;
// T = float: Precision::Single (tensor-core or FMA half-steps).
template <typename T>
void solve_impl(const fsk_measure& src, const fsk_measure& tgt, const fsk_cost* cost,
                const fsk_config& cfg, const fsk_tiles& tiles, fsk_ledger* ledger,
                fsk_report* rep, double* grad_out, const double* f_init = nullptr,
                const double* g_init = nullptr, bool points_unchecked = false) {
    constexpr bool kSingle = std::is_same_v<T, float>;
    const int64_t n = src.n, m = tgt.n, d = src.d;
    const double fs = feature_scale(cost);
    if (num_devices_setting() >= 1 && cfg.schedule == 0) {
        // sharded over the configured devices (multi_device.cpp)
        const std::vector<double> alpha_m = host_sqnorm(src, fs), beta_m = host_sqnorm(tgt, fs);
        const double diam2_m = cfg.eps_scaling_factor < 1.0
                                   ? joint_sq_diameter_raw(src.points, n, tgt.points, m, d)
                                   : 0.0;
        if (solve_multi_device<T>(src, tgt, cost, cfg, eps_schedule_raw(cfg, diam2_m), alpha_m,
                                  beta_m, f_init, g_init, tiles, ledger, rep, grad_out))
            return;
    }
    auto& C = exec_ctx();
    PhaseTimer timer(C.s);
    DevProblem<T> P;
    // the gradient's host pages are faulted in while the device iterates
    HostPrefault prefault;
    if (grad_out) prefault.start(grad_out, sizeof(double) * size_t(n) * size_t(d));
    // alpha = |x|^2, beta = |y|^2 (core.cpp:83-96) on the host, for the dual value
    std::vector<double> alpha_v, beta_v;
    PinnedHost<double> alpha_h, beta_h;
    const double* alpha = nullptr;
    const double* beta = nullptr;
    DevBuf<T> f, g;
    if (kSingle && points_unchecked) {
        // single-precision ingest: the caller's doubles cross the link once and the
        // device narrows them, checks their finiteness (validate_measure, deferred
        // here by the entry point) and forms alpha, beta and the initial potentials
        // f_hat = -alpha, g_hat = -beta (solver.cpp:27-32): no host pass over the clouds
        f.alloc(size_t(n), C.s);
        g.alloc(size_t(m), C.s);
        DevBuf<double> alpha_d, beta_d;
        if (!P.ingest(src, tgt, fs, C.s, alpha_d, beta_d, f_init ? nullptr : f.get(),
                      g_init ? nullptr : g.get()))
            throw ValidationFailure(kNonFiniteCoordinate);
        if (f_init) f = dev_from<T>(f_init, n, C.s);
        if (g_init) g = dev_from<T>(g_init, m, C.s);
        alpha_h = PinnedHost<double>(size_t(n));
        beta_h = PinnedHost<double>(size_t(m));
        FSKB_CUDA(cudaMemcpyAsync(alpha_h.get(), alpha_d.get(), sizeof(double) * size_t(n),
                                  cudaMemcpyDeviceToHost, C.s));
        FSKB_CUDA(cudaMemcpyAsync(beta_h.get(), beta_d.get(), sizeof(double) * size_t(m),
                                  cudaMemcpyDeviceToHost, C.s));
        alpha = alpha_h.get();
        beta = beta_h.get();
        timer.mark("upload + ingest");
        if constexpr (kSingle) enable_tensor_path(P, tensor_mode_from_env());
        timer.mark("operand images");
    } else {
        P.upload(src, tgt, cost, C.s);
        timer.mark("upload");
        if constexpr (kSingle) enable_tensor_path(P, tensor_mode_from_env());
        timer.mark("operand images");
        alpha_v = host_sqnorm(src, fs);
        beta_v = host_sqnorm(tgt, fs);
        alpha = alpha_v.data();
        beta = beta_v.data();
        std::vector<double> f0((size_t)(n)), g0((size_t)(m));
        // reference init f = g = 0, i.e. f_hat = -alpha, g_hat = -beta (solver.cpp:27-32);
        // a warm start (fsk_sinkhorn_solve_warm) starts from the caller's shifted pair
        for (int64_t i = 0; i < n; ++i) f0[size_t(i)] = f_init ? f_init[i] : -alpha[size_t(i)];
        for (int64_t j = 0; j < m; ++j) g0[size_t(j)] = g_init ? g_init[j] : -beta[size_t(j)];
        f = dev_from<T>(f0.data(), n, C.s);
        g = dev_from<T>(g0.data(), m, C.s);
    }
    DevBuf<T> f2, g2;
    if (cfg.schedule == 1) {
        f2.alloc(size_t(n), C.s);
        g2.alloc(size_t(m), C.s);
    }

    timer.mark("initial potentials");
    // the squared diameter only feeds the geometric eps decay (schedule.cpp:27-44)
    const double diam2 =
        cfg.eps_scaling_factor < 1.0 ? joint_sq_diameter_raw(src.points, n, tgt.points, m, d) : 0.0;
    const auto schedule = eps_schedule_raw(cfg, diam2);
    timer.mark("eps schedule");
    int iters = 0;
    double viol = 0.0, dual = 0.0, final_eps = 0.0;
    bool stopped = false;
    std::vector<double> hist;
    double cur_tc_eps = -1.0;
    // Fused convergence check (alternating schedule, fp64, marginal_tol > 0; SURVEY
    // §8a): the violation of iterate k needs f+ = the f-update of iteration k + 1,
    // so that f-update emits r_i = a_i exp((f_k - f_{k+1})/eps) and sum |r - a| as a
    // by-product (c = b exactly: g_k is the g-update of f_k). Stopping returns
    // iterate k and drops f_{k+1}: the reference's result (solver.cpp:51-60) for one
    // extra pass at the stop instead of two marginal passes every iteration.
    const bool fused_check = !kSingle && cfg.marginal_tol > 0.0 && cfg.schedule == 0;
    DevBuf<T> f_next, r_dev;
    DevBuf<double> viol_dev;
    bool check_pending = false;   // iterate `iters` awaits its violation
    if (fused_check) {
        f_next.alloc(size_t(n), C.s);
        r_dev.alloc(size_t(n), C.s);
        viol_dev.alloc(1, C.s);
    }
    bool persistent_done = false;
    if constexpr (kSingle) {
        // small fp32 CUDA-core problems: the whole alternating loop (the f32 path has no
        // early stop, solver.cpp:87-108) is one persistent kernel (small_solve.cu)
        const char* penv = std::getenv("FSK_PERSIST");
        if (!P.tc && !P.labeled && cfg.schedule == 0 && !schedule.empty() &&
            !(penv && penv[0] == '0') && small_solve_fits(n, m, d)) {
            const std::vector<float> es(schedule.begin(), schedule.end());
            DevBuf<float> es_d(es.size(), C.s);
            FSKB_CUDA(cudaMemcpyAsync(es_d.get(), es.data(), es.size() * sizeof(float),
                                      cudaMemcpyHostToDevice, C.s));
            SmallSolveParams sp{};
            sp.X = P.src.pts.get();
            sp.Y = P.tgt.pts.get();
            sp.logw_x = P.src.logw.get();
            sp.logw_y = P.tgt.logw.get();
            sp.f = f.get();
            sp.g = g.get();
            sp.eps_sched = es_d.get();
            sp.iters = int(es.size());
            sp.n = n;
            sp.m = m;
            sp.d = int(d);
            sp.fscale = float(P.fscale);
            sp.flags = C.flags;
            sp.bad_iter = C.bad_iter;
            launch_small_solve(sp, C.s);
            FSKB_CUDA(cudaStreamSynchronize(C.s));
            for (double eps_d : schedule) {
                ledger_update_f32(ledger, n, m, d, tiles.block_rows, tiles.block_cols);
                ledger_update_f32(ledger, m, n, d, tiles.block_cols, tiles.block_rows);
                hist.push_back(eps_d);
                final_eps = eps_d;
                ++iters;
            }
            persistent_done = true;
        }
    }
    for (double eps_d : schedule) {
        if (persistent_done) break;
        const T eps = T(eps_d);
        final_eps = eps_d;
        if constexpr (kSingle) {
            if (P.tc && cur_tc_eps != eps_d) {
                P.tc->set_eps(P, eps_d);
                cur_tc_eps = eps_d;
            }
        }
        FinalizeArgs<T> fa{};
        fa.eps = eps;
        fa.flags = C.flags;
        fa.bad_iter = C.bad_iter;
        fa.iter = iters + 1;
        if (cfg.schedule == 0 && check_pending) {
            // f_{k+1} with the lagged violation of iterate k fused into its epilogue
            FinalizeArgs<T> fv = fa;
            fv.out_pot = f_next.get();
            fv.old_pot = f.get();
            fv.w = P.src.w.get();
            fv.out_marg = r_dev.get();
            fv.marg_flag = kFlagNonFiniteRowMarginal;
            fv.viol = viol_dev.get();
            viol_dev.zero();
            half_step<T>(P, 0, g.get(), eps, fv);
            double hv = 0.0;
            FSKB_CUDA(cudaMemcpyAsync(&hv, viol_dev.get(), sizeof(double), cudaMemcpyDeviceToHost,
                                      C.s));
            FSKB_CUDA(cudaStreamSynchronize(C.s));
            // the reference's induced_marginals + violation of iterate k
            ledger_marginals(ledger, n, m, d, tiles, cost);
            check_pending = false;
            viol = hv;
            if (viol <= cfg.marginal_tol) {
                const int fl = read_and_clear_flags(C);
                if (fl) throw_for_flags(fl, " at iteration " + std::to_string(iters));
                HostMarginals hm;
                hm.r.resize(size_t(n));
                dev_to<T>(r_dev, hm.r.data(), n, C.s);
                std::vector<double> fh((size_t)(n)), gh((size_t)(m));
                dev_to<T>(f, fh.data(), n, C.s);
                dev_to<T>(g, gh.data(), m, C.s);
                ledger_marginals(ledger, n, m, d, tiles, cost);
                dual = dual_value(src, tgt, fh.data(), gh.data(), alpha, beta, hm.r, final_eps);
                stopped = true;
                break;
            }
            std::swap(f, f_next);
            fa.out_pot = g.get();
            half_step<T>(P, 1, f.get(), eps, fa);
            ledger_update_f(ledger, n, m, d, tiles, cost);
            ledger_update_g(ledger, n, m, d, tiles, cost);
        } else if (cfg.schedule == 0) {
            fa.out_pot = f.get();
            half_step<T>(P, 0, g.get(), eps, fa);
            fa.out_pot = g.get();
            half_step<T>(P, 1, f.get(), eps, fa);
            if (kSingle) {
                ledger_update_f32(ledger, n, m, d, tiles.block_rows, tiles.block_cols);
                ledger_update_f32(ledger, m, n, d, tiles.block_cols, tiles.block_rows);
            } else {
                ledger_update_f(ledger, n, m, d, tiles, cost);
                ledger_update_g(ledger, n, m, d, tiles, cost);
            }
        } else {
            fa.out_pot = f2.get();
            fa.sym_old = f.get();
            half_step<T>(P, 0, g.get(), eps, fa);
            fa.out_pot = g2.get();
            fa.sym_old = g.get();
            half_step<T>(P, 1, f.get(), eps, fa);
            std::swap(f, f2);
            std::swap(g, g2);
            if (kSingle) {
                ledger_update_f32(ledger, n, m, d, tiles.block_rows, tiles.block_cols);
                ledger_update_f32(ledger, m, n, d, tiles.block_cols, tiles.block_rows);
                if (ledger) ledger->slow_to_fast_scalars += uint64_t(n + m);
            } else {
                ledger_symmetric(ledger, n, m, d, tiles, cost);
            }
        }
        ++iters;
        hist.push_back(eps_d);
        // early stopping is checked at the final eps only; the reference's
        // single-precision loop ignores it (solver.cpp:87-108)
        if (fused_check && eps_d == cfg.eps) {
            check_pending = true;   // decided by the next iteration's f-update
        } else if (!kSingle && !fused_check && cfg.marginal_tol > 0.0 && eps_d == cfg.eps) {
            const int fl = read_and_clear_flags(C);
            if (fl) throw_for_flags(fl, " at iteration " + std::to_string(iters));
            HostMarginals hm = marginals_to_host<T>(P, f.get(), g.get(), eps, C);
            ledger_marginals(ledger, n, m, d, tiles, cost);
            sync_and_check(C);
            viol = violation(hm, src, tgt);
            if (viol <= cfg.marginal_tol) {
                std::vector<double> fh((size_t)(n)), gh((size_t)(m));
                dev_to<T>(f, fh.data(), n, C.s);
                dev_to<T>(g, gh.data(), m, C.s);
                // dual_cost recomputes the same marginals (deterministic kernels)
                ledger_marginals(ledger, n, m, d, tiles, cost);
                dual = dual_value(src, tgt, fh.data(), gh.data(), alpha, beta, hm.r, eps_d);
                stopped = true;
                break;
            }
        }
    }
    timer.mark("iterations");
    {
        const int bad = bad_iteration(C);
        const int fl = read_and_clear_flags(C);
        if (fl) throw_for_flags(fl, bad != INT_MAX ? " at iteration " + std::to_string(bad) : "");
    }
    const double pot_eps = kSingle ? cfg.eps : final_eps;
    std::vector<double> fh((size_t)(n)), gh((size_t)(m));
    dev_to<T>(f, fh.data(), n, C.s);
    dev_to<T>(g, gh.data(), m, C.s);
    DevBuf<T> lse_f(size_t(n), C.s), mx_f(size_t(n), C.s);
    EarlyDownload early_grad;
    DevBuf<T> r_keep;
    DevBuf<float> l2h_keep, l2l_keep;
    if (!stopped) {
        if constexpr (kSingle) {
            if (P.tc && cur_tc_eps != pot_eps) P.tc->set_eps(P, pot_eps);
        }
        const bool keep = kSingle && P.tc && grad_out;
        if (keep) {
            l2h_keep.alloc(size_t(n), C.s);
            l2l_keep.alloc(size_t(n), C.s);
        }
        HostMarginals hm = marginals_to_host<T>(P, f.get(), g.get(), T(pot_eps), C, &lse_f, &mx_f,
                                                keep ? &r_keep : nullptr,
                                                keep ? &l2h_keep : nullptr,
                                                keep ? &l2l_keep : nullptr);
        sync_and_check(C);   // (the stream is idle here: the marginals were downloaded)
        const char* ov = std::getenv("FSK_OVERLAP_GRAD");
        if constexpr (kSingle) {
            if (keep && host_pinned(grad_out) && !(ov && ov[0] == '0')) {
                // page-locked gradient output: enqueue the gradient (fused K3 on the
                // f-side pass's LSE) and its download on a copy stream now, so the
                // host's violation / dual work below overlaps them. The gradient
                // reports into its own status word, read after the marginals' (the
                // sequential order of the checks).
                early_grad.flags.alloc(1, C.s);
                early_grad.flags.zero();
                DevBuf<T> G(size_t(n * d), C.s);
                P.tc->grad(P, 0, g.get(), f.get(), T(pot_eps), 0, n, G.get(),
                           early_grad.flags.get(), l2h_keep.get(), l2l_keep.get(),
                           r_keep.get());
                early_grad.wide.alloc(size_t(n * d), C.s);
                launch_f32_to_f64(G.get(), early_grad.wide.get(), n * d, C.s);
                early_grad.start(grad_out, sizeof(double) * size_t(n * d), C.s);
            }
        }
        ledger_marginals(ledger, n, m, d, tiles, cost);
        viol = violation(hm, src, tgt);
        // the last iterate's own tolerance check (fused path: never run in the loop);
        // the reference charges it unless that check stopped the solve
        if (check_pending && !(viol <= cfg.marginal_tol)) ledger_marginals(ledger, n, m, d, tiles, cost);
        ledger_marginals(ledger, n, m, d, tiles, cost);
        dual = dual_value(src, tgt, fh.data(), gh.data(), alpha, beta, hm.r, pot_eps);
    }
    if (rep) {
        rep->iterations = iters;
        rep->marginal_violation = viol;
        rep->dual_cost = dual;
        rep->eps = pot_eps;
        if (rep->f_hat) std::memcpy(rep->f_hat, fh.data(), sizeof(double) * size_t(n));
        if (rep->g_hat) std::memcpy(rep->g_hat, gh.data(), sizeof(double) * size_t(m));
        if (rep->eps_history)
            for (int64_t k = 0; k < rep->eps_history_cap && k < int64_t(hist.size()); ++k)
                rep->eps_history[k] = hist[size_t(k)];
    }
    timer.mark("marginals + dual");
    if (grad_out && early_grad.started()) {
        early_grad.finish(C.s);
        timer.mark("gradient (overlapped) + download");
        int fl = 0;
        FSKB_CUDA(cudaMemcpy(&fl, early_grad.flags.get(), sizeof(int), cudaMemcpyDeviceToHost));
        throw_for_flags(fl);
        sync_and_check(C);
        if (ledger) {
            ledger_marginals(ledger, n, m, d, tiles, cost);
            ledger_apply(ledger, n, m, d, d, tiles, cost, false);
        }
    } else if (grad_out) {
        // grad_X = 2 r (X - softmax(S) Y) at the returned potentials
        const T eps = T(pot_eps);
        DevBuf<T> G(size_t(n * d), C.s);
        bool done = false;
        if constexpr (kSingle) {
            if (P.tc) {
                // fused tcgen05 path: K1 row LSE + split-fp16 transport kernel
                if (!r_keep.get()) P.tc->set_eps(P, pot_eps);
                if constexpr (kSingle)
                    P.tc->grad(P, 0, g.get(), f.get(), eps, 0, n, G.get(), C.flags, l2h_keep.get(),
                               l2l_keep.get(), r_keep.get());
                done = true;
            }
        }
        if constexpr (kSingle) {
            if (!done) {
                // CUDA-core fp32 problem: the gradient pass in fp64 (grad_rows_fp64)
                DevBuf<double> G64(size_t(n * d), C.s);
                grad_rows_fp64(P, f.get(), g.get(), pot_eps, 0, n, G64.get(), C.flags, C.s);
                prefault.join();
                G64.download(grad_out, size_t(n * d));
                done = true;
                sync_and_check(C);
                if (ledger) {
                    ledger_marginals(ledger, n, m, d, tiles, cost);
                    ledger_apply(ledger, n, m, d, d, tiles, cost, false);
                }
                return;
            }
        }
        if (!done) {
            if (stopped) {
                FinalizeArgs<T> fa{};
                fa.eps = eps;
                fa.flags = C.flags;
                fa.out_lse = lse_f.get();
                fa.out_max = mx_f.get();
                half_step<T>(P, 0, g.get(), eps, fa);
            }
            DevBuf<T> O(size_t(n * d), C.s);
            launch_apply<T>(P.params(0, g.get(), eps), lse_f.get(), P.tgt.pts.get(), d, nullptr,
                            nullptr, 0, O.get(), C.s);
            launch_grad_epilogue<T>(P.src.pts.get(), O.get(), P.src.w.get(), f.get(),
                                    lse_f.get(), n, d, eps, G.get(), C.flags, C.s);
        }
        timer.mark("gradient");
        prefault.join();
        timer.mark("output page faults + lock (join)");
        if (prefault.pinned()) {
            // one DMA into the page-locked caller buffer (widened on the device)
            if constexpr (std::is_same_v<T, double>) {
                FSKB_CUDA(cudaMemcpyAsync(grad_out, G.get(), sizeof(double) * size_t(n * d),
                                          cudaMemcpyDeviceToHost, C.s));
                FSKB_CUDA(cudaStreamSynchronize(C.s));
            } else {
                DevBuf<double> wide(size_t(n * d), C.s);
                launch_f32_to_f64(G.get(), wide.get(), n * d, C.s);
                FSKB_CUDA(cudaMemcpyAsync(grad_out, wide.get(), sizeof(double) * size_t(n * d),
                                          cudaMemcpyDeviceToHost, C.s));
                FSKB_CUDA(cudaStreamSynchronize(C.s));
            }
        } else {
            dev_to<T>(G, grad_out, n * d, C.s);
        }
        prefault.release();
        timer.mark("gradient download");
        sync_and_check(C);
        if (ledger) {
            ledger_marginals(ledger, n, m, d, tiles, cost);
            ledger_apply(ledger, n, m, d, d, tiles, cost, false);
        }
    }
}

}  // namespace
}  // namespace fskb

using namespace fskb;

extern "C" {

const char* fsk_last_error(void) { return g_err.c_str(); }

int fsk_update_f_hat(const fsk_measure* src, const fsk_measure* tgt, const double* g_hat,
                     const fsk_cost* cost, double eps, const fsk_tiles* tiles, fsk_ledger* ledger,
                     double* out) {
    return guarded([&] {
        common_checks(src, tgt, cost, tiles);
        if (!(eps > 0.0)) throw ValidationFailure("eps must be positive");
        if (!all_finite(g_hat, tgt->n)) throw ValidationFailure("non-finite g_hat entry");
        ledger_update_f(ledger, src->n, tgt->n, src->d, *tiles, cost);
        auto& C = exec_ctx();
        DevProblem<double> P;
        P.upload(*src, *tgt, cost, C.s);
        DevBuf<double> g = dev_from<double>(g_hat, tgt->n, C.s), f(size_t(src->n), C.s);
        FinalizeArgs<double> fa{};
        fa.eps = eps;
        fa.out_pot = f.get();
        fa.flags = C.flags;
        half_step<double>(P, 0, g.get(), eps, fa);
        dev_to<double>(f, out, src->n, C.s);
        sync_and_check(C);
    });
}

int fsk_update_g_hat(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                     const fsk_cost* cost, double eps, const fsk_tiles* tiles, fsk_ledger* ledger,
                     double* out) {
    return guarded([&] {
        common_checks(src, tgt, cost, tiles);
        if (!(eps > 0.0)) throw ValidationFailure("eps must be positive");
        if (!all_finite(f_hat, src->n)) throw ValidationFailure("non-finite f_hat entry");
        ledger_update_g(ledger, src->n, tgt->n, src->d, *tiles, cost);
        auto& C = exec_ctx();
        DevProblem<double> P;
        P.upload(*src, *tgt, cost, C.s);
        DevBuf<double> f = dev_from<double>(f_hat, src->n, C.s), g(size_t(tgt->n), C.s);
        FinalizeArgs<double> fa{};
        fa.eps = eps;
        fa.out_pot = g.get();
        fa.flags = C.flags;
        half_step<double>(P, 1, f.get(), eps, fa);
        dev_to<double>(g, out, tgt->n, C.s);
        sync_and_check(C);
    });
}

int fsk_symmetric_update(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                         const double* g_hat, double eps, const fsk_cost* cost,
                         const fsk_tiles* tiles, fsk_ledger* ledger, double* out_f,
                         double* out_g) {
    return guarded([&] {
        common_checks(src, tgt, cost, tiles);
        check_potentials_raw(f_hat, src->n, g_hat, tgt->n, eps);
        ledger_symmetric(ledger, src->n, tgt->n, src->d, *tiles, cost);
        auto& C = exec_ctx();
        DevProblem<double> P;
        P.upload(*src, *tgt, cost, C.s);
        DevBuf<double> f = dev_from<double>(f_hat, src->n, C.s);
        DevBuf<double> g = dev_from<double>(g_hat, tgt->n, C.s);
        DevBuf<double> fn(size_t(src->n), C.s), gn(size_t(tgt->n), C.s);
        FinalizeArgs<double> fa{};
        fa.eps = eps;
        fa.flags = C.flags;
        fa.out_pot = fn.get();
        fa.sym_old = f.get();
        half_step<double>(P, 0, g.get(), eps, fa);
        fa.out_pot = gn.get();
        fa.sym_old = g.get();
        half_step<double>(P, 1, f.get(), eps, fa);
        dev_to<double>(fn, out_f, src->n, C.s);
        dev_to<double>(gn, out_g, tgt->n, C.s);
        sync_and_check(C);
    });
}

namespace {
// P V (side 0) or P^T U (side 1) with optional Hadamard factors, host buffers.
int transport_host(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                   const double* g_hat, double eps, const fsk_cost* cost, const double* A,
                   const double* B, int64_t r, const double* V, int64_t p, int side,
                   double* out) {
    auto& C = exec_ctx();
    DevProblem<double> P;
    P.upload(*src, *tgt, cost, C.s);
    const int64_t R = side == 0 ? src->n : tgt->n, Cn = side == 0 ? tgt->n : src->n;
    DevBuf<double> f = dev_from<double>(f_hat, src->n, C.s);
    DevBuf<double> g = dev_from<double>(g_hat, tgt->n, C.s);
    DevBuf<double> Vd = dev_from<double>(V, Cn * p, C.s);
    DevBuf<double> Ad, Bd;
    if (A) {
        Ad = dev_from<double>(A, src->n * r, C.s);
        Bd = dev_from<double>(B, tgt->n * r, C.s);
    }
    DevBuf<double> lse(size_t(R), C.s), mx(size_t(R), C.s), o(size_t(R * p), C.s);
    const double* kpot = side == 0 ? g.get() : f.get();
    const double* pot = side == 0 ? f.get() : g.get();
    FinalizeArgs<double> fa{};
    fa.eps = eps;
    fa.flags = C.flags;
    fa.out_lse = lse.get();
    fa.out_max = mx.get();
    half_step<double>(P, side, kpot, eps, fa);
    if (p > 0)
        transport<double>(P, side, kpot, pot, eps, lse.get(), mx.get(), Vd.get(), p, Ad.get(),
                          Bd.get(), r, o.get(), C.flags);
    dev_to<double>(o, out, R * p, C.s);
    sync_and_check(C, kFlagNonFinitePotential);
    return 0;
}
}  // namespace

int fsk_apply_plan(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                   const double* g_hat, double eps, const fsk_cost* cost, const double* V,
                   int64_t p, const fsk_tiles* tiles, fsk_ledger* ledger, double* out) {
    return guarded([&] {
        common_checks(src, tgt, cost, tiles);
        check_potentials_raw(f_hat, src->n, g_hat, tgt->n, eps);
        if (!all_finite(V, tgt->n * p)) throw ValidationFailure("apply_plan: non-finite V");
        ledger_apply(ledger, src->n, tgt->n, src->d, p, *tiles, cost, false);
        transport_host(src, tgt, f_hat, g_hat, eps, cost, nullptr, nullptr, 0, V, p, 0, out);
    });
}

int fsk_apply_plan_adjoint(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                           const double* g_hat, double eps, const fsk_cost* cost, const double* U,
                           int64_t p, const fsk_tiles* tiles, fsk_ledger* ledger, double* out) {
    return guarded([&] {
        common_checks(src, tgt, cost, tiles);
        check_potentials_raw(f_hat, src->n, g_hat, tgt->n, eps);
        if (!all_finite(U, src->n * p))
            throw ValidationFailure("apply_plan_adjoint: non-finite U");
        ledger_apply(ledger, src->n, tgt->n, src->d, p, *tiles, cost, true);
        transport_host(src, tgt, f_hat, g_hat, eps, cost, nullptr, nullptr, 0, U, p, 1, out);
    });
}

int fsk_apply_hadamard_plan(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                            const double* g_hat, double eps, const fsk_cost* cost,
                            const double* A, const double* B, int64_t r, const double* V,
                            int64_t p, const fsk_tiles* tiles, fsk_ledger* ledger, double* out) {
    return guarded([&] {
        common_checks(src, tgt, cost, tiles);
        check_potentials_raw(f_hat, src->n, g_hat, tgt->n, eps);
        if (r < 1) throw ValidationFailure("apply_hadamard_plan: rank factor r must be >= 1");
        ledger_hadamard(ledger, src->n, tgt->n, src->d, r, p, *tiles, cost);
        transport_host(src, tgt, f_hat, g_hat, eps, cost, A, B, r, V, p, 0, out);
    });
}

int fsk_induced_marginals(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                          const double* g_hat, double eps, const fsk_cost* cost,
                          const fsk_tiles* tiles, fsk_ledger* ledger, double* out_r,
                          double* out_c) {
    return guarded([&] {
        common_checks(src, tgt, cost, tiles);
        check_potentials_raw(f_hat, src->n, g_hat, tgt->n, eps);
        ledger_marginals(ledger, src->n, tgt->n, src->d, *tiles, cost);
        auto& C = exec_ctx();
        DevProblem<double> P;
        P.upload(*src, *tgt, cost, C.s);
        DevBuf<double> f = dev_from<double>(f_hat, src->n, C.s);
        DevBuf<double> g = dev_from<double>(g_hat, tgt->n, C.s);
        HostMarginals hm = marginals_to_host<double>(P, f.get(), g.get(), eps, C);
        sync_and_check(C);
        std::memcpy(out_r, hm.r.data(), sizeof(double) * hm.r.size());
        std::memcpy(out_c, hm.c.data(), sizeof(double) * hm.c.size());
    });
}

namespace {
int half_step_f32_host(const float* sp, const float* sw, int64_t n, const float* tp,
                       const float* tw, int64_t m, int64_t d, const float* pot, float eps,
                       int side, float* out) {
    auto& C = exec_ctx();
    DevProblem<float> P;
    P.upload_f32(sp, sw, n, tp, tw, m, d, C.s);
    if (enable_tensor_path(P, tensor_mode_from_env())) P.tc->set_eps(P, eps);
    const int64_t R = side == 0 ? n : m, Cn = side == 0 ? m : n;
    DevBuf<float> k(size_t(Cn), C.s), o(size_t(R), C.s);
    k.upload(pot, size_t(Cn));
    FinalizeArgs<float> fa{};
    fa.eps = eps;
    fa.out_pot = o.get();
    fa.flags = C.flags;
    half_step<float>(P, side, k.get(), eps, fa);
    o.download(out, size_t(R));
    sync_and_check(C);
    return 0;
}
}  // namespace

int fsk_update_f_hat_f32(const float* src_points, const float* src_weights, int64_t n,
                         const float* tgt_points, const float* tgt_weights, int64_t m, int64_t d,
                         const float* g_hat, float eps, const fsk_tiles* tiles,
                         fsk_ledger* ledger, float* out) {
    return guarded([&] {
        ledger_update_f32(ledger, n, m, d, tiles ? tiles->block_rows : 64,
                          tiles ? tiles->block_cols : 64);
        half_step_f32_host(src_points, src_weights, n, tgt_points, tgt_weights, m, d, g_hat, eps,
                           0, out);
    });
}

int fsk_update_g_hat_f32(const float* src_points, const float* src_weights, int64_t n,
                         const float* tgt_points, const float* tgt_weights, int64_t m, int64_t d,
                         const float* f_hat, float eps, const fsk_tiles* tiles,
                         fsk_ledger* ledger, float* out) {
    return guarded([&] {
        ledger_update_f32(ledger, m, n, d, tiles ? tiles->block_cols : 64,
                          tiles ? tiles->block_rows : 64);
        half_step_f32_host(src_points, src_weights, n, tgt_points, tgt_weights, m, d, f_hat, eps,
                           1, out);
    });
}

uint64_t fsk_io_count_f_update(int64_t n, int64_t m, int64_t d, const fsk_tiles* t) {
    const Counts c = lse_counts(n, m, d, t->block_rows, t->block_cols, false);
    return c.load + c.store;
}
uint64_t fsk_io_count_g_update(int64_t n, int64_t m, int64_t d, const fsk_tiles* t) {
    const Counts c = lse_counts(m, n, d, t->block_cols, t->block_rows, false);
    return c.load + c.store;
}
uint64_t fsk_io_count_symmetric_update(int64_t n, int64_t m, int64_t d, const fsk_tiles* t) {
    return fsk_io_count_f_update(n, m, d, t) + fsk_io_count_g_update(n, m, d, t) + uint64_t(n + m);
}
uint64_t fsk_io_count_apply_plan(int64_t n, int64_t m, int64_t d, int64_t p, const fsk_tiles* t) {
    const Counts c = apply_counts(n, m, d, p, 0, t->block_rows, t->block_cols, false);
    return c.load + c.store;
}
uint64_t fsk_io_count_apply_plan_adjoint(int64_t n, int64_t m, int64_t d, int64_t p,
                                         const fsk_tiles* t) {
    const Counts c = apply_counts(m, n, d, p, 0, t->block_cols, t->block_rows, false);
    return c.load + c.store;
}
uint64_t fsk_io_count_apply_hadamard(int64_t n, int64_t m, int64_t d, int64_t r, int64_t p,
                                     const fsk_tiles* t) {
    const Counts c = apply_counts(n, m, d, p, r, t->block_rows, t->block_cols, false);
    return c.load + c.store;
}
uint64_t fsk_io_count_induced_marginals(int64_t n, int64_t m, int64_t d, const fsk_tiles* t) {
    return fsk_io_count_f_update(n, m, d, t) + 2 * uint64_t(n) + fsk_io_count_g_update(n, m, d, t) +
           2 * uint64_t(m);
}

int fsk_tiles_fit_sram(const fsk_tiles* t, int64_t d, int64_t sram_scalars) {
    const uint64_t need = uint64_t(t->block_cols) * d + uint64_t(t->block_rows) * d +
                          uint64_t(t->block_cols) + 2 * uint64_t(t->block_rows);
    return need <= uint64_t(sram_scalars) ? 1 : 0;
}

void fsk_debug_break_lse(int broken) { break_lse_flag() = broken != 0; }

int fsk_sinkhorn_solve(const fsk_measure* src, const fsk_measure* tgt, const fsk_cost* cost,
                       const fsk_config* cfg, const fsk_tiles* tiles, fsk_ledger* ledger,
                       fsk_report* report) {
    return guarded([&] {
        const bool deferred = checks_deferring_points(src, tgt, cost, tiles, cfg);
        validate_config_raw(*cfg);
        if (cfg->precision == 0) {
            if (labeled_cost(cost))
                throw ValidationFailure(
                    "single-precision solve supports the squared-Euclidean cost only");
            solve_impl<float>(*src, *tgt, cost, *cfg, *tiles, ledger, report, nullptr, nullptr,
                              nullptr, deferred);
        } else {
            solve_impl<double>(*src, *tgt, cost, *cfg, *tiles, ledger, report, nullptr);
        }
    });
}

int fsk_sinkhorn_solve_grad(const fsk_measure* src, const fsk_measure* tgt, const fsk_cost* cost,
                            const fsk_config* cfg, const fsk_tiles* tiles, fsk_ledger* ledger,
                            fsk_report* report, double* out_grad) {
    return guarded([&] {
        PhaseTimer timer(nullptr);
        const bool deferred = checks_deferring_points(src, tgt, cost, tiles, cfg);
        validate_config_raw(*cfg);
        timer.mark("validation");
        if (cfg->precision == 0) {
            if (labeled_cost(cost))
                throw ValidationFailure(
                    "single-precision solve supports the squared-Euclidean cost only");
            solve_impl<float>(*src, *tgt, cost, *cfg, *tiles, ledger, report, out_grad, nullptr,
                              nullptr, deferred);
        } else {
            solve_impl<double>(*src, *tgt, cost, *cfg, *tiles, ledger, report, out_grad);
        }
        timer.mark("solve incl. teardown");
    });
}

int fsk_sinkhorn_solve_warm(const fsk_measure* src, const fsk_measure* tgt, const fsk_cost* cost,
                            const fsk_config* cfg, const fsk_tiles* tiles, fsk_ledger* ledger,
                            const double* f_init, const double* g_init, fsk_report* report,
                            double* out_grad) {
    return guarded([&] {
        common_checks(src, tgt, cost, tiles);
        validate_config_raw(*cfg);
        if (!f_init || !g_init) throw ValidationFailure("warm start needs both potentials");
        check_potentials_raw(f_init, src->n, g_init, tgt->n, cfg->eps);
        if (cfg->precision == 0) {
            if (labeled_cost(cost))
                throw ValidationFailure(
                    "single-precision solve supports the squared-Euclidean cost only");
            solve_impl<float>(*src, *tgt, cost, *cfg, *tiles, ledger, report, out_grad, f_init,
                              g_init);
        } else {
            solve_impl<double>(*src, *tgt, cost, *cfg, *tiles, ledger, report, out_grad, f_init,
                               g_init);
        }
    });
}

int fsk_dual_cost(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                  const double* g_hat, double eps, const fsk_cost* cost, const fsk_tiles* tiles,
                  fsk_ledger* ledger, double* out) {
    return guarded([&] {
        common_checks(src, tgt, cost, tiles);
        check_potentials_raw(f_hat, src->n, g_hat, tgt->n, eps);
        ledger_marginals(ledger, src->n, tgt->n, src->d, *tiles, cost);
        auto& C = exec_ctx();
        DevProblem<double> P;
        P.upload(*src, *tgt, cost, C.s);
        DevBuf<double> f = dev_from<double>(f_hat, src->n, C.s);
        DevBuf<double> g = dev_from<double>(g_hat, tgt->n, C.s);
        HostMarginals hm = marginals_to_host<double>(P, f.get(), g.get(), eps, C);
        sync_and_check(C);
        const double fs = feature_scale(cost);
        *out = dual_value(*src, *tgt, f_hat, g_hat, host_sqnorm(*src, fs).data(),
                          host_sqnorm(*tgt, fs).data(), hm.r, eps);
    });
}

namespace {
double solve_dual(const fsk_measure& a, const fsk_measure& b, const fsk_cost* cost,
                  const fsk_config& cfg, const fsk_tiles& tiles, fsk_ledger* ledger) {
    fsk_report rep{};
    if (cfg.precision == 0) {
        if (labeled_cost(cost))
            throw ValidationFailure(
                "single-precision solve supports the squared-Euclidean cost only");
        solve_impl<float>(a, b, cost, cfg, tiles, ledger, &rep, nullptr);
    } else {
        solve_impl<double>(a, b, cost, cfg, tiles, ledger, &rep, nullptr);
    }
    return rep.dual_cost;
}
}  // namespace

int fsk_sinkhorn_divergence_mixed(const fsk_measure* mu, const fsk_measure* nu,
                                  const fsk_cost* cost_cross, const fsk_cost* cost_mu,
                                  const fsk_cost* cost_nu, const fsk_config* cfg,
                                  const fsk_tiles* tiles, fsk_ledger* ledger, double* out) {
    return guarded([&] {
        common_checks(mu, nu, cost_cross, tiles);
        validate_config_raw(*cfg);
        const double cross = solve_dual(*mu, *nu, cost_cross, *cfg, *tiles, ledger);
        common_checks(mu, mu, cost_mu, tiles);
        const double smu = solve_dual(*mu, *mu, cost_mu, *cfg, *tiles, ledger);
        common_checks(nu, nu, cost_nu, tiles);
        const double snu = solve_dual(*nu, *nu, cost_nu, *cfg, *tiles, ledger);
        *out = cross - 0.5 * smu - 0.5 * snu;
    });
}

int fsk_sinkhorn_divergence_batch(const fsk_measure* mus, const fsk_measure* nus, int64_t pairs,
                                  const fsk_cost* cost, const fsk_config* cfg,
                                  const fsk_tiles* tiles, fsk_ledger* ledger, double* out) {
    return guarded([&] {
        validate_config_raw(*cfg);
        {
            BatchMemoScope memo;   // each distinct cloud is validated once
            for (int64_t k = 0; k < pairs; ++k) common_checks(&mus[k], &nus[k], cost, tiles);
        }
        // pairs are independent: FSK_BATCH_WORKERS host workers, each with its own
        // stream (exec_ctx), upload cache and host memo, can run them concurrently.
        // Default 1: at cfg5 two or three workers measured the same throughput (the
        // busier GPU drops to the power-capped clock)
        static const int workers_env = [] {
            const char* e = std::getenv("FSK_BATCH_WORKERS");
            return e ? std::max(1, std::atoi(e)) : 1;
        }();
        const int W = int(std::min<int64_t>(workers_env, pairs));
        int dev = 0;
        FSKB_CUDA(cudaGetDevice(&dev));
        std::vector<fsk_ledger> led(size_t(W), fsk_ledger{});
        std::vector<std::exception_ptr> err(static_cast<std::size_t>(W));
        auto work = [&](int w) {
            try {
                FSKB_CUDA(cudaSetDevice(dev));
                UploadCacheScope uploads;   // each distinct cloud crosses the host link once
                BatchMemoScope memo;        // (per worker) and is scanned / normed once
                fsk_ledger* L = ledger ? &led[size_t(w)] : nullptr;
                for (int64_t k = w; k < pairs; k += W) {
                    const double cross = solve_dual(mus[k], nus[k], cost, *cfg, *tiles, L);
                    const double smu = solve_dual(mus[k], mus[k], cost, *cfg, *tiles, L);
                    const double snu = solve_dual(nus[k], nus[k], cost, *cfg, *tiles, L);
                    out[k] = cross - 0.5 * smu - 0.5 * snu;
                }
            } catch (...) {
                err[size_t(w)] = std::current_exception();
            }
        };
        if (W <= 1) {
            work(0);
        } else {
            std::vector<std::thread> th;
            for (int w = 0; w < W; ++w) th.emplace_back(work, w);
            for (auto& t : th) t.join();
        }
        for (auto& e : err)
            if (e) std::rethrow_exception(e);
        if (ledger)
            for (const auto& l : led) {
                ledger->slow_to_fast_scalars += l.slow_to_fast_scalars;
                ledger->fast_to_slow_scalars += l.fast_to_slow_scalars;
                ledger->kernel_invocations += l.kernel_invocations;
                ledger->transport_vector_applies += l.transport_vector_applies;
                ledger->transport_matrix_applies += l.transport_matrix_applies;
                ledger->hadamard_applies += l.hadamard_applies;
            }
    });
}

namespace {
// side 0: grad_source / barycentric (rows of X, V = Y); side 1: grad_target (rows of Y, V = X)
int autodiff_host(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                  const double* g_hat, double eps, const fsk_cost* cost, int side, bool grad,
                  double* out) {
    auto& C = exec_ctx();
    DevProblem<double> P;
    P.upload(*src, *tgt, cost, C.s);
    const int64_t R = side == 0 ? src->n : tgt->n, d = src->d;
    DevBuf<double> f = dev_from<double>(f_hat, src->n, C.s);
    DevBuf<double> g = dev_from<double>(g_hat, tgt->n, C.s);
    const double* kpot = side == 0 ? g.get() : f.get();
    const double* pot = side == 0 ? f.get() : g.get();
    DevBuf<double> lse(size_t(R), C.s), mx(size_t(R), C.s), O(size_t(R * d), C.s);
    FinalizeArgs<double> fa{};
    fa.eps = eps;
    fa.flags = C.flags;
    fa.out_lse = lse.get();
    fa.out_max = mx.get();
    half_step<double>(P, side, kpot, eps, fa);
    const double* Q = side == 0 ? P.src.pts.get() : P.tgt.pts.get();
    const double* V = side == 0 ? P.tgt.pts.get() : P.src.pts.get();
    const double* w = side == 0 ? P.src.w.get() : P.tgt.w.get();
    launch_apply<double>(P.params(side, kpot, eps), lse.get(), V, d, nullptr, nullptr, 0, O.get(),
                         C.s);
    if (grad) {
        DevBuf<double> G(size_t(R * d), C.s);
        launch_grad_epilogue<double>(Q, O.get(), w, pot, lse.get(), R, d, eps, G.get(), C.flags,
                                     C.s);
        dev_to<double>(G, out, R * d, C.s);
    } else {
        dev_to<double>(O, out, R * d, C.s);
    }
    sync_and_check(C);
    return 0;
}
}  // namespace

int fsk_grad_source(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                    const double* g_hat, double eps, const fsk_cost* cost, const fsk_tiles* tiles,
                    fsk_ledger* ledger, double* out) {
    return guarded([&] {
        common_checks(src, tgt, cost, tiles);
        check_potentials_raw(f_hat, src->n, g_hat, tgt->n, eps);
        ledger_marginals(ledger, src->n, tgt->n, src->d, *tiles, cost);
        ledger_apply(ledger, src->n, tgt->n, src->d, src->d, *tiles, cost, false);
        autodiff_host(src, tgt, f_hat, g_hat, eps, cost, 0, true, out);
    });
}

int fsk_grad_target(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                    const double* g_hat, double eps, const fsk_cost* cost, const fsk_tiles* tiles,
                    fsk_ledger* ledger, double* out) {
    return guarded([&] {
        common_checks(src, tgt, cost, tiles);
        check_potentials_raw(f_hat, src->n, g_hat, tgt->n, eps);
        ledger_marginals(ledger, src->n, tgt->n, src->d, *tiles, cost);
        ledger_apply(ledger, src->n, tgt->n, src->d, src->d, *tiles, cost, true);
        autodiff_host(src, tgt, f_hat, g_hat, eps, cost, 1, true, out);
    });
}

int fsk_barycentric_projection(const fsk_measure* src, const fsk_measure* tgt,
                               const double* f_hat, const double* g_hat, double eps,
                               const fsk_cost* cost, const fsk_tiles* tiles, fsk_ledger* ledger,
                               double* out) {
    return guarded([&] {
        common_checks(src, tgt, cost, tiles);
        check_potentials_raw(f_hat, src->n, g_hat, tgt->n, eps);
        ledger_marginals(ledger, src->n, tgt->n, src->d, *tiles, cost);
        ledger_apply(ledger, src->n, tgt->n, src->d, src->d, *tiles, cost, false);
        autodiff_host(src, tgt, f_hat, g_hat, eps, cost, 0, false, out);
    });
}

void fsk_rng_normal_fill(uint64_t seed, double* out, int64_t count) {
    rng_normal_fill(seed, out, count);
}

const char* fsk_version(void) { return "fsk_b200 0.1 (sm_100a; tcgen05 split-fp16 + fp64/fp32 CUDA-core)"; }

int fsk_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
    return c;
}

void* fsk_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (guarded([&] { p = host_alloc(bytes); }) != 0) return nullptr;
    return p;
}

int fsk_host_free(void* p) {
    return guarded([&] { host_free(p); });
}

int64_t fsk_device_peak_bytes(int device, int reset) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return -1;
    if (reset) {
        unsigned long long zero = 0;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &zero);
    }
    unsigned long long v = 0;
    if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &v) != cudaSuccess) return -1;
    return int64_t(v);
}

}  // extern "C"
