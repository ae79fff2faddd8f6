// Multi-GPU sinkhorn_solve inside the library: the C ABI and the
// C++ drop-in scale over the devices of one box without a Python driver.
//
//   fsk_set_num_devices(N)   N >= 1: solves shard over devices 0..N-1
//
// One host thread and one non-blocking stream per device; every device holds
// both clouds resident (its own DevProblem, operand images and warm bounds) and
// updates only its shard of rows of f (rows of X) and of g (rows of Y), 256-row
// aligned; the only exchange is an NCCL all-gather of the potential shards after
// each half-step (ncclCommInitAll over the devices: NVLink / NVSwitch). The fp64
// early stop (marginal_tol) reads the lagged violation of the next f-update, whose
// per-device partials are all-reduced in the same NCCL group as that all-gather
// (one launch). The final marginals, the dual and the gradient are computed on
// the shards and assembled on the host. NCCL is loaded with dlopen on first use
// (the process may already hold torch's libnccl.so.2, which is then reused).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/fsk_b200.h"
#include "common.h"
#include "core_kernels.h"
#include "device_ops.h"
#include "hostlib.h"
#include "multi_device.h"
#include "tc_engine.h"

namespace fskb {
extern thread_local std::string g_err;
namespace {

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                               ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*comm_abort)(ncclComm_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (n.h) break;
        }
        if (!n.h) return;
        auto sym = [](const char* s) { return dlsym(n.h, s); };
        n.comm_init_all = reinterpret_cast<decltype(n.comm_init_all)>(sym("ncclCommInitAll"));
        n.all_gather = reinterpret_cast<decltype(n.all_gather)>(sym("ncclAllGather"));
        n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(sym("ncclAllReduce"));
        n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
        n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
        n.comm_abort = reinterpret_cast<decltype(n.comm_abort)>(sym("ncclCommAbort"));
        n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(sym("ncclCommDestroy"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
    });
    if (!n.h || !n.comm_init_all || !n.all_gather || !n.all_reduce || !n.group_start)
        throw CudaFailure("multi-device solve: NCCL (libnccl.so.2) not available");
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw CudaFailure(std::string(what) + ": " +
                          (nccl().error_string ? nccl().error_string(r) : "nccl error"));
}

std::atomic<int> g_num_devices{0};

// communicators and streams of devices 0..N-1, created once per N
struct DeviceGroup {
    int n = 0;
    std::vector<ncclComm_t> comms;
    std::vector<cudaStream_t> streams;
};
std::mutex g_group_mu;
DeviceGroup g_group;

DeviceGroup& device_group(int n) {
    if (g_group.n == n) return g_group;
    for (size_t k = 0; k < g_group.comms.size(); ++k) {
        cudaSetDevice(int(k));
        if (nccl().comm_destroy) nccl().comm_destroy(g_group.comms[k]);
        cudaStreamDestroy(g_group.streams[k]);
    }
    g_group = DeviceGroup();
    std::vector<int> devs(static_cast<size_t>(n));
    for (int k = 0; k < n; ++k) devs[size_t(k)] = k;
    g_group.comms.resize(static_cast<size_t>(n));
    nccl_check(nccl().comm_init_all(g_group.comms.data(), n, devs.data()), "ncclCommInitAll");
    g_group.streams.resize(static_cast<size_t>(n));
    for (int k = 0; k < n; ++k) {
        FSKB_CUDA(cudaSetDevice(k));
        configure_device_pool(k);
        FSKB_CUDA(cudaStreamCreateWithFlags(&g_group.streams[size_t(k)], cudaStreamNonBlocking));
    }
    g_group.n = n;
    return g_group;
}

// 256-aligned contiguous shards (the last one ragged), as sharded.py shard_bounds
std::vector<std::pair<int64_t, int64_t>> shards(int64_t rows, int world) {
    int64_t per = (rows + world - 1) / world;
    per = (per + 255) / 256 * 256;
    std::vector<std::pair<int64_t, int64_t>> b;
    for (int k = 0; k < world; ++k)
        b.push_back({std::min(rows, int64_t(k) * per), std::min(rows, int64_t(k + 1) * per)});
    return b;
}

template <typename T>
constexpr ncclDataType_t nccl_type() {
    return std::is_same_v<T, double> ? ncclFloat64 : ncclFloat32;
}

}  // namespace

int num_devices_setting() { return g_num_devices.load(); }

template <typename T>
bool solve_multi_device(const fsk_measure& src, const fsk_measure& tgt, const fsk_cost* cost,
                        const fsk_config& cfg, const std::vector<double>& schedule,
                        const std::vector<double>& alpha, const std::vector<double>& beta,
                        const double* f_init, const double* g_init, const fsk_tiles& tiles,
                        fsk_ledger* ledger, fsk_report* rep, double* grad_out) {
    constexpr bool kSingle = std::is_same_v<T, float>;
    const int world = num_devices_setting();
    if (world < 1 || cfg.schedule != 0 || schedule.empty()) return false;
    int visible = 0;
    FSKB_CUDA(cudaGetDeviceCount(&visible));
    if (world > visible)
        throw ValidationFailure("fsk_set_num_devices: more devices than are visible");
    std::lock_guard<std::mutex> lock(g_group_mu);
    DeviceGroup& G = device_group(world);
    const int64_t n = src.n, m = tgt.n, d = src.d;
    const auto fb = shards(n, world), gb = shards(m, world);
    const int64_t fper = fb[0].second - fb[0].first, gper = gb[0].second - gb[0].first;
    const bool fused_check = !kSingle && cfg.marginal_tol > 0.0;
    // per-device results, assembled on the host
    std::vector<double> fh(static_cast<size_t>(n)), gh(static_cast<size_t>(m)), r(static_cast<size_t>(n)), c(static_cast<size_t>(m));
    std::atomic<bool> failed{false};
    std::string first_error;
    int first_kind = 0;   // 1 validation, 2 numerical, 3 other
    std::mutex err_mu;
    int iters_done = 0, stop_at = -1;
    double viol_stop = 0.0;
    const int cap_iters = int(schedule.size());

    auto body = [&](int k) {
        FSKB_CUDA(cudaSetDevice(k));
        cudaStream_t s = G.streams[size_t(k)];
        ncclComm_t comm = G.comms[size_t(k)];
        int* flags = nullptr;
        FSKB_CUDA(cudaMalloc(reinterpret_cast<void**>(&flags), 2 * sizeof(int)));
        struct FlagFree {
            int* p;
            ~FlagFree() { cudaFree(p); }
        } ff{flags};
        const int init_flags[2] = {0, INT_MAX};
        FSKB_CUDA(cudaMemcpyAsync(flags, init_flags, sizeof(init_flags), cudaMemcpyHostToDevice, s));
        DevProblem<T> P;
        P.upload(src, tgt, cost, s);
        if constexpr (kSingle) enable_tensor_path(P, tensor_mode_from_env());
        // potentials: world * per long (the all-gather layout), the first n / m real
        DevBuf<T> f(size_t(world) * size_t(fper), s), g(size_t(world) * size_t(gper), s);
        DevBuf<T> f_next, r_dev;
        DevBuf<double> viol(1, s), viol_all(1, s);
        {
            std::vector<T> hf(static_cast<size_t>(n)), hg(static_cast<size_t>(m));
            for (int64_t i = 0; i < n; ++i) hf[size_t(i)] = T(f_init ? f_init[i] : -alpha[size_t(i)]);
            for (int64_t j = 0; j < m; ++j) hg[size_t(j)] = T(g_init ? g_init[j] : -beta[size_t(j)]);
            f.upload(hf.data(), size_t(n));
            g.upload(hg.data(), size_t(m));
            FSKB_CUDA(cudaStreamSynchronize(s));
        }
        if (fused_check) {
            f_next.alloc(size_t(world) * size_t(fper), s);
            r_dev.alloc(size_t(n), s);
        }
        const auto [f0, f1] = fb[size_t(k)];
        const auto [g0, g1] = gb[size_t(k)];
        auto gather = [&](DevBuf<T>& buf, int64_t per, double* vsend, double* vrecv) {
            nccl_check(nccl().group_start(), "ncclGroupStart");
            nccl_check(nccl().all_gather(buf.get() + int64_t(k) * per, buf.get(), size_t(per),
                                         nccl_type<T>(), comm, s),
                       "ncclAllGather");
            if (vsend)
                nccl_check(nccl().all_reduce(vsend, vrecv, 1, ncclFloat64, ncclSum, comm, s),
                           "ncclAllReduce");
            nccl_check(nccl().group_end(), "ncclGroupEnd");
        };
        double cur_eps = -1.0;
        bool pending = false;
        int it = 0;
        for (; it < cap_iters; ++it) {
            if (failed.load()) return;
            const double eps_d = schedule[size_t(it)];
            const T eps = T(eps_d);
            if constexpr (kSingle) {
                if (P.tc && cur_eps != eps_d) P.tc->set_eps(P, eps_d);
            }
            cur_eps = eps_d;
            FinalizeArgs<T> fa{};
            fa.eps = eps;
            fa.flags = flags;
            fa.bad_iter = flags + 1;
            fa.iter = it + 1;
            if (pending) {
                // f_{it+1} with the lagged violation of iterate `it` (partials all-reduced
                // in the same NCCL group as the shard all-gather)
                FinalizeArgs<T> fv = fa;
                fv.out_pot = f_next.get();
                fv.old_pot = f.get();
                fv.w = P.src.w.get();
                fv.out_marg = r_dev.get();
                fv.marg_flag = kFlagNonFiniteRowMarginal;
                fv.viol = viol.get();
                viol.zero();
                half_step_rows<T>(P, 0, g.get(), eps, fv, f0, f1);
                gather(f_next, fper, viol.get(), viol_all.get());
                double hv = 0.0;
                FSKB_CUDA(cudaMemcpyAsync(&hv, viol_all.get(), sizeof(double),
                                          cudaMemcpyDeviceToHost, s));
                FSKB_CUDA(cudaStreamSynchronize(s));
                pending = false;
                if (hv <= cfg.marginal_tol) {
                    // iterate `it` is the answer: its r rows (from this f-update), f, g
                    std::vector<T> rl(static_cast<size_t>(f1 - f0));
                    FSKB_CUDA(cudaMemcpyAsync(rl.data(), r_dev.get() + f0, rl.size() * sizeof(T),
                                              cudaMemcpyDeviceToHost, s));
                    FSKB_CUDA(cudaStreamSynchronize(s));
                    for (int64_t i = f0; i < f1; ++i) r[size_t(i)] = double(rl[size_t(i - f0)]);
                    if (k == 0) {
                        stop_at = it;
                        viol_stop = hv;
                    }
                    break;
                }
                std::swap(f, f_next);
            } else {
                fa.out_pot = f.get();
                half_step_rows<T>(P, 0, g.get(), eps, fa, f0, f1);
                gather(f, fper, nullptr, nullptr);
            }
            fa.out_pot = g.get();
            half_step_rows<T>(P, 1, f.get(), eps, fa, g0, g1);
            gather(g, gper, nullptr, nullptr);
            if (fused_check && eps_d == cfg.eps) pending = true;
        }
        FSKB_CUDA(cudaStreamSynchronize(s));
        {
            int hflags[2];
            FSKB_CUDA(cudaMemcpy(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost));
            if (hflags[0])
                throw_for_flags(hflags[0], hflags[1] != INT_MAX
                                               ? " at iteration " + std::to_string(hflags[1])
                                               : "");
        }
        const bool stopped_here = it < cap_iters;
        if (k == 0) iters_done = stopped_here ? it : cap_iters;
        const double pot_eps = kSingle ? cfg.eps : cur_eps;
        // final potentials (every device holds them whole after the last all-gather)
        if (k == 0) {
            std::vector<T> hf(static_cast<size_t>(n)), hg(static_cast<size_t>(m));
            FSKB_CUDA(cudaMemcpy(hf.data(), f.get(), size_t(n) * sizeof(T), cudaMemcpyDeviceToHost));
            FSKB_CUDA(cudaMemcpy(hg.data(), g.get(), size_t(m) * sizeof(T), cudaMemcpyDeviceToHost));
            for (int64_t i = 0; i < n; ++i) fh[size_t(i)] = double(hf[size_t(i)]);
            for (int64_t j = 0; j < m; ++j) gh[size_t(j)] = double(hg[size_t(j)]);
        }
        if (!stopped_here) {
            if constexpr (kSingle) {
                if (P.tc && cur_eps != pot_eps) P.tc->set_eps(P, pot_eps);
            }
            // induced marginals on the shards (r rows of X, c rows of Y)
            DevBuf<T> rr(size_t(n), s), cc(size_t(m), s);
            FinalizeArgs<T> fr{};
            fr.eps = T(pot_eps);
            fr.flags = flags;
            fr.old_pot = f.get();
            fr.w = P.src.w.get();
            fr.out_marg = rr.get();
            fr.marg_flag = kFlagNonFiniteRowMarginal;
            half_step_rows<T>(P, 0, g.get(), T(pot_eps), fr, f0, f1);
            FinalizeArgs<T> fc{};
            fc.eps = T(pot_eps);
            fc.flags = flags;
            fc.old_pot = g.get();
            fc.w = P.tgt.w.get();
            fc.out_marg = cc.get();
            fc.marg_flag = kFlagNonFiniteColMarginal;
            half_step_rows<T>(P, 1, f.get(), T(pot_eps), fc, g0, g1);
            std::vector<T> rl(static_cast<size_t>(f1 - f0)), cl(static_cast<size_t>(g1 - g0));
            FSKB_CUDA(cudaMemcpyAsync(rl.data(), rr.get() + f0, rl.size() * sizeof(T),
                                      cudaMemcpyDeviceToHost, s));
            FSKB_CUDA(cudaMemcpyAsync(cl.data(), cc.get() + g0, cl.size() * sizeof(T),
                                      cudaMemcpyDeviceToHost, s));
            FSKB_CUDA(cudaStreamSynchronize(s));
            for (int64_t i = f0; i < f1; ++i) r[size_t(i)] = double(rl[size_t(i - f0)]);
            for (int64_t j = g0; j < g1; ++j) c[size_t(j)] = double(cl[size_t(j - g0)]);
        } else {
            // stopped: c = b exactly (g is the g-update of f), r rows came with the check
            for (int64_t j = g0; j < g1; ++j) c[size_t(j)] = tgt.weights[j];
        }
        if (grad_out && f1 > f0) {
            // gradient rows of this shard, straight into out_grad
            const int64_t R = f1 - f0;
            std::vector<double> hgr(static_cast<size_t>(R * d));
            if constexpr (kSingle) {
                if (P.tc) {
                    DevBuf<T> Gd(size_t(R * d), s);
                    P.s = s;
                    P.tc->grad(P, 0, g.get(), f.get(), T(pot_eps), f0, f1, Gd.get(), flags);
                    DevBuf<double> wide(size_t(R * d), s);
                    launch_f32_to_f64(Gd.get(), wide.get(), R * d, s);
                    wide.download(hgr.data(), hgr.size());
                } else {
                    DevBuf<double> G64(size_t(R * d), s);
                    grad_rows_fp64(P, f.get(), g.get(), pot_eps, f0, f1, G64.get(), flags, s);
                    G64.download(hgr.data(), hgr.size());
                }
            } else {
                DevBuf<double> lse(size_t(n), s), mx(size_t(n), s), O(size_t(R * d), s),
                    Gd(size_t(R * d), s);
                FinalizeArgs<double> fl{};
                fl.eps = pot_eps;
                fl.flags = flags;
                fl.out_lse = lse.get();
                fl.out_max = mx.get();
                half_step_rows<double>(P, 0, g.get(), pot_eps, fl, f0, f1);
                ScoreParams<double> sp = P.params(0, g.get(), pot_eps);
                sp.Q += f0 * d;
                sp.R = R;
                launch_apply<double>(sp, lse.get() + f0, P.tgt.pts.get(), d, nullptr, nullptr, 0,
                                     O.get(), s);
                launch_grad_epilogue<double>(P.src.pts.get() + f0 * d, O.get(),
                                             P.src.w.get() + f0, f.get() + f0, lse.get() + f0, R,
                                             d, pot_eps, Gd.get(), flags, s);
                Gd.download(hgr.data(), hgr.size());
            }
            FSKB_CUDA(cudaStreamSynchronize(s));
            std::memcpy(grad_out + f0 * d, hgr.data(), hgr.size() * sizeof(double));
        }
        int hflags[2];
        FSKB_CUDA(cudaMemcpy(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost));
        if (hflags[0] & ~kFlagNonFinitePotential) throw_for_flags(hflags[0]);
        // (teardown after every device is done with its collectives)
        FSKB_CUDA(cudaStreamSynchronize(s));
    };
    std::vector<std::thread> th;
    for (int k = 0; k < world; ++k)
        th.emplace_back([&, k] {
            try {
                body(k);
            } catch (const std::exception& e) {
                std::lock_guard<std::mutex> l(err_mu);
                if (!failed.exchange(true)) {
                    first_error = e.what();
                    first_kind = dynamic_cast<const ValidationFailure*>(&e)   ? 1
                                 : dynamic_cast<const NumericalFailure*>(&e) ? 2
                                                                             : 3;
                    // the other devices may wait in a collective: abort the group
                    if (nccl().comm_abort)
                        for (auto cm : G.comms) nccl().comm_abort(cm);
                    G.n = 0;
                    G.comms.clear();
                }
            }
        });
    for (auto& t : th) t.join();
    if (failed.load()) {
        for (auto st : g_group.streams) cudaStreamDestroy(st);
        g_group = DeviceGroup();
        if (first_kind == 1) throw ValidationFailure(first_error);
        if (first_kind == 2) throw NumericalFailure(first_error);
        throw CudaFailure(first_error);
    }
    // ledger: the reference's closed forms for its own loop (solver.cpp:36-66): two
    // updates per iteration, the tolerance check's marginals for every iterate at the
    // final eps, then final marginals (unless a check stopped the solve) + dual_cost
    bool last_check_passed = false;
    for (int it = 0; it < iters_done; ++it) {
        if (kSingle) {
            ledger_update_f32(ledger, n, m, d, tiles.block_rows, tiles.block_cols);
            ledger_update_f32(ledger, m, n, d, tiles.block_cols, tiles.block_rows);
        } else {
            ledger_update_f(ledger, n, m, d, tiles, cost);
            ledger_update_g(ledger, n, m, d, tiles, cost);
        }
        if (fused_check && schedule[size_t(it)] == cfg.eps)
            ledger_marginals(ledger, n, m, d, tiles, cost);
    }
    const bool stopped = stop_at >= 0;
    double viol = viol_stop;
    if (!stopped) {
        viol = 0.0;
        for (int64_t i = 0; i < n; ++i) viol += std::abs(r[size_t(i)] - src.weights[i]);
        for (int64_t j = 0; j < m; ++j) viol += std::abs(c[size_t(j)] - tgt.weights[j]);
        last_check_passed = fused_check && iters_done > 0 &&
                            schedule[size_t(iters_done - 1)] == cfg.eps && viol <= cfg.marginal_tol;
        if (!last_check_passed) ledger_marginals(ledger, n, m, d, tiles, cost);
    }
    ledger_marginals(ledger, n, m, d, tiles, cost);   // dual_cost's marginals
    const double pot_eps = kSingle ? cfg.eps : schedule[size_t(std::max(0, iters_done - 1))];
    const double mass = cascade_sum(r.data(), r.size());
    double value = 0.0;
    for (int64_t i = 0; i < n; ++i) value += (fh[size_t(i)] + alpha[size_t(i)]) * src.weights[i];
    for (int64_t j = 0; j < m; ++j) value += (gh[size_t(j)] + beta[size_t(j)]) * tgt.weights[j];
    const double dual = value - pot_eps * (mass - 1.0);
    if (rep) {
        rep->iterations = iters_done;
        rep->marginal_violation = viol;
        rep->dual_cost = dual;
        rep->eps = pot_eps;
        if (rep->f_hat) std::memcpy(rep->f_hat, fh.data(), sizeof(double) * size_t(n));
        if (rep->g_hat) std::memcpy(rep->g_hat, gh.data(), sizeof(double) * size_t(m));
        if (rep->eps_history)
            for (int64_t q = 0; q < rep->eps_history_cap && q < iters_done; ++q)
                rep->eps_history[q] = schedule[size_t(q)];
    }
    if (grad_out) {
        ledger_marginals(ledger, n, m, d, tiles, cost);
        ledger_apply(ledger, n, m, d, d, tiles, cost, false);
    }
    return true;
}

template bool solve_multi_device<float>(const fsk_measure&, const fsk_measure&, const fsk_cost*,
                                        const fsk_config&, const std::vector<double>&,
                                        const std::vector<double>&, const std::vector<double>&,
                                        const double*, const double*, const fsk_tiles&,
                                        fsk_ledger*, fsk_report*, double*);
template bool solve_multi_device<double>(const fsk_measure&, const fsk_measure&, const fsk_cost*,
                                         const fsk_config&, const std::vector<double>&,
                                         const std::vector<double>&, const std::vector<double>&,
                                         const double*, const double*, const fsk_tiles&,
                                         fsk_ledger*, fsk_report*, double*);

}  // namespace fskb

extern "C" int fsk_set_num_devices(int n) {
    if (n < 0) {
        fskb::g_err = "fsk_set_num_devices: n must be >= 0";
        return FSK_EVALIDATION;
    }
    fskb::g_num_devices.store(n);
    return FSK_OK;
}

extern "C" int fsk_num_devices(void) { return fskb::num_devices_setting(); }
