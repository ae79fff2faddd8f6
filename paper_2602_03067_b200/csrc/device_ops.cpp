#include <memory>
#include <utility>
#include <vector>
#include <atomic>
#include "device_ops.h"

#include <climits>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "tc_engine.h"

namespace fskb {

std::atomic<int64_t>& launch_counter() {
    static std::atomic<int64_t> c{0};
    return c;
}

bool& break_lse_flag() {
    static bool b = false;
    return b;
}

int num_sms() {
    static int n = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

// Every DevBuf is a stream-ordered allocation from the device's default pool. Its
// default release threshold (0) hands freed memory back to the driver at every
// synchronization, so the next pass re-maps its partial buffers (and a solve its
// operand images): keep what the pool holds instead. Once per device.
void configure_device_pool(int device) {
    static std::atomic<uint64_t> done_mask{0};
    if (device < 0 || device >= 64 || (done_mask.load() >> device) & 1u) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = ~uint64_t(0);
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        // Map a block into the pool up front (one allocation, freed at once and kept):
        // later requests are carved from resident memory. Without it, the per-call
        // buffers of the C ABI solves (hundreds of MB each at cfg3) fragment the pool
        // and some calls grow it: measured 0.15-2 s stalls in 4 of 10 cfg3 calls,
        // none with the reserve (gpurun_out/e2eab3). FSK_POOL_RESERVE_GB overrides
        // the default of 24 GB on devices of >= 100 GB (0 disables).
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        const char* e = std::getenv("FSK_POOL_RESERVE_GB");
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) cudaGetLastError();
        const double gb = e ? std::atof(e) : (total_b >= (size_t(100) << 30) ? 24.0 : 0.0);
        if (gb > 0.0 && double(free_b) > 2.0 * gb * double(1ull << 30)) {
            void* p = nullptr;
            if (cudaMallocAsync(&p, size_t(gb * double(1ull << 30)), cudaStreamPerThread) ==
                cudaSuccess) {
                cudaFreeAsync(p, cudaStreamPerThread);
                cudaStreamSynchronize(cudaStreamPerThread);
            } else {
                cudaGetLastError();
            }
        }
        cudaSetDevice(prev);
    }
    done_mask.fetch_or(uint64_t(1) << device);
}

ExecCtx& exec_ctx() {
    thread_local ExecCtx c;
    if (!c.s) {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
            throw CudaFailure("no CUDA device available (the B200 engine has no CPU fallback)");
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) configure_device_pool(dev);
        FSKB_CUDA(cudaStreamCreateWithFlags(&c.s, cudaStreamNonBlocking));
        FSKB_CUDA(cudaMalloc(reinterpret_cast<void**>(&c.flags), 2 * sizeof(int)));
        c.bad_iter = c.flags + 1;
        int init[2] = {0, INT_MAX};
        FSKB_CUDA(cudaMemcpy(c.flags, init, sizeof(init), cudaMemcpyHostToDevice));
    }
    return c;
}

int read_and_clear_flags(ExecCtx& c) {
    int h[2];
    FSKB_CUDA(cudaMemcpyAsync(h, c.flags, sizeof(h), cudaMemcpyDeviceToHost, c.s));
    FSKB_CUDA(cudaStreamSynchronize(c.s));
    if (h[0] != 0 || h[1] != INT_MAX) {
        int init[2] = {0, INT_MAX};
        FSKB_CUDA(cudaMemcpyAsync(c.flags, init, sizeof(init), cudaMemcpyHostToDevice, c.s));
        FSKB_CUDA(cudaStreamSynchronize(c.s));
    }
    return h[0];
}

void throw_for_flags(int flags, const std::string& suffix) {
    if (!flags) return;
    if (flags & kFlagNonFinitePotential)
        throw NumericalFailure("non-finite potential produced by streaming LSE update" + suffix);
    if (flags & kFlagTransportOverflow)
        throw NumericalFailure("overflow in transport application, potentials are not stabilized" +
                               suffix);
    if (flags & kFlagNonFiniteTransport)
        throw NumericalFailure("non-finite entry in transport application output" + suffix);
    if (flags & kFlagNonFiniteRowMarginal)
        throw NumericalFailure("non-finite induced row marginal" + suffix);
    if (flags & kFlagNonFiniteColMarginal)
        throw NumericalFailure("non-finite induced column marginal" + suffix);
}

namespace {

// Batch-scoped cache of uploaded measures, keyed by the caller's host buffers
// (read-only for the duration of the call): a batch of solves over a few
// distinct clouds ships each cloud over the host link once; later uses are
// device-to-device copies.
struct UploadKey {
    const double* pts;
    const double* w;
    const int32_t* lab;
    int64_t n, d;
    bool labels;
    bool operator==(const UploadKey& o) const {
        return pts == o.pts && w == o.w && lab == o.lab && n == o.n && d == o.d &&
               labels == o.labels;
    }
};
template <typename T>
using UploadCacheT = std::vector<std::pair<UploadKey, std::unique_ptr<DevSide<T>>>>;
struct UploadCache {
    UploadCacheT<float> f;
    UploadCacheT<double> d;
    template <typename T>
    UploadCacheT<T>& get() {
        if constexpr (std::is_same_v<T, float>) return f;
        else return d;
    }
};
thread_local UploadCache* t_upload_cache = nullptr;

template <typename T>
void copy_side(DevSide<T>& dst, const DevSide<T>& src, cudaStream_t s) {
    dst.n = src.n;
    dst.d = src.d;
    auto cp = [&](auto& to, const auto& from) {
        using E = std::remove_pointer_t<decltype(from.get())>;
        if (!from.get()) return;
        to.alloc(from.size(), s);
        FSKB_CUDA(cudaMemcpyAsync(to.get(), from.get(), from.size() * sizeof(E),
                                  cudaMemcpyDeviceToDevice, s));
    };
    cp(dst.pts, src.pts);
    cp(dst.w, src.w);
    cp(dst.logw, src.logw);
    cp(dst.lab, src.lab);
}

template <typename T>
void upload_side_host(DevSide<T>& side, const fsk_measure& m, bool want_labels, cudaStream_t s);

template <typename T>
void upload_side(DevSide<T>& side, const fsk_measure& m, bool want_labels, cudaStream_t s) {
    if (!t_upload_cache) return upload_side_host(side, m, want_labels, s);
    const UploadKey key{m.points, m.weights, m.labels, m.n, m.d, want_labels && m.labels};
    auto& cache = t_upload_cache->get<T>();
    for (auto& [k, v] : cache)
        if (k == key) return copy_side(side, *v, s);
    upload_side_host(side, m, want_labels, s);
    auto keep = std::make_unique<DevSide<T>>();
    copy_side(*keep, side, s);
    cache.emplace_back(key, std::move(keep));
}

template <typename T>
void upload_side_host(DevSide<T>& side, const fsk_measure& m, bool want_labels, cudaStream_t s) {
    side.n = m.n;
    side.d = m.d;
    side.pts.alloc(size_t(m.n * m.d), s);
    side.w.alloc(size_t(m.n), s);
    side.logw.alloc(size_t(m.n), s);
    if constexpr (std::is_same_v<T, double>) {
        side.pts.upload(m.points, size_t(m.n * m.d));
        side.w.upload(m.weights, size_t(m.n));
    } else {
        // ship the caller's doubles as they are and narrow on the device (no host
        // conversion pass over n x d values)
        DevBuf<double> tmp(size_t(m.n * m.d), s), wtmp(size_t(m.n), s);
        tmp.upload(m.points, size_t(m.n * m.d));
        wtmp.upload(m.weights, size_t(m.n));
        launch_f64_to_f32(tmp.get(), side.pts.get(), m.n * m.d, s);
        launch_f64_to_f32(wtmp.get(), side.w.get(), m.n, s);
        FSKB_CUDA(cudaStreamSynchronize(s));
    }
    launch_log<T>(side.w.get(), side.logw.get(), m.n, s);
    if (want_labels && m.labels) {
        side.lab.alloc(size_t(m.n), s);
        side.lab.upload(m.labels, size_t(m.n));
    }
}

}  // namespace

UploadCacheScope::UploadCacheScope() : prev_(t_upload_cache) { t_upload_cache = new UploadCache; }
UploadCacheScope::~UploadCacheScope() {
    delete t_upload_cache;
    t_upload_cache = static_cast<UploadCache*>(prev_);
}

template <typename T>
void DevProblem<T>::upload(const fsk_measure& a, const fsk_measure& b, const fsk_cost* cost,
                           cudaStream_t stream) {
    s = stream;
    labeled = cost && cost->kind == 1;
    fscale = labeled ? cost->lambda1 : 1.0;
    lambda2 = labeled ? cost->lambda2 : 0.0;
    upload_side(src, a, labeled, s);
    upload_side(tgt, b, labeled, s);
    if (labeled) {
        wdim = cost->num_labels;
        wtab.alloc(size_t(wdim * wdim), s);
        wtab.upload(cost->label_cost, size_t(wdim * wdim));
    }
    FSKB_CUDA(cudaStreamSynchronize(s));
}

template <typename T>
bool DevProblem<T>::ingest(const fsk_measure& a, const fsk_measure& b, double scale,
                           cudaStream_t stream, DevBuf<double>& alpha, DevBuf<double>& beta,
                           T* f0, T* g0) {
    if constexpr (!std::is_same_v<T, float>) {
        throw CudaFailure("ingest on a double problem");
    } else {
        s = stream;
        labeled = false;
        fscale = 1.0;
        lambda2 = 0.0;
        DevBuf<int> bad(1, s);
        bad.zero();
        auto side_in = [&](DevSide<T>& side, const fsk_measure& m, DevBuf<double>& sq, T* p0) {
            side.n = m.n;
            side.d = m.d;
            side.pts.alloc(size_t(m.n * m.d), s);
            side.w.alloc(size_t(m.n), s);
            side.logw.alloc(size_t(m.n), s);
            sq.alloc(size_t(m.n), s);
            DevBuf<double> tmp(size_t(m.n * m.d), s), wtmp(size_t(m.n), s);
            tmp.upload(m.points, size_t(m.n * m.d));
            wtmp.upload(m.weights, size_t(m.n));
            launch_ingest_f32(tmp.get(), m.n, m.d, scale, side.pts.get(), sq.get(), p0, bad.get(),
                              s);
            launch_f64_to_f32(wtmp.get(), side.w.get(), m.n, s);
            launch_log<T>(side.w.get(), side.logw.get(), m.n, s);
        };
        side_in(src, a, alpha, f0);
        side_in(tgt, b, beta, g0);
        int h = 0;
        FSKB_CUDA(cudaMemcpyAsync(&h, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
        FSKB_CUDA(cudaStreamSynchronize(s));
        return h == 0;
    }
}

template <typename T>
void DevProblem<T>::upload_f32(const float* xa, const float* wa, int64_t n, const float* xb,
                               const float* wb, int64_t m, int64_t d, cudaStream_t stream) {
    if constexpr (!std::is_same_v<T, float>) throw CudaFailure("upload_f32 on a double problem");
    else {
    s = stream;
    labeled = false;
    fscale = 1.0;
    src.n = n;
    src.d = d;
    tgt.n = m;
    tgt.d = d;
    src.pts.alloc(size_t(n * d), s);
    src.pts.upload(xa, size_t(n * d));
    tgt.pts.alloc(size_t(m * d), s);
    tgt.pts.upload(xb, size_t(m * d));
    src.w.alloc(size_t(n), s);
    src.w.upload(wa, size_t(n));
    tgt.w.alloc(size_t(m), s);
    tgt.w.upload(wb, size_t(m));
    src.logw.alloc(size_t(n), s);
    tgt.logw.alloc(size_t(m), s);
    launch_log<T>(src.w.get(), src.logw.get(), n, s);
    launch_log<T>(tgt.w.get(), tgt.logw.get(), m, s);
    }
}

template <typename T>
ScoreParams<T> DevProblem<T>::params(int side, const T* kpot, T eps) const {
    ScoreParams<T> p{};
    const DevSide<T>& q = side == 0 ? src : tgt;
    const DevSide<T>& k = side == 0 ? tgt : src;
    p.Q = q.pts.get();
    p.K = k.pts.get();
    p.R = q.n;
    p.C = k.n;
    p.d = q.d;
    p.kscale = T(2.0 * fscale / double(eps));
    if constexpr (std::is_same_v<T, float>) p.kscale = 2.0f * float(fscale) / eps;
    p.kpot = kpot;
    p.klogw = k.logw.get();
    p.eps = eps;
    if (labeled) {
        p.qlab = q.lab.get();
        p.klab = k.lab.get();
        p.wtab = wtab.get();
        p.wdim = wdim;
        p.lam2_eps = T(lambda2 / double(eps));
    }
    return p;
}

template <typename T>
void half_step(DevProblem<T>& P, int side, const T* kpot, T eps, const FinalizeArgs<T>& fa) {
    if constexpr (std::is_same_v<T, float>) {
        if (P.tc) {
            P.tc->run(P, side, kpot, eps, fa, 0, P.rows(side));
            return;
        }
    }
    const ScoreParams<T> sp = P.params(side, kpot, eps);
    const int splits = lse_splits(sp.R, sp.C);
    DevBuf<T> pm(size_t(splits) * size_t(sp.R), P.s), ps(size_t(splits) * size_t(sp.R), P.s);
    launch_lse<T>(sp, splits, pm.get(), ps.get(), P.s);
    launch_lse_finalize<T>(pm.get(), ps.get(), splits, sp.R, fa, P.s);
}

template <typename T>
void half_step_rows(DevProblem<T>& P, int side, const T* kpot, T eps, const FinalizeArgs<T>& fa,
                    int64_t row_begin, int64_t row_end) {
    if (row_end <= row_begin) return;
    if constexpr (std::is_same_v<T, float>) {
        if (P.tc) {
            P.tc->run(P, side, kpot, eps, fa, row_begin, row_end);
            return;
        }
    }
    ScoreParams<T> sp = P.params(side, kpot, eps);
    sp.Q += row_begin * sp.d;
    sp.R = row_end - row_begin;
    if (sp.qlab) sp.qlab += row_begin;
    FinalizeArgs<T> f = fa;
    auto off = [&](auto* p) { return p ? p + row_begin : p; };
    f.out_pot = off(f.out_pot);
    f.sym_old = off(f.sym_old);
    f.out_lse = off(f.out_lse);
    f.out_max = off(f.out_max);
    f.old_pot = off(f.old_pot);
    f.w = off(f.w);
    f.out_marg = off(f.out_marg);
    const int splits = lse_splits(sp.R, sp.C);
    DevBuf<T> pm(size_t(splits) * size_t(sp.R), P.s), ps(size_t(splits) * size_t(sp.R), P.s);
    launch_lse<T>(sp, splits, pm.get(), ps.get(), P.s);
    launch_lse_finalize<T>(pm.get(), ps.get(), splits, sp.R, f, P.s);
}

template <typename T>
void transport(DevProblem<T>& P, int side, const T* kpot, const T* pot, T eps, const T* lse,
               const T* mx, const T* V, int64_t p, const T* A, const T* B, int64_t r, T* out,
               int* flags) {
    const ScoreParams<T> sp = P.params(side, kpot, eps);
    DevBuf<T> O(size_t(sp.R) * size_t(p), P.s);
    launch_apply<T>(sp, lse, V, p, A, B, r, O.get(), P.s);
    const T* w = side == 0 ? P.src.w.get() : P.tgt.w.get();
    launch_apply_finalize<T>(O.get(), sp.R, p, w, pot, lse, mx, eps, out, flags, P.s);
}

template struct DevProblem<float>;
template struct DevProblem<double>;
void grad_rows_fp64(const DevProblem<float>& P, const float* f, const float* g, double eps,
                    int64_t row_begin, int64_t row_end, double* out_dev, int* flags,
                    cudaStream_t s) {
    const int64_t n = P.src.n, m = P.tgt.n, d = P.src.d, R = row_end - row_begin;
    if (R <= 0) return;
    static const bool fused = [] {
        const char* e = std::getenv("FSK_GRAD_FUSED");
        return !(e && e[0] == '0');
    }();
    if (fused && !P.labeled &&
        launch_grad_small_fp64(P.src.pts.get(), P.src.w.get(), f, P.tgt.pts.get(), P.tgt.w.get(),
                               g, row_begin, R, m, int(d), eps, 2.0 * P.fscale / eps, out_dev,
                               flags, s))
        return;
    DevProblem<double> Pd;
    Pd.s = s;
    Pd.fscale = P.fscale;
    auto widen = [&](DevSide<double>& o, const DevSide<float>& i) {
        o.n = i.n;
        o.d = i.d;
        o.pts.alloc(size_t(i.n * i.d), s);
        o.w.alloc(size_t(i.n), s);
        o.logw.alloc(size_t(i.n), s);
        launch_f32_to_f64(i.pts.get(), o.pts.get(), i.n * i.d, s);
        launch_f32_to_f64(i.w.get(), o.w.get(), i.n, s);
        launch_log<double>(o.w.get(), o.logw.get(), i.n, s);
    };
    widen(Pd.src, P.src);
    widen(Pd.tgt, P.tgt);
    if (P.labeled) {
        // label-augmented cost: labels and the V x V table as they are
        Pd.labeled = true;
        Pd.lambda2 = P.lambda2;
        Pd.wdim = P.wdim;
        Pd.wtab.alloc(size_t(P.wdim * P.wdim), s);
        FSKB_CUDA(cudaMemcpyAsync(Pd.wtab.get(), P.wtab.get(),
                                  size_t(P.wdim * P.wdim) * sizeof(double),
                                  cudaMemcpyDeviceToDevice, s));
        for (auto [o, i] : {std::pair{&Pd.src, &P.src}, std::pair{&Pd.tgt, &P.tgt}}) {
            o->lab.alloc(size_t(i->n), s);
            FSKB_CUDA(cudaMemcpyAsync(o->lab.get(), i->lab.get(), size_t(i->n) * sizeof(int32_t),
                                      cudaMemcpyDeviceToDevice, s));
        }
    }
    DevBuf<double> fd(size_t(n), s), gd(size_t(m), s), lse(size_t(n), s), mx(size_t(n), s);
    launch_f32_to_f64(f, fd.get(), n, s);
    launch_f32_to_f64(g, gd.get(), m, s);
    FinalizeArgs<double> fa{};
    fa.eps = eps;
    fa.flags = flags;
    fa.out_lse = lse.get();
    fa.out_max = mx.get();
    half_step_rows<double>(Pd, 0, gd.get(), eps, fa, row_begin, row_end);
    ScoreParams<double> sp = Pd.params(0, gd.get(), eps);
    sp.Q += row_begin * d;
    sp.R = R;
    DevBuf<double> O(size_t(R * d), s);
    launch_apply<double>(sp, lse.get() + row_begin, Pd.tgt.pts.get(), d, nullptr, nullptr, 0,
                         O.get(), s);
    launch_grad_epilogue<double>(Pd.src.pts.get() + row_begin * d, O.get(),
                                 Pd.src.w.get() + row_begin, fd.get() + row_begin,
                                 lse.get() + row_begin, R, d, eps, out_dev, flags, s);
}

template void half_step<float>(DevProblem<float>&, int, const float*, float,
                               const FinalizeArgs<float>&);
template void half_step<double>(DevProblem<double>&, int, const double*, double,
                                const FinalizeArgs<double>&);
template void half_step_rows<float>(DevProblem<float>&, int, const float*, float,
                                    const FinalizeArgs<float>&, int64_t, int64_t);
template void half_step_rows<double>(DevProblem<double>&, int, const double*, double,
                                     const FinalizeArgs<double>&, int64_t, int64_t);
template void transport<float>(DevProblem<float>&, int, const float*, const float*, float,
                               const float*, const float*, const float*, int64_t, const float*,
                               const float*, int64_t, float*, int*);
template void transport<double>(DevProblem<double>&, int, const double*, const double*, double,
                                const double*, const double*, const double*, int64_t,
                                const double*, const double*, int64_t, double*, int*);

}  // namespace fskb
