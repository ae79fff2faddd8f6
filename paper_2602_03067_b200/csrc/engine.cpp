// Device engine (fsk_engine_*): one problem resident in HBM, potentials in
// caller-owned device buffers, half-steps over row ranges. This is the unit a
// multi-GPU driver shards: rank k updates rows [k n/N, (k+1) n/N) of f, the
// collective library all-gathers the length-n vector in place, then the same
// for g. No collective lives in here.
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/fsk_b200.h"
#include "common.h"
#include "core_kernels.h"
#include "device_ops.h"
#include "hostlib.h"
#include "small_solve.h"
#include "tc_engine.h"

namespace fskb {
extern thread_local std::string g_err;
}

using namespace fskb;

struct fsk_engine {
    // CUDA graph of `iterate` (CUDA-core path only): the whole f/g loop as one launch
    cudaGraphExec_t graph = nullptr;
    int graph_iters = 0;
    cudaStream_t graph_stream = nullptr;
    const float* graph_f = nullptr;
    const float* graph_g = nullptr;
    double graph_eps = 0.0;
    int device = 0;
    DevProblem<float> P;
    float* f = nullptr;
    float* g = nullptr;
    double eps = 0.0;
    cudaStream_t own = nullptr;
    int* flags = nullptr;
    int64_t launches_at_create = 0;
    // stream fence: the engine's persistent buffers are used (and regrown) on
    // whatever stream each call passes; a call on a new stream first waits for
    // the last call's work
    cudaEvent_t fence = nullptr;
    cudaStream_t last = nullptr;
    bool fenced = false;
    DevBuf<float> eps_sched;   // persistent small-problem loop: eps per iteration
    double eps_sched_val = 0.0;
    // fixed-potential transport state over row shards (fsk_engine_transport_prepare):
    // the HVP workspace of SPEC.md:442-446, per orientation
    struct Prep {
        bool valid = false;
        const float* f = nullptr;
        const float* g = nullptr;
        double eps = 0.0;
        int64_t rb[2] = {0, 0}, re[2] = {0, 0};
        DevBuf<float> marg[2], lse[2], mx[2], l2h[2], l2l[2];
    } prep;
};

namespace {

template <typename F>
int eguard(F&& f) {
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

// The stream argument is a plain cudaStream_t: NULL is the legacy default
// stream (CUDA convention), so work is ordered with whatever the caller - e.g.
// torch and its NCCL collectives - runs on that stream. The engine's private
// stream is only used by create/set_eps, which synchronize before returning.
cudaStream_t pick(fsk_engine* e, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (e->fenced && s != e->last) FSKB_CUDA(cudaStreamWaitEvent(s, e->fence, 0));
    return s;
}

// records the fence after a call's work on `s` (RAII at the top of each call)
struct Fence {
    fsk_engine* e;
    cudaStream_t s;
    ~Fence() {
        if (cudaEventRecord(e->fence, s) == cudaSuccess) {
            e->last = s;
            e->fenced = true;
        }
    }
};

void drop_graph(fsk_engine* e) {
    if (e->graph) cudaGraphExecDestroy(e->graph);
    e->graph = nullptr;
}

}  // namespace

extern "C" {

int fsk_engine_create(int device, const double* X, const double* a, int64_t n, const double* Y,
                      const double* b, int64_t m, int64_t d, int mode, fsk_engine** out) {
    return eguard([&] {
        fsk_measure src{X, a, nullptr, n, d}, tgt{Y, b, nullptr, m, d};
        validate_problem_raw(src, tgt, nullptr);
        FSKB_CUDA(cudaSetDevice(device));
        configure_device_pool(device);
        auto* e = new fsk_engine();
        e->device = device;
        FSKB_CUDA(cudaStreamCreateWithFlags(&e->own, cudaStreamNonBlocking));
        FSKB_CUDA(cudaEventCreateWithFlags(&e->fence, cudaEventDisableTiming));
        FSKB_CUDA(cudaMalloc(reinterpret_cast<void**>(&e->flags), 2 * sizeof(int)));
        FSKB_CUDA(cudaMemset(e->flags, 0, 2 * sizeof(int)));
        e->P.upload(src, tgt, nullptr, e->own);
        enable_tensor_path(e->P, mode);
        FSKB_CUDA(cudaStreamSynchronize(e->own));
        *out = e;
    });
}

int fsk_engine_create_labeled(int device, const double* X, const double* a, const int32_t* la,
                              int64_t n, const double* Y, const double* b, const int32_t* lb,
                              int64_t m, int64_t d, double lambda1, double lambda2,
                              const double* label_cost, int64_t num_labels, int mode,
                              fsk_engine** out) {
    return eguard([&] {
        fsk_measure src{X, a, la, n, d}, tgt{Y, b, lb, m, d};
        fsk_cost cost{1, lambda1, lambda2, label_cost, num_labels};
        validate_problem_raw(src, tgt, &cost);
        FSKB_CUDA(cudaSetDevice(device));
        configure_device_pool(device);
        auto* e = new fsk_engine();
        e->device = device;
        FSKB_CUDA(cudaStreamCreateWithFlags(&e->own, cudaStreamNonBlocking));
        FSKB_CUDA(cudaEventCreateWithFlags(&e->fence, cudaEventDisableTiming));
        FSKB_CUDA(cudaMalloc(reinterpret_cast<void**>(&e->flags), 2 * sizeof(int)));
        FSKB_CUDA(cudaMemset(e->flags, 0, 2 * sizeof(int)));
        e->P.upload(src, tgt, &cost, e->own);
        enable_tensor_path(e->P, mode);
        FSKB_CUDA(cudaStreamSynchronize(e->own));
        *out = e;
    });
}

void fsk_engine_destroy(fsk_engine* e) {
    if (!e) return;
    cudaSetDevice(e->device);
    if (e->graph) cudaGraphExecDestroy(e->graph);
    // the buffers may sit on caller streams that are gone by now: drain the device,
    // then free on the legacy stream
    cudaDeviceSynchronize();
    {
        DevBufTeardown td;
        e->P.tc.reset();
        e->P = DevProblem<float>();   // clouds, labels, label table (on e->own)
        e->eps_sched.release();
        e->prep = fsk_engine::Prep();
    }
    cudaDeviceSynchronize();
    cudaFree(e->flags);
    cudaEventDestroy(e->fence);
    cudaStreamDestroy(e->own);
    delete e;
}

int fsk_engine_set_eps(fsk_engine* e, double eps) {
    return eguard([&] {
        if (!(eps > 0.0)) throw ValidationFailure("eps must be positive");
        // the captured iterate graph bakes eps (2/eps key scale, finalize eps) into
        // its launches: a new eps needs a new capture
        if (eps != e->eps) drop_graph(e);
        e->eps = eps;
        e->P.s = pick(e, e->own);
        Fence fence_{e, e->own};
        if (e->P.tc) e->P.tc->set_eps(e->P, eps);
        FSKB_CUDA(cudaStreamSynchronize(e->own));
    });
}

int fsk_engine_bind_potentials(fsk_engine* e, float* f_dev, float* g_dev) {
    if (f_dev != e->f || g_dev != e->g) drop_graph(e);
    e->f = f_dev;
    e->g = g_dev;
    return FSK_OK;
}

int fsk_engine_init_potentials(fsk_engine* e, void* stream) {
    return eguard([&] {
        cudaStream_t s = pick(e, stream);
        Fence fence_{e, s};
        // f_hat = -s |x|^2, g_hat = -s |y|^2 (solver.cpp:27-32; s = lambda1 for labels)
        const float fs = float(e->P.fscale);
        launch_neg_sqnorm<float>(e->P.src.pts.get(), e->P.src.n, e->P.src.d, fs, e->f, s);
        launch_neg_sqnorm<float>(e->P.tgt.pts.get(), e->P.tgt.n, e->P.tgt.d, fs, e->g, s);
        // a new solve: the skip decisions start from scratch (same bits as a fresh engine)
        if (e->P.tc) e->P.tc->reset_history(s);
    });
}

int fsk_engine_half_step(fsk_engine* e, int side, int64_t row_begin, int64_t row_end,
                         double* viol_accum, void* stream) {
    return eguard([&] {
        if (!e->f || !e->g) throw ValidationFailure("engine potentials not bound");
        if (!(e->eps > 0.0)) throw ValidationFailure("engine eps not set");
        const int64_t R = side == 0 ? e->P.src.n : e->P.tgt.n;
        if (row_begin < 0 || row_end > R || row_begin > row_end)
            throw ValidationFailure("engine row range out of bounds");
        e->P.s = pick(e, stream);
        Fence fence_{e, e->P.s};
        const float eps = float(e->eps);
        float* pot = side == 0 ? e->f : e->g;
        const float* kpot = side == 0 ? e->g : e->f;
        FinalizeArgs<float> fa{};
        fa.eps = eps;
        fa.flags = e->flags;
        fa.out_pot = pot;
        if (viol_accum) {
            fa.old_pot = pot;
            fa.w = side == 0 ? e->P.src.w.get() : e->P.tgt.w.get();
            fa.viol = viol_accum;
            fa.marg_flag = side == 0 ? kFlagNonFiniteRowMarginal : kFlagNonFiniteColMarginal;
        }
        half_step_rows<float>(e->P, side, kpot, eps, fa, row_begin, row_end);
    });
}

int fsk_engine_iterate(fsk_engine* e, int iters, void* stream) {
    return eguard([&] {
        if (!e->f || !e->g) throw ValidationFailure("engine potentials not bound");
        if (!(e->eps > 0.0)) throw ValidationFailure("engine eps not set");
        if (iters < 1) throw ValidationFailure("iters must be positive");
        cudaStream_t s = pick(e, stream);
        Fence fence_{e, s};
        e->P.s = s;
        const float eps = float(e->eps);
        auto body = [&] {
            for (int k = 0; k < iters; ++k) {
                FinalizeArgs<float> fa{};
                fa.eps = eps;
                fa.flags = e->flags;
                fa.out_pot = e->f;
                half_step_rows<float>(e->P, 0, e->g, eps, fa, 0, e->P.src.n);
                fa.out_pot = e->g;
                half_step_rows<float>(e->P, 1, e->f, eps, fa, 0, e->P.tgt.n);
            }
        };
        // small CUDA-core problems (keys fit in shared memory, d <= 16): the whole
        // loop is one persistent cooperative kernel (small_solve.cu)
        const char* penv = std::getenv("FSK_PERSIST");
        if (!e->P.tc && !e->P.labeled && !(penv && penv[0] == '0') &&
            small_solve_fits(e->P.src.n, e->P.tgt.n, e->P.src.d)) {
            if (e->eps_sched.size() < size_t(iters) || e->eps_sched_val != e->eps) {
                const std::vector<float> h(size_t(iters), float(e->eps));
                e->eps_sched.alloc(size_t(iters), s);
                FSKB_CUDA(cudaMemcpyAsync(e->eps_sched.get(), h.data(), h.size() * sizeof(float),
                                          cudaMemcpyHostToDevice, s));
                FSKB_CUDA(cudaStreamSynchronize(s));
                e->eps_sched_val = e->eps;
            }
            SmallSolveParams sp{};
            sp.X = e->P.src.pts.get();
            sp.Y = e->P.tgt.pts.get();
            sp.logw_x = e->P.src.logw.get();
            sp.logw_y = e->P.tgt.logw.get();
            sp.f = e->f;
            sp.g = e->g;
            sp.eps_sched = e->eps_sched.get();
            sp.iters = iters;
            sp.n = e->P.src.n;
            sp.m = e->P.tgt.n;
            sp.d = int(e->P.src.d);
            sp.fscale = float(e->P.fscale);
            sp.flags = e->flags;
            launch_small_solve(sp, s);
            return;
        }
        // the tensor path decides screening per pass on the host: run it eagerly;
        // the CUDA-core path (small / low-d problems, launch-bound) replays a graph
        const char* env = std::getenv("FSK_GRAPH");
        const bool use_graph = !e->P.tc && s != nullptr && !(env && env[0] == '0');
        if (!use_graph) {
            body();
            return;
        }
        if (!e->graph || e->graph_iters != iters || e->graph_stream != s || e->graph_f != e->f ||
            e->graph_g != e->g || e->graph_eps != e->eps) {
            drop_graph(e);
            cudaGraph_t g = nullptr;
            FSKB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            try {
                body();
            } catch (...) {
                cudaStreamEndCapture(s, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            FSKB_CUDA(cudaStreamEndCapture(s, &g));
            FSKB_CUDA(cudaGraphInstantiate(&e->graph, g, 0));
            cudaGraphDestroy(g);
            e->graph_iters = iters;
            e->graph_stream = s;
            e->graph_f = e->f;
            e->graph_g = e->g;
            e->graph_eps = e->eps;
        } else {
            count_launch(4 * iters);  // the captured launches (host-side counter)
        }
        FSKB_CUDA(cudaGraphLaunch(e->graph, s));
    });
}

int fsk_engine_grad(fsk_engine* e, int64_t row_begin, int64_t row_end, float* grad_dev,
                    void* stream) {
    return eguard([&] {
        if (!e->f || !e->g) throw ValidationFailure("engine potentials not bound");
        const int64_t n = e->P.src.n, d = e->P.src.d;
        if (row_begin < 0 || row_end > n || row_begin > row_end)
            throw ValidationFailure("engine row range out of bounds");
        const int64_t R = row_end - row_begin;
        if (R == 0) return;
        cudaStream_t s = pick(e, stream);
        Fence fence_{e, s};
        e->P.s = s;
        const float eps = float(e->eps);
        if (e->P.tc) {
            e->P.tc->grad(e->P, 0, e->g, e->f, eps, row_begin, row_end, grad_dev, e->flags);
            return;
        }
        // CUDA-core path: the gradient pass in fp64 (grad_rows_fp64)
        (void)eps;
        DevBuf<double> G64(size_t(R * d), s);
        grad_rows_fp64(e->P, e->f, e->g, e->eps, row_begin, row_end, G64.get(), e->flags, s);
        launch_f64_to_f32(G64.get(), grad_dev, R * d, s);
    });
}

namespace {
// One LSE pass of `side` at the bound potentials: marginal, natural LSE/max and
// (tensor path) the log2 LSE split, as consumed by the transport applications.
struct SideLse {
    DevBuf<float> marg, lse, mx, l2h, l2l;
};
SideLse side_lse(fsk_engine* e, int side, cudaStream_t s) {
    const int64_t R = side == 0 ? e->P.src.n : e->P.tgt.n;
    SideLse o;
    o.marg.alloc(size_t(R), s);
    o.lse.alloc(size_t(R), s);
    o.mx.alloc(size_t(R), s);
    FinalizeArgs<float> fa{};
    fa.eps = float(e->eps);
    fa.flags = e->flags;
    fa.old_pot = side == 0 ? e->f : e->g;
    fa.w = side == 0 ? e->P.src.w.get() : e->P.tgt.w.get();
    fa.out_marg = o.marg.get();
    fa.marg_flag = side == 0 ? kFlagNonFiniteRowMarginal : kFlagNonFiniteColMarginal;
    fa.out_lse = o.lse.get();
    fa.out_max = o.mx.get();
    if (e->P.tc) {
        o.l2h.alloc(size_t(R), s);
        o.l2l.alloc(size_t(R), s);
        fa.out_l2h = o.l2h.get();
        fa.out_l2l = o.l2l.get();
    }
    half_step_rows<float>(e->P, side, side == 0 ? e->g : e->f, float(e->eps), fa, 0, R);
    return o;
}
}  // namespace

int fsk_engine_transport_mat(fsk_engine* e, int side, const float* v_dev, int64_t p,
                             float* out_dev, void* stream) {
    return eguard([&] {
        if (!e->f || !e->g) throw ValidationFailure("engine potentials not bound");
        if (side != 0 && side != 1) throw ValidationFailure("side must be 0 or 1");
        if (p < 1) throw ValidationFailure("p must be positive");
        cudaStream_t s = pick(e, stream);
        Fence fence_{e, s};
        e->P.s = s;
        const float eps = float(e->eps);
        const float* kpot = side == 0 ? e->g : e->f;
        const float* pot = side == 0 ? e->f : e->g;
        SideLse L = side_lse(e, side, s);
        if (e->P.tc) {
            e->P.tc->apply_mat(e->P, side, kpot, eps, L.l2h.get(), L.l2l.get(), L.marg.get(),
                               v_dev, p, out_dev, e->flags);
        } else {
            transport<float>(e->P, side, kpot, pot, eps, L.lse.get(), L.mx.get(), v_dev, p,
                             nullptr, nullptr, 0, out_dev, e->flags);
        }
    });
}

int fsk_engine_transport_hadamard(fsk_engine* e, const float* a_dev, const float* v_dev,
                                  int64_t p, float* out_dev, void* stream) {
    return eguard([&] {
        if (!e->f || !e->g) throw ValidationFailure("engine potentials not bound");
        if (p < 1) throw ValidationFailure("p must be positive");
        cudaStream_t s = pick(e, stream);
        Fence fence_{e, s};
        e->P.s = s;
        const float eps = float(e->eps);
        SideLse L = side_lse(e, 0, s);
        if (e->P.tc) {
            e->P.tc->apply_mat(e->P, 0, e->g, eps, L.l2h.get(), L.l2l.get(), L.marg.get(), v_dev,
                               p, out_dev, e->flags, a_dev);
        } else {
            transport<float>(e->P, 0, e->g, e->f, eps, L.lse.get(), L.mx.get(), v_dev, p, a_dev,
                             e->P.tgt.pts.get(), e->P.src.d, out_dev, e->flags);
        }
    });
}

int fsk_engine_transport_vec(fsk_engine* e, int side, const float* v_dev, double* out_dev,
                             void* stream) {
    return eguard([&] {
        if (!e->f || !e->g) throw ValidationFailure("engine potentials not bound");
        if (side != 0 && side != 1) throw ValidationFailure("side must be 0 or 1");
        cudaStream_t s = pick(e, stream);
        Fence fence_{e, s};
        e->P.s = s;
        const float eps = float(e->eps);
        const int64_t R = side == 0 ? e->P.src.n : e->P.tgt.n;
        const float* kpot = side == 0 ? e->g : e->f;
        const float* pot = side == 0 ? e->f : e->g;
        DevBuf<float> marg(size_t(R), s), lse(size_t(R), s), mx(size_t(R), s);
        DevBuf<float> l2h, l2l;
        FinalizeArgs<float> fa{};
        fa.eps = eps;
        fa.flags = e->flags;
        fa.old_pot = pot;
        fa.w = side == 0 ? e->P.src.w.get() : e->P.tgt.w.get();
        fa.out_marg = marg.get();
        fa.marg_flag = side == 0 ? kFlagNonFiniteRowMarginal : kFlagNonFiniteColMarginal;
        fa.out_lse = lse.get();
        fa.out_max = mx.get();
        if (e->P.tc) {
            l2h.alloc(size_t(R), s);
            l2l.alloc(size_t(R), s);
            fa.out_l2h = l2h.get();
            fa.out_l2l = l2l.get();
        }
        half_step_rows<float>(e->P, side, kpot, eps, fa, 0, R);
        if (e->P.tc) {
            e->P.tc->vec(e->P, side, kpot, eps, l2h.get(), l2l.get(), marg.get(), v_dev, out_dev,
                         e->flags);
        } else {
            DevBuf<float> outf(size_t(R), s);
            transport<float>(e->P, side, kpot, pot, eps, lse.get(), mx.get(), v_dev, 1, nullptr,
                             nullptr, 0, outf.get(), e->flags);
            launch_f32_to_f64(outf.get(), out_dev, R, s);
        }
    });
}

int fsk_engine_transport_prepare(fsk_engine* e, int64_t f_begin, int64_t f_end, int64_t g_begin,
                                 int64_t g_end, void* stream) {
    return eguard([&] {
        if (!e->f || !e->g) throw ValidationFailure("engine potentials not bound");
        if (!(e->eps > 0.0)) throw ValidationFailure("engine eps not set");
        const int64_t rb[2] = {f_begin, g_begin}, re[2] = {f_end, g_end};
        cudaStream_t s = pick(e, stream);
        Fence fence_{e, s};
        e->P.s = s;
        auto& pr = e->prep;
        pr.valid = false;
        for (int side = 0; side < 2; ++side) {
            const int64_t R = side == 0 ? e->P.src.n : e->P.tgt.n;
            if (rb[side] < 0 || re[side] > R || rb[side] > re[side])
                throw ValidationFailure("engine row range out of bounds");
            if (e->P.tc && rb[side] % 256 != 0)
                throw ValidationFailure("transport row shards must start on a 256-row boundary");
            for (DevBuf<float>* b : {&pr.marg[side], &pr.lse[side], &pr.mx[side]})
                if (b->size() < size_t(R)) b->alloc(size_t(R), s);
            FinalizeArgs<float> fa{};
            fa.eps = float(e->eps);
            fa.flags = e->flags;
            fa.old_pot = side == 0 ? e->f : e->g;
            fa.w = side == 0 ? e->P.src.w.get() : e->P.tgt.w.get();
            fa.out_marg = pr.marg[side].get();
            fa.marg_flag = side == 0 ? kFlagNonFiniteRowMarginal : kFlagNonFiniteColMarginal;
            fa.out_lse = pr.lse[side].get();
            fa.out_max = pr.mx[side].get();
            if (e->P.tc) {
                for (DevBuf<float>* b : {&pr.l2h[side], &pr.l2l[side]})
                    if (b->size() < size_t(R)) b->alloc(size_t(R), s);
                fa.out_l2h = pr.l2h[side].get();
                fa.out_l2l = pr.l2l[side].get();
            }
            const float* kpot = side == 0 ? e->g : e->f;
            half_step_rows<float>(e->P, side, kpot, float(e->eps), fa, rb[side], re[side]);
            // exact row-max seeds: the recorded live sets keep only blocks within 2^-64
            // of a row max (the transport passes below score only those)
            if (e->P.tc)
                e->P.tc->tighten_live(e->P, side, kpot, float(e->eps), pr.mx[side].get(),
                                      e->flags, rb[side], re[side]);
            pr.rb[side] = rb[side];
            pr.re[side] = re[side];
        }
        pr.f = e->f;
        pr.g = e->g;
        pr.eps = e->eps;
        pr.valid = true;
    });
}

namespace {
const fsk_engine::Prep& check_prep(fsk_engine* e, int side, int64_t rb, int64_t re) {
    const auto& pr = e->prep;
    if (!pr.valid || pr.f != e->f || pr.g != e->g || pr.eps != e->eps)
        throw ValidationFailure("transport state not prepared for the bound potentials / eps");
    if (side != 0 && side != 1) throw ValidationFailure("side must be 0 or 1");
    if (rb < pr.rb[side] || re > pr.re[side] || rb > re)
        throw ValidationFailure("transport rows outside the prepared range");
    return pr;
}
}  // namespace

int fsk_engine_marginal(fsk_engine* e, int side, float* out_dev, void* stream) {
    return eguard([&] {
        const auto& pr = check_prep(e, side, e->prep.rb[side & 1], e->prep.re[side & 1]);
        cudaStream_t s = pick(e, stream);
        Fence fence_{e, s};
        const int64_t R = side == 0 ? e->P.src.n : e->P.tgt.n;
        FSKB_CUDA(cudaMemcpyAsync(out_dev, pr.marg[side].get(), size_t(R) * sizeof(float),
                                  cudaMemcpyDeviceToDevice, s));
    });
}

int fsk_engine_transport_vec_rows(fsk_engine* e, int side, int64_t row_begin, int64_t row_end,
                                  const float* v_dev, double* out_dev, void* stream) {
    return eguard([&] {
        const auto& pr = check_prep(e, side, row_begin, row_end);
        cudaStream_t s = pick(e, stream);
        Fence fence_{e, s};
        e->P.s = s;
        const float eps = float(e->eps);
        const float* kpot = side == 0 ? e->g : e->f;
        const float* pot = side == 0 ? e->f : e->g;
        const int64_t R = row_end - row_begin;
        if (R == 0) return;
        if (e->P.tc) {
            e->P.tc->vec(e->P, side, kpot, eps, pr.l2h[side].get(), pr.l2l[side].get(),
                         pr.marg[side].get(), v_dev, out_dev, e->flags, row_begin, row_end);
            return;
        }
        ScoreParams<float> sp = e->P.params(side, kpot, eps);
        sp.Q += row_begin * sp.d;
        sp.R = R;
        DevBuf<float> O(size_t(R), s), outf(size_t(R), s);
        launch_apply<float>(sp, pr.lse[side].get() + row_begin, v_dev, 1, nullptr, nullptr, 0,
                            O.get(), s);
        const float* w = side == 0 ? e->P.src.w.get() : e->P.tgt.w.get();
        launch_apply_finalize<float>(O.get(), R, 1, w + row_begin, pot + row_begin,
                                     pr.lse[side].get() + row_begin, pr.mx[side].get() + row_begin,
                                     eps, outf.get(), e->flags, s);
        launch_f32_to_f64(outf.get(), out_dev, R, s);
    });
}

int fsk_engine_transport_mat_rows(fsk_engine* e, int side, int64_t row_begin, int64_t row_end,
                                  const float* v_dev, int64_t p, const float* a_dev,
                                  float* out_dev, void* stream) {
    return eguard([&] {
        const auto& pr = check_prep(e, side, row_begin, row_end);
        if (p < 1) throw ValidationFailure("p must be positive");
        if (a_dev && side != 0) throw ValidationFailure("the Hadamard form is side 0 only");
        cudaStream_t s = pick(e, stream);
        Fence fence_{e, s};
        e->P.s = s;
        const float eps = float(e->eps);
        const float* kpot = side == 0 ? e->g : e->f;
        const float* pot = side == 0 ? e->f : e->g;
        const int64_t R = row_end - row_begin, d = e->P.src.d;
        if (R == 0) return;
        if (e->P.tc) {
            e->P.tc->apply_mat(e->P, side, kpot, eps, pr.l2h[side].get(), pr.l2l[side].get(),
                               pr.marg[side].get(), v_dev, p, out_dev, e->flags, a_dev, row_begin,
                               row_end);
            return;
        }
        ScoreParams<float> sp = e->P.params(side, kpot, eps);
        sp.Q += row_begin * sp.d;
        sp.R = R;
        DevBuf<float> O(size_t(R * p), s);
        launch_apply<float>(sp, pr.lse[side].get() + row_begin, v_dev, p,
                            a_dev ? a_dev + row_begin * d : nullptr,
                            a_dev ? e->P.tgt.pts.get() : nullptr, a_dev ? d : 0, O.get(), s);
        const float* w = side == 0 ? e->P.src.w.get() : e->P.tgt.w.get();
        launch_apply_finalize<float>(O.get(), R, p, w + row_begin, pot + row_begin,
                                     pr.lse[side].get() + row_begin, pr.mx[side].get() + row_begin,
                                     eps, out_dev, e->flags, s);
    });
}

uint64_t fsk_engine_screen_live_tiles(const fsk_engine* e) {
    return e && e->P.tc ? uint64_t(e->P.tc->live_tiles()) : 0;
}

double fsk_engine_live_set_fraction(const fsk_engine* e, int side) {
    return e && e->P.tc ? e->P.tc->live_set_fraction(side) : -1.0;
}

uint64_t fsk_engine_screen_blocks(const fsk_engine* e) {
    if (!e || !e->P.tc) return 0;
    e->P.tc->live_tiles();  // drains the pending read-backs
    return uint64_t(e->P.tc->screened_blocks());
}

void fsk_engine_pass_counts(const fsk_engine* e, uint64_t out[3]) {
    unsigned long long c[3] = {0, 0, 0};
    if (e && e->P.tc) {
        e->P.tc->live_tiles();   // drains the pending read-backs
        e->P.tc->pass_counts(c);
    }
    for (int k = 0; k < 3; ++k) out[k] = uint64_t(c[k]);
}

int64_t fsk_engine_kernel_launches(const fsk_engine* e) {
    (void)e;
    return launch_counter().load();
}

const char* fsk_engine_path(const fsk_engine* e) { return tensor_path_name(e->P); }

}  // extern "C"
