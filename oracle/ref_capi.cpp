// ctypes-friendly C wrapper around the (patched) reference CPU library.
//
// TEST INFRASTRUCTURE ONLY. Compiled by oracle/build_ref.py together with the
// reference's own sources under /root/reference/proj/src into
// oracle/_ref/libfsk_ref.so. Used by tests/ (as a checker), by
// tests/golden/make_golden.py (to produce committed fixtures) and by
// bench.py's cpu_baseline / --impl reference arm (to time the reference's
// own CPU path). Never linked into the product.
//
// Every entry point forwards to the reference API declared in
// proj/include/fsk/stream.hpp:20-98 and proj/include/fsk/solver.hpp:17-40.
#include <cstdint>
#include <cstring>
#include <string>

#include "fsk/core.hpp"
#include "fsk/ledger.hpp"
#include "fsk/solver.hpp"
#include "fsk/stream.hpp"
#include "fsk/threads.hpp"

namespace {

thread_local std::string g_err;

struct RefMeasure {
    const double* pts;
    const double* w;
    const int32_t* labels;  // nullable
    int64_t n, d;
};

struct RefCost {
    int32_t kind;  // 0 squared Euclidean, 1 label augmented
    double lambda1, lambda2;
    const double* label_cost;  // V x V row-major
    int64_t num_labels;
};

fsk::DiscreteMeasure to_measure(const RefMeasure& m) {
    fsk::DiscreteMeasure out;
    out.points = fsk::Mat(static_cast<std::size_t>(m.n), static_cast<std::size_t>(m.d));
    if (m.n * m.d > 0) std::memcpy(out.points.data(), m.pts, sizeof(double) * m.n * m.d);
    out.weights.assign(m.w, m.w + m.n);
    if (m.labels) out.labels = std::vector<int32_t>(m.labels, m.labels + m.n);
    return out;
}

fsk::CostSpec to_cost(const RefCost* c) {
    if (!c || c->kind == 0) return fsk::CostSpec::squared_euclidean();
    fsk::Mat W(static_cast<std::size_t>(c->num_labels), static_cast<std::size_t>(c->num_labels));
    if (c->num_labels > 0)
        std::memcpy(W.data(), c->label_cost, sizeof(double) * c->num_labels * c->num_labels);
    return fsk::CostSpec::label_augmented(c->lambda1, c->lambda2, std::move(W));
}

fsk::Mat to_mat(const double* p, int64_t rows, int64_t cols) {
    fsk::Mat m(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
    if (rows * cols > 0) std::memcpy(m.data(), p, sizeof(double) * rows * cols);
    return m;
}

void export_ledger(const fsk::IoLedger& l, uint64_t* out) {
    if (!out) return;
    out[0] = l.slow_to_fast_scalars.load();
    out[1] = l.fast_to_slow_scalars.load();
    out[2] = l.kernel_invocations.load();
    out[3] = l.transport_vector_applies.load();
    out[4] = l.transport_matrix_applies.load();
    out[5] = l.hadamard_applies.load();
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const fsk::ValidationError& e) {
        g_err = e.what();
        return 1;
    } catch (const fsk::NumericalError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

fsk::ShiftedPotentials pots(const double* f, int64_t n, const double* g, int64_t m, double eps) {
    fsk::ShiftedPotentials p;
    p.f_hat.assign(f, f + n);
    p.g_hat.assign(g, g + m);
    p.eps = eps;
    return p;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_num_threads(int64_t n) { fsk::set_num_threads(static_cast<std::size_t>(n)); }
int64_t ref_num_threads() { return static_cast<int64_t>(fsk::num_threads()); }

int ref_update_f_hat(const RefMeasure* src, const RefMeasure* tgt, const double* g_hat,
                     const RefCost* cost, double eps, int64_t bn, int64_t bm, double* out,
                     uint64_t* ledger) {
    return guarded([&] {
        fsk::IoLedger led;
        fsk::Vec g(g_hat, g_hat + tgt->n);
        auto r = fsk::stream::update_f_hat(to_measure(*src), to_measure(*tgt), g, to_cost(cost),
                                           eps, {std::size_t(bn), std::size_t(bm)}, led);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
        export_ledger(led, ledger);
    });
}

int ref_update_g_hat(const RefMeasure* src, const RefMeasure* tgt, const double* f_hat,
                     const RefCost* cost, double eps, int64_t bn, int64_t bm, double* out,
                     uint64_t* ledger) {
    return guarded([&] {
        fsk::IoLedger led;
        fsk::Vec f(f_hat, f_hat + src->n);
        auto r = fsk::stream::update_g_hat(to_measure(*src), to_measure(*tgt), f, to_cost(cost),
                                           eps, {std::size_t(bn), std::size_t(bm)}, led);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
        export_ledger(led, ledger);
    });
}

int ref_symmetric_update(const RefMeasure* src, const RefMeasure* tgt, const double* f_hat,
                         const double* g_hat, double eps, const RefCost* cost, int64_t bn,
                         int64_t bm, double* out_f, double* out_g, uint64_t* ledger) {
    return guarded([&] {
        fsk::IoLedger led;
        auto r = fsk::stream::symmetric_update(to_measure(*src), to_measure(*tgt),
                                               pots(f_hat, src->n, g_hat, tgt->n, eps),
                                               to_cost(cost), {std::size_t(bn), std::size_t(bm)},
                                               led);
        std::memcpy(out_f, r.f_hat.data(), sizeof(double) * r.f_hat.size());
        std::memcpy(out_g, r.g_hat.data(), sizeof(double) * r.g_hat.size());
        export_ledger(led, ledger);
    });
}

int ref_apply_plan(const RefMeasure* src, const RefMeasure* tgt, const double* f_hat,
                   const double* g_hat, double eps, const RefCost* cost, const double* V,
                   int64_t p, int64_t bn, int64_t bm, double* out, uint64_t* ledger) {
    return guarded([&] {
        fsk::IoLedger led;
        auto r = fsk::stream::apply_plan(to_measure(*src), to_measure(*tgt),
                                         pots(f_hat, src->n, g_hat, tgt->n, eps), to_cost(cost),
                                         to_mat(V, tgt->n, p), {std::size_t(bn), std::size_t(bm)},
                                         led);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
        export_ledger(led, ledger);
    });
}

int ref_apply_plan_adjoint(const RefMeasure* src, const RefMeasure* tgt, const double* f_hat,
                           const double* g_hat, double eps, const RefCost* cost, const double* U,
                           int64_t p, int64_t bn, int64_t bm, double* out, uint64_t* ledger) {
    return guarded([&] {
        fsk::IoLedger led;
        auto r = fsk::stream::apply_plan_adjoint(
            to_measure(*src), to_measure(*tgt), pots(f_hat, src->n, g_hat, tgt->n, eps),
            to_cost(cost), to_mat(U, src->n, p), {std::size_t(bn), std::size_t(bm)}, led);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
        export_ledger(led, ledger);
    });
}

int ref_apply_hadamard_plan(const RefMeasure* src, const RefMeasure* tgt, const double* f_hat,
                            const double* g_hat, double eps, const RefCost* cost, const double* A,
                            const double* B, int64_t r, const double* V, int64_t p, int64_t bn,
                            int64_t bm, double* out, uint64_t* ledger) {
    return guarded([&] {
        fsk::IoLedger led;
        auto o = fsk::stream::apply_hadamard_plan(
            to_measure(*src), to_measure(*tgt), pots(f_hat, src->n, g_hat, tgt->n, eps),
            to_cost(cost), to_mat(A, src->n, r), to_mat(B, tgt->n, r), to_mat(V, tgt->n, p),
            {std::size_t(bn), std::size_t(bm)}, led);
        std::memcpy(out, o.data(), sizeof(double) * o.size());
        export_ledger(led, ledger);
    });
}

int ref_induced_marginals(const RefMeasure* src, const RefMeasure* tgt, const double* f_hat,
                          const double* g_hat, double eps, const RefCost* cost, int64_t bn,
                          int64_t bm, double* out_r, double* out_c, uint64_t* ledger) {
    return guarded([&] {
        fsk::IoLedger led;
        auto [r, c] = fsk::stream::induced_marginals(to_measure(*src), to_measure(*tgt),
                                                     pots(f_hat, src->n, g_hat, tgt->n, eps),
                                                     to_cost(cost),
                                                     {std::size_t(bn), std::size_t(bm)}, led);
        std::memcpy(out_r, r.data(), sizeof(double) * r.size());
        std::memcpy(out_c, c.data(), sizeof(double) * c.size());
        export_ledger(led, ledger);
    });
}

// fp32 half-steps (stream.cpp:437-451). Points/weights already float.
int ref_update_f_hat_f32(const float* src_pts, const float* src_w, int64_t n, const float* tgt_pts,
                         const float* tgt_w, int64_t m, int64_t d, const float* g_hat, float eps,
                         int64_t bn, int64_t bm, float* out, uint64_t* ledger) {
    return guarded([&] {
        fsk::IoLedger led;
        fsk::stream::FloatCloud s, t;
        s.points.assign(src_pts, src_pts + n * d);
        s.weights.assign(src_w, src_w + n);
        s.n = n;
        s.d = d;
        t.points.assign(tgt_pts, tgt_pts + m * d);
        t.weights.assign(tgt_w, tgt_w + m);
        t.n = m;
        t.d = d;
        std::vector<float> g(g_hat, g_hat + m);
        auto r = fsk::stream::update_f_hat_f32(s, t, g, eps, {std::size_t(bn), std::size_t(bm)},
                                               led);
        std::memcpy(out, r.data(), sizeof(float) * r.size());
        export_ledger(led, ledger);
    });
}

int ref_update_g_hat_f32(const float* src_pts, const float* src_w, int64_t n, const float* tgt_pts,
                         const float* tgt_w, int64_t m, int64_t d, const float* f_hat, float eps,
                         int64_t bn, int64_t bm, float* out, uint64_t* ledger) {
    return guarded([&] {
        fsk::IoLedger led;
        fsk::stream::FloatCloud s, t;
        s.points.assign(src_pts, src_pts + n * d);
        s.weights.assign(src_w, src_w + n);
        s.n = n;
        s.d = d;
        t.points.assign(tgt_pts, tgt_pts + m * d);
        t.weights.assign(tgt_w, tgt_w + m);
        t.n = m;
        t.d = d;
        std::vector<float> f(f_hat, f_hat + n);
        auto r = fsk::stream::update_g_hat_f32(s, t, f, eps, {std::size_t(bn), std::size_t(bm)},
                                               led);
        std::memcpy(out, r.data(), sizeof(float) * r.size());
        export_ledger(led, ledger);
    });
}

struct RefConfig {
    double eps;
    int32_t schedule;  // 0 alternating, 1 symmetric
    int32_t max_iters;
    double marginal_tol;
    double eps_scaling_factor;
    int32_t extra_iters_at_final_eps;
    int32_t precision;  // 0 single, 1 double
};

fsk::SinkhornConfig to_cfg(const RefConfig& c) {
    fsk::SinkhornConfig cfg;
    cfg.eps = c.eps;
    cfg.schedule = c.schedule ? fsk::Schedule::Symmetric : fsk::Schedule::Alternating;
    cfg.max_iters = c.max_iters;
    cfg.marginal_tol = c.marginal_tol;
    cfg.eps_scaling_factor = c.eps_scaling_factor;
    cfg.extra_iters_at_final_eps = c.extra_iters_at_final_eps;
    cfg.precision = c.precision ? fsk::Precision::Double : fsk::Precision::Single;
    return cfg;
}

// out_f/out_g: n/m doubles; out_scalars: [iterations, marginal_violation, dual_cost, final eps]
int ref_sinkhorn_solve(const RefMeasure* src, const RefMeasure* tgt, const RefCost* cost,
                       const RefConfig* cfg, int64_t bn, int64_t bm, double* out_f, double* out_g,
                       double* out_scalars, double* eps_history, int64_t eps_cap,
                       uint64_t* ledger) {
    return guarded([&] {
        fsk::IoLedger led;
        auto rep = fsk::solver::sinkhorn_solve(to_measure(*src), to_measure(*tgt), to_cost(cost),
                                               to_cfg(*cfg), {std::size_t(bn), std::size_t(bm)},
                                               led);
        std::memcpy(out_f, rep.potentials.f_hat.data(), sizeof(double) * src->n);
        std::memcpy(out_g, rep.potentials.g_hat.data(), sizeof(double) * tgt->n);
        out_scalars[0] = rep.iterations;
        out_scalars[1] = rep.marginal_violation;
        out_scalars[2] = rep.dual_cost;
        out_scalars[3] = rep.potentials.eps;
        for (int64_t k = 0; k < eps_cap && k < (int64_t)rep.eps_history.size(); ++k)
            eps_history[k] = rep.eps_history[k];
        export_ledger(led, ledger);
    });
}

int ref_dual_cost(const RefMeasure* src, const RefMeasure* tgt, const double* f_hat,
                  const double* g_hat, double eps, const RefCost* cost, int64_t bn, int64_t bm,
                  double* out, uint64_t* ledger) {
    return guarded([&] {
        fsk::IoLedger led;
        *out = fsk::solver::dual_cost(to_measure(*src), to_measure(*tgt),
                                      pots(f_hat, src->n, g_hat, tgt->n, eps), to_cost(cost),
                                      {std::size_t(bn), std::size_t(bm)}, led);
        export_ledger(led, ledger);
    });
}

int ref_sinkhorn_divergence(const RefMeasure* mu, const RefMeasure* nu, const RefCost* cost,
                            const RefConfig* cfg, int64_t bn, int64_t bm, double* out,
                            uint64_t* ledger) {
    return guarded([&] {
        fsk::IoLedger led;
        *out = fsk::solver::sinkhorn_divergence(to_measure(*mu), to_measure(*nu), to_cost(cost),
                                                to_cfg(*cfg), {std::size_t(bn), std::size_t(bm)},
                                                led);
        export_ledger(led, ledger);
    });
}

}  // extern "C"
