// fsk core / schedule / threads API (include/fsk/{core,schedule,threads}.hpp).
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <thread>
#include <vector>

#include "../../../include/fsk/core.hpp"
#include "../../../include/fsk/schedule.hpp"
#include "../../../include/fsk/threads.hpp"
#include "../common.h"
#include "../hostlib.h"
#include "bridge.h"

namespace fsk {

namespace {
template <typename F>
void as_fsk(F&& f) {
    try {
        f();
    } catch (const fskb::ValidationFailure& e) {
        throw ValidationError(e.what());
    }
}
}  // namespace

DiscreteMeasure make_uniform_measure(Mat points, std::optional<std::vector<int32_t>> labels) {
    DiscreteMeasure m;
    const std::size_t n = points.rows();
    m.points = std::move(points);
    m.weights.assign(n, 1.0 / double(n));
    m.labels = std::move(labels);
    return m;
}

void validate_measure(const DiscreteMeasure& m) {
    if (m.points.rows() < 1 || m.points.cols() < 1)
        throw ValidationError("measure must have n >= 1 points of dimension d >= 1");
    bridge::check_measure_shapes(m);
    as_fsk([&] { fskb::validate_measure_raw(bridge::view(m)); });
}

void validate_problem(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
                      const CostSpec& spec) {
    validate_measure(src);
    validate_measure(tgt);
    bridge::check_spec_shape(spec);
    const fsk_cost c = bridge::view(spec);
    as_fsk([&] { fskb::validate_problem_raw(bridge::view(src), bridge::view(tgt), &c); });
}

void validate_sinkhorn_config(const SinkhornConfig& cfg) {
    const fsk_config c = bridge::view(cfg);
    as_fsk([&] { fskb::validate_config_raw(c); });
}

void validate_tiles(const TileConfig& tiles) {
    const fsk_tiles t = bridge::view(tiles);
    as_fsk([&] { fskb::validate_tiles_raw(&t); });
}

Vec squared_norms(const Mat& points) {
    if (!fskb::all_finite(points.data(), int64_t(points.size())))
        throw ValidationError("non-finite coordinate in squared_norms input");
    Vec out(points.rows());
    for (std::size_t i = 0; i < points.rows(); ++i) {
        double s = 0.0;
        for (std::size_t t = 0; t < points.cols(); ++t) s += points(i, t) * points(i, t);
        out[i] = s;
    }
    return out;
}

std::pair<Vec, Vec> unshift_potentials(const ShiftedPotentials& p, const Vec& alpha,
                                       const Vec& beta) {
    if (p.f_hat.size() != alpha.size() || p.g_hat.size() != beta.size())
        throw ValidationError("potential/shift length mismatch in unshift_potentials");
    Vec f(alpha.size()), g(beta.size());
    for (std::size_t i = 0; i < f.size(); ++i) f[i] = p.f_hat[i] + alpha[i];
    for (std::size_t j = 0; j < g.size(); ++j) g[j] = p.g_hat[j] + beta[j];
    return {std::move(f), std::move(g)};
}

ShiftedPotentials shift_potentials(const Vec& f, const Vec& g, const Vec& alpha, const Vec& beta,
                                   double eps) {
    if (f.size() != alpha.size() || g.size() != beta.size())
        throw ValidationError("potential/shift length mismatch in shift_potentials");
    ShiftedPotentials p;
    p.eps = eps;
    p.f_hat.resize(f.size());
    p.g_hat.resize(g.size());
    for (std::size_t i = 0; i < f.size(); ++i) p.f_hat[i] = f[i] - alpha[i];
    for (std::size_t j = 0; j < g.size(); ++j) p.g_hat[j] = g[j] - beta[j];
    return p;
}

Vec potential_shift(const Mat& points, const CostSpec& spec) {
    Vec a = squared_norms(points);
    const double s = spec.feature_scale();
    if (s != 1.0)
        for (double& v : a) v *= s;
    return a;
}

double joint_sq_diameter(const Mat& X, const Mat& Y) {
    return fskb::joint_sq_diameter_raw(X.data(), int64_t(X.rows()), Y.data(), int64_t(Y.rows()),
                                       int64_t(X.cols()));
}

std::vector<double> eps_schedule(const SinkhornConfig& cfg, double sq_diam) {
    std::vector<double> out;
    const fsk_config c = bridge::view(cfg);
    as_fsk([&] { out = fskb::eps_schedule_raw(c, sq_diam); });
    return out;
}

// ---- host worker utility (threads.hpp) -----------------------------------------

namespace {
std::atomic<std::size_t> g_workers{0};
}

void set_num_threads(std::size_t n) { g_workers.store(n == 0 ? 1 : n); }

std::size_t num_threads() {
    const std::size_t n = g_workers.load();
    if (n) return n;
    if (const char* s = std::getenv("FSK_THREADS")) {
        const long v = std::atol(s);
        if (v >= 1) return std::size_t(v);
    }
    const std::size_t hw = std::thread::hardware_concurrency();
    return hw ? hw : 1;
}

namespace detail {
void run_parallel(std::size_t nblocks, std::size_t nworkers,
                  void (*trampoline)(void*, std::size_t), void* ctx) {
    std::vector<std::thread> pool;
    pool.reserve(nworkers);
    for (std::size_t w = 0; w < nworkers; ++w)
        pool.emplace_back([=] {
            for (std::size_t b = w; b < nblocks; b += nworkers) trampoline(ctx, b);
        });
    for (auto& t : pool) t.join();
}
}  // namespace detail

}  // namespace fsk
