#include "hostlib.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>
#include <limits>

#include "../../include/fsk/rng.hpp"
#include "common.h"

namespace fskb {

namespace {
std::string num(double v) { return std::to_string(v); }
}  // namespace

namespace {
// non-finite <=> all exponent bits set: a branch-free integer scan (vectorizes)
bool finite_range(const double* p, int64_t n) {
    const uint64_t* b = reinterpret_cast<const uint64_t*>(p);
    uint64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) bad |= uint64_t((b[i] & 0x7FF0000000000000ull) == 0x7FF0000000000000ull);
    return bad == 0;
}
}  // namespace

bool all_finite(const double* p, int64_t n) {
    const int64_t per = int64_t(1) << 22;
    if (n < 2 * per) return finite_range(p, n);
    // the cloud scan runs on every validated call: split it over host threads
    const int T = int(std::min<int64_t>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())),
                                        n / per));
    std::vector<char> ok(size_t(T), 1);
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
            const int64_t lo = n * t / T, hi = n * (t + 1) / T;
            ok[size_t(t)] = finite_range(p + lo, hi - lo) ? 1 : 0;
        });
    for (auto& x : th) x.join();
    for (char v : ok)
        if (!v) return false;
    return true;
}

void validate_measure_raw(const fsk_measure& m, bool check_points) {
    if (m.n < 1 || m.d < 1)
        throw ValidationFailure("measure must have n >= 1 points of dimension d >= 1");
    if (check_points && !all_finite(m.points, m.n * m.d))
        throw ValidationFailure(kNonFiniteCoordinate);
    double sum = 0.0;
    for (int64_t i = 0; i < m.n; ++i) {
        const double w = m.weights[i];
        if (!(w > 0.0)) throw ValidationFailure("weights must be strictly positive");
        sum += w;
    }
    if (std::abs(sum - 1.0) > 1e-12)
        throw ValidationFailure("weights must sum to 1 (got " + num(sum) + ")");
    if (m.labels) {
        for (int64_t i = 0; i < m.n; ++i)
            if (m.labels[i] < 0) throw ValidationFailure("labels must be nonnegative");
    }
}

void validate_problem_raw(const fsk_measure& src, const fsk_measure& tgt, const fsk_cost* cost,
                          bool measures_checked, bool check_points) {
    if (!measures_checked) {
        validate_measure_raw(src, check_points);
        validate_measure_raw(tgt, check_points);
    }
    if (src.d != tgt.d)
        throw ValidationFailure("source dimension " + std::to_string(src.d) +
                                " != target dimension " + std::to_string(tgt.d));
    if (labeled_cost(cost)) {
        if (!src.labels || !tgt.labels)
            throw ValidationFailure("label-augmented cost requires labels on both measures");
        if (cost->lambda1 < 0.0 || cost->lambda2 < 0.0)
            throw ValidationFailure("lambda1/lambda2 must be nonnegative");
        const int64_t v = cost->num_labels;
        for (int64_t i = 0; i < src.n; ++i)
            if (src.labels[i] >= v)
                throw ValidationFailure("source label " + std::to_string(src.labels[i]) +
                                        " out of range of label cost table");
        for (int64_t j = 0; j < tgt.n; ++j)
            if (tgt.labels[j] >= v)
                throw ValidationFailure("target label " + std::to_string(tgt.labels[j]) +
                                        " out of range of label cost table");
        if (!all_finite(cost->label_cost, v * v))
            throw ValidationFailure("non-finite entry in label cost table");
    }
}

void validate_config_raw(const fsk_config& cfg) {
    if (!(cfg.eps > 0.0)) throw ValidationFailure("eps must be positive");
    if (cfg.max_iters < 1) throw ValidationFailure("max_iters must be positive");
    if (cfg.marginal_tol < 0.0) throw ValidationFailure("marginal_tol must be nonnegative");
    if (!(cfg.eps_scaling_factor > 0.0 && cfg.eps_scaling_factor <= 1.0))
        throw ValidationFailure("eps_scaling_factor must lie in (0, 1]");
    if (cfg.extra_iters_at_final_eps < 0)
        throw ValidationFailure("extra_iters_at_final_eps must be nonnegative");
}

void validate_tiles_raw(const fsk_tiles* tiles) {
    if (!tiles || tiles->block_rows < 1 || tiles->block_cols < 1)
        throw ValidationFailure("tile block sizes must be >= 1");
}

void check_potentials_raw(const double* f, int64_t n, const double* g, int64_t m, double eps) {
    if (!(eps > 0.0)) throw ValidationFailure("potentials carry nonpositive eps");
    if (!all_finite(f, n) || !all_finite(g, m))
        throw ValidationFailure("non-finite potential entry");
}

// ---- ledger -----------------------------------------------------------------

Counts lse_counts(int64_t R, int64_t C, int64_t d, int64_t br, int64_t bc, bool labeled) {
    const uint64_t L = labeled ? 1 : 0;
    br = std::min(br, R);
    const uint64_t nblocks = uint64_t((R + br - 1) / br);
    Counts c;
    // per block: bn*d (+bn labels); per tile: bm*d + 2bm (+bm labels); store bn
    c.load = uint64_t(R) * d + L * R + nblocks * (uint64_t(C) * (d + 2) + L * C);
    c.store = uint64_t(R);
    return c;
}

Counts apply_counts(int64_t R, int64_t C, int64_t d, int64_t p, int64_t r, int64_t br, int64_t bc,
                    bool labeled) {
    const uint64_t L = labeled ? 1 : 0;
    br = std::min(br, R);
    const uint64_t nblocks = uint64_t((R + br - 1) / br);
    Counts c;
    c.load = uint64_t(R) * (d + 2 + L + r) + nblocks * uint64_t(C) * (d + 2 + p + L + r);
    c.store = uint64_t(R) * p;
    return c;
}

void ledger_add(fsk_ledger* l, const Counts& c) {
    if (!l) return;
    l->slow_to_fast_scalars += c.load;
    l->fast_to_slow_scalars += c.store;
}

namespace {
uint64_t wtab_scalars(const fsk_cost* c) {
    return labeled_cost(c) ? uint64_t(c->num_labels) * uint64_t(c->num_labels) : 0;
}
}  // namespace

void ledger_update_f(fsk_ledger* l, int64_t n, int64_t m, int64_t d, const fsk_tiles& t,
                     const fsk_cost* cost) {
    if (!l) return;
    l->kernel_invocations += 1;
    l->slow_to_fast_scalars += wtab_scalars(cost);
    ledger_add(l, lse_counts(n, m, d, t.block_rows, t.block_cols, labeled_cost(cost)));
}

void ledger_update_g(fsk_ledger* l, int64_t n, int64_t m, int64_t d, const fsk_tiles& t,
                     const fsk_cost* cost) {
    if (!l) return;
    l->kernel_invocations += 1;
    l->slow_to_fast_scalars += wtab_scalars(cost);
    ledger_add(l, lse_counts(m, n, d, t.block_cols, t.block_rows, labeled_cost(cost)));
}

void ledger_symmetric(fsk_ledger* l, int64_t n, int64_t m, int64_t d, const fsk_tiles& t,
                      const fsk_cost* cost) {
    if (!l) return;
    l->kernel_invocations += 1;
    l->slow_to_fast_scalars += wtab_scalars(cost);
    ledger_add(l, lse_counts(n, m, d, t.block_rows, t.block_cols, labeled_cost(cost)));
    ledger_add(l, lse_counts(m, n, d, t.block_cols, t.block_rows, labeled_cost(cost)));
    l->slow_to_fast_scalars += uint64_t(n + m);
}

void ledger_apply(fsk_ledger* l, int64_t n, int64_t m, int64_t d, int64_t p, const fsk_tiles& t,
                  const fsk_cost* cost, bool adjoint) {
    if (!l) return;
    l->kernel_invocations += 1;
    (p == 1 ? l->transport_vector_applies : l->transport_matrix_applies) += 1;
    l->slow_to_fast_scalars += wtab_scalars(cost);
    if (!adjoint)
        ledger_add(l, apply_counts(n, m, d, p, 0, t.block_rows, t.block_cols, labeled_cost(cost)));
    else
        ledger_add(l, apply_counts(m, n, d, p, 0, t.block_cols, t.block_rows, labeled_cost(cost)));
}

void ledger_hadamard(fsk_ledger* l, int64_t n, int64_t m, int64_t d, int64_t r, int64_t p,
                     const fsk_tiles& t, const fsk_cost* cost) {
    if (!l) return;
    l->kernel_invocations += 1;
    l->hadamard_applies += 1;
    l->slow_to_fast_scalars += wtab_scalars(cost);
    ledger_add(l, apply_counts(n, m, d, p, r, t.block_rows, t.block_cols, labeled_cost(cost)));
}

void ledger_marginals(fsk_ledger* l, int64_t n, int64_t m, int64_t d, const fsk_tiles& t,
                      const fsk_cost* cost) {
    if (!l) return;
    l->kernel_invocations += 1;
    l->slow_to_fast_scalars += wtab_scalars(cost);
    ledger_add(l, lse_counts(n, m, d, t.block_rows, t.block_cols, labeled_cost(cost)));
    l->slow_to_fast_scalars += 2 * uint64_t(n);
    ledger_add(l, lse_counts(m, n, d, t.block_cols, t.block_rows, labeled_cost(cost)));
    l->slow_to_fast_scalars += 2 * uint64_t(m);
}

void ledger_update_f32(fsk_ledger* l, int64_t R, int64_t C, int64_t d, int64_t br, int64_t bc) {
    if (!l) return;
    l->kernel_invocations += 1;
    ledger_add(l, lse_counts(R, C, d, br, bc, false));
}

// ---- schedule -----------------------------------------------------------------

// schedule.cpp:8-25, one row-major pass (min / max are order-independent, so the
// result is identical to the reference's per-column scans)
double joint_sq_diameter_raw(const double* X, int64_t n, const double* Y, int64_t m, int64_t d) {
    std::vector<double> lo(size_t(d), std::numeric_limits<double>::infinity());
    std::vector<double> hi(size_t(d), -std::numeric_limits<double>::infinity());
    auto scan = [&](const double* P, int64_t rows) {
        for (int64_t i = 0; i < rows; ++i)
            for (int64_t t = 0; t < d; ++t) {
                const double v = P[i * d + t];
                lo[size_t(t)] = v < lo[size_t(t)] ? v : lo[size_t(t)];
                hi[size_t(t)] = hi[size_t(t)] < v ? v : hi[size_t(t)];
            }
    };
    scan(X, n);
    scan(Y, m);
    double diam2 = 0.0;
    for (int64_t t = 0; t < d; ++t) diam2 += (hi[size_t(t)] - lo[size_t(t)]) * (hi[size_t(t)] - lo[size_t(t)]);
    return diam2;
}

std::vector<double> eps_schedule_raw(const fsk_config& cfg, double sq_diam) {
    validate_config_raw(cfg);
    std::vector<double> out;
    const std::size_t cap = std::size_t(cfg.max_iters);
    if (cfg.eps_scaling_factor >= 1.0) {
        out.assign(cap, cfg.eps);
        return out;
    }
    // geometric decay from the squared diameter; the clamped final value is
    // emitted before the loop stops (schedule.cpp:36-40), then the extras
    double e = sq_diam;
    while (out.size() < cap) {
        out.push_back(e > cfg.eps ? e : cfg.eps);
        if (e <= cfg.eps) break;
        e *= cfg.eps_scaling_factor;
    }
    for (int k = 0; k < cfg.extra_iters_at_final_eps && out.size() < cap; ++k) out.push_back(cfg.eps);
    return out;
}

void rng_normal_fill(uint64_t seed, double* out, int64_t count) {
    fsk::Rng rng(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = rng.normal();
}

double cascade_sum(const double* a, std::size_t n) {
    if (n == 0) return 0.0;
    if (n <= 8) {
        double s = a[0];
        for (std::size_t i = 1; i < n; ++i) s += a[i];
        return s;
    }
    const std::size_t h = n / 2;
    return cascade_sum(a, h) + cascade_sum(a + h, n - h);
}

}  // namespace fskb
