// Host-side pieces shared by the C ABI (capi.cpp) and the C++ drop-in API
// (api/*.cpp): input validation with the reference's messages, the IO-ledger
// closed forms, the eps schedule, and the seeded generator.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/fsk_b200.h"

namespace fskb {

// ---- validation (proj/src/core.cpp:18-81, stream.cpp:253-259) -------------
// check_points = false skips the coordinate finiteness scan (a caller that checks it
// elsewhere, e.g. on the device after the upload, and throws the same message)
void validate_measure_raw(const fsk_measure& m, bool check_points = true);
// measures_checked: validate_measure_raw already ran on both (batch entry points)
void validate_problem_raw(const fsk_measure& src, const fsk_measure& tgt, const fsk_cost* cost,
                          bool measures_checked = false, bool check_points = true);
inline constexpr const char* kNonFiniteCoordinate = "non-finite coordinate in measure";
void validate_config_raw(const fsk_config& cfg);
void validate_tiles_raw(const fsk_tiles* tiles);
bool all_finite(const double* p, int64_t n);
void check_potentials_raw(const double* f, int64_t n, const double* g, int64_t m, double eps);

inline bool labeled_cost(const fsk_cost* c) { return c && c->kind == 1; }
inline double feature_scale(const fsk_cost* c) { return labeled_cost(c) ? c->lambda1 : 1.0; }

// ---- ledger closed forms (stream.cpp:93-136 / :140-207 increments) --------
// Totals of the reference's per-block add_load/add_store calls, valid for any
// tile shape (ragged blocks included) and for labeled costs.
struct Counts {
    uint64_t load = 0, store = 0;
};
Counts lse_counts(int64_t R, int64_t C, int64_t d, int64_t br, int64_t bc, bool labeled);
Counts apply_counts(int64_t R, int64_t C, int64_t d, int64_t p, int64_t r, int64_t br, int64_t bc,
                    bool labeled);
void ledger_add(fsk_ledger* l, const Counts& c);

// Per-operation accounting exactly as the reference's public ops increment it.
void ledger_update_f(fsk_ledger* l, int64_t n, int64_t m, int64_t d, const fsk_tiles& t,
                     const fsk_cost* cost);
void ledger_update_g(fsk_ledger* l, int64_t n, int64_t m, int64_t d, const fsk_tiles& t,
                     const fsk_cost* cost);
void ledger_symmetric(fsk_ledger* l, int64_t n, int64_t m, int64_t d, const fsk_tiles& t,
                      const fsk_cost* cost);
void ledger_apply(fsk_ledger* l, int64_t n, int64_t m, int64_t d, int64_t p, const fsk_tiles& t,
                  const fsk_cost* cost, bool adjoint);
void ledger_hadamard(fsk_ledger* l, int64_t n, int64_t m, int64_t d, int64_t r, int64_t p,
                     const fsk_tiles& t, const fsk_cost* cost);
void ledger_marginals(fsk_ledger* l, int64_t n, int64_t m, int64_t d, const fsk_tiles& t,
                      const fsk_cost* cost);
void ledger_update_f32(fsk_ledger* l, int64_t R, int64_t C, int64_t d, int64_t br, int64_t bc);

// ---- schedule (proj/src/schedule.cpp) ------------------------------------
double joint_sq_diameter_raw(const double* X, int64_t n, const double* Y, int64_t m, int64_t d);
std::vector<double> eps_schedule_raw(const fsk_config& cfg, double sq_diam);

// ---- seeded generator (proj/include/fsk/rng.hpp) --------------------------
void rng_normal_fill(uint64_t seed, double* out, int64_t count);

// cascade sum with the reference's association (<= 8 sequential, split n/2)
double cascade_sum(const double* a, std::size_t n);

}  // namespace fskb
