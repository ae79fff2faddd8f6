// Conversions between the C++ drop-in types (include/fsk/*.hpp) and the C ABI
// (include/fsk_b200.h), and status -> exception mapping.
#pragma once

#include <string>

#include "../../../include/fsk/core.hpp"
#include "../../../include/fsk/ledger.hpp"
#include "../../../include/fsk_b200.h"

namespace fsk::bridge {

inline fsk_measure view(const DiscreteMeasure& m) {
    return fsk_measure{m.points.data(), m.weights.data(),
                       m.labels ? m.labels->data() : nullptr, int64_t(m.points.rows()),
                       int64_t(m.points.cols())};
}

inline fsk_cost view(const CostSpec& c) {
    if (c.kind != CostKind::LabelAugmented) return fsk_cost{0, 1.0, 0.0, nullptr, 0};
    return fsk_cost{1, c.lambda1, c.lambda2, c.label_cost.data(), int64_t(c.label_cost.rows())};
}

inline fsk_tiles view(const TileConfig& t) {
    return fsk_tiles{int64_t(t.block_rows), int64_t(t.block_cols)};
}

inline fsk_config view(const SinkhornConfig& c) {
    return fsk_config{c.eps,
                      c.schedule == Schedule::Symmetric ? 1 : 0,
                      c.max_iters,
                      c.marginal_tol,
                      c.eps_scaling_factor,
                      c.extra_iters_at_final_eps,
                      c.precision == Precision::Double ? 1 : 0};
}

// Adds the C-ABI counters into the (atomic) IoLedger.
struct LedgerScope {
    explicit LedgerScope(IoLedger& l) : led(l) {}
    ~LedgerScope() {
        led.slow_to_fast_scalars.fetch_add(raw.slow_to_fast_scalars);
        led.fast_to_slow_scalars.fetch_add(raw.fast_to_slow_scalars);
        led.kernel_invocations.fetch_add(raw.kernel_invocations);
        led.transport_vector_applies.fetch_add(raw.transport_vector_applies);
        led.transport_matrix_applies.fetch_add(raw.transport_matrix_applies);
        led.hadamard_applies.fetch_add(raw.hadamard_applies);
    }
    fsk_ledger* get() { return &raw; }
    IoLedger& led;
    fsk_ledger raw{};
};

inline void check(int status) {
    if (status == FSK_OK) return;
    const std::string msg = fsk_last_error();
    if (status == FSK_EVALIDATION) throw ValidationError(msg);
    if (status == FSK_ENUMERICAL) throw NumericalError(msg);
    throw std::runtime_error("fsk_b200 device failure: " + msg);
}

// shape checks the C ABI cannot see (it receives one n per measure)
inline void check_measure_shapes(const DiscreteMeasure& m) {
    const std::size_t n = m.points.rows();
    if (n >= 1 && m.points.cols() >= 1 && m.weights.size() != n)
        throw ValidationError("weight count " + std::to_string(m.weights.size()) +
                              " does not match point count " + std::to_string(n));
    if (m.labels && m.labels->size() != n)
        throw ValidationError("label count does not match point count");
}

inline void check_spec_shape(const CostSpec& spec) {
    if (spec.kind == CostKind::LabelAugmented && spec.label_cost.cols() != spec.label_cost.rows())
        throw ValidationError("label cost table must be square");
}

}  // namespace fsk::bridge
