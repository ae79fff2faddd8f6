// fsk::stream on the B200 (include/fsk/stream.hpp). Argument checks happen in
// the reference's order (stream.cpp:270-375), then the C ABI runs the kernels.
#include "../../../include/fsk/stream.hpp"

#include <cmath>

#include "../hostlib.h"
#include "bridge.h"

namespace fsk::stream {

namespace {

void check_pots(const ShiftedPotentials& p, std::size_t n, std::size_t m) {
    if (p.f_hat.size() != n || p.g_hat.size() != m)
        throw ValidationError("potential lengths do not match the measures");
    if (!(p.eps > 0.0)) throw ValidationError("potentials carry nonpositive eps");
    if (!fskb::all_finite(p.f_hat.data(), int64_t(n)) ||
        !fskb::all_finite(p.g_hat.data(), int64_t(m)))
        throw ValidationError("non-finite potential entry");
}

void prelude(const DiscreteMeasure& src, const DiscreteMeasure& tgt, const CostSpec& spec,
             const TileConfig& tiles) {
    validate_problem(src, tgt, spec);
    validate_tiles(tiles);
}

}  // namespace

Vec update_f_hat(const DiscreteMeasure& src, const DiscreteMeasure& tgt, const Vec& g_hat,
                 const CostSpec& spec, double eps, const TileConfig& tiles, IoLedger& ledger) {
    prelude(src, tgt, spec, tiles);
    if (!(eps > 0.0)) throw ValidationError("eps must be positive");
    if (g_hat.size() != tgt.size()) throw ValidationError("g_hat length mismatch");
    const fsk_measure a = bridge::view(src), b = bridge::view(tgt);
    const fsk_cost c = bridge::view(spec);
    const fsk_tiles t = bridge::view(tiles);
    bridge::LedgerScope led(ledger);
    Vec out(src.size());
    bridge::check(fsk_update_f_hat(&a, &b, g_hat.data(), &c, eps, &t, led.get(), out.data()));
    return out;
}

Vec update_g_hat(const DiscreteMeasure& src, const DiscreteMeasure& tgt, const Vec& f_hat,
                 const CostSpec& spec, double eps, const TileConfig& tiles, IoLedger& ledger) {
    prelude(src, tgt, spec, tiles);
    if (!(eps > 0.0)) throw ValidationError("eps must be positive");
    if (f_hat.size() != src.size()) throw ValidationError("f_hat length mismatch");
    const fsk_measure a = bridge::view(src), b = bridge::view(tgt);
    const fsk_cost c = bridge::view(spec);
    const fsk_tiles t = bridge::view(tiles);
    bridge::LedgerScope led(ledger);
    Vec out(tgt.size());
    bridge::check(fsk_update_g_hat(&a, &b, f_hat.data(), &c, eps, &t, led.get(), out.data()));
    return out;
}

ShiftedPotentials symmetric_update(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
                                   const ShiftedPotentials& p, const CostSpec& spec,
                                   const TileConfig& tiles, IoLedger& ledger) {
    prelude(src, tgt, spec, tiles);
    check_pots(p, src.size(), tgt.size());
    const fsk_measure a = bridge::view(src), b = bridge::view(tgt);
    const fsk_cost c = bridge::view(spec);
    const fsk_tiles t = bridge::view(tiles);
    bridge::LedgerScope led(ledger);
    ShiftedPotentials out;
    out.eps = p.eps;
    out.f_hat.resize(src.size());
    out.g_hat.resize(tgt.size());
    bridge::check(fsk_symmetric_update(&a, &b, p.f_hat.data(), p.g_hat.data(), p.eps, &c, &t,
                                       led.get(), out.f_hat.data(), out.g_hat.data()));
    return out;
}

Mat apply_plan(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
               const ShiftedPotentials& p, const CostSpec& spec, const Mat& V,
               const TileConfig& tiles, IoLedger& ledger) {
    prelude(src, tgt, spec, tiles);
    check_pots(p, src.size(), tgt.size());
    if (V.rows() != tgt.size()) throw ValidationError("apply_plan: V row count != m");
    const fsk_measure a = bridge::view(src), b = bridge::view(tgt);
    const fsk_cost c = bridge::view(spec);
    const fsk_tiles t = bridge::view(tiles);
    bridge::LedgerScope led(ledger);
    Mat out(src.size(), V.cols());
    bridge::check(fsk_apply_plan(&a, &b, p.f_hat.data(), p.g_hat.data(), p.eps, &c, V.data(),
                                 int64_t(V.cols()), &t, led.get(), out.data()));
    return out;
}

Mat apply_plan_adjoint(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
                       const ShiftedPotentials& p, const CostSpec& spec, const Mat& U,
                       const TileConfig& tiles, IoLedger& ledger) {
    prelude(src, tgt, spec, tiles);
    check_pots(p, src.size(), tgt.size());
    if (U.rows() != src.size()) throw ValidationError("apply_plan_adjoint: U row count != n");
    const fsk_measure a = bridge::view(src), b = bridge::view(tgt);
    const fsk_cost c = bridge::view(spec);
    const fsk_tiles t = bridge::view(tiles);
    bridge::LedgerScope led(ledger);
    Mat out(tgt.size(), U.cols());
    bridge::check(fsk_apply_plan_adjoint(&a, &b, p.f_hat.data(), p.g_hat.data(), p.eps, &c,
                                         U.data(), int64_t(U.cols()), &t, led.get(), out.data()));
    return out;
}

Mat apply_hadamard_plan(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
                        const ShiftedPotentials& p, const CostSpec& spec, const Mat& A,
                        const Mat& B, const Mat& V, const TileConfig& tiles, IoLedger& ledger) {
    prelude(src, tgt, spec, tiles);
    check_pots(p, src.size(), tgt.size());
    if (A.rows() != src.size() || B.rows() != tgt.size() || A.cols() != B.cols())
        throw ValidationError("apply_hadamard_plan: weight factor shape mismatch");
    if (A.cols() < 1) throw ValidationError("apply_hadamard_plan: rank factor r must be >= 1");
    if (V.rows() != tgt.size()) throw ValidationError("apply_hadamard_plan: V row count != m");
    const fsk_measure a = bridge::view(src), b = bridge::view(tgt);
    const fsk_cost c = bridge::view(spec);
    const fsk_tiles t = bridge::view(tiles);
    bridge::LedgerScope led(ledger);
    Mat out(src.size(), V.cols());
    bridge::check(fsk_apply_hadamard_plan(&a, &b, p.f_hat.data(), p.g_hat.data(), p.eps, &c,
                                          A.data(), B.data(), int64_t(A.cols()), V.data(),
                                          int64_t(V.cols()), &t, led.get(), out.data()));
    return out;
}

std::pair<Vec, Vec> induced_marginals(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
                                      const ShiftedPotentials& p, const CostSpec& spec,
                                      const TileConfig& tiles, IoLedger& ledger) {
    prelude(src, tgt, spec, tiles);
    check_pots(p, src.size(), tgt.size());
    const fsk_measure a = bridge::view(src), b = bridge::view(tgt);
    const fsk_cost c = bridge::view(spec);
    const fsk_tiles t = bridge::view(tiles);
    bridge::LedgerScope led(ledger);
    Vec r(src.size()), cc(tgt.size());
    bridge::check(fsk_induced_marginals(&a, &b, p.f_hat.data(), p.g_hat.data(), p.eps, &c, &t,
                                        led.get(), r.data(), cc.data()));
    return {std::move(r), std::move(cc)};
}

FloatCloud to_float_cloud(const DiscreteMeasure& m) {
    FloatCloud f;
    f.n = m.size();
    f.d = m.dim();
    f.points.resize(f.n * f.d);
    for (std::size_t i = 0; i < f.points.size(); ++i) f.points[i] = float(m.points.data()[i]);
    f.weights.resize(f.n);
    for (std::size_t i = 0; i < f.n; ++i) f.weights[i] = float(m.weights[i]);
    return f;
}

std::vector<float> update_f_hat_f32(const FloatCloud& src, const FloatCloud& tgt,
                                    const std::vector<float>& g_hat, float eps,
                                    const TileConfig& tiles, IoLedger& ledger) {
    const fsk_tiles t = bridge::view(tiles);
    bridge::LedgerScope led(ledger);
    std::vector<float> out(src.n);
    bridge::check(fsk_update_f_hat_f32(src.points.data(), src.weights.data(), int64_t(src.n),
                                       tgt.points.data(), tgt.weights.data(), int64_t(tgt.n),
                                       int64_t(src.d), g_hat.data(), eps, &t, led.get(),
                                       out.data()));
    return out;
}

std::vector<float> update_g_hat_f32(const FloatCloud& src, const FloatCloud& tgt,
                                    const std::vector<float>& f_hat, float eps,
                                    const TileConfig& tiles, IoLedger& ledger) {
    const fsk_tiles t = bridge::view(tiles);
    bridge::LedgerScope led(ledger);
    std::vector<float> out(tgt.n);
    bridge::check(fsk_update_g_hat_f32(src.points.data(), src.weights.data(), int64_t(src.n),
                                       tgt.points.data(), tgt.weights.data(), int64_t(tgt.n),
                                       int64_t(src.d), f_hat.data(), eps, &t, led.get(),
                                       out.data()));
    return out;
}

uint64_t io_count_f_update(std::size_t n, std::size_t m, std::size_t d, const TileConfig& tiles) {
    const fsk_tiles t = bridge::view(tiles);
    return fsk_io_count_f_update(int64_t(n), int64_t(m), int64_t(d), &t);
}
uint64_t io_count_g_update(std::size_t n, std::size_t m, std::size_t d, const TileConfig& tiles) {
    const fsk_tiles t = bridge::view(tiles);
    return fsk_io_count_g_update(int64_t(n), int64_t(m), int64_t(d), &t);
}
uint64_t io_count_symmetric_update(std::size_t n, std::size_t m, std::size_t d,
                                   const TileConfig& tiles) {
    const fsk_tiles t = bridge::view(tiles);
    return fsk_io_count_symmetric_update(int64_t(n), int64_t(m), int64_t(d), &t);
}
uint64_t io_count_apply_plan(std::size_t n, std::size_t m, std::size_t d, std::size_t p,
                             const TileConfig& tiles) {
    const fsk_tiles t = bridge::view(tiles);
    return fsk_io_count_apply_plan(int64_t(n), int64_t(m), int64_t(d), int64_t(p), &t);
}
uint64_t io_count_apply_plan_adjoint(std::size_t n, std::size_t m, std::size_t d, std::size_t p,
                                     const TileConfig& tiles) {
    const fsk_tiles t = bridge::view(tiles);
    return fsk_io_count_apply_plan_adjoint(int64_t(n), int64_t(m), int64_t(d), int64_t(p), &t);
}
uint64_t io_count_apply_hadamard(std::size_t n, std::size_t m, std::size_t d, std::size_t r,
                                 std::size_t p, const TileConfig& tiles) {
    const fsk_tiles t = bridge::view(tiles);
    return fsk_io_count_apply_hadamard(int64_t(n), int64_t(m), int64_t(d), int64_t(r), int64_t(p),
                                       &t);
}
uint64_t io_count_induced_marginals(std::size_t n, std::size_t m, std::size_t d,
                                    const TileConfig& tiles) {
    const fsk_tiles t = bridge::view(tiles);
    return fsk_io_count_induced_marginals(int64_t(n), int64_t(m), int64_t(d), &t);
}

bool tiles_fit_sram(const TileConfig& tiles, std::size_t d, std::size_t sram_scalars) {
    const fsk_tiles t = bridge::view(tiles);
    return fsk_tiles_fit_sram(&t, int64_t(d), int64_t(sram_scalars)) != 0;
}

void debug_break_lse(bool broken) { fsk_debug_break_lse(broken ? 1 : 0); }

}  // namespace fsk::stream
