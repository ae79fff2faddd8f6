// fsk::solver, fsk::autodiff, fsk::hvp on the B200 (include/fsk/*.hpp).
#include "../../../include/fsk/solver.hpp"

#include "../../../include/fsk/autodiff.hpp"
#include "../../../include/fsk/devices.hpp"
#include "../../../include/fsk/hvp.hpp"
#include "../hostlib.h"
#include "bridge.h"

namespace fsk {

namespace {
void check_pots(const ShiftedPotentials& p, std::size_t n, std::size_t m) {
    if (p.f_hat.size() != n || p.g_hat.size() != m)
        throw ValidationError("potential lengths do not match the measures");
}
}  // namespace

void set_num_devices(int n) { bridge::check(fsk_set_num_devices(n)); }
int num_devices() { return fsk_num_devices(); }

namespace solver {

SolveReport sinkhorn_solve(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
                           const CostSpec& spec, const SinkhornConfig& cfg,
                           const TileConfig& tiles, IoLedger& ledger) {
    validate_problem(src, tgt, spec);
    validate_sinkhorn_config(cfg);
    validate_tiles(tiles);
    const fsk_measure a = bridge::view(src), b = bridge::view(tgt);
    const fsk_cost c = bridge::view(spec);
    const fsk_tiles t = bridge::view(tiles);
    const fsk_config k = bridge::view(cfg);
    bridge::LedgerScope led(ledger);
    SolveReport rep;
    rep.potentials.f_hat.resize(src.size());
    rep.potentials.g_hat.resize(tgt.size());
    std::vector<double> hist(std::size_t(cfg.max_iters));
    fsk_report r{rep.potentials.f_hat.data(), rep.potentials.g_hat.data(), hist.data(),
                 int64_t(hist.size()), 0, 0.0, 0.0, 0.0};
    bridge::check(fsk_sinkhorn_solve(&a, &b, &c, &k, &t, led.get(), &r));
    rep.iterations = r.iterations;
    rep.marginal_violation = r.marginal_violation;
    rep.dual_cost = r.dual_cost;
    rep.potentials.eps = r.eps;
    hist.resize(std::size_t(r.iterations));
    rep.eps_history = std::move(hist);
    return rep;
}

SolveReport sinkhorn_solve_warm(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
                                const CostSpec& spec, const SinkhornConfig& cfg,
                                const TileConfig& tiles, IoLedger& ledger,
                                const ShiftedPotentials& init) {
    validate_problem(src, tgt, spec);
    validate_sinkhorn_config(cfg);
    validate_tiles(tiles);
    check_pots(init, src.size(), tgt.size());
    const fsk_measure a = bridge::view(src), b = bridge::view(tgt);
    const fsk_cost c = bridge::view(spec);
    const fsk_tiles t = bridge::view(tiles);
    const fsk_config k = bridge::view(cfg);
    bridge::LedgerScope led(ledger);
    SolveReport rep;
    rep.potentials.f_hat.resize(src.size());
    rep.potentials.g_hat.resize(tgt.size());
    std::vector<double> hist(std::size_t(cfg.max_iters));
    fsk_report r{rep.potentials.f_hat.data(), rep.potentials.g_hat.data(), hist.data(),
                 int64_t(hist.size()), 0, 0.0, 0.0, 0.0};
    bridge::check(fsk_sinkhorn_solve_warm(&a, &b, &c, &k, &t, led.get(), init.f_hat.data(),
                                          init.g_hat.data(), &r, nullptr));
    rep.iterations = r.iterations;
    rep.marginal_violation = r.marginal_violation;
    rep.dual_cost = r.dual_cost;
    rep.potentials.eps = r.eps;
    hist.resize(std::size_t(r.iterations));
    rep.eps_history = std::move(hist);
    return rep;
}

double dual_cost(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
                 const ShiftedPotentials& p, const CostSpec& spec, const TileConfig& tiles,
                 IoLedger& ledger) {
    validate_problem(src, tgt, spec);
    validate_tiles(tiles);
    check_pots(p, src.size(), tgt.size());
    const fsk_measure a = bridge::view(src), b = bridge::view(tgt);
    const fsk_cost c = bridge::view(spec);
    const fsk_tiles t = bridge::view(tiles);
    bridge::LedgerScope led(ledger);
    double out = 0.0;
    bridge::check(fsk_dual_cost(&a, &b, p.f_hat.data(), p.g_hat.data(), p.eps, &c, &t, led.get(),
                                &out));
    return out;
}

double sinkhorn_divergence_mixed(const DiscreteMeasure& mu, const DiscreteMeasure& nu,
                                 const CostSpec& spec_cross, const CostSpec& spec_mu,
                                 const CostSpec& spec_nu, const SinkhornConfig& cfg,
                                 const TileConfig& tiles, IoLedger& ledger) {
    validate_problem(mu, nu, spec_cross);
    validate_problem(mu, mu, spec_mu);
    validate_problem(nu, nu, spec_nu);
    validate_sinkhorn_config(cfg);
    validate_tiles(tiles);
    const fsk_measure a = bridge::view(mu), b = bridge::view(nu);
    const fsk_cost cx = bridge::view(spec_cross), cm = bridge::view(spec_mu),
                   cn = bridge::view(spec_nu);
    const fsk_tiles t = bridge::view(tiles);
    const fsk_config k = bridge::view(cfg);
    bridge::LedgerScope led(ledger);
    double out = 0.0;
    bridge::check(fsk_sinkhorn_divergence_mixed(&a, &b, &cx, &cm, &cn, &k, &t, led.get(), &out));
    return out;
}

double sinkhorn_divergence(const DiscreteMeasure& mu, const DiscreteMeasure& nu,
                           const CostSpec& spec, const SinkhornConfig& cfg,
                           const TileConfig& tiles, IoLedger& ledger) {
    return sinkhorn_divergence_mixed(mu, nu, spec, spec, spec, cfg, tiles, ledger);
}

}  // namespace solver

namespace autodiff {

namespace {
using AdFn = int (*)(const fsk_measure*, const fsk_measure*, const double*, const double*, double,
                     const fsk_cost*, const fsk_tiles*, fsk_ledger*, double*);

Mat run(AdFn fn, std::size_t rows, const DiscreteMeasure& src, const DiscreteMeasure& tgt,
        const ShiftedPotentials& p, const CostSpec& spec, const TileConfig& tiles,
        IoLedger& ledger) {
    validate_problem(src, tgt, spec);
    validate_tiles(tiles);
    check_pots(p, src.size(), tgt.size());
    const fsk_measure a = bridge::view(src), b = bridge::view(tgt);
    const fsk_cost c = bridge::view(spec);
    const fsk_tiles t = bridge::view(tiles);
    bridge::LedgerScope led(ledger);
    Mat out(rows, src.dim());
    bridge::check(fn(&a, &b, p.f_hat.data(), p.g_hat.data(), p.eps, &c, &t, led.get(),
                     out.data()));
    return out;
}
}  // namespace

Mat barycentric_projection(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
                           const ShiftedPotentials& p, const CostSpec& spec,
                           const TileConfig& tiles, IoLedger& ledger) {
    return run(fsk_barycentric_projection, src.size(), src, tgt, p, spec, tiles, ledger);
}

Mat grad_source(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
                const ShiftedPotentials& p, const CostSpec& spec, const TileConfig& tiles,
                IoLedger& ledger) {
    return run(fsk_grad_source, src.size(), src, tgt, p, spec, tiles, ledger);
}

Mat grad_target(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
                const ShiftedPotentials& p, const CostSpec& spec, const TileConfig& tiles,
                IoLedger& ledger) {
    return run(fsk_grad_target, tgt.size(), src, tgt, p, spec, tiles, ledger);
}

}  // namespace autodiff

namespace hvp {

HvpResult hvp_apply(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
                    const ShiftedPotentials& p, const CostSpec& spec, const Mat& A,
                    const HvpConfig& cfg, const TileConfig& tiles, IoLedger& ledger) {
    validate_problem(src, tgt, spec);
    validate_tiles(tiles);
    check_pots(p, src.size(), tgt.size());
    if (A.rows() != src.size() || A.cols() != src.dim())
        throw ValidationError("hvp: direction shape mismatch");
    const fsk_measure a = bridge::view(src), b = bridge::view(tgt);
    const fsk_cost c = bridge::view(spec);
    const fsk_tiles t = bridge::view(tiles);
    const fsk_hvp_config h{cfg.tau, cfg.cg_tol, cfg.cg_max_iters};
    bridge::LedgerScope led(ledger);
    HvpResult res;
    res.value = Mat(src.size(), src.dim());
    fsk_hvp_report rep{};
    bridge::check(fsk_hvp_apply(&a, &b, p.f_hat.data(), p.g_hat.data(), p.eps, &c, A.data(), &h,
                                &t, led.get(), res.value.data(), &rep));
    res.cg_iters = rep.cg_iters;
    res.cg_rel_residual = rep.cg_rel_residual;
    res.converged = rep.converged != 0;
    return res;
}

}  // namespace hvp
}  // namespace fsk
