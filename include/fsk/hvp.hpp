// fsk::hvp - SPEC.md "hvp" module (Thm. 3.5),
// specified by the reference but never implemented there. Streaming
// Hessian-vector product of OT_eps w.r.t. the source points: explicit term via
// one Hadamard-weighted transport, implicit term via damped Schur-complement CG
// over transport-vector products. O((n + m) d) memory, never n x m (the opt-in
// FSK_PLAN_CACHE=1 plan-block cache of the single-precision path trades that
// contract for speed; it is off by default).
#pragma once

#include "fsk/core.hpp"
#include "fsk/ledger.hpp"

namespace fsk::hvp {

struct HvpConfig {
    double tau = 1e-5;      // Schur damping
    double cg_tol = 1e-6;   // relative residual target
    int cg_max_iters = 50;  // K_CG
};

struct HvpResult {
    Mat value;              // n x d
    int cg_iters = 0;
    double cg_rel_residual = 0.0;
    bool converged = false;
};

HvpResult hvp_apply(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
                    const ShiftedPotentials& p, const CostSpec& spec, const Mat& A,
                    const HvpConfig& cfg, const TileConfig& tiles, IoLedger& ledger);

}  // namespace fsk::hvp
