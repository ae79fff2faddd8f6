// fsk::autodiff - SPEC.md "autodiff" module, specified by
// the reference but never implemented there (SURVEY.md finding 5). Provided by
// the B200 library as fused streaming kernels (one LSE pass + one transport
// pass, no n x m buffer). Induced-marginal form throughout.
#pragma once

#include "fsk/core.hpp"
#include "fsk/ledger.hpp"

namespace fsk::autodiff {

// T = diag(r)^-1 P Y  (softmax-weighted target average per source point)
Mat barycentric_projection(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
                           const ShiftedPotentials& p, const CostSpec& spec,
                           const TileConfig& tiles, IoLedger& ledger);

// grad_X OT = 2 (diag(r) X - P Y)
Mat grad_source(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
                const ShiftedPotentials& p, const CostSpec& spec, const TileConfig& tiles,
                IoLedger& ledger);

// grad_Y OT = 2 (diag(c) Y - P^T X)
Mat grad_target(const DiscreteMeasure& src, const DiscreteMeasure& tgt,
                const ShiftedPotentials& p, const CostSpec& spec, const TileConfig& tiles,
                IoLedger& ledger);

}  // namespace fsk::autodiff
