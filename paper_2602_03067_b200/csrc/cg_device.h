// Device-resident conjugate-gradient vector algebra for the HVP's Schur system
// (cg_solve of hvp.hvp_apply). The iterate, residual and search
// direction stay in HBM (fp64); dot products are fixed-order two-stage
// reductions (run-to-run bit-identical); the host reads one scalar per
// iteration (the new residual norm) to decide termination.
#pragma once

#include <cstdint>

#include "common.h"

namespace fskb {

struct DeviceCg {
    int64_t m = 0;
    cudaStream_t s = nullptr;
    DevBuf<double> w2, res, pdir, ap, partial, scal;   // scal: [rs0, rs1, pAp]
    DevBuf<float> pf;                                   // fp32 copy of pdir (transport input)
    double* h_rs = nullptr;                             // pinned: the last rs_new
    int k = 0;                                          // iteration parity

    DeviceCg(int64_t m_, cudaStream_t s_);
    ~DeviceCg();
    DeviceCg(const DeviceCg&) = delete;
    DeviceCg& operator=(const DeviceCg&) = delete;

    // res = pdir = rhs, w2 = 0; returns <rhs, rhs> (synchronizes)
    double init(const double* rhs_dev);
    // tmpf_i = float(pv_i / r_i)  (P p scaled by diag(r)^-1 for the P^T pass)
    void div_rows(const double* pv, const float* r, int64_t n, float* tmpf);
    // Ap = c p - ptq + tau p; alpha = rs / <p, Ap>; w2 += alpha p; res -= alpha Ap;
    // returns rs_new = <res, res> (one synchronize)
    double step(const float* c, const double* ptq, double tau);
    // pdir = res + (rs_new / rs) pdir (and its fp32 copy); advances the parity
    void direction();
};

}  // namespace fskb
