// placeholder: replaced by the tcgen05 implementation
#include "device_ops.h"
#include "tc_engine.h"

namespace fskb {

struct TcHalfStep::Impl {};

bool TcHalfStep::supported(int64_t) { return false; }
TcHalfStep::TcHalfStep(DevProblem<float>&) : impl_(nullptr) {}
TcHalfStep::~TcHalfStep() {}
void TcHalfStep::set_eps(DevProblem<float>&, double) {}
void TcHalfStep::run(DevProblem<float>&, int, const float*, float, const FinalizeArgs<float>&,
                     int64_t, int64_t) {
    throw CudaFailure("tensor path unavailable");
}

bool enable_tensor_path(DevProblem<float>& P, int mode) {
    (void)P;
    (void)mode;
    return false;
}

const char* tensor_path_name(const DevProblem<float>& P) {
    return P.tc ? "tcgen05-split3" : "fma-f32";
}

}  // namespace fskb
