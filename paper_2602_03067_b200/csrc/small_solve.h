// Persistent small-problem Sinkhorn loop (small_solve.cu): all iterations of an
// alternating fp32 solve in one cooperative launch, for problems whose key side
// fits in shared memory (cfg1-class: n, m ~ 4096, d <= 16).
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace fskb {

constexpr int kSmallSolveMaxD = 16;
constexpr std::size_t kSmallSolveSmem = 192 * 1024;
constexpr std::size_t kSmallSolveResSmem = 220 * 1024;   // resident-cloud variant

struct SmallSolveParams {
    const float* X;        // n x d row-major
    const float* Y;        // m x d row-major
    const float* logw_x;   // log a (n)
    const float* logw_y;   // log b (m)
    float* f;              // shifted potentials, in/out
    float* g;
    const float* eps_sched;  // device, one eps per iteration
    int iters;
    int iter0;             // iteration number of the first (for bad_iter reports)
    int64_t n, m;
    int d;
    int64_t cpad;          // set by the launcher
    int64_t npad, mpad;    // set by the launcher (resident variant)
    float fscale;          // feature scale s (1 for the squared-Euclidean cost)
    int* flags;
    int* bad_iter;         // nullable
};

bool small_solve_fits(int64_t n, int64_t m, int64_t d);
void launch_small_solve(const SmallSolveParams& p, cudaStream_t s);

}  // namespace fskb
