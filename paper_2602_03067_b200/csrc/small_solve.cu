// Persistent small-problem Sinkhorn loop (CUDA-core FP32, d <= 16): the whole
// alternating iteration sequence of sinkhorn_solve (solver.cpp:36-48; the f32
// loop of solver.cpp:69-117) in ONE cooperative launch. cfg1 (n = m = 4096,
// d = 3) is launch-bound: its half-step is ~4 us of MUFU work, while a graph of
// per-half-step LSE + finalize kernels costs ~49 us per half-step in launch
// gaps. Here every half-step is
//   stage:  all keys of the side (pre-scaled by 2/eps, SoA) + their bias
//           (pot_j + eps log w_j)/eps into shared memory (<= 192 KB)
//   rows:   one warp per query row, lanes stride the keys; pass 1 row max,
//           pass 2 sum of exp(s - max) (one exp per score, no online rescale),
//           warp reductions; f_i = -eps (max + log sum)
//   sync:   grid-wide barrier, then the other side reads the new potential.
// Scores are formed exactly as the FP32 tile kernel does (fma over features in
// order, then + bias), so the result differs from the per-launch path only in
// the LSE summation order (fp32 contract of SURVEY §8d).
#include <cooperative_groups.h>

#include "common.h"
#include "small_solve.h"

namespace cg = cooperative_groups;

namespace fskb {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = 32 * kWarps;

template <int D>
__global__ void __launch_bounds__(kThreads, 1) small_solve_kernel(const SmallSolveParams p) {
    extern __shared__ __align__(16) float sm[];
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t cpad = p.cpad;
    for (int it = 0; it < p.iters; ++it) {
        const float eps = p.eps_sched[it];
        const float kscale = 2.0f * p.fscale / eps;
        for (int side = 0; side < 2; ++side) {
            const float* Q = side == 0 ? p.X : p.Y;
            const float* K = side == 0 ? p.Y : p.X;
            const float* kpot = side == 0 ? p.g : p.f;
            const float* klogw = side == 0 ? p.logw_y : p.logw_x;
            float* out = side == 0 ? p.f : p.g;
            const int64_t R = side == 0 ? p.n : p.m;
            const int64_t C = side == 0 ? p.m : p.n;
            // stage the keys (SoA, x 2/eps) and their bias
            for (int64_t j = threadIdx.x; j < C; j += kThreads) {
#pragma unroll
                for (int t = 0; t < D; ++t) sm[t * cpad + j] = K[j * D + t] * kscale;
                sm[D * cpad + j] = (kpot[j] + eps * klogw[j]) / eps;
            }
            __syncthreads();
            for (int64_t r = int64_t(blockIdx.x) * kWarps + warp; r < R;
                 r += int64_t(gridDim.x) * kWarps) {
                float q[D];
#pragma unroll
                for (int t = 0; t < D; ++t) q[t] = Q[r * D + t];
                float mx = -INFINITY;
                for (int64_t j = lane; j < C; j += 32) {
                    float acc = 0.0f;
#pragma unroll
                    for (int t = 0; t < D; ++t) acc = fmaf(q[t], sm[t * cpad + j], acc);
                    mx = fmaxf(mx, acc + sm[D * cpad + j]);
                }
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1)
                    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
                float sum = 0.0f;
                for (int64_t j = lane; j < C; j += 32) {
                    float acc = 0.0f;
#pragma unroll
                    for (int t = 0; t < D; ++t) acc = fmaf(q[t], sm[t * cpad + j], acc);
                    sum += __expf(acc + sm[D * cpad + j] - mx);
                }
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1)
                    sum += __shfl_xor_sync(0xffffffffu, sum, off);
                if (lane == 0) {
                    const float pot = -eps * (mx + logf(sum));
                    if (!isfinite(pot)) {
                        atomicOr(p.flags, kFlagNonFinitePotential);
                        if (p.bad_iter) atomicMin(p.bad_iter, p.iter0 + it + 1);
                    }
                    out[r] = pot;
                }
            }
            // the other side stages this side's new potential next
            grid.sync();
        }
    }
}

template <int D>
void launch_d(const SmallSolveParams& p, int grid, size_t smem, cudaStream_t s) {
    static bool configured = false;
    if (!configured) {
        FSKB_CUDA(cudaFuncSetAttribute(small_solve_kernel<D>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kSmallSolveSmem)));
        configured = true;
    }
    SmallSolveParams q = p;
    void* args[] = {&q};
    FSKB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(small_solve_kernel<D>),
                                          dim3(unsigned(grid)), dim3(kThreads), args, smem, s));
}

}  // namespace

bool small_solve_fits(int64_t n, int64_t m, int64_t d) {
    if (d < 1 || d > kSmallSolveMaxD || n < 1 || m < 1) return false;
    const int64_t cmax = n > m ? n : m;
    const int64_t cpad = (cmax + 3) / 4 * 4;
    return size_t(cpad) * size_t(d + 1) * sizeof(float) <= kSmallSolveSmem;
}

void launch_small_solve(const SmallSolveParams& p0, cudaStream_t s) {
    if (p0.iters < 1) return;
    SmallSolveParams p = p0;
    const int64_t cmax = p.n > p.m ? p.n : p.m;
    p.cpad = (cmax + 3) / 4 * 4;
    const size_t smem = size_t(p.cpad) * size_t(p.d + 1) * sizeof(float);
    // one CTA per SM (co-residency is what the grid barrier needs)
    const int grid = num_sms();
    switch (p.d) {
#define FSKB_SMALL_CASE(DD) \
    case DD:                \
        launch_d<DD>(p, grid, smem, s); \
        break;
        FSKB_SMALL_CASE(1) FSKB_SMALL_CASE(2) FSKB_SMALL_CASE(3) FSKB_SMALL_CASE(4)
        FSKB_SMALL_CASE(5) FSKB_SMALL_CASE(6) FSKB_SMALL_CASE(7) FSKB_SMALL_CASE(8)
        FSKB_SMALL_CASE(9) FSKB_SMALL_CASE(10) FSKB_SMALL_CASE(11) FSKB_SMALL_CASE(12)
        FSKB_SMALL_CASE(13) FSKB_SMALL_CASE(14) FSKB_SMALL_CASE(15) FSKB_SMALL_CASE(16)
#undef FSKB_SMALL_CASE
        default:
            throw CudaFailure("small_solve: unsupported d");
    }
    FSKB_CUDA(cudaGetLastError());
    count_launch();
}

}  // namespace fskb
