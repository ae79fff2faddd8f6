// Persistent small-problem Sinkhorn loop (CUDA-core FP32, d <= 16): the whole
// alternating iteration sequence of sinkhorn_solve (solver.cpp:36-48; the f32
// loop of solver.cpp:69-117) in ONE cooperative launch. cfg1 (n = m = 4096,
// d = 3) is launch-bound: its half-step is ~4 us of MUFU work, while a graph of
// per-half-step LSE + finalize kernels costs ~49 us per half-step in launch
// gaps. Here every half-step is
//   stage:  all keys of the side (pre-scaled by 2/eps, SoA) + their bias
//           (pot_j + eps log w_j)/eps into shared memory (<= 192 KB)
//   rows:   one warp per query row (32 warps per CTA), lanes stride groups of 4
//           keys (float4 shared loads), online (max, sum) in log2 units with one
//           rescale per group at most and one ex2 per score, warp reduction;
//           f_i = -eps ln2 (max + log2 sum)
//   sync:   grid-wide barrier, then the other side reads the new potential.
// Scores are formed as the FP32 tile kernel does (fma over features in order onto
// the bias), with keys and bias pre-scaled to log2 units at staging, so the
// result differs from the per-launch path at fp32 rounding (contract of SURVEY §8d).
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.h"
#include "small_solve.h"

namespace cg = cooperative_groups;

namespace fskb {
namespace {

constexpr int kWarps = 32;
constexpr int kThreads = 32 * kWarps;

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) small_solve_kernel(const SmallSolveParams p) {
    extern __shared__ __align__(16) float sm[];
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t cpad = p.cpad;   // multiple of 128: every lane's float4 group is in range
    constexpr float kLog2e = 1.4426950408889634f;
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
            // stage the keys (SoA, x 2 s / eps, in log2 units) and their bias; padded
            // keys get a -inf bias
            for (int64_t j = threadIdx.x; j < cpad; j += kThreads) {
                if (j < C) {
#pragma unroll
                    for (int t = 0; t < D; ++t)
                        sm[t * cpad + j] = (K[j * D + t] * kscale) * kLog2e;
                    sm[D * cpad + j] = ((kpot[j] + eps * klogw[j]) / eps) * kLog2e;
                } else {
#pragma unroll
                    for (int t = 0; t < D; ++t) sm[t * cpad + j] = 0.0f;
                    sm[D * cpad + j] = -INFINITY;
                }
            }
            __syncthreads();
            const float4* s4 = reinterpret_cast<const float4*>(sm);
            const int64_t c4 = cpad / 4;
            for (int64_t r = int64_t(blockIdx.x) * kWarps + warp; r < R;
                 r += int64_t(gridDim.x) * kWarps) {
                float q[D];
#pragma unroll
                for (int t = 0; t < D; ++t) q[t] = Q[r * D + t];
                // online (max, sum) per lane over groups of 4 keys: one rescale per
                // group at most, one ex2 per score
                float mx = -INFINITY, sum = 0.0f;
                for (int64_t g = lane; g < c4; g += 32) {
                    float4 acc = s4[D * c4 + g];
#pragma unroll
                    for (int t = 0; t < D; ++t) {
                        const float4 k = s4[t * c4 + g];
                        acc.x = fmaf(q[t], k.x, acc.x);
                        acc.y = fmaf(q[t], k.y, acc.y);
                        acc.z = fmaf(q[t], k.z, acc.z);
                        acc.w = fmaf(q[t], k.w, acc.w);
                    }
                    const float gm = fmaxf(fmaxf(acc.x, acc.y), fmaxf(acc.z, acc.w));
                    if (gm > mx) {
                        sum *= ex2(mx - gm);
                        mx = gm;
                    }
                    if (mx > -INFINITY)   // (a lane whose groups are all padding stays empty)
                        sum += ex2(acc.x - mx) + ex2(acc.y - mx) + ex2(acc.z - mx) +
                               ex2(acc.w - mx);
                }
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                    const float mo = __shfl_xor_sync(0xffffffffu, mx, off);
                    const float so = __shfl_xor_sync(0xffffffffu, sum, off);
                    const float M = fmaxf(mx, mo);
                    sum = (mx > -INFINITY ? sum * ex2(mx - M) : 0.0f) +
                          (mo > -INFINITY ? so * ex2(mo - M) : 0.0f);
                    mx = M;
                }
                if (lane == 0) {
                    // f = -eps ln 2 (max + log2 sum)
                    const float pot = -eps * 0.6931471805599453f * (mx + __log2f(sum));
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

// Resident variant (both clouds fit in shared memory next to the bias row): the
// clouds (SoA) and the log2 weights are staged ONCE per launch; a half-step only
// refreshes the key bias from the other side's new potential (one coalesced read
// of m floats per CTA). Rows are dealt round-robin over the grid (row r -> CTA
// r mod G, warp r / G), so every SM holds ceil(R / G) rows instead of 32 rows on
// R / 32 SMs. Scores: bias_j + sum_t (x_t 2 s log2e / eps) y_t, the query
// pre-scaled in registers.
template <int D>
__global__ void __launch_bounds__(kThreads, 1) small_solve_res_kernel(const SmallSolveParams p) {
    extern __shared__ __align__(16) float sm[];
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t np = p.npad, mp = p.mpad;
    float* xs = sm;             // D x np
    float* ys = xs + D * np;    // D x mp
    float* lx = ys + D * mp;    // log2 a, -inf past n
    float* ly = lx + np;        // log2 b, -inf past m
    float* bias = ly + mp;      // max(np, mp)
    constexpr float kLog2e = 1.4426950408889634f;
    for (int64_t j = threadIdx.x; j < np; j += kThreads) {
        const bool v = j < p.n;
#pragma unroll
        for (int t = 0; t < D; ++t) xs[t * np + j] = v ? p.X[j * D + t] : 0.0f;
        lx[j] = v ? p.logw_x[j] * kLog2e : -INFINITY;
    }
    for (int64_t j = threadIdx.x; j < mp; j += kThreads) {
        const bool v = j < p.m;
#pragma unroll
        for (int t = 0; t < D; ++t) ys[t * mp + j] = v ? p.Y[j * D + t] : 0.0f;
        ly[j] = v ? p.logw_y[j] * kLog2e : -INFINITY;
    }
    const int64_t G = gridDim.x;
    for (int it = 0; it < p.iters; ++it) {
        const float eps = p.eps_sched[it];
        const float qscale = 2.0f * p.fscale / eps * kLog2e;
        const float bscale = kLog2e / eps;
        for (int side = 0; side < 2; ++side) {
            const float* Qs = side == 0 ? xs : ys;
            const float* Ks = side == 0 ? ys : xs;
            const float* klw = side == 0 ? ly : lx;
            const float* kpot = side == 0 ? p.g : p.f;   // written by this launch: no __ldg
            float* out = side == 0 ? p.f : p.g;
            const int64_t qp = side == 0 ? np : mp, kp = side == 0 ? mp : np;
            const int64_t R = side == 0 ? p.n : p.m, C = side == 0 ? p.m : p.n;
            __syncthreads();   // (the previous half-step's rows are done with bias)
            for (int64_t j = threadIdx.x; j < kp; j += kThreads)
                bias[j] = fmaf(j < C ? kpot[j] : 0.0f, bscale, klw[j]);
            __syncthreads();
            const float4* k4 = reinterpret_cast<const float4*>(Ks);
            const float4* b4 = reinterpret_cast<const float4*>(bias);
            const int64_t c4 = kp / 4;
            for (int64_t r = blockIdx.x + G * warp; r < R; r += G * kWarps) {
                float q[D];
#pragma unroll
                for (int t = 0; t < D; ++t) q[t] = Qs[t * qp + r] * qscale;
                float mx = -INFINITY, sum = 0.0f;
                for (int64_t g = lane; g < c4; g += 32) {
                    float4 acc = b4[g];
#pragma unroll
                    for (int t = 0; t < D; ++t) {
                        const float4 k = k4[t * c4 + g];
                        acc.x = fmaf(q[t], k.x, acc.x);
                        acc.y = fmaf(q[t], k.y, acc.y);
                        acc.z = fmaf(q[t], k.z, acc.z);
                        acc.w = fmaf(q[t], k.w, acc.w);
                    }
                    const float gm = fmaxf(fmaxf(acc.x, acc.y), fmaxf(acc.z, acc.w));
                    if (gm > mx) {
                        sum *= ex2(mx - gm);
                        mx = gm;
                    }
                    if (mx > -INFINITY)
                        sum += ex2(acc.x - mx) + ex2(acc.y - mx) + ex2(acc.z - mx) +
                               ex2(acc.w - mx);
                }
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                    const float mo = __shfl_xor_sync(0xffffffffu, mx, off);
                    const float so = __shfl_xor_sync(0xffffffffu, sum, off);
                    const float M = fmaxf(mx, mo);
                    sum = (mx > -INFINITY ? sum * ex2(mx - M) : 0.0f) +
                          (mo > -INFINITY ? so * ex2(mo - M) : 0.0f);
                    mx = M;
                }
                if (lane == 0) {
                    const float pot = -eps * 0.6931471805599453f * (mx + __log2f(sum));
                    if (!isfinite(pot)) {
                        atomicOr(p.flags, kFlagNonFinitePotential);
                        if (p.bad_iter) atomicMin(p.bad_iter, p.iter0 + it + 1);
                    }
                    out[r] = pot;
                }
            }
            grid.sync();
        }
    }
}

size_t resident_smem(int64_t n, int64_t m, int64_t d) {
    const int64_t np = (n + 127) / 128 * 128, mp = (m + 127) / 128 * 128;
    return size_t((d + 1) * (np + mp) + (np > mp ? np : mp)) * sizeof(float);
}

template <int D>
void launch_d(const SmallSolveParams& p, int grid, size_t smem, bool resident, cudaStream_t s) {
    static bool configured = false;
    if (!configured) {
        FSKB_CUDA(cudaFuncSetAttribute(small_solve_kernel<D>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kSmallSolveSmem)));
        FSKB_CUDA(cudaFuncSetAttribute(small_solve_res_kernel<D>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kSmallSolveResSmem)));
        configured = true;
    }
    SmallSolveParams q = p;
    void* args[] = {&q};
    void* fn = resident ? reinterpret_cast<void*>(small_solve_res_kernel<D>)
                        : reinterpret_cast<void*>(small_solve_kernel<D>);
    FSKB_CUDA(cudaLaunchCooperativeKernel(fn, dim3(unsigned(grid)), dim3(kThreads), args, smem, s));
}

}  // namespace

bool small_solve_fits(int64_t n, int64_t m, int64_t d) {
    if (d < 1 || d > kSmallSolveMaxD || n < 1 || m < 1) return false;
    const int64_t cmax = n > m ? n : m;
    const int64_t cpad = (cmax + 127) / 128 * 128;
    return size_t(cpad) * size_t(d + 1) * sizeof(float) <= kSmallSolveSmem;
}

void launch_small_solve(const SmallSolveParams& p0, cudaStream_t s) {
    if (p0.iters < 1) return;
    SmallSolveParams p = p0;
    const int64_t cmax = p.n > p.m ? p.n : p.m;
    p.cpad = (cmax + 127) / 128 * 128;
    p.npad = (p.n + 127) / 128 * 128;
    p.mpad = (p.m + 127) / 128 * 128;
    const char* renv = std::getenv("FSK_SMALL_RESIDENT");
    const bool resident = !(renv && renv[0] == '0') &&
                          resident_smem(p.n, p.m, p.d) <= kSmallSolveResSmem;
    const size_t smem = resident ? resident_smem(p.n, p.m, p.d)
                                 : size_t(p.cpad) * size_t(p.d + 1) * sizeof(float);
    // one CTA per SM (co-residency is what the grid barrier needs)
    const int grid = num_sms();
    switch (p.d) {
#define FSKB_SMALL_CASE(DD) \
    case DD:                \
        launch_d<DD>(p, grid, smem, resident, s); \
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
