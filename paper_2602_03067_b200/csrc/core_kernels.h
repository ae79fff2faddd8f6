// CUDA-core (FMA) streaming kernels: the exact-precision engine.
//
// One templated kernel family serves fp64 (the reference's default Double
// precision; 1e-12 parity with stream.cpp) and fp32 (the small-d FMA path of
// the Single precision engine). Each pass streams 64-column key tiles through
// shared memory against a 64-row query block held by 256 threads (4x4 scores
// per thread); nothing n x m ever reaches HBM.
//
//   lse_partial   per (row block, column split): per-row online max / sum-exp
//                 partials (stream.cpp:93-136 lse_reduce, split over columns to
//                 fill 148 SMs when n is small)
//   lse_finalize  combines the partials and writes the requested epilogues:
//                 potential (-eps LSE), symmetric average, LSE/max, induced
//                 marginal r = w exp((pot - pot+)/eps), violation sum
//   apply         O = softmax(S) V (optionally (.)(A B^T)), p in 64-wide chunks
//                 (stream.cpp:140-207 apply_core)
//   apply_finalize  out = w exp(pot/eps + LSE) O, overflow / finiteness flags
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace fskb {

// Biased score S_ij = kscale <q_i, k_j> + (kpot_j + eps klogw_j)/eps
//                     - lam2_eps W[qlab_i, klab_j]            (stream.cpp:61-79)
template <typename T>
struct ScoreParams {
    const T* Q;       // R x d row-major (query side: rows being updated)
    const T* K;       // C x d row-major (key side: streamed)
    int64_t R, C, d;
    T kscale;         // 2 * feature_scale / eps  (stream.cpp:224 scaled2_eps)
    const T* kpot;    // C   key-side shifted potential (g_hat for the f-update)
    const T* klogw;   // C   log key weights
    T eps;
    const int32_t* qlab;  // nullable
    const int32_t* klab;
    const double* wtab;   // V x V label cost
    int64_t wdim;
    T lam2_eps;
};

template <typename T>
struct FinalizeArgs {
    T eps;
    T* out_pot;          // -eps LSE (or symmetric average when sym_old != null)
    const T* sym_old;
    T* out_lse;          // LSE_j S_ij
    T* out_max;          // max_j S_ij
    const T* old_pot;    // for marginals: r_i = w_i exp((old_pot_i - pot_i) / eps)
    const T* w;
    T* out_marg;
    double* viol;        // += sum_i |r_i - w_i| (fixed-order: per-block partials in
                         // viol_part, summed by launch_viol_accumulate)
    int marg_flag;       // which flag bit a non-finite marginal raises
    int* flags;
    int* bad_iter;       // nullable: atomicMin(iter) on a non-finite potential
    int iter;
    int break_lse;       // negative control (set by the launchers)
    float* out_l2h = nullptr;  // tcgen05 path only: log2(e) LSE split hi + lo (float pair)
    float* out_l2l = nullptr;
    double* viol_part = nullptr;  // set by the launchers when viol != null
};

// *viol += sum of part[0 .. nb) in index order (one block): the marginal
// violation is bit-identical run to run.
void launch_viol_accumulate(const double* part, int nb, double* viol, cudaStream_t s);

#ifdef __CUDACC__
// Block-level partial of the violation, in a fixed order (256-thread blocks).
__device__ __forceinline__ void viol_block_partial(double v, double* part) {
    __shared__ double wsum[8];
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t += wsum[w];
        part[blockIdx.x] = t;
    }
}
#endif

// Number of column splits used for R rows (fills the machine when R is small).
int lse_splits(int64_t R, int64_t C);

template <typename T>
void launch_lse(const ScoreParams<T>& P, int splits, T* part_m, T* part_s, cudaStream_t s);

template <typename T>
void launch_lse_finalize(const T* part_m, const T* part_s, int splits, int64_t R,
                         const FinalizeArgs<T>& a, cudaStream_t s);

// O (R x p) = sum_j exp(S_ij - lse_i) [* <A_i, B_j>] V_j ; A/B nullable.
template <typename T>
void launch_apply(const ScoreParams<T>& P, const T* lse, const T* V, int64_t p, const T* A,
                  const T* B, int64_t r, T* O, cudaStream_t s);

// out_ic = w_i exp(pot_i/eps + lse_i) O_ic ; flags overflow when pot/eps + max > 709.
template <typename T>
void launch_apply_finalize(const T* O, int64_t R, int64_t p, const T* w, const T* pot,
                           const T* lse, const T* mx, T eps, T* out, int* flags, cudaStream_t s);

// Elementwise helpers.
template <typename T>
void launch_log(const T* in, T* out, int64_t n, cudaStream_t s);
template <typename T>
void launch_neg_sqnorm(const T* P, int64_t n, int64_t d, T scale, T* out, cudaStream_t s);
void launch_f64_to_f32(const double* in, float* out, int64_t n, cudaStream_t s);
// out (m x d) = diag(w) Y, rounded to float
void launch_scale_rows(const float* Y, const double* w, int64_t m, int64_t d, float* out,
                       cudaStream_t s);
void launch_f32_to_f64(const float* in, double* out, int64_t n, cudaStream_t s);
// pts64 (n x d doubles, device) -> pts32; sqnorm_i = scale * sum_t x_it^2 in fp64 in the
// host loop's order; pot0_i = float(-sqnorm_i) (nullable); *bad |= 1 on a non-finite value
void launch_ingest_f32(const double* pts64, int64_t n, int64_t d, double scale, float* pts32,
                       double* sqnorm, float* pot0, int* bad, cudaStream_t s);
// G_i = 2 (r_i X_i - O_i) with r_i = w_i exp(pot_i/eps + lse_i)
template <typename T>
void launch_grad_epilogue(const T* X, const T* O, const T* w, const T* pot, const T* lse,
                          int64_t R, int64_t d, T eps, T* G, int* flags, cudaStream_t s);
// d <= 16, float problem: G rows [row_begin, row_begin + R) = 2 (r_i x_i - (P Y)_i) in
// fp64 in one pass (online max / sum / transport); false when d is out of range
bool launch_grad_small_fp64(const float* X, const float* wx, const float* f, const float* Y,
                            const float* wy, const float* g, int64_t row_begin, int64_t R,
                            int64_t C, int d, double eps, double kscale, double* G, int* flags,
                            cudaStream_t s);

}  // namespace fskb
