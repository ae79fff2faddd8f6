// CUDA-core streaming kernels (fp64 exact path, fp32 FMA path). See core_kernels.h.
#include <cfloat>
#include <cmath>

#include "common.h"
#include "core_kernels.h"

namespace fskb {

namespace {

constexpr int BM = 64;   // query rows per block
constexpr int BN = 64;   // key columns per tile
constexpr int DK = 16;   // depth chunk staged in shared memory
constexpr int NT = 256;  // threads: 16 (tx, columns) x 16 (ty, rows)
constexpr int PC = 64;   // output columns per apply block

template <typename T>
__device__ __forceinline__ T dexp(T x);
template <>
__device__ __forceinline__ double dexp<double>(double x) { return exp(x); }
// full-precision expf (not __expf: its ex2(x log2e) loses |x| 2^-24 relative, which
// put the fp32 CUDA-core gradient at 2.5x the reference fp32 path's error on cfg1)
template <>
__device__ __forceinline__ float dexp<float>(float x) { return expf(x); }

template <typename T>
__device__ __forceinline__ T dlog(T x);
template <>
__device__ __forceinline__ double dlog<double>(double x) { return log(x); }
template <>
__device__ __forceinline__ float dlog<float>(float x) { return logf(x); }

template <typename T>
__device__ __forceinline__ T ninf() { return -INFINITY; }

// acc[ii][jj] = sum_t Q[I0+ty*4+ii][t] * (K[J0+tx+16jj][t] * kscale)
template <typename T>
__device__ __forceinline__ void dot_tile(const T* __restrict__ Q, const T* __restrict__ K,
                                         int64_t R, int64_t C, int64_t d, T kscale, int64_t I0,
                                         int64_t J0, T (&acc)[4][4], T* Qs, T* Ks) {
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[ii][jj] = T(0);
    for (int64_t k0 = 0; k0 < d; k0 += DK) {
        __syncthreads();
#pragma unroll
        for (int u = 0; u < (BM * DK) / NT; ++u) {
            const int e = tid + u * NT;
            const int row = e / DK, kk = e % DK;
            const int64_t gk = k0 + kk;
            const int64_t gi = I0 + row, gj = J0 + row;
            Qs[kk * (BM + 1) + row] = (gi < R && gk < d) ? Q[gi * d + gk] : T(0);
            Ks[kk * (BN + 1) + row] = (gj < C && gk < d) ? K[gj * d + gk] * kscale : T(0);
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < DK; ++kk) {
            T qv[4], kv[4];
#pragma unroll
            for (int ii = 0; ii < 4; ++ii) qv[ii] = Qs[kk * (BM + 1) + ty * 4 + ii];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) kv[jj] = Ks[kk * (BN + 1) + tx + 16 * jj];
#pragma unroll
            for (int ii = 0; ii < 4; ++ii)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) acc[ii][jj] = fma(qv[ii], kv[jj], acc[ii][jj]);
        }
    }
}

// Scores for the 4x4 micro-tile, -inf outside [.., Jend).
template <typename T, bool LAB>
__device__ __forceinline__ void score_tile(const ScoreParams<T>& P, int64_t I0, int64_t J0,
                                           int64_t Jend, T (&sc)[4][4], T* Qs, T* Ks) {
    dot_tile(P.Q, P.K, P.R, P.C, P.d, P.kscale, I0, J0, sc, Qs, Ks);
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
        const int64_t j = J0 + tx + 16 * jj;
        const bool ok = j < Jend;
        const T bias = ok ? (P.kpot[j] + P.eps * P.klogw[j]) / P.eps : T(0);
        int32_t kl = 0;
        if (LAB && ok) kl = P.klab[j];
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
            T v = sc[ii][jj] + bias;
            if (LAB) {
                const int64_t i = I0 + ty * 4 + ii;
                if (ok && i < P.R) v -= P.lam2_eps * T(P.wtab[int64_t(P.qlab[i]) * P.wdim + kl]);
            }
            sc[ii][jj] = ok ? v : ninf<T>();
        }
    }
}

template <typename T, bool LAB>
__global__ void __launch_bounds__(NT) lse_partial_kernel(ScoreParams<T> P, int64_t cols_per_split,
                                                         T* __restrict__ part_m,
                                                         T* __restrict__ part_s, int break_lse) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* Qs = reinterpret_cast<T*>(smem_raw);
    T* Ks = Qs + DK * (BM + 1);
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t I0 = int64_t(blockIdx.x) * BM;
    const int64_t Jbeg = int64_t(blockIdx.y) * cols_per_split;
    const int64_t Jend = min(P.C, Jbeg + cols_per_split);
    T m[4], s[4];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
        m[ii] = ninf<T>();
        s[ii] = T(0);
    }
    for (int64_t J0 = Jbeg; J0 < Jend; J0 += BN) {
        T sc[4][4];
        score_tile<T, LAB>(P, I0, J0, Jend, sc, Qs, Ks);
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
            T tmax = sc[ii][0];
#pragma unroll
            for (int jj = 1; jj < 4; ++jj) tmax = fmax(tmax, sc[ii][jj]);
            if (tmax > m[ii]) {
                // online rescale (stream.cpp:81-87); the negative control flips it
                if (s[ii] != T(0)) s[ii] *= break_lse ? dexp(tmax - m[ii]) : dexp(m[ii] - tmax);
                m[ii] = tmax;
            }
            if (m[ii] != ninf<T>()) {
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) s[ii] += dexp(sc[ii][jj] - m[ii]);
            }
        }
    }
    // combine the 16 column-threads sharing each row
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
#pragma unroll
        for (int off = 8; off >= 1; off >>= 1) {
            const T mo = __shfl_xor_sync(0xffffffffu, m[ii], off);
            const T so = __shfl_xor_sync(0xffffffffu, s[ii], off);
            const T M = fmax(m[ii], mo);
            T acc = T(0);
            if (m[ii] != ninf<T>()) acc += s[ii] * dexp(break_lse ? M - m[ii] : m[ii] - M);
            if (mo != ninf<T>()) acc += so * dexp(break_lse ? M - mo : mo - M);
            m[ii] = M;
            s[ii] = acc;
        }
        const int64_t i = I0 + ty * 4 + ii;
        if (tx == 0 && i < P.R) {
            part_m[int64_t(blockIdx.y) * P.R + i] = m[ii];
            part_s[int64_t(blockIdx.y) * P.R + i] = s[ii];
        }
    }
}

template <typename T>
__global__ void lse_finalize_kernel(const T* __restrict__ part_m, const T* __restrict__ part_s,
                                    int splits, int64_t R, FinalizeArgs<T> a) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    double vsum = 0.0;
    if (i < R) {
        T M = ninf<T>();
        for (int k = 0; k < splits; ++k) M = fmax(M, part_m[k * R + i]);
        T S = T(0);
        for (int k = 0; k < splits; ++k) {
            const T mk = part_m[k * R + i];
            if (mk != ninf<T>()) S += part_s[k * R + i] * dexp(a.break_lse ? M - mk : mk - M);
        }
        const T lse = M + dlog(S);
        if (a.out_lse) a.out_lse[i] = lse;
        if (a.out_max) a.out_max[i] = M;
        const T pot = -a.eps * lse;
        if (!isfinite(pot)) {
            atomicOr(a.flags, kFlagNonFinitePotential);
            if (a.bad_iter) atomicMin(a.bad_iter, a.iter);
        }
        // marginals read old_pot before out_pot is written (they may alias)
        if (a.out_marg || a.viol) {
            const T r = a.w[i] * dexp((a.old_pot[i] - pot) * (T(1) / a.eps));
            if (!isfinite(r)) atomicOr(a.flags, a.marg_flag);
            if (a.out_marg) a.out_marg[i] = r;
            vsum = fabs(double(r) - double(a.w[i]));
        }
        if (a.out_pot) a.out_pot[i] = a.sym_old ? T(0.5) * a.sym_old[i] + T(0.5) * pot : pot;
    }
    if (a.viol) viol_block_partial(vsum, a.viol_part);
}

__global__ void viol_accumulate_kernel(const double* __restrict__ part, int nb,
                                       double* __restrict__ viol) {
    __shared__ double sh[256];
    double v = 0.0;
    for (int i = threadIdx.x; i < nb; i += 256) v += part[i];
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *viol += sh[0];
}

template <typename T, bool LAB, bool HAD>
__global__ void __launch_bounds__(NT) apply_kernel(ScoreParams<T> P, const T* __restrict__ lse,
                                                   const T* __restrict__ V, int64_t p,
                                                   const T* __restrict__ A,
                                                   const T* __restrict__ B, int64_t r,
                                                   T* __restrict__ O, int64_t per) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* Qs = reinterpret_cast<T*>(smem_raw);
    T* Ks = Qs + DK * (BM + 1);
    T* Ps = Ks + DK * (BN + 1);       // BM x (BN+1)
    T* Vs = Ps + BM * (BN + 1);       // BN x (PC+1)
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int64_t I0 = int64_t(blockIdx.x) * BM;
    const int64_t c0 = int64_t(blockIdx.y) * PC;
    T li[4];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
        const int64_t i = I0 + ty * 4 + ii;
        li[ii] = i < P.R ? lse[i] : T(0);
    }
    T o[4][4];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) o[ii][cc] = T(0);
    // key split blockIdx.z: keys [z per, z per + per); partial O at O + z R p
    const int64_t Jb = int64_t(blockIdx.z) * per, Je = min(P.C, Jb + per);
    O += int64_t(blockIdx.z) * P.R * p;
    for (int64_t J0 = Jb; J0 < Je; J0 += BN) {
        T sc[4][4];
        score_tile<T, LAB>(P, I0, J0, Je, sc, Qs, Ks);
#pragma unroll
        for (int ii = 0; ii < 4; ++ii)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
                sc[ii][jj] = sc[ii][jj] == ninf<T>() ? T(0) : dexp(sc[ii][jj] - li[ii]);
        if (HAD) {
            T wd[4][4];
            dot_tile(A, B, P.R, P.C, r, T(1), I0, J0, wd, Qs, Ks);
#pragma unroll
            for (int ii = 0; ii < 4; ++ii)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) sc[ii][jj] *= wd[ii][jj];
        }
        __syncthreads();
#pragma unroll
        for (int ii = 0; ii < 4; ++ii)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) Ps[(ty * 4 + ii) * (BN + 1) + tx + 16 * jj] = sc[ii][jj];
#pragma unroll
        for (int u = 0; u < (BN * PC) / NT; ++u) {
            const int e = tid + u * NT;
            const int j = e / PC, c = e % PC;
            const int64_t gj = J0 + j, gc = c0 + c;
            Vs[j * (PC + 1) + c] = (gj < P.C && gc < p) ? V[gj * p + gc] : T(0);
        }
        __syncthreads();
#pragma unroll 8
        for (int j = 0; j < BN; ++j) {
            T pv[4], vv[4];
#pragma unroll
            for (int ii = 0; ii < 4; ++ii) pv[ii] = Ps[(ty * 4 + ii) * (BN + 1) + j];
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) vv[cc] = Vs[j * (PC + 1) + tx + 16 * cc];
#pragma unroll
            for (int ii = 0; ii < 4; ++ii)
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) o[ii][cc] = fma(pv[ii], vv[cc], o[ii][cc]);
        }
    }
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
        const int64_t i = I0 + ty * 4 + ii;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
            const int64_t c = c0 + tx + 16 * cc;
            if (i < P.R && c < p) O[i * p + c] = o[ii][cc];
        }
    }
}

template <typename T>
__global__ void apply_finalize_kernel(const T* __restrict__ O, int64_t R, int64_t p,
                                      const T* __restrict__ w, const T* __restrict__ pot,
                                      const T* __restrict__ lse, const T* __restrict__ mx, T eps,
                                      T* __restrict__ out, int* flags) {
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= R * p) return;
    const int64_t i = idx / p;
    const T argmax = pot[i] / eps + mx[i];
    if (argmax > T(709)) {
        atomicOr(flags, kFlagTransportOverflow);
        out[idx] = T(0);
        return;
    }
    const T v = w[i] * dexp(pot[i] / eps + lse[i]) * O[idx];
    if (!isfinite(v)) atomicOr(flags, kFlagNonFiniteTransport);
    out[idx] = v;
}

template <typename T>
__global__ void log_kernel(const T* in, T* out, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = dlog(in[i]);
}

template <typename T>
__global__ void neg_sqnorm_kernel(const T* P, int64_t n, int64_t d, T scale, T* out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    T s = T(0);
    for (int64_t t = 0; t < d; ++t) s += P[i * d + t] * P[i * d + t];
    out[i] = -(scale == T(1) ? s : s * scale);
}

__global__ void f64_to_f32_kernel(const double* in, float* out, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = float(in[i]);
}
__global__ void f32_to_f64_kernel(const float* in, double* out, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = double(in[i]);
}

template <typename T>
__global__ void grad_epilogue_kernel(const T* X, const T* O, const T* w, const T* pot,
                                     const T* lse, int64_t R, int64_t d, T eps, T* G,
                                     int* flags) {
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= R * d) return;
    const int64_t i = idx / d;
    const T ri = w[i] * dexp(pot[i] / eps + lse[i]);
    const T v = T(2) * ri * (X[idx] - O[idx]);
    if (!isfinite(v)) atomicOr(flags, kFlagNonFiniteTransport);
    G[idx] = v;
}

// Small-d fp64 gradient in ONE pass (grad_rows_fp64 for d <= 16 without labels):
// per row an online (max, sum, sum e^s y) over all keys, one warp per row, lanes
// striding the keys, merged across lanes at the end; G_i = 2 r_i (x_i - O_i) with
// O_i = (sum e^s y) / sum, r_i = a_i exp(f_i / eps + lse_i) (the epilogue above).
// The per-key terms are prepared once: kb_j = (g_j + eps log b_j) / eps, ky_j =
// y_j 2 s / eps, the scores formed as the two-pass path forms them.
__global__ void grad_small_prep_kernel(const float* __restrict__ Y, const float* __restrict__ wy,
                                       const float* __restrict__ g, int64_t C, int d, double eps,
                                       double kscale, double* __restrict__ kb,
                                       double* __restrict__ ky) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= C) return;
    kb[j] = (double(g[j]) + eps * log(double(wy[j]))) / eps;
    for (int t = 0; t < d; ++t) ky[j * d + t] = double(Y[j * d + t]) * kscale;
}

template <int D>
__global__ void __launch_bounds__(256) grad_small_fp64_kernel(
    const float* __restrict__ X, const float* __restrict__ wx, const float* __restrict__ f,
    const float* __restrict__ Y, const double* __restrict__ kb, const double* __restrict__ ky,
    int64_t row_begin, int64_t R, int64_t C, double eps, double* __restrict__ G, int* flags) {
    const int lane = threadIdx.x & 31;
    const int64_t li = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (li >= R) return;   // whole warps
    const int64_t i = row_begin + li;
    double q[D], v[D];
#pragma unroll
    for (int t = 0; t < D; ++t) {
        q[t] = double(X[i * D + t]);
        v[t] = 0.0;
    }
    double m = -INFINITY, s = 0.0;
    for (int64_t j = lane; j < C; j += 32) {
        double sc = 0.0;
#pragma unroll
        for (int t = 0; t < D; ++t) sc = fma(q[t], __ldg(ky + j * D + t), sc);
        sc += __ldg(kb + j);
        if (!(sc > -INFINITY)) continue;   // zero-weight key
        if (sc > m) {
            const double a = exp(m - sc);
            s *= a;
#pragma unroll
            for (int t = 0; t < D; ++t) v[t] *= a;
            m = sc;
        }
        const double e = exp(sc - m);
        s += e;
#pragma unroll
        for (int t = 0; t < D; ++t) v[t] = fma(e, double(__ldg(Y + j * D + t)), v[t]);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const double mo = __shfl_xor_sync(0xffffffffu, m, off);
        const double so = __shfl_xor_sync(0xffffffffu, s, off);
        const double M = fmax(m, mo);
        const double a = m > -INFINITY ? exp(m - M) : 0.0;
        const double b = mo > -INFINITY ? exp(mo - M) : 0.0;
        s = s * a + so * b;
#pragma unroll
        for (int t = 0; t < D; ++t) {
            const double vo = __shfl_xor_sync(0xffffffffu, v[t], off);
            v[t] = v[t] * a + vo * b;
        }
        m = M;
    }
    if (lane == 0) {
        const double lse = m + log(s);
        const double ri = double(wx[i]) * exp(double(f[i]) / eps + lse);
        bool bad = false;
#pragma unroll
        for (int t = 0; t < D; ++t) {
            const double gv = 2.0 * ri * (q[t] - v[t] / s);
            bad |= !isfinite(gv);
            G[li * D + t] = gv;
        }
        if (bad) atomicOr(flags, kFlagNonFiniteTransport);
    }
}

inline unsigned blocks_for(int64_t n, int t = 256) { return unsigned((n + t - 1) / t); }

template <typename T>
std::size_t lse_smem() {
    return sizeof(T) * (DK * (BM + 1) + DK * (BN + 1));
}
template <typename T>
std::size_t apply_smem() {
    return sizeof(T) * (DK * (BM + 1) + DK * (BN + 1) + BM * (BN + 1) + BN * (PC + 1));
}

}  // namespace

int lse_splits(int64_t R, int64_t C) {
    const int64_t rowblocks = (R + BM - 1) / BM;
    const int64_t target = int64_t(num_sms()) * 4;
    int64_t splits = (target + rowblocks - 1) / rowblocks;
    const int64_t max_splits = (C + BN - 1) / BN;
    if (splits > max_splits) splits = max_splits;
    if (splits < 1) splits = 1;
    if (splits > 64) splits = 64;
    return int(splits);
}

template <typename T>
void launch_lse(const ScoreParams<T>& P, int splits, T* part_m, T* part_s, cudaStream_t s) {
    const int64_t per = ((P.C + splits - 1) / splits + BN - 1) / BN * BN;
    dim3 grid(unsigned((P.R + BM - 1) / BM), unsigned(splits));
    const int brk = break_lse_flag() ? 1 : 0;
    if (P.qlab)
        lse_partial_kernel<T, true><<<grid, NT, lse_smem<T>(), s>>>(P, per, part_m, part_s, brk);
    else
        lse_partial_kernel<T, false><<<grid, NT, lse_smem<T>(), s>>>(P, per, part_m, part_s, brk);
    FSKB_CUDA(cudaGetLastError());
    count_launch();
}

template <typename T>
void launch_lse_finalize(const T* part_m, const T* part_s, int splits, int64_t R,
                         const FinalizeArgs<T>& a, cudaStream_t s) {
    FinalizeArgs<T> fa = a;
    fa.break_lse = break_lse_flag() ? 1 : 0;
    const unsigned nb = blocks_for(R);
    DevBuf<double> vpart;
    if (fa.viol) {
        vpart.alloc(nb, s);
        fa.viol_part = vpart.get();
    }
    lse_finalize_kernel<T><<<nb, 256, 0, s>>>(part_m, part_s, splits, R, fa);
    FSKB_CUDA(cudaGetLastError());
    count_launch();
    if (fa.viol) launch_viol_accumulate(vpart.get(), int(nb), fa.viol, s);
}

void launch_viol_accumulate(const double* part, int nb, double* viol, cudaStream_t s) {
    viol_accumulate_kernel<<<1, 256, 0, s>>>(part, nb, viol);
    FSKB_CUDA(cudaGetLastError());
    count_launch();
}

// O = sum over the key splits' partials, in split order (deterministic)
template <typename T>
__global__ void sum_splits_kernel(const T* __restrict__ part, int splits, int64_t n,
                                  T* __restrict__ out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    T v = part[i];
    for (int k = 1; k < splits; ++k) v += part[size_t(k) * n + i];
    out[i] = v;
}

template <typename T>
void launch_apply(const ScoreParams<T>& P, const T* lse, const T* V, int64_t p, const T* A,
                  const T* B, int64_t r, T* O, cudaStream_t s) {
    // small row counts fill the GPU with key splits (partials summed in split order)
    const int64_t tiles = ((P.R + BM - 1) / BM) * ((p + PC - 1) / PC);
    int64_t splits = (2 * int64_t(num_sms()) + tiles - 1) / tiles;
    splits = std::max<int64_t>(1, std::min<int64_t>({splits, (P.C + BN - 1) / BN, 16}));
    const int64_t per = ((P.C + splits - 1) / splits + BN - 1) / BN * BN;
    splits = (P.C + per - 1) / per;
    DevBuf<T> part;
    T* dst = O;
    if (splits > 1) {
        part.alloc(size_t(splits) * size_t(P.R) * size_t(p), s);
        dst = part.get();
    }
    dim3 grid(unsigned((P.R + BM - 1) / BM), unsigned((p + PC - 1) / PC), unsigned(splits));
    const std::size_t sm = apply_smem<T>();
    static bool configured = false;
    if (!configured) {
        FSKB_CUDA(cudaFuncSetAttribute(apply_kernel<T, false, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        FSKB_CUDA(cudaFuncSetAttribute(apply_kernel<T, true, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        FSKB_CUDA(cudaFuncSetAttribute(apply_kernel<T, false, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        FSKB_CUDA(cudaFuncSetAttribute(apply_kernel<T, true, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        configured = true;
    }
    const bool lab = P.qlab != nullptr, had = A != nullptr;
    if (lab && had)
        apply_kernel<T, true, true><<<grid, NT, sm, s>>>(P, lse, V, p, A, B, r, dst, per);
    else if (lab)
        apply_kernel<T, true, false><<<grid, NT, sm, s>>>(P, lse, V, p, A, B, r, dst, per);
    else if (had)
        apply_kernel<T, false, true><<<grid, NT, sm, s>>>(P, lse, V, p, A, B, r, dst, per);
    else
        apply_kernel<T, false, false><<<grid, NT, sm, s>>>(P, lse, V, p, A, B, r, dst, per);
    FSKB_CUDA(cudaGetLastError());
    count_launch();
    if (splits > 1) {
        const int64_t n = P.R * p;
        sum_splits_kernel<T><<<blocks_for(n), 256, 0, s>>>(part.get(), int(splits), n, O);
        FSKB_CUDA(cudaGetLastError());
        count_launch();
    }
}

template <typename T>
void launch_apply_finalize(const T* O, int64_t R, int64_t p, const T* w, const T* pot,
                           const T* lse, const T* mx, T eps, T* out, int* flags, cudaStream_t s) {
    apply_finalize_kernel<T><<<blocks_for(R * p), 256, 0, s>>>(O, R, p, w, pot, lse, mx, eps, out,
                                                              flags);
    FSKB_CUDA(cudaGetLastError());
    count_launch();
}

template <typename T>
void launch_log(const T* in, T* out, int64_t n, cudaStream_t s) {
    if (!n) return;
    log_kernel<T><<<blocks_for(n), 256, 0, s>>>(in, out, n);
    FSKB_CUDA(cudaGetLastError());
    count_launch();
}

template <typename T>
void launch_neg_sqnorm(const T* P, int64_t n, int64_t d, T scale, T* out, cudaStream_t s) {
    if (!n) return;
    neg_sqnorm_kernel<T><<<blocks_for(n), 256, 0, s>>>(P, n, d, scale, out);
    FSKB_CUDA(cudaGetLastError());
    count_launch();
}

__global__ void scale_rows_kernel(const float* __restrict__ Y, const double* __restrict__ w,
                                  int64_t m, int64_t d, float* __restrict__ out) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < m * d;
         k += int64_t(gridDim.x) * blockDim.x)
        out[k] = float(w[k / d] * double(Y[k]));
}
void launch_scale_rows(const float* Y, const double* w, int64_t m, int64_t d, float* out,
                       cudaStream_t s) {
    if (!m || !d) return;
    scale_rows_kernel<<<blocks_for(m * d), 256, 0, s>>>(Y, w, m, d, out);
    FSKB_CUDA(cudaGetLastError());
    count_launch();
}

// Single-precision ingest of a caller cloud (n x d doubles already on the device):
// narrows the points to float, flags any non-finite coordinate (validate_measure,
// core.cpp:18-66, deferred to the device) and writes each row's squared norm in fp64
// in the host loop's order (s += x_t * x_t, t = 0..d-1, no contraction: bit-identical
// to host_sqnorm_compute) times scale, and the negated, narrowed initial potential
// -alpha (solver.cpp:27-32) when pot0 is given.
__global__ void ingest_narrow_kernel(const double* __restrict__ in, float* __restrict__ out,
                                     int64_t n, int* bad) {
    int found = 0;
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
         k += int64_t(gridDim.x) * blockDim.x) {
        const double v = in[k];
        found |= int((__double_as_longlong(v) & 0x7FF0000000000000ll) == 0x7FF0000000000000ll);
        out[k] = float(v);
    }
    if (__any_sync(0xffffffffu, found) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}
__global__ void ingest_sqnorm_kernel(const double* __restrict__ P, int64_t n, int64_t d,
                                     double scale, double* __restrict__ sq,
                                     float* __restrict__ pot0) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const double* r = P + i * d;
        double s = 0.0;
        for (int64_t t = 0; t < d; ++t) s = __dadd_rn(s, __dmul_rn(r[t], r[t]));
        const double a = scale != 1.0 ? __dmul_rn(s, scale) : s;
        sq[i] = a;
        if (pot0) pot0[i] = float(-a);
    }
}
void launch_ingest_f32(const double* pts64, int64_t n, int64_t d, double scale, float* pts32,
                       double* sqnorm, float* pot0, int* bad, cudaStream_t s) {
    if (!n) return;
    ingest_narrow_kernel<<<blocks_for(n * d), 256, 0, s>>>(pts64, pts32, n * d, bad);
    FSKB_CUDA(cudaGetLastError());
    ingest_sqnorm_kernel<<<blocks_for(n, 128), 128, 0, s>>>(pts64, n, d, scale, sqnorm, pot0);
    FSKB_CUDA(cudaGetLastError());
    count_launch(2);
}

void launch_f64_to_f32(const double* in, float* out, int64_t n, cudaStream_t s) {
    if (!n) return;
    f64_to_f32_kernel<<<blocks_for(n), 256, 0, s>>>(in, out, n);
    FSKB_CUDA(cudaGetLastError());
    count_launch();
}
void launch_f32_to_f64(const float* in, double* out, int64_t n, cudaStream_t s) {
    if (!n) return;
    f32_to_f64_kernel<<<blocks_for(n), 256, 0, s>>>(in, out, n);
    FSKB_CUDA(cudaGetLastError());
    count_launch();
}

template <typename T>
void launch_grad_epilogue(const T* X, const T* O, const T* w, const T* pot, const T* lse,
                          int64_t R, int64_t d, T eps, T* G, int* flags, cudaStream_t s) {
    if (!R) return;
    grad_epilogue_kernel<T><<<blocks_for(R * d), 256, 0, s>>>(X, O, w, pot, lse, R, d, eps, G,
                                                              flags);
    FSKB_CUDA(cudaGetLastError());
    count_launch();
}

bool launch_grad_small_fp64(const float* X, const float* wx, const float* f, const float* Y,
                            const float* wy, const float* g, int64_t row_begin, int64_t R,
                            int64_t C, int d, double eps, double kscale, double* G, int* flags,
                            cudaStream_t s) {
    if (d < 1 || d > 16) return false;
    if (!R) return true;
    DevBuf<double> kb(size_t(C), s), ky(size_t(C) * size_t(d), s);
    grad_small_prep_kernel<<<blocks_for(C), 256, 0, s>>>(Y, wy, g, C, d, eps, kscale, kb.get(),
                                                         ky.get());
    const unsigned blocks = unsigned((R * 32 + 255) / 256);
    switch (d) {
#define FSKB_GS_CASE(DD)                                                                     \
    case DD:                                                                                 \
        grad_small_fp64_kernel<DD><<<blocks, 256, 0, s>>>(X, wx, f, Y, kb.get(), ky.get(),   \
                                                          row_begin, R, C, eps, G, flags);   \
        break;
        FSKB_GS_CASE(1) FSKB_GS_CASE(2) FSKB_GS_CASE(3) FSKB_GS_CASE(4) FSKB_GS_CASE(5)
        FSKB_GS_CASE(6) FSKB_GS_CASE(7) FSKB_GS_CASE(8) FSKB_GS_CASE(9) FSKB_GS_CASE(10)
        FSKB_GS_CASE(11) FSKB_GS_CASE(12) FSKB_GS_CASE(13) FSKB_GS_CASE(14) FSKB_GS_CASE(15)
        FSKB_GS_CASE(16)
#undef FSKB_GS_CASE
    }
    FSKB_CUDA(cudaGetLastError());
    count_launch(2);
    return true;
}

#define FSKB_INSTANTIATE(T)                                                                     \
    template void launch_lse<T>(const ScoreParams<T>&, int, T*, T*, cudaStream_t);              \
    template void launch_lse_finalize<T>(const T*, const T*, int, int64_t,                      \
                                         const FinalizeArgs<T>&, cudaStream_t);                 \
    template void launch_apply<T>(const ScoreParams<T>&, const T*, const T*, int64_t, const T*, \
                                  const T*, int64_t, T*, cudaStream_t);                         \
    template void launch_apply_finalize<T>(const T*, int64_t, int64_t, const T*, const T*,      \
                                           const T*, const T*, T, T*, int*, cudaStream_t);      \
    template void launch_log<T>(const T*, T*, int64_t, cudaStream_t);                           \
    template void launch_neg_sqnorm<T>(const T*, int64_t, int64_t, T, T*, cudaStream_t);        \
    template void launch_grad_epilogue<T>(const T*, const T*, const T*, const T*, const T*,     \
                                          int64_t, int64_t, T, T*, int*, cudaStream_t);

FSKB_INSTANTIATE(float)
FSKB_INSTANTIATE(double)

}  // namespace fskb
