// Device-resident problem and the operations composed from the kernels.
// Used by capi.cpp (host-buffer C ABI) and engine.cpp (device engine).
#pragma once

#include <memory>
#include <vector>

#include "../../include/fsk_b200.h"
#include "common.h"
#include "core_kernels.h"

namespace fskb {

class TcHalfStep;  // tcgen05 split-fp16 half-step (tc_engine.h)

// Per-thread execution context: one non-blocking stream on the current device
// and a device status word.
struct ExecCtx {
    cudaStream_t s = nullptr;
    int* flags = nullptr;  // device int
    int* bad_iter = nullptr;
};
ExecCtx& exec_ctx();
// Keep freed stream-ordered allocations in the device's default pool (release
// threshold = max) instead of returning them to the driver at every sync.
void configure_device_pool(int device);
int read_and_clear_flags(ExecCtx& c);
void throw_for_flags(int flags, const std::string& suffix = "");

template <typename T>
struct DevSide {
    DevBuf<T> pts, w, logw;
    DevBuf<int32_t> lab;
    int64_t n = 0, d = 0;
};

// While alive (one per host thread), DevProblem::upload ships each distinct
// caller measure once and serves repeats from device copies (batch entry points).
struct UploadCacheScope {
    UploadCacheScope();
    ~UploadCacheScope();
    UploadCacheScope(const UploadCacheScope&) = delete;
    UploadCacheScope& operator=(const UploadCacheScope&) = delete;

  private:
    void* prev_;
};

template <typename T>
struct DevProblem {
    DevSide<T> src, tgt;
    DevBuf<double> wtab;
    int64_t wdim = 0;
    bool labeled = false;
    double fscale = 1.0, lambda2 = 0.0;
    cudaStream_t s = nullptr;
    std::shared_ptr<TcHalfStep> tc;  // tensor-core half-step (float only), null = FMA path
    double tc_eps = 0.0;

    void upload(const fsk_measure& a, const fsk_measure& b, const fsk_cost* cost,
                cudaStream_t stream);
    // Single-precision solve ingest (squared Euclidean, float problems): ships the
    // caller's doubles, narrows them on the device and computes there what the host
    // would otherwise scan for: the coordinate finiteness check (returned; the caller
    // throws validate_measure's message) and each row's fp64 squared norm (alpha, beta:
    // device vectors, bit-identical to host_sqnorm) plus the initial potentials
    // f = -alpha, g = -beta when f0 / g0 are given. Synchronizes the stream.
    bool ingest(const fsk_measure& a, const fsk_measure& b, double scale, cudaStream_t stream,
                DevBuf<double>& alpha, DevBuf<double>& beta, T* f0, T* g0);
    // float clouds straight from FloatCloud buffers (squared Euclidean)
    void upload_f32(const float* xa, const float* wa, int64_t n, const float* xb,
                    const float* wb, int64_t m, int64_t d, cudaStream_t stream);

    ScoreParams<T> params(int side, const T* kpot, T eps) const;
    int64_t rows(int side) const { return side == 0 ? src.n : tgt.n; }
    int64_t cols(int side) const { return side == 0 ? tgt.n : src.n; }
};

// One LSE pass over all key columns for every row of `side`, plus epilogues.
template <typename T>
void half_step(DevProblem<T>& P, int side, const T* kpot, T eps, const FinalizeArgs<T>& fa);

// Rows [row_begin, row_end) only; FinalizeArgs pointers address full-length
// vectors. Used by the sharded device engine.
template <typename T>
void half_step_rows(DevProblem<T>& P, int side, const T* kpot, T eps, const FinalizeArgs<T>& fa,
                    int64_t row_begin, int64_t row_end);

// Transport application out = P V (side 0) or P^T V (side 1) given the LSE of
// that orientation (lse, mx from a half_step pass).
template <typename T>
void transport(DevProblem<T>& P, int side, const T* kpot, const T* pot, T eps, const T* lse,
               const T* mx, const T* V, int64_t p, const T* A, const T* B, int64_t r, T* out,
               int* flags);

// CUDA-core fp32 problems: gradient rows [row_begin, row_end) of G = 2 (diag(r) X -
// P Y) evaluated in fp64 (scores, LSE, transport) from the float clouds and
// potentials; out_dev is (row_end - row_begin) x d doubles. fp32 score arithmetic
// alone moves plan entries by |S| 2^-24 (~1e-5 at cfg1), above the gradient contract.
void grad_rows_fp64(const DevProblem<float>& P, const float* f, const float* g, double eps,
                    int64_t row_begin, int64_t row_end, double* out_dev, int* flags,
                    cudaStream_t s);

// Enables the tcgen05 path for a float problem when the shape allows it.
// mode: 0 auto, 1 force FMA, 2 force tensor. Returns true when enabled.
bool enable_tensor_path(DevProblem<float>& P, int mode);
// FSK_TENSOR_MODE (auto | fma | tensor) -> the mode argument above (capi.cpp).
int tensor_mode_from_env();
const char* tensor_path_name(const DevProblem<float>& P);

}  // namespace fskb
