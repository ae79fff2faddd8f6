// tcgen05 half-step engine (fp32-accurate split-fp16 tensor-core path).
//
// The X Y^T contraction of a half-step runs on the 5th-gen tensor cores as a
// K = 3d + 16 fp16 GEMM (hi/lo split of both operands, three products, bias
// folded in as three extra K columns), accumulated in fp32 in TMEM; the
// epilogue warps keep the online max / sum-exp per row in registers and write
// only the new potential. Operands are pre-formatted once per eps into
// UMMA-canonical SW128/SW32 tile images so one bulk copy (TMA engine) moves a
// whole key tile. See DESIGN.md "K1 lse_half_step (tcgen05)".
#pragma once

#include <cstdint>

#include "common.h"
#include "core_kernels.h"

namespace fskb {

template <typename T>
struct DevProblem;

class TcHalfStep {
public:
    // 1 <= d <= 4096; d is padded to a multiple of 64 in the images and d > 64
    // runs the chunked kernels (operands streamed 64 features at a time).
    explicit TcHalfStep(DevProblem<float>& P);
    ~TcHalfStep();
    static bool supported(int64_t d);
    int chunks() const;
    // Screening diagnostics: (query tile pair, key tile) blocks scored in full by
    // phase 2 of screened passes, and blocks those passes covered.
    unsigned long long live_tiles() const;
    unsigned long long screened_blocks() const;
    // LSE passes run so far: [screened cold, warm-bound, plain]
    void pass_counts(unsigned long long out[3]) const;
    // Fraction of (query tile pair, key tile) blocks in the live set of the last
    // LSE pass of `side` (-1 when none is recorded); synchronizes the device.
    double live_set_fraction(int side) const;

    // (Re)builds the scaled key images for this eps (O((n+m) d) work).
    void set_eps(DevProblem<float>& P, double eps);
    // Forget the skip state carried from earlier passes (warm bounds, pass-kind
    // history): a solve restarted from fresh potentials then runs exactly like the
    // first solve of the problem, whatever ran before (history-independent bits).
    void reset_history(cudaStream_t s);

    // One half-step for rows [row_begin, row_end) of `side` (0: f from g over
    // keys Y, 1: g from f over keys X). FinalizeArgs pointers address full-length
    // vectors (row i of the side is element i).
    void run(DevProblem<float>& P, int side, const float* kpot, float eps,
             const FinalizeArgs<float>& fa, int64_t row_begin, int64_t row_end);

    // Gradient of the EOT loss w.r.t. the query cloud of `side` (side 0: X) for
    // rows [row_begin, row_end): G_i = 2 r_i (x_i - (softmax_j S_ij) y_j) with
    // r_i = w_i exp((pot_i - pot+_i)/eps). Two passes: K1 for
    // the row LSE, then the fused tcgen05 transport kernel. G is (end-begin) x d.
    // pre_*: the row log2 LSE (hi, lo) and marginal of a pass over the same rows
    // at the same potentials (e.g. the solver's final marginals) - skips pass 1.
    void grad(DevProblem<float>& P, int side, const float* kpot, const float* pot, float eps,
              int64_t row_begin, int64_t row_end, float* G, int* flags,
              const float* pre_l2h = nullptr, const float* pre_l2l = nullptr,
              const float* pre_r = nullptr);

    // Keeps the live blocks of the transport plan at potentials (f, g) in HBM
    // (row-normalized fp32, union of both orientations' live sets; needs both sides'
    // live sets recorded at these potentials and l2h0/l2l0/r of side 0); while it
    // is valid, vec() at those potentials sweeps it instead of recomputing scores.
    // Returns false (nothing cached) for d <= 64 or when it would not fit.
    bool build_plan(DevProblem<float>& P, const float* g, const float* f, float eps,
                    const float* l2h0, const float* l2l0, const float* r, int* flags);
    void drop_plan();
    double plan_fraction() const;   // cached blocks / all blocks, -1 when none

    // Re-records the live key-tile set of `side` at fixed potentials with every
    // row's running max seeded just below its true max (mx_nat: the natural-log row
    // max of a pass at the same potentials): only tiles holding terms within 2^-64
    // of a row's max stay live, so the transport passes that follow (HVP/CG) skip
    // the rest. One extra LSE pass.
    void tighten_live(DevProblem<float>& P, int side, const float* kpot, float eps,
                      const float* mx_nat, int* flags, int64_t row_begin = 0,
                      int64_t row_end = -1);

    // Transport-vector application with fixed potentials: out_i = marg_i sum_j
    // 2^(t_ij - L_i) v_j = (P v)_i (side 0) or (P^T v)_j (side 1), given the row
    // LSE of that orientation in log2 units (l2h + l2l) and its induced marginal
    // (from a `run` with out_l2h/out_l2l/out_marg at the same potentials). v is
    // indexed by the key side; out (double) by the updated side.
    void vec(DevProblem<float>& P, int side, const float* kpot, float eps, const float* l2h,
             const float* l2l, const float* marg, const float* v, double* out, int* flags,
             int64_t row_begin = 0, int64_t row_end = -1);

    // Transport-matrix application with fixed potentials: out (rows x p, float) =
    // P V (side 0) or P^T V (side 1) for a general V (key rows x p, float, device),
    // any d, via the tcgen05 general apply kernel (p in passes of 128 columns).
    // With A (rows x d, device): the Hadamard form (P (.) A K^T) V where K is the
    // key cloud (apply_hadamard_plan with B = the key cloud, as in the HVP).
    void apply_mat(DevProblem<float>& P, int side, const float* kpot, float eps, const float* l2h,
                   const float* l2l, const float* marg, const float* V, int64_t p_cols,
                   float* out, int* flags, const float* A = nullptr, int64_t row_begin = 0,
                   int64_t row_end = -1);

private:
    void poll_screen(int side, double max_live);
    struct PassExtras {
        const float* m_init;        // running-max seeds (LSE passes)
        const uint32_t* live_in;    // caller-supplied live set
        int in_splits, in_kps, in_kwords;
        float* plan_out;            // VEC passes: store the visited plan blocks
        const int* plan_slot;
    };
    int pass(DevProblem<float>& P, int side, const float* kpot, float eps, int64_t row_begin,
             int64_t row_end, const float* const* vec, int* flags, DevBuf<double>& pm,
             DevBuf<double>& ps, const PassExtras* ex = nullptr);
    struct Impl;
    Impl* impl_;
};

}  // namespace fskb
