/*
 * fsk_b200.h - C ABI of the B200-native FlashSinkhorn engine (libfsk_b200.so).
 *
 * This is the drop-in boundary. The reference (arxiv/paper_2602_03067,
 * /root/reference/proj) is a C++20 library whose public surface is
 * fsk::stream / fsk::solver in proj/include/fsk/{stream,solver}.hpp. An FFI to
 * that path would bind exactly the functions below: plain pointers and sizes,
 * host (CPU) buffers in row-major order, double precision at the boundary,
 * outputs written into caller-provided buffers, an int status instead of C++
 * exceptions. The C++ API in include/fsk/*.hpp is a thin layer over this ABI
 * that restores the reference's types and exceptions; see INTEGRATION.md for
 * the reference-side binding.
 *
 * Status codes: FSK_OK (0), FSK_EVALIDATION (1) -> fsk::ValidationError,
 * FSK_ENUMERICAL (2) -> fsk::NumericalError, FSK_ECUDA (3) -> device failure.
 * fsk_last_error() returns the message of the last failure on this thread
 * (messages match the reference's exception texts).
 *
 * All compute runs on the current CUDA device with hand-written sm_100a
 * kernels; there is no CPU fallback. Calls are synchronous with respect to
 * the host buffers they receive.
 */
#ifndef FSK_B200_H_
#define FSK_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSK_OK 0
#define FSK_EVALIDATION 1
#define FSK_ENUMERICAL 2
#define FSK_ECUDA 3

/* fsk::DiscreteMeasure (proj/include/fsk/core.hpp:57-65): n x d row-major
 * points, n weights, optional n int32 labels (NULL when unlabeled). */
typedef struct fsk_measure {
    const double* points;
    const double* weights;
    const int32_t* labels;
    int64_t n;
    int64_t d;
} fsk_measure;

/* fsk::CostSpec (core.hpp:78-101). kind 0 = SquaredEuclidean,
 * 1 = LabelAugmented (lambda1 * |x-y|^2 + lambda2 * W[l_i, l_j]). */
typedef struct fsk_cost {
    int32_t kind;
    double lambda1;
    double lambda2;
    const double* label_cost; /* num_labels x num_labels row-major */
    int64_t num_labels;
} fsk_cost;

/* fsk::TileConfig (core.hpp:105-108). Only used for the IO-ledger accounting
 * and validation: the GPU tiling is fixed by the kernels. */
typedef struct fsk_tiles {
    int64_t block_rows;
    int64_t block_cols;
} fsk_tiles;

/* fsk::IoLedger (proj/include/fsk/ledger.hpp:12-40). Counters are ADDED to. */
typedef struct fsk_ledger {
    uint64_t slow_to_fast_scalars;
    uint64_t fast_to_slow_scalars;
    uint64_t kernel_invocations;
    uint64_t transport_vector_applies;
    uint64_t transport_matrix_applies;
    uint64_t hadamard_applies;
} fsk_ledger;

/* fsk::SinkhornConfig (core.hpp:113-121). schedule 0 = Alternating,
 * 1 = Symmetric; precision 0 = Single, 1 = Double. */
typedef struct fsk_config {
    double eps;
    int32_t schedule;
    int32_t max_iters;
    double marginal_tol;
    double eps_scaling_factor;
    int32_t extra_iters_at_final_eps;
    int32_t precision;
} fsk_config;

/* fsk::solver::SolveReport (proj/include/fsk/solver.hpp:8-14). The caller
 * provides f_hat (n), g_hat (m) and eps_history (eps_history_cap) buffers. */
typedef struct fsk_report {
    double* f_hat;
    double* g_hat;
    double* eps_history;
    int64_t eps_history_cap;
    int32_t iterations;
    double marginal_violation;
    double dual_cost;
    double eps;
} fsk_report;

/* HvpConfig: damping tau, CG tolerance eta, CG cap. */
typedef struct fsk_hvp_config {
    double tau;
    double cg_tol;
    int32_t cg_max_iters;
} fsk_hvp_config;

typedef struct fsk_hvp_report {
    int32_t cg_iters;
    double cg_rel_residual;
    int32_t converged;
} fsk_hvp_report;

const char* fsk_last_error(void);

/* ---- streaming half-steps and transport operators ------------------------ */

/* fsk::stream::update_f_hat (stream.hpp:20-21, stream.cpp:270-281) */
int fsk_update_f_hat(const fsk_measure* src, const fsk_measure* tgt, const double* g_hat,
                     const fsk_cost* cost, double eps, const fsk_tiles* tiles, fsk_ledger* ledger,
                     double* out_f_hat);

/* fsk::stream::update_g_hat (stream.hpp:24-25, stream.cpp:283-294) */
int fsk_update_g_hat(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                     const fsk_cost* cost, double eps, const fsk_tiles* tiles, fsk_ledger* ledger,
                     double* out_g_hat);

/* fsk::stream::symmetric_update (stream.hpp:30-32, stream.cpp:296-322) */
int fsk_symmetric_update(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                         const double* g_hat, double eps, const fsk_cost* cost,
                         const fsk_tiles* tiles, fsk_ledger* ledger, double* out_f_hat,
                         double* out_g_hat);

/* fsk::stream::apply_plan (stream.hpp:37-39, stream.cpp:324-339): out = P V,
 * V is m x p, out n x p. */
int fsk_apply_plan(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                   const double* g_hat, double eps, const fsk_cost* cost, const double* V,
                   int64_t p, const fsk_tiles* tiles, fsk_ledger* ledger, double* out);

/* fsk::stream::apply_plan_adjoint (stream.hpp:42-44, stream.cpp:341-357):
 * out = P^T U, U is n x p, out m x p. */
int fsk_apply_plan_adjoint(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                           const double* g_hat, double eps, const fsk_cost* cost, const double* U,
                           int64_t p, const fsk_tiles* tiles, fsk_ledger* ledger, double* out);

/* fsk::stream::apply_hadamard_plan (stream.hpp:47-49, stream.cpp:359-375):
 * out = (P (.) A B^T) V with A n x r, B m x r, V m x p. */
int fsk_apply_hadamard_plan(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                            const double* g_hat, double eps, const fsk_cost* cost,
                            const double* A, const double* B, int64_t r, const double* V,
                            int64_t p, const fsk_tiles* tiles, fsk_ledger* ledger, double* out);

/* fsk::stream::induced_marginals (stream.hpp:53-55, stream.cpp:377-404) */
int fsk_induced_marginals(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                          const double* g_hat, double eps, const fsk_cost* cost,
                          const fsk_tiles* tiles, fsk_ledger* ledger, double* out_r,
                          double* out_c);

/* fsk::stream::update_f_hat_f32 / update_g_hat_f32 (stream.hpp:66-71,
 * stream.cpp:437-451): FloatCloud inputs (float points n x d, float weights).
 * Runs the single-precision engine: tcgen05 split-fp16 tensor-core kernel for
 * d >= 32, CUDA-core FMA kernel for small d. */
int fsk_update_f_hat_f32(const float* src_points, const float* src_weights, int64_t n,
                         const float* tgt_points, const float* tgt_weights, int64_t m, int64_t d,
                         const float* g_hat, float eps, const fsk_tiles* tiles,
                         fsk_ledger* ledger, float* out_f_hat);
int fsk_update_g_hat_f32(const float* src_points, const float* src_weights, int64_t n,
                         const float* tgt_points, const float* tgt_weights, int64_t m, int64_t d,
                         const float* f_hat, float eps, const fsk_tiles* tiles,
                         fsk_ledger* ledger, float* out_g_hat);

/* Closed-form scalar-transfer schedules (stream.hpp:76-91, stream.cpp:459-499) */
uint64_t fsk_io_count_f_update(int64_t n, int64_t m, int64_t d, const fsk_tiles* tiles);
uint64_t fsk_io_count_g_update(int64_t n, int64_t m, int64_t d, const fsk_tiles* tiles);
uint64_t fsk_io_count_symmetric_update(int64_t n, int64_t m, int64_t d, const fsk_tiles* tiles);
uint64_t fsk_io_count_apply_plan(int64_t n, int64_t m, int64_t d, int64_t p,
                                 const fsk_tiles* tiles);
uint64_t fsk_io_count_apply_plan_adjoint(int64_t n, int64_t m, int64_t d, int64_t p,
                                         const fsk_tiles* tiles);
uint64_t fsk_io_count_apply_hadamard(int64_t n, int64_t m, int64_t d, int64_t r, int64_t p,
                                     const fsk_tiles* tiles);
uint64_t fsk_io_count_induced_marginals(int64_t n, int64_t m, int64_t d, const fsk_tiles* tiles);

/* fsk::stream::tiles_fit_sram (stream.hpp:95-96, stream.cpp:501-505) */
int fsk_tiles_fit_sram(const fsk_tiles* tiles, int64_t d, int64_t sram_scalars);

/* fsk::stream::debug_break_lse (stream.hpp:98, stream.cpp:268): negative
 * control - flips the online-LSE rescale exponent in every kernel. */
void fsk_debug_break_lse(int broken);

/* ---- solver ------------------------------------------------------------- */

/* fsk::solver::sinkhorn_solve (solver.hpp:17-19, solver.cpp:121-129). The
 * whole iteration loop runs device-resident. */
int fsk_sinkhorn_solve(const fsk_measure* src, const fsk_measure* tgt, const fsk_cost* cost,
                       const fsk_config* cfg, const fsk_tiles* tiles, fsk_ledger* ledger,
                       fsk_report* report);

/* Warm-started solve (the downstream re-solve loops of SPEC.md:656):
 * sinkhorn_solve from the caller's shifted potentials (f_init n, g_init m) instead
 * of the reference init f_hat = -alpha, g_hat = -beta (solver.cpp:27-32); same
 * schedule, stopping rule and report. out_grad (n x d, nullable) as in
 * fsk_sinkhorn_solve_grad. */
int fsk_sinkhorn_solve_warm(const fsk_measure* src, const fsk_measure* tgt, const fsk_cost* cost,
                            const fsk_config* cfg, const fsk_tiles* tiles, fsk_ledger* ledger,
                            const double* f_init, const double* g_init, fsk_report* report,
                            double* out_grad);

/* fsk::solver::dual_cost (solver.hpp:23-25, solver.cpp:131-143) */
int fsk_dual_cost(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                  const double* g_hat, double eps, const fsk_cost* cost, const fsk_tiles* tiles,
                  fsk_ledger* ledger, double* out);

/* fsk::solver::sinkhorn_divergence_mixed (solver.hpp:35-40, solver.cpp:145-153);
 * fsk::solver::sinkhorn_divergence is the call with the same spec thrice. */
int fsk_sinkhorn_divergence_mixed(const fsk_measure* mu, const fsk_measure* nu,
                                  const fsk_cost* cost_cross, const fsk_cost* cost_mu,
                                  const fsk_cost* cost_nu, const fsk_config* cfg,
                                  const fsk_tiles* tiles, fsk_ledger* ledger, double* out);

/* Batched debiased divergences: `pairs` independent (mu_k, nu_k), each three
 * solves, results in out[k]. One call, device-resident (cfg5 workload). */
int fsk_sinkhorn_divergence_batch(const fsk_measure* mus, const fsk_measure* nus, int64_t pairs,
                                  const fsk_cost* cost, const fsk_config* cfg,
                                  const fsk_tiles* tiles, fsk_ledger* ledger, double* out);

/* ---- SPEC modules the reference specifies but never implemented ----------- */

/* autodiff.grad_source: G = 2 (diag(r) X - P Y), n x d. */
int fsk_grad_source(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                    const double* g_hat, double eps, const fsk_cost* cost, const fsk_tiles* tiles,
                    fsk_ledger* ledger, double* out_grad);

/* autodiff.grad_target: G = 2 (diag(c) Y - P^T X), m x d. */
int fsk_grad_target(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                    const double* g_hat, double eps, const fsk_cost* cost, const fsk_tiles* tiles,
                    fsk_ledger* ledger, double* out_grad);

/* autodiff.barycentric_projection: T = diag(r)^-1 P Y. */
int fsk_barycentric_projection(const fsk_measure* src, const fsk_measure* tgt,
                               const double* f_hat, const double* g_hat, double eps,
                               const fsk_cost* cost, const fsk_tiles* tiles, fsk_ledger* ledger,
                               double* out);

/* Forward + gradient in one call (the cfg2/cfg3 workload): sinkhorn_solve,
 * then grad_source at the returned potentials, without leaving the device. */
int fsk_sinkhorn_solve_grad(const fsk_measure* src, const fsk_measure* tgt, const fsk_cost* cost,
                            const fsk_config* cfg, const fsk_tiles* tiles, fsk_ledger* ledger,
                            fsk_report* report, double* out_grad);

/* hvp.hvp_apply (Thm. 3.5): HVP of OT_eps w.r.t. X
 * along A (n x d) at the given potentials, damped Schur-complement CG. */
int fsk_hvp_apply(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                  const double* g_hat, double eps, const fsk_cost* cost, const double* A,
                  const fsk_hvp_config* hcfg, const fsk_tiles* tiles, fsk_ledger* ledger,
                  double* out, fsk_hvp_report* hrep);
/* Same contract in single precision (the paper's strict-FP32 HVP):
 * fp32 device problem; when the tensor path is enabled (FSK_TENSOR_MODE / d >= 32)
 * every transport-vector application runs on the tcgen05 split-fp16 kernel.
 * Squared-Euclidean cost only. */
int fsk_hvp_apply_single(const fsk_measure* src, const fsk_measure* tgt, const double* f_hat,
                         const double* g_hat, double eps, const fsk_cost* cost, const double* A,
                         const fsk_hvp_config* hcfg, const fsk_tiles* tiles, fsk_ledger* ledger,
                         double* out, fsk_hvp_report* hrep);

/* ---- device engine (device-resident, sharded; used for multi-GPU) ---------- */

/* An engine holds one problem resident in HBM (fp32 clouds, log-weights, the
 * tcgen05 operand images). Potentials live in caller-owned device buffers
 * (float, length n / m) so a collective library can all-gather them in place. */
typedef struct fsk_engine fsk_engine;

/* mode: 0 = auto (split-fp16 tensor cores for 1 <= d <= 4096, except small d < 32
 *       problems whose keys fit in shared memory, which run the persistent CUDA-core
 *       loop; measured in profiles/r02_dsweep.md),
 *       1 = force CUDA-core FMA fp32, 2 = force tensor (split-fp16). */
int fsk_engine_create(int device, const double* X, const double* a, int64_t n, const double* Y,
                      const double* b, int64_t m, int64_t d, int mode, fsk_engine** out);
/* Same with the label-augmented cost C_ij = lambda1 |x_i - y_j|^2 + lambda2 W[la_i, lb_j]
 * (CostSpec::LabelAugmented, core.hpp; stream.cpp:73-77): labels int32 in [0, V), W
 * row-major V x V. The tensor path applies lambda2 W / eps in the chunked / general
 * kernels' epilogues (V <= 64), the CUDA-core path in its score tiles. */
int fsk_engine_create_labeled(int device, const double* X, const double* a, const int32_t* la,
                              int64_t n, const double* Y, const double* b, const int32_t* lb,
                              int64_t m, int64_t d, double lambda1, double lambda2,
                              const double* label_cost, int64_t num_labels, int mode,
                              fsk_engine** out);
void fsk_engine_destroy(fsk_engine* e);
/* Sets eps (rebuilds the scaled key images) and the potential buffers. */
int fsk_engine_set_eps(fsk_engine* e, double eps);
int fsk_engine_bind_potentials(fsk_engine* e, float* f_dev, float* g_dev);
/* `stream` arguments below are cudaStream_t handles used as given: NULL is the
 * legacy default stream (CUDA convention), not an engine-private stream, so the
 * engine's kernels are ordered with the caller's collectives on that stream. */
/* Initialise f = -|x|^2, g = -|y|^2 (f = g = 0 unshifted) on rows
 * [row_begin, row_end) of each side. */
int fsk_engine_init_potentials(fsk_engine* e, void* stream);
/* One half-step restricted to rows [row_begin, row_end) of the updated side:
 * side 0 = f-update (rows of X, reads all of g), 1 = g-update (rows of Y).
 * viol_accum (device double*, nullable) receives += sum_i |a_i e^{(old-new)/eps} - a_i|
 * over those rows (the lagged marginal violation of the previous iterate). */
int fsk_engine_half_step(fsk_engine* e, int side, int64_t row_begin, int64_t row_end,
                         double* viol_accum, void* stream);
/* `iters` alternating iterations over all rows (single GPU). On the CUDA-core
 * path the loop is captured once into a CUDA graph and replayed (launch-bound
 * small problems; FSK_GRAPH=0 disables); the tensor path runs it eagerly.
 * `stream` must be a non-NULL stream for graph capture. */
int fsk_engine_iterate(fsk_engine* e, int iters, void* stream);
/* Gradient w.r.t. X for rows [row_begin,row_end): grad_dev (float, (end-begin) x d). */
int fsk_engine_grad(fsk_engine* e, int64_t row_begin, int64_t row_end, float* grad_dev,
                    void* stream);
/* Transport-vector application at the bound potentials: out_dev (double, device)
 * = P v (side 0, v indexed by Y, out by X) or P^T v (side 1). One LSE pass for the
 * row marginal, then the tcgen05 VEC pass (or the fp32 CUDA-core apply). */
int fsk_engine_transport_vec(fsk_engine* e, int side, const float* v_dev, double* out_dev,
                             void* stream);
/* Transport-matrix application at the bound potentials: out_dev (float, rows x p,
 * device) = P V (side 0; V indexed by Y, m x p) or P^T V (side 1; V n x p). One LSE
 * pass, then the tcgen05 general apply kernel (any d, p in passes of 128 columns)
 * or the fp32 CUDA-core apply. */
int fsk_engine_transport_mat(fsk_engine* e, int side, const float* v_dev, int64_t p,
                             float* out_dev, void* stream);
/* Hadamard-weighted transport (apply_hadamard_plan with B = Y, stream.cpp:359-375):
 * out_dev (float, n x p) = (P (.) A Y^T) V for A (n x d) and V (m x p), device. */
int fsk_engine_transport_hadamard(fsk_engine* e, const float* a_dev, const float* v_dev,
                                  int64_t p, float* out_dev, void* stream);
/* Cumulative count of (query tile, key tile) blocks scored in full by tracked
 * tcgen05 LSE passes (warm-bound passes, or screened passes' phase 2); the rest
 * were proven below 2^-64 of every row's max (diagnostics for the bench line).
 * Tracking is adaptive (warm bounds). */
uint64_t fsk_engine_screen_live_tiles(const fsk_engine* e);
/* Fraction of (query tile pair, key tile) blocks in the live-tile set recorded by
 * the last LSE pass of `side` (reused by transport passes at the same potentials);
 * -1 when none. Synchronizes the device (diagnostics). */
double fsk_engine_live_set_fraction(const fsk_engine* e, int side);
/* (query tile, key tile) blocks covered by those tracked passes. */
uint64_t fsk_engine_screen_blocks(const fsk_engine* e);
/* Launch counter of this engine's kernels (for bench accounting). */
/* Fixed-potential transport over row shards (the HVP workspace, SPEC.md:442-446;
 * the multi-GPU HVP of SURVEY §8e). prepare runs the LSE pass of each orientation
 * over rows [f_begin, f_end) of X and [g_begin, g_end) of Y at the bound potentials
 * and eps (tensor path: shards start on 256-row boundaries) and keeps the row
 * LSE, max and induced marginal; it stays valid until the potentials / eps change.
 *   marginal:         out (float, n or m) = r (side 0) / c (side 1), prepared rows
 *   transport_vec_rows:  out (double, rows) = rows [b, e) of P v (side 0, v: m) or
 *                        P^T v (side 1, v: n)
 *   transport_mat_rows:  out (float, rows x p) = rows of P V / P^T V (V: key rows x p);
 *                        a_dev (n x d, side 0 only): the Hadamard form (P (.) A Y^T) V */
int fsk_engine_transport_prepare(fsk_engine* e, int64_t f_begin, int64_t f_end, int64_t g_begin,
                                 int64_t g_end, void* stream);
int fsk_engine_marginal(fsk_engine* e, int side, float* out_dev, void* stream);
int fsk_engine_transport_vec_rows(fsk_engine* e, int side, int64_t row_begin, int64_t row_end,
                                  const float* v_dev, double* out_dev, void* stream);
int fsk_engine_transport_mat_rows(fsk_engine* e, int side, int64_t row_begin, int64_t row_end,
                                  const float* v_dev, int64_t p, const float* a_dev,
                                  float* out_dev, void* stream);

/* LSE passes the tensor path ran so far, by kind: out[0] screened cold passes
 * (5-MMA phase 1 + live blocks), out[1] warm-bound passes, out[2] plain passes. */
void fsk_engine_pass_counts(const fsk_engine* e, uint64_t out[3]);

int64_t fsk_engine_kernel_launches(const fsk_engine* e);
/* Name of the kernel path the engine uses for half-steps ("tcgen05-split3" / "fma-f32"). */
const char* fsk_engine_path(const fsk_engine* e);

/* ---- misc ----------------------------------------------------------------- */
/* Fills out[0..count) with fsk::Rng(seed).normal() (proj/include/fsk/rng.hpp:44-57). */
void fsk_rng_normal_fill(uint64_t seed, double* out, int64_t count);
/* Library build/version string and device check. */
const char* fsk_version(void);
int fsk_device_count(void);

/* Multi-GPU solves inside the library: n >= 1 makes sinkhorn_solve,
 * _solve_grad and _solve_warm (alternating schedule) shard rows of X and Y over
 * devices 0..n-1 of this process - one host thread and stream per device, both
 * clouds resident on each, an NCCL all-gather of the potential shards after every
 * half-step (ncclCommInitAll; the fp64 early stop's violation partials ride in the
 * same NCCL group), marginals / dual / gradient assembled from the shards.
 * n = 0 (default) is the single-device path on the current device. */
int fsk_set_num_devices(int n);
int fsk_num_devices(void);

/* High-water mark (bytes) of the device's default memory pool, which holds every
 * allocation the library makes; reset != 0 restarts it at the current usage.
 * The HVP memory contract (peak <= c (n + m) d scalars, never n m)
 * is asserted through this. */
int64_t fsk_device_peak_bytes(int device, int reset);

/* Page-locked host buffers from a process-wide pool (no reference counterpart: the
 * reference API is host-only). Inputs and outputs of the solve entry points that live
 * in such a buffer (or in any cudaHostRegister'ed memory) move by one DMA instead of
 * being staged through pinned bounce buffers. fsk_host_free returns the block to the
 * pool (cached up to 8 GB for the next fsk_host_alloc of a similar size). NULL on
 * failure (fsk_last_error). */
void* fsk_host_alloc(size_t bytes);
int fsk_host_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* FSK_B200_H_ */
