/*
 * stochinv_b200 — C ABI of the B200-native RBFGS / AdaRBFGS iteration.
 *
 * This is the drop-in boundary for the reference's hot path (arxiv 1602.01768,
 * `stochinv` C++ library).  The reference has no FFI layer; its boundary is the
 * C++ API in proj/include/stochinv/ (SURVEY §8b).  Each entry point below names
 * the reference interface it replaces.  The C++ facade
 * include/stochinv_b200.hpp re-exposes the reference signatures on top of it;
 * INTEGRATION.md shows the ctypes / C++ bindings.
 *
 * Conventions
 *   - Dense matrices are column-major doubles (Eigen::MatrixXd layout,
 *     proj/include/stochinv/types.hpp:8).  Pointers named *_host are host
 *     memory; *_dev are device memory of the context's GPU.
 *   - Every function returns an si_status.  Non-zero codes mirror the
 *     reference's exception classes and CLI exit codes
 *     (proj/include/stochinv/errors.hpp:9-26, tools/stochinv_cli.cpp:269-285):
 *     SI_ERR_CONFIG = ConfigError / std::invalid_argument (exit 2),
 *     SI_ERR_NUMERICAL = NumericalError / GramRankDeficientError (exit 3),
 *     SI_ERR_IO = IoError (exit 4).  si_last_error() returns the message
 *     (thread-local).  SI_ERR_RESAMPLE is the NumericalError a step kernel
 *     raises when the sketched Gram fails (callers redraw, simi.cpp:331-333).
 *   - A context is owned by one host thread (the reference's single-owner
 *     inverter state); kernels run on the context stream.
 *   - There is no CPU fallback: without a CUDA device every call that needs
 *     the GPU returns SI_ERR_CUDA.
 */
#ifndef STOCHINV_B200_H
#define STOCHINV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum si_status {
    SI_OK = 0,
    SI_ERR_CONFIG = 2,
    SI_ERR_NUMERICAL = 3,
    SI_ERR_IO = 4,
    SI_ERR_CUDA = 5,
    SI_ERR_RESAMPLE = 6
} si_status;

typedef enum si_symmetry { SI_GENERAL = 0, SI_SYMMETRIC = 1, SI_SPD = 2 } si_symmetry; /* problem_matrix.hpp:7 */

typedef enum si_sketch_kind {
    SI_SKETCH_GAUSSIAN = 0,           /* SketchRule::gaussian(q), host RngStream draws (bit-exact parity mode) */
    SI_SKETCH_GAUSSIAN_DEVICE = 1,    /* Gaussian from the device counter-based RNG (Philox4x32-10) */
    SI_SKETCH_COORDINATE_BLOCK = 2,   /* SketchRule::coordinate_block(n, q), sketching.cpp:20-28 */
    SI_SKETCH_ADAPTIVE_COLS = 3,      /* SketchRule::adaptive_cols(n, q): contiguous blocks + Eq 8.2 */
    SI_SKETCH_ADAPTIVE_GAUSS = 4,     /* SketchRule::adaptive_gauss(q) */
    SI_SKETCH_ADAPTIVE_COLS_UNIFORM = 5, /* paper sampler: q distinct coordinates uniformly */
    SI_SKETCH_ADAPTIVE_GAUSS_DEVICE = 6  /* adaptive_gauss with device RNG */
} si_sketch_kind;

typedef enum si_probability { SI_PROB_UNIFORM = 0, SI_PROB_CONVENIENT = 1 } si_probability;
typedef enum si_termination { SI_TOL_REACHED = 0, SI_MAX_ITERS = 1, SI_TERMINATION_ERROR = 2 } si_termination;

typedef struct si_context si_context;
typedef struct si_problem si_problem;

/* HistoryPoint, simi.hpp:73-78 */
typedef struct si_history_point {
    int64_t k;
    double residual; /* ||I - A X_k||_F / ||I - A X_0||_F */
    double flops;    /* cumulative, step kernels only (flops.cpp tallies) */
    double seconds;  /* cumulative, step kernels only (device time) */
} si_history_point;

/* Per-checkpoint observer (an addition; the reference has none). */
typedef void (*si_checkpoint_fn)(const si_history_point* point, void* user);

/* InverterConfig (simi.hpp:59-71) / AdaConfig (adarbfgs.hpp:46-56) */
typedef struct si_inverter_config {
    int sketch;        /* si_sketch_kind */
    int probabilities; /* si_probability, coordinate_block only */
    int64_t q;
    double tol;                 /* relative residual target; 0 = unreachable */
    int64_t max_iters;          /* default 1000 */
    double time_budget_seconds; /* 0 = unlimited; checked at checkpoints */
    uint64_t seed;
    int64_t residual_every_k; /* TrackOptions::residual_every_k, default 10 */
    int track_flops;
    int track_wall_time;
    int max_redraws;          /* default 100 */
    const double* x0_host;    /* optional X0 (RBFGS) or L0 (AdaRBFGS), n×n; NULL = identity */
    si_checkpoint_fn on_checkpoint;
    void* user;
    int update;               /* si_update: MethodSpec::named_method for run_inverter (default bfgs) */
} si_inverter_config;

/* The named updates on the B200 path (qn_updates.hpp UpdateName subset, SURVEY §8 a1 + f3). */
typedef enum si_update { SI_UPDATE_BFGS = 0, SI_UPDATE_PSB = 1, SI_UPDATE_AIP = 2, SI_UPDATE_DFP = 3 } si_update;
/* run_baseline methods (baselines.hpp:36). */
typedef enum si_baseline { SI_BASELINE_NEWTON_SCHULZ = 0, SI_BASELINE_MINIMAL_RESIDUAL = 1 } si_baseline;

/* RunResult + InverterState scalars (simi.hpp:82-96) */
typedef struct si_run_result {
    int termination; /* si_termination */
    int64_t k;
    double max_symmetry_drift;
    double flops;
    double seconds;
    int64_t history_count; /* points produced (may exceed the caller's capacity) */
    int64_t redraws;
    double condition_estimate; /* AdaRBFGS cond(L), n <= 256 only; 0 otherwise */
    char message[256];
} si_run_result;

/* ---- library / context ----------------------------------------------- */
const char* si_last_error(void);
const char* si_version(void);
void si_default_config(si_inverter_config* cfg); /* reference defaults (simi.hpp:53-71) */

int si_context_create(int device, si_context** out);
/* Run on a caller-provided cudaStream_t (e.g. torch.cuda.current_stream()).  For the legacy default
 * stream (NULL) the context uses a private blocking stream, which is ordered with it implicitly. */
int si_context_create_on_stream(int device, void* cuda_stream, si_context** out);
int si_context_destroy(si_context* ctx);

/* ---- multi-GPU contexts -----------------------
 * A multi-GPU context drives P ranks over NCCL (NVLink / NVSwitch); si_run_inverter (bfgs),
 * si_run_adarbfgs and the si_solver_* calls on it run the iteration sharded — X's upper
 * triangle in 2P row chunks (RBFGS), L in P row panels (AdaRBFGS), A replicated — with the
 * reference's run semantics (run_inverter simi.hpp:105, run_adarbfgs adarbfgs.hpp:59).
 * Problems created on it are replicated to every local rank.  NCCL is loaded on demand.
 *   _multi:    one process driving `ndev` distinct devices (ncclCommInitAll);
 *   _rank:     one process per GPU (torchrun / MPI): every rank passes the id rank 0 got
 *              from si_nccl_unique_id (the caller broadcasts the bytes); cuda_stream may be
 *              NULL (private stream) or the caller's stream; x_out / l_out of the drivers are
 *              filled on rank 0 only;
 *   _loopback: `nranks` virtual ranks on ONE device sharing one stream, the collectives
 *              replayed as device copies — a single-GPU harness for the P > 1 logic (tests),
 *              not a performance configuration. */
#define SI_NCCL_ID_BYTES 128
int si_nccl_unique_id(void* id_out);
int si_context_create_multi(const int* devices, int ndev, si_context** out);
int si_context_create_rank(int device, void* cuda_stream, int nranks, int rank, const void* nccl_id, si_context** out);
int si_context_create_loopback(int device, int nranks, si_context** out);
/* global rank count, the global rank of this process's first local rank, local rank count
 * (1, 0, 1 for a single-GPU context) */
int si_context_ranks(si_context* ctx, int* nranks, int* first_rank, int* local_ranks);
int si_context_synchronize(si_context* ctx);
/* si_run_inverter / si_run_adarbfgs keep their last workspace (the n×n iterate and panels,
 * when it is at most a quarter of device memory) in the context so a rerun of the same
 * shape allocates nothing; this frees it now (it is also freed by si_context_destroy). */
int si_context_release_workspaces(si_context* ctx);
/* Kernel launches issued by this context so far (the bench's gpu_launches). */
int64_t si_context_launch_count(si_context* ctx);
/* Draw log (an addition for parity checks): from now on the drivers append every executed
 * sampling attempt's outcome to buf (up to cap entries) — the block index for coordinate_block /
 * adaptive_cols (rng.hpp:28-36 categorical), the q coordinates for adaptive_cols_uniform —
 * in draw order, rejected attempts included.  NULL turns it off.  si_context_draw_count returns
 * the entries produced (may exceed cap). */
int si_context_set_draw_log(si_context* ctx, int64_t* buf, int64_t cap);
int64_t si_context_draw_count(si_context* ctx);
/* Per-kernel-class device timing (CUDA events around each launch). */
int si_context_set_profiling(si_context* ctx, int enabled);
/* Returns the number of classes; fills up to cap entries (name, launches, total ms). */
int si_context_profile(si_context* ctx, char (*names)[32], int64_t* launches, double* total_ms, int cap);
int si_context_reset_profile(si_context* ctx);

/* ---- problem matrix: ProblemMatrix(Matrix, Symmetry), problem_matrix.hpp:14 */
int si_problem_create_dense(si_context* ctx, int64_t n, const double* a_host, int symmetry, si_problem** out);
int si_problem_create_dense_device(si_context* ctx, int64_t n, const double* a_dev, int symmetry, si_problem** out);
/* CSR (int64 rowptr, int32 colind, double val), SURVEY §8b item 2 — sparse A (configs 4/5). */
int si_problem_create_csr(si_context* ctx, int64_t n, int64_t nnz, const int64_t* rowptr_host,
                          const int32_t* colind_host, const double* val_host, int symmetry, si_problem** out);
int si_problem_destroy(si_problem* prob);
int64_t si_problem_n(si_problem* prob);
/* ProblemMatrix::validate_spd (problem_matrix.cpp:28-41): SI_ERR_CONFIG if not spd-flagged,
 * SI_ERR_NUMERICAL if the Cholesky fails. */
int si_problem_validate_spd(si_problem* prob);
/* Copy A (dense or densified CSR) to host, n×n column-major. */
int si_problem_get_dense(si_problem* prob, double* a_host);
/* ProblemMatrix load_matrix_market(path), io.hpp:14 / io.cpp:28-121 (same checks and messages,
 * SI_ERR_IO on parse errors).  symmetry < 0 takes the header's (general / symmetric); coordinate
 * files stay sparse (CSR) when keep_sparse != 0 instead of being densified (io.cpp:72). */
int si_problem_load_matrix_market(si_context* ctx, const char* path, int symmetry, int keep_sparse,
                                  si_problem** out);
/* ProblemMatrix build_ridge_hessian(path, lambda), io.hpp:19 / io.cpp:123-166: A = BᵀB + λI from a
 * LIBSVM file, the product on the GPU; SPD-flagged when λ > 0. */
int si_problem_ridge_hessian(si_context* ctx, const char* libsvm_path, double lambda, si_problem** out);
/* ProblemMatrix gen_synthetic(n, seed), io.hpp:23 / io.cpp:168-171: A = ĀᵀĀ, Ā ~ U(0,1) from RngStream(seed). */
int si_problem_synthetic(si_context* ctx, int64_t n, uint64_t seed, si_problem** out);
/* Host-side parse only (no device work): the same reader and error texts as
 * si_problem_load_matrix_market.  info: n, header symmetry, stored entries after
 * mirroring/deduplication.  dense: the n×n column-major matrix the reference's
 * load_matrix_market(path).data() holds. */
int si_io_matrix_market_info(const char* path, int64_t* n, int* symmetric, int64_t* stored);
int si_io_matrix_market_dense(const char* path, double* out_colmajor);
/* LIBSVM scan (io.cpp:128-161): sample and feature counts, SI_ERR_IO on the reference's errors. */
int si_io_libsvm_info(const char* path, int64_t* samples, int64_t* features);

/* ---- step-level drop-ins (host buffers, reference semantics) ----------- */
/* Matrix bfgs_step(const Matrix& x, const Matrix& a, const Matrix& s), qn_updates.hpp:70.
 * Returns SI_ERR_RESAMPLE when SᵀAS is not positive definite (GramRankDeficientError). */
int si_bfgs_step(si_context* ctx, int64_t n, int64_t q, const double* x_host, const double* a_host,
                 const double* s_host, double* x_out_host);
/* Same step with A given as a problem handle (A resident on the device). */
int si_bfgs_step_problem(si_context* ctx, si_problem* prob, int64_t q, const double* x_host, const double* s_host,
                         double* x_out_host);
/* Matrix adarbfgs_update_factor(l, a, stilde), adarbfgs.hpp:28.
 * Returns SI_ERR_RESAMPLE when an inverse square root hits its floor. */
int si_adarbfgs_update_factor(si_context* ctx, int64_t n, int64_t q, const double* l_host, const double* a_host,
                              const double* stilde_host, double* l_out_host);
/* Matrix sym_inv_sqrt(const Matrix& m, double floor_rel = 1e-14), linalg.hpp (linalg.cpp:144-155):
 * r_out (q×q) = M^{-1/2} for symmetric M; SI_ERR_NUMERICAL ("matrix is not positive definite") iff
 * an eigenvalue λ ≤ 1e-14·λmax or λ ≤ 0 — the rule the AdaRBFGS update applies to SᵀAS. */
int si_sym_inv_sqrt(si_context* ctx, int64_t q, const double* m_host, double* r_out_host);
/* Vector adaptive_block_probabilities(l, a, blocks), adarbfgs.hpp:32-33; blocks given in CSR
 * form (block_offsets[nblocks+1], block_indices[n]). */
int si_adaptive_block_probabilities(si_context* ctx, int64_t n, const double* l_host, const double* a_host,
                                    int64_t nblocks, const int64_t* block_offsets, const int64_t* block_indices,
                                    double* p_out_host);
/* psb_step / aip_step (qn_updates.hpp, qn_updates.cpp:121-129, 147-152) and the dfp_step pair
 * (:154-174), host buffers; SI_ERR_RESAMPLE on a non-PD sketched Gram. */
int si_psb_step(si_context* ctx, int64_t n, int64_t q, const double* x_host, const double* a_host,
                const double* s_host, double* x_out_host);
int si_aip_step(si_context* ctx, int64_t n, int64_t q, const double* x_host, const double* a_host,
                const double* s_host, double* x_out_host);
int si_dfp_step(si_context* ctx, int64_t n, int64_t q, const double* x_host, const double* x_inv_host,
                const double* a_host, const double* s_host, double* x_out_host, double* x_inv_out_host);
/* Newton-Schulz / minimal-residual building blocks (baselines.hpp:13-33, linalg.cpp:106-129). */
int si_newton_schulz_step(si_context* ctx, int64_t n, const double* x_host, const double* a_host, double* x_out_host);
int si_newton_schulz_init(si_context* ctx, si_problem* prob, uint64_t seed, double* x_out_host);
int si_spectral_norm_estimate(si_context* ctx, si_problem* prob, int iters, uint64_t seed, double* out);
int si_mr_step_cached(si_context* ctx, int64_t n, const double* x_host, const double* r_host, const double* a_host,
                      double* x_out_host, double* r_out_host, double* alpha, int* stagnated);
int si_mr_init(si_context* ctx, si_problem* prob, double* x_out_host);
/* ||I - A X||_F (simi.cpp:242-244). */
int si_residual(si_context* ctx, si_problem* prob, const double* x_host, double* out);

/* ---- drivers --------------------------------------------------------- */
/* RunResult run_inverter(const InverterConfig&) for MethodSpec::named_method(bfgs),
 * simi.hpp:105 / simi.cpp:217-381.  x_out_host (n×n) receives the final X. */
int si_run_inverter(si_context* ctx, si_problem* prob, const si_inverter_config* cfg, double* x_out_host,
                    si_history_point* history, int64_t history_cap, si_run_result* result);
/* run_inverter for any si_update (cfg->update); x_inv_out_host (optional) receives the tracked
 * inverse iterate of dfp (simi.cpp:227-229; tracks_inverse_iterate), ignored otherwise. */
int si_run_inverter_pair(si_context* ctx, si_problem* prob, const si_inverter_config* cfg, double* x_out_host,
                         double* x_inv_out_host, si_history_point* history, int64_t history_cap,
                         si_run_result* result);
/* RunResult run_baseline(const BaselineConfig&), baselines.hpp:68 / baselines.cpp:52-151: method
 * si_baseline; uses cfg->tol, max_iters, time_budget_seconds, seed (spectral-norm start vector),
 * residual_every_k, track_*, x0_host (NULL = the method's paper initialisation), on_checkpoint. */
int si_run_baseline(si_context* ctx, si_problem* prob, int method, const si_inverter_config* cfg,
                    double* x_out_host, si_history_point* history, int64_t history_cap, si_run_result* result);
/* RunResult run_adarbfgs(const AdaConfig&), adarbfgs.hpp:59 / adarbfgs.cpp:91-200.
 * l_out_host (optional) receives L; x_out_host (optional) receives X = L Lᵀ. */
int si_run_adarbfgs(si_context* ctx, si_problem* prob, const si_inverter_config* cfg, double* l_out_host,
                    double* x_out_host, si_history_point* history, int64_t history_cap, si_run_result* result);

/* ---- device-resident solver (bench / multi-GPU plumbing) -------------- */
typedef struct si_solver si_solver;
typedef enum si_method { SI_METHOD_RBFGS = 0, SI_METHOD_ADARBFGS = 1 } si_method;
int si_solver_create(si_context* ctx, si_problem* prob, int method, int sketch, int64_t q, uint64_t seed,
                     si_solver** out);
int si_solver_destroy(si_solver* s);
int si_solver_set_identity(si_solver* s);
int si_solver_set_iterate(si_solver* s, const double* host);  /* X (RBFGS) or L (AdaRBFGS) */
int si_solver_get_iterate(si_solver* s, double* host);
/* Device pointer to the n×n iterate (column-major, ld n). */
double* si_solver_iterate_device(si_solver* s);
/* Run `iters` iterations with device-side sketches, no host round trip except the
 * resample check; returns SI_ERR_NUMERICAL if max_redraws is exceeded. */
int si_solver_step(si_solver* s, int64_t iters);
/* One iteration with a host-supplied sketch (S for RBFGS, coordinate indices for AdaRBFGS cols). */
int si_solver_step_with_sketch(si_solver* s, const double* s_host, const int64_t* idx_host);
int si_solver_residual(si_solver* s, double* out); /* absolute ||I - A X||_F */
int64_t si_solver_redraws(si_solver* s);

/* ---- device-pointer operations ---------------------------------------
 * The row-sharded multi-GPU driver (paper_1602_01768_b200/dist.py) composes an
 * RBFGS iteration from these on each rank's panels; pointers are device memory
 * of the context's GPU, column-major.  All are asynchronous on the context
 * stream except si_rbfgs_core_device (reads the PD status) and
 * si_residual_rows_device (returns a host scalar). */
/* C = alpha·op(A)·op(B) + beta·C.  A is M×K (a_kmajor: A(m,k) = A[m*lda + k], else A[m + k*lda]);
 * B is K×N (b_kmajor: B(k,n) = B[k + n*ldb], else B[n + k*ldb]); FP64 DMMA. */
int si_gemm_device(si_context* ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int a_kmajor,
                   const double* B, int64_t ldb, int b_kmajor, double* C, int64_t ldc, double alpha, double beta);
/* Y (m×k, ld ldy) = A_rows·P for a CSR row panel on the device (m rows, int64 rowptr relative to
 * the panel, int32 global column indices < n) and a dense n×k operand P (ld ldp): the sharded
 * drivers' A·S for sparse A (configs 4/5). */
int si_spmm_csr_device(si_context* ctx, int64_t m, int64_t n, const int64_t* rowptr, const int32_t* colind,
                       const double* val, const double* P, int64_t ldp, int64_t k, double* Y, int64_t ldy);
/* X (m×m symmetric, ld ldx) += V·Uᵀ (V, U m×k) on the upper tiles, written mirrored (exactly
 * symmetric): the K-SYMUPD kernel, used on the diagonal blocks of the symmetric sharded driver. */
int si_symupd_device(si_context* ctx, int64_t m, int64_t k, const double* V, int64_t ldv, const double* U,
                     int64_t ldu, double* X, int64_t ldx);
/* S (n×q, ld lds) ~ N(0,1) from Philox4x32-10(seed, draw): identical bytes on every rank. */
int si_sketch_gaussian_device(si_context* ctx, double* S, int64_t n, int64_t q, int64_t lds, uint64_t seed,
                              uint64_t draw);
/* From P = [SᵀY | YᵀW] (q×2q, ld ldp) build M = [[G⁻¹ + G⁻¹HG⁻¹, −G⁻¹], [−G⁻¹, 0]] (2q×2q, ld 2q).
 * scratch: 6q² + 2q + 16 doubles.  Returns SI_ERR_RESAMPLE when G = SᵀAS is not positive definite. */
int si_rbfgs_core_device(si_context* ctx, const double* P, int64_t ldp, int64_t q, double* M, double* scratch);
/* The same core, fully asynchronous: the PD status goes to status_dev (one device int, 0 = G
 * positive definite) and M is written as 0 on rejection, so an update enqueued behind it leaves
 * X unchanged.  The caller reads status_dev later (deferred check: the driver enqueues the
 * update and the next iteration before it knows whether this draw is accepted). */
int si_rbfgs_core_device_async(si_context* ctx, const double* P, int64_t ldp, int64_t q, double* M,
                               double* scratch, int* status_dev);
/* Σ_{i<m, j<n} (δ(r0+i, j) − (X_rows·A)(i, j))², X_rows = rows [r0, r0+m) of X (ld ldx), dense A. */
int si_residual_rows_device(si_context* ctx, si_problem* prob, int64_t m, int64_t r0, const double* x_rows,
                            int64_t ldx, double* out_host);
/* AdaRBFGS panel ops (adarbfgs.cpp:12-21 split over row panels).
 * gather: out (rows×q, ld rows) = L[:, idx] for a rows×? panel L (ld ldl), idx on the device. */
int si_gather_columns_device(si_context* ctx, const double* L, int64_t rows, int64_t ldl, const int64_t* idx_dev,
                             int64_t q, double* out);
/* q×n stage: R = G^{-1/2} (q×q) and B = T − R·Z (q×n, ld q) from the all-reduced G and Z = (AS)ᵀL.
 * Coordinate S̃: St = NULL, T = S̃ᵀ from idx_dev.  Gaussian S̃ (St n×q): T = (S̃ᵀS̃)^{-1/2}S̃ᵀ is
 * also written to T_out (q×n).  scratch: 8q² + 8q + 32 doubles.  SI_ERR_RESAMPLE on the
 * sym_inv_sqrt floor (linalg.cpp:144-155). */
int si_ada_core_device(si_context* ctx, const double* G, int64_t q, const double* Z, int64_t n,
                       const int64_t* idx_dev, const double* St, double* T_out, double* R, double* B, double* scratch);
/* d_j += 2⟨T_j, B_j⟩ − ‖B_j‖² — diag(LᵀAL) carried across L += (S·R)·B; T = NULL
 * means T = S̃ᵀ from idx_dev. */
int si_pdiag_update_device(si_context* ctx, const double* B, int64_t q, int64_t n, const double* T,
                           const int64_t* idx_dev, double* d);
/* Device pointer to the problem's dense A (column-major, ld n); NULL for CSR. */
const double* si_problem_dense_device(si_problem* prob);

/* ---- host RngStream (rng.hpp:13-71), exposed for input generation and tests */
typedef struct si_rng si_rng;
/* FactoredState adarbfgs_step(state, a, rule, rng, max_redraws), adarbfgs.hpp:37-38: one factored
 * update L -> L⁺ drawing from the caller's RngStream (sketch = SI_SKETCH_ADAPTIVE_COLS, _GAUSS or
 * _COLS_UNIFORM); SI_ERR_NUMERICAL when max_redraws + 1 draws are rejected. */
int si_adarbfgs_step(si_context* ctx, si_problem* prob, int sketch, int64_t q, si_rng* rng, int max_redraws,
                     const double* l_host, double* l_out_host);
int si_rng_create(uint64_t seed, si_rng** out);
int si_rng_substream(si_rng* r, uint64_t index, si_rng** out); /* rng.hpp:18-20 */
int si_rng_destroy(si_rng* r);
double si_rng_uniform(si_rng* r);
double si_rng_gaussian(si_rng* r);
int64_t si_rng_categorical(si_rng* r, const double* p, int64_t n);
int64_t si_rng_uniform_index(si_rng* r, int64_t n);
int si_rng_gaussian_matrix(si_rng* r, int64_t rows, int64_t cols, double* out); /* column-major fill */
int si_rng_uniform_matrix(si_rng* r, int64_t rows, int64_t cols, double* out);
int si_rng_uniform_subset(si_rng* r, int64_t n, int64_t q, int64_t* out); /* paper sampler */

#ifdef __cplusplus
}
#endif
#endif /* STOCHINV_B200_H */
