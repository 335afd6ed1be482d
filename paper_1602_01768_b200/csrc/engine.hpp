// Internal engine interface: device context, problem storage, and the enqueue
// functions of the RBFGS / AdaRBFGS iteration.  Implemented in engine.cu
// (nvcc; kernels + launch logic); used by driver.cpp (host C++: C ABI, drivers,
// reference RNG).  No CUDA kernel code here.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace si {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// errors.hpp:9-22 (ConfigError is a std::invalid_argument, NumericalError a std::runtime_error)
struct ConfigError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct NumericalError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what);

struct KernelStat {
    int64_t launches = 0;
    double ms = 0.0;
};

struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int num_sms = 148;
    double* ws = nullptr;  // split-K partials / reduction scratch
    size_t ws_doubles = 0;
    double* scalar_dev = nullptr;   // 8 doubles
    double* scalar_host = nullptr;  // pinned mirror
    int64_t launches = 0;
    bool profiling = false;
    std::vector<std::string> class_names;
    std::vector<KernelStat> stats;
    struct Pending {
        int cls;
        cudaEvent_t a, b;
    };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> event_pool;
    int* aux_status = nullptr;      // status words of device-pointer entry points

    // second stream + split-K workspace for work that overlaps a single-CTA stage
    // (AdaRBFGS: Z = (AS)ᵀ·L under the inverse square root); fork / join by events
    cudaStream_t side = nullptr, side_hi = nullptr;  // side_hi: highest stream priority
    double* ws_side = nullptr;
    size_t ws_side_doubles = 0;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    void fork(bool high = false);  // side (or side_hi) waits for everything enqueued on `stream` so far
    void join(bool high = false);  // `stream` waits for everything enqueued on side (side_hi) so far
    // run_inverter's bfgs workspace kept between calls (take / keep, driver.cpp)
    struct RbfgsWork* cached_rw = nullptr;
    struct RbfgsWork* take_rbfgs(int64_t n, int64_t q);
    void keep_rbfgs(struct RbfgsWork* w);
    // run_adarbfgs's workspace, same policy
    struct AdaWork* cached_aw = nullptr;
    bool cached_aw_gauss = false;
    struct AdaWork* take_ada(int64_t n, int64_t q, bool gaussian);
    void keep_ada(struct AdaWork* w, bool gaussian);
    double* ensure_ws(size_t doubles);
    int class_id(const char* name);
    void resolve_profile();
    ~Context();
};

// RAII launch accounting: counts the launch and (when profiling) brackets it
// with CUDA events on the context stream.
struct LaunchScope {
    Context& c;
    int cls = -1;
    cudaEvent_t a = nullptr, b = nullptr;
    LaunchScope(Context& ctx, const char* name);
    ~LaunchScope();
};

struct Problem {
    Context* ctx = nullptr;
    int64_t n = 0;
    int symmetry = 2;
    bool dense = true;
    double* a = nullptr;  // dense n×n column-major
    // CSR
    int64_t nnz = 0;
    int64_t* rowptr = nullptr;
    int32_t* colind = nullptr;
    double* val = nullptr;
    bool spd_checked = false;
    bool spd_ok = false;
    ~Problem();
};

// Workspace of one RBFGS iterate (SURVEY App. C1 rank-2q form):
//   U = [S W] (n×2q), Y = A·S, P = Yᵀ·U = [G | H], Ginv, T = H·Ginv,
//   M = [[Ginv + Ginv H Ginv, −Ginv], [−Ginv, 0]], V = U·M, X ← X + V·Uᵀ.
enum UpdateKind { UPD_BFGS = 0, UPD_PSB = 1, UPD_AIP = 2, UPD_DFP = 3 };  // si_update

struct RbfgsWork {
    int64_t n = 0, q = 0;
    int update = UPD_BFGS;
    double* X = nullptr;
    // other named updates (family.cuh): basis buffers, second core, DFP inverse iterate H
    double *Bs = nullptr, *Bs2 = nullptr, *V2 = nullptr, *M2 = nullptr, *H = nullptr, *Ginv2 = nullptr;
    double *Y = nullptr, *U = nullptr, *P = nullptr, *Ginv = nullptr, *T = nullptr, *M = nullptr, *V = nullptr;
    double* factor_scratch = nullptr;
    int* status = nullptr;  // [0] Gram not PD (skip), [1] non-finite iterate, [2] rejected draws,
                            // [3] accepted steps, [4] batch stopped (8 ints)
    unsigned long long* counter = nullptr;
    double* s_pinned = nullptr;  // host staging for host-drawn sketches (lazy: pinned())
    double* lowrank = nullptr;   // n×2q scratch of the rank-2q first checkpoint (lazy)
    double* pinned();
    void alloc(int64_t n, int64_t q, bool own_x);
    void release();
    bool own_x = true;
    // run_inverter's batched device-sketch mode: iterations are enqueued back to back
    // between checkpoints and advance_batch_kernel keeps the accounting (status[3..4])
    bool batch = false;
};

// Workspace of one AdaRBFGS factor update (adarbfgs.cpp:12-21):
//   S = L·S̃, AS = A·S, G = Sᵀ·AS, R = G^{-1/2}, Z = (AS)ᵀ·L,
//   L ← L + (S·R)·(T − R·Z),  T = (S̃ᵀS̃)^{-1/2} S̃ᵀ.
struct AdaWork {
    int64_t n = 0, q = 0;
    double* L = nullptr;
    double *S = nullptr, *AS = nullptr, *G = nullptr, *R = nullptr, *SR = nullptr, *Z = nullptr, *B = nullptr;
    double *St = nullptr, *G2 = nullptr, *R2 = nullptr, *Tm = nullptr;  // Gaussian S̃ path
    double* eig_scratch = nullptr;
    int64_t* idx_dev = nullptr;
    int64_t* idx_pinned = nullptr;
    double* st_pinned = nullptr;
    double* AL = nullptr;  // n×n scratch for residual / probabilities (lazy)
    double* pdiag = nullptr;  // n: diag(LᵀAL), exact or carried by App. C3
    // run_adarbfgs's batched loop: index sets of up to ring_cap attempts (device + pinned),
    // ada_advance_batch_kernel accounting in status[4] (stopped) / status[5] (accepted)
    bool batch = false;
    int64_t* idx_ring = nullptr;
    int64_t* idx_ring_pinned = nullptr;
    int ring_cap = 0;
    void ensure_ring(int cap);
    // the next attempt's sketch pipelined ahead (coordinate sampler, batched loops):
    // S' = L[:, idx'] + SR·B[:, idx'] (= the next L's columns) and A·S', S'ᵀ·A·S' computed on the
    // side stream while the main stream runs this attempt's L update
    const int64_t* idx_next = nullptr;  // device, q entries; null: no next attempt in this batch
    bool have_next = false;
    double *S_next = nullptr, *AS_next = nullptr, *G_next = nullptr, *Bsel = nullptr;
    bool pdiag_valid = false;
    int pdiag_age = 0;       // incremental updates since the last exact refresh
    int pdiag_refresh = 64;  // exact A·L refresh period (SI_PDIAG_REFRESH; 1 = every iteration)
    double* p_pinned = nullptr;
    int* status = nullptr;
    unsigned long long* counter = nullptr;
    void alloc(int64_t n, int64_t q, bool gaussian);
    void release();
};

// ---- engine entry points (engine.cu) -------------------------------------
// external == nullptr && !on_stream: a private non-blocking stream.  on_stream: the caller's
// stream; the legacy default stream (0) is served by a private *blocking* stream, which the
// legacy stream orders against implicitly in both directions (graphs cannot be captured on 0).
Context* context_create(int device, cudaStream_t external, bool on_stream = false);
void problem_upload_dense(Problem& p, const double* host, bool device_src);
void problem_upload_csr(Problem& p, const int64_t* rowptr, const int32_t* colind, const double* val);
bool problem_validate_spd(Problem& p, double* scratch_nn = nullptr);  // blocked Schur-complement pivots (own kernels)
void problem_download_dense(Problem& p, double* host);

// generic dense product C = alpha·op(A)·op(B) + beta·C with leading dimensions
void gemm(Context& c, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, bool a_kmajor, const double* B,
          int64_t ldb, bool b_kmajor, double* C, int64_t ldc, double alpha, double beta, const int* skip = nullptr,
          int* nonfinite = nullptr, const double* Csrc = nullptr);  // Csrc: beta·Csrc (ld ldc) instead of beta·C
// Y = A·P for the problem matrix (dense GEMM or CSR SpMM), P n×k
void apply_a(Context& c, Problem& a, const double* P, int64_t ldp, int64_t k, double* Y, int64_t ldy,
             const int* skip = nullptr);

void spmm_csr_rows(Context& c, int64_t m, int64_t n, const int64_t* rowptr, const int32_t* colind, const double* val,
                   const double* P, int64_t ldp, int64_t k, double* Y, int64_t ldy);
void rbfgs_enqueue_iteration(Context& c, Problem& a, RbfgsWork& w, bool device_sketch, uint64_t seed);
// the q×q stage: Gram inverse (PD check into status[0]) and the 2q×2q core M
void rbfgs_core_enqueue(Context& c, const double* P, int64_t ldp, int64_t q, double* Ginv, double* T, double* M,
                        double* scratch, int* status);
// M from a given G⁻¹ (the part of rbfgs_core_enqueue after the inverse)
void rbfgs_core_tail(Context& c, const double* P, int64_t ldp, int64_t q, const double* Ginv, double* T, double* M,
                     int* status);
// M[0:count) = 0 when status[0] != 0 (the deferred PD check of the sharded driver)
void zero_on_status(Context& c, double* M, int64_t count, const int* status);
// the q×q stage of the single-GPU iteration: G⁻¹ (PD check into status[0]) and Ĝ = G + H
void rbfgs_gram_enqueue(Context& c, const double* P, int64_t ldp, int64_t q, double* Ginv, double* Ghat,
                        double* scratch, int* status);
// Gaussian sketch from Philox(seed, draw): draw read from counter_dev if non-null
void philox_sketch(Context& c, double* S, int64_t n, int64_t q, int64_t lds, uint64_t seed,
                   const unsigned long long* counter_dev, uint64_t draw, const int* skip);
void residual_rows_sq_enqueue(Context& c, Problem& a, int64_t m, int64_t r0, const double* Xrows, int64_t ldx,
                              double* out_dev);
void rbfgs_enqueue_sketch_upload(Context& c, RbfgsWork& w);  // s_pinned -> S
// sum of squares of I − A·X into *out_dev (no n×n write); returns nothing (async)
void residual_sq_enqueue(Context& c, Problem& a, const double* X, double* out_dev, double* scratch_nxn);
// ‖I − A‖²_F: the base residual when X0 = I (default), O(n²) instead of 2n³
void identity_residual_sq_enqueue(Context& c, Problem& a, double* out_dev);
// ‖I − A·(I + sign·V·Uᵀ)‖²_F with V, U n×k (dense A): the k = 1 checkpoint from X0 = I, 4n²k flops
void lowrank_residual_sq_enqueue(Context& c, Problem& a, int64_t k, const double* V, int64_t ldv, const double* U,
                                 int64_t ldu, double sign, double* P, double* out_dev);
void factored_residual_sq_enqueue(Context& c, Problem& a, const double* L, double* AL, double* out_dev);
void set_identity(Context& c, double* X, int64_t n);

void ada_enqueue_update(Context& c, Problem& a, AdaWork& w, int mode /*0 cols idx, 1 gaussian host, 2 gaussian dev*/,
                        uint64_t seed);
void ada_enqueue_probabilities(Context& c, Problem& a, AdaWork& w);
// ---- family.cuh: psb / aip / dfp iterations and the NS / MR baselines ----
void family_alloc(RbfgsWork& w, int update);
void family_release(RbfgsWork& w);
void family_enqueue_iteration(Context& c, Problem& a, RbfgsWork& w, bool device_sketch, uint64_t seed);
void symupd_device(Context& c, int64_t m, int64_t k, const double* V, int64_t ldv, const double* U, int64_t ldu,
                   double* X, int64_t ldx);
// C += A·B (A M×K, B(k, j) = B[j + k·ldb]) on 128×128 persistent tiles seeded from C: the
// sharded driver's off-diagonal update block
void gemm_update(Context& c, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                 int64_t ldb, double* C, int64_t ldc, const int* skip, int* nonfinite);
// K-SYMUPD with the iteration's device flags: skipped when *skip, non-finite results flagged
void symupd_ex(Context& c, int64_t m, int64_t k, const double* V, int64_t ldv, const double* U, int64_t ldu, double* X,
               int64_t ldx, const int* skip, int* nonfinite);
// the same on a trapezoid X (m×ncols, ld ldx): leading m×m block mirrored, the rest plain
void symupd_trapezoid(Context& c, int64_t m, int64_t ncols, int64_t k, const double* V, int64_t ldv, const double* U,
                      int64_t ldu, double* X, int64_t ldx, const int* skip, int* nonfinite);
// ---- shard.cu: helpers of the sharded drivers (shard.cpp) ----
// Y (n×k, ld ldy) from `parts` all-gathered k×mc slots (symmetric_chunks: the 2P-chunk pairing)
void place_rows(Context& c, const double* g, int64_t mc, int parts, bool symmetric_chunks, int64_t n, int64_t k,
                double* Y, int64_t ldy);
// dst (rows×cols, ld ldd) = srcᵀ (src cols×rows, ld lds)
void transpose_block(Context& c, const double* src, int64_t lds, int64_t rows, int64_t cols, double* dst,
                     int64_t ldd);
// Σ over rows [r0, r0+m) of ‖I − X·A‖² for CSR A and a row panel X[R, :] (column-major m×n, ld m)
void csr_residual_rows_sq(Context& c, Problem& a, int64_t m, int64_t r0, const double* Xrows, double* out_dev);
void accumulate(Context& c, double* dst, const double* src, int64_t count);  // dst += src
void combine(Context& c, void* dst, const void* src, int64_t count, bool is_int, bool is_max);  // dst ∘= src
void panel_column_dots(Context& c, const double* AL, const double* L, int64_t m, int64_t n, double* d);
void problem_diagonal(Context& c, Problem& a, double* d);  // d = diag(A)
void ghat_split(Context& c, const double* G, const double* H, int64_t q, double* Ghat, const int* skip);  // Ĝ = G − H'
// enqueue on the context's highest-priority side stream (fork() / join(true) around it)
struct SideHi {
    Context& c;
    cudaStream_t s0;
    double* w0;
    size_t n0;
    explicit SideHi(Context& ctx);
    ~SideHi();
};
void set_identity_rows(Context& c, double* X, int64_t m, int64_t cols, int64_t diag_off);  // X(i, j) = δ(j, i + off)
// the single-GPU iteration's counters: advance_batch_kernel (RBFGS) / ada_advance_batch_kernel
void advance_batch(Context& c, unsigned long long* counter, int* status, bool ada);
void residual_general_sq_enqueue(Context& c, Problem& a, const double* X, double* scratch_nn, double* out_dev);
void column_weights(Context& c, Problem& a, int mode, std::vector<double>& out);
void lu_inverse_device(Context& c, const double* M, int64_t n, double* out);  // SPD M (block inverse)
// G⁻¹ (ld ldo) of an SPD q×q block (ld ldp), any q: fused K-FACTOR (q ≤ 128) or 2×2 block
// recursion on the GEMM engine; status[0] = 1 when a pivot is not > 0.  scratch: 4q² doubles.
void spd_inverse_device(Context& c, const double* P, int64_t ldp, int64_t q, double* ginv, int64_t ldo,
                        double* scratch, int* status);
void spd_inverse_diagonal(Context& c, Problem& a, std::vector<double>& out);
struct BaselineWork {
    int64_t n = 0;
    double *X = nullptr, *Xn = nullptr, *T = nullptr, *R = nullptr, *part = nullptr;
    int* flag = nullptr;
    void alloc(int64_t n);
    void release();
};
double baseline_residual(Context& c, Problem& a, BaselineWork& w);
bool newton_schulz_enqueue(Context& c, Problem& a, BaselineWork& w);
int mr_enqueue(Context& c, Problem& a, BaselineWork& w, double* alpha_out);
double sumsq_device(Context& c, const double* x, int64_t count);
void newton_schulz_init_device(Context& c, Problem& a, BaselineWork& w, double spectral_norm);
void mr_init_device(Context& c, Problem& a, BaselineWork& w);

void ada_core_enqueue(Context& c, const double* G, int64_t q, const double* Z, int64_t n, const int64_t* idx,
                      const double* St, double* G2, double* R2, double* Tq, double* R, double* B, double* scratch,
                      int* st);
// sym_inv_sqrt (linalg.cpp:144-155): R = M^{-1/2}, status[0] = 1 on the floor (λ ≤ 1e-14·λmax or
// λ ≤ 0); scratch 6q² + 8q + 32 doubles, status 8 ints
void sym_inv_sqrt_device(Context& c, const double* M, int64_t q, double* R, double* scratch, int* status);
void gather_columns(Context& c, const double* L, int64_t rows, int64_t ld, const int64_t* idx, int64_t q, double* out);
void pdiag_update(Context& c, const double* B, int64_t q, int64_t n, const double* T, const int64_t* idx,
                  const int* skip, double* d);
void ada_init_pdiag_identity(Context& c, Problem& a, AdaWork& w);  // diag(A): the L = I diagonal  // pdiag = diag(LᵀAL) -> p_pinned (async)

// ---- ingestion (io.cpp) --------------------------------
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct LoadedMatrix {
    int64_t n = 0;
    bool symmetric = false;
    bool sparse = false;
    std::vector<double> dense;  // column-major n×n (array format, or coordinate with keep_sparse = false)
    std::vector<int64_t> rowptr;
    std::vector<int32_t> colind;
    std::vector<double> val;
};
LoadedMatrix load_matrix_market(const std::string& path, bool keep_sparse);  // io.cpp:28-121
struct LibsvmRows {
    int64_t n = 0, m = 0;
    std::vector<std::vector<std::pair<int64_t, double>>> samples;
};
LibsvmRows read_libsvm(const std::string& path);                          // io.cpp:123-157
double* ridge_hessian_device(Context& c, const LibsvmRows& r, double lambda);  // BᵀB + λI, n×n device
double* synthetic_device(Context& c, int64_t n, uint64_t seed);           // ĀᵀĀ (io.cpp:168-176)

}  // namespace si
