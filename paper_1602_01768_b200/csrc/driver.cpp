// Host side of the drop-in: the C ABI (include/stochinv_b200.h) and the
// run_inverter / run_adarbfgs drivers.  Sampling (RngStream, categorical,
// redraw control flow) stays here on the host so indices and RNG consumption
// follow the reference bit for bit; all matrix arithmetic is enqueued on the
// device through engine.cu.  Compiled with g++ -O3 -march=x86-64-v3 (the
// oracle's flags) so host Gaussian draws match the oracle's bytes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/stochinv_b200.h"
#include "engine.hpp"
#include "host_rng.hpp"

#include "capi_internal.hpp"

using namespace si_capi;


extern "C" {

const char* si_last_error(void) { return g_err.c_str(); }
const char* si_version(void) { return "stochinv_b200 0.1 (sm_100a, FP64 DMMA)"; }

void si_default_config(si_inverter_config* cfg) {
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->sketch = SI_SKETCH_GAUSSIAN;
    cfg->probabilities = SI_PROB_UNIFORM;
    cfg->q = 1;
    cfg->tol = 1e-2;          // simi.hpp:64
    cfg->max_iters = 1000;    // simi.hpp:65
    cfg->residual_every_k = 10;  // simi.hpp:54
    cfg->track_flops = 1;
    cfg->track_wall_time = 1;
    cfg->max_redraws = 100;   // simi.hpp:70
    cfg->update = SI_UPDATE_BFGS;
}

int si_context_create(int device, si_context** out) {
    return guard([&] {
        auto* h = new si_context();
        h->c.reset(si::context_create(device, nullptr));
        *out = h;
    });
}

int si_context_create_on_stream(int device, void* stream, si_context** out) {
    return guard([&] {
        auto* h = new si_context();
        h->c.reset(si::context_create(device, static_cast<cudaStream_t>(stream), true));
        *out = h;
    });
}

int si_context_destroy(si_context* ctx) {
    return guard([&] { delete ctx; });
}

int si_context_synchronize(si_context* ctx) {
    return guard([&] { ck(cudaStreamSynchronize(ctx->c->stream), "sync"); });
}

int si_context_release_workspaces(si_context* ctx) {
    return guard([&] {
        ck(cudaStreamSynchronize(ctx->c->stream), "sync");
        ctx->c->keep_rbfgs(nullptr);
        ctx->c->keep_ada(nullptr, false);
    });
}

int64_t si_context_launch_count(si_context* ctx) { return ctx->c->launches; }

int si_context_set_draw_log(si_context* ctx, int64_t* buf, int64_t cap) {
    ctx->draw_log = buf;
    ctx->draw_cap = buf ? cap : 0;
    ctx->draw_count = 0;
    return SI_OK;
}

int64_t si_context_draw_count(si_context* ctx) { return ctx->draw_count; }

int si_context_set_profiling(si_context* ctx, int enabled) {
    return guard([&] {
        ctx->c->resolve_profile();
        ctx->c->profiling = enabled != 0;
    });
}

int si_context_profile(si_context* ctx, char (*names)[32], int64_t* launches, double* total_ms, int cap) {
    int count = 0;
    const int rc = guard([&] {
        ctx->c->resolve_profile();
        auto& c = *ctx->c;
        count = int(c.class_names.size());
        for (int i = 0; i < count && i < cap; ++i) {
            std::snprintf(names[i], 32, "%s", c.class_names[size_t(i)].c_str());
            launches[i] = c.stats[size_t(i)].launches;
            total_ms[i] = c.stats[size_t(i)].ms;
        }
    });
    return rc == SI_OK ? count : -rc;
}

int si_context_reset_profile(si_context* ctx) {
    return guard([&] {
        ctx->c->resolve_profile();
        for (auto& s : ctx->c->stats) s = si::KernelStat{};
    });
}

// ------------------------------------------------------------- problems ---
static si_problem* new_problem(si_context* ctx, int64_t n, int symmetry) {
    require(n >= 1, "ProblemMatrix: matrix must be square with n >= 1");
    require(symmetry >= 0 && symmetry <= 2, "ProblemMatrix: unknown symmetry flag");
    auto* h = new si_problem();
    h->owner = ctx;
    h->p = std::make_unique<si::Problem>();
    h->p->ctx = ctx->c.get();
    h->p->n = n;
    h->p->symmetry = symmetry;
    return h;
}

int si_problem_create_dense(si_context* ctx, int64_t n, const double* a_host, int symmetry, si_problem** out) {
    return guard([&] {
        std::unique_ptr<si_problem> h(new_problem(ctx, n, symmetry));
        // symmetric / spd flags symmetrize (M + Mᵀ)/2 on the device (problem_matrix.cpp:9-18)
        si::problem_upload_dense(*h->p, a_host, false);
        si::shard_replicate_problem(ctx, h.get());
        *out = h.release();
    });
}

int si_problem_create_dense_device(si_context* ctx, int64_t n, const double* a_dev, int symmetry, si_problem** out) {
    return guard([&] {
        std::unique_ptr<si_problem> h(new_problem(ctx, n, symmetry));
        si::problem_upload_dense(*h->p, a_dev, true);
        si::shard_replicate_problem(ctx, h.get());
        *out = h.release();
    });
}

int si_problem_create_csr(si_context* ctx, int64_t n, int64_t nnz, const int64_t* rowptr, const int32_t* colind,
                          const double* val, int symmetry, si_problem** out) {
    return guard([&] {
        std::unique_ptr<si_problem> h(new_problem(ctx, n, symmetry));
        require(rowptr[0] == 0 && rowptr[n] == nnz, "CSR: rowptr must start at 0 and end at nnz");
        for (int64_t i = 0; i < n; ++i) require(rowptr[i + 1] >= rowptr[i], "CSR: rowptr must be non-decreasing");
        for (int64_t t = 0; t < nnz; ++t) require(colind[t] >= 0 && colind[t] < n, "CSR: column index out of range");
        h->p->nnz = nnz;
        si::problem_upload_csr(*h->p, rowptr, colind, val);
        si::shard_replicate_problem(ctx, h.get());
        *out = h.release();
    });
}

int si_problem_destroy(si_problem* prob) {
    return guard([&] { delete prob; });
}

int64_t si_problem_n(si_problem* prob) { return prob->p->n; }

int si_problem_validate_spd(si_problem* prob) {
    return guard([&] { validate_spd(prob); });
}

int si_problem_get_dense(si_problem* prob, double* a_host) {
    return guard([&] { si::problem_download_dense(*prob->p, a_host); });
}

// ------------------------------------------------------------ steps -------
static void bfgs_step_impl(si_context* ctx, si::Problem& a, int64_t q, const double* x_host, const double* s_host,
                           double* x_out) {
    auto& c = *ctx->c;
    const int64_t n = a.n;
    require(q >= 1, "bfgs_step: q must be >= 1");
    si::RbfgsWork w;
    struct Rel {
        si::RbfgsWork& w;
        ~Rel() { w.release(); }
    } rel{w};
    w.alloc(n, q, true);
    ck(cudaMemcpyAsync(w.X, x_host, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyHostToDevice, c.stream), "h2d");
    std::memcpy(w.pinned(), s_host, size_t(n) * size_t(q) * sizeof(double));
    si::rbfgs_enqueue_sketch_upload(c, w);
    si::rbfgs_enqueue_iteration(c, a, w, false, 0);
    int st[4];
    read_status(c, w.status, st);
    if (st[0]) throw ResampleError("bfgs_step: sketched Gram matrix is not positive definite");
    ck(cudaMemcpyAsync(x_out, w.X, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "d2h");
    ck(cudaStreamSynchronize(c.stream), "sync");
}

int si_bfgs_step(si_context* ctx, int64_t n, int64_t q, const double* x_host, const double* a_host,
                 const double* s_host, double* x_out_host) {
    return guard([&] {
        si::Problem a;
        a.ctx = ctx->c.get();
        a.n = n;
        a.symmetry = SI_GENERAL;  // bfgs_step takes A as given (qn_updates.cpp:176)
        si::problem_upload_dense(a, a_host, false);
        bfgs_step_impl(ctx, a, q, x_host, s_host, x_out_host);
    });
}

int si_bfgs_step_problem(si_context* ctx, si_problem* prob, int64_t q, const double* x_host, const double* s_host,
                         double* x_out_host) {
    return guard([&] { bfgs_step_impl(ctx, *prob->p, q, x_host, s_host, x_out_host); });
}

int si_adarbfgs_update_factor(si_context* ctx, int64_t n, int64_t q, const double* l_host, const double* a_host,
                              const double* stilde_host, double* l_out_host) {
    return guard([&] {
        auto& c = *ctx->c;
        si::Problem a;
        a.ctx = &c;
        a.n = n;
        a.symmetry = SI_GENERAL;
        si::problem_upload_dense(a, a_host, false);
        si::AdaWork w;
        struct Rel {
            si::AdaWork& w;
            ~Rel() { w.release(); }
        } rel{w};
        w.alloc(n, q, true);
        ck(cudaMemcpyAsync(w.L, l_host, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyHostToDevice, c.stream),
           "h2d");
        std::memcpy(w.st_pinned, stilde_host, size_t(n) * size_t(q) * sizeof(double));
        si::ada_enqueue_update(c, a, w, 1, 0);
        int st[4];
        read_status(c, w.status, st);
        if (st[0]) throw ResampleError("sym_inv_sqrt: matrix is not positive definite");
        ck(cudaMemcpyAsync(l_out_host, w.L, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, c.stream),
           "d2h");
        ck(cudaStreamSynchronize(c.stream), "sync");
    });
}

int si_sym_inv_sqrt(si_context* ctx, int64_t q, const double* m_host, double* r_out_host) {
    return guard([&] {
        auto& c = *ctx->c;
        require(q >= 1, "sym_inv_sqrt: matrix must be square with n >= 1");
        double *m = nullptr, *r = nullptr, *scratch = nullptr;
        int* status = nullptr;
        struct Rel {
            double **m, **r, **s;
            int** st;
            ~Rel() {
                for (double** p : {m, r, s})
                    if (*p) cudaFree(*p);
                if (*st) cudaFree(*st);
            }
        } rel{&m, &r, &scratch, &status};
        const size_t qq = size_t(q) * size_t(q);
        ck(cudaMalloc(&m, qq * sizeof(double)), "malloc");
        ck(cudaMalloc(&r, qq * sizeof(double)), "malloc");
        ck(cudaMalloc(&scratch, (6 * qq + 8 * size_t(q) + 32) * sizeof(double)), "malloc");
        ck(cudaMalloc(&status, 8 * sizeof(int)), "malloc");
        ck(cudaMemsetAsync(status, 0, 8 * sizeof(int), c.stream), "memset");
        ck(cudaMemcpyAsync(m, m_host, qq * sizeof(double), cudaMemcpyHostToDevice, c.stream), "h2d");
        si::sym_inv_sqrt_device(c, m, q, r, scratch, status);
        int st[4];
        read_status(c, status, st);
        if (st[0]) throw NumericalError("sym_inv_sqrt: matrix is not positive definite");  // linalg.cpp:150
        ck(cudaMemcpyAsync(r_out_host, r, qq * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "d2h");
        ck(cudaStreamSynchronize(c.stream), "sync");
    });
}

int si_adaptive_block_probabilities(si_context* ctx, int64_t n, const double* l_host, const double* a_host,
                                    int64_t nblocks, const int64_t* offs, const int64_t* idx, double* p_out) {
    return guard([&] {
        auto& c = *ctx->c;
        si::Problem a;
        a.ctx = &c;
        a.n = n;
        a.symmetry = SI_GENERAL;
        si::problem_upload_dense(a, a_host, false);
        si::AdaWork w;
        struct Rel {
            si::AdaWork& w;
            ~Rel() { w.release(); }
        } rel{w};
        w.alloc(n, 1, false);
        ck(cudaMemcpyAsync(w.L, l_host, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyHostToDevice, c.stream),
           "h2d");
        si::ada_enqueue_probabilities(c, a, w);
        ck(cudaStreamSynchronize(c.stream), "sync");
        std::vector<std::vector<si::Index>> blocks(static_cast<size_t>(nblocks));
        for (int64_t b = 0; b < nblocks; ++b)
            for (int64_t t = offs[b]; t < offs[b + 1]; ++t) blocks[size_t(b)].push_back(idx[t]);
        std::vector<double> p;
        block_probabilities(w.p_pinned, blocks, p);
        std::copy(p.begin(), p.end(), p_out);
    });
}

int si_residual(si_context* ctx, si_problem* prob, const double* x_host, double* out) {
    return guard([&] {
        auto& c = *ctx->c;
        const int64_t n = prob->p->n;
        double* X = nullptr;
        ck(cudaMalloc(&X, size_t(n) * size_t(n) * sizeof(double)), "malloc");
        ck(cudaMemcpyAsync(X, x_host, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyHostToDevice, c.stream), "h2d");
        *out = residual_norm(c, *prob->p, X);
        cudaFree(X);
    });
}

// ---------------------------------------------------------- run_inverter ---
// simi.cpp:217-381 for MethodSpec::named_method(UpdateName::bfgs).
static const char* update_name(int u) {
    switch (u) {
        case SI_UPDATE_BFGS: return "bfgs";
        case SI_UPDATE_PSB: return "psb";
        case SI_UPDATE_AIP: return "aip";
        case SI_UPDATE_DFP: return "dfp";
    }
    return "?";
}

static double flops_named(int u, double n, double q) {  // flops.cpp:22-46
    switch (u) {
        case SI_UPDATE_PSB: return 8 * n * n * q + 8 * n * q * q + 2 * q * q * q + n * q + 3 * n * n;
        case SI_UPDATE_AIP: return 6 * n * n * q + 4 * n * q * q + 2 * q * q * q + n * q + n * n;
        case SI_UPDATE_DFP: return 14 * n * n * q + 14 * n * q * q + 4 * q * q * q + 6 * n * n;
    }
    return flops_bfgs(n, q);
}

// validate_update (qn_updates.cpp:79-92): psb needs a symmetric A, bfgs / aip / dfp an SPD one
static void validate_update(int u, si_problem* prob, double* scratch_nn = nullptr) {
    if (u == SI_UPDATE_PSB) {
        if (prob->p->symmetry == SI_GENERAL) throw ConfigError("psb requires a symmetric matrix");
        return;
    }
    validate_spd(prob, scratch_nn);
}

// ---------------------------------------------------------- run_inverter ---
// simi.cpp:217-381 for MethodSpec::named_method(bfgs | psb | aip | dfp).
// SI_TRACE=1: wall time of the driver's phases on stderr (stream synchronised at each mark)
struct PhaseTrace {
    bool on = std::getenv("SI_TRACE") != nullptr;
    cudaStream_t s;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
    explicit PhaseTrace(cudaStream_t st) : s(st) {}
    void mark(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[si trace] %-28s %9.3f ms (total %9.3f ms)\n", what,
                     std::chrono::duration<double, std::milli>(now - last).count(),
                     std::chrono::duration<double, std::milli>(now - t0).count());
        last = now;
    }
    ~PhaseTrace() { mark("release"); }
};

static void run_inverter_impl(si_context* ctx, si_problem* prob, const si_inverter_config* cfg, double* x_out,
                              double* x_inv_out, si_history_point* history, int64_t history_cap,
                              si_run_result* result) {
    auto& c = *ctx->c;
    PhaseTrace trace(c.stream);
    si::Problem& a = *prob->p;
    const int64_t n = a.n, q = cfg->q;
    const int upd = cfg->update;
    std::memset(result, 0, sizeof(*result));
    // validate_config (simi.cpp:185-213)
    require(upd >= SI_UPDATE_BFGS && upd <= SI_UPDATE_DFP, "unknown update name");
    require(q >= 1 && q <= n, "SketchRule: q must satisfy 1 <= q <= n");
    const int sk = cfg->sketch;
    if (sk == SI_SKETCH_ADAPTIVE_COLS || sk == SI_SKETCH_ADAPTIVE_GAUSS || sk == SI_SKETCH_ADAPTIVE_COLS_UNIFORM ||
        sk == SI_SKETCH_ADAPTIVE_GAUSS_DEVICE)
        throw ConfigError("run_inverter: adaptive sketch rules belong to the adarbfgs driver");
    require(sk == SI_SKETCH_GAUSSIAN || sk == SI_SKETCH_GAUSSIAN_DEVICE || sk == SI_SKETCH_COORDINATE_BLOCK,
            "run_inverter: unknown sketch rule");
    require(cfg->tol >= 0.0, "run_inverter: tol must be >= 0");
    require(cfg->max_iters >= 1, "run_inverter: max_iters must be >= 1");
    require(cfg->max_redraws >= 0, "run_inverter: max_redraws must be >= 0");
    require(cfg->residual_every_k >= 1, "run_inverter: residual_every_k must be >= 1");
    if (upd == SI_UPDATE_PSB) validate_update(upd, prob);  // (spd checks below, on the workspace)
    const bool symmetric_iterates = upd != SI_UPDATE_AIP;  // simi.cpp:77-81
    const bool tracks_inverse = upd == SI_UPDATE_DFP;

    // the bfgs workspace stays in the context between calls when X is at most a quarter of
    // device memory: re-running a problem of the same shape allocates and frees nothing
    // (cudaFree / cudaFreeHost of gigabyte buffers measured 3-400 ms)
    size_t mem_free = 0, mem_total = 0;
    ck(cudaMemGetInfo(&mem_free, &mem_total), "meminfo");
    const bool cacheable = upd == SI_UPDATE_BFGS && double(n) * double(n) * 8.0 <= 0.25 * double(mem_total);
    si::RbfgsWork* wp = cacheable ? c.take_rbfgs(n, q) : nullptr;
    if (!wp) {
        wp = new si::RbfgsWork;
        wp->alloc(n, q, true);
        si::family_alloc(*wp, upd);
    }
    si::RbfgsWork& w = *wp;
    w.q = q;
    struct Rel {
        si::Context& c;
        si::RbfgsWork* w;
        bool cacheable;
        double* scratch = nullptr;
        ~Rel() {
            if (scratch) cudaFree(scratch);
            if (cacheable) {
                c.keep_rbfgs(w);
                return;
            }
            si::family_release(*w);
            w->release();
            delete w;
        }
    } rel{c, wp, cacheable};
    trace.mark("alloc");
    // validate_config (simi.cpp:185-213): the Cholesky of A runs in the iterate's buffer,
    // which is initialised right after
    validate_update(upd, prob, w.X);
    if (cfg->x0_host && symmetric_iterates) {
        double nrm = 0.0;
        const double asym = host_frobenius_asym(cfg->x0_host, n, &nrm);
        if (asym > 1e-10 * std::max(1.0, nrm)) throw ConfigError("run_inverter: this method requires a symmetric x0");
    }
    trace.mark("validate (Cholesky)");
    if (cfg->x0_host)
        ck(cudaMemcpyAsync(w.X, cfg->x0_host, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyHostToDevice,
                           c.stream),
           "h2d x0");
    else
        si::set_identity(c, w.X, n);
    if (tracks_inverse) {  // simi.cpp:227-229: x_inv = lu_inverse(x0) or I
        if (cfg->x0_host)
            si::lu_inverse_device(c, w.X, n, w.H);
        else
            si::set_identity(c, w.H, n);
    }
    const double* tracked = tracks_inverse ? w.H : w.X;  // simi.cpp:236-238
    auto residual = [&]() -> double {
        if (upd == SI_UPDATE_AIP && !a.dense) {  // general X with a CSR A
            if (!rel.scratch) ck(cudaMalloc(&rel.scratch, size_t(n) * size_t(n) * sizeof(double)), "malloc");
            si::residual_general_sq_enqueue(c, a, w.X, rel.scratch, c.scalar_dev);
            ck(cudaMemcpyAsync(c.scalar_host, c.scalar_dev, sizeof(double), cudaMemcpyDeviceToHost, c.stream), "d2h");
            ck(cudaStreamSynchronize(c.stream), "sync");
            return std::sqrt(c.scalar_host[0]);
        }
        return residual_norm(c, a, tracked);
    };
    // k = 1 from the default X0 = I: X1 = I + [Z R]·[W' Z]ᵀ (the BFGS rank-2q form still in
    // the workspace), so the checkpoint needs 4n²·2q flops instead of the 2n³ product
    const bool lowrank_first = !cfg->x0_host && upd == SI_UPDATE_BFGS && a.dense;
    auto first_residual = [&]() -> double {
        if (!w.lowrank) ck(cudaMalloc(&w.lowrank, size_t(n) * size_t(2 * q) * sizeof(double)), "malloc");
        // X1 = I + [Z R]·[W' Z]ᵀ (rbfgs_enqueue_iteration's buffers: U = [S | W' | Z | R])
        const int64_t nq = n * w.q;
        si::lowrank_residual_sq_enqueue(c, a, 2 * w.q, w.U + 2 * nq, n, w.U + nq, n, 1.0, w.lowrank, c.scalar_dev);
        ck(cudaMemcpyAsync(c.scalar_host, c.scalar_dev, sizeof(double), cudaMemcpyDeviceToHost, c.stream), "d2h");
        ck(cudaStreamSynchronize(c.stream), "sync");
        return std::sqrt(c.scalar_host[0]);
    };

    HistoryWriter hist{history, history_cap, 0, cfg};
    double flops = 0.0, seconds = 0.0;
    int64_t k = 0;
    bool x_early = false;  // X download issued before the last checkpoint (overlaps its 2n³ residual)
    auto finish = [&](int term, const std::string& msg) {
        result->termination = term;
        result->k = k;
        result->flops = flops;
        result->seconds = seconds;
        result->history_count = hist.count;
        result->max_symmetry_drift = 0.0;  // symmetric updates write X (and H) exactly symmetric (mirrored tiles)
        set_message(result, msg);
        if (x_early) {  // the final X is already on its way on the side stream
            c.join();
        } else if (x_out) {
            ck(cudaMemcpyAsync(x_out, w.X, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, c.stream),
               "d2h x");
        }
        if (x_inv_out && tracks_inverse)
            ck(cudaMemcpyAsync(x_inv_out, w.H, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyDeviceToHost,
                               c.stream),
               "d2h x_inv");
        ck(cudaStreamSynchronize(c.stream), "sync");
        trace.mark("finish (x download)");
    };

    // simi.cpp:242-246; for the default X0 = I (and H0 = I), ‖I − A·I‖ = ‖I − A‖ needs no GEMM
    double base;
    if (cfg->x0_host) {
        base = residual();
    } else {
        si::identity_residual_sq_enqueue(c, a, c.scalar_dev);
        ck(cudaMemcpyAsync(c.scalar_host, c.scalar_dev, sizeof(double), cudaMemcpyDeviceToHost, c.stream), "d2h");
        ck(cudaStreamSynchronize(c.stream), "sync");
        base = std::sqrt(c.scalar_host[0]);
    }
    trace.mark("x0 + base residual");
    if (base == 0.0) {
        hist.record(0, 0.0, 0.0, 0.0);
        finish(SI_TOL_REACHED, "");
        return;
    }
    hist.record(0, 1.0, 0.0, 0.0);

    // coordinate-block rule (sketching.cpp:20-28) with uniform or convenient p (simi.cpp:121-150)
    std::vector<std::vector<si::Index>> blocks;
    std::vector<double> p;
    if (sk == SI_SKETCH_COORDINATE_BLOCK) {
        blocks = si::contiguous_partition(n, q);
        p.assign(blocks.size(), 1.0 / double(blocks.size()));
        if (cfg->probabilities == SI_PROB_CONVENIENT) {
            std::vector<double> wts;
            if (upd == SI_UPDATE_DFP)
                si::spd_inverse_diagonal(c, a, wts);  // Tr(SᵢᵀA⁻¹Sᵢ)
            else
                si::column_weights(c, a, upd == SI_UPDATE_PSB ? 1 : 0, wts);  // ‖ASᵢ‖² or Tr(SᵢᵀASᵢ)
            double sum = 0.0;
            for (size_t i = 0; i < blocks.size(); ++i) {
                double t = 0.0;
                for (auto j : blocks[i]) t += wts[size_t(j)];
                if (!(t > 0.0))
                    throw ConfigError(upd == SI_UPDATE_PSB
                                          ? "convenient_probabilities: family member with zero sketched norm"
                                          : "trace probabilities: member with non-positive sketched trace");
                p[i] = t;
                sum += t;
            }
            for (double& v : p) v /= sum;
        }
    }

    si::RngStream rng(cfg->seed);  // simi.cpp:275
    const bool device_sketch = sk == SI_SKETCH_GAUSSIAN_DEVICE;
    DeviceTimer tm;
    int st[8];
    // simi.cpp:361-375: the residual checkpoint after iteration k
    auto checkpoint = [&]() -> bool {
        trace.mark("iterations");
        const double rel_res = (k == 1 && lowrank_first ? first_residual() : residual()) / base;
        trace.mark(k == 1 && lowrank_first ? "checkpoint (rank-2q)" : "checkpoint");
        hist.record(k, rel_res, flops, seconds);
        if (rel_res <= cfg->tol) {
            finish(SI_TOL_REACHED, "");
            return true;
        }
        if (cfg->time_budget_seconds > 0.0 && seconds > cfg->time_budget_seconds) {
            finish(SI_MAX_ITERS, "time budget exhausted");
            return true;
        }
        return false;
    };
    // Device sketches (bfgs): the iterations between two checkpoints are enqueued back to
    // back — one captured CUDA graph per iteration, no host round trip — and the device
    // keeps the accounting (advance_batch_kernel): a rejected draw or a non-finite iterate
    // stops the batch at the exact iteration, so k, the redraw count and limit, the draws
    // and the iterates are those of the eager loop below.  SI_RUN_EAGER=1 forces the latter.
    if (device_sketch && upd == SI_UPDATE_BFGS && std::getenv("SI_RUN_EAGER") == nullptr) {
        w.batch = true;
        struct Graph {
            cudaGraphExec_t exec = nullptr;
            PhaseTrace* tr = nullptr;
            ~Graph() {
                if (exec) cudaGraphExecDestroy(exec);
                if (tr) tr->mark("graph destroy");
            }
        } g;
        g.tr = &trace;
        const bool graphs = !c.profiling && std::getenv("SI_NO_GRAPH") == nullptr;
        bool warmed = false;
        int64_t graph_launches = 0;
        int consecutive = 0;  // failed attempts of iteration k + 1
        const int64_t every = cfg->residual_every_k, kmax = cfg->max_iters;
        k = 0;
        while (k < kmax) {
            const int64_t kc = k == 0 ? 1 : std::min(((k + every) / every) * every, kmax);  // next checkpoint
            ck(cudaMemsetAsync(w.status, 0, 8 * sizeof(int), c.stream), "reset");
            ck(cudaEventRecord(tm.a, c.stream), "event");
            for (int64_t b = k; b < kc; ++b) {
                if (!graphs || !warmed) {  // the first iteration runs eagerly: sizes workspaces, sets attributes
                    si::family_enqueue_iteration(c, a, w, true, cfg->seed);
                    warmed = true;
                    continue;
                }
                if (!g.exec) {
                    const int64_t l0 = c.launches;
                    cudaGraph_t gr = nullptr;
                    ck(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal), "capture");
                    si::family_enqueue_iteration(c, a, w, true, cfg->seed);
                    ck(cudaStreamEndCapture(c.stream, &gr), "end capture");
                    ck(cudaGraphInstantiate(&g.exec, gr, 0), "instantiate");
                    cudaGraphDestroy(gr);
                    graph_launches = c.launches - l0;
                    c.launches = l0;
                }
                ck(cudaGraphLaunch(g.exec, c.stream), "graph launch");
                c.launches += graph_launches;
            }
            ck(cudaEventRecord(tm.b, c.stream), "event");
            ck(cudaMemcpyAsync(st, w.status, 8 * sizeof(int), cudaMemcpyDeviceToHost, c.stream), "status d2h");
            ck(cudaStreamSynchronize(c.stream), "sync");
            const int64_t accepted = st[3];
            k += accepted;
            result->redraws += st[2];
            if (cfg->track_wall_time) seconds += tm.seconds();
            if (cfg->track_flops) flops += double(accepted) * flops_named(upd, double(n), double(w.q));
            if (st[1]) {  // simi.cpp:342-347
                finish(SI_TERMINATION_ERROR, "diverged: non-finite entries at iteration " + std::to_string(k));
                return;
            }
            if (st[4]) {  // a rejected draw of iteration k + 1 stopped the batch (simi.cpp:331-333)
                consecutive = (accepted > 0 ? 0 : consecutive) + 1;
                if (consecutive > cfg->max_redraws) {
                    k += 1;
                    finish(SI_TERMINATION_ERROR, "sketch rejection limit exceeded for " + describe(sk, q) +
                                                     " at iteration " + std::to_string(k));
                    return;
                }
                continue;
            }
            consecutive = 0;
            if (k == kmax && x_out) {  // X is final: download it on the side stream under the last residual
                c.fork();
                ck(cudaMemcpyAsync(x_out, w.X, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyDeviceToHost,
                                   c.side),
                   "d2h x");
                x_early = true;
            }
            if (checkpoint()) return;
        }
        k = kmax;
        finish(SI_MAX_ITERS, "");
        return;
    }
    for (k = 1; k <= cfg->max_iters; ++k) {
        bool stepped = false;
        for (int failures = 0; !stepped; ++failures) {
            if (failures > cfg->max_redraws) {
                finish(SI_TERMINATION_ERROR, "sketch rejection limit exceeded for " + describe(sk, q) +
                                                 " at iteration " + std::to_string(k));
                return;
            }
            if (sk == SI_SKETCH_GAUSSIAN) {
                rng.gaussian_fill(w.pinned(), n, q, n);  // rng.hpp:42-49
            } else if (sk == SI_SKETCH_COORDINATE_BLOCK) {
                const si::Index i = rng.categorical(p.data(), si::Index(p.size()));
                ctx->log_draw(i);
                const auto& blk = blocks[size_t(i)];
                // the last block of contiguous_partition may be narrower: this draw has q' = |C_i| columns
                w.q = int64_t(blk.size());
                double* sp = w.pinned();
                std::fill(sp, sp + n * w.q, 0.0);
                for (size_t j = 0; j < blk.size(); ++j) sp[blk[j] + int64_t(j) * n] = 1.0;
            }
            if (!device_sketch) si::rbfgs_enqueue_sketch_upload(c, w);
            ck(cudaEventRecord(tm.a, c.stream), "event");  // timer starts after the draw (simi.cpp:298)
            si::family_enqueue_iteration(c, a, w, device_sketch, cfg->seed);
            ck(cudaEventRecord(tm.b, c.stream), "event");
            read_status(c, w.status, st);
            if (st[0] || st[2]) {  // GramRankDeficientError -> redraw (simi.cpp:331-333)
                st[0] = st[2] = 0;
                ck(cudaMemsetAsync(w.status, 0, 4 * sizeof(int), c.stream), "reset");
                result->redraws++;
                continue;
            }
            if (cfg->track_wall_time) seconds += tm.seconds();
            if (cfg->track_flops) flops += flops_named(upd, double(n), double(w.q));  // s.cols()
            stepped = true;
        }
        if (st[1]) {  // simi.cpp:342-347
            finish(SI_TERMINATION_ERROR, "diverged: non-finite entries at iteration " + std::to_string(k));
            return;
        }
        if (k == 1 || k == cfg->max_iters || k % cfg->residual_every_k == 0) {  // simi.cpp:361-375
            if (checkpoint()) return;
        }
    }
    k = cfg->max_iters;
    finish(SI_MAX_ITERS, "");
}

int si_run_inverter(si_context* ctx, si_problem* prob, const si_inverter_config* cfg, double* x_out,
                    si_history_point* history, int64_t history_cap, si_run_result* result) {
    return guard([&] {
        if (ctx->group)  // multi-GPU context: the sharded iteration (shard.cpp)
            si::shard_run_inverter(ctx, prob, cfg, x_out, history, history_cap, result);
        else
            run_inverter_impl(ctx, prob, cfg, x_out, nullptr, history, history_cap, result);
    });
}

int si_run_inverter_pair(si_context* ctx, si_problem* prob, const si_inverter_config* cfg, double* x_out,
                         double* x_inv_out, si_history_point* history, int64_t history_cap, si_run_result* result) {
    return guard([&] {
        if (ctx->group)  // multi-GPU context: the sharded driver (bfgs; other updates are rejected there)
            si::shard_run_inverter(ctx, prob, cfg, x_out, history, history_cap, result);
        else
            run_inverter_impl(ctx, prob, cfg, x_out, x_inv_out, history, history_cap, result);
    });
}

// ---------------------------------------------------------- run_baseline ---
// spectral_norm_estimate (linalg.cpp:106-129) with the start vector drawn here
// (host RngStream, the oracle's bytes); products on the device.
static double spectral_norm_estimate(si::Context& c, si::Problem& a, int iters, uint64_t seed) {
    const int64_t n = a.n;
    require(iters >= 1, "spectral_norm_estimate: iters must be >= 1");
    if (!a.dense && a.symmetry == SI_GENERAL)
        throw ConfigError("spectral_norm_estimate: a general CSR A is not supported (needs Aᵀ)");
    if (si::sumsq_device(c, a.dense ? a.a : a.val, a.dense ? n * n : a.nnz) == 0.0) return 0.0;
    si::RngStream rng(seed);
    std::vector<double> v(static_cast<size_t>(n)), wv(static_cast<size_t>(n));
    auto nrm = [](const std::vector<double>& x) {
        double t = 0.0;
        for (double e : x) t += e * e;
        return std::sqrt(t);
    };
    double *dv = nullptr, *dw = nullptr;
    ck(cudaMalloc(&dv, size_t(n) * sizeof(double)), "malloc");
    ck(cudaMalloc(&dw, size_t(n) * sizeof(double)), "malloc");
    struct Free {
        double *p1, *p2;
        ~Free() {
            cudaFree(p1);
            cudaFree(p2);
        }
    } fr{dv, dw};
    rng.gaussian_fill(v.data(), n, 1, n);
    if (nrm(v) == 0.0) std::fill(v.begin(), v.end(), 1.0);
    double s0 = nrm(v);
    for (double& e : v) e /= s0;
    double est = 0.0;
    for (int it = 0; it < iters; ++it) {
        ck(cudaMemcpyAsync(dv, v.data(), size_t(n) * sizeof(double), cudaMemcpyHostToDevice, c.stream), "h2d");
        si::apply_a(c, a, dv, n, 1, dw, n, nullptr);  // w = A·v
        ck(cudaMemcpyAsync(wv.data(), dw, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "d2h");
        ck(cudaStreamSynchronize(c.stream), "sync");
        est = nrm(wv);
        if (est == 0.0) {  // v in the null space: restart from a fresh direction
            rng.gaussian_fill(v.data(), n, 1, n);
            s0 = nrm(v);
            for (double& e : v) e /= s0;
            continue;
        }
        if (a.dense && a.symmetry == SI_GENERAL)
            si::gemm(c, n, 1, n, a.a, n, true, dw, n, true, dv, n, 1.0, 0.0);  // v = Aᵀ·w
        else
            si::apply_a(c, a, dw, n, 1, dv, n, nullptr);  // symmetric A: Aᵀ·w = A·w
        ck(cudaMemcpyAsync(v.data(), dv, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "d2h");
        ck(cudaStreamSynchronize(c.stream), "sync");
        const double nv = nrm(v);
        if (nv == 0.0) break;
        for (double& e : v) e /= nv;
    }
    return est;
}

int si_run_baseline(si_context* ctx, si_problem* prob, int method, const si_inverter_config* cfg, double* x_out,
                    si_history_point* history, int64_t history_cap, si_run_result* result) {
    return guard([&] {
        auto& c = *ctx->c;
        si::Problem& a = *prob->p;
        const int64_t n = a.n;
        std::memset(result, 0, sizeof(*result));
        require(method == SI_BASELINE_NEWTON_SCHULZ || method == SI_BASELINE_MINIMAL_RESIDUAL,
                "run_baseline: unknown method");
        require(cfg->tol >= 0.0, "run_baseline: tol must be >= 0");
        require(cfg->max_iters >= 1, "run_baseline: max_iters must be >= 1");
        require(cfg->residual_every_k >= 1, "run_baseline: residual_every_k must be >= 1");
        const bool ns = method == SI_BASELINE_NEWTON_SCHULZ;
        si::BaselineWork w;
        struct Rel {
            si::BaselineWork& w;
            ~Rel() { w.release(); }
        } rel{w};
        w.alloc(n);
        if (cfg->x0_host)
            ck(cudaMemcpyAsync(w.X, cfg->x0_host, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyHostToDevice,
                               c.stream),
               "h2d x0");
        else if (ns)
            si::newton_schulz_init_device(c, a, w, spectral_norm_estimate(c, a, 100, cfg->seed));
        else
            si::mr_init_device(c, a, w);

        HistoryWriter hist{history, history_cap, 0, cfg};
        double flops = 0.0, seconds = 0.0;
        int64_t k = 0;
        auto finish = [&](int term, const std::string& msg) {
            result->termination = term;
            result->k = k;
            result->flops = flops;
            result->seconds = seconds;
            result->history_count = hist.count;
            set_message(result, msg);
            if (x_out)
                ck(cudaMemcpyAsync(x_out, w.X, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyDeviceToHost,
                                   c.stream),
                   "d2h x");
            ck(cudaStreamSynchronize(c.stream), "sync");
        };
        const double base = si::baseline_residual(c, a, w);  // R = I − A X0 (baselines.cpp:70-71)
        if (base == 0.0) {
            hist.record(0, 0.0, 0.0, 0.0);
            finish(SI_TOL_REACHED, "");
            return;
        }
        hist.record(0, 1.0, 0.0, 0.0);
        const double fl = ns ? 4.0 * double(n) * n * n + 2.0 * double(n) * n   // flops.cpp:76-79
                             : 4.0 * double(n) * n * n + 8.0 * double(n) * n;  // flops.cpp:81-85
        for (k = 1; k <= cfg->max_iters; ++k) {
            const auto t0 = std::chrono::steady_clock::now();
            bool finite = true, stagnated = false;
            if (ns) {
                finite = si::newton_schulz_enqueue(c, a, w);
            } else {
                double alpha = 0.0;
                const int r = si::mr_enqueue(c, a, w, &alpha);
                stagnated = r == 1;
                finite = r != 2;
            }
            const auto t1 = std::chrono::steady_clock::now();
            if (cfg->track_wall_time) seconds += std::chrono::duration<double>(t1 - t0).count();
            if (cfg->track_flops) flops += fl;
            if (!finite) {
                finish(SI_TERMINATION_ERROR, "diverged: non-finite entries at iteration " + std::to_string(k));
                return;
            }
            if (stagnated) {  // baselines.cpp:110-119: ‖R‖ of the carried residual
                const double rel_res = std::sqrt(si::sumsq_device(c, w.R, n * n)) / base;
                hist.record(k, rel_res, flops, seconds);
                if (rel_res <= cfg->tol) {
                    finish(SI_TOL_REACHED, "");
                } else {
                    finish(SI_TERMINATION_ERROR,
                           "minimal residual stagnated (zero step denominator) at iteration " + std::to_string(k));
                }
                return;
            }
            if (k == 1 || k == cfg->max_iters || k % cfg->residual_every_k == 0) {  // baselines.cpp:121-146
                const double rel_res = si::baseline_residual(c, a, w) / base;     // replaces the carried R
                hist.record(k, rel_res, flops, seconds);
                if (!std::isfinite(rel_res)) {
                    finish(SI_TERMINATION_ERROR, "diverged: residual overflow at iteration " + std::to_string(k));
                    return;
                }
                if (rel_res <= cfg->tol) {
                    finish(SI_TOL_REACHED, "");
                    return;
                }
                if (cfg->time_budget_seconds > 0.0 && seconds > cfg->time_budget_seconds) {
                    finish(SI_MAX_ITERS, "time budget exhausted");
                    return;
                }
            }
        }
        k = cfg->max_iters;
        finish(SI_MAX_ITERS, "");
    });
}

// ------------------------------------------------ step-level (f3 / f4) -----
static void upload_general(si::Problem& a, si_context* ctx, int64_t n, const double* a_host) {
    a.ctx = ctx->c.get();
    a.n = n;
    a.symmetry = SI_GENERAL;  // the step kernels take A as given
    si::problem_upload_dense(a, a_host, false);
}

static void named_step_impl(si_context* ctx, int update, int64_t n, int64_t q, const double* x_host,
                            const double* x_inv_host, const double* a_host, const double* s_host, double* x_out,
                            double* x_inv_out) {
    auto& c = *ctx->c;
    require(q >= 1 && n >= 1, "named step: bad shape");
    si::Problem a;
    upload_general(a, ctx, n, a_host);
    si::RbfgsWork w;
    struct Rel {
        si::RbfgsWork& w;
        ~Rel() {
            si::family_release(w);
            w.release();
        }
    } rel{w};
    w.alloc(n, q, true);
    si::family_alloc(w, update);
    const size_t nn = size_t(n) * size_t(n) * sizeof(double);
    ck(cudaMemcpyAsync(w.X, x_host, nn, cudaMemcpyHostToDevice, c.stream), "h2d");
    if (update == SI_UPDATE_DFP) ck(cudaMemcpyAsync(w.H, x_inv_host, nn, cudaMemcpyHostToDevice, c.stream), "h2d");
    std::memcpy(w.pinned(), s_host, size_t(n) * size_t(q) * sizeof(double));
    si::rbfgs_enqueue_sketch_upload(c, w);
    si::family_enqueue_iteration(c, a, w, false, 0);
    int st[4];
    read_status(c, w.status, st);
    if (st[0])
        throw ResampleError(std::string(update_name(update)) + "_step: sketched Gram matrix is not positive definite");
    ck(cudaMemcpyAsync(x_out, w.X, nn, cudaMemcpyDeviceToHost, c.stream), "d2h");
    if (update == SI_UPDATE_DFP) ck(cudaMemcpyAsync(x_inv_out, w.H, nn, cudaMemcpyDeviceToHost, c.stream), "d2h");
    ck(cudaStreamSynchronize(c.stream), "sync");
}

int si_psb_step(si_context* ctx, int64_t n, int64_t q, const double* x, const double* a, const double* s, double* o) {
    return guard([&] { named_step_impl(ctx, SI_UPDATE_PSB, n, q, x, nullptr, a, s, o, nullptr); });
}
int si_aip_step(si_context* ctx, int64_t n, int64_t q, const double* x, const double* a, const double* s, double* o) {
    return guard([&] { named_step_impl(ctx, SI_UPDATE_AIP, n, q, x, nullptr, a, s, o, nullptr); });
}
int si_dfp_step(si_context* ctx, int64_t n, int64_t q, const double* x, const double* xi, const double* a,
                const double* s, double* o, double* oi) {
    return guard([&] { named_step_impl(ctx, SI_UPDATE_DFP, n, q, x, xi, a, s, o, oi); });
}

int si_newton_schulz_step(si_context* ctx, int64_t n, const double* x_host, const double* a_host, double* x_out) {
    return guard([&] {
        auto& c = *ctx->c;
        si::Problem a;
        upload_general(a, ctx, n, a_host);
        si::BaselineWork w;
        struct Rel {
            si::BaselineWork& w;
            ~Rel() { w.release(); }
        } rel{w};
        w.alloc(n);
        ck(cudaMemcpyAsync(w.X, x_host, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyHostToDevice, c.stream),
           "h2d");
        si::newton_schulz_enqueue(c, a, w);
        ck(cudaMemcpyAsync(x_out, w.X, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, c.stream),
           "d2h");
        ck(cudaStreamSynchronize(c.stream), "sync");
    });
}

int si_spectral_norm_estimate(si_context* ctx, si_problem* prob, int iters, uint64_t seed, double* out) {
    return guard([&] { *out = spectral_norm_estimate(*ctx->c, *prob->p, iters, seed); });
}

int si_newton_schulz_init(si_context* ctx, si_problem* prob, uint64_t seed, double* x_out) {
    return guard([&] {
        auto& c = *ctx->c;
        const int64_t n = prob->p->n;
        si::BaselineWork w;
        struct Rel {
            si::BaselineWork& w;
            ~Rel() { w.release(); }
        } rel{w};
        w.alloc(n);
        si::newton_schulz_init_device(c, *prob->p, w, spectral_norm_estimate(c, *prob->p, 100, seed));
        ck(cudaMemcpyAsync(x_out, w.X, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, c.stream),
           "d2h");
        ck(cudaStreamSynchronize(c.stream), "sync");
    });
}

int si_mr_init(si_context* ctx, si_problem* prob, double* x_out) {
    return guard([&] {
        auto& c = *ctx->c;
        const int64_t n = prob->p->n;
        si::BaselineWork w;
        struct Rel {
            si::BaselineWork& w;
            ~Rel() { w.release(); }
        } rel{w};
        w.alloc(n);
        si::mr_init_device(c, *prob->p, w);
        ck(cudaMemcpyAsync(x_out, w.X, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, c.stream),
           "d2h");
        ck(cudaStreamSynchronize(c.stream), "sync");
    });
}

int si_mr_step_cached(si_context* ctx, int64_t n, const double* x_host, const double* r_host, const double* a_host,
                      double* x_out, double* r_out, double* alpha, int* stagnated) {
    return guard([&] {
        auto& c = *ctx->c;
        si::Problem a;
        upload_general(a, ctx, n, a_host);
        si::BaselineWork w;
        struct Rel {
            si::BaselineWork& w;
            ~Rel() { w.release(); }
        } rel{w};
        w.alloc(n);
        const size_t nn = size_t(n) * size_t(n) * sizeof(double);
        ck(cudaMemcpyAsync(w.X, x_host, nn, cudaMemcpyHostToDevice, c.stream), "h2d");
        ck(cudaMemcpyAsync(w.R, r_host, nn, cudaMemcpyHostToDevice, c.stream), "h2d");
        const int r = si::mr_enqueue(c, a, w, alpha);
        *stagnated = r == 1 ? 1 : 0;
        ck(cudaMemcpyAsync(x_out, w.X, nn, cudaMemcpyDeviceToHost, c.stream), "d2h");
        ck(cudaMemcpyAsync(r_out, w.R, nn, cudaMemcpyDeviceToHost, c.stream), "d2h");
        ck(cudaStreamSynchronize(c.stream), "sync");
    });
}

// ---------------------------------------------------------- run_adarbfgs ---
// adarbfgs.cpp:91-200.
int si_run_adarbfgs(si_context* ctx, si_problem* prob, const si_inverter_config* cfg, double* l_out,
                    double* x_out, si_history_point* history, int64_t history_cap, si_run_result* result) {
    return guard([&] {
        if (ctx->group) {  // multi-GPU context: L row-sharded (shard.cpp)
            si::shard_run_adarbfgs(ctx, prob, cfg, l_out, x_out, history, history_cap, result);
            return;
        }
        auto& c = *ctx->c;
        si::Problem& a = *prob->p;
        const int64_t n = a.n, q = cfg->q;
        std::memset(result, 0, sizeof(*result));
        require(q >= 1 && q <= n, "SketchRule: q must satisfy 1 <= q <= n");
        const int sk = cfg->sketch;
        if (!(sk == SI_SKETCH_ADAPTIVE_COLS || sk == SI_SKETCH_ADAPTIVE_GAUSS || sk == SI_SKETCH_ADAPTIVE_COLS_UNIFORM ||
              sk == SI_SKETCH_ADAPTIVE_GAUSS_DEVICE))
            throw ConfigError("run_adarbfgs: rule must be adaptive");
        require(cfg->tol >= 0.0, "run_adarbfgs: tol must be >= 0");
        require(cfg->max_iters >= 1, "run_adarbfgs: max_iters must be >= 1");
        if (prob->p->symmetry != SI_SPD)
            throw std::invalid_argument("ProblemMatrix: operation requires an spd-flagged matrix");
        const bool cols = sk == SI_SKETCH_ADAPTIVE_COLS;
        const bool gauss = sk == SI_SKETCH_ADAPTIVE_GAUSS || sk == SI_SKETCH_ADAPTIVE_GAUSS_DEVICE;

        // the workspace stays in the context between calls when L is at most a quarter of
        // device memory (as run_inverter's)
        size_t mem_free = 0, mem_total = 0;
        ck(cudaMemGetInfo(&mem_free, &mem_total), "meminfo");
        const bool cacheable = double(n) * double(n) * 8.0 <= 0.25 * double(mem_total);
        si::AdaWork* wp = cacheable ? c.take_ada(n, q, gauss) : nullptr;
        if (!wp) {
            wp = new si::AdaWork;
            wp->alloc(n, q, gauss);
        }
        si::AdaWork& w = *wp;
        w.q = q;
        struct Rel {
            si::Context& c;
            si::AdaWork* w;
            bool cacheable, gauss;
            ~Rel() {
                if (cacheable) {
                    c.keep_ada(w, gauss);
                    return;
                }
                w->release();
                delete w;
            }
        } rel{c, wp, cacheable, gauss};
        validate_spd(prob, w.L);  // adarbfgs.cpp:97; the Cholesky runs in L's buffer, initialised next
        if (cfg->x0_host)
            ck(cudaMemcpyAsync(w.L, cfg->x0_host, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyHostToDevice,
                               c.stream),
               "h2d l0");
        else
            si::set_identity(c, w.L, n);
        if (const char* e = std::getenv("SI_PDIAG_REFRESH")) w.pdiag_refresh = std::max(1, std::atoi(e));
        if (cols && !cfg->x0_host) si::ada_init_pdiag_identity(c, a, w);  // diag(I·A·I) = diag(A)

        HistoryWriter hist{history, history_cap, 0, cfg};
        double flops = 0.0, seconds = 0.0;
        int64_t k = 0;
        auto finish = [&](int term, const std::string& msg) {
            result->termination = term;
            result->k = k;
            result->flops = flops;
            result->seconds = seconds;
            result->history_count = hist.count;
            set_message(result, msg);
            if (l_out)
                ck(cudaMemcpyAsync(l_out, w.L, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyDeviceToHost,
                                   c.stream),
                   "d2h l");
            if (x_out) {  // state.x = L Lᵀ (adarbfgs.cpp:89,122)
                double* X = nullptr;
                ck(cudaMalloc(&X, size_t(n) * size_t(n) * sizeof(double)), "malloc");
                si::gemm(c, n, n, n, w.L, n, false, w.L, n, false, X, n, 1.0, 0.0);
                ck(cudaMemcpyAsync(x_out, X, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, c.stream),
                   "d2h x");
                ck(cudaStreamSynchronize(c.stream), "sync");
                cudaFree(X);
            }
            ck(cudaStreamSynchronize(c.stream), "sync");
        };

        // adarbfgs.cpp:112-115,126; for the default L0 = I the base is ‖I − A‖ (no GEMM)
        double base;
        if (cfg->x0_host) {
            base = factored_residual_norm(c, a, w);
        } else {
            si::identity_residual_sq_enqueue(c, a, c.scalar_dev);
            ck(cudaMemcpyAsync(c.scalar_host, c.scalar_dev, sizeof(double), cudaMemcpyDeviceToHost, c.stream), "d2h");
            ck(cudaStreamSynchronize(c.stream), "sync");
            base = std::sqrt(c.scalar_host[0]);
        }
        if (base == 0.0) {
            hist.record(0, 0.0, 0.0, 0.0);
            finish(SI_TOL_REACHED, "");
            return;
        }
        hist.record(0, 1.0, 0.0, 0.0);

        const auto blocks = cols ? si::contiguous_partition(n, q) : std::vector<std::vector<si::Index>>{};
        si::RngStream rng(cfg->seed);
        std::vector<double> p;
        int st[8];
        // adarbfgs.cpp:179-194: the factored residual checkpoint after iteration k
        auto checkpoint = [&]() -> bool {
            const double rel = factored_residual_norm(c, a, w) / base;
            hist.record(k, rel, flops, seconds);
            if (rel <= cfg->tol) {
                finish(SI_TOL_REACHED, "");
                return true;
            }
            if (cfg->time_budget_seconds > 0.0 && seconds > cfg->time_budget_seconds) {
                finish(SI_MAX_ITERS, "time budget exhausted");
                return true;
            }
            return false;
        };
        // Samplers whose draws do not depend on the iterate (q uniform coordinates; device
        // Gaussian S̃): up to 64 attempts between two checkpoints are drawn on the host, their
        // index sets uploaded once, and enqueued back to back; ada_advance_batch_kernel stops
        // the batch at a rejected square root or a non-finite factor, and the host rewinds the
        // RngStream to just after the rejected draw — the same attempts, draws, k and
        // iterates as the per-iteration loop (SI_RUN_EAGER=1), without a round trip per
        // iteration.  The reference's Eq. 8.2 sampler needs the device probabilities before
        // every draw and stays per-iteration.
        if ((sk == SI_SKETCH_ADAPTIVE_COLS_UNIFORM || sk == SI_SKETCH_ADAPTIVE_GAUSS_DEVICE) &&
            std::getenv("SI_RUN_EAGER") == nullptr) {
            const int mode = sk == SI_SKETCH_ADAPTIVE_COLS_UNIFORM ? 0 : 2;
            constexpr int64_t CAP = 64;
            w.batch = true;
            if (mode == 0) w.ensure_ring(int(CAP));
            int64_t* const idx0 = w.idx_dev;
            std::vector<si::RngStream> snaps;
            int consecutive = 0;
            const int64_t every = cfg->residual_every_k, kmax = cfg->max_iters;
            k = 0;
            while (k < kmax) {
                const int64_t kc = k == 0 ? 1 : std::min(((k + every) / every) * every, kmax);  // next checkpoint
                const int64_t nb = std::min(kc - k, CAP);
                const auto t0 = std::chrono::steady_clock::now();
                if (mode == 0) {
                    snaps.clear();
                    for (int64_t b = 0; b < nb; ++b) {
                        snaps.push_back(rng);  // the stream before draw b
                        const auto idx = si::uniform_subset(rng, n, q);
                        for (int64_t j = 0; j < q; ++j) w.idx_ring_pinned[b * q + j] = idx[size_t(j)];
                    }
                    snaps.push_back(rng);
                    ck(cudaMemcpyAsync(w.idx_ring, w.idx_ring_pinned, size_t(nb) * size_t(q) * sizeof(int64_t),
                                       cudaMemcpyHostToDevice, c.stream),
                       "h2d idx");
                }
                ck(cudaMemsetAsync(w.status, 0, 8 * sizeof(int), c.stream), "reset");
                for (int64_t b = 0; b < nb; ++b) {
                    if (mode == 0) {
                        w.idx_dev = w.idx_ring + b * q;
                        w.idx_next = b + 1 < nb ? w.idx_ring + (b + 1) * q : nullptr;  // S pipelined ahead
                    }
                    si::ada_enqueue_update(c, a, w, mode, cfg->seed);
                }
                w.idx_dev = idx0;
                w.idx_next = nullptr;
                ck(cudaMemcpyAsync(st, w.status, 8 * sizeof(int), cudaMemcpyDeviceToHost, c.stream), "status d2h");
                ck(cudaStreamSynchronize(c.stream), "sync");
                const auto t1 = std::chrono::steady_clock::now();
                const int64_t accepted = st[5];
                if (mode == 0) {  // the attempts that executed: all, or up to the rejected one
                    const int64_t ran = st[4] ? accepted + 1 : nb;
                    for (int64_t b = 0; b < ran * q; ++b) ctx->log_draw(w.idx_ring_pinned[b]);
                }
                k += accepted;
                result->redraws += st[2];
                if (cfg->track_wall_time) seconds += std::chrono::duration<double>(t1 - t0).count();
                if (cfg->track_flops) flops += double(accepted) * flops_adarbfgs(double(n), double(q));
                if (st[1]) {
                    finish(SI_TERMINATION_ERROR, "diverged: non-finite factor at iteration " + std::to_string(k));
                    return;
                }
                if (st[4]) {  // attempt `accepted` of this batch was rejected: redraw from just after it
                    if (mode == 0) rng = snaps[size_t(accepted) + 1];
                    consecutive = (accepted > 0 ? 0 : consecutive) + 1;
                    if (consecutive > cfg->max_redraws) {
                        k += 1;
                        finish(SI_TERMINATION_ERROR, "sketch rejection limit exceeded for " + describe(sk, q) +
                                                         " at iteration " + std::to_string(k));
                        return;
                    }
                    continue;
                }
                consecutive = 0;
                if (k == kc && checkpoint()) return;
            }
            k = kmax;
            finish(SI_MAX_ITERS, "");
            return;
        }
        for (k = 1; k <= cfg->max_iters; ++k) {
            bool stepped = false;
            const auto t0 = std::chrono::steady_clock::now();  // timer includes probabilities + draws (:143)
            if (cols) {
                si::ada_enqueue_probabilities(c, a, w);
                ck(cudaStreamSynchronize(c.stream), "sync");
                block_probabilities(w.p_pinned, blocks, p);
            }
            for (int attempt = 0; attempt <= cfg->max_redraws && !stepped; ++attempt) {
                int mode = 0;
                if (cols) {
                    const si::Index i = rng.categorical(p.data(), si::Index(p.size()));
                    ctx->log_draw(i);
                    const auto& blk = blocks[size_t(i)];
                    w.q = int64_t(blk.size());  // a narrower last block draws q' = |C_i| columns
                    for (size_t j = 0; j < blk.size(); ++j) w.idx_pinned[j] = blk[j];
                } else if (sk == SI_SKETCH_ADAPTIVE_COLS_UNIFORM) {
                    const auto idx = si::uniform_subset(rng, n, q);
                    for (int64_t j = 0; j < q; ++j) {
                        w.idx_pinned[j] = idx[size_t(j)];
                        ctx->log_draw(idx[size_t(j)]);
                    }
                } else if (sk == SI_SKETCH_ADAPTIVE_GAUSS) {
                    rng.gaussian_fill(w.st_pinned, n, q, n);
                    mode = 1;
                } else {
                    mode = 2;
                }
                if (mode == 0)
                    ck(cudaMemcpyAsync(w.idx_dev, w.idx_pinned, size_t(w.q) * sizeof(int64_t), cudaMemcpyHostToDevice,
                                       c.stream),
                       "h2d idx");
                si::ada_enqueue_update(c, a, w, mode, cfg->seed);
                read_status(c, w.status, st);
                if (st[0] || st[2]) {
                    st[0] = st[2] = 0;
                    ck(cudaMemsetAsync(w.status, 0, 4 * sizeof(int), c.stream), "reset");
                    result->redraws++;
                    continue;
                }
                stepped = true;
            }
            const auto t1 = std::chrono::steady_clock::now();
            if (!stepped) {
                finish(SI_TERMINATION_ERROR, "sketch rejection limit exceeded for " + describe(sk, q) +
                                                 " at iteration " + std::to_string(k));
                return;
            }
            if (cfg->track_wall_time) seconds += std::chrono::duration<double>(t1 - t0).count();
            if (cfg->track_flops) {
                flops += flops_adarbfgs(double(n), double(q));  // adarbfgs.cpp:166 uses rule.q
                if (cols) flops += 2.0 * double(n) * double(n) * double(n);  // adarbfgs.cpp:168
            }
            if (st[1]) {
                finish(SI_TERMINATION_ERROR, "diverged: non-finite factor at iteration " + std::to_string(k));
                return;
            }
            if (k == 1 || k == cfg->max_iters || k % cfg->residual_every_k == 0) {
                if (checkpoint()) return;
            }
        }
        k = cfg->max_iters;
        finish(SI_MAX_ITERS, "");
    });
}

// ------------------------------------------------------------- solver -----
int si_solver_create(si_context* ctx, si_problem* prob, int method, int sketch, int64_t q, uint64_t seed,
                     si_solver** out) {
    return guard([&] {
        const int64_t n = prob->p->n;
        require(q >= 1 && q <= n, "SketchRule: q must satisfy 1 <= q <= n");
        require(method == SI_METHOD_RBFGS || method == SI_METHOD_ADARBFGS, "solver: unknown method");
        auto s = std::make_unique<si_solver>();
        s->ctx = ctx;
        s->prob = prob;
        s->method = method;
        s->sketch = sketch;
        s->q = q;
        s->seed = seed;
        s->rng = std::make_unique<si::RngStream>(seed);
        ck(cudaMallocHost(&s->status_host, 4 * sizeof(int)), "pinned");
        if (ctx->group) {  // multi-GPU context: the sharded iteration (shard.cpp)
            s->shard = si::shard_solver_create(ctx, prob, method, sketch, q, seed);
            *out = s.release();
            return;
        }
        if (method == SI_METHOD_RBFGS) {
            require(sketch == SI_SKETCH_GAUSSIAN || sketch == SI_SKETCH_GAUSSIAN_DEVICE,
                    "solver: RBFGS supports gaussian sketches");
            s->rw.alloc(n, q, true);
            si::set_identity(*ctx->c, s->rw.X, n);
        } else {
            require(sketch == SI_SKETCH_ADAPTIVE_COLS_UNIFORM || sketch == SI_SKETCH_ADAPTIVE_GAUSS ||
                        sketch == SI_SKETCH_ADAPTIVE_GAUSS_DEVICE || sketch == SI_SKETCH_ADAPTIVE_COLS,
                    "solver: AdaRBFGS needs an adaptive rule");
            s->aw.alloc(n, q, sketch == SI_SKETCH_ADAPTIVE_GAUSS || sketch == SI_SKETCH_ADAPTIVE_GAUSS_DEVICE);
            si::set_identity(*ctx->c, s->aw.L, n);
        }
        ck(cudaStreamSynchronize(ctx->c->stream), "sync");
        *out = s.release();
    });
}

int si_solver_destroy(si_solver* s) {
    return guard([&] { delete s; });
}

static double* solver_iterate(si_solver* s) { return s->method == SI_METHOD_RBFGS ? s->rw.X : s->aw.L; }

int si_solver_set_identity(si_solver* s) {
    return guard([&] {
        require(!s->shard, "solver: use si_solver_set_iterate on a multi-GPU context");
        si::set_identity(*s->ctx->c, solver_iterate(s), s->prob->p->n);
    });
}

int si_solver_set_iterate(si_solver* s, const double* host) {
    return guard([&] {
        if (s->shard) {
            si::shard_solver_set(s->shard, host);
            return;
        }
        const int64_t n = s->prob->p->n;
        ck(cudaMemcpyAsync(solver_iterate(s), host, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyHostToDevice,
                           s->ctx->c->stream),
           "h2d");
    });
}

int si_solver_get_iterate(si_solver* s, double* host) {
    return guard([&] {
        if (s->shard) {
            si::shard_solver_get(s->shard, host);
            return;
        }
        const int64_t n = s->prob->p->n;
        ck(cudaMemcpyAsync(host, solver_iterate(s), size_t(n) * size_t(n) * sizeof(double), cudaMemcpyDeviceToHost,
                           s->ctx->c->stream),
           "d2h");
        ck(cudaStreamSynchronize(s->ctx->c->stream), "sync");
    });
}

double* si_solver_iterate_device(si_solver* s) { return s->shard ? nullptr : solver_iterate(s); }

int64_t si_solver_redraws(si_solver* s) { return s->shard ? si::shard_solver_redraws(s->shard) : s->redraws; }

static void solver_one(si_solver* s, const double* s_host, const int64_t* idx_host, bool check) {
    auto& c = *s->ctx->c;
    si::Problem& a = *s->prob->p;
    const int64_t n = a.n, q = s->q;
    if (s->method == SI_METHOD_RBFGS) {
        const bool dev = s_host == nullptr && s->sketch == SI_SKETCH_GAUSSIAN_DEVICE;
        if (!dev) {
            if (s_host)
                std::memcpy(s->rw.pinned(), s_host, size_t(n) * size_t(q) * sizeof(double));
            else
                s->rng->gaussian_fill(s->rw.pinned(), n, q, n);
            si::rbfgs_enqueue_sketch_upload(c, s->rw);
        }
        si::rbfgs_enqueue_iteration(c, a, s->rw, dev, s->seed);
    } else {
        int mode = 0;
        if (idx_host) {
            std::memcpy(s->aw.idx_pinned, idx_host, size_t(q) * sizeof(int64_t));
        } else if (s->sketch == SI_SKETCH_ADAPTIVE_COLS_UNIFORM) {
            const auto idx = si::uniform_subset(*s->rng, n, q);
            for (int64_t j = 0; j < q; ++j) s->aw.idx_pinned[j] = idx[size_t(j)];
        } else if (s->sketch == SI_SKETCH_ADAPTIVE_GAUSS) {
            if (s_host)
                std::memcpy(s->aw.st_pinned, s_host, size_t(n) * size_t(q) * sizeof(double));
            else
                s->rng->gaussian_fill(s->aw.st_pinned, n, q, n);
            mode = 1;
        } else if (s->sketch == SI_SKETCH_ADAPTIVE_GAUSS_DEVICE) {
            mode = s_host ? 1 : 2;
            if (s_host) std::memcpy(s->aw.st_pinned, s_host, size_t(n) * size_t(q) * sizeof(double));
        } else {
            throw ConfigError("solver: adaptive_cols needs explicit indices (use si_run_adarbfgs)");
        }
        if (mode == 0)
            ck(cudaMemcpyAsync(s->aw.idx_dev, s->aw.idx_pinned, size_t(q) * sizeof(int64_t), cudaMemcpyHostToDevice,
                               c.stream),
               "h2d idx");
        si::ada_enqueue_update(c, a, s->aw, mode, s->seed);
    }
    if (check) {
        int* status = s->method == SI_METHOD_RBFGS ? s->rw.status : s->aw.status;
        read_status(c, status, s->status_host);
        if (s->status_host[1]) throw NumericalError("diverged: non-finite iterate");
        if (s->status_host[0] || s->status_host[2]) {
            ck(cudaMemsetAsync(status, 0, 4 * sizeof(int), c.stream), "reset");
            s->redraws++;
            throw ResampleError("solver: sketch rejected (resample)");
        }
    }
}

int si_solver_step(si_solver* s, int64_t iters) {
    return guard([&] {
        if (s->shard) {
            si::shard_solver_step(s->shard, iters, *s->rng, 100);
            return;
        }
        auto& c = *s->ctx->c;
        const bool device = s->sketch == SI_SKETCH_GAUSSIAN_DEVICE || s->sketch == SI_SKETCH_ADAPTIVE_GAUSS_DEVICE;
        int* status = s->method == SI_METHOD_RBFGS ? s->rw.status : s->aw.status;
        if (!device && s->method == SI_METHOD_ADARBFGS && s->sketch == SI_SKETCH_ADAPTIVE_COLS_UNIFORM &&
            std::getenv("SI_RUN_EAGER") == nullptr) {
            // the paper sampler's draws do not depend on the iterate: up to 64 index sets are
            // drawn ahead, uploaded once and enqueued back to back (run_adarbfgs's batched loop;
            // a rejected attempt stops the batch on the device and the stream is rewound to it)
            si::AdaWork& w = s->aw;
            const int64_t n = s->prob->p->n, q = s->q;
            constexpr int64_t CAP = 64;
            w.ensure_ring(int(CAP));
            int64_t* const idx0 = w.idx_dev;
            std::vector<si::RngStream> snaps;
            int st[8];
            int consecutive = 0;
            for (int64_t done = 0; done < iters;) {
                const int64_t nb = std::min(iters - done, CAP);
                snaps.clear();
                for (int64_t b = 0; b < nb; ++b) {
                    snaps.push_back(*s->rng);
                    const auto idx = si::uniform_subset(*s->rng, n, q);
                    for (int64_t j = 0; j < q; ++j) w.idx_ring_pinned[b * q + j] = idx[size_t(j)];
                }
                snaps.push_back(*s->rng);
                ck(cudaMemcpyAsync(w.idx_ring, w.idx_ring_pinned, size_t(nb) * size_t(q) * sizeof(int64_t),
                                   cudaMemcpyHostToDevice, c.stream),
                   "h2d idx");
                ck(cudaMemsetAsync(w.status, 0, 8 * sizeof(int), c.stream), "reset");
                w.batch = true;
                for (int64_t b = 0; b < nb; ++b) {
                    w.idx_dev = w.idx_ring + b * q;
                    w.idx_next = b + 1 < nb ? w.idx_ring + (b + 1) * q : nullptr;
                    si::ada_enqueue_update(c, *s->prob->p, w, 0, s->seed);
                }
                w.batch = false;
                w.idx_dev = idx0;
                w.idx_next = nullptr;
                ck(cudaMemcpyAsync(st, w.status, 8 * sizeof(int), cudaMemcpyDeviceToHost, c.stream), "status d2h");
                ck(cudaStreamSynchronize(c.stream), "sync");
                const int64_t accepted = st[5];
                done += accepted;
                s->redraws += st[2];
                if (st[1]) throw NumericalError("diverged: non-finite iterate");
                if (st[4]) {
                    *s->rng = snaps[size_t(accepted) + 1];
                    consecutive = (accepted > 0 ? 0 : consecutive) + 1;
                    if (consecutive > 100) throw NumericalError("solver: rejection limit exceeded");
                } else {
                    consecutive = 0;
                }
            }
            ck(cudaMemsetAsync(w.status, 0, 8 * sizeof(int), c.stream), "reset");
            return;
        }
        if (!device) {
            // host-drawn sketches share one pinned staging buffer: one iteration at a time
            for (int64_t i = 0; i < iters;) {
                for (int attempt = 0;; ++attempt) {
                    try {
                        solver_one(s, nullptr, nullptr, true);
                        break;
                    } catch (const ResampleError&) {
                        if (attempt >= 100) throw NumericalError("solver: rejection limit exceeded");
                    }
                }
                ++i;
            }
            return;
        }
        // device sketches: enqueue back to back with no host round trip.  A rejected
        // Gram makes the rest of its iteration a no-op and is counted on the device
        // (advance_counter_kernel); those iterations are re-run with fresh counters,
        // i.e. redrawn, as simi.cpp:287-340.
        int64_t remaining = iters;
        int64_t total_redraws = 0;
        const char* ng = std::getenv("SI_NO_GRAPH");
        const bool graphs = !(ng && ng[0] == '1') && !c.profiling;
        auto one = [&]() {
            if (!graphs) {
                solver_one(s, nullptr, nullptr, false);
                return;
            }
            if (!s->warmed) {  // first iteration eagerly: sizes workspaces, sets kernel attributes
                solver_one(s, nullptr, nullptr, false);
                s->warmed = true;
                return;
            }
            if (!s->graph) {
                const int64_t l0 = c.launches;
                cudaGraph_t g = nullptr;
                ck(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal), "capture");
                solver_one(s, nullptr, nullptr, false);
                ck(cudaStreamEndCapture(c.stream, &g), "end capture");
                ck(cudaGraphInstantiate(&s->graph, g, 0), "instantiate");
                cudaGraphDestroy(g);
                s->graph_launches = c.launches - l0;
                c.launches = l0;
            }
            ck(cudaGraphLaunch(s->graph, c.stream), "graph launch");
            c.launches += s->graph_launches;
        };
        while (remaining > 0) {
            for (int64_t i = 0; i < remaining; ++i) one();
            read_status(c, status, s->status_host);
            if (s->status_host[1]) throw NumericalError("diverged: non-finite iterate");
            remaining = s->status_host[2] + s->status_host[0];
            if (remaining) {
                ck(cudaMemsetAsync(status, 0, 4 * sizeof(int), c.stream), "reset");
                s->redraws += remaining;
                total_redraws += remaining;
                if (total_redraws > 100 * iters) throw NumericalError("solver: rejection limit exceeded");
            }
        }
    });
}

int si_solver_step_with_sketch(si_solver* s, const double* s_host, const int64_t* idx_host) {
    return guard([&] {
        require(!s->shard, "solver: host sketches on a multi-GPU context go through si_run_inverter");
        solver_one(s, s_host, idx_host, true);
    });
}

int si_solver_residual(si_solver* s, double* out) {
    return guard([&] {
        if (s->shard) {
            *out = si::shard_solver_residual(s->shard);
            return;
        }
        auto& c = *s->ctx->c;
        if (s->method == SI_METHOD_RBFGS)
            *out = residual_norm(c, *s->prob->p, s->rw.X);
        else
            *out = factored_residual_norm(c, *s->prob->p, s->aw);
    });
}

// ------------------------------------------------------- device pointers --
int si_gemm_device(si_context* ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int a_kmajor,
                   const double* B, int64_t ldb, int b_kmajor, double* C, int64_t ldc, double alpha, double beta) {
    return guard([&] {
        require(M >= 0 && N >= 0 && K >= 0, "gemm: negative dimension");
        si::gemm(*ctx->c, M, N, K, A, lda, a_kmajor != 0, B, ldb, b_kmajor != 0, C, ldc, alpha, beta);
    });
}

int si_spmm_csr_device(si_context* ctx, int64_t m, int64_t n, const int64_t* rowptr, const int32_t* colind,
                       const double* val, const double* P, int64_t ldp, int64_t k, double* Y, int64_t ldy) {
    return guard([&] {
        require(m >= 0 && n >= 1 && k >= 0 && ldp >= n && ldy >= m, "spmm_csr: bad shape");
        if (m > 0 && k > 0) si::spmm_csr_rows(*ctx->c, m, n, rowptr, colind, val, P, ldp, k, Y, ldy);
    });
}

int si_symupd_device(si_context* ctx, int64_t m, int64_t k, const double* V, int64_t ldv, const double* U,
                     int64_t ldu, double* X, int64_t ldx) {
    return guard([&] {
        require(m >= 0 && k >= 1 && ldv >= m && ldu >= m && ldx >= m, "symupd: bad shape");
        if (m > 0) si::symupd_device(*ctx->c, m, k, V, ldv, U, ldu, X, ldx);
    });
}

int si_sketch_gaussian_device(si_context* ctx, double* S, int64_t n, int64_t q, int64_t lds, uint64_t seed,
                              uint64_t draw) {
    return guard([&] {
        require(n >= 1 && q >= 1 && lds >= n, "sketch: bad shape");
        si::philox_sketch(*ctx->c, S, n, q, lds, seed, nullptr, draw, nullptr);
    });
}

// The sharded drivers' q×q core: for q ≤ 128 G⁻¹ comes from the single-GPU iteration's fused
// K-FACTOR kernel (one CTA, 72 µs at q = 128 against 113 µs for the blocked inverse; Ĝ goes to
// scratch and is not used), then M as in rbfgs_core_enqueue.  scratch: 6q² + 2q + 16 doubles.
static void shard_core_enqueue(si::Context& c, const double* P, int64_t ldp, int64_t q, double* M, double* scratch,
                               int* status) {
    double* ginv = scratch;
    double* t = scratch + q * q;
    double* fs = scratch + 2 * q * q;
    if (q <= 128) {
        si::rbfgs_gram_enqueue(c, P, ldp, q, ginv, fs, fs + q * q, status);
        si::rbfgs_core_tail(c, P, ldp, q, ginv, t, M, status);
    } else {
        si::rbfgs_core_enqueue(c, P, ldp, q, ginv, t, M, fs, status);
    }
}

int si_rbfgs_core_device(si_context* ctx, const double* P, int64_t ldp, int64_t q, double* M, double* scratch) {
    return guard([&] {
        auto& c = *ctx->c;
        require(q >= 1 && ldp >= q, "rbfgs_core: bad shape");
        if (!c.aux_status) ck(cudaMalloc(&c.aux_status, 4 * sizeof(int)), "malloc");
        ck(cudaMemsetAsync(c.aux_status, 0, 4 * sizeof(int), c.stream), "memset");
        shard_core_enqueue(c, P, ldp, q, M, scratch, c.aux_status);
        int st[4];
        read_status(c, c.aux_status, st);
        if (st[0]) throw ResampleError("bfgs_step: sketched Gram matrix is not positive definite");
    });
}

int si_rbfgs_core_device_async(si_context* ctx, const double* P, int64_t ldp, int64_t q, double* M,
                               double* scratch, int* status_dev) {
    return guard([&] {
        auto& c = *ctx->c;
        require(q >= 1 && ldp >= q && status_dev != nullptr, "rbfgs_core_async: bad shape");
        ck(cudaMemsetAsync(status_dev, 0, sizeof(int), c.stream), "memset");
        shard_core_enqueue(c, P, ldp, q, M, scratch, status_dev);
        si::zero_on_status(c, M, 4 * q * q, status_dev);
    });
}

int si_gather_columns_device(si_context* ctx, const double* L, int64_t rows, int64_t ldl, const int64_t* idx_dev,
                             int64_t q, double* out) {
    return guard([&] {
        require(rows >= 0 && q >= 0 && ldl >= rows, "gather_columns: bad shape");
        if (rows * q > 0) si::gather_columns(*ctx->c, L, rows, ldl, idx_dev, q, out);
    });
}

int si_ada_core_device(si_context* ctx, const double* G, int64_t q, const double* Z, int64_t n,
                       const int64_t* idx_dev, const double* St, double* T_out, double* R, double* B, double* scratch) {
    return guard([&] {
        auto& c = *ctx->c;
        require(q >= 1 && n >= q, "ada_core: bad shape");
        require(St == nullptr || T_out != nullptr, "ada_core: Gaussian S̃ needs T_out");
        if (!c.aux_status) ck(cudaMalloc(&c.aux_status, 4 * sizeof(int)), "malloc");
        ck(cudaMemsetAsync(c.aux_status, 0, 4 * sizeof(int), c.stream), "memset");
        double* g2 = scratch;
        double* r2 = scratch + q * q;
        double* es = scratch + 2 * q * q;
        si::ada_core_enqueue(c, G, q, Z, n, idx_dev, St, g2, r2, T_out, R, B, es, c.aux_status);
        int st[4];
        read_status(c, c.aux_status, st);
        if (st[0]) throw ResampleError("sym_inv_sqrt: matrix is not positive definite");
    });
}

int si_pdiag_update_device(si_context* ctx, const double* B, int64_t q, int64_t n, const double* T,
                           const int64_t* idx_dev, double* d) {
    return guard([&] {
        require(q >= 1 && n >= 1, "pdiag_update: bad shape");
        si::pdiag_update(*ctx->c, B, q, n, T, idx_dev, nullptr, d);
    });
}

int si_residual_rows_device(si_context* ctx, si_problem* prob, int64_t m, int64_t r0, const double* x_rows,
                            int64_t ldx, double* out_host) {
    return guard([&] {
        auto& c = *ctx->c;
        si::residual_rows_sq_enqueue(c, *prob->p, m, r0, x_rows, ldx, c.scalar_dev);
        ck(cudaMemcpyAsync(c.scalar_host, c.scalar_dev, sizeof(double), cudaMemcpyDeviceToHost, c.stream), "d2h");
        ck(cudaStreamSynchronize(c.stream), "sync");
        *out_host = c.scalar_host[0];
    });
}

const double* si_problem_dense_device(si_problem* prob) { return prob->p->dense ? prob->p->a : nullptr; }

// ------------------------------------------------------------ ingestion ---
int si_problem_load_matrix_market(si_context* ctx, const char* path, int symmetry, int keep_sparse,
                                  si_problem** out) {
    return guard([&] {
        const si::LoadedMatrix m = si::load_matrix_market(path, keep_sparse != 0);
        const int sym = symmetry >= 0 ? symmetry : (m.symmetric ? SI_SYMMETRIC : SI_GENERAL);
        std::unique_ptr<si_problem> h(new_problem(ctx, m.n, sym));
        if (m.sparse) {
            h->p->nnz = int64_t(m.val.size());
            si::problem_upload_csr(*h->p, m.rowptr.data(), m.colind.data(), m.val.data());
        } else {
            si::problem_upload_dense(*h->p, m.dense.data(), false);
        }
        si::shard_replicate_problem(ctx, h.get());
        *out = h.release();
    });
}

int si_problem_ridge_hessian(si_context* ctx, const char* libsvm_path, double lambda, si_problem** out) {
    return guard([&] {
        require(lambda >= 0.0, "build_ridge_hessian: lambda must be >= 0");
        const si::LibsvmRows rows = si::read_libsvm(libsvm_path);
        double* a = si::ridge_hessian_device(*ctx->c, rows, lambda);
        struct Free {
            double* p;
            ~Free() { cudaFree(p); }
        } f{a};
        std::unique_ptr<si_problem> h(new_problem(ctx, rows.n, lambda > 0.0 ? SI_SPD : SI_SYMMETRIC));
        si::problem_upload_dense(*h->p, a, true);
        si::shard_replicate_problem(ctx, h.get());
        *out = h.release();
    });
}

int si_problem_synthetic(si_context* ctx, int64_t n, uint64_t seed, si_problem** out) {
    return guard([&] {
        if (n < 2) throw ConfigError("gen_synthetic: n must be >= 2");
        double* a = si::synthetic_device(*ctx->c, n, seed);
        struct Free {
            double* p;
            ~Free() { cudaFree(p); }
        } f{a};
        std::unique_ptr<si_problem> h(new_problem(ctx, n, SI_SPD));
        si::problem_upload_dense(*h->p, a, true);
        si::shard_replicate_problem(ctx, h.get());
        *out = h.release();
    });
}

int si_io_matrix_market_info(const char* path, int64_t* n, int* symmetric, int64_t* stored) {
    return guard([&] {
        const si::LoadedMatrix m = si::load_matrix_market(path, true);
        if (n) *n = m.n;
        if (symmetric) *symmetric = m.symmetric ? 1 : 0;
        if (stored) *stored = m.sparse ? int64_t(m.val.size()) : m.n * m.n;
    });
}

int si_io_matrix_market_dense(const char* path, double* out_colmajor) {
    return guard([&] {
        const si::LoadedMatrix m = si::load_matrix_market(path, false);
        std::copy(m.dense.begin(), m.dense.end(), out_colmajor);
    });
}

int si_io_libsvm_info(const char* path, int64_t* samples, int64_t* features) {
    return guard([&] {
        const si::LibsvmRows r = si::read_libsvm(path);
        if (samples) *samples = r.m;
        if (features) *features = r.n;
    });
}

// ---------------------------------------------------------------- rng ------
struct si_rng {
    si::RngStream r;
};

int si_rng_create(uint64_t seed, si_rng** out) {
    return guard([&] { *out = new si_rng{si::RngStream(seed)}; });
}
int si_rng_substream(si_rng* r, uint64_t index, si_rng** out) {
    return guard([&] { *out = new si_rng{r->r.substream(index)}; });
}
int si_rng_destroy(si_rng* r) {
    return guard([&] { delete r; });
}
double si_rng_uniform(si_rng* r) { return r->r.uniform(); }
double si_rng_gaussian(si_rng* r) { return r->r.gaussian(); }
int64_t si_rng_categorical(si_rng* r, const double* p, int64_t n) { return r->r.categorical(p, n); }
int64_t si_rng_uniform_index(si_rng* r, int64_t n) { return r->r.uniform_index(n); }
int si_rng_gaussian_matrix(si_rng* r, int64_t rows, int64_t cols, double* out) {
    return guard([&] { r->r.gaussian_fill(out, rows, cols, rows); });
}
int si_rng_uniform_matrix(si_rng* r, int64_t rows, int64_t cols, double* out) {
    return guard([&] { r->r.uniform_fill(out, rows, cols, rows); });
}
int si_rng_uniform_subset(si_rng* r, int64_t n, int64_t q, int64_t* out) {
    return guard([&] {
        require(q >= 1 && q <= n, "uniform_subset: need 1 <= q <= n");
        const auto v = si::uniform_subset(r->r, n, q);
        std::copy(v.begin(), v.end(), out);
    });
}

}  // extern "C"

// ---------------------------------------------------------- adarbfgs_step ---
// FactoredState adarbfgs_step(state, a, rule, rng, max_redraws), adarbfgs.cpp:49-75:
// one factored update drawing from the caller's RngStream (probabilities once,
// then one draw per attempt), NumericalError after max_redraws + 1 rejections.
int si_adarbfgs_step(si_context* ctx, si_problem* prob, int sketch, int64_t q, si_rng* rng, int max_redraws,
                     const double* l_host, double* l_out_host) {
    return guard([&] {
        auto& c = *ctx->c;
        si::Problem& a = *prob->p;
        const int64_t n = a.n;
        const bool cols = sketch == SI_SKETCH_ADAPTIVE_COLS, uniform = sketch == SI_SKETCH_ADAPTIVE_COLS_UNIFORM,
                   gauss = sketch == SI_SKETCH_ADAPTIVE_GAUSS;
        if (!cols && !uniform && !gauss)
            throw ConfigError("adarbfgs_step: rule must be adaptive-factor-cols or -gauss");
        require(q >= 1 && q <= n, "SketchRule: q must satisfy 1 <= q <= n");
        require(max_redraws >= 0, "adarbfgs_step: max_redraws must be >= 0");
        validate_spd(prob);  // adarbfgs.cpp:53
        si::AdaWork w;
        struct Rel {
            si::AdaWork& w;
            ~Rel() { w.release(); }
        } rel{w};
        w.alloc(n, q, gauss);
        w.pdiag_refresh = 1;  // a single step: the exact diagonal, as the reference
        ck(cudaMemcpyAsync(w.L, l_host, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyHostToDevice, c.stream),
           "h2d l");
        const auto blocks = cols ? si::contiguous_partition(n, q) : std::vector<std::vector<si::Index>>{};
        std::vector<double> p;
        if (cols) {
            si::ada_enqueue_probabilities(c, a, w);
            ck(cudaStreamSynchronize(c.stream), "sync");
            block_probabilities(w.p_pinned, blocks, p);
        }
        int st[4];
        for (int attempt = 0; attempt <= max_redraws; ++attempt) {
            int mode = 0;
            w.q = q;
            if (cols) {
                const auto& blk = blocks[size_t(rng->r.categorical(p.data(), si::Index(p.size())))];
                w.q = int64_t(blk.size());
                for (size_t j = 0; j < blk.size(); ++j) w.idx_pinned[j] = blk[j];
            } else if (uniform) {
                const auto idx = si::uniform_subset(rng->r, n, q);
                for (int64_t j = 0; j < q; ++j) w.idx_pinned[j] = idx[size_t(j)];
            } else {
                rng->r.gaussian_fill(w.st_pinned, n, q, n);
                mode = 1;
            }
            if (mode == 0)
                ck(cudaMemcpyAsync(w.idx_dev, w.idx_pinned, size_t(w.q) * sizeof(int64_t), cudaMemcpyHostToDevice,
                                   c.stream),
                   "h2d idx");
            si::ada_enqueue_update(c, a, w, mode, 0);
            read_status(c, w.status, st);
            if (st[0]) {
                ck(cudaMemsetAsync(w.status, 0, 4 * sizeof(int), c.stream), "reset");
                continue;
            }
            ck(cudaMemcpyAsync(l_out_host, w.L, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyDeviceToHost,
                               c.stream),
               "d2h l");
            ck(cudaStreamSynchronize(c.stream), "sync");
            return;
        }
        throw NumericalError("adarbfgs_step: rejection limit exceeded for " + describe(sketch, q));
    });
}

si_solver::~si_solver() {
    if (shard) si::shard_solver_delete(shard);
    release();
}
