// Internal to the C ABI implementation (driver.cpp, shard.cpp): the opaque handle types
// of include/stochinv_b200.h and the helpers both translation units use (error mapping,
// flop tallies, history recording).  Not installed; not part of the public interface.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
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

struct si_context;
struct si_problem;

namespace si {
struct ShardGroup;  // shard.cpp: the ranks a multi-GPU context drives and their communicator
struct ShardSolver;
void shard_group_delete(ShardGroup* g);
void shard_solver_delete(ShardSolver* s);
// multi-GPU contexts (shard.cpp): A on every local rank, the sharded drivers and solver
void shard_replicate_problem(si_context* ctx, si_problem* h);
void shard_run_inverter(si_context* ctx, si_problem* prob, const si_inverter_config* cfg, double* x_out,
                        si_history_point* history, int64_t history_cap, si_run_result* result);
void shard_run_adarbfgs(si_context* ctx, si_problem* prob, const si_inverter_config* cfg, double* l_out,
                        double* x_out, si_history_point* history, int64_t history_cap, si_run_result* result);
ShardSolver* shard_solver_create(si_context* ctx, si_problem* prob, int method, int sketch, int64_t q, uint64_t seed);
void shard_solver_step(ShardSolver* s, int64_t iters, RngStream& rng, int max_redraws);
double shard_solver_residual(ShardSolver* s);
void shard_solver_get(ShardSolver* s, double* host);
void shard_solver_set(ShardSolver* s, const double* host);
int64_t shard_solver_redraws(ShardSolver* s);
}  // namespace si

namespace si_capi {

inline thread_local std::string g_err;

using si::ConfigError;
using si::NumericalError;
struct ResampleError : NumericalError {
    using NumericalError::NumericalError;
};

template <class F>
inline int guard(F&& f) {
    try {
        f();
        return SI_OK;
    } catch (const ResampleError& e) {
        g_err = e.what();
        return SI_ERR_RESAMPLE;
    } catch (const NumericalError& e) {
        g_err = e.what();
        return SI_ERR_NUMERICAL;
    } catch (const si::IoError& e) {  // errors.hpp:24-26 (CLI exit 4)
        g_err = e.what();
        return SI_ERR_IO;
    } catch (const si::CudaError& e) {
        g_err = e.what();
        return SI_ERR_CUDA;
    } catch (const std::invalid_argument& e) {  // ConfigError and ProblemMatrix's plain invalid_argument
        g_err = e.what();
        return SI_ERR_CONFIG;
    } catch (const std::bad_alloc& e) {
        g_err = std::string("allocation failed: ") + e.what();
        return SI_ERR_CUDA;
    } catch (const std::exception& e) {  // stochinv_cli.cpp:281-283 maps other std::exception to exit 2
        g_err = e.what();
        return SI_ERR_CONFIG;
    }
}

inline void ck(cudaError_t e, const char* what) { si::cuda_check(e, what); }

inline double flops_bfgs(double n, double q) { return 10 * n * n * q + 10 * n * q * q + 2 * q * q * q + 4 * n * n; }  // flops.cpp:43-46
inline double flops_adarbfgs(double n, double q) {  // flops.cpp:70-74
    return 8 * n * n * q + 10 * n * q * q + 4 * q * q * q + n * q + n * n;
}

struct DeviceTimer {
    cudaEvent_t a{}, b{};
    explicit DeviceTimer() {
        ck(cudaEventCreate(&a), "event");
        ck(cudaEventCreate(&b), "event");
    }
    ~DeviceTimer() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
    double seconds() {
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, a, b), "elapsed");
        return ms * 1e-3;
    }
};

}  // namespace si_capi

struct si_context {
    std::unique_ptr<si::Context> c;  // the (first local) device; the single-GPU API runs here
    // multi-GPU contexts (si_context_create_multi / _rank / _loopback): every local rank and
    // the communicator; null for a single-GPU context
    si::ShardGroup* group = nullptr;
    ~si_context() {
        if (group) si::shard_group_delete(group);
    }
    // optional draw log (si_context_set_draw_log): every executed sampling attempt of the
    // drivers appends its outcome — the block index (coordinate_block, adaptive_cols) or the q
    // coordinates (adaptive_cols_uniform) — in the order the reference draws them
    int64_t* draw_log = nullptr;
    int64_t draw_cap = 0;
    int64_t draw_count = 0;
    void log_draw(int64_t v) {
        if (draw_log && draw_count < draw_cap) draw_log[draw_count] = v;
        ++draw_count;
    }
};

struct si_problem {
    si_context* owner = nullptr;
    std::unique_ptr<si::Problem> p;
    // multi-GPU contexts: A on every local rank (replicas[0] = p; virtual ranks on one device share it)
    std::vector<si::Problem*> replicas;
    std::vector<std::unique_ptr<si::Problem>> owned_replicas;
};

struct si_solver {
    si_context* ctx = nullptr;
    si_problem* prob = nullptr;
    int method = 0, sketch = 0;
    int64_t q = 0;
    uint64_t seed = 0;
    si::RbfgsWork rw;
    si::AdaWork aw;
    int* status_host = nullptr;
    int64_t redraws = 0;
    std::unique_ptr<si::RngStream> rng;
    // one device-sketched iteration captured as a CUDA graph (launch-bound small n)
    cudaGraphExec_t graph = nullptr;
    int64_t graph_launches = 0;
    bool warmed = false;
    si::ShardSolver* shard = nullptr;  // multi-GPU context: the sharded iteration (shard.cpp)
    ~si_solver();
    void release() {
        if (graph) cudaGraphExecDestroy(graph);
        rw.release();
        aw.release();
        if (status_host) cudaFreeHost(status_host);
    }
};

namespace si_capi {

inline void require(bool cond, const char* msg) {
    if (!cond) throw ConfigError(msg);
}

// ProblemMatrix::validate_spd semantics (problem_matrix.cpp:28-41)
inline void validate_spd(si_problem* prob, double* scratch_nn = nullptr) {
    if (prob->p->symmetry != SI_SPD)
        throw std::invalid_argument("ProblemMatrix: operation requires an spd-flagged matrix");
    if (!si::problem_validate_spd(*prob->p, scratch_nn))
        throw std::runtime_error("ProblemMatrix: spd flag set but Cholesky failed");
}

inline double host_frobenius_asym(const double* x, int64_t n, double* norm_out) {
    double d = 0.0, nn = 0.0;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) {
            const double v = x[i + j * n];
            const double e = v - x[j + i * n];
            d += e * e;
            nn += v * v;
        }
    *norm_out = std::sqrt(nn);
    return std::sqrt(d);
}

inline std::string describe(int sketch, int64_t q) {
    const char* k = "gaussian";
    switch (sketch) {
        case SI_SKETCH_COORDINATE_BLOCK: k = "coordinate-block"; break;
        case SI_SKETCH_ADAPTIVE_COLS: k = "adaptive-factor-cols"; break;
        case SI_SKETCH_ADAPTIVE_GAUSS:
        case SI_SKETCH_ADAPTIVE_GAUSS_DEVICE: k = "adaptive-factor-gauss"; break;
        case SI_SKETCH_ADAPTIVE_COLS_UNIFORM: k = "adaptive-factor-cols-uniform"; break;
        default: break;
    }
    return std::string(k) + "(q=" + std::to_string(q) + ")";
}

// status[0..3] -> host (sync)
inline void read_status(si::Context& c, const int* status_dev, int* host) {
    ck(cudaMemcpyAsync(host, status_dev, 4 * sizeof(int), cudaMemcpyDeviceToHost, c.stream), "status d2h");
    ck(cudaStreamSynchronize(c.stream), "sync");
}

inline double residual_norm(si::Context& c, si::Problem& a, const double* X) {
    si::residual_sq_enqueue(c, a, X, c.scalar_dev, nullptr);
    ck(cudaMemcpyAsync(c.scalar_host, c.scalar_dev, sizeof(double), cudaMemcpyDeviceToHost, c.stream), "d2h");
    ck(cudaStreamSynchronize(c.stream), "sync");
    return std::sqrt(c.scalar_host[0]);
}

inline double factored_residual_norm(si::Context& c, si::Problem& a, si::AdaWork& w) {
    if (!w.AL) ck(cudaMalloc(&w.AL, size_t(w.n) * size_t(w.n) * sizeof(double)), "malloc AL");
    si::factored_residual_sq_enqueue(c, a, w.L, w.AL, c.scalar_dev);
    ck(cudaMemcpyAsync(c.scalar_host, c.scalar_dev, sizeof(double), cudaMemcpyDeviceToHost, c.stream), "d2h");
    ck(cudaStreamSynchronize(c.stream), "sync");
    return std::sqrt(c.scalar_host[0]);
}

struct HistoryWriter {
    si_history_point* buf;
    int64_t cap;
    int64_t count = 0;
    const si_inverter_config* cfg;
    void record(int64_t k, double rel, double flops, double seconds) {
        si_history_point hp{k, rel, flops, seconds};
        if (buf && count < cap) buf[count] = hp;
        ++count;
        if (cfg->on_checkpoint) cfg->on_checkpoint(&hp, cfg->user);
    }
};

inline void set_message(si_run_result* r, const std::string& m) {
    std::snprintf(r->message, sizeof(r->message), "%s", m.c_str());
}

inline void block_probabilities(const double* pdiag, const std::vector<std::vector<si::Index>>& blocks,
                                std::vector<double>& p) {
    // adarbfgs.cpp:23-36: p_i = sum_{j in C_i} l_jᵀ A l_j, then p / p.sum()
    p.assign(blocks.size(), 0.0);
    for (size_t i = 0; i < blocks.size(); ++i) {
        double tr = 0.0;
        for (si::Index j : blocks[i]) tr += pdiag[j];
        p[i] = tr;
    }
    double mn = p.empty() ? 1.0 : *std::min_element(p.begin(), p.end());
    if (mn <= 0.0)
        throw NumericalError(
            "adaptive_block_probabilities: non-positive block trace; the factor has degenerated");
    double sum = 0.0;
    for (double v : p) sum += v;
    for (double& v : p) v /= sum;
}

}  // namespace si_capi
