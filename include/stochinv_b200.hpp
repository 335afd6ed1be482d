// C++ facade over the stochinv_b200 C ABI that re-exposes the reference's
// solver API (proj/include/stochinv/*.hpp) for the RBFGS / AdaRBFGS hot path:
//
//   Matrix bfgs_step(const Matrix& x, const Matrix& a, const Matrix& s)          qn_updates.hpp:70
//   Matrix adarbfgs_update_factor(const Matrix& l, const Matrix& a, const Matrix& stilde)  adarbfgs.hpp:28
//   Vector adaptive_block_probabilities(l, a, blocks)                            adarbfgs.hpp:32-33
//   RunResult run_inverter(const InverterConfig&)     (named bfgs)               simi.hpp:105
//   RunResult run_adarbfgs(const AdaConfig&)                                     adarbfgs.hpp:59
//   ProblemMatrix, SketchRule, MethodSpec, TrackOptions, HistoryPoint, RngStream ...
//
// Matrix is Eigen::MatrixXd when STOCHINV_B200_WITH_EIGEN is defined (a drop-in
// for reference callers), otherwise the small column-major stochinv::Matrix
// below.  Errors are re-thrown as the reference's exception classes
// (errors.hpp:9-26).  Header-only; link with -lstochinv_b200.
#pragma once

#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "stochinv_b200.h"

#ifdef STOCHINV_B200_WITH_EIGEN
#include <Eigen/Dense>
#endif

namespace stochinv {

#ifdef STOCHINV_B200_WITH_EIGEN
using Matrix = Eigen::MatrixXd;
using Vector = Eigen::VectorXd;
using Index = Eigen::Index;
#else
using Index = std::ptrdiff_t;
/// Dense column-major matrix with the Eigen::MatrixXd members the facade uses.
class Matrix {
public:
    Matrix() = default;
    Matrix(Index rows, Index cols) : r_(rows), c_(cols), v_(static_cast<size_t>(rows * cols), 0.0) {}
    static Matrix Identity(Index rows, Index cols) {
        Matrix m(rows, cols);
        for (Index i = 0; i < rows && i < cols; ++i) m(i, i) = 1.0;
        return m;
    }
    static Matrix Zero(Index rows, Index cols) { return Matrix(rows, cols); }
    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    double& operator()(Index i, Index j) { return v_[static_cast<size_t>(i + j * r_)]; }
    double operator()(Index i, Index j) const { return v_[static_cast<size_t>(i + j * r_)]; }

private:
    Index r_ = 0, c_ = 0;
    std::vector<double> v_;
};
class Vector {
public:
    Vector() = default;
    explicit Vector(Index n) : v_(static_cast<size_t>(n), 0.0) {}
    Index size() const { return Index(v_.size()); }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    double& operator[](Index i) { return v_[static_cast<size_t>(i)]; }
    double operator[](Index i) const { return v_[static_cast<size_t>(i)]; }

private:
    std::vector<double> v_;
};
#endif

// ---------------------------------------------------------------- errors (errors.hpp:9-26)
struct ConfigError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct NumericalError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct GramRankDeficientError : NumericalError {
    explicit GramRankDeficientError(const std::string& what) : NumericalError(what) {}
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int rc) {
    if (rc == SI_OK) return;
    const std::string msg = si_last_error();
    switch (rc) {
        case SI_ERR_CONFIG: throw ConfigError(msg);
        case SI_ERR_NUMERICAL: throw NumericalError(msg);
        case SI_ERR_RESAMPLE: throw GramRankDeficientError(msg);
        case SI_ERR_IO: throw IoError(msg);
        default: throw DeviceError(msg);
    }
}
/// One context per host thread (the reference's single-owner state).
inline si_context* context() {
    struct Holder {
        si_context* c = nullptr;
        ~Holder() {
            if (c) si_context_destroy(c);
        }
    };
    thread_local Holder h;
    if (!h.c) check(si_context_create(0, &h.c));
    return h.c;
}
template <class M>
M make(Index r, Index c) {
    return M(r, c);
}
}  // namespace detail

// ---------------------------------------------------------------- problem_matrix.hpp:7-35
enum class Symmetry { general = SI_GENERAL, symmetric = SI_SYMMETRIC, spd = SI_SPD };

class ProblemMatrix {
public:
    ProblemMatrix(const Matrix& data, Symmetry symmetry) : sym_(symmetry) {
        if (data.rows() != data.cols() || data.rows() < 1)
            throw std::invalid_argument("ProblemMatrix: matrix must be square with n >= 1");
        si_problem* p = nullptr;
        detail::check(si_problem_create_dense(detail::context(), data.rows(), data.data(), int(symmetry), &p));
        h_.reset(p, [](si_problem* q) { si_problem_destroy(q); });
    }
    /// CSR constructor (sparse A; an addition — the reference densifies, io.cpp:72)
    ProblemMatrix(Index n, const std::vector<int64_t>& rowptr, const std::vector<int32_t>& colind,
                  const std::vector<double>& val, Symmetry symmetry)
        : sym_(symmetry) {
        si_problem* p = nullptr;
        detail::check(si_problem_create_csr(detail::context(), n, int64_t(val.size()), rowptr.data(), colind.data(),
                                            val.data(), int(symmetry), &p));
        h_.reset(p, [](si_problem* q) { si_problem_destroy(q); });
    }
    Index n() const { return Index(si_problem_n(h_.get())); }
    Symmetry symmetry() const { return sym_; }
    bool is_symmetric() const { return sym_ != Symmetry::general; }
    void validate_spd() const { detail::check(si_problem_validate_spd(h_.get())); }
    Matrix data() const {
        Matrix m = detail::make<Matrix>(n(), n());
        detail::check(si_problem_get_dense(h_.get(), m.data()));
        return m;
    }
    si_problem* handle() const { return h_.get(); }

private:
    Symmetry sym_;
    std::shared_ptr<si_problem> h_;
};

// ---------------------------------------------------------------- sketching.hpp:15-77
enum class SketchKind {
    gaussian_dense = SI_SKETCH_GAUSSIAN,
    gaussian_device = SI_SKETCH_GAUSSIAN_DEVICE,
    coordinate_block = SI_SKETCH_COORDINATE_BLOCK,
    adaptive_factor_cols = SI_SKETCH_ADAPTIVE_COLS,
    adaptive_factor_gauss = SI_SKETCH_ADAPTIVE_GAUSS,
    adaptive_factor_cols_uniform = SI_SKETCH_ADAPTIVE_COLS_UNIFORM,
    adaptive_factor_gauss_device = SI_SKETCH_ADAPTIVE_GAUSS_DEVICE,
};
enum class ProbabilityRule { uniform, convenient, none };

struct SketchRule {
    SketchKind kind = SketchKind::gaussian_dense;
    Index q = 1;
    ProbabilityRule probabilities = ProbabilityRule::none;
    static SketchRule gaussian(Index q) { return {SketchKind::gaussian_dense, q, ProbabilityRule::none}; }
    static SketchRule gaussian_device(Index q) { return {SketchKind::gaussian_device, q, ProbabilityRule::none}; }
    static SketchRule coordinate_block(Index /*n*/, Index q, ProbabilityRule p = ProbabilityRule::uniform) {
        return {SketchKind::coordinate_block, q, p};
    }
    static SketchRule adaptive_cols(Index /*n*/, Index q) {
        return {SketchKind::adaptive_factor_cols, q, ProbabilityRule::uniform};
    }
    static SketchRule adaptive_gauss(Index q) { return {SketchKind::adaptive_factor_gauss, q, ProbabilityRule::none}; }
    static SketchRule adaptive_cols_uniform(Index q) {
        return {SketchKind::adaptive_factor_cols_uniform, q, ProbabilityRule::uniform};
    }
    bool is_adaptive() const {
        return kind == SketchKind::adaptive_factor_cols || kind == SketchKind::adaptive_factor_gauss ||
               kind == SketchKind::adaptive_factor_cols_uniform || kind == SketchKind::adaptive_factor_gauss_device;
    }
};

inline std::vector<std::vector<Index>> contiguous_partition(Index n, Index q) {  // sketching.cpp:106-115
    if (q < 1 || q > n) throw ConfigError("contiguous_partition: need 1 <= q <= n");
    std::vector<std::vector<Index>> blocks;
    for (Index s = 0; s < n; s += q) {
        std::vector<Index> b;
        for (Index i = s; i < std::min(s + q, n); ++i) b.push_back(i);
        blocks.push_back(std::move(b));
    }
    return blocks;
}

// ---------------------------------------------------------------- simi.hpp:36-107
enum class UpdateName { kaczmarz, bad_broyden, psb, good_broyden, aip, dfp, bfgs, column };
enum class VariantKind { generic_row, generic_col, generic_sym, named };
struct MethodSpec {
    VariantKind kind = VariantKind::named;
    UpdateName name = UpdateName::bfgs;
    static MethodSpec named_method(UpdateName n) { return {VariantKind::named, n}; }
};

struct TrackOptions {
    Index residual_every_k = 10;
    bool flops = true;
    bool wall_time = true;
};

struct HistoryPoint {
    long k = 0;
    double residual = 0.0;
    double flops = 0.0;
    double seconds = 0.0;
};

enum class Termination { tol_reached = SI_TOL_REACHED, max_iters = SI_MAX_ITERS, error = SI_TERMINATION_ERROR };

struct InverterState {
    Matrix x;
    std::optional<Matrix> x_inv;  // dfp's tracked inverse (tracks_inverse_iterate)
    long k = 0;
    std::vector<HistoryPoint> history;
    double max_symmetry_drift = 0.0;
    double flops = 0.0;
    double seconds = 0.0;
};

struct RunResult {
    InverterState state;
    Termination termination = Termination::error;
    std::string message;
    Matrix l;  // AdaRBFGS factor (FactoredState::l)
};

struct InverterConfig {
    ProblemMatrix a;
    SketchRule rule;
    MethodSpec method;
    double tol = 1e-2;
    long max_iters = 1000;
    double time_budget_seconds = 0.0;
    std::uint64_t seed = 0;
    TrackOptions track;
    std::optional<Matrix> x0;
    int max_redraws = 100;
    std::function<void(const HistoryPoint&)> on_checkpoint;  // addition
};

struct AdaConfig {
    ProblemMatrix a;
    SketchRule rule;
    double tol = 1e-2;
    long max_iters = 1000;
    double time_budget_seconds = 0.0;
    std::uint64_t seed = 0;
    TrackOptions track;
    std::optional<Matrix> l0;
    int max_redraws = 100;
    std::function<void(const HistoryPoint&)> on_checkpoint;
};

namespace detail {
inline void trampoline(const si_history_point* p, void* user) {
    auto* f = static_cast<std::function<void(const HistoryPoint&)>*>(user);
    (*f)(HistoryPoint{long(p->k), p->residual, p->flops, p->seconds});
}
template <class Cfg>
si_inverter_config to_c(const Cfg& c, const std::optional<Matrix>& start,
                        const std::function<void(const HistoryPoint&)>* cb) {
    si_inverter_config o;
    si_default_config(&o);
    o.sketch = int(c.rule.kind);
    o.probabilities = c.rule.probabilities == ProbabilityRule::convenient ? SI_PROB_CONVENIENT : SI_PROB_UNIFORM;
    o.q = c.rule.q;
    o.tol = c.tol;
    o.max_iters = c.max_iters;
    o.time_budget_seconds = c.time_budget_seconds;
    o.seed = c.seed;
    o.residual_every_k = c.track.residual_every_k;
    o.track_flops = c.track.flops;
    o.track_wall_time = c.track.wall_time;
    o.max_redraws = c.max_redraws;
    o.x0_host = start ? start->data() : nullptr;
    if (cb && *cb) {
        o.on_checkpoint = &trampoline;
        o.user = const_cast<void*>(static_cast<const void*>(cb));
    }
    return o;
}
inline std::vector<HistoryPoint> history(const std::vector<si_history_point>& h, int64_t count) {
    std::vector<HistoryPoint> out;
    for (int64_t i = 0; i < count && i < int64_t(h.size()); ++i)
        out.push_back({long(h[size_t(i)].k), h[size_t(i)].residual, h[size_t(i)].flops, h[size_t(i)].seconds});
    return out;
}
}  // namespace detail

namespace detail {
inline int update_code(const MethodSpec& m) {
    if (m.kind == VariantKind::named) {
        switch (m.name) {
            case UpdateName::bfgs: return SI_UPDATE_BFGS;
            case UpdateName::psb: return SI_UPDATE_PSB;
            case UpdateName::aip: return SI_UPDATE_AIP;
            case UpdateName::dfp: return SI_UPDATE_DFP;
            default: break;
        }
    }
    throw ConfigError("stochinv_b200: only the named bfgs / psb / aip / dfp updates are on the GPU path");
}
}  // namespace detail

/// RunResult run_inverter(const InverterConfig&), simi.hpp:105 (named bfgs / psb / aip / dfp).
inline RunResult run_inverter(const InverterConfig& config) {
    const int upd = detail::update_code(config.method);
    const Index n = config.a.n();
    if (config.x0 && (config.x0->rows() != n || config.x0->cols() != n))
        throw ConfigError("run_inverter: x0 dimension mismatch");
    si_inverter_config c = detail::to_c(config, config.x0, &config.on_checkpoint);
    c.update = upd;
    std::vector<si_history_point> h(size_t(config.max_iters / std::max<Index>(1, config.track.residual_every_k) + 4));
    si_run_result r;
    RunResult out;
    out.state.x = detail::make<Matrix>(n, n);
    if (upd == SI_UPDATE_DFP) out.state.x_inv = detail::make<Matrix>(n, n);
    detail::check(si_run_inverter_pair(detail::context(), config.a.handle(), &c, out.state.x.data(),
                                       out.state.x_inv ? out.state.x_inv->data() : nullptr, h.data(),
                                       int64_t(h.size()), &r));
    out.state.k = long(r.k);
    out.state.history = detail::history(h, r.history_count);
    out.state.max_symmetry_drift = r.max_symmetry_drift;
    out.state.flops = r.flops;
    out.state.seconds = r.seconds;
    out.termination = Termination(r.termination);
    out.message = r.message;
    return out;
}

// ---------------------------------------------------------------- baselines.hpp:36-68
enum class BaselineMethod { newton_schulz = SI_BASELINE_NEWTON_SCHULZ, minimal_residual = SI_BASELINE_MINIMAL_RESIDUAL };
struct BaselineConfig {
    ProblemMatrix a;
    BaselineMethod method = BaselineMethod::newton_schulz;
    double tol = 1e-2;
    long max_iters = 1000;
    double time_budget_seconds = 0.0;
    std::uint64_t seed = 0;
    TrackOptions track;
    std::optional<Matrix> x0;
    std::function<void(const HistoryPoint&)> on_checkpoint;
};

/// RunResult run_baseline(const BaselineConfig&), baselines.hpp:68.
inline RunResult run_baseline(const BaselineConfig& config) {
    const Index n = config.a.n();
    if (config.x0 && (config.x0->rows() != n || config.x0->cols() != n))
        throw ConfigError("run_baseline: x0 dimension mismatch");
    si_inverter_config c;
    si_default_config(&c);
    c.tol = config.tol;
    c.max_iters = config.max_iters;
    c.time_budget_seconds = config.time_budget_seconds;
    c.seed = config.seed;
    c.residual_every_k = config.track.residual_every_k;
    c.track_flops = config.track.flops;
    c.track_wall_time = config.track.wall_time;
    c.x0_host = config.x0 ? config.x0->data() : nullptr;
    if (config.on_checkpoint) {
        c.on_checkpoint = &detail::trampoline;
        c.user = const_cast<void*>(static_cast<const void*>(&config.on_checkpoint));
    }
    std::vector<si_history_point> h(size_t(config.max_iters / std::max<Index>(1, config.track.residual_every_k) + 4));
    si_run_result r;
    RunResult out;
    out.state.x = detail::make<Matrix>(n, n);
    detail::check(si_run_baseline(detail::context(), config.a.handle(), int(config.method), &c, out.state.x.data(),
                                  h.data(), int64_t(h.size()), &r));
    out.state.k = long(r.k);
    out.state.history = detail::history(h, r.history_count);
    out.state.flops = r.flops;
    out.state.seconds = r.seconds;
    out.termination = Termination(r.termination);
    out.message = r.message;
    return out;
}

/// Matrix newton_schulz_step(x, a) = 2X − XAX, baselines.hpp:15.
inline Matrix newton_schulz_step(const Matrix& x, const Matrix& a) {
    const Index n = x.rows();
    Matrix out = detail::make<Matrix>(n, n);
    detail::check(si_newton_schulz_step(detail::context(), n, x.data(), a.data(), out.data()));
    return out;
}

/// RunResult run_adarbfgs(const AdaConfig&), adarbfgs.hpp:59; state.x = L Lᵀ.
inline RunResult run_adarbfgs(const AdaConfig& config) {
    const Index n = config.a.n();
    if (config.l0 && (config.l0->rows() != n || config.l0->cols() != n))
        throw ConfigError("run_adarbfgs: l0 dimension mismatch");
    si_inverter_config c = detail::to_c(config, config.l0, &config.on_checkpoint);
    std::vector<si_history_point> h(size_t(config.max_iters / std::max<Index>(1, config.track.residual_every_k) + 4));
    si_run_result r;
    RunResult out;
    out.state.x = detail::make<Matrix>(n, n);
    out.l = detail::make<Matrix>(n, n);
    detail::check(si_run_adarbfgs(detail::context(), config.a.handle(), &c, out.l.data(), out.state.x.data(),
                                  h.data(), int64_t(h.size()), &r));
    out.state.k = long(r.k);
    out.state.history = detail::history(h, r.history_count);
    out.state.flops = r.flops;
    out.state.seconds = r.seconds;
    out.termination = Termination(r.termination);
    out.message = r.message;
    return out;
}

/// Matrix bfgs_step(x, a, s), qn_updates.hpp:70.  Throws GramRankDeficientError.
inline Matrix bfgs_step(const Matrix& x, const Matrix& a, const Matrix& s) {
    const Index n = s.rows(), q = s.cols();
    if (x.rows() != n || x.cols() != n || a.rows() != n || a.cols() != n)
        throw ConfigError("bfgs_step: dimension mismatch");
    Matrix out = detail::make<Matrix>(n, n);
    detail::check(si_bfgs_step(detail::context(), n, q, x.data(), a.data(), s.data(), out.data()));
    return out;
}

/// Matrix psb_step / aip_step (x, a, s), qn_updates.hpp.  Throw GramRankDeficientError.
inline Matrix psb_step(const Matrix& x, const Matrix& a, const Matrix& s) {
    const Index n = s.rows(), q = s.cols();
    Matrix out = detail::make<Matrix>(n, n);
    detail::check(si_psb_step(detail::context(), n, q, x.data(), a.data(), s.data(), out.data()));
    return out;
}
inline Matrix aip_step(const Matrix& x, const Matrix& a, const Matrix& s) {
    const Index n = s.rows(), q = s.cols();
    Matrix out = detail::make<Matrix>(n, n);
    detail::check(si_aip_step(detail::context(), n, q, x.data(), a.data(), s.data(), out.data()));
    return out;
}
struct IteratePair {
    Matrix primal, inverse;
};
/// IteratePair dfp_step(x, x_inv, a, s), qn_updates.hpp.
inline IteratePair dfp_step(const Matrix& x, const Matrix& x_inv, const Matrix& a, const Matrix& s) {
    const Index n = s.rows(), q = s.cols();
    IteratePair out{detail::make<Matrix>(n, n), detail::make<Matrix>(n, n)};
    detail::check(si_dfp_step(detail::context(), n, q, x.data(), x_inv.data(), a.data(), s.data(), out.primal.data(),
                              out.inverse.data()));
    return out;
}

/// Matrix adarbfgs_update_factor(l, a, stilde), adarbfgs.hpp:28.  Throws NumericalError.
inline Matrix adarbfgs_update_factor(const Matrix& l, const Matrix& a, const Matrix& stilde) {
    const Index n = stilde.rows(), q = stilde.cols();
    Matrix out = detail::make<Matrix>(n, n);
    const int rc = si_adarbfgs_update_factor(detail::context(), n, q, l.data(), a.data(), stilde.data(), out.data());
    if (rc == SI_ERR_RESAMPLE) throw NumericalError(si_last_error());  // linalg.cpp:150-151
    detail::check(rc);
    return out;
}

/// Vector adaptive_block_probabilities(l, a, blocks), adarbfgs.hpp:32-33.
inline Vector adaptive_block_probabilities(const Matrix& l, const Matrix& a,
                                           const std::vector<std::vector<Index>>& blocks) {
    std::vector<int64_t> offs{0}, idx;
    for (const auto& b : blocks) {
        for (Index i : b) idx.push_back(int64_t(i));
        offs.push_back(int64_t(idx.size()));
    }
    Vector p(Index(blocks.size()));
    detail::check(si_adaptive_block_probabilities(detail::context(), l.rows(), l.data(), a.data(),
                                                  int64_t(blocks.size()), offs.data(), idx.data(), p.data()));
    return p;
}

/// RngStream, rng.hpp:13-71 (the same host stream the drivers draw from).
class RngStream {
public:
    explicit RngStream(std::uint64_t seed) {
        si_rng* r = nullptr;
        detail::check(si_rng_create(seed, &r));
        h_.reset(r, [](si_rng* p) { si_rng_destroy(p); });
    }
    RngStream substream(std::uint64_t index) const {
        si_rng* r = nullptr;
        detail::check(si_rng_substream(h_.get(), index, &r));
        return RngStream(r);
    }
    double uniform() { return si_rng_uniform(h_.get()); }
    double gaussian() { return si_rng_gaussian(h_.get()); }
    Index categorical(const Vector& p) { return Index(si_rng_categorical(h_.get(), p.data(), p.size())); }
    Index uniform_index(Index n) { return Index(si_rng_uniform_index(h_.get(), n)); }
    Matrix gaussian_matrix(Index rows, Index cols) {
        Matrix m = detail::make<Matrix>(rows, cols);
        detail::check(si_rng_gaussian_matrix(h_.get(), rows, cols, m.data()));
        return m;
    }
    Matrix uniform_matrix(Index rows, Index cols) {
        Matrix m = detail::make<Matrix>(rows, cols);
        detail::check(si_rng_uniform_matrix(h_.get(), rows, cols, m.data()));
        return m;
    }

    si_rng* handle() const { return h_.get(); }

private:
    explicit RngStream(si_rng* r) { h_.reset(r, [](si_rng* p) { si_rng_destroy(p); }); }
    std::shared_ptr<si_rng> h_;
};

/// FactoredState (adarbfgs.hpp:15-22, the step-level subset) and
/// FactoredState adarbfgs_step(state, a, rule, rng, max_redraws), adarbfgs.hpp:37-38.
struct FactoredState {
    Matrix l;
    long k = 0;
};
inline FactoredState adarbfgs_step(const FactoredState& state, const ProblemMatrix& a, const SketchRule& rule,
                                   RngStream& rng, int max_redraws = 100) {
    const Index n = a.n();
    FactoredState next{detail::make<Matrix>(n, n), state.k + 1};
    const int rc = si_adarbfgs_step(detail::context(), a.handle(), int(rule.kind), rule.q, rng.handle(), max_redraws,
                                    state.l.data(), next.l.data());
    if (rc == SI_ERR_CONFIG) throw ConfigError(si_last_error());
    if (rc != SI_OK) throw NumericalError(si_last_error());
    return next;
}

// flops.cpp:43-46, 70-74
namespace flops {
inline double bfgs(Index n_, Index q_) {
    const double n = double(n_), q = double(q_);
    return 10 * n * n * q + 10 * n * q * q + 2 * q * q * q + 4 * n * n;
}
inline double adarbfgs(Index n_, Index q_) {
    const double n = double(n_), q = double(q_);
    return 8 * n * n * q + 10 * n * q * q + 4 * q * q * q + n * q + n * n;
}
}  // namespace flops

}  // namespace stochinv
