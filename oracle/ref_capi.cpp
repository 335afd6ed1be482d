// TEST INFRASTRUCTURE — a C entry layer over the reference's OWN sources
// (/root/reference/proj/src/*.cpp, compiled unmodified against ref_shim/, the Eigen-API
// subset), built by oracle/Makefile into oracle/_ref/libstochinv_ref.so.  It lets the tests
// check the oracle restatement (stochinv_oracle.cpp) against the reference code itself and
// lets bench.py's reference arm time the reference's run_inverter.  Nothing here is part
// of the product; the reference sources are not copied into the repository.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <optional>
#include <stdexcept>
#include <string>

#include "stochinv/adarbfgs.hpp"
#include "stochinv/errors.hpp"
#include "stochinv/linalg.hpp"
#include "stochinv/qn_updates.hpp"
#include "stochinv/simi.hpp"

using namespace stochinv;

namespace {
thread_local std::string g_err;

Matrix wrap(const double* p, Index r, Index c) {
    Matrix m(r, c);
    std::memcpy(m.data(), p, sizeof(double) * size_t(r) * size_t(c));
    return m;
}
void out(const Matrix& m, double* p) { std::memcpy(p, m.data(), sizeof(double) * size_t(m.size())); }

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const GramRankDeficientError& e) {
        g_err = e.what();
        return 6;
    } catch (const NumericalError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

void history_out(const RunResult& r, int* term, int64_t* k, int64_t* hk, double* hres, double* hflops, double* hsec,
                 int64_t hcap, int64_t* hcount) {
    *term = int(r.termination);
    *k = r.state.k;
    const auto& h = r.state.history;
    *hcount = int64_t(h.size());
    for (size_t i = 0; i < h.size() && int64_t(i) < hcap; ++i) {
        hk[i] = h[i].k;
        hres[i] = h[i].residual;
        hflops[i] = h[i].flops;
        hsec[i] = h[i].seconds;
    }
}
}  // namespace

extern "C" {

const char* rf_last_error() { return g_err.c_str(); }

int rf_bfgs_step(int64_t n, int64_t q, const double* x, const double* a, const double* s, double* x_out) {
    return guard([&] { out(bfgs_step(wrap(x, n, n), wrap(a, n, n), wrap(s, n, q)), x_out); });
}

int rf_adarbfgs_update_factor(int64_t n, int64_t q, const double* l, const double* a, const double* st, double* l_out) {
    return guard([&] { out(adarbfgs_update_factor(wrap(l, n, n), wrap(a, n, n), wrap(st, n, q)), l_out); });
}

int rf_sym_inv_sqrt(int64_t n, const double* m, double* r_out) {
    return guard([&] { out(sym_inv_sqrt(wrap(m, n, n)), r_out); });
}

// run_inverter(MethodSpec::named_method(bfgs)) — rule 0 gaussian(q), 1 coordinate_block(n, q)
int rf_run_inverter_bfgs(int64_t n, const double* a, int rule, int64_t q, double tol, int64_t max_iters,
                         int64_t every_k, uint64_t seed, int max_redraws, const double* x0, double* x_out, int* term,
                         int64_t* k, int64_t* hk, double* hres, double* hflops, double* hsec, int64_t hcap,
                         int64_t* hcount, double* drift, char* message, int64_t message_cap) {
    return guard([&] {
        InverterConfig cfg{ProblemMatrix(wrap(a, n, n), Symmetry::spd),
                           WeightSpec::identity(),
                           rule == 0 ? SketchRule::gaussian(q) : SketchRule::coordinate_block(n, q),
                           MethodSpec::named_method(UpdateName::bfgs)};
        cfg.tol = tol;
        cfg.max_iters = long(max_iters);
        cfg.seed = seed;
        cfg.track.residual_every_k = every_k;
        cfg.max_redraws = max_redraws;
        if (x0) cfg.x0 = wrap(x0, n, n);
        const RunResult r = run_inverter(cfg);
        history_out(r, term, k, hk, hres, hflops, hsec, hcap, hcount);
        *drift = r.state.max_symmetry_drift;
        if (x_out) out(r.state.x, x_out);
        if (message && message_cap > 0) std::snprintf(message, size_t(message_cap), "%s", r.message.c_str());
    });
}

// run_adarbfgs — rule 0 adaptive_cols(n, q) (contiguous blocks + Eq. 8.2), 1 adaptive_gauss(q)
int rf_run_adarbfgs(int64_t n, const double* a, int rule, int64_t q, double tol, int64_t max_iters, int64_t every_k,
                    uint64_t seed, int max_redraws, const double* l0, double* x_out, int* term, int64_t* k,
                    int64_t* hk, double* hres, double* hflops, double* hsec, int64_t hcap, int64_t* hcount) {
    return guard([&] {
        AdaConfig cfg{ProblemMatrix(wrap(a, n, n), Symmetry::spd),
                      rule == 0 ? SketchRule::adaptive_cols(n, q) : SketchRule::adaptive_gauss(q)};
        cfg.tol = tol;
        cfg.max_iters = long(max_iters);
        cfg.seed = seed;
        cfg.track.residual_every_k = every_k;
        cfg.max_redraws = max_redraws;
        if (l0) cfg.l0 = wrap(l0, n, n);
        const RunResult r = run_adarbfgs(cfg);
        history_out(r, term, k, hk, hres, hflops, hsec, hcap, hcount);
        if (x_out) out(r.state.x, x_out);  // state.x = L·Lᵀ (adarbfgs.cpp:89,122)
    });
}

}  // extern "C"
