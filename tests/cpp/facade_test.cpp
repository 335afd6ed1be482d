// Reference-style tests against the C++ facade (include/stochinv_b200.hpp):
// the same calls a stochinv user makes, now served by the sm_100a library.
// Mirrors proj/tests/test_qn_updates.cpp:199-228, test_adarbfgs.cpp:15-23,94-112,
// test_simi.cpp:163-173.  Prints one line per check; exit code = #failures.
#include <cmath>
#include <cstdio>

#include "stochinv_b200.hpp"

using namespace stochinv;

static int failures = 0;
#define CHECK(cond)                                                      \
    do {                                                                 \
        if (!(cond)) {                                                   \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                  \
        } else {                                                         \
            std::printf("ok   %s\n", #cond);                             \
        }                                                                \
    } while (0)

static double diff_norm(const Matrix& a, const Matrix& b) {
    double s = 0;
    for (Index j = 0; j < a.cols(); ++j)
        for (Index i = 0; i < a.rows(); ++i) s += (a(i, j) - b(i, j)) * (a(i, j) - b(i, j));
    return std::sqrt(s);
}

static Matrix random_spd(Index n, RngStream& rng) {  // tests/helpers.hpp:19-22
    Matrix b = rng.gaussian_matrix(n, n);
    Matrix a(n, n);
    for (Index i = 0; i < n; ++i)
        for (Index j = 0; j < n; ++j) {
            double s = 0;
            for (Index k = 0; k < n; ++k) s += b(i, k) * b(j, k);
            a(i, j) = s + (i == j ? 0.5 * double(n) : 0.0);
        }
    return a;
}

int main() {
    // BFGS hand fixture (test_qn_updates.cpp:199-207)
    Matrix a(2, 2);
    a(0, 0) = 2; a(0, 1) = 1; a(1, 0) = 1; a(1, 1) = 2;
    Matrix s(2, 1);
    s(0, 0) = 1;
    Matrix expected(2, 2);
    expected(0, 0) = 0.75; expected(0, 1) = -0.5; expected(1, 0) = -0.5; expected(1, 1) = 1.0;
    const Matrix stepped = bfgs_step(Matrix::Identity(2, 2), a, s);
    CHECK(diff_norm(stepped, expected) <= 1e-12);

    // resample signal (test_qn_updates.cpp:253-268)
    bool threw = false;
    try {
        (void)bfgs_step(Matrix::Identity(2, 2), a, Matrix::Zero(2, 1));
    } catch (const GramRankDeficientError&) {
        threw = true;
    }
    CHECK(threw);

    // scalar factored update (test_adarbfgs.cpp:15-23)
    Matrix a1(1, 1), l1(1, 1), s1(1, 1);
    a1(0, 0) = 4; l1(0, 0) = 1; s1(0, 0) = 1;
    CHECK(std::abs(adarbfgs_update_factor(l1, a1, s1)(0, 0) - 0.5) <= 1e-12);

    // run_inverter(bfgs, coordinate_block(5,2)) stays exactly symmetric (test_simi.cpp:163-173)
    RngStream rng(67);
    const Matrix spd = random_spd(5, rng);
    InverterConfig cfg{ProblemMatrix(spd, Symmetry::spd), SketchRule::coordinate_block(5, 1),
                       MethodSpec::named_method(UpdateName::bfgs)};
    cfg.tol = 0.0;
    cfg.max_iters = 30;
    int seen = 0;
    cfg.on_checkpoint = [&](const HistoryPoint&) { ++seen; };
    const RunResult res = run_inverter(cfg);
    Matrix xt(5, 5);
    for (Index i = 0; i < 5; ++i)
        for (Index j = 0; j < 5; ++j) xt(i, j) = res.state.x(j, i);
    CHECK(diff_norm(res.state.x, xt) == 0.0);
    CHECK(res.state.max_symmetry_drift < 1e-8);
    CHECK(res.termination == Termination::max_iters);
    CHECK(seen == int(res.state.history.size()));

    // AdaRBFGS converges (test_adarbfgs.cpp:94-112)
    RngStream rng2(89);
    const Matrix spd10 = random_spd(10, rng2);
    AdaConfig acfg{ProblemMatrix(spd10, Symmetry::spd), SketchRule::adaptive_gauss(2)};
    acfg.tol = 1e-6;
    acfg.max_iters = 4000;
    acfg.seed = 5;
    acfg.track.residual_every_k = 20;
    const RunResult ares = run_adarbfgs(acfg);
    CHECK(ares.termination == Termination::tol_reached);
    CHECK(ares.state.history.front().residual == 1.0);

    // configuration errors propagate as ConfigError (simi.cpp:185-213)
    bool cfg_err = false;
    try {
        InverterConfig bad{ProblemMatrix(spd, Symmetry::spd), SketchRule::gaussian(9),
                           MethodSpec::named_method(UpdateName::bfgs)};
        (void)run_inverter(bad);
    } catch (const ConfigError&) {
        cfg_err = true;
    }
    CHECK(cfg_err);

    // row f3: psb keeps X exactly symmetric and satisfies X⁺AS = S (test_qn_updates.cpp:119-132)
    Matrix sk(5, 2);
    sk(1, 0) = 1.0;
    sk(3, 1) = 1.0;
    const Matrix xp = psb_step(Matrix::Identity(5, 5), spd, sk);
    double sec = 0.0;
    for (Index j = 0; j < 2; ++j)
        for (Index i = 0; i < 5; ++i) {
            double v = 0.0;
            for (Index k = 0; k < 5; ++k)
                for (Index l = 0; l < 5; ++l) v += xp(i, k) * spd(k, l) * sk(l, j);
            sec += (v - sk(i, j)) * (v - sk(i, j));
        }
    CHECK(std::sqrt(sec) <= 1e-9);
    // dfp with S = I lands on A (test_qn_updates.cpp:176-185)
    const IteratePair full = dfp_step(Matrix::Identity(5, 5), Matrix::Identity(5, 5), spd, Matrix::Identity(5, 5));
    CHECK(diff_norm(full.primal, spd) <= 1e-9 * 10.0);
    // named dfp run tracks its inverse
    InverterConfig dcfg{ProblemMatrix(spd, Symmetry::spd), SketchRule::gaussian(2),
                        MethodSpec::named_method(UpdateName::dfp)};
    dcfg.tol = 1e-8;
    dcfg.max_iters = 3000;
    const RunResult dres = run_inverter(dcfg);
    CHECK(dres.termination == Termination::tol_reached);
    CHECK(dres.state.x_inv.has_value());
    // row f4: Newton–Schulz scalar regression and a converging run (test_baselines.cpp:14-21, 85-99)
    Matrix a2(1, 1), x2(1, 1);
    a2(0, 0) = 2.0;
    x2(0, 0) = 0.4;
    CHECK(std::abs(newton_schulz_step(x2, a2)(0, 0) - 0.48) <= 1e-14);
    BaselineConfig bcfg{ProblemMatrix(spd, Symmetry::spd)};
    bcfg.tol = 1e-8;
    bcfg.max_iters = 200;
    const RunResult bres = run_baseline(bcfg);
    CHECK(bres.termination == Termination::tol_reached);
    std::printf("%d failure(s)\n", failures);
    return failures;
}
