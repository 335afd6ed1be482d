// ============================================================================
// stochinv CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A from-scratch C++ restatement of the reference's RBFGS / AdaRBFGS hot path
// (arxiv 1602.01768, `stochinv` C++ library under /root/reference/proj).  It is
// the parity checker for the CUDA product path and the CPU baseline timed by
// bench.py (`cpu_baseline.kind = "port"`).  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it; the product
// library (paper_1602_01768_b200/) never links or calls it.
//
// Why a restatement: the reference needs Eigen3 + vendored doctest/CLI11 which
// are absent from this image (no network), so per the task rules it is treated
// as unbuildable; see DESIGN.md §Oracle.  Every function cites the reference
// file:line it follows.  Parity is pinned against the reference's own
// known-answer tests (tests/test_oracle_pins.py, SURVEY §4 pin table).
//
// Dense matrices are column-major like Eigen::MatrixXd (types.hpp:8).  GEMMs go
// through OpenBLAS (numpy's bundled ILP64 build, dlopen'ed) when present, else
// a plain blocked loop; either way the arithmetic follows the reference's
// expression order operation by operation (rounding of a single GEMM differs
// from Eigen's blocking at the 1e-16 level, as SURVEY §8c notes).
// ============================================================================
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <glob.h>
#include <malloc.h>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace oracle {

// Host threads for the elementwise passes and OpenBLAS (or_set_threads; 0 = all).
static int g_threads = 0;

// Minimal parallel-for over [0, count) on the host threads (this image has no
// OpenMP runtime); used for the O(n²) elementwise passes, GEMMs use OpenBLAS.
template <class F>
void parallel_for(long count, F&& f) {
    const long hw = g_threads > 0 ? long(g_threads) : long(std::thread::hardware_concurrency());
    const long nt = std::max(1L, std::min<long>(count, hw));
    if (nt <= 1) {
        for (long i = 0; i < count; ++i) f(i);
        return;
    }
    std::vector<std::thread> pool;
    for (long t = 0; t < nt; ++t)
        pool.emplace_back([&, t] {
            for (long i = t; i < count; i += nt) f(i);
        });
    for (auto& th : pool) th.join();
}

using Index = std::ptrdiff_t;

struct ConfigError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct NumericalError : std::runtime_error { using std::runtime_error::runtime_error; };
struct GramRankDeficientError : NumericalError { using NumericalError::NumericalError; };

// ---------------------------------------------------------------- Mat ------
struct Mat {
    Index r = 0, c = 0;
    std::vector<double> v;
    Mat() = default;
    Mat(Index rows, Index cols, double fill = 0.0) : r(rows), c(cols), v(size_t(rows * cols), fill) {}
    double& operator()(Index i, Index j) { return v[size_t(i + j * r)]; }
    double operator()(Index i, Index j) const { return v[size_t(i + j * r)]; }
    double* data() { return v.data(); }
    const double* data() const { return v.data(); }
    static Mat identity(Index n) {
        Mat m(n, n);
        for (Index i = 0; i < n; ++i) m(i, i) = 1.0;
        return m;
    }
    Mat t() const {
        Mat o(c, r);
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) o(j, i) = (*this)(i, j);
        return o;
    }
    double squared_norm() const {
        double s = 0.0;
        for (double x : v) s += x * x;
        return s;
    }
    double norm() const { return std::sqrt(squared_norm()); }
    bool all_finite() const {
        for (double x : v)
            if (!std::isfinite(x)) return false;
        return true;
    }
};

Mat operator+(const Mat& a, const Mat& b) {
    Mat o = a;
    for (size_t i = 0; i < o.v.size(); ++i) o.v[i] += b.v[i];
    return o;
}
Mat operator-(const Mat& a, const Mat& b) {
    Mat o = a;
    for (size_t i = 0; i < o.v.size(); ++i) o.v[i] -= b.v[i];
    return o;
}
Mat operator*(double s, const Mat& a) {
    Mat o = a;
    for (double& x : o.v) x *= s;
    return o;
}

// ---------------------------------------------------------------- GEMM -----
// C = op(A) * op(B); column-major; OpenBLAS ILP64 when available.
using cblas_dgemm_t = void (*)(int, int, int, int64_t, int64_t, int64_t, double, const double*, int64_t,
                               const double*, int64_t, double, double*, int64_t);
static cblas_dgemm_t g_dgemm = nullptr;
using blas_threads_t = void (*)(int);
static blas_threads_t g_blas_threads = nullptr;
static bool g_blas_probed = false;

static void probe_blas() {
    if (g_blas_probed) return;
    g_blas_probed = true;
    if (const char* off = std::getenv("SI_ORACLE_NO_BLAS"); off && off[0] == '1') return;
    std::vector<std::string> candidates;
    if (const char* p = std::getenv("SI_ORACLE_BLAS")) candidates.emplace_back(p);
    glob_t g;
    const char* pats[] = {"/opt/prime-rl/.venv/lib/python3.12/site-packages/numpy.libs/libscipy_openblas64_*.so",
                          "/usr/lib/x86_64-linux-gnu/libopenblas*.so*"};
    for (const char* pat : pats) {
        if (glob(pat, 0, nullptr, &g) == 0) {
            for (size_t i = 0; i < g.gl_pathc; ++i) candidates.emplace_back(g.gl_pathv[i]);
        }
        globfree(&g);
    }
    for (const auto& path : candidates) {
        void* h = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL);
        if (!h) continue;
        auto f = reinterpret_cast<cblas_dgemm_t>(dlsym(h, "scipy_cblas_dgemm64_"));
        if (f) {
            g_dgemm = f;
            g_blas_threads = reinterpret_cast<blas_threads_t>(dlsym(h, "scipy_openblas_set_num_threads64_"));
            return;
        }
    }
}

Mat gemm(const Mat& a, bool ta, const Mat& b, bool tb) {
    probe_blas();
    const Index m = ta ? a.c : a.r, k = ta ? a.r : a.c;
    const Index kb = tb ? b.c : b.r, n = tb ? b.r : b.c;
    if (k != kb) throw std::invalid_argument("gemm: inner dimension mismatch");
    Mat out(m, n);
    if (m == 0 || n == 0) return out;
    if (k == 0) return out;
    if (g_dgemm) {
        g_dgemm(102, ta ? 112 : 111, tb ? 112 : 111, m, n, k, 1.0, a.data(), std::max<Index>(1, a.r), b.data(),
                std::max<Index>(1, b.r), 0.0, out.data(), std::max<Index>(1, m));
        return out;
    }
    auto A = [&](Index i, Index p) { return ta ? a(p, i) : a(i, p); };
    auto B = [&](Index p, Index j) { return tb ? b(j, p) : b(p, j); };
    for (Index j = 0; j < n; ++j)
        for (Index p = 0; p < k; ++p) {
            const double bpj = B(p, j);
            for (Index i = 0; i < m; ++i) out(i, j) += A(i, p) * bpj;
        }
    return out;
}
Mat mul(const Mat& a, const Mat& b) { return gemm(a, false, b, false); }

// ---------------------------------------------------------------- RNG ------
// Restates proj/include/stochinv/rng.hpp:13-71 verbatim in behaviour: splitmix64
// seeding (rng.hpp:62-67), std::mt19937_64, libstdc++ distributions, a fresh
// normal_distribution per gaussian_matrix call, column-major fill (rng.hpp:42-49).
class RngStream {
public:
    explicit RngStream(std::uint64_t seed) : state_(mix(seed)), engine_(state_) {}
    RngStream substream(std::uint64_t index) const {  // rng.hpp:18-20
        return RngStream(state_ ^ (0x9e3779b97f4a7c15ULL * (index + 1)));
    }
    double uniform() { return std::uniform_real_distribution<double>(0.0, 1.0)(engine_); }  // rng.hpp:24
    double gaussian() { return std::normal_distribution<double>(0.0, 1.0)(engine_); }      // rng.hpp:25
    Index categorical(const double* p, Index n) {                                          // rng.hpp:28-36
        double u = uniform();
        double acc = 0.0;
        for (Index i = 0; i < n; ++i) {
            acc += p[i];
            if (u < acc) return i;
        }
        return n - 1;
    }
    Index uniform_index(Index n) { return std::uniform_int_distribution<Index>(0, n - 1)(engine_); }  // rng.hpp:38-40
    void gaussian_fill(double* m, Index rows, Index cols) {                                           // rng.hpp:42-49
        std::normal_distribution<double> dist(0.0, 1.0);
        for (Index j = 0; j < cols; ++j)
            for (Index i = 0; i < rows; ++i) m[i + j * rows] = dist(engine_);
    }
    Mat gaussian_matrix(Index rows, Index cols) {
        Mat m(rows, cols);
        gaussian_fill(m.data(), rows, cols);
        return m;
    }
    void uniform_fill(double* m, Index rows, Index cols) {  // rng.hpp:51-58
        std::uniform_real_distribution<double> dist(0.0, 1.0);
        for (Index j = 0; j < cols; ++j)
            for (Index i = 0; i < rows; ++i) m[i + j * rows] = dist(engine_);
    }

private:
    static std::uint64_t mix(std::uint64_t x) {
        x += 0x9e3779b97f4a7c15ULL;
        x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
        x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
        return x ^ (x >> 31);
    }
    std::uint64_t state_;
    std::mt19937_64 engine_;
};

// ------------------------------------------------------------ LLT ----------
// Eigen::LLT semantics as used by gram_llt (qn_updates.cpp:37-43): lower
// Cholesky of the symmetric input (lower triangle read); failure on a
// non-positive or non-finite pivot.
struct Llt {
    Mat l;
    bool ok = true;
    explicit Llt(const Mat& g) : l(g.r, g.c) {
        const Index q = g.r;
        for (Index j = 0; j < q; ++j) {
            double d = g(j, j);
            for (Index p = 0; p < j; ++p) d -= l(j, p) * l(j, p);
            if (!(d > 0.0)) {
                ok = false;
                return;
            }
            const double ljj = std::sqrt(d);
            l(j, j) = ljj;
            for (Index i = j + 1; i < q; ++i) {
                double s = g(i, j);
                for (Index p = 0; p < j; ++p) s -= l(i, p) * l(j, p);
                l(i, j) = s / ljj;
            }
        }
    }
    // solve (L L^T) X = B
    Mat solve(const Mat& b) const {
        const Index q = l.r;
        Mat x = b;
        for (Index c = 0; c < x.c; ++c) {
            double* col = &x(0, c);
            for (Index i = 0; i < q; ++i) {
                double s = col[i];
                for (Index p = 0; p < i; ++p) s -= l(i, p) * col[p];
                col[i] = s / l(i, i);
            }
            for (Index i = q - 1; i >= 0; --i) {
                double s = col[i];
                for (Index p = i + 1; p < q; ++p) s -= l(p, i) * col[p];
                col[i] = s / l(i, i);
            }
        }
        return x;
    }
};

Llt gram_llt(const Mat& gram, const char* kernel) {  // qn_updates.cpp:37-43
    Llt llt(gram);
    if (!llt.ok) throw GramRankDeficientError(std::string(kernel) + ": sketched Gram matrix is not positive definite");
    return llt;
}

// ------------------------------------------------------------ bfgs_step ----
// proj/src/qn_updates.cpp:176-186, same expression order.
// Raw-pointer GEMM on column-major operands: C(m×n) = op(A)·op(B).
void gemm_raw(Index m, Index n, Index k, const double* A, Index lda, bool ta, const double* B, Index ldb, bool tb,
              double* C, Index ldc) {
    probe_blas();
    if (m == 0 || n == 0) return;
    if (g_dgemm && k > 0) {
        g_dgemm(102, ta ? 112 : 111, tb ? 112 : 111, m, n, k, 1.0, A, std::max<Index>(1, lda), B,
                std::max<Index>(1, ldb), 0.0, C, std::max<Index>(1, ldc));
        return;
    }
    for (Index j = 0; j < n; ++j) {
        for (Index i = 0; i < m; ++i) C[i + j * ldc] = 0.0;
        for (Index p = 0; p < k; ++p) {
            const double bpj = tb ? B[j + p * ldb] : B[p + j * ldb];
            for (Index i = 0; i < m; ++i) C[i + j * ldc] += (ta ? A[p + i * lda] : A[i + p * lda]) * bpj;
        }
    }
}

// proj/src/qn_updates.cpp:176-186, same expression order; operands borrowed
// (the reference takes const Matrix&), n×n temporaries as Eigen evaluates them.
void bfgs_step_raw(Index n, Index q, const double* x, const double* a, const double* s, double* out) {
    Mat as(n, q);
    gemm_raw(n, q, n, a, n, false, s, n, false, as.data(), n);  // :177  A S
    Mat gram(q, q);
    gemm_raw(q, q, n, s, n, true, as.data(), n, false, gram.data(), q);  // :178  S^T A S
    const Llt llt = gram_llt(gram, "bfgs_step");                         // :179
    const Mat t1 = llt.solve(as.t());                                    // :180
    Mat st(q, n);
    for (Index j = 0; j < q; ++j)
        for (Index i = 0; i < n; ++i) st(j, i) = s[i + j * n];
    const Mat t2 = llt.solve(st);  // :181
    Mat k(q, n);
    gemm_raw(q, n, n, t1.data(), q, false, x, n, false, k.data(), q);  // :182
    Mat pax(n, n);
    gemm_raw(n, n, q, s, n, false, k.data(), q, false, pax.data(), n);  // :183
    // :185  s*t2 + x - pax - pax^T + s*((k*t1^T)*s^T)
    Mat st2(n, n);
    gemm_raw(n, n, q, s, n, false, t2.data(), q, false, st2.data(), n);
    const Mat core = gemm(k, false, t1, true);
    Mat cst(q, n);
    gemm_raw(q, n, q, core.data(), q, false, s, n, true, cst.data(), q);
    Mat last(n, n);
    gemm_raw(n, n, q, s, n, false, cst.data(), q, false, last.data(), n);
    // combine in cache blocks so the transposed read of pax stays in cache
    const Index B = 64;
    const Index nb = (n + B - 1) / B;
    parallel_for(long(nb), [&](long jbi) {
        const Index jb = Index(jbi) * B;
        for (Index ib = 0; ib < n; ib += B)
            for (Index j = jb; j < std::min(n, jb + B); ++j)
                for (Index i = ib; i < std::min(n, ib + B); ++i)
                    out[i + j * n] = st2(i, j) + x[i + j * n] - pax(i, j) - pax(j, i) + last(i, j);
    });
}

Mat bfgs_step(const Mat& x, const Mat& a, const Mat& s) {
    Mat out(x.r, x.c);
    bfgs_step_raw(x.r, s.c, x.data(), a.data(), s.data(), out.data());
    return out;
}

// run_inverter's symmetrization (simi.cpp:351-357): drift = ‖X − Xᵀ‖_F, X = (X + Xᵀ)/2, blocked.
double symmetrize_inplace(Index n, double* x) {
    const Index B = 64;
    const Index nb = (n + B - 1) / B;
    std::vector<double> part(static_cast<size_t>(nb), 0.0);
    parallel_for(long(nb), [&](long jbi) {
        const Index jb = Index(jbi) * B;
        double d = 0.0;
        for (Index ib = 0; ib <= jb; ib += B)
            for (Index j = jb; j < std::min(n, jb + B); ++j)
                for (Index i = ib; i < std::min(n, ib + B); ++i) {
                    if (i >= j) continue;
                    const double u = x[i + j * n], l = x[j + i * n];
                    d += 2.0 * (u - l) * (u - l);
                    const double v = 0.5 * (u + l);
                    x[i + j * n] = v;
                    x[j + i * n] = v;
                }
        part[size_t(jbi)] = d;
    });
    double drift = 0.0;
    for (double d : part) drift += d;
    return std::sqrt(drift);
}

// ------------------------------------------------------------ Jacobi -------
// proj/src/linalg.cpp:13-79 (cyclic Jacobi, <= 60 sweeps, ascending sort).
struct EigenDecomposition {
    std::vector<double> values;
    Mat vectors;
};

EigenDecomposition jacobi_eigendecomposition(const Mat& m) {
    if (m.r != m.c) throw std::invalid_argument("jacobi_eigendecomposition: matrix must be square");
    const Index n = m.r;
    Mat a(n, n);
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) a(i, j) = 0.5 * (m(i, j) + m(j, i));  // :19
    Mat q = Mat::identity(n);
    const double scale = std::max(a.norm(), 1e-300);  // :22
    const int max_sweeps = 60;
    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
        double off = 0.0;
        for (Index p = 0; p < n; ++p)
            for (Index r = p + 1; r < n; ++r) off += a(p, r) * a(p, r);
        if (std::sqrt(2.0 * off) <= 1e-15 * scale) break;  // :28
        for (Index p = 0; p < n - 1; ++p) {
            for (Index r = p + 1; r < n; ++r) {
                const double apq = a(p, r);
                if (std::abs(apq) <= 1e-300) continue;
                const double theta = (a(r, r) - a(p, p)) / (2.0 * apq);
                const double t = (theta >= 0.0) ? 1.0 / (theta + std::sqrt(1.0 + theta * theta))
                                                : 1.0 / (theta - std::sqrt(1.0 + theta * theta));
                const double c = 1.0 / std::sqrt(1.0 + t * t);
                const double s = t * c;
                for (Index k = 0; k < n; ++k) {
                    const double akp = a(k, p), akr = a(k, r);
                    a(k, p) = c * akp - s * akr;
                    a(k, r) = s * akp + c * akr;
                }
                for (Index k = 0; k < n; ++k) {
                    const double apk = a(p, k), ark = a(r, k);
                    a(p, k) = c * apk - s * ark;
                    a(r, k) = s * apk + c * ark;
                }
                for (Index k = 0; k < n; ++k) {
                    const double qkp = q(k, p), qkr = q(k, r);
                    q(k, p) = c * qkp - s * qkr;
                    q(k, r) = s * qkp + c * qkr;
                }
            }
        }
    }
    std::vector<Index> order(static_cast<size_t>(n));
    std::iota(order.begin(), order.end(), Index{0});
    std::vector<double> diag(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) diag[size_t(i)] = a(i, i);
    std::sort(order.begin(), order.end(), [&](Index i, Index j) { return diag[size_t(i)] < diag[size_t(j)]; });
    EigenDecomposition dec;
    dec.values.resize(static_cast<size_t>(n));
    dec.vectors = Mat(n, n);
    for (Index j = 0; j < n; ++j) {
        const Index o = order[size_t(j)];
        dec.values[size_t(j)] = diag[size_t(o)];
        for (Index i = 0; i < n; ++i) dec.vectors(i, j) = q(i, o);
    }
    return dec;
}

// proj/src/linalg.cpp:144-155
Mat sym_inv_sqrt(const Mat& m, double floor_rel = 1e-14) {
    const EigenDecomposition dec = jacobi_eigendecomposition(m);
    const Index n = m.r;
    double lam_max = 0.0;
    if (n) lam_max = *std::max_element(dec.values.begin(), dec.values.end());
    std::vector<double> inv_roots(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) {
        const double lam = dec.values[size_t(i)];
        if (lam <= floor_rel * lam_max || lam <= 0.0) throw NumericalError("sym_inv_sqrt: matrix is not positive definite");
        inv_roots[size_t(i)] = 1.0 / std::sqrt(lam);
    }
    Mat vd = dec.vectors;
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) vd(i, j) *= inv_roots[size_t(j)];
    return gemm(vd, false, dec.vectors, true);
}

// ------------------------------------------------------- adarbfgs ----------
// proj/src/adarbfgs.cpp:12-21
Mat adarbfgs_update_factor(const Mat& l, const Mat& a, const Mat& stilde) {
    const Mat s = mul(l, stilde);                            // :13
    const Mat as = mul(a, s);                                // :14
    const Mat gram = gemm(s, true, as, false);               // :15
    const Mat r = sym_inv_sqrt(gram);                        // :16
    const Mat g2 = gemm(stilde, true, stilde, false);        // :17
    const Mat term = gemm(sym_inv_sqrt(g2), false, stilde, true);  // :18
    const Mat asl = gemm(as, true, l, false);                // :19
    return l + mul(s, mul(r, term - mul(r, asl)));           // :20
}

// proj/src/adarbfgs.cpp:23-36
std::vector<double> adaptive_block_probabilities(const Mat& l, const Mat& a,
                                                 const std::vector<std::vector<Index>>& blocks) {
    const Mat al = mul(a, l);
    std::vector<double> p(blocks.size());
    const Index n = l.r;
    for (size_t i = 0; i < blocks.size(); ++i) {
        double trace = 0.0;
        for (Index j : blocks[i]) {
            double d = 0.0;
            for (Index k = 0; k < n; ++k) d += al(k, j) * l(k, j);
            trace += d;
        }
        p[i] = trace;
    }
    double mn = p.empty() ? 1.0 : *std::min_element(p.begin(), p.end());
    if (mn <= 0.0)
        throw NumericalError("adaptive_block_probabilities: non-positive block trace; the factor has degenerated");
    double sum = 0.0;
    for (double x : p) sum += x;
    for (double& x : p) x /= sum;
    return p;
}

// proj/src/sketching.cpp:106-115
std::vector<std::vector<Index>> contiguous_partition(Index n, Index q) {
    if (q < 1 || q > n) throw ConfigError("contiguous_partition: need 1 <= q <= n");
    std::vector<std::vector<Index>> blocks;
    for (Index start = 0; start < n; start += q) {
        std::vector<Index> block;
        for (Index i = start; i < std::min(start + q, n); ++i) block.push_back(i);
        blocks.push_back(std::move(block));
    }
    return blocks;
}

// Paper / BASELINE sampler (ref/"q distinct coordinate vectors
// selected uniformly at random"): NOT in the reference.  Builder
// definition: partial Fisher-Yates over RngStream::uniform_index (rng.hpp:38-40)
// -> indices perm[0..q).  Shared bit-for-bit with the product host sampler.
std::vector<Index> uniform_subset(RngStream& rng, Index n, Index q) {
    std::vector<Index> perm(static_cast<size_t>(n));
    std::iota(perm.begin(), perm.end(), Index{0});
    for (Index i = 0; i < q; ++i) {
        const Index j = i + rng.uniform_index(n - i);
        std::swap(perm[size_t(i)], perm[size_t(j)]);
    }
    perm.resize(size_t(q));
    return perm;
}

Mat coordinate_block_member(Index n, const std::vector<Index>& block) {  // adarbfgs.cpp:40-45
    Mat s(n, Index(block.size()));
    for (size_t j = 0; j < block.size(); ++j) s(block[j], Index(j)) = 1.0;
    return s;
}

// ------------------------------------------------------------ flops --------
double flops_bfgs(double n, double q) { return 10 * n * n * q + 10 * n * q * q + 2 * q * q * q + 4 * n * n; }  // flops.cpp:43-46
double flops_adarbfgs(double n, double q) {                                                                 // flops.cpp:70-74
    return 8 * n * n * q + 10 * n * q * q + 4 * q * q * q + n * q + n * n;
}

// ------------------------------------------------------------ drivers ------
struct HistoryPoint {
    long k;
    double residual, flops, seconds;
};
enum Termination { tol_reached = 0, max_iters = 1, error = 2 };

double residual_dense(const Mat& a, const Mat& x) {  // simi.cpp:242-244
    Mat ax = mul(a, x);
    const Index n = a.r;
    double s = 0.0;
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) {
            const double d = (i == j ? 1.0 : 0.0) - ax(i, j);
            s += d * d;
        }
    return std::sqrt(s);
}

// ------------------------------------------- other rank-q updates (row f3) --
// proj/src/qn_updates.cpp:121-129
Mat psb_step(const Mat& x, const Mat& a, const Mat& s) {
    const Mat as = mul(a, s);
    const Mat gram = gemm(as, true, as, false);                    // SᵀAAS
    const Mat t = gram_llt(gram, "psb_step").solve(as.t());        // q×n
    const Mat u = mul(x, as) - s;                                  // (XA − I)S
    const Mat mtheta = mul(u, t);
    const Mat c = gemm(as, true, u, false);                        // q×q
    return x - mtheta - mtheta.t() + gemm(t, true, mul(c, t), false);
}

// proj/src/qn_updates.cpp:147-152
Mat aip_step(const Mat& x, const Mat& a, const Mat& s) {
    const Mat as = mul(a, s);
    const Mat gram = gemm(s, true, as, false);                     // SᵀAS
    const Mat rhs = s.t() - gemm(as, true, x, false);              // Sᵀ − (AS)ᵀX
    return x + mul(s, gram_llt(gram, "aip_step").solve(rhs));
}

struct IteratePair {
    Mat primal, inverse;
};

// proj/src/qn_updates.cpp:154-174 (primal DFP update and the BFGS-form update of its inverse)
IteratePair dfp_step(const Mat& x, const Mat& x_inv, const Mat& a, const Mat& s) {
    const Mat as = mul(a, s);
    const Mat gram = gemm(s, true, as, false);
    const Llt llt = gram_llt(gram, "dfp_step");
    const Mat t1 = llt.solve(as.t());
    const Mat t2 = llt.solve(s.t());
    const Mat k = mul(t2, x);
    const Mat aox = mul(as, k);
    const Mat aoa = mul(as, t1);
    IteratePair next;
    next.primal = x + aoa - aox - aox.t() + mul(as, mul(gemm(k, false, t2, true), as.t()));
    const Mat hy = mul(x_inv, as);
    const Mat gram2 = gemm(as, true, hy, false);
    next.inverse = x_inv + mul(s, t2) - mul(hy, gram_llt(gram2, "dfp_step (inverse)").solve(hy.t()));
    return next;
}

// Eigen::PartialPivLU(m).inverse() (linalg.cpp:157-160): row-pivoted LU, then solve against I
Mat lu_inverse(const Mat& m) {
    const Index n = m.r;
    Mat lu = m;
    std::vector<Index> piv(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) piv[size_t(i)] = i;
    for (Index k = 0; k < n; ++k) {
        Index p = k;
        for (Index i = k + 1; i < n; ++i)
            if (std::fabs(lu(i, k)) > std::fabs(lu(p, k))) p = i;
        if (p != k) {
            for (Index j = 0; j < n; ++j) std::swap(lu(k, j), lu(p, j));
            std::swap(piv[size_t(k)], piv[size_t(p)]);
        }
        const double d = lu(k, k);
        for (Index i = k + 1; i < n; ++i) {
            lu(i, k) /= d;
            const double l = lu(i, k);
            for (Index j = k + 1; j < n; ++j) lu(i, j) -= l * lu(k, j);
        }
    }
    Mat inv(n, n);
    for (Index c = 0; c < n; ++c) {
        std::vector<double> y(static_cast<size_t>(n));
        for (Index i = 0; i < n; ++i) {
            double v = piv[size_t(i)] == c ? 1.0 : 0.0;
            for (Index j = 0; j < i; ++j) v -= lu(i, j) * y[size_t(j)];
            y[size_t(i)] = v;
        }
        for (Index i = n - 1; i >= 0; --i) {
            double v = y[size_t(i)];
            for (Index j = i + 1; j < n; ++j) v -= lu(i, j) * inv(j, c);
            inv(i, c) = v / lu(i, i);
        }
    }
    return inv;
}

// flops.cpp:22-25, 32-35, 37-41
double flops_psb(double n, double q) { return 8 * n * n * q + 8 * n * q * q + 2 * q * q * q + n * q + 3 * n * n; }
double flops_aip(double n, double q) { return 6 * n * n * q + 4 * n * q * q + 2 * q * q * q + n * q + n * n; }
double flops_dfp(double n, double q) { return 14 * n * n * q + 14 * n * q * q + 4 * q * q * q + 6 * n * n; }
double flops_newton_schulz(double n) { return 4 * n * n * n + 2 * n * n; }   // flops.cpp:76-79
double flops_minimal_residual(double n) { return 4 * n * n * n + 8 * n * n; }  // flops.cpp:81-85

// --------------------------------------------------- baselines (row f4) ------
// proj/src/baselines.cpp:12-14
Mat newton_schulz_step(const Mat& x, const Mat& a) { return 2.0 * x - mul(x, mul(a, x)); }

// proj/src/linalg.cpp:106-129 (power iteration on MᵀM from a seeded Gaussian start)
double spectral_norm_estimate(const Mat& m, int iters, uint64_t seed) {
    if (iters < 1) throw std::invalid_argument("spectral_norm_estimate: iters must be >= 1");
    if (m.v.empty() || m.norm() == 0.0) return 0.0;
    RngStream rng(seed);
    Mat v = rng.gaussian_matrix(m.c, 1);
    if (v.norm() == 0.0)
        for (double& e : v.v) e = 1.0;
    v = (1.0 / v.norm()) * v;
    double est = 0.0;
    for (int it = 0; it < iters; ++it) {
        const Mat w = mul(m, v);
        est = w.norm();
        if (est == 0.0) {
            v = rng.gaussian_matrix(m.c, 1);
            v = (1.0 / v.norm()) * v;
            continue;
        }
        v = gemm(m, true, w, false);
        const double nv = v.norm();
        if (nv == 0.0) break;
        for (double& e : v.v) e /= nv;
    }
    return est;
}

// proj/src/baselines.cpp:16-20
Mat newton_schulz_init(const Mat& a, uint64_t seed) {
    const double s = spectral_norm_estimate(a, 100, seed);
    if (s <= 0.0) throw ConfigError("newton_schulz_init: zero matrix");
    return (0.99 / (s * s)) * a.t();
}

struct MrStep {
    Mat x, r;
    double alpha = 0.0;
    bool stagnated = false;
};

// proj/src/baselines.cpp:22-37
MrStep mr_step_cached(const Mat& x, const Mat& r, const Mat& a) {
    MrStep out;
    const Mat xr = mul(x, r);
    const Mat axr = mul(a, xr);
    const double denom = axr.squared_norm();
    if (denom == 0.0) {
        out.x = x;
        out.r = r;
        out.stagnated = true;
        return out;
    }
    double num = 0.0;
    for (size_t i = 0; i < r.v.size(); ++i) num += r.v[i] * axr.v[i];
    out.alpha = num / denom;
    out.x = x + out.alpha * xr;
    out.r = r - out.alpha * axr;
    return out;
}

// proj/src/baselines.cpp:45-50
Mat mr_init(const Mat& a) {
    const double denom = gemm(a, false, a, true).v.empty() ? 0.0 : a.squared_norm();  // Tr(AAᵀ) = ‖A‖_F²
    if (denom == 0.0) throw ConfigError("mr_init: zero matrix");
    double tr = 0.0;
    for (Index i = 0; i < a.r; ++i) tr += a(i, i);
    return (tr / denom) * Mat::identity(a.r);
}

Mat identity_minus(const Mat& m) {
    Mat o = (-1.0) * m;
    for (Index i = 0; i < o.r; ++i) o(i, i) += 1.0;
    return o;
}

}  // namespace oracle

// =================================================================== C ABI ==
using namespace oracle;

namespace {
thread_local std::string g_err;
int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}
// status codes mirror the product C-ABI: 0 ok, 2 config, 3 numerical, 5 other
#define OR_GUARD(...)                                                    \
    try {                                                                \
        __VA_ARGS__;                                                        \
        return 0;                                                        \
    } catch (const GramRankDeficientError& e) { return fail(e, 3); }     \
    catch (const NumericalError& e) { return fail(e, 3); }               \
    catch (const ConfigError& e) { return fail(e, 2); }                  \
    catch (const std::invalid_argument& e) { return fail(e, 2); }        \
    catch (const std::exception& e) { return fail(e, 5); }

Mat wrap(const double* p, int64_t r, int64_t c) {
    Mat m(r, c);
    if (r > 0 && c > 0) std::memcpy(m.data(), p, sizeof(double) * size_t(r * c));
    return m;
}
void out(const Mat& m, double* p) {
    if (!m.v.empty()) std::memcpy(p, m.data(), sizeof(double) * m.v.size());
}
}  // namespace

// The reference (like this restatement) allocates several n×n temporaries per
// bfgs_step (qn_updates.cpp:183-185).  glibc serves blocks > 32 MB with fresh
// mmaps, so every call would page-fault gigabytes; as a CPU baseline we give the
// port a tuned allocator instead (heap reuse, no trimming).
__attribute__((constructor)) static void oracle_tune_malloc() {
    mallopt(M_MMAP_MAX, 0);
    mallopt(M_TRIM_THRESHOLD, 1 << 30);
}

extern "C" {

const char* or_last_error() { return g_err.c_str(); }
// host threads for the CPU baseline: n > 0 limits OpenBLAS and the elementwise passes, 0 = all
void or_set_threads(int n) {
    probe_blas();
    g_threads = n;
    if (g_blas_threads) g_blas_threads(n > 0 ? n : int(std::thread::hardware_concurrency()));
}
int or_have_blas() {
    probe_blas();
    return g_dgemm != nullptr;
}

// --- RngStream handle (rng.hpp) ---
void* or_rng_create(uint64_t seed) { return new RngStream(seed); }
void* or_rng_substream(void* h, uint64_t index) { return new RngStream(static_cast<RngStream*>(h)->substream(index)); }
void or_rng_destroy(void* h) { delete static_cast<RngStream*>(h); }
double or_rng_uniform(void* h) { return static_cast<RngStream*>(h)->uniform(); }
double or_rng_gaussian(void* h) { return static_cast<RngStream*>(h)->gaussian(); }
int64_t or_rng_categorical(void* h, const double* p, int64_t n) { return static_cast<RngStream*>(h)->categorical(p, n); }
int64_t or_rng_uniform_index(void* h, int64_t n) { return static_cast<RngStream*>(h)->uniform_index(n); }
void or_rng_gaussian_matrix(void* h, int64_t rows, int64_t cols, double* out_) {
    static_cast<RngStream*>(h)->gaussian_fill(out_, rows, cols);
}
void or_rng_uniform_matrix(void* h, int64_t rows, int64_t cols, double* out_) {
    static_cast<RngStream*>(h)->uniform_fill(out_, rows, cols);
}
void or_uniform_subset(void* h, int64_t n, int64_t q, int64_t* idx) {
    auto v = uniform_subset(*static_cast<RngStream*>(h), n, q);
    for (int64_t i = 0; i < q; ++i) idx[i] = v[size_t(i)];
}

// --- step kernels ---
int or_bfgs_step(int64_t n, int64_t q, const double* x, const double* a, const double* s, double* x_out) {
    OR_GUARD(bfgs_step_raw(n, q, x, a, s, x_out))
}
// in place: returns the drift ‖X − Xᵀ‖_F removed (simi.cpp:351-357)
double or_symmetrize(int64_t n, double* x) { return symmetrize_inplace(n, x); }
int or_adarbfgs_update_factor(int64_t n, int64_t q, const double* l, const double* a, const double* st, double* l_out) {
    OR_GUARD(out(adarbfgs_update_factor(wrap(l, n, n), wrap(a, n, n), wrap(st, n, q)), l_out))
}
int or_adaptive_block_probabilities(int64_t n, int64_t q, const double* l, const double* a, double* p_out) {
    OR_GUARD({
        auto blocks = contiguous_partition(n, q);
        auto p = adaptive_block_probabilities(wrap(l, n, n), wrap(a, n, n), blocks);
        std::copy(p.begin(), p.end(), p_out);
    })
}
int or_sym_inv_sqrt(int64_t n, const double* m, double* o) { OR_GUARD(out(sym_inv_sqrt(wrap(m, n, n)), o)) }
int or_jacobi(int64_t n, const double* m, double* values, double* vectors) {
    OR_GUARD({
        auto d = jacobi_eigendecomposition(wrap(m, n, n));
        std::copy(d.values.begin(), d.values.end(), values);
        out(d.vectors, vectors);
    })
}
int or_gemm(int64_t m, int64_t n, int64_t k, int ta, int tb, const double* a, const double* b, double* c) {
    OR_GUARD({
        Mat A = ta ? wrap(a, k, m) : wrap(a, m, k);
        Mat B = tb ? wrap(b, n, k) : wrap(b, k, n);
        out(gemm(A, ta, B, tb), c);
    })
}
double or_residual(int64_t n, const double* a, const double* x) { return residual_dense(wrap(a, n, n), wrap(x, n, n)); }
double or_flops_bfgs(int64_t n, int64_t q) { return flops_bfgs(double(n), double(q)); }
double or_flops_adarbfgs(int64_t n, int64_t q) { return flops_adarbfgs(double(n), double(q)); }

// --- run_inverter for the named bfgs method (simi.cpp:217-381) ---
// rule: 0 = gaussian(q) (sketching.cpp:30-36), 1 = coordinate_block(n,q) uniform p
// (sketching.cpp:20-28).  x0 may be NULL (identity).  Returns the termination in
// *term, history points into (hk, hres, hflops, hsec) up to hcap entries.
int or_run_inverter_bfgs(int64_t n, const double* a_in, int rule, int64_t q, double tol, int64_t max_iters_,
                         int64_t every_k, uint64_t seed, int max_redraws, const double* x0, double* x_out,
                         int* term, int64_t* k_out, int64_t* hk, double* hres, double* hflops, double* hsec,
                         int64_t hcap, int64_t* hcount, double* max_drift, int64_t* redraws_out) {
    OR_GUARD({
        if (tol < 0.0) throw ConfigError("run_inverter: tol must be >= 0");
        if (max_iters_ < 1) throw ConfigError("run_inverter: max_iters must be >= 1");
        if (max_redraws < 0) throw ConfigError("run_inverter: max_redraws must be >= 0");
        if (every_k < 1) throw ConfigError("run_inverter: residual_every_k must be >= 1");
        if (q < 1 || q > n) throw ConfigError("SketchRule: q must satisfy 1 <= q <= n");
        const Mat a = wrap(a_in, n, n);
        Mat x = x0 ? wrap(x0, n, n) : Mat::identity(n);
        std::vector<std::vector<Index>> blocks;
        std::vector<double> p;
        if (rule == 1) {
            blocks = contiguous_partition(n, q);
            p.assign(blocks.size(), 1.0 / double(blocks.size()));
        }
        int64_t hc = 0;
        double flops_total = 0.0, seconds = 0.0, drift_max = 0.0;
        int64_t redraws = 0;
        long k = 0;
        long kfinal = max_iters_;
        auto record = [&](double rel) {
            if (hc < hcap) {
                hk[hc] = k;
                hres[hc] = rel;
                hflops[hc] = flops_total;
                hsec[hc] = seconds;
            }
            ++hc;
        };
        const double base = residual_dense(a, x);  // :242-246
        *term = max_iters;
        bool done = false;
        if (base == 0.0) {
            record(0.0);
            *term = tol_reached;
            done = true;
        } else {
            record(1.0);
        }
        RngStream rng(seed);  // :275
        for (k = 1; !done && k <= max_iters_; ++k) {
            Mat next;
            bool stepped = false;
            for (int failures = 0; !stepped; ++failures) {  // :287
                if (failures > max_redraws) {
                    *term = error;
                    g_err = "sketch rejection limit exceeded";
                    done = true;
                    kfinal = k;
                    break;
                }
                Mat s;
                if (rule == 0) {
                    s = rng.gaussian_matrix(n, q);
                } else {
                    const Index i = rng.categorical(p.data(), Index(p.size()));
                    s = coordinate_block_member(n, blocks[size_t(i)]);
                }
                const auto start = std::chrono::steady_clock::now();
                try {
                    next = bfgs_step(x, a, s);
                } catch (const NumericalError&) {
                    ++redraws;
                    continue;
                }
                const auto stop = std::chrono::steady_clock::now();
                seconds += std::chrono::duration<double>(stop - start).count();
                flops_total += flops_bfgs(double(n), double(s.c));
                stepped = true;
            }
            if (done) break;
            if (!next.all_finite()) {  // :342-347
                *term = error;
                g_err = "diverged";
                kfinal = k;
                break;
            }
            x = std::move(next);
            // :351-357 symmetrize + drift
            drift_max = std::max(drift_max, symmetrize_inplace(n, x.data()));
            if (k == 1 || k == max_iters_ || k % every_k == 0) {  // :361-375
                const double rel = residual_dense(a, x) / base;
                record(rel);
                if (rel <= tol) {
                    *term = tol_reached;
                    done = true;
                    kfinal = k;
                    break;
                }
            }
        }
        *k_out = kfinal;
        *hcount = hc;
        *max_drift = drift_max;
        *redraws_out = redraws;
        out(x, x_out);
    })
}

// --- run_adarbfgs (adarbfgs.cpp:91-200) ---
// rule: 0 = adaptive_cols (contiguous blocks + Eq 8.2, adarbfgs.cpp:144-149),
//       1 = adaptive_gauss (rng.gaussian_matrix), 2 = paper uniform q-subset
//       (builder sampler, not in the reference; see uniform_subset).
int or_run_adarbfgs(int64_t n, const double* a_in, int rule, int64_t q, double tol, int64_t max_iters_,
                    int64_t every_k, uint64_t seed, int max_redraws, const double* l0, double* l_out, int* term,
                    int64_t* k_out, int64_t* hk, double* hres, double* hflops, double* hsec, int64_t hcap,
                    int64_t* hcount, int64_t* outcomes, int64_t outcap) {
    OR_GUARD({
        if (q < 1 || q > n) throw ConfigError("SketchRule: q must satisfy 1 <= q <= n");
        if (tol < 0.0) throw ConfigError("run_adarbfgs: tol must be >= 0");
        if (max_iters_ < 1) throw ConfigError("run_adarbfgs: max_iters must be >= 1");
        const Mat a = wrap(a_in, n, n);
        Mat l = l0 ? wrap(l0, n, n) : Mat::identity(n);
        std::vector<std::vector<Index>> blocks;
        if (rule == 0) blocks = contiguous_partition(n, q);
        int64_t hc = 0;
        double flops_total = 0.0, seconds = 0.0;
        long k = 0;
        long kfinal = max_iters_;
        auto record = [&](double rel) {
            if (hc < hcap) {
                hk[hc] = k;
                hres[hc] = rel;
                hflops[hc] = flops_total;
                hsec[hc] = seconds;
            }
            ++hc;
        };
        auto residual = [&]() {  // :112-115
            const Mat al = mul(a, l);
            const Mat x = gemm(al, false, l, true);
            double s = 0.0;
            for (Index j = 0; j < n; ++j)
                for (Index i = 0; i < n; ++i) {
                    const double d = (i == j ? 1.0 : 0.0) - x(i, j);
                    s += d * d;
                }
            return std::sqrt(s);
        };
        const double base = residual();
        *term = max_iters;
        bool done = false;
        if (base == 0.0) {
            record(0.0);
            *term = tol_reached;
            done = true;
        } else {
            record(1.0);
        }
        RngStream rng(seed);
        int64_t noutcome = 0;
        for (k = 1; !done && k <= max_iters_; ++k) {
            std::vector<double> p;
            Mat next_l;
            bool stepped = false;
            const auto start = std::chrono::steady_clock::now();
            if (rule == 0) p = adaptive_block_probabilities(l, a, blocks);
            for (int attempt = 0; attempt <= max_redraws && !stepped; ++attempt) {
                Mat stilde;
                if (rule == 0) {
                    const Index i = rng.categorical(p.data(), Index(p.size()));
                    if (noutcome < outcap) outcomes[noutcome] = i;
                    ++noutcome;
                    stilde = coordinate_block_member(n, blocks[size_t(i)]);
                } else if (rule == 1) {
                    stilde = rng.gaussian_matrix(n, q);
                } else {
                    auto idx = uniform_subset(rng, n, q);
                    for (Index j = 0; j < q; ++j) {
                        if (noutcome < outcap) outcomes[noutcome] = idx[size_t(j)];
                        ++noutcome;
                    }
                    stilde = coordinate_block_member(n, idx);
                }
                try {
                    next_l = adarbfgs_update_factor(l, a, stilde);
                    stepped = true;
                } catch (const NumericalError&) {
                }
            }
            const auto stop = std::chrono::steady_clock::now();
            if (!stepped) {
                *term = error;
                g_err = "sketch rejection limit exceeded";
                kfinal = k;
                break;
            }
            seconds += std::chrono::duration<double>(stop - start).count();
            flops_total += flops_adarbfgs(double(n), double(q));
            if (rule == 0) flops_total += 2.0 * double(n) * double(n) * double(n);
            if (!next_l.all_finite()) {
                *term = error;
                g_err = "diverged";
                kfinal = k;
                break;
            }
            l = std::move(next_l);
            if (k == 1 || k == max_iters_ || k % every_k == 0) {
                const double rel = residual() / base;
                record(rel);
                if (rel <= tol) {
                    *term = tol_reached;
                    kfinal = k;
                    break;
                }
            }
        }
        *k_out = kfinal;
        *hcount = hc;
        out(l, l_out);
    })
}

// --- row f3: psb / aip / dfp steps ---
int or_psb_step(int64_t n, int64_t q, const double* x, const double* a, const double* s, double* x_out) {
    OR_GUARD(out(psb_step(wrap(x, n, n), wrap(a, n, n), wrap(s, n, q)), x_out))
}
int or_aip_step(int64_t n, int64_t q, const double* x, const double* a, const double* s, double* x_out) {
    OR_GUARD(out(aip_step(wrap(x, n, n), wrap(a, n, n), wrap(s, n, q)), x_out))
}
int or_dfp_step(int64_t n, int64_t q, const double* x, const double* x_inv, const double* a, const double* s,
                double* x_out, double* x_inv_out) {
    OR_GUARD({
        const IteratePair p = dfp_step(wrap(x, n, n), wrap(x_inv, n, n), wrap(a, n, n), wrap(s, n, q));
        out(p.primal, x_out);
        out(p.inverse, x_inv_out);
    })
}
int or_lu_inverse(int64_t n, const double* m, double* o) { OR_GUARD(out(lu_inverse(wrap(m, n, n)), o)) }
double or_flops_named(int update, int64_t n, int64_t q) {
    const double nn = double(n), qq = double(q);
    switch (update) {
        case 0: return flops_bfgs(nn, qq);
        case 1: return flops_psb(nn, qq);
        case 2: return flops_aip(nn, qq);
        case 3: return flops_dfp(nn, qq);
    }
    return 0.0;
}

// --- row f4: Newton-Schulz / minimal residual ---
int or_newton_schulz_step(int64_t n, const double* x, const double* a, double* x_out) {
    OR_GUARD(out(newton_schulz_step(wrap(x, n, n), wrap(a, n, n)), x_out))
}
int or_newton_schulz_init(int64_t n, const double* a, uint64_t seed, double* x_out) {
    OR_GUARD(out(newton_schulz_init(wrap(a, n, n), seed), x_out))
}
int or_spectral_norm_estimate(int64_t r, int64_t c, const double* m, int iters, uint64_t seed, double* est) {
    OR_GUARD(*est = spectral_norm_estimate(wrap(m, r, c), iters, seed))
}
int or_mr_step_cached(int64_t n, const double* x, const double* r, const double* a, double* x_out, double* r_out,
                      double* alpha, int* stagnated) {
    OR_GUARD({
        const MrStep st = mr_step_cached(wrap(x, n, n), wrap(r, n, n), wrap(a, n, n));
        out(st.x, x_out);
        out(st.r, r_out);
        *alpha = st.alpha;
        *stagnated = st.stagnated ? 1 : 0;
    })
}
int or_mr_init(int64_t n, const double* a, double* x_out) { OR_GUARD(out(mr_init(wrap(a, n, n)), x_out)) }

// run_baseline (baselines.cpp:52-151); method 0 = newton-schulz, 1 = minimal residual.
int or_run_baseline(int64_t n, const double* a_in, int method, double tol, int64_t max_iters_, int64_t every_k,
                    uint64_t seed, const double* x0, double* x_out, int* term, int64_t* k_out, int64_t* hk,
                    double* hres, double* hflops, double* hsec, int64_t hcap, int64_t* hcount) {
    OR_GUARD({
        if (tol < 0.0) throw ConfigError("run_baseline: tol must be >= 0");
        if (max_iters_ < 1) throw ConfigError("run_baseline: max_iters must be >= 1");
        const bool ns = method == 0;
        const Mat a = wrap(a_in, n, n);
        Mat x = x0 ? wrap(x0, n, n) : (ns ? newton_schulz_init(a, seed) : mr_init(a));
        Mat r = identity_minus(mul(a, x));
        const double base = r.norm();
        int64_t hc = 0;
        double flops_total = 0.0, seconds = 0.0;
        long k = 0;
        auto record = [&](double rel) {
            if (hc < hcap) {
                hk[hc] = k;
                hres[hc] = rel;
                hflops[hc] = flops_total;
                hsec[hc] = seconds;
            }
            ++hc;
        };
        *term = max_iters;
        long kfinal = max_iters_;
        g_err.clear();
        if (base == 0.0) {
            record(0.0);
            *term = tol_reached;
            kfinal = 0;
        } else {
            record(1.0);
            for (k = 1; k <= max_iters_; ++k) {
                const auto start = std::chrono::steady_clock::now();
                bool stagnated = false;
                Mat next;
                if (ns) {
                    next = newton_schulz_step(x, a);
                } else {
                    MrStep st = mr_step_cached(x, r, a);
                    stagnated = st.stagnated;
                    next = std::move(st.x);
                    r = std::move(st.r);
                }
                seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
                flops_total += ns ? flops_newton_schulz(double(n)) : flops_minimal_residual(double(n));
                if (!next.all_finite()) {
                    *term = error;
                    g_err = "diverged: non-finite entries at iteration " + std::to_string(k);
                    kfinal = k;
                    break;
                }
                x = std::move(next);
                if (stagnated) {
                    const double rel = r.norm() / base;
                    record(rel);
                    *term = rel <= tol ? tol_reached : error;
                    if (*term == error)
                        g_err = "minimal residual stagnated (zero step denominator) at iteration " + std::to_string(k);
                    kfinal = k;
                    break;
                }
                if (k == 1 || k == max_iters_ || k % every_k == 0) {
                    r = identity_minus(mul(a, x));
                    const double rel = r.norm() / base;
                    record(rel);
                    if (!std::isfinite(rel)) {
                        *term = error;
                        g_err = "diverged: residual overflow at iteration " + std::to_string(k);
                        kfinal = k;
                        break;
                    }
                    if (rel <= tol) {
                        *term = tol_reached;
                        kfinal = k;
                        break;
                    }
                }
            }
        }
        *k_out = kfinal;
        *hcount = hc;
        out(x, x_out);
    })
}

// run_inverter for the named updates on the GPU path (simi.cpp:217-381):
// update 0 bfgs, 1 psb, 2 aip, 3 dfp.  rule 0 = gaussian(q), 1 = coordinate_block(n, q)
// with probabilities prob (0 uniform, 1 convenient: simi.cpp:121-150 per update).
// x_inv_out receives the tracked inverse for dfp (may be NULL otherwise).
int or_run_inverter(int update, int64_t n, const double* a_in, int rule, int prob, int64_t q, double tol,
                    int64_t max_iters_, int64_t every_k, uint64_t seed, int max_redraws, const double* x0,
                    double* x_out, double* x_inv_out, int* term, int64_t* k_out, int64_t* hk, double* hres,
                    double* hflops, double* hsec, int64_t hcap, int64_t* hcount, double* max_drift,
                    int64_t* redraws_out) {
    OR_GUARD({
        if (tol < 0.0) throw ConfigError("run_inverter: tol must be >= 0");
        if (max_iters_ < 1) throw ConfigError("run_inverter: max_iters must be >= 1");
        if (max_redraws < 0) throw ConfigError("run_inverter: max_redraws must be >= 0");
        if (every_k < 1) throw ConfigError("run_inverter: residual_every_k must be >= 1");
        if (q < 1 || q > n) throw ConfigError("SketchRule: q must satisfy 1 <= q <= n");
        const Mat a = wrap(a_in, n, n);
        const bool dfp = update == 3, symmetric = update != 2;
        Mat x = x0 ? wrap(x0, n, n) : Mat::identity(n);
        Mat x_inv = dfp ? (x0 ? lu_inverse(x) : Mat::identity(n)) : Mat();
        std::vector<std::vector<Index>> blocks;
        std::vector<double> p;
        if (rule == 1) {
            blocks = contiguous_partition(n, q);
            p.assign(blocks.size(), 1.0 / double(blocks.size()));
            if (prob == 1) {  // convenient (simi.cpp:121-150)
                std::vector<double> w(static_cast<size_t>(n));
                if (update == 0 || update == 2) {  // Tr(SᵢᵀASᵢ)
                    for (Index j = 0; j < n; ++j) w[size_t(j)] = a(j, j);
                } else if (update == 1) {  // ‖A Sᵢ‖_F² (col side, identity weight)
                    for (Index j = 0; j < n; ++j) {
                        double t = 0.0;
                        for (Index i = 0; i < n; ++i) t += a(i, j) * a(i, j);
                        w[size_t(j)] = t;
                    }
                } else {  // Tr(SᵢᵀA⁻¹Sᵢ)
                    const Llt llt(a);
                    const Mat ai = llt.solve(Mat::identity(n));
                    for (Index j = 0; j < n; ++j) w[size_t(j)] = ai(j, j);
                }
                double sum = 0.0;
                for (size_t i = 0; i < blocks.size(); ++i) {
                    double t = 0.0;
                    for (Index j : blocks[i]) t += w[size_t(j)];
                    if (!(t > 0.0))
                        throw ConfigError(update == 1 ? "convenient_probabilities: family member with zero sketched norm"
                                                      : "trace probabilities: member with non-positive sketched trace");
                    p[i] = t;
                    sum += t;
                }
                for (double& v : p) v /= sum;
            }
        }
        auto residual = [&]() { return residual_dense(a, dfp ? x_inv : x); };
        int64_t hc = 0;
        double flops_total = 0.0, seconds = 0.0, drift_max = 0.0;
        int64_t redraws = 0;
        long k = 0;
        long kfinal = max_iters_;
        auto record = [&](double rel) {
            if (hc < hcap) {
                hk[hc] = k;
                hres[hc] = rel;
                hflops[hc] = flops_total;
                hsec[hc] = seconds;
            }
            ++hc;
        };
        const double base = residual();
        *term = max_iters;
        bool done = false;
        g_err.clear();
        if (base == 0.0) {
            record(0.0);
            *term = tol_reached;
            done = true;
            kfinal = 0;
        } else {
            record(1.0);
        }
        RngStream rng(seed);
        for (k = 1; !done && k <= max_iters_; ++k) {
            Mat next, next_inv;
            bool stepped = false;
            for (int failures = 0; !stepped; ++failures) {
                if (failures > max_redraws) {
                    *term = error;
                    g_err = "sketch rejection limit exceeded";
                    done = true;
                    kfinal = k;
                    break;
                }
                Mat s;
                if (rule == 0) {
                    s = rng.gaussian_matrix(n, q);
                } else {
                    const Index i = rng.categorical(p.data(), Index(p.size()));
                    s = coordinate_block_member(n, blocks[size_t(i)]);
                }
                const auto start = std::chrono::steady_clock::now();
                try {
                    switch (update) {
                        case 0: next = bfgs_step(x, a, s); break;
                        case 1: next = psb_step(x, a, s); break;
                        case 2: next = aip_step(x, a, s); break;
                        default: {
                            IteratePair pr = dfp_step(x, x_inv, a, s);
                            next = std::move(pr.primal);
                            next_inv = std::move(pr.inverse);
                        }
                    }
                } catch (const NumericalError&) {
                    ++redraws;
                    continue;
                }
                seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
                flops_total += or_flops_named(update, n, s.c);
                stepped = true;
            }
            if (done) break;
            if (!next.all_finite() || (dfp && !next_inv.all_finite())) {
                *term = error;
                g_err = "diverged: non-finite entries at iteration " + std::to_string(k);
                kfinal = k;
                break;
            }
            x = std::move(next);
            if (dfp) x_inv = std::move(next_inv);
            if (symmetric) {
                drift_max = std::max(drift_max, symmetrize_inplace(n, x.data()));
                if (dfp) symmetrize_inplace(n, x_inv.data());
            }
            if (k == 1 || k == max_iters_ || k % every_k == 0) {
                const double rel = residual() / base;
                record(rel);
                if (rel <= tol) {
                    *term = tol_reached;
                    kfinal = k;
                    break;
                }
            }
        }
        *k_out = kfinal;
        *hcount = hc;
        *max_drift = drift_max;
        *redraws_out = redraws;
        out(x, x_out);
        if (dfp && x_inv_out) out(x_inv, x_inv_out);
    })
}

}  // extern "C"
