// Problem ingestion: the reference's readers and synthetic
// generator, with sparse inputs kept sparse and the Gram products on the GPU.
//
//   load_matrix_market  proj/src/io.cpp:28-121 — the same header checks, the
//                       same IoError texts with "path:line:" prefixes, the same
//                       duplicate rule (a later coordinate entry overwrites an
//                       earlier one, as the reference's dense m(i,j) = v does)
//                       and symmetric mirroring; coordinate files become CSR
//                       instead of being densified (io.cpp:72).
//   build_ridge_hessian proj/src/io.cpp:123-166 — A = Σ x xᵀ + λI from LIBSVM
//                       rows, formed as BᵀB + λI by the DMMA GEMM engine.
//   gen_synthetic       proj/src/io.cpp:168-176 — A = ĀᵀĀ with Ā uniform from
//                       RngStream(seed) (host draws, device product).
//
// The parser is a small cursor over the file (MmCursor) that owns the line
// number, so every diagnostic carries the line it was raised on.
#include <cuda_runtime.h>

#include <algorithm>
#include <cctype>
#include <cstdlib>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/stochinv_b200.h"
#include "engine.hpp"
#include "host_rng.hpp"

namespace si {

namespace {

struct MmCursor {
    std::string path;
    std::ifstream in;
    long line_no = 0;
    std::string line;

    explicit MmCursor(const std::string& p) : path(p), in(p) {
        if (!in) throw IoError("cannot open " + path);
    }
    [[noreturn]] void fail(const std::string& what) const {
        throw IoError(path + ":" + std::to_string(line_no) + ": " + what);
    }
    bool next() {  // any line
        if (!std::getline(in, line)) return false;
        ++line_no;
        return true;
    }
    bool next_data() {  // skips blank lines and '%' comments
        while (next())
            if (!line.empty() && line[0] != '%') return true;
        return false;
    }
};

std::string folded(std::string s) {
    for (char& ch : s) ch = char(std::tolower(static_cast<unsigned char>(ch)));
    return s;
}

struct MmBanner {
    bool coordinate = false, symmetric = false;
};

MmBanner read_banner(MmCursor& cur) {
    if (!cur.next()) throw IoError(cur.path + ": empty file");
    std::istringstream words(cur.line);
    std::string tag, obj, fmt, fld, sym;
    words >> tag >> obj >> fmt >> fld >> sym;
    obj = folded(obj), fmt = folded(fmt), fld = folded(fld), sym = folded(sym);
    if (tag != "%%MatrixMarket") cur.fail("missing %%MatrixMarket banner");
    if (obj != "matrix") cur.fail("unsupported object '" + obj + "'");
    if (fmt != "coordinate" && fmt != "array") cur.fail("unsupported format '" + fmt + "'");
    if (fld != "real" && fld != "integer") cur.fail("unsupported field '" + fld + "' (real values required)");
    if (sym != "general" && sym != "symmetric") cur.fail("unsupported symmetry '" + sym + "'");
    return MmBanner{fmt == "coordinate", sym == "symmetric"};
}

// (row, col) -> value for a coordinate body; ordered row-major so CSR fills in order
using EntryMap = std::map<std::pair<int64_t, int64_t>, double>;

EntryMap read_coordinate_body(MmCursor& cur, long dim, long count, bool mirror) {
    EntryMap cells;
    long got = 0;
    while (got < count && cur.next()) {
        if (cur.line.empty() || cur.line[0] == '%') continue;
        std::istringstream rec(cur.line);
        long r = 0, c = 0;
        double v = 0.0;
        if (!(rec >> r >> c >> v)) cur.fail("malformed coordinate entry");
        if (r < 1 || c < 1 || r > dim || c > dim) cur.fail("index out of range");
        cells[{r - 1, c - 1}] = v;
        if (mirror) cells[{c - 1, r - 1}] = v;
        ++got;
    }
    if (got < count)
        throw IoError(cur.path + ": truncated file, expected " + std::to_string(count) + " entries, got " +
                      std::to_string(got));
    return cells;
}

// array body: column-major values; the symmetric variant lists the lower
// triangle of each column (io.cpp:88-119)
void read_array_body(MmCursor& cur, int64_t n, bool lower_only, std::vector<double>& dense) {
    const long want = lower_only ? long(n) * (long(n) + 1) / 2 : long(n) * long(n);
    long got = 0;
    int64_t row = 0, col = 0;
    while (got < want && cur.next()) {
        if (cur.line.empty() || cur.line[0] == '%') continue;
        std::istringstream vals(cur.line);
        for (double v; vals >> v;) {
            if (got >= want) cur.fail("surplus array entry");
            dense[size_t(row + col * n)] = v;
            if (lower_only) dense[size_t(col + row * n)] = v;
            ++got;
            if (++row == n) row = lower_only ? ++col : (++col, 0);
        }
        if (!vals.eof()) cur.fail("malformed array entry");
    }
    if (got < want)
        throw IoError(cur.path + ": truncated file, expected " + std::to_string(want) + " entries, got " +
                      std::to_string(got));
}

}  // namespace

LoadedMatrix load_matrix_market(const std::string& path, bool keep_sparse) {
    MmCursor cur(path);
    const MmBanner banner = read_banner(cur);
    if (!cur.next_data() && cur.line.empty()) throw IoError(path + ": missing size line");
    std::istringstream dims(cur.line);
    long rows = 0, cols = 0, count = 0;
    if (banner.coordinate ? !(dims >> rows >> cols >> count) : !(dims >> rows >> cols))
        cur.fail(banner.coordinate ? "malformed coordinate size line" : "malformed array size line");
    if (rows != cols) cur.fail("matrix must be square");
    if (rows < 1) cur.fail("empty matrix");

    LoadedMatrix out;
    out.n = rows;
    out.symmetric = banner.symmetric;
    const size_t nn = size_t(rows) * size_t(rows);
    if (!banner.coordinate) {
        out.dense.assign(nn, 0.0);
        read_array_body(cur, out.n, banner.symmetric, out.dense);
        return out;
    }
    const EntryMap cells = read_coordinate_body(cur, rows, count, banner.symmetric);
    if (!keep_sparse) {
        out.dense.assign(nn, 0.0);
        for (const auto& kv : cells) out.dense[size_t(kv.first.first + kv.first.second * out.n)] = kv.second;
        return out;
    }
    out.sparse = true;
    out.rowptr.assign(size_t(out.n) + 1, 0);
    out.colind.reserve(cells.size());
    out.val.reserve(cells.size());
    for (const auto& kv : cells) {
        ++out.rowptr[size_t(kv.first.first) + 1];
        out.colind.push_back(int32_t(kv.first.second));
        out.val.push_back(kv.second);
    }
    for (size_t i = 1; i < out.rowptr.size(); ++i) out.rowptr[i] += out.rowptr[i - 1];
    return out;
}

// LIBSVM rows "label idx:val idx:val ..." (io.cpp:128-160): 1-based indices,
// '#' comment lines, n = largest index seen.
LibsvmRows read_libsvm(const std::string& path) {
    MmCursor cur(path);
    LibsvmRows r;
    while (cur.next()) {
        if (cur.line.empty() || cur.line[0] == '#') continue;
        std::istringstream toks(cur.line);
        std::string tok;
        if (!(toks >> tok)) continue;  // the label (unused by the Hessian)
        std::vector<std::pair<int64_t, double>> feats;
        while (toks >> tok) {
            const auto colon = tok.find(':');
            if (colon == std::string::npos) cur.fail("malformed feature token '" + tok + "'");
            const std::string key = tok.substr(0, colon), val = tok.substr(colon + 1);
            char* end_k = nullptr;
            char* end_v = nullptr;
            const long long idx = std::strtoll(key.c_str(), &end_k, 10);
            const double v = std::strtod(val.c_str(), &end_v);
            if (key.empty() || val.empty() || end_k == key.c_str() || end_v == val.c_str())
                cur.fail("malformed feature token '" + tok + "'");
            if (idx < 1) cur.fail("feature indices are 1-based");
            r.n = std::max<int64_t>(r.n, idx);
            feats.emplace_back(int64_t(idx) - 1, v);
        }
        r.samples.push_back(std::move(feats));
    }
    if (r.n == 0) throw IoError(path + ": no features found (n = 0)");
    r.m = int64_t(r.samples.size());
    return r;
}

// A = lambda·I + Σ_samples x xᵀ = lambda·I + BᵀB, B (m×n) densified on the host
// in row chunks, the product accumulated by the DMMA engine.  Duplicate
// feature indices in one row are summed into B, which gives the same Σ vi·vj
// over all pairs as the reference's double loop.  Returns a device pointer.
double* ridge_hessian_device(Context& c, const LibsvmRows& r, double lambda) {
    const int64_t n = r.n;
    double* A = nullptr;
    cuda_check(cudaMalloc(&A, size_t(n) * size_t(n) * sizeof(double)), "malloc A");
    {
        std::vector<double> diag(size_t(n) * size_t(n), 0.0);
        for (int64_t i = 0; i < n; ++i) diag[size_t(i + i * n)] = lambda;
        cuda_check(cudaMemcpyAsync(A, diag.data(), diag.size() * sizeof(double), cudaMemcpyHostToDevice, c.stream),
                   "h2d");
        cuda_check(cudaStreamSynchronize(c.stream), "sync");
    }
    const int64_t chunk = std::max<int64_t>(64, std::min<int64_t>(r.m, (int64_t(1) << 27) / std::max<int64_t>(n, 1)));
    std::vector<double> hb;
    double* B = nullptr;
    cuda_check(cudaMalloc(&B, size_t(chunk) * size_t(n) * sizeof(double)), "malloc B");
    for (int64_t r0 = 0; r0 < r.m; r0 += chunk) {
        const int64_t mc = std::min(chunk, r.m - r0);
        hb.assign(size_t(mc) * size_t(n), 0.0);
        for (int64_t s = 0; s < mc; ++s)
            for (const auto& [j, v] : r.samples[size_t(r0 + s)]) hb[size_t(s + j * mc)] += v;
        cuda_check(cudaMemcpyAsync(B, hb.data(), hb.size() * sizeof(double), cudaMemcpyHostToDevice, c.stream), "h2d");
        gemm(c, n, n, mc, B, mc, true, B, mc, true, A, n, 1.0, 1.0);  // A += Bᵀ·B
        cuda_check(cudaStreamSynchronize(c.stream), "sync");
    }
    cudaFree(B);
    return A;
}

// A = ĀᵀĀ, Ā = RngStream(seed).uniform_matrix(n, n) (io.cpp:168-176)
double* synthetic_device(Context& c, int64_t n, uint64_t seed) {
    std::vector<double> abar(size_t(n) * size_t(n));
    RngStream rng(seed);
    rng.uniform_fill(abar.data(), n, n, n);
    double *Ab = nullptr, *A = nullptr;
    cuda_check(cudaMalloc(&Ab, abar.size() * sizeof(double)), "malloc");
    cuda_check(cudaMalloc(&A, abar.size() * sizeof(double)), "malloc");
    cuda_check(cudaMemcpyAsync(Ab, abar.data(), abar.size() * sizeof(double), cudaMemcpyHostToDevice, c.stream), "h2d");
    gemm(c, n, n, n, Ab, n, true, Ab, n, true, A, n, 1.0, 0.0);  // ĀᵀĀ
    cuda_check(cudaStreamSynchronize(c.stream), "sync");
    cudaFree(Ab);
    return A;
}

}  // namespace si
