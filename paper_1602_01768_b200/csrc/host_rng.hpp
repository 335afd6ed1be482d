// Host-side sampling for the drop-in: the reference's seeded stream, kept on
// the host so coordinate indices and redraw RNG consumption are bit-exact with
// the reference.
//
// Restates proj/include/stochinv/rng.hpp:13-71 (splitmix64-seeded
// std::mt19937_64 + libstdc++ distributions; a fresh normal_distribution per
// gaussian_matrix call, column-major fill) and proj/src/sketching.cpp:106-115
// (contiguous_partition).  Compiled with the same -O3 -march=x86-64-v3 flags as
// the oracle so FMA contraction inside libstdc++'s polar method matches.
#pragma once
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <random>
#include <vector>

namespace si {

using Index = std::ptrdiff_t;

class RngStream {
public:
    explicit RngStream(std::uint64_t seed) : state_(mix(seed)), engine_(state_) {}
    RngStream substream(std::uint64_t index) const { return RngStream(state_ ^ (0x9e3779b97f4a7c15ULL * (index + 1))); }
    double uniform() { return std::uniform_real_distribution<double>(0.0, 1.0)(engine_); }
    double gaussian() { return std::normal_distribution<double>(0.0, 1.0)(engine_); }
    Index categorical(const double* p, Index n) {  // rng.hpp:28-36
        const double u = uniform();
        double acc = 0.0;
        for (Index i = 0; i < n; ++i) {
            acc += p[i];
            if (u < acc) return i;
        }
        return n - 1;
    }
    Index uniform_index(Index n) { return std::uniform_int_distribution<Index>(0, n - 1)(engine_); }
    void gaussian_fill(double* m, Index rows, Index cols, Index ld) {  // rng.hpp:42-49
        std::normal_distribution<double> dist(0.0, 1.0);
        for (Index j = 0; j < cols; ++j)
            for (Index i = 0; i < rows; ++i) m[i + j * ld] = dist(engine_);
    }
    void uniform_fill(double* m, Index rows, Index cols, Index ld) {  // rng.hpp:51-58
        std::uniform_real_distribution<double> dist(0.0, 1.0);
        for (Index j = 0; j < cols; ++j)
            for (Index i = 0; i < rows; ++i) m[i + j * ld] = dist(engine_);
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

// Paper / BASELINE sampler ("q distinct coordinate vectors selected uniformly at
// random", ref/PAPER.md:1179); absent from the reference, builder-defined as a
// partial Fisher-Yates over RngStream::uniform_index.
inline std::vector<Index> uniform_subset(RngStream& rng, Index n, Index q) {
    std::vector<Index> perm(static_cast<size_t>(n));
    std::iota(perm.begin(), perm.end(), Index{0});
    for (Index i = 0; i < q; ++i) {
        const Index j = i + rng.uniform_index(n - i);
        std::swap(perm[static_cast<size_t>(i)], perm[static_cast<size_t>(j)]);
    }
    perm.resize(static_cast<size_t>(q));
    return perm;
}

inline std::vector<std::vector<Index>> contiguous_partition(Index n, Index q) {
    std::vector<std::vector<Index>> blocks;
    for (Index start = 0; start < n; start += q) {
        std::vector<Index> block;
        for (Index i = start; i < std::min(start + q, n); ++i) block.push_back(i);
        blocks.push_back(std::move(block));
    }
    return blocks;
}

}  // namespace si
