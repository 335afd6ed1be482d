// Kernels of the sharded (multi-GPU) drivers (shard.cpp): row placement of
// all-gathered panels, block transposes for the residual's row exchange, the CSR row-panel
// residual, and the in-device collectives of the loopback communicator (the test harness
// that runs P virtual ranks on one GPU).  No GEMM here: the products go through engine.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "engine.hpp"

namespace si {

namespace {

// row i of a contiguous partition of n rows into `parts` near-equal parts (row_partition:
// the first n % parts parts one row longer) -> (part, offset in part)
__device__ __forceinline__ void part_of_row(int64_t i, int64_t n, int parts, int& p, int64_t& off) {
    const int64_t base = n / parts, extra = n % parts;
    const int64_t big = extra * (base + 1);
    if (i < big) {
        p = int(i / (base + 1));
        off = i - int64_t(p) * (base + 1);
    } else {
        const int64_t j = i - big;
        p = int(extra + j / base);
        off = j - (int64_t(p) - extra) * base;
    }
}

// Y (n×k, ld ldy) from an all-gathered buffer of `parts` slots, each slot a k×mc block
// (column-major, ld mc) holding its part's rows.  symmetric_chunks: parts = 2P chunks, chunk
// c sits in slot 2·owner + j with owner = c (j = 0) or 2P−1−c (j = 1) — the chunk pairs of
// the symmetric RBFGS distribution; otherwise part p sits in slot p.
__global__ void place_rows_kernel(const double* __restrict__ g, int64_t mc, int parts, int symmetric_chunks,
                                  int64_t n, int64_t k, double* __restrict__ Y, int64_t ldy) {
    const int64_t total = n * k;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % n, col = e / n;
        int p;
        int64_t off;
        part_of_row(i, n, parts, p, off);
        int slot = p;
        if (symmetric_chunks) {
            const int P = parts / 2;
            slot = p < P ? 2 * p : 2 * (2 * P - 1 - p) + 1;
        }
        Y[i + col * ldy] = g[(int64_t)slot * k * mc + col * mc + off];
    }
}

// dst (rows×cols block, ld ldd) = srcᵀ, src cols×rows (ld lds): 32×32 tiles through shared
// memory, coalesced on both sides
__global__ void transpose_block_kernel(const double* __restrict__ src, int64_t lds, int64_t rows, int64_t cols,
                                       double* __restrict__ dst, int64_t ldd) {
    __shared__ double t[32][33];
    const int64_t r0 = int64_t(blockIdx.x) * 32, c0 = int64_t(blockIdx.y) * 32;
    for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {  // t[a][b] = src(c0 + b, r0 + a)
        const int64_t sr = c0 + threadIdx.x, sc = r0 + yy;
        if (sr < cols && sc < rows) t[yy][threadIdx.x] = src[sr + sc * lds];
    }
    __syncthreads();
    for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {  // dst(r0 + x, c0 + yy) = src(c0 + yy, r0 + x)
        const int64_t rr = r0 + threadIdx.x, cc = c0 + yy;
        if (rr < rows && cc < cols) dst[rr + cc * ldd] = t[threadIdx.x][yy];
    }
}

// Σ_{k<n, i<m} (δ(k, r0+i) − (A·B)(k, i))² for CSR A (n rows, absolute rowptr) and a dense
// row-major B (n×m, row stride m) — B is a column-major m×n row panel X[R, :] read as its
// transpose, so A·B = (X[R, :]·A)ᵀ for symmetric A: the residual rows of a sharded X with
// no n×m product written.  One warp per row k of A, lanes over i.
__global__ void csr_resid_rows_kernel(int64_t n, const int64_t* __restrict__ rowptr,
                                      const int32_t* __restrict__ colind, const double* __restrict__ val,
                                      const double* __restrict__ B, int64_t m, int64_t r0, double* partial) {
    __shared__ double red[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double acc = 0.0;
    for (int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; k < n; k += warps) {
        const int64_t b = rowptr[k], e = rowptr[k + 1];
        for (int64_t i = lane; i < m; i += 32) {
            double s = 0.0;
            for (int64_t t = b; t < e; ++t) s = fma(val[t], B[(int64_t)colind[t] * m + i], s);
            const double d = (k == r0 + i ? 1.0 : 0.0) - s;
            acc = fma(d, d, acc);
        }
    }
    acc = warp_sum(acc);
    if (lane == 0) red[wid] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
        partial[blockIdx.x] = t;
    }
}

__global__ void sum_partials_kernel(const double* __restrict__ part, int count, double* out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < count; i += blockDim.x) s += part[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
        *out = t;
    }
}

__global__ void accumulate_kernel(double* __restrict__ dst, const double* __restrict__ src, int64_t count) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
        dst[e] += src[e];
}

__global__ void identity_rows_kernel(double* X, int64_t m, int64_t cols, int64_t diag_off) {
    const int64_t total = m * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % m, j = e / m;
        X[e] = (j == i + diag_off) ? 1.0 : 0.0;
    }
}

template <typename T>
__global__ void combine_kernel(T* __restrict__ dst, const T* __restrict__ src, int64_t count, int is_max) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
        dst[e] = is_max ? (src[e] > dst[e] ? src[e] : dst[e]) : T(dst[e] + src[e]);
}

// d_j = Σ_i AL(i, j)·L(i, j) over an m×n row panel (ld m): one warp per column
__global__ void panel_column_dots_kernel(const double* __restrict__ AL, const double* __restrict__ L, int64_t m,
                                         int64_t n, double* __restrict__ d) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < n; j += warps) {
        double s = 0.0;
        for (int64_t i = lane; i < m; i += 32) s = fma(AL[i + j * m], L[i + j * m], s);
        s = warp_sum(s);
        if (lane == 0) d[j] = s;
    }
}

// Ĝ = G − H' with G read from its upper triangle and H' symmetrised (ghat_kernel's formula,
// kernels_aux.cuh) when G and H' sit in separate buffers (ld q)
__global__ void ghat_split_kernel(const double* __restrict__ G, const double* __restrict__ H, int q,
                                  double* __restrict__ gh, const int* skip) {
    if (skip && *skip) return;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < q * q; idx += gridDim.x * blockDim.x) {
        const int i = idx % q, j = idx / q;
        const double g = i <= j ? G[i + (int64_t)j * q] : G[j + (int64_t)i * q];
        const double h = 0.5 * (H[i + (int64_t)j * q] + H[j + (int64_t)i * q]);
        gh[idx] = g - h;
    }
}

int blocks_for(int64_t work) { return int(std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 8))); }

}  // namespace

void place_rows(Context& c, const double* g, int64_t mc, int parts, bool symmetric_chunks, int64_t n, int64_t k,
                double* Y, int64_t ldy) {
    LaunchScope ls(c, "place_rows");
    place_rows_kernel<<<blocks_for(n * k), 256, 0, c.stream>>>(g, mc, parts, symmetric_chunks ? 1 : 0, n, k, Y, ldy);
    cuda_check(cudaGetLastError(), "place_rows");
}

void transpose_block(Context& c, const double* src, int64_t lds, int64_t rows, int64_t cols, double* dst,
                     int64_t ldd) {
    if (rows <= 0 || cols <= 0) return;
    LaunchScope ls(c, "transpose_block");
    dim3 grid(unsigned((rows + 31) / 32), unsigned((cols + 31) / 32));
    transpose_block_kernel<<<grid, dim3(32, 8), 0, c.stream>>>(src, lds, rows, cols, dst, ldd);
    cuda_check(cudaGetLastError(), "transpose_block");
}

void csr_residual_rows_sq(Context& c, Problem& a, int64_t m, int64_t r0, const double* Xrows, double* out_dev) {
    const int blocks = c.num_sms * 4;
    double* part = c.ensure_ws(size_t(blocks));
    {
        LaunchScope ls(c, "csr_resid_rows");
        csr_resid_rows_kernel<<<blocks, 256, 0, c.stream>>>(a.n, a.rowptr, a.colind, a.val, Xrows, m, r0, part);
        cuda_check(cudaGetLastError(), "csr_resid_rows");
    }
    LaunchScope ls(c, "sum_reduce");
    sum_partials_kernel<<<1, 1024, 0, c.stream>>>(part, blocks, out_dev);
    cuda_check(cudaGetLastError(), "sum_partials");
}

void accumulate(Context& c, double* dst, const double* src, int64_t count) {
    LaunchScope ls(c, "loopback_sum");
    accumulate_kernel<<<blocks_for(count), 256, 0, c.stream>>>(dst, src, count);
    cuda_check(cudaGetLastError(), "accumulate");
}

void combine(Context& c, void* dst, const void* src, int64_t count, bool is_int, bool is_max) {
    LaunchScope ls(c, "loopback_reduce");
    if (is_int)
        combine_kernel<int><<<blocks_for(count), 256, 0, c.stream>>>(static_cast<int*>(dst), static_cast<const int*>(src),
                                                                     count, is_max ? 1 : 0);
    else
        combine_kernel<double><<<blocks_for(count), 256, 0, c.stream>>>(
            static_cast<double*>(dst), static_cast<const double*>(src), count, is_max ? 1 : 0);
    cuda_check(cudaGetLastError(), "combine");
}

void panel_column_dots(Context& c, const double* AL, const double* L, int64_t m, int64_t n, double* d) {
    LaunchScope ls(c, "column_dots");
    panel_column_dots_kernel<<<blocks_for(n * 32), 256, 0, c.stream>>>(AL, L, m, n, d);
    cuda_check(cudaGetLastError(), "panel_column_dots");
}

void ghat_split(Context& c, const double* G, const double* H, int64_t q, double* Ghat, const int* skip) {
    LaunchScope ls(c, "ghat");
    ghat_split_kernel<<<blocks_for(q * q), 256, 0, c.stream>>>(G, H, int(q), Ghat, skip);
    cuda_check(cudaGetLastError(), "ghat_split");
}

void set_identity_rows(Context& c, double* X, int64_t m, int64_t cols, int64_t diag_off) {
    LaunchScope ls(c, "set_identity");
    identity_rows_kernel<<<blocks_for(m * cols), 256, 0, c.stream>>>(X, m, cols, diag_off);
    cuda_check(cudaGetLastError(), "identity_rows");
}

}  // namespace si
