// q×q kernels of the AdaRBFGS factor update and sparse/elementwise helpers.
//   - K-ISQRT: symmetric inverse square root R = G^{-1/2} by cyclic Jacobi in a
//     parallel (round-robin tournament) ordering inside one CTA.  Same stopping
//     rule (off-norm ≤ 1e-15‖G‖_F, ≤ 60 sweeps), same eigenvalue floor
//     (λ ≤ 1e-14 λ_max or λ ≤ 0 → resample) as linalg.cpp:13-79,144-155; the
//     symmetric root is unique, so R matches the reference's to rounding.
//   - K-SPMM: Y = A·P for CSR A (warp per row, vectorised row-major P).
//   - column dots for diag(LᵀAL) (Eq 8.2, adarbfgs.cpp:23-36).
#pragma once
#include "common.cuh"

namespace si {

// The reference's sym_inv_sqrt (linalg.cpp:144-155) in one CTA: cyclic Jacobi
// (linalg.cpp:13-79: A = (G + Gᵀ)/2, off-norm stop ≤ 1e-15‖A‖_F, ≤ 60 sweeps) with the
// rotations of a round-robin tournament applied in parallel, then the floor test
// "λ ≤ floor_rel·λ_max or λ ≤ 0" → *status = 1 (NumericalError → redraw), else
// R = Q·diag(λ^{-1/2})·Qᵀ (ld ldr).  `base` holds 2q² + 2(q/2 + 1) doubles + q + 2 ints
// (shared or global memory); every thread of the block must call it.
__device__ __noinline__ void jacobi_isqrt_block(const double* __restrict__ Gm, int64_t ldg, int q, double* base,
                                                double* __restrict__ R, int64_t ldr, int* status, double floor_rel) {
    const int qe = q + (q & 1);  // even count for the tournament (index q is a bye when q is odd)
    const int half = qe / 2;
    double* a = base;                       // q×q
    double* Q = base + (size_t)q * q;       // q×q
    double* cs = Q + (size_t)q * q;         // half
    double* sn = cs + half;                 // half
    int* pp = reinterpret_cast<int*>(sn + half);  // half
    int* rr = pp + half;                          // half
    __shared__ double red[32];
    __shared__ double s_scale, s_off;
    __shared__ int s_fail;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;

    for (int idx = tid; idx < q * q; idx += nt) {
        const int i = idx % q, j = idx / q;
        a[idx] = 0.5 * (Gm[i + (int64_t)j * ldg] + Gm[j + (int64_t)i * ldg]);  // linalg.cpp:19
        Q[idx] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    auto block_sum = [&](double v) -> double {  // result valid in thread 0
        v = warp_sum(v);
        __syncthreads();
        if (lane == 0) red[wid] = v;
        __syncthreads();
        double t = 0.0;
        if (tid == 0) {
            for (int w = 0; w < (nt >> 5); ++w) t += red[w];
        }
        return t;
    };
    {
        double v = 0.0;
        for (int idx = tid; idx < q * q; idx += nt) v += a[idx] * a[idx];
        const double t = block_sum(v);
        if (tid == 0) s_scale = fmax(sqrt(t), 1e-300);  // linalg.cpp:22
        __syncthreads();
    }
    const double scale = s_scale;
    for (int sweep = 0; sweep < 60; ++sweep) {
        double v = 0.0;
        for (int idx = tid; idx < q * q; idx += nt) {
            const int i = idx % q, j = idx / q;
            if (i < j) v += a[idx] * a[idx];
        }
        const double t = block_sum(v);
        if (tid == 0) s_off = t;
        __syncthreads();
        if (sqrt(2.0 * s_off) <= 1e-15 * scale) break;  // linalg.cpp:28
        for (int round = 0; round < qe - 1; ++round) {
            // tournament pairing: slot 0 fixed, others rotate
            for (int k = tid; k < half; k += nt) {
                auto slot = [&](int s) { return s == 0 ? 0 : ((s - 1 + round) % (qe - 1)) + 1; };
                int p = slot(k), r = slot(qe - 1 - k);
                if (p > r) {
                    const int tmp = p;
                    p = r;
                    r = tmp;
                }
                double c = 1.0, s = 0.0;
                if (r < q) {
                    const double apq = a[p + r * q];
                    if (fabs(apq) > 1e-300) {  // linalg.cpp:32-37
                        const double theta = (a[r + r * q] - a[p + p * q]) / (2.0 * apq);
                        const double tt = (theta >= 0.0) ? 1.0 / (theta + sqrt(1.0 + theta * theta))
                                                         : 1.0 / (theta - sqrt(1.0 + theta * theta));
                        c = 1.0 / sqrt(1.0 + tt * tt);
                        s = tt * c;
                    }
                }
                pp[k] = p;
                rr[k] = r;
                cs[k] = c;
                sn[k] = s;
            }
            __syncthreads();
            // A <- A J and Q <- Q J (column rotations)
            for (int w = tid; w < half * q * 2; w += nt) {
                const int which = w / (half * q);  // 0: a, 1: Q
                const int rem = w % (half * q);
                const int k = rem / q, row = rem % q;
                const int p = pp[k], r = rr[k];
                if (r >= q || sn[k] == 0.0) continue;
                double* m = which ? Q : a;
                const double c = cs[k], s = sn[k];
                const double xp = m[row + p * q], xr = m[row + r * q];
                m[row + p * q] = c * xp - s * xr;
                m[row + r * q] = s * xp + c * xr;
            }
            __syncthreads();
            // A <- Jᵀ A (row rotations)
            for (int w = tid; w < half * q; w += nt) {
                const int k = w / q, col = w % q;
                const int p = pp[k], r = rr[k];
                if (r >= q || sn[k] == 0.0) continue;
                const double c = cs[k], s = sn[k];
                const double xp = a[p + col * q], xr = a[r + col * q];
                a[p + col * q] = c * xp - s * xr;
                a[r + col * q] = s * xp + c * xr;
            }
            __syncthreads();
        }
    }
    // eigenvalue floor (linalg.cpp:146-152): λ ≤ floor_rel·λ_max or λ ≤ 0 → NumericalError
    if (tid == 0) {
        double lmax = -1e308;
        for (int i = 0; i < q; ++i) lmax = fmax(lmax, a[i + i * q]);
        int fail = 0;
        for (int i = 0; i < q; ++i) {
            const double lam = a[i + i * q];
            if (lam <= floor_rel * lmax || lam <= 0.0) fail = 1;
        }
        s_fail = fail;
    }
    __syncthreads();
    if (s_fail) {
        if (tid == 0) *status = 1;
        return;
    }
    // Q ← Q·diag(λ^{-1/4}) in place, then R = Q·Qᵀ (linalg.cpp:154; same root to rounding)
    for (int idx = tid; idx < q * q; idx += nt) {
        const int j = idx / q;
        Q[idx] *= 1.0 / sqrt(sqrt(a[j + j * q]));
    }
    __syncthreads();
    for (int idx = tid; idx < q * q; idx += nt) {
        const int i = idx % q, j = idx / q;
        if (i > j) continue;
        double acc = 0.0;
        for (int k = 0; k < q; ++k) acc = fma(Q[i + k * q], Q[j + k * q], acc);
        R[i + (int64_t)j * ldr] = acc;
        R[j + (int64_t)i * ldr] = acc;
    }
}

constexpr double ISQRT_FLOOR = 1e-14;        // linalg.hpp sym_inv_sqrt default floor_rel
constexpr double ISQRT_FAST_ACCEPT = 1e-12;  // certified λmin/λmax above which Newton–Schulz's R is kept

// Stand-alone exact inverse square root (q×q, global work): runs when `need` is set
// (need == nullptr: always), clears it.  The fallback of the multi-kernel Newton–Schulz.
__global__ void __launch_bounds__(1024) jacobi_isqrt_kernel(const double* __restrict__ Gm, int64_t ldg, int q,
                                                            double* work, double* __restrict__ R, int* status,
                                                            int* need) {
    if (*status) return;
    if (need) {
        if (!*need) return;
        __syncthreads();
        if (threadIdx.x == 0) *need = 0;
    }
    jacobi_isqrt_block(Gm, ldg, q, work, R, q, status, ISQRT_FLOOR);
}

// Y(i,:) = sum_c A(i,c) P(c,:) for CSR A; P and Y column-major (ld n).  One warp
// per row; lanes stride over the k columns.  P is read through the read-only
// path; for k >= 32 the loads of one nonzero are 32 distinct columns.
__global__ void spmm_csr_kernel(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
                                const double* __restrict__ val, const double* __restrict__ P, int64_t ldp, int64_t k,
                                double* __restrict__ Y, int64_t ldy, const int* skip) {
    if (skip && *skip) return;
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < n; row += warps) {
        const int64_t b = rowptr[row], e = rowptr[row + 1];
        for (int64_t c0 = 0; c0 < k; c0 += 32) {
            const int64_t col = c0 + lane;
            double acc = 0.0;
            if (col < k) {
                for (int64_t t = b; t < e; ++t) acc += __ldg(val + t) * __ldg(P + colind[t] + col * ldp);
                Y[row + col * ldy] = acc;
            }
        }
    }
}

// Row-major SpMM: Yr(i,:) = sum_c A(i,c) Pr(c,:) with Pr, Yr row-major (ld = k).
// Coalesced: the warp reads one contiguous k-row of Pr per nonzero.
__global__ void spmm_csr_rowmajor_kernel(int64_t n, const int64_t* __restrict__ rowptr,
                                         const int32_t* __restrict__ colind, const double* __restrict__ val,
                                         const double* __restrict__ Pr, int64_t k, double* __restrict__ Y,
                                         int64_t ldy, const int* skip) {
    if (skip && *skip) return;
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < n; row += warps) {
        const int64_t b = rowptr[row], e = rowptr[row + 1];
        for (int64_t c0 = 0; c0 < k; c0 += 64) {
            const int64_t col = c0 + 2 * lane;
            double2 acc = make_double2(0.0, 0.0);
            if (col + 1 < k) {
                for (int64_t t = b; t < e; ++t) {
                    const double v = __ldg(val + t);
                    const double2 x = __ldg(reinterpret_cast<const double2*>(Pr + (int64_t)colind[t] * k + col));
                    acc.x += v * x.x;
                    acc.y += v * x.y;
                }
                Y[row + col * ldy] = acc.x;
                Y[row + (col + 1) * ldy] = acc.y;
            } else if (col < k) {
                for (int64_t t = b; t < e; ++t) acc.x += __ldg(val + t) * __ldg(Pr + (int64_t)colind[t] * k + col);
                Y[row + col * ldy] = acc.x;
            }
        }
    }
}

// Row-blocked row-major SpMM: one warp computes R consecutive rows of Y for 64·NS columns.
// The warp-per-row kernel above reads one k-row of Pr per nonzero (config 5: 129 nonzeros per
// row, q = 512: 52 GB of L2 → SM traffic per product, 54× the algorithmic bytes) although
// neighbouring rows of a banded or stencil matrix touch nearly the same columns.  Here the R
// rows' column lists are walked together, smallest pending column first: its Pr row is
// loaded once (NS 16-byte loads per lane) and used by every row of the block that holds that
// column, and each (colind, val) load is amortised over 64·NS columns.  Every row still
// accumulates its nonzeros in storage order, so the result is bitwise that of the per-row
// kernel; unsorted or duplicate column indices only cost sharing, not correctness.
template <int R, int NS>
__global__ void __launch_bounds__(256)
    spmm_csr_rowblock_kernel(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
                             const double* __restrict__ val, const double* __restrict__ Pr, int64_t k,
                             double* __restrict__ Y, int64_t ldy, const int* skip) {
    if (skip && *skip) return;
    static_assert(R % 2 == 0, "row pairs are stored together");
    constexpr int32_t NONE = 0x7fffffff;
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t passes = k / (64 * NS), blocks = (n + R - 1) / R;
    const bool pair16 = (ldy & 1) == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
    for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < blocks * passes; u += warps) {
        const int64_t rb = u / passes, pass = u - rb * passes;
        const int64_t row0 = rb * R, c0 = pass * (64 * NS) + 2 * lane;
        int64_t ptr[R], end[R];
        int32_t cur[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const bool ok = row0 + r < n;
            ptr[r] = ok ? rowptr[row0 + r] : 0;
            end[r] = ok ? rowptr[row0 + r + 1] : 0;
            cur[r] = ptr[r] < end[r] ? __ldg(colind + ptr[r]) : NONE;
        }
        double2 acc[R][NS];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int s = 0; s < NS; ++s) acc[r][s] = make_double2(0.0, 0.0);
        for (;;) {
            int32_t cmin = cur[0];
#pragma unroll
            for (int r = 1; r < R; ++r) cmin = min(cmin, cur[r]);
            if (cmin == NONE) break;
            const double2* prow = reinterpret_cast<const double2*>(Pr + (int64_t)cmin * k + c0);
            double2 x[NS];
#pragma unroll
            for (int s = 0; s < NS; ++s) x[s] = __ldg(prow + s * 32);
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (cur[r] == cmin) {
                    const double v = __ldg(val + ptr[r]);
#pragma unroll
                    for (int s = 0; s < NS; ++s) {
                        acc[r][s].x += v * x[s].x;
                        acc[r][s].y += v * x[s].y;
                    }
                    ++ptr[r];
                    cur[r] = ptr[r] < end[r] ? __ldg(colind + ptr[r]) : NONE;
                }
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            double* y0 = Y + row0 + (c0 + s * 64) * ldy;  // column c, rows row0..; column c + 1 at y0 + ldy
#pragma unroll
            for (int r = 0; r < R; r += 2) {
                if (pair16 && row0 + r + 1 < n) {
                    *reinterpret_cast<double2*>(y0 + r) = make_double2(acc[r][s].x, acc[r + 1][s].x);
                    *reinterpret_cast<double2*>(y0 + ldy + r) = make_double2(acc[r][s].y, acc[r + 1][s].y);
                } else {
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        if (row0 + r + h < n) {
                            y0[r + h] = acc[r + h][s].x;
                            y0[ldy + r + h] = acc[r + h][s].y;
                        }
                }
            }
        }
    }
}

// Column-major SpMM for very wide dense operands (k ≫ 1, e.g. A·L with k = n):
// thread per (row i, column j); consecutive rows of a banded / stencil A touch
// consecutive rows of P, so the P loads of a warp coalesce.
__global__ void spmm_csr_colmajor_kernel(int64_t n, const int64_t* __restrict__ rowptr,
                                         const int32_t* __restrict__ colind, const double* __restrict__ val,
                                         const double* __restrict__ P, int64_t ldp, int64_t k, double* __restrict__ Y,
                                         int64_t ldy, const int* skip) {
    if (skip && *skip) return;
    for (int64_t j = blockIdx.y; j < k; j += gridDim.y) {
        const double* pj = P + j * ldp;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
            double acc = 0.0;
            for (int64_t t = rowptr[i]; t < rowptr[i + 1]; ++t) acc += __ldg(val + t) * __ldg(pj + colind[t]);
            Y[i + j * ldy] = acc;
        }
    }
}

// out (k×n row-major, i.e. Pᵀ col-major) = transpose of P (n×k col-major)
__global__ void transpose_kernel(const double* __restrict__ P, int64_t n, int64_t k, int64_t ldp,
                                 double* __restrict__ out, const int* skip) {
    if (skip && *skip) return;
    __shared__ double tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int64_t i = i0 + threadIdx.x, j = j0 + dy;
        if (i < n && j < k) tile[dy][threadIdx.x] = P[i + j * ldp];
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int64_t i = i0 + dy, j = j0 + threadIdx.x;
        if (i < n && j < k) out[j + i * k] = tile[threadIdx.x][dy];
    }
}

// out(j, i) = P(i, j) for an n×k block P (ld ldp) into a k×n block (ld ldo): the block row of a
// symmetric working matrix refreshed from its block column (validate_spd's left-looking sweep)
__global__ void transpose_ld_kernel(const double* __restrict__ P, int64_t n, int64_t k, int64_t ldp,
                                    double* __restrict__ out, int64_t ldo, const int* skip) {
    if (skip && *skip) return;
    __shared__ double tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int64_t i = i0 + threadIdx.x, j = j0 + dy;
        if (i < n && j < k) tile[dy][threadIdx.x] = P[i + j * ldp];
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int64_t i = i0 + dy, j = j0 + threadIdx.x;
        if (i < n && j < k) out[j + i * ldo] = tile[threadIdx.x][dy];
    }
}

// d_j = sum_i AL(i,j) * L(i,j)  (diag(Lᵀ A L)); one warp per column.
__global__ void column_dots_kernel(const double* __restrict__ AL, const double* __restrict__ L, int64_t n,
                                   double* __restrict__ d) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < n; j += warps) {
        double s = 0.0;
        for (int64_t i = lane; i < n; i += 32) s += AL[i + j * n] * L[i + j * n];
        s = warp_sum(s);
        if (lane == 0) d[j] = s;
    }
}

// Eq. 8.2 diagonal d_j = l_jᵀ·A·l_j carried across L⁺ = L + (S·R)·B, B = T − R·Z
// (SURVEY App. C3): Lᵀ·A·(S·R) = Zᵀ·R and (S·R)ᵀ·A·(S·R) = R·G·R = I, so
//   d⁺_j = d_j + 2⟨(R·Z)_j, B_j⟩ + ‖B_j‖² = d_j + 2⟨T_j, B_j⟩ − ‖B_j‖².
// B and T are q×n (ld q); T = S̃ᵀ is given by the index list when T is null.
// One warp per column, O(n·q) in total instead of the 2n³ of A·L.
__global__ void pdiag_update_kernel(const double* __restrict__ B, int64_t q, int64_t n, const double* __restrict__ T,
                                    const int64_t* __restrict__ idx, const int* skip, double* __restrict__ d) {
    if (skip && *skip) return;
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < n; j += warps) {
        double bb = 0.0, tb = 0.0;
        for (int64_t i = lane; i < q; i += 32) {
            const double b = B[i + j * q];
            bb += b * b;
            if (T)
                tb += T[i + j * q] * b;
            else if (idx[i] == j)
                tb += b;
        }
        bb = warp_sum(bb);
        tb = warp_sum(tb);
        if (lane == 0) d[j] += 2.0 * tb - bb;
    }
}

// d_j = A_jj (the Eq. 8.2 diagonal at L = I), dense or CSR A
__global__ void problem_diagonal_kernel(const double* __restrict__ a, const int64_t* __restrict__ rowptr,
                                        const int32_t* __restrict__ colind, const double* __restrict__ val, int64_t n,
                                        double* __restrict__ d) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        if (a) {
            d[j] = a[j + j * n];
        } else {
            double v = 0.0;
            for (int64_t t = rowptr[j]; t < rowptr[j + 1]; ++t)
                if (colind[t] == j) v += val[t];
            d[j] = v;
        }
    }
}

// B = T − R·Z precursor for coordinate S̃: after B = −R·Z, add T = S̃ᵀ (B[j, idx[j]] += 1).
__global__ void add_selector_kernel(double* B, int64_t q, const int64_t* __restrict__ idx, const int* skip) {
    if (skip && *skip) return;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < q; j += (int64_t)gridDim.x * blockDim.x)
        B[j + idx[j] * q] += 1.0;
}

// ‖X‖ entries of a dense matrix into a scaled copy (used for QD-style scaling)
__global__ void scatter_coordinate_kernel(double* S, int64_t n, int64_t q, const int64_t* __restrict__ idx) {
    // S = I[:, idx] (n×q, ld n), S zero-initialised by the caller
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < q; j += (int64_t)gridDim.x * blockDim.x)
        S[idx[j] + j * n] = 1.0;
}

}  // namespace si

namespace si {

// ---- K-ISQRT for larger q: coupled Newton–Schulz iteration (one CTA per small
// kernel, GEMMs on the DMMA engine in between).  With c = ‖G‖_F:
//   Y0 = G/c, Z0 = I;  T = (3I − Z·Y)/2;  Y ← Y·T;  Z ← T·Z
// Y → (G/c)^{1/2}, Z → (G/c)^{-1/2} quadratically; R = Z/√c is the unique
// symmetric root the reference's Jacobi produces (linalg.cpp:144-155), so L⁺
// matches it to rounding.  Flags: conv (int) skips the remaining GEMMs once
// ‖Z·Y − I‖_F ≤ tol; a non-converged or non-finite result sets status (the
// reference's floor / resample signal).
__global__ void ns_init_kernel(const double* __restrict__ G, int64_t ldg, int q, double* Y, double* Z, double* scal,
                               int* status, int* conv) {
    __shared__ double red[32];
    const int tid = threadIdx.x, nt = blockDim.x;
    double s = 0.0;
    for (int idx = tid; idx < q * q; idx += nt) {
        const int i = idx % q, j = idx / q;
        const double v = 0.5 * (G[i + (int64_t)j * ldg] + G[j + (int64_t)i * ldg]);
        s += v * v;
    }
    s = warp_sum(s);
    if ((tid & 31) == 0) red[tid >> 5] = s;
    __syncthreads();
    double rmax = 0.0;  // ‖G‖_∞ (see ns_fused_kernel: a tighter λmax bound than ‖G‖_F)
    for (int i = tid; i < q; i += nt) {
        double r = 0.0;
        for (int j = 0; j < q; ++j) r += fabs(0.5 * (G[i + (int64_t)j * ldg] + G[j + (int64_t)i * ldg]));
        rmax = fmax(rmax, r);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
    __shared__ double rm[32];
    if ((tid & 31) == 0) rm[tid >> 5] = rmax;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0, m = 0.0;
        for (int w = 0; w < nt / 32; ++w) {
            t += red[w];
            m = fmax(m, rm[w]);
        }
        scal[0] = fmin(sqrt(t), m);
        scal[1] = 1e300;  // previous error
    }
    __syncthreads();
    const double c = scal[0];
    const bool bad = !(c > 0.0) || !isfinite(c) || *status;
    for (int idx = tid; idx < q * q; idx += nt) {
        const int i = idx % q, j = idx / q;
        Y[idx] = bad ? 0.0 : 0.5 * (G[i + (int64_t)j * ldg] + G[j + (int64_t)i * ldg]) / c;
        Z[idx] = (i == j) ? 1.0 : 0.0;
    }
    if (tid == 0) {
        *conv = bad ? 1 : 0;
        if (bad) *status = 1;
    }
}

// T = (3I − ZY)/2 from Tmp = Z·Y; err = ‖ZY − I‖_F; stop once err ≤ tol or it stagnates
__global__ void ns_step_kernel(const double* __restrict__ ZY, int q, double* T, double* scal, int* conv, double tol) {
    __shared__ double red[32];
    if (*conv) return;
    const int tid = threadIdx.x, nt = blockDim.x;
    double s = 0.0;
    for (int idx = tid; idx < q * q; idx += nt) {
        const int i = idx % q, j = idx / q;
        const double d = ZY[idx] - (i == j ? 1.0 : 0.0);
        s += d * d;
        T[idx] = (i == j ? 1.5 : 0.0) - 0.5 * ZY[idx];
    }
    s = warp_sum(s);
    if ((tid & 31) == 0) red[tid >> 5] = s;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < nt / 32; ++w) t += red[w];
        const double err = sqrt(t);
        if (err <= tol || (err < 1e-8 && err >= scal[1])) *conv = 2;  // converged (2: stop after this check)
        scal[1] = err;
    }
}

__global__ void ns_copy2_kernel(double* Y, const double* Yn, double* Z, const double* Zn, int q, const int* conv) {
    if (*conv) return;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < q * q; idx += gridDim.x * blockDim.x) {
        Y[idx] = Yn[idx];
        Z[idx] = Zn[idx];
    }
}

// R = Z/√c (symmetrized) when the iteration converged and certifies the floor:
// ‖R‖²_F = Σ 1/λ_i ≥ 1/λmin and c ≥ λmax, so 1/(‖R‖²_F·c) is a lower bound of λmin/λmax;
// above ISQRT_FAST_ACCEPT (100× the reference's 1e-14 floor) R is kept.  Otherwise (no
// convergence, a near-singular G) *need is set and jacobi_isqrt_kernel decides with the
// reference's own rule (linalg.cpp:144-155).  One CTA.
__global__ void __launch_bounds__(1024) ns_finish_kernel(const double* __restrict__ Z, int q, const double* scal,
                                                         double* R, int* status, const int* conv, int* need) {
    __shared__ double red[32];
    __shared__ int s_ok;
    if (*status) return;
    const int tid = threadIdx.x, nt = blockDim.x;
    const double rc = 1.0 / sqrt(scal[0]);
    double ss = 0.0;
    for (int idx = tid; idx < q * q; idx += nt) {
        const int i = idx % q, j = idx / q;
        const double v = 0.5 * (Z[i + j * q] + Z[j + i * q]) * rc;
        ss += v * v;
    }
    ss = warp_sum(ss);
    if ((tid & 31) == 0) red[tid >> 5] = ss;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < nt / 32; ++w) t += red[w];
        const bool conv_ok = *conv == 2 && scal[1] < 1e-6;
        s_ok = conv_ok && isfinite(t) && t > 0.0 && 1.0 / (t * scal[0]) > ISQRT_FAST_ACCEPT;
        *need = s_ok ? 0 : 1;
    }
    __syncthreads();
    if (!s_ok) return;
    for (int idx = tid; idx < q * q; idx += nt) {
        const int i = idx % q, j = idx / q;
        R[idx] = 0.5 * (Z[i + j * q] + Z[j + i * q]) * rc;
    }
}

// ---- fused Newton–Schulz for q ≤ 64: one CTA, all five QP×QP operands in
// shared memory (pitch QP+4 ≡ 4 mod 16 → conflict-free fragment loads), each
// product on the DMMA pipe (mma.m16n8k8), no global round trips between
// iterations.  Padding rows/cols carry an identity block, which the iteration
// leaves invariant.  Same contract as the multi-kernel variant above.
// C_j = A_j·B_j for NP independent QP×QP products in the dynamic shared buffer
// `nsm` (operands addressed by offsets, pitch QP+4 ≡ 4 mod 16: conflict-free
// fragment loads).  Every product in the Newton–Schulz iteration is a polynomial
// in the same symmetric G (Y, Z, T commute and stay symmetric), so only the
// m16×n8 output blocks that meet the upper triangle are computed (20 of 32 at
// QP = 64) and each element (r ≤ c) is stored to (r, c) and (c, r): every entry
// is written exactly once and the result is exactly symmetric.  Each warp owns
// PER blocks across the NP products and advances all of their accumulation
// chains together, so the DMMA pipe sees NP·PER independent chains.
extern __shared__ __align__(16) double nsm[];

template <int QP>
__device__ __forceinline__ void upper_block(int idx, int& m0, int& n0) {
    constexpr int MB = QP / 16, NB = QP / 8;
#pragma unroll
    for (int mb = 0; mb < MB; ++mb) {
        const int cnt = NB - 2 * mb;
        if (idx < cnt) {
            m0 = mb * 16;
            n0 = (2 * mb + idx) * 8;
            return;
        }
        idx -= cnt;
    }
    m0 = n0 = 0;
}

template <int QP, int NW, int NP>
__device__ __forceinline__ void cta_symm_products(const int (&aoff)[NP], const int (&boff)[NP], const int (&coff)[NP],
                                                  int warp, int lane) {
    constexpr int LD = QP + 4;
    constexpr int MB = QP / 16, NB = QP / 8;
    constexpr int NBLK = MB * NB - MB * (MB - 1);  // blocks meeting the upper triangle
    constexpr int TOT = NP * NBLK;
    constexpr int PER = (TOT + NW - 1) / NW;
    const int g = lane >> 2, t = lane & 3;
    int m0s[PER], n0s[PER], ao[PER], bo[PER], co[PER];
#pragma unroll
    for (int p = 0; p < PER; ++p) {
        const int job = min(warp + p * NW, TOT - 1);
        const int u = job / NBLK;
        upper_block<QP>(job % NBLK, m0s[p], n0s[p]);
        ao[p] = aoff[0];
        bo[p] = boff[0];
        co[p] = coff[0];
#pragma unroll
        for (int v = 1; v < NP; ++v)
            if (u == v) {
                ao[p] = aoff[v];
                bo[p] = boff[v];
                co[p] = coff[v];
            }
    }
    double c[PER][4];
#pragma unroll
    for (int p = 0; p < PER; ++p)
#pragma unroll
        for (int e = 0; e < 4; ++e) c[p][e] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < QP; k0 += 8) {
#pragma unroll
        for (int p = 0; p < PER; ++p) {
            if (warp + p * NW < TOT) {
                const double* Au = nsm + ao[p];
                const double* Bu = nsm + bo[p];
                const int m0 = m0s[p], n0 = n0s[p];
                double a[4], b[2];
                a[0] = Au[(m0 + g) + (k0 + t) * LD];
                a[1] = Au[(m0 + g + 8) + (k0 + t) * LD];
                a[2] = Au[(m0 + g) + (k0 + t + 4) * LD];
                a[3] = Au[(m0 + g + 8) + (k0 + t + 4) * LD];
                b[0] = Bu[(k0 + t) + (n0 + g) * LD];
                b[1] = Bu[(k0 + t + 4) + (n0 + g) * LD];
                dmma_1688(c[p], a, b);
            }
        }
    }
#pragma unroll
    for (int p = 0; p < PER; ++p) {
        if (warp + p * NW < TOT) {
            double* Cu = nsm + co[p];
            const int m0 = m0s[p], n0 = n0s[p];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int r = m0 + g + ((e >> 1) << 3), cc = n0 + 2 * t + (e & 1);
                if (r <= cc) {
                    Cu[r + cc * LD] = c[p][e];
                    Cu[cc + r * LD] = c[p][e];
                }
            }
        }
    }
}

template <int QP>
__global__ void __launch_bounds__(512) ns_fused_kernel(const double* __restrict__ G, int64_t ldg, int q,
                                                       double* __restrict__ R, int* status, double tol, int max_it,
                                                       int accelerate) {
    constexpr int LD = QP + 4, SZ = QP * LD, NW = 16;
    __shared__ double red[NW];
    __shared__ double s_c, s_err, s_prev;
    __shared__ int s_stop, s_accel;
    if (*status) return;
    // operand offsets in nsm: Y, Z, T, Yn, Zn
    int oY = 0, oZ = SZ, oYn = 3 * SZ, oZn = 4 * SZ;
    const int oT = 2 * SZ;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    auto block_sum = [&](double v) {
        v = warp_sum(v);
        if (lane == 0) red[warp] = v;
        __syncthreads();
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) s += red[w];
        __syncthreads();
        return s;
    };
    // scale c ≥ λmax(G): min(‖G‖_F, ‖G‖_∞) (both bound the spectral radius of a
    // symmetric G; ‖G‖_∞ is far tighter for the near-diagonal Grams of coordinate
    // sketches, which saves Newton–Schulz iterations — the small eigenvalues of
    // G/c grow by at most 1.5× per iteration until they reach 1)
    double fro = 0.0;
    for (int idx = tid; idx < q * q; idx += nt) {
        const int i = idx % q, j = idx / q;
        const double v = 0.5 * (G[i + (int64_t)j * ldg] + G[j + (int64_t)i * ldg]);
        fro += v * v;
    }
    fro = block_sum(fro);
    __shared__ double s_rowmax[NW];
    double rmax = 0.0;
    for (int i = tid; i < q; i += nt) {  // row abs sums
        double r = 0.0;
        for (int j = 0; j < q; ++j) r += fabs(0.5 * (G[i + (int64_t)j * ldg] + G[j + (int64_t)i * ldg]));
        rmax = fmax(rmax, r);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
    if (lane == 0) s_rowmax[warp] = rmax;
    __syncthreads();
    if (tid == 0) {
        double m = 0.0;
        for (int w = 0; w < NW; ++w) m = fmax(m, s_rowmax[w]);
        s_c = fmin(sqrt(fro), m);
        s_prev = 1e300;
        s_stop = 0;
        s_accel = 1;
    }
    __syncthreads();
    const double cc = s_c;
    if (!(cc > 0.0) || !isfinite(cc)) {
        if (tid == 0) *status = 1;
        return;
    }
    for (int idx = tid; idx < QP * QP; idx += nt) {
        const int i = idx % QP, j = idx / QP;
        const bool in = i < q && j < q;
        nsm[oY + i + j * LD] = in ? 0.5 * (G[i + (int64_t)j * ldg] + G[j + (int64_t)i * ldg]) / cc : (i == j ? 1.0 : 0.0);
        nsm[oZ + i + j * LD] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int it = 0; it < max_it; ++it) {
        {
            const int a1[1] = {oZ}, b1[1] = {oY}, c1[1] = {oT};
            cta_symm_products<QP, NW, 1>(a1, b1, c1, warp, lane);  // T ← Z·Y
        }
        __syncthreads();
        // T = a·I − b·ZY with a − b = 1 (fixed point ZY = I).  Eigenvalue-wise (every
        // iterate is a polynomial in G) x = λ(ZY) maps to x·(a − b·x)².  The Newton step
        // a = 3/2 grows a small x by 2.25× per iteration; the kernel starts with a = 2
        // (4× growth; from a spectrum in (0, 1] it stays in (0, 32/27]) and switches to
        // Newton for good once ‖ZY − I‖_F < 1/2 or stops falling by a quarter per step
        // (a = 2 is neutral at x = 1, so eigenvalues near 1 only oscillate under it).
        // Same unique limit (G/c)^{-1/2}.  SI_NS_NEWTON_ONLY=1 disables it.
        const bool accel = accelerate && s_accel;
        const double ca = accel ? 2.0 : 1.5, cb = ca - 1.0;
        double e = 0.0;
        for (int idx = tid; idx < QP * QP; idx += nt) {
            const int i = idx % QP, j = idx / QP;
            const double zy = nsm[oT + i + j * LD];
            const double d = zy - (i == j ? 1.0 : 0.0);
            e += d * d;
            nsm[oT + i + j * LD] = (i == j ? ca : 0.0) - cb * zy;
        }
        e = block_sum(e);
        if (tid == 0) {
            const double err = sqrt(e);
            if (err < 0.5 || err > 0.75 * s_prev) s_accel = 0;
            s_stop = (err <= tol || (err < 1e-8 && err >= s_prev)) ? 1 : 0;
            s_prev = err;
            s_err = err;
        }
        __syncthreads();
        if (s_stop) break;
        {
            const int a2[2] = {oY, oT}, b2[2] = {oT, oZ}, c2[2] = {oYn, oZn};
            cta_symm_products<QP, NW, 2>(a2, b2, c2, warp, lane);  // Y ← Y·T, Z ← T·Z
        }
        __syncthreads();
        int tmp = oY;
        oY = oYn;
        oYn = tmp;
        tmp = oZ;
        oZ = oZn;
        oZn = tmp;
    }
    // keep R = Z/√c when Newton–Schulz converged and certifies λmin/λmax > ISQRT_FAST_ACCEPT
    // (‖R‖²_F = Σ 1/λ_i ≥ 1/λmin, c ≥ λmax); otherwise the reference's Jacobi + floor rule
    // decides in this CTA (linalg.cpp:144-155), its work arrays in the operand buffers
    const double rc = 1.0 / sqrt(cc);
    double ss = 0.0;
    for (int idx = tid; idx < q * q; idx += nt) {
        const int i = idx % q, j = idx / q;
        const double v = nsm[oZ + i + j * LD] * rc;
        ss += v * v;
    }
    ss = block_sum(ss);
    const bool fast = s_stop && s_err < 1e-6 && isfinite(ss) && ss > 0.0 && 1.0 / (ss * cc) > ISQRT_FAST_ACCEPT;
    if (!fast) {
        jacobi_isqrt_block(G, ldg, q, nsm, R, q, status, ISQRT_FLOOR);
        return;
    }
    for (int idx = tid; idx < q * q; idx += nt) {
        const int i = idx % q, j = idx / q;
        R[idx] = nsm[oZ + i + j * LD] * rc;  // Z is exactly symmetric
    }
}

// ---- recursive SPD inverse helpers (q > 128): Gi21 := Gi12ᵀ and scaled copies
__global__ void scale_copy_kernel(const double* __restrict__ src, int64_t lds, double* __restrict__ dst, int64_t ldd,
                                  int64_t rows, int64_t cols, double alpha, const int* skip) {
    if (skip && *skip) return;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < rows * cols;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx % rows, j = idx / rows;
        dst[i + j * ldd] = alpha * src[i + j * lds];
    }
}

// lower triangle := upper triangle (q×q, ld) — exact symmetry of an assembled inverse
__global__ void mirror_upper_kernel(double* g, int64_t q, int64_t ld, const int* skip) {
    if (skip && *skip) return;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < q * q;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx % q, j = idx / q;
        if (i > j) g[i + j * ld] = g[j + i * ld];
    }
}

}  // namespace si
