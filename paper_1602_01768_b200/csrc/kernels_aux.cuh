// Non-GEMM kernels of the RBFGS / AdaRBFGS iteration (sm_100a):
//   - split-K and scalar reductions (deterministic order),
//   - K-FACTOR: SPD check + inverse of the q×q Gram (Gauss-Jordan without
//     pivoting, single CTA; its pivots are the squared Cholesky diagonals, so
//     the failure test matches gram_llt, qn_updates.cpp:37-43),
//   - K-CORE: assembly of the 2q×2q core M of the rank-2q update,
//   - K-RNG: counter-based (Philox4x32-10) Gaussian sketch generator,
//   - small fill / copy helpers.
#pragma once
#include "common.cuh"

namespace si {

// C(m,n) = alpha * sum_z ws[z][m,n] + beta * C(m,n)
__global__ void splitk_reduce_kernel(const double* __restrict__ ws, int splits, int64_t M, int64_t N, double* C,
                                     int64_t ldc, double alpha, double beta, const int* skip,
                                     const double* Csrc = nullptr) {
    griddep_wait();
    griddep_launch();
    if (skip && *skip) return;
    const int64_t total = M * N;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int z = 0; z < splits; ++z) s += ws[z * total + idx];
        int64_t m, n;
        if (total < (int64_t(1) << 31)) {  // 32-bit index arithmetic
            const uint32_t i32 = (uint32_t)idx, m32 = (uint32_t)M, q32 = i32 / m32;
            n = q32;
            m = i32 - q32 * m32;
        } else {
            n = idx / M;
            m = idx - n * M;
        }
        double* c = C + m + n * ldc;
        const double* cs = Csrc ? Csrc + m + n * ldc : c;
        *c = beta != 0.0 ? alpha * s + beta * *cs : alpha * s;
    }
}

// out[0] = sum ws[0..count) in a fixed order (one CTA).
__global__ void sum_reduce_kernel(const double* __restrict__ ws, int64_t count, double* out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) s += ws[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        out[0] = t;
    }
}

// K-FACTOR.  G_ref(i,j) = P(min(i,j), max(i,j)) (the reference's LLT reads the
// lower triangle of gram = SᵀAS; P = YᵀS = gramᵀ).  Writes Ginv (q×q, ldo) and
// sets *status = 1 when a pivot is not > 0 (the GramRankDeficientError
// resample signal, qn_updates.cpp:37-43).
//
// Gauss-Jordan without pivoting, register resident: thread t owns column
// j = t % q and rows [r0, r0 + RPT) with r0 = (t / q)·RPT, so one elimination
// step is: owners of row k / column k publish them to shared memory, barrier,
// RPT register FMAs, barrier.  Used for q ≤ 128 (RPT ≤ 32); larger q falls back
// to the shared/global-memory variant below.
template <int RPT, int MAXT>
__global__ void __launch_bounds__(MAXT) spd_inverse_reg_kernel(const double* __restrict__ P, int64_t ldp, int q,
                                                               double* __restrict__ ginv, int64_t ldo, int* status) {
    __shared__ double rowk[128], colk[128];
    if (*status) return;
    const int tid = threadIdx.x;
    const int j = tid % q, grp = tid / q, r0 = grp * RPT;
    const int ngrp = (q + RPT - 1) / RPT;
    const bool active = grp < ngrp;
    double a[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int i = r0 + r;
        a[r] = (active && i < q) ? (i <= j ? P[i + (int64_t)j * ldp] : P[j + (int64_t)i * ldp]) : 0.0;
    }
    // k = kb·RPT + kr with kr unrolled, so the owner of pivot row k reads the
    // compile-time register a[kr] and the update needs no dynamic indexing
    for (int kb = 0; kb < ngrp; ++kb) {
        const bool own_row = active && grp == kb;
#pragma unroll
        for (int kr = 0; kr < RPT; ++kr) {
            const int k = kb * RPT + kr;
            if (k >= q) break;  // uniform
            if (own_row) rowk[j] = a[kr];
            if (active && j == k) {
#pragma unroll
                for (int r = 0; r < RPT; ++r) colk[r0 + r] = a[r];
            }
            __syncthreads();
            const double piv = colk[k];
            if (!(piv > 0.0)) {  // uniform: every thread read the same shared value
                if (tid == 0) *status = 1;
                return;
            }
            const double inv = 1.0 / piv;
            const bool jk = j == k;
            const double rk = (jk ? 1.0 : rowk[j]) * inv;  // new row k, column j
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                const double base = jk ? 0.0 : a[r];
                const double upd = base - colk[r0 + r] * rk;
                a[r] = (r == kr && own_row) ? rk : upd;
            }
            __syncthreads();
        }
    }
    if (active) {
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const int i = r0 + r;
            if (i < q) ginv[i + (int64_t)j * ldo] = a[r];
        }
    }
}

// Ĝ = G − H' for the RBFGS update X⁺ = X + [Z R]·[W' Z]ᵀ (engine.cu): G read from
// the upper triangle of P[:, 0:q] (as K-FACTOR reads it), H' = P[:, q:2q] = −YᵀXY symmetrised
__global__ void ghat_kernel(const double* __restrict__ P, int64_t ldp, int q, double* __restrict__ gh, const int* skip) {
    if (skip && *skip) return;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < q * q; idx += gridDim.x * blockDim.x) {
        const int i = idx % q, j = idx / q;
        const double g = i <= j ? P[i + (int64_t)j * ldp] : P[j + (int64_t)i * ldp];
        const double h = 0.5 * (P[i + (int64_t)(q + j) * ldp] + P[j + (int64_t)(q + i) * ldp]);
        gh[idx] = g - h;
    }
}

// symmetrize Ginv in place: (G + Gᵀ)/2 (exact symmetry of the implied projector)
__global__ void symmetrize_small_kernel(double* g, int q, int64_t ld, const int* skip) {
    if (skip && *skip) return;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < q * q; idx += gridDim.x * blockDim.x) {
        const int i = idx % q, j = idx / q;
        if (i < j) {
            const double v = 0.5 * (g[i + j * ld] + g[j + i * ld]);
            g[i + j * ld] = v;
            g[j + i * ld] = v;
        }
    }
}

// K-FACTOR, blocked.  G⁻¹ for SPD G (q ≤ 128, read as G(i,j) = P(min, max)) by
// Gauss-Jordan in 16-column panels, the whole matrix resident in shared memory
// (padded to QP = 16·⌈q/16⌉ with an identity block, which keeps it SPD):
//   D = G[p,p] → D⁻¹ by one warp (16 scalar GJ steps, warp-synchronous; every
//       scalar pivot is the one the unblocked elimination meets, so "pivot ≤ 0"
//       is still gram_llt's failure test),
//   R' = D⁻¹·G[p,:],  C = G[:,p],
//   G[i,j] −= C[i,:]·R'[:,j] for the whole matrix — a rank-16 update on the DMMA
//       pipe (16 warps × 32×32 tiles) — then G[p,:] = R', G[:,p] = −C·D⁻¹, G[p,p] = D⁻¹.
// Eight panels at q = 128: ~40 CTA barriers instead of the 256 of the scalar
// elimination, and one launch instead of the recursion's eleven (measured: the q×q
// stage of a config-3 iteration 232 vs 268 µs).  Output symmetrised exactly.
template <int QP, int PB>
__global__ void __launch_bounds__(512) spd_inverse_blocked_kernel(const double* __restrict__ P, int64_t ldp, int q,
                                                                 double* __restrict__ ginv, int64_t ldo, int* status) {
    constexpr int LDG = QP + 4, LDC = PB + 4, LDR = QP + 4, LDD = PB + 1;
    static_assert(PB == 16 || PB == 32, "panel width");
    extern __shared__ __align__(16) double gsm[];
    double* Gs = gsm;                  // QP × LDG
    double* Cb = Gs + QP * LDG;        // QP × LDC  (column panel, m-major rows: Cb[i*LDC + l])
    double* Rb = Cb + QP * LDC;        // PB × LDR  (new row panel)
    double* Db = Rb + PB * LDR;        // PB × LDD
    __shared__ int s_bad;
    if (*status) return;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < QP * QP; e += nt) {
        const int i = e % QP, j = e / QP;
        double v;
        if (i < q && j < q)
            v = i <= j ? P[i + (int64_t)j * ldp] : P[j + (int64_t)i * ldp];
        else
            v = i == j ? 1.0 : 0.0;
        Gs[i * LDG + j] = v;
    }
    if (tid == 0) s_bad = 0;
    __syncthreads();
    for (int k0 = 0; k0 < QP; k0 += PB) {
        // D⁻¹ by warp 0: lane j < 16 holds column j of D in registers; row and column k
        // of each elimination step travel by shuffles (no shared-memory round trips)
        if (warp == 0) {
            const int j = lane & (PB - 1);
            double d[PB];
#pragma unroll
            for (int i = 0; i < PB; ++i) d[i] = Gs[(k0 + i) * LDG + k0 + j];
            bool bad = false;
#pragma unroll
            for (int k = 0; k < PB; ++k) {
                const double piv = __shfl_sync(0xffffffffu, d[k], k);
                bad |= !(piv > 0.0);  // uniform; once set the values are discarded
                const double inv = 1.0 / piv;
                const double rk = d[k];  // row k, column j (old)
#pragma unroll
                for (int i = 0; i < PB; ++i) {
                    const double cki = __shfl_sync(0xffffffffu, d[i], k);  // column k, row i (old)
                    if (i == k)
                        d[i] = j == k ? inv : rk * inv;
                    else
                        d[i] = j == k ? -cki * inv : d[i] - cki * rk * inv;
                }
            }
            if (lane < PB) {
#pragma unroll
                for (int i = 0; i < PB; ++i) Db[i * LDD + j] = d[i];
            }
            if (bad && lane == 0) s_bad = 1;
        }
        // C = G[:, p] (old) for every thread
        for (int e = tid; e < QP * PB; e += nt) {
            const int i = e / PB, l = e % PB;
            Cb[i * LDC + l] = Gs[i * LDG + k0 + l];
        }
        __syncthreads();
        if (s_bad) {
            if (tid == 0) *status = 1;  // not positive definite: the resample signal
            return;
        }
        // R' = D⁻¹·G[p, :]
        for (int e = tid; e < PB * QP; e += nt) {
            const int r = e / QP, j = e % QP;
            double acc = 0.0;
#pragma unroll
            for (int l = 0; l < PB; ++l) acc += Db[r * LDD + l] * Gs[(k0 + l) * LDG + j];
            Rb[r * LDR + j] = acc;
        }
        __syncthreads();
        // G −= C·R' (rank-16, DMMA): 16 warps as 4×4, warp tile (QP/4)×(QP/4)
        {
            constexpr int WT = QP / 4, MI = WT / 16, NI = WT / 8;
            const int g = lane >> 2, t4 = lane & 3, wm0 = (warp >> 2) * WT, wn0 = (warp & 3) * WT;
            if (WT >= 16) {
                double acc[MI > 0 ? MI : 1][NI > 0 ? NI : 1][4];
#pragma unroll
                for (int i = 0; i < MI; ++i)
#pragma unroll
                    for (int j = 0; j < NI; ++j)
#pragma unroll
                        for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;
#pragma unroll
                for (int kk = 0; kk < PB; kk += 8) {
                    double a[MI > 0 ? MI : 1][4], b[NI > 0 ? NI : 1][2];
#pragma unroll
                    for (int i = 0; i < MI; ++i)
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            a[i][e] = Cb[(wm0 + i * 16 + g + ((e & 1) << 3)) * LDC + kk + t4 + ((e >> 1) << 2)];
#pragma unroll
                    for (int j = 0; j < NI; ++j)
#pragma unroll
                        for (int e = 0; e < 2; ++e) b[j][e] = Rb[(kk + t4 + (e << 2)) * LDR + wn0 + j * 8 + g];
#pragma unroll
                    for (int i = 0; i < MI; ++i)
#pragma unroll
                        for (int j = 0; j < NI; ++j) dmma_1688(acc[i][j], a[i], b[j]);
                }
#pragma unroll
                for (int i = 0; i < MI; ++i)
#pragma unroll
                    for (int j = 0; j < NI; ++j)
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int r = wm0 + i * 16 + g + ((e >> 1) << 3), c = wn0 + j * 8 + 2 * t4 + (e & 1);
                            Gs[r * LDG + c] -= acc[i][j][e];
                        }
            } else {
                for (int e = tid; e < QP * QP; e += nt) {
                    const int r = e / QP, c = e % QP;
                    double acc = 0.0;
#pragma unroll
                    for (int l = 0; l < PB; ++l) acc += Cb[r * LDC + l] * Rb[l * LDR + c];
                    Gs[r * LDG + c] -= acc;
                }
            }
        }
        __syncthreads();
        // the pivot rows / columns: G[p,:] = R', G[:,p] = −C·D⁻¹, G[p,p] = D⁻¹
        for (int e = tid; e < PB * QP; e += nt) {
            const int r = e / QP, j = e % QP;
            if (j < k0 || j >= k0 + PB) Gs[(k0 + r) * LDG + j] = Rb[r * LDR + j];
        }
        for (int e = tid; e < QP * PB; e += nt) {
            const int i = e / PB, l = e % PB;
            if (i < k0 || i >= k0 + PB) {
                double acc = 0.0;
#pragma unroll
                for (int m = 0; m < PB; ++m) acc += Cb[i * LDC + m] * Db[m * LDD + l];
                Gs[i * LDG + k0 + l] = -acc;
            }
        }
        for (int e = tid; e < PB * PB; e += nt) Gs[(k0 + e / PB) * LDG + k0 + e % PB] = Db[(e / PB) * LDD + e % PB];
        __syncthreads();
    }
    for (int e = tid; e < q * q; e += nt) {  // exact symmetrisation
        const int i = e % q, j = e / q;
        ginv[i + (int64_t)j * ldo] = 0.5 * (Gs[i * LDG + j] + Gs[j * LDG + i]);
    }
}

// Shared/global-memory Gauss-Jordan for large q (same arithmetic).
__global__ void __launch_bounds__(1024) spd_inverse_kernel(const double* __restrict__ P, int64_t ldp, int q,
                                                           double* __restrict__ ginv, int64_t ldo, double* work,
                                                           int* status, int use_smem) {
    extern __shared__ __align__(16) double sm[];
    if (*status) return;
    double* a = use_smem ? sm : work;  // q×q col-major, ld = q
    double* rowk = use_smem ? sm + (size_t)q * q : work + (size_t)q * q;
    double* colk = rowk + q;
    __shared__ int fail;
    const int tid = threadIdx.x, nt = blockDim.x;
    if (tid == 0) fail = 0;
    for (int idx = tid; idx < q * q; idx += nt) {
        const int i = idx % q, j = idx / q;
        a[idx] = i <= j ? P[i + (int64_t)j * ldp] : P[j + (int64_t)i * ldp];
    }
    __syncthreads();
    for (int k = 0; k < q; ++k) {
        const double piv = a[k + k * q];
        if (!(piv > 0.0)) {
            if (tid == 0) fail = 1;
            break;
        }
        const double inv = 1.0 / piv;
        for (int j = tid; j < q; j += nt) {
            rowk[j] = (j == k ? 1.0 : a[k + j * q]) * inv;
            colk[j] = a[j + k * q];
        }
        __syncthreads();
        for (int idx = tid; idx < q * q; idx += nt) {
            const int i = idx % q, j = idx / q;
            if (i == k) {
                a[idx] = rowk[j];
            } else {
                const double base = (j == k) ? 0.0 : a[idx];
                a[idx] = base - colk[i] * rowk[j];
            }
        }
        __syncthreads();
    }
    __syncthreads();
    if (fail) {
        if (tid == 0) *status = 1;
        return;
    }
    for (int idx = tid; idx < q * q; idx += nt) {
        const int i = idx % q, j = idx / q;
        ginv[i + (int64_t)j * ldo] = 0.5 * (a[i + j * q] + a[j + i * q]);
    }
}

// K-CORE (part 1): lay out M = [[Ginv, −Ginv], [−Ginv, 0]] (2q×2q, ld 2q) from
// Ginv so that the follow-up GEMM M11 += Ginv·(H·Ginv) completes
// M11 = Ginv + Ginv·H·Ginv.
__global__ void core_layout_kernel(const double* __restrict__ ginv, int q, double* __restrict__ M, const int* skip) {
    if (skip && *skip) return;
    const int q2 = 2 * q;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < q2 * q2; idx += gridDim.x * blockDim.x) {
        const int i = idx % q2, j = idx / q2;
        double v;
        if (i < q && j < q) v = ginv[i + j * q];
        else if (i >= q && j >= q) v = 0.0;
        else v = -ginv[(i % q) + (j % q) * q];
        M[idx] = v;
    }
}

// A rejected core (status[0] != 0) leaves M = 0, so the update that follows it,
// X += V·Uᵀ with V = U·M, adds exact zeros: the sharded driver enqueues the update
// before it reads the PD status (deferred check, dist.py SymmetricShardedRBFGS).
__global__ void zero_on_status_kernel(double* __restrict__ M, int64_t count, const int* status) {
    if (!*status) return;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
        M[i] = 0.0;
}

// ---------------------------------------------------------------- K-RNG --
struct Philox {
    __device__ static void round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0, uint32_t k1) {
        const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
        const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
        const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    __device__ static void gen(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            round(c[0], c[1], c[2], c[3], k0, k1);
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
    }
};

// S(i,j) ~ N(0,1), column-major n×q with leading dimension lds.  Element pair
// (2e, 2e+1) in linear order comes from Philox(key = seed, counter = (e, draw)).
// `draw_counter` lives in device memory so one captured iteration can be
// replayed; K-FACTOR's launcher advances it.
__global__ void philox_gaussian_kernel(double* __restrict__ S, int64_t n, int64_t q, int64_t lds, uint64_t seed,
                                       const unsigned long long* draw_counter, const int* skip,
                                       unsigned long long draw_value = 0) {
    griddep_wait();
    griddep_launch();
    if (skip && *skip) return;
    const uint64_t draw = draw_counter ? *draw_counter : draw_value;
    const int64_t total = n * q;
    const int64_t pairs = (total + 1) / 2;
    const bool pair16 = (n & 1) == 0 && (lds & 1) == 0 && (reinterpret_cast<uintptr_t>(S) & 15) == 0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < pairs; e += (int64_t)gridDim.x * blockDim.x) {
        uint32_t c[4] = {(uint32_t)e, (uint32_t)(e >> 32), (uint32_t)draw, (uint32_t)(draw >> 32)};
        Philox::gen(c, (uint32_t)seed, (uint32_t)(seed >> 32));
        const uint64_t x0 = ((uint64_t)c[0] << 32) | c[1];
        const uint64_t x1 = ((uint64_t)c[2] << 32) | c[3];
        const double u1 = ((double)(x0 >> 11) + 0.5) * 0x1.0p-53;  // (0,1)
        const double u2 = ((double)(x1 >> 11)) * 0x1.0p-53;        // [0,1)
        const double r = sqrt(-2.0 * log(u1));
        double sn, cs;
        sincospi(2.0 * u2, &sn, &cs);
        const int64_t l0 = 2 * e, l1 = 2 * e + 1;
        int64_t i0, j0, i1, j1;
        if (total < (int64_t(1) << 31)) {  // 32-bit index arithmetic (a 64-bit division is a long software sequence)
            const uint32_t n32 = (uint32_t)n, a = (uint32_t)l0, b = (uint32_t)l1;
            j0 = a / n32;
            i0 = a - (uint32_t)j0 * n32;
            j1 = b / n32;
            i1 = b - (uint32_t)j1 * n32;
        } else {
            j0 = l0 / n;
            i0 = l0 - j0 * n;
            j1 = l1 / n;
            i1 = l1 - j1 * n;
        }
        if (pair16) {  // n even: the pair shares a column and is 16-byte aligned — one full-width store
            *reinterpret_cast<double2*>(S + i0 + j0 * lds) = make_double2(r * cs, r * sn);
        } else {
            S[i0 + j0 * lds] = r * cs;
            if (l1 < total) S[i1 + j1 * lds] = r * sn;
        }
    }
}

// End of a device-sketched iteration: advance the draw counter and, when the
// iteration's Gram was rejected, count it (status[2]) and clear the skip flag so
// the next enqueued iteration runs -- a rejected draw becomes a redraw.
__global__ void advance_counter_kernel(unsigned long long* counter, int* status) {
    griddep_wait();
    griddep_launch();
    *counter += 1ull;
    if (status[0]) {
        status[2] += 1;
        status[0] = 0;
    }
}

// End of an iteration in run_inverter's batched mode (iterations enqueued back to
// back between two checkpoints, no host round trip): every executed attempt
// advances the draw counter once, exactly as the eager loop does; an accepted step
// is counted in status[3]; a rejected Gram (status[0]) or a non-finite iterate
// (status[1]) stops the batch (status[4], with status[0] left set so every later
// launch of the batch is a no-op) and the host resumes from the exact iteration —
// so a batched run draws the same sketches and produces the same iterates as the
// eager loop.
__global__ void advance_batch_kernel(unsigned long long* counter, int* status) {
    griddep_wait();
    griddep_launch();
    if (status[4]) return;
    *counter += 1ull;
    if (status[0]) {
        status[2] += 1;
        status[4] = 1;
        return;
    }
    status[3] += 1;
    if (status[1]) {
        status[4] = 1;
        status[0] = 1;
    }
}

// run_adarbfgs's batched loop (AdaRBFGS analogue of advance_batch_kernel; status[3] is
// the Newton–Schulz stop flag there, so the accepted count lives in status[5]): a
// rejected square root (status[0]) or a non-finite factor (status[1]) stops the batch
// at that attempt; every executed attempt advances the Philox counter (device-Gaussian
// S̃) exactly once.
__global__ void ada_advance_batch_kernel(unsigned long long* counter, int* status) {
    if (status[4]) return;
    if (counter) *counter += 1ull;
    if (status[0]) {
        status[2] += 1;
        status[4] = 1;
        return;
    }
    status[5] += 1;
    if (status[1]) {
        status[4] = 1;
        status[0] = 1;
    }
}

// A <- (A + Aᵀ)/2 in place (ProblemMatrix construction, problem_matrix.cpp:9-18).
// Block (bx, by) with bx <= by owns tile pair (I=bx, J=by) and its mirror.
__global__ void symmetrize_kernel(double* A, int64_t n) {
    __shared__ double t1[32][33], t2[32][33];
    const int64_t I = blockIdx.x, J = blockIdx.y;
    if (I > J) return;
    const int tx = threadIdx.x;
    for (int ty = threadIdx.y; ty < 32; ty += blockDim.y) {
        const int64_t r1 = I * 32 + tx, c1 = J * 32 + ty;  // tile (I,J): A[r1, c1]
        const int64_t r2 = J * 32 + tx, c2 = I * 32 + ty;  // tile (J,I): A[r2, c2]
        t1[ty][tx] = (r1 < n && c1 < n) ? A[r1 + c1 * n] : 0.0;
        t2[ty][tx] = (r2 < n && c2 < n) ? A[r2 + c2 * n] : 0.0;
    }
    __syncthreads();
    for (int ty = threadIdx.y; ty < 32; ty += blockDim.y) {
        // new A[I*32+tx, J*32+ty] = 0.5 (t1[ty][tx] + A[J*32+ty, I*32+tx]) = 0.5 (t1[ty][tx] + t2[tx][ty])
        const int64_t r1 = I * 32 + tx, c1 = J * 32 + ty;
        const int64_t r2 = J * 32 + tx, c2 = I * 32 + ty;
        const double v1 = 0.5 * (t1[ty][tx] + t2[tx][ty]);
        const double v2 = 0.5 * (t2[ty][tx] + t1[tx][ty]);
        if (r1 < n && c1 < n) A[r1 + c1 * n] = v1;
        if (r2 < n && c2 < n) A[r2 + c2 * n] = v2;
    }
}

__global__ void set_identity_kernel(double* X, int64_t n, int64_t ldx) {
    const int64_t total = n * n;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx % n, j = idx / n;
        X[i + j * ldx] = (i == j) ? 1.0 : 0.0;
    }
}

// Columns `idx[0..q)` of L (n×n, ld) gathered into S (n×q, ld n): S = L·S̃ for a
// coordinate S̃ (adarbfgs.cpp:13 without the dense GEMM).
__global__ void gather_columns_kernel(const double* __restrict__ L, int64_t n, int64_t ldl,
                                      const int64_t* __restrict__ idx, int64_t q, double* __restrict__ S) {
    // grid.y walks the q gathered columns, grid.x the rows: coalesced, no index division
    for (int64_t j = blockIdx.y; j < q; j += gridDim.y) {
        const double* __restrict__ src = L + idx[j] * ldl;
        double* __restrict__ dst = S + j * n;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
            dst[i] = src[i];
    }
}

// all-finite check: flag |= any non-finite entry
__global__ void nonfinite_kernel(const double* __restrict__ X, int64_t count, int* flag) {
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(X[i]);
    bad = __syncthreads_or(bad);
    if (bad && threadIdx.x == 0) atomicOr(flag, 1);
}

}  // namespace si
