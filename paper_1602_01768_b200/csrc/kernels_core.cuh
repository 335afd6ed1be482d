// K-FACTOR (fused, q ≤ 128): the whole q×q stage of one RBFGS iteration in ONE
// single-CTA launch.  From P = [G | H'] (q×2q, G = YᵀS read from its upper
// triangle as gram_llt reads the lower one of SᵀAS, H' = YᵀW' = −YᵀXY):
//
//   G⁻¹ + PD test   recursive 2×2 block (Schur-complement) inverse in shared
//                   memory; LF×LF leaves by symmetric sweeps in one warp
//                   (registers + broadcast rows, warp barriers only);
//                   the block products on the DMMA pipe (m16n8k8 .f64)
//   Ĝ = G − H'      (symmetrised), written straight from the load
//
// It replaces spd_inverse + symmetrize_small + ghat (two or three launches).
//
// PD test: block elimination meets the same Schur-complement pivots, in the
// same order, as the unblocked elimination / Cholesky; a leaf pivot that is not
// > 0 is exactly gram_llt's failure (qn_updates.cpp:37-43) and sets status[0]
// (GramRankDeficientError → redraw), after which every later launch of the
// iteration is a no-op.
//
// Block inverse of G = [[A, B], [Bᵀ, D]] (h = N/2), in place:
//   A ← A⁻¹;  T1 = A⁻¹·B;  D ← S = D − Bᵀ·T1;  D ← S⁻¹;
//   B ← −T1·S⁻¹;  A ← A⁻¹ − B·T1ᵀ (= A⁻¹ + T2·T1ᵀ);  lower-left ← Bᵀ.
#pragma once
#include "common.cuh"

namespace si {
namespace core {


// Code size matters more than anything else here: the kernel runs once per
// iteration right after the big GEMMs have flushed the instruction caches, so
// every phase is one out-of-line copy shared by all its call sites (a fully
// inlined recursion measured 139 µs in place against 72 µs with a warm cache).

// C(M×M) ∘= A(M×M)·B(M×M) on the DMMA pipe by warp tiles of (16·MI)×(8·NI)
// fragments; element (i, k) of A is A[i·asi + k·ask], B(k, j) = B[k·bsk + j·bsj],
// C(i, j) = C[i·ldc + j].  mode: 0 C = AB, 1 C −= AB, 2 C = −AB,
// 3 C −= AB and Mr(j, i) = Xs(i, j) (pitch ldm: the lower-left mirror of B).
template <int M, int NWARP>
__device__ __noinline__ void mma_phase(const double* A, int asi, int ask, const double* B, int bsk, int bsj, double* C,
                                       int ldc, int mode, double* Mr, const double* Xs, int ldm) {
    constexpr bool BIG = M >= 32 && (M / 32) * (M / 32) >= NWARP;
    constexpr int MI = BIG ? 2 : 1;
    constexpr int NI = BIG ? 4 : ((M / 16) * (M / 16) >= NWARP ? 2 : 1);
    constexpr int TM = 16 * MI, TN = 8 * NI;
    static_assert(M % TM == 0 && M % TN == 0 && M % 8 == 0, "mma_phase tiling");
    constexpr int TILES = (M / TM) * (M / TN);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    for (int tile = warp; tile < TILES; tile += NWARP) {
        const int m0 = (tile % (M / TM)) * TM, n0 = (tile / (M / TM)) * TN;
        double acc[MI][NI][4];
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;
#pragma unroll 1
        for (int kk = 0; kk < M; kk += 8) {
            double a[MI][4], b[NI][2];
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    a[i][e] = A[(m0 + i * 16 + g + ((e & 1) << 3)) * asi + (kk + t4 + ((e >> 1) << 2)) * ask];
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) b[j][e] = B[(kk + t4 + (e << 2)) * bsk + (n0 + j * 8 + g) * bsj];
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
                    const int r = m0 + i * 16 + g + ((e >> 1) << 3), c = n0 + j * 8 + 2 * t4 + (e & 1);
                    const double v = acc[i][j][e];
                    double* cp = C + r * ldc + c;
                    if (mode == 0)
                        *cp = v;
                    else if (mode == 2)
                        *cp = -v;
                    else
                        *cp -= v;
                    if (mode == 3) Mr[c * ldm + r] = Xs[r * ldm + c];
                }
    }
    __syncthreads();
}

// LF×LF leaf (row-major, pitch ld) inverted in place by one warp with the
// symmetric sweep operator (ã_kk = −1/p, ã_ik = a_ik/p, ã_ij = a_ij − a_ik·a_kj/p;
// sweeping every pivot gives −A⁻¹, and the working matrix stays symmetric): lane j
// keeps column j in registers, and since column k = row k, step k only needs every
// lane's d[k] — one shared-memory store per lane, a warp barrier and broadcast
// loads.  Row k+1 is updated and published first, so the next pivot's reciprocal
// overlaps the rest of the step.  The pivots p are the Schur-complement pivots of
// the whole matrix.
template <int LF>
__device__ __noinline__ void leaf_inverse(double* Gb, int ld, double* pp, int* s_bad) {
    static_assert(LF == 16 || LF == 32, "leaf size");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp == 0) {
        const int j = lane & (LF - 1);
        double d[LF];
#pragma unroll
        for (int i = 0; i < LF; ++i) d[i] = Gb[i * ld + j];
        bool bad = false;
        if (lane < LF) pp[lane] = d[0];
        __syncwarp();
        double inv_next = 1.0 / pp[0];
        bad |= !(pp[0] > 0.0);
#pragma unroll
        for (int k = 0; k < LF; ++k) {
            const double* buf = pp + (k & 1) * LF;
            double* nbuf = pp + ((k + 1) & 1) * LF;
            const double inv = inv_next;
            const double akj = d[k] * inv;
            if (k + 1 < LF) {
                const double r1 = buf[k + 1];
                d[k + 1] = j == k ? r1 * inv : d[k + 1] - r1 * akj;
                if (lane < LF) nbuf[lane] = d[k + 1];
                __syncwarp();
                const double piv = nbuf[k + 1];
                bad |= !(piv > 0.0);
                inv_next = 1.0 / piv;
            }
#pragma unroll
            for (int i = 0; i < LF; i += 2) {
                const double2 r = *reinterpret_cast<const double2*>(buf + i);
                const double ri[2] = {r.x, r.y};
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int ii = i + u;
                    if (ii == k)
                        d[ii] = j == k ? -inv : akj;
                    else if (ii != k + 1)
                        d[ii] = j == k ? ri[u] * inv : d[ii] - ri[u] * akj;
                }
            }
            __syncwarp();  // every lane has read buf before step k+1 overwrites it (as nbuf)
        }
        if (lane < LF) {
#pragma unroll
            for (int i = 0; i < LF; ++i) Gb[i * ld + j] = -d[i];
        }
        if (bad && lane == 0) *s_bad = 1;
    }
    __syncthreads();
}

// In-place inverse of the N×N block at (o, o); scr holds the T1 panels of this
// level and the ones below ((N/2)×(N/2+4), then (N/4)×(N/4+4), ...) and the
// leaf ping-pong rows.
template <int N, int LF, int LDG, int NW>
__device__ __forceinline__ void block_inverse(double* Gs, int o, double* scr, int* s_bad) {
    if constexpr (N <= LF) {
        leaf_inverse<N>(Gs + o * LDG + o, LDG, scr, s_bad);
    } else {
        constexpr int h = N / 2, LDT = h + 4;
        double* T1 = scr;                // h×h, pitch LDT
        double* sub = scr + h * LDT;
        double* A = Gs + o * LDG + o;   // A block; B = A + h, D = A + h·LDG + h, lower-left = A + h·LDG
        block_inverse<h, LF, LDG, NW>(Gs, o, sub, s_bad);                                     // A ← A⁻¹
        mma_phase<h, NW>(A, LDG, 1, A + h, LDG, 1, T1, LDT, 0, nullptr, nullptr, 0);           // T1 = A⁻¹·B
        mma_phase<h, NW>(A + h, 1, LDG, T1, LDT, 1, A + h * LDG + h, LDG, 1, nullptr, nullptr, 0);  // D −= Bᵀ·T1
        block_inverse<h, LF, LDG, NW>(Gs, o + h, sub, s_bad);                                 // D ← S⁻¹
        mma_phase<h, NW>(T1, LDT, 1, A + h * LDG + h, LDG, 1, A + h, LDG, 2, nullptr, nullptr, 0);  // B ← −T1·S⁻¹
        // A −= B·T1ᵀ and lower-left ← Bᵀ (mirror of the B block into A + h·LDG)
        mma_phase<h, NW>(A + h, LDG, 1, T1, 1, LDT, A, LDG, 3, A + h * LDG, A + h, LDG);
    }
}

template <int N, int LF, int LDG>
constexpr int scratch_doubles() {
    if constexpr (N <= LF)
        return 2 * N;  // leaf ping-pong rows
    else
        return (N / 2) * (N / 2 + 4) + scratch_doubles<N / 2, LF, LDG>();
}

template <int QP, int LF>
struct GramSmem {
    static constexpr int LDG = QP + 4;
    static constexpr size_t BYTES = sizeof(double) * size_t(QP * LDG + scratch_doubles<QP, LF, LDG>());
};

}  // namespace core

// One CTA of NT threads: ginv (q×q, ld q) = G⁻¹ symmetrised,
// ghat (q×q, ld q) = G − (H' + H'ᵀ)/2; status[0] = 1 when G is not PD.
template <int QP, int LF, int NT>
__global__ void __launch_bounds__(NT, 1)
    rbfgs_gram_kernel(const double* __restrict__ P, int64_t ldp, int q, double* __restrict__ ginv,
                      double* __restrict__ ghat, int* status) {
    using SM = core::GramSmem<QP, LF>;
    constexpr int LDG = SM::LDG;
    extern __shared__ __align__(16) double gsm_[];
    __shared__ int s_bad;
    griddep_wait();
    griddep_launch();
    if (*status) return;
    double* Gs = gsm_;
    double* scr = Gs + QP * LDG;
    const int tid = threadIdx.x;
    if (tid == 0) s_bad = 0;
    for (int e = tid; e < QP * QP; e += NT) {
        const int i = e % QP, j = e / QP;  // column-major walk: coalesced reads of P
        double v;
        if (i < q && j < q) {
            v = i <= j ? P[i + (int64_t)j * ldp] : P[j + (int64_t)i * ldp];
            if (ghat) ghat[i + (int64_t)j * q] = v - 0.5 * (P[i + (int64_t)(q + j) * ldp] + P[j + (int64_t)(q + i) * ldp]);
        } else {
            v = i == j ? 1.0 : 0.0;  // identity padding keeps the block SPD
        }
        Gs[i * LDG + j] = v;
    }
    __syncthreads();
    core::block_inverse<QP, LF, LDG, NT / 32>(Gs, 0, scr, &s_bad);
    __syncthreads();
    if (s_bad) {  // uniform
        if (tid == 0) *status = 1;
        return;
    }
    for (int e = tid; e < q * q; e += NT) {  // exact symmetrisation
        const int i = e % q, j = e / q;
        ginv[e] = 0.5 * (Gs[i * LDG + j] + Gs[j * LDG + i]);
    }
}

}  // namespace si
