// K-CORE (fused): the whole q×q stage of one RBFGS iteration in ONE single-CTA
// launch for q ≤ 128.  From P = [G | H] (q×2q, G = YᵀS read from its upper
// triangle as gram_llt reads the lower one of SᵀAS, H = YᵀW):
//
//   G⁻¹ + PD test          recursive 2×2 block (Schur) inverse in shared memory,
//                          leaves of LF×LF inverted by one warp in registers
//   T   = H·G⁻¹            (global scratch for q = 128, shared memory otherwise)
//   M   = [[G⁻¹ + G⁻¹·T, −G⁻¹], [−G⁻¹, 0]]   (2q×2q, ld 2q), G⁻¹ (q×q, ld q)
//
// This replaces K-FACTOR + core_layout + two q×q×q GEMM launches (five to
// seven launches, each a separate dependency step of the graph) of the
// RBFGS iteration (qn_updates.cpp:176-186 via SURVEY App. C1).
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
// Products run on the DMMA pipe (m16n8k8 .f64) with all 16 warps.
#pragma once
#include "common.cuh"

namespace si {
namespace core {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;

// C(M×N) = A(M×K)·B(K×N) by warp tiles of (16·MI)×(8·NI) fragments; operands
// come from the accessors a(i, k), b(k, j) (shared or global memory, any
// layout) and every result element is handed to epi(i, j, v).
template <int M, int N, int K, class FA, class FB, class FE>
__device__ __forceinline__ void block_mma(int warp, int lane, FA a_at, FB b_at, FE epi) {
    constexpr int MI = (M >= 32 && N >= 32 && (M / 32) * (N / 32) >= kWarps) ? 2 : 1;
    constexpr int NI = (M >= 32 && N >= 32 && (M / 32) * (N / 32) >= kWarps) ? 4 : ((M / 16) * (N / 16) >= kWarps ? 2 : 1);
    constexpr int TM = 16 * MI, TN = 8 * NI;
    static_assert(M % TM == 0 && N % TN == 0 && K % 8 == 0, "block_mma tiling");
    constexpr int TILES = (M / TM) * (N / TN);
    const int g = lane >> 2, t4 = lane & 3;
    for (int tile = warp; tile < TILES; tile += kWarps) {
        const int m0 = (tile % (M / TM)) * TM, n0 = (tile / (M / TM)) * TN;
        double acc[MI][NI][4];
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;
#pragma unroll 4
        for (int kk = 0; kk < K; kk += 8) {
            double a[MI][4], b[NI][2];
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) a[i][e] = a_at(m0 + i * 16 + g + ((e & 1) << 3), kk + t4 + ((e >> 1) << 2));
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) b[j][e] = b_at(kk + t4 + (e << 2), n0 + j * 8 + g);
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
                for (int e = 0; e < 4; ++e)
                    epi(m0 + i * 16 + g + ((e >> 1) << 3), n0 + j * 8 + 2 * t4 + (e & 1), acc[i][j][e]);
    }
}

// LF×LF leaf at (o, o) of Gs (row-major, pitch LDG) inverted in place by warp 0:
// lane j holds column j, row and column k of each Gauss-Jordan step travel by
// shuffles.  Pivots are the Schur-complement pivots of the whole matrix.
template <int LF, int LDG>
__device__ __forceinline__ void leaf_inverse(double* Gs, int o, int warp, int lane, int* s_bad) {
    if (warp == 0) {
        const int j = lane & (LF - 1);
        double d[LF];
#pragma unroll
        for (int i = 0; i < LF; ++i) d[i] = Gs[(o + i) * LDG + o + j];
        bool bad = false;
#pragma unroll
        for (int k = 0; k < LF; ++k) {
            const double piv = __shfl_sync(0xffffffffu, d[k], k);
            bad |= !(piv > 0.0);
            const double inv = 1.0 / piv;
            const double rk = d[k];
#pragma unroll
            for (int i = 0; i < LF; ++i) {
                const double cki = __shfl_sync(0xffffffffu, d[i], k);
                if (i == k)
                    d[i] = j == k ? inv : rk * inv;
                else
                    d[i] = j == k ? -cki * inv : d[i] - cki * rk * inv;
            }
        }
        if (lane < LF) {
#pragma unroll
            for (int i = 0; i < LF; ++i) Gs[(o + i) * LDG + o + j] = d[i];
        }
        if (bad && lane == 0) *s_bad = 1;
    }
    __syncthreads();
}

// In-place inverse of the N×N block at (o, o); scr holds the T1 panels of this
// level and the ones below ((N/2)×(N/2+4), then (N/4)×(N/4+4), ...).
template <int N, int LF, int LDG>
__device__ void block_inverse(double* Gs, int o, double* scr, int warp, int lane, int* s_bad) {
    if constexpr (N <= LF) {
        leaf_inverse<N, LDG>(Gs, o, warp, lane, s_bad);
    } else {
        constexpr int h = N / 2, LDT = h + 4;
        double* T1 = scr;
        double* sub = scr + h * LDT;
        block_inverse<h, LF, LDG>(Gs, o, sub, warp, lane, s_bad);  // A ← A⁻¹
        block_mma<h, h, h>(  // T1 = A⁻¹·B
            warp, lane, [&](int i, int k) { return Gs[(o + i) * LDG + o + k]; },
            [&](int k, int j) { return Gs[(o + k) * LDG + o + h + j]; },
            [&](int i, int j, double v) { T1[i * LDT + j] = v; });
        __syncthreads();
        block_mma<h, h, h>(  // D ← D − Bᵀ·T1
            warp, lane, [&](int i, int k) { return Gs[(o + k) * LDG + o + h + i]; },
            [&](int k, int j) { return T1[k * LDT + j]; },
            [&](int i, int j, double v) { Gs[(o + h + i) * LDG + o + h + j] -= v; });
        __syncthreads();
        block_inverse<h, LF, LDG>(Gs, o + h, sub, warp, lane, s_bad);  // D ← S⁻¹
        block_mma<h, h, h>(  // B ← −T1·S⁻¹
            warp, lane, [&](int i, int k) { return T1[i * LDT + k]; },
            [&](int k, int j) { return Gs[(o + h + k) * LDG + o + h + j]; },
            [&](int i, int j, double v) { Gs[(o + i) * LDG + o + h + j] = -v; });
        __syncthreads();
        block_mma<h, h, h>(  // A ← A⁻¹ − B·T1ᵀ, lower-left ← Bᵀ
            warp, lane, [&](int i, int k) { return Gs[(o + i) * LDG + o + h + k]; },
            [&](int k, int j) { return T1[j * LDT + k]; },
            [&](int i, int j, double v) {
                Gs[(o + i) * LDG + o + j] -= v;
                Gs[(o + h + j) * LDG + o + i] = Gs[(o + i) * LDG + o + h + j];
            });
        __syncthreads();
    }
}

template <int N, int LF>
constexpr int scratch_doubles() {
    if constexpr (N <= LF)
        return 0;
    else
        return (N / 2) * (N / 2 + 4) + scratch_doubles<N / 2, LF>();
}

template <int QP>
struct CoreSmem {
    static constexpr int LDG = QP + 4;
    static constexpr bool H_SMEM = QP <= 64;  // H and T in shared memory; global (L2) at QP = 128
    static constexpr int G_ELEMS = QP * LDG;
    static constexpr int HT_ELEMS = H_SMEM ? 2 * QP * LDG : 0;
    template <int LF>
    static constexpr size_t bytes() {
        return sizeof(double) * size_t(G_ELEMS + HT_ELEMS + scratch_doubles<QP, LF>());
    }
};

}  // namespace core

// One CTA of core::kThreads threads.  tg: q×q global scratch for T (used when QP = 128).
template <int QP, int LF>
__global__ void __launch_bounds__(core::kThreads, 1)
    rbfgs_core_fused_kernel(const double* __restrict__ P, int64_t ldp, int q, double* __restrict__ ginv,
                            double* __restrict__ tg, double* __restrict__ M, int* status) {
    using SM = core::CoreSmem<QP>;
    constexpr int LDG = SM::LDG;
    extern __shared__ __align__(16) double csm[];
    __shared__ int s_bad;
    if (*status) return;
    double* Gs = csm;
    double* Hs = Gs + SM::G_ELEMS;                             // H_SMEM only
    double* Ts = Hs + (SM::H_SMEM ? QP * LDG : 0);             // H_SMEM only
    double* scr = Gs + SM::G_ELEMS + SM::HT_ELEMS;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double* H = P + (int64_t)q * ldp;
    if (tid == 0) s_bad = 0;
    for (int e = tid; e < QP * QP; e += core::kThreads) {
        const int i = e % QP, j = e / QP;  // column-major walk: coalesced reads of P
        double v;
        if (i < q && j < q)
            v = i <= j ? P[i + (int64_t)j * ldp] : P[j + (int64_t)i * ldp];
        else
            v = i == j ? 1.0 : 0.0;  // identity padding keeps the block SPD
        Gs[i * LDG + j] = v;
        if constexpr (SM::H_SMEM) Hs[i * LDG + j] = (i < q && j < q) ? H[i + (int64_t)j * ldp] : 0.0;
    }
    __syncthreads();
    core::block_inverse<QP, LF, LDG>(Gs, 0, scr, warp, lane, &s_bad);
    if (s_bad) {  // uniform (read after the leaf's barrier)
        if (tid == 0) *status = 1;
        return;
    }
    // exact symmetrisation of G⁻¹ (the implied projector is symmetric); write G⁻¹
    for (int e = tid; e < QP * QP; e += core::kThreads) {
        const int i = e % QP, j = e / QP;
        if (i < j) {
            const double v = 0.5 * (Gs[i * LDG + j] + Gs[j * LDG + i]);
            Gs[i * LDG + j] = v;
            Gs[j * LDG + i] = v;
        }
    }
    __syncthreads();
    for (int e = tid; e < q * q; e += core::kThreads) {
        const int i = e % q, j = e / q;
        const double v = Gs[i * LDG + j];
        ginv[e] = v;
        M[i + (int64_t)(q + j) * (2 * q)] = -v;  // M12
        M[q + i + (int64_t)j * (2 * q)] = -v;    // M21
        M[q + i + (int64_t)(q + j) * (2 * q)] = 0.0;
    }
    // T = H·G⁻¹
    if constexpr (SM::H_SMEM) {
        core::block_mma<QP, QP, QP>(
            warp, lane, [&](int i, int k) { return Hs[i * LDG + k]; }, [&](int k, int j) { return Gs[k * LDG + j]; },
            [&](int i, int j, double v) { Ts[i * LDG + j] = v; });
    } else {
        core::block_mma<QP, QP, QP>(
            warp, lane, [&](int i, int k) { return (i < q && k < q) ? H[i + (int64_t)k * ldp] : 0.0; },
            [&](int k, int j) { return Gs[k * LDG + j]; },
            [&](int i, int j, double v) {
                if (i < q && j < q) tg[i + (int64_t)j * q] = v;
            });
    }
    __syncthreads();  // T visible to the block (shared or global)
    // M11 = G⁻¹ + G⁻¹·T
    if constexpr (SM::H_SMEM) {
        core::block_mma<QP, QP, QP>(
            warp, lane, [&](int i, int k) { return Gs[i * LDG + k]; }, [&](int k, int j) { return Ts[k * LDG + j]; },
            [&](int i, int j, double v) {
                if (i < q && j < q) M[i + (int64_t)j * (2 * q)] = Gs[i * LDG + j] + v;
            });
    } else {
        core::block_mma<QP, QP, QP>(
            warp, lane, [&](int i, int k) { return Gs[i * LDG + k]; },
            [&](int k, int j) { return (k < q && j < q) ? tg[k + (int64_t)j * q] : 0.0; },
            [&](int i, int j, double v) {
                if (i < q && j < q) M[i + (int64_t)j * (2 * q)] = Gs[i * LDG + j] + v;
            });
    }
}

}  // namespace si
