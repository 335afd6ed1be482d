// FP64 tensor-core (DMMA) GEMM engine for sm_100a.
//
// One templated mainloop serves every dense contraction on the RBFGS/AdaRBFGS
// path (SURVEY §2.4 compute-site table):
//   Y = A·S, W = X·Y, V = U·M              (EPI_STORE / EPI_PARTIAL + split-K)
//   [G | H] = Yᵀ·[S W], Z = (AS)ᵀ·L        (A operand K-major)
//   X ← X + V·Uᵀ on upper tiles, mirrored   (EPI_SYMUPD, the fused rank-2q update)
//   ‖I − A·X‖²_F partials, no n×n write     (EPI_RESID)
//
// Tiles are staged global→shared by a STAGES-deep cp.async ring (zero-filled
// out of bounds), fragments are read from padded shared memory (row pitch ≡ 4
// doubles mod 16 → conflict-free 64-bit LDS), and each warp issues
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4, measured 36.9 TFLOP/s peak on B200,
// profiles/r01_fp64_peak.txt).
#pragma once
#include "common.cuh"

namespace si {

enum Epi { EPI_STORE = 0, EPI_PARTIAL = 1, EPI_SYMUPD = 2, EPI_RESID = 3 };

struct GemmArgs {
    int64_t M, N, K;
    const double* A;
    int64_t lda;  // A_KMAJOR ? A(m,k) = A[m*lda + k] : A[m + k*lda]
    const double* B;
    int64_t ldb;  // B_KMAJOR ? B(k,n) = B[k + n*ldb] : B[n + k*ldb]
    double* C;
    int64_t ldc;  // C(m,n) = C[m + n*ldc]
    double alpha, beta;
    int64_t k_chunk;  // split-K chunk (multiple of BK); gridDim.z = #splits
    double* ws;       // EPI_PARTIAL: ws[z*M*N + m + n*M]; EPI_RESID: ws[linear block]
    const int* skip;  // if set and nonzero, the launch is a no-op (failed Gram upstream)
    int* nonfinite;   // EPI_SYMUPD: set to 1 when a written entry is not finite (simi.cpp:342-347 guard)
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool A_KMAJOR, bool B_KMAJOR>
struct GemmSmem {
    static constexpr int A_ELEMS = A_KMAJOR ? BM * (BK + 4) : BK * (BM + 4);
    static constexpr int B_ELEMS = B_KMAJOR ? BN * (BK + 4) : BK * (BN + 4);
    static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
    static constexpr size_t BYTES = size_t(STAGES) * STAGE_ELEMS * sizeof(double);
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool A_KMAJOR, bool B_KMAJOR, int VEC, int EPI>
__global__ void __launch_bounds__(WM* WN * 32) gemm_f64_kernel(GemmArgs p) {
    static_assert(BM % (WM * 8) == 0 && BN % (WN * 8) == 0, "warp tiling");
    static_assert(BK % 4 == 0 && (BK + 4) % 16 == 4 && (BM + 4) % 16 == 4 && (BN + 4) % 16 == 4, "smem pitch");
    constexpr int NT = WM * WN * 32;
    constexpr int MI = BM / WM / 8;
    constexpr int NI = BN / WN / 8;
    using SM = GemmSmem<BM, BN, BK, WM, WN, STAGES, A_KMAJOR, B_KMAJOR>;
    constexpr int LDA_S = A_KMAJOR ? BK + 4 : BM + 4;
    constexpr int LDB_S = B_KMAJOR ? BK + 4 : BN + 4;

    if (p.skip && *p.skip) return;
    extern __shared__ __align__(128) double smem[];

    // ---- tile coordinates
    int64_t tile_m, tile_n;
    if constexpr (EPI == EPI_SYMUPD) {
        // linear index over upper-triangular tile pairs (ti <= tj)
        const int64_t t = blockIdx.x;
        int64_t tj = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
        while (tj * (tj + 1) / 2 > t) --tj;
        while ((tj + 1) * (tj + 2) / 2 <= t) ++tj;
        tile_n = tj;
        tile_m = t - tj * (tj + 1) / 2;
    } else {
        tile_m = blockIdx.x;
        tile_n = blockIdx.y;
    }
    const int64_t m0 = tile_m * BM, n0 = tile_n * BN;
    const int64_t k_begin = (int64_t)blockIdx.z * p.k_chunk;
    const int64_t k_end = min(p.K, k_begin + p.k_chunk);
    const int num_kt = (int)((k_end - k_begin + BK - 1) / BK);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int wm0 = (warp / WN) * (BM / WM), wn0 = (warp % WN) * (BN / WN);

    // ---- global -> shared stage loader
    auto load_stage = [&](int stage, int kt) {
        double* As = smem + stage * SM::STAGE_ELEMS;
        double* Bs = As + SM::A_ELEMS;
        const int64_t kbase = k_begin + (int64_t)kt * BK;
        // A tile
        if constexpr (!A_KMAJOR) {  // columns of BM contiguous doubles
            constexpr int CH = BK * BM / VEC;
            for (int c = tid; c < CH; c += NT) {
                const int kk = c / (BM / VEC), mm = (c % (BM / VEC)) * VEC;
                const int64_t gm = m0 + mm, gk = kbase + kk;
                const bool ok = gm < p.M && gk < k_end;
                const double* src = ok ? p.A + gm + gk * p.lda : p.A;
                cp_async<VEC * 8>(As + kk * LDA_S + mm, src, ok);
            }
        } else {  // rows of BK contiguous doubles
            constexpr int CH = BM * BK / VEC;
            for (int c = tid; c < CH; c += NT) {
                const int mm = c / (BK / VEC), kk = (c % (BK / VEC)) * VEC;
                const int64_t gm = m0 + mm, gk = kbase + kk;
                const bool ok = gm < p.M && gk < k_end;
                const double* src = ok ? p.A + gm * p.lda + gk : p.A;
                cp_async<VEC * 8>(As + mm * LDA_S + kk, src, ok);
            }
        }
        // B tile
        if constexpr (B_KMAJOR) {  // columns n: BK contiguous doubles
            constexpr int CH = BN * BK / VEC;
            for (int c = tid; c < CH; c += NT) {
                const int nn = c / (BK / VEC), kk = (c % (BK / VEC)) * VEC;
                const int64_t gn = n0 + nn, gk = kbase + kk;
                const bool ok = gn < p.N && gk < k_end;
                const double* src = ok ? p.B + gk + gn * p.ldb : p.B;
                cp_async<VEC * 8>(Bs + nn * LDB_S + kk, src, ok);
            }
        } else {  // rows k: BN contiguous doubles
            constexpr int CH = BK * BN / VEC;
            for (int c = tid; c < CH; c += NT) {
                const int kk = c / (BN / VEC), nn = (c % (BN / VEC)) * VEC;
                const int64_t gn = n0 + nn, gk = kbase + kk;
                const bool ok = gn < p.N && gk < k_end;
                const double* src = ok ? p.B + gn + gk * p.ldb : p.B;
                cp_async<VEC * 8>(Bs + kk * LDB_S + nn, src, ok);
            }
        }
    };

    double acc[MI][NI][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < num_kt) load_stage(s, s);
        cp_async_commit();
    }

    for (int kt = 0; kt < num_kt; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int nk = kt + STAGES - 1;
            if (nk < num_kt) load_stage(nk % STAGES, nk);
            cp_async_commit();
        }
        const double* As = smem + (kt % STAGES) * SM::STAGE_ELEMS;
        const double* Bs = As + SM::A_ELEMS;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double a[MI], b[NI];
#pragma unroll
            for (int i = 0; i < MI; ++i) {
                const int m = wm0 + i * 8 + g, k = kk + t4;
                a[i] = A_KMAJOR ? As[m * LDA_S + k] : As[k * LDA_S + m];
            }
#pragma unroll
            for (int j = 0; j < NI; ++j) {
                const int n = wn0 + j * 8 + g, k = kk + t4;
                b[j] = B_KMAJOR ? Bs[n * LDB_S + k] : Bs[k * LDB_S + n];
            }
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < NI; ++j) dmma_884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
    }
    cp_async_wait<0>();

    // ---- epilogues
    if constexpr (EPI == EPI_RESID) {
        double local = 0.0;
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int64_t row = m0 + wm0 + i * 8 + g, col = n0 + wn0 + j * 8 + 2 * t4 + e;
                    if (row < p.M && col < p.N) {
                        const double d = (row == col ? 1.0 : 0.0) - acc[i][j][e];
                        local += d * d;
                    }
                }
        local = warp_sum(local);
        __shared__ double red[NT / 32];
        __syncthreads();
        if (lane == 0) red[warp] = local;
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int w = 0; w < NT / 32; ++w) s += red[w];
            p.ws[(int64_t)blockIdx.x + (int64_t)gridDim.x * ((int64_t)blockIdx.y + (int64_t)gridDim.y * blockIdx.z)] =
                s;
        }
        return;
    } else {
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int64_t row = m0 + wm0 + i * 8 + g, col = n0 + wn0 + j * 8 + 2 * t4 + e;
                    if (row >= p.M || col >= p.N) continue;
                    const double v = acc[i][j][e];
                    if constexpr (EPI == EPI_STORE) {
                        double* c = p.C + row + col * p.ldc;
                        const double nv = p.beta != 0.0 ? p.alpha * v + p.beta * *c : p.alpha * v;
                        *c = nv;
                        if (p.nonfinite && !isfinite(nv)) atomicOr(p.nonfinite, 1);
                    } else if constexpr (EPI == EPI_PARTIAL) {
                        p.ws[(int64_t)blockIdx.z * p.M * p.N + row + col * p.M] = v;
                    } else {  // EPI_SYMUPD: X(row,col) += alpha*acc on the upper triangle, mirrored
                        if (tile_m < tile_n || row <= col) {
                            double* c = p.C + row + col * p.ldc;
                            const double nv = *c + p.alpha * v;
                            *c = nv;
                            if (row != col) p.C[col + row * p.ldc] = nv;
                            if (!isfinite(nv) && p.nonfinite) atomicOr(p.nonfinite, 1);
                        }
                    }
                }
    }
}

}  // namespace si
