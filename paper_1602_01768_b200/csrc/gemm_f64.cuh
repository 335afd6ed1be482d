// FP64 tensor-core (DMMA) GEMM engine for sm_100a.
//
// One templated tile engine serves every dense contraction on the RBFGS /
// AdaRBFGS path (SURVEY §2.4 compute-site table):
//   Y = A·S, W = X·Y, V = U·M              (EPI_STORE / EPI_PARTIAL + split-K)
//   [G | H] = Yᵀ·[S W], Z = (AS)ᵀ·L        (A operand K-major)
//   X ← X + V·Uᵀ on upper tiles, mirrored   (EPI_SYMUPD, the fused rank-2q update)
//   ‖I − A·X‖²_F partials, no n×n write     (EPI_RESID)
//
// Two mainloops feed the same warp tiles:
//   gemm_tma_kernel  — Blackwell path: one elected thread issues TMA
//                      (cp.async.bulk.tensor) boxes into a STAGES-deep ring
//                      guarded by mbarriers (full / empty); the WM×WN warps
//                      never block on a CTA-wide barrier.  Boxes are 4
//                      doubles wider than the tile so shared memory keeps a
//                      pitch ≡ 4 (mod 16) doubles → conflict-free 64-bit LDS.
//   gemm_f64_kernel  — cp.async ring for operands TMA cannot describe (odd
//                      leading dimensions / unaligned bases).
// Warps issue mma.sync.aligned.m16n8k8.f64 (SASS DMMA.8x8x4; measured FP64
// DMMA peak 36.9 TFLOP/s on B200, profiles/r01_fp64_peak.txt).
#pragma once
#include <cuda.h>

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
    int* nonfinite;   // STORE / SYMUPD: set to 1 when a written entry is not finite (simi.cpp:342-347)
    int64_t diag_off; // RESID: the identity's diagonal is at (r, r + diag_off) (row panels of a sharded X)
    int c_in_acc;     // STORE: accumulators start from beta·C (set by the host when alpha == 1, beta != 0);
                      // RESID: from beta·C (the A + P·Uᵀ form of the first checkpoint)
    const double* Csrc;  // STORE: beta·Csrc(m,n) (ld ldc) instead of beta·C — out-of-place C = alpha·A·B + beta·Csrc
    int dbg;          // SYMUPD experiments (SI_SYMUPD_DBG): 1 = no stores, 2 = no C loads, 4 = no C prefetch
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool A_KMAJOR, bool B_KMAJOR>
struct GemmSmem {
    static constexpr int A_ELEMS = A_KMAJOR ? BM * (BK + 4) : BK * (BM + 4);
    static constexpr int B_ELEMS = B_KMAJOR ? BN * (BK + 4) : BK * (BN + 4);
    static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
    static constexpr size_t BYTES = size_t(STAGES) * STAGE_ELEMS * sizeof(double);
    static constexpr size_t BAR_OFFSET = (BYTES + 127) / 128 * 128;
    static constexpr size_t TMA_BYTES = BAR_OFFSET + 2 * STAGES * sizeof(uint64_t);
};

// Shared per-tile logic of both mainloops.
template <int BM, int BN, int BK, int WM, int WN, bool A_KMAJOR, bool B_KMAJOR, int EPI>
struct TileOps {
    static constexpr int MI = BM / WM / 16;  // m16 blocks per warp
    static constexpr int NI = BN / WN / 8;   // n8 blocks per warp
    static constexpr int LDA_S = A_KMAJOR ? BK + 4 : BM + 4;
    static constexpr int LDB_S = B_KMAJOR ? BK + 4 : BN + 4;
    static_assert(BM % (WM * 16) == 0 && BN % (WN * 8) == 0, "warp tiling");
    static_assert(BK % 8 == 0 && (BM + 4) % 16 == 4 && (BN + 4) % 16 == 4, "smem pitch");
    static_assert((!A_KMAJOR && !B_KMAJOR) || (BK + 4) % 16 == 4, "smem pitch (K-major operands)");

    int64_t m0, n0, tile_m, tile_n, split;
    int g, t4, wm0, wn0;

    // Work item w of a launch: SYMUPD enumerates upper-triangular tile pairs
    // (ti <= tj); otherwise w = tile_m + tm·(tile_n + tn·split).
    struct Work {
        int64_t tile_m, tile_n, split;
    };
    // SYMUPD tiles: BM×BN blocks (BM = R·BN) that meet the upper triangle.  Column
    // block tn needs row blocks 0..tn/R, so column chunk c (R column blocks) holds
    // R·(c+1) tiles and chunks 0..c−1 hold R·c(c+1)/2; w runs row blocks fastest.
    // (the host launches SYMUPD only with BM a multiple of BN)
    static constexpr int R_SYM = BM % BN == 0 ? BM / BN : 1;
    __host__ __device__ __forceinline__ static int64_t sym_work_count(int64_t n) {
        const int64_t tn = (n + BN - 1) / BN;
        const int64_t full = tn / R_SYM, rest = tn % R_SYM;  // complete chunks, columns of the last one
        return R_SYM * full * (full + 1) / 2 + rest * (full + 1);
    }
    // 32-bit integer arithmetic and an fp32 square-root estimate (exact after the ±1
    // integer correction): the per-tile decode runs on every work item of a
    // persistent CTA, where FP64 sqrt and 64-bit divisions were measurable
    __device__ __forceinline__ static void sym_tile(int64_t w64, int64_t& tile_m, int64_t& tile_n) {
        const uint32_t w = (uint32_t)w64;
        uint32_t c = (uint32_t)((sqrtf(8.0f * (float)w / (float)R_SYM + 1.0f) - 1.0f) * 0.5f);
        while (c > 0 && (uint32_t)R_SYM * c * (c + 1) / 2 > w) --c;
        while ((uint32_t)R_SYM * (c + 1) * (c + 2) / 2 <= w) ++c;
        const uint32_t rem = w - (uint32_t)R_SYM * c * (c + 1) / 2;
        tile_n = (int64_t)(c * R_SYM + rem / (c + 1));
        tile_m = (int64_t)(rem % (c + 1));
    }
    // Trapezoid SYMUPD (M < N: the rows [0, M) of a symmetric block's row panel, X[R, r0:],
    // the sharded driver's chunk): the upper tiles of the leading M×M block (mirrored inside
    // it), then every tile of the columns right of it (no mirror)
    __host__ __device__ __forceinline__ static int64_t sym_trap_count(int64_t M, int64_t N) {
        const int64_t tmM = (M + BM - 1) / BM, tnM = (M + BN - 1) / BN, tn = (N + BN - 1) / BN;
        return sym_work_count(M) + (tn - tnM) * tmM;
    }
    __device__ __forceinline__ static Work decode(int64_t w, const GemmArgs& p) {
        Work r;
        if constexpr (EPI == EPI_SYMUPD) {
            const int64_t wsq = p.M < p.N ? sym_work_count(p.M) : INT64_MAX;
            if (w < wsq) {
                sym_tile(w, r.tile_m, r.tile_n);
            } else {
                const int64_t tmM = (p.M + BM - 1) / BM, tnM = (p.M + BN - 1) / BN, v = w - wsq;
                r.tile_m = v % tmM;
                r.tile_n = tnM + v / tmM;
            }
            r.split = 0;
        } else {
            const uint32_t tm = (uint32_t)((p.M + BM - 1) / BM), tn = (uint32_t)((p.N + BN - 1) / BN);
            const uint32_t w32 = (uint32_t)w, q1 = w32 / tm;
            r.tile_m = w32 - q1 * tm;
            r.tile_n = q1 % tn;
            r.split = q1 / tn;
        }
        return r;
    }
    __device__ __forceinline__ static int64_t work_count(const GemmArgs& p) {
        const int64_t tm = (p.M + BM - 1) / BM, tn = (p.N + BN - 1) / BN;
        if constexpr (EPI == EPI_SYMUPD) return p.M < p.N ? sym_trap_count(p.M, p.N) : sym_work_count(p.N);
        return tm * tn * ((p.K + p.k_chunk - 1) / p.k_chunk > 0 ? (p.K + p.k_chunk - 1) / p.k_chunk : 1);
    }
    __device__ __forceinline__ void setup_work(int64_t w, const GemmArgs& p, int warp, int lane) {
        const Work r = decode(w, p);
        tile_m = r.tile_m;
        tile_n = r.tile_n;
        split = r.split;
        m0 = tile_m * BM;
        n0 = tile_n * BN;
        g = lane >> 2;
        t4 = lane & 3;
        wm0 = (warp / WN) * (BM / WM);
        wn0 = (warp % WN) * (BN / WN);
    }

    __device__ __forceinline__ void setup(int warp, int lane, const GemmArgs& p) {
        if constexpr (EPI == EPI_SYMUPD) {
            const Work r = decode(blockIdx.x, p);
            tile_m = r.tile_m;
            tile_n = r.tile_n;
        } else {
            tile_m = blockIdx.x;
            tile_n = blockIdx.y;
        }
        split = blockIdx.z;
        m0 = tile_m * BM;
        n0 = tile_n * BN;
        g = lane >> 2;
        t4 = lane & 3;
        wm0 = (warp / WN) * (BM / WM);
        wn0 = (warp % WN) * (BN / WN);
    }

    // L2 prefetch of this thread's part of a C tile (the next work item's X block)
    __device__ __forceinline__ void prefetch_c(const GemmArgs& p) const {
        const double* src = (EPI == EPI_STORE && p.Csrc) ? p.Csrc : p.C;
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j) {
                const int64_t r = row(i, 0), c = col(j, 0);
                if (r < p.M && c < p.N) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(src + r + c * p.ldc));
                if (r < p.M && c + 1 < p.N)
                    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(src + r + (c + 1) * p.ldc));
            }
    }
    // fragment element e of block (i, j) sits at (wm0 + 16i + g + 8(e>>1), wn0 + 8j + 2t + (e&1))
    __device__ __forceinline__ int64_t row(int i, int e) const { return m0 + wm0 + i * 16 + g + ((e >> 1) << 3); }
    __device__ __forceinline__ int64_t col(int j, int e) const { return n0 + wn0 + j * 8 + 2 * t4 + (e & 1); }

    // STORE with alpha = 1 and beta ≠ 0 also starts from C (p.c_in_acc)
    __device__ __forceinline__ bool c_in_acc(const GemmArgs& p) const {
        if constexpr (EPI == EPI_SYMUPD) return true;
        if constexpr (EPI == EPI_STORE || EPI == EPI_RESID) return p.c_in_acc != 0;
        return false;
    }

    __device__ __forceinline__ void init_acc(double (&acc)[MI][NI][4], const GemmArgs& p) const {
        if (c_in_acc(p) && !(EPI == EPI_SYMUPD && (p.dbg & 2))) {
            // accumulate onto the C tile itself (C = beta·C + A·B with alpha = 1; for
            // SYMUPD X + V·Uᵀ): the loads are issued under the pipeline fill and the
            // epilogue becomes store-only
            const double b = EPI == EPI_SYMUPD ? 1.0 : p.beta;
            const double* src = (EPI == EPI_STORE && p.Csrc) ? p.Csrc : p.C;
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < NI; ++j)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int64_t r = row(i, e), c = col(j, e);
                        if constexpr (EPI == EPI_SYMUPD)  // SI_SYMUPD_DBG & 64: streaming (evict-first) X loads and stores
                            acc[i][j][e] = (r < p.M && c < p.N) ? ((p.dbg & 64) ? __ldcs(src + r + c * p.ldc) : src[r + c * p.ldc]) : 0.0;
                        else
                            acc[i][j][e] = (r < p.M && c < p.N) ? b * src[r + c * p.ldc] : 0.0;
                    }
        } else {
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < NI; ++j)
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;
        }
    }

    __device__ __forceinline__ void compute_stage(double (&acc)[MI][NI][4], const double* As, const double* Bs) const {
        compute_part<0, BK>(acc, As, Bs);
    }
    // the k8 steps [K0, K1) of a stage
    template <int K0, int K1>
    __device__ __forceinline__ void compute_part(double (&acc)[MI][NI][4], const double* As, const double* Bs) const {
#pragma unroll
        for (int kk = K0; kk < K1; kk += 8) {
            double a[MI][4], b[NI][2];
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int m = wm0 + i * 16 + g + ((e & 1) << 3), k = kk + t4 + ((e >> 1) << 2);
                    a[i][e] = A_KMAJOR ? As[m * LDA_S + k] : As[k * LDA_S + m];
                }
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int n = wn0 + j * 8 + g, k = kk + t4 + (e << 2);
                    b[j][e] = B_KMAJOR ? Bs[n * LDB_S + k] : Bs[k * LDB_S + n];
                }
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < NI; ++j) dmma_1688(acc[i][j], a[i], b[j]);
        }
    }

    // `sync_consumers` synchronises exactly the threads that hold accumulators
    template <class Sync>
    __device__ __forceinline__ void epilogue(const double (&acc)[MI][NI][4], const GemmArgs& p, int tid, int nthreads,
                                             Sync sync_consumers) const {
        if constexpr (EPI == EPI_RESID) {
            double local = 0.0;
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < NI; ++j)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int64_t r = row(i, e), c = col(j, e);
                        if (r < p.M && c < p.N) {
                            const double d = (r + p.diag_off == c ? 1.0 : 0.0) - p.alpha * acc[i][j][e];
                            local += d * d;
                        }
                    }
            local = warp_sum(local);
            __shared__ double red[32];
            const int lane = tid & 31, w = tid >> 5;
            if (lane == 0) red[w] = local;
            sync_consumers();
            if (tid == 0) {
                double s = 0.0;
                for (int k = 0; k < nthreads / 32; ++k) s += red[k];
                p.ws[tile_m + ((p.M + BM - 1) / BM) * (tile_n + ((p.N + BN - 1) / BN) * split)] = s;
            }
            sync_consumers();  // `red` is reused by the next work item of a persistent CTA
        } else {
            if constexpr (EPI == EPI_SYMUPD) {
                // off-diagonal full tiles: the mirror X(c, r), X(c+1, r) of the fragment
                // pair (r, c), (r, c+1) is one aligned 16-byte store
                const bool fast = m0 + BM <= n0 && m0 + BM <= p.M && n0 + BN <= p.M && (p.ldc & 1) == 0 &&
                                  (reinterpret_cast<uintptr_t>(p.C) & 15) == 0;
                if (n0 >= p.M && m0 + BM <= p.M && n0 + BN <= p.N) {  // trapezoid columns right of the block
                    bool bad = false;
#pragma unroll
                    for (int i = 0; i < MI; ++i)
#pragma unroll
                        for (int j = 0; j < NI; ++j)
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const int64_t r = row(i, e), c = col(j, e);
                                p.C[r + c * p.ldc] = acc[i][j][e];
                                bad |= !isfinite(acc[i][j][e]);
                            }
                    if (bad && p.nonfinite) atomicOr(p.nonfinite, 1);
                    return;
                }
                if (fast && (p.dbg & 1)) {  // experiment: keep the accumulators live, store nothing
                    double t = 0.0;
#pragma unroll
                    for (int i = 0; i < MI; ++i)
#pragma unroll
                        for (int j = 0; j < NI; ++j)
#pragma unroll
                            for (int e = 0; e < 4; ++e) t += acc[i][j][e];
                    if (t == 1.2345e300) p.C[0] = t;
                    return;
                }
                if (fast) {
                    bool bad = false;
#pragma unroll
                    for (int i = 0; i < MI; ++i)
#pragma unroll
                        for (int j = 0; j < NI; ++j)
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const int64_t r = row(i, 2 * h), c = col(j, 2 * h);
                                const double v0 = acc[i][j][2 * h], v1 = acc[i][j][2 * h + 1];
                                if (!(p.dbg & 64)) {
                                    p.C[r + c * p.ldc] = v0;
                                    p.C[r + (c + 1) * p.ldc] = v1;
                                    *reinterpret_cast<double2*>(p.C + c + r * p.ldc) = make_double2(v0, v1);
                                } else {  // experiment: DRAM reads 1.42 -> 1.26 GB per launch at config 3, 0.5% slower
                                    __stcs(p.C + r + c * p.ldc, v0);
                                    __stcs(p.C + r + (c + 1) * p.ldc, v1);
                                    __stcs(reinterpret_cast<double2*>(p.C + c + r * p.ldc), make_double2(v0, v1));
                                }
                                bad |= !isfinite(v0) || !isfinite(v1);
                            }
                    if (bad && p.nonfinite) atomicOr(p.nonfinite, 1);
                    return;
                }
            }
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < NI; ++j)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int64_t r = row(i, e), c = col(j, e);
                        if (r >= p.M || c >= p.N) continue;
                        const double v = acc[i][j][e];
                        if constexpr (EPI == EPI_STORE) {
                            double* cp = p.C + r + c * p.ldc;
                            const double* cs = p.Csrc ? p.Csrc + r + c * p.ldc : cp;
                            const double nv = p.c_in_acc ? v : (p.beta != 0.0 ? p.alpha * v + p.beta * *cs : p.alpha * v);
                            *cp = nv;
                            if (p.nonfinite && !isfinite(nv)) atomicOr(p.nonfinite, 1);
                        } else if constexpr (EPI == EPI_PARTIAL) {
                            p.ws[split * p.M * p.N + r + c * p.M] = v;
                        } else {  // EPI_SYMUPD: X(r,c) = acc (= X + V·Uᵀ) on the upper triangle, mirrored
                            if (r <= c) {
                                p.C[r + c * p.ldc] = v;
                                if (r != c && c < p.M) p.C[c + r * p.ldc] = v;
                                if (!isfinite(v) && p.nonfinite) atomicOr(p.nonfinite, 1);
                            }
                        }
                    }
        }
    }
};

// --------------------------------------------------------------- TMA path --
// Persistent: gridDim.x CTAs stride over the launch's work items (tiles ×
// split-K chunks; upper-triangular tile pairs for SYMUPD).  Threads: WM·WN
// warps, all of them compute.  Lane 0 of warp 0 is also the TMA producer: it
// keeps STAGES−1 k-stages in flight *across work-item boundaries*, so the next
// tile's operands stream in while the current tile finishes and stores, arming
// full[s] with the stage's byte count and issuing one box for A and one for B.
// Every warp waits on full[s], computes, and arrives on empty[s] (count WM·WN);
// the producer waits on empty[s] only before refilling that slot — no CTA-wide
// barrier in the mainloop.  Each CTA also prefetches the next tile's C block to
// L2 when the epilogue will read it.  (A separate producer warp would cost a
// whole warpgroup of registers: ptxas allocates in 4-warp units.)
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool A_KMAJOR, bool B_KMAJOR, int EPI>
__global__ void __launch_bounds__(WM* WN * 32, ((EPI == EPI_SYMUPD || EPI == EPI_STORE) && BM == 128 && BN == 64) ? 2 : 1)
    gemm_tma_persistent_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                               GemmArgs p) {
    using SM = GemmSmem<BM, BN, BK, WM, WN, STAGES, A_KMAJOR, B_KMAJOR>;
    using T = TileOps<BM, BN, BK, WM, WN, A_KMAJOR, B_KMAJOR, EPI>;
    constexpr int NW = WM * WN;
    constexpr uint32_t STAGE_BYTES = SM::STAGE_ELEMS * sizeof(double);

    extern __shared__ __align__(128) double smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + SM::BAR_OFFSET);
    uint64_t* empty = full + STAGES;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool producer = tid == 0;
    if (producer) {  // prologue before the dependency wait (overlaps the predecessor's tail under PDL)
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        mbar_fence_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    griddep_wait();
    griddep_launch();
    if (p.skip && *p.skip) return;
    const int64_t W = T::work_count(p);
    auto chunk_kt = [&](int64_t split) {
        const int64_t kb = split * p.k_chunk;
        return (int)((min(p.K, kb + p.k_chunk) - kb + BK - 1) / BK);
    };

    // producer cursor: work item pw, k-stage pk within it, ring slot ps with its
    // use count (parity) — 32-bit incremental counters keep the issue path short
    int64_t pw = blockIdx.x;
    int pk = 0, ps = 0, pround = 0, pissued = 0;
    typename T::Work pwork{};
    int pnk = 0;
    const uint64_t keep = EPI == EPI_SYMUPD ? l2_policy_evict_last() : 0;
    if (producer && pw < W) {
        pwork = T::decode(pw, p);
        pnk = chunk_kt(pwork.split);
    }
    auto issue_next = [&]() {  // issue the next stage for (pw, pk) and advance the cursor
        const int s = ps;
        if (pround > 0) mbar_wait(&empty[s], (uint32_t)((pround - 1) & 1));
        double* As = smem + s * SM::STAGE_ELEMS;
        double* Bs = As + SM::A_ELEMS;
        const int32_t kc = (int32_t)(pwork.split * p.k_chunk + (int64_t)pk * BK);
        const int32_t mc = (int32_t)(pwork.tile_m * BM), nc = (int32_t)(pwork.tile_n * BN);
        mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
        if (EPI == EPI_SYMUPD && !A_KMAJOR && !B_KMAJOR && !(p.dbg & 32)) {
            // the rank-2q panels are re-read by every tile of their block row / column while 4 GB of
            // X stream through the L2: keep them (evict-last; DRAM reads 1.63 -> 1.42 GB per launch at
            // config 3, time unchanged; SI_SYMUPD_DBG & 32 turns the hint off)
            tma_load_2d_hint(As, &tmA, mc, kc, &full[s], keep);
            tma_load_2d_hint(Bs, &tmB, nc, kc, &full[s], keep);
        } else {
            if constexpr (A_KMAJOR)
                tma_load_2d(As, &tmA, kc, mc, &full[s]);
            else
                tma_load_2d(As, &tmA, mc, kc, &full[s]);
            if constexpr (B_KMAJOR)
                tma_load_2d(Bs, &tmB, kc, nc, &full[s]);
            else
                tma_load_2d(Bs, &tmB, nc, kc, &full[s]);
        }
        ++pissued;
        if (++ps == STAGES) {
            ps = 0;
            ++pround;
        }
        if (++pk == pnk) {
            pk = 0;
            pw += gridDim.x;
            if (pw < W) {
                pwork = T::decode(pw, p);
                pnk = chunk_kt(pwork.split);
            }
        }
    };
    // keep the producer STAGES−1 stages ahead of consumer stage cg
    auto pump = [&](int cg) {
        while (pw < W && pissued < cg + STAGES - 1) issue_next();
    };

    __syncthreads();
    if (producer) pump(0);

    T t;
    int cg = 0, cs = 0;
    uint32_t cphase = 0;
    for (int64_t w = blockIdx.x; w < W; w += gridDim.x) {
        t.setup_work(w, p, warp, lane);
        const int nk = chunk_kt(t.split);
        double acc[T::MI][T::NI][4];
        t.init_acc(acc, p);
        for (int kt = 0; kt < nk; ++kt, ++cg) {
            if (warp == 0) {
                if (producer) pump(cg);
                __syncwarp();
            }
            const int s = cs;
            mbar_wait(&full[s], cphase);
            if (++cs == STAGES) {
                cs = 0;
                cphase ^= 1u;
            }
            const double* As = smem + s * SM::STAGE_ELEMS;
            t.compute_stage(acc, As, As + SM::A_ELEMS);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (kt == nk - 1 && w + gridDim.x < W && t.c_in_acc(p) && !(EPI == EPI_SYMUPD && (p.dbg & 4))) {
                T nt = t;  // warm L2 with the next tile's C block before its init_acc
                nt.setup_work(w + gridDim.x, p, warp, lane);
                nt.prefetch_c(p);
            }
        }
        t.epilogue(acc, p, tid, NW * 32, [] { __syncthreads(); });
    }
}

// ------------------------------------------- warp-specialised K-SYMUPD --
// X ← X + V·Uᵀ on the upper BM×BN tiles, mirrored (the fused rank-2q update), with the
// tile epilogue taken off the DMMA warps.  Warps 0..7 only compute: they run the TMA-fed
// mainloop from zero accumulators, drop the accumulators into a shared-memory hand-off
// buffer (interleaved by thread: conflict-free on both sides) and go straight on to their
// next tile.  Warps 8..11 are memory warps: lane 0 of warp 8 issues the TMA operand stages
// (running ahead across tiles, polled between epilogue chunks), and the four warps retire
// the previous tile — its X block is prefetched to L2 while the tile is computed, then each
// memory warp adds X to two compute warps' fragments and writes them and their mirror (8-byte
// stores down a column, 16-byte stores along the mirror row: full sectors) — so the X read
// and the 2·BM·BN·8-byte write of a tile overlap the next tile's DMMA work instead of
// stalling it (the ≈ 2.9 µs per tile of the single-role kernel).  Registers are granted in
// 4-warp units, so the 4 memory warps cost no more than 1 (12 warps × 168 ≤ 65 536).
template <int BM, int BN, int BK, int STAGES>
struct SymWsSmem {
    static constexpr int A_ELEMS = BK * (BM + 4);
    static constexpr int B_ELEMS = BK * (BN + 4);
    static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
    static constexpr int HAND_ELEMS = BM * BN;
    static constexpr size_t HAND_OFFSET = size_t(STAGES) * STAGE_ELEMS * sizeof(double);
    static constexpr size_t BAR_OFFSET = (HAND_OFFSET + size_t(HAND_ELEMS) * sizeof(double) + 127) / 128 * 128;
    static constexpr size_t BYTES = BAR_OFFSET + (2 * STAGES + 2) * sizeof(uint64_t);
    static constexpr int MEM_WARPS = 4;
};

// 12 warps at ≤ 168 registers (__maxnreg__; the compute warps need ≈ 166 without the epilogue)
template <int BM, int BN, int BK, int WM, int WN, int STAGES>
__global__ void __maxnreg__(168)
    gemm_symupd_ws_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs p) {
    using SM = SymWsSmem<BM, BN, BK, STAGES>;
    using T = TileOps<BM, BN, BK, WM, WN, false, false, EPI_SYMUPD>;
    constexpr int NW = WM * WN;            // compute warps
    constexpr int NC = NW * 32;            // compute threads
    constexpr int NMEM = SM::MEM_WARPS;    // memory warps
    constexpr uint32_t STAGE_BYTES = SM::STAGE_ELEMS * sizeof(double);

    extern __shared__ __align__(128) double smem[];
    double* hand = smem + size_t(STAGES) * SM::STAGE_ELEMS;
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + SM::BAR_OFFSET);
    uint64_t* empty = full + STAGES;
    uint64_t* hfull = empty + STAGES;  // compute warps → memory warps (count NW)
    uint64_t* hfree = hfull + 1;       // memory warps → compute warps (count NMEM)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == NC) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        mbar_init(hfull, NW);
        mbar_init(hfree, NMEM);
        mbar_fence_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    griddep_wait();
    griddep_launch();
    if (p.skip && *p.skip) return;
    const int64_t W = T::sym_work_count(p.N);
    const int nk = (int)((p.K + BK - 1) / BK);
    __syncthreads();

    if (warp < NW) {  // ---------------------------------------- compute warps
        T t;
        int cs = 0;
        uint32_t cphase = 0;
        int tiles = 0;
        for (int64_t w = blockIdx.x; w < W; w += gridDim.x, ++tiles) {
            t.setup_work(w, p, warp, lane);
            double acc[T::MI][T::NI][4];
#pragma unroll
            for (int i = 0; i < T::MI; ++i)
#pragma unroll
                for (int j = 0; j < T::NI; ++j)
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;
            for (int kt = 0; kt < nk; ++kt) {
                const int s = cs;
                mbar_wait(&full[s], cphase);
                if (++cs == STAGES) {
                    cs = 0;
                    cphase ^= 1u;
                }
                const double* As = smem + s * SM::STAGE_ELEMS;
                t.compute_stage(acc, As, As + SM::A_ELEMS);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
            if (tiles > 0) mbar_wait(hfree, (uint32_t)((tiles - 1) & 1));  // the previous tile is retired
#pragma unroll
            for (int i = 0; i < T::MI; ++i)
#pragma unroll
                for (int j = 0; j < T::NI; ++j)
#pragma unroll
                    for (int e = 0; e < 4; ++e) hand[((i * T::NI + j) * 4 + e) * NC + tid] = acc[i][j][e];
            __syncwarp();
            if (lane == 0) mbar_arrive(hfull);
        }
        return;
    }

    // ------------------------------------------------------------ memory warps
    const int mw = warp - NW;
    const bool producer = mw == 0 && lane == 0;
    int64_t pw = blockIdx.x;
    int pk = 0, ps = 0, pround = 0;
    int64_t ptm = 0, ptn = 0;
    if (pw < W) T::sym_tile(pw, ptm, ptn);
    // issue every stage whose slot is free, never blocking (polled between epilogue rounds)
    auto pump = [&](bool block) {
        while (pw < W) {
            const int s = ps;
            if (pround > 0) {
                if (block)
                    mbar_wait(&empty[s], (uint32_t)((pround - 1) & 1));
                else if (!mbar_try_wait(&empty[s], (uint32_t)((pround - 1) & 1)))
                    return;
            }
            double* As = smem + s * SM::STAGE_ELEMS;
            double* Bs = As + SM::A_ELEMS;
            const int32_t kc = (int32_t)(pk * BK);
            mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
            tma_load_2d(As, &tmA, (int32_t)(ptm * BM), kc, &full[s]);
            tma_load_2d(Bs, &tmB, (int32_t)(ptn * BN), kc, &full[s]);
            if (++ps == STAGES) {
                ps = 0;
                ++pround;
            }
            if (++pk == nk) {
                pk = 0;
                pw += gridDim.x;
                if (pw < W) T::sym_tile(pw, ptm, ptn);
            }
            block = false;
        }
    };
    if (producer) pump(false);
    __syncwarp();
    int tiles = 0;
    for (int64_t w = blockIdx.x; w < W; w += gridDim.x, ++tiles) {
        int64_t tm, tn;
        T::sym_tile(w, tm, tn);
        const int64_t m0 = tm * BM, n0 = tn * BN;
        {  // the tile's X block to L2 while it is computed: one prefetch per 128-byte line
            constexpr int LINES = BN * (BM / 16);  // 16 doubles per line
            for (int l = mw * 32 + lane; l < LINES; l += NMEM * 32) {
                const int64_t c = n0 + l / (BM / 16), r = m0 + (l % (BM / 16)) * 16;
                if (r < p.M && c < p.N) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p.C + r + c * p.ldc));
            }
        }
        // wait for the compute warps' hand-off, keeping the operand ring fed meanwhile
        for (;;) {
            if (producer) pump(false);
            if (mbar_try_wait(hfull, (uint32_t)(tiles & 1))) break;
        }
        __syncwarp();
        const bool fast = m0 + BM <= n0 && m0 + BM <= p.M && n0 + BN <= p.N && (p.ldc & 1) == 0 &&
                          (reinterpret_cast<uintptr_t>(p.C) & 15) == 0;
        bool bad = false;
        for (int cw = mw; cw < NW; cw += NMEM) {  // retire compute warp cw's fragments as its lane would
            const int ct = cw * 32 + lane;
            const int g = lane >> 2, t4 = lane & 3;
            const int64_t wm0 = (cw / WN) * (BM / WM), wn0 = (cw % WN) * (BN / WN);
#pragma unroll 1
            for (int i = 0; i < T::MI; ++i) {  // one m16 row block at a time: 4·NI values in flight
                const int64_t rb = m0 + wm0 + i * 16 + g;
                const int64_t cb = n0 + wn0 + 2 * t4;
                const double* xc = p.C + rb + cb * p.ldc;
                double x[T::NI * 4];
#pragma unroll
                for (int j = 0; j < T::NI; ++j)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int64_t r = rb + ((e >> 1) << 3), c = cb + j * 8 + (e & 1);
                        x[j * 4 + e] = (fast || (r < p.M && c < p.N))
                                           ? xc[((e >> 1) << 3) + (j * 8 + (e & 1)) * p.ldc]
                                           : 0.0;
                    }
#pragma unroll
                for (int j = 0; j < T::NI; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int f = (i * T::NI + j) * 4 + 2 * h;
                        const double v0 = x[j * 4 + 2 * h] + hand[f * NC + ct];
                        const double v1 = x[j * 4 + 2 * h + 1] + hand[(f + 1) * NC + ct];
                        const int64_t r = rb + (h << 3), c = cb + j * 8;
                        bad |= !isfinite(v0) || !isfinite(v1);
                        if (fast) {
                            double* d = p.C + r + c * p.ldc;
                            d[0] = v0;
                            d[p.ldc] = v1;
                            *reinterpret_cast<double2*>(p.C + c + r * p.ldc) = make_double2(v0, v1);
                        } else {
                            if (r < p.M && c < p.N && r <= c) {
                                p.C[r + c * p.ldc] = v0;
                                if (r != c) p.C[c + r * p.ldc] = v0;
                            }
                            if (r < p.M && c + 1 < p.N && r <= c + 1) {
                                p.C[r + (c + 1) * p.ldc] = v1;
                                if (r != c + 1) p.C[c + 1 + r * p.ldc] = v1;
                            }
                        }
                    }
            }
            if (producer) pump(false);
            __syncwarp();
        }
        if (bad && p.nonfinite) atomicOr(p.nonfinite, 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(hfree);
    }
}

// ------------------------------------------- deferred-epilogue K-SYMUPD --
// X ← X + V·Uᵀ on the upper BM×BN tiles, mirrored, with the tile epilogue folded into the
// NEXT tile's mainloop and the X read-modify-write done by the L2 (red.global.add.f64).
// In the single-role kernel all 8 warps reach the epilogue together: 64 X loads and 96 stores
// per thread go through the LSU while the DMMA pipe idles (≈ 2–3 µs of a 36 µs tile).  Here
// the accumulators start from zero; a finished tile's fragment blocks are dropped into a
// shared-memory hand-off area — thread-interleaved, so every thread only ever reads back its
// own slots: no barrier, no bank conflict — and the warps start the next tile at once.  After
// each k8 step of that tile a thread retires one 16×8 fragment block of the previous one:
// eight fire-and-forget reductions, X(r, c) += v on the tile and X(c, r) += v on its mirror.
// Both halves start bitwise equal and receive the same addend, so X stays exactly symmetric;
// every element receives exactly one addend per launch, so the result is deterministic and
// rounded once (X + Σ instead of a running sum seeded with X).  No X value ever enters a
// register: register loads of X measured +0.6 ms per launch at config 3 (their scoreboard
// is shared with the fragment loads, so every DMMA waited on L2), cp.async staging +0.19 ms,
// the reductions +0.06 ms.  HB = fragment blocks handed off per thread (of MI·NI); the
// remaining blocks are retired from registers at the hand-off.  HB = 15 of 16 leaves room
// for three BK = 16 stages beside the 120 KB hand-off area (BK = 8 × 5 stages with all 16
// blocks measured 15% slower in the mainloop).  Diagonal and ragged tiles take a guarded
// load-add-store epilogue.
template <int BM, int BN, int BK, int WM, int WN, int STAGES, int HB>
struct SymDefSmem {
    static constexpr int A_ELEMS = BK * (BM + 4);
    static constexpr int B_ELEMS = BK * (BN + 4);
    static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
    static constexpr size_t HAND_OFFSET = size_t(STAGES) * STAGE_ELEMS * sizeof(double);
    static constexpr size_t HAND_BYTES = size_t(HB) * 4 * WM * WN * 32 * sizeof(double);
    static constexpr size_t BAR_OFFSET = (HAND_OFFSET + HAND_BYTES + 127) / 128 * 128;
    static constexpr size_t BYTES = BAR_OFFSET + 2 * STAGES * sizeof(uint64_t);
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int HB>
__global__ void __launch_bounds__(WM* WN * 32, 1)
    gemm_symupd_deferred_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                                GemmArgs p) {
    using SM = SymDefSmem<BM, BN, BK, WM, WN, STAGES, HB>;
    using T = TileOps<BM, BN, BK, WM, WN, false, false, EPI_SYMUPD>;
    constexpr int NW = WM * WN, NC = NW * 32;
    constexpr int MI = T::MI, NI = T::NI, NBLK = MI * NI;
    constexpr uint32_t STAGE_BYTES = SM::STAGE_ELEMS * sizeof(double);
    static_assert(BM == BN, "mirror classification assumes square tiles");
    static_assert(HB >= 0 && HB <= NBLK, "hand-off blocks");

    extern __shared__ __align__(128) double smem[];
    double2* hand = reinterpret_cast<double2*>(reinterpret_cast<char*>(smem) + SM::HAND_OFFSET);
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + SM::BAR_OFFSET);
    uint64_t* empty = full + STAGES;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool producer = tid == 0;
    if (producer) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        mbar_fence_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    griddep_wait();
    griddep_launch();
    if (p.skip && *p.skip) return;
    const int64_t W = T::work_count(p);
    const int nk = (int)((p.K + BK - 1) / BK);
    const int64_t ldc = p.ldc;

    // TMA producer cursor (thread 0), STAGES−1 stages ahead across work items
    int64_t pw = blockIdx.x;
    int pk = 0, ps = 0, pround = 0, pissued = 0;
    typename T::Work pwork{};
    if (producer && pw < W) pwork = T::decode(pw, p);
    auto issue_next = [&]() {
        const int s = ps;
        if (pround > 0) mbar_wait(&empty[s], (uint32_t)((pround - 1) & 1));
        double* As = smem + s * SM::STAGE_ELEMS;
        double* Bs = As + SM::A_ELEMS;
        const int32_t kc = (int32_t)(pk * BK);
        mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
        tma_load_2d(As, &tmA, (int32_t)(pwork.tile_m * BM), kc, &full[s]);
        tma_load_2d(Bs, &tmB, (int32_t)(pwork.tile_n * BN), kc, &full[s]);
        ++pissued;
        if (++ps == STAGES) {
            ps = 0;
            ++pround;
        }
        if (++pk == nk) {
            pk = 0;
            pw += gridDim.x;
            if (pw < W) pwork = T::decode(pw, p);
        }
    };
    auto pump = [&](int cg) {
        while (pw < W && pissued < cg + STAGES - 1) issue_next();
    };
    __syncthreads();
    if (producer) pump(0);

    // deferred tile (control flow below is CTA-uniform)
    bool d_mirror = false, bad = false;
    int d_blk = HB;             // next handed-off block to retire (HB: none pending)
    double* d_base = nullptr;   // &X(m0 + wm0 + g, n0 + wn0 + 2·t4) of the deferred tile
    double* d_mbase = nullptr;  // &X(n0 + wn0 + 2·t4, m0 + wm0 + g): its mirror
    const double2* myhand = hand + tid;
    // X += v on one fragment block (16×8: rows g, g+8; columns 2·t4, 2·t4+1) and on its mirror
    auto red_block = [&](double* base, double* mbase, bool mirror, int i, int j, double v0, double v1, double v2,
                         double v3) {
        double* x = base + i * 16 + (int64_t)(j * 8) * ldc;
        atomicAdd(x, v0);
        atomicAdd(x + ldc, v1);
        atomicAdd(x + 8, v2);
        atomicAdd(x + 8 + ldc, v3);
        if (mirror) {
            double* m = mbase + (int64_t)(i * 16) * ldc + j * 8;
            atomicAdd(m, v0);
            atomicAdd(m + 1, v1);
            atomicAdd(m + 8 * ldc, v2);
            atomicAdd(m + 8 * ldc + 1, v3);
        }
        bad |= !isfinite(v0) || !isfinite(v1) || !isfinite(v2) || !isfinite(v3);
    };
    auto hook = [&]() {  // one handed-off block of the deferred tile per call
        if (d_blk >= HB) return;
        const double2 h0 = myhand[(d_blk * 2 + 0) * NC], h1 = myhand[(d_blk * 2 + 1) * NC];
        red_block(d_base, d_mbase, d_mirror, d_blk / NI, d_blk % NI, h0.x, h0.y, h1.x, h1.y);
        ++d_blk;
    };

    T t;
    int cg = 0, cs = 0;
    uint32_t cphase = 0;
    for (int64_t w = blockIdx.x; w < W; w += gridDim.x) {
        t.setup_work(w, p, warp, lane);
        const int64_t m0 = t.m0, n0 = t.n0;
        // full off-diagonal tile of the symmetric block (mirrored) / full tile right of it (plain)
        const bool t_mirror = m0 + BM <= n0 && n0 + BN <= p.M;
        const bool t_plain = n0 >= p.M && m0 + BM <= p.M && n0 + BN <= p.N;
        {  // this tile's X block (and its mirror) to L2 while it is computed: one prefetch per line
            constexpr int LINES = BN * (BM / 16);
            for (int l = tid; l < LINES; l += NC) {
                const int64_t c = n0 + l / (BM / 16), r = m0 + (l % (BM / 16)) * 16;
                if (r < p.M && c < p.N) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p.C + r + c * ldc));
                if (t_mirror) {
                    const int64_t mc = m0 + l / (BN / 16), mr = n0 + (l % (BN / 16)) * 16;
                    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p.C + mr + mc * ldc));
                }
            }
        }
        double acc[MI][NI][4];
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;
        for (int kt = 0; kt < nk; ++kt, ++cg) {
            if (warp == 0) {
                if (producer) pump(cg);
                __syncwarp();
            }
            const int s = cs;
            mbar_wait(&full[s], cphase);
            if (++cs == STAGES) {
                cs = 0;
                cphase ^= 1u;
            }
            const double* As = smem + s * SM::STAGE_ELEMS;
            t.compute_stage(acc, As, As + SM::A_ELEMS);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
#pragma unroll
            for (int h = 0; h < BK / 8; ++h) hook();
        }
        while (d_blk < HB) hook();  // short K: the rest of the previous tile
        if (t_mirror || t_plain) {
            const int64_t r = t.row(0, 0), c = t.col(0, 0);
            double* base = p.C + r + c * ldc;
            double* mbase = p.C + c + r * ldc;
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < NI; ++j) {
                    if (i * NI + j < HB) {
                        hand[((i * NI + j) * 2 + 0) * NC + tid] = make_double2(acc[i][j][0], acc[i][j][1]);
                        hand[((i * NI + j) * 2 + 1) * NC + tid] = make_double2(acc[i][j][2], acc[i][j][3]);
                    } else {
                        red_block(base, mbase, t_mirror, i, j, acc[i][j][0], acc[i][j][1], acc[i][j][2], acc[i][j][3]);
                    }
                }
            d_base = base;
            d_mbase = mbase;
            d_mirror = t_mirror;
            d_blk = 0;
        } else {  // diagonal / ragged tiles: immediate guarded epilogue
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < NI; ++j)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int64_t r = t.row(i, e), c = t.col(j, e);
                        if (r < p.M && c < p.N && r <= c) {
                            const double v = p.C[r + c * ldc] + acc[i][j][e];
                            p.C[r + c * ldc] = v;
                            if (r != c && c < p.M) p.C[c + r * ldc] = v;
                            bad |= !isfinite(v);
                        }
                    }
        }
    }
    while (d_blk < HB) hook();
    if (bad && p.nonfinite) atomicOr(p.nonfinite, 1);
}

// ------------------------------------------------------ C-panel TMA path --
// Short-K panel updates C ← beta·C + A·B (the AdaRBFGS factor update L += SR·B, K = q):
// with only a few k-stages per tile the C-tile loads dominate (ncu: long-scoreboard
// stalls, DMMA half idle), so the producer also fetches every work item's C tile by TMA
// into one of two shared-memory buffers, one work item ahead, and the accumulators are
// seeded from shared memory.  Persistent, one CTA per SM; EPI_STORE with beta·C seeding.
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool A_KMAJOR, bool B_KMAJOR>
struct CPanelSmem {
    using SM = GemmSmem<BM, BN, BK, WM, WN, STAGES, A_KMAJOR, B_KMAJOR>;
    static constexpr int LDCS = BM + 4;                       // C buffer pitch (column-major tile)
    static constexpr size_t RING = size_t(STAGES) * SM::STAGE_ELEMS * sizeof(double);
    static constexpr size_t CBUF = size_t(BN) * LDCS * sizeof(double);
    static constexpr size_t BAR_OFFSET = (RING + 2 * CBUF + 127) / 128 * 128;
    static constexpr size_t BYTES = BAR_OFFSET + (2 * STAGES + 4) * sizeof(uint64_t);
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool A_KMAJOR, bool B_KMAJOR>
__global__ void __launch_bounds__(WM* WN * 32, 1)
    gemm_tma_cpanel_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           const __grid_constant__ CUtensorMap tmC, GemmArgs p) {
    using SM = GemmSmem<BM, BN, BK, WM, WN, STAGES, A_KMAJOR, B_KMAJOR>;
    using CP = CPanelSmem<BM, BN, BK, WM, WN, STAGES, A_KMAJOR, B_KMAJOR>;
    using T = TileOps<BM, BN, BK, WM, WN, A_KMAJOR, B_KMAJOR, EPI_STORE>;
    constexpr int NW = WM * WN;
    constexpr uint32_t STAGE_BYTES = SM::STAGE_ELEMS * sizeof(double);
    constexpr uint32_t C_BYTES = uint32_t(BN) * CP::LDCS * sizeof(double);

    extern __shared__ __align__(128) double smem[];
    double* cbuf = reinterpret_cast<double*>(reinterpret_cast<char*>(smem) + CP::RING);
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + CP::BAR_OFFSET);
    uint64_t* empty = full + STAGES;
    uint64_t* cfull = empty + STAGES;  // [2]
    uint64_t* cempty = cfull + 2;      // [2]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool producer = tid == 0;
    if (producer) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&cfull[s], 1);
            mbar_init(&cempty[s], NW);
        }
        mbar_fence_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        tma_prefetch_desc(&tmC);
    }
    griddep_wait();
    griddep_launch();
    if (p.skip && *p.skip) return;
    const int64_t W = T::work_count(p);
    const int nk = (int)((p.K + BK - 1) / BK);  // unsplit

    // C tile of this CTA's i-th work item into buffer i & 1
    int64_t cw = blockIdx.x;
    int ci = 0;
    auto issue_c = [&]() {
        const int b = ci & 1;
        if (ci >= 2) mbar_wait(&cempty[b], (uint32_t)(((ci >> 1) - 1) & 1));
        const typename T::Work wk = T::decode(cw, p);
        mbar_arrive_expect_tx(&cfull[b], C_BYTES);
        tma_load_2d(cbuf + size_t(b) * BN * CP::LDCS, &tmC, (int32_t)(wk.tile_m * BM), (int32_t)(wk.tile_n * BN),
                    &cfull[b]);
        ++ci;
        cw += gridDim.x;
    };
    int64_t pw = blockIdx.x;
    int pk = 0, ps = 0, pround = 0, pissued = 0;
    typename T::Work pwork{};
    if (producer && pw < W) pwork = T::decode(pw, p);
    auto issue_next = [&]() {
        if (pk == 0) {  // entering work item pw: its successor's C tile goes out now (one item ahead)
            if (cw < W && cw <= pw + gridDim.x) issue_c();
        }
        const int s = ps;
        if (pround > 0) mbar_wait(&empty[s], (uint32_t)((pround - 1) & 1));
        double* As = smem + s * SM::STAGE_ELEMS;
        double* Bs = As + SM::A_ELEMS;
        const int32_t kc = (int32_t)((int64_t)pk * BK);
        const int32_t mc = (int32_t)(pwork.tile_m * BM), nc = (int32_t)(pwork.tile_n * BN);
        mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
        if constexpr (A_KMAJOR)
            tma_load_2d(As, &tmA, kc, mc, &full[s]);
        else
            tma_load_2d(As, &tmA, mc, kc, &full[s]);
        if constexpr (B_KMAJOR)
            tma_load_2d(Bs, &tmB, kc, nc, &full[s]);
        else
            tma_load_2d(Bs, &tmB, nc, kc, &full[s]);
        ++pissued;
        if (++ps == STAGES) {
            ps = 0;
            ++pround;
        }
        if (++pk == nk) {
            pk = 0;
            pw += gridDim.x;
            if (pw < W) pwork = T::decode(pw, p);
        }
    };
    auto pump = [&](int cg) {
        while (pw < W && pissued < cg + STAGES - 1) issue_next();
    };
    __syncthreads();
    if (producer) {
        if (cw < W) issue_c();  // the first item's C tile, then the stages (which send the second's)
        pump(0);
    }

    T t;
    int cg = 0, cs = 0, item = 0;
    uint32_t cphase = 0;
    for (int64_t w = blockIdx.x; w < W; w += gridDim.x, ++item) {
        t.setup_work(w, p, warp, lane);
        double acc[T::MI][T::NI][4];
        {  // seed from the C tile in shared memory (beta·C)
            const int b = item & 1;
            mbar_wait(&cfull[b], (uint32_t)((item >> 1) & 1));
            const double* Cs = cbuf + size_t(b) * BN * CP::LDCS;
#pragma unroll
            for (int i = 0; i < T::MI; ++i)
#pragma unroll
                for (int j = 0; j < T::NI; ++j)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int lr = t.wm0 + i * 16 + t.g + ((e >> 1) << 3), lc = t.wn0 + j * 8 + 2 * t.t4 + (e & 1);
                        acc[i][j][e] = p.beta * Cs[lc * CP::LDCS + lr];
                    }
            __syncwarp();
            if (lane == 0) mbar_arrive(&cempty[b]);
        }
        for (int kt = 0; kt < nk; ++kt, ++cg) {
            if (warp == 0) {
                if (producer) pump(cg);
                __syncwarp();
            }
            const int s = cs;
            mbar_wait(&full[s], cphase);
            if (++cs == STAGES) {
                cs = 0;
                cphase ^= 1u;
            }
            const double* As = smem + s * SM::STAGE_ELEMS;
            t.compute_stage(acc, As, As + SM::A_ELEMS);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        t.epilogue(acc, p, tid, NW * 32, [] {});  // c_in_acc: store-only
    }
}

// ------------------------------------------- C-panel, bulk-store epilogue --
// C ← beta·C + A·B for a short-K panel update (the AdaRBFGS factor update L += SR·B, K = q)
// with both directions of the C traffic on the bulk-copy engine.  The C-panel kernel above still
// pays, per 128×64 tile of only K/16 stages, a 64 KB store burst from registers (SM → L2 at
// ≈ 64 B/clk: every warp stalled in its stores while the DMMA pipe idles).  Here a tile's C
// block arrives by TMA into `cin` during the previous tile's mainloop (issued as soon as every
// warp has seeded its accumulators from the previous block), and the finished tile is written
// to a second shared-memory tile `cout` (column pitch BM + 4: the conflict-free fragment
// layout) and leaves as BN bulk copies of one 1 KB column each (cp.async.bulk shared → global,
// SASS UBLKCP, one per thread of warps 0–1) that drain while the warps are already in the
// next tile's mainloop.  `cout` is rewritten only after its issuing threads saw their copies'
// reads complete (mbarrier ofree), a whole mainloop later.  (Letting the L2 do the
// read-modify-write — cp.reduce.async.bulk .add.f64 from a zero-seeded tile, no C load at all —
// measured 94 µs against 105 µs at config 2 but is capped by the L2's FP64 atomic rate,
// ≈ 190 G elements/s: 88 µs for n² = 16.8 M elements.)
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool A_KMAJOR, bool B_KMAJOR>
struct CBulkSmem {
    using SM = GemmSmem<BM, BN, BK, WM, WN, STAGES, A_KMAJOR, B_KMAJOR>;
    static constexpr int LDC = BM + 4;  // pitch of both C tiles (column-major)
    static constexpr size_t RING = size_t(STAGES) * SM::STAGE_ELEMS * sizeof(double);
    static constexpr size_t CBUF = size_t(BN) * LDC * sizeof(double);
    static constexpr size_t BAR_OFFSET = (RING + 2 * CBUF + 127) / 128 * 128;
    static constexpr size_t BYTES = BAR_OFFSET + (2 * STAGES + 3) * sizeof(uint64_t);
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool A_KMAJOR, bool B_KMAJOR>
__global__ void __launch_bounds__(WM* WN * 32, 1)
    gemm_tma_cbulk_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmC, GemmArgs p) {
    using SM = GemmSmem<BM, BN, BK, WM, WN, STAGES, A_KMAJOR, B_KMAJOR>;
    using CB = CBulkSmem<BM, BN, BK, WM, WN, STAGES, A_KMAJOR, B_KMAJOR>;
    using T = TileOps<BM, BN, BK, WM, WN, A_KMAJOR, B_KMAJOR, EPI_STORE>;
    constexpr int NW = WM * WN, NC = NW * 32;
    constexpr uint32_t STAGE_BYTES = SM::STAGE_ELEMS * sizeof(double);
    constexpr uint32_t C_BYTES = uint32_t(BN) * CB::LDC * sizeof(double);
    static_assert(BN <= NC, "one bulk copy per thread");

    extern __shared__ __align__(128) double smem[];
    double* cin = reinterpret_cast<double*>(reinterpret_cast<char*>(smem) + CB::RING);
    double* cout = cin + size_t(BN) * CB::LDC;
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + CB::BAR_OFFSET);
    uint64_t* empty = full + STAGES;
    uint64_t* cfull = empty + STAGES;  // the item's C block has landed in cin
    uint64_t* cseeded = cfull + 1;     // every warp has read cin (count NW)
    uint64_t* ofree = cseeded + 1;     // the previous item's bulk copies have left cout (count BN)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool producer = tid == 0;
    if (producer) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        mbar_init(cfull, 1);
        mbar_init(cseeded, NW);
        mbar_init(ofree, BN);
        mbar_fence_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        tma_prefetch_desc(&tmC);
    }
    griddep_wait();
    griddep_launch();
    if (p.skip && *p.skip) return;
    const int64_t W = T::work_count(p);
    const int nk = (int)((p.K + BK - 1) / BK);  // unsplit

    auto issue_c = [&](int64_t w) {  // C block of work item w into cin
        const typename T::Work wk = T::decode(w, p);
        mbar_arrive_expect_tx(cfull, C_BYTES);
        tma_load_2d(cin, &tmC, (int32_t)(wk.tile_m * BM), (int32_t)(wk.tile_n * BN), cfull);
    };
    int64_t pw = blockIdx.x;
    int pk = 0, ps = 0, pround = 0, pissued = 0;
    typename T::Work pwork{};
    if (producer && pw < W) pwork = T::decode(pw, p);
    auto issue_next = [&]() {
        const int s = ps;
        if (pround > 0) mbar_wait(&empty[s], (uint32_t)((pround - 1) & 1));
        double* As = smem + s * SM::STAGE_ELEMS;
        double* Bs = As + SM::A_ELEMS;
        const int32_t kc = (int32_t)((int64_t)pk * BK);
        const int32_t mc = (int32_t)(pwork.tile_m * BM), nc = (int32_t)(pwork.tile_n * BN);
        mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
        if constexpr (A_KMAJOR)
            tma_load_2d(As, &tmA, kc, mc, &full[s]);
        else
            tma_load_2d(As, &tmA, mc, kc, &full[s]);
        if constexpr (B_KMAJOR)
            tma_load_2d(Bs, &tmB, kc, nc, &full[s]);
        else
            tma_load_2d(Bs, &tmB, nc, kc, &full[s]);
        ++pissued;
        if (++ps == STAGES) {
            ps = 0;
            ++pround;
        }
        if (++pk == nk) {
            pk = 0;
            pw += gridDim.x;
            if (pw < W) pwork = T::decode(pw, p);
        }
    };
    auto pump = [&](int cg) {
        while (pw < W && pissued < cg + STAGES - 1) issue_next();
    };
    __syncthreads();
    if (producer) {
        if (blockIdx.x < W) issue_c(blockIdx.x);
        pump(0);
    }

    T t;
    int cg = 0, cs = 0, item = 0;
    uint32_t cphase = 0;
    bool bad = false;
    for (int64_t w = blockIdx.x; w < W; w += gridDim.x, ++item) {
        t.setup_work(w, p, warp, lane);
        double acc[T::MI][T::NI][4];
        {  // seed from the C block in shared memory (beta·C)
            mbar_wait(cfull, (uint32_t)(item & 1));
#pragma unroll
            for (int i = 0; i < T::MI; ++i)
#pragma unroll
                for (int j = 0; j < T::NI; ++j)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int lr = t.wm0 + i * 16 + t.g + ((e >> 1) << 3), lc = t.wn0 + j * 8 + 2 * t.t4 + (e & 1);
                        acc[i][j][e] = p.beta * cin[lc * CB::LDC + lr];
                    }
            __syncwarp();
            if (lane == 0) mbar_arrive(cseeded);
            if (producer && w + gridDim.x < W) {  // cin is free once every warp has seeded: fetch the next block
                mbar_wait(cseeded, (uint32_t)(item & 1));
                issue_c(w + gridDim.x);
            }
        }
        for (int kt = 0; kt < nk; ++kt, ++cg) {
            if (warp == 0) {
                if (producer) pump(cg);
                __syncwarp();
            }
            const int s = cs;
            mbar_wait(&full[s], cphase);
            if (++cs == STAGES) {
                cs = 0;
                cphase ^= 1u;
            }
            const double* As = smem + s * SM::STAGE_ELEMS;
            t.compute_stage(acc, As, As + SM::A_ELEMS);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        // the finished tile leaves through cout; the previous item's copies were issued a mainloop ago
        if (item >= 1) {
            if (tid < BN) {
                bulk_wait_read<0>();
                mbar_arrive(ofree);
            }
            mbar_wait(ofree, (uint32_t)((item - 1) & 1));
        }
#pragma unroll
        for (int i = 0; i < T::MI; ++i)
#pragma unroll
            for (int j = 0; j < T::NI; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int lr = t.wm0 + i * 16 + t.g + ((e >> 1) << 3), lc = t.wn0 + j * 8 + 2 * t.t4 + (e & 1);
                    cout[lc * CB::LDC + lr] = acc[i][j][e];
                    bad |= !isfinite(acc[i][j][e]);
                }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid < BN) {
            const int64_t col = t.n0 + tid;
            const int64_t rows = min((int64_t)BM, p.M - t.m0);
            if (col < p.N && rows > 0) bulk_store(p.C + t.m0 + col * p.ldc, cout + tid * CB::LDC, (uint32_t)(rows * sizeof(double)));
            bulk_commit();
        }
    }
    if (tid < BN) bulk_wait<0>();
    if (bad && p.nonfinite) atomicOr(p.nonfinite, 1);
}

// ------------------------------------------- C-panel, A-stationary (K ≤ 64) --
// C ← beta·C + A·B for a panel update whose whole K fits one shared-memory operand (the
// AdaRBFGS factor update L += SR·B at q ≤ 64).  With K = 64 a 128×64 tile is only four BK = 16
// stages: the ring kernels above spend as long waiting on operand stages and tile changes as
// on DMMA (ncu: the warps sit on full[]; 100 µs for 58 µs of DMMA work at config 2).  Here
// each CTA owns a contiguous run of tiles in row-strip order, so the 128×K slice of A stays
// in shared memory for the whole strip (reloaded at most once per CTA), the K×64 slice of B
// arrives as ONE TMA box per tile (double-buffered, a whole tile ahead) and the C tile by TMA
// into a third buffer, one tile ahead: two barrier waits per tile instead of five, and
// 100 KB instead of 170 KB fetched per tile.  A not K-major, B K-major (the L-update layout).
template <int BM, int BN, int KMAX>
struct CStatSmem {
    static constexpr int LDA = BM + 4, LDB = KMAX + 4, LDC = BM + 4;
    static constexpr size_t A_BYTES = size_t(KMAX) * LDA * sizeof(double);
    static constexpr size_t B_BYTES = size_t(BN) * LDB * sizeof(double);
    static constexpr size_t C_BYTES = size_t(BN) * LDC * sizeof(double);
    static constexpr size_t B_OFFSET = A_BYTES, C_OFFSET = A_BYTES + 2 * B_BYTES;
    static constexpr size_t BAR_OFFSET = (C_OFFSET + C_BYTES + 127) / 128 * 128;
    static constexpr size_t BYTES = BAR_OFFSET + 8 * sizeof(uint64_t);
};

template <int BM, int BN, int KMAX, int WM, int WN>
__global__ void __launch_bounds__(WM* WN * 32, 1)
    gemm_tma_cstat_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmC, GemmArgs p) {
    using SM = CStatSmem<BM, BN, KMAX>;
    using T = TileOps<BM, BN, KMAX, WM, WN, false, true, EPI_STORE>;
    constexpr int NW = WM * WN;
    static_assert(SM::A_BYTES % 128 == 0 && SM::B_BYTES % 128 == 0 && SM::C_BYTES % 128 == 0, "TMA destinations");

    extern __shared__ __align__(128) double smem[];
    double* As = smem;
    double* Bs = reinterpret_cast<double*>(reinterpret_cast<char*>(smem) + SM::B_OFFSET);
    double* Cs = reinterpret_cast<double*>(reinterpret_cast<char*>(smem) + SM::C_OFFSET);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + SM::BAR_OFFSET);
    uint64_t* afull = bars;        // the strip's A slice has landed
    uint64_t* adone = bars + 1;    // every warp has finished the strip (count NW)
    uint64_t* bfull = bars + 2;    // [2] B slice of item i in buffer i & 1
    uint64_t* bdone = bars + 4;    // [2] every warp has finished with that buffer (count NW)
    uint64_t* cfull = bars + 6;    // the item's C block has landed
    uint64_t* cseeded = bars + 7;  // every warp has read it (count NW)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool producer = tid == 0;
    if (producer) {
        mbar_init(afull, 1);
        mbar_init(adone, NW);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&bfull[b], 1);
            mbar_init(&bdone[b], NW);
        }
        mbar_init(cfull, 1);
        mbar_init(cseeded, NW);
        mbar_fence_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        tma_prefetch_desc(&tmC);
    }
    griddep_wait();
    griddep_launch();
    if (p.skip && *p.skip) return;
    // this CTA's run of tiles, row strips outermost: item t = strip · tn + column tile
    const int64_t tm = (p.M + BM - 1) / BM, tn = (p.N + BN - 1) / BN, W = tm * tn;
    const int64_t w0 = W * blockIdx.x / gridDim.x, w1 = W * (blockIdx.x + 1) / gridDim.x;
    auto issue_a = [&](int64_t strip) {
        mbar_arrive_expect_tx(afull, (uint32_t)SM::A_BYTES);
        tma_load_2d(As, &tmA, (int32_t)(strip * BM), 0, afull);
    };
    auto issue_b = [&](int64_t w, int item) {
        const int b = item & 1;
        if (item >= 2) mbar_wait(&bdone[b], (uint32_t)(((item >> 1) - 1) & 1));
        mbar_arrive_expect_tx(&bfull[b], (uint32_t)SM::B_BYTES);
        tma_load_2d(Bs + size_t(b) * BN * SM::LDB, &tmB, 0, (int32_t)((w % tn) * BN), &bfull[b]);
    };
    auto issue_c = [&](int64_t w) {
        mbar_arrive_expect_tx(cfull, (uint32_t)SM::C_BYTES);
        tma_load_2d(Cs, &tmC, (int32_t)((w / tn) * BM), (int32_t)((w % tn) * BN), cfull);
    };
    __syncthreads();
    if (producer && w0 < w1) {
        issue_a(w0 / tn);
        issue_c(w0);
        issue_b(w0, 0);
        if (w0 + 1 < w1) issue_b(w0 + 1, 1);
    }

    T t;
    int strips = 0;  // A slices consumed so far
    int64_t cur_strip = -1;
    bool bad = false;
    for (int64_t w = w0; w < w1; ++w) {
        const int item = (int)(w - w0);
        // TileOps::setup_work decodes column-major tile order; this kernel walks strips, so set the tile here
        t.tile_m = w / tn;
        t.tile_n = w % tn;
        t.split = 0;
        t.m0 = t.tile_m * BM;
        t.n0 = t.tile_n * BN;
        t.g = lane >> 2;
        t.t4 = lane & 3;
        t.wm0 = (warp / WN) * (BM / WM);
        t.wn0 = (warp % WN) * (BN / WN);
        if (t.tile_m != cur_strip) {
            if (cur_strip >= 0) {  // the previous strip is finished: its A slice may be replaced
                __syncwarp();
                if (lane == 0) mbar_arrive(adone);
                if (producer) {
                    mbar_wait(adone, (uint32_t)((strips - 1) & 1));
                    issue_a(t.tile_m);
                }
            }
            cur_strip = t.tile_m;
            mbar_wait(afull, (uint32_t)(strips & 1));
            ++strips;
        }
        double acc[T::MI][T::NI][4];
        mbar_wait(cfull, (uint32_t)(item & 1));
#pragma unroll
        for (int i = 0; i < T::MI; ++i)
#pragma unroll
            for (int j = 0; j < T::NI; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int lr = t.wm0 + i * 16 + t.g + ((e >> 1) << 3), lc = t.wn0 + j * 8 + 2 * t.t4 + (e & 1);
                    acc[i][j][e] = p.beta * Cs[lc * SM::LDC + lr];
                }
        __syncwarp();
        if (lane == 0) mbar_arrive(cseeded);
        if (producer && w + 1 < w1) {  // the C buffer is free once every warp has seeded
            mbar_wait(cseeded, (uint32_t)(item & 1));
            issue_c(w + 1);
        }
        const int b = item & 1;
        mbar_wait(&bfull[b], (uint32_t)((item >> 1) & 1));
        {
            const double* Bb = Bs + size_t(b) * BN * SM::LDB;
#pragma unroll 1
            for (int kk = 0; kk < KMAX; kk += 16)  // rolled: a full unroll keeps every fragment of the slice live
                t.template compute_part<0, 16>(acc, As + kk * SM::LDA, Bb + kk);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bdone[b]);
        // store-only epilogue (the accumulators hold beta·C + A·B)
#pragma unroll
        for (int i = 0; i < T::MI; ++i)
#pragma unroll
            for (int j = 0; j < T::NI; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int64_t r = t.row(i, e), c = t.col(j, e);
                    if (r < p.M && c < p.N) {
                        p.C[r + c * p.ldc] = acc[i][j][e];
                        bad |= !isfinite(acc[i][j][e]);
                    }
                }
        if (producer && w + 2 < w1) issue_b(w + 2, item + 2);  // buffer b again, once every warp has left it
    }
    if (bad && p.nonfinite) atomicOr(p.nonfinite, 1);
}

// One CTA per work item (grid = tiles × splits): the long-K products (Y = A·S,
// W = X·Y), whose pipeline fill is amortised over ≥ 100 k-stages.
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool A_KMAJOR, bool B_KMAJOR, int EPI>
__global__ void __launch_bounds__(WM* WN * 32, 1)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs p) {
    using SM = GemmSmem<BM, BN, BK, WM, WN, STAGES, A_KMAJOR, B_KMAJOR>;
    using T = TileOps<BM, BN, BK, WM, WN, A_KMAJOR, B_KMAJOR, EPI>;
    constexpr int NW = WM * WN;
    constexpr uint32_t STAGE_BYTES = SM::STAGE_ELEMS * sizeof(double);

    extern __shared__ __align__(128) double smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + SM::BAR_OFFSET);
    uint64_t* empty = full + STAGES;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {  // prologue before the dependency wait (overlaps the predecessor's tail under PDL)
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        mbar_fence_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    griddep_wait();
    griddep_launch();
    if (p.skip && *p.skip) return;
    T t;
    t.setup(warp, lane, p);
    const int64_t k_begin = (int64_t)blockIdx.z * p.k_chunk;
    const int64_t k_end = min(p.K, k_begin + p.k_chunk);
    const int num_kt = (int)((k_end - k_begin + BK - 1) / BK);
    const bool producer = tid == 0;

    auto issue = [&](int kt) {
        const int s = kt % STAGES;
        if (kt >= STAGES) mbar_wait(&empty[s], ((kt / STAGES) - 1) & 1);
        double* As = smem + s * SM::STAGE_ELEMS;
        double* Bs = As + SM::A_ELEMS;
        const int32_t kc = (int32_t)(k_begin + (int64_t)kt * BK);
        mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
        if constexpr (A_KMAJOR)
            tma_load_2d(As, &tmA, kc, (int32_t)t.m0, &full[s]);
        else
            tma_load_2d(As, &tmA, (int32_t)t.m0, kc, &full[s]);
        if constexpr (B_KMAJOR)
            tma_load_2d(Bs, &tmB, kc, (int32_t)t.n0, &full[s]);
        else
            tma_load_2d(Bs, &tmB, (int32_t)t.n0, kc, &full[s]);
    };

    __syncthreads();
    if (producer)
        for (int kt = 0; kt < STAGES - 1 && kt < num_kt; ++kt) issue(kt);

    double acc[T::MI][T::NI][4];
    t.init_acc(acc, p);
    for (int kt = 0; kt < num_kt; ++kt) {
        if (warp == 0) {
            if (producer && kt + STAGES - 1 < num_kt) issue(kt + STAGES - 1);
            __syncwarp();
        }
        const int s = kt % STAGES;
        mbar_wait(&full[s], (kt / STAGES) & 1);
        const double* As = smem + s * SM::STAGE_ELEMS;
        t.compute_stage(acc, As, As + SM::A_ELEMS);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    t.epilogue(acc, p, tid, NW * 32, [] { __syncthreads(); });
}

// ---------------------------------------------------------- cp.async path --
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool A_KMAJOR, bool B_KMAJOR, int VEC, int EPI>
__global__ void __launch_bounds__(WM* WN * 32) gemm_f64_kernel(GemmArgs p) {
    using SM = GemmSmem<BM, BN, BK, WM, WN, STAGES, A_KMAJOR, B_KMAJOR>;
    using T = TileOps<BM, BN, BK, WM, WN, A_KMAJOR, B_KMAJOR, EPI>;
    constexpr int NT = WM * WN * 32;
    constexpr int LDA_S = T::LDA_S, LDB_S = T::LDB_S;

    if (p.skip && *p.skip) return;
    extern __shared__ __align__(128) double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    T t;
    t.setup(warp, lane, p);
    const int64_t m0 = t.m0, n0 = t.n0;
    const int64_t k_begin = (int64_t)blockIdx.z * p.k_chunk;
    const int64_t k_end = min(p.K, k_begin + p.k_chunk);
    const int num_kt = (int)((k_end - k_begin + BK - 1) / BK);

    auto load_stage = [&](int stage, int kt) {
        double* As = smem + stage * SM::STAGE_ELEMS;
        double* Bs = As + SM::A_ELEMS;
        const int64_t kbase = k_begin + (int64_t)kt * BK;
        if constexpr (!A_KMAJOR) {  // columns of BM contiguous doubles
            constexpr int CH = BK * BM / VEC;
            for (int c = tid; c < CH; c += NT) {
                const int kk = c / (BM / VEC), mm = (c % (BM / VEC)) * VEC;
                const int64_t gm = m0 + mm, gk = kbase + kk;
                const bool ok = gm < p.M && gk < k_end;
                cp_async<VEC * 8>(As + kk * LDA_S + mm, ok ? p.A + gm + gk * p.lda : p.A, ok);
            }
        } else {  // rows of BK contiguous doubles
            constexpr int CH = BM * BK / VEC;
            for (int c = tid; c < CH; c += NT) {
                const int mm = c / (BK / VEC), kk = (c % (BK / VEC)) * VEC;
                const int64_t gm = m0 + mm, gk = kbase + kk;
                const bool ok = gm < p.M && gk < k_end;
                cp_async<VEC * 8>(As + mm * LDA_S + kk, ok ? p.A + gm * p.lda + gk : p.A, ok);
            }
        }
        if constexpr (B_KMAJOR) {  // columns n: BK contiguous doubles
            constexpr int CH = BN * BK / VEC;
            for (int c = tid; c < CH; c += NT) {
                const int nn = c / (BK / VEC), kk = (c % (BK / VEC)) * VEC;
                const int64_t gn = n0 + nn, gk = kbase + kk;
                const bool ok = gn < p.N && gk < k_end;
                cp_async<VEC * 8>(Bs + nn * LDB_S + kk, ok ? p.B + gk + gn * p.ldb : p.B, ok);
            }
        } else {  // rows k: BN contiguous doubles
            constexpr int CH = BK * BN / VEC;
            for (int c = tid; c < CH; c += NT) {
                const int kk = c / (BN / VEC), nn = (c % (BN / VEC)) * VEC;
                const int64_t gn = n0 + nn, gk = kbase + kk;
                const bool ok = gn < p.N && gk < k_end;
                cp_async<VEC * 8>(Bs + kk * LDB_S + nn, ok ? p.B + gn + gk * p.ldb : p.B, ok);
            }
        }
    };

    double acc[T::MI][T::NI][4];
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < num_kt) load_stage(s, s);
        cp_async_commit();
    }
    t.init_acc(acc, p);
    for (int kt = 0; kt < num_kt; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int nk = kt + STAGES - 1;
            if (nk < num_kt) load_stage(nk % STAGES, nk);
            cp_async_commit();
        }
        const double* As = smem + (kt % STAGES) * SM::STAGE_ELEMS;
        t.compute_stage(acc, As, As + SM::A_ELEMS);
    }
    cp_async_wait<0>();
    t.epilogue(acc, p, tid, NT, [] { __syncthreads(); });
}

}  // namespace si
