// Engine: launch logic of the RBFGS / AdaRBFGS iteration on one B200.
// See engine.hpp for the data each pipeline keeps resident in HBM.
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "engine.hpp"
#include "gemm_f64.cuh"
#include "kernels_aux.cuh"
#include "kernels_small.cuh"
#include "kernels_core.cuh"

namespace si {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

// ----------------------------------------------------------------- context --
Context* context_create(int device, cudaStream_t external, bool on_stream) {
    CK(cudaSetDevice(device));
    auto* c = new Context();
    c->device = device;
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    if (external) {
        c->stream = external;
        c->own_stream = false;
    } else if (on_stream) {
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamDefault));  // blocking: ordered with stream 0
        c->own_stream = true;
    } else {
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    CK(cudaMalloc(&c->scalar_dev, 8 * sizeof(double)));
    CK(cudaMallocHost(&c->scalar_host, 8 * sizeof(double)));
    return c;
}

Context::~Context() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (auto& p : pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (auto e : event_pool) cudaEventDestroy(e);
    if (ws) cudaFree(ws);
    if (ws_side) cudaFree(ws_side);
    if (side) cudaStreamDestroy(side);
    if (side_hi) cudaStreamDestroy(side_hi);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (cached_rw) {
        cached_rw->release();
        delete cached_rw;
    }
    if (cached_aw) {
        cached_aw->release();
        delete cached_aw;
    }
    if (aux_status) cudaFree(aux_status);
    if (scalar_dev) cudaFree(scalar_dev);
    if (scalar_host) cudaFreeHost(scalar_host);
    if (own_stream && stream) cudaStreamDestroy(stream);
}

void Context::fork(bool high) {
    if (!side) {
        CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&side_hi, cudaStreamNonBlocking, hi));
        CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(ev_fork, stream));
    CK(cudaStreamWaitEvent(high ? side_hi : side, ev_fork, 0));
}

void Context::join(bool high) {
    CK(cudaEventRecord(ev_join, high ? side_hi : side));
    CK(cudaStreamWaitEvent(stream, ev_join, 0));
}

// Enqueue on the side stream with its own split-K workspace (RAII swap of stream / ws).
struct SideScope {
    Context& c;
    cudaStream_t s0;
    double* w0;
    size_t n0;
    explicit SideScope(Context& ctx, bool high = false) : c(ctx), s0(ctx.stream), w0(ctx.ws), n0(ctx.ws_doubles) {
        c.stream = high ? c.side_hi : c.side;
        c.ws = c.ws_side;
        c.ws_doubles = c.ws_side_doubles;
    }
    ~SideScope() {
        c.ws_side = c.ws;
        c.ws_side_doubles = c.ws_doubles;
        c.stream = s0;
        c.ws = w0;
        c.ws_doubles = n0;
    }
};

SideHi::SideHi(Context& ctx) : c(ctx), s0(ctx.stream), w0(ctx.ws), n0(ctx.ws_doubles) {
    c.stream = c.side_hi;
    c.ws = c.ws_side;
    c.ws_doubles = c.ws_side_doubles;
}
SideHi::~SideHi() {
    c.ws_side = c.ws;
    c.ws_side_doubles = c.ws_doubles;
    c.stream = s0;
    c.ws = w0;
    c.ws_doubles = n0;
}

RbfgsWork* Context::take_rbfgs(int64_t n, int64_t q) {
    if (!cached_rw || cached_rw->n != n || cached_rw->q != q) return nullptr;
    RbfgsWork* w = cached_rw;
    cached_rw = nullptr;
    CK(cudaMemsetAsync(w->status, 0, 8 * sizeof(int), stream));
    CK(cudaMemsetAsync(w->counter, 0, sizeof(unsigned long long), stream));
    w->batch = false;
    return w;
}

void Context::keep_rbfgs(RbfgsWork* w) {
    if (cached_rw) {
        cached_rw->release();
        delete cached_rw;
    }
    cached_rw = w;
}

AdaWork* Context::take_ada(int64_t n, int64_t q, bool gaussian) {
    if (!cached_aw || cached_aw->n != n || cached_aw->q != q || cached_aw_gauss != gaussian) return nullptr;
    AdaWork* w = cached_aw;
    cached_aw = nullptr;
    CK(cudaMemsetAsync(w->status, 0, 8 * sizeof(int), stream));
    CK(cudaMemsetAsync(w->counter, 0, sizeof(unsigned long long), stream));
    w->batch = false;
    w->pdiag_valid = false;
    w->pdiag_age = 0;
    w->pdiag_refresh = 64;
    return w;
}

void Context::keep_ada(AdaWork* w, bool gaussian) {
    if (cached_aw) {
        cached_aw->release();
        delete cached_aw;
    }
    cached_aw = w;
    cached_aw_gauss = gaussian;
}

double* Context::ensure_ws(size_t doubles) {
    if (doubles <= ws_doubles) return ws;
    CK(cudaStreamSynchronize(stream));
    if (ws) CK(cudaFree(ws));
    ws_doubles = std::max(doubles, ws_doubles * 2);
    CK(cudaMalloc(&ws, ws_doubles * sizeof(double)));
    return ws;
}

int Context::class_id(const char* name) {
    for (size_t i = 0; i < class_names.size(); ++i)
        if (class_names[i] == name) return int(i);
    class_names.emplace_back(name);
    stats.emplace_back();
    return int(class_names.size() - 1);
}

void Context::resolve_profile() {
    if (pending.empty()) return;
    CK(cudaStreamSynchronize(stream));
    for (auto& p : pending) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, p.a, p.b));
        stats[size_t(p.cls)].ms += ms;
        event_pool.push_back(p.a);
        event_pool.push_back(p.b);
    }
    pending.clear();
}

LaunchScope::LaunchScope(Context& ctx, const char* name) : c(ctx) {
    c.launches++;
    cls = c.class_id(name);
    c.stats[size_t(cls)].launches++;
    if (c.profiling) {
        auto get = [&]() {
            if (!c.event_pool.empty()) {
                cudaEvent_t e = c.event_pool.back();
                c.event_pool.pop_back();
                return e;
            }
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            return e;
        };
        a = get();
        b = get();
        CK(cudaEventRecord(a, c.stream));
    }
}

LaunchScope::~LaunchScope() {
    if (a) {
        cudaEventRecord(b, c.stream);
        c.pending.push_back({cls, a, b});
    }
}

static void check_launch(const char* what) { cuda_check(cudaGetLastError(), what); }

static int grid_for(int64_t work, int threads, int max_blocks = 148 * 16) {
    int64_t b = (work + threads - 1) / threads;
    return int(std::max<int64_t>(1, std::min<int64_t>(b, max_blocks)));
}

// --------------------------------------------------------------- GEMM ------
enum TileCfg { T128x128 = 0, T128x64 = 1, T128x32 = 2, T128x128W16 = 3, T64x128 = 4, T128x128K32 = 5, T128x128W8K32 = 6, T128x128W16S6 = 7, T64x64 = 8 };

// development switches: SI_WARPS16=1 selects 16 consumer warps for 128×128
// tiles; SI_NO_TMA=1 forces the cp.async mainloop.
static bool env_flag(const char* name) {
    const char* s = std::getenv(name);
    return s && s[0] == '1';
}
static bool use_w16() {
    static int v = -1;
    if (v < 0) v = env_flag("SI_WARPS16") ? 1 : 0;
    return v == 1;
}
static bool tma_disabled() {
    static int v = -1;
    if (v < 0) v = env_flag("SI_NO_TMA") ? 1 : 0;
    return v == 1;
}

// Kernel attributes (dynamic shared memory limit) are per device: set once per device
// the first time a context on that device launches the kernel.
struct DeviceOnce {
    std::atomic<uint64_t> mask{0};
    bool first(int device) {
        const uint64_t bit = 1ull << (device & 63);
        return !(mask.fetch_or(bit) & bit);
    }
};

template <int BM, int BN, int BK, int WM, int WN, int ST, bool AK, bool BKM, int VEC, int EPI>
static void launch_gemm_cfg(Context& c, const GemmArgs& a, dim3 grid, const char* name) {
    using SM = GemmSmem<BM, BN, BK, WM, WN, ST, AK, BKM>;
    auto kern = gemm_f64_kernel<BM, BN, BK, WM, WN, ST, AK, BKM, VEC, EPI>;
    static DeviceOnce once;
    if (once.first(c.device)) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SM::BYTES)));
    LaunchScope ls(c, name);
    kern<<<grid, WM * WN * 32, SM::BYTES, c.stream>>>(a);
    check_launch(name);
}

// ---- programmatic dependent launch: the iteration's kernels call griddep_wait()
// before touching their inputs, so each may be launched while its predecessor
// drains (SI_NO_PDL=1 turns the attribute off)
static bool pdl_enabled() {
    static const bool on = std::getenv("SI_NO_PDL") == nullptr;
    return on;
}
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, kern, args...));
}

// ---- TMA descriptors (cuTensorMapEncodeTiled through the runtime's driver entry point)
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw CudaError("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2-D FP64 tensor: `inner` contiguous elements per line, `outer` lines `ld` apart.
static void make_tmap(CUtensorMap* m, const double* base, int64_t inner, int64_t outer, int64_t ld, uint32_t box_inner,
                      uint32_t box_outer) {
    cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
    cuuint64_t strides[1] = {cuuint64_t(ld) * sizeof(double)};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

template <int BM, int BN, int BK, int WM, int WN, int ST, bool AK, bool BKM, int EPI>
static void launch_tma_cfg(Context& c, const GemmArgs& a, dim3 grid, const char* name) {
    using SM = GemmSmem<BM, BN, BK, WM, WN, ST, AK, BKM>;
    // Short-K products (the rank-2q updates) run persistent — one CTA per resident
    // slot striding over the work items, so the next tile's TMA stages stream in
    // under the current tile's epilogue; long-K products keep one CTA per item
    // (measured faster: their fill is amortised over >= 100 k-stages).
    const bool persist = EPI == EPI_SYMUPD || a.K <= 1024;
    auto kern_p = gemm_tma_persistent_kernel<BM, BN, BK, WM, WN, ST, AK, BKM, EPI>;
    auto kern_g = gemm_tma_kernel<BM, BN, BK, WM, WN, ST, AK, BKM, EPI>;
    static DeviceOnce once;
    static int per_sm = 1;  // same for every B200
    if (once.first(c.device)) {
        CK(cudaFuncSetAttribute(kern_p, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SM::TMA_BYTES)));
        CK(cudaFuncSetAttribute(kern_g, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SM::TMA_BYTES)));
        int v = 1;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern_p, WM * WN * 32, SM::TMA_BYTES));
        per_sm = std::max(v, 1);
    }
    const int64_t work = int64_t(grid.x) * grid.y * grid.z;
    CUtensorMap ta, tb;
    if (AK)
        make_tmap(&ta, a.A, a.K, a.M, a.lda, BK + 4, BM);
    else
        make_tmap(&ta, a.A, a.M, a.K, a.lda, BM + 4, BK);
    if (BKM)
        make_tmap(&tb, a.B, a.K, a.N, a.ldb, BK + 4, BN);
    else
        make_tmap(&tb, a.B, a.N, a.K, a.ldb, BN + 4, BK);
    LaunchScope ls(c, name);
    if (persist)
        launch_pdl(kern_p, dim3(unsigned(std::min<int64_t>(work, int64_t(c.num_sms) * per_sm))), dim3(WM * WN * 32),
                   SM::TMA_BYTES, c.stream, ta, tb, a);
    else
        launch_pdl(kern_g, grid, dim3(WM * WN * 32), SM::TMA_BYTES, c.stream, ta, tb, a);
    check_launch(name);
}

// C-panel TMA launch (gemm_tma_cpanel_kernel): 128×64 tiles, 8 warps, 3 stages, C tiles
// double-buffered in shared memory, one CTA per SM
template <bool AK, bool BKM>
static void launch_cpanel_cfg(Context& c, const GemmArgs& a, int64_t work) {
    constexpr int BM = 128, BN = 64, BK = 16, WM = 4, WN = 2, ST = 3;
    using CP = CPanelSmem<BM, BN, BK, WM, WN, ST, AK, BKM>;
    auto kern = gemm_tma_cpanel_kernel<BM, BN, BK, WM, WN, ST, AK, BKM>;
    static DeviceOnce once;
    if (once.first(c.device)) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(CP::BYTES)));
    CUtensorMap ta, tb, tc;
    if (AK)
        make_tmap(&ta, a.A, a.K, a.M, a.lda, BK + 4, BM);
    else
        make_tmap(&ta, a.A, a.M, a.K, a.lda, BM + 4, BK);
    if (BKM)
        make_tmap(&tb, a.B, a.K, a.N, a.ldb, BK + 4, BN);
    else
        make_tmap(&tb, a.B, a.N, a.K, a.ldb, BN + 4, BK);
    make_tmap(&tc, a.Csrc ? a.Csrc : a.C, a.M, a.N, a.ldc, BM + 4, BN);  // the seed (beta·Csrc or beta·C)
    LaunchScope ls(c, "gemm_cpanel");
    launch_pdl(kern, dim3(unsigned(std::min<int64_t>(work, int64_t(c.num_sms)))), dim3(WM * WN * 32), CP::BYTES, c.stream,
               ta, tb, tc, a);
}

// C-panel launch with the bulk-copy epilogue (gemm_tma_cbulk_kernel): C = beta·Csrc + A·B, 128×64
// tiles, 8 warps, 3 stages, one C-in and one C-out tile in shared memory, one CTA per SM
template <bool AK, bool BKM>
static void launch_cbulk_cfg(Context& c, const GemmArgs& a, int64_t work) {
    constexpr int BM = 128, BN = 64, BK = 16, WM = 4, WN = 2, ST = 3;
    using CB = CBulkSmem<BM, BN, BK, WM, WN, ST, AK, BKM>;
    static_assert(CB::BYTES <= 232448, "shared memory per CTA");
    auto kern = gemm_tma_cbulk_kernel<BM, BN, BK, WM, WN, ST, AK, BKM>;
    static DeviceOnce once;
    if (once.first(c.device)) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(CB::BYTES)));
    CUtensorMap ta, tb, tc;
    if (AK)
        make_tmap(&ta, a.A, a.K, a.M, a.lda, BK + 4, BM);
    else
        make_tmap(&ta, a.A, a.M, a.K, a.lda, BM + 4, BK);
    if (BKM)
        make_tmap(&tb, a.B, a.K, a.N, a.ldb, BK + 4, BN);
    else
        make_tmap(&tb, a.B, a.N, a.K, a.ldb, BN + 4, BK);
    make_tmap(&tc, a.Csrc ? a.Csrc : a.C, a.M, a.N, a.ldc, BM + 4, BN);  // the seed (beta·Csrc or beta·C)
    LaunchScope ls(c, "gemm_cpanel");
    launch_pdl(kern, dim3(unsigned(std::min<int64_t>(work, int64_t(c.num_sms)))), dim3(WM * WN * 32), CB::BYTES, c.stream,
               ta, tb, tc, a);
}

// A-stationary C-panel launch (gemm_tma_cstat_kernel): C = beta·Csrc + A·B for K ≤ 64, A M-major,
// B K-major; 128×64 tiles in row-strip order, 8 warps, one CTA per SM
static void launch_cstat(Context& c, const GemmArgs& a) {
    constexpr int BM = 128, BN = 64, KMAX = 64, WM = 4, WN = 2;
    using SM = CStatSmem<BM, BN, KMAX>;
    static_assert(SM::BYTES <= 232448, "shared memory per CTA");
    auto kern = gemm_tma_cstat_kernel<BM, BN, KMAX, WM, WN>;
    static DeviceOnce once;
    if (once.first(c.device)) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SM::BYTES)));
    CUtensorMap ta, tb, tc;
    make_tmap(&ta, a.A, a.M, a.K, a.lda, BM + 4, KMAX);
    make_tmap(&tb, a.B, a.K, a.N, a.ldb, KMAX + 4, BN);
    make_tmap(&tc, a.Csrc ? a.Csrc : a.C, a.M, a.N, a.ldc, BM + 4, BN);
    const int64_t work = ((a.M + BM - 1) / BM) * ((a.N + BN - 1) / BN);
    LaunchScope ls(c, "gemm_cpanel");
    launch_pdl(kern, dim3(unsigned(std::min<int64_t>(work, int64_t(c.num_sms)))), dim3(WM * WN * 32), SM::BYTES, c.stream,
               ta, tb, tc, a);
}

template <bool AK, bool BKM, int VEC, int EPI>
static void launch_gemm_tile(Context& c, TileCfg t, const GemmArgs& a, dim3 grid, const char* name, bool tma) {
    if (EPI == EPI_SYMUPD && t == T64x128) throw std::logic_error("gemm_symupd: tile height must be a multiple of its width");
    if (tma) {
        switch (t) {
            case T128x128: launch_tma_cfg<128, 128, 16, 4, 2, 5, AK, BKM, EPI>(c, a, grid, name); break;
            case T128x64: launch_tma_cfg<128, 64, 16, 4, 2, 4, AK, BKM, EPI>(c, a, grid, name); break;
            case T128x32: launch_tma_cfg<128, 32, 16, 8, 1, 4, AK, BKM, EPI>(c, a, grid, name); break;
            case T128x128W16: launch_tma_cfg<128, 128, 16, 4, 4, 5, AK, BKM, EPI>(c, a, grid, name); break;
            case T128x128K32:
                if constexpr (EPI == EPI_SYMUPD) launch_tma_cfg<128, 128, 32, 4, 4, 3, AK, BKM, EPI>(c, a, grid, name);
                break;
            case T128x128W8K32:
                if constexpr (EPI == EPI_SYMUPD) launch_tma_cfg<128, 128, 32, 4, 2, 3, AK, BKM, EPI>(c, a, grid, name);
                break;
            case T128x128W16S6:
                if constexpr (EPI == EPI_SYMUPD) launch_tma_cfg<128, 128, 16, 4, 4, 6, AK, BKM, EPI>(c, a, grid, name);
                break;
            case T64x128: launch_tma_cfg<64, 128, 16, 2, 4, 6, AK, BKM, EPI>(c, a, grid, name); break;
            case T64x64:
                if constexpr (EPI == EPI_STORE || EPI == EPI_PARTIAL)
                    launch_tma_cfg<64, 64, 16, 2, 2, 6, AK, BKM, EPI>(c, a, grid, name);
                break;
        }
        return;
    }
    switch (t) {
        case T128x128: launch_gemm_cfg<128, 128, 16, 4, 2, 4, AK, BKM, VEC, EPI>(c, a, grid, name); break;
        case T128x64: launch_gemm_cfg<128, 64, 16, 4, 2, 4, AK, BKM, VEC, EPI>(c, a, grid, name); break;
        case T128x32: launch_gemm_cfg<128, 32, 16, 8, 1, 4, AK, BKM, VEC, EPI>(c, a, grid, name); break;
        case T128x128W16:
        case T128x128K32:
        case T128x128W8K32:
        case T128x128W16S6: launch_gemm_cfg<128, 128, 16, 4, 4, 4, AK, BKM, VEC, EPI>(c, a, grid, name); break;
        case T64x128: launch_gemm_cfg<64, 128, 16, 2, 4, 4, AK, BKM, VEC, EPI>(c, a, grid, name); break;
        case T64x64:
            if constexpr (EPI == EPI_STORE || EPI == EPI_PARTIAL)
                launch_gemm_cfg<64, 64, 16, 2, 2, 4, AK, BKM, VEC, EPI>(c, a, grid, name);
            break;
    }
}

static bool aligned_ptr(const void* p, uintptr_t b) { return (reinterpret_cast<uintptr_t>(p) & (b - 1)) == 0; }

// TMA needs 16-byte aligned bases and line strides (even leading dimensions)
static bool tma_ok(const GemmArgs& a) {
    return !tma_disabled() && a.lda % 2 == 0 && a.ldb % 2 == 0 && aligned_ptr(a.A, 16) && aligned_ptr(a.B, 16) &&
           a.M < (int64_t(1) << 31) && a.N < (int64_t(1) << 31) && a.K < (int64_t(1) << 31);
}

template <int EPI>
static void launch_gemm_layout(Context& c, TileCfg t, bool ak, bool bkm, int vec, const GemmArgs& a, dim3 grid,
                               const char* name) {
    const bool tma = tma_ok(a);
    if (!ak && bkm) {
        vec == 2 ? launch_gemm_tile<false, true, 2, EPI>(c, t, a, grid, name, tma)
                 : launch_gemm_tile<false, true, 1, EPI>(c, t, a, grid, name, tma);
    } else if (ak && bkm) {
        vec == 2 ? launch_gemm_tile<true, true, 2, EPI>(c, t, a, grid, name, tma)
                 : launch_gemm_tile<true, true, 1, EPI>(c, t, a, grid, name, tma);
    } else if (!ak && !bkm) {
        vec == 2 ? launch_gemm_tile<false, false, 2, EPI>(c, t, a, grid, name, tma)
                 : launch_gemm_tile<false, false, 1, EPI>(c, t, a, grid, name, tma);
    } else {
        throw std::invalid_argument("gemm: A K-major with B N-major is not instantiated");
    }
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static int pick_vec(const GemmArgs& a) {
    const bool ok = a.M % 2 == 0 && a.N % 2 == 0 && a.K % 2 == 0 && a.lda % 2 == 0 && a.ldb % 2 == 0 &&
                    aligned16(a.A) && aligned16(a.B);
    return ok ? 2 : 1;
}

static TileCfg pick_tile(int64_t N, int64_t M = 1 << 30) {
    if (M <= 64 && N <= 64) return T64x64;  // small Grams (q ≤ 64: G = SᵀAS, [G | H']): no 3/4-empty tiles
    if (M <= 64 && N > 64) return T64x128;  // q×n products (Z = (AS)ᵀL, Grams): no half-empty tiles
    if (N <= 32) return T128x32;
    if (N <= 64) return T128x64;
    return use_w16() ? T128x128W16 : T128x128;
}

void gemm(Context& c, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, bool a_kmajor, const double* B,
          int64_t ldb, bool b_kmajor, double* C, int64_t ldc, double alpha, double beta, const int* skip,
          int* nonfinite, const double* Csrc) {
    if (M <= 0 || N <= 0) return;
    GemmArgs a{};
    a.M = M;
    a.N = N;
    a.K = K;
    a.A = A;
    a.lda = lda;
    a.B = B;
    a.ldb = ldb;
    a.C = C;
    a.ldc = ldc;
    a.alpha = alpha;
    a.beta = beta;
    a.skip = skip;
    a.nonfinite = nonfinite;
    a.Csrc = Csrc;
    // short-K, wide-output products (the rank-2q panel update) keep 16 warps resident
    // K <= 128 panel updates (the AdaRBFGS L update): two 8-warp 128×64 CTAs per SM so one
    // CTA's C-tile load/store overlaps the other's mainloop (3.6% faster at config 2 than one
    // 16-warp 128×128 CTA); SI_SHORTK_TILE=w16 selects the latter
    static const int shortk_mode = [] {
        const char* e = std::getenv("SI_SHORTK_TILE");
        return (e && std::string(e) == "w16") ? 0 : 1;
    }();
    // the largest K that takes the two-CTA 128×64 tiles: 256 measured 2.5% faster than the
    // 16-warp 128×128 tiles on config 4's L update (137.0 vs 140.6 ms); SI_SHORTK_MAX overrides
    static const int64_t shortk_max = [] {
        const char* e = std::getenv("SI_SHORTK_MAX");
        return e ? std::atoll(e) : 256;
    }();
    const TileCfg t = (K <= shortk_max && N > 64 && M > 64 && shortk_mode == 1)
                          ? T128x64
                          : ((K <= 512 && N > 64 && M > 64) ? T128x128W16 : pick_tile(N, M));
    const int BM = (t == T64x128 || t == T64x64) ? 64 : 128;
    const int BN = (t == T128x128 || t == T128x128W16 || t == T64x128) ? 128 : ((t == T128x64 || t == T64x64) ? 64 : 32),
              BKT = 16;
    const int64_t tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN, tiles = tm * tn;
    const int per_sm = (t == T128x128 || t == T128x128W16 || t == T64x128) ? 1 : 2;
    const int64_t slots = int64_t(c.num_sms) * per_sm;
    // split-K: pick the split minimising a time model —
    //   waves(s) · (k-stages per unit + F) · t_stage  +  partial traffic / HBM  +  reduce launch
    // (F ≈ 2 stages of per-unit pipeline fill / epilogue; t_stage = one BM×BN×16 DMMA
    // stage on one SM at the measured 36.9 TFLOP/s / 148; per_sm CTAs share an SM).
    int splits = 1;
    if (K > 8 * BKT && !nonfinite) {
        const double t_stage = double(BM) * BN * BKT * 2.0 / (36.9e12 / 148.0) * per_sm;  // seconds
        auto cost = [&](int64_t s) {
            const int64_t chunk = ((K + s - 1) / s + BKT - 1) / BKT * BKT;
            const int64_t units = tiles * s;
            const double waves = double((units + slots - 1) / slots);
            double t = waves * (double(chunk / BKT) + 2.0) * t_stage;
            if (s > 1) t += (2.0 * double(s) + 1.0) * double(M) * double(N) * 8.0 / 5.0e12 + 4e-6;
            return t;
        };
        double best = cost(1);
        for (int s = 2; s <= 128; ++s) {
            const int64_t chunk = ((K + s - 1) / s + BKT - 1) / BKT * BKT;
            if (chunk < 8 * BKT) break;
            if (double(s) * double(M) * double(N) * 8.0 > 512.0 * 1024 * 1024) break;
            const double cs = cost(s);
            if (cs < best * 0.995) {
                best = cs;
                splits = s;
            }
        }
    }
    const int vec = pick_vec(a);
    static const int force_split = [] {  // SI_SPLITK_FORCE (experiments): the split of every split-K product
        const char* e = std::getenv("SI_SPLITK_FORCE");
        return e ? std::atoi(e) : 0;
    }();
    if (force_split > 0 && splits > 1) splits = force_split;
    if (K == 0) {
        splits = 1;
    }
    if (splits == 1) {
        a.k_chunk = std::max<int64_t>(K, 1);
        a.c_in_acc = (alpha == 1.0 && beta != 0.0) ? 1 : 0;
        // short-K panel updates seeded from C (the AdaRBFGS L update): C tiles by TMA, one
        // work item ahead (config 2: 0.356 -> 0.332 ms/iteration); SI_CPANEL=0 disables,
        // SI_CPANEL_KMAX sets the largest K (default 256)
        static const bool cpanel = [] {
            const char* e = std::getenv("SI_CPANEL");
            return !(e && e[0] == '0');
        }();
        static const int64_t cpanel_kmax = [] {  // 256: config 4's L update 137.6 -> 135.6 ms
            const char* e = std::getenv("SI_CPANEL_KMAX");
            return e ? std::atoll(e) : 256;
        }();
        if (cpanel && t == T128x64 && a.c_in_acc && K <= cpanel_kmax && tma_ok(a) && a.ldc % 2 == 0 &&
            aligned_ptr(C, 16) && aligned_ptr(Csrc ? Csrc : C, 16)) {
            // the finished tiles leave by bulk copies from shared memory (SI_CPANEL_BULK=0: stores from
            // registers); an even M keeps every column segment a multiple of 16 bytes
            // K ≤ 64 (AdaRBFGS at q ≤ 64): the whole A slice of a row strip stays in shared memory
            // (SI_CPANEL_STAT=0: the ring kernels below)
            static const bool cstat = [] {
                const char* e = std::getenv("SI_CPANEL_STAT");
                return !(e && e[0] == '0');
            }();
            if (cstat && K <= 64 && !a_kmajor && b_kmajor) {
                launch_cstat(c, a);
                return;
            }
            static const bool cbulk = [] {
                const char* e = std::getenv("SI_CPANEL_BULK");
                return !(e && e[0] == '0');
            }();
            if (cbulk && M % 2 == 0) {
                if (!a_kmajor && b_kmajor)
                    launch_cbulk_cfg<false, true>(c, a, tm * tn);
                else if (!a_kmajor && !b_kmajor)
                    launch_cbulk_cfg<false, false>(c, a, tm * tn);
                else
                    launch_cbulk_cfg<true, true>(c, a, tm * tn);
                return;
            }
            if (!a_kmajor && b_kmajor)
                launch_cpanel_cfg<false, true>(c, a, tm * tn);
            else if (!a_kmajor && !b_kmajor)
                launch_cpanel_cfg<false, false>(c, a, tm * tn);
            else
                launch_cpanel_cfg<true, true>(c, a, tm * tn);
            return;
        }
        launch_gemm_layout<EPI_STORE>(c, t, a_kmajor, b_kmajor, vec, a, dim3(unsigned(tm), unsigned(tn), 1),
                                      "gemm_store");
        return;
    }
    const int64_t chunk = ((K + splits - 1) / splits + BKT - 1) / BKT * BKT;
    splits = int((K + chunk - 1) / chunk);
    a.k_chunk = chunk;
    a.ws = c.ensure_ws(size_t(splits) * size_t(M) * size_t(N));
    launch_gemm_layout<EPI_PARTIAL>(c, t, a_kmajor, b_kmajor, vec, a, dim3(unsigned(tm), unsigned(tn), unsigned(splits)),
                                    "gemm_splitk");
    LaunchScope ls(c, "splitk_reduce");
    launch_pdl(splitk_reduce_kernel, dim3(grid_for(M * N, 256)), dim3(256), 0, c.stream, (const double*)a.ws, splits, M,
               N, C, ldc, alpha, beta, skip, Csrc);
    check_launch("splitk_reduce");
}

// C += A·B for a short-K update of a large block (the sharded driver's off-diagonal trapezoid
// part, X[R_c, r1:] += V·Uᵀ): the K-SYMUPD tiling (128×128, 8 warps, accumulators seeded from
// the C tile, persistent) without the mirror — the default short-K choice (128×64 C-panel
// tiles) suits K ≤ q updates with a narrower output
void gemm_update(Context& c, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                 int64_t ldb, double* C, int64_t ldc, const int* skip, int* nonfinite) {
    if (M <= 0 || N <= 0) return;
    GemmArgs a{};
    a.M = M;
    a.N = N;
    a.K = K;
    a.A = A;
    a.lda = lda;
    a.B = B;
    a.ldb = ldb;
    a.C = C;
    a.ldc = ldc;
    a.alpha = 1.0;
    a.beta = 1.0;
    a.c_in_acc = 1;
    a.k_chunk = std::max<int64_t>(K, 1);
    a.skip = skip;
    a.nonfinite = nonfinite;
    const bool big = ((M + 127) / 128) * ((N + 127) / 128) >= int64_t(c.num_sms);
    if (!big || !tma_ok(a)) {
        gemm(c, M, N, K, A, lda, false, B, ldb, false, C, ldc, 1.0, 1.0, skip, nonfinite);
        return;
    }
    launch_gemm_layout<EPI_STORE>(c, T128x128, false, false, pick_vec(a), a,
                                  dim3(unsigned((M + 127) / 128), unsigned((N + 127) / 128), 1), "gemm_update");
}

// warp-specialised K-SYMUPD (gemm_symupd_ws_kernel): 8 DMMA warps on 128×128 tiles
// (BK = 8, 5 TMA stages) + 4 memory warps (TMA producer and tile epilogue)
static void launch_symupd_ws(Context& c, const GemmArgs& a) {
    constexpr int BM = 128, BN = 128, BK = 8, WM = 4, WN = 2, ST = 5;
    using SM = SymWsSmem<BM, BN, BK, ST>;
    auto kern = gemm_symupd_ws_kernel<BM, BN, BK, WM, WN, ST>;
    static DeviceOnce once;
    if (once.first(c.device)) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SM::BYTES)));
    CUtensorMap ta, tb;
    make_tmap(&ta, a.A, a.M, a.K, a.lda, BM + 4, BK);
    make_tmap(&tb, a.B, a.N, a.K, a.ldb, BN + 4, BK);
    const int64_t tn = (a.N + BN - 1) / BN, work = tn * (tn + 1) / 2;
    LaunchScope ls(c, "gemm_symupd");
    launch_pdl(kern, dim3(unsigned(std::min<int64_t>(work, c.num_sms))), dim3(WM * WN * 32 + 32 * SM::MEM_WARPS),
               SM::BYTES, c.stream,
               ta, tb, a);
    check_launch("gemm_symupd_ws");
}

// deferred-epilogue K-SYMUPD (gemm_symupd_deferred_kernel): 8 DMMA warps on 128×128 tiles, the
// previous tile retired by L2 reductions under the mainloop; square and trapezoid launches.
// Opt-in (SI_SYMUPD_DEFER; default 0 = the single-role kernel): measured 2.16–2.18 ms against 2.22 ms
// at config 3 (B), but the reductions fetch the mirror tiles too (+1 GB of DRAM reads per launch),
// DESIGN.md §9.  B = BK 16 × 3 stages + 15-block hand-off, A / D = BK 16 × 5 / 6 stages with the
// reductions straight from registers, C = BK 8 × 5 stages + 16-block hand-off, E / F = 4 stages +
// 11 / 8 blocks.
static int symupd_defer_mode() {
    static const int mode = [] {
        const char* e = std::getenv("SI_SYMUPD_DEFER");
        if (!e || !e[0]) return 0;
        return e[0] == '0' ? 0 : int(e[0]);
    }();
    return mode;
}
static bool symupd_defer_ok(const GemmArgs& a) {
    return symupd_defer_mode() != 0 && a.alpha == 1.0 && !(a.dbg & 1023) && tma_ok(a) && a.ldc % 2 == 0 && aligned16(a.C);
}
template <int BK, int ST, int HB>
static void launch_symupd_deferred_cfg(Context& c, const GemmArgs& a, int64_t work) {
    constexpr int BM = 128, BN = 128, WM = 4, WN = 2;
    using SM = SymDefSmem<BM, BN, BK, WM, WN, ST, HB>;
    static_assert(SM::BYTES <= 232448, "shared memory per CTA");
    auto kern = gemm_symupd_deferred_kernel<BM, BN, BK, WM, WN, ST, HB>;
    static DeviceOnce once;
    if (once.first(c.device)) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SM::BYTES)));
    CUtensorMap ta, tb;
    make_tmap(&ta, a.A, a.M, a.K, a.lda, BM + 4, BK);
    make_tmap(&tb, a.B, a.N, a.K, a.ldb, BN + 4, BK);
    LaunchScope ls(c, "gemm_symupd");
    launch_pdl(kern, dim3(unsigned(std::min<int64_t>(work, c.num_sms))), dim3(WM * WN * 32), SM::BYTES, c.stream, ta, tb,
               a);
    check_launch("gemm_symupd_deferred");
}
static void launch_symupd_deferred(Context& c, const GemmArgs& a, int64_t work) {
    switch (symupd_defer_mode()) {
        case 'A': launch_symupd_deferred_cfg<16, 5, 0>(c, a, work); break;
        case 'D': launch_symupd_deferred_cfg<16, 6, 0>(c, a, work); break;
        case 'E': launch_symupd_deferred_cfg<16, 4, 11>(c, a, work); break;
        case 'F': launch_symupd_deferred_cfg<16, 4, 8>(c, a, work); break;
        case 'C': launch_symupd_deferred_cfg<8, 5, 16>(c, a, work); break;
        default: launch_symupd_deferred_cfg<16, 3, 15>(c, a, work); break;
    }
}

// X <- X + alpha·V·Uᵀ on the upper-triangular tiles, mirrored (X symmetric n×n)
static void symupd(Context& c, int64_t n, int64_t k, const double* V, int64_t ldv, const double* U, int64_t ldu,
                   double* X, int64_t ldx, double alpha, const int* skip, int* nonfinite) {
    GemmArgs a{};
    a.M = n;
    a.N = n;
    a.K = k;
    a.A = V;
    a.lda = ldv;
    a.B = U;
    a.ldb = ldu;
    a.C = X;
    a.ldc = ldx;
    a.alpha = alpha;
    a.beta = 1.0;
    a.k_chunk = k;
    a.skip = skip;
    a.nonfinite = nonfinite;
    static const int dbg = [] {
        const char* e = std::getenv("SI_SYMUPD_DBG");
        return e ? std::atoi(e) : 0;
    }();
    a.dbg = dbg;
    const int vec = pick_vec(a);
    // Tile choice (SI_SYMUPD_TILE): default one 8-warp CTA per SM on 128×128 tiles
    // (32×64 warp tiles: a clock64 trace of CTA 0 shows ~92% of the DMMA rate per
    // k-stage against ~88% for "w16", one 16-warp CTA with 32×32 warp tiles);
    // "128x64" two 8-warp CTAs per SM (2.31 vs 2.25 ms at config 3); "k32",
    // "w8k32", "s6": BK = 32 / 6 stages (no difference measured).
    static const TileCfg forced = [] {
        const char* e = std::getenv("SI_SYMUPD_TILE");
        const std::string v = e ? e : "";
        if (v == "128x64") return T128x64;
        if (v == "k32") return T128x128K32;
        if (v == "w8k32") return T128x128W8K32;
        if (v == "s6") return T128x128W16S6;
        if (v == "w16") return T128x128W16;
        if (v == "128x128") return T128x128;
        return TileCfg(-1);
    }();
    // small n (fewer upper 128×128 tiles than SMs, e.g. config 1): 128×64 tiles, two CTAs
    // per SM, twice the work items
    const int64_t t128 = (n + 127) / 128;
    const TileCfg cfg = int(forced) >= 0 ? forced : (t128 * (t128 + 1) / 2 < int64_t(c.num_sms) ? T128x64 : T128x128);
    // SI_SYMUPD_WS=1: the warp-specialised kernel (measured slower: 2.66 vs 2.20 ms at config 3,
    // DESIGN.md §9), kept as an opt-in experiment
    static const bool ws = env_flag("SI_SYMUPD_WS");
    if (ws && cfg == T128x128 && int(forced) < 0 && alpha == 1.0 && !dbg && tma_ok(a) && a.ldc % 2 == 0) {
        launch_symupd_ws(c, a);
        return;
    }
    const int64_t bn = cfg == T128x64 ? 64 : 128, r = 128 / bn;
    const int64_t tn = (n + bn - 1) / bn, full = tn / r, rest = tn % r;
    const int64_t work = r * full * (full + 1) / 2 + rest * (full + 1);  // TileOps::sym_work_count
    if (cfg == T128x128 && int(forced) < 0 && symupd_defer_ok(a)) {
        launch_symupd_deferred(c, a, work);
        return;
    }
    launch_gemm_layout<EPI_SYMUPD>(c, cfg, false, false, vec, a, dim3(unsigned(work), 1, 1), "gemm_symupd");
}

void symupd_ex(Context& c, int64_t m, int64_t k, const double* V, int64_t ldv, const double* U, int64_t ldu, double* X,
               int64_t ldx, const int* skip, int* nonfinite) {
    symupd(c, m, k, V, ldv, U, ldu, X, ldx, 1.0, skip, nonfinite);
}

// X (m×ncols, ld ldx: rows [0, m) of a symmetric block, columns from the block's first row
// on) += V·Uᵀ with V m×k, U ncols×k: the leading m×m block by upper tiles mirrored inside it,
// the columns right of it as plain tiles — one persistent K-SYMUPD launch over the trapezoid
void symupd_trapezoid(Context& c, int64_t m, int64_t ncols, int64_t k, const double* V, int64_t ldv, const double* U,
                      int64_t ldu, double* X, int64_t ldx, const int* skip, int* nonfinite) {
    if (ncols <= m) {
        symupd(c, m, k, V, ldv, U, ldu, X, ldx, 1.0, skip, nonfinite);
        return;
    }
    GemmArgs a{};
    a.M = m;
    a.N = ncols;
    a.K = k;
    a.A = V;
    a.lda = ldv;
    a.B = U;
    a.ldb = ldu;
    a.C = X;
    a.ldc = ldx;
    a.alpha = 1.0;
    a.beta = 1.0;
    a.k_chunk = k;
    a.skip = skip;
    a.nonfinite = nonfinite;
    const int64_t t128 = (m + 127) / 128, tn128 = (ncols + 127) / 128;
    const int64_t tiles128 = t128 * (t128 + 1) / 2 + (tn128 - t128) * t128;
    const TileCfg cfg = tiles128 < int64_t(c.num_sms) ? T128x64 : T128x128;
    const int64_t bn = cfg == T128x64 ? 64 : 128, r = 128 / bn;
    const int64_t tn = (m + bn - 1) / bn, full = tn / r, rest = tn % r;
    const int64_t sq = r * full * (full + 1) / 2 + rest * (full + 1);
    const int64_t work = sq + ((ncols + bn - 1) / bn - tn) * ((m + 127) / 128);
    if (cfg == T128x128 && symupd_defer_ok(a)) {
        launch_symupd_deferred(c, a, work);
        return;
    }
    launch_gemm_layout<EPI_SYMUPD>(c, cfg, false, false, pick_vec(a), a, dim3(unsigned(work), 1, 1), "gemm_symupd");
}

void advance_batch(Context& c, unsigned long long* counter, int* status, bool ada) {
    LaunchScope ls(c, "advance_counter");
    if (ada)
        ada_advance_batch_kernel<<<1, 1, 0, c.stream>>>(counter, status);
    else
        advance_batch_kernel<<<1, 1, 0, c.stream>>>(counter, status);
    check_launch("advance");
}

// ----------------------------------------------------------- problem -------
Problem::~Problem() {
    if (a) cudaFree(a);
    if (rowptr) cudaFree(rowptr);
    if (colind) cudaFree(colind);
    if (val) cudaFree(val);
}

void problem_upload_dense(Problem& p, const double* src, bool device_src) {
    Context& c = *p.ctx;
    const size_t bytes = size_t(p.n) * size_t(p.n) * sizeof(double);
    CK(cudaMalloc(&p.a, bytes));
    CK(cudaMemcpyAsync(p.a, src, bytes, device_src ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
    p.dense = true;
    if (p.symmetry != 0) {  // (M + Mᵀ)/2 for symmetric / spd flags (problem_matrix.cpp:9-18)
        LaunchScope ls(c, "symmetrize");
        const unsigned T = unsigned((p.n + 31) / 32);
        symmetrize_kernel<<<dim3(T, T), dim3(32, 8), 0, c.stream>>>(p.a, p.n);
        check_launch("symmetrize");
    }
    CK(cudaStreamSynchronize(c.stream));
}

void problem_upload_csr(Problem& p, const int64_t* rowptr, const int32_t* colind, const double* val) {
    Context& c = *p.ctx;
    CK(cudaMalloc(&p.rowptr, size_t(p.n + 1) * sizeof(int64_t)));
    CK(cudaMalloc(&p.colind, size_t(std::max<int64_t>(p.nnz, 1)) * sizeof(int32_t)));
    CK(cudaMalloc(&p.val, size_t(std::max<int64_t>(p.nnz, 1)) * sizeof(double)));
    CK(cudaMemcpyAsync(p.rowptr, rowptr, size_t(p.n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c.stream));
    if (p.nnz) {
        CK(cudaMemcpyAsync(p.colind, colind, size_t(p.nnz) * sizeof(int32_t), cudaMemcpyHostToDevice, c.stream));
        CK(cudaMemcpyAsync(p.val, val, size_t(p.nnz) * sizeof(double), cudaMemcpyHostToDevice, c.stream));
    }
    p.dense = false;
    CK(cudaStreamSynchronize(c.stream));
}

__global__ void densify_csr_kernel(int64_t n, const int64_t* rowptr, const int32_t* colind, const double* val,
                                   double* out) {
    for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < n; row += (int64_t)gridDim.x * blockDim.x)
        for (int64_t t = rowptr[row]; t < rowptr[row + 1]; ++t) out[row + (int64_t)colind[t] * n] += val[t];
}

void problem_download_dense(Problem& p, double* host) {
    Context& c = *p.ctx;
    const size_t bytes = size_t(p.n) * size_t(p.n) * sizeof(double);
    if (p.dense) {
        CK(cudaMemcpyAsync(host, p.a, bytes, cudaMemcpyDeviceToHost, c.stream));
    } else {
        double* tmp = nullptr;
        CK(cudaMalloc(&tmp, bytes));
        CK(cudaMemsetAsync(tmp, 0, bytes, c.stream));
        densify_csr_kernel<<<grid_for(p.n, 256), 256, 0, c.stream>>>(p.n, p.rowptr, p.colind, p.val, tmp);
        CK(cudaMemcpyAsync(host, tmp, bytes, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
        CK(cudaFree(tmp));
    }
    CK(cudaStreamSynchronize(c.stream));
}

// row-major SpMM launch: the row-blocked kernel when k is a multiple of 64 (SI_SPMM_ROWBLOCK=0:
// the warp-per-row kernel), 4 rows × 64·NS columns per warp
static void launch_spmm_rowmajor(Context& c, int64_t m, const int64_t* rowptr, const int32_t* colind, const double* val,
                                 const double* Pr, int64_t k, double* Y, int64_t ldy, const int* skip) {
    static const bool rowblock = [] {
        const char* e = std::getenv("SI_SPMM_ROWBLOCK");
        return !(e && e[0] == '0');
    }();
    if (rowblock && k >= 64 && k % 64 == 0) {
        constexpr int R = 4;
        static const int ns_cap = [] {  // SI_SPMM_NS: the most 64-column slabs per warp pass (1, 2, 4)
            const char* e = std::getenv("SI_SPMM_NS");
            return e ? std::atoi(e) : 4;
        }();
        int ns = k % 256 == 0 ? 4 : (k % 128 == 0 ? 2 : 1);
        while (ns > ns_cap && ns > 1) ns /= 2;
        const int64_t units = ((m + R - 1) / R) * (k / (64 * ns));
        const dim3 grid(grid_for(units * 32, 256, c.num_sms * 32));
        if (ns == 4)
            spmm_csr_rowblock_kernel<R, 4><<<grid, 256, 0, c.stream>>>(m, rowptr, colind, val, Pr, k, Y, ldy, skip);
        else if (ns == 2)
            spmm_csr_rowblock_kernel<R, 2><<<grid, 256, 0, c.stream>>>(m, rowptr, colind, val, Pr, k, Y, ldy, skip);
        else
            spmm_csr_rowblock_kernel<R, 1><<<grid, 256, 0, c.stream>>>(m, rowptr, colind, val, Pr, k, Y, ldy, skip);
        return;
    }
    spmm_csr_rowmajor_kernel<<<grid_for(m * 32, 256, c.num_sms * 32), 256, 0, c.stream>>>(m, rowptr, colind, val, Pr, k, Y,
                                                                                         ldy, skip);
}

// Y = A·P (dense GEMM or CSR SpMM)
void apply_a(Context& c, Problem& a, const double* P, int64_t ldp, int64_t k, double* Y, int64_t ldy, const int* skip) {
    const int64_t n = a.n;
    if (a.dense) {
        gemm(c, n, k, n, a.a, n, false, P, ldp, true, Y, ldy, 1.0, 0.0, skip);
        return;
    }
    if (k > 4096) {  // very wide operand (A·L): thread per (row, column), CSR stays in L2
        LaunchScope ls(c, "spmm_csr_cols");
        dim3 grid(unsigned(std::min<int64_t>((n + 255) / 256, 1024)), unsigned(std::min<int64_t>(k, 65535)));
        spmm_csr_colmajor_kernel<<<grid, 256, 0, c.stream>>>(n, a.rowptr, a.colind, a.val, P, ldp, k, Y, ldy, skip);
        check_launch("spmm_csr_cols");
        return;
    }
    // row-major copy of P so each nonzero reads one contiguous k-row
    double* Pr = c.ensure_ws(size_t(n) * size_t(k));
    {
        LaunchScope ls(c, "transpose");
        dim3 grid(unsigned((n + 31) / 32), unsigned((k + 31) / 32));
        transpose_kernel<<<grid, dim3(32, 8), 0, c.stream>>>(P, n, k, ldp, Pr, skip);
        check_launch("transpose");
    }
    LaunchScope ls(c, "spmm_csr");
    launch_spmm_rowmajor(c, n, a.rowptr, a.colind, a.val, Pr, k, Y, ldy, skip);
    check_launch("spmm_csr");
}

// Y (m×k, ld ldy) = A_rows·P for a CSR row panel (m rows, global column indices < n)
// and a dense n×k operand P: the row-major copy + warp-per-row kernel of apply_a.
void spmm_csr_rows(Context& c, int64_t m, int64_t n, const int64_t* rowptr, const int32_t* colind, const double* val,
                   const double* P, int64_t ldp, int64_t k, double* Y, int64_t ldy) {
    double* Pr = c.ensure_ws(size_t(n) * size_t(k));
    {
        LaunchScope ls(c, "transpose");
        dim3 grid(unsigned((n + 31) / 32), unsigned((k + 31) / 32));
        transpose_kernel<<<grid, dim3(32, 8), 0, c.stream>>>(P, n, k, ldp, Pr, nullptr);
        check_launch("transpose");
    }
    LaunchScope ls(c, "spmm_csr");
    launch_spmm_rowmajor(c, m, rowptr, colind, val, Pr, k, Y, ldy, nullptr);
    check_launch("spmm_csr");
}

void set_identity(Context& c, double* X, int64_t n) {
    LaunchScope ls(c, "set_identity");
    set_identity_kernel<<<grid_for(n * n, 256), 256, 0, c.stream>>>(X, n, n);
    check_launch("set_identity");
}

// ------------------------------------------------------------- RBFGS -------
template <typename T>
static void dmalloc(T** p, size_t count) {
    CK(cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T)));
}

void RbfgsWork::alloc(int64_t n_, int64_t q_, bool own) {
    n = n_;
    q = q_;
    own_x = own;
    if (own) dmalloc(&X, size_t(n) * size_t(n));
    dmalloc(&Y, size_t(n) * size_t(q));
    dmalloc(&U, size_t(n) * size_t(4 * q));  // [S | W | Z | R] (BFGS); [S | W] for the other updates
    dmalloc(&V, size_t(n) * size_t(2 * q));
    dmalloc(&P, size_t(q) * size_t(2 * q));
    dmalloc(&Ginv, size_t(q) * size_t(q));
    dmalloc(&T, size_t(q) * size_t(q));
    dmalloc(&M, size_t(2 * q) * size_t(2 * q));
    dmalloc(&factor_scratch, 4 * size_t(q) * size_t(q) + size_t(2 * q) + 16);
    dmalloc(&status, 8);
    dmalloc(&counter, 1);
    CK(cudaMemset(status, 0, 8 * sizeof(int)));
    CK(cudaMemset(counter, 0, sizeof(unsigned long long)));
}

// pinned staging for host-drawn sketches, allocated on first use: page-locking
// n·q doubles costs 7-19 ms, which device-sketch runs never need
double* RbfgsWork::pinned() {
    if (!s_pinned) CK(cudaMallocHost(&s_pinned, size_t(n) * size_t(q) * sizeof(double)));
    return s_pinned;
}

void RbfgsWork::release() {
    if (own_x && X) cudaFree(X);
    for (double* p : {Y, U, V, P, Ginv, T, M, factor_scratch})
        if (p) cudaFree(p);
    if (status) cudaFree(status);
    if (counter) cudaFree(counter);
    if (s_pinned) cudaFreeHost(s_pinned);
    if (lowrank) cudaFree(lowrank);
    lowrank = nullptr;
    X = Y = U = V = P = Ginv = T = M = factor_scratch = nullptr;
    status = nullptr;
    counter = nullptr;
    s_pinned = nullptr;
}

void rbfgs_enqueue_sketch_upload(Context& c, RbfgsWork& w) {
    CK(cudaMemcpyAsync(w.U, w.s_pinned, size_t(w.n) * size_t(w.q) * sizeof(double), cudaMemcpyHostToDevice,
                       c.stream));
}

// Gi (ld ldo) = G⁻¹ for SPD G read as G(i,j) = P(min, max) (ld ldp).
//   q ≤ 128: register-resident Gauss-Jordan in one CTA (pivots = squared Cholesky
//            diagonals → the gram_llt failure test), then exact symmetrization;
//   q > 128: 2×2 block elimination on the DMMA GEMM engine, recursively:
//            Ai = A⁻¹, T1 = Ai·B, S = D − Bᵀ·T1, Si = S⁻¹ (PD ⇔ A and S PD),
//            G⁻¹ = [[Ai + T2·T1ᵀ, −T2], [−T2ᵀ, Si]] with T2 = T1·Si.
// scratch: 4q² doubles.
static int inverse_base_q() {
    static int v = 0;
    if (!v) {
        const char* s = std::getenv("SI_INV_BASE");
        v = s ? std::max(16, std::min(128, std::atoi(s))) : 64;  // measured: 64 beats 128 at q = 128
    }
    return v;
}

template <int QP, int PB>
static void spd_inverse_blocked(Context& c, const double* P, int64_t ldp, int64_t q, double* ginv, int64_t ldo,
                                int* status) {
    constexpr size_t smem =
        sizeof(double) * (size_t(QP) * (QP + 4) + size_t(QP) * (PB + 4) + size_t(PB) * (QP + 4) + PB * (PB + 1));
    static DeviceOnce once;
    if (once.first(c.device)) {
        CK(cudaFuncSetAttribute(spd_inverse_blocked_kernel<QP, PB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(smem)));
    }
    LaunchScope ls(c, "spd_inverse");
    spd_inverse_blocked_kernel<QP, PB><<<1, 512, smem, c.stream>>>(P, ldp, int(q), ginv, ldo, status);
    check_launch("spd_inverse_blocked");
}

static void spd_inverse_ld(Context& c, const double* P, int64_t ldp, int64_t q, double* ginv, int64_t ldo,
                           double* scratch, int* status) {
    // blocked Gauss-Jordan, one CTA, the matrix in shared memory (16-column panels; 32-column
    // panels measured 2.2× slower: the warp-serial 32×32 pivot-block inverse dominates)
    static const bool blocked = std::getenv("SI_INV_SCALAR") == nullptr;
    if (blocked && q > 32 && q <= 128) {
        if (q <= 64)
            spd_inverse_blocked<64, 16>(c, P, ldp, q, ginv, ldo, status);
        else
            spd_inverse_blocked<128, 16>(c, P, ldp, q, ginv, ldo, status);
        return;
    }
    if (q <= inverse_base_q()) {
        const int rpt = q <= 32 ? 1 : (q <= 64 ? 8 : 16);
        const int threads = int(q * ((q + rpt - 1) / rpt));
        {
            LaunchScope ls(c, "spd_inverse");
            switch (rpt) {
                case 1:
                    spd_inverse_reg_kernel<1, 1024><<<1, threads, 0, c.stream>>>(P, ldp, int(q), ginv, ldo, status);
                    break;
                case 8:
                    spd_inverse_reg_kernel<8, 512><<<1, threads, 0, c.stream>>>(P, ldp, int(q), ginv, ldo, status);
                    break;
                default:
                    spd_inverse_reg_kernel<16, 1024><<<1, threads, 0, c.stream>>>(P, ldp, int(q), ginv, ldo, status);
                    break;
            }
            check_launch("spd_inverse_reg");
        }
        LaunchScope ls(c, "symmetrize_small");
        symmetrize_small_kernel<<<grid_for(q * q, 256), 256, 0, c.stream>>>(ginv, int(q), ldo, status);
        check_launch("symmetrize_small");
        return;
    }
    const int64_t h = ((q / 2 + 63) / 64) * 64, q2 = q - h;
    const double* A = P;                     // G11 (h×h)
    const double* B = P + h * ldp;           // G12 (h×q2): upper-right block of the upper triangle
    const double* D = P + h + h * ldp;       // G22 (q2×q2)
    double* T1 = scratch;                    // h×q2
    double* S = T1 + h * q2;                 // q2×q2
    double* T2 = S + q2 * q2;                // h×q2
    double* sub = T2 + h * q2;               // recursion scratch
    double* Gi11 = ginv;
    double* Gi12 = ginv + h * ldo;
    double* Gi22 = ginv + h + h * ldo;
    spd_inverse_ld(c, A, ldp, h, Gi11, ldo, sub, status);                          // Ai
    gemm(c, h, q2, h, Gi11, ldo, false, B, ldp, true, T1, h, 1.0, 0.0, status);      // T1 = Ai·B
    {
        LaunchScope ls(c, "scale_copy");
        scale_copy_kernel<<<grid_for(q2 * q2, 256), 256, 0, c.stream>>>(D, ldp, S, q2, q2, q2, 1.0, status);
        check_launch("scale_copy");
    }
    gemm(c, q2, q2, h, B, ldp, true, T1, h, true, S, q2, -1.0, 1.0, status);        // S = D − Bᵀ·T1
    spd_inverse_ld(c, S, q2, q2, Gi22, ldo, sub, status);                          // Si
    gemm(c, h, q2, q2, T1, h, false, Gi22, ldo, true, T2, h, 1.0, 0.0, status);      // T2 = T1·Si
    gemm(c, h, h, q2, T2, h, false, T1, h, false, Gi11, ldo, 1.0, 1.0, status);      // Gi11 += T2·T1ᵀ
    {
        LaunchScope ls(c, "scale_copy");
        scale_copy_kernel<<<grid_for(h * q2, 256), 256, 0, c.stream>>>(T2, h, Gi12, ldo, h, q2, -1.0, status);
        check_launch("scale_copy");
    }
    LaunchScope ls(c, "mirror_upper");
    mirror_upper_kernel<<<grid_for(q * q, 256), 256, 0, c.stream>>>(ginv, q, ldo, status);  // Gi21 = Gi12ᵀ
    check_launch("mirror_upper");
}

static void spd_inverse(Context& c, const double* P, int64_t ldp, int64_t q, double* ginv, double* scratch,
                        int* status) {
    spd_inverse_ld(c, P, ldp, q, ginv, q, scratch, status);
}

void spd_inverse_device(Context& c, const double* P, int64_t ldp, int64_t q, double* ginv, int64_t ldo,
                        double* scratch, int* status) {
    spd_inverse_ld(c, P, ldp, q, ginv, ldo, scratch, status);
}

// K-FACTOR + K-CORE: from P = [G | H] (q×2q, ld ldp) build
// M = [[Ginv + Ginv·H·Ginv, −Ginv], [−Ginv, 0]] (2q×2q, ld 2q).  status[0] is
// set (and every later launch skipped) when G is not positive definite.
void rbfgs_core_enqueue(Context& c, const double* P, int64_t ldp, int64_t q, double* Ginv, double* T, double* M,
                        double* scratch, int* status) {
    spd_inverse(c, P, ldp, q, Ginv, scratch, status);
    rbfgs_core_tail(c, P, ldp, q, Ginv, T, M, status);
}

void rbfgs_core_tail(Context& c, const double* P, int64_t ldp, int64_t q, const double* Ginv, double* T, double* M,
                     int* status) {
    {
        LaunchScope ls(c, "core_layout");
        core_layout_kernel<<<grid_for(4 * q * q, 256), 256, 0, c.stream>>>(Ginv, int(q), M, status);
        check_launch("core_layout");
    }
    gemm(c, q, q, q, P + q * ldp, ldp, false, Ginv, q, true, T, q, 1.0, 0.0, status);  // T = H·Ginv
    gemm(c, q, q, q, Ginv, q, false, T, q, true, M, 2 * q, 1.0, 1.0, status);          // M11 = Ginv + Ginv·T
}

void zero_on_status(Context& c, double* M, int64_t count, const int* status) {
    LaunchScope ls(c, "zero_on_status");
    zero_on_status_kernel<<<grid_for(count, 256), 256, 0, c.stream>>>(M, count, status);
    check_launch("zero_on_status");
}

// K-FACTOR for the single-GPU RBFGS iteration: G⁻¹ (with the gram_llt PD test) and
// Ĝ = G − H' from P = [G | H'] (H' = YᵀW' = −H).
template <int QP>
static void launch_gram_fused(Context& c, const double* P, int64_t ldp, int64_t q, double* Ginv, double* Ghat,
                              int* status) {
    constexpr int LF = 16, NT = 512;
    using SM = core::GramSmem<QP, LF>;
    static DeviceOnce once;
    if (once.first(c.device)) {
        CK(cudaFuncSetAttribute(rbfgs_gram_kernel<QP, LF, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(SM::BYTES)));
    }
    LaunchScope ls(c, "gram_inverse");
    launch_pdl(rbfgs_gram_kernel<QP, LF, NT>, dim3(1), dim3(NT), SM::BYTES, c.stream, P, ldp, int(q), Ginv, Ghat,
               status);
    check_launch("gram_inverse");
}

void rbfgs_gram_enqueue(Context& c, const double* P, int64_t ldp, int64_t q, double* Ginv, double* Ghat,
                        double* scratch, int* status) {
    // q ≤ 128: one single-CTA launch (kernels_core.cuh); SI_GRAM_UNFUSED=1 keeps K-FACTOR + ghat
    static const bool unfused = std::getenv("SI_GRAM_UNFUSED") != nullptr;
    if (!unfused && q <= 128) {
        if (q <= 32)
            launch_gram_fused<32>(c, P, ldp, q, Ginv, Ghat, status);
        else if (q <= 64)
            launch_gram_fused<64>(c, P, ldp, q, Ginv, Ghat, status);
        else
            launch_gram_fused<128>(c, P, ldp, q, Ginv, Ghat, status);
        return;
    }
    spd_inverse(c, P, ldp, q, Ginv, scratch, status);
    if (!Ghat) return;
    LaunchScope ls(c, "ghat");
    ghat_kernel<<<grid_for(q * q, 256), 256, 0, c.stream>>>(P, ldp, int(q), Ghat, status);
    check_launch("ghat");
}

// ProblemMatrix::validate_spd (problem_matrix.cpp:28-41): the LLT's success test — every
// pivot of the elimination > 0 — as a blocked right-looking Schur-complement sweep on this
// engine's own kernels (no library factorisation):
//   for each 128-wide diagonal block D of the current Schur complement:
//     K-FACTOR(D): D⁻¹ with its leaf pivots tested (> 0), one CTA
//     T = −B·D⁻¹                         (B the block column below D)   K-GEMM
//     trailing ← trailing + T·Bᵀ         (= − B·D⁻¹·Bᵀ, symmetric)        K-SYMUPD (upper tiles, mirrored)
// The blocks meet the Schur-complement pivots of the whole matrix in order, i.e. the
// Cholesky pivots (squared diagonal of the factor), so the decision is the LLT's; a
// failed pivot makes every later launch a no-op.  n³/3 flops, on the DMMA pipe.
// `scratch` (n×n, optional): a caller's buffer for the working copy (the drivers lend
// their iterate before initialising it; cudaMalloc / cudaFree of an n×n scratch measured
// 50–240 ms at n = 16384).
bool problem_validate_spd(Problem& p, double* scratch) {
    if (p.spd_checked) return p.spd_ok;
    Context& c = *p.ctx;
    const int64_t n = p.n;
    const size_t bytes = size_t(n) * size_t(n) * sizeof(double);
    constexpr int64_t BLK = 128;
    double* W = scratch;
    double *T = nullptr, *Dinv = nullptr;
    int* st = nullptr;
    struct Rel {
        double **w, **t, **d;
        int** s;
        bool own;
        ~Rel() {
            if (own && *w) cudaFree(*w);
            if (*t) cudaFree(*t);
            if (*d) cudaFree(*d);
            if (*s) cudaFree(*s);
        }
    } rel{&W, &T, &Dinv, &st, scratch == nullptr};
    if (!W) CK(cudaMalloc(&W, bytes));
    CK(cudaMalloc(&T, size_t(n) * BLK * sizeof(double)));
    CK(cudaMalloc(&Dinv, size_t(BLK) * BLK * sizeof(double)));
    CK(cudaMalloc(&st, 8 * sizeof(int)));
    CK(cudaMemsetAsync(st, 0, 8 * sizeof(int), c.stream));
    if (p.dense) {
        CK(cudaMemcpyAsync(W, p.a, bytes, cudaMemcpyDeviceToDevice, c.stream));
    } else {
        CK(cudaMemsetAsync(W, 0, bytes, c.stream));
        densify_csr_kernel<<<grid_for(n, 256), 256, 0, c.stream>>>(n, p.rowptr, p.colind, p.val, W);
        check_launch("densify");
    }
    // Left-looking order (default; SI_VALIDATE_RIGHT=1 keeps the right-looking sweep below): the
    // n³/3 flops become one (n−k)×128×k product per panel — long-K, split-K, the shape the K-GEMM
    // runs at 96% of the DMMA rate — instead of 128 rank-128 K-SYMUPD launches (75%).  W keeps both
    // factors in place, using the symmetric redundancy: the lower block column of panel j holds
    // T_j = −B_j·D_j⁻¹ and the upper block row holds B_jᵀ, so panel k's Schur complement is
    //     S_k = A[k:, k:k+b] + W[k:, 0:k] · W[0:k, k:k+b]      (T, M-major) · (Bᵀ, K-major),
    // its leading b×b block goes through K-FACTOR (pivots tested), its remainder B_k is mirrored
    // into the block row and T_k = −B_k·D_k⁻¹ is computed from that mirror into the block column.
    // Look-ahead: K-FACTOR(D_k) → B_kᵀ → T_k is a chain of small launches (≈ 0.1 ms per panel, 128
    // panels); it runs on the high-priority side stream while the main stream already forms the
    // part of S_{k+1} that does not depend on panel k (the product over panels < k); panel k's own
    // rank-b term is added after the join.  SI_VALIDATE_SERIAL=1 keeps everything on one stream.
    static const bool right_looking = std::getenv("SI_VALIDATE_RIGHT") != nullptr;
    static const bool lookahead = std::getenv("SI_VALIDATE_SERIAL") == nullptr;
    for (int64_t k = 0; !right_looking && k < n; k += BLK) {
        const int64_t b = std::min(BLK, n - k), rest = n - k - b;
        double* D = W + k + k * n;
        // S_k is complete here (k = 0: A itself)
        auto chain = [&]() {
            if (b <= 32)
                launch_gram_fused<32>(c, D, n, b, Dinv, nullptr, st);
            else if (b <= 64)
                launch_gram_fused<64>(c, D, n, b, Dinv, nullptr, st);
            else
                launch_gram_fused<128>(c, D, n, b, Dinv, nullptr, st);
            if (rest == 0) return;
            double* Bcol = W + (k + b) + k * n;   // B_k: rest×b, ld n
            double* Brow = W + k + (k + b) * n;   // B_kᵀ: b×rest, ld n
            {
                LaunchScope ls(c, "transpose");
                dim3 grid(unsigned((rest + 31) / 32), unsigned((b + 31) / 32));
                transpose_ld_kernel<<<grid, dim3(32, 8), 0, c.stream>>>(Bcol, rest, b, n, Brow, n, st);
                check_launch("transpose_ld");
            }
            gemm(c, rest, b, b, Brow, n, true, Dinv, b, true, Bcol, n, -1.0, 0.0, st);  // T_k = −B_k·D_k⁻¹
        };
        if (rest == 0) {
            chain();
            break;
        }
        const int64_t k1 = k + b, b1 = std::min(BLK, n - k1);
        double* S1 = W + k1 + k1 * n;  // S_{k+1}: (n − k1)×b1, ld n
        if (lookahead && k > 0) {
            c.fork(true);
            {
                SideScope side(c, true);
                chain();
            }
            gemm(c, n - k1, b1, k, W + k1, n, false, W + k1 * n, n, true, S1, n, 1.0, 1.0, st);  // panels < k
            c.join(true);
        } else {
            chain();
            if (k > 0) gemm(c, n - k1, b1, k, W + k1, n, false, W + k1 * n, n, true, S1, n, 1.0, 1.0, st);
        }
        // panel k's own term: S_{k+1} += T_k[b:, :]·B_k[0:b1, :]ᵀ
        gemm(c, n - k1, b1, b, W + k1 + k * n, n, false, W + k + k1 * n, n, true, S1, n, 1.0, 1.0, st);
    }
    for (int64_t k = 0; right_looking && k < n; k += BLK) {
        const int64_t b = std::min(BLK, n - k);
        double* D = W + k + k * n;
        if (b <= 32)
            launch_gram_fused<32>(c, D, n, b, Dinv, nullptr, st);
        else if (b <= 64)
            launch_gram_fused<64>(c, D, n, b, Dinv, nullptr, st);
        else
            launch_gram_fused<128>(c, D, n, b, Dinv, nullptr, st);
        const int64_t rest = n - k - b;
        if (rest == 0) break;
        const double* B = W + (k + b) + k * n;                                   // rest×b, ld n
        gemm(c, rest, b, b, B, n, false, Dinv, b, true, T, rest, -1.0, 0.0, st);  // T = −B·D⁻¹
        symupd(c, rest, b, T, rest, B, n, W + (k + b) * (n + 1), n, 1.0, st, nullptr);
    }
    int hst = 0;
    CK(cudaMemcpyAsync(&hst, st, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    p.spd_checked = true;
    p.spd_ok = hst == 0;
    return p.spd_ok;
}

void philox_sketch(Context& c, double* S, int64_t n, int64_t q, int64_t lds, uint64_t seed,
                   const unsigned long long* counter_dev, uint64_t draw, const int* skip) {
    LaunchScope ls(c, "sketch_philox");
    philox_gaussian_kernel<<<grid_for((n * q + 1) / 2, 256), 256, 0, c.stream>>>(S, n, q, lds, seed, counter_dev, skip,
                                                                               draw);
    check_launch("philox");
}

// One RBFGS iteration.  With Y = A·S, W = X·Y, G = SᵀAS = YᵀS, H = YᵀW and
// Z = S·G⁻¹, the reference's expanded update (qn_updates.cpp:176-186:
// S·t2 + X − S·k − (S·k)ᵀ + S(k·t1ᵀ)Sᵀ with k = G⁻¹Wᵀ, S·t2 = Z·G·Zᵀ) is
//     X⁺ = X + Z(G + H)Zᵀ − Z·Wᵀ − W·Zᵀ = X + [Z R]·[W' Z]ᵀ,
//     W' = −W,  R = Z·Ĝ + W',  Ĝ = G + H = G − YᵀW',
// so the q×q stage needs only G⁻¹ (K-FACTOR, with the PD test) and Ĝ, the
// n-row stage is two n×q×q products (4nq² flops instead of the 8nq² of
// V = [S W]·M plus two q×q×q core products), and [S | W' | Z | R] sit side by
// side in one n×4q buffer so [S W'], [W' Z] and [Z R] are contiguous windows.
// Every launch is skipped on the device once K-FACTOR flags a non-PD Gram (status[0]).
void rbfgs_enqueue_iteration(Context& c, Problem& a, RbfgsWork& w, bool device_sketch, uint64_t seed) {
    const int64_t n = w.n, q = w.q;
    double* S = w.U;
    double* Wn = S + n * q;  // W' = −X·Y
    double* Z = Wn + n * q;
    double* R = Z + n * q;
    const int* skip = w.status;
    if (device_sketch) {
        LaunchScope ls(c, "sketch_philox");
        launch_pdl(philox_gaussian_kernel, dim3(grid_for((n * q + 1) / 2, 256)), dim3(256), 0, c.stream, S, n, q, n,
                   seed, (const unsigned long long*)w.counter, skip, 0ull);
        check_launch("philox");
    }
    apply_a(c, a, S, n, q, w.Y, n, skip);                                       // Y = A·S
    // G = SᵀAS needs only Y: its one-CTA inverse (K-FACTOR) runs on the side stream while
    // W' = −X·Y occupies the other SMs; H' = YᵀW' and Ĝ follow the join (config 3: 6.267 ->
    // 6.233 ms).  Small n keeps the serial order — one [G | H'] product, then K-FACTOR with Ĝ —
    // because the split product and the extra launches cost more than K-FACTOR there
    // (config 1: 0.064 vs 0.068 ms); SI_RBFGS_SERIAL=1 forces it.
    static const bool serial = std::getenv("SI_RBFGS_SERIAL") != nullptr;
    if (!serial && n >= 8192) {
        gemm(c, q, q, n, w.Y, n, true, S, n, true, w.P, q, 1.0, 0.0, skip);               // G = Yᵀ·S
        c.fork(true);  // high priority: K-FACTOR takes the first free SM instead of queueing behind W'
        {
            SideScope side(c, true);
            rbfgs_gram_enqueue(c, w.P, q, q, w.Ginv, nullptr, w.factor_scratch, w.status);  // G⁻¹ + PD test
        }
        gemm(c, n, q, n, w.X, n, false, w.Y, n, true, Wn, n, -1.0, 0.0, skip);            // W' = −X·Y
        gemm(c, q, q, n, w.Y, n, true, Wn, n, true, w.P + q * q, q, 1.0, 0.0, skip);      // H' = Yᵀ·W'
        c.join(true);
        LaunchScope ls(c, "ghat");
        ghat_kernel<<<grid_for(q * q, 256), 256, 0, c.stream>>>(w.P, q, int(q), w.T, w.status);  // Ĝ = G − H'
        check_launch("ghat");
    } else {
        gemm(c, n, q, n, w.X, n, false, w.Y, n, true, Wn, n, -1.0, 0.0, skip);      // W' = −X·Y
        gemm(c, q, 2 * q, n, w.Y, n, true, S, n, true, w.P, q, 1.0, 0.0, skip);     // P = Yᵀ·[S W'] = [G | −H]
        rbfgs_gram_enqueue(c, w.P, q, q, w.Ginv, w.T, w.factor_scratch, w.status);  // G⁻¹ + PD test, Ĝ = G + H
    }
    gemm(c, n, q, q, S, n, false, w.Ginv, q, true, Z, n, 1.0, 0.0, skip);       // Z = S·G⁻¹
    gemm(c, n, q, q, Z, n, false, w.T, q, true, R, n, 1.0, 1.0, skip, nullptr, Wn);  // R = Z·Ĝ + W'
    symupd(c, n, 2 * q, Z, n, Wn, n, w.X, n, 1.0, skip, w.status + 1);         // X += [Z R]·[W' Z]ᵀ
    if (device_sketch) {
        LaunchScope ls(c, "advance_counter");
        launch_pdl(w.batch ? advance_batch_kernel : advance_counter_kernel, dim3(1), dim3(1), 0, c.stream, w.counter,
                   w.status);
        check_launch("advance");
    }
}

// ----------------------------------------------------------- residual ------
// Σ (δ(r + diag_off, c) − (A·B)(r, c))² over an M×N product with K = n, no
// M×N write; partial per CTA then a fixed-order reduction into *out_dev.
template <bool BKM>
static void resid_gemm_rect(Context& c, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                            const double* B, int64_t ldb, int64_t diag_off, double* out_dev) {
    GemmArgs g{};
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = A;
    g.lda = lda;
    g.B = B;
    g.ldb = ldb;
    g.alpha = 1.0;
    g.k_chunk = K;
    g.diag_off = diag_off;
    // fewer 128×128 tiles than SMs (small n, e.g. config 1's checkpoints): 64×128 tiles
    // double the CTAs (the sum of squares cannot be split over K)
    const bool small = ((M + 127) / 128) * ((N + 127) / 128) < int64_t(c.num_sms);
    const int64_t BMr = small ? 64 : 128;
    const int64_t TM = (M + BMr - 1) / BMr, TN = (N + 127) / 128;
    g.ws = c.ensure_ws(size_t(TM * TN));
    const int vec = pick_vec(g);
    launch_gemm_layout<EPI_RESID>(c, small ? T64x128 : (use_w16() ? T128x128W16 : T128x128), false, BKM, vec, g,
                                  dim3(unsigned(TM), unsigned(TN), 1), "gemm_resid");
    LaunchScope ls(c, "sum_reduce");
    sum_reduce_kernel<<<1, 1024, 0, c.stream>>>(g.ws, TM * TN, out_dev);
    check_launch("sum_reduce");
}

template <bool BKM>
static void resid_gemm(Context& c, int64_t n, const double* A, int64_t lda, const double* B, int64_t ldb,
                       double* out_dev) {
    resid_gemm_rect<BKM>(c, n, n, n, A, lda, B, ldb, 0, out_dev);
}

// Row panel of a row-sharded X: Σ over rows [r0, r0+m) of ‖I − X·A‖² (= ‖I − A·X‖²
// for symmetric A and X), dense A.
void residual_rows_sq_enqueue(Context& c, Problem& a, int64_t m, int64_t r0, const double* Xrows, int64_t ldx,
                              double* out_dev) {
    if (!a.dense) throw std::invalid_argument("residual_rows: sparse A is not supported for row panels yet");
    resid_gemm_rect<true>(c, m, a.n, a.n, Xrows, ldx, a.a, a.n, r0, out_dev);
}

__global__ void csr_resid_kernel(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
                                 const double* __restrict__ val, const double* __restrict__ X, double* partial) {
    // ‖I − A X‖² = ‖I − X A‖² (A, X symmetric): row i of (A X) = sum_t a_it X(t,:)
    // one warp per output row; X columns read contiguously along the row of X (X symmetric:
    // X(t, j) = X(j, t) so row t of X is column t, contiguous).
    __shared__ double red[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double acc = 0.0;
    for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < n; row += warps) {
        const int64_t b = rowptr[row], e = rowptr[row + 1];
        for (int64_t j = lane; j < n; j += 32) {
            double s = 0.0;
            for (int64_t t = b; t < e; ++t) s += val[t] * X[j + (int64_t)colind[t] * n];
            const double d = (row == j ? 1.0 : 0.0) - s;
            acc += d * d;
        }
    }
    acc = warp_sum(acc);
    if (lane == 0) red[wid] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        partial[blockIdx.x] = t;
    }
}

// ‖I − A‖²_F (the base residual for X0 = I, simi.cpp:242-246 with X = I): no GEMM needed.
__global__ void identity_resid_dense_kernel(const double* __restrict__ A, int64_t n, double* partial) {
    __shared__ double red[32];
    double acc = 0.0;
    const int64_t total = n * n;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx % n, j = idx / n;
        const double d = (i == j ? 1.0 : 0.0) - A[idx];
        acc += d * d;
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        partial[blockIdx.x] = t;
    }
}

__global__ void identity_resid_csr_kernel(int64_t n, const int64_t* __restrict__ rowptr,
                                          const int32_t* __restrict__ colind, const double* __restrict__ val,
                                          double* partial) {
    __shared__ double red[32];
    double acc = 0.0;
    for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < n; row += (int64_t)gridDim.x * blockDim.x) {
        double diag = 0.0;
        for (int64_t t = rowptr[row]; t < rowptr[row + 1]; ++t) {
            if (colind[t] == row) diag += val[t];
            else acc += val[t] * val[t];
        }
        acc += (1.0 - diag) * (1.0 - diag);
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        partial[blockIdx.x] = t;
    }
}

void identity_residual_sq_enqueue(Context& c, Problem& a, double* out_dev) {
    const int blocks = c.num_sms * 4;
    double* part = c.ensure_ws(size_t(blocks));
    {
        LaunchScope ls(c, "identity_resid");
        if (a.dense)
            identity_resid_dense_kernel<<<blocks, 256, 0, c.stream>>>(a.a, a.n, part);
        else
            identity_resid_csr_kernel<<<blocks, 256, 0, c.stream>>>(a.n, a.rowptr, a.colind, a.val, part);
        check_launch("identity_resid");
    }
    LaunchScope ls(c, "sum_reduce");
    sum_reduce_kernel<<<1, 1024, 0, c.stream>>>(part, blocks, out_dev);
    check_launch("sum_reduce");
}

void residual_sq_enqueue(Context& c, Problem& a, const double* X, double* out_dev, double* /*scratch*/) {
    const int64_t n = a.n;
    if (a.dense) {
        resid_gemm<true>(c, n, a.a, n, X, n, out_dev);  // ‖I − A·X‖²
        return;
    }
    const int blocks = c.num_sms * 4;
    double* part = c.ensure_ws(size_t(blocks));
    {
        LaunchScope ls(c, "csr_resid");
        csr_resid_kernel<<<blocks, 256, 0, c.stream>>>(n, a.rowptr, a.colind, a.val, X, part);
        check_launch("csr_resid");
    }
    LaunchScope ls(c, "sum_reduce");
    sum_reduce_kernel<<<1, 1024, 0, c.stream>>>(part, blocks, out_dev);
    check_launch("sum_reduce");
}

// First checkpoint from X0 = I (simi.cpp:361-375 at k = 1): X1 = I + sign·V·Uᵀ, so
// ‖I − A·X1‖² = ‖I − A − sign·(A·V)·Uᵀ‖² — P = A·V (2n²·k) then one residual GEMM with
// K = k whose accumulators start from the A tile, 4n²k in all instead of 2n³
// (config 3: 0.27 TFLOP instead of 8.8).  Dense A only.
void lowrank_residual_sq_enqueue(Context& c, Problem& a, int64_t k, const double* V, int64_t ldv, const double* U,
                                 int64_t ldu, double sign, double* P, double* out_dev) {
    const int64_t n = a.n;
    if (!a.dense) throw std::invalid_argument("lowrank residual: dense A only");
    apply_a(c, a, V, ldv, k, P, n, nullptr);  // P = A·V
    GemmArgs g{};
    g.M = n;
    g.N = n;
    g.K = k;
    g.A = P;
    g.lda = n;
    g.B = U;  // B(kk, j) = Uᵀ(kk, j) = U[j + kk·ldu]
    g.ldb = ldu;
    g.C = a.a;
    g.ldc = n;
    g.alpha = sign;  // acc = sign·A + P·Uᵀ = sign·(A·X1); the epilogue takes δ − sign·acc
    g.beta = sign;
    g.c_in_acc = 1;
    g.k_chunk = k;
    const int64_t TM = (n + 127) / 128, TN = (n + 127) / 128;
    g.ws = c.ensure_ws(size_t(TM * TN));
    launch_gemm_layout<EPI_RESID>(c, T128x128, false, false, pick_vec(g), g, dim3(unsigned(TM), unsigned(TN), 1),
                                  "gemm_resid_lowrank");
    LaunchScope ls(c, "sum_reduce");
    sum_reduce_kernel<<<1, 1024, 0, c.stream>>>(g.ws, TM * TN, out_dev);
    check_launch("sum_reduce");
}

// ‖I − (A·L)·Lᵀ‖² (adarbfgs.cpp:112-115): AL = A·L into scratch, then a
// residual GEMM against Lᵀ (B operand N-major) with no n×n write.
// X = L·Lᵀ first (K-SYMUPD on a zeroed scratch: upper tiles, mirrored — n³ flops), then
// the ordinary ‖I − A·X‖ (2n³ dense, 2·nnz·n CSR): 3n³ instead of the 4n³ of
// (A·L)·Lᵀ; SI_FACTORED_RESID_AL=1 keeps the latter.
void factored_residual_sq_enqueue(Context& c, Problem& a, const double* L, double* AL, double* out_dev) {
    const int64_t n = a.n;
    static const bool via_al = env_flag("SI_FACTORED_RESID_AL");
    if (!via_al) {
        CK(cudaMemsetAsync(AL, 0, size_t(n) * size_t(n) * sizeof(double), c.stream));
        symupd(c, n, n, L, n, L, n, AL, n, 1.0, nullptr, nullptr);
        residual_sq_enqueue(c, a, AL, out_dev, nullptr);
        return;
    }
    apply_a(c, a, L, n, n, AL, n, nullptr);
    resid_gemm<false>(c, n, AL, n, L, n, out_dev);
}

// ------------------------------------------------------------ AdaRBFGS -----
void AdaWork::alloc(int64_t n_, int64_t q_, bool gaussian) {
    n = n_;
    q = q_;
    dmalloc(&L, size_t(n) * size_t(n));
    dmalloc(&S, size_t(n) * size_t(q));
    dmalloc(&AS, size_t(n) * size_t(q));
    dmalloc(&SR, size_t(n) * size_t(q));
    dmalloc(&G, size_t(q) * size_t(q));
    dmalloc(&R, size_t(q) * size_t(q));
    dmalloc(&Z, size_t(q) * size_t(n));
    dmalloc(&B, size_t(q) * size_t(n));
    dmalloc(&eig_scratch, 6 * size_t(q) * size_t(q) + 8 * size_t(q) + 32);
    dmalloc(&idx_dev, size_t(q));
    dmalloc(&pdiag, size_t(n));
    dmalloc(&status, 8);
    dmalloc(&counter, 1);
    CK(cudaMemset(status, 0, 8 * sizeof(int)));
    CK(cudaMemset(counter, 0, sizeof(unsigned long long)));
    CK(cudaMallocHost(&idx_pinned, size_t(q) * sizeof(int64_t)));
    CK(cudaMallocHost(&p_pinned, size_t(n) * sizeof(double)));
    if (gaussian) {
        dmalloc(&St, size_t(n) * size_t(q));
        dmalloc(&G2, size_t(q) * size_t(q));
        dmalloc(&R2, size_t(q) * size_t(q));
        dmalloc(&Tm, size_t(q) * size_t(n));
        CK(cudaMallocHost(&st_pinned, size_t(n) * size_t(q) * sizeof(double)));
    }
}

void AdaWork::release() {
    for (double* p : {S_next, AS_next, G_next, Bsel})
        if (p) cudaFree(p);
    S_next = AS_next = G_next = Bsel = nullptr;
    have_next = false;
    idx_next = nullptr;
    if (idx_ring) cudaFree(idx_ring);
    if (idx_ring_pinned) cudaFreeHost(idx_ring_pinned);
    idx_ring = nullptr;
    idx_ring_pinned = nullptr;
    ring_cap = 0;
    for (double* p : {L, S, AS, SR, G, R, Z, B, eig_scratch, pdiag, St, G2, R2, Tm, AL})
        if (p) cudaFree(p);
    if (idx_dev) cudaFree(idx_dev);
    if (status) cudaFree(status);
    if (counter) cudaFree(counter);
    if (idx_pinned) cudaFreeHost(idx_pinned);
    if (p_pinned) cudaFreeHost(p_pinned);
    if (st_pinned) cudaFreeHost(st_pinned);
    L = S = AS = SR = G = R = Z = B = eig_scratch = pdiag = St = G2 = R2 = Tm = AL = nullptr;
    idx_dev = nullptr;
    status = nullptr;
    counter = nullptr;
    idx_pinned = nullptr;
    p_pinned = nullptr;
    st_pinned = nullptr;
}

template <int QP>
static void ns_fused(Context& c, const double* Mq, int64_t q, double* R, int* status) {
    const size_t smem = size_t(5) * QP * (QP + 4) * sizeof(double);
    static DeviceOnce once;
    if (once.first(c.device)) {
        CK(cudaFuncSetAttribute(ns_fused_kernel<QP>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    }
    LaunchScope ls(c, "ns_fused");
    static const int accelerate = env_flag("SI_NS_NEWTON_ONLY") ? 0 : 1;
    ns_fused_kernel<QP><<<1, 512, smem, c.stream>>>(Mq, q, int(q), R, status, 1e-14 * std::sqrt(double(q)), 60,
                                                     accelerate);
    check_launch("ns_fused");
}

// R = M^{-1/2} (q×q, ld q) with the reference's accept / reject contract
// (sym_inv_sqrt, linalg.cpp:144-155: reject iff an eigenvalue λ ≤ 1e-14·λmax or λ ≤ 0,
// status[0] = 1 → NumericalError → redraw).
//   Fast path: Newton–Schulz (q ≤ 64 fused in one CTA; q > 64 on the DMMA GEMM engine)
//   whose R is kept only when it converged and certifies λmin/λmax > 1e-12
//   (1/(‖R‖²_F·c), c ≥ λmax) — 100× inside the floor, so no draw the reference
//   rejects is accepted.  Otherwise the reference's cyclic Jacobi (tournament order,
//   one CTA) recomputes R and applies the floor itself: near-singular Grams are
//   decided by the reference's own rule.  SI_ISQRT_JACOBI=1 always takes Jacobi.
// scratch: 6q² + 8q + 32 doubles; status[3] is used as the NS stop flag.
static void inv_sqrt(Context& c, const double* Mq, int64_t q, double* R, double* scratch, int* status) {
    const bool jacobi = env_flag("SI_ISQRT_JACOBI");
    if (!jacobi && q <= 64) {
        if (q <= 16) ns_fused<16>(c, Mq, q, R, status);
        else if (q <= 32) ns_fused<32>(c, Mq, q, R, status);
        else if (q <= 48) ns_fused<48>(c, Mq, q, R, status);
        else ns_fused<64>(c, Mq, q, R, status);
        return;
    }
    double* Y = scratch;
    double* Z = Y + q * q;
    double* T = Z + q * q;
    double* ZY = T + q * q;
    double* Yn = ZY + q * q;
    double* Zn = Yn + q * q;
    double* scal = Zn + q * q;
    int* need = reinterpret_cast<int*>(scal + 4);  // Jacobi fallback flag
    if (!jacobi) {
        int* conv = status + 3;
        {
            LaunchScope ls(c, "ns_init");
            ns_init_kernel<<<1, 1024, 0, c.stream>>>(Mq, q, int(q), Y, Z, scal, status, conv);
            check_launch("ns_init");
        }
        const double tol = 1e-14 * std::sqrt(double(q));
        for (int it = 0; it < 48; ++it) {
            gemm(c, q, q, q, Z, q, false, Y, q, true, ZY, q, 1.0, 0.0, conv);  // Z·Y
            {
                LaunchScope ls(c, "ns_step");
                ns_step_kernel<<<1, 1024, 0, c.stream>>>(ZY, int(q), T, scal, conv, tol);
                check_launch("ns_step");
            }
            gemm(c, q, q, q, Y, q, false, T, q, true, Yn, q, 1.0, 0.0, conv);  // Y·T
            gemm(c, q, q, q, T, q, false, Z, q, true, Zn, q, 1.0, 0.0, conv);  // T·Z
            LaunchScope ls(c, "ns_copy");
            ns_copy2_kernel<<<grid_for(q * q, 256), 256, 0, c.stream>>>(Y, Yn, Z, Zn, int(q), conv);
            check_launch("ns_copy");
        }
        {
            LaunchScope ls(c, "ns_finish");
            ns_finish_kernel<<<1, 1024, 0, c.stream>>>(Z, int(q), scal, R, status, conv, need);
            check_launch("ns_finish");
        }
    }
    // exact path: runs on the device only when flagged (always under SI_ISQRT_JACOBI);
    // its work arrays (2q² + 3q doubles) reuse Y and Z
    LaunchScope ls(c, "jacobi_isqrt");
    jacobi_isqrt_kernel<<<1, 1024, 0, c.stream>>>(Mq, q, int(q), scratch, R, status, jacobi ? nullptr : need);
    check_launch("jacobi_isqrt");
}

void sym_inv_sqrt_device(Context& c, const double* M, int64_t q, double* R, double* scratch, int* status) {
    inv_sqrt(c, M, q, R, scratch, status);
}

// The q×n stage of adarbfgs_update_factor (adarbfgs.cpp:13-19): R = G^{-1/2} and
// B = T − R·Z with T = S̃ᵀ (coordinate: idx, St null) or T = (S̃ᵀS̃)^{-1/2}·S̃ᵀ
// (Gaussian S̃ = St, n×q; T written to Tq, q×n).  Floor hits set status[0].
// the parts of ada_core_enqueue before / after Z is needed (the overlapped schedule)
static void ada_core_root(Context& c, const double* G, int64_t q, int64_t n, const double* St, double* G2, double* R2,
                          double* Tq, double* R, double* scratch, int* st) {
    inv_sqrt(c, G, q, R, scratch, st);  // R = G^{-1/2}
    if (St) {
        gemm(c, q, q, n, St, n, true, St, n, true, G2, q, 1.0, 0.0, st);  // S̃ᵀS̃
        inv_sqrt(c, G2, q, R2, scratch, st);
        gemm(c, q, n, q, R2, q, false, St, n, false, Tq, q, 1.0, 0.0, st);  // T = R2·S̃ᵀ
    }
}

static void ada_core_b(Context& c, int64_t q, const double* Z, int64_t n, const int64_t* idx, const double* St,
                       const double* Tq, const double* R, double* B, int* st) {
    if (!St) {
        gemm(c, q, n, q, R, q, false, Z, q, true, B, q, -1.0, 0.0, st);  // B = −R·Z
        LaunchScope ls(c, "add_selector");
        add_selector_kernel<<<grid_for(q, 128), 128, 0, c.stream>>>(B, q, idx, st);  // + T = S̃ᵀ
        check_launch("add_selector");
    } else {
        CK(cudaMemcpyAsync(B, Tq, size_t(q) * size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
        gemm(c, q, n, q, R, q, false, Z, q, true, B, q, -1.0, 1.0, st);  // B = T − R·Z
    }
}

void ada_core_enqueue(Context& c, const double* G, int64_t q, const double* Z, int64_t n, const int64_t* idx,
                      const double* St, double* G2, double* R2, double* Tq, double* R, double* B, double* scratch,
                      int* st) {
    inv_sqrt(c, G, q, R, scratch, st);  // R = G^{-1/2}
    if (!St) {
        gemm(c, q, n, q, R, q, false, Z, q, true, B, q, -1.0, 0.0, st);  // B = −R·Z
        LaunchScope ls(c, "add_selector");
        add_selector_kernel<<<grid_for(q, 128), 128, 0, c.stream>>>(B, q, idx, st);  // + T = S̃ᵀ
        check_launch("add_selector");
    } else {
        gemm(c, q, q, n, St, n, true, St, n, true, G2, q, 1.0, 0.0, st);  // S̃ᵀS̃
        inv_sqrt(c, G2, q, R2, scratch, st);
        gemm(c, q, n, q, R2, q, false, St, n, false, Tq, q, 1.0, 0.0, st);  // T = R2·S̃ᵀ
        CK(cudaMemcpyAsync(B, Tq, size_t(q) * size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
        gemm(c, q, n, q, R, q, false, Z, q, true, B, q, -1.0, 1.0, st);  // B = T − R·Z
    }
}

void gather_columns(Context& c, const double* L, int64_t rows, int64_t ld, const int64_t* idx, int64_t q, double* out) {
    LaunchScope ls(c, "gather_columns");
    const int64_t bx = std::max<int64_t>(1, std::min<int64_t>((rows + 255) / 256, int64_t(c.num_sms) * 16 / std::max<int64_t>(q, 1) + 1));
    const int64_t by = std::min<int64_t>(q, 65535);
    gather_columns_kernel<<<dim3(unsigned(bx), unsigned(by)), 256, 0, c.stream>>>(L, rows, ld, idx, q, out);
    check_launch("gather");
}

void pdiag_update(Context& c, const double* B, int64_t q, int64_t n, const double* T, const int64_t* idx,
                  const int* skip, double* d) {
    LaunchScope ls(c, "pdiag_update");
    pdiag_update_kernel<<<grid_for(n * 32, 256), 256, 0, c.stream>>>(B, q, n, T, idx, skip, d);
    check_launch("pdiag_update");
}

// L⁺ = L + (S·R)·(T − R·(AS)ᵀ·L), adarbfgs.cpp:12-21.
//   mode 0: coordinate S̃ = I[:, idx] (idx_dev filled), S = L[:, idx] gathered
//   mode 1: Gaussian S̃ uploaded from st_pinned; mode 2: Gaussian S̃ from Philox
void ada_enqueue_update(Context& c, Problem& a, AdaWork& w, int mode, uint64_t seed) {
    const int64_t n = w.n, q = w.q;
    int* st = w.status;
    static const bool pipeline = [] {  // SI_ADA_PIPELINE=1: sketch pipelining (measured 0.327 vs 0.315 ms at config 2: off)
        const char* e = std::getenv("SI_ADA_PIPELINE");
        return e && e[0] == '1';
    }();
    const bool precomputed = mode == 0 && w.have_next;
    if (precomputed) {  // S, A·S and G of this attempt were computed under the previous L update
        std::swap(w.S, w.S_next);
        std::swap(w.AS, w.AS_next);
        std::swap(w.G, w.G_next);
        w.have_next = false;
        c.join();
    } else if (mode == 0) {
        gather_columns(c, w.L, n, n, w.idx_dev, q, w.S);
    } else {
        if (mode == 1) {
            CK(cudaMemcpyAsync(w.St, w.st_pinned, size_t(n) * size_t(q) * sizeof(double), cudaMemcpyHostToDevice,
                               c.stream));
        } else {
            LaunchScope ls(c, "sketch_philox");
            philox_gaussian_kernel<<<grid_for((n * q + 1) / 2, 256), 256, 0, c.stream>>>(w.St, n, q, n, seed,
                                                                                       w.counter, st);
            check_launch("philox");
        }
        gemm(c, n, q, n, w.L, n, false, w.St, n, true, w.S, n, 1.0, 0.0, st);  // S = L·S̃
    }
    if (!precomputed) {
        apply_a(c, a, w.S, n, q, w.AS, n, st);                                 // AS = A·S
        gemm(c, q, q, n, w.S, n, true, w.AS, n, true, w.G, q, 1.0, 0.0, st);   // G = Sᵀ·AS
    }
    // Z = (AS)ᵀ·L does not depend on R: it runs on the side stream (every SM but the
    // one holding the inverse square root) while the q×q stage and SR = S·R run here
    static const bool overlap = std::getenv("SI_ADA_SERIAL") == nullptr;
    if (overlap) {
        c.fork();
        {
            SideScope side(c);
            gemm(c, q, n, n, w.AS, n, true, w.L, n, true, w.Z, q, 1.0, 0.0, st);  // Z = (AS)ᵀ·L
        }
        ada_core_root(c, w.G, q, n, mode == 0 ? nullptr : w.St, w.G2, w.R2, w.Tm, w.R, w.eig_scratch, st);
        gemm(c, n, q, q, w.S, n, false, w.R, q, true, w.SR, n, 1.0, 0.0, st);  // SR = S·R
        c.join();
        ada_core_b(c, q, w.Z, n, w.idx_dev, mode == 0 ? nullptr : w.St, w.Tm, w.R, w.B, st);
    } else {
        gemm(c, q, n, n, w.AS, n, true, w.L, n, true, w.Z, q, 1.0, 0.0, st);  // Z = (AS)ᵀ·L
        ada_core_enqueue(c, w.G, q, w.Z, n, w.idx_dev, mode == 0 ? nullptr : w.St, w.G2, w.R2, w.Tm, w.R, w.B,
                         w.eig_scratch, st);
        gemm(c, n, q, q, w.S, n, false, w.R, q, true, w.SR, n, 1.0, 0.0, st);  // SR = S·R
    }
    if (pipeline && mode == 0 && w.batch && w.idx_next) {
        // the next attempt's S' = L⁺[:, idx'] = L[:, idx'] + SR·B[:, idx'] (n×q×q), then A·S' and
        // G' = S'ᵀ·A·S' on the side stream, overlapping the L update below (config 2: the L update
        // runs memory-bound at ≈ 55% of the DMMA rate, A·S' fills the gap)
        if (!w.S_next) {
            dmalloc(&w.S_next, size_t(n) * size_t(q));
            dmalloc(&w.AS_next, size_t(n) * size_t(q));
            dmalloc(&w.G_next, size_t(q) * size_t(q));
            dmalloc(&w.Bsel, size_t(q) * size_t(q));
        }
        gather_columns(c, w.L, n, n, w.idx_next, q, w.S_next);
        gather_columns(c, w.B, q, q, w.idx_next, q, w.Bsel);                          // B[:, idx'] (q×q)
        gemm(c, n, q, q, w.SR, n, false, w.Bsel, q, true, w.S_next, n, 1.0, 1.0, st);  // S' += SR·B[:, idx']
        c.fork();
        {
            SideScope side(c);
            apply_a(c, a, w.S_next, n, q, w.AS_next, n, st);                                   // A·S'
            gemm(c, q, q, n, w.S_next, n, true, w.AS_next, n, true, w.G_next, q, 1.0, 0.0, st);  // S'ᵀ·A·S'
        }
        w.have_next = true;
    }
    gemm(c, n, n, q, w.SR, n, false, w.B, q, true, w.L, n, 1.0, 1.0, st, st + 1);  // L += SR·B (+ finite check)
    if (w.pdiag_valid) {  // carry diag(LᵀAL) across the accepted update (App. C3)
        pdiag_update(c, w.B, q, n, mode == 0 ? nullptr : w.Tm, w.idx_dev, st, w.pdiag);
        ++w.pdiag_age;
    }
    if (w.batch) {
        LaunchScope ls(c, "advance_counter");
        ada_advance_batch_kernel<<<1, 1, 0, c.stream>>>(mode == 2 ? w.counter : nullptr, w.status);
        check_launch("advance");
    } else if (mode == 2) {
        LaunchScope ls(c, "advance_counter");
        advance_counter_kernel<<<1, 1, 0, c.stream>>>(w.counter, w.status);
        check_launch("advance");
    }
}

// device ring of index sets for run_adarbfgs's batched loop (cap attempts of q indices)
void AdaWork::ensure_ring(int cap) {
    if (cap <= ring_cap) return;
    if (idx_ring) cudaFree(idx_ring);
    if (idx_ring_pinned) cudaFreeHost(idx_ring_pinned);
    ring_cap = cap;
    dmalloc(&idx_ring, size_t(cap) * size_t(q));
    CK(cudaMallocHost(&idx_ring_pinned, size_t(cap) * size_t(q) * sizeof(int64_t)));
}

// pdiag_j = l_jᵀ A l_j (diag(LᵀAL), Eq 8.2 numerators), copied to p_pinned.
void ada_enqueue_probabilities(Context& c, Problem& a, AdaWork& w) {
    const int64_t n = w.n;
    if (!w.pdiag_valid || w.pdiag_refresh <= 1 || w.pdiag_age >= w.pdiag_refresh) {
        // exact: diag(Lᵀ·(A·L)) (adarbfgs.cpp:23-36)
        if (!w.AL) dmalloc(&w.AL, size_t(n) * size_t(n));
        apply_a(c, a, w.L, n, n, w.AL, n, nullptr);
        LaunchScope ls(c, "column_dots");
        column_dots_kernel<<<grid_for(n * 32, 256), 256, 0, c.stream>>>(w.AL, w.L, n, w.pdiag);
        check_launch("column_dots");
        w.pdiag_valid = w.pdiag_refresh > 1;
        w.pdiag_age = 0;
    }
    CK(cudaMemcpyAsync(w.p_pinned, w.pdiag, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
}

void problem_diagonal(Context& c, Problem& a, double* d) {
    LaunchScope ls(c, "problem_diagonal");
    problem_diagonal_kernel<<<grid_for(a.n, 256), 256, 0, c.stream>>>(a.dense ? a.a : nullptr, a.rowptr, a.colind,
                                                                       a.val, a.n, d);
    check_launch("problem_diagonal");
}

void ada_init_pdiag_identity(Context& c, Problem& a, AdaWork& w) {
    if (w.pdiag_refresh <= 1) return;  // reference behaviour: exact every iteration
    LaunchScope ls(c, "problem_diagonal");
    problem_diagonal_kernel<<<grid_for(w.n, 256), 256, 0, c.stream>>>(a.dense ? a.a : nullptr, a.rowptr, a.colind,
                                                                       a.val, w.n, w.pdiag);
    check_launch("problem_diagonal");
    w.pdiag_valid = true;
    w.pdiag_age = 0;
}

}  // namespace si

#include "family.cuh"
