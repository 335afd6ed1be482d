// Multi-GPU C ABI and the sharded RBFGS / AdaRBFGS drivers.
//
// A multi-GPU si_context drives P ranks — several devices of this process
// (si_context_create_multi, ncclCommInitAll), one device per process
// (si_context_create_rank: torchrun / MPI style, ncclCommInitRank), or P virtual ranks on
// one device (si_context_create_loopback, the single-GPU test harness).  si_run_inverter,
// si_run_adarbfgs and the si_solver_* calls on such a context run the iteration sharded,
// with the reference's run-level semantics (checkpoint schedule, HistoryPoints, tol /
// time-budget termination, redraw limit, non-finite guard, the checkpoint callback):
//
// RBFGS — the upper triangle of X in 2P row chunks, rank g owning chunks g and 2P−1−g
// (balanced triangle work), each stored as its trapezoid X[R_c, r0_c:n]; A replicated:
//     S            Philox(seed, draw) on every rank (no traffic), or the host RngStream bytes
//     Y[R_c]       = A[R_c, :]·S                                 local          2·m·n·q
//     Y            = all-gather                                  NCCL           n×q
//     W'loc        = −(X_c·Y[r0:] at rows R_c, X_c[:, m:]ᵀ·Y[R_c] at rows r1:)       4·area·q
//     [G | H']loc  = Σ_c Y[R_c]ᵀS[R_c] | Y[r0:]ᵀ·W'loc[r0:]
//     [W' | G | H'] = all-reduce(one packed buffer)               NCCL           n·q + 2q²
//     K-FACTOR     G⁻¹ (PD test) and Ĝ = G − H'                  replicated, one CTA
//     Z = S·G⁻¹ (rows ≥ r0), R[R_c] = Z[R_c]·Ĝ + W'[R_c]
//     X_c         += [R Z][R_c]·[Z W'][r0:]ᵀ   (diagonal block by K-SYMUPD: exactly symmetric)
//   — per rank ≈ 6n²q/P flops, the single-GPU count split evenly; two collectives per
//   iteration; the iterations between checkpoints are captured once as a CUDA graph per
//   stream (collectives included) and replayed.
// AdaRBFGS — L row-sharded in P contiguous panels L_p = L[R_p, :]; A replicated:
//     S_p = L_p[:, C] or L_p·S̃; S = all-gather; (AS)_p = A[R_p, :]·S;
//     [G | Z] = all-reduce([S_pᵀ(AS)_p | (AS)_pᵀL_p]); R = G^{-1/2}, B = T − R·Z replicated;
//     L_p += (S_p·R)·B; the Eq. 8.2 diagonal carried on the replicated B (App. C3).
// Checkpoints use no n×n gather: RBFGS rebuilds its chunks' full rows from the trapezoids
// (each off-diagonal block sent once, point to point) and sums ‖I − X[R_c,:]·A‖² with one
// scalar all-reduce; AdaRBFGS forms X[R_p, :] = L_p·Lᵀ by streaming the panels (broadcast).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <tuple>

#include "capi_internal.hpp"
#include "shard.hpp"

using namespace si_capi;

namespace si {

// ------------------------------------------------------------------ NCCL --
namespace {

struct NcclApi {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommInitAll) commInitAll = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
};

// NCCL is loaded on first use: the copy already in the process when there is one (torch
// bundles its own libnccl.so.2 — loading a second copy would clash), else SI_NCCL_LIBRARY
// or the system libnccl.so.2.
const NcclApi& nccl() {
    static const NcclApi api = [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) {
            const char* path = std::getenv("SI_NCCL_LIBRARY");
            h = dlopen(path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) throw CudaError(std::string("NCCL is unavailable: ") + dlerror());
        NcclApi a;
        auto sym = [&](auto& f, const char* name) {
            f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
            if (!f) throw CudaError(std::string("NCCL symbol missing: ") + name);
        };
        sym(a.getUniqueId, "ncclGetUniqueId");
        sym(a.commInitRank, "ncclCommInitRank");
        sym(a.commInitAll, "ncclCommInitAll");
        sym(a.commDestroy, "ncclCommDestroy");
        sym(a.allReduce, "ncclAllReduce");
        sym(a.allGather, "ncclAllGather");
        sym(a.broadcast, "ncclBroadcast");
        sym(a.send, "ncclSend");
        sym(a.recv, "ncclRecv");
        sym(a.groupStart, "ncclGroupStart");
        sym(a.groupEnd, "ncclGroupEnd");
        sym(a.errorString, "ncclGetErrorString");
        return a;
    }();
    return api;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + nccl().errorString(r));
}

void dev(Context* c) { cuda_check(cudaSetDevice(c->device), "cudaSetDevice"); }

}  // namespace

struct NcclComm : Comm {
    std::vector<ncclComm_t> comms;  // one per local rank
    ~NcclComm() override {
        for (auto c : comms)
            if (c) nccl().commDestroy(c);
    }
    void group_start() override { nck(nccl().groupStart(), "ncclGroupStart"); }
    void group_end() override { nck(nccl().groupEnd(), "ncclGroupEnd"); }
    void all_reduce(int l, void* buf, size_t count, bool is_int, RedOp op, cudaStream_t s) override {
        nck(nccl().allReduce(buf, buf, count, is_int ? ncclInt32 : ncclFloat64, op == RedOp::sum ? ncclSum : ncclMax,
                             comms[size_t(l)], s),
            "ncclAllReduce");
    }
    void all_gather(int l, const double* send, double* recv, size_t count, cudaStream_t s) override {
        nck(nccl().allGather(send, recv, count, ncclFloat64, comms[size_t(l)], s), "ncclAllGather");
    }
    void broadcast(int l, const double* send, double* recv, size_t count, int root, cudaStream_t s) override {
        nck(nccl().broadcast(send, recv, count, ncclFloat64, root, comms[size_t(l)], s), "ncclBroadcast");
    }
    void send(int l, const double* buf, size_t count, int peer, cudaStream_t s) override {
        nck(nccl().send(buf, count, ncclFloat64, peer, comms[size_t(l)], s), "ncclSend");
    }
    void recv(int l, double* buf, size_t count, int peer, cudaStream_t s) override {
        nck(nccl().recv(buf, count, ncclFloat64, peer, comms[size_t(l)], s), "ncclRecv");
    }
};

// P virtual ranks on one device sharing one stream: collectives are recorded until the
// group ends and then replayed as device copies and element-wise reductions in rank order.
struct LoopbackComm : Comm {
    Context* c0 = nullptr;
    struct Op {
        int kind;  // 0 all_reduce, 1 all_gather, 2 broadcast, 3 send, 4 recv
        int l;
        const void* src;
        void* dst;
        size_t count;
        bool is_int;
        RedOp op;
        int peer;
    };
    std::vector<Op> ops;
    int depth = 0;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    ~LoopbackComm() override {
        if (tmp) cudaFree(tmp);
    }
    void reserve(size_t bytes) override {
        if (bytes <= tmp_bytes) return;
        if (tmp) cuda_check(cudaFree(tmp), "free");
        cuda_check(cudaMalloc(&tmp, bytes), "loopback scratch");
        tmp_bytes = bytes;
    }
    void group_start() override { ++depth; }
    void group_end() override {
        if (--depth == 0) run();
    }
    void push(const Op& o) {
        ops.push_back(o);
        if (depth == 0) run();
    }
    void copy(void* dst, const void* src, size_t bytes) {
        if (dst != src && bytes)
            cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c0->stream), "loopback copy");
    }
    void run() {
        std::vector<Op> red, gat, bc, snd, rcv;
        for (auto& o : ops) {
            switch (o.kind) {
                case 0: red.push_back(o); break;
                case 1: gat.push_back(o); break;
                case 2: bc.push_back(o); break;
                case 3: snd.push_back(o); break;
                default: rcv.push_back(o); break;
            }
        }
        ops.clear();
        auto by_rank = [](const Op& a, const Op& b) { return a.l < b.l; };
        if (!red.empty()) {
            if (int(red.size()) != nranks) throw std::logic_error("loopback all_reduce: every rank must take part");
            std::sort(red.begin(), red.end(), by_rank);
            const size_t es = red[0].is_int ? sizeof(int) : sizeof(double);
            reserve(red[0].count * es);
            copy(tmp, red[0].dst, red[0].count * es);
            for (size_t r = 1; r < red.size(); ++r)
                combine(*c0, tmp, red[r].dst, int64_t(red[0].count), red[0].is_int, red[0].op == RedOp::max);
            for (auto& o : red) copy(o.dst, tmp, o.count * es);
        }
        if (!gat.empty()) {
            std::sort(gat.begin(), gat.end(), by_rank);
            for (auto& o : gat)
                for (auto& src : gat)
                    copy(static_cast<double*>(o.dst) + size_t(src.l) * o.count, src.src, o.count * sizeof(double));
        }
        if (!bc.empty()) {
            const void* root_src = nullptr;
            for (auto& o : bc)
                if (o.l == o.peer) root_src = o.src;
            for (auto& o : bc) copy(o.dst, root_src, o.count * sizeof(double));
        }
        for (auto& s : snd) {  // the first unmatched recv posted by the peer for this sender
            auto it = std::find_if(rcv.begin(), rcv.end(), [&](const Op& r) { return r.l == s.peer && r.peer == s.l; });
            if (it == rcv.end()) throw std::logic_error("loopback send without a matching recv");
            copy(it->dst, s.src, s.count * sizeof(double));
            rcv.erase(it);
        }
        if (!rcv.empty()) throw std::logic_error("loopback recv without a matching send");
    }
    void all_reduce(int l, void* buf, size_t count, bool is_int, RedOp op, cudaStream_t) override {
        push({0, l, buf, buf, count, is_int, op, 0});
    }
    void all_gather(int l, const double* send, double* recv, size_t count, cudaStream_t) override {
        push({1, l, send, recv, count, false, RedOp::sum, 0});
    }
    void broadcast(int l, const double* send, double* recv, size_t count, int root, cudaStream_t) override {
        push({2, l, send, recv, count, false, RedOp::sum, root});
    }
    void send(int l, const double* buf, size_t count, int peer, cudaStream_t) override {
        push({3, l, buf, nullptr, count, false, RedOp::sum, peer});
    }
    void recv(int l, double* buf, size_t count, int peer, cudaStream_t) override {
        push({4, l, nullptr, buf, count, false, RedOp::sum, peer});
    }
};

ShardGroup::~ShardGroup() {
    for (auto* c : ctx) {
        cudaSetDevice(c->device);
        cudaStreamSynchronize(c->stream);
    }
    comm.reset();
    owned.clear();
}

void shard_group_delete(ShardGroup* g) { delete g; }

static std::vector<int64_t> row_partition(int64_t n, int parts) {  // dist.py row_partition
    std::vector<int64_t> b(size_t(parts) + 1, 0);
    const int64_t base = n / parts, extra = n % parts;
    for (int p = 0; p < parts; ++p) b[size_t(p) + 1] = b[size_t(p)] + base + (p < extra ? 1 : 0);
    return b;
}

// ----------------------------------------------------------- the solver --
struct ShardSolver {
    si_context* sctx;
    ShardGroup& G;
    si_problem* prob;
    int method, sketch;
    int64_t n, q;
    uint64_t seed;
    int P = 1, NL = 1;
    std::vector<int64_t> cb;  // RBFGS: 2P chunk bounds; AdaRBFGS: P panel bounds
    int64_t mc = 0;           // rows of the largest chunk / panel
    bool gauss_ada = false;

    struct Rank {
        Context* c = nullptr;
        Problem* a = nullptr;
        int g = 0;
        int chunk[2] = {0, 0};
        double* X[2] = {nullptr, nullptr};
        double *U = nullptr, *Y = nullptr, *send = nullptr, *gath = nullptr, *Ginv = nullptr, *Ghat = nullptr,
               *fscr = nullptr;
        double *Lp = nullptr, *Sp = nullptr, *S = nullptr, *ASp = nullptr, *GZ = nullptr, *R = nullptr, *B = nullptr,
               *SRp = nullptr, *St = nullptr, *G2 = nullptr, *R2 = nullptr, *Tq = nullptr, *escr = nullptr,
               *d = nullptr;
        int64_t* idx = nullptr;
        int64_t* idx_ring = nullptr;
        int* status = nullptr;
        unsigned long long* counter = nullptr;
        double* scal = nullptr;
        double *xfull = nullptr, *stage = nullptr;
        std::vector<void*> allocs;
    };
    std::vector<Rank> R;
    double* s_pinned = nullptr;
    int64_t* idx_pinned = nullptr;
    int ring_cap = 0;
    int* st_host = nullptr;
    double* scal_host = nullptr;
    std::vector<cudaGraphExec_t> graphs;
    std::vector<cudaStream_t> gstreams;
    bool warmed = false;
    int64_t graph_launches = 0;
    int64_t redraws = 0;
    bool pdiag_valid = false;

    ShardSolver(si_context* ctx, si_problem* pr, int meth, int sk, int64_t q_, uint64_t seed_)
        : sctx(ctx), G(*ctx->group), prob(pr), method(meth), sketch(sk), n(pr->p->n), q(q_), seed(seed_) {
        P = G.nranks();
        NL = G.nlocal();
        gauss_ada = sk == SI_SKETCH_ADAPTIVE_GAUSS || sk == SI_SKETCH_ADAPTIVE_GAUSS_DEVICE;
        if (method == SI_METHOD_RBFGS) {
            if (n < 2 * P) throw ConfigError("multi-GPU run_inverter: n must be at least twice the rank count");
            cb = row_partition(n, 2 * P);
        } else {
            if (n < P) throw ConfigError("multi-GPU run_adarbfgs: n must be at least the rank count");
            cb = row_partition(n, P);
        }
        for (size_t i = 0; i + 1 < cb.size(); ++i) mc = std::max(mc, cb[i + 1] - cb[i]);
        R.resize(size_t(NL));
        for (int l = 0; l < NL; ++l) {
            R[size_t(l)].c = G.ctx[size_t(l)];
            R[size_t(l)].a = pr->replicas[size_t(l)];
            R[size_t(l)].g = G.rank(l);
        }
        alloc();
    }
    ~ShardSolver() {
        for (auto e : graphs) cudaGraphExecDestroy(e);
        for (auto& r : R) {
            cudaSetDevice(r.c->device);
            cudaStreamSynchronize(r.c->stream);
            for (void* p : r.allocs) cudaFree(p);
        }
        if (s_pinned) cudaFreeHost(s_pinned);
        if (idx_pinned) cudaFreeHost(idx_pinned);
        if (st_host) cudaFreeHost(st_host);
        if (scal_host) cudaFreeHost(scal_host);
    }

    template <class T>
    T* dalloc(Rank& r, size_t count) {
        dev(r.c);
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc (sharded)");
        r.allocs.push_back(p);
        return static_cast<T*>(p);
    }
    int owner(int c) const { return c < P ? c : 2 * P - 1 - c; }
    int64_t r0(int c) const { return cb[size_t(c)]; }
    int64_t rows(int c) const { return cb[size_t(c) + 1] - cb[size_t(c)]; }
    bool local(int g) const { return G.owns(g); }
    int lidx(int g) const { return g - G.rank(0); }

    void alloc() {
        const size_t nq = size_t(n) * size_t(q), qq = size_t(q) * size_t(q);
        for (auto& r : R) {
            r.status = dalloc<int>(r, 8);
            r.counter = dalloc<unsigned long long>(r, 1);
            r.scal = dalloc<double>(r, 8);
            cuda_check(cudaMemsetAsync(r.status, 0, 8 * sizeof(int), r.c->stream), "memset");
            cuda_check(cudaMemsetAsync(r.counter, 0, sizeof(unsigned long long), r.c->stream), "memset");
            if (method == SI_METHOD_RBFGS) {
                r.chunk[0] = r.g;
                r.chunk[1] = 2 * P - 1 - r.g;
                for (int j = 0; j < 2; ++j)
                    r.X[j] = dalloc<double>(r, size_t(rows(r.chunk[j])) * size_t(n - r0(r.chunk[j])));
                r.U = dalloc<double>(r, 4 * nq + 2 * qq);  // [S | R | Z | W' | H' | G]
                r.Y = dalloc<double>(r, nq);
                r.send = dalloc<double>(r, 2 * size_t(mc) * size_t(q));
                r.gath = P > 1 ? dalloc<double>(r, 2 * size_t(P) * size_t(mc) * size_t(q)) : r.send;
                r.Ginv = dalloc<double>(r, qq);
                r.Ghat = dalloc<double>(r, qq);
                r.fscr = dalloc<double>(r, 4 * qq + 2 * size_t(q) + 16);
            } else {
                const size_t m = size_t(rows(r.g));
                r.Lp = dalloc<double>(r, m * size_t(n));
                r.Sp = dalloc<double>(r, size_t(mc) * size_t(q));
                r.S = dalloc<double>(r, nq);
                r.gath = P > 1 ? dalloc<double>(r, size_t(P) * size_t(mc) * size_t(q)) : nullptr;
                r.ASp = dalloc<double>(r, m * size_t(q));
                r.GZ = dalloc<double>(r, qq + nq);
                r.R = dalloc<double>(r, qq);
                r.B = dalloc<double>(r, nq);
                r.SRp = dalloc<double>(r, m * size_t(q));
                r.escr = dalloc<double>(r, 8 * qq + 8 * size_t(q) + 32);
                r.idx = dalloc<int64_t>(r, size_t(q));
                r.d = dalloc<double>(r, size_t(n));
                if (gauss_ada) {
                    r.St = dalloc<double>(r, nq);
                    r.G2 = dalloc<double>(r, qq);
                    r.R2 = dalloc<double>(r, qq);
                    r.Tq = dalloc<double>(r, nq);
                }
            }
        }
        cuda_check(cudaMallocHost(&st_host, 8 * sizeof(int)), "pinned");
        cuda_check(cudaMallocHost(&scal_host, 8 * sizeof(double)), "pinned");
        if (method == SI_METHOD_RBFGS)
            G.comm->reserve((nq + 2 * qq) * sizeof(double));  // [W' | H'] is the largest reduction
        else
            G.comm->reserve((nq + qq) * sizeof(double));
        sync();
    }

    void sync() {
        for (auto& r : R) {
            dev(r.c);
            cuda_check(cudaStreamSynchronize(r.c->stream), "sync");
        }
    }

    double* pinned_sketch() {
        if (!s_pinned) cuda_check(cudaMallocHost(&s_pinned, size_t(n) * size_t(q) * sizeof(double)), "pinned");
        return s_pinned;
    }
    void ensure_ring(int cap) {
        if (cap <= ring_cap) return;
        if (idx_pinned) cudaFreeHost(idx_pinned);
        cuda_check(cudaMallocHost(&idx_pinned, size_t(cap) * size_t(q) * sizeof(int64_t)), "pinned");
        for (auto& r : R) r.idx_ring = dalloc<int64_t>(r, size_t(cap) * size_t(q));
        ring_cap = cap;
    }

    // ---- iterate set / get ------------------------------------------------
    void set_identity() {
        for (auto& r : R) {
            dev(r.c);
            if (method == SI_METHOD_RBFGS) {
                for (int j = 0; j < 2; ++j) set_identity_rows(*r.c, r.X[j], rows(r.chunk[j]), n - r0(r.chunk[j]), 0);
            } else {
                set_identity_rows(*r.c, r.Lp, rows(r.g), n, r0(r.g));
            }
        }
        pdiag_valid = false;
    }
    void set_from_host(const double* x) {  // X0 (its trapezoids) or L0 (its row panels), column-major n×n
        for (auto& r : R) {
            dev(r.c);
            if (method == SI_METHOD_RBFGS) {
                for (int j = 0; j < 2; ++j) {
                    const int c = r.chunk[j];
                    const int64_t a0 = r0(c), m = rows(c);
                    cuda_check(cudaMemcpy2DAsync(r.X[j], size_t(m) * 8, x + a0 + a0 * n, size_t(n) * 8, size_t(m) * 8,
                                                 size_t(n - a0), cudaMemcpyHostToDevice, r.c->stream),
                               "h2d x0");
                }
            } else {
                const int64_t a0 = r0(r.g), m = rows(r.g);
                cuda_check(cudaMemcpy2DAsync(r.Lp, size_t(m) * 8, x + a0, size_t(n) * 8, size_t(m) * 8, size_t(n),
                                             cudaMemcpyHostToDevice, r.c->stream),
                           "h2d l0");
            }
        }
        pdiag_valid = false;
        sync();
    }

    // ---- one RBFGS attempt (qq = this draw's sketch width) ------------------
    void enqueue_rbfgs(int64_t qq, bool device_sketch, bool batch) {
        const size_t nq = size_t(n) * size_t(qq);
        for (auto& r : R) {
            dev(r.c);
            Context& c = *r.c;
            const int* skip = r.status;
            double* S = r.U;
            if (device_sketch) philox_sketch(c, S, n, qq, n, seed, r.counter, 0, skip);
            for (int j = 0; j < 2; ++j) {
                const int ch = r.chunk[j];
                const int64_t a0 = r0(ch), m = rows(ch);
                double* dst = r.send + size_t(j) * size_t(mc) * size_t(qq);
                if (r.a->dense)
                    gemm(c, m, qq, n, r.a->a + a0 * n, n, true, S, n, true, dst, mc, 1.0, 0.0, skip);  // A[R_c,:]·S
                else
                    spmm_csr_rows(c, m, n, r.a->rowptr + a0, r.a->colind, r.a->val, S, n, qq, dst, mc);
            }
            // G = Σ_c Y[R_c]ᵀ·S[R_c] from the local rows (before the gather), all-reduced in the
            // same NCCL group as the Y all-gather, so its one-CTA K-FACTOR can run on the
            // high-priority side stream under the W' products (the single-GPU arrangement); W' and
            // H' share the second all-reduce.  Buffer tail after W': [H' | G] (q×q each).
            double* Gq = r.U + 4 * nq + size_t(qq) * size_t(qq);
            for (int j = 0; j < 2; ++j) {
                const int ch = r.chunk[j];
                gemm(c, qq, qq, rows(ch), r.send + size_t(j) * size_t(mc) * size_t(qq), mc, true, S + r0(ch), n, true,
                     Gq, qq, 1.0, j ? 1.0 : 0.0, skip);
            }
        }
        if (P > 1) {
            G.comm->group_start();
            for (int l = 0; l < NL; ++l) {
                auto& r = R[size_t(l)];
                dev(r.c);
                G.comm->all_gather(l, r.send, r.gath, 2 * size_t(mc) * size_t(qq), r.c->stream);
                G.comm->all_reduce(l, r.U + 4 * nq + size_t(qq) * size_t(qq), size_t(qq) * size_t(qq), false,
                                   RedOp::sum, r.c->stream);
            }
            G.comm->group_end();
        }
        for (auto& r : R) {
            dev(r.c);
            Context& c = *r.c;
            const int* skip = r.status;
            double* Wn = r.U + 3 * nq;
            double* Hq = Wn + nq;
            double* Gq = Hq + qq * qq;
            place_rows(c, r.gath, mc, 2 * P, true, n, qq, r.Y, n);
            c.fork(true);
            {
                SideHi side(c);
                rbfgs_gram_enqueue(c, Gq, qq, qq, r.Ginv, nullptr, r.fscr, r.status);  // G⁻¹ + PD test
            }
            cuda_check(cudaMemsetAsync(Wn, 0, nq * sizeof(double), c.stream), "memset W");
            for (int j = 0; j < 2; ++j) {
                const int ch = r.chunk[j];
                const int64_t a0 = r0(ch), m = rows(ch), a1 = a0 + m;
                gemm(c, m, qq, n - a0, r.X[j], m, false, r.Y + a0, n, true, Wn + a0, n, -1.0, 1.0, skip);
                if (a1 < n)
                    gemm(c, n - a1, qq, m, r.X[j] + m * m, m, true, r.Y + a0, n, true, Wn + a1, n, -1.0, 1.0, skip);
            }
            const int64_t f0 = r0(r.chunk[0]);  // H' = Y[f0:]ᵀ·W'loc[f0:] (W'loc is zero above f0)
            gemm(c, qq, qq, n - f0, r.Y + f0, n, true, Wn + f0, n, true, Hq, qq, 1.0, 0.0, skip);
        }
        if (P > 1) {
            G.comm->group_start();
            for (int l = 0; l < NL; ++l) {
                auto& r = R[size_t(l)];
                dev(r.c);
                G.comm->all_reduce(l, r.U + 3 * nq, nq + size_t(qq) * size_t(qq), false, RedOp::sum, r.c->stream);
            }
            G.comm->group_end();
        }
        for (auto& r : R) {
            dev(r.c);
            Context& c = *r.c;
            const int* skip = r.status;
            double* S = r.U;
            double* Rm = r.U + nq;
            double* Z = r.U + 2 * nq;
            double* Wn = r.U + 3 * nq;
            double* Hq = Wn + nq;
            double* Gq = Hq + qq * qq;
            c.join(true);
            ghat_split(c, Gq, Hq, qq, r.Ghat, r.status);  // Ĝ = G − H'
            const int64_t f0 = r0(r.chunk[0]);
            gemm(c, n - f0, qq, qq, S + f0, n, false, r.Ginv, qq, true, Z + f0, n, 1.0, 0.0, skip);  // Z = S·G⁻¹
            for (int j = 0; j < 2; ++j) {
                const int ch = r.chunk[j];
                const int64_t a0 = r0(ch), m = rows(ch), a1 = a0 + m;
                gemm(c, m, qq, qq, Z + a0, n, false, r.Ghat, qq, true, Rm + a0, n, 1.0, 1.0, skip, nullptr,
                     Wn + a0);  // R = Z·Ĝ + W'
                // X_c += [R Z][R_c]·[Z W'][r0:]ᵀ: the whole trapezoid in one K-SYMUPD launch (the
                // diagonal block by upper tiles mirrored, the rest plain)
                symupd_trapezoid(c, m, n - a0, 2 * qq, Rm + a0, n, Z + a0, n, r.X[j], m, skip, r.status + 1);
                (void)a1;
            }
            if (batch) advance_batch(c, r.counter, r.status, false);
        }
    }

    // ---- one AdaRBFGS attempt ----------------------------------------------
    // mode 0: coordinate indices (idx_src: per-rank device arrays); 1: host Gaussian S̃ in
    // s_pinned; 2: Philox S̃.  qq = this draw's width.
    void enqueue_ada(int mode, int64_t qq, int64_t ring_slot, bool batch) {
        for (auto& r : R) {
            dev(r.c);
            Context& c = *r.c;
            int* st = r.status;
            const int64_t m = rows(r.g);
            const int64_t* idx = ring_slot >= 0 ? r.idx_ring + ring_slot * q : r.idx;
            if (mode == 0) {
                gather_columns(c, r.Lp, m, m, idx, qq, r.Sp);  // S_p = L_p[:, C] (ld m)
            } else {
                if (mode == 2) philox_sketch(c, r.St, n, qq, n, seed, r.counter, 0, st);
                gemm(c, m, qq, n, r.Lp, m, false, r.St, n, true, r.Sp, m, 1.0, 0.0, st);  // S_p = L_p·S̃
            }
        }
        if (P > 1) {
            for (auto& r : R) {  // pad the panel to mc rows for the all-gather
                dev(r.c);
                const int64_t m = rows(r.g);
                if (m != mc)
                    cuda_check(cudaMemcpy2DAsync(r.S, size_t(mc) * 8, r.Sp, size_t(m) * 8, size_t(m) * 8, size_t(qq),
                                                 cudaMemcpyDeviceToDevice, r.c->stream),
                               "pad");
            }
            G.comm->group_start();
            for (int l = 0; l < NL; ++l) {
                auto& r = R[size_t(l)];
                dev(r.c);
                const int64_t m = rows(r.g);
                G.comm->all_gather(l, m == mc ? r.Sp : r.S, r.gath, size_t(mc) * size_t(qq), r.c->stream);
            }
            G.comm->group_end();
        }
        for (auto& r : R) {
            dev(r.c);
            Context& c = *r.c;
            int* st = r.status;
            const int64_t a0 = r0(r.g), m = rows(r.g);
            if (P > 1)
                place_rows(c, r.gath, mc, P, false, n, qq, r.S, n);
            else
                cuda_check(cudaMemcpyAsync(r.S, r.Sp, size_t(n) * size_t(qq) * 8, cudaMemcpyDeviceToDevice, c.stream),
                           "copy S");
            if (r.a->dense)
                gemm(c, m, qq, n, r.a->a + a0 * n, n, true, r.S, n, true, r.ASp, m, 1.0, 0.0, st);  // (AS)_p
            else
                spmm_csr_rows(c, m, n, r.a->rowptr + a0, r.a->colind, r.a->val, r.S, n, qq, r.ASp, m);
            gemm(c, qq, qq, m, r.Sp, m, true, r.ASp, m, true, r.GZ, qq, 1.0, 0.0, st);           // S_pᵀ(AS)_p
            gemm(c, qq, n, m, r.ASp, m, true, r.Lp, m, true, r.GZ + qq * qq, qq, 1.0, 0.0, st);  // (AS)_pᵀ L_p
        }
        if (P > 1) {
            G.comm->group_start();
            for (int l = 0; l < NL; ++l) {
                auto& r = R[size_t(l)];
                dev(r.c);
                G.comm->all_reduce(l, r.GZ, size_t(qq) * size_t(qq) + size_t(qq) * size_t(n), false, RedOp::sum,
                                   r.c->stream);
            }
            G.comm->group_end();
        }
        for (auto& r : R) {
            dev(r.c);
            Context& c = *r.c;
            int* st = r.status;
            const int64_t m = rows(r.g);
            const int64_t* idx = ring_slot >= 0 ? r.idx_ring + ring_slot * q : r.idx;
            ada_core_enqueue(c, r.GZ, qq, r.GZ + qq * qq, n, mode == 0 ? idx : nullptr, mode == 0 ? nullptr : r.St,
                             r.G2, r.R2, r.Tq, r.R, r.B, r.escr, st);                        // R, B = T − R·Z
            gemm(c, m, qq, qq, r.Sp, m, false, r.R, qq, true, r.SRp, m, 1.0, 0.0, st);       // (S·R)_p
            gemm(c, m, n, qq, r.SRp, m, false, r.B, qq, true, r.Lp, m, 1.0, 1.0, st, st + 1);  // L_p += (S·R)_p·B
            if (pdiag_valid) pdiag_update(c, r.B, qq, n, mode == 0 ? nullptr : r.Tq, idx, st, r.d);
            if (batch) advance_batch(c, mode == 2 ? r.counter : nullptr, st, true);
        }
    }

    // ---- status (max over ranks) -------------------------------------------
    void reset_status() {
        for (auto& r : R) {
            dev(r.c);
            cuda_check(cudaMemsetAsync(r.status, 0, 8 * sizeof(int), r.c->stream), "reset");
        }
    }
    void read_status(int* st) {
        if (P > 1) {
            G.comm->group_start();
            for (int l = 0; l < NL; ++l) {
                auto& r = R[size_t(l)];
                dev(r.c);
                G.comm->all_reduce(l, r.status, 8, true, RedOp::max, r.c->stream);
            }
            G.comm->group_end();
        }
        dev(R[0].c);
        cuda_check(cudaMemcpyAsync(st_host, R[0].status, 8 * sizeof(int), cudaMemcpyDeviceToHost, R[0].c->stream),
                   "status d2h");
        sync();
        std::memcpy(st, st_host, 8 * sizeof(int));
    }
    double reduce_scalar() {  // Σ over ranks of scal[0] + scal[1]
        for (auto& r : R) {
            dev(r.c);
            combine(*r.c, r.scal, r.scal + 1, 1, false, false);
        }
        if (P > 1) {
            G.comm->group_start();
            for (int l = 0; l < NL; ++l) {
                auto& r = R[size_t(l)];
                dev(r.c);
                G.comm->all_reduce(l, r.scal, 1, false, RedOp::sum, r.c->stream);
            }
            G.comm->group_end();
        }
        dev(R[0].c);
        cuda_check(cudaMemcpyAsync(scal_host, R[0].scal, sizeof(double), cudaMemcpyDeviceToHost, R[0].c->stream),
                   "d2h");
        sync();
        return scal_host[0];
    }

    // ---- graphs: one attempt captured per stream (collectives included) ------
    template <class F>
    void replay(F&& enqueue_one) {
        const bool graphs_ok = !R[0].c->profiling && std::getenv("SI_NO_GRAPH") == nullptr;
        if (!graphs_ok || !warmed) {  // first attempt eagerly: sizes workspaces, sets kernel attributes
            enqueue_one();
            warmed = true;
            return;
        }
        if (graphs.empty()) {
            gstreams.clear();
            for (auto& r : R)
                if (std::find(gstreams.begin(), gstreams.end(), r.c->stream) == gstreams.end())
                    gstreams.push_back(r.c->stream);
            const int64_t l0 = R[0].c->launches;
            for (auto st : gstreams) cuda_check(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed), "capture");
            enqueue_one();
            for (size_t i = 0; i < gstreams.size(); ++i) {
                cudaGraph_t gr = nullptr;
                for (auto& r : R)
                    if (r.c->stream == gstreams[i]) dev(r.c);
                cuda_check(cudaStreamEndCapture(gstreams[i], &gr), "end capture");
                cudaGraphExec_t e = nullptr;
                cuda_check(cudaGraphInstantiate(&e, gr, 0), "instantiate");
                cudaGraphDestroy(gr);
                graphs.push_back(e);
            }
            graph_launches = R[0].c->launches - l0;
            R[0].c->launches = l0;
        }
        for (size_t i = 0; i < gstreams.size(); ++i) {
            for (auto& r : R)
                if (r.c->stream == gstreams[i]) dev(r.c);
            cuda_check(cudaGraphLaunch(graphs[i], gstreams[i]), "graph launch");
        }
        R[0].c->launches += graph_launches;
    }

    // ---- checkpoints ------------------------------------------------------------
    void ensure_full_buffers() {
        for (auto& r : R) {
            if (!r.xfull) r.xfull = dalloc<double>(r, size_t(mc) * size_t(n));
            if (!r.stage) r.stage = dalloc<double>(r, size_t(mc) * size_t(n));
        }
    }
    // RBFGS: X[R_c, :] (m×n, ld m) in the owner's xfull, for chunks c = 0..2P−1 in turn; the
    // blocks left of the trapezoid come from the earlier chunks' owners (one send each)
    template <class F>
    void for_each_full_rows(F&& on_rows) {
        ensure_full_buffers();
        for (int c = 0; c < 2 * P; ++c) {
            const int oc = owner(c);
            const int64_t a0 = r0(c), m = rows(c);
            G.comm->group_start();
            for (int l = 0; l < NL; ++l) {
                auto& r = R[size_t(l)];
                dev(r.c);
                for (int cp = 0; cp < c; ++cp) {
                    const int op = owner(cp);
                    if (op == oc) continue;
                    if (r.g == oc)
                        G.comm->recv(l, r.stage + r0(cp) * m, size_t(rows(cp)) * size_t(m), op, r.c->stream);
                    if (r.g == op) {
                        const int j = r.chunk[0] == cp ? 0 : 1;
                        G.comm->send(l, r.X[j] + (a0 - r0(cp)) * rows(cp), size_t(rows(cp)) * size_t(m), oc,
                                     r.c->stream);
                    }
                }
            }
            G.comm->group_end();
            if (!local(oc)) {
                on_rows(-1, c);
                continue;
            }
            auto& r = R[size_t(lidx(oc))];
            dev(r.c);
            for (int cp = 0; cp < c; ++cp) {
                const int64_t mp = rows(cp);
                const double* src;
                if (owner(cp) == oc) {
                    const int j = r.chunk[0] == cp ? 0 : 1;
                    src = r.X[j] + (a0 - r0(cp)) * mp;
                } else {
                    src = r.stage + r0(cp) * m;
                }
                transpose_block(*r.c, src, mp, m, mp, r.xfull + r0(cp) * m, m);  // X[R_c, R_cp] = X[R_cp, R_c]ᵀ
            }
            const int j = r.chunk[0] == c ? 0 : 1;
            cuda_check(cudaMemcpyAsync(r.xfull + a0 * m, r.X[j], size_t(m) * size_t(n - a0) * 8,
                                       cudaMemcpyDeviceToDevice, r.c->stream),
                       "copy trapezoid");
            on_rows(lidx(oc), c);
        }
    }
    // AdaRBFGS: X[R_p, :] = L_p·Lᵀ into xfull, streaming the panels L_s by broadcast
    void ada_form_x_rows() {
        ensure_full_buffers();
        for (int s = 0; s < P; ++s) {
            const int64_t ms = rows(s);
            if (P > 1) {
                G.comm->group_start();
                for (int l = 0; l < NL; ++l) {
                    auto& r = R[size_t(l)];
                    dev(r.c);
                    G.comm->broadcast(l, r.g == s ? r.Lp : nullptr, r.g == s ? r.Lp : r.stage, size_t(ms) * size_t(n), s,
                                      r.c->stream);
                }
                G.comm->group_end();
            }
            for (auto& r : R) {
                dev(r.c);
                const int64_t m = rows(r.g);
                const double* Ls = r.g == s ? r.Lp : r.stage;
                gemm(*r.c, m, ms, n, r.Lp, m, false, Ls, ms, false, r.xfull + r0(s) * m, m, 1.0, 0.0);  // L_p·L_sᵀ
            }
        }
    }
    void rows_residual(Rank& r, int slot, int64_t m, int64_t a0, const double* Xrows) {
        if (r.a->dense)
            residual_rows_sq_enqueue(*r.c, *r.a, m, a0, Xrows, m, r.scal + slot);
        else
            csr_residual_rows_sq(*r.c, *r.a, m, a0, Xrows, r.scal + slot);
    }
    double residual() {  // ‖I − A·X‖_F
        for (auto& r : R) {
            dev(r.c);
            cuda_check(cudaMemsetAsync(r.scal, 0, 8 * sizeof(double), r.c->stream), "memset");
        }
        if (method == SI_METHOD_RBFGS) {
            for_each_full_rows([&](int l, int c) {
                if (l < 0) return;
                auto& r = R[size_t(l)];
                rows_residual(r, r.chunk[0] == c ? 0 : 1, rows(c), r0(c), r.xfull);
            });
        } else {
            ada_form_x_rows();
            for (auto& r : R) {
                dev(r.c);
                rows_residual(r, 0, rows(r.g), r0(r.g), r.xfull);
            }
        }
        return std::sqrt(std::max(reduce_scalar(), 0.0));
    }

    // rows [a0, a0+m) of the n×n column-major host matrix from local rank l's m×n panel (ld m)
    void rows_to_host(int l, int64_t a0, int64_t m, const double* panel, double* host) {
        auto& r = R[size_t(l)];
        dev(r.c);
        if (host)
            cuda_check(cudaMemcpy2DAsync(host + a0, size_t(n) * 8, panel, size_t(m) * 8, size_t(m) * 8, size_t(n),
                                         cudaMemcpyDeviceToHost, r.c->stream),
                       "d2h rows");
    }
    // download for one-process-per-GPU groups: every panel is sent to global rank 0
    template <class PanelFn>
    void gather_rows_to_rank0(int nparts, PanelFn&& panel_of, double* host) {
        // panel_of(part) -> (owner global rank, a0, m, device pointer on the owner or nullptr)
        for (int part = 0; part < nparts; ++part) {
            auto [og, a0, m, ptr] = panel_of(part);
            G.comm->group_start();
            for (int l = 0; l < NL; ++l) {
                auto& r = R[size_t(l)];
                dev(r.c);
                if (og != 0 && r.g == og) G.comm->send(l, ptr, size_t(m) * size_t(n), 0, r.c->stream);
                if (og != 0 && r.g == 0) G.comm->recv(l, r.stage, size_t(m) * size_t(n), og, r.c->stream);
            }
            G.comm->group_end();
            if (local(0) && host) {
                auto& r = R[size_t(lidx(0))];
                dev(r.c);
                const double* src = og == 0 ? ptr : r.stage;
                cuda_check(cudaMemcpy2DAsync(host + a0, size_t(n) * 8, src, size_t(m) * 8, size_t(m) * 8, size_t(n),
                                             cudaMemcpyDeviceToHost, r.c->stream),
                           "d2h rows");
                cuda_check(cudaStreamSynchronize(r.c->stream), "sync");
            }
        }
    }
    void download_x(double* host) {  // RBFGS X, or AdaRBFGS X = L·Lᵀ
        const bool multiproc = G.nranks() > G.nlocal();
        if (method == SI_METHOD_RBFGS) {
            if (!multiproc) {
                for_each_full_rows([&](int l, int c) {
                    if (l >= 0) rows_to_host(l, r0(c), rows(c), R[size_t(l)].xfull, host);
                    sync();  // xfull is reused by the next chunk
                });
                return;
            }
            // one process per GPU: chunk by chunk, the owner's full rows go to rank 0
            ensure_full_buffers();
            for (int c = 0; c < 2 * P; ++c) {
                double* full = nullptr;
                for_each_full_rows_one(c, &full);
                gather_rows_to_rank0(
                    1, [&](int) { return std::tuple<int, int64_t, int64_t, const double*>(owner(c), r0(c), rows(c), full); },
                    host);
            }
            return;
        }
        ada_form_x_rows();
        download_panels([&](Rank& r) { return r.xfull; }, host);
    }
    void download_l(double* host) {
        download_panels([&](Rank& r) { return r.Lp; }, host);
    }
    template <class Sel>
    void download_panels(Sel&& sel, double* host) {
        const bool multiproc = G.nranks() > G.nlocal();
        if (!multiproc) {
            for (int l = 0; l < NL; ++l) rows_to_host(l, r0(R[size_t(l)].g), rows(R[size_t(l)].g), sel(R[size_t(l)]), host);
            sync();
            return;
        }
        ensure_full_buffers();
        gather_rows_to_rank0(
            P,
            [&](int part) {
                const double* ptr = local(part) ? sel(R[size_t(lidx(part))]) : nullptr;
                return std::tuple<int, int64_t, int64_t, const double*>(part, r0(part), rows(part), ptr);
            },
            host);
    }
    // the full rows of one chunk c (multi-process download): runs the exchange for c only
    void for_each_full_rows_one(int c_target, double** full_out) {
        ensure_full_buffers();
        const int oc = owner(c_target);
        const int64_t a0 = r0(c_target), m = rows(c_target);
        G.comm->group_start();
        for (int l = 0; l < NL; ++l) {
            auto& r = R[size_t(l)];
            dev(r.c);
            for (int cp = 0; cp < c_target; ++cp) {
                const int op = owner(cp);
                if (op == oc) continue;
                if (r.g == oc) G.comm->recv(l, r.stage + r0(cp) * m, size_t(rows(cp)) * size_t(m), op, r.c->stream);
                if (r.g == op) {
                    const int j = r.chunk[0] == cp ? 0 : 1;
                    G.comm->send(l, r.X[j] + (a0 - r0(cp)) * rows(cp), size_t(rows(cp)) * size_t(m), oc, r.c->stream);
                }
            }
        }
        G.comm->group_end();
        *full_out = nullptr;
        if (!local(oc)) return;
        auto& r = R[size_t(lidx(oc))];
        dev(r.c);
        for (int cp = 0; cp < c_target; ++cp) {
            const int64_t mp = rows(cp);
            const double* src = owner(cp) == oc ? r.X[r.chunk[0] == cp ? 0 : 1] + (a0 - r0(cp)) * mp : r.stage + r0(cp) * m;
            transpose_block(*r.c, src, mp, m, mp, r.xfull + r0(cp) * m, m);
        }
        const int j = r.chunk[0] == c_target ? 0 : 1;
        cuda_check(cudaMemcpyAsync(r.xfull + a0 * m, r.X[j], size_t(m) * size_t(n - a0) * 8, cudaMemcpyDeviceToDevice,
                                   r.c->stream),
                   "copy trapezoid");
        *full_out = r.xfull;
    }

    // ---- Eq. 8.2 diagonal ------------------------------------------------------------
    void pdiag_init() {  // diag(LᵀAL): diag(A) at L = I; the exact Σ_p diag(L_pᵀ(A·L)_p) otherwise
        if (!identity_start) {
            ensure_full_buffers();
            for (auto& r : R)
                if (!r.a->dense) throw ConfigError("multi-GPU run_adarbfgs: adaptive_cols with l0 needs a dense A");
            for (int s = 0; s < P; ++s) {  // (A·L)_p = Σ_s A[R_p, R_s]·L_s
                const int64_t ms = rows(s);
                if (P > 1) {
                    G.comm->group_start();
                    for (int l = 0; l < NL; ++l) {
                        auto& r = R[size_t(l)];
                        dev(r.c);
                        G.comm->broadcast(l, r.g == s ? r.Lp : nullptr, r.g == s ? r.Lp : r.stage, size_t(ms) * size_t(n),
                                          s, r.c->stream);
                    }
                    G.comm->group_end();
                }
                for (auto& r : R) {
                    dev(r.c);
                    const int64_t m = rows(r.g);
                    const double* Ls = r.g == s ? r.Lp : r.stage;
                    gemm(*r.c, m, n, ms, r.a->a + r0(r.g) + r0(s) * n, n, false, Ls, ms, true, r.xfull, m, 1.0,
                         s ? 1.0 : 0.0);
                }
            }
            for (auto& r : R) {
                dev(r.c);
                panel_column_dots(*r.c, r.xfull, r.Lp, rows(r.g), n, r.d);
            }
            if (P > 1) {
                G.comm->group_start();
                for (int l = 0; l < NL; ++l) {
                    auto& r = R[size_t(l)];
                    dev(r.c);
                    G.comm->all_reduce(l, r.d, size_t(n), false, RedOp::sum, r.c->stream);
                }
                G.comm->group_end();
            }
        } else {
            for (auto& r : R) {
                dev(r.c);
                problem_diagonal(*r.c, *r.a, r.d);
            }
        }
        pdiag_valid = true;
    }
    bool identity_start = true;
};

void shard_solver_delete(ShardSolver* s) { delete s; }

// --------------------------------------------------------- drivers ------
static void validate_shared(si_problem* prob) {  // validate_spd on local rank 0's replica
    validate_spd(prob);
}

static double identity_residual(ShardSolver& sv) {  // ‖I − A‖_F: the base for X0 = I
    auto& r = sv.R[0];
    dev(r.c);
    identity_residual_sq_enqueue(*r.c, *r.a, r.scal);
    cuda_check(cudaMemcpyAsync(sv.scal_host, r.scal, sizeof(double), cudaMemcpyDeviceToHost, r.c->stream), "d2h");
    cuda_check(cudaStreamSynchronize(r.c->stream), "sync");
    return std::sqrt(sv.scal_host[0]);
}

void shard_run_inverter(si_context* ctx, si_problem* prob, const si_inverter_config* cfg, double* x_out,
                        si_history_point* history, int64_t history_cap, si_run_result* result) {
    const int64_t n = prob->p->n, q = cfg->q;
    std::memset(result, 0, sizeof(*result));
    require(cfg->update == SI_UPDATE_BFGS, "multi-GPU run_inverter: the sharded iteration is bfgs");
    require(q >= 1 && q <= n, "SketchRule: q must satisfy 1 <= q <= n");
    const int sk = cfg->sketch;
    if (sk == SI_SKETCH_ADAPTIVE_COLS || sk == SI_SKETCH_ADAPTIVE_GAUSS || sk == SI_SKETCH_ADAPTIVE_COLS_UNIFORM ||
        sk == SI_SKETCH_ADAPTIVE_GAUSS_DEVICE)
        throw ConfigError("run_inverter: adaptive sketch rules belong to the adarbfgs driver");
    require(sk == SI_SKETCH_GAUSSIAN || sk == SI_SKETCH_GAUSSIAN_DEVICE || sk == SI_SKETCH_COORDINATE_BLOCK,
            "run_inverter: unknown sketch rule");
    require(cfg->tol >= 0.0, "run_inverter: tol must be >= 0");
    require(cfg->max_iters >= 1, "run_inverter: max_iters must be >= 1");
    require(cfg->max_redraws >= 0, "run_inverter: max_redraws must be >= 0");
    require(cfg->residual_every_k >= 1, "run_inverter: residual_every_k must be >= 1");
    validate_shared(prob);  // simi.cpp:185-213 (validate_update for bfgs: spd)
    if (cfg->x0_host) {
        double nrm = 0.0;
        const double asym = host_frobenius_asym(cfg->x0_host, n, &nrm);
        if (asym > 1e-10 * std::max(1.0, nrm)) throw ConfigError("run_inverter: this method requires a symmetric x0");
    }
    ShardSolver sv(ctx, prob, SI_METHOD_RBFGS, sk, q, cfg->seed);
    if (cfg->x0_host)
        sv.set_from_host(cfg->x0_host);
    else
        sv.set_identity();
    HistoryWriter hist{history, history_cap, 0, cfg};
    double flops = 0.0, seconds = 0.0;
    int64_t k = 0;
    auto finish = [&](int term, const std::string& msg) {
        result->termination = term;
        result->k = k;
        result->flops = flops;
        result->seconds = seconds;
        result->history_count = hist.count;
        result->max_symmetry_drift = 0.0;  // the trapezoids hold each entry once: X is exactly symmetric
        result->redraws = sv.redraws;
        set_message(result, msg);
        if (x_out) sv.download_x(x_out);
        sv.sync();
    };
    const double base = cfg->x0_host ? sv.residual() : identity_residual(sv);  // simi.cpp:242-246
    if (base == 0.0) {
        hist.record(0, 0.0, 0.0, 0.0);
        finish(SI_TOL_REACHED, "");
        return;
    }
    hist.record(0, 1.0, 0.0, 0.0);
    std::vector<std::vector<si::Index>> blocks;
    std::vector<double> p;
    if (sk == SI_SKETCH_COORDINATE_BLOCK) {
        if (cfg->probabilities == SI_PROB_CONVENIENT)
            throw ConfigError("multi-GPU run_inverter: coordinate_block supports uniform probabilities");
        blocks = si::contiguous_partition(n, q);
        p.assign(blocks.size(), 1.0 / double(blocks.size()));
    }
    si::RngStream rng(cfg->seed);  // simi.cpp:275
    const bool device_sketch = sk == SI_SKETCH_GAUSSIAN_DEVICE;
    auto& r0c = *sv.R[0].c;
    dev(&r0c);
    cudaEvent_t ta, tb;
    cuda_check(cudaEventCreate(&ta), "event");
    cuda_check(cudaEventCreate(&tb), "event");
    struct Ev {
        cudaEvent_t a, b;
        ~Ev() {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    } evs{ta, tb};
    auto elapsed = [&]() {
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, ta, tb), "elapsed");
        return double(ms) * 1e-3;
    };
    auto checkpoint = [&]() -> bool {  // simi.cpp:361-375
        const double rel = sv.residual() / base;
        hist.record(k, rel, flops, seconds);
        if (rel <= cfg->tol) {
            finish(SI_TOL_REACHED, "");
            return true;
        }
        if (cfg->time_budget_seconds > 0.0 && seconds > cfg->time_budget_seconds) {
            finish(SI_MAX_ITERS, "time budget exhausted");
            return true;
        }
        return false;
    };
    int st[8];
    if (device_sketch && std::getenv("SI_RUN_EAGER") == nullptr) {
        // the iterations between two checkpoints back to back as graph replays; the device keeps
        // the accounting (advance_batch_kernel), as in the single-GPU driver
        int consecutive = 0;
        const int64_t every = cfg->residual_every_k, kmax = cfg->max_iters;
        while (k < kmax) {
            const int64_t kc = k == 0 ? 1 : std::min(((k + every) / every) * every, kmax);
            sv.reset_status();
            dev(&r0c);
            cuda_check(cudaEventRecord(ta, r0c.stream), "event");
            for (int64_t b = k; b < kc; ++b) sv.replay([&] { sv.enqueue_rbfgs(q, true, true); });
            dev(&r0c);
            cuda_check(cudaEventRecord(tb, r0c.stream), "event");
            sv.read_status(st);
            const int64_t accepted = st[3];
            k += accepted;
            sv.redraws += st[2];
            if (cfg->track_wall_time) seconds += elapsed();
            if (cfg->track_flops) flops += double(accepted) * flops_bfgs(double(n), double(q));
            if (st[1]) {
                finish(SI_TERMINATION_ERROR, "diverged: non-finite entries at iteration " + std::to_string(k));
                return;
            }
            if (st[4]) {
                consecutive = (accepted > 0 ? 0 : consecutive) + 1;
                if (consecutive > cfg->max_redraws) {
                    k += 1;
                    finish(SI_TERMINATION_ERROR, "sketch rejection limit exceeded for " + describe(sk, q) +
                                                     " at iteration " + std::to_string(k));
                    return;
                }
                continue;
            }
            consecutive = 0;
            if (checkpoint()) return;
        }
        k = kmax;
        finish(SI_MAX_ITERS, "");
        return;
    }
    for (k = 1; k <= cfg->max_iters; ++k) {
        bool stepped = false;
        for (int failures = 0; !stepped; ++failures) {
            if (failures > cfg->max_redraws) {
                finish(SI_TERMINATION_ERROR, "sketch rejection limit exceeded for " + describe(sk, q) +
                                                 " at iteration " + std::to_string(k));
                return;
            }
            int64_t qq = q;
            if (sk == SI_SKETCH_GAUSSIAN) {
                rng.gaussian_fill(sv.pinned_sketch(), n, q, n);  // rng.hpp:42-49
            } else if (sk == SI_SKETCH_COORDINATE_BLOCK) {
                const si::Index i = rng.categorical(p.data(), si::Index(p.size()));
                ctx->log_draw(i);
                const auto& blk = blocks[size_t(i)];
                qq = int64_t(blk.size());
                double* sp = sv.pinned_sketch();
                std::fill(sp, sp + n * qq, 0.0);
                for (size_t j = 0; j < blk.size(); ++j) sp[blk[j] + int64_t(j) * n] = 1.0;
            }
            if (!device_sketch)
                for (auto& r : sv.R) {
                    dev(r.c);
                    cuda_check(cudaMemcpyAsync(r.U, sv.s_pinned, size_t(n) * size_t(qq) * 8, cudaMemcpyHostToDevice,
                                               r.c->stream),
                               "h2d sketch");
                }
            sv.reset_status();
            dev(&r0c);
            cuda_check(cudaEventRecord(ta, r0c.stream), "event");  // after the draw (simi.cpp:298)
            sv.enqueue_rbfgs(qq, device_sketch, device_sketch);
            dev(&r0c);
            cuda_check(cudaEventRecord(tb, r0c.stream), "event");
            sv.read_status(st);
            if (st[0] || st[2]) {  // GramRankDeficientError -> redraw (simi.cpp:331-333)
                sv.redraws++;
                continue;
            }
            if (cfg->track_wall_time) seconds += elapsed();
            if (cfg->track_flops) flops += flops_bfgs(double(n), double(qq));
            stepped = true;
        }
        if (st[1]) {
            finish(SI_TERMINATION_ERROR, "diverged: non-finite entries at iteration " + std::to_string(k));
            return;
        }
        if (k == 1 || k == cfg->max_iters || k % cfg->residual_every_k == 0)
            if (checkpoint()) return;
    }
    k = cfg->max_iters;
    finish(SI_MAX_ITERS, "");
}

void shard_run_adarbfgs(si_context* ctx, si_problem* prob, const si_inverter_config* cfg, double* l_out,
                        double* x_out, si_history_point* history, int64_t history_cap, si_run_result* result) {
    const int64_t n = prob->p->n, q = cfg->q;
    std::memset(result, 0, sizeof(*result));
    require(q >= 1 && q <= n, "SketchRule: q must satisfy 1 <= q <= n");
    const int sk = cfg->sketch;
    if (!(sk == SI_SKETCH_ADAPTIVE_COLS || sk == SI_SKETCH_ADAPTIVE_GAUSS || sk == SI_SKETCH_ADAPTIVE_COLS_UNIFORM ||
          sk == SI_SKETCH_ADAPTIVE_GAUSS_DEVICE))
        throw ConfigError("run_adarbfgs: rule must be adaptive");
    require(cfg->tol >= 0.0, "run_adarbfgs: tol must be >= 0");
    require(cfg->max_iters >= 1, "run_adarbfgs: max_iters must be >= 1");
    if (prob->p->symmetry != SI_SPD)
        throw std::invalid_argument("ProblemMatrix: operation requires an spd-flagged matrix");
    const bool cols = sk == SI_SKETCH_ADAPTIVE_COLS;
    validate_shared(prob);  // adarbfgs.cpp:97
    ShardSolver sv(ctx, prob, SI_METHOD_ADARBFGS, sk, q, cfg->seed);
    if (cfg->x0_host) {
        sv.set_from_host(cfg->x0_host);
        sv.identity_start = false;
    } else {
        sv.set_identity();
    }
    if (cols) sv.pdiag_init();
    HistoryWriter hist{history, history_cap, 0, cfg};
    double flops = 0.0, seconds = 0.0;
    int64_t k = 0;
    auto finish = [&](int term, const std::string& msg) {
        result->termination = term;
        result->k = k;
        result->flops = flops;
        result->seconds = seconds;
        result->history_count = hist.count;
        result->redraws = sv.redraws;
        set_message(result, msg);
        if (l_out) sv.download_l(l_out);
        if (x_out) sv.download_x(x_out);  // state.x = L Lᵀ (adarbfgs.cpp:89,122)
        sv.sync();
    };
    const double base = cfg->x0_host ? sv.residual() : identity_residual(sv);  // adarbfgs.cpp:112-115,126
    if (base == 0.0) {
        hist.record(0, 0.0, 0.0, 0.0);
        finish(SI_TOL_REACHED, "");
        return;
    }
    hist.record(0, 1.0, 0.0, 0.0);
    const auto blocks = cols ? si::contiguous_partition(n, q) : std::vector<std::vector<si::Index>>{};
    si::RngStream rng(cfg->seed);
    std::vector<double> p, dhost;
    auto checkpoint = [&]() -> bool {  // adarbfgs.cpp:179-194
        const double rel = sv.residual() / base;
        hist.record(k, rel, flops, seconds);
        if (rel <= cfg->tol) {
            finish(SI_TOL_REACHED, "");
            return true;
        }
        if (cfg->time_budget_seconds > 0.0 && seconds > cfg->time_budget_seconds) {
            finish(SI_MAX_ITERS, "time budget exhausted");
            return true;
        }
        return false;
    };
    int st[8];
    auto upload_idx = [&](const int64_t* idx, int64_t count, bool ring) {
        for (auto& r : sv.R) {
            dev(r.c);
            cuda_check(cudaMemcpyAsync(ring ? r.idx_ring : r.idx, idx, size_t(count) * sizeof(int64_t),
                                       cudaMemcpyHostToDevice, r.c->stream),
                       "h2d idx");
        }
    };
    if ((sk == SI_SKETCH_ADAPTIVE_COLS_UNIFORM || sk == SI_SKETCH_ADAPTIVE_GAUSS_DEVICE) &&
        std::getenv("SI_RUN_EAGER") == nullptr) {
        // as the single-GPU driver: up to 64 attempts between checkpoints drawn on the host,
        // enqueued back to back, the batch stopped on the device at a rejected attempt and the
        // host stream rewound to just after it
        const int mode = sk == SI_SKETCH_ADAPTIVE_COLS_UNIFORM ? 0 : 2;
        constexpr int64_t CAP = 64;
        if (mode == 0) sv.ensure_ring(int(CAP));
        std::vector<si::RngStream> snaps;
        int consecutive = 0;
        const int64_t every = cfg->residual_every_k, kmax = cfg->max_iters;
        while (k < kmax) {
            const int64_t kc = k == 0 ? 1 : std::min(((k + every) / every) * every, kmax);
            const int64_t nb = std::min(kc - k, CAP);
            const auto t0 = std::chrono::steady_clock::now();
            if (mode == 0) {
                snaps.clear();
                for (int64_t b = 0; b < nb; ++b) {
                    snaps.push_back(rng);
                    const auto idx = si::uniform_subset(rng, n, q);
                    for (int64_t j = 0; j < q; ++j) sv.idx_pinned[b * q + j] = idx[size_t(j)];
                }
                snaps.push_back(rng);
                upload_idx(sv.idx_pinned, nb * q, true);
            }
            sv.reset_status();
            for (int64_t b = 0; b < nb; ++b) sv.enqueue_ada(mode, q, mode == 0 ? b : -1, true);
            sv.read_status(st);
            const auto t1 = std::chrono::steady_clock::now();
            const int64_t accepted = st[5];
            if (mode == 0) {
                const int64_t ran = st[4] ? accepted + 1 : nb;
                for (int64_t b = 0; b < ran * q; ++b) ctx->log_draw(sv.idx_pinned[b]);
            }
            k += accepted;
            sv.redraws += st[2];
            if (cfg->track_wall_time) seconds += std::chrono::duration<double>(t1 - t0).count();
            if (cfg->track_flops) flops += double(accepted) * flops_adarbfgs(double(n), double(q));
            if (st[1]) {
                finish(SI_TERMINATION_ERROR, "diverged: non-finite factor at iteration " + std::to_string(k));
                return;
            }
            if (st[4]) {
                if (mode == 0) rng = snaps[size_t(accepted) + 1];
                consecutive = (accepted > 0 ? 0 : consecutive) + 1;
                if (consecutive > cfg->max_redraws) {
                    k += 1;
                    finish(SI_TERMINATION_ERROR, "sketch rejection limit exceeded for " + describe(sk, q) +
                                                     " at iteration " + std::to_string(k));
                    return;
                }
                continue;
            }
            consecutive = 0;
            if (k == kc && checkpoint()) return;
        }
        k = kmax;
        finish(SI_MAX_ITERS, "");
        return;
    }
    int64_t* idx_host = nullptr;
    cuda_check(cudaMallocHost(&idx_host, size_t(q) * sizeof(int64_t)), "pinned");
    struct Pin {
        int64_t* p;
        ~Pin() { cudaFreeHost(p); }
    } pin{idx_host};
    for (k = 1; k <= cfg->max_iters; ++k) {
        bool stepped = false;
        const auto t0 = std::chrono::steady_clock::now();  // probabilities + draws inside (:143)
        if (cols) {  // the carried diagonal of the replicated B, read from local rank 0
            auto& r = sv.R[0];
            dev(r.c);
            dhost.resize(size_t(n));
            cuda_check(cudaMemcpyAsync(dhost.data(), r.d, size_t(n) * 8, cudaMemcpyDeviceToHost, r.c->stream), "d2h");
            cuda_check(cudaStreamSynchronize(r.c->stream), "sync");
            block_probabilities(dhost.data(), blocks, p);
        }
        for (int attempt = 0; attempt <= cfg->max_redraws && !stepped; ++attempt) {
            int mode = 0;
            int64_t qq = q;
            if (cols) {
                const si::Index i = rng.categorical(p.data(), si::Index(p.size()));
                ctx->log_draw(i);
                const auto& blk = blocks[size_t(i)];
                qq = int64_t(blk.size());
                for (size_t j = 0; j < blk.size(); ++j) idx_host[j] = blk[j];
            } else if (sk == SI_SKETCH_ADAPTIVE_COLS_UNIFORM) {
                const auto idx = si::uniform_subset(rng, n, q);
                for (int64_t j = 0; j < q; ++j) {
                    idx_host[j] = idx[size_t(j)];
                    ctx->log_draw(idx[size_t(j)]);
                }
            } else if (sk == SI_SKETCH_ADAPTIVE_GAUSS) {
                rng.gaussian_fill(sv.pinned_sketch(), n, q, n);
                for (auto& r : sv.R) {
                    dev(r.c);
                    cuda_check(cudaMemcpyAsync(r.St, sv.s_pinned, size_t(n) * size_t(q) * 8, cudaMemcpyHostToDevice,
                                               r.c->stream),
                               "h2d st");
                }
                mode = 1;
            } else {
                mode = 2;
            }
            if (mode == 0) upload_idx(idx_host, qq, false);
            sv.reset_status();
            sv.enqueue_ada(mode, qq, -1, mode == 2);
            sv.read_status(st);
            if (st[0] || st[2]) {
                sv.redraws++;
                continue;
            }
            stepped = true;
        }
        const auto t1 = std::chrono::steady_clock::now();
        if (!stepped) {
            finish(SI_TERMINATION_ERROR, "sketch rejection limit exceeded for " + describe(sk, q) + " at iteration " +
                                             std::to_string(k));
            return;
        }
        if (cfg->track_wall_time) seconds += std::chrono::duration<double>(t1 - t0).count();
        if (cfg->track_flops) {
            flops += flops_adarbfgs(double(n), double(q));
            if (cols) flops += 2.0 * double(n) * double(n) * double(n);  // adarbfgs.cpp:168
        }
        if (st[1]) {
            finish(SI_TERMINATION_ERROR, "diverged: non-finite factor at iteration " + std::to_string(k));
            return;
        }
        if (k == 1 || k == cfg->max_iters || k % cfg->residual_every_k == 0)
            if (checkpoint()) return;
    }
    k = cfg->max_iters;
    finish(SI_MAX_ITERS, "");
}

// ------------------------------------------------ device-resident solver ---
ShardSolver* shard_solver_create(si_context* ctx, si_problem* prob, int method, int sketch, int64_t q, uint64_t seed) {
    if (method == SI_METHOD_RBFGS) {
        require(sketch == SI_SKETCH_GAUSSIAN_DEVICE, "multi-GPU solver: RBFGS runs with device Gaussian sketches");
    } else {
        require(sketch == SI_SKETCH_ADAPTIVE_COLS_UNIFORM || sketch == SI_SKETCH_ADAPTIVE_GAUSS_DEVICE,
                "multi-GPU solver: AdaRBFGS runs adaptive_cols_uniform or device Gaussian sketches");
    }
    validate_shared(prob);
    auto* s = new ShardSolver(ctx, prob, method, sketch, q, seed);
    s->set_identity();
    s->sync();
    return s;
}

// iters accepted iterations, the device keeping the accounting; returns the redraws
void shard_solver_step(ShardSolver* s, int64_t iters, si::RngStream& rng, int max_redraws) {
    int st[8];
    int64_t done = 0;
    int consecutive = 0;
    const int mode = s->method == SI_METHOD_RBFGS ? -1 : (s->sketch == SI_SKETCH_ADAPTIVE_COLS_UNIFORM ? 0 : 2);
    constexpr int64_t CAP = 64;
    if (mode == 0) s->ensure_ring(int(CAP));
    std::vector<si::RngStream> snaps;
    while (done < iters) {
        const int64_t nb = mode == 0 ? std::min(iters - done, CAP) : iters - done;
        if (mode == 0) {
            snaps.clear();
            for (int64_t b = 0; b < nb; ++b) {
                snaps.push_back(rng);
                const auto idx = si::uniform_subset(rng, s->n, s->q);
                for (int64_t j = 0; j < s->q; ++j) s->idx_pinned[b * s->q + j] = idx[size_t(j)];
            }
            snaps.push_back(rng);
            for (auto& r : s->R) {
                dev(r.c);
                cuda_check(cudaMemcpyAsync(r.idx_ring, s->idx_pinned, size_t(nb * s->q) * sizeof(int64_t),
                                           cudaMemcpyHostToDevice, r.c->stream),
                           "h2d idx");
            }
        }
        s->reset_status();
        for (int64_t b = 0; b < nb; ++b) {
            if (mode < 0)
                s->replay([&] { s->enqueue_rbfgs(s->q, true, true); });
            else
                s->enqueue_ada(mode, s->q, mode == 0 ? b : -1, true);
        }
        s->read_status(st);
        const int64_t accepted = mode < 0 ? st[3] : st[5];
        done += accepted;
        s->redraws += st[2];
        if (st[1]) throw NumericalError("diverged: non-finite iterate");
        if (st[4]) {
            if (mode == 0) rng = snaps[size_t(accepted) + 1];
            consecutive = (accepted > 0 ? 0 : consecutive) + 1;
            if (consecutive > max_redraws) throw NumericalError("solver: rejection limit exceeded");
        } else {
            consecutive = 0;
        }
    }
}

double shard_solver_residual(ShardSolver* s) { return s->residual(); }
void shard_solver_get(ShardSolver* s, double* host) {
    if (s->method == SI_METHOD_RBFGS)
        s->download_x(host);
    else
        s->download_l(host);
    s->sync();
}
void shard_solver_set(ShardSolver* s, const double* host) { s->set_from_host(host); }
int64_t shard_solver_redraws(ShardSolver* s) { return s->redraws; }

// ------------------------------------------------------- replication ---
void shard_replicate_problem(si_context* ctx, si_problem* h) {
    h->replicas.assign(1, h->p.get());
    if (!ctx->group) return;
    ShardGroup& G = *ctx->group;
    Problem& src = *h->p;
    for (int l = 1; l < G.nlocal(); ++l) {
        Context* c = G.ctx[size_t(l)];
        if (c->device == src.ctx->device) {  // virtual ranks of one device share A
            h->replicas.push_back(&src);
            continue;
        }
        auto p = std::make_unique<Problem>();
        p->ctx = c;
        p->n = src.n;
        p->symmetry = src.symmetry;
        p->dense = src.dense;
        p->nnz = src.nnz;
        dev(c);
        auto peer = [&](void** dst, const void* from, size_t bytes) {
            cuda_check(cudaMalloc(dst, std::max<size_t>(bytes, 8)), "cudaMalloc (replica)");
            cuda_check(cudaMemcpyPeer(*dst, c->device, from, src.ctx->device, bytes), "replicate A");
        };
        if (src.dense) {
            peer(reinterpret_cast<void**>(&p->a), src.a, size_t(src.n) * size_t(src.n) * 8);
        } else {
            peer(reinterpret_cast<void**>(&p->rowptr), src.rowptr, size_t(src.n + 1) * 8);
            peer(reinterpret_cast<void**>(&p->colind), src.colind, size_t(src.nnz) * 4);
            peer(reinterpret_cast<void**>(&p->val), src.val, size_t(src.nnz) * 8);
        }
        p->spd_checked = src.spd_checked;
        p->spd_ok = src.spd_ok;
        h->replicas.push_back(p.get());
        h->owned_replicas.push_back(std::move(p));
    }
}

}  // namespace si

// ------------------------------------------------------------------ C ABI --
extern "C" {

int si_nccl_unique_id(void* id_out) {
    return guard([&] {
        ncclUniqueId id;
        si::nck(si::nccl().getUniqueId(&id), "ncclGetUniqueId");
        static_assert(sizeof(id) == SI_NCCL_ID_BYTES, "ncclUniqueId size");
        std::memcpy(id_out, &id, sizeof(id));
    });
}

int si_context_create_rank(int device, void* stream, int nranks, int rank, const void* nccl_id, si_context** out) {
    return guard([&] {
        require(nranks >= 1 && rank >= 0 && rank < nranks, "context: rank out of range");
        auto h = std::make_unique<si_context>();
        h->c.reset(si::context_create(device, static_cast<cudaStream_t>(stream), stream != nullptr));
        auto g = std::make_unique<si::ShardGroup>();
        g->ctx.push_back(h->c.get());
        auto comm = std::make_unique<si::NcclComm>();
        comm->nranks = nranks;
        comm->rank0 = rank;
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        ncclComm_t cm = nullptr;
        si::dev(h->c.get());
        si::nck(si::nccl().commInitRank(&cm, nranks, id, rank), "ncclCommInitRank");
        comm->comms.push_back(cm);
        g->comm = std::move(comm);
        h->group = g.release();
        *out = h.release();
    });
}

int si_context_create_multi(const int* devices, int ndev, si_context** out) {
    return guard([&] {
        require(ndev >= 1, "context: at least one device");
        for (int i = 0; i < ndev; ++i)
            for (int j = 0; j < i; ++j)
                require(devices[i] != devices[j], "context: a device may appear once (use si_context_create_loopback)");
        auto h = std::make_unique<si_context>();
        h->c.reset(si::context_create(devices[0], nullptr));
        auto g = std::make_unique<si::ShardGroup>();
        g->ctx.push_back(h->c.get());
        for (int i = 1; i < ndev; ++i) {
            g->owned.emplace_back(si::context_create(devices[i], nullptr));
            g->ctx.push_back(g->owned.back().get());
        }
        auto comm = std::make_unique<si::NcclComm>();
        comm->nranks = ndev;
        comm->rank0 = 0;
        comm->comms.assign(size_t(ndev), nullptr);
        si::nck(si::nccl().commInitAll(comm->comms.data(), ndev, devices), "ncclCommInitAll");
        g->comm = std::move(comm);
        h->group = g.release();
        *out = h.release();
    });
}

int si_context_create_loopback(int device, int nranks, si_context** out) {
    return guard([&] {
        require(nranks >= 1, "context: at least one rank");
        auto h = std::make_unique<si_context>();
        h->c.reset(si::context_create(device, nullptr));
        auto g = std::make_unique<si::ShardGroup>();
        g->loopback = true;
        g->ctx.push_back(h->c.get());
        for (int i = 1; i < nranks; ++i) {  // every virtual rank on the first one's stream
            g->owned.emplace_back(si::context_create(device, h->c->stream));
            g->ctx.push_back(g->owned.back().get());
        }
        auto comm = std::make_unique<si::LoopbackComm>();
        comm->nranks = nranks;
        comm->rank0 = 0;
        comm->c0 = h->c.get();
        g->comm = std::move(comm);
        h->group = g.release();
        *out = h.release();
    });
}

int si_context_ranks(si_context* ctx, int* nranks, int* first_rank, int* local_ranks) {
    if (!ctx->group) {
        *nranks = 1;
        *first_rank = 0;
        *local_ranks = 1;
        return SI_OK;
    }
    *nranks = ctx->group->nranks();
    *first_rank = ctx->group->rank(0);
    *local_ranks = ctx->group->nlocal();
    return SI_OK;
}

}  // extern "C"
