// Multi-GPU plumbing of the C ABI (shard.cpp): the communicator abstraction the sharded
// drivers use and the group of ranks a multi-GPU si_context drives.
//
//   NcclComm      NCCL over NVLink / NVSwitch, loaded on demand (dlopen of libnccl.so.2,
//                 reusing an already-loaded copy such as torch's): one communicator per
//                 local device, calls of all local ranks inside one ncclGroupStart/End.
//   LoopbackComm  P virtual ranks on ONE device sharing one stream, the collectives
//                 replayed as device copies / reductions at group end — the harness that
//                 runs the sharded drivers' P > 1 logic on a single GPU (tests only; no
//                 rank ever waits on another, nothing here is a performance claim).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <memory>
#include <vector>

#include "engine.hpp"

namespace si {

enum class RedOp { sum, max };

struct Comm {
    int nranks = 1;  // global ranks
    int rank0 = 0;   // global rank of local rank 0 (local ranks are consecutive)
    virtual ~Comm() = default;
    virtual void group_start() {}
    virtual void group_end() {}
    // in place; doubles or int32
    virtual void all_reduce(int l, void* buf, size_t count, bool is_int, RedOp op, cudaStream_t s) = 0;
    // recv = concat over ranks of each rank's `count` doubles
    virtual void all_gather(int l, const double* send, double* recv, size_t count, cudaStream_t s) = 0;
    // root's `send` to every rank's `recv` (root may pass recv == send)
    virtual void broadcast(int l, const double* send, double* recv, size_t count, int root, cudaStream_t s) = 0;
    virtual void send(int l, const double* buf, size_t count, int peer, cudaStream_t s) = 0;
    virtual void recv(int l, double* buf, size_t count, int peer, cudaStream_t s) = 0;
    // device scratch the collectives may need (loopback reductions), sized before graph capture
    virtual void reserve(size_t) {}
};

struct ShardGroup {
    std::vector<Context*> ctx;                   // local ranks; ctx[0] is the si_context's own
    std::vector<std::unique_ptr<Context>> owned;  // ctx[1..]
    std::unique_ptr<Comm> comm;
    bool loopback = false;
    int nranks() const { return comm->nranks; }
    int rank(int l) const { return comm->rank0 + l; }
    int nlocal() const { return int(ctx.size()); }
    bool owns(int g) const { return g >= comm->rank0 && g < comm->rank0 + nlocal(); }
    ~ShardGroup();
};

}  // namespace si
