// Transport under the multi-rank schedules (sigma.cu sigma_gather_rank and
// the ring, davidson.cu reductions and argmin).  The rank code is written
// once against this interface; two implementations sit under it:
//
//   NCCL      one process (or host thread) per GPU, ncclComm_t over
//             NVLink/NVSwitch -- the production transport;
//   loopback  `world` handles in one process, each driven by its own host
//             thread, usually on one GPU: point-to-point and broadcast are
//             device copies ordered by CUDA events, all-reduce sums the
//             ranks' buffers in rank order, and a host barrier separates the
//             phases.  It runs the SAME rank functions as NCCL, so the
//             multi-rank code is exercised on a single-GPU box.
//
// Semantics follow NCCL: calls between group_start/group_end form one
// group; the k-th send from a to b matches the k-th recv on b from a (counts
// must agree); the k-th broadcast / all-reduce of a group is the same
// collective on every rank.  Every rank enters every group (possibly empty).
// All operations of one group are enqueued on one stream.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>

namespace detci_gpu {

class Comm {
public:
    virtual ~Comm() = default;
    virtual const char* name() const = 0;
    virtual void group_start() = 0;
    virtual void group_end() = 0;
    // in-place: root's buf is copied into every other rank's buf
    virtual void broadcast(double* buf, size_t n, int root, cudaStream_t s) = 0;
    virtual void send(const double* buf, size_t n, int peer, cudaStream_t s) = 0;
    virtual void recv(double* buf, size_t n, int peer, cudaStream_t s) = 0;
    // in-place sum over ranks; every rank receives the same bits
    virtual void allreduce_sum(double* buf, size_t n, cudaStream_t s) = 0;
    // After a local failure: make peers blocked in (or later entering) a
    // collective fail instead of waiting forever.  The communicator is
    // unusable afterwards.
    virtual void abort() noexcept = 0;
    virtual bool aborted() const = 0;
};

std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const uint8_t id[128]);
// Ranks passing the same `group` id (and world) form one loopback group.
std::unique_ptr<Comm> make_loopback_comm(uint64_t group, int rank, int world);

// Kernel attributes are per device and several host threads may launch the
// same kernel concurrently: raise a kernel's dynamic shared-memory limit on
// the current device to at least `smem` (never lowers it; thread-safe).
void ensure_dynamic_smem(const void* func, size_t smem);
// Set the preferred shared-memory carveout once per (device, kernel).
void ensure_carveout(const void* func, int percent);

} // namespace detci_gpu
