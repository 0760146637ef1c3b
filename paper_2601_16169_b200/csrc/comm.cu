// Transports under the multi-rank schedules (comm.hpp): NCCL, and the
// in-process loopback that runs the same rank code with P host threads.
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "comm.hpp"
#include "common.cuh"

namespace detci_gpu {

// ---------------------------------------------------------------------------
// Kernel attribute records (per device, per kernel; thread-safe).
// ---------------------------------------------------------------------------
namespace {
std::mutex g_attr_mu;
std::map<std::pair<int, const void*>, size_t> g_smem;
std::map<std::pair<int, const void*>, int> g_carveout;
} // namespace

void ensure_dynamic_smem(const void* func, size_t smem) {
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_attr_mu);
    size_t& cur = g_smem[{dev, func}];
    if (smem <= cur) return;
    CUDA_CHECK(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    cur = smem;
}

void ensure_carveout(const void* func, int percent) {
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto it = g_carveout.find({dev, func});
    if (it != g_carveout.end() && it->second == percent) return;
    CUDA_CHECK(cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, percent));
    g_carveout[{dev, func}] = percent;
}

namespace {

// ---------------------------------------------------------------------------
// NCCL
// ---------------------------------------------------------------------------
void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(7, std::string(what) + ": " + ncclGetErrorString(r));
}

class NcclComm final : public Comm {
public:
    NcclComm(int rank, int world, const uint8_t id[128]) {
        ncclUniqueId uid;
        static_assert(sizeof(uid) == 128, "ncclUniqueId size");
        std::memcpy(&uid, id, sizeof(uid));
        nccl_check(ncclCommInitRank(&comm_, world, uid, rank), "ncclCommInitRank");
    }
    ~NcclComm() override {
        if (comm_) ncclCommDestroy(comm_);
    }
    const char* name() const override { return "nccl"; }
    void group_start() override {
        live();
        nccl_check(ncclGroupStart(), "ncclGroupStart");
    }
    void group_end() override { nccl_check(ncclGroupEnd(), "ncclGroupEnd"); }
    void broadcast(double* buf, size_t n, int root, cudaStream_t s) override {
        live();
        if (n) nccl_check(ncclBroadcast(buf, buf, n, ncclDouble, root, comm_, s), "ncclBroadcast");
    }
    void send(const double* buf, size_t n, int peer, cudaStream_t s) override {
        live();
        if (n) nccl_check(ncclSend(buf, n, ncclDouble, peer, comm_, s), "ncclSend");
    }
    void recv(double* buf, size_t n, int peer, cudaStream_t s) override {
        live();
        if (n) nccl_check(ncclRecv(buf, n, ncclDouble, peer, comm_, s), "ncclRecv");
    }
    void allreduce_sum(double* buf, size_t n, cudaStream_t s) override {
        live();
        if (n) nccl_check(ncclAllReduce(buf, buf, n, ncclDouble, ncclSum, comm_, s), "ncclAllReduce");
    }
    void abort() noexcept override {
        if (comm_) ncclCommAbort(comm_);
        comm_ = nullptr;
    }
    bool aborted() const override { return comm_ == nullptr; }

private:
    void live() const {
        if (!comm_) fail(1, "communicator aborted after an earlier failure");
    }
    ncclComm_t comm_ = nullptr;
};

// ---------------------------------------------------------------------------
// Loopback
// ---------------------------------------------------------------------------
enum class OpKind { Send, Recv, Bcast, AllReduce };

struct Op {
    OpKind kind;
    double* buf;
    size_t n;
    int peer;   // send/recv peer, broadcast root
};

// Shared state of one loopback rank group.
struct LoopGroup {
    explicit LoopGroup(int w) : world(w), posted(w), ready(w, nullptr), done(w, nullptr) {}
    const int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    bool aborted = false;
    std::vector<std::vector<Op>> posted;   // this group call's ops, per rank
    std::vector<cudaEvent_t> ready, done;  // per rank, owned by the rank's Comm

    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (aborted) fail(1, "loopback: a peer rank failed (group aborted)");
        const uint64_t gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
            return;
        }
        cv.wait(lk, [&] { return generation != gen || aborted; });
        if (generation == gen) fail(1, "loopback: a peer rank failed (group aborted)");
    }
    void abort() {
        std::lock_guard<std::mutex> lk(mu);
        aborted = true;
        cv.notify_all();
    }
};

std::mutex g_groups_mu;
std::map<uint64_t, std::weak_ptr<LoopGroup>> g_groups;

std::shared_ptr<LoopGroup> join_group(uint64_t id, int world) {
    std::lock_guard<std::mutex> lk(g_groups_mu);
    auto& slot = g_groups[id];
    std::shared_ptr<LoopGroup> g = slot.lock();
    if (!g || g->aborted) {
        g = std::make_shared<LoopGroup>(world);
        slot = g;
    }
    if (g->world != world) fail(4, "loopback: ranks of one group disagree on world_size");
    return g;
}

// out[i] = sum_{q < P} stage[q * n + i], summed in rank order (the same bits
// on every rank).
__global__ void k_rank_sum(const double* __restrict__ stage, size_t n, int P, double* __restrict__ out) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        double acc = stage[i];
        for (int q = 1; q < P; ++q) acc += stage[static_cast<size_t>(q) * n + i];
        out[i] = acc;
    }
}

class LoopbackComm final : public Comm {
public:
    LoopbackComm(uint64_t id, int rank, int world) : rank_(rank), world_(world), group_(join_group(id, world)) {
        CUDA_CHECK(cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming));
        CUDA_CHECK(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
        std::lock_guard<std::mutex> lk(group_->mu);
        if (group_->ready[rank_]) fail(4, "loopback: rank " + std::to_string(rank_) + " joined twice");
        group_->ready[rank_] = ready_;
        group_->done[rank_] = done_;
    }
    ~LoopbackComm() override {
        {
            std::lock_guard<std::mutex> lk(group_->mu);
            group_->ready[rank_] = nullptr;
            group_->done[rank_] = nullptr;
        }
        if (stage_) cudaFree(stage_);
        cudaEventDestroy(ready_);
        cudaEventDestroy(done_);
    }
    const char* name() const override { return "loopback"; }
    void group_start() override {
        if (in_group_) fail(1, "loopback: nested group");
        in_group_ = true;
        ops_.clear();
        stream_ = nullptr;
    }
    void group_end() override {
        if (!in_group_) fail(1, "loopback: group_end without group_start");
        in_group_ = false;
        try {
            run();
        } catch (...) {
            abort();   // peers waiting in this group's barriers fail too
            throw;
        }
    }
    void broadcast(double* buf, size_t n, int root, cudaStream_t s) override { add({OpKind::Bcast, buf, n, root}, s); }
    void send(const double* buf, size_t n, int peer, cudaStream_t s) override {
        add({OpKind::Send, const_cast<double*>(buf), n, peer}, s);
    }
    void recv(double* buf, size_t n, int peer, cudaStream_t s) override { add({OpKind::Recv, buf, n, peer}, s); }
    void allreduce_sum(double* buf, size_t n, cudaStream_t s) override { add({OpKind::AllReduce, buf, n, 0}, s); }
    void abort() noexcept override {
        aborted_ = true;
        group_->abort();
    }
    bool aborted() const override { return aborted_; }

private:
    void add(const Op& op, cudaStream_t s) {
        if (aborted_) fail(1, "communicator aborted after an earlier failure");
        if ((op.kind == OpKind::Send || op.kind == OpKind::Recv || op.kind == OpKind::Bcast) &&
            (op.peer < 0 || op.peer >= world_))
            fail(4, "loopback: peer rank out of range");
        if (stream_ && s != stream_) fail(1, "loopback: one group must use one stream");
        stream_ = s;
        ops_.push_back(op);
        if (!in_group_) {   // a lone call is a group of one
            in_group_ = true;
            group_end();
        }
    }

    // The exchange of one group:
    //   1. record `ready` (every op's buffer is final), post the ops, barrier;
    //   2. copy what this rank receives out of the peers' posted buffers
    //      (after their `ready`), record `done`, barrier;
    //   3. wait for every peer's `done` (nobody overwrites a buffer a peer
    //      still reads), then reduce the staged all-reduce operands.
    void run() {
        LoopGroup& G = *group_;
        const cudaStream_t s = stream_;
        if (s) CUDA_CHECK(cudaEventRecord(ready_, s));
        {
            std::lock_guard<std::mutex> lk(G.mu);
            G.posted[rank_] = ops_;
        }
        G.barrier();
        std::vector<size_t> stage_off;
        size_t stage_need = 0;
        for (const Op& op : ops_)
            if (op.kind == OpKind::AllReduce) {
                stage_off.push_back(stage_need);
                stage_need += op.n * static_cast<size_t>(world_);
            }
        if (stage_need > stage_n_) {
            if (stage_) CUDA_CHECK(cudaFree(stage_));
            stage_ = nullptr;
            CUDA_CHECK(cudaMalloc(&stage_, stage_need * sizeof(double)));
            stage_n_ = stage_need;
        }
        std::vector<char> waited(world_, 0);
        auto wait_ready = [&](int q) {
            if (q == rank_ || waited[q]) return;
            CUDA_CHECK(cudaStreamWaitEvent(s, G.ready[q], 0));
            waited[q] = 1;
        };
        auto nth = [&](int q, OpKind kind, int peer, int k) -> const Op* {
            int seen = 0;
            for (const Op& op : G.posted[q])
                if (op.kind == kind && (peer < 0 || op.peer == peer) && seen++ == k) return &op;
            return nullptr;
        };
        std::vector<int> recv_k(world_, 0);
        int bcast_k = 0, red_k = 0;
        for (const Op& op : ops_) {
            if (op.kind == OpKind::Recv) {
                const Op* src = nth(op.peer, OpKind::Send, rank_, recv_k[op.peer]++);
                if (!src) fail(7, "loopback: recv from rank " + std::to_string(op.peer) + " has no matching send");
                if (src->n != op.n)
                    fail(7, "loopback: recv count " + std::to_string(op.n) + " != send count " +
                                std::to_string(src->n) + " (rank " + std::to_string(op.peer) + " -> " +
                                std::to_string(rank_) + ")");
                wait_ready(op.peer);
                if (op.n) CUDA_CHECK(cudaMemcpyAsync(op.buf, src->buf, op.n * 8, cudaMemcpyDeviceToDevice, s));
            } else if (op.kind == OpKind::Bcast) {
                const Op* src = nth(op.peer, OpKind::Bcast, -1, bcast_k++);
                if (!src || src->peer != op.peer || src->n != op.n)
                    fail(7, "loopback: broadcast " + std::to_string(bcast_k - 1) + " differs between ranks");
                if (op.peer != rank_ && op.n) {
                    wait_ready(op.peer);
                    CUDA_CHECK(cudaMemcpyAsync(op.buf, src->buf, op.n * 8, cudaMemcpyDeviceToDevice, s));
                }
            } else if (op.kind == OpKind::AllReduce) {
                const int k = red_k++;
                for (int q = 0; q < world_; ++q) {
                    const Op* src = nth(q, OpKind::AllReduce, -1, k);
                    if (!src || src->n != op.n)
                        fail(7, "loopback: all-reduce " + std::to_string(k) + " differs between ranks");
                    wait_ready(q);
                    if (op.n)
                        CUDA_CHECK(cudaMemcpyAsync(stage_ + stage_off[k] + static_cast<size_t>(q) * op.n, src->buf,
                                                   op.n * 8, cudaMemcpyDeviceToDevice, s));
                }
            }
        }
        // sends nobody received: the peer's group differs
        for (int q = 0; q < world_; ++q) {
            if (q == rank_) continue;
            int posted_sends = 0;
            for (const Op& op : G.posted[q])
                if (op.kind == OpKind::Send && op.peer == rank_) ++posted_sends;
            if (posted_sends != recv_k[q])
                fail(7, "loopback: rank " + std::to_string(q) + " sent " + std::to_string(posted_sends) +
                            " messages to rank " + std::to_string(rank_) + ", " + std::to_string(recv_k[q]) +
                            " received");
        }
        if (s) CUDA_CHECK(cudaEventRecord(done_, s));
        G.barrier();
        if (s) {
            for (int q = 0; q < world_; ++q)
                if (q != rank_) CUDA_CHECK(cudaStreamWaitEvent(s, G.done[q], 0));
            int k = 0;
            for (const Op& op : ops_)
                if (op.kind == OpKind::AllReduce) {
                    if (op.n) {
                        const unsigned grid = static_cast<unsigned>(std::min<size_t>((op.n + 255) / 256, 1184));
                        k_rank_sum<<<grid, 256, 0, s>>>(stage_ + stage_off[k], op.n, world_, op.buf);
                        CUDA_LAUNCH_CHECK();
                    }
                    ++k;
                }
        }
        ops_.clear();
        stream_ = nullptr;
    }

    const int rank_, world_;
    std::shared_ptr<LoopGroup> group_;
    cudaEvent_t ready_ = nullptr, done_ = nullptr;
    std::vector<Op> ops_;
    cudaStream_t stream_ = nullptr;
    bool in_group_ = false, aborted_ = false;
    double* stage_ = nullptr;
    size_t stage_n_ = 0;
};

} // namespace

std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const uint8_t id[128]) {
    return std::make_unique<NcclComm>(rank, world, id);
}

std::unique_ptr<Comm> make_loopback_comm(uint64_t group, int rank, int world) {
    return std::make_unique<LoopbackComm>(group, rank, world);
}

} // namespace detci_gpu
