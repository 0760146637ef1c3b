// extern "C" boundary of libdetci_gpu.so (include/detci_gpu.h).  Every entry
// point converts internal failures to a status code (no exception crosses
// the ABI) and records the message for detci_gpu_last_error.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include <nccl.h>

#include "comm.hpp"
#include "formulas.cuh"
#include "handle.hpp"

using namespace detci_gpu;

namespace detci_gpu {
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
} // namespace detci_gpu

struct detci_gpu_handle {
    Handle h;
};

namespace {

thread_local std::string g_last_error;

// collective: the call may enter rank collectives (build, sigma, Davidson).
// A failure there aborts the rank transport, so peers blocked in (or later
// entering) a collective fail instead of waiting forever; the handle's
// multi-rank calls fail from then on (recreate the group).
template <class F>
int guarded(detci_gpu_handle* hh, F&& body, bool collective = false) {
    int code = DETCI_GPU_OK;
    try {
        body();
        return DETCI_GPU_OK;
    } catch (const Failure& f) {
        if (hh) hh->h.err = f.what();
        g_last_error = f.what();
        code = f.code;
    } catch (const std::bad_alloc&) {
        const char* msg = "host allocation failed";
        if (hh) hh->h.err = msg;
        g_last_error = msg;
        code = DETCI_GPU_E_CAPACITY;
    } catch (const std::exception& e) {
        if (hh) hh->h.err = e.what();
        g_last_error = e.what();
        code = DETCI_GPU_E_ERROR;
    }
    if (collective && hh && hh->h.comm) hh->h.comm->abort();
    return code;
}

void require(bool ok, int code, const std::string& msg) {
    if (!ok) fail(code, msg);
}

void activate(const Handle& h) { CUDA_CHECK(cudaSetDevice(h.device)); }

__global__ void k_precondition(const double* __restrict__ r, const double* __restrict__ d, uint64_t n,
                               double theta, double* __restrict__ out) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double denom = d[i] - theta;
        if (fabs(denom) < 1e-8) denom = copysign(1e-8, denom);
        out[i] = r[i] / denom;
    }
}

__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, uint64_t n, double a) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        y[i] -= a * x[i];
}

__global__ void k_div(double* __restrict__ y, uint64_t n, double a) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        y[i] /= a;
}

double host_j(const double* eri, int n, int p, int q, Bits spec) {
    double acc = 0.0;
    while (any(spec)) {
        const int r = lowest(spec);
        spec = drop_lowest(spec);
        acc += eri_at(eri, n, p, q, r, r);
    }
    return acc;
}

// <bra|H|ket> from the kernels' factorized forms (detci_gpu_factorized_element).
double factorized_element_bits(int norbs, double core, const double* h1, const double* eri, Bits bra_a,
                               Bits bra_b, Bits ket_a, Bits ket_b) {
    const int da = popc(bra_a ^ ket_a) / 2;
    const int db = popc(bra_b ^ ket_b) / 2;
    require(popc(bra_a) == popc(ket_a) && popc(bra_b) == popc(ket_b), DETCI_GPU_E_INPUT,
            "factorized_element: spin-nonconserving pair");
    if (da + db > 2) return 0.0;
    if (da == 0 && db == 0) {  // diagonal, regrouped as in k_diag
        auto energy = [&](Bits s) {
            double acc = 0.0;
            for (Bits a = s; any(a);) {
                const int p = lowest(a);
                a = drop_lowest(a);
                acc += h1[p * norbs + p];
                for (Bits b = a; any(b);) {
                    const int q = lowest(b);
                    b = drop_lowest(b);
                    acc += eri_at(eri, norbs, p, p, q, q) - eri_at(eri, norbs, p, q, q, p);
                }
            }
            return acc;
        };
        double x = 0.0;
        for (Bits a = bra_a; any(a); a = drop_lowest(a)) {
            const int p = lowest(a);
            for (Bits b = bra_b; any(b); b = drop_lowest(b)) x += eri_at(eri, norbs, p, p, lowest(b), lowest(b));
        }
        return core + energy(bra_a) + energy(bra_b) + x;
    }
    // separated-ordering element times eps(bra) eps(ket) (formulas.cuh)
    const int eps = eps_parity(bra_a, prefix_parity(bra_b)) ^ eps_parity(ket_a, prefix_parity(ket_b));
    if (db == 0 || da == 0) {  // same-spin: alpha (ch 0) or beta (ch 1)
        const int ch = db == 0 ? 0 : 1;
        const Bits si = ch == 0 ? bra_a : bra_b, sj = ch == 0 ? ket_a : ket_b;
        const Bits spec = ch == 0 ? bra_b : bra_a;
        const int kind = (ch == 0 ? da : db) - 1;
        const PairEntry e = make_pair_entry(kind, si, sj, h1, eri, norbs);
        double v = e.v;
        if (kind == 0) {
            const double j = host_j(eri, norbs, lowest(si & ~sj), lowest(sj & ~si), spec);
            v += (e.ab_sign >> 31) ? -j : j;
        }
        return eps ? -v : v;
    }
    // mixed alpha single x beta single
    const int pa = lowest(bra_a & ~ket_a), qa = lowest(ket_a & ~bra_a);
    const MixedMove mv = mixed_move(bra_b, ket_b, norbs);
    const int cd = static_cast<int>(mv.cd);
    double w = mixed_weight(eri, norbs, pa, qa, cd / norbs, cd % norbs);
    if (mv.sbit ^ mixed_alpha_parity(bra_a, pa, qa) ^ eps) w = -w;
    return w;
}

} // namespace

extern "C" {

int detci_gpu_abi_version(void) { return DETCI_GPU_ABI_VERSION; }

const char* detci_gpu_last_error(const detci_gpu_handle* h) {
    return h ? h->h.err.c_str() : g_last_error.c_str();
}

int detci_gpu_nccl_unique_id(uint8_t out[128]) {
    return guarded(nullptr, [&] {
        ncclUniqueId id;
        if (ncclGetUniqueId(&id) != ncclSuccess) fail(DETCI_GPU_E_CUDA, "ncclGetUniqueId failed");
        static_assert(sizeof(id) == 128, "ncclUniqueId size");
        std::memcpy(out, &id, 128);
    });
}

namespace {
// transport: 0 NCCL (desc->nccl_id), 1 loopback group `group`
int create_handle(const detci_gpu_desc* desc, detci_gpu_handle** out, int transport, uint64_t group) {
    return guarded(nullptr, [&] {
        require(desc && out, DETCI_GPU_E_INPUT, "create: null argument");
        *out = nullptr;
        require(desc->world_size >= 1 && desc->rank >= 0 && desc->rank < desc->world_size,
                DETCI_GPU_E_CONFIG, "create: invalid rank/world_size");
        require(desc->virtual_blocks >= 0, DETCI_GPU_E_CONFIG, "create: negative virtual_blocks");
        require(!(desc->world_size > 1 && desc->virtual_blocks > 1), DETCI_GPU_E_CONFIG,
                "create: virtual_blocks requires world_size 1");
        int ndev = 0;
        CUDA_CHECK(cudaGetDeviceCount(&ndev));
        require(ndev > 0, DETCI_GPU_E_CUDA, "create: no CUDA device");
        auto* hh = new detci_gpu_handle();
        Handle& h = hh->h;
        try {
            h.device = desc->device >= 0 ? desc->device : 0;
            if (desc->device < 0) CUDA_CHECK(cudaGetDevice(&h.device));
            require(h.device < ndev, DETCI_GPU_E_CONFIG, "create: device ordinal out of range");
            CUDA_CHECK(cudaSetDevice(h.device));
            h.rank = desc->rank;
            h.world = desc->world_size;
            h.vblocks = std::max(1, desc->virtual_blocks);
            h.weighted = desc->weighted_partition;
            h.budget = desc->memory_budget_bytes;
            CUDA_CHECK(cudaStreamCreateWithFlags(&h.stream, cudaStreamNonBlocking));
            CUDA_CHECK(cudaStreamCreateWithFlags(&h.comm_stream, cudaStreamNonBlocking));
            for (auto& e : h.ev) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            if (h.world > 1 && transport == 0) {
                require(desc->nccl_id != nullptr, DETCI_GPU_E_CONFIG, "create: nccl_id required");
                h.comm = make_nccl_comm(h.rank, h.world, desc->nccl_id);
            } else if (h.world > 1) {
                h.comm = make_loopback_comm(group, h.rank, h.world);
            }
        } catch (...) {
            detci_gpu_destroy(hh);
            throw;
        }
        *out = hh;
    });
}
} // namespace

int detci_gpu_create(const detci_gpu_desc* desc, detci_gpu_handle** out) {
    return create_handle(desc, out, 0, 0);
}

int detci_gpu_create_loopback(const detci_gpu_desc* desc, uint64_t group, detci_gpu_handle** out) {
    return create_handle(desc, out, 1, group);
}

void detci_gpu_destroy(detci_gpu_handle* hh) {
    if (!hh) return;
    Handle& h = hh->h;
    cudaSetDevice(h.device);
    if (h.stream) cudaStreamSynchronize(h.stream);
    if (h.comm_stream) cudaStreamSynchronize(h.comm_stream);
    release_basis(h);
    for (auto& c : h.ch) {
        c.strings.reset();
        c.prefix.reset();
    }
    h.d_h1.reset();
    h.d_eri.reset();
    h.red.reset();
    h.red_count.reset();
    h.comm.reset();
    if (h.pin_x) cudaFreeHost(h.pin_x);
    if (h.pin_y) cudaFreeHost(h.pin_y);
    for (auto& e : h.ev)
        if (e) cudaEventDestroy(e);
    if (h.stream) cudaStreamDestroy(h.stream);
    if (h.comm_stream) cudaStreamDestroy(h.comm_stream);
    delete hh;
}

int detci_gpu_set_strings(detci_gpu_handle* hh, int norbs, const uint64_t* alpha, size_t na,
                          const uint64_t* beta, size_t nb) {
    return detci_gpu_set_strings_words(hh, norbs, 1, alpha, na, beta, nb);
}

int detci_gpu_set_strings_words(detci_gpu_handle* hh, int norbs, int words, const uint64_t* alpha, size_t na,
                                const uint64_t* beta, size_t nb) {
    return guarded(hh, [&] {
        require(hh != nullptr, DETCI_GPU_E_INPUT, "set_strings: null handle");
        Handle& h = hh->h;
        require(norbs >= 1, DETCI_GPU_E_INPUT, "set_strings: norbs must be positive");
        // Reference limit is kMaxKernelBits = 256 spin-orbitals (basis.cpp:83-87);
        // the device strings are one or two uint64 words per channel.
        require(2 * norbs <= 256, DETCI_GPU_E_INPUT,
                "build_basis: " + std::to_string(2 * norbs) + " spin-orbitals exceed the kernel limit of 256");
        require(words == 1 || words == 2, DETCI_GPU_E_INPUT, "set_strings: words must be 1 or 2");
        require(norbs <= 64 * words, DETCI_GPU_E_INPUT,
                "set_strings: " + std::to_string(norbs) + " orbitals need " + std::to_string((norbs + 63) / 64) +
                    " words per string");
        require(norbs <= 64 || mixed_scatter_enabled(), DETCI_GPU_E_UNSUPPORTED,
                "set_strings: norbs > 64 needs the scatter mixed kernel (DETCI_MIXED=gather is set)");
        require(h.have_ints == false || norbs == h.norbs, DETCI_GPU_E_INPUT,
                "set_strings: norbs does not match the integrals");
        const char* names[2] = {"alpha", "beta"};
        const uint64_t* src[2] = {alpha, beta};
        const size_t cnt[2] = {na, nb};
        // allowed bits per word
        uint64_t allowed[2] = {0, 0};
        for (int w = 0; w < 2; ++w) {
            const int bits = std::max(0, std::min(64, norbs - 64 * w));
            allowed[w] = bits == 64 ? ~0ull : ((1ull << bits) - 1);
        }
        const bool wide = norbs > 64;
        for (int c = 0; c < 2; ++c) {
            require(cnt[c] > 0 && src[c] != nullptr, DETCI_GPU_E_INPUT,
                    std::string("build_basis: empty ") + names[c] + " string list");
            require(cnt[c] < (1ull << 31), DETCI_GPU_E_UNSUPPORTED, "set_strings: more than 2^31 strings");
            int ne = -1;
            for (size_t i = 0; i < cnt[c]; ++i) {
                int pc = 0;
                for (int w = 0; w < words; ++w) {
                    const uint64_t x = src[c][i * words + w];
                    require((x & ~allowed[w]) == 0, DETCI_GPU_E_INPUT,
                            std::string("build_basis: ") + names[c] + " string " + std::to_string(i) +
                                " has wrong orbital count");
                    pc += __builtin_popcountll(x);
                }
                if (ne < 0) ne = pc;
                require(pc == ne, DETCI_GPU_E_INPUT,
                        std::string("build_basis: inconsistent electron count in ") + names[c] +
                            " strings (string " + std::to_string(i) + ")");
            }
            h.ch[c].n_elec = ne;
        }
        activate(h);
        release_basis(h);
        h.norbs = norbs;
        for (int c = 0; c < 2; ++c) {
            ChannelTables& t = h.ch[c];
            t.n = cnt[c];
            t.h_strings.resize(t.n);
            t.h_strings_hi.assign(wide ? t.n : 0, 0ull);
            for (size_t i = 0; i < t.n; ++i) {
                t.h_strings[i] = src[c][i * words];
                if (wide) t.h_strings_hi[i] = src[c][i * words + 1];
            }
            t.strings.alloc(t.n);
            copy_sync(t.strings.p, t.h_strings.data(), t.n * sizeof(uint64_t), cudaMemcpyHostToDevice, h.stream);
            // exclusive prefix parities P(s) for eps(A,B) = popc(A & P(B)) & 1
            std::vector<uint64_t> pre(t.n), pre_hi(wide ? t.n : 0);
            for (size_t i = 0; i < t.n; ++i) {
                const Bits p = prefix_parity(Bits(t.h_strings[i], wide ? t.h_strings_hi[i] : 0ull));
                pre[i] = p.lo;
                if (wide) pre_hi[i] = p.hi;
            }
            t.prefix.alloc(t.n);
            copy_sync(t.prefix.p, pre.data(), t.n * sizeof(uint64_t), cudaMemcpyHostToDevice, h.stream);
            if (wide) {
                t.strings_hi.alloc(t.n);
                t.prefix_hi.alloc(t.n);
                copy_sync(t.strings_hi.p, t.h_strings_hi.data(), t.n * 8, cudaMemcpyHostToDevice, h.stream);
                copy_sync(t.prefix_hi.p, pre_hi.data(), t.n * 8, cudaMemcpyHostToDevice, h.stream);
            } else {
                t.strings_hi.reset();
                t.prefix_hi.reset();
            }
        }
        h.have_strings = true;
    });
}

int detci_gpu_set_integrals(detci_gpu_handle* hh, double core, const double* h1, const double* eri) {
    return guarded(hh, [&] {
        require(hh != nullptr, DETCI_GPU_E_INPUT, "set_integrals: null handle");
        Handle& h = hh->h;
        require(h.have_strings, DETCI_GPU_E_INPUT, "set_integrals: call set_strings first");
        require(h1 && eri, DETCI_GPU_E_INPUT, "set_integrals: null integrals");
        activate(h);
        release_basis(h);
        const size_t n = static_cast<size_t>(h.norbs);
        h.core = core;
        h.h1.assign(h1, h1 + n * n);
        h.eri.assign(eri, eri + n * n * n * n);
        h.d_h1.alloc(n * n);
        h.d_eri.alloc(n * n * n * n);
        copy_sync(h.d_h1.p, h.h1.data(), n * n * 8, cudaMemcpyHostToDevice, h.stream);
        copy_sync(h.d_eri.p, h.eri.data(), n * n * n * n * 8, cudaMemcpyHostToDevice, h.stream);
        h.have_ints = true;
    });
}

int detci_gpu_build_basis(detci_gpu_handle* hh) {
    return guarded(hh, [&] {
        require(hh != nullptr, DETCI_GPU_E_INPUT, "build_basis: null handle");
        activate(hh->h);
        build_device_basis(hh->h);
    }, true);
}

int detci_gpu_helper_size(const detci_gpu_handle* hh, int channel, int kind, uint64_t* nflat) {
    return guarded(const_cast<detci_gpu_handle*>(hh), [&] {
        require(hh && hh->h.built, DETCI_GPU_E_INPUT, "helpers: basis not built");
        require(channel >= 0 && channel < 2 && kind >= 0 && kind < 2, DETCI_GPU_E_INPUT,
                "helpers: bad channel/kind");
        *nflat = hh->h.ch[channel].nflat[kind];
    });
}

int detci_gpu_get_helpers(const detci_gpu_handle* hh, int channel, int kind, uint32_t* flat,
                          uint64_t* offset, uint32_t* len) {
    return guarded(const_cast<detci_gpu_handle*>(hh), [&] {
        require(hh && hh->h.built, DETCI_GPU_E_INPUT, "helpers: basis not built");
        require(channel >= 0 && channel < 2 && kind >= 0 && kind < 2, DETCI_GPU_E_INPUT,
                "helpers: bad channel/kind");
        const Handle& h = hh->h;
        activate(h);
        const ChannelTables& t = h.ch[channel];
        if (flat && t.nflat[kind])
            copy_sync(flat, t.flat[kind].p, t.nflat[kind] * 4, cudaMemcpyDeviceToHost, h.stream);
        if (offset) copy_sync(offset, t.offset[kind].p, t.n * 8, cudaMemcpyDeviceToHost, h.stream);
        if (len) copy_sync(len, t.len[kind].p, t.n * 4, cudaMemcpyDeviceToHost, h.stream);
    });
}

int detci_gpu_local_rows(const detci_gpu_handle* hh, uint64_t* row_begin, uint64_t* row_end,
                         uint64_t* n_beta) {
    return guarded(const_cast<detci_gpu_handle*>(hh), [&] {
        require(hh && hh->h.built, DETCI_GPU_E_INPUT, "local_rows: basis not built");
        *row_begin = hh->h.a0;
        *row_end = hh->h.a1;
        *n_beta = hh->h.nb();
    });
}

int detci_gpu_nnz(const detci_gpu_handle* hh, uint64_t* total, uint64_t* a, uint64_t* b, uint64_t* m) {
    return guarded(const_cast<detci_gpu_handle*>(hh), [&] {
        require(hh && hh->h.built, DETCI_GPU_E_INPUT, "nnz: basis not built");
        const Handle& h = hh->h;
        if (a) *a = h.nnz_alpha;
        if (b) *b = h.nnz_beta;
        if (m) *m = h.nnz_mixed;
        if (total) *total = h.nnz_alpha + h.nnz_beta + h.nnz_mixed;
    });
}

int detci_gpu_diag(const detci_gpu_handle* hh, double* out) {
    return guarded(const_cast<detci_gpu_handle*>(hh), [&] {
        require(hh && hh->h.built, DETCI_GPU_E_INPUT, "diag: basis not built");
        activate(hh->h);
        copy_sync(out, hh->h.diag.p, hh->h.local_len() * 8, cudaMemcpyDeviceToHost, hh->h.stream);
    });
}

int detci_gpu_plan_partition(uint64_t na, uint64_t nb, const uint32_t* sa, const uint32_t* da,
                             const uint32_t* sb, const uint32_t* db, int P, int weighted, uint64_t* blk) {
    return guarded(nullptr, [&] {
        require(blk && (!weighted || (sa && da && sb && db)), DETCI_GPU_E_INPUT,
                "plan_partition: null argument");
        plan_partition(na, nb, sa, da, sb, db, P, weighted, blk);
    });
}

int detci_gpu_sigma_device(detci_gpu_handle* hh, const double* dx, double* dy, detci_gpu_timings* tm) {
    return guarded(hh, [&] {
        require(hh != nullptr && dx && dy, DETCI_GPU_E_INPUT, "sigma: null argument");
        require(dx != dy, DETCI_GPU_E_INPUT, "sigma: x and y must not alias");
        activate(hh->h);
        if (tm) *tm = detci_gpu_timings{};
        sigma_device(hh->h, dx, dy, tm);
    }, true);
}

int detci_gpu_rebalance(detci_gpu_handle* hh, int rounds, double* max_over_mean) {
    return guarded(hh, [&] {
        require(hh != nullptr && hh->h.built, DETCI_GPU_E_INPUT, "rebalance: basis not built");
        require(rounds >= 0, DETCI_GPU_E_CONFIG, "rebalance: rounds must be >= 0");
        Handle& h = hh->h;
        activate(h);
        const int P = std::max(h.world, h.vblocks);
        for (int r = 0; r < rounds && P > 1; ++r) {
            // a timed sigma of a constant vector (the kernels' cost does not
            // depend on the values)
            DevBuf<double> x, y;
            const size_t n = std::max<size_t>(h.local_len(), 1);
            x.alloc(n);
            y.alloc(n);
            CUDA_CHECK(cudaMemsetAsync(x.p, 0x3f, n * sizeof(double), h.stream));
            detci_gpu_timings tm{};
            sigma_device(h, x.p, y.p, &tm);
            std::vector<double> t(4 * static_cast<size_t>(P), 0.0);
            if (h.world > 1) {
                for (int q = 0; q < 4; ++q) t[4 * static_cast<size_t>(h.rank) + q] = h.own_phase_seconds[q];
                allreduce_sum(h, t.data(), static_cast<int>(t.size()));
            } else {
                t = h.rank_phase_seconds;
            }
            if (max_over_mean && r == 0) {
                double mx = 0.0, sum = 0.0;
                for (int g = 0; g < P; ++g) {
                    const double v = t[4 * g] + t[4 * g + 1] + t[4 * g + 2] + t[4 * g + 3];
                    mx = std::max(mx, v);
                    sum += v;
                }
                *max_over_mean = sum > 0 ? mx * P / sum : 1.0;
            }
            rebalance_partition(h, t);
        }
    }, true);
}

int detci_gpu_sigma_async(detci_gpu_handle* hh, const double* dx, double* dy) {
    return guarded(hh, [&] {
        require(hh != nullptr && dx && dy, DETCI_GPU_E_INPUT, "sigma: null argument");
        require(dx != dy, DETCI_GPU_E_INPUT, "sigma: x and y must not alias");
        activate(hh->h);
        sigma_enqueue(hh->h, dx, dy);
    }, true);
}

int detci_gpu_stream(const detci_gpu_handle* hh, void** stream) {
    return guarded(const_cast<detci_gpu_handle*>(hh), [&] {
        require(hh && stream, DETCI_GPU_E_INPUT, "stream: null argument");
        *stream = reinterpret_cast<void*>(hh->h.stream);
    });
}

int detci_gpu_launch_count(uint64_t* count) {
    return guarded(nullptr, [&] {
        require(count != nullptr, DETCI_GPU_E_INPUT, "launch_count: null argument");
        *count = g_launches.load();
    });
}

int detci_gpu_sigma(detci_gpu_handle* hh, const double* x, double* y, detci_gpu_timings* tm) {
    return guarded(hh, [&] {
        require(hh != nullptr && x && y, DETCI_GPU_E_INPUT, "sigma: null argument");
        Handle& h = hh->h;
        require(h.built, DETCI_GPU_E_INPUT, "sigma: basis not built");
        activate(h);
        if (sigma_host(h, x, y, tm)) return;
        const size_t n = h.local_len();
        h.xbuf.alloc(n);
        h.ybuf.alloc(n);
        cudaEvent_t e[4];
        for (auto& ev : e) CUDA_CHECK(cudaEventCreate(&ev));
        CUDA_CHECK(cudaEventRecord(e[0], h.stream));
        CUDA_CHECK(cudaMemcpyAsync(h.xbuf.p, x, n * 8, cudaMemcpyHostToDevice, h.stream));
        CUDA_CHECK(cudaEventRecord(e[1], h.stream));
        if (tm) *tm = detci_gpu_timings{};
        sigma_device(h, h.xbuf.p, h.ybuf.p, tm);
        CUDA_CHECK(cudaEventRecord(e[2], h.stream));
        CUDA_CHECK(cudaMemcpyAsync(y, h.ybuf.p, n * 8, cudaMemcpyDeviceToHost, h.stream));
        CUDA_CHECK(cudaEventRecord(e[3], h.stream));
        CUDA_CHECK(cudaEventSynchronize(e[3]));
        if (tm) {
            float a = 0.f, b = 0.f, c = 0.f;
            CUDA_CHECK(cudaEventElapsedTime(&a, e[0], e[1]));
            CUDA_CHECK(cudaEventElapsedTime(&b, e[2], e[3]));
            CUDA_CHECK(cudaEventElapsedTime(&c, e[0], e[3]));
            tm->h2d_seconds = a * 1e-3;
            tm->d2h_seconds = b * 1e-3;
            tm->total_seconds = c * 1e-3;
        }
        for (auto& ev : e) cudaEventDestroy(ev);
    }, true);
}

int detci_gpu_sigma_plan(const detci_gpu_handle* hh, detci_gpu_plan* out) {
    return guarded(const_cast<detci_gpu_handle*>(hh), [&] {
        require(hh && out && hh->h.built, DETCI_GPU_E_INPUT, "sigma_plan: basis not built");
        const Handle& h = hh->h;
        *out = detci_gpu_plan{};
        const SellTable& t = h.sell_scatter[0];
        out->mixed_kmax = t.kmax;
        out->mixed_segments = static_cast<int>(t.nseg);
        out->mixed_windows = h.scatter_plan.empty() ? 0 : static_cast<int>(h.scatter_plan[0].size());
        out->mixed_sell_entries = t.sell.n;
        out->d_bytes = h.dbuf.bytes();
        // single-GPU plan (P = 1): one item per ja with its whole singles
        // list, cut into passes of kmax rows plus one remainder pass padded
        // to the next power of two; every pass walks all SELL entries and
        // issues (K + 1) 8-byte loads per entry (K V rows, one Cs gather)
        if (t.kmax > 0 && h.h_sa_off.size() == h.na() + 1) {
            uint64_t loads_per_entry = 0, pairs = 0;
            for (size_t ja = 0; ja < h.na(); ++ja) {
                const uint64_t len = h.h_sa_off[ja + 1] - h.h_sa_off[ja];
                pairs += len;
                const uint64_t full = len / t.kmax, rem = len % t.kmax;
                loads_per_entry += full * (t.kmax + 1);
                if (rem) {
                    uint64_t k = 1;
                    while (k < rem) k <<= 1;
                    loads_per_entry += k + 1;
                }
            }
            out->mixed_lds_bytes = 8 * t.sell.n * loads_per_entry;
            out->d_read_bytes = h.scatter_plan.empty() ? 0 : 8 * pairs * h.nb();
        }
    });
}

int detci_gpu_rank_seconds(const detci_gpu_handle* hh, double* out, int cap, int* count) {
    return guarded(const_cast<detci_gpu_handle*>(hh), [&] {
        require(hh && count, DETCI_GPU_E_INPUT, "rank_seconds: null argument");
        const auto& r = hh->h.rank_seconds;
        *count = static_cast<int>(r.size());
        for (int i = 0; i < cap && i < static_cast<int>(r.size()); ++i) out[i] = r[i];
    });
}

int detci_gpu_rank_phase_seconds(const detci_gpu_handle* hh, double* out, int cap, int* count) {
    return guarded(const_cast<detci_gpu_handle*>(hh), [&] {
        require(hh && count, DETCI_GPU_E_INPUT, "rank_phase_seconds: null argument");
        const auto& r = hh->h.rank_phase_seconds;
        *count = static_cast<int>(r.size());
        for (int i = 0; i < cap && i < static_cast<int>(r.size()); ++i) out[i] = r[i];
    });
}

int detci_gpu_alloc_vector(detci_gpu_handle* hh, double** dptr) {
    return guarded(hh, [&] {
        require(hh && hh->h.built && dptr, DETCI_GPU_E_INPUT, "alloc_vector: basis not built");
        activate(hh->h);
        CUDA_CHECK(cudaMalloc(dptr, std::max<size_t>(hh->h.local_len(), 1) * 8));
    });
}

int detci_gpu_free_vector(detci_gpu_handle* hh, double* dptr) {
    return guarded(hh, [&] {
        require(hh != nullptr, DETCI_GPU_E_INPUT, "free_vector: null handle");
        activate(hh->h);
        CUDA_CHECK(cudaFree(dptr));
    });
}

// kind: 0 host->device, 1 device->host, 2 device->device (local length)
int detci_gpu_copy_vector(detci_gpu_handle* hh, double* dst, const double* src, int kind) {
    return guarded(hh, [&] {
        require(hh && hh->h.built && dst && src, DETCI_GPU_E_INPUT, "copy_vector: bad argument");
        activate(hh->h);
        const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice
                                          : (kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
        CUDA_CHECK(cudaMemcpyAsync(dst, src, hh->h.local_len() * 8, k, hh->h.stream));
        CUDA_CHECK(cudaStreamSynchronize(hh->h.stream));
    });
}

int detci_gpu_davidson(detci_gpu_handle* hh, const detci_dav_opts* opts, detci_dav_result* res,
                       detci_trace_cb cb, void* user) {
    return guarded(hh, [&] {
        require(hh && opts && res, DETCI_GPU_E_INPUT, "davidson: null argument");
        activate(hh->h);
        davidson_device(hh->h, *opts, res, cb, user);
    }, true);
}

int detci_gpu_davidson_roots(detci_gpu_handle* hh, const detci_dav_block_opts* opts,
                             detci_dav_block_result* res) {
    return guarded(hh, [&] {
        require(hh && opts && res, DETCI_GPU_E_INPUT, "davidson_roots: null argument");
        activate(hh->h);
        davidson_roots_device(hh->h, *opts, res);
    }, true);
}

int detci_gpu_sigma_block(detci_gpu_handle* hh, const double* const* dx, double* const* dy, int m) {
    return guarded(hh, [&] {
        require(hh && dx && dy && m >= 1, DETCI_GPU_E_INPUT, "sigma_block: bad argument");
        activate(hh->h);
        sigma_block(hh->h, dx, dy, m);
    }, true);
}

int detci_gpu_build_stored(detci_gpu_handle* hh, uint64_t memory_budget_bytes, uint64_t* nnz) {
    return guarded(hh, [&] {
        require(hh != nullptr, DETCI_GPU_E_INPUT, "build_stored_matrix: null handle");
        activate(hh->h);
        build_stored(hh->h, memory_budget_bytes, nnz);
    });
}

int detci_gpu_stored_arrays(const detci_gpu_handle* hh, uint64_t* row_offset, uint32_t* col, double* value) {
    return guarded(const_cast<detci_gpu_handle*>(hh), [&] {
        require(hh != nullptr, DETCI_GPU_E_INPUT, "stored_arrays: null handle");
        const Handle& h = hh->h;
        require(h.st_off.p != nullptr, DETCI_GPU_E_INPUT, "stored_arrays: matrix not built");
        activate(const_cast<Handle&>(h));
        const uint64_t dim = h.na() * h.nb();
        if (row_offset) copy_sync(row_offset, h.st_off.p, (dim + 1) * 8, cudaMemcpyDeviceToHost, h.stream);
        if (col) copy_sync(col, h.st_col.p, h.st_nnz * 4, cudaMemcpyDeviceToHost, h.stream);
        if (value) copy_sync(value, h.st_val.p, h.st_nnz * 8, cudaMemcpyDeviceToHost, h.stream);
    });
}

int detci_gpu_set_operator(detci_gpu_handle* hh, int kind) {
    return guarded(hh, [&] {
        require(hh != nullptr, DETCI_GPU_E_INPUT, "set_operator: null handle");
        require(kind == 0 || kind == 1, DETCI_GPU_E_CONFIG, "set_operator: kind must be 0 or 1");
        require(kind == 0 || hh->h.st_off.p != nullptr, DETCI_GPU_E_INPUT,
                "set_operator: build the stored matrix first");
        hh->h.use_stored = kind == 1;
    });
}

int detci_gpu_release_stored(detci_gpu_handle* hh) {
    return guarded(hh, [&] {
        require(hh != nullptr, DETCI_GPU_E_INPUT, "release_stored: null handle");
        activate(hh->h);
        release_stored(hh->h);
    });
}

int detci_gpu_inner_product(detci_gpu_handle* hh, const double* x, const double* y, uint64_t n,
                            double* out) {
    return guarded(hh, [&] {
        require(hh && x && y && out, DETCI_GPU_E_INPUT, "inner_product: null argument");
        require(hh->h.world == 1, DETCI_GPU_E_UNSUPPORTED, "inner_product: single-GPU helper");
        activate(hh->h);
        DevBuf<double> dx, dy;
        dx.alloc(std::max<uint64_t>(n, 1));
        dy.alloc(std::max<uint64_t>(n, 1));
        copy_sync(dx.p, x, n * 8, cudaMemcpyHostToDevice, hh->h.stream);
        copy_sync(dy.p, y, n * 8, cudaMemcpyHostToDevice, hh->h.stream);
        *out = device_dot(hh->h, dx.p, dy.p, n);
    });
}

int detci_gpu_orthonormalize(detci_gpu_handle* hh, const double* vs, int k, uint64_t n,
                             const double* candidate, double* out, int* accepted) {
    return guarded(hh, [&] {
        require(hh && candidate && out && accepted && (k == 0 || vs), DETCI_GPU_E_INPUT,
                "orthonormalize: null argument");
        require(hh->h.world == 1, DETCI_GPU_E_UNSUPPORTED, "orthonormalize: single-GPU helper");
        Handle& h = hh->h;
        activate(h);
        DevBuf<double> dv, dc;
        dv.alloc(std::max<uint64_t>(static_cast<uint64_t>(k) * n, 1));
        dc.alloc(std::max<uint64_t>(n, 1));
        if (k) copy_sync(dv.p, vs, static_cast<size_t>(k) * n * 8, cudaMemcpyHostToDevice, h.stream);
        copy_sync(dc.p, candidate, n * 8, cudaMemcpyHostToDevice, h.stream);
        for (int pass = 0; pass < 2; ++pass)
            for (int j = 0; j < k; ++j) {
                const double* bv = dv.p + static_cast<size_t>(j) * n;
                const double o = device_dot(h, bv, dc.p, n);
                k_axpy<<<592, 256, 0, h.stream>>>(dc.p, bv, n, o);
                CUDA_LAUNCH_CHECK();
            }
        const double norm = std::sqrt(device_dot(h, dc.p, dc.p, n));
        *accepted = norm >= 1e-10 ? 1 : 0;
        if (*accepted) {
            k_div<<<592, 256, 0, h.stream>>>(dc.p, n, norm);
            CUDA_LAUNCH_CHECK();
        }
        CUDA_CHECK(cudaStreamSynchronize(h.stream));
        copy_sync(out, dc.p, n * 8, cudaMemcpyDeviceToHost, h.stream);
    });
}

int detci_gpu_precondition(detci_gpu_handle* hh, const double* residual, const double* diag,
                           uint64_t n, double theta, double* out) {
    return guarded(hh, [&] {
        require(hh && residual && diag && out, DETCI_GPU_E_INPUT, "precondition: null argument");
        Handle& h = hh->h;
        activate(h);
        DevBuf<double> dr, dd;
        dr.alloc(std::max<uint64_t>(n, 1));
        dd.alloc(std::max<uint64_t>(n, 1));
        copy_sync(dr.p, residual, n * 8, cudaMemcpyHostToDevice, h.stream);
        copy_sync(dd.p, diag, n * 8, cudaMemcpyHostToDevice, h.stream);
        k_precondition<<<592, 256, 0, h.stream>>>(dr.p, dd.p, n, theta, dr.p);
        CUDA_LAUNCH_CHECK();
        CUDA_CHECK(cudaStreamSynchronize(h.stream));
        copy_sync(out, dr.p, n * 8, cudaMemcpyDeviceToHost, h.stream);
    });
}

// Diagnostic (host execution, no GPU): the element <bra|H|ket> as the sigma
// kernels assemble it from the factorized closed forms of formulas.cuh.
// E_INPUT when the pair is not connected by <= 2 spin-conserving moves.
int detci_gpu_factorized_element(int norbs, double core, const double* h1, const double* eri,
                                 uint64_t bra_a, uint64_t bra_b, uint64_t ket_a, uint64_t ket_b,
                                 double* out) {
    return guarded(nullptr, [&] {
        *out = factorized_element_bits(norbs, core, h1, eri, Bits(bra_a), Bits(bra_b), Bits(ket_a), Bits(ket_b));
    });
}

int detci_gpu_factorized_element_words(int norbs, int words, double core, const double* h1, const double* eri,
                                       const uint64_t* bra_a, const uint64_t* bra_b, const uint64_t* ket_a,
                                       const uint64_t* ket_b, double* out) {
    return guarded(nullptr, [&] {
        require(words == 1 || words == 2, DETCI_GPU_E_INPUT, "factorized_element: words must be 1 or 2");
        require(norbs <= 64 * words, DETCI_GPU_E_INPUT, "factorized_element: norbs exceeds the words");
        auto w = [&](const uint64_t* x) { return Bits(x[0], words > 1 ? x[1] : 0ull); };
        *out = factorized_element_bits(norbs, core, h1, eri, w(bra_a), w(bra_b), w(ket_a), w(ket_b));
    });
}

} // extern "C"
