// sigma = H C over the alpha x beta tensor-product basis (matvec,
// matvec.cpp:125-228), B200-native, for M = 1, 2 or 4 vectors per pass.
//
// The kernels work in the separated determinant ordering (formulas.cuh):
// with Cs = eps o C and eps(A,B) = (-1)^{popc(A & P(B))},
//   y  = diag*C + eps o sum_ja Ha(ia,ja;B_ib) Cs[ja,ib]       k_samespin on Cs
//   yT =          sum_jb Hb(ib,jb;A_ia) Cs^T[jb,ia]           k_samespin on Cs^T
//   y += eps o sum_ja sum_jb Hm Cs[ja,jb]                     k_mixed
//   y += eps o yT^T                                           k_transpose_add_eps
// where every separated-ordering element carries only same-channel signs, so
// no kernel evaluates a per-element spectator parity; eps is applied once per
// determinant in the prologue (k_eps_transpose writes Cs and Cs^T) and in the
// epilogues.
//
// Gather formulation: every output element is owned by exactly one thread,
// so there are no atomics and the result is deterministic.  The beta term
// runs the alpha kernel on the transposed block, which turns its per-row
// gathers into coalesced row reads (the transposes cost 32 B/det against
// ~8 B x thousands of elements per det).  With M vectors, every element's
// value work (same-spin) and its W gather and SELL entry (mixed) are
// shared by the M vectors (the multi-root block Davidson's new block).
//
// This file: the eps prologue/epilogue kernels, the schedules (one block,
// the multi-block gather schedule, the ring) and the entry points; the
// same-spin kernels live in samespin.cu, the mixed term in mixed.cu.
//
// Multi-GPU / virtual blocks: alpha rows are partitioned into P blocks;
// the alpha and mixed terms need Cs rows from every block, which rotate
// ring-wise (NCCL send/recv on a comm stream, double-buffered, overlapped
// with the compute of the resident block).  The beta term and diagonal are
// block-local.
#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "formulas.cuh"
#include "handle.hpp"
#include "sigma_device.cuh"
#include "sigma_internal.hpp"

namespace detci_gpu {

namespace {

// ---------------------------------------------------------------------------
// eps prologue / epilogue, through 32x32 smem tiles (coalesced both ways).
// ---------------------------------------------------------------------------
constexpr int kTile = 32;

// Local block x (rows x cols, row r = alpha string a_str[r], column c = beta
// string with prefix parity b_pre[c]):
//   xs[r * ldx + c] = eps x      (if xs)     xsT[c * ldt + r] = eps x (if xsT)
__global__ void k_eps_transpose(const double* __restrict__ x, size_t ldx, double* __restrict__ xs,
                                double* __restrict__ xsT, size_t ldt, uint32_t rows, uint32_t cols,
                                const EpsRows e) {
    __shared__ double tile[kTile][kTile + 1];
    __shared__ uint64_t s_a[2][kTile];
    const uint32_t c0 = blockIdx.x * kTile, r0 = blockIdx.y * kTile;
    const uint32_t cc = c0 + threadIdx.x;
    const Bits pb = cc < cols ? load_bits(e.b, e.b_hi, cc) : Bits();
    if (threadIdx.y == 0 && r0 + threadIdx.x < rows) {
        s_a[0][threadIdx.x] = e.a[r0 + threadIdx.x];
        s_a[1][threadIdx.x] = e.a_hi ? e.a_hi[r0 + threadIdx.x] : 0ull;
    }
    __syncthreads();
    for (uint32_t y = threadIdx.y; y < kTile; y += blockDim.y) {
        const uint32_t rr = r0 + y;
        if (rr < rows && cc < cols) {
            const size_t i = static_cast<size_t>(rr) * ldx + cc;
            const double v = flip_sign(x[i], static_cast<uint32_t>(eps_parity(Bits(s_a[0][y], s_a[1][y]), pb)));
            if (xs) xs[i] = v;
            tile[y][threadIdx.x] = v;
        }
    }
    if (!xsT) return;
    __syncthreads();
    for (uint32_t y = threadIdx.y; y < kTile; y += blockDim.y) {
        const uint32_t c = c0 + y, rr = r0 + threadIdx.x;
        if (rr < rows && c < cols) xsT[static_cast<size_t>(c) * ldt + rr] = tile[threadIdx.x][y];
    }
}

// dst[r * ldd + c] += eps(a_str[r], b_pre[c]) src[c * lds + r], dst rows x cols
__global__ void k_transpose_add_eps(const double* __restrict__ src, size_t lds, double* __restrict__ dst,
                                    size_t ldd, uint32_t rows, uint32_t cols,
                                    const EpsRows e) {
    __shared__ double tile[kTile][kTile + 1];
    __shared__ uint64_t s_a[2][kTile];
    const uint32_t c0 = blockIdx.x * kTile, r0 = blockIdx.y * kTile;
    for (uint32_t y = threadIdx.y; y < kTile; y += blockDim.y) {
        const uint32_t c = c0 + y, rr = r0 + threadIdx.x;
        if (rr < rows && c < cols) tile[y][threadIdx.x] = src[static_cast<size_t>(c) * lds + rr];
    }
    if (threadIdx.y == 0 && r0 + threadIdx.x < rows) {
        s_a[0][threadIdx.x] = e.a[r0 + threadIdx.x];
        s_a[1][threadIdx.x] = e.a_hi ? e.a_hi[r0 + threadIdx.x] : 0ull;
    }
    __syncthreads();
    const uint32_t cc = c0 + threadIdx.x;
    const Bits pb = cc < cols ? load_bits(e.b, e.b_hi, cc) : Bits();
    for (uint32_t y = threadIdx.y; y < kTile; y += blockDim.y) {
        const uint32_t rr = r0 + y;
        if (rr < rows && cc < cols)
            dst[static_cast<size_t>(rr) * ldd + cc] +=
                flip_sign(tile[threadIdx.x][y], static_cast<uint32_t>(eps_parity(Bits(s_a[0][y], s_a[1][y]), pb)));
    }
}

// ---------------------------------------------------------------------------
// Host orchestration.
// ---------------------------------------------------------------------------


// Scratch for M vectors: Cs^T / sigma^T blocks, the eps-signed Cs (the
// whole vector for virtual blocks, whose ring reads other blocks before
// their own prologue ran) and ring buffers.
void ensure_scratch(Handle& h, int M, int P) {
    const size_t block = static_cast<size_t>(h.max_blk) * h.nb();
    if (h.ct.n < M * block) {
        h.ct.alloc(M * block);
        h.yt.alloc(M * block);
    }
    const size_t xs = M * (h.vblocks > 1 ? h.na() * h.nb() : block);
    if (h.xs.n < xs) h.xs.alloc(xs);
    if (P > 1 && h.ring[0].n < M * block) {
        h.ring[0].alloc(M * block);
        h.ring[1].alloc(M * block);
    }
}

// eps prologue for rows [a0, a1): Cs (row-major, if xs_loc) and Cs^T (h.ct).
template <int M>
void eps_prologue(Handle& h, const Ptrs& x_loc, const MPtrs& xs_loc, bool transpose, uint64_t a0,
                  uint64_t a1) {
    const uint32_t nloc = static_cast<uint32_t>(a1 - a0), nb = static_cast<uint32_t>(h.nb());
    const size_t block = static_cast<size_t>(h.max_blk) * h.nb();
    if (nloc == 0 || nb == 0) return;
    dim3 tb(kTile, 8), tg((nb + kTile - 1) / kTile, (nloc + kTile - 1) / kTile);
    for (int v = 0; v < M; ++v) {
        k_eps_transpose<<<tg, tb, 0, h.stream>>>(x_loc[v], nb, xs_loc[v], transpose ? h.ct.p + v * block : nullptr,
                                                 nloc, nloc, nb, eps_rows(h, a0));
        CUDA_LAUNCH_CHECK();
    }
}

// The beta term for rows [a0, a1): same-spin kernel on Cs^T (h.ct, written
// by the prologue), raw result in h.yt (M x [nb][nloc]); eps is applied by
// the combine.
template <int M>
void beta_term(Handle& h, uint64_t a0, uint64_t a1) {
    const uint32_t nloc = static_cast<uint32_t>(a1 - a0), nb = static_cast<uint32_t>(h.nb());
    const size_t block = static_cast<size_t>(h.max_blk) * h.nb();
    SameSpinArgs s{};
    for (int v = 0; v < M; ++v) {
        s.C[v] = h.ct.p + v * block;
        s.Y[v] = h.yt.p + v * block;
    }
    s.ldc = nloc;
    s.c_row0 = 0;
    s.j0 = 0;
    s.j1 = nb;
    s.ldy = nloc;
    s.row0 = 0;
    s.nrows = nb;
    s.ncols = nloc;
    s.J = h.ch[0].J.p + a0;
    s.ldj = h.na();
    fill_lists(s, h.ch[1]);
    s.accumulate = 0;
    launch_samespin<M>(s, h.stream);
}

template <int M>
void combine(Handle& h, const MPtrs& y_loc, uint64_t a0, uint64_t a1, PhaseTimer& tm) {
    const uint32_t nloc = static_cast<uint32_t>(a1 - a0), nb = static_cast<uint32_t>(h.nb());
    const size_t block = static_cast<size_t>(h.max_blk) * h.nb();
    if (nloc == 0 || nb == 0) return;
    const int id = tm.begin(3);
    dim3 tb(kTile, 8), tg((nb + kTile - 1) / kTile, (nloc + kTile - 1) / kTile);
    for (int v = 0; v < M; ++v) {
        k_transpose_add_eps<<<tg, tb, 0, h.stream>>>(h.yt.p + v * block, nloc, y_loc[v], nb, nloc, nb,
                                                     eps_rows(h, a0));
        CUDA_LAUNCH_CHECK();
    }
    tm.end(id);
}

// One block-rank's sigma with the Cs ring.  `fetch(s, held, dst, block)`
// enqueues on h.comm_stream the transfer that makes alpha block `block`
// resident in dst (M consecutive block-sized slabs) for step s + 1 (NCCL
// send/recv, or a device copy for virtual blocks).
template <int M, class Fetch>
void sigma_ring(Handle& h, int g, int P, const Ptrs& x_loc, const MPtrs& xs_loc, const MPtrs& y_loc,
                PhaseTimer& tm, Fetch&& fetch) {
    const uint64_t a0 = h.blk[g], a1 = h.blk[g + 1];
    const size_t block = static_cast<size_t>(h.max_blk) * h.nb();
    cudaEvent_t* done_compute = h.ev;      // [0..1]
    cudaEvent_t* done_comm = h.ev + 2;     // [2..3]
    int id = tm.begin(1);
    eps_prologue<M>(h, x_loc, xs_loc, true, a0, a1);
    // Cs and the ring buffers are produced / last read on the compute
    // stream: the comm stream must not send or overwrite them before that.
    CUDA_CHECK(cudaEventRecord(h.ev[4], h.stream));
    CUDA_CHECK(cudaStreamWaitEvent(h.comm_stream, h.ev[4], 0));
    beta_term<M>(h, a0, a1);
    tm.end(id);
    Ptrs held{};
    for (int v = 0; v < M; ++v) held[v] = xs_loc[v];
    for (int s = 0; s < P; ++s) {
        const int b = (g + s) % P;
        if (s + 1 < P) {
            // ring[s%2] was read by compute at step s-1
            if (s >= 1) CUDA_CHECK(cudaStreamWaitEvent(h.comm_stream, done_compute[(s - 1) % 2], 0));
            fetch(s, held, h.ring[s % 2].p, (g + s + 1) % P);
            CUDA_CHECK(cudaEventRecord(done_comm[s % 2], h.comm_stream));
        }
        const uint32_t b0 = static_cast<uint32_t>(h.blk[b]), b1 = static_cast<uint32_t>(h.blk[b + 1]);
        id = tm.begin(0);
        launch_alpha<M>(h, held, b0, b1, x_loc, y_loc, a0, a1, s == 0);
        tm.end(id);
        id = tm.begin(2);
        if (M <= 2 && mixed_scatter_enabled())
            launch_mixed_scatter<M == 2 ? 2 : 1>(h, g, P, b, held, b0, b1, y_loc, a0);
        else
            launch_mixed<M>(h, held, b0, b1, y_loc, a0, a1);
        tm.end(id);
        CUDA_CHECK(cudaEventRecord(done_compute[s % 2], h.stream));
        if (s + 1 < P) {
            CUDA_CHECK(cudaStreamWaitEvent(h.stream, done_comm[s % 2], 0));
            for (int v = 0; v < M; ++v) held[v] = h.ring[s % 2].p + v * block;
        }
    }
    combine<M>(h, y_loc, a0, a1, tm);
}

// ---------------------------------------------------------------------------
// Multi-block "gather" schedule (default for P > 1; DETCI_MULTI=ring keeps the
// ring).  The ring's mixed term restricts each CTA item (ja, K outputs) to
// the outputs of one rank, i.e. to ~|S(ja)|/P rows, so items shrink to K of
// 4-8 at P = 8 (1.2-1.6x the per-element cost, measured with virtual
// blocks).  Here every rank holds the whole Cs (allgather, dim x 8 B, under
// the beta term), runs the alpha term in one launch, and computes the mixed
// term for ALL alpha rows but only its 1/P of the beta slots, with the full
// K = 16 items; the resulting column slab is exchanged all-to-all (dim/P x
// 8 B per rank) and unpacked into the local rows.
// ---------------------------------------------------------------------------
// Scratch of the gather schedule: the whole Cs (M vectors), this rank's
// column slab T (na x ns_g) and the received slabs R (nloc x ns_g' each).
void ensure_gather_scratch(Handle& h, int M, int P) {
    const size_t na = h.na(), nb = h.nb();
    const size_t full = na * nb;
    if (h.world > 1 && h.cs_full.n < M * full) h.cs_full.alloc(M * full);
    size_t tmax = 0;
    for (int g = 0; g < P; ++g) {
        const auto [s0, s1] = mixed_slots(h, g, P);
        tmax = std::max<size_t>(tmax, s1 - s0);
    }
    const size_t t = (h.world > 1 ? na * tmax : full + na * kWarp * static_cast<size_t>(P));
    if (h.mix_t.n < M * t) h.mix_t.alloc(M * t);
    if (h.world > 1) {
        const size_t r = static_cast<size_t>(h.max_blk) * (nb + kWarp * static_cast<size_t>(P));
        if (h.mix_r.n < M * r) h.mix_r.alloc(M * r);
    }
}

// One rank (world > 1) of the gather schedule over the rank transport
// (comm.hpp: NCCL, or the in-process loopback).
template <int M>
void sigma_gather_rank(Handle& h, const Ptrs& x_loc, const MPtrs& y_loc, PhaseTimer& tm) {
    const int g = h.rank, P = h.world;
    const uint64_t a0 = h.blk[g], a1 = h.blk[g + 1], nloc = a1 - a0;
    const size_t na = h.na(), nb = h.nb(), full = na * nb;
    Ptrs cf{};
    MPtrs cfw{};
    for (int v = 0; v < M; ++v) {
        cf[v] = h.cs_full.p + v * full;
        cfw[v] = h.cs_full.p + v * full + a0 * nb;
    }
    int id = tm.begin(1);
    eps_prologue<M>(h, x_loc, cfw, true, a0, a1);   // own rows of Cs, and Cs^T
    CUDA_CHECK(cudaEventRecord(h.ev[4], h.stream));
    CUDA_CHECK(cudaStreamWaitEvent(h.comm_stream, h.ev[4], 0));
    // allgather of the P row blocks (in-place broadcasts from each owner)
    h.comm->group_start();
    for (int v = 0; v < M; ++v)
        for (int b = 0; b < P; ++b) {
            double* blk = h.cs_full.p + v * full + h.blk[b] * nb;
            h.comm->broadcast(blk, (h.blk[b + 1] - h.blk[b]) * nb, b, h.comm_stream);
        }
    h.comm->group_end();
    CUDA_CHECK(cudaEventRecord(h.ev[5], h.comm_stream));
    beta_term<M>(h, a0, a1);                        // local, under the allgather
    tm.end(id);
    CUDA_CHECK(cudaStreamWaitEvent(h.stream, h.ev[5], 0));
    id = tm.begin(0);
    launch_alpha<M>(h, cf, 0, static_cast<uint32_t>(na), x_loc, y_loc, a0, a1, true);
    tm.end(id);
    id = tm.begin(2);
    const auto [s0, s1] = mixed_slots(h, g, P);
    const size_t ns = s1 - s0;
    double* T[kMaxM] = {};
    for (int v = 0; v < M; ++v) T[v] = h.mix_t.p + v * na * ns;
    mixed_columns<M>(h, g, P, cf, T, ns);
    // all-to-all of the slab: rows of rank b go to b; slabs from every rank
    // land in R (source-major, nloc x ns_src each)
    CUDA_CHECK(cudaEventRecord(h.ev[6], h.stream));
    CUDA_CHECK(cudaStreamWaitEvent(h.comm_stream, h.ev[6], 0));
    const size_t rstride = static_cast<size_t>(h.max_blk) * (nb + kWarp * static_cast<size_t>(P));
    std::vector<size_t> roff(P + 1, 0);
    for (int b = 0; b < P; ++b) {
        const auto [t0, t1] = mixed_slots(h, b, P);
        roff[b + 1] = roff[b] + nloc * (t1 - t0);
    }
    h.comm->group_start();
    for (int v = 0; v < M; ++v)
        for (int b = 0; b < P; ++b) {
            const auto [t0, t1] = mixed_slots(h, b, P);
            const size_t send_n = (h.blk[b + 1] - h.blk[b]) * ns, recv_n = nloc * (t1 - t0);
            double* src = T[v] + h.blk[b] * ns;
            double* dst = h.mix_r.p + v * rstride + roff[b];
            if (b == g) {
                if (send_n)
                    CUDA_CHECK(cudaMemcpyAsync(dst, src, send_n * 8, cudaMemcpyDeviceToDevice, h.comm_stream));
                continue;
            }
            h.comm->send(src, send_n, b, h.comm_stream);
            h.comm->recv(dst, recv_n, b, h.comm_stream);
        }
    h.comm->group_end();
    CUDA_CHECK(cudaEventRecord(h.ev[7], h.comm_stream));
    CUDA_CHECK(cudaStreamWaitEvent(h.stream, h.ev[7], 0));
    for (int v = 0; v < M; ++v)
        for (int b = 0; b < P; ++b) {
            const auto [t0, t1] = mixed_slots(h, b, P);
            unpack_slab<M>(h, h.mix_r.p + v * rstride + roff[b], t1 - t0, t1 - t0, nloc, t0, y_loc[v]);
        }
    tm.end(id);
    combine<M>(h, y_loc, a0, a1, tm);
}

// The gather schedule emulated on one GPU (virtual blocks): every rank's
// work in turn; the allgather is the whole Cs signed up front, the
// all-to-all is the column slabs of all ranks unpacked into the whole y.
template <int M>
void sigma_gather_virtual(Handle& h, const Ptrs& dx, const MPtrs& dy, PhaseTimer& tm) {
    const int P = h.vblocks;
    const size_t na = h.na(), nb = h.nb(), full = na * nb;
    const size_t tstride = full + na * kWarp * static_cast<size_t>(P);
    Ptrs cf{};
    MPtrs cfw{};
    for (int v = 0; v < M; ++v) {
        cf[v] = h.xs.p + v * full;
        cfw[v] = h.xs.p + v * full;
    }
    eps_prologue<M>(h, dx, cfw, false, 0, na);
    for (int g = 0; g < P; ++g) {
        tm.rank_tag = g;
        const uint64_t a0 = h.blk[g], a1 = h.blk[g + 1];
        Ptrs xg{};
        MPtrs yg{}, cg{};
        for (int v = 0; v < M; ++v) {
            xg[v] = dx[v] + a0 * nb;
            yg[v] = dy[v] + a0 * nb;
            cg[v] = h.xs.p + v * full + a0 * nb;
        }
        int id = tm.begin(1);
        eps_prologue<M>(h, xg, cg, true, a0, a1);
        beta_term<M>(h, a0, a1);
        tm.end(id);
        id = tm.begin(0);
        launch_alpha<M>(h, cf, 0, static_cast<uint32_t>(na), xg, yg, a0, a1, true);
        tm.end(id);
        combine<M>(h, yg, a0, a1, tm);
    }
    size_t toff = 0;
    for (int g = 0; g < P; ++g) {
        tm.rank_tag = g;
        const int id = tm.begin(2);
        const auto [s0, s1] = mixed_slots(h, g, P);
        const size_t ns = s1 - s0;
        double* T[kMaxM] = {};
        for (int v = 0; v < M; ++v) T[v] = h.mix_t.p + v * tstride + toff;
        mixed_columns<M>(h, g, P, cf, T, ns);
        for (int v = 0; v < M; ++v) unpack_slab<M>(h, T[v], ns, static_cast<uint32_t>(ns), na, s0, dy[v]);
        toff += na * ns;
        tm.end(id);
    }
    tm.rank_tag = -1;
}

template <int M>
void sigma_schedule_m(Handle& h, const Ptrs& dx, const MPtrs& dy, PhaseTimer& tm) {
    const int Pm = std::max(h.world, h.vblocks);
    if constexpr (M <= 2) {   // the scatter kernel runs M <= 2
        if (Pm > 1 && mixed_scatter_enabled() && !multi_ring()) {
            ensure_scratch(h, M, 1);
            ensure_gather_scratch(h, M, Pm);
            if (h.world > 1) sigma_gather_rank<M>(h, dx, dy, tm);
            else sigma_gather_virtual<M>(h, dx, dy, tm);
            return;
        }
    }
    const size_t nb = h.nb();
    const int P = std::max(h.world, h.vblocks);
    const size_t block = static_cast<size_t>(h.max_blk) * nb;
    ensure_scratch(h, M, P);
    if (h.world > 1) {
        const int g = h.rank;
        MPtrs xs{};
        for (int v = 0; v < M; ++v) xs[v] = h.xs.p + v * block;
        sigma_ring<M>(h, g, P, dx, xs, dy, tm, [&](int s, const Ptrs& held, double* dst, int next) {
            const int cur = (g + s) % P;
            const size_t send_n = (h.blk[cur + 1] - h.blk[cur]) * nb;
            const size_t recv_n = (h.blk[next + 1] - h.blk[next]) * nb;
            h.comm->group_start();
            for (int v = 0; v < M; ++v) {
                h.comm->send(held[v], send_n, (g - 1 + P) % P, h.comm_stream);
                h.comm->recv(dst + v * block, recv_n, (g + 1) % P, h.comm_stream);
            }
            h.comm->group_end();
        });
    } else if (P > 1) {
        // Virtual blocks: every block-rank's schedule runs in turn on this GPU;
        // the ring transport is a device copy out of the whole Cs, which is
        // signed up front (a real rank signs its own block in its prologue).
        const size_t full = h.na() * nb;
        MPtrs xs_all{};
        for (int v = 0; v < M; ++v) xs_all[v] = h.xs.p + v * full;
        eps_prologue<M>(h, dx, xs_all, false, 0, h.na());
        for (int g = 0; g < P; ++g) {
            Ptrs xg{};
            MPtrs yg{}, xsg{};
            for (int v = 0; v < M; ++v) {
                xg[v] = dx[v] + h.blk[g] * nb;
                yg[v] = dy[v] + h.blk[g] * nb;
                xsg[v] = xs_all[v] + h.blk[g] * nb;
            }
            tm.rank_tag = g;
            sigma_ring<M>(h, g, P, xg, xsg, yg, tm, [&](int, const Ptrs&, double* dst, int next) {
                const size_t n = (h.blk[next + 1] - h.blk[next]) * nb;
                for (int v = 0; v < M; ++v)
                    CUDA_CHECK(cudaMemcpyAsync(dst + v * block, xs_all[v] + h.blk[next] * nb, n * sizeof(double),
                                               cudaMemcpyDeviceToDevice, h.comm_stream));
            });
        }
    } else {
        MPtrs xs{};
        for (int v = 0; v < M; ++v) xs[v] = h.xs.p + v * block;
        sigma_ring<M>(h, 0, 1, dx, xs, dy, tm, [](int, const Ptrs&, double*, int) {});
    }
}

void sigma_schedule(Handle& h, const double* dx, double* dy, PhaseTimer& tm) {
    if (h.use_stored) {   // Method::Stored (run.cpp:87-95): CSR SpMV
        const int id = tm.begin(0);
        stored_spmv(h, dx, dy);
        tm.end(id);
        return;
    }
    Ptrs x{};
    MPtrs y{};
    x[0] = dx;
    y[0] = dy;
    sigma_schedule_m<1>(h, x, y, tm);
}

// Pageable host memory (not registered with CUDA): its async copies are
// staged synchronously by the driver and serialise the pipeline.
bool pageable(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
}

// memcpy on the host's cores (the bounce copies through the pinned mirrors)
void host_copy(double* dst, const double* src, size_t n) {
    constexpr size_t kBlock = size_t{1} << 20;   // doubles per task (8 MB)
    const int64_t nb = static_cast<int64_t>((n + kBlock - 1) / kBlock);
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < nb; ++b) {
        const size_t o = static_cast<size_t>(b) * kBlock;
        std::memcpy(dst + o, src + o, std::min(kBlock, n - o) * sizeof(double));
    }
}

// Row chunks of the pipelined host sigma.  Front (H2D under the beta term):
// growing chunks, ratio ~1.4 < (beta time / H2D time) per row, so each chunk
// lands before the previous chunk's beta work ends.  Tail (D2H under the
// alpha term and reduction): shrinking chunks, so only the last, small
// chunk's copy is exposed.
constexpr int kFrontChunks = 9, kTailChunks = 5;
constexpr double kFrontWeight[kFrontChunks] = {1, 1.4, 2, 2.8, 3.9, 5.4, 7.5, 10.5, 14.7};
constexpr double kTailWeight[kTailChunks] = {16, 8, 4, 2, 1};

// Chunk edges (multiples of 128 rows, so the beta term's column chunks and
// the alpha term's row groups have no partial tiles inside the pipe).
template <int N>
std::vector<uint64_t> pipe_edges(uint64_t nloc, const double (&w)[N]) {
    double sum = 0.0;
    for (double x : w) sum += x;
    std::vector<uint64_t> e(N + 1, 0);
    double acc = 0.0;
    for (int c = 1; c < N; ++c) {
        acc += w[c - 1];
        e[c] = std::min<uint64_t>(nloc, static_cast<uint64_t>(nloc * acc / sum + 64) / 128 * 128);
        e[c] = std::max(e[c], e[c - 1]);
    }
    e[N] = nloc;
    return e;
}

// Host-pointer sigma with the host copies overlapped (one block, one vector,
// matrix-free).  x arrives in growing row chunks on the copy stream; as each lands, its eps prologue runs and the beta term
// over its alpha columns (the beta term reads only the x rows of its own
// column chunk).  The scatter kernels then need all of Cs.  Finally, per row
// chunk: the alpha term (y = diag*C + ...), the beta combine, the D
// reduction, and that chunk's D2H on the copy stream under the next chunk's
// kernels.  Returns false (nothing enqueued) when the shape does not allow it.
bool sigma_host_pipelined(Handle& h, const double* x, double* y, detci_gpu_timings* out) {
    if (h.world > 1 || h.vblocks > 1 || h.use_stored || !mixed_scatter_enabled()) return false;
    const uint64_t nloc = h.nloc(), nb = h.nb(), n = nloc * nb;
    if (nloc < 128 * kFrontChunks || nb == 0) return false;
    ensure_scratch(h, 1, 1);
    const SellTable& t = scatter_table(h, 1);
    const auto& wins = scatter_windows(h, 0, 1, 1, t.kmax);
    h.xbuf.alloc(n);
    h.ybuf.alloc(n);
    double* dx = h.xbuf.p;
    double* dy = h.ybuf.p;
    const uint64_t a0 = h.a0;
    // pageable caller buffers: bounce through page-locked mirrors (chunk by
    // chunk on the host's cores, so the DMA and the kernels stay overlapped)
    const bool bounce_x = pageable(x), bounce_y = pageable(y);
    if ((bounce_x || bounce_y) && h.pin_n < n) {
        if (h.pin_x) cudaFreeHost(h.pin_x);
        if (h.pin_y) cudaFreeHost(h.pin_y);
        h.pin_x = h.pin_y = nullptr;
        h.pin_n = 0;
        CUDA_CHECK(cudaMallocHost(&h.pin_x, n * sizeof(double)));
        CUDA_CHECK(cudaMallocHost(&h.pin_y, n * sizeof(double)));
        h.pin_n = n;
    }
    const double* xs_src = bounce_x ? h.pin_x : x;   // the H2D source
    double* yd_dst = bounce_y ? h.pin_y : y;         // the D2H destination
    const std::vector<uint64_t> fe = pipe_edges(nloc, kFrontWeight), te = pipe_edges(nloc, kTailWeight);
    cudaEvent_t ev[kFrontChunks + kTailChunks + 2];
    const bool dbg = std::getenv("DETCI_PIPE_DEBUG") != nullptr;
    for (auto& e : ev) CUDA_CHECK(cudaEventCreateWithFlags(&e, out || dbg ? cudaEventDefault : cudaEventDisableTiming));
    cudaEvent_t* landed = ev;                    // H2D of front chunk c done
    cudaEvent_t* final_rows = ev + kFrontChunks; // y rows of tail chunk c final
    cudaEvent_t t0 = ev[kFrontChunks + kTailChunks], t1 = ev[kFrontChunks + kTailChunks + 1];
    CUDA_CHECK(cudaEventRecord(t0, h.stream));
    CUDA_CHECK(cudaStreamWaitEvent(h.comm_stream, t0, 0));   // previous work on the buffers is done
    auto front_copy = [&](int c) {
        const uint64_t r0 = fe[c], r1 = fe[c + 1];
        if (r1 > r0) {
            if (bounce_x) host_copy(h.pin_x + r0 * nb, x + r0 * nb, (r1 - r0) * nb);
            CUDA_CHECK(cudaMemcpyAsync(dx + r0 * nb, xs_src + r0 * nb, (r1 - r0) * nb * 8, cudaMemcpyHostToDevice,
                                       h.comm_stream));
        }
        CUDA_CHECK(cudaEventRecord(landed[c], h.comm_stream));
    };
    // with page-locked x every chunk's copy is enqueued up front; with a
    // bounce, chunk c is copied on the host while the GPU runs chunk c - 1
    if (!bounce_x)
        for (int c = 0; c < kFrontChunks; ++c) front_copy(c);
    // prologue + beta term per landed chunk
    for (int c = 0; c < kFrontChunks; ++c) {
        const uint64_t r0 = fe[c], r1 = fe[c + 1];
        if (bounce_x) front_copy(c);
        CUDA_CHECK(cudaStreamWaitEvent(h.stream, landed[c], 0));
        if (r1 == r0) continue;
        const uint32_t rc = static_cast<uint32_t>(r1 - r0);
        dim3 tb(kTile, 8), tg(static_cast<unsigned>((nb + kTile - 1) / kTile), (rc + kTile - 1) / kTile);
        k_eps_transpose<<<tg, tb, 0, h.stream>>>(dx + r0 * nb, nb, h.xs.p + r0 * nb, h.ct.p + r0, nloc, rc,
                                                 static_cast<uint32_t>(nb), eps_rows(h, a0 + r0));
        CUDA_LAUNCH_CHECK();
        SameSpinArgs s{};
        s.C[0] = h.ct.p + r0;
        s.Y[0] = h.yt.p + r0;
        s.ldc = nloc;
        s.c_row0 = 0;
        s.j0 = 0;
        s.j1 = static_cast<uint32_t>(nb);
        s.ldy = nloc;
        s.row0 = 0;
        s.nrows = static_cast<uint32_t>(nb);
        s.ncols = rc;
        s.J = h.ch[0].J.p + a0 + r0;
        s.ldj = h.na();
        fill_lists(s, h.ch[1]);
        s.accumulate = 0;
        launch_samespin<1>(s, h.stream);
    }
    cudaEvent_t e_front = nullptr, e_scatter = nullptr;
    if (dbg) {
        CUDA_CHECK(cudaEventCreate(&e_front));
        CUDA_CHECK(cudaEventCreate(&e_scatter));
        CUDA_CHECK(cudaEventRecord(e_front, h.stream));
    }
    // per scatter window: the scatter kernels (D partials of the window's
    // rows), then per row chunk of the window: alpha term, combine, D
    // reduction, D2H.  A window's D2H runs under the next window's scatter;
    // the last window's rows go in shrinking chunks.
    Ptrs held{};
    held[0] = h.xs.p;
    MPtrs yl{};
    yl[0] = dy;
    const int nw = static_cast<int>(wins.size());
    int last_chunk = -1;
    // D2H of each tail chunk into the pinned mirror, then (bounce) the host
    // copies it out once that chunk's event fires
    struct TailCopy {
        uint64_t r0, r1;
        cudaEvent_t done;
    };
    std::vector<TailCopy> tails;
    auto tail_chunk = [&](uint64_t r0, uint64_t r1, bool alpha_combine, int wi) {
        if (r1 == r0) return;
        if (alpha_combine) {
            Ptrs xl{};
            xl[0] = dx + r0 * nb;
            MPtrs yc{};
            yc[0] = dy + r0 * nb;
            launch_alpha<1>(h, held, 0, static_cast<uint32_t>(h.na()), xl, yc, a0 + r0, a0 + r1, true, nw > 1);
            const uint32_t rc = static_cast<uint32_t>(r1 - r0);
            dim3 tb(kTile, 8), tg(static_cast<unsigned>((nb + kTile - 1) / kTile), (rc + kTile - 1) / kTile);
            k_transpose_add_eps<<<tg, tb, 0, h.stream>>>(h.yt.p + r0, nloc, dy + r0 * nb, nb, rc,
                                                         static_cast<uint32_t>(nb), eps_rows(h, a0 + r0));
            CUDA_LAUNCH_CHECK();
        }
        launch_mixed_scatter<1>(h, 0, 1, 0, held, 0, static_cast<uint32_t>(h.na()), yl, a0, 2, a0 + r0, a0 + r1, wi);
        last_chunk = (last_chunk + 1) % kTailChunks;
        cudaEvent_t done = final_rows[last_chunk];
        CUDA_CHECK(cudaEventRecord(done, h.stream));
        CUDA_CHECK(cudaStreamWaitEvent(h.comm_stream, done, 0));
        CUDA_CHECK(cudaMemcpyAsync(yd_dst + r0 * nb, dy + r0 * nb, (r1 - r0) * nb * 8, cudaMemcpyDeviceToHost,
                                   h.comm_stream));
        if (bounce_y) {
            cudaEvent_t e;
            CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CUDA_CHECK(cudaEventRecord(e, h.comm_stream));
            tails.push_back({r0, r1, e});
        }
    };
    const std::vector<uint64_t> edges = pipe_edges(nloc, kTailWeight);
    if (nw == 1) {
        // one window: the scatter, then per row chunk alpha term, combine,
        // reduction and D2H (the chunk's copy runs under the next chunk)
        launch_mixed_scatter<1>(h, 0, 1, 0, held, 0, static_cast<uint32_t>(h.na()), yl, a0, 1, 0, ~0ull, 0);
        if (dbg) CUDA_CHECK(cudaEventRecord(e_scatter, h.stream));
        for (size_t c = 0; c + 1 < edges.size(); ++c) tail_chunk(edges[c], edges[c + 1], true, 0);
    } else {
        // ja windows add into every row: y starts at zero, every window but
        // the last adds its mixed part whole, then per row chunk the alpha
        // term (y += diag*C + alpha), the combine, the last window's
        // reduction and the D2H
        CUDA_CHECK(cudaMemsetAsync(dy, 0, n * sizeof(double), h.stream));
        for (int wi = 0; wi + 1 < nw; ++wi)
            launch_mixed_scatter<1>(h, 0, 1, 0, held, 0, static_cast<uint32_t>(h.na()), yl, a0, 3, 0, ~0ull, wi);
        launch_mixed_scatter<1>(h, 0, 1, 0, held, 0, static_cast<uint32_t>(h.na()), yl, a0, 1, 0, ~0ull, nw - 1);
        if (dbg) CUDA_CHECK(cudaEventRecord(e_scatter, h.stream));
        for (size_t c = 0; c + 1 < edges.size(); ++c) tail_chunk(edges[c], edges[c + 1], true, nw - 1);
    }
    for (auto& tc : tails) {
        CUDA_CHECK(cudaEventSynchronize(tc.done));
        host_copy(y + tc.r0 * nb, h.pin_y + tc.r0 * nb, (tc.r1 - tc.r0) * nb);
        cudaEventDestroy(tc.done);
    }
    CUDA_CHECK(cudaEventRecord(t1, h.comm_stream));
    CUDA_CHECK(cudaEventSynchronize(t1));
    if (dbg) {
        float f = 0.f, sc = 0.f, lastland = 0.f, tail = 0.f, tot = 0.f;
        CUDA_CHECK(cudaEventElapsedTime(&f, t0, e_front));
        CUDA_CHECK(cudaEventElapsedTime(&sc, e_front, e_scatter));
        CUDA_CHECK(cudaEventElapsedTime(&lastland, t0, landed[kFrontChunks - 1]));
        CUDA_CHECK(cudaEventElapsedTime(&tail, e_scatter, final_rows[std::max(last_chunk, 0)]));
        CUDA_CHECK(cudaEventElapsedTime(&tot, t0, t1));
        std::fprintf(stderr, "pipe: front %.2f (H2D done %.2f) scatter %.2f tail %.2f total %.2f ms\n", f, lastland,
                     sc, tail, tot);
        cudaEventDestroy(e_front);
        cudaEventDestroy(e_scatter);
    }
    if (out) {
        float total = 0.f, h2d = 0.f, tail = 0.f;
        CUDA_CHECK(cudaEventElapsedTime(&total, t0, t1));
        CUDA_CHECK(cudaEventElapsedTime(&h2d, t0, landed[kFrontChunks - 1]));
        CUDA_CHECK(cudaEventElapsedTime(&tail, final_rows[std::max(last_chunk, 0)], t1));
        *out = detci_gpu_timings{};
        out->h2d_seconds = h2d * 1e-3;    // overlapped with the beta term
        out->d2h_seconds = tail * 1e-3;   // exposed tail (last chunk)
        out->total_seconds = total * 1e-3;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    return true;
}

} // namespace

bool sigma_host(Handle& h, const double* x, double* y, detci_gpu_timings* tm) {
    if (!h.built) fail(DETCI_GPU_E_INPUT, "sigma: basis not built");
    if (std::getenv("DETCI_SIGMA_PIPELINE") && std::string(std::getenv("DETCI_SIGMA_PIPELINE")) == "0") return false;
    if (tm) return false;   // the phase split needs the plain schedule
    return sigma_host_pipelined(h, x, y, nullptr);
}

void sigma_enqueue(Handle& h, const double* dx, double* dy) {
    if (!h.built) fail(DETCI_GPU_E_INPUT, "sigma: basis not built");
    PhaseTimer tm(h, false);
    sigma_schedule(h, dx, dy, tm);
}

void sigma_block(Handle& h, const double* const* dx, double* const* dy, int m) {
    if (!h.built) fail(DETCI_GPU_E_INPUT, "sigma: basis not built");
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j)
            if (dx[i] == dy[j]) fail(DETCI_GPU_E_INPUT, "sigma: x and y must not alias");
    PhaseTimer tm(h, false);
    if (h.use_stored) {
        for (int i = 0; i < m; ++i) stored_spmv(h, dx[i], dy[i]);
        CUDA_CHECK(cudaStreamSynchronize(h.stream));
        return;
    }
    int i = 0;
    while (i < m) {
        Ptrs x{};
        MPtrs y{};
        // pairs: M = 2 shares the V gathers and SELL stream; M = 4 shrinks
        // the staged row segments 4x and loses (measured 1.35-1.6x slower
        // per vector with the gather kernel), so it is not used
        const int take = m - i >= 2 ? 2 : 1;
        for (int v = 0; v < take; ++v) {
            x[v] = dx[i + v];
            y[v] = dy[i + v];
        }
        if (take == 2) sigma_schedule_m<2>(h, x, y, tm);
        else sigma_schedule_m<1>(h, x, y, tm);
        i += take;
    }
    CUDA_CHECK(cudaStreamSynchronize(h.stream));
}

void sigma_device(Handle& h, const double* dx, double* dy, detci_gpu_timings* out) {
    if (!h.built) fail(DETCI_GPU_E_INPUT, "sigma: basis not built");
    PhaseTimer tm(h, out != nullptr);
    h.timer = out ? &tm : nullptr;
    struct Reset {
        Handle& h;
        ~Reset() { h.timer = nullptr; }
    } reset{h};
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (out) {
        CUDA_CHECK(cudaEventCreate(&t0));
        CUDA_CHECK(cudaEventCreate(&t1));
        CUDA_CHECK(cudaEventRecord(t0, h.stream));
    }
    sigma_schedule(h, dx, dy, tm);
    if (out) {
        CUDA_CHECK(cudaEventRecord(t1, h.stream));
        CUDA_CHECK(cudaEventSynchronize(t1));
        double parts[5];
        tm.collect(parts);
        out->mixed_reduce_seconds = parts[4];
        const int vP = std::max(h.world, h.vblocks) > 1 && h.world == 1 ? h.vblocks : 0;
        h.rank_seconds = tm.per_rank(vP);
        h.rank_phase_seconds = tm.per_rank_phase(vP);
        for (int q = 0; q < 4; ++q) h.own_phase_seconds[q] = parts[q];
        float ms = 0.f;
        CUDA_CHECK(cudaEventElapsedTime(&ms, t0, t1));
        out->alpha_seconds = parts[0];
        out->beta_seconds = parts[1];
        out->mixed_seconds = parts[2];
        out->combine_seconds = parts[3];
        out->total_seconds = ms * 1e-3;
        out->comm_seconds = std::max(0.0, out->total_seconds - parts[0] - parts[1] - parts[2] - parts[3]);
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
    } else {
        CUDA_CHECK(cudaStreamSynchronize(h.stream));
    }
}

} // namespace detci_gpu
