// Internal state of a detci_gpu_handle: the device-resident basis.
//
// HBM layout: per channel the uint64 string table
// and its prefix parities, the four helper lists exactly as
// FlatExcitationTable (flat u32, offset u64, len u32;
// connectivity.hpp:24-33), a same-spin pair table parallel to each list
// (separated-ordering value f64, J index u32), a spectator J table
// J[tri(p,q)][string] = sum_{r in string} (pq|rr), the beta-singles SELL-32
// table for the mixed term, this rank's diagonal and the C/sigma scratch.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "../../include/detci_gpu.h"
#include "comm.hpp"
#include "common.cuh"

namespace detci_gpu {

// Scatter formulation of the mixed term (sigma.cu k_mixed_scatter): largest
// number of output alpha rows per pass (kmax is one of 16, 8, 4, 2, 1),
// shared-memory budget, V-table row pitch (doubles).
constexpr int kScatterKMax = 16;
constexpr int kScatterClasses = 5;   // possible kmax values (item lists cached per kmax)
constexpr uint32_t kScatterSmem = 222u * 1024;   // dynamic; + 4.3 KB static row tables <= 227 KB
// V rows of the scatter kernel are rows of the pair-ERI matrix
// PE[tri(pa,qa)][tri(pb,qb)] = (pa qa|pb qb) (8-fold symmetry: one value per
// unordered beta move), pitch even so every row is 16-byte aligned.
inline uint32_t pair_count(int n) { return static_cast<uint32_t>(n * (n - 1) / 2); }
inline uint32_t scatter_vpitch(int n) { return std::max<uint32_t>(2, (pair_count(n) + 1) & ~1u); }
// Staged Cs row segment of seg_cols doubles: one double of alignment shift
// (the bulk copy needs source and destination congruent mod 16 bytes) and
// the zero slot the padding entries read, rounded to an even pitch.
__host__ __device__ inline uint32_t scatter_segpad(uint32_t seg_cols) { return (seg_cols + 3) & ~1u; }
// DETCI_MIXED=gather selects the gather kernel (k_mixed) for M = 1.
inline bool mixed_scatter_enabled() {
    const char* e = std::getenv("DETCI_MIXED");
    return !(e && std::string(e) == "gather");
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { reset(); }
    void reset() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t count) {
        if (count == n && p) return;
        reset();
        if (count == 0) return;
        CUDA_CHECK(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    size_t bytes() const { return n * sizeof(T); }
};

struct PhaseTimer;   // sigma_internal.hpp

struct ChannelTables {
    size_t n = 0;                      // strings in this channel (global)
    int n_elec = 0;
    std::vector<uint64_t> h_strings;
    DevBuf<uint64_t> strings;
    DevBuf<uint64_t> prefix;           // prefix_parity(strings[i]) (eps sign)
    // norbs > 64: orbitals 64..127 of each string and of its prefix parity
    // (empty otherwise; kernels read them through load_bits)
    std::vector<uint64_t> h_strings_hi;
    DevBuf<uint64_t> strings_hi;
    DevBuf<uint64_t> prefix_hi;
    const uint64_t* hi() const { return strings_hi.p; }
    const uint64_t* prefix_hi_p() const { return prefix_hi.p; }
    // kind 0 = singles, 1 = doubles
    DevBuf<uint32_t> flat[2];
    DevBuf<uint64_t> offset[2];
    DevBuf<uint32_t> len[2];
    uint64_t nflat[2] = {0, 0};
    std::vector<uint32_t> h_len[2];
    // same-spin pair tables (this channel moves, the other is spectator)
    DevBuf<double> pv[2];
    DevBuf<uint32_t> pab;              // singles: tri(p,q) | sign << 31
    // this channel as spectator: J[tri * n + i]
    DevBuf<double> J;
};

struct SellTable {
    DevBuf<uint32_t> sell;
    DevBuf<uint64_t> off;              // [slice * nseg + seg]
    DevBuf<uint32_t> len;              // [slice * nseg + seg]
    uint32_t seg_cols = 0, nseg = 0;
    bool double_buffer = true;         // C stages double-buffered (else one)
    int format = 1;                    // 1 gather (k_mixed), 2 scatter (k_mixed_scatter)
    int kmax = 0;                      // format 2: largest K class (16 or 8)
    bool built = false;
};

// One output window of the scatter mixed term: alpha rows [i_lo, i_hi) of
// this rank, whose D rows (one per (ia, position of ja in ia's singles list))
// are sa_off[ia] - d_base; per alpha block b the CTA items (ja, kbeg | len <<
// 20): the run of ja's singles list whose outputs ia_k lie in the window (the
// CTA cuts it into passes of kmax rows and one padded remainder pass).
struct ScatterWindow {
    uint64_t i_lo = 0, i_hi = 0, d_base = 0, d_rows = 0;
    // Single-block plans cut the work by ja instead (items stay whole): the
    // window holds ja in [j0, j1) for all output rows, and its D is
    // compacted per row: D row of (ia, pos) = base[ia] + pos - lo[ia], where
    // [lo[ia], lo[ia] + base[ia+1] - base[ia]) are the positions of the
    // window's ja in ia's list.  (No arrays when one window covers all ja.)
    bool by_ja = false;
    uint64_t j0 = 0, j1 = 0;
    DevBuf<uint32_t> lo;
    DevBuf<uint64_t> base;
    DevBuf<uint2> items[kScatterClasses];            // by log2(kmax) (built on demand)
    std::vector<uint64_t> item_off[kScatterClasses]; // per alpha block, size P + 1
};

struct Handle {
    int device = 0;
    int rank = 0;
    int world = 1;
    int vblocks = 1;   // virtual alpha blocks on one GPU (tests the ring schedule)
    int weighted = 0;
    uint64_t budget = 0;
    std::string err;

    int norbs = 0;
    bool have_strings = false, have_ints = false, built = false;
    double core = 0.0;
    std::vector<double> h1, eri;
    DevBuf<double> d_h1, d_eri;
    DevBuf<double> d_pair;             // pair-ERI matrix (scatter_vpitch rows), scatter V rows

    ChannelTables ch[2];

    // mixed term: beta singles in SELL-32, bucketed by jb segment; one
    // segmentation per vector count M in {1, 2, 4} (the staged C rows of M
    // vectors share the CTA's shared memory), built on first use
    SellTable sell_m[3];
    SellTable sell_scatter[2];         // format 2, M = 1, 2
    DevBuf<uint32_t> sell_perm;        // slot -> beta string (degree-sorted)
    std::vector<uint64_t> slice_prefix;   // prefix of the scatter work per 32-slot slice (mixed_slots)
    // scatter mixed term: tpos[sa_off[ja] + k] = position of ja in the
    // singles list of its k-th single ia; host copies of the alpha singles;
    // windows per block-rank g (built on first use, dropped with dbuf)
    DevBuf<uint32_t> tpos;
    std::vector<uint32_t> h_sa_flat;
    std::vector<uint64_t> h_sa_off;
    std::vector<std::vector<std::unique_ptr<ScatterWindow>>> scatter_plan;
    DevBuf<double> dbuf;               // D partials of the current window
    uint64_t dcap_rows = 0;            // D rows per vector that fit (set with the plan)
    int dplan_m = 0;                   // vectors per pass the plan reserved D for
    uint32_t nslices = 0;

    // alpha-block partition: P = world (NCCL) or vblocks (virtual)
    std::vector<uint64_t> blk;
    std::vector<uint32_t> slot_cut;   // measured mixed column shares (rebalance_partition), else empty
    uint64_t a0 = 0, a1 = 0;           // this rank's rows
    uint64_t max_blk = 0;

    DevBuf<double> diag;               // (a1 - a0) * nb

    // sigma scratch
    DevBuf<double> ct, yt;             // nb * max_blk
    DevBuf<double> xs;                 // eps o C of the local block (ring payload)
    DevBuf<double> cs_full;            // gather schedule (P > 1): the whole Cs
    DevBuf<double> mix_t, mix_r;       // gather schedule: own / received mixed slabs
    DevBuf<double> ring[2];            // max_blk * nb
    DevBuf<double> xbuf, ybuf;         // host-pointer staging, local length
    // page-locked mirrors of x and y for callers that hand pageable memory
    // (detci_gpu_sigma bounces through them so the copies stay overlapped)
    double* pin_x = nullptr;
    double* pin_y = nullptr;
    size_t pin_n = 0;
    DevBuf<double> red;                // reduction partials
    DevBuf<double> dav_store;          // Davidson subspace, cached across solves
    DevBuf<unsigned int> red_count;

    // stored-matrix method (stored.cu): CSR of H, used by every sigma call
    // while use_stored is set (detci_gpu_set_operator)
    DevBuf<uint64_t> st_off;
    DevBuf<uint32_t> st_col;
    DevBuf<double> st_val;
    uint64_t st_nnz = 0;
    bool use_stored = false;

    PhaseTimer* timer = nullptr;       // set while a timed sigma runs
    std::vector<double> rank_seconds;  // virtual blocks: device seconds per block-rank, last timed sigma
    std::vector<double> rank_phase_seconds;   // the same per (rank, phase alpha/beta/mixed/combine)
    double own_phase_seconds[4] = {};         // world > 1: this rank's phases, last timed sigma
    cudaStream_t stream = nullptr, comm_stream = nullptr;
    cudaEvent_t ev[16] = {};
    std::unique_ptr<Comm> comm;        // world > 1: NCCL or loopback (comm.hpp)
    DevBuf<double> red_host;           // allreduce_sum staging (grown to the count)

    uint64_t nnz_alpha = 0, nnz_beta = 0, nnz_mixed = 0;

    size_t na() const { return ch[0].n; }
    size_t nb() const { return ch[1].n; }
    uint64_t nloc() const { return a1 - a0; }
    size_t local_len() const { return static_cast<size_t>(a1 - a0) * nb(); }
};

// basis.cu
void plan_partition(uint64_t na, uint64_t nb, const uint32_t* sa, const uint32_t* da,
                    const uint32_t* sb, const uint32_t* db, int P, int weighted, uint64_t* blk);
void build_device_basis(Handle& h);
const SellTable& mixed_table(Handle& h, int M);   // M in {1, 2, 4}
const SellTable& scatter_table(Handle& h, int M);   // M in {1, 2}
void release_basis(Handle& h);
void build_scatter_tpos(Handle& h);
// Drop the scatter D buffer and windows (re-planned against the free memory
// at the next sigma); the Davidson solvers call it before allocating.
void release_sigma_scratch(Handle& h);
void rebalance_partition(Handle& h, const std::vector<double>& t);

// sigma.cu
void sigma_device(Handle& h, const double* dx, double* dy, detci_gpu_timings* tm);
void sigma_enqueue(Handle& h, const double* dx, double* dy);  // no host sync
// y = H x on host buffers with the copies overlapped (chunked H2D under the
// beta term, chunked D2H under the alpha term / reduction); false when the
// shape needs the plain copy-sigma-copy schedule.  Synchronous.
bool sigma_host(Handle& h, const double* x, double* y, detci_gpu_timings* tm);
// m vectors through one blocked pass (element evaluations shared across
// vectors where the kernels support it); synchronous.
void sigma_block(Handle& h, const double* const* dx, double* const* dy, int m);

// stored.cu
void build_stored(Handle& h, uint64_t budget, uint64_t* nnz);
void release_stored(Handle& h);
void stored_spmv(Handle& h, const double* dx, double* dy);   // enqueued on h.stream

// davidson.cu
struct DavidsonOutcome {
    int status = 0, iterations = 0;
    double energy = 0.0, seconds = 0.0;
};
void davidson_device(Handle& h, const detci_dav_opts& opts, detci_dav_result* res,
                     detci_trace_cb cb, void* user);
double device_dot(Handle& h, const double* x, const double* y, uint64_t n);
void device_dot_many(Handle& h, const double* x, const double* const* ys, int k, uint64_t n,
                     double* out_host);
void allreduce_sum(Handle& h, double* host_vals, int count);
// Collective agreement: true when every rank passes ok (world 1: ok).  Used
// before committing to work that one rank alone could refuse (capacity), so
// no rank is left waiting in a collective its peer never enters.
bool all_ranks_ok(Handle& h, bool ok);
// Every rank fails when any rank fails `ok`: the failing rank with its own
// (code, msg), the others with E_ERROR "<what>: another rank failed".
void collective_require(Handle& h, bool ok, int code, const std::string& msg, const char* what);
double smallest_eigenpair(const std::vector<double>& lower, int ld, int k, std::vector<double>& vec);
void jacobi_eigen(const std::vector<double>& lower, int ld, int k, std::vector<double>& evals,
                  std::vector<double>& vecs);
void davidson_roots_device(Handle& h, const detci_dav_block_opts& opts, detci_dav_block_result* res);

// Strings of the eps sign eps(A_r, B_c) for local rows from `row` on: alpha
// strings and beta prefix parities, high words null for norbs <= 64.
struct EpsRows {
    const uint64_t* a;
    const uint64_t* a_hi;
    const uint64_t* b;
    const uint64_t* b_hi;
};
inline EpsRows eps_rows(const Handle& h, uint64_t row) {
    return EpsRows{h.ch[0].strings.p + row, h.ch[0].hi() ? h.ch[0].hi() + row : nullptr, h.ch[1].prefix.p,
                   h.ch[1].prefix_hi_p()};
}

} // namespace detci_gpu
