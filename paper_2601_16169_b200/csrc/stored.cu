// Stored-matrix method on the device: build_stored_matrix / stored_matvec
// (matvec.cpp:240-334, matvec.hpp:73-90).
//
// CSR in HBM with the reference's exact row layout, so row_offset and col
// are byte-identical to the reference StoredMatrix and values agree to
// rounding (the elements come from the separated-ordering closed forms of
// formulas.cuh, not hij_words):
//   row I = ia * nb + ib:  [ diagonal (col I)
//                          | alpha singles u doubles of ia, ascending ja
//                          | beta singles u doubles of ib, ascending jb
//                          | alpha singles x beta singles, ja-major, jb ascending ]
// Costs 12 B per nonzero (u32 col + f64 value) + 8 B per row, so it fits only
// small problems (C1: 1.28e9 nonzeros, 15 GB); the matrix-free sigma is the
// production path.  Single GPU only, like the reference's in-process matrix.
//
// Build: one kernel writes every row length, a CUB scan makes row_offset,
// one warp per row fills the row (each lane places its entries by rank: a
// singles entry's position in the merged alpha run is its own index plus the
// number of doubles targets below it).  SpMV: one warp per row, lanes over
// the row's entries, fixed-order warp reduction (deterministic).
#include <cub/cub.cuh>

#include <string>

#include "formulas.cuh"
#include "handle.hpp"

namespace detci_gpu {

namespace {

__global__ void k_stored_rowlen(uint32_t na, uint32_t nb, const uint32_t* __restrict__ lsa,
                                const uint32_t* __restrict__ lda, const uint32_t* __restrict__ lsb,
                                const uint32_t* __restrict__ ldb, uint64_t* __restrict__ rowlen) {
    const uint64_t dim = static_cast<uint64_t>(na) * nb;
    for (uint64_t I = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; I < dim;
         I += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t ia = static_cast<uint32_t>(I / nb), ib = static_cast<uint32_t>(I % nb);
        rowlen[I] = 1ull + lsa[ia] + lda[ia] + lsb[ib] + ldb[ib] + static_cast<uint64_t>(lsa[ia]) * lsb[ib];
    }
}

__device__ __forceinline__ uint32_t count_below(const uint32_t* a, uint32_t n, uint32_t key) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

struct StoredFillArgs {
    uint32_t na, nb;
    int norbs;
    const uint64_t* sa;   // alpha strings
    const uint64_t* sb;   // beta strings
    const uint64_t* pb;   // prefix parities of the beta strings (eps)
    const uint64_t* sa_hi;   // norbs > 64: high words (else null)
    const uint64_t* sb_hi;
    const uint64_t* pb_hi;
    // [channel][kind] helper lists and same-spin pair tables
    const uint32_t* flat[2][2];
    const uint64_t* off[2][2];
    const uint32_t* len[2][2];
    const double* pv[2][2];
    const uint32_t* pab[2];
    const double* J[2];   // J[c][tri * n_c + i]: channel c as spectator
    const double* eri;
    const double* diag;
    const uint64_t* row_offset;
    uint32_t* col;
    double* value;
};

__device__ __forceinline__ int eps_of(Bits a, Bits pb) { return eps_parity(a, pb); }

// One warp per row (grid-strided over rows).
__global__ void __launch_bounds__(256) k_stored_fill(const StoredFillArgs a) {
    const uint64_t dim = static_cast<uint64_t>(a.na) * a.nb;
    const uint32_t lane = threadIdx.x % kWarp;
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x / kWarp);
    const int n = a.norbs;
    for (uint64_t I = blockIdx.x * static_cast<uint64_t>(blockDim.x / kWarp) + threadIdx.x / kWarp; I < dim;
         I += warps) {
        const uint32_t ia = static_cast<uint32_t>(I / a.nb), ib = static_cast<uint32_t>(I % a.nb);
        const Bits A = load_bits(a.sa, a.sa_hi, ia), B = load_bits(a.sb, a.sb_hi, ib),
                   PB = load_bits(a.pb, a.pb_hi, ib);
        const int eI = eps_of(A, PB);
        uint64_t at = a.row_offset[I];
        if (lane == 0) {
            a.col[at] = static_cast<uint32_t>(I);
            a.value[at] = a.diag[I];
        }
        ++at;
        // alpha same-spin: spectator B, J of the beta channel
        {
            const uint32_t* fs = a.flat[0][0] + a.off[0][0][ia];
            const uint32_t* fd = a.flat[0][1] + a.off[0][1][ia];
            const uint32_t ns = a.len[0][0][ia], nd = a.len[0][1][ia];
            for (uint32_t k = lane; k < ns + nd; k += kWarp) {
                const bool single = k < ns;
                const uint32_t kk = single ? k : k - ns;
                const uint32_t ja = single ? fs[kk] : fd[kk];
                const uint32_t pos = kk + (single ? count_below(fd, nd, ja) : count_below(fs, ns, ja));
                const uint64_t e = (single ? a.off[0][0][ia] : a.off[0][1][ia]) + kk;
                double v = a.pv[0][single ? 0 : 1][e];
                if (single) {
                    const uint32_t ab = a.pab[0][e];
                    const double j = a.J[1][static_cast<size_t>(ab & 0x7fffffffu) * a.nb + ib];
                    v += (ab >> 31) ? -j : j;
                }
                const int s = eI ^ eps_of(load_bits(a.sa, a.sa_hi, ja), PB);
                a.col[at + pos] = static_cast<uint32_t>(static_cast<uint64_t>(ja) * a.nb + ib);
                a.value[at + pos] = s ? -v : v;
            }
            at += ns + nd;
        }
        // beta same-spin: spectator A, J of the alpha channel
        {
            const uint32_t* fs = a.flat[1][0] + a.off[1][0][ib];
            const uint32_t* fd = a.flat[1][1] + a.off[1][1][ib];
            const uint32_t ns = a.len[1][0][ib], nd = a.len[1][1][ib];
            for (uint32_t k = lane; k < ns + nd; k += kWarp) {
                const bool single = k < ns;
                const uint32_t kk = single ? k : k - ns;
                const uint32_t jb = single ? fs[kk] : fd[kk];
                const uint32_t pos = kk + (single ? count_below(fd, nd, jb) : count_below(fs, ns, jb));
                const uint64_t e = (single ? a.off[1][0][ib] : a.off[1][1][ib]) + kk;
                double v = a.pv[1][single ? 0 : 1][e];
                if (single) {
                    const uint32_t ab = a.pab[1][e];
                    const double j = a.J[0][static_cast<size_t>(ab & 0x7fffffffu) * a.na + ia];
                    v += (ab >> 31) ? -j : j;
                }
                const int s = eI ^ eps_of(A, load_bits(a.pb, a.pb_hi, jb));
                a.col[at + pos] = static_cast<uint32_t>(static_cast<uint64_t>(ia) * a.nb + jb);
                a.value[at + pos] = s ? -v : v;
            }
            at += ns + nd;
        }
        // mixed: alpha singles x beta singles
        {
            const uint32_t* fa = a.flat[0][0] + a.off[0][0][ia];
            const uint32_t* fb = a.flat[1][0] + a.off[1][0][ib];
            const uint32_t nsa = a.len[0][0][ia], nsb = a.len[1][0][ib];
            for (uint32_t t = lane; t < nsa * nsb; t += kWarp) {
                const uint32_t ka = t / nsb, kb = t - ka * nsb;
                const uint32_t ja = fa[ka], jb = fb[kb];
                const Bits Aj = load_bits(a.sa, a.sa_hi, ja);
                const int pa = lowest(A & ~Aj), qa = lowest(Aj & ~A);
                const MixedMove mv = mixed_move(B, load_bits(a.sb, a.sb_hi, jb), n);
                const int c = static_cast<int>(mv.cd) / n, d = static_cast<int>(mv.cd) % n;
                const double v = mixed_weight(a.eri, n, pa, qa, c, d);
                const int s = static_cast<int>(mv.sbit) ^ mixed_alpha_parity(A, pa, qa) ^ eI ^ eps_of(Aj, load_bits(a.pb, a.pb_hi, jb));
                a.col[at + t] = static_cast<uint32_t>(static_cast<uint64_t>(ja) * a.nb + jb);
                a.value[at + t] = s ? -v : v;
            }
        }
    }
}

// y[I] = sum_at value[at] * x[col[at]], one warp per row.
__global__ void __launch_bounds__(256)
k_stored_spmv(const uint64_t* __restrict__ row_offset, const uint32_t* __restrict__ col,
              const double* __restrict__ value, const double* __restrict__ x, double* __restrict__ y,
              uint64_t dim) {
    const uint32_t lane = threadIdx.x % kWarp;
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x / kWarp);
    for (uint64_t I = blockIdx.x * static_cast<uint64_t>(blockDim.x / kWarp) + threadIdx.x / kWarp; I < dim;
         I += warps) {
        const uint64_t b = row_offset[I], e = row_offset[I + 1];
        double acc = 0.0;
        for (uint64_t at = b + lane; at < e; at += kWarp) acc = fma(__ldcs(value + at), x[__ldcs(col + at)], acc);
        for (int s = 16; s > 0; s >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, s);
        if (lane == 0) y[I] = acc;
    }
}

} // namespace

void build_stored(Handle& h, uint64_t budget, uint64_t* nnz_out) {
    if (!h.built) fail(DETCI_GPU_E_INPUT, "build_stored_matrix: basis not built");
    if (h.world > 1 || h.vblocks > 1)
        fail(DETCI_GPU_E_UNSUPPORTED, "build_stored_matrix: single GPU only");
    const uint64_t na = h.na(), nb = h.nb(), dim = na * nb;
    if (dim > 0xffffffffull)  // matvec.cpp:245-246
        fail(DETCI_GPU_E_CAPACITY, "stored matrix: dimension exceeds 32-bit column indexing");
    release_stored(h);
    DevBuf<uint64_t> rowlen;
    rowlen.alloc(dim);
    h.st_off.alloc(dim + 1);
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((dim + 255) / 256, 148 * 16));
    k_stored_rowlen<<<grid, 256, 0, h.stream>>>(static_cast<uint32_t>(na), static_cast<uint32_t>(nb),
                                                h.ch[0].len[0].p, h.ch[0].len[1].p, h.ch[1].len[0].p,
                                                h.ch[1].len[1].p, rowlen.p);
    CUDA_LAUNCH_CHECK();
    CUDA_CHECK(cudaMemsetAsync(h.st_off.p, 0, sizeof(uint64_t), h.stream));
    size_t tmp_bytes = 0;
    CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, rowlen.p, h.st_off.p + 1, dim, h.stream));
    DevBuf<unsigned char> tmp;
    tmp.alloc(std::max<size_t>(tmp_bytes, 1));
    CUDA_CHECK(cub::DeviceScan::InclusiveSum(tmp.p, tmp_bytes, rowlen.p, h.st_off.p + 1, dim, h.stream));
    uint64_t nnz = 0;
    CUDA_CHECK(cudaMemcpyAsync(&nnz, h.st_off.p + dim, sizeof(uint64_t), cudaMemcpyDeviceToHost, h.stream));
    CUDA_CHECK(cudaStreamSynchronize(h.stream));
    rowlen.reset();
    tmp.reset();
    // matvec.cpp:262-269 convention and message
    const uint64_t required = nnz * (sizeof(double) + sizeof(uint32_t)) + (dim + 1) * sizeof(uint64_t);
    size_t free_b = 0, total_b = 0;
    CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
    const uint64_t cap = budget ? budget : static_cast<uint64_t>(free_b);
    if (required > cap || nnz * 12 > free_b) {
        h.st_off.reset();
        fail(DETCI_GPU_E_CAPACITY, "stored matrix requires " + std::to_string(required) + " bytes, budget is " +
                                       std::to_string(std::min<uint64_t>(cap, free_b)) + " bytes");
    }
    h.st_col.alloc(std::max<uint64_t>(nnz, 1));
    h.st_val.alloc(std::max<uint64_t>(nnz, 1));
    StoredFillArgs a{};
    a.na = static_cast<uint32_t>(na);
    a.nb = static_cast<uint32_t>(nb);
    a.norbs = h.norbs;
    a.sa = h.ch[0].strings.p;
    a.sb = h.ch[1].strings.p;
    a.pb = h.ch[1].prefix.p;
    a.sa_hi = h.ch[0].hi();
    a.sb_hi = h.ch[1].hi();
    a.pb_hi = h.ch[1].prefix_hi_p();
    for (int c = 0; c < 2; ++c) {
        for (int k = 0; k < 2; ++k) {
            a.flat[c][k] = h.ch[c].flat[k].p;
            a.off[c][k] = h.ch[c].offset[k].p;
            a.len[c][k] = h.ch[c].len[k].p;
            a.pv[c][k] = h.ch[c].pv[k].p;
        }
        a.pab[c] = h.ch[c].pab.p;
        a.J[c] = h.ch[c].J.p;
    }
    a.eri = h.d_eri.p;
    a.diag = h.diag.p;
    a.row_offset = h.st_off.p;
    a.col = h.st_col.p;
    a.value = h.st_val.p;
    k_stored_fill<<<148 * 8, 256, 0, h.stream>>>(a);
    CUDA_LAUNCH_CHECK();
    CUDA_CHECK(cudaStreamSynchronize(h.stream));
    h.st_nnz = nnz;
    if (nnz_out) *nnz_out = nnz;
}

void release_stored(Handle& h) {
    h.st_off.reset();
    h.st_col.reset();
    h.st_val.reset();
    h.st_nnz = 0;
    h.use_stored = false;
}

void stored_spmv(Handle& h, const double* dx, double* dy) {
    if (!h.st_off.p) fail(DETCI_GPU_E_INPUT, "stored_matvec: matrix not built");
    const uint64_t dim = h.na() * h.nb();
    k_stored_spmv<<<148 * 16, 256, 0, h.stream>>>(h.st_off.p, h.st_col.p, h.st_val.p, dx, dy, dim);
    CUDA_LAUNCH_CHECK();
}

} // namespace detci_gpu
