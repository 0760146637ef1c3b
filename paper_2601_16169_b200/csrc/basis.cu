// Device basis construction: helper lists, pair tables, J tables, the mixed
// SELL table, the diagonal and the alpha-block partition (build_basis,
// basis.cpp:78-148; generate_singles/doubles, connectivity.cpp:64-122).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <string>
#include <vector>

#include "formulas.cuh"
#include "handle.hpp"
#include "sigma_internal.hpp"

namespace detci_gpu {

// alpha-block boundaries: reference formula na*g/P (matvec.cpp:108-111) or
// balanced by each row's element count.
void plan_partition(uint64_t na, uint64_t nb, const uint32_t* sa, const uint32_t* da,
                    const uint32_t* sb, const uint32_t* db, int P, int weighted, uint64_t* blk) {
    if (P < 1) fail(DETCI_GPU_E_INPUT, "partition: P must be positive");
    if (static_cast<uint64_t>(P) > na)
        fail(DETCI_GPU_E_INPUT, "partition: " + std::to_string(P) + " alpha blocks exceed n_alpha " +
                                    std::to_string(na));
    if (!weighted || P == 1) {
        for (int g = 0; g <= P; ++g) blk[g] = na * static_cast<uint64_t>(g) / P;
        return;
    }
    uint64_t sum_sb = 0, sum_db = 0;
    for (uint64_t i = 0; i < nb; ++i) {
        sum_sb += sb[i];
        sum_db += db[i];
    }
    std::vector<double> prefix(na + 1, 0.0);
    for (uint64_t i = 0; i < na; ++i)
        prefix[i + 1] = prefix[i] + static_cast<double>(sa[i] + da[i]) * nb +
                        static_cast<double>(sum_sb + sum_db) +
                        (weighted == 2 ? 0.0 : static_cast<double>(sa[i]) * sum_sb);
    blk[0] = 0;
    blk[P] = na;
    for (int g = 1; g < P; ++g) {
        const double target = prefix[na] * g / P;
        uint64_t cut = std::lower_bound(prefix.begin(), prefix.end(), target) - prefix.begin();
        cut = std::max<uint64_t>(cut, blk[g - 1] + 1);
        cut = std::min<uint64_t>(cut, na - (P - g));
        blk[g] = cut;
    }
}

namespace {

constexpr int kPairTile = 2048;   // strings staged in smem per pass (16 KB)
constexpr int kPairBlock = 512;   // 16 warps = 16 source rows per CTA

// Helper lists by pairwise comparison.  For source row i every string j is
// tested with popc(s_i ^ s_j): 2 = one electron moved (singles), 4 = two
// (doubles) -- equivalent to the reference's move probing because every
// string of a channel has the same electron count (basis.cpp:39-44).  Rows
// come out ascending by construction: a warp tests 32 consecutive j, and a
// ballot + prefix popcount compacts the hits in order.  Pass 1 counts,
// pass 2 fills at the scanned offsets.
// kWide: norbs > 64, the high words of the strings in `shi`.
template <bool kFill, bool kWide>
__global__ void __launch_bounds__(kPairBlock)
k_pair_scan(const uint64_t* __restrict__ s, const uint64_t* __restrict__ shi, uint32_t n, uint32_t* __restrict__ len_s,
            uint32_t* __restrict__ len_d, const uint64_t* __restrict__ off_s,
            const uint64_t* __restrict__ off_d, uint32_t* __restrict__ flat_s,
            uint32_t* __restrict__ flat_d, unsigned int* __restrict__ dup_index) {
    __shared__ uint64_t tile[kWide ? 2 : 1][kPairTile];
    const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    const uint32_t i = blockIdx.x * (kPairBlock / kWarp) + warp;
    const uint64_t si = i < n ? s[i] : 0ull;
    const uint64_t si_hi = kWide && i < n ? shi[i] : 0ull;
    const unsigned lt_mask = (1u << lane) - 1u;
    uint32_t cs = 0, cd = 0;
    uint64_t base_s = 0, base_d = 0;
    if (kFill && i < n) {
        base_s = off_s[i];
        base_d = off_d[i];
    }
    for (uint32_t t0 = 0; t0 < n; t0 += kPairTile) {
        const uint32_t tn = min(static_cast<uint32_t>(kPairTile), n - t0);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < tn; k += kPairBlock) {
            tile[0][k] = s[t0 + k];
            if (kWide) tile[kWide ? 1 : 0][k] = shi[t0 + k];
        }
        __syncthreads();
        if (i >= n) continue;
        for (uint32_t k = 0; k < tn; k += kWarp) {
            const uint32_t kk = k + lane;
            const int d = kk < tn ? __popcll(si ^ tile[0][kk]) + (kWide ? __popcll(si_hi ^ tile[kWide ? 1 : 0][kk]) : 0)
                                  : -1;
            const unsigned bs = __ballot_sync(0xffffffffu, d == 2);
            const unsigned bd = __ballot_sync(0xffffffffu, d == 4);
            if (kFill) {
                if (d == 2) flat_s[base_s + cs + __popc(bs & lt_mask)] = t0 + kk;
                if (d == 4) flat_d[base_d + cd + __popc(bd & lt_mask)] = t0 + kk;
            } else {
                const unsigned b0 = __ballot_sync(0xffffffffu, d == 0 && t0 + kk != i);
                if (b0 && lane == 0) {
                    const uint32_t j = t0 + k + static_cast<uint32_t>(__ffs(b0) - 1);
                    atomicMin(dup_index, max(i, j));
                }
            }
            cs += __popc(bs);
            cd += __popc(bd);
        }
    }
    if (!kFill && i < n && lane == 0) {
        len_s[i] = cs;
        len_d[i] = cd;
    }
}

// Exclusive scan of u32 counts into u64 offsets (FlatExcitationTable::offset
// has size n, connectivity.cpp:41-54); one CTA, total in out[n].
__global__ void __launch_bounds__(1024)
k_scan_offsets(const uint32_t* __restrict__ len, uint64_t* __restrict__ off, uint32_t n) {
    __shared__ uint64_t sums[1024];
    const uint32_t t = threadIdx.x;
    const uint32_t chunk = (n + 1023) / 1024;
    const uint32_t b = min(n, t * chunk), e = min(n, b + chunk);
    uint64_t local = 0;
    for (uint32_t i = b; i < e; ++i) local += len[i];
    sums[t] = local;
    __syncthreads();
    for (int stride = 1; stride < 1024; stride <<= 1) {
        const uint64_t v = t >= static_cast<uint32_t>(stride) ? sums[t - stride] : 0;
        __syncthreads();
        sums[t] += v;
        __syncthreads();
    }
    uint64_t run = sums[t] - local;
    for (uint32_t i = b; i < e; ++i) {
        off[i] = run;
        run += len[i];
    }
    if (t == 1023) off[n] = sums[1023];
}

// Transpose positions of the alpha singles lists (scatter mixed term):
// tpos[off[ja] + k] = index of ja in the list of ia = flat[off[ja] + k]
// (singles are mutual, so it exists).
__global__ void k_tpos(const uint32_t* __restrict__ flat, const uint64_t* __restrict__ off,
                       const uint32_t* __restrict__ len, uint32_t n, uint32_t* __restrict__ tpos) {
    const uint32_t ja = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    const int lane = threadIdx.x % kWarp;
    if (ja >= n) return;
    const uint64_t o = off[ja];
    for (uint32_t k = lane; k < len[ja]; k += kWarp) {
        const uint32_t ia = flat[o + k];
        const uint32_t* f = flat + off[ia];
        uint32_t lo = 0, hi = len[ia];
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (f[mid] < ja) lo = mid + 1;
            else hi = mid;
        }
        tpos[o + k] = lo;
    }
}

// Same-spin pair tables, one warp per source row, lanes over entries.
__global__ void k_pair_tables(int kind, const uint64_t* __restrict__ s, const uint64_t* __restrict__ shi, uint32_t n,
                              const uint32_t* __restrict__ flat, const uint64_t* __restrict__ off,
                              const uint32_t* __restrict__ len, const double* __restrict__ h1,
                              const double* __restrict__ eri, int norbs, double* __restrict__ pv,
                              uint32_t* __restrict__ pab) {
    const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    const int lane = threadIdx.x % kWarp;
    if (i >= n) return;
    const Bits si = load_bits(s, shi, i);
    const uint64_t o = off[i];
    for (uint32_t k = lane; k < len[i]; k += kWarp) {
        const PairEntry e = make_pair_entry(kind, si, load_bits(s, shi, flat[o + k]), h1, eri, norbs);
        pv[o + k] = e.v;
        if (kind == 0) pab[o + k] = e.ab_sign;
    }
}

// J[t * n + i] = sum_{r in s_i} (p q | r r), t = tri(p, q), p > q.
__global__ void k_jtable(const uint64_t* __restrict__ s, const uint64_t* __restrict__ shi, uint32_t n,
                         const double* __restrict__ eri, int norbs, double* __restrict__ J) {
    const uint32_t t = blockIdx.y;
    int p = 1;
    while ((p + 1) * p / 2 <= static_cast<int>(t)) ++p;
    const int q = static_cast<int>(t) - p * (p - 1) / 2;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        Bits bits = load_bits(s, shi, i);
        double acc = 0.0;
        while (any(bits)) {
            const int r = lowest(bits);
            bits = drop_lowest(bits);
            acc += eri_at(eri, norbs, p, q, r, r);
        }
        J[static_cast<size_t>(t) * n + i] = acc;
    }
}

// Diagonal pieces: E[i] = sum_{p in s} h_pp + sum_{p<q in s} [(pp|qq) - (pq|qp)].
__global__ void k_string_energy(const uint64_t* __restrict__ s, const uint64_t* __restrict__ shi, uint32_t n,
                                const double* __restrict__ h1, const double* __restrict__ eri,
                                int norbs, double* __restrict__ E) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Bits a = load_bits(s, shi, i);
    double acc = 0.0;
    while (any(a)) {
        const int p = lowest(a);
        a = drop_lowest(a);
        acc += h1[p * norbs + p];
        Bits b = a;
        while (any(b)) {
            const int q = lowest(b);
            b = drop_lowest(b);
            acc += eri_at(eri, norbs, p, p, q, q) - eri_at(eri, norbs, p, q, q, p);
        }
    }
    E[i] = acc;
}

// U[p * nb + ib] = sum_{q in B_ib} (pp|qq): the opposite-spin Coulomb part.
__global__ void k_u_table(const uint64_t* __restrict__ sb, const uint64_t* __restrict__ sbhi, uint32_t nb,
                          const double* __restrict__ eri, int norbs, double* __restrict__ U) {
    const uint32_t ib = blockIdx.x * blockDim.x + threadIdx.x;
    const int p = blockIdx.y;
    if (ib >= nb) return;
    Bits b = load_bits(sb, sbhi, ib);
    double acc = 0.0;
    while (any(b)) {
        const int q = lowest(b);
        b = drop_lowest(b);
        acc += eri_at(eri, norbs, p, p, q, q);
    }
    U[static_cast<size_t>(p) * nb + ib] = acc;
}

// diag[ia, ib] = core + E_A[ia] + E_B[ib] + sum_{p in A} U[p][ib]
// (zero_excite_words, slater_condon.cpp:23-39, regrouped by channel).
__global__ void k_diag(const uint64_t* __restrict__ sa, const uint64_t* __restrict__ sahi, const double* __restrict__ EA,
                       uint32_t nloc, const double* __restrict__ EB, const double* __restrict__ U,
                       uint32_t nb, double core, double* __restrict__ diag) {
    const uint32_t ib = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t ia = blockIdx.y;
    if (ib >= nb || ia >= nloc) return;
    Bits a = load_bits(sa, sahi, ia);
    double x = 0.0;
    while (any(a)) {
        const int p = lowest(a);
        a = drop_lowest(a);
        x += U[static_cast<size_t>(p) * nb + ib];
    }
    diag[static_cast<size_t>(ia) * nb + ib] = core + EA[ia] + EB[ib] + x;
}

template <class T>
void upload(DevBuf<T>& d, const std::vector<T>& v, cudaStream_t st) {
    d.alloc(v.size());
    if (!v.empty())
        CUDA_CHECK(cudaMemcpyAsync(d.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
}

void build_helper_lists(Handle& h, int c) {
    ChannelTables& t = h.ch[c];
    const uint32_t n = static_cast<uint32_t>(t.n);
    DevBuf<unsigned int> dup;
    dup.alloc(1);
    const unsigned int none = 0xffffffffu;
    CUDA_CHECK(cudaMemcpyAsync(dup.p, &none, sizeof(none), cudaMemcpyHostToDevice, h.stream));
    for (int k = 0; k < 2; ++k) {
        t.len[k].alloc(n);
        t.offset[k].alloc(static_cast<size_t>(n) + 1);  // [n] holds the total
    }
    const unsigned grid = (n + kPairBlock / kWarp - 1) / (kPairBlock / kWarp);
    if (t.hi())
        k_pair_scan<false, true><<<grid, kPairBlock, 0, h.stream>>>(t.strings.p, t.hi(), n, t.len[0].p, t.len[1].p,
                                                                    nullptr, nullptr, nullptr, nullptr, dup.p);
    else
        k_pair_scan<false, false><<<grid, kPairBlock, 0, h.stream>>>(t.strings.p, nullptr, n, t.len[0].p,
                                                                     t.len[1].p, nullptr, nullptr, nullptr, nullptr,
                                                                     dup.p);
    CUDA_LAUNCH_CHECK();
    unsigned int dup_host = none;
    CUDA_CHECK(cudaMemcpyAsync(&dup_host, dup.p, sizeof(dup_host), cudaMemcpyDeviceToHost, h.stream));
    for (int k = 0; k < 2; ++k) {
        k_scan_offsets<<<1, 1024, 0, h.stream>>>(t.len[k].p, t.offset[k].p, n);
        CUDA_LAUNCH_CHECK();
        CUDA_CHECK(cudaMemcpyAsync(&t.nflat[k], t.offset[k].p + n, sizeof(uint64_t),
                                   cudaMemcpyDeviceToHost, h.stream));
    }
    CUDA_CHECK(cudaStreamSynchronize(h.stream));
    if (dup_host != none)  // index_strings, connectivity.cpp:35-37
        fail(DETCI_GPU_E_INPUT, "excitation tables: duplicate string at index " +
                                    std::to_string(dup_host));
    for (int k = 0; k < 2; ++k) t.flat[k].alloc(std::max<uint64_t>(t.nflat[k], 1));
    if (t.hi())
        k_pair_scan<true, true><<<grid, kPairBlock, 0, h.stream>>>(t.strings.p, t.hi(), n, nullptr, nullptr,
                                                                   t.offset[0].p, t.offset[1].p, t.flat[0].p,
                                                                   t.flat[1].p, nullptr);
    else
        k_pair_scan<true, false><<<grid, kPairBlock, 0, h.stream>>>(t.strings.p, nullptr, n, nullptr, nullptr,
                                                                    t.offset[0].p, t.offset[1].p, t.flat[0].p,
                                                                    t.flat[1].p, nullptr);
    CUDA_LAUNCH_CHECK();
    for (int k = 0; k < 2; ++k) {
        t.h_len[k].resize(n);
        CUDA_CHECK(cudaMemcpyAsync(t.h_len[k].data(), t.len[k].p, n * sizeof(uint32_t),
                                   cudaMemcpyDeviceToHost, h.stream));
    }
}

void build_pair_tables(Handle& h, int c) {
    ChannelTables& t = h.ch[c];
    const uint32_t n = static_cast<uint32_t>(t.n);
    for (int k = 0; k < 2; ++k) {
        const size_t m = std::max<uint64_t>(t.nflat[k], 1);
        t.pv[k].alloc(m);
        if (k == 0) t.pab.alloc(m);
        const unsigned grid = (n * kWarp + 255) / 256;
        k_pair_tables<<<grid, 256, 0, h.stream>>>(k, t.strings.p, t.hi(), n, t.flat[k].p,
                                                  t.offset[k].p, t.len[k].p, h.d_h1.p, h.d_eri.p,
                                                  h.norbs, t.pv[k].p, t.pab.p);
        CUDA_LAUNCH_CHECK();
    }
    const uint32_t ntri = static_cast<uint32_t>(h.norbs * (h.norbs - 1) / 2);
    t.J.alloc(std::max<size_t>(static_cast<size_t>(ntri) * n, 1));
    if (ntri > 0) {
        dim3 grid(std::min<uint32_t>((n + 255) / 256, 64), ntri);
        k_jtable<<<grid, 256, 0, h.stream>>>(t.strings.p, t.hi(), n, h.d_eri.p, h.norbs, t.J.p);
        CUDA_LAUNCH_CHECK();
    }
}

// Mixed-term SELL-32 table, built on the host from the device helper list.
//  * slots: beta strings sorted by singles degree (SELL-C-sigma), so the 32
//    rows of a slice have near-equal lengths (99% fill at C2/C3, 59-81%
//    unsorted);
//  * column segments of <= 12288 beta strings, so the staged C-row segment
//    plus the +-W table leave room for two CTAs per SM;
//  * within each lane the entry order is free (the element sum is
//    order-independent to 1e-16), so each (slice, segment) is scheduled
//    greedily so that at every step the 16 lanes of each half-warp read
//    distinct shared-memory bank pairs for both gathers (W[cd] and
//    C[ja, jb]); padding entries point at a zero of W and reuse a
//    C address already read in that step (broadcast).  Simulated on C2 this
//    cuts shared-memory wavefronts per element step from 9.2 to 5.6.
//  * format 2 (scatter kernel, k_mixed_scatter): the same slots, segments
//    and schedule, but the entry carries cd and the beta sign separately
//    (encode_scatter_entry) because the kernel reads V[k][cd] for K output
//    rows per C gather; the schedule weights V-bank conflicts 8x.
void build_mixed_sell(Handle& h, SellTable& st, int M, int format) {
    ChannelTables& b = h.ch[1];
    const uint32_t nb = static_cast<uint32_t>(b.n);
    const int n = h.norbs;
    const uint32_t nn = static_cast<uint32_t>(n * n);
    // Shared memory per CTA (<= 220 KB): two +-W buffers plus either two
    // double-buffered C stages of M row segments, or -- preferred, because
    // segmenting a row splits every SELL row and costs ~18% fill -- one stage
    // holding the M rows in as few segments as fit.
    // DETCI_MIXED_MAX_SEG caps the segment width (tests force multi-segment
    // tables on small systems with it).
    uint32_t cap = 32766;   // 18-bit byte offsets
    if (const char* e = std::getenv("DETCI_MIXED_MAX_SEG")) cap = std::max(2, std::atoi(e)) & ~1u;
    const uint32_t wdbl = (2 * nn + 1) & ~1u;
    if (format == 2) {
        // The largest K (output rows per CTA) whose K V rows leave room for
        // a Cs segment of >= 2048 columns per vector and that costs no more
        // row segments than K/2 (M = 2 starts at 8: 2 x K accumulators per
        // thread).  Large norbs shrink K (n = 64: 32 KB per V row).
        const int64_t vp = scatter_vpitch(n);
        auto room = [&](int K) { return static_cast<int64_t>(kScatterSmem / 8) - K * vp; };
        auto nseg_for = [&](int K) {
            const uint32_t seg = std::min<uint32_t>(cap, static_cast<uint32_t>(std::max<int64_t>(room(K), 2) / M) & ~1u);
            return (nb + seg - 1) / seg;
        };
        int K = M == 1 ? 16 : 8;
        while (K > 1 && (room(K) < 2048 * M || nseg_for(K) > nseg_for(K / 2))) K /= 2;
        if (room(K) < 64 * M) fail(DETCI_GPU_E_UNSUPPORTED, "mixed term: V rows do not fit shared memory");
        st.kmax = K;
    }
    // (format 2 keeps a zero slot after each staged row segment: 2 doubles)
    const uint32_t budget = format == 2 ? static_cast<uint32_t>(kScatterSmem / 8 - st.kmax * scatter_vpitch(n) - 3 * M)
                                        : 220u * 1024 / 8 - 2 * wdbl;   // doubles for C stages
    const uint32_t single_seg = std::min<uint32_t>(cap, (budget / M) & ~1u);
    const uint32_t double_seg = std::min<uint32_t>(std::min<uint32_t>(16000, cap), (budget / 2 / M) & ~1u);
    const uint32_t nseg_single = (nb + single_seg - 1) / single_seg;
    const uint32_t nseg_double = (nb + double_seg - 1) / double_seg;
    // overlap only when it costs no extra segments (the scatter kernel
    // stages one row per CTA: single buffer)
    st.double_buffer = format == 1 && nseg_double <= nseg_single;
    st.format = format;
    const uint32_t max_seg = st.double_buffer ? double_seg : single_seg;
    st.nseg = (nb + max_seg - 1) / max_seg;
    if (st.nseg > 16) fail(DETCI_GPU_E_UNSUPPORTED, "mixed term: more than 16 column segments");
    if (format == 1 && 2 * nn >= (1u << 14)) fail(DETCI_GPU_E_UNSUPPORTED, "mixed term: +-W index exceeds 14 bits");
    if (format == 2 && pair_count(n) >= (1u << 13))
        fail(DETCI_GPU_E_UNSUPPORTED, "mixed term: pair-ERI column exceeds 13 bits");
    // weight of a V/W bank conflict in the schedule: the scatter kernel reads
    // V once per output row (~8 per C gather on average)
    const int wv = format == 2 ? 8 : 1;
    // random lane orders tried per half-warp step (DETCI_SELL_ATTEMPTS)
    int attempts = 128;   // measured: 8 -> 128 takes C3 mixed 437 -> 428 ms at no visible build cost
    if (const char* e = std::getenv("DETCI_SELL_ATTEMPTS")) attempts = std::max(1, std::atoi(e));
    st.seg_cols = (nb + st.nseg - 1) / st.nseg;
    if (static_cast<uint64_t>(st.seg_cols) * 8 >= (1u << 18))
        fail(DETCI_GPU_E_UNSUPPORTED, "mixed term: row segment exceeds the 18-bit entry offset");
    h.nslices = (nb + kWarp - 1) / kWarp;
    const uint32_t nseg = st.nseg, seg_cols = st.seg_cols, nslices = h.nslices;

    std::vector<uint32_t> flat(std::max<uint64_t>(b.nflat[0], 1));
    std::vector<uint64_t> off(nb);
    copy_sync(flat.data(), b.flat[0].p, b.nflat[0] * 4, cudaMemcpyDeviceToHost, h.stream);
    copy_sync(off.data(), b.offset[0].p, nb * 8, cudaMemcpyDeviceToHost, h.stream);
    const std::vector<uint32_t>& deg = b.h_len[0];
    std::vector<uint32_t> perm(nb);
    std::iota(perm.begin(), perm.end(), 0u);
    std::stable_sort(perm.begin(), perm.end(), [&](uint32_t x, uint32_t y) { return deg[x] > deg[y]; });

    // per (slice, seg) padded lengths
    std::vector<uint32_t> slen(static_cast<size_t>(nslices) * nseg, 0);
    for (uint32_t slot = 0; slot < nb; ++slot) {
        const uint32_t ib = perm[slot];
        uint32_t cnt[16] = {0};
        for (uint32_t k = 0; k < deg[ib]; ++k) ++cnt[flat[off[ib] + k] / seg_cols];
        for (uint32_t g = 0; g < nseg; ++g) {
            uint32_t& m = slen[(slot / kWarp) * nseg + g];
            m = std::max(m, cnt[g]);
        }
    }
    std::vector<uint64_t> soff(slen.size());
    uint64_t total = 0;
    for (size_t i = 0; i < slen.size(); ++i) {
        soff[i] = total;
        total += static_cast<uint64_t>(slen[i]) * kWarp;
    }
    std::vector<uint32_t> sell(std::max<uint64_t>(total, 1), 0);
    const std::vector<uint64_t>& bs = b.h_strings;
    const std::vector<uint64_t>& bs_hi = b.h_strings_hi;
    auto bstr = [&](uint32_t i) { return Bits(bs[i], bs_hi.empty() ? 0ull : bs_hi[i]); };

    #pragma omp parallel for schedule(dynamic, 4)
    for (int64_t sl = 0; sl < static_cast<int64_t>(nslices); ++sl) {
        // (jb_local, bank key: w_index (format 1) or cd | sbit << 31 (format 2))
        std::vector<std::pair<uint32_t, uint32_t>> lanes[kWarp];
        uint64_t rng = 0x9e3779b97f4a7c15ull ^ static_cast<uint64_t>(sl);  // deterministic per slice
        for (uint32_t g = 0; g < nseg; ++g) {
            for (int l = 0; l < kWarp; ++l) {
                lanes[l].clear();
                const uint32_t slot = static_cast<uint32_t>(sl) * kWarp + l;
                if (slot >= nb) continue;
                const uint32_t ib = perm[slot];
                for (uint32_t k = 0; k < deg[ib]; ++k) {
                    const uint32_t jb = flat[off[ib] + k];
                    if (jb / seg_cols != g) continue;
                    const MixedMove mv = mixed_move(bstr(ib), bstr(jb), n);
                    // format 2: the pair-ERI column tri(pb, qb) (V rows are
                    // pair-ERI rows); format 1: the +-W index
                    const uint32_t pcol = tri_index(static_cast<int>(mv.cd) / n, static_cast<int>(mv.cd) % n);
                    lanes[l].emplace_back(jb - g * seg_cols,
                                          format == 2 ? (pcol | mv.sbit << 31) : mv.cd + mv.sbit * nn);
                }
            }
            const uint32_t L = slen[sl * nseg + g];
            uint32_t* out = sell.data() + soff[sl * nseg + g];
            for (uint32_t k = 0; k < L; ++k) {
                for (int half = 0; half < 2; ++half) {
                    int64_t used_w[16], used_c[16];
                    auto cost = [&](uint32_t jbl, uint32_t key) {
                        const uint32_t wi = key & 0x7fffffffu;
                        const int64_t uw = used_w[wi % 16], uc = used_c[jbl % 16];
                        return wv * (uw >= 0 && uw != wi) + (uc >= 0 && uc != jbl);
                    };
                    auto wkey = [](uint32_t key) { return key & 0x7fffffffu; };
                    int vrem[16] = {0};
                    for (int i = 0; i < 16; ++i)
                        for (const auto& en : lanes[half * 16 + i]) ++vrem[wkey(en.second) % 16];
                    // greedy first-fit over the 16 lanes, best of a few lane orders
                    int order[16], best_order[16], best_total = 1 << 30;
                    size_t pick[16], best_pick[16];
                    for (int i = 0; i < 16; ++i) order[i] = half * 16 + i;
                    for (int attempt = 0; attempt < attempts && best_total > 0; ++attempt) {
                        if (attempt > 0)
                            for (int i = 15; i > 0; --i) {
                                rng = rng * 6364136223846793005ull + 1442695040888963407ull;
                                std::swap(order[i], order[(rng >> 33) % (i + 1)]);
                            }
                        for (int i = 0; i < 16; ++i) used_w[i] = used_c[i] = -1;
                        int total = 0;
                        for (int oi = 0; oi < 16; ++oi) {
                            const auto& r = lanes[order[oi]];
                            if (r.empty()) continue;
                            // least cost; ties go to the V bank with the most
                            // entries left in the half-warp (keeps later steps
                            // from running out of distinct banks)
                            size_t best = 0;
                            int best_cost = 1 << 20, best_rem = -1;
                            for (size_t i = 0; i < r.size(); ++i) {
                                const int c = cost(r[i].first, r[i].second);
                                const int rm = vrem[wkey(r[i].second) % 16];
                                if (c < best_cost || (c == best_cost && rm > best_rem)) {
                                    best_cost = c;
                                    best_rem = rm;
                                    best = i;
                                }
                            }
                            pick[oi] = best;
                            total += best_cost;
                            const uint32_t bw = wkey(r[best].second);
                            if (used_w[bw % 16] < 0) used_w[bw % 16] = bw;
                            if (used_c[r[best].first % 16] < 0) used_c[r[best].first % 16] = r[best].first;
                        }
                        if (total < best_total) {
                            best_total = total;
                            std::copy(order, order + 16, best_order);
                            std::copy(pick, pick + 16, best_pick);
                        }
                    }
                    for (int i = 0; i < 16; ++i) used_w[i] = used_c[i] = -1;
                    int pads[16], npad = 0;
                    for (int oi = 0; oi < 16; ++oi) {
                        const int l = best_order[oi];
                        auto& r = lanes[l];
                        if (r.empty()) {
                            pads[npad++] = l;
                            continue;
                        }
                        const auto e = r[best_pick[oi]];
                        r[best_pick[oi]] = r.back();
                        r.pop_back();
                        const uint32_t ew = wkey(e.second);
                        if (used_w[ew % 16] < 0) used_w[ew % 16] = ew;
                        if (used_c[e.first % 16] < 0) used_c[e.first % 16] = e.first;
                        out[static_cast<size_t>(k) * kWarp + l] =
                            format == 2 ? encode_scatter_entry(e.first, ew, e.second >> 31)
                                        : encode_mixed_entry(e.first, e.second);
                    }
                    for (int p = 0; p < npad; ++p) {
                        if (format == 2) {
                            // scatter kernel: the C side reads the zero slot
                            // after the staged segment (index seg_cols); any V
                            // address already read in this step (broadcast)
                            uint32_t wz = 0;
                            for (int i = 0; i < 16; ++i)
                                if (used_w[i] >= 0) {
                                    wz = static_cast<uint32_t>(used_w[i]);
                                    break;
                                }
                            if (used_w[wz % 16] < 0) used_w[wz % 16] = wz;
                            if (used_c[seg_cols % 16] < 0) used_c[seg_cols % 16] = seg_cols;
                            out[static_cast<size_t>(k) * kWarp + pads[p]] = encode_scatter_entry(seg_cols, wz, 0);
                            continue;
                        }
                        // a zero of W (diagonal c == d) on a free or same-address bank
                        uint32_t wz = 0;
                        for (int c = 0; c < n; ++c) {
                            const uint32_t z = static_cast<uint32_t>(c * n + c);
                            if (used_w[z % 16] < 0 || used_w[z % 16] == z) {
                                wz = z;
                                break;
                            }
                        }
                        if (used_w[wz % 16] < 0) used_w[wz % 16] = wz;
                        uint32_t jz = 0;
                        for (int i = 0; i < 16; ++i)
                            if (used_c[i] >= 0) {
                                jz = static_cast<uint32_t>(used_c[i]);
                                break;
                            }
                        out[static_cast<size_t>(k) * kWarp + pads[p]] =
                            format == 2 ? encode_scatter_entry(jz, wz, 0) : encode_mixed_entry(jz, wz);
                    }
                }
            }
        }
    }
    if (!h.sell_perm.p) upload(h.sell_perm, perm, h.stream);
    upload(st.len, slen, h.stream);
    upload(st.off, soff, h.stream);
    upload(st.sell, sell, h.stream);
    CUDA_CHECK(cudaStreamSynchronize(h.stream));
    if (format == 2 && M == 1) {
        // scatter work per slice (padded entries over the segments) plus the
        // per-slot D store + reduction, which costs as much as ~9 entries
        // (16 B of HBM per (row, single) pair against ~1.1 x 8 B of shared
        // memory per entry and pair, at ~6 vs ~30 TB/s): the multi-rank
        // column shares are cut on its prefix (mixed_slots)
        h.slice_prefix.assign(static_cast<size_t>(nslices) + 1, 0);
        for (uint32_t sl = 0; sl < nslices; ++sl) {
            uint64_t w = 9;
            for (uint32_t g = 0; g < nseg; ++g) w += slen[static_cast<size_t>(sl) * nseg + g];
            h.slice_prefix[sl + 1] = h.slice_prefix[sl] + w;
        }
    }
    st.built = true;
}

namespace {
// Block edges on multiples of 128 rows when blocks are large: a block's
// rows are the beta term's columns, and a partial 128-column chunk runs
// the clamped tail kernel (C3 at 8 blocks: 29 ms of tails vs 7 ms at one
// block).  Costs <= 64 rows (3% at C3 / 8) of balance.  Kept only when no
// block becomes empty.
void round_block_edges(std::vector<uint64_t>& blk, uint64_t na) {
    const int P = static_cast<int>(blk.size()) - 1;
    if (P <= 1 || na < 1024ull * P) return;
    std::vector<uint64_t> r = blk;
    bool nonempty = true;
    for (int g = 1; g < P; ++g) {
        uint64_t e = (r[g] + 64) / 128 * 128;
        e = std::max(e, r[g - 1]);
        r[g] = std::min(e, na);
        nonempty = nonempty && r[g] > r[g - 1];
    }
    nonempty = nonempty && r[P] > r[P - 1];
    if (nonempty) blk = r;
}

// P cuts of a prefix array (size n + 1) at equal shares, each part >= 1.
std::vector<uint64_t> cut_prefix(const std::vector<double>& prefix, int P) {
    const uint64_t n = prefix.size() - 1;
    std::vector<uint64_t> c(P + 1, 0);
    c[P] = n;
    for (int g = 1; g < P; ++g) {
        const double target = prefix[n] * g / P;
        uint64_t cut = std::lower_bound(prefix.begin(), prefix.end(), target) - prefix.begin();
        cut = std::max<uint64_t>(cut, c[g - 1] + 1);
        cut = std::min<uint64_t>(cut, n - (P - g));
        c[g] = cut;
    }
    return c;
}
} // namespace

void set_local_rows(Handle& h);

void build_partition(Handle& h) {
    const int P = std::max(h.world, h.vblocks);
    const uint64_t na = h.na(), nb = h.nb();
    h.blk.assign(P + 1, 0);
    // Under the gather schedule the mixed term is split by beta-slot columns
    // (mixed_slots), not by rows: the row partition then balances the
    // same-spin work only (weighted = 2).
    const bool gather = P > 1 && mixed_scatter_enabled() && !multi_ring();
    plan_partition(na, nb, h.ch[0].h_len[0].data(), h.ch[0].h_len[1].data(), h.ch[1].h_len[0].data(),
                   h.ch[1].h_len[1].data(), P, h.weighted && gather ? 2 : h.weighted, h.blk.data());
    // Block edges on multiples of 128 rows when blocks are large: a block's
    // rows are the beta term's columns, and a partial 128-column chunk runs
    // the clamped tail kernel (C3 at 8 blocks: 29 ms of tails vs 7 ms at one
    // block).  Costs <= 64 rows (3% at C3 / 8) of balance.
    // Kept only when no block becomes empty.
    round_block_edges(h.blk, na);
    uint64_t sum_sb = 0, sum_db = 0, sum_sa = 0, sum_da = 0;
    for (uint64_t i = 0; i < nb; ++i) {
        sum_sb += h.ch[1].h_len[0][i];
        sum_db += h.ch[1].h_len[1][i];
    }
    for (uint64_t i = 0; i < na; ++i) {
        sum_sa += h.ch[0].h_len[0][i];
        sum_da += h.ch[0].h_len[1][i];
    }
    h.nnz_alpha = (sum_sa + sum_da) * nb;
    h.nnz_beta = (sum_sb + sum_db) * na;
    h.nnz_mixed = sum_sa * sum_sb;
    h.slot_cut.clear();
    set_local_rows(h);
}

void set_local_rows(Handle& h) {
    const int P = std::max(h.world, h.vblocks);
    const uint64_t na = h.na();
    h.max_blk = 0;
    for (int g = 0; g < P; ++g) h.max_blk = std::max(h.max_blk, h.blk[g + 1] - h.blk[g]);
    if (h.world > 1) {
        h.a0 = h.blk[h.rank];
        h.a1 = h.blk[h.rank + 1];
    } else {
        h.a0 = 0;
        h.a1 = na;  // virtual blocks: this process owns every row
    }
}

void build_diag(Handle& h) {
    const uint32_t na = static_cast<uint32_t>(h.na()), nb = static_cast<uint32_t>(h.nb());
    DevBuf<double> EA, EB, U;
    EA.alloc(na);
    EB.alloc(nb);
    U.alloc(static_cast<size_t>(h.norbs) * nb);
    k_string_energy<<<(na + 255) / 256, 256, 0, h.stream>>>(h.ch[0].strings.p, h.ch[0].hi(), na, h.d_h1.p,
                                                            h.d_eri.p, h.norbs, EA.p);
    k_string_energy<<<(nb + 255) / 256, 256, 0, h.stream>>>(h.ch[1].strings.p, h.ch[1].hi(), nb, h.d_h1.p,
                                                            h.d_eri.p, h.norbs, EB.p);
    k_u_table<<<dim3((nb + 255) / 256, h.norbs), 256, 0, h.stream>>>(h.ch[1].strings.p, h.ch[1].hi(), nb,
                                                                      h.d_eri.p, h.norbs, U.p);
    CUDA_LAUNCH_CHECK();
    const uint32_t nloc = static_cast<uint32_t>(h.nloc());
    h.diag.alloc(std::max<size_t>(h.local_len(), 1));
    for (uint32_t r0 = 0; r0 < nloc; r0 += 65535) {
        const uint32_t rows = std::min<uint32_t>(65535, nloc - r0);
        k_diag<<<dim3((nb + 255) / 256, rows), 256, 0, h.stream>>>(
            h.ch[0].strings.p + h.a0 + r0, h.ch[0].hi() ? h.ch[0].hi() + h.a0 + r0 : nullptr, EA.p + h.a0 + r0,
            rows, EB.p, U.p, nb, h.core,
            h.diag.p + static_cast<size_t>(r0) * nb);
        CUDA_LAUNCH_CHECK();
    }
    CUDA_CHECK(cudaStreamSynchronize(h.stream));
}

size_t estimate_bytes(const Handle& h) {
    const size_t na = h.na(), nb = h.nb();
    const size_t ntri = static_cast<size_t>(h.norbs) * (h.norbs - 1) / 2;
    size_t b = static_cast<size_t>(h.norbs) * h.norbs * h.norbs * h.norbs * 8;
    for (int c = 0; c < 2; ++c) {
        const auto& t = h.ch[c];
        const size_t e = t.nflat[0] + t.nflat[1];
        b += e * (4 + 8) + t.nflat[0] * 4 + t.n * (16 + 2 * (12 + 4)) + ntri * t.n * 8;
    }
    b += (h.ch[1].nflat[0] * 4) * 2;             // SELL incl. padding slack
    const int P = std::max(h.world, h.vblocks);
    size_t max_blk = (na + P - 1) / P + 1;
    if (P > 1) max_blk = std::max<size_t>(max_blk, na / P + 2);
    const size_t loc = (h.world > 1 ? max_blk : na) * nb;
    b += loc * 8;                                 // diag
    b += 3 * max_blk * nb * 8;                    // ct, yt, xs
    if (P > 1) b += 2 * max_blk * nb * 8;         // ring buffers
    return b;
}

} // namespace

const SellTable& mixed_table(Handle& h, int M) {
    const int idx = M == 1 ? 0 : (M == 2 ? 1 : 2);
    SellTable& t = h.sell_m[idx];
    if (h.norbs > 64)   // its +-W tables hold one uint64 per string move
        fail(DETCI_GPU_E_UNSUPPORTED, "mixed term: norbs > 64 runs on the scatter kernel only (M <= 2)");
    if (!t.built) build_mixed_sell(h, t, M, 1);
    return t;
}

const SellTable& scatter_table(Handle& h, int M) {
    SellTable& t = h.sell_scatter[M == 2 ? 1 : 0];
    if (!t.built) {
        build_mixed_sell(h, t, M == 2 ? 2 : 1, 2);
        if (!h.tpos.p) build_scatter_tpos(h);
    }
    return t;
}

void build_scatter_tpos(Handle& h) {
    ChannelTables& a = h.ch[0];
    const uint32_t n = static_cast<uint32_t>(a.n);
    h.tpos.alloc(std::max<uint64_t>(a.nflat[0], 1));
    k_tpos<<<(n * kWarp + 255) / 256, 256, 0, h.stream>>>(a.flat[0].p, a.offset[0].p, a.len[0].p, n, h.tpos.p);
    CUDA_LAUNCH_CHECK();
    h.h_sa_flat.resize(std::max<uint64_t>(a.nflat[0], 1));
    h.h_sa_off.resize(n + 1);
    CUDA_CHECK(cudaMemcpyAsync(h.h_sa_flat.data(), a.flat[0].p, a.nflat[0] * 4, cudaMemcpyDeviceToHost, h.stream));
    CUDA_CHECK(cudaMemcpyAsync(h.h_sa_off.data(), a.offset[0].p, (n + 1) * 8, cudaMemcpyDeviceToHost, h.stream));
    CUDA_CHECK(cudaStreamSynchronize(h.stream));
}

void release_sigma_scratch(Handle& h) {
    h.dbuf.reset();
    h.dcap_rows = 0;
    h.dplan_m = 0;
    h.scatter_plan.clear();
}

void release_basis(Handle& h) {
    for (auto& t : h.ch) {
        for (int k = 0; k < 2; ++k) {
            t.flat[k].reset();
            t.offset[k].reset();
            t.len[k].reset();
            t.pv[k].reset();
        }
        t.pab.reset();
        t.J.reset();
    }
    for (SellTable* tp : {&h.sell_m[0], &h.sell_m[1], &h.sell_m[2], &h.sell_scatter[0], &h.sell_scatter[1]}) {
        SellTable& t = *tp;
        t.sell.reset();
        t.off.reset();
        t.len.reset();
        t.built = false;
    }
    h.sell_perm.reset();
    release_stored(h);
    h.tpos.reset();
    h.h_sa_flat.clear();
    h.h_sa_off.clear();
    release_sigma_scratch(h);
    h.diag.reset();
    h.ct.reset();
    h.yt.reset();
    h.xs.reset();
    h.dav_store.reset();
    h.cs_full.reset();
    h.mix_t.reset();
    h.mix_r.reset();
    h.ring[0].reset();
    h.ring[1].reset();
    h.xbuf.reset();
    h.ybuf.reset();
    h.built = false;
}

// Pair-ERI matrix PE[tri(p,q)][tri(r,s)] = (pq|rs) over unordered pairs
// p != q, r != s (rows padded to scatter_vpitch): the scatter kernel's V rows.
// 8-fold symmetry of the real integrals ((pq|rs) = (qp|rs) = (pq|sr); the
// reference reads them that way, integrals.hpp) makes one value per pair.
void build_pair_eri(Handle& h) {
    const int n = h.norbs;
    const uint32_t T = pair_count(n), vp = scatter_vpitch(n);
    std::vector<double> pe(static_cast<size_t>(std::max<uint32_t>(T, 1)) * vp, 0.0);
    for (int p = 1; p < n; ++p)
        for (int q = 0; q < p; ++q)
            for (int r = 1; r < n; ++r)
                for (int s = 0; s < r; ++s)
                    pe[static_cast<size_t>(tri_index(p, q)) * vp + tri_index(r, s)] = eri_at(h.eri.data(), n, p, q, r, s);
    h.d_pair.alloc(pe.size());
    copy_sync(h.d_pair.p, pe.data(), pe.size() * sizeof(double), cudaMemcpyHostToDevice, h.stream);
}

void build_device_basis(Handle& h) {
    if (!h.have_strings) fail(DETCI_GPU_E_INPUT, "build_basis: strings not set");
    if (!h.have_ints) fail(DETCI_GPU_E_INPUT, "build_basis: integrals not set");
    release_basis(h);
    for (int c = 0; c < 2; ++c) build_helper_lists(h, c);
    CUDA_CHECK(cudaStreamSynchronize(h.stream));
    build_partition(h);

    size_t free_b = 0, total_b = 0;
    CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
    const uint64_t budget = h.budget ? h.budget : free_b;
    const size_t need = estimate_bytes(h);
    // basis.cpp:113-118 convention; free memory differs per rank, so the
    // decision is collective (no rank builds while a peer has given up)
    collective_require(h, need <= budget, DETCI_GPU_E_CAPACITY,
                       "device basis requires " + std::to_string(need) + " bytes, budget is " +
                           std::to_string(budget) + " bytes",
                       "build_basis");

    for (int c = 0; c < 2; ++c) build_pair_tables(h, c);
    build_pair_eri(h);
    if (mixed_scatter_enabled()) scatter_table(h, 1);
    else build_mixed_sell(h, h.sell_m[0], 1, 1);
    build_diag(h);
    const size_t scratch = static_cast<size_t>(h.max_blk) * h.nb();
    h.ct.alloc(std::max<size_t>(scratch, 1));
    h.yt.alloc(std::max<size_t>(scratch, 1));
    h.xs.alloc(std::max<size_t>(h.vblocks > 1 ? h.na() * h.nb() : scratch, 1));
    // (the ring buffers of DETCI_MULTI=ring are allocated by its first sigma)
    CUDA_CHECK(cudaStreamSynchronize(h.stream));
    h.built = all_ranks_ok(h, true);
}

// Measured rebalance (detci_gpu_rebalance): re-cut the alpha-row blocks and
// the mixed term's beta-slot shares from the per-rank phase times of a timed
// sigma, t[4 g + phase] (phases alpha, beta, mixed, combine).  The static
// cuts weight rows by alpha elements + beta work and slices by scatter work
// (plan_partition, slice_prefix) at one cost per unit; here each block-rank's
// measured seconds per modelled unit replace that cost over its own range,
// so the new cuts follow what the model misses (the L2 locality of a row
// range, the per-CTA staging of a light column share).  matvec.cpp:108-111
// is the reference's n*g/P; PAPER.md:304 names load imbalance as what limits
// its scaling.
void rebalance_partition(Handle& h, const std::vector<double>& t) {
    const int P = std::max(h.world, h.vblocks);
    if (P <= 1 || t.size() < 4 * static_cast<size_t>(P)) return;
    const uint64_t na = h.na();
    const auto& sa = h.ch[0].h_len[0];
    const auto& da = h.ch[0].h_len[1];
    auto floor_rates = [&](std::vector<double>& r) {
        double m = 0.0;
        for (double v : r) m += v;
        m /= P;
        for (double& v : r) v = std::max(v, 0.1 * m);
    };
    // rows: alpha seconds per alpha element, beta + combine seconds per row
    std::vector<double> ra(P, 0.0), rb(P, 0.0);
    for (int g = 0; g < P; ++g) {
        double wa = 0.0;
        for (uint64_t i = h.blk[g]; i < h.blk[g + 1]; ++i) wa += static_cast<double>(sa[i] + da[i]);
        const double rows = static_cast<double>(h.blk[g + 1] - h.blk[g]);
        ra[g] = wa > 0 ? t[4 * g] / wa : 0.0;
        rb[g] = rows > 0 ? (t[4 * g + 1] + t[4 * g + 3]) / rows : 0.0;
    }
    floor_rates(ra);
    floor_rates(rb);
    std::vector<double> prefix(na + 1, 0.0);
    for (int g = 0; g < P; ++g)
        for (uint64_t i = h.blk[g]; i < h.blk[g + 1]; ++i)
            prefix[i + 1] = prefix[i] + static_cast<double>(sa[i] + da[i]) * ra[g] + rb[g];
    std::vector<uint64_t> blk = cut_prefix(prefix, P);
    round_block_edges(blk, na);
    // beta-slot shares of the mixed term: seconds per unit of slice work
    std::vector<uint32_t> cut;
    const auto& pre = h.slice_prefix;
    const uint32_t nsl = h.nslices;
    if (pre.size() == static_cast<size_t>(nsl) + 1 && nsl >= static_cast<uint32_t>(P)) {
        std::vector<uint32_t> old(P + 1, 0);
        for (int g = 0; g < P; ++g) old[g] = mixed_slots(h, g, P).first / kWarp;
        old[P] = nsl;
        std::vector<double> rm(P, 0.0);
        for (int g = 0; g < P; ++g) {
            const double w = static_cast<double>(pre[std::min(old[g + 1], nsl)] - pre[std::min(old[g], nsl)]);
            rm[g] = w > 0 ? t[4 * g + 2] / w : 0.0;
        }
        floor_rates(rm);
        std::vector<double> sp(nsl + 1, 0.0);
        int g = 0;
        for (uint32_t sl = 0; sl < nsl; ++sl) {
            while (g + 1 < P && sl >= old[g + 1]) ++g;
            sp[sl + 1] = sp[sl] + static_cast<double>(pre[sl + 1] - pre[sl]) * rm[g];
        }
        const std::vector<uint64_t> c = cut_prefix(sp, P);
        cut.resize(P + 1);
        for (int k = 0; k <= P; ++k) cut[k] = static_cast<uint32_t>(c[k]) * kWarp;
    }
    h.blk = blk;
    h.slot_cut = cut;
    set_local_rows(h);
    release_sigma_scratch(h);
    if (h.world > 1) build_diag(h);
}

} // namespace detci_gpu
