// Per-channel Slater-Condon closed forms used by the sigma kernels.
//
// The reference evaluates every element from the full interleaved
// determinant (hij_words, slater_condon.cpp:96-105).  The kernels instead
// factor each element into a part that depends only on the moving channel's
// string pair (precomputed once per helper-list entry) and a spectator part
// evaluated per determinant with one AND + POPC.  These functions are
// __host__ __device__ so the same code runs in the table-building kernels and
// in the CPU self-check exported as detci_gpu_factorized_element (tests
// compare it with the reference hij on random pairs, no GPU needed).
#pragma once

#include "common.cuh"

namespace detci_gpu {

#ifdef __CUDACC__
#define DG_HD __host__ __device__ __forceinline__
#else
#define DG_HD inline
#endif

DG_HD int popc64(uint64_t x) {
#ifdef __CUDA_ARCH__
    return __popcll(x);
#else
    return __builtin_popcountll(x);
#endif
}

DG_HD int ctz64(uint64_t x) {
#ifdef __CUDA_ARCH__
    return __ffsll(static_cast<long long>(x)) - 1;
#else
    return __builtin_ctzll(x);
#endif
}

DG_HD double eri_at(const double* eri, int n, int p, int q, int r, int s) {
    return eri[((static_cast<size_t>(p) * n + q) * n + r) * n + s];
}

// One same-spin helper-list entry: bra string si (row), ket string sj
// (target).  ch = channel that moves (0 alpha, 1 beta), kind 0 single,
// 1 double.  Element for spectator string S:
//   single: (-1)^{popc(S & mask)} * (v + (-1)^{sgn} * J_S[tri])
//   double: (-1)^{popc(S & mask)} * v
// one_excite_words / two_excite_words, slater_condon.cpp:41-94.
struct PairEntry {
    double v;
    uint64_t mask;
    uint32_t ab_sign; // singles: tri(p,q) | sgn << 31
};

DG_HD PairEntry make_pair_entry(int ch, int kind, uint64_t si, uint64_t sj, const double* h1,
                                const double* eri, int n) {
    PairEntry e;
    const uint64_t x = si & ~sj; // bra-only: annihilated
    const uint64_t y = sj & ~si; // ket-only: created
    if (kind == 0) {
        const int p = ctz64(x), q = ctz64(y);
        const int sgn = popc64(si & open_mask(p, q)) & 1;
        double v = h1[p * n + q];
        // ket-occupied r of the moving channel, r == q included (its direct
        // and exchange parts cancel, slater_condon.cpp:55-63)
        uint64_t r_bits = sj;
        while (r_bits) {
            const int r = ctz64(r_bits);
            r_bits &= r_bits - 1;
            v += eri_at(eri, n, p, q, r, r);
            v -= eri_at(eri, n, p, r, r, q);
        }
        e.v = sgn ? -v : v;
        e.mask = spectator_mask(ch, p, q);
        e.ab_sign = tri_index(p, q) | (static_cast<uint32_t>(sgn) << 31);
    } else {
        const int p1 = ctz64(x), p2 = ctz64(x & (x - 1));
        const int q1 = ctz64(y), q2 = ctz64(y & (y - 1));
        // parity_double_words (bitstring.cpp:100-107): p1->q1 on the bra,
        // then p2->q2 on the intermediate string
        const int s1 = popc64(si & open_mask(p1, q1)) & 1;
        const uint64_t mid = (si & ~(1ull << p1)) | (1ull << q1);
        const int s2 = popc64(mid & open_mask(p2, q2)) & 1;
        const double v = eri_at(eri, n, p1, q1, p2, q2) - eri_at(eri, n, p1, q2, p2, q1);
        e.v = (s1 ^ s2) ? -v : v;
        e.mask = spectator_mask(ch, p1, q1) ^ spectator_mask(ch, p2, q2);
        e.ab_sign = 0;
    }
    return e;
}

// Packed beta-single entry for the mixed term (SELL-32 table):
//   bits 0..17  byte offset of C[ja, jb] inside the staged row segment
//               (jb relative to its segment, times 8; segments <= 32767 cols)
//   bits 18..31 index into the +-W table: cd + sbit * n^2 with cd = pb*n+qb
//               and sbit = parity of popc(B_ib & open(pb, qb)) (< 2*64^2)
// so the kernel needs one AND and one shift to address both gathers and the
// sign of the beta half is folded into which half of +-W is read.
struct MixedMove {
    uint32_t cd;
    uint32_t sbit;
};

DG_HD MixedMove mixed_move(uint64_t b_bra, uint64_t b_ket, int n) {
    const uint64_t x = b_bra & ~b_ket, y = b_ket & ~b_bra;
    const int pb = ctz64(x), qb = ctz64(y);
    MixedMove m;
    m.cd = static_cast<uint32_t>(pb * n + qb);
    m.sbit = static_cast<uint32_t>(popc64(b_bra & open_mask(pb, qb)) & 1);
    return m;
}

DG_HD uint32_t encode_mixed_entry(uint32_t jb_local, uint32_t w_index) {
    return (jb_local * 8u) | (w_index << 18);
}

// W_ja[cd] of the mixed term: (pa qa | c d) * (-1)^{popc(A'_ja & Mbeta(c,d))}
// with the alpha move pa (bra-only) -> qa (ket-only); zero on the diagonal
// c == d (also the value padding entries point at).
DG_HD double mixed_weight(const double* eri, int n, int pa, int qa, uint64_t a_ket, int c, int d) {
    if (c == d) return 0.0;
    const double v = eri_at(eri, n, pa, qa, c, d);
    return (popc64(a_ket & spectator_mask(1, c, d)) & 1) ? -v : v;
}

// Sign of the alpha half of a mixed element that depends on the bra pair:
// popc(A & open(pa,qa)) + popc(B & [lo, hi-1]).
DG_HD int mixed_outer_parity(uint64_t a_bra, uint64_t b_bra, int pa, int qa) {
    return (popc64(a_bra & open_mask(pa, qa)) + popc64(b_bra & spectator_mask(0, pa, qa))) & 1;
}

} // namespace detci_gpu
