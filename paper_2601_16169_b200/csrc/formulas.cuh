// Per-channel Slater-Condon closed forms used by the sigma kernels.
//
// The reference evaluates every element from the full interleaved
// determinant (hij_words, slater_condon.cpp:96-105; alpha p is spin-orbital
// 2p, beta p is 2p+1, bitstring.hpp:13-16).  The kernels work in the
// *separated* ordering instead (all alpha spin-orbitals, then all beta).
// The two orderings of a determinant |A,B> differ by the permutation sign
//   eps(A,B) = (-1)^{#{(p in A, q in B) : q < p}} = (-1)^{popc(A & P(B))},
// P(B) bit p = parity of popc(B & ((1<<p)-1)) (exclusive prefix parity), so
//   H_ref[(A,B),(A',B')] = eps(A,B) eps(A',B') H_sep[(A,B),(A',B')]
// and sigma = eps o (H_sep (eps o C)).  In H_sep every sign is a
// same-channel parity: the spectator masks of the interleaved phase
// (popc(B & [lo,hi-1]) for alpha moves, popc(A & [lo+1,hi]) for beta moves)
// are exactly eps(A,B)eps(A',B) resp. eps(A,B)eps(A,B'), so same-spin
// elements and the mixed element
//   H_sep = (-1)^{popc(A & open(pa,qa)) + popc(B & open(pb,qb))} (pa qa|pb qb)
// no longer depend on the other channel's string except through the J term
// of singles.  These functions are __host__ __device__ so the same code runs
// in the table-building kernels and in the CPU self-check exported as
// detci_gpu_factorized_element (tests compare it with the reference hij on
// random pairs, no GPU needed).
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

// Exclusive prefix parity P(B): bit p = parity(popc(B & ((1 << p) - 1))).
DG_HD uint64_t prefix_parity(uint64_t b) {
    uint64_t x = b << 1;
    x ^= x << 1;
    x ^= x << 2;
    x ^= x << 4;
    x ^= x << 8;
    x ^= x << 16;
    x ^= x << 32;
    return x;
}

// eps(A,B) of the separated <-> interleaved reordering as a parity bit.
DG_HD int eps_parity(uint64_t a, uint64_t pb) { return popc64(a & pb) & 1; }

// One same-spin helper-list entry: bra string si (row), ket string sj
// (target), kind 0 single, 1 double.  Separated-ordering element for
// spectator string S:
//   single: v + (-1)^{sgn} * J_S[tri]
//   double: v
// one_excite_words / two_excite_words, slater_condon.cpp:41-94.
struct PairEntry {
    double v;
    uint32_t ab_sign; // singles: tri(p,q) | sgn << 31
};

DG_HD PairEntry make_pair_entry(int kind, uint64_t si, uint64_t sj, const double* h1,
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

// Format 2 (scatter kernel):
//   bits 0..17  byte offset of Cs[ja, jb] in the staged row segment
//   bits 18..29 cd = pb * n + qb (n <= 64)
//   bit  31     sbit (beta same-channel parity)
DG_HD uint32_t encode_scatter_entry(uint32_t jb_local, uint32_t cd, uint32_t sbit) {
    return (jb_local * 8u) | (cd << 18) | (sbit << 31);
}

// W_m[cd] of the mixed term for the alpha move m = pa -> qa:
// (pa qa | c d), zero on the diagonal c == d (also the value padding
// entries point at).
DG_HD double mixed_weight(const double* eri, int n, int pa, int qa, int c, int d) {
    return c == d ? 0.0 : eri_at(eri, n, pa, qa, c, d);
}

// Same-channel parity of the alpha half of a mixed element: popc(A & open(pa,qa)).
DG_HD int mixed_alpha_parity(uint64_t a_bra, int pa, int qa) {
    return popc64(a_bra & open_mask(pa, qa)) & 1;
}

} // namespace detci_gpu
