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

// A channel string of up to 128 spatial orbitals: orbital p is bit p % 64
// of word p / 64, as the reference's multi-word BitString lays them out
// (bitstring.hpp:33-51; kMaxKernelBits = 256 spin-orbitals,
// slater_condon.hpp:26).  Systems with norbs <= 64 keep hi == 0, and every
// helper below reduces to the one-word form.
struct Bits {
    uint64_t lo, hi;
    DG_HD Bits(uint64_t l = 0, uint64_t h = 0) : lo(l), hi(h) {}
};
DG_HD Bits operator&(Bits a, Bits b) { return Bits(a.lo & b.lo, a.hi & b.hi); }
DG_HD Bits operator|(Bits a, Bits b) { return Bits(a.lo | b.lo, a.hi | b.hi); }
DG_HD Bits operator^(Bits a, Bits b) { return Bits(a.lo ^ b.lo, a.hi ^ b.hi); }
DG_HD Bits operator~(Bits a) { return Bits(~a.lo, ~a.hi); }
DG_HD bool any(Bits a) { return (a.lo | a.hi) != 0; }
DG_HD int popc(Bits a) { return popc64(a.lo) + popc64(a.hi); }
// lowest set orbital of a nonzero string
DG_HD int lowest(Bits a) { return a.lo ? ctz64(a.lo) : 64 + ctz64(a.hi); }
DG_HD Bits drop_lowest(Bits a) {
    if (a.lo) a.lo &= a.lo - 1;
    else a.hi &= a.hi - 1;
    return a;
}
DG_HD Bits bit_at(int p) { return p < 64 ? Bits(1ull << p, 0) : Bits(0, 1ull << (p - 64)); }
// orbitals strictly between a and b
DG_HD Bits open_bits(int a, int b) {
    const int lo = (a < b ? a : b) + 1, hi = (a < b ? b : a) - 1;
    Bits r;
    if (lo <= 63) r.lo = bit_range(lo, hi < 63 ? hi : 63);
    if (hi >= 64) r.hi = bit_range(lo > 64 ? lo - 64 : 0, hi - 64);
    return r;
}
// string i of a channel table: the high words live in a second array, null
// for norbs <= 64
DG_HD Bits load_bits(const uint64_t* lo, const uint64_t* hi, size_t i) { return Bits(lo[i], hi ? hi[i] : 0ull); }

// Exclusive prefix parity over both words: the high word also carries the
// parity of the whole low word.
DG_HD Bits prefix_parity(Bits b) {
    Bits r(prefix_parity(b.lo), prefix_parity(b.hi));
    if (popc64(b.lo) & 1) r.hi = ~r.hi;
    return r;
}

// eps(A,B) of the separated <-> interleaved reordering as a parity bit.
DG_HD int eps_parity(Bits a, Bits pb) { return popc(a & pb) & 1; }

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

DG_HD PairEntry make_pair_entry(int kind, Bits si, Bits sj, const double* h1,
                                const double* eri, int n) {
    PairEntry e;
    const Bits x = si & ~sj; // bra-only: annihilated
    const Bits y = sj & ~si; // ket-only: created
    if (kind == 0) {
        const int p = lowest(x), q = lowest(y);
        const int sgn = popc(si & open_bits(p, q)) & 1;
        double v = h1[p * n + q];
        // ket-occupied r of the moving channel, r == q included (its direct
        // and exchange parts cancel, slater_condon.cpp:55-63)
        Bits r_bits = sj;
        while (any(r_bits)) {
            const int r = lowest(r_bits);
            r_bits = drop_lowest(r_bits);
            v += eri_at(eri, n, p, q, r, r);
            v -= eri_at(eri, n, p, r, r, q);
        }
        e.v = sgn ? -v : v;
        e.ab_sign = tri_index(p, q) | (static_cast<uint32_t>(sgn) << 31);
    } else {
        const int p1 = lowest(x), p2 = lowest(drop_lowest(x));
        const int q1 = lowest(y), q2 = lowest(drop_lowest(y));
        // parity_double_words (bitstring.cpp:100-107): p1->q1 on the bra,
        // then p2->q2 on the intermediate string
        const int s1 = popc(si & open_bits(p1, q1)) & 1;
        const Bits mid = (si & ~bit_at(p1)) | bit_at(q1);
        const int s2 = popc(mid & open_bits(p2, q2)) & 1;
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

DG_HD MixedMove mixed_move(Bits b_bra, Bits b_ket, int n) {
    const Bits x = b_bra & ~b_ket, y = b_ket & ~b_bra;
    const int pb = lowest(x), qb = lowest(y);
    MixedMove m;
    m.cd = static_cast<uint32_t>(pb * n + qb);
    m.sbit = static_cast<uint32_t>(popc(b_bra & open_bits(pb, qb)) & 1);
    return m;
}

DG_HD uint32_t encode_mixed_entry(uint32_t jb_local, uint32_t w_index) {
    return (jb_local * 8u) | (w_index << 18);
}

// Format 2 (scatter kernel):
//   bits 0..17  byte offset of Cs[ja, jb] in the staged row segment
//   bits 18..30 pair-ERI column tri(pb, qb) (< 8128 for n <= 128)
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
DG_HD int mixed_alpha_parity(Bits a_bra, int pa, int qa) {
    return popc(a_bra & open_bits(pa, qa)) & 1;
}

} // namespace detci_gpu
