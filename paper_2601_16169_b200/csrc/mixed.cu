// Mixed alpha-beta sigma term (matvec's mixed loop, matvec.cpp:193-219): the
// scatter kernel with its D reduction (default) and the gather kernel
// (DETCI_MIXED=gather), the work plans, and the multi-block column share.
#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
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
// Mixed alpha-beta kernel.  CTA = (output row ia, 2048 beta slots).  Stage =
// (alpha single ja of ia in the window, column segment g).  Two stage
// buffers, each [ +W | -W | Cs_0[ja, seg] | ... | Cs_{M-1}[ja, seg] ]; the
// next stage's row segments stream in with cp.async (and its W is built)
// while the current one is consumed:
//   W[cd] = (-1)^{popc(A_ia & open(pa,qa))} (pa qa|c d)
// (separated ordering: the whole alpha half of the sign is uniform over the
// stage), then each thread walks its beta strings' singles from the SELL-32
// table (one coalesced 4 B entry per element, shared by the M vectors)
// gathering W[cd] once and Cs_v[ja, jb] per vector from smem.  eps is
// applied once per output in the epilogue.
// ---------------------------------------------------------------------------

// beta slots per thread (1024 * R slots per CTA); M = 4 keeps 64 registers
template <int M>
struct MxR {
    static constexpr int value = 2;
};

struct MixedArgs {
    const double* C[kMaxM];
    size_t ldc;
    uint32_t c_row0, j0, j1;
    double* Y[kMaxM];
    size_t ldy;
    uint32_t row0, nrows, nb, nparts;
    const uint64_t* alpha;
    const uint64_t* beta_prefix;  // prefix_parity of the beta strings (eps)
    const uint32_t* sa_flat;
    const uint64_t* sa_off;
    const uint32_t* sa_len;
    const uint32_t* sell;
    const uint64_t* sell_off;
    const uint32_t* sell_len;
    const uint32_t* perm;     // slot -> beta string
    uint32_t seg_cols, nseg, nslices;
    const double* eri;
    int norbs;
};


// kDB: C stages double-buffered (row segments stream in under the compute of
// the previous stage); otherwise one C stage, refilled after a barrier (used
// when a whole row fits, which avoids segmenting the SELL table).
template <int M, bool kDB>
__global__ void __launch_bounds__(kMxBlock, 1)
k_mixed(const MixedArgs a) {
    constexpr int kMxR = MxR<M>::value;
    extern __shared__ double smem[];
    // layout: [ W buffer 0 | W buffer 1 | C stage 0 (M rows) | C stage 1 ]
    // W is double-buffered per alpha single (built once per ja), the C row
    // segments per stage = (ja, segment).
    const int nn = a.norbs * a.norbs;
    const uint32_t wdbl = static_cast<uint32_t>((2 * nn + 1) & ~1);
    const uint32_t segpad = (a.seg_cols + 1) & ~1u;
    double* const wbuf0 = smem;
    double* const cbuf0 = smem + 2 * wdbl;
    const uint32_t cstage = M * segpad;

    const uint32_t r = blockIdx.x / a.nparts;
    const uint32_t part = blockIdx.x % a.nparts;
    const uint32_t ia = a.row0 + r;
    const uint32_t tid = threadIdx.x;
    const uint32_t lane = tid % kWarp;
    const uint64_t A = a.alpha[ia];

    uint32_t slice[kMxR];
    double acc[M][kMxR];
#pragma unroll
    for (int q = 0; q < kMxR; ++q) {
        const uint32_t slot = part * (kMxBlock * kMxR) + q * kMxBlock + tid;
        slice[q] = slot / kWarp;
#pragma unroll
        for (int v = 0; v < M; ++v) acc[v][q] = 0.0;
    }

    const uint64_t o = a.sa_off[ia];
    const uint32_t n = a.sa_len[ia];
    const uint32_t* f = a.sa_flat + o;
    const uint32_t kb = a.j0 == 0 ? 0 : lower_bound_u32(f, n, a.j0);
    const uint32_t ke = lower_bound_u32(f, n, a.j1);
    const uint32_t nstages = (ke - kb) * a.nseg;

    // issue stage i: C row segments (async) into C buffer i & 1, and, on the
    // first segment of a new ja, +-W into W buffer (ja index) & 1
    auto issue = [&](uint32_t i) {
        const uint32_t kk = i / a.nseg, g = i % a.nseg;
        const uint32_t ja = f[kb + kk];
        const uint32_t segw = min(a.seg_cols, a.nb - g * a.seg_cols);
        const size_t src_off = static_cast<size_t>(ja - a.c_row0) * a.ldc + g * a.seg_cols;
        double* cb = cbuf0 + (kDB ? (i & 1) * cstage : 0);
#pragma unroll
        for (int v = 0; v < M; ++v) {
            double* crow = cb + v * segpad;
            const double* src = a.C[v] + src_off;
            for (uint32_t c = tid; c < segw; c += kMxBlock) cp_async8(crow + c, src + c);
        }
        cp_async_commit();
        if (g == 0) {
            double* wb = wbuf0 + (kk & 1) * wdbl;
            const uint64_t Ak = a.alpha[ja];
            const int pa = __ffsll(static_cast<long long>(A & ~Ak)) - 1;
            const int qa = __ffsll(static_cast<long long>(Ak & ~A)) - 1;
            const double* erow = a.eri + static_cast<size_t>(pa * a.norbs + qa) * nn;
            const uint32_t sA = static_cast<uint32_t>(mixed_alpha_parity(A, pa, qa));
            for (int cd = tid; cd < nn; cd += kMxBlock) {
                const int c = cd / a.norbs, d = cd - c * a.norbs;
                const double v = flip_sign(c != d ? erow[cd] : 0.0, sA);
                wb[cd] = v;
                wb[nn + cd] = -v;
            }
        }
    };

    if (kDB && nstages > 0) issue(0);
#pragma unroll 1
    for (uint32_t i = 0; i < nstages; ++i) {
        if (kDB) {
            if (i + 1 < nstages) {
                // C buffer (i+1)&1 was released by the barrier ending stage
                // i-1; W buffer ((i+1)/nseg)&1 differs from the one in use
                // when the next stage starts a new ja
                issue(i + 1);
                cp_async_wait_prev();  // stage i's rows have landed
            } else {
                cp_async_wait_all();
            }
        } else {
            issue(i);  // the barrier ending stage i-1 released the C buffer
            cp_async_wait_all();
        }
        __syncthreads();
        const uint32_t kk = i / a.nseg, g = i % a.nseg;
        const char* wbase = reinterpret_cast<const char*>(wbuf0 + (kk & 1) * wdbl);
        const char* cbase = reinterpret_cast<const char*>(cbuf0 + (kDB ? (i & 1) * cstage : 0));
        const uint32_t cstride = segpad * 8;  // bytes between the M staged rows
#pragma unroll
        for (int q = 0; q < kMxR; ++q) {
            if (slice[q] >= a.nslices) continue;
            const uint32_t L = a.sell_len[slice[q] * a.nseg + g];
            const uint32_t* ent = a.sell + a.sell_off[slice[q] * a.nseg + g] + lane;
            if (M == 1) {
                double s0 = 0.0, s1 = 0.0;
                uint32_t t = 0;
#pragma unroll 1
                for (; t + 8 <= L; t += 8) {
                    uint32_t e[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) e[u] = __ldg(ent + static_cast<size_t>(t + u) * kWarp);
#pragma unroll
                    for (int u = 0; u < 8; u += 2) {
                        const double w0 = *reinterpret_cast<const double*>(wbase + ((e[u] >> 18) << 3));
                        const double c0 = *reinterpret_cast<const double*>(cbase + (e[u] & 0x3ffffu));
                        const double w1 = *reinterpret_cast<const double*>(wbase + ((e[u + 1] >> 18) << 3));
                        const double c1 = *reinterpret_cast<const double*>(cbase + (e[u + 1] & 0x3ffffu));
                        s0 = fma(w0, c0, s0);
                        s1 = fma(w1, c1, s1);
                    }
                }
#pragma unroll 1
                for (; t < L; ++t) {
                    const uint32_t e0 = __ldg(ent + static_cast<size_t>(t) * kWarp);
                    s0 = fma(*reinterpret_cast<const double*>(wbase + ((e0 >> 18) << 3)),
                             *reinterpret_cast<const double*>(cbase + (e0 & 0x3ffffu)), s0);
                }
                acc[0][q] += s0 + s1;
            } else {
                // M independent FMA chains already; one accumulator per vector
                double s[M];
#pragma unroll
                for (int v = 0; v < M; ++v) s[v] = 0.0;
                uint32_t t = 0;
#pragma unroll 1
                for (; t + 8 <= L; t += 8) {
                    uint32_t e[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) e[u] = __ldg(ent + static_cast<size_t>(t + u) * kWarp);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const double w = *reinterpret_cast<const double*>(wbase + ((e[u] >> 18) << 3));
                        const char* c = cbase + (e[u] & 0x3ffffu);
#pragma unroll
                        for (int v = 0; v < M; ++v) s[v] = fma(w, *reinterpret_cast<const double*>(c + v * cstride), s[v]);
                    }
                }
#pragma unroll 1
                for (; t < L; ++t) {
                    const uint32_t e0 = __ldg(ent + static_cast<size_t>(t) * kWarp);
                    const double w = *reinterpret_cast<const double*>(wbase + ((e0 >> 18) << 3));
                    const char* c = cbase + (e0 & 0x3ffffu);
#pragma unroll
                    for (int v = 0; v < M; ++v) s[v] = fma(w, *reinterpret_cast<const double*>(c + v * cstride), s[v]);
                }
#pragma unroll
                for (int v = 0; v < M; ++v) acc[v][q] += s[v];
            }
        }
        __syncthreads();  // C buffer i&1 (and a finished W buffer) free
    }

#pragma unroll
    for (int q = 0; q < kMxR; ++q) {
        const uint32_t slot = part * (kMxBlock * kMxR) + q * kMxBlock + tid;
        if (slot < a.nb) {
            const uint32_t ib = a.perm[slot];
            const uint32_t flip = static_cast<uint32_t>(__popcll(A & a.beta_prefix[ib]));
            const size_t yi = static_cast<size_t>(r) * a.ldy + ib;
#pragma unroll
            for (int v = 0; v < M; ++v) a.Y[v][yi] += flip_sign(acc[v][q], flip);
        }
    }
}

// ---------------------------------------------------------------------------
// Scatter formulation of the mixed term (the default for M = 1).
//
// The gather kernel above spends two shared-memory gathers (W[cd] and
// Cs[ja, jb]) per FMA.  Turned around, one staged row Cs[ja, .] feeds every
// output row ia_k in the singles list of ja, and each gathered Cs[ja, jb]
// is reused for K of them:
//   D[ia_k, pos_k, ib] = sum_{jb in S(ib)} (-1)^{sb} V_k[cd(ib,jb)] Cs[ja, jb]
//   V_k[cd] = (-1)^{popc(A_k & open(pa,qa))} (pa qa|cd),  ia_k -> ja = pa -> qa
// so an element costs 1 + 1/K gathers instead of 2.  CTA = (item (ja, K
// consecutive entries of its list), 1024 beta slots); smem holds the K V rows
// and the row Cs[ja, .] (in segments when it does not fit).  Each partial is
// stored to its own slot of D (pos_k = position of ja in ia_k's list), and
// k_mixed_reduce sums D over the positions in ascending order, so the result
// is deterministic without atomics.
// ---------------------------------------------------------------------------
struct ScatterArgs {
    const double* C[2];         // Cs_v row ja at C[v] + (ja - c_row0) * ldc
    size_t ldc;
    uint32_t c_row0;
    const uint2* items;         // (ja, kbeg | cnt << 24)
    uint32_t nparts, nslices, nb, seg_cols, nseg, vpitch;
    const uint64_t* alpha;
    const uint64_t* alpha_hi;   // norbs > 64 (else null)
    const uint32_t* sa_flat;
    const uint64_t* sa_off;
    const uint32_t* tpos;
    const uint32_t* sell;
    const uint64_t* sell_off;
    const uint32_t* sell_len;
    const double* pair;         // pair-ERI matrix, rows of vpitch doubles
    double* D[2];               // D_v row (sa_off[ia] + pos - d_base), ldd slots
    uint64_t d_base;
    uint32_t ldd;
    uint32_t slot0, slot_end;   // beta slots [slot0, slot_end) (multi-GPU column share)
    const uint32_t* w_lo;       // ja-window D compaction (ScatterWindow::by_ja), or null
    const uint64_t* w_base;
};

// (V row offset | alpha sign << 63, D row) of output ia = list(ja)[pos].
// The V row of the alpha move pa -> qa is row tri(pa, qa) of the pair-ERI
// matrix: V[tri(pb, qb)] = (pa qa|pb qb).
__device__ __forceinline__ void scatter_row(const ScatterArgs& a, uint32_t ja, uint64_t oja, uint32_t pos,
                                            uint64_t& vr, uint64_t& dr) {
    const Bits Aj = load_bits(a.alpha, a.alpha_hi, ja);
    const uint32_t ia = a.sa_flat[oja + pos];
    const Bits Ak = load_bits(a.alpha, a.alpha_hi, ia);
    const int pa = lowest(Ak & ~Aj);
    const int qa = lowest(Aj & ~Ak);
    vr = static_cast<uint64_t>(tri_index(pa, qa)) * a.vpitch |
         static_cast<uint64_t>(mixed_alpha_parity(Ak, pa, qa)) << 63;
    dr = a.w_lo ? a.w_base[ia] + a.tpos[oja + pos] - a.w_lo[ia] : a.sa_off[ia] + a.tpos[oja + pos] - a.d_base;
}

// Entries of a CTA's run whose (V row, D row) are computed once up front
// (one latency for all passes instead of one per pass).
constexpr uint32_t kRunPre = 256;

// Staging of one Cs row segment (doubles [g * seg_cols, + segw) of row ja,
// vector v) into its smem slot by 1-D TMA: the 16-byte aligned interior by
// one bulk copy (issued by the elected thread, completing on `bar`), the
// unaligned first / last double by plain stores.  The smem row is shifted
// by one double when the source starts at 8 mod 16 so that source and
// destination stay congruent; returns that shift.
__device__ __forceinline__ uint32_t seg_shift(const double* src) {
    return static_cast<uint32_t>((reinterpret_cast<uintptr_t>(src) >> 3) & 1u);
}
// bytes the elected thread's bulk copy of the segment moves
__device__ __forceinline__ uint32_t seg_bulk_bytes(const double* src, uint32_t segw) {
    const uintptr_t s = reinterpret_cast<uintptr_t>(src), e = s + static_cast<uintptr_t>(segw) * 8;
    const uintptr_t s0 = (s + 15) & ~uintptr_t{15}, e0 = e & ~uintptr_t{15};
    return e0 > s0 ? static_cast<uint32_t>(e0 - s0) : 0u;
}
__device__ __forceinline__ void seg_issue(double* dst, const double* src, uint32_t segw, uint64_t* bar) {
    const uint32_t sh = seg_shift(src);
    const uint32_t bytes = seg_bulk_bytes(src, segw);
    if (bytes) bulk_g2s(dst + sh + sh, src + sh, bytes, bar);   // element i at dst + sh + i
}
// The doubles outside the bulk copy (at most one at each end) by plain
// stores, and the zero slot the padding entries read (element seg_cols of
// the shifted row; never overlaps the copy, segpad >= seg_cols + 2).
__device__ __forceinline__ void seg_edges(double* dst, const double* src, uint32_t segw, uint32_t seg_cols,
                                          uint32_t t) {
    const uint32_t sh = seg_shift(src);
    const uint32_t bytes = seg_bulk_bytes(src, segw);
    const uint32_t first = sh, last = first + bytes / 8;   // bulk covers [first, last)
    if (t == 0) {
        if (first > 0 && segw > 0) dst[sh] = src[0];
        dst[sh + seg_cols] = 0.0;
    }
    if (t == 1)
        for (uint32_t i = (bytes ? last : first); i < segw; ++i) dst[sh + i] = src[i];
}

// One pass of the scatter CTA: K output rows ia_k = list(ja)[kbeg + k], k <
// cnt (rows cnt..K-1 padded: computed, never stored).  The elected thread
// stages the pass's K V rows (pair-ERI rows, one 1-D TMA bulk copy each) and,
// unless the whole row is already resident (`staged`), the Cs row segments,
// all completing on the CTA's mbarrier; every thread then walks its SELL
// entries (one 4-byte entry per element, prefetched a batch ahead) and
// stores its K partials.  M = 1 or 2 vectors share the V gathers (the
// multi-root block's pairs): an element costs (M + K) / (M K) gathers per
// FMA.
template <int K, int M>
__device__ __forceinline__ void scatter_pass(const ScatterArgs& a, double* vsub, double* cseg, uint64_t* s_vrow,
                                             uint64_t* s_drow, uint64_t* bar, uint32_t& phase, uint32_t ja,
                                             uint64_t oja, uint32_t kbeg, uint32_t cnt, bool staged, bool stage_row,
                                             uint32_t part, bool precomputed) {
    const uint32_t tid = threadIdx.x, lane = tid % kWarp;
    const uint32_t segpad = scatter_segpad(a.seg_cols);
    const size_t crow = static_cast<size_t>(ja - a.c_row0) * a.ldc;
    const uint32_t vbytes = a.vpitch * 8;
    __syncthreads();   // the previous pass is done with V, the row tables and the segment
    if (!precomputed) {
        if (tid < K) {
            uint64_t vr = ~0ull, dr = 0;
            if (tid < cnt) scatter_row(a, ja, oja, kbeg + tid, vr, dr);
            s_vrow[tid] = vr;
            s_drow[tid] = dr;
        }
        __syncthreads();
    }
    // segment g of vector v: source and smem slot
    auto seg_src = [&](int v, uint32_t g) { return a.C[v] + crow + static_cast<size_t>(g) * a.seg_cols; };
    auto seg_w = [&](uint32_t g) { return min(a.seg_cols, a.nb - g * a.seg_cols); };
    // elected thread: V rows of this pass (+ segment 0, or the whole row on
    // the CTA's first pass), one arrive with the byte count
    if (tid == 0) {
        fence_proxy_async_smem();   // the CTA's reads of the old V / segment precede the new writes
        uint32_t bytes = static_cast<uint32_t>(K) * vbytes;
        const bool seg0 = stage_row || !staged;
        if (seg0)
            for (int v = 0; v < M; ++v) bytes += seg_bulk_bytes(seg_src(v, 0), seg_w(0));
        mbar_arrive_expect_tx(bar, bytes);
        for (int k = 0; k < K; ++k) {
            const uint64_t vr = s_vrow[k < static_cast<int>(cnt) ? k : 0];
            bulk_g2s(vsub + k * a.vpitch, a.pair + (vr & 0x7fffffffffffffffull), vbytes, bar);
        }
        if (seg0)
            for (int v = 0; v < M; ++v) seg_issue(cseg + v * segpad, seg_src(v, 0), seg_w(0), bar);
    }
    if ((stage_row || !staged) && tid < 2)
        for (int v = 0; v < M; ++v) seg_edges(cseg + v * segpad, seg_src(v, 0), seg_w(0), a.seg_cols, tid);

    const uint32_t slot = a.slot0 + part * kMxBlock + tid;
    const uint32_t sl = slot / kWarp;
    const bool active = sl < a.nslices && slot < a.slot_end;
    double acc[M][K];
#pragma unroll
    for (int v = 0; v < M; ++v)
#pragma unroll
        for (int k = 0; k < K; ++k) acc[v][k] = 0.0;
    const char* vb = reinterpret_cast<const char*>(vsub);
    const uint32_t vstride = a.vpitch * 8;

#pragma unroll 1
    for (uint32_t g = 0; g < a.nseg; ++g) {
        if (g > 0) {
            __syncthreads();   // previous segment consumed
            if (tid == 0) {
                fence_proxy_async_smem();
                uint32_t bytes = 0;
                for (int v = 0; v < M; ++v) bytes += seg_bulk_bytes(seg_src(v, g), seg_w(g));
                mbar_arrive_expect_tx(bar, bytes);
                for (int v = 0; v < M; ++v) seg_issue(cseg + v * segpad, seg_src(v, g), seg_w(g), bar);
            }
            if (tid < 2)
                for (int v = 0; v < M; ++v) seg_edges(cseg + v * segpad, seg_src(v, g), seg_w(g), a.seg_cols, tid);
        }
        const bool fresh = g > 0 || stage_row || !staged;   // this segment was (re)staged just now
        mbar_wait(bar, phase);   // V rows (g == 0) and the segment's bulk bytes landed
        phase ^= 1u;
        if (fresh) __syncthreads();   // plain-store edges and zero slot visible
        if (!active) continue;
        // per vector: the staged row starts one double in when its source
        // was misaligned (seg_shift)
        const char* cbv[M];
#pragma unroll
        for (int v = 0; v < M; ++v)
            cbv[v] = reinterpret_cast<const char*>(cseg + v * segpad + seg_shift(seg_src(v, g)));
        auto element = [&](uint32_t e) {
            const uint32_t co = e & 0x3ffffu;
            double c[M];
#pragma unroll
            for (int v = 0; v < M; ++v)
                c[v] = xor_sign(*reinterpret_cast<const double*>(cbv[v] + co), e & 0x80000000u);
            const char* vp = vb + ((e >> 15) & 0xfff8u);
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const double w = *reinterpret_cast<const double*>(vp + k * vstride);
#pragma unroll
                for (int v = 0; v < M; ++v) acc[v][k] = fma(w, c[v], acc[v][k]);
            }
        };
        const uint32_t L = a.sell_len[sl * a.nseg + g];
        const uint32_t* ent = a.sell + a.sell_off[sl * a.nseg + g] + lane;
        uint32_t t = 0;
        if (L >= 4) {
            // batches of 4 entries, the next batch's loads in flight while
            // the current one is consumed
            uint32_t e[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) e[u] = __ldg(ent + static_cast<size_t>(u) * kWarp);
#pragma unroll 1
            for (; t + 8 <= L; t += 4) {
                uint32_t nx[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) nx[u] = __ldg(ent + static_cast<size_t>(t + 4 + u) * kWarp);
#pragma unroll
                for (int u = 0; u < 4; ++u) element(e[u]);
#pragma unroll
                for (int u = 0; u < 4; ++u) e[u] = nx[u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) element(e[u]);
            t += 4;
        }
#pragma unroll 1
        for (; t < L; ++t) element(__ldg(ent + static_cast<size_t>(t) * kWarp));
    }
    if (!active) return;
#pragma unroll
    for (int k = 0; k < K; ++k)
        if (k < static_cast<int>(cnt)) {
            const uint32_t sgn = static_cast<uint32_t>(s_vrow[k] >> 63);
#pragma unroll
            for (int v = 0; v < M; ++v) a.D[v][s_drow[k] * a.ldd + (slot - a.slot0)] = flip_sign(acc[v][k], sgn);
        }
}

// CTA = (item = (ja, a run of len entries of its singles list), 1024 beta
// slots).  The row Cs[ja, .] is staged once when it fits whole (nseg == 1)
// and serves every pass: full passes of KMAX output rows, then one padded
// remainder pass of the next power of two >= the rest.  All staging is 1-D
// TMA (cp.async.bulk) issued by one thread and completing on one mbarrier
// (one phase per pass and segment).
template <int KMAX, int M>
__global__ void __launch_bounds__(kMxBlock, 1)
k_mixed_scatter(const ScatterArgs a) {
    extern __shared__ __align__(16) double smem[];
    double* const vsub = smem;                      // KMAX rows of vpitch
    double* const cseg = smem + KMAX * a.vpitch;    // Cs_v[ja, segment], v < M (scatter_segpad each)
    __shared__ uint64_t s_vrow[KMAX];               // pair row offset | sign << 63 (runs past kRunPre)
    __shared__ uint64_t s_drow[KMAX];               // D row of output k
    __shared__ uint64_t s_vall[kRunPre], s_dall[kRunPre];   // the run's first kRunPre rows
    __shared__ uint64_t bar;

    const uint32_t item = blockIdx.x / a.nparts, part = blockIdx.x % a.nparts;
    const uint2 it = a.items[item];
    const uint32_t ja = it.x, kbeg = it.y & 0xfffffu, len = it.y >> 20;
    const uint64_t oja = a.sa_off[ja];
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    for (uint32_t t = threadIdx.x; t < min(len, kRunPre); t += kMxBlock) {
        uint64_t vr, dr;
        scatter_row(a, ja, oja, kbeg + t, vr, dr);
        s_vall[t] = vr;
        s_dall[t] = dr;
    }   // visible after the first pass's barrier
    const bool whole = a.nseg == 1;
    uint32_t phase = 0;
    uint32_t p = kbeg;
    const uint32_t end = kbeg + len;
    // row tables of a pass: the precomputed slice, or s_vrow/s_drow
    auto tabs = [&](uint32_t pp, uint32_t k, uint64_t*& v, uint64_t*& d) {
        const bool pre = pp - kbeg + k <= kRunPre;
        v = pre ? s_vall + (pp - kbeg) : s_vrow;
        d = pre ? s_dall + (pp - kbeg) : s_drow;
        return pre;
    };
    uint64_t *tv, *td;
    bool first = true;
#pragma unroll 1
    for (; p + KMAX <= end; p += KMAX) {
        const bool pre = tabs(p, KMAX, tv, td);
        scatter_pass<KMAX, M>(a, vsub, cseg, tv, td, &bar, phase, ja, oja, p, KMAX, whole && !first,
                              whole && first, part, pre);
        first = false;
    }
    const uint32_t r = end - p;
    if (r == 0) return;
    const bool pre = tabs(p, r, tv, td);
    const bool st = whole && !first, sr = whole && first;
    if constexpr (KMAX > 8) { if (r > 8) { scatter_pass<16, M>(a, vsub, cseg, tv, td, &bar, phase, ja, oja, p, r, st, sr, part, pre); return; } }
    if constexpr (KMAX > 4) { if (r > 4) { scatter_pass<8, M>(a, vsub, cseg, tv, td, &bar, phase, ja, oja, p, r, st, sr, part, pre); return; } }
    if constexpr (KMAX > 2) { if (r > 2) { scatter_pass<4, M>(a, vsub, cseg, tv, td, &bar, phase, ja, oja, p, r, st, sr, part, pre); return; } }
    if constexpr (KMAX > 1) { if (r > 1) { scatter_pass<2, M>(a, vsub, cseg, tv, td, &bar, phase, ja, oja, p, r, st, sr, part, pre); return; } }
    scatter_pass<1, M>(a, vsub, cseg, tv, td, &bar, phase, ja, oja, p, r, st, sr, part, pre);
}

// y[ia, ib] += eps(A_ia, B_ib) sum_{pos in [lo, hi)} D[sa_off[ia] + pos - d_base, slot]
// with [lo, hi) the positions of the held block's ja in ia's singles list,
// summed in ascending order (deterministic).  CTA = (row, 256 slots).
struct ReduceArgs {
    const double* D;
    uint64_t d_base;
    uint32_t ldd, nb, nparts;
    uint32_t i_lo, j0, j1;
    const uint32_t* sa_flat;
    const uint64_t* sa_off;
    const uint32_t* sa_len;
    const uint64_t* alpha;
    const uint64_t* beta_prefix;
    const uint64_t* alpha_hi;         // norbs > 64 (else null)
    const uint64_t* beta_prefix_hi;
    const uint32_t* perm;
    double* Y;                  // row ia at Y + (ia - y_row0) * ldy (accumulate, by perm)
    size_t ldy;
    uint32_t y_row0;
    uint32_t slot0, slot_end;   // slots [slot0, slot_end); D column = slot - slot0
    double* T;                  // if set: T[(ia - y_row0) * ldt + slot - slot0] = result (slot order)
    size_t ldt;
    int t_accumulate;           // T += instead of = (later ja windows)
    const uint32_t* w_lo;       // ja-window D compaction, or null
    const uint64_t* w_base;
};

constexpr int kRedBlock = 256;

__global__ void __launch_bounds__(kRedBlock)
k_mixed_reduce(const ReduceArgs a) {
    __shared__ uint32_t s_rng[2];
    const uint32_t ia = a.i_lo + blockIdx.x / a.nparts;
    const uint32_t slot = a.slot0 + (blockIdx.x % a.nparts) * kRedBlock + threadIdx.x;
    const uint64_t o = a.sa_off[ia];
    if (a.w_lo) {   // ja window: the positions and D rows come compacted
        if (threadIdx.x == 0) {
            s_rng[0] = a.w_lo[ia];
            s_rng[1] = a.w_lo[ia] + static_cast<uint32_t>(a.w_base[ia + 1] - a.w_base[ia]);
        }
    } else if (threadIdx.x < 2) {
        const uint32_t* f = a.sa_flat + o;
        s_rng[threadIdx.x] = lower_bound_u32(f, a.sa_len[ia], threadIdx.x == 0 ? a.j0 : a.j1);
    }
    __syncthreads();
    if (slot >= a.nb || slot >= a.slot_end) return;
    const uint32_t lo = s_rng[0], hi = s_rng[1];
    if (lo == hi && (!a.T || a.t_accumulate)) return;
    const uint64_t drow = a.w_lo ? a.w_base[ia] : o + lo - a.d_base;
    const double* d = a.D + drow * a.ldd + (slot - a.slot0);
    double s = 0.0;
    uint32_t p = lo;
#pragma unroll 1
    for (; p + 8 <= hi; p += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(d + static_cast<size_t>(p - lo + u) * a.ldd);
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; p < hi; ++p) s += __ldcs(d + static_cast<size_t>(p - lo) * a.ldd);
    const uint32_t ib = a.perm[slot];
    const uint32_t flip = static_cast<uint32_t>(
        eps_parity(load_bits(a.alpha, a.alpha_hi, ia), load_bits(a.beta_prefix, a.beta_prefix_hi, ib)));
    if (a.T) {
        double& t = a.T[static_cast<size_t>(ia - a.y_row0) * a.ldt + (slot - a.slot0)];
        t = a.t_accumulate ? t + flip_sign(s, flip) : flip_sign(s, flip);
    } else {
        a.Y[static_cast<size_t>(ia - a.y_row0) * a.ldy + ib] += flip_sign(s, flip);
    }
}

// y[r * ldy + perm[s]] += R[r * ldr + s], s < ns (perm already offset to the
// source's first slot): the column-partitioned mixed term back into rows.
__global__ void k_unpack_mixed(const double* __restrict__ R, size_t ldr, uint32_t ns, uint32_t rows,
                               const uint32_t* __restrict__ perm, double* __restrict__ y, size_t ldy) {
    const uint32_t r = blockIdx.y;
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += gridDim.x * blockDim.x)
        if (r < rows) y[static_cast<size_t>(r) * ldy + perm[s]] += R[static_cast<size_t>(r) * ldr + s];
}

} // namespace

size_t mixed_smem(const Handle& h, const SellTable& t, int M) {
    const size_t nn = static_cast<size_t>(h.norbs) * h.norbs;
    const size_t w = (2 * nn + 1) & ~size_t{1}, c = M * ((t.seg_cols + 1) & ~size_t{1});
    return (2 * w + (t.double_buffer ? 2 : 1) * c) * sizeof(double);   // 2 W buffers + 1 or 2 C stages
}

template <int M>
void launch_mixed(Handle& h, const Ptrs& Cb, uint32_t b0, uint32_t b1, const MPtrs& y_loc, uint64_t a0,
                  uint64_t a1) {
    const SellTable& t = mixed_table(h, M);
    MixedArgs m{};
    for (int v = 0; v < M; ++v) {
        m.C[v] = Cb[v];
        m.Y[v] = y_loc[v];
    }
    m.ldc = h.nb();
    m.c_row0 = b0;
    m.j0 = b0;
    m.j1 = b1;
    m.ldy = h.nb();
    m.row0 = static_cast<uint32_t>(a0);
    m.nrows = static_cast<uint32_t>(a1 - a0);
    m.nb = static_cast<uint32_t>(h.nb());
    m.nparts = (m.nb + kMxBlock * MxR<M>::value - 1) / (kMxBlock * MxR<M>::value);
    m.alpha = h.ch[0].strings.p;
    m.beta_prefix = h.ch[1].prefix.p;
    m.sa_flat = h.ch[0].flat[0].p;
    m.sa_off = h.ch[0].offset[0].p;
    m.sa_len = h.ch[0].len[0].p;
    m.sell = t.sell.p;
    m.sell_off = t.off.p;
    m.sell_len = t.len.p;
    m.perm = h.sell_perm.p;
    m.seg_cols = t.seg_cols;
    m.nseg = t.nseg;
    m.nslices = h.nslices;
    m.eri = h.d_eri.p;
    m.norbs = h.norbs;
    if (m.nrows == 0) return;
    const size_t smem = mixed_smem(h, t, M);
    const int db = t.double_buffer ? 1 : 0;
    if (db) ensure_dynamic_smem(reinterpret_cast<const void*>(k_mixed<M, true>), smem);
    else ensure_dynamic_smem(reinterpret_cast<const void*>(k_mixed<M, false>), smem);
    const uint64_t grid = static_cast<uint64_t>(m.nrows) * m.nparts;
    if (db)
        k_mixed<M, true><<<static_cast<unsigned>(grid), kMxBlock, smem, h.stream>>>(m);
    else
        k_mixed<M, false><<<static_cast<unsigned>(grid), kMxBlock, smem, h.stream>>>(m);
    CUDA_LAUNCH_CHECK();
}


// D row stride (slots): all slots, or under the multi-block gather schedule
// the largest per-rank column share.
uint32_t mixed_ldd(const Handle& h) {
    const int P = std::max(h.world, h.vblocks);
    if (P == 1 || multi_ring()) return h.nslices * kWarp;
    uint32_t m = 0;
    for (int g = 0; g < P; ++g) {
        const auto [s0, s1] = mixed_slots(h, g, P);
        m = std::max(m, s1 - s0);
    }
    return m;
}

// Scatter plan for block-rank g (rows [blk[g], blk[g+1])): output windows
// whose D fits the capacity, and per window, K grid (kmax 16 or 8) and alpha
// block the CTA items.  D capacity: DETCI_MIXED_DBYTES if set (tests force
// several windows), else 60% of the free device memory at the first sigma,
// shared by the M vectors of a pass (release_sigma_scratch re-plans after
// the Davidson solvers allocate their subspace, and a pass with more vectors
// than the plan reserved for re-plans).
const std::vector<std::unique_ptr<ScatterWindow>>& scatter_windows(Handle& h, int g, int P, int M, int kmax) {
    const uint64_t ldd = mixed_ldd(h);
    if (h.dplan_m != 0 && h.dplan_m < M) release_sigma_scratch(h);
    if (h.scatter_plan.size() != static_cast<size_t>(P)) {
        h.scatter_plan.clear();
        h.scatter_plan.resize(P);
    }
    const uint64_t* off = h.h_sa_off.data();
    const uint32_t* flat = h.h_sa_flat.data();
    if (h.dcap_rows == 0) {
        size_t fr = 0, tot = 0;
        CUDA_CHECK(cudaMemGetInfo(&fr, &tot));
        uint64_t bytes = static_cast<uint64_t>(0.6 * static_cast<double>(fr + h.dbuf.bytes()));
        if (const char* e = std::getenv("DETCI_MIXED_DBYTES")) bytes = std::strtoull(e, nullptr, 10);
        h.dbuf.reset();
        uint64_t maxlen = 1;
        for (size_t i = 0; i < h.na(); ++i) maxlen = std::max<uint64_t>(maxlen, off[i + 1] - off[i]);
        h.dcap_rows = std::max<uint64_t>(bytes / (ldd * 8 * M), maxlen);
        h.dplan_m = M;
    }
    auto& wins = h.scatter_plan[g];
    if (wins.empty() && P == 1) {
        // P == 1 (also the gather schedule's column share on a multi-block
        // handle): all output rows; windows cut the ja range, so every item
        // keeps its whole list
        const uint64_t na = h.na();
        uint64_t j = 0;
        while (j < na) {
            auto w = std::make_unique<ScatterWindow>();
            w->j0 = j;
            uint64_t rows = 0;
            while (j < na && (j == w->j0 || rows + (off[j + 1] - off[j]) <= h.dcap_rows)) {
                rows += off[j + 1] - off[j];
                ++j;
            }
            w->j1 = j;
            w->i_lo = 0;
            w->i_hi = na;
            w->d_base = 0;
            w->d_rows = rows;
            w->by_ja = !(w->j0 == 0 && w->j1 == na);
            if (w->by_ja) {
                std::vector<uint32_t> lo(na);
                std::vector<uint64_t> base(na + 1, 0);
                for (uint64_t ia = 0; ia < na; ++ia) {
                    const uint32_t* f = flat + off[ia];
                    const uint32_t* e = flat + off[ia + 1];
                    const uint32_t l = static_cast<uint32_t>(std::lower_bound(f, e, static_cast<uint32_t>(w->j0)) - f);
                    const uint32_t hgh = static_cast<uint32_t>(std::lower_bound(f, e, static_cast<uint32_t>(w->j1)) - f);
                    lo[ia] = l;
                    base[ia + 1] = base[ia] + (hgh - l);
                }
                if (base[na] != rows) fail(DETCI_GPU_E_CUDA, "mixed term: singles lists are not mutual");
                w->lo.alloc(na);
                w->base.alloc(na + 1);
                copy_sync(w->lo.p, lo.data(), na * 4, cudaMemcpyHostToDevice, h.stream);
                copy_sync(w->base.p, base.data(), (na + 1) * 8, cudaMemcpyHostToDevice, h.stream);
            }
            wins.push_back(std::move(w));
        }
    }
    if (wins.empty()) {
        // block-rank of the ring schedule: windows over the rank's output rows
        const uint64_t r0 = h.blk[g], r1 = h.blk[g + 1];
        uint64_t i = r0;
        while (i < r1) {
            auto w = std::make_unique<ScatterWindow>();
            w->i_lo = i;
            while (i < r1 && (i == w->i_lo || off[i + 1] - off[w->i_lo] <= h.dcap_rows)) ++i;
            w->i_hi = i;
            w->d_base = off[w->i_lo];
            w->d_rows = off[w->i_hi] - w->d_base;
            wins.push_back(std::move(w));
        }
    }
    const int ki = __builtin_ctz(static_cast<unsigned>(kmax));   // items depend on kmax
    for (auto& w : wins) {
        if (!w->item_off[ki].empty()) continue;
        // one item per ja: the run of its (window-restricted) singles list;
        // the CTA cuts it into passes of kmax and a padded remainder
        std::vector<uint2> items;
        w->item_off[ki].assign(static_cast<size_t>(P) + 1, 0);
        for (int b = 0; b < P; ++b) {
            w->item_off[ki][b] = items.size();
            const uint64_t j0 = P == 1 ? w->j0 : h.blk[b], j1 = P == 1 ? w->j1 : h.blk[b + 1];
            for (uint64_t ja = j0; ja < j1; ++ja) {
                const uint32_t* f = flat + off[ja];
                const uint32_t* e = flat + off[ja + 1];
                const uint32_t p_lo = P == 1 ? 0u : static_cast<uint32_t>(std::lower_bound(f, e, static_cast<uint32_t>(w->i_lo)) - f);
                const uint32_t p_hi = P == 1 ? static_cast<uint32_t>(e - f)
                                             : static_cast<uint32_t>(std::lower_bound(f, e, static_cast<uint32_t>(w->i_hi)) - f);
                if (p_hi > p_lo) {
                    if (p_hi - p_lo >= (1u << 12) || p_lo >= (1u << 20))
                        fail(DETCI_GPU_E_UNSUPPORTED, "mixed term: singles list too long for the item encoding");
                    items.push_back(make_uint2(static_cast<uint32_t>(ja), p_lo | (p_hi - p_lo) << 20));
                }
            }
        }
        w->item_off[ki][P] = items.size();
        w->items[ki].alloc(std::max<size_t>(items.size(), 1));
        if (!items.empty())
            copy_sync(w->items[ki].p, items.data(), items.size() * sizeof(uint2), cudaMemcpyHostToDevice, h.stream);
    }
    uint64_t need = 0;
    for (auto& w : wins) need = std::max(need, w->d_rows);
    if (h.dbuf.n < need * ldd * M) h.dbuf.alloc(need * ldd * M);
    return wins;
}

template <int KMAX, int M>
void launch_scatter_k(const ScatterArgs& a, uint64_t grid, uint32_t vpitch, size_t cbytes, cudaStream_t st) {
    const size_t smem = static_cast<size_t>(KMAX) * vpitch * sizeof(double) + M * cbytes;
    if (smem > kScatterSmem) fail(DETCI_GPU_E_CUDA, "mixed term: scatter plan exceeds shared memory");
    ensure_dynamic_smem(reinterpret_cast<const void*>(k_mixed_scatter<KMAX, M>), smem);
    k_mixed_scatter<KMAX, M><<<static_cast<unsigned>(grid), kMxBlock, smem, st>>>(a);
    CUDA_LAUNCH_CHECK();
}


// Mixed term through the scatter kernel for block-rank g, held alpha block
// b = rows [b0, b1) of Cs in Cb, outputs rows [a0, a1) of y_loc.
// phases: 1 = scatter kernels only, 2 = D reduction only (of output rows
// [r_lo, r_hi) within each window), 3 = both (per window).
template <int M>
void launch_mixed_scatter(Handle& h, int g, int P, int b, const Ptrs& Cb, uint32_t b0, uint32_t b1,
                          const MPtrs& y_loc, uint64_t a0, int phases, uint64_t r_lo, uint64_t r_hi,
                          int only_window, const MixedTarget& tgt) {
    const SellTable& t = scatter_table(h, M);
    const auto& wins = scatter_windows(h, g, P, M, t.kmax);
    const int ki = __builtin_ctz(static_cast<unsigned>(t.kmax));
    const uint32_t ldd = mixed_ldd(h);
    const uint32_t vpitch = scatter_vpitch(h.norbs);
    const size_t cbytes = scatter_segpad(t.seg_cols) * sizeof(double);   // + shift and zero slot
    for (size_t wi = 0; wi < wins.size(); ++wi) {
        if (only_window >= 0 && static_cast<size_t>(only_window) != wi) continue;
        const auto& w = wins[wi];
        const auto& io = w->item_off[ki];
        const uint64_t i0 = io[b], i1 = io[b + 1];
        if (i1 == i0) continue;
        ScatterArgs a{};
        for (int v = 0; v < M; ++v) {
            a.C[v] = Cb[v];
            a.D[v] = h.dbuf.p + static_cast<size_t>(v) * w->d_rows * ldd;
        }
        a.ldc = h.nb();
        a.c_row0 = b0;
        a.nslices = h.nslices;
        a.nb = static_cast<uint32_t>(h.nb());
        a.seg_cols = t.seg_cols;
        a.nseg = t.nseg;
        a.vpitch = vpitch;
        a.alpha = h.ch[0].strings.p;
        a.alpha_hi = h.ch[0].hi();
        a.sa_flat = h.ch[0].flat[0].p;
        a.sa_off = h.ch[0].offset[0].p;
        a.tpos = h.tpos.p;
        a.sell = t.sell.p;
        a.sell_off = t.off.p;
        a.sell_len = t.len.p;
        a.pair = h.d_pair.p;
        a.d_base = w->d_base;
        a.ldd = ldd;
        a.w_lo = w->by_ja ? w->lo.p : nullptr;
        a.w_base = w->by_ja ? w->base.p : nullptr;
        a.slot0 = tgt.slot0;
        a.slot_end = std::min<uint32_t>(tgt.slot_end, h.nslices * kWarp);
        if (a.slot_end <= a.slot0) return;   // empty column share (more ranks than slices)
        if (a.slot_end - a.slot0 > ldd) fail(DETCI_GPU_E_CUDA, "mixed term: slot share exceeds the D stride");
        a.nparts = (a.slot_end - a.slot0 + kMxBlock - 1) / kMxBlock;
        if (phases & 1) {
            a.items = w->items[ki].p + i0;
            const uint64_t grid = (i1 - i0) * a.nparts;
            if (grid >= (1ull << 31)) fail(DETCI_GPU_E_UNSUPPORTED, "mixed term: scatter grid too large");
            switch (t.kmax) {
                case 16: launch_scatter_k<16, 1>(a, grid, vpitch, cbytes, h.stream); break;   // kmax 16 => M == 1
                case 8: launch_scatter_k<8, M>(a, grid, vpitch, cbytes, h.stream); break;
                case 4: launch_scatter_k<4, M>(a, grid, vpitch, cbytes, h.stream); break;
                case 2: launch_scatter_k<2, M>(a, grid, vpitch, cbytes, h.stream); break;
                default: launch_scatter_k<1, M>(a, grid, vpitch, cbytes, h.stream); break;
            }
        }

        const uint64_t lo = std::max<uint64_t>(w->i_lo, r_lo), hi = std::min<uint64_t>(w->i_hi, r_hi);
        for (int v = 0; v < M && (phases & 2) && lo < hi; ++v) {
            ReduceArgs r{};
            r.D = a.D[v];
            r.d_base = w->d_base;
            r.ldd = ldd;
            r.nb = a.nb;
            r.slot0 = a.slot0;
            r.slot_end = std::min<uint32_t>(a.slot_end, a.nb);
            r.nparts = (r.slot_end - r.slot0 + kRedBlock - 1) / kRedBlock;
            r.T = tgt.T[v];
            r.ldt = tgt.ldt;
            r.t_accumulate = wi > 0 ? 1 : 0;
            r.w_lo = a.w_lo;
            r.w_base = a.w_base;
            r.i_lo = static_cast<uint32_t>(lo);
            r.j0 = b0;
            r.j1 = b1;
            r.sa_flat = a.sa_flat;
            r.sa_off = a.sa_off;
            r.sa_len = h.ch[0].len[0].p;
            r.alpha = a.alpha;
            r.beta_prefix = h.ch[1].prefix.p;
            r.alpha_hi = a.alpha_hi;
            r.beta_prefix_hi = h.ch[1].prefix_hi_p();
            r.perm = h.sell_perm.p;
            r.Y = y_loc[v];
            r.ldy = h.nb();
            r.y_row0 = static_cast<uint32_t>(a0);
            const uint64_t rgrid = (hi - lo) * r.nparts;
            const int tid = h.timer ? h.timer->begin(4) : -1;
            k_mixed_reduce<<<static_cast<unsigned>(rgrid), kRedBlock, 0, h.stream>>>(r);
            CUDA_LAUNCH_CHECK();
            if (h.timer) h.timer->end(tid);
        }
    }
}

bool multi_ring() {
    const char* e = std::getenv("DETCI_MULTI");
    return e && std::string(e) == "ring";
}

// Beta slots of the mixed term owned by block-rank g (32-slot aligned),
// cut on the prefix of the scatter work per slice: the slots are sorted by
// descending singles degree, so equal slot counts would give rank 0 the
// heaviest strings (1.5x the mean at C3 / P = 8).
std::pair<uint32_t, uint32_t> mixed_slots(const Handle& h, int g, int P) {
    const uint64_t total = static_cast<uint64_t>(h.nslices) * kWarp;
    if (h.slot_cut.size() == static_cast<size_t>(P) + 1) return {h.slot_cut[g], h.slot_cut[g + 1]};
    const auto& pre = h.slice_prefix;
    const bool weighted = pre.size() == static_cast<size_t>(h.nslices) + 1 && pre.back() > 0;
    auto at = [&](int k) -> uint32_t {
        if (k <= 0) return 0;
        if (k >= P) return static_cast<uint32_t>(total);
        if (!weighted) return static_cast<uint32_t>(total * k / P / kWarp * kWarp);
        const double target = static_cast<double>(pre.back()) * k / P;
        const size_t s = std::lower_bound(pre.begin(), pre.end(), target,
                                          [](uint64_t v, double t) { return static_cast<double>(v) < t; }) -
                         pre.begin();
        return static_cast<uint32_t>(std::min<uint64_t>(s * kWarp, total));
    };
    return {at(g), at(g + 1)};
}

// Unpack a column slab of slots [s0, s0 + ns): only slots < nb are real
// (the last slice is padded to 32).
template <int M>
void unpack_slab(Handle& h, const double* R, size_t ldr, uint32_t ns, uint64_t rows, uint32_t s0, double* y) {
    ns = static_cast<uint32_t>(std::min<uint64_t>(ns, h.nb() > s0 ? h.nb() - s0 : 0));
    if (rows == 0 || ns == 0) return;
    for (uint64_t r0 = 0; r0 < rows; r0 += 65535) {
        const uint32_t rr = static_cast<uint32_t>(std::min<uint64_t>(65535, rows - r0));
        dim3 grid((ns + 255) / 256, rr);
        k_unpack_mixed<<<grid, 256, 0, h.stream>>>(R + r0 * ldr, ldr, ns, rr, h.sell_perm.p + s0, y + r0 * h.nb(),
                                                   h.nb());
        CUDA_LAUNCH_CHECK();
    }
}

// Mixed term of block-rank g, column-partitioned: all alpha rows (Cs whole
// in Cfull), beta slots of g, result (eps applied) into T (na x ldt, slot
// order).
template <int M>
void mixed_columns(Handle& h, int g, int P, const Ptrs& Cfull, double* const* T, size_t ldt) {
    const auto [s0, s1] = mixed_slots(h, g, P);
    MixedTarget tgt;
    tgt.slot0 = s0;
    tgt.slot_end = s1;
    tgt.ldt = ldt;
    for (int v = 0; v < M; ++v) tgt.T[v] = T[v];
    MPtrs none{};
    launch_mixed_scatter<M>(h, 0, 1, 0, Cfull, 0, static_cast<uint32_t>(h.na()), none, 0, 3, 0, ~0ull, -1, tgt);
}


template void launch_mixed<1>(Handle&, const Ptrs&, uint32_t, uint32_t, const MPtrs&, uint64_t, uint64_t);
template void launch_mixed<2>(Handle&, const Ptrs&, uint32_t, uint32_t, const MPtrs&, uint64_t, uint64_t);
template void launch_mixed<4>(Handle&, const Ptrs&, uint32_t, uint32_t, const MPtrs&, uint64_t, uint64_t);
template void launch_mixed_scatter<1>(Handle&, int, int, int, const Ptrs&, uint32_t, uint32_t, const MPtrs&, uint64_t,
                                      int, uint64_t, uint64_t, int, const MixedTarget&);
template void launch_mixed_scatter<2>(Handle&, int, int, int, const Ptrs&, uint32_t, uint32_t, const MPtrs&, uint64_t,
                                      int, uint64_t, uint64_t, int, const MixedTarget&);
template void unpack_slab<1>(Handle&, const double*, size_t, uint32_t, uint64_t, uint32_t, double*);
template void unpack_slab<2>(Handle&, const double*, size_t, uint32_t, uint64_t, uint32_t, double*);
template void mixed_columns<1>(Handle&, int, int, const Ptrs&, double* const*, size_t);
template void mixed_columns<2>(Handle&, int, int, const Ptrs&, double* const*, size_t);

} // namespace detci_gpu
