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
// Multi-GPU / virtual blocks: alpha rows are partitioned into P blocks;
// the alpha and mixed terms need Cs rows from every block, which rotate
// ring-wise (NCCL send/recv on a comm stream, double-buffered, overlapped
// with the compute of the resident block).  The beta term and diagonal are
// block-local.
#include <algorithm>
#include <cstdio>
#include <array>
#include <cstdlib>
#include <string>
#include <vector>

#include "formulas.cuh"
#include "handle.hpp"

namespace detci_gpu {

namespace {

constexpr int kMaxM = 4;

// ---------------------------------------------------------------------------
// Same-spin kernel.  CTA = (output row, column chunk); threads own R columns
// each (coalesced), loop over the row's helper-list entries staged in smem.
// Per element: one coalesced 8 B load of Cs[ja, col] per vector and a DFMA
// (+ one coalesced J load and a sign flip for singles).  Grid is chunk-major
// so CTAs in flight share Cs[:, chunk] in L2.
// ---------------------------------------------------------------------------
constexpr int kSSBlock = 128;
constexpr int kStage = 256;

template <int M>
struct SSR {
    static constexpr int value = M == 1 ? 4 : (M == 2 ? 2 : 1);
};

struct SameSpinArgs {
    const double* C[kMaxM];   // Cs row ja of vector v at C[v] + (ja - c_row0) * ldc
    size_t ldc;
    uint32_t c_row0, j0, j1;  // window [j0, j1) of target rows
    double* Y[kMaxM];         // output row r at Y[v] + r * ldy
    size_t ldy;
    uint32_t row0, nrows;     // list rows [row0, row0 + nrows)
    uint32_t ncols;
    const double* J;          // J[tri * ldj + col]
    size_t ldj;
    const uint32_t* flat[2];
    const uint64_t* off[2];
    const uint32_t* len[2];
    const double* pv[2];
    const uint32_t* pab;
    const uint64_t* eps_row;  // if set: output *= eps(eps_row[row], eps_col[col])
    const uint64_t* eps_col;
    const double* diag;       // if set (write mode): Y = diag * Cself + acc
    const double* Cself[kMaxM];
    int accumulate;
};

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t n, uint32_t key) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// x * (-1)^{bit 31 of sign31}, by flipping the IEEE sign bit.
__device__ __forceinline__ double xor_sign(double x, uint32_t sign31) {
    return __hiloint2double(__double2hiint(x) ^ static_cast<int>(sign31), __double2loint(x));
}

// Epilogue shared by both same-spin variants: eps sign, then write,
// accumulate, or diag * Cself + acc.
template <int M>
__device__ __forceinline__ void samespin_store(const SameSpinArgs& a, uint64_t arow, uint32_t r, uint32_t c,
                                               const double (&acc)[M]) {
    const size_t yi = static_cast<size_t>(r) * a.ldy + c;
    const uint32_t flip = a.eps_row ? static_cast<uint32_t>(__popcll(arow & a.eps_col[c])) : 0u;
#pragma unroll
    for (int vv = 0; vv < M; ++vv) {
        const double v = flip_sign(acc[vv], flip);
        if (a.accumulate && a.diag) {   // accumulate the diagonal term too
            a.Y[vv][yi] += fma(a.diag[yi], a.Cself[vv][yi], v);
        } else if (a.accumulate) {
            a.Y[vv][yi] += v;
        } else if (a.diag) {
            a.Y[vv][yi] = fma(a.diag[yi], a.Cself[vv][yi], v);
        } else {
            a.Y[vv][yi] = v;
        }
    }
}

// kTail: the CTA's column chunk crosses ncols, so column indices are clamped
// (loads stay in bounds, stores are masked); full chunks use one base
// pointer per entry with immediate offsets.
template <bool kTail, int M>
__global__ void __launch_bounds__(kSSBlock)
k_samespin(const SameSpinArgs a, uint32_t chunk0) {
    constexpr int R = SSR<M>::value;
    __shared__ uint32_t s_ja[kStage];
    __shared__ double s_v[kStage];
    __shared__ uint32_t s_ab[kStage];
    __shared__ uint64_t s_range[4];

    const uint32_t r = blockIdx.x % a.nrows;
    const uint32_t chunk = chunk0 + blockIdx.x / a.nrows;
    const uint32_t row = a.row0 + r;
    const uint32_t tid = threadIdx.x;
    const uint32_t col0 = chunk * (kSSBlock * R) + tid;

    uint32_t col[R];
    double acc[R][M];
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const uint32_t c = col0 + q * kSSBlock;
        col[q] = kTail ? min(c, a.ncols - 1) : c;
#pragma unroll
        for (int v = 0; v < M; ++v) acc[q][v] = 0.0;
    }

    if (tid < 2) {
        const uint64_t o = a.off[tid][row];
        const uint32_t n = a.len[tid][row];
        const uint32_t* f = a.flat[tid] + o;
        const uint32_t b = a.j0 == 0 ? 0 : lower_bound_u32(f, n, a.j0);
        const uint32_t e = lower_bound_u32(f, n, a.j1);
        s_range[2 * tid] = o + b;
        s_range[2 * tid + 1] = o + e;
    }
    __syncthreads();

#pragma unroll 1
    for (int kind = 0; kind < 2; ++kind) {
        const uint64_t kb = s_range[2 * kind], ke = s_range[2 * kind + 1];
#pragma unroll 1
        for (uint64_t k0 = kb; k0 < ke; k0 += kStage) {
            const int cnt = static_cast<int>(min(static_cast<uint64_t>(kStage), ke - k0));
            __syncthreads();
            for (int t = tid; t < cnt; t += kSSBlock) {
                s_ja[t] = a.flat[kind][k0 + t] - a.c_row0;
                s_v[t] = a.pv[kind][k0 + t];
                if (kind == 0) s_ab[t] = a.pab[k0 + t];
            }
            __syncthreads();
            if (kind == 0) {
#pragma unroll 2
                for (int e = 0; e < cnt; ++e) {
                    const size_t rowoff = static_cast<size_t>(s_ja[e]) * a.ldc;
                    const uint32_t ab = s_ab[e];
                    const double* jrow = a.J + static_cast<size_t>(ab & 0x7fffffffu) * a.ldj;
                    const double v = s_v[e];
                    const uint32_t jsign = ab & 0x80000000u;
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        const uint32_t cq = kTail ? col[q] : col0 + q * kSSBlock;
                        const double val = v + xor_sign(__ldg(jrow + cq), jsign);
#pragma unroll
                        for (int vv = 0; vv < M; ++vv)
                            acc[q][vv] = fma(val, __ldg(a.C[vv] + rowoff + cq), acc[q][vv]);
                    }
                }
            } else {
#pragma unroll 4
                for (int e = 0; e < cnt; ++e) {
                    const size_t rowoff = static_cast<size_t>(s_ja[e]) * a.ldc + (kTail ? 0 : col0);
                    const double v = s_v[e];
#pragma unroll
                    for (int q = 0; q < R; ++q) {
#pragma unroll
                        for (int vv = 0; vv < M; ++vv) {
                            const double* base = a.C[vv] + rowoff;
                            const double c = __ldg(kTail ? base + col[q] : base + q * kSSBlock);
                            acc[q][vv] = fma(v, c, acc[q][vv]);
                        }
                    }
                }
            }
        }
    }

    const uint64_t arow = a.eps_row ? a.eps_row[row] : 0;
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const uint32_t c = col0 + q * kSSBlock;
        if (kTail && c >= a.ncols) continue;
        samespin_store<M>(a, arow, r, c, acc[q]);
    }
}

// Grouped variant: CTA = (8 consecutive output rows, one 32*R-column chunk),
// one row per warp.  Consecutive rows share most of their helper-list
// targets (sorted strings), and the warps walk their own sorted lists at
// similar paces, so Cs[ja, chunk] lines fetched by one warp are re-read by
// the others from L1 (simulated 45-59% L1 hits at C2) instead of L2, which
// bounds the one-row-per-CTA kernel (84.6% L2 throughput, 98% L2 hits).
constexpr int kGStage = 32;   // entries staged per warp
// Warps per SM the grouped kernel is compiled for (64 registers).  Measured:
// 40 or 48 warps per SM (48 / 40 registers) are slower (C3 alpha 121 vs 114
// ms): more rows in flight thrash L1.
constexpr int kSSMinBlocks = 32;

// GW warps = output rows per CTA (8 or 16; 1024 threads per SM either way)
// kV2 (M = 1, full chunks, 16-byte aligned rows): each lane owns two pairs
// of adjacent columns and reads them with one 16-byte load each, halving
// the load instructions per element.
template <bool kTail, int M, int GW, bool kV2 = false>
__global__ void __launch_bounds__(GW * kWarp, kSSMinBlocks / GW)
k_samespin_g(const SameSpinArgs a, uint32_t chunk0, uint32_t ngroups) {
    constexpr int kGW = GW;
    constexpr int R = SSR<M>::value;
    static_assert(!kV2 || (M == 1 && !kTail && R == 4), "kV2: one vector, full chunks");
    __shared__ uint32_t s_ja[kGW][kGStage];
    __shared__ double s_v[kGW][kGStage];
    __shared__ uint32_t s_ab[kGW][kGStage];

    const uint32_t warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    const uint32_t group = blockIdx.x % ngroups;
    const uint32_t chunk = chunk0 + blockIdx.x / ngroups;
    const uint32_t r = group * kGW + warp;
    if (r >= a.nrows) return;   // no CTA-wide barriers below
    const uint32_t row = a.row0 + r;
    const uint32_t col0 = chunk * (kWarp * R) + lane;

    uint32_t col[R];
    double acc[R][M];
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const uint32_t c = col0 + q * kWarp;
        col[q] = kTail ? min(c, a.ncols - 1) : c;
#pragma unroll
        for (int v = 0; v < M; ++v) acc[q][v] = 0.0;
    }

    uint64_t rb = 0, re = 0;
    if (lane < 2) {
        const uint64_t o = a.off[lane][row];
        const uint32_t n = a.len[lane][row];
        const uint32_t* f = a.flat[lane] + o;
        rb = o + (a.j0 == 0 ? 0 : lower_bound_u32(f, n, a.j0));
        re = o + lower_bound_u32(f, n, a.j1);
    }
    uint32_t* sja = s_ja[warp];
    double* sv = s_v[warp];
    uint32_t* sab = s_ab[warp];

#pragma unroll 1
    for (int kind = 0; kind < 2; ++kind) {
        const uint64_t kb = __shfl_sync(0xffffffffu, rb, kind), ke = __shfl_sync(0xffffffffu, re, kind);
#pragma unroll 1
        for (uint64_t k0 = kb; k0 < ke; k0 += kGStage) {
            const int cnt = static_cast<int>(min(static_cast<uint64_t>(kGStage), ke - k0));
            __syncwarp();
            for (int t = lane; t < cnt; t += kWarp) {
                sja[t] = a.flat[kind][k0 + t] - a.c_row0;
                sv[t] = a.pv[kind][k0 + t];
                if (kind == 0) sab[t] = a.pab[k0 + t];
            }
            __syncwarp();
            if constexpr (kV2) {
                // columns chunk*128 + q*64 + 2*lane + {0, 1}, q < 2
                const uint32_t cb = chunk * (kWarp * R) + 2 * lane;
                if (kind == 0) {
#pragma unroll 2
                    for (int e = 0; e < cnt; ++e) {
                        const double* crow = a.C[0] + static_cast<size_t>(sja[e]) * a.ldc + cb;
                        const uint32_t ab = sab[e];
                        const double* jrow = a.J + static_cast<size_t>(ab & 0x7fffffffu) * a.ldj + cb;
                        const double v = sv[e];
                        const uint32_t jsign = ab & 0x80000000u;
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            const double2 j = __ldg(reinterpret_cast<const double2*>(jrow + q * 2 * kWarp));
                            const double2 c = __ldg(reinterpret_cast<const double2*>(crow + q * 2 * kWarp));
                            acc[2 * q][0] = fma(v + xor_sign(j.x, jsign), c.x, acc[2 * q][0]);
                            acc[2 * q + 1][0] = fma(v + xor_sign(j.y, jsign), c.y, acc[2 * q + 1][0]);
                        }
                    }
                } else {
#pragma unroll 4
                    for (int e = 0; e < cnt; ++e) {
                        const double* crow = a.C[0] + static_cast<size_t>(sja[e]) * a.ldc + cb;
                        const double v = sv[e];
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            const double2 c = __ldg(reinterpret_cast<const double2*>(crow + q * 2 * kWarp));
                            acc[2 * q][0] = fma(v, c.x, acc[2 * q][0]);
                            acc[2 * q + 1][0] = fma(v, c.y, acc[2 * q + 1][0]);
                        }
                    }
                }
                continue;
            }
            if (kind == 0) {
#pragma unroll 2
                for (int e = 0; e < cnt; ++e) {
                    const size_t rowoff = static_cast<size_t>(sja[e]) * a.ldc;
                    const uint32_t ab = sab[e];
                    const double* jrow = a.J + static_cast<size_t>(ab & 0x7fffffffu) * a.ldj;
                    const double v = sv[e];
                    const uint32_t jsign = ab & 0x80000000u;
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        const uint32_t cq = kTail ? col[q] : col0 + q * kWarp;
                        const double val = v + xor_sign(__ldg(jrow + cq), jsign);
#pragma unroll
                        for (int vv = 0; vv < M; ++vv)
                            acc[q][vv] = fma(val, __ldg(a.C[vv] + rowoff + cq), acc[q][vv]);
                    }
                }
            } else {
#pragma unroll 4
                for (int e = 0; e < cnt; ++e) {
                    const size_t rowoff = static_cast<size_t>(sja[e]) * a.ldc + (kTail ? 0 : col0);
                    const double v = sv[e];
#pragma unroll
                    for (int q = 0; q < R; ++q) {
#pragma unroll
                        for (int vv = 0; vv < M; ++vv) {
                            const double* base = a.C[vv] + rowoff;
                            const double c = __ldg(kTail ? base + col[q] : base + q * kWarp);
                            acc[q][vv] = fma(v, c, acc[q][vv]);
                        }
                    }
                }
            }
        }
    }

    const uint64_t arow = a.eps_row ? a.eps_row[row] : 0;
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const uint32_t c = kV2 ? chunk * (kWarp * R) + (q / 2) * 2 * kWarp + 2 * lane + (q % 2) : col0 + q * kWarp;
        if (kTail && c >= a.ncols) continue;
        samespin_store<M>(a, arow, r, c, acc[q]);
    }
}

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
constexpr int kMxBlock = 1024;   // one CTA per SM, 32 warps

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

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_prev() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

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
    const uint32_t* sa_flat;
    const uint64_t* sa_off;
    const uint32_t* tpos;
    const uint32_t* sell;
    const uint64_t* sell_off;
    const uint32_t* sell_len;
    const double* eri;
    int norbs;
    double* D[2];               // D_v row (sa_off[ia] + pos - d_base), ldd slots
    uint64_t d_base;
    uint32_t ldd;
    uint32_t slot0, slot_end;   // beta slots [slot0, slot_end) (multi-GPU column share)
    const uint32_t* w_lo;       // ja-window D compaction (ScatterWindow::by_ja), or null
    const uint64_t* w_base;
};

// One pass of the scatter CTA: K output rows ia_k = list(ja)[kbeg + k], k <
// cnt (rows cnt..K-1 padded: computed, never stored).  Builds V for the pass, runs
// the row segments (reusing the staged row when it fits whole: `staged`),
// and stores the partials.  M = 1 or 2 vectors share the V gathers (the
// multi-root block's pairs): an element costs (M + K) / (M K) gathers per
// FMA.
// (V row offset | alpha sign << 63, D row) of output ia = list(ja)[pos].
__device__ __forceinline__ void scatter_row(const ScatterArgs& a, uint32_t ja, uint64_t oja, uint32_t pos,
                                            uint64_t& vr, uint64_t& dr) {
    const int n = a.norbs, nn = n * n;
    const uint64_t Aj = a.alpha[ja];
    const uint32_t ia = a.sa_flat[oja + pos];
    const uint64_t Ak = a.alpha[ia];
    const int pa = __ffsll(static_cast<long long>(Ak & ~Aj)) - 1;
    const int qa = __ffsll(static_cast<long long>(Aj & ~Ak)) - 1;
    vr = static_cast<uint64_t>(pa * n + qa) * nn | static_cast<uint64_t>(mixed_alpha_parity(Ak, pa, qa)) << 63;
    dr = a.w_lo ? a.w_base[ia] + a.tpos[oja + pos] - a.w_lo[ia] : a.sa_off[ia] + a.tpos[oja + pos] - a.d_base;
}

// Entries of a CTA's run whose (V row, D row) are computed once up front
// (one latency for all passes instead of one per pass).
constexpr uint32_t kRunPre = 256;

template <int K, int M>
__device__ __forceinline__ void scatter_pass(const ScatterArgs& a, double* vsub, double* cseg, uint64_t* s_vrow,
                                             uint64_t* s_drow, uint32_t ja, uint64_t oja, uint32_t kbeg,
                                             uint32_t cnt, bool staged, uint32_t part, bool precomputed) {
    const int n = a.norbs, nn = n * n;
    const uint32_t tid = threadIdx.x, lane = tid % kWarp;
    const uint32_t segpad = (a.seg_cols + 2) & ~1u;   // + the zero slot at seg_cols
    const size_t crow = static_cast<size_t>(ja - a.c_row0) * a.ldc;
    auto stage = [&](uint32_t g) {
        const uint32_t segw = min(a.seg_cols, a.nb - g * a.seg_cols);
#pragma unroll
        for (int v = 0; v < M; ++v) {
            const double* src = a.C[v] + crow + static_cast<size_t>(g) * a.seg_cols;
            double* dst = cseg + v * segpad;
            for (uint32_t c = tid; c < segw; c += kMxBlock) cp_async8(dst + c, src + c);
        }
        cp_async_commit();
    };
    __syncthreads();   // the previous pass is done with V, the row tables and the segment
    if (!precomputed && tid < K) {
        uint64_t vr = ~0ull, dr = 0;
        if (tid < cnt) scatter_row(a, ja, oja, kbeg + tid, vr, dr);
        s_vrow[tid] = vr;
        s_drow[tid] = dr;
    }
    if (!staged) stage(0);   // streams in under the V copies
    __syncthreads();
    // V rows: the raw ERI rows (pa qa|..) by cp.async; the alpha sign goes on
    // the partial at the store, padding entries read the C zero slot, and
    // rows k >= cnt copy row 0 (finite, never stored)
    if ((nn & 1) == 0) {
        const uint32_t h2 = static_cast<uint32_t>(nn) / 2;
        for (uint32_t t = tid; t < static_cast<uint32_t>(K) * h2; t += kMxBlock) {
            const uint32_t k = t / h2, u = t - k * h2;
            const uint64_t vr = s_vrow[k < cnt ? k : 0];
            cp_async16(vsub + k * a.vpitch + 2 * u, a.eri + (vr & 0x7fffffffffffffffull) + 2 * u);
        }
    } else {
        for (uint32_t t = tid; t < static_cast<uint32_t>(K * nn); t += kMxBlock) {
            const uint32_t k = t / nn, cd = t - k * nn;
            const uint64_t vr = s_vrow[k < cnt ? k : 0];
            cp_async8(vsub + k * a.vpitch + cd, a.eri + (vr & 0x7fffffffffffffffull) + cd);
        }
    }
    cp_async_commit();   // waited for with the first segment below

    const uint32_t slot = a.slot0 + part * kMxBlock + tid;
    const uint32_t sl = slot / kWarp;
    const bool active = sl < a.nslices && slot < a.slot_end;
    double acc[M][K];
#pragma unroll
    for (int v = 0; v < M; ++v)
#pragma unroll
        for (int k = 0; k < K; ++k) acc[v][k] = 0.0;
    const char* vb = reinterpret_cast<const char*>(vsub);
    const char* cb = reinterpret_cast<const char*>(cseg);
    const uint32_t vstride = a.vpitch * 8, cstride = segpad * 8;

    auto element = [&](uint32_t e) {
        const char* cp = cb + (e & 0x3ffffu);
        double c[M];
#pragma unroll
        for (int v = 0; v < M; ++v)
            c[v] = xor_sign(*reinterpret_cast<const double*>(cp + v * cstride), e & 0x80000000u);
        const char* vp = vb + ((e >> 15) & 0x7ff8u);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const double w = *reinterpret_cast<const double*>(vp + k * vstride);
#pragma unroll
            for (int v = 0; v < M; ++v) acc[v][k] = fma(w, c[v], acc[v][k]);
        }
    };

#pragma unroll 1
    for (uint32_t g = 0; g < a.nseg; ++g) {
        if (g > 0) {
            __syncthreads();   // previous segment consumed
            stage(g);
        }
        cp_async_wait_all();
        __syncthreads();
        if (!active) continue;
        const uint32_t L = a.sell_len[sl * a.nseg + g];
        const uint32_t* ent = a.sell + a.sell_off[sl * a.nseg + g] + lane;
        uint32_t t = 0;
#pragma unroll 1
        for (; t + 4 <= L; t += 4) {
            uint32_t e[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) e[u] = __ldg(ent + static_cast<size_t>(t + u) * kWarp);
#pragma unroll
            for (int u = 0; u < 4; ++u) element(e[u]);
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
// remainder pass of the next power of two >= the rest.
template <int KMAX, int M>
__global__ void __launch_bounds__(kMxBlock, 1)
k_mixed_scatter(const ScatterArgs a) {
    extern __shared__ double smem[];
    double* const vsub = smem;                      // KMAX rows of vpitch
    double* const cseg = smem + KMAX * a.vpitch;    // Cs_v[ja, segment], v < M
    __shared__ uint64_t s_vrow[KMAX];               // eri row offset | sign << 63 (runs past kRunPre)
    __shared__ uint64_t s_drow[KMAX];               // D row of output k
    __shared__ uint64_t s_vall[kRunPre], s_dall[kRunPre];   // the run's first kRunPre rows

    const uint32_t item = blockIdx.x / a.nparts, part = blockIdx.x % a.nparts;
    const uint2 it = a.items[item];
    const uint32_t ja = it.x, kbeg = it.y & 0xfffffu, len = it.y >> 20;
    const uint64_t oja = a.sa_off[ja];
    for (uint32_t t = threadIdx.x; t < min(len, kRunPre); t += kMxBlock) {
        uint64_t vr, dr;
        scatter_row(a, ja, oja, kbeg + t, vr, dr);
        s_vall[t] = vr;
        s_dall[t] = dr;
    }   // visible after the first pass's barrier
    const bool whole = a.nseg == 1;
    const uint32_t segpad = (a.seg_cols + 2) & ~1u;
    if (threadIdx.x < M) cseg[threadIdx.x * segpad + a.seg_cols] = 0.0;   // zero slot (padding entries)
    if (whole) {
        const size_t crow = static_cast<size_t>(ja - a.c_row0) * a.ldc;
#pragma unroll
        for (int v = 0; v < M; ++v) {
            const double* src = a.C[v] + crow;
            double* dst = cseg + v * segpad;
            for (uint32_t c = threadIdx.x; c < a.nb; c += kMxBlock) cp_async8(dst + c, src + c);
        }
        cp_async_commit();
    }
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
#pragma unroll 1
    for (; p + KMAX <= end; p += KMAX) {
        const bool pre = tabs(p, KMAX, tv, td);
        scatter_pass<KMAX, M>(a, vsub, cseg, tv, td, ja, oja, p, KMAX, whole, part, pre);
    }
    const uint32_t r = end - p;
    if (r == 0) return;
    const bool pre = tabs(p, r, tv, td);
    if constexpr (KMAX > 8) { if (r > 8) { scatter_pass<16, M>(a, vsub, cseg, tv, td, ja, oja, p, r, whole, part, pre); return; } }
    if constexpr (KMAX > 4) { if (r > 4) { scatter_pass<8, M>(a, vsub, cseg, tv, td, ja, oja, p, r, whole, part, pre); return; } }
    if constexpr (KMAX > 2) { if (r > 2) { scatter_pass<4, M>(a, vsub, cseg, tv, td, ja, oja, p, r, whole, part, pre); return; } }
    if constexpr (KMAX > 1) { if (r > 1) { scatter_pass<2, M>(a, vsub, cseg, tv, td, ja, oja, p, r, whole, part, pre); return; } }
    scatter_pass<1, M>(a, vsub, cseg, tv, td, ja, oja, p, r, whole, part, pre);
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
    for (; p + 4 <= hi; p += 4) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcs(d + static_cast<size_t>(p - lo + u) * a.ldd);
#pragma unroll
        for (int u = 0; u < 4; ++u) s += v[u];
    }
    for (; p < hi; ++p) s += __ldcs(d + static_cast<size_t>(p - lo) * a.ldd);
    const uint32_t ib = a.perm[slot];
    const uint32_t flip = static_cast<uint32_t>(__popcll(a.alpha[ia] & a.beta_prefix[ib]));
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

// ---------------------------------------------------------------------------
// eps prologue / epilogue, through 32x32 smem tiles (coalesced both ways).
// ---------------------------------------------------------------------------
constexpr int kTile = 32;

// Local block x (rows x cols, row r = alpha string a_str[r], column c = beta
// string with prefix parity b_pre[c]):
//   xs[r * ldx + c] = eps x      (if xs)     xsT[c * ldt + r] = eps x (if xsT)
__global__ void k_eps_transpose(const double* __restrict__ x, size_t ldx, double* __restrict__ xs,
                                double* __restrict__ xsT, size_t ldt, uint32_t rows, uint32_t cols,
                                const uint64_t* __restrict__ a_str, const uint64_t* __restrict__ b_pre) {
    __shared__ double tile[kTile][kTile + 1];
    __shared__ uint64_t s_a[kTile];
    const uint32_t c0 = blockIdx.x * kTile, r0 = blockIdx.y * kTile;
    const uint32_t cc = c0 + threadIdx.x;
    const uint64_t pb = cc < cols ? b_pre[cc] : 0;
    if (threadIdx.y == 0 && r0 + threadIdx.x < rows) s_a[threadIdx.x] = a_str[r0 + threadIdx.x];
    __syncthreads();
    for (uint32_t y = threadIdx.y; y < kTile; y += blockDim.y) {
        const uint32_t rr = r0 + y;
        if (rr < rows && cc < cols) {
            const size_t i = static_cast<size_t>(rr) * ldx + cc;
            const double v = flip_sign(x[i], static_cast<uint32_t>(__popcll(s_a[y] & pb)));
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
                                    const uint64_t* __restrict__ a_str, const uint64_t* __restrict__ b_pre) {
    __shared__ double tile[kTile][kTile + 1];
    __shared__ uint64_t s_a[kTile];
    const uint32_t c0 = blockIdx.x * kTile, r0 = blockIdx.y * kTile;
    for (uint32_t y = threadIdx.y; y < kTile; y += blockDim.y) {
        const uint32_t c = c0 + y, rr = r0 + threadIdx.x;
        if (rr < rows && c < cols) tile[y][threadIdx.x] = src[static_cast<size_t>(c) * lds + rr];
    }
    if (threadIdx.y == 0 && r0 + threadIdx.x < rows) s_a[threadIdx.x] = a_str[r0 + threadIdx.x];
    __syncthreads();
    const uint32_t cc = c0 + threadIdx.x;
    const uint64_t pb = cc < cols ? b_pre[cc] : 0;
    for (uint32_t y = threadIdx.y; y < kTile; y += blockDim.y) {
        const uint32_t rr = r0 + y;
        if (rr < rows && cc < cols)
            dst[static_cast<size_t>(rr) * ldd + cc] +=
                flip_sign(tile[threadIdx.x][y], static_cast<uint32_t>(__popcll(s_a[y] & pb)));
    }
}

// ---------------------------------------------------------------------------
// Host orchestration.
// ---------------------------------------------------------------------------

struct PhaseTimer {
    Handle& h;
    bool on;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    std::vector<int> cat;
    PhaseTimer(Handle& hh, bool enabled) : h(hh), on(enabled) {}
    ~PhaseTimer() {
        for (auto& p : ev) {
            cudaEventDestroy(p.first);
            cudaEventDestroy(p.second);
        }
    }
    int begin(int category) {
        if (!on) return -1;
        cudaEvent_t a, b;
        CUDA_CHECK(cudaEventCreate(&a));
        CUDA_CHECK(cudaEventCreate(&b));
        CUDA_CHECK(cudaEventRecord(a, h.stream));
        ev.emplace_back(a, b);
        cat.push_back(category);
        return static_cast<int>(ev.size()) - 1;
    }
    void end(int id) {
        if (id >= 0) CUDA_CHECK(cudaEventRecord(ev[id].second, h.stream));
    }
    // categories: 0 alpha, 1 beta, 2 mixed, 3 combine
    void collect(double out[4]) {
        for (int i = 0; i < 4; ++i) out[i] = 0.0;
        for (size_t i = 0; i < ev.size(); ++i) {
            float ms = 0.f;
            CUDA_CHECK(cudaEventElapsedTime(&ms, ev[i].first, ev[i].second));
            out[cat[i]] += ms * 1e-3;
        }
    }
};

using Ptrs = std::array<const double*, kMaxM>;
using MPtrs = std::array<double*, kMaxM>;

// The grouped kernel (8 rows per CTA, L1 reuse) is the default; set
// DETCI_SAMESPIN=row for the one-row-per-CTA kernel.  With the spectator
// parities gone (separated ordering) the grouped kernel is no longer
// issue-bound: measured on B200, alpha term C2 19.9 vs 25.4 ms, C3 115 vs
// 159 ms.
bool grouped_samespin() {
    const char* e = std::getenv("DETCI_SAMESPIN");
    return !(e && std::string(e) == "row");
}

// DETCI_SAMESPIN_VEC=1: 16-byte loads in the grouped kernel.  Off by
// default: measured level or slightly slower (C2 alpha 20.1 vs 19.8 ms, C3
// 117.4 vs 116.3 ms), i.e. the kernel is bound by L1/L2 data, not by load
// instructions.
bool samespin_vec2() {
    const char* e = std::getenv("DETCI_SAMESPIN_VEC");
    return e && std::string(e) == "1";
}

template <int M, int GW>
void launch_samespin_g(const SameSpinArgs& s, cudaStream_t st) {
    constexpr uint32_t kChunk = kWarp * SSR<M>::value;
    const uint64_t full = s.ncols / kChunk;
    const bool tail = s.ncols % kChunk != 0;
    const uint32_t ngroups = (s.nrows + GW - 1) / GW;
    static bool configured = false;
    if (!configured) {  // favour L1 over shared memory (the kernel uses <= 32 KB)
        CUDA_CHECK(cudaFuncSetAttribute(k_samespin_g<false, M, GW>, cudaFuncAttributePreferredSharedMemoryCarveout, 10));
        CUDA_CHECK(cudaFuncSetAttribute(k_samespin_g<true, M, GW>, cudaFuncAttributePreferredSharedMemoryCarveout, 10));
        if constexpr (M == 1)
            CUDA_CHECK(cudaFuncSetAttribute(k_samespin_g<false, 1, GW, true>,
                                            cudaFuncAttributePreferredSharedMemoryCarveout, 10));
        configured = true;
    }
    // 16-byte loads need even strides and 16-byte aligned bases
    const bool v2 = M == 1 && samespin_vec2() && s.ldc % 2 == 0 && s.ldj % 2 == 0 &&
                    reinterpret_cast<uintptr_t>(s.C[0]) % 16 == 0 && reinterpret_cast<uintptr_t>(s.J) % 16 == 0;
    if (full && v2) {
        if constexpr (M == 1) {
            k_samespin_g<false, 1, GW, true><<<static_cast<unsigned>(full * ngroups), GW * kWarp, 0, st>>>(s, 0, ngroups);
            CUDA_LAUNCH_CHECK();
        }
    } else if (full) {
        k_samespin_g<false, M, GW><<<static_cast<unsigned>(full * ngroups), GW * kWarp, 0, st>>>(s, 0, ngroups);
        CUDA_LAUNCH_CHECK();
    }
    if (tail) {
        k_samespin_g<true, M, GW><<<ngroups, GW * kWarp, 0, st>>>(s, static_cast<uint32_t>(full), ngroups);
        CUDA_LAUNCH_CHECK();
    }
}

// DETCI_SAMESPIN_ROWS=16: 16 rows per grouped CTA (default 8).
int samespin_group_rows() {
    const char* e = std::getenv("DETCI_SAMESPIN_ROWS");
    return (e && std::string(e) == "16") ? 16 : 8;
}

template <int M>
void launch_samespin(const SameSpinArgs& s, cudaStream_t st) {
    if (s.nrows == 0 || s.ncols == 0) return;
    if (grouped_samespin()) {
        if (samespin_group_rows() == 16) launch_samespin_g<M, 16>(s, st);
        else launch_samespin_g<M, 8>(s, st);
        return;
    }
    constexpr uint32_t kChunk = kSSBlock * SSR<M>::value;
    const uint64_t full = s.ncols / kChunk;
    const bool tail = s.ncols % kChunk != 0;
    if (full) {
        k_samespin<false, M><<<static_cast<unsigned>(full * s.nrows), kSSBlock, 0, st>>>(s, 0);
        CUDA_LAUNCH_CHECK();
    }
    if (tail) {
        k_samespin<true, M><<<s.nrows, kSSBlock, 0, st>>>(s, static_cast<uint32_t>(full));
        CUDA_LAUNCH_CHECK();
    }
}

void fill_lists(SameSpinArgs& s, const ChannelTables& t) {
    for (int k = 0; k < 2; ++k) {
        s.flat[k] = t.flat[k].p;
        s.off[k] = t.offset[k].p;
        s.len[k] = t.len[k].p;
        s.pv[k] = t.pv[k].p;
    }
    s.pab = t.pab.p;
}

template <int M>
void launch_alpha(const Handle& h, const Ptrs& Cb, uint32_t b0, uint32_t b1, const Ptrs& x_loc,
                  const MPtrs& y_loc, uint64_t a0, uint64_t a1, bool first, bool add_to_y = false) {
    SameSpinArgs s{};
    for (int v = 0; v < M; ++v) {
        s.C[v] = Cb[v];
        s.Y[v] = y_loc[v];
        s.Cself[v] = x_loc[v];
    }
    s.ldc = h.nb();
    s.c_row0 = b0;
    s.j0 = b0;
    s.j1 = b1;
    s.ldy = h.nb();
    s.row0 = static_cast<uint32_t>(a0);
    s.nrows = static_cast<uint32_t>(a1 - a0);
    s.ncols = static_cast<uint32_t>(h.nb());
    s.J = h.ch[1].J.p;
    s.ldj = h.nb();
    fill_lists(s, h.ch[0]);
    s.eps_row = h.ch[0].strings.p;
    s.eps_col = h.ch[1].prefix.p;
    s.diag = first ? h.diag.p + (a0 - h.a0) * h.nb() : nullptr;
    s.accumulate = (first && !add_to_y) ? 0 : 1;   // first && add_to_y: y += diag*C + alpha
    launch_samespin<M>(s, h.stream);
}

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
    static size_t configured[2][kMaxM + 1] = {};
    const int db = t.double_buffer ? 1 : 0;
    if (smem > configured[db][M]) {
        if (db)
            CUDA_CHECK(cudaFuncSetAttribute(k_mixed<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem)));
        else
            CUDA_CHECK(cudaFuncSetAttribute(k_mixed<M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem)));
        configured[db][M] = smem;
    }
    const uint64_t grid = static_cast<uint64_t>(m.nrows) * m.nparts;
    if (db)
        k_mixed<M, true><<<static_cast<unsigned>(grid), kMxBlock, smem, h.stream>>>(m);
    else
        k_mixed<M, false><<<static_cast<unsigned>(grid), kMxBlock, smem, h.stream>>>(m);
    CUDA_LAUNCH_CHECK();
}


bool multi_ring();
std::pair<uint32_t, uint32_t> mixed_slots(const Handle& h, int g, int P);

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
                CUDA_CHECK(cudaMemcpy(w->lo.p, lo.data(), na * 4, cudaMemcpyHostToDevice));
                CUDA_CHECK(cudaMemcpy(w->base.p, base.data(), (na + 1) * 8, cudaMemcpyHostToDevice));
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
            CUDA_CHECK(cudaMemcpy(w->items[ki].p, items.data(), items.size() * sizeof(uint2), cudaMemcpyHostToDevice));
    }
    uint64_t need = 0;
    for (auto& w : wins) need = std::max(need, w->d_rows);
    if (h.dbuf.n < need * ldd * M) h.dbuf.alloc(need * ldd * M);
    return wins;
}

template <int KMAX, int M>
void launch_scatter_k(const ScatterArgs& a, uint64_t grid, uint32_t vpitch, size_t cbytes, cudaStream_t st) {
    const size_t smem = static_cast<size_t>(KMAX) * vpitch * sizeof(double) + M * cbytes;
    static size_t configured = 0;
    if (smem > configured) {
        CUDA_CHECK(cudaFuncSetAttribute(k_mixed_scatter<KMAX, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
        configured = smem;
    }
    k_mixed_scatter<KMAX, M><<<static_cast<unsigned>(grid), kMxBlock, smem, st>>>(a);
    CUDA_LAUNCH_CHECK();
}

// Where the mixed term goes: beta slots [slot0, slot_end) and, if T is set,
// overwrite T[v][(ia - a0) * ldt + slot - slot0] (slot order) instead of
// accumulating into y[ia][perm[slot]].
struct MixedTarget {
    uint32_t slot0 = 0, slot_end = 0xffffffffu;
    double* T[kMaxM] = {};
    size_t ldt = 0;
};

// Mixed term through the scatter kernel for block-rank g, held alpha block
// b = rows [b0, b1) of Cs in Cb, outputs rows [a0, a1) of y_loc.
// phases: 1 = scatter kernels only, 2 = D reduction only (of output rows
// [r_lo, r_hi) within each window), 3 = both (per window).
template <int M>
void launch_mixed_scatter(Handle& h, int g, int P, int b, const Ptrs& Cb, uint32_t b0, uint32_t b1,
                          const MPtrs& y_loc, uint64_t a0, int phases = 3, uint64_t r_lo = 0,
                          uint64_t r_hi = ~0ull, int only_window = -1, const MixedTarget& tgt = MixedTarget{}) {
    const SellTable& t = scatter_table(h, M);
    const auto& wins = scatter_windows(h, g, P, M, t.kmax);
    const int ki = __builtin_ctz(static_cast<unsigned>(t.kmax));
    const uint32_t ldd = mixed_ldd(h);
    const uint32_t vpitch = scatter_vpitch(h.norbs);
    const size_t cbytes = ((t.seg_cols + 2) & ~1u) * sizeof(double);   // + zero slot
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
        a.sa_flat = h.ch[0].flat[0].p;
        a.sa_off = h.ch[0].offset[0].p;
        a.tpos = h.tpos.p;
        a.sell = t.sell.p;
        a.sell_off = t.off.p;
        a.sell_len = t.len.p;
        a.eri = h.d_eri.p;
        a.norbs = h.norbs;
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
            r.perm = h.sell_perm.p;
            r.Y = y_loc[v];
            r.ldy = h.nb();
            r.y_row0 = static_cast<uint32_t>(a0);
            const uint64_t rgrid = (hi - lo) * r.nparts;
            k_mixed_reduce<<<static_cast<unsigned>(rgrid), kRedBlock, 0, h.stream>>>(r);
            CUDA_LAUNCH_CHECK();
        }
    }
}

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
                                                 nloc, nloc, nb, h.ch[0].strings.p + a0, h.ch[1].prefix.p);
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
                                                     h.ch[0].strings.p + a0, h.ch[1].prefix.p);
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
bool multi_ring() {
    const char* e = std::getenv("DETCI_MULTI");
    return e && std::string(e) == "ring";
}

// Beta slots of the mixed term owned by block-rank g (32-slot aligned).
std::pair<uint32_t, uint32_t> mixed_slots(const Handle& h, int g, int P) {
    const uint64_t total = static_cast<uint64_t>(h.nslices) * kWarp;
    auto at = [&](int k) { return static_cast<uint32_t>(k == P ? total : total * k / P / kWarp * kWarp); };
    return {at(g), at(g + 1)};
}

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

// One rank (world > 1) of the gather schedule over NCCL.
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
    if (ncclGroupStart() != ncclSuccess) fail(DETCI_GPU_E_CUDA, "ncclGroupStart");
    for (int v = 0; v < M; ++v)
        for (int b = 0; b < P; ++b) {
            double* blk = h.cs_full.p + v * full + h.blk[b] * nb;
            const size_t n = (h.blk[b + 1] - h.blk[b]) * nb;
            if (n && ncclBroadcast(blk, blk, n, ncclDouble, b, h.nccl, h.comm_stream) != ncclSuccess)
                fail(DETCI_GPU_E_CUDA, "ncclBroadcast (Cs allgather)");
        }
    if (ncclGroupEnd() != ncclSuccess) fail(DETCI_GPU_E_CUDA, "ncclGroupEnd (Cs allgather)");
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
    if (ncclGroupStart() != ncclSuccess) fail(DETCI_GPU_E_CUDA, "ncclGroupStart");
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
            if (send_n && ncclSend(src, send_n, ncclDouble, b, h.nccl, h.comm_stream) != ncclSuccess)
                fail(DETCI_GPU_E_CUDA, "ncclSend (mixed slab)");
            if (recv_n && ncclRecv(dst, recv_n, ncclDouble, b, h.nccl, h.comm_stream) != ncclSuccess)
                fail(DETCI_GPU_E_CUDA, "ncclRecv (mixed slab)");
        }
    if (ncclGroupEnd() != ncclSuccess) fail(DETCI_GPU_E_CUDA, "ncclGroupEnd (mixed slab)");
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
    const int id = tm.begin(2);
    size_t toff = 0;
    for (int g = 0; g < P; ++g) {
        const auto [s0, s1] = mixed_slots(h, g, P);
        const size_t ns = s1 - s0;
        double* T[kMaxM] = {};
        for (int v = 0; v < M; ++v) T[v] = h.mix_t.p + v * tstride + toff;
        mixed_columns<M>(h, g, P, cf, T, ns);
        for (int v = 0; v < M; ++v) unpack_slab<M>(h, T[v], ns, static_cast<uint32_t>(ns), na, s0, dy[v]);
        toff += na * ns;
    }
    tm.end(id);
}

template <int M>
void sigma_schedule_m(Handle& h, const Ptrs& dx, const MPtrs& dy, PhaseTimer& tm) {
    const int Pm = std::max(h.world, h.vblocks);
    if (Pm > 1 && M <= 2 && mixed_scatter_enabled() && !multi_ring()) {
        ensure_scratch(h, M, 1);
        ensure_gather_scratch(h, M, Pm);
        if (h.world > 1) sigma_gather_rank<M>(h, dx, dy, tm);
        else sigma_gather_virtual<M>(h, dx, dy, tm);
        return;
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
            if (ncclGroupStart() != ncclSuccess) fail(DETCI_GPU_E_CUDA, "ncclGroupStart");
            for (int v = 0; v < M; ++v) {
                ncclSend(held[v], send_n, ncclDouble, (g - 1 + P) % P, h.nccl, h.comm_stream);
                ncclRecv(dst + v * block, recv_n, ncclDouble, (g + 1) % P, h.nccl, h.comm_stream);
            }
            if (ncclGroupEnd() != ncclSuccess) fail(DETCI_GPU_E_CUDA, "ncclGroupEnd (ring)");
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
    const std::vector<uint64_t> fe = pipe_edges(nloc, kFrontWeight), te = pipe_edges(nloc, kTailWeight);
    cudaEvent_t ev[kFrontChunks + kTailChunks + 2];
    const bool dbg = std::getenv("DETCI_PIPE_DEBUG") != nullptr;
    for (auto& e : ev) CUDA_CHECK(cudaEventCreateWithFlags(&e, out || dbg ? cudaEventDefault : cudaEventDisableTiming));
    cudaEvent_t* landed = ev;                    // H2D of front chunk c done
    cudaEvent_t* final_rows = ev + kFrontChunks; // y rows of tail chunk c final
    cudaEvent_t t0 = ev[kFrontChunks + kTailChunks], t1 = ev[kFrontChunks + kTailChunks + 1];
    CUDA_CHECK(cudaEventRecord(t0, h.stream));
    CUDA_CHECK(cudaStreamWaitEvent(h.comm_stream, t0, 0));   // previous work on the buffers is done
    for (int c = 0; c < kFrontChunks; ++c) {
        const uint64_t r0 = fe[c], r1 = fe[c + 1];
        if (r1 > r0)
            CUDA_CHECK(cudaMemcpyAsync(dx + r0 * nb, x + r0 * nb, (r1 - r0) * nb * 8, cudaMemcpyHostToDevice,
                                       h.comm_stream));
        CUDA_CHECK(cudaEventRecord(landed[c], h.comm_stream));
    }
    // prologue + beta term per landed chunk
    for (int c = 0; c < kFrontChunks; ++c) {
        const uint64_t r0 = fe[c], r1 = fe[c + 1];
        CUDA_CHECK(cudaStreamWaitEvent(h.stream, landed[c], 0));
        if (r1 == r0) continue;
        const uint32_t rc = static_cast<uint32_t>(r1 - r0);
        dim3 tb(kTile, 8), tg(static_cast<unsigned>((nb + kTile - 1) / kTile), (rc + kTile - 1) / kTile);
        k_eps_transpose<<<tg, tb, 0, h.stream>>>(dx + r0 * nb, nb, h.xs.p + r0 * nb, h.ct.p + r0, nloc, rc,
                                                 static_cast<uint32_t>(nb), h.ch[0].strings.p + a0 + r0,
                                                 h.ch[1].prefix.p);
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
                                                         static_cast<uint32_t>(nb), h.ch[0].strings.p + a0 + r0,
                                                         h.ch[1].prefix.p);
            CUDA_LAUNCH_CHECK();
        }
        launch_mixed_scatter<1>(h, 0, 1, 0, held, 0, static_cast<uint32_t>(h.na()), yl, a0, 2, a0 + r0, a0 + r1, wi);
        last_chunk = (last_chunk + 1) % kTailChunks;
        cudaEvent_t done = final_rows[last_chunk];
        CUDA_CHECK(cudaEventRecord(done, h.stream));
        CUDA_CHECK(cudaStreamWaitEvent(h.comm_stream, done, 0));
        CUDA_CHECK(cudaMemcpyAsync(y + r0 * nb, dy + r0 * nb, (r1 - r0) * nb * 8, cudaMemcpyDeviceToHost,
                                   h.comm_stream));
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
        double parts[4];
        tm.collect(parts);
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
