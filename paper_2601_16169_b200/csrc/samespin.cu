// Same-spin sigma kernels (the alpha term on Cs, the beta term on Cs^T):
// matvec's alpha and beta loops (matvec.cpp:144-191) in the separated
// ordering (sigma.cu header).
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




// Epilogue shared by both same-spin variants: eps sign, then write,
// accumulate, or diag * Cself + acc.
template <int M>
__device__ __forceinline__ void samespin_store(const SameSpinArgs& a, Bits arow, uint32_t r, uint32_t c,
                                               const double (&acc)[M]) {
    const size_t yi = static_cast<size_t>(r) * a.ldy + c;
    const uint32_t flip =
        a.eps_row ? static_cast<uint32_t>(eps_parity(arow, load_bits(a.eps_col, a.eps_col_hi, c))) : 0u;
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

    const Bits arow = a.eps_row ? load_bits(a.eps_row, a.eps_row_hi, row) : Bits();
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
// RT > 0 (tail launches): RT column groups of 32 per lane instead of the
// default R, so the partial last chunk (e.g. 40 of 128 columns at C3) does not
// walk every entry for R x 32 clamped columns.
template <bool kTail, int M, int GW, bool kV2 = false, int RT = 0>
__global__ void __launch_bounds__(GW * kWarp, kSSMinBlocks / GW)
k_samespin_g(const SameSpinArgs a, uint32_t chunk0, uint32_t ngroups) {
    constexpr int kGW = GW;
    constexpr int R = RT > 0 ? RT : SSR<M>::value;
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
    const uint32_t col0 = chunk * (kWarp * SSR<M>::value) + lane;

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

    const Bits arow = a.eps_row ? load_bits(a.eps_row, a.eps_row_hi, row) : Bits();
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const uint32_t c = kV2 ? chunk * (kWarp * R) + (q / 2) * 2 * kWarp + 2 * lane + (q % 2) : col0 + q * kWarp;
        if (kTail && c >= a.ncols) continue;
        samespin_store<M>(a, arow, r, c, acc[q]);
    }
}

} // namespace

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
    // favour L1 over shared memory (the kernel uses <= 32 KB)
    ensure_carveout(reinterpret_cast<const void*>(k_samespin_g<false, M, GW>), 10);
    ensure_carveout(reinterpret_cast<const void*>(k_samespin_g<true, M, GW>), 10);
    if constexpr (M == 1) ensure_carveout(reinterpret_cast<const void*>(k_samespin_g<false, 1, GW, true>), 10);
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
        const uint32_t tail_cols = s.ncols - static_cast<uint32_t>(full) * kChunk;
        if (SSR<M>::value > 1 && tail_cols <= kWarp) {
            ensure_carveout(reinterpret_cast<const void*>(k_samespin_g<true, M, GW, false, 1>), 10);
            k_samespin_g<true, M, GW, false, 1><<<ngroups, GW * kWarp, 0, st>>>(s, static_cast<uint32_t>(full), ngroups);
        } else if (SSR<M>::value > 2 && tail_cols <= 2 * kWarp) {
            ensure_carveout(reinterpret_cast<const void*>(k_samespin_g<true, M, GW, false, 2>), 10);
            k_samespin_g<true, M, GW, false, 2><<<ngroups, GW * kWarp, 0, st>>>(s, static_cast<uint32_t>(full), ngroups);
        } else {
            k_samespin_g<true, M, GW><<<ngroups, GW * kWarp, 0, st>>>(s, static_cast<uint32_t>(full), ngroups);
        }
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
                  const MPtrs& y_loc, uint64_t a0, uint64_t a1, bool first, bool add_to_y) {
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
    s.eps_row_hi = h.ch[0].hi();
    s.eps_col_hi = h.ch[1].prefix_hi_p();
    s.diag = first ? h.diag.p + (a0 - h.a0) * h.nb() : nullptr;
    s.accumulate = (first && !add_to_y) ? 0 : 1;   // first && add_to_y: y += diag*C + alpha
    launch_samespin<M>(s, h.stream);
}


template void launch_samespin<1>(const SameSpinArgs&, cudaStream_t);
template void launch_samespin<2>(const SameSpinArgs&, cudaStream_t);
template void launch_samespin<4>(const SameSpinArgs&, cudaStream_t);
template void launch_alpha<1>(const Handle&, const Ptrs&, uint32_t, uint32_t, const Ptrs&, const MPtrs&, uint64_t,
                              uint64_t, bool, bool);
template void launch_alpha<2>(const Handle&, const Ptrs&, uint32_t, uint32_t, const Ptrs&, const MPtrs&, uint64_t,
                              uint64_t, bool, bool);
template void launch_alpha<4>(const Handle&, const Ptrs&, uint32_t, uint32_t, const Ptrs&, const MPtrs&, uint64_t,
                              uint64_t, bool, bool);

} // namespace detci_gpu
