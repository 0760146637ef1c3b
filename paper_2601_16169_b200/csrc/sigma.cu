// sigma = H C over the alpha x beta tensor-product basis (matvec,
// matvec.cpp:125-228), B200-native.
//
//   y  = diag*C + sum_ja Ha(ia,ja;B_ib) C[ja,ib]              k_samespin on C
//   yT =          sum_jb Hb(ib,jb;A_ia) C^T[jb,ia]            k_samespin on C^T
//   y += sum_ja sum_jb Hm C[ja,jb]                            k_mixed
//   y += yT^T                                                 k_transpose_add
//
// Gather formulation: every output element is owned by exactly one thread,
// so there are no atomics and the result is deterministic.  The beta term
// runs the alpha kernel on the transposed block, which turns its per-row
// gathers into coalesced row reads (the transposes cost 32 B/det against
// ~8 B x thousands of elements per det).
//
// Multi-GPU / virtual blocks: alpha rows are partitioned into P blocks;
// the alpha and mixed terms need C rows from every block, which rotate
// ring-wise (NCCL send/recv on a comm stream, double-buffered, overlapped
// with the compute of the resident block).  The beta term and diagonal are
// block-local.
#include <algorithm>
#include <vector>

#include "formulas.cuh"
#include "handle.hpp"

namespace detci_gpu {

namespace {

// ---------------------------------------------------------------------------
// Same-spin kernel.  CTA = (output row, column chunk); threads own R columns
// each (coalesced), loop over the row's helper-list entries staged in smem.
// Per element: one coalesced 8 B load of C[ja, col], AND+POPC against the
// spectator string, sign flip, DFMA (+ one coalesced J load for singles).
// Grid is chunk-major so CTAs in flight share C[:, chunk] in L2.
// ---------------------------------------------------------------------------
constexpr int kSSBlock = 128;
constexpr int kSSR = 4;
constexpr int kStage = 256;

struct SameSpinArgs {
    const double* C;        // C row ja at C + (ja - c_row0) * ldc
    size_t ldc;
    uint32_t c_row0, j0, j1;  // window [j0, j1) of target rows
    double* Y;              // output row r at Y + r * ldy
    size_t ldy;
    uint32_t row0, nrows;   // list rows [row0, row0 + nrows)
    uint32_t ncols;
    const uint64_t* spec;   // spectator string per column
    const double* J;        // J[tri * ldj + col]
    size_t ldj;
    const uint32_t* flat[2];
    const uint64_t* off[2];
    const uint32_t* len[2];
    const double* pv[2];
    const uint64_t* pm[2];
    const uint32_t* pab;
    const double* diag;     // if set (write mode): Y = diag * Cself + acc
    const double* Cself;
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

// (-1)^{popc(S & M)} applied to the high word of x: parity of a 64-bit AND
// via one 32-bit POPC of (lo ^ hi).
__device__ __forceinline__ double spectator_signed(double x, uint32_t slo, uint32_t shi, uint32_t mlo,
                                                   uint32_t mhi) {
    const uint32_t par = __popc((slo & mlo) ^ (shi & mhi));
    return __hiloint2double(__double2hiint(x) ^ static_cast<int>(par << 31), __double2loint(x));
}

// kTail: the CTA's column chunk crosses ncols, so column indices are clamped
// (loads stay in bounds, stores are masked); full chunks use one base
// pointer per entry with immediate offsets.
template <bool kTail>
__global__ void __launch_bounds__(kSSBlock)
k_samespin(const SameSpinArgs a, uint32_t chunk0) {
    __shared__ uint32_t s_ja[kStage];
    __shared__ double s_v[kStage];
    __shared__ uint64_t s_m[kStage];
    __shared__ uint32_t s_ab[kStage];
    __shared__ uint64_t s_range[4];

    const uint32_t r = blockIdx.x % a.nrows;
    const uint32_t chunk = chunk0 + blockIdx.x / a.nrows;
    const uint32_t row = a.row0 + r;
    const uint32_t tid = threadIdx.x;
    const uint32_t col0 = chunk * (kSSBlock * kSSR) + tid;

    uint32_t col[kSSR];
    uint32_t slo[kSSR], shi[kSSR];
    double acc[kSSR];
#pragma unroll
    for (int q = 0; q < kSSR; ++q) {
        const uint32_t c = col0 + q * kSSBlock;
        col[q] = kTail ? min(c, a.ncols - 1) : c;
        const uint64_t sp = a.spec[col[q]];
        slo[q] = static_cast<uint32_t>(sp);
        shi[q] = static_cast<uint32_t>(sp >> 32);
        acc[q] = 0.0;
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
                s_m[t] = a.pm[kind][k0 + t];
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
                    const uint64_t m = s_m[e];
                    const uint32_t mlo = static_cast<uint32_t>(m), mhi = static_cast<uint32_t>(m >> 32);
                    const uint32_t jsign = ab & 0x80000000u;
#pragma unroll
                    for (int q = 0; q < kSSR; ++q) {
                        const uint32_t cq = kTail ? col[q] : col0 + q * kSSBlock;
                        const double c = __ldg(a.C + rowoff + cq);
                        const double j = __ldg(jrow + cq);
                        const double val =
                            v + __hiloint2double(__double2hiint(j) ^ static_cast<int>(jsign), __double2loint(j));
                        acc[q] = fma(val, spectator_signed(c, slo[q], shi[q], mlo, mhi), acc[q]);
                    }
                }
            } else {
#pragma unroll 4
                for (int e = 0; e < cnt; ++e) {
                    const double* base = a.C + static_cast<size_t>(s_ja[e]) * a.ldc + (kTail ? 0 : col0);
                    const double v = s_v[e];
                    const uint64_t m = s_m[e];
                    const uint32_t mlo = static_cast<uint32_t>(m), mhi = static_cast<uint32_t>(m >> 32);
#pragma unroll
                    for (int q = 0; q < kSSR; ++q) {
                        const double c = __ldg(kTail ? base + col[q] : base + q * kSSBlock);
                        acc[q] = fma(v, spectator_signed(c, slo[q], shi[q], mlo, mhi), acc[q]);
                    }
                }
            }
        }
    }

#pragma unroll
    for (int q = 0; q < kSSR; ++q) {
        const uint32_t c = col0 + q * kSSBlock;
        if (kTail && c >= a.ncols) continue;
        const size_t yi = static_cast<size_t>(r) * a.ldy + c;
        if (a.accumulate) {
            a.Y[yi] += acc[q];
        } else if (a.diag) {
            a.Y[yi] = fma(a.diag[yi], a.Cself[yi], acc[q]);
        } else {
            a.Y[yi] = acc[q];
        }
    }
}

// ---------------------------------------------------------------------------
// Mixed alpha-beta kernel.  CTA = (output row ia, column part of
// kMxBlock*kMxR beta strings).  For each alpha single ja of ia in the window:
//   W[cd] = (pa qa|c d) (-1)^{popc(A_ja & Mbeta(c,d))}   built in smem,
//   C[ja, segment] staged in smem (cp.async),
// then each thread walks its beta strings' singles from the SELL-32 table
// (one coalesced 4 B entry per element) gathering W[cd] and C[ja, jb] from
// smem.  The ib-dependent alpha sign is applied once per (ja, ib).
// ---------------------------------------------------------------------------
constexpr int kMxBlock = 1024;   // one CTA per SM, 32 warps
constexpr int kMxR = 2;          // beta slots per thread -> 2048 slots per CTA

struct MixedArgs {
    const double* C;
    size_t ldc;
    uint32_t c_row0, j0, j1;
    double* Y;
    size_t ldy;
    uint32_t row0, nrows, nb, nparts;
    const uint64_t* alpha;
    const uint64_t* beta;
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
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_prev() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// Stage = (alpha single ja, column segment g).  Two stage buffers, each
// [ +W | -W | C[ja, segment] ]; the next stage's row segment streams in with
// cp.async (and its W is built) while the current one is consumed.
__global__ void __launch_bounds__(kMxBlock, 1)
k_mixed(const MixedArgs a) {
    extern __shared__ double smem[];
    const int nn = a.norbs * a.norbs;
    const uint32_t wdbl = static_cast<uint32_t>((2 * nn + 1) & ~1);
    const uint32_t stage_dbl = wdbl + ((a.seg_cols + 1) & ~1u);

    const uint32_t r = blockIdx.x / a.nparts;
    const uint32_t part = blockIdx.x % a.nparts;
    const uint32_t ia = a.row0 + r;
    const uint32_t tid = threadIdx.x;
    const uint32_t lane = tid % kWarp;
    const uint64_t A = a.alpha[ia];

    uint64_t B[kMxR];
    uint32_t slice[kMxR];
    double sig[kMxR], acc[kMxR];
#pragma unroll
    for (int q = 0; q < kMxR; ++q) {
        const uint32_t slot = part * (kMxBlock * kMxR) + q * kMxBlock + tid;
        B[q] = a.beta[a.perm[min(slot, a.nb - 1)]];
        slice[q] = slot / kWarp;
        sig[q] = 0.0;
        acc[q] = 0.0;
    }

    const uint64_t o = a.sa_off[ia];
    const uint32_t n = a.sa_len[ia];
    const uint32_t* f = a.sa_flat + o;
    const uint32_t kb = a.j0 == 0 ? 0 : lower_bound_u32(f, n, a.j0);
    const uint32_t ke = lower_bound_u32(f, n, a.j1);
    const uint32_t nstages = (ke - kb) * a.nseg;

    // issue stage i into buffer i & 1: C row segment (async) + +-W (threads)
    auto issue = [&](uint32_t i) {
        double* buf = smem + (i & 1) * stage_dbl;
        const uint32_t k = kb + i / a.nseg, g = i % a.nseg;
        const uint32_t ja = f[k];
        const double* src = a.C + static_cast<size_t>(ja - a.c_row0) * a.ldc + g * a.seg_cols;
        const uint32_t segw = min(a.seg_cols, a.nb - g * a.seg_cols);
        double* crow = buf + wdbl;
        for (uint32_t c = tid; c < segw; c += kMxBlock) cp_async8(crow + c, src + c);
        cp_async_commit();
        const uint64_t Ak = a.alpha[ja];
        const int pa = __ffsll(static_cast<long long>(A & ~Ak)) - 1;
        const int qa = __ffsll(static_cast<long long>(Ak & ~A)) - 1;
        const double* erow = a.eri + static_cast<size_t>(pa * a.norbs + qa) * nn;
        for (int cd = tid; cd < nn; cd += kMxBlock) {
            const int c = cd / a.norbs, d = cd - c * a.norbs;
            double v = 0.0;
            if (c != d) {
                v = erow[cd];
                if (__popcll(Ak & spectator_mask(1, c, d)) & 1) v = -v;
            }
            buf[cd] = v;
            buf[nn + cd] = -v;
        }
    };

    if (nstages > 0) issue(0);
#pragma unroll 1
    for (uint32_t i = 0; i < nstages; ++i) {
        if (i + 1 < nstages) {
            issue(i + 1);          // buffer (i+1)&1 was released by the barrier ending stage i-1
            cp_async_wait_prev();  // stage i's row has landed
        } else {
            cp_async_wait_all();
        }
        __syncthreads();
        const char* wbase = reinterpret_cast<const char*>(smem + (i & 1) * stage_dbl);
        const char* cbase = reinterpret_cast<const char*>(smem + (i & 1) * stage_dbl + wdbl);
        const uint32_t g = i % a.nseg;
#pragma unroll
        for (int q = 0; q < kMxR; ++q) {
            if (slice[q] >= a.nslices) continue;
            const uint32_t L = a.sell_len[slice[q] * a.nseg + g];
            const uint32_t* ent = a.sell + a.sell_off[slice[q] * a.nseg + g] + lane;
            double s0 = 0.0, s1 = 0.0;
            uint32_t t = 0;
#pragma unroll 1
            for (; t + 8 <= L; t += 8) {
                uint32_t e[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) e[u] = __ldg(ent + static_cast<size_t>(t + u) * kWarp);
#pragma unroll
                for (int u = 0; u < 8; u += 2) {
                    const double w0 = *reinterpret_cast<const double*>(wbase + ((e[u] >> 17) << 3));
                    const double c0 = *reinterpret_cast<const double*>(cbase + (e[u] & 0x1ffffu));
                    const double w1 = *reinterpret_cast<const double*>(wbase + ((e[u + 1] >> 17) << 3));
                    const double c1 = *reinterpret_cast<const double*>(cbase + (e[u + 1] & 0x1ffffu));
                    s0 = fma(w0, c0, s0);
                    s1 = fma(w1, c1, s1);
                }
            }
#pragma unroll 1
            for (; t < L; ++t) {
                const uint32_t e0 = __ldg(ent + static_cast<size_t>(t) * kWarp);
                const double w0 = *reinterpret_cast<const double*>(wbase + ((e0 >> 17) << 3));
                const double c0 = *reinterpret_cast<const double*>(cbase + (e0 & 0x1ffffu));
                s0 = fma(w0, c0, s0);
            }
            acc[q] += s0 + s1;
        }
        if (g + 1 == a.nseg) {  // last segment of this ja: apply the alpha sign
            const uint32_t ja = f[kb + i / a.nseg];
            const uint64_t Ak = a.alpha[ja];
            const int pa = __ffsll(static_cast<long long>(A & ~Ak)) - 1;
            const int qa = __ffsll(static_cast<long long>(Ak & ~A)) - 1;
            const int sA = __popcll(A & open_mask(pa, qa)) & 1;
            const uint64_t ma = spectator_mask(0, pa, qa);
#pragma unroll
            for (int q = 0; q < kMxR; ++q) {
                sig[q] += flip_sign(acc[q], static_cast<uint32_t>(sA ^ (__popcll(B[q] & ma) & 1)));
                acc[q] = 0.0;
            }
        }
        __syncthreads();  // buffer i&1 free for stage i+2
    }

#pragma unroll
    for (int q = 0; q < kMxR; ++q) {
        const uint32_t slot = part * (kMxBlock * kMxR) + q * kMxBlock + tid;
        if (slot < a.nb) a.Y[static_cast<size_t>(r) * a.ldy + a.perm[slot]] += sig[q];
    }
}

// ---------------------------------------------------------------------------
// Transposes through 32x32 smem tiles (coalesced both ways).
// ---------------------------------------------------------------------------
constexpr int kTile = 32;

// dst[c * ldd + r] = src[r * lds + c], src rows x cols
__global__ void k_transpose(const double* __restrict__ src, size_t lds, double* __restrict__ dst,
                            size_t ldd, uint32_t rows, uint32_t cols) {
    __shared__ double tile[kTile][kTile + 1];
    const uint32_t c0 = blockIdx.x * kTile, r0 = blockIdx.y * kTile;
    for (uint32_t y = threadIdx.y; y < kTile; y += blockDim.y) {
        const uint32_t rr = r0 + y, cc = c0 + threadIdx.x;
        if (rr < rows && cc < cols) tile[y][threadIdx.x] = src[static_cast<size_t>(rr) * lds + cc];
    }
    __syncthreads();
    for (uint32_t y = threadIdx.y; y < kTile; y += blockDim.y) {
        const uint32_t cc = c0 + y, rr = r0 + threadIdx.x;
        if (rr < rows && cc < cols) dst[static_cast<size_t>(cc) * ldd + rr] = tile[threadIdx.x][y];
    }
}

// dst[r * ldd + c] += src[c * lds + r], dst rows x cols
__global__ void k_transpose_add(const double* __restrict__ src, size_t lds,
                                double* __restrict__ dst, size_t ldd, uint32_t rows,
                                uint32_t cols) {
    __shared__ double tile[kTile][kTile + 1];
    const uint32_t c0 = blockIdx.x * kTile, r0 = blockIdx.y * kTile;
    for (uint32_t y = threadIdx.y; y < kTile; y += blockDim.y) {
        const uint32_t cc = c0 + y, rr = r0 + threadIdx.x;
        if (rr < rows && cc < cols) tile[y][threadIdx.x] = src[static_cast<size_t>(cc) * lds + rr];
    }
    __syncthreads();
    for (uint32_t y = threadIdx.y; y < kTile; y += blockDim.y) {
        const uint32_t rr = r0 + y, cc = c0 + threadIdx.x;
        if (rr < rows && cc < cols) dst[static_cast<size_t>(rr) * ldd + cc] += tile[threadIdx.x][y];
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

SameSpinArgs alpha_args(const Handle& h, const double* Cb, uint32_t b0, uint32_t b1,
                        const double* x_loc, double* y_loc, uint64_t a0, uint64_t a1, bool first) {
    const ChannelTables& A = h.ch[0];
    const ChannelTables& B = h.ch[1];
    SameSpinArgs s{};
    s.C = Cb;
    s.ldc = h.nb();
    s.c_row0 = b0;
    s.j0 = b0;
    s.j1 = b1;
    s.Y = y_loc;
    s.ldy = h.nb();
    s.row0 = static_cast<uint32_t>(a0);
    s.nrows = static_cast<uint32_t>(a1 - a0);
    s.ncols = static_cast<uint32_t>(h.nb());
    s.spec = B.strings.p;
    s.J = B.J.p;
    s.ldj = h.nb();
    for (int k = 0; k < 2; ++k) {
        s.flat[k] = A.flat[k].p;
        s.off[k] = A.offset[k].p;
        s.len[k] = A.len[k].p;
        s.pv[k] = A.pv[k].p;
        s.pm[k] = A.pmask[k].p;
    }
    s.pab = A.pab.p;
    s.diag = first ? h.diag.p + (a0 - h.a0) * h.nb() : nullptr;
    s.Cself = x_loc;
    s.accumulate = first ? 0 : 1;
    return s;
}

void launch_samespin(const SameSpinArgs& s, cudaStream_t st) {
    if (s.nrows == 0 || s.ncols == 0) return;
    constexpr uint32_t kChunk = kSSBlock * kSSR;
    const uint64_t full = s.ncols / kChunk;
    const bool tail = s.ncols % kChunk != 0;
    if (full) {
        k_samespin<false><<<static_cast<unsigned>(full * s.nrows), kSSBlock, 0, st>>>(s, 0);
        CUDA_LAUNCH_CHECK();
    }
    if (tail) {
        k_samespin<true><<<s.nrows, kSSBlock, 0, st>>>(s, static_cast<uint32_t>(full));
        CUDA_LAUNCH_CHECK();
    }
}

size_t mixed_smem(const Handle& h) {
    const size_t nn = static_cast<size_t>(h.norbs) * h.norbs;
    return 2 * (((2 * nn + 1) & ~size_t{1}) + ((h.seg_cols + 1) & ~size_t{1})) * sizeof(double);
}

void launch_mixed(const Handle& h, const double* Cb, uint32_t b0, uint32_t b1, double* y_loc,
                  uint64_t a0, uint64_t a1, cudaStream_t st) {
    MixedArgs m{};
    m.C = Cb;
    m.ldc = h.nb();
    m.c_row0 = b0;
    m.j0 = b0;
    m.j1 = b1;
    m.Y = y_loc;
    m.ldy = h.nb();
    m.row0 = static_cast<uint32_t>(a0);
    m.nrows = static_cast<uint32_t>(a1 - a0);
    m.nb = static_cast<uint32_t>(h.nb());
    m.nparts = (m.nb + kMxBlock * kMxR - 1) / (kMxBlock * kMxR);
    m.alpha = h.ch[0].strings.p;
    m.beta = h.ch[1].strings.p;
    m.sa_flat = h.ch[0].flat[0].p;
    m.sa_off = h.ch[0].offset[0].p;
    m.sa_len = h.ch[0].len[0].p;
    m.sell = h.sell.p;
    m.sell_off = h.sell_off.p;
    m.sell_len = h.sell_len.p;
    m.perm = h.sell_perm.p;
    m.seg_cols = h.seg_cols;
    m.nseg = h.nseg;
    m.nslices = h.nslices;
    m.eri = h.d_eri.p;
    m.norbs = h.norbs;
    if (m.nrows == 0) return;
    const size_t smem = mixed_smem(h);
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        CUDA_CHECK(cudaFuncSetAttribute(k_mixed, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
        configured = smem;
    }
    const uint64_t grid = static_cast<uint64_t>(m.nrows) * m.nparts;
    k_mixed<<<static_cast<unsigned>(grid), kMxBlock, smem, st>>>(m);
    CUDA_LAUNCH_CHECK();
}

// The beta term for rows [a0, a1): transpose, same-spin kernel on C^T with
// the alpha strings as spectators, result in h.yt ([nb][nloc]).
void beta_term(Handle& h, const double* x_loc, uint64_t a0, uint64_t a1, PhaseTimer& tm) {
    const uint32_t nloc = static_cast<uint32_t>(a1 - a0), nb = static_cast<uint32_t>(h.nb());
    const int id = tm.begin(1);
    dim3 tb(kTile, 8), tg((nb + kTile - 1) / kTile, (nloc + kTile - 1) / kTile);
    k_transpose<<<tg, tb, 0, h.stream>>>(x_loc, nb, h.ct.p, nloc, nloc, nb);
    CUDA_LAUNCH_CHECK();
    const ChannelTables& A = h.ch[0];
    const ChannelTables& B = h.ch[1];
    SameSpinArgs s{};
    s.C = h.ct.p;
    s.ldc = nloc;
    s.c_row0 = 0;
    s.j0 = 0;
    s.j1 = nb;
    s.Y = h.yt.p;
    s.ldy = nloc;
    s.row0 = 0;
    s.nrows = nb;
    s.ncols = nloc;
    s.spec = A.strings.p + a0;
    s.J = A.J.p + a0;
    s.ldj = h.na();
    for (int k = 0; k < 2; ++k) {
        s.flat[k] = B.flat[k].p;
        s.off[k] = B.offset[k].p;
        s.len[k] = B.len[k].p;
        s.pv[k] = B.pv[k].p;
        s.pm[k] = B.pmask[k].p;
    }
    s.pab = B.pab.p;
    s.accumulate = 0;
    launch_samespin(s, h.stream);
    tm.end(id);
}

void combine(Handle& h, double* y_loc, uint64_t a0, uint64_t a1, PhaseTimer& tm) {
    const uint32_t nloc = static_cast<uint32_t>(a1 - a0), nb = static_cast<uint32_t>(h.nb());
    const int id = tm.begin(3);
    dim3 tb(kTile, 8), tg((nb + kTile - 1) / kTile, (nloc + kTile - 1) / kTile);
    k_transpose_add<<<tg, tb, 0, h.stream>>>(h.yt.p, nloc, y_loc, nb, nloc, nb);
    CUDA_LAUNCH_CHECK();
    tm.end(id);
}

// One block-rank's sigma with the C ring.  `fetch(s, dst, block)` enqueues on
// h.comm_stream the transfer that makes block `block` resident in dst for
// step s (NCCL send/recv, or a device copy for virtual blocks).
template <class Fetch>
void sigma_ring(Handle& h, int g, int P, const double* x_loc, double* y_loc, PhaseTimer& tm,
                Fetch&& fetch) {
    const uint64_t a0 = h.blk[g], a1 = h.blk[g + 1];
    cudaEvent_t* done_compute = h.ev;      // [0..1]
    cudaEvent_t* done_comm = h.ev + 2;     // [2..3]
    // x and the ring buffers are produced / last read on the compute stream:
    // the comm stream must not send or overwrite them before that work ends.
    CUDA_CHECK(cudaEventRecord(h.ev[4], h.stream));
    CUDA_CHECK(cudaStreamWaitEvent(h.comm_stream, h.ev[4], 0));
    beta_term(h, x_loc, a0, a1, tm);
    const double* held = x_loc;
    for (int s = 0; s < P; ++s) {
        const int b = (g + s) % P;
        if (s + 1 < P) {
            // ring[s%2] was read by compute at step s-1
            if (s >= 1) CUDA_CHECK(cudaStreamWaitEvent(h.comm_stream, done_compute[(s - 1) % 2], 0));
            fetch(s, held, h.ring[s % 2].p, (g + s + 1) % P);
            CUDA_CHECK(cudaEventRecord(done_comm[s % 2], h.comm_stream));
        }
        const uint32_t b0 = static_cast<uint32_t>(h.blk[b]), b1 = static_cast<uint32_t>(h.blk[b + 1]);
        int id = tm.begin(0);
        launch_samespin(alpha_args(h, held, b0, b1, x_loc, y_loc, a0, a1, s == 0), h.stream);
        tm.end(id);
        id = tm.begin(2);
        launch_mixed(h, held, b0, b1, y_loc, a0, a1, h.stream);
        tm.end(id);
        CUDA_CHECK(cudaEventRecord(done_compute[s % 2], h.stream));
        if (s + 1 < P) {
            CUDA_CHECK(cudaStreamWaitEvent(h.stream, done_comm[s % 2], 0));
            held = h.ring[s % 2].p;
        }
    }
    combine(h, y_loc, a0, a1, tm);
}

} // namespace

namespace {

void sigma_schedule(Handle& h, const double* dx, double* dy, PhaseTimer& tm) {
    const size_t nb = h.nb();
    const int P = std::max(h.world, h.vblocks);
    if (h.world > 1) {
        const int g = h.rank;
        sigma_ring(h, g, P, dx, dy, tm, [&](int s, const double* held, double* dst, int next) {
            const int cur = (g + s) % P;
            const size_t send_n = (h.blk[cur + 1] - h.blk[cur]) * nb;
            const size_t recv_n = (h.blk[next + 1] - h.blk[next]) * nb;
            if (ncclGroupStart() != ncclSuccess) fail(DETCI_GPU_E_CUDA, "ncclGroupStart");
            ncclSend(held, send_n, ncclDouble, (g - 1 + P) % P, h.nccl, h.comm_stream);
            ncclRecv(dst, recv_n, ncclDouble, (g + 1) % P, h.nccl, h.comm_stream);
            if (ncclGroupEnd() != ncclSuccess) fail(DETCI_GPU_E_CUDA, "ncclGroupEnd (ring)");
        });
    } else if (P > 1) {
        // Virtual blocks: every block-rank's schedule runs in turn on this GPU;
        // the ring transport is a device copy out of the full x.
        for (int g = 0; g < P; ++g) {
            const double* xg = dx + h.blk[g] * nb;
            double* yg = dy + h.blk[g] * nb;
            sigma_ring(h, g, P, xg, yg, tm, [&](int, const double*, double* dst, int next) {
                const size_t n = (h.blk[next + 1] - h.blk[next]) * nb;
                CUDA_CHECK(cudaMemcpyAsync(dst, dx + h.blk[next] * nb, n * sizeof(double),
                                           cudaMemcpyDeviceToDevice, h.comm_stream));
            });
        }
    } else {
        sigma_ring(h, 0, 1, dx, dy, tm, [](int, const double*, double*, int) {});
    }
}

} // namespace

void sigma_enqueue(Handle& h, const double* dx, double* dy) {
    if (!h.built) fail(DETCI_GPU_E_INPUT, "sigma: basis not built");
    PhaseTimer tm(h, false);
    sigma_schedule(h, dx, dy, tm);
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
