// Device-resident Davidson (davidson_solve, davidson.cpp:73-206).
//
// Every per-iteration vector operation is a fused, bandwidth-bound kernel
// over HBM-resident vectors; only scalars (<= 2k dot products, two norms)
// cross to the host, where the k x k Rayleigh-Ritz problem is solved
// (Jacobi on the lower triangle, as Eigen's SelfAdjointEigenSolver reads
// it).  Reductions are two-stage with a fixed order, so a run is bitwise
// reproducible; with several GPUs the per-rank partials are summed with
// an all-reduce over the rank transport (comm.hpp) before use.  Algorithmic rules kept from the reference:
// argmin-diagonal guess with lowest-index ties, lower-triangle projected
// fill, 2-pass modified Gram-Schmidt with the 1e-10 dependence threshold,
// the 1e-8 preconditioner clamp, collapse to the Ritz pair at
// max_subspace, and the per-iteration trace (Gram deviation included).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "handle.hpp"
#include "sigma_device.cuh"

namespace detci_gpu {

namespace {

constexpr int kRedBlocks = 592;   // 4 x 148 SMs
constexpr int kRedThreads = 256;
constexpr int kMaxVec = 64;

struct VecList {
    const double* p[2 * kMaxVec];
};

__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int s = 16; s > 0; s >>= 1) v += __shfl_down_sync(0xffffffffu, v, s);
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : 0.0;
        for (int s = 16; s > 0; s >>= 1) t += __shfl_down_sync(0xffffffffu, t, s);
    }
    return t;  // valid in thread 0
}

// Vector kernels process kU elements per thread per step (stride
// blockDim.x, coalesced) so that every thread keeps several independent
// loads in flight: one outstanding load per thread reaches only a fraction
// of HBM bandwidth at 592 x 256 threads.
constexpr int kU = 4;

// Tiles of kU * blockDim.x consecutive elements, grid-strided so that all
// blocks sweep memory together (per-block contiguous chunks would open
// hundreds of concurrent DRAM streams per vector).
#define TILE_LOOP(i0, n)                                                                          \
    for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * kU * blockDim.x + threadIdx.x; i0 < (n); \
         i0 += static_cast<uint64_t>(gridDim.x) * kU * blockDim.x)

// partial[j * gridDim.x + blk] = sum over this block's tiles of x * y_j
// (groups of 8 vectors per sweep: x is re-read per group).
__global__ void __launch_bounds__(kRedThreads)
k_dot_many(const double* __restrict__ x, VecList ys, int k, uint64_t n, double* __restrict__ partial) {
    __shared__ double sh[32];
    const uint64_t e = n;
    for (int j0 = 0; j0 < k; j0 += 8) {
        const int kk = min(8, k - j0);
        double acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.0;
        TILE_LOOP(i0, e) {
            double xv[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint64_t i = i0 + static_cast<uint64_t>(u) * blockDim.x;
                xv[u] = i < e ? x[i] : 0.0;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (j < kk) {
                    const double* y = ys.p[j0 + j];
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const uint64_t i = i0 + static_cast<uint64_t>(u) * blockDim.x;
                        if (i < e) acc[j] = fma(xv[u], y[i], acc[j]);
                    }
                }
            }
        }
        for (int j = 0; j < kk; ++j) {
            const double s = block_sum(acc[j], sh);
            if (threadIdx.x == 0) partial[static_cast<size_t>(j0 + j) * gridDim.x + blockIdx.x] = s;
        }
    }
}

// out[j] = sum_b partial[j * nblk + b], fixed order (one warp per j)
__global__ void k_finalize(const double* __restrict__ partial, int nblk, int k, double* __restrict__ out) {
    const int j = blockIdx.x;
    if (j >= k) return;
    double v = 0.0;
    for (int b = threadIdx.x; b < nblk; b += 32) v += partial[static_cast<size_t>(j) * nblk + b];
    for (int s = 16; s > 0; s >>= 1) v += __shfl_down_sync(0xffffffffu, v, s);
    if (threadIdx.x == 0) out[j] = v;
}

struct RitzArgs {
    const double* v[kMaxVec];
    const double* w[kMaxVec];
    double c[kMaxVec];
    int k;
    double theta;
};

// ritz = sum c_j v_j, img = sum c_j w_j, res = img - theta ritz,
// corr = res / clamp(diag - theta); partials of |res|^2 and |corr|^2.
// (davidson.cpp:134-146 and precondition, :59-71)
__global__ void __launch_bounds__(kRedThreads)
k_ritz(const RitzArgs a, const double* __restrict__ diag, uint64_t n, double* __restrict__ ritz,
       double* __restrict__ img, double* __restrict__ corr, double* __restrict__ partial) {
    __shared__ double sh[32];
    double rr = 0.0, cc = 0.0;
    const uint64_t e = n;
    TILE_LOOP(i0, e) {
        double r[kU], m[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) r[u] = m[u] = 0.0;
        for (int j = 0; j < a.k; ++j) {
            const double cj = a.c[j];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint64_t i = i0 + static_cast<uint64_t>(u) * blockDim.x;
                if (i < e) {
                    r[u] += cj * a.v[j][i];
                    m[u] += cj * a.w[j][i];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint64_t i = i0 + static_cast<uint64_t>(u) * blockDim.x;
            if (i >= e) continue;
            ritz[i] = r[u];
            img[i] = m[u];
            const double res = m[u] - a.theta * r[u];
            double denom = diag[i] - a.theta;
            if (fabs(denom) < 1e-8) denom = copysign(1e-8, denom);
            const double cr = res / denom;
            corr[i] = cr;
            rr += res * res;
            cc += cr * cr;
        }
    }
    const double s1 = block_sum(rr, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s1;
    const double s2 = block_sum(cc, sh);
    if (threadIdx.x == 0) partial[gridDim.x + blockIdx.x] = s2;
}

// One modified Gram-Schmidt step: cand -= (*o_prev) vprev (if vprev), then
// partial of <vnext, cand> (or |cand|^2 when vnext is null).  When src is
// set the step starts from cand = src / divisor.
__global__ void __launch_bounds__(kRedThreads)
k_mgs_step(double* __restrict__ cand, const double* __restrict__ src, double divisor,
           const double* __restrict__ vprev, const double* __restrict__ o_prev,
           const double* __restrict__ vnext, uint64_t n, double* __restrict__ partial) {
    __shared__ double sh[32];
    const double o = vprev ? *o_prev : 0.0;
    double acc = 0.0;
    const uint64_t e = n;
    TILE_LOOP(i0, e) {
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint64_t i = i0 + static_cast<uint64_t>(u) * blockDim.x;
            if (i >= e) continue;
            double c = src ? src[i] / divisor : cand[i];
            if (vprev) c -= o * vprev[i];
            cand[i] = c;
            acc += (vnext ? vnext[i] : c) * c;
        }
    }
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// Classical Gram-Schmidt update over the whole subspace in one pass:
// dst = (src - sum_j d[j] v_j) * scale, d on the device (finalized dots);
// with `partial`, also the block partials of |dst|^2.  dst may alias src.
__global__ void __launch_bounds__(kRedThreads)
k_combine(double* dst, const double* src, double scale, VecList v, const double* __restrict__ d, int k,
          uint64_t n, double* __restrict__ partial) {
    __shared__ double sd[kMaxVec];
    __shared__ double sh[32];
    for (int j = threadIdx.x; j < k; j += blockDim.x) sd[j] = d[j];
    __syncthreads();
    double acc = 0.0;
    const uint64_t e = n;
    TILE_LOOP(i0, e) {
        double sv[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint64_t i = i0 + static_cast<uint64_t>(u) * blockDim.x;
            sv[u] = i < e ? src[i] : 0.0;
        }
        for (int j = 0; j < k; ++j) {
            const double dj = sd[j];
            const double* vj = v.p[j];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint64_t i = i0 + static_cast<uint64_t>(u) * blockDim.x;
                if (i < e) sv[u] -= dj * vj[i];
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint64_t i = i0 + static_cast<uint64_t>(u) * blockDim.x;
            if (i >= e) continue;
            const double t = sv[u] * scale;
            dst[i] = t;
            acc += t * t;
        }
    }
    if (partial) {
        const double t = block_sum(acc, sh);
        if (threadIdx.x == 0) partial[blockIdx.x] = t;
    }
}

// ---------------------------------------------------------------------------
// Fused single-root iteration passes over the subspace (davidson.cpp:126-176
// restated as 3 + 1 streaming passes instead of ~6.5k vector passes).
// Every pass streams ns vectors tile by tile into shared memory with 1-D TMA
// bulk copies (one elected thread, NS-stage mbarrier ring, one persistent
// CTA per SM), so the bytes in flight do not depend on the thread count;
// the element-wise part reads the staged tiles, and the dot products of
// the pass (one stream against a per-element "probe") are accumulated per
// warp (warp w owns subspace vectors w, w + 8, ...) and written as per-CTA
// partials for the fixed-order finalize.
//   kPassProj  streams x, w_0..w_{k-1}:     <x, w_j>                    (projected row)
//   kPassRitz  streams v_j, w_j, diag:      corr = (W c - theta V c) / clamp(diag - theta),
//              |res|^2, |corr|^2, <v_j, corr>, <v_{k-1}, v_j>          (Ritz residual + CGS dots + Gram row)
//   kPassOrth1 streams corr, v_j:           cand = (corr - sum d_j v_j) / |corr|, <v_j, cand>
//   kPassOrth2 streams cand, v_j:           cand -= sum e_j v_j, |cand|^2
// ---------------------------------------------------------------------------
enum StreamPass { kPassProj = 0, kPassRitz = 1, kPassOrth1 = 2, kPassOrth2 = 3 };
constexpr int kStMaxS = 2 * kMaxVec + 1;
constexpr int kStMaxStages = 6;
constexpr size_t kStSmem = 210 * 1024;   // per SM

struct StreamArgs {
    // kPassRitz with tma2d: V[0..k) and W[0..k) as two 2-D tensor maps (rows
    // ld apart), one box of k rows x T columns each per tile
    CUtensorMap tm[2];
    int tma2d;
    uint64_t ld;             // row stride (elements) of the V / W blocks (tma2d)
    const double* s[kStMaxS];
    double c[kMaxVec];       // kPassRitz: Ritz coefficients
    int ns, k;
    uint32_t T;              // tile elements (multiple of 32)
    int nst;                 // pipeline stages (<= kStMaxStages)
    int split;               // kPassRitz: two threads per element (DETCI_DAV_RITZ_SPLIT=1)
    uint64_t n;
    double theta;
    const double* coef;      // kPassOrth1: d_j (unnormalised <v_j, corr>); kPassOrth2: e_j (device slots)
    const double* norm2;     // kPassOrth1: |corr|^2 (device slot)
    double* out;             // corr / cand
    double* partial;         // [reduction][gridDim.x]
};

__device__ __forceinline__ void tma_2d_g2s(void* dst, const CUtensorMap* map, int c0, int r0, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r0), "r"(smem_u32(bar))
        : "memory");
}

template <int MODE, int kStThreads>
__global__ void __launch_bounds__(kStThreads, 512 / kStThreads)
k_dav_stream(const __grid_constant__ StreamArgs a) {
    constexpr int kStWarps = kStThreads / 32;
    constexpr int kStJ = kMaxVec / kStWarps;   // subspace vectors per warp
    const int kStStages = a.nst;
    extern __shared__ __align__(128) double st_smem[];   // 2-D TMA boxes land 128-byte aligned
    __shared__ uint64_t bars[kStMaxStages];
    __shared__ double sh[32];
    __shared__ double s_coef[kMaxVec];
    const uint32_t T = a.T;
    const int ns = a.ns, k = a.k;
    double* const probe = st_smem + static_cast<size_t>(kStStages) * ns * T;
    const uint32_t tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
    const uint64_t ntiles = (a.n + T - 1) / T;
    const uint32_t my_tiles = blockIdx.x < ntiles
                                  ? static_cast<uint32_t>((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x)
                                  : 0u;
    auto tile_base = [&](uint32_t it) { return (static_cast<uint64_t>(it) * gridDim.x + blockIdx.x) * T; };
    auto tile_cnt = [&](uint32_t it) { const uint64_t rem = a.n - tile_base(it); return static_cast<uint32_t>(rem < T ? rem : T); };
    auto stage = [&](uint32_t st) { return st_smem + static_cast<size_t>(st) * ns * T; };
    auto issue = [&](uint32_t it) {   // warp 0: lane 0 arms the barrier, the lanes issue the copies
        const uint32_t st = it % kStStages, bytes = (tile_cnt(it) * 8u) & ~15u;
        if (MODE == kPassRitz && a.tma2d) {
            // two boxes (V, W: k rows x T, zero-filled past n, always full
            // box bytes) and the diagonal by a 1-D copy
            if (lane == 0) {
                mbar_arrive_expect_tx(&bars[st], 2u * static_cast<uint32_t>(k) * T * 8u + bytes);
                const int c0 = static_cast<int>(tile_base(it));
                tma_2d_g2s(stage(st), &a.tm[0], c0, 0, &bars[st]);
                tma_2d_g2s(stage(st) + static_cast<size_t>(k) * T, &a.tm[1], c0, 0, &bars[st]);
                if (bytes) bulk_g2s(stage(st) + static_cast<size_t>(2 * k) * T, a.s[2 * k] + tile_base(it), bytes, &bars[st]);
            }
            return;
        }
        if (lane == 0) mbar_arrive_expect_tx(&bars[st], bytes * static_cast<uint32_t>(ns));
        __syncwarp();
        if (bytes)
            for (int s = static_cast<int>(lane); s < ns; s += 32)
                bulk_g2s(stage(st) + static_cast<size_t>(s) * T, a.s[s] + tile_base(it), bytes, &bars[st]);
    };
    if (tid == 0) {
        for (int s = 0; s < kStStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (warp == 0)
        for (uint32_t it = 0; it < my_tiles && it < static_cast<uint32_t>(kStStages); ++it) issue(it);
    if (MODE == kPassOrth1 || MODE == kPassOrth2)
        for (int j = tid; j < k; j += kStThreads) s_coef[j] = a.coef[j];
    __syncthreads();

    // per-element scalars
    double inv_cnorm = 0.0;
    if (MODE == kPassOrth1) inv_cnorm = 1.0 / sqrt(*a.norm2);
    double out_scale = 1.0;   // kPassOrth2: 1 / nu, nu^2 = |cand1|^2 - sum e_j^2
    if (MODE == kPassOrth2) {
        double e2 = 0.0;
        for (int j = 0; j < k; ++j) e2 += s_coef[j] * s_coef[j];
        const double nu2 = *a.norm2 - e2;
        out_scale = nu2 > 0.0 ? 1.0 / sqrt(nu2) : 1.0;
    }
    double r1 = 0.0, r2 = 0.0;            // |res|^2, |corr|^2 / |cand|^2
    double acc[kStJ], acc2[kStJ];         // per-warp dots (vector j = warp + kStWarps * jj)
#pragma unroll
    for (int jj = 0; jj < kStJ; ++jj) acc[jj] = acc2[jj] = 0.0;

#pragma unroll 1
    for (uint32_t it = 0; it < my_tiles; ++it) {
        const uint32_t st = it % kStStages;
        const uint32_t cnt = tile_cnt(it);
        const uint64_t base = tile_base(it);
        double* const S = stage(st);
        mbar_wait(&bars[st], (it / kStStages) & 1u);
        if ((cnt & 1u) && static_cast<int>(tid) < ns) S[static_cast<size_t>(tid) * T + cnt - 1] = a.s[tid][base + cnt - 1];
        __syncthreads();
        // element-wise part (kPassRitz with a.split: two threads per
        // element, each summing half of the subspace, combined by a shuffle)
        const uint32_t esplit = MODE == kPassRitz && a.split ? 1u : 0u;
        const uint32_t ehalf = tid & esplit;
        const uint32_t cnt_up = esplit ? ((cnt + (kStThreads / 2) - 1) / (kStThreads / 2)) * (kStThreads / 2) : cnt;
        for (uint32_t i = tid >> esplit; i < cnt_up; i += kStThreads >> esplit) {
            if constexpr (MODE == kPassRitz) {
                const bool live = i < cnt;
                const uint32_t ii = live ? i : 0;
                double r = 0.0, m = 0.0;
#pragma unroll 4
                for (int j = static_cast<int>(ehalf); j < k; j += 1 + static_cast<int>(esplit)) {
                    r += a.c[j] * S[static_cast<size_t>(j) * T + ii];
                    m += a.c[j] * S[static_cast<size_t>(k + j) * T + ii];
                }
                if (esplit) {
                    r += __shfl_xor_sync(0xffffffffu, r, 1);
                    m += __shfl_xor_sync(0xffffffffu, m, 1);
                }
                if (!live || ehalf) continue;
                const double res = m - a.theta * r;
                double denom = S[static_cast<size_t>(2 * k) * T + i] - a.theta;
                if (fabs(denom) < 1e-8) denom = copysign(1e-8, denom);
                const double cr = res / denom;
                probe[i] = cr;
                a.out[base + i] = cr;
                r1 += res * res;
                r2 += cr * cr;
            } else if constexpr (MODE == kPassOrth1 || MODE == kPassOrth2) {
                double x = S[i];
#pragma unroll 4
                for (int j = 0; j < k; ++j) x -= s_coef[j] * S[static_cast<size_t>(1 + j) * T + i];
                if (MODE == kPassOrth1) x *= inv_cnorm;
                probe[i] = x;
                a.out[base + i] = MODE == kPassOrth2 ? x * out_scale : x;
                r2 += x * x;
            }
        }
        if constexpr (MODE != kPassOrth2) {
            if (MODE != kPassProj) __syncthreads();   // probe complete
            const double* pr = MODE == kPassProj ? S : probe;
            const int off = MODE == kPassRitz ? 0 : 1;   // first subspace stream
            const double* last = S + static_cast<size_t>(k - 1) * T;   // v_{k-1} (kPassRitz Gram row)
#pragma unroll
            for (int jj = 0; jj < kStJ; ++jj) {
                const int j = static_cast<int>(warp) + kStWarps * jj;
                if (j < k) {
                    const double* sj = S + static_cast<size_t>(off + j) * T;
                    double x = 0.0, g = 0.0;
                    for (uint32_t i = lane; i < cnt; i += 32) {
                        const double v = sj[i];
                        x = fma(v, pr[i], x);
                        if (MODE == kPassRitz) g = fma(v, last[i], g);
                    }
                    acc[jj] += x;
                    if (MODE == kPassRitz) acc2[jj] += g;
                }
            }
        }
        __syncthreads();   // stage and probe consumed
        if (warp == 0 && it + kStStages < my_tiles) {
            fence_proxy_async_smem();
            issue(it + kStStages);
        }
    }
    // partials: [0] |res|^2, [1] |corr|^2 (kPassRitz) or [0] |cand|^2 (kPassOrth2);
    // kPassOrth1 also [k] |cand1|^2
    // dots at [dbase + j] (and the Gram row at [dbase + k + j])
    const int dbase = MODE == kPassRitz ? 2 : 0;
    if constexpr (MODE == kPassRitz || MODE == kPassOrth2 || MODE == kPassOrth1) {
        const double s2 = block_sum(r2, sh);
        const int slot = MODE == kPassRitz ? 1 : (MODE == kPassOrth1 ? k : 0);
        if (tid == 0) a.partial[static_cast<size_t>(slot) * gridDim.x + blockIdx.x] = s2;
    }
    if constexpr (MODE == kPassRitz) {
        const double s1 = block_sum(r1, sh);
        if (tid == 0) a.partial[blockIdx.x] = s1;
    }
    if constexpr (MODE != kPassOrth2) {
#pragma unroll
        for (int jj = 0; jj < kStJ; ++jj) {
            const int j = static_cast<int>(warp) + kStWarps * jj;
            double x = acc[jj], g = acc2[jj];
            for (int s = 16; s > 0; s >>= 1) {
                x += __shfl_down_sync(0xffffffffu, x, s);
                g += __shfl_down_sync(0xffffffffu, g, s);
            }
            if (lane == 0 && j < k) {
                a.partial[static_cast<size_t>(dbase + j) * gridDim.x + blockIdx.x] = x;
                if (MODE == kPassRitz) a.partial[static_cast<size_t>(dbase + k + j) * gridDim.x + blockIdx.x] = g;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Register-dot variant of the fused passes (default for k <= 20).  Same
// streams, same TMA ring, but one thread owns one element of the tile and
// keeps every dot of the pass in registers (KMAX accumulators), so a tile
// costs one barrier and 2k + 1 (Ritz) / k + 1 shared-memory loads per
// element instead of the element phase + probe + warp-per-vector dot phase
// (5k + 1 / 3k + 1 loads, three barriers).  The bulk copies of a stage are
// issued by the 32 lanes of warp 0 (one elected thread issued ns copies
// serially before).  Dots are reduced once per CTA at the end: per warp by
// shuffles, then over warps in warp order into the per-CTA partials (fixed
// order, so the solve stays bitwise reproducible).
//   kPassOrth1 additionally reduces |cand|^2 into partial slot k, and
//   kPassOrth2 writes cand / nu with nu^2 = |cand1|^2 - sum e_j^2 (exact for
//   an orthonormal V; the host checks it against the directly reduced
//   |cand2|^2 and rescales in the rare case they disagree), which removes
//   the normalisation pass.
// ---------------------------------------------------------------------------
constexpr int kRsThreads = 512;

template <int MODE, int KMAX>
__global__ void __launch_bounds__(kRsThreads, 1)
k_dav_stream_r(const StreamArgs a) {
    constexpr int kWarps = kRsThreads / 32;
    constexpr int kVals = 2 + 2 * KMAX;
    const int kStStages = a.nst;
    extern __shared__ __align__(16) double st_smem[];
    __shared__ uint64_t bars[kStMaxStages];
    __shared__ double s_coef[KMAX];
    __shared__ double s_red[kWarps][kVals];
    const uint32_t T = a.T;
    const int ns = a.ns, k = a.k;
    const uint32_t tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
    const uint64_t ntiles = (a.n + T - 1) / T;
    const uint32_t my_tiles = blockIdx.x < ntiles
                                  ? static_cast<uint32_t>((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x)
                                  : 0u;
    auto tile_base = [&](uint32_t it) { return (static_cast<uint64_t>(it) * gridDim.x + blockIdx.x) * T; };
    auto tile_cnt = [&](uint32_t it) { const uint64_t rem = a.n - tile_base(it); return static_cast<uint32_t>(rem < T ? rem : T); };
    auto stage = [&](uint32_t st) { return st_smem + static_cast<size_t>(st) * ns * T; };
    auto issue = [&](uint32_t it) {   // warp 0
        const uint32_t st = it % kStStages, bytes = (tile_cnt(it) * 8u) & ~15u;
        if (lane == 0) mbar_arrive_expect_tx(&bars[st], bytes * static_cast<uint32_t>(ns));
        __syncwarp();
        if (bytes)
            for (int s = static_cast<int>(lane); s < ns; s += 32)
                bulk_g2s(stage(st) + static_cast<size_t>(s) * T, a.s[s] + tile_base(it), bytes, &bars[st]);
    };
    if (tid == 0) {
        for (int s = 0; s < kStStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (warp == 0)
        for (uint32_t it = 0; it < my_tiles && it < static_cast<uint32_t>(kStStages); ++it) issue(it);
    if (MODE == kPassOrth1 || MODE == kPassOrth2)
        for (int j = tid; j < k; j += kRsThreads) s_coef[j] = a.coef[j];
    __syncthreads();

    double scale = 1.0;
    if (MODE == kPassOrth1) scale = 1.0 / sqrt(*a.norm2);
    if (MODE == kPassOrth2) {
        // nu^2 = |cand1|^2 - sum_j e_j^2 (cand1 = this pass's input)
        double e2 = 0.0;
        for (int j = 0; j < k; ++j) e2 += s_coef[j] * s_coef[j];
        const double nu2 = *a.norm2 - e2;
        scale = nu2 > 0.0 ? 1.0 / sqrt(nu2) : 1.0;
    }
    double r1 = 0.0, r2 = 0.0;
    double acc[KMAX], acc2[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) acc[j] = acc2[j] = 0.0;

#pragma unroll 1
    for (uint32_t it = 0; it < my_tiles; ++it) {
        const uint32_t st = it % kStStages;
        const uint32_t cnt = tile_cnt(it);
        const uint64_t base = tile_base(it);
        const double* const S = stage(st);
        mbar_wait(&bars[st], (it / kStStages) & 1u);
        if (cnt & 1u) {   // the bulk copies moved 16-byte multiples
            if (static_cast<int>(tid) < ns)
                const_cast<double*>(S)[static_cast<size_t>(tid) * T + cnt - 1] = a.s[tid][base + cnt - 1];
            __syncthreads();
        }
        for (uint32_t i = tid; i < cnt; i += kRsThreads) {
            if constexpr (MODE == kPassRitz) {
                double r = 0.0, m = 0.0;
#pragma unroll
                for (int j = 0; j < KMAX; ++j)
                    if (j < k) {
                        r = fma(a.c[j], S[static_cast<size_t>(j) * T + i], r);
                        m = fma(a.c[j], S[static_cast<size_t>(k + j) * T + i], m);
                    }
                const double res = m - a.theta * r;
                double denom = S[static_cast<size_t>(2 * k) * T + i] - a.theta;
                if (fabs(denom) < 1e-8) denom = copysign(1e-8, denom);
                const double cr = res / denom;
                a.out[base + i] = cr;
                r1 = fma(res, res, r1);
                r2 = fma(cr, cr, r2);
                const double last = S[static_cast<size_t>(k - 1) * T + i];
#pragma unroll
                for (int j = 0; j < KMAX; ++j)
                    if (j < k) {
                        const double v = S[static_cast<size_t>(j) * T + i];
                        acc[j] = fma(v, cr, acc[j]);
                        acc2[j] = fma(v, last, acc2[j]);
                    }
            } else if constexpr (MODE == kPassProj) {
                const double x = S[i];
#pragma unroll
                for (int j = 0; j < KMAX; ++j)
                    if (j < k) acc[j] = fma(S[static_cast<size_t>(1 + j) * T + i], x, acc[j]);
            } else {
                double x = S[i];
#pragma unroll
                for (int j = 0; j < KMAX; ++j)
                    if (j < k) x = fma(-s_coef[j], S[static_cast<size_t>(1 + j) * T + i], x);
                r2 = fma(x, x, r2);   // Orth1: |corr - sum d v|^2 (scaled below); Orth2: |cand2|^2
                x *= scale;
                a.out[base + i] = x;
                if constexpr (MODE == kPassOrth1) {
#pragma unroll
                    for (int j = 0; j < KMAX; ++j)
                        if (j < k) acc[j] = fma(S[static_cast<size_t>(1 + j) * T + i], x, acc[j]);
                }
            }
        }
        __syncthreads();   // stage consumed
        if (warp == 0 && it + kStStages < my_tiles) {
            fence_proxy_async_smem();
            issue(it + kStStages);
        }
    }
    if (MODE == kPassOrth1) r2 *= scale * scale;

    // Per-CTA partials, layout as k_dav_stream: kPassRitz [0] |res|^2,
    // [1] |corr|^2, [2 + j] <v_j, corr>, [2 + k + j] <v_{k-1}, v_j>;
    // kPassProj [j]; kPassOrth1 [j] and [k] |cand1|^2; kPassOrth2 [0] |cand2|^2.
    auto wsum = [&](double v) {
        for (int s = 16; s > 0; s >>= 1) v += __shfl_down_sync(0xffffffffu, v, s);
        return v;
    };
    int nv = 0;
    auto put = [&](int slot, double v) {
        v = wsum(v);
        if (lane == 0) s_red[warp][slot] = v;
    };
    if constexpr (MODE == kPassRitz) {
        put(0, r1);
        put(1, r2);
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
            if (j < k) {
                put(2 + j, acc[j]);
                put(2 + k + j, acc2[j]);
            }
        nv = 2 + 2 * k;
    } else if constexpr (MODE == kPassProj) {
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
            if (j < k) put(j, acc[j]);
        nv = k;
    } else if constexpr (MODE == kPassOrth1) {
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
            if (j < k) put(j, acc[j]);
        put(k, r2);
        nv = k + 1;
    } else {
        put(0, r2);
        nv = 1;
    }
    __syncthreads();
    for (int v = tid; v < nv; v += kRsThreads) {
        double s = 0.0;
        for (int w = 0; w < kWarps; ++w) s += s_red[w][v];
        a.partial[static_cast<size_t>(v) * gridDim.x + blockIdx.x] = s;
    }
}

// ---------------------------------------------------------------------------
// Block (multi-root) residual pass: one stream over V[0..k), W[0..k) and the
// diagonal forms the preconditioned correction of all m <= 4 roots,
//   corr_r = (W c_r - theta_r V c_r) / clamp(diag - theta_r),
// and |res_r|^2, |corr_r|^2 -- 2k + 1 vector reads and m writes instead of
// m Ritz passes of 2k reads and 3 writes each (Ritz vectors and images are
// formed only when the subspace collapses onto them, or at the end).
// One element per thread (512 threads), the same TMA ring as the single-root
// passes; partials [r] |res_r|^2, [m + r] |corr_r|^2.
// ---------------------------------------------------------------------------
constexpr int kBlkMaxRoots = 4;
struct BlockRitzArgs {
    const double* s[kStMaxS];        // V[0..k), W[0..k), diag
    double c[kBlkMaxRoots][kMaxVec]; // Ritz coefficients per root
    double theta[kBlkMaxRoots];
    double* out[kBlkMaxRoots];       // corr_r
    int k, m, ns, nst;
    uint32_t T;
    uint64_t n;
    double* partial;
};

__global__ void __launch_bounds__(512, 1)
k_ritz_block(const BlockRitzArgs a) {
    constexpr int kThreads = 512, kWarps = kThreads / 32;
    extern __shared__ __align__(16) double st_smem[];
    __shared__ uint64_t bars[kStMaxStages];
    __shared__ double s_red[kWarps][2 * kBlkMaxRoots];
    const int nst = a.nst, ns = a.ns, k = a.k, m = a.m;
    const uint32_t T = a.T;
    const uint32_t tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
    const uint64_t ntiles = (a.n + T - 1) / T;
    const uint32_t my_tiles = blockIdx.x < ntiles
                                  ? static_cast<uint32_t>((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x)
                                  : 0u;
    auto tile_base = [&](uint32_t it) { return (static_cast<uint64_t>(it) * gridDim.x + blockIdx.x) * T; };
    auto tile_cnt = [&](uint32_t it) { const uint64_t rem = a.n - tile_base(it); return static_cast<uint32_t>(rem < T ? rem : T); };
    auto stage = [&](uint32_t st) { return st_smem + static_cast<size_t>(st) * ns * T; };
    auto issue = [&](uint32_t it) {   // warp 0
        const uint32_t st = it % nst, bytes = (tile_cnt(it) * 8u) & ~15u;
        if (lane == 0) mbar_arrive_expect_tx(&bars[st], bytes * static_cast<uint32_t>(ns));
        __syncwarp();
        if (bytes)
            for (int s = static_cast<int>(lane); s < ns; s += 32)
                bulk_g2s(stage(st) + static_cast<size_t>(s) * T, a.s[s] + tile_base(it), bytes, &bars[st]);
    };
    if (tid == 0) {
        for (int s = 0; s < nst; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (warp == 0)
        for (uint32_t it = 0; it < my_tiles && it < static_cast<uint32_t>(nst); ++it) issue(it);
    __syncthreads();

    double s1[kBlkMaxRoots], s2[kBlkMaxRoots];
#pragma unroll
    for (int r = 0; r < kBlkMaxRoots; ++r) s1[r] = s2[r] = 0.0;
#pragma unroll 1
    for (uint32_t it = 0; it < my_tiles; ++it) {
        const uint32_t st = it % nst;
        const uint32_t cnt = tile_cnt(it);
        const uint64_t base = tile_base(it);
        const double* const S = stage(st);
        mbar_wait(&bars[st], (it / nst) & 1u);
        if (cnt & 1u) {
            if (static_cast<int>(tid) < ns)
                const_cast<double*>(S)[static_cast<size_t>(tid) * T + cnt - 1] = a.s[tid][base + cnt - 1];
            __syncthreads();
        }
        for (uint32_t i = tid; i < cnt; i += kThreads) {
            double rv[kBlkMaxRoots], rw[kBlkMaxRoots];
#pragma unroll
            for (int r = 0; r < kBlkMaxRoots; ++r) rv[r] = rw[r] = 0.0;
#pragma unroll 2
            for (int j = 0; j < k; ++j) {
                const double v = S[static_cast<size_t>(j) * T + i];
                const double w = S[static_cast<size_t>(k + j) * T + i];
#pragma unroll
                for (int r = 0; r < kBlkMaxRoots; ++r)
                    if (r < m) {
                        rv[r] = fma(a.c[r][j], v, rv[r]);
                        rw[r] = fma(a.c[r][j], w, rw[r]);
                    }
            }
            const double dg = S[static_cast<size_t>(2 * k) * T + i];
#pragma unroll
            for (int r = 0; r < kBlkMaxRoots; ++r)
                if (r < m) {
                    const double res = rw[r] - a.theta[r] * rv[r];
                    double denom = dg - a.theta[r];
                    if (fabs(denom) < 1e-8) denom = copysign(1e-8, denom);
                    const double cr = res / denom;
                    a.out[r][base + i] = cr;
                    s1[r] = fma(res, res, s1[r]);
                    s2[r] = fma(cr, cr, s2[r]);
                }
        }
        __syncthreads();   // stage consumed
        if (warp == 0 && it + nst < my_tiles) {
            fence_proxy_async_smem();
            issue(it + nst);
        }
    }
#pragma unroll
    for (int r = 0; r < kBlkMaxRoots; ++r) {
        double x = s1[r], y = s2[r];
        for (int o = 16; o > 0; o >>= 1) {
            x += __shfl_down_sync(0xffffffffu, x, o);
            y += __shfl_down_sync(0xffffffffu, y, o);
        }
        if (lane == 0) {
            s_red[warp][r] = x;
            s_red[warp][kBlkMaxRoots + r] = y;
        }
    }
    __syncthreads();
    if (tid < 2 * static_cast<uint32_t>(m)) {
        const int r = static_cast<int>(tid) % m, which = static_cast<int>(tid) / m;
        double acc = 0.0;
        for (int w = 0; w < kWarps; ++w) acc += s_red[w][which * kBlkMaxRoots + r];
        a.partial[static_cast<size_t>(tid) * gridDim.x + blockIdx.x] = acc;
    }
}

__global__ void k_scale_div(double* __restrict__ x, uint64_t n, double divisor) {
    TILE_LOOP(i0, n) {
        double v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint64_t i = i0 + static_cast<uint64_t>(u) * blockDim.x;
            v[u] = i < n ? x[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint64_t i = i0 + static_cast<uint64_t>(u) * blockDim.x;
            if (i < n) x[i] = v[u] / divisor;
        }
    }
}

__global__ void k_set_unit(double* __restrict__ x, uint64_t n, uint64_t at) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        x[i] = i == at ? 1.0 : 0.0;
}

// Per-block (min value, lowest index) of diag, then a final pass.
__global__ void k_argmin(const double* __restrict__ d, uint64_t n, double* __restrict__ pv,
                         uint64_t* __restrict__ pi) {
    __shared__ double sv[kRedThreads];
    __shared__ uint64_t si[kRedThreads];
    double bv = INFINITY;
    uint64_t bi = ~0ull;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double v = d[i];
        if (v < bv || (v == bv && i < bi)) {
            bv = v;
            bi = i;
        }
    }
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            const double ov = sv[threadIdx.x + s];
            const uint64_t oi = si[threadIdx.x + s];
            if (ov < sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
                sv[threadIdx.x] = ov;
                si[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        pv[blockIdx.x] = sv[0];
        pi[blockIdx.x] = si[0];
    }
}

// Per-block smallest (value, index) pair lexicographically above (v0, i0):
// round r of the block solver's guesses finds the r-th lowest diagonal entry
// (lowest index on ties) without sorting the diagonal on the host.
__global__ void k_argmin_after(const double* __restrict__ d, uint64_t n, double v0, uint64_t i0, int first,
                               double* __restrict__ pv, uint64_t* __restrict__ pi) {
    __shared__ double sv[kRedThreads];
    __shared__ uint64_t si[kRedThreads];
    double bv = INFINITY;
    uint64_t bi = ~0ull;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double v = d[i];
        const bool above = first || v > v0 || (v == v0 && i > i0);
        if (above && (v < bv || (v == bv && i < bi))) {
            bv = v;
            bi = i;
        }
    }
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            const double ov = sv[threadIdx.x + s];
            const uint64_t oi = si[threadIdx.x + s];
            if (ov < sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
                sv[threadIdx.x] = ov;
                si[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        pv[blockIdx.x] = sv[0];
        pi[blockIdx.x] = si[0];
    }
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void ensure_red(Handle& h) {
    if (h.red.n < static_cast<size_t>(2 * kMaxVec * kRedBlocks + 8 * kMaxVec))
        h.red.alloc(static_cast<size_t>(2 * kMaxVec * kRedBlocks + 8 * kMaxVec));
}

// Device scalar slot (after the partials region) for MGS overlaps.
double* scalar_slot(Handle& h, int i) { return h.red.p + 2 * kMaxVec * kRedBlocks + i; }

void allreduce_device(Handle& h, double* dptr, int count) {
    if (h.world <= 1) return;
    h.comm->allreduce_sum(dptr, static_cast<size_t>(count), h.stream);
}

// Finalize `k` partial rows into device slots [slot, slot + k), allreduced.
void finalize_to(Handle& h, int k, int slot) {
    k_finalize<<<k, 32, 0, h.stream>>>(h.red.p, kRedBlocks, k, scalar_slot(h, slot));
    CUDA_LAUNCH_CHECK();
    allreduce_device(h, scalar_slot(h, slot), k);
}

void read_slots(Handle& h, int slot, int k, double* out) {
    CUDA_CHECK(cudaMemcpyAsync(out, scalar_slot(h, slot), k * sizeof(double), cudaMemcpyDeviceToHost,
                               h.stream));
    CUDA_CHECK(cudaStreamSynchronize(h.stream));
}

// DETCI_DAVIDSON_ORTHO=mgs: the reference's sequential 2-pass MGS (2k
// dependent projection kernels).  Default: classical Gram-Schmidt twice,
// measured at C2 0.119 vs 0.124 s per iteration (sigma 0.105 s).
bool ortho_mgs() {
    const char* e = std::getenv("DETCI_DAVIDSON_ORTHO");
    return e && std::string(e) == "mgs";
}

// One classical Gram-Schmidt pass: d = <v_j, src> (device slots 64..), then
// dst = (src - sum_j d_j v_j) * scale; with `norm`, |dst|^2 lands in slot 4.
template <class VF>
void cgs_pass(Handle& h, double* dst, const double* src, double scale, VF&& V, int k, uint64_t n, bool norm) {
    VecList vl{};
    for (int j = 0; j < k; ++j) vl.p[j] = V(j);
    k_dot_many<<<kRedBlocks, kRedThreads, 0, h.stream>>>(src, vl, k, n, h.red.p);
    CUDA_LAUNCH_CHECK();
    finalize_to(h, k, kMaxVec);
    k_combine<<<kRedBlocks, kRedThreads, 0, h.stream>>>(dst, src, scale, vl, scalar_slot(h, kMaxVec), k, n,
                                                        norm ? h.red.p : nullptr);
    CUDA_LAUNCH_CHECK();
    if (norm) finalize_to(h, 1, 4);
}

// Device slots of the fused passes (after the CGS region at kMaxVec..2kMaxVec)
constexpr int kSlotRitz = 2 * kMaxVec;            // |res|^2, |corr|^2, d_j (k), Gram row (k)
constexpr int kSlotOrth1 = kSlotRitz + 2 * kMaxVec + 4;   // e_j (k)
constexpr int kSlotOrth2 = kSlotOrth1 + kMaxVec + 4;      // |cand|^2

int sm_count() {
    int dev = 0, v = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    return v;
}

// One fused pass (k_dav_stream<MODE>) over the ns streams, its nred
// reductions finalized (fixed order) and allreduced into device slots
// [slot, slot + nred).  Stream bases must be 16-byte aligned.
// Pipeline shape of the fused passes: threads per CTA, CTAs per SM, stages
// (DETCI_DAV_CFG="threads,ctas,stages" overrides the default 512,1,3).
// Two stages (C2, 60 iterations, one box: subspace solve + vector work 8.8 ms
// per iteration at 512 x 1 x 2, 10.7 ms at 512 x 1 x 3, 9.0 ms at 256 x 2 x 2,
// 11.6 ms at 256 x 2 x 3): larger tiles, fewer barriers per byte.
struct StreamCfg {
    int threads = 512, ctas = 1, stages = 2;
};
StreamCfg stream_cfg() {
    StreamCfg c;
    if (const char* e = std::getenv("DETCI_DAV_CFG")) {
        int t = 0, k = 0, s = 0;
        if (std::sscanf(e, "%d,%d,%d", &t, &k, &s) == 3 && (t == 256 || t == 512) && k >= 1 && k <= 4 && s >= 2 &&
            s <= kStMaxStages) {
            c.threads = t;
            c.ctas = k;
            c.stages = s;
        }
    }
    return c;
}

// Default for k <= 20: the register-dot kernel (k_dav_stream_r, 512 threads).
// Measured on C2, 12 iterations (ncu launch lists, 2 stages): the four passes
// 56.6 ms vs 61.1 ms with the warp-per-vector dot phase (Ritz pass 24.7 vs
// 29.1 ms); at 256 threads it was slower (86.9 vs 65.5 ms at 3 stages): one
// element per thread needs the full 16 warps to hide its FMA chains.
// DETCI_DAV_STREAM=warp: the warp-per-vector kernel for every k;
// DETCI_DAV_STREAM=reg_ritz: the register kernel for the Ritz pass only.
constexpr int kRsMaxK = 20;
bool register_stream(int k, int mode = -1) {
    static const int sel = [] {
        const char* e = std::getenv("DETCI_DAV_STREAM");
        if (e && std::string(e) == "warp") return 0;
        if (e && std::string(e) == "reg_ritz") return 2;
        return 1;
    }();
    return k <= kRsMaxK && (sel == 1 || (sel == 2 && mode == kPassRitz));
}

// 2-D tensor map over `rows` vectors of n doubles, ld apart, box T x rows
// (cuTensorMapEncodeTiled through the runtime's driver entry point).
bool encode_rows_map(CUtensorMap* m, const double* base, uint64_t n, uint32_t rows, uint64_t ld, uint32_t T) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    if (!fn || rows == 0 || rows > 256 || T == 0 || T > 256 || (ld * 8) % 16 != 0) return false;
    const cuuint64_t dims[2] = {n, rows};
    const cuuint64_t strides[1] = {ld * 8};
    const cuuint32_t box[2] = {T, rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// DETCI_DAV_TMA2D=1: the Ritz pass stages V and W as two 2-D tensor boxes
// per tile instead of one 1-D copy per vector.  Measured level or slower
// (C2, 60 iterations: vector work 7.73-7.87 vs 7.61 ms per iteration; the
// box width caps T at 256), so the per-copy cost is not what holds the Ritz
// pass below the others; off by default.
bool tma2d_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DETCI_DAV_TMA2D");
        return e && std::string(e) == "1";
    }();
    return on;
}

template <int MODE>
void stream_pass(Handle& h, StreamArgs& a, int nred, int slot) {
    for (int s = 0; s < a.ns; ++s)
        if (reinterpret_cast<uintptr_t>(a.s[s]) & 15u) fail(DETCI_GPU_E_ERROR, "davidson: misaligned vector");
    static const StreamCfg cfg = stream_cfg();
    a.nst = cfg.stages;
    if (MODE == kPassRitz && a.tma2d) {
        // V rows and W rows must each be one strided block
        bool ok = tma2d_enabled() && a.k >= 1;
        for (int j = 0; ok && j < a.k; ++j)
            ok = a.s[j] == a.s[0] + j * a.ld && a.s[a.k + j] == a.s[a.k] + j * a.ld;
        const size_t per = static_cast<size_t>(a.nst) * a.ns + 1;
        const uint32_t T = static_cast<uint32_t>(std::min<size_t>(256, kStSmem / cfg.ctas / 8 / per) & ~size_t{31});
        ok = ok && T >= 32 && cfg.threads == 512 &&
             encode_rows_map(&a.tm[0], a.s[0], a.n, static_cast<uint32_t>(a.k), a.ld, T) &&
             encode_rows_map(&a.tm[1], a.s[a.k], a.n, static_cast<uint32_t>(a.k), a.ld, T);
        a.tma2d = ok ? 1 : 0;
        if (ok) {
            a.T = T;
            const size_t smem = per * a.T * sizeof(double);
            const int grid = sm_count() * cfg.ctas;
            a.partial = h.red.p;
            ensure_dynamic_smem(reinterpret_cast<const void*>(&k_dav_stream<MODE, 512>), smem);
            k_dav_stream<MODE, 512><<<grid, 512, smem, h.stream>>>(a);
            CUDA_LAUNCH_CHECK();
            if (nred > 0) {
                k_finalize<<<nred, 32, 0, h.stream>>>(h.red.p, grid, nred, scalar_slot(h, slot));
                CUDA_LAUNCH_CHECK();
                allreduce_device(h, scalar_slot(h, slot), nred);
            }
            return;
        }
    }
    static const bool split = [] {
        const char* e = std::getenv("DETCI_DAV_RITZ_SPLIT");
        return e && std::string(e) == "1";
    }();
    a.split = split ? 1 : 0;
    if (register_stream(a.k, MODE)) {
        a.T = static_cast<uint32_t>(std::min<size_t>(4096, kStSmem / 8 / (static_cast<size_t>(a.nst) * a.ns)) &
                                    ~size_t{31});
        if (a.T < 32) fail(DETCI_GPU_E_ERROR, "davidson: stream tile below 32 elements");
        const size_t smem = static_cast<size_t>(a.nst) * a.ns * a.T * sizeof(double);
        const int grid = sm_count();
        a.partial = h.red.p;
        auto go = [&](auto kern) {
            ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
            kern<<<grid, kRsThreads, smem, h.stream>>>(a);
        };
        if (a.k <= 8) go(&k_dav_stream_r<MODE, 8>);
        else if (a.k <= 12) go(&k_dav_stream_r<MODE, 12>);
        else if (a.k <= 16) go(&k_dav_stream_r<MODE, 16>);
        else go(&k_dav_stream_r<MODE, kRsMaxK>);
        CUDA_LAUNCH_CHECK();
        if (nred > 0) {
            k_finalize<<<nred, 32, 0, h.stream>>>(h.red.p, grid, nred, scalar_slot(h, slot));
            CUDA_LAUNCH_CHECK();
            allreduce_device(h, scalar_slot(h, slot), nred);
        }
        return;
    }
    const size_t per = static_cast<size_t>(a.nst) * a.ns + 1;   // doubles per tile element (stages + probe)
    a.T = static_cast<uint32_t>(std::min<size_t>(4096, kStSmem / cfg.ctas / 8 / per) & ~size_t{31});
    if (a.T < 32) fail(DETCI_GPU_E_ERROR, "davidson: stream tile below 32 elements");
    const size_t smem = per * a.T * sizeof(double);
    const int grid = sm_count() * cfg.ctas;
    a.partial = h.red.p;
    if (cfg.threads == 512) {
        ensure_dynamic_smem(reinterpret_cast<const void*>(&k_dav_stream<MODE, 512>), smem);
        k_dav_stream<MODE, 512><<<grid, 512, smem, h.stream>>>(a);
    } else {
        ensure_dynamic_smem(reinterpret_cast<const void*>(&k_dav_stream<MODE, 256>), smem);
        k_dav_stream<MODE, 256><<<grid, 256, smem, h.stream>>>(a);
    }
    CUDA_LAUNCH_CHECK();
    if (nred > 0) {
        k_finalize<<<nred, 32, 0, h.stream>>>(h.red.p, grid, nred, scalar_slot(h, slot));
        CUDA_LAUNCH_CHECK();
        allreduce_device(h, scalar_slot(h, slot), nred);
    }
}

// DETCI_DAVIDSON_FUSED=0: the previous per-operation kernels (k_dot_many,
// k_ritz, two CGS passes), kept for comparison.
// DETCI_DAVIDSON_BLOCK_RITZ=0: one k_ritz pass per root in the block solver.
bool fused_block_ritz(int m, int k, uint64_t n) {
    const char* e = std::getenv("DETCI_DAVIDSON_BLOCK_RITZ");   // read per call (tests switch it)
    const bool off = e && std::string(e) == "0";
    const size_t ns = 2 * static_cast<size_t>(k) + 1;
    // the block solver's vectors sit n doubles apart: 16-byte bulk copies need n even
    return !off && m <= kBlkMaxRoots && ns <= static_cast<size_t>(kStMaxS) && n > 0 && n % 2 == 0 &&
           kStSmem / 8 / (2 * ns) >= 32;
}

bool fused_passes() {
    const char* e = std::getenv("DETCI_DAVIDSON_FUSED");
    return !(e && std::string(e) == "0");
}

} // namespace

void allreduce_sum(Handle& h, double* host_vals, int count) {
    if (h.world <= 1 || count <= 0) return;
    if (h.red_host.n < static_cast<size_t>(count)) h.red_host.alloc(static_cast<size_t>(count));
    double* d = h.red_host.p;
    CUDA_CHECK(cudaMemcpyAsync(d, host_vals, count * sizeof(double), cudaMemcpyHostToDevice, h.stream));
    allreduce_device(h, d, count);
    CUDA_CHECK(cudaMemcpyAsync(host_vals, d, count * sizeof(double), cudaMemcpyDeviceToHost, h.stream));
    CUDA_CHECK(cudaStreamSynchronize(h.stream));
}

bool all_ranks_ok(Handle& h, bool ok) {
    if (h.world <= 1) return ok;
    double bad = ok ? 0.0 : 1.0;
    allreduce_sum(h, &bad, 1);
    return bad == 0.0;
}

void collective_require(Handle& h, bool ok, int code, const std::string& msg, const char* what) {
    if (all_ranks_ok(h, ok)) return;
    if (!ok) fail(code, msg);
    fail(DETCI_GPU_E_ERROR, std::string(what) + ": another rank failed");
}

void device_dot_many(Handle& h, const double* x, const double* const* ys, int k, uint64_t n,
                     double* out_host) {
    if (k > 2 * kMaxVec) fail(DETCI_GPU_E_CONFIG, "dot_many: too many vectors");
    ensure_red(h);
    VecList vl{};
    for (int j = 0; j < k; ++j) vl.p[j] = ys[j];
    k_dot_many<<<kRedBlocks, kRedThreads, 0, h.stream>>>(x, vl, k, n, h.red.p);
    CUDA_LAUNCH_CHECK();
    for (int j0 = 0; j0 < k; j0 += kMaxVec) {
        const int kk = std::min(kMaxVec, k - j0);
        k_finalize<<<kk, 32, 0, h.stream>>>(h.red.p + static_cast<size_t>(j0) * kRedBlocks, kRedBlocks,
                                             kk, scalar_slot(h, 0));
        CUDA_LAUNCH_CHECK();
        allreduce_device(h, scalar_slot(h, 0), kk);
        read_slots(h, 0, kk, out_host + j0);
    }
}

double device_dot(Handle& h, const double* x, const double* y, uint64_t n) {
    double v = 0.0;
    device_dot_many(h, x, &y, 1, n, &v);
    return v;
}

// All eigenpairs of the k x k symmetric matrix given by its lower triangle
// lower[i * ld + j], j <= i (Eigen's SelfAdjointEigenSolver reads only that
// triangle, davidson.cpp:22-30).  Cyclic Jacobi to machine precision;
// eigenvalues ascending, vecs[m * k + i] = component i of eigenvector m.
void jacobi_eigen(const std::vector<double>& lower, int ld, int k, std::vector<double>& evals,
                  std::vector<double>& vecs) {
    std::vector<double> a(static_cast<size_t>(k) * k), v(static_cast<size_t>(k) * k, 0.0);
    for (int i = 0; i < k; ++i) {
        for (int j = 0; j < k; ++j) a[i * k + j] = i >= j ? lower[i * ld + j] : lower[j * ld + i];
        v[i * k + i] = 1.0;
    }
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, tot = 0.0;
        for (int i = 0; i < k; ++i)
            for (int j = 0; j < k; ++j) {
                tot += a[i * k + j] * a[i * k + j];
                if (i != j) off += a[i * k + j] * a[i * k + j];
            }
        if (off == 0.0 || off <= 1e-30 * tot) break;
        for (int p = 0; p < k; ++p)
            for (int q = p + 1; q < k; ++q) {
                const double apq = a[p * k + q];
                if (apq == 0.0) continue;
                const double tau = (a[q * k + q] - a[p * k + p]) / (2.0 * apq);
                const double t = (tau >= 0 ? 1.0 : -1.0) / (std::fabs(tau) + std::sqrt(1.0 + tau * tau));
                const double c = 1.0 / std::sqrt(1.0 + t * t), s = t * c;
                for (int r = 0; r < k; ++r) {
                    const double arp = a[r * k + p], arq = a[r * k + q];
                    a[r * k + p] = c * arp - s * arq;
                    a[r * k + q] = s * arp + c * arq;
                }
                for (int r = 0; r < k; ++r) {
                    const double apr = a[p * k + r], aqr = a[q * k + r];
                    a[p * k + r] = c * apr - s * aqr;
                    a[q * k + r] = s * apr + c * aqr;
                }
                for (int r = 0; r < k; ++r) {
                    const double vrp = v[r * k + p], vrq = v[r * k + q];
                    v[r * k + p] = c * vrp - s * vrq;
                    v[r * k + q] = s * vrp + c * vrq;
                }
            }
    }
    std::vector<int> order(k);
    for (int i = 0; i < k; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return a[x * k + x] < a[y * k + y]; });
    evals.resize(k);
    vecs.assign(static_cast<size_t>(k) * k, 0.0);
    for (int m = 0; m < k; ++m) {
        evals[m] = a[order[m] * k + order[m]];
        for (int i = 0; i < k; ++i) vecs[static_cast<size_t>(m) * k + i] = v[i * k + order[m]];
    }
}

double smallest_eigenpair(const std::vector<double>& lower, int ld, int k, std::vector<double>& vec) {
    std::vector<double> evals, vecs;
    jacobi_eigen(lower, ld, k, evals, vecs);
    vec.assign(vecs.begin(), vecs.begin() + k);
    return evals[0];
}

void davidson_device(Handle& h, const detci_dav_opts& opts, detci_dav_result* res,
                     detci_trace_cb cb, void* user) {
    if (!h.built) fail(DETCI_GPU_E_INPUT, "davidson_solve: basis not built");
    const uint64_t n = h.local_len();
    if (!(opts.tol > 0.0)) fail(DETCI_GPU_E_CONFIG, "davidson_solve: tol must be positive");
    if (opts.max_subspace < 2) fail(DETCI_GPU_E_CONFIG, "davidson_solve: max_subspace must be >= 2");
    if (opts.max_iter < 1) fail(DETCI_GPU_E_CONFIG, "davidson_solve: max_iter must be positive");
    if (opts.max_subspace > kMaxVec)
        fail(DETCI_GPU_E_UNSUPPORTED, "davidson_solve: max_subspace above 64");
    ensure_red(h);
    const int ms = opts.max_subspace;
    const auto wall0 = std::chrono::steady_clock::now();

    size_t free_b = 0, total_b = 0;
    CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
    // the scatter D buffer is scratch: count it as free, and drop it (it is
    // re-planned around the subspace at the next sigma) only when the
    // subspace does not fit next to it
    // the subspace buffer is cached in the handle across solves (freeing
    // hundreds of MB per solve costs 0.1-0.4 s); a cached buffer counts as free
    // vector stride rounded to 16 bytes (the fused passes stream each
    // vector with 1-D TMA bulk copies)
    const uint64_t ld = (n + 1) & ~uint64_t{1};
    const size_t need = (2 * static_cast<size_t>(ms) + 3) * ld * sizeof(double);
    const bool grow = h.dav_store.bytes() < need;
    const bool drop_d = grow && need + (1ull << 30) > free_b + h.dav_store.bytes();
    free_b += h.dbuf.bytes() + h.dav_store.bytes();
    const uint64_t budget = h.budget ? h.budget : free_b;
    // per-rank conditions, decided collectively
    if (n == 0) collective_require(h, false, DETCI_GPU_E_INPUT, "davidson_solve: empty diagonal", "davidson_solve");
    else
        collective_require(h, need <= std::min<uint64_t>(budget, free_b), DETCI_GPU_E_CAPACITY,
                           "davidson vectors require " + std::to_string(need) + " bytes, budget is " +
                               std::to_string(std::min<uint64_t>(budget, free_b)) + " bytes",
                           "davidson_solve");
    DevBuf<double>& store = h.dav_store;
    if (drop_d) release_sigma_scratch(h);
    if (grow) {
        store.reset();
        store.alloc((2 * static_cast<size_t>(ms) + 3) * ld);
    }
    auto V = [&](int j) { return store.p + static_cast<size_t>(j) * ld; };
    auto Wv = [&](int j) { return store.p + static_cast<size_t>(ms + j) * ld; };
    double* ritz = store.p + static_cast<size_t>(2 * ms) * ld;
    double* img = ritz + ld;
    double* corr = img + ld;
    const bool fused = fused_passes();
    const unsigned vgrid = kRedBlocks;

    // Initial vector (davidson.cpp:84-97).
    if (opts.initial_guess) {
        CUDA_CHECK(cudaMemcpyAsync(V(0), opts.initial_guess, n * sizeof(double), cudaMemcpyHostToDevice,
                                   h.stream));
        const double nrm2 = device_dot(h, V(0), V(0), n);
        const double norm = std::sqrt(nrm2);
        if (!(norm > 0.0)) fail(DETCI_GPU_E_INPUT, "davidson_solve: zero initial guess");
        k_scale_div<<<vgrid, kRedThreads, 0, h.stream>>>(V(0), n, norm);
        CUDA_LAUNCH_CHECK();
    } else {
        DevBuf<double> pv;
        DevBuf<uint64_t> pi;
        pv.alloc(kRedBlocks);
        pi.alloc(kRedBlocks);
        k_argmin<<<kRedBlocks, kRedThreads, 0, h.stream>>>(h.diag.p, n, pv.p, pi.p);
        CUDA_LAUNCH_CHECK();
        std::vector<double> hv(kRedBlocks);
        std::vector<uint64_t> hi(kRedBlocks);
        CUDA_CHECK(cudaMemcpyAsync(hv.data(), pv.p, kRedBlocks * sizeof(double), cudaMemcpyDeviceToHost, h.stream));
        CUDA_CHECK(cudaMemcpyAsync(hi.data(), pi.p, kRedBlocks * sizeof(uint64_t), cudaMemcpyDeviceToHost, h.stream));
        CUDA_CHECK(cudaStreamSynchronize(h.stream));
        double bv = INFINITY;
        uint64_t bi = ~0ull;
        for (int b = 0; b < kRedBlocks; ++b)
            if (hv[b] < bv || (hv[b] == bv && hi[b] < bi)) {
                bv = hv[b];
                bi = hi[b];
            }
        // Global argmin across ranks: lowest value, then lowest global index.
        uint64_t owner_index = bi + h.a0 * h.nb();
        if (h.world > 1) {
            std::vector<double> all(2 * h.world, 0.0);
            all[2 * h.rank] = bv;
            all[2 * h.rank + 1] = static_cast<double>(owner_index);
            allreduce_sum(h, all.data(), 2 * h.world);
            double gv = INFINITY;
            double gi = 0;
            for (int r = 0; r < h.world; ++r)
                if (all[2 * r] < gv || (all[2 * r] == gv && all[2 * r + 1] < gi)) {
                    gv = all[2 * r];
                    gi = all[2 * r + 1];
                }
            owner_index = static_cast<uint64_t>(gi);
        }
        const uint64_t lo = h.a0 * h.nb(), local_at = owner_index >= lo && owner_index < lo + n
                                                          ? owner_index - lo
                                                          : ~0ull;
        k_set_unit<<<vgrid, kRedThreads, 0, h.stream>>>(V(0), n, local_at);
        CUDA_LAUNCH_CHECK();
    }

    std::vector<double> proj(static_cast<size_t>(ms) * ms, 0.0);
    std::vector<double> gram(static_cast<size_t>(ms) * ms, 0.0);
    std::vector<double> coeffs;
    int k_sub = 1, k_img = 0;
    bool restart_pending = false;
    double theta = 0.0;
    int status = 0, iters = 0;
    bool ritz_fresh = false;
    std::vector<detci_dav_iter> trace;

    for (int iter = 0; iter < opts.max_iter; ++iter) {
        detci_dav_iter st{};
        st.restarted = restart_pending ? 1 : 0;
        restart_pending = false;

        auto t0 = std::chrono::steady_clock::now();
        while (k_img < k_sub) {
            sigma_device(h, V(k_img), Wv(k_img), nullptr);
            ++k_img;
        }
        st.matvec_seconds = seconds_since(t0);

        const int k = k_sub;
        t0 = std::chrono::steady_clock::now();
        if (fused) {
            // projected row k-1: <V[k-1], W_j> in one pass (the Gram row
            // comes out of the Ritz pass below)
            StreamArgs pa{};
            pa.ns = k + 1;
            pa.k = k;
            pa.n = n;
            pa.s[0] = V(k - 1);
            for (int j = 0; j < k; ++j) pa.s[1 + j] = Wv(j);
            stream_pass<kPassProj>(h, pa, k, 0);
            std::vector<double> dots(k);
            read_slots(h, 0, k, dots.data());
            for (int j = 0; j < k; ++j) proj[(k - 1) * ms + j] = dots[j];
        } else {
            // projected row k-1 and Gram row k-1 in one pass over V[k-1]
            std::vector<const double*> ys(2 * k);
            for (int j = 0; j < k; ++j) {
                ys[j] = Wv(j);
                ys[k + j] = V(j);
            }
            std::vector<double> dots(2 * k);
            device_dot_many(h, V(k - 1), ys.data(), 2 * k, n, dots.data());
            for (int j = 0; j < k; ++j) {
                proj[(k - 1) * ms + j] = dots[j];
                gram[(k - 1) * ms + j] = dots[k + j];
            }
        }
        theta = smallest_eigenpair(proj, ms, k, coeffs);
        st.subspace_solve_seconds = seconds_since(t0);

        t0 = std::chrono::steady_clock::now();
        // the Ritz vector and its image are materialised only when the
        // subspace collapses onto them (or, after the loop, for the
        // returned eigenvector)
        const bool collapse = k_sub >= ms;
        double rnorm = 0.0, cnorm = 0.0;
        ritz_fresh = false;
        if (fused) {
            // residual, preconditioned correction, <v_j, corr> and the Gram
            // row in one pass over V, W and the diagonal
            StreamArgs ra{};
            ra.ns = 2 * k + 1;
            ra.k = k;
            ra.n = n;
            for (int j = 0; j < k; ++j) {
                ra.s[j] = V(j);
                ra.s[k + j] = Wv(j);
                ra.c[j] = coeffs[j];
            }
            ra.s[2 * k] = h.diag.p;
            ra.theta = theta;
            ra.out = corr;
            ra.tma2d = 1;
            ra.ld = ld;
            stream_pass<kPassRitz>(h, ra, 2 * k + 2, kSlotRitz);
            std::vector<double> sc(2 * k + 2);
            read_slots(h, kSlotRitz, 2 * k + 2, sc.data());
            rnorm = std::sqrt(sc[0]);
            cnorm = std::sqrt(sc[1]);
            for (int j = 0; j < k; ++j) gram[(k - 1) * ms + j] = sc[2 + k + j];
        }

        if (!fused || collapse) {
            RitzArgs ra{};
            for (int j = 0; j < k; ++j) {
                ra.v[j] = V(j);
                ra.w[j] = Wv(j);
                ra.c[j] = coeffs[j];
            }
            ra.k = k;
            ra.theta = theta;
            k_ritz<<<kRedBlocks, kRedThreads, 0, h.stream>>>(ra, h.diag.p, n, ritz, img, corr, h.red.p);
            CUDA_LAUNCH_CHECK();
            ritz_fresh = true;
            finalize_to(h, 2, 0);
            double norms2[2];
            read_slots(h, 0, 2, norms2);
            rnorm = std::sqrt(norms2[0]);
            cnorm = std::sqrt(norms2[1]);
        }
        double gdev = 0.0;
        for (int i = 0; i < k; ++i)
            for (int j = 0; j <= i; ++j)
                gdev = std::max(gdev, std::fabs(gram[i * ms + j] - (i == j ? 1.0 : 0.0)));
        st.max_gram_deviation = gdev;
        st.ritz_value = theta;
        st.residual_norm = rnorm;

        const bool converged = rnorm <= opts.tol;
        const bool last = iter + 1 == opts.max_iter;
        auto push = [&]() {
            st.orthogonalization_seconds = seconds_since(t0);
            trace.push_back(st);
            if (cb) cb(&trace.back(), iters, user);
            ++iters;
        };
        if (converged || last) {
            push();
            status = converged ? 0 : 1;
            break;
        }
        if (!(cnorm > 0.0)) {
            push();
            status = 2;
            break;
        }
        if (collapse) {  // collapse (davidson.cpp:178-184)
            CUDA_CHECK(cudaMemcpyAsync(V(0), ritz, n * sizeof(double), cudaMemcpyDeviceToDevice, h.stream));
            CUDA_CHECK(cudaMemcpyAsync(Wv(0), img, n * sizeof(double), cudaMemcpyDeviceToDevice, h.stream));
            k_sub = k_img = 1;
            const double* y2[2] = {Wv(0), V(0)};
            double d2[2];
            device_dot_many(h, V(0), y2, 2, n, d2);
            proj[0] = d2[0];
            gram[0] = d2[1];
            restart_pending = true;
        }
        // corr / |corr| orthogonalized twice against V[0..k_sub) into
        // V[k_sub] (orthonormalize, davidson.cpp:43-57)
        double* cand = V(k_sub);
        double nrm2 = 0.0;
        bool prenormalised = false;
        if (ortho_mgs()) {
            // the reference's 2-pass modified Gram-Schmidt, one projection per kernel
            const int steps = 2 * k_sub;
            for (int t = 0; t <= steps; ++t) {
                const double* src = t == 0 ? corr : nullptr;
                const double* vprev = t == 0 ? nullptr : V((t - 1) % k_sub);
                const double* vnext = t == steps ? nullptr : V(t % k_sub);
                k_mgs_step<<<kRedBlocks, kRedThreads, 0, h.stream>>>(cand, src, cnorm, vprev,
                                                                      scalar_slot(h, 4 + (t + 1) % 2),
                                                                      vnext, n, h.red.p);
                CUDA_LAUNCH_CHECK();
                finalize_to(h, 1, 4 + t % 2);
            }
            read_slots(h, 4 + steps % 2, 1, &nrm2);
        } else if (fused && !collapse) {
            // classical Gram-Schmidt twice from the Ritz pass's dots: pass 1
            // also forms the second pass's dots, pass 2 the norm
            StreamArgs oa{};
            oa.ns = k + 1;
            oa.k = k;
            oa.n = n;
            for (int j = 0; j < k; ++j) oa.s[1 + j] = V(j);
            oa.s[0] = corr;
            oa.coef = scalar_slot(h, kSlotRitz + 2);
            oa.norm2 = scalar_slot(h, kSlotRitz + 1);
            oa.out = cand;
            // pass 1 also reduces |cand1|^2 (slot k); pass 2 writes the
            // candidate normalised by nu = sqrt(|cand1|^2 - sum e_j^2)
            stream_pass<kPassOrth1>(h, oa, k + 1, kSlotOrth1);
            oa.s[0] = cand;
            oa.coef = scalar_slot(h, kSlotOrth1);
            oa.norm2 = scalar_slot(h, kSlotOrth1 + k);
            stream_pass<kPassOrth2>(h, oa, 1, kSlotOrth2);
            {
                std::vector<double> sl(k + 1);
                read_slots(h, kSlotOrth1, k + 1, sl.data());
                read_slots(h, kSlotOrth2, 1, &nrm2);
                double nu2 = sl[k];
                for (int j = 0; j < k; ++j) nu2 -= sl[j] * sl[j];
                const double nu_a = nu2 > 0.0 ? std::sqrt(nu2) : 1.0;
                const double nu_d = std::sqrt(nrm2);
                // cand holds cand2 / nu_a; the reference divides by the
                // directly computed norm (davidson.cpp:54-56)
                if (nu_d >= 1e-10 && std::fabs(nu_a / nu_d - 1.0) > 1e-12) {
                    k_scale_div<<<vgrid, kRedThreads, 0, h.stream>>>(cand, n, nu_d / nu_a);
                    CUDA_LAUNCH_CHECK();
                }
                prenormalised = true;
            }
        } else {
            // classical Gram-Schmidt twice ("twice is enough"): each pass is
            // one multi-dot and one fused update, 2k + 3 vector passes
            // instead of 4k for the k sequential projections of a MGS pass
            cgs_pass(h, cand, corr, 1.0 / cnorm, V, k_sub, n, false);
            cgs_pass(h, cand, cand, 1.0, V, k_sub, n, true);
            read_slots(h, 4, 1, &nrm2);
        }
        const double norm = std::sqrt(nrm2);
        push();
        if (!(norm >= 1e-10)) {
            status = 2;
            break;
        }
        if (!prenormalised) {
            k_scale_div<<<vgrid, kRedThreads, 0, h.stream>>>(cand, n, norm);
            CUDA_LAUNCH_CHECK();
        }
        ++k_sub;
    }

    res->status = status;
    res->converged = status == 0;
    res->iterations = iters;
    res->energy = theta;
    if (res->eigenvector) {
        if (!ritz_fresh && !coeffs.empty()) {   // fused passes: materialise the Ritz vector now
            RitzArgs ra{};
            for (int j = 0; j < static_cast<int>(coeffs.size()); ++j) {
                ra.v[j] = V(j);
                ra.w[j] = Wv(j);
                ra.c[j] = coeffs[j];
            }
            ra.k = static_cast<int>(coeffs.size());
            ra.theta = theta;
            k_ritz<<<kRedBlocks, kRedThreads, 0, h.stream>>>(ra, h.diag.p, n, ritz, img, corr, h.red.p);
            CUDA_LAUNCH_CHECK();
        }
        const double nrm = std::sqrt(device_dot(h, ritz, ritz, n));
        k_scale_div<<<vgrid, kRedThreads, 0, h.stream>>>(ritz, n, nrm);
        CUDA_LAUNCH_CHECK();
        CUDA_CHECK(cudaMemcpyAsync(res->eigenvector, ritz, n * sizeof(double), cudaMemcpyDeviceToHost,
                                   h.stream));
    }
    if (res->trace)
        for (int i = 0; i < std::min(res->trace_cap, iters); ++i) res->trace[i] = trace[i];
    CUDA_CHECK(cudaStreamSynchronize(h.stream));
    res->seconds = seconds_since(wall0);
}


// ---------------------------------------------------------------------------
// Multi-root block Davidson (Davidson-Liu): SURVEY.md 8(f) rank 1, BASELINE
// config C5.  A capability beyond the reference (single root,
// davidson.hpp:83-86) built from the same rules: guesses are unit vectors at
// the nroots lowest diagonal entries (lowest index on ties), lower-triangle
// projected fill, Jacobi on the host, per-root residual and the clamped
// diagonal preconditioner, 2-pass MGS against the subspace (and the
// corrections added before it in the same iteration) with the 1e-10
// dependence threshold, and collapse to the nroots Ritz pairs when the next
// block would exceed max_subspace.  New vectors of one iteration go through
// one blocked sigma call.
// ---------------------------------------------------------------------------
void davidson_roots_device(Handle& h, const detci_dav_block_opts& opts, detci_dav_block_result* res) {
    if (!h.built) fail(DETCI_GPU_E_INPUT, "davidson_solve: basis not built");
    const uint64_t n = h.local_len();
    const int m = opts.nroots;
    if (m < 1) fail(DETCI_GPU_E_CONFIG, "davidson_roots: nroots must be positive");
    if (!(opts.tol > 0.0)) fail(DETCI_GPU_E_CONFIG, "davidson_solve: tol must be positive");
    if (opts.max_iter < 1) fail(DETCI_GPU_E_CONFIG, "davidson_solve: max_iter must be positive");
    if (opts.max_subspace < 2 * m) fail(DETCI_GPU_E_CONFIG, "davidson_roots: max_subspace must be >= 2*nroots");
    if (opts.max_subspace > kMaxVec) fail(DETCI_GPU_E_UNSUPPORTED, "davidson_solve: max_subspace above 64");
    const uint64_t dim_global = static_cast<uint64_t>(h.na()) * h.nb();
    if (static_cast<uint64_t>(m) > dim_global) fail(DETCI_GPU_E_INPUT, "davidson_roots: nroots exceeds the dimension");
    ensure_red(h);
    const int ms = opts.max_subspace;
    const auto wall0 = std::chrono::steady_clock::now();

    size_t free_b = 0, total_b = 0;
    CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
    const size_t nvec = 2 * static_cast<size_t>(ms) + 3 * static_cast<size_t>(m);
    const size_t need = nvec * n * sizeof(double);
    const bool grow = h.dav_store.bytes() < need;   // as in davidson_device
    const bool drop_d = grow && need + (1ull << 30) > free_b + h.dav_store.bytes();
    free_b += h.dbuf.bytes() + h.dav_store.bytes();
    const uint64_t budget = std::min<uint64_t>(h.budget ? h.budget : free_b, free_b);
    if (n == 0) collective_require(h, false, DETCI_GPU_E_INPUT, "davidson_solve: empty diagonal", "davidson_roots");
    else
        collective_require(h, need <= budget, DETCI_GPU_E_CAPACITY,
                       "davidson vectors require " + std::to_string(need) + " bytes, budget is " +
                           std::to_string(budget) + " bytes",
                       "davidson_roots");
    DevBuf<double>& store = h.dav_store;
    if (drop_d) release_sigma_scratch(h);
    if (grow) {
        store.reset();
        store.alloc(nvec * n);
    }
    auto V = [&](int j) { return store.p + static_cast<size_t>(j) * n; };
    auto Wv = [&](int j) { return store.p + static_cast<size_t>(ms + j) * n; };
    auto RZ = [&](int r) { return store.p + static_cast<size_t>(2 * ms + r) * n; };
    auto IM = [&](int r) { return store.p + static_cast<size_t>(2 * ms + m + r) * n; };
    auto CR = [&](int r) { return store.p + static_cast<size_t>(2 * ms + 2 * m + r) * n; };

    // guesses: the m lowest diagonal entries (lowest index first on ties),
    // found on the device one rank-local pick per round
    {
        const uint64_t keep = std::min<uint64_t>(n, static_cast<uint64_t>(m));
        std::vector<double> cand(2 * m, INFINITY);  // (value, global index) of local best
        DevBuf<double> pv;
        DevBuf<uint64_t> pi;
        pv.alloc(kRedBlocks);
        pi.alloc(kRedBlocks);
        std::vector<double> hv(kRedBlocks);
        std::vector<uint64_t> hi(kRedBlocks);
        double v0 = 0.0;
        uint64_t i0 = 0;
        for (uint64_t r = 0; r < keep; ++r) {
            k_argmin_after<<<kRedBlocks, kRedThreads, 0, h.stream>>>(h.diag.p, n, v0, i0, r == 0 ? 1 : 0, pv.p, pi.p);
            CUDA_LAUNCH_CHECK();
            CUDA_CHECK(cudaMemcpyAsync(hv.data(), pv.p, kRedBlocks * sizeof(double), cudaMemcpyDeviceToHost, h.stream));
            CUDA_CHECK(cudaMemcpyAsync(hi.data(), pi.p, kRedBlocks * sizeof(uint64_t), cudaMemcpyDeviceToHost, h.stream));
            CUDA_CHECK(cudaStreamSynchronize(h.stream));
            double bv = INFINITY;
            uint64_t bi = ~0ull;
            for (int b = 0; b < kRedBlocks; ++b)
                if (hv[b] < bv || (hv[b] == bv && hi[b] < bi)) {
                    bv = hv[b];
                    bi = hi[b];
                }
            if (bi == ~0ull) break;
            cand[2 * r] = bv;
            cand[2 * r + 1] = static_cast<double>(bi + h.a0 * h.nb());
            v0 = bv;
            i0 = bi;
        }
        std::vector<double> all(2 * static_cast<size_t>(m) * h.world, 0.0);
        std::copy(cand.begin(), cand.end(), all.begin() + 2 * static_cast<size_t>(m) * h.rank);
        allreduce_sum(h, all.data(), static_cast<int>(all.size()));
        std::vector<std::pair<double, double>> pool;
        for (size_t i = 0; i < all.size(); i += 2)
            if (std::isfinite(all[i])) pool.emplace_back(all[i], all[i + 1]);
        std::sort(pool.begin(), pool.end());
        const uint64_t lo = h.a0 * h.nb();
        for (int r = 0; r < m; ++r) {
            const uint64_t gi = static_cast<uint64_t>(pool[r].second);
            k_set_unit<<<kRedBlocks, kRedThreads, 0, h.stream>>>(V(r), n, gi >= lo && gi < lo + n ? gi - lo : ~0ull);
            CUDA_LAUNCH_CHECK();
        }
    }

    std::vector<double> proj(static_cast<size_t>(ms) * ms, 0.0), gram(static_cast<size_t>(ms) * ms, 0.0);
    std::vector<double> evals, evecs, theta(m, 0.0), rnorm(m, 0.0);
    int k_sub = m, k_img = 0, status = 0, iters = 0;
    bool restart_pending = false;
    std::vector<detci_dav_iter> trace;

    auto fill_rows = [&](int from, int to) {  // projected + Gram rows [from, to)
        for (int i = from; i < to; ++i) {
            std::vector<const double*> ys(2 * (i + 1));
            for (int j = 0; j <= i; ++j) {
                ys[j] = Wv(j);
                ys[i + 1 + j] = V(j);
            }
            std::vector<double> dots(2 * (i + 1));
            device_dot_many(h, V(i), ys.data(), 2 * (i + 1), n, dots.data());
            for (int j = 0; j <= i; ++j) {
                proj[i * ms + j] = dots[j];
                gram[i * ms + j] = dots[i + 1 + j];
            }
        }
    };

    bool ritz_fresh = false;
    int last_k = 0;
    // Ritz vector, image and correction of root r from the current
    // subspace (k vectors) and eigenpairs
    auto ritz_root = [&](int r, int k) {
        RitzArgs ra{};
        for (int j = 0; j < k; ++j) {
            ra.v[j] = V(j);
            ra.w[j] = Wv(j);
            ra.c[j] = evecs[static_cast<size_t>(r) * k + j];
        }
        ra.k = k;
        ra.theta = evals[r];
        k_ritz<<<kRedBlocks, kRedThreads, 0, h.stream>>>(ra, h.diag.p, n, RZ(r), IM(r), CR(r), h.red.p);
        CUDA_LAUNCH_CHECK();
    };
    for (int iter = 0; iter < opts.max_iter; ++iter) {
        detci_dav_iter st{};
        st.restarted = restart_pending ? 1 : 0;
        restart_pending = false;
        auto t0 = std::chrono::steady_clock::now();
        if (k_img < k_sub) {  // one blocked sigma for the new vectors
            std::vector<const double*> xs;
            std::vector<double*> ys;
            for (int j = k_img; j < k_sub; ++j) {
                xs.push_back(V(j));
                ys.push_back(Wv(j));
            }
            sigma_block(h, xs.data(), ys.data(), static_cast<int>(xs.size()));
            const int first = k_img;
            k_img = k_sub;
            st.matvec_seconds = seconds_since(t0);
            t0 = std::chrono::steady_clock::now();
            fill_rows(first, k_sub);
        } else {
            st.matvec_seconds = seconds_since(t0);
            t0 = std::chrono::steady_clock::now();
        }
        const int k = k_sub;
        jacobi_eigen(proj, ms, k, evals, evecs);
        last_k = k;
        st.subspace_solve_seconds = seconds_since(t0);

        t0 = std::chrono::steady_clock::now();
        double worst = 0.0;
        std::vector<double> cnorm(m, 0.0);
        if (fused_block_ritz(m, k, n)) {
            // all m corrections in one pass; Ritz vectors / images later
            BlockRitzArgs ba{};
            for (int j = 0; j < k; ++j) {
                ba.s[j] = V(j);
                ba.s[k + j] = Wv(j);
            }
            ba.s[2 * k] = h.diag.p;
            for (int r = 0; r < m; ++r) {
                for (int j = 0; j < k; ++j) ba.c[r][j] = evecs[static_cast<size_t>(r) * k + j];
                ba.theta[r] = evals[r];
                ba.out[r] = CR(r);
            }
            ba.k = k;
            ba.m = m;
            ba.ns = 2 * k + 1;
            ba.nst = 2;
            ba.n = n;
            ba.T = static_cast<uint32_t>(std::min<size_t>(4096, kStSmem / 8 / (2 * static_cast<size_t>(ba.ns))) &
                                         ~size_t{31});
            ba.partial = h.red.p;
            const size_t smem = 2 * static_cast<size_t>(ba.ns) * ba.T * sizeof(double);
            const int grid = sm_count();
            ensure_dynamic_smem(reinterpret_cast<const void*>(&k_ritz_block), smem);
            k_ritz_block<<<grid, 512, smem, h.stream>>>(ba);
            CUDA_LAUNCH_CHECK();
            k_finalize<<<2 * m, 32, 0, h.stream>>>(h.red.p, grid, 2 * m, scalar_slot(h, 0));
            CUDA_LAUNCH_CHECK();
            allreduce_device(h, scalar_slot(h, 0), 2 * m);
            std::vector<double> nn(2 * m);
            read_slots(h, 0, 2 * m, nn.data());
            for (int r = 0; r < m; ++r) {
                theta[r] = evals[r];
                rnorm[r] = std::sqrt(nn[r]);
                cnorm[r] = std::sqrt(nn[m + r]);
                worst = std::max(worst, rnorm[r]);
            }
            ritz_fresh = false;
        } else {
            for (int r = 0; r < m; ++r) {
                ritz_root(r, k);
                finalize_to(h, 2, 0);
                double nn2[2];
                read_slots(h, 0, 2, nn2);
                theta[r] = evals[r];
                rnorm[r] = std::sqrt(nn2[0]);
                cnorm[r] = std::sqrt(nn2[1]);
                worst = std::max(worst, rnorm[r]);
            }
            ritz_fresh = true;
        }
        double gdev = 0.0;
        for (int i = 0; i < k; ++i)
            for (int j = 0; j <= i; ++j)
                gdev = std::max(gdev, std::fabs(gram[i * ms + j] - (i == j ? 1.0 : 0.0)));
        st.max_gram_deviation = gdev;
        st.ritz_value = theta[0];
        st.residual_norm = worst;
        auto push = [&]() {
            st.orthogonalization_seconds = seconds_since(t0);
            trace.push_back(st);
            ++iters;
        };
        const bool converged = worst <= opts.tol;
        if (converged || iter + 1 == opts.max_iter) {
            push();
            status = converged ? 0 : 1;
            break;
        }
        int unconverged = 0;
        for (int r = 0; r < m; ++r) unconverged += rnorm[r] > opts.tol && cnorm[r] > 0.0;
        if (k_sub + unconverged > ms) {  // collapse to the m Ritz pairs
            if (!ritz_fresh) {
                // Ritz vectors and images (and, again, the corrections) by
                // the per-root pass before V[0..m) is overwritten
                for (int r = 0; r < m; ++r) ritz_root(r, k);
                ritz_fresh = true;
            }
            for (int r = 0; r < m; ++r) {
                CUDA_CHECK(cudaMemcpyAsync(V(r), RZ(r), n * 8, cudaMemcpyDeviceToDevice, h.stream));
                CUDA_CHECK(cudaMemcpyAsync(Wv(r), IM(r), n * 8, cudaMemcpyDeviceToDevice, h.stream));
            }
            k_sub = k_img = m;
            fill_rows(0, m);
            restart_pending = true;
        }
        int added = 0;
        for (int r = 0; r < m; ++r) {
            if (!(rnorm[r] > opts.tol) || !(cnorm[r] > 0.0)) continue;
            if (k_sub >= ms) break;
            double* cand = V(k_sub);
            const int kk = k_sub;
            double nrm2 = 0.0;
            if (ortho_mgs()) {
                const int steps = 2 * kk;
                for (int t = 0; t <= steps; ++t) {
                    const double* src = t == 0 ? CR(r) : nullptr;
                    const double* vprev = t == 0 ? nullptr : V((t - 1) % kk);
                    const double* vnext = t == steps ? nullptr : V(t % kk);
                    k_mgs_step<<<kRedBlocks, kRedThreads, 0, h.stream>>>(cand, src, cnorm[r], vprev,
                                                                          scalar_slot(h, 4 + (t + 1) % 2), vnext,
                                                                          n, h.red.p);
                    CUDA_LAUNCH_CHECK();
                    finalize_to(h, 1, 4 + t % 2);
                }
                read_slots(h, 4 + steps % 2, 1, &nrm2);
            } else {
                cgs_pass(h, cand, CR(r), 1.0 / cnorm[r], V, kk, n, false);
                cgs_pass(h, cand, cand, 1.0, V, kk, n, true);
                read_slots(h, 4, 1, &nrm2);
            }
            const double norm = std::sqrt(nrm2);
            if (!(norm >= 1e-10)) continue;
            k_scale_div<<<kRedBlocks, kRedThreads, 0, h.stream>>>(cand, n, norm);
            CUDA_LAUNCH_CHECK();
            ++k_sub;
            ++added;
        }
        push();
        if (added == 0) {
            status = 2;
            break;
        }
    }

    res->status = status;
    res->converged = status == 0;
    res->iterations = iters;
    if (res->eigenvectors && !ritz_fresh && last_k > 0)
        for (int r = 0; r < m; ++r) ritz_root(r, last_k);
    for (int r = 0; r < m; ++r) {
        if (res->energies) res->energies[r] = theta[r];
        if (res->residuals) res->residuals[r] = rnorm[r];
        if (res->eigenvectors) {
            const double nrm = std::sqrt(device_dot(h, RZ(r), RZ(r), n));
            k_scale_div<<<kRedBlocks, kRedThreads, 0, h.stream>>>(RZ(r), n, nrm);
            CUDA_LAUNCH_CHECK();
            CUDA_CHECK(cudaMemcpyAsync(res->eigenvectors + static_cast<size_t>(r) * n, RZ(r), n * 8,
                                       cudaMemcpyDeviceToHost, h.stream));
        }
    }
    if (res->trace)
        for (int i = 0; i < std::min(res->trace_cap, iters); ++i) res->trace[i] = trace[i];
    CUDA_CHECK(cudaStreamSynchronize(h.stream));
    res->seconds = seconds_since(wall0);
}

} // namespace detci_gpu
