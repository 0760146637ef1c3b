// Shared device helpers and the error convention of libdetci_gpu.so.
//
// Bit conventions follow the reference (paths relative to
// /root/reference/proj/core): spatial orbital p of a channel string is bit p
// of one uint64 mask; in the interleaved determinant alpha p is spin-orbital
// 2p and beta p is 2p+1 (bitstring.hpp:13-16).  Fermionic signs are
// (-1)^(occupied spin-orbitals strictly between the moved pair in the bra)
// (bitstring.hpp:109-114).  Splitting that count per channel gives the masks
// below (re-derived in DESIGN.md "phase"):
//   alpha move a<->b : same-channel open(a,b) plus beta bits [lo, hi-1]
//   beta  move a<->b : same-channel open(a,b) plus alpha bits [lo+1, hi]
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace detci_gpu {

// Exception carrying a detci_gpu_status code; converted at the C-ABI.
struct Failure : std::runtime_error {
    int code;
    Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Failure(code, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess)
        fail(7, std::string("CUDA error in ") + what + " (" + file + ":" + std::to_string(line) +
                    "): " + cudaGetErrorString(e));
}

#define CUDA_CHECK(expr) ::detci_gpu::cuda_check((expr), #expr, __FILE__, __LINE__)
// Host<->device copy ordered on `s` and complete at return.  (A plain
// cudaMemcpy runs on the legacy stream, which does not order with the
// non-blocking streams the kernels run on, and a pageable H2D cudaMemcpy may
// return before its DMA lands: a kernel launched right after on another
// stream could read stale data.)
inline void copy_sync(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
    if (bytes == 0) return;
    cuda_check(cudaMemcpyAsync(dst, src, bytes, kind, s), "cudaMemcpyAsync", __FILE__, __LINE__);
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize", __FILE__, __LINE__);
}

// Every kernel launch site ends with CUDA_LAUNCH_CHECK(), which also counts
// the launch (detci_gpu_launch_count; bench.py reports it as gpu_launches).
void count_launch();
#define CUDA_LAUNCH_CHECK()                                                                  \
    do {                                                                                     \
        ::detci_gpu::count_launch();                                                         \
        ::detci_gpu::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__);    \
    } while (0)

// Bits [lo, hi] inclusive of a 64-bit word (empty when lo > hi).
__host__ __device__ __forceinline__ uint64_t bit_range(int lo, int hi) {
    if (lo > hi) return 0ull;
    return (~0ull >> (63 - hi)) & (~0ull << lo);
}

// Bits strictly between a and b.
__host__ __device__ __forceinline__ uint64_t open_mask(int a, int b) {
    const int lo = a < b ? a : b, hi = a < b ? b : a;
    return bit_range(lo + 1, hi - 1);
}

// Spectator mask of a move a<->b in channel `ch` (0 alpha, 1 beta): the
// other channel's bits that lie between spin-orbitals of the moved pair.
__host__ __device__ __forceinline__ uint64_t spectator_mask(int ch, int a, int b) {
    const int lo = a < b ? a : b, hi = a < b ? b : a;
    return ch == 0 ? bit_range(lo, hi - 1) : bit_range(lo + 1, hi);
}

#ifdef __CUDACC__
__device__ __forceinline__ int parity64(uint64_t x) { return __popcll(x) & 1; }

// v * (-1)^bit by flipping the IEEE sign bit (exact, branch-free).
__device__ __forceinline__ double flip_sign(double v, uint32_t bit) {
    return __longlong_as_double(__double_as_longlong(v) ^ (static_cast<unsigned long long>(bit & 1u) << 63));
}

// Sign bit already in position 31 of `word` (the packed SELL entry format).
__device__ __forceinline__ double flip_sign_hi(double v, uint32_t word) {
    const int lo = __double2loint(v);
    const int hi = __double2hiint(v) ^ static_cast<int>(word & 0x80000000u);
    return __hiloint2double(hi, lo);
}
#endif

// Triangular index of an unordered orbital pair p != q (J tables).
__host__ __device__ __forceinline__ uint32_t tri_index(int p, int q) {
    const int lo = p < q ? p : q, hi = p < q ? q : p;
    return static_cast<uint32_t>(hi * (hi - 1) / 2 + lo);
}

constexpr int kWarp = 32;

} // namespace detci_gpu
