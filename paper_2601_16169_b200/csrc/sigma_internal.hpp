// Internal interface of the sigma translation units (sigma.cu: schedules
// and entry points; samespin.cu: same-spin kernels; mixed.cu: mixed-term
// kernels).  Not part of the C-ABI.
#pragma once

#include <array>
#include <vector>
#include <cstdint>
#include <utility>

#include "comm.hpp"
#include "handle.hpp"

namespace detci_gpu {

constexpr int kMaxM = 4;   // vectors per blocked pass
constexpr int kMxBlock = 1024;   // mixed-term CTA: one per SM, 32 warps

// CUDA-event phase timer on the compute stream (detci_gpu_timings split).
struct PhaseTimer {
    Handle& h;
    bool on;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    std::vector<int> cat, rk;
    int rank_tag = -1;   // virtual block-rank the following phases belong to (-1: none)
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
        rk.push_back(rank_tag);
        return static_cast<int>(ev.size()) - 1;
    }
    void end(int id) {
        if (id >= 0) CUDA_CHECK(cudaEventRecord(ev[id].second, h.stream));
    }
    // categories: 0 alpha, 1 beta, 2 mixed, 3 combine, 4 the D reductions
    // (inside the mixed phase)
    void collect(double out[5]) {
        for (int i = 0; i < 5; ++i) out[i] = 0.0;
        for (size_t i = 0; i < ev.size(); ++i) {
            float ms = 0.f;
            CUDA_CHECK(cudaEventElapsedTime(&ms, ev[i].first, ev[i].second));
            out[cat[i]] += ms * 1e-3;
        }
    }
    // device seconds per tagged block-rank (phases 0-3; the reductions are
    // inside the mixed phase)
    std::vector<double> per_rank(int P) {
        std::vector<double> t(std::max(P, 0), 0.0);
        for (size_t i = 0; i < ev.size(); ++i) {
            if (rk[i] < 0 || rk[i] >= P || cat[i] == 4) continue;
            float ms = 0.f;
            CUDA_CHECK(cudaEventElapsedTime(&ms, ev[i].first, ev[i].second));
            t[rk[i]] += ms * 1e-3;
        }
        return t;
    }
    // the same by phase: t[rank * 4 + phase], phases 0-3
    std::vector<double> per_rank_phase(int P) {
        std::vector<double> t(4 * static_cast<size_t>(std::max(P, 0)), 0.0);
        for (size_t i = 0; i < ev.size(); ++i) {
            if (rk[i] < 0 || rk[i] >= P || cat[i] == 4) continue;
            float ms = 0.f;
            CUDA_CHECK(cudaEventElapsedTime(&ms, ev[i].first, ev[i].second));
            t[4 * static_cast<size_t>(rk[i]) + cat[i]] += ms * 1e-3;
        }
        return t;
    }
};

using Ptrs = std::array<const double*, kMaxM>;
using MPtrs = std::array<double*, kMaxM>;

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
    const uint64_t* eps_row_hi;   // norbs > 64: high words (else null)
    const uint64_t* eps_col_hi;
    const double* diag;       // if set (write mode): Y = diag * Cself + acc
    const double* Cself[kMaxM];
    int accumulate;
};

// Where the mixed term goes: beta slots [slot0, slot_end) and, if T is set,
// overwrite T[v][(ia - a0) * ldt + slot - slot0] (slot order) instead of
// accumulating into y[ia][perm[slot]].
struct MixedTarget {
    uint32_t slot0 = 0, slot_end = 0xffffffffu;
    double* T[kMaxM] = {};
    size_t ldt = 0;
};

// samespin.cu
template <int M> void launch_samespin(const SameSpinArgs& s, cudaStream_t st);
void fill_lists(SameSpinArgs& s, const ChannelTables& t);
// alpha term for list rows [a0, a1): Cs rows [b0, b1) in Cb; first: y =
// diag*C + ... (add_to_y: y += diag*C + ...), else y += ...
template <int M>
void launch_alpha(const Handle& h, const Ptrs& Cb, uint32_t b0, uint32_t b1, const Ptrs& x_loc,
                  const MPtrs& y_loc, uint64_t a0, uint64_t a1, bool first, bool add_to_y = false);

// mixed.cu
template <int M>
void launch_mixed(Handle& h, const Ptrs& Cb, uint32_t b0, uint32_t b1, const MPtrs& y_loc, uint64_t a0,
                  uint64_t a1);
const std::vector<std::unique_ptr<ScatterWindow>>& scatter_windows(Handle& h, int g, int P, int M, int kmax);
template <int M>
void launch_mixed_scatter(Handle& h, int g, int P, int b, const Ptrs& Cb, uint32_t b0, uint32_t b1,
                          const MPtrs& y_loc, uint64_t a0, int phases = 3, uint64_t r_lo = 0,
                          uint64_t r_hi = ~0ull, int only_window = -1, const MixedTarget& tgt = MixedTarget{});
bool multi_ring();
std::pair<uint32_t, uint32_t> mixed_slots(const Handle& h, int g, int P);
template <int M>
void unpack_slab(Handle& h, const double* R, size_t ldr, uint32_t ns, uint64_t rows, uint32_t s0, double* y);
template <int M>
void mixed_columns(Handle& h, int g, int P, const Ptrs& Cfull, double* const* T, size_t ldt);

} // namespace detci_gpu
