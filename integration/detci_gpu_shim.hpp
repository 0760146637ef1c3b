// detci_gpu_shim.hpp -- the drop-in for code inside the reference tree
// (proj/core).  Converts the reference's value types to the C-ABI
// (include/detci_gpu.h) and rethrows status codes as detci::Error subclasses,
// keeping the reference signatures:
//
//   build_basis_gpu(const detci::Basis&)          device copy of a host Basis
//   build_basis_gpu(alpha, beta, IntegralTable, BasisOptions)
//                                                 build_basis (basis.hpp:85-86)
//                                                 with tables + diag built on
//                                                 the device
//   matvec(DeviceBasis, x, y, MatvecTimings*)     matvec.hpp:64-65 (plan and
//                                                 workers are scheduling-only
//                                                 in the reference and have no
//                                                 device meaning)
//   linear_operator(DeviceBasis) -> detci::LinearOperator   davidson.hpp:28
//   davidson_solve(DeviceBasis, DavidsonOptions) -> detci::DavidsonResult
//
// INTEGRATION.md shows the run.cpp hook (Method::Gpu) that uses these.
#pragma once

#include <chrono>
#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include <detci/basis.hpp>
#include <detci/davidson.hpp>
#include <detci/error.hpp>
#include <detci/matvec.hpp>
#include <detci/slater_condon.hpp>

#include "../include/detci_gpu.h"

namespace detci::gpu {

inline void rethrow(int code, const detci_gpu_handle* h) {
    if (code == DETCI_GPU_OK) return;
    const std::string msg = detci_gpu_last_error(h);
    switch (code) {
        case DETCI_GPU_E_INPUT: throw InputError(msg);
        case DETCI_GPU_E_FORMAT: throw FormatError(msg);
        case DETCI_GPU_E_CONFIG: throw ConfigError(msg);
        case DETCI_GPU_E_CAPACITY: throw CapacityError(msg);
        case DETCI_GPU_E_UNSUPPORTED: throw UnsupportedError(msg);
        default: throw Error(msg);
    }
}

/// uint64 words per channel string on the device: 1 for norbs <= 64, 2 up
/// to 128 (the reference itself allows kMaxKernelBits = 256 spin-orbitals).
inline int string_words(int norbs) {
    if (norbs > 128) throw UnsupportedError("gpu: norbs > 128 is not supported on the device path");
    return norbs > 64 ? 2 : 1;
}

/// Channel strings as string_words(norbs) uint64 words each, word w holding
/// orbitals 64w .. 64w+63 (from occupied_list, whatever the BitString's
/// bit_length).
inline std::vector<std::uint64_t> channel_masks(const std::vector<BitString>& strings, int norbs) {
    const int w = string_words(norbs);
    std::vector<std::uint64_t> out(strings.size() * w, 0);
    for (std::size_t k = 0; k < strings.size(); ++k)
        for (int i : occupied_list(strings[k])) out[k * w + i / 64] |= std::uint64_t{1} << (i % 64);
    return out;
}

struct DeviceOptions {
    int device = 0, rank = 0, world_size = 1, virtual_blocks = 1;
    bool weighted_partition = true;
    const std::uint8_t* nccl_id = nullptr;
    std::uint64_t memory_budget_bytes = 0;
    // > 0: the world_size ranks are host threads of this process over the
    // loopback transport (group id), not NCCL (detci_gpu_create_loopback)
    std::uint64_t loopback_group = 0;
    // > 0: rounds of the measured rebalance after the build (world_size or
    // virtual_blocks > 1; detci_gpu_rebalance)
    int balance_rounds = 0;
};

class DeviceBasis {
public:
    /// Device copy of a host Basis built by the reference build_basis.
    explicit DeviceBasis(const Basis& basis, const DeviceOptions& o = {}) {
        init(basis.norbs, channel_masks(basis.alpha_strings, basis.norbs),
             channel_masks(basis.beta_strings, basis.norbs), basis.integrals, o);
    }
    /// Device basis straight from the string lists and integrals (the
    /// host never builds tables, cache or diagonal).
    DeviceBasis(int norbs, const std::vector<std::uint64_t>& a, const std::vector<std::uint64_t>& b,
                const IntegralTable& table, const DeviceOptions& o = {}) {
        init(norbs, a, b, table, o);
    }
    DeviceBasis(const DeviceBasis&) = delete;
    DeviceBasis& operator=(const DeviceBasis&) = delete;
    ~DeviceBasis() { detci_gpu_destroy(h_); }

    detci_gpu_handle* handle() const { return h_; }
    std::size_t local_dimension() const { return local_dim_; }
    std::uint64_t row_begin() const { return row_begin_; }
    std::uint64_t row_end() const { return row_end_; }

private:
    void init(int n, const std::vector<std::uint64_t>& a, const std::vector<std::uint64_t>& b,
              const IntegralTable& table, const DeviceOptions& o) {
        detci_gpu_desc d{o.device, o.rank, o.world_size, o.nccl_id, o.virtual_blocks,
                         o.weighted_partition ? 1 : 0, o.memory_budget_bytes};
        if (o.loopback_group) rethrow(detci_gpu_create_loopback(&d, o.loopback_group, &h_), nullptr);
        else rethrow(detci_gpu_create(&d, &h_), nullptr);
        try {
            const int w = string_words(n);
            rethrow(detci_gpu_set_strings_words(h_, n, w, a.data(), a.size() / w, b.data(), b.size() / w), h_);
            const std::size_t nn = static_cast<std::size_t>(n);
            std::vector<double> h1(nn * nn), eri(nn * nn * nn * nn);
            for (int p = 0; p < n; ++p)
                for (int q = 0; q < n; ++q) h1[p * nn + q] = table.one_electron(p, q);
            for (int p = 0; p < n; ++p)
                for (int q = 0; q < n; ++q)
                    for (int r = 0; r < n; ++r)
                        for (int s = 0; s < n; ++s)
                            eri[((p * nn + q) * nn + r) * nn + s] = table.two_electron(p, q, r, s);
            rethrow(detci_gpu_set_integrals(h_, table.core_energy(), h1.data(), eri.data()), h_);
            rethrow(detci_gpu_build_basis(h_), h_);
            if (o.balance_rounds > 0) rethrow(detci_gpu_rebalance(h_, o.balance_rounds, nullptr), h_);
            std::uint64_t nb = 0;
            rethrow(detci_gpu_local_rows(h_, &row_begin_, &row_end_, &nb), h_);
            local_dim_ = (row_end_ - row_begin_) * nb;
        } catch (...) {
            detci_gpu_destroy(h_);
            h_ = nullptr;
            throw;
        }
    }

    detci_gpu_handle* h_ = nullptr;
    std::uint64_t row_begin_ = 0, row_end_ = 0;
    std::size_t local_dim_ = 0;
};

inline std::unique_ptr<DeviceBasis> build_basis_gpu(const Basis& basis, const DeviceOptions& o = {}) {
    return std::make_unique<DeviceBasis>(basis, o);
}

/// build_basis (basis.hpp:85-86, basis.cpp:78-148)
/// end to end on the device.  The helper lists and the diagonal are built in
/// HBM and copied back into a host Basis with the reference's field layout
/// (strings repacked at the same bit_length, integrals, J/K, the four
/// FlatExcitationTables, diag); the determinant cache is left empty, which the
/// reference treats as "compute on the fly" (basis.hpp:63-70), and the
/// budget check on it does not apply.  Errors follow build_basis: too many
/// spin-orbitals, empty lists, bad popcounts and duplicates are InputError.
struct GpuBuiltBasis {
    std::unique_ptr<DeviceBasis> device;
    Basis host;
};

inline GpuBuiltBasis build_basis_gpu(std::vector<BitString> alpha, std::vector<BitString> beta, IntegralTable table,
                                     const BasisOptions& opts = {}, const DeviceOptions& o = {}) {
    const auto t0 = std::chrono::steady_clock::now();
    const int n = table.norbs();
    if (2 * n > kMaxKernelBits)
        throw InputError("build_basis: " + std::to_string(2 * n) + " spin-orbitals exceed the kernel limit of " +
                         std::to_string(kMaxKernelBits));
    GpuBuiltBasis out;
    out.device = std::make_unique<DeviceBasis>(n, channel_masks(alpha, n), channel_masks(beta, n), table, o);
    detci_gpu_handle* h = out.device->handle();
    Basis& B = out.host;
    B.norbs = n;
    const int bit_length = opts.bit_length != 0 ? opts.bit_length : (2 * n <= 64 ? 2 * n : 20);
    B.channel_packing = make_packing(n, bit_length);
    B.det_packing = make_packing(2 * n, bit_length);
    B.alpha_strings.reserve(alpha.size());
    B.beta_strings.reserve(beta.size());
    for (const BitString& s : alpha) B.alpha_strings.push_back(repack(s, bit_length));
    for (const BitString& s : beta) B.beta_strings.push_back(repack(s, bit_length));
    B.n_elec_alpha = static_cast<int>(occupied_list(B.alpha_strings.front()).size());
    B.n_elec_beta = static_cast<int>(occupied_list(B.beta_strings.front()).size());
    B.integrals = std::move(table);
    B.jk = build_direct_exchange(B.integrals);
    FlatExcitationTable* tabs[2][2] = {{&B.singles_a, &B.doubles_a}, {&B.singles_b, &B.doubles_b}};
    for (int ch = 0; ch < 2; ++ch)
        for (int kind = 0; kind < 2; ++kind) {
            std::uint64_t nflat = 0;
            rethrow(detci_gpu_helper_size(h, ch, kind, &nflat), h);
            FlatExcitationTable& t = *tabs[ch][kind];
            const std::size_t ns = ch == 0 ? B.alpha_strings.size() : B.beta_strings.size();
            std::vector<std::uint64_t> off(ns);
            t.flat.resize(nflat);
            t.len.resize(ns);
            rethrow(detci_gpu_get_helpers(h, ch, kind, t.flat.data(), off.data(), t.len.data()), h);
            t.offset.assign(off.begin(), off.end());
        }
    B.diag.resize(out.device->local_dimension());
    rethrow(detci_gpu_diag(h, B.diag.data()), h);
    B.stats.connectivity_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return out;
}

inline void matvec(const DeviceBasis& db, std::span<const double> x, std::span<double> y,
                   MatvecTimings* timings = nullptr) {
    if (x.size() != db.local_dimension() || y.size() != db.local_dimension())
        throw InputError("matvec: vector length " + std::to_string(x.size()) +
                         " does not match basis dimension " + std::to_string(db.local_dimension()));
    detci_gpu_timings t{};
    rethrow(detci_gpu_sigma(db.handle(), x.data(), y.data(), timings ? &t : nullptr), db.handle());
    if (timings) {
        timings->alpha_seconds = t.alpha_seconds;
        timings->beta_seconds = t.beta_seconds;
        timings->mixed_seconds = t.mixed_seconds;
        timings->combine_seconds = t.combine_seconds;
    }
}

inline LinearOperator linear_operator(const DeviceBasis& db) {
    return [&db](std::span<const double> x, std::span<double> y) { matvec(db, x, y); };
}

inline DavidsonResult davidson_solve(const DeviceBasis& db, const DavidsonOptions& o = {}) {
    if (!o.initial_guess.empty() && o.initial_guess.size() != db.local_dimension())
        throw InputError("davidson_solve: initial guess length mismatch");
    detci_dav_opts opts{o.tol, o.max_iter, o.max_subspace,
                        o.initial_guess.empty() ? nullptr : o.initial_guess.data()};
    std::vector<detci_dav_iter> trace(static_cast<std::size_t>(o.max_iter > 0 ? o.max_iter : 1));
    DavidsonResult r;
    r.eigenvector.resize(db.local_dimension());
    detci_dav_result res{};
    res.eigenvector = r.eigenvector.data();
    res.trace = trace.data();
    res.trace_cap = static_cast<int>(trace.size());
    rethrow(detci_gpu_davidson(db.handle(), &opts, &res, nullptr, nullptr), db.handle());
    r.status = res.status == 0 ? SolveStatus::Converged
                               : (res.status == 1 ? SolveStatus::MaxIterationsReached : SolveStatus::Stagnated);
    r.converged = res.converged != 0;
    r.energy = res.energy;
    for (int i = 0; i < res.iterations; ++i) {
        IterationStats s;
        s.ritz_value = trace[i].ritz_value;
        s.residual_norm = trace[i].residual_norm;
        s.matvec_seconds = trace[i].matvec_seconds;
        s.orthogonalization_seconds = trace[i].orthogonalization_seconds;
        s.subspace_solve_seconds = trace[i].subspace_solve_seconds;
        s.max_gram_deviation = trace[i].max_gram_deviation;
        s.restarted = trace[i].restarted != 0;
        r.trace.iterations.push_back(s);
    }
    return r;
}

} // namespace detci::gpu
