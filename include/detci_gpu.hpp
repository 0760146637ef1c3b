// detci_gpu.hpp -- header-only C++ wrapper over the C-ABI (detci_gpu.h).
//
// RAII handle, exceptions rethrown from status codes with the same class
// names as detci::Error (error.hpp:12-48), and the reference's call shapes:
//   detci_gpu::Basis          ~ detci::Basis + build_basis (basis.hpp:42-90)
//   detci_gpu::matvec         ~ detci::matvec (matvec.hpp:64-65)
//   Basis::linear_operator()  ~ detci::LinearOperator (davidson.hpp:28)
//   detci_gpu::davidson_solve ~ detci::davidson_solve (davidson.hpp:85-86)
// Standalone: does not include the reference headers.  For code inside the
// reference tree use integration/detci_gpu_shim.hpp, which converts
// detci::Basis / IntegralTable and rethrows detci::Error subclasses.
#pragma once

#include <cstdint>
#include <functional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "detci_gpu.h"

namespace detci_gpu {

struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct InputError : Error { using Error::Error; };
struct FormatError : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct CapacityError : Error { using Error::Error; };
struct UnsupportedError : Error { using Error::Error; };
struct CudaError : Error { using Error::Error; };

inline void check(int code, const detci_gpu_handle* h = nullptr) {
    if (code == DETCI_GPU_OK) return;
    const std::string msg = detci_gpu_last_error(h);
    switch (code) {
        case DETCI_GPU_E_INPUT: throw InputError(msg);
        case DETCI_GPU_E_FORMAT: throw FormatError(msg);
        case DETCI_GPU_E_CONFIG: throw ConfigError(msg);
        case DETCI_GPU_E_CAPACITY: throw CapacityError(msg);
        case DETCI_GPU_E_UNSUPPORTED: throw UnsupportedError(msg);
        case DETCI_GPU_E_CUDA: throw CudaError(msg);
        default: throw Error(msg);
    }
}

struct Integrals {
    int norbs = 0;
    double core = 0.0;
    std::vector<double> h1;   // norbs^2
    std::vector<double> eri;  // norbs^4, chemist (pq|rs)
};

struct Options {
    int device = 0, rank = 0, world_size = 1, virtual_blocks = 1;
    bool weighted_partition = false;
    const uint8_t* nccl_id = nullptr;
    uint64_t memory_budget_bytes = 0;
};

class Basis {
public:
    Basis(const std::vector<uint64_t>& alpha, const std::vector<uint64_t>& beta, const Integrals& ints,
          const Options& o = {}) {
        detci_gpu_desc d{o.device, o.rank, o.world_size, o.nccl_id, o.virtual_blocks,
                         o.weighted_partition ? 1 : 0, o.memory_budget_bytes};
        check(detci_gpu_create(&d, &h_));
        try {
            check(detci_gpu_set_strings(h_, ints.norbs, alpha.data(), alpha.size(), beta.data(), beta.size()), h_);
            check(detci_gpu_set_integrals(h_, ints.core, ints.h1.data(), ints.eri.data()), h_);
            check(detci_gpu_build_basis(h_), h_);
            uint64_t nbeta = 0;
            check(detci_gpu_local_rows(h_, &row_begin_, &row_end_, &nbeta), h_);
            local_dim_ = (row_end_ - row_begin_) * nbeta;
        } catch (...) {
            detci_gpu_destroy(h_);
            throw;
        }
    }
    Basis(const Basis&) = delete;
    Basis& operator=(const Basis&) = delete;
    ~Basis() { detci_gpu_destroy(h_); }

    detci_gpu_handle* handle() const { return h_; }
    std::size_t local_dimension() const { return local_dim_; }
    uint64_t row_begin() const { return row_begin_; }
    uint64_t row_end() const { return row_end_; }

    std::vector<double> diag() const {
        std::vector<double> d(local_dim_);
        check(detci_gpu_diag(h_, d.data()), h_);
        return d;
    }

    /// y = H x on host spans of the local length.
    std::function<void(std::span<const double>, std::span<double>)> linear_operator() const {
        return [this](std::span<const double> x, std::span<double> y) {
            if (x.size() != local_dim_ || y.size() != local_dim_)
                throw InputError("matvec: vector length does not match basis dimension");
            check(detci_gpu_sigma(h_, x.data(), y.data(), nullptr), h_);
        };
    }

private:
    detci_gpu_handle* h_ = nullptr;
    uint64_t row_begin_ = 0, row_end_ = 0;
    std::size_t local_dim_ = 0;
};

inline void matvec(const Basis& b, std::span<const double> x, std::span<double> y,
                   detci_gpu_timings* timings = nullptr) {
    if (x.size() != b.local_dimension() || y.size() != b.local_dimension())
        throw InputError("matvec: vector length " + std::to_string(x.size()) + " does not match basis dimension " +
                         std::to_string(b.local_dimension()));
    check(detci_gpu_sigma(b.handle(), x.data(), y.data(), timings), b.handle());
}

struct DavidsonOptions {
    double tol = 1e-8;
    int max_iter = 200;
    int max_subspace = 20;
    std::vector<double> initial_guess;
};

struct DavidsonResult {
    int status = 0;  // 0 Converged, 1 MaxIterationsReached, 2 Stagnated
    bool converged = false;
    double energy = 0.0;
    std::vector<double> eigenvector;
    std::vector<detci_dav_iter> trace;
};

inline DavidsonResult davidson_solve(const Basis& b, const DavidsonOptions& o = {}) {
    detci_dav_opts opts{o.tol, o.max_iter, o.max_subspace,
                        o.initial_guess.empty() ? nullptr : o.initial_guess.data()};
    if (!o.initial_guess.empty() && o.initial_guess.size() != b.local_dimension())
        throw InputError("davidson_solve: initial guess length mismatch");
    DavidsonResult r;
    r.eigenvector.resize(b.local_dimension());
    r.trace.resize(static_cast<std::size_t>(o.max_iter > 0 ? o.max_iter : 1));
    detci_dav_result res{};
    res.eigenvector = r.eigenvector.data();
    res.trace = r.trace.data();
    res.trace_cap = static_cast<int>(r.trace.size());
    check(detci_gpu_davidson(b.handle(), &opts, &res, nullptr, nullptr), b.handle());
    r.status = res.status;
    r.converged = res.converged != 0;
    r.energy = res.energy;
    r.trace.resize(static_cast<std::size_t>(res.iterations));
    return r;
}

} // namespace detci_gpu
