// run_gpu -- the reference pipeline with the device sigma plugged in
// (what Method::Gpu in run.cpp does).  Built by
// oracle/Makefile against the unmodified reference library; used by
// tests/test_gpu_integration.py.
//
//   run_gpu <fcidump> [<det-list>]
//
// Prints three GROUND_ENERGY lines:
//   reference   davidson_solve over the reference matvec (CPU)
//   mixed       the reference davidson_solve over the device sigma through
//               detci::LinearOperator (SURVEY.md 7.2.7 "mixed oracle")
//   device      the device-resident Davidson (detci_gpu_davidson)
#include <chrono>
#include <cstdio>
#include <fstream>
#include <random>
#include <string>

#include <detci/basis.hpp>
#include <detci/davidson.hpp>
#include <detci/detfile.hpp>
#include <detci/integrals.hpp>
#include <detci/matvec.hpp>
#include <detci/oracle.hpp>

#include "detci_gpu_shim.hpp"

using namespace detci;

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: run_gpu <fcidump> [<det-list>]\n");
        return 1;
    }
    try {
        std::ifstream fin(argv[1]);
        IntegralTable table = parse_fcidump(fin);
        std::vector<BitString> alpha, beta;
        if (argc > 2) {
            std::ifstream din(argv[2]);
            DetList list = parse_det_list(din);
            alpha = std::move(list.alpha);
            beta = std::move(list.beta);
        } else {
            const auto [na, nb] = channel_electron_counts(table.n_elec(), table.ms2());
            alpha = full_channel_strings(table.norbs(), na);
            beta = full_channel_strings(table.norbs(), nb);
        }
        const Basis basis = build_basis(std::move(alpha), std::move(beta), std::move(table));
        const DecompositionPlan plan = plan_decomposition(1, 1, 1, 1, basis);
        const auto dev = gpu::build_basis_gpu(basis);

        // sigma parity on a random vector
        std::vector<double> x(basis.dimension()), y_ref(basis.dimension()), y_gpu(basis.dimension());
        std::mt19937_64 rng(11);
        std::uniform_real_distribution<double> u(-1.0, 1.0);
        for (double& v : x) v = u(rng);
        matvec(basis, plan, x, y_ref);
        gpu::matvec(*dev, x, y_gpu);
        double worst = 0.0;
        for (std::size_t i = 0; i < x.size(); ++i)
            worst = std::max(worst, std::abs(y_ref[i] - y_gpu[i]) /
                                        std::max({1.0, std::abs(y_ref[i]), std::abs(y_gpu[i])}));
        std::printf("SIGMA_MAX_REL_DIFF %.3e\n", worst);

        const DavidsonResult ref = davidson_solve(
            [&](std::span<const double> in, std::span<double> out) { matvec(basis, plan, in, out); }, basis.diag);
        const DavidsonResult mixed = davidson_solve(gpu::linear_operator(*dev), basis.diag);
        const DavidsonResult device = gpu::davidson_solve(*dev);
        std::printf("GROUND_ENERGY reference %.12e %zu\n", ref.energy, ref.trace.iterations.size());
        std::printf("GROUND_ENERGY mixed %.12e %zu\n", mixed.energy, mixed.trace.iterations.size());
        std::printf("GROUND_ENERGY device %.12e %zu\n", device.energy, device.trace.iterations.size());
        return ref.converged && mixed.converged && device.converged ? 0 : 2;
    } catch (const Error& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
