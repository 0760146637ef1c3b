// run_gpu -- the reference pipeline with the device sigma plugged in
// (what Method::Gpu in run.cpp does).  Built by
// oracle/Makefile against the unmodified reference library; used by
// tests/test_gpu_integration.py.
//
//   run_gpu <fcidump> [<det-list>]
//
// Prints GPU_BUILD (the device build_basis against the reference one) and
// four GROUND_ENERGY lines:
//   reference   davidson_solve over the reference matvec (CPU)
//   mixed       the reference davidson_solve over the device sigma through
//               detci::LinearOperator (SURVEY.md 7.2.7 "mixed oracle")
//   device      the device-resident Davidson (detci_gpu_davidson)
//   gpu_built   the reference davidson_solve over build_basis_gpu's basis
//               (tables and diagonal built on the device)
#include <algorithm>
#include <chrono>
#include <cmath>
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
        const IntegralTable table_copy = table;
        const std::vector<BitString> alpha_copy = alpha, beta_copy = beta;
        auto tb0 = std::chrono::steady_clock::now();
        const Basis basis = build_basis(std::move(alpha), std::move(beta), std::move(table));
        const double t_host = std::chrono::duration<double>(std::chrono::steady_clock::now() - tb0).count();
        tb0 = std::chrono::steady_clock::now();
        gpu::GpuBuiltBasis built = gpu::build_basis_gpu(alpha_copy, beta_copy, table_copy);
        const double t_dev = std::chrono::duration<double>(std::chrono::steady_clock::now() - tb0).count();
        // the device-built host Basis against the reference one: helper lists
        // byte-identical, diagonal within 1e-12
        bool tables_equal = true;
        const FlatExcitationTable* ra[4] = {&basis.singles_a, &basis.doubles_a, &basis.singles_b, &basis.doubles_b};
        const FlatExcitationTable* ga[4] = {&built.host.singles_a, &built.host.doubles_a, &built.host.singles_b,
                                            &built.host.doubles_b};
        for (int i = 0; i < 4; ++i)
            tables_equal = tables_equal && ra[i]->flat == ga[i]->flat && ra[i]->offset == ga[i]->offset &&
                           ra[i]->len == ga[i]->len;
        double diag_worst = 0.0;
        for (std::size_t i = 0; i < basis.diag.size(); ++i)
            diag_worst = std::max(diag_worst, std::abs(basis.diag[i] - built.host.diag[i]) /
                                                  std::max(1.0, std::abs(basis.diag[i])));
        const bool same_shape = built.host.dimension() == basis.dimension() && built.host.norbs == basis.norbs &&
                                built.host.n_elec_alpha == basis.n_elec_alpha &&
                                built.host.channel_packing.bit_length == basis.channel_packing.bit_length &&
                                built.host.det_packing.nwords == basis.det_packing.nwords;
        std::printf("GPU_BUILD tables_equal %d diag_max_rel %.3e shape %d host_s %.4f device_s %.4f\n",
                    tables_equal ? 1 : 0, diag_worst, same_shape ? 1 : 0, t_host, t_dev);
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
        // the reference solver over the GPU-built basis (its diag and sigma)
        const DavidsonResult gbuilt = davidson_solve(gpu::linear_operator(*built.device), built.host.diag);
        std::printf("GROUND_ENERGY reference %.12e %zu\n", ref.energy, ref.trace.iterations.size());
        std::printf("GROUND_ENERGY mixed %.12e %zu\n", mixed.energy, mixed.trace.iterations.size());
        std::printf("GROUND_ENERGY device %.12e %zu\n", device.energy, device.trace.iterations.size());
        std::printf("GROUND_ENERGY gpu_built %.12e %zu\n", gbuilt.energy, gbuilt.trace.iterations.size());
        return ref.converged && mixed.converged && device.converged && gbuilt.converged ? 0 : 2;
    } catch (const Error& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
