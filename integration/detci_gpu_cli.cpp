// detci_gpu -- `detci run` (tools/detci.cpp:44-62, run.cpp:44-125) with the
// device methods: --method gpu | stored, --devices N,
// and a "gpu" block in the JSON report.  The text and JSON reports are the
// reference's own emit_report output (run.cpp:127-242), so tools that parse
// `GROUND_ENERGY` or the JSON schema keep working.  Built by oracle/Makefile
// against the unmodified reference objects (+ run.cpp, which needs
// nlohmann/json) and libdetci_gpu.so.
//
//   detci_gpu run --integrals F --dets D [--method gpu|stored|matrix_free]
//       [--devices N] [--transport nccl|loopback] [--virtual-blocks V]
//       [--balance-rounds R] [--bit-length B] [--shuffle]
//       [--seed S] [--tol T] [--max-iter N] [--max-subspace K]
//       [--memory-budget BYTES] [--workers W] [--format text|json]
//       [--no-timings] [--out PATH]
//
// --method matrix_free runs the reference CPU pipeline unchanged.  gpu: the
// device basis (tables + diagonal in HBM), the device sigma
// and the device Davidson.  stored: the device CSR (build_stored_matrix
// layout) behind the same device Davidson.  --devices N > 1 runs one host
// thread per GPU, each with its own handle and an NCCL communicator over the
// N devices (alpha blocks + C allgather / column-share exchange), cut by R
// (default 2) rounds of the measured rebalance; rank 0 reports.  --transport loopback
// runs the N ranks as threads on ONE GPU over the in-process transport (the
// same rank code, for single-GPU machines).  Exit codes follow the reference
// CLI (tools/detci.cpp:32-34, 59-63): 0 converged, 1 error (message on
// stderr), 2 reported but not converged.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include <nlohmann/json.hpp>

#include <detci/detfile.hpp>
#include <detci/integrals.hpp>
#include <detci/run.hpp>

#include "detci_gpu_shim.hpp"

using namespace detci;

namespace {

double since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

struct GpuConfig {
    std::string method = "gpu";   // gpu | stored | matrix_free
    int devices = 1;
    int virtual_blocks = 1;
    std::string transport = "nccl";   // nccl | loopback
    int balance_rounds = 2;           // measured rebalance rounds (devices > 1)
};

constexpr int kExitOk = 0, kExitError = 1, kExitNotConverged = 2;   // tools/detci.cpp:32-34

struct GpuRun {
    DavidsonResult solved;
    double build_seconds = 0.0, stored_build_seconds = 0.0, solve_seconds = 0.0;
    std::uint64_t nnz_stored = 0;
    std::size_t n_alpha = 0, n_beta = 0;
};

constexpr std::uint64_t kBetaSeedOffset = 0x9e3779b97f4a7c15ULL;   // run.cpp:41

// One rank's pipeline (rank 0 of 1 for a single device).
GpuRun run_rank(const RunConfig& cfg, const GpuConfig& g, int norbs, const std::vector<std::uint64_t>& a,
                const std::vector<std::uint64_t>& b, const IntegralTable& table, int rank,
                const std::uint8_t* nccl_id) {
    GpuRun out;
    gpu::DeviceOptions o;
    const bool loop = g.transport == "loopback";
    o.device = loop ? 0 : rank;
    o.loopback_group = loop && g.devices > 1 ? 1 : 0;
    o.rank = rank;
    o.world_size = g.devices;
    o.nccl_id = nccl_id;
    o.virtual_blocks = g.virtual_blocks;
    o.memory_budget_bytes = 0;
    o.balance_rounds = g.devices > 1 ? g.balance_rounds : 0;
    auto t0 = std::chrono::steady_clock::now();
    gpu::DeviceBasis dev(norbs, a, b, table, o);
    out.build_seconds = since(t0);
    if (g.method == "stored") {
        t0 = std::chrono::steady_clock::now();
        gpu::rethrow(detci_gpu_build_stored(dev.handle(), cfg.memory_budget_bytes, &out.nnz_stored), dev.handle());
        gpu::rethrow(detci_gpu_set_operator(dev.handle(), 1), dev.handle());
        out.stored_build_seconds = since(t0);
    }
    DavidsonOptions opts;
    opts.tol = cfg.tol;
    opts.max_iter = cfg.max_iter;
    opts.max_subspace = cfg.max_subspace;
    t0 = std::chrono::steady_clock::now();
    out.solved = gpu::davidson_solve(dev, opts);
    out.solve_seconds = since(t0);
    return out;
}

std::string usage() {
    return "usage: detci_gpu run --integrals F --dets D [--method gpu|stored|matrix_free] [--devices N]\n"
           "       [--transport nccl|loopback] [--virtual-blocks V] [--balance-rounds R] [--bit-length B]\n"
           "       [--shuffle] [--seed S]\n"
           "       [--tol T] [--max-iter N]\n"
           "       [--max-subspace K] [--memory-budget BYTES] [--workers W] [--format text|json]\n"
           "       [--no-timings] [--out PATH]\n";
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 2 || std::string(argv[1]) != "run") {
        std::fprintf(stderr, "%s", usage().c_str());
        return 1;
    }
    RunConfig cfg;
    GpuConfig g;
    std::string format = "text", out_path;
    try {
        for (int i = 2; i < argc; ++i) {
            const std::string k = argv[i];
            auto val = [&]() -> std::string {
                if (i + 1 >= argc) throw ConfigError("option " + k + " needs a value");
                return argv[++i];
            };
            if (k == "--integrals") cfg.integrals_path = val();
            else if (k == "--dets") cfg.dets_path = val();
            else if (k == "--method") g.method = val();
            else if (k == "--devices") g.devices = std::stoi(val());
            else if (k == "--virtual-blocks") g.virtual_blocks = std::stoi(val());
            else if (k == "--transport") g.transport = val();
            else if (k == "--balance-rounds") g.balance_rounds = std::stoi(val());
            else if (k == "--bit-length") cfg.bit_length = std::stoi(val());
            else if (k == "--shuffle") cfg.shuffle = true;
            else if (k == "--seed") cfg.seed = std::stoull(val());
            else if (k == "--tol") cfg.tol = std::stod(val());
            else if (k == "--max-iter") cfg.max_iter = std::stoi(val());
            else if (k == "--max-subspace") cfg.max_subspace = std::stoi(val());
            else if (k == "--memory-budget") cfg.memory_budget_bytes = std::stoull(val());
            else if (k == "--workers") cfg.workers = std::stoi(val());
            else if (k == "--format") format = val();
            else if (k == "--no-timings") cfg.include_timings = false;
            else if (k == "--out") out_path = val();
            else throw ConfigError("unknown option " + k);
        }
        if (g.method != "gpu" && g.method != "stored" && g.method != "matrix_free")
            throw ConfigError("--method must be gpu, stored or matrix_free");
        if (format != "text" && format != "json") throw ConfigError("--format must be text or json");
        if (g.transport != "nccl" && g.transport != "loopback")
            throw ConfigError("--transport must be nccl or loopback");
        if (g.devices < 1 || g.virtual_blocks < 1) throw ConfigError("--devices and --virtual-blocks must be >= 1");
        if (g.method == "stored" && (g.devices > 1 || g.virtual_blocks > 1))
            throw UnsupportedError("--method stored runs on one GPU");
        const ReportFormat fmt = format == "json" ? ReportFormat::Json : ReportFormat::Text;

        std::string text;
        bool converged = false;
        if (g.method == "matrix_free") {
            cfg.method = Method::MatrixFree;
            const RunReport rep = run_diagonalization(cfg);
            converged = rep.converged;
            text = emit_report(rep, fmt);
        } else {
            cfg.method = g.method == "stored" ? Method::Stored : Method::MatrixFree;
            const auto wall0 = std::chrono::steady_clock::now();
            RunReport report;
            report.config = cfg;
            // inputs as run.cpp:48-67
            auto t0 = std::chrono::steady_clock::now();
            std::ifstream fcidump(cfg.integrals_path);
            if (!fcidump) throw InputError("cannot open integrals file '" + cfg.integrals_path + "'");
            IntegralTable table = parse_fcidump(fcidump);
            std::ifstream dets(cfg.dets_path);
            if (!dets) throw InputError("cannot open determinant list '" + cfg.dets_path + "'");
            DetList list = parse_det_list(dets);
            report.timings.io = since(t0);
            if (list.norbs != table.norbs())
                throw InputError("determinant list norbs " + std::to_string(list.norbs) +
                                 " does not match FCIDUMP NORB " + std::to_string(table.norbs()));
            if (cfg.shuffle) {
                shuffle_strings(list.alpha, cfg.seed);
                shuffle_strings(list.beta, cfg.seed + kBetaSeedOffset);
            }
            const int n = table.norbs();
            if (2 * n > kMaxKernelBits)
                throw InputError("build_basis: " + std::to_string(2 * n) +
                                 " spin-orbitals exceed the kernel limit of " + std::to_string(kMaxKernelBits));
            const auto a = gpu::channel_masks(list.alpha, n);
            const auto b = gpu::channel_masks(list.beta, n);

            std::vector<GpuRun> runs(g.devices);
            if (g.devices == 1) {
                runs[0] = run_rank(cfg, g, n, a, b, table, 0, nullptr);
            } else {
                std::uint8_t id[128] = {};
                if (g.transport == "nccl") gpu::rethrow(detci_gpu_nccl_unique_id(id), nullptr);
                std::vector<std::exception_ptr> errs(g.devices);
                std::vector<std::thread> th;
                for (int r = 0; r < g.devices; ++r)
                    th.emplace_back([&, r] {
                        try {
                            runs[r] = run_rank(cfg, g, n, a, b, table, r, id);
                        } catch (...) {
                            errs[r] = std::current_exception();
                        }
                    });
                for (auto& t : th) t.join();
                for (auto& e : errs)
                    if (e) std::rethrow_exception(e);
            }
            const GpuRun& r0 = runs[0];
            report.dimension = list.alpha.size() * list.beta.size();
            report.n_alpha = list.alpha.size();
            report.n_beta = list.beta.size();
            report.norbs = n;
            report.timings.diag_precompute = r0.build_seconds;   // tables + diagonal, on the device
            report.timings.stored_build = r0.stored_build_seconds;
            report.ground_energy = r0.solved.energy;
            report.iterations = static_cast<int>(r0.solved.trace.iterations.size());
            report.converged = r0.solved.converged;
            converged = report.converged;
            report.status = r0.solved.status;
            report.trace = r0.solved.trace;
            double matvec = 0.0;
            for (const IterationStats& it : report.trace.iterations) {
                report.timings.orthogonalization += it.orthogonalization_seconds;
                report.timings.subspace_solve += it.subspace_solve_seconds;
                matvec += it.matvec_seconds;
            }
            if (g.method == "stored") report.timings.matvec_stored = matvec;
            report.timings.total = since(wall0);
            text = emit_report(report, fmt);
            const std::string label = g.method == "stored" ? "stored (gpu)" : "gpu";
            if (fmt == ReportFormat::Json) {
                nlohmann::json doc = nlohmann::json::parse(text);
                doc["config"]["method"] = g.method == "stored" ? "stored_gpu" : "gpu";
                doc["gpu"] = {
                    {"devices", g.devices},
                    {"virtual_blocks", g.virtual_blocks},
                    {"device_basis_build_seconds", r0.build_seconds},
                    {"stored_nnz", r0.nnz_stored},
                    {"solver_seconds", r0.solve_seconds},
                    {"matvec_seconds", matvec},
                    {"abi_version", detci_gpu_abi_version()},
                };
                text = doc.dump(2) + "\n";
            } else {
                const std::string from = g.method == "stored" ? "  method         stored" : "  method         matrix_free";
                const auto at = text.find(from);
                if (at != std::string::npos)
                    text.replace(at, from.size(), "  method         " + label + " (devices " +
                                                      std::to_string(g.devices) + ")");
                if (cfg.include_timings) {
                    const auto gl = text.find("GROUND_ENERGY");
                    char line[160];
                    std::snprintf(line, sizeof line, "  gpu (s)        basis %.4f, solver %.4f, matvec %.4f\n",
                                  r0.build_seconds, r0.solve_seconds, matvec);
                    text.insert(gl, line);
                }
            }
        }
        if (out_path.empty()) {
            std::fwrite(text.data(), 1, text.size(), stdout);
        } else {
            std::ofstream f(out_path);
            if (!f) throw InputError("cannot write '" + out_path + "'");
            f << text;
        }
        return converged ? kExitOk : kExitNotConverged;   // tools/detci.cpp:59-63
    } catch (const Error& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return kExitError;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return kExitError;
    }
}
