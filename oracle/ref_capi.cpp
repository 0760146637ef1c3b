// extern "C" harness over the UNMODIFIED reference library (detci, compiled
// from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libdetci_ref.so).
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library, and
// only as the checker or the timed CPU baseline -- never on the product path.
//
// Everything here is glue written for this repo: it converts plain arrays to
// the reference's value types and calls the reference's public API
// (parse_fcidump, build_basis, matvec, davidson_solve, dense_hamiltonian,
// hij_words, ...).  The one piece of new logic is ref_matvec_rows, the
// row-sampled sigma harness of SURVEY.md 8(d): it evaluates whole alpha rows
// of sigma with the reference's own hij_words / determinant_words /
// neighbors in the exact contribution order of matvec.cpp:144-227, so every
// sampled row is bit-identical to the corresponding row of the full
// reference product.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include <detci/basis.hpp>
#include <detci/bitstring.hpp>
#include <detci/connectivity.hpp>
#include <detci/davidson.hpp>
#include <detci/detfile.hpp>
#include <detci/integrals.hpp>
#include <detci/matvec.hpp>
#include <detci/oracle.hpp>
#include <detci/slater_condon.hpp>

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace detci;

namespace {

thread_local std::string g_err;

// Status codes shared with include/detci_gpu.h (DETCI_GPU_E_*).
int map_exception() {
    try {
        throw;
    } catch (const InputError& e) {
        g_err = e.what();
        return 2;
    } catch (const FormatError& e) {
        g_err = e.what();
        return 3;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 4;
    } catch (const CapacityError& e) {
        g_err = e.what();
        return 5;
    } catch (const UnsupportedError& e) {
        g_err = e.what();
        return 6;
    } catch (const Error& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 7;
    }
}

#define GUARD(...)                  \
    try {                           \
        __VA_ARGS__;                \
        return 0;                   \
    } catch (...) {                 \
        return map_exception();     \
    }

BitString mask_to_string(std::uint64_t mask, int norbs) {
    std::vector<int> occ;
    for (int i = 0; i < norbs; ++i)
        if ((mask >> i) & 1u) occ.push_back(i);
    return from_occupied(occ, make_packing(norbs, norbs));
}

// `words` uint64 per string, word w = orbitals 64w .. 64w+63 (norbs <= 128)
BitString words_to_string(const std::uint64_t* w, int words, int norbs) {
    std::vector<int> occ;
    for (int i = 0; i < norbs && i < 64 * words; ++i)
        if ((w[i / 64] >> (i % 64)) & 1u) occ.push_back(i);
    return from_occupied(occ, make_packing(norbs, std::min(norbs, 64)));
}

std::uint64_t string_to_mask(const BitString& s) {
    std::uint64_t m = 0;
    for (int i : occupied_list(s)) m |= std::uint64_t{1} << i;
    return m;
}

const FlatExcitationTable& pick_table(const Basis& b, int channel, int kind) {
    if (channel == 0) return kind == 0 ? b.singles_a : b.doubles_a;
    return kind == 0 ? b.singles_b : b.doubles_b;
}

template <class F>
inline void union_ascending(std::span<const std::uint32_t> s, std::span<const std::uint32_t> d,
                            F&& f) {
    std::size_t i = 0, j = 0;
    while (i < s.size() && j < d.size()) f(s[i] < d[j] ? s[i++] : d[j++]);
    while (i < s.size()) f(s[i++]);
    while (j < d.size()) f(d[j++]);
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_max_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// ---- integrals --------------------------------------------------------------

int ref_table_from_fcidump(const char* path, void** out) {
    GUARD({
        std::ifstream in(path);
        if (!in) throw InputError(std::string("cannot open ") + path);
        *out = new IntegralTable(parse_fcidump(in));
    })
}

// eri: dense n^4 chemist-notation array; every 8-fold canonical quadruple is
// stored (the dense synthetic generator of SURVEY.md 8(d)).
int ref_table_from_dense(int norbs, int nelec, int ms2, double core, const double* h1,
                         const double* eri, void** out) {
    GUARD({
        auto t = std::make_unique<IntegralTable>(norbs, nelec, ms2);
        t->set_core_energy(core);
        const std::size_t n = static_cast<std::size_t>(norbs);
        for (int p = 0; p < norbs; ++p)
            for (int q = 0; q <= p; ++q) t->set_one_electron(p, q, h1[p * n + q]);
        for (int p = 0; p < norbs; ++p)
            for (int q = 0; q <= p; ++q)
                for (int r = 0; r <= p; ++r)
                    for (int s = 0; s <= r; ++s) {
                        if (r == p && s > q) continue;
                        t->set_two_electron(p, q, r, s, eri[((p * n + q) * n + r) * n + s]);
                    }
        *out = t.release();
    })
}

void ref_table_free(void* t) { delete static_cast<IntegralTable*>(t); }

int ref_table_info(void* tp, int* norbs, int* nelec, int* ms2, double* core) {
    GUARD({
        const auto* t = static_cast<IntegralTable*>(tp);
        *norbs = t->norbs();
        *nelec = t->n_elec();
        *ms2 = t->ms2();
        *core = t->core_energy();
    })
}

// Dense h (n^2) and ERI (n^4) exactly as the reference resolves them.
int ref_table_dense(void* tp, double* h1, double* eri) {
    GUARD({
        const auto* t = static_cast<IntegralTable*>(tp);
        const int n = t->norbs();
        for (int p = 0; p < n; ++p)
            for (int q = 0; q < n; ++q) h1[p * n + q] = t->one_electron(p, q);
        for (int p = 0; p < n; ++p)
            for (int q = 0; q < n; ++q)
                for (int r = 0; r < n; ++r)
                    for (int s = 0; s < n; ++s)
                        eri[((static_cast<std::size_t>(p) * n + q) * n + r) * n + s] =
                            t->two_electron(p, q, r, s);
    })
}

int ref_write_fcidump(void* tp, const char* path) {
    GUARD({
        std::ofstream out(path);
        write_fcidump(*static_cast<IntegralTable*>(tp), out);
    })
}

// ---- strings ----------------------------------------------------------------

long ref_full_channel_strings(int norbs, int nelec, std::uint64_t* out, long cap) {
    try {
        const auto strings = full_channel_strings(norbs, nelec);
        if (out) {
            const long n = std::min<long>(cap, static_cast<long>(strings.size()));
            for (long i = 0; i < n; ++i) out[i] = string_to_mask(strings[i]);
        }
        return static_cast<long>(strings.size());
    } catch (...) {
        return -map_exception();
    }
}

int ref_channel_electron_counts(int nelec, int ms2, int* na, int* nb) {
    GUARD({
        const auto [a, b] = channel_electron_counts(nelec, ms2);
        *na = a;
        *nb = b;
    })
}

// Parses a determinant list; call with null buffers to get the counts.
int ref_parse_det_list(const char* path, int* norbs, std::uint64_t* alpha, long* na,
                       std::uint64_t* beta, long* nb) {
    GUARD({
        std::ifstream in(path);
        if (!in) throw InputError(std::string("cannot open ") + path);
        const DetList list = parse_det_list(in);
        *norbs = list.norbs;
        if (alpha)
            for (std::size_t i = 0; i < list.alpha.size(); ++i)
                alpha[i] = string_to_mask(list.alpha[i]);
        if (beta)
            for (std::size_t i = 0; i < list.beta.size(); ++i)
                beta[i] = string_to_mask(list.beta[i]);
        *na = static_cast<long>(list.alpha.size());
        *nb = static_cast<long>(list.beta.size());
    })
}

int ref_shuffle_masks(std::uint64_t* masks, long n, int norbs, std::uint64_t seed) {
    GUARD({
        std::vector<BitString> s;
        for (long i = 0; i < n; ++i) s.push_back(mask_to_string(masks[i], norbs));
        shuffle_strings(s, seed);
        for (long i = 0; i < n; ++i) masks[i] = string_to_mask(s[static_cast<std::size_t>(i)]);
    })
}

// Helper lists for a bare string list (reference generate_singles/doubles).
int ref_generate_table(const std::uint64_t* masks, long n, int norbs, int kind,
                       std::uint32_t* flat, std::uint64_t* offset, std::uint32_t* len,
                       std::uint64_t* nflat) {
    GUARD({
        std::vector<BitString> s;
        for (long i = 0; i < n; ++i) s.push_back(mask_to_string(masks[i], norbs));
        const FlatExcitationTable t =
            kind == 0 ? generate_singles(s, norbs) : generate_doubles(s, norbs);
        *nflat = t.flat.size();
        if (flat) std::copy(t.flat.begin(), t.flat.end(), flat);
        if (offset)
            for (std::size_t i = 0; i < t.offset.size(); ++i) offset[i] = t.offset[i];
        if (len) std::copy(t.len.begin(), t.len.end(), len);
    })
}

// ---- basis ------------------------------------------------------------------

int ref_basis_create(void* tp, const std::uint64_t* alpha, long na, const std::uint64_t* beta,
                     long nb, int bit_length, int cache, std::uint64_t budget, int workers,
                     void** out) {
    GUARD({
        const auto* t = static_cast<IntegralTable*>(tp);
        std::vector<BitString> a, b;
        for (long i = 0; i < na; ++i) a.push_back(mask_to_string(alpha[i], t->norbs()));
        for (long i = 0; i < nb; ++i) b.push_back(mask_to_string(beta[i], t->norbs()));
        BasisOptions o;
        o.bit_length = bit_length;
        o.cache = cache != 0;
        o.memory_budget_bytes = budget;
        o.workers = workers;
        *out = new Basis(build_basis(std::move(a), std::move(b), *t, o));
    })
}

// Multi-word variant of ref_basis_create (norbs up to 128 here; the
// reference itself allows kMaxKernelBits = 256 spin-orbitals).
int ref_basis_create_words(void* tp, int words, const std::uint64_t* alpha, long na, const std::uint64_t* beta,
                           long nb, int bit_length, int cache, std::uint64_t budget, int workers, void** out) {
    GUARD({
        const auto* t = static_cast<IntegralTable*>(tp);
        std::vector<BitString> a, b;
        for (long i = 0; i < na; ++i) a.push_back(words_to_string(alpha + i * words, words, t->norbs()));
        for (long i = 0; i < nb; ++i) b.push_back(words_to_string(beta + i * words, words, t->norbs()));
        BasisOptions o;
        o.bit_length = bit_length;
        o.cache = cache != 0;
        o.memory_budget_bytes = budget;
        o.workers = workers;
        *out = new Basis(build_basis(std::move(a), std::move(b), *t, o));
    })
}

void ref_basis_free(void* b) { delete static_cast<Basis*>(b); }

int ref_basis_stats(void* bp, double* stats3, int* det_words) {
    GUARD({
        const auto* b = static_cast<Basis*>(bp);
        stats3[0] = b->stats.connectivity_seconds;
        stats3[1] = b->stats.cache_seconds;
        stats3[2] = b->stats.diag_seconds;
        *det_words = b->det_packing.nwords;
    })
}

int ref_basis_diag(void* bp, double* out) {
    GUARD({
        const auto* b = static_cast<Basis*>(bp);
        std::copy(b->diag.begin(), b->diag.end(), out);
    })
}

int ref_basis_table(void* bp, int channel, int kind, std::uint32_t* flat, std::uint64_t* offset,
                    std::uint32_t* len, std::uint64_t* nflat) {
    GUARD({
        const FlatExcitationTable& t = pick_table(*static_cast<Basis*>(bp), channel, kind);
        *nflat = t.flat.size();
        if (flat) std::copy(t.flat.begin(), t.flat.end(), flat);
        if (offset)
            for (std::size_t i = 0; i < t.offset.size(); ++i) offset[i] = t.offset[i];
        if (len) std::copy(t.len.begin(), t.len.end(), len);
    })
}

// Full reference product; timings4 = {alpha, beta, mixed, combine} seconds.
int ref_matvec(void* bp, int a, int b, int t, int r, const double* x, double* y, int workers,
               double* timings4) {
    GUARD({
        const auto* basis = static_cast<Basis*>(bp);
        const DecompositionPlan plan = plan_decomposition(a, b, t, r, *basis);
        const std::size_t dim = basis->dimension();
        MatvecTimings tm;
        matvec(*basis, plan, std::span<const double>(x, dim), std::span<double>(y, dim), workers,
               &tm);
        if (timings4) {
            timings4[0] = tm.alpha_seconds;
            timings4[1] = tm.beta_seconds;
            timings4[2] = tm.mixed_seconds;
            timings4[3] = tm.combine_seconds;
        }
    })
}

// Row-sampled reference sigma: y_rows[k*nb + ib] = sigma[rows[k], ib], built
// with the reference kernels in the reference contribution order
// (matvec.cpp:152-163 alpha, :176-187 beta, :201-215 mixed, :224-227 combine).
// Parallel over sampled rows; each row is independent.
static void matvec_rows_impl(const Basis& basis, const std::uint64_t* rows, long nrows,
                             const double* x, double* y_rows, int workers) {
    const std::size_t nb = basis.n_beta();
    const std::size_t det_words = static_cast<std::size_t>(basis.det_packing.nwords);
    const IntegralTable& table = basis.integrals;
    const DirectExchange& jk = basis.jk;
    const PackingConfig& cfg = basis.det_packing;
    const int nthreads = resolve_workers(workers);
    #pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (long k = 0; k < nrows; ++k) {
        const std::size_t ia = rows[k];
        std::vector<std::uint64_t> bra(det_words), ket(det_words);
        const auto sa = basis.singles_a.neighbors(ia);
        const auto da = basis.doubles_a.neighbors(ia);
        for (std::size_t ib = 0; ib < nb; ++ib) {
            basis.determinant_words(ia, ib, bra.data());
            double pa = 0.0;
            union_ascending(sa, da, [&](std::uint32_t ja) {
                basis.determinant_words(ja, ib, ket.data());
                pa += hij_words(bra.data(), ket.data(), cfg, table, jk) * x[ja * nb + ib];
            });
            double pb = 0.0;
            union_ascending(basis.singles_b.neighbors(ib), basis.doubles_b.neighbors(ib),
                            [&](std::uint32_t jb) {
                                basis.determinant_words(ia, jb, ket.data());
                                pb += hij_words(bra.data(), ket.data(), cfg, table, jk) *
                                      x[ia * nb + jb];
                            });
            double pm = 0.0;
            const auto sb = basis.singles_b.neighbors(ib);
            for (const std::uint32_t ja : sa) {
                const double* xrow = x + ja * nb;
                for (const std::uint32_t jb : sb) {
                    basis.determinant_words(ja, jb, ket.data());
                    pm += hij_words(bra.data(), ket.data(), cfg, table, jk) * xrow[jb];
                }
            }
            const std::size_t I = ia * nb + ib;
            y_rows[static_cast<std::size_t>(k) * nb + ib] = basis.diag[I] * x[I] + pa + pb + pm;
        }
    }
}

int ref_matvec_rows(void* bp, const std::uint64_t* rows, long nrows, const double* x,
                    double* y_rows, int workers) {
    GUARD(matvec_rows_impl(*static_cast<Basis*>(bp), rows, nrows, x, y_rows, workers))
}

// Reference Davidson over the reference matvec.  trace (may be null) receives
// up to trace_cap rows of {ritz, residual, gram_dev, restarted}.
int ref_davidson(void* bp, double tol, int max_iter, int max_subspace, int workers,
                 double* energy, int* iterations, int* status, double* eigenvector,
                 double* trace, int trace_cap, double* seconds) {
    GUARD({
        const Basis& basis = *static_cast<Basis*>(bp);
        const DecompositionPlan plan = plan_decomposition(1, 1, 1, 1, basis);
        DavidsonOptions o;
        o.tol = tol;
        o.max_iter = max_iter;
        o.max_subspace = max_subspace;
        const auto t0 = std::chrono::steady_clock::now();
        const DavidsonResult res = davidson_solve(
            [&](std::span<const double> x, std::span<double> y) {
                matvec(basis, plan, x, y, workers);
            },
            basis.diag, o);
        if (seconds)
            *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *energy = res.energy;
        *iterations = static_cast<int>(res.trace.iterations.size());
        *status = static_cast<int>(res.status);
        if (eigenvector) std::copy(res.eigenvector.begin(), res.eigenvector.end(), eigenvector);
        if (trace)
            for (int i = 0; i < std::min(trace_cap, *iterations); ++i) {
                const auto& it = res.trace.iterations[static_cast<std::size_t>(i)];
                trace[4 * i + 0] = it.ritz_value;
                trace[4 * i + 1] = it.residual_norm;
                trace[4 * i + 2] = it.max_gram_deviation;
                trace[4 * i + 3] = it.restarted ? 1.0 : 0.0;
            }
    })
}

// Reference Davidson over a caller-supplied operator (the "mixed oracle" of
// reference solver, external sigma).
typedef void (*ref_apply_fn)(const double* x, double* y, std::uint64_t n, void* user);

int ref_davidson_operator(ref_apply_fn apply, void* user, const double* diag, std::uint64_t n,
                          double tol, int max_iter, int max_subspace, double* energy,
                          int* iterations, int* status, double* trace, int trace_cap) {
    GUARD({
        DavidsonOptions o;
        o.tol = tol;
        o.max_iter = max_iter;
        o.max_subspace = max_subspace;
        const DavidsonResult res = davidson_solve(
            [&](std::span<const double> x, std::span<double> y) {
                apply(x.data(), y.data(), n, user);
            },
            std::span<const double>(diag, n), o);
        *energy = res.energy;
        *iterations = static_cast<int>(res.trace.iterations.size());
        *status = static_cast<int>(res.status);
        if (trace)
            for (int i = 0; i < std::min(trace_cap, *iterations); ++i) {
                const auto& it = res.trace.iterations[static_cast<std::size_t>(i)];
                trace[4 * i + 0] = it.ritz_value;
                trace[4 * i + 1] = it.residual_norm;
                trace[4 * i + 2] = it.max_gram_deviation;
                trace[4 * i + 3] = it.restarted ? 1.0 : 0.0;
            }
    })
}

int ref_dense_hamiltonian(void* bp, double* out, std::uint64_t cap) {
    GUARD({
        const DenseHamiltonian d = dense_hamiltonian(*static_cast<Basis*>(bp), cap);
        std::copy(d.values.begin(), d.values.end(), out);
    })
}

// <bra|H|ket> for interleaved determinants built from channel masks, through
// the reference's validated hij (Slater-Condon) at the given bit_length.
int ref_hij(void* tp, std::uint64_t bra_a, std::uint64_t bra_b, std::uint64_t ket_a,
            std::uint64_t ket_b, int bit_length, double* out) {
    GUARD({
        const auto* t = static_cast<IntegralTable*>(tp);
        const int n = t->norbs();
        const int bl = bit_length > 0 ? bit_length : std::min(64, 2 * n);
        const BitString ba = repack(mask_to_string(bra_a, n), bl);
        const BitString bb = repack(mask_to_string(bra_b, n), bl);
        const BitString ka = repack(mask_to_string(ket_a, n), bl);
        const BitString kb = repack(mask_to_string(ket_b, n), bl);
        const DirectExchange jk = build_direct_exchange(*t);
        *out = hij(interleave(ba, bb), interleave(ka, kb), *t, jk);
    })
}

// Oracle element (explicit second quantization, oracle.cpp:70-126).
// ref_hij for strings of `words` uint64 each (norbs <= 128), interleaved at
// bit_length 64 (multi-word determinants).
int ref_hij_words(void* tp, int words, const std::uint64_t* bra_a, const std::uint64_t* bra_b,
                  const std::uint64_t* ket_a, const std::uint64_t* ket_b, double* out) {
    GUARD({
        const auto* t = static_cast<IntegralTable*>(tp);
        const int n = t->norbs();
        const int bl = std::min(64, 2 * n);
        const BitString ba = repack(words_to_string(bra_a, words, n), bl);
        const BitString bb = repack(words_to_string(bra_b, words, n), bl);
        const BitString ka = repack(words_to_string(ket_a, words, n), bl);
        const BitString kb = repack(words_to_string(ket_b, words, n), bl);
        const DirectExchange jk = build_direct_exchange(*t);
        *out = hij(interleave(ba, bb), interleave(ka, kb), *t, jk);
    })
}

int ref_brute_force_hij(void* tp, std::uint64_t bra_a, std::uint64_t bra_b, std::uint64_t ket_a,
                        std::uint64_t ket_b, double* out) {
    GUARD({
        const auto* t = static_cast<IntegralTable*>(tp);
        const int n = t->norbs();
        const int bl = std::min(64, 2 * n);
        const BitString ba = repack(mask_to_string(bra_a, n), bl);
        const BitString bb = repack(mask_to_string(bra_b, n), bl);
        const BitString ka = repack(mask_to_string(ket_a, n), bl);
        const BitString kb = repack(mask_to_string(ket_b, n), bl);
        *out = brute_force_hij(interleave(ba, bb), interleave(ka, kb), *t);
    })
}

// Reference StoredMatrix (build_stored_matrix, matvec.cpp:240-316): build,
// copy out, stored_matvec (matvec.cpp:318-332).
int ref_stored_build(void* bp, std::uint64_t budget, int workers, void** out, std::uint64_t* nnz) {
    GUARD({
        auto* m = new StoredMatrix(build_stored_matrix(*static_cast<Basis*>(bp), budget, workers));
        *nnz = m->nonzero_count();
        *out = m;
    })
}

void ref_stored_free(void* m) { delete static_cast<StoredMatrix*>(m); }

int ref_stored_arrays(void* mp, std::uint64_t* row_offset, std::uint32_t* col, double* value) {
    GUARD({
        const auto* m = static_cast<StoredMatrix*>(mp);
        for (std::size_t i = 0; i < m->row_offset.size(); ++i) row_offset[i] = m->row_offset[i];
        std::copy(m->col.begin(), m->col.end(), col);
        std::copy(m->value.begin(), m->value.end(), value);
    })
}

int ref_stored_matvec(void* mp, const double* x, double* y, int workers) {
    GUARD({
        const auto* m = static_cast<StoredMatrix*>(mp);
        stored_matvec(*m, std::span<const double>(x, m->dimension), std::span<double>(y, m->dimension), workers);
    })
}

} // extern "C"
