/* CPU restatement of the reference detci sigma path (C11).
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load oracle/_ref/libdetci_oracle.so.  The product path
 * (paper_2601_16169_b200/, libdetci_gpu.so) never links or calls it.
 *
 * Parity pinned: every function below is checked in tests/test_oracle.py
 * against the reference library compiled from /root/reference
 * (oracle/_ref/libdetci_ref.so) and against the committed golden vectors in
 * tests/golden/ (generated from that library by tests/golden/make_golden.py),
 * including the shipped chain8 golden E = -2.420193979007e+00
 * (proj/test_output.txt:33).
 *
 * Representation: one uint64 occupation mask per channel string
 * (norbs <= 64); determinants are the interleaved 2*norbs spin-orbital
 * occupation (alpha p -> 2p, beta p -> 2p+1; bitstring.hpp:13-16) held in two
 * 64-bit words.  The reference's results are independent of its packing
 * (test_bitstring.cpp:200-228), so this is the same algorithm.
 */
#ifndef DETCI_ORACLE_H
#define DETCI_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror detci::Error subclasses (error.hpp:12-48). */
enum { ORC_OK = 0, ORC_E_ERROR = 1, ORC_E_INPUT = 2, ORC_E_CONFIG = 4 };

typedef struct {
    int norbs;
    double core;
    const double* h1;  /* norbs^2, symmetric */
    const double* eri; /* norbs^4, chemist (pq|rs), 8-fold symmetric */
} orc_integrals;

typedef struct {
    const uint32_t* flat;
    const uint64_t* offset;
    const uint32_t* len;
} orc_table;

typedef struct {
    orc_integrals ints;
    const uint64_t* alpha;
    uint64_t na;
    const uint64_t* beta;
    uint64_t nb;
    orc_table sa, da, sb, db; /* singles/doubles, alpha/beta */
    const double* diag;
} orc_basis;

/* connectivity.cpp:64-122.  kind 0 = singles, 1 = doubles.  Call with
 * flat == NULL to get len/offset/nflat, then again with flat allocated. */
int orc_generate_table(const uint64_t* strings, uint64_t n, int norbs, int kind, uint32_t* flat,
                       uint64_t* offset, uint32_t* len, uint64_t* nflat);

/* slater_condon.cpp:96-105 on interleaved (alpha, beta) channel masks. */
double orc_hij(const orc_integrals* ints, uint64_t bra_a, uint64_t bra_b, uint64_t ket_a,
               uint64_t ket_b);

/* basis.cpp:134-145: diag[ia*nb+ib] = zero_excite(det(ia, ib)). */
int orc_diag(const orc_integrals* ints, const uint64_t* alpha, uint64_t na, const uint64_t* beta,
             uint64_t nb, double* diag, int threads);

/* matvec.cpp:125-228, same contribution order, y fully overwritten. */
int orc_matvec(const orc_basis* b, const double* x, double* y, int threads);

/* Rows rows[0..nrows) of sigma, y_rows[k*nb + ib]. */
int orc_matvec_rows(const orc_basis* b, const uint64_t* rows, uint64_t nrows, const double* x,
                    double* y_rows, int threads);

/* davidson.cpp:34-71 vector helpers. */
double orc_inner_product(const double* x, const double* y, uint64_t n);
int orc_orthonormalize(const double* vs, int k, uint64_t n, const double* candidate, double* out);
void orc_precondition(const double* residual, const double* diag, uint64_t n, double theta,
                      double* out);

/* davidson.cpp:73-206 over orc_matvec.  trace rows: {ritz, residual,
 * gram_dev, restarted}.  status: 0 converged, 1 max_iter, 2 stagnated
 * (davidson.hpp:53-57). */
int orc_davidson(const orc_basis* b, double tol, int max_iter, int max_subspace, int threads,
                 double* energy, int* iterations, int* status, double* eigenvector,
                 double* trace, int trace_cap);

#ifdef __cplusplus
}
#endif

#endif
