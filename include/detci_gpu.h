/* detci_gpu.h -- C-ABI of the B200-native Davidson sigma build (H*C) for the
 * selected alpha x beta determinant space of detci (arxiv 2601.16169).
 *
 * This is the drop-in boundary: everything above it (CLI, reports, the
 * reference's Davidson API types) is unchanged; a C++ shim
 * (include/detci_gpu.hpp, integration/detci_gpu_shim.hpp) turns it back into
 * the reference's signatures.  Plain pointers and sizes only, no exceptions
 * across the boundary, one handle per host thread, every call synchronous at
 * return.  All citations are relative to /root/reference/proj/core.
 *
 * Reference interfaces each entry point replaces:
 *   detci_gpu_create / _destroy     Basis lifetime (basis.hpp:42-79)
 *   detci_gpu_create_loopback       the same, with the in-process rank
 *                                   transport standing in for the paper's
 *                                   MPI ranks (PAPER.md "Mpi2dSlide") 
 *   detci_gpu_set_strings           Basis::alpha_strings/beta_strings, the
 *                                   prepare_channel checks (basis.cpp:26-47)
 *   detci_gpu_set_integrals         IntegralTable + build_direct_exchange
 *                                   (integrals.hpp:25-72, integrals.cpp:72-85)
 *   detci_gpu_build_basis           build_basis (basis.cpp:78-148): helper
 *                                   lists, diagonal; the det cache is not
 *                                   needed on the device
 *   detci_gpu_get_helpers           Basis::singles_a/doubles_a/singles_b/
 *                                   doubles_b (FlatExcitationTable,
 *                                   connectivity.hpp:24-33)
 *   detci_gpu_diag                  Basis::diag (basis.hpp:74)
 *   detci_gpu_sigma[_device]        matvec (matvec.hpp:64-65) / the
 *                                   LinearOperator apply_h (davidson.hpp:28,
 *                                   run.cpp:96-103)
 *   detci_gpu_davidson              davidson_solve (davidson.hpp:85-86)
 *   detci_gpu_build_stored, _stored_arrays, _set_operator, _release_stored
 *                                   build_stored_matrix / stored_matvec
 *                                   (matvec.hpp:73-90), Method::Stored
 *   detci_gpu_inner_product, _orthonormalize, _precondition
 *                                   davidson.hpp:67-81 vector helpers
 *   detci_gpu_last_error            what() of the detci::Error thrown
 *
 * Status codes map 1:1 onto detci::Error subclasses (error.hpp:12-48).
 */
#ifndef DETCI_GPU_H
#define DETCI_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DETCI_GPU_ABI_VERSION 3

enum detci_gpu_status {
    DETCI_GPU_OK = 0,
    DETCI_GPU_E_ERROR = 1,       /* detci::Error */
    DETCI_GPU_E_INPUT = 2,       /* detci::InputError */
    DETCI_GPU_E_FORMAT = 3,      /* detci::FormatError */
    DETCI_GPU_E_CONFIG = 4,      /* detci::ConfigError */
    DETCI_GPU_E_CAPACITY = 5,    /* detci::CapacityError */
    DETCI_GPU_E_UNSUPPORTED = 6, /* detci::UnsupportedError */
    DETCI_GPU_E_CUDA = 7,        /* CUDA / NCCL runtime failure (detci::Error) */
};

typedef struct detci_gpu_handle detci_gpu_handle;

typedef struct {
    int device;                   /* CUDA ordinal; -1 = LOCAL_RANK-style current device */
    int rank;                     /* this process's rank, 0..world_size-1 */
    int world_size;               /* GPUs (one process each); 1 = single GPU */
    const uint8_t* nccl_id;       /* 128-byte ncclUniqueId (world_size > 1) */
    int virtual_blocks;           /* >1: emulate that many alpha blocks + C ring on
                                     one GPU (tests the multi-GPU schedule) */
    int weighted_partition;       /* 1: alpha blocks balanced by per-row work,
                                     0: reference formula n*i/P (matvec.cpp:108-111) */
    uint64_t memory_budget_bytes; /* 0 = free device memory */
} detci_gpu_desc;

typedef struct {
    /* Mirrors MatvecTimings (matvec.hpp:56-61) plus the GPU split; seconds,
     * measured with CUDA events on the compute stream. */
    double alpha_seconds;     /* alpha-alpha singles+doubles (+ diagonal) */
    double beta_seconds;      /* beta-beta singles+doubles incl. transposes */
    double mixed_seconds;     /* alpha-beta singles x singles */
    double combine_seconds;   /* transpose-add of the beta part */
    double comm_seconds;      /* ring exposure not hidden behind compute */
    double h2d_seconds;       /* host -> device copy of x (host-pointer calls) */
    double d2h_seconds;       /* device -> host copy of y */
    double total_seconds;
    double mixed_reduce_seconds; /* of mixed_seconds: the deterministic D
                                    reductions (k_mixed_reduce) */
} detci_gpu_timings;

typedef struct {
    double tol;         /* residual 2-norm threshold (davidson.hpp:31) */
    int max_iter;
    int max_subspace;
    const double* initial_guess; /* NULL: unit vector at argmin diag; else
                                    local-length host array */
} detci_dav_opts;

typedef struct {
    double ritz_value;
    double residual_norm;
    double matvec_seconds;
    double orthogonalization_seconds;
    double subspace_solve_seconds;
    double max_gram_deviation;
    int restarted;
} detci_dav_iter;

typedef struct {
    int status;      /* 0 Converged, 1 MaxIterationsReached, 2 Stagnated (davidson.hpp:53-57) */
    int converged;
    int iterations;
    double energy;
    double seconds;
    double* eigenvector;     /* optional caller buffer, local length, or NULL */
    detci_dav_iter* trace;   /* optional caller buffer of trace_cap entries */
    int trace_cap;
} detci_dav_result;

/* Multi-root block Davidson (BASELINE config C5).  A
 * capability beyond the reference's single-root davidson_solve
 * (davidson.hpp:83-86), built from the same rules. */
typedef struct {
    double tol;         /* max over roots of the residual 2-norm */
    int max_iter;
    int max_subspace;   /* >= 2 * nroots */
    int nroots;
} detci_dav_block_opts;

typedef struct {
    int status;             /* as detci_dav_result */
    int converged;
    int iterations;
    double seconds;
    double* energies;       /* nroots, ascending, or NULL */
    double* residuals;      /* nroots, or NULL */
    double* eigenvectors;   /* nroots * local length (root-major), or NULL */
    detci_dav_iter* trace;  /* ritz_value = lowest root, residual_norm = max over roots */
    int trace_cap;
} detci_dav_block_result;

/* Called once per Davidson iteration (after the trace entry is final). */
typedef void (*detci_trace_cb)(const detci_dav_iter* it, int iteration, void* user);

/* ---- lifetime ------------------------------------------------------------ */
int detci_gpu_abi_version(void);
int detci_gpu_create(const detci_gpu_desc* desc, detci_gpu_handle** out);
void detci_gpu_destroy(detci_gpu_handle* h);
const char* detci_gpu_last_error(const detci_gpu_handle* h); /* h may be NULL */

/* world_size > 1 without NCCL: the ranks of one loopback group (same
 * `group` id, same world_size) live in ONE process, each handle driven by
 * its own host thread, usually all on one GPU.  They exchange through device
 * copies ordered by CUDA events and a host barrier, and run exactly the
 * multi-rank code paths the NCCL transport runs (sigma schedules, Davidson
 * reductions and argmin).  desc->nccl_id is ignored.  A failing collective
 * call on one rank makes its peers' calls fail (E_ERROR) instead of hang. */
int detci_gpu_create_loopback(const detci_gpu_desc* desc, uint64_t group, detci_gpu_handle** out);

/* 128-byte NCCL unique id for rank 0 to broadcast (torch.distributed). */
int detci_gpu_nccl_unique_id(uint8_t out[128]);

/* ---- inputs ---------------------------------------------------------------
 * Channel strings: one uint64 occupation mask per string, bit p = spatial
 * orbital p (norbs <= 64).  Global lists on every rank.  Errors follow
 * prepare_channel/index_strings: empty list, bits beyond norbs or
 * inconsistent popcounts -> E_INPUT.  Duplicates are reported by
 * detci_gpu_build_basis (as generate_singles does).
 * Replaces Basis::alpha_strings / beta_strings (basis.hpp:40-60) for one-word
 * packings. */
int detci_gpu_set_strings(detci_gpu_handle* h, int norbs, const uint64_t* alpha, size_t na,
                          const uint64_t* beta, size_t nb);

/* The same for norbs <= 128: `words` (1 or 2) consecutive uint64 per string,
 * word w holding orbitals 64w .. 64w+63 (the word order of the reference's
 * BitString, bitstring.hpp:33-51, at bit_length 64).  The reference accepts
 * up to kMaxKernelBits = 256 spin-orbitals (slater_condon.hpp:26,
 * basis.cpp:83-87); norbs > 128 -> E_INPUT.  Systems with norbs > 64 run the
 * scatter mixed kernel only: DETCI_MIXED=gather or 4-vector blocks ->
 * E_UNSUPPORTED. */
int detci_gpu_set_strings_words(detci_gpu_handle* h, int norbs, int words, const uint64_t* alpha,
                                size_t na, const uint64_t* beta, size_t nb);

/* h1: norbs^2 row-major; eri: norbs^4 dense chemist (pq|rs), 8-fold symmetric. */
int detci_gpu_set_integrals(detci_gpu_handle* h, double core, const double* h1,
                            const double* eri);

/* Builds the device basis: string index, helper lists (byte-identical to
 * generate_singles/doubles), pair tables, spectator J tables, the diagonal,
 * and the alpha-block partition.  E_CAPACITY when the device footprint
 * exceeds the budget. */
int detci_gpu_build_basis(detci_gpu_handle* h);

/* ---- parity read-back ----------------------------------------------------- */
/* channel 0 = alpha, 1 = beta; kind 0 = singles, 1 = doubles. */
int detci_gpu_helper_size(const detci_gpu_handle* h, int channel, int kind, uint64_t* nflat);
int detci_gpu_get_helpers(const detci_gpu_handle* h, int channel, int kind, uint32_t* flat,
                          uint64_t* offset, uint32_t* len);

/* This rank's alpha rows [row_begin, row_end); local vectors are
 * (row_end - row_begin) * n_beta doubles, row-major (basis.hpp:10). */
int detci_gpu_local_rows(const detci_gpu_handle* h, uint64_t* row_begin, uint64_t* row_end,
                         uint64_t* n_beta);

/* Off-diagonal structural nonzeros of H (the per-row count of
 * build_stored_matrix minus the diagonal, matvec.cpp:251-260), global. */
int detci_gpu_nnz(const detci_gpu_handle* h, uint64_t* nnz_offdiag, uint64_t* nnz_alpha,
                  uint64_t* nnz_beta, uint64_t* nnz_mixed);

int detci_gpu_diag(const detci_gpu_handle* h, double* out_local);

/* Host-only planning (no GPU): alpha-block boundaries blk[0..P] for P ranks
 * from the helper-list row lengths.  weighted 0 reproduces the reference
 * block formula n_alpha*g/P (matvec.cpp:108-111); 1 balances the per-row
 * element count (len_sa+len_da)*n_beta + sum(len_sb+len_db)
 * + len_sa*sum(len_sb).  E_INPUT when P exceeds n_alpha
 * (plan_decomposition, matvec.cpp:95-96). */
int detci_gpu_plan_partition(uint64_t n_alpha, uint64_t n_beta, const uint32_t* len_sa,
                             const uint32_t* len_da, const uint32_t* len_sb,
                             const uint32_t* len_db, int P, int weighted, uint64_t* blk);

/* ---- sigma ----------------------------------------------------------------- */
/* y = H x over this rank's rows; host pointers (copies inside). */
int detci_gpu_sigma(detci_gpu_handle* h, const double* x_local, double* y_local,
                    detci_gpu_timings* timings);
/* Device pointers (local length), enqueued on the handle's stream and
 * synchronised before return.  x and y must not alias. */
int detci_gpu_sigma_device(detci_gpu_handle* h, const double* dx, double* dy,
                           detci_gpu_timings* timings);
/* Enqueue sigma on the handle's stream without a host synchronisation
 * (back-to-back benchmark steps); pair with detci_gpu_stream + events. */
int detci_gpu_sigma_async(detci_gpu_handle* h, const double* dx, double* dy);
/* The handle's compute stream (a cudaStream_t) so callers can record events
 * on the stream the kernels run on. */
int detci_gpu_stream(const detci_gpu_handle* h, void** stream);
/* Kernels this library has launched in the process so far (all handles). */
int detci_gpu_launch_count(uint64_t* count);
/* Device scratch sized for one local vector (for benchmarks/tests). */
int detci_gpu_alloc_vector(detci_gpu_handle* h, double** dptr);
int detci_gpu_free_vector(detci_gpu_handle* h, double* dptr);
int detci_gpu_copy_vector(detci_gpu_handle* h, double* dst, const double* src, int kind);

/* Shape of the single-GPU sigma plan (diagnostics, bench roofline): the
 * mixed term's scatter pass width K, Cs row segments, ja windows of the D
 * partials (0 before the first sigma), SELL entries incl. padding, and the
 * D buffer size. */
typedef struct {
    int mixed_kmax;
    int mixed_segments;
    int mixed_windows;
    uint64_t mixed_sell_entries;
    uint64_t d_bytes;
    /* per sigma (one vector), from the plan: shared-memory load bytes the
     * scatter kernels issue (V and Cs gathers incl. padding), and the D bytes
     * the reductions read (0 before the first sigma) */
    uint64_t mixed_lds_bytes;
    uint64_t d_read_bytes;
} detci_gpu_plan;
int detci_gpu_sigma_plan(const detci_gpu_handle* h, detci_gpu_plan* out);

/* Virtual blocks (desc.virtual_blocks > 1): device seconds of each
 * block-rank's share of the last timed sigma (detci_gpu_sigma_device with
 * timings), i.e. what one rank of a P-GPU run computes, transfers excluded.
 * *count = P (0 when none); up to cap values are written. */
int detci_gpu_rank_seconds(const detci_gpu_handle* h, double* out, int cap, int* count);
/* The same split by phase: out[4 * rank + phase], phases alpha, beta, mixed,
 * combine (count = 4 * P). */
int detci_gpu_rank_phase_seconds(const detci_gpu_handle* h, double* out, int cap, int* count);

/* Measured rebalance (P = world or virtual blocks > 1; collective when
 * world > 1): `rounds` timed sigmas, each followed by a re-cut of the alpha
 * row blocks and of the mixed term's beta-slot column shares from the
 * per-rank phase times (each rank's measured cost per modelled unit).  The
 * local row range changes: call before allocating rank-local vectors or
 * running a solver, and re-query detci_gpu_local_rows.  *max_over_mean
 * (optional) = the slowest rank over the mean rank of the first timed
 * sigma, i.e. before rebalancing. */
int detci_gpu_rebalance(detci_gpu_handle* h, int rounds, double* max_over_mean);

/* ---- Davidson -------------------------------------------------------------- */
int detci_gpu_davidson(detci_gpu_handle* h, const detci_dav_opts* opts, detci_dav_result* res,
                       detci_trace_cb cb, void* user);

int detci_gpu_davidson_roots(detci_gpu_handle* h, const detci_dav_block_opts* opts,
                             detci_dav_block_result* res);

/* m vectors through one blocked sigma: dx[i], dy[i] device pointers of the
 * local length (the multi-root Davidson's new block). */
int detci_gpu_sigma_block(detci_gpu_handle* h, const double* const* dx, double* const* dy, int m);

/* ---- stored-matrix method (Method::Stored) ------------
 * build_stored_matrix (matvec.cpp:240-316): CSR of H in HBM with the
 * reference's row layout -- row I = ia*nb + ib holds the diagonal, the alpha
 * singles u doubles (ascending ja), the beta singles u doubles (ascending
 * jb), then alpha singles x beta singles (ja-major) -- so row_offset and col
 * are identical to the reference StoredMatrix.  Budget: required = nnz*12 +
 * (dim+1)*8 bytes against memory_budget_bytes (0 = free device memory), else
 * DETCI_GPU_E_CAPACITY with the reference message; dim > 2^32-1 is
 * DETCI_GPU_E_CAPACITY too (matvec.cpp:245-246).  Single GPU only.
 * set_operator(h, 1) makes every sigma call (sigma, sigma_device, the
 * Davidson solvers) the stored SpMV (stored_matvec, matvec.cpp:318-332);
 * set_operator(h, 0) returns to the matrix-free sigma. */
int detci_gpu_build_stored(detci_gpu_handle* h, uint64_t memory_budget_bytes, uint64_t* nnz);
int detci_gpu_stored_arrays(const detci_gpu_handle* h, uint64_t* row_offset /* dim+1 */,
                            uint32_t* col /* nnz */, double* value /* nnz */);
int detci_gpu_set_operator(detci_gpu_handle* h, int kind);   /* 0 matrix-free, 1 stored */
int detci_gpu_release_stored(detci_gpu_handle* h);

/* davidson.hpp:67-81 helpers on host arrays of length n (single GPU). */
int detci_gpu_inner_product(detci_gpu_handle* h, const double* x, const double* y, uint64_t n,
                            double* out);
/* vs: k row-major vectors; returns 1 in *accepted, 0 on linear dependence. */
int detci_gpu_orthonormalize(detci_gpu_handle* h, const double* vs, int k, uint64_t n,
                             const double* candidate, double* out, int* accepted);
int detci_gpu_precondition(detci_gpu_handle* h, const double* residual, const double* diag,
                           uint64_t n, double theta, double* out);

/* ---- diagnostics (host only, no GPU needed) ------------------------------- */
/* <bra|H|ket> assembled from the factorized per-channel closed forms the
 * sigma kernels use (pair value x spectator sign, mixed W table); lets the
 * phase convention be checked against the reference hij on the CPU. */
int detci_gpu_factorized_element(int norbs, double core, const double* h1, const double* eri,
                                 uint64_t bra_alpha, uint64_t bra_beta, uint64_t ket_alpha,
                                 uint64_t ket_beta, double* out);

/* The same for strings of `words` (1 or 2) uint64 each (norbs <= 128, word
 * order as detci_gpu_set_strings_words). */
int detci_gpu_factorized_element_words(int norbs, int words, double core, const double* h1,
                                       const double* eri, const uint64_t* bra_alpha,
                                       const uint64_t* bra_beta, const uint64_t* ket_alpha,
                                       const uint64_t* ket_beta, double* out);

#ifdef __cplusplus
}
#endif

#endif /* DETCI_GPU_H */
