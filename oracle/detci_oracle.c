/* CPU restatement of the reference detci sigma path -- see detci_oracle.h.
 *
 * TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Each function names the reference file:line it restates (paths relative to
 * /root/reference/proj/core).  Loop and accumulation orders follow the
 * reference so that, given bit-identical integrals, the sigma vectors here
 * are bit-identical to the reference's (checked in tests/test_oracle.py).
 */
#include "detci_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- interleaved determinant (bitstring.hpp:13-16, bitstring.cpp:109-126) */

typedef struct {
    uint64_t w[2];
} det_t;

static inline int det_bit(const det_t* d, int i) { return (int)((d->w[i >> 6] >> (i & 63)) & 1u); }
static inline void det_set(det_t* d, int i) { d->w[i >> 6] |= (uint64_t)1 << (i & 63); }
static inline void det_clear(det_t* d, int i) { d->w[i >> 6] &= ~((uint64_t)1 << (i & 63)); }

static det_t interleave(uint64_t a, uint64_t b) {
    det_t d = {{0, 0}};
    while (a) {
        det_set(&d, 2 * __builtin_ctzll(a));
        a &= a - 1;
    }
    while (b) {
        det_set(&d, 2 * __builtin_ctzll(b) + 1);
        b &= b - 1;
    }
    return d;
}

/* count_set_between (bitstring.cpp:39-55): set bits strictly between p, q. */
static int count_between(const det_t* d, int p, int q) {
    int lo = (p < q ? p : q) + 1, hi = (p < q ? q : p) - 1, c = 0;
    for (int i = lo; i <= hi; ++i) c += det_bit(d, i);
    return c;
}

/* parity_single_words (bitstring.hpp:111-114). */
static inline int parity_single(const det_t* d, int p, int q) {
    return (count_between(d, p, q) & 1) ? -1 : 1;
}

typedef struct {
    int degree; /* 0, 1, 2 or 3 (= kBeyondDouble) */
    int ann[2], cre[2];
} diff_t;

/* difference_words (bitstring.cpp:70-98). */
static diff_t difference(const det_t* bra, const det_t* ket) {
    diff_t d = {0, {0, 0}, {0, 0}};
    int bits = __builtin_popcountll(bra->w[0] ^ ket->w[0]) + __builtin_popcountll(bra->w[1] ^ ket->w[1]);
    if (bits == 0) return d;
    if (bits > 4 || (bits & 1)) {
        d.degree = 3;
        return d;
    }
    d.degree = bits / 2;
    int na = 0, nc = 0;
    for (int w = 0; w < 2; ++w) {
        uint64_t a = bra->w[w] & ~ket->w[w];
        while (a) {
            if (na == d.degree) { d.degree = 3; return d; }
            d.ann[na++] = 64 * w + __builtin_ctzll(a);
            a &= a - 1;
        }
        uint64_t c = ket->w[w] & ~bra->w[w];
        while (c) {
            if (nc == d.degree) { d.degree = 3; return d; }
            d.cre[nc++] = 64 * w + __builtin_ctzll(c);
            c &= c - 1;
        }
    }
    return d;
}

static inline double eri(const orc_integrals* t, int p, int q, int r, int s) {
    const size_t n = (size_t)t->norbs;
    return t->eri[((p * n + q) * n + r) * n + s];
}

/* zero_excite_words (slater_condon.cpp:23-39) with J/K of
 * build_direct_exchange (integrals.cpp:72-85). */
static double zero_excite(const orc_integrals* t, const det_t* d) {
    int occ[128], n = 0;
    for (int w = 0; w < 2; ++w) {
        uint64_t v = d->w[w];
        while (v) {
            occ[n++] = 64 * w + __builtin_ctzll(v);
            v &= v - 1;
        }
    }
    const int no = t->norbs;
    double value = t->core;
    for (int i = 0; i < n; ++i) {
        const int si = occ[i] >> 1;
        value += t->h1[si * no + si];
        for (int j = i + 1; j < n; ++j) {
            const int sj = occ[j] >> 1;
            value += eri(t, si, si, sj, sj);
            if ((occ[i] & 1) == (occ[j] & 1)) value -= eri(t, si, sj, sj, si);
        }
    }
    return value;
}

/* one_excite_words (slater_condon.cpp:41-66). */
static double one_excite(const orc_integrals* t, const det_t* bra, const det_t* ket, const diff_t* df) {
    const int p = df->ann[0], q = df->cre[0];
    if ((p & 1) != (q & 1)) return 0.0;
    const int ps = p >> 1, qs = q >> 1;
    double value = t->h1[ps * t->norbs + qs];
    for (int w = 0; w < 2; ++w) {
        uint64_t v = ket->w[w];
        while (v) {
            const int r = 64 * w + __builtin_ctzll(v);
            v &= v - 1;
            if (r == p) continue;
            const int rs = r >> 1;
            value += eri(t, ps, qs, rs, rs);
            if ((r & 1) == (p & 1)) value -= eri(t, ps, rs, rs, qs);
        }
    }
    return parity_single(bra, p, q) * value;
}

/* two_excite_words + parity_double_words (slater_condon.cpp:68-94,
 * bitstring.cpp:100-107). */
static double two_excite(const orc_integrals* t, const det_t* bra, const diff_t* df) {
    const int p1 = df->ann[0], p2 = df->ann[1], q1 = df->cre[0], q2 = df->cre[1];
    const int direct_ok = (p1 & 1) == (q1 & 1) && (p2 & 1) == (q2 & 1);
    const int cross_ok = (p1 & 1) == (q2 & 1) && (p2 & 1) == (q1 & 1);
    if (!direct_ok && !cross_ok) return 0.0;
    const int s1 = parity_single(bra, p1, q1);
    det_t mid = *bra;
    det_clear(&mid, p1);
    det_set(&mid, q1);
    const int sign = s1 * parity_single(&mid, p2, q2);
    if (direct_ok) {
        double value = eri(t, p1 >> 1, q1 >> 1, p2 >> 1, q2 >> 1);
        if (cross_ok) value -= eri(t, p1 >> 1, q2 >> 1, p2 >> 1, q1 >> 1);
        return sign * value;
    }
    return -sign * eri(t, p1 >> 1, q2 >> 1, p2 >> 1, q1 >> 1);
}

/* hij_words (slater_condon.cpp:96-105). */
static double hij_det(const orc_integrals* t, const det_t* bra, const det_t* ket) {
    const diff_t df = difference(bra, ket);
    switch (df.degree) {
        case 0: return zero_excite(t, bra);
        case 1: return one_excite(t, bra, ket, &df);
        case 2: return two_excite(t, bra, &df);
        default: return 0.0;
    }
}

double orc_hij(const orc_integrals* t, uint64_t bra_a, uint64_t bra_b, uint64_t ket_a, uint64_t ket_b) {
    const det_t bra = interleave(bra_a, bra_b), ket = interleave(ket_a, ket_b);
    return hij_det(t, &bra, &ket);
}

/* ---- helper lists (connectivity.cpp:26-122) ------------------------------ */

typedef struct {
    uint64_t mask;
    uint32_t idx;
} keyed_t;

static int keyed_cmp(const void* a, const void* b) {
    const keyed_t* x = (const keyed_t*)a;
    const keyed_t* y = (const keyed_t*)b;
    if (x->mask != y->mask) return x->mask < y->mask ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

static int u32_cmp(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y);
}

static int64_t lookup(const keyed_t* idx, uint64_t n, uint64_t mask) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (idx[mid].mask < mask) lo = mid + 1;
        else hi = mid;
    }
    return (lo < n && idx[lo].mask == mask) ? (int64_t)idx[lo].idx : -1;
}

/* Row i: every string j reachable from i by one (kind 0) or two (kind 1)
 * electron moves, ascending -- generate_singles/doubles probe each move
 * against an index (connectivity.cpp:70-84, :94-120) and sort the row. */
int orc_generate_table(const uint64_t* s, uint64_t n, int norbs, int kind, uint32_t* flat,
                       uint64_t* offset, uint32_t* len, uint64_t* nflat) {
    keyed_t* index = (keyed_t*)malloc(sizeof(keyed_t) * (n ? n : 1));
    for (uint64_t i = 0; i < n; ++i) {
        index[i].mask = s[i];
        index[i].idx = (uint32_t)i;
    }
    qsort(index, n, sizeof(keyed_t), keyed_cmp);
    for (uint64_t i = 1; i < n; ++i)
        if (index[i].mask == index[i - 1].mask) {  /* index_strings :36-37 */
            free(index);
            return ORC_E_INPUT;
        }
    const uint64_t full = norbs == 64 ? ~(uint64_t)0 : (((uint64_t)1 << norbs) - 1);
    uint64_t total = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t src = s[i];
        int occ[64], vir[64], no = 0, nv = 0;
        for (int p = 0; p < norbs; ++p) {
            if ((src >> p) & 1u) occ[no++] = p;
            else vir[nv++] = p;
        }
        uint32_t* row = flat ? flat + offset[i] : NULL;
        uint32_t cnt = 0;
        if (kind == 0) {
            for (int a = 0; a < no; ++a)
                for (int c = 0; c < nv; ++c) {
                    const uint64_t probe = (src & ~((uint64_t)1 << occ[a])) | ((uint64_t)1 << vir[c]);
                    const int64_t j = lookup(index, n, probe & full);
                    if (j >= 0) {
                        if (row) row[cnt] = (uint32_t)j;
                        ++cnt;
                    }
                }
        } else {
            for (int a = 0; a < no; ++a)
                for (int b = a + 1; b < no; ++b)
                    for (int c = 0; c < nv; ++c)
                        for (int d = c + 1; d < nv; ++d) {
                            const uint64_t probe = (src & ~(((uint64_t)1 << occ[a]) | ((uint64_t)1 << occ[b]))) |
                                                   ((uint64_t)1 << vir[c]) | ((uint64_t)1 << vir[d]);
                            const int64_t j = lookup(index, n, probe);
                            if (j >= 0) {
                                if (row) row[cnt] = (uint32_t)j;
                                ++cnt;
                            }
                        }
        }
        if (row) qsort(row, cnt, sizeof(uint32_t), u32_cmp);
        if (!flat) {  /* flatten (connectivity.cpp:41-54): offset has size n */
            offset[i] = total;
            len[i] = cnt;
        }
        total += cnt;
    }
    *nflat = total;
    free(index);
    return ORC_OK;
}

/* ---- diagonal (basis.cpp:134-145) ---------------------------------------- */

int orc_diag(const orc_integrals* t, const uint64_t* alpha, uint64_t na, const uint64_t* beta,
             uint64_t nb, double* diag, int threads) {
    if (threads < 1) threads = 1;
    #pragma omp parallel for schedule(static) num_threads(threads)
    for (int64_t ia = 0; ia < (int64_t)na; ++ia)
        for (uint64_t ib = 0; ib < nb; ++ib) {
            const det_t d = interleave(alpha[ia], beta[ib]);
            diag[ia * nb + ib] = zero_excite(t, &d);
        }
    return ORC_OK;
}

/* ---- sigma (matvec.cpp:125-228) ------------------------------------------ */

/* part_alpha + part_beta + part_mixed of one element, in the reference's
 * per-element order: union of singles and doubles ascending (for_each_union,
 * matvec.cpp:21-29), then mixed singles x singles lexicographic. */
static void element_parts(const orc_basis* b, uint64_t ia, uint64_t ib, const double* x,
                          double* pa_out, double* pb_out, double* pm_out) {
    const uint64_t nb = b->nb;
    const det_t bra = interleave(b->alpha[ia], b->beta[ib]);
    double pa = 0.0, pb = 0.0, pm = 0.0;
    {
        const uint32_t* s = b->sa.flat + b->sa.offset[ia];
        const uint32_t* d = b->da.flat + b->da.offset[ia];
        uint32_t ns = b->sa.len[ia], nd = b->da.len[ia], i = 0, j = 0;
        while (i < ns || j < nd) {
            uint32_t ja;
            if (i < ns && (j >= nd || s[i] < d[j])) ja = s[i++];
            else ja = d[j++];
            const det_t ket = interleave(b->alpha[ja], b->beta[ib]);
            pa += hij_det(&b->ints, &bra, &ket) * x[ja * nb + ib];
        }
    }
    {
        const uint32_t* s = b->sb.flat + b->sb.offset[ib];
        const uint32_t* d = b->db.flat + b->db.offset[ib];
        uint32_t ns = b->sb.len[ib], nd = b->db.len[ib], i = 0, j = 0;
        while (i < ns || j < nd) {
            uint32_t jb;
            if (i < ns && (j >= nd || s[i] < d[j])) jb = s[i++];
            else jb = d[j++];
            const det_t ket = interleave(b->alpha[ia], b->beta[jb]);
            pb += hij_det(&b->ints, &bra, &ket) * x[ia * nb + jb];
        }
    }
    {
        const uint32_t* s = b->sa.flat + b->sa.offset[ia];
        const uint32_t* t = b->sb.flat + b->sb.offset[ib];
        for (uint32_t i = 0; i < b->sa.len[ia]; ++i) {
            const uint32_t ja = s[i];
            const double* xrow = x + (uint64_t)ja * nb;
            for (uint32_t j = 0; j < b->sb.len[ib]; ++j) {
                const det_t ket = interleave(b->alpha[ja], b->beta[t[j]]);
                pm += hij_det(&b->ints, &bra, &ket) * xrow[t[j]];
            }
        }
    }
    *pa_out = pa;
    *pb_out = pb;
    *pm_out = pm;
}

int orc_matvec(const orc_basis* b, const double* x, double* y, int threads) {
    if (threads < 1) threads = 1;
    const uint64_t nb = b->nb;
    #pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
    for (int64_t ia = 0; ia < (int64_t)b->na; ++ia)
        for (uint64_t ib = 0; ib < nb; ++ib) {
            double pa, pb, pm;
            element_parts(b, (uint64_t)ia, ib, x, &pa, &pb, &pm);
            const uint64_t I = (uint64_t)ia * nb + ib;
            y[I] = b->diag[I] * x[I] + pa + pb + pm;  /* combine :224-227 */
        }
    return ORC_OK;
}

int orc_matvec_rows(const orc_basis* b, const uint64_t* rows, uint64_t nrows, const double* x,
                    double* y_rows, int threads) {
    if (threads < 1) threads = 1;
    const uint64_t nb = b->nb;
    #pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
    for (int64_t k = 0; k < (int64_t)nrows; ++k) {
        const uint64_t ia = rows[k];
        for (uint64_t ib = 0; ib < nb; ++ib) {
            double pa, pb, pm;
            element_parts(b, ia, ib, x, &pa, &pb, &pm);
            const uint64_t I = ia * nb + ib;
            y_rows[(uint64_t)k * nb + ib] = b->diag[I] * x[I] + pa + pb + pm;
        }
    }
    return ORC_OK;
}

/* ---- Davidson (davidson.cpp:34-206) -------------------------------------- */

double orc_inner_product(const double* x, const double* y, uint64_t n) {
    double acc = 0.0;
    for (uint64_t i = 0; i < n; ++i) acc += x[i] * y[i];
    return acc;
}

int orc_orthonormalize(const double* vs, int k, uint64_t n, const double* candidate, double* out) {
    memcpy(out, candidate, n * sizeof(double));
    for (int pass = 0; pass < 2; ++pass)
        for (int j = 0; j < k; ++j) {
            const double* bv = vs + (uint64_t)j * n;
            const double overlap = orc_inner_product(bv, out, n);
            for (uint64_t i = 0; i < n; ++i) out[i] -= overlap * bv[i];
        }
    const double norm = sqrt(orc_inner_product(out, out, n));
    if (!(norm >= 1e-10)) return 0;
    for (uint64_t i = 0; i < n; ++i) out[i] /= norm;
    return 1;
}

void orc_precondition(const double* r, const double* diag, uint64_t n, double theta, double* out) {
    for (uint64_t i = 0; i < n; ++i) {
        double denom = diag[i] - theta;
        if (fabs(denom) < 1e-8) denom = copysign(1e-8, denom);
        out[i] = r[i] / denom;
    }
}

/* Smallest eigenpair of the k x k symmetric matrix whose lower triangle is
 * g[i*ld + j], j <= i (davidson.cpp:22-30 uses only that triangle).  Cyclic
 * Jacobi; eigenvector sign is arbitrary, as with Eigen. */
static void smallest_eigenpair(const double* g, int ld, int k, double* theta, double* vec) {
    double a[64 * 64], v[64 * 64];
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) {
            a[i * k + j] = i >= j ? g[i * ld + j] : g[j * ld + i];
            v[i * k + j] = i == j ? 1.0 : 0.0;
        }
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, tot = 0.0;
        for (int i = 0; i < k; ++i)
            for (int j = 0; j < k; ++j) {
                tot += a[i * k + j] * a[i * k + j];
                if (i != j) off += a[i * k + j] * a[i * k + j];
            }
        if (off <= 1e-30 * tot || off == 0.0) break;
        for (int p = 0; p < k; ++p)
            for (int q = p + 1; q < k; ++q) {
                const double apq = a[p * k + q];
                if (apq == 0.0) continue;
                const double tau = (a[q * k + q] - a[p * k + p]) / (2.0 * apq);
                const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
                for (int r = 0; r < k; ++r) {
                    const double arp = a[r * k + p], arq = a[r * k + q];
                    a[r * k + p] = c * arp - s * arq;
                    a[r * k + q] = s * arp + c * arq;
                }
                for (int r = 0; r < k; ++r) {
                    const double apr = a[p * k + r], aqr = a[q * k + r];
                    a[p * k + r] = c * apr - s * aqr;
                    a[q * k + r] = s * apr + c * aqr;
                }
                for (int r = 0; r < k; ++r) {
                    const double vrp = v[r * k + p], vrq = v[r * k + q];
                    v[r * k + p] = c * vrp - s * vrq;
                    v[r * k + q] = s * vrp + c * vrq;
                }
            }
    }
    int m = 0;
    for (int i = 1; i < k; ++i)
        if (a[i * k + i] < a[m * k + m]) m = i;
    *theta = a[m * k + m];
    for (int i = 0; i < k; ++i) vec[i] = v[i * k + m];
}

int orc_davidson(const orc_basis* b, double tol, int max_iter, int max_subspace, int threads,
                 double* energy, int* iterations, int* status, double* eigenvector,
                 double* trace, int trace_cap) {
    const uint64_t n = b->na * b->nb;
    if (n == 0) return ORC_E_INPUT;
    if (!(tol > 0.0) || max_subspace < 2 || max_iter < 1) return ORC_E_CONFIG;
    if (max_subspace > 64) return ORC_E_CONFIG;

    double* V = (double*)calloc((size_t)max_subspace * n, sizeof(double)); /* subspace */
    double* W = (double*)calloc((size_t)max_subspace * n, sizeof(double)); /* images */
    double* ritz = (double*)calloc(n, sizeof(double));
    double* ritz_img = (double*)calloc(n, sizeof(double));
    double* res = (double*)calloc(n, sizeof(double));
    double* corr = (double*)calloc(n, sizeof(double));
    double* cand = (double*)calloc(n, sizeof(double));
    double proj[64 * 64];
    double coeffs[64];

    uint64_t argmin = 0; /* davidson.cpp:91-97: lowest index wins ties */
    for (uint64_t i = 1; i < n; ++i)
        if (b->diag[i] < b->diag[argmin]) argmin = i;
    V[argmin] = 1.0;
    int k_sub = 1, k_img = 0, restart_pending = 0, iters = 0, st = 0;
    double theta = 0.0;

    for (int iter = 0; iter < max_iter; ++iter) {
        const int restarted = restart_pending;
        restart_pending = 0;
        while (k_img < k_sub) {
            orc_matvec(b, V + (uint64_t)k_img * n, W + (uint64_t)k_img * n, threads);
            ++k_img;
        }
        const int k = k_sub;
        for (int j = 0; j < k; ++j)
            proj[(k - 1) * max_subspace + j] =
                orc_inner_product(V + (uint64_t)(k - 1) * n, W + (uint64_t)j * n, n);
        smallest_eigenpair(proj, max_subspace, k, &theta, coeffs);

        memset(ritz, 0, n * sizeof(double));
        memset(ritz_img, 0, n * sizeof(double));
        for (int j = 0; j < k; ++j) {
            const double c = coeffs[j];
            const double* vj = V + (uint64_t)j * n;
            const double* wj = W + (uint64_t)j * n;
            for (uint64_t i = 0; i < n; ++i) {
                ritz[i] += c * vj[i];
                ritz_img[i] += c * wj[i];
            }
        }
        for (uint64_t i = 0; i < n; ++i) res[i] = ritz_img[i] - theta * ritz[i];
        const double rnorm = sqrt(orc_inner_product(res, res, n));
        double gdev = 0.0;
        for (int i = 0; i < k; ++i)
            for (int j = 0; j <= i; ++j) {
                const double g = orc_inner_product(V + (uint64_t)i * n, V + (uint64_t)j * n, n);
                const double dv = fabs(g - (i == j ? 1.0 : 0.0));
                if (dv > gdev) gdev = dv;
            }
        if (trace && iters < trace_cap) {
            trace[4 * iters + 0] = theta;
            trace[4 * iters + 1] = rnorm;
            trace[4 * iters + 2] = gdev;
            trace[4 * iters + 3] = restarted;
        }
        ++iters;
        if (rnorm <= tol || iter + 1 == max_iter) {
            st = rnorm <= tol ? 0 : 1;
            break;
        }
        orc_precondition(res, b->diag, n, theta, corr);
        const double cnorm = sqrt(orc_inner_product(corr, corr, n));
        if (!(cnorm > 0.0)) {
            st = 2;
            break;
        }
        for (uint64_t i = 0; i < n; ++i) corr[i] /= cnorm;
        if (k_sub >= max_subspace) {  /* collapse, davidson.cpp:178-184 */
            memcpy(V, ritz, n * sizeof(double));
            memcpy(W, ritz_img, n * sizeof(double));
            k_sub = k_img = 1;
            proj[0] = orc_inner_product(V, W, n);
            restart_pending = 1;
        }
        if (!orc_orthonormalize(V, k_sub, n, corr, cand)) {
            st = 2;
            break;
        }
        memcpy(V + (uint64_t)k_sub * n, cand, n * sizeof(double));
        ++k_sub;
    }
    *energy = theta;
    *iterations = iters;
    *status = st;
    if (eigenvector) {
        const double norm = sqrt(orc_inner_product(ritz, ritz, n));
        for (uint64_t i = 0; i < n; ++i) eigenvector[i] = ritz[i] / norm;
    }
    free(V);
    free(W);
    free(ritz);
    free(ritz_img);
    free(res);
    free(corr);
    free(cand);
    return ORC_OK;
}
