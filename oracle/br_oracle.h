/*
 * br_oracle.h -- CPU restatement of the boundary-row (BR) eigenvalue-only
 * divide-and-conquer tridiagonal eigensolver of arXiv 2605.26599.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker and the CPU baseline
 * ("port") for bench.py.  It is never linked into, loaded by, or called from
 * the product library (libbrgpu.so); only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may use it.
 *
 * Two arithmetic modes:
 *   ref_arith = 1  -- the reference's own arithmetic: IEEE divisions in the
 *                     secular sums (/root/reference/proj/src/secular.cpp:33-43),
 *                     libm hypot (qrql.cpp:29,35; deflate.cpp:85), normalise
 *                     then dot (secular.cpp:272-286, dense.hpp:48-53).
 *                     Pinned bitwise against the compiled reference blocks
 *                     (oracle/_ref) on eigenvalues.
 *   ref_arith = 0  -- the GPU product's arithmetic specification: one correctly
 *                     rounded reciprocal per pole term, a fixed portable
 *                     hypot, fused multiply-adds in the boundary-row dots.  The
 *                     CUDA kernels are required to reproduce this mode bit for
 *                     bit.
 * and the secular stopping rule of secular.cpp:154-158, either verbatim
 * (patched_stop = 0) or tau-relative (patched_stop = 1).
 */
#ifndef BR_ORACLE_H
#define BR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: identical numbering to include/brgpu.h. */
enum {
    BRO_OK = 0,
    BRO_INVALID_ARGUMENT = 1,
    BRO_NO_CONVERGENCE = 2,
    BRO_BUDGET_EXCEEDED = 3,
    BRO_POLE_HIT = 4,
    BRO_ZERO_DENOMINATOR = 5,
    BRO_MALFORMED_COMPACT_ROOT = 6,
    BRO_DIMENSION_MISMATCH = 7,
    BRO_DOMAIN_ERROR = 8,
    BRO_OUT_OF_MEMORY = 9
};

typedef struct bro_opts {
    int leaf_cutoff;     /* 25 */
    int zhat;            /* 1: Gu-Eisenstat refreshed weights (secular.cpp:288-313) */
    int patched_stop;    /* 1: tau-relative bracket stop */
    int ref_arith;       /* see header comment */
    int threads;         /* OpenMP threads (<=0: runtime default) */
    double tol_scale;    /* deflation tol scale (deflate.hpp:55-56), 1.0 */
} bro_opts;

typedef struct bro_stats {
    int64_t merges;          /* internal nodes merged */
    int64_t sum_k;           /* sum of active ranks K */
    double sum_k2;           /* sum of K^2 */
    int64_t sum_nn;          /* sum of non-negligible poles */
    int64_t rotations;       /* close-pole Givens deflations */
    int64_t evals;           /* secular evaluations (incl. the bracket probe) */
    double pole_terms;       /* sum over evaluations of K */
    double zhat_terms;       /* K^2 summed over non-root merges with zhat */
    double row_terms;        /* K^2 summed over non-root merges */
    int64_t max_k;
    int32_t height;          /* max tree height over blocks */
    int32_t blocks;          /* irreducible blocks */
} bro_stats;

/* Per-merge trace record (level-ordered, offset-ordered). */
typedef struct bro_trace {
    int32_t level;
    int32_t is_root;
    int64_t offset;          /* global row offset */
    int64_t size;
    int64_t nn;              /* non-negligible poles */
    int64_t k;               /* active rank */
    double tol;
    double rho;
} bro_trace;

void bro_default_opts(bro_opts* o);

/* All eigenvalues of T = tridiag(e, d, e), ascending, into w[n].
 * trace (may be NULL) receives up to trace_cap records; *trace_len gets the
 * number of merges (which may exceed trace_cap). */
int bro_eigvals(int64_t n, const double* d, const double* e, double* w,
                const bro_opts* o, bro_stats* st,
                bro_trace* trace, int64_t trace_cap, int64_t* trace_len);

/* batch independent matrices of order n: d[b*n..], e[b*(n-1)..], w[b*n..]. */
int bro_eigvals_batched(int64_t batch, int64_t n, const double* d, const double* e,
                        double* w, const bro_opts* o, bro_stats* st);

/* Values-only implicit QL/QR (the eigenvalues_qrql shape), ascending. */
/* Selected rows (Algorithm 1's sigma): rows is nsel x n, rows[r*n+j] = Q(sel[r], j). */
int bro_eigvals_rows(int64_t n, const double* d, const double* e, double* w, int64_t nsel,
                     const int64_t* sel, double* rows, const bro_opts* o);

int bro_qrql_values(int64_t n, const double* d, const double* e, double* w, int ref_arith);

/* Leaf solve: eigenvalues ascending plus first/last eigenvector rows. */
int bro_leaf_full(int m, const double* d, const double* e, double* lam, double* Q, int ref);
int bro_leaf(int m, const double* d, const double* e, double* lam, double* blo,
             double* bhi, int ref_arith);

/* One secular root j of diag(d) + rho z z^T (d strictly ascending). */
int bro_solve_root(int k, const double* d, const double* z, double rho, int j,
                   int patched_stop, int ref_arith, int* origin, double* tau,
                   int* nevals);

/* Deflation of one merge: returns K; fills d_active/z_active (K), the
 * deflated eigenvalues in walk order (n-K) and the number of rotations. */
int bro_deflate(int n, const double* d, const double* z, double tol_scale, int ref_arith,
                double* d_active, double* z_active, double* deflated, int* k_out,
                int* nrot_out, double* tol_out);

/* Gu-Eisenstat refreshed weights for K roots (origin, tau). */
int bro_refreshed_weights(int k, const double* d, const double* z, const int* origin,
                          const double* tau, int ref_arith, double* zhat);

/* Test hook: record (offset, size, n_left, D[size], z[size]) of every merge --
 * merged child eigenvalues and z = (sign*bhi_L, blo_R) before deflation -- into
 * buf (doubles); NULL disables.  bro_merge_dump_used: doubles written/needed. */
void bro_set_merge_dump(double* buf, int64_t cap);
int64_t bro_merge_dump_used(void);

/* Sturm count: number of eigenvalues of T strictly less than x. */
int64_t bro_sturm_count(int64_t n, const double* d, const double* e, double x);

#ifdef __cplusplus
}
#endif

#endif
