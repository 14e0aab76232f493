/*
 * br_oracle.c -- CPU restatement of the eigenvalue-only boundary-row (BR)
 * divide-and-conquer solver (arXiv 2605.26599, Algorithm 1 at PAPER.md:1766-1784).
 *
 * TEST INFRASTRUCTURE ONLY: parity checker + CPU baseline.  Never linked into
 * the product.  See br_oracle.h for the two arithmetic modes.
 *
 * Reference anchors (all under /root/reference/proj):
 *   validate / inf_norm / blocks   src/tridiagonal.cpp:17-58
 *   split tree, Cuppen cuts        src/merge_tree.cpp:34-92
 *   QL/QR sweeps, leaf             src/qrql.cpp:22-135, 146-346, 348-364, 386-413
 *   z, deflation walk, row replay  src/deflate.cpp:31-140
 *   secular eval / root / delta    src/secular.cpp:26-52, 80-241, 243-270
 *   secular column, dots           src/secular.cpp:272-286, include/br/dense.hpp:48-53
 *   refreshed weights              src/secular.cpp:288-313
 *   BR driver (spec only)
 *
 * Compile with -ffp-contract=off: every expression below is evaluated exactly
 * as written (left to right, one rounding per operation), which is what the
 * CUDA kernels (built with --fmad=false) reproduce.
 */
#include "br_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define U_RND 0x1p-53 /* unit roundoff, kEps in secular.cpp:14 / deflate.cpp:13 */

/* ------------------------------------------------------------------------- */
/* primitives                                                                */
/* ------------------------------------------------------------------------- */

/* Portable hypot used by the GPU arithmetic mode (the product reproduces it). */
static double hyp_port(double a, double b) {
    double x = fabs(a), y = fabs(b);
    double big = x > y ? x : y;
    double small = x > y ? y : x;
    if (small == 0.0) return big;
    double t = small / big;
    return big * sqrt(1.0 + t * t);
}

static inline double hyp(double a, double b, int ref) { return ref ? hypot(a, b) : hyp_port(a, b); }

static inline double sign_of(double a, double b) { return b >= 0 ? fabs(a) : -fabs(a); }

/* qrql.cpp:22-40 */
static void make_givens(double g, double f, double* c, double* s, double* r, int ref) {
    if (f == 0.0) {
        *c = 1.0; *s = 0.0; *r = g;
    } else if (fabs(f) > fabs(g)) {
        double t = g / f;
        double tt = hyp(1.0, t, ref);
        *s = 1.0 / tt;
        *c = t * (*s);
        *r = f * tt;
    } else {
        double t = f / g;
        double tt = hyp(1.0, t, ref);
        *c = 1.0 / tt;
        *s = t * (*c);
        *r = g * tt;
    }
}

/* qrql.cpp:43-122: symmetric 2x2 [[a,b],[b,c]]; rt1 larger magnitude, (cs1,sn1) its vector */
static void eig2x2(double a, double b, double c, double* rt1, double* rt2, double* cs1, double* sn1) {
    double sm = a + c, df = a - c, adf = fabs(df), tb = b + b, ab = fabs(tb);
    double acmx, acmn, rt;
    if (fabs(a) > fabs(c)) { acmx = a; acmn = c; } else { acmx = c; acmn = a; }
    if (adf > ab) rt = adf * sqrt(1.0 + (ab / adf) * (ab / adf));
    else if (adf < ab) rt = ab * sqrt(1.0 + (adf / ab) * (adf / ab));
    else rt = ab * sqrt(2.0);
    if (sm < 0.0) {
        *rt1 = 0.5 * (sm - rt);
        *rt2 = (acmx / *rt1) * acmn - (b / *rt1) * b;
    } else if (sm > 0.0) {
        *rt1 = 0.5 * (sm + rt);
        *rt2 = (acmx / *rt1) * acmn - (b / *rt1) * b;
    } else {
        *rt1 = 0.5 * rt;
        *rt2 = -0.5 * rt;
    }
    int sgn1 = sm < 0.0 ? -1 : 1, sgn2;
    double cs;
    if (df >= 0.0) { cs = df + rt; sgn2 = 1; } else { cs = df - rt; sgn2 = -1; }
    double acs = fabs(cs), c1, s1;
    if (acs > ab) {
        double ct = -tb / cs;
        s1 = 1.0 / sqrt(1.0 + ct * ct);
        c1 = ct * s1;
    } else if (ab == 0.0) {
        c1 = 1.0; s1 = 0.0;
    } else {
        double tn = -cs / tb;
        c1 = 1.0 / sqrt(1.0 + tn * tn);
        s1 = tn * c1;
    }
    if (sgn1 == sgn2) { double tn = c1; c1 = -s1; s1 = tn; }
    *cs1 = c1; *sn1 = s1;
}

/* qrql.cpp:126-135 on up to two tracked rows */
static inline void rot_rows(double* r0, double* r1, int64_t j, double c, double s) {
    if (r0) { double xi = r0[j], xj = r0[j + 1]; r0[j] = c * xi - s * xj; r0[j + 1] = s * xi + c * xj; }
    if (r1) { double xi = r1[j], xj = r1[j + 1]; r1[j] = c * xi - s * xj; r1[j + 1] = s * xi + c * xj; }
}

/* ------------------------------------------------------------------------- */
/* implicit QL/QR sweeps: qrql.cpp:146-346, tracking at most two rows        */
/* ------------------------------------------------------------------------- */
static int steqr(int64_t n, double* d, double* e, double* r0, double* r1, int ref) {
    if (n <= 1) return BRO_OK;
    const double eps2 = U_RND * U_RND;
    const double safmin = DBL_MIN;
    const double ssfmax = sqrt(1.0 / safmin) / 3.0;
    const double ssfmin = sqrt(safmin) / eps2;
    const long nmaxit = (long)n * 30;
    long jtot = 0;
    int64_t l1 = 0;
    while (l1 < n) {
        if (l1 > 0) e[l1 - 1] = 0.0;
        int64_t m = n - 1;
        for (int64_t k = l1; k < n - 1; ++k) {
            double tst = fabs(e[k]);
            if (tst == 0.0) { m = k; break; }
            if (tst <= sqrt(fabs(d[k])) * sqrt(fabs(d[k + 1])) * U_RND) { e[k] = 0.0; m = k; break; }
        }
        int64_t l = l1, lsv = l, lend = m, lendsv = lend;
        l1 = m + 1;
        if (lend == l) continue;
        double anorm = 0.0;
        for (int64_t k = l; k <= lend; ++k) anorm = fmax(anorm, fabs(d[k]));
        for (int64_t k = l; k < lend; ++k) anorm = fmax(anorm, fabs(e[k]));
        int iscale = 0;
        if (anorm == 0.0) continue;
        if (anorm > ssfmax) {
            iscale = 1;
            double f = ssfmax / anorm;
            for (int64_t k = l; k <= lend; ++k) d[k] *= f;
            for (int64_t k = l; k < lend; ++k) e[k] *= f;
        } else if (anorm < ssfmin) {
            iscale = 2;
            double f = ssfmin / anorm;
            for (int64_t k = l; k <= lend; ++k) d[k] *= f;
            for (int64_t k = l; k < lend; ++k) e[k] *= f;
        }
        if (fabs(d[lend]) < fabs(d[l])) { int64_t t = l; l = lend; lend = t; }
        if (lend > l) {
            for (;;) { /* QL */
                int64_t mm = lend;
                for (int64_t k = l; k < lend; ++k) {
                    double tst = e[k] * e[k];
                    if (tst <= eps2 * fabs(d[k]) * fabs(d[k + 1]) + safmin) { mm = k; break; }
                }
                if (mm < lend) e[mm] = 0.0;
                double p = d[l];
                if (mm == l) { ++l; if (l <= lend) continue; break; }
                if (mm == l + 1) {
                    double rt1, rt2, c, s;
                    eig2x2(d[l], e[l], d[l + 1], &rt1, &rt2, &c, &s);
                    rot_rows(r0, r1, l, c, -s);
                    d[l] = rt1; d[l + 1] = rt2; e[l] = 0.0;
                    l += 2;
                    if (l <= lend) continue;
                    break;
                }
                if (jtot == nmaxit) break;
                ++jtot;
                double g = (d[l + 1] - p) / (2.0 * e[l]);
                double r = hyp(g, 1.0, ref);
                g = d[mm] - p + e[l] / (g + sign_of(r, g));
                double s = 1.0, c = 1.0;
                p = 0.0;
                for (int64_t i = mm - 1; i >= l; --i) {
                    double f = s * e[i];
                    double b = c * e[i];
                    make_givens(g, f, &c, &s, &r, ref);
                    if (i != mm - 1) e[i + 1] = r;
                    g = d[i + 1] - p;
                    r = (d[i] - g) * s + 2.0 * c * b;
                    p = s * r;
                    d[i + 1] = g + p;
                    g = c * r - b;
                    rot_rows(r0, r1, i, c, s);
                }
                d[l] -= p;
                e[l] = g;
            }
        } else {
            for (;;) { /* QR */
                int64_t mm = lend;
                for (int64_t k = l; k > lend; --k) {
                    double tst = e[k - 1] * e[k - 1];
                    if (tst <= eps2 * fabs(d[k]) * fabs(d[k - 1]) + safmin) { mm = k; break; }
                }
                if (mm > lend) e[mm - 1] = 0.0;
                double p = d[l];
                if (mm == l) { --l; if (l >= lend) continue; break; }
                if (mm == l - 1) {
                    double rt1, rt2, c, s;
                    eig2x2(d[l - 1], e[l - 1], d[l], &rt1, &rt2, &c, &s);
                    rot_rows(r0, r1, l - 1, c, -s);
                    d[l - 1] = rt1; d[l] = rt2; e[l - 1] = 0.0;
                    l -= 2;
                    if (l >= lend) continue;
                    break;
                }
                if (jtot == nmaxit) break;
                ++jtot;
                double g = (d[l - 1] - p) / (2.0 * e[l - 1]);
                double r = hyp(g, 1.0, ref);
                g = d[mm] - p + e[l - 1] / (g + sign_of(r, g));
                double s = 1.0, c = 1.0;
                p = 0.0;
                for (int64_t i = mm; i < l; ++i) {
                    double f = s * e[i];
                    double b = c * e[i];
                    make_givens(g, f, &c, &s, &r, ref);
                    if (i != mm) e[i - 1] = r;
                    g = d[i] - p;
                    r = (d[i + 1] - g) * s + 2.0 * c * b;
                    p = s * r;
                    d[i] = g + p;
                    g = c * r - b;
                    rot_rows(r0, r1, i, c, -s);
                }
                d[l] -= p;
                e[l - 1] = g;
            }
        }
        if (iscale == 1) {
            double f = anorm / ssfmax;
            for (int64_t k = lsv; k <= lendsv; ++k) d[k] *= f;
            for (int64_t k = lsv; k < lendsv; ++k) e[k] *= f;
        } else if (iscale == 2) {
            double f = anorm / ssfmin;
            for (int64_t k = lsv; k <= lendsv; ++k) d[k] *= f;
            for (int64_t k = lsv; k < lendsv; ++k) e[k] *= f;
        }
        if (jtot >= nmaxit) {
            for (int64_t k = 0; k < n - 1; ++k)
                if (e[k] != 0.0) return BRO_NO_CONVERGENCE;
        }
    }
    return BRO_OK;
}

/* Stable ascending sort (ties by index; qrql.cpp:348-364) of m values with
 * up to two rows permuted alongside.  rank_i = #{j: d_j < d_i} + #{j < i: d_j == d_i}. */
static void stable_sort_rows(int m, double* d, double* r0, double* r1) {
    double td[64], t0[64], t1[64];
    for (int i = 0; i < m; ++i) {
        int rank = 0;
        for (int j = 0; j < m; ++j)
            if (d[j] < d[i] || (j < i && d[j] == d[i])) ++rank;
        td[rank] = d[i];
        if (r0) t0[rank] = r0[i];
        if (r1) t1[rank] = r1[i];
    }
    memcpy(d, td, sizeof(double) * (size_t)m);
    if (r0) memcpy(r0, t0, sizeof(double) * (size_t)m);
    if (r1) memcpy(r1, t1, sizeof(double) * (size_t)m);
}

/* ------------------------------------------------------------------------- */
/* secular equation: secular.cpp:26-52, 80-241                                */
/* ------------------------------------------------------------------------- */
typedef struct { double f, fp, abs_sum, psi; int pole; } ev_t;

static ev_t eval_shifted(int k, const double* d, const double* z, double rho, int org,
                         double tau, int jsplit, int ref) {
    ev_t r = {0.0, 0.0, 0.0, 0.0, 0};
    const double dorg = d[org];
    double sum = 0.0, sum_abs = 0.0, sum_d = 0.0, psi_d = 0.0, psum = 0.0;
    for (int i = 0; i < k; ++i) {
        const double del = (d[i] - dorg) - tau;
        if (del == 0.0) { r.pole = 1; return r; }
        const double zz = z[i] * z[i];
        if (ref) {
            const double term = zz / del;
            const double dterm = term / del;
            sum += term;
            sum_abs += fabs(term);
            sum_d += dterm;
            if (i <= jsplit) { psi_d += dterm; psum = sum; }
        } else {
            /* GPU spec: one reciprocal, t = z^2 r, f' accumulates fma(t, r, .) */
            const double rr = 1.0 / del;
            const double term = zz * rr;
            sum += term;
            sum_d = fma(term, rr, sum_d);
            if (i <= jsplit) { psi_d = sum_d; psum = sum; }
        }
    }
    r.f = 1.0 + rho * sum;
    r.fp = rho * sum_d;
    /* GPU arithmetic: the bracket fixes the term signs (t_i < 0 for i <= j,
     * t_i > 0 for i > j), so sum|t| = sum t - 2 * sum_{i<=j} t. */
    r.abs_sum = ref ? rho * sum_abs : rho * (sum - 2.0 * psum);
    r.psi = rho * psi_d;
    return r;
}

/* ---- 32-way split arithmetic (GPU spec for merges larger than 8192 or of
 * active rank K > 1024): a warp owns one root / pole; lane l
 * accumulates the terms i = l, l+32, ... in increasing order; the 32 partials
 * are combined by the xor butterfly a[l] <- a[l] + a[l ^ off], off = 16..1
 * (every lane ends with the same value; this is lane 0's). */
#define BRO_SPLIT 32
#ifndef BRO_SPLIT_MIN_SIZE
#define BRO_SPLIT_MIN_SIZE 8192
#endif
#define BRO_SPLIT_MIN_K 1024
/* split iff the merge is larger than 8192 or its active rank exceeds 1024 */

static double bfly_add(double* a) {
    double b[BRO_SPLIT];
    for (int off = BRO_SPLIT / 2; off >= 1; off >>= 1) {
        for (int l = 0; l < BRO_SPLIT; ++l) b[l] = a[l] + a[l ^ off];
        memcpy(a, b, sizeof(b));
    }
    return a[0];
}

static double bfly_mul(double* a) {
    double b[BRO_SPLIT];
    for (int off = BRO_SPLIT / 2; off >= 1; off >>= 1) {
        for (int l = 0; l < BRO_SPLIT; ++l) b[l] = a[l] * a[l ^ off];
        memcpy(a, b, sizeof(b));
    }
    return a[0];
}

static ev_t eval_split(int k, const double* d, const double* z, double rho, int org, double tau,
                       int jsplit) {
    ev_t r = {0.0, 0.0, 0.0, 0.0, 0};
    const double dorg = d[org];
    double S[BRO_SPLIT], SD[BRO_SPLIT], PS[BRO_SPLIT], PU[BRO_SPLIT];
    for (int l = 0; l < BRO_SPLIT; ++l) {
        S[l] = 0.0; SD[l] = 0.0; PS[l] = 0.0; PU[l] = 0.0;
        for (int i = l; i < k; i += BRO_SPLIT) {
            const double del = (d[i] - dorg) - tau;
            if (del == 0.0) r.pole = 1;
            const double zz = z[i] * z[i];
            const double rr = 1.0 / del;
            const double t = zz * rr;
            S[l] += t;
            SD[l] = fma(t, rr, SD[l]);
            if (i <= jsplit) { PS[l] = SD[l]; PU[l] = S[l]; }
        }
    }
    if (r.pole) return r;
    const double sum = bfly_add(S), sd = bfly_add(SD), ps = bfly_add(PS), pu = bfly_add(PU);
    r.f = 1.0 + rho * sum;
    r.fp = rho * sd;
    r.abs_sum = rho * (sum - 2.0 * pu);
    r.psi = rho * ps;
    return r;
}

static double zsq_split(int k, const double* z) {
    double S[BRO_SPLIT];
    for (int l = 0; l < BRO_SPLIT; ++l) {
        S[l] = 0.0;
        for (int i = l; i < k; i += BRO_SPLIT) S[l] += z[i] * z[i];
    }
    return bfly_add(S);
}

static int solve_root_impl(int k, const double* d, const double* z, double rho, int j, int patched,
                           int ref, int split, int* origin, double* tau_out, int* nevals);

/* Root in (lo, hi) of A t^2 + B t + C = 0 (stable form), NaN if none. */
static double quad_root_in(double A, double B, double C, double lo, double hi) {
    double t = NAN;
    if (A == 0.0) {
        if (B != 0.0) t = -C / B;
        return (isfinite(t) && t > lo && t < hi) ? t : NAN;
    }
    const double disc = B * B - 4.0 * A * C;
    if (disc >= 0.0) {
        const double sq = sqrt(disc);
        const double q = -0.5 * (B + (B >= 0 ? sq : -sq));
        const double r1 = q / A;
        const double r2 = (q != 0.0) ? C / q : NAN;
        if (isfinite(r1) && r1 > lo && r1 < hi) t = r1;
        else if (isfinite(r2) && r2 > lo && r2 < hi) t = r2;
    }
    return t;
}

int bro_solve_root(int k, const double* d, const double* z, double rho, int j,
                   int patched, int ref, int* origin, double* tau_out, int* nevals) {
    return solve_root_impl(k, d, z, rho, j, patched, ref, 0, origin, tau_out, nevals);
}

/* GPU arithmetic: a bracket on one side of the origin spanning more than a
 * factor 4 is bisected geometrically (sqrt(lo) sqrt(hi), same sign): the
 * iterate reaches the root's scale in O(log log(hi/lo)) evaluations instead of
 * halving its way down (glued Wilkinson roots within 1e-15 of a pole). */
static inline int geo_ok(double lo, double hi) {
    return (lo > 0.0 && hi > 4.0 * lo) || (hi < 0.0 && lo < 4.0 * hi);
}
static inline double geo_mid(double lo, double hi) {
    return lo > 0.0 ? sqrt(lo) * sqrt(hi) : -(sqrt(-lo) * sqrt(-hi));
}

static int solve_root_impl(int k, const double* d, const double* z, double rho, int j, int patched,
                           int ref, int split, int* origin, double* tau_out, int* nevals) {
    int ne = 0;
    if (j < 0 || j >= k) return BRO_INVALID_ARGUMENT;
    if (k == 1) {
        *origin = 0;
        *tau_out = rho * z[0] * z[0];
        if (nevals) *nevals = 0;
        return BRO_OK;
    }
    const int last = (j == k - 1);
    int org;
    double lo, hi, other_gap = 0.0;
    int reuse = 0;
    ev_t mid_ev = {0.0, 0.0, 0.0, 0.0, 0};
    int gmode = 0;
    double gA = 0.0, gB = 0.0, gC = 0.0;
    if (last) {
        double zsq = 0.0;
        if (split) zsq = zsq_split(k, z);
        else for (int i = 0; i < k; ++i) zsq += z[i] * z[i];
        org = k - 1;
        lo = 0.0;
        hi = rho * zsq;
    } else {
        const double gap = d[j + 1] - d[j];
        ev_t mid = split ? eval_split(k, d, z, rho, j, 0.5 * gap, j)
                         : eval_shifted(k, d, z, rho, j, 0.5 * gap, j, ref);
        ++ne;
        if (mid.pole || mid.f > 0.0) {
            org = j; lo = 0.0; hi = gap; other_gap = d[j + 1] - d[j];
        } else {
            org = j + 1; lo = -(d[j + 1] - d[j]); hi = 0.0; other_gap = d[j] - d[j + 1];
        }
        /* GPU arithmetic: the first iterate (the bracket midpoint) is the probe
         * point in either origin; reuse its evaluation (f, f', psi' depend on
         * lambda only) instead of evaluating it again. */
        if (!ref) { reuse = 1; mid_ev = mid; }
        /* GPU arithmetic, dlaed4-style start: when the rest of the secular sum
         * (all poles but j, j+1) varies little over the half bracket
         * (|f'_rest| gap/2 <= |f_rest| at the probe), the first step solves the
         * two-nearest-poles-plus-constant model exactly instead of the lumped
         * two-pole model. */
        if (!ref && !mid.pole) {
            const double tp = 0.5 * gap;
            const double rj = 1.0 / ((d[j] - d[j]) - tp);
            const double rj1 = 1.0 / ((d[j + 1] - d[j]) - tp);
            const double z2j = z[j] * z[j], z2j1 = z[j + 1] * z[j + 1];
            const double tj = z2j * rj, tj1 = z2j1 * rj1;
            const double crest = mid.f - rho * tj - rho * tj1;
            const double fprest = mid.fp - rho * (tj * rj) - rho * (tj1 * rj1);
            if (fabs(fprest) * tp <= fabs(crest)) {
                const double a = rho * z2j, b = rho * z2j1;
                gmode = 1;
                gA = crest;
                if (org == j) { gB = -(crest * gap + a + b); gC = a * gap; }
                else { gB = crest * gap - a - b; gC = -(b * gap); }
            }
        }
    }
    /* GPU arithmetic, dlaed4-style model switch: the interior model is the
     * middle way (psi'/phi' lumped on the two nearest poles, secular.cpp:172-213)
     * or, after a slow step, the fixed-weight model (the origin pole keeps its
     * exact weight worg = rho z_org^2, the rest of f' is lumped on the other
     * pole).  The middle way alone converges linearly when the derivative at the
     * origin comes from other poles of a cluster (glued Wilkinson: up to 46
     * evaluations per root; with the safeguards below at most 19). */
    int swtch = 0, nslow = 0;
    double prevf = 0.0;
    const double worg = rho * (z[org] * z[org]);
    double tau = 0.5 * (lo + hi);
    int converged = 0;
    for (int iter = 0; iter < 400; ++iter) {
        double pole_tau = NAN;
        ev_t ev;
        if (reuse) {
            ev = mid_ev;
            reuse = 0;
        } else {
            ev = split ? eval_split(k, d, z, rho, org, tau, j) : eval_shifted(k, d, z, rho, org, tau, j, ref);
            ++ne;
        }
        if (ev.pole) {
            tau = 0.5 * (lo + hi);
            ev = split ? eval_split(k, d, z, rho, org, tau, j) : eval_shifted(k, d, z, rho, org, tau, j, ref);
            ++ne;
            if (ev.pole) break;
        }
        const double ftol = (double)k * U_RND * (1.0 + ev.abs_sum);
        if (fabs(ev.f) <= ftol) { converged = 1; break; }
        if (ev.f < 0.0) lo = tau; else hi = tau;
        const double lambda_abs = fabs(d[org] + tau);
        const double scale = patched ? fmin(lambda_abs, fabs(tau)) : lambda_abs;
        if (hi - lo <= 4.0 * U_RND * scale) { converged = 1; break; }
        /* GPU arithmetic, slow-step safeguards (a step is slow when f kept its
         * sign and more than a tenth of its magnitude):
         *  - a slow step toggles the interior model (middle way / fixed weight);
         *  - after two slow steps in a row, the origin-pole bound: f = rest +
         *    worg/(-tau) with every term of rest increasing in tau, so an
         *    iterate beyond the root bounds it by worg/rest on the origin side
         *    (halved: safe while the computed rest is within a quarter of its
         *    value, |rest| > 4 ftol), and the step bisects a one-sided bracket
         *    spanning more than a factor 4 geometrically;
         *  - a rejected model step bisects geometrically under the same rule.
         * Thresholds tuned on the eval-count tails (random 2^20: the share of
         * roots needing >= 12 evaluations is unchanged; glued Wilkinson 2^18:
         * max 46 -> 18 evaluations). */
        int slow = 0;
        if (!ref) {
            slow = iter >= 1 && ev.f * prevf > 0.0 && fabs(ev.f) > 0.1 * fabs(prevf);
            nslow = slow ? nslow + 1 : 0;
            if (nslow >= 2) {
                const double rest = ev.f + worg / tau;
                if (tau > 0.0 && ev.f > 0.0 && rest > 4.0 * ftol) {
                    const double q = worg / rest;
                    const double bnd = 0.5 * q;
                    if (bnd > lo && bnd < tau) lo = bnd;
                    pole_tau = q;
                } else if (tau < 0.0 && ev.f < 0.0 && rest < -4.0 * ftol) {
                    const double q = worg / rest;
                    const double bnd = 0.5 * q;
                    if (bnd < hi && bnd > tau) hi = bnd;
                    pole_tau = q;
                }
            }
            if (slow && !last) swtch = !swtch;
            prevf = ev.f;
        }
        double tau_next = NAN;
        /* GPU arithmetic, pole step: after the origin bound applied, a root three
         * orders of magnitude closer to the origin pole than the iterate is taken
         * from the pole-dominant model f ~ rest + worg/(-t) (root worg/rest), not
         * halved towards it geometrically (random 2^17: the slowest root per merge
         * 7.90 -> 7.35 evaluations; eigenvalues within 1e-16 relative) */
        const int pstep = !ref && isfinite(pole_tau) && pole_tau > lo && pole_tau < hi && pole_tau != tau &&
                          fabs(pole_tau) < 1e-3 * fabs(tau);
        const int geo_step = pstep || (nslow >= 2 && geo_ok(lo, hi));
#ifndef BRO_NO_LAST_GUESS
        /* GPU arithmetic, the last root's start (dlaed4's case i = n): its first
         * iterate is the bracket midpoint, often far from the root; the first
         * step solves the model of the two largest poles plus a constant fitted
         * at that point, c + rho z_{k-2}^2/(delta - t) + rho z_{k-1}^2/(-t) = 0
         * (delta = d_{k-2} - d_{k-1}), instead of the one-pole model. */
        if (!ref && last && iter == 0 && k >= 2) {
            const double delta = d[k - 2] - d[k - 1];
            const double a = rho * (z[k - 2] * z[k - 2]), b = rho * (z[k - 1] * z[k - 1]);
            const double ta = a / (delta - tau), tb = b / (-tau);
            const double c = ev.f - ta - tb;
            const double fprest = ev.fp - ta / (delta - tau) - tb / (-tau);
            if (fabs(fprest) * tau <= fabs(c)) {  /* the rest is flat over [0, tau] */
                gmode = 1;
                gA = c;
                gB = -(c * delta + a + b);
                gC = b * delta;
            }
        }
#endif
        if (pstep) {
            tau_next = pole_tau;
        } else if (nslow >= 2 && geo_ok(lo, hi)) {
            tau_next = geo_mid(lo, hi);
        } else
        if (iter == 0 && gmode) {
            tau_next = quad_root_in(gA, gB, gC, lo, hi);
        } else if (iter < 100) {
            const double dl = -tau;
            if (last) {
                const double b = ev.fp * dl * dl;
                const double a = ev.f - ev.fp * dl;
                if (a != 0.0) tau_next = tau + (dl + b / a);
            } else {
                const double d_left = (org == j) ? -tau : other_gap - tau;
                const double d_right = (org == j) ? other_gap - tau : -tau;
                /* middle way: psi' on the left pole, phi' on the right; fixed
                 * weight (swtch): the origin pole's share of f' is its own term
                 * worg/d^2, the rest of f' goes to the other pole */
                double psi_p = ev.psi;
                double phi_p = ev.fp - ev.psi;
                if (swtch) {
                    if (org == j) {
                        psi_p = worg / (d_left * d_left);
                        phi_p = ev.fp - psi_p;
                    } else {
                        phi_p = worg / (d_right * d_right);
                        psi_p = ev.fp - phi_p;
                    }
                }
                const double b = psi_p * d_left * d_left;
                const double c = phi_p * d_right * d_right;
                const double a = ev.f - psi_p * d_left - phi_p * d_right;
                const double qa = a;
                const double qb = -(a * (d_left + d_right) + b + c);
                const double qc = a * d_left * d_right + b * d_right + c * d_left;
                double eta1 = NAN, eta2 = NAN;
                if (qa == 0.0) {
                    if (qb != 0.0) eta1 = -qc / qb;
                } else {
                    const double disc = qb * qb - 4.0 * qa * qc;
                    if (disc >= 0.0) {
                        const double sq = sqrt(disc);
                        const double qq = -0.5 * (qb + (qb >= 0 ? sq : -sq));
                        eta1 = qq / qa;
                        if (qq != 0.0) eta2 = qc / qq;
                    }
                }
                const double cand1 = tau + eta1;
                const double cand2 = tau + eta2;
                const int ok1 = isfinite(cand1) && cand1 > lo && cand1 < hi;
                const int ok2 = isfinite(cand2) && cand2 > lo && cand2 < hi;
                if (ok1 && ok2) tau_next = fabs(eta1) <= fabs(eta2) ? cand1 : cand2;
                else if (ok1) tau_next = cand1;
                else if (ok2) tau_next = cand2;
            }
        }
        const int model_ok = isfinite(tau_next) && tau_next > lo && tau_next < hi && tau_next != tau;
        if (!model_ok)
            tau_next = (!ref && geo_ok(lo, hi)) ? geo_mid(lo, hi) : 0.5 * (lo + hi);
        /* GPU arithmetic, step stop: a model step (not a bisection) of at most
         * 2^-27 |tau_next| ends the iteration at tau_next -- the model converges
         * at least quadratically, so the remaining error is ~2^-54 |tau|; this
         * saves the evaluation that would only confirm |f| <= ftol (random:
         * -9.5% evaluations, Toeplitz -19%, eigenvalues within 2e-14 of the
         * previous rule, accuracy against LAPACK unchanged) */
        if (!ref && model_ok && !geo_step && fabs(tau_next - tau) <= 0x1p-27 * fabs(tau_next)) {
            tau = tau_next;
            converged = 1;
            break;
        }
        tau = tau_next;
    }
    if (nevals) *nevals = ne;
    if (!converged) return BRO_NO_CONVERGENCE;
    *origin = org;
    *tau_out = tau;
    return BRO_OK;
}

/* secular.cpp:288-313 (w *= factor in sequential root order; w starts at 1). */
int bro_refreshed_weights(int k, const double* d, const double* z, const int* origin,
                          const double* tau, int ref, double* zhat) {
    for (int i = 0; i < k; ++i) {
        const double di = d[i];
        double w = 1.0;
        for (int j = 0; j < k; ++j) {
            const double del = (di - d[origin[j]]) - tau[j];
            if (i == j) w *= del;
            else if (ref) w *= del / (di - d[j]);
            else w *= del * (1.0 / (di - d[j]));
        }
        const double mag = sqrt(fmax(0.0, -w));
        zhat[i] = z[i] >= 0.0 ? mag : -mag;
    }
    return BRO_OK;
}

/* One parent boundary-row pair for root (org, tau): secular.cpp:272-286 + dense.hpp:48-53. */
static int root_rows(int k, const double* d, const double* zh, const double* r0, const double* r1,
                     int org, double tau, int ref, int split, double* blo, double* bhi, double* ybuf) {
    const double dorg = d[org];
    if (ref) {
        double norm_sq = 0.0;
        for (int i = 0; i < k; ++i) {
            const double del = (d[i] - dorg) - tau;
            if (del == 0.0) return BRO_ZERO_DENOMINATOR;
            const double y = zh[i] / del;
            ybuf[i] = y;
            norm_sq += y * y;
        }
        const double inv = 1.0 / sqrt(norm_sq);
        double a0 = 0.0, a1 = 0.0;
        for (int i = 0; i < k; ++i) {
            const double y = ybuf[i] * inv;
            a0 += r0[i] * y;
            a1 += r1[i] * y;
        }
        *blo = a0; *bhi = a1;
    } else if (split) {
        double NN[BRO_SPLIT], S0[BRO_SPLIT], S1[BRO_SPLIT];
        for (int l = 0; l < BRO_SPLIT; ++l) {
            NN[l] = 0.0; S0[l] = 0.0; S1[l] = 0.0;
            for (int i = l; i < k; i += BRO_SPLIT) {
                const double del = (d[i] - dorg) - tau;
                if (del == 0.0) return BRO_ZERO_DENOMINATOR;
                const double y = zh[i] * (1.0 / del);
                NN[l] = fma(y, y, NN[l]);
                S0[l] = fma(r0[i], y, S0[l]);
                S1[l] = fma(r1[i], y, S1[l]);
            }
        }
        const double nn = bfly_add(NN), s0 = bfly_add(S0), s1 = bfly_add(S1);
        const double inv = 1.0 / sqrt(nn);
        *blo = s0 * inv; *bhi = s1 * inv;
    } else {
        double nn = 0.0, s0 = 0.0, s1 = 0.0;
        for (int i = 0; i < k; ++i) {
            const double del = (d[i] - dorg) - tau;
            if (del == 0.0) return BRO_ZERO_DENOMINATOR;
            const double y = zh[i] * (1.0 / del);
            nn = fma(y, y, nn);
            s0 = fma(r0[i], y, s0);
            s1 = fma(r1[i], y, s1);
        }
        const double inv = 1.0 / sqrt(nn);
        *blo = s0 * inv; *bhi = s1 * inv;
    }
    return BRO_OK;
}

/* One selected row's entry for root (org, tau): R_parent(i, j) = R_child(i,:) y_j
 * (Algorithm 1, "(Q_v)_sigma = (Q_L + Q_R)_sigma S_v").
 * GPU arithmetic: one sequential pass in pole order, fused multiply-adds for
 * ||y||^2 and the dot product (the non-split root_rows order). */
static int sigma_root_row(int k, const double* d, const double* zh, const double* x, int org,
                          double tau, int ref, double* out) {
    const double dorg = d[org];
    double nn = 0.0, s = 0.0;
    for (int i = 0; i < k; ++i) {
        const double del = (d[i] - dorg) - tau;
        if (del == 0.0) return BRO_ZERO_DENOMINATOR;
        const double y = ref ? zh[i] / del : zh[i] * (1.0 / del);
        if (ref) { nn += y * y; s += x[i] * y; }
        else { nn = fma(y, y, nn); s = fma(x[i], y, s); }
    }
    *out = ref ? s / sqrt(nn) : s * (1.0 / sqrt(nn));
    return BRO_OK;
}

/* ------------------------------------------------------------------------- */
/* deflation: deflate.cpp:43-107 (walk) + 109-140 (row replay, fused)         */
/* ------------------------------------------------------------------------- */
typedef struct {
    int n, K, nn, nrot;
    double tol;
} defl_info;

/* GPU arithmetic of a close-pole group (deflate.cpp:76-95, 109-140 restated):
 * a survivor s absorbs its members k1, k2, ... (consecutive non-negligible
 * poles within tol of d_s) by the rotation chain of the reference.  Composed,
 * the chain is r_i = |(z_s, z_k1, .., z_ki)|, survivor row r_i x_s = sum of
 * z x over the group so far, member row x_k' = c x_k - s x_p with c =
 * r_{i-1}/r_i, s = z_k/r_i, x_p = S_{i-1}/r_{i-1}.  Here it is evaluated from
 * sequential prefix sums Q = sum z^2, S0/S1 = sum z x (one add per member on
 * the dependency chain instead of a hypot + two divisions), so a walk of a
 * glued-Wilkinson cluster (runs of ~10^4) is a cheap prefix pass followed by
 * independent per-member updates.  The survivor's z becomes sqrt(Q) >= 0. */
static void group_member(double Qp, double S0p, double S1p, double zk, double* x0, double* x1) {
    const double Qn = Qp + zk * zk;
    const double rp = sqrt(Qp), R = sqrt(Qn);
    const double irp = 1.0 / rp, iR = 1.0 / R;
    const double c = rp * iR, sn = zk * iR;
    const double xp0 = S0p * irp, xp1 = S1p * irp;
    if (x0) *x0 = c * *x0 - sn * xp0;
    if (x1) *x1 = c * *x1 - sn * xp1;
}

/* D, Z, R0, R1: merged (sorted) order, modified in place by the rotations.
 * act[K]: sorted positions of survivors.  defl[n-K]: sorted positions of the
 * deflated poles in walk order.  R0/R1 may be NULL (root-only merge). */
static void deflate_walk(int n, const double* D, double* Z, double* R0, double* R1, double tol,
                         int ref, int* act, int* defl, defl_info* info, int nx, double* X, double* SX) {
    /* X: nx extra selected rows (stride n, merged order), SX: nx group sums */
    int prev = -1, K = 0, nd = 0, nn = 0, nrot = 0;
    /* GPU arithmetic: running group sums of the current survivor */
    int L = 0;
    double Q = 0.0, S0 = 0.0, S1 = 0.0;
#define GROUP_CLOSE()                                              \
    do {                                                           \
        if (!ref && prev >= 0 && L > 0) {                          \
            const double R_ = sqrt(Q), iR_ = 1.0 / R_;            \
            Z[prev] = R_;                                          \
            if (R0) R0[prev] = S0 * iR_;                           \
            if (R1) R1[prev] = S1 * iR_;                           \
            for (int x_ = 0; x_ < nx; ++x_)                        \
                X[(int64_t)x_ * n + prev] = SX[x_] * iR_;          \
        }                                                          \
    } while (0)
    for (int k = 0; k < n; ++k) {
        if (fabs(Z[k]) <= tol) { defl[nd++] = k; continue; }
        ++nn;
        if (prev >= 0 && fabs(D[k] - D[prev]) <= tol) {
            if (ref) {
                const double zp = Z[prev], zq = Z[k];
                const double r = hyp(zp, zq, ref);
                const double c = zp / r, s = zq / r;
                Z[prev] = r;
                Z[k] = 0.0;
                if (R0) { double xp = R0[prev], xq = R0[k]; R0[prev] = c * xp + s * xq; R0[k] = c * xq - s * xp; }
                if (R1) { double xp = R1[prev], xq = R1[k]; R1[prev] = c * xp + s * xq; R1[k] = c * xq - s * xp; }
                for (int x = 0; x < nx; ++x) {
                    double* Xr = X + (int64_t)x * n;
                    double xp = Xr[prev], xq = Xr[k];
                    Xr[prev] = c * xp + s * xq;
                    Xr[k] = c * xq - s * xp;
                }
            } else {
                const double zk = Z[k];
                const double x0 = R0 ? R0[k] : 0.0, x1 = R1 ? R1[k] : 0.0;
                group_member(Q, S0, S1, zk, R0 ? &R0[k] : NULL, R1 ? &R1[k] : NULL);
                for (int x = 0; x < nx; ++x) {  /* same per-row arithmetic as R0/R1 */
                    double* Xr = X + (int64_t)x * n;
                    const double xk = Xr[k];
                    group_member(Q, SX[x], SX[x], zk, &Xr[k], NULL);
                    SX[x] = SX[x] + zk * xk;
                }
                Q = Q + zk * zk;
                S0 = S0 + zk * x0;
                S1 = S1 + zk * x1;
                Z[k] = 0.0;
                ++L;
            }
            defl[nd++] = k;
            ++nrot;
            continue;
        }
        GROUP_CLOSE();
        prev = k;
        act[K++] = k;
        if (!ref) {
            const double zs = Z[k];
            L = 0;
            Q = zs * zs;
            S0 = R0 ? zs * R0[k] : 0.0;
            S1 = R1 ? zs * R1[k] : 0.0;
            for (int x = 0; x < nx; ++x) SX[x] = zs * X[(int64_t)x * n + k];
        }
    }
    GROUP_CLOSE();
#undef GROUP_CLOSE
    info->n = n; info->K = K; info->nn = nn; info->nrot = nrot; info->tol = tol;
}

int bro_deflate(int n, const double* d, const double* z, double tol_scale, int ref,
                double* d_active, double* z_active, double* deflated, int* k_out,
                int* nrot_out, double* tol_out) {
    /* d, z in child order; stable sort + walk, returns compacted problem. */
    int* perm = (int*)malloc(sizeof(int) * (size_t)n * 3);
    double* D = (double*)malloc(sizeof(double) * (size_t)n * 2);
    if (!perm || !D) { free(perm); free(D); return BRO_OUT_OF_MEMORY; }
    double* Z = D + n;
    int* act = perm + n;
    int* defl = perm + 2 * n;
    double dmax = 0.0, zmax = 0.0;
    for (int i = 0; i < n; ++i) { dmax = fmax(dmax, fabs(d[i])); zmax = fmax(zmax, fabs(z[i])); }
    const double tol = 8.0 * U_RND * fmax(dmax, zmax) * tol_scale;
    /* stable sort by d (insertion-by-rank, O(n^2): small test sizes only) */
    for (int i = 0; i < n; ++i) {
        int rank = 0;
        for (int j = 0; j < n; ++j)
            if (d[j] < d[i] || (j < i && d[j] == d[i])) ++rank;
        perm[rank] = i;
    }
    for (int k = 0; k < n; ++k) { D[k] = d[perm[k]]; Z[k] = z[perm[k]]; }
    defl_info info;
    deflate_walk(n, D, Z, NULL, NULL, tol, ref, act, defl, &info, 0, NULL, NULL);
    for (int a = 0; a < info.K; ++a) { d_active[a] = D[act[a]]; z_active[a] = Z[act[a]]; }
    for (int t = 0; t < n - info.K; ++t) deflated[t] = D[defl[t]];
    *k_out = info.K;
    *nrot_out = info.nrot;
    *tol_out = tol;
    free(perm);
    free(D);
    return BRO_OK;
}

/* ------------------------------------------------------------------------- */
/* leaf + qrql values                                                        */
/* ------------------------------------------------------------------------- */
int bro_leaf(int m, const double* d, const double* e, double* lam, double* blo, double* bhi,
             int ref) {
    double ee[64];
    if (m <= 0 || m > 64) return BRO_INVALID_ARGUMENT;
    memcpy(lam, d, sizeof(double) * (size_t)m);
    if (m > 1) memcpy(ee, e, sizeof(double) * (size_t)(m - 1));
    for (int i = 0; i < m; ++i) { blo[i] = 0.0; bhi[i] = 0.0; }
    blo[0] = 1.0;
    bhi[m - 1] = 1.0;
    int st = steqr(m, lam, ee, blo, bhi, ref);
    if (st) return st;
    stable_sort_rows(m, lam, blo, bhi);
    return BRO_OK;
}

/* Full eigenvector matrix of a leaf (Q[i*m + k] = row i of eigenvector k) by the
 * same QL/QR sweeps, tracking one row per run: the conventional full-eigenvector
 * D&C restatement of the Theorem 1 check (tests/test_theorem1_gpu.py) starts
 * from exactly the leaf vectors whose boundary rows the BR path carries. */
int bro_leaf_full(int m, const double* d, const double* e, double* lam, double* Q, int ref) {
    double ee[64], x[64], l2[64];
    if (m <= 0 || m > 64) return BRO_INVALID_ARGUMENT;
    for (int i = 0; i < m; ++i) {
        memcpy(l2, d, sizeof(double) * (size_t)m);
        if (m > 1) memcpy(ee, e, sizeof(double) * (size_t)(m - 1));
        for (int k = 0; k < m; ++k) x[k] = k == i ? 1.0 : 0.0;
        int st = steqr(m, l2, ee, x, NULL, ref);
        if (st) return st;
        stable_sort_rows(m, l2, x, NULL);
        memcpy(Q + (size_t)i * (size_t)m, x, sizeof(double) * (size_t)m);
        if (i == 0) memcpy(lam, l2, sizeof(double) * (size_t)m);
    }
    return BRO_OK;
}

static int cmp_double(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x < y) ? -1 : (y < x) ? 1 : 0;
}

/* stable merge sort (ascending by '<') */
static void stable_sort_values(int64_t n, double* a, double* tmp) {
    for (int64_t w = 1; w < n; w *= 2) {
        for (int64_t lo = 0; lo < n; lo += 2 * w) {
            int64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
            int64_t i = lo, j = mid, k = lo;
            while (i < mid && j < hi) tmp[k++] = (a[j] < a[i]) ? a[j++] : a[i++];
            while (i < mid) tmp[k++] = a[i++];
            while (j < hi) tmp[k++] = a[j++];
        }
        memcpy(a, tmp, sizeof(double) * (size_t)n);
    }
}

int bro_qrql_values(int64_t n, const double* d, const double* e, double* w, int ref) {
    if (n <= 0) return BRO_INVALID_ARGUMENT;
    double* ee = (double*)malloc(sizeof(double) * (size_t)(n > 1 ? n - 1 : 1));
    if (!ee) return BRO_OUT_OF_MEMORY;
    memcpy(w, d, sizeof(double) * (size_t)n);
    if (n > 1) memcpy(ee, e, sizeof(double) * (size_t)(n - 1));
    int st = steqr(n, w, ee, NULL, NULL, ref);
    free(ee);
    if (st) return st;
    qsort(w, (size_t)n, sizeof(double), cmp_double);
    return BRO_OK;
}

/* ------------------------------------------------------------------------- */
/* merge tree: merge_tree.cpp:34-60                                          */
/* ------------------------------------------------------------------------- */
typedef struct {
    int64_t off, size;  /* global offset */
    int32_t left, right, level;
    int32_t block;
} node_t;

typedef struct {
    node_t* nodes;
    int64_t count, cap;
} tree_t;

static int32_t build_node(tree_t* t, int64_t off, int64_t size, int cutoff, int32_t block) {
    int32_t id = (int32_t)t->count++;
    node_t* nd = &t->nodes[id];
    nd->off = off; nd->size = size; nd->left = -1; nd->right = -1; nd->level = 0; nd->block = block;
    if (size > cutoff) {
        int64_t nl = size / 2;
        int32_t l = build_node(t, off, nl, cutoff, block);
        int32_t r = build_node(t, off + nl, size - nl, cutoff, block);
        nd = &t->nodes[id];
        nd->left = l; nd->right = r;
        int32_t ll = t->nodes[l].level, rl = t->nodes[r].level;
        nd->level = 1 + (ll > rl ? ll : rl);
    }
    return id;
}

/* ------------------------------------------------------------------------- */
/* merge step                                              */
/* ------------------------------------------------------------------------- */
typedef struct {
    int status;
    int K, nn, nrot;
    int64_t evals;
    double pole_terms;
    double tol;
} merge_out;

/* lam/blo/bhi hold both children at [off, off+size); replaced by the parent.
 * par != 0 allows OpenMP inside the merge. */
/* Merge-input dump for the Theorem 1 test (test infrastructure): records
 * (offset, size, n_left, D[size], z[size]) per merge while buf is set. */
static struct { double* buf; int64_t cap, used; } g_dump;
void bro_set_merge_dump(double* buf, int64_t cap) { g_dump.buf = buf; g_dump.cap = cap; g_dump.used = 0; }
int64_t bro_merge_dump_used(void) { return g_dump.used; }

/* Selected rows sigma (global row indices) of the whole solve: S holds, per
 * requested row r, the row sel[r] of the current node's eigenvector matrix at
 * that node's positions (stride N), in the node's ascending eigenvalue order. */
typedef struct {
    int64_t nsel, N;
    const int64_t* sel;
    double* S;
} sigma_t;

static merge_out merge_node(double* lam, double* blo, double* bhi, int64_t off, int64_t size,
                            double rho, int sign, int is_root, const bro_opts* o, int par,
                            const sigma_t* sg) {
    merge_out mo;
    memset(&mo, 0, sizeof(mo));
    const int n = (int)size, nL = (int)(size / 2), nR = n - nL;
    const int ref = o->ref_arith;
    int split = !ref && n > BRO_SPLIT_MIN_SIZE;
    double* lamL = lam + off;
    double* lamR = lam + off + nL;
    double* buf = (double*)malloc(sizeof(double) * (size_t)n * 11);
    int* ibuf = (int*)malloc(sizeof(int) * (size_t)n * 3);
    if (!buf || !ibuf) { free(buf); free(ibuf); mo.status = BRO_OUT_OF_MEMORY; return mo; }
    double *D = buf, *Z = buf + n, *R0 = buf + 2 * n, *R1 = buf + 3 * n;
    double *dA = buf + 4 * n, *zA = buf + 5 * n, *r0A = buf + 6 * n, *r1A = buf + 7 * n;
    double *tau = buf + 8 * n, *zh = buf + 9 * n, *outb = buf + 10 * n;
    int *act = ibuf, *defl = ibuf + n, *org = ibuf + 2 * n;
    /* selected rows inside this node (split_row_request: the
     * child that holds a row contributes it, the other child's columns are 0) */
    int nx = 0;
    int64_t* xr = NULL;
    double *X = NULL, *XA = NULL, *XO = NULL, *SX = NULL;
    if (sg && sg->nsel) {
        xr = (int64_t*)malloc(sizeof(int64_t) * (size_t)sg->nsel);
        for (int64_t r = 0; r < sg->nsel; ++r)
            if (sg->sel[r] >= off && sg->sel[r] < off + size) xr[nx++] = r;
        if (nx) {
            X = (double*)malloc(sizeof(double) * (size_t)n * (size_t)nx * 3);
            SX = (double*)malloc(sizeof(double) * (size_t)nx);
            XA = X + (size_t)n * nx;
            XO = XA + (size_t)n * nx;
        }
    }

    /* tol: deflate.cpp:55-60 over D = lam_L ++ lam_R and z = (sign*bhi_L, blo_R) */
    double dmax = 0.0, zmax = 0.0;
    for (int i = 0; i < n; ++i) {
        dmax = fmax(dmax, fabs(lam[off + i]));
        zmax = fmax(zmax, fabs(i < nL ? bhi[off + i] : blo[off + i]));
    }
    const double tol = 8.0 * U_RND * fmax(dmax, zmax) * o->tol_scale;
    mo.tol = tol;

    /* stable merge of the sorted children (== std::stable_sort, deflate.cpp:62-66) */
    {
        int a = 0, b = 0;
        for (int k = 0; k < n; ++k) {
            int take_right = (a == nL) || (b < nR && lamR[b] < lamL[a]);
            if (!take_right) {
                const int64_t p = off + a;
                D[k] = lamL[a];
                Z[k] = sign < 0 ? -bhi[p] : bhi[p];
                R0[k] = blo[p];
                R1[k] = 0.0;
                for (int x = 0; x < nx; ++x)
                    X[(int64_t)x * n + k] = sg->sel[xr[x]] < off + nL ? sg->S[xr[x] * sg->N + p] : 0.0;
                ++a;
            } else {
                const int64_t p = off + nL + b;
                D[k] = lamR[b];
                Z[k] = blo[p];
                R0[k] = 0.0;
                R1[k] = bhi[p];
                for (int x = 0; x < nx; ++x)
                    X[(int64_t)x * n + k] = sg->sel[xr[x]] >= off + nL ? sg->S[xr[x] * sg->N + p] : 0.0;
                ++b;
            }
        }
    }
    /* test hook (Theorem 1 check): merged poles and z of every merge, before deflation */
    if (g_dump.buf) {
        int64_t at;
#pragma omp atomic capture
        { at = g_dump.used; g_dump.used += 3 + 2 * (int64_t)n; }
        if (at + 3 + 2 * (int64_t)n <= g_dump.cap) {
            double* q = g_dump.buf + at;
            q[0] = (double)off; q[1] = (double)n; q[2] = (double)nL;
            memcpy(q + 3, D, sizeof(double) * (size_t)n);
            memcpy(q + 3 + n, Z, sizeof(double) * (size_t)n);
        }
    }
    defl_info info;
    deflate_walk(n, D, Z, is_root ? NULL : R0, is_root ? NULL : R1, tol, ref, act, defl, &info, nx, X, SX);
    const int K = info.K;
    mo.K = K; mo.nn = info.nn; mo.nrot = info.nrot;
    if (!ref && K > BRO_SPLIT_MIN_K) split = 1;
    for (int a = 0; a < K; ++a) {
        dA[a] = D[act[a]];
        zA[a] = Z[act[a]];
        if (!is_root) { r0A[a] = R0[act[a]]; r1A[a] = R1[act[a]]; }
        for (int x = 0; x < nx; ++x) XA[(int64_t)x * n + a] = X[(int64_t)x * n + act[a]];
    }

    /* secular roots (secular.cpp:80-241), independent per root */
    int st_all = BRO_OK;
    int64_t evals = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : evals) if (par && K >= 64)
    for (int j = 0; j < K; ++j) {
        int ne = 0;
        int st = solve_root_impl(K, dA, zA, rho, j, o->patched_stop, ref, split, &org[j], &tau[j], &ne);
        evals += ne;
        if (st) {
#pragma omp atomic write
            st_all = st;
        }
    }
    mo.evals = evals;
    mo.pole_terms = (double)evals * (double)K;
    if (st_all) { mo.status = st_all; goto done; }

    if (!is_root && K > 0) {
        if (o->zhat && K > 1) {
            /* refreshed weights, one pole per iteration (sequential root order inside) */
#pragma omp parallel for schedule(static) if (par && K >= 64)
            for (int i = 0; i < K; ++i) {
                const double di = dA[i];
                double w = 1.0;
                if (split) {
                    double W[BRO_SPLIT];
                    for (int l = 0; l < BRO_SPLIT; ++l) {
                        W[l] = 1.0;
                        for (int j = l; j < K; j += BRO_SPLIT) {
                            const double del = (di - dA[org[j]]) - tau[j];
                            if (i == j) W[l] *= del;
                            else W[l] *= del * (1.0 / (di - dA[j]));
                        }
                    }
                    w = bfly_mul(W);
                } else {
                    for (int j = 0; j < K; ++j) {
                        const double del = (di - dA[org[j]]) - tau[j];
                        if (i == j) w *= del;
                        else if (ref) w *= del / (di - dA[j]);
                        else w *= del * (1.0 / (di - dA[j]));
                    }
                }
                const double mag = sqrt(fmax(0.0, -w));
                zh[i] = zA[i] >= 0.0 ? mag : -mag;
            }
        } else {
            memcpy(zh, zA, sizeof(double) * (size_t)K);
        }
        /* stream secular columns through the two selected rows:
         * blo' -> outb[j], bhi' -> zA[j] */
#pragma omp parallel if (par && K >= 64)
        {
            double* ybuf = ref ? (double*)malloc(sizeof(double) * (size_t)K) : NULL;
#pragma omp for schedule(static)
            for (int j = 0; j < K; ++j) {
                double b0, b1;
                int st = root_rows(K, dA, zh, r0A, r1A, org[j], tau[j], ref, split, &b0, &b1, ybuf);
                if (st) {
#pragma omp atomic write
                    st_all = st;
                }
                outb[j] = b0;
                zA[j] = b1; /* zA is dead once zh is formed; reuse it for bhi' */
            }
            free(ybuf);
        }
        if (st_all) { mo.status = st_all; goto done; }
        /* selected rows: R_parent(sigma, j) = R_child(sigma, :) y_j */
        for (int x = 0; x < nx; ++x)
            for (int j = 0; j < K; ++j) {
                int st = sigma_root_row(K, dA, zh, XA + (int64_t)x * n, org[j], tau[j], ref,
                                        &XO[(int64_t)x * n + j]);
                if (st) st_all = st;
            }
        if (st_all) { mo.status = st_all; goto done; }
    }

    /* parent order: stable merge of deflated list (walk order) then roots */
    {
        const int ndef = n - K;
        int a = 0, b = 0;
        for (int k = 0; k < n; ++k) {
            double lr = 0.0;
            int take_root = 0;
            if (b < K) {
                lr = dA[org[b]] + tau[b];
                take_root = (a == ndef) || (lr < D[defl[a]]);
            }
            const int64_t p = off + k;
            if (take_root) {
                lam[p] = lr;
                if (!is_root) { blo[p] = outb[b]; bhi[p] = zA[b]; }
                for (int x = 0; x < nx; ++x) sg->S[xr[x] * sg->N + p] = XO[(int64_t)x * n + b];
                ++b;
            } else {
                const int s = defl[a];
                lam[p] = D[s];
                if (!is_root) { blo[p] = R0[s]; bhi[p] = R1[s]; }
                for (int x = 0; x < nx; ++x) sg->S[xr[x] * sg->N + p] = X[(int64_t)x * n + s];
                ++a;
            }
        }
    }
done:
    free(buf);
    free(ibuf);
    free(xr);
    free(X);
    free(SX);
    return mo;
}

/* ------------------------------------------------------------------------- */
/* driver: SPEC.md:348-356                                                   */
/* ------------------------------------------------------------------------- */
void bro_default_opts(bro_opts* o) {
    o->leaf_cutoff = 25;
    o->zhat = 1;
    o->patched_stop = 1;
    o->ref_arith = 0;
    o->threads = 0;
    o->tol_scale = 1.0;
}

static int solve_impl(int64_t n, const double* d, const double* e, double* w, const bro_opts* o,
                      bro_stats* st, bro_trace* trace, int64_t trace_cap, int64_t* trace_len,
                      int allow_par, int64_t nsel, const int64_t* sel, double* rows) {
    if (n <= 0 || !d || (!e && n > 1) || !w) return BRO_INVALID_ARGUMENT;
    for (int64_t i = 0; i < n; ++i) if (!isfinite(d[i])) return BRO_INVALID_ARGUMENT;
    for (int64_t i = 0; i + 1 < n; ++i) if (!isfinite(e[i])) return BRO_INVALID_ARGUMENT;
    if (o->leaf_cutoff < 5 || o->leaf_cutoff > 64) return BRO_INVALID_ARGUMENT;
    const int cutoff = o->leaf_cutoff;
    int status = BRO_OK;
    for (int64_t r = 0; r < nsel; ++r)
        if (sel[r] < 0 || sel[r] >= n) return BRO_INVALID_ARGUMENT;
    sigma_t sg = {nsel, n, sel, NULL};
    int64_t* pos = NULL;

    /* irreducible blocks: tridiagonal.cpp:45-58 with tol = u */
    int64_t nblk = 0;
    int64_t* bstart = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
    double* scale = (double*)malloc(sizeof(double) * (size_t)n);
    double* dw = (double*)malloc(sizeof(double) * (size_t)n);
    double* ew = (double*)malloc(sizeof(double) * (size_t)(n > 1 ? n : 1));
    double* blo = (double*)malloc(sizeof(double) * (size_t)n);
    double* bhi = (double*)malloc(sizeof(double) * (size_t)n);
    tree_t t;
    t.cap = 2 * (n / ((cutoff + 1) / 2) + 1) + 2 * n / 8 + 16;
    t.count = 0;
    t.nodes = (node_t*)malloc(sizeof(node_t) * (size_t)t.cap);
    if (nsel) sg.S = (double*)calloc((size_t)(nsel * n), sizeof(double));
    if (!bstart || !scale || !dw || !ew || !blo || !bhi || !t.nodes || (nsel && !sg.S)) { status = BRO_OUT_OF_MEMORY; goto out; }

    bstart[nblk++] = 0;
    for (int64_t i = 0; i + 1 < n; ++i)
        if (fabs(e[i]) <= U_RND * (fabs(d[i]) + fabs(d[i + 1]))) bstart[nblk++] = i + 1;
    bstart[nblk] = n;

    /* scale each block by max(|d|,|e|,1) and build its tree.
     * GPU mode also lifts TINY blocks (max < 2^-500) by the power of two
     * 2^ilogb(max): exact, and it keeps y = zhat/Delta and its square from
     * overflowing when every pole gap is below ~1e-154 (the reference's
     * max(.,1) never enlarges, so such blocks end in inf/NaN there). */
    int32_t height = 0;
    for (int64_t b = 0; b < nblk; ++b) {
        const int64_t off = bstart[b], sz = bstart[b + 1] - off;
        double mx = 0.0;
        for (int64_t i = 0; i < sz; ++i) mx = fmax(mx, fabs(d[off + i]));
        for (int64_t i = 0; i + 1 < sz; ++i) mx = fmax(mx, fabs(e[off + i]));
        double s = fmax(1.0, mx);
        if (!o->ref_arith && mx > 0.0 && mx < 0x1p-500) s = ldexp(1.0, ilogb(mx));
        scale[b] = s;
        for (int64_t i = 0; i < sz; ++i) dw[off + i] = d[off + i] / s;
        for (int64_t i = 0; i + 1 < sz; ++i) ew[off + i] = e[off + i] / s;
        if (off + sz < n) ew[off + sz - 1] = 0.0;
        if (sz > cutoff) {
            int32_t root = build_node(&t, off, sz, cutoff, (int32_t)b);
            if (t.nodes[root].level > height) height = t.nodes[root].level;
        }
    }
    if (t.count > t.cap) { status = BRO_OUT_OF_MEMORY; goto out; }

    /* Cuppen cuts, pre-order (merge_tree.cpp:78-92) */
    for (int64_t i = 0; i < t.count; ++i) {
        node_t* nd = &t.nodes[i];
        if (nd->left < 0) continue;
        const int64_t m = nd->off + nd->size / 2 - 1;
        const double rho = fabs(ew[m]);
        dw[m] -= rho;
        dw[m + 1] -= rho;
    }

    /* leaves of every tree + blocks <= cutoff (values only) */
    {
        int64_t nleaf = 0;
        for (int64_t i = 0; i < t.count; ++i) if (t.nodes[i].left < 0) ++nleaf;
        int lerr = BRO_OK;
#pragma omp parallel for schedule(dynamic, 64) if (allow_par)
        for (int64_t i = 0; i < t.count; ++i) {
            const node_t* nd = &t.nodes[i];
            if (nd->left >= 0) continue;
            int r = bro_leaf((int)nd->size, dw + nd->off, ew + nd->off, w + nd->off,
                             blo + nd->off, bhi + nd->off, o->ref_arith);
            if (r) {
#pragma omp atomic write
                lerr = r;
            }
        }
#pragma omp parallel for schedule(dynamic, 64) if (allow_par)
        for (int64_t b = 0; b < nblk; ++b) {
            const int64_t off = bstart[b], sz = bstart[b + 1] - off;
            if (sz > cutoff) continue;
            double lam[64], ee[64];
            memcpy(lam, dw + off, sizeof(double) * (size_t)sz);
            if (sz > 1) memcpy(ee, ew + off, sizeof(double) * (size_t)(sz - 1));
            int r = steqr(sz, lam, ee, NULL, NULL, o->ref_arith);
            if (r) {
#pragma omp atomic write
                lerr = r;
            }
            stable_sort_rows((int)sz, lam, NULL, NULL);
            memcpy(w + off, lam, sizeof(double) * (size_t)sz);
        }
        (void)nleaf;
        /* selected rows of the leaves (and of blocks <= cutoff): the leaf QL/QR
         * tracking row sel-off instead of the boundary rows (inc/qrql.hpp:38-42) */
        for (int64_t r = 0; r < nsel && !lerr; ++r) {
            const int64_t i = sel[r];
            int64_t off = -1, sz = 0;
            for (int64_t q = 0; q < t.count; ++q)
                if (t.nodes[q].left < 0 && t.nodes[q].off <= i && i < t.nodes[q].off + t.nodes[q].size) {
                    off = t.nodes[q].off; sz = t.nodes[q].size;
                    break;
                }
            if (off < 0)
                for (int64_t b = 0; b < nblk; ++b)
                    if (bstart[b] <= i && i < bstart[b + 1]) { off = bstart[b]; sz = bstart[b + 1] - off; break; }
            double lam[64], ee[64], x[64];
            memcpy(lam, dw + off, sizeof(double) * (size_t)sz);
            if (sz > 1) memcpy(ee, ew + off, sizeof(double) * (size_t)(sz - 1));
            for (int64_t k = 0; k < sz; ++k) x[k] = k == i - off ? 1.0 : 0.0;
            int rr = steqr(sz, lam, ee, x, NULL, o->ref_arith);
            if (rr) lerr = rr;
            stable_sort_rows((int)sz, lam, x, NULL);
            memcpy(sg.S + r * n + off, x, sizeof(double) * (size_t)sz);
        }
        if (lerr) { status = lerr; goto out; }
    }

    /* level loop (level-synchronous, disjoint merges) */
    {
        int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(t.count + 1));
        int64_t tl = 0;
        if (!order) { status = BRO_OUT_OF_MEMORY; goto out; }
        int nthreads = 1;
#ifdef _OPENMP
        if (allow_par) nthreads = omp_get_max_threads();
#endif
        for (int32_t lev = 1; lev <= height && status == BRO_OK; ++lev) {
            int64_t cnt = 0;
            for (int64_t i = 0; i < t.count; ++i)
                if (t.nodes[i].left >= 0 && t.nodes[i].level == lev) order[cnt++] = i;
            /* offset order == pre-order within a block; blocks are offset ordered */
            const int par_inside = allow_par && cnt < nthreads;
            int lerr = BRO_OK;
            int64_t sk = 0, snn = 0, srot = 0, sev = 0, mk = 0;
            double sk2 = 0.0, spt = 0.0, szt = 0.0;
#pragma omp parallel for schedule(dynamic, 1) if (allow_par && !par_inside) \
    reduction(+ : sk, snn, srot, sev, sk2, spt, szt) reduction(max : mk)
            for (int64_t q = 0; q < cnt; ++q) {
                const node_t* nd = &t.nodes[order[q]];
                const int64_t m = nd->off + nd->size / 2 - 1;
                const double rho = fabs(ew[m]);
                const int sign = ew[m] < 0 ? -1 : 1;
                /* root-only mode unless rows are requested */
                const int is_root = !nsel && (nd->off == bstart[nd->block]) &&
                                    (nd->size == bstart[nd->block + 1] - bstart[nd->block]);
                merge_out mo = merge_node(w, blo, bhi, nd->off, nd->size, rho, sign, is_root, o,
                                          par_inside, nsel ? &sg : NULL);
                if (mo.status) {
#pragma omp atomic write
                    lerr = mo.status;
                }
                sk += mo.K; sk2 += (double)mo.K * (double)mo.K; snn += mo.nn; srot += mo.nrot;
                sev += mo.evals; spt += mo.pole_terms;
                if (!is_root) szt += (double)mo.K * (double)mo.K;
                if (mo.K > mk) mk = mo.K;
                if (trace && tl + q < trace_cap) {
                    bro_trace* tr = &trace[tl + q];
                    tr->level = lev; tr->is_root = is_root; tr->offset = nd->off; tr->size = nd->size;
                    tr->nn = mo.nn; tr->k = mo.K; tr->tol = mo.tol; tr->rho = rho;
                }
            }
            tl += cnt;
            if (st) {
                st->merges += cnt; st->sum_k += sk; st->sum_k2 += sk2; st->sum_nn += snn;
                st->rotations += srot; st->evals += sev; st->pole_terms += spt;
                st->row_terms += szt;
                if (o->zhat) st->zhat_terms += szt;
                if (mk > st->max_k) st->max_k = mk;
            }
            if (lerr) status = lerr;
        }
        if (trace_len) *trace_len = tl;
        free(order);
        if (status) goto out;
    }

    /* rescale, then global ascending (stable) sort across blocks */
    for (int64_t b = 0; b < nblk; ++b)
        for (int64_t i = bstart[b]; i < bstart[b + 1]; ++i) w[i] *= scale[b];
    if (nsel) {
        /* selected rows to the global column order: element i of block b goes
         * to its stable rank #{j: w_j < w_i} + #{j < i: w_j == w_i} (the order
         * of the stable cross-block sort below); other blocks' columns are 0 */
        pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
        if (!pos) { status = BRO_OUT_OF_MEMORY; goto out; }
        for (int64_t i = 0; i < n; ++i) pos[i] = i;
        if (nblk > 1) {
            int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)n * 2);
            if (!idx) { status = BRO_OUT_OF_MEMORY; goto out; }
            int64_t* tmp = idx + n;
            for (int64_t i = 0; i < n; ++i) idx[i] = i;
            for (int64_t wd = 1; wd < n; wd *= 2) {  /* stable merge sort of indices by value */
                for (int64_t lo = 0; lo < n; lo += 2 * wd) {
                    int64_t mid = lo + wd < n ? lo + wd : n, hi = lo + 2 * wd < n ? lo + 2 * wd : n;
                    int64_t a = lo, b = mid, k = lo;
                    while (a < mid && b < hi) tmp[k++] = (w[idx[b]] < w[idx[a]]) ? idx[b++] : idx[a++];
                    while (a < mid) tmp[k++] = idx[a++];
                    while (b < hi) tmp[k++] = idx[b++];
                }
                memcpy(idx, tmp, sizeof(int64_t) * (size_t)n);
            }
            for (int64_t k = 0; k < n; ++k) pos[idx[k]] = k;
            free(idx);
        }
        memset(rows, 0, sizeof(double) * (size_t)(nsel * n));
        for (int64_t r = 0; r < nsel; ++r) {
            int64_t b = 0;
            while (bstart[b + 1] <= sel[r]) ++b;
            for (int64_t i = bstart[b]; i < bstart[b + 1]; ++i) rows[r * n + pos[i]] = sg.S[r * n + i];
        }
    }
    if (nblk > 1) stable_sort_values(n, w, dw);
    if (st) { st->height = height; st->blocks = (int32_t)nblk; }

out:
    free(bstart); free(scale); free(dw); free(ew); free(blo); free(bhi); free(t.nodes);
    free(sg.S); free(pos);
    return status;
}

int bro_eigvals(int64_t n, const double* d, const double* e, double* w, const bro_opts* o,
                bro_stats* st, bro_trace* trace, int64_t trace_cap, int64_t* trace_len) {
    bro_opts def;
    if (!o) { bro_default_opts(&def); o = &def; }
    if (st) memset(st, 0, sizeof(*st));
#ifdef _OPENMP
    int saved = omp_get_max_threads();
    if (o->threads > 0) omp_set_num_threads(o->threads);
    int r = solve_impl(n, d, e, w, o, st, trace, trace_cap, trace_len, o->threads != 1, 0, NULL, NULL);
    omp_set_num_threads(saved);
    return r;
#else
    return solve_impl(n, d, e, w, o, st, trace, trace_cap, trace_len, 0, 0, NULL, NULL);
#endif
}

/* Algorithm 1 with requested rows sigma: eigenvalues w
 * ascending plus rows[r*n + j] = Q(sel[r], j), Q the eigenvector matrix of T
 * with columns in the order of w (0-based global row indices, duplicates and
 * any order allowed).  Every merge, the block root included, propagates the
 * requested rows; with nsel == 0 this is bro_eigvals. */
int bro_eigvals_rows(int64_t n, const double* d, const double* e, double* w, int64_t nsel,
                     const int64_t* sel, double* rows, const bro_opts* o) {
    bro_opts def;
    if (!o) { bro_default_opts(&def); o = &def; }
    if (nsel < 0 || (nsel && (!sel || !rows))) return BRO_INVALID_ARGUMENT;
#ifdef _OPENMP
    int saved = omp_get_max_threads();
    if (o->threads > 0) omp_set_num_threads(o->threads);
    int r = solve_impl(n, d, e, w, o, NULL, NULL, 0, NULL, o->threads != 1, nsel, sel, rows);
    omp_set_num_threads(saved);
    return r;
#else
    return solve_impl(n, d, e, w, o, NULL, NULL, 0, NULL, 0, nsel, sel, rows);
#endif
}

int bro_eigvals_batched(int64_t batch, int64_t n, const double* d, const double* e, double* w,
                        const bro_opts* o, bro_stats* st) {
    bro_opts def;
    if (!o) { bro_default_opts(&def); o = &def; }
    if (batch < 0 || n <= 0) return BRO_INVALID_ARGUMENT;
    if (st) memset(st, 0, sizeof(*st));
    int status = BRO_OK;
#ifdef _OPENMP
    int saved = omp_get_max_threads();
    if (o->threads > 0) omp_set_num_threads(o->threads);
#endif
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < batch; ++b) {
        bro_stats s1;
        memset(&s1, 0, sizeof(s1));
        int r = solve_impl(n, d + b * n, e + b * (n - 1), w + b * n, o, st ? &s1 : NULL, NULL, 0,
                           NULL, 0, 0, NULL, NULL);
        if (r) {
#pragma omp atomic write
            status = r;
        }
        if (st) {
#pragma omp critical
            {
                st->merges += s1.merges; st->sum_k += s1.sum_k; st->sum_k2 += s1.sum_k2;
                st->sum_nn += s1.sum_nn; st->rotations += s1.rotations; st->evals += s1.evals;
                st->pole_terms += s1.pole_terms; st->zhat_terms += s1.zhat_terms;
                st->row_terms += s1.row_terms;
                if (s1.max_k > st->max_k) st->max_k = s1.max_k;
                if (s1.height > st->height) st->height = s1.height;
                st->blocks += s1.blocks;
            }
        }
    }
#ifdef _OPENMP
    omp_set_num_threads(saved);
#endif
    return status;
}

/* Number of eigenvalues < x (LDL^T inertia), for Sturm certificates. */
int64_t bro_sturm_count(int64_t n, const double* d, const double* e, double x) {
    const double pivmin = DBL_MIN * 4.0;
    int64_t cnt = 0;
    double q = d[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    if (q < 0) ++cnt;
    for (int64_t i = 1; i < n; ++i) {
        q = (d[i] - x) - e[i - 1] * e[i - 1] / q;
        if (fabs(q) < pivmin) q = -pivmin;
        if (q < 0) ++cnt;
    }
    return cnt;
}
