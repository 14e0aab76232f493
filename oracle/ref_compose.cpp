// ref_compose.cpp -- the BR driver of SPEC.md:312-380 composed from the
// UNMODIFIED reference building blocks compiled from /root/reference/proj/src.
//
// TEST INFRASTRUCTURE ONLY (built by oracle/Makefile into oracle/_ref/).  The
// reference ships every block but no driver; this file is the
// composition the survey probed, with OpenMP over same-level
// merges and over roots inside a merge.  It is
// (a) the pin for the C restatement in br_oracle.c (ref_arith mode must agree
// bitwise on eigenvalues) and (b) bench.py's "reference" CPU arm.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "br/boundary_state.hpp"
#include "br/deflate.hpp"
#include "br/dense.hpp"
#include "br/errors.hpp"
#include "br/merge_tree.hpp"
#include "br/oracle.hpp"
#include "br/qrql.hpp"
#include "br/secular.hpp"
#include "br/tridiagonal.hpp"

namespace {

int code_of(const std::exception& ex) {
    if (dynamic_cast<const br::InvalidArgument*>(&ex)) return 1;
    if (dynamic_cast<const br::NoConvergence*>(&ex)) return 2;
    if (dynamic_cast<const br::BudgetExceeded*>(&ex)) return 3;
    if (dynamic_cast<const br::PoleHit*>(&ex)) return 4;
    if (dynamic_cast<const br::ZeroDenominator*>(&ex)) return 5;
    if (dynamic_cast<const br::MalformedCompactRoot*>(&ex)) return 6;
    if (dynamic_cast<const br::DimensionMismatch*>(&ex)) return 7;
    if (dynamic_cast<const br::DomainError*>(&ex)) return 8;
    return 99;
}

struct NodeState {
    std::vector<double> lam, blo, bhi;
};

// merge_step(left, right, rho, sign, internal|root).
NodeState merge_step(const NodeState& L, const NodeState& R, double rho, int sign, bool is_root,
                     bool zhat, bool par) {
    const std::size_t nL = L.lam.size(), nR = R.lam.size(), n = nL + nR;
    br::BoundaryState bl, br_;
    bl.bhi = L.bhi; bl.local_lambda = L.lam;
    br_.blo = R.blo; br_.local_lambda = R.lam;
    std::vector<double> z = br::build_z(bl, br_, sign);            // deflate.cpp:31-41
    std::vector<double> D(L.lam);
    D.insert(D.end(), R.lam.begin(), R.lam.end());
    br::MergePrep prep = br::deflate_merge(D, z, rho);              // deflate.cpp:43-107
    br::Matrix rows(2, n);
    for (std::size_t i = 0; i < nL; ++i) rows(0, i) = L.blo[i];
    for (std::size_t i = 0; i < nR; ++i) rows(1, nL + i) = R.bhi[i];
    br::Matrix rowsp = br::apply_prep_to_rows(rows, prep);          // deflate.cpp:121-140
    std::vector<std::int32_t> inv(n);
    for (std::size_t k = 0; k < n; ++k) inv[static_cast<std::size_t>(prep.perm[k])] = static_cast<std::int32_t>(k);

    const std::size_t K = prep.active_rank();
    br::SecularProblem P{prep.d_active, prep.z_active, rho};
    std::vector<br::CompactRoot> roots(K);
    std::vector<double> rl(K);
    std::string err;
    int errc = 0;
#pragma omp parallel for schedule(dynamic, 16) if (par && K >= 64)
    for (std::int64_t j = 0; j < static_cast<std::int64_t>(K); ++j) {
        try {
            roots[j] = br::solve_root(static_cast<std::size_t>(j), P);   // secular.cpp:80-241
            rl[j] = br::root_value(P, roots[j]);
        } catch (const std::exception& ex) {
#pragma omp critical
            { errc = code_of(ex); err = ex.what(); }
        }
    }
    if (errc) throw br::NoConvergence(err);

    std::vector<double> bl_out(K), bh_out(K);
    if (!is_root && K > 0) {
        br::SecularProblem P2 = P;
        if (zhat) P2.z = br::refreshed_weights(P, roots);            // secular.cpp:288-313
        std::vector<double> r0(K), r1(K);
        for (std::size_t a = 0; a < K; ++a) {
            r0[a] = rowsp(0, static_cast<std::size_t>(prep.active_pos[a]));
            r1[a] = rowsp(1, static_cast<std::size_t>(prep.active_pos[a]));
        }
#pragma omp parallel for schedule(static) if (par && K >= 64)
        for (std::int64_t j = 0; j < static_cast<std::int64_t>(K); ++j) {
            try {
                std::vector<double> y = br::secular_column(P2, roots[j]);   // secular.cpp:272-286
                bl_out[j] = br::dot(r0, y);                                 // dense.hpp:48-53
                bh_out[j] = br::dot(r1, y);
            } catch (const std::exception& ex) {
#pragma omp critical
                { errc = code_of(ex); err = ex.what(); }
            }
        }
        if (errc == 5) throw br::ZeroDenominator(err);
        if (errc) throw br::NoConvergence(err);
    }

    // parent: ascending (deflated poles U roots), stable with deflated first
    NodeState out;
    out.lam.resize(n);
    if (!is_root) { out.blo.resize(n); out.bhi.resize(n); }
    const std::size_t nd = prep.deflated.size();
    std::size_t a = 0, b = 0;
    for (std::size_t k = 0; k < n; ++k) {
        bool take_root = b < K && (a == nd || rl[b] < prep.deflated[a].second);
        if (take_root) {
            out.lam[k] = rl[b];
            if (!is_root) { out.blo[k] = bl_out[b]; out.bhi[k] = bh_out[b]; }
            ++b;
        } else {
            const auto& dfl = prep.deflated[a];
            out.lam[k] = dfl.second;
            if (!is_root) {
                const std::size_t col = static_cast<std::size_t>(inv[static_cast<std::size_t>(dfl.first)]);
                out.blo[k] = rowsp(0, col);
                out.bhi[k] = rowsp(1, col);
            }
            ++a;
        }
    }
    return out;
}

std::vector<double> solve_block(const std::vector<double>& d, const std::vector<double>& e,
                                std::size_t cutoff, bool zhat, int nthreads) {
    const std::size_t n = d.size();
    if (n <= cutoff)
        return br::eigenvalues_qrql(br::TridiagonalMatrix(d, e));     // qrql.cpp:386-394
    br::MergeTree tree = br::build_merge_tree(n, cutoff);            // merge_tree.cpp:53-60
    std::vector<double> dm(d);
    br::apply_all_splits(tree, dm, e);                               // merge_tree.cpp:78-92
    std::vector<NodeState> st(tree.nodes.size());
    std::vector<std::int32_t> leaves = tree.leaves();
    bool leaf_fail = false;
#pragma omp parallel for schedule(dynamic, 64) if (nthreads > 1)
    for (std::int64_t q = 0; q < static_cast<std::int64_t>(leaves.size()); ++q) {
        const br::MergeNode& nd = tree.at(leaves[q]);
        std::vector<double> ld(dm.begin() + nd.offset, dm.begin() + nd.offset + nd.size);
        std::vector<double> le(e.begin() + nd.offset, e.begin() + nd.offset + nd.size - 1);
        try {
            br::LeafEigenResult r = br::leaf_eig(br::TridiagonalMatrix(ld, le));  // qrql.cpp:396-413
            NodeState& s = st[leaves[q]];
            s.lam = r.lambda;
            s.blo.assign(r.q.row(0).begin(), r.q.row(0).end());
            s.bhi.assign(r.q.row(nd.size - 1).begin(), r.q.row(nd.size - 1).end());
        } catch (const std::exception&) {
#pragma omp critical
            leaf_fail = true;
        }
    }
    if (leaf_fail) throw br::NoConvergence("leaf_eig failed");
    for (std::int32_t lev = 1; lev <= tree.height(); ++lev) {
        std::vector<std::int32_t> ids = tree.internal_at_level(lev);
        const bool par_inside = nthreads > 1 && static_cast<int>(ids.size()) < nthreads;
        std::string err;
        int errc = 0;
#pragma omp parallel for schedule(dynamic, 1) if (nthreads > 1 && !par_inside)
        for (std::int64_t q = 0; q < static_cast<std::int64_t>(ids.size()); ++q) {
            const br::MergeNode& nd = tree.at(ids[q]);
            try {
                NodeState s = merge_step(st[nd.left], st[nd.right], nd.rho, nd.split_sign,
                                         ids[q] == tree.root, zhat, par_inside);
                st[ids[q]] = std::move(s);
                st[nd.left] = NodeState{};
                st[nd.right] = NodeState{};
            } catch (const std::exception& ex) {
#pragma omp critical
                { errc = code_of(ex); err = ex.what(); }
            }
        }
        if (errc == 2) throw br::NoConvergence(err);
        if (errc == 5) throw br::ZeroDenominator(err);
        if (errc) throw br::InvalidArgument(err);
    }
    return st[tree.root].lam;
}

} // namespace

extern "C" {

// br_eigenvalues(T, threads) of SPEC.md:348-356 from the reference blocks.
int brref_eigvals(std::int64_t n, const double* d, const double* e, double* w, int threads,
                  int zhat, int leaf_cutoff) {
    try {
#ifdef _OPENMP
        const int saved = omp_get_max_threads();
        if (threads > 0) omp_set_num_threads(threads);
        const int nth = omp_get_max_threads();
#else
        const int nth = 1;
#endif
        if (n <= 0) throw br::InvalidArgument("order must be positive");
        br::TridiagonalMatrix T(std::vector<double>(d, d + n),
                                std::vector<double>(e, e + (n > 1 ? n - 1 : 0)));   // validates
        const std::vector<br::Block> blocks = br::find_irreducible_blocks(T, 0x1p-53);
        std::vector<double> out;
        out.reserve(static_cast<std::size_t>(n));
        for (const br::Block& b : blocks) {
            double s = 1.0;
            for (std::size_t i = 0; i < b.size; ++i) s = std::max(s, std::abs(T.d[b.offset + i]));
            for (std::size_t i = 0; i + 1 < b.size; ++i) s = std::max(s, std::abs(T.e[b.offset + i]));
            std::vector<double> bd(b.size), be(b.size - 1);
            for (std::size_t i = 0; i < b.size; ++i) bd[i] = T.d[b.offset + i] / s;
            for (std::size_t i = 0; i + 1 < b.size; ++i) be[i] = T.e[b.offset + i] / s;
            std::vector<double> lam = solve_block(bd, be, static_cast<std::size_t>(leaf_cutoff), zhat != 0, nth);
            for (double v : lam) out.push_back(v * s);
        }
        std::sort(out.begin(), out.end());
        std::memcpy(w, out.data(), sizeof(double) * out.size());
#ifdef _OPENMP
        omp_set_num_threads(saved);
#endif
        return 0;
    } catch (const std::exception& ex) {
        return code_of(ex);
    }
}

// The reference's own eigenvalue-only entry point (inc/qrql.hpp:20-23).
int brref_eigenvalues_qrql(std::int64_t n, const double* d, const double* e, double* w) {
    try {
        br::TridiagonalMatrix T(std::vector<double>(d, d + n),
                                std::vector<double>(e, e + (n > 1 ? n - 1 : 0)));
        std::vector<double> v = br::eigenvalues_qrql(T);
        std::memcpy(w, v.data(), sizeof(double) * v.size());
        return 0;
    } catch (const std::exception& ex) {
        return code_of(ex);
    }
}

int brref_dense_eig(std::int64_t n, const double* d, const double* e, double* w) {
    try {
        br::TridiagonalMatrix T(std::vector<double>(d, d + n),
                                std::vector<double>(e, e + (n > 1 ? n - 1 : 0)));
        std::vector<double> v = br::dense_eig(T);
        std::memcpy(w, v.data(), sizeof(double) * v.size());
        return 0;
    } catch (const std::exception& ex) {
        return code_of(ex);
    }
}

int brref_leaf_eig(int m, const double* d, const double* e, double* lam, double* blo, double* bhi) {
    try {
        br::TridiagonalMatrix T(std::vector<double>(d, d + m), std::vector<double>(e, e + (m - 1)));
        br::LeafEigenResult r = br::leaf_eig(T);
        for (int i = 0; i < m; ++i) {
            lam[i] = r.lambda[i];
            blo[i] = r.q(0, i);
            bhi[i] = r.q(m - 1, i);
        }
        return 0;
    } catch (const std::exception& ex) {
        return code_of(ex);
    }
}

int brref_solve_root(int k, const double* d, const double* z, double rho, int j, int* origin,
                     double* tau) {
    try {
        br::SecularProblem P{std::vector<double>(d, d + k), std::vector<double>(z, z + k), rho};
        br::CompactRoot r = br::solve_root(static_cast<std::size_t>(j), P);
        *origin = r.origin_index;
        *tau = r.tau;
        return 0;
    } catch (const std::exception& ex) {
        return code_of(ex);
    }
}

int brref_deflate(int n, const double* d, const double* z, double rho, double* d_active,
                  double* z_active, double* deflated, int* k_out, int* nrot_out, double* tol_out) {
    try {
        br::MergePrep p = br::deflate_merge(std::vector<double>(d, d + n), std::vector<double>(z, z + n), rho);
        for (std::size_t a = 0; a < p.d_active.size(); ++a) {
            d_active[a] = p.d_active[a];
            z_active[a] = p.z_active[a];
        }
        for (std::size_t t = 0; t < p.deflated.size(); ++t) deflated[t] = p.deflated[t].second;
        *k_out = static_cast<int>(p.d_active.size());
        *nrot_out = static_cast<int>(p.givens.size());
        *tol_out = p.tol;
        return 0;
    } catch (const std::exception& ex) {
        return code_of(ex);
    }
}

int brref_refreshed_weights(int k, const double* d, const double* z, double rho,
                            const int* origin, const double* tau, double* zhat) {
    try {
        br::SecularProblem P{std::vector<double>(d, d + k), std::vector<double>(z, z + k), rho};
        std::vector<br::CompactRoot> roots(static_cast<std::size_t>(k));
        for (int j = 0; j < k; ++j) {
            roots[j].origin_index = origin[j];
            roots[j].tau = tau[j];
        }
        std::vector<double> w = br::refreshed_weights(P, roots);
        std::memcpy(zhat, w.data(), sizeof(double) * w.size());
        return 0;
    } catch (const std::exception& ex) {
        return code_of(ex);
    }
}

}  // extern "C"
