// brgpu.hpp -- header-only C++ wrapper over the C ABI (brgpu.h).
//
// Mirrors the reference's C++ surface for this path:
//   std::vector<double> br::eigenvalues_qrql(const TridiagonalMatrix&)   (inc/qrql.hpp:20-23)
//   br_eigenvalues(T, threads) -> BrResult{lambda, ledger}
// and rethrows the matching exception class of inc/errors.hpp:9-60.
//
// Define BRGPU_USE_BR_ERRORS *after* including "br/errors.hpp" to throw the
// reference's own br::Error subclasses; otherwise brgpu:: mirrors with the same
// names are thrown.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "brgpu.h"

namespace brgpu {

#ifdef BRGPU_USE_BR_ERRORS
using Error = br::Error;
using InvalidArgument = br::InvalidArgument;
using NoConvergence = br::NoConvergence;
using BudgetExceeded = br::BudgetExceeded;
using PoleHit = br::PoleHit;
using ZeroDenominator = br::ZeroDenominator;
using MalformedCompactRoot = br::MalformedCompactRoot;
using DimensionMismatch = br::DimensionMismatch;
using DomainError = br::DomainError;
#else
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};
#define BRGPU_ERR_CLASS(N) \
    class N : public Error { \
    public: \
        explicit N(const std::string& what) : Error(what) {} \
    };
BRGPU_ERR_CLASS(InvalidArgument)
BRGPU_ERR_CLASS(NoConvergence)
BRGPU_ERR_CLASS(BudgetExceeded)
BRGPU_ERR_CLASS(PoleHit)
BRGPU_ERR_CLASS(ZeroDenominator)
BRGPU_ERR_CLASS(MalformedCompactRoot)
BRGPU_ERR_CLASS(DimensionMismatch)
BRGPU_ERR_CLASS(DomainError)
#undef BRGPU_ERR_CLASS
#endif

/// Device / CUDA / NCCL failures (no reference counterpart).
class DeviceError : public std::runtime_error {
public:
    explicit DeviceError(const std::string& what) : std::runtime_error(what) {}
};

[[noreturn]] inline void throw_status(int code, const std::string& msg) {
    switch (code) {
        case BRGPU_ERR_INVALID_ARGUMENT: throw InvalidArgument(msg);
        case BRGPU_ERR_NO_CONVERGENCE: throw NoConvergence(msg);
        case BRGPU_ERR_BUDGET_EXCEEDED: throw BudgetExceeded(msg);
        case BRGPU_ERR_POLE_HIT: throw PoleHit(msg);
        case BRGPU_ERR_ZERO_DENOMINATOR: throw ZeroDenominator(msg);
        case BRGPU_ERR_MALFORMED_COMPACT_ROOT: throw MalformedCompactRoot(msg);
        case BRGPU_ERR_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
        case BRGPU_ERR_DOMAIN_ERROR: throw DomainError(msg);
        default: throw DeviceError(msg + " (" + brgpu_status_string(code) + ")");
    }
}

/// LedgerSnapshot analogue (inc/workspace.hpp:15-26).
struct Ledger {
    std::int64_t live_doubles, peak_doubles, live_ints, peak_ints, limit_doubles, limit_ints;
    std::int64_t rows_doubles = 0, rows_ints = 0;  // requested-rows state (outside 16N / 7N)
    std::int64_t limit_bytes() const { return limit_doubles * 8 + limit_ints * 4; }
};

struct BrResult {
    std::vector<double> lambda;  // ascending
    Ledger ledger;
    /// |sigma| x n, row-major: selected_rows[r*n + j] = Q(sigma_r, j); empty if no request
    std::vector<double> selected_rows;
};

/// One handle = one device + one stream; use one Solver per host thread.
class Solver {
public:
    explicit Solver(int device = 0) {
        const int rc = brgpu_create(&h_, device);
        if (rc) throw_status(rc, "brgpu_create");
    }
    ~Solver() { brgpu_destroy(h_); }
    Solver(const Solver&) = delete;
    Solver& operator=(const Solver&) = delete;

    void set_option(int option, std::int64_t value) { check(brgpu_set_option(h_, option, value)); }

    /// All eigenvalues of tridiag(e, d, e), ascending (the eigenvalues_qrql shape).
    std::vector<double> eigenvalues(const std::vector<double>& d, const std::vector<double>& e) {
        if (d.empty()) throw InvalidArgument("tridiagonal: order must be positive");
        if (e.size() + 1 != d.size()) throw InvalidArgument("tridiagonal: off-diagonal length != n-1");
        std::vector<double> w(d.size());
        check(brgpu_eigvals(h_, static_cast<std::int64_t>(d.size()), d.data(),
                            e.empty() ? nullptr : e.data(), w.data()));
        return w;
    }

    /// Any matrix type with members d and e (e.g. br::TridiagonalMatrix).
    template <class TM>
    std::vector<double> eigenvalues(const TM& t) {
        return eigenvalues(t.d, t.e);
    }

    template <class TM>
    BrResult br_eigenvalues(const TM& t) {
        BrResult r;
        r.lambda = eigenvalues(t.d, t.e);
        brgpu_ledger l;
        check(brgpu_get_ledger(h_, &l));
        r.ledger = Ledger{l.live_doubles, l.peak_doubles, l.live_ints, l.peak_ints, l.limit_doubles,
                          l.limit_ints, l.rows_doubles, l.rows_ints};
        return r;
    }

    /// Algorithm 1 with a row request: eigenvalues plus rows Q(sigma_r, :) (0-based
    /// row indices, duplicates and any order allowed).
    template <class TM>
    BrResult br_eigenvalues(const TM& t, const std::vector<std::int64_t>& sigma) {
        if (t.d.empty()) throw InvalidArgument("tridiagonal: order must be positive");
        if (t.e.size() + 1 != t.d.size()) throw InvalidArgument("tridiagonal: off-diagonal length != n-1");
        BrResult r;
        const std::int64_t n = static_cast<std::int64_t>(t.d.size());
        r.lambda.resize(t.d.size());
        r.selected_rows.resize(sigma.size() * t.d.size());
        check(brgpu_eigvals_rows(h_, n, t.d.data(), t.e.empty() ? nullptr : t.e.data(),
                                 static_cast<std::int64_t>(sigma.size()), sigma.empty() ? nullptr : sigma.data(),
                                 r.lambda.data(), sigma.empty() ? nullptr : r.selected_rows.data()));
        brgpu_ledger l;
        check(brgpu_get_ledger(h_, &l));
        r.ledger = Ledger{l.live_doubles, l.peak_doubles, l.live_ints, l.peak_ints, l.limit_doubles,
                          l.limit_ints, l.rows_doubles, l.rows_ints};
        return r;
    }

    brgpu_handle* handle() const { return h_; }

private:
    void check(int rc) {
        if (rc) throw_status(rc, brgpu_last_error_message(h_));
    }
    brgpu_handle* h_ = nullptr;
};

/// The calling thread's default solver on device 0 (one handle = one device +
/// one stream per host thread, created on first use).
inline Solver& thread_solver() {
    static thread_local Solver solver(0);
    return solver;
}

/// Free function with the exact shape of br::eigenvalues_qrql
/// (inc/qrql.hpp:20-23): all eigenvalues of T, ascending, same exceptions.
/// TM is any matrix type with members d (n) and e (n-1), e.g. br::TridiagonalMatrix.
template <class TM>
std::vector<double> eigenvalues(const TM& t) {
    return thread_solver().eigenvalues(t.d, t.e);
}

/// SPEC.md:348-356 br_eigenvalues(T) -> BrResult{lambda, ledger}.
template <class TM>
BrResult br_eigenvalues(const TM& t) {
    return thread_solver().br_eigenvalues(t);
}

/// ... with Algorithm 1's requested rows sigma (0-based).
template <class TM>
BrResult br_eigenvalues(const TM& t, const std::vector<std::int64_t>& sigma) {
    return thread_solver().br_eigenvalues(t, sigma);
}

}  // namespace brgpu
