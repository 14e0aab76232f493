// tests/cpp/dropin_main.cpp -- drives integration/br_gpu.cpp linked with the
// reference's own src/tridiagonal.cpp + src/qrql.cpp (built by oracle/Makefile
// into oracle/_ref/cpp_dropin; TEST ONLY).  For each case it prints
//   case <name> n <n> maxdiff <max|lambda_gpu - lambda_qrql|> tol <8 n eps ||T||>
// and then the exception mapping checks.  tests/test_cpp_dropin.py parses it.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "br/errors.hpp"
#include "br/qrql.hpp"
#include "br/tridiagonal.hpp"
#define BRGPU_USE_BR_ERRORS
#include "brgpu.hpp"

namespace br {
std::vector<double> eigenvalues_br_gpu(const TridiagonalMatrix& t);
}

static std::uint64_t st = 0x9E3779B97F4A7C15ull;
static double uni() {  // xorshift64*, U(-1, 1)
    st ^= st >> 12; st ^= st << 25; st ^= st >> 27;
    return 2.0 * (double)((st * 0x2545F4914F6CDD1Dull) >> 11) * 0x1p-53 - 1.0;
}

static void run_case(const char* name, std::vector<double> d, std::vector<double> e) {
    br::TridiagonalMatrix t(std::move(d), std::move(e));
    const std::vector<double> g = br::eigenvalues_br_gpu(t);
    const std::vector<double> q = br::eigenvalues_qrql(t);
    double md = 0.0;
    for (std::size_t i = 0; i < g.size(); ++i) md = std::fmax(md, std::fabs(g[i] - q[i]));
    const double tol = 8.0 * (double)t.n * 0x1p-52 * t.inf_norm();
    std::printf("case %s n %zu maxdiff %.6e tol %.6e sorted %d\n", name, t.n, md, tol,
                (int)std::is_sorted(g.begin(), g.end()));
}

int main() {
    try {
        for (std::size_t n : {1u, 2u, 7u, 26u, 100u, 1000u, 4096u}) {
            std::vector<double> d(n), e(n ? n - 1 : 0);
            for (auto& x : d) x = uni();
            for (auto& x : e) x = uni();
            char nm[32];
            std::snprintf(nm, sizeof nm, "random%zu", n);
            run_case(nm, d, e);
        }
        run_case("toeplitz121", std::vector<double>(2048, 2.0), std::vector<double>(2047, 1.0));
        {
            std::vector<double> d(2100), e(2099, 1.0);
            for (std::size_t i = 0; i < d.size(); ++i) d[i] = std::fabs((double)(i % 21) - 10.0);
            for (std::size_t i = 20; i < e.size(); i += 21) e[i] = 1e-10;
            run_case("wilkinson", d, e);
        }
        // the reference's validation runs first (src/tridiagonal.cpp:17-30) ...
        try {
            br::TridiagonalMatrix t({1.0, NAN}, {1.0});
            std::printf("no-throw-ctor\n");
        } catch (const br::InvalidArgument&) {
            std::printf("ctor-invalid-argument\n");
        }
        // ... and a non-finite entry that reaches the GPU maps to br::InvalidArgument
        try {
            br::TridiagonalMatrix t;
            t.n = 3; t.d = {1.0, INFINITY, 2.0}; t.e = {0.5, 0.5};
            brgpu::eigenvalues(t);
            std::printf("no-throw-gpu\n");
        } catch (const br::InvalidArgument&) {
            std::printf("gpu-invalid-argument\n");
        }
        // SPEC.md:348-356 br_eigenvalues(T) with the ledger, and requested rows
        br::TridiagonalMatrix t({2.0, 2.0, 2.0}, {1.0, 1.0});
        brgpu::BrResult r = brgpu::br_eigenvalues(t, std::vector<std::int64_t>{0, 2});
        std::printf("br_eigenvalues lambda %zu rows %zu ledger_ok %d\n", r.lambda.size(), r.selected_rows.size(),
                    (int)(r.ledger.peak_doubles <= r.ledger.limit_doubles));
    } catch (const brgpu::DeviceError& ex) {
        std::printf("device-error %s\n", ex.what());
        return 3;
    }
    std::printf("done\n");
    return 0;
}
