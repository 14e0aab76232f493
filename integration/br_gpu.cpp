// integration/br_gpu.cpp -- the one file a reference maintainer adds to the
// reference tree to get a drop-in for
// br::eigenvalues_qrql (proj/include/br/qrql.hpp:20-23) backed by the B200 BR
// solver: same signature, same ascending output, the reference's own
// br::Error subclasses.  tests/test_cpp_dropin.py compiles it together with
// the reference's src/tridiagonal.cpp and src/qrql.cpp (oracle/Makefile) and
// checks it against br::eigenvalues_qrql on the GPU.
#include "br/errors.hpp"
#include "br/qrql.hpp"
#include "br/tridiagonal.hpp"
#define BRGPU_USE_BR_ERRORS  // rethrow br::InvalidArgument, br::NoConvergence, ...
#include "brgpu.hpp"         // this repository's include/

namespace br {

// Drop-in for eigenvalues_qrql: same signature, same ascending output, same exceptions.
std::vector<double> eigenvalues_br_gpu(const TridiagonalMatrix& t) {
    t.validate();                   // src/tridiagonal.cpp:17-30
    return brgpu::eigenvalues(t);   // one solver handle (device 0 + stream) per host thread
}

}  // namespace br
