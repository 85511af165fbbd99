// Compatibility include: the reference's "krylov/csr_matrix.hpp" resolved to the
// B200 drop-in API, so the reference's own tests compile unchanged
// (tests/cpp/Makefile: ref_sparse_core).  Everything of krylov:: comes from
// include/krylov_b200 (spmv runs on the GPU).
#pragma once
#include "krylov_b200/io.hpp"
#include "krylov_b200/krylov.hpp"
namespace krylov {
using namespace krylov_b200;
}
