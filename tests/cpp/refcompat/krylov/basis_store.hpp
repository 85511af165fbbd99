// Compatibility include: the reference's "krylov/basis_store.hpp" resolved to the
// B200 drop-in API (plus the test inputs of refcompat_support.hpp), so the
// reference's own tests/test_block_ortho.cpp compiles unchanged
// (tests/cpp/Makefile: ref_block_ortho).
#pragma once
#include "../refcompat_support.hpp"
