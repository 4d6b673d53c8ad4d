// tilesim/complex_matrix.hpp -- the reference's header name, kept so translation units
// written against the reference include it unchanged.  Provides:
//   ScalarKind, classify_scalar, GateMatrix, SparsityProfile, op_count, sparsity_profile, is_unitary, random_unitary (proj/include/tilesim/complex_matrix.hpp)
// The declarations live in tilesim/core.hpp (the B200 build's gatecore, one
// header); the definitions are in libtilesim_b200.so.
#pragma once

#include "tilesim/core.hpp"
