// tilesim/gate.hpp -- the reference's header name, kept so translation units
// written against the reference include it unchanged.  Provides:
//   Gate, kFusedQubitCap, make_gate, make_gate_arg_order, expand_gate, fuse_matrices, wire_union (proj/include/tilesim/gate.hpp)
// The declarations live in tilesim/core.hpp (the B200 build's gatecore, one
// header); the definitions are in libtilesim_b200.so.
#pragma once

#include "tilesim/core.hpp"
