// tilesim/circuit.hpp -- the reference's header name, kept so translation
// units written against the reference include it unchanged.  Provides:
//   Circuit, make_named_gate, named_gate_arity, named_gate_param_count,
//   parse_circuit, serialize_circuit, load_circuit_file, save_circuit_file
//   (proj/include/tilesim/circuit.hpp:12-43), plus gen_benchmark
// The declarations live in tilesim/ir.hpp; the definitions are in
// libtilesim_b200.so.
#pragma once

#include "tilesim/ir.hpp"
