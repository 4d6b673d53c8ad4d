// tilesim/ir.hpp -- circuit IR, named-gate lowering, text format, generators.
//
// Reference surface:
//   Circuit, make_named_gate, named_gate_arity/param_count  proj/include/tilesim/circuit.hpp:12-27
//   parse_circuit / serialize_circuit / load / save          proj/include/tilesim/circuit.hpp:29-43
//   gen_benchmark (QFT ALA RQC QVC IQP HES)                  SPEC.md:170-178 (SPEC-only)
// plus QAOA MaxCut (BASELINE.json configs[2]); recipes pinned in DESIGN.md §3.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "tilesim/core.hpp"

namespace tilesim {

struct Circuit {
  int n_qubits = 0;
  std::vector<Gate> gates;  // program order == application order
};

Gate make_named_gate(const std::string& name, const std::vector<double>& params, const std::vector<int>& qubits);
int named_gate_arity(const std::string& name);        // 0 if unknown
int named_gate_param_count(const std::string& name);

Circuit parse_circuit(const std::string& text);        // throws ParseError
std::string serialize_circuit(const Circuit& c);
Circuit load_circuit_file(const std::string& path);
void save_circuit_file(const Circuit& c, const std::string& path);

enum class BenchmarkKind { QFT, ALA, RQC, QVC, IQP, HES, QAOA };
BenchmarkKind parse_benchmark_kind(const std::string& s);  // throws ConfigError
Circuit gen_benchmark(BenchmarkKind kind, int n, int depth, uint64_t seed);

}  // namespace tilesim
