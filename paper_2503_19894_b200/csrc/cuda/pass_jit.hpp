// JIT-compiled tile passes (pass_jit.cu): host interface.
#pragma once

#include <string>

#include "gate_launch.hpp"

namespace tsg {

// JIT on for passes over states of at least TSG_PASS_JIT_MIN_N qubits, unless TSG_PASS_JIT=0
bool pass_jit_enabled(int n_qubits);
// CUDA source of the pass whose op table is ops[0, n_ops); *name = its kernel name (hash)
std::string pass_jit_source(int precision_bits, const PassOp* ops, int n_ops, std::string* name);
// compile (or fetch from the disk cache) without loading: no device needed
void pass_jit_cubin(const std::string& source, const std::string& name);
// compile (or fetch from the caches) and load; returns a cudaKernel_t usable as a launch handle
const void* pass_jit_kernel(const std::string& source, const std::string& name);

}  // namespace tsg
