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

// CUDA source of a complex128 k_stream_dmma product with its nonzero 8 x 4
// tiles of [Mr | Mi | Mr + Mi] compiled in (DmmaStaticNz); *name = its kernel name
std::string dmma_jit_source(int ks, int stages, const uint32_t nz[3], bool tpose, std::string* name);
// The JIT source of a full-range complex128 launch that takes the DMMA
// stream kernel and has at least one zero tile; false otherwise (apply_f64.cu)
bool dmma_jit_spec(const GateLaunch& g, std::string* source, std::string* name);
// JIT DMMA products on (n >= TSG_PASS_JIT_MIN_N, unless TSG_PASS_JIT=0 or TSG_DMMA_JIT=0)
bool dmma_jit_enabled(int n_qubits);

}  // namespace tsg
