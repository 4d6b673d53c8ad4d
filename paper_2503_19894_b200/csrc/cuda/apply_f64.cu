// complex128 instantiations of the gate kernels (see kernels.cuh).
#include "apply_impl.cuh"

namespace tsg {
int launch_gate_f64(const GateLaunch& g, cudaStream_t s, int num_sms) { return launch_gate_impl<double>(g, s, num_sms); }
}  // namespace tsg
