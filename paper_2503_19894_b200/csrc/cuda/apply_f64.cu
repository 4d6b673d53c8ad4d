// complex128 instantiations of the gate kernels (see kernels*.cuh).
#include "apply_impl.cuh"

namespace tsg {
int launch_gate_f64(const GateLaunch& g, cudaStream_t s, int num_sms) { return launch_gate_impl<double>(g, s, num_sms); }
int launch_diag_batch_f64(const DiagBatchLaunch& b, cudaStream_t s, int num_sms) {
  return launch_diag_batch_impl<double>(b, s, num_sms);
}
}  // namespace tsg
