// complex64 instantiations of the gate kernels (see kernels*.cuh).
#include "apply_impl.cuh"

namespace tsg {
int launch_gate_f32(const GateLaunch& g, cudaStream_t s, int num_sms) { return launch_gate_impl<float>(g, s, num_sms); }
int launch_diag_batch_f32(const DiagBatchLaunch& b, cudaStream_t s, int num_sms) {
  return launch_diag_batch_impl<float>(b, s, num_sms);
}

std::string kernel_name(const GateLaunch& g, int precision_bits) {
  return precision_bits == 64 ? kernel_name_impl<double>(g) : kernel_name_impl<float>(g);
}
}  // namespace tsg
