// complex128 instantiations of the gate kernels (see kernels*.cuh).
#include "apply_impl.cuh"
#include "pass_jit.hpp"

namespace tsg {
namespace {
template <int KS>
bool dmma_jit_spec_ks(const GateLaunch& g, std::string* source, std::string* name) {
  DmmaSetup<double, KS> st;
  if (!dmma_setup<double, KS>(g, st)) return false;
  // Measured on RQC-30's 5-qubit gates (profiles/r02/dmma_jit_ab.txt): the
  // compiled-in masks win where a third to two thirds of the tiles are
  // nonzero (40-48 of 96: 0.1-0.7 ms faster, FP64 work halved without the
  // runtime predicates), and lose at a quarter (24 of 96, HBM-bound: +0.1-0.5 ms)
  // and near-dense (88 of 96: +0.9 ms): one code path per row block costs
  // more than the skipped work saves there.
  const int all = 3 * DShape<double, KS>::RB * DShape<double, KS>::KST;
  const char* mode = std::getenv("TSG_DMMA_JIT");  // "2": every launch with a zero tile (experiments)
  const bool every = mode && mode[0] == '2';
  if (st.nonzero == all || (!every && (3 * st.nonzero < all || 3 * st.nonzero > 2 * all))) return false;
  *source = dmma_jit_source(KS, st.stages, st.p.nzblk, st.tpose, name);
  return true;
}
}  // namespace

bool dmma_jit_spec(const GateLaunch& g, std::string* source, std::string* name) {
  if (!g.full_range || (g.klass != 2 && g.klass != 3) || !g.m_re || dmma_mode() == 1) return false;
  switch (g.ks) {
    case 3: return dmma_jit_spec_ks<3>(g, source, name);
    case 4: return dmma_jit_spec_ks<4>(g, source, name);
    case 5: return dmma_jit_spec_ks<5>(g, source, name);
    default: return false;
  }
}

int launch_gate_f64(const GateLaunch& g, cudaStream_t s, int num_sms) { return launch_gate_impl<double>(g, s, num_sms); }
int launch_diag_batch_f64(const DiagBatchLaunch& b, cudaStream_t s, int num_sms) {
  return launch_diag_batch_impl<double>(b, s, num_sms);
}
}  // namespace tsg
