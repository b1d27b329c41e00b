// Parameter-space row-per-i contraction kernels, float (see jt_contract_rowip.cuh).
#include "jt_contract_rowip.cuh"

namespace jt {

cudaError_t launch_contract_rowi_param_float(int fold, int longk, int ng, const CArgs& a, const RowiParam& rp,
                                          int grid, cudaStream_t s, bool xw, int kp) {
  auto k = rowi_p_select<float, false>(fold, longk, ng, xw, kp);
  if (!k) return cudaErrorInvalidValue;
  return launch_pdl(k, grid, NT, 0, s, a, rp);
}

int contract_rowi_param_max_ctas_float(int fold, int longk, int ng, bool xw, int kp) {
  auto k = rowi_p_select<float, false>(fold, longk, ng, xw, kp);
  int n = 0;
  if (k) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, NT, 0);
  return n > 0 ? n : 1;
}

}  // namespace jt
