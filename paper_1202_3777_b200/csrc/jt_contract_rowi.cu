// Row-per-i contraction launchers (plain, long-K, i-grouped, parameter-space) and the
// contraction dispatchers.
#include "jt_contract.cuh"

namespace jt {

cudaError_t launch_contract_tile(int dtype, int fold, int ng, const CArgs& a, int grid, cudaStream_t s);
int contract_tile_max_ctas_per_sm(int dtype, int fold, int ng);

cudaError_t launch_contract_rowi_param(int dtype, int fold, int longk, const CArgs& a, const RowiParam& rp, int grid,
                                       cudaStream_t s, bool xw) {
  if (grid <= 0 || a.n_units <= 0) return cudaSuccess;
  if (xw) {  // paired short-K passes that also write the clique's product X
    if (longk) return cudaErrorInvalidValue;
    if (dtype == 0)
      return fold ? launch_pdl(contract_rowi_p_kernel<float, true, false, true>, grid, NT, 0, s, a, rp)
                  : launch_pdl(contract_rowi_p_kernel<float, false, false, true>, grid, NT, 0, s, a, rp);
    return launch_pdl(contract_rowi_p_kernel<double, false, false, true>, grid, NT, 0, s, a, rp);
  }
  if (dtype == 0) {
    if (fold)
      return longk ? launch_pdl(contract_rowi_p_kernel<float, true, true>, grid, NT, 0, s, a, rp)
                   : launch_pdl(contract_rowi_p_kernel<float, true, false>, grid, NT, 0, s, a, rp);
    return longk ? launch_pdl(contract_rowi_p_kernel<float, false, true>, grid, NT, 0, s, a, rp)
                 : launch_pdl(contract_rowi_p_kernel<float, false, false>, grid, NT, 0, s, a, rp);
  }
  return longk ? launch_pdl(contract_rowi_p_kernel<double, false, true>, grid, NT, 0, s, a, rp)
               : launch_pdl(contract_rowi_p_kernel<double, false, false>, grid, NT, 0, s, a, rp);
}

cudaError_t launch_contract(int dtype, int fold, int rowi, int ng, const CArgs& a, int grid, cudaStream_t s) {
  if (grid <= 0 || a.n_units <= 0) return cudaSuccess;
  if (rowi == 2 || rowi == 3) {  // i-groups: IGM 4 (rowi 2) or 8 (rowi 3)
    if (dtype == 0) {
      if (fold)
        return rowi == 2 ? launch_pdl(contract_rowg_kernel<float, true, 4>, grid, NT, 0, s, a)
                         : launch_pdl(contract_rowg_kernel<float, true, 8>, grid, NT, 0, s, a);
      return rowi == 2 ? launch_pdl(contract_rowg_kernel<float, false, 4>, grid, NT, 0, s, a)
                       : launch_pdl(contract_rowg_kernel<float, false, 8>, grid, NT, 0, s, a);
    }
    return rowi == 2 ? launch_pdl(contract_rowg_kernel<double, false, 4>, grid, NT, 0, s, a)
                     : launch_pdl(contract_rowg_kernel<double, false, 8>, grid, NT, 0, s, a);
  }
  if (rowi) {
    if (dtype == 0)
      return rowi == 4 ? (fold ? launch_pdl(contract_rowi_kernel<float, true, true>, grid, NT, 0, s, a)
                               : launch_pdl(contract_rowi_kernel<float, false, true>, grid, NT, 0, s, a))
             : fold ? launch_pdl(contract_rowi_kernel<float, true>, grid, NT, 0, s, a)
                    : launch_pdl(contract_rowi_kernel<float, false>, grid, NT, 0, s, a);
    return rowi == 4 ? launch_pdl(contract_rowi_kernel<double, false, true>, grid, NT, 0, s, a)
                     : launch_pdl(contract_rowi_kernel<double, false>, grid, NT, 0, s, a);
  }
  return launch_contract_tile(dtype, fold, ng, a, grid, s);
}

int contract_max_ctas_per_sm(int dtype, int fold, int rowi, int ng) {
  int n = 0;
  if (rowi == 2 || rowi == 3) {
    if (dtype == 0 && fold)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rowi == 2 ? contract_rowg_kernel<float, true, 4>
                                                                  : contract_rowg_kernel<float, true, 8>, NT, 0);
    else if (dtype == 0)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rowi == 2 ? contract_rowg_kernel<float, false, 4>
                                                                  : contract_rowg_kernel<float, false, 8>, NT, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rowi == 2 ? contract_rowg_kernel<double, false, 4>
                                                                  : contract_rowg_kernel<double, false, 8>, NT, 0);
    return n > 0 ? n : 1;
  }
  if (rowi) {
    const bool lk = rowi == 4;
    if (dtype == 0 && fold)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, lk ? contract_rowi_kernel<float, true, true>
                                                           : contract_rowi_kernel<float, true>, NT, 0);
    else if (dtype == 0)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, lk ? contract_rowi_kernel<float, false, true>
                                                           : contract_rowi_kernel<float, false>, NT, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, lk ? contract_rowi_kernel<double, false, true>
                                                           : contract_rowi_kernel<double, false>, NT, 0);
    return n > 0 ? n : 1;
  }
  return contract_tile_max_ctas_per_sm(dtype, fold, ng);
}

}  // namespace jt
