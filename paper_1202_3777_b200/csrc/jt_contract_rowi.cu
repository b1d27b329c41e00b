// Row-per-i contraction launchers (plain, long-K, i-grouped, parameter-space) and the
// contraction dispatchers.
#include <cstdlib>

#include "jt_contract.cuh"

namespace jt {

cudaError_t launch_contract_tile(int dtype, int fold, int ng, const CArgs& a, int grid, cudaStream_t s);
int contract_tile_max_ctas_per_sm(int dtype, int fold, int ng);

#define ROWIP_DECL(T)                                                                                          \
  cudaError_t launch_contract_rowi_param_##T(int fold, int longk, int ng, const CArgs& a, const RowiParam& rp,    \
                                             int grid, cudaStream_t s, bool xw, int kp);                         \
  int contract_rowi_param_max_ctas_##T(int fold, int longk, int ng, bool xw, int kp);
ROWIP_DECL(float)
ROWIP_DECL(double)
ROWIP_DECL(floatv)
ROWIP_DECL(doublev)
#undef ROWIP_DECL

// row-per-i kernels with the output kinds fixed at compile time (JT_ROWI_KP=0: off)
static int rowi_kind_pattern(int ka, int kb) {
  static const int on = getenv("JT_ROWI_KP") ? atoi(getenv("JT_ROWI_KP")) : 1;
  if (!on) return 0;
  if (ka == OUT_SEP_FRESH && kb == OUT_NONE) return 1;
  if (ka == OUT_SEP_DFRESH && kb == OUT_SEP_DRATIO) return 2;
  if (ka == OUT_SEP_DRATIO && kb == OUT_NONE) return 3;
  return 0;
}

// JT_ROWI_NGC=0: the descriptor-driven kernel for every factor count (A/B switch)
static int rowi_ngc(int ng) {
  static const int on = getenv("JT_ROWI_NGC") ? atoi(getenv("JT_ROWI_NGC")) : 1;
  return on ? ng : 0;
}

// xw: paired short-K passes that also write the clique's product X; vs: the pass
// reads virtual separators
cudaError_t launch_contract_rowi_param(int dtype, int fold, int longk, const CArgs& a, const RowiParam& rp, int grid,
                                       cudaStream_t s, bool xw, bool vs) {
  if (grid <= 0 || a.n_units <= 0) return cudaSuccess;
  const int ng = rowi_ngc(rp.cp.nG);
  const int kp = rowi_kind_pattern(rp.cp.out_kind, rp.cp.out_kind_b);
  if (vs)
    return dtype == 0 ? launch_contract_rowi_param_floatv(fold, longk, ng, a, rp, grid, s, xw, kp)
                      : launch_contract_rowi_param_doublev(fold, longk, ng, a, rp, grid, s, xw, kp);
  return dtype == 0 ? launch_contract_rowi_param_float(fold, longk, ng, a, rp, grid, s, xw, kp)
                    : launch_contract_rowi_param_double(fold, longk, ng, a, rp, grid, s, xw, kp);
}

int contract_rowi_param_max_ctas(int dtype, int fold, int longk, int ng, bool xw, bool vs, int ka, int kb) {
  ng = rowi_ngc(ng);
  const int kp = rowi_kind_pattern(ka, kb);
  if (vs)
    return dtype == 0 ? contract_rowi_param_max_ctas_floatv(fold, longk, ng, xw, kp)
                      : contract_rowi_param_max_ctas_doublev(fold, longk, ng, xw, kp);
  return dtype == 0 ? contract_rowi_param_max_ctas_float(fold, longk, ng, xw, kp)
                    : contract_rowi_param_max_ctas_double(fold, longk, ng, xw, kp);
}

template <typename T, bool FOLD, bool LONGK>
static cudaError_t launch_rowi_t(bool vs, const CArgs& a, int grid, cudaStream_t s) {
  return vs ? launch_pdl(contract_rowi_kernel<T, FOLD, LONGK, true>, grid, NT, 0, s, a)
            : launch_pdl(contract_rowi_kernel<T, FOLD, LONGK, false>, grid, NT, 0, s, a);
}

cudaError_t launch_contract(int dtype, int fold, int rowi, int ng, const CArgs& a, int grid, cudaStream_t s, bool vs) {
  if (grid <= 0 || a.n_units <= 0) return cudaSuccess;
  if (vs && rowi != 1 && rowi != 4) return cudaErrorInvalidValue;
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
      return rowi == 4 ? (fold ? launch_rowi_t<float, true, true>(vs, a, grid, s)
                               : launch_rowi_t<float, false, true>(vs, a, grid, s))
             : fold ? launch_rowi_t<float, true, false>(vs, a, grid, s)
                    : launch_rowi_t<float, false, false>(vs, a, grid, s);
    return rowi == 4 ? launch_rowi_t<double, false, true>(vs, a, grid, s)
                     : launch_rowi_t<double, false, false>(vs, a, grid, s);
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
