// Tile contraction launchers (one pass group per launch, tables in global memory).
#include "jt_contract.cuh"

namespace jt {

cudaError_t launch_contract_tile(int dtype, int fold, int ng, const CArgs& a, int grid, cudaStream_t s) {
  if (dtype == 0 && fold)
    return by_ng<float, true>(ng, [&](auto c) { return launch_contract_t<float, true, decltype(c)::value>(a, grid, s); });
  if (dtype == 0)
    return by_ng<float, false>(ng, [&](auto c) { return launch_contract_t<float, false, decltype(c)::value>(a, grid, s); });
  return by_ng<double, false>(ng, [&](auto c) { return launch_contract_t<double, false, decltype(c)::value>(a, grid, s); });
}

int contract_tile_max_ctas_per_sm(int dtype, int fold, int ng) {
  if (dtype == 0 && fold) return by_ng<float, true>(ng, [&](auto c) { return occ_contract_t<float, true, decltype(c)::value>(); });
  if (dtype == 0) return by_ng<float, false>(ng, [&](auto c) { return occ_contract_t<float, false, decltype(c)::value>(); });
  return by_ng<double, false>(ng, [&](auto c) { return occ_contract_t<double, false, decltype(c)::value>(); });
}

}  // namespace jt
