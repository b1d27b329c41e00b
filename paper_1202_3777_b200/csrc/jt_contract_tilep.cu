// Tile contraction launchers with the pass descriptor and tables in kernel parameters.
#include "jt_contract.cuh"

namespace jt {

cudaError_t launch_contract_tile_param(int dtype, int fold, int ng, const CArgs& a, const TileParam& tp, int grid,
                                       cudaStream_t s) {
  if (grid <= 0 || a.n_units <= 0) return cudaSuccess;
  if (dtype == 0 && fold)
    return by_ng<float, true>(ng, [&](auto c) { return launch_contract_p_t<float, true, decltype(c)::value>(a, tp, grid, s); });
  if (dtype == 0)
    return by_ng<float, false>(ng, [&](auto c) { return launch_contract_p_t<float, false, decltype(c)::value>(a, tp, grid, s); });
  return by_ng<double, false>(ng, [&](auto c) { return launch_contract_p_t<double, false, decltype(c)::value>(a, tp, grid, s); });
}

}  // namespace jt
