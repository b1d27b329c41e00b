// Parameter-space row-per-i launchers, one translation unit per dtype
// (jt_contract_rowip32.cu / jt_contract_rowip64.cu): the factor count per k is a
// compile-time constant for nG <= 4, so the k loop issues exactly nG vector
// loads per k (no per-factor predicates) — see rowi_body.
#pragma once
#include "jt_contract.cuh"

namespace jt {

template <typename T, bool FOLD, bool LONGK, bool XW, bool VS, int KP = 0>
static auto rowi_p_fn(int ng) {
  switch (ng) {
    case 1: return contract_rowi_p_kernel<T, FOLD, LONGK, XW, 1, VS, KP>;
    case 2: return contract_rowi_p_kernel<T, FOLD, LONGK, XW, 2, VS, KP>;
    case 3: return contract_rowi_p_kernel<T, FOLD, LONGK, XW, 3, VS, KP>;
    case 4: return contract_rowi_p_kernel<T, FOLD, LONGK, XW, 4, VS, KP>;
    default: return contract_rowi_p_kernel<T, FOLD, LONGK, XW, 0, VS, KP>;
  }
}

// ng <= 0: the generic (descriptor-driven) kernel; kp (short K, unfolded): the
// output-kind pattern fixed at compile time (rowi_body KP; 2 for VS kernels only)
template <typename T, bool VS>
static void (*rowi_p_select(int fold, int longk, int ng, bool xw, int kp = 0))(const CArgs, const RowiParam) {
  if (kp && !fold && !longk) {
    if (kp == 1 && !xw) return rowi_p_fn<T, false, false, false, VS, 1>(ng);
    if (kp == 3 && !xw) return rowi_p_fn<T, false, false, false, VS, 3>(ng);
    if constexpr (VS)
      if (kp == 2) return xw ? rowi_p_fn<T, false, false, true, VS, 2>(ng) : rowi_p_fn<T, false, false, false, VS, 2>(ng);
  }
  if (xw) {
    if (longk) return nullptr;
    if constexpr (sizeof(T) == 4)
      return fold ? rowi_p_fn<T, true, false, true, VS>(ng) : rowi_p_fn<T, false, false, true, VS>(ng);
    else return rowi_p_fn<T, false, false, true, VS>(ng);
  }
  if constexpr (sizeof(T) == 4) {
    if (fold) return longk ? rowi_p_fn<T, true, true, false, VS>(ng) : rowi_p_fn<T, true, false, false, VS>(ng);
  }
  return longk ? rowi_p_fn<T, false, true, false, VS>(ng) : rowi_p_fn<T, false, false, false, VS>(ng);
}

}  // namespace jt
