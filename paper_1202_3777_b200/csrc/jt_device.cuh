// Device helpers shared by the kernel translation units (jt_kernels.cu,
// jt_contract.cu): vector loads/stores, programmatic dependent launch.
#pragma once
#include "jt_internal.h"
#include <utility>

namespace jt {

template <typename T, int VEC> struct VecT;
template <> struct VecT<float, 4> { using type = float4; };
template <> struct VecT<float, 2> { using type = float2; };
template <> struct VecT<float, 1> { using type = float; };
template <> struct VecT<double, 2> { using type = double2; };
template <> struct VecT<double, 1> { using type = double; };

template <typename T, int VEC>
__device__ __forceinline__ void load_vec(const T* p, T (&v)[VEC]) {
  using V = typename VecT<T, VEC>::type;
  V x = *reinterpret_cast<const V*>(p);
  const T* xs = reinterpret_cast<const T*>(&x);
#pragma unroll
  for (int l = 0; l < VEC; ++l) v[l] = xs[l];
}

template <typename T, int VEC>
__device__ __forceinline__ void load_vec_ro(const T* p, T (&v)[VEC]) {
  using V = typename VecT<T, VEC>::type;
  V x = __ldg(reinterpret_cast<const V*>(p));
  const T* xs = reinterpret_cast<const T*>(&x);
#pragma unroll
  for (int l = 0; l < VEC; ++l) v[l] = xs[l];
}

template <typename T, int VEC>
__device__ __forceinline__ void load_vec_cs(const T* p, T (&v)[VEC]) {
  using V = typename VecT<T, VEC>::type;
  V x = __ldcs(reinterpret_cast<const V*>(p));
  const T* xs = reinterpret_cast<const T*>(&x);
#pragma unroll
  for (int l = 0; l < VEC; ++l) v[l] = xs[l];
}

template <typename T, int VEC>
__device__ __forceinline__ void store_vec(T* p, const T (&v)[VEC]) {
  using V = typename VecT<T, VEC>::type;
  V x;
  T* xs = reinterpret_cast<T*>(&x);
#pragma unroll
  for (int l = 0; l < VEC; ++l) xs[l] = v[l];
  *reinterpret_cast<V*>(p) = x;
}

template <typename T, int VEC>
__device__ __forceinline__ void store_vec_cs(T* p, const T (&v)[VEC]) {
  using V = typename VecT<T, VEC>::type;
  V x;
  T* xs = reinterpret_cast<T*>(&x);
#pragma unroll
  for (int l = 0; l < VEC; ++l) xs[l] = v[l];
  __stcs(reinterpret_cast<V*>(p), x);
}

// Programmatic dependent launch: wave kernels are launched with the
// programmatic-serialization attribute, so a kernel's CTAs may be scheduled
// while the previous wave drains; every such kernel waits for the previous
// grid's completion (griddepcontrol.wait) before touching any data and lets its
// own dependents launch right away.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}


}  // namespace jt
