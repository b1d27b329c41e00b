// Persistent single-launch propagation for small single trees (sm_100a).
//
// Small junction trees (c1 12 cliques, c2 368, c4M 870) are
// latency-bound: every wave moves a few KB to a few MB and the cost is the
// chain of dependent steps, not bandwidth.  Here the whole collect+distribute
// program is ONE cooperative launch; its waves are separated by a grid barrier
// and every pass is a "tiny pass" (jt_internal.h): one thread per separator
// entry walks the entry's row of the clique (Alg. 1 step 1, the row sum of
// _pass_block, propagate.py:67) multiplying the pass's factors in on the fly
// (children's ratios, parent ratio), writes the clique back when the pass owns
// the write (propagate.py:74-75), and applies the Hugin update to its entry
// (ratio = new/old, 0/0 = 0, nonzero/0 flagged; propagate.py:68-76).  Long
// rows are split over a group of 2..32 lanes (lane chunks in order + a fixed
// shuffle tree: deterministic), so no lane waits on more than a few L2 round
// trips per wave.  Every offset is stride arithmetic over merged mixed-radix
// dims (potential.py:42-63) -- no index maps, no block tables.
#include "jt_internal.h"

namespace jt {

__device__ __forceinline__ unsigned tiny_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier: arrive counter + generation word; the last CTA to arrive
// resets the counter and bumps the generation.  The fences order every table
// write of a wave before any read of the next (all loads below are coherent:
// tables change between the waves of the launch).
__device__ __forceinline__ void tiny_grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = tiny_ld_acquire(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (tiny_ld_acquire(bar + 1) == gen) __nanosleep(8);
    }
    __threadfence();
  }
  __syncthreads();
}

// oldv: the entry's current separator value, loaded before the row walk (one
// L2 round trip fewer on the wave's critical path)
template <typename T>
__device__ __forceinline__ void tiny_finalize(const TPass& P, int64_t j, double star, T* aux, double* qout, int* err,
                                              T oldv) {
  if (P.out_kind == OUT_SEP_FRESH) {
    aux[P.out_off + j] = (T)star;
  } else if (P.out_kind == OUT_SEP_DFRESH) {
    const double c = (double)oldv;
    aux[P.ratio_off + j] = (T)(c != 0.0 ? star : 0.0);
    aux[(P.out2_off >= 0 ? P.out2_off : P.out_off) + j] = (T)(c * star);
  } else if (P.out_kind == OUT_SEP) {
    const double old = (double)oldv;
    if (old == 0.0 && star != 0.0) atomicOr(err, EB_INCONSISTENT);
    aux[P.ratio_off + j] = (T)((old != 0.0) ? star / old : 0.0);
    aux[(P.out2_off >= 0 ? P.out2_off : P.out_off) + j] = (T)star;
  } else if (P.out_kind == OUT_RAW) {
    qout[P.out_off + j] = star;
  }
}

// n / d and n % d for n < 2^31 by multiply-high with a host-built magic number
__device__ __forceinline__ int tiny_div(int n, unsigned mul, int shr) {
  return (int)((__umulhi((unsigned)n, mul) + (unsigned)n) >> shr);
}

// Row walk state of one lane: base offsets of its output entry plus the
// odometer at its first row position.
template <int NFM>
struct TRow {
  int so, dd, oo;
  int fo[NFM];
  int dig[TD];
};

// Decompose output entry j and row position r0 (program constants only: runs
// before the wait on the previous wave).
template <int NFM>
__device__ __forceinline__ void tiny_prep(const TPass& P, int j, int r0, TRow<NFM>& R) {
  const int nf = P.nf;
  R.so = R.dd = R.oo = 0;
#pragma unroll
  for (int f = 0; f < NFM; ++f) R.fo[f] = 0;
  int x = j;
  for (int d = P.nod - 1; d >= 0; --d) {
    const int q = tiny_div(x, P.omul[d], P.oshr[d]);
    const int dig = x - q * P.ocard[d];
    x = q;
    R.so += dig * P.osrc[d];
    R.dd += dig * P.odst[d];
    R.oo += dig * P.oout[d];
#pragma unroll
    for (int f = 0; f < NFM; ++f)
      if (f < nf) R.fo[f] += dig * P.ofac[f][d];
  }
  x = r0;
  for (int d = P.nrd - 1; d >= 0; --d) {
    const int q = tiny_div(x, P.rmul[d], P.rshr[d]);
    R.dig[d] = x - q * P.rcard[d];
    x = q;
    R.so += R.dig[d] * P.rsrc[d];
    R.dd += R.dig[d] * P.rdst[d];
#pragma unroll
    for (int f = 0; f < NFM; ++f)
      if (f < nf) R.fo[f] += R.dig[d] * P.rfac[f][d];
  }
}

// Sum (and optionally write) positions [r0, r1) of the row.  Positions go in
// batches of TB: the odometer first produces every offset of the batch (32-bit
// integer work only), then all loads of the batch issue back to back, so a lane
// waits for one L2 round trip per batch, not per position.
constexpr int TB = 4;
template <typename T, int NFM>
__device__ __forceinline__ double tiny_exec(const TPass& P, const T* __restrict__ src, T* __restrict__ dst,
                                            const T* __restrict__ aux, TRow<NFM>& R, int r0, int r1) {
  const int nf = P.nf;
  if (r0 >= r1) return 0.0;
  const bool wr = P.dst_off >= 0;
  const T* __restrict__ fb[NFM];
#pragma unroll
  for (int f = 0; f < NFM; ++f) fb[f] = aux + (f < nf ? P.fac_off[f] : 0);
  const int d0 = P.nrd - 1;  // innermost row dim: its step needs no carry most of the time
  const int c0 = d0 >= 0 ? P.rcard[d0] : 1;
  const int s0 = d0 >= 0 ? P.rsrc[d0] : 0, t0 = d0 >= 0 ? P.rdst[d0] : 0;
  int f0[NFM];
#pragma unroll
  for (int f = 0; f < NFM; ++f) f0[f] = (d0 >= 0 && f < nf) ? P.rfac[f][d0] : 0;
  int so = R.so, dd = R.dd;
  int fo[NFM];
#pragma unroll
  for (int f = 0; f < NFM; ++f) fo[f] = R.fo[f];
  double acc = 0.0;
  for (int rb = r0; rb < r1; rb += TB) {
    const int nb = r1 - rb < TB ? r1 - rb : TB;
    int bs[TB], bd[TB], bf[NFM][TB];
#pragma unroll
    for (int q = 0; q < TB; ++q) {
      bs[q] = so;
      bd[q] = dd;
#pragma unroll
      for (int f = 0; f < NFM; ++f) bf[f][q] = fo[f];
      if (q < nb && d0 >= 0) {
        // odometer step over the row dims (last fastest)
        so += s0;
        dd += t0;
#pragma unroll
        for (int f = 0; f < NFM; ++f) fo[f] += f0[f];
        if (++R.dig[d0] == c0) {
          so -= c0 * s0;
          dd -= c0 * t0;
#pragma unroll
          for (int f = 0; f < NFM; ++f) fo[f] -= c0 * f0[f];
          R.dig[d0] = 0;
          for (int d = d0 - 1; d >= 0; --d) {
            so += P.rsrc[d];
            dd += P.rdst[d];
#pragma unroll
            for (int f = 0; f < NFM; ++f)
              if (f < nf) fo[f] += P.rfac[f][d];
            if (++R.dig[d] < P.rcard[d]) break;
            const int c = P.rcard[d];
            so -= c * P.rsrc[d];
            dd -= c * P.rdst[d];
#pragma unroll
            for (int f = 0; f < NFM; ++f)
              if (f < nf) fo[f] -= c * P.rfac[f][d];
            R.dig[d] = 0;
          }
        }
      }
    }
    T v[TB];
#pragma unroll
    for (int q = 0; q < TB; ++q) v[q] = q < nb ? src[bs[q]] : (T)0;
#pragma unroll
    for (int f = 0; f < NFM; ++f) {
      if (f < nf) {
#pragma unroll
        for (int q = 0; q < TB; ++q)
          if (q < nb) v[q] *= fb[f][bf[f][q]];
      }
    }
#pragma unroll
    for (int q = 0; q < TB; ++q) {
      if (q < nb) {
        if (wr) dst[bd[q]] = v[q];
        acc += (double)v[q];
      }
    }
  }
  return acc;
}

// One wave: every thread finds its pass (binary search over the wave's compact
// unit0 list), decomposes its entry and row start, and -- with PDL -- only then
// waits for the previous wave: descriptor reads and index math overlap the
// previous kernel's tail.
// One lane's unit of a wave: its pass, output entry, row chunk and the row
// walk's start state -- all from program constants (descriptor reads and index
// math), so it can be prepared before the previous wave's writes are visible.
template <int NFM>
struct TinyLane {
  const TPass* P;
  int G, sub, r0, r1;
  bool in, live;
  TRow<NFM> R;
};

template <int NFM>
__device__ __forceinline__ void tiny_lane_prep(const TinyArgs& a, int w, int64_t t, TinyLane<NFM>& L) {
  const TinyWave tw = a.waves[w];
  const TPass* __restrict__ ps = a.passes + tw.pass0;
  const int64_t* __restrict__ u0 = a.unit0s + tw.pass0;
  L.in = t < tw.n_threads;
  int lo = 0;
  if (L.in) {
    int hi = tw.n_passes - 1;
    while (lo < hi) {
      const int m = (lo + hi + 1) >> 1;
      if (__ldg(u0 + m) <= t) lo = m;
      else hi = m - 1;
    }
  }
  L.P = ps + lo;
  const TPass& P = *L.P;
  const int u = L.in ? (int)(t - __ldg(u0 + lo)) : 0;
  // P.warp = lanes per output entry (1, 2, 4, 8, 16 or 32): lane chunks of the
  // row in lane order, then a fixed shuffle tree inside the lane group
  L.G = L.in ? P.warp : 1;
  const int j = u / L.G;
  L.sub = u - j * L.G;
  L.live = L.in && j < P.n_out;  // lanes of the pass's padding compute nothing
  const int nr = L.live ? (int)P.n_rest : 0;
  const int per = (nr + L.G - 1) / L.G;
  L.r0 = L.live ? L.sub * per : 0;
  L.r1 = L.live ? (L.r0 + per < nr ? L.r0 + per : nr) : 0;
  if (L.live) tiny_prep<NFM>(P, j, L.r0, L.R);
}

// The data part: row loads, the lane-group shuffle tree, the Hugin update.
template <typename T, int NFM>
__device__ __forceinline__ void tiny_lane_exec(const TinyArgs& a, TinyLane<NFM>& L) {
  T* __restrict__ clique = reinterpret_cast<T*>(a.clique);
  const T* __restrict__ base = reinterpret_cast<const T*>(a.base);
  T* __restrict__ aux = reinterpret_cast<T*>(a.aux);
  const TPass& P = *L.P;
  const T* src = (P.src_arena == A_BASE ? base : P.src_arena == A_AUX ? aux : clique) + P.src_off;
  T* dst = clique + (P.dst_off >= 0 ? P.dst_off : 0);
  const bool fin = L.live && L.sub == 0 && P.out_kind != OUT_NONE;
  T oldv = (T)0;
  if (fin && (P.out_kind == OUT_SEP || P.out_kind == OUT_SEP_DFRESH)) oldv = aux[P.out_off + L.R.oo];
  double s = L.live ? tiny_exec<T, NFM>(P, src, dst, aux, L.R, L.r0, L.r1) : 0.0;
  for (int o = 1; o < L.G; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (fin) tiny_finalize<T>(P, L.R.oo, s, aux, a.qout, a.err, oldv);
}

// One wave, grid-stride over its units; with PDL the first unit is prepared
// before the wait on the previous wave, overlapping that kernel's tail.
template <typename T, int NFM, bool PDL>
__device__ __forceinline__ void tiny_wave(const TinyArgs& a, int w) {
  const int64_t stride = (int64_t)gridDim.x * NT;
  const int64_t n = a.waves[w].n_threads;
  bool waited = !PDL;
  for (int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x; t < n || !waited; t += stride) {
    TinyLane<NFM> L;
    tiny_lane_prep<NFM>(a, w, t, L);
    if (!waited) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      waited = true;
    }
    if (!L.in) break;
    tiny_lane_exec<T, NFM>(a, L);
  }
}

// every wave in one cooperative launch, grid barriers between waves
template <typename T, int NFM>
__global__ void __launch_bounds__(NT, 2) tiny_persist_kernel(const TinyArgs a) {
  for (int w = 0; w < a.n_waves; ++w) {
    tiny_wave<T, NFM, false>(a, w);
    if (w + 1 < a.n_waves) tiny_grid_barrier(a.bar);
  }
}

// one wave per launch (programmatic dependent launch chains the waves; the
// program is replayed as a CUDA graph)
template <typename T, int NFM>
__global__ void __launch_bounds__(NT, 2) tiny_wave_kernel(const TinyArgs a, int w) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  tiny_wave<T, NFM, true>(a, w);
}

// The whole program in ONE thread-block cluster (<= 16 CTAs): waves separated
// by the hardware cluster barrier (release/acquire at cluster scope orders the
// global-memory tables between waves) -- for trees whose every wave fits a
// cluster's threads, where a grid barrier or a launch per wave costs more than
// the wave itself.
template <typename T, int NFM>
__global__ void __launch_bounds__(NT, 1) tiny_cluster_kernel(const TinyArgs a) {
  // every wave fits the cluster's threads (one unit per thread): the next
  // wave's unit is prepared while this wave's stores drain, before the barrier
  const int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  TinyLane<NFM> L;
  tiny_lane_prep<NFM>(a, 0, t, L);
  for (int w = 0; w < a.n_waves; ++w) {
    if (L.in) tiny_lane_exec<T, NFM>(a, L);
    if (w + 1 < a.n_waves) {
      tiny_lane_prep<NFM>(a, w + 1, t, L);
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
  }
}

template <typename T, int NFM>
static cudaError_t launch_tiny_cluster_t(const TinyArgs& a, int grid, cudaStream_t s) {
  auto k = tiny_cluster_kernel<T, NFM>;
  if (grid > 8) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = grid;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, a);
}

template <typename T>
static cudaError_t launch_tiny_cluster_nf(int nfm, const TinyArgs& a, int grid, cudaStream_t s) {
  if (nfm <= 2) return launch_tiny_cluster_t<T, 2>(a, grid, s);
  if (nfm <= 4) return launch_tiny_cluster_t<T, 4>(a, grid, s);
  return launch_tiny_cluster_t<T, MAXF>(a, grid, s);
}

cudaError_t launch_tiny_cluster(int dtype, int nfm, const TinyArgs& a, int grid, cudaStream_t s) {
  return dtype == 0 ? launch_tiny_cluster_nf<float>(nfm, a, grid, s)
                    : launch_tiny_cluster_nf<double>(nfm, a, grid, s);
}

template <typename T, int NFM>
static cudaError_t launch_tiny_t(const TinyArgs& a, int grid, cudaStream_t s, int* occ_out) {
  auto k = tiny_persist_kernel<T, NFM>;
  if (occ_out) {
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, NT, 0);
    *occ_out = n > 0 ? n : 1;
    return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, a);
}

template <typename T, int NFM>
static cudaError_t launch_tiny_wave_t(const TinyArgs& a, int w, int grid, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, tiny_wave_kernel<T, NFM>, a, w);
}

template <typename T>
static cudaError_t launch_tiny_wave_nf(int nfm, const TinyArgs& a, int w, int grid, cudaStream_t s) {
  if (nfm <= 2) return launch_tiny_wave_t<T, 2>(a, w, grid, s);
  if (nfm <= 4) return launch_tiny_wave_t<T, 4>(a, w, grid, s);
  return launch_tiny_wave_t<T, MAXF>(a, w, grid, s);
}

cudaError_t launch_tiny_wave(int dtype, int nfm, const TinyArgs& a, int w, int grid, cudaStream_t s) {
  return dtype == 0 ? launch_tiny_wave_nf<float>(nfm, a, w, grid, s) : launch_tiny_wave_nf<double>(nfm, a, w, grid, s);
}

template <typename T>
static cudaError_t launch_tiny_nf(int nfm, const TinyArgs& a, int grid, cudaStream_t s, int* occ_out) {
  if (nfm <= 2) return launch_tiny_t<T, 2>(a, grid, s, occ_out);
  if (nfm <= 4) return launch_tiny_t<T, 4>(a, grid, s, occ_out);
  return launch_tiny_t<T, MAXF>(a, grid, s, occ_out);
}

cudaError_t launch_tiny(int dtype, int nfm, const TinyArgs& a, int grid, cudaStream_t s, int* occ_out) {
  return dtype == 0 ? launch_tiny_nf<float>(nfm, a, grid, s, occ_out) : launch_tiny_nf<double>(nfm, a, grid, s, occ_out);
}

}  // namespace jt
