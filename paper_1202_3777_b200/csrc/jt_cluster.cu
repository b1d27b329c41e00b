// Small trees in distributed shared memory: the whole single-tree state (clique
// tables, separators, ratio scratch) is loaded into the shared memory of one
// thread-block cluster (up to 16 CTAs), and the whole collect + distribute runs
// in ONE launch, level after level, separated by cluster barriers instead of
// kernel launches.  Each level is the paper's Alg. 1 for all its messages:
//   phase A — one thread (short rows) or one warp (long rows) per separator
//             entry j sums its row of the source clique (stride arithmetic, no
//             μ tables), forms ratio = new/old (0/0 = 0, nonzero/0 flagged) and
//             stores the new separator value;
//   phase B — every element of every target clique of the level is multiplied
//             by the ratios of all its incoming messages.
// Tables are bin-packed whole onto cluster ranks, so an element address is
// (rank, local offset) without per-element division; remote ranks are reached
// through DSMEM (cluster.map_shared_rank).  Sums are fixed-order: deterministic.
#include <cooperative_groups.h>

#include "jt_internal.h"

namespace cg = cooperative_groups;

namespace jt {

template <typename T>
__device__ __forceinline__ T* rank_ptr(T* const* bases, int rank, int off) {
  return bases[rank] + off;
}

// last index i in [0, n) with key(i) <= q (keys ascending, key(0) <= q)
template <class K>
__device__ __forceinline__ int upper_idx(K key, int n, int64_t q) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (key(mid) <= q) lo = mid;
    else hi = mid;
  }
  return lo;
}

template <typename T>
__global__ void __launch_bounds__(CL_THREADS) cluster_prop_kernel(const ClusterArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char csm[];
  __shared__ T* bases[CL_MAX_RANKS];
  const int rank = (int)cl.block_rank();
  const int nr = (int)cl.num_blocks();
  const int tid = threadIdx.x;
  const int nthr = nr * blockDim.x;
  const int gtid = rank * blockDim.x + tid;
  const int lane = tid & 31, warp = tid >> 5;
  const int gwarp = gtid >> 5, nwarps = nthr >> 5;
  T* my = reinterpret_cast<T*>(csm);
  if (tid < nr) bases[tid] = cl.map_shared_rank(my, tid);
  T* clique = reinterpret_cast<T*>(a.clique);
  T* aux = reinterpret_cast<T*>(a.aux);
  const int s0 = a.seg_begin[rank], s1 = a.seg_begin[rank + 1];
  for (int si = s0 + warp; si < s1; si += blockDim.x / 32) {  // a warp per table
    const ClusterSeg g = a.segs[si];
    const T* src = (g.arena == A_CLIQUE ? clique : aux) + g.gofs;
    for (int e = lane; e < g.len; e += 32) my[g.lofs + e] = src[e];
  }
  cl.sync();
  for (int lv = 0; lv < a.n_levels; ++lv) {
    const ClusterLevel L = a.levels[lv];
    // the level's descriptors: read through L1 (every thread of the SM touches the same few lines)
    const int* __restrict__ blob = a.blob + L.blob_off;
    const int nm = L.n_msgs;
    const int* toff = blob + nm * CL_MREC;  // target record offsets
    // ---- phase A: marginalize every message of the level onto its separator ----
    for (int pass = 0; pass < 2; ++pass) {  // 0: short rows (thread/entry), 1: long rows (warp/entry)
      const int64_t total = pass == 0 ? L.n_short : L.n_long;
      const int64_t stride = pass == 0 ? nthr : nwarps;
      const int koff = pass == 0 ? 9 : 10;
      for (int64_t q = pass == 0 ? gtid : gwarp; q < total; q += stride) {
        const int m = upper_idx([&](int i) { return (int64_t)blob[i * CL_MREC + koff]; }, nm, q);
        const int* M = blob + m * CL_MREC;
        const int j = (int)(q - M[koff]);
        const int nsd = M[7], nrd = M[8], Lr = M[6];
        int rem = j, base = 0;
        for (int d = nsd - 1; d >= 0; --d) {  // separator digits (separator order, last fastest)
          const int c = M[11 + d];
          base += (rem % c) * M[11 + CL_MAXD + d];
          rem /= c;
        }
        const T* src = rank_ptr<T>(bases, M[0], M[1]);
        const int* rc = M + 11 + 2 * CL_MAXD;
        const int* rs = M + 11 + 3 * CL_MAXD;
        double star = 0.0;
        if (pass == 0) {
          int dig[CL_MAXD];
          int off = base;
          for (int d = 0; d < nrd; ++d) dig[d] = 0;
          for (int p = 0; p < Lr; ++p) {
            star += (double)src[off];
            for (int d = nrd - 1; d >= 0; --d) {  // odometer over the rest dims
              off += rs[d];
              if (++dig[d] < rc[d]) break;
              off -= rs[d] * rc[d];
              dig[d] = 0;
            }
          }
        } else {
          for (int p = lane; p < Lr; p += 32) {
            int r2 = p, off = base;
            for (int d = nrd - 1; d >= 0; --d) {
              const int c = rc[d];
              off += (r2 % c) * rs[d];
              r2 /= c;
            }
            star += (double)src[off];
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) star += __shfl_xor_sync(0xffffffffu, star, o);
          if (lane != 0) continue;
        }
        T* sep = rank_ptr<T>(bases, M[2], M[3]);
        T* rat = rank_ptr<T>(bases, M[4], M[5]);
        const double old = (double)sep[j];
        if (old == 0.0 && star != 0.0) atomicOr(a.err, EB_INCONSISTENT);
        rat[j] = (T)(old != 0.0 ? star / old : 0.0);
        sep[j] = (T)star;
      }
    }
    cl.sync();
    // ---- phase B: every target element times the ratios of its incoming messages ----
    for (int64_t q = gtid; q < L.n_elem_chunks; q += nthr) {
      const int t = upper_idx([&](int i) { return (int64_t)blob[toff[i] + 5]; }, L.n_tgts, q);
      const int* G = blob + toff[t];
      const int size = G[2], nd = G[3], nin = G[4];
      const int* card = G + 6;
      const int e0 = (int)(q - G[5]) * CL_CHUNK;
      const int e1 = min(size, e0 + CL_CHUNK);
      int dig[CL_MAXD];
      int rem = e0;
      for (int d = nd - 1; d >= 0; --d) {
        dig[d] = rem % card[d];
        rem /= card[d];
      }
      int sidx[CL_MAXIN];
      const T* rp[CL_MAXIN];
      for (int k = 0; k < nin; ++k) {
        const int* R = G + 6 + nd + k * (2 + nd);
        int x = 0;
        for (int d = 0; d < nd; ++d) x += dig[d] * R[2 + d];
        sidx[k] = x;
        rp[k] = rank_ptr<T>(bases, R[0], R[1]);
      }
      T* tg = rank_ptr<T>(bases, G[0], G[1]);
      for (int e = e0; e < e1; ++e) {
        T v = tg[e];
        for (int k = 0; k < nin; ++k) v *= rp[k][sidx[k]];
        tg[e] = v;
        for (int d = nd - 1; d >= 0; --d) {  // odometer: digits and separator indices
          for (int k = 0; k < nin; ++k) sidx[k] += G[6 + nd + k * (2 + nd) + 2 + d];
          if (++dig[d] < card[d]) break;
          for (int k = 0; k < nin; ++k) sidx[k] -= G[6 + nd + k * (2 + nd) + 2 + d] * card[d];
          dig[d] = 0;
        }
      }
    }
    cl.sync();
  }
  for (int si = s0 + warp; si < s1; si += blockDim.x / 32) {  // write back (ratio scratch stays on chip)
    const ClusterSeg g = a.segs[si];
    T* dst = (g.arena == A_CLIQUE ? clique : aux) + g.gofs;
    for (int e = lane; e < g.len; e += 32) dst[e] = my[g.lofs + e];
  }
}

cudaError_t launch_cluster_prop(int dtype, const ClusterArgs& a, int n_ranks, int smem_bytes, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_ranks);
  cfg.blockDim = dim3(CL_THREADS);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = n_ranks;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (dtype == 0) return cudaLaunchKernelEx(&cfg, cluster_prop_kernel<float>, a);
  return cudaLaunchKernelEx(&cfg, cluster_prop_kernel<double>, a);
}

// Can a cluster of n_ranks CTAs with smem_bytes each be co-scheduled?
int cluster_prop_supported(int dtype, int n_ranks, int smem_bytes) {
  auto setup = [&](auto kern) -> int {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes) != cudaSuccess) return 0;
    if (n_ranks > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
      return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_ranks);
    cfg.blockDim = dim3(CL_THREADS);
    cfg.dynamicSmemBytes = smem_bytes;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = n_ranks;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return n;
  };
  return dtype == 0 ? setup(cluster_prop_kernel<float>) : setup(cluster_prop_kernel<double>);
}

}  // namespace jt
