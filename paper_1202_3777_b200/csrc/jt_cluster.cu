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

// last index i in [lo, hi) with pre[i] <= q (pre ascending, pre[lo] <= q)
__device__ __forceinline__ int upper_idx(const int64_t* pre, int lo, int hi, int64_t q) {
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pre[mid] <= q) lo = mid;
    else hi = mid;
  }
  return lo;
}

constexpr int CL_LVL_MAX = 512;  // messages / targets of one level staged in shared memory

template <typename T>
__global__ void cluster_prop_kernel(const ClusterArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char csm[];
  __shared__ T* bases[CL_MAX_RANKS];
  // per-level prefix tables (item -> message / target by binary search in smem)
  __shared__ int64_t s_short[CL_LVL_MAX], s_long[CL_LVL_MAX], s_chunk[CL_LVL_MAX];
  const int rank = (int)cl.block_rank();
  const int nr = (int)cl.num_blocks();
  const int tid = threadIdx.x;
  const int nthr = nr * blockDim.x;
  const int gtid = rank * blockDim.x + tid;
  const int lane = tid & 31;
  const int gwarp = gtid >> 5, nwarps = nthr >> 5;
  T* my = reinterpret_cast<T*>(csm);
  if (tid < nr) bases[tid] = cl.map_shared_rank(my, tid);
  T* clique = reinterpret_cast<T*>(a.clique);
  T* aux = reinterpret_cast<T*>(a.aux);
  // load this rank's tables from HBM
  for (int s = 0; s < a.n_segs; ++s) {
    const ClusterSeg g = a.segs[s];
    if (g.rank != rank) continue;
    const T* src = (g.arena == A_CLIQUE ? clique : aux) + g.gofs;
    for (int e = tid; e < g.len; e += blockDim.x) my[g.lofs + e] = src[e];
  }
  cl.sync();
  for (int lv = 0; lv < a.n_levels; ++lv) {
    const ClusterLevel L = a.levels[lv];
    for (int i = tid; i < L.m1 - L.m0; i += blockDim.x) {
      s_short[i] = a.msgs[L.m0 + i].short0;
      s_long[i] = a.msgs[L.m0 + i].long0;
    }
    for (int i = tid; i < L.t1 - L.t0; i += blockDim.x) s_chunk[i] = a.tgts[L.t0 + i].chunk0;
    __syncthreads();
    // ---- phase A: marginalize every message of the level onto its separator ----
    for (int pass = 0; pass < 2; ++pass) {  // 0: short rows (thread/entry), 1: long rows (warp/entry)
      const int64_t total = pass == 0 ? L.n_short : L.n_long;
      const int64_t stride = pass == 0 ? nthr : nwarps;
      for (int64_t q = pass == 0 ? gtid : gwarp; q < total; q += stride) {
        // locate (message, entry): messages of the level are in [m0, m1), with
        // prefix counts of short / long entries
        const int m = L.m0 + upper_idx(pass == 0 ? s_short : s_long, 0, L.m1 - L.m0, q);
        const ClusterMsg M = a.msgs[m];  // one bulk copy: no dependent loads per field
        const int j = (int)(q - (pass == 0 ? M.short0 : M.long0));
        // row base of entry j: separator digits (separator order, last fastest)
        int rem = j, base = 0;
        for (int d = M.nsd - 1; d >= 0; --d) {
          const int c = M.sd_card[d];
          base += (rem % c) * M.sd_stride[d];
          rem /= c;
        }
        const T* src = rank_ptr<T>(bases, M.src_rank, M.src_off);
        double star = 0.0;
        if (pass == 0) {
          int dig[CL_MAXD];
          int off = base;
          for (int d = 0; d < M.nrd; ++d) dig[d] = 0;
          for (int p = 0; p < M.L; ++p) {
            star += (double)src[off];
            for (int d = M.nrd - 1; d >= 0; --d) {  // odometer over the rest dims
              off += M.rd_stride[d];
              if (++dig[d] < M.rd_card[d]) break;
              off -= M.rd_stride[d] * M.rd_card[d];
              dig[d] = 0;
            }
          }
        } else {
          for (int p = lane; p < M.L; p += 32) {
            int r2 = p, off = base;
            for (int d = M.nrd - 1; d >= 0; --d) {
              const int c = M.rd_card[d];
              off += (r2 % c) * M.rd_stride[d];
              r2 /= c;
            }
            star += (double)src[off];
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) star += __shfl_xor_sync(0xffffffffu, star, o);
          if (lane != 0) continue;
        }
        T* sep = rank_ptr<T>(bases, M.sep_rank, M.sep_off);
        T* rat = rank_ptr<T>(bases, M.rat_rank, M.rat_off);
        const double old = (double)sep[j];
        if (old == 0.0 && star != 0.0) atomicOr(a.err, EB_INCONSISTENT);
        rat[j] = (T)(old != 0.0 ? star / old : 0.0);
        sep[j] = (T)star;
      }
    }
    cl.sync();
    // ---- phase B: every target element times the ratios of its incoming messages ----
    for (int64_t q = gtid; q < L.n_elem_chunks; q += nthr) {
      const int t = L.t0 + upper_idx(s_chunk, 0, L.t1 - L.t0, q);
      const ClusterTgt& G = a.tgts[t];
      const int e0 = (int)(q - G.chunk0) * CL_CHUNK;
      const int e1 = min(G.size, e0 + CL_CHUNK);
      int dig[CL_MAXD];
      int rem = e0;
      for (int d = G.nd - 1; d >= 0; --d) {
        dig[d] = rem % G.card[d];
        rem /= G.card[d];
      }
      const int nin = G.nin, nd = G.nd;
      int sidx[CL_MAXIN];
      const T* rp[CL_MAXIN];
      int card[CL_MAXD];
      for (int d = 0; d < nd; ++d) card[d] = G.card[d];
      for (int k = 0; k < nin; ++k) {
        int x = 0;
        for (int d = 0; d < nd; ++d) x += dig[d] * G.sstride[k][d];
        sidx[k] = x;
        const int mi = G.msg[k];
        rp[k] = rank_ptr<T>(bases, a.msgs[mi].rat_rank, a.msgs[mi].rat_off);
      }
      T* tg = rank_ptr<T>(bases, G.rank, G.off);
      for (int e = e0; e < e1; ++e) {
        T v = tg[e];
        for (int k = 0; k < nin; ++k) v *= rp[k][sidx[k]];
        tg[e] = v;
        for (int d = nd - 1; d >= 0; --d) {  // odometer: digits and separator indices
          for (int k = 0; k < nin; ++k) sidx[k] += G.sstride[k][d];
          if (++dig[d] < card[d]) break;
          for (int k = 0; k < nin; ++k) sidx[k] -= G.sstride[k][d] * card[d];
          dig[d] = 0;
        }
      }
    }
    cl.sync();
  }
  // write this rank's tables back (ratio scratch stays on chip)
  for (int s = 0; s < a.n_segs; ++s) {
    const ClusterSeg g = a.segs[s];
    if (g.rank != rank || !g.writeback) continue;
    T* dst = (g.arena == A_CLIQUE ? clique : aux) + g.gofs;
    for (int e = tid; e < g.len; e += blockDim.x) dst[e] = my[g.lofs + e];
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
