// Device kernels of the B200 junction-tree engine (sm_100a).
//
// wave_kernel  — one launch per scheduler wave; every CTA walks a list of work
//   items, each a contiguous run of blocks of one *pass* (one sweep over one
//   clique table).  Per element: read the clique (or the shared base replica),
//   multiply the factor tensors in (separator ratios new/old of Alg. 1 step 2,
//   evidence masks), optionally write it back, and accumulate it into its
//   output separator entry (Alg. 1 step 1, Eq. 2).  Index maps are never read:
//   the separator/ratio indices come from stride arithmetic on the block's
//   outer offsets (host-precomputed per block) plus per-thread inner offsets.
//   Reductions are fixed-order (per-thread sequential → smem tree → chunk
//   order), so results are run-to-run deterministic.  The last CTA of an output
//   group sums the chunk partials and applies the Hugin update
//   (ratio = star/old with 0/0 = 0, nonzero/0 flagged; propagate.py:67-76).
#include "jt_internal.h"
#include "jt_device.cuh"
#include <cfloat>
#include <algorithm>
#include <type_traits>
#include <utility>

namespace jt {

// out[b] = Σ_{r<R} get(b, r): r ascending within a thread group, groups combined
// in order — deterministic for a given (n_bins, R).  `out` must not alias the
// values read by `get` (callers reduce from global partials or from `red`
// into a separate buffer).
template <class F>
__device__ __forceinline__ void reduce_bins(F get, int n_bins, int R, double* out, double* part2) {
  const int tid = threadIdx.x;
  if (n_bins >= NT) {
    for (int b = tid; b < n_bins; b += NT) {
      double s = 0.0;
      for (int r = 0; r < R; ++r) s += get(b, r);
      out[b] = s;
    }
    __syncthreads();
  } else {
    int G = NT / n_bins;
    if (G > R) G = R;
    if (G < 1) G = 1;
    if (tid < n_bins * G) {
      const int b = tid / G, g = tid - (tid / G) * G;
      double s = 0.0;
      for (int r = g; r < R; r += G) s += get(b, r);
      part2[tid] = s;
    }
    __syncthreads();
    if (tid < n_bins) {
      double t = 0.0;
      for (int g = 0; g < G; ++g) t += part2[tid * G + g];
      out[tid] = t;
    }
    __syncthreads();
  }
}

template <typename T>
__device__ __forceinline__ void finalize_entry(const DevPass& P, int64_t j, double star, T* aux,
                                               double* qout, int* err) {
  if (P.out_kind == OUT_SEP_FRESH) {
    aux[P.out_off + j] = (T)star;
  } else if (P.out_kind == OUT_SEP_DFRESH) {
    const double c = (double)aux[P.out_off + j];
    aux[P.ratio_off + j] = (T)(c != 0.0 ? star : 0.0);
    aux[(P.out2_off >= 0 ? P.out2_off : P.out_off) + j] = (T)(c * star);
  } else if (P.out_kind == OUT_SEP) {
    const double old = (double)aux[P.out_off + j];
    if (old == 0.0 && star != 0.0) atomicOr(err, EB_INCONSISTENT);
    const double r = (old != 0.0) ? star / old : 0.0;
    aux[P.ratio_off + j] = (T)r;
    aux[(P.out2_off >= 0 ? P.out2_off : P.out_off) + j] = (T)star;
  } else {
    qout[P.out_off + j] = star;
  }
}

// Deterministic cross-CTA combine of one output group's chunk partials.  The
// block's n_in values are in red[0..n_in).  Chunks are combined in fixed
// groups of CHUNK_GROUP (level 1) and the groups in order (level 2); the last
// CTA to arrive at each level does that level's sum, so no CTA reduces more
// than CHUNK_GROUP × n_in values.
template <typename T>
__device__ __noinline__ void chunk_finalize(const DevPass& P, const Item& item, const WaveArgs& a, double* red,
                               double* part2, int* s_last, T* aux) {
  const int tid = threadIdx.x;
  const int n_in = P.n_in, nch = P.n_chunks;
  const int ng = (nch + CHUNK_GROUP - 1) / CHUNK_GROUP;
  const int g = item.chunk / CHUNK_GROUP;
  const int gsz = min(CHUNK_GROUP, nch - g * CHUNK_GROUP);
  double* L1 = a.partials + P.part_off + item.j_out * (int64_t)(nch + ng) * n_in;
  double* L2 = L1 + (int64_t)nch * n_in;
  int* cnt = a.counters + P.cnt_off + item.j_out * (int64_t)(ng + 1);
  for (int b = tid; b < n_in; b += NT) L1[(int64_t)item.chunk * n_in + b] = red[b];
  __threadfence();
  __syncthreads();
  if (tid == 0) *s_last = (atomicAdd(&cnt[g], 1) == gsz - 1);
  __syncthreads();
  if (!*s_last) return;
  __threadfence();
  const double* Lg = L1 + (int64_t)g * CHUNK_GROUP * n_in;
  reduce_bins([&](int b, int r) { return __ldcg(Lg + (int64_t)r * n_in + b); }, n_in, gsz, red, part2);
  if (tid == 0) cnt[g] = 0;
  if (ng > 1) {
    for (int b = tid; b < n_in; b += NT) L2[(int64_t)g * n_in + b] = red[b];
    __threadfence();
    __syncthreads();
    if (tid == 0) *s_last = (atomicAdd(&cnt[ng], 1) == ng - 1);
    __syncthreads();
    if (!*s_last) return;
    __threadfence();
    reduce_bins([&](int b, int r) { return __ldcg(L2 + (int64_t)r * n_in + b); }, n_in, ng, red, part2);
    if (tid == 0) cnt[ng] = 0;
  }
  const int64_t j0 = item.j_out * (int64_t)n_in;
  for (int b = tid; b < n_in; b += NT) finalize_entry<T>(P, j0 + b, red[b], aux, a.qout, a.err);
}

// Thread-owned bins (P.own): each thread owns the VEC output lanes of its
// position in every block (n_in == T == NT*VEC), streams OKV blocks per
// iteration and finalizes its own lanes at every output-group boundary —
// no barriers, no shared memory in the steady state.  This is the batched
// layout's natural path (case = innermost index).
// VEC consecutive output entries [j, j+VEC) at once (j multiple of VEC): the
// thread-owned epilogue, with vector loads/stores of the separator arrays.
template <typename T, int VEC>
__device__ __forceinline__ void finalize_vec(const DevPass& P, int64_t j, const double (&star)[VEC], T* aux,
                                             double* qout) {
  if (P.out_kind == OUT_RAW) {
#pragma unroll
    for (int l = 0; l < VEC; ++l) qout[P.out_off + j + l] = star[l];
    return;
  }
  T nw[VEC];
  if (P.out_kind == OUT_SEP_FRESH) {
#pragma unroll
    for (int l = 0; l < VEC; ++l) nw[l] = (T)star[l];
    store_vec<T, VEC>(aux + P.out_off + j, nw);
    return;
  }
  T old[VEC], rt[VEC];
  load_vec<T, VEC>(aux + P.out_off + j, old);
  if (P.out_kind == OUT_SEP_DFRESH) {
#pragma unroll
    for (int l = 0; l < VEC; ++l) {
      const double c = (double)old[l];
      rt[l] = (T)(c != 0.0 ? star[l] : 0.0);
      nw[l] = (T)(c * star[l]);
    }
  } else {
#pragma unroll
    for (int l = 0; l < VEC; ++l) {
      const double o = (double)old[l];
      rt[l] = (T)(o != 0.0 ? star[l] / o : 0.0);
      nw[l] = (T)star[l];
    }
  }
  store_vec<T, VEC>(aux + P.ratio_off + j, rt);
  store_vec<T, VEC>(aux + (P.out2_off >= 0 ? P.out2_off : P.out_off) + j, nw);
}

template <typename T, int VEC>
__device__ __forceinline__ bool any_inconsistent(const DevPass& P, int64_t j, const double (&star)[VEC], const T* aux) {
  if (P.out_kind != OUT_SEP) return false;
  T old[VEC];
  load_vec<T, VEC>(aux + P.out_off + j, old);
  bool bad = false;
#pragma unroll
  for (int l = 0; l < VEC; ++l) bad |= ((double)old[l] == 0.0 && star[l] != 0.0);
  return bad;
}

constexpr int OWIN = 64;    // block-table window staged in shared memory

// Group flush of the thread-owned kernel, compiled once (not inlined into the
// unrolled block loop): multiply the group-constant factors in, check, and
// write the VEC lanes of each of the M vectors.
template <typename T, int VEC, int LM, int M>
__device__ __noinline__ void own_flush(const DevPass& P, const T* __restrict__ aux_c, T* aux, double* qout, int* err,
                                       const int32_t* e, const int* qfo, int64_t j, double s0, double s1, double s2,
                                       double s3, double s4, double s5, double s6, double s7, double s8, double s9,
                                       double s10, double s11, double s12, double s13, double s14, double s15) {
  constexpr int CH = NT * VEC;
  const double sv[16] = {s0, s1, s2, s3, s4, s5, s6, s7, s8, s9, s10, s11, s12, s13, s14, s15};
#pragma unroll
  for (int m = 0; m < M; ++m) {
    double sum[VEC];
#pragma unroll
    for (int l = 0; l < VEC; ++l) sum[l] = sv[m * VEC + l];
    for (int f = 0; f < P.nf; ++f) {
      if (!((P.flush_fac >> f) & 1u)) continue;
      const bool fv = LM == 0 ? (bool)((P.fac_vec >> f) & 1u) : true;
      const T* p = aux_c + P.fac_off[f] + e[2 + f] + qfo[f] + m * CH;
      T g[VEC];
      if (VEC == 1 || fv) {
        load_vec_ro<T, VEC>(p, g);
      } else {
#pragma unroll
        for (int l = 0; l < VEC; ++l) g[l] = __ldg(p);
      }
#pragma unroll
      for (int l = 0; l < VEC; ++l) sum[l] *= (double)g[l];
    }
    if (any_inconsistent<T, VEC>(P, j + m * CH, sum, aux)) atomicOr(err, EB_INCONSISTENT);
    finalize_vec<T, VEC>(P, j + m * CH, sum, aux, qout);
  }
}

// M vectors (lane chunks NT*VEC apart) per thread per block; OKV*M = 8 vectors
// in flight per tensor per iteration.  Block-table entries are int32 element
// offsets staged per window in shared memory; per-thread inner factor offsets
// live in shared memory so the factor loop stays a runtime loop (compact code).
template <typename T, int VEC, int LM, int M>
__global__ void __launch_bounds__(NT) wave_own_kernel(const WaveArgs a) {
  pdl_enter();
  static_assert(M * VEC <= 16, "flush passes at most 16 lanes");
  constexpr int OKV = 8 / M;
  __shared__ DevPass P;
  __shared__ double part2[NT];
  __shared__ int s_last;
  __shared__ double red[NT * 4 * 4];
  __shared__ int32_t s_blk[OWIN * (2 + MAXF)];
  __shared__ int s_qf[MAXF][NT];
  T* __restrict__ clique = reinterpret_cast<T*>(a.clique);
  const T* __restrict__ base = reinterpret_cast<const T*>(a.base);
  T* __restrict__ aux = reinterpret_cast<T*>(a.aux);
  const T* __restrict__ aux_c = aux;
  const int tid = threadIdx.x;
  const int lane0 = tid * VEC;
  constexpr int CH = NT * VEC;  // lanes per chunk
  static_assert(LM != 0 || M == 1, "generic load shapes use one vector per thread");
  int cur = -1;
  int q_src = 0, q_dst = 0;
  for (int it = blockIdx.x; it < a.n_items; it += gridDim.x) {
    const Item item = a.items[it];
    if (item.pass != cur) {
      __syncthreads();
      const int* sw = reinterpret_cast<const int*>(a.passes + item.pass);
      int* dw = reinterpret_cast<int*>(&P);
      for (int w = tid; w < (int)(sizeof(DevPass) / 4); w += NT) dw[w] = sw[w];
      __syncthreads();
      cur = item.pass;
      int rem = lane0, sacc = 0, dd = 0;
      for (int f = 0; f < MAXF; ++f) s_qf[f][tid] = 0;
      for (int d = P.ndi - 1; d >= 0; --d) {
        const int c = P.icard[d];
        const int dig = rem % c;
        rem /= c;
        sacc += dig * P.isrc[d];
        dd += dig * P.idst[d];
        for (int f = 0; f < P.nf; ++f) s_qf[f][tid] += dig * P.ifac[f][d];
      }
      q_src = sacc;
      q_dst = dd;
    }
    const int64_t r_out = P.n_blocks_per_jout;
    const bool chunked = P.n_chunks > 1;
    int64_t b0, b1;
    if (!chunked) {
      b0 = item.j_out * r_out;
      b1 = (item.j_out + item.j_count) * r_out;
    } else {
      b0 = item.j_out * r_out + (int64_t)item.chunk * P.blocks_per_chunk;
      b1 = min(b0 + P.blocks_per_chunk, (item.j_out + 1) * r_out);
    }
    const T* __restrict__ srcA =
        (P.src_arena == A_BASE ? base : P.src_arena == A_AUX ? aux_c : clique) + P.src_off + q_src;
    const bool wr = P.dst_off >= 0;
    T* __restrict__ dstA = clique + (wr ? P.dst_off : 0) + q_dst;
    const int bs = 2 + P.nf, nf = P.nf;
    const bool svec = LM == 0 ? (bool)P.src_vec : LM == 2;
    const uint32_t ffm = P.flush_fac;
    int qfo[MAXF];
#pragma unroll
    for (int f = 0; f < MAXF; ++f) qfo[f] = s_qf[f][tid];
    double acc[M][VEC];
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
      for (int l = 0; l < VEC; ++l) acc[m][l] = 0.0;
    int64_t gidx = b0 / r_out;
    int left = chunked ? INT32_MAX : (int)((gidx + 1) * r_out - b0);
    for (int64_t w0 = b0; w0 < b1; w0 += OWIN) {
      const int wn = (int)((b1 - w0) < OWIN ? (b1 - w0) : OWIN);
      __syncthreads();
      const int32_t* g = a.blk32 + P.blk32_off + w0 * bs;
      for (int i = tid; i < wn * bs; i += NT) s_blk[i] = __ldg(g + i);
      __syncthreads();
      for (int wb = 0; wb < wn; wb += OKV) {
        const int nb = wn - wb < OKV ? wn - wb : OKV;
        const int32_t* eb = &s_blk[wb * bs];
        T v[OKV][M][VEC];
#pragma unroll
        for (int u = 0; u < OKV; ++u) {
          if (u < nb) {
            const T* p = srcA + eb[u * bs];
#pragma unroll
            for (int m = 0; m < M; ++m) {
              if (VEC == 1 || svec) {
                load_vec<T, VEC>(p + m * CH, v[u][m]);
              } else {
                const T x = *p;
#pragma unroll
                for (int l = 0; l < VEC; ++l) v[u][m][l] = x;
              }
            }
          }
        }
        for (int f = 0; f < nf; ++f) {
          if ((ffm >> f) & 1u) continue;
          const T* fb = aux_c + P.fac_off[f] + s_qf[f][tid];
          const bool fv = LM == 0 ? (bool)((P.fac_vec >> f) & 1u) : true;
#pragma unroll
          for (int u = 0; u < OKV; ++u) {
            if (u < nb) {
              const T* p = fb + eb[u * bs + 2 + f];
#pragma unroll
              for (int m = 0; m < M; ++m) {
                T gv[VEC];
                if (VEC == 1 || fv) {
                  load_vec_ro<T, VEC>(p + m * CH, gv);
                } else {
                  const T x = __ldg(p);
#pragma unroll
                  for (int l = 0; l < VEC; ++l) gv[l] = x;
                }
#pragma unroll
                for (int l = 0; l < VEC; ++l) v[u][m][l] *= gv[l];
              }
            }
          }
        }
        // ≤ OKV-term partial sums in the storage type, folded into the fp64
        // accumulator once per iteration or output group
        T part[M][VEC];
#pragma unroll
        for (int m = 0; m < M; ++m)
#pragma unroll
          for (int l = 0; l < VEC; ++l) part[m][l] = (T)0;
#pragma unroll
        for (int u = 0; u < OKV; ++u) {
          if (u >= nb) continue;
          if (wr) {
            T* dp = dstA + eb[u * bs + 1];
#pragma unroll
            for (int m = 0; m < M; ++m) store_vec<T, VEC>(dp + m * CH, v[u][m]);
          }
#pragma unroll
          for (int m = 0; m < M; ++m)
#pragma unroll
            for (int l = 0; l < VEC; ++l) part[m][l] += v[u][m][l];
          if (--left == 0) {
            double sv[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) sv[i] = 0.0;
#pragma unroll
            for (int m = 0; m < M; ++m)
#pragma unroll
              for (int l = 0; l < VEC; ++l) {
                sv[m * VEC + l] = acc[m][l] + (double)part[m][l];
                acc[m][l] = 0.0;
                part[m][l] = (T)0;
              }
            own_flush<T, VEC, LM, M>(P, aux_c, aux, a.qout, a.err, eb + u * bs, qfo, gidx * (int64_t)P.n_in + lane0,
                                     sv[0], sv[1], sv[2], sv[3], sv[4], sv[5], sv[6], sv[7], sv[8], sv[9], sv[10],
                                     sv[11], sv[12], sv[13], sv[14], sv[15]);
            ++gidx;
            left = (int)r_out;
          }
        }
#pragma unroll
        for (int m = 0; m < M; ++m)
#pragma unroll
          for (int l = 0; l < VEC; ++l) acc[m][l] += (double)part[m][l];
      }
    }
    if (chunked) {
      // group-constant factors: apply to this chunk's partial (Σ F·S_c = F·Σ S_c)
      const int32_t* e = &s_blk[0];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        double sum[VEC];
#pragma unroll
        for (int l = 0; l < VEC; ++l) sum[l] = acc[m][l];
        for (int f = 0; f < nf; ++f) {
          if (!((ffm >> f) & 1u)) continue;
          const bool fv = LM == 0 ? (bool)((P.fac_vec >> f) & 1u) : true;
          const T* p = aux_c + P.fac_off[f] + e[2 + f] + qfo[f] + m * CH;
#pragma unroll
          for (int l = 0; l < VEC; ++l) sum[l] *= (double)__ldg(p + (fv ? l : 0));
        }
#pragma unroll
        for (int l = 0; l < VEC; ++l) red[lane0 + m * CH + l] = sum[l];
      }
      __syncthreads();
      chunk_finalize<T>(P, item, a, red, part2, &s_last, aux);
      __syncthreads();
    }
  }
}

#ifndef WK2_MINB
#define WK2_MINB 3
#endif
// KVT vectors per thread per iteration: 4 for large waves; 2 at three CTAs per
// SM for small, latency-bound waves (more warps in flight, less work per step)
// The general pass interpreter over one wave's items.  COH (persistent
// program): tables change between the waves of one launch, so factor loads
// take the coherent path instead of the read-only (non-coherent) cache.
template <typename T, int VEC, int KVT, bool COH>
__device__ __forceinline__ void wave_body(const WaveArgs& a) {
  constexpr int TH = NT * KVT * VEC;  // positions per CTA iteration
  __shared__ DevPass P;
  __shared__ double part2[NT];
  __shared__ int s_last;
  extern __shared__ __align__(16) double dsm[];
  double* red = dsm;                                              // [TH] block partials
  double* outb = dsm + TH;                                        // [TH] reduced bins
  uint16_t (*s_qfac)[KVT][NT] = reinterpret_cast<uint16_t (*)[KVT][NT]>(dsm + 2 * TH);  // inner factor offsets

  T* __restrict__ clique = reinterpret_cast<T*>(a.clique);
  const T* __restrict__ base = reinterpret_cast<const T*>(a.base);
  T* __restrict__ aux = reinterpret_cast<T*>(a.aux);
  const int tid = threadIdx.x;

  int cur = -1;
  int q_slot[KVT];
  bool q_ok[KVT];
  int q_src[KVT], q_dst[KVT];

  for (int it = blockIdx.x; it < a.n_items; it += gridDim.x) {
    const Item item = a.items[it];
    if (item.pass != cur) {
      __syncthreads();
      const int* sw = reinterpret_cast<const int*>(a.passes + item.pass);
      int* dw = reinterpret_cast<int*>(&P);
      for (int w = tid; w < (int)(sizeof(DevPass) / 4); w += NT) dw[w] = sw[w];
      __syncthreads();
      cur = item.pass;
      const int TV = P.T / VEC;
      const int nq = P.BPI * TV;
#pragma unroll
      for (int k = 0; k < KVT; ++k) {
        const int q = tid + k * NT;
        q_ok[k] = q < nq;
        const int slot = q_ok[k] ? q / TV : 0;
        const int iv = q_ok[k] ? q - slot * TV : 0;
        q_slot[k] = slot;
        int rem = iv * VEC, s = 0, dd = 0;
        int fo[MAXF];
#pragma unroll
        for (int f = 0; f < MAXF; ++f) fo[f] = 0;
        for (int d = P.ndi - 1; d >= 0; --d) {
          const int c = P.icard[d];
          const int dig = rem % c;
          rem /= c;
          s += dig * P.isrc[d];
          dd += dig * P.idst[d];
#pragma unroll
          for (int f = 0; f < MAXF; ++f)
            if (f < P.nf) fo[f] += dig * P.ifac[f][d];
        }
        q_src[k] = s;
        q_dst[k] = dd;
#pragma unroll
        for (int f = 0; f < MAXF; ++f) s_qfac[f][k][tid] = (uint16_t)fo[f];
      }
    }

    const bool multi = P.gpi > 1;
    const int64_t jb = item.j_out * P.n_blocks_per_jout;
    const int64_t b0 = jb + (int64_t)item.chunk * P.blocks_per_chunk;
    int64_t b1 = multi ? (item.j_out + item.j_count) * P.n_blocks_per_jout : b0 + P.blocks_per_chunk;
    if (!multi && b1 > jb + P.n_blocks_per_jout) b1 = jb + P.n_blocks_per_jout;
    const T* __restrict__ srcA = (P.src_arena == A_BASE ? base : P.src_arena == A_AUX ? aux : clique) + P.src_off;
    const bool wr = P.dst_off >= 0;
    T* __restrict__ dstA = clique + (wr ? P.dst_off : 0);
    const int64_t* __restrict__ blk = a.blk + P.blk_off;
    const int bs = P.blk_stride;
    const int nf = P.nf;

    double acc[KVT][VEC];
#pragma unroll
    for (int k = 0; k < KVT; ++k)
#pragma unroll
      for (int l = 0; l < VEC; ++l) acc[k][l] = 0.0;

    for (int64_t bb = b0; bb < b1; bb += P.BPI) {
      T v[KVT][VEC];
      const int64_t* e[KVT];
      bool ok[KVT];
      // block-table lookups of every slot first, then the data loads: the KVT
      // loads issue back to back instead of each waiting on its own lookup
      int64_t so[KVT];
#pragma unroll
      for (int k = 0; k < KVT; ++k) {
        const int64_t bi = bb + q_slot[k];
        ok[k] = q_ok[k] && bi < b1;
        e[k] = blk + (ok[k] ? bi : b0) * bs;
        so[k] = __ldg(e[k]) + q_src[k];
      }
#pragma unroll
      for (int k = 0; k < KVT; ++k) {
        if (ok[k]) {
          const T* p = srcA + so[k];
          if (VEC == 1 || P.src_vec) {
            load_vec<T, VEC>(p, v[k]);
          } else {
            const T x = *p;
#pragma unroll
            for (int l = 0; l < VEC; ++l) v[k][l] = x;
          }
        } else {
#pragma unroll
          for (int l = 0; l < VEC; ++l) v[k][l] = (T)0;
        }
      }
#pragma unroll
      for (int f = 0; f < MAXF; ++f) {
        if (f < nf) {
          const T* fb = aux + P.fac_off[f];
          const bool fv = (P.fac_vec >> f) & 1u;
          int64_t fo[KVT];
#pragma unroll
          for (int k = 0; k < KVT; ++k) fo[k] = __ldg(e[k] + 2 + f) + s_qfac[f][k][tid];
#pragma unroll
          for (int k = 0; k < KVT; ++k) {
            if (ok[k]) {
              const T* p = fb + fo[k];
              T g[VEC];
              if (VEC == 1 || fv) {
                if (COH) load_vec<T, VEC>(p, g);
                else load_vec_ro<T, VEC>(p, g);
              } else {
                const T x = COH ? *p : __ldg(p);
#pragma unroll
                for (int l = 0; l < VEC; ++l) g[l] = x;
              }
#pragma unroll
              for (int l = 0; l < VEC; ++l) v[k][l] *= g[l];
            }
          }
        }
      }
      if (wr) {
#pragma unroll
        for (int k = 0; k < KVT; ++k)
          if (ok[k]) store_vec<T, VEC>(dstA + e[k][1] + q_dst[k], v[k]);
      }
#pragma unroll
      for (int k = 0; k < KVT; ++k)
#pragma unroll
        for (int l = 0; l < VEC; ++l) acc[k][l] += (double)v[k][l];
      if (multi) {
        // this iteration holds gpi complete output groups: reduce and finalize now
        const int n_in = P.n_in;
        const int64_t g0 = (bb - jb) / P.n_blocks_per_jout + item.j_out;
        const int64_t rem_g = item.j_out + item.j_count - g0;
        const int ng = (int)(rem_g < P.gpi ? rem_g : P.gpi);
#pragma unroll
        for (int k = 0; k < KVT; ++k) {
          if (q_ok[k]) {
            const int q = tid + k * NT;
#pragma unroll
            for (int l = 0; l < VEC; ++l) {
              red[q * VEC + l] = acc[k][l];
              acc[k][l] = 0.0;
            }
          }
        }
        __syncthreads();
        const int rest = P.T / n_in;
        const int ro = (int)P.n_blocks_per_jout;
        const int32_t* __restrict__ bbase = a.bins + P.bin_off;
        const int32_t* __restrict__ brest = bbase + n_in;
        const int T_ = P.T;
        reduce_bins(
            [&](int gb, int r) {
              const int g = gb / n_in, b = gb - (gb / n_in) * n_in;
              const int slot = g * ro + r / rest;
              return red[slot * T_ + (n_in == 1 ? 0 : bbase[b]) + (n_in == 1 ? r % rest : brest[r % rest])];
            },
            ng * n_in, ro * rest, outb, part2);
        for (int b = tid; b < ng * n_in; b += NT) finalize_entry<T>(P, g0 * n_in + b, outb[b], aux, a.qout, a.err);
        __syncthreads();
      }
    }

    if (P.out_kind == OUT_NONE || multi) continue;

    // ---- block partials -> n_in bins (fixed order) ----
    const int n_in = P.n_in;
    double* vals = outb;  // reduced bins of this item
    if (n_in == 1) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < KVT; ++k)
#pragma unroll
        for (int l = 0; l < VEC; ++l) s += acc[k][l];
      s = warp_sum(s);
      if ((tid & 31) == 0) part2[tid >> 5] = s;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < NT / 32; ++w) t += part2[w];
        outb[0] = t;
      }
      __syncthreads();
    } else {
#pragma unroll
      for (int k = 0; k < KVT; ++k) {
        if (q_ok[k]) {
          const int q = tid + k * NT;
#pragma unroll
          for (int l = 0; l < VEC; ++l) red[q * VEC + l] = acc[k][l];
        }
      }
      __syncthreads();
      if (!(P.BPI == 1 && n_in == P.T)) {
        const int rest = P.T / n_in;
        const int R = P.BPI * rest;
        const int32_t* __restrict__ bbase = a.bins + P.bin_off;
        const int32_t* __restrict__ brest = bbase + n_in;
        const int T_ = P.T;
        reduce_bins(
            [&](int b, int r) {
              const int slot = r / rest;
              const int p = r - slot * rest;
              return red[slot * T_ + bbase[b] + brest[p]];
            },
            n_in, R, outb, part2);
      } else {
        vals = red;  // identity bins: every position is its own output entry
      }
    }

    // ---- output: direct or via chunk partials + last-CTA finalize ----
    const int64_t j0 = item.j_out * (int64_t)n_in;
    if (P.n_chunks == 1) {
      for (int b = tid; b < n_in; b += NT) finalize_entry<T>(P, j0 + b, vals[b], aux, a.qout, a.err);
    } else {
      if (vals != red) {
        for (int b = tid; b < n_in; b += NT) red[b] = vals[b];
        __syncthreads();
      }
      chunk_finalize<T>(P, item, a, red, part2, &s_last, aux);
    }
    __syncthreads();
  }
}

template <typename T, int VEC, int KVT>
__global__ void __launch_bounds__(NT, KVT == 2 ? WK2_MINB : 2) wave_kernel(const WaveArgs a) {
  pdl_enter();
  wave_body<T, VEC, KVT, false>(a);
}

// Row passes: every position of a unit reduces into ONE output entry (n_in <= 1:
// the separator is a prefix of the merged outer dims — Alg. 1 row sums — or
// there is no output, e.g. a pure absorb/write pass).  Warp-centric: a unit is
// one output group (or `j_count` small groups, or one chunk of a huge group)
// walked by ONE warp, KR vectors per lane in flight per tensor, reduced with
// shuffles — no barriers, no shared memory.  Units are handed out dynamically
// (one atomic per unit), so SMs that run ahead take more of them; the results
// do not depend on which warp took a unit (each group is summed in a fixed
// order, chunk partials are combined in chunk order), so they are
// run-to-run deterministic.  Inner offsets of the T positions of a block come
// from a host-built table (RowTab, L1-resident); block offsets from the block
// table.
constexpr int KR = KROW;

template <typename T>
__device__ __forceinline__ double warp_chunk_combine(const DevPass& P, const Item& u, const WaveArgs& a,
                                                     double part, bool* last) {
  // n_in == 1 chunk partials: level 1 groups of CHUNK_GROUP chunks, level 2 the
  // groups in order; the last warp to arrive at a level sums it (lane i holds
  // partial i, fixed xor-tree order)
  const int lane = threadIdx.x & 31;
  const int nch = P.n_chunks;
  const int ng = (nch + CHUNK_GROUP - 1) / CHUNK_GROUP;
  const int g = u.chunk / CHUNK_GROUP;
  const int gsz = min(CHUNK_GROUP, nch - g * CHUNK_GROUP);
  double* L1 = a.partials + P.part_off + u.j_out * (int64_t)(nch + ng);
  double* L2 = L1 + nch;
  int* cnt = a.counters + P.cnt_off + u.j_out * (int64_t)(ng + 1);
  if (lane == 0) L1[u.chunk] = part;
  __threadfence();
  __syncwarp();
  int arrived = 0;
  if (lane == 0) arrived = atomicAdd(&cnt[g], 1);
  arrived = __shfl_sync(0xffffffffu, arrived, 0);
  *last = false;
  if (arrived != gsz - 1) return 0.0;
  __threadfence();
  double s = lane < gsz ? __ldcg(L1 + g * CHUNK_GROUP + lane) : 0.0;
  s = warp_sum(s);
  if (lane == 0) cnt[g] = 0;
  if (ng > 1) {
    if (lane == 0) L2[g] = s;
    __threadfence();
    __syncwarp();
    if (lane == 0) arrived = atomicAdd(&cnt[ng], 1);
    arrived = __shfl_sync(0xffffffffu, arrived, 0);
    if (arrived != ng - 1) return 0.0;
    __threadfence();
    s = 0.0;
    for (int i0 = 0; i0 < ng; i0 += 32) {  // ng <= 32 for any realistic split
      const double x = i0 + lane < ng ? __ldcg(L2 + i0 + lane) : 0.0;
      s += warp_sum(x);
    }
    if (lane == 0) cnt[ng] = 0;
  }
  *last = true;
  return s;
}

// LIN: the pass's blocks are at least KR vectors per lane (TW >= KR) and the
// src/dst inner offsets are the positions themselves (the clique's own layout):
// one block entry per batch, slot addresses are immediates off one pointer.
template <typename T, int VEC, bool LIN>
#ifndef ROW_MINB
#define ROW_MINB 2
#endif
__global__ void __launch_bounds__(NT, ROW_MINB) wave_row_kernel(const WaveArgs a) {
  pdl_enter();
  T* __restrict__ clique = reinterpret_cast<T*>(a.clique);
  const T* __restrict__ base = reinterpret_cast<const T*>(a.base);
  T* __restrict__ aux = reinterpret_cast<T*>(a.aux);
  const T* __restrict__ aux_c = aux;
  const int lane = threadIdx.x & 31;
  const int n_warps = gridDim.x * (NT / 32);
  // static round-robin over the warps of the grid: unit i -> warp i mod n_warps
  for (int ui = blockIdx.x * (NT / 32) + (threadIdx.x >> 5); ui < a.n_items; ui += n_warps) {
    const Item u = a.items[ui];
    const DevPass* __restrict__ P = a.passes + u.pass;
    const int TW = LIN ? P->T / (32 * VEC) : P->T / (32 * VEC);  // {1,2,4} or a multiple of KR
    const int lg = (LIN || TW >= KR) ? 0 : (TW == 1 ? 0 : TW == 2 ? 1 : 2);
    const int TV = P->T / VEC;
    const int64_t r_out = P->n_blocks_per_jout;
    const bool chunked = P->n_chunks > 1;
    const T* __restrict__ srcA =
        (P->src_arena == A_BASE ? base : P->src_arena == A_AUX ? aux_c : clique) + P->src_off;
    const bool wr = P->dst_off >= 0;
    T* __restrict__ dstA = clique + (wr ? P->dst_off : 0);
    const int32_t* __restrict__ blk = a.blk32 + P->blk32_off;
    const int32_t* __restrict__ tab = a.rowtab + P->row_tab_off;  // [2+nf][T/VEC]
    const int bs = 2 + P->nf;
    const int nf = P->nf;
    const bool svec = VEC == 1 || P->src_vec;
    const uint32_t fvm = P->fac_vec;
    const uint32_t fmode = P->row_fmode;
    const int out_kind = P->out_kind;
    const int n_groups = chunked ? 1 : (int)u.j_count;
    for (int gi = 0; gi < n_groups; ++gi) {
      const int64_t j = u.j_out + gi;
      int64_t b = j * r_out, b1 = b + r_out;
      if (chunked) {
        b += (int64_t)u.chunk * P->blocks_per_chunk;
        b1 = min(b + P->blocks_per_chunk, (j + 1) * r_out);
      }
      double acc = 0.0;
      int kk = 0;  // TW >= KR: next vector index within block b
      while (b < b1) {
        // phase 1: every slot's block entry and inner offset (no data yet), so the
        // KR data loads below issue back to back instead of each waiting on its index
        T v[KR][VEC];
        int ioff[KR];
        uint32_t okm = (1u << KR) - 1u;
        int e0 = 0;
        if (LIN) {
          e0 = __ldg(blk + b * bs);
          const T* p0 = srcA + e0 + (kk * 32 + lane) * VEC;
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            ioff[k] = (kk + k) * 32 + lane;
            load_vec_cs<T, VEC>(p0 + k * 32 * VEC, v[k]);
          }
        } else {
          int soff[KR];
          okm = 0;
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            const int64_t bk = TW >= KR ? b : b + (k >> lg);
            const bool ok = bk < b1;
            okm |= (ok ? 1u : 0u) << k;
            ioff[k] = (TW >= KR ? kk + k : (k & (TW - 1))) * 32 + lane;
            soff[k] = __ldg(blk + (ok ? bk : b) * bs) + __ldg(tab + ioff[k]);
          }
          // phase 2: the data loads (streaming: evict-first, keeps L1 for the tables)
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            const T* p = srcA + soff[k];
            if (svec) {
              load_vec_cs<T, VEC>(p, v[k]);
            } else {
              const T x = __ldcs(p);
#pragma unroll
              for (int l = 0; l < VEC; ++l) v[k][l] = x;
            }
          }
        }
        // phase 3: factors (separator ratios / evidence masks: small, L1/L2-resident).
        // Per factor the host chose how its inner offsets are formed: a table
        // lookup, the position itself (linear), or zero (constant over the block).
        for (int f = 0; f < nf; ++f) {
          const T* fb = aux_c + P->fac_off[f];
          const int mode = (fmode >> (2 * f)) & 3;
          if ((LIN || TW >= KR) && mode == 2) {  // one value per block: scalar broadcast
            const T x = __ldg(fb + __ldg(blk + b * bs + 2 + f));
#pragma unroll
            for (int k = 0; k < KR; ++k)
#pragma unroll
              for (int l = 0; l < VEC; ++l) v[k][l] *= x;
            continue;
          }
          const int32_t* tf = tab + (int64_t)(2 + f) * TV;
          const bool fv = (fvm >> f) & 1u;
          int fo[KR];
          if (LIN || TW >= KR) {
            const int e = __ldg(blk + b * bs + 2 + f);
#pragma unroll
            for (int k = 0; k < KR; ++k)
              fo[k] = e + (mode == 1 ? ioff[k] * VEC : mode == 2 ? 0 : __ldg(tf + ioff[k]));
          } else {
#pragma unroll
            for (int k = 0; k < KR; ++k) {
              const int64_t bk = b + (k >> lg);
              fo[k] = __ldg(blk + (bk < b1 ? bk : b) * bs + 2 + f) +
                      (mode == 1 ? ioff[k] * VEC : mode == 2 ? 0 : __ldg(tf + ioff[k]));
            }
          }
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            T g[VEC];
            if (VEC == 1 || fv) {
              load_vec_ro<T, VEC>(fb + fo[k], g);
            } else {
              const T x = __ldg(fb + fo[k]);
#pragma unroll
              for (int l = 0; l < VEC; ++l) g[l] = x;
            }
#pragma unroll
            for (int l = 0; l < VEC; ++l) v[k][l] *= g[l];
          }
        }
        if (wr) {
          if (LIN) {
            T* q0 = dstA + __ldg(blk + b * bs + 1) + (kk * 32 + lane) * VEC;
#pragma unroll
            for (int k = 0; k < KR; ++k) store_vec<T, VEC>(q0 + k * 32 * VEC, v[k]);
          } else {
            const int32_t* td = tab + TV;
#pragma unroll
            for (int k = 0; k < KR; ++k) {
              if ((okm >> k) & 1u) {
                const int64_t bk = TW >= KR ? b : b + (k >> lg);
                store_vec<T, VEC>(dstA + __ldg(blk + bk * bs + 1) + __ldg(td + ioff[k]), v[k]);
              }
            }
          }
        }
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          T part = (T)0;
#pragma unroll
          for (int l = 0; l < VEC; ++l) part += v[k][l];
          acc += ((okm >> k) & 1u) ? (double)part : 0.0;
        }
        if (LIN || TW >= KR) {
          kk += KR;
          if (kk == TW) {
            kk = 0;
            ++b;
          }
        } else {
          b += KR >> lg;
        }
      }
      if (out_kind == OUT_NONE) continue;
      double sum = warp_sum(acc);
      if (chunked) {
        bool last;
        sum = warp_chunk_combine<T>(*P, u, a, sum, &last);
        if (!last) continue;
      }
      if (lane == 0) finalize_entry<T>(*P, j, sum, aux, a.qout, a.err);
    }
  }
}

template <typename T, int VEC>
static cudaError_t launch_row_t(int lin, const WaveArgs& a, int grid, cudaStream_t s) {
  return lin ? launch_pdl(wave_row_kernel<T, VEC, true>, grid, NT, 0, s, a)
             : launch_pdl(wave_row_kernel<T, VEC, false>, grid, NT, 0, s, a);
}

cudaError_t launch_wave_row(int dtype, int vec, int lin, const WaveArgs& a, int grid, cudaStream_t s) {
  if (grid <= 0 || a.n_items <= 0) return cudaSuccess;
  if (dtype == 0) {
    if (vec == 4) return launch_row_t<float, 4>(lin, a, grid, s);
    if (vec == 2) return launch_row_t<float, 2>(lin, a, grid, s);
    return launch_row_t<float, 1>(lin, a, grid, s);
  }
  if (vec == 2) return launch_row_t<double, 2>(lin, a, grid, s);
  return launch_row_t<double, 1>(lin, a, grid, s);
}

template <typename T, int VEC>
static int occ_row_t() {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, wave_row_kernel<T, VEC, false>, NT, 0);
  return n > 0 ? n : 1;
}

int wave_row_max_ctas_per_sm(int dtype, int vec) {
  if (dtype == 0) {
    if (vec == 4) return occ_row_t<float, 4>();
    if (vec == 2) return occ_row_t<float, 2>();
    return occ_row_t<float, 1>();
  }
  if (vec == 2) return occ_row_t<double, 2>();
  return occ_row_t<double, 1>();
}

template <int VEC, int KVT>
constexpr size_t wave_smem() {
  return (size_t)2 * NT * KVT * VEC * sizeof(double) + (size_t)MAXF * KVT * NT * sizeof(uint16_t);
}

template <typename T, int VEC, int KVT>
static cudaError_t launch_t(const WaveArgs& a, int grid, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(wave_kernel<T, VEC, KVT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)wave_smem<VEC, KVT>());
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(wave_kernel<T, VEC, KVT>, grid, NT, wave_smem<VEC, KVT>(), s, a);
}

template <typename T, int VEC, int LM, int M>
static cudaError_t launch_own_t(const WaveArgs& a, int grid, cudaStream_t s) {
  return launch_pdl(wave_own_kernel<T, VEC, LM, M>, grid, NT, 0, s, a);
}

template <typename T, int VEC, int LM>
static cudaError_t launch_own_m(int m, const WaveArgs& a, int grid, cudaStream_t s) {
  if (m == 4) return launch_own_t<T, VEC, LM, 4>(a, grid, s);
  if (m == 2) return launch_own_t<T, VEC, LM, 2>(a, grid, s);
  return launch_own_t<T, VEC, LM, 1>(a, grid, s);
}

cudaError_t launch_wave_own(int dtype, int vec, int lm, int m, const WaveArgs& a, int grid, cudaStream_t s) {
  if (grid <= 0 || a.n_items <= 0) return cudaSuccess;
  if (dtype == 0) {
    if (vec == 4) {
      if (lm == 1) return launch_own_m<float, 4, 1>(m, a, grid, s);
      if (lm == 2) return launch_own_m<float, 4, 2>(m, a, grid, s);
      return launch_own_t<float, 4, 0, 1>(a, grid, s);
    }
    if (vec == 2) return launch_own_t<float, 2, 0, 1>(a, grid, s);
    return launch_own_t<float, 1, 0, 1>(a, grid, s);
  }
  if (vec == 2) {
    if (lm == 1) return launch_own_m<double, 2, 1>(m, a, grid, s);
    if (lm == 2) return launch_own_m<double, 2, 2>(m, a, grid, s);
    return launch_own_t<double, 2, 0, 1>(a, grid, s);
  }
  return launch_own_t<double, 1, 0, 1>(a, grid, s);
}

template <typename T, int VEC>
static int occ_own_t() {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, wave_own_kernel<T, VEC, 0, 1>, NT, 0);
  return n > 0 ? n : 1;
}

int wave_own_max_ctas_per_sm(int dtype, int vec) {
  if (dtype == 0) {
    if (vec == 4) return occ_own_t<float, 4>();
    if (vec == 2) return occ_own_t<float, 2>();
    return occ_own_t<float, 1>();
  }
  if (vec == 2) return occ_own_t<double, 2>();
  return occ_own_t<double, 1>();
}

template <int KVT>
static cudaError_t launch_kv(int dtype, int vec, const WaveArgs& a, int grid, cudaStream_t s) {
  if (dtype == 0) {
    if (vec == 4) return launch_t<float, 4, KVT>(a, grid, s);
    if (vec == 2) return launch_t<float, 2, KVT>(a, grid, s);
    return launch_t<float, 1, KVT>(a, grid, s);
  }
  if (vec == 2) return launch_t<double, 2, KVT>(a, grid, s);
  return launch_t<double, 1, KVT>(a, grid, s);
}

cudaError_t launch_wave(int dtype, int vec, int kv, const WaveArgs& a, int grid, cudaStream_t s) {
  if (grid <= 0 || a.n_items <= 0) return cudaSuccess;
  return kv == 2 ? launch_kv<2>(dtype, vec, a, grid, s) : launch_kv<4>(dtype, vec, a, grid, s);
}

template <typename T, int VEC, int KVT>
static int occ_t() {
  int n = 0;
  cudaFuncSetAttribute(wave_kernel<T, VEC, KVT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)wave_smem<VEC, KVT>());
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, wave_kernel<T, VEC, KVT>, NT, wave_smem<VEC, KVT>());
  return n > 0 ? n : 1;
}

template <int KVT>
static int occ_kv(int dtype, int vec) {
  if (dtype == 0) {
    if (vec == 4) return occ_t<float, 4, KVT>();
    if (vec == 2) return occ_t<float, 2, KVT>();
    return occ_t<float, 1, KVT>();
  }
  if (vec == 2) return occ_t<double, 2, KVT>();
  return occ_t<double, 1, KVT>();
}

int wave_max_ctas_per_sm(int dtype, int vec, int kv) { return kv == 2 ? occ_kv<2>(dtype, vec) : occ_kv<4>(dtype, vec); }

// ---- posteriors: raw marginals [var][card][B] -> normalized [B][Σcard] ----
// normalize (potential.py:181-186): total <= 0 raises ZeroMassError; here the
// case's row is NaN-filled and the zero-mass bit is set.
// q_exp (nullable: exp_all for every query): the queried tables are stored
// scaled by 2^q_exp (power-of-two prescaling); unnormalized results undo it.
__global__ void normalize_kernel(const double* __restrict__ qout, const int64_t* __restrict__ q_off,
                                 const int32_t* __restrict__ q_card, const int32_t* __restrict__ q_col,
                                 int nq, int B, int rows, int total_cols, int normalize,
                                 double* __restrict__ post, int* err, const int* __restrict__ q_exp, int exp_all) {
  // qout is [card][B] (B = padded case lanes); posteriors are written for the first `rows` cases
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nq * rows) return;
  const int i = (int)(idx / rows);
  const int b = (int)(idx - (int64_t)i * rows);
  const double* q = qout + q_off[i];
  const int card = q_card[i];
  double* o = post + (int64_t)b * total_cols + q_col[i];
  double s = 0.0;
  for (int d = 0; d < card; ++d) s += q[(int64_t)d * B + b];
  if (!normalize) {
    const int ex = q_exp ? q_exp[i] : exp_all;
    for (int d = 0; d < card; ++d) o[d] = ldexp(q[(int64_t)d * B + b], -ex);
    return;
  }
  if (!(s > 0.0)) {
    atomicOr(err, EB_ZERO_MASS);
    atomicMin(err + 1, b);  // lowest failing case (jt_error_case)
    for (int d = 0; d < card; ++d) o[d] = __longlong_as_double(0x7ff8000000000000ULL);
    return;
  }
  for (int d = 0; d < card; ++d) o[d] = q[(int64_t)d * B + b] / s;
}

cudaError_t launch_normalize(const double* qout, const int64_t* q_off, const int32_t* q_card,
                             const int32_t* q_col, int nq, int B, int rows, int total_cols, int normalize,
                             double* post, int* err, const int* q_exp, int exp_all, cudaStream_t s) {
  const int64_t n = (int64_t)nq * rows;
  if (n == 0) return cudaSuccess;
  normalize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(qout, q_off, q_card, q_col, nq, B, rows,
                                                               total_cols, normalize, post, err, q_exp, exp_all);
  return cudaGetLastError();
}

// ---- host<->arena conversion (f64 staging <-> storage type, batch lanes) ----
// exp2: stored = value * 2^exp2 (power-of-two prescaling, exact: ldexp only
// moves the exponent)
template <typename T>
__global__ void d2t_kernel(const double* __restrict__ src, T* __restrict__ dst, int64_t n,
                           int64_t stride, int64_t bcount, int exp2) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * bcount) return;
  const int64_t e = idx / bcount, l = idx - (idx / bcount) * bcount;
  dst[e * stride + l] = (T)(exp2 ? ldexp(src[e], exp2) : src[e]);
}

template <typename T>
__global__ void t2d_kernel(const T* __restrict__ src, int64_t stride, double* __restrict__ dst, int64_t n, int exp2) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < n) dst[idx] = exp2 ? ldexp((double)src[idx * stride], -exp2) : (double)src[idx * stride];
}

template <typename T>
__global__ void scale_pow2_kernel(T* p, int64_t n, int exp2) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < n) p[idx] = (T)ldexp((double)p[idx], exp2);
}

template <typename T>
__global__ void fill_kernel(T* dst, int64_t n, double v) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < n) dst[idx] = (T)v;
}

cudaError_t launch_convert_d2t(int dtype, const double* src, void* dst, int64_t n, int64_t stride,
                               int64_t bcount, cudaStream_t s, int exp2) {
  const int64_t tot = n * bcount;
  if (tot == 0) return cudaSuccess;
  const unsigned g = (unsigned)((tot + 255) / 256);
  if (dtype == 0) d2t_kernel<float><<<g, 256, 0, s>>>(src, (float*)dst, n, stride, bcount, exp2);
  else d2t_kernel<double><<<g, 256, 0, s>>>(src, (double*)dst, n, stride, bcount, exp2);
  return cudaGetLastError();
}

cudaError_t launch_convert_t2d(int dtype, const void* src, int64_t stride, double* dst, int64_t n,
                               cudaStream_t s, int exp2) {
  if (n == 0) return cudaSuccess;
  const unsigned g = (unsigned)((n + 255) / 256);
  if (dtype == 0) t2d_kernel<float><<<g, 256, 0, s>>>((const float*)src, stride, dst, n, exp2);
  else t2d_kernel<double><<<g, 256, 0, s>>>((const double*)src, stride, dst, n, exp2);
  return cudaGetLastError();
}

cudaError_t launch_scale_pow2(int dtype, void* p, int64_t n, int exp2, cudaStream_t s) {
  if (n == 0 || exp2 == 0) return cudaSuccess;
  const unsigned g = (unsigned)((n + 255) / 256);
  if (dtype == 0) scale_pow2_kernel<float><<<g, 256, 0, s>>>((float*)p, n, exp2);
  else scale_pow2_kernel<double><<<g, 256, 0, s>>>((double*)p, n, exp2);
  return cudaGetLastError();
}

template <typename T>
__global__ void mul_kernel(T* __restrict__ dst, const T* __restrict__ a, const T* __restrict__ b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = a[i] * b[i];
}

// dst = a * b elementwise (a separator's final table from its collect message and
// distribute ratio)
cudaError_t launch_mul(int dtype, void* dst, const void* a, const void* b, int64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (dtype == 0) mul_kernel<float><<<g, 256, 0, s>>>((float*)dst, (const float*)a, (const float*)b, n);
  else mul_kernel<double><<<g, 256, 0, s>>>((double*)dst, (const double*)a, (const double*)b, n);
  return cudaGetLastError();
}

cudaError_t launch_fill(int dtype, void* dst, int64_t n, double v, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const unsigned g = (unsigned)((n + 255) / 256);
  if (dtype == 0) fill_kernel<float><<<g, 256, 0, s>>>((float*)dst, n, v);
  else fill_kernel<double><<<g, 256, 0, s>>>((double*)dst, n, v);
  return cudaGetLastError();
}

// ---- evidence masks (apply_evidence, propagate.py:243-260) ----
// mask_v[d][b] = 1 except d != observed state of case b.  Masks of the listed
// variables are reset to ones, then every observation zeroes its lane.
__global__ void ev_fill_kernel(void* aux, int dtype, const int32_t* __restrict__ vars, int nv,
                               const int64_t* __restrict__ var_off, const int32_t* __restrict__ cards, int B) {
  const int k = blockIdx.y;
  if (k >= nv) return;
  const int v = vars[k];
  const int64_t len = (int64_t)cards[v] * B, off = var_off[v];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    if (dtype == 0) ((float*)aux)[off + i] = 1.0f;
    else ((double*)aux)[off + i] = 1.0;
  }
}

__global__ void ev_zero_kernel(void* aux, int dtype, const int32_t* __restrict__ obs, int n,
                               const int64_t* __restrict__ var_off, const int32_t* __restrict__ cards, int B) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = obs[3 * i], v = obs[3 * i + 1], x = obs[3 * i + 2];
  const int card = cards[v];
  const int64_t base = var_off[v];
  const int lo = b < 0 ? 0 : b, hi = b < 0 ? B : b + 1;
  for (int l = lo; l < hi; ++l)
    for (int d = 0; d < card; ++d)
      if (d != x) {
        if (dtype == 0) ((float*)aux)[base + (int64_t)d * B + l] = 0.0f;
        else ((double*)aux)[base + (int64_t)d * B + l] = 0.0;
      }
}

cudaError_t launch_ev_fill(void* aux, int dtype, const int32_t* vars, int nv, const int64_t* var_off,
                           const int32_t* cards, int B, cudaStream_t s) {
  if (nv == 0) return cudaSuccess;
  ev_fill_kernel<<<dim3(8, nv), 256, 0, s>>>(aux, dtype, vars, nv, var_off, cards, B);
  return cudaGetLastError();
}

// Per-case code of an evidence mask (virtual separators, VDesc): -1 all ones
// (unobserved), -2 all zeros (conflicting observations), else the one state
// left (ev_zero leaves at most one).
__global__ void ev_code_kernel(const void* aux, int dtype, const VCodeTask* __restrict__ tasks, int B,
                               int32_t* __restrict__ codes) {
  const VCodeTask t = tasks[blockIdx.y];
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
    int ones = 0, first = -1;
    for (int d = 0; d < t.card; ++d) {
      const int64_t i = t.mask_off + (int64_t)d * B + b;
      const bool one = dtype == 0 ? ((const float*)aux)[i] != 0.0f : ((const double*)aux)[i] != 0.0;
      ones += one;
      if (one && first < 0) first = d;
    }
    codes[(int64_t)blockIdx.y * B + b] = ones == t.card ? -1 : ones == 0 ? -2 : first;
  }
}

cudaError_t launch_ev_code(const void* aux, int dtype, const VCodeTask* tasks, int nt, int B, int32_t* codes,
                           cudaStream_t s) {
  if (nt == 0) return cudaSuccess;
  ev_code_kernel<<<dim3((B + 255) / 256, nt), 256, 0, s>>>(aux, dtype, tasks, B, codes);
  return cudaGetLastError();
}

cudaError_t launch_ev_zero(void* aux, int dtype, const int32_t* obs, int n, const int64_t* var_off,
                           const int32_t* cards, int B, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  ev_zero_kernel<<<(n + 127) / 128, 128, 0, s>>>(aux, dtype, obs, n, var_off, cards, B);
  return cudaGetLastError();
}

// ---- initialize (propagate.py:204-222): clique tables = product of assigned CPTs ----
// One CTA row per clique (blockIdx.y); every entry decodes its digits for each
// CPT variable (clique stride, card) and gathers the CPT value (CPT stride).
__global__ void init_kernel(void* base, int dtype, const double* __restrict__ cpt,
                            const InitClique* __restrict__ cl, const InitTerm* __restrict__ terms,
                            const int64_t* __restrict__ vdesc) {
  const InitClique c = cl[blockIdx.y];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < c.size;
       e += (int64_t)gridDim.x * blockDim.x) {
    double p = 1.0;
    for (int t = c.first_term; t < c.first_term + c.n_terms; ++t) {
      const InitTerm tm = terms[t];
      int64_t idx = 0;
      for (int v = 0; v < tm.nv; ++v) {
        const int64_t* d = vdesc + 3 * (tm.first_var + v);
        idx += ((e / d[0]) % d[1]) * d[2];
      }
      p *= cpt[tm.cpt_off + idx];
    }
    if (dtype == 0) ((float*)base)[c.off + e] = (float)p;
    else ((double*)base)[c.off + e] = p;
  }
}

cudaError_t launch_init(void* base, int dtype, const double* cpt, const InitClique* cl, int n_cliques,
                        const InitTerm* terms, const int64_t* vdesc, int64_t max_size, cudaStream_t s) {
  if (n_cliques == 0) return cudaSuccess;
  const unsigned gx = (unsigned)std::min<int64_t>((max_size + 255) / 256, 1024);
  init_kernel<<<dim3(gx, n_cliques), 256, 0, s>>>(base, dtype, cpt, cl, terms, vdesc);
  return cudaGetLastError();
}

// ---- K0: device μ builder, μ[j][p] = row_base(j) + rest(p) (compiler.py:285-304) ----
struct MuDims {
  int nsd, nrd;
  int64_t sc[32], ss[32], rc[32], rs[32];
};

__global__ void mapping_table_kernel(int64_t* __restrict__ out, int64_t n_sep, int64_t n_rest, MuDims m) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_sep * n_rest) return;
  int64_t j = idx / n_rest, p = idx - (idx / n_rest) * n_rest;
  int64_t v = 0;
  for (int d = m.nsd - 1; d >= 0; --d) {  // separator digits, separator order, last fastest
    v += (j % m.sc[d]) * m.ss[d];
    j /= m.sc[d];
  }
  for (int d = m.nrd - 1; d >= 0; --d) {  // remaining clique positions, ascending
    v += (p % m.rc[d]) * m.rs[d];
    p /= m.rc[d];
  }
  out[idx] = v;
}

cudaError_t launch_mapping_table(int64_t* out, int64_t n_sep, int64_t n_rest, int nsd,
                                 const int64_t* sep_card, const int64_t* sep_stride, int nrd,
                                 const int64_t* rest_card, const int64_t* rest_stride, cudaStream_t s) {
  MuDims m;
  if (nsd > 32 || nrd > 32) return cudaErrorInvalidValue;
  m.nsd = nsd;
  m.nrd = nrd;
  for (int i = 0; i < nsd; ++i) { m.sc[i] = sep_card[i]; m.ss[i] = sep_stride[i]; }
  for (int i = 0; i < nrd; ++i) { m.rc[i] = rest_card[i]; m.rs[i] = rest_stride[i]; }
  const int64_t n = n_sep * n_rest;
  if (n == 0) return cudaSuccess;
  mapping_table_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(out, n_sep, n_rest, m);
  return cudaGetLastError();
}

// ---- engine-protocol path: Alg. 1 driven by host μ tables (paper §3.2) ----
// phase 0: one warp per separator entry j: star_j = Σ_p φ_src[μ_src[j][p]]
//          (lane-strided, fixed shuffle order), error check, ratio, sep_j = star_j.
// phase 1: one thread per (j, p): φ_tgt[μ_tgt[j][p]] *= ratio_j.
template <typename I>
__global__ void mu_marg_kernel(const double* __restrict__ src, double* __restrict__ sep,
                               double* __restrict__ ratio, const I* __restrict__ mu, int64_t row,
                               int64_t n_sep, int* err) {
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= n_sep) return;
  double s = 0.0;
  const I* m = mu + j * row;
  for (int64_t p = lane; p < row; p += 32) s += src[m[p]];
  s = warp_sum(s);
  if (lane == 0) {
    const double old = sep[j];
    if (old == 0.0 && s != 0.0) atomicOr(err, EB_INCONSISTENT);
    ratio[j] = (old != 0.0) ? s / old : 0.0;
    sep[j] = s;
  }
}

template <typename I>
__global__ void mu_scatter_kernel(double* __restrict__ tgt, const double* __restrict__ ratio,
                                  const I* __restrict__ mu, int64_t row, int64_t n_sep) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_sep * row) return;
  const int64_t j = idx / row;
  tgt[mu[idx]] *= ratio[j];
}

cudaError_t launch_mu_message(const double* src, double* tgt, double* sep, double* ratio,
                              const void* mu_src, int64_t row_src, const void* mu_tgt,
                              int64_t row_tgt, int64_t n_sep, int is64, int* err, int phase,
                              cudaStream_t s) {
  if (n_sep == 0) return cudaSuccess;
  if (phase == 0) {
    const int64_t threads = n_sep * 32;
    const unsigned g = (unsigned)((threads + 255) / 256);
    if (is64) mu_marg_kernel<int64_t><<<g, 256, 0, s>>>(src, sep, ratio, (const int64_t*)mu_src, row_src, n_sep, err);
    else mu_marg_kernel<int32_t><<<g, 256, 0, s>>>(src, sep, ratio, (const int32_t*)mu_src, row_src, n_sep, err);
  } else {
    const int64_t n = n_sep * row_tgt;
    if (n == 0) return cudaSuccess;
    const unsigned g = (unsigned)((n + 255) / 256);
    if (is64) mu_scatter_kernel<int64_t><<<g, 256, 0, s>>>(tgt, ratio, (const int64_t*)mu_tgt, row_tgt, n_sep);
    else mu_scatter_kernel<int32_t><<<g, 256, 0, s>>>(tgt, ratio, (const int32_t*)mu_tgt, row_tgt, n_sep);
  }
  return cudaGetLastError();
}

}  // namespace jt
