// Contraction kernels of the shared-base batch path, sm_100a:
// templates only.  The launchers live in jt_contract_{tile,tilep,rowi}.cu so the
// instantiations compile in parallel.
#pragma once
#include "jt_internal.h"
#include "jt_device.cuh"
#include <algorithm>
#include <type_traits>
#include <utility>

namespace jt {

// ---- contraction passes (shared-base batches) ----
// Hugin update of VEC consecutive case lanes of one output entry (element
// offset j of case 0) from sums in the accumulator type A (fp32 sums of the
// unfolded fp32 kernels stay fp32: the ratio and product are the same IEEE
// results as via fp64); returns "nonzero / 0 seen" for the caller to flag once.
template <typename T, typename A, int VEC>
__device__ __forceinline__ bool finalize_lanes(int kind, int64_t out_off, int64_t ratio_off, int64_t out2_off,
                                               int64_t j, const A (&star)[VEC], const T (&old)[VEC], T* aux,
                                               double* qout, bool cs = false) {
  if (kind == OUT_RAW) {
#pragma unroll
    for (int l = 0; l < VEC; ++l) qout[out_off + j + l] = (double)star[l];
    return false;
  }
  T nw[VEC];
  if (kind == OUT_SEP_FRESH || kind == OUT_SEP_DRATIO) {
#pragma unroll
    for (int l = 0; l < VEC; ++l) nw[l] = (T)star[l];
    T* dst = aux + (kind == OUT_SEP_FRESH ? out_off : ratio_off) + j;
    if (cs) store_vec_cs<T, VEC>(dst, nw);
    else store_vec<T, VEC>(dst, nw);
    return false;
  }
  T rt[VEC];
  bool bad = false;
#pragma unroll
  for (int l = 0; l < VEC; ++l) {
    const A o = (A)old[l];
    if (kind == OUT_SEP_DFRESH) {
      rt[l] = (T)(o != (A)0 ? star[l] : (A)0);
      nw[l] = (T)(o * star[l]);
    } else {
      bad |= (o == (A)0 && star[l] != (A)0);
      rt[l] = (T)(o != (A)0 ? star[l] / o : (A)0);
      nw[l] = (T)star[l];
    }
  }
  const bool keep = out2_off != OUT2_SKIP;
  if (cs) {
    store_vec_cs<T, VEC>(aux + ratio_off + j, rt);
    if (keep) store_vec_cs<T, VEC>(aux + (out2_off >= 0 ? out2_off : out_off) + j, nw);
  } else {
    store_vec<T, VEC>(aux + ratio_off + j, rt);
    if (keep) store_vec<T, VEC>(aux + (out2_off >= 0 ? out2_off : out_off) + j, nw);
  }
  return bad;
}

template <typename T> struct CTraits;
template <> struct CTraits<float> { static constexpr int VEC = 4; };
template <> struct CTraits<double> { static constexpr int VEC = 2; };

// Per-warp cp.async ring of the contraction kernel: stage = NG factor-row
// slices (16 B per lane each) + the TMC-entry W row; depth by a per-warp budget
// (fold kernels also hold 64 KB of fp64 accumulators per CTA).
#ifndef CON_RING_NF
#define CON_RING_NF 2048
#endif
#ifndef CON_RING_F
#define CON_RING_F 2048
#endif
// CON_WRING: the stage also carries the k's W row (TMC entries, copied by the
// first lanes, read by all after a warp barrier), so W loads are as far ahead
// as the factor slices instead of one k in registers.
#ifndef CON_WRING
#define CON_WRING 1
#endif
template <typename T, int NG, bool FOLD> struct CRing {
  static constexpr int SF = NG * 512;                          // NG factor slices of 16 B per lane
  static constexpr int WB = CON_WRING ? TMC * (int)sizeof(T) : 0;  // the W row
  static constexpr int SB = SF + WB;                           // one stage
  static constexpr int BUDGET = FOLD ? CON_RING_F : CON_RING_NF;
  static constexpr int D = NG == 0 ? (CON_WRING ? 4 : 2) : (BUDGET / SF > 8 ? 8 : (BUDGET / SF < 2 ? 2 : BUDGET / SF));
  static constexpr size_t BYTES = (size_t)(NT / 32) * D * SB;
};
constexpr size_t CFOLD_SMEM = (size_t)TMC * 4 * NT * sizeof(double);  // fp32 fold accumulators

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// One warp per unit (i, tile of TMC rows of S', share of the case chunks); each
// epilogue inputs (old separator values, E factors) are read once: streaming
// loads keep them from evicting the units' W rows from L1
#ifndef CON_EPI_CS
#define CON_EPI_CS 1
#endif
template <typename T, int VEC>
__device__ __forceinline__ void con_epi_load(const T* p, T (&v)[VEC]) {
  if (CON_EPI_CS) load_vec_cs<T, VEC>(p, v);
  else load_vec<T, VEC>(p, v);
}

// Epilogue of one half tile (TMC/2 rows) for one output kind: the rows' old
// separator values are loaded before any store (stores would otherwise order
// the loads behind them); returns "nonzero / 0 seen".
template <typename T, typename A, int VEC, int KIND, bool FOLD, int NG, bool PRM = false>
__device__ __forceinline__ bool contract_epilogue_half(const CPass* __restrict__ P, const CArgs& a, int h, int rows,
                                                       int s0, const int32_t* __restrict__ ti,
                                                       const int32_t* __restrict__ ts, int b0,
                                                       const T (&part)[TMC][VEC], const double* cacc) {
  T* __restrict__ aux = reinterpret_cast<T*>(a.aux);
  const T* __restrict__ aux_c = aux;
  const int nE = P->nE;
  int jo[TMC / 2];
  const int jb = __ldg(ti + NG + nE);
#pragma unroll
  for (int r = 0; r < TMC / 2; ++r) {
    const int32_t* q = ts + (int64_t)(s0 + h + r) * (nE + 1) + nE;
    jo[r] = h + r < rows ? jb + (PRM ? *q : __ldg(q)) : 0;
  }
  T old[TMC / 2][VEC];
#pragma unroll
  for (int r = 0; r < TMC / 2; ++r) {
    if ((KIND == OUT_SEP || KIND == OUT_SEP_DFRESH) && h + r < rows)
      con_epi_load<T, VEC>(aux_c + P->out_off + jo[r] + b0, old[r]);
    else
#pragma unroll
      for (int l = 0; l < VEC; ++l) old[r][l] = (T)0;
  }
  bool bad = false;
#pragma unroll
  for (int r = 0; r < TMC / 2; ++r) {
    if (h + r >= rows) continue;
    A v[VEC];
#pragma unroll
    for (int l = 0; l < VEC; ++l) v[l] = FOLD ? (A)cacc[((h + r) * VEC + l) * NT + threadIdx.x] : (A)part[h + r][l];
    if (nE > 0) {
      const int32_t* tsr = ts + (int64_t)(s0 + h + r) * (nE + 1);
      for (int e = 0; e < nE; ++e) {
        T f[VEC];
        con_epi_load<T, VEC>(aux_c + P->efac_off[e] + __ldg(ti + NG + e) + (PRM ? tsr[e] : __ldg(tsr + e)) + b0, f);
#pragma unroll
        for (int l = 0; l < VEC; ++l) v[l] *= (A)f[l];
      }
    }
    bad |= finalize_lanes<T, A, VEC>(KIND, P->out_off, P->ratio_off, P->out2_off, (int64_t)jo[r] + b0, v, old[r], aux,
                                     a.qout, a.stream_epi != 0);
  }
  return bad;
}

// One warp per unit (i, tile of TMC rows of S', share of the case chunks); each
// lane owns VEC consecutive cases.  Per k: the product of the NG factor rows
// (one VEC-vector per lane, coalesced across the warp) is reused by the TMC
// rows of W: TMC x VEC FMAs per lane per k.  Factor slices stream through a
// lane-private cp.async ring D stages deep (each lane consumes only what it
// copied: no barriers, no registers held), so D k-steps of factor loads are in
// flight per warp; the W row (a warp-uniform 8-entry broadcast, L1-resident
// across the unit's case-chunk warps) is prefetched one k ahead in registers.
// fp32 sums stay in registers for CKF consecutive k and are then folded into
// per-thread fp64 accumulators in shared memory (fp64 passes accumulate in
// registers).
#ifndef CON_MINB
#define CON_MINB 2
#endif
#ifndef CON_FOLD_K
#define CON_FOLD_K 32  // fp32 k-terms per register partial before the fp64 fold (16: -1.5%)
#endif
#ifndef CON_WPF
#define CON_WPF 1
#endif
template <typename T, bool FOLD, int NG, bool PRM>
__device__ __forceinline__ void tile_body(const CArgs& a, const CPass* __restrict__ P0, const int32_t* __restrict__ tk0,
                                          const int32_t* __restrict__ ts0) {
  constexpr int VEC = CTraits<T>::VEC;
  constexpr int WV = sizeof(T) == 4 ? 4 : 2;  // W row loaded as TMC / WV vectors
  using R = CRing<T, NG, FOLD>;
  using A = typename std::conditional<FOLD || sizeof(T) == 8, double, T>::type;  // epilogue type
  static_assert(TMC == 8, "W rows are TMC entries");
  extern __shared__ __align__(16) unsigned char csm_c[];
  double* cacc = reinterpret_cast<double*>(csm_c);  // FOLD: [TMC * VEC][NT] fp64 accumulators
  const int lane = threadIdx.x & 31;
  // this warp's stage 0; stage q: slice g of lane l at + q * SB + g * 512 + l * 16, W row at + q * SB + SF
  unsigned char* const ring = csm_c + (FOLD ? CFOLD_SMEM : 0) + (size_t)(threadIdx.x >> 5) * R::D * R::SB;
  constexpr bool WR = CON_WRING != 0;
  constexpr int WL = R::WB / 16;  // lanes copying the W row (16 B each)
  const T* __restrict__ W = reinterpret_cast<const T*>(a.w);
  const T* __restrict__ aux_c = reinterpret_cast<const T*>(a.aux);
  const int n_warps = gridDim.x * (NT / 32);
  int pi = 0;
  for (int64_t u = blockIdx.x * (NT / 32) + (threadIdx.x >> 5); u < a.n_units; u += n_warps) {
    int64_t ul;
    if (PRM) {
      ul = u;  // one pass per launch, starting at unit 0
    } else if (a.interleave) {
      pi = (int)(u % a.n_passes);
      ul = u / a.n_passes;
    } else {
      while (pi + 1 < a.n_passes && u >= a.passes[pi + 1].unit0) ++pi;
      while (pi > 0 && u < a.passes[pi].unit0) --pi;
      ul = u - a.passes[pi].unit0;
    }
    const CPass* __restrict__ P = PRM ? P0 : a.passes + pi;
    const int nT = P->nT, nCG = P->nCG, nKS = P->nKS;
    // unit = (i, t, ks, cg), case chunk fastest: concurrent warps share factor rows
    // (cmaj: case chunk slowest)
    int cg, ks, t;
    int64_t i;
    if (P->cmaj) {
      const int64_t per = (int64_t)P->nI * nT * nKS;
      cg = (int)(ul / per);
      const int64_t r = ul - (int64_t)cg * per;
      ks = (int)(r % nKS);
      t = (int)((r / nKS) % nT);
      i = r / ((int64_t)nKS * nT);
    } else {
      cg = (int)(ul % nCG);
      ks = (int)((ul / nCG) % nKS);
      t = (int)((ul / ((int64_t)nCG * nKS)) % nT);
      i = ul / ((int64_t)nCG * nKS * nT);
    }
    const int nS = P->nS, nE = P->nE;
    const int kb = ks * P->kch;                      // this unit's k range [kb, kb + nK)
    const int nK = min(P->nK - kb, P->kch);
    const int nKall = P->nK;
    const int nSp = (nS + 7) & ~7;
    const int bstep = 32 * VEC * nCG;
    const int s0 = t * TMC;
    const int rows = min(TMC, nS - s0);
    const int32_t* __restrict__ ti = a.tab + P->ti_off + i * (NG + nE + 1);
    const int32_t* __restrict__ tk = (PRM ? tk0 : a.tab + P->tk_off) + (int64_t)kb * NG;
    const int32_t* __restrict__ ts = PRM ? ts0 : a.tab + P->ts_off;
    const T* __restrict__ wrow = W + P->w_off + (i * (int64_t)nKall + kb) * nSp + s0;
    const T* gq[NG > 0 ? NG : 1];  // factor g at (i, k = kb, case 0)
#pragma unroll
    for (int g = 0; g < NG; ++g) gq[g] = aux_c + P->gfac_off[g] + __ldg(ti + g);
    for (int b0 = cg * 32 * VEC + lane * VEC; b0 < a.B; b0 += bstep) {
      // lanes of this warp with cases left (a prefix): the W row copy and the warp barrier
      const int na = min(32, (a.B - (b0 - lane * VEC) + VEC - 1) / VEC);
      const unsigned wm = na >= 32 ? 0xffffffffu : ((1u << na) - 1u);
      const T* gb[NG > 0 ? NG : 1];  // this lane's case vector of each factor (per k: + the k-offset)
#pragma unroll
      for (int g = 0; g < NG; ++g) gb[g] = gq[g] + b0;
      auto issue = [&](int k, unsigned char* sp) {
#pragma unroll
        for (int g = 0; g < NG; ++g)
          cp_async16(sp + g * 512 + lane * 16, gb[g] + (PRM ? tk[k * NG + g] : __ldg(tk + k * NG + g)));
        if (WR) {
          const T* wk = wrow + k * nSp;
          if (na >= WL) {
            if (lane < WL) cp_async16(sp + R::SF + lane * 16, wk + lane * (16 / (int)sizeof(T)));
          } else if (lane == 0) {
#pragma unroll
            for (int c = 0; c < WL; ++c) cp_async16(sp + R::SF + c * 16, wk + c * (16 / (int)sizeof(T)));
          }
        }
      };
      if (NG > 0 || WR) {
#pragma unroll
        for (int q = 0; q < R::D - 1; ++q) {
          if (q < nK) issue(q, ring + q * R::SB);
          cp_async_commit();
        }
      }
      T part[TMC][VEC];
#pragma unroll
      for (int r = 0; r < TMC; ++r)
#pragma unroll
        for (int l = 0; l < VEC; ++l) part[r][l] = (T)0;
      if (FOLD)
#pragma unroll
        for (int q = 0; q < TMC * VEC; ++q) cacc[q * NT + threadIdx.x] = 0.0;
      constexpr int WPF = WR ? 1 : CON_WPF;
      T wn[WPF][TMC];  // !WR: W rows of the next CON_WPF k
      if (!WR) {
#pragma unroll
        for (int q = 0; q < WPF; ++q)
#pragma unroll
          for (int h = 0; h < TMC / WV; ++h) {
            T x[WV];
            if (q < nK) load_vec_ro<T, WV>(wrow + (int64_t)q * nSp + h * WV, x);
#pragma unroll
            for (int l = 0; l < WV; ++l) wn[q][h * WV + l] = q < nK ? x[l] : (T)0;
          }
      }
      unsigned char* sp = ring;                          // stage of k
      unsigned char* spn = ring + (R::D - 1) * R::SB;    // stage refilled at k (k + D - 1)
      int since = 0;
      for (int k = 0; k < nK; ++k) {
        T w[TMC];
        if (NG > 0 || WR) cp_async_wait<R::D - 2>();
        if (WR) {
          __syncwarp(wm);  // the W row of this stage was copied by the first lanes
#pragma unroll
          for (int h = 0; h < TMC / WV; ++h) {
            T x[WV];
            load_vec<T, WV>(reinterpret_cast<const T*>(sp + R::SF) + h * WV, x);
#pragma unroll
            for (int l = 0; l < WV; ++l) w[h * WV + l] = x[l];
          }
        } else {
#pragma unroll
          for (int r = 0; r < TMC; ++r) w[r] = wn[0][r];
#pragma unroll
          for (int q = 0; q + 1 < WPF; ++q)
#pragma unroll
            for (int r = 0; r < TMC; ++r) wn[q][r] = wn[q + 1][r];
          if (k + WPF < nK) {
#pragma unroll
            for (int h = 0; h < TMC / WV; ++h) {
              T x[WV];
              load_vec_ro<T, WV>(wrow + (int64_t)(k + WPF) * nSp + h * WV, x);
#pragma unroll
              for (int l = 0; l < WV; ++l) wn[WPF - 1][h * WV + l] = x[l];
            }
          }
        }
        T pv[VEC];
#pragma unroll
        for (int l = 0; l < VEC; ++l) pv[l] = (T)1;
        if (NG > 0 || WR) {
#pragma unroll
          for (int g = 0; g < NG; ++g) {
            T f[VEC];
            load_vec<T, VEC>(reinterpret_cast<const T*>(sp + g * 512 + lane * 16), f);
#pragma unroll
            for (int l = 0; l < VEC; ++l) pv[l] = g == 0 ? f[l] : pv[l] * f[l];
          }
          // refill the stage consumed last iteration (this lane's own slot)
          if (k + R::D - 1 < nK) issue(k + R::D - 1, spn);
          cp_async_commit();
          spn = sp;
          sp = sp + R::SB == ring + R::D * R::SB ? ring : sp + R::SB;
        }
#pragma unroll
        for (int r = 0; r < TMC; ++r)
#pragma unroll
          for (int l = 0; l < VEC; ++l) part[r][l] += w[r] * pv[l];
        if (FOLD && ++since == CON_FOLD_K) {
          since = 0;
#pragma unroll
          for (int r = 0; r < TMC; ++r)
#pragma unroll
            for (int l = 0; l < VEC; ++l) {
              cacc[(r * VEC + l) * NT + threadIdx.x] += (double)part[r][l];
              part[r][l] = (T)0;
            }
        }
      }
      if (FOLD)
#pragma unroll
        for (int r = 0; r < TMC; ++r)
#pragma unroll
          for (int l = 0; l < VEC; ++l) {
            cacc[(r * VEC + l) * NT + threadIdx.x] += (double)part[r][l];
            part[r][l] = (T)0;
          }
      if (nKS > 1) {
        // K-split: park this chunk's sums; the last warp of the (i, t, case chunk)
        // group adds the nKS partials in chunk order and runs the epilogue
        const int64_t grp = ((i * nT + t) * (int64_t)nCG + cg);
        double* pp = a.partials + P->part_off + (grp * nKS) * (TMC * 32 * VEC);
#pragma unroll
        for (int r = 0; r < TMC; ++r)
#pragma unroll
          for (int l = 0; l < VEC; ++l)
            __stcg(pp + (int64_t)ks * (TMC * 32 * VEC) + (r * 32 + lane) * VEC + l,
                   FOLD ? cacc[(r * VEC + l) * NT + threadIdx.x] : (double)part[r][l]);
        __threadfence();
        __syncwarp();  // K-split passes need B % (32 VEC) == 0 (compile_contract): every lane is here
        int arrived = 0;
        if (lane == 0) arrived = atomicAdd(a.counters + P->cnt_off + grp, 1);
        arrived = __shfl_sync(0xffffffffu, arrived, 0);
        if (arrived != nKS - 1) continue;
        __threadfence();
        if (lane == 0) a.counters[P->cnt_off + grp] = 0;
#pragma unroll
        for (int r = 0; r < TMC; ++r)
#pragma unroll
          for (int l = 0; l < VEC; ++l) {
            double t_ = 0.0;
            for (int q = 0; q < nKS; ++q) t_ += __ldcg(pp + (int64_t)q * (TMC * 32 * VEC) + (r * 32 + lane) * VEC + l);
            if (FOLD) cacc[(r * VEC + l) * NT + threadIdx.x] = t_;
            else part[r][l] = (T)t_;  // fp64 passes only (fp32 K-split passes always fold)
          }
      }
      bool bad = false;
      switch (P->out_kind) {  // warp-uniform: one specialised epilogue per kind
        case OUT_SEP_FRESH:
#pragma unroll
          for (int h = 0; h < TMC; h += TMC / 2)
            contract_epilogue_half<T, A, VEC, OUT_SEP_FRESH, FOLD, NG, PRM>(P, a, h, rows, s0, ti, ts, b0, part, cacc);
          break;
        case OUT_RAW:
#pragma unroll
          for (int h = 0; h < TMC; h += TMC / 2)
            contract_epilogue_half<T, A, VEC, OUT_RAW, FOLD, NG, PRM>(P, a, h, rows, s0, ti, ts, b0, part, cacc);
          break;
        case OUT_SEP_DFRESH:
#pragma unroll
          for (int h = 0; h < TMC; h += TMC / 2)
            contract_epilogue_half<T, A, VEC, OUT_SEP_DFRESH, FOLD, NG, PRM>(P, a, h, rows, s0, ti, ts, b0, part, cacc);
          break;
        case OUT_SEP_DRATIO:
#pragma unroll
          for (int h = 0; h < TMC; h += TMC / 2)
            contract_epilogue_half<T, A, VEC, OUT_SEP_DRATIO, FOLD, NG, PRM>(P, a, h, rows, s0, ti, ts, b0, part, cacc);
          break;
        default:
#pragma unroll
          for (int h = 0; h < TMC; h += TMC / 2)
            bad |= contract_epilogue_half<T, A, VEC, OUT_SEP, FOLD, NG, PRM>(P, a, h, rows, s0, ti, ts, b0, part, cacc);
      }
      if (bad) atomicOr(a.err, EB_INCONSISTENT);
    }
  }
}

template <typename T, bool FOLD, int NG>
__global__ void __launch_bounds__(NT, CON_MINB) contract_kernel(const CArgs a) {
  pdl_enter();
  tile_body<T, FOLD, NG, false>(a, nullptr, nullptr, nullptr);
}

// one tile pass per launch, its descriptor and k / s' tables in the kernel parameters
template <typename T, bool FOLD, int NG>
__global__ void __launch_bounds__(NT, CON_MINB) contract_p_kernel(const CArgs a, const __grid_constant__ TileParam tp) {
  pdl_enter();
  tile_body<T, FOLD, NG, true>(a, &tp.cp, tp.tk, tp.ts);
}

// Row-per-i contraction passes (nS == 1: every output variable is also a factor
// variable, e.g. Hugin messages between cliques whose separators cover each
// other): no W reuse exists, so the unit is TMC consecutive i values and the
// warp streams their factor rows — KU x TMC x nG independent vector loads in
// flight per lane — with the same epilogue.
// occupancy / loads-in-flight trade-offs, chosen by a variant sweep on the c5
// batch program (tools/build_variant.sh, tools/sweep_variants.sh; profiles r06):
// one or two k per step at 4-8 CTAs/SM beat deeper per-warp unrolling
#ifndef ROWI_KU_NF
#define ROWI_KU_NF 1
#endif
#ifndef ROWI_MINB_NF
#define ROWI_MINB_NF 6
#endif
#ifndef ROWI_KU_F
#define ROWI_KU_F 2
#endif
#ifndef ROWI_MINB_F
#define ROWI_MINB_F 5
#endif
#ifndef ROWI_MINB_D
#define ROWI_MINB_D 6
#endif
// LONGK: passes with long K sums (nK >= 16) keep ROWI_KU_L values of k in flight
// per lane (their loads would otherwise chain one memory latency per k) at a
// larger register budget
#ifndef ROWI_KU_L
#define ROWI_KU_L 4
#endif
#ifndef ROWI_MINB_L
#define ROWI_MINB_L 4
#endif
// Virtual separators (VDesc): per case lane, the column of the entry's Wv row
// the leaf's collect pass would have summed to — the observed state, nK (the row
// sum: unobserved / no evidence) — or -1 (conflicting evidence: zero).
template <int VEC>
__device__ __forceinline__ void vsep_cols(const VDesc& d, const int32_t* __restrict__ codes, int b0, int (&c)[VEC]) {
  if (d.code_off < 0) {
#pragma unroll
    for (int l = 0; l < VEC; ++l) c[l] = d.nK;
    return;
  }
  if constexpr (VEC == 4) {
    const int4 x = __ldg(reinterpret_cast<const int4*>(codes + d.code_off + b0));
    c[0] = x.x, c[1] = x.y, c[2] = x.z, c[3] = x.w;
  } else if constexpr (VEC == 2) {
    const int2 x = __ldg(reinterpret_cast<const int2*>(codes + d.code_off + b0));
    c[0] = x.x, c[1] = x.y;
  } else {
#pragma unroll
    for (int l = 0; l < VEC; ++l) c[l] = __ldg(codes + d.code_off + b0 + l);
  }
#pragma unroll
  for (int l = 0; l < VEC; ++l) c[l] = c[l] >= 0 ? c[l] : c[l] == -1 ? d.nK : -1;
}
// the value at a Wv row (pointer to its first column) for the lanes' columns
template <typename T, int VEC>
__device__ __forceinline__ void vsep_gather(const T* __restrict__ row, const int (&c)[VEC], T (&f)[VEC]) {
#pragma unroll
  for (int l = 0; l < VEC; ++l) f[l] = c[l] >= 0 ? __ldg(row + c[l]) : (T)0;
}
template <typename T, int VEC>
__device__ __forceinline__ void vsep_pick(int v, const T (&vv)[CMAXV][VEC], T (&f)[VEC]) {
#pragma unroll
  for (int l = 0; l < VEC; ++l) f[l] = v == 0 ? vv[0][l] : vv[1][l];
}

// NGC: the pass's factor count when fixed at compile time (1..4; 0 = read from
// the descriptor, loops bounded by CMAXG and predicated per factor)
// VS: the pass reads virtual separators (the epilogue evaluates them; a separate
// instantiation at a larger register budget, so plain passes keep theirs)
#ifndef ROWI_MINB_V
#define ROWI_MINB_V 4
#endif
#ifndef ROWI_KU_V
#define ROWI_KU_V 1  // k per step of the VS variant (2 and 4 measured slower)
#endif
// KP: output kinds fixed at compile time — 1: (collect FRESH, no second output),
// 2: (DFRESH, ratio-only second output), 3: (ratio-only, none); 0: read from the descriptor
template <typename T, bool FOLD, bool LONGK, bool PRM, bool XW = false, int NGC = 0, bool VS = false, int KP = 0>
__device__ __forceinline__ void rowi_body(const CArgs& a, const CPass* __restrict__ P0, const int32_t* __restrict__ tk0,
                                          const int32_t* __restrict__ ts0) {
  // one i per warp unit (few registers: three or four CTAs per SM), KU values
  // of k in flight, each with its nG factor-row vectors
  constexpr int VEC = CTraits<T>::VEC;
  constexpr int KU = LONGK ? ROWI_KU_L : VS ? ROWI_KU_V : FOLD ? ROWI_KU_F : ROWI_KU_NF;
  constexpr int KF = 16;
  T* __restrict__ aux = reinterpret_cast<T*>(a.aux);
  const T* __restrict__ aux_c = aux;
  const T* __restrict__ W = reinterpret_cast<const T*>(a.w);
  const int lane = threadIdx.x & 31;
  const int n_warps = gridDim.x * (NT / 32);
  int pi = 0;
  for (int64_t u = blockIdx.x * (NT / 32) + (threadIdx.x >> 5); u < a.n_units; u += n_warps) {
    int64_t ul;
    if (PRM) {
      ul = u;  // one pass per launch, starting at unit 0
    } else if (a.interleave) {
      pi = (int)(u % a.n_passes);
      ul = u / a.n_passes;
    } else {
      while (pi + 1 < a.n_passes && u >= a.passes[pi + 1].unit0) ++pi;
      while (pi > 0 && u < a.passes[pi].unit0) --pi;
      ul = u - a.passes[pi].unit0;
    }
    const CPass* __restrict__ P = PRM ? P0 : a.passes + pi;
    const int nCG = P->nCG;
    const int cg = P->cmaj ? (int)(ul / P->nI) : (int)(ul % nCG);
    const int64_t i = P->cmaj ? ul % P->nI : ul / nCG;
    constexpr int GM = NGC ? NGC : CMAXG;
    const int nK = P->nK, nG = NGC ? NGC : P->nG, nE = P->nE;
    constexpr int KA = KP == 1 ? OUT_SEP_FRESH : KP == 2 ? OUT_SEP_DFRESH : KP == 3 ? OUT_SEP_DRATIO : -1;
    constexpr int KB = KP == 1 || KP == 3 ? OUT_NONE : KP == 2 ? OUT_SEP_DRATIO : -1;
    const int ka = KA >= 0 ? KA : P->out_kind, kb = KB >= 0 ? KB : P->out_kind_b;
    const bool two = kb != OUT_NONE;  // paired sibling output (same K-sum)
    const int nV = VS ? P->nV : 0;  // virtual separators (entry indices at the end of the ti row)
    const int tw = nG + nE + 1 + (two ? P->nE_b + 1 : 0) + nV;
    const int32_t* __restrict__ tir = a.tab + P->ti_off + i * tw;
    const int32_t* __restrict__ tk = PRM ? tk0 : a.tab + P->tk_off;
    const int32_t* __restrict__ ts = PRM ? ts0 : a.tab + P->ts_off;
    const T* gq[GM];
#pragma unroll
    for (int g = 0; g < GM; ++g) gq[g] = aux_c + (g < nG ? P->gfac_off[g] + __ldg(tir + g) : 0);
    const T* __restrict__ wrow = W + P->w_off + i * (int64_t)nK;
    const int bstep = 32 * VEC * nCG;
    for (int b0 = cg * 32 * VEC + lane * VEC; b0 < a.B; b0 += bstep) {
      // VS: the virtual separators at this i (epilogue factors / old separators),
      // gathered before the K-sum so their latency hides behind it
      T vv[CMAXV][VEC];
      if (VS && nV > 0) {
#pragma unroll
        for (int q = 0; q < CMAXV; ++q)
          if (q < nV) {
            int vc[VEC];  // the lanes' Wv columns
            vsep_cols<VEC>(P->vd[q], a.codes, b0, vc);
            vsep_gather<T, VEC>(W + P->vd[q].w_off + __ldg(tir + tw - nV + q), vc, vv[q]);
          }
      }
      double acc[VEC];
#pragma unroll
      for (int l = 0; l < VEC; ++l) acc[l] = 0.0;
      T part[VEC];
#pragma unroll
      for (int l = 0; l < VEC; ++l) part[l] = (T)0;
      int since = 0;
      const T* gb[GM];  // this lane's case vector of each factor (per k: + the k-offset, one IMAD.WIDE)
#pragma unroll
      for (int g = 0; g < GM; ++g) gb[g] = gq[g] + b0;
      for (int k = 0; k < nK; k += KU) {
        T pv[KU][VEC];
        T w[KU];
#pragma unroll
        for (int q = 0; q < KU; ++q) {
          const int kq = min(k + q, nK - 1);
#pragma unroll
          for (int l = 0; l < VEC; ++l) pv[q][l] = (T)1;
#pragma unroll
          for (int g = 0; g < GM; ++g) {
            if (NGC || g < nG) {
              T f[VEC];
              load_vec_ro<T, VEC>(gb[g] + (PRM ? tk[kq * nG + g] : __ldg(tk + kq * nG + g)), f);
#pragma unroll
              for (int l = 0; l < VEC; ++l) pv[q][l] *= f[l];
            }
          }
          w[q] = k + q < nK ? __ldg(wrow + kq) : (T)0;
        }
#pragma unroll
        for (int q = 0; q < KU; ++q)
#pragma unroll
          for (int l = 0; l < VEC; ++l) part[l] += w[q] * pv[q][l];
        if (FOLD && (since += KU) >= KF) {
#pragma unroll
          for (int l = 0; l < VEC; ++l) {
            acc[l] += (double)part[l];
            part[l] = (T)0;
          }
          since = 0;
        }
      }
#define TSV(x) (PRM ? ts[(x)] : __ldg(ts + (x)))
#define SBV(x) (PRM ? sb[(x)] : __ldg(sb + (x)))
      double vsum[VEC], v[VEC];
#pragma unroll
      for (int l = 0; l < VEC; ++l) v[l] = vsum[l] = acc[l] + (double)part[l];
      const bool cs = a.stream_epi != 0;
      double xp[XW ? VEC : 1];  // XW: product of the E factors (times old below) -> X
#pragma unroll
      for (int l = 0; l < (XW ? VEC : 1); ++l) xp[l] = 1.0;
      for (int e = 0; e < nE; ++e) {
        T f[VEC];
        const int ev = nV > 0 ? P->e_v[e] : -1;
        if (ev >= 0) {
          vsep_pick<T, VEC>(ev, vv, f);
        } else {
          const T* ep = aux_c + P->efac_off[e] + __ldg(tir + nG + e) + TSV(e) + b0;
          if (cs) load_vec_cs<T, VEC>(ep, f);
          else load_vec_ro<T, VEC>(ep, f);
        }
#pragma unroll
        for (int l = 0; l < VEC; ++l) {
          v[l] *= (double)f[l];
          if (XW) xp[l % (XW ? VEC : 1)] *= (double)f[l];
        }
      }
      const int64_t j = (int64_t)__ldg(tir + nG + nE) + TSV(nE) + b0;
      T old[VEC] = {};
      if (ka == OUT_SEP || ka == OUT_SEP_DFRESH) {
        if (nV > 0 && P->old_v >= 0) vsep_pick<T, VEC>(P->old_v, vv, old);
        else if (cs) load_vec_cs<T, VEC>(aux_c + P->out_off + j, old);
        else load_vec<T, VEC>(aux_c + P->out_off + j, old);
      }
      if (XW) {  // X = old * Π E (the product of every factor over the output scope)
        T xv[VEC];
#pragma unroll
        for (int l = 0; l < VEC; ++l) xv[l] = (T)(xp[l % (XW ? VEC : 1)] * (double)old[l]);
        if (cs) store_vec_cs<T, VEC>(aux + P->x_off + j, xv);
        else store_vec<T, VEC>(aux + P->x_off + j, xv);
      }
      bool bad = finalize_lanes<T, double, VEC>(ka, P->out_off, P->ratio_off, P->out2_off, j, v, old, aux,
                                                a.qout, cs);
      if (two) {
        const int32_t* tb = tir + nG + nE + 1;  // [E_b..., out_b] of this i
        const int32_t* sb = ts + nE + 1;        // [E_b..., out_b] of the (single) s' row
        const int nEb = P->nE_b;
#pragma unroll
        for (int l = 0; l < VEC; ++l) v[l] = vsum[l];
        for (int e = 0; e < nEb; ++e) {
          T f[VEC];
          const int ev = nV > 0 ? P->e_v_b[e] : -1;
          if (ev >= 0) {
            vsep_pick<T, VEC>(ev, vv, f);
          } else {
            const T* ep = aux_c + P->efac_off_b[e] + __ldg(tb + e) + SBV(e) + b0;
            if (cs) load_vec_cs<T, VEC>(ep, f);
            else load_vec_ro<T, VEC>(ep, f);
          }
#pragma unroll
          for (int l = 0; l < VEC; ++l) v[l] *= (double)f[l];
        }
        const int64_t jb = (int64_t)__ldg(tb + nEb) + SBV(nEb) + b0;
        T oldb[VEC] = {};
        if (kb == OUT_SEP || kb == OUT_SEP_DFRESH) {
          if (nV > 0 && P->old_v_b >= 0) vsep_pick<T, VEC>(P->old_v_b, vv, oldb);
          else if (cs) load_vec_cs<T, VEC>(aux_c + P->out_off_b + jb, oldb);
          else load_vec<T, VEC>(aux_c + P->out_off_b + jb, oldb);
        }
        bad |= finalize_lanes<T, double, VEC>(kb, P->out_off_b, P->ratio_off_b, P->out2_off_b, jb, v, oldb,
                                              aux, a.qout, cs);
      }
      if (bad) atomicOr(a.err, EB_INCONSISTENT);
#undef TSV
#undef SBV
    }
  }
}

#define ROWI_MINB(T, FOLD, LONGK, VS) \
  (LONGK ? ROWI_MINB_L : VS ? ROWI_MINB_V : FOLD ? ROWI_MINB_F : sizeof(T) == 8 ? ROWI_MINB_D : ROWI_MINB_NF)
template <typename T, bool FOLD, bool LONGK = false, bool VS = false>
__global__ void __launch_bounds__(NT, ROWI_MINB(T, FOLD, LONGK, VS)) contract_rowi_kernel(const CArgs a) {
  pdl_enter();
  rowi_body<T, FOLD, LONGK, false, false, 0, VS>(a, nullptr, nullptr, nullptr);
}

template <typename T, bool FOLD, bool LONGK, bool XW = false, int NGC = 0, bool VS = false, int KP = 0>
__global__ void __launch_bounds__(NT, ROWI_MINB(T, FOLD, LONGK, VS))
    contract_rowi_p_kernel(const CArgs a, const __grid_constant__ RowiParam rp) {
  pdl_enter();
  rowi_body<T, FOLD, LONGK, true, XW, NGC, VS, KP>(a, &rp.cp, rp.tk, rp.ts);
}


// Row-per-i passes over i-groups: igs consecutive i differ only in the
// innermost i variable, which most factors (the large ones) do not index.  One
// warp walks the whole group: per k the shared factor rows are loaded once and
// reused by every member (each member multiplies in its own few small factors
// and W entry), so the large rows stream from DRAM once instead of igs times
// through L2.  IGM: compile-time bound of igs (registers for the accumulators).
#ifndef ROWG_MINB
#define ROWG_MINB 4
#endif
template <typename T, bool FOLD, int IGM>
__global__ void __launch_bounds__(NT, ROWG_MINB) contract_rowg_kernel(const CArgs a) {
  pdl_enter();
  constexpr int VEC = CTraits<T>::VEC;
  constexpr int KF = 16;
  T* __restrict__ aux = reinterpret_cast<T*>(a.aux);
  const T* __restrict__ aux_c = aux;
  const T* __restrict__ W = reinterpret_cast<const T*>(a.w);
  const int lane = threadIdx.x & 31;
  const int n_warps = gridDim.x * (NT / 32);
  int pi = 0;
  for (int64_t u = blockIdx.x * (NT / 32) + (threadIdx.x >> 5); u < a.n_units; u += n_warps) {
    int64_t ul;
    if (a.interleave) {
      pi = (int)(u % a.n_passes);
      ul = u / a.n_passes;
    } else {
      while (pi + 1 < a.n_passes && u >= a.passes[pi + 1].unit0) ++pi;
      while (pi > 0 && u < a.passes[pi].unit0) --pi;
      ul = u - a.passes[pi].unit0;
    }
    const CPass* __restrict__ P = a.passes + pi;
    const int nCG = P->nCG, igs = P->igs;
    const int64_t n_grp = P->nI / igs;
    const int cg = P->cmaj ? (int)(ul / n_grp) : (int)(ul % nCG);
    const int64_t i0 = (P->cmaj ? ul % n_grp : ul / nCG) * igs;
    const int nK = P->nK, nG = P->nG, nE = P->nE;
    const int tw = nG + nE + 1;
    const int32_t* __restrict__ tir = a.tab + P->ti_off + i0 * tw;  // member q: + q * tw
    const int32_t* __restrict__ tk = a.tab + P->tk_off;
    const int32_t* __restrict__ ts = a.tab + P->ts_off;
    const T* gq[CMAXG];
    int gs[CMAXG];
#pragma unroll
    for (int g = 0; g < CMAXG; ++g) {
      gq[g] = aux_c + (g < nG ? P->gfac_off[g] + __ldg(tir + g) : 0);
      gs[g] = g < nG ? P->gstride[g] : 0;
    }
    const T* __restrict__ wrow = W + P->w_off + i0 * (int64_t)nK;  // member q: + q * nK
    const int bstep = 32 * VEC * nCG;
    for (int b0 = cg * 32 * VEC + lane * VEC; b0 < a.B; b0 += bstep) {
      double acc[IGM][VEC];
      T part[IGM][VEC];
#pragma unroll
      for (int q = 0; q < IGM; ++q)
#pragma unroll
        for (int l = 0; l < VEC; ++l) {
          acc[q][l] = 0.0;
          part[q][l] = (T)0;
        }
      int since = 0;
      for (int k = 0; k < nK; ++k) {
        T ps[VEC];  // product of the shared factor rows
#pragma unroll
        for (int l = 0; l < VEC; ++l) ps[l] = (T)1;
#pragma unroll
        for (int g = 0; g < CMAXG; ++g) {
          if (g < nG && gs[g] == 0) {
            T f[VEC];
            load_vec_ro<T, VEC>(gq[g] + b0 + __ldg(tk + k * nG + g), f);
#pragma unroll
            for (int l = 0; l < VEC; ++l) ps[l] *= f[l];
          }
        }
#pragma unroll
        for (int q = 0; q < IGM; ++q) {
          if (q < igs) {
            T pv[VEC];
#pragma unroll
            for (int l = 0; l < VEC; ++l) pv[l] = ps[l];
#pragma unroll
            for (int g = 0; g < CMAXG; ++g) {
              if (g < nG && gs[g] != 0) {
                T f[VEC];
                load_vec_ro<T, VEC>(gq[g] + (int64_t)q * gs[g] + b0 + __ldg(tk + k * nG + g), f);
#pragma unroll
                for (int l = 0; l < VEC; ++l) pv[l] *= f[l];
              }
            }
            const T w = __ldg(wrow + (int64_t)q * nK + k);
#pragma unroll
            for (int l = 0; l < VEC; ++l) part[q][l] += w * pv[l];
          }
        }
        if (FOLD && ++since == KF) {
#pragma unroll
          for (int q = 0; q < IGM; ++q)
#pragma unroll
            for (int l = 0; l < VEC; ++l) {
              acc[q][l] += (double)part[q][l];
              part[q][l] = (T)0;
            }
          since = 0;
        }
      }
      bool bad = false;
#pragma unroll
      for (int q = 0; q < IGM; ++q) {
        if (q >= igs) continue;
        const int32_t* tq = tir + (int64_t)q * tw;
        double v[VEC];
#pragma unroll
        for (int l = 0; l < VEC; ++l) v[l] = acc[q][l] + (double)part[q][l];
        const bool cs = a.stream_epi != 0;
        for (int e = 0; e < nE; ++e) {
          T f[VEC];
          const T* ep = aux_c + P->efac_off[e] + __ldg(tq + nG + e) + __ldg(ts + e) + b0;
          if (cs) load_vec_cs<T, VEC>(ep, f);
          else load_vec_ro<T, VEC>(ep, f);
#pragma unroll
          for (int l = 0; l < VEC; ++l) v[l] *= (double)f[l];
        }
        const int64_t j = (int64_t)__ldg(tq + nG + nE) + __ldg(ts + nE) + b0;
        T old[VEC] = {};
        if (P->out_kind == OUT_SEP || P->out_kind == OUT_SEP_DFRESH) {
          if (cs) load_vec_cs<T, VEC>(aux_c + P->out_off + j, old);
          else load_vec<T, VEC>(aux_c + P->out_off + j, old);
        }
        bad |= finalize_lanes<T, double, VEC>(P->out_kind, P->out_off, P->ratio_off, P->out2_off, j, v, old, aux,
                                              a.qout, cs);
      }
      if (bad) atomicOr(a.err, EB_INCONSISTENT);
    }
  }
}

template <typename T, bool FOLD, int NG>
static size_t contract_smem() {
  return (FOLD ? CFOLD_SMEM : 0) + CRing<T, NG, FOLD>::BYTES;
}

template <typename T, bool FOLD, int NG>
static cudaError_t contract_prepare() {
  static bool done = false;  // one attribute call per instantiation (host thread of the plan owner)
  if (done) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(contract_kernel<T, FOLD, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)contract_smem<T, FOLD, NG>());
  if (e == cudaSuccess) done = true;
  return e;
}

template <typename T, bool FOLD, int NG>
static cudaError_t launch_contract_t(const CArgs& a, int grid, cudaStream_t s) {
  cudaError_t e = contract_prepare<T, FOLD, NG>();
  if (e != cudaSuccess) return e;
  return launch_pdl(contract_kernel<T, FOLD, NG>, grid, NT, contract_smem<T, FOLD, NG>(), s, a);
}

template <typename T, bool FOLD, int NG>
static int occ_contract_t() {
  if (contract_prepare<T, FOLD, NG>() != cudaSuccess) return 1;
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, contract_kernel<T, FOLD, NG>, NT, contract_smem<T, FOLD, NG>());
  return n > 0 ? n : 1;
}

template <typename T, bool FOLD, class F>
static auto by_ng(int ng, F f) {
  switch (ng) {
    case 0: return f(std::integral_constant<int, 0>());
    case 1: return f(std::integral_constant<int, 1>());
    case 2: return f(std::integral_constant<int, 2>());
    case 3: return f(std::integral_constant<int, 3>());
    default: return f(std::integral_constant<int, 4>());
  }
}

template <typename T, bool FOLD, int NG>
static cudaError_t launch_contract_p_t(const CArgs& a, const TileParam& tp, int grid, cudaStream_t s) {
  static bool done = false;
  if (!done) {
    cudaError_t e = cudaFuncSetAttribute(contract_p_kernel<T, FOLD, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)contract_smem<T, FOLD, NG>());
    if (e != cudaSuccess) return e;
    done = true;
  }
  return launch_pdl(contract_p_kernel<T, FOLD, NG>, grid, NT, contract_smem<T, FOLD, NG>(), s, a, tp);
}





}  // namespace jt
