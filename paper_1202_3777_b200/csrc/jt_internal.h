// Internal types shared by the host planner (jt_plan.cpp) and the kernels
// (jt_kernels.cu).  See DESIGN.md §3 for the pass/wave model.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace jt {

constexpr int NT = 256;     // threads per CTA of the wave kernel
constexpr int KV = 4;       // vectors owned per thread per iteration (large waves; small waves use 2)
constexpr int MAXF = 8;     // factors (ratio / evidence tensors) multiplied in per pass
constexpr int MAXDI = 8;    // merged inner dimensions per pass

enum ArenaId : int { A_CLIQUE = 0, A_BASE = 1, A_AUX = 2 };
enum OutKind : int { OUT_NONE = 0, OUT_SEP = 1, OUT_RAW = 2, OUT_SEP_FRESH = 3, OUT_SEP_DFRESH = 4, OUT_SEP_DRATIO = 5 };
// OUT_SEP_DRATIO (contraction passes of fused propagations): a fresh distribute output
// whose final table is rebuilt on demand writes only the ratio Σ (no old read).  Where
// the old separator is 0 the reference's ratio is 0 and this one is Σ; every consumer
// multiplies it into clique entries that sum to that 0 — nonnegative, hence all 0 —
// so every table, posterior and rebuilt final separator is the same.
// out2_off == OUT2_SKIP: a distribute pass of a fused propagation does not store the
// separator's final table (old x ratio, rebuilt on demand: materialize_final)
constexpr int64_t OUT2_SKIP = -2;
// OUT_SEP_DFRESH: distribute output of a fresh propagation; the pass sums
// WITHOUT the target separator's own collect message c (= old value), so
// new = c*S and ratio = new/old = S (0 where c == 0): the Hugin division cancels.
// OUT_SEP_FRESH: collect output of a fresh propagation (old separator known to be
// ones): ratio == star, so only the separator itself is written and consumers
// read it as the ratio.
enum ErrBits : int { EB_INCONSISTENT = 1, EB_ZERO_MASS = 2 };

// One pass = one sweep over one clique table: read (src), multiply the
// factors in, optionally write (dst), optionally reduce onto one output
// tensor.  The clique is seen as [outer blocks] x [inner block of T positions].
struct DevPass {
  int64_t src_off;          // element offset of the clique in the src arena
  int64_t dst_off;          // element offset in the clique arena, -1: no write
  int64_t fac_off[MAXF];    // element offsets of the factor tensors (aux arena)
  int64_t out_off;          // aux (OUT_SEP) or qout (OUT_RAW) offset of the output
  int64_t ratio_off;        // aux offset of the ratio array written by OUT_SEP
  int64_t out2_off;         // OUT_SEP: >= 0 writes the new separator here (old stays at out_off)
  int64_t blk_off;          // offset into the block table (int64 entries)
  int64_t bin_off;          // offset into the bin table (int32: binbase[n_in], binrest[T/n_in])
  int64_t part_off;         // offset into the partials arena (doubles)
  int64_t cnt_off;          // offset into the counters arena (ints)
  int64_t n_blocks_per_jout;// rest-outer blocks per output group (r_out)
  int64_t blocks_per_chunk; // multiple of BPI
  int src_arena;            // A_CLIQUE, A_BASE or A_AUX (separator-sized sources)
  int src_vec;              // 1: innermost stride 1 (vector load), 0: broadcast
  int nf;
  uint32_t fac_vec;         // bit f set: factor f has the innermost dim (vector), else broadcast
  uint32_t flush_fac;       // bit f set: factor f is constant over an output group (own passes):
                            //   multiplied once into the group sum instead of per element
  int out_kind;
  int n_in;                 // output bins per block
  int n_chunks;
  int T;                    // positions per block (multiple of VEC)
  int BPI;                  // blocks per CTA iteration
  int blk_stride;           // 2 + nf
  int gpi;                  // >1: each iteration covers gpi whole output groups (BPI = gpi*r_out),
                            //     reduced and finalized per iteration; items span j_count groups
  int64_t blk32_off;        // OWN passes: offset into the int32 block table (entries in units)
  int unit_src, unit_dst;   // element offset = entry * unit
  int unit_fac[MAXF];
  int own_m;                // own passes: vectors (lane chunks) per thread per block
  int kv;                   // general kernel: vectors per thread per iteration (2 or 4)
  int row;                  // 1: row pass (n_in <= 1, no gpi, T % (32*VEC) == 0): wave_row_kernel
  int64_t row_tab_off;      // row passes: offset of the inner-offset table [2+nf][T/VEC] (int32)
  int row_lin;              // row passes: src and dst inner offsets equal the position (tab rows 0/1 unused)
  uint32_t row_fmode;       // row passes, 2 bits per factor: 0 table, 1 offset = position, 2 offset = 0
  int own;                  // 1: thread-owned bins (n_in == T == NT*VEC): sync-free epilogue,
                            //    items span j_count whole output groups
  int ndi;                  // merged inner dims
  int icard[MAXDI];         // innermost last
  int isrc[MAXDI];
  int idst[MAXDI];
  int iout[MAXDI];
  int ifac[MAXF][MAXDI];
};

struct Item {               // one CTA work unit
  int pass;
  int chunk;
  int64_t j_out;
  int64_t j_count;          // OWN passes without chunking: consecutive output groups
};

struct WaveArgs {
  void* clique;             // T*
  const void* base;         // const T*
  void* aux;                // T*
  double* qout;
  double* partials;
  int* counters;
  int* err;
  const int64_t* blk;
  const int32_t* blk32;
  const int32_t* bins;
  const DevPass* passes;
  const Item* items;
  int n_items;
  const int32_t* rowtab;    // row kernel inner-offset tables
};

// Contraction pass (shared-base batches): the base replica never
// changes, so a pass over clique c with factors G (batched, over vars U), output
// over vars s and epilogue factors E (vars within s) is
//   out[I, S', b] = Π_E E[., b] · Σ_{K'} W[I, K', S'] · Π_G F_g[I, K', b]
// with I = s∩U, S' = s∖U, K' = U∖s and W = base summed over R = c∖(s∪U),
// precomputed on the host.  A warp owns one (i, row tile of TMC rows of S')
// unit and walks all cases.
constexpr int TMC = 8;     // W rows per warp unit
constexpr int CVEC = 4;    // B must be a multiple of this (fp32 lanes per vector; fp64 uses 2)
constexpr int CMAXG = 4;   // factors multiplied per k (more: the pass takes the general kernels)
// Virtual separator (shared-base fresh programs): a leaf clique's collect message
// phi*(j, b) = Σ_k Wv[j][k] · mask_v[k][b] (the leaf's one private variable v and
// its 0/1 evidence mask) is not materialised.  The row-per-i passes that read it
// (as an epilogue factor or as the old separator of a distribute output) gather
// it: with the mask's per-case code c (a one-hot state, -1 all ones, -2 all
// zeros) the sum is Wv[j][c], the precomputed row sum Wv[j][nK], or 0.
struct VDesc {
  int64_t w_off;            // W arena offset of Wv, layout [entries][nK + 1] (row sum last)
  int64_t code_off;         // int32 offset of the leaf's mask codes [B] in CArgs::codes; -1: no evidence
  int nK, pad;
};
struct VCodeTask {          // per-program mask code of one evidence variable
  int64_t mask_off;         // aux offset of its mask [card][B]
  int card, pad;
};
constexpr int CMAXV = 2;    // virtual separators per pass

struct CPass {
  int64_t w_off;            // W arena offset, layout [nI][nK][nS]
  int64_t ti_off;           // int32 [nI][nG + nE + 1]: G i-offsets, E i-offsets, out i-offset
  int64_t tk_off;           // int32 [nK][nG]: G k-offsets
  int64_t ts_off;           // int32 [nS][nE + 1]: E s-offsets, out s-offset
  int64_t unit0;            // first global unit of this pass in its launch
  int64_t n_units;
  int nI, nS, nK, nG, nE, nT, nBC;
  int nCG;                  // case-chunk groups: a unit walks chunks cg, cg + nCG, ...
  int cmaj;                 // 1: units enumerate the case-chunk group outermost (concurrent warps
                            //    share one case chunk of every i: i-reused factor rows stay in L2)
  int rowi;                 // 1: nS == 1, one i per unit (W layout [nI][nK]); 2/3: i-groups (below)
  int igs;                  // rowi 2/3: a unit is igs consecutive i (the innermost i variable) that
  int gstride[CMAXG];       //   share every G factor with gstride 0 (loaded once per k); factor g
                            //   of member q sits at + q * gstride[g]
  int nKS;                  // > 1: K split into nKS chunks of kch (units also index the chunk);
  int kch;                  //   partial sums combined in chunk order by the last warp of a group
  int64_t part_off, cnt_off;
  int out_kind;
  int64_t out_off, ratio_off, out2_off;
  int64_t gfac_off[MAXF];   // aux offsets of the G factors
  int64_t efac_off[MAXF];   // aux offsets of the E factors
  // second output (row-per-i passes): a sibling pass of the same clique with the
  // same output scope and the same K-sum (G factors) -- e.g. the distribute
  // messages to two children over equal separators -- shares the sum; only its
  // epilogue factors and output differ.  out_kind_b == OUT_NONE: no second output.
  // ti rows then hold [G, E, out, E_b, out_b]; ts rows [E, out, E_b, out_b].
  int64_t x_off;            // >= 0 (paired passes): also write X = old_a * Π E_a (the product of every
                            // factor over the output scope) here, for the clique's other passes
  int out_kind_b, nE_b;
  int64_t out_off_b, ratio_off_b, out2_off_b;
  int64_t efac_off_b[MAXF];
  // virtual separators read by this (row-per-i) pass: ti rows end with their nV Wv
  // row offsets; E slot e (E_b slot) is virtual separator e_v[e] (e_v_b[e]) when >= 0, the
  // old separator of the output (second output) when old_v (old_v_b) >= 0
  int nV;
  int8_t e_v[MAXF], e_v_b[MAXF];
  int8_t old_v, old_v_b;
  VDesc vd[CMAXV];
};
struct CArgs {
  const void* w;
  void* aux;
  double* qout;
  int* err;
  const int32_t* tab;
  const CPass* passes;
  int n_passes;
  int64_t n_units;
  int B;
  double* partials;         // K-split partial sums
  int* counters;            // K-split arrival counters (reset by the last warp)
  const int32_t* codes;     // virtual separators: per-case evidence mask codes (VDesc::code_off)
  int stream_epi;           // 1: epilogue inputs (E factors, old separators) load and outputs store
                            //    with evict-first hints: the streams do not flush reused factor rows
  int interleave;           // 1: every pass has n_units / n_passes units and unit u belongs to
                            // pass u % n_passes (passes reading the same tensors run side by side)
};
constexpr int CKF = 16;     // fp32 contraction sums longer than this fold into fp64
// ng: factors per k (0..CMAXG) of every pass of the launch (compile-time in the kernel; ignored for rowi)
cudaError_t launch_contract(int dtype, int fold, int rowi, int ng, const CArgs& a, int grid, cudaStream_t s, bool vs = false);
// A single row-per-i pass with its descriptor and k-table carried in the kernel
// parameters (__grid_constant__): the per-k, warp-uniform table lookups come from
// the constant bank instead of competing with the factor streams for L1.
constexpr int RP_TK = 448;  // ints of the k-table (nK x nG)
constexpr int RP_TS = 24;   // ints of the s'-row table (nS == 1: E, out, E_b, out_b)
struct RowiParam {
  CPass cp;
  int32_t tk[RP_TK];
  int32_t ts[RP_TS];
};
cudaError_t launch_contract_rowi_param(int dtype, int fold, int longk, const CArgs& a, const RowiParam& rp, int grid,
                                       cudaStream_t s, bool xw = false, bool vs = false);
constexpr int TP_TS = 1024;  // ints of the s'-row table of a tile pass (nS x (nE + 1))
struct TileParam {
  CPass cp;
  int32_t tk[RP_TK];
  int32_t ts[TP_TS];
};
cudaError_t launch_contract_tile_param(int dtype, int fold, int ng, const CArgs& a, const TileParam& tp, int grid,
                                       cudaStream_t s);
int contract_max_ctas_per_sm(int dtype, int fold, int rowi, int ng);
// occupancy of the parameter-space row-per-i kernel a pass launches (nG specialised)
int contract_rowi_param_max_ctas(int dtype, int fold, int longk, int ng, bool xw, bool vs = false, int ka = 0,
                                 int kb = 0);

// device initialize: one entry per clique, one term per CPT, 3 int64 per CPT variable
// (clique stride, card, CPT stride)
struct InitClique {
  int64_t off, size;
  int first_term, n_terms;
};
struct InitTerm {
  int64_t cpt_off;
  int first_var, nv;
};

// launchers (jt_kernels.cu)
cudaError_t launch_init(void* base, int dtype, const double* cpt, const InitClique* cl, int n_cliques,
                        const InitTerm* terms, const int64_t* vdesc, int64_t max_size, cudaStream_t s);
cudaError_t launch_wave(int dtype, int vec, int kv, const WaveArgs& a, int grid, cudaStream_t s);
// ---- persistent single-launch programs for small single trees (jt_tiny.cu) ----
// A tiny pass is one sweep over one clique table seen as [output entries] x
// [row]: one thread (or, for long rows, one warp) per output entry walks its
// row with mixed-radix odometers -- every factor, source, destination and
// output offset from stride arithmetic, no tables.  Rows are summed in a fixed
// order, so results are deterministic.  Passes without output: one thread per
// element.  All waves of a propagation run in ONE cooperative launch, separated
// by grid barriers.
constexpr int TD = 16;  // merged dims per side (output / row)
struct TPass {
  int64_t src_off, dst_off, out_off, ratio_off, out2_off;
  int64_t fac_off[MAXF];
  int64_t unit0;            // first thread of the pass in its wave (multiple of 32)
  int64_t n_out, n_rest;    // output entries (elements, without output), row length
  int src_arena, nf, out_kind, warp;  // warp: lanes per output entry (power of two <= 32)
  int nod, nrd;
  int ocard[TD], rcard[TD];
  unsigned omul[TD], rmul[TD];  // fast division by the cards: q = (umulhi(n, mul) + n) >> shr
  int oshr[TD], rshr[TD];
  int osrc[TD], odst[TD], oout[TD], rsrc[TD], rdst[TD];
  int ofac[MAXF][TD], rfac[MAXF][TD];
};
struct TinyWave {
  int64_t pass0;            // first TPass of the wave
  int64_t n_threads;        // threads of the wave (sum of the passes' units)
  int n_passes, pad;
};
struct TinyArgs {
  void* clique;
  const void* base;
  void* aux;
  double* qout;
  int* err;
  const TPass* passes;
  const int64_t* unit0s;    // TPass::unit0 of every pass, compact (binary search)
  const TinyWave* waves;
  int n_waves;
  unsigned* bar;            // [counter, generation]
};
// occ_out != nullptr: only report the kernel's CTAs per SM
// nfm: factor count bound of the program's passes (2, 4 or 8; template of the kernel)
cudaError_t launch_tiny(int dtype, int nfm, const TinyArgs& a, int grid, cudaStream_t s, int* occ_out = nullptr);
// the whole tiny program in one thread-block cluster of `grid` (<= 16) CTAs
cudaError_t launch_tiny_cluster(int dtype, int nfm, const TinyArgs& a, int grid, cudaStream_t s);
// one wave of a tiny program as its own launch (PDL-chained, graph-replayable)
cudaError_t launch_tiny_wave(int dtype, int nfm, const TinyArgs& a, int w, int grid, cudaStream_t s);
int wave_max_ctas_per_sm(int dtype, int vec, int kv);
cudaError_t launch_wave_row(int dtype, int vec, int lin, const WaveArgs& a, int grid, cudaStream_t s);
int wave_row_max_ctas_per_sm(int dtype, int vec);
#ifndef KROW_V
#define KROW_V 8
#endif
constexpr int KROW = KROW_V;
constexpr int CHUNK_GROUP = 32;  // chunk partials combined in groups of this many (two levels)     // vectors per thread per iteration of the row kernel
cudaError_t launch_wave_own(int dtype, int vec, int lm, int m, const WaveArgs& a, int grid, cudaStream_t s);
int wave_own_max_ctas_per_sm(int dtype, int vec);
cudaError_t launch_normalize(const double* qout, const int64_t* q_off, const int32_t* q_card,
                             const int32_t* q_col, int nq, int B, int rows, int total_cols,
                             int normalize, double* post, int* err, const int* q_exp, int exp_all,
                             cudaStream_t s);
// exp2: arena values are stored scaled by 2^exp2 (power-of-two prescaling)
cudaError_t launch_convert_d2t(int dtype, const double* src, void* dst, int64_t n,
                               int64_t dst_stride, int64_t bcount, cudaStream_t s, int exp2 = 0);
cudaError_t launch_convert_t2d(int dtype, const void* src, int64_t src_stride,
                               double* dst, int64_t n, cudaStream_t s, int exp2 = 0);
cudaError_t launch_scale_pow2(int dtype, void* p, int64_t n, int exp2, cudaStream_t s);
cudaError_t launch_fill(int dtype, void* dst, int64_t n, double v, cudaStream_t s);
cudaError_t launch_mul(int dtype, void* dst, const void* a, const void* b, int64_t n, cudaStream_t s);
cudaError_t launch_ev_fill(void* aux, int dtype, const int32_t* vars, int nv, const int64_t* var_off,
                           const int32_t* cards, int B, cudaStream_t s);
cudaError_t launch_ev_code(const void* aux, int dtype, const VCodeTask* tasks, int nt, int B, int32_t* codes,
                           cudaStream_t s);
cudaError_t launch_ev_zero(void* aux, int dtype, const int32_t* obs, int n, const int64_t* var_off,
                           const int32_t* cards, int B, cudaStream_t s);
cudaError_t launch_mapping_table(int64_t* out, int64_t n_sep, int64_t n_rest,
                                 int nsd, const int64_t* sep_card, const int64_t* sep_stride,
                                 int nrd, const int64_t* rest_card, const int64_t* rest_stride,
                                 cudaStream_t s);
cudaError_t launch_mu_message(const double* src, double* tgt, double* sep, double* ratio,
                              const void* mu_src, int64_t row_src, const void* mu_tgt,
                              int64_t row_tgt, int64_t n_sep, int is64, int* err,
                              int phase, cudaStream_t s);

}  // namespace jt
