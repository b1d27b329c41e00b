// Host side of libjtb200.so: plan (tree structure), state (HBM arenas), the
// wave scheduler that turns Hugin collect/distribute into passes, the pass
// compiler (block split, stride tables, chunking), and the C ABI.
//
// Reference correspondence (paths relative to the reference repo):
//   jt_plan_create        JunctionTree (pkg/src/jtprop/compiler.py:40-80)
//   jt_state_*            PropagationState / from_potentials (propagate.py:172-240)
//   jt_apply_evidence     apply_evidence (propagate.py:243-260)
//   jt_message            message_passing → _pass_block (propagate.py:56-76, 263-274)
//   jt_propagate          belief_propagation = collect_evidence + distribute_evidence
//                         per component (propagate.py:296-360)
//   jt_query              query_marginal / posterior_marginals (propagate.py:363-390)
//   jt_plan_mapping_table build_mapping_table (compiler.py:285-304)
//   jt_run_message_mu     SequentialEngine.run_message (propagate.py:79-94)
#include "jt_b200.h"
#include "jt_internal.h"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <iterator>
#include <cstdlib>
#include <array>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

using namespace jt;

#define CK(x)                                  \
  do {                                         \
    cudaError_t e__ = (x);                     \
    if (e__ != cudaSuccess) {                  \
      last_cuda_error() = e__;                 \
      return e__ == cudaErrorMemoryAllocation ? JT_ERR_OOM : JT_ERR_CUDA; \
    }                                          \
  } while (0)

static cudaError_t& last_cuda_error() {
  static thread_local cudaError_t e = cudaSuccess;
  return e;
}

// ---------------------------------------------------------------- plan ----
struct jt_plan {
  int n_vars = 0;
  std::vector<int> cards;
  int n_cliques = 0;
  std::vector<std::vector<int>> cvars;
  int n_seps = 0;
  std::vector<std::array<int, 2>> sedge;
  std::vector<std::vector<int>> svars;
  std::vector<int> roots;
  std::vector<std::vector<std::pair<int, int>>> nbrs;  // (clique, sep) ascending clique id
  std::vector<int64_t> csize, ssize;
  std::vector<int> comp;  // component index (position in roots) per clique
  int dtype = JT_F32;
  int device = 0;
};

static int64_t prod_cards(const jt_plan* p, const std::vector<int>& vars) {
  int64_t n = 1;
  for (int v : vars) n *= p->cards[v];
  return n;
}

extern "C" int jt_plan_create(int n_vars, const int32_t* cards, int n_cliques, const int32_t* clique_off,
                              const int32_t* clique_vars, int n_seps, const int32_t* sep_edge,
                              const int32_t* sep_off, const int32_t* sep_vars, int n_roots,
                              const int32_t* roots, int dtype, int device, jt_plan** out) {
  if (!out || n_vars < 0 || n_cliques <= 0 || n_seps < 0 || n_roots <= 0) return JT_ERR_BAD_ARG;
  if (dtype != JT_F32 && dtype != JT_F64) return JT_ERR_BAD_ARG;
  auto p = std::make_unique<jt_plan>();
  p->n_vars = n_vars;
  p->cards.assign(cards, cards + n_vars);
  for (int c : p->cards)
    if (c < 1) return JT_ERR_BAD_ARG;
  p->n_cliques = n_cliques;
  p->cvars.resize(n_cliques);
  for (int c = 0; c < n_cliques; ++c) {
    for (int i = clique_off[c]; i < clique_off[c + 1]; ++i) {
      const int v = clique_vars[i];
      if (v < 0 || v >= n_vars) return JT_ERR_BAD_ARG;
      if (!p->cvars[c].empty() && v <= p->cvars[c].back()) return JT_ERR_BAD_ARG;
      p->cvars[c].push_back(v);
    }
  }
  p->n_seps = n_seps;
  p->sedge.resize(n_seps);
  p->svars.resize(n_seps);
  p->nbrs.resize(n_cliques);
  for (int s = 0; s < n_seps; ++s) {
    const int a = sep_edge[2 * s], b = sep_edge[2 * s + 1];
    if (a < 0 || b < 0 || a >= n_cliques || b >= n_cliques || a == b) return JT_ERR_BAD_ARG;
    p->sedge[s] = {a, b};
    for (int i = sep_off[s]; i < sep_off[s + 1]; ++i) {
      const int v = sep_vars[i];
      if (v < 0 || v >= n_vars) return JT_ERR_BAD_ARG;
      if (!p->svars[s].empty() && v <= p->svars[s].back()) return JT_ERR_BAD_ARG;
      for (int c : {a, b})
        if (!std::binary_search(p->cvars[c].begin(), p->cvars[c].end(), v)) return JT_ERR_BAD_ARG;
      p->svars[s].push_back(v);
    }
    p->nbrs[a].push_back({b, s});
    p->nbrs[b].push_back({a, s});
  }
  for (auto& l : p->nbrs) std::sort(l.begin(), l.end());
  p->roots.assign(roots, roots + n_roots);
  p->comp.assign(n_cliques, -1);
  for (int r = 0; r < n_roots; ++r) {
    const int root = p->roots[r];
    if (root < 0 || root >= n_cliques || p->comp[root] != -1) return JT_ERR_BAD_ARG;
    std::vector<int> stack{root};
    p->comp[root] = r;
    while (!stack.empty()) {
      const int c = stack.back();
      stack.pop_back();
      for (auto& nb : p->nbrs[c]) {
        if (p->comp[nb.first] == -1) {
          p->comp[nb.first] = r;
          stack.push_back(nb.first);
        } else if (p->comp[nb.first] != r) {
          return JT_ERR_BAD_ARG;
        }
      }
    }
  }
  for (int c = 0; c < n_cliques; ++c)
    if (p->comp[c] == -1) return JT_ERR_BAD_ARG;  // a component without a root
  if (n_seps != n_cliques - n_roots) return JT_ERR_BAD_ARG;  // forest check (compiler.py:402)
  for (int c = 0; c < n_cliques; ++c) p->csize.push_back(prod_cards(p.get(), p->cvars[c]));
  for (int s = 0; s < n_seps; ++s) p->ssize.push_back(prod_cards(p.get(), p->svars[s]));
  p->dtype = dtype;
  p->device = device;
  *out = p.release();
  return JT_OK;
}

extern "C" void jt_plan_destroy(jt_plan* plan) { delete plan; }

// --------------------------------------------------------- tensors / specs --
struct Tensor {
  int arena = A_AUX;  // where it lives
  int64_t off = 0;
  std::vector<int> vars;  // ascending
  bool batch = false;     // trailing batch dim
  // virtual separator (VDesc): the collect message of leaf clique vclique is not
  // materialised; its readers evaluate Σ_k base · Π vfac (the leaf's evidence)
  int vclique = -1;
  std::vector<Tensor> vfac;
};

struct PassSpec {
  int clique = 0;
  std::vector<int> scope;   // non-empty: iterate this scope (a separator) instead of the clique's
  int64_t src_off = -1;     // A_AUX source: aux offset of the scope's table
  int src_arena = A_CLIQUE;
  bool write = false;
  std::vector<Tensor> factors;
  int out_kind = OUT_NONE;
  Tensor out;
  int64_t ratio_off = -1;
  int64_t out2_off = -1;
  int64_t x_off = -1;       // >= 0: this (paired) pass also writes its clique's product X here
  int sep = -1;             // distribute passes: the separator of the output
  bool skip_out2 = false;   // fused propagation: the final table of `sep` is rebuilt on demand
};

struct LaunchGrp {  // one kernel launch of a wave
  int kind = 0;      // 0: general kernel, 1: thread-owned-bins kernel, 2: row kernel
  int vec = 1;       // lanes per vector load (kind 3: factors per k, nG)
  int lm = 0;        // own kernel load shapes: 0 generic, 1 src bcast + vector factors, 2 all vector
  int m = 1;         // own kernel vectors per thread per block
  int grid = 0;
  int n_items = 0;
  int64_t item_off = 0;  // relative to the wave's item_base
  // kind 3 (contraction): CPass range and unit count
  int64_t cpass_off = 0;
  int n_cpasses = 0;
  int64_t n_units = 0;
  int interleave = 0;  // CArgs::interleave
  int rp_idx = -1;     // >= 0: single row-per-i pass launched with its tables in the parameters
  int xw = 0;          // 1: that pass writes the clique product X (rowi_p kernel with XW)
  int tp_idx = -1;     // >= 0: single tile pass launched with its tables in the parameters
  int vs = 0;          // 1: a pass of the launch reads virtual separators (VS kernel variant)
};

struct WaveRt {
  int n_items = 0;  // all items of the wave
  std::vector<LaunchGrp> groups;
  int64_t pass_base = 0, item_base = 0;
};

struct Program {
  std::vector<WaveRt> waves;
  DevPass* d_passes = nullptr;
  Item* d_items = nullptr;
  int64_t* d_blk = nullptr;
  int32_t* d_blk32 = nullptr;
  int32_t* d_bins = nullptr;
  int32_t* d_rowtab = nullptr;
  double* d_part = nullptr;
  int* d_cnt = nullptr;
  CPass* d_cpass = nullptr;
  int32_t* d_ctab = nullptr;
  void* d_w = nullptr;
  VCodeTask* d_vtask = nullptr;  // virtual separators: mask-code tasks and their codes
  int32_t* d_vcode = nullptr;
  int n_vtask = 0;
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t gstream = nullptr;
  // persistent single-launch program (small single trees, jt_tiny.cu)
  std::vector<RowiParam> rparams;  // per single row-per-i launch (LaunchGrp::rp_idx)
  std::vector<TileParam> tparams;  // per single tile launch (LaunchGrp::tp_idx)
  int tiny = 0, tiny_grid = 0, n_twaves = 0, tiny_nfm = MAXF;
  int tiny_cluster = 0;                // > 0: the whole program in one cluster of this many CTAs
  int tiny_waves_launch = 0;           // 1: per-wave launches (PDL), tiny kernel on the waves flagged below
  std::vector<char> tiny_w;            // per (non-empty) wave: run as a tiny-pass launch
  std::vector<int> tiny_wave_grid;     // per-wave grids of the per-wave launches
  std::vector<int> vsep_leaves;        // leaves whose collect message this program does not store
  std::vector<int> final_skip;         // separators whose final table it does not store
  TPass* d_tpass = nullptr;
  int64_t* d_unit0 = nullptr;
  TinyWave* d_twaves = nullptr;
  unsigned* d_bar = nullptr;
  int runs = 0;
  int64_t n_launches = 0;  // kernel launches per run
  ~Program() {
    if (gexec) cudaGraphExecDestroy(gexec);
    cudaFree(d_passes);
    cudaFree(d_items);
    cudaFree(d_blk);
    cudaFree(d_blk32);
    cudaFree(d_bins);
    cudaFree(d_rowtab);
    cudaFree(d_part);
    cudaFree(d_cnt);
    cudaFree(d_cpass);
    cudaFree(d_ctab);
    cudaFree(d_vtask);
    cudaFree(d_vcode);
    cudaFree(d_w);
    cudaFree(d_tpass);
    cudaFree(d_unit0);
    cudaFree(d_twaves);
    cudaFree(d_bar);
  }
};


// ------------------------------------------------------------------ state --
struct jt_state {
  const jt_plan* plan = nullptr;
  int B = 1;       // case lanes of every batched tensor (padded, see padded_batch)
  int B_user = 1;  // cases the caller asked for: API bounds, posterior rows
  int mode = JT_MATERIALIZED;
  int esz = 4;
  int num_sms = 148;
  void* d_clique = nullptr;
  void* d_base = nullptr;
  void* d_aux = nullptr;
  double* d_qout = nullptr;
  double* d_post = nullptr;
  int64_t post_cap = 0;
  double* d_stage = nullptr;
  int64_t stage_cap = 0;
  int* d_err = nullptr;
  std::map<std::string, std::pair<int64_t*, int>> qmeta;  // per var list: device metadata, total cols
  cudaStream_t stream = nullptr;
  // fork/join resources: independent launch groups of one wave run on side
  // streams (parallel branches once the program is captured as a graph)
  static constexpr int N_SIDE = 7;
  cudaStream_t side[N_SIDE] = {};
  cudaEvent_t ev_fork = nullptr;
  cudaEvent_t ev_join[N_SIDE] = {};
  std::vector<int64_t> coff, boff, sep_off, ratC_off, ratD_off, ev_off, q_off;
  int64_t msg_ratio_off = 0;
  int64_t n_clique = 0, n_base = 0, n_aux = 0, n_qout = 0;
  std::vector<int> ev_clique;               // per var: clique holding its active factor, -1 none
  int64_t* d_evoff = nullptr;               // per var: aux offset of its mask [card][B]
  int32_t* d_cards = nullptr;               // per var cardinality
  int32_t* d_obs = nullptr;                 // observation staging (case, var, state)
  int64_t obs_cap = 0;
  int32_t* d_fill = nullptr;                // variables whose masks are (re)filled with ones
  int64_t fill_cap = 0;
  std::vector<int32_t> fill_host;           // contents of d_fill
  std::map<std::string, std::unique_ptr<Program>> programs;
  int64_t launches = 0;
  int64_t device_bytes = 0;
  // shared-base mode: cliques whose passes would need more than MAXF factors keep
  // per-case tables in the clique arena (initialised from base x evidence at the
  // start of each propagation, children absorbed eagerly); every other clique
  // stays a shared base table
  std::vector<char> hub;
  int* d_qexp = nullptr;    // per-query exponents of unnormalized queries
  int64_t qexp_cap = 0;
  int err_case = -1;        // lowest case index of the last zero-mass error (jt_sync_error)
  // Power-of-two prescaling (exact: only exponents move).  Every table is stored
  // as exact * 2^e: pre_e per clique is chosen at load/initialize so each clique
  // sums to about the size of its parent separator (root: 1) -- the balance the
  // reference's own generator lacks (uniform(0.1,1) tables reach 2e107 on a
  // Pigs-shaped tree), so fp32 states neither overflow nor
  // underflow on unscaled inputs.  e_c / e_s track the current exponent of every
  // clique / separator table through messages and propagations (host integers:
  // the scaling is data-independent per state); host views and unnormalized
  // queries (P(e), propagate.py:363-377) undo it exactly.
  std::vector<int> pre_e, e_c, e_s;
  bool fresh = true;        // separators hold ones (reset/load): collect may skip old/ratio
  bool seps_stale = false;  // separators logically ones but not yet filled
  // Two tables per separator (X at sep_off, Y at ratC_off): one holds the
  // current separator values, the other the last collect ratios.  A fresh
  // propagation writes the collect messages into the current table and the
  // distribute results into the other one, then the roles swap.
  bool sep_in_y = false;
  // leaves whose collect message the last propagation did not store (virtual
  // separators): materialised before a later query reads it (materialize_vsep)
  std::vector<int> vsep_pending;
  // separators whose final table the last propagation did not store (rebuilt as
  // collect message x distribute ratio before it is read: materialize_final)
  std::vector<int> final_pending;
  // host copy of the base replica (shared-base states): contraction passes
  // precompute W = base summed over the variables no factor or output sees
  std::vector<double> h_base;
  ~jt_state() {
    programs.clear();
    cudaFree(d_clique);
    cudaFree(d_base);
    cudaFree(d_aux);
    cudaFree(d_qout);
    cudaFree(d_post);
    cudaFree(d_stage);
    cudaFree(d_err);
    cudaFree(d_evoff);
    cudaFree(d_cards);
    cudaFree(d_obs);
    cudaFree(d_fill);
    cudaFree(d_qexp);
    for (auto& kv : qmeta) cudaFree(kv.second.first);
    for (int i = 0; i < N_SIDE; ++i) {
      if (side[i]) cudaStreamDestroy(side[i]);
      if (ev_join[i]) cudaEventDestroy(ev_join[i]);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (stream) cudaStreamDestroy(stream);
  }
};

static int64_t align4(int64_t x) { return (x + 3) & ~int64_t(3); }

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}
static int64_t sep_cur(const jt_state* st, int sp) { return st->sep_in_y ? st->ratC_off[sp] : st->sep_off[sp]; }
static int64_t sep_alt(const jt_state* st, int sp) { return st->sep_in_y ? st->sep_off[sp] : st->ratC_off[sp]; }

struct DevGuard {
  int prev = 0;
  explicit DevGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DevGuard() {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != prev) cudaSetDevice(prev);
  }
};

static int smallest_holder(const jt_plan* p, int v);

// Case lanes: micro-batches above one thread-owned block (NT*VEC lanes) are
// padded to a whole number of blocks, others of >= one case chunk (32*VEC
// lanes) to whole chunks, so every pass keeps its vector, thread-owned and
// K-split kernels (an odd size such as 4000 otherwise fell to the general kernels
// at half the speed, or failed to plan in fp64).  Padded lanes carry no evidence,
// are propagated like any case and never reach the caller.
static int padded_batch(const jt_plan* plan, int batch) {
  const int vec = plan->dtype == JT_F32 ? 4 : 2;
  const int L = NT * vec, chunk = 32 * vec;
  if (batch > L) return (batch + L - 1) / L * L;
  if (batch >= chunk) return (batch + chunk - 1) / chunk * chunk;
  return batch;
}

static void layout_state(jt_state* st) {
  const jt_plan* plan = st->plan;
  const int mode = st->mode;
  const int64_t B = st->B;
  st->esz = plan->dtype == JT_F32 ? 4 : 8;
  // clique arena: every clique (materialized); in shared-base mode only the hub
  // cliques (more neighbour ratios + owned evidence masks than a pass carries,
  // MAXF) get per-case tables: they absorb their children eagerly (jt_state::hub)
  int64_t off = 0;
  st->hub.assign(plan->n_cliques, 0);
  for (int c = 0; c < plan->n_cliques; ++c) {
    if (mode == JT_MATERIALIZED) {
      st->coff.push_back(off);
      off = align4(off + plan->csize[c] * B);
      continue;
    }
    int owned = 0;
    for (int v = 0; v < plan->n_vars; ++v)
      if (smallest_holder(plan, v) == c) ++owned;
    st->hub[c] = (int)plan->nbrs[c].size() + owned > MAXF;
    st->coff.push_back(st->hub[c] ? off : -1);
    if (st->hub[c]) off = align4(off + plan->csize[c] * B);
  }
  st->n_clique = off;
  // base replica (one copy of every table, no batch dim): the shared-base
  // engine reads it directly; materialized states reset from it (jt_state_reset)
  int64_t boff = 0;
  for (int c = 0; c < plan->n_cliques; ++c) {
    st->boff.push_back(boff);
    boff = align4(boff + plan->csize[c]);
  }
  st->n_base = boff;
  // aux arena: seps | ratioC | ratioD | msg ratio | evidence vectors
  off = 0;
  auto take = [&](int64_t n) {
    const int64_t o = off;
    off = align4(off + n);
    return o;
  };
  int64_t max_s = 1;
  for (int s = 0; s < plan->n_seps; ++s) st->sep_off.push_back(take(plan->ssize[s] * B));
  for (int s = 0; s < plan->n_seps; ++s) st->ratC_off.push_back(take(plan->ssize[s] * B));
  for (int s = 0; s < plan->n_seps; ++s) st->ratD_off.push_back(take(plan->ssize[s] * B));
  for (int s = 0; s < plan->n_seps; ++s) max_s = std::max(max_s, plan->ssize[s]);
  st->msg_ratio_off = take(max_s * B);
  for (int v = 0; v < plan->n_vars; ++v) st->ev_off.push_back(take((int64_t)plan->cards[v] * B));
  st->n_aux = off;
  int64_t qo = 0;
  for (int v = 0; v < plan->n_vars; ++v) {
    st->q_off.push_back(qo);
    qo += (int64_t)plan->cards[v] * B;
  }
  st->n_qout = std::max<int64_t>(qo, 1);
  st->ev_clique.assign(plan->n_vars, -1);
  st->pre_e.assign(plan->n_cliques, 0);
  st->e_c.assign(plan->n_cliques, 0);
  st->e_s.assign(plan->n_seps, 0);
}

// Exponent that brings a clique table summing to `sum` to about `target`.
static int balance_exp(double sum, double target) {
  if (!(sum > 0.0) || !std::isfinite(sum)) return 0;
  const double e = std::round(std::log2(target / sum));
  return (int)std::max(-900.0, std::min(900.0, e));
}

// pre_e from the clique tables (host, fp64, clique-id order at `at(c)`): each
// clique scaled to sum to its BFS-parent separator's size, roots to 1
// (SURVEY Appendix A balance, as powers of two).
template <class F>
static void choose_prescale(jt_state* st, F at) {
  const jt_plan* p = st->plan;
  std::vector<int64_t> target(p->n_cliques, 1);
  std::vector<char> seen(p->n_cliques, 0);
  std::vector<int> q(p->roots.begin(), p->roots.end());
  for (int r : p->roots) seen[r] = 1;
  for (size_t h = 0; h < q.size(); ++h)
    for (auto& nb : p->nbrs[q[h]])
      if (!seen[nb.first]) {
        seen[nb.first] = 1;
        target[nb.first] = p->ssize[nb.second];
        q.push_back(nb.first);
      }
  for (int c = 0; c < p->n_cliques; ++c) {
    const double* v = at(c);
    double sum = 0.0;
    for (int64_t i = 0; i < p->csize[c]; ++i) sum += v[i];
    st->pre_e[c] = balance_exp(sum, (double)target[c]);
  }
}

// exponent of the joint Π φ_c / Π φ_s: every table of a calibrated state
static int joint_exp(const jt_state* st) {
  int64_t e = 0;
  for (int x : st->e_c) e += x;
  for (int x : st->e_s) e -= x;
  return (int)e;
}

static void set_all_exp(jt_state* st, int e) {
  std::fill(st->e_c.begin(), st->e_c.end(), e);
  std::fill(st->e_s.begin(), st->e_s.end(), e);
}

extern "C" int jt_state_create(const jt_plan* plan, int batch, int mode, jt_state** out) {
  if (!plan || !out || batch < 1 || (mode != JT_MATERIALIZED && mode != JT_SHARED_BASE))
    return JT_ERR_BAD_ARG;
  DevGuard g(plan->device);
  auto st = std::make_unique<jt_state>();
  st->plan = plan;
  st->B = padded_batch(plan, batch);
  st->B_user = batch;
  st->mode = mode;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, plan->device));
  st->num_sms = prop.multiProcessorCount;
  layout_state(st.get());
  const size_t es = st->esz;
  if (st->n_clique) CK(cudaMalloc(&st->d_clique, st->n_clique * es));
  if (st->n_base) CK(cudaMalloc(&st->d_base, st->n_base * es));
  CK(cudaMalloc(&st->d_aux, std::max<int64_t>(st->n_aux, 4) * es));
  CK(cudaMalloc(&st->d_qout, st->n_qout * sizeof(double)));
  // error word [flags, lowest failing case index (INT_MAX: none)]
  CK(cudaMalloc(&st->d_err, 2 * sizeof(int)));
  {
    const int init[2] = {0, INT_MAX};
    CK(cudaMemcpy(st->d_err, init, sizeof init, cudaMemcpyHostToDevice));
  }
  CK(cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking));
  CK(cudaMalloc(&st->d_evoff, std::max(1, plan->n_vars) * sizeof(int64_t)));
  CK(cudaMalloc(&st->d_cards, std::max(1, plan->n_vars) * sizeof(int32_t)));
  if (plan->n_vars) {
    CK(cudaMemcpy(st->d_evoff, st->ev_off.data(), plan->n_vars * sizeof(int64_t), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(st->d_cards, plan->cards.data(), plan->n_vars * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  st->device_bytes = (st->n_clique + st->n_base + st->n_aux) * es + st->n_qout * 8;
  // initial contents: cliques 1 (initialize's np.ones, propagate.py:209), seps 1 (236)
  if (st->n_clique) CK(launch_fill(plan->dtype, st->d_clique, st->n_clique, 1.0, st->stream));
  CK(launch_fill(plan->dtype, st->d_base, st->n_base, 1.0, st->stream));
  CK(launch_fill(plan->dtype, st->d_aux, st->n_aux, 1.0, st->stream));
  CK(cudaStreamSynchronize(st->stream));
  *out = st.release();
  return JT_OK;
}

extern "C" void jt_state_destroy(jt_state* st) {
  if (!st) return;
  DevGuard g(st->plan->device);
  delete st;
}

extern "C" int64_t jt_state_device_bytes(const jt_state* st) { return st ? st->device_bytes : 0; }
extern "C" int64_t jt_state_launch_count(const jt_state* st) { return st ? st->launches : 0; }

static cudaStream_t pick_stream(jt_state* st, void* s) {
  return s ? reinterpret_cast<cudaStream_t>(s) : st->stream;
}

static int ensure_stage(jt_state* st, int64_t n) {
  if (n <= st->stage_cap) return JT_OK;
  cudaFree(st->d_stage);
  st->d_stage = nullptr;
  st->stage_cap = 0;
  CK(cudaMalloc(&st->d_stage, std::max<int64_t>(n, 1) * sizeof(double)));
  st->stage_cap = n;
  return JT_OK;
}

// ------------------------------------------------------- pass compiler ----
struct Dim {
  int64_t card;
  int64_t src, dst, out;
  int64_t fac[MAXF];
};

static int64_t tensor_stride(const jt_plan* p, const Tensor& t, int var, int64_t B) {
  // var < 0 denotes the batch dim
  if (var < 0) return t.batch ? 1 : 0;
  auto it = std::find(t.vars.begin(), t.vars.end(), var);
  if (it == t.vars.end()) return 0;
  int64_t s = t.batch ? B : 1;
  for (auto j = it + 1; j != t.vars.end(); ++j) s *= p->cards[*j];
  return s;
}

struct BuiltPass {
  DevPass d;
  std::vector<int64_t> blk;
  std::vector<int32_t> blk32;
  std::vector<int32_t> bins;
  std::vector<int32_t> rowtab;
  int64_t n_part = 0;
  int64_t n_cnt = 0;
  std::vector<Item> items;
};

static std::vector<Dim> pass_dims(const jt_state* st, const PassSpec& ps) {
  const jt_plan* p = st->plan;
  const int64_t B = st->B;
  const auto& cv = ps.scope.empty() ? p->cvars[ps.clique] : ps.scope;
  std::vector<int> vars(cv.begin(), cv.end());
  if (B > 1) vars.push_back(-1);
  // lanes per block for the thread-owned path: one vector per thread
  const int64_t L = (int64_t)NT * (st->esz == 4 ? 4 : 2);
  Tensor src;
  src.vars = cv;
  src.batch = (B > 1) && (ps.src_arena == A_CLIQUE || ps.src_arena == A_AUX);
  Tensor dst;
  dst.vars = cv;
  dst.batch = B > 1;
  std::vector<Dim> dims;
  for (int v : vars) {
    Dim d{};
    d.card = v < 0 ? B : p->cards[v];
    d.src = tensor_stride(p, src, v, B);
    d.dst = ps.write ? tensor_stride(p, dst, v, B) : 0;
    d.out = ps.out_kind != OUT_NONE ? tensor_stride(p, ps.out, v, B) : 0;
    for (size_t f = 0; f < ps.factors.size(); ++f) d.fac[f] = tensor_stride(p, ps.factors[f], v, B);
    if (v < 0 && B > L && B % L == 0) {
      // split the case dim into (B/L outer, L inner lanes); every stride of the
      // outer part is the lane stride times L
      Dim hi = d;
      hi.card = B / L;
      hi.src *= L;
      hi.dst *= L;
      hi.out *= L;
      for (size_t f = 0; f < ps.factors.size(); ++f) hi.fac[f] *= L;
      d.card = L;
      dims.push_back(hi);
    }
    dims.push_back(d);
  }
  if (dims.empty()) {  // empty clique scope: a single entry
    Dim d{};
    d.card = 1;
    dims.push_back(d);
  }
  return dims;
}

static int pass_max_vec(const jt_state* st, const PassSpec& ps) {
  auto dims = pass_dims(st, ps);
  const int64_t c = dims.back().card;
  const int maxv = st->esz == 4 ? 4 : 2;
  for (int v = maxv; v > 1; v >>= 1)
    if (c % v == 0) return v;
  return 1;
}

static bool mergeable(const Dim& a, const Dim& b, int nf) {
  auto ok = [](int64_t sa, int64_t sb, int64_t cb) { return (sa == 0 && sb == 0) || (sb != 0 && sa == sb * cb); };
  if (!ok(a.src, b.src, b.card) || !ok(a.dst, b.dst, b.card) || !ok(a.out, b.out, b.card)) return false;
  for (int f = 0; f < nf; ++f)
    if (!ok(a.fac[f], b.fac[f], b.card)) return false;
  return true;
}

static std::vector<Dim> merge_dims(const std::vector<Dim>& in, int nf) {
  std::vector<Dim> out;
  for (const Dim& d : in) {
    if (!out.empty() && mergeable(out.back(), d, nf)) {
      Dim m = d;  // strides of the inner dim, card multiplied
      m.card = out.back().card * d.card;
      out.back() = m;
    } else {
      out.push_back(d);
    }
  }
  return out;
}

static int compile_pass(const jt_state* st, const PassSpec& ps, int vec, int pass_idx, BuiltPass& bp,
                        bool allow_row = true, int kv = KV, bool allow_own = true) {
  const int nf = (int)ps.factors.size();
  if (nf > MAXF) return JT_ERR_UNSUPPORTED;
  std::vector<Dim> dims = pass_dims(st, ps);
  const int nd = (int)dims.size();
  const int TH = NT * kv * vec;
  const bool has_out = ps.out_kind != OUT_NONE;
  if (ps.write && !ps.scope.empty()) return JT_ERR_UNSUPPORTED;
  int64_t total = 1;
  for (auto& d : dims) total *= d.card;

  struct Cand {
    int k;
    bool own = false;
    bool row = false;
    int own_m = 0;
    int gpi = 1;
    int64_t j_per_item = 1;
    int64_t T, n_in, n_out, r_out;
    int BPI;
    int64_t n_chunks, bpc;
    double cost;
    std::vector<Dim> inner;
  };
  Cand best{};
  best.cost = 1e300;
  bool found = false;
  int64_t T = 1;
  for (int k = nd - 1; k >= 0; --k) {
    T *= dims[k].card;
    if (T > TH) break;
    if (T % vec) continue;
    std::vector<Dim> inner(dims.begin() + k, dims.end());
    std::vector<Dim> im = merge_dims(inner, nf);
    if ((int)im.size() > MAXDI) continue;
    Cand c;
    c.k = k;
    c.T = T;
    c.inner = im;
    c.n_in = 1;
    for (auto& d : inner)
      if (has_out && d.out) c.n_in *= d.card;
    c.n_out = 1;
    c.r_out = 1;
    for (int i = 0; i < k; ++i) {
      if (has_out && dims[i].out) c.n_out *= dims[i].card;
      else c.r_out *= dims[i].card;
    }
    c.own_m = 0;
    if (has_out && c.n_in == T && T % ((int64_t)NT * vec) == 0) {
      const int64_t m = T / ((int64_t)NT * vec);
      // M > 1 only for full-width vectors (the templated load-shape kernels)
      bool allf = true;  // M > 1 kernels load every factor as a full vector
      for (int f = 0; f < nf; ++f) allf = allf && dims.back().fac[f] == 1;
      if (m == 1 || ((m == 2 || m == 4) && vec == (st->esz == 4 ? 4 : 2) && allf)) c.own_m = (int)m;
    }
    // the thread-owned kernel is validated for one merged inner dimension only
    // (batched states: the case dim); multi-dim inner blocks take the general kernel
    static const bool own_multi = env_int("JT_OWN_MULTI", 0) != 0;
    if ((im.size() > 1 && !own_multi) || !allow_own) c.own_m = 0;
    c.own = c.own_m > 0;
    c.BPI = c.own ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(TH / T, c.r_out));
    // several whole output groups per iteration when a group is smaller than an iteration
    c.gpi = 1;
    if (!c.own && has_out && c.r_out * T * 2 <= TH && c.n_out > 1) {
      c.gpi = (int)std::min<int64_t>(TH / (c.r_out * T), c.n_out);
      if (c.gpi * c.n_in > 4096) c.gpi = (int)std::max<int64_t>(1, 4096 / c.n_in);
      if (c.gpi > 1) c.BPI = (int)(c.gpi * c.r_out);
    }
    // row passes (one output entry per item, or none) run on the lean row kernel
    const int64_t tw = T / (32 * vec);
    if (allow_row && !c.own && c.gpi == 1 && (!has_out || c.n_in == 1) && T % (32 * vec) == 0 &&
        (tw == 1 || tw == 2 || tw == 4 || tw % KROW == 0)) {
      c.row = true;
      c.BPI = 1;
    }
    // chunking: ~8 items per SM slot for big passes, >= 2 iterations per item otherwise
    // single trees: ~2 items per SM slot (measured: c3 0.278 -> 0.238 ms fp32, 0.561 -> 0.534 fp64;
    // the batch program does not move); batches keep 8
    const int ips = env_int("JT_ITEMS_PER_SM", st->B == 1 ? 2 : 8);
    static const int min_it = env_int("JT_MIN_ITERS", 2);
    const int64_t per_item = std::max<int64_t>((int64_t)min_it * TH, total / (int64_t)(st->num_sms * ips));
    const int64_t desired = std::max<int64_t>(1, (total + per_item - 1) / per_item);
    const int64_t max_chunks = (c.r_out + c.BPI - 1) / c.BPI;
    int64_t nch = has_out ? (desired + c.n_out - 1) / c.n_out : desired;
    // thread-owned column passes: every chunk costs n_in partials, so split only as far
    // as one item per resident CTA needs (~3 per SM)
    if (c.own && has_out)
      nch = std::min<int64_t>(nch, ((int64_t)st->num_sms * 3 + c.n_out - 1) / c.n_out);
    if ((c.own || c.gpi > 1) && c.r_out * T <= per_item) nch = 1;  // whole groups per item instead
    if (c.own && getenv("JT_OWN_NOCHUNK")) nch = 1;
    nch = std::max<int64_t>(1, std::min(nch, max_chunks));
    int64_t bpc = (c.r_out + nch - 1) / nch;
    bpc = (bpc + c.BPI - 1) / c.BPI * c.BPI;
    c.bpc = bpc;
    c.n_chunks = (c.r_out + bpc - 1) / bpc;
    c.j_per_item = 1;
    // own items: ~16 blocks, so concurrently running CTAs walk neighbouring
    // output groups and share their factor rows in L2
    if (c.own && c.n_chunks == 1)
      c.j_per_item = std::max<int64_t>(1, (16 / c.own_m) / std::max<int64_t>(1, c.r_out));
    if (c.gpi > 1) {
      c.n_chunks = 1;
      c.bpc = c.r_out;
      c.j_per_item = std::max<int64_t>(c.gpi, per_item / std::max<int64_t>(1, c.r_out * T) / c.gpi * c.gpi);
    }
    const double esz = st->esz;
    double bytes = (double)total * esz * ((ps.src_arena == A_CLIQUE ? 1.0 : 0.05) + (ps.write ? 1.0 : 0.0));
    const int64_t ng = (c.n_chunks + 31) / 32;
    double part = (has_out && c.n_chunks > 1) ? (double)c.n_out * (c.n_chunks + ng) * c.n_in * 16.0 : 0.0;
    double items = (double)c.n_out * c.n_chunks / c.j_per_item;
    // per-item epilogue: block reduction (general path) or nothing (own path);
    // the last CTA of a group sums <= 32 partial rows of n_in values per level
    double epi = c.own ? 256.0 : 4096.0;
    if (c.gpi > 1) epi = 4096.0 * c.j_per_item / c.gpi;  // one smem reduction per iteration
    double fin = (has_out && c.n_chunks > 1) ? (double)c.n_out * std::min<int64_t>(32, c.n_chunks) * c.n_in * 64.0 : 0.0;
    // single-tree states: the measured streaming efficiency of the kernels
    // (profiles/README.md: general ~2 TB/s, row 3.5-5.7 TB/s) weighs the bytes
    if (st->B == 1) bytes *= c.row ? 1.0 : c.own ? 1.25 : 2.0;
    double pen = 0.0;
    if (T * esz < 128) pen = bytes * (128.0 / (T * esz) - 1.0) * 0.5;
    c.cost = bytes + part + items * epi + fin + pen + (double)c.n_out * c.r_out * (c.own ? (st->B == 1 ? 64.0 : 2048.0) : 16.0);
    if (getenv("JT_DEBUG_COST"))
      fprintf(stderr, "cand clique %d T %lld n_in %lld n_out %lld r_out %lld own %d/%d row %d gpi %d nch %lld cost %.3g "
              "(bytes %.3g part %.3g items %.3g fin %.3g pen %.3g)\n", ps.clique, (long long)c.T, (long long)c.n_in,
              (long long)c.n_out, (long long)c.r_out, (int)c.own, c.own_m, (int)c.row, c.gpi, (long long)c.n_chunks,
              c.cost, bytes, part, items * epi, fin, pen);
    if (!found || c.cost < best.cost * 0.999) {
      best = c;
      found = true;
    }
  }
  if (!found) return JT_ERR_UNSUPPORTED;

  DevPass& d = bp.d;
  std::memset(&d, 0, sizeof(d));
  d.src_arena = ps.src_arena;
  d.src_off = ps.src_arena == A_AUX ? ps.src_off : ps.src_arena == A_CLIQUE ? st->coff[ps.clique] : st->boff[ps.clique];
  d.dst_off = ps.write ? st->coff[ps.clique] : -1;
  d.nf = nf;
  d.fac_vec = 0;
  for (int f = 0; f < nf; ++f) {
    d.fac_off[f] = ps.factors[f].off;
    if (dims.back().fac[f] == 1) d.fac_vec |= 1u << f;
  }
  d.src_vec = dims.back().src == 1 ? 1 : 0;
  d.out_kind = ps.out_kind;
  d.out_off = has_out ? ps.out.off : 0;
  d.ratio_off = ps.ratio_off;
  d.out2_off = ps.out2_off;
  d.T = (int)best.T;
  d.BPI = best.BPI;
  d.n_in = (int)best.n_in;
  d.n_chunks = (int)best.n_chunks;
  d.n_blocks_per_jout = best.r_out;
  d.blocks_per_chunk = best.bpc;
  d.blk_stride = 2 + nf;
  d.own = best.own ? 1 : 0;
  d.row = best.row ? 1 : 0;
  d.kv = kv;
  d.own_m = best.own_m;
  d.flush_fac = 0;
  // group-constant factors are multiplied into the group SUM at the flush, so a
  // pass that also writes its clique table must take every factor per element
  // (otherwise the written table misses them: wrong posteriors downstream)
  if (best.own && !ps.write && !getenv("JT_OWN_NOFLUSH")) {
    for (int f = 0; f < nf; ++f) {
      bool constant = true;
      for (int i = 0; i < best.k; ++i)
        if (!(has_out && dims[i].out) && dims[i].fac[f] != 0) constant = false;
      if (constant) d.flush_fac |= 1u << f;
    }
  }
  d.gpi = best.gpi;
  d.ndi = (int)best.inner.size();
  for (int i = 0; i < d.ndi; ++i) {
    const Dim& x = best.inner[i];
    d.icard[i] = (int)x.card;
    d.isrc[i] = (int)x.src;
    d.idst[i] = (int)x.dst;
    d.iout[i] = (int)x.out;
    for (int f = 0; f < nf; ++f) d.ifac[f][i] = (int)x.fac[f];
  }
  // block table: j_out-major over the separator dims outside the block, then
  // the remaining outer dims
  std::vector<int> so, ro;
  for (int i = 0; i < best.k; ++i) ((has_out && dims[i].out) ? so : ro).push_back(i);
  const int64_t nblk = best.n_out * best.r_out;
  bp.blk.assign(nblk * (2 + nf), 0);
  std::vector<int64_t> dig_s(so.size(), 0), dig_r(ro.size(), 0);
  int64_t bi = 0;
  for (int64_t jo = 0; jo < best.n_out; ++jo) {
    int64_t s_src = 0, s_dst = 0, s_fac[MAXF] = {0};
    {
      int64_t x = jo;
      for (int t = (int)so.size() - 1; t >= 0; --t) {
        const Dim& dd = dims[so[t]];
        const int64_t dg = x % dd.card;
        x /= dd.card;
        s_src += dg * dd.src;
        s_dst += dg * dd.dst;
        for (int f = 0; f < nf; ++f) s_fac[f] += dg * dd.fac[f];
      }
    }
    std::fill(dig_r.begin(), dig_r.end(), 0);
    int64_t r_src = 0, r_dst = 0, r_fac[MAXF] = {0};
    for (int64_t po = 0; po < best.r_out; ++po) {
      int64_t* e = &bp.blk[bi * (2 + nf)];
      e[0] = s_src + r_src;
      e[1] = s_dst + r_dst;
      for (int f = 0; f < nf; ++f) e[2 + f] = s_fac[f] + r_fac[f];
      ++bi;
      // odometer increment over the rest-outer dims (last fastest)
      for (int t = (int)ro.size() - 1; t >= 0; --t) {
        const Dim& dd = dims[ro[t]];
        dig_r[t]++;
        r_src += dd.src;
        r_dst += dd.dst;
        for (int f = 0; f < nf; ++f) r_fac[f] += dd.fac[f];
        if (dig_r[t] < dd.card) break;
        r_src -= dd.src * dd.card;
        r_dst -= dd.dst * dd.card;
        for (int f = 0; f < nf; ++f) r_fac[f] -= dd.fac[f] * dd.card;
        dig_r[t] = 0;
      }
    }
  }
  // row passes: inner-offset table [2+nf][T/VEC] and warp units
  if (best.row) {
    const int TV = (int)(best.T / vec);
    bp.rowtab.assign((size_t)(2 + nf) * TV, 0);
    d.row_lin = 1;
    for (int iv = 0; iv < TV; ++iv) {
      int64_t rem = (int64_t)iv * vec, so = 0, dd = 0, fo[MAXF] = {0};
      for (int i = d.ndi - 1; i >= 0; --i) {
        const int64_t dig = rem % d.icard[i];
        rem /= d.icard[i];
        so += dig * d.isrc[i];
        dd += dig * d.idst[i];
        for (int f = 0; f < nf; ++f) fo[f] += dig * d.ifac[f][i];
      }
      if (so != (int64_t)iv * vec || (ps.write && dd != (int64_t)iv * vec) || !d.src_vec || TV / 32 < KROW)
        d.row_lin = 0;
      bp.rowtab[iv] = (int32_t)so;
      bp.rowtab[TV + iv] = (int32_t)dd;
      for (int f = 0; f < nf; ++f) bp.rowtab[(size_t)(2 + f) * TV + iv] = (int32_t)fo[f];
    }
    d.row_fmode = 0;
    for (int f = 0; f < nf; ++f) {
      bool lin = true, zero = true;
      for (int iv = 0; iv < TV; ++iv) {
        const int32_t x = bp.rowtab[(size_t)(2 + f) * TV + iv];
        lin = lin && x == iv * vec && ((d.fac_vec >> f) & 1u);
        zero = zero && x == 0 && !((d.fac_vec >> f) & 1u);  // the VEC lanes of a vector must agree too
      }
      d.row_fmode |= (uint32_t)(zero ? 2 : lin ? 1 : 0) << (2 * f);
    }
    const int64_t grp_el = best.r_out * best.T;
    // ~4 units per warp of a full-occupancy grid (3 CTAs x 8 warps per SM), >= one batch each
    const int64_t unit = std::max<int64_t>((int64_t)32 * vec * KROW, total / ((int64_t)st->num_sms * 24 * 4));
    if (has_out && grp_el > 2 * unit) {
      int64_t bpc = std::max<int64_t>(1, unit / best.T);
      while ((best.r_out + bpc - 1) / bpc > 32 * CHUNK_GROUP) bpc *= 2;
      d.blocks_per_chunk = bpc;
      d.n_chunks = (int)((best.r_out + bpc - 1) / bpc);
    } else if (!has_out) {
      // no output: any split of the blocks is fine; units of ~unit elements
      int64_t bpc = std::max<int64_t>(1, unit / best.T);
      d.blocks_per_chunk = bpc;
      d.n_chunks = (int)((best.r_out + bpc - 1) / bpc);
    } else {
      d.n_chunks = 1;
      d.blocks_per_chunk = best.r_out;
    }
    best.n_chunks = d.n_chunks;
    best.j_per_item = d.n_chunks == 1 ? std::max<int64_t>(1, unit / grp_el) : 1;
  }
  // thread-owned passes read a compact int32 table: every column in units of
  // the largest power-of-two-free common step (T for lane-strided tensors)
  if (best.own || best.row) {
    const int ncol = 2 + nf;
    std::vector<int64_t> unit(ncol, 1);  // plain int32 element offsets
    bp.blk32.resize(bp.blk.size());
    bool fits = true;
    for (int64_t b = 0; b < nblk && fits; ++b)
      for (int c = 0; c < ncol; ++c) {
        const int64_t q = bp.blk[b * ncol + c] / unit[c];
        if (q > INT32_MAX) fits = false;
        bp.blk32[b * ncol + c] = (int32_t)q;
      }
    if (!fits || unit[0] > INT32_MAX || unit[1] > INT32_MAX) return JT_ERR_UNSUPPORTED;
    d.unit_src = (int)unit[0];
    d.unit_dst = (int)unit[1];
    for (int f = 0; f < nf; ++f) {
      if (unit[2 + f] > INT32_MAX) return JT_ERR_UNSUPPORTED;
      d.unit_fac[f] = (int)unit[2 + f];
    }
  }
  // bin tables: position(b, p) = binbase[b] + binrest[p] over the inner block
  if (has_out && d.n_in > 1) {
    std::vector<int64_t> pstride(d.ndi, 1);
    for (int i = d.ndi - 2; i >= 0; --i) pstride[i] = pstride[i + 1] * d.icard[i + 1];
    std::vector<int64_t> bb{0}, br{0};
    for (int i = 0; i < d.ndi; ++i) {
      auto& tgt = d.iout[i] ? bb : br;
      std::vector<int64_t> nx;
      nx.reserve(tgt.size() * d.icard[i]);
      for (int64_t o : tgt)
        for (int c = 0; c < d.icard[i]; ++c) nx.push_back(o + c * pstride[i]);
      tgt.swap(nx);
    }
    for (auto x : bb) bp.bins.push_back((int32_t)x);
    for (auto x : br) bp.bins.push_back((int32_t)x);
  }
  if (has_out && d.n_chunks > 1) {
    const int64_t ng = (best.n_chunks + 31) / 32;
    bp.n_part = best.n_out * (best.n_chunks + ng) * best.n_in;
    bp.n_cnt = best.n_out * (ng + 1);
  }
  if ((best.own || best.gpi > 1 || best.row) && best.n_chunks == 1) {
    for (int64_t jo = 0; jo < best.n_out; jo += best.j_per_item)
      bp.items.push_back(Item{pass_idx, 0, jo, std::min(best.j_per_item, best.n_out - jo)});
  } else {
    for (int64_t jo = 0; jo < best.n_out; ++jo)
      for (int64_t ch = 0; ch < best.n_chunks; ++ch) bp.items.push_back(Item{pass_idx, (int)ch, jo, 1});
  }
  return JT_OK;
}

// waves touching fewer elements than this are launch-latency bound
#ifndef SMALL_WAVE_LOG2
#define SMALL_WAVE_LOG2 21
#endif
constexpr int64_t SMALL_WAVE_ELEMS = int64_t(1) << SMALL_WAVE_LOG2;

struct HostProgram {
  std::vector<WaveRt> waves;
  std::vector<DevPass> passes;
  std::vector<Item> items;
  std::vector<int64_t> blk;
  std::vector<int32_t> blk32;
  std::vector<int32_t> bins;
  std::vector<int32_t> rowtab;
  std::vector<int> pass_clique;
  int64_t n_part = 0, n_cnt = 0;
  std::vector<CPass> cpasses;
  std::vector<int32_t> ctab;
  std::vector<double> w;
  std::vector<int> cpass_clique;
  std::vector<RowiParam> rparams;
  std::vector<TileParam> tparams;
  std::map<int, VDesc> vdesc;  // virtual separators by leaf clique (Wv built once)
  std::vector<VCodeTask> vcode;  // their evidence mask codes, computed at the start of every run
};

// ----------------------------------------------------- contraction passes --

static bool has_virtual(const PassSpec& ps) {
  if (ps.out.vclique >= 0) return true;
  for (auto& f : ps.factors)
    if (f.vclique >= 0) return true;
  return false;
}

static bool contract_eligible(const jt_state* st, const PassSpec& ps) {
  return st->mode == JT_SHARED_BASE && st->B > 1 && st->B % CVEC == 0 && !st->h_base.empty() &&
         ps.src_arena == A_BASE && !ps.write && ps.scope.empty() && ps.out_kind != OUT_NONE &&
         !getenv("JT_NO_CONTRACT");
}

// Mixed-radix enumeration of a var group: offsets (per tensor) of every index.
static std::vector<int64_t> group_offsets(const jt_plan* p, const std::vector<int>& vars,
                                          const std::vector<int64_t>& stride_of_var) {
  std::vector<int64_t> out{0};
  for (size_t a = 0; a < vars.size(); ++a) {
    const int c = p->cards[vars[a]];
    std::vector<int64_t> nx;
    nx.reserve(out.size() * c);
    for (int64_t o : out)
      for (int d = 0; d < c; ++d) nx.push_back(o + d * stride_of_var[a]);
    out.swap(nx);
  }
  return out;
}

// Wv[j][k] (the leaf's base summed onto its separator entry j and private state
// k; the row sum, accumulated in the arena type in k order, at [j][nK]) and the
// mask-code task of a virtual separator; built once per program and leaf.
// Appends to hp.w (rolled back with the pass that built it).
static int64_t tsize_entries(const jt_plan* p, const Tensor& t) {
  int64_t n = 1;
  for (int v : t.vars) n *= p->cards[v];
  return n;
}

static int virtual_sep(const jt_state* st, const Tensor& t, HostProgram& hp, VDesc& vd) {
  auto it = hp.vdesc.find(t.vclique);
  if (it != hp.vdesc.end()) {
    vd = it->second;
    return JT_OK;
  }
  const jt_plan* p = st->plan;
  const int c = t.vclique;
  const auto& C = p->cvars[c];
  std::vector<int> K;
  std::set_difference(C.begin(), C.end(), t.vars.begin(), t.vars.end(), std::back_inserter(K));
  // the gather form needs the leaf's evidence to be the 0/1 mask of its one private variable
  if (t.vfac.size() > 1 || (t.vfac.size() == 1 && t.vfac[0].vars != K)) return JT_ERR_UNSUPPORTED;
  int64_t nK = 1, nJ = 1;
  for (int v : K) nK *= p->cards[v];
  for (int v : t.vars) nJ *= p->cards[v];
  if (nJ * (nK + 1) > INT32_MAX) return JT_ERR_UNSUPPORTED;
  Tensor te = t;
  te.batch = false;
  std::vector<int64_t> cj(C.size(), 0), ck(C.size(), 0);
  for (size_t a = 0; a < C.size(); ++a) {
    cj[a] = tensor_stride(p, te, C[a], 1);
    int64_t st_ = 1;
    bool in = false;
    for (int b = (int)K.size() - 1; b >= 0; --b) {
      if (K[b] == C[a]) {
        in = true;
        break;
      }
      st_ *= p->cards[K[b]];
    }
    ck[a] = in ? st_ : 0;
  }
  const int64_t w0 = ((int64_t)hp.w.size() + 7) & ~int64_t(7);
  hp.w.resize(w0 + nJ * (nK + 1), 0.0);
  double* W = hp.w.data() + w0;
  const double* src = st->h_base.data() + st->boff[c];
  std::vector<int> dig(C.size(), 0);
  int64_t xj = 0, xk = 0;
  for (int64_t e = 0; e < p->csize[c]; ++e) {
    W[xj * (nK + 1) + xk] += src[e];
    for (int a = (int)C.size() - 1; a >= 0; --a) {
      xj += cj[a];
      xk += ck[a];
      if (++dig[a] < p->cards[C[a]]) break;
      xj -= cj[a] * p->cards[C[a]];
      xk -= ck[a] * p->cards[C[a]];
      dig[a] = 0;
    }
  }
  for (int64_t j = 0; j < nJ; ++j) {  // the unobserved case: Σ_k in k order, arena precision
    double* r = W + j * (nK + 1);
    if (st->esz == 8) {
      double acc = 0.0;
      for (int64_t k = 0; k < nK; ++k) acc += r[k];
      r[nK] = acc;
    } else {
      float acc = 0.0f;
      for (int64_t k = 0; k < nK; ++k) acc += (float)r[k];
      r[nK] = (double)acc;
    }
  }
  std::memset(&vd, 0, sizeof(vd));
  vd.w_off = w0;
  vd.nK = (int)nK;
  vd.code_off = -1;
  if (!t.vfac.empty()) {
    VCodeTask tk;
    std::memset(&tk, 0, sizeof(tk));
    tk.mask_off = t.vfac[0].off;
    tk.card = (int)nK;
    vd.code_off = (int64_t)hp.vcode.size() * st->B;
    hp.vcode.push_back(tk);
  }
  hp.vdesc[c] = vd;
  return JT_OK;
}

#ifndef CON_NCG_MID
#define CON_NCG_MID 4  // case chunks per unit group for 8 <= nK < 32
#endif
#ifndef CON_NCG_SMALL
#define CON_NCG_SMALL 1  // and for nK < 8 (a unit walks all case chunks)
#endif
static int compile_contract(const jt_state* st, const PassSpec& ps, HostProgram& hp, CPass& cp,
                            const PassSpec* ps_b = nullptr) {
  const jt_plan* p = st->plan;
  const int64_t B = st->B;
  const auto& C = p->cvars[ps.clique];
  const auto& s = ps.out.vars;
  auto subset = [](const std::vector<int>& a, const std::vector<int>& b) {
    return std::includes(b.begin(), b.end(), a.begin(), a.end());
  };
  std::vector<const Tensor*> G, E;
  for (auto& f : ps.factors) (subset(f.vars, s) ? E : G).push_back(&f);
  if ((int)G.size() > CMAXG || (int)E.size() > MAXF) return JT_ERR_UNSUPPORTED;

  std::vector<int> U;
  for (auto* f : G) U.insert(U.end(), f->vars.begin(), f->vars.end());
  std::sort(U.begin(), U.end());
  U.erase(std::unique(U.begin(), U.end()), U.end());
  std::vector<int> I, S, K;
  std::set_intersection(s.begin(), s.end(), U.begin(), U.end(), std::back_inserter(I));
  std::set_difference(s.begin(), s.end(), U.begin(), U.end(), std::back_inserter(S));
  std::set_difference(U.begin(), U.end(), s.begin(), s.end(), std::back_inserter(K));
  const int nG = (int)G.size(), nE = (int)E.size();
  // second output: same scope, same G factors (hence same I, K', W); its own E factors
  std::vector<const Tensor*> Eb;
  if (ps_b) {
    std::vector<const Tensor*> Gb;
    for (auto& f : ps_b->factors) (subset(f.vars, s) ? Eb : Gb).push_back(&f);
    if (ps_b->out.vars != s || ps_b->clique != ps.clique || Gb.size() != G.size() || (int)Eb.size() > MAXF)
      return JT_ERR_UNSUPPORTED;
    for (size_t g = 0; g < G.size(); ++g)
      if (Gb[g]->off != G[g]->off || Gb[g]->vars != G[g]->vars) return JT_ERR_UNSUPPORTED;
    if (!std::includes(U.begin(), U.end(), s.begin(), s.end())) return JT_ERR_UNSUPPORTED;  // row-per-i only
  }
  const int nEb = (int)Eb.size();
  // virtual separators read by this pass (E factors, old separators), distinct by leaf
  std::vector<const Tensor*> V;
  auto vid = [&](const Tensor* t) -> int {
    if (t->vclique < 0) return -1;
    for (size_t q = 0; q < V.size(); ++q)
      if (V[q]->vclique == t->vclique) return (int)q;
    V.push_back(t);
    return (int)V.size() - 1;
  };
  for (auto* f : G)
    if (f->vclique >= 0) return JT_ERR_UNSUPPORTED;  // (gathered in the epilogue only)
  int8_t e_v[MAXF], e_v_b[MAXF];
  for (int e = 0; e < nE; ++e) e_v[e] = (int8_t)vid(E[e]);
  for (int e = 0; e < nEb; ++e) e_v_b[e] = (int8_t)vid(Eb[e]);
  // a fresh distribute output whose final table is rebuilt on demand needs no old
  // separator (unless it feeds the clique product X): ratio only
  auto kind_of = [](const PassSpec& q) {
    return q.out_kind == OUT_SEP_DFRESH && q.skip_out2 && q.x_off < 0 && env_int("JT_DRATIO", 1) ? OUT_SEP_DRATIO
                                                                                                 : q.out_kind;
  };
  const int8_t old_v = kind_of(ps) == OUT_SEP_DRATIO ? (int8_t)-1 : (int8_t)vid(&ps.out);
  const int8_t old_v_b = ps_b && kind_of(*ps_b) != OUT_SEP_DRATIO ? (int8_t)vid(&ps_b->out) : (int8_t)-1;
  if ((int)V.size() > CMAXV) return JT_ERR_UNSUPPORTED;
  if (old_v >= 0 && ps.out_kind != OUT_SEP && ps.out_kind != OUT_SEP_DFRESH) return JT_ERR_UNSUPPORTED;
  if (old_v_b >= 0 && ps_b->out_kind != OUT_SEP && ps_b->out_kind != OUT_SEP_DFRESH) return JT_ERR_UNSUPPORTED;
  const int nV = (int)V.size();
  // enumeration order of i (any order works: every i-dependent offset comes from
  // the per-i table): the variables that index the largest factor tensors vary
  // slowest, so consecutive i (consecutive warps) re-read the same factor rows
  // while they are still in L2
  {
    std::vector<std::pair<double, int>> cost;
    for (size_t a = 0; a < I.size(); ++a) {
      double c = 0.0;
      for (auto* f : G)
        if (std::binary_search(f->vars.begin(), f->vars.end(), I[a])) {
          double n = (double)B;
          for (int v : f->vars) n *= p->cards[v];
          c += n;
        }
      cost.push_back({-c, (int)a});  // most expensive first (outermost)
    }
    std::stable_sort(cost.begin(), cost.end());
    std::vector<int> Io;
    for (auto& x : cost) Io.push_back(I[x.second]);
    if (getenv("JT_IPERM_REV")) std::reverse(Io.begin(), Io.end());
    if (!getenv("JT_NO_IPERM")) I.swap(Io);
  }
  auto strides = [&](const std::vector<int>& vars, const Tensor& t) {
    std::vector<int64_t> o;
    if (t.vclique >= 0) {  // virtual separator: offsets of its Wv rows ([entries][nK + 1])
      Tensor te = t;
      te.batch = false;
      const int64_t row = p->csize[t.vclique] / std::max<int64_t>(1, tsize_entries(p, t)) + 1;
      for (int v : vars) o.push_back(tensor_stride(p, te, v, 1) * row);
      return o;
    }
    for (int v : vars) o.push_back(tensor_stride(p, t, v, B));
    return o;
  };
  // per-group offset lists of every tensor
  std::vector<std::vector<int64_t>> gI(nG), gK(nG), eI(nE), eS(nE);
  for (int g = 0; g < nG; ++g) {
    gI[g] = group_offsets(p, I, strides(I, *G[g]));
    gK[g] = group_offsets(p, K, strides(K, *G[g]));
  }
  for (int e = 0; e < nE; ++e) {
    eI[e] = group_offsets(p, I, strides(I, *E[e]));
    eS[e] = group_offsets(p, S, strides(S, *E[e]));
  }
  std::vector<std::vector<int64_t>> ebI(nEb), ebS(nEb);
  for (int e = 0; e < nEb; ++e) {
    ebI[e] = group_offsets(p, I, strides(I, *Eb[e]));
    ebS[e] = group_offsets(p, S, strides(S, *Eb[e]));
  }
  // outputs are written in the batch layout (a virtual old separator's other
  // outputs — ratio, final table — are stored tensors at the same offsets)
  auto stored = [](const Tensor& t) {
    Tensor x = t;
    x.vclique = -1;
    return x;
  };
  std::vector<int64_t> obI, obS;
  if (ps_b) {
    obI = group_offsets(p, I, strides(I, stored(ps_b->out)));
    obS = group_offsets(p, S, strides(S, stored(ps_b->out)));
  }
  const std::vector<int64_t> oI = group_offsets(p, I, strides(I, stored(ps.out)));
  const std::vector<int64_t> oS = group_offsets(p, S, strides(S, stored(ps.out)));
  const int64_t nI = (int64_t)oI.size(), nS = (int64_t)oS.size();
  if (nV > 0 && nS != 1) return JT_ERR_UNSUPPORTED;  // the row-per-i epilogue evaluates them
  // per-i entry index of each virtual separator (its vars are output = i variables)
  std::vector<std::vector<int64_t>> vI(nV);
  for (int q = 0; q < nV; ++q) vI[q] = group_offsets(p, I, strides(I, *V[q]));
  const int64_t nK = (int64_t)group_offsets(p, K, std::vector<int64_t>(K.size(), 0)).size();
  if (nI * nK * (nS + 7) > (int64_t)1 << 31) return JT_ERR_UNSUPPORTED;
  auto fits = [](const std::vector<int64_t>& v) {
    for (int64_t x : v)
      if (x > INT32_MAX) return false;
    return true;
  };
  for (int g = 0; g < nG; ++g)
    if (!fits(gI[g]) || !fits(gK[g])) return JT_ERR_UNSUPPORTED;
  for (int e = 0; e < nE; ++e)
    if (!fits(eI[e]) || !fits(eS[e])) return JT_ERR_UNSUPPORTED;
  if (!fits(oI) || !fits(oS)) return JT_ERR_UNSUPPORTED;
  for (int e = 0; e < nEb; ++e)
    if (!fits(ebI[e]) || !fits(ebS[e])) return JT_ERR_UNSUPPORTED;
  if (ps_b && (!fits(obI) || !fits(obS))) return JT_ERR_UNSUPPORTED;
  // W[i][k][s'] = Σ_R base: walk the clique once, odometer over its variables
  // nS == 1 uses the row-per-i kernel
  const bool rowi = nS == 1;
  const int64_t nSp = rowi ? 1 : (nS + 7) & ~int64_t(7);  // W rows padded: two 4-vector loads per k
  // every pass's W starts 64-byte aligned: the tile kernel loads W rows as
  // 16-byte vectors, and a preceding row-per-i pass leaves an arbitrary length
  const int64_t w0 = ((int64_t)hp.w.size() + 7) & ~int64_t(7);
  hp.w.resize(w0 + nI * nK * nSp, 0.0);
  {
    // per clique position: contribution to i, k, s' linear indices (R: none)
    std::vector<int64_t> ci(C.size(), 0), ck(C.size(), 0), cs(C.size(), 0);
    auto lin = [&](const std::vector<int>& grp, int v) {
      int64_t st_ = 1;
      bool in = false;
      for (int a = (int)grp.size() - 1; a >= 0; --a) {
        if (grp[a] == v) {
          in = true;
          break;
        }
        st_ *= p->cards[grp[a]];
      }
      return in ? st_ : 0;
    };
    for (size_t a = 0; a < C.size(); ++a) {
      ci[a] = lin(I, C[a]);
      ck[a] = lin(K, C[a]);
      cs[a] = lin(S, C[a]);
    }
    const double* src = st->h_base.data() + st->boff[ps.clique];
    const int64_t n = p->csize[ps.clique];
    std::vector<int> dig(C.size(), 0);
    int64_t xi = 0, xk = 0, xs = 0;
    double* W = hp.w.data() + w0;
    for (int64_t e = 0; e < n; ++e) {
      W[(xi * nK + xk) * nSp + xs] += src[e];
      for (int a = (int)C.size() - 1; a >= 0; --a) {
        xi += ci[a];
        xk += ck[a];
        xs += cs[a];
        if (++dig[a] < p->cards[C[a]]) break;
        const int64_t c = p->cards[C[a]];
        xi -= ci[a] * c;
        xk -= ck[a] * c;
        xs -= cs[a] * c;
        dig[a] = 0;
      }
    }
  }
  std::memset(&cp, 0, sizeof(cp));
  cp.w_off = w0;
  cp.ti_off = (int64_t)hp.ctab.size();
  for (int64_t i = 0; i < nI; ++i) {
    for (int g = 0; g < nG; ++g) hp.ctab.push_back((int32_t)gI[g][i]);
    for (int e = 0; e < nE; ++e) hp.ctab.push_back((int32_t)eI[e][i]);
    hp.ctab.push_back((int32_t)oI[i]);
    if (ps_b) {
      for (int e = 0; e < nEb; ++e) hp.ctab.push_back((int32_t)ebI[e][i]);
      hp.ctab.push_back((int32_t)obI[i]);
    }
    for (int q = 0; q < nV; ++q) hp.ctab.push_back((int32_t)vI[q][i]);
  }
  cp.tk_off = (int64_t)hp.ctab.size();
  for (int64_t k = 0; k < nK; ++k)
    for (int g = 0; g < nG; ++g) hp.ctab.push_back((int32_t)gK[g][k]);
  cp.ts_off = (int64_t)hp.ctab.size();
  for (int64_t x = 0; x < nS; ++x) {
    for (int e = 0; e < nE; ++e) hp.ctab.push_back((int32_t)eS[e][x]);
    hp.ctab.push_back((int32_t)oS[x]);
    if (ps_b) {
      for (int e = 0; e < nEb; ++e) hp.ctab.push_back((int32_t)ebS[e][x]);
      hp.ctab.push_back((int32_t)obS[x]);
    }
  }
  cp.nI = (int)nI;
  cp.nS = (int)nS;
  cp.nK = (int)nK;
  cp.nG = nG;
  cp.nE = nE;
  cp.rowi = rowi ? 1 : 0;
  const int trows = rowi ? 1 : TMC;  // rowi: one i per unit
  cp.nT = rowi ? (int)((nI + trows - 1) / trows) : (int)((nS + trows - 1) / trows);
  {
    const int cvec = st->esz == 4 ? 4 : 2;  // case lanes per vector of the kernels
    cp.nBC = (int)((B + 32 * cvec - 1) / (32 * cvec));
  }
  // a unit walks a share of the case chunks of its (i, row tile): all of them for
  // short sums (amortises the unit's setup), one per unit for long ones (parallelism)
  {
    static const int ncg_small = env_int("JT_NCG_SMALL", CON_NCG_SMALL);
    static const int ncg_mid = env_int("JT_NCG_MID", CON_NCG_MID);
    static const int ncg_long = env_int("JT_NCG_LONG", 1 << 30);
    cp.nCG = nK >= 32 ? std::min(ncg_long, cp.nBC) : nK >= 8 ? std::min(ncg_mid, cp.nBC) : std::min(ncg_small, cp.nBC);
    // bit 0: rowi passes, bit 1: tile passes (default: rowi chunk-major, measured +2-6%)
    const int cmaj = env_int("JT_CMAJ", 1);
    cp.cmaj = (cmaj >> (rowi ? 0 : 1)) & 1;
  }
  cp.nKS = 1;
  cp.kch = (int)nK;
  cp.n_units = (rowi ? 1 : nI) * cp.nT * cp.nCG;
  int64_t min_units = (int64_t)st->num_sms * 8;
  cp.igs = 1;
  // (opt-in, JT_ROWG=1: measured slower than plain row-per-i once paired passes and
  // evict-first epilogue streams cut the re-reads it was built against)
  if (rowi && !I.empty() && nV == 0 && env_int("JT_ROWG", 0)) {
    // i-groups: the innermost i variable's values share every factor that does not
    // index it; group them into one warp unit when those shared factors dominate
    const int v = I.back();
    const int igs = p->cards[v];
    double shared = 0.0, own = 0.0;
    int gst[CMAXG] = {0};
    for (int g = 0; g < nG; ++g) {
      double n = (double)B;
      for (int x : G[g]->vars) n *= p->cards[x];
      gst[g] = (int)tensor_stride(p, *G[g], v, B);
      (gst[g] == 0 ? shared : own) += n;
    }
    const int64_t units = (nI / igs) * (int64_t)cp.nCG;
    static const int igs_max = env_int("JT_ROWG_MAX", 8);
    if (igs >= 2 && igs <= igs_max && nI % igs == 0 && shared > own && units >= min_units) {
      cp.rowi = igs <= 4 ? 2 : 3;
      cp.igs = igs;
      for (int g = 0; g < nG; ++g) cp.gstride[g] = gst[g];
      cp.n_units = units;
    }
  }
  // (the K-split combine is a warp collective: every lane must own cases, so B
  // must fill whole case chunks; otherwise the pass takes the general kernels)
  const int kvec = st->esz == 4 ? 4 : 2;
  if (!rowi && cp.n_units < min_units && nK >= 256 && B % (32 * kvec) == 0) {
    // long sums with few units (posteriors of a clique-private variable): split K
    // into chunks of >= 64 k so every warp has work; partials combined in order
    const int vec = st->esz == 4 ? 4 : 2;
    cp.nBC = (int)((B + 32 * vec - 1) / (32 * vec));
    cp.nCG = cp.nBC;  // one case chunk per unit: the combine group is (i, t, chunk)
    const int64_t base_units = nI * cp.nT * cp.nCG;
    int64_t nks = std::min<int64_t>((min_units * 4 + base_units - 1) / base_units, (nK + 63) / 64);
    nks = std::max<int64_t>(2, nks);
    cp.kch = (int)((nK + nks - 1) / nks);
    cp.nKS = (int)((nK + cp.kch - 1) / cp.kch);
    cp.n_units = base_units * cp.nKS;
    const int64_t groups = base_units;
    cp.part_off = hp.n_part;
    hp.n_part += groups * cp.nKS * (int64_t)TMC * 32 * vec;
    cp.cnt_off = hp.n_cnt;
    hp.n_cnt += groups;
  }
  // too few units: first split the case chunks finer (more units of fewer chunks,
  // e.g. leaf messages with short sums over a few thousand separator rows)
  while (cp.nKS == 1 && cp.n_units < min_units && cp.nCG < cp.nBC) {
    cp.nCG = std::min(cp.nBC, cp.nCG * 2);
    cp.n_units = (rowi ? 1 : nI) * cp.nT * cp.nCG;
  }
  // still too few (e.g. a posterior over a long factor row): the chunked
  // thread-owned/general passes parallelise over the clique instead
  if (cp.n_units < min_units) {
    hp.w.resize(w0);
    hp.ctab.resize(cp.ti_off);
    return JT_ERR_UNSUPPORTED;
  }
  cp.out_kind = kind_of(ps);
  cp.out_off = ps.out.off;
  cp.ratio_off = ps.ratio_off;
  cp.out2_off = ps.skip_out2 && ps.out_kind == OUT_SEP_DFRESH ? OUT2_SKIP : ps.out2_off;
  for (int g = 0; g < nG; ++g) cp.gfac_off[g] = G[g]->off;
  for (int e = 0; e < nE; ++e) cp.efac_off[e] = E[e]->off;
  cp.out_kind_b = OUT_NONE;
  cp.x_off = -1;
  // long K sums on the row-per-i kernel: several k in flight per lane (rowi code 4);
  // fp64 only (fp32 long sums fold, at two k per step already; measured -2% with it)
  const int longk = env_int("JT_ROWI_LONGK", st->esz == 8 ? 16 : 0);
  if (cp.rowi == 1 && longk > 0 && nK >= longk) cp.rowi = 4;
  if (ps_b) {
    cp.igs = 1;  // the paired epilogue lives in the plain row-per-i kernel
    cp.rowi = cp.rowi == 4 ? 4 : 1;
    cp.n_units = cp.nT * cp.nCG;
    cp.out_kind_b = kind_of(*ps_b);
    cp.nE_b = nEb;
    cp.out_off_b = ps_b->out.off;
    cp.ratio_off_b = ps_b->ratio_off;
    cp.out2_off_b = ps_b->skip_out2 && ps_b->out_kind == OUT_SEP_DFRESH ? OUT2_SKIP : ps_b->out2_off;
    for (int e = 0; e < nEb; ++e) cp.efac_off_b[e] = Eb[e]->off;
    cp.x_off = ps.x_off;
  }
  if (ps.x_off >= 0 && (!ps_b || cp.rowi != 1 || cp.out_kind != OUT_SEP_DFRESH)) {
    hp.w.resize(w0);
    hp.ctab.resize(cp.ti_off);
    return JT_ERR_UNSUPPORTED;  // X is written by the paired short-K row-per-i epilogue only
  }
  cp.nV = nV;
  for (int e = 0; e < MAXF; ++e) {
    cp.e_v[e] = e < nE ? e_v[e] : (int8_t)-1;
    cp.e_v_b[e] = e < nEb ? e_v_b[e] : (int8_t)-1;
  }
  cp.old_v = old_v;
  cp.old_v_b = old_v_b;
  for (int q = 0; q < nV; ++q) {
    int rc = virtual_sep(st, *V[q], hp, cp.vd[q]);
    if (rc != JT_OK) {
      for (auto it = hp.vdesc.begin(); it != hp.vdesc.end();)  // built by this call: rolled back below
        it = it->second.w_off >= w0 ? hp.vdesc.erase(it) : std::next(it);
      (void)0;
      hp.w.resize(w0);
      hp.ctab.resize(cp.ti_off);
      return rc;
    }
  }
  return JT_OK;
}

// Disjointness check of one program (the device analogue of the reference's
// ParallelEngine(validate=True), propagate.py:135-140): within a wave no two
// passes write the same tensor element, and no pass reads what another pass of
// the same wave writes.  Runs at every program build (host only, O(passes^2)).
static int validate_waves(const jt_state* st, const std::vector<std::vector<PassSpec>>& waves) {
  const jt_plan* p = st->plan;
  struct Iv { int arena; int64_t lo, hi; };
  auto tsize = [&](const Tensor& t) {
    int64_t n = t.batch ? st->B : 1;
    for (int v : t.vars) n *= p->cards[v];
    return n;
  };
  auto overlap = [](const Iv& a, const Iv& b) { return a.arena == b.arena && a.lo < b.hi && b.lo < a.hi; };
  for (const auto& w : waves) {
    std::vector<std::vector<Iv>> wr(w.size()), rd(w.size());
    for (size_t i = 0; i < w.size(); ++i) {
      const PassSpec& ps = w[i];
      const int64_t csz = p->csize[ps.clique] * (st->mode == JT_MATERIALIZED ? st->B : 1);
      if (ps.write) wr[i].push_back({A_CLIQUE, st->coff[ps.clique], st->coff[ps.clique] + csz});
      if (ps.src_arena == A_AUX) {
        Tensor t;
        t.vars = ps.scope;
        t.batch = st->B > 1;
        rd[i].push_back({A_AUX, ps.src_off, ps.src_off + tsize(t)});
      } else if (ps.src_arena == A_CLIQUE) {
        rd[i].push_back({A_CLIQUE, st->coff[ps.clique], st->coff[ps.clique] + csz});
      }
      for (const auto& f : ps.factors) rd[i].push_back({A_AUX, f.off, f.off + tsize(f)});
      if (ps.out_kind == OUT_RAW) {
        wr[i].push_back({-1, ps.out.off, ps.out.off + tsize(ps.out)});
      } else if (ps.out_kind != OUT_NONE) {
        const int64_t n = tsize(ps.out);
        if (ps.out_kind == OUT_SEP_FRESH) {
          wr[i].push_back({A_AUX, ps.out.off, ps.out.off + n});
        } else {
          rd[i].push_back({A_AUX, ps.out.off, ps.out.off + n});
          if (ps.out2_off < 0) wr[i].push_back({A_AUX, ps.out.off, ps.out.off + n});
          else wr[i].push_back({A_AUX, ps.out2_off, ps.out2_off + n});
          wr[i].push_back({A_AUX, ps.ratio_off, ps.ratio_off + n});
        }
      }
    }
    for (size_t i = 0; i < w.size(); ++i)
      for (size_t j = 0; j < w.size(); ++j) {
        if (i == j) continue;
        for (const Iv& a : wr[i]) {
          for (const Iv& b : rd[j])
            if (overlap(a, b)) return JT_ERR_BAD_ARG;
          if (j > i)
            for (const Iv& b : wr[j])
              if (overlap(a, b)) return JT_ERR_BAD_ARG;
        }
      }
  }
  return JT_OK;
}

// Sibling passes of one wave that may share a K-sum (compile_contract with a
// second output): same clique, same output scope, both contraction passes.
static std::vector<int> pair_specs(const jt_state* st, const std::vector<PassSpec>& w) {
  std::vector<int> partner(w.size(), -1);
  if (!env_int("JT_PAIR", 1)) return partner;
  for (size_t a = 0; a < w.size(); ++a) {
    if (partner[a] >= 0 || !contract_eligible(st, w[a]) || w[a].out_kind == OUT_RAW) continue;
    for (size_t b = a + 1; b < w.size(); ++b) {
      if (partner[b] >= 0 || !contract_eligible(st, w[b]) || w[b].out_kind == OUT_RAW) continue;
      if (w[b].clique != w[a].clique || w[b].out.vars != w[a].out.vars) continue;
      partner[a] = (int)b;
      partner[b] = (int)a;
      break;
    }
  }
  return partner;
}

static int compile_program(const jt_state* st, const std::vector<std::vector<PassSpec>>& waves, HostProgram& hp,
                           int occ_override = 0, const std::vector<std::vector<char>>* skip = nullptr) {
  auto& passes = hp.passes;
  auto& items = hp.items;
  auto& blk = hp.blk;
  auto& bins = hp.bins;
  int64_t& n_part = hp.n_part;
  int64_t& n_cnt = hp.n_cnt;
  for (size_t wix = 0; wix < waves.size(); ++wix) {
    const auto& w = waves[wix];
    if (w.empty()) continue;
    auto skipped = [&](size_t q) { return skip && !(*skip)[wix].empty() && (*skip)[wix][q]; };
    WaveRt rt;
    rt.pass_base = (int64_t)passes.size();
    rt.item_base = (int64_t)items.size();
    // launch groups of the wave: (kind, vec, lm, m) -> items, in first-seen order
    std::vector<std::pair<std::array<int, 4>, std::vector<Item>>> grp;
    // launch-bound (small) waves: one vector width and no row kernel, so the
    // wave is one or two launches; big waves give every pass its own best kernel
    int64_t wave_el = 0;
    int wave_vec = st->esz == 4 ? 4 : 2;
    for (auto& ps : w) {
      const auto dd = pass_dims(st, ps);
      int64_t n = 1;
      for (auto& x : dd) n *= x.card;
      wave_el += n;
      wave_vec = std::min(wave_vec, pass_max_vec(st, ps));
    }
    const bool small_wave = wave_el < SMALL_WAVE_ELEMS;
    // contraction passes, split by accumulator kind (fp32 sums over > CKF terms fold into fp64)
    // contraction launch groups keyed by (fold, rowi, nG): fold = fp32 sums over > CKF
    // terms fold into fp64; nG is a compile-time parameter of the tile kernel
    constexpr int NGK = CMAXG + 1;
    std::vector<CPass> cps[10 * NGK];
    std::vector<int> cpc[10 * NGK];
    // row-per-i siblings sharing a K-sum (same clique, output scope and G factors,
    // e.g. distribute messages to children over equal separators) become ONE pass
    // with two epilogues: the shared factor rows stream once
    std::vector<int> partner = pair_specs(st, w);
    for (size_t wi = 0; wi < w.size(); ++wi) {
      const PassSpec& ps = w[wi];
      if (has_virtual(ps)) {  // virtual separators: row-per-i contraction passes only
        bool ok = contract_eligible(st, ps) && !skipped(wi);
        if (!ok) return JT_ERR_UNSUPPORTED;
      }
      if (skipped(wi)) continue;  // a tiny pass (jt_tiny.cu)
      // the clique product X is written only by a paired contraction pass
      if (ps.x_off >= 0 && (!contract_eligible(st, ps) || partner[wi] < 0)) return JT_ERR_UNSUPPORTED;
      if (partner[wi] >= 0 && partner[wi] < (int)wi) continue;  // compiled with its partner
      if (contract_eligible(st, ps)) {
        CPass cp;
        bool paired = false;
        if (partner[wi] >= 0) {
          const size_t n_w = hp.w.size(), n_t = hp.ctab.size();
          paired = compile_contract(st, ps, hp, cp, &w[partner[wi]]) == JT_OK;
          if (!paired && ps.x_off >= 0) return JT_ERR_UNSUPPORTED;  // caller rebuilds without X
          if (!paired) {  // fall back to two separate passes
            hp.w.resize(n_w);
            hp.ctab.resize(n_t);
            partner[partner[wi]] = -1;
          }
        }
        if (!paired && ps.x_off >= 0) return JT_ERR_UNSUPPORTED;
        if (paired || compile_contract(st, ps, hp, cp) == JT_OK) {
          if (cp.nV > 0 && !(cp.rowi == 1 || cp.rowi == 4)) return JT_ERR_UNSUPPORTED;
          const int key = ((st->esz == 4 && cp.nK > CKF ? 1 : 0) + 2 * cp.rowi) * NGK + (cp.rowi ? 0 : cp.nG);
          cps[key].push_back(cp);
          cpc[key].push_back(ps.clique);
          continue;
        }
      }
      if (has_virtual(ps)) return JT_ERR_UNSUPPORTED;  // caller rebuilds without virtual separators
      BuiltPass bp;
      const int local = (int)(passes.size() - rt.pass_base);
      const int vec = small_wave ? wave_vec : pass_max_vec(st, ps);
      // single trees, small (latency-bound) waves or scalar passes: the general kernel
      // at 2 vectors per thread, 3 CTAs per SM (more warps in flight)
      static const bool no_row = getenv("JT_NO_ROW") != nullptr, no_own = getenv("JT_NO_OWN") != nullptr;
      // single trees: 2 vectors per thread (3 CTAs/SM, more warps in flight) unless the pass
      // streams a clique above 2^23 elements from HBM (c3), where 4 per thread measure better
      // (c4B 0.73 -> 0.66 ms, c5 0.32 -> 0.30 ms fp32; c3 keeps 0.24)
      static const int single_kv = env_int("JT_SINGLE_KV", 0);  // > 0: forced for every single-tree pass
      int64_t pass_el = 1;
      for (auto& x : pass_dims(st, ps)) pass_el *= x.card;
      const int kv = st->B == 1 && single_kv > 0 ? single_kv
                   : st->B == 1 && (small_wave || vec == 1 || pass_el <= (int64_t(1) << 23)) ? 2 : KV;
      int rc = compile_pass(st, ps, vec, local, bp, !small_wave && !no_row, kv, !no_own);
      if (rc != JT_OK) return rc;
      bp.d.blk_off = (int64_t)blk.size();
      bp.d.blk32_off = (int64_t)hp.blk32.size();
      hp.blk32.insert(hp.blk32.end(), bp.blk32.begin(), bp.blk32.end());
      if (bp.d.own || bp.d.row) bp.blk.clear();  // these kernels read only the int32 table
      bp.d.bin_off = (int64_t)bins.size();
      bp.d.row_tab_off = (int64_t)hp.rowtab.size();
      hp.rowtab.insert(hp.rowtab.end(), bp.rowtab.begin(), bp.rowtab.end());
      bp.d.part_off = n_part;
      bp.d.cnt_off = n_cnt;
      blk.insert(blk.end(), bp.blk.begin(), bp.blk.end());
      bins.insert(bins.end(), bp.bins.begin(), bp.bins.end());
      n_part += bp.n_part;
      n_cnt += bp.n_cnt;
      passes.push_back(bp.d);
      hp.pass_clique.push_back(ps.clique);
      std::array<int, 4> key{bp.d.row ? 2 : 0, vec, bp.d.row ? bp.d.row_lin : 0, bp.d.row ? 1 : bp.d.kv};
      if (bp.d.own) {
        const bool allf = bp.d.fac_vec == ((1u << bp.d.nf) - 1u);
        const bool full_vec = vec == (st->esz == 4 ? 4 : 2);
        const int lm = full_vec && allf && !getenv("JT_OWN_LM0") ? (bp.d.src_vec ? 2 : 1) : 0;
        if (lm == 0 && bp.d.own_m != 1) return JT_ERR_UNSUPPORTED;
        key = {1, vec, lm, bp.d.own_m};
      }
      auto it = std::find_if(grp.begin(), grp.end(), [&](const auto& g) { return g.first == key; });
      if (it == grp.end()) {
        grp.push_back({key, {}});
        it = grp.end() - 1;
      }
      it->second.insert(it->second.end(), bp.items.begin(), bp.items.end());
    }
    for (auto& g : grp) {
      LaunchGrp lg;
      lg.kind = g.first[0];
      lg.vec = g.first[1];
      lg.lm = g.first[2];
      lg.m = g.first[3];
      int occ = occ_override;
      if (!occ) {
        const int dt = st->plan->dtype;
        occ = lg.kind == 1 ? wave_own_max_ctas_per_sm(dt, lg.vec)
            : lg.kind == 2 ? wave_row_max_ctas_per_sm(dt, lg.vec) : wave_max_ctas_per_sm(dt, lg.vec, lg.m);
      }
      lg.n_items = (int)g.second.size();
      lg.item_off = (int64_t)items.size() - rt.item_base;
      lg.grid = (int)std::min<int64_t>(lg.n_items, (int64_t)occ * st->num_sms);
      if (lg.kind == 2)  // warp units: enough CTAs for every unit to have a warp, up to full occupancy
        lg.grid = (int)std::min<int64_t>((lg.n_items + NT / 32 - 1) / (NT / 32), (int64_t)occ * st->num_sms);
      items.insert(items.end(), g.second.begin(), g.second.end());
      rt.groups.push_back(lg);
    }
    // JT_SPLIT_CPASS=1: one launch per contraction pass (also what an ncu launch
    // list needs to attribute time and DRAM bytes to single passes)
    // (default: the measured program is 2-8% faster with the passes
    // as separate parallel graph branches)
    if (env_int("JT_SPLIT_CPASS", 1)) {
      std::vector<CPass> cps2[10 * NGK];
      std::vector<int> cpc2[10 * NGK];
      for (int key = 0; key < 10 * NGK; ++key) {
        cps2[key].swap(cps[key]);
        cpc2[key].swap(cpc[key]);
      }
      for (int key = 0; key < 10 * NGK; ++key)
        for (size_t q = 0; q < cps2[key].size(); ++q) {
          const int fold = (key / NGK) & 1;
          LaunchGrp cg;
          cg.kind = 3;
          cg.lm = fold;
          cg.m = (key / NGK) >> 1;
          cg.vec = key % NGK;
          cg.cpass_off = (int64_t)hp.cpasses.size();
          CPass cp = cps2[key][q];
          cp.unit0 = 0;
          cg.n_units = cp.n_units;
          cg.n_cpasses = 1;
          hp.cpasses.push_back(cp);
          // row-per-i pass: descriptor and tables in the kernel parameters (constant bank)
          const int tsw = cp.nE + 1 + (cp.out_kind_b != OUT_NONE ? cp.nE_b + 1 : 0);
          if (cp.x_off >= 0 && !((cp.rowi == 1) && cp.nK * cp.nG <= RP_TK && tsw <= RP_TS))
            return JT_ERR_UNSUPPORTED;  // X needs the parameter-space row-per-i kernel
          if ((cp.rowi == 1 || cp.rowi == 4) && cp.nK * cp.nG <= RP_TK && tsw <= RP_TS &&
              (env_int("JT_ROWI_PARAM", 1) || cp.x_off >= 0)) {
            RowiParam rp;
            std::memset(&rp, 0, sizeof(rp));
            rp.cp = cp;
            for (int x = 0; x < cp.nK * cp.nG; ++x) rp.tk[x] = hp.ctab[cp.tk_off + x];
            for (int x = 0; x < tsw; ++x) rp.ts[x] = hp.ctab[cp.ts_off + x];
            cg.rp_idx = (int)hp.rparams.size();
            cg.xw = cp.x_off >= 0 ? 1 : 0;
            hp.rparams.push_back(rp);
          }
          const int64_t tsn = (int64_t)cp.nS * (cp.nE + 1);
          if (cp.rowi == 0 && cp.nK * cp.nG <= RP_TK && tsn <= TP_TS && env_int("JT_TILE_PARAM", 1)) {
            TileParam tpm;
            std::memset(&tpm, 0, sizeof(tpm));
            tpm.cp = cp;
            for (int x = 0; x < cp.nK * cp.nG; ++x) tpm.tk[x] = hp.ctab[cp.tk_off + x];
            for (int64_t x = 0; x < tsn; ++x) tpm.ts[x] = hp.ctab[cp.ts_off + x];
            cg.tp_idx = (int)hp.tparams.size();
            hp.tparams.push_back(tpm);
          }
          hp.cpass_clique.push_back(cpc2[key][q]);
          cg.vs = cp.nV > 0;
          const int occ = occ_override ? occ_override
                          : cg.rp_idx >= 0
                              ? contract_rowi_param_max_ctas(st->plan->dtype, fold, cg.m == 4, cp.nG, cg.xw != 0, cg.vs,
                                                             cp.out_kind, cp.out_kind_b)
                              : contract_max_ctas_per_sm(st->plan->dtype, fold, cg.m, cg.vec);
          cg.grid = (int)std::min<int64_t>((cg.n_units + NT / 32 - 1) / (NT / 32), (int64_t)occ * st->num_sms);
          rt.groups.push_back(cg);
        }
    }
    for (int key = 0; key < 10 * NGK; ++key) {
      const int fold = (key / NGK) & 1;
      if (cps[key].empty()) continue;
      for (auto& x : cps[key])
        if (x.x_off >= 0) return JT_ERR_UNSUPPORTED;  // X needs one pass per launch
      LaunchGrp cg;
      cg.kind = 3;
      cg.lm = fold;
      cg.m = (key / NGK) >> 1;
      cg.vec = key % NGK;
      cg.cpass_off = (int64_t)hp.cpasses.size();
      for (size_t q = 0; q < cps[key].size(); ++q) {
        CPass cp = cps[key][q];
        cp.unit0 = cg.n_units;
        cg.n_units += cp.n_units;
        cg.n_cpasses++;
        cg.vs |= cp.nV > 0;
        hp.cpasses.push_back(cp);
        hp.cpass_clique.push_back(cpc[key][q]);
      }
      // passes of one clique with equal unit counts (e.g. the distribute messages to
      // children with equal separators) read the same factor tensors: interleave their
      // units so the second reader finds them in L1/L2
      if (cps[key].size() > 1 && !getenv("JT_NO_INTERLEAVE")) {
        bool same = true;
        for (size_t q = 1; q < cps[key].size(); ++q)
          same = same && cps[key][q].n_units == cps[key][0].n_units && cpc[key][q] == cpc[key][0];
        cg.interleave = same ? 1 : 0;
      }
      const int occ = occ_override ? occ_override : contract_max_ctas_per_sm(st->plan->dtype, fold, cg.m, cg.vec);
      cg.grid = (int)std::min<int64_t>((cg.n_units + NT / 32 - 1) / (NT / 32), (int64_t)occ * st->num_sms);
      rt.groups.push_back(cg);
    }
    rt.n_items = (int)(items.size() - rt.item_base);
    hp.waves.push_back(rt);
  }
  return JT_OK;
}

// Small waves of single trees run as tiny-pass launches (jt_tiny.cu): their
// work is a few thousand entries, latency-bound, and the general kernel's
// per-item block tables and smem epilogues dominate.  JT_TINY=2 (default):
// per wave, a tiny launch when the wave touches at most 2^JT_TINY_WAVE_LOG2
// elements, else the general launch groups (PDL chains every launch, the
// program is graph-replayed); JT_TINY=1: the whole program as ONE cooperative
// launch with grid barriers (every wave small); JT_TINY=0: off.
#ifndef TINY_MAX_LOG2
#define TINY_MAX_LOG2 22
#endif
#ifndef TINY_WAVE_LOG2
#define TINY_WAVE_LOG2 18
#endif
#ifndef TINY_ROW_MAX
#define TINY_ROW_MAX 0
#endif
static int tiny_mode() { return env_int("JT_TINY", 2); }

// Row shape of a pass as a tiny pass: output entries x row length (merged dims).
static void tiny_shape(const jt_state* st, const PassSpec& ps, int64_t& n_out, int64_t& n_rest) {
  const std::vector<Dim> dims = merge_dims(pass_dims(st, ps), (int)ps.factors.size());
  n_out = n_rest = 1;
  for (const Dim& d : dims) ((ps.out_kind == OUT_NONE || d.out != 0) ? n_out : n_rest) *= d.card;
}

// Per wave and pass: run as a tiny pass?  Mode 2: every pass of a wave touching
// at most 2^JT_TINY_WAVE_LOG2 elements, and (JT_TINY_ROW_MAX > 0) any pass whose
// rows are at most that long; mode 1: all passes when every wave is small.
static bool tiny_masks(const jt_state* st, const std::vector<std::vector<PassSpec>>& waves,
                       std::vector<std::vector<char>>& mask) {
  mask.assign(waves.size(), {});
  const int mode = tiny_mode();
  if (st->B != 1 || st->mode != JT_MATERIALIZED || mode == 0) return false;
  static const int lg = env_int("JT_TINY_MAX_LOG2", TINY_MAX_LOG2);
  static const int lgw = env_int("JT_TINY_WAVE_LOG2", TINY_WAVE_LOG2);
  static const int row_max = env_int("JT_TINY_ROW_MAX", TINY_ROW_MAX);
  int nw = 0, ntiny = 0;
  bool all_small = true;
  for (size_t wi = 0; wi < waves.size(); ++wi) {
    const auto& w = waves[wi];
    mask[wi].assign(w.size(), 0);
    if (w.empty()) continue;
    ++nw;
    int64_t el = 0;
    std::vector<int64_t> rows(w.size());
    for (size_t q = 0; q < w.size(); ++q) {
      int64_t no, nr;
      tiny_shape(st, w[q], no, nr);
      el += no * nr;
      rows[q] = nr;
    }
    all_small = all_small && el <= (int64_t(1) << lg);
    for (size_t q = 0; q < w.size(); ++q) {
      const bool t = mode == 1 || el <= (int64_t(1) << lgw) || (row_max > 0 && rows[q] <= row_max);
      mask[wi][q] = t ? 1 : 0;
      ntiny += t;
    }
  }
  if (mode == 1) {
    if (!(all_small && nw >= 3)) {
      for (auto& m : mask) std::fill(m.begin(), m.end(), 0);
      return false;
    }
    return true;
  }
  return ntiny > 0 && nw >= 2;
}

// q = (umulhi(n, mul) + n) >> shr == n / d for 0 <= n < 2^31 (round-up method)
static void fast_div(int64_t d, unsigned& mul, int& shr) {
  int l = 0;
  while ((int64_t(1) << l) < d) ++l;
  mul = (unsigned)(((uint64_t(1) << 32) * ((uint64_t(1) << l) - (uint64_t)d)) / (uint64_t)d + 1);
  shr = l;
}

// Tiny passes of a program: per pass, the merged dims split into output dims
// (those the output tensor indexes; every dim when there is no output) and row
// dims; one thread per output entry, one warp when the row is long.
static int build_tiny(const jt_state* st, const std::vector<std::vector<PassSpec>>& waves,
                      const std::vector<std::vector<char>>& mask, std::vector<TPass>& tp, std::vector<TinyWave>& tw) {
  auto fits = [](int64_t x) { return x >= INT32_MIN && x <= INT32_MAX; };
  for (size_t wi = 0; wi < waves.size(); ++wi) {
    const auto& w = waves[wi];
    if (w.empty()) continue;
    TinyWave wv{};
    wv.pass0 = (int64_t)tp.size();
    int64_t units = 0;
    for (size_t q = 0; q < w.size(); ++q) {
      if (!mask[wi][q]) continue;
      const PassSpec& ps = w[q];
      const int nf = (int)ps.factors.size();
      if (nf > MAXF || (ps.write && !ps.scope.empty())) return JT_ERR_UNSUPPORTED;
      const std::vector<Dim> dims = merge_dims(pass_dims(st, ps), nf);
      const bool has_out = ps.out_kind != OUT_NONE;
      TPass P;
      std::memset(&P, 0, sizeof(P));
      P.src_arena = ps.src_arena;
      P.src_off = ps.src_arena == A_AUX ? ps.src_off : ps.src_arena == A_CLIQUE ? st->coff[ps.clique] : st->boff[ps.clique];
      P.dst_off = ps.write ? st->coff[ps.clique] : -1;
      P.nf = nf;
      for (int f = 0; f < nf; ++f) P.fac_off[f] = ps.factors[f].off;
      P.out_kind = ps.out_kind;
      P.out_off = has_out ? ps.out.off : 0;
      P.ratio_off = ps.ratio_off;
      P.out2_off = ps.out2_off;
      P.n_out = 1;
      P.n_rest = 1;
      for (const Dim& d : dims) {
        if (!fits(d.src) || !fits(d.dst) || !fits(d.out) || d.card > INT32_MAX) return JT_ERR_UNSUPPORTED;
        for (int f = 0; f < nf; ++f)
          if (!fits(d.fac[f])) return JT_ERR_UNSUPPORTED;
        if (!has_out || d.out != 0) {
          if (P.nod == TD) return JT_ERR_UNSUPPORTED;
          const int k = P.nod++;
          P.ocard[k] = (int)d.card;
          fast_div(d.card, P.omul[k], P.oshr[k]);
          P.osrc[k] = (int)d.src;
          P.odst[k] = (int)d.dst;
          P.oout[k] = (int)d.out;
          for (int f = 0; f < nf; ++f) P.ofac[f][k] = (int)d.fac[f];
          P.n_out *= d.card;
        } else {
          if (P.nrd == TD) return JT_ERR_UNSUPPORTED;
          const int k = P.nrd++;
          P.rcard[k] = (int)d.card;
          fast_div(d.card, P.rmul[k], P.rshr[k]);
          P.rsrc[k] = (int)d.src;
          P.rdst[k] = (int)d.dst;
          for (int f = 0; f < nf; ++f) P.rfac[f][k] = (int)d.fac[f];
          P.n_rest *= d.card;
        }
      }
      // lanes per output entry: rows split into lane chunks of <= 2 batches (jt_tiny.cu)
      if (P.n_out * 32 > INT32_MAX || P.n_rest > INT32_MAX) return JT_ERR_UNSUPPORTED;
      int G = 1;
      while (G < 32 && P.n_rest > (int64_t)G * 8) G *= 2;
      P.warp = G;
      P.unit0 = units;
      const int64_t nu = P.n_out * G;
      units += (nu + 31) / 32 * 32;
      tp.push_back(P);
    }
    wv.n_passes = (int)(tp.size() - wv.pass0);
    wv.n_threads = units;
    tw.push_back(wv);
  }
  return JT_OK;
}

static int build_program(jt_state* st, const std::vector<std::vector<PassSpec>>& waves,
                         std::unique_ptr<Program>& out) {
  HostProgram hp;
  int rc0 = validate_waves(st, waves);
  if (rc0) return rc0;
  std::vector<std::vector<char>> tmask;
  std::vector<TPass> tp;
  std::vector<TinyWave> tw;
  bool tiny = tiny_masks(st, waves, tmask);
  if (tiny && (build_tiny(st, waves, tmask, tp, tw) != JT_OK || tp.empty())) {
    tiny = false;
    tp.clear();
    tw.clear();
  }
  rc0 = compile_program(st, waves, hp, 0, tiny ? &tmask : nullptr);
  if (rc0) return rc0;
  auto prog = std::make_unique<Program>();
  for (auto& w : waves)
    for (auto& ps : w) {
      auto note = [&](const Tensor& t) {
        if (t.vclique >= 0 && std::find(prog->vsep_leaves.begin(), prog->vsep_leaves.end(), t.vclique) ==
                                  prog->vsep_leaves.end())
          prog->vsep_leaves.push_back(t.vclique);
      };
      note(ps.out);
      for (auto& f : ps.factors) note(f);
      if (ps.skip_out2 && ps.sep >= 0) prog->final_skip.push_back(ps.sep);
    }
  prog->waves = hp.waves;
  prog->rparams = hp.rparams;
  prog->tparams = hp.tparams;
  for (auto& w : hp.waves) prog->n_launches += (int64_t)w.groups.size();
  if (tiny) {
    {
      int occ = 1, nfm = 1;
      for (auto& x : tp) nfm = std::max(nfm, x.nf);
      TinyArgs dummy{};
      CK(launch_tiny(st->plan->dtype, nfm, dummy, 0, nullptr, &occ));
      prog->tiny_nfm = nfm;
      int64_t max_ctas = 1;
      for (auto& w : tw) max_ctas = std::max<int64_t>(max_ctas, (w.n_threads + NT - 1) / NT);
      prog->tiny = 1;
      prog->tiny_grid = (int)std::min<int64_t>(max_ctas, (int64_t)occ * st->num_sms);
      prog->n_twaves = (int)tw.size();
      prog->n_launches = 1;
      prog->tiny_waves_launch = tiny_mode() == 2;
      // every wave all tiny and within one cluster's threads: one cluster launch
      {
        // (opt-in, JT_TINY_CLUSTER=<ctas>: measured slower than per-wave launches on c1,
        // 39 vs 29 us -- fewer threads per wave lengthen each wave more than the
        // cluster barrier saves)
        static const int cmax = env_int("JT_TINY_CLUSTER", 0);
        bool all_tiny = tiny_mode() == 2 && cmax > 0;
        int64_t max_thr = 0;
        for (size_t w = 0; w < tw.size() && all_tiny; ++w) {
          all_tiny = hp.waves[w].groups.empty();
          max_thr = std::max(max_thr, tw[w].n_threads);
        }
        // one unit per thread: every wave must fit the cluster's threads
        if (all_tiny && max_thr <= (int64_t)cmax * NT) {
          prog->tiny_cluster = (int)std::min<int64_t>(cmax, std::max<int64_t>(1, (max_thr + NT - 1) / NT));
          prog->tiny_waves_launch = 0;
          prog->n_launches = 1;
        }
      }
      if (prog->tiny_waves_launch) {
        prog->n_launches = 0;
        for (size_t w = 0; w < tw.size(); ++w) {
          prog->tiny_wave_grid.push_back(
              (int)std::min<int64_t>((tw[w].n_threads + NT - 1) / NT, (int64_t)occ * st->num_sms));
          prog->tiny_w.push_back(tw[w].n_passes > 0 ? 1 : 0);
          prog->n_launches += (tw[w].n_passes > 0 ? 1 : 0) + (int64_t)hp.waves[w].groups.size();
        }
      }
      std::vector<int64_t> u0;
      for (auto& x : tp) u0.push_back(x.unit0);
      CK(cudaMalloc(&prog->d_unit0, u0.size() * sizeof(int64_t)));
      CK(cudaMemcpy(prog->d_unit0, u0.data(), u0.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
      CK(cudaMalloc(&prog->d_tpass, tp.size() * sizeof(TPass)));
      CK(cudaMemcpy(prog->d_tpass, tp.data(), tp.size() * sizeof(TPass), cudaMemcpyHostToDevice));
      CK(cudaMalloc(&prog->d_twaves, tw.size() * sizeof(TinyWave)));
      CK(cudaMemcpy(prog->d_twaves, tw.data(), tw.size() * sizeof(TinyWave), cudaMemcpyHostToDevice));
      CK(cudaMalloc(&prog->d_bar, 2 * sizeof(unsigned)));
      CK(cudaMemset(prog->d_bar, 0, 2 * sizeof(unsigned)));
    }
  }
  auto& passes = hp.passes;
  auto& items = hp.items;
  auto& blk = hp.blk;
  auto& bins = hp.bins;
  const int64_t n_part = hp.n_part, n_cnt = hp.n_cnt;
  auto up = [&](auto** dptr, const auto& vec) -> int {
    using E = typename std::decay_t<decltype(vec)>::value_type;
    const size_t n = std::max<size_t>(vec.size(), 1);
    CK(cudaMalloc((void**)dptr, n * sizeof(E)));
    if (!vec.empty()) CK(cudaMemcpy(*dptr, vec.data(), vec.size() * sizeof(E), cudaMemcpyHostToDevice));
    return JT_OK;
  };
  int rc;
  if ((rc = up(&prog->d_passes, passes))) return rc;
  if ((rc = up(&prog->d_items, items))) return rc;
  if ((rc = up(&prog->d_blk, blk))) return rc;
  if ((rc = up(&prog->d_bins, bins))) return rc;
  if ((rc = up(&prog->d_blk32, hp.blk32))) return rc;
  if ((rc = up(&prog->d_rowtab, hp.rowtab))) return rc;
  if ((rc = up(&prog->d_cpass, hp.cpasses))) return rc;
  if ((rc = up(&prog->d_ctab, hp.ctab))) return rc;
  if (!hp.vcode.empty()) {
    if ((rc = up(&prog->d_vtask, hp.vcode))) return rc;
    CK(cudaMalloc(&prog->d_vcode, hp.vcode.size() * st->B * sizeof(int32_t)));
    prog->n_vtask = (int)hp.vcode.size();
    prog->n_launches += 1;  // the mask-code launch (launch_program_waves)
  }
  {
    const size_t n = std::max<size_t>(hp.w.size(), 1);
    CK(cudaMalloc(&prog->d_w, n * st->esz));
    if (!hp.w.empty()) {
      if (st->esz == 8) {
        CK(cudaMemcpy(prog->d_w, hp.w.data(), hp.w.size() * 8, cudaMemcpyHostToDevice));
      } else {
        std::vector<float> wf(hp.w.begin(), hp.w.end());
        CK(cudaMemcpy(prog->d_w, wf.data(), wf.size() * 4, cudaMemcpyHostToDevice));
      }
    }
  }
  CK(cudaMalloc(&prog->d_part, std::max<int64_t>(n_part, 1) * sizeof(double)));
  CK(cudaMalloc(&prog->d_cnt, std::max<int64_t>(n_cnt, 1) * sizeof(int)));
  CK(cudaMemset(prog->d_cnt, 0, std::max<int64_t>(n_cnt, 1) * sizeof(int)));
  out = std::move(prog);
  return JT_OK;
}

static int launch_group(jt_state* st, const Program* pr, const WaveRt& w, const LaunchGrp& g, cudaStream_t s) {
  if (g.kind == 3) {
    CArgs c;
    c.w = pr->d_w;
    c.aux = st->d_aux;
    c.qout = st->d_qout;
    c.err = st->d_err;
    c.tab = pr->d_ctab;
    c.codes = pr->d_vcode;
    c.passes = pr->d_cpass + g.cpass_off;
    c.n_passes = g.n_cpasses;
    c.n_units = g.n_units;
    c.B = st->B;
    c.partials = pr->d_part;
    c.counters = pr->d_cnt;
    c.interleave = g.interleave;
    static const int stream_epi = env_int("JT_EPI_CS", 1);
    c.stream_epi = stream_epi;
    if (g.rp_idx >= 0)
      CK(launch_contract_rowi_param(st->plan->dtype, g.lm, g.m == 4, c, pr->rparams[g.rp_idx], g.grid, s, g.xw != 0,
                                    g.vs != 0));
    else if (g.tp_idx >= 0)
      CK(launch_contract_tile_param(st->plan->dtype, g.lm, g.vec, c, pr->tparams[g.tp_idx], g.grid, s));
    else
      CK(launch_contract(st->plan->dtype, g.lm, g.m, g.vec, c, g.grid, s, g.vs != 0));
    st->launches++;
    return JT_OK;
  }
  WaveArgs a;
  a.clique = st->d_clique;
  a.base = st->d_base;
  a.aux = st->d_aux;
  a.qout = st->d_qout;
  a.partials = pr->d_part;
  a.counters = pr->d_cnt;
  a.err = st->d_err;
  a.blk = pr->d_blk;
  a.blk32 = pr->d_blk32;
  a.bins = pr->d_bins;
  a.rowtab = pr->d_rowtab;
  a.passes = pr->d_passes + w.pass_base;
  a.items = pr->d_items + w.item_base + g.item_off;
  a.n_items = g.n_items;
  if (g.kind == 1) CK(launch_wave_own(st->plan->dtype, g.vec, g.lm, g.m, a, g.grid, s));
  else if (g.kind == 2) CK(launch_wave_row(st->plan->dtype, g.vec, g.lm, a, g.grid, s));
  else CK(launch_wave(st->plan->dtype, g.vec, g.m, a, g.grid, s));
  st->launches++;
  return JT_OK;
}

static int ensure_side(jt_state* st) {
  if (st->ev_fork) return JT_OK;
  for (int i = 0; i < jt_state::N_SIDE; ++i) {
    CK(cudaStreamCreateWithFlags(&st->side[i], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&st->ev_join[i], cudaEventDisableTiming));
  }
  CK(cudaEventCreateWithFlags(&st->ev_fork, cudaEventDisableTiming));
  return JT_OK;
}

static int launch_program_waves(jt_state* st, Program* pr, cudaStream_t s) {
  if (pr->n_vtask > 0) {  // virtual separators: the current evidence masks' codes
    CK(launch_ev_code(st->d_aux, st->plan->dtype, pr->d_vtask, pr->n_vtask, (int)st->B, pr->d_vcode, s));
    st->launches++;
  }
  TinyArgs ta{};
  if (pr->tiny && pr->tiny_waves_launch) {
    TinyArgs& a = ta;
    a.clique = st->d_clique;
    a.base = st->d_base;
    a.aux = st->d_aux;
    a.qout = st->d_qout;
    a.err = st->d_err;
    a.passes = pr->d_tpass;
    a.unit0s = pr->d_unit0;
    a.waves = pr->d_twaves;
    a.n_waves = pr->n_twaves;
    a.bar = pr->d_bar;
  }
  int wi = -1;
  for (auto& w : pr->waves) {
    ++wi;
    // the wave's tiny passes run as one more (independent) launch group
    const bool has_tiny = pr->tiny && pr->tiny_waves_launch && pr->tiny_w[wi];
    const int ng = (int)w.groups.size() + (has_tiny ? 1 : 0);
    auto launch_gi = [&](int gi, cudaStream_t gs) -> int {
      if (gi < (int)w.groups.size()) return launch_group(st, pr, w, w.groups[gi], gs);
      CK(launch_tiny_wave(st->plan->dtype, pr->tiny_nfm, ta, wi, pr->tiny_wave_grid[wi], gs));
      st->launches++;
      return JT_OK;
    };
    if (ng == 0) continue;
    if (ng == 1) {
      int rc = launch_gi(0, s);
      if (rc) return rc;
      continue;
    }
    // independent launch groups: fork onto side streams, join back into s
    int rc = ensure_side(st);
    if (rc) return rc;
    CK(cudaEventRecord(st->ev_fork, s));
    const int nside = std::min(ng - 1, (int)jt_state::N_SIDE);
    for (int i = 0; i < nside; ++i) CK(cudaStreamWaitEvent(st->side[i], st->ev_fork, 0));
    for (int gi = 0; gi < ng; ++gi) {
      cudaStream_t gs = gi == 0 ? s : st->side[(gi - 1) % jt_state::N_SIDE];
      if ((rc = launch_gi(gi, gs))) return rc;
    }
    for (int i = 0; i < nside; ++i) {
      CK(cudaEventRecord(st->ev_join[i], st->side[i]));
      CK(cudaStreamWaitEvent(s, st->ev_join[i], 0));
    }
  }
  return JT_OK;
}

// First run launches directly; from the second run on the wave sequence is
// replayed as a CUDA graph on that stream (launch-bound small trees).
static int run_program(jt_state* st, Program* pr, cudaStream_t s) {
  pr->runs++;
  if (pr->tiny && pr->tiny_waves_launch) {
    // per-wave launches: captured into a graph from the second run on (below)
  } else if (pr->tiny && pr->tiny_cluster) {
    TinyArgs a{};
    a.clique = st->d_clique;
    a.base = st->d_base;
    a.aux = st->d_aux;
    a.qout = st->d_qout;
    a.err = st->d_err;
    a.passes = pr->d_tpass;
    a.unit0s = pr->d_unit0;
    a.waves = pr->d_twaves;
    a.n_waves = pr->n_twaves;
    a.bar = pr->d_bar;
    CK(launch_tiny_cluster(st->plan->dtype, pr->tiny_nfm, a, pr->tiny_cluster, s));
    st->launches++;
    return JT_OK;
  } else if (pr->tiny) {
    TinyArgs a{};
    a.clique = st->d_clique;
    a.base = st->d_base;
    a.aux = st->d_aux;
    a.qout = st->d_qout;
    a.err = st->d_err;
    a.passes = pr->d_tpass;
    a.unit0s = pr->d_unit0;
    a.waves = pr->d_twaves;
    a.n_waves = pr->n_twaves;
    a.bar = pr->d_bar;
    CK(launch_tiny(st->plan->dtype, pr->tiny_nfm, a, pr->tiny_grid, s));
    st->launches++;
    return JT_OK;
  }
  if (pr->waves.size() <= 1 || pr->runs < 2) return launch_program_waves(st, pr, s);
  if (pr->gexec && pr->gstream == s) {
    CK(cudaGraphLaunch(pr->gexec, s));
    st->launches += pr->n_launches;
    return JT_OK;
  }
  cudaStreamCaptureStatus cs;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone || s == nullptr)
    return launch_program_waves(st, pr, s);
  cudaGraph_t graph;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  const int64_t before = st->launches;
  int rc = launch_program_waves(st, pr, s);
  cudaError_t ec = cudaStreamEndCapture(s, &graph);
  st->launches = before;
  if (rc != JT_OK) return rc;
  CK(ec);
  if (pr->gexec) cudaGraphExecDestroy(pr->gexec);
  pr->gexec = nullptr;
  CK(cudaGraphInstantiate(&pr->gexec, graph, 0));
  cudaGraphDestroy(graph);
  pr->gstream = s;
  CK(cudaGraphLaunch(pr->gexec, s));
  st->launches += pr->n_launches;
  return JT_OK;
}

// ------------------------------------------------------------ scheduler ----
static Tensor sep_tensor(const jt_state* st, int s, int64_t off) {
  Tensor t;
  t.arena = A_AUX;
  t.off = off;
  t.vars = st->plan->svars[s];
  t.batch = st->B > 1;
  return t;
}

static Tensor ev_tensor(const jt_state* st, int v) {
  Tensor t;
  t.arena = A_AUX;
  t.off = st->ev_off[v];
  t.vars = {v};
  t.batch = st->B > 1;
  return t;
}

static Tensor var_out_tensor(const jt_state* st, int v) {
  Tensor t;
  t.arena = -1;
  t.off = st->q_off[v];
  t.vars = {v};
  t.batch = st->B > 1;
  return t;
}

struct Orient {
  std::vector<int> parent, psep, depth, height;
  std::vector<std::vector<std::pair<int, int>>> children;  // (child, sep) ascending
  int max_depth = 0, max_height = 0;
};

static Orient orient(const jt_plan* p, const std::vector<int>& roots) {
  Orient o;
  const int n = p->n_cliques;
  o.parent.assign(n, -1);
  o.psep.assign(n, -1);
  o.depth.assign(n, 0);
  o.height.assign(n, 0);
  o.children.resize(n);
  std::vector<int> order;
  for (int r : roots) {
    std::vector<int> stack{r};
    o.parent[r] = -1;
    std::vector<char> seen(n, 0);
    seen[r] = 1;
    while (!stack.empty()) {
      const int c = stack.back();
      stack.pop_back();
      order.push_back(c);
      for (auto& nb : p->nbrs[c]) {
        if (nb.first == o.parent[c] && nb.second == o.psep[c]) continue;
        if (seen[nb.first]) continue;
        seen[nb.first] = 1;
        o.parent[nb.first] = c;
        o.psep[nb.first] = nb.second;
        o.depth[nb.first] = o.depth[c] + 1;
        o.children[c].push_back(nb);
        stack.push_back(nb.first);
      }
    }
  }
  for (auto it = order.rbegin(); it != order.rend(); ++it) {
    const int c = *it;
    if (o.parent[c] >= 0) o.height[o.parent[c]] = std::max(o.height[o.parent[c]], o.height[c] + 1);
  }
  for (int c = 0; c < n; ++c) {
    o.max_depth = std::max(o.max_depth, o.depth[c]);
    o.max_height = std::max(o.max_height, o.height[c]);
    std::sort(o.children[c].begin(), o.children[c].end());
  }
  return o;
}

// Hugin collect+distribute as waves of passes.  Lazy scheme: a clique is read
// (not written) in collect, with its children's collect ratios multiplied in
// on the fly; its final table = original × Π children ratios × parent ratio is
// written once in distribute.  Cliques with more factors than a pass carries
// absorb their children's ratios eagerly (in-place) during collect instead.
static int build_propagate_waves(jt_state* st, const std::vector<int>& roots, const std::vector<int>& qvars,
                                 std::vector<std::vector<PassSpec>>& waves, bool fresh, bool hub_x,
                                 std::vector<char>& vleaf, bool lazy_final) {
  const jt_plan* p = st->plan;
  const bool shared = st->mode == JT_SHARED_BASE;
  const int src_arena = shared ? A_BASE : A_CLIQUE;
  Orient o = orient(p, roots);
  const int n = p->n_cliques;
  std::vector<std::vector<int>> evs(n);  // active evidence vars per clique (shared mode)
  if (shared)
    for (int v = 0; v < p->n_vars; ++v)
      if (st->ev_clique[v] >= 0) evs[st->ev_clique[v]].push_back(v);
  std::vector<char> eager(n, 0);
  for (int c = 0; c < n; ++c) {
    const int nfac = (int)o.children[c].size() + (o.parent[c] >= 0 ? 1 : 0) + (int)evs[c].size();
    eager[c] = nfac > MAXF;
  }
  // virtual separators (fresh shared-base programs): a leaf's collect message over a
  // large separator is evaluated by its readers instead of stored (vleaf[c] requested
  // by the caller; kept when the leaf qualifies)
  vleaf.resize(n, 0);
  for (int c = 0; c < n; ++c) {
    if (!vleaf[c]) continue;
    bool ok = shared && fresh && o.children[c].empty() && o.parent[c] >= 0 && !eager[c] && !eager[o.parent[c]] &&
              evs[c].size() <= 1;
    if (ok && evs[c].size() == 1) {  // the gather form: evidence on the leaf's one private variable
      std::vector<int> K;
      const auto& sv = p->svars[o.psep[c]];
      std::set_difference(p->cvars[c].begin(), p->cvars[c].end(), sv.begin(), sv.end(), std::back_inserter(K));
      ok = K == std::vector<int>{evs[c][0]};
    }
    vleaf[c] = ok;
  }
  auto ev_list = [&](int c) {
    std::vector<Tensor> f;
    for (int v : evs[c]) f.push_back(ev_tensor(st, v));
    return f;
  };
  auto virt = [&](Tensor t, int c) {  // the collect message of leaf c (separator tensor t)
    if (vleaf[c]) {
      t.vclique = c;
      t.vfac = ev_list(c);
    }
    return t;
  };
  std::fill(eager.begin(), eager.end(), 0);
  std::vector<PassSpec> hub_init;  // shared-base hubs: per-case table = base x evidence
  std::vector<std::vector<PassSpec>> hub_init_more;
  for (int c = 0; c < n; ++c) {
    const int nfac = (int)o.children[c].size() + (o.parent[c] >= 0 ? 1 : 0) + (int)evs[c].size();
    if (nfac > MAXF) {
      if (shared && !st->hub[c]) return JT_ERR_UNSUPPORTED;
      eager[c] = 1;
      if (shared) {
        for (size_t i = 0; i == 0 || i < evs[c].size(); i += MAXF) {
          PassSpec ps;
          ps.clique = c;
          ps.src_arena = i == 0 ? A_BASE : A_CLIQUE;
          ps.write = true;
          for (size_t k = i; k < std::min(evs[c].size(), i + MAXF); ++k) ps.factors.push_back(ev_tensor(st, evs[c][k]));
          if (i == 0) hub_init.push_back(ps);
          else {
            if (hub_init_more.size() < i / MAXF) hub_init_more.resize(i / MAXF);
            hub_init_more[i / MAXF - 1].push_back(ps);
          }
        }
      }
    }
  }
  if (!hub_init.empty()) {
    waves.push_back(hub_init);
    for (auto& w : hub_init_more) waves.push_back(w);
  }
  // collect ratio of a child separator: fresh propagations keep it in the
  // separator table itself (old == 1 ⇒ ratio == new)
  auto ratC = [&](int sp) { return fresh ? sep_cur(st, sp) : sep_alt(st, sp); };
  const int c_kind = fresh ? OUT_SEP_FRESH : OUT_SEP;
  auto child_ratios = [&](int c) {
    std::vector<Tensor> f;
    for (auto& ch : o.children[c]) f.push_back(virt(sep_tensor(st, ch.second, ratC(ch.second)), ch.first));
    return f;
  };
  auto ev_factors = [&](int c) {
    std::vector<Tensor> f;
    for (int v : evs[c]) f.push_back(ev_tensor(st, v));
    return f;
  };
  // ---- collect: by height, leaves first ----
  for (int h = 0; h <= o.max_height; ++h) {
    std::vector<std::vector<PassSpec>> pre;  // absorb sub-waves for eager cliques
    std::vector<PassSpec> main;
    for (int c = 0; c < n; ++c) {
      if (o.height[c] != h) continue;
      const bool is_root = o.parent[c] < 0;
      if (is_root && !eager[c]) continue;
      std::vector<Tensor> cf = child_ratios(c);
      std::vector<Tensor> ef = ev_factors(c);
      if (eager[c]) {
        // absorb children ratios MAXF at a time, in place
        size_t i = 0;
        int sub = 0;
        const size_t last_chunk = is_root ? cf.size() : (cf.size() > 0 ? cf.size() - ((cf.size() - 1) % MAXF + 1) : 0);
        while (i < last_chunk) {
          PassSpec ps;
          ps.clique = c;
          ps.src_arena = A_CLIQUE;
          ps.write = true;
          for (size_t k = i; k < std::min(last_chunk, i + MAXF); ++k) ps.factors.push_back(cf[k]);
          i += ps.factors.size();
          if ((int)pre.size() <= sub) pre.resize(sub + 1);
          pre[sub++].push_back(ps);
        }
        if (!is_root) {
          PassSpec ps;
          ps.clique = c;
          ps.src_arena = A_CLIQUE;
          ps.write = true;
          for (size_t k = i; k < cf.size(); ++k) ps.factors.push_back(cf[k]);
          ps.out_kind = c_kind;
          ps.out = sep_tensor(st, o.psep[c], sep_cur(st, o.psep[c]));
          ps.ratio_off = sep_alt(st, o.psep[c]);
          main.push_back(ps);
        }
      } else if (!vleaf[c]) {  // (a virtual separator's producer is not run)
        PassSpec ps;
        ps.clique = c;
        ps.src_arena = src_arena;
        ps.factors = cf;
        ps.factors.insert(ps.factors.end(), ef.begin(), ef.end());
        ps.out_kind = c_kind;
        ps.out = sep_tensor(st, o.psep[c], sep_cur(st, o.psep[c]));
        ps.ratio_off = sep_alt(st, o.psep[c]);
        main.push_back(ps);
      }
    }
    for (auto& w : pre) waves.push_back(w);
    // roots absorb after their children's ratios exist: eager roots are at max height;
    // their absorb passes were queued in `pre` of their own height, which runs after
    // all lower heights — correct since every child has a lower height.
    waves.push_back(main);
  }
  // query assignment (fused queries, shared mode): a variable held by some
  // separator is read from the smallest such separator's final table (after
  // propagation every separator equals both adjacent clique marginals,
  // propagate.py:393-402), otherwise from its smallest clique with all factors
  std::vector<std::vector<int>> qby(n), qsep(p->n_seps);
  for (int v : qvars) {
    int bs = -1;
    if (shared)
      for (int sp = 0; sp < p->n_seps; ++sp)
        if (std::binary_search(p->svars[sp].begin(), p->svars[sp].end(), v))
          if (bs < 0 || p->ssize[sp] < p->ssize[bs]) bs = sp;
    if (bs >= 0) {
      qsep[bs].push_back(v);
      continue;
    }
    int best = -1;
    for (int c = 0; c < n; ++c)
      if (std::binary_search(p->cvars[c].begin(), p->cvars[c].end(), v))
        if (best < 0 || p->csize[c] < p->csize[best]) best = c;
    if (best < 0) return JT_ERR_BAD_ARG;
    qby[best].push_back(v);
  }
  // ---- distribute: by depth, root first ----
  // dwx[d]: passes of depth d that read a clique product X written at depth d
  std::vector<std::vector<PassSpec>> dw(o.max_depth + 3), dwx(o.max_depth + 3);
  std::vector<char> x_used(o.max_depth + 3, 0);
  for (int c = 0; c < n; ++c) {
    const int d = o.depth[c];
    const size_t dw0 = dw[d].size();
    std::vector<Tensor> fac;
    if (!eager[c]) fac = child_ratios(c);
    if (o.parent[c] >= 0) fac.push_back(sep_tensor(st, o.psep[c], st->ratD_off[o.psep[c]]));
    if (!eager[c]) {  // eager shared-base hubs took their evidence in at initialisation
      std::vector<Tensor> ef = ev_factors(c);
      fac.insert(fac.end(), ef.begin(), ef.end());
    }
    const auto& ch = o.children[c];
    for (size_t i = 0; i < ch.size(); ++i) {
      PassSpec ps;
      ps.clique = c;
      ps.src_arena = eager[c] ? A_CLIQUE : src_arena;
      ps.factors = fac;
      ps.write = !shared && ch.size() == 1;
      ps.out_kind = OUT_SEP;
      ps.out = sep_tensor(st, ch[i].second, sep_cur(st, ch[i].second));
      if (fresh) ps.out = virt(ps.out, ch[i].first);  // (ratC == sep_cur: the child's collect message)
      if (fresh) ps.out2_off = sep_alt(st, ch[i].second);
      ps.sep = ch[i].second;
      // (fused queries of this separator read its final table in this program)
      ps.skip_out2 = lazy_final && fresh && shared && qsep[ch[i].second].empty();
      ps.ratio_off = st->ratD_off[ch[i].second];
      if (fresh && !ps.write && !eager[c]) {
        // message to child k: product of the OTHER messages, marginalised
        // (new/old == Σ without k's own collect message)
        const int64_t own_off = ratC(ch[i].second);
        std::vector<Tensor> f2;
        for (auto& t : fac)
          if (!(t.off == own_off && t.vars == p->svars[ch[i].second])) f2.push_back(t);
        if (f2.size() + 1 == fac.size()) {
          ps.factors = f2;
          ps.out_kind = OUT_SEP_DFRESH;
        }
      }
      dw[d].push_back(ps);
    }
    if (!shared && ch.size() != 1 && !fac.empty()) {
      PassSpec ps;
      ps.clique = c;
      ps.src_arena = A_CLIQUE;
      ps.factors = fac;
      ps.write = true;
      dw[ch.empty() ? d : d + 1].push_back(ps);
    }
    for (int v : qby[c]) {
      PassSpec ps;
      ps.clique = c;
      ps.src_arena = shared && !eager[c] ? A_BASE : A_CLIQUE;
      ps.factors = shared ? fac : std::vector<Tensor>{};
      ps.out_kind = OUT_RAW;
      ps.out = var_out_tensor(st, v);
      // materialized: queries read the final table, after its writer
      dw[shared ? d : d + 2].push_back(ps);
    }
    // Clique product X (shared-base, fresh): when two children share a separator
    // scope S, their paired pass reads every factor over S anyway; it also writes
    // X = Π{factors of c over S} (into the per-program message scratch), and the
    // clique's other passes that multiply all of those factors read X instead,
    // one sub-wave later (c5's hub: its other two distribute passes read one
    // tensor instead of three 140000-entry separators).
    if (hub_x && shared && fresh && !eager[c] && !x_used[d] && dw[d].size() > dw0) {
      std::map<std::vector<int>, int> by_scope;
      for (auto& chp : ch) by_scope[p->svars[chp.second]]++;
      const std::vector<int>* S = nullptr;
      for (auto& kv : by_scope)
        if (kv.second >= 2 && (!S || kv.first.size() > S->size())) S = &kv.first;
      std::vector<Tensor> fin;
      if (S)
        for (auto& t : fac)
          if (std::includes(S->begin(), S->end(), t.vars.begin(), t.vars.end())) fin.push_back(t);
      if (S && fin.size() >= 2) {
        auto has = [](const std::vector<Tensor>& fs, const Tensor& t) {
          for (auto& f : fs)
            if (f.off == t.off && f.vars == t.vars) return true;
          return false;
        };
        int writer = -1, consumers = 0;
        for (size_t q = dw0; q < dw[d].size(); ++q) {
          PassSpec& ps = dw[d][q];
          if (ps.clique != c || !ps.scope.empty()) continue;
          if (ps.out.vars == *S) {
            if (writer < 0 && ps.out_kind == OUT_SEP_DFRESH) writer = (int)q;
            continue;
          }
          bool all = true;
          for (auto& t : fin) all = all && has(ps.factors, t);
          consumers += all;
        }
        if (writer >= 0 && consumers > 0) {
          int s_id = -1;
          for (auto& chp : ch)
            if (p->svars[chp.second] == *S) s_id = chp.second;
          Tensor X = sep_tensor(st, s_id, st->msg_ratio_off);
          dw[d][writer].x_off = st->msg_ratio_off;
          std::vector<PassSpec> keep;
          for (size_t q = dw0; q < dw[d].size(); ++q) {
            PassSpec ps = dw[d][q];
            bool all = ps.clique == c && ps.scope.empty() && ps.out.vars != *S;
            for (auto& t : fin) all = all && has(ps.factors, t);
            if (!all) {
              keep.push_back(ps);
              continue;
            }
            std::vector<Tensor> f2{X};
            for (auto& t : ps.factors)
              if (!has(fin, t)) f2.push_back(t);
            ps.factors = f2;
            dwx[d].push_back(ps);
          }
          dw[d].resize(dw0);
          dw[d].insert(dw[d].end(), keep.begin(), keep.end());
          x_used[d] = 1;
        }
      }
    }
  }
  for (int sp = 0; sp < p->n_seps; ++sp) {
    if (qsep[sp].empty()) continue;
    // the separator's final table is written by its parent's distribute pass
    const int a = p->sedge[sp][0], b = p->sedge[sp][1];
    const int par = o.parent[a] == b ? b : a;
    for (int v : qsep[sp]) {
      PassSpec ps;
      ps.clique = par;
      ps.scope = p->svars[sp];
      ps.src_arena = A_AUX;
      ps.src_off = fresh ? sep_alt(st, sp) : sep_cur(st, sp);
      ps.out_kind = OUT_RAW;
      ps.out = var_out_tensor(st, v);
      dw[o.depth[par] + 1].push_back(ps);
    }
  }
  for (size_t d = 0; d < dw.size(); ++d) {
    waves.push_back(dw[d]);
    if (!dwx[d].empty()) waves.push_back(dwx[d]);
  }
  return JT_OK;
}

// Can a pass read its virtual separators (compile_contract's classification: as
// epilogue factors or old separators of a row-per-i contraction pass, at most CMAXV)?
static bool vsep_readable(const jt_state* st, const PassSpec& ps) {
  if (!has_virtual(ps)) return true;
  if (!contract_eligible(st, ps)) return false;
  const auto& s = ps.out.vars;
  std::vector<int> U, vs;
  auto subset = [](const std::vector<int>& a, const std::vector<int>& b) {
    return std::includes(b.begin(), b.end(), a.begin(), a.end());
  };
  // (as K-sum factors, gathered per k, they measured slower on c5 than the factor
  // rows they replace: epilogue reads only)
  for (auto& f : ps.factors) {
    if (f.vclique >= 0 && std::find(vs.begin(), vs.end(), f.vclique) == vs.end()) vs.push_back(f.vclique);
    if (!subset(f.vars, s)) {
      if (f.vclique >= 0) return false;
      U.insert(U.end(), f.vars.begin(), f.vars.end());
    }
  }
  std::sort(U.begin(), U.end());
  if (ps.out.vclique >= 0) {
    if (ps.out_kind != OUT_SEP && ps.out_kind != OUT_SEP_DFRESH) return false;
    if (std::find(vs.begin(), vs.end(), ps.out.vclique) == vs.end()) vs.push_back(ps.out.vclique);
  }
  return (int)vs.size() <= CMAXV && subset(s, U);
}

// Leaves whose collect message is at least JT_VSEP_MIN_MB (default 256; 0: every
// leaf) become virtual separators where every reader can gather them (JT_VSEP=0: off).
static int build_propagate(jt_state* st, const std::vector<int>& roots, const std::vector<int>& qvars,
                           std::vector<std::vector<PassSpec>>& waves, bool fresh = false, bool hub_x = false,
                           bool vsep = false) {
  const jt_plan* p = st->plan;
  std::vector<char> vleaf(p->n_cliques, 0);
  const int64_t min_mb = env_int("JT_VSEP_MIN_MB", 256);
  if (vsep && fresh && st->mode == JT_SHARED_BASE && env_int("JT_VSEP", 1)) {
    Orient o = orient(p, roots);
    for (int c = 0; c < p->n_cliques; ++c)
      if (o.parent[c] >= 0 && o.children[c].empty())
        vleaf[c] = (double)p->ssize[o.psep[c]] * st->B * st->esz >= (double)min_mb * (1 << 20);
  }
  for (int it = 0; it < 16; ++it) {
    waves.clear();
    int rc = build_propagate_waves(st, roots, qvars, waves, fresh, hub_x, vleaf, vsep && env_int("JT_LAZY_FINAL", 1));
    if (rc) return rc;
    bool again = false;
    for (auto& w : waves)
      for (auto& ps : w)
        if (!vsep_readable(st, ps)) {  // its leaves' messages are stored after all
          if (getenv("JT_DEBUG_VSEP"))
            fprintf(stderr, "vsep: pass of clique %d (out kind %d, %zu factors, eligible %d) cannot read leaf %d\n",
                    ps.clique, ps.out_kind, ps.factors.size(), (int)contract_eligible(st, ps),
                    ps.out.vclique >= 0 ? ps.out.vclique : [&] {
                      for (auto& f : ps.factors)
                        if (f.vclique >= 0) return f.vclique;
                      return -1;
                    }());
          for (auto& f : ps.factors)
            if (f.vclique >= 0) vleaf[f.vclique] = 0, again = true;
          if (ps.out.vclique >= 0) vleaf[ps.out.vclique] = 0, again = true;
        }
    if (!again) return JT_OK;
  }
  return JT_ERR_UNSUPPORTED;
}

static std::string key_of(const char* tag, const std::vector<int>& a, const std::vector<int>& b = {}) {
  std::string k(tag);
  for (int x : a) k += "," + std::to_string(x);
  k += "|";
  for (int x : b) k += "," + std::to_string(x);
  return k;
}

static std::vector<int> active_ev(const jt_state* st) {
  std::vector<int> k;
  if (st->mode == JT_SHARED_BASE)
    for (int v = 0; v < st->plan->n_vars; ++v)
      if (st->ev_clique[v] >= 0) {
        k.push_back(v);
        k.push_back(st->ev_clique[v]);
      }
  return k;
}

static int get_program(jt_state* st, const std::string& key,
                       const std::vector<std::vector<PassSpec>>& waves, Program** out) {
  auto it = st->programs.find(key);
  if (it == st->programs.end()) {
    std::unique_ptr<Program> pr;
    int rc = build_program(st, waves, pr);
    if (rc != JT_OK) return rc;
    it = st->programs.emplace(key, std::move(pr)).first;
  }
  *out = it->second.get();
  return JT_OK;
}

// Fill the current separator tables with ones if a reset deferred it.
static int ensure_seps(jt_state* st, cudaStream_t s) {
  if (!st->seps_stale) return JT_OK;
  const jt_plan* p = st->plan;
  const int64_t x0 = st->sep_off[0], y0 = st->ratC_off[0], z0 = st->ratD_off[0];
  const int64_t off = st->sep_in_y ? y0 : x0, n = st->sep_in_y ? z0 - y0 : y0 - x0;
  CK(launch_fill(p->dtype, (char*)st->d_aux + off * st->esz, n, 1.0, s));
  st->launches++;
  st->seps_stale = false;
  return JT_OK;
}

// ------------------------------------------------------------------ C ABI --
extern "C" int jt_state_load(jt_state* st, int case_idx, const double* clique_concat, const double* sep_concat) {
  if (!st || case_idx < -1 || case_idx >= st->B_user) return JT_ERR_BAD_ARG;
  const jt_plan* p = st->plan;
  DevGuard g(p->device);
  const bool shared = st->mode == JT_SHARED_BASE;
  if (shared && case_idx != -1 && clique_concat) return JT_ERR_UNSUPPORTED;
  int64_t tot_c = std::accumulate(p->csize.begin(), p->csize.end(), int64_t(0));
  int64_t tot_s = std::accumulate(p->ssize.begin(), p->ssize.end(), int64_t(0));
  int rc = ensure_stage(st, std::max(tot_c, tot_s));
  if (rc) return rc;
  cudaStream_t s = st->stream;
  const int64_t B = st->B;
  if ((rc = ensure_seps(st, s))) return rc;
  st->fresh = (case_idx < 0 && !sep_concat) || (st->fresh && !sep_concat);
  if (clique_concat && case_idx < 0) {
    // new base tables: fresh prescale exponents; separators (ones or given) unscaled
    std::vector<int64_t> co(p->n_cliques + 1, 0);
    for (int c = 0; c < p->n_cliques; ++c) co[c + 1] = co[c] + p->csize[c];
    choose_prescale(st, [&](int c) { return clique_concat + co[c]; });
    st->e_c = st->pre_e;
    std::fill(st->e_s.begin(), st->e_s.end(), 0);
  }
  if (clique_concat && case_idx < 0 && shared) {
    // host copy of the (prescaled) base for contraction passes; programs built on the old base are stale
    st->h_base.assign(st->n_base, 1.0);
    int64_t o = 0;
    for (int c = 0; c < p->n_cliques; ++c) {
      for (int64_t i = 0; i < p->csize[c]; ++i)
        st->h_base[st->boff[c] + i] = std::ldexp(clique_concat[o + i], st->pre_e[c]);
      o += p->csize[c];
    }
    st->programs.clear();
  }
  if (clique_concat) {
    CK(cudaMemcpyAsync(st->d_stage, clique_concat, tot_c * 8, cudaMemcpyHostToDevice, s));
    int64_t o = 0;
    for (int c = 0; c < p->n_cliques; ++c) {
      const int64_t nc = p->csize[c];
      if (case_idx < 0) {
        char* dst = (char*)st->d_base + st->boff[c] * st->esz;
        CK(launch_convert_d2t(p->dtype, st->d_stage + o, dst, nc, 1, 1, s, st->pre_e[c]));
      }
      if (!shared) {
        char* dst = (char*)st->d_clique + (st->coff[c] + (case_idx < 0 ? 0 : case_idx)) * st->esz;
        CK(launch_convert_d2t(p->dtype, st->d_stage + o, dst, nc, B, case_idx < 0 ? B : 1, s, st->e_c[c]));
      }
      o += nc;
    }
    CK(cudaStreamSynchronize(s));
  }
  if (sep_concat) {
    CK(cudaMemcpyAsync(st->d_stage, sep_concat, tot_s * 8, cudaMemcpyHostToDevice, s));
  }
  int64_t o = 0;
  for (int sp = 0; sp < p->n_seps; ++sp) {
    const int64_t ns = p->ssize[sp];
    char* dst = (char*)st->d_aux + (sep_cur(st, sp) + (case_idx < 0 ? 0 : case_idx)) * st->esz;
    if (sep_concat) {
      CK(launch_convert_d2t(p->dtype, st->d_stage + o, dst, ns, B, case_idx < 0 ? B : 1, s, st->e_s[sp]));
    } else if (case_idx < 0) {
      CK(launch_fill(p->dtype, dst, ns * B, 1.0, s));
    }
    o += ns;
  }
  CK(cudaStreamSynchronize(s));
  return JT_OK;
}

extern "C" int jt_state_initialize(jt_state* st, int n_cpts, const int32_t* cpt_clique, const int32_t* cpt_off,
                                   const int32_t* cpt_vars, const double* cpt_values) {
  if (!st || n_cpts < 0 || (n_cpts > 0 && (!cpt_clique || !cpt_off || !cpt_vars || !cpt_values)))
    return JT_ERR_BAD_ARG;
  const jt_plan* p = st->plan;
  DevGuard g(p->device);
  std::vector<std::vector<int>> by_clique(p->n_cliques);
  std::vector<int64_t> val_off(n_cpts + 1, 0);
  for (int k = 0; k < n_cpts; ++k) {
    const int c = cpt_clique[k];
    if (c < 0 || c >= p->n_cliques || cpt_off[k + 1] < cpt_off[k]) return JT_ERR_BAD_ARG;
    int64_t n = 1;
    for (int i = cpt_off[k]; i < cpt_off[k + 1]; ++i) {
      const int v = cpt_vars[i];
      if (v < 0 || v >= p->n_vars || !std::binary_search(p->cvars[c].begin(), p->cvars[c].end(), v))
        return JT_ERR_BAD_ARG;  // NoCoveringCliqueError territory: the CPT must fit its clique
      n *= p->cards[v];
    }
    val_off[k + 1] = val_off[k] + n;
    by_clique[c].push_back(k);
  }
  std::vector<InitClique> cl(p->n_cliques);
  std::vector<InitTerm> terms;
  std::vector<int64_t> vdesc;
  int64_t max_size = 1;
  for (int c = 0; c < p->n_cliques; ++c) {
    const auto& cv = p->cvars[c];
    std::vector<int64_t> cstride(cv.size(), 1);
    for (int i = (int)cv.size() - 2; i >= 0; --i) cstride[i] = cstride[i + 1] * p->cards[cv[i + 1]];
    cl[c].off = st->boff[c];
    cl[c].size = p->csize[c];
    cl[c].first_term = (int)terms.size();
    cl[c].n_terms = (int)by_clique[c].size();
    max_size = std::max(max_size, p->csize[c]);
    for (int k : by_clique[c]) {
      InitTerm t;
      t.cpt_off = val_off[k];
      t.first_var = (int)(vdesc.size() / 3);
      t.nv = cpt_off[k + 1] - cpt_off[k];
      int64_t ts = 1;
      std::vector<int64_t> tstr(t.nv);
      for (int i = t.nv - 1; i >= 0; --i) {
        tstr[i] = ts;
        ts *= p->cards[cpt_vars[cpt_off[k] + i]];
      }
      for (int i = 0; i < t.nv; ++i) {
        const int v = cpt_vars[cpt_off[k] + i];
        const int pos = (int)(std::lower_bound(cv.begin(), cv.end(), v) - cv.begin());
        vdesc.push_back(cstride[pos]);
        vdesc.push_back(p->cards[v]);
        vdesc.push_back(tstr[i]);
      }
      terms.push_back(t);
    }
  }
  int rc = ensure_stage(st, std::max<int64_t>(val_off[n_cpts], 1));
  if (rc) return rc;
  cudaStream_t s = st->stream;
  InitClique* d_cl = nullptr;
  InitTerm* d_terms = nullptr;
  int64_t* d_vd = nullptr;
  auto cleanup = [&]() {
    cudaFree(d_cl);
    cudaFree(d_terms);
    cudaFree(d_vd);
  };
  cudaError_t e = cudaMalloc(&d_cl, std::max<size_t>(cl.size(), 1) * sizeof(InitClique));
  if (e == cudaSuccess) e = cudaMalloc(&d_terms, std::max<size_t>(terms.size(), 1) * sizeof(InitTerm));
  if (e == cudaSuccess) e = cudaMalloc(&d_vd, std::max<size_t>(vdesc.size(), 1) * sizeof(int64_t));
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_cl, cl.data(), cl.size() * sizeof(InitClique), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && !terms.empty())
    e = cudaMemcpyAsync(d_terms, terms.data(), terms.size() * sizeof(InitTerm), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && !vdesc.empty())
    e = cudaMemcpyAsync(d_vd, vdesc.data(), vdesc.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && val_off[n_cpts] > 0)
    e = cudaMemcpyAsync(st->d_stage, cpt_values, val_off[n_cpts] * sizeof(double), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = launch_init(st->d_base, p->dtype, st->d_stage, d_cl, p->n_cliques, d_terms, d_vd, max_size, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cleanup();
  if (e != cudaSuccess) {
    last_cuda_error() = e;
    return e == cudaErrorMemoryAllocation ? JT_ERR_OOM : JT_ERR_CUDA;
  }
  st->launches++;
  {
    // prescale the new base (power-of-two balance, see jt_state) from its clique sums
    std::vector<char> raw(st->n_base * st->esz);
    CK(cudaMemcpy(raw.data(), st->d_base, raw.size(), cudaMemcpyDeviceToHost));
    std::vector<double> hb(st->n_base);
    for (int64_t i = 0; i < st->n_base; ++i)
      hb[i] = st->esz == 8 ? ((const double*)raw.data())[i] : (double)((const float*)raw.data())[i];
    choose_prescale(st, [&](int c) { return hb.data() + st->boff[c]; });
    for (int c = 0; c < p->n_cliques; ++c) {
      CK(launch_scale_pow2(p->dtype, (char*)st->d_base + st->boff[c] * st->esz, p->csize[c], st->pre_e[c], s));
      for (int64_t i = 0; i < p->csize[c]; ++i) hb[st->boff[c] + i] = std::ldexp(hb[st->boff[c] + i], st->pre_e[c]);
    }
    CK(cudaStreamSynchronize(s));
    if (st->mode == JT_SHARED_BASE) {  // host copy of the new base (contraction passes)
      st->h_base.swap(hb);
      st->programs.clear();
    }
  }
  // every case starts from the new base tables; separators ones, no evidence
  rc = jt_state_reset(st, nullptr);
  if (rc) return rc;
  CK(cudaStreamSynchronize(s));
  return JT_OK;
}

static int materialize_final(jt_state* st, cudaStream_t s);

extern "C" int jt_state_store(jt_state* st, int case_idx, double* clique_concat, double* sep_concat) {
  if (!st || case_idx < 0 || case_idx >= st->B_user) return JT_ERR_BAD_ARG;
  const jt_plan* p = st->plan;
  DevGuard g(p->device);
  if (st->mode == JT_SHARED_BASE && clique_concat) return JT_ERR_UNSUPPORTED;
  int64_t tot_c = std::accumulate(p->csize.begin(), p->csize.end(), int64_t(0));
  int64_t tot_s = std::accumulate(p->ssize.begin(), p->ssize.end(), int64_t(0));
  int rc = ensure_stage(st, std::max(tot_c, tot_s));
  if (rc) return rc;
  cudaStream_t s = st->stream;
  const int64_t B = st->B;
  if ((rc = ensure_seps(st, s))) return rc;
  if (clique_concat) {
    int64_t o = 0;
    for (int c = 0; c < p->n_cliques; ++c) {
      const char* src = (const char*)st->d_clique + (st->coff[c] + case_idx) * st->esz;
      CK(launch_convert_t2d(p->dtype, src, B, st->d_stage + o, p->csize[c], s, st->e_c[c]));
      o += p->csize[c];
    }
    CK(cudaMemcpyAsync(clique_concat, st->d_stage, tot_c * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  if (sep_concat) {
    if (!st->final_pending.empty() && (rc = materialize_final(st, s))) return rc;
    int64_t o = 0;
    for (int sp = 0; sp < p->n_seps; ++sp) {
      const char* src = (const char*)st->d_aux + (sep_cur(st, sp) + case_idx) * st->esz;
      CK(launch_convert_t2d(p->dtype, src, B, st->d_stage + o, p->ssize[sp], s, st->e_s[sp]));
      o += p->ssize[sp];
    }
    CK(cudaMemcpyAsync(sep_concat, st->d_stage, tot_s * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  return JT_OK;
}

extern "C" int jt_state_clone(jt_state* src, jt_state** out) {
  if (!src || !out) return JT_ERR_BAD_ARG;
  DevGuard g(src->plan->device);
  jt_state* dst = nullptr;
  int rc = jt_state_create(src->plan, src->B, src->mode, &dst);
  if (rc) return rc;
  std::unique_ptr<jt_state> own(dst);
  cudaStream_t s = dst->stream;
  // src work may be queued on any stream of the caller's: order after all of it
  CK(cudaDeviceSynchronize());
  const size_t es = src->esz;
  if (src->n_clique) CK(cudaMemcpyAsync(dst->d_clique, src->d_clique, src->n_clique * es, cudaMemcpyDeviceToDevice, s));
  if (src->n_base) CK(cudaMemcpyAsync(dst->d_base, src->d_base, src->n_base * es, cudaMemcpyDeviceToDevice, s));
  if (src->n_aux) CK(cudaMemcpyAsync(dst->d_aux, src->d_aux, src->n_aux * es, cudaMemcpyDeviceToDevice, s));
  CK(cudaStreamSynchronize(s));
  dst->fresh = src->fresh;
  dst->seps_stale = src->seps_stale;
  dst->sep_in_y = src->sep_in_y;
  dst->vsep_pending = src->vsep_pending;
  dst->final_pending = src->final_pending;
  dst->ev_clique = src->ev_clique;
  dst->h_base = src->h_base;
  dst->pre_e = src->pre_e;
  dst->e_c = src->e_c;
  dst->e_s = src->e_s;
  *out = own.release();
  return JT_OK;
}

extern "C" int jt_clear_evidence(jt_state* st) {
  if (!st) return JT_ERR_BAD_ARG;
  std::fill(st->ev_clique.begin(), st->ev_clique.end(), -1);
  return JT_OK;
}

extern "C" int jt_state_reset(jt_state* st, void* stream) {
  if (!st) return JT_ERR_BAD_ARG;
  const jt_plan* p = st->plan;
  DevGuard g(p->device);
  cudaStream_t s = pick_stream(st, stream);
  jt_clear_evidence(st);
  // separators back to ones: deferred — a fresh propagation never reads them
  st->seps_stale = p->n_seps > 0;
  st->fresh = true;
  st->e_c = st->pre_e;
  std::fill(st->e_s.begin(), st->e_s.end(), 0);
  if (st->mode == JT_SHARED_BASE) return JT_OK;
  Program* pr;
  auto it = st->programs.find("reset");
  if (it != st->programs.end()) {
    pr = it->second.get();
  } else {
    std::vector<std::vector<PassSpec>> waves(1);
    for (int c = 0; c < p->n_cliques; ++c) {
      PassSpec ps;
      ps.clique = c;
      ps.src_arena = A_BASE;
      ps.write = true;
      waves[0].push_back(ps);
    }
    int rc = get_program(st, "reset", waves, &pr);
    if (rc) return rc;
  }
  return run_program(st, pr, s);
}

// Observations arrive as (case, var, state) triples (host or device); masks are
// built on the device.  Shared-base states keep them as persistent factors
// (observations accumulate until reset, like repeated apply_evidence calls on
// the reference state); materialized states multiply them into the owning
// cliques right away (propagate.py:257-258).
static int evidence_common(jt_state* st, int n, const int32_t* d_obs, const std::vector<int>& vars,
                           const std::vector<int>& cliques, cudaStream_t s) {
  const jt_plan* p = st->plan;
  const bool shared = st->mode == JT_SHARED_BASE;
  std::vector<int32_t> fill;
  for (size_t i = 0; i < vars.size(); ++i) {
    const int v = vars[i], c = cliques[i];
    if (shared) {
      if (st->ev_clique[v] >= 0 && st->ev_clique[v] != c) return JT_ERR_UNSUPPORTED;
      if (st->ev_clique[v] < 0) fill.push_back(v);
      st->ev_clique[v] = c;
    } else {
      fill.push_back(v);
    }
  }
  // The fill list (variables whose masks start as ones) is the same for every
  // micro-batch of a batch run: it lives in its own device buffer and is
  // re-uploaded only when it changes, so the steady state issues no pageable
  // host->device copy (which may synchronize the stream and stall pipelining).
  if (!fill.empty()) {
    if (fill != st->fill_host) {
      if ((int64_t)fill.size() > st->fill_cap) {
        CK(cudaStreamSynchronize(s));
        cudaFree(st->d_fill);
        st->d_fill = nullptr;
        st->fill_cap = 0;
        CK(cudaMalloc(&st->d_fill, fill.size() * sizeof(int32_t)));
        st->fill_cap = (int64_t)fill.size();
      }
      CK(cudaMemcpyAsync(st->d_fill, fill.data(), fill.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
      st->fill_host = fill;
    }
    CK(launch_ev_fill(st->d_aux, p->dtype, st->d_fill, (int)fill.size(), st->d_evoff, st->d_cards, st->B, s));
    st->launches++;
  }
  CK(launch_ev_zero(st->d_aux, p->dtype, d_obs, n, st->d_evoff, st->d_cards, st->B, s));
  st->launches++;
  if (shared) return JT_OK;
  std::map<int, std::vector<int>> by_clique;
  for (size_t i = 0; i < vars.size(); ++i) by_clique[cliques[i]].push_back(vars[i]);
  std::vector<std::vector<PassSpec>> waves;
  std::vector<int> kk;
  for (auto& kv : by_clique) {
    kk.push_back(kv.first);
    for (size_t i = 0; i < kv.second.size(); i += MAXF) {
      PassSpec ps;
      ps.clique = kv.first;
      ps.src_arena = A_CLIQUE;
      ps.write = true;
      for (size_t k = i; k < std::min(kv.second.size(), i + MAXF); ++k) {
        ps.factors.push_back(ev_tensor(st, kv.second[k]));
        kk.push_back(kv.second[k]);
      }
      const size_t wi = i / MAXF;
      if (waves.size() <= wi) waves.resize(wi + 1);
      waves[wi].push_back(ps);
    }
    kk.push_back(-1);
  }
  Program* pr;
  int rc = get_program(st, key_of("ev", kk), waves, &pr);
  if (rc) return rc;
  return run_program(st, pr, s);
}

static int collect_vars(const jt_state* st, int n, const int32_t* var, const int32_t* clique,
                        std::vector<int>& vars, std::vector<int>& cliques) {
  const jt_plan* p = st->plan;
  std::map<int, int> owner;
  for (int i = 0; i < n; ++i) {
    const int v = var[i], c = clique[i];
    if (v < 0 || v >= p->n_vars || c < 0 || c >= p->n_cliques) return JT_ERR_BAD_ARG;
    if (!std::binary_search(p->cvars[c].begin(), p->cvars[c].end(), v)) return JT_ERR_BAD_ARG;
    auto it = owner.find(v);
    if (it != owner.end() && it->second != c) return JT_ERR_BAD_ARG;
    owner[v] = c;
  }
  for (auto& kv : owner) {
    vars.push_back(kv.first);
    cliques.push_back(kv.second);
  }
  return JT_OK;
}

extern "C" int jt_apply_evidence(jt_state* st, int n, const int32_t* case_idx, const int32_t* var,
                                 const int32_t* clique, const int32_t* value, void* stream) {
  if (!st || n < 0) return JT_ERR_BAD_ARG;
  if (n == 0) return JT_OK;
  const jt_plan* p = st->plan;
  DevGuard g(p->device);
  std::vector<int> vars, cliques;
  int rc = collect_vars(st, n, var, clique, vars, cliques);
  if (rc) return rc;
  std::vector<int32_t> obs(3 * (size_t)n);
  for (int i = 0; i < n; ++i) {
    const int b = case_idx ? case_idx[i] : -1;
    if (b < -1 || b >= st->B_user || value[i] < 0 || value[i] >= p->cards[var[i]]) return JT_ERR_BAD_ARG;
    obs[3 * i] = b;
    obs[3 * i + 1] = var[i];
    obs[3 * i + 2] = value[i];
  }
  const int64_t need = 3 * (int64_t)n;
  if (need > st->obs_cap) {
    cudaFree(st->d_obs);
    st->d_obs = nullptr;
    CK(cudaMalloc(&st->d_obs, need * sizeof(int32_t)));
    st->obs_cap = need;
  }
  cudaStream_t s = pick_stream(st, stream);
  // pageable source: the copy is staged before cudaMemcpyAsync returns
  CK(cudaMemcpyAsync(st->d_obs, obs.data(), obs.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  return evidence_common(st, n, st->d_obs, vars, cliques, s);
}

extern "C" int jt_apply_evidence_device(jt_state* st, int n, const int32_t* d_obs, int n_vars,
                                        const int32_t* var, const int32_t* clique, void* stream) {
  if (!st || n < 0 || n_vars < 0 || (n > 0 && !d_obs)) return JT_ERR_BAD_ARG;
  if (n == 0) return JT_OK;
  DevGuard g(st->plan->device);
  std::vector<int> vars, cliques;
  int rc = collect_vars(st, n_vars, var, clique, vars, cliques);
  if (rc) return rc;
  return evidence_common(st, n, d_obs, vars, cliques, pick_stream(st, stream));
}

extern "C" int jt_message(jt_state* st, int src, int tgt, int sep, void* stream) {
  if (!st) return JT_ERR_BAD_ARG;
  const jt_plan* p = st->plan;
  if (src < 0 || tgt < 0 || sep < 0 || src >= p->n_cliques || tgt >= p->n_cliques || sep >= p->n_seps)
    return JT_ERR_BAD_ARG;
  const auto& e = p->sedge[sep];
  if (!((e[0] == src && e[1] == tgt) || (e[0] == tgt && e[1] == src))) return JT_ERR_BAD_ARG;
  if (st->mode != JT_MATERIALIZED) return JT_ERR_UNSUPPORTED;
  DevGuard g(p->device);
  cudaStream_t s = pick_stream(st, stream);
  int rc0 = ensure_seps(st, s);
  if (rc0) return rc0;
  st->fresh = false;
  // exponents (jt_state): new sep = star of src; tgt *= new/old
  {
    const int es_old = st->e_s[sep];
    st->e_s[sep] = st->e_c[src];
    st->e_c[tgt] += st->e_c[src] - es_old;
  }
  const std::string mkey = key_of("msg", {src, tgt, sep, (int)st->sep_in_y});
  Program* pr;
  auto it = st->programs.find(mkey);
  if (it != st->programs.end()) {
    pr = it->second.get();
  } else {
    std::vector<std::vector<PassSpec>> waves(2);
    PassSpec m;
    m.clique = src;
    m.out_kind = OUT_SEP;
    m.out = sep_tensor(st, sep, sep_cur(st, sep));
    m.ratio_off = st->msg_ratio_off;
    waves[0].push_back(m);
    PassSpec sc;
    sc.clique = tgt;
    sc.write = true;
    sc.factors.push_back(sep_tensor(st, sep, st->msg_ratio_off));
    waves[1].push_back(sc);
    int rc = get_program(st, mkey, waves, &pr);
    if (rc) return rc;
  }
  return run_program(st, pr, s);
}

static int resolve_roots(const jt_state* st, const int32_t* roots_or_null, std::vector<int>& roots) {
  const jt_plan* p = st->plan;
  roots = p->roots;
  if (roots_or_null) {
    for (size_t i = 0; i < roots.size(); ++i) {
      const int r = roots_or_null[i];
      if (r < 0 || r >= p->n_cliques || p->comp[r] != (int)i) return JT_ERR_BAD_ARG;
      roots[i] = r;
    }
  }
  return JT_OK;
}


// Shared-base states keep only the latest propagation's ratios: the base never
// absorbs a message, so the Hugin update new/old of a second propagation has no
// table to apply to.  A re-propagation (or one after incremental evidence)
// therefore restarts from the base and every active evidence mask (evidence
// accumulates as masks until reset): calibrated tables are P(C, e) whatever the
// message history, so this equals the reference's repeated belief_propagation.
static void shared_restart(jt_state* st) {
  st->vsep_pending.clear();
  st->final_pending.clear();
  if (st->mode != JT_SHARED_BASE || st->fresh) return;
  st->fresh = true;
  st->seps_stale = st->plan->n_seps > 0;
  st->e_c = st->pre_e;
  std::fill(st->e_s.begin(), st->e_s.end(), 0);
}

extern "C" int jt_propagate(jt_state* st, const int32_t* roots_or_null, void* stream) {
  if (!st) return JT_ERR_BAD_ARG;
  DevGuard g(st->plan->device);
  std::vector<int> roots;
  int rc = resolve_roots(st, roots_or_null, roots);
  if (rc) return rc;
  cudaStream_t s = pick_stream(st, stream);
  shared_restart(st);
  const bool fresh = st->fresh;
  if (!fresh && (rc = ensure_seps(st, s))) return rc;
  std::vector<int> tag{(int)fresh, (int)st->sep_in_y};
  std::vector<int> kv = active_ev(st);
  kv.insert(kv.end(), tag.begin(), tag.end());
  const std::string key = key_of("bp", roots, kv);
  Program* pr;
  auto it = st->programs.find(key);
  if (it != st->programs.end()) {
    pr = it->second.get();
  } else {
    std::vector<std::vector<PassSpec>> waves;
    rc = build_propagate(st, roots, {}, waves, fresh);
    if (rc) return rc;
    rc = get_program(st, key, waves, &pr);
    if (rc) return rc;
  }
  rc = run_program(st, pr, s);
  if (rc) return rc;
  set_all_exp(st, joint_exp(st));  // calibrated: every table is a marginal of the joint
  if (fresh) st->sep_in_y = !st->sep_in_y;
  st->fresh = false;
  st->seps_stale = false;
  return JT_OK;
}

static int smallest_holder(const jt_plan* p, int v) {
  int best = -1;
  for (int c = 0; c < p->n_cliques; ++c)
    if (std::binary_search(p->cvars[c].begin(), p->cvars[c].end(), v))
      if (best < 0 || p->csize[c] < p->csize[best]) best = c;
  return best;
}

// raw marginals are already in qout; normalize into out_device [B][Σcard].
// Per-variable-list metadata is uploaded once and cached, so this is async.
static int finish_query(jt_state* st, int n, const int32_t* var, int normalize, double* out_device,
                        cudaStream_t s, int* total_cols_out, const std::vector<int>& exps) {
  const jt_plan* p = st->plan;
  std::vector<int> vs(var, var + n);
  const std::string key = key_of("qm", vs);
  auto it = st->qmeta.find(key);
  if (it == st->qmeta.end()) {
    std::vector<int64_t> meta(3 * (size_t)n + 4);
    int64_t* qo = meta.data();
    int32_t* qc = reinterpret_cast<int32_t*>(meta.data() + n);
    int32_t* qcol = qc + n;
    int cols = 0;
    for (int i = 0; i < n; ++i) {
      qo[i] = st->q_off[var[i]];
      qc[i] = p->cards[var[i]];
      qcol[i] = cols;
      cols += p->cards[var[i]];
    }
    int64_t* d = nullptr;
    CK(cudaMalloc(&d, meta.size() * sizeof(int64_t)));
    CK(cudaMemcpy(d, meta.data(), meta.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    it = st->qmeta.emplace(key, std::make_pair(d, cols)).first;
  }
  const int64_t* dqo = it->second.first;
  const int32_t* dqc = reinterpret_cast<const int32_t*>(dqo + n);
  const int32_t* dqcol = dqc + n;
  const int cols = it->second.second;
  // stored tables are exact * 2^e: unnormalized results undo it (one exponent, or per query)
  const int* d_qexp = nullptr;
  int exp_all = exps.empty() ? 0 : exps[0];
  if (!normalize && std::any_of(exps.begin(), exps.end(), [&](int e) { return e != exp_all; })) {
    if ((int64_t)exps.size() > st->qexp_cap) {
      CK(cudaStreamSynchronize(s));
      cudaFree(st->d_qexp);
      st->d_qexp = nullptr;
      st->qexp_cap = 0;
      CK(cudaMalloc(&st->d_qexp, exps.size() * sizeof(int)));
      st->qexp_cap = (int64_t)exps.size();
    }
    CK(cudaMemcpyAsync(st->d_qexp, exps.data(), exps.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    d_qexp = st->d_qexp;
  }
  CK(launch_normalize(st->d_qout, dqo, dqc, dqcol, n, st->B, st->B_user, cols, normalize, out_device, st->d_err, d_qexp,
                      exp_all, s));
  st->launches++;
  if (total_cols_out) *total_cols_out = cols;
  return JT_OK;
}

// The collect messages of the leaves the last (fused) propagation gathered
// instead of storing (virtual separators), written where a stored one would be
// now (sep_alt after the run's swap), for the queries that read them.
static int materialize_vsep(jt_state* st, cudaStream_t s) {
  const jt_plan* p = st->plan;
  Orient o = orient(p, p->roots);
  std::vector<PassSpec> w;
  for (int c : st->vsep_pending) {
    PassSpec ps;
    ps.clique = c;
    ps.src_arena = A_BASE;
    for (int v = 0; v < p->n_vars; ++v)
      if (st->ev_clique[v] == c) ps.factors.push_back(ev_tensor(st, v));
    ps.out_kind = OUT_SEP_FRESH;
    ps.out = sep_tensor(st, o.psep[c], sep_alt(st, o.psep[c]));
    w.push_back(ps);
  }
  std::vector<int> kv = active_ev(st);
  kv.push_back((int)st->sep_in_y);
  Program* pr;
  int rc = get_program(st, key_of("vm", st->vsep_pending, kv), {w}, &pr);
  if (rc) return rc;
  if ((rc = run_program(st, pr, s))) return rc;
  st->vsep_pending.clear();
  return JT_OK;
}

// Final separator tables the last fused propagation did not store: collect
// message (sep_alt after the run's swap) x distribute ratio, as its distribute
// pass would have written them (OUT_SEP_DFRESH: new = old * Σ, ratio = Σ or 0).
static int materialize_final(jt_state* st, cudaStream_t s) {
  int rc;
  if (!st->vsep_pending.empty() && (rc = materialize_vsep(st, s))) return rc;
  for (int sp : st->final_pending) {
    char* aux = (char*)st->d_aux;
    const int64_t n = st->plan->ssize[sp] * st->B;
    CK(launch_mul(st->plan->dtype, aux + sep_cur(st, sp) * st->esz, aux + sep_alt(st, sp) * st->esz,
                  aux + st->ratD_off[sp] * st->esz, n, s));
    st->launches++;
  }
  st->final_pending.clear();
  return JT_OK;
}

static int query_program(jt_state* st, int n, const int32_t* var, const int32_t* clique, cudaStream_t s,
                         std::vector<int>& exps) {
  const jt_plan* p = st->plan;
  std::vector<int> vs, cs;
  for (int i = 0; i < n; ++i) {
    const int v = var[i];
    if (v < 0 || v >= p->n_vars) return JT_ERR_BAD_ARG;
    int c = clique ? clique[i] : -1;
    if (c < 0) c = smallest_holder(p, v);
    if (c < 0) return JT_ERR_BAD_ARG;
    if (!std::binary_search(p->cvars[c].begin(), p->cvars[c].end(), v)) return JT_ERR_BAD_ARG;
    vs.push_back(v);
    cs.push_back(c);
    exps.push_back(st->e_c[c]);
  }
  std::vector<int> kk = vs;
  kk.insert(kk.end(), cs.begin(), cs.end());
  const bool shared = st->mode == JT_SHARED_BASE;
  // shared-base state not propagated since reset/load: its tables are base × evidence
  const bool unprop = shared && st->fresh;
#ifndef JT_NO_VSEP_MATERIALIZE  // (test-sensitivity variant only)
  if (shared && !unprop && !st->vsep_pending.empty()) {
    int rc = materialize_vsep(st, s);
    if (rc) return rc;
  }
#endif
  std::vector<int> kv = active_ev(st);
  kv.push_back((int)st->sep_in_y);
  kv.push_back((int)unprop);
  std::string key = key_of("q", kk, kv);
  Program* pr;
  auto it = st->programs.find(key);
  if (it != st->programs.end()) {
    pr = it->second.get();
  } else {
    std::vector<std::vector<PassSpec>> waves(1);
    Orient o;
    if (shared) o = orient(p, p->roots);
    for (int i = 0; i < n; ++i) {
      PassSpec ps;
      ps.clique = cs[i];
      ps.src_arena = shared ? A_BASE : A_CLIQUE;
      ps.out_kind = OUT_RAW;
      ps.out = var_out_tensor(st, vs[i]);
      if (shared) {
        // final table of the clique = base × evidence × Π neighbour ratios; a hub
        // (eager clique) holds base × evidence × children's ratios per case already
        const int c = cs[i];
        int nev = 0;
        for (int v = 0; v < p->n_vars; ++v) nev += st->ev_clique[v] == c;
        const bool eager = (int)o.children[c].size() + (o.parent[c] >= 0 ? 1 : 0) + nev > MAXF;
        if (eager && !st->hub[c]) return JT_ERR_UNSUPPORTED;
        if (eager && !unprop) {
          ps.src_arena = A_CLIQUE;
          if (o.parent[c] >= 0) ps.factors.push_back(sep_tensor(st, o.psep[c], st->ratD_off[o.psep[c]]));
        } else {
          if (!unprop) {
            for (auto& ch : o.children[c]) ps.factors.push_back(sep_tensor(st, ch.second, sep_alt(st, ch.second)));
            if (o.parent[c] >= 0) ps.factors.push_back(sep_tensor(st, o.psep[c], st->ratD_off[o.psep[c]]));
          }
          for (int v = 0; v < p->n_vars; ++v)
            if (st->ev_clique[v] == c) ps.factors.push_back(ev_tensor(st, v));
          if ((int)ps.factors.size() > MAXF) return JT_ERR_UNSUPPORTED;
        }
      }
      waves[0].push_back(ps);
    }
    int rc = get_program(st, key, waves, &pr);
    if (rc) return rc;
  }
  return run_program(st, pr, s);
}

extern "C" int jt_query_device(jt_state* st, int n, const int32_t* var, const int32_t* clique, int normalize,
                               double* out_device, void* stream) {
  if (!st || n < 0 || !out_device) return JT_ERR_BAD_ARG;
  if (n == 0) return JT_OK;
  DevGuard g(st->plan->device);
  cudaStream_t s = pick_stream(st, stream);
  std::vector<int> exps;
  int rc = query_program(st, n, var, clique, s, exps);
  if (rc) return rc;
  return finish_query(st, n, var, normalize, out_device, s, nullptr, exps);
}

extern "C" int jt_query(jt_state* st, int n, const int32_t* var, const int32_t* clique, int normalize,
                        double* out_host, void* stream) {
  if (!st || n < 0 || !out_host) return JT_ERR_BAD_ARG;
  if (n == 0) return JT_OK;
  DevGuard g(st->plan->device);
  const jt_plan* p = st->plan;
  int64_t cols = 0;
  for (int i = 0; i < n; ++i) {
    if (var[i] < 0 || var[i] >= p->n_vars) return JT_ERR_BAD_ARG;
    cols += p->cards[var[i]];
  }
  const int64_t need = cols * st->B_user;
  if (need > st->post_cap) {
    cudaFree(st->d_post);
    st->d_post = nullptr;
    CK(cudaMalloc(&st->d_post, need * sizeof(double)));
    st->post_cap = need;
  }
  cudaStream_t s = pick_stream(st, stream);
  int rc = jt_query_device(st, n, var, clique, normalize, st->d_post, s);
  if (rc) return rc;
  CK(cudaMemcpyAsync(out_host, st->d_post, need * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return JT_OK;
}

extern "C" int jt_propagate_query(jt_state* st, int n, const int32_t* var, int normalize, double* out_device,
                                  void* stream) {
  if (!st || n < 0 || (n > 0 && !out_device)) return JT_ERR_BAD_ARG;
  const jt_plan* p = st->plan;
  DevGuard g(p->device);
  std::vector<int> vs;
  for (int i = 0; i < n; ++i) {
    if (var[i] < 0 || var[i] >= p->n_vars) return JT_ERR_BAD_ARG;
    vs.push_back(var[i]);
  }
  if (st->mode != JT_SHARED_BASE) {
    int rc = jt_propagate(st, nullptr, stream);
    if (rc) return rc;
    return n ? jt_query_device(st, n, var, nullptr, normalize, out_device, stream) : JT_OK;
  }
  cudaStream_t s = pick_stream(st, stream);
  shared_restart(st);
  const bool fresh = st->fresh;
  if (!fresh) {
    int rc = ensure_seps(st, s);
    if (rc) return rc;
  }
  std::vector<int> kv = active_ev(st);
  kv.push_back((int)fresh);
  kv.push_back((int)st->sep_in_y);
  const std::string key = key_of("bpq", vs, kv);
  Program* pr;
  auto it = st->programs.find(key);
  if (it != st->programs.end()) {
    pr = it->second.get();
  } else {
    std::vector<std::vector<PassSpec>> waves;
    // clique product X (with virtual separators: fp64 -7%, fp32 -11% program time);
    // virtual separators; when a program cannot place them, the plainer ones
    const bool hx = env_int("JT_HUBX", 1) != 0;
    const bool attempts[3][2] = {{hx, true}, {hx, false}, {false, false}};
    int rc = JT_ERR_UNSUPPORTED;
    for (int a = 0; a < 3 && rc == JT_ERR_UNSUPPORTED; ++a) {
      if (a > 0 && attempts[a][0] == attempts[a - 1][0] && attempts[a][1] == attempts[a - 1][1]) continue;
      if ((rc = build_propagate(st, p->roots, vs, waves, fresh, attempts[a][0], attempts[a][1]))) return rc;
      rc = get_program(st, key, waves, &pr);
    }
    if (rc) return rc;
  }
  int rc = run_program(st, pr, s);
  if (rc) return rc;
  st->vsep_pending = pr->vsep_leaves;
  st->final_pending = pr->final_skip;
  set_all_exp(st, joint_exp(st));
  if (fresh) st->sep_in_y = !st->sep_in_y;
  st->fresh = false;
  st->seps_stale = false;
  return n ? finish_query(st, n, var, normalize, out_device, s, nullptr, std::vector<int>(n, st->e_c[0])) : JT_OK;
}

extern "C" int jt_sync_error(jt_state* st) {
  if (!st) return JT_ERR_BAD_ARG;
  DevGuard g(st->plan->device);
  CK(cudaDeviceSynchronize());
  int h[2] = {0, INT_MAX};
  const int init[2] = {0, INT_MAX};
  CK(cudaMemcpy(h, st->d_err, sizeof h, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(st->d_err, init, sizeof init, cudaMemcpyHostToDevice));
  st->err_case = (h[0] & EB_ZERO_MASS) && h[1] != INT_MAX ? h[1] : -1;
  if (h[0] & EB_INCONSISTENT) return JT_ERR_INCONSISTENT_DIVISION;
  if (h[0] & EB_ZERO_MASS) return JT_ERR_ZERO_MASS;
  return JT_OK;
}

extern "C" int jt_error_case(const jt_state* st) { return st ? st->err_case : -1; }

extern "C" const char* jt_error_string(int code) {
  switch (code) {
    case JT_OK: return "ok";
    case JT_ERR_BAD_ARG: return "bad argument";
    case JT_ERR_INCONSISTENT_DIVISION: return "separator entry is zero but its fresh marginal is not";
    case JT_ERR_ZERO_MASS: return "cannot normalize a zero-mass table";
    case JT_ERR_CUDA: return cudaGetErrorString(last_cuda_error());
    case JT_ERR_OOM: return "device out of memory";
    case JT_ERR_UNSUPPORTED: return "unsupported configuration";
    default: return "unknown error";
  }
}

extern "C" int jt_plan_mapping_table(const jt_plan* p, int clique, int sep, int64_t* out_host) {
  if (!p || !out_host || clique < 0 || clique >= p->n_cliques || sep < 0 || sep >= p->n_seps) return JT_ERR_BAD_ARG;
  const auto& cv = p->cvars[clique];
  const auto& sv = p->svars[sep];
  for (int v : sv)
    if (!std::binary_search(cv.begin(), cv.end(), v)) return JT_ERR_BAD_ARG;
  DevGuard g(p->device);
  std::vector<int64_t> stride(cv.size(), 1);
  for (int i = (int)cv.size() - 2; i >= 0; --i) stride[i] = stride[i + 1] * p->cards[cv[i + 1]];
  std::vector<int64_t> sc, ss, rc_, rs;
  for (int v : sv) {  // separator order (compiler.py:294-299)
    const int pos = (int)(std::find(cv.begin(), cv.end(), v) - cv.begin());
    sc.push_back(p->cards[v]);
    ss.push_back(stride[pos]);
  }
  for (size_t i = 0; i < cv.size(); ++i)  // remaining positions ascending (288-292)
    if (!std::binary_search(sv.begin(), sv.end(), cv[i])) {
      rc_.push_back(p->cards[cv[i]]);
      rs.push_back(stride[i]);
    }
  const int64_t n_sep = p->ssize[sep], n_rest = p->csize[clique] / std::max<int64_t>(1, p->ssize[sep]);
  int64_t* d = nullptr;
  CK(cudaMalloc(&d, std::max<int64_t>(1, n_sep * n_rest) * sizeof(int64_t)));
  cudaError_t e = launch_mapping_table(d, n_sep, n_rest, (int)sc.size(), sc.data(), ss.data(), (int)rc_.size(),
                                       rc_.data(), rs.data(), nullptr);
  if (e == cudaSuccess) e = cudaMemcpy(out_host, d, n_sep * n_rest * sizeof(int64_t), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) {
    last_cuda_error() = e;
    return JT_ERR_CUDA;
  }
  return JT_OK;
}

// engine protocol: one message on host arrays through device buffers
struct MuScratch {
  int device = -1;
  void* buf = nullptr;
  size_t cap = 0;
  int* err = nullptr;
  cudaStream_t s = nullptr;
};

extern "C" int jt_run_message_mu(const double* phi_src, int64_t n_src, double* phi_tgt, int64_t n_tgt, double* phi_sep,
                                 int64_t n_sep, const void* mu_src, int64_t row_src, const void* mu_tgt,
                                 int64_t row_tgt, int mu_is_int64, int device) {
  if (!phi_src || !phi_tgt || !phi_sep || !mu_src || !mu_tgt || n_sep < 0 || row_src < 0 || row_tgt < 0)
    return JT_ERR_BAD_ARG;
  if (n_sep * row_src != n_src || n_sep * row_tgt != n_tgt) return JT_ERR_BAD_ARG;
  static std::mutex mtx;
  static std::map<int, MuScratch> scratch;
  std::lock_guard<std::mutex> lock(mtx);
  DevGuard g(device);
  MuScratch& m = scratch[device];
  const size_t isz = mu_is_int64 ? 8 : 4;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t need = al(n_src * 8) + al(n_tgt * 8) + al(n_sep * 8) * 2 + al(n_src * isz) + al(n_tgt * isz) + 256;
  if (!m.s) {
    CK(cudaStreamCreateWithFlags(&m.s, cudaStreamNonBlocking));
    CK(cudaMalloc(&m.err, sizeof(int)));
  }
  if (need > m.cap) {
    cudaFree(m.buf);
    m.buf = nullptr;
    m.cap = 0;
    CK(cudaMalloc(&m.buf, need));
    m.cap = need;
  }
  char* b = (char*)m.buf;
  double* d_src = (double*)b; b += al(n_src * 8);
  double* d_tgt = (double*)b; b += al(n_tgt * 8);
  double* d_sep = (double*)b; b += al(n_sep * 8);
  double* d_ratio = (double*)b; b += al(n_sep * 8);
  void* d_mus = b; b += al(n_src * isz);
  void* d_mut = b;
  cudaStream_t s = m.s;
  CK(cudaMemsetAsync(m.err, 0, sizeof(int), s));
  CK(cudaMemcpyAsync(d_src, phi_src, n_src * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_sep, phi_sep, n_sep * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_mus, mu_src, n_src * isz, cudaMemcpyHostToDevice, s));
  CK(launch_mu_message(d_src, nullptr, d_sep, d_ratio, d_mus, row_src, nullptr, row_tgt, n_sep, mu_is_int64, m.err, 0, s));
  int herr = 0;
  CK(cudaMemcpyAsync(&herr, m.err, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (herr & EB_INCONSISTENT) return JT_ERR_INCONSISTENT_DIVISION;  // nothing written back
  CK(cudaMemcpyAsync(d_tgt, phi_tgt, n_tgt * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_mut, mu_tgt, n_tgt * isz, cudaMemcpyHostToDevice, s));
  CK(launch_mu_message(nullptr, d_tgt, d_sep, d_ratio, nullptr, row_src, d_mut, row_tgt, n_sep, mu_is_int64, m.err, 1, s));
  CK(cudaMemcpyAsync(phi_tgt, d_tgt, n_tgt * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(phi_sep, d_sep, n_sep * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return JT_OK;
}

extern "C" const char* jt_version(void) { return "libjtb200 0.1 sm_100a"; }

// ----------------------------------------------------------------- debug --
// Host-only: compile the propagation program of a (plan, batch, mode) without
// touching a device and describe every wave/pass.  kind 0: jt_propagate;
// kind 1: jt_propagate_query over all variables with every variable observed
// (the batch program); kind 2: jt_propagate on a freshly reset state.  Used by tools/plan_report.py and the CPU tests.
extern "C" int jt_debug_plan(const jt_plan* plan, int batch, int mode, int kind, int num_sms, int occ,
                             char* buf, int64_t len) {
  if (!plan || !buf || len <= 0 || batch < 1) return JT_ERR_BAD_ARG;
  jt_state st;
  st.plan = plan;
  st.B = padded_batch(plan, batch);
  st.B_user = batch;
  st.mode = mode;
  st.num_sms = num_sms > 0 ? num_sms : 148;
  layout_state(&st);
  if (mode == JT_SHARED_BASE) st.h_base.assign(st.n_base, 1.0);  // W values do not matter here
  std::vector<int> qv;
  if (kind == 1) {
    for (int v = 0; v < plan->n_vars; ++v) {
      qv.push_back(v);
      if (mode == JT_SHARED_BASE) st.ev_clique[v] = smallest_holder(plan, v);
    }
  }
  std::vector<std::vector<PassSpec>> waves;
  int rc = JT_OK;
  {
    // as the runtime does: clique product X and virtual separators, else plainer programs
    const bool hx = env_int("JT_HUBX", 1) != 0;
    const bool attempts[3][2] = {{hx, true}, {hx, false}, {false, false}};
    for (int a = 0; a < 3; ++a) {
      if ((rc = build_propagate(&st, plan->roots, qv, waves, kind >= 1, attempts[a][0], attempts[a][1]))) return rc;
      if ((rc = validate_waves(&st, waves))) return rc;
      HostProgram probe;
      if (compile_program(&st, waves, probe, occ > 0 ? occ : 2) != JT_ERR_UNSUPPORTED) break;
    }
  }
  HostProgram hp;
  std::vector<std::vector<char>> tmask;
  std::vector<TPass> tp;
  std::vector<TinyWave> tw;
  bool tiny = tiny_masks(&st, waves, tmask);
  if (tiny && (build_tiny(&st, waves, tmask, tp, tw) != JT_OK || tp.empty())) tiny = false;
  rc = compile_program(&st, waves, hp, occ > 0 ? occ : 2, tiny ? &tmask : nullptr);
  if (rc) return rc;
  std::string out;
  char line[512];
  if (tiny) {
    {
      int64_t warp_passes = 0, threads = 0;
      for (auto& x : tp) warp_passes += x.warp > 1;
      for (auto& x : tw) threads += x.n_threads;
      int64_t nt = 0;
      for (auto& x : tw) nt += x.n_passes > 0;
      snprintf(line, sizeof line, "tiny passes (mode %d): %lld of %zu waves, %zu passes (%lld with several lanes per "
               "entry), %lld threads over all waves\n", tiny_mode(), (long long)nt, tw.size(), tp.size(),
               (long long)warp_passes, (long long)threads);
      out += line;
    }
  }
  {
    // compulsory HBM traffic per wave: every factor tensor read once, outputs
    // written once (separator updates also read the old values and write ratios)
    double tot = 0.0;
    for (size_t w = 0; w < waves.size(); ++w) {
      double bytes = 0.0;
      // paired row-per-i siblings read their shared (K-sum) factors once
      const std::vector<int> partner = pair_specs(&st, waves[w]);
      for (size_t a = 0; a < waves[w].size(); ++a) {
        const int b = partner[a];
        if (b < 0 || b < (int)a) continue;
        // a tensor the paired pass reads for both outputs (a shared factor, or one
        // output's old separator that is the other's factor) comes from DRAM once
        const auto& A = waves[w][a];
        const auto& Bp = waves[w][b];
        auto nbytes = [&](const Tensor& t) {
          double n = t.batch ? (double)st.B : 1.0;
          for (int v : t.vars) n *= plan->cards[v];
          return n * st.esz;
        };
        auto same = [](const Tensor& x, const Tensor& y) { return x.off == y.off && x.vars == y.vars; };
        for (auto& f : Bp.factors) {
          bool dup = same(f, A.out);
          for (auto& g : A.factors) dup = dup || same(g, f);
          if (dup && f.vclique < 0) bytes -= nbytes(f);
        }
        for (auto& g : A.factors)
          if (same(g, Bp.out) && g.vclique < 0) bytes -= nbytes(g);
      }
      for (auto& ps : waves[w]) {
        auto tsize = [&](const Tensor& t) {
          double n = t.batch ? (double)st.B : 1.0;
          for (int v : t.vars) n *= plan->cards[v];
          return n;
        };
        for (auto& f : ps.factors) bytes += f.vclique >= 0 ? 0.0 : tsize(f) * st.esz;
        if (ps.out_kind == OUT_RAW) bytes += tsize(ps.out) * 8;
        else if (ps.out_kind == OUT_SEP_FRESH) bytes += tsize(ps.out) * st.esz;
        else if (ps.out_kind == OUT_SEP_DFRESH && ps.skip_out2 && ps.x_off < 0 && env_int("JT_DRATIO", 1))
          bytes += tsize(ps.out) * st.esz;  // ratio only (OUT_SEP_DRATIO)
        else if (ps.out_kind != OUT_NONE)
          bytes += tsize(ps.out) * st.esz * (3 - (ps.out.vclique >= 0) - (ps.skip_out2 && ps.out_kind == OUT_SEP_DFRESH));
        const double csz = (double)plan->csize[ps.clique] * (ps.src_arena == A_BASE ? 1.0 : (double)st.B);
        if (ps.scope.empty()) bytes += csz * st.esz * (ps.write ? 2 : 1);
        if (ps.x_off >= 0) bytes += tsize(ps.out) * st.esz;  // the clique product X
        if (getenv("JT_DEBUG_SPECS")) {
          double fb = 0.0;
          for (auto &f : ps.factors) fb += f.vclique >= 0 ? 0.0 : tsize(f) * st.esz;
          int nvs = ps.out.vclique >= 0;
          for (auto& f : ps.factors) nvs += f.vclique >= 0;
          snprintf(line, sizeof line, "  spec w%zu clique %d src %d out %d nf %zu factors MB %.1f out MB %.1f vsep %d\n", w,
                   ps.clique, ps.src_arena, ps.out_kind, ps.factors.size(), fb / 1e6,
                   ps.out_kind != OUT_NONE ? tsize(ps.out) * st.esz / 1e6 : 0.0, nvs);
          out += line;
        }
      }
      tot += bytes;
      snprintf(line, sizeof line, "compulsory wave %zu MB %.1f\n", w, bytes / 1e6);
      out += line;
    }
    snprintf(line, sizeof line, "compulsory total MB %.1f\n", tot / 1e6);
    out += line;
  }
  for (size_t w = 0; w < hp.waves.size(); ++w) {
    const WaveRt& rt = hp.waves[w];
    snprintf(line, sizeof line, "wave %zu items %d launches %zu:", w, rt.n_items, rt.groups.size());
    out += line;
    for (const LaunchGrp& g : rt.groups) {
      if (g.kind == 3)
        snprintf(line, sizeof line, " [contract passes %d units %lld grid %d%s]", g.n_cpasses, (long long)g.n_units,
                 g.grid, g.interleave ? " interleaved" : "");
      else
        snprintf(line, sizeof line, " [%s vec %d items %d grid %d]", g.kind == 1 ? "own" : g.kind == 2 ? "row" : "gen",
                 g.vec, g.n_items, g.grid);
      out += line;
    }
    out += "\n";
    const int64_t pe = (w + 1 < hp.waves.size()) ? hp.waves[w + 1].pass_base : (int64_t)hp.passes.size();
    for (int64_t pi = rt.pass_base; pi < pe; ++pi) {
      const DevPass& d = hp.passes[pi];
      int64_t n_items = 0, n_out = 0;
      for (int64_t i = rt.item_base; i < rt.item_base + rt.n_items; ++i)
        if (hp.items[i].pass == pi - rt.pass_base) {
          ++n_items;
          if (hp.items[i].chunk == 0) n_out += hp.items[i].j_count;
        }
      snprintf(line, sizeof line,
               "  pass clique %d src %d nf %d wr %d out %d T %d n_in %d n_out %lld r_out %lld BPI %d chunks %d "
               "bpc %lld items %lld ndi %d own %d/%d row %d gpi %d ffac %x part %lld\n",
               hp.pass_clique[pi], d.src_arena, d.nf, d.dst_off >= 0, d.out_kind, d.T, d.n_in, (long long)n_out,
               (long long)d.n_blocks_per_jout, d.BPI, d.n_chunks, (long long)d.blocks_per_chunk,
               (long long)n_items, d.ndi, d.own, d.own_m, d.row, d.gpi, d.flush_fac,
               (long long)(d.n_chunks > 1 && d.out_kind ? n_out * d.n_chunks * d.n_in : 0));
      out += line;
    }
    for (const LaunchGrp& g : rt.groups) {
      if (g.kind != 3) continue;
      for (int q = 0; q < g.n_cpasses; ++q) {
        const CPass& c = hp.cpasses[g.cpass_off + q];
        snprintf(line, sizeof line,
                 "  contract clique %d out %d nI %d nS %d nK %d nG %d nE %d units %lld rowi %d ks %d igs %d gI-dep",
                 hp.cpass_clique[g.cpass_off + q], c.out_kind, c.nI, c.nS, c.nK, c.nG, c.nE, (long long)c.n_units,
                 c.rowi, c.nKS, c.igs);
        out += line;
        for (int gg = 0; gg < c.nG; ++gg) {  // does factor gg depend on i?
          bool dep = false;
          for (int ii = 1; ii < c.nI && !dep; ++ii) dep = hp.ctab[c.ti_off + ii * (c.nG + c.nE + 1) + gg] != 0;
          out += dep ? " 1" : " 0";
        }
        out += "\n";
      }
    }
  }
  const int64_t n = std::min<int64_t>((int64_t)out.size(), len - 1);
  memcpy(buf, out.data(), n);
  buf[n] = 0;
  return (int64_t)out.size() < len ? JT_OK : JT_ERR_BAD_ARG;
}
