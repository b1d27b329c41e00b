/*
 * jt_b200.h — C ABI of the B200 junction-tree propagation engine (libjtb200.so).
 *
 * The reference (`jtprop`, pure Python/numpy) has no native boundary; its
 * plug-in seams are:
 *   - the duck-typed engine protocol `run_message(phi_src, phi_tgt, phi_sep,
 *     mu_src, mu_tgt)` (propagate.py:79-161), replaced by jt_run_message_mu;
 *   - the functional API initialize / from_potentials / apply_evidence /
 *     message_passing / belief_propagation / query_marginal
 *     (propagate.py:204-390), replaced by the plan/state calls below.
 * Every entry point names the reference function it stands in for.
 *
 * Conventions: host buffers are caller-owned and copied during the call;
 * handles are library-owned; a state is bound to one device and is not
 * thread-safe; `stream` may be NULL (the state's own stream) or a
 * cudaStream_t.  Every call returns a JT_* code; kernels record data errors
 * (0/0 vs nonzero/0, zero mass) in a device error word read by jt_sync_error.
 * Tables are flat, C order, LAST scope variable fastest (potential.py:50-55);
 * clique and separator member lists are ascending variable ids
 * (compiler.py:28, 204).  Batched states store case b of every table as the
 * innermost (stride-1) index.
 */
#ifndef JT_B200_H
#define JT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct jt_plan jt_plan;
typedef struct jt_state jt_state;

enum {
  JT_OK = 0,
  JT_ERR_BAD_ARG = 1,
  JT_ERR_INCONSISTENT_DIVISION = 2, /* errors.py:114 InconsistentDivisionError */
  JT_ERR_ZERO_MASS = 3,             /* errors.py:98  ZeroMassError */
  JT_ERR_CUDA = 4,
  JT_ERR_OOM = 5,
  JT_ERR_UNSUPPORTED = 6
};
enum { JT_F32 = 0, JT_F64 = 1 };
/* state modes */
enum {
  JT_MATERIALIZED = 0, /* every case owns its clique tables in HBM (reference semantics) */
  JT_SHARED_BASE = 1   /* one base replica shared by all cases; evidence and messages
                          enter as factors, clique tables are never written (batch API) */
};

/* Tree structure; replaces handing a `JunctionTree` (compiler.py:40-80) to the
 * engine.  CSR member lists; sep_edge holds (lower id, higher id) per separator;
 * neighbors are derived (sorted by clique id, compiler.py:228-229). */
int jt_plan_create(int n_vars, const int32_t* cards,
                   int n_cliques, const int32_t* clique_off, const int32_t* clique_vars,
                   int n_seps, const int32_t* sep_edge, const int32_t* sep_off,
                   const int32_t* sep_vars, int n_roots, const int32_t* roots,
                   int dtype, int device, jt_plan** out);
void jt_plan_destroy(jt_plan* plan);

/* Device-built μ table (|φ_s| × |φ_c|/|φ_s|, C order) for (clique, sep);
 * bit-exact with build_mapping_table (compiler.py:285-304). */
int jt_plan_mapping_table(const jt_plan* plan, int clique, int sep, int64_t* out_host);

/* State = potential store (PropagationState, propagate.py:172-201).
 * batch >= 1 evidence cases; mode JT_MATERIALIZED or JT_SHARED_BASE. */
int jt_state_create(const jt_plan* plan, int batch, int mode, jt_state** out);
void jt_state_destroy(jt_state* st);
int64_t jt_state_device_bytes(const jt_state* st);

/* from_potentials (propagate.py:225-240): clique tables concatenated in clique-id
 * order (Σ|φ_c| doubles); sep tables likewise or NULL for all-ones.
 * case_idx = -1 broadcasts to every case (and, in shared mode, loads the base). */
int jt_state_load(jt_state* st, int case_idx, const double* clique_concat,
                  const double* sep_concat);
/* initialize (propagate.py:204-222) on the device: every clique's base table
 * becomes the product of the CPTs assigned to it (ones when none), then every
 * case is reset to it (separators ones, no evidence).  CPT k belongs to clique
 * cpt_clique[k] (tree.cpt_assignment[child]); its variables are
 * cpt_vars[cpt_off[k] .. cpt_off[k+1]) in the CPT table's own axis order (C order,
 * last fastest; potential.py:50-55) and its values follow in cpt_values. */
int jt_state_initialize(jt_state* st, int n_cpts, const int32_t* cpt_clique, const int32_t* cpt_off,
                        const int32_t* cpt_vars, const double* cpt_values);
/* Restore every case to the loaded base tables (clique tables from the base
 * replica, separators to ones) and drop all evidence: PropagationState.copy()
 * of a template state (cli.py:194-201), done on device for the whole batch. */
int jt_state_reset(jt_state* st, void* stream);
/* PropagationState.copy() (propagate.py:193-201) on the device: a new state over
 * the same plan, batch and mode whose arenas, separator roles and evidence are a
 * device-to-device copy of src. */
int jt_state_clone(jt_state* src, jt_state** out);
/* Read back one case (host views of state.clique_values / state.sep_values).
 * Shared-base states materialise the final tables of that case on the fly. */
int jt_state_store(jt_state* st, int case_idx, double* clique_concat, double* sep_concat);

/* apply_evidence (propagate.py:243-260): n observations (case, var, clique, state).
 * clique = owning clique (tree.cpt_assignment[var]).  case = -1 → every case. */
int jt_apply_evidence(jt_state* st, int n, const int32_t* case_idx, const int32_t* var,
                      const int32_t* clique, const int32_t* value, void* stream);
/* Same, with the observations already resident on the device: d_obs holds n
 * int32 triples (case, var, state); var/clique (host, n_vars entries) list every
 * variable observed in d_obs with its owning clique.  Asynchronous. */
int jt_apply_evidence_device(jt_state* st, int n, const int32_t* d_obs, int n_vars,
                             const int32_t* var, const int32_t* clique, void* stream);
/* Drop all evidence factors (shared-base mode: back to the bare base replica). */
int jt_clear_evidence(jt_state* st);

/* message_passing (propagate.py:263-274): one Hugin message src→tgt over sep,
 * all cases (per-message compatibility path; materialized states only). */
int jt_message(jt_state* st, int src, int tgt, int sep, void* stream);

/* belief_propagation (propagate.py:337-360): full collect + distribute for every
 * component; roots_or_null overrides the per-component roots (n = plan's n_roots). */
int jt_propagate(jt_state* st, const int32_t* roots_or_null, void* stream);

/* query_marginal / posterior_marginals (propagate.py:363-390): n variables;
 * clique[i] = -1 picks the smallest holding clique (ties → lowest id).
 * out_host: [batch][Σ_i card(var_i)] doubles, normalized when normalize != 0. */
int jt_query(jt_state* st, int n, const int32_t* var, const int32_t* clique,
             int normalize, double* out_host, void* stream);
/* Same, writing into a device buffer (for NCCL gathers); does not synchronize. */
int jt_query_device(jt_state* st, int n, const int32_t* var, const int32_t* clique,
                    int normalize, double* out_device, void* stream);
/* Batch step for shared-base states: propagate + posteriors of n variables in
 * one fused program (queries ride in the distribute waves). */
int jt_propagate_query(jt_state* st, int n, const int32_t* var, int normalize,
                       double* out_device, void* stream);

/* Synchronize the stream, return and clear the device error word. */
int jt_sync_error(jt_state* st);
/* Lowest case index whose posterior had zero mass at the last jt_sync_error
 * that returned JT_ERR_ZERO_MASS, else -1 (the reference raises per case:
 * potential.py:181-186 via estimator.py:130-133). */
int jt_error_case(const jt_state* st);
const char* jt_error_string(int code);
/* Kernel launches issued by this state since creation (for bench accounting). */
int64_t jt_state_launch_count(const jt_state* st);

/* Engine protocol: SequentialEngine.run_message (propagate.py:79-94 → _pass_block
 * 56-76) on host float64 arrays with host μ tables (int32 or int64, C order).
 * Raises JT_ERR_INCONSISTENT_DIVISION before writing anything, like the
 * reference. */
int jt_run_message_mu(const double* phi_src, int64_t n_src, double* phi_tgt, int64_t n_tgt,
                      double* phi_sep, int64_t n_sep, const void* mu_src, int64_t row_src,
                      const void* mu_tgt, int64_t row_tgt, int mu_is_int64, int device);

/* Host-only planner report (no device needed): compiles the propagation
 * program for (batch, mode) — kind 0: jt_propagate, kind 1: the batch program
 * with posteriors of every variable — and writes one line per wave and pass. */
int jt_debug_plan(const jt_plan* plan, int batch, int mode, int kind, int num_sms, int occ,
                  char* buf, int64_t len);

/* Library build/version string. */
const char* jt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* JT_B200_H */
