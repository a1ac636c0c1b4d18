/* C ABI of the B200 ACOPF callback evaluator (libacopf_b200.so).
 *
 * Drop-in boundary for the reference's callback path.  The
 * reference binds these callbacks through Python (`opfkit.nlp.NlpProblem`,
 * pkg/src/opfkit/nlp.py:26-49); the Python package in this repo binds this
 * header through ctypes and rebuilds the same NlpProblem, and INTEGRATION.md
 * shows the equivalent ctypes stub a maintainer would add to opfkit.
 *
 * Entry point -> reference interface it replaces:
 *   acopf_topo_create      _Engine.__init__ packing + _build_patterns   (acopf.py:77-195)
 *   acopf_batch_create     composer._Builder.assemble: build_acopf per stage (composer.py:199-203)
 *   acopf_batch_stage_sizes  NlpProblem.n/m_eq/m_ineq + nnz of each stage (acopf.py:392-410)
 *   acopf_batch_set_layout   composite offsets, coupling rows        (composer.py:206-242)
 *   acopf_batch_eval       objective/gradient/constraints/jacobian/lagrangian_hessian
 *                          of every stage at once, device buffers     (acopf.py:266-373,
 *                                                                     composer.py:256-311)
 *   acopf_batch_eval_host  same with host buffers (H2D + eval + D2H on the handle's stream)
 *   acopf_batch_flows      per-branch flows and per-bus network injections of every stage
 *                          (pu) -- the device half of extract_solution / residuals_at /
 *                          solution_from_case                        (acopf.py:448-546, 230-264)
 *   acopf_batch_pattern    CSR indptr/indices of J or H (stage or composite) -- the fixed
 *                          pattern scipy would produce (acopf.py:308-311, 370-373)
 *   acopf_multi_create / acopf_batch_eval_multi   the sharded evaluation over GPUs with the
 *                          NCCL communicator inside (EMPAR pool analogue, runner.py:305-312)
 *   acopf_format_matrix    MATPOWER text of a solved stage's matrices   (matpower.py:151-190)
 *   acopf_last_error       error text (Python raises DeviceError / Disconnected ...)
 *
 * Conventions: plain pointers and sizes, no exceptions across the ABI.  Every
 * function returns 0 on success and nonzero on failure; the message is in
 * acopf_last_error() (thread-local).  Device pointers are CUDA global memory on
 * the handle's device.  Evaluation is stream-ordered on the given stream
 * (NULL = the legacy default stream, CUDA's convention; torch's default
 * stream is that stream); one handle must not be evaluated concurrently from
 * two streams or two host threads (it owns one objective scratch buffer, the
 * host-evaluation staging buffers and their graphs); callers serialise per
 * handle (the Python layer holds a lock).
 */
#ifndef ACOPF_B200_H
#define ACOPF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct acopf_topo acopf_topo;
typedef struct acopf_batch acopf_batch;

/* what-mask bits for acopf_batch_eval */
#define ACOPF_OBJ 1u
#define ACOPF_GRAD 2u
#define ACOPF_CONS 4u
#define ACOPF_JAC 8u
#define ACOPF_HESS 16u
#define ACOPF_ALL 31u

/* objective modes for acopf_batch_set_layout */
#define ACOPF_OBJ_PER_STAGE 0   /* obj[slot_s] = f_s (independent points)            */
#define ACOPF_OBJ_WEIGHTED 1    /* obj[0] = ((0 + w_0 f_0) + w_1 f_1) + ... (composite) */
#define ACOPF_OBJ_TERMS 2       /* obj[slot_s] = w_s f_s, summed by the caller (sharded) */

const char* acopf_last_error(void);
int acopf_version(void);

/* One packed topology (active buses, live branches and generators) in the
 * reference's per-unit conventions.  fo/to: bus slots per live branch; adm:
 * 8 doubles per branch (gff, bff, gft, bft, gtf, btf, gtt, btt), branch-major;
 * rated: 1 when rate_a > 0; gbus: bus slot per live generator; gs/bs: per unit. */
int acopf_topo_create(int32_t nb, int32_t nbr, int32_t ng, const int32_t* fo, const int32_t* to,
                      const double* adm, const uint8_t* rated, const int32_t* gbus,
                      const double* gs, const double* bs, acopf_topo** out);
int acopf_topo_destroy(acopf_topo* t);

/* A batch of stages on one device.  Stage s uses topology stage_topo[s] minus
 * the branches removed_idx[removed_ptr[s] .. removed_ptr[s+1]) (topology-local
 * branch indices), loads set stage_load[s] (pd/qd, nb values each, at
 * load_off[set]) and cost set stage_cost[s] (ca/cb/cc, ng values each, at
 * cost_off[set]), objective weight weight[s]. */
int acopf_batch_create(int32_t device, int32_t n_topos, acopf_topo* const* topos, int32_t n_stages,
                       const int32_t* stage_topo, const int64_t* removed_ptr, const int32_t* removed_idx,
                       const int32_t* stage_load, const int64_t* load_off, int64_t n_load_values,
                       const double* pd, const double* qd, const int32_t* stage_cost,
                       const int64_t* cost_off, int64_t n_cost_values, const double* ca,
                       const double* cb, const double* cc, const double* weight, acopf_batch** out);
int acopf_batch_destroy(acopf_batch* b);

/* Per stage, 6 values: n, m_eq, m_ineq, nnz of the J equality rows, nnz of the
 * J inequality rows, nnz of H. */
int acopf_batch_stage_sizes(const acopf_batch* b, int64_t* out6);

/* Output placement of every stage inside the caller's flat buffers (6 int64
 * per stage: var_off, eq_row, ineq_row, jeq_base, jineq_base, h_base), the
 * objective mode and slots, and the coupling rows: cons row, position of the
 * row's 2 J values, x index of the child (a) and base (b) quantity, and
 * whether the base column sorts first (J values -1, +1) or not (+1, -1). */
int acopf_batch_set_layout(acopf_batch* b, const int64_t* offsets6, int32_t obj_mode,
                           const int32_t* obj_slot, int64_t n_coupling, const int64_t* cp_row,
                           const int64_t* cp_jpos, const int64_t* cp_a, const int64_t* cp_b,
                           const int8_t* cp_base_first);

/* Evaluate the requested callbacks of every stage at (x, obj_factor, mult).
 * Unrequested outputs may be NULL.  All pointers are device pointers. */
int acopf_batch_eval(acopf_batch* b, const double* x, double obj_factor, const double* mult,
                     uint32_t what, double* obj, double* grad, double* cons, double* jval,
                     double* hval, void* stream);

/* Same, host pointers (pinned memory gives asynchronous copies); sizes of the
 * flat buffers in doubles.  Every requested output must be non-NULL with at
 * least the layout's size (x: the flat variable count, obj: 1 or the largest
 * objective slot + 1, cons: rows, jval / hval: values), and the Hessian needs
 * mult with at least the row count; otherwise the call fails before any copy.
 * Copies in, evaluates and copies out on `stream` (NULL = the handle's own
 * stream; its device buffers are internal), then synchronises that stream.
 * Layouts whose stages are contiguous and in order (independent points) are
 * pipelined in chunks over three streams; any other layout runs as one
 * H2D / evaluate / D2H sequence, which on the handle's own stream with pinned
 * host buffers is captured once per (what, sizes) as a CUDA graph and replayed
 * with its host pointers patched (ACOPF_HOST_GRAPHS=0 disables this). */
int acopf_batch_eval_host(acopf_batch* b, const double* x, int64_t nx, double obj_factor,
                          const double* mult, int64_t nm, uint32_t what, double* obj, int64_t nobj,
                          double* grad, int64_t ngrad, double* cons, int64_t ncons, double* jval,
                          int64_t nj, double* hval, int64_t nh, void* stream);

/* Branch flows and network injections of every stage at x (device pointers),
 * per-unit, exactly as Engine.first_order / Engine.injections compute them
 * (acopf.py:230-264).  Stage s (in batch order) owns
 *   flows[F_s + 0*nbr + k], [F_s + 1*nbr + k], [F_s + 2*nbr + k], [F_s + 3*nbr + k]
 *       = pf, qf, pt, qt of topology branch k (nbr = the stage topology's branches;
 *         F_s = sum over earlier stages of 4*nbr); branches a contingency removes
 *         are not written (the caller zero-fills);
 *   inj[I_s + i], inj[I_s + nb + i] = p, q of bus i, shunts included
 *       (I_s = sum over earlier stages of 2*nb).
 * Needs set_layout (x is read at each stage's var_off). */
int acopf_batch_flows(acopf_batch* b, const double* x, double* flows, double* inj, void* stream);

/* CSR pattern of one stage (stage >= 0; rows: that stage's constraints or
 * variables; columns stage-local) or of the whole laid-out batch (stage = -1,
 * needs set_layout; n_rows/n_cols are the flat sizes).  which: 0 = J, 1 = H.
 * indptr has rows+1 entries (int64), indices nnz entries (int32). */
int acopf_batch_pattern(const acopf_batch* b, int32_t stage, int32_t which, int64_t n_rows,
                        int64_t* indptr, int32_t* indices);

/* Host utility: the order in which one CSR row's COO terms (given by their
 * columns, in COO order) are visited after scipy's canonicalisation
 * (csr_sort_indices = std::sort on the column only).  perm[t] = COO index of
 * the t-th term; equal columns are adjacent and summed left to right.  Used by
 * the tests to pin the replay against scipy itself. */
int acopf_canonical_order(int64_t n, const int32_t* cols, int32_t* perm);

/* ---- multi-GPU: one process per GPU, a composite sharded into contiguous stage
 * blocks (the reference's EMPAR pool analogue, runner.py:305-312).
 * Each rank makes a batch of its own stages with a composite layout whose
 * coupling rows may read base-stage values owned by other ranks from a halo at
 * x[halo_dst0 ...], and objective mode ACOPF_OBJ_TERMS. */
typedef struct acopf_multi acopf_multi;

/* ncclGetUniqueId: rank 0 makes the 128-byte id, the caller broadcasts it. */
int acopf_nccl_unique_id(void* id128);

/* The exchange plan and (with nccl_id) the NCCL communicator, made inside with
 * ncclCommInitRank (collective: every rank calls it).  x_lo/x_hi: every rank's
 * global x range; need_ptr (world+1) / need_idx: every rank's sorted global x
 * indices it reads from other ranks (the halo, in this rank's halo order);
 * halo_dst0: local x index of this rank's first halo value; obj_counts: stages
 * (objective terms) per rank.  nccl_id NULL makes a plan-only handle (host,
 * acopf_multi_plan).  The batch must stay alive while the handle is used. */
int acopf_multi_create(acopf_batch* b, int32_t rank, int32_t world, const int64_t* x_lo, const int64_t* x_hi,
                       const int64_t* need_ptr, const int64_t* need_idx, int64_t halo_dst0,
                       const int32_t* obj_counts, const void* nccl_id, acopf_multi** out);

/* Host view of the plan: sizes3 = (exports, export slots per rank, halo values);
 * export_idx = local x indices this rank sends; halo_src = position of each halo
 * value in the gathered [world][export slots] buffer (either may be NULL). */
int acopf_multi_plan(const acopf_multi* m, int64_t* sizes3, int64_t* export_idx, int64_t* halo_src);
int acopf_multi_destroy(acopf_multi* m);

/* One sharded evaluation on this rank (device pointers, stream-ordered on
 * `stream`, NULL = legacy default stream): the halo chain (pack kernel ->
 * ncclAllGather -> unpack kernel -> coupling rows) runs on a forked stream and
 * overlaps the tile kernel; every rank's w_s f_s terms are all-gathered and
 * summed in global stage order on the device into obj[0] (bit-identical to one
 * GPU).  x must hold the halo slots (it is written there); outputs are this
 * rank's local blocks in its layout. */
int acopf_batch_eval_multi(acopf_multi* m, double* x, double obj_factor, const double* mult, uint32_t what,
                           double* obj, double* grad, double* cons, double* jval, double* hval, void* stream);

/* The reference IPM's Newton matrix on the device (ipm.py:463-477, 173-189), dense,
 * K = [[0.5 (Hfull + Hfull^T) + reg I, Je^T], [Je, -delta I]]
 * with Hfull = H + diag(dx) + Ji^T diag(ds) Ji over the nf free variables, from
 * device J / H value arrays (jval / hval of acopf_batch_eval) and device index
 * structures: H as CSR over free rows (h_ptr nf+1, free column h_col, value index
 * h_vi), Ji as CSC over free columns (jt_*: inequality row, value index) and as CSR
 * over inequality rows (ji_*: free column, value index), Je as CSR over equality
 * rows (je_*); sc_e / sc_i: the reference view's row scales s_c of the equality and
 * inequality rows (NULL = 1).  K must hold (nf+me)^2 zeros; both triangles are
 * written.  Deterministic (no atomics). */
int acopf_kkt_assemble(int64_t nf, int64_t me, double* K, const int64_t* h_ptr, const int32_t* h_col,
                       const int64_t* h_vi, const double* hval, const double* dx, const int64_t* jt_ptr,
                       const int32_t* jt_row, const int64_t* jt_vi, const int64_t* ji_ptr, const int32_t* ji_col,
                       const int64_t* ji_vi, const double* jval, const double* ds, const int64_t* je_ptr,
                       const int32_t* je_col, const int64_t* je_vi, const double* sc_e, const double* sc_i,
                       double reg, double delta, void* stream);

/* Host graph utilities of the composite builder (network.py:232-262, 339-344):
 * islands of the in-service network over buses with alive[v] != 0 (edges with an
 * endpoint not alive are ignored; edge_live may be NULL = all), labels in the
 * order of their first bus, -1 for buses not alive; and the bridges of the live
 * multigraph (a parallel twin is not a bridge), is_bridge[k] per edge. */
int acopf_graph_islands(int32_t nbus, const uint8_t* alive, int64_t nedge, const int32_t* ea, const int32_t* eb,
                        const uint8_t* edge_live, int32_t* n_islands, int32_t* label);
int acopf_graph_bridges(int32_t nbus, int64_t nedge, const int32_t* ea, const int32_t* eb, const uint8_t* edge_live,
                        uint8_t* is_bridge);

/* Host utility of the composite builder: dst[dst_off[i] ..+ len[i]) = src[src_off[i] ..+ len[i])
 * for i < n, on the host cores (the per-stage bound blocks of composer.py:244-251). */
int acopf_copy_runs(int64_t n, double* dst, const int64_t* dst_off, const double* src, const int64_t* src_off,
                    const int64_t* len);

/* MATPOWER text of one matrix section of a solved stage (the reference's
 * matpower._fmt_matrix, matpower.py:151-157): "mpc.<section> = [", one line
 * per row ("\t" + the row's values as "%.10g" joined by "\t" + ";"), "];",
 * lines joined by "\n".  Row r holds values[row_ptr[r] .. row_ptr[r+1]).
 * Writes at most cap bytes to out (no terminating NUL); *len receives the
 * text's length (out may be NULL to size it).  Host only, thread-safe. */
int acopf_format_matrix(const char* section, int64_t rows, const int64_t* row_ptr, const double* values,
                        char* out, int64_t cap, int64_t* len);

/* Kernel launches issued by this handle since creation (evidence counter). */
int64_t acopf_batch_launches(const acopf_batch* b);

/* Host check of every tile table of the batch (planner invariants, no GPU):
 * each staging position and each round term slot has exactly one producer
 * (an end or bus store, a constant, or a sum), padding slots hold -0.0, and
 * all locations lie inside the tile's area.  stats (may be NULL) receives 12
 * values: tables, tiles of the base topologies, branch ends in base tiles,
 * area doubles (sum over tables), -0.0 padding slots (sum), largest tile CTA
 * shared memory in bytes, sum rounds, round lane-terms (sum of terms x width),
 * round chain terms (sum of terms per round), and the modeled shared-memory
 * wavefronts of one stage's area stores over all tables (half-warp model,
 * whole-warp model, conflict-free ideal).  Returns nonzero with acopf_last_error() on the
 * first violation. */
int acopf_batch_verify(const acopf_batch* b, int64_t* stats);

#ifdef __cplusplus
}
#endif
#endif
