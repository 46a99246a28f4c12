/* =============================================================================
 * toast.h — C ABI of the B200-native TOAST hot path (libtoast.so)
 *
 * What it computes: batched evaluation of MCTS rollouts over the sharding-
 * decision space of arXiv 2508.15010 ("TOAST"), /root/reference/PAPER.md
 * (cited as P:<line>).  For each candidate action sequence it materialises the
 * sharding, derives local FLOPs, inserts and costs the
 * implied collectives, runs the live-range sweep for peak memory
 * and returns runtime and score C(s) = RT(s) + MP(s).
 * The exact definitions are SURVEY.md §8(c) C0-C16 and DESIGN.md.
 *
 * Conventions (all calls):
 *   - Every call returns toast_status (0 = TOAST_OK) and never throws across
 *     the ABI; toast_last_error() returns a thread-local message valid until
 *     the next call on that thread.
 *   - Handles (toast_graph, toast_analysis, toast_search_state) are owned by
 *     the library and freed with the matching toast_free_* call.  Caller
 *     buffers are never freed or retained.
 *   - Candidate buffers (seqs, out, prefixes, out_seqs) may be host or device
 *     pointers.  Device pointers: the call is asynchronous on `cuda_stream`
 *     (a cudaStream_t, NULL = legacy default stream); the caller synchronises.
 *     Host pointers (pageable or pinned): the library copies through device
 *     scratch on `cuda_stream` and returns after the results are in host
 *     memory.  All buffers must use the same kind of memory.
 *   - Candidate-level problems never fail a call; they are reported in
 *     toast_cost.status with every other field zero.
 *   - A toast_analysis is immutable after toast_nda and safe for concurrent
 *     calls on different streams (host-pointer calls serialise on a mutex).
 * ============================================================================= */
#ifndef TOAST_H
#define TOAST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TOAST_OK = 0,
  TOAST_E_INVALID_ARG = 1,  /* NULL pointer, negative size, bad option value */
  TOAST_E_PARSE = 2,        /* syntax error; message holds "line:col: ..." */
  TOAST_E_SHAPE = 3,        /* shape/attribute mismatch; message names the binding */
  TOAST_E_UNDEFINED = 4,    /* use before definition */
  TOAST_E_DUPLICATE = 5,    /* a name bound twice */
  TOAST_E_MESH = 6,         /* duplicate axis name, size < 2, 0 or > 4 axes, bw <= 0 */
  TOAST_E_MACHINE = 7,      /* flops_per_sec <= 0, penalty_c < 0 */
  TOAST_E_DEGENERATE = 8,   /* baseline runtime 0: no contraction op */
  TOAST_E_LIMIT = 9,        /* > 8 SetGroups in a super-color, > 1023 actions, > 64 SetGroups,
                               > 8 loops or operands per op, rank > 8, > 2^31 loops */
  TOAST_E_CUDA = 10,        /* CUDA runtime error, or no device attached to the graph */
  TOAST_E_NCCL = 11,        /* reserved: collectives run in the caller (torch.distributed) */
  TOAST_E_OOM = 12          /* host or device allocation failed */
} toast_status;

/* candidate status bits (toast_cost.status) */
#define TOAST_ST_BAD_ACTION_ID 1u        /* an id >= number of actions */
#define TOAST_ST_DUP_COLOR_AXIS 2u       /* the same (super-color, axis) twice */
#define TOAST_ST_RES_MISMATCH 4u         /* a SetGroup bit disagrees with an earlier action's */
#define TOAST_ST_NONZERO_AFTER_STOP 8u   /* a nonzero entry after the first 0 (STOP) */

/* collective kinds, index of toast_cost.payload[axis][kind] */
#define TOAST_AG 0
#define TOAST_RS 1
#define TOAST_AR 2
#define TOAST_A2A 3

/* One mesh axis.  Mesh order = array order.  bytes_per_sec is
   the link bandwidth used by the ring cost model. */
typedef struct {
  const char* name;
  int32_t size;          /* >= 2 */
  double bytes_per_sec;  /* > 0 */
} toast_axis;

/* Machine characteristics: FLOP rate for matmul-class ops,
   per-device memory DM and penalty constant C of MP(s). */
typedef struct {
  double flops_per_sec;
  uint64_t device_memory_bytes;
  double penalty_c;
} toast_machine;

/* NDA options: prune super-colors with fewer than min_unique_dims value
   dims (default 10); maximum trajectory depth (default 30);
   cost_model: how runtime accumulates — TOAST_COST_SUM (0, reading
   G14: compute + every collective, straight-line) or TOAST_COST_CRITICAL_PATH
   (1, reading R22: the latest finish over the op DAG, finish(t) = max over
   operands of (finish(def) + the edge's collective time) + t's compute time).
   Every other record field is the same under both.
   conflict_grouping: how conflicts are grouped into sets whose resolution is
   decided together — TOAST_GROUP_COMPAT (0, §3.5: the closure of
   the "compatible conflicts" box relation) or
   TOAST_GROUP_CONTRACTION (1, the dimension-graph contraction heuristic of
   the [comment] block P:1346-1357, reading R23: eagerly contract
   M edges unless a directed path would join the two endpoints of a
   conflict; conflicts on the same pair of contracted nodes form one set).
   dedup ("any action sequence yielding the
   same sharded model resolves to the same unique state"): 0 = every
   candidate of a rollout launch is evaluated on its own; 1 = a rollout launch
   materialises every candidate (H1, H2, H3, H7), then costs each distinct
   materialised state once (H4-H6, and the critical path) and copies its
   record to the candidates that reached it — the same bits either way
   (states are compared exactly: equal state key AND equal per-class axis
   maps); 2 = on under TOAST_COST_CRITICAL_PATH (where the per-state walk
   dominates: 1.3-5x measured), off under TOAST_COST_SUM (where it depends on
   how often states repeat: 0.96x on GPT-24, 2.1x on U-Net).  Any other value
   of these three: TOAST_E_INVALID_ARG. */
enum { TOAST_COST_SUM = 0, TOAST_COST_CRITICAL_PATH = 1 };
enum { TOAST_GROUP_COMPAT = 0, TOAST_GROUP_CONTRACTION = 1 };
typedef struct {
  int32_t min_unique_dims;
  int32_t max_depth;
  int32_t cost_model;
  int32_t conflict_grouping;
  int32_t dedup;
} toast_nda_opts;

typedef struct toast_graph toast_graph;        /* opaque, library-owned */
typedef struct toast_analysis toast_analysis;  /* opaque, library-owned, immutable */

/* 256-byte cost record, one per candidate (16-byte aligned). */
typedef struct {
  double runtime_s;        /* C13: flops/F + sum over axes of ring collective time */
  double score;            /* RT + MP */
  uint64_t peak_bytes;     /* C12: max over program points of live device-local bytes */
  uint64_t flops;          /* C10: low 64 bits of the local matmul-class FLOP total */
  uint64_t state_key;      /* C14 (R14): sum over (op, axis A, role r holding A) of mix64(first loop << 8 | A << 4 | r) */
  uint32_t status;         /* TOAST_ST_* bits; 0 = ok */
  uint32_t n_collectives;  /* total number of collectives (count[][] saturates at 65535) */
  uint64_t payload[4][4];  /* C11 bytes per [axis][AG, RS, AR, A2A] */
  uint16_t count[4][4];    /* number of collectives per [axis][kind] */
  uint64_t flops_hi;       /* high 64 bits of the FLOP total */
  uint8_t pad[40];
} toast_cost;

/* action id -> (super-color, resolution bits r, axis index, #value dims). id 0 = STOP. */
typedef struct {
  int32_t super_color, resolution, axis, n_value_dims;
} toast_action_info;

/* ---------------------------------------------------------------------------
 * toast_load_graph — parse the text IR (SPEC grammar S:92-104
 * extended with dot_general/conv/gather/... ) and bind it to a mesh and
 * machine.  `ir_text` need not be NUL-terminated (`len` bytes are read).
 * `cuda_device` >= 0 selects the device the tables are uploaded to by
 * toast_nda; -1 builds a host-only graph (analysis and dumps only; eval calls
 * then fail with TOAST_E_CUDA).  On error *out is NULL.
 * ------------------------------------------------------------------------- */
toast_status toast_load_graph(const char* ir_text, size_t len, const toast_axis* axes, int32_t n_axes,
                              const toast_machine* m, int32_t cuda_device, toast_graph** out);

/* toast_nda — H0 (once per graph): loop table from the NDA rules (Fig. 3,
 * P:443-558), I∪M components, conflicts,
 * compatibility sets (§3.5), cross-layer SetGroups (§3.6),
 * argument groups / super-colors (§4.4), the action table
 * (§4.2) and the baseline cost; uploads the device tables.
 * `g` stays owned by the caller and may be freed after this call. */
toast_status toast_nda(const toast_graph* g, const toast_nda_opts* o, toast_analysis** out);

/* number of actions including STOP (id 0): the action table of §4.2 (
 * SURVEY §8(c) C8).  Errors: TOAST_E_INVALID_ARG (NULL). */
toast_status toast_num_actions(const toast_analysis* a, int32_t* n);
/* the action table (§4.2, C8): per action id (index; id 0 = STOP,
 * all -1 but n_value_dims 0) the super-color (§4.4), the
 * resolution bits over its SetGroups (§3.5-3.6), the mesh axis,
 * and the number of value dims of the super-color ("at least 10 unique
 * dimensions").  Fills up to cap entries (caller-owned host array); *n = the
 * number of actions.  Errors: TOAST_E_INVALID_ARG (NULL, or cap > 0 with out NULL). */
toast_status toast_query_actions(const toast_analysis* a, toast_action_info* out, int32_t cap, int32_t* n);
/* the empty sequence's record — the unsharded module at the root of the tree
 * (P:1418), whose runtime and peak are the normalisers t0 and peak0 of
 * RT / MP, so its RT = 1.  out: caller-owned host toast_cost.
 * Errors: TOAST_E_INVALID_ARG (NULL). */
toast_status toast_query_baseline(const toast_analysis* a, toast_cost* out);
/* candidates one full wave of the GPU evaluates at once (resident warps x 32);
 * batch sizes that are multiples of it leave no partially filled last wave
 * (the "many trajectories in parallel" of P:1400, sized for this GPU).
 * Errors: TOAST_E_INVALID_ARG (NULL); TOAST_E_CUDA for a host-only analysis. */
toast_status toast_preferred_batch(const toast_analysis* a, int64_t* n);
/* JSON dump of the H0 tables (loops with their Fig. 3 names' classes P:443-558,
 * conflicts P:743-746, compatibility sets P:924-946, SetGroups P:949-959,
 * super-colors P:1442-1449, actions P:1407-1417, baseline P:1461-1477) plus
 * "kernel_tables": the sizes of the per-candidate tables the kernels read,
 * the dispatched kernel variant [mesh axes, power-of-two, cost model] and the
 * op index of every peak-memory frontier point (reading R19).
 * *needed = bytes incl. NUL; writes only if cap >= *needed (caller-owned host
 * buffer).  Errors: TOAST_E_INVALID_ARG (NULL). */
toast_status toast_dump_analysis(const toast_analysis* a, char* buf, size_t cap, size_t* needed);

/* toast_eval_batch — H1-H7 for n candidates.  seqs: uint16[n][32] action ids,
 * 0 = STOP; out: toast_cost[n]. */
toast_status toast_eval_batch(const toast_analysis* a, const uint16_t* seqs, int64_t n, toast_cost* out,
                              void* cuda_stream);

/* toast_rollout_batch — H8: from each prefix (uint16[n][32]),
 * extend with Philox4x32-10 draws (key = seed, counter = (id_base + i, depth))
 * until STOP (p = depth/max_depth), no legal action, or
 * max_depth; writes the sequence to out_seqs[n][32] and its cost to out[n].
 * A prefix with an invalid id or nonzero after STOP is returned unextended. */
toast_status toast_rollout_batch(const toast_analysis* a, const uint16_t* prefixes, int64_t n, uint64_t seed,
                                 uint64_t id_base, uint16_t* out_seqs, toast_cost* out, void* cuda_stream);

/* The search-facing result of one candidate, 16 B: the score C(s) = RT(s) +
 * MP(s) and the state key (reading R14) — what the
 * tree backs up and identifies states by.  Bit-identical to the `score` and
 * `state_key` of the full toast_cost record; a candidate whose record would
 * carry a nonzero status has score = NaN (0x7FF8000000000000) and state_key =
 * that status.  For callers that do not need the payload breakdown: a 16-B
 * record moves 1/16 of the bytes of toast_cost across PCIe on the host path. */
typedef struct {
  double score;
  uint64_t state_key;
} toast_score;

/* toast_eval_scores / toast_rollout_scores — toast_eval_batch /
 * toast_rollout_batch with toast_score[n] results (same computation, same
 * memory rules: all buffers host or all device; device pointers run
 * asynchronously on cuda_stream, host pointers synchronously). */
toast_status toast_eval_scores(const toast_analysis* a, const uint16_t* seqs, int64_t n, toast_score* out,
                               void* cuda_stream);
toast_status toast_rollout_scores(const toast_analysis* a, const uint16_t* prefixes, int64_t n, uint64_t seed,
                                  uint64_t id_base, uint16_t* out_seqs, toast_score* out, void* cuda_stream);

/* per-loop axis masks of one sequence (debug / tests; NEXT-1 lowering) — the
 * "attempt" materialisation of C9 (reading G1).
 * masks: uint8[cap]; *n = number of loops. seq is a host pointer.
 * Errors: TOAST_E_INVALID_ARG for NULL, or (when masks is written) for a
 * sequence the kernels' decode would flag (any TOAST_ST_* bit: an id >= the
 * action count, a repeated (super-color, axis), a resolution disagreeing with
 * an earlier fixed SetGroup bit, a nonzero id after STOP). */
toast_status toast_materialize(const toast_analysis* a, const uint16_t seq[32], uint8_t* masks, int64_t cap,
                               int64_t* n);

/* toast_lower — the device-local program one sequence implies (SURVEY §8(f)
 * NEXT-1): every value's local shape, layout (per dim, the mesh axes sharding
 * it) and partial axes, and in front of every use edge the collectives of the
 * cost model (C11: phase 1 all_to_all/all_gather, phase 2 reduce_scatter /
 * all_reduce, phase 3 local slice), each with the payload bytes the cost
 * model charges — the notation of Fig. 2c / Fig. 5b.
 * Text, one statement per line; format in DESIGN.md "Lowering" and
 * csrc/lower.cpp.  seq: host uint16[32] (0 = STOP).  *needed = bytes incl.
 * NUL; writes only if cap >= *needed.  Host-side (no GPU needed).
 * Errors: TOAST_E_INVALID_ARG (NULL, or a sequence the kernels' decode would
 * flag with any TOAST_ST_* bit — see toast_materialize). */
toast_status toast_lower(const toast_analysis* a, const uint16_t seq[32], char* buf, size_t cap, size_t* needed);

/* ---------------------------------------------------------------------------
 * Search (C16).  Single GPU: toast_search.  Root-parallel
 * multi-GPU: the caller drives begin / round / (all_gather of the export
 * bytes across ranks) / import / end, e.g. with torch.distributed (NCCL).
 * ------------------------------------------------------------------------- */
typedef struct {
  uint64_t seed;
  int64_t max_evals;        /* 0 = unlimited */
  double time_limit_s;      /* 0 = unlimited */
  int32_t leaves_per_round; /* L */
  int32_t rollouts_per_leaf;/* R */
  int32_t patience;         /* stop after this many non-improving rounds (1) */
  int32_t transpositions;   /* 0 = a tree of action sequences; 1 = each materialised state
                               once (reading R24): a selected leaf
                               whose exactly evaluated state another node already holds
                               (equal state key) leaves the tree after its round */
  double uct_c;             /* UCT exploration constant (sqrt 2) */
  double target_score;      /* stop once best <= target; NaN = disabled */
  void* cuda_stream;
} toast_search_opts;

typedef struct {
  uint16_t best_seq[32];
  toast_cost best;
  int64_t evals;
  int32_t rounds, hit_target;
  double wall_s, time_to_target_s; /* time_to_target_s < 0 if never reached */
} toast_search_result;

typedef struct toast_search_state toast_search_state;

/* The per-round record one rank contributes to the all-gather (host memory,
   toast_search_export_bytes() bytes).  Written by toast_search_round; the
   gathered array [world] is passed to toast_search_import on every rank. */
typedef struct {
  double best_score;       /* this rank's best score (after adopting the last global best) */
  uint64_t best_key;
  uint16_t best_seq[32];
  int64_t evals;           /* evaluations done by this rank so far */
  double elapsed_s;        /* this rank's wall clock since begin (rank 0's decides time limits) */
  int32_t rank;
  int32_t pad;
  toast_cost best;         /* full record of the rank's best */
} toast_search_export;
/* The export record is this header followed by one toast_root_stat per action
   id (index = action id, entry 0 unused): the rank's root-child visit count
   and reward sum (the ranks exchange best sequences AND visit
   statistics).  toast_search_import sums them over the ranks; read the sums
   with toast_search_root_stats. */
typedef struct {
  int64_t visits;
  double value_sum;
} toast_root_stat;

toast_status toast_search(const toast_analysis* a, const toast_search_opts* o, toast_search_result* out);

/* bytes one rank contributes to the per-round all_gather */
size_t toast_search_export_bytes(const toast_analysis* a);
/* seed of rank r = o->seed + r.  A host-only analysis (cuda_device = -1) may
   begin and import (the exchange logic is host code) but not run rounds. */
toast_status toast_search_begin(const toast_analysis* a, const toast_search_opts* o, int32_t rank, int32_t world,
                                toast_search_state** out);
/* runs one round on the GPU; writes this rank's toast_search_export to `export_buf` (host memory) */
toast_status toast_search_round(toast_search_state* s, void* export_buf);
/* imports world records ([world][export_bytes], host memory); *stop = 1 when all ranks must stop */
toast_status toast_search_import(toast_search_state* s, const void* gathered, int32_t* stop);
/* the same with the exchange in device memory: the round's
   record is copied to `export_dev` (device, toast_search_export_bytes()
   bytes) on `cuda_stream`, so an NCCL all-gather enqueued on that stream
   after the call reads it without a host round trip; `gathered_dev` (device,
   [world][export_bytes]) is read back on `cuda_stream` and imported.  Both
   return once their copy is complete.  Errors: TOAST_E_INVALID_ARG (NULL, a
   host pointer), TOAST_E_CUDA. */
toast_status toast_search_round_dev(toast_search_state* s, void* export_dev, void* cuda_stream);
toast_status toast_search_import_dev(toast_search_state* s, const void* gathered_dev, int32_t* stop, void* cuda_stream);
toast_status toast_search_end(toast_search_state* s, toast_search_result* out);
/* root-child statistics summed over the ranks at the last import (index =
   action id; visits 0 = the child is not expanded on any rank).  out: cap
   entries; *n = number of actions. */
toast_status toast_search_root_stats(const toast_search_state* s, toast_root_stat* out, int32_t cap, int32_t* n);

const char* toast_last_error(void);
void toast_free_graph(toast_graph* g);
void toast_free_analysis(toast_analysis* a);

#ifdef __cplusplus
}
#endif

#endif /* TOAST_H */
