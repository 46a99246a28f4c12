// Internal structures of libtoast: host-side graph/analysis and the packed
// device tables the sm_100a kernels read.
#pragma once

#include <cstdint>
#include <vector_types.h>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/toast.h"

namespace toast {

// ----------------------------------------------------------------- op kinds
enum OpKind : uint8_t {
  OK_PARAM, OK_RET, OK_UNARY, OK_BINARY, OK_TRANSPOSE, OK_REDUCE, OK_BROADCAST, OK_MATMUL, OK_DOT,
  OK_CONV, OK_CONV_BI, OK_CONV_BF, OK_RESAMPLE, OK_CONCAT, OK_SLICE, OK_PAD, OK_GATHER, OK_SEGSUM
};

enum LoopType : uint8_t { T_P = 0, T_R = 1, T_X = 2 };

struct GValue {
  int32_t dtype_code;          // index into the dtype table (f32, bf16, f16, i32, f64, i64)
  int32_t elem_bytes;
  std::vector<int64_t> shape;
  int32_t def_op;
  std::string name;
};

struct GOp {
  OpKind kind;
  std::string name;            // IR spelling (hash input for C6/C7)
  std::vector<int64_t> ia;     // integer attributes (meaning per kind)
  std::vector<int32_t> operands;
  int32_t result = -1;
  std::string binding;
  std::string attr_text;       // the bracket attributes as written (groups ';', atoms ',')
};

}  // namespace toast

struct toast_graph {
  std::vector<toast::GValue> values;
  std::vector<toast::GOp> ops;   // params, body, rets
  int32_t n_params = 0;
  std::vector<std::string> axis_names;
  std::vector<int32_t> axis_size;
  std::vector<double> axis_bw;
  toast_machine machine;
  int32_t device = -1;
};

namespace toast {

// ------------------------------------------------------------ host tables
// (used by toast_materialize on the host and to build the device tables)
// one op, 32 bytes
struct DOp {
  uint32_t loop_begin;   // global id of the op's role-0 loop
  uint8_t n_loops;
  uint8_t rank;          // result rank (0 for ret)
  uint8_t rmask;         // bit r set <=> role r is a reduction (R) loop
  uint8_t flags;         // bit0 matmul-class, bit1 ret
  uint32_t res_roles;    // 4 bits per result dim: role of dim i
  uint32_t use_begin;    // first entry in uses[]
  uint32_t death_begin;  // first entry in deaths[]
  uint16_t n_death;
  uint8_t n_uses;
  uint8_t pad;
  uint64_t gbytes;       // global bytes of the result (0 for ret)
};
static_assert(sizeof(DOp) == 32, "DOp is 32 B");

// one use (op t, operand k), 8 bytes
struct DUse {
  uint32_t def_op;       // value id == defining op
  uint32_t use_roles;    // 4 bits per dim: role in op t of operand dim i
};

// packed loop word (uint64):
//   [0,10)  acolor (0x3FF = no action can touch this loop)
//   [10,12) type
//   [12,28) div_ok: bit S <=> extent % prod(sizes of axis subset S) == 0
//   [28,44) deselection id (0 = never deselected)
constexpr uint32_t NO_ACOLOR = 0x3FF;

constexpr int MAX_LOOPS_PER_OP = 8;
constexpr int MAX_USES_PER_OP = 8;
constexpr int MAX_RANK = 8;
constexpr int MAX_ACTIONS = 1024;
constexpr int MAX_GROUPS = 64;

// ------------------------------------------------------------ device tables
// An op's SIGNATURE fixes how it materialises (per role: action color,
// divisibility, deselection class, result dim), so per candidate the kernel
// keeps one entry per signature: axis->role | axis->result dim.  Everything
// per op is then aggregated per signature (state key, FLOPs), per edge
// template (collectives) and per frontier point (peak memory, reading R19).
struct KUse {            // 16 B: one "special" use edge (a value used more than once by one op)
  uint16_t def_sig;      // signature of the defining op
  uint16_t tmpl;         // NO_TMPL
  uint32_t use_dimof;    // nibble r: operand dim held by this op's role r (0xF: none)
  uint64_t gb_flags;     // def global bytes (bits 0-55) | flags << 56 (bit0 first use of the value here, bit1 last)
};
// one kept op of the peak-memory frontier: M_t = constant + n_sig signature
// terms + n_tmpl template terms (+ its special edges).  Points come in groups
// of FRONTIER_GROUP: the first carries the constant and the signature terms
// absolutely, the others as signed differences from the previous point.
// A term is a signed 48-bit value | feature id << 48.
constexpr int FRONTIER_GROUP = 8;
struct KPoint {          // 16 B
  uint32_t term_begin;
  uint16_t n_sig, n_tmpl;
  uint32_t spec_begin;
  uint16_t n_spec;
  uint16_t use_sig;      // the op's own signature (special edges)
};
constexpr uint16_t NO_TMPL = 0xFFFF;
// edge template: use edges with the same (def signature, use signature, use
// role->dim map) communicate identically for every candidate; their payloads
// are costed once per candidate from the template's summed def bytes
struct KTmpl {           // 24 B
  uint16_t def_sig;
  uint16_t use_sig;      // the use op's materialisation class
  uint32_t use_dimof;
  uint64_t sum_gbytes;
  uint32_t n_edges;
  uint32_t fslot;        // the template's growth-code slot for the frontier (0xFFFFFFFF: no frontier term uses it)
};
// one op signature, 64 B (one warp-uniform 4 x 16-B load): per role its
// divisibility word, per distinct action color of the signature the roles it
// covers, each role's deselection class and result dim
struct KSig {
  uint32_t div[4];       // role r: div_ok (bit S <=> extent divisible by prod(axis subset S)) = div[r >> 1] >> 16 * (r & 1)
  uint32_t col[8];       // k < m: acolor | role mask << 10
  uint32_t div1;         // byte A: the roles (with a color) whose extent axis A alone divides (the walk's test for a role holding no axis yet)
  uint8_t m;             // distinct action colors among the roles
  uint8_t dsel_roles;    // roles with a deselection class
  uint8_t nr;
  uint8_t pad;           // bit0: every axis subset divides every shardable role (one-round materialisation)
  uint64_t cls;          // byte r: deselection class of role r (0 = never deselected)
};
// critical-path stream (reading R22), 8-byte records (2 x u32) in program
// order: per op {result slot, compute class | #operands << 16}, then per
// operand {its def's finish slot, communication class}
struct KCpComm {         // 16 B: an edge duration class
  uint16_t def_sig;
  uint16_t use_mc;       // the use op's materialisation class
  uint32_t use_dimof;    // nibble r: operand dim held by the op's role r (0xF: none)
  uint64_t gb;           // def global bytes
};
struct KCpComp {         // 16 B: a compute-time class
  uint32_t sig;
  uint32_t pad;
  uint64_t gflops;
};
constexpr uint32_t NO_SLOT = 0xFFFFFFFFu;   // a parameter's "slot": finish 0
constexpr uint32_t NO_CLASS = 0xFFFFu;      // no compute time
constexpr uint32_t ZERO_COMM = 0xFFFFFFFFu; // an edge that never communicates: the def's finish as is
// The walk is a sequence of bundles of <= CP_EMAX operand edges (8-B records:
// x = the operand's finish slot | duration class << 16 | first edge of its op
// << 31; y = the op's result slot | compute-time class << 16 | last edge << 31,
// indices into the block's scratch, kernels.cu cp_stride; "none" indices name
// a 0.0 entry, a non-last edge names the trash slot); no edge of a bundle
// reads a slot its bundle writes.
constexpr int CP_EMAX = 8;
constexpr int PIPE_STREAMS = 8;   // host-buffer pipeline streams (at most)
constexpr int CP_WINDOW = 96;
static_assert(sizeof(KCpComm) == 16 && sizeof(KCpComp) == 16, "cp records");
// Device images of the records above (built by upload_tables): every
// signature reference a kernel resolves per candidate is replaced by the
// signature's materialisation class (whose axis -> role map the kernels keep
// per lane) and its role -> result-dim map, so no per-signature entry table
// is needed on chip.
struct KTmplDev {        // 32 B (2 x 16-B loads)
  uint32_t mcs;          // def class | use class << 16
  uint32_t use_dimof;
  uint64_t sum_gbytes;
  uint32_t n_edges;
  uint32_t fslot;
  uint32_t def_rdm;      // nibble r: result dim of the def signature's role r (0xF: none)
  uint32_t pad;
};
struct KUseDev {         // 32 B
  uint32_t def_mc;
  uint32_t use_dimof;
  uint64_t gb_flags;
  uint32_t def_rdm;
  uint32_t pad[3];
};
struct KCpCommDev {      // 32 B
  uint32_t mcs;          // def class | use class << 16
  uint32_t use_dimof;
  uint64_t gb;
  uint32_t def_rdm;
  uint32_t pad[3];
};
static_assert(sizeof(KTmplDev) == 32 && sizeof(KUseDev) == 32 && sizeof(KCpCommDev) == 32, "device records");
static_assert(sizeof(KSig) == 64 && sizeof(KPoint) == 16 && sizeof(KUse) == 16 && sizeof(KTmpl) == 24, "records");


// search round reduction record (K3), one per leaf
struct LeafRed {
  double reward_sum;     // sum of the leaf's R+1 rewards (-score), in order (R16)
  int32_t best;          // -1 = the leaf's own state, j = rollout j, -2 = none valid
  uint32_t leaf_status;  // the leaf's own state: status and key (transpositions, reading R24)
  uint64_t leaf_key;
  toast_cost cost;       // the leaf's best record
  uint16_t seq[32];      // and its sequence
};

// NEXT-3 in-launch dedup (toast_nda_opts.dedup): per launch, scratch for the
// front kernel's per-candidate results, the hash set of distinct states and
// the compact list of their representatives (kernels.cu "dedup")
struct DedupCtx {
  uint64_t* key = nullptr;        // [n] state key (H7); null: dedup off
  uint64_t* flo = nullptr;        // [n] FLOP total, low / high word (H3)
  uint64_t* fhi = nullptr;
  uint32_t* status = nullptr;     // [n] decode status (H1)
  uint32_t* rep = nullptr;        // [n] the candidate whose state this is (itself if first), ~0u if invalid
  uint32_t* slot = nullptr;       // [n] a representative's index in the compact list
  uint32_t* rep_of_slot = nullptr;// [n] the compact list
  uint32_t* rows = nullptr;       // [n][row_words] the class maps (the materialised state)
  uint32_t* table = nullptr;      // [cap] candidate + 1 (0 = empty), open addressing on the key
  unsigned int* count = nullptr;  // [1] representatives
  uint32_t cap_mask = 0, row_words = 0;
};

// signature role word: acolor [0,10) | div_ok [10,26) | deselection class [26,34)
struct DeviceTables {
  const KPoint* points = nullptr;        // [n_points] peak-memory frontier (R19); use_sig holds the op's class
  const uint64_t* terms = nullptr;       // per point: constant, then value | feature << 48
  const KUseDev* spec = nullptr;         // special edges of the points
  const KSig* sigs = nullptr;            // [n_mc] per materialisation class
  const uint64_t* fsig = nullptr;        // [n_fsig] per frontier signature slot: class | result dims << 32
  const uint64_t* mc_key = nullptr;      // [n_mc][4 axes][8 roles] summed state-key terms (R14)
  const uint64_t* mc_flops = nullptr;    // [n_mc][2] summed global FLOPs of matmul-class ops (lo, hi)
  const KTmplDev* tmpl = nullptr;        // [n_tmpl]
  const uint4* tmpl_b = nullptr;         // [n_tmpl][2] the same with byte maps (prmt lookups), when tmpl_bytes
  int32_t tmpl_bytes = 0;                // every op has <= 7 roles: H4 reads the byte-map templates
  const uint64_t* desel = nullptr;       // [class][2] = need0, need1 (class 0 = none)
  const uint32_t* actions = nullptr;     // acolor | r << 10 | axis << 18
  const uint64_t* acol_groups = nullptr; // 8 x 8-bit group ids (0xFF = unused)
  const uint32_t* kill = nullptr;        // [n_actions][n_words]
  const uint64_t* action_grp = nullptr;  // [n_actions][2]: the SetGroups an action fixes, and those it fixes to 1
  int32_t n_desel = 0;                   // deselection classes (class 0 = none)
  // constants
  int32_t n_ops, n_loops, n_actions, n_acolors, n_words, n_axes, max_depth, n_sigs;
  int32_t n_tmpl, pow2;  // pow2: every axis size is a power of two (exact division = shift)
  int32_t n_points, n_mc;
  int32_t n_fsig, n_ftmpl;  // signatures / templates the frontier terms use (their per-lane code tables)
  int32_t n_spec = 0;       // special edges (a value used twice by one op) of the frontier points
  int32_t n_terms = 0;      // frontier terms (the TOAST_SMEM_TABLES copy)
  int32_t cost_model, n_slots;   // R22: critical path; finish-time slots per candidate
  int32_t n_comm, n_comp;        // R22: edge-duration and compute-time classes
  const uint2* cp = nullptr;     // critical-path stream
  const uint32_t* cp_bsize = nullptr;  // per bundle: edges | prefetch slot << 4 | prefetch slot << 18 (0x3FFF: none)
  int32_t n_bundles = 0;
  const KCpCommDev* cp_comm = nullptr;
  const KCpComp* cp_comp = nullptr;      // sig holds the op's class
  double* cp_scratch = nullptr;  // per launched block: [cp_stride][32] doubles (allocated per launch)
  unsigned int* ticket = nullptr; // per launch: the next batch counter (dynamic batch scheduling; null: static)
  DedupCtx dd;                    // per launch (dedup launches only)
  int32_t sizes[4];
  double bw[4];
  double F, C, t0;
  uint64_t DM, peak0;
  uint64_t inv[16];     // exact division by prod(subset): (x >> shift) * inv
  uint32_t shift[16];
  uint64_t shift_pack;  // nibble S = shift[S] (pow2 meshes, every subset shift <= 15)
  uint64_t inv128_lo[16], inv128_hi[16];   // the same inverse mod 2^128 (FLOP totals)
};

}  // namespace toast

struct toast_analysis {
  // host-side results (also used for the JSON dump)
  int32_t n_ops = 0;
  int64_t n_loops = 0, n_edges = 0;
  std::vector<int32_t> loop_op, loop_role, loop_type, loop_comp, loop_scolor;
  std::vector<int64_t> loop_ext;
  struct Conf { int32_t op, u, v, set, side0; };
  std::vector<Conf> conflicts;
  int64_t n_boxes = 0, dropped_boxes = 0;
  int32_t grouping = 0;                      // TOAST_GROUP_COMPAT / TOAST_GROUP_CONTRACTION (reading R23)
  int64_t contracted = 0, contract_rejected = 0;
  std::vector<int32_t> cnode;                // R23: contracted node (smallest member loop) per loop
  std::vector<int32_t> set_group;
  std::vector<uint64_t> set_sig;
  int32_t n_groups = 0;
  std::vector<int32_t> sc_min_loop;
  std::vector<int64_t> sc_value_dims;
  std::vector<std::vector<int32_t>> sc_groups;
  std::vector<toast_action_info> actions;   // [0] = STOP
  toast_cost baseline;
  double t0 = 0;
  uint64_t peak0 = 0;

  // host copies of the packed tables (kept for toast_materialize and tests)
  std::vector<toast::DOp> h_ops;
  std::vector<uint64_t> h_gflops, h_loops, h_desel, h_acol_groups;
  std::vector<toast::DUse> h_uses;
  std::vector<uint32_t> h_deaths, h_actions, h_kill;
  // device-table images
  std::vector<toast::KPoint> h_points;      // peak-memory frontier
  std::vector<uint64_t> h_terms;
  std::vector<toast::KUse> h_spec;
  std::vector<int32_t> point_op;            // op index of each frontier point
  // the reduced method's work per evaluation, before the kernels' table
  // sharing (materialisation classes, class-keyed templates, delta terms):
  // roles over signatures, signature-keyed templates, absolute frontier terms
  int64_t work_sig_roles = 0, work_tmpl = 0, work_terms = 0;
  std::vector<uint32_t> h_cp;               // critical-path stream (8-B records as 2 x u32)
  std::vector<uint32_t> h_cp_bsize;         // per bundle of the stream: edges | two prefetch hints
  std::vector<toast::KCpComm> h_cp_comm;
  std::vector<toast::KCpComp> h_cp_comp;
  int32_t cost_model = 0;
  int32_t cp_walked_ops = 0, cp_walked_edges = 0;   // R22 walk after the exact reductions
  std::vector<toast::KSig> h_sigs;          // per materialisation class
  std::vector<uint64_t> h_sig_mr;           // per signature: class | resdim << 32
  std::vector<uint64_t> h_sig_roles, h_desel_cls;
  std::vector<uint8_t> h_sig_nroles;
  std::vector<uint32_t> h_sig_resdim;
  std::vector<uint64_t> h_sig_key, h_sig_flops;
  std::vector<uint64_t> h_mc_key, h_mc_flops;   // the same summed per materialisation class (uploaded)
  std::vector<toast::KTmpl> h_tmpl;
  std::vector<uint32_t> op_sig;
  std::vector<int32_t> axis_size;

  std::shared_ptr<const toast_graph> graph;   // the program (names, attributes) for toast_lower
  toast::DeviceTables dt;       // device pointers valid iff device >= 0
  int32_t device = -1;
  std::vector<void*> dev_allocs;

  // scratch for host-pointer calls
  std::mutex scratch_mu;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  int32_t smem_per_warp = 0, warps_per_block = 8;
  int32_t eval_blocks = 0, rollout_blocks = 0;
  int32_t occ_eval[4] = {0, 0, 0, 0}, occ_roll[4] = {0, 0, 0, 0};   // blocks per SM for K = 1, 2, 4, 8
  int32_t n_sms = 0, k_throughput = 1;
  int32_t k_force = 0;   // autotune: every launch uses this K (0: pick)
  int32_t dedup = 0;     // NEXT-3: rollout launches cost each distinct state once
  int32_t occ_back = 1;  // resident blocks per SM of the dedup back kernel
  int32_t back_warps = 1;  // ... and its warps per block
  void* pipe_stream[toast::PIPE_STREAMS] = {};      // host-buffer path: chunked H2D / kernel / D2H overlap
  // search buffers, kept between searches (a search that finds them in use allocates its own)
  struct SearchPool {
    void* d = nullptr;
    size_t d_bytes = 0;
    void* h_pre = nullptr;
    size_t h_pre_bytes = 0;
    void* h_red = nullptr;
    size_t h_red_bytes = 0;
    bool in_use = false;
  } spool;
  void* pipe_event = nullptr;
  void* cp_pool = nullptr;      // cudaMemPool_t of the per-launch scratch (batch ticket; R22 finish slots)
};

namespace toast {
// ir.cpp
toast_status parse_ir(const char* text, size_t len, toast_graph* g, std::string& err);
// analysis.cpp
toast_status build_analysis(const toast_graph* g, const toast_nda_opts* o, toast_analysis* a, std::string& err);
std::string dump_json(const toast_analysis* a);
uint32_t host_validate(const toast_analysis* a, const uint16_t* seq);
void host_materialize(const toast_analysis* a, const uint16_t* seq, uint8_t* masks);
// lower.cpp: the device-local program of one action sequence (NEXT-1)
toast_status lower_program(const toast_analysis* a, const uint16_t* seq, std::string& out, std::string& err);
// kernels.cu
toast_status upload_tables(toast_analysis* a, std::string& err);
toast_status autotune_k(toast_analysis* a, std::string& err);   // measured throughput K (after upload_tables)
void free_tables(toast_analysis* a);
// d_out: toast_cost[n], or toast_score[n] when compact
toast_status launch_eval(const toast_analysis* a, const uint16_t* d_seqs, int64_t n, void* d_out, void* stream,
                         std::string& err, bool compact = false);
toast_status launch_rollout(const toast_analysis* a, const uint16_t* d_pre, int64_t n, uint64_t seed, uint64_t id_base,
                            uint16_t* d_seqs, void* d_out, void* stream, std::string& err, int64_t rep = 1,
                            bool compact = false);
// search round reduction (K3): per leaf, reward sum + best candidate; d_out = [L] records of leaf_red_bytes()
toast_status launch_round_reduce(const toast_cost* d_lcost, const uint16_t* d_lpre, const toast_cost* d_cost,
                                 const uint16_t* d_seqs, int L, int R, void* d_out, void* stream, std::string& err);
size_t leaf_red_bytes();
toast_status run_host_buffers(toast_analysis* a, bool rollout, const uint16_t* h_in, int64_t n, uint64_t seed,
                              uint64_t id_base, uint16_t* h_seqs, void* h_out, void* stream, std::string& err,
                              bool compact = false);
bool is_device_pointer(const void* p);
}  // namespace toast
