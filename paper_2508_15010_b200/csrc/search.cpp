// Host MCTS around the K1/K2 kernels.
// One tree per rank rooted at the unsharded module.  A round
// selects L leaves by UCT with virtual loss, expands the lowest untried legal
// action of each, evaluates each leaf's own state exactly (K1) plus R Philox
// rollouts from it (K2, "generating many trajectories"), backs up
// reward = -score, and stops when a round fails to improve the best
// (patience configurable) or the budget is spent.
// Root-parallel ranks exchange one fixed-size record per round; the caller
// all-gathers the records (torch.distributed / NCCL) and imports them.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "toast_internal.h"

namespace toast {

struct SNode {
  std::vector<uint16_t> prefix;
  std::vector<int32_t> untried;
  std::vector<SNode*> children;
  SNode* parent = nullptr;
  double W = 0.0;
  int64_t N = 0;
};

using ExportRec = toast_search_export;   // include/toast.h
size_t search_export_bytes(const toast_analysis* a);

}  // namespace toast

struct toast_search_state {
  const toast_analysis* a = nullptr;
  toast_search_opts o{};
  int32_t rank = 0, world = 1;
  uint64_t seed = 0;
  toast::SNode* root = nullptr;
  std::unordered_map<uint64_t, toast::SNode*> states;   // transpositions (R24): state key -> the node holding it
  // local incumbent (reset to the global one after each import) and global incumbent
  toast_cost best{};
  uint16_t best_seq[32] = {0};
  toast_cost gbest{};
  uint16_t gbest_seq[32] = {0};
  int64_t evals = 1;           // this rank (the root eval counts once)
  int64_t global_evals = 1;
  int64_t rollouts_done = 0;
  int32_t rounds = 0, nonimprove = 0, hit_target = 0, done = 0;
  std::vector<toast_root_stat> groot;   // root-child statistics summed over the ranks (last import)
  double time_to_target = -1.0;
  std::chrono::steady_clock::time_point t_start;
  // buffers: pinned host (prefixes in, per-leaf reductions out) and device scratch
  uint16_t* h_lpre = nullptr;
  toast::LeafRed* h_red = nullptr;
  void* d_buf = nullptr;
  size_t d_bytes = 0;
  bool pooled = false;     // the buffers belong to the analysis' search pool
  ~toast_search_state();
};

namespace toast {
namespace {

void free_tree(SNode* n) {
  if (!n) return;
  std::vector<SNode*> st{n};
  while (!st.empty()) {
    SNode* x = st.back();
    st.pop_back();
    for (SNode* c : x->children) st.push_back(c);
    delete x;
  }
}

std::vector<int32_t> legal_after(const toast_analysis* a, const std::vector<uint16_t>& prefix) {
  std::vector<int32_t> out;
  if ((int)prefix.size() >= a->dt.max_depth) return out;
  const int nw = a->dt.n_words;
  std::vector<uint32_t> legal(nw, 0xffffffffu);
  legal[0] &= ~1u;
  for (uint16_t p : prefix)
    for (int w = 0; w < nw; ++w) legal[w] &= ~a->h_kill[(size_t)p * nw + w];
  for (int32_t x = 1; x < a->dt.n_actions; ++x)
    if ((legal[x >> 5] >> (x & 31)) & 1) out.push_back(x);
  return out;
}

bool better(const toast_cost& x, const uint16_t* sx, const toast_cost& y, const uint16_t* sy) {
  if (x.score != y.score) return x.score < y.score;
  if (x.state_key != y.state_key) return x.state_key < y.state_key;
  for (int i = 0; i < 32; ++i) if (sx[i] != sy[i]) return sx[i] < sy[i];
  return false;
}

double elapsed(const toast_search_state* s) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - s->t_start).count();
}

}  // namespace

toast_status search_begin(const toast_analysis* a, const toast_search_opts* o, int32_t rank, int32_t world,
                          toast_search_state** out, std::string& err) {
  if (o->leaves_per_round < 1 || o->rollouts_per_leaf < 0 || o->patience < 1 || world < 1 || rank < 0 || rank >= world) {
    err = "bad search options";
    return TOAST_E_INVALID_ARG;
  }
  auto s = std::make_unique<toast_search_state>();
  s->a = a;
  s->o = *o;
  s->rank = rank;
  s->world = world;
  s->seed = o->seed + (uint64_t)rank;
  s->t_start = std::chrono::steady_clock::now();
  s->root = new SNode();
  s->root->untried = legal_after(a, s->root->prefix);
  s->states[a->baseline.state_key] = s->root;   // the unsharded module (key 0)
  s->best = a->baseline;              // the unsharded root is the first incumbent
  memset(s->best_seq, 0, sizeof s->best_seq);
  s->gbest = s->best;
  memset(s->gbest_seq, 0, sizeof s->gbest_seq);
  const int64_t L = o->leaves_per_round, R = o->rollouts_per_leaf;
  // device: [L][32] prefixes | [L] leaf records | [L*R][32] sequences | [L*R] records | [L] reductions
  s->d_bytes = (size_t)L * 64 + (size_t)L * sizeof(toast_cost) + (size_t)L * R * (64 + sizeof(toast_cost)) +
               (size_t)L * sizeof(LeafRed);
  if (a->device >= 0) {
    // buffers: the analysis' pool when it is free (grown to fit), else our own
    toast_analysis* ma = const_cast<toast_analysis*>(a);
    std::lock_guard<std::mutex> lk(ma->scratch_mu);
    auto& P = ma->spool;
    const size_t hp = (size_t)L * 64, hr = (size_t)L * sizeof(LeafRed);
    cudaError_t e = cudaSuccess;
    if (!P.in_use) {
      if (P.d_bytes < s->d_bytes) {
        if (P.d) cudaFree(P.d);
        P.d = nullptr; P.d_bytes = 0;
        e = cudaMalloc(&P.d, s->d_bytes);
        if (e == cudaSuccess) P.d_bytes = s->d_bytes;
      }
      if (e == cudaSuccess && P.h_pre_bytes < hp) {
        if (P.h_pre) cudaFreeHost(P.h_pre);
        P.h_pre = nullptr; P.h_pre_bytes = 0;
        e = cudaMallocHost(&P.h_pre, hp);
        if (e == cudaSuccess) P.h_pre_bytes = hp;
      }
      if (e == cudaSuccess && P.h_red_bytes < hr) {
        if (P.h_red) cudaFreeHost(P.h_red);
        P.h_red = nullptr; P.h_red_bytes = 0;
        e = cudaMallocHost(&P.h_red, hr);
        if (e == cudaSuccess) P.h_red_bytes = hr;
      }
      if (e != cudaSuccess) { err = cudaGetErrorString(e); return TOAST_E_OOM; }
      P.in_use = true;
      s->pooled = true;
      s->d_buf = P.d;
      s->h_lpre = reinterpret_cast<uint16_t*>(P.h_pre);
      s->h_red = reinterpret_cast<LeafRed*>(P.h_red);
    } else {
      e = cudaMalloc(&s->d_buf, s->d_bytes);
      if (e == cudaSuccess) e = cudaMallocHost((void**)&s->h_lpre, hp);
      if (e == cudaSuccess) e = cudaMallocHost((void**)&s->h_red, hr);
      if (e != cudaSuccess) { err = cudaGetErrorString(e); return TOAST_E_OOM; }
    }
  }
  *out = s.release();
  return TOAST_OK;
}

toast_status search_round(toast_search_state* s, void* export_buf, std::string& err) {
  const toast_analysis* a = s->a;
  if (!s->d_buf) { err = "search rounds need device tables (the analysis is host-only)"; return TOAST_E_CUDA; }
  const int L = s->o.leaves_per_round, R = s->o.rollouts_per_leaf;
  std::vector<SNode*> leaves;
  for (int l = 0; l < L; ++l) {
    SNode* node = s->root;
    while (true) {
      if (!node->untried.empty()) {
        SNode* ch = new SNode();
        ch->prefix = node->prefix;
        ch->prefix.push_back((uint16_t)node->untried.front());
        node->untried.erase(node->untried.begin());
        ch->parent = node;
        ch->untried = legal_after(a, ch->prefix);
        node->children.push_back(ch);
        node = ch;
        break;
      }
      if (node->children.empty()) break;
      SNode* bc = nullptr;
      double bv = 0;
      for (SNode* ch : node->children) {
        double v = ch->W / (double)ch->N + s->o.uct_c * std::sqrt(std::log((double)node->N) / (double)ch->N);
        if (!bc || v > bv) { bc = ch; bv = v; }
      }
      node = bc;
    }
    for (SNode* x = node; x; x = x->parent) { x->N += 1; x->W -= 1.0; }   // virtual loss
    leaves.push_back(node);
  }
  // device batch: L exact leaf evals + L*R rollouts (R per leaf prefix) + the per-leaf reduction
  memset(s->h_lpre, 0, (size_t)L * 64);
  for (int l = 0; l < L; ++l) {
    const auto& p = leaves[l]->prefix;
    for (size_t i = 0; i < p.size(); ++i) s->h_lpre[(size_t)l * 32 + i] = p[i];
  }
  char* d = reinterpret_cast<char*>(s->d_buf);
  uint16_t* d_lpre = reinterpret_cast<uint16_t*>(d);
  toast_cost* d_lcost = reinterpret_cast<toast_cost*>(d + (size_t)L * 64);
  uint16_t* d_outs = reinterpret_cast<uint16_t*>(d + (size_t)L * (64 + sizeof(toast_cost)));
  toast_cost* d_cost = reinterpret_cast<toast_cost*>(reinterpret_cast<char*>(d_outs) + (size_t)L * R * 64);
  void* d_red = reinterpret_cast<char*>(d_cost) + (size_t)L * R * sizeof(toast_cost);
  cudaStream_t st = (cudaStream_t)s->o.cuda_stream;
  auto ck = [&](cudaError_t e) { if (e != cudaSuccess) { err = cudaGetErrorString(e); return false; } return true; };
  if (!ck(cudaMemcpyAsync(d_lpre, s->h_lpre, (size_t)L * 64, cudaMemcpyHostToDevice, st))) return TOAST_E_CUDA;
  toast_status ts = launch_eval(a, d_lpre, L, d_lcost, st, err);
  if (ts) return ts;
  if (R > 0) {
    ts = launch_rollout(a, d_lpre, (int64_t)L * R, s->seed, (uint64_t)s->rollouts_done, d_outs, d_cost, st, err, R);
    if (ts) return ts;
  }
  ts = launch_round_reduce(d_lcost, d_lpre, d_cost, d_outs, L, R, d_red, st, err);
  if (ts) return ts;
  if (!ck(cudaMemcpyAsync(s->h_red, d_red, (size_t)L * sizeof(LeafRed), cudaMemcpyDeviceToHost, st))) return TOAST_E_CUDA;
  if (!ck(cudaStreamSynchronize(st))) return TOAST_E_CUDA;
  s->rollouts_done += (int64_t)L * R;
  for (SNode* lf : leaves) for (SNode* x = lf; x; x = x->parent) { x->N -= 1; x->W += 1.0; }
  // backup (R16): each leaf's in-order reward sum, once per node on its path
  for (int l = 0; l < L; ++l) {
    const LeafRed& rr = s->h_red[l];
    for (SNode* x = leaves[l]; x; x = x->parent) { x->N += R + 1; x->W += rr.reward_sum; }
    if (rr.best != -2 && better(rr.cost, rr.seq, s->best, s->best_seq)) {
      s->best = rr.cost;
      memcpy(s->best_seq, rr.seq, 64);
    }
  }
  // reading R24 ("any action sequence yielding the same sharded
  // model resolves to the same unique state, eliminating duplication by
  // construction"): with transpositions on, the tree holds each materialised
  // state once — a selected leaf whose exactly evaluated state another node
  // already holds leaves the tree (its rewards stay backed up on its path)
  if (s->o.transpositions) {
    std::vector<SNode*> gone;
    for (int l = 0; l < L; ++l) {
      const LeafRed& rr = s->h_red[l];
      if (rr.leaf_status != 0) continue;
      SNode* lf = leaves[l];
      auto it = s->states.find(rr.leaf_key);
      if (it == s->states.end()) s->states.emplace(rr.leaf_key, lf);
      else if (it->second != lf && std::find(gone.begin(), gone.end(), lf) == gone.end()) gone.push_back(lf);
    }
    for (SNode* g : gone) {
      auto& ch = g->parent->children;
      ch.erase(std::find(ch.begin(), ch.end(), g));
      delete g;
    }
  }
  s->evals += (int64_t)L * (R + 1);
  s->rounds++;
  ExportRec* ex = reinterpret_cast<ExportRec*>(export_buf);
  memset(ex, 0, sizeof(ExportRec));
  ex->best_score = s->best.score;
  ex->best_key = s->best.state_key;
  memcpy(ex->best_seq, s->best_seq, 64);
  ex->evals = s->evals;
  ex->elapsed_s = elapsed(s);
  ex->rank = s->rank;
  ex->best = s->best;
  // this rank's root-child statistics, indexed by action id
  toast_root_stat* rs = reinterpret_cast<toast_root_stat*>(reinterpret_cast<char*>(export_buf) + sizeof(ExportRec));
  memset(rs, 0, sizeof(toast_root_stat) * (size_t)a->dt.n_actions);
  for (SNode* ch : s->root->children) {
    rs[ch->prefix[0]].visits = ch->N;
    rs[ch->prefix[0]].value_sum = ch->W;
  }
  return TOAST_OK;
}

toast_status search_import(toast_search_state* s, const void* gathered, int32_t* stop, std::string& err) {
  (void)err;
  const size_t rb = search_export_bytes(s->a);
  auto rec = [&](int i) { return reinterpret_cast<const ExportRec*>(reinterpret_cast<const char*>(gathered) + rb * i); };
  int gb = 0;
  int64_t tot = 0;
  const int NA = s->a->dt.n_actions;
  s->groot.assign(NA, toast_root_stat{0, 0.0});
  for (int i = 0; i < s->world; ++i) {
    tot += rec(i)->evals;
    if (i && better(rec(i)->best, rec(i)->best_seq, rec(gb)->best, rec(gb)->best_seq)) gb = i;
    const toast_root_stat* rs = reinterpret_cast<const toast_root_stat*>(rec(i) + 1);
    for (int x = 0; x < NA; ++x) {   // rank order: the sums are identical on every rank
      s->groot[x].visits += rs[x].visits;
      s->groot[x].value_sum += rs[x].value_sum;
    }
  }

  // the global incumbent before this round is identical on every rank
  bool improved = better(rec(gb)->best, rec(gb)->best_seq, s->gbest, s->gbest_seq);
  if (improved) {
    s->gbest = rec(gb)->best;
    memcpy(s->gbest_seq, rec(gb)->best_seq, 64);
  }
  s->best = s->gbest;
  memcpy(s->best_seq, s->gbest_seq, 64);
  s->global_evals = tot;
  const double el = rec(0)->elapsed_s;   // rank 0's clock decides time limits on every rank
  if (s->time_to_target < 0 && !std::isnan(s->o.target_score) && s->best.score <= s->o.target_score) {
    s->time_to_target = el;
    s->hit_target = 1;
  }
  if (improved) s->nonimprove = 0;
  else s->nonimprove++;
  int st = 0;
  if (s->nonimprove >= s->o.patience) st = 1;
  if (s->o.max_evals > 0 && tot >= s->o.max_evals) st = 1;
  if (s->o.time_limit_s > 0 && el >= s->o.time_limit_s) st = 1;
  if (s->hit_target) st = 1;
  s->done = st;
  *stop = st;
  return TOAST_OK;
}

// the same round / import with the exchange buffers in device memory, ordered
// on the caller's stream (the NCCL all-gather runs between them on that stream)
toast_status search_round_dev(toast_search_state* s, void* export_dev, void* stream, std::string& err) {
  std::vector<char> buf(search_export_bytes(s->a));
  toast_status st = search_round(s, buf.data(), err);
  if (st) return st;
  cudaError_t e = cudaMemcpyAsync(export_dev, buf.data(), buf.size(), cudaMemcpyHostToDevice, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);   // the host record dies with this call
  if (e != cudaSuccess) { err = cudaGetErrorString(e); return TOAST_E_CUDA; }
  return TOAST_OK;
}

toast_status search_import_dev(toast_search_state* s, const void* gathered_dev, int32_t* stop, void* stream,
                               std::string& err) {
  std::vector<char> buf(search_export_bytes(s->a) * (size_t)s->world);
  cudaError_t e = cudaMemcpyAsync(buf.data(), gathered_dev, buf.size(), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) { err = cudaGetErrorString(e); return TOAST_E_CUDA; }
  return search_import(s, buf.data(), stop, err);
}

void search_result(const toast_search_state* s, toast_search_result* out) {
  memset(out, 0, sizeof(*out));
  memcpy(out->best_seq, s->best_seq, 64);
  out->best = s->best;
  out->evals = s->global_evals;
  out->rounds = s->rounds;
  out->hit_target = s->hit_target;
  out->wall_s = elapsed(s);
  out->time_to_target_s = s->time_to_target;
}

size_t search_export_bytes(const toast_analysis* a) {
  return sizeof(ExportRec) + sizeof(toast_root_stat) * (size_t)a->dt.n_actions;
}

int32_t search_root_stats(const toast_search_state* s, toast_root_stat* out, int32_t cap) {
  const int32_t n = s->a->dt.n_actions;
  for (int32_t x = 0; x < cap && x < n; ++x)
    out[x] = x < (int32_t)s->groot.size() ? s->groot[x] : toast_root_stat{0, 0.0};
  return n;
}

void search_free(toast_search_state* s) { delete s; }

}  // namespace toast

toast_search_state::~toast_search_state() {
  toast::free_tree(root);
  if (pooled) {
    toast_analysis* ma = const_cast<toast_analysis*>(a);
    std::lock_guard<std::mutex> lk(ma->scratch_mu);
    ma->spool.in_use = false;
    return;
  }
  if (d_buf) cudaFree(d_buf);
  if (h_lpre) cudaFreeHost(h_lpre);
  if (h_red) cudaFreeHost(h_red);
}
