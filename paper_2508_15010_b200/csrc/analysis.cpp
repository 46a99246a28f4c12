// H0: the once-per-graph analysis of libtoast, written for
// graphs of 10^4-10^5 loops: CSR edge lists, union-find, per-component
// bitset reachability for the "box" test, parity union-find for the
// compatibility closure.  Produces the packed device tables of
// toast_internal.h.  Definitions: SURVEY §8(c) C1-C8 / DESIGN.md.
#include <algorithm>
#include <chrono>
#include <array>
#include <cstring>
#include <map>
#include <set>
#include <numeric>
#include <cstdio>
#include <cstdlib>

#include "toast_internal.h"

namespace toast {
namespace {

// ---------------------------------------------------------------- hashing (C6/C14)
inline uint64_t splitmix_fin(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline uint64_t hc(uint64_t h, uint64_t x) { return splitmix_fin(h ^ (x + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2))); }
uint64_t hfold(const uint64_t* xs, size_t n) {
  uint64_t h = 0;
  for (size_t i = 0; i < n; ++i) h = hc(h, xs[i]);
  return h;
}
uint64_t hfold(std::vector<uint64_t> v, bool sort_first) {
  if (sort_first) std::sort(v.begin(), v.end());
  return hfold(v.data(), v.size());
}
uint64_t fnv(const std::string& s) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (unsigned char c : s) h = (h ^ c) * 0x100000001b3ULL;
  return h;
}

struct DSU {
  std::vector<int32_t> par;
  explicit DSU(size_t n) : par(n) { std::iota(par.begin(), par.end(), 0); }
  int32_t root(int32_t x) {
    while (par[x] != x) { par[x] = par[par[x]]; x = par[x]; }
    return x;
  }
  void join(int32_t a, int32_t b) {
    a = root(a); b = root(b);
    if (a == b) return;
    if (b < a) std::swap(a, b);
    par[b] = a;   // root = smallest member
  }
};

// per-op loop structure (C1 table, written directly per op kind)
struct OpLoops {
  std::vector<int64_t> ext;
  std::vector<uint8_t> type;
  std::vector<uint8_t> res_role;                // per result dim
  std::vector<std::vector<uint8_t>> use_role;   // per operand, per dim
};

OpLoops loops_of(const toast_graph* g, const GOp& op) {
  OpLoops L;
  auto S = [&](int k) -> const std::vector<int64_t>& { return g->values[op.operands[k]].shape; };
  const std::vector<int64_t> none;
  const std::vector<int64_t>& R = op.result >= 0 ? g->values[op.result].shape : none;
  auto add = [&](int64_t e, uint8_t t) { L.ext.push_back(e); L.type.push_back(t); };
  auto ident_roles = [](size_t n) { std::vector<uint8_t> v(n); for (size_t i = 0; i < n; ++i) v[i] = (uint8_t)i; return v; };
  switch (op.kind) {
    case OK_PARAM:
      for (int64_t e : R) add(e, T_P);
      L.res_role = ident_roles(R.size());
      break;
    case OK_RET:
      for (int64_t e : S(0)) add(e, T_P);
      L.use_role.push_back(ident_roles(S(0).size()));
      break;
    case OK_UNARY: case OK_BINARY:
      for (int64_t e : R) add(e, T_P);
      L.res_role = ident_roles(R.size());
      for (size_t k = 0; k < op.operands.size(); ++k) L.use_role.push_back(ident_roles(R.size()));
      break;
    case OK_TRANSPOSE:
      for (int64_t e : S(0)) add(e, T_P);
      L.use_role.push_back(ident_roles(S(0).size()));
      for (int64_t p : op.ia) L.res_role.push_back((uint8_t)p);
      break;
    case OK_REDUCE:
      for (size_t i = 0; i < S(0).size(); ++i) {
        add(S(0)[i], op.ia[i] ? T_R : T_P);
        if (!op.ia[i]) L.res_role.push_back((uint8_t)i);
      }
      L.use_role.push_back(ident_roles(S(0).size()));
      break;
    case OK_BROADCAST: {
      for (int64_t e : R) add(e, T_P);
      L.res_role = ident_roles(R.size());
      std::vector<uint8_t> u;
      for (size_t i = 0; i < S(0).size(); ++i) u.push_back((uint8_t)((int64_t)i < op.ia[0] ? i : i + 1));
      L.use_role.push_back(u);
      break;
    }
    case OK_MATMUL:
      add(R[0], T_P); add(R[1], T_P); add(S(0)[1], T_R);
      L.res_role = {0, 1};
      L.use_role = {{0, 2}, {2, 1}};
      break;
    case OK_DOT: {
      int64_t nb = op.ia[0], nc = op.ia[1];
      const int64_t* lb = &op.ia[2];
      const int64_t* rb = lb + nb;
      const int64_t* lc = rb + nb;
      const int64_t* rc = lc + nc;
      const auto& A = S(0); const auto& B = S(1);
      std::vector<int> ra(A.size(), -1), rbv(B.size(), -1);
      int role = 0;
      for (int64_t t = 0; t < nb; ++t) { add(A[lb[t]], T_P); ra[lb[t]] = role; rbv[rb[t]] = role; ++role; }
      std::vector<char> ua(A.size(), 0), ub(B.size(), 0);
      for (int64_t t = 0; t < nb; ++t) { ua[lb[t]] = 1; ub[rb[t]] = 1; }
      for (int64_t t = 0; t < nc; ++t) { ua[lc[t]] = 1; ub[rc[t]] = 1; }
      for (size_t i = 0; i < A.size(); ++i) if (!ua[i]) { add(A[i], T_P); ra[i] = role++; }
      for (size_t i = 0; i < B.size(); ++i) if (!ub[i]) { add(B[i], T_P); rbv[i] = role++; }
      int nres = role;
      for (int64_t t = 0; t < nc; ++t) { add(A[lc[t]], T_R); ra[lc[t]] = role; rbv[rc[t]] = role; ++role; }
      L.res_role = ident_roles(nres);
      std::vector<uint8_t> ua8, ub8;
      for (int x : ra) ua8.push_back((uint8_t)x);
      for (int x : rbv) ub8.push_back((uint8_t)x);
      L.use_role = {ua8, ub8};
      break;
    }
    case OK_CONV:     // roles N Ho Wo Co | Ci | KH KW
      add(R[0], T_P); add(R[1], T_X); add(R[2], T_X); add(R[3], T_P); add(S(0)[3], T_R); add(S(1)[0], T_X); add(S(1)[1], T_X);
      L.res_role = {0, 1, 2, 3};
      L.use_role = {{0, 1, 2, 4}, {5, 6, 4, 3}};
      break;
    case OK_CONV_BI:  // roles N H W Ci | Co | KH KW
      add(R[0], T_P); add(R[1], T_X); add(R[2], T_X); add(R[3], T_P); add(S(0)[3], T_R); add(S(1)[0], T_X); add(S(1)[1], T_X);
      L.res_role = {0, 1, 2, 3};
      L.use_role = {{0, 1, 2, 4}, {5, 6, 3, 4}};
      break;
    case OK_CONV_BF:  // roles KH KW Ci Co | N | H W
      add(R[0], T_X); add(R[1], T_X); add(R[2], T_P); add(R[3], T_P); add(S(0)[0], T_R); add(S(0)[1], T_X); add(S(0)[2], T_X);
      L.res_role = {0, 1, 2, 3};
      L.use_role = {{4, 5, 6, 2}, {4, 5, 6, 3}};
      break;
    case OK_RESAMPLE:
      add(R[0], T_P); add(R[1], T_X); add(R[2], T_X); add(R[3], T_P);
      L.res_role = {0, 1, 2, 3};
      L.use_role = {{0, 1, 2, 3}};
      break;
    case OK_CONCAT: case OK_SLICE: case OK_PAD:
      for (size_t i = 0; i < R.size(); ++i) add(R[i], (int64_t)i == op.ia[0] ? T_X : T_P);
      L.res_role = ident_roles(R.size());
      for (size_t k = 0; k < op.operands.size(); ++k) L.use_role.push_back(ident_roles(R.size()));
      break;
    case OK_GATHER: {   // roles e.. f | n(X)
      size_t ke = S(1).size();
      for (size_t t = 0; t <= ke; ++t) add(R[t], T_P);
      add(S(0)[0], T_X);
      L.res_role = ident_roles(ke + 1);
      L.use_role = {{(uint8_t)(ke + 1), (uint8_t)ke}, ident_roles(ke)};
      break;
    }
    case OK_SEGSUM: {   // roles e..(R) f | n(X)
      size_t ke = S(1).size();
      for (size_t t = 0; t < ke; ++t) add(S(0)[t], T_R);
      add(R[1], T_P);
      add(R[0], T_X);
      L.res_role = {(uint8_t)(ke + 1), (uint8_t)ke};
      L.use_role = {ident_roles(ke + 1), ident_roles(ke)};
      break;
    }
  }
  return L;
}

inline bool is_matmul_class(OpKind k) { return k == OK_MATMUL || k == OK_DOT || k == OK_CONV || k == OK_CONV_BI || k == OK_CONV_BF; }


// NEXT-4, reading R23: the dimension-graph contraction heuristic
// ([comment] §3.5) — "eagerly contract edges in the dimension graph
// unless this produces a (directed) path between two nodes that participate in
// a conflict".  M edges are taken once each in (def loop, use loop) order.
// Per contracted node of a component with conflicts, bitsets over the conflict
// endpoints: A = endpoints reaching it, D = endpoints it reaches (both including
// its own members), PA = the conflict partners of A.  Merging X and Y creates
// exactly the new paths through the merged node, so it joins a conflict iff
// (PA(X) | PA(Y)) & (D(X) | D(Y)) != 0.  After a merge the merged A / D are
// pushed to the node's descendants / ancestors; a node that already contains
// them stops the push (A only grows along edges, D only against them).
// Conflicts on the same unordered pair of contracted nodes form one set
// (contracting both vertical edges of a box identifies its
// conflicts as compatible), side 0 = the endpoint in the node of the set's
// smallest conflict's u.  The WL hash (C6) sees the contracted M edges between
// the set's endpoints.
static void build_contraction_sets(toast_analysis* a, int64_t NL, const std::vector<uint64_t>& ekeys,
                                   const std::vector<int64_t>& out_off, const std::vector<int32_t>& out_dst,
                                   const std::vector<int32_t>& ep_index, int32_t NE, const std::vector<uint64_t>& reach,
                                   const std::vector<int64_t>& reach_off, int32_t& n_sets,
                                   std::vector<std::vector<std::pair<int32_t, int32_t>>>& set_medges) {
  const size_t W = (size_t)(NE + 63) / 64;
  const int32_t NC = (int32_t)a->conflicts.size();
  auto bit = [](uint64_t* b, int32_t i) { b[i >> 6] |= 1ULL << (i & 63); };
  std::vector<uint64_t> partner((size_t)NE * W, 0);
  for (const auto& c : a->conflicts) {
    bit(&partner[(size_t)ep_index[c.u] * W], ep_index[c.v]);
    bit(&partner[(size_t)ep_index[c.v] * W], ep_index[c.u]);
  }
  int64_t nreach = 0;
  for (int64_t l = 0; l < NL; ++l) if (reach_off[l] >= 0) nreach = std::max(nreach, reach_off[l] + 1);
  std::vector<uint64_t> A((size_t)nreach * W, 0), D((size_t)nreach * W, 0), PA((size_t)nreach * W, 0);
  auto row = [&](std::vector<uint64_t>& v, int32_t l) { return &v[(size_t)reach_off[l] * W]; };
  // contracted adjacency (loop ids, resolved through the DSU when read)
  std::vector<std::vector<int32_t>> gout(NL), gin(NL);
  for (uint64_t e : ekeys) {
    const int32_t x = (int32_t)(e >> 32), y = (int32_t)(uint32_t)e;
    if (reach_off[x] < 0) continue;
    gout[x].push_back(y);
    gin[y].push_back(x);
  }
  // initial A / PA in loop order (every M edge goes from a lower to a higher loop id), D = reach + itself
  for (int64_t l = 0; l < NL; ++l) {
    if (reach_off[l] < 0) continue;
    uint64_t *al = row(A, (int32_t)l), *pl = row(PA, (int32_t)l), *dl = row(D, (int32_t)l);
    const uint64_t* rl = &reach[(size_t)reach_off[l] * W];
    for (size_t w = 0; w < W; ++w) dl[w] = rl[w];
    if (ep_index[l] >= 0) {
      bit(al, ep_index[l]);
      bit(dl, ep_index[l]);
      const uint64_t* pp = &partner[(size_t)ep_index[l] * W];
      for (size_t w = 0; w < W; ++w) pl[w] |= pp[w];
    }
    for (int32_t p : gin[l]) {
      const uint64_t *ap = row(A, p), *ppa = row(PA, p);
      for (size_t w = 0; w < W; ++w) { al[w] |= ap[w]; pl[w] |= ppa[w]; }
    }
  }
  const auto t_init = std::chrono::steady_clock::now();
  int64_t pushed = 0;
  DSU cg(NL);
  std::vector<int32_t> stack;
  // adjacency lists are concatenated (the shorter into the longer) and
  // compacted (roots, no duplicates, no self) only when they have doubled
  // since their last compaction, so a large node absorbing many small ones
  // costs amortised linear time
  std::vector<size_t> compacted(NL, 0), in_compacted(NL, 0);
  auto merge_adj = [&](std::vector<int32_t>& into, std::vector<int32_t>& from, size_t& cin, size_t cfrom, int32_t z) {
    if (from.size() > into.size()) { into.swap(from); cin = cfrom; }
    into.insert(into.end(), from.begin(), from.end());
    std::vector<int32_t>().swap(from);
    if (into.size() >= 2 * std::max<size_t>(cin, 16)) {
      for (int32_t& v : into) v = cg.root(v);
      std::sort(into.begin(), into.end());
      into.erase(std::unique(into.begin(), into.end()), into.end());
      into.erase(std::remove(into.begin(), into.end(), z), into.end());
      cin = into.size();
    }
  };
  auto push = [&](std::vector<uint64_t>& S, std::vector<uint64_t>* S2, std::vector<std::vector<int32_t>>& adj, int32_t z) {
    const uint64_t* sz = row(S, z);
    const uint64_t* sz2 = S2 ? row(*S2, z) : nullptr;
    stack.assign(adj[z].begin(), adj[z].end());
    while (!stack.empty()) {
      const int32_t w = cg.root(stack.back());
      stack.pop_back();
      if (w == z) continue;
      uint64_t* sw = row(S, w);
      bool sub = true;
      for (size_t q = 0; q < W && sub; ++q) sub = (sz[q] & ~sw[q]) == 0;
      if (sub) continue;
      for (size_t q = 0; q < W; ++q) sw[q] |= sz[q];
      ++pushed;
      if (S2) { uint64_t* s2 = row(*S2, w); for (size_t q = 0; q < W; ++q) s2[q] |= sz2[q]; }
      for (int32_t v : adj[w]) stack.push_back(v);
    }
  };
  for (uint64_t e : ekeys) {
    const int32_t x0 = (int32_t)(e >> 32), y0 = (int32_t)(uint32_t)e;
    const int32_t x = cg.root(x0), y = cg.root(y0);
    if (x == y) continue;
    if (reach_off[x0] < 0) { cg.join(x, y); a->contracted++; continue; }   // no conflict in this component
    {
      const uint64_t *ax = row(PA, x), *ay = row(PA, y), *dx = row(D, x), *dy = row(D, y);
      bool joins = false;
      for (size_t q = 0; q < W && !joins; ++q) joins = ((ax[q] | ay[q]) & (dx[q] | dy[q])) != 0;
      if (joins) { a->contract_rejected++; continue; }
    }
    const int32_t z = std::min(x, y), o2 = std::max(x, y);
    cg.join(x, y);
    a->contracted++;
    {
      uint64_t *az = row(A, z), *dz = row(D, z), *pz = row(PA, z);
      const uint64_t *ao = row(A, o2), *dox = row(D, o2), *po = row(PA, o2);
      for (size_t q = 0; q < W; ++q) { az[q] |= ao[q]; dz[q] |= dox[q]; pz[q] |= po[q]; }
    }
    {
      std::vector<size_t>& c = compacted;
      size_t co = c[o2];
      merge_adj(gout[z], gout[o2], c[z], co, z);
    }
    merge_adj(gin[z], gin[o2], in_compacted[z], in_compacted[o2], z);
    push(A, &PA, gout, z);   // descendants are now reached by A(z)
    push(D, nullptr, gin, z);   // ancestors now reach D(z)
  }
  if (getenv("TOAST_DEBUG"))
    fprintf(stderr, "[toast] contraction: %zu-word endpoint bitsets, %lld node updates pushed, main loop %.3f s\n", W,
            (long long)pushed, std::chrono::duration<double>(std::chrono::steady_clock::now() - t_init).count());
  a->cnode.resize(NL);
  for (int64_t l = 0; l < NL; ++l) a->cnode[l] = cg.root((int32_t)l);
  // sets
  std::map<std::pair<int32_t, int32_t>, int32_t> pair_set;
  std::vector<int32_t> set_first;
  for (int32_t i = 0; i < NC; ++i) {
    auto& c = a->conflicts[i];
    const int32_t U = a->cnode[c.u], V = a->cnode[c.v];
    auto it = pair_set.emplace(std::make_pair(std::min(U, V), std::max(U, V)), (int32_t)set_first.size());
    if (it.second) set_first.push_back(i);
    c.set = it.first->second;
    c.side0 = U == a->cnode[a->conflicts[set_first[c.set]].u] ? c.u : c.v;
  }
  n_sets = (int32_t)set_first.size();
  set_medges.assign(n_sets, {});
  std::vector<std::vector<int32_t>> ep_sets(NE);
  for (int32_t i = 0; i < NC; ++i) {
    const auto& c = a->conflicts[i];
    for (int32_t l : {c.u, c.v}) {
      auto& v = ep_sets[ep_index[l]];
      if (std::find(v.begin(), v.end(), c.set) == v.end()) v.push_back(c.set);
    }
  }
  for (uint64_t e : ekeys) {
    const int32_t x = (int32_t)(e >> 32), y = (int32_t)(uint32_t)e;
    if (ep_index[x] < 0 || ep_index[y] < 0 || a->cnode[x] != a->cnode[y]) continue;
    for (int32_t sx : ep_sets[ep_index[x]])
      for (int32_t sy : ep_sets[ep_index[y]])
        if (sx == sy) set_medges[sx].push_back({x, y});
  }
}

}  // namespace

toast_status build_analysis(const toast_graph* g, const toast_nda_opts* o, toast_analysis* a, std::string& err) {
  const int32_t n_ops = (int32_t)g->ops.size();
  const int n_axes = (int)g->axis_size.size();
  a->n_ops = n_ops;
  a->axis_size = g->axis_size;

  // ------------------------------------------------------------ C1 loops
  std::vector<OpLoops> OL(n_ops);
  std::vector<int64_t> lbeg(n_ops + 1, 0);
  for (int32_t t = 0; t < n_ops; ++t) {
    OL[t] = loops_of(g, g->ops[t]);
    if (OL[t].ext.size() > (size_t)MAX_LOOPS_PER_OP) { err = "op '" + g->ops[t].binding + "' has more than 8 loops"; return TOAST_E_LIMIT; }
    if (g->ops[t].operands.size() > (size_t)MAX_USES_PER_OP) { err = "op '" + g->ops[t].binding + "' has more than 8 operands"; return TOAST_E_LIMIT; }
    lbeg[t + 1] = lbeg[t] + (int64_t)OL[t].ext.size();
  }
  const int64_t NL = lbeg[n_ops];
  if (NL >= (int64_t)1 << 31) { err = "too many loops"; return TOAST_E_LIMIT; }
  a->n_loops = NL;
  a->loop_op.resize(NL); a->loop_role.resize(NL); a->loop_type.resize(NL); a->loop_ext.resize(NL);
  for (int32_t t = 0; t < n_ops; ++t)
    for (size_t r = 0; r < OL[t].ext.size(); ++r) {
      int64_t l = lbeg[t] + (int64_t)r;
      a->loop_op[l] = t; a->loop_role[l] = (int32_t)r; a->loop_type[l] = OL[t].type[r]; a->loop_ext[l] = OL[t].ext[r];
    }
  auto def_loop = [&](int32_t v, int i) { int32_t o2 = g->values[v].def_op; return (int32_t)(lbeg[o2] + OL[o2].res_role[i]); };
  auto use_loop = [&](int32_t t, int k, int i) { return (int32_t)(lbeg[t] + OL[t].use_role[k][i]); };

  // M edges over loops (deduplicated), CSR out-adjacency
  std::vector<uint64_t> ekeys;
  for (int32_t t = 0; t < n_ops; ++t)
    for (size_t k = 0; k < g->ops[t].operands.size(); ++k) {
      int32_t v = g->ops[t].operands[k];
      for (size_t i = 0; i < g->values[v].shape.size(); ++i)
        ekeys.push_back(((uint64_t)(uint32_t)def_loop(v, (int)i) << 32) | (uint32_t)use_loop(t, (int)k, (int)i));
    }
  std::sort(ekeys.begin(), ekeys.end());
  ekeys.erase(std::unique(ekeys.begin(), ekeys.end()), ekeys.end());
  a->n_edges = (int64_t)ekeys.size();
  std::vector<int64_t> out_off(NL + 1, 0);
  std::vector<int32_t> out_dst(ekeys.size());
  for (uint64_t e : ekeys) out_off[(e >> 32) + 1]++;
  for (int64_t l = 0; l < NL; ++l) out_off[l + 1] += out_off[l];
  for (size_t i = 0; i < ekeys.size(); ++i) out_dst[i] = (int32_t)(uint32_t)ekeys[i];   // sorted by src then dst

  // ------------------------------------------------------------ C2 components
  DSU cd(NL);
  for (uint64_t e : ekeys) cd.join((int32_t)(e >> 32), (int32_t)(uint32_t)e);
  a->loop_comp.resize(NL);
  for (int64_t l = 0; l < NL; ++l) a->loop_comp[l] = cd.root((int32_t)l);

  // ------------------------------------------------------------ C3 conflicts
  std::map<std::pair<int32_t, int32_t>, int32_t> conf_index;
  for (int32_t t = 0; t < n_ops; ++t) {
    const int nl = (int)OL[t].ext.size();
    uint64_t pairbits = 0;   // bit (u*8+v) for u<v roles that co-occur
    auto site = [&](const std::vector<uint8_t>& roles) {
      for (size_t x = 0; x < roles.size(); ++x)
        for (size_t y = x + 1; y < roles.size(); ++y) {
          int u = std::min(roles[x], roles[y]), v = std::max(roles[x], roles[y]);
          if (u != v) pairbits |= 1ULL << (u * 8 + v);
        }
    };
    if (g->ops[t].result >= 0) site(OL[t].res_role);
    for (auto& ur : OL[t].use_role) site(ur);
    for (int u = 0; u < nl; ++u)
      for (int v = u + 1; v < nl; ++v) {
        if (!(pairbits >> (u * 8 + v) & 1)) continue;
        if (OL[t].type[u] == T_X || OL[t].type[v] == T_X) continue;
        int32_t lu = (int32_t)(lbeg[t] + u), lv = (int32_t)(lbeg[t] + v);
        if (a->loop_comp[lu] != a->loop_comp[lv]) continue;
        conf_index[{lu, lv}] = (int32_t)a->conflicts.size();
        a->conflicts.push_back({t, lu, lv, -1, -1});
      }
  }
  const int32_t NC = (int32_t)a->conflicts.size();

  // ------------------------------------------------------------ C4 boxes
  // reachability bitsets over conflict endpoints, computed in reverse loop order
  // (every M edge goes from a lower to a higher loop id)
  std::vector<int32_t> ep_index(NL, -1);
  int32_t NE = 0;
  for (auto& c : a->conflicts) {
    if (ep_index[c.u] < 0) ep_index[c.u] = NE++;
    if (ep_index[c.v] < 0) ep_index[c.v] = NE++;
  }
  const size_t W = (size_t)(NE + 63) / 64;
  std::vector<char> comp_has_ep(NL, 0);
  for (auto& c : a->conflicts) comp_has_ep[a->loop_comp[c.u]] = 1;
  std::vector<int64_t> reach_off(NL, -1);
  int64_t nreach = 0;
  for (int64_t l = 0; l < NL; ++l) if (comp_has_ep[a->loop_comp[l]]) reach_off[l] = nreach++;
  std::vector<uint64_t> reach((size_t)nreach * W, 0);
  if (NC > 0) {
    for (int64_t l = NL - 1; l >= 0; --l) {
      if (reach_off[l] < 0) continue;
      uint64_t* dst = &reach[(size_t)reach_off[l] * W];
      for (int64_t e = out_off[l]; e < out_off[l + 1]; ++e) {
        int32_t m = out_dst[e];
        const uint64_t* src = &reach[(size_t)reach_off[m] * W];
        for (size_t w = 0; w < W; ++w) dst[w] |= src[w];
        if (ep_index[m] >= 0) dst[ep_index[m] >> 6] |= 1ULL << (ep_index[m] & 63);
      }
    }
  }
  auto reaches = [&](int32_t from, int32_t to) {
    int32_t e = ep_index[to];
    return (reach[(size_t)reach_off[from] * W + (e >> 6)] >> (e & 63)) & 1;
  };
  a->grouping = o->conflict_grouping;
  int32_t n_sets = 0;
  std::vector<std::vector<std::pair<int32_t, int32_t>>> set_medges;   // per set: the M edges its WL hash sees (C6)
  if (o->conflict_grouping == TOAST_GROUP_CONTRACTION) {
    build_contraction_sets(a, NL, ekeys, out_off, out_dst, ep_index, NE, reach, reach_off, n_sets, set_medges);
  } else {
  struct BoxRec { int32_t c1, c2, N, O, L, R, parity; };
  std::vector<BoxRec> boxes;
  for (int32_t ci = 0; ci < NC; ++ci) {
    const auto c1 = a->conflicts[ci];
    std::vector<BoxRec> mine;
    for (int lab = 0; lab < 2; ++lab) {
      int32_t N = lab ? c1.v : c1.u, O = lab ? c1.u : c1.v;
      for (int64_t e1 = out_off[N]; e1 < out_off[N + 1]; ++e1)
        for (int64_t e2 = out_off[O]; e2 < out_off[O + 1]; ++e2) {
          int32_t L = out_dst[e1], R = out_dst[e2];
          if (L == R || a->loop_op[L] != a->loop_op[R]) continue;
          auto it = conf_index.find({std::min(L, R), std::max(L, R)});
          if (it == conf_index.end()) continue;
          if (reaches(N, R) || reaches(O, L)) continue;
          const auto& c2 = a->conflicts[it->second];
          mine.push_back({ci, it->second, N, O, L, R, (int32_t)((N == c1.u) ^ (L == c2.u))});
        }
    }
    std::stable_sort(mine.begin(), mine.end(), [](const BoxRec& x, const BoxRec& y) { return x.c2 < y.c2; });
    for (size_t i = 0; i < mine.size(); ++i)
      if (i == 0 || mine[i].c2 != mine[i - 1].c2) boxes.push_back(mine[i]);
  }
  a->n_boxes = (int64_t)boxes.size();

  // ------------------------------------------------------------ C5 compatibility sets
  std::vector<int32_t> pp(NC);
  std::vector<uint8_t> px(NC, 0);   // parity to parent
  std::iota(pp.begin(), pp.end(), 0);
  auto pfind = [&](int32_t x, uint8_t& par) {
    // iterative: collect path, then compress
    std::vector<int32_t> path;
    while (pp[x] != x) { path.push_back(x); x = pp[x]; }
    uint8_t acc = 0;
    for (size_t i = path.size(); i-- > 0;) {
      int32_t y = path[i];
      acc ^= px[y];
      px[y] = acc;
      pp[y] = x;
    }
    par = path.empty() ? 0 : px[path[0]];
    return x;
  };
  std::vector<char> box_ok(boxes.size(), 0);
  for (size_t b = 0; b < boxes.size(); ++b) {
    uint8_t p1, p2;
    int32_t r1 = pfind(boxes[b].c1, p1), r2 = pfind(boxes[b].c2, p2);
    if (r1 == r2) {
      if ((p1 ^ p2) != boxes[b].parity) { a->dropped_boxes++; continue; }
      box_ok[b] = 1;
      continue;
    }
    pp[r2] = r1;
    px[r2] = (uint8_t)(p1 ^ p2 ^ boxes[b].parity);
    box_ok[b] = 1;
  }
  std::vector<int32_t> root_first(NC, -1);   // root -> smallest conflict
  std::vector<uint8_t> cpar(NC);
  std::vector<int32_t> croot(NC);
  for (int32_t i = 0; i < NC; ++i) {
    croot[i] = pfind(i, cpar[i]);
    if (root_first[croot[i]] < 0) root_first[croot[i]] = i;
  }
  std::vector<int32_t> set_of_root(NC, -1);
  for (int32_t i = 0; i < NC; ++i)
    if (root_first[croot[i]] == i) set_of_root[croot[i]] = n_sets++;
  for (int32_t i = 0; i < NC; ++i) {
    auto& c = a->conflicts[i];
    int32_t first = root_first[croot[i]];
    c.set = set_of_root[croot[i]];
    c.side0 = (cpar[i] ^ cpar[first]) ? c.v : c.u;
  }

  set_medges.assign(n_sets, {});
  for (size_t b = 0; b < boxes.size(); ++b) {
    if (!box_ok[b]) continue;
    auto& E = set_medges[a->conflicts[boxes[b].c1].set];
    E.push_back({boxes[b].N, boxes[b].L});
    E.push_back({boxes[b].O, boxes[b].R});
  }
  }   // compatibility sets

  // ------------------------------------------------------------ C6 SetGroups (3-round WL)
  a->set_sig.assign(n_sets, 0);
  {
    std::vector<std::vector<int32_t>> set_conf(n_sets);
    for (int32_t i = 0; i < NC; ++i) set_conf[a->conflicts[i].set].push_back(i);
    for (int32_t s = 0; s < n_sets; ++s) {
      std::map<int32_t, int> side;   // node -> side mask
      std::vector<std::pair<int32_t, int32_t>> cedges;
      for (int32_t i : set_conf[s]) {
        const auto& c = a->conflicts[i];
        int32_t s1 = c.side0 == c.u ? c.v : c.u;
        side[c.side0] |= 1;
        side[s1] |= 2;
        cedges.push_back({c.u, c.v});
      }
      auto& me = set_medges[s];
      std::sort(me.begin(), me.end());
      me.erase(std::unique(me.begin(), me.end()), me.end());
      std::sort(cedges.begin(), cedges.end());
      cedges.erase(std::unique(cedges.begin(), cedges.end()), cedges.end());
      std::vector<int32_t> nodes;
      for (auto& kv : side) nodes.push_back(kv.first);
      std::map<int32_t, size_t> pos;
      for (size_t i = 0; i < nodes.size(); ++i) pos[nodes[i]] = i;
      std::vector<uint64_t> lab(nodes.size());
      for (size_t i = 0; i < nodes.size(); ++i) {
        int32_t l = nodes[i];
        uint64_t x[4] = {fnv(g->ops[a->loop_op[l]].name), (uint64_t)a->loop_role[l], (uint64_t)a->loop_type[l],
                         (uint64_t)side[l]};
        lab[i] = hfold(x, 4);
      }
      for (int round = 0; round < 3; ++round) {
        std::vector<std::vector<uint64_t>> outs(nodes.size()), ins(nodes.size()), cfs(nodes.size());
        for (auto& e : me) { outs[pos[e.first]].push_back(lab[pos[e.second]]); ins[pos[e.second]].push_back(lab[pos[e.first]]); }
        for (auto& e : cedges) { cfs[pos[e.first]].push_back(lab[pos[e.second]]); cfs[pos[e.second]].push_back(lab[pos[e.first]]); }
        std::vector<uint64_t> nl(nodes.size());
        for (size_t i = 0; i < nodes.size(); ++i) {
          uint64_t x[4] = {lab[i], hfold(outs[i], true), hfold(ins[i], true), hfold(cfs[i], true)};
          nl[i] = hfold(x, 4);
        }
        lab.swap(nl);
      }
      a->set_sig[s] = hfold(lab, true);
    }
    std::map<uint64_t, int32_t> gid;
    a->set_group.assign(n_sets, -1);
    for (int32_t s = 0; s < n_sets; ++s) {
      auto it = gid.find(a->set_sig[s]);
      if (it == gid.end()) it = gid.emplace(a->set_sig[s], a->n_groups++).first;
      a->set_group[s] = it->second;
    }
  }
  if (a->n_groups > MAX_GROUPS) { err = "more than 64 SetGroups"; return TOAST_E_LIMIT; }

  // ------------------------------------------------------------ C7 argument groups, super-colors
  {
    std::map<std::vector<int64_t>, std::vector<int32_t>> groups;
    for (int32_t p = 0; p < g->n_params; ++p) {
      int32_t v = g->ops[p].result;
      const auto& shp = g->values[v].shape;
      std::vector<std::vector<std::array<int64_t, 4>>> per(shp.size());
      for (int32_t t = 0; t < n_ops; ++t)
        for (size_t k = 0; k < g->ops[t].operands.size(); ++k)
          if (g->ops[t].operands[k] == v)
            for (size_t i = 0; i < shp.size(); ++i) {
              int32_t l = use_loop(t, (int)k, (int)i);
              per[i].push_back({(int64_t)fnv(g->ops[t].name), (int64_t)k, (int64_t)a->loop_role[l], (int64_t)a->loop_type[l]});
            }
      std::vector<int64_t> key = {g->values[v].dtype_code, (int64_t)shp.size()};
      key.insert(key.end(), shp.begin(), shp.end());
      for (auto& d : per) {
        std::sort(d.begin(), d.end());
        key.push_back((int64_t)d.size());
        for (auto& q : d) key.insert(key.end(), q.begin(), q.end());
      }
      groups[key].push_back(v);
    }
    DSU sd(NL);
    for (int64_t l = 0; l < NL; ++l) sd.join((int32_t)l, a->loop_comp[l]);
    for (auto& kv : groups) {
      const auto& mem = kv.second;
      for (size_t j = 1; j < mem.size(); ++j)
        for (size_t i = 0; i < g->values[mem[0]].shape.size(); ++i) sd.join(def_loop(mem[0], (int)i), def_loop(mem[j], (int)i));
    }
    std::vector<int32_t> sc_of_root(NL, -1);
    a->loop_scolor.resize(NL);
    for (int64_t l = 0; l < NL; ++l) {
      int32_t r = sd.root((int32_t)l);
      if (sc_of_root[r] < 0) { sc_of_root[r] = (int32_t)a->sc_min_loop.size(); a->sc_min_loop.push_back((int32_t)l); }
      a->loop_scolor[l] = sc_of_root[r];
    }
  }
  const int32_t NSC = (int32_t)a->sc_min_loop.size();
  a->sc_value_dims.assign(NSC, 0);
  for (size_t v = 0; v < g->values.size(); ++v)
    for (size_t i = 0; i < g->values[v].shape.size(); ++i) a->sc_value_dims[a->loop_scolor[def_loop((int32_t)v, (int)i)]]++;
  a->sc_groups.assign(NSC, {});
  for (auto& c : a->conflicts) a->sc_groups[a->loop_scolor[c.u]].push_back(a->set_group[c.set]);
  for (auto& sg : a->sc_groups) { std::sort(sg.begin(), sg.end()); sg.erase(std::unique(sg.begin(), sg.end()), sg.end()); }

  // ------------------------------------------------------------ C8 action table
  a->actions.clear();
  a->actions.push_back({-1, 0, -1, 0});
  std::vector<int32_t> acolor_of_sc(NSC, -1), sc_of_acolor;
  for (int32_t c = 0; c < NSC; ++c) {
    if (a->sc_value_dims[c] < o->min_unique_dims) continue;
    if (a->sc_groups[c].size() > 8) { err = "more than 8 SetGroups in one super-color"; return TOAST_E_LIMIT; }
    acolor_of_sc[c] = (int32_t)sc_of_acolor.size();
    sc_of_acolor.push_back(c);
    for (int32_t r = 0; r < (1 << a->sc_groups[c].size()); ++r)
      for (int ax = 0; ax < n_axes; ++ax) a->actions.push_back({c, r, ax, (int32_t)a->sc_value_dims[c]});
  }
  if (a->actions.size() > (size_t)MAX_ACTIONS) { err = "more than 1023 actions"; return TOAST_E_LIMIT; }

  // ------------------------------------------------------------ packed tables
  const int32_t NA = (int32_t)a->actions.size();
  const int32_t nwords = (NA + 31) / 32;
  // deselection ids: need0 = groups where the loop is a side-1 endpoint (deselected when bit = 0),
  //                  need1 = groups where it is a side-0 endpoint (deselected when bit = 1)
  std::map<int32_t, std::pair<uint64_t, uint64_t>> dsel;
  for (auto& c : a->conflicts) {
    uint64_t gb = 1ULL << a->set_group[c.set];
    int32_t s1 = c.side0 == c.u ? c.v : c.u;
    dsel[s1].first |= gb;
    dsel[c.side0].second |= gb;
  }
  a->h_desel.assign(2, 0);   // id 0 = none
  std::map<int32_t, uint32_t> dsel_id;
  for (auto& kv : dsel) {
    dsel_id[kv.first] = (uint32_t)(a->h_desel.size() / 2);
    a->h_desel.push_back(kv.second.first);
    a->h_desel.push_back(kv.second.second);
  }
  if (a->h_desel.size() / 2 >= 65536) { err = "too many conflict endpoints"; return TOAST_E_LIMIT; }
  a->h_loops.resize(NL);
  for (int64_t l = 0; l < NL; ++l) {
    uint32_t ac = acolor_of_sc[a->loop_scolor[l]] >= 0 ? (uint32_t)acolor_of_sc[a->loop_scolor[l]] : NO_ACOLOR;
    if (a->loop_type[l] == T_X) ac = NO_ACOLOR;
    uint32_t div = 0;
    for (int S = 0; S < 16; ++S) {
      int64_t prod = 1;
      bool valid = true;
      for (int A = 0; A < 4; ++A) if (S >> A & 1) { if (A >= n_axes) valid = false; else prod *= g->axis_size[A]; }
      if (valid && a->loop_ext[l] % prod == 0) div |= 1u << S;
    }
    auto it = dsel_id.find((int32_t)l);
    uint64_t did = it == dsel_id.end() ? 0 : it->second;
    a->h_loops[l] = (uint64_t)ac | ((uint64_t)a->loop_type[l] << 10) | ((uint64_t)div << 12) | (did << 28);
  }
  // last uses and deaths (C12)
  std::vector<int32_t> last_use(g->values.size());
  for (size_t v = 0; v < g->values.size(); ++v) last_use[v] = g->values[v].def_op;
  for (int32_t t = 0; t < n_ops; ++t)
    for (int32_t v : g->ops[t].operands) last_use[v] = std::max(last_use[v], t);
  std::vector<std::vector<int32_t>> deaths(n_ops);
  for (size_t v = 0; v < g->values.size(); ++v) deaths[last_use[v]].push_back(g->values[v].def_op);
  a->h_ops.resize(n_ops);
  a->h_gflops.assign(n_ops, 0);
  a->h_uses.clear();
  a->h_deaths.clear();
  for (int32_t t = 0; t < n_ops; ++t) {
    const GOp& op = g->ops[t];
    DOp d{};
    d.loop_begin = (uint32_t)lbeg[t];
    d.n_loops = (uint8_t)OL[t].ext.size();
    d.rank = op.result >= 0 ? (uint8_t)g->values[op.result].shape.size() : 0;
    for (size_t r = 0; r < OL[t].type.size(); ++r) if (OL[t].type[r] == T_R) d.rmask |= (uint8_t)(1u << r);
    d.flags = (is_matmul_class(op.kind) ? 1 : 0) | (op.kind == OK_RET ? 2 : 0);
    for (size_t i = 0; i < OL[t].res_role.size(); ++i) d.res_roles |= (uint32_t)OL[t].res_role[i] << (4 * i);
    d.use_begin = (uint32_t)a->h_uses.size();
    d.n_uses = (uint8_t)op.operands.size();
    for (size_t k = 0; k < op.operands.size(); ++k) {
      DUse u{};
      u.def_op = (uint32_t)g->values[op.operands[k]].def_op;
      for (size_t i = 0; i < OL[t].use_role[k].size(); ++i) u.use_roles |= (uint32_t)OL[t].use_role[k][i] << (4 * i);
      a->h_uses.push_back(u);
    }
    d.death_begin = (uint32_t)a->h_deaths.size();
    d.n_death = (uint16_t)deaths[t].size();
    if (deaths[t].size() > 65535) { err = "too many values die at one op"; return TOAST_E_LIMIT; }
    for (int32_t v : deaths[t]) a->h_deaths.push_back((uint32_t)v);
    if (op.result >= 0) {
      uint64_t b = (uint64_t)g->values[op.result].elem_bytes;
      for (int64_t e : g->values[op.result].shape) b *= (uint64_t)e;
      d.gbytes = b;
    }
    if (d.flags & 1) {
      uint64_t f = 2;
      for (int64_t e : OL[t].ext) f *= (uint64_t)e;
      a->h_gflops[t] = f;
    }
    a->h_ops[t] = d;
  }
  // actions and per-acolor groups
  a->h_actions.assign(NA, 0);
  for (int32_t i = 1; i < NA; ++i) {
    const auto& ai = a->actions[i];
    a->h_actions[i] = (uint32_t)acolor_of_sc[ai.super_color] | ((uint32_t)ai.resolution << 10) | ((uint32_t)ai.axis << 18);
  }
  a->h_acol_groups.assign(sc_of_acolor.size(), 0);
  for (size_t ac = 0; ac < sc_of_acolor.size(); ++ac) {
    const auto& gs = a->sc_groups[sc_of_acolor[ac]];
    uint64_t w = 0;
    for (int t = 0; t < 8; ++t) w |= (uint64_t)(t < (int)gs.size() ? gs[t] : 0xFF) << (8 * t);
    a->h_acol_groups[ac] = w;
  }
  // kill masks (C15): chosen a kills b iff same (color, axis) or a shared group's bit disagrees
  a->h_kill.assign((size_t)NA * nwords, 0);
  for (int32_t x = 1; x < NA; ++x) {
    const auto& ax = a->actions[x];
    const auto& gx = a->sc_groups[ax.super_color];
    for (int32_t y = 1; y < NA; ++y) {
      const auto& ay = a->actions[y];
      bool kill = ax.super_color == ay.super_color && ax.axis == ay.axis;
      if (!kill) {
        const auto& gy = a->sc_groups[ay.super_color];
        for (size_t i = 0; i < gx.size() && !kill; ++i)
          for (size_t j = 0; j < gy.size(); ++j)
            if (gx[i] == gy[j] && (((ax.resolution >> i) ^ (ay.resolution >> j)) & 1)) { kill = true; break; }
      }
      if (kill) a->h_kill[(size_t)x * nwords + (y >> 5)] |= 1u << (y & 31);
    }
  }

  // ------------------------------------------------------------ device stream
  {
    // deselection classes: distinct (need0, need1) pairs; class 0 = never deselected
    std::map<std::pair<uint64_t, uint64_t>, uint32_t> cls_id;
    a->h_desel_cls.assign(2, 0);
    std::vector<uint32_t> loop_cls(NL, 0);
    for (auto& kv : dsel) {
      auto it = cls_id.find(kv.second);
      if (it == cls_id.end()) {
        it = cls_id.emplace(kv.second, (uint32_t)(a->h_desel_cls.size() / 2)).first;
        a->h_desel_cls.push_back(kv.second.first);
        a->h_desel_cls.push_back(kv.second.second);
      }
      loop_cls[kv.first] = it->second;
    }
    if (a->h_desel_cls.size() / 2 > 255) { err = "more than 255 deselection classes"; return TOAST_E_LIMIT; }
    // op signatures: the per-role words that decide materialisation (C9) plus
    // each role's result dim (so a candidate's entry also gives the result layout)
    auto resdim_of = [&](int32_t t) {
      uint32_t m = ~0u;
      for (size_t i = 0; i < OL[t].res_role.size(); ++i) {
        uint32_t r = OL[t].res_role[i];
        m = (m & ~(0xFu << (4 * r))) | ((uint32_t)i << (4 * r));
      }
      return m;
    };
    std::map<std::vector<uint64_t>, uint32_t> sig_id;
    std::vector<std::vector<uint64_t>> sig_words;
    std::vector<uint32_t> sig_rd;
    a->op_sig.assign(n_ops, 0);
    for (int32_t t = 0; t < n_ops; ++t) {
      std::vector<uint64_t> w;
      for (int64_t l = lbeg[t]; l < lbeg[t + 1]; ++l) {
        uint64_t ac = a->h_loops[l] & 0x3FF;
        if (ac == NO_ACOLOR) w.push_back(NO_ACOLOR);
        else w.push_back(ac | (((a->h_loops[l] >> 12) & 0xFFFF) << 10) | ((uint64_t)loop_cls[l] << 26));
      }
      while (!w.empty() && w.back() == NO_ACOLOR) w.pop_back();
      const uint32_t rd = resdim_of(t);
      std::vector<uint64_t> key = w;
      key.push_back((uint64_t)rd << 40 | 0xFFull << 32);   // disjoint from role words
      auto it = sig_id.find(key);
      if (it == sig_id.end()) {
        it = sig_id.emplace(key, (uint32_t)sig_words.size()).first;
        sig_words.push_back(w);
        sig_rd.push_back(rd);
      }
      a->op_sig[t] = it->second;
    }
    if (sig_words.size() > 65535) { err = "more than 65535 op signatures"; return TOAST_E_LIMIT; }
    if (getenv("TOAST_DEBUG")) {
      int hist[9] = {0};
      for (auto& w : sig_words) {
        std::vector<uint64_t> cs;
        for (uint64_t x : w) if ((x & 0x3FF) != NO_ACOLOR && std::find(cs.begin(), cs.end(), x & 0x3FF) == cs.end()) cs.push_back(x & 0x3FF);
        hist[std::min<size_t>(cs.size(), 8)]++;
      }
      int fast = 0;
      const uint32_t full = (1u << (1u << n_axes)) - 1u;
      for (auto& w : sig_words) {
        bool f = true;
        for (uint64_t x : w) if ((x & 0x3FF) != NO_ACOLOR && (((x >> 10) & 0xFFFF) & full) != full) f = false;
        fast += f;
      }
      fprintf(stderr, "[toast] signatures with every axis subset dividing every shardable role: %d of %zu\n", fast, sig_words.size());
      {
        std::map<std::vector<uint64_t>, int> uw;
        for (auto& w : sig_words) uw[w]++;
        fprintf(stderr, "[toast] materialisation classes (distinct role-word tuples): %zu of %zu signatures\n", uw.size(), sig_words.size());
      }
      fprintf(stderr, "[toast] signatures by distinct action colors:");
      for (int i = 0; i <= 8; ++i) fprintf(stderr, " %d:%d", i, hist[i]);
      fprintf(stderr, "\n");
    }
    a->h_sig_roles.assign(sig_words.size() * 8, NO_ACOLOR);
    a->h_sig_nroles.assign(sig_words.size(), 0);
    a->h_sig_resdim = sig_rd;
    for (size_t q = 0; q < sig_words.size(); ++q) {
      a->h_sig_nroles[q] = (uint8_t)sig_words[q].size();
      for (size_t r = 0; r < sig_words[q].size(); ++r) a->h_sig_roles[q * 8 + r] = sig_words[q][r];
    }
    // materialisation classes: signatures with the same role words (they differ
    // only in which role lands on which result dim) materialise identically
    std::vector<uint32_t> sig_mc(sig_words.size());
    std::vector<size_t> mc_rep;
    {
      std::map<std::vector<uint64_t>, uint32_t> mcid;
      for (size_t q = 0; q < sig_words.size(); ++q) {
        auto it = mcid.emplace(sig_words[q], (uint32_t)mc_rep.size());
        if (it.second) mc_rep.push_back(q);
        sig_mc[q] = it.first->second;
      }
    }
    a->h_sig_mr.assign(sig_words.size(), 0);
    for (size_t q = 0; q < sig_words.size(); ++q) a->h_sig_mr[q] = (uint64_t)sig_mc[q] | ((uint64_t)sig_rd[q] << 32);
    a->h_sigs.assign(mc_rep.size(), KSig{});
    for (size_t mcq = 0; mcq < mc_rep.size(); ++mcq) {
      const size_t q = mc_rep[mcq];
      KSig& k = a->h_sigs[mcq];
      k.nr = (uint8_t)sig_words[q].size();
      for (size_t r = 0; r < sig_words[q].size(); ++r) {
        const uint64_t w = sig_words[q][r];
        const uint32_t ac = (uint32_t)(w & 0x3FF);
        if (ac == NO_ACOLOR) continue;
        k.div[r >> 1] |= (uint32_t)((w >> 10) & 0xFFFF) << (16 * (r & 1));
        for (int A = 0; A < n_axes; ++A)
          if ((w >> (10 + (1u << A))) & 1) k.div1 |= 1u << (8 * A + r);
        const uint32_t cls = (uint32_t)(w >> 26) & 0xFF;
        if (cls) { k.dsel_roles |= (uint8_t)(1u << r); k.cls |= (uint64_t)cls << (8 * r); }
        int kk = 0;
        while (kk < k.m && (k.col[kk] & 0x3FF) != ac) ++kk;
        if (kk == k.m) k.col[k.m++] = ac;
        k.col[kk] |= 1u << (10 + r);
      }
      // every axis subset divides every shardable role: materialisation needs one round
      const uint32_t full = (1u << (1u << n_axes)) - 1u;
      bool all = true;
      for (size_t r = 0; r < sig_words[q].size(); ++r)
        if ((sig_words[q][r] & 0x3FF) != NO_ACOLOR && (((sig_words[q][r] >> 10) & 0xFFFF) & full) != full) all = false;
      k.pad = all ? 1 : 0;
    }
    // per-signature state-key terms (R14) and FLOP sums
    const size_t NS = sig_words.size();
    a->h_sig_key.assign(NS * 32, 0);
    a->h_sig_flops.assign(NS * 2, 0);
    for (int32_t t = 0; t < n_ops; ++t) {
      const uint32_t q = a->op_sig[t];
      for (int A = 0; A < 4; ++A)
        for (int r = 0; r < (int)OL[t].ext.size(); ++r)
          a->h_sig_key[q * 32 + A * 8 + r] += splitmix_fin(((uint64_t)lbeg[t] << 8) | ((uint64_t)A << 4) | (uint64_t)r);
      unsigned __int128 f = ((unsigned __int128)a->h_sig_flops[q * 2 + 1] << 64) | a->h_sig_flops[q * 2];
      f += a->h_gflops[t];
      a->h_sig_flops[q * 2] = (uint64_t)f;
      a->h_sig_flops[q * 2 + 1] = (uint64_t)(f >> 64);
    }
    // per materialisation class: the signatures share one axis -> role map, so
    // their state-key terms add per (axis, role) and their FLOP sums share one
    // exact divisor (every op's FLOPs divide exactly) — the kernels take both
    // once per class
    a->h_mc_key.assign(a->h_sigs.size() * 32, 0);
    a->h_mc_flops.assign(a->h_sigs.size() * 2, 0);
    for (size_t q = 0; q < NS; ++q) {
      const size_t c = (size_t)(a->h_sig_mr[q] & 0xFFFF);
      for (int i = 0; i < 32; ++i) a->h_mc_key[c * 32 + i] += a->h_sig_key[q * 32 + i];
      unsigned __int128 f = ((unsigned __int128)a->h_mc_flops[c * 2 + 1] << 64) | a->h_mc_flops[c * 2];
      f += ((unsigned __int128)a->h_sig_flops[q * 2 + 1] << 64) | a->h_sig_flops[q * 2];
      a->h_mc_flops[c * 2] = (uint64_t)f;
      a->h_mc_flops[c * 2 + 1] = (uint64_t)(f >> 64);
    }
    // edge templates (C11): use edges with the same (def signature, use
    // signature, use role->dim map) communicate identically for a candidate;
    // a value used more than once by one op is a "special" edge group, costed
    // edge by edge (within-op dedup, G26)
    // An edge whose def and use ops are of one materialisation class (the same
    // axis -> role map for every candidate) and whose every shardable role is
    // the same result dim and operand dim (none off the result: no partial sum)
    // has D == U and P empty for every candidate: it never communicates and
    // never grows a temporary, so it is left out of the tables altogether.
    // So is an edge from a def op no action can shard (D and P empty: at most
    // free slices, C11 phase 3).
    auto never_communicates = [&](int32_t d, int32_t t, uint32_t um) {
      const uint32_t sd = a->op_sig[d], su = a->op_sig[t];
      bool any = false;   // a def op no action can shard: D and P are empty, at most free slices
      for (int r = 0; r < 8; ++r) any |= (a->h_sig_roles[(size_t)sd * 8 + r] & 0x3FF) != NO_ACOLOR;
      if (!any) return true;
      if ((a->h_sig_mr[sd] & 0xFFFF) != (a->h_sig_mr[su] & 0xFFFF)) return false;
      const uint32_t rd = a->h_sig_resdim[sd];
      for (int r = 0; r < 8; ++r) {
        if ((a->h_sig_roles[(size_t)sd * 8 + r] & 0x3FF) == NO_ACOLOR) continue;
        const uint32_t dd = (rd >> (4 * r)) & 15, du = (um >> (4 * r)) & 15;
        if (dd == 15 || dd != du) return false;
      }
      return true;
    };
    int64_t n_silent = 0;
    std::map<std::tuple<uint32_t, uint32_t, uint32_t>, uint32_t> tmpl_id;
    std::set<std::tuple<uint32_t, uint32_t, uint32_t>> sig_tmpl;   // templates keyed by signatures (work count)
    a->h_tmpl.clear();
    std::vector<std::vector<std::pair<uint32_t, uint64_t>>> op_tmpl(n_ops);   // per op: (template, def bytes)
    std::vector<std::vector<KUse>> op_spec(n_ops);                            // per op: its special edges
    for (int32_t t = 0; t < n_ops; ++t) {
      const GOp& op = g->ops[t];
      std::vector<int> order(op.operands.size());
      std::iota(order.begin(), order.end(), 0);
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
        return g->values[op.operands[x]].def_op < g->values[op.operands[y]].def_op;
      });
      for (size_t q = 0; q < order.size(); ++q) {
        int k = order[q];
        int32_t v = g->values[op.operands[k]].def_op;
        bool first = q == 0 || g->values[op.operands[order[q - 1]]].def_op != v;
        bool last = q + 1 == order.size() || g->values[op.operands[order[q + 1]]].def_op != v;
        uint32_t um = ~0u;
        for (size_t i = 0; i < OL[t].use_role[k].size(); ++i) {
          uint32_t r = OL[t].use_role[k][i];
          um = (um & ~(0xFu << (4 * r))) | ((uint32_t)i << (4 * r));
        }
        const uint64_t gb = a->h_ops[v].gbytes;
        if (gb >> 48) { err = "a value larger than 2^48 bytes"; return TOAST_E_LIMIT; }
        if (first && last && never_communicates(v, t, um)) {
          ++n_silent;   // the same layout for every candidate: no collective, no growth (frontier weight 0)
          continue;
        }
        if (first && last) {   // the value is used once here: cost it through its template
          // keyed by the use op's materialisation class: only its axis -> role
          // map and this edge's role -> operand dim map decide the use layout
          const uint32_t umc = (uint32_t)(a->h_sig_mr[a->op_sig[t]] & 0xFFFFFFFFu);
          auto key = std::make_tuple(a->op_sig[v], umc, um);
          auto it = tmpl_id.find(key);
          if (it == tmpl_id.end()) {
            it = tmpl_id.emplace(key, (uint32_t)a->h_tmpl.size()).first;
            KTmpl tm{};
            tm.def_sig = (uint16_t)a->op_sig[v];
            tm.use_sig = (uint16_t)umc;
            tm.use_dimof = um;
            a->h_tmpl.push_back(tm);
          }
          KTmpl& tm = a->h_tmpl[it->second];
          if (tm.sum_gbytes + gb < tm.sum_gbytes) { err = "template byte sum overflows"; return TOAST_E_LIMIT; }
          tm.sum_gbytes += gb;
          tm.n_edges += 1;
          op_tmpl[t].push_back({it->second, gb});
          sig_tmpl.insert(std::make_tuple(a->op_sig[v], a->op_sig[t], um));
        } else {
          KUse u{};
          u.def_sig = (uint16_t)a->op_sig[v];
          u.tmpl = NO_TMPL;
          u.use_dimof = um;
          u.gb_flags = gb | ((uint64_t)((first ? 1 : 0) | (last ? 2 : 0)) << 56);
          op_spec[t].push_back(u);
        }
      }
    }
    if (a->h_tmpl.size() >= NO_TMPL) { err = "more than 65534 edge templates"; return TOAST_E_LIMIT; }
    if (getenv("TOAST_DEBUG"))
      fprintf(stderr, "[toast] %lld single use edges never communicate (no template)\n", (long long)n_silent);
    a->work_tmpl = (int64_t)sig_tmpl.size();
    a->work_sig_roles = 0;
    for (auto& w : sig_words) a->work_sig_roles += (int64_t)w.size();

    // peak-memory frontier (C12, reading R19).  For a candidate with
    // per-signature result divisors d_s and per-template growth factors g_tm,
    //   M_t = sum_s Live_t[s] / d_s + sum_tm Tmp_t[tm] * g_tm + special_t,
    // where Live_t[s] = global bytes of signature-s values live after t-1 plus
    // t's result, and Tmp_t[tm] = global bytes of t's template-tm edges (every
    // term is an exact integer: each value divides exactly).  M_t is linear in
    // the weights w = (1/d_s, g_tm), and w lies in the box
    //   1/prod(all axes) <= 1/d_s <= 1,   0 <= g_tm <= 1 - 1/prod(all axes)
    // (a signature none of whose result dims an action can shard has
    // 1/d_s = 1; a template whose def signature is such has g_tm = 0).  So op t
    // can be dropped whenever another kept op q has M_q >= M_t for EVERY w in
    // the box — peak = max_t M_t is unchanged, bit for bit.  Ops with special
    // edges are always kept (their own term is not linear).
    {
      const size_t NS = sig_words.size(), NT = a->h_tmpl.size(), D = 1 + NS + NT;   // [0] = constant
      int64_t prodall = 1;
      for (int A = 0; A < n_axes; ++A) prodall *= g->axis_size[A];
      std::vector<char> sig_fixed(NS, 1);
      for (size_t q = 0; q < NS; ++q)
        for (size_t r = 0; r < sig_words[q].size(); ++r)
          if ((sig_words[q][r] & 0x3FF) != NO_ACOLOR && ((sig_rd[q] >> (4 * r)) & 15) != 15) sig_fixed[q] = 0;
      // dmax[q]: the largest divisor a candidate can give signature q's result
      // layout — over every placement of distinct axes on its shardable
      // result-dim roles that keeps each role's extent divisible (div_ok)
      std::vector<int64_t> dmax(NS, 1);
      for (size_t q = 0; q < NS; ++q) {
        if (sig_fixed[q]) continue;
        int64_t n_assign = 1;
        for (int A = 0; A < n_axes; ++A) n_assign *= 9;   // each axis: one of 8 roles or none
        for (int64_t code = 0; code < n_assign; ++code) {
          int64_t c = code, d = 1;
          uint32_t per_role[8] = {0};
          bool ok = true;
          for (int A = 0; A < n_axes && ok; ++A) {
            const int r = (int)(c % 9) - 1;
            c /= 9;
            if (r < 0) continue;
            if (r >= (int)sig_words[q].size() || (sig_words[q][r] & 0x3FF) == NO_ACOLOR ||
                ((sig_rd[q] >> (4 * r)) & 15) == 15) { ok = false; break; }
            per_role[r] |= 1u << A;
            d *= g->axis_size[A];
          }
          for (int r = 0; r < 8 && ok; ++r)
            if (per_role[r] && !(((sig_words[q][r] >> 10) & 0xFFFF) >> per_role[r] & 1)) ok = false;
          if (ok && d > dmax[q]) dmax[q] = d;
        }
      }
      std::vector<int64_t> lo(D), hi(D);   // weight bounds x prodall (exact: dmax divides prodall)
      lo[0] = hi[0] = prodall;
      for (size_t q = 0; q < NS; ++q) { lo[1 + q] = prodall / dmax[q]; hi[1 + q] = prodall; }
      for (size_t q = 0; q < NT; ++q) { lo[1 + NS + q] = 0; hi[1 + NS + q] = prodall - prodall / dmax[a->h_tmpl[q].def_sig]; }
      // x >= y for every feasible w.  The feasible set is the box plus the
      // coupling g_tm <= 1 - 1/d_D (a template's growth 1/d_U - 1/d_D never
      // exceeds 1 - 1/d_D, with d_D its def signature's divisor — the same
      // weight as that signature's live-byte coordinate).  The minimum over
      // this set separates per signature s: with B_s = the sum of s's
      // templates' negative differences (each taking g at its cap) the
      // signature's coefficient becomes (diff_s - B_s), minimised at an
      // endpoint of [lo_s, hi_s]; positive template differences take g = 0.
      std::vector<std::vector<uint32_t>> sig_tmpls(NS);
      for (size_t q = 0; q < NT; ++q) sig_tmpls[a->h_tmpl[q].def_sig].push_back((uint32_t)q);
      auto geq = [&](const std::vector<int64_t>& x, const std::vector<int64_t>& y) {
        __int128 m = (__int128)(x[0] - y[0]) * prodall;
        for (size_t q = 0; q < NS; ++q) {
          const __int128 a_s = (__int128)x[1 + q] - y[1 + q];
          __int128 B = 0;
          for (uint32_t tm : sig_tmpls[q]) {
            const __int128 b = (__int128)x[1 + NS + tm] - y[1 + NS + tm];
            if (b < 0) B += b;
          }
          const __int128 coef = a_s - B;
          m += coef * (coef >= 0 ? lo[1 + q] : hi[1 + q]) + B * prodall;
        }
        return m >= 0;
      };
      std::vector<int64_t> Lv(NS, 0);
      std::vector<std::vector<int64_t>> P;
      std::vector<int32_t> Pt;
      for (int32_t t = 0; t < n_ops; ++t) {
        std::vector<int64_t> p(D, 0);
        for (size_t q = 0; q < NS; ++q) p[1 + q] = Lv[q];
        p[1 + a->op_sig[t]] += (int64_t)a->h_ops[t].gbytes;
        for (auto& e : op_tmpl[t]) p[1 + NS + e.first] += (int64_t)e.second;
        // fold the fixed weights into the constant
        for (size_t q = 0; q < NS; ++q)
          if (sig_fixed[q]) { p[0] += p[1 + q]; p[1 + q] = 0; }
        for (size_t q = 0; q < NT; ++q)
          if (hi[1 + NS + q] == 0) p[1 + NS + q] = 0;
        Lv[a->op_sig[t]] += (int64_t)a->h_ops[t].gbytes;
        for (int32_t v : deaths[t]) Lv[a->op_sig[v]] -= (int64_t)a->h_ops[v].gbytes;
        const bool special = !op_spec[t].empty();
        if (!special) {
          bool dom = false;
          for (auto& x : P) if (geq(x, p)) { dom = true; break; }
          if (dom) continue;
        }
        for (size_t i = 0; i < P.size();) {
          if (op_spec[Pt[i]].empty() && geq(p, P[i])) {
            P[i] = std::move(P.back()); P.pop_back();
            Pt[i] = Pt.back(); Pt.pop_back();
          } else {
            ++i;
          }
        }
        P.push_back(std::move(p));
        Pt.push_back(t);
      }
      std::vector<size_t> ord(P.size());
      std::iota(ord.begin(), ord.end(), 0);
      std::sort(ord.begin(), ord.end(), [&](size_t x, size_t y) { return Pt[x] < Pt[y]; });
      a->h_points.clear();
      a->h_terms.clear();
      a->h_spec.clear();
      a->point_op.clear();
      // points in program order, in groups of FRONTIER_GROUP: a group's first
      // point carries its constant and signature terms absolutely, the others
      // as signed differences from the previous point (consecutive frontier
      // ops share most of their live set); template terms are per point
      const std::vector<int64_t>* prev = nullptr;
      for (size_t n = 0; n < ord.size(); ++n) {
        const auto& p = P[ord[n]];
        const int32_t t = Pt[ord[n]];
        const bool anchor = n % FRONTIER_GROUP == 0;
        for (size_t d = 0; d < D; ++d)
          if ((uint64_t)p[d] >> 47) { err = "a live-byte sum of 2^47 bytes or more"; return TOAST_E_LIMIT; }
        KPoint kp{};
        kp.term_begin = (uint32_t)a->h_terms.size();
        auto term = [&](int64_t v, size_t fid) { return ((uint64_t)v & ((1ULL << 48) - 1)) | ((uint64_t)fid << 48); };
        a->h_terms.push_back((uint64_t)(anchor ? p[0] : p[0] - (*prev)[0]));
        a->work_terms += 1;
        for (size_t d = 1; d < D; ++d) a->work_terms += p[d] != 0;   // the point's absolute terms
        for (size_t q = 0; q < NS; ++q) {
          const int64_t v = anchor ? p[1 + q] : p[1 + q] - (*prev)[1 + q];
          if (v) { a->h_terms.push_back(term(v, q)); ++kp.n_sig; }
        }
        for (size_t q = 0; q < NT; ++q)
          if (p[1 + NS + q]) { a->h_terms.push_back(term(p[1 + NS + q], q)); ++kp.n_tmpl; }
        kp.spec_begin = (uint32_t)a->h_spec.size();
        kp.n_spec = (uint16_t)op_spec[t].size();
        if (op_spec[t].size() > 65535) { err = "too many repeated operands at one op"; return TOAST_E_LIMIT; }
        kp.use_sig = (uint16_t)a->op_sig[t];
        for (auto& u : op_spec[t]) a->h_spec.push_back(u);
        a->h_points.push_back(kp);
        a->point_op.push_back(t);
        prev = &p;
      }
      // compact the frontier's feature ids: only the signatures and templates
      // a term uses get a per-lane code slot in the kernels' shared memory
      std::vector<uint32_t> sslot(NS, 0xFFFFu), tslot(NT, 0xFFFFFFFFu);
      uint32_t nfs = 0, nft = 0;
      for (const KPoint& kp : a->h_points) {
        uint64_t* tp = a->h_terms.data() + kp.term_begin + 1;
        for (uint32_t k = 0; k < kp.n_sig; ++k, ++tp) {
          const uint32_t f = (uint32_t)(*tp >> 48);
          if (sslot[f] == 0xFFFFu) sslot[f] = nfs++;
          *tp = (*tp & ((1ULL << 48) - 1)) | ((uint64_t)sslot[f] << 48);
        }
        for (uint32_t k = 0; k < kp.n_tmpl; ++k, ++tp) {
          const uint32_t f = (uint32_t)(*tp >> 48);
          if (tslot[f] == 0xFFFFFFFFu) tslot[f] = nft++;
          *tp = (*tp & ((1ULL << 48) - 1)) | ((uint64_t)tslot[f] << 48);
        }
      }
      for (size_t q = 0; q < NS; ++q) a->h_sig_mr[q] = (a->h_sig_mr[q] & ~0xFFFF0000ULL) | ((uint64_t)sslot[q] << 16);
      for (size_t q = 0; q < NT; ++q) a->h_tmpl[q].fslot = tslot[q];
      a->dt.n_fsig = (int32_t)nfs;
      a->dt.n_ftmpl = (int32_t)nft;
    }
    if (getenv("TOAST_DEBUG"))
      fprintf(stderr, "[toast] ops %d loops %lld signatures %zu templates %zu frontier points %zu terms %zu actions %zu desel classes %zu\n",
              n_ops, (long long)NL, sig_words.size(), a->h_tmpl.size(), a->h_points.size(), a->h_terms.size(),
              a->actions.size(), a->h_desel_cls.size() / 2);
  }

  // ------------------------------------------------------------ critical-path stream (reading R22)
  a->cost_model = o->cost_model;
  int32_t n_slots = 0;
  a->h_cp.clear();
  a->h_cp_comm.clear();
  a->h_cp_comp.clear();
  if (o->cost_model == TOAST_COST_CRITICAL_PATH) {
    // Edge durations are shared by every edge of the same communication class
    // (def signature, use materialisation class, use role -> dim map, bytes),
    // compute times by every op of the same (signature, FLOPs) class: the
    // kernels evaluate each class once per candidate.
    //
    // Exact reductions of the max-plus walk (every finish time is >= +0, so
    // x + 0.0 == x bit for bit):
    //  * an edge whose def and use ops are of one materialisation class and
    //    whose every shardable role is the same result / operand dim, with no
    //    shardable role off the result (no partial sum), never communicates:
    //    its duration is 0 for every candidate, the walk takes the def's
    //    finish as is (ZERO_COMM, no class, no add);
    //  * an op without compute time whose single operand edge is such an edge
    //    finishes exactly when its operand does: it is elided and its result
    //    shares the operand's finish (an alias), so it costs nothing per
    //    candidate and the latest finish is unchanged.
    // Finish-time slots are then held per alias class, from the def of its
    // first value to the last use of any of its values (reused greedily);
    // parameters finish at 0 and need none.
    auto shardable_roles = [&](uint32_t sig) {
      uint32_t m = 0;
      for (int r = 0; r < 8; ++r)
        if ((a->h_sig_roles[(size_t)sig * 8 + r] & 0x3FF) != NO_ACOLOR) m |= 1u << r;
      return m;
    };
    auto use_dimof = [&](int32_t t, size_t k) {
      uint32_t um = ~0u;
      for (size_t i = 0; i < OL[t].use_role[k].size(); ++i) {
        uint32_t rr = OL[t].use_role[k][i];
        um = (um & ~(0xFu << (4 * rr))) | ((uint32_t)i << (4 * rr));
      }
      return um;
    };
    auto zero_edge = [&](int32_t t, size_t k) {
      const int32_t d = g->values[g->ops[t].operands[k]].def_op;
      const uint32_t sd = a->op_sig[d], su = a->op_sig[t];
      if (!shardable_roles(sd)) return true;   // a def no action can shard: at most free slices
      if ((a->h_sig_mr[sd] & 0xFFFF) != (a->h_sig_mr[su] & 0xFFFF)) return false;
      const uint32_t rd = a->h_sig_resdim[sd], um = use_dimof(t, k), sh = shardable_roles(sd);
      for (int r = 0; r < 8; ++r) {
        if (!((sh >> r) & 1)) continue;
        const uint32_t dd = (rd >> (4 * r)) & 15, du = (um >> (4 * r)) & 15;
        if (dd == 15 || dd != du) return false;
      }
      return true;
    };
    const size_t NV = g->values.size();
    std::vector<int32_t> fid(NV);                 // alias class of each value's finish (a value id)
    std::iota(fid.begin(), fid.end(), 0);
    std::vector<char> elided(n_ops, 0);
    std::vector<uint32_t> zero_bits(n_ops, 0);    // bit k: operand k's edge never communicates
    for (int32_t t = 0; t < n_ops; ++t)
      for (size_t k = 0; k < g->ops[t].operands.size(); ++k)
        if (zero_edge(t, k)) zero_bits[t] |= 1u << k;
    // Dominated edges.  A finish is never below the finish of anything that
    // reaches it (every term is >= 0 and rounding is monotone), so an edge from
    // x into t can never win t's max over another operand edge from y when x
    // reaches y (or x is a parameter, finish 0) and the x edge's duration is
    // never larger: it never communicates (term finish(x) <= finish(y) <=
    // finish(y) + d), or both edges are of one duration class (finish(x) + d <=
    // finish(y) + d, rounding is monotone).  Such edges are dropped.  Among
    // edges from one value with one duration the first is kept; an operand
    // that reaches no other operand always keeps an edge.
    auto edge_class_key = [&](int32_t t, size_t k) {
      const int32_t d = g->values[g->ops[t].operands[k]].def_op;
      return std::make_tuple((uint32_t)a->op_sig[d], (uint32_t)(a->h_sig_mr[a->op_sig[t]] & 0xFFFFFFFFu),
                             use_dimof(t, k), a->h_ops[d].gbytes);
    };
    std::vector<uint32_t> drop_bits(n_ops, 0);
    {
      std::vector<int32_t> src_of(n_ops, -1);   // source index of non-parameter defs feeding multi-operand ops
      int32_t NSRC = 0;
      for (int32_t t = 0; t < n_ops; ++t) {
        const GOp& op = g->ops[t];
        if (op.operands.size() < 2) continue;
        for (int32_t v : op.operands) {
          const int32_t d = g->values[v].def_op;
          if (g->ops[d].kind != OK_PARAM && src_of[d] < 0) src_of[d] = NSRC++;
        }
      }
      const size_t WS = (size_t)(NSRC + 63) / 64;
      std::vector<uint64_t> R((size_t)n_ops * WS, 0);   // R[op]: sources reaching op (itself included)
      for (int32_t t = 0; t < n_ops && WS; ++t) {
        uint64_t* rt = &R[(size_t)t * WS];
        for (int32_t v : g->ops[t].operands) {
          const uint64_t* rd = &R[(size_t)g->values[v].def_op * WS];
          for (size_t w = 0; w < WS; ++w) rt[w] |= rd[w];
        }
        if (src_of[t] >= 0) rt[src_of[t] >> 6] |= 1ULL << (src_of[t] & 63);
      }
      for (int32_t t = 0; t < n_ops; ++t) {
        const GOp& op = g->ops[t];
        const size_t nk = op.operands.size();
        if (nk < 2) continue;
        for (size_t k = 0; k < nk; ++k) {
          const bool zk = (zero_bits[t] >> k) & 1;
          const int32_t xk = op.operands[k], dk = g->values[xk].def_op;
          bool dom = false;
          for (size_t j = 0; j < nk && !dom; ++j) {
            if (j == k) continue;
            const bool zj = (zero_bits[t] >> j) & 1;
            const bool no_longer = zk || (!zj && edge_class_key(t, k) == edge_class_key(t, j));
            if (!no_longer) continue;
            const int32_t xj = op.operands[j], dj = g->values[xj].def_op;
            if (xj == xk) dom = zk == zj ? j < k : zk;   // same value: keep the first of equal durations
            else if (g->ops[dk].kind == OK_PARAM) dom = true;
            else dom = (R[(size_t)dj * WS + (src_of[dk] >> 6)] >> (src_of[dk] & 63)) & 1;
          }
          if (dom) drop_bits[t] |= 1u << k;
        }
      }
    }
    for (int32_t t = 0; t < n_ops; ++t) {
      const GOp& op = g->ops[t];
      if (op.kind == OK_PARAM || (a->h_ops[t].flags & 1)) continue;
      int32_t kept = -1, n_kept = 0;
      for (size_t k = 0; k < op.operands.size(); ++k)
        if (!((drop_bits[t] >> k) & 1)) { kept = (int32_t)k; ++n_kept; }
      if (n_kept == 1 && ((zero_bits[t] >> kept) & 1)) {
        elided[t] = 1;
        if (op.result >= 0) fid[op.result] = fid[op.operands[kept]];
      }
    }
    // The walk runs in BUNDLES of at most CP_EMAX operand edges whose ops read
    // no finish produced inside the same bundle: the kernel issues all of a
    // bundle's loads before it combines them, so a bundle costs one memory
    // round trip instead of one per op.  Any topological order gives the same
    // finish times (each is a function of its operands', in operand order) and
    // the same latest finish (max is exact), so the schedule is free: ops are
    // taken greedily in program order from a window of CP_WINDOW ops past the
    // first unscheduled one (the window bounds how far liveness can stretch).
    std::map<std::tuple<uint32_t, uint32_t, uint32_t, uint64_t>, uint32_t> comm_id;
    std::map<std::pair<uint32_t, uint64_t>, uint32_t> comp_id;
    struct WOp { int32_t t; uint32_t comp; int32_t e0, ne; };
    struct WEdge { int32_t cls_val; uint32_t comm; };   // alias class of the operand (value id), class / ZERO_COMM
    std::vector<WOp> wops;
    std::vector<WEdge> wedges;
    std::vector<int32_t> producer(NV, -1);   // walked op index producing an alias class
    for (int32_t t = 0; t < n_ops; ++t) {
      const GOp& op = g->ops[t];
      if (elided[t] || op.kind == OK_PARAM) continue;   // parameters finish at 0 and hold no slot
      WOp w{t, NO_CLASS, (int32_t)wedges.size(), 0};
      if (a->h_ops[t].flags & 1) {
        auto it = comp_id.emplace(std::make_pair(a->op_sig[t], a->h_gflops[t]), (uint32_t)a->h_cp_comp.size());
        if (it.second) {
          KCpComp c{};
          c.sig = a->op_sig[t];
          c.gflops = a->h_gflops[t];
          a->h_cp_comp.push_back(c);
        }
        w.comp = it.first->second;
      }
      const uint32_t umc = (uint32_t)(a->h_sig_mr[a->op_sig[t]] & 0xFFFFFFFFu);
      for (size_t k = 0; k < op.operands.size(); ++k) {
        if ((drop_bits[t] >> k) & 1) continue;
        const int32_t v = op.operands[k];
        const int32_t d = g->values[v].def_op;
        uint32_t cls = ZERO_COMM;
        if (!((zero_bits[t] >> k) & 1)) {
          const uint32_t um = use_dimof(t, k);
          auto it = comm_id.emplace(std::make_tuple((uint32_t)a->op_sig[d], umc, um, a->h_ops[d].gbytes),
                                    (uint32_t)a->h_cp_comm.size());
          if (it.second) {
            KCpComm c{};
            c.def_sig = (uint16_t)a->op_sig[d];
            c.use_mc = (uint16_t)umc;
            c.use_dimof = um;
            c.gb = a->h_ops[d].gbytes;
            a->h_cp_comm.push_back(c);
          }
          cls = it.first->second;
        }
        wedges.push_back({fid[v], cls});
      }
      if (op.operands.empty()) wedges.push_back({-1, ZERO_COMM});   // finish = its own compute time
      w.ne = (int32_t)wedges.size() - w.e0;
      if (op.result >= 0) producer[op.result] = (int32_t)wops.size();
      wops.push_back(w);
    }
    const int32_t NW = (int32_t)wops.size();
    // bundles
    std::vector<int32_t> bundle_of(NW, -1), order;
    std::vector<uint32_t> bsize;
    {
      int32_t lo = 0, nb = 0;
      const char* em = getenv("TOAST_CP_EMAX");   // bundle width experiments (<= CP_EMAX)
      const int32_t emax = em ? std::max(1, std::min(CP_EMAX, atoi(em))) : CP_EMAX;
      const char* fw = getenv("TOAST_CP_FWD");    // 0: no in-bundle forwarding (experiments)
      const bool fwd = !fw || atoi(fw) != 0;
      while (lo < NW) {
        int32_t used = 0;
        for (int32_t i = lo; i < NW && i < lo + CP_WINDOW; ++i) {
          if (bundle_of[i] >= 0 || (used + wops[i].ne > emax && used > 0)) continue;
          bool ready = true;
          for (int32_t e = wops[i].e0; e < wops[i].e0 + wops[i].ne && ready; ++e) {
            const int32_t cv = wedges[e].cls_val;
            const int32_t pr = cv >= 0 ? producer[cv] : -1;
            // a producer in this bundle hands its finish over in a register
            if (pr >= 0 && (bundle_of[pr] < 0 || (!fwd && bundle_of[pr] == nb))) ready = false;
          }
          if (!ready) continue;
          bundle_of[i] = nb;
          order.push_back(i);
          used += wops[i].ne;
        }
        bsize.push_back((uint32_t)used);
        ++nb;
        while (lo < NW && bundle_of[lo] >= 0) ++lo;
      }
    }
    const int32_t NB = (int32_t)bsize.size();
    if (getenv("TOAST_DEBUG")) {   // the walked DAG's depth: no schedule needs fewer bundles
      std::vector<int32_t> lvl(NW, 0);
      int32_t depth = 0;
      for (int32_t i = 0; i < NW; ++i) {
        for (int32_t e = wops[i].e0; e < wops[i].e0 + wops[i].ne; ++e) {
          const int32_t cv = wedges[e].cls_val;
          const int32_t pr = cv >= 0 ? producer[cv] : -1;
          if (pr >= 0) lvl[i] = std::max(lvl[i], lvl[pr] + 1);
        }
        depth = std::max(depth, lvl[i] + 1);
      }
      fprintf(stderr, "[toast] critical path: walked DAG depth %d, %d bundles\n", depth, NB);
    }
    // finish slots per alias class, held from its producer's bundle to the last
    // bundle reading it; a class read only inside its producer's bundle (in
    // registers) needs none
    std::vector<int32_t> last_b(NV, -1);
    std::vector<char> needs_slot(NV, 0);
    for (int32_t i = 0; i < NW; ++i)
      if (g->ops[wops[i].t].result >= 0) last_b[g->ops[wops[i].t].result] = bundle_of[i];
    for (int32_t i = 0; i < NW; ++i)
      for (int32_t e = wops[i].e0; e < wops[i].e0 + wops[i].ne; ++e) {
        const int32_t cv = wedges[e].cls_val;
        if (cv < 0 || producer[cv] < 0) continue;
        last_b[cv] = std::max(last_b[cv], bundle_of[i]);
        if (bundle_of[producer[cv]] != bundle_of[i]) needs_slot[cv] = 1;
      }
    std::vector<std::vector<int32_t>> b_deaths(NB);
    for (size_t v = 0; v < NV; ++v) if (last_b[v] >= 0) b_deaths[last_b[v]].push_back((int32_t)v);
    std::vector<uint32_t> slot_of(NV, NO_SLOT), free_slots;
    std::vector<int32_t> recs;   // walked ops in bundle order
    size_t oi = 0;
    for (int32_t b = 0; b < NB; ++b) {
      const size_t ob = oi;
      for (; oi < order.size() && bundle_of[order[oi]] == b; ++oi) {
        const int32_t res = g->ops[wops[order[oi]].t].result;
        if (res >= 0 && needs_slot[res]) {
          if (free_slots.empty()) free_slots.push_back((uint32_t)n_slots++);
          slot_of[res] = free_slots.back();
          free_slots.pop_back();
        }
      }
      for (size_t q = ob; q < oi; ++q) recs.push_back((int32_t)order[q]);
      for (int32_t c : b_deaths[b])
        if (slot_of[c] != NO_SLOT) free_slots.push_back(slot_of[c]);
    }
    if (n_slots + 2 > 0x7FFF || a->h_cp_comm.size() + a->h_cp_comp.size() + 1 > 0x7FFF) {
      err = "critical-path stream limits (32765 finish slots, 32766 duration classes)";
      return TOAST_E_LIMIT;
    }
    // records in bundle order; indices into the block's scratch (kernels.cu cp_stride):
    // classes [communication | compute | zero], slots [finish slots | zero | trash]
    const uint32_t zero_cls = (uint32_t)(a->h_cp_comm.size() + a->h_cp_comp.size());
    const uint32_t zero_slot = (uint32_t)n_slots, trash_slot = (uint32_t)n_slots + 1;
    std::vector<int32_t> last_pos(NW, -1);   // position of an op's last edge inside its bundle
    {
      int32_t cur_b = -1, pos = 0;
      for (int32_t wi : recs) {
        const WOp& w = wops[wi];
        if (bundle_of[wi] != cur_b) { cur_b = bundle_of[wi]; pos = 0; }
        const int32_t res = g->ops[w.t].result;
        const uint32_t rs = (res >= 0 && slot_of[res] != NO_SLOT) ? slot_of[res] : trash_slot;
        const uint32_t ct = w.comp == NO_CLASS ? zero_cls : (uint32_t)a->h_cp_comm.size() + w.comp;
        for (int32_t e = w.e0; e < w.e0 + w.ne; ++e, ++pos) {
          const int32_t cv = wedges[e].cls_val;
          const int32_t pr = (cv >= 0) ? producer[cv] : -1;
          const bool fwd_e = pr >= 0 && bundle_of[pr] == cur_b;   // x bit 15: the finish of edge fs of this bundle
          const uint32_t fs = fwd_e ? (uint32_t)last_pos[pr] : pr >= 0 ? slot_of[cv] : zero_slot;
          const uint32_t dur = wedges[e].comm == ZERO_COMM ? zero_cls : wedges[e].comm;
          const uint32_t first = e == w.e0, last = e == w.e0 + w.ne - 1;
          a->h_cp.push_back(fs | (uint32_t)fwd_e << 15 | dur << 16 | first << 31);
          a->h_cp.push_back((last ? rs : trash_slot) | (last ? ct : zero_cls) << 16 | last << 31);
        }
        last_pos[wi] = pos - 1;
      }
    }
    // Prefetch hints: a finish read long after it was written (a forward
    // activation read by the backward pass) has left the L2 by then; the bundle
    // PF_DIST bundles before the read prefetches it into L2 (two hints per
    // bundle header; a read with no free header slot in reach goes without).
    {
      const char* pd = getenv("TOAST_CP_PF_DIST");
      const char* pc = getenv("TOAST_CP_PF_COLD");
      const int32_t dist = pd ? atoi(pd) : 6, cold = pc ? atoi(pc) : 16;
      std::vector<uint32_t> pf(NB * 2, 0x3FFF);
      for (int32_t wi : recs) {
        const int32_t b = bundle_of[wi];
        const WOp& w = wops[wi];
        for (int32_t e = w.e0; e < w.e0 + w.ne && dist > 0 && n_slots < 0x3FFF; ++e) {
          const int32_t cv = wedges[e].cls_val;
          if (cv < 0 || producer[cv] < 0 || slot_of[cv] == NO_SLOT) continue;
          const int32_t pb = bundle_of[producer[cv]];
          if (b - pb <= cold) continue;
          for (int32_t t = std::max(pb + 1, b - dist); t >= pb + 1 && t >= b - 4 * dist; --t) {
            if (pf[2 * t] == 0x3FFF) { pf[2 * t] = slot_of[cv]; break; }
            if (pf[2 * t + 1] == 0x3FFF) { pf[2 * t + 1] = slot_of[cv]; break; }
          }
        }
      }
      for (int32_t i = 0; i < NB; ++i) bsize[i] |= pf[2 * i] << 4 | pf[2 * i + 1] << 18;
    }
    a->h_cp_bsize = bsize;
    a->cp_walked_ops = NW;
    a->cp_walked_edges = (int32_t)wedges.size();
    if (getenv("TOAST_DEBUG"))
      fprintf(stderr, "[toast] critical path: %d of %d ops walked (%zu edges) in %d bundles, %d finish slots, "
              "%zu communication classes, %zu compute classes\n", NW, n_ops, wedges.size(), NB, n_slots,
              a->h_cp_comm.size(), a->h_cp_comp.size());
  }
  a->dt.n_slots = n_slots;
  a->dt.n_comm = (int32_t)a->h_cp_comm.size();
  a->dt.n_comp = (int32_t)a->h_cp_comp.size();
  a->dt.cost_model = o->cost_model;

  // ------------------------------------------------------------ baseline (empty sequence)
  {
    unsigned __int128 fl = 0;
    for (int32_t t = 0; t < n_ops; ++t) fl += a->h_gflops[t];
    int64_t L = 0, peak = 0;
    for (int32_t t = 0; t < n_ops; ++t) {
      int64_t res = (int64_t)a->h_ops[t].gbytes;
      peak = std::max(peak, L + res);
      int64_t dy = 0;
      for (int32_t v : deaths[t]) dy += (int64_t)a->h_ops[v].gbytes;
      L += res - dy;
    }
    uint64_t lo = (uint64_t)fl, hi = (uint64_t)(fl >> 64);
    volatile double fhi = (double)hi;
    double fd = fhi * 18446744073709551616.0;
    fd = fd + (double)lo;
    double t0 = fd / g->machine.flops_per_sec;
    if (o->cost_model == TOAST_COST_CRITICAL_PATH) {
      // R22 with nothing sharded: no collectives; finish(t) = max over operands
      // of finish(def) + t's compute time (global FLOPs / F)
      std::vector<double> fin(g->values.size(), 0.0);
      double cp = 0.0;
      for (int32_t t = 0; t < n_ops; ++t) {
        const GOp& op = g->ops[t];
        double ready = 0.0;
        for (int32_t v : op.operands) {
          volatile double f = fin[v] + 0.0;
          if (f > ready) ready = f;
        }
        const double ct = (double)a->h_gflops[t] / g->machine.flops_per_sec;
        const double ft = ready + ct;
        if (op.result >= 0) fin[op.result] = ft;
        if (ft > cp) cp = ft;
      }
      t0 = cp;
    }
    if (!(t0 > 0.0)) { err = "baseline runtime is 0: the program has no contraction op"; return TOAST_E_DEGENERATE; }
    a->t0 = t0;
    a->peak0 = (uint64_t)peak;
    memset(&a->baseline, 0, sizeof(a->baseline));
    a->baseline.runtime_s = t0;
    a->baseline.peak_bytes = (uint64_t)peak;
    a->baseline.flops = lo;
    a->baseline.flops_hi = hi;
    double MP = (uint64_t)peak > g->machine.device_memory_bytes
                    ? (g->machine.penalty_c * (double)((uint64_t)peak - g->machine.device_memory_bytes)) / (double)peak
                    : 0.0;
    a->baseline.score = t0 / t0 + MP;
  }

  // ------------------------------------------------------------ constants
  DeviceTables& T = a->dt;
  T.n_ops = n_ops;
  T.n_loops = (int32_t)NL;
  T.n_actions = NA;
  T.n_acolors = (int32_t)sc_of_acolor.size();
  T.n_words = nwords;
  T.n_axes = n_axes;
  T.max_depth = o->max_depth;
  T.n_sigs = (int32_t)a->h_sig_nroles.size();
  T.n_mc = (int32_t)a->h_sigs.size();
  T.n_tmpl = (int32_t)a->h_tmpl.size();
  T.n_points = (int32_t)a->h_points.size();
  T.pow2 = 1;
  for (int A = 0; A < n_axes; ++A) if (g->axis_size[A] & (g->axis_size[A] - 1)) T.pow2 = 0;
  for (int A = 0; A < 4; ++A) {
    T.sizes[A] = A < n_axes ? g->axis_size[A] : 1;
    T.bw[A] = A < n_axes ? g->axis_bw[A] : 1.0;
  }
  T.F = g->machine.flops_per_sec;
  T.C = g->machine.penalty_c;
  T.DM = g->machine.device_memory_bytes;
  T.t0 = a->t0;
  T.peak0 = a->peak0;
  for (int S = 0; S < 16; ++S) {
    uint64_t d = 1;
    for (int A = 0; A < n_axes; ++A) if (S >> A & 1) d *= (uint64_t)g->axis_size[A];
    uint32_t sh = 0;
    while (!(d & 1)) { d >>= 1; ++sh; }
    uint64_t inv = d;                 // Newton iteration for the inverse of an odd d mod 2^64
    for (int it = 0; it < 6; ++it) inv *= 2 - d * inv;
    T.shift[S] = sh;
    T.inv[S] = inv;
    unsigned __int128 d128 = d, inv128 = d;   // Newton for the inverse mod 2^128
    for (int it = 0; it < 7; ++it) inv128 *= (unsigned __int128)2 - d128 * inv128;
    T.inv128_lo[S] = (uint64_t)inv128;
    T.inv128_hi[S] = (uint64_t)(inv128 >> 64);
  }
  T.shift_pack = 0;
  for (int S = 0; S < 16; ++S) {
    if (T.shift[S] > 15) T.pow2 = 0;   // the shift path packs 4-bit codes; larger meshes take the general path
    T.shift_pack |= (uint64_t)(T.shift[S] & 15) << (4 * S);
  }
  return TOAST_OK;
}

// ---------------------------------------------------------------- host materialisation (debug)
// The decode checks of C9 (the kernels' H1) on the host: 0, or the TOAST_ST_*
// bits of an invalid sequence (which toast_lower / toast_materialize refuse).
uint32_t host_validate(const toast_analysis* a, const uint16_t* seq) {
  const DeviceTables& T = a->dt;
  uint32_t status = 0;
  bool stopped = false;
  uint64_t fixed = 0, ones = 0;
  std::vector<uint32_t> axes_of(T.n_acolors, 0);   // per action color: the axes its actions used
  for (int j = 0; j < 32; ++j) {
    const uint32_t id = seq[j];
    if (stopped) { if (id) status |= TOAST_ST_NONZERO_AFTER_STOP; continue; }
    if (id == 0) { stopped = true; continue; }
    if (id >= a->h_actions.size()) { status |= TOAST_ST_BAD_ACTION_ID; continue; }
    const uint32_t w = a->h_actions[id];
    const uint32_t ac = w & 0x3FF, r = (w >> 10) & 0xFF, ax = (w >> 18) & 3;
    if ((axes_of[ac] >> ax) & 1) status |= TOAST_ST_DUP_COLOR_AXIS;
    axes_of[ac] |= 1u << ax;
    const uint64_t gw = a->h_acol_groups[ac];
    for (int t = 0; t < 8; ++t) {
      const uint32_t gid = (gw >> (8 * t)) & 0xFF;
      if (gid == 0xFF) continue;
      const uint64_t g = 1ULL << gid, bit = (r >> t) & 1;
      if ((fixed & g) && (((ones >> gid) & 1) != bit)) status |= TOAST_ST_RES_MISMATCH;
      if (!(fixed & g)) { fixed |= g; if (bit) ones |= g; }
    }
  }
  return status;
}

// masks of a VALID sequence (host_validate == 0): an action color holds at
// most one action per mesh axis, so at most 4 events fit its 4 slots
void host_materialize(const toast_analysis* a, const uint16_t* seq, uint8_t* masks) {
  const DeviceTables& T = a->dt;
  std::vector<uint32_t> lists(T.n_acolors, 0);
  uint64_t fixed = 0, ones = 0;
  int n = 0;
  while (n < 32 && seq[n]) ++n;
  for (int j = 0; j < n; ++j) {
    uint32_t w = a->h_actions[seq[j]];
    uint32_t ac = w & 0x3FF, r = (w >> 10) & 0xFF, ax = (w >> 18) & 3;
    int rank = 0;
    while (rank < 4 && ((lists[ac] >> (8 * rank)) & 0x80)) ++rank;
    if (rank == 4) continue;   // unreachable for a valid sequence (see host_validate)
    lists[ac] |= (0x80u | (ax << 5) | (uint32_t)j) << (8 * rank);
    uint64_t gw = a->h_acol_groups[ac];
    for (int t = 0; t < 8; ++t) {
      uint32_t gid = (gw >> (8 * t)) & 0xFF;
      if (gid == 0xFF) break;
      fixed |= 1ULL << gid;
      if ((r >> t) & 1) ones |= 1ULL << gid;
    }
  }
  memset(masks, 0, (size_t)T.n_loops);
  for (int32_t t = 0; t < T.n_ops; ++t) {
    const DOp& op = a->h_ops[t];
    uint32_t l8[8] = {0};
    uint32_t div[8] = {0};
    for (int r = 0; r < op.n_loops; ++r) {
      uint64_t L = a->h_loops[op.loop_begin + r];
      uint32_t ac = L & 0x3FF;
      div[r] = (L >> 12) & 0xFFFF;
      if (ac == NO_ACOLOR) continue;
      uint32_t did = (L >> 28) & 0xFFFF;
      if (did && ((((fixed & ~ones) & a->h_desel[2 * did]) | (ones & a->h_desel[2 * did + 1])) != 0)) continue;
      l8[r] = lists[ac];
    }
    uint32_t opmask = 0, mk[8] = {0};
    while (true) {
      int best = -1;
      uint32_t bj = 99;
      for (int r = 0; r < op.n_loops; ++r)
        if ((l8[r] & 0x80) && (l8[r] & 31) < bj) { bj = l8[r] & 31; best = r; }
      if (best < 0) break;
      uint32_t A = (l8[best] >> 5) & 3;
      if (!(opmask >> A & 1) && ((div[best] >> (mk[best] | (1u << A))) & 1)) { mk[best] |= 1u << A; opmask |= 1u << A; }
      l8[best] >>= 8;
    }
    for (int r = 0; r < op.n_loops; ++r) masks[op.loop_begin + r] = (uint8_t)mk[r];
  }
}

// ---------------------------------------------------------------- JSON dump (same schema as the oracle's)
std::string dump_json(const toast_analysis* a) {
  std::string s;
  s.reserve(64 * (size_t)a->n_loops + 4096);
  auto I = [](int64_t x) { return std::to_string(x); };
  s += "{\"n_ops\":" + I(a->n_ops) + ",\"n_loops\":" + I(a->n_loops) + ",\"n_edges\":" + I(a->n_edges) + ",\"loops\":[";
  for (int64_t l = 0; l < a->n_loops; ++l) {
    if (l) s += ',';
    s += '[' + I(a->loop_op[l]) + ',' + I(a->loop_role[l]) + ',' + I(a->loop_ext[l]) + ',' + I(a->loop_type[l]) + ',' +
         I(a->loop_comp[l]) + ',' + I(a->loop_scolor[l]) + ']';
  }
  s += "],\"conflicts\":[";
  for (size_t i = 0; i < a->conflicts.size(); ++i) {
    const auto& c = a->conflicts[i];
    if (i) s += ',';
    s += '[' + I(c.op) + ',' + I(c.u) + ',' + I(c.v) + ',' + I(c.set) + ',' + I(c.side0) + ']';
  }
  {   // the per-candidate tables the kernels read (signatures, templates, peak-memory frontier)
    int64_t roles = 0, cols = 0;
    for (const auto& k : a->h_sigs) { roles += k.nr; cols += k.m; }
    s += "],\"kernel_tables\":{\"n_sigs\":" + I((int64_t)a->h_sig_mr.size()) + ",\"n_mc\":" +
         I((int64_t)a->h_sigs.size()) + ",\"sig_roles\":" + I(roles) +
         ",\"sig_colors\":" + I(cols) + ",\"n_tmpl\":" + I((int64_t)a->h_tmpl.size()) + ",\"n_points\":" +
         I((int64_t)a->h_points.size()) + ",\"n_terms\":" + I((int64_t)a->h_terms.size()) + ",\"n_spec\":" +
         I((int64_t)a->h_spec.size()) + ",\"n_slots\":" + I((int64_t)a->dt.n_slots) + ",\"cp_walked_ops\":" +
         I((int64_t)a->cp_walked_ops) + ",\"cp_walked_edges\":" + I((int64_t)a->cp_walked_edges) + ",\"cp_bundles\":" + I((int64_t)a->h_cp_bsize.size()) + ",\"n_acolors\":" + I((int64_t)a->dt.n_acolors) +
         ",\"n_words\":" + I((int64_t)a->dt.n_words) + ",\"n_fsig\":" + I((int64_t)a->dt.n_fsig) + ",\"n_ftmpl\":" +
         I((int64_t)a->dt.n_ftmpl) + ",\"warps_per_batch\":" +
         I((int64_t)a->k_throughput) + ",\"kernel_variant\":[" + I((int64_t)a->dt.n_axes) + "," +
         I((int64_t)a->dt.pow2) + "," + I((int64_t)a->dt.cost_model) + "],\"blocks_per_sm\":" +
         I((int64_t)a->occ_roll[a->k_throughput >= 8 ? 3 : a->k_throughput >= 4 ? 2 : a->k_throughput >= 2 ? 1 : 0]) + ",\"work\":{\"sig_roles\":" + I(a->work_sig_roles) + ",\"n_tmpl\":" +
         I(a->work_tmpl) + ",\"n_terms\":" + I(a->work_terms) + "},\"frontier_ops\":[";
    for (size_t q = 0; q < a->point_op.size(); ++q) { if (q) s += ','; s += I(a->point_op[q]); }
    s += "]}";
  }
  s += ",\"n_boxes\":" + I(a->n_boxes) + ",\"dropped_boxes\":" + I(a->dropped_boxes);
  s += ",\"contracted\":" + I(a->contracted) + ",\"contract_rejected\":" + I(a->contract_rejected);
  if (a->grouping == TOAST_GROUP_CONTRACTION) {
    s += ",\"cnode\":[";
    for (size_t l = 0; l < a->cnode.size(); ++l) { if (l) s += ','; s += I(a->cnode[l]); }
    s += "]";
  }
  s += ",\"set_group\":[";
  for (size_t i = 0; i < a->set_group.size(); ++i) { if (i) s += ','; s += I(a->set_group[i]); }
  s += "],\"set_sig\":[";
  for (size_t i = 0; i < a->set_sig.size(); ++i) {
    if (i) s += ',';
    char b[32];
    snprintf(b, sizeof b, "\"%016llx\"", (unsigned long long)a->set_sig[i]);
    s += b;
  }
  s += "],\"n_groups\":" + I(a->n_groups) + ",\"scolors\":[";
  for (size_t c = 0; c < a->sc_min_loop.size(); ++c) {
    if (c) s += ',';
    s += '[' + I(a->sc_min_loop[c]) + ',' + I(a->sc_value_dims[c]) + ",[";
    for (size_t j = 0; j < a->sc_groups[c].size(); ++j) { if (j) s += ','; s += I(a->sc_groups[c][j]); }
    s += "]]";
  }
  s += "],\"actions\":[";
  for (size_t i = 1; i < a->actions.size(); ++i) {
    if (i > 1) s += ',';
    s += '[' + I(a->actions[i].super_color) + ',' + I(a->actions[i].resolution) + ',' + I(a->actions[i].axis) + ']';
  }
  char b[160];
  snprintf(b, sizeof b, "],\"baseline\":{\"runtime\":%.17g,\"peak\":%llu,\"flops\":%llu}}", a->t0,
           (unsigned long long)a->peak0, (unsigned long long)a->baseline.flops);
  s += b;
  return s;
}

}  // namespace toast
