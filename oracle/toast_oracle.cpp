// =============================================================================
// TOAST oracle — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, deliberately literal CPU implementation of what the hot path
// computes (SURVEY.md §8(c), C0–C17), written from the paper:
//   arXiv 2508.15010, /root/reference/PAPER.md ("P:n" = line n).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this library.  The product path
// (paper_2508_15010_b200/) shares NO code with it: no headers, no helpers, no
// generated tables.  Every function cites the passage it follows.
//
// Parity status per part (see DESIGN.md §"Oracle pins"):
//   C1–C5, C9–C14 pinned by paper worked examples / closed forms / invariants /
//   brute force; the C1 rules of the extension ops (dot_general, conv2d and its
//   adjoints, resample, concat / slice / pad, gather, segment_sum) pinned by
//   what the lowered programs compute on every device of 2- and 3-axis meshes
//   (tests/test_lowering.py, the sharded interpreter); C15 pinned by Philox KAT vectors; C6 (WL signatures) pinned by
//   brute-force isomorphism of the sets' labelled graphs; C7 (argument keys) and
//   C8 (action table order) are "parity unpinned" beyond the structural
//   invariants in tests/test_oracle_pins.py.  The contraction
//   heuristic (reading R23, NEXT-4) is pinned by the paper's box / incompatible
//   listings, by "all conflicts of the attention layer
//   compatible" and by brute-force path checks on random programs.
//
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fPIC -shared -pthread
// =============================================================================
#include <algorithm>
#include <chrono>
#include <functional>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

namespace orc {

using u64 = uint64_t;
using u32 = uint32_t;
using u16 = uint16_t;
using i64 = int64_t;
typedef unsigned __int128 u128;

struct OracleError : std::runtime_error {
  std::string code;
  OracleError(const std::string& c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// ---------------------------------------------------------------------------
// Text IR (SPEC grammar S:92–104, extended per SURVEY §8(c) C0/C1)
// ---------------------------------------------------------------------------
struct Tok {
  int kind;  // 0 ident, 1 number, 2 punct, 3 eof
  std::string s;
  int line, col;
};

static std::vector<Tok> tokenize(const std::string& src) {
  std::vector<Tok> out;
  int line = 1, col = 1;
  size_t i = 0;
  while (i < src.size()) {
    char c = src[i];
    if (c == '\n') { line++; col = 1; i++; continue; }
    if (c == ' ' || c == '\t' || c == '\r') { i++; col++; continue; }
    if (c == '#') { while (i < src.size() && src[i] != '\n') i++; continue; }
    Tok t; t.line = line; t.col = col;
    if (isalpha((unsigned char)c) || c == '_') {
      size_t j = i;
      while (j < src.size() && (isalnum((unsigned char)src[j]) || src[j] == '_' || src[j] == '.')) j++;
      t.kind = 0; t.s = src.substr(i, j - i);
      col += (int)(j - i); i = j; out.push_back(t); continue;
    }
    if (isdigit((unsigned char)c) || (c == '-' && i + 1 < src.size() && (isdigit((unsigned char)src[i + 1]) || src[i+1]=='.')) || c == '.') {
      size_t j = i + 1;
      while (j < src.size()) {
        char d = src[j];
        if (isdigit((unsigned char)d) || d == '.' ) { j++; continue; }
        if ((d == 'e' || d == 'E') && j + 1 < src.size()) {
          j++; if (src[j] == '-' || src[j] == '+') j++; continue;
        }
        break;
      }
      t.kind = 1; t.s = src.substr(i, j - i);
      col += (int)(j - i); i = j; out.push_back(t); continue;
    }
    if (strchr("()[]{},;:=", c)) {
      t.kind = 2; t.s = std::string(1, c); i++; col++; out.push_back(t); continue;
    }
    throw OracleError("E_PARSE", std::to_string(line) + ":" + std::to_string(col) + ": unexpected character '" + std::string(1, c) + "'");
  }
  Tok e; e.kind = 3; e.line = line; e.col = col; out.push_back(e);
  return out;
}

struct Value {
  std::string name;
  std::string dtype;
  std::vector<i64> shape;
  int def_op;
};

struct Op {
  std::string kind;                              // IR op name, "param" or "ret"
  std::vector<std::vector<std::string>> attrs;   // groups split by ';', items by ','
  std::vector<int> operands;                     // value ids
  int result = -1;                               // value id; -1 for ret
  std::string binding;
};

static int dtype_bytes(const std::string& dt) {
  if (dt == "f32" || dt == "i32") return 4;
  if (dt == "bf16" || dt == "f16") return 2;
  if (dt == "f64" || dt == "i64") return 8;
  return -1;
}

static const std::set<std::string>& unary_ops() {
  static const std::set<std::string> s = {
      "relu", "neg", "exp", "log", "recip", "rsqrt", "sqrt", "tanh", "gelu", "silu", "sigmoid",
      "square", "abs", "sign", "ones_like", "scale", "add_s", "pow_s", "convert", "d_relu",
      "d_gelu", "d_silu", "d_tanh", "d_sigmoid", "stop_gradient", "cos", "sin"};
  return s;
}
// any "d_<name>" (a derivative of an elementwise function) follows the (function) rule too
static bool is_unary(const std::string& k) { return unary_ops().count(k) || (k.size() > 2 && k[0] == 'd' && k[1] == '_'); }
static const std::set<std::string>& binary_ops() {
  static const std::set<std::string> s = {"add", "sub", "mul", "div", "max", "min", "pow"};
  return s;
}

struct Module {
  std::string name;
  std::vector<Value> values;
  std::vector<Op> ops;       // params, body, rets (in this order)
  int n_params = 0, n_body = 0, n_rets = 0;
};

static i64 to_int(const std::string& s, const std::string& ctx) {
  char* end = nullptr;
  long long v = strtoll(s.c_str(), &end, 10);
  if (!end || *end) throw OracleError("E_SHAPE", ctx + ": expected integer attribute, got '" + s + "'");
  return v;
}

static std::vector<i64> infer_shape(Module& M, Op& op, std::string& dtype) {
  const std::string ctx = "binding '" + op.binding + "'";
  auto sh = [&](int k) -> const std::vector<i64>& { return M.values[op.operands[k]].shape; };
  auto dt = [&](int k) -> const std::string& { return M.values[op.operands[k]].dtype; };
  auto need = [&](size_t n) {
    if (op.operands.size() != n) throw OracleError("E_SHAPE", ctx + ": expected " + std::to_string(n) + " operands");
  };
  auto attr_ints = [&](size_t g) {
    std::vector<i64> v;
    if (g < op.attrs.size()) for (auto& s : op.attrs[g]) v.push_back(to_int(s, ctx));
    return v;
  };
  const std::string& k = op.kind;
  if (is_unary(k)) {
    need(1);
    dtype = dt(0);
    if (k == "convert") {
      if (op.attrs.empty() || op.attrs[0].empty() || dtype_bytes(op.attrs[0][0]) < 0)
        throw OracleError("E_SHAPE", ctx + ": convert needs a dtype");
      dtype = op.attrs[0][0];
    }
    return sh(0);
  }
  if (binary_ops().count(k)) {
    need(2);
    if (sh(0) != sh(1)) throw OracleError("E_SHAPE", ctx + ": elementwise operands differ in shape");
    dtype = dt(0);
    return sh(0);
  }
  if (k == "transpose") {
    need(1);
    auto p = attr_ints(0);
    const auto& s = sh(0);
    if (p.size() != s.size()) throw OracleError("E_SHAPE", ctx + ": bad permutation");
    std::vector<int> seen(s.size(), 0);
    std::vector<i64> r;
    for (auto x : p) {
      if (x < 0 || x >= (i64)s.size() || seen[x]) throw OracleError("E_SHAPE", ctx + ": bad permutation");
      seen[x] = 1; r.push_back(s[x]);
    }
    dtype = dt(0);
    return r;
  }
  if (k == "reduce") {
    need(1);
    if (op.attrs.size() != 1 || op.attrs[0].size() < 2) throw OracleError("E_SHAPE", ctx + ": reduce[dims..., comb]");
    std::string comb = op.attrs[0].back();
    if (comb != "add" && comb != "mul" && comb != "max" && comb != "min") throw OracleError("E_SHAPE", ctx + ": bad combiner");
    const auto& s = sh(0);
    std::vector<int> red(s.size(), 0);
    for (size_t i = 0; i + 1 < op.attrs[0].size(); i++) {
      i64 d = to_int(op.attrs[0][i], ctx);
      if (d < 0 || d >= (i64)s.size() || red[d]) throw OracleError("E_SHAPE", ctx + ": bad reduce dim");
      red[d] = 1;
    }
    std::vector<i64> r;
    for (size_t i = 0; i < s.size(); i++) if (!red[i]) r.push_back(s[i]);
    dtype = dt(0);
    return r;
  }
  if (k == "broadcast") {
    need(1);
    auto a = attr_ints(0);
    const auto& s = sh(0);
    if (a.size() != 2 || a[0] < 0 || a[0] > (i64)s.size() || a[1] < 1) throw OracleError("E_SHAPE", ctx + ": broadcast[l, e]");
    std::vector<i64> r = s;
    r.insert(r.begin() + a[0], a[1]);
    dtype = dt(0);
    return r;
  }
  if (k == "matmul") {
    need(2);
    if (sh(0).size() != 2 || sh(1).size() != 2 || sh(0)[1] != sh(1)[0])
      throw OracleError("E_SHAPE", ctx + ": matmul contraction extents differ");
    dtype = dt(0);
    return {sh(0)[0], sh(1)[1]};
  }
  if (k == "dot_general") {
    need(2);
    if (op.attrs.size() != 4) throw OracleError("E_SHAPE", ctx + ": dot_general[lb;rb;lc;rc]");
    auto lb = attr_ints(0), rb = attr_ints(1), lc = attr_ints(2), rc = attr_ints(3);
    const auto& L = sh(0); const auto& R = sh(1);
    if (lb.size() != rb.size() || lc.size() != rc.size()) throw OracleError("E_SHAPE", ctx + ": dot_general dims");
    std::vector<int> ul(L.size(), 0), ur(R.size(), 0);
    for (size_t t = 0; t < lb.size(); t++) {
      if (lb[t] < 0 || lb[t] >= (i64)L.size() || rb[t] < 0 || rb[t] >= (i64)R.size() || ul[lb[t]] || ur[rb[t]] || L[lb[t]] != R[rb[t]])
        throw OracleError("E_SHAPE", ctx + ": dot_general batch dims");
      ul[lb[t]] = ur[rb[t]] = 1;
    }
    for (size_t t = 0; t < lc.size(); t++) {
      if (lc[t] < 0 || lc[t] >= (i64)L.size() || rc[t] < 0 || rc[t] >= (i64)R.size() || ul[lc[t]] || ur[rc[t]] || L[lc[t]] != R[rc[t]])
        throw OracleError("E_SHAPE", ctx + ": dot_general contracting dims");
      ul[lc[t]] = ur[rc[t]] = 1;
    }
    std::vector<i64> r;
    for (auto x : lb) r.push_back(L[x]);
    for (size_t i = 0; i < L.size(); i++) if (!ul[i]) r.push_back(L[i]);
    for (size_t i = 0; i < R.size(); i++) if (!ur[i]) r.push_back(R[i]);
    dtype = dt(0);
    return r;
  }
  if (k == "conv2d") {
    need(2);
    const auto& x = sh(0); const auto& w = sh(1);
    if (x.size() != 4 || w.size() != 4 || x[3] != w[2]) throw OracleError("E_SHAPE", ctx + ": conv2d shapes");
    dtype = dt(0);
    return {x[0], x[1], x[2], w[3]};
  }
  if (k == "conv2d_bwd_input") {
    need(2);
    const auto& dy = sh(0); const auto& w = sh(1);
    if (dy.size() != 4 || w.size() != 4 || dy[3] != w[3]) throw OracleError("E_SHAPE", ctx + ": conv2d_bwd_input shapes");
    dtype = dt(0);
    return {dy[0], dy[1], dy[2], w[2]};
  }
  if (k == "conv2d_bwd_filter") {
    need(2);
    auto a = attr_ints(0);
    const auto& x = sh(0); const auto& dy = sh(1);
    if (a.size() != 2 || x.size() != 4 || dy.size() != 4 || x[0] != dy[0] || x[1] != dy[1] || x[2] != dy[2] || a[0] < 1 || a[1] < 1)
      throw OracleError("E_SHAPE", ctx + ": conv2d_bwd_filter shapes");
    dtype = dt(0);
    return {a[0], a[1], x[3], dy[3]};
  }
  if (k == "resample") {
    need(1);
    const auto& x = sh(0);
    if (op.attrs.size() != 1 || op.attrs[0].size() != 2 || x.size() != 4) throw OracleError("E_SHAPE", ctx + ": resample[up|down,f]");
    i64 f = to_int(op.attrs[0][1], ctx);
    std::vector<i64> r = x;
    if (f < 1) throw OracleError("E_SHAPE", ctx + ": resample factor");
    if (op.attrs[0][0] == "up") { r[1] *= f; r[2] *= f; }
    else if (op.attrs[0][0] == "down") {
      if (x[1] % f || x[2] % f) throw OracleError("E_SHAPE", ctx + ": resample factor does not divide");
      r[1] /= f; r[2] /= f;
    } else throw OracleError("E_SHAPE", ctx + ": resample mode");
    dtype = dt(0);
    return r;
  }
  if (k == "concat") {
    if (op.operands.empty()) throw OracleError("E_SHAPE", ctx + ": concat needs operands");
    auto a = attr_ints(0);
    const auto& s0 = sh(0);
    if (a.size() != 1 || a[0] < 0 || a[0] >= (i64)s0.size()) throw OracleError("E_SHAPE", ctx + ": concat[d]");
    std::vector<i64> r = s0;
    r[a[0]] = 0;
    for (size_t j = 0; j < op.operands.size(); j++) {
      const auto& s = sh(j);
      if (s.size() != s0.size()) throw OracleError("E_SHAPE", ctx + ": concat rank");
      for (size_t i = 0; i < s.size(); i++)
        if ((i64)i != a[0] && s[i] != s0[i]) throw OracleError("E_SHAPE", ctx + ": concat extents");
      r[a[0]] += s[a[0]];
    }
    dtype = dt(0);
    return r;
  }
  if (k == "slice") {
    need(1);
    auto a = attr_ints(0);
    const auto& s = sh(0);
    if (a.size() != 3 || a[0] < 0 || a[0] >= (i64)s.size() || a[1] < 0 || a[2] < 1 || a[1] + a[2] > s[a[0]])
      throw OracleError("E_SHAPE", ctx + ": slice[d,start,len]");
    std::vector<i64> r = s; r[a[0]] = a[2];
    dtype = dt(0);
    return r;
  }
  if (k == "pad") {
    need(1);
    auto a = attr_ints(0);
    const auto& s = sh(0);
    if (a.size() != 3 || a[0] < 0 || a[0] >= (i64)s.size() || a[1] < 0 || a[2] < 0)
      throw OracleError("E_SHAPE", ctx + ": pad[d,lo,hi]");
    std::vector<i64> r = s; r[a[0]] += a[1] + a[2];
    dtype = dt(0);
    return r;
  }
  if (k == "gather") {
    need(2);
    const auto& t = sh(0); const auto& ix = sh(1);
    if (t.size() != 2 || ix.empty()) throw OracleError("E_SHAPE", ctx + ": gather(tbl[n,f], idx[e...])");
    std::vector<i64> r = ix; r.push_back(t[1]);
    dtype = dt(0);
    return r;
  }
  if (k == "segment_sum") {
    need(2);
    auto a = attr_ints(0);
    const auto& d = sh(0); const auto& ix = sh(1);
    if (a.size() != 1 || a[0] < 1 || ix.empty() || d.size() != ix.size() + 1) throw OracleError("E_SHAPE", ctx + ": segment_sum[n](dat, idx)");
    for (size_t i = 0; i < ix.size(); i++) if (d[i] != ix[i]) throw OracleError("E_SHAPE", ctx + ": segment_sum extents");
    dtype = dt(0);
    return {a[0], d.back()};
  }
  throw OracleError("E_PARSE", ctx + ": unknown op '" + k + "'");
}

static Module parse_module(const std::string& src) {
  auto toks = tokenize(src);
  size_t p = 0;
  auto where = [&](const Tok& t) { return std::to_string(t.line) + ":" + std::to_string(t.col) + ": "; };
  auto expect = [&](const std::string& s) {
    if (toks[p].s != s || toks[p].kind == 3) throw OracleError("E_PARSE", where(toks[p]) + "expected '" + s + "'");
    p++;
  };
  auto ident = [&]() {
    if (toks[p].kind != 0) throw OracleError("E_PARSE", where(toks[p]) + "expected identifier");
    return toks[p++].s;
  };
  Module M;
  std::map<std::string, int> env;
  if (toks[p].s != "def") throw OracleError("E_PARSE", where(toks[p]) + "expected 'def'");
  p++;
  M.name = ident();
  expect("(");
  std::vector<Op> params;
  while (toks[p].s != ")") {
    Tok nt = toks[p];
    std::string nm = ident();
    expect(":");
    std::string dt = ident();
    if (dtype_bytes(dt) < 0) throw OracleError("E_PARSE", where(toks[p - 1]) + "unknown dtype '" + dt + "'");
    expect("[");
    std::vector<i64> shape;
    while (toks[p].s != "]") {
      if (toks[p].kind != 1) throw OracleError("E_PARSE", where(toks[p]) + "expected extent");
      i64 e = strtoll(toks[p].s.c_str(), nullptr, 10);
      if (e < 1) throw OracleError("E_SHAPE", "parameter '" + nm + "': extent must be >= 1");
      shape.push_back(e); p++;
      if (toks[p].s == ",") p++;
    }
    expect("]");
    if (env.count(nm)) throw OracleError("E_DUPLICATE", where(nt) + "duplicate binding '" + nm + "'");
    Value v; v.name = nm; v.dtype = dt; v.shape = shape; v.def_op = (int)M.ops.size();
    env[nm] = (int)M.values.size();
    Op op; op.kind = "param"; op.result = (int)M.values.size(); op.binding = nm;
    M.values.push_back(v);
    M.ops.push_back(op);
    M.n_params++;
    if (toks[p].s == ",") p++;
    else if (toks[p].s != ")") throw OracleError("E_PARSE", where(toks[p]) + "expected ',' or ')'");
  }
  expect(")");
  expect("{");
  std::vector<int> rets;
  bool have_return = false;
  while (toks[p].s != "}") {
    if (toks[p].kind == 3) throw OracleError("E_PARSE", where(toks[p]) + "unexpected end of input");
    if (toks[p].kind == 0 && toks[p].s == "return") {
      p++;
      while (true) {
        Tok nt = toks[p];
        std::string nm = ident();
        if (!env.count(nm)) throw OracleError("E_UNDEFINED", where(nt) + "use of undefined '" + nm + "'");
        rets.push_back(env[nm]);
        if (toks[p].s == ",") { p++; continue; }
        break;
      }
      have_return = true;
      if (toks[p].s != "}") throw OracleError("E_PARSE", where(toks[p]) + "expected '}' after return");
      break;
    }
    Tok bt = toks[p];
    std::string nm = ident();
    expect("=");
    Op op;
    op.kind = ident();
    op.binding = nm;
    if (toks[p].s == "[") {
      p++;
      op.attrs.push_back({});
      while (toks[p].s != "]") {
        if (toks[p].kind == 3) throw OracleError("E_PARSE", where(toks[p]) + "unterminated attributes");
        if (toks[p].s == ";") { op.attrs.push_back({}); p++; continue; }
        if (toks[p].s == ",") { p++; continue; }
        if (toks[p].kind != 0 && toks[p].kind != 1) throw OracleError("E_PARSE", where(toks[p]) + "bad attribute");
        op.attrs.back().push_back(toks[p].s); p++;
      }
      p++;
    }
    expect("(");
    while (toks[p].s != ")") {
      Tok at = toks[p];
      std::string a = ident();
      if (!env.count(a)) throw OracleError("E_UNDEFINED", where(at) + "use of undefined '" + a + "'");
      op.operands.push_back(env[a]);
      if (toks[p].s == ",") p++;
      else if (toks[p].s != ")") throw OracleError("E_PARSE", where(toks[p]) + "expected ',' or ')'");
    }
    expect(")");
    if (env.count(nm)) throw OracleError("E_DUPLICATE", where(bt) + "duplicate binding '" + nm + "'");
    std::string dtype;
    std::vector<i64> shape = infer_shape(M, op, dtype);
    Value v; v.name = nm; v.dtype = dtype; v.shape = shape; v.def_op = (int)M.ops.size();
    op.result = (int)M.values.size();
    env[nm] = op.result;
    M.values.push_back(v);
    M.ops.push_back(op);
    M.n_body++;
  }
  if (!have_return) throw OracleError("E_PARSE", where(toks[p]) + "missing return");
  expect("}");
  if (toks[p].kind != 3) throw OracleError("E_PARSE", where(toks[p]) + "trailing input");
  for (int v : rets) {
    Op op; op.kind = "ret"; op.operands = {v}; op.binding = "return " + M.values[v].name;
    M.ops.push_back(op);
    M.n_rets++;
  }
  return M;
}

// ---------------------------------------------------------------------------
// C1: the Named Dimension Analysis, literally (Fig. 3; §3.1)
//   Every definition site and every use site gets fresh dimension names.
//   (variable use) adds M edges def-name_i -> use-name_i,
//   including the returned variable.  Each op rule adds identities I.
//   Quotienting by I alone gives one class per "way of partitioning one op"
//   (P:877–878): these classes are the loops.
// ---------------------------------------------------------------------------
enum LoopType { LP = 0, LR = 1, LX = 2 };

struct Loop {
  int op;
  int role;
  i64 ext;
  int type;
};

struct NDA {
  int n_names = 0;
  std::vector<std::vector<int>> def_names;               // per value
  std::vector<std::vector<std::vector<int>>> use_names;  // per op, per operand
  std::vector<std::pair<int, int>> M;                    // name -> name
  std::vector<std::pair<int, int>> I;                    // name ≗ name
  std::vector<std::vector<int>> role_rep;                // per op: representative name per role
  std::vector<std::vector<int>> role_type;               // per op: loop type per role
  std::vector<std::vector<i64>> role_ext;                // per op: extent per role
};

static NDA run_nda(const Module& M) {
  NDA N;
  N.def_names.resize(M.values.size());
  N.use_names.resize(M.ops.size());
  N.role_rep.resize(M.ops.size());
  N.role_type.resize(M.ops.size());
  N.role_ext.resize(M.ops.size());
  auto fresh = [&]() { return N.n_names++; };
  auto fresh_vec = [&](size_t n) { std::vector<int> v; for (size_t i = 0; i < n; i++) v.push_back(fresh()); return v; };
  auto ident = [&](int a, int b) { N.I.push_back({a, b}); };
  for (size_t t = 0; t < M.ops.size(); t++) {
    const Op& op = M.ops[t];
    // (variable use): fresh names per use site + M edges from the definition's names
    for (int v : op.operands) {
      std::vector<int> u = fresh_vec(M.values[v].shape.size());
      for (size_t i = 0; i < u.size(); i++) N.M.push_back({N.def_names[v][i], u[i]});
      N.use_names[t].push_back(u);
    }
    const auto& U = N.use_names[t];
    std::vector<int> A;
    if (op.result >= 0) { A = fresh_vec(M.values[op.result].shape.size()); N.def_names[op.result] = A; }
    auto ushape = [&](int k) -> const std::vector<i64>& { return M.values[op.operands[k]].shape; };
    const std::vector<i64> rshape = op.result >= 0 ? M.values[op.result].shape : std::vector<i64>{};
    auto& rep = N.role_rep[t];
    auto& typ = N.role_type[t];
    auto& ext = N.role_ext[t];
    auto role = [&](int name, int ty, i64 e) { rep.push_back(name); typ.push_back(ty); ext.push_back(e); };
    const std::string& k = op.kind;
    auto attr_ints = [&](size_t g) {
      std::vector<i64> v;
      if (g < op.attrs.size()) for (auto& s : op.attrs[g]) v.push_back(strtoll(s.c_str(), nullptr, 10));
      return v;
    };
    if (k == "param") {
      // linear context: definition names, one loop each
      for (size_t i = 0; i < A.size(); i++) role(A[i], LP, rshape[i]);
    } else if (k == "ret") {
      // the returned variable is a use site
      for (size_t i = 0; i < U[0].size(); i++) role(U[0][i], LP, ushape(0)[i]);
    } else if (is_unary(k)) {
      // (function) P:519–523: {a_i ≗ d_i}
      for (size_t i = 0; i < A.size(); i++) { ident(A[i], U[0][i]); role(A[i], LP, rshape[i]); }
    } else if (binary_ops().count(k)) {
      // (op) P:525–531: {a_i ≗ d_i, a_i ≗ c_i}
      for (size_t i = 0; i < A.size(); i++) { ident(A[i], U[0][i]); ident(A[i], U[1][i]); role(A[i], LP, rshape[i]); }
    } else if (k == "transpose") {
      // (transpose) P:539–543: result position j carries operand dim perm[j]
      auto perm = attr_ints(0);
      for (size_t j = 0; j < A.size(); j++) ident(A[j], U[0][perm[j]]);
      for (size_t i = 0; i < U[0].size(); i++) role(U[0][i], LP, ushape(0)[i]);
    } else if (k == "reduce") {
      // (reduce) P:494–499: result drops the reduced dims; the rest identified
      std::vector<int> red(U[0].size(), 0);
      for (size_t i = 0; i + 1 < op.attrs[0].size(); i++) red[strtoll(op.attrs[0][i].c_str(), nullptr, 10)] = 1;
      size_t j = 0;
      for (size_t i = 0; i < U[0].size(); i++) if (!red[i]) ident(A[j++], U[0][i]);
      for (size_t i = 0; i < U[0].size(); i++) role(U[0][i], red[i] ? LR : LP, ushape(0)[i]);
    } else if (k == "broadcast") {
      // (broadcast) P:545–551 (reading G5): fresh unconstrained name at position l
      auto a = attr_ints(0);
      size_t l = (size_t)a[0];
      for (size_t j = 0; j < A.size(); j++) {
        if (j < l) ident(A[j], U[0][j]);
        else if (j > l) ident(A[j], U[0][j - 1]);
      }
      for (size_t j = 0; j < A.size(); j++) role(A[j], LP, rshape[j]);
    } else if (k == "matmul") {
      // (matmul) P:501–506: {a1 ≗ d1, a2 ≗ c2, d2 ≗ c1}
      ident(A[0], U[0][0]); ident(A[1], U[1][1]); ident(U[0][1], U[1][0]);
      role(A[0], LP, rshape[0]); role(A[1], LP, rshape[1]); role(U[0][1], LR, ushape(0)[1]);
    } else if (k == "dot_general") {
      // extension "analogously to PartIR/Shardy"
      auto lb = attr_ints(0), rb = attr_ints(1), lc = attr_ints(2), rc = attr_ints(3);
      std::vector<int> ul(U[0].size(), 0), ur(U[1].size(), 0);
      for (auto x : lb) ul[x] = 1;
      for (auto x : lc) ul[x] = 1;
      for (auto x : rb) ur[x] = 1;
      for (auto x : rc) ur[x] = 1;
      size_t j = 0;
      for (size_t t2 = 0; t2 < lb.size(); t2++) { ident(A[j], U[0][lb[t2]]); ident(U[0][lb[t2]], U[1][rb[t2]]); j++; }
      for (size_t i = 0; i < U[0].size(); i++) if (!ul[i]) ident(A[j++], U[0][i]);
      for (size_t i = 0; i < U[1].size(); i++) if (!ur[i]) ident(A[j++], U[1][i]);
      for (size_t t2 = 0; t2 < lc.size(); t2++) ident(U[0][lc[t2]], U[1][rc[t2]]);
      for (size_t jj = 0; jj < A.size(); jj++) role(A[jj], LP, rshape[jj]);
      for (size_t t2 = 0; t2 < lc.size(); t2++) role(U[0][lc[t2]], LR, ushape(0)[lc[t2]]);
    } else if (k == "conv2d") {
      // x[N,H,W,Ci] * w[KH,KW,Ci,Co] -> [N,Ho,Wo,Co]; spatial loops unshardable (G23)
      ident(A[0], U[0][0]); ident(A[1], U[0][1]); ident(A[2], U[0][2]); ident(A[3], U[1][3]); ident(U[0][3], U[1][2]);
      role(A[0], LP, rshape[0]); role(A[1], LX, rshape[1]); role(A[2], LX, rshape[2]); role(A[3], LP, rshape[3]);
      role(U[0][3], LR, ushape(0)[3]); role(U[1][0], LX, ushape(1)[0]); role(U[1][1], LX, ushape(1)[1]);
    } else if (k == "conv2d_bwd_input") {
      // dy[N,H,W,Co], w[KH,KW,Ci,Co] -> dx[N,H,W,Ci]
      ident(A[0], U[0][0]); ident(A[1], U[0][1]); ident(A[2], U[0][2]); ident(A[3], U[1][2]); ident(U[0][3], U[1][3]);
      role(A[0], LP, rshape[0]); role(A[1], LX, rshape[1]); role(A[2], LX, rshape[2]); role(A[3], LP, rshape[3]);
      role(U[0][3], LR, ushape(0)[3]); role(U[1][0], LX, ushape(1)[0]); role(U[1][1], LX, ushape(1)[1]);
    } else if (k == "conv2d_bwd_filter") {
      // x[N,H,W,Ci], dy[N,H,W,Co] -> dw[KH,KW,Ci,Co]
      ident(A[2], U[0][3]); ident(A[3], U[1][3]); ident(U[0][0], U[1][0]); ident(U[0][1], U[1][1]); ident(U[0][2], U[1][2]);
      role(A[0], LX, rshape[0]); role(A[1], LX, rshape[1]); role(A[2], LP, rshape[2]); role(A[3], LP, rshape[3]);
      role(U[0][0], LR, ushape(0)[0]); role(U[0][1], LX, ushape(0)[1]); role(U[0][2], LX, ushape(0)[2]);
    } else if (k == "resample") {
      for (size_t i = 0; i < A.size(); i++) ident(A[i], U[0][i]);
      role(A[0], LP, rshape[0]); role(A[1], LX, rshape[1]); role(A[2], LX, rshape[2]); role(A[3], LP, rshape[3]);
    } else if (k == "concat" || k == "slice" || k == "pad") {
      i64 d = attr_ints(0)[0];
      for (size_t q = 0; q < U.size(); q++)
        for (size_t i = 0; i < A.size(); i++) ident(A[i], U[q][i]);
      for (size_t i = 0; i < A.size(); i++) role(A[i], (i64)i == d ? LX : LP, rshape[i]);
    } else if (k == "gather") {
      // tbl[n,f], idx[e..] -> [e.., f]
      size_t ke = U[1].size();
      for (size_t t2 = 0; t2 < ke; t2++) ident(A[t2], U[1][t2]);
      ident(A[ke], U[0][1]);
      for (size_t t2 = 0; t2 <= ke; t2++) role(A[t2], LP, rshape[t2]);
      role(U[0][0], LX, ushape(0)[0]);
    } else if (k == "segment_sum") {
      // dat[e.., f], idx[e..] -> [n, f]
      size_t ke = U[1].size();
      for (size_t t2 = 0; t2 < ke; t2++) ident(U[0][t2], U[1][t2]);
      ident(A[1], U[0][ke]);
      for (size_t t2 = 0; t2 < ke; t2++) role(U[0][t2], LR, ushape(0)[t2]);
      role(A[1], LP, rshape[1]);
      role(A[0], LX, rshape[0]);
    } else {
      throw OracleError("E_PARSE", "unknown op kind " + k);
    }
  }
  return N;
}

// ---------------------------------------------------------------------------
// Plain union-find (used for the I-quotient, components, super-colors)
// ---------------------------------------------------------------------------
struct UF {
  std::vector<int> p;
  explicit UF(int n) : p(n) { for (int i = 0; i < n; i++) p[i] = i; }
  int find(int x) { while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; } return x; }
  void unite(int a, int b) { a = find(a); b = find(b); if (a != b) { if (a < b) p[b] = a; else p[a] = b; } }
};

// ---------------------------------------------------------------------------
// Hashes for C6/C14
// ---------------------------------------------------------------------------
static u64 mix64(u64 z) {
  z ^= z >> 30; z *= 0xbf58476d1ce4e5b9ULL;
  z ^= z >> 27; z *= 0x94d049bb133111ebULL;
  z ^= z >> 31;
  return z;
}
static u64 hcombine(u64 h, u64 x) { return mix64(h ^ (x + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2))); }
static u64 hseq(const std::vector<u64>& xs) { u64 h = 0; for (u64 x : xs) h = hcombine(h, x); return h; }
static u64 fnv1a(const std::string& s) {
  u64 h = 0xcbf29ce484222325ULL;
  for (unsigned char c : s) { h ^= c; h *= 0x100000001b3ULL; }
  return h;
}

// ---------------------------------------------------------------------------
// Philox4x32-10 (Random123), for C15
// ---------------------------------------------------------------------------
static void philox4x32_10(const u32 ctr_in[4], const u32 key_in[2], u32 out[4]) {
  u32 c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
  u32 k[2] = {key_in[0], key_in[1]};
  for (int r = 0; r < 10; r++) {
    if (r > 0) { k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u; }
    u64 p0 = (u64)0xD2511F53u * c[0];
    u64 p1 = (u64)0xCD9E8D57u * c[2];
    u32 hi0 = (u32)(p0 >> 32), lo0 = (u32)p0;
    u32 hi1 = (u32)(p1 >> 32), lo1 = (u32)p1;
    u32 n0 = hi1 ^ c[1] ^ k[0];
    u32 n1 = lo1;
    u32 n2 = hi0 ^ c[3] ^ k[1];
    u32 n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
  }
  for (int i = 0; i < 4; i++) out[i] = c[i];
}

// ---------------------------------------------------------------------------
// The whole analysis state
// ---------------------------------------------------------------------------
struct Axis { std::string name; i64 size; double bw; };

struct Conflict { int op; int u, v; };   // loop ids, u has the lower role
struct Box { int c1, c2; int N, O, L, R; int parity; };

struct Cost {
  double runtime_s, score;
  u64 peak_bytes, flops, state_key;
  u32 status, n_collectives;
  u64 payload[4][4];
  u16 count[4][4];
  u64 flops_hi;
  uint8_t pad[40];
};
static_assert(sizeof(Cost) == 256, "cost record is 256 B");

enum { ST_BAD_ACTION_ID = 1, ST_DUP_COLOR_AXIS = 2, ST_RES_MISMATCH = 4, ST_NONZERO_AFTER_STOP = 8 };
enum { K_AG = 0, K_RS = 1, K_AR = 2, K_A2A = 3 };

struct Action { int sc; int r; int axis; };

struct Oracle {
  Module M;
  NDA nda;
  std::vector<Axis> axes;
  double F = 1e12; u64 DM = 0; double C = 100.0;
  int min_dims = 10, max_depth = 30;
  int cost_model = 0;   // 0: straight-line sum (G14); 1: critical path (reading R22)
  int grouping = 0;     // 0: compatibility sets (C4/C5); 1: graph contraction heuristic (reading R23)

  std::vector<Loop> loops;
  std::vector<int> op_loop_begin;                       // loops of op t: [begin[t], begin[t+1])
  std::vector<int> name_loop;                           // name -> loop
  std::set<std::pair<int, int>> edges;                  // M over loops (deduplicated)
  std::vector<std::vector<int>> out_adj;
  std::vector<int> comp;                                // smallest member loop
  std::vector<Conflict> conflicts;
  std::map<std::pair<int, int>, int> conflict_of;       // (min loop, max loop) -> index
  std::vector<Box> boxes;                               // candidate boxes in canonical order
  std::vector<int> box_accepted;
  int dropped_boxes = 0;
  std::vector<int> cnode;                               // R23: contracted node of each loop (smallest member)
  int contracted = 0, contract_rejected = 0;            // R23: edges contracted / skipped
  std::vector<int> conf_set, conf_side0;
  std::vector<int> set_root;                            // smallest conflict per set
  std::vector<u64> set_sig;
  struct SetGraph { std::map<int, int> side; std::set<std::pair<int, int>> medges, cedges; };
  std::vector<SetGraph> set_graphs;                     // C6 input per set (dumped for the isomorphism pin)
  std::vector<int> set_group;
  int n_groups = 0;
  std::vector<int> scolor;                              // per loop
  std::vector<int> sc_min_loop;
  std::vector<i64> sc_value_dims;
  std::vector<std::vector<int>> sc_groups;              // SetGroups with a conflict in c, ascending
  std::vector<Action> actions;                          // index 0 = STOP (unused entry)
  double t0 = 0; u64 peak0 = 0; u64 flops0 = 0;
  std::vector<int> value_last_use;
  std::vector<std::vector<int>> dying;                  // per op: values whose last use is that op

  int loop_of(int op, int role) const { return op_loop_begin[op] + role; }
  int nloops(int op) const { return op_loop_begin[op + 1] - op_loop_begin[op]; }

  // loop of (op t, operand k, dim i) and of (value v's definition, dim i)
  int use_loop(int t, int k, int i) const { return name_loop[nda.use_names[t][k][i]]; }
  int def_loop(int v, int i) const { return name_loop[nda.def_names[v][i]]; }

  void build() {
    nda = run_nda(M);
    // I-quotient: union-find over names; each class must contain exactly one role rep
    UF uf(nda.n_names);
    for (auto& pr : nda.I) uf.unite(pr.first, pr.second);
    name_loop.assign(nda.n_names, -1);
    op_loop_begin.assign(M.ops.size() + 1, 0);
    std::map<int, int> root_loop;
    for (size_t t = 0; t < M.ops.size(); t++) {
      op_loop_begin[t] = (int)loops.size();
      for (size_t r = 0; r < nda.role_rep[t].size(); r++) {
        int root = uf.find(nda.role_rep[t][r]);
        if (root_loop.count(root)) throw OracleError("E_INTERNAL", "two roles identified in op " + M.ops[t].binding);
        root_loop[root] = (int)loops.size();
        loops.push_back(Loop{(int)t, (int)r, nda.role_ext[t][r], nda.role_type[t][r]});
      }
    }
    op_loop_begin[M.ops.size()] = (int)loops.size();
    for (int n = 0; n < nda.n_names; n++) {
      int root = uf.find(n);
      if (!root_loop.count(root)) throw OracleError("E_INTERNAL", "name without a loop");
      name_loop[n] = root_loop[root];
    }
    // sanity: each op's site names map to that op's loops
    for (size_t t = 0; t < M.ops.size(); t++) {
      for (auto& u : nda.use_names[t]) for (int n : u) if (loops[name_loop[n]].op != (int)t) throw OracleError("E_INTERNAL", "use name escapes op");
      if (M.ops[t].result >= 0) for (int n : nda.def_names[M.ops[t].result]) if (loops[name_loop[n]].op != (int)t) throw OracleError("E_INTERNAL", "def name escapes op");
    }
    // M over loops, deduplicated (C1)
    for (auto& e : nda.M) edges.insert({name_loop[e.first], name_loop[e.second]});
    out_adj.assign(loops.size(), {});
    for (auto& e : edges) out_adj[e.first].push_back(e.second);
    // C2: components = I∪M quotient (A11): weakly connected classes
    UF cu((int)loops.size());
    for (auto& e : edges) cu.unite(e.first, e.second);
    comp.resize(loops.size());
    for (size_t l = 0; l < loops.size(); l++) comp[l] = cu.find((int)l);   // smallest member (unite keeps min root)
    find_conflicts();
    if (grouping == 0) {
      find_boxes();
      build_sets();
    } else {
      build_sets_contraction();
    }
    build_groups();
    build_supercolors();
    build_actions();
    // last uses (C12)
    value_last_use.assign(M.values.size(), -1);
    for (size_t v = 0; v < M.values.size(); v++) value_last_use[v] = M.values[v].def_op;
    for (size_t t = 0; t < M.ops.size(); t++)
      for (int v : M.ops[t].operands) value_last_use[v] = std::max(value_last_use[v], (int)t);
    dying.assign(M.ops.size(), {});
    for (size_t v = 0; v < M.values.size(); v++) dying[value_last_use[v]].push_back((int)v);
    // baseline (C13): the empty sequence
    std::vector<u16> empty(32, 0);
    Cost c0;
    raw_eval(empty.data(), c0, /*baseline=*/true);
    flops0 = c0.flops;
    peak0 = c0.peak_bytes;
    t0 = c0.runtime_s;
    if (!(t0 > 0.0)) throw OracleError("E_DEGENERATE", "baseline runtime is 0 (no contraction op)");
  }

  // C3: conflicts — pairs of non-X loops of one op, co-occurring at one of its
  // sites, in the same component
  void find_conflicts() {
    for (size_t t = 0; t < M.ops.size(); t++) {
      std::vector<std::vector<int>> sites;
      if (M.ops[t].result >= 0) {
        std::vector<int> s;
        for (int n : nda.def_names[M.ops[t].result]) s.push_back(name_loop[n]);
        sites.push_back(s);
      }
      for (auto& u : nda.use_names[t]) {
        std::vector<int> s;
        for (int n : u) s.push_back(name_loop[n]);
        sites.push_back(s);
      }
      std::set<std::pair<int, int>> pairs;
      for (auto& s : sites)
        for (size_t a = 0; a < s.size(); a++)
          for (size_t b = 0; b < s.size(); b++) {
            int x = s[a], y = s[b];
            if (x == y) continue;
            if (loops[x].type == LX || loops[y].type == LX) continue;
            if (comp[x] != comp[y]) continue;
            pairs.insert({std::min(x, y), std::max(x, y)});   // lower loop id = lower role
          }
      for (auto& pr : pairs) {
        conflict_of[pr] = (int)conflicts.size();
        conflicts.push_back(Conflict{(int)t, pr.first, pr.second});
      }
    }
  }

  // directed path src ~> dst over M edges (ops only increase along edges)
  bool path(int src, int dst) const {
    int lim = loops[dst].op;
    std::vector<char> seen(loops.size(), 0);
    std::deque<int> q;
    q.push_back(src); seen[src] = 1;
    while (!q.empty()) {
      int x = q.front(); q.pop_front();
      if (x == dst) return true;
      for (int y : out_adj[x]) {
        if (seen[y] || loops[y].op > lim) continue;
        seen[y] = 1; q.push_back(y);
      }
    }
    return false;
  }

  // C4: the "box" relation (§3.5, Fig. 6; directed "across" paths, reading G7)
  void find_boxes() {
    std::map<std::pair<int, int>, Box> found;
    for (size_t ci = 0; ci < conflicts.size(); ci++) {
      const Conflict& c1 = conflicts[ci];
      for (int lab = 0; lab < 2; lab++) {
        int N = lab == 0 ? c1.u : c1.v;
        int O = lab == 0 ? c1.v : c1.u;
        for (int L : out_adj[N])
          for (int R : out_adj[O]) {
            if (L == R || loops[L].op != loops[R].op) continue;
            auto it = conflict_of.find({std::min(L, R), std::max(L, R)});
            if (it == conflict_of.end()) continue;
            int cj = it->second;
            if (path(N, R) || path(O, L)) continue;
            const Conflict& c2 = conflicts[cj];
            Box b{(int)ci, cj, N, O, L, R, (int)((N == c1.u) ^ (L == c2.u))};
            if (!found.count({(int)ci, cj})) found[{(int)ci, cj}] = b;
          }
      }
    }
    for (auto& kv : found) boxes.push_back(kv.second);
  }

  // C5: compatibility sets = closure of compatibility, parity union-find
  std::vector<int> pp, ppar;
  std::pair<int, int> pfind(int x) {
    if (pp[x] == x) return {x, 0};
    auto r = pfind(pp[x]);
    ppar[x] ^= r.second;
    pp[x] = r.first;
    return {pp[x], ppar[x]};
  }
  void build_sets() {
    int n = (int)conflicts.size();
    pp.resize(n); ppar.assign(n, 0);
    for (int i = 0; i < n; i++) pp[i] = i;
    box_accepted.assign(boxes.size(), 0);
    for (size_t bi = 0; bi < boxes.size(); bi++) {
      const Box& b = boxes[bi];
      auto a = pfind(b.c1), c = pfind(b.c2);
      if (a.first == c.first) {
        if ((a.second ^ c.second) != b.parity) { dropped_boxes++; continue; }
        box_accepted[bi] = 1;
        continue;
      }
      pp[c.first] = a.first;
      ppar[c.first] = a.second ^ c.second ^ b.parity;
      box_accepted[bi] = 1;
    }
    // set ids ordered by smallest conflict; side0 relative to that smallest conflict
    std::map<int, int> root_min;
    for (int i = 0; i < n; i++) {
      int r = pfind(i).first;
      if (!root_min.count(r)) root_min[r] = i;
    }
    std::map<int, int> min_set;
    for (auto& kv : root_min) min_set[kv.second] = 0;
    int sid = 0;
    for (auto& kv : min_set) { kv.second = sid++; set_root.push_back(kv.first); }
    conf_set.resize(n); conf_side0.resize(n);
    for (int i = 0; i < n; i++) {
      auto r = pfind(i);
      int mn = root_min[r.first];
      conf_set[i] = min_set[mn];
      int q = r.second ^ pfind(mn).second;
      conf_side0[i] = q == 0 ? conflicts[i].u : conflicts[i].v;
    }
  }

  // NEXT-4 (reading R23): the dimension-graph contraction heuristic
  // ([comment] §3.5): "Eagerly contract edges in the dimension
  // graph unless this produces a (directed) path between two nodes that
  // participate in a conflict."  Edges are taken once each in canonical
  // (def loop, use loop) order (contraction only adds paths, so a skipped edge
  // stays skipped and one pass is the fixpoint).  A contraction is skipped when,
  // in the contracted graph, the two endpoints of some conflict would share a
  // node or one would reach the other.  "Both vertical edges will be
  // contracted, which amounts to identifying the conflicts at the top and
  // bottom of the box as compatible": conflicts whose endpoints
  // land on the same pair of contracted nodes form one set; side 0 of a
  // conflict is its endpoint in the node of the set's smallest conflict's u.
  // Contraction never joins components, so a conflict can only acquire a path
  // through an edge of its own component: only those conflicts are checked.
  bool contracted_conflict_path(UF& t, int component) {
    std::map<int, std::set<int>> adj;   // contracted graph of the component
    for (auto& e : edges) {
      if (comp[e.first] != component) continue;
      int a = t.find(e.first), b = t.find(e.second);
      if (a != b) adj[a].insert(b);
    }
    for (auto& c : conflicts) {
      if (comp[c.u] != component) continue;
      int U = t.find(c.u), V = t.find(c.v);
      if (U == V) return true;
      for (int dir = 0; dir < 2; dir++) {   // U ~> V, then V ~> U (breadth-first)
        int src = dir == 0 ? U : V, dst = dir == 0 ? V : U;
        std::set<int> seen{src};
        std::deque<int> q{src};
        while (!q.empty()) {
          int x = q.front(); q.pop_front();
          if (x == dst) return true;
          for (int y : adj[x]) if (seen.insert(y).second) q.push_back(y);
        }
      }
    }
    return false;
  }
  void build_sets_contraction() {
    UF g((int)loops.size());
    for (auto& e : edges) {                 // std::set order: (def loop, use loop) ascending
      if (g.find(e.first) == g.find(e.second)) continue;
      UF trial = g;
      trial.unite(e.first, e.second);
      if (contracted_conflict_path(trial, comp[e.first])) { contract_rejected++; continue; }
      g = trial;
      contracted++;
    }
    cnode.resize(loops.size());
    for (size_t l = 0; l < loops.size(); l++) cnode[l] = g.find((int)l);   // unite keeps the smallest member
    // sets: conflicts on the same unordered pair of contracted nodes, numbered by smallest conflict
    int n = (int)conflicts.size();
    std::map<std::pair<int, int>, int> pair_set;
    conf_set.assign(n, -1); conf_side0.assign(n, -1);
    for (int i = 0; i < n; i++) {
      int U = cnode[conflicts[i].u], V = cnode[conflicts[i].v];
      std::pair<int, int> key{std::min(U, V), std::max(U, V)};
      if (!pair_set.count(key)) {
        pair_set[key] = (int)set_root.size();
        set_root.push_back(i);
      }
      conf_set[i] = pair_set[key];
      int root_u = cnode[conflicts[set_root[conf_set[i]]].u];
      conf_side0[i] = cnode[conflicts[i].u] == root_u ? conflicts[i].u : conflicts[i].v;
    }
  }

  // C6: SetGroups — isomorphic sets across layers (§3.6), 3-round WL
  void build_groups() {
    int ns = (int)set_root.size();
    set_sig.assign(ns, 0);
    std::vector<std::vector<int>> set_confs(ns);
    for (size_t i = 0; i < conflicts.size(); i++) set_confs[conf_set[i]].push_back((int)i);
    std::vector<std::vector<int>> set_boxes(ns);
    for (size_t bi = 0; bi < boxes.size(); bi++)
      if (box_accepted[bi]) set_boxes[conf_set[boxes[bi].c1]].push_back((int)bi);
    for (int s = 0; s < ns; s++) {
      std::map<int, int> sidemask;
      std::set<std::pair<int, int>> conf_edges;
      for (int c : set_confs[s]) {
        const Conflict& cf = conflicts[c];
        int s0 = conf_side0[c];
        int s1 = s0 == cf.u ? cf.v : cf.u;
        sidemask[s0] |= 1;
        sidemask[s1] |= 2;
        conf_edges.insert({cf.u, cf.v});
      }
      std::set<std::pair<int, int>> m_edges;
      if (grouping == 0) {
        for (int bi : set_boxes[s]) {
          m_edges.insert({boxes[bi].N, boxes[bi].L});
          m_edges.insert({boxes[bi].O, boxes[bi].R});
        }
      } else {
        // R23: the contracted M edges between the set's endpoints (the analogue of its boxes' vertical edges)
        for (auto& e : edges)
          if (sidemask.count(e.first) && sidemask.count(e.second) && cnode[e.first] == cnode[e.second])
            m_edges.insert(e);
      }
      set_graphs.push_back(SetGraph{sidemask, m_edges, conf_edges});
      std::map<int, u64> label;
      for (auto& kv : sidemask) {
        int l = kv.first;
        label[l] = hseq({fnv1a(M.ops[loops[l].op].kind), (u64)loops[l].role, (u64)loops[l].type, (u64)kv.second});
      }
      for (int round = 0; round < 3; round++) {
        std::map<int, u64> next;
        for (auto& kv : label) {
          int n = kv.first;
          std::vector<u64> outs, ins, cfs;
          for (auto& e : m_edges) {
            if (e.first == n) outs.push_back(label[e.second]);
            if (e.second == n) ins.push_back(label[e.first]);
          }
          for (auto& e : conf_edges) {
            if (e.first == n) cfs.push_back(label[e.second]);
            if (e.second == n) cfs.push_back(label[e.first]);
          }
          std::sort(outs.begin(), outs.end());
          std::sort(ins.begin(), ins.end());
          std::sort(cfs.begin(), cfs.end());
          next[n] = hseq({kv.second, hseq(outs), hseq(ins), hseq(cfs)});
        }
        label = next;
      }
      std::vector<u64> fin;
      for (auto& kv : label) fin.push_back(kv.second);
      std::sort(fin.begin(), fin.end());
      set_sig[s] = hseq(fin);
    }
    std::map<u64, int> sig_group;
    set_group.assign(ns, -1);
    for (int s = 0; s < ns; s++) {   // sets are in smallest-conflict order
      if (!sig_group.count(set_sig[s])) sig_group[set_sig[s]] = n_groups++;
      set_group[s] = sig_group[set_sig[s]];
    }
  }

  // C7: argument groups by keys from all uses (§4.4) -> super-colors
  void build_supercolors() {
    typedef std::tuple<std::string, int, int, int> UseKey;
    std::map<std::tuple<std::string, std::vector<i64>, std::vector<std::vector<UseKey>>>, std::vector<int>> groups;
    for (int p = 0; p < M.n_params; p++) {
      int v = M.ops[p].result;
      size_t rank = M.values[v].shape.size();
      std::vector<std::vector<UseKey>> per_dim(rank);
      for (size_t t = 0; t < M.ops.size(); t++)
        for (size_t k = 0; k < M.ops[t].operands.size(); k++)
          if (M.ops[t].operands[k] == v)
            for (size_t i = 0; i < rank; i++) {
              int l = use_loop((int)t, (int)k, (int)i);
              per_dim[i].push_back(UseKey{M.ops[t].kind, (int)k, loops[l].role, loops[l].type});
            }
      for (auto& d : per_dim) std::sort(d.begin(), d.end());
      groups[std::make_tuple(M.values[v].dtype, M.values[v].shape, per_dim)].push_back(v);
    }
    UF su((int)loops.size());
    for (size_t l = 0; l < loops.size(); l++) su.unite((int)l, comp[l]);
    for (auto& kv : groups) {
      const auto& members = kv.second;
      for (size_t j = 1; j < members.size(); j++)
        for (size_t i = 0; i < M.values[members[0]].shape.size(); i++)
          su.unite(def_loop(members[0], (int)i), def_loop(members[j], (int)i));
    }
    std::map<int, int> root_id;
    for (size_t l = 0; l < loops.size(); l++) {
      int r = su.find((int)l);
      if (!root_id.count(r)) { root_id[r] = (int)sc_min_loop.size(); sc_min_loop.push_back((int)l); }
    }
    scolor.resize(loops.size());
    for (size_t l = 0; l < loops.size(); l++) scolor[l] = root_id[su.find((int)l)];
    int nsc = (int)sc_min_loop.size();
    sc_value_dims.assign(nsc, 0);
    for (size_t v = 0; v < M.values.size(); v++)
      for (size_t i = 0; i < M.values[v].shape.size(); i++) sc_value_dims[scolor[def_loop((int)v, (int)i)]]++;
    std::vector<std::set<int>> g(nsc);
    for (size_t c = 0; c < conflicts.size(); c++) g[scolor[conflicts[c].u]].insert(set_group[conf_set[c]]);
    sc_groups.resize(nsc);
    for (int c = 0; c < nsc; c++) sc_groups[c] = std::vector<int>(g[c].begin(), g[c].end());
  }

  // C8: action table (§4.2)
  void build_actions() {
    actions.push_back(Action{-1, 0, -1});   // id 0 = STOP
    for (size_t c = 0; c < sc_min_loop.size(); c++) {
      if (sc_value_dims[c] < min_dims) continue;
      if (sc_groups[c].size() > 8) throw OracleError("E_LIMIT", "more than 8 SetGroups in one super-color");
      int nr = 1 << sc_groups[c].size();
      for (int r = 0; r < nr; r++)
        for (size_t a = 0; a < axes.size(); a++) actions.push_back(Action{(int)c, r, (int)a});
    }
    if (actions.size() > 1024) throw OracleError("E_LIMIT", "more than 1023 actions");
  }

  int group_bit(int sc, int r, int g) const {
    for (size_t t = 0; t < sc_groups[sc].size(); t++) if (sc_groups[sc][t] == g) return (r >> t) & 1;
    return -1;
  }

  // ------------------------------------------------------------------
  // C9–C14: one candidate
  // ------------------------------------------------------------------
  void raw_eval(const u16* seq, Cost& out, bool baseline = false) const {
    memset(&out, 0, sizeof(out));
    // C9 decode
    u32 status = 0;
    std::vector<int> acts;
    bool stopped = false;
    for (int i = 0; i < 32; i++) {
      int id = seq[i];
      if (stopped) { if (id != 0) status |= ST_NONZERO_AFTER_STOP; continue; }
      if (id == 0) { stopped = true; continue; }
      if (id >= (int)actions.size()) { status |= ST_BAD_ACTION_ID; continue; }
      acts.push_back(id);
    }
    std::set<std::pair<int, int>> seen_ca;
    std::map<int, int> fixed;   // group -> bit
    for (int id : acts) {
      const Action& a = actions[id];
      if (seen_ca.count({a.sc, a.axis})) status |= ST_DUP_COLOR_AXIS;
      seen_ca.insert({a.sc, a.axis});
      for (size_t t = 0; t < sc_groups[a.sc].size(); t++) {
        int g = sc_groups[a.sc][t];
        int b = (a.r >> t) & 1;
        if (fixed.count(g) && fixed[g] != b) status |= ST_RES_MISMATCH;
        if (!fixed.count(g)) fixed[g] = b;
      }
    }
    if (status) { out.status = status; return; }
    // deselected loops: the deselected endpoint of a conflict whose group bit is fixed
    std::vector<char> desel(loops.size(), 0);
    for (size_t c = 0; c < conflicts.size(); c++) {
      int g = set_group[conf_set[c]];
      auto it = fixed.find(g);
      if (it == fixed.end()) continue;
      int s0 = conf_side0[c];
      int s1 = s0 == conflicts[c].u ? conflicts[c].v : conflicts[c].u;
      desel[it->second == 0 ? s1 : s0] = 1;
    }
    // C9 materialize ("attempts to shard all dimensions"; one axis per op P:744)
    std::vector<int> mask(loops.size(), 0);
    for (size_t t = 0; t < M.ops.size(); t++) {
      for (int id : acts) {
        const Action& a = actions[id];
        for (int r = 0; r < nloops((int)t); r++) {
          int l = loop_of((int)t, r);
          if (scolor[l] != a.sc) continue;
          if (loops[l].type == LX) continue;
          if (desel[l]) continue;
          int opm = 0;
          for (int r2 = 0; r2 < nloops((int)t); r2++) opm |= mask[loop_of((int)t, r2)];
          if (opm & (1 << a.axis)) continue;
          i64 prod = axes[a.axis].size;
          for (size_t A = 0; A < axes.size(); A++) if (mask[l] & (1 << A)) prod *= axes[A].size;
          if (loops[l].ext % prod != 0) continue;
          mask[l] |= 1 << a.axis;
        }
      }
    }
    eval_masks(mask, out);
    (void)baseline;
  }

  u64 axes_prod(int m) const {
    u64 p = 1;
    for (size_t A = 0; A < axes.size(); A++) if (m & (1 << A)) p *= (u64)axes[A].size;
    return p;
  }
  u64 elem(int v) const { return (u64)dtype_bytes(M.values[v].dtype); }
  u64 global_bytes(int v) const {
    u64 b = elem(v);
    for (i64 e : M.values[v].shape) b *= (u64)e;
    return b;
  }
  std::vector<int> layout_D(const std::vector<int>& mask, int v) const {
    std::vector<int> D;
    for (size_t i = 0; i < M.values[v].shape.size(); i++) D.push_back(mask[def_loop(v, (int)i)]);
    return D;
  }
  int partial_P(const std::vector<int>& mask, int v) const {
    int t = M.values[v].def_op, P = 0;
    for (int r = 0; r < nloops(t); r++) if (loops[loop_of(t, r)].type == LR) P |= mask[loop_of(t, r)];
    return P;
  }
  u64 local_bytes_of(int v, const std::vector<int>& D) const {
    int all = 0;
    for (int m : D) all |= m;
    return global_bytes(v) / axes_prod(all);
  }

  // profile (optional): M_t of every op t, the quantity C12 maximises
  void eval_masks(const std::vector<int>& mask, Cost& out, std::vector<i64>* profile = nullptr) const {
    // C10: FLOPs over matmul-class ops only
    u128 flops = 0;
    std::vector<u128> op_flops(M.ops.size(), 0);   // per op, for the critical path (R22)
    for (size_t t = 0; t < M.ops.size(); t++) {
      const std::string& k = M.ops[t].kind;
      if (k != "matmul" && k != "dot_general" && k != "conv2d" && k != "conv2d_bwd_input" && k != "conv2d_bwd_filter") continue;
      u128 f = 2;
      for (int r = 0; r < nloops((int)t); r++) {
        int l = loop_of((int)t, r);
        f *= (u128)((u64)loops[l].ext / axes_prod(mask[l]));
      }
      flops += f;
      op_flops[t] = f;
    }
    // C11: collectives per use edge (Fig. 2c; Fig. 5b)
    std::vector<u64> temp_total(M.ops.size(), 0);
    int nA = (int)axes.size();
    u64 ncount[4][4] = {{0}};   // true counts; the record keeps them saturated to 16 bits
    // R22: per use edge, the duration of its own collectives (the same ring
    // formula as C13 over this edge's payloads); a within-op duplicate waits
    // for the same collectives
    std::vector<std::vector<double>> edge_m(M.ops.size());
    for (size_t t = 0; t < M.ops.size(); t++) {
      const Op& op = M.ops[t];
      std::vector<std::pair<int, std::vector<int>>> done;   // (value, U) already costed at this op
      std::vector<double> done_m;
      std::map<int, i64> temp;                              // per distinct operand value
      edge_m[t].assign(op.operands.size(), 0.0);
      for (size_t k = 0; k < op.operands.size(); k++) {
        int v = op.operands[k];
        std::vector<int> U;
        for (size_t i = 0; i < M.values[v].shape.size(); i++) U.push_back(mask[use_loop((int)t, (int)k, (int)i)]);
        if (!temp.count(v)) temp[v] = 0;
        int dup = -1;
        for (size_t q = 0; q < done.size(); q++) if (done[q].first == v && done[q].second == U) dup = (int)q;
        if (dup >= 0) { edge_m[t][k] = done_m[dup]; continue; }
        done.push_back({v, U});
        done_m.push_back(0.0);
        std::vector<int> D = layout_D(mask, v);
        int P = partial_P(mask, v);
        if (D == U && P == 0) continue;
        std::vector<int> cur = D;
        u64 size = local_bytes_of(v, D);
        u64 ep[4][4] = {{0}};   // this edge's payloads [axis][kind]
        // phase 1: axes of D not kept in the same dim (reading R20):
        // 1a all_gather every axis U holds on no dim, then 1b all_to_all every
        // axis U holds on another dim — so every intermediate layout keeps
        // only axes of D (1a) or of U (1b) on each dim and stays divisible
        for (int A = 0; A < nA; A++) {
          for (size_t i = 0; i < D.size(); i++) {
            if (!(cur[i] & (1 << A)) || (U[i] & (1 << A))) continue;
            bool elsewhere = false;
            for (size_t j = 0; j < U.size(); j++) if (j != i && (U[j] & (1 << A))) elsewhere = true;
            if (elsewhere) continue;
            ep[A][K_AG] += size; ncount[A][K_AG]++;
            cur[i] &= ~(1 << A); size *= (u64)axes[A].size;
          }
        }
        for (int A = 0; A < nA; A++) {
          for (size_t i = 0; i < D.size(); i++) {
            if (!(cur[i] & (1 << A)) || (U[i] & (1 << A))) continue;
            int j_other = -1;
            for (size_t j = 0; j < U.size(); j++) if (j != i && (U[j] & (1 << A))) j_other = (int)j;
            ep[A][K_A2A] += size; ncount[A][K_A2A]++;
            cur[i] &= ~(1 << A); cur[j_other] |= 1 << A;
          }
        }
        // phase 2: partial sums
        for (int A = 0; A < nA; A++) {
          if (!(P & (1 << A))) continue;
          int j_u = -1;
          for (size_t j = 0; j < U.size(); j++) if (U[j] & (1 << A)) j_u = (int)j;
          if (j_u >= 0) {
            size /= (u64)axes[A].size;
            ep[A][K_RS] += size; ncount[A][K_RS]++;
            cur[j_u] |= 1 << A;
          } else {
            ep[A][K_AR] += size; ncount[A][K_AR]++;
          }
        }
        // phase 3: free local slices (no payload)
        double m = 0.0;
        for (int A = 0; A < nA; A++) {
          for (int kk = 0; kk < 4; kk++) out.payload[A][kk] += ep[A][kk];
          double n = (double)axes[A].size;
          double ag = (double)ep[A][K_AG], rs = (double)ep[A][K_RS];
          double ar = (double)ep[A][K_AR], a2a = (double)ep[A][K_A2A];
          double term = ((n - 1.0) * (ag + rs) + ((n - 1.0) * (2.0 * ar + a2a)) / n) / axes[A].bw;
          m = m + term;
        }
        edge_m[t][k] = m;
        done_m.back() = m;
        // temporaries: only gathers grow the operand buffer
        u64 use_local = local_bytes_of(v, U);
        i64 grow = (i64)use_local - (i64)local_bytes_of(v, D);
        if (grow > temp[v]) temp[v] = grow;
      }
      for (auto& kv : temp) temp_total[t] += (u64)kv.second;
    }
    // C12: liveness
    i64 L = 0, peak = 0;
    for (size_t t = 0; t < M.ops.size(); t++) {
      int rv = M.ops[t].result;
      i64 res = rv >= 0 ? (i64)local_bytes_of(rv, layout_D(mask, rv)) : 0;
      i64 Mt = L + res + (i64)temp_total[t];
      if (profile) profile->push_back(Mt);
      if (Mt > peak) peak = Mt;
      i64 dying_bytes = 0;
      for (int v : dying[t]) dying_bytes += (i64)local_bytes_of(v, layout_D(mask, v));
      L = L + res - dying_bytes;
    }
    // C14 (reading R14): the state is "the final sharding configuration
    // itself": the set of (op, axis, loop role holding the axis).
    // key = sum over that set of mix64(first loop id << 8 | axis << 4 | role), mod 2^64.
    u64 key = 0;
    for (size_t t = 0; t < M.ops.size(); t++)
      for (int r = 0; r < nloops((int)t); r++)
        for (int A = 0; A < 4; A++)
          if (mask[loop_of((int)t, r)] & (1 << A)) key += mix64(((u64)op_loop_begin[t] << 8) | ((u64)A << 4) | (u64)r);
    // C13: runtime and score
    u64 flo = (u64)flops, fhi = (u64)(flops >> 64);
    double fl = (double)fhi * 18446744073709551616.0 + (double)flo;
    double t = fl / F;
    for (int A = 0; A < nA; A++) {
      double n = (double)axes[A].size;
      double ag = (double)out.payload[A][K_AG], rs = (double)out.payload[A][K_RS];
      double ar = (double)out.payload[A][K_AR], a2a = (double)out.payload[A][K_A2A];
      double term = ((n - 1.0) * (ag + rs) + ((n - 1.0) * (2.0 * ar + a2a)) / n) / axes[A].bw;
      t = t + term;
    }
    if (cost_model == 1) {
      // R22 ("runtime cost is accumulated along the critical path"):
      // finish(t) = max over t's operands, in operand order, of (finish of the
      // operand's def + its edge's collective duration) + t's compute time;
      // parameters finish at 0; runtime = the latest finish
      std::vector<double> fin(M.values.size(), 0.0);
      double cp = 0.0;
      for (size_t tt = 0; tt < M.ops.size(); tt++) {
        const Op& op = M.ops[tt];
        double ready = 0.0;
        for (size_t k = 0; k < op.operands.size(); k++) {
          double f = fin[op.operands[k]] + edge_m[tt][k];
          if (f > ready) ready = f;
        }
        double ct = (double)(u64)op_flops[tt] / F;
        double ft = ready + ct;
        if (op.result >= 0) fin[op.result] = ft;
        if (ft > cp) cp = ft;
      }
      t = cp;
    }
    out.runtime_s = t;
    out.peak_bytes = (u64)peak;
    out.flops = flo;
    out.flops_hi = fhi;
    out.state_key = key;
    u64 nc = 0;
    for (int A = 0; A < 4; A++)
      for (int k = 0; k < 4; k++) {
        nc += ncount[A][k];
        out.count[A][k] = (u16)(ncount[A][k] > 65535 ? 65535 : ncount[A][k]);
      }
    out.n_collectives = (u32)nc;
    if (t0 > 0.0) {
      double RT = t / t0;
      double MP = (u64)peak > DM ? (C * (double)((u64)peak - DM)) / (double)peak0 : 0.0;
      out.score = RT + MP;
    }
  }

  // C9 materialization only (for tests): per-loop masks
  void materialize(const u16* seq, std::vector<int>& mask_out) const {
    Cost c; raw_eval(seq, c);
    mask_out.assign(loops.size(), 0);
    if (c.status) return;
    // recompute (raw_eval keeps masks local); duplicate of the C9 loop by design
    std::vector<int> acts;
    for (int i = 0; i < 32 && seq[i]; i++) acts.push_back(seq[i]);
    std::map<int, int> fixed;
    for (int id : acts) {
      const Action& a = actions[id];
      for (size_t t = 0; t < sc_groups[a.sc].size(); t++) fixed[sc_groups[a.sc][t]] = (a.r >> t) & 1;
    }
    std::vector<char> desel(loops.size(), 0);
    for (size_t c2 = 0; c2 < conflicts.size(); c2++) {
      auto it = fixed.find(set_group[conf_set[c2]]);
      if (it == fixed.end()) continue;
      int s0 = conf_side0[c2];
      int s1 = s0 == conflicts[c2].u ? conflicts[c2].v : conflicts[c2].u;
      desel[it->second == 0 ? s1 : s0] = 1;
    }
    for (size_t t = 0; t < M.ops.size(); t++)
      for (int id : acts) {
        const Action& a = actions[id];
        for (int r = 0; r < nloops((int)t); r++) {
          int l = loop_of((int)t, r);
          if (scolor[l] != a.sc || loops[l].type == LX || desel[l]) continue;
          int opm = 0;
          for (int r2 = 0; r2 < nloops((int)t); r2++) opm |= mask_out[loop_of((int)t, r2)];
          if (opm & (1 << a.axis)) continue;
          i64 prod = axes[a.axis].size;
          for (size_t A = 0; A < axes.size(); A++) if (mask_out[l] & (1 << A)) prod *= axes[A].size;
          if (loops[l].ext % prod != 0) continue;
          mask_out[l] |= 1 << a.axis;
        }
      }
  }

  // ------------------------------------------------------------------
  // C15: legality / kills and rollout
  // ------------------------------------------------------------------
  bool kills(int chosen, int other) const {
    const Action& a = actions[chosen];
    const Action& b = actions[other];
    if (a.sc == b.sc && a.axis == b.axis) return true;
    for (size_t t = 0; t < sc_groups[a.sc].size(); t++) {
      int g = sc_groups[a.sc][t];
      int bb = group_bit(b.sc, b.r, g);
      if (bb >= 0 && bb != ((a.r >> t) & 1)) return true;
    }
    return false;
  }

  void rollout(const u16* prefix, u64 seed, u64 id, u16* out_seq, Cost& out) const {
    std::vector<u16> seq;
    bool bad = false, stopped = false;
    for (int i = 0; i < 32; i++) {
      if (stopped) { if (prefix[i]) bad = true; continue; }
      if (prefix[i] == 0) { stopped = true; continue; }
      if (prefix[i] >= actions.size()) bad = true;
      seq.push_back(prefix[i]);
    }
    if (!bad) {
      std::set<int> legal;
      for (size_t a = 1; a < actions.size(); a++) legal.insert((int)a);
      for (u16 a : seq) {
        std::vector<int> dead;
        for (int b : legal) if (kills(a, b)) dead.push_back(b);
        for (int b : dead) legal.erase(b);
      }
      int d = (int)seq.size();
      while (d < max_depth) {
        u32 ctr[4] = {(u32)id, (u32)(id >> 32), (u32)d, 0u};
        u32 key[2] = {(u32)seed, (u32)(seed >> 32)};
        u32 r[4];
        philox4x32_10(ctr, key, r);
        if ((u64)r[0] * (u64)max_depth < ((u64)d << 32)) break;   // p_stop = d / max_depth
        if (legal.empty()) break;
        u64 k = ((u64)r[1] * (u64)legal.size()) >> 32;
        auto it = legal.begin();
        std::advance(it, (long)k);
        int a = *it;
        std::vector<int> dead;
        for (int b : legal) if (kills(a, b)) dead.push_back(b);
        for (int b : dead) legal.erase(b);
        seq.push_back((u16)a);
        d++;
      }
    }
    for (int i = 0; i < 32; i++) out_seq[i] = 0;
    if (bad) { for (int i = 0; i < 32; i++) out_seq[i] = prefix[i]; }
    else for (size_t i = 0; i < seq.size() && i < 32; i++) out_seq[i] = seq[i];
    raw_eval(out_seq, out);
  }

  // ------------------------------------------------------------------
  // C17: brute force over all legal sequences
  // ------------------------------------------------------------------
  static bool better(const Cost& a, const u16* sa, const Cost& b, const u16* sb) {
    if (a.score != b.score) return a.score < b.score;
    if (a.state_key != b.state_key) return a.state_key < b.state_key;
    for (int i = 0; i < 32; i++) if (sa[i] != sb[i]) return sa[i] < sb[i];
    return false;
  }
  i64 brute(std::vector<u16>& seq, std::set<int> legal, u16* best_seq, Cost& best, bool& have) const {
    u16 s[32] = {0};
    for (size_t i = 0; i < seq.size(); i++) s[i] = seq[i];
    Cost c; raw_eval(s, c);
    i64 n = 1;
    if (!have || better(c, s, best, best_seq)) { best = c; memcpy(best_seq, s, sizeof(s)); have = true; }
    if ((int)seq.size() >= max_depth) return n;
    for (int a : legal) {
      std::set<int> nl;
      for (int b : legal) if (!kills(a, b)) nl.insert(b);
      seq.push_back((u16)a);
      n += brute(seq, nl, best_seq, best, have);
      seq.pop_back();
    }
    return n;
  }
};

// ---------------------------------------------------------------------------
// C16: MCTS, the spec in DESIGN.md §"Search"
// ---------------------------------------------------------------------------
struct Node {
  std::vector<u16> prefix;
  std::vector<int> untried;            // ascending legal action ids not yet expanded
  std::vector<Node*> children;
  Node* parent = nullptr;
  double W = 0.0;
  i64 N = 0;
  bool expanded_all() const { return untried.empty(); }
};

struct SearchOut {
  u16 best_seq[32];
  Cost best;
  i64 evals;
  int rounds;
  int hit_target;
  double wall_s;
  double time_to_target_s;
};

static void free_tree(Node* n) { for (Node* c : n->children) free_tree(c); delete n; }

static std::vector<int> legal_after(const Oracle& O, const std::vector<u16>& prefix) {
  std::vector<int> legal;
  for (size_t a = 1; a < O.actions.size(); a++) {
    bool ok = true;
    for (u16 p : prefix) if (O.kills(p, (int)a)) { ok = false; break; }
    if (ok) legal.push_back((int)a);
  }
  if ((int)prefix.size() >= O.max_depth) legal.clear();
  return legal;
}

}  // namespace orc

// =============================================================================
// C ABI for the tests (ctypes) — test infrastructure only
// =============================================================================
using namespace orc;

static thread_local std::string g_err;

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// axes: "name=size:bw,name=size:bw"
void* orc_new(const char* ir, const char* mesh, double F, uint64_t DM, double C, int min_dims, int max_depth,
              int cost_model, int grouping) {
  try {
    auto* O = new Oracle();
    std::string ms(mesh);
    size_t p = 0;
    while (p < ms.size()) {
      size_t q = ms.find(',', p);
      if (q == std::string::npos) q = ms.size();
      std::string item = ms.substr(p, q - p);
      size_t eq = item.find('='), col = item.find(':');
      Axis a;
      a.name = item.substr(0, eq);
      a.size = strtoll(item.substr(eq + 1, col - eq - 1).c_str(), nullptr, 10);
      a.bw = strtod(item.substr(col + 1).c_str(), nullptr);
      O->axes.push_back(a);
      p = q + 1;
    }
    if (O->axes.empty() || O->axes.size() > 4) throw OracleError("E_MESH", "mesh must have 1..4 axes");
    for (auto& a : O->axes) if (a.size < 2 || !(a.bw > 0)) throw OracleError("E_MESH", "axis size < 2 or bw <= 0");
    O->F = F; O->DM = DM; O->C = C; O->min_dims = min_dims; O->max_depth = max_depth;
    if (cost_model != 0 && cost_model != 1) throw OracleError("E_INVALID_ARG", "cost_model must be 0 or 1");
    O->cost_model = cost_model;
    if (grouping != 0 && grouping != 1) throw OracleError("E_INVALID_ARG", "grouping must be 0 or 1");
    O->grouping = grouping;
    O->M = parse_module(ir);
    O->build();
    return O;
  } catch (OracleError& e) {
    g_err = e.code + ": " + e.what();
    return nullptr;
  } catch (std::exception& e) {
    g_err = std::string("E_INTERNAL: ") + e.what();
    return nullptr;
  }
}

void orc_free(void* h) { delete (Oracle*)h; }
int orc_n_actions(void* h) { return (int)((Oracle*)h)->actions.size(); }
int orc_n_loops(void* h) { return (int)((Oracle*)h)->loops.size(); }
int orc_n_ops(void* h) { return (int)((Oracle*)h)->M.ops.size(); }

static void run_threads(int64_t n, int threads, const std::function<void(int64_t)>& f) {
  if (threads <= 1 || n < 2) { for (int64_t i = 0; i < n; i++) f(i); return; }
  std::vector<std::thread> th;
  for (int w = 0; w < threads; w++)
    th.emplace_back([&, w]() { for (int64_t i = w; i < n; i += threads) f(i); });
  for (auto& t : th) t.join();
}

void orc_eval(void* h, const uint16_t* seqs, int64_t n, void* out, int threads) {
  Oracle* O = (Oracle*)h;
  Cost* c = (Cost*)out;
  run_threads(n, threads, [&](int64_t i) { O->raw_eval(seqs + 32 * i, c[i]); });
}

void orc_rollout(void* h, const uint16_t* prefixes, int64_t n, uint64_t seed, uint64_t id_base, uint16_t* out_seqs, void* out, int threads) {
  Oracle* O = (Oracle*)h;
  Cost* c = (Cost*)out;
  run_threads(n, threads, [&](int64_t i) { O->rollout(prefixes + 32 * i, seed, id_base + (uint64_t)i, out_seqs + 32 * i, c[i]); });
}

void orc_materialize(void* h, const uint16_t* seq, uint8_t* masks) {
  Oracle* O = (Oracle*)h;
  std::vector<int> m;
  O->materialize(seq, m);
  for (size_t i = 0; i < m.size(); i++) masks[i] = (uint8_t)m[i];
}

// the liveness profile of one sequence: M_t for every op t (C12), n_ops values
void orc_profile(void* h, const uint16_t* seq, int64_t* out) {
  Oracle* O = (Oracle*)h;
  std::vector<int> m;
  O->materialize(seq, m);
  Cost c;
  std::vector<i64> prof;
  O->eval_masks(m, c, &prof);
  for (size_t t = 0; t < prof.size(); t++) out[t] = prof[t];
}

int64_t orc_bruteforce(void* h, uint16_t* best_seq, void* best_cost) {
  Oracle* O = (Oracle*)h;
  std::vector<u16> seq;
  std::set<int> legal;
  for (size_t a = 1; a < O->actions.size(); a++) legal.insert((int)a);
  bool have = false;
  Cost best;
  int64_t n = O->brute(seq, legal, best_seq, best, have);
  memcpy(best_cost, &best, sizeof(Cost));
  return n;
}

// I-quotient lookups (Fig. 4b): loop of (op t, operand k, dim i) / of the definition of op t's result, dim i
int orc_use_loop(void* h, int t, int k, int i) { return ((Oracle*)h)->use_loop(t, k, i); }
int orc_def_loop(void* h, int t, int i) { Oracle* O = (Oracle*)h; return O->def_loop(O->M.ops[t].result, i); }
int orc_n_names(void* h) { return ((Oracle*)h)->nda.n_names; }
int orc_n_identities(void* h) { return (int)((Oracle*)h)->nda.I.size(); }
int orc_n_map(void* h) { return (int)((Oracle*)h)->nda.M.size(); }
// the deduplicated M edges over loops (C1), as (def loop, use loop) pairs in canonical order; returns the count
int orc_edges(void* h, int* out, int cap) {
  Oracle* O = (Oracle*)h;
  int n = 0;
  for (auto& e : O->edges) {
    if (n < cap) { out[2 * n] = e.first; out[2 * n + 1] = e.second; }
    n++;
  }
  return n;
}

void orc_philox(const uint32_t* ctr, const uint32_t* key, uint32_t* out) { philox4x32_10(ctr, key, out); }

// baseline: flops(lo), peak0, t0
void orc_baseline(void* h, double* t0, uint64_t* peak0, uint64_t* flops0) {
  Oracle* O = (Oracle*)h;
  *t0 = O->t0; *peak0 = O->peak0; *flops0 = O->flops0;
}

// JSON dump of the analysis (for library-vs-oracle parity of H0)
int64_t orc_dump(void* h, char* buf, int64_t cap) {
  Oracle* O = (Oracle*)h;
  std::string s = "{";
  auto num = [](i64 x) { return std::to_string(x); };
  s += "\"n_ops\":" + num(O->M.ops.size()) + ",\"n_loops\":" + num(O->loops.size()) + ",\"n_edges\":" + num(O->edges.size());
  s += ",\"loops\":[";
  for (size_t l = 0; l < O->loops.size(); l++) {
    if (l) s += ",";
    const Loop& L = O->loops[l];
    s += "[" + num(L.op) + "," + num(L.role) + "," + num(L.ext) + "," + num(L.type) + "," + num(O->comp[l]) + "," + num(O->scolor[l]) + "]";
  }
  s += "],\"conflicts\":[";
  for (size_t c = 0; c < O->conflicts.size(); c++) {
    if (c) s += ",";
    const Conflict& C = O->conflicts[c];
    s += "[" + num(C.op) + "," + num(C.u) + "," + num(C.v) + "," + num(O->conf_set[c]) + "," + num(O->conf_side0[c]) + "]";
  }
  s += "],\"n_boxes\":" + num(O->boxes.size()) + ",\"dropped_boxes\":" + num(O->dropped_boxes);
  s += ",\"contracted\":" + num(O->contracted) + ",\"contract_rejected\":" + num(O->contract_rejected);
  if (O->grouping == 1) {
    s += ",\"cnode\":[";
    for (size_t l = 0; l < O->cnode.size(); l++) { if (l) s += ","; s += num(O->cnode[l]); }
    s += "]";
  }
  s += ",\"set_group\":[";
  for (size_t i = 0; i < O->set_group.size(); i++) { if (i) s += ","; s += num(O->set_group[i]); }
  s += "],\"set_sig\":[";
  for (size_t i = 0; i < O->set_sig.size(); i++) {
    if (i) s += ",";
    char b[32]; snprintf(b, sizeof b, "\"%016llx\"", (unsigned long long)O->set_sig[i]); s += b;
  }
  s += "],\"set_graphs\":[";
  for (size_t i = 0; i < O->set_graphs.size(); i++) {
    const auto& G = O->set_graphs[i];
    if (i) s += ",";
    s += "{\"nodes\":[";
    bool first = true;
    for (auto& kv : G.side) {
      const Loop& L = O->loops[kv.first];
      if (!first) s += ",";
      first = false;
      s += "[" + num(kv.first) + ",\"" + O->M.ops[L.op].kind + "\"," + num(L.role) + "," + num(L.type) + "," + num(kv.second) + "]";
    }
    s += "],\"medges\":[";
    first = true;
    for (auto& e : G.medges) { if (!first) s += ","; first = false; s += "[" + num(e.first) + "," + num(e.second) + "]"; }
    s += "],\"cedges\":[";
    first = true;
    for (auto& e : G.cedges) { if (!first) s += ","; first = false; s += "[" + num(e.first) + "," + num(e.second) + "]"; }
    s += "]}";
  }
  s += "],\"n_groups\":" + num(O->n_groups);
  s += ",\"scolors\":[";
  for (size_t c = 0; c < O->sc_min_loop.size(); c++) {
    if (c) s += ",";
    s += "[" + num(O->sc_min_loop[c]) + "," + num(O->sc_value_dims[c]) + ",[";
    for (size_t g = 0; g < O->sc_groups[c].size(); g++) { if (g) s += ","; s += num(O->sc_groups[c][g]); }
    s += "]]";
  }
  s += "],\"actions\":[";
  for (size_t a = 1; a < O->actions.size(); a++) {
    if (a > 1) s += ",";
    s += "[" + num(O->actions[a].sc) + "," + num(O->actions[a].r) + "," + num(O->actions[a].axis) + "]";
  }
  char b[128];
  snprintf(b, sizeof b, "],\"baseline\":{\"runtime\":%.17g,\"peak\":%llu,\"flops\":%llu}}", O->t0,
           (unsigned long long)O->peak0, (unsigned long long)O->flops0);
  s += b;
  if ((int64_t)s.size() + 1 <= cap) memcpy(buf, s.c_str(), s.size() + 1);
  return (int64_t)s.size() + 1;
}

// C16 search (single process).  rollout_threads = CPU threads for the batch.
int orc_search(void* h, uint64_t seed, int64_t max_evals, double time_limit_s, int L, int R, int patience,
               double uct_c, double target_score, int threads, void* result, double* trace, int trace_cap,
               int transpositions) {
  Oracle* O = (Oracle*)h;
  SearchOut* res = (SearchOut*)result;
  memset(res, 0, sizeof(SearchOut));
  auto tstart = std::chrono::steady_clock::now();
  auto elapsed = [&]() { return std::chrono::duration<double>(std::chrono::steady_clock::now() - tstart).count(); };
  Node* root = new Node();
  root->untried = legal_after(*O, root->prefix);
  std::map<u64, Node*> holder;   // reading R24: which node holds each materialised state (by its key)
  // the root is the unsharded module: it is the first incumbent
  bool have = true;
  Cost best;
  u16 best_seq[32] = {0};
  O->raw_eval(best_seq, best);
  holder[best.state_key] = root;
  i64 evals = 1, rollouts_done = 0;
  int rounds = 0, nonimprove = 0;
  res->time_to_target_s = -1.0;
  while (true) {
    std::vector<Node*> leaves;
    for (int l = 0; l < L; l++) {
      Node* node = root;
      while (true) {
        if (!node->untried.empty()) {
          Node* ch = new Node();
          ch->prefix = node->prefix;
          ch->prefix.push_back((u16)node->untried.front());
          node->untried.erase(node->untried.begin());
          ch->parent = node;
          ch->untried = legal_after(*O, ch->prefix);
          node->children.push_back(ch);
          node = ch;
          break;
        }
        if (node->children.empty()) break;
        Node* bestc = nullptr; double bv = 0;
        for (Node* ch : node->children) {
          double v = ch->W / (double)ch->N + uct_c * std::sqrt(std::log((double)node->N) / (double)ch->N);
          if (!bestc || v > bv) { bestc = ch; bv = v; }
        }
        node = bestc;
      }
      for (Node* x = node; x; x = x->parent) { x->N += 1; x->W -= 1.0; }   // virtual loss
      leaves.push_back(node);
    }
    // (1) each selected leaf's own state, evaluated exactly; (2) R rollouts from it
    std::vector<u16> lpre((size_t)L * 32, 0);
    for (int l = 0; l < L; l++)
      for (size_t i = 0; i < leaves[l]->prefix.size(); i++) lpre[(size_t)l * 32 + i] = leaves[l]->prefix[i];
    std::vector<Cost> lcost((size_t)L);
    orc_eval(O, lpre.data(), (int64_t)L, lcost.data(), threads);
    std::vector<u16> pre((size_t)L * R * 32, 0), outs((size_t)L * R * 32, 0);
    for (int l = 0; l < L; l++)
      for (int j = 0; j < R; j++)
        for (size_t i = 0; i < leaves[l]->prefix.size(); i++) pre[((size_t)l * R + j) * 32 + i] = leaves[l]->prefix[i];
    std::vector<Cost> costs((size_t)L * R);
    orc_rollout(O, pre.data(), (int64_t)L * R, seed, (uint64_t)rollouts_done, outs.data(), costs.data(), threads);
    rollouts_done += (i64)L * R;
    for (Node* lf : leaves) for (Node* x = lf; x; x = x->parent) { x->N -= 1; x->W += 1.0; }
    bool improved = false;
    auto consider = [&](const Cost& c, const u16* s) {
      if (c.status == 0 && (!have || Oracle::better(c, s, best, best_seq))) {
        best = c; memcpy(best_seq, s, 32 * sizeof(u16)); have = true; improved = true;
      }
    };
    // backup (reading R16): a leaf's R+1 rewards are summed in order (its own
    // state first, then rollouts 0..R-1), then added once to every node on its path
    for (int l = 0; l < L; l++) {
      double sum = -lcost[l].score;
      for (int j = 0; j < R; j++) sum = sum + (-costs[(size_t)l * R + j].score);
      for (Node* x = leaves[l]; x; x = x->parent) { x->N += R + 1; x->W += sum; }
      consider(lcost[l], &lpre[(size_t)l * 32]);
      for (int j = 0; j < R; j++) consider(costs[(size_t)l * R + j], &outs[((size_t)l * R + j) * 32]);
    }
    // reading R24: "any action sequence yielding the same sharded
    // model resolves to the same unique state, eliminating duplication by
    // construction" — with transpositions on, a selected leaf whose state (its
    // exactly evaluated key) another node already holds leaves the tree; leaves
    // are taken in selection order, so the first to reach a state keeps it
    if (transpositions) {
      std::vector<Node*> gone;
      for (int l = 0; l < L; l++) {
        if (lcost[l].status != 0) continue;
        auto it = holder.find(lcost[l].state_key);
        if (it == holder.end()) holder[lcost[l].state_key] = leaves[l];
        else if (it->second != leaves[l] && std::find(gone.begin(), gone.end(), leaves[l]) == gone.end())
          gone.push_back(leaves[l]);
      }
      for (Node* g : gone) {
        std::vector<Node*>& ch = g->parent->children;
        ch.erase(std::find(ch.begin(), ch.end(), g));
        delete g;
      }
    }
    evals += (i64)L * (R + 1);
    if (trace && rounds < trace_cap) trace[rounds] = best.score;
    rounds++;
    if (res->time_to_target_s < 0 && !std::isnan(target_score) && best.score <= target_score) {
      res->time_to_target_s = elapsed(); res->hit_target = 1;
    }
    if (improved) nonimprove = 0; else nonimprove++;
    if (nonimprove >= patience) break;
    if (max_evals > 0 && evals >= max_evals) break;
    if (time_limit_s > 0 && elapsed() >= time_limit_s) break;
    if (res->hit_target) break;
  }
  memcpy(res->best_seq, best_seq, sizeof best_seq);
  res->best = best;
  res->evals = evals;
  res->rounds = rounds;
  res->wall_s = elapsed();
  free_tree(root);
  return 0;
}

}  // extern "C"
