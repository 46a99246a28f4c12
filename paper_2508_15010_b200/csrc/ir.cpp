// Text-IR front end of libtoast.  Grammar (SPEC S:92-104,
// extended):
//   module := 'def' ID '(' [param {',' param}] ')' '{' {stmt} 'return' ID {',' ID} '}'
//   param  := ID ':' DTYPE '[' [INT {',' INT}] ']'
//   stmt   := ID '=' ID ['[' attrs ']'] '(' [ID {',' ID}] ')'
//   attrs  := items separated by ',' and ';' (';' starts a new group)
// Shapes of bindings are inferred and checked here; errors carry line:col or
// the binding's name.
#include <cctype>
#include <cstdlib>
#include <cstring>
#include <unordered_map>

#include "toast_internal.h"

namespace toast {
namespace {

struct Cursor {
  const char* p;
  const char* end;
  int line = 1;
  const char* line_start;
  std::string* err;

  void skip() {
    while (p < end) {
      if (*p == '\n') { ++line; ++p; line_start = p; continue; }
      if (*p == ' ' || *p == '\t' || *p == '\r') { ++p; continue; }
      if (*p == '#') { while (p < end && *p != '\n') ++p; continue; }
      break;
    }
  }
  std::string loc() {
    return std::to_string(line) + ":" + std::to_string((int)(p - line_start) + 1) + ": ";
  }
  bool peek(char c) { skip(); return p < end && *p == c; }
  bool accept(char c) { if (peek(c)) { ++p; return true; } return false; }
  bool expect(char c) {
    if (accept(c)) return true;
    *err = loc() + "expected '" + std::string(1, c) + "'";
    return false;
  }
  bool ident(std::string& out) {
    skip();
    const char* s = p;
    if (p < end && (isalpha((unsigned char)*p) || *p == '_')) {
      while (p < end && (isalnum((unsigned char)*p) || *p == '_' || *p == '.')) ++p;
      out.assign(s, p);
      return true;
    }
    *err = loc() + "expected identifier";
    return false;
  }
  // a number or identifier token inside attribute brackets
  bool atom(std::string& out) {
    skip();
    const char* s = p;
    if (p < end && (isalnum((unsigned char)*p) || *p == '_' || *p == '-' || *p == '+' || *p == '.')) {
      ++p;
      while (p < end) {
        char c = *p;
        if (isalnum((unsigned char)c) || c == '_' || c == '.') { ++p; continue; }
        if ((c == '-' || c == '+') && (p[-1] == 'e' || p[-1] == 'E')) { ++p; continue; }
        break;
      }
      out.assign(s, p);
      return true;
    }
    *err = loc() + "bad attribute";
    return false;
  }
};

struct DType { const char* name; int bytes; };
const DType kDTypes[] = {{"f32", 4}, {"bf16", 2}, {"f16", 2}, {"i32", 4}, {"f64", 8}, {"i64", 8}};

int dtype_lookup(const std::string& s) {
  for (int i = 0; i < 6; ++i) if (s == kDTypes[i].name) return i;
  return -1;
}

bool is_unary_name(const std::string& k) {
  static const char* names[] = {"relu", "neg", "exp", "log", "recip", "rsqrt", "sqrt", "tanh", "gelu", "silu",
                                "sigmoid", "square", "abs", "sign", "ones_like", "scale", "add_s", "pow_s",
                                "convert", "stop_gradient", "cos", "sin"};
  for (const char* n : names) if (k == n) return true;
  return k.size() > 2 && k.compare(0, 2, "d_") == 0;   // derivative of an elementwise function
}
bool is_binary_name(const std::string& k) {
  return k == "add" || k == "sub" || k == "mul" || k == "div" || k == "max" || k == "min" || k == "pow";
}

bool parse_int(const std::string& s, int64_t& v) {
  if (s.empty()) return false;
  char* e = nullptr;
  v = strtoll(s.c_str(), &e, 10);
  return e && *e == 0;
}

// infer result (shape, dtype) and the integer attributes of one binding
toast_status infer(toast_graph* g, GOp& op, const std::vector<std::vector<std::string>>& attrs, GValue& res,
                   std::string& err) {
  auto fail = [&](const std::string& m) { err = "binding '" + op.binding + "': " + m; return TOAST_E_SHAPE; };
  auto V = [&](int k) -> GValue& { return g->values[op.operands[k]]; };
  auto nops = [&](size_t n) { return op.operands.size() == n; };
  auto ints = [&](size_t grp, std::vector<int64_t>& out) {
    out.clear();
    if (grp >= attrs.size()) return true;
    for (auto& s : attrs[grp]) { int64_t v; if (!parse_int(s, v)) return false; out.push_back(v); }
    return true;
  };
  const std::string& k = op.name;
  res.dtype_code = op.operands.empty() ? 0 : V(0).dtype_code;
  if (is_unary_name(k)) {
    op.kind = OK_UNARY;
    if (!nops(1)) return fail("expected 1 operand");
    res.shape = V(0).shape;
    if (k == "convert") {
      int dc = attrs.empty() || attrs[0].empty() ? -1 : dtype_lookup(attrs[0][0]);
      if (dc < 0) return fail("convert needs a dtype");
      res.dtype_code = dc;
    }
  } else if (is_binary_name(k)) {
    op.kind = OK_BINARY;
    if (!nops(2)) return fail("expected 2 operands");
    if (V(0).shape != V(1).shape) return fail("elementwise operands differ in shape");
    res.shape = V(0).shape;
  } else if (k == "transpose") {
    op.kind = OK_TRANSPOSE;
    if (!nops(1) || !ints(0, op.ia)) return fail("transpose[perm]");
    const auto& s = V(0).shape;
    if (op.ia.size() != s.size()) return fail("bad permutation");
    std::vector<char> seen(s.size(), 0);
    for (int64_t x : op.ia) {
      if (x < 0 || x >= (int64_t)s.size() || seen[x]) return fail("bad permutation");
      seen[x] = 1;
      res.shape.push_back(s[x]);
    }
  } else if (k == "reduce") {
    op.kind = OK_REDUCE;
    if (!nops(1) || attrs.size() != 1 || attrs[0].size() < 2) return fail("reduce[dims..., comb]");
    const std::string& comb = attrs[0].back();
    if (comb != "add" && comb != "mul" && comb != "max" && comb != "min") return fail("bad combiner");
    const auto& s = V(0).shape;
    std::vector<char> red(s.size(), 0);
    for (size_t i = 0; i + 1 < attrs[0].size(); ++i) {
      int64_t d;
      if (!parse_int(attrs[0][i], d) || d < 0 || d >= (int64_t)s.size() || red[d]) return fail("bad reduce dim");
      red[d] = 1;
    }
    op.ia.clear();
    for (size_t i = 0; i < s.size(); ++i) { op.ia.push_back(red[i]); if (!red[i]) res.shape.push_back(s[i]); }
  } else if (k == "broadcast") {
    op.kind = OK_BROADCAST;
    if (!nops(1) || !ints(0, op.ia) || op.ia.size() != 2) return fail("broadcast[l, e]");
    const auto& s = V(0).shape;
    if (op.ia[0] < 0 || op.ia[0] > (int64_t)s.size() || op.ia[1] < 1) return fail("broadcast[l, e]");
    res.shape = s;
    res.shape.insert(res.shape.begin() + op.ia[0], op.ia[1]);
  } else if (k == "matmul") {
    op.kind = OK_MATMUL;
    if (!nops(2)) return fail("expected 2 operands");
    const auto& a = V(0).shape; const auto& b = V(1).shape;
    if (a.size() != 2 || b.size() != 2 || a[1] != b[0]) return fail("matmul contraction extents differ");
    res.shape = {a[0], b[1]};
  } else if (k == "dot_general") {
    op.kind = OK_DOT;
    std::vector<int64_t> lb, rb, lc, rc;
    if (!nops(2) || attrs.size() != 4 || !ints(0, lb) || !ints(1, rb) || !ints(2, lc) || !ints(3, rc))
      return fail("dot_general[lb;rb;lc;rc]");
    const auto& a = V(0).shape; const auto& b = V(1).shape;
    if (lb.size() != rb.size() || lc.size() != rc.size()) return fail("dot_general dims");
    std::vector<char> ua(a.size(), 0), ub(b.size(), 0);
    auto mark = [&](const std::vector<int64_t>& x, const std::vector<int64_t>& y) {
      for (size_t t = 0; t < x.size(); ++t) {
        if (x[t] < 0 || x[t] >= (int64_t)a.size() || y[t] < 0 || y[t] >= (int64_t)b.size()) return false;
        if (ua[x[t]] || ub[y[t]] || a[x[t]] != b[y[t]]) return false;
        ua[x[t]] = ub[y[t]] = 1;
      }
      return true;
    };
    if (!mark(lb, rb)) return fail("dot_general batch dims");
    if (!mark(lc, rc)) return fail("dot_general contracting dims");
    // ia = [nb, nc, lb..., rb..., lc..., rc...]
    op.ia = {(int64_t)lb.size(), (int64_t)lc.size()};
    op.ia.insert(op.ia.end(), lb.begin(), lb.end());
    op.ia.insert(op.ia.end(), rb.begin(), rb.end());
    op.ia.insert(op.ia.end(), lc.begin(), lc.end());
    op.ia.insert(op.ia.end(), rc.begin(), rc.end());
    for (int64_t x : lb) res.shape.push_back(a[x]);
    for (size_t i = 0; i < a.size(); ++i) if (!ua[i]) res.shape.push_back(a[i]);
    for (size_t i = 0; i < b.size(); ++i) if (!ub[i]) res.shape.push_back(b[i]);
  } else if (k == "conv2d" || k == "conv2d_bwd_input") {
    op.kind = k == "conv2d" ? OK_CONV : OK_CONV_BI;
    if (!nops(2)) return fail("expected 2 operands");
    const auto& x = V(0).shape; const auto& w = V(1).shape;
    if (x.size() != 4 || w.size() != 4) return fail("conv shapes");
    if (op.kind == OK_CONV) {
      if (x[3] != w[2]) return fail("conv2d shapes");
      res.shape = {x[0], x[1], x[2], w[3]};
    } else {
      if (x[3] != w[3]) return fail("conv2d_bwd_input shapes");
      res.shape = {x[0], x[1], x[2], w[2]};
    }
  } else if (k == "conv2d_bwd_filter") {
    op.kind = OK_CONV_BF;
    if (!nops(2) || !ints(0, op.ia) || op.ia.size() != 2) return fail("conv2d_bwd_filter[KH,KW]");
    const auto& x = V(0).shape; const auto& d = V(1).shape;
    if (x.size() != 4 || d.size() != 4 || x[0] != d[0] || x[1] != d[1] || x[2] != d[2] || op.ia[0] < 1 || op.ia[1] < 1)
      return fail("conv2d_bwd_filter shapes");
    res.shape = {op.ia[0], op.ia[1], x[3], d[3]};
  } else if (k == "resample") {
    op.kind = OK_RESAMPLE;
    int64_t f;
    if (!nops(1) || attrs.size() != 1 || attrs[0].size() != 2 || !parse_int(attrs[0][1], f) || f < 1)
      return fail("resample[up|down,f]");
    const auto& x = V(0).shape;
    if (x.size() != 4) return fail("resample needs rank 4");
    res.shape = x;
    if (attrs[0][0] == "up") { res.shape[1] *= f; res.shape[2] *= f; }
    else if (attrs[0][0] == "down") {
      if (x[1] % f || x[2] % f) return fail("resample factor does not divide");
      res.shape[1] /= f; res.shape[2] /= f;
    } else return fail("resample mode");
  } else if (k == "concat") {
    op.kind = OK_CONCAT;
    if (op.operands.empty() || !ints(0, op.ia) || op.ia.size() != 1) return fail("concat[d]");
    const auto& s0 = V(0).shape;
    int64_t d = op.ia[0];
    if (d < 0 || d >= (int64_t)s0.size()) return fail("concat[d]");
    res.shape = s0;
    res.shape[d] = 0;
    for (size_t j = 0; j < op.operands.size(); ++j) {
      const auto& s = V((int)j).shape;
      if (s.size() != s0.size()) return fail("concat rank");
      for (size_t i = 0; i < s.size(); ++i) if ((int64_t)i != d && s[i] != s0[i]) return fail("concat extents");
      res.shape[d] += s[d];
    }
  } else if (k == "slice" || k == "pad") {
    op.kind = k == "slice" ? OK_SLICE : OK_PAD;
    if (!nops(1) || !ints(0, op.ia) || op.ia.size() != 3) return fail(k + "[d,a,b]");
    const auto& s = V(0).shape;
    int64_t d = op.ia[0];
    if (d < 0 || d >= (int64_t)s.size()) return fail("bad dim");
    res.shape = s;
    if (op.kind == OK_SLICE) {
      if (op.ia[1] < 0 || op.ia[2] < 1 || op.ia[1] + op.ia[2] > s[d]) return fail("slice[d,start,len]");
      res.shape[d] = op.ia[2];
    } else {
      if (op.ia[1] < 0 || op.ia[2] < 0) return fail("pad[d,lo,hi]");
      res.shape[d] += op.ia[1] + op.ia[2];
    }
  } else if (k == "gather") {
    op.kind = OK_GATHER;
    if (!nops(2)) return fail("expected 2 operands");
    const auto& t = V(0).shape; const auto& ix = V(1).shape;
    if (t.size() != 2 || ix.empty()) return fail("gather(tbl[n,f], idx[e...])");
    res.shape = ix;
    res.shape.push_back(t[1]);
  } else if (k == "segment_sum") {
    op.kind = OK_SEGSUM;
    if (!nops(2) || !ints(0, op.ia) || op.ia.size() != 1 || op.ia[0] < 1) return fail("segment_sum[n](dat, idx)");
    const auto& d = V(0).shape; const auto& ix = V(1).shape;
    if (ix.empty() || d.size() != ix.size() + 1) return fail("segment_sum ranks");
    for (size_t i = 0; i < ix.size(); ++i) if (d[i] != ix[i]) return fail("segment_sum extents");
    res.shape = {op.ia[0], d.back()};
  } else {
    err = "binding '" + op.binding + "': unknown op '" + k + "'";
    return TOAST_E_PARSE;
  }
  if ((int)res.shape.size() > MAX_RANK) return fail("rank > 8");
  res.elem_bytes = kDTypes[res.dtype_code].bytes;
  return TOAST_OK;
}

}  // namespace

toast_status parse_ir(const char* text, size_t len, toast_graph* g, std::string& err) {
  Cursor c{text, text + len, 1, text, &err};
  std::unordered_map<std::string, int32_t> env;
  std::string w;
  if (!c.ident(w) || w != "def") { err = c.loc() + "expected 'def'"; return TOAST_E_PARSE; }
  if (!c.ident(w)) return TOAST_E_PARSE;
  if (!c.expect('(')) return TOAST_E_PARSE;
  if (!c.peek(')')) {
    do {
      c.skip();
      std::string at = c.loc();
      std::string name, dt;
      if (!c.ident(name) || !c.expect(':') || !c.ident(dt)) return TOAST_E_PARSE;
      int dc = dtype_lookup(dt);
      if (dc < 0) { err = c.loc() + "unknown dtype '" + dt + "'"; return TOAST_E_PARSE; }
      if (!c.expect('[')) return TOAST_E_PARSE;
      GValue v;
      v.dtype_code = dc;
      v.elem_bytes = kDTypes[dc].bytes;
      if (!c.peek(']')) {
        do {
          std::string tok;
          int64_t e;
          if (!c.atom(tok) || !parse_int(tok, e)) { err = c.loc() + "expected extent"; return TOAST_E_PARSE; }
          if (e < 1) { err = "parameter '" + name + "': extent must be >= 1"; return TOAST_E_SHAPE; }
          v.shape.push_back(e);
        } while (c.accept(','));
      }
      if (!c.expect(']')) return TOAST_E_PARSE;
      if ((int)v.shape.size() > MAX_RANK) { err = "parameter '" + name + "': rank > 8"; return TOAST_E_SHAPE; }
      if (env.count(name)) { err = at + "duplicate binding '" + name + "'"; return TOAST_E_DUPLICATE; }
      v.def_op = (int32_t)g->ops.size();
      v.name = name;
      env[name] = (int32_t)g->values.size();
      GOp op;
      op.kind = OK_PARAM;
      op.name = "param";
      op.binding = name;
      op.result = (int32_t)g->values.size();
      g->values.push_back(v);
      g->ops.push_back(op);
      g->n_params++;
    } while (c.accept(','));
  }
  if (!c.expect(')') || !c.expect('{')) return TOAST_E_PARSE;
  std::vector<int32_t> rets;
  while (true) {
    c.skip();
    if (c.p >= c.end) { err = c.loc() + "unexpected end of input"; return TOAST_E_PARSE; }
    std::string at = c.loc();
    std::string name;
    if (!c.ident(name)) return TOAST_E_PARSE;
    if (name == "return") {
      do {
        c.skip();
        std::string rl = c.loc();
        std::string r;
        if (!c.ident(r)) return TOAST_E_PARSE;
        auto it = env.find(r);
        if (it == env.end()) { err = rl + "use of undefined '" + r + "'"; return TOAST_E_UNDEFINED; }
        rets.push_back(it->second);
      } while (c.accept(','));
      if (!c.expect('}')) return TOAST_E_PARSE;
      break;
    }
    if (!c.expect('=')) return TOAST_E_PARSE;
    GOp op;
    op.binding = name;
    if (!c.ident(op.name)) return TOAST_E_PARSE;
    std::vector<std::vector<std::string>> attrs;
    if (c.accept('[')) {
      attrs.emplace_back();
      while (!c.peek(']')) {
        if (c.p >= c.end) { err = c.loc() + "unterminated attributes"; return TOAST_E_PARSE; }
        if (c.accept(';')) { attrs.emplace_back(); continue; }
        if (c.accept(',')) continue;
        std::string tok;
        if (!c.atom(tok)) return TOAST_E_PARSE;
        attrs.back().push_back(tok);
      }
      c.accept(']');
      for (size_t gi = 0; gi < attrs.size(); ++gi) {
        if (gi) op.attr_text += ';';
        for (size_t ai = 0; ai < attrs[gi].size(); ++ai) op.attr_text += (ai ? "," : "") + attrs[gi][ai];
      }
    }
    if (!c.expect('(')) return TOAST_E_PARSE;
    if (!c.peek(')')) {
      do {
        c.skip();
        std::string al = c.loc();
        std::string a;
        if (!c.ident(a)) return TOAST_E_PARSE;
        auto it = env.find(a);
        if (it == env.end()) { err = al + "use of undefined '" + a + "'"; return TOAST_E_UNDEFINED; }
        op.operands.push_back(it->second);
      } while (c.accept(','));
    }
    if (!c.expect(')')) return TOAST_E_PARSE;
    if (env.count(name)) { err = at + "duplicate binding '" + name + "'"; return TOAST_E_DUPLICATE; }
    GValue res;
    toast_status st = infer(g, op, attrs, res, err);
    if (st != TOAST_OK) return st;
    res.def_op = (int32_t)g->ops.size();
    res.name = name;
    op.result = (int32_t)g->values.size();
    env[name] = op.result;
    g->values.push_back(res);
    g->ops.push_back(op);
  }
  c.skip();
  if (c.p != c.end) { err = c.loc() + "trailing input"; return TOAST_E_PARSE; }
  for (int32_t v : rets) {
    GOp op;
    op.kind = OK_RET;
    op.name = "ret";
    op.operands = {v};
    op.binding = "return " + g->values[v].name;
    g->ops.push_back(op);
  }
  return TOAST_OK;
}

}  // namespace toast
