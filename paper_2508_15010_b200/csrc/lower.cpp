// toast_lower: the device-local program one action sequence implies (SURVEY
// §8(f) NEXT-1).  The sequence is materialised on the host (C9), every value
// gets its layout D (per dim, the mesh axes sharding it) and partial axes P
// (the axes sharding a reduction loop of its def op), and every use edge whose
// layout U differs, or whose value is partial, gets the collectives of C11 in
// front of the use, in the notation of Fig. 2c / Fig. 5b (P:336-344,
// P:796-810):
//   phase 1  per axis A (mesh order) held on a dim of D that U does not keep
//            there: first every all_gather (U holds A on no dim), then every
//            all_to_all (U holds A on another dim), an axis waiting while its
//            target dim would not divide; moves that block one another run
//            as one all_to_all listing them all — reading R20
//   phase 2  per partial axis A: reduce_scatter onto the dim U holds A on,
//            else all_reduce
//   phase 3  per axis U holds that the current layout lacks: a local slice
// with the payload the cost model charges (reading G12/G13).  Within one op a
// value used twice with the same U is resharded once (G26); every use of a
// partial value reduces it (G27).  Local extents divide exactly (C9 only
// shards divisible loops).
//
// Text format, one statement per line:
//   mesh <name>=<size> ...
//   %v = <op>[attrs](%a, ...) <dtype> [global dims] local[dims] layout[m0,...] partial[m]
//   %v.k = all_gather{axis=A,dim=i}(%v) ... bytes=<payload>
//   %v.k = all_to_all{axis=A,from=i,to=j}+{axis=B,from=j,to=i}(%v) ... bytes=<payload A>+<payload B>
//   return %a, ...
// m = bitmask over mesh axes (bit A = axis A of the mesh line).
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "toast_internal.h"

namespace toast {

namespace {

const char* kDtypeName[] = {"f32", "bf16", "f16", "i32", "f64", "i64"};

std::string dims_str(const std::vector<int64_t>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
  return s + "]";
}
std::string masks_str(const std::vector<uint32_t>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
  return s + "]";
}

}  // namespace

toast_status lower_program(const toast_analysis* a, const uint16_t* seq, std::string& out, std::string& err) {
  if (!a->graph) { err = "the analysis holds no program"; return TOAST_E_INVALID_ARG; }
  const toast_graph& g = *a->graph;
  const int n_axes = (int)g.axis_size.size();
  std::vector<uint8_t> mask((size_t)a->n_loops, 0);
  host_materialize(a, seq, mask.data());

  auto prod = [&](uint32_t m) {
    int64_t p = 1;
    for (int A = 0; A < n_axes; ++A) if ((m >> A) & 1) p *= g.axis_size[A];
    return p;
  };
  auto local_shape = [&](const std::vector<int64_t>& gs, const std::vector<uint32_t>& L) {
    std::vector<int64_t> ls(gs.size());
    for (size_t i = 0; i < gs.size(); ++i) ls[i] = gs[i] / prod(L[i]);
    return ls;
  };
  // layout D and partial axes P of the value defined by op t
  auto def_layout = [&](int32_t t, std::vector<uint32_t>& D, uint32_t& P) {
    const DOp& d = a->h_ops[t];
    D.assign(d.rank, 0);
    for (int i = 0; i < d.rank; ++i) D[i] = mask[d.loop_begin + ((d.res_roles >> (4 * i)) & 15)];
    P = 0;
    for (int r = 0; r < d.n_loops; ++r)
      if ((d.rmask >> r) & 1) P |= mask[d.loop_begin + r];
  };

  std::string s;
  s += "# device-local program lowered by libtoast (SURVEY 8(f) NEXT-1)\nmesh";
  for (int A = 0; A < n_axes; ++A) s += " " + g.axis_names[A] + "=" + std::to_string(g.axis_size[A]);
  s += "\n";
  std::vector<std::string> rets;
  std::vector<int> n_tmp(g.values.size(), 0);
  for (int32_t t = 0; t < (int32_t)g.ops.size(); ++t) {
    const GOp& op = g.ops[t];
    const DOp& dop = a->h_ops[t];
    // operands: reshard each use edge (deduplicated within the op)
    std::map<std::pair<int32_t, std::vector<uint32_t>>, std::string> done;
    std::vector<std::string> args;
    for (size_t k = 0; k < op.operands.size(); ++k) {
      const int32_t v = op.operands[k];
      const GValue& val = g.values[v];
      const int rank = (int)val.shape.size();
      const DUse& u = a->h_uses[dop.use_begin + k];
      std::vector<uint32_t> U(rank), D;
      for (int i = 0; i < rank; ++i) U[i] = mask[dop.loop_begin + ((u.use_roles >> (4 * i)) & 15)];
      uint32_t P;
      def_layout(val.def_op, D, P);
      const std::string src = "%" + val.name;
      auto key = std::make_pair(v, U);
      auto it = done.find(key);
      if (it != done.end()) { args.push_back(it->second); continue; }
      if (D == U && P == 0) { done[key] = src; args.push_back(src); continue; }
      std::vector<uint32_t> cur = D;
      uint32_t part = P;
      uint64_t size = (uint64_t)val.elem_bytes;
      for (int64_t e : local_shape(val.shape, D)) size *= (uint64_t)e;
      std::string prev = src;
      auto emit_spec = [&](const std::string& coll, const std::string& bytes) {
        const std::string name = "%" + val.name + "." + std::to_string(++n_tmp[v]);
        s += name + " = " + coll + "(" + prev + ") " + kDtypeName[val.dtype_code] + " " + dims_str(val.shape) +
             " local" + dims_str(local_shape(val.shape, cur)) + " layout" + masks_str(cur) + " partial[" +
             std::to_string(part) + "] bytes=" + bytes + "\n";
        prev = name;
      };
      auto emit = [&](const std::string& coll, uint64_t bytes, bool has_bytes) {
        const std::string name = "%" + val.name + "." + std::to_string(++n_tmp[v]);
        s += name + " = " + coll + "(" + prev + ") " + kDtypeName[val.dtype_code] + " " + dims_str(val.shape) +
             " local" + dims_str(local_shape(val.shape, cur)) + " layout" + masks_str(cur) + " partial[" +
             std::to_string(part) + "]";
        if (has_bytes) s += " bytes=" + std::to_string(bytes);
        s += "\n";
        prev = name;
      };
      // phase 1 (reading R20): 1a all_gather the axes U holds on no dim, then
      // 1b all_to_all the axes U holds on another dim (ascending mesh axis,
      // then dim) — every intermediate layout stays divisible
      // 1a: all_gather every axis of D that U holds on no dim
      struct Move { int A, i, j; };
      std::vector<Move> moves;
      for (int A = 0; A < n_axes; ++A) {
        const uint32_t bit = 1u << A;
        for (int i = 0; i < rank; ++i) {
          if (!(cur[i] & bit) || (U[i] & bit)) continue;
          int j_other = -1;
          for (int j = 0; j < rank; ++j) if (j != i && (U[j] & bit)) j_other = j;
          if (j_other >= 0) { moves.push_back({A, i, j_other}); continue; }
          const uint64_t pay = size;
          cur[i] &= ~bit;
          size *= (uint64_t)g.axis_size[A];
          emit("all_gather{axis=" + std::to_string(A) + ",dim=" + std::to_string(i) + "}", pay, true);
        }
      }
      // 1b: all_to_all every axis U holds on another dim.  An all_to_all keeps
      // the local size, so its payload (and the cost) does not depend on the
      // order; the moves run in ascending axis order except that an axis waits
      // while its target dim would not divide (it still holds an axis that is
      // about to leave), so every intermediate layout stays divisible.  Moves
      // that block one another (a cycle, e.g. two axes swapping dims whose
      // extents cannot hold both) run as ONE all_to_all over the product of
      // their axes: one statement listing every move, each axis charged as
      // its own all_to_all (reading R20).
      while (!moves.empty()) {
        size_t pick = moves.size();
        for (size_t q = 0; q < moves.size() && pick == moves.size(); ++q) {
          const Move& m = moves[q];
          if (val.shape[m.j] % (prod(cur[m.j]) * g.axis_size[m.A]) == 0) pick = q;
        }
        std::vector<Move> step;
        if (pick == moves.size()) {
          step.swap(moves);
        } else {
          step.push_back(moves[pick]);
          moves.erase(moves.begin() + (long)pick);
        }
        std::string spec, bytes;
        for (const Move& m : step) {
          const uint32_t bit = 1u << m.A;
          cur[m.i] &= ~bit;
          cur[m.j] |= bit;
          spec += std::string(spec.empty() ? "" : "+") + "{axis=" + std::to_string(m.A) + ",from=" + std::to_string(m.i) +
                  ",to=" + std::to_string(m.j) + "}";
          bytes += (bytes.empty() ? "" : "+") + std::to_string(size);
        }
        emit_spec("all_to_all" + spec, bytes);
      }
      // phase 2: reduce_scatter / all_reduce of the partial axes
      for (int A = 0; A < n_axes; ++A) {
        const uint32_t bit = 1u << A;
        if (!(part & bit)) continue;
        int j_u = -1;
        for (int j = 0; j < rank; ++j) if (U[j] & bit) j_u = j;
        part &= ~bit;
        if (j_u >= 0) {
          size /= (uint64_t)g.axis_size[A];
          cur[j_u] |= bit;
          emit("reduce_scatter{axis=" + std::to_string(A) + ",dim=" + std::to_string(j_u) + "}", size, true);
        } else {
          emit("all_reduce{axis=" + std::to_string(A) + "}", size, true);
        }
      }
      // phase 3: free local slices
      for (int A = 0; A < n_axes; ++A) {
        const uint32_t bit = 1u << A;
        for (int j = 0; j < rank; ++j) {
          if (!(U[j] & bit) || (cur[j] & bit)) continue;
          cur[j] |= bit;
          size /= (uint64_t)g.axis_size[A];
          emit("slice{axis=" + std::to_string(A) + ",dim=" + std::to_string(j) + "}", 0, false);
        }
      }
      if (cur != U) { err = "internal: resharding did not reach the use layout"; return TOAST_E_INVALID_ARG; }
      done[key] = prev;
      args.push_back(prev);
    }
    if (op.kind == OK_RET) { rets.push_back(args[0]); continue; }
    const GValue& res = g.values[op.result];
    std::vector<uint32_t> D;
    uint32_t P;
    def_layout(t, D, P);
    s += "%" + res.name + " = " + op.name;
    if (!op.attr_text.empty()) s += "[" + op.attr_text + "]";
    if (op.kind != OK_PARAM) {
      s += "(";
      for (size_t k = 0; k < args.size(); ++k) s += (k ? ", " : "") + args[k];
      s += ")";
    }
    s += std::string(" ") + kDtypeName[res.dtype_code] + " " + dims_str(res.shape) + " local" +
         dims_str(local_shape(res.shape, D)) + " layout" + masks_str(D) + " partial[" + std::to_string(P) + "]\n";
  }
  s += "return";
  for (size_t i = 0; i < rets.size(); ++i) s += (i ? ", " : " ") + rets[i];
  s += "\n";
  out.swap(s);
  return TOAST_OK;
}

}  // namespace toast
