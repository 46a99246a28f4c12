// extern "C" entry points of libtoast (include/toast.h).  Argument checks,
// error strings and host/device pointer dispatch; the work happens in
// ir.cpp (parse), analysis.cpp (H0), kernels.cu (H1-H8) and search.cpp.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <set>
#include <string>

#include "toast_internal.h"

namespace toast {
toast_status search_begin(const toast_analysis* a, const toast_search_opts* o, int32_t rank, int32_t world,
                          toast_search_state** out, std::string& err);
toast_status search_round(toast_search_state* s, void* export_buf, std::string& err);
toast_status search_import(toast_search_state* s, const void* gathered, int32_t* stop, std::string& err);
toast_status search_round_dev(toast_search_state* s, void* export_dev, void* stream, std::string& err);
toast_status search_import_dev(toast_search_state* s, const void* gathered_dev, int32_t* stop, void* stream,
                               std::string& err);
void search_result(const toast_search_state* s, toast_search_result* out);
size_t search_export_bytes(const toast_analysis* a);
int32_t search_root_stats(const toast_search_state* s, toast_root_stat* out, int32_t cap);
void search_free(toast_search_state* s);
}  // namespace toast

namespace {
thread_local std::string g_err;

toast_status fail(toast_status st, const std::string& msg) {
  g_err = msg;
  return st;
}
toast_status ret(toast_status st, const std::string& msg) {
  g_err = st == TOAST_OK ? std::string() : msg;
  return st;
}
bool has_device(const toast_analysis* a) { return a && a->device >= 0 && a->dt.points != nullptr; }
}  // namespace

extern "C" {

const char* toast_last_error(void) { return g_err.c_str(); }

toast_status toast_load_graph(const char* ir_text, size_t len, const toast_axis* axes, int32_t n_axes,
                              const toast_machine* m, int32_t cuda_device, toast_graph** out) {
  if (!out) return fail(TOAST_E_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!ir_text || !axes || !m) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  if (n_axes < 1 || n_axes > 4) return fail(TOAST_E_MESH, "the mesh must have 1 to 4 axes");
  std::set<std::string> names;
  for (int i = 0; i < n_axes; ++i) {
    if (!axes[i].name) return fail(TOAST_E_MESH, "axis without a name");
    if (!names.insert(axes[i].name).second) return fail(TOAST_E_MESH, std::string("duplicate axis '") + axes[i].name + "'");
    if (axes[i].size < 2) return fail(TOAST_E_MESH, std::string("axis '") + axes[i].name + "' has size < 2");
    if (!(axes[i].bytes_per_sec > 0)) return fail(TOAST_E_MESH, std::string("axis '") + axes[i].name + "' has bandwidth <= 0");
  }
  if (!(m->flops_per_sec > 0) || !(m->penalty_c >= 0)) return fail(TOAST_E_MACHINE, "flops_per_sec must be > 0, penalty_c >= 0");
  toast_graph* g = new (std::nothrow) toast_graph();
  if (!g) return fail(TOAST_E_OOM, "out of host memory");
  try {
    std::string err;
    toast_status st = toast::parse_ir(ir_text, len, g, err);
    if (st != TOAST_OK) { delete g; return fail(st, err); }
  } catch (std::bad_alloc&) {
    delete g;
    return fail(TOAST_E_OOM, "out of host memory");
  }
  for (int i = 0; i < n_axes; ++i) {
    g->axis_names.push_back(axes[i].name);
    g->axis_size.push_back(axes[i].size);
    g->axis_bw.push_back(axes[i].bytes_per_sec);
  }
  g->machine = *m;
  g->device = cuda_device;
  *out = g;
  return ret(TOAST_OK, "");
}

toast_status toast_nda(const toast_graph* g, const toast_nda_opts* o, toast_analysis** out) {
  if (!out) return fail(TOAST_E_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!g || !o) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  if (o->min_unique_dims < 0 || o->max_depth < 1 || o->max_depth > 32)
    return fail(TOAST_E_INVALID_ARG, "min_unique_dims must be >= 0 and max_depth in [1, 32]");
  if (o->cost_model != TOAST_COST_SUM && o->cost_model != TOAST_COST_CRITICAL_PATH)
    return fail(TOAST_E_INVALID_ARG, "cost_model must be TOAST_COST_SUM or TOAST_COST_CRITICAL_PATH");
  if (o->conflict_grouping != TOAST_GROUP_COMPAT && o->conflict_grouping != TOAST_GROUP_CONTRACTION)
    return fail(TOAST_E_INVALID_ARG, "conflict_grouping must be TOAST_GROUP_COMPAT or TOAST_GROUP_CONTRACTION");
  if (o->dedup < 0 || o->dedup > 2) return fail(TOAST_E_INVALID_ARG, "dedup must be 0, 1 or 2");
  toast_analysis* a = new (std::nothrow) toast_analysis();
  if (!a) return fail(TOAST_E_OOM, "out of host memory");
  std::string err;
  try {
    toast_status st = toast::build_analysis(g, o, a, err);
    if (st != TOAST_OK) { delete a; return fail(st, err); }
    a->device = g->device;
    a->graph = std::make_shared<const toast_graph>(*g);
    if (a->device >= 0) {
      st = toast::upload_tables(a, err);
      if (st == TOAST_OK) st = toast::autotune_k(a, err);
      if (st != TOAST_OK) { toast::free_tables(a); delete a; return fail(st, err); }
    }
    // (after the autotune, which times the one-kernel path); 2 = on for the critical path only
    a->dedup = o->dedup == 2 ? (o->cost_model == TOAST_COST_CRITICAL_PATH ? 1 : 0) : o->dedup;
  } catch (std::bad_alloc&) {
    delete a;
    return fail(TOAST_E_OOM, "out of host memory");
  }
  *out = a;
  return ret(TOAST_OK, "");
}

toast_status toast_num_actions(const toast_analysis* a, int32_t* n) {
  if (!a || !n) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  *n = (int32_t)a->actions.size();
  return ret(TOAST_OK, "");
}

toast_status toast_query_actions(const toast_analysis* a, toast_action_info* out, int32_t cap, int32_t* n) {
  if (!a || !n || (cap > 0 && !out)) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  *n = (int32_t)a->actions.size();
  for (int32_t i = 0; i < cap && i < *n; ++i) out[i] = a->actions[i];
  return ret(TOAST_OK, "");
}

toast_status toast_query_baseline(const toast_analysis* a, toast_cost* out) {
  if (!a || !out) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  *out = a->baseline;
  return ret(TOAST_OK, "");
}

toast_status toast_preferred_batch(const toast_analysis* a, int64_t* n) {
  if (!a || !n) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  if (!has_device(a)) return fail(TOAST_E_CUDA, "the analysis has no device tables");
  const int i = a->k_throughput >= 8 ? 3 : a->k_throughput >= 4 ? 2 : a->k_throughput >= 2 ? 1 : 0;
  *n = (int64_t)std::min(a->occ_eval[i], a->occ_roll[i]) * a->n_sms * 32;
  return ret(TOAST_OK, "");
}

toast_status toast_dump_analysis(const toast_analysis* a, char* buf, size_t cap, size_t* needed) {
  if (!a || !needed) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  std::string s = toast::dump_json(a);
  *needed = s.size() + 1;
  if (buf && cap >= *needed) memcpy(buf, s.c_str(), s.size() + 1);
  return ret(TOAST_OK, "");
}

toast_status toast_eval_batch(const toast_analysis* a, const uint16_t* seqs, int64_t n, toast_cost* out,
                              void* cuda_stream) {
  if (!a || n < 0 || (n > 0 && (!seqs || !out))) return fail(TOAST_E_INVALID_ARG, "bad argument");
  if (!has_device(a)) return fail(TOAST_E_CUDA, "the analysis has no device tables (cuda_device = -1 or no GPU)");
  if (n == 0) return ret(TOAST_OK, "");
  std::string err;
  cudaSetDevice(a->device);
  bool dev_in = toast::is_device_pointer(seqs), dev_out = toast::is_device_pointer(out);
  if (dev_in != dev_out) return fail(TOAST_E_INVALID_ARG, "seqs and out must both be host or both be device memory");
  toast_status st = dev_in ? toast::launch_eval(a, seqs, n, out, cuda_stream, err)
                           : toast::run_host_buffers(const_cast<toast_analysis*>(a), false, seqs, n, 0, 0, nullptr, out,
                                                     cuda_stream, err);
  return ret(st, err);
}

toast_status toast_rollout_batch(const toast_analysis* a, const uint16_t* prefixes, int64_t n, uint64_t seed,
                                 uint64_t id_base, uint16_t* out_seqs, toast_cost* out, void* cuda_stream) {
  if (!a || n < 0 || (n > 0 && (!prefixes || !out || !out_seqs))) return fail(TOAST_E_INVALID_ARG, "bad argument");
  if (!has_device(a)) return fail(TOAST_E_CUDA, "the analysis has no device tables (cuda_device = -1 or no GPU)");
  if (n == 0) return ret(TOAST_OK, "");
  std::string err;
  cudaSetDevice(a->device);
  bool d1 = toast::is_device_pointer(prefixes), d2 = toast::is_device_pointer(out_seqs), d3 = toast::is_device_pointer(out);
  if (d1 != d2 || d1 != d3) return fail(TOAST_E_INVALID_ARG, "buffers must all be host or all be device memory");
  toast_status st = d1 ? toast::launch_rollout(a, prefixes, n, seed, id_base, out_seqs, out, cuda_stream, err, 1)
                       : toast::run_host_buffers(const_cast<toast_analysis*>(a), true, prefixes, n, seed, id_base,
                                                 out_seqs, out, cuda_stream, err);
  return ret(st, err);
}

toast_status toast_eval_scores(const toast_analysis* a, const uint16_t* seqs, int64_t n, toast_score* out,
                               void* cuda_stream) {
  if (!a || n < 0 || (n > 0 && (!seqs || !out))) return fail(TOAST_E_INVALID_ARG, "bad argument");
  if (!has_device(a)) return fail(TOAST_E_CUDA, "the analysis has no device tables (cuda_device = -1 or no GPU)");
  if (n == 0) return ret(TOAST_OK, "");
  std::string err;
  cudaSetDevice(a->device);
  bool dev_in = toast::is_device_pointer(seqs), dev_out = toast::is_device_pointer(out);
  if (dev_in != dev_out) return fail(TOAST_E_INVALID_ARG, "seqs and out must both be host or both be device memory");
  toast_status st = dev_in ? toast::launch_eval(a, seqs, n, out, cuda_stream, err, true)
                           : toast::run_host_buffers(const_cast<toast_analysis*>(a), false, seqs, n, 0, 0, nullptr, out,
                                                     cuda_stream, err, true);
  return ret(st, err);
}

toast_status toast_rollout_scores(const toast_analysis* a, const uint16_t* prefixes, int64_t n, uint64_t seed,
                                  uint64_t id_base, uint16_t* out_seqs, toast_score* out, void* cuda_stream) {
  if (!a || n < 0 || (n > 0 && (!prefixes || !out || !out_seqs))) return fail(TOAST_E_INVALID_ARG, "bad argument");
  if (!has_device(a)) return fail(TOAST_E_CUDA, "the analysis has no device tables (cuda_device = -1 or no GPU)");
  if (n == 0) return ret(TOAST_OK, "");
  std::string err;
  cudaSetDevice(a->device);
  bool d1 = toast::is_device_pointer(prefixes), d2 = toast::is_device_pointer(out_seqs), d3 = toast::is_device_pointer(out);
  if (d1 != d2 || d1 != d3) return fail(TOAST_E_INVALID_ARG, "buffers must all be host or all be device memory");
  toast_status st = d1 ? toast::launch_rollout(a, prefixes, n, seed, id_base, out_seqs, out, cuda_stream, err, 1, true)
                       : toast::run_host_buffers(const_cast<toast_analysis*>(a), true, prefixes, n, seed, id_base,
                                                 out_seqs, out, cuda_stream, err, true);
  return ret(st, err);
}

toast_status toast_materialize(const toast_analysis* a, const uint16_t seq[32], uint8_t* masks, int64_t cap, int64_t* n) {
  if (!a || !seq || !n) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  *n = a->n_loops;
  if (masks && cap >= a->n_loops) {
    if (const uint32_t st = toast::host_validate(a, seq))
      return fail(TOAST_E_INVALID_ARG, "invalid sequence (TOAST_ST_* bits " + std::to_string(st) + ")");
    toast::host_materialize(a, seq, masks);
  }
  return ret(TOAST_OK, "");
}

toast_status toast_lower(const toast_analysis* a, const uint16_t seq[32], char* buf, size_t cap, size_t* needed) {
  if (!a || !seq || !needed) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  if (const uint32_t st = toast::host_validate(a, seq))
    return fail(TOAST_E_INVALID_ARG, "invalid sequence (TOAST_ST_* bits " + std::to_string(st) + ")");
  std::string s, err;
  toast_status st = toast::lower_program(a, seq, s, err);
  if (st != TOAST_OK) return fail(st, err);
  *needed = s.size() + 1;
  if (buf && cap >= *needed) memcpy(buf, s.c_str(), s.size() + 1);
  return ret(TOAST_OK, "");
}

size_t toast_search_export_bytes(const toast_analysis* a) {
  return a ? toast::search_export_bytes(a) : 0;
}

toast_status toast_search_root_stats(const toast_search_state* s, toast_root_stat* out, int32_t cap, int32_t* n) {
  if (!s || !n || (cap > 0 && !out)) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  *n = toast::search_root_stats(s, out, cap);
  return ret(TOAST_OK, "");
}

toast_status toast_search_begin(const toast_analysis* a, const toast_search_opts* o, int32_t rank, int32_t world,
                                toast_search_state** out) {
  if (!a || !o || !out) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  if (a->device >= 0) cudaSetDevice(a->device);
  std::string err;
  return ret(toast::search_begin(a, o, rank, world, out, err), err);
}

toast_status toast_search_round(toast_search_state* s, void* export_buf) {
  if (!s || !export_buf) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  std::string err;
  return ret(toast::search_round(s, export_buf, err), err);
}

toast_status toast_search_import(toast_search_state* s, const void* gathered, int32_t* stop) {
  if (!s || !gathered || !stop) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  std::string err;
  return ret(toast::search_import(s, gathered, stop, err), err);
}

toast_status toast_search_round_dev(toast_search_state* s, void* export_dev, void* cuda_stream) {
  if (!s || !export_dev) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  if (!toast::is_device_pointer(export_dev)) return fail(TOAST_E_INVALID_ARG, "export_dev is not device memory");
  std::string err;
  return ret(toast::search_round_dev(s, export_dev, cuda_stream, err), err);
}

toast_status toast_search_import_dev(toast_search_state* s, const void* gathered_dev, int32_t* stop, void* cuda_stream) {
  if (!s || !gathered_dev || !stop) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  if (!toast::is_device_pointer(gathered_dev)) return fail(TOAST_E_INVALID_ARG, "gathered_dev is not device memory");
  std::string err;
  return ret(toast::search_import_dev(s, gathered_dev, stop, cuda_stream, err), err);
}

toast_status toast_search_end(toast_search_state* s, toast_search_result* out) {
  if (!s) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  if (out) toast::search_result(s, out);
  toast::search_free(s);
  return ret(TOAST_OK, "");
}

toast_status toast_search(const toast_analysis* a, const toast_search_opts* o, toast_search_result* out) {
  if (!a || !o || !out) return fail(TOAST_E_INVALID_ARG, "NULL argument");
  if (!has_device(a)) return fail(TOAST_E_CUDA, "the analysis has no device tables");
  toast_search_state* s = nullptr;
  toast_status st = toast_search_begin(a, o, 0, 1, &s);
  if (st) return st;
  std::string buf(toast::search_export_bytes(a), '\0');
  int32_t stop = 0;
  while (!stop) {
    st = toast_search_round(s, &buf[0]);
    if (!st) st = toast_search_import(s, buf.data(), &stop);
    if (st) {
      std::string keep = g_err;
      toast::search_free(s);
      return fail(st, keep);
    }
  }
  return toast_search_end(s, out);
}

void toast_free_graph(toast_graph* g) { delete g; }

void toast_free_analysis(toast_analysis* a) {
  if (!a) return;
  toast::free_tables(a);
  delete a;
}

}  // extern "C"
