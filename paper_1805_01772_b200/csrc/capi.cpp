// extern "C" graph-construction entry points of libcf (include/cf.h). Execution entry points
// (cf_session_*, cf_run) live in runtime.cu.
#include <cstring>
#include <cstdlib>
#include <string>

#include "compiler.h"
#include "ir.h"

struct cf_graph {
  cf::Graph g;
};

namespace cf {
thread_local std::string g_last_error;
void set_error(const std::string& m) { g_last_error = m; }
}  // namespace cf

using cf::CfError;
using cf::TRef;

#define CF_TRY try {
#define CF_CATCH                                   \
  }                                                \
  catch (const CfError& e) {                       \
    cf::set_error(e.what());                       \
    return e.code;                                 \
  }                                                \
  catch (const std::exception& e) {                \
    cf::set_error(std::string("internal: ") + e.what()); \
    return CF_E_INVALID_GRAPH;                     \
  }                                                \
  return CF_OK;

static TRef tr(cf_tensor t) { return TRef{t.node, t.port}; }
static cf_tensor ct(TRef t) { return cf_tensor{t.node, t.port}; }

static void check(const cf_graph* g, cf_tensor t) {
  if (!g) throw CfError(CF_E_INVALID_GRAPH, "null graph");
  if (t.node < 0 || t.node >= (int)g->g.nodes.size() || t.port < 0 ||
      t.port >= (int)g->g.nodes[t.node].odt.size())
    throw CfError(CF_E_INVALID_GRAPH, "invalid tensor handle");
}

extern "C" {

const char* cf_last_error(void) { return cf::g_last_error.c_str(); }
const char* cf_version(void) { return "libcf 0.1 (sm_100a)"; }

cf_status cf_graph_create(cf_graph** out) {
  CF_TRY
  if (!out) throw CfError(CF_E_INVALID_GRAPH, "null out");
  *out = new cf_graph();
  CF_CATCH
}

void cf_graph_destroy(cf_graph* g) { delete g; }

cf_status cf_placeholder(cf_graph* g, const char* name, int32_t dtype, int32_t rank,
                         const int64_t* shape, cf_tensor* out) {
  CF_TRY
  if (!g || !name || !out || rank < 0 || rank > 8) throw CfError(CF_E_ARITY, "bad arguments");
  if (dtype < 0 || dtype > CF_FLOW) throw CfError(CF_E_DTYPE, "bad dtype");
  *out = ct(g->g.placeholder(name, dtype, cf::Shape(shape, shape + rank)));
  CF_CATCH
}

cf_status cf_const(cf_graph* g, int32_t dtype, int32_t rank, const int64_t* shape,
                   const void* host_data, cf_tensor* out) {
  CF_TRY
  if (!g || !out || rank < 0 || rank > 8) throw CfError(CF_E_ARITY, "bad arguments");
  *out = ct(g->g.constant(dtype, cf::Shape(shape, shape + rank), host_data));
  CF_CATCH
}

cf_status cf_op(cf_graph* g, const char* op, int32_t n_in, const cf_tensor* in,
                const char* attrs, int32_t* n_out, cf_tensor* out) {
  CF_TRY
  if (!g || !op) throw CfError(CF_E_ARITY, "bad arguments");
  std::vector<TRef> ins;
  for (int i = 0; i < n_in; ++i) {
    check(g, in[i]);
    ins.push_back(tr(in[i]));
  }
  std::string o(op);
  if (o == "Placeholder" || o == "Const" || o == "Switch" || o == "Merge" || o == "Enter" ||
      o == "Exit" || o == "NextIteration")
    throw CfError(CF_E_INVALID_GRAPH, "use cf_placeholder/cf_const/cf_cond/cf_while_loop for " + o);
  auto r = g->g.op(o, ins, cf::Attrs::parse(attrs));
  if (r.size() > 8) throw CfError(CF_E_ARITY, "too many outputs");
  if (n_out) *n_out = (int32_t)r.size();
  for (size_t j = 0; j < r.size() && out; ++j) out[j] = ct(r[j]);
  CF_CATCH
}

static cf_status while_impl(cf_graph* g, cf_pred_fn pred, cf_body_fn body, void* user, int32_t n,
                            const cf_tensor* inits, int32_t K, const char* name, cf_tensor* outs,
                            cf_tensor* trip) {
  CF_TRY
  if (!g || !pred || !body || n < 0) throw CfError(CF_E_ARITY, "bad arguments");
  std::vector<TRef> iv;
  for (int i = 0; i < n; ++i) {
    check(g, inits[i]);
    iv.push_back(tr(inits[i]));
  }
  auto pf = [&](const std::vector<TRef>& v) {
    std::vector<cf_tensor> a;
    for (auto& t : v) a.push_back(ct(t));
    cf_tensor p{-1, 0};
    cf_status st = pred(g, (int32_t)a.size(), a.data(), &p, user);
    if (st != CF_OK) throw CfError(st, "pred callback failed: " + cf::g_last_error);
    check(g, p);
    return tr(p);
  };
  auto bf = [&](const std::vector<TRef>& v) {
    std::vector<cf_tensor> a, o(v.size(), cf_tensor{-1, 0});
    for (auto& t : v) a.push_back(ct(t));
    cf_status st = body(g, (int32_t)a.size(), a.data(), o.data(), user);
    if (st != CF_OK) throw CfError(st, "body callback failed: " + cf::g_last_error);
    std::vector<TRef> r;
    for (auto& t : o) {
      check(g, t);
      r.push_back(tr(t));
    }
    return r;
  };
  TRef ce;
  auto r = g->g.while_loop(pf, bf, iv, K, name ? name : "", &ce);
  for (size_t j = 0; j < r.size(); ++j) outs[j] = ct(r[j]);
  if (trip) *trip = ct(ce);
  CF_CATCH
}

cf_status cf_while_loop(cf_graph* g, cf_pred_fn pred, cf_body_fn body, void* user, int32_t n,
                        const cf_tensor* inits, int32_t K, const char* name, cf_tensor* outs) {
  return while_impl(g, pred, body, user, n, inits, K, name, outs, nullptr);
}

cf_status cf_while_loop_counted(cf_graph* g, cf_pred_fn pred, cf_body_fn body, void* user,
                                int32_t n, const cf_tensor* inits, int32_t K, const char* name,
                                cf_tensor* outs, cf_tensor* trip) {
  return while_impl(g, pred, body, user, n, inits, K, name, outs, trip);
}

cf_status cf_cond(cf_graph* g, cf_tensor pred, cf_branch_fn t, cf_branch_fn f, void* user,
                  int32_t n_out, cf_tensor* outs) {
  CF_TRY
  if (!g || !t || !f || n_out < 0) throw CfError(CF_E_ARITY, "bad arguments");
  check(g, pred);
  auto mk = [&](cf_branch_fn fn) {
    return [&, fn]() {
      std::vector<cf_tensor> o(n_out, cf_tensor{-1, 0});
      cf_status st = fn(g, n_out, o.data(), user);
      if (st != CF_OK) throw CfError(st, "branch callback failed: " + cf::g_last_error);
      std::vector<TRef> r;
      for (auto& x : o) {
        check(g, x);
        r.push_back(tr(x));
      }
      return r;
    };
  };
  auto r = g->g.cond(tr(pred), mk(t), mk(f));
  for (size_t j = 0; j < r.size(); ++j) outs[j] = ct(r[j]);
  CF_CATCH
}

cf_status cf_ta_create(cf_graph* g, int64_t size, int32_t dtype, int32_t elem_rank,
                       const int64_t* elem_shape, cf_tensor* handle, cf_tensor* flow) {
  CF_TRY
  if (!g || size < 0 || elem_rank < 0 || elem_rank > 7) throw CfError(CF_E_ARITY, "bad arguments");
  cf::Attrs a;
  a.set("size", size);
  a.set("dtype", dtype);
  a.setv("elem_shape", cf::Shape(elem_shape, elem_shape + elem_rank));
  auto r = g->g.op("TACreate", {}, a);
  *handle = ct(r[0]);
  *flow = ct(r[1]);
  CF_CATCH
}

static cf::Attrs ta_attrs(cf_graph* g, cf_tensor h) {
  // TA attrs travel with the handle: find the TACreate behind Enter/Switch/Identity routing
  TRef t = tr(h);
  for (int guard = 0; guard < 10000; ++guard) {
    const cf::Node& n = g->g.nodes[t.node];
    if (n.op == "TACreate" || n.op == "TAGrad") {
      if (n.op == "TAGrad") {
        t = n.in[0];
        continue;
      }
      cf::Attrs a;
      a.set("size", n.attrs.i("size"));
      a.set("dtype", n.attrs.i("dtype"));
      a.setv("elem_shape", n.attrs.v("elem_shape"));
      return a;
    }
    if (n.in.empty()) break;
    t = n.in[0];
  }
  throw CfError(CF_E_INVALID_GRAPH, "TensorArray handle does not come from cf_ta_create");
}

cf_status cf_ta_read(cf_graph* g, cf_tensor h, cf_tensor ix, cf_tensor flow, cf_tensor* value) {
  CF_TRY
  check(g, h);
  check(g, ix);
  check(g, flow);
  *value = ct(g->g.op1("TARead", {tr(h), tr(ix), tr(flow)}, ta_attrs(g, h)));
  CF_CATCH
}

cf_status cf_ta_write(cf_graph* g, cf_tensor h, cf_tensor ix, cf_tensor v, cf_tensor flow,
                      cf_tensor* flow_out) {
  CF_TRY
  check(g, h);
  check(g, ix);
  check(g, v);
  check(g, flow);
  *flow_out = ct(g->g.op1("TAWrite", {tr(h), tr(ix), tr(v), tr(flow)}, ta_attrs(g, h)));
  CF_CATCH
}

cf_status cf_ta_unstack(cf_graph* g, cf_tensor h, cf_tensor v, cf_tensor flow, cf_tensor* flow_out) {
  CF_TRY
  check(g, h);
  check(g, v);
  check(g, flow);
  *flow_out = ct(g->g.op1("TAUnstack", {tr(h), tr(v), tr(flow)}, ta_attrs(g, h)));
  CF_CATCH
}

cf_status cf_ta_stack(cf_graph* g, cf_tensor h, cf_tensor flow, cf_tensor* value) {
  CF_TRY
  check(g, h);
  check(g, flow);
  *value = ct(g->g.op1("TAStack", {tr(h), tr(flow)}, ta_attrs(g, h)));
  CF_CATCH
}

cf_status cf_gradients(cf_graph* g, cf_tensor y, int32_t n_x, const cf_tensor* xs,
                       cf_tensor* out_grads) {
  CF_TRY
  check(g, y);
  std::vector<TRef> xv;
  for (int i = 0; i < n_x; ++i) {
    check(g, xs[i]);
    xv.push_back(tr(xs[i]));
  }
  auto r = cf::gradients(g->g, tr(y), xv);
  for (size_t j = 0; j < r.size(); ++j) out_grads[j] = ct(r[j]);
  CF_CATCH
}

cf_status cf_validate(const cf_graph* g, char* report, size_t cap) {
  if (!g) return CF_E_INVALID_GRAPH;
  auto errs = g->g.validate();
  std::string s;
  for (auto& e : errs) s += e + "\n";
  if (report && cap) {
    std::strncpy(report, s.c_str(), cap - 1);
    report[cap - 1] = 0;
  }
  if (!errs.empty()) {
    cf::set_error(errs[0]);
    return CF_E_INVALID_GRAPH;
  }
  return CF_OK;
}

cf_status cf_graph_json(const cf_graph* g, char* buf, size_t cap, size_t* needed) {
  if (!g) return CF_E_INVALID_GRAPH;
  std::string s = g->g.json();
  if (needed) *needed = s.size() + 1;
  if (buf && cap) {
    std::strncpy(buf, s.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  return CF_OK;
}

cf_status cf_graph_num_nodes(const cf_graph* g, int32_t* n) {
  if (!g || !n) return CF_E_INVALID_GRAPH;
  *n = (int32_t)g->g.nodes.size();
  return CF_OK;
}

cf_status cf_tensor_info(const cf_graph* g, cf_tensor t, int32_t* dtype, int32_t* rank,
                         int64_t* shape) {
  CF_TRY
  check(g, t);
  const auto& s = g->g.shape(tr(t));
  if (dtype) *dtype = g->g.dtype(tr(t));
  if (rank) *rank = (int32_t)s.size();
  if (shape)
    for (size_t j = 0; j < s.size() && j < 8; ++j) shape[j] = s[j];
  CF_CATCH
}

// debug hook (include/cf_debug.h): compile without a device and list the body programs
int32_t cf_debug_program_listing(const cf_graph* g, int32_t precision, int32_t parallel_iterations,
                                 int32_t n_fetch, const cf_tensor* fetches, char* buf, size_t cap,
                                 size_t* needed) {
  CF_TRY
  if (!g) throw CfError(CF_E_INVALID_GRAPH, "null graph");
  cf::CompileOpts o;
  o.precision = precision ? precision : CF_F32;
  o.parallel_iterations = parallel_iterations;
  // iteration bound of frames without a TensorArray (cf_run_opts.max_iterations)
  if (const char* mi = std::getenv("CF_DEBUG_MAX_ITERATIONS")) o.max_iterations = atoll(mi);
  std::vector<TRef> fv;
  for (int i = 0; i < n_fetch; ++i) fv.push_back(tr(fetches[i]));
  cf::HostProgram P = cf::compile(g->g, o, fv);
  std::string txt = P.describe + P.listing;
  if (needed) *needed = txt.size() + 1;
  if (buf && cap) {
    std::strncpy(buf, txt.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  CF_CATCH
}

}  // extern "C"

// accessor used by runtime.cu
const cf::Graph& cf_graph_ir(const cf_graph* g) { return g->g; }
