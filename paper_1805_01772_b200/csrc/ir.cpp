// libcf host IR + builder + validate + JSON (see ir.h).
#include "ir.h"

#include <algorithm>
#include <cstring>
#include <set>
#include <sstream>

namespace cf {

int dt_size(int32_t d) {
  switch (d) {
    case BOOL: return 1;
    case I32: return 4;
    case I64: return 8;
    case F32: return 4;
    case F64: return 8;
    case BF16: return 2;
    default: return 0;
  }
}

const char* dt_name(int32_t d) {
  static const char* n[] = {"bool", "i32", "i64", "f32", "f64", "bf16", "flow", "res"};
  return (d >= 0 && d < 8) ? n[d] : "?";
}

// ------------------------------------------------------------------------------ attrs
int64_t Attrs::i(const std::string& k, int64_t d) const {
  auto it = kv.find(k);
  return it == kv.end() ? d : std::stoll(it->second);
}
double Attrs::f(const std::string& k, double d) const {
  auto it = kv.find(k);
  return it == kv.end() ? d : std::stod(it->second);
}
std::string Attrs::s(const std::string& k, const std::string& d) const {
  auto it = kv.find(k);
  return it == kv.end() ? d : it->second;
}
std::vector<int64_t> Attrs::v(const std::string& k) const {
  std::vector<int64_t> r;
  auto it = kv.find(k);
  if (it == kv.end() || it->second.empty()) return r;
  std::stringstream ss(it->second);
  std::string tok;
  while (std::getline(ss, tok, ',')) if (!tok.empty()) r.push_back(std::stoll(tok));
  return r;
}
void Attrs::setf(const std::string& k, double x) {
  std::ostringstream o;
  o.precision(17);
  o << x;
  kv[k] = o.str();
}
void Attrs::setv(const std::string& k, const std::vector<int64_t>& x) {
  std::string s;
  for (size_t j = 0; j < x.size(); ++j) s += (j ? "," : "") + std::to_string(x[j]);
  kv[k] = s;
}
Attrs Attrs::parse(const char* s) {
  Attrs a;
  if (!s) return a;
  std::string str(s);
  size_t p = 0;
  while (p < str.size()) {
    size_t e = str.find(';', p);
    if (e == std::string::npos) e = str.size();
    std::string item = str.substr(p, e - p);
    size_t eq = item.find('=');
    if (eq != std::string::npos) a.kv[item.substr(0, eq)] = item.substr(eq + 1);
    p = e + 1;
  }
  return a;
}

// ------------------------------------------------------------------------------ inference
static Shape bcast(const Shape& a, const Shape& b) {
  if (a == b) return a;
  if (a.empty()) return b;
  if (b.empty()) return a;
  throw CfError(CF_E_SHAPE, "incompatible shapes");
}

void infer(const Graph& g, const std::string& op, const std::vector<TRef>& in, const Attrs& a,
           std::vector<int32_t>* odt, std::vector<Shape>* osh) {
  std::vector<int32_t> dt;
  std::vector<Shape> sh;
  for (auto& t : in) {
    dt.push_back(g.dtype(t));
    sh.push_back(g.shape(t));
  }
  auto need = [&](size_t n) {
    if (in.size() != n)
      throw CfError(CF_E_ARITY, op + " expects " + std::to_string(n) + " inputs, got " +
                                    std::to_string(in.size()));
  };
  auto out1 = [&](int32_t d, Shape s) { odt->assign(1, d); osh->assign(1, std::move(s)); };
  if (op == "Placeholder") return out1((int32_t)a.i("dtype"), a.v("shape"));
  if (op == "Const") return out1((int32_t)a.i("dtype"), a.v("shape"));
  if (op == "Identity" || op == "ZerosLike" || op == "StopGradient") {
    need(1);
    return out1(dt[0], sh[0]);
  }
  if (op == "Neg" || op == "Sigmoid" || op == "Tanh" || op == "Relu") {
    need(1);
    if (!is_float(dt[0])) throw CfError(CF_E_DTYPE, op + " on non-float");
    return out1(dt[0], sh[0]);
  }
  if (op == "Add" || op == "Sub" || op == "Mul") {
    need(2);
    if (dt[0] != dt[1] || dt[0] == BOOL || dt[0] == RES) throw CfError(CF_E_DTYPE, op + " dtypes");
    return out1(dt[0], bcast(sh[0], sh[1]));
  }
  if (op == "AddN") {
    if (in.empty()) throw CfError(CF_E_ARITY, "AddN of nothing");
    for (size_t j = 0; j < in.size(); ++j)
      if (dt[j] != dt[0] || sh[j] != sh[0]) throw CfError(CF_E_SHAPE, "AddN mismatch");
    return out1(dt[0], sh[0]);
  }
  if (op == "ReluGrad") { need(2); return out1(dt[0], sh[0]); }
  if (op == "BiasAdd") {
    need(2);
    if (sh[0].size() != 2 || sh[1] != Shape{sh[0][1]}) throw CfError(CF_E_SHAPE, "BiasAdd");
    return out1(dt[0], sh[0]);
  }
  if (op == "MatMul") {
    need(2);
    if (!is_float(dt[0]) || dt[0] != dt[1]) throw CfError(CF_E_DTYPE, "MatMul on non-float");
    if (sh[0].size() != 2 || sh[1].size() != 2) throw CfError(CF_E_SHAPE, "MatMul needs rank 2");
    bool ta = a.b("ta"), tb = a.b("tb");
    int64_t m = ta ? sh[0][1] : sh[0][0], k1 = ta ? sh[0][0] : sh[0][1];
    int64_t k2 = tb ? sh[1][1] : sh[1][0], n = tb ? sh[1][0] : sh[1][1];
    if (k1 != k2) throw CfError(CF_E_SHAPE, "MatMul inner dimensions differ");
    return out1(dt[0], {m, n});
  }
  if (op == "Transpose") {
    need(1);
    Shape s(sh[0].rbegin(), sh[0].rend());
    return out1(dt[0], s);
  }
  if (op == "ReduceSum" || op == "ReduceMax" || op == "ReduceMin") {
    need(1);
    if (a.i("axis", -1) == 0) return out1(dt[0], Shape(sh[0].begin() + 1, sh[0].end()));
    return out1(dt[0], {});
  }
  if (op == "Fill") {
    need(1);
    if (!sh[0].empty()) throw CfError(CF_E_SHAPE, "Fill value must be a scalar");
    return out1(dt[0], a.v("shape"));
  }
  if (op == "Less" || op == "LessEqual" || op == "Greater" || op == "Equal") {
    need(2);
    if (dt[0] != dt[1]) throw CfError(CF_E_DTYPE, op + " dtypes differ");
    return out1(BOOL, bcast(sh[0], sh[1]));
  }
  if (op == "LogicalAnd") { need(2); return out1(BOOL, bcast(sh[0], sh[1])); }
  if (op == "LogicalNot") { need(1); return out1(BOOL, sh[0]); }
  if (op == "Select") {
    need(3);
    if (dt[0] != BOOL) throw CfError(CF_E_DTYPE, "Select condition must be bool");
    return out1(dt[1], bcast(sh[1], sh[2]));
  }
  if (op == "Concat") {
    int64_t ax = a.i("axis");
    Shape s = sh.at(0);
    s[ax] = 0;
    for (auto& x : sh) s[ax] += x[ax];
    return out1(dt[0], s);
  }
  if (op == "Slice") { need(1); return out1(dt[0], a.v("size")); }
  if (op == "SliceGrad") { need(1); return out1(dt[0], a.v("shape")); }
  if (op == "Reshape") {
    need(1);
    Shape s = a.v("shape");
    if (numel(s) != numel(sh[0])) throw CfError(CF_E_SHAPE, "Reshape size mismatch");
    return out1(dt[0], s);
  }
  if (op == "Cast") { need(1); return out1((int32_t)a.i("dtype"), sh[0]); }
  if (op == "LSTMCell") {
    need(a.b("masked") ? 7 : 5);
    if (sh[0].size() != 2 || sh[1].size() != 2) throw CfError(CF_E_SHAPE, "LSTMCell x/h rank");
    int64_t B = sh[0][0], I = sh[0][1], H = sh[1][1];
    if (sh[3] != Shape{4 * H, I + H} || sh[4] != Shape{4 * H} || sh[2] != Shape{B, H} ||
        sh[1] != Shape{B, H})
      throw CfError(CF_E_SHAPE, "LSTMCell shapes");
    odt->assign(4, dt[0]);
    *osh = {{B, H}, {B, H}, {B, H}, {B, 4 * H}};
    return;
  }
  if (op == "LSTMCellGrad") {
    need(a.b("masked") ? 10 : 8);
    int64_t B = sh[0][0], I = sh[0][1], H = sh[1][1];
    odt->assign(5, dt[0]);
    *osh = {{B, I}, {B, H}, {B, H}, {4 * H, I + H}, {4 * H}};
    return;
  }
  if (op == "Switch") {
    need(2);
    if (dt[1] != BOOL || !sh[1].empty())
      throw CfError(CF_E_NONBOOL_PRED, "Switch predicate must be a bool scalar");
    *odt = {dt[0], dt[0]};
    *osh = {sh[0], sh[0]};
    return;
  }
  if (op == "Merge") {
    need(2);
    if (dt[0] != dt[1]) throw CfError(CF_E_BRANCH_MISMATCH, "Merge dtypes differ");
    return out1(dt[0], sh[0]);
  }
  if (op == "Enter" || op == "Exit" || op == "NextIteration") { need(1); return out1(dt[0], sh[0]); }
  if (op == "TACreate") {
    *odt = {RES, FLOW};
    *osh = {{}, {}};
    return;
  }
  if (op == "TARead") { need(3); return out1((int32_t)a.i("dtype"), a.v("elem_shape")); }
  if (op == "TAWrite") { need(4); return out1(FLOW, {}); }
  if (op == "TAStack") {
    need(2);
    Shape s = a.v("elem_shape");
    s.insert(s.begin(), a.i("size"));
    return out1((int32_t)a.i("dtype"), s);
  }
  if (op == "TAUnstack") { need(3); return out1(FLOW, {}); }
  if (op == "TAGrad") {
    need(2);
    *odt = {RES, FLOW};
    *osh = {{}, {}};
    return;
  }
  if (op == "StackCreate") return out1(RES, {});
  if (op == "StackPush") { need(2); odt->clear(); osh->clear(); return; }
  if (op == "StackPop") { need(1); return out1((int32_t)a.i("dtype"), a.v("elem_shape")); }
  // cross-partition edges: message key = (channel, iteration tag)
  if (op == "Send") {
    need(2);
    if (dt[1] != I64 || !sh[1].empty()) throw CfError(CF_E_DTYPE, "Send index must be an int64 scalar");
    if (!a.has("channel") || !a.has("peer")) throw CfError(CF_E_ARITY, "Send needs channel and peer");
    odt->clear();
    osh->clear();
    return;
  }
  if (op == "Recv") {
    need(1);
    if (dt[0] != I64 || !sh[0].empty()) throw CfError(CF_E_DTYPE, "Recv index must be an int64 scalar");
    if (!a.has("channel") || !a.has("peer")) throw CfError(CF_E_ARITY, "Recv needs channel and peer");
    return out1((int32_t)a.i("dtype"), a.v("shape"));
  }
  throw CfError(CF_E_UNSUPPORTED, "unknown op " + op);
}

// ------------------------------------------------------------------------------ graph
bool Graph::is_ancestor(int anc, int c) const {
  for (int x = c; x >= 0; x = ctxs[x].parent)
    if (x == anc) return true;
  return false;
}

int Graph::enclosing_while(int c) const {
  for (int x = c; x >= 0; x = ctxs[x].parent)
    if (ctxs[x].kind == WHILE) return x;
  return -1;
}

int Graph::add(const std::string& op, const std::vector<TRef>& in, const Attrs& a, int ctx,
               const std::vector<int>& ctrl) {
  Node n;
  infer(*this, op, in, a, &n.odt, &n.osh);
  n.id = (int)nodes.size();
  n.op = op;
  n.in = in;
  n.ctrl = ctrl;
  n.attrs = a;
  n.ctx = ctx;
  nodes.push_back(std::move(n));
  return nodes.back().id;
}

TRef Graph::capture(TRef t, int c) {
  int d = ctx_of(t);
  if (d == c) return t;
  if (ctxs[c].kind == ROOT || !is_ancestor(d, c))
    throw CfError(CF_E_INVALID_GRAPH, "tensor used outside its control-flow context");
  TRef tp = capture(t, ctxs[c].parent);
  auto it = ctxs[c].captured.find(tp);
  if (it != ctxs[c].captured.end()) return it->second;
  TRef out;
  if (ctxs[c].kind == WHILE) {
    Attrs a;
    a.sets("frame", ctxs[c].name);
    a.set("is_constant", 1);
    int id = add("Enter", {tp}, a, c);
    ctxs[c].constants.push_back(id);
    out = {id, 0};
  } else {
    TRef p = capture(ctxs[c].pred, ctxs[c].parent);
    Attrs a;
    a.set("capture", 1);
    a.set("cond_id", ctxs[c].cond_id);
    int id = add("Switch", {tp, p}, a, c);
    out = {id, ctxs[c].branch};
  }
  ctxs[c].captured[tp] = out;
  return out;
}

TRef Graph::pivot_of(int c) {
  if (!ctxs[c].pivot.valid()) {
    // cond pivot: Identity(Switch(pred, pred)[branch])
    TRef p = capture(ctxs[c].pred, ctxs[c].parent);
    Attrs a;
    a.set("pivot", 1);
    a.set("cond_id", ctxs[c].cond_id);
    int sw = add("Switch", {p, p}, a, c);
    Attrs b;
    b.set("pivot", 1);
    int idn = add("Identity", {{sw, ctxs[c].branch}}, b, c);
    ctxs[c].pivot = {idn, 0};
  }
  return ctxs[c].pivot;
}

bool Graph::is_capture(TRef t) const {
  const Node& n = nodes[t.node];
  return (n.op == "Enter" && n.attrs.b("is_constant")) || (n.op == "Switch" && n.attrs.b("capture"));
}

std::vector<TRef> Graph::op(const std::string& o, const std::vector<TRef>& in, const Attrs& a) {
  std::vector<TRef> ins;
  for (auto& t : in) ins.push_back(capture(t, cur));
  std::vector<int> ctrl;
  // zero-input ops need the construct's pivot; in a loop body, ops fed only by loop
  // constants would otherwise also run on the exiting iteration
  bool all_cap = std::all_of(ins.begin(), ins.end(), [&](TRef t) { return is_capture(t); });
  if ((ctxs[cur].kind == COND && ins.empty()) || (ctxs[cur].kind == WHILE && all_cap))
    ctrl.push_back(pivot_of(cur).node);
  int id = add(o, ins, a, cur, ctrl);
  std::vector<TRef> r;
  for (size_t p = 0; p < nodes[id].odt.size(); ++p) r.push_back({id, (int32_t)p});
  return r;
}

TRef Graph::placeholder(const std::string& name, int32_t dt, const Shape& s) {
  if (placeholders.count(name)) throw CfError(CF_E_INVALID_GRAPH, "duplicate placeholder " + name);
  Attrs a;
  a.sets("name", name);
  a.set("dtype", dt);
  a.setv("shape", s);
  int id = add("Placeholder", {}, a, 0);
  placeholders[name] = id;
  return {id, 0};
}

TRef Graph::constant(int32_t dt, const Shape& s, const void* data) {
  Attrs a;
  a.set("dtype", dt);
  a.setv("shape", s);
  TRef r = op1("Const", {}, a);
  size_t bytes = (size_t)numel(s) * dt_size(dt);
  nodes[r.node].data.resize(bytes);
  if (bytes) {
    if (data) std::memcpy(nodes[r.node].data.data(), data, bytes);
    else std::memset(nodes[r.node].data.data(), 0, bytes);
  }
  return r;
}

TRef Graph::zeros(int32_t dt, const Shape& s) { return constant(dt, s, nullptr); }

std::vector<TRef> Graph::cond(TRef pred, const std::function<std::vector<TRef>()>& tf,
                              const std::function<std::vector<TRef>()>& ff) {
  if (dtype(pred) != BOOL || !shape(pred).empty())
    throw CfError(CF_E_NONBOOL_PRED, "cond predicate must be a bool scalar");
  pred = capture(pred, cur);
  int cid = n_conds++;
  std::vector<TRef> outs[2];
  for (int br : {1, 0}) {
    Ctx c;
    c.id = (int)ctxs.size();
    c.kind = COND;
    c.parent = cur;
    c.pred = pred;
    c.branch = br;
    c.cond_id = cid;
    ctxs.push_back(c);
    CtxGuard guard(*this, c.id);
    auto r = br ? tf() : ff();
    for (auto& t : r) outs[br].push_back(capture(t, cur));
  }
  if (outs[0].size() != outs[1].size())
    throw CfError(CF_E_BRANCH_MISMATCH, "cond branches return different arity");
  std::vector<TRef> merges;
  for (size_t j = 0; j < outs[0].size(); ++j) {
    if (dtype(outs[0][j]) != dtype(outs[1][j]))
      throw CfError(CF_E_BRANCH_MISMATCH, "cond branch dtypes differ");
    Attrs a;
    a.set("cond_id", cid);
    merges.push_back({add("Merge", {outs[0][j], outs[1][j]}, a, cur), 0});
  }
  return merges;
}

std::vector<TRef> Graph::while_loop(
    const std::function<TRef(const std::vector<TRef>&)>& pred,
    const std::function<std::vector<TRef>(const std::vector<TRef>&)>& body,
    const std::vector<TRef>& inits, int K, const std::string& name_in, TRef* counter_exit) {
  if (K < 1) throw CfError(CF_E_ARITY, "parallel_iterations must be >= 1");
  std::string name = name_in.empty() ? "while" + std::to_string(whiles.size()) : name_in;
  if (whiles.count(name)) throw CfError(CF_E_INVALID_GRAPH, "duplicate frame " + name);
  int parent = cur;
  std::vector<TRef> all{const_i64(0)};
  for (auto& t : inits) all.push_back(capture(t, cur));
  Ctx c;
  c.id = (int)ctxs.size();
  c.kind = WHILE;
  c.parent = parent;
  c.name = name;
  c.K = K;
  ctxs.push_back(c);
  int cid = c.id;
  whiles[name] = cid;
  frame_order.push_back(name);
  std::vector<LoopVar> lv(all.size());
  for (size_t j = 0; j < all.size(); ++j) {
    Attrs ea;
    ea.sets("frame", name);
    ea.set("is_constant", 0);
    lv[j].enter = add("Enter", {all[j]}, ea, cid);
    Attrs ma;
    ma.set("loop", 1);
    ma.sets("frame", name);
    lv[j].merge = add("Merge", {{lv[j].enter, 0}, {lv[j].enter, 0}}, ma, cid);
  }
  ctxs[cid].pivot = {lv[0].merge, 0};
  TRef p;
  {
    CtxGuard guard(*this, cid);
    std::vector<TRef> mv;
    for (size_t j = 1; j < lv.size(); ++j) mv.push_back({lv[j].merge, 0});
    p = pred(mv);
    if (dtype(p) != BOOL || !shape(p).empty())
      throw CfError(CF_E_NONBOOL_PRED, "loop predicate must be a bool scalar");
    p = capture(p, cid);
  }
  for (auto& v : lv) {
    Attrs sa;
    sa.set("loop", 1);
    sa.sets("frame", name);
    v.sw = add("Switch", {{v.merge, 0}, p}, sa, cid);
    Attrs xa;
    xa.sets("frame", name);
    v.exit = add("Exit", {{v.sw, 0}}, xa, parent);
  }
  Attrs pa;
  pa.set("pivot", 1);
  ctxs[cid].pivot = {add("Identity", {{lv[0].sw, 1}}, pa, cid), 0};
  std::vector<TRef> outs;
  TRef cnext;
  {
    CtxGuard guard(*this, cid);
    std::vector<TRef> bv;
    for (size_t j = 1; j < lv.size(); ++j) bv.push_back({lv[j].sw, 1});
    outs = body(bv);
    if (outs.size() != inits.size())
      throw CfError(CF_E_ARITY, "body returns wrong number of loop variables");
    for (auto& t : outs) t = capture(t, cid);
    cnext = op1("Add", {TRef{lv[0].sw, 1}, const_i64(1)});
  }
  outs.insert(outs.begin(), cnext);
  for (size_t j = 0; j < lv.size(); ++j) {
    if (dtype(outs[j]) != nodes[lv[j].merge].odt[0])
      throw CfError(CF_E_DTYPE, "body output dtype differs from loop variable");
    Attrs na;
    na.sets("frame", name);
    lv[j].next = add("NextIteration", {outs[j]}, na, cid);
    nodes[lv[j].merge].in[1] = {lv[j].next, 0};
  }
  ctxs[cid].loop_vars = lv;
  std::vector<TRef> res;
  for (size_t j = 1; j < lv.size(); ++j) res.push_back({lv[j].exit, 0});
  if (counter_exit) *counter_exit = {lv[0].exit, 0};
  return res;
}

// ------------------------------------------------------------------------------ validate
std::vector<std::string> Graph::validate() const {
  std::vector<std::string> errs;
  for (auto& n : nodes) {
    if ((n.op == "Merge" || n.op == "Switch") && n.in.size() != 2)
      errs.push_back("node " + std::to_string(n.id) + ": " + n.op + " arity");
    for (auto& t : n.in)
      if (t.node < 0 || t.node >= (int)nodes.size() || t.port >= (int)nodes[t.node].odt.size())
        errs.push_back("node " + std::to_string(n.id) + ": dangling input");
  }
  if (!errs.empty()) return errs;
  // cycles must pass through NextIteration
  std::vector<std::vector<int>> adj(nodes.size());
  for (auto& n : nodes)
    for (auto& t : n.in)
      if (nodes[t.node].op != "NextIteration") adj[t.node].push_back(n.id);
  std::vector<int> color(nodes.size(), 0);
  for (size_t s = 0; s < nodes.size(); ++s) {
    if (color[s]) continue;
    std::vector<std::pair<int, size_t>> st{{(int)s, 0}};
    color[s] = 1;
    while (!st.empty()) {
      auto& [v, k] = st.back();
      if (k < adj[v].size()) {
        int w = adj[v][k++];
        if (color[w] == 1) {
          errs.push_back("cycle lacks NextIteration (through node " + std::to_string(w) + ")");
          return errs;
        }
        if (!color[w]) {
          color[w] = 1;
          st.push_back({w, 0});
        }
      } else {
        color[v] = 2;
        st.pop_back();
      }
    }
  }
  // context crossing only via Enter / Exit / cond Switch / Merge
  for (auto& n : nodes) {
    for (auto& t : n.in) {
      const Node& s = nodes[t.node];
      if (s.ctx == n.ctx) continue;
      bool ok = false;
      const Ctx& nc = ctxs[n.ctx];
      const Ctx& sc = ctxs[s.ctx];
      if (n.op == "Enter" && s.ctx == nc.parent) ok = true;
      else if (n.op == "Exit" && sc.parent == n.ctx) ok = true;
      else if (n.op == "Switch" && nc.kind == COND && s.ctx == nc.parent) ok = true;
      else if (n.op == "Merge" && sc.kind == COND && sc.parent == n.ctx) ok = true;
      else if (s.op == "Exit" && s.ctx == n.ctx) ok = true;
      if (!ok)
        errs.push_back("node " + std::to_string(n.id) + " (" + n.op + ") crosses context from node " +
                       std::to_string(s.id) + " (" + s.op + ")");
    }
  }
  return errs;
}

std::string Graph::json() const {
  std::ostringstream o;
  o << "{\"version\":1,\"nodes\":[";
  for (size_t j = 0; j < nodes.size(); ++j) {
    const Node& n = nodes[j];
    o << (j ? "," : "") << "{\"id\":" << n.id << ",\"op\":\"" << n.op << "\",\"ctx\":" << n.ctx
      << ",\"inputs\":[";
    for (size_t k = 0; k < n.in.size(); ++k)
      o << (k ? "," : "") << "[" << n.in[k].node << "," << n.in[k].port << "]";
    o << "],\"ctrl\":[";
    for (size_t k = 0; k < n.ctrl.size(); ++k) o << (k ? "," : "") << n.ctrl[k];
    o << "],\"attrs\":{";
    size_t k = 0;
    for (auto& [key, val] : n.attrs.kv) o << (k++ ? "," : "") << "\"" << key << "\":\"" << val << "\"";
    o << "},\"dtypes\":[";
    for (size_t q = 0; q < n.odt.size(); ++q) o << (q ? "," : "") << "\"" << dt_name(n.odt[q]) << "\"";
    o << "]}";
  }
  o << "],\"contexts\":[";
  for (size_t j = 0; j < ctxs.size(); ++j) {
    const Ctx& c = ctxs[j];
    o << (j ? "," : "") << "{\"id\":" << c.id << ",\"kind\":" << (int)c.kind
      << ",\"parent\":" << c.parent << ",\"name\":\"" << c.name << "\",\"K\":" << c.K
      << ",\"cond_id\":" << c.cond_id << ",\"branch\":" << c.branch << "}";
  }
  o << "]}";
  return o.str();
}

}  // namespace cf
