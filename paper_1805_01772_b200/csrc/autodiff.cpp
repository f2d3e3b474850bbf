// libcf gradients(): PAPER.md §5.1-5.2.
//
//  * Four-step reverse-mode algorithm: Grads[y] := 1, reverse topological
//    traversal, gradient function per op, contributions summed.
//  * The traversal runs per control-flow context; a nested cond / while is one item of its
//    enclosing context and "generates a corresponding control-flow construct in the gradient
//    graph":
//      - cond -> cond(pred, true_fn_grad(g_z), false_fn_grad(g_z));
//      - while -> a gradient while_loop running the forward trip count (hidden counter) in
//        reverse; loop-variable grads as gradient loop variables; loop-constant grads summed
//        eagerly into extra loop variables.
//  * Forward values referenced by gradient code inside a loop are saved on one stack each:
//    StackPush in the forward context, StackPop in the mirrored gradient context
//    (PAPER.md:1046-1066). The predicate of a cond nested in a loop is such a value, hence the
//    per-iteration predicate stack. Loop constants are not pushed.
//  * MatMulGrad; TensorArray duality.
#include <algorithm>
#include <cstring>
#include <functional>
#include <map>
#include <set>

#include "ir.h"

namespace cf {
namespace {

struct Item {
  int kind = 0;      // 0 node, 1 cond, 2 while
  int key = 0;       // node id / cond id / frame ctx id
  std::vector<int> nodes;
  std::vector<TRef> inputs, outputs;
};

class AD {
 public:
  explicit AD(Graph& g) : g_(g) { mirror_[0] = 0; }

  TRef zeros_like(TRef t) {
    int32_t d = g_.dtype(t);
    if (d == FLOW) {
      float z = 0;
      (void)z;
      return g_.constant(FLOW, {}, nullptr);
    }
    return g_.zeros(d, g_.shape(t));
  }

  TRef sum(const std::vector<TRef>& v) {
    if (v.size() == 1) return v[0];
    return g_.op1("AddN", v);
  }

  // A forward value referenced from gradient code (loop constants resolve outward; values
  // inside a loop being differentiated are stack-saved).
  TRef fwd(TRef t) {
    const Node& n = g_.nodes[t.node];
    if (n.op == "Enter" && n.attrs.b("is_constant")) return fwd(n.in[0]);
    int C = n.ctx;
    int W = g_.enclosing_while(C);
    if (W < 0 || !mirror_.count(W)) return t;
    auto pit = pop_of_.find(t);
    if (pit != pop_of_.end()) return pit->second;
    if (!stack_of_.count(t)) {
      Attrs a;
      a.sets("frame", g_.ctxs[W].name);
      a.set("dtype", g_.dtype(t));
      a.setv("elem_shape", g_.shape(t));
      TRef h;
      {
        CtxGuard guard(g_, g_.ctxs[W].parent);
        h = g_.op1("StackCreate", {}, a);
      }
      {
        CtxGuard guard(g_, C);
        g_.op("StackPush", {h, t});
      }
      stack_of_[t] = h;
    }
    Attrs pa;
    pa.set("dtype", g_.dtype(t));
    pa.setv("elem_shape", g_.shape(t));
    // a loop nested in another loop ("for nested loops, we apply our
    // techniques recursively"): its stack is created once per outer iteration, in the outer
    // body, so the handle is itself an outer-loop value the gradient needs -- saved on a
    // stack of the outer loop in turn (fwd recursion)
    const TRef hp = fwd(stack_of_[t]);
    TRef v;
    {
      CtxGuard guard(g_, mirror_.at(C));
      v = g_.op1("StackPop", {hp}, pa);
    }
    pop_of_[t] = v;
    return v;
  }

  TRef reduce_to(TRef gt, TRef like, TRef out) {
    if (g_.shape(like).empty() && !g_.shape(out).empty()) return g_.op1("ReduceSum", {gt});
    return gt;
  }

  bool machinery(const Node& n, int ctx) {
    const Ctx& c = g_.ctxs[ctx];
    if (c.kind == COND)
      return (n.op == "Switch" && n.ctx == ctx) || (n.op == "Identity" && n.attrs.b("pivot"));
    if (c.kind != WHILE) return false;
    if (n.attrs.s("frame") == c.name &&
        (n.op == "Enter" || n.op == "NextIteration" ||
         ((n.op == "Merge" || n.op == "Switch") && n.attrs.b("loop"))))
      return true;
    return n.op == "Identity" && n.attrs.b("pivot");
  }

  void items(int ctx, std::vector<Item>* out_items, std::vector<int>* topo) {
    std::map<std::pair<int, int>, int> index;
    std::vector<Item>& its = *out_items;
    for (const Node& n : g_.nodes) {
      std::pair<int, int> key;
      if (n.ctx == ctx) {
        if (machinery(n, ctx)) continue;
        if (n.op == "Merge" && n.attrs.has("cond_id") && !n.attrs.b("loop"))
          key = {1, (int)n.attrs.i("cond_id")};
        else if (n.op == "Exit")
          key = {2, g_.whiles.at(n.attrs.s("frame"))};
        else
          key = {0, n.id};
      } else {
        int cc = n.ctx;
        while (cc >= 0 && g_.ctxs[cc].parent != ctx) cc = g_.ctxs[cc].parent;
        if (cc < 0) continue;
        key = g_.ctxs[cc].kind == COND ? std::make_pair(1, g_.ctxs[cc].cond_id)
                                       : std::make_pair(2, cc);
      }
      auto it = index.find(key);
      if (it == index.end()) {
        Item item;
        item.kind = key.first;
        item.key = key.second;
        index[key] = (int)its.size();
        its.push_back(item);
        it = index.find(key);
      }
      its[it->second].nodes.push_back(n.id);
    }
    for (Item& it : its) {
      if (it.kind == 0) {
        const Node& n = g_.nodes[it.nodes[0]];
        it.inputs = n.in;
        for (size_t p = 0; p < n.odt.size(); ++p) it.outputs.push_back({n.id, (int32_t)p});
      } else if (it.kind == 1) {
        for (int id : it.nodes) {
          const Node& n = g_.nodes[id];
          if (n.op == "Merge" && n.ctx == ctx) it.outputs.push_back({id, 0});
          if (n.op == "Switch" && g_.ctxs[n.ctx].kind == COND && g_.ctxs[n.ctx].parent == ctx)
            for (auto& t : n.in) it.inputs.push_back(t);
        }
      } else {
        const std::string& name = g_.ctxs[it.key].name;
        for (int id : it.nodes) {
          const Node& n = g_.nodes[id];
          if (n.op == "Exit" && n.ctx == ctx) it.outputs.push_back({id, 0});
          if (n.op == "Enter" && n.attrs.s("frame") == name) it.inputs.push_back(n.in[0]);
        }
      }
    }
    std::map<int, int> prod;
    for (size_t k = 0; k < its.size(); ++k)
      for (int id : its[k].nodes) prod[id] = (int)k;
    std::vector<std::set<int>> deps(its.size());
    for (size_t k = 0; k < its.size(); ++k)
      for (auto& t : its[k].inputs) {
        auto p = prod.find(t.node);
        if (p != prod.end() && p->second != (int)k) deps[k].insert(p->second);
      }
    std::vector<int> seen(its.size(), 0);
    std::function<void(int)> visit = [&](int k) {
      if (seen[k]) return;
      seen[k] = 1;
      for (int d : deps[k]) visit(d);
      topo->push_back(k);
    };
    for (size_t k = 0; k < its.size(); ++k) visit((int)k);
  }

  std::map<TRef, TRef> backprop(int ctx, const std::map<TRef, std::vector<TRef>>& ups,
                                const std::vector<TRef>& wrt) {
    std::vector<Item> its;
    std::vector<int> topo;
    items(ctx, &its, &topo);
    std::set<TRef> from_wrt(wrt.begin(), wrt.end());
    // Send/Recv pairs carry the dependence across partitions: a Recv's value depends on the
    // peer's parameters, and every Send/Recv gets its mirrored gradient message, so items
    // holding one are never pruned (the peer would wait forever otherwise).
    std::vector<char> comm(its.size(), 0), recv(its.size(), 0);
    for (size_t k = 0; k < its.size(); ++k)
      for (int id : its[k].nodes) {
        const std::string& o = g_.nodes[id].op;
        if (o == "Send" || o == "Recv") comm[k] = 1;
        if (o == "Recv") recv[k] = 1;
      }
    for (int k : topo) {
      bool hit = recv[k] != 0;
      for (auto& t : its[k].inputs) hit |= from_wrt.count(t) > 0;
      if (hit) from_wrt.insert(its[k].outputs.begin(), its[k].outputs.end());
    }
    std::map<TRef, std::vector<TRef>> grads = ups;
    for (auto r = topo.rbegin(); r != topo.rend(); ++r) {
      Item& it = its[*r];
      std::vector<TRef> g_outs;
      bool any = false;
      for (auto& o : it.outputs) {
        auto gi = grads.find(o);
        if (gi != grads.end() && !gi->second.empty()) {
          TRef s = sum(gi->second);
          gi->second = {s};
          g_outs.push_back(s);
          any = true;
        } else {
          g_outs.push_back(TRef{});
        }
      }
      if (!any && !comm[*r]) continue;
      bool reach = comm[*r] != 0;
      for (auto& t : it.inputs) reach |= from_wrt.count(t) > 0;
      if (!reach) continue;
      std::vector<std::pair<TRef, TRef>> pairs;
      if (it.kind == 0) {
        auto gs = op_grad(g_.nodes[it.nodes[0]].id, g_outs);
        for (size_t j = 0; j < it.inputs.size(); ++j) pairs.push_back({it.inputs[j], gs[j]});
      } else if (it.kind == 1) {
        pairs = cond_grad(ctx, it, g_outs);
      } else {
        pairs = while_grad(ctx, it, g_outs);
      }
      for (auto& [t, gt] : pairs)
        if (gt.valid() && from_wrt.count(t) && differentiable(g_.dtype(t))) grads[t].push_back(gt);
    }
    std::map<TRef, TRef> res;
    for (auto& t : wrt) {
      auto gi = grads.find(t);
      if (gi != grads.end() && !gi->second.empty()) res[t] = sum(gi->second);
    }
    return res;
  }

  std::vector<std::pair<TRef, TRef>> cond_grad(int ctx, const Item& it,
                                               const std::vector<TRef>& g_outs) {
    int cond_id = it.key;
    std::map<int, int> branch_ctx;
    std::vector<std::pair<TRef, TRef>> captures[2];
    TRef pred;
    for (int id : it.nodes) {
      const Node& n = g_.nodes[id];
      const Ctx& c = g_.ctxs[n.ctx];
      if (c.kind == COND && c.parent == ctx && c.cond_id == cond_id) {
        branch_ctx[c.branch] = n.ctx;
        if (n.op == "Switch") {
          pred = n.in[1];
          if (n.attrs.b("capture")) captures[c.branch].push_back({n.in[0], {id, c.branch}});
        }
      }
    }
    std::vector<TRef> externals;
    for (int br : {1, 0})
      for (auto& [e, s] : captures[br])
        if (differentiable(g_.dtype(e)) &&
            std::find(externals.begin(), externals.end(), e) == externals.end())
          externals.push_back(e);
    bool has_comm = false;
    for (int id : it.nodes) has_comm |= g_.nodes[id].op == "Send" || g_.nodes[id].op == "Recv";
    if (externals.empty() && !has_comm) return {};
    TRef pred_g = fwd(pred);
    std::vector<const Node*> merges;
    for (auto& o : it.outputs) merges.push_back(&g_.nodes[o.node]);
    std::vector<TRef> merge_in[2];
    for (auto* m : merges) {
      merge_in[0].push_back(m->in[0]);
      merge_in[1].push_back(m->in[1]);
    }
    auto make = [&](int br) {
      return [&, br]() {
        std::vector<TRef> res;
        auto bc = branch_ctx.find(br);
        std::map<TRef, TRef> gd;
        std::vector<TRef> leaves;
        for (auto& [e, s] : captures[br]) leaves.push_back(s);
        if (bc != branch_ctx.end()) {
          mirror_[bc->second] = g_.cur;
          std::map<TRef, std::vector<TRef>> ups;
          for (size_t j = 0; j < merge_in[br].size(); ++j)
            if (g_outs[j].valid()) ups[merge_in[br][j]].push_back(g_outs[j]);
          gd = backprop(bc->second, ups, leaves);
        }
        for (auto& e : externals) {
          std::vector<TRef> gs;
          for (auto& [ee, s] : captures[br])
            if (ee == e && gd.count(s)) gs.push_back(gd[s]);
          res.push_back(gs.empty() ? zeros_like(e) : sum(gs));
        }
        return res;
      };
    };
    auto outs = g_.cond(pred_g, make(1), make(0));
    std::vector<std::pair<TRef, TRef>> pairs;
    for (size_t j = 0; j < externals.size(); ++j) pairs.push_back({externals[j], outs[j]});
    return pairs;
  }

  std::vector<std::pair<TRef, TRef>> while_grad(int ctx, const Item& it,
                                                const std::vector<TRef>& g_outs) {
    (void)ctx;
    int W = it.key;
    const std::string name = g_.ctxs[W].name;
    const std::vector<LoopVar> lv = g_.ctxs[W].loop_vars;
    std::map<int, TRef> g_exit;
    for (size_t j = 0; j < it.outputs.size(); ++j) g_exit[it.outputs[j].node] = g_outs[j];
    TRef n_trip = fwd(TRef{lv[0].exit, 0});
    std::vector<size_t> var_js;
    for (size_t j = 1; j < lv.size(); ++j)
      if (differentiable(g_.nodes[lv[j].enter].odt[0])) var_js.push_back(j);
    std::vector<int> consts;
    for (int e : g_.ctxs[W].constants)
      if (differentiable(g_.nodes[e].odt[0])) consts.push_back(e);
    std::vector<TRef> inits{n_trip};
    for (size_t j : var_js) {
      auto ge = g_exit.find(lv[j].exit);
      TRef init_in = g_.nodes[lv[j].enter].in[0];
      inits.push_back(ge != g_exit.end() && ge->second.valid() ? ge->second : zeros_like(init_in));
    }
    for (int e : consts) inits.push_back(zeros_like(g_.nodes[e].in[0]));
    size_t nv = var_js.size();
    auto pred = [&](const std::vector<TRef>& v) {
      return g_.op1("Greater", {v[0], g_.const_i64(0)});
    };
    auto body = [&](const std::vector<TRef>& v) {
      mirror_[W] = g_.cur;
      std::map<TRef, std::vector<TRef>> ups;
      for (size_t q = 0; q < nv; ++q)
        ups[g_.nodes[lv[var_js[q]].next].in[0]].push_back(v[1 + q]);
      std::vector<TRef> leaves;
      for (size_t j : var_js) leaves.push_back({lv[j].sw, 1});
      for (int e : consts) leaves.push_back({e, 0});
      auto gd = backprop(W, ups, leaves);
      std::vector<TRef> out{g_.op1("Sub", {v[0], g_.const_i64(1)})};
      for (size_t j : var_js) {
        TRef s{lv[j].sw, 1};
        out.push_back(gd.count(s) ? gd[s] : zeros_like(g_.nodes[lv[j].enter].in[0]));
      }
      for (size_t q = 0; q < consts.size(); ++q) {
        TRef s{consts[q], 0};
        TRef acc = v[1 + nv + q];
        out.push_back(gd.count(s) ? g_.op1("Add", {acc, gd[s]}) : acc);
      }
      return out;
    };
    auto outs = g_.while_loop(pred, body, inits, g_.ctxs[W].K, name + "_grad", nullptr);
    std::vector<std::pair<TRef, TRef>> pairs;
    for (size_t q = 0; q < nv; ++q) pairs.push_back({g_.nodes[lv[var_js[q]].enter].in[0], outs[1 + q]});
    for (size_t q = 0; q < consts.size(); ++q)
      pairs.push_back({g_.nodes[consts[q]].in[0], outs[1 + nv + q]});
    return pairs;
  }

  std::vector<TRef> op_grad(int nid, const std::vector<TRef>& g_outs) {
    // copy: the node vector may grow while building
    const Node n = g_.nodes[nid];
    const std::string& op = n.op;
    TRef g = g_outs.empty() ? TRef{} : g_outs[0];
    TRef out{nid, 0};
    const auto& in = n.in;
    auto none = std::vector<TRef>(in.size());
    auto mm = [&](TRef a, TRef b, bool ta, bool tb) {
      Attrs at;
      at.set("ta", ta);
      at.set("tb", tb);
      return g_.op1("MatMul", {a, b}, at);
    };
    auto one = [&]() {
      float v = 1.0f;
      return g_.constant(F32, {}, &v);
    };
    if (op == "Identity" || op == "Cast") return {g};
    if (op == "Send") {
      // the gradient of a sent value comes back from the receiver on the mirrored edge
      Attrs a;
      a.set("channel", n.attrs.i("channel") ^ kGradChannel);
      a.set("peer", n.attrs.i("peer"));
      a.set("dtype", g_.dtype(in[0]));
      a.setv("shape", g_.shape(in[0]));
      return {g_.op1("Recv", {fwd(in[1])}, a), TRef{}};
    }
    if (op == "Recv") {
      TRef gv = g.valid() ? g : zeros_like(out);
      Attrs a;
      a.set("channel", n.attrs.i("channel") ^ kGradChannel);
      a.set("peer", n.attrs.i("peer"));
      g_.op("Send", {gv, fwd(in[0])}, a);
      return none;
    }
    static const std::set<std::string> nograd = {
        "StopGradient", "Placeholder", "Const", "ZerosLike", "Less", "LessEqual", "Greater",
        "Equal", "LogicalAnd", "LogicalNot", "ReduceMax", "ReduceMin", "TACreate",
        "StackCreate", "StackPush", "StackPop", "TAGrad"};
    if (nograd.count(op)) return none;
    if (op == "Add") return {reduce_to(g, in[0], out), reduce_to(g, in[1], out)};
    if (op == "Sub") return {reduce_to(g, in[0], out), reduce_to(g_.op1("Neg", {g}), in[1], out)};
    if (op == "AddN") return std::vector<TRef>(in.size(), g);
    if (op == "Mul")
      return {reduce_to(g_.op1("Mul", {g, fwd(in[1])}), in[0], out),
              reduce_to(g_.op1("Mul", {g, fwd(in[0])}), in[1], out)};
    if (op == "Neg") return {g_.op1("Neg", {g})};
    if (op == "MatMul") {
      TRef x = fwd(in[0]), y = fwd(in[1]);
      bool ta = n.attrs.b("ta"), tb = n.attrs.b("tb");
      if (!ta && !tb) return {mm(g, y, false, true), mm(x, g, true, false)};
      if (ta && !tb) return {mm(y, g, false, true), mm(x, g, false, false)};
      if (!ta && tb) return {mm(g, y, false, false), mm(g, x, true, false)};
      return {mm(y, g, true, true), mm(g, x, true, true)};
    }
    if (op == "Transpose") return {g_.op1("Transpose", {g})};
    if (op == "BiasAdd") {
      Attrs a;
      a.set("axis", 0);
      return {g, g_.op1("ReduceSum", {g}, a)};
    }
    if (op == "ReduceSum") {
      if (n.attrs.i("axis", -1) == 0) throw CfError(CF_E_NO_GRADIENT, "ReduceSum(axis=0)");
      Attrs a;
      a.setv("shape", g_.shape(in[0]));
      return {g_.op1("Fill", {g}, a)};
    }
    if (op == "Fill") return {g_.op1("ReduceSum", {g})};
    if (op == "Sigmoid") {
      TRef y = fwd(out);
      return {g_.op1("Mul", {g, g_.op1("Mul", {y, g_.op1("Sub", {one(), y})})})};
    }
    if (op == "Tanh") {
      TRef y = fwd(out);
      return {g_.op1("Mul", {g, g_.op1("Sub", {one(), g_.op1("Mul", {y, y})})})};
    }
    if (op == "Relu") return {g_.op1("ReluGrad", {g, fwd(out)})};
    if (op == "Select") {
      TRef c = fwd(in[0]);
      TRef z = g_.op1("ZerosLike", {g});
      return {TRef{}, g_.op1("Select", {c, g, z}), g_.op1("Select", {c, z, g})};
    }
    if (op == "Concat") {
      int64_t ax = n.attrs.i("axis");
      std::vector<TRef> res;
      int64_t off = 0;
      for (auto& t : in) {
        Shape s = g_.shape(t);
        std::vector<int64_t> begin(s.size(), 0);
        begin[ax] = off;
        off += s[ax];
        Attrs a;
        a.setv("begin", begin);
        a.setv("size", s);
        res.push_back(g_.op1("Slice", {g}, a));
      }
      return res;
    }
    if (op == "Slice") {
      Attrs a;
      a.setv("shape", g_.shape(in[0]));
      a.setv("begin", n.attrs.v("begin"));
      a.setv("size", n.attrs.v("size"));
      return {g_.op1("SliceGrad", {g}, a)};
    }
    if (op == "Reshape") {
      Attrs a;
      a.setv("shape", g_.shape(in[0]));
      return {g_.op1("Reshape", {g}, a)};
    }
    if (op == "LSTMCell") {
      bool masked = n.attrs.b("masked");
      std::vector<TRef> ins{fwd(in[0]), fwd(in[1]), fwd(in[2]), fwd(in[3]), fwd(TRef{nid, 3})};
      if (masked) {
        ins.push_back(fwd(in[5]));
        ins.push_back(fwd(in[6]));
      }
      for (int p = 0; p < 3; ++p)
        ins.push_back(g_outs[p].valid() ? g_outs[p] : zeros_like(TRef{nid, p}));
      Attrs a;
      a.set("masked", masked);
      a.setf("forget_bias", n.attrs.f("forget_bias", 0.0));
      auto gr = g_.op("LSTMCellGrad", ins, a);
      std::vector<TRef> res{gr[0], gr[1], gr[2], gr[3], gr[4]};
      if (masked) {
        res.push_back(TRef{});
        res.push_back(TRef{});
      }
      return res;
    }
    if (op == "TARead") {
      auto gh = g_.op("TAGrad", {fwd(in[0]), fwd(in[2])});
      TRef wf = g_.op1("TAWrite", {gh[0], fwd(in[1]), g, gh[1]}, n.attrs);
      return {TRef{}, TRef{}, wf};
    }
    if (op == "TAWrite") {
      auto gh = g_.op("TAGrad", {fwd(in[0]), g});
      TRef gv = g_.op1("TARead", {gh[0], fwd(in[1]), gh[1]}, n.attrs);
      return {TRef{}, TRef{}, gv, g};
    }
    if (op == "TAStack") {
      auto gh = g_.op("TAGrad", {fwd(in[0]), fwd(in[1])});
      TRef uf = g_.op1("TAUnstack", {gh[0], g, gh[1]}, n.attrs);
      return {TRef{}, uf};
    }
    if (op == "TAUnstack") {
      auto gh = g_.op("TAGrad", {fwd(in[0]), g});
      TRef gv = g_.op1("TAStack", {gh[0], gh[1]}, n.attrs);
      return {TRef{}, gv, g};
    }
    throw CfError(CF_E_NO_GRADIENT, "no gradient for op " + op);
  }

 private:
  Graph& g_;
  std::map<int, int> mirror_;
  std::map<TRef, TRef> stack_of_, pop_of_;
};

}  // namespace

std::vector<TRef> gradients(Graph& g, TRef y, const std::vector<TRef>& xs) {
  if (!is_float(g.dtype(y)) || !g.shape(y).empty())
    throw CfError(CF_E_NONSCALAR_OBJECTIVE, "y must be a float scalar");
  if (g.ctx_of(y) != 0) throw CfError(CF_E_INVALID_GRAPH, "y must be in the root context");
  AD ad(g);
  CtxGuard guard(g, 0);
  float one = 1.0f;
  TRef seed = g.constant(g.dtype(y), {}, nullptr);
  if (g.dtype(y) == F32) std::memcpy(g.nodes[seed.node].data.data(), &one, 4);
  else {
    double d = 1.0;
    std::memcpy(g.nodes[seed.node].data.data(), &d, 8);
  }
  auto gd = ad.backprop(0, {{y, {seed}}}, xs);
  std::vector<TRef> res;
  for (auto& x : xs) res.push_back(gd.count(x) ? gd[x] : ad.zeros_like(x));
  return res;
}

}  // namespace cf
