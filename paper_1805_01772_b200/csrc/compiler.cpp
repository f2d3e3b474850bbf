// libcf device compiler: lowers a cf::Graph to the table the persistent driver kernel
// interprets (program.h).
//
// Every node becomes a device node. Control-flow primitives, integer/bool scalar ops,
// TensorArray and Stack ops are evaluated by the driver itself (device-resident control,
// north star subsystem (1)); float-tensor ops become "heavy" instances executed by the
// worker CTAs. Each heavy output gets a static placement:
//   * TA    -- written straight into the TensorArray slot its TAWrite targets (zero-copy
//              TensorArray write);
//   * ARENA -- one slot per iteration, for values that reach a StackPush: the stack then
//              holds pointers to immutable slots (the contiguous-array lowering of stacks
//              when "the loop variables have a static shape and the iteration count has a
//              static upper bound");
//   * RING  -- K+1 slots for everything else in a loop: the parallel_iterations window
//               guarantees a slot is dead before it is reused;
//   * ROOT  -- one buffer for values outside loops.
#include "compiler.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <set>
#include <sstream>

namespace cf {

using namespace cfdev;

namespace {

// gradient-loop steps accumulated per dW tile (K = 8 * batch). Measured on cfg3 (tools/
// dwchunk_ab.py): 1 step 113.8 ms, 2 94.6, 4 76.6, 8 72.7, 12 71.3-71.9, 16 72.3 -> 8 (the dz and
// swap-in rings grow by one slot per chunk step); kDwMax bounds it
constexpr int kDwChunk = 8;
static_assert(kDwChunk <= kDwMax, "dW chunk records");

int32_t dev_dt(int32_t d, int32_t precision) {
  (void)precision;
  switch (d) {
    case BOOL: return D_BOOL;
    case I32: return D_I32;
    case I64: return D_I64;
    case F32:
    case F64:
    case BF16: return D_F32;
    default: return D_NONE;
  }
}
int dev_size(int32_t d) {
  switch (d) {
    case D_BOOL: return 1;
    case D_I32: return 4;
    case D_I64: return 8;
    case D_F32: return 4;
    case D_BF16: return 2;
    default: return 0;
  }
}

struct Compiler {
  const Graph& g;
  CompileOpts o;
  HostProgram P;
  std::vector<int> vbase, ctrl_vid, frame_of;   // per node
  std::vector<bool> root_dead;                  // per node: root code nothing needs
  std::map<int, int> one_mul;                  // root Mul by a constant one -> kept input
  std::map<int, TRef> wt_root;                 // LSTMCellGrad node -> root value of its W
  std::map<int, int> wt_buf;                   // 2 W value id (+1 packed W) -> shared buffer
  std::map<int, int> wt_leader;                // 2 W value id (+1 packed W) -> preparing node
  std::vector<std::vector<std::pair<int, int>>> cons;   // per value: (consumer node, input idx)
  std::map<std::string, int> frame_id;
  std::vector<int> frame_ctx;
  std::vector<int> frame_parent;      // enclosing frame of each frame (-1: root context)
  std::vector<int64_t> frame_total;   // iteration indices over all instances of a frame
  std::map<int, int> ta_id;           // TACreate node -> ta id
  std::map<int, int> stack_id;        // StackCreate node -> stack id
  std::vector<std::vector<std::pair<int, int>>> extra_edges;   // per frame: (before, after)
  std::vector<uint8_t> vdt;           // device dtype per value id
  std::vector<int> ta_dt;             // device dtype per TensorArray
  std::map<int, int> acc_of_loopvar;  // loop Merge node -> acc id
  std::map<int, int> acc_of_add;      // fused Add node -> acc id
  std::map<std::pair<int, int>, int> acc_of_src;   // (LSTMCellGrad node, port) -> acc id
  std::vector<std::pair<int, int>> reg_bufs;       // (buffer id, registry index)
  bool bf16() const { return o.precision == CF_BF16; }

  Compiler(const Graph& gg, const CompileOpts& oo) : g(gg), o(oo) {}

  int vid(TRef t) const { return vbase[t.node] + t.port; }
  int32_t vdt_of(TRef t) const { return vdt[vid(t)]; }

  // handle -> creator node (TACreate / TAGrad / StackCreate) through routing
  int trace_creator(TRef h) const {
    for (int k = 0; k < 256; ++k) {
      const Node& n = g.nodes[h.node];
      if (n.op == "TACreate" || n.op == "StackCreate") return n.id;
      if (n.op == "TAGrad" && h.port == 0) return n.id;
      if (n.in.empty()) break;
      h = n.in[0];
    }
    return -1;
  }

  // Device dtypes (reading R16 / DESIGN.md "bf16 policy"): values connected through routing
  // (Switch/Merge/Enter/Exit/NextIteration/Identity), TensorArray slots and stacks share one
  // storage dtype; in bf16 mode the LSTM GEMM operands (x, h, gates, out) are bf16, every
  // other float (cell state c, gradients, accumulators, loss) stays fp32.
  void assign_dtypes() {
    const int N = (int)g.nodes.size();
    int nv = P.n_vids;
    int extra = (int)P.tas.size() + (int)P.stacks.size();
    std::vector<int> uf(nv + extra);
    for (size_t i = 0; i < uf.size(); ++i) uf[i] = (int)i;
    std::function<int(int)> find = [&](int x) { return uf[x] == x ? x : uf[x] = find(uf[x]); };
    auto unite = [&](int a, int b) { uf[find(a)] = find(b); };
    auto ta_cls = [&](int ta) { return nv + ta; };
    auto st_cls = [&](int sid) { return nv + (int)P.tas.size() + sid; };
    for (int i = 0; i < N; ++i) {
      const Node& n = g.nodes[i];
      const std::string& op = n.op;
      int o0 = vbase[i];
      if (op == "Identity" || op == "StopGradient" || op == "Reshape" || op == "Enter" ||
          op == "Exit" || op == "NextIteration" ||
          (op == "Cast" && is_float(n.odt[0]) && is_float(g.dtype(n.in[0]))))
        unite(vid(n.in[0]), o0);
      else if (op == "Switch") {
        unite(vid(n.in[0]), o0);
        unite(vid(n.in[0]), o0 + 1);
      } else if (op == "Merge") {
        unite(vid(n.in[0]), o0);
        unite(vid(n.in[1]), o0);
      } else if (op == "TAWrite" || op == "TARead" || op == "TAUnstack" || op == "TAStack") {
        int ta = trace_ta(n.in[0]);
        if (op == "TAWrite") unite(vid(n.in[2]), ta_cls(ta));
        if (op == "TARead" || op == "TAStack") unite(o0, ta_cls(ta));
        if (op == "TAUnstack") unite(vid(n.in[1]), ta_cls(ta));
      } else if (op == "StackPush" || op == "StackPop") {
        int c = trace_creator(n.in[0]);
        if (c >= 0 && stack_id.count(c)) {
          int sid = stack_id.at(c);
          unite(op == "StackPush" ? vid(n.in[1]) : o0, st_cls(sid));
        }
      }
    }
    std::vector<uint8_t> want(uf.size(), 0);
    if (bf16()) {
      for (int i = 0; i < N; ++i) {
        const Node& n = g.nodes[i];
        if (n.op == "LSTMCell") {
          for (int j : {0, 1}) want[find(vid(n.in[j]))] = 1;
          for (int p : {0, 2, 3}) want[find(vbase[i] + p)] = 1;
        } else if (n.op == "LSTMCellGrad") {
          for (int j : {0, 1, 4}) want[find(vid(n.in[j]))] = 1;
        } else if (n.op == "MatMul" && std::getenv("CF_NO_TC_MATMUL") == nullptr) {
          // generic GEMM operands (the MoE-style experts and their gradients) stored in bf16:
          // TMA operands of the tcgen05 GEMM (runtime.cu HK_MATMUL_TC); fp32 accumulation
          for (int j : {0, 1}) want[find(vid(n.in[j]))] = 1;
        }
      }
    }
    vdt.assign(nv, D_NONE);
    for (int i = 0; i < N; ++i) {
      const Node& n = g.nodes[i];
      for (size_t p = 0; p < n.odt.size(); ++p) {
        int v = vbase[i] + (int)p;
        int32_t d = n.odt[p];
        vdt[v] = is_float(d) ? (want[find(v)] ? D_BF16 : D_F32) : (uint8_t)dev_dt(d, o.precision);
      }
    }
    ta_dt.assign(P.tas.size(), D_F32);
    for (size_t t = 0; t < P.tas.size(); ++t) {
      int32_t gd = P.tas[t].dt;   // graph dtype stored temporarily
      ta_dt[t] = is_float(gd) ? (want[find(ta_cls((int)t))] ? D_BF16 : D_F32) : dev_dt(gd, o.precision);
    }
  }
  bool is_heavy(const Node& n) const {
    if (n.op == "Placeholder" || n.op == "Const" || n.op == "Identity" || n.op == "StopGradient" ||
        n.op == "Reshape" || n.op == "Switch" || n.op == "Merge" || n.op == "Enter" ||
        n.op == "Exit" || n.op == "NextIteration" || n.op.rfind("TA", 0) == 0 ||
        n.op.rfind("Stack", 0) == 0)
      return false;
    for (auto d : n.odt)
      if (is_float(d)) return true;
    return false;
  }

  [[noreturn]] void unsupported(const Node& n, const std::string& why) {
    throw CfError(CF_E_UNSUPPORTED, "device compiler: node " + std::to_string(n.id) + " (" +
                                        n.op + "): " + why);
  }

  int add_buf(size_t bytes, bool zero, const std::string& what, const void* init = nullptr) {
    BufPlan b;
    b.bytes = std::max<size_t>(bytes, 16);
    b.zero = zero;
    b.what = what;
    if (init) {
      b.init.resize(bytes);
      std::memcpy(b.init.data(), init, bytes);
    }
    P.bufs.push_back(std::move(b));
    return (int)P.bufs.size() - 1;
  }

  // root value of a tensor-core LSTMCellGrad node's weight (-1: not a root value). The weight
  // reaches the gradient loop through a stack (autodiff saves the forward body's Enter'ed W,
  // PAPER.md:416-420): follow the pop to its pushes, and the pushed value through Switch /
  // Identity / Enter to the root value (all pushes must agree)
  TRef weight_root(const Node& n) {
    auto stack_of = [&](TRef h) -> int {
      for (int k = 0; k < 64; ++k) {
        const Node& hn = g.nodes[h.node];
        if (hn.op == "StackCreate") return hn.id;
        if (hn.in.empty()) return -1;
        h = hn.in[0];
      }
      return -1;
    };
    std::function<TRef(TRef, int)> root_of = [&](TRef v, int depth) -> TRef {
      for (int k = 0; k < 64 && v.node >= 0 && depth < 4; ++k) {
        const Node& m = g.nodes[v.node];
        if (frame_of[m.id] < 0 && m.op != "Exit") return v;
        if (m.op == "Enter" || m.op == "Identity" || m.op == "Switch") {
          v = m.in[0];
        } else if (m.op == "StackPop") {
          const int sid = stack_of(m.in[0]);
          TRef r{-1, 0};
          for (auto& q : g.nodes)
            if (q.op == "StackPush" && stack_of(q.in[0]) == sid) {
              const TRef rq = root_of(q.in[1], depth + 1);
              if (rq.node < 0 || (r.node >= 0 && !(rq == r))) return TRef{-1, 0};
              r = rq;
            }
          return r;
        } else {
          return TRef{-1, 0};
        }
      }
      return TRef{-1, 0};
    };
    return root_of(n.in[3], 0);
  }

  // trace a TensorArray handle back to its static TA id
  int trace_ta(TRef h, int depth = 0) {
    if (depth > 64) throw CfError(CF_E_UNSUPPORTED, "TensorArray handle routing too deep");
    const Node& n = g.nodes[h.node];
    if (n.op == "TACreate") return ta_id.at(n.id);
    if (n.op == "TAGrad") {
      int f = trace_ta(n.in[0], depth + 1);
      return P.tas[f].grad_id;
    }
    if (n.op == "Enter" || n.op == "Identity" || n.op == "Switch" || n.op == "Exit" ||
        n.op == "NextIteration")
      return trace_ta(n.in[0], depth + 1);
    if (n.op == "Merge") return trace_ta(n.in[0], depth + 1);
    throw CfError(CF_E_UNSUPPORTED, "TensorArray handle from op " + n.op);
  }

  void run(const std::vector<TRef>& fetches) {
    const int N = (int)g.nodes.size();
    vbase.resize(N);
    ctrl_vid.resize(N);
    int nv = 0;
    for (int i = 0; i < N; ++i) {
      vbase[i] = nv;
      nv += (int)g.nodes[i].odt.size();
    }
    for (int i = 0; i < N; ++i) ctrl_vid[i] = nv++;
    P.n_vids = nv;
    cons.assign(nv, {});
    for (auto& n : g.nodes)
      for (size_t j = 0; j < n.in.size(); ++j) cons[vid(n.in[j])].push_back({n.id, (int)j});

    // ---- frames
    frame_of.assign(N, -1);
    for (auto& name : g.frame_order) {
      int c = g.whiles.at(name);
      frame_id[name] = (int)frame_ctx.size();
      frame_ctx.push_back(c);
      P.frame_names.push_back(name);
    }
    // a while_loop nested in another one's body: a
    // frame instance per iteration of the enclosing frame, run by the driver as one step of
    // the enclosing body (runtime.cu OP_FRAME)
    frame_parent.assign(frame_ctx.size(), -1);
    for (size_t f = 0; f < frame_ctx.size(); ++f) {
      const int pw = g.enclosing_while(g.ctxs[frame_ctx[f]].parent);
      if (pw >= 0) {
        frame_parent[f] = frame_id.at(g.ctxs[pw].name);
        P.nested = true;
        if (o.stack_budget_bytes >= 0)
          throw CfError(CF_E_UNSUPPORTED, "stack swapping with nested while_loops");
      }
    }
    for (auto& n : g.nodes) {
      int w = g.enclosing_while(n.ctx);
      if (w >= 0) frame_of[n.id] = frame_id.at(g.ctxs[w].name);
    }
    extra_edges.assign(frame_ctx.size() + 1, {});

    // ---- TensorArrays and stacks
    for (auto& n : g.nodes) {
      if (n.op == "TACreate") {
        DTA t{};
        t.size = (int32_t)n.attrs.i("size");
        t.dt = (int32_t)n.attrs.i("dtype");   // graph dtype until assign_dtypes()
        t.elem_bytes = numel(n.attrs.v("elem_shape"));   // elements until assign_dtypes()
        t.grad_id = -1;
        ta_id[n.id] = (int)P.tas.size();
        P.tas.push_back(t);
        ta_shape.push_back(n.attrs.v("elem_shape"));
      }
    }
    for (auto& n : g.nodes) {
      if (n.op == "TAGrad") {
        int f = trace_ta(n.in[0]);
        if (P.tas[f].grad_id < 0) {
          DTA t = P.tas[f];
          t.is_grad = 1;
          t.grad_id = -1;
          P.tas[f].grad_id = (int)P.tas.size();
          P.tas.push_back(t);
          ta_shape.push_back(ta_shape[f]);
        }
      }
    }
    // stack ids (capacity set after bounds)
    for (auto& n : g.nodes)
      if (n.op == "StackCreate") {
        stack_id[n.id] = (int)P.stacks.size();
        P.stacks.push_back(DStack{});
      }
    assign_dtypes();
    for (size_t k = 0; k < P.tas.size(); ++k) {
      DTA& t = P.tas[k];
      t.dt = ta_dt[k];
      t.elem_bytes *= dev_size(t.dt);
      t.base = add_buf((size_t)t.size * t.elem_bytes, t.is_grad != 0,
                       std::string(t.is_grad ? "grad " : "") + "TensorArray " + std::to_string(k));
      if (t.dt == D_BF16) register_buf((int)t.base, t.size, ta_rows_cols(k));
    }
    int slot_total = 0;
    for (auto& t : P.tas) slot_total += t.size;
    P.ta_slots = slot_total;

    // ---- frame bounds (iteration upper bound from TensorArray sizes, or opts)
    std::vector<int64_t> bound(frame_ctx.size(), 0);
    for (auto& n : g.nodes) {
      int f = frame_of[n.id];
      if (f < 0) continue;
      if (n.op == "TARead" || n.op == "TAWrite")
        bound[f] = std::max<int64_t>(bound[f], P.tas[trace_ta(n.in[0])].size);
    }
    for (size_t f = 0; f < frame_ctx.size(); ++f) {
      if (o.max_iterations > 0) bound[f] = o.max_iterations;
      if (bound[f] <= 0)
        throw CfError(CF_E_UNSUPPORTED, "cannot bound iterations of frame " + P.frame_names[f] +
                                            " (no TensorArray; set max_iterations)");
    }
    // a nested frame's iteration indices run on over its instances (one instance per
    // iteration of the enclosing frame): arenas and stack instances are indexed by them
    frame_total.assign(frame_ctx.size(), 0);
    std::function<int64_t(int)> total_of = [&](int f) -> int64_t {
      if (frame_total[f] > 0) return frame_total[f];
      return frame_total[f] = bound[f] * (frame_parent[f] >= 0 ? total_of(frame_parent[f]) : 1);
    };
    for (size_t f = 0; f < frame_ctx.size(); ++f) total_of((int)f);
    for (auto& n : g.nodes) {
      if (n.op == "StackCreate") {
        DStack& s = P.stacks[stack_id.at(n.id)];
        auto it = frame_id.find(n.attrs.s("frame"));
        if (it == frame_id.end()) unsupported(n, "stack of unknown frame");
        s.capacity = (int32_t)bound[it->second];
        // created once per iteration of the frame around it (a nested loop's stack): one
        // instance per iteration index of that frame
        s.instances = frame_of[n.id] >= 0 ? (int32_t)frame_total[frame_of[n.id]] : 1;
        s.entry_off = P.stack_pool;
        s.depth_off = P.stack_depths;
        P.stack_pool += s.capacity * s.instances;
        P.stack_depths += s.instances;
      }
    }
    // ---- root algebra: 1 * v is v exactly. autodiff's gradient of a loss term sum(R * out)
    // is Fill(dy) * R with dy the seed 1: the Mul becomes a view of R and the Fill dies below
    auto is_one = [&](TRef t, auto&& self) -> bool {
      const Node& n = g.nodes[t.node];
      if (n.op == "Fill" || n.op == "Identity") return self(n.in[0], self);
      if (n.op != "Const" || !g.shape(t).empty()) return false;
      if (n.odt[0] == F32 && n.data.size() == 4) {
        float v;
        std::memcpy(&v, n.data.data(), 4);
        return v == 1.0f;
      }
      if (n.odt[0] == F64 && n.data.size() == 8) {
        double v;
        std::memcpy(&v, n.data.data(), 8);
        return v == 1.0;
      }
      return false;
    };
    for (auto& n : g.nodes) {
      if (n.op != "Mul" || frame_of[n.id] >= 0) continue;
      for (int j = 0; j < 2; ++j)
        if (is_one(n.in[j], is_one) && g.shape(n.in[1 - j]) == n.osh[0] &&
            g.dtype(n.in[1 - j]) == n.odt[0]) {
          one_mul[n.id] = 1 - j;
          break;
        }
    }
    // ---- root dead-code elimination: a side-effect-free root op none of whose results reaches
    // a fetch, a frame or an effectful op is never evaluated (e.g. the gradients autodiff
    // builds for inputs nobody asked for: d R_out = dy * out of a Mul in the loss)
    root_dead.assign(N, false);
    {
      static const std::set<std::string> pure = {
          "Mul", "Add", "Sub", "Neg", "Fill", "ReduceSum", "ReduceMax", "ReduceMin", "MatMul",
          "Tanh", "Sigmoid", "Relu", "Const", "Identity", "Cast", "Transpose", "BiasAdd", "AddN",
          "ZerosLike", "Less", "LessEqual", "Greater", "Equal", "LogicalAnd", "LogicalNot",
          "Reshape", "Slice"};
      std::vector<char> live(N, 0);
      std::vector<int> work;
      auto mark = [&](int x) {
        if (!live[x]) { live[x] = 1; work.push_back(x); }
      };
      for (auto& t : fetches) mark(t.node);
      for (auto& n : g.nodes)
        if (frame_of[n.id] >= 0 || n.op == "Exit" || !pure.count(n.op)) mark(n.id);
      while (!work.empty()) {
        const int x = work.back();
        work.pop_back();
        auto om = one_mul.find(x);
        if (om != one_mul.end()) {   // only the operand the view keeps
          mark(g.nodes[x].in[om->second].node);
          continue;
        }
        for (auto& t : g.nodes[x].in) mark(t.node);
        for (int c : g.nodes[x].ctrl) mark(c);
      }
      for (int i = 0; i < N; ++i) root_dead[i] = !live[i];
    }
    detect_accumulators();
    fuse_dout_sums();

    // ---- device nodes
    P.nodes.resize(N);
    int max_cond = -1;
    std::vector<int> heavy_nodes;
    for (auto& n : g.nodes) {
      DNode d{};
      d.n_in = (int)n.in.size();
      d.in_off = (int)P.in_vids.size();
      auto fz = fused_dout.find(n.id);
      auto om = one_mul.find(n.id);
      if (om != one_mul.end()) {   // 1 * v: a view of v
        d.n_in = 1;
        P.in_vids.push_back(vid(n.in[om->second]));
      } else if (fz == fused_dout.end()) {
        for (auto& t : n.in) P.in_vids.push_back(vid(t));
      } else {
        // LSTMCellGrad with its dout AddN folded in: dout = AddN input 0, the other AddN
        // inputs appended after the regular inputs (aux5 = how many)
        const Node& an = g.nodes[fz->second];
        const int o = n.attrs.b("masked") ? 7 : 5;
        for (size_t j = 0; j < n.in.size(); ++j)
          P.in_vids.push_back(vid((int)j == o + 2 ? an.in[0] : n.in[j]));
        for (size_t j = 1; j < an.in.size(); ++j) P.in_vids.push_back(vid(an.in[j]));
        d.n_in = (int)(n.in.size() + an.in.size() - 1);
      }
      d.n_ctrl = (int)n.ctrl.size();
      d.ctrl_off = (int)P.in_vids.size();
      for (int c : n.ctrl) P.in_vids.push_back(ctrl_vid[c]);
      d.n_out = (int)n.odt.size();
      d.out_vid = vbase[n.id];
      d.ctrl_vid = ctrl_vid[n.id];
      d.place_off = -1;
      for (auto& a : d.aux) a = 0;
      const std::string& op = n.op;
      int32_t odt = n.odt.empty() ? -1 : n.odt[0];
      if (op == "Placeholder") {
        d.op = OP_PLACEHOLDER;
        FeedInfo fi;
        fi.vid = vbase[n.id];
        fi.graph_dt = odt;
        fi.dev_dt = vdt[vbase[n.id]];
        fi.bytes = numel(n.osh[0]) * dev_size(fi.dev_dt);
        fi.scalar_ctrl = !is_float(odt) && n.osh[0].empty();
        P.feeds[n.attrs.s("name")] = fi;
      } else if (op == "Const") {
        d.op = OP_CONST;
        if (odt == FLOW || odt == RES) {
          d.op = OP_FLOW;
        } else if (!is_float(odt) && n.osh[0].empty()) {
          d.aux[0] = 1;
          int64_t v = 0;
          if (odt == I64) std::memcpy(&v, n.data.data(), 8);
          else if (odt == I32) { int32_t x; std::memcpy(&x, n.data.data(), 4); v = x; }
          else if (odt == BOOL) v = n.data[0] != 0;
          d.imm[0] = v;
          d.aux[1] = dev_dt(odt, o.precision);
        } else {
          int32_t dd = vdt[vbase[n.id]];
          int64_t ne = numel(n.osh[0]);
          std::vector<uint8_t> bytes((size_t)ne * dev_size(dd));
          for (int64_t k = 0; k < ne && is_float(odt); ++k) {
            float f;
            if (odt == F64) {
              double x;
              std::memcpy(&x, n.data.data() + 8 * k, 8);
              f = (float)x;
            } else {
              std::memcpy(&f, n.data.data() + 4 * k, 4);
            }
            if (dd == D_BF16) {
              uint32_t u;
              std::memcpy(&u, &f, 4);
              u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16;
              uint16_t h = (uint16_t)u;
              std::memcpy(bytes.data() + 2 * k, &h, 2);
            } else {
              std::memcpy(bytes.data() + 4 * k, &f, 4);
            }
          }
          if (!is_float(odt)) std::memcpy(bytes.data(), n.data.data(), std::min(bytes.size(), n.data.size()));
          d.aux[0] = 0;
          d.aux[1] = dd;
          d.imm[0] = add_buf(bytes.size(), false, "const " + std::to_string(n.id), bytes.data());
          if (dd == D_BF16 && n.osh[0].size() >= 2) register_shape((int)d.imm[0], n.osh[0], 1);
        }
      } else if (op == "Identity" || op == "StopGradient" || op == "Reshape" ||
                 (op == "Cast" && is_float(odt) && is_float(g.dtype(n.in[0]))) ||
                 one_mul.count(n.id)) {
        d.op = OP_PASS;
      } else if (op == "Switch") {
        d.op = OP_SWITCH;
        d.aux[0] = n.attrs.has("cond_id") ? (int)n.attrs.i("cond_id") : -1;
        d.aux[1] = n.attrs.b("loop");
        if (d.aux[0] > max_cond) max_cond = d.aux[0];
      } else if (op == "Merge") {
        if (n.attrs.b("loop")) {
          d.op = OP_MERGE_LOOP;
          d.aux[0] = frame_id.at(n.attrs.s("frame"));
        } else {
          d.op = OP_MERGE;
        }
      } else if (op == "Enter") {
        d.op = OP_ENTER;
        d.aux[0] = frame_id.at(n.attrs.s("frame"));
      } else if (op == "Exit") {
        d.op = OP_EXIT;
        d.aux[0] = frame_id.at(n.attrs.s("frame"));
      } else if (op == "NextIteration") {
        d.op = OP_NEXTITER;
        d.aux[0] = frame_id.at(n.attrs.s("frame"));
      } else if (op == "TACreate") {
        d.op = OP_TA_CREATE;
        d.aux[0] = ta_id.at(n.id);
      } else if (op == "TARead") {
        d.op = OP_TA_READ;
      } else if (op == "TAWrite") {
        d.op = OP_TA_WRITE;
      } else if (op == "TAStack") {
        d.op = OP_TA_STACK;
      } else if (op == "TAUnstack") {
        d.op = OP_TA_UNSTACK;
      } else if (op == "TAGrad") {
        d.op = OP_TA_GRAD;
        d.aux[0] = trace_ta(TRef{n.id, 0});
      } else if (op == "StackCreate") {
        d.op = OP_STACK_CREATE;
        d.aux[0] = stack_id.at(n.id);
      } else if (op == "StackPush") {
        d.op = OP_STACK_PUSH;
      } else if (op == "StackPop") {
        d.op = OP_STACK_POP;
      } else if (op == "Send" || op == "Recv") {
        d.op = op == "Send" ? OP_SEND : OP_RECV;
        d.aux[0] = add_chan(n);
        if (op == "Recv") heavy_nodes.push_back(n.id);   // output placed like a heavy output
      } else if (odt == FLOW) {
        d.op = OP_FLOW;
      } else if (fused_addn.count(n.id) || root_dead[n.id]) {
        // folded into its LSTMCellGrad consumer (not in any body program), or dead root code
      } else if (acc_of_add.count(n.id)) {
        d.op = OP_ACC;
        d.aux[0] = acc_of_add.at(n.id);
      } else if (!is_heavy(n)) {
        // integer / bool control arithmetic on the device driver
        bool all_scalar = true;
        for (auto& t : n.in) all_scalar &= g.shape(t).empty();
        if (op == "ReduceMax" || op == "ReduceMin") {
          if (g.shape(n.in[0]).size() != 1) unsupported(n, "integer reduction of rank != 1");
          d.op = OP_REDUCE_I;
          d.aux[0] = op == "ReduceMin";
          d.aux[1] = (int)g.shape(n.in[0])[0];
          d.aux[2] = dev_dt(g.dtype(n.in[0]), o.precision);
        } else if (op == "Slice" && g.shape(n.in[0]).size() == 1) {
          d.op = OP_SLICE_I;
          int32_t dd = dev_dt(g.dtype(n.in[0]), o.precision);
          d.imm[0] = n.attrs.v("begin").at(0) * dev_size(dd);
          d.aux[1] = dd;
        } else if (all_scalar) {
          d.op = OP_SCALAR;
          static const std::map<std::string, int> sc = {
              {"Add", SC_ADD}, {"Sub", SC_SUB}, {"Mul", SC_MUL}, {"Less", SC_LESS},
              {"LessEqual", SC_LEQ}, {"Greater", SC_GREATER}, {"Equal", SC_EQ},
              {"LogicalAnd", SC_AND}, {"LogicalNot", SC_NOT}, {"Cast", SC_CAST}};
          auto it = sc.find(op);
          if (it == sc.end()) unsupported(n, "integer op not lowered");
          d.aux[0] = it->second;
          d.aux[1] = dev_dt(odt, o.precision);
        } else {
          unsupported(n, "non-scalar integer/bool tensor op");
        }
      } else {
        d.op = OP_HEAVY;
        heavy_nodes.push_back(n.id);
        lower_heavy(n, d);
        if (fused_dout.count(n.id)) d.aux[5] = (int)g.nodes[fused_dout.at(n.id)].in.size() - 1;
      }
      P.nodes[n.id] = d;
    }
    P.n_conds = max_cond + 1;

    // ---- placements of heavy outputs
    P.dw_chunk = bf16() ? kDwChunk : 1;
    if (const char* e = std::getenv("CF_DW_CHUNK"); e && bf16())   // A/B (tools/dwchunk_ab.py)
      P.dw_chunk = std::max(1, std::min(kDwMax, std::atoi(e)));
    // weights of the tensor-core LSTM nodes: the nodes of one root weight (a layer's masked and
    // unmasked cells) share one prepared buffer (packed W forward, W^T backward) and one
    // preparation, issued as a root step (kRootPrep)
    if (bf16() && std::getenv("CF_NO_ROOT_HINTS") == nullptr)
      for (int nid : heavy_nodes) {
        const Node& n = g.nodes[nid];
        if ((n.op != "LSTMCellGrad" && n.op != "LSTMCell") || frame_of[nid] < 0) continue;
        const TRef w = weight_root(n);
        if (w.node < 0 || frame_of[w.node] >= 0 || g.nodes[w.node].op == "Exit") continue;
        wt_root[nid] = w;
        const int key = 2 * vid(w) + (n.op == "LSTMCell" ? 1 : 0);   // W^T or packed W of it
        if (!wt_leader.count(key)) wt_leader[key] = nid;
        // low 32 bits: root W value id + 1; high 32: the node whose preparation it shares + 1
        P.nodes[nid].imm[3] = (int64_t)(vid(w) + 1) | ((int64_t)(wt_leader.at(key) + 1) << 32);
      }
    for (int nid : heavy_nodes) place_outputs(g.nodes[nid]);

    // ---- evaluation orders
    build_orders(bound);

    // ---- fetches
    for (auto& t : fetches) {
      FetchInfo fi;
      fi.vid = vid(t);
      fi.dev_dt = vdt[fi.vid];
      fi.bytes = numel(g.shape(t)) * dev_size(fi.dev_dt);
      P.fetches.push_back(fi);
      P.fetch_vids.push_back(fi.vid);
    }

    // ---- bounds for runtime pools
    int64_t per_iter_heavy = 0, root_heavy = 0, max_tiles = 1;
    std::vector<int64_t> frame_heavy(frame_ctx.size(), 0);
    for (int nid : heavy_nodes) {
      int f = frame_of[nid];
      int k = g.nodes[nid].op == "LSTMCellGrad" ? 3 : xproj(g.nodes[nid]) ? 2 : 1;
      if (g.nodes[nid].op == "AddN" && g.nodes[nid].in.size() > 8)   // a chain of 8-input sums
        k = 1 + (int)((g.nodes[nid].in.size() - 8 + 6) / 7);
      if (f >= 0) frame_heavy[f] += k + 4;
      else root_heavy += k + 1;
    }
    for (auto& n : g.nodes)
      if (n.op == "TAWrite" || n.op == "TAStack" || n.op == "TAUnstack" || n.op == "Send") {
        int f = frame_of[n.id];
        if (f >= 0) frame_heavy[f] += 2;
        else root_heavy += 2;
      }
    int64_t total = root_heavy + 64 + (int64_t)fetches.size() + 2 * (int64_t)heavy_nodes.size() +
                    2 * (int64_t)P.accs.size();
    for (size_t f = 0; f < frame_ctx.size(); ++f)
      total += frame_heavy[f] * (frame_total[f] + (frame_parent[f] >= 0 ? frame_total[frame_parent[f]] : 1));
    (void)per_iter_heavy;
    (void)max_tiles;
    P.inst_bound = total + 1024;
    P.branch_bound = 1;
    // branch bits are indexed by the iteration index over all instances of a nested frame
    for (size_t f = 0; f < bound.size(); ++f)
      P.branch_bound = (int)std::max<int64_t>(P.branch_bound, frame_total[f] + 1);

    // ---- describe
    std::ostringstream ds;
    ds << "nodes=" << N << " values=" << P.n_vids << " frames=" << frame_ctx.size()
       << " tas=" << P.tas.size() << " stacks=" << P.stacks.size()
       << " heavy_nodes=" << heavy_nodes.size() << " inst_bound=" << P.inst_bound << "\n";
    size_t tot = 0;
    for (auto& b : P.bufs) tot += b.bytes;
    ds << "device bytes=" << tot << " buffers=" << P.bufs.size() << "\n";
    for (size_t f = 0; f < frame_ctx.size(); ++f)
      ds << "frame " << P.frame_names[f] << " K=" << P.frames[f].K << " bound=" << bound[f]
         << " body=" << P.frames[f].n_body << "\n";
    int counts[6] = {0, 0, 0, 0, 0, 0};
    for (auto& pl : P.places) counts[pl.kind]++;
    ds << "accumulators=" << P.accs.size() << " tma_operands=" << P.reg.size() << "\n";
    ds << "structured frames=" << P.structured_frames << " cond contexts="
       << (P.ctxs.empty() ? 0 : P.ctxs.size() - 1) << " waves=" << P.n_waves
       << " heavy_batches=" << P.n_batches << (P.nested ? " nested_frames=1" : "") << "\n";
    ds << "stacks: resident bytes=" << P.stack_resident_bytes << " swapped arenas=" << P.swaps.size()
       << " swapped bytes=" << P.stack_swapped_bytes << "\n";
    ds << "placements root=" << counts[0] << " ring=" << counts[1] << " arena=" << counts[2]
       << " ta=" << counts[3] << " acc=" << counts[4] << "\n";
    P.describe = ds.str();
  }

  // one half of a Send/Recv channel. Both partitions derive slots and payload bytes the same
  // way (K + 1 slots of the enclosing loop, payload = value shape x device dtype); the runtime
  // checks that the halves agree when the peers connect.
  int add_chan(const Node& n) {
    const bool send = n.op == "Send";
    ChanPlan c;
    c.channel = (int32_t)n.attrs.i("channel");
    c.role = send ? 1 : 0;
    c.peer = (int32_t)n.attrs.i("peer");
    c.frame = frame_of[n.id];
    for (auto& o : P.chans)
      if (o.channel == c.channel && o.role == c.role)
        unsupported(n, "channel " + std::to_string(c.channel) + " used twice in one partition");
    int K = 0;
    if (c.frame >= 0) K = o.parallel_iterations > 0 ? o.parallel_iterations : g.ctxs[frame_ctx[c.frame]].K;
    c.slots = K + 1;
    int v = send ? vid(n.in[0]) : vbase[n.id];
    c.dt = vdt[v];
    const Shape& sh = send ? g.shape(n.in[0]) : n.osh[0];
    c.elem_bytes = numel(sh) * dev_size(c.dt);
    const int64_t flags = ((int64_t)c.slots * 8 + 255) / 256 * 256;
    c.bytes = send ? flags + 256 : flags + (int64_t)c.slots * ((c.elem_bytes + 255) / 256 * 256);
    c.offset = P.chan_bytes;
    P.chan_bytes += c.bytes;
    P.chans.push_back(c);
    return (int)P.chans.size() - 1;
  }

  void lower_heavy(const Node& n, DNode& d) {
    const std::string& op = n.op;
    auto ew = [&](int sub) {
      d.aux[0] = HK_EW;
      d.aux[1] = sub;
      d.imm[0] = numel(n.osh[0]);
      int flags = 0;
      for (size_t j = 0; j < n.in.size() && j < 8; ++j)
        if (g.shape(n.in[j]).empty() && !n.osh[0].empty()) flags |= 1 << j;
      d.aux[2] = flags;
    };
    if (op == "Add") return ew(EW_ADD);
    if (op == "Sub") return ew(EW_SUB);
    if (op == "Mul") return ew(EW_MUL);
    if (op == "Neg") return ew(EW_NEG);
    if (op == "Sigmoid") return ew(EW_SIGMOID);
    if (op == "Tanh") return ew(EW_TANH);
    if (op == "Relu") return ew(EW_RELU);
    if (op == "ReluGrad") return ew(EW_RELUGRAD);
    if (op == "ZerosLike") return ew(EW_ZEROS);
    if (op == "AddN") return ew(EW_ADDN);   // > 8 inputs: a chain of instances (runtime.cu)
    if (op == "BiasAdd") {
      ew(EW_BIASADD);
      d.imm[1] = n.osh[0].at(1);
      return;
    }
    if (op == "Select") {
      ew(EW_SELECT);
      d.imm[1] = g.shape(n.in[0]).empty() ? 0 : (n.osh[0].size() == 2 && g.shape(n.in[0]).size() == 1
                                                     ? n.osh[0][1] : 1);
      d.aux[3] = g.shape(n.in[0]).empty() ? 1 : 0;
      return;
    }
    if (op == "Fill") {
      d.aux[0] = HK_FILL;
      d.imm[0] = numel(n.osh[0]);
      return;
    }
    if (op == "ReduceSum") {
      if (n.attrs.i("axis", -1) == 0) {
        auto s = g.shape(n.in[0]);
        if (s.size() != 2) unsupported(n, "ReduceSum(axis=0) needs rank 2");
        d.aux[0] = HK_REDUCE_SUM0;
        d.imm[0] = s[0];
        d.imm[1] = s[1];
      } else {
        d.aux[0] = HK_REDUCE_SUM;
        d.imm[0] = numel(g.shape(n.in[0]));
      }
      return;
    }
    if (op == "MatMul") {
      d.aux[0] = HK_MATMUL;
      d.aux[1] = (n.attrs.b("ta") ? 1 : 0) | (n.attrs.b("tb") ? 2 : 0);
      auto sa = g.shape(n.in[0]), sb = g.shape(n.in[1]);
      d.imm[0] = n.osh[0][0];
      d.imm[1] = n.osh[0][1];
      d.imm[2] = n.attrs.b("ta") ? sa[0] : sa[1];
      d.imm[3] = sa[1] | (sb[1] << 32);   // leading dims of A and B
      return;
    }
    if (op == "LSTMCell" || op == "LSTMCellGrad") {
      if (bf16()) {
        int64_t I = g.shape(n.in[0])[1], H = g.shape(n.in[1])[1];
        if (I % 256 != 0 || H % 256 != 0)
          unsupported(n, "bf16 tcgen05 LSTM path needs input and hidden sizes that are multiples "
                         "of 256 (use CF_F32 for other shapes)");
      }
      d.aux[0] = op == "LSTMCell" ? HK_LSTM_FWD : HK_LSTM_BWD_EW;
      d.aux[1] = n.attrs.b("masked") | (xproj(n) ? 4 : 0);   // bit 2: x-projection split
      d.imm[0] = g.shape(n.in[0])[0];
      d.imm[1] = g.shape(n.in[0])[1];
      d.imm[2] = g.shape(n.in[1])[1];
      double fb = n.attrs.f("forget_bias", 0.0);
      float ff = (float)fb;
      int32_t fbits;
      std::memcpy(&fbits, &ff, 4);
      d.aux[2] = fbits;
      d.aux[3] = acc_of_src.count({n.id, 3}) ? acc_of_src.at({n.id, 3}) : -1;
      d.aux[4] = acc_of_src.count({n.id, 4}) ? acc_of_src.at({n.id, 4}) : -1;
      return;
    }
    unsupported(n, "float op not lowered");
  }

  // routing closure of a value through control-flow primitives and views
  void closure(int v0, bool* pinned, int* ta_write, int frame) {
    std::set<int> seen{v0};
    std::vector<std::pair<int, bool>> st{{v0, true}};   // (vid, same iteration)
    *pinned = false;
    *ta_write = -1;
    while (!st.empty()) {
      auto [v, same] = st.back();
      st.pop_back();
      for (auto [c, idx] : cons[v]) {
        const Node& cn = g.nodes[c];
        const std::string& op = cn.op;
        if (op == "StackPush" && idx == 1) *pinned = true;
        if (op == "TAWrite" && idx == 2 && same && frame_of[c] == frame && *ta_write < 0)
          *ta_write = c;
        // Enter too: a value entering a nested frame (f2) may reach a StackPush there (e.g. a
        // loop variable's initial value, pushed in the inner frame's first iteration); it must
        // then live in an immutable arena slot, not the enclosing frame's ring
        bool route = op == "Identity" || op == "StopGradient" || op == "Reshape" ||
                     op == "Switch" || op == "Merge" || op == "NextIteration" || op == "Exit" ||
                     op == "Enter";
        if (!route || (op == "Switch" && idx != 0)) continue;
        bool nsame = same && op != "NextIteration" && op != "Exit" && op != "Enter";
        for (int p = 0; p < (int)cn.odt.size(); ++p) {
          int w = vbase[c] + p;
          if (seen.insert(w).second) st.push_back({w, nsame});
        }
      }
    }
  }

  std::vector<int64_t> frame_bound_cache;
  std::vector<Shape> ta_shape;

  // ---- TMA operand registry (bf16 buffers viewed as [slots][rows][cols])
  void register_buf(int buf, int slots, std::pair<int, int> rc) {
    if (rc.first <= 0 || rc.second <= 0 || rc.second % 64 != 0) return;
    DReg r{};
    r.base = buf;
    r.slots = slots;
    r.rows = rc.first;
    r.cols = rc.second;
    r.slot_bytes = (int64_t)rc.first * rc.second * 2;
    P.reg.push_back(r);
  }
  void register_shape(int buf, const Shape& shp, int slots) {
    if (shp.size() == 2) register_buf(buf, slots, {(int)shp[0], (int)shp[1]});
    else if (shp.size() == 3) register_buf(buf, slots * (int)shp[0], {(int)shp[1], (int)shp[2]});
  }
  std::pair<int, int> ta_rows_cols(size_t k) {
    const Shape& s = ta_shape.at(k);
    if (s.size() != 2) return {0, 0};
    return {(int)s[0], (int)s[1]};
  }

  // ---- in-place accumulator fusion: loop variable v with
  //   Switch_v:1 -> Add(., X) -> NextIteration_v   and X routed (within the iteration) from
  //   LSTMCellGrad dW/db outputs or zero constants  ==>  one fp32 buffer updated in place.
  void detect_accumulators() {
    for (size_t f = 0; f < frame_ctx.size(); ++f) {
      const Ctx& ctx = g.ctxs[frame_ctx[f]];
      for (size_t j = 1; j < ctx.loop_vars.size(); ++j) {
        const LoopVar& lv = ctx.loop_vars[j];
        if (!is_float(g.nodes[lv.merge].odt[0])) continue;
        const auto& sc = cons[vbase[lv.sw] + 1];
        if (sc.size() != 1) continue;
        const Node& add = g.nodes[sc[0].first];
        if (add.op != "Add" || add.in.size() != 2) continue;
        const auto& ac = cons[vbase[add.id]];
        if (ac.size() != 1 || ac[0].first != lv.next) continue;
        TRef other = add.in[sc[0].second == 0 ? 1 : 0];
        if (g.shape(other) != g.nodes[lv.merge].osh[0]) continue;
        // backward routing closure of `other`
        std::vector<TRef> st{other};
        std::set<int> seen;
        std::vector<std::pair<int, int>> srcs;
        bool ok = true;
        int port_kind = -1;
        while (!st.empty() && ok) {
          TRef t = st.back();
          st.pop_back();
          if (!seen.insert(vid(t)).second) continue;
          const Node& p = g.nodes[t.node];
          if (p.op == "Merge" && !p.attrs.b("loop")) {
            st.push_back(p.in[0]);
            st.push_back(p.in[1]);
          } else if (p.op == "Identity" || (p.op == "Switch" && !p.attrs.b("loop"))) {
            st.push_back(p.in[0]);
          } else if (p.op == "LSTMCellGrad" && (t.port == 3 || t.port == 4)) {
            if (port_kind >= 0 && port_kind != t.port) ok = false;
            port_kind = t.port;
            // the port must only feed this routing chain
            for (auto [c, idx] : cons[vid(t)]) {
              const std::string& cop = g.nodes[c].op;
              if (!(cop == "Merge" || cop == "Identity" || cop == "Switch" || c == add.id)) ok = false;
            }
            srcs.push_back({p.id, t.port});
          } else if (p.op == "Const") {
            for (auto b : p.data) ok &= (b == 0);
          } else {
            ok = false;
          }
        }
        if (!ok || srcs.empty()) continue;
        DAcc a{};
        a.frame = (int)f;
        a.bytes = numel(g.nodes[lv.merge].osh[0]) * 4;
        a.base = add_buf(a.bytes, false, "accumulator " + std::to_string(lv.merge));
        TRef init = g.nodes[lv.enter].in[0];
        a.init_vid = vid(init);
        const Node& in = g.nodes[init.node];
        a.init_zero = in.op == "Const" && std::all_of(in.data.begin(), in.data.end(), [](uint8_t b) { return b == 0; });
        int id = (int)P.accs.size();
        P.accs.push_back(a);
        acc_of_loopvar[lv.merge] = id;
        acc_of_add[add.id] = id;
        for (auto& sp : srcs) acc_of_src[sp] = id;
      }
    }
  }

  // number of placement slots of a heavy node: outputs + internal scratch / prep buffers
  // forward cells whose input projection runs as its own instance ahead of the recurrence
  // (runtime.cu HK_LSTM_XPROJ_TC). Off by default, CF_XPROJ=1 enables it: measured on cfg3 the
  // forward took 33.4 ms with the split vs 24.0 ms fused (the cell tile's time is its
  // epilogue, which the split does not shorten, and the projection adds 1.5 SM-s of tiles)
  bool xproj(const Node& n) const {
    return bf16() && n.op == "LSTMCell" && std::getenv("CF_XPROJ") != nullptr;
  }
  int n_places(const Node& n) const {
    int np = (int)n.odt.size();
    if (n.op == "LSTMCellGrad") np += bf16() ? 2 : 1;   // dz scratch (+ W^T prep)
    if (n.op == "LSTMCell" && bf16()) np += xproj(n) ? 2 : 1;   // W prep (+ x-projection scratch)
    return np;
  }

  void place_outputs(const Node& n) {
    DNode& d = P.nodes[n.id];
    d.place_off = (int)P.places.size();
    int f = frame_of[n.id];
    int nout = (int)n.odt.size();
    const int np = n_places(n);
    for (int p = 0; p < np; ++p) {
      PlaceDesc pl{};
      Shape shp;
      int32_t dd;
      bool internal = p >= nout;
      enum { NONE, DZ, WPREP, WTPREP, ZX } kind = NONE;
      int64_t extra_bytes = 0;
      if (!internal) {
        shp = n.osh[p];
        dd = vdt[vbase[n.id] + p];
      } else if (n.op == "LSTMCellGrad" && p == nout) {
        kind = DZ;
        int64_t B = g.shape(n.in[0])[0], H = g.shape(n.in[1])[1];
        shp = {B, 4 * H};
        dd = bf16() ? D_BF16 : D_F32;
        if (bf16()) extra_bytes = ((B + 127) / 128) * 4 * H * 4;   // db partials
      } else if (n.op == "LSTMCell" && p == nout + 1) {
        kind = ZX;   // x-projection [B, 4H] fp32, gate-interleaved like the gates
        shp = {g.shape(n.in[0])[0], 4 * g.shape(n.in[1])[1]};
        dd = D_F32;
      } else {
        kind = n.op == "LSTMCell" ? WPREP : WTPREP;
        Shape w = g.shape(n.in[3]);
        shp = kind == WPREP ? w : Shape{w[1], w[0]};
        dd = D_BF16;
      }
      pl.dt = dd;
      int64_t body = numel(shp) * dev_size(dd);
      pl.elem_bytes = ((body + 1023) / 1024) * 1024 + extra_bytes;
      if (!internal) pl.elem_bytes = body;
      if (n.op == "ReduceSum" && n.attrs.i("axis", -1) != 0) pl.elem_bytes = 8192;  // + partials
      bool pinned = false;
      int taw = -1;
      if (!internal) closure(vbase[n.id] + p, &pinned, &taw, f);
      auto acc_it = acc_of_src.find({n.id, p});
      if (acc_it != acc_of_src.end()) {
        pl.kind = PL_ACC;
        pl.slots = acc_it->second;   // acc id
        pl.base = -1;
        pl.dt = D_F32;
      } else if ((kind == WTPREP || kind == WPREP) && wt_root.count(n.id) &&
                 wt_buf.count(2 * vid(wt_root.at(n.id)) + (kind == WPREP ? 1 : 0))) {
        pl.kind = PL_ROOT;   // the prepared weight another node of the same root weight prepares
        pl.slots = 1;
        pl.base = wt_buf.at(2 * vid(wt_root.at(n.id)) + (kind == WPREP ? 1 : 0));
      } else if (kind == WPREP || kind == WTPREP || f < 0) {
        pl.kind = PL_ROOT;
        pl.slots = 1;
        pl.base = add_buf(pl.elem_bytes, false, "root " + n.op + std::to_string(n.id));
        if (dd == D_BF16) register_shape((int)pl.base, shp, 1);
        if ((kind == WTPREP || kind == WPREP) && wt_root.count(n.id))
          wt_buf[2 * vid(wt_root.at(n.id)) + (kind == WPREP ? 1 : 0)] = (int)pl.base;
      } else if (taw >= 0 && P.tas[trace_ta(g.nodes[taw].in[0])].elem_bytes == body &&
                 P.tas[trace_ta(g.nodes[taw].in[0])].dt == dd) {
        const Node& w = g.nodes[taw];
        pl.kind = PL_TA;
        pl.ta = trace_ta(w.in[0]);
        pl.index_vid = vid(w.in[1]);
        // the write index and the handle must be evaluated before this heavy node
        extra_edges[f].push_back({w.in[1].node, n.id});
        extra_edges[f].push_back({w.in[0].node, n.id});
      } else if (pinned) {
        pl.kind = PL_ARENA;
        pl.slots = -1;   // allocated with the frame bound
        pl.base = -1;
      } else {
        int K = o.parallel_iterations > 0 ? o.parallel_iterations : g.ctxs[frame_ctx[f]].K;
        pl.kind = PL_RING;
        pl.slots = K + 1;
        // chunked dW reads the dz of the last P.dw_chunk steps: keep them alive past the window
        if (kind == DZ && bf16()) pl.slots = K + P.dw_chunk + 1;
        pl.base = add_buf((size_t)pl.elem_bytes * pl.slots, false, "ring " + n.op + std::to_string(n.id));
        if (dd == D_BF16 && shp.size() == 2)
          register_buf_stride((int)pl.base, pl.slots, (int)shp[0], (int)shp[1], pl.elem_bytes);
      }
      P.places.push_back(pl);
    }
  }

  void register_buf_stride(int buf, int slots, int rows, int cols, int64_t slot_bytes) {
    if (cols % 64 != 0) return;
    DReg r{};
    r.base = buf;
    r.slots = slots;
    r.rows = rows;
    r.cols = cols;
    r.slot_bytes = slot_bytes;
    P.reg.push_back(r);
  }

  // ---- structured conds (reading R20). A frame body qualifies when every cond context in it
  // is a builder cond (Switch/Merge only through cf_cond) holding no Send/Recv, and no control
  // edge leaves a cond Switch. Fills alias (Switch output vid -> its data input vid) and the
  // device context of every node of `ord`.
  std::map<int, int> gctx_to_dctx;
  int dctx_of(int c) {
    if (g.ctxs[c].kind != COND) return 0;
    auto it = gctx_to_dctx.find(c);
    if (it != gctx_to_dctx.end()) return it->second;
    if (P.ctxs.empty()) P.ctxs.push_back(DCtx{0, -1, 0, -1});
    DCtx d{};
    d.parent = dctx_of(g.ctxs[c].parent);
    d.pred_vid = vid(g.ctxs[c].pred);
    d.branch = g.ctxs[c].branch;
    d.cond_id = g.ctxs[c].cond_id;
    P.ctxs.push_back(d);
    return gctx_to_dctx[c] = (int)P.ctxs.size() - 1;
  }
  bool structure_conds(const std::vector<int>& ord, std::map<int, int>* alias, std::vector<int>* nctx) {
    if (std::getenv("CF_NO_STRUCT")) return false;   // debugging switch
    std::set<int> sw;
    for (int v : ord) {
      const Node& n = g.nodes[v];
      const bool in_cond = g.ctxs[n.ctx].kind == COND;
      if (in_cond && (n.op == "Send" || n.op == "Recv")) return false;
      if (in_cond && n.op == "Switch") {
        if (n.attrs.b("loop")) return false;
        sw.insert(v);
      }
    }
    if (sw.empty()) return false;
    for (int v : ord)
      for (int c : g.nodes[v].ctrl)
        if (sw.count(c)) return false;
    // cond Merges must have both inputs produced inside their two branches
    for (int v : ord)
      if (g.nodes[v].op == "Merge" && !g.nodes[v].attrs.b("loop"))
        if (merge_branch_ctx_g(v, 0) < 0 || merge_branch_ctx_g(v, 1) < 0) return false;
    for (int v : sw) {
      const Node& n = g.nodes[v];
      (*alias)[vbase[v]] = vid(n.in[0]);
      (*alias)[vbase[v] + 1] = vid(n.in[0]);
    }
    nctx->clear();
    for (int v : ord) nctx->push_back(dctx_of(g.nodes[v].ctx));
    if (P.ctxs.size() > 128) throw CfError(CF_E_UNSUPPORTED, "more than 127 cond contexts in one program");
    // predicates may themselves be captures
    for (auto& d : P.ctxs)
      for (auto it = alias->find(d.pred_vid); it != alias->end(); it = alias->find(d.pred_vid))
        d.pred_vid = it->second;
    return true;
  }
  // graph cond context of Merge node m's input j (the branch child of m's context), or -1
  int merge_branch_ctx_g(int m, int j) {
    const Node& mn = g.nodes[m];
    int c = g.nodes[mn.in[j].node].ctx;
    while (c >= 0 && g.ctxs[c].parent != mn.ctx) c = g.ctxs[c].parent;
    if (c < 0 || g.ctxs[c].kind != COND || g.ctxs[c].branch != j) return -1;
    return c;
  }
  int merge_branch_ctx(int m, int j) { return dctx_of(merge_branch_ctx_g(m, j)); }

  // ---- AddN -> LSTMCellGrad dout fusion: the gradient of a layer output is the sum of the
  // next layer's d[x] and the output TensorArray's gradient; the cell-gradient tile adds the
  // (up to 3) terms itself, so the sum is never materialised (one instance and one
  // [B, H] write + read less per layer and step).
  std::map<int, int> fused_dout;   // LSTMCellGrad node -> folded AddN node
  std::set<int> fused_addn;
  void fuse_dout_sums() {
    if (std::getenv("CF_NO_FUSE")) return;   // debugging switch
    for (const Node& n : g.nodes) {
      if (n.op != "LSTMCellGrad") continue;
      const int o = n.attrs.b("masked") ? 7 : 5;
      const TRef din = n.in[o + 2];
      const Node& a = g.nodes[din.node];
      if (a.op != "AddN" || a.in.size() < 2 || a.in.size() > 3) continue;
      if (cons[vid(din)].size() != 1 || a.ctx != n.ctx || frame_of[a.id] != frame_of[n.id]) continue;
      if (acc_of_add.count(a.id) || vdt[vid(din)] != D_F32) continue;
      bool ok = true;
      for (auto& t : a.in) ok &= vdt[vid(t)] == D_F32 && g.shape(t) == g.shape(din);
      if (!ok) continue;
      fused_dout[n.id] = a.id;
      fused_addn.insert(a.id);
      const int f = frame_of[n.id];
      if (f >= 0)
        for (auto& t : a.in) extra_edges[f].push_back({t.node, n.id});
    }
  }

  bool waveable(int v) const {
    const DNode& d = P.nodes[v];
    switch (d.op) {
      // value-free ops with a fast path on the helper warps (runtime.cu fast_node); control
      // inputs allowed. TA reads / zero-copy writes and scalar ops on immediates too: a node
      // the fast path declines is evaluated by the driver right after its wave.
      case OP_CONST: case OP_PASS: case OP_FLOW: case OP_SCALAR: case OP_ACC: case OP_TA_GRAD:
      case OP_TA_READ: case OP_TA_WRITE:
        return true;
      case OP_STACK_PUSH: case OP_STACK_POP: return P.swaps.empty();   // control inputs too
      default: break;
    }
    if (d.n_ctrl != 0) return false;
    switch (d.op) {
      case OP_MERGE: case OP_MERGE_LOOP: case OP_NEXTITER: case OP_SWITCH: return true;
      case OP_STACK_PUSH: case OP_STACK_POP: return P.swaps.empty();
      default: return false;
    }
  }
  // heavy nodes the driver constructs as one batch (runtime.cu run_batch): the tensor-core LSTM
  // cell nodes of the bf16 path (no swapped stacks: a swap copy is created while a node is built)
  bool batchable(int v) const {
    const DNode& d = P.nodes[v];
    return bf16() && P.swaps.empty() && !std::getenv("CF_NO_BATCH") && d.op == OP_HEAVY &&
           (d.aux[0] == HK_LSTM_FWD || d.aux[0] == HK_LSTM_BWD_EW) && d.n_in <= 32 && d.n_ctrl <= 32;
  }
  void form_waves(int f, std::vector<int>* ord, std::vector<int>* nctx, const std::map<int, int>& alias,
                  std::vector<int>* wave_len, std::vector<int>* batch_len) {
    const int n = (int)ord->size();
    wave_len->assign(n, 0);
    batch_len->assign(n, 0);
    if (std::getenv("CF_NO_LEVEL_ORDER")) return;   // debugging switch
    std::map<int, int> pos;
    for (int k = 0; k < n; ++k) pos[(*ord)[k]] = k;
    std::vector<int> prod_of_vid(P.n_vids, -1);
    for (int k = 0; k < n; ++k) {
      const Node& nd = g.nodes[(*ord)[k]];
      for (size_t p2 = 0; p2 < nd.odt.size(); ++p2) prod_of_vid[vbase[nd.id] + p2] = nd.id;
    }
    auto res = [&](int v) {
      for (auto it = alias.find(v); it != alias.end(); it = alias.find(v)) v = it->second;
      return v;
    };
    std::vector<int> level(n, 0);
    std::vector<std::vector<int>> preds(n);
    for (int k = 0; k < n; ++k) {
      const int v = (*ord)[k];
      if (P.nodes[v].op == OP_MERGE_LOOP) continue;   // sources within an iteration
      const Node& nd = g.nodes[v];
      for (auto& t : nd.in) {
        int pv = prod_of_vid[res(vid(t))];
        if (pv >= 0 && pos.count(pv)) preds[k].push_back(pos[pv]);
      }
      for (int c : nd.ctrl)
        if (pos.count(c)) preds[k].push_back(pos[c]);
    }
    // extra edges may name a compiled-away cond Switch: use its data input's producer
    auto node_res = [&](int a) {
      for (int k2 = 0; k2 < 64 && !pos.count(a); ++k2) {
        const Node& an = g.nodes[a];
        if (an.op != "Switch" || an.in.empty()) break;
        a = an.in[0].node;
      }
      return a;
    };
    for (auto& [a0, b] : extra_edges[f]) {
      const int a = node_res(a0);
      if (pos.count(a) && pos.count(b)) preds[pos[b]].push_back(pos[a]);
    }
    // a node of a structured cond branch reads its context's liveness, i.e. the predicates of
    // the context chain: it must come after their producers (the compiled-away Switches
    // carried that dependence)
    for (int k = 0; k < n; ++k)
      for (int c = (*nctx)[k]; c > 0; c = P.ctxs[c].parent) {
        const int pv = prod_of_vid[P.ctxs[c].pred_vid];
        if (pv >= 0 && pos.count(pv)) preds[k].push_back(pos[pv]);
      }
    for (int k = 0; k < n; ++k) {
      const DNode& dn = P.nodes[(*ord)[k]];
      if (dn.op == OP_MERGE && dn.aux[5] == 0 && g.nodes[(*ord)[k]].attrs.has("cond_id")) {
        // structured Merge (aux set later): after its cond's predicate
        for (int j = 0; j < 2; ++j) {
          int bc = merge_branch_ctx_g((*ord)[k], j);
          if (bc >= 0) {
            const int pv = prod_of_vid[res(vid(g.ctxs[bc].pred))];
            if (pv >= 0 && pos.count(pv)) preds[k].push_back(pos[pv]);
          }
        }
      }
    }
    // a loop Merge reads the previous iteration's NextIteration token: the NextIteration of
    // this iteration must come later (the Kahn order guarantees it; levels must too)
    for (int k = 0; k < n; ++k)
      if (P.nodes[(*ord)[k]].op == OP_NEXTITER)
        for (auto [c, idx] : cons[vbase[(*ord)[k]]])
          if (pos.count(c) && pos[c] < k) preds[k].push_back(pos[c]);
    for (int k = 0; k < n; ++k)   // ord is topological: predecessors come first
      for (int q : preds[k]) level[k] = std::max(level[k], level[q] + 1);
    // phases: a chain of batchable heavy nodes (e.g. the layers of one cell branch) stays in one
    // phase; any other node that consumes a batchable node's output starts the next phase. Within
    // a phase the other nodes come first (level order, waves), then the phase's batchable nodes
    // as ONE batch: the driver builds their instances together (runtime.cu run_batch) instead of
    // one node at a time between routing waves. Any topological order is a valid evaluation
    // order of the dataflow graph (PAPER.md:209-214 non-strict semantics).
    std::vector<int> phase(n, 0), bat(n, 0);
    for (int k = 0; k < n; ++k) bat[k] = batchable((*ord)[k]) ? 1 : 0;
    for (int k = 0; k < n; ++k)
      for (int q : preds[k]) phase[k] = std::max(phase[k], phase[q] + ((bat[q] && !bat[k]) ? 1 : 0));
    // a batch completes as a unit: a node that reads batch members starts one level after the
    // batch's LAST member, not after the member it reads (the layers of a cell branch chain
    // inside the batch, which otherwise turns the routing after it into one level per layer)
    if (!std::getenv("CF_NO_BATCH_LEVELS")) {
      std::map<int, int> blev;   // phase -> deepest batchable member
      for (int k = 0; k < n; ++k)
        if (bat[k]) blev[phase[k]] = std::max(blev[phase[k]], level[k]);
      for (int k = 0; k < n; ++k) {
        if (bat[k]) continue;
        int lv = 0;
        for (int q : preds[k]) lv = std::max(lv, (bat[q] ? blev[phase[q]] : level[q]) + 1);
        level[k] = lv;
      }
    }
    std::vector<int> idx(n);
    for (int k = 0; k < n; ++k) idx[k] = k;
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
      if (phase[a] != phase[b]) return phase[a] < phase[b];
      if (bat[a] != bat[b]) return bat[a] < bat[b];
      if (level[a] != level[b]) return level[a] < level[b];
      return waveable((*ord)[a]) > waveable((*ord)[b]);
    });
    std::vector<int> o2, c2;
    for (int k : idx) {
      o2.push_back((*ord)[k]);
      c2.push_back((*nctx)[k]);
    }
    wave_len->assign(n, 0);
    batch_len->assign(n, 0);
    for (int k = 0; k < n;) {   // batches: consecutive batchable nodes of one phase (<= 32)
      if (!bat[idx[k]]) {
        ++k;
        continue;
      }
      int e = k;
      while (e < n && bat[idx[e]] && phase[idx[e]] == phase[idx[k]] && e - k < 32) ++e;
      if (e - k >= 2) (*batch_len)[k] = e - k;
      k = e;
    }
    // smallest level group evaluated as a wave (helper round trip vs serial evaluation);
    // CF_MIN_WAVE overrides it (A/B)
    int min_wave = 1;   // measured on cfg3: 1 -> 80.5 ms, 2 -> 81.7, 4 -> 81.9 ms per step
    if (const char* mw = std::getenv("CF_MIN_WAVE")) min_wave = std::max(1, atoi(mw));
    // waves pay for themselves by overlapping the construction of tensor-core nodes; a body
    // without one (e.g. the trivial control-overhead loop) evaluates its nodes inline
    // (measured on that loop: 27.5 -> 23.4 us per iteration); CF_WAVES_ALWAYS for A/B
    bool has_mm = std::getenv("CF_WAVES_ALWAYS") != nullptr;
    for (int k = 0; k < n && !has_mm; ++k) {
      const std::string& op = g.nodes[(*ord)[k]].op;
      has_mm = op == "LSTMCell" || op == "LSTMCellGrad" || op == "MatMul";
    }
    for (int k = 0; k < n && has_mm && !std::getenv("CF_NO_WAVES");) {
      int e = k;
      while (e < n && waveable(o2[e]) && level[idx[e]] == level[idx[k]] && e - k < 256) ++e;
      if (e - k >= min_wave) (*wave_len)[k] = e - k;
      k = std::max(e, k + 1);
    }
    *ord = o2;
    *nctx = c2;
  }

  // the top-most frame below `anc` on node x's frame chain (x inside a frame nested in anc), or -1
  int child_frame_of(int x, int anc) const {
    int f = frame_of[x];
    if (g.nodes[x].op == "Exit") f = frame_id.at(g.nodes[x].attrs.s("frame"));
    for (; f >= 0; f = frame_parent[f])
      if (frame_parent[f] == anc) return f;
    return -1;
  }
  // body program of a frame whose body holds nested frames: the nested
  // frames are single steps (OP_FRAME) of the body, placed after the producers of their Enter
  // inputs and before the consumers of their Exits; plain topological order (no level order,
  // routing waves, heavy batches or structured conds in such a body)
  void build_parent_frame(int f, const Ctx& ctx, const std::vector<int>& body, const std::vector<int>& enters,
                          const std::vector<int>& exits, const std::vector<int>& children,
                          const std::vector<int64_t>& bound, int* iter_base) {
    const int N = (int)g.nodes.size();
    std::set<int> bset(body.begin(), body.end());
    auto item_of = [&](int x) -> int {
      if (bset.count(x)) return x;
      const int c = child_frame_of(x, f);
      return c >= 0 ? N + c : -1;
    };
    std::vector<int> items(body.begin(), body.end());
    for (int c : children) items.push_back(N + c);
    std::map<int, std::set<int>> succ;
    std::map<int, int> indeg;
    for (int it : items) indeg[it] = 0;
    auto edge = [&](int a, int b) {
      if (a < 0 || b < 0 || a == b || !indeg.count(a) || !indeg.count(b)) return;
      if (succ[a].insert(b).second) indeg[b]++;
    };
    for (int i = 0; i < N; ++i) {
      const int dst = item_of(i);
      if (dst < 0) continue;
      if (dst == i && P.nodes[i].op == OP_MERGE_LOOP) continue;   // sources within an iteration
      for (auto& t : g.nodes[i].in) edge(item_of(t.node), dst);
      for (int cc : g.nodes[i].ctrl) edge(item_of(cc), dst);
    }
    for (auto& [a, b] : extra_edges[f]) edge(item_of(a), item_of(b));
    std::vector<int> ready, ord;
    for (int it : items)
      if (indeg[it] == 0) ready.push_back(it);
    std::sort(ready.rbegin(), ready.rend());
    while (!ready.empty()) {
      const int v = ready.back();
      ready.pop_back();
      ord.push_back(v);
      for (int w : succ[v])
        if (--indeg[w] == 0) {
          ready.push_back(w);
          std::sort(ready.rbegin(), ready.rend());
        }
    }
    if (ord.size() != items.size())
      throw CfError(CF_E_INVALID_GRAPH, "frame " + ctx.name + " body has a cycle without NextIteration");
    DFrame& F = P.frames[f];
    F.K = o.parallel_iterations > 0 ? o.parallel_iterations : ctx.K;
    F.bound = (int32_t)bound[f];
    F.parent = frame_parent[f];
    F.body_off = (int)P.order.size();
    for (int v : ord) P.order.push_back(v >= N ? ctx.loop_vars.at(0).enter : v);
    F.n_body = (int)P.order.size() - F.body_off;
    F.enter_off = (int)P.order.size();
    F.n_enter = (int)enters.size();
    P.order.insert(P.order.end(), enters.begin(), enters.end());
    F.exit_off = (int)P.order.size();
    F.n_exit = (int)exits.size();
    P.order.insert(P.order.end(), exits.begin(), exits.end());
    F.counter_switch = ctx.loop_vars.at(0).sw;
    F.counter_enter = ctx.loop_vars.at(0).enter;
    F.iter_base = *iter_base;
    *iter_base += (int)bound[f] + 2;
    F.bn_off = (int)P.body_nodes.size();
    F.bi_off = (int)P.body_ivids.size();
    for (int v : ord) {
      DNode bn{};
      if (v >= N) {
        bn.op = OP_FRAME;
        bn.aux[0] = v - N;
        bn.place_off = -1;
        ((int16_t*)bn.pad)[5] = -1;
        bn.in_off = bn.ctrl_off = (int)P.body_ivids.size() - F.bi_off;
        P.body_nodes.push_back(bn);
        continue;
      }
      bn = P.nodes[v];
      ((int16_t*)bn.pad)[5] = (int16_t)(v < 32768 ? v : -1);
      bn.ctx = 0;
      const int base = (int)P.body_ivids.size() - F.bi_off;
      for (int j = 0; j < bn.n_in; ++j) P.body_ivids.push_back(P.in_vids[bn.in_off + j]);
      for (int j = 0; j < bn.n_ctrl; ++j) P.body_ivids.push_back(P.in_vids[bn.ctrl_off + j]);
      bn.in_off = base;
      bn.ctrl_off = base + bn.n_in;
      P.body_nodes.push_back(bn);
    }
    F.bi_count = (int)P.body_ivids.size() - F.bi_off;
    while (P.body_ivids.size() % 4) P.body_ivids.push_back(0);
    P.max_body = std::max(P.max_body, F.n_body);
    P.max_bi = std::max(P.max_bi, F.bi_count);
    F.acc_off = (int)P.order.size();
    F.n_acc = 0;
    for (size_t a = 0; a < P.accs.size(); ++a)
      if (P.accs[a].frame == f) {
        P.order.push_back((int)a);
        F.n_acc++;
      }
  }

  void build_orders(const std::vector<int64_t>& bound) {
    const int N = (int)g.nodes.size();
    // arena allocation needs the bound. Stack swapping: when all arenas
    // exceed the stack budget, the largest ones (each >= swap_min_bytes) become swapped
    // arenas: a (K + 1)-slot device ring + host backing (reading R19).
    struct Ar { int node, port, frame; int64_t bytes; };
    std::vector<Ar> ars;
    for (int i = 0; i < N; ++i) {
      const DNode& d = P.nodes[i];
      if (d.op != OP_HEAVY && d.op != OP_RECV) continue;
      int np = n_places(g.nodes[i]);
      for (int p = 0; p < np; ++p)
        if (P.places[d.place_off + p].kind == PL_ARENA)
          ars.push_back({i, p, frame_of[i], P.places[d.place_off + p].elem_bytes * frame_total[frame_of[i]]});
    }
    std::set<std::pair<int, int>> swap_set;
    if (o.stack_budget_bytes >= 0) {
      int64_t total = 0;
      for (auto& a : ars) total += a.bytes;
      std::vector<Ar> cand;
      for (auto& a : ars)
        if (P.places[P.nodes[a.node].place_off + a.port].elem_bytes >= o.swap_min_bytes) cand.push_back(a);
      const bool small = o.swap_smallest_first;
      std::stable_sort(cand.begin(), cand.end(),
                       [small](const Ar& x, const Ar& y) { return small ? x.bytes < y.bytes : x.bytes > y.bytes; });
      for (auto& a : cand) {
        if (total <= o.stack_budget_bytes) break;
        swap_set.insert({a.node, a.port});
        total -= a.bytes;
      }
    }
    for (auto& a : ars) {
      const int i = a.node, p = a.port, f = a.frame;
      PlaceDesc& pl = P.places[P.nodes[i].place_off + p];
      int slots = (int)frame_total[f];   // = bound[f] for a top-level frame
      if (swap_set.count({i, p})) {
        const int K = o.parallel_iterations > 0 ? o.parallel_iterations : g.ctxs[frame_ctx[f]].K;
        slots = std::min<int>(K + 1, (int)bound[f]);
        pl.kind = PL_SWAP;
        pl.ta = (int32_t)P.swaps.size();   // swap id
        SwapPlan sp;
        sp.place = P.nodes[i].place_off + p;
        sp.elem_bytes = pl.elem_bytes;
        sp.ring = slots;
        sp.capacity = (int32_t)bound[f];
        // swap-ins land in a ring of their own, indexed by the gradient loop's iteration: the
        // forward ring may still hold values that left the loop through an Exit. In bf16 mode a
        // chunked dW instance reads the popped x / h of its last P.dw_chunk steps after those
        // iterations left the window, so the ring keeps that many more slots (like the dz ring)
        sp.in_ring = std::min<int>(bf16() ? K + P.dw_chunk + 1 : K + 1, (int)bound[f]);
        sp.in_buf = add_buf((size_t)pl.elem_bytes * sp.in_ring, false, "swap-in ring " + std::to_string(i));
        if (pl.dt == D_BF16 && p < (int)g.nodes[i].osh.size() && g.nodes[i].osh[p].size() == 2)
          register_buf_stride(sp.in_buf, sp.in_ring, (int)g.nodes[i].osh[p][0], (int)g.nodes[i].osh[p][1],
                              pl.elem_bytes);
        P.swaps.push_back(sp);
        P.stack_swapped_bytes += a.bytes;
      } else {
        P.stack_resident_bytes += a.bytes;
      }
      pl.slots = slots;
      pl.base = add_buf((size_t)pl.elem_bytes * slots, false,
                        (pl.kind == PL_SWAP ? "swap ring " : "arena ") + g.nodes[i].op + std::to_string(i));
      if (pl.dt == D_BF16 && p < (int)g.nodes[i].osh.size() && g.nodes[i].osh[p].size() == 2)
        register_buf_stride((int)pl.base, slots, (int)g.nodes[i].osh[p][0], (int)g.nodes[i].osh[p][1],
                            pl.elem_bytes);
    }
    // ---- frames
    P.frames.resize(frame_ctx.size());
    int iter_base = 0;
    for (size_t f = 0; f < frame_ctx.size(); ++f) {
      int c = frame_ctx[f];
      const Ctx& ctx = g.ctxs[c];
      std::vector<int> body, enters, exits;
      for (int i = 0; i < N; ++i) {
        if (frame_of[i] != (int)f || fused_addn.count(i)) continue;
        if (g.nodes[i].op == "Enter" && g.nodes[i].attrs.s("frame") == ctx.name) enters.push_back(i);
        else if (g.nodes[i].op == "Exit" && g.nodes[i].attrs.s("frame") != ctx.name) continue;   // a child's
        else body.push_back(i);
      }
      for (int i = 0; i < N; ++i)
        if (g.nodes[i].op == "Exit" && g.nodes[i].attrs.s("frame") == ctx.name) exits.push_back(i);
      std::vector<int> children;
      for (size_t c2 = 0; c2 < frame_ctx.size(); ++c2)
        if (frame_parent[c2] == (int)f) children.push_back((int)c2);
      if (!children.empty()) {
        build_parent_frame((int)f, ctx, body, enters, exits, children, bound, &iter_base);
        continue;
      }
      std::set<int> bset(body.begin(), body.end());
      std::map<int, std::vector<int>> succ;
      std::map<int, int> indeg;
      for (int i : body) indeg[i] = 0;
      auto edge = [&](int a, int b) {
        if (!bset.count(a) || !bset.count(b) || a == b) return;
        succ[a].push_back(b);
        indeg[b]++;
      };
      for (int i : body) {
        const Node& n = g.nodes[i];
        if (P.nodes[i].op == OP_MERGE_LOOP) continue;   // sources within an iteration
        for (auto& t : n.in) edge(t.node, i);
        for (int c : n.ctrl) edge(c, i);
      }
      for (auto& [a, b] : extra_edges[f]) edge(a, b);
      std::vector<int> ord;
      std::vector<int> ready;
      for (int i : body)
        if (indeg[i] == 0) ready.push_back(i);
      std::sort(ready.rbegin(), ready.rend());
      while (!ready.empty()) {
        int v = ready.back();
        ready.pop_back();
        ord.push_back(v);
        for (int w : succ[v])
          if (--indeg[w] == 0) {
            ready.push_back(w);
            std::sort(ready.rbegin(), ready.rend());
          }
      }
      if (ord.size() != body.size())
        throw CfError(CF_E_INVALID_GRAPH, "frame " + ctx.name + " body has a cycle without NextIteration");
      // ---- structured conds (reading R20): compile capture Switches away
      std::map<int, int> alias;
      std::vector<int> node_ctx;
      if (structure_conds(ord, &alias, &node_ctx)) {
        std::vector<int> kept, kctx;
        for (size_t k = 0; k < ord.size(); ++k)
          if (!(g.nodes[ord[k]].op == "Switch" && g.ctxs[g.nodes[ord[k]].ctx].kind == COND)) {
            kept.push_back(ord[k]);
            kctx.push_back(node_ctx[k]);
          }
        ord = kept;
        node_ctx = kctx;
        P.structured_frames++;
      } else {
        alias.clear();
        node_ctx.assign(ord.size(), 0);
      }
      auto res = [&](int v) {
        for (auto it = alias.find(v); it != alias.end(); it = alias.find(v)) v = it->second;
        return v;
      };
      for (int v : ord) {
        DNode& dn = P.nodes[v];
        if (dn.place_off >= 0)
          for (int p2 = 0; p2 < n_places(g.nodes[v]); ++p2) {
            PlaceDesc& pl = P.places[dn.place_off + p2];
            if (pl.kind == PL_TA) pl.index_vid = res(pl.index_vid);
          }
      }
      // ---- waves: order the body by dependency level and group each level's routing / stack
      //      nodes (independent by construction) behind an OP_WAVE marker
      std::vector<int> wave_len;   // per ord position: > 0 = a wave of that many starts here
      std::vector<int> batch_len;  // per ord position: > 0 = a heavy batch of that many starts here
      form_waves(f, &ord, &node_ctx, alias, &wave_len, &batch_len);
      DFrame& F = P.frames[f];
      F.K = o.parallel_iterations > 0 ? o.parallel_iterations : ctx.K;
      F.bound = (int32_t)bound[f];
      F.parent = frame_parent[f];
      F.body_off = (int)P.order.size();
      for (size_t k = 0; k < ord.size(); ++k) {
        if (wave_len[k] > 0 || batch_len[k] > 0) P.order.push_back(ord[k]);   // the marker's slot (never evaluated)
        P.order.push_back(ord[k]);
      }
      F.n_body = (int)P.order.size() - F.body_off;
      F.enter_off = (int)P.order.size();
      F.n_enter = (int)enters.size();
      P.order.insert(P.order.end(), enters.begin(), enters.end());
      F.exit_off = (int)P.order.size();
      F.n_exit = (int)exits.size();
      P.order.insert(P.order.end(), exits.begin(), exits.end());
      F.counter_switch = ctx.loop_vars.at(0).sw;
      F.counter_enter = ctx.loop_vars.at(0).enter;
      F.iter_base = iter_base;
      iter_base += (int)bound[f] + 2;
      // body program: node records in evaluation order with rebased input ids, so the
      // driver can stage one frame's control program in shared memory
      F.bn_off = (int)P.body_nodes.size();
      F.bi_off = (int)P.body_ivids.size();
      for (size_t k = 0; k < ord.size(); ++k) {
        const int v = ord[k];
        if (wave_len[k] > 0) {
          DNode wm{};
          wm.op = OP_WAVE;
          wm.aux[0] = wave_len[k];
          unsigned long long mask[2] = {0, 0};   // contexts the wave's nodes read (128 bits)
          auto add = [&](int c) { mask[c >> 6] |= 1ULL << (c & 63); };
          for (int q = 0; q < wave_len[k]; ++q) {
            const int u = ord[k + q];
            if (node_ctx[k + q] > 0) add(node_ctx[k + q]);
            if (P.nodes[u].op == OP_MERGE && g.nodes[u].attrs.has("cond_id") && !alias.empty()) {
              int c0 = merge_branch_ctx(u, 0), c1 = merge_branch_ctx(u, 1);
              if (c0 > 0) add(c0);
              if (c1 > 0) add(c1);
            }
          }
          wm.imm[0] = (int64_t)mask[0];
          wm.imm[1] = (int64_t)mask[1];
          wm.place_off = -1;
          wm.in_off = wm.ctrl_off = (int)P.body_ivids.size() - F.bi_off;
          P.body_nodes.push_back(wm);
          P.n_waves++;
        }
        if (batch_len[k] > 0) {
          DNode bm{};
          bm.op = OP_HEAVY_BATCH;
          bm.aux[0] = batch_len[k];
          bm.place_off = -1;
          bm.in_off = bm.ctrl_off = (int)P.body_ivids.size() - F.bi_off;
          P.body_nodes.push_back(bm);
          P.n_batches++;
          // per member: bit j of aux[6] = data input j is an output of an earlier member of the
          // same batch (its liveness follows that member's; the driver checks the others)
          std::map<int, int> out_of;   // value id -> member
          for (int q = 0; q < batch_len[k]; ++q) {
            const int u = ord[k + q];
            for (int p2 = 0; p2 < P.nodes[u].n_out; ++p2) out_of[P.nodes[u].out_vid + p2] = q;
          }
          for (int q = 0; q < batch_len[k]; ++q) {
            DNode& mu = P.nodes[ord[k + q]];
            uint32_t m = 0;
            for (int j = 0; j < mu.n_in && j < 32; ++j) {
              auto it = out_of.find(res(P.in_vids[mu.in_off + j]));
              if (it != out_of.end() && it->second < q) m |= 1u << j;
            }
            mu.aux[6] = (int32_t)m;
          }
        }
        DNode bn = P.nodes[v];
        // node id for the device driver (pad[2] high half; pad[0..2] low are registry hints)
        ((int16_t*)bn.pad)[5] = (int16_t)(v < 32768 ? v : -1);
        bn.ctx = node_ctx[k];
        if (bn.ctx || alias.size()) P.nodes[v].ctx = bn.ctx;
        if (bn.op == OP_MERGE && !alias.empty()) {
          // structured cond Merge: inputs [false branch, true branch] (ir.cpp Graph::cond)
          bn.aux[5] = merge_branch_ctx(v, 0);
          bn.aux[6] = merge_branch_ctx(v, 1);
          P.nodes[v].aux[5] = bn.aux[5];
          P.nodes[v].aux[6] = bn.aux[6];
        }
        int base = (int)P.body_ivids.size() - F.bi_off;
        for (int j = 0; j < bn.n_in; ++j) P.body_ivids.push_back(res(P.in_vids[bn.in_off + j]));
        for (int j = 0; j < bn.n_ctrl; ++j) P.body_ivids.push_back(P.in_vids[bn.ctrl_off + j]);
        bn.in_off = base;
        bn.ctrl_off = base + bn.n_in;
        P.body_nodes.push_back(bn);
      }
      F.bi_count = (int)P.body_ivids.size() - F.bi_off;
      while (P.body_ivids.size() % 4) P.body_ivids.push_back(0);   // 16 B aligned segments
      P.max_body = std::max(P.max_body, F.n_body);
      P.max_bi = std::max(P.max_bi, F.bi_count);
      F.acc_off = (int)P.order.size();
      F.n_acc = 0;
      for (size_t a = 0; a < P.accs.size(); ++a)
        if (P.accs[a].frame == (int)f) {
          P.order.push_back((int)a);
          F.n_acc++;
        }
    }
    P.iter_counters = iter_base;
    // ---- root steps: root nodes + frames as super nodes
    // item id: node i -> i ; frame f -> N + f
    std::vector<int> items;
    for (int i = 0; i < N; ++i)
      if (frame_of[i] < 0 && g.nodes[i].op != "Exit" && !root_dead[i]) items.push_back(i);
    for (size_t f = 0; f < frame_ctx.size(); ++f)
      if (frame_parent[f] < 0) items.push_back(N + (int)f);
    auto item_of = [&](int node) -> int {
      if (frame_of[node] >= 0 || g.nodes[node].op == "Exit") return N + child_frame_of(node, -1);
      return node;
    };
    std::map<int, std::set<int>> succ;
    std::map<int, int> indeg;
    for (int it : items) indeg[it] = 0;
    auto edge = [&](int a, int b) {
      if (a == b || (a < N && root_dead[a])) return;   // a view's dropped operand (1 * v)
      if (succ[a].insert(b).second) indeg[b]++;
    };
    for (int i = 0; i < N; ++i) {
      if (root_dead[i]) continue;   // (its inputs may be live; no edge into a dead item)
      int dst = item_of(i);
      for (auto& t : g.nodes[i].in) edge(item_of(t.node), dst);
      for (int c : g.nodes[i].ctrl) edge(item_of(c), dst);
    }
    // pops after pushes: frame that pushes precedes the frame that pops
    for (auto& n : g.nodes) {
      if (n.op != "StackPop") continue;
      int sid = -1;
      TRef h = n.in[0];
      for (int k = 0; k < 64 && sid < 0; ++k) {
        const Node& hn = g.nodes[h.node];
        if (hn.op == "StackCreate") sid = hn.id;
        else if (!hn.in.empty()) h = hn.in[0];
        else break;
      }
      if (sid < 0) continue;
      for (auto& m : g.nodes)
        if (m.op == "StackPush") {
          TRef hh = m.in[0];
          for (int k = 0; k < 64; ++k) {
            const Node& hn = g.nodes[hh.node];
            if (hn.op == "StackCreate") {
              if (hn.id == sid) edge(item_of(m.id), item_of(n.id));
              break;
            }
            if (hn.in.empty()) break;
            hh = hn.in[0];
          }
        }
    }
    // ready items by key, smallest first: nodes by id, frames after the ready nodes, root-level
    // Recvs last. A Recv's wait instance occupies a slot of the driver's in-flight ring until
    // the peer's message arrives, so it is created only when nothing else is ready (a Recv
    // ready at the start would otherwise sit in the ring through both loops and, once the
    // ring wrapped, block both ranks' drivers on each other: f3's gradient exchange)
    auto key = [&](int it) { return it < N && g.nodes[it].op == "Recv" ? 2 * N + it : it; };
    auto by_key = [&](int a, int b) { return key(a) > key(b); };
    std::vector<int> ready, ord;
    for (int it : items)
      if (indeg[it] == 0) ready.push_back(it);
    std::sort(ready.begin(), ready.end(), by_key);
    while (!ready.empty()) {
      int v = ready.back();
      ready.pop_back();
      ord.push_back(v);
      for (int w : succ[v])
        if (--indeg[w] == 0) {
          ready.push_back(w);
          std::sort(ready.begin(), ready.end(), by_key);
        }
    }
    if (ord.size() != items.size()) throw CfError(CF_E_INVALID_GRAPH, "root graph has a cycle");
    // Root scheduling hints (program.h kRootLow / kRootPrep):
    // - heavy root work no frame depends on (the loss value, fetch-only sums) goes to the
    //   low-priority queue, where it fills idle workers instead of delaying the next loop;
    // - each tensor-core LSTMCellGrad's W^T preparation is issued right after its weight is
    //   available (low priority), so it runs under the forward loop instead of between loops.
    std::vector<char> for_frame(N, 0);
    {
      std::vector<int> work;
      for (auto& n : g.nodes)
        if (frame_of[n.id] >= 0 || n.op == "Exit")
          for (auto& t : n.in)
            if (frame_of[t.node] < 0 && !for_frame[t.node]) {
              for_frame[t.node] = 1;
              work.push_back(t.node);
            }
      while (!work.empty()) {
        const int x = work.back();
        work.pop_back();
        for (auto& t : g.nodes[x].in)
          if (!for_frame[t.node]) {
            for_frame[t.node] = 1;
            work.push_back(t.node);
          }
      }
    }
    const bool hints = std::getenv("CF_NO_ROOT_HINTS") == nullptr;   // A/B switch
    std::map<int, std::vector<int>> prep_after;   // root producer of W -> leader LSTM nodes
    if (hints)
      for (auto& [key, nid] : wt_leader) prep_after[wt_root.at(nid).node].push_back(nid);
    for (auto& [wn, v] : prep_after)   // the forward's packed W first (LSTMCell ids are lower)
      std::sort(v.begin(), v.end());
    for (int it : ord) {
      if (it >= N) {
        P.root_steps.push_back(-(it - N + 1));
        continue;
      }
      const bool low = hints && P.nodes[it].op == OP_HEAVY && !for_frame[it];
      P.root_steps.push_back(low ? it | kRootLow : it);
      for (int gn : prep_after[it]) P.root_steps.push_back(gn | kRootPrep);
    }
  }
};

}  // namespace

HostProgram compile(const Graph& g, const CompileOpts& o, const std::vector<TRef>& fetches) {
  auto errs = g.validate();
  if (!errs.empty()) throw CfError(CF_E_INVALID_GRAPH, errs[0]);
  Compiler c(g, o);
  c.run(fetches);
  // body program listing (debug hook cf_debug_program_listing)
  {
    std::ostringstream ls;
    ls << "root";
    for (int s : c.P.root_steps) {
      if (s < 0) ls << " [frame " << c.P.frame_names[-s - 1] << "]";
      else if (s & kRootPrep) ls << " prep(" << g.nodes[s & kRootNode].op << (s & kRootNode) << ")";
      else if (s & kRootLow) ls << " " << g.nodes[s & kRootNode].op << (s & kRootNode) << "(low)";
      else ls << " " << g.nodes[s].op << s;
    }
    ls << "\n";
    for (size_t f = 0; f < c.P.frames.size(); ++f) {
      const auto& F = c.P.frames[f];
      ls << "frame " << c.P.frame_names[f] << "\n";
      for (int k = 0; k < F.n_body; ++k) {
        const auto& bn = c.P.body_nodes[F.bn_off + k];
        const int nid = c.P.order[F.body_off + k];
        ls << k << " " << (bn.op == OP_WAVE ? std::string("WAVE") : bn.op == OP_HEAVY_BATCH ? std::string("BATCH")
                           : bn.op == OP_FRAME ? "FRAME " + c.P.frame_names[bn.aux[0]] : g.nodes[nid].op) << " node=" << nid
           << " ctx=" << bn.ctx << " gctx=" << g.nodes[nid].ctx;
        if (bn.op == OP_WAVE || bn.op == OP_HEAVY_BATCH) ls << " n=" << bn.aux[0];
        ls << " in=";
        for (int j = 0; j < bn.n_in; ++j) ls << c.P.body_ivids[F.bi_off + bn.in_off + j] << ",";
        ls << " out=" << bn.out_vid;
        if (bn.op != OP_WAVE && bn.n_out > 0) ls << " dt=" << (int)c.vdt[bn.out_vid];
        ls << "\n";
      }
    }
    c.P.listing = ls.str();
  }
  c.P.vdt = c.vdt;
  c.P.precision = o.precision;
  return std::move(c.P);
}

}  // namespace cf
