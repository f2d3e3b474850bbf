// Host-side IR, builder and autodiff of libcf (C++17). No CUDA here.
//
// Graph construction follows PAPER.md §4.2 (lines 620-667): cond -> Switch/Merge with one
// Switch per captured external tensor and one Merge per output; while_loop -> per loop
// variable Enter/Merge/Switch/NextIteration/Exit, Enter(is_constant) per captured external
// tensor, plus a hidden int64 counter loop variable.
#pragma once
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cf.h"

namespace cf {

struct CfError : std::runtime_error {
  cf_status code;
  CfError(cf_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

enum DT : int32_t { BOOL = CF_BOOL, I32 = CF_I32, I64 = CF_I64, F32 = CF_F32, F64 = CF_F64,
                    BF16 = CF_BF16, FLOW = CF_FLOW, RES = CF_RES };

inline bool is_float(int32_t d) { return d == F32 || d == F64 || d == BF16; }
inline bool differentiable(int32_t d) { return is_float(d) || d == FLOW; }
int dt_size(int32_t d);
const char* dt_name(int32_t d);

using Shape = std::vector<int64_t>;
inline int64_t numel(const Shape& s) { int64_t n = 1; for (auto v : s) n *= v; return n; }

struct TRef {
  int32_t node = -1, port = 0;
  bool operator<(const TRef& o) const { return node != o.node ? node < o.node : port < o.port; }
  bool operator==(const TRef& o) const { return node == o.node && port == o.port; }
  bool operator!=(const TRef& o) const { return !(*this == o); }
  bool valid() const { return node >= 0; }
};

struct Attrs {
  std::map<std::string, std::string> kv;
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  int64_t i(const std::string& k, int64_t d = 0) const;
  double f(const std::string& k, double d = 0) const;
  bool b(const std::string& k, bool d = false) const { return i(k, d ? 1 : 0) != 0; }
  std::string s(const std::string& k, const std::string& d = "") const;
  std::vector<int64_t> v(const std::string& k) const;
  void set(const std::string& k, int64_t x) { kv[k] = std::to_string(x); }
  void setf(const std::string& k, double x);
  void sets(const std::string& k, const std::string& x) { kv[k] = x; }
  void setv(const std::string& k, const std::vector<int64_t>& x);
  static Attrs parse(const char* s);
};

enum CtxKind { ROOT = 0, WHILE = 1, COND = 2 };

// channel id of the gradient edge mirroring a Send/Recv edge
constexpr int64_t kGradChannel = 1 << 20;

struct LoopVar { int enter = -1, merge = -1, sw = -1, next = -1, exit = -1; };

struct Ctx {
  int id = 0;
  CtxKind kind = ROOT;
  int parent = -1;
  std::string name;      // while frame name
  int K = 32;            // parallel_iterations
  TRef pred;             // cond predicate (in parent ctx)
  int branch = -1;       // cond: 1 = true branch (Switch port 1), 0 = false
  int cond_id = -1;
  TRef pivot;
  std::map<TRef, TRef> captured;
  std::vector<LoopVar> loop_vars;   // [0] = hidden counter
  std::vector<int> constants;       // Enter(is_constant) node ids
};

struct Node {
  int id = 0;
  std::string op;
  std::vector<TRef> in;
  std::vector<int> ctrl;
  Attrs attrs;
  int ctx = 0;
  std::vector<int32_t> odt;
  std::vector<Shape> osh;
  std::vector<uint8_t> data;  // Const payload
};

struct Graph {
  std::vector<Node> nodes;
  std::vector<Ctx> ctxs;
  int cur = 0;
  std::map<std::string, int> placeholders;
  std::map<std::string, int> whiles;     // frame name -> ctx id
  std::vector<std::string> frame_order;  // frames in creation order
  int n_conds = 0;

  Graph() { ctxs.push_back(Ctx{}); }

  int32_t dtype(TRef t) const { return nodes.at(t.node).odt.at(t.port); }
  const Shape& shape(TRef t) const { return nodes.at(t.node).osh.at(t.port); }
  int ctx_of(TRef t) const { return nodes.at(t.node).ctx; }
  bool is_ancestor(int anc, int c) const;   // anc == c or anc encloses c
  int enclosing_while(int c) const;

  // raw creation (no capture)
  int add(const std::string& op, const std::vector<TRef>& in, const Attrs& a, int ctx,
          const std::vector<int>& ctrl = {});
  TRef capture(TRef t, int ctx);
  TRef pivot_of(int ctx);
  bool is_capture(TRef t) const;
  std::vector<TRef> op(const std::string& op, const std::vector<TRef>& in, const Attrs& a = {});
  TRef op1(const std::string& o, const std::vector<TRef>& in, const Attrs& a = {}) {
    return op(o, in, a).at(0);
  }
  TRef placeholder(const std::string& name, int32_t dt, const Shape& s);
  TRef constant(int32_t dt, const Shape& s, const void* data);
  TRef const_i64(int64_t v) { return constant(I64, {}, &v); }
  TRef zeros(int32_t dt, const Shape& s);

  std::vector<TRef> cond(TRef pred, const std::function<std::vector<TRef>()>& tf,
                         const std::function<std::vector<TRef>()>& ff);
  std::vector<TRef> while_loop(
      const std::function<TRef(const std::vector<TRef>&)>& pred,
      const std::function<std::vector<TRef>(const std::vector<TRef>&)>& body,
      const std::vector<TRef>& inits, int K, const std::string& name, TRef* counter_exit);

  std::vector<std::string> validate() const;
  std::string json() const;
};

struct CtxGuard {
  Graph& g; int old;
  CtxGuard(Graph& gg, int c) : g(gg), old(gg.cur) { g.cur = c; }
  ~CtxGuard() { g.cur = old; }
};

void infer(const Graph& g, const std::string& op, const std::vector<TRef>& in, const Attrs& a,
           std::vector<int32_t>* odt, std::vector<Shape>* osh);

std::vector<TRef> gradients(Graph& g, TRef y, const std::vector<TRef>& xs);

}  // namespace cf
