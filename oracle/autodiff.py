"""Reverse-mode autodiff through cond / while_loop / TensorArray (test infrastructure only).

Follows PAPER.md §5.1-5.2:

* ``gradients(y, xs)``: the four-step algorithm: Grads[y] := 1, traverse
  the subgraph between y and xs in reverse topological order, call each op's gradient
  function, "Add each di_k to Grads[i_k]".
* Each op belongs to a control-flow context; "When the backpropagation traversal first
  encounters a new control-flow context, it generates a corresponding control-flow construct
  in the gradient graph". The traversal therefore treats a nested cond /
  while as one item of its enclosing context.
* cond: "The gradient for tf.cond(pred, true_fn, false_fn) with output gradients g_z is
  tf.cond(pred, true_fn_grad(g_z), false_fn_grad(g_z))" where each branch gradient applies the
  algorithm to the branch with Grads[t_i] := g_z[i].
* while_loop: (1) a gradient loop running the forward trip count in reverse, driven by the
  hidden counter; (2) loop-variable gradients become gradient-loop variables initialised from
  the gradients of the loop outputs; (3) gradients of loop constants are summed over
  iterations, eagerly, as extra loop variables.
* Forward intermediates needed by the gradient loop are saved on one stack each, pushed in
  the forward loop and popped in the gradient loop; for a cond nested in
  a loop the predicate is such an intermediate, so it is pushed every forward iteration and
  popped to drive the gradient cond. Loop constants (Enter is_constant)
  are not pushed: the gradient graph reads the outer tensor directly.
* TensorArray duality: grad(read) = grad-TA write, grad(write) = grad-TA
  read, grad(unstack) = grad-TA stack, grad(stack) = grad-TA unstack; flows carry ordering.
* MatMul gradient exactly as MatMulGrad.
"""
from __future__ import annotations

import collections
from typing import Dict, List, Optional

from .graph import (BOOL, DIFFERENTIABLE, FLOAT, FLOW, GRAD_CHANNEL, INT, RES, Builder, Ctx,
                    GraphError, Node, T)


class _AD:
    def __init__(self, b: Builder):
        self.b = b
        self.g = b.g
        self.mirror: Dict[int, Ctx] = {self.g.root.id: self.g.root}
        self.stack_of: Dict[T, T] = {}
        self.pop_of: Dict[T, T] = {}

    # ---------------------------------------------------------------- helpers
    def dtype(self, t):
        return self.g.dtype(t)

    def shape(self, t):
        return self.g.shape(t)

    def zeros_like_static(self, t: T) -> T:
        dt = self.dtype(t)
        if dt == FLOW:
            return self.b.const(0.0, FLOW)
        return self.b.zeros(self.shape(t), FLOAT)

    def sum(self, gl: List[T]) -> Optional[T]:
        if not gl:
            return None
        if len(gl) == 1:
            return gl[0]
        return self.b.op1("AddN", gl)

    def fwd(self, t: T) -> T:
        """A forward value referenced from gradient code (TF GetRealValue): loop constants
        resolve to the outer tensor; values inside a forward loop are stack-saved."""
        n = self.g.nodes[t.node]
        if n.op == "Enter" and n.attrs.get("is_constant"):
            return self.fwd(n.inputs[0])
        C = n.ctx
        W = C.enclosing_while()
        if W is None or W.id not in self.mirror:
            return t
        if t in self.pop_of:
            return self.pop_of[t]
        b = self.b
        if t not in self.stack_of:
            with b.in_ctx(W.parent):
                h = b.op1("StackCreate", [], {"frame": W.name, "dtype": self.dtype(t),
                                              "elem_shape": self.shape(t)})
            with b.in_ctx(C):
                b.op("StackPush", [h, t])
            self.stack_of[t] = h
        # a loop nested in another loop ("for nested loops, we apply our
        # techniques recursively"): its stack is created once per outer iteration, in the outer
        # body, so the handle itself is an outer-loop value the gradient needs -- saved on a
        # stack of the outer loop in turn (fwd recursion); the outer gradient iteration pops
        # the handle of its own forward iteration, whose inner gradient loop pops the values
        hp = self.fwd(self.stack_of[t])
        with b.in_ctx(self.mirror[C.id]):
            v = b.op1("StackPop", [hp], {"dtype": self.dtype(t), "elem_shape": self.shape(t)})
        self.pop_of[t] = v
        return v

    def _reduce_to(self, gt: T, like: T, out: T) -> T:
        if self.shape(like) == () and self.shape(out) != ():
            return self.b.op1("ReduceSum", [gt])
        return gt

    # ---------------------------------------------------------------- items
    def _is_machinery(self, n: Node, ctx: Ctx) -> bool:
        if ctx.kind == "cond":
            # capture / pivot Switches of the branch are its leaves
            return (n.op == "Switch" and n.ctx is ctx) or \
                (n.op == "Identity" and n.attrs.get("pivot", False))
        if ctx.kind != "while":
            return False
        if n.op == "Enter" and n.attrs.get("frame") == ctx.name:
            return True
        if n.op in ("Merge", "Switch") and n.attrs.get("loop") and n.attrs.get("frame") == ctx.name:
            return True
        if n.op == "NextIteration" and n.attrs.get("frame") == ctx.name:
            return True
        if n.op == "Identity" and n.attrs.get("pivot"):
            return True
        return False

    def _items(self, ctx: Ctx):
        items: Dict[tuple, dict] = {}
        order = []
        for n in self.g.nodes:
            c = n.ctx
            if c is ctx:
                if self._is_machinery(n, ctx):
                    continue
                if n.op == "Merge" and "cond_id" in n.attrs and not n.attrs.get("loop"):
                    key = ("cond", n.attrs["cond_id"])
                elif n.op == "Exit":
                    key = ("while", n.attrs["frame"])
                else:
                    key = ("node", n.id)
            else:
                cc = c
                while cc is not None and cc.parent is not ctx:
                    cc = cc.parent
                if cc is None:
                    continue
                key = ("cond", cc.cond_id) if cc.kind == "cond" else ("while", cc.name)
            if key not in items:
                items[key] = {"nodes": []}
                order.append(key)
            items[key]["nodes"].append(n)
        for key, it in items.items():
            nodes = it["nodes"]
            if key[0] == "node":
                n = nodes[0]
                it["inputs"] = list(n.inputs)
                it["outputs"] = [T(n.id, p) for p in range(len(n.out_dtypes))]
            elif key[0] == "cond":
                it["outputs"] = [T(m.id, 0) for m in nodes if m.op == "Merge" and m.ctx is ctx]
                it["inputs"] = [t for s in nodes if s.op == "Switch" and s.ctx.parent is ctx
                                and s.ctx.kind == "cond" for t in s.inputs]
            else:
                it["outputs"] = [T(x.id, 0) for x in nodes if x.op == "Exit" and x.ctx is ctx]
                it["inputs"] = [e.inputs[0] for e in nodes if e.op == "Enter"
                                and e.attrs["frame"] == key[1]]
        prod = {}
        for key, it in items.items():
            for n in it["nodes"]:
                prod[n.id] = key
        deps = {k: set() for k in items}
        for key, it in items.items():
            for t in it["inputs"]:
                pk = prod.get(t.node)
                if pk is not None and pk != key:
                    deps[key].add(pk)
        topo, seen = [], set()

        def visit(k):
            if k in seen:
                return
            seen.add(k)
            for d in sorted(deps[k], key=order.index):
                visit(d)
            topo.append(k)
        for k in order:
            visit(k)
        return items, topo

    # ---------------------------------------------------------------- traversal
    def backprop(self, ctx: Ctx, ups: Dict[T, List[T]], wrt: List[T]) -> Dict[T, T]:
        items, topo = self._items(ctx)
        from_wrt = set(wrt)
        # Send/Recv pairs carry the dependence across partitions: a Recv's
        # value depends on the peer's parameters, and every Send/Recv gets its mirrored
        # gradient message, so items holding one are never pruned (else a peer would wait).
        comm = {k: any(n.op in ("Send", "Recv") for n in items[k]["nodes"]) for k in topo}
        recv = {k: any(n.op == "Recv" for n in items[k]["nodes"]) for k in topo}
        for k in topo:
            it = items[k]
            if any(t in from_wrt for t in it["inputs"]) or recv[k]:
                from_wrt.update(it["outputs"])
        grads: Dict[T, List[T]] = collections.defaultdict(list)
        for t, gl in ups.items():
            grads[t].extend(gl if isinstance(gl, list) else [gl])
        for k in reversed(topo):
            it = items[k]
            g_outs = [self.sum(grads[o]) if grads.get(o) else None for o in it["outputs"]]
            for o, go in zip(it["outputs"], g_outs):
                if go is not None:
                    grads[o] = [go]
            if all(go is None for go in g_outs) and not comm[k]:
                continue
            if not any(t in from_wrt for t in it["inputs"]) and not comm[k]:
                continue
            if k[0] == "node":
                pairs = zip(it["inputs"], self.op_grad(it["nodes"][0], g_outs))
            elif k[0] == "cond":
                pairs = self.cond_grad(ctx, k[1], it, g_outs)
            else:
                pairs = self.while_grad(ctx, k[1], it, g_outs)
            for t, gt in pairs:
                if gt is not None and t in from_wrt and self.dtype(t) in DIFFERENTIABLE:
                    grads[t].append(gt)
        return {t: self.sum(grads[t]) for t in wrt if grads.get(t)}

    # ---------------------------------------------------------------- constructs
    def cond_grad(self, ctx, cond_id, it, g_outs):
        """tf.cond(pred, true_fn_grad(g_z), false_fn_grad(g_z))."""
        b = self.b
        merges = [self.g.nodes[o.node] for o in it["outputs"]]
        branch_ctx = {}
        captures = {0: [], 1: []}
        pred = None
        for n in it["nodes"]:
            if n.ctx.kind == "cond" and n.ctx.parent is ctx and n.ctx.cond_id == cond_id:
                branch_ctx[n.ctx.branch] = n.ctx
                if n.op == "Switch" and n.attrs.get("capture"):
                    captures[n.ctx.branch].append((n.inputs[0], T(n.id, n.ctx.branch)))
                if n.op == "Switch":
                    pred = n.inputs[1]
        externals = []
        for br in (1, 0):
            for e, _ in captures[br]:
                if e not in externals and self.dtype(e) in DIFFERENTIABLE:
                    externals.append(e)
        if not externals and not any(n.op in ("Send", "Recv") for n in it["nodes"]):
            return []
        pred_g = self.fwd(pred)

        def make(br):
            def fn():
                bc = branch_ctx.get(br)
                if bc is not None:
                    self.mirror[bc.id] = b.cur
                ups = {}
                for (m, go) in zip(merges, g_outs):
                    if go is not None:
                        ups.setdefault(m.inputs[br], []).append(go)
                leaves = [s for e, s in captures[br]]
                gd = self.backprop(bc, ups, leaves) if bc is not None else {}
                res = []
                for e in externals:
                    gs = [gd[s] for ee, s in captures[br] if ee == e and s in gd]
                    res.append(self.sum(gs) if gs else self.zeros_like_static(e))
                return res
            return fn

        outs = b.cond(pred_g, make(1), make(0))
        return list(zip(externals, outs))

    def while_grad(self, ctx, name, it, g_outs):
        """Gradient loop per PAPER.md:1022-1035 features 1-3."""
        b = self.b
        W = self.g.whiles[name]
        lv = W.loop_vars
        exit_ids = [o.node for o in it["outputs"]]
        g_exit = dict(zip(exit_ids, g_outs))
        counter_exit = T(lv[0]["exit"], 0)
        n_trip = self.fwd(counter_exit)
        var_js = [j for j in range(1, len(lv))
                  if self.g.nodes[lv[j]["enter"]].out_dtypes[0] in DIFFERENTIABLE]
        consts = [self.g.nodes[e] for e in W.constants
                  if self.g.nodes[e].out_dtypes[0] in DIFFERENTIABLE]
        inits = [n_trip]
        for j in var_js:
            ge = g_exit.get(lv[j]["exit"])
            inits.append(ge if ge is not None else
                         self.zeros_like_static(self.g.nodes[lv[j]["enter"]].inputs[0]))
        for e in consts:
            inits.append(self.zeros_like_static(e.inputs[0]))
        nv = len(var_js)

        def pred(k, *rest):
            return b.op1("Greater", [k, b.const(0, INT)])

        def body(k, *vals):
            self.mirror[W.id] = b.cur
            gs, accs = vals[:nv], vals[nv:]
            ups = {}
            for j, gj in zip(var_js, gs):
                nxt = self.g.nodes[lv[j]["next"]].inputs[0]
                ups.setdefault(nxt, []).append(gj)
            leaves = [T(lv[j]["switch"], 1) for j in var_js] + [T(e.id, 0) for e in consts]
            gd = self.backprop(W, ups, leaves)
            new_gs = []
            for j in var_js:
                s = T(lv[j]["switch"], 1)
                new_gs.append(gd[s] if s in gd else
                              self.zeros_like_static(self.g.nodes[lv[j]["enter"]].inputs[0]))
            new_accs = []
            for e, acc in zip(consts, accs):
                s = T(e.id, 0)
                new_accs.append(b.add(acc, gd[s]) if s in gd else acc)
            return [b.op1("Sub", [k, b.const(1, INT)])] + new_gs + new_accs

        outs = b.while_loop(pred, body, inits, parallel_iterations=W.K, name=name + "_grad")
        pairs = []
        for j, o in zip(var_js, outs[1:1 + nv]):
            pairs.append((self.g.nodes[lv[j]["enter"]].inputs[0], o))
        for e, o in zip(consts, outs[1 + nv:]):
            pairs.append((e.inputs[0], o))
        return pairs

    # ---------------------------------------------------------------- op gradients
    def op_grad(self, n: Node, g_outs: List[Optional[T]]) -> List[Optional[T]]:
        b = self.b
        op = n.op
        g = g_outs[0] if g_outs else None
        out = T(n.id, 0)
        ins = n.inputs
        F = self.fwd
        if op in ("Identity", "Cast"):
            return [g]
        if op == "Send":
            # the gradient of a sent value comes back from the receiver on the mirrored edge
            v = ins[0]
            return [b.recv(F(ins[1]), n.attrs["channel"] ^ GRAD_CHANNEL, n.attrs["peer"],
                           self.dtype(v), self.shape(v)), None]
        if op == "Recv":
            gv = g if g is not None else self.zeros_like_static(out)
            b.send(gv, F(ins[0]), n.attrs["channel"] ^ GRAD_CHANNEL, n.attrs["peer"])
            return [None]
        if op in ("StopGradient", "Placeholder", "Const", "ZerosLike", "Less", "LessEqual",
                  "Greater", "Equal", "LogicalAnd", "LogicalNot", "ReduceMax", "ReduceMin",
                  "TACreate", "StackCreate", "StackPush", "StackPop", "TAGrad"):
            return [None] * len(ins)
        if op == "Add":
            return [self._reduce_to(g, ins[0], out), self._reduce_to(g, ins[1], out)]
        if op == "Sub":
            return [self._reduce_to(g, ins[0], out),
                    self._reduce_to(b.op1("Neg", [g]), ins[1], out)]
        if op == "AddN":
            return [g] * len(ins)
        if op == "Mul":
            return [self._reduce_to(b.mul(g, F(ins[1])), ins[0], out),
                    self._reduce_to(b.mul(g, F(ins[0])), ins[1], out)]
        if op == "Neg":
            return [b.op1("Neg", [g])]
        if op == "MatMul":
            # MatMulGrad: g_x = g_z y^T, g_y = x^T g_z
            x, y = F(ins[0]), F(ins[1])
            ta, tb = n.attrs.get("ta", False), n.attrs.get("tb", False)
            if not ta and not tb:
                return [b.matmul(g, y, tb=True), b.matmul(x, g, ta=True)]
            if ta and not tb:
                return [b.matmul(y, g, tb=True), b.matmul(x, g)]
            if not ta and tb:
                return [b.matmul(g, y), b.matmul(g, x, ta=True)]
            return [b.matmul(y, g, ta=True, tb=True), b.matmul(g, x, ta=True, tb=True)]
        if op == "Transpose":
            return [b.op1("Transpose", [g])]
        if op == "BiasAdd":
            return [g, b.op1("ReduceSum", [g], {"axis": 0})]
        if op == "ReduceSum" and n.attrs.get("axis") == 0:
            raise GraphError("CF_E_NO_GRADIENT", "no gradient for ReduceSum(axis=0)")
        if op == "ReduceSum":
            # "The gradient of reduce_sum is broadcast"
            return [b.op1("Fill", [g], {"shape": self.shape(ins[0])})]
        if op == "Fill":
            return [b.op1("ReduceSum", [g])]
        if op == "Sigmoid":
            y = F(out)
            return [b.mul(g, b.mul(y, b.sub(b.const(1.0), y)))]
        if op == "Tanh":
            y = F(out)
            return [b.mul(g, b.sub(b.const(1.0), b.mul(y, y)))]
        if op == "Relu":
            return [b.op1("ReluGrad", [g, F(out)])]
        if op == "Select":
            c = F(ins[0])
            z = b.op1("ZerosLike", [g])
            return [None, b.op1("Select", [c, g, z]), b.op1("Select", [c, z, g])]
        if op == "Concat":
            ax = n.attrs["axis"]
            res, off = [], 0
            for t in ins:
                s = self.shape(t)
                begin = [0] * len(s)
                begin[ax] = off
                off += s[ax]
                res.append(b.op1("Slice", [g], {"begin": tuple(begin), "size": tuple(s)}))
            return res
        if op == "Slice":
            return [b.op1("SliceGrad", [g], {"shape": self.shape(ins[0]),
                                             "begin": n.attrs["begin"], "size": n.attrs["size"]})]
        if op == "Reshape":
            return [b.op1("Reshape", [g], {"shape": self.shape(ins[0])})]
        if op == "LSTMCell":
            masked = n.attrs.get("masked", False)
            ups = []
            for p in range(3):
                gp = g_outs[p]
                ups.append(gp if gp is not None else self.zeros_like_static(T(n.id, p)))
            fin = [F(ins[0]), F(ins[1]), F(ins[2]), F(ins[3]), F(T(n.id, 3))]
            if masked:
                fin += [F(ins[5]), F(ins[6])]
            gr = b.op("LSTMCellGrad", fin + ups, {"masked": masked,
                                                  "forget_bias": n.attrs.get("forget_bias", 0.0)})
            res = [gr[0], gr[1], gr[2], gr[3], gr[4]]
            if masked:
                res += [None, None]
            return res
        # ---- TensorArray duality, flows per TF
        if op == "TARead":
            h, ix, flow = ins
            gh, gf = b.op("TAGrad", [F(h), F(flow)])
            wf = b.op1("TAWrite", [gh, F(ix), g, gf], dict(n.attrs))
            return [None, None, wf]
        if op == "TAWrite":
            h, ix, v, flow = ins
            gh, gf = b.op("TAGrad", [F(h), g])
            gv = b.op1("TARead", [gh, F(ix), gf], dict(n.attrs))
            return [None, None, gv, g]
        if op == "TAStack":
            h, flow = ins
            gh, gf = b.op("TAGrad", [F(h), F(flow)])
            uf = b.op1("TAUnstack", [gh, g, gf], dict(n.attrs))
            return [None, uf]
        if op == "TAUnstack":
            h, v, flow = ins
            gh, gf = b.op("TAGrad", [F(h), g])
            gv = b.op1("TAStack", [gh, gf], dict(n.attrs))
            return [None, gv, g]
        raise GraphError("CF_E_NO_GRADIENT", f"no gradient for op {op}")


def gradients(b: Builder, y: T, xs: List[T]) -> List[T]:
    """tf.gradients(y, xs)."""
    g = b.g
    if g.dtype(y) != FLOAT or g.shape(y) != ():
        raise GraphError("CF_E_NONSCALAR_OBJECTIVE", "y must be a float scalar")
    if g.ctx_of(y) is not g.root:
        raise GraphError("CF_E_INVALID_GRAPH", "y must be a root-context tensor")
    ad = _AD(b)
    with b.in_ctx(g.root):
        one = b.const(1.0)
        gd = ad.backprop(g.root, {y: [one]}, list(xs))
        return [gd[x] if x in gd else ad.zeros_like_static(x) for x in xs]
