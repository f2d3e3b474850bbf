"""Oracle IR and builder (test infrastructure only; see oracle/__init__.py).

Graph construction follows PAPER.md §4.2 "Compilation of Control-Flow Constructs"
(lines 620-667):

* ``cond(p, true_fn, false_fn)`` uses only Switch and Merge; "we capture any external tensor
  (not created in the branch), and insert a Switch to guard its entering into the branch"
  with "one Switch for each external tensor" and "For each output, we add a Merge"
  (PAPER.md:624-637).
* ``while_loop(pred, body, inits)``: per loop variable Enter -> Merge -> G_pred -> Switch ->
  G_body -> NextIteration -> Merge, Switch-false -> Exit; "We automatically insert an Enter
  for each external tensor" (loop constants).
* A hidden counter loop variable is always added, because "the forward loop must be augmented
  with a loop counter" (SPEC.md:193 makes it unconditional).
* TensorArray read/write/stack/unstack thread a "flow" scalar for ordering.

Zero-input ops (and ops whose inputs are all captured externals) created inside a cond
branch or loop body get a control input from the construct's *pivot* (the Switch output that
carries the branch / loop predicate), so that they execute once per frame and are dead on
untaken branches and on the exiting iteration -- the reading of "each operation executes at
most once per frame" for operations with no data inputs (reading R7).
"""
from __future__ import annotations

import contextlib
import dataclasses
from typing import Any, Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

FLOAT = "f64"
INT = "i64"
GRAD_CHANNEL = 1 << 20     # channel id of the gradient edge mirroring a Send/Recv edge
BOOL = "bool"
FLOW = "flow"   # TensorArray flow scalar (ordering token); differentiable (TF convention)
RES = "res"     # resource handle (TensorArray, Stack)

DIFFERENTIABLE = (FLOAT, FLOW)

CONTROL_OPS = ("Switch", "Merge", "Enter", "Exit", "NextIteration")


class GraphError(Exception):
    """Build-time error; ``code`` mirrors the C-ABI status names."""

    def __init__(self, code: str, msg: str):
        super().__init__(f"{code}: {msg}")
        self.code = code


@dataclasses.dataclass(frozen=True)
class T:
    """Symbolic tensor = (producer node id, output port)."""
    node: int
    port: int = 0


@dataclasses.dataclass
class Ctx:
    kind: str                      # "root" | "while" | "cond"
    parent: Optional["Ctx"] = None
    name: str = ""                 # frame name (while)
    K: int = 32                    # parallel_iterations (while)
    pred: Optional[T] = None       # cond predicate (lives in parent ctx)
    branch: int = -1               # cond: 1 = true, 0 = false (Switch port, reading R6)
    cond_id: int = -1
    pivot: Optional[T] = None
    captured: Dict[T, T] = dataclasses.field(default_factory=dict)
    # while bookkeeping
    loop_vars: List[dict] = dataclasses.field(default_factory=list)
    constants: List[int] = dataclasses.field(default_factory=list)  # Enter(is_constant) ids
    id: int = 0

    def ancestors(self):
        c = self
        while c is not None:
            yield c
            c = c.parent

    def enclosing_while(self) -> Optional["Ctx"]:
        for c in self.ancestors():
            if c.kind == "while":
                return c
        return None


@dataclasses.dataclass
class Node:
    id: int
    op: str
    inputs: List[T]
    ctrl: List[int]
    attrs: Dict[str, Any]
    ctx: Ctx
    out_dtypes: List[str]
    out_shapes: List[Optional[Tuple[int, ...]]]


class Graph:
    def __init__(self):
        self.nodes: List[Node] = []
        self.root = Ctx("root", id=0)
        self.ctxs: List[Ctx] = [self.root]
        self.placeholders: Dict[str, int] = {}
        self.n_conds = 0
        self.whiles: Dict[str, Ctx] = {}

    def dtype(self, t: T) -> str:
        return self.nodes[t.node].out_dtypes[t.port]

    def shape(self, t: T):
        return self.nodes[t.node].out_shapes[t.port]

    def ctx_of(self, t: T) -> Ctx:
        return self.nodes[t.node].ctx

    def consumers(self):
        """(node, port) -> list of (consumer id, consumer input index)."""
        cons: Dict[Tuple[int, int], List[Tuple[int, int]]] = {}
        for n in self.nodes:
            for i, t in enumerate(n.inputs):
                cons.setdefault((t.node, t.port), []).append((n.id, i))
        return cons

    def count_ops(self) -> Dict[str, int]:
        out: Dict[str, int] = {}
        for n in self.nodes:
            out[n.op] = out.get(n.op, 0) + 1
        return out


# ----------------------------------------------------------------------------------------
# shape / dtype inference
# ----------------------------------------------------------------------------------------

def _bcast(sa, sb):
    if sa == sb:
        return sa
    if sa == ():
        return sb
    if sb == ():
        return sa
    raise GraphError("CF_E_SHAPE", f"incompatible shapes {sa} {sb}")


def infer(g: Graph, op: str, inputs: Sequence[T], attrs: Dict[str, Any]):
    dt = [g.dtype(t) for t in inputs]
    sh = [g.shape(t) for t in inputs]

    def need(n):
        if len(inputs) != n:
            raise GraphError("CF_E_ARITY", f"{op} expects {n} inputs, got {len(inputs)}")

    if op == "Placeholder":
        return [attrs["dtype"]], [tuple(attrs["shape"])]
    if op == "Const":
        v = attrs["value"]
        return [attrs["dtype"]], [tuple(np.shape(v))]
    if op in ("Identity", "Neg", "Sigmoid", "Tanh", "Relu", "ZerosLike", "StopGradient"):
        need(1)
        if op not in ("Identity", "ZerosLike", "StopGradient") and dt[0] != FLOAT:
            raise GraphError("CF_E_DTYPE", f"{op} on {dt[0]}")
        return [dt[0]], [sh[0]]
    if op in ("Add", "Sub", "Mul"):
        need(2)
        if dt[0] != dt[1] or dt[0] in (BOOL, RES):
            raise GraphError("CF_E_DTYPE", f"{op} dtypes {dt}")
        return [dt[0]], [_bcast(sh[0], sh[1])]
    if op == "AddN":
        if not inputs:
            raise GraphError("CF_E_ARITY", "AddN of nothing")
        for d, s in zip(dt, sh):
            if d != dt[0] or s != sh[0]:
                raise GraphError("CF_E_SHAPE", "AddN mismatch")
        return [dt[0]], [sh[0]]
    if op == "ReluGrad":
        need(2)
        return [FLOAT], [sh[0]]
    if op == "MatMul":
        need(2)
        if dt[0] != FLOAT or dt[1] != FLOAT:
            raise GraphError("CF_E_DTYPE", "MatMul on non-float")
        a, b = sh
        if len(a) != 2 or len(b) != 2:
            raise GraphError("CF_E_SHAPE", "MatMul needs rank 2")
        m, k1 = (a[1], a[0]) if attrs.get("ta") else a
        k2, n = (b[1], b[0]) if attrs.get("tb") else b
        if k1 != k2:
            raise GraphError("CF_E_SHAPE", f"MatMul inner {k1} != {k2}")
        return [FLOAT], [(m, n)]
    if op == "Transpose":
        need(1)
        return [dt[0]], [tuple(reversed(sh[0]))]
    if op in ("ReduceSum", "ReduceMax", "ReduceMin"):
        need(1)
        if attrs.get("axis") == 0:
            return [dt[0]], [tuple(sh[0][1:])]
        return [dt[0]], [()]
    if op == "BiasAdd":
        need(2)
        if len(sh[0]) != 2 or sh[1] != (sh[0][1],):
            raise GraphError("CF_E_SHAPE", f"BiasAdd shapes {sh}")
        return [dt[0]], [sh[0]]
    if op == "Fill":
        need(1)
        if sh[0] != ():
            raise GraphError("CF_E_SHAPE", "Fill value must be scalar")
        return [dt[0]], [tuple(attrs["shape"])]
    if op in ("Less", "LessEqual", "Greater", "Equal"):
        need(2)
        if dt[0] != dt[1]:
            raise GraphError("CF_E_DTYPE", f"{op} dtypes {dt}")
        return [BOOL], [_bcast(sh[0], sh[1])]
    if op == "LogicalAnd":
        need(2)
        return [BOOL], [_bcast(sh[0], sh[1])]
    if op == "LogicalNot":
        need(1)
        return [BOOL], [sh[0]]
    if op == "Select":
        need(3)
        if dt[0] != BOOL:
            raise GraphError("CF_E_DTYPE", "Select condition must be bool")
        return [dt[1]], [_bcast(sh[1], sh[2])]
    if op == "Concat":
        ax = attrs["axis"]
        s = list(sh[0])
        s[ax] = sum(x[ax] for x in sh)
        return [dt[0]], [tuple(s)]
    if op == "Slice":
        need(1)
        return [dt[0]], [tuple(attrs["size"])]
    if op == "SliceGrad":   # pad g (shape = size) into zeros of attrs["shape"] at begin
        need(1)
        return [dt[0]], [tuple(attrs["shape"])]
    if op == "Reshape":
        need(1)
        return [dt[0]], [tuple(attrs["shape"])]
    if op == "Cast":
        need(1)
        return [attrs["dtype"]], [sh[0]]
    if op == "LSTMCell":
        # inputs x[B,I], h[B,H], c[B,H], W[4H,I+H], b[4H] (+ t scalar, len[B] when masked)
        need(7 if attrs.get("masked") else 5)
        B, I = sh[0]
        H = sh[1][1]
        if sh[3] != (4 * H, I + H) or sh[4] != (4 * H,) or sh[2] != (B, H):
            raise GraphError("CF_E_SHAPE", f"LSTMCell shapes {sh}")
        return [FLOAT] * 4, [(B, H), (B, H), (B, H), (B, 4 * H)]
    if op == "LSTMCellGrad":
        # x, h, c, W, gates, [t, len], dh_next, dc_next, dout
        need(10 if attrs.get("masked") else 8)
        B, I = sh[0]
        H = sh[1][1]
        return [FLOAT] * 5, [(B, I), (B, H), (B, H), (4 * H, I + H), (4 * H,)]
    # ---- control-flow primitives
    if op == "Switch":
        need(2)
        if dt[1] != BOOL or sh[1] != ():
            raise GraphError("CF_E_NONBOOL_PRED", "Switch predicate must be a bool scalar")
        return [dt[0], dt[0]], [sh[0], sh[0]]
    if op == "Merge":
        need(2)
        if dt[0] != dt[1]:
            raise GraphError("CF_E_BRANCH_MISMATCH", f"Merge dtypes {dt}")
        return [dt[0]], [sh[0] if sh[0] == sh[1] else None]
    if op in ("Enter", "Exit", "NextIteration"):
        need(1)
        return [dt[0]], [sh[0]]
    # ---- TensorArray and stacks
    if op == "TACreate":
        return [RES, FLOW], [(), ()]
    if op == "TARead":
        need(3)
        return [attrs["dtype"]], [tuple(attrs["elem_shape"])]
    if op == "TAWrite":
        need(4)
        return [FLOW], [()]
    if op == "TAStack":
        need(2)
        return [attrs["dtype"]], [(attrs["size"],) + tuple(attrs["elem_shape"])]
    if op == "TAUnstack":
        need(3)
        return [FLOW], [()]
    if op == "TAGrad":
        need(2)
        return [RES, FLOW], [(), ()]
    if op == "StackCreate":
        return [RES], [()]
    if op == "StackPush":
        need(2)
        return [], []
    if op == "StackPop":
        need(1)
        return [attrs["dtype"]], [tuple(attrs["elem_shape"]) if attrs.get("elem_shape") is not None else None]
    # ---- cross-device Send / Recv (§4.4): rendezvous on (channel, tag)
    if op == "Send":
        need(2)     # value, ix (a scalar of the sending context; places the op in it)
        return [], []
    if op == "Recv":
        need(1)     # ix (a scalar of the receiving context)
        return [attrs["dtype"]], [tuple(attrs["shape"])]
    raise GraphError("CF_E_UNSUPPORTED", f"unknown op {op}")


# ----------------------------------------------------------------------------------------
# builder
# ----------------------------------------------------------------------------------------

class TensorArray:
    """Builder-side TensorArray handle: handle + current flow."""

    def __init__(self, b: "Builder", size: int, dtype: str, elem_shape, handle: T, flow: T):
        self.b, self.size, self.dtype, self.elem_shape = b, size, dtype, tuple(elem_shape)
        self.handle, self.flow = handle, flow

    def _attrs(self):
        return {"dtype": self.dtype, "elem_shape": self.elem_shape, "size": self.size}

    def with_flow(self, flow: T) -> "TensorArray":
        return TensorArray(self.b, self.size, self.dtype, self.elem_shape, self.handle, flow)

    def read(self, ix: T) -> T:
        return self.b.op("TARead", [self.handle, ix, self.flow], self._attrs())[0]

    def write(self, ix: T, v: T) -> "TensorArray":
        f = self.b.op("TAWrite", [self.handle, ix, v, self.flow], self._attrs())[0]
        return self.with_flow(f)

    def stack(self) -> T:
        return self.b.op("TAStack", [self.handle, self.flow], self._attrs())[0]

    def unstack(self, v: T) -> "TensorArray":
        f = self.b.op("TAUnstack", [self.handle, v, self.flow], self._attrs())[0]
        return self.with_flow(f)


class Builder:
    """Graph construction API (§2.1)."""

    def __init__(self, g: Optional[Graph] = None):
        self.g = g or Graph()
        self.cur = self.g.root

    # ---- contexts -------------------------------------------------------------------
    @contextlib.contextmanager
    def in_ctx(self, c: Ctx):
        old = self.cur
        self.cur = c
        try:
            yield
        finally:
            self.cur = old

    def _new_ctx(self, **kw) -> Ctx:
        c = Ctx(id=len(self.g.ctxs), **kw)
        self.g.ctxs.append(c)
        return c

    # ---- raw node creation ------------------------------------------------------------
    def _add(self, op, inputs, attrs=None, ctrl=None, ctx=None) -> Node:
        attrs = dict(attrs or {})
        dts, shs = infer(self.g, op, inputs, attrs)
        n = Node(len(self.g.nodes), op, list(inputs), list(ctrl or []), attrs,
                 ctx or self.cur, dts, shs)
        self.g.nodes.append(n)
        return n

    def capture(self, t: T, c: Optional[Ctx] = None) -> T:
        """Make tensor ``t`` usable in ctx ``c``: Enter(is_constant) into loops, Switch into
        cond branches, recursively."""
        c = c or self.cur
        d = self.g.ctx_of(t)
        if d is c:
            return t
        if c.kind == "root" or d not in list(c.ancestors()):
            raise GraphError("CF_E_INVALID_GRAPH",
                             "tensor used outside its control-flow context without Exit/Merge")
        tp = self.capture(t, c.parent)
        if tp in c.captured:
            return c.captured[tp]
        if c.kind == "while":
            n = self._add("Enter", [tp], {"frame": c.name, "is_constant": True}, ctx=c)
            c.constants.append(n.id)
            out = T(n.id, 0)
        elif c.kind == "cond":
            pred = self.capture(c.pred, c.parent)
            n = self._add("Switch", [tp, pred], {"capture": True, "cond_id": c.cond_id}, ctx=c)
            out = T(n.id, c.branch)
        else:  # pragma: no cover
            raise GraphError("CF_E_INVALID_GRAPH", "bad capture")
        c.captured[tp] = out
        return out

    def _pivot(self, c: Ctx) -> T:
        # while ctx: the counter Merge while the predicate is built (every iteration incl.
        # the exiting one), then the body pivot Identity(Switch_true(counter)).
        if c.pivot is None:
            assert c.kind == "cond"
            p = self.capture(c.pred, c.parent)
            sw = self._add("Switch", [p, p], {"pivot": True, "cond_id": c.cond_id}, ctx=c)
            piv = self._add("Identity", [T(sw.id, c.branch)], {"pivot": True}, ctx=c)
            c.pivot = T(piv.id, 0)
        return c.pivot

    def _is_capture(self, t: T) -> bool:
        n = self.g.nodes[t.node]
        return (n.op == "Enter" and n.attrs.get("is_constant")) or \
               (n.op == "Switch" and n.attrs.get("capture"))

    def op(self, op: str, inputs: Sequence[T], attrs=None) -> List[T]:
        """Create op ``op`` in the current context, capturing external inputs."""
        ins = [self.capture(t) for t in inputs]
        ctrl = []
        # zero-input ops need the pivot in any construct; in a loop body, ops whose inputs are
        # all loop constants would otherwise also run on the exiting iteration
        if (self.cur.kind == "cond" and not ins) or \
                (self.cur.kind == "while" and all(self._is_capture(t) for t in ins)):
            ctrl = [self._pivot(self.cur).node]
        n = self._add(op, ins, attrs, ctrl)
        return [T(n.id, i) for i in range(len(n.out_dtypes))]

    def op1(self, op, inputs, attrs=None) -> T:
        return self.op(op, inputs, attrs)[0]

    # ---- sources ------------------------------------------------------------------
    def placeholder(self, name: str, dtype: str, shape) -> T:
        n = self._add("Placeholder", [], {"name": name, "dtype": dtype, "shape": tuple(shape)},
                      ctx=self.g.root)
        self.g.placeholders[name] = n.id
        return T(n.id, 0)

    def const(self, value, dtype: Optional[str] = None) -> T:
        v = np.asarray(value)
        if dtype is None:
            dtype = BOOL if v.dtype == bool else (INT if np.issubdtype(v.dtype, np.integer) else FLOAT)
        v = v.astype({FLOAT: np.float64, FLOW: np.float64, INT: np.int64, BOOL: bool}[dtype])
        return self.op1("Const", [], {"value": v, "dtype": dtype})

    def zeros(self, shape, dtype=FLOAT) -> T:
        return self.const(np.zeros(shape), dtype)

    # ---- convenience ops ----------------------------------------------------------------
    def add(self, a, b): return self.op1("Add", [a, b])
    def sub(self, a, b): return self.op1("Sub", [a, b])
    def mul(self, a, b): return self.op1("Mul", [a, b])
    def matmul(self, a, b, ta=False, tb=False): return self.op1("MatMul", [a, b], {"ta": ta, "tb": tb})
    def less(self, a, b): return self.op1("Less", [a, b])

    # Send / Recv between partitions. `channel` names the edge; the message
    # key is (channel, iteration tag), so a Send and its Recv must sit in mirrored contexts.
    def send(self, v: T, ix: T, channel: int, peer: int) -> None:
        self.op("Send", [v, ix], {"channel": channel, "peer": peer})

    def recv(self, ix: T, channel: int, peer: int, dtype: str, shape) -> T:
        return self.op1("Recv", [ix], {"channel": channel, "peer": peer, "dtype": dtype,
                                       "shape": tuple(shape)})
    def reduce_sum(self, a): return self.op1("ReduceSum", [a])

    # ---- cond -------------------------------------------------------
    def cond(self, pred: T, true_fn: Callable[[], Sequence[T]],
             false_fn: Callable[[], Sequence[T]]) -> List[T]:
        if self.g.dtype(pred) != BOOL or self.g.shape(pred) != ():
            raise GraphError("CF_E_NONBOOL_PRED", "cond predicate must be a bool scalar")
        pred = self.capture(pred)
        cid = self.g.n_conds
        self.g.n_conds += 1
        outs = {}
        for branch, fn in ((1, true_fn), (0, false_fn)):
            c = self._new_ctx(kind="cond", parent=self.cur, pred=pred, branch=branch, cond_id=cid)
            with self.in_ctx(c):
                r = [self.capture(t) for t in fn()]
            outs[branch] = r
        if len(outs[0]) != len(outs[1]):
            raise GraphError("CF_E_BRANCH_MISMATCH", "branches return different arity")
        merges = []
        for f, t in zip(outs[0], outs[1]):
            if self.g.dtype(f) != self.g.dtype(t):
                raise GraphError("CF_E_BRANCH_MISMATCH", "branch dtypes differ")
            n = self._add("Merge", [f, t], {"cond_id": cid})
            merges.append(T(n.id, 0))
        return merges

    # ---- while_loop ---------------------------------------------------
    def while_loop(self, pred_fn, body_fn, inits: Sequence[T], parallel_iterations: int = 32,
                   name: Optional[str] = None, return_counter: bool = False):
        if parallel_iterations < 1:
            raise GraphError("CF_E_ARITY", "parallel_iterations must be >= 1")
        name = name or f"while{len(self.g.whiles)}"
        if name in self.g.whiles:
            raise GraphError("CF_E_INVALID_GRAPH", f"duplicate frame {name}")
        parent = self.cur
        counter0 = self.const(0, INT)
        all_inits = [counter0] + [self.capture(t) for t in inits]
        c = self._new_ctx(kind="while", parent=parent, name=name, K=parallel_iterations)
        self.g.whiles[name] = c
        lv = []
        for t in all_inits:
            e = self._add("Enter", [t], {"frame": name, "is_constant": False}, ctx=c)
            m = self._add("Merge", [T(e.id, 0), T(e.id, 0)], {"loop": True, "frame": name}, ctx=c)
            lv.append({"enter": e.id, "merge": m.id})
        c.pivot = T(lv[0]["merge"], 0)
        with self.in_ctx(c):
            p = pred_fn(*[T(v["merge"], 0) for v in lv[1:]])
            if self.g.dtype(p) != BOOL or self.g.shape(p) != ():
                raise GraphError("CF_E_NONBOOL_PRED", "loop predicate must be a bool scalar")
            p = self.capture(p)
        for v in lv:
            s = self._add("Switch", [T(v["merge"], 0), p], {"loop": True, "frame": name}, ctx=c)
            v["switch"] = s.id
            x = self._add("Exit", [T(s.id, 0)], {"frame": name}, ctx=parent)
            v["exit"] = x.id
        piv = self._add("Identity", [T(lv[0]["switch"], 1)], {"pivot": True}, ctx=c)
        c.pivot = T(piv.id, 0)
        with self.in_ctx(c):
            body_in = [T(v["switch"], 1) for v in lv[1:]]
            outs = list(body_fn(*body_in))
            if len(outs) != len(inits):
                raise GraphError("CF_E_ARITY", "body returns wrong number of loop variables")
            outs = [self.capture(t) for t in outs]
            cnext = self.op1("Add", [T(lv[0]["switch"], 1), self.const(1, INT)])
        for v, o in zip(lv, [cnext] + outs):
            merge = self.g.nodes[v["merge"]]
            if self.g.dtype(o) != merge.out_dtypes[0]:
                raise GraphError("CF_E_DTYPE", "body output dtype differs from loop variable")
            ni = self._add("NextIteration", [o], {"frame": name}, ctx=c)
            v["next"] = ni.id
            merge.inputs[1] = T(ni.id, 0)
        c.loop_vars = lv
        res = [T(v["exit"], 0) for v in lv[1:]]
        if return_counter:
            return res, T(lv[0]["exit"], 0)
        return res

    # ---- TensorArray --------------------------------------------------------------------
    def tensor_array(self, size: int, dtype: str, elem_shape) -> TensorArray:
        h, f = self.op("TACreate", [], {"size": int(size), "dtype": dtype,
                                         "elem_shape": tuple(elem_shape)})
        return TensorArray(self, size, dtype, elem_shape, h, f)

    def ta_in_loop(self, ta: TensorArray, flow: T) -> TensorArray:
        return ta.with_flow(flow)

    # ---- scan (Fig. "scan") ------------------------------------------------
    def scan(self, fn, elems: T, init: T, parallel_iterations: int = 32) -> T:
        n = self.g.shape(elems)[0]
        elem_ta = self.tensor_array(n, self.g.dtype(elems), self.g.shape(elems)[1:]).unstack(elems)
        result_ta = self.tensor_array(n, self.g.dtype(init), self.g.shape(init))
        nt = self.const(n, INT)

        def pred(i, a, flow):
            return self.less(i, nt)

        def body(i, a, flow):
            a_out = fn(a, elem_ta.read(i))
            flow2 = result_ta.with_flow(flow).write(i, a_out).flow
            return (self.add(i, self.const(1, INT)), a_out, flow2)

        _, _, rflow = self.while_loop(pred, body, (self.const(0, INT), init, result_ta.flow),
                                      parallel_iterations)
        return result_ta.with_flow(rflow).stack()


def validate(g: Graph) -> List[str]:
    """Structural checks: Merge/Switch arity, cycles only through
    NextIteration, no context crossing without Enter/Exit/Switch/Merge."""
    errs = []
    for n in g.nodes:
        if n.op == "Merge" and len(n.inputs) != 2:
            errs.append(f"node {n.id}: Merge arity {len(n.inputs)}")
        if n.op == "Switch" and len(n.inputs) != 2:
            errs.append(f"node {n.id}: Switch arity {len(n.inputs)}")
    # cycles: DFS over data edges skipping NextIteration outputs
    adj: Dict[int, List[int]] = {n.id: [] for n in g.nodes}
    for n in g.nodes:
        for t in n.inputs:
            if g.nodes[t.node].op != "NextIteration":
                adj[t.node].append(n.id)
    color = {}
    for s in adj:
        if s in color:
            continue
        stack = [(s, iter(adj[s]))]
        color[s] = 1
        while stack:
            v, it = stack[-1]
            for w in it:
                if color.get(w) == 1:
                    errs.append(f"cycle lacks NextIteration (through node {w})")
                    break
                if w not in color:
                    color[w] = 1
                    stack.append((w, iter(adj[w])))
                    break
            else:
                color[v] = 2
                stack.pop()
    # context crossing
    for n in g.nodes:
        for t in n.inputs:
            src = g.nodes[t.node]
            if src.ctx is n.ctx:
                continue
            ok = False
            if n.op == "Enter" and src.ctx is n.ctx.parent:
                ok = True
            elif src.op == "Exit" and src.ctx is n.ctx:
                ok = True
            elif n.op == "Exit" and src.ctx.parent is n.ctx:
                ok = True
            elif n.op == "Switch" and n.ctx.kind == "cond" and src.ctx is n.ctx.parent:
                ok = True
            elif n.op == "Merge" and src.ctx.kind == "cond" and src.ctx.parent is n.ctx:
                ok = True
            elif n.op == "Merge" and n.attrs.get("loop") and src.op in ("Enter", "NextIteration"):
                ok = True
            if not ok:
                errs.append(f"node {n.id} ({n.op}) crosses context from node {src.id} ({src.op})")
    return errs
