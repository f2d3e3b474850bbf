"""Tagged-token dataflow interpreter -- the oracle's "local executor" (test infrastructure only).

Follows PAPER.md §4.3 "Local Execution" (lines 676-764):

* "It starts from the source nodes and repeatedly executes the nodes that become ready. A
  node, with the exception of Merge, becomes ready when all its inputs are available"
  (PAPER.md:683-687).
* Each tensor is a tuple (value, is_dead, tag); tags are tuples of
  (frame name, iteration) pairs, i.e. ``root/frame/i[/frame2/j...]`` (reading R6).
* The evaluation rules of Fig. "Evaluation rules for control-flow operators"
  (PAPER.md:712-735), with the readings R1-R3 of DESIGN.md for the points the figure leaves
  open: a dead token at NextIteration is dropped (R1); dead Exit tokens are held and an Exit
  fires once per frame instance, live at the final iteration or dead once for a dead frame
  (R2); a cond Merge fires on its first live input and outputs dead only when all inputs
  arrived dead (R3).
* Non-control ops: "the actual computation is performed only when none of the inputs are
  dead. If there is a dead input, we skip the computation and propagate a dead signal"
  (PAPER.md:749-755). Control inputs count as inputs for deadness.
* Loop constants are re-delivered to every iteration.
* parallel_iterations with the admission rule of SPEC.md:358 (reading R5):
  iteration i starts only if i - (oldest incomplete iteration) < K.
* Stacks: push/pop of the same stack node run in iteration order (the
  "explicit control dependencies to enforce ordering"), and a pop waits
  until the frame instance that pushed is complete.

A control trace is recorded for parity checks.
"""
from __future__ import annotations

import collections
import random
from typing import Any, Dict, List, Optional, Tuple

import numpy as np

from . import kernels
from .graph import BOOL, FLOAT, FLOW, INT, Graph, T


class InterpError(Exception):
    def __init__(self, code: str, msg: str):
        super().__init__(f"{code}: {msg}")
        self.code = code


class _Dead:
    def __repr__(self):
        return "DeadMarker"


DEAD = _Dead()   # fetch result for a dead tensor


class Token:
    __slots__ = ("value", "dead", "tag")

    def __init__(self, value, dead, tag):
        self.value, self.dead, self.tag = value, dead, tag


class TensorArrayObj:
    """Write-once TensorArray resource; grad TAs accumulate
    ("the gradient TensorArray holds the sum of the partial gradients")."""

    def __init__(self, size, dtype, elem_shape, is_grad=False):
        self.size, self.dtype, self.elem_shape = size, dtype, tuple(elem_shape)
        self.elems: List[Optional[np.ndarray]] = [None] * size
        self.is_grad = is_grad
        self.grad: Optional["TensorArrayObj"] = None

    def _ix(self, i):
        i = int(i)
        if not 0 <= i < self.size:
            raise InterpError("CF_E_SHAPE", f"TensorArray index {i} out of range {self.size}")
        return i

    def write(self, i, v):
        i = self._ix(i)
        if self.elems[i] is not None:
            if not self.is_grad:
                raise InterpError("CF_E_DOUBLE_WRITE", f"TensorArray slot {i} written twice")
            self.elems[i] = self.elems[i] + v
        else:
            self.elems[i] = np.array(v, dtype=np.float64 if self.dtype in (FLOAT, FLOW) else None)

    def read(self, i):
        i = self._ix(i)
        if self.elems[i] is None:
            if self.is_grad:
                return np.zeros(self.elem_shape)
            raise InterpError("CF_E_INVALID_GRAPH", f"TensorArray slot {i} read before write")
        return self.elems[i].copy()

    def stack(self):
        return np.stack([self.read(i) for i in range(self.size)]) if self.size else \
            np.zeros((0,) + self.elem_shape)

    def get_grad(self):
        if self.grad is None:
            self.grad = TensorArrayObj(self.size, self.dtype, self.elem_shape, is_grad=True)
        return self.grad


class StackObj:
    def __init__(self, stack_id, owner_key):
        self.id, self.owner_key = stack_id, owner_key
        self.entries: List[Any] = []
        self.pushes = self.pops = self.max_depth = 0


class Frame:
    def __init__(self, key, name, K, n_enters):
        self.key, self.name, self.K = key, name, K
        self.started = 0            # iterations 0..started-1 have started
        self.complete_upto = 0      # iterations < complete_upto are complete
        self.pending: Dict[int, int] = collections.defaultdict(int)
        self.parked: Dict[int, List[Tuple[int, int, Token]]] = collections.defaultdict(list)
        self.consts: List[Tuple[int, Token]] = []
        self.enters_left = n_enters
        self.dead = False
        self.exit_iter: Optional[int] = None
        self.done = False
        self.max_inflight = 0


class Trace:
    def __init__(self):
        self.trip_counts: Dict[Tuple, int] = {}       # (parent_tag, frame) -> n
        self.branch: Dict[Tuple[int, Tuple], bool] = {}   # (cond_id, tag) -> pred
        self.pushes: Dict[int, int] = collections.defaultdict(int)
        self.pops: Dict[int, int] = collections.defaultdict(int)
        self.max_depth: Dict[int, int] = collections.defaultdict(int)
        self.exit_fires: Dict[Tuple[int, Tuple], int] = collections.defaultdict(int)
        self.max_inflight: Dict[str, int] = collections.defaultdict(int)
        self.fires = 0
        self.dead_fires = 0
        self.live_merge_dead_inputs = 0   # a loop Merge that received a dead token
        self.sends = 0
        self.recvs = 0
        self.push_log: List[Tuple[int, Tuple]] = []
        self.pop_log: List[Tuple[int, Tuple]] = []


class Interpreter:
    def __init__(self, g: Graph, K_override: Optional[int] = None, sched_seed: Optional[int] = None,
                 transport=None):
        self.g = g
        self.transport = transport   # oracle.transport.*: Send/Recv between partitions
        self.K_override = K_override
        self.rng = random.Random(sched_seed) if sched_seed is not None else None
        self.cons = g.consumers()
        self.ctrl_cons: Dict[int, List[int]] = collections.defaultdict(list)
        for n in g.nodes:
            for c in n.ctrl:
                self.ctrl_cons[c].append(n.id)
        self.enters_per_frame: Dict[str, int] = collections.defaultdict(int)
        for n in g.nodes:
            if n.op == "Enter":
                self.enters_per_frame[n.attrs["frame"]] += 1

    # ------------------------------------------------------------------------------
    def run(self, feeds: Dict[str, np.ndarray], fetches: List[T]):
        g = self.g
        self.inbox: Dict[Tuple[int, Tuple], Dict[Any, Token]] = {}
        self.fired: set = set()
        self.queued: set = set()
        self.ready: collections.deque = collections.deque()
        self.frames: Dict[Tuple, Frame] = {}
        self.trace = Trace()
        self.root_vals: Dict[Tuple[int, int], Token] = {}
        self.seq: Dict[Tuple[int, Tuple], int] = collections.defaultdict(int)
        self.parked_ordered: Dict[Tuple[int, Tuple], Dict[int, Tuple]] = collections.defaultdict(dict)
        self.waiting_pops: List[Tuple[int, Tuple]] = []
        self.fetch_set = {(t.node, t.port) for t in fetches}

        for name, nid in g.placeholders.items():
            if name not in feeds:
                raise InterpError("CF_E_MISSING_FEED", f"no feed for placeholder {name}")
        for n in g.nodes:
            if not n.inputs and not n.ctrl:
                if n.ctx.kind != "root":
                    raise InterpError("CF_E_INVALID_GRAPH", f"source node {n.id} inside a construct")
                self.ready.append((n.id, ()))
                self.inbox[(n.id, ())] = {}
        while True:
            while self.ready:
                if self.rng is not None and len(self.ready) > 1:
                    k = self.rng.randrange(len(self.ready))
                    self.ready.rotate(-k)
                    item = self.ready.popleft()
                    self.ready.rotate(k)
                else:
                    item = self.ready.popleft()
                self._fire(*item, feeds)
            if not self._wake_pops():
                break
        if self.inbox:
            left = sorted({(g.nodes[k[0]].op, k[0]) for k in self.inbox})[:8]
            raise InterpError("CF_E_DEADLOCK", f"no ready nodes but pending instances: {left}")
        out = []
        for t in fetches:
            tok = self.root_vals.get((t.node, t.port))
            if tok is None:
                raise InterpError("CF_E_INVALID_GRAPH", f"fetch {t} never produced at root")
            out.append(DEAD if tok.dead else tok.value)
        return out

    # ------------------------------------------------------------------------------
    def _frame_iters(self, tag):
        for k in range(len(tag)):
            yield (tag[:k], tag[k][0]), tag[k][1]

    def _count(self, tag, d):
        for fk, it in self._frame_iters(tag):
            self.frames[fk].pending[it] += d

    def _deliver(self, cnid: int, port, tok: Token):
        key = (cnid, tok.tag)
        if key in self.fired:
            node = self.g.nodes[cnid]
            if node.op == "Merge":
                return      # second input of an already-fired cond Merge
            raise InterpError("CF_E_INVALID_GRAPH", f"node {cnid} fed twice at tag {tok.tag}")
        box = self.inbox.get(key)
        if box is None:
            box = self.inbox[key] = {}
            self._count(tok.tag, +1)
        if port in box:
            raise InterpError("CF_E_INVALID_GRAPH", f"input {port} of node {cnid} delivered twice")
        box[port] = tok
        if key not in self.queued and self._is_ready(cnid, box):
            self.queued.add(key)
            self.ready.append(key)

    def _is_ready(self, nid, box):
        n = self.g.nodes[nid]
        if n.op == "Merge":
            if n.attrs.get("loop"):
                return len(box) >= 1
            if any(not t.dead for p, t in box.items() if isinstance(p, int)):
                return True
            return len(box) == 2
        return len(box) == len(n.inputs) + len(n.ctrl)

    def _emit(self, nid, port, tok: Token):
        if tok.tag == () and (nid, port) in self.fetch_set:
            self.root_vals[(nid, port)] = tok
        for cnid, cport in self.cons.get((nid, port), ()):
            self._deliver(cnid, cport, tok)

    def _emit_ctrl(self, nid, dead, tag):
        for cnid in self.ctrl_cons.get(nid, ()):
            self._deliver(cnid, ("c", nid), Token(None, dead, tag))

    # ------------------------------------------------------------------------------
    def _frame_for_enter(self, n, parent_tag):
        name = n.attrs["frame"]
        key = (parent_tag, name)
        fr = self.frames.get(key)
        if fr is None:
            ctx = self.g.whiles[name]
            K = self.K_override or ctx.K
            fr = self.frames[key] = Frame(key, name, K, self.enters_per_frame[name])
            fr.started = 1      # "The child frame is created when the first Enter is executed"
        return fr

    def _admit(self, fr: Frame, it: int) -> bool:
        return it - fr.complete_upto < fr.K

    def _start_iter(self, fr: Frame, it: int):
        assert it == fr.started
        fr.started += 1
        fr.max_inflight = max(fr.max_inflight, fr.started - fr.complete_upto)
        self.trace.max_inflight[fr.name] = max(self.trace.max_inflight[fr.name], fr.max_inflight)
        tag = fr.key[0] + ((fr.name, it),)
        for enid, tok in fr.consts:
            self._emit(enid, 0, Token(tok.value, tok.dead, tag))
        for cnid, cport, tok in fr.parked.pop(it, []):
            self._deliver(cnid, cport, tok)

    def _advance(self, fr: Frame):
        changed = False
        while fr.complete_upto < fr.started:
            it = fr.complete_upto
            if fr.pending.get(it, 0) != 0 or (it == 0 and fr.enters_left > 0):
                break
            fr.complete_upto += 1
            changed = True
        while fr.started in fr.parked and self._admit(fr, fr.started):
            self._start_iter(fr, fr.started)
            changed = True
        if (fr.exit_iter is not None or fr.dead) and fr.complete_upto == fr.started \
                and not fr.parked and not fr.done:
            fr.done = True
            self.trace.trip_counts[fr.key] = 0 if fr.dead else fr.exit_iter
        return changed

    def _wake_pops(self) -> bool:
        woke = False
        still = []
        for key in self.waiting_pops:
            nid, tag = key
            box = self.inbox[key]
            st = box[0].value
            fr = self.frames.get(st.owner_key) if st is not None else None
            if st is None or fr is None or fr.done:
                self.ready.append(key)
                woke = True
            else:
                still.append(key)
        self.waiting_pops = still
        return woke

    # ------------------------------------------------------------------------------
    def _fire(self, nid, tag, feeds):
        g = self.g
        n = g.nodes[nid]
        key = (nid, tag)
        box = self.inbox[key]
        # ordered stack ops: one per iteration, in iteration order
        if n.op in ("StackPush", "StackPop") and tag:
            fk = (tag[:-1], tag[-1][0])
            okey = (nid, fk)
            it = tag[-1][1]
            if self.seq[okey] != it:
                self.parked_ordered[okey][it] = key
                return
            if n.op == "StackPop" and not any(t.dead for t in box.values()):
                st = box[0].value
                fr = self.frames.get(st.owner_key)
                if fr is not None and not fr.done:
                    self.waiting_pops.append(key)
                    return
        del self.inbox[key]
        self.queued.discard(key)
        if key in self.fired:
            raise InterpError("CF_E_INVALID_GRAPH", f"node {nid} fired twice at {tag}")
        self.fired.add(key)
        self.trace.fires += 1
        self._eval(n, tag, box, feeds)
        self._count(tag, -1)
        if n.op in ("StackPush", "StackPop") and tag:
            fk = (tag[:-1], tag[-1][0])
            okey = (nid, fk)
            self.seq[okey] += 1
            nxt = self.parked_ordered[okey].pop(self.seq[okey], None)
            if nxt is not None:
                self.ready.append(nxt)
        for fk, _ in self._frame_iters(tag):
            self._advance(self.frames[fk])

    def _eval(self, n, tag, box, feeds):
        op = n.op
        ins = [box[i] for i in range(len(n.inputs))] if op != "Merge" else None
        ctrl_dead = any(box[("c", c)].dead for c in n.ctrl)
        tr = self.trace
        if op == "Switch":
            d, p = ins
            dead = d.dead or p.dead or ctrl_dead
            if dead:
                o0 = o1 = True
            else:
                pv = bool(p.value)
                o0, o1 = pv, not pv        # r1 = p || dead(d); r2 = !p || dead(d)
                if "cond_id" in n.attrs:
                    tr.branch[(n.attrs["cond_id"], tag)] = pv
            self._emit(n.id, 0, Token(d.value, o0, tag))
            self._emit(n.id, 1, Token(d.value, o1, tag))
            self._emit_ctrl(n.id, dead, tag)
            return
        if op == "Merge":
            live = [(p, t) for p, t in sorted(box.items(), key=lambda kv: str(kv[0]))
                    if isinstance(p, int) and not t.dead]
            if n.attrs.get("loop"):
                t0 = next(iter(box.values()))
                if t0.dead and tag[-1][1] > 0:
                    tr.live_merge_dead_inputs += 1
                out = t0
            else:
                out = live[0][1] if live else next(t for p, t in box.items() if isinstance(p, int))
            self._emit(n.id, 0, Token(out.value, out.dead, tag))
            self._emit_ctrl(n.id, out.dead, tag)
            return
        if op == "Enter":
            d = ins[0]
            dead = d.dead or ctrl_dead
            fr = self._frame_for_enter(n, tag)
            fr.enters_left -= 1
            ctx = self.g.whiles[n.attrs["frame"]]
            if ctx.loop_vars and n.id == ctx.loop_vars[0]["enter"] and dead:
                fr.dead = True
            tok = Token(d.value, dead, tag + ((fr.name, 0),))
            if n.attrs.get("is_constant"):
                fr.consts.append((n.id, tok))
                for it in range(fr.started):
                    self._emit(n.id, 0, Token(d.value, dead, tag + ((fr.name, it),)))
            else:
                self._count(tok.tag, +1)     # keep iteration 0 pending while delivering
                self._emit(n.id, 0, tok)
                self._count(tok.tag, -1)
            self._advance(fr)
            return
        if op == "Exit":
            d = ins[0]
            fk = (tag[:-1], tag[-1][0])
            fr = self.frames[fk]
            ptag = tag[:-1]
            if d.dead or ctrl_dead:
                if fr.dead:
                    tr.exit_fires[(n.id, ptag)] += 1
                    self._emit(n.id, 0, Token(None, True, ptag))
                return      # reading R2: dead Exit tokens of a live frame are held
            tr.exit_fires[(n.id, ptag)] += 1
            if tr.exit_fires[(n.id, ptag)] > 1:
                raise InterpError("CF_E_INVALID_GRAPH", "Exit fired twice for one frame")
            fr.exit_iter = tag[-1][1]
            self._emit(n.id, 0, Token(d.value, False, ptag))
            return
        if op == "NextIteration":
            d = ins[0]
            if d.dead or ctrl_dead:
                return      # reading R1: dead NextIteration tokens are dropped
            fk = (tag[:-1], tag[-1][0])
            fr = self.frames[fk]
            it = tag[-1][1] + 1
            ntag = tag[:-1] + ((fr.name, it),)
            tok = Token(d.value, False, ntag)
            targets = [(c, p, tok) for c, p in self.cons.get((n.id, 0), ())]
            if it < fr.started:
                for c, p, t in targets:
                    self._deliver(c, p, t)
            elif it == fr.started and self._admit(fr, it) and it not in fr.parked:
                self._start_iter(fr, it)
                for c, p, t in targets:
                    self._deliver(c, p, t)
            else:
                # park; count the targets as pending for the source iteration so the
                # "first NextIteration starts N+1" transition is not lost
                fr.parked[it].extend(targets)
            return
        # ---------------- Send / Recv: the is_dead signal crosses devices;
        # a Recv "is always ready" and takes whatever its Send delivered for this tag
        if op in ("Send", "Recv"):
            if self.transport is None:
                raise InterpError("CF_E_UNSUPPORTED", f"{op} without a transport")
            key = tuple(it for _, it in tag)
            peer, ch = n.attrs["peer"], n.attrs["channel"]
            if op == "Send":
                v, ix = ins
                dead = ctrl_dead or v.dead or ix.dead
                self.transport.send(peer, ch, key, None if dead else np.array(v.value, copy=True), dead,
                                    tuple(self.g.shape(n.inputs[0])))
                tr.sends += 1
                self._emit_ctrl(n.id, dead, tag)
                return
            val, mdead = self.transport.recv(peer, ch, key, tuple(n.attrs["shape"]))
            dead = ctrl_dead or ins[0].dead or mdead
            tr.recvs += 1
            self._emit(n.id, 0, Token(None if dead else val, dead, tag))
            self._emit_ctrl(n.id, dead, tag)
            return
        # ---------------- non-control ops: dead propagation
        dead = ctrl_dead or any(t.dead for t in ins)
        nout = len(n.out_dtypes)
        if dead:
            tr.dead_fires += 1
            for p in range(nout):
                self._emit(n.id, p, Token(None, True, tag))
            self._emit_ctrl(n.id, True, tag)
            return
        vals = [t.value for t in ins]
        outs = self._compute(n, vals, tag, feeds)
        for p in range(nout):
            self._emit(n.id, p, Token(outs[p], False, tag))
        self._emit_ctrl(n.id, False, tag)

    def _compute(self, n, vals, tag, feeds):
        op = n.op
        a = n.attrs
        if op == "Placeholder":
            v = np.asarray(feeds[a["name"]])
            v = v.astype({FLOAT: np.float64, INT: np.int64, BOOL: bool}[a["dtype"]])
            if tuple(v.shape) != tuple(a["shape"]):
                raise InterpError("CF_E_SHAPE", f"feed {a['name']} shape {v.shape} != {a['shape']}")
            return [v]
        if op == "TACreate":
            return [TensorArrayObj(a["size"], a["dtype"], a["elem_shape"]), np.float64(0.0)]
        if op == "TARead":
            return [vals[0].read(vals[1])]
        if op == "TAWrite":
            vals[0].write(vals[1], vals[2])
            return [np.float64(0.0)]
        if op == "TAStack":
            return [vals[0].stack()]
        if op == "TAUnstack":
            v = vals[1]
            if v.shape[0] != vals[0].size:
                raise InterpError("CF_E_SHAPE", "unstack size mismatch")
            for i in range(v.shape[0]):
                vals[0].write(i, v[i])
            return [np.float64(0.0)]
        if op == "TAGrad":
            return [vals[0].get_grad(), np.float64(0.0)]
        if op == "StackCreate":
            return [StackObj(n.id, (tag, a["frame"]))]
        if op == "StackPush":
            st: StackObj = vals[0]
            # a handle (a nested loop's stack, saved for the outer gradient loop) by reference
            v = vals[1]
            st.entries.append(v if isinstance(v, StackObj) else np.array(v, copy=True))
            st.pushes += 1
            st.max_depth = max(st.max_depth, len(st.entries))
            self.trace.pushes[st.id] += 1
            self.trace.max_depth[st.id] = max(self.trace.max_depth[st.id], len(st.entries))
            self.trace.push_log.append((st.id, tag))
            return []
        if op == "StackPop":
            st = vals[0]
            if not st.entries:
                raise InterpError("CF_E_POP_EMPTY", f"pop of empty stack {st.id}")
            st.pops += 1
            self.trace.pops[st.id] += 1
            self.trace.pop_log.append((st.id, tag))
            return [st.entries.pop()]
        if op in ("Add", "Sub", "AddN") and n.out_dtypes[0] == FLOW:
            return [np.float64(0.0)]
        return kernels.eval_op(op, vals, a)


def run(g: Graph, feeds, fetches, K_override=None, sched_seed=None, return_trace=False,
        transport=None):
    it = Interpreter(g, K_override, sched_seed, transport)
    vals = it.run(feeds, fetches)
    return (vals, it.trace) if return_trace else vals
