"""Thin ctypes binding over libcf (include/cf.h): argument marshalling only.

Every step of graph construction, differentiation, compilation and execution happens inside
libcf.so (C++ host code + sm_100a kernels). PyTorch is used only for device memory and
streams. There is no CPU fallback: if libcf.so is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Callable, Dict, List, Optional, Sequence

HERE = os.path.dirname(os.path.abspath(__file__))
# CF_LIB=libcf_prof.so selects the profiling build (tools/profile_run.py); default libcf.so
LIB_PATH = os.path.join(HERE, os.environ.get("CF_LIB", "libcf.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libcf.so not built ({LIB_PATH}); run python -c 'import __graft_entry__ as "
                      f"g; g.build()' -- there is no CPU fallback")
_lib = C.CDLL(LIB_PATH)

# cf_dtype
BOOL, I32, I64, F32, F64, BF16, FLOW, RES = range(8)
STATUS = {0: "CF_OK", 1: "CF_E_ARITY", 2: "CF_E_DTYPE", 3: "CF_E_SHAPE", 4: "CF_E_NONBOOL_PRED",
          5: "CF_E_BRANCH_MISMATCH", 6: "CF_E_INVALID_GRAPH", 7: "CF_E_NONSCALAR_OBJECTIVE",
          8: "CF_E_NO_GRADIENT", 9: "CF_E_MISSING_FEED", 10: "CF_E_UNSUPPORTED",
          11: "CF_E_DEADLOCK", 12: "CF_E_POP_EMPTY", 13: "CF_E_DOUBLE_WRITE",
          14: "CF_E_STACK_BUDGET", 15: "CF_E_CUDA", 16: "CF_E_NCCL"}


class CfError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.code = STATUS.get(status, str(status))


class cf_tensor(C.Structure):
    _fields_ = [("node", C.c_int32), ("port", C.c_int32)]


class cf_buffer(C.Structure):
    _fields_ = [("data", C.c_void_p), ("dtype", C.c_int32), ("rank", C.c_int32),
                ("shape", C.c_int64 * 8)]


class cf_run_opts(C.Structure):
    _fields_ = [("precision", C.c_int32), ("parallel_iterations", C.c_int32),
                ("device", C.c_int32), ("num_workers", C.c_int32), ("stream", C.c_void_p),
                ("max_iterations", C.c_int64), ("watchdog_ms", C.c_int64),
                ("sched_seed", C.c_int32), ("reserved", C.c_int32 * 7),
                ("stack_budget_bytes", C.c_int64), ("swap_min_bytes", C.c_int64),
                ("swap_smallest_first", C.c_int32), ("pad_", C.c_int32),
                ("dev_alloc", C.c_void_p), ("dev_free", C.c_void_p), ("alloc_user", C.c_void_p),
                ("d2h_stream", C.c_void_p), ("h2d_stream", C.c_void_p)]

# caller allocator callbacks (cf_run_opts.dev_alloc / dev_free)
DEV_ALLOC = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
DEV_FREE = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class cf_trace(C.Structure):
    _fields_ = [("n_frames", C.c_int32), ("trip_count", C.c_int32 * 16),
                ("max_inflight", C.c_int32 * 16), ("pushes", C.c_int64), ("pops", C.c_int64),
                ("max_depth", C.c_int32), ("exit_fires", C.c_int32), ("instances", C.c_int64),
                ("tiles", C.c_int64), ("dead_skipped", C.c_int64), ("n_branch_bits", C.c_int32),
                ("branch_bits", C.POINTER(C.c_uint8)), ("branch_bits_cap", C.c_int32),
                ("wall_ms", C.c_double), ("sends", C.c_int64), ("recvs", C.c_int64),
                ("swap_out", C.c_int64), ("swap_in", C.c_int64), ("bytes_d2h", C.c_int64),
                ("bytes_h2d", C.c_int64)]


PRED_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int32, C.POINTER(cf_tensor),
                      C.POINTER(cf_tensor), C.c_void_p)
BODY_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int32, C.POINTER(cf_tensor),
                      C.POINTER(cf_tensor), C.c_void_p)
BRANCH_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int32, C.POINTER(cf_tensor), C.c_void_p)

_P = C.c_void_p
IPC_HANDLE_BYTES = 64
GRAD_CHANNEL = 1 << 20
_sig = {
    "cf_last_error": (C.c_char_p, []),
    "cf_version": (C.c_char_p, []),
    "cf_graph_create": (C.c_int32, [C.POINTER(_P)]),
    "cf_graph_destroy": (None, [_P]),
    "cf_placeholder": (C.c_int32, [_P, C.c_char_p, C.c_int32, C.c_int32, C.POINTER(C.c_int64),
                                   C.POINTER(cf_tensor)]),
    "cf_const": (C.c_int32, [_P, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.c_void_p,
                             C.POINTER(cf_tensor)]),
    "cf_op": (C.c_int32, [_P, C.c_char_p, C.c_int32, C.POINTER(cf_tensor), C.c_char_p,
                          C.POINTER(C.c_int32), C.POINTER(cf_tensor)]),
    "cf_while_loop": (C.c_int32, [_P, PRED_FN, BODY_FN, C.c_void_p, C.c_int32,
                                  C.POINTER(cf_tensor), C.c_int32, C.c_char_p,
                                  C.POINTER(cf_tensor)]),
    "cf_while_loop_counted": (C.c_int32, [_P, PRED_FN, BODY_FN, C.c_void_p, C.c_int32,
                                          C.POINTER(cf_tensor), C.c_int32, C.c_char_p,
                                          C.POINTER(cf_tensor), C.POINTER(cf_tensor)]),
    "cf_cond": (C.c_int32, [_P, cf_tensor, BRANCH_FN, BRANCH_FN, C.c_void_p, C.c_int32,
                            C.POINTER(cf_tensor)]),
    "cf_ta_create": (C.c_int32, [_P, C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64),
                                 C.POINTER(cf_tensor), C.POINTER(cf_tensor)]),
    "cf_ta_read": (C.c_int32, [_P, cf_tensor, cf_tensor, cf_tensor, C.POINTER(cf_tensor)]),
    "cf_ta_write": (C.c_int32, [_P, cf_tensor, cf_tensor, cf_tensor, cf_tensor,
                                C.POINTER(cf_tensor)]),
    "cf_ta_unstack": (C.c_int32, [_P, cf_tensor, cf_tensor, cf_tensor, C.POINTER(cf_tensor)]),
    "cf_ta_stack": (C.c_int32, [_P, cf_tensor, cf_tensor, C.POINTER(cf_tensor)]),
    "cf_gradients": (C.c_int32, [_P, cf_tensor, C.c_int32, C.POINTER(cf_tensor),
                                 C.POINTER(cf_tensor)]),
    "cf_validate": (C.c_int32, [_P, C.c_char_p, C.c_size_t]),
    "cf_graph_json": (C.c_int32, [_P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "cf_graph_num_nodes": (C.c_int32, [_P, C.POINTER(C.c_int32)]),
    "cf_tensor_info": (C.c_int32, [_P, cf_tensor, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                   C.POINTER(C.c_int64)]),
    "cf_session_create": (C.c_int32, [_P, C.POINTER(cf_run_opts), C.c_int32,
                                      C.POINTER(cf_tensor), C.POINTER(_P)]),
    "cf_run": (C.c_int32, [_P, C.c_int32, C.POINTER(C.c_char_p), C.POINTER(cf_buffer),
                           C.POINTER(cf_buffer), C.POINTER(C.c_uint8), C.POINTER(cf_trace)]),
    "cf_session_feed_dtype": (C.c_int32, [_P, C.c_char_p, C.POINTER(C.c_int32)]),
    "cf_session_fetch_dtype": (C.c_int32, [_P, C.c_int32, C.POINTER(C.c_int32)]),
    "cf_session_describe": (C.c_int32, [_P, C.c_char_p, C.c_size_t]),
    "cf_session_destroy": (None, [_P]),
    "cf_session_channels": (C.c_int32, [_P, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    "cf_session_ipc_handle": (C.c_int32, [_P, C.c_void_p]),
    "cf_session_connect": (C.c_int32, [_P, C.c_int32, C.c_void_p, C.c_int32, C.POINTER(C.c_int64)]),
    # include/cf_debug.h (test hooks)
    "cf_debug_set_m2_rows": (C.c_int32, [C.c_int32]),
    "cf_debug_set_worker_roles": (C.c_int32, [C.c_int32, C.c_int32]),
    "cf_debug_tile_phases": (C.c_int32, [C.c_void_p, C.c_int32]),
    "cf_debug_set_knob": (C.c_int32, [C.c_int32, C.c_int32]),
    "cf_debug_tc_pipe": (C.c_int32, [C.c_int32] * 6 + [C.c_void_p, C.c_void_p, C.POINTER(C.c_float)]),
    "cf_debug_set_flags": (C.c_int32, [C.c_int32]),
    "cf_debug_program_listing": (C.c_int32, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                             C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "cf_debug_session_profile": (C.c_int32, [_P, C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                                             C.c_void_p]),
    "cf_debug_tc_gemm": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                     C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = list(_sig)


def _dtype_size(d: int) -> int:
    return {BOOL: 1, I32: 4, I64: 8, F32: 4, F64: 8, BF16: 2}[d]


def _check(st: int):
    if st != 0:
        raise CfError(st, _lib.cf_last_error().decode())


def _attrs(d: Optional[Dict]) -> bytes:
    if not d:
        return b""
    parts = []
    for k, v in d.items():
        if isinstance(v, bool):
            v = int(v)
        if isinstance(v, (list, tuple)):
            v = ",".join(str(int(x)) for x in v)
        parts.append(f"{k}={v}")
    return ";".join(parts).encode()


class Tensor:
    __slots__ = ("g", "node", "port")

    def __init__(self, g: "Graph", node: int, port: int):
        self.g, self.node, self.port = g, node, port

    @property
    def c(self) -> cf_tensor:
        return cf_tensor(self.node, self.port)

    def info(self):
        dt, rk = C.c_int32(), C.c_int32()
        sh = (C.c_int64 * 8)()
        _check(_lib.cf_tensor_info(self.g.h, self.c, C.byref(dt), C.byref(rk), sh))
        return dt.value, tuple(sh[i] for i in range(rk.value))

    @property
    def dtype(self):
        return self.info()[0]

    @property
    def shape(self):
        return self.info()[1]

    def __repr__(self):
        return f"Tensor({self.node}:{self.port})"


class TensorArray:
    def __init__(self, g: "Graph", handle: Tensor, flow: Tensor):
        self.g, self.handle, self.flow = g, handle, flow

    def with_flow(self, flow: Tensor) -> "TensorArray":
        return TensorArray(self.g, self.handle, flow)

    def read(self, ix: Tensor) -> Tensor:
        out = cf_tensor()
        _check(_lib.cf_ta_read(self.g.h, self.handle.c, ix.c, self.flow.c, C.byref(out)))
        return Tensor(self.g, out.node, out.port)

    def write(self, ix: Tensor, v: Tensor) -> "TensorArray":
        out = cf_tensor()
        _check(_lib.cf_ta_write(self.g.h, self.handle.c, ix.c, v.c, self.flow.c, C.byref(out)))
        return self.with_flow(Tensor(self.g, out.node, out.port))

    def unstack(self, v: Tensor) -> "TensorArray":
        out = cf_tensor()
        _check(_lib.cf_ta_unstack(self.g.h, self.handle.c, v.c, self.flow.c, C.byref(out)))
        return self.with_flow(Tensor(self.g, out.node, out.port))

    def stack(self) -> Tensor:
        out = cf_tensor()
        _check(_lib.cf_ta_stack(self.g.h, self.handle.c, self.flow.c, C.byref(out)))
        return Tensor(self.g, out.node, out.port)


class Graph:
    """cf_graph handle with builder methods."""

    def __init__(self):
        h = _P()
        _check(_lib.cf_graph_create(C.byref(h)))
        self.h = h
        self._keep = []      # callback objects alive during construction
        self._exc = None

    def __del__(self):
        try:
            if self.h:
                _lib.cf_graph_destroy(self.h)
        except Exception:
            pass

    def _t(self, ct: cf_tensor) -> Tensor:
        return Tensor(self, ct.node, ct.port)

    def num_nodes(self) -> int:
        n = C.c_int32()
        _check(_lib.cf_graph_num_nodes(self.h, C.byref(n)))
        return n.value

    def placeholder(self, name: str, dtype: int, shape: Sequence[int]) -> Tensor:
        sh = (C.c_int64 * max(len(shape), 1))(*shape)
        out = cf_tensor()
        _check(_lib.cf_placeholder(self.h, name.encode(), dtype, len(shape), sh, C.byref(out)))
        return self._t(out)

    def const(self, value, dtype: int) -> Tensor:
        import numpy as np
        npdt = {F32: np.float32, I64: np.int64, BOOL: np.bool_, I32: np.int32, F64: np.float64}
        if dtype == FLOW:
            arr = np.zeros((), np.float32)
            data, shape = None, ()
        else:
            arr = np.array(value, dtype=npdt[dtype], order="C", copy=True)
            data, shape = arr.ctypes.data_as(C.c_void_p), arr.shape
        sh = (C.c_int64 * max(len(shape), 1))(*shape)
        out = cf_tensor()
        _check(_lib.cf_const(self.h, dtype, len(shape), sh, data, C.byref(out)))
        return self._t(out)

    def op(self, name: str, inputs: Sequence[Tensor], attrs: Optional[Dict] = None) -> List[Tensor]:
        arr = (cf_tensor * max(len(inputs), 1))(*[t.c for t in inputs])
        outs = (cf_tensor * 8)()
        n = C.c_int32()
        _check(_lib.cf_op(self.h, name.encode(), len(inputs), arr, _attrs(attrs), C.byref(n), outs))
        return [self._t(outs[i]) for i in range(n.value)]

    def op1(self, name, inputs, attrs=None) -> Tensor:
        return self.op(name, inputs, attrs)[0]

    def _call(self, fn, args):
        try:
            return fn(*args)
        except Exception as e:   # surface Python errors after the C call returns
            self._exc = e
            raise

    def while_loop(self, pred: Callable, body: Callable, inits: Sequence[Tensor],
                   parallel_iterations: int = 32, name: Optional[str] = None,
                   return_counter: bool = False):
        n = len(inits)

        def _pred(gh, nv, vars_, out, user):
            try:
                r = pred(*[self._t(vars_[i]) for i in range(nv)])
                out[0] = r.c
                return 0
            except CfError as e:
                self._exc = e
                return e.status
            except Exception as e:
                self._exc = e
                return 6

        def _body(gh, nv, vars_, out, user):
            try:
                r = list(body(*[self._t(vars_[i]) for i in range(nv)]))
                if len(r) != nv:
                    raise CfError(1, "body returned wrong number of loop variables")
                for i, t in enumerate(r):
                    out[i] = t.c
                return 0
            except CfError as e:
                self._exc = e
                return e.status
            except Exception as e:
                self._exc = e
                return 6
        pf, bf = PRED_FN(_pred), BODY_FN(_body)
        self._keep += [pf, bf]
        arr = (cf_tensor * max(n, 1))(*[t.c for t in inits])
        outs = (cf_tensor * max(n, 1))()
        trip = cf_tensor()
        self._exc = None
        st = _lib.cf_while_loop_counted(self.h, pf, bf, None, n, arr, parallel_iterations,
                                        name.encode() if name else None, outs, C.byref(trip))
        if st != 0 and self._exc is not None:
            e, self._exc = self._exc, None
            raise e
        _check(st)
        res = [self._t(outs[i]) for i in range(n)]
        return (res, self._t(trip)) if return_counter else res

    def cond(self, pred: Tensor, true_fn: Callable, false_fn: Callable, n_out: int) -> List[Tensor]:
        """cond(pred, true_fn, false_fn); n_out = outputs per branch."""
        return self.cond_n(pred, true_fn, false_fn, n_out)

    def cond_n(self, pred: Tensor, true_fn: Callable, false_fn: Callable, n_out: int) -> List[Tensor]:
        def mk(fn):
            def _b(gh, n, out, user):
                try:
                    r = list(fn())
                    if len(r) != n:
                        raise CfError(5, "cond branch returned %d outputs, expected %d" % (len(r), n))
                    for i, t in enumerate(r):
                        out[i] = t.c
                    return 0
                except CfError as e:
                    self._exc = e
                    return e.status
                except Exception as e:
                    self._exc = e
                    return 6
            return BRANCH_FN(_b)
        tf, ff = mk(true_fn), mk(false_fn)
        self._keep += [tf, ff]
        outs = (cf_tensor * max(n_out, 1))()
        self._exc = None
        st = _lib.cf_cond(self.h, pred.c, tf, ff, None, n_out, outs)
        if st != 0 and self._exc is not None:
            e, self._exc = self._exc, None
            raise e
        _check(st)
        return [self._t(outs[i]) for i in range(n_out)]

    # cross-GPU edges of a partitioned program; channel ^ GRAD_CHANNEL is
    # the mirrored gradient edge
    def send(self, v: Tensor, ix: Tensor, channel: int, peer: int) -> None:
        self.op("Send", [v, ix], {"channel": channel, "peer": peer})

    def recv(self, ix: Tensor, channel: int, peer: int, dtype: int, shape: Sequence[int]) -> Tensor:
        return self.op1("Recv", [ix], {"channel": channel, "peer": peer, "dtype": dtype,
                                       "shape": list(shape)})

    def tensor_array(self, size: int, dtype: int, elem_shape: Sequence[int]) -> TensorArray:
        sh = (C.c_int64 * max(len(elem_shape), 1))(*elem_shape)
        h, f = cf_tensor(), cf_tensor()
        _check(_lib.cf_ta_create(self.h, size, dtype, len(elem_shape), sh, C.byref(h), C.byref(f)))
        return TensorArray(self, self._t(h), self._t(f))

    def gradients(self, y: Tensor, xs: Sequence[Tensor]) -> List[Tensor]:
        arr = (cf_tensor * max(len(xs), 1))(*[x.c for x in xs])
        out = (cf_tensor * max(len(xs), 1))()
        _check(_lib.cf_gradients(self.h, y.c, len(xs), arr, out))
        return [self._t(out[i]) for i in range(len(xs))]

    def validate(self) -> List[str]:
        buf = C.create_string_buffer(1 << 16)
        st = _lib.cf_validate(self.h, buf, len(buf))
        txt = buf.value.decode()
        return [l for l in txt.splitlines() if l] if st != 0 else []

    def json(self) -> dict:
        import json
        need = C.c_size_t()
        _lib.cf_graph_json(self.h, None, 0, C.byref(need))
        buf = C.create_string_buffer(need.value)
        _check(_lib.cf_graph_json(self.h, buf, len(buf), None))
        return json.loads(buf.value.decode())

    def count_ops(self) -> Dict[str, int]:
        out: Dict[str, int] = {}
        for n in self.json()["nodes"]:
            out[n["op"]] = out.get(n["op"], 0) + 1
        return out


# ----------------------------------------------------------------------------- execution
_TORCH_DT = None


def _torch_dtypes():
    global _TORCH_DT
    if _TORCH_DT is None:
        import torch
        _TORCH_DT = {BOOL: torch.bool, I32: torch.int32, I64: torch.int64, F32: torch.float32,
                     BF16: torch.bfloat16}
    return _TORCH_DT


class Session:
    """Compiled graph on one GPU (cf_session_create) + cf_run."""

    def __init__(self, g: Graph, fetches: Sequence[Tensor], precision: int = F32,
                 parallel_iterations: int = 0, device: int = 0, stream=None,
                 max_iterations: int = 0, watchdog_ms: int = 0, num_workers: int = 0,
                 sched_seed: int = 0, profile: bool = False, stack_budget_bytes: int = 0,
                 swap_min_bytes: int = 0, swap_smallest_first: bool = False,
                 dev_alloc=None, dev_free=None, d2h_stream=None, h2d_stream=None):
        """dev_alloc(bytes) -> int device pointer and dev_free(ptr) (Python callables, both
        or neither): the session's device buffers come from the caller's allocator
        (cf_run_opts.dev_alloc / dev_free). d2h_stream / h2d_stream: cudaStream_t handles for
        the swap copies (cf_run_opts)."""
        self.g = g
        self.fetches = list(fetches)
        o = cf_run_opts()
        o.precision = precision
        o.parallel_iterations = parallel_iterations
        o.device = device
        o.num_workers = num_workers
        o.stream = stream
        o.max_iterations = max_iterations
        o.watchdog_ms = watchdog_ms
        o.sched_seed = sched_seed
        o.reserved[0] = 1 if profile else 0
        o.stack_budget_bytes = stack_budget_bytes
        o.swap_min_bytes = swap_min_bytes
        o.swap_smallest_first = 1 if swap_smallest_first else 0
        if (dev_alloc is None) != (dev_free is None):
            raise ValueError("dev_alloc and dev_free go together")
        if dev_alloc is not None:   # kept alive with the session: the library calls them
            self._alloc_cb = DEV_ALLOC(lambda n, _u: int(dev_alloc(int(n))) or None)
            self._free_cb = DEV_FREE(lambda ptr, _u: dev_free(int(ptr or 0)))
            o.dev_alloc = C.cast(self._alloc_cb, C.c_void_p)
            o.dev_free = C.cast(self._free_cb, C.c_void_p)
        o.d2h_stream = d2h_stream
        o.h2d_stream = h2d_stream
        arr = (cf_tensor * max(len(fetches), 1))(*[t.c for t in fetches])
        h = _P()
        _check(_lib.cf_session_create(g.h, C.byref(o), len(fetches), arr, C.byref(h)))
        self.h = h
        self.fetch_dtypes = []
        for i in range(len(fetches)):
            d = C.c_int32()
            _check(_lib.cf_session_fetch_dtype(self.h, i, C.byref(d)))
            self.fetch_dtypes.append(d.value)
        self.fetch_shapes = [t.shape for t in fetches]

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib.cf_session_destroy(self.h)
        except Exception:
            pass

    def profile(self):
        """Per-instance device timing of the last run (needs profile=True): numpy array of
        [create, publish, first_start, last_end, busy_ns, kind, ntiles] rows and (t0, t1)."""
        import numpy as np
        n = C.c_int64()
        t = (C.c_uint64 * 130)()
        _check(_lib.cf_debug_session_profile(self.h, None, 0, C.byref(n), t))
        buf = np.zeros(6 * n.value, dtype=np.uint64)
        _check(_lib.cf_debug_session_profile(self.h, buf.ctypes.data, buf.size, C.byref(n), t))
        r = buf.reshape(-1, 6)
        out = np.zeros((r.shape[0], 7), dtype=np.float64)
        out[:, :5] = r[:, :5].astype(np.float64)
        out[:, 5] = (r[:, 5] >> np.uint64(32)).astype(np.float64)
        out[:, 6] = (r[:, 5] & np.uint64(0xffffffff)).astype(np.float64)
        self.driver_ops = [(int(t[2 + k]), int(t[66 + k])) for k in range(64)]
        return out, (float(t[0]), float(t[1]))

    # ---- multi-GPU pipeline (include/cf.h "multi-GPU layer pipeline")
    def channels(self):
        """This session's channel halves: list of (channel, role, peer, slots, bytes, dtype,
        offset); role 0 = receives, 1 = sends."""
        n = C.c_int32()
        _check(_lib.cf_session_channels(self.h, 0, None, C.byref(n)))
        tab = (C.c_int64 * max(7 * n.value, 1))()
        _check(_lib.cf_session_channels(self.h, n.value, tab, C.byref(n)))
        return [tuple(tab[7 * i + k] for k in range(7)) for i in range(n.value)]

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(IPC_HANDLE_BYTES)
        _check(_lib.cf_session_ipc_handle(self.h, buf))
        return buf.raw

    def connect(self, peer: int, handle: bytes, table) -> None:
        flat = [int(v) for row in table for v in row]
        tab = (C.c_int64 * max(len(flat), 1))(*flat)
        _check(_lib.cf_session_connect(self.h, peer, C.c_char_p(handle), len(table), tab))

    def connect_pipeline(self, group=None) -> None:
        """Exchange channel memory with every other rank through torch.distributed (any
        backend) and connect the peers this partition talks to."""
        import torch.distributed as dist
        mine = (dist.get_rank(group), self.ipc_handle(), self.channels())
        allv = [None] * dist.get_world_size(group)
        dist.all_gather_object(allv, mine, group=group)
        peers = {c[2] for c in mine[2]}
        for rank, handle, table in allv:
            if rank in peers:
                self.connect(rank, handle, table)

    def has_feed(self, name: str) -> bool:
        d = C.c_int32()
        return _lib.cf_session_feed_dtype(self.h, name.encode(), C.byref(d)) == 0

    def feed_dtype(self, name: str) -> int:
        d = C.c_int32()
        _check(_lib.cf_session_feed_dtype(self.h, name.encode(), C.byref(d)))
        return d.value

    def describe(self) -> str:
        buf = C.create_string_buffer(1 << 14)
        _check(_lib.cf_session_describe(self.h, buf, len(buf)))
        return buf.value.decode()

    def alloc_outputs(self, device="cuda"):
        import torch
        tdt = _torch_dtypes()
        return [torch.empty(s, dtype=tdt[d], device=device)
                for s, d in zip(self.fetch_shapes, self.fetch_dtypes)]

    def run(self, feeds: Dict, outs=None, trace: bool = False, branch_cap: int = 0):
        """feeds: name -> CUDA torch tensor (contiguous, session dtype). Returns
        (outputs, dead flags, trace dict | None)."""
        import torch
        names = list(feeds)
        if outs is None:
            outs = self.alloc_outputs()
        # the marshalled argument arrays of the previous call are reused when the same tensors
        # come again (a training loop's resident inputs): one key comparison instead of a
        # per-feed rebuild
        key = (tuple((nm, feeds[nm].data_ptr(), feeds[nm].dtype, tuple(feeds[nm].shape),
                      tuple(feeds[nm].stride()), feeds[nm].is_cuda) for nm in names),
               tuple((t.data_ptr(), t.dtype, tuple(t.shape), tuple(t.stride())) for t in outs))
        cached = getattr(self, "_args_cache", None)
        if cached is not None and cached[0] == key:
            bufs, cnames, obufs = cached[1]
        else:
            bufs = (cf_buffer * max(len(names), 1))()
            for i, nm in enumerate(names):
                t = feeds[nm]
                if not t.is_cuda or not t.is_contiguous():
                    raise CfError(2, f"feed {nm} must be a contiguous CUDA tensor")
                bufs[i].data = t.data_ptr()
                bufs[i].dtype = {torch.bool: BOOL, torch.int32: I32, torch.int64: I64,
                                 torch.float32: F32, torch.bfloat16: BF16}[t.dtype]
                bufs[i].rank = t.dim()
                for k, s in enumerate(t.shape):
                    bufs[i].shape[k] = s
            cnames = (C.c_char_p * max(len(names), 1))(*[n.encode() for n in names])
            obufs = (cf_buffer * max(len(outs), 1))()
            for i, t in enumerate(outs):
                obufs[i].data = t.data_ptr()
                obufs[i].dtype = self.fetch_dtypes[i]
                obufs[i].rank = t.dim()
                for k, sz in enumerate(t.shape):
                    obufs[i].shape[k] = sz
                if not t.is_contiguous() or t.element_size() != _dtype_size(self.fetch_dtypes[i]):
                    raise CfError(2, f"fetch buffer {i} must be contiguous with the session dtype")
            self._args_cache = (key, (bufs, cnames, obufs))
        dead = (C.c_uint8 * max(len(outs), 1))()
        tr = cf_trace()
        bits = None
        if trace and branch_cap:
            bits = (C.c_uint8 * branch_cap)()
            tr.branch_bits = C.cast(bits, C.POINTER(C.c_uint8))
            tr.branch_bits_cap = branch_cap
        st = _lib.cf_run(self.h, len(names), cnames, bufs, obufs, dead,
                         C.byref(tr) if trace else None)
        _check(st)
        tdict = None
        if trace:
            tdict = {
                "n_frames": tr.n_frames,
                "trip_count": [tr.trip_count[i] for i in range(tr.n_frames)],
                "max_inflight": [tr.max_inflight[i] for i in range(tr.n_frames)],
                "pushes": tr.pushes, "pops": tr.pops, "max_depth": tr.max_depth,
                "exit_fires": tr.exit_fires, "instances": tr.instances, "tiles": tr.tiles,
                "dead_skipped": tr.dead_skipped, "wall_ms": tr.wall_ms,
                "sends": tr.sends, "recvs": tr.recvs, "swap_out": tr.swap_out,
                "swap_in": tr.swap_in, "bytes_d2h": tr.bytes_d2h, "bytes_h2d": tr.bytes_h2d,
                "n_branch_bits": tr.n_branch_bits,
                "branch_bits": bytes(bits)[:min(branch_cap, tr.n_branch_bits)] if bits else b"",
            }
        return outs, [bool(dead[i]) for i in range(len(outs))], tdict


def debug_tc_gemm(M, N, K, bn, a_mn, b_mn, A, B, Cout, stream=None):
    """Test hook (include/cf_debug.h): C = A(m,k) . B(n,k) on the tcgen05 tile engine."""
    _check(_lib.cf_debug_tc_gemm(M, N, K, bn, a_mn, b_mn, A.data_ptr(), B.data_ptr(),
                                 Cout.data_ptr(), stream))


def version() -> str:
    return _lib.cf_version().decode()


def debug_set_flags(flags: int) -> None:
    """Profiling knob (cf_debug.h): bit 0 = workers skip tile bodies (driver cost alone)."""
    _check(_lib.cf_debug_set_flags(flags))


def debug_set_knob(which: int, value: int) -> None:
    """A/B knob (cf_debug.h): 0 = claim-ahead lead in k-blocks (0 = default)."""
    _check(_lib.cf_debug_set_knob(which, value))


def debug_tile_phases(reset: bool = True) -> list:
    """Tile phase clocks (cf_debug.h; collected under debug flag bit 22): 20 counters."""
    buf = (C.c_uint64 * 20)()
    _check(_lib.cf_debug_tile_phases(buf, 1 if reset else 0))
    return list(buf)


def debug_tc_pipe(M, N, K, nb, reps, prefetch, A, B) -> float:
    """Test hook (include/cf_debug.h): mainloop throughput probe; returns device ms."""
    ms = C.c_float()
    _check(_lib.cf_debug_tc_pipe(M, N, K, nb, reps, prefetch, A.data_ptr(), B.data_ptr(), C.byref(ms)))
    return ms.value


def debug_set_worker_roles(low_first: int, strict: bool = False) -> None:
    """Test hook (include/cf_debug.h): workers that take dW chunks first / strict roles."""
    _check(_lib.cf_debug_set_worker_roles(low_first, 1 if strict else 0))


def debug_set_m2_rows(rows: int) -> None:
    """Test hook (include/cf_debug.h): batch size from which 256-row GEMM tiles are used."""
    _check(_lib.cf_debug_set_m2_rows(rows))


def debug_program_listing(g: "Graph", fetches, precision: int = F32, parallel_iterations: int = 0) -> str:
    """Test hook: the device program (description + body programs) without a GPU."""
    arr = (cf_tensor * max(len(fetches), 1))(*[t.c for t in fetches])
    need = C.c_size_t()
    _check(_lib.cf_debug_program_listing(g.h, precision, parallel_iterations, len(fetches), arr,
                                          None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    _check(_lib.cf_debug_program_listing(g.h, precision, parallel_iterations, len(fetches), arr,
                                          buf, len(buf), None))
    return buf.value.decode()
