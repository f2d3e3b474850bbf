/*
 * cf.h -- C-ABI of libcf, a B200-native implementation of in-graph dynamic control flow
 * (Yu et al., "Dynamic Control Flow in Large-Scale Machine Learning", arXiv 1805.01772).
 *
 * Citations "PAPER.md:a-b" refer to lines of the paper's LaTeX source; "SPEC.md:n" to the
 * CPU-program specification written from it (used for error names only).
 *
 * Conventions (all entry points):
 *  - Every call returns a cf_status; CF_OK = 0. On error, cf_last_error() returns a
 *    thread-local message valid until the next cf_* call on that thread. A failing build
 *    call leaves the graph unchanged except for nodes already appended (never mutated).
 *  - Ownership: cf_graph and cf_session are library-owned until *_destroy. Tensor memory
 *    passed in (feeds) or out (fetch buffers) is caller-owned and BORROWED for the duration
 *    of the call; the library never frees it. Library scratch (token tables, rings, stacks,
 *    TensorArray storage, work queues) is allocated by cf_session_create and freed by
 *    cf_session_destroy.
 *  - Layout: every tensor buffer is dense row-major (C order) of the declared shape.
 *  - Symbolic tensors (cf_tensor) are (node, port) handles into one graph; they carry no
 *    ownership ("SymbolicTensor").
 *  - No CPU fallback: a graph the device compiler cannot lower is rejected with
 *    CF_E_UNSUPPORTED; a machine without a CUDA device gets CF_E_CUDA from
 *    cf_session_create. Graph construction, gradients and validation are host-only and
 *    work without a GPU.
 */
#ifndef CF_H_
#define CF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t cf_status;
enum {
  CF_OK = 0,
  CF_E_ARITY = 1,               /* wrong number of inputs / loop variables   */
  CF_E_DTYPE = 2,               /* dtype mismatch                             */
  CF_E_SHAPE = 3,               /* shape mismatch / index out of range   */
  CF_E_NONBOOL_PRED = 4,        /* cond / loop predicate not a bool scalar   */
  CF_E_BRANCH_MISMATCH = 5,     /* cond branches differ in arity or dtype    */
  CF_E_INVALID_GRAPH = 6,       /* validate(): illegal cycle, arity, context crossing      */
  CF_E_NONSCALAR_OBJECTIVE = 7, /* gradients of a non-scalar y               */
  CF_E_NO_GRADIENT = 8,         /* op on the path has no gradient function                 */
  CF_E_MISSING_FEED = 9,        /* placeholder without a feed                */
  CF_E_UNSUPPORTED = 10,        /* graph the device compiler cannot lower (no fallback)    */
  CF_E_DEADLOCK = 11,           /* device watchdog fired (SPEC.md:317 DeadlockDetected)    */
  CF_E_POP_EMPTY = 12,          /* StackPop of an empty stack                */
  CF_E_DOUBLE_WRITE = 13,       /* TensorArray slot written twice     */
  CF_E_STACK_BUDGET = 14,       /* stack / iteration bound exceeded          */
  CF_E_CUDA = 15,               /* CUDA runtime error or no device                         */
  CF_E_NCCL = 16
};

typedef enum {
  CF_BOOL = 0, CF_I32 = 1, CF_I64 = 2, CF_F32 = 3, CF_F64 = 4, CF_BF16 = 5,
  CF_FLOW = 6,  /* TensorArray flow scalar: an ordering token, differentiable (TF convention) */
  CF_RES = 7    /* resource handle (TensorArray, Stack) */
} cf_dtype;

typedef struct cf_graph cf_graph;
typedef struct { int32_t node; int32_t port; } cf_tensor;

/* Dense buffer descriptor. data is a device pointer for cf_run feeds/fetches. */
typedef struct {
  void* data;
  int32_t dtype;     /* cf_dtype */
  int32_t rank;
  int64_t shape[8];
} cf_buffer;

const char* cf_last_error(void);
const char* cf_version(void);

/* ---------------------------------------------------------------- graph construction */
cf_status cf_graph_create(cf_graph** out);
void cf_graph_destroy(cf_graph* g);

/* Feedable input; name must be unique. Lives in the root context. */
cf_status cf_placeholder(cf_graph* g, const char* name, int32_t dtype, int32_t rank,
                         const int64_t* shape, cf_tensor* out);
/* Constant from host memory (copied). Created in the current construction context. */
cf_status cf_const(cf_graph* g, int32_t dtype, int32_t rank, const int64_t* shape,
                   const void* host_data, cf_tensor* out);
/* Generic op. op names: Identity Add Sub Mul Neg AddN MatMul Transpose ReduceSum ReduceMax
 * ReduceMin BiasAdd Fill ZerosLike Less LessEqual Greater Equal LogicalAnd LogicalNot Select
 * Sigmoid Tanh Relu ReluGrad Concat Slice Reshape Cast LSTMCell LSTMCellGrad StackCreate
 * StackPush StackPop Send Recv. attrs: "key=value;key=v1,v2" (ints, floats, bools as 0/1).
 * Send(value, ix; channel, peer) / Recv(ix; channel, peer, dtype, shape): one edge of a program
 * partitioned across GPUs (§4.4). The message key is (channel, iteration of
 * the enclosing loop); a dead Send delivers the is_dead signal. Gradients:
 * grad(Send) = Recv and grad(Recv) = Send on channel ^ (1 << 20) (the mirrored edge).
 * External inputs are captured automatically: Enter into loop bodies, Switch into cond
 * branches, "one Switch for each external tensor".
 * *n_out receives the number of outputs written to out (capacity 8). */
cf_status cf_op(cf_graph* g, const char* op, int32_t n_in, const cf_tensor* in,
                const char* attrs, int32_t* n_out, cf_tensor* out);

/* while_loop(pred, body, inits) compiled to Enter/Merge/Switch/
 * NextIteration/Exit per loop variable plus a hidden int64 counter
 * (PAPER.md:1025-1028). pred/body are called once, at construction, with the Merge
 * (pred) / Switch-true (body) outputs of the n user loop variables. parallel_iterations
 * >= 1 bounds the iterations in flight. outs receives the n Exit
 * outputs; frame_name may be NULL (auto) and must be unique per graph. */
typedef cf_status (*cf_pred_fn)(cf_graph* g, int32_t n, const cf_tensor* vars,
                                cf_tensor* out_pred, void* user);
typedef cf_status (*cf_body_fn)(cf_graph* g, int32_t n, const cf_tensor* vars,
                                cf_tensor* out_vars, void* user);
cf_status cf_while_loop(cf_graph* g, cf_pred_fn pred, cf_body_fn body, void* user,
                        int32_t n, const cf_tensor* inits, int32_t parallel_iterations,
                        const char* frame_name, cf_tensor* outs);
/* Same, also returning the hidden counter's Exit (the trip count). */
cf_status cf_while_loop_counted(cf_graph* g, cf_pred_fn pred, cf_body_fn body, void* user,
                                int32_t n, const cf_tensor* inits, int32_t parallel_iterations,
                                const char* frame_name, cf_tensor* outs, cf_tensor* trip_count);

/* cond(pred, true_fn, false_fn) compiled to Switch/Merge only
 * (PAPER.md:624-637). Each branch fills n_out tensors; both must agree in dtype. outs
 * receives one Merge per output. pred must be a bool scalar. */
typedef cf_status (*cf_branch_fn)(cf_graph* g, int32_t n_out, cf_tensor* outs, void* user);
cf_status cf_cond(cf_graph* g, cf_tensor pred, cf_branch_fn true_fn, cf_branch_fn false_fn,
                  void* user, int32_t n_out, cf_tensor* outs);

/* TensorArray: write-once indexed container, reads allowed many times.
 * handle (CF_RES) and flow (CF_FLOW) are separate tensors; every op consumes the current
 * flow and write/unstack return the new flow (ordering). */
cf_status cf_ta_create(cf_graph* g, int64_t size, int32_t dtype, int32_t elem_rank,
                       const int64_t* elem_shape, cf_tensor* handle, cf_tensor* flow);
cf_status cf_ta_read(cf_graph* g, cf_tensor handle, cf_tensor index, cf_tensor flow,
                     cf_tensor* value);
cf_status cf_ta_write(cf_graph* g, cf_tensor handle, cf_tensor index, cf_tensor value,
                      cf_tensor flow, cf_tensor* flow_out);
cf_status cf_ta_unstack(cf_graph* g, cf_tensor handle, cf_tensor value, cf_tensor flow,
                        cf_tensor* flow_out);
cf_status cf_ta_stack(cf_graph* g, cf_tensor handle, cf_tensor flow, cf_tensor* value);

/* gradients(y, xs): appends the gradient graph -- gradient conds
 * (PAPER.md:960-969), gradient loops with stack-saved intermediates and predicate stacks
 * (PAPER.md:1022-1098), TensorArray duals. y must be a float scalar
 * in the root context. Unreached xs get zeros. */
cf_status cf_gradients(cf_graph* g, cf_tensor y, int32_t n_x, const cf_tensor* xs,
                       cf_tensor* out_grads);

/* Structural validation. Writes a newline-separated report of violations
 * (empty = valid) into report (NUL-terminated, truncated to cap). Returns CF_OK if valid,
 * CF_E_INVALID_GRAPH otherwise. */
cf_status cf_validate(const cf_graph* g, char* report, size_t cap);
/* JSON dump of the graph (SPEC.md:125 style). *needed receives the full length + 1. */
cf_status cf_graph_json(const cf_graph* g, char* buf, size_t cap, size_t* needed);
cf_status cf_graph_num_nodes(const cf_graph* g, int32_t* n);
cf_status cf_tensor_info(const cf_graph* g, cf_tensor t, int32_t* dtype, int32_t* rank,
                         int64_t* shape /* cap 8 */);

/* ---------------------------------------------------------------- execution */
typedef struct cf_session cf_session;

typedef struct {
  int32_t precision;            /* CF_F32: SIMT fp32 parity path; CF_BF16: tcgen05 path   */
  int32_t parallel_iterations;  /* 0 = per-loop value; else overrides every loop          */
  int32_t device;               /* CUDA device ordinal                                    */
  int32_t num_workers;          /* 0 = one worker CTA per SM (minus the driver CTA)       */
  void* stream;                 /* cudaStream_t; NULL = a library-owned stream, each run
                                   ordered after the legacy default stream's prior work  */
  int64_t max_iterations;       /* per-frame iteration bound for stack arenas; 0 = infer
                                   from TensorArray sizes                                */
  int64_t watchdog_ms;          /* device watchdog; 0 = 60000                             */
  int32_t sched_seed;           /* 0 = FIFO; else shuffled worker claim order (race check) */
  int32_t reserved[7];
  /* Stack swapping: stacked activations stay in
   * device memory up to stack_budget_bytes; beyond it the largest stacked values (each at
   * least swap_min_bytes) keep only a (parallel_iterations + 1)-slot device ring and move to
   * pinned host memory after the push (device -> host on a copy stream), coming back ahead
   * of the pop (host -> device). <= 0 = never swap (a zero-initialised struct swaps
   * nothing); 1 = swap every eligible value. */
  int64_t stack_budget_bytes;
  int64_t swap_min_bytes;       /* 0 = 4096 ("do not swap small tensors") */
  int32_t swap_smallest_first;  /* 0: swap the largest stacked values first (fewest swaps);
                                   1: smallest first (fewest bytes per step, for a link that
                                   cannot hide the largest ones)                           */
  int32_t pad_;
  /* Caller allocator: when dev_alloc is set, every device buffer the
   * session owns (arenas, rings, stack pool, instance records, queues, scratch) comes from
   * dev_alloc(bytes, alloc_user) -- 256-byte aligned, or NULL to fail with CF_E_CUDA -- and
   * goes back through dev_free(ptr, alloc_user) in cf_session_destroy. NULL = cudaMalloc /
   * cudaFree. The IPC-exported channel block of a multi-GPU session (cf_session_ipc_handle)
   * is always cudaMalloc'ed: cudaIpcGetMemHandle needs an allocation of its own. */
  void* (*dev_alloc)(size_t bytes, void* alloc_user);
  void (*dev_free)(void* ptr, void* alloc_user);
  void* alloc_user;
  /* Swap copy streams (a8; "separate streams for GPU-to-CPU and
   * CPU-to-GPU transfers"): cudaStream_t for the device -> host and host -> device copies of
   * swapped stack entries; NULL = library-owned non-blocking streams (three each). */
  void* d2h_stream;
  void* h2d_stream;
} cf_run_opts;

/* Control trace -- compared bit-exact with the oracle's. */
typedef struct {
  int32_t n_frames;
  int32_t trip_count[16];       /* per loop frame, in frame creation order               */
  int32_t max_inflight[16];     /* max iterations in flight per frame (<= K)             */
  int64_t pushes, pops;         /* total stack pushes / pops                            */
  int32_t max_depth;            /* max depth over all stacks                             */
  int32_t exit_fires;           /* Exit firings (each Exit once per frame instance)      */
  int64_t instances;            /* device work items (heavy op instances) executed       */
  int64_t tiles;                /* device tiles executed                                 */
  int64_t dead_skipped;         /* heavy ops skipped because an input was dead           */
  int32_t n_branch_bits;        /* bits written into branch_bits                        */
  uint8_t* branch_bits;         /* caller buffer or NULL: per (cond, iteration) taken bit */
  int32_t branch_bits_cap;
  double wall_ms;               /* device time of the run (CUDA events)                 */
  int64_t sends, recvs;         /* cross-GPU messages sent / received, live or dead (a14)  */
  int64_t swap_out, swap_in;    /* stack entries moved device -> host / host -> device (a8) */
  int64_t bytes_d2h, bytes_h2d; /* their bytes                                            */
} cf_trace;

/* Compile the graph for the device (placement of every value, lowering to the device
 * driver's node table) and allocate device state. fetches: tensors cf_run returns. */
cf_status cf_session_create(const cf_graph* g, const cf_run_opts* opts, int32_t n_fetch,
                            const cf_tensor* fetches, cf_session** out);
/* Run the whole graph once: ONE launch of the persistent driver kernel, which evaluates
 * every control decision on the device (no host round trip per iteration). feeds are
 * device buffers matched to placeholders by name; outs are caller-allocated device buffers
 * (one per fetch, dtype per cf_session_fetch_dtype). out_dead[i] = 1 marks a dead fetch
 * (DeadMarker): its buffer is left untouched. Synchronous. trace may be NULL. */
cf_status cf_run(cf_session* s, int32_t n_feed, const char* const* feed_names,
                 const cf_buffer* feeds, cf_buffer* outs, uint8_t* out_dead, cf_trace* trace);
/* Device dtype the session expects for a placeholder feed / produces for a fetch. */
cf_status cf_session_feed_dtype(const cf_session* s, const char* name, int32_t* dtype);
cf_status cf_session_fetch_dtype(const cf_session* s, int32_t i, int32_t* dtype);
/* Human-readable summary of the compiled program (node kinds, placements, bytes). */
cf_status cf_session_describe(const cf_session* s, char* buf, size_t cap);
void cf_session_destroy(cf_session* s);

/* ---- multi-GPU layer pipeline ---------------------
 * A graph holding Send/Recv nodes is one partition of a program split across GPUs, one
 * process per GPU. Every Send/Recv is one half of a channel; the session keeps its halves in
 * one device allocation: the receiving half holds `slots` payload slots + 64-bit flags written
 * by the sender over NVLink, the sending half holds 64-bit acks + a "run done" word written
 * by the receiver. slots = parallel_iterations + 1 of the enclosing loop.
 *
 * cf_session_channels: this session's halves, 7 int64 per row: channel, role (0 = receives,
 *   1 = sends), peer rank, slots, payload bytes, device dtype, byte offset in the allocation.
 *   *n = number of rows (rows beyond cap are not written; table may be NULL).
 * cf_session_ipc_handle: the allocation's cudaIpcMemHandle_t (CF_IPC_HANDLE_BYTES bytes,
 *   zeros if the session has no channel).
 * cf_session_connect: import a peer's handle + table (exchanged by the caller, e.g. with
 *   torch.distributed.all_gather_object) before the first cf_run. CF_E_UNSUPPORTED when the
 *   peer lacks the mirrored half or the halves disagree (slots, payload bytes, dtype);
 *   CF_E_CUDA when the handle cannot be opened (peers must be separate processes).
 * cf_run on a session with an unconnected channel fails with CF_E_UNSUPPORTED. All partitions
 * must call cf_run the same number of times (run epochs tag the messages). */
#define CF_IPC_HANDLE_BYTES 64
cf_status cf_session_channels(const cf_session* s, int32_t cap, int64_t* table, int32_t* n);
cf_status cf_session_ipc_handle(const cf_session* s, void* handle);
cf_status cf_session_connect(cf_session* s, int32_t peer, const void* handle, int32_t n,
                             const int64_t* table);

#ifdef __cplusplus
}
#endif
#endif /* CF_H_ */
