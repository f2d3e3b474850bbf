// Device program: what the host compiler (compiler.cpp) hands to the persistent driver
// kernel (runtime.cu). Plain structs, identical layout on host and device.
#pragma once
#include <cstdint>

namespace cfdev {

// ---- token: the device form of the paper's (value, is_dead, tag) tuple.
// The tag is implicit: the driver evaluates one iteration of a frame at a time, so every
// token in the table belongs to the current (frame, iteration); tensors flowing across
// iterations carry their storage address, which encodes the producing iteration.
enum TokKind : uint8_t { TK_UNSET = 0, TK_IMM = 1, TK_PTR = 2, TK_HANDLE = 3, TK_FLOW = 4 };
enum DevDT : uint8_t { D_BOOL = 0, D_I32 = 1, D_I64 = 2, D_F32 = 3, D_BF16 = 5, D_NONE = 7 };

struct Tok {
  int64_t v;       // immediate scalar, device address, or handle id
  int32_t writer;  // heavy instance producing the bytes at v (-1: ready)
  uint8_t dead;
  uint8_t kind;
  uint8_t dt;
  uint8_t pad;
};
static_assert(sizeof(Tok) == 16, "Tok layout");

// ---- interpreter opcodes
enum Op : int32_t {
  OP_NOP = 0,
  OP_PLACEHOLDER,   // token preset at run start
  OP_CONST,         // aux0: 1 = immediate scalar (imm0), 0 = pointer (imm0 = device address)
  OP_PASS,          // Identity / StopGradient / Reshape (views)
  OP_SWITCH,        // aux0: cond_id (-1 loop), aux1: is loop switch
  OP_MERGE,         // cond merge
  OP_MERGE_LOOP,    // aux0: frame; in0 = Enter, in1 = NextIteration
  OP_ENTER,         // aux0: frame
  OP_EXIT,          // aux0: frame
  OP_NEXTITER,      // aux0: frame
  OP_SCALAR,        // aux0: scalar sub-op (SC_*)
  OP_REDUCE_I,      // aux0: 0 max, 1 min; aux1: element count
  OP_SLICE_I,       // 1-D int/bool slice view: imm0 = byte offset
  OP_FLOW,          // flow-valued arithmetic (Add/AddN/Const/ZerosLike of flows)
  OP_TA_CREATE,     // aux0: ta id
  OP_TA_READ,       // aux0: ta id (static, for checks)
  OP_TA_WRITE,
  OP_TA_STACK,
  OP_TA_UNSTACK,
  OP_TA_GRAD,       // aux0: grad ta id
  OP_STACK_CREATE,  // aux0: stack id
  OP_STACK_PUSH,
  OP_STACK_POP,
  OP_HEAVY,         // aux0: heavy kind (HK_*), aux1: sub-op / flags
  OP_ACC,           // fused accumulator Add (aux0: acc id): output = the accumulator buffer
  OP_SEND,          // cross-GPU Send (aux0: channel index)
  OP_RECV,          // cross-GPU Recv (aux0: channel index); output placed like a heavy output
  OP_WAVE,          // body-program marker: the next aux0 nodes are independent routing / stack
                    // nodes, evaluated in parallel by the driver CTA's helper warps
  OP_FRAME,         // body-program step: run a nested frame (aux0: frame id) to its Exits
  OP_HEAVY_BATCH,   // body-program marker: the next aux0 nodes are tensor-core LSTM nodes of one
                    // phase (each input an earlier member's output or ready before the marker);
                    // their instances are built together, one helper lane per node
  OP__COUNT
};

enum ScalarOp : int32_t {
  SC_ADD = 0, SC_SUB, SC_MUL, SC_LESS, SC_LEQ, SC_GREATER, SC_EQ, SC_AND, SC_NOT, SC_CAST
};

// ---- heavy work kinds (executed by worker CTAs, tiled)
enum HeavyKind : int32_t {
  HK_NOP = 0,       // join: completes when its dependencies complete (0 tiles)
  HK_EW,            // elementwise; sub = EW_*
  HK_FILL,          // out[i] = scalar at p1 (or imm)
  HK_COPY,          // bytes
  HK_REDUCE_SUM,    // all elements -> scalar (deterministic two-level)
  HK_REDUCE_SUM0,   // [M,N] -> [N]
  HK_MATMUL,        // sub bit0 ta, bit1 tb
  HK_LSTM_FWD,      // fused LSTM cell (sub bit0: masked)
  HK_LSTM_BWD_EW,   // dz, dc_prev
  HK_LSTM_BWD_MM,   // dxh = dz W, dW = dz^T [x,h], db = colsum dz
  HK_ACC,           // dst += src (grad TensorArray double write)
  HK_PREP_WP,       // bf16 gate-interleaved W rows for the forward GEMM (B operand)
  HK_PREP_WT,       // bf16 W^T for the d[x,h] GEMM (B operand)
  HK_LSTM_FWD_TC,   // tcgen05 gate GEMM + fused LSTM epilogue
  HK_LSTM_BWD_EW_BF,// dz (bf16) + dc + db partials
  HK_LSTM_DXH_TC,   // tcgen05 d[x,h] = dz W
  HK_LSTM_DW_TC,    // tcgen05 dW (+)= dz^T [x,h] (MN-major operands) + db
  HK_SWAP,          // stack swap copy on the host I/O thread's copy stream (sub 0: D2H, 1: H2D)
  HK_WAIT,          // no tiles: completes when a channel flag shows the expected message (a14)
  HK_LSTM_XPROJ_TC, // tcgen05 x-projection of a cell: Zx = x Wx^T (fp32), ahead of the recurrence
  HK_MATMUL_TC,     // tcgen05 generic GEMM of registered bf16 operands (sub bit0 ta, bit1 tb)
  HK__COUNT
};

enum EwOp : int32_t {
  EW_ADD = 0, EW_SUB, EW_MUL, EW_NEG, EW_SIGMOID, EW_TANH, EW_RELU, EW_RELUGRAD,
  EW_BIASADD, EW_SELECT, EW_ADDN, EW_ZEROS
};

// ---- placement of a heavy output (SURVEY.md §7.2 "static buffer pointer per (edge, slot)")
enum Place : int32_t { PL_ROOT = 0, PL_RING = 1, PL_ARENA = 2, PL_TA = 3, PL_ACC = 4,
                       PL_SWAP = 5 /* stacked value with host backing: device ring of K + 1 */ };

struct PlaceDesc {
  int32_t kind;
  int32_t slots;       // RING: R = K + 1; ARENA: frame iteration bound
  int32_t ta;          // PL_TA: static TensorArray id
  int32_t index_vid;   // PL_TA: value id of the write index
  int64_t base;        // device address (ROOT / RING / ARENA)
  int64_t elem_bytes;
  int32_t dt;          // DevDT of the stored elements
  int32_t pad;
};

struct DNode {
  int32_t op;
  int32_t n_in;
  int32_t in_off;      // into prog.in_vids
  int32_t n_ctrl;
  int32_t ctrl_off;    // into prog.in_vids (value ids of producers' ctrl tokens)
  int32_t n_out;
  int32_t out_vid;     // first output value id
  int32_t ctrl_vid;    // this node's own ctrl token
  int32_t place_off;   // into prog.places (n_out entries) for heavy nodes; -1 otherwise
  int32_t aux[7];
  int64_t imm[4];      // op-specific sizes / constants
  int32_t ctx;         // structured cond context (prog.ctxs index; 0 = loop level)
  int32_t pad[3];      // 16-byte records (the driver stages body programs with int4 copies)
};

// Structured cond context of a frame body (reading R20): a branch of a cond is live iff its
// parent is live and the predicate (a driver scalar) selects it; nodes of a dead branch are not
// evaluated at all, capture Switches are compiled away, and the cond's Merges pick the live
// branch's input.
struct DCtx {
  int32_t parent;      // 0 = loop level
  int32_t pred_vid;    // value id of the cond predicate (in the parent context)
  int32_t branch;      // 1 = true branch (Switch port 1)
  int32_t cond_id;     // for the branch-bit trace
};
static_assert(sizeof(DNode) % 16 == 0, "DNode layout");

// Fused loop accumulator ("sum gradients eagerly into new loop
// variables"): one buffer updated in place by its producers, initialised at frame start.
struct DAcc {
  int64_t base;         // device buffer (fp32)
  int64_t bytes;
  int32_t frame;
  int32_t init_vid;     // value id of the loop variable's init (Enter input)
  int32_t init_zero;    // 1: init is a zeros constant (fill), else copy from init_vid
  int32_t pad;
};

// TMA operand registry entry: a bf16 buffer viewed as [slots][rows][cols]
struct DReg {
  int64_t base;
  int64_t slot_bytes;
  int32_t slots, rows, cols, map0;   // map0: index of its 3 tensor maps (KA, KB, MN)
  double inv_slot;                    // 1 / slot_bytes (division-free slot index on device)
};

struct DFrame {
  int32_t K;            // parallel_iterations
  int32_t bound;        // iteration bound (arena slots / stack capacity)
  int32_t body_off, n_body;     // node ids in evaluation order, into prog.order
  int32_t enter_off, n_enter;   // Enter node ids
  int32_t exit_off, n_exit;     // Exit node ids
  int32_t counter_switch;       // node id of the hidden counter's Switch
  int32_t counter_enter;        // node id of the hidden counter's Enter
  int32_t iter_base;            // offset into per-iteration counters (size bound + 1)
  int32_t acc_off, n_acc;       // accumulators initialised at frame start (into prog.order)
  int32_t bn_off;               // body program: DNodes in evaluation order (prog.body_nodes)
  int32_t bi_off, bi_count;     // their input ids (prog.body_ivids), offsets rebased
  int32_t parent;               // enclosing frame (-1: root): one instance per parent iteration
};

struct DTA {
  int64_t base;         // static buffer (device)
  int64_t elem_bytes;
  int32_t size;
  int32_t is_grad;
  int32_t grad_id;      // id of its gradient TA (-1 none)
  int32_t dt;
};

struct DStack {
  int32_t capacity;     // entries per instance
  int32_t entry_off;    // into the stack entry pool (Tok); instance k at entry_off + k * capacity
  int32_t instances;    // 1, or one per iteration index of the frame that creates the stack
  int32_t depth_off;    // into the stack depth array (one depth per instance)
};

// Root program step: a node id (>= 0) or a frame (-(frame + 1)).
// ---- swapped stack arena: the value's device storage
// is a ring of `ring` slots (slot = iteration % ring); each push also copies the entry to host
// slot = push index; a pop whose ring slot no longer holds the entry brings it back first.
struct DSwap {
  int64_t dev_base;       // device ring
  int64_t elem_bytes;
  int64_t host_base;      // pinned host backing, [capacity][elem_bytes]
  int64_t in_base;        // swap-in ring [ring][elem_bytes], slot = gradient-loop iteration % ring
  int32_t ring, owner_off;   // owner_off: into RunArgs.swap_owner ([ring] stack entry ids)
  int32_t capacity;
  int32_t in_ring;        // swap-in ring slots: K + 1, or K + 9 in bf16 mode (a chunked dW reads
                          // the popped x / h of its last 8 gradient steps after they left the window)
};

// ---- cross-GPU channel (one Send/Recv edge). Each session holds one
// half of the channel in its IPC-exported channel memory:
//   receiving half: flags[slots] (u64) + data[slots][elem_bytes]   (written by the sender)
//   sending half:   acks[slots]  (u64) + done (u64)                  (written by the receiver)
// flag = epoch << 32 | (2 * (iter + 1) + dead); ack = epoch << 32 | (iter + 1); done = epoch of
// the receiver's last finished run. Message slot = iter % slots.
struct DChan {
  int32_t channel, role;     // role 0: this session receives, 1: sends
  int32_t peer, slots;
  int64_t elem_bytes;
  int32_t dt, frame;
  unsigned long long* flags;        // receiving half (local)  | sending half: peer's flags
  uint8_t* data;                    // receiving half (local)  | sending half: peer's data
  unsigned long long* acks;         // sending half (local)    | receiving half: peer's acks
  unsigned long long* done;         // sending half (local)    | receiving half: peer's done
};

constexpr int kDwMax = 16;   // most gradient-loop steps one dW instance accumulates
// root step tags (Prog.root_steps: node id, or -(frame + 1)): a heavy root node no frame
// depends on, published to the low-priority queue; the early W^T preparation of a tensor-core
// LSTMCellGrad node (the node's imm[3]: root weight's value id + 1 in the low 32 bits, the
// node whose preparation and W^T buffer it shares + 1 in the high 32 bits)
constexpr int32_t kRootLow = 1 << 29, kRootPrep = 1 << 30, kRootNode = kRootLow - 1;

struct Prog {
  int32_t n_nodes, n_vids, n_frames, n_tas, n_stacks;
  int32_t n_root_steps;
  int32_t n_fetch;
  int32_t n_conds;
  int32_t branch_bound;         // iterations recorded per cond in the branch-bit array
  int32_t dw_chunk;             // gradient-loop steps per dW instance (rings sized for it)
  const DNode* nodes;
  const int32_t* in_vids;
  const PlaceDesc* places;
  const DFrame* frames;
  const int32_t* order;         // frame bodies / enters / exits
  const int32_t* root_steps;
  const DTA* tas;
  const DStack* stacks;
  const int32_t* fetch_vids;
  const DAcc* accs;
  int32_t n_accs;
  int32_t n_reg;                // registry entries (static part; feeds appended per run)
  const DReg* reg;
  const void* maps;             // CUtensorMap[3 * n_reg], 64-byte aligned
  const DNode* body_nodes;      // per-frame body programs (staged into driver smem)
  const int32_t* body_ivids;
  int32_t max_body, max_bi;     // largest body (nodes, input ids)
  int32_t n_places, iter_counters;
  int32_t precision;            // 3 = f32 SIMT, 5 = bf16 tcgen05
  int32_t n_chans;
  const DChan* chans;
  int32_t n_swaps, n_ctxs;
  const DSwap* swaps;
  const DCtx* ctxs;
  int32_t nested;               // 1: a frame runs inside another frame's body (f2)
  int32_t n_stack_depths;       // stack instances (depth counters)
};

// ---- heavy instance record (written by the driver, read by workers)
struct Inst {
  int32_t kind, sub;
  int32_t ntiles, frame;
  int32_t iter, pad;
  int64_t n, m, k;      // sizes
  int64_t p[20];        // pointers (p[13] = primary output for generic kinds)
  int64_t s[8];         // scalars
  int64_t dts;          // device dtypes: input j at bits [4j, 4j+4), output at [32, 36)
  unsigned long long* signal;        // optional: written (release, system scope) with
  unsigned long long signal_value;   // signal_value when the last tile completes
};

// ---- run-time state shared by the driver CTA and the worker CTAs
struct RunState {
  // job queue: entries = (inst << 20 | tile) encoded as uint64; tail published by driver
  unsigned long long q_head;     // high-priority ring: claimed by workers (CAS)
  unsigned long long q_tail;     // published by driver (release)
  unsigned long long lq_head;    // low-priority ring (filler work: dW chunks, preps)
  unsigned long long lq_tail;
  unsigned long long q_done;     // tiles finished (for ring capacity)
  int32_t quit;                  // 1 = workers exit
  int32_t error;                 // cf_status from the device
  unsigned long long cq_tail;    // completion queue reserve (workers)
  unsigned long long cq_head;    // consumed by driver
  int64_t error_info;
  // trace
  int32_t trip[16];
  int32_t max_inflight[16];
  long long pushes, pops;
  long long sends, recvs;
  long long swap_out, swap_in, bytes_d2h, bytes_h2d;
  int32_t smem_mask, smem_used;   // driver arrays staged in shared memory (bit per array)
  int32_t max_depth, exit_fires;
  long long instances, tiles, dead_skipped;
  unsigned long long t_start, t_end;
  long long op_count[64], op_cycles[64];   // driver self-profile: opcodes [0,32), regions [32,64)
};

// a placeholder's token for this run, applied to the token table by the driver CTA at start
struct PresetTok {
  int64_t vid;
  Tok t;
};

struct RunArgs {
  Prog prog;
  RunState* st;
  Tok* toks;                 // [n_vids]
  int32_t* wait_ovf;         // [4096] channel waits published while the driver's table is full
  const PresetTok* preset;   // [n_preset] this run's placeholder tokens (one upload per run)
  int32_t n_preset;
  int32_t pad_preset;
  Tok* stack_pool;           // stack entries
  int32_t* stack_depth;      // [n_stacks]
  int64_t* ta_base;          // [n_tas] runtime base (may alias on unstack)
  int32_t* ta_writer;        // [sum sizes] per-slot writer instance
  uint8_t* ta_written;       // [sum sizes]
  int32_t* ta_slot_off;      // [n_tas] offset into ta_writer / ta_written
  Inst* insts;               // [inst_cap]
  int32_t inst_cap;
  int32_t* tile_next;        // per instance: next tile to claim (atomic, workers)
  int32_t* inst_tiles_done;  // atomic per instance
  int32_t* edge_next;        // [edge_cap]
  int32_t* edge_to;
  int32_t edge_cap;
  unsigned long long* queue; // [q_cap] ready instance ids (tiles claimed via tile_next)
  unsigned long long q_cap;
  int32_t* cq;               // [cq_cap] completion queue (inst + 1; 0 = empty)
  unsigned long long cq_cap;
  int32_t* iter_outstanding; // per frame iteration
  uint8_t* branch_bits;      // [n_conds * branch_bound]
  void** fetch_out;          // caller buffers
  uint8_t* fetch_dead;
  int64_t* fetch_bytes;
  int64_t watchdog_ns;
  int32_t sched_seed;
  int32_t num_workers;
  int64_t dyn_smem;          // dynamic shared memory per CTA (driver: token table if it fits)
  int64_t* inst_aux;         // [inst_cap][kDwMax * 6] per-instance side data (chunked dW steps)
  int32_t* dw_count;         // [n_nodes] pending dW steps per LSTMCellGrad node (chunking)
  int64_t* dw_pend;          // [n_nodes][kDwMax][10] pending step records
  unsigned long long* lq;    // low-priority job ring (same capacity as queue)
  unsigned long long* prof;  // optional: per instance {create, publish, first start, last end,
                             //  busy ns, kind|ntiles} (profiling hook, cf_debug.h)
  int32_t* prep_inst;        // [n_nodes] per-run weight-prep instance of LSTM nodes (-1)
  int32_t* acc_writer;       // [n_accs] latest instance writing each accumulator
  const uint8_t* vdt;        // [n_vids] device dtype of every value
  unsigned long long epoch;  // run counter (channel message tags)
  // swap I/O (a8): requests go to the host I/O thread through a mapped ring; the thread's
  // copy streams write completions (instance id + 1) into io_cq in stream order
  int32_t* swap_owner;       // [sum of rings] stack entry id held by each device ring slot
  unsigned long long* io_req;        // mapped host ring [io_cap][4]: src, dst, bytes, id|dir<<32
  unsigned long long* io_req_tail;   // mapped host word: requests published
  int32_t* io_cq;            // device ring [io_cap]
  int32_t io_cap;
  int32_t pad4;
};

}  // namespace cfdev
