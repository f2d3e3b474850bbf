// Host compiler: cf::Graph -> device program (program.h) + buffer plan.
#pragma once
#include <map>
#include <string>
#include <vector>

#include "ir.h"
#include "program.h"

namespace cf {

struct BufPlan {
  size_t bytes = 0;
  bool zero = false;                 // zero-filled at every run start
  std::vector<uint8_t> init;         // uploaded once (constants)
  std::string what;
};

struct FeedInfo {
  int vid = -1;
  int32_t graph_dt = 0;
  int32_t dev_dt = 0;
  int64_t bytes = 0;
  bool scalar_ctrl = false;
};

struct FetchInfo {
  int vid = -1;
  int32_t dev_dt = 0;
  int64_t bytes = 0;
};

// one half of a cross-GPU channel (program.h DChan); offset into the session's channel memory
struct ChanPlan {
  int32_t channel = 0, role = 0, peer = 0, slots = 1, dt = 0, frame = -1;
  int64_t elem_bytes = 0;
  int64_t offset = 0, bytes = 0;
};

// swapped stack arena (program.h DSwap); dev_base = buffer id until the runtime patches it
struct SwapPlan {
  int place = -1;          // index into places
  int in_buf = -1;         // buffer id of the swap-in ring (pops of the gradient loop)
  int64_t elem_bytes = 0;
  int32_t ring = 0, capacity = 0;
  int32_t in_ring = 0;     // swap-in ring slots (program.h DSwap)
};

struct HostProgram {
  std::vector<cfdev::DNode> nodes;
  std::vector<int32_t> in_vids;
  std::vector<cfdev::PlaceDesc> places;
  std::vector<cfdev::DFrame> frames;
  std::vector<int32_t> order;
  std::vector<int32_t> root_steps;
  std::vector<cfdev::DTA> tas;
  std::vector<cfdev::DStack> stacks;
  std::vector<int32_t> fetch_vids;
  std::vector<cfdev::DAcc> accs;
  std::vector<cfdev::DReg> reg;       // base = buffer id until the runtime patches it
  std::vector<uint8_t> vdt;
  std::vector<cfdev::DNode> body_nodes;
  std::vector<int32_t> body_ivids;
  int max_body = 0, max_bi = 0;
  int32_t precision = CF_F32;
  std::vector<std::string> frame_names;
  int n_vids = 0;
  int n_conds = 0;
  int branch_bound = 1;
  int dw_chunk = 1;              // gradient-loop steps per dW instance (bf16 mode: kDwChunk)
  int iter_counters = 0;
  int stack_pool = 0;
  int stack_depths = 0;              // stack instances (one depth counter each)
  bool nested = false;               // a frame inside another frame's body
  int ta_slots = 0;
  int64_t inst_bound = 0;            // upper bound of heavy instances per run
  int64_t tile_bound = 0;            // max tiles of one instance
  std::vector<BufPlan> bufs;
  std::vector<ChanPlan> chans;
  std::vector<SwapPlan> swaps;
  std::vector<cfdev::DCtx> ctxs;     // [0] = loop level (unused entry)
  int structured_frames = 0;
  int n_waves = 0;
  int n_batches = 0;
  int64_t stack_resident_bytes = 0, stack_swapped_bytes = 0;
  int64_t chan_bytes = 0;
  std::map<std::string, FeedInfo> feeds;
  std::vector<FetchInfo> fetches;
  std::string describe;
  std::string listing;   // body programs, one node per line (debug hook)
};

struct CompileOpts {
  int32_t precision = CF_F32;
  int32_t parallel_iterations = 0;
  int64_t max_iterations = 0;
  int64_t stack_budget_bytes = -1;   // -1: never swap
  int64_t swap_min_bytes = 4096;
  bool swap_smallest_first = false;
};

HostProgram compile(const Graph& g, const CompileOpts& o, const std::vector<TRef>& fetches);

}  // namespace cf
