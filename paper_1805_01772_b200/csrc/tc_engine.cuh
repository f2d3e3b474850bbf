// tcgen05 GEMM tile engine: one 128 x BN output tile per call, warp-specialized inside a
// 256-thread CTA (warp 0 lane 0 = TMA producer, warp 1 lane 0 = MMA issuer, all 8 warps =
// epilogue readers of TMEM). A 4-stage smem ring (full/empty mbarriers) pipelines TMA and MMA
// across the K loop; running k-block counters keep barrier phases consistent across tiles.
#pragma once
#include <cuda.h>

#include "tc.cuh"

namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kStages = 4;
constexpr int kStageA = BM * BK * 2;      // 16 KiB
constexpr int kStageBmax = 256 * BK * 2;  // 32 KiB
constexpr int kSmemTC = kStages * (kStageA + kStageBmax) + 1024 /*align*/ + 256 /*barriers*/;
// 256-row mode (two 128 x 256 accumulators sharing each B stage): 3 stages of 64 KiB in the
// same shared memory; 1.5x fewer operand bytes per flop than 128-row tiles
constexpr int kStages2 = 3;
constexpr int kStage2A = 2 * kStageA;     // 32 KiB: rows [0,128) then [128,256)
constexpr int kStage2 = kStage2A + kStageBmax;
static_assert(kStages2 * kStage2 <= kStages * (kStageA + kStageBmax), "256-row stages fit");

struct TcShared {
  uint8_t* a[kStages];
  uint8_t* b[kStages];
  uint8_t* a2[kStages2];
  uint8_t* b2[kStages2];
  uint64_t* full;    // [kStages]
  uint64_t* empty;   // [kStages]
  uint64_t* done;    // [1]
  uint32_t* tmem_slot;
  volatile uint32_t* kb_issued;   // running k-block counter of the last MMA issued (hook pacing)
  uint64_t* full2;   // [kStages2]
  uint64_t* empty2;  // [kStages2]
};

// carve the dynamic smem buffer (1024-aligned for SWIZZLE_128B)
__device__ inline TcShared tc_carve(uint8_t* dyn) {
  TcShared s;
  uintptr_t base = ((uintptr_t)dyn + 1023) & ~(uintptr_t)1023;
  uint8_t* p = (uint8_t*)base;
  for (int i = 0; i < kStages; ++i) {
    s.a[i] = p;
    p += kStageA;
  }
  for (int i = 0; i < kStages; ++i) {
    s.b[i] = p;
    p += kStageBmax;
  }
  s.full = (uint64_t*)p;
  s.empty = s.full + kStages;
  s.done = s.empty + kStages;
  s.full2 = s.done + 1;
  s.empty2 = s.full2 + kStages2;
  s.tmem_slot = (uint32_t*)(s.empty2 + kStages2);
  s.kb_issued = (volatile uint32_t*)(s.tmem_slot + 1);
  for (int i = 0; i < kStages2; ++i) {
    s.a2[i] = (uint8_t*)base + i * kStage2;
    s.b2[i] = s.a2[i] + kStage2A;
  }
  return s;
}

// one-time per CTA: barrier init (thread 0) + TMEM allocation (warp 2); all threads sync
__device__ inline void tc_setup(TcShared& s) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1);
    }
    for (int i = 0; i < kStages2; ++i) {
      mbar_init(&s.full2[i], 1);
      mbar_init(&s.empty2[i], 1);
    }
    mbar_init(s.done, 1);
    *s.kb_issued = 0;
    fence_barrier_init();
  }
  if (threadIdx.x / 32 == 2) tmem_alloc<512>(s.tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
}
__device__ inline void tc_teardown(TcShared& s) {
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x / 32 == 2) tmem_dealloc<512>(*s.tmem_slot);
}

// box load request: which map, coordinates, smem byte offset within the stage buffer
struct Box {
  const CUtensorMap* map;
  int c0, c1, c2;
  int off;
  int keep = 0;   // 1: L2 evict-last hint (operands re-read across tiles, e.g. the weights)
};
__device__ __forceinline__ void box_load(uint8_t* stage, const Box& b, uint64_t* bar) {
  if (b.keep) tma_load_3d_hint(stage + b.off, b.map, bar, b.c0, b.c1, b.c2, kL2EvictLast);
  else tma_load_3d(stage + b.off, b.map, bar, b.c0, b.c1, b.c2);
}

// Operand plan callbacks: fill up to 4 boxes for operand A / B of k-block kb; return count.
// Run the K loop of one tile. `cnt` is the CTA-wide running k-block counter (same value in
// the producer and MMA threads), `tiles` the running tile counter (epilogue done-barrier
// phase). After return, all threads may read the accumulator with tmem_ld16.
struct NoHook {
  __device__ void operator()() const {}
};
// run the hook once the MMA issuer is within 3 k-blocks of the end of the tile's mainloop
// (end = the running k-block counter after the tile): late enough that a tile claimed there
// does not wait long behind this one, early enough to hide the claim's round trips
// A/B knobs (cf_debug_set_knob): [0] hook lead in k-blocks (0 = the default 8). A late hook
// delays its warp's share of the epilogue (every warp waits for it at the staging barrier):
// measured on cfg3 with lead 3 the forward epilogue's barrier wait was 3.1 us, with 16 0.6 us
__device__ int kKnobs[8];
template <class Hook>
__device__ __forceinline__ void hook_paced(TcShared& s, uint32_t end, Hook& hook) {
  const int lead = kKnobs[0] > 0 ? kKnobs[0] : 8;
  while ((int)(end - *s.kb_issued) > lead) __nanosleep(256);
  hook();
}
// hook: run by thread 64 (an epilogue thread, idle during the mainloop) before it waits for the
// accumulator; the worker claims its next tile there (runtime.cu worker_loop)
template <class PlanA, class PlanB, class Hook = NoHook>
__device__ inline void tc_tile(TcShared& s, int nk, int bn, int a_mn, int b_mn, uint32_t& cnt,
                               uint32_t& tiles, PlanA plan_a, PlanB plan_b, Hook hook = Hook()) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t stage_b = (uint32_t)bn * BK * 2;
  // Role warps: lane 0 works, lanes 1-31 park at __syncwarp (NOT in a suspending
  // mbarrier.try_wait, which would stall the working lane of the same warp).
  if (warp == 0) {
    if (lane == 0) {
    uint32_t c = cnt;
    for (int kb = 0; kb < nk; ++kb, ++c) {
      const int st = c % kStages;
      const uint32_t round = c / kStages;
      mbar_wait(&s.empty[st], (round & 1) ^ 1);
      mbar_arrive_expect_tx(&s.full[st], kStageA + stage_b);
      Box bx[4];
      int na = plan_a(kb, bx);
      for (int i = 0; i < na; ++i) box_load(s.a[st], bx[i], &s.full[st]);
      int nb = plan_b(kb, bx);
      for (int i = 0; i < nb; ++i) box_load(s.b[st], bx[i], &s.full[st]);
    }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
    const uint32_t idesc = idesc_bf16(BM, bn, a_mn, b_mn);
    const uint32_t tmem = *s.tmem_slot;
    uint32_t c = cnt;
    for (int kb = 0; kb < nk; ++kb, ++c) {
      const int st = c % kStages;
      const uint32_t round = c / kStages;
      mbar_wait(&s.full[st], round & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(s.a[st]), sb = smem_u32(s.b[st]);
#pragma unroll
      for (int k = 0; k < BK / 16; ++k) {
        uint64_t da = a_mn ? sdesc_sw128(sa + k * 2048, 8192, 1024) : sdesc_sw128(sa + k * 32, 16, 1024);
        uint64_t db = b_mn ? sdesc_sw128(sb + k * 2048, 8192, 1024) : sdesc_sw128(sb + k * 32, 16, 1024);
        mma_bf16(tmem, da, db, idesc, (kb | k) != 0);
      }
      mma_commit(&s.empty[st]);   // frees the stage when these MMAs have read it
      *s.kb_issued = c + 1;
    }
    mma_commit(s.done);           // accumulator complete
    }
    __syncwarp();
  }
  if (threadIdx.x == 64) hook_paced(s, cnt + nk, hook);
  cnt += nk;
  // everyone waits for the accumulator
  mbar_wait(s.done, tiles & 1);
  tiles++;
  tc_fence_after();
}

// 256-row tile: rows [0,128) accumulate in TMEM columns [0,bn), rows [128,256) in [256,256+bn);
// both MMAs of a k16 step read the same B stage (bn = 256 or 128 columns). Plans fill A boxes at offsets within the
// 32 KiB A region (rows 128.. at +16 KiB) and B boxes as in tc_tile. Own barriers and k-block
// counter (cnt2); the done barrier / tile counter are shared with tc_tile.
template <class PlanA, class PlanB, class Hook = NoHook>
__device__ inline void tc_tile2(TcShared& s, int nk, int a_mn, int b_mn, uint32_t& cnt2,
                                uint32_t& tiles, PlanA plan_a, PlanB plan_b, int bn = 256,
                                int prefetch_ahead = 0, Hook hook = Hook()) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    if (lane == 0) {
      uint32_t c = cnt2;
      for (int kb = 0; kb < nk; ++kb, ++c) {
        const int st = c % kStages2;
        const uint32_t round = c / kStages2;
        mbar_wait(&s.empty2[st], (round & 1) ^ 1);
        mbar_arrive_expect_tx(&s.full2[st], kStage2A + (uint32_t)bn * BK * 2);
        Box bx[8];
        int na = plan_a(kb, bx);
        for (int i = 0; i < na; ++i) box_load(s.a2[st], bx[i], &s.full2[st]);
        int nb = plan_b(kb, bx);
        for (int i = 0; i < nb; ++i) box_load(s.b2[st], bx[i], &s.full2[st]);
        if (prefetch_ahead > 0) {   // the same boxes a few k-blocks ahead, into L2 only
          const int kp = kb == 0 ? 1 : kb + prefetch_ahead;
          for (int q = kp; q <= kb + prefetch_ahead && q < nk; ++q) {
            const int n1 = plan_a(q, bx);
            for (int i = 0; i < n1; ++i) tma_prefetch_l2_3d(bx[i].map, bx[i].c0, bx[i].c1, bx[i].c2);
            const int n2 = plan_b(q, bx);
            for (int i = 0; i < n2; ++i) tma_prefetch_l2_3d(bx[i].map, bx[i].c0, bx[i].c1, bx[i].c2);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(BM, bn, a_mn, b_mn);
      const uint32_t tmem = *s.tmem_slot;
      uint32_t c = cnt2;
      for (int kb = 0; kb < nk; ++kb, ++c) {
        const int st = c % kStages2;
        const uint32_t round = c / kStages2;
        mbar_wait(&s.full2[st], round & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(s.a2[st]), sb = smem_u32(s.b2[st]);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint32_t ko = a_mn ? k * 2048 : k * 32;
          uint64_t da0 = a_mn ? sdesc_sw128(sa + ko, 8192, 1024) : sdesc_sw128(sa + ko, 16, 1024);
          uint64_t da1 = a_mn ? sdesc_sw128(sa + kStageA + ko, 8192, 1024)
                              : sdesc_sw128(sa + kStageA + ko, 16, 1024);
          uint64_t db = b_mn ? sdesc_sw128(sb + k * 2048, 8192, 1024) : sdesc_sw128(sb + k * 32, 16, 1024);
          mma_bf16(tmem, da0, db, idesc, (kb | k) != 0);
          mma_bf16(tmem + 256, da1, db, idesc, (kb | k) != 0);
        }
        mma_commit(&s.empty2[st]);
        *s.kb_issued = c + 1;
      }
      mma_commit(s.done);
    }
    __syncwarp();
  }
  if (threadIdx.x == 64) hook_paced(s, cnt2 + nk, hook);
  cnt2 += nk;
  mbar_wait(s.done, tiles & 1);
  tiles++;
  tc_fence_after();
}

// accumulator element access for the epilogue: warp w reads TMEM lanes 32*(w%4)..+31 (tile
// rows), columns [col0, col0+16)
__device__ inline void tc_acc16(TcShared& s, int col0, float* v) {
  const int warp = threadIdx.x / 32;
  const uint32_t taddr = *s.tmem_slot + ((uint32_t)(32 * (warp % 4)) << 16) + (uint32_t)col0;
  tmem_ld16(taddr, v);
}

// end of tile: all TMEM reads done before the next tile's MMAs overwrite the accumulator
__device__ inline void tc_tile_end() {
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
}

}  // namespace tc
