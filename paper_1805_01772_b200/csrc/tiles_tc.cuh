// bf16 tensor-core tiles of the LSTM cell (forward and backward) for the persistent worker.
//
// Forward (reading R9): Z = [x_t, h_{t-1}] W^T + b as ONE tcgen05 GEMM per 128-row x 256-col
// tile, where the 256 columns are the four gates (i, f, g, o) of 64 hidden units (W rows
// permuted once per run by HK_PREP_WP). Every TMEM lane (= batch row) therefore holds all four
// gates of its units and the sigma / tanh / cell-update / length-mask epilogue is
// thread-local; it writes h (bf16), c (fp32), out (bf16) and the saved gates (bf16, the
// StackPush of PAPER.md:1046-1066 landing directly in its arena slot).
//
// Backward: an elementwise tile computes dz (pre-activation gate grads, bf16) and dc; then
//   d[x,h] = dz W     : tcgen05, A = dz (K-major), B = W^T (K-major, HK_PREP_WT)
//   dW (+)= dz^T [x,h]: tcgen05 with MN-major A (dz) and B (x, h) straight from the saved
//                        activations -- no transposed copies; fp32 read-modify-write into the
//                        fused accumulator ("sum of the gradients ... at
//                        each iteration"); db from per-row-tile partials in a fixed order.
#pragma once
#include <cuda_bf16.h>

#include "program.h"
#include "tc_engine.cuh"

namespace cfdev {

// debug flags for the tile code (cf_debug_set_flags; this header belongs to runtime.cu only)
__device__ int kDbgFlagsTC = 0;
// debug flag bit 22: per-kind tile phase clocks read by cf_debug_tile_phases. Slot k*4: tiles,
// +1 cycles entry -> mainloop issue, +2 mainloop (until the accumulator is complete), +3 epilogue
// (k: 0 forward, 1 d[x,h], 2 dW, 3 backward EW)
__device__ unsigned long long g_tile_phase[20];   // 16..19: forward epilogue sub-phases
__device__ __forceinline__ long long phase_now() {
  return (kDbgFlagsTC & (1 << 22)) && threadIdx.x == 0 ? clock64() : 0;
}
__device__ __forceinline__ void phase_add(int k, long long t0, long long t1) {
  if (t0 == 0) return;
  const long long t2 = clock64();
  atomicAdd(&g_tile_phase[4 * k + 0], 1ULL);
  atomicAdd(&g_tile_phase[4 * k + 1], (unsigned long long)(t1 - t0));
  atomicAdd(&g_tile_phase[4 * k + 2], (unsigned long long)(t2 - t1));
}
__device__ __forceinline__ void phase_epi(int k, long long t2) {
  if (t2 == 0) return;
  atomicAdd(&g_tile_phase[4 * k + 3], (unsigned long long)(clock64() - t2));
}

__device__ __forceinline__ float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float ldf(const void* p, int dt, int64_t i) {
  return dt == D_BF16 ? __bfloat162float(((const __nv_bfloat16*)p)[i]) : ((const float*)p)[i];
}
__device__ __forceinline__ void stf(void* p, int dt, int64_t i, float v) {
  if (dt == D_BF16) ((__nv_bfloat16*)p)[i] = __float2bfloat16(v);
  else ((float*)p)[i] = v;
}
__device__ __forceinline__ float sigmoidf_(float x) { return 1.0f / (1.0f + __expf(-x)); }
__device__ __forceinline__ float tanhf_(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct bf16x8 {
  __nv_bfloat162 v[4];
};
__device__ __forceinline__ void store_bf16x16(__nv_bfloat16* dst, const float* v) {
  bf16x8 a, b;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    a.v[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    b.v[i] = __floats2bfloat162_rn(v[8 + 2 * i], v[8 + 2 * i + 1]);
  }
  ((uint4*)dst)[0] = *(uint4*)&a;
  ((uint4*)dst)[1] = *(uint4*)&b;
}
__device__ __forceinline__ void load_bf16x16(const __nv_bfloat16* src, float* v) {
  uint4 ra = ((const uint4*)src)[0], rb = ((const uint4*)src)[1];
  const __nv_bfloat162* a = (const __nv_bfloat162*)&ra;
  const __nv_bfloat162* b = (const __nv_bfloat162*)&rb;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 x = __bfloat1622float2(a[i]), y = __bfloat1622float2(b[i]);
    v[2 * i] = x.x;
    v[2 * i + 1] = x.y;
    v[8 + 2 * i] = y.x;
    v[8 + 2 * i + 1] = y.y;
  }
}

// ---------------------------------------------------------------- weight preparation
// Wp[n][k] = bf16(W[src(n)][k]); n = j*256 + g*64 + u' -> src = g*H + j*64 + u'
__device__ void tile_prep_wp(const Inst& I, int tile) {
  const int64_t H = I.n, KT = I.k;
  const float* W = (const float*)I.p[0];
  __nv_bfloat16* Wp = (__nv_bfloat16*)I.p[13];
  const int rows_per_tile = 16;
  for (int rr = 0; rr < rows_per_tile; ++rr) {
    int64_t n = (int64_t)tile * rows_per_tile + rr;
    if (n >= 4 * H) break;
    int64_t j = n / 256, r = n % 256, g = r / 64, u = j * 64 + r % 64;
    const float* src = W + (g * H + u) * KT;
    __nv_bfloat16* dst = Wp + n * KT;
    for (int64_t k = threadIdx.x * 2; k < KT; k += 512)
      *(__nv_bfloat162*)(dst + k) = __floats2bfloat162_rn(src[k], src[k + 1]);
  }
}
// WT[n][g] = bf16(W[g][n]); W: [G = 4H][KT]; tile = 64 (n) x 128 (g)
__device__ void tile_prep_wt(const Inst& I, int tile, float* sm) {
  const int64_t G = 4 * I.n, KT = I.k;
  const float* W = (const float*)I.p[0];
  __nv_bfloat16* WT = (__nv_bfloat16*)I.p[13];
  const int64_t tg = G / 128;
  const int64_t n0 = (tile / tg) * 64, g0 = (tile % tg) * 128;
  float* t = sm;   // [128][65]
  for (int idx = threadIdx.x; idx < 128 * 64; idx += 256) {
    int gg = idx / 64, nn = idx % 64;
    t[gg * 65 + nn] = W[(g0 + gg) * KT + n0 + nn];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < 64 * 128; idx += 256) {
    int nn = idx / 128, gg = idx % 128;
    WT[(n0 + nn) * G + g0 + gg] = __float2bfloat16(t[gg * 65 + nn]);
  }
  __syncthreads();
}

// ---------------------------------------------------------------- forward
// p: 0 x-map, 1 h-map, 2 c_prev(f32), 3 Wp-map, 4 bias(f32), 5 lens(i64), 6 h_prev(bf16),
//    8 h_next(bf16), 9 c_next(f32), 10 out(bf16), 11 gates(bf16, tile-interleaved)
// s: 0 t, 1 forget bias bits, 2 x slot, 3 h slot
//
// Epilogue latency: the tile's bias slice goes to shared memory and each thread's first c_prev
// vector and length are loaded BEFORE the mainloop's accumulator wait; inside the epilogue the
// next cell group's c_prev is in flight while the current one computes, and the four gates'
// TMEM loads share one wait. sigma(x) = 0.5 tanh(x / 2) + 0.5 (one MUFU op instead of ex2 + a
// division).
__device__ __forceinline__ float sigm_tanh(float x) { return fmaf(0.5f, tanhf_(0.5f * x), 0.5f); }
// staging of the forward epilogue in the tile engine's stage buffers (free once the mainloop
// completed): gates rows of 512 B and h rows of 128 B, each padded by 16 B (a quarter warp's
// 16-byte stores to 8 consecutive rows hit distinct banks), then one live flag per row
constexpr int kFwdGRow = 512 + 16, kFwdHRow = 128 + 16;
constexpr int kFwdHOff = 256 * kFwdGRow, kFwdLOff = kFwdHOff + 256 * kFwdHRow;
static_assert(kFwdLOff + 256 <= tc::kStages * (tc::kStageA + tc::kStageBmax), "forward staging fits");
template <class Hook>
__device__ void tile_lstm_fwd_tc(const Inst& I, int tile, tc::TcShared& ts, uint32_t& cnt,
                                 uint32_t& cnt2, uint32_t& ntile, float* sm, Hook hook) {
  const int B = (int)I.m, In = (int)I.k, H = (int)I.n;
  const int nkx = In / 64, nk = (In + H) / 64;
  const int tn = H / 64;
  const bool m2 = I.sub & 2;   // 256-row tile (two accumulators)
  // sub bit 2: the x-projection Zx = x Wx^T was computed ahead (HK_LSTM_XPROJ_TC, p[7], fp32,
  // same gate-interleaved columns): only the recurrent k-blocks run here, the epilogue adds Zx
  const bool xproj = I.sub & 4;
  const float* zx = (const float*)I.p[7];
  const int kb0 = xproj ? nkx : 0;
  const int mt = tile / tn, nt = tile % tn;
  const int m0 = mt * (m2 ? 2 * tc::BM : tc::BM);
  const CUtensorMap* mx = (const CUtensorMap*)I.p[0];
  const CUtensorMap* mh = (const CUtensorMap*)I.p[1];
  const CUtensorMap* mw = (const CUtensorMap*)I.p[3];
  const int sx = (int)I.s[2], sh = (int)I.s[3];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const bool masked = I.sub & 1;
  const int64_t t = I.s[0];
  const float fb = __int_as_float((int)I.s[1]);
  const float* bias = (const float*)I.p[4];
  const float* c_prev = (const float*)I.p[2];
  const __nv_bfloat16* h_prev = (const __nv_bfloat16*)I.p[6];
  const int64_t* lens = (const int64_t*)I.p[5];
  __nv_bfloat16* h_next = (__nv_bfloat16*)I.p[8];
  float* c_next = (float*)I.p[9];
  __nv_bfloat16* out = (__nv_bfloat16*)I.p[10];
  __nv_bfloat16* gates = (__nv_bfloat16*)I.p[11];
  const int nh = m2 ? 2 : 1;
  const long long ph0 = phase_now();
  unsigned long long gt0 = 0;   // wall-clock ns beside the SM cycles (the clock under load)
  if (ph0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
  // ---- before the mainloop: bias slice -> smem (forget bias folded in), first c_prev, lengths
  {
    const int g = threadIdx.x / 64, u = threadIdx.x % 64;   // 256 threads = 4 gates x 64 units
    sm[threadIdx.x] = bias[g * H + nt * 64 + u] + (g == 1 ? fb : 0.f);
  }
  const int cbase = (warp / 4) * 32;   // this warp's 32 units of the tile's 64
  auto row_of = [&](int half) { return m0 + 128 * half + 32 * (warp % 4) + lane; };
  auto cp_ptr = [&](int it) {   // iteration it = half * 2 + j: 16 units starting at cbase + 16 j
    const int r = row_of(it >> 1);
    return c_prev + (int64_t)(r < B ? r : 0) * H + nt * 64 + cbase + 16 * (it & 1);
  };
  float4 cpb[2][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) cpb[0][q] = ((const float4*)cp_ptr(0))[q];
  bool live_h[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = row_of(h);
    live_h[h] = h < nh && r < B && (!masked || t < lens[r]);
  }
  // a tile whose rows have all finished (t >= len for every row, "we skip
  // the computation"): no GEMM; every row copies its state through and emits zeros (R10)
  if (__syncthreads_or(live_h[0] || live_h[1]) == 0) {
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      if (it >= 2 * nh) break;
      const int r = row_of(it >> 1);
      if (r >= B) continue;
      const int64_t o = (int64_t)r * H + nt * 64 + cbase + 16 * (it & 1);
      float v[16];
      load_bf16x16(h_prev + o, v);
      store_bf16x16(h_next + o, v);
      float z[16] = {};
      store_bf16x16(out + o, z);
#pragma unroll
      for (int q = 0; q < 4; ++q) ((float4*)(c_next + o))[q] = ((const float4*)(c_prev + o))[q];
    }
    return;
  }
  auto plan_a = [&](int kb, tc::Box* b) {
    kb += kb0;
    for (int hh = 0; hh < (m2 ? 2 : 1); ++hh) {
      if (kb < nkx) b[hh] = {mx, kb * 64, m0 + 128 * hh, sx, hh * tc::kStageA};
      else b[hh] = {mh, (kb - nkx) * 64, m0 + 128 * hh, sh, hh * tc::kStageA};
    }
    return m2 ? 2 : 1;
  };
  const int keep_w = !(kDbgFlagsTC & 32);   // A/B: debug flag bit 5 drops the L2 hint
  auto plan_b = [&](int kb, tc::Box* b) {
    b[0] = {mw, (kb + kb0) * 64, nt * 256, 0, 0, keep_w};
    return 1;
  };
  // debug flags bits 16-19: L2 prefetch distance in k-blocks (A/B; 0 = the default 4, 15 = off)
  const int pfd = (kDbgFlagsTC >> 16) & 15;
  const int ahead = pfd == 15 ? 0 : pfd ? pfd : 4;
  const long long ph1 = ph0 ? clock64() : 0;
  if (m2) tc::tc_tile2(ts, nk - kb0, 0, 0, cnt2, ntile, plan_a, plan_b, 256, ahead, hook);
  else tc::tc_tile(ts, nk - kb0, 256, 0, 0, cnt, ntile, plan_a, plan_b, hook);
  phase_add(0, ph0, ph1);
  const long long ph2 = ph0 ? clock64() : 0;
  // ---- fused epilogue: 2 (or 4) groups of 16 units x 4 gates per thread. The gates and h are
  // staged in the (now idle) pipeline stage buffers and written out coalesced (debug flag bit
  // 21: direct per-row stores, A/B)
  const bool staged = !(kDbgFlagsTC & (1 << 21));
  uint8_t* stg = ts.a[0];
  const int nit = 2 * nh;
  // fully unrolled: the double-buffered c_prev registers are indexed by constants (a runtime
  // index would put them in local memory)
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    if (it >= nit) break;
    const int half = it >> 1, cu = cbase + 16 * (it & 1);
    const int r = row_of(half);
    if (it + 1 < nit) {   // next group's c_prev in flight while this one computes
#pragma unroll
      for (int q = 0; q < 4; ++q) cpb[(it + 1) & 1][q] = ((const float4*)cp_ptr(it + 1))[q];
    }
    uint32_t zr[4][16];
    const uint32_t ta = *ts.tmem_slot + ((uint32_t)(32 * (warp % 4)) << 16) + (uint32_t)(256 * half + cu);
#pragma unroll
    for (int g = 0; g < 4; ++g) tc::tmem_ld16_nowait(ta + 64 * g, zr[g]);
    float4 zxv[4][4];
    if (xproj) {   // the precomputed x-projection of this row's 16 units x 4 gates
      const float* zrow = zx + (int64_t)(r < B ? r : 0) * 4 * H + nt * 256 + cu;
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int q = 0; q < 4; ++q) zxv[g][q] = ((const float4*)(zrow + g * 64))[q];
    }
    tc::tmem_wait_ld();
    if (r >= B || (kDbgFlagsTC & (1 << 20))) continue;   // bit 20: no epilogue (timing only)
    if (xproj) {
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          zr[g][4 * q + 0] = __float_as_uint(__uint_as_float(zr[g][4 * q + 0]) + zxv[g][q].x);
          zr[g][4 * q + 1] = __float_as_uint(__uint_as_float(zr[g][4 * q + 1]) + zxv[g][q].y);
          zr[g][4 * q + 2] = __float_as_uint(__uint_as_float(zr[g][4 * q + 2]) + zxv[g][q].z);
          zr[g][4 * q + 3] = __float_as_uint(__uint_as_float(zr[g][4 * q + 3]) + zxv[g][q].w);
        }
    }
    const int u0 = nt * 64 + cu;
    const int64_t o = (int64_t)r * H + u0;
    float cp[16], hn[16], cn[16], zi[16], zf[16], zg[16], zo[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) *(float4*)&cp[4 * q] = cpb[it & 1][q];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      zi[i] = sigm_tanh(__uint_as_float(zr[0][i]) + sm[0 * 64 + cu + i]);
      zf[i] = sigm_tanh(__uint_as_float(zr[1][i]) + sm[1 * 64 + cu + i]);
      zg[i] = tanhf_(__uint_as_float(zr[2][i]) + sm[2 * 64 + cu + i]);
      zo[i] = sigm_tanh(__uint_as_float(zr[3][i]) + sm[3 * 64 + cu + i]);
      cn[i] = zf[i] * cp[i] + zi[i] * zg[i];
      hn[i] = zo[i] * tanhf_(cn[i]);
    }
    if (staged) {
      // gates and h into shared memory (padded rows: conflict-free 16-byte stores), c direct
      const int rl = 128 * half + 32 * (warp % 4) + lane;
      uint8_t* g0 = stg + rl * kFwdGRow + cu * 2;
      store_bf16x16((__nv_bfloat16*)(g0 + 0), zi);
      store_bf16x16((__nv_bfloat16*)(g0 + 128), zf);
      store_bf16x16((__nv_bfloat16*)(g0 + 256), zg);
      store_bf16x16((__nv_bfloat16*)(g0 + 384), zo);
      __nv_bfloat16* h0 = (__nv_bfloat16*)(stg + kFwdHOff + rl * kFwdHRow + cu * 2);
      if (live_h[half]) {
        store_bf16x16(h0, hn);
#pragma unroll
        for (int q = 0; q < 4; ++q) ((float4*)(c_next + o))[q] = *(float4*)&cn[4 * q];
      } else {
        // finished row (reading R10): state copied through, output zero (at the copy-out)
        float hp[16];
        load_bf16x16(h_prev + o, hp);
        store_bf16x16(h0, hp);
#pragma unroll
        for (int q = 0; q < 4; ++q) ((float4*)(c_next + o))[q] = *(float4*)&cp[4 * q];
      }
      if ((it & 1) == 0) stg[kFwdLOff + rl] = live_h[half] ? 1 : 0;
      continue;
    }
    __nv_bfloat16* gr = gates + (int64_t)r * 4 * H + nt * 256 + cu;
    store_bf16x16(gr + 0, zi);
    store_bf16x16(gr + 64, zf);
    store_bf16x16(gr + 128, zg);
    store_bf16x16(gr + 192, zo);
    if (live_h[half]) {
      store_bf16x16(h_next + o, hn);
      store_bf16x16(out + o, hn);
#pragma unroll
      for (int q = 0; q < 4; ++q) ((float4*)(c_next + o))[q] = *(float4*)&cn[4 * q];
    } else {
      // finished row (reading R10): state copied through, output zero
      float hp[16];
      load_bf16x16(h_prev + o, hp);
      store_bf16x16(h_next + o, hp);
      float z[16] = {};
      store_bf16x16(out + o, z);
#pragma unroll
      for (int q = 0; q < 4; ++q) ((float4*)(c_next + o))[q] = *(float4*)&cp[4 * q];
    }
  }
  const long long ph3 = ph0 ? clock64() : 0;
  if (staged && !(kDbgFlagsTC & (1 << 20))) {
    // coalesced copy-out: a warp writes a whole 512-byte gates row (or four 128-byte h / out
    // rows) per instruction instead of 32 row fragments
    __syncthreads();
    if (ph0) {
      const long long ph4 = clock64();
      atomicAdd(&g_tile_phase[16], (unsigned long long)(ph3 - ph2));   // TMEM + math + staging
      atomicAdd(&g_tile_phase[17], (unsigned long long)(ph4 - ph3));   // barrier (warp imbalance)
    }
    const int nrows = min(128 * nh, B - m0);
    for (int rr = warp; rr < nrows; rr += 8) {
      const uint4 v = *(const uint4*)(stg + rr * kFwdGRow + lane * 16);
      *(uint4*)((uint8_t*)(gates + (int64_t)(m0 + rr) * 4 * H + nt * 256) + lane * 16) = v;
    }
    for (int q = threadIdx.x; q < nrows * 8; q += 256) {
      const int rr = q >> 3, ch = q & 7;
      const uint4 v = *(const uint4*)(stg + kFwdHOff + rr * kFwdHRow + ch * 16);
      const int64_t ob = ((int64_t)(m0 + rr) * H + nt * 64) * 2 + ch * 16;
      *(uint4*)((uint8_t*)h_next + ob) = v;
      *(uint4*)((uint8_t*)out + ob) = stg[kFwdLOff + rr] ? v : make_uint4(0, 0, 0, 0);
    }
    // the next tile's TMA (async proxy) overwrites these stage buffers
    tc::fence_proxy_async_smem();
  }
  tc::tc_tile_end();
  phase_epi(0, ph2);
  if (ph0) {
    unsigned long long gt1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
    atomicAdd(&g_tile_phase[18], gt1 - gt0);
    atomicAdd(&g_tile_phase[19], (unsigned long long)(clock64() - ph0));
  }
}

// ---------------------------------------------------------------- forward x-projection
// Zx = x Wx^T for one (row tile, 256-column gate-interleaved tile): the input part of the gate
// pre-activations does not depend on h_{t-1}, so it runs as its own instance as soon as x_t is
// ready (the layer below's step t), off the recurrence's critical chain; the cell instance
// then runs only the recurrent k-blocks (sub bit 2). fp32 out through the idle stage buffers.
// p: 0 x-map, 3 Wp-map, 7 Zx (f32 [B][4H]); s: 2 x slot; sub bit 1: 256-row tile
template <class Hook>
__device__ void tile_lstm_xproj_tc(const Inst& I, int tile, tc::TcShared& ts, uint32_t& cnt,
                                   uint32_t& cnt2, uint32_t& ntile, Hook hook) {
  const int B = (int)I.m, In = (int)I.k, H = (int)I.n;
  const int nkx = In / 64, tn = H / 64;
  const bool m2 = I.sub & 2;
  const int mt = tile / tn, nt = tile % tn;
  const int m0 = mt * (m2 ? 2 * tc::BM : tc::BM);
  const CUtensorMap* mx = (const CUtensorMap*)I.p[0];
  const CUtensorMap* mw = (const CUtensorMap*)I.p[3];
  float* zx = (float*)I.p[7];
  const int sx = (int)I.s[2];
  auto plan_a = [&](int kb, tc::Box* b) {
    b[0] = {mx, kb * 64, m0, sx, 0};
    if (m2) b[1] = {mx, kb * 64, m0 + 128, sx, tc::kStageA};
    return m2 ? 2 : 1;
  };
  const int keep_w = !(kDbgFlagsTC & 32);
  auto plan_b = [&](int kb, tc::Box* b) {
    b[0] = {mw, kb * 64, nt * 256, 0, 0, keep_w};
    return 1;
  };
  if (m2) tc::tc_tile2(ts, nkx, 0, 0, cnt2, ntile, plan_a, plan_b, 256, 0, hook);
  else tc::tc_tile(ts, nkx, 256, 0, 0, cnt, ntile, plan_a, plan_b, hook);
  uint8_t* stg = ts.a[0];
  constexpr int kRow = 1024 + 16;   // 256 fp32 + pad
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int half = 0; half < (m2 ? 2 : 1); ++half) {
    const int rl = 32 * (warp % 4) + lane;
    for (int c = (warp / 4) * 128; c < (warp / 4) * 128 + 128; c += 16) {
      float v[16];
      tc::tc_acc16(ts, 256 * half + c, v);
#pragma unroll
      for (int q = 0; q < 4; ++q) *(float4*)(stg + rl * kRow + (c + 4 * q) * 4) = *(float4*)&v[4 * q];
    }
    __syncthreads();
    const int nrows = min(128, B - (m0 + 128 * half));
    for (int q = threadIdx.x; q < nrows * 64; q += 256) {
      const int rr = q >> 6, ch = q & 63;
      *(uint4*)((uint8_t*)(zx + (int64_t)(m0 + 128 * half + rr) * 4 * H + nt * 256) + ch * 16) =
          *(const uint4*)(stg + rr * kRow + ch * 16);
    }
    __syncthreads();
  }
  tc::fence_proxy_async_smem();
  tc::tc_tile_end();
}

// ---------------------------------------------------------------- backward elementwise
// p: 2 c_prev(f32), 4 gates(bf16 interleaved), 5 lens, 6 dh_next(f32), 7 dc_next(f32),
//    8 dout(dt s[4]), 9 dc(f32 out), 10 dz(bf16 out, [B][4H] natural) + partials,
//    14/15 folded AddN terms of dout (f32, optional)
// tile = 128 rows x 64 units; thread: 4 consecutive units (16-byte fp32 / 8-byte bf16 vector
// accesses), rows t/16 + 16i. HBM-bound: every operand is read once, dz / dc written once.
__device__ __forceinline__ float4 ld4f(const float* p) { return *(const float4*)p; }
__device__ __forceinline__ void bf4(const __nv_bfloat16* p, float* o) {
  const uint2 v = *(const uint2*)p;
  const __nv_bfloat162 a = *(const __nv_bfloat162*)&v.x, b = *(const __nv_bfloat162*)&v.y;
  const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
  o[0] = fa.x; o[1] = fa.y; o[2] = fb.x; o[3] = fb.y;
}
// one row's 4 units of the LSTM cell backward (the forward pass's c recomputed from the stored
// gates): dz for the 4 gates, dc to the previous step; a finished row (reading R10) passes
// dc through and has zero dz
__device__ __forceinline__ void ew_cell4(const float* ig, const float* fg, const float* gg,
                                         const float* og, const float* cpa, const float* dna,
                                         const float* dca, const float* dov, bool live,
                                         float (&zf)[4][4], float (&dco)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float cn = fg[k] * cpa[k] + ig[k] * gg[k];
    // tanh of the recomputed cell state with the same one-MUFU approximation the forward
    // epilogue used for h (libm tanhf is ~20 instructions; the EW tile issues ~0.8 IPC)
    const float tc_ = (kDbgFlagsTC & (1 << 23)) ? tanhf(cn) : tanhf_(cn);
    const float dh = dna[k] + dov[k];
    const float dcs = dh * og[k] * (1.0f - tc_ * tc_) + dca[k];
    zf[0][k] = dcs * gg[k] * ig[k] * (1.0f - ig[k]);
    zf[1][k] = dcs * cpa[k] * fg[k] * (1.0f - fg[k]);
    zf[2][k] = dcs * ig[k] * (1.0f - gg[k] * gg[k]);
    zf[3][k] = dh * tc_ * og[k] * (1.0f - og[k]);
    dco[k] = dcs * fg[k];
    if (!live) {
      zf[0][k] = zf[1][k] = zf[2][k] = zf[3][k] = 0.0f;
      dco[k] = dca[k];
    }
  }
}
// dz (bf16, natural [B][4H] layout) and dc stores of one row's 4 units; db sums the bf16-rounded
// dz, exactly what the dW GEMM consumes
__device__ __forceinline__ void ew_store4(__nv_bfloat16* zr, int64_t H, float* dcp,
                                          const float (&zf)[4][4], const float (&dco)[4],
                                          float (&sdb)[4][4]) {
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const __nv_bfloat162 lo = __floats2bfloat162_rn(zf[g][0], zf[g][1]);
    const __nv_bfloat162 hi = __floats2bfloat162_rn(zf[g][2], zf[g][3]);
    sdb[g][0] += __low2float(lo);
    sdb[g][1] += __high2float(lo);
    sdb[g][2] += __low2float(hi);
    sdb[g][3] += __high2float(hi);
    uint2 pk;
    pk.x = *(const uint32_t*)&lo;
    pk.y = *(const uint32_t*)&hi;
    *(uint2*)(zr + (int64_t)g * H) = pk;
  }
  *(float4*)dcp = make_float4(dco[0], dco[1], dco[2], dco[3]);
}
// tile = 128 rows x kEwUnits units (64-unit gate-interleaved slices). Small tiles: the
// instance's latency is on the gradient loop's critical path (EW -> d[x,h] -> next step's EW).
// Operands go through registers, four rows at a time: the loads of four rows first, then their
// math and stores (the stores may alias the loads as far as the compiler knows; row by row,
// every row's loads waited for the previous row's stores: 13.1 -> 11.1 us per tile). Staging
// the operands in shared memory was measured no better: bulk copies issued by one warp (640 of
// 128-512 B per tile) 14.6 us, per-thread cp.async copies of all 8 rows 14.5 us (cfg3; the
// tile's stalls are spread over memory, instruction fetch and issue).
constexpr int kEwUnits = 64;   // 256 measured: 4x fewer tiles, no faster per cell, longer chain
__device__ void tile_lstm_bwd_ew_bf(const Inst& I, int tile, float* sm) {
  const int B = (int)I.m, H = (int)I.n;
  const int tu = (H + kEwUnits - 1) / kEwUnits;
  const int rt = tile / tu, ut0 = (tile % tu) * (kEwUnits / 64);   // first 64-unit slice
  const int nsl = min(kEwUnits / 64, H / 64 - ut0);
  const int ul = (threadIdx.x % 16) * 4;          // unit within a 64-unit slice
  const int rg = threadIdx.x / 16;
  const float* c_prev = (const float*)I.p[2];
  const __nv_bfloat16* gates = (const __nv_bfloat16*)I.p[4];
  const int64_t* lens = (const int64_t*)I.p[5];
  const float* dhn = (const float*)I.p[6];
  const float* dcn = (const float*)I.p[7];
  const void* dout = (const void*)I.p[8];
  const bool dout_bf = (int)I.s[4] == D_BF16;
  const float* add0 = (const float*)I.p[14];
  const float* add1 = (const float*)I.p[15];
  float* dc = (float*)I.p[9];
  __nv_bfloat16* dz = (__nv_bfloat16*)I.p[10];
  float* partial = (float*)(I.p[10] + I.s[5]);
  const bool masked = I.sub & 1;
  const int64_t t = I.s[0];
  const int nrow = min(128, B - rt * 128);
  const long long ph0 = phase_now();
  bool live_r[8];
  bool any = false;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int rr = rg + 16 * i;
    live_r[i] = !masked || (rr < nrow && t < lens[rt * 128 + rr]);
    any |= rr < nrow && live_r[i];
  }
  if (masked && __syncthreads_or(any) == 0) {
    // no live row: dz = 0, dc passes through, the db partials are 0
    for (int sl = 0; sl < nsl; ++sl) {
      const int ut = ut0 + sl;
      const int u = ut * 64 + ul;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rr = rg + 16 * i;
        if (rr >= nrow) continue;
        const int64_t r = (int64_t)rt * 128 + rr, e = r * H + u;
        __nv_bfloat16* zr = dz + r * 4 * H + u;
#pragma unroll
        for (int g = 0; g < 4; ++g) *(uint2*)(zr + (int64_t)g * H) = make_uint2(0u, 0u);
        *(float4*)(dc + e) = ld4f(dcn + e);
      }
      const int g = threadIdx.x / 64, uu = threadIdx.x % 64;
      partial[(int64_t)rt * 4 * H + g * H + ut * 64 + uu] = 0.f;
    }
    return;
  }
  for (int sl = 0; sl < nsl; ++sl) {
    const int ut = ut0 + sl;
    const int u = ut * 64 + ul;
    float sdb[4][4] = {};
    {
      // rows past the batch read row 0 and store nothing
#pragma unroll
      for (int i0 = 0; i0 < 8; i0 += 4) {
        float ga[4][4][4], cpv[4][4], dnv[4][4], dcv4[4][4], dov4[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int rr = rg + 16 * (i0 + j);
          const int r = rt * 128 + (rr < nrow ? rr : 0);
          const int64_t e = (int64_t)r * H + u;
          const __nv_bfloat16* gr = gates + (int64_t)r * 4 * H + ut * 256 + ul;
#pragma unroll
          for (int g = 0; g < 4; ++g) bf4(gr + 64 * g, ga[j][g]);
          const float4 cp = ld4f(c_prev + e), dn = ld4f(dhn + e), dc4 = ld4f(dcn + e);
          float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
          if (add0) a0 = ld4f(add0 + e);   // folded AddN terms
          if (add1) a1 = ld4f(add1 + e);
          if (dout_bf) bf4((const __nv_bfloat16*)dout + e, dov4[j]);
          else *(float4*)dov4[j] = ld4f((const float*)dout + e);
          *(float4*)cpv[j] = cp;
          *(float4*)dcv4[j] = dc4;
          *(float4*)dnv[j] = make_float4(dn.x + a0.x + a1.x, dn.y + a0.y + a1.y, dn.z + a0.z + a1.z,
                                         dn.w + a0.w + a1.w);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = i0 + j;
          const int rr = rg + 16 * i;
          if (rr >= nrow) continue;
          float zf[4][4], dco[4];
          ew_cell4(ga[j][0], ga[j][1], ga[j][2], ga[j][3], cpv[j], dnv[j], dcv4[j], dov4[j],
                   live_r[i], zf, dco);
          const int64_t r = (int64_t)rt * 128 + rr;
          ew_store4(dz + r * 4 * H + u, H, dc + r * H + u, zf, dco, sdb);
        }
      }
    }
    // reduce the 16 row groups of this slice: sm[rg][g][64]
#pragma unroll
    for (int g = 0; g < 4; ++g)
      *(float4*)&sm[(rg * 4 + g) * 64 + ul] = make_float4(sdb[g][0], sdb[g][1], sdb[g][2], sdb[g][3]);
    __syncthreads();
    {
      const int g = threadIdx.x / 64, uu = threadIdx.x % 64;   // 256 threads = 4 gates x 64 units
      float acc = 0.f;
#pragma unroll
      for (int q = 0; q < 16; ++q) acc += sm[(q * 4 + g) * 64 + uu];
      partial[(int64_t)rt * 4 * H + g * H + ut * 64 + uu] = acc;
    }
    __syncthreads();
  }
  phase_add(3, ph0, ph0);
}

// ---------------------------------------------------------------- generic GEMM (MatMul)
// C[M][N] = op(A) op(B) for bf16 operands in the TMA operand registry (the MoE-style experts
// and their gradients, cfg5): 128 x 256 tiles on the tcgen05 engine, fp32 accumulation.
// A stored [M][K] (K-major) or, transposed, [K][M] (MN-major); B stored [K][N] (MN-major) or,
// transposed, [N][K] (K-major). p: 0 A map, 1 B map, 13 C; s: 0 A slot, 1 B slot, 2 C dtype;
// sub: bit 0 ta, bit 1 tb
template <class Hook>
__device__ void tile_matmul_tc(const Inst& I, int tile, tc::TcShared& ts, uint32_t& cnt,
                               uint32_t& ntile, Hook hook) {
  const int M = (int)I.m, N = (int)I.n, K = (int)I.k;
  const bool ta = I.sub & 1, tb = I.sub & 2;
  const int tn = N / 256;
  const int mt = tile / tn, nt = tile % tn;
  const int m0 = mt * tc::BM, n0 = nt * 256;
  const CUtensorMap* ma = (const CUtensorMap*)I.p[0];
  const CUtensorMap* mb = (const CUtensorMap*)I.p[1];
  const int sa = (int)I.s[0], sb = (int)I.s[1];
  auto plan_a = [&](int kb, tc::Box* b) {
    if (!ta) {
      b[0] = {ma, kb * 64, m0, sa, 0};
      return 1;
    }
    for (int j = 0; j < 2; ++j) b[j] = {ma, m0 + 64 * j, kb * 64, sa, j * 8192};
    return 2;
  };
  auto plan_b = [&](int kb, tc::Box* b) {
    if (tb) {
      b[0] = {mb, kb * 64, n0, sb, 0};
      return 1;
    }
    for (int j = 0; j < 4; ++j) b[j] = {mb, n0 + 64 * j, kb * 64, sb, j * 8192};
    return 4;
  };
  tc::tc_tile(ts, K / 64, 256, ta ? 1 : 0, tb ? 0 : 1, cnt, ntile, plan_a, plan_b, hook);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int r = m0 + 32 * (warp % 4) + lane;
  const bool cbf = (int)I.s[2] == D_BF16;
  for (int c = (warp / 4) * 128; c < (warp / 4) * 128 + 128; c += 16) {
    float v[16];
    tc::tc_acc16(ts, c, v);
    if (r >= M) continue;
    const int64_t o = (int64_t)r * N + n0 + c;
    if (cbf) {
      store_bf16x16((__nv_bfloat16*)I.p[13] + o, v);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) ((float4*)((float*)I.p[13] + o))[q] = *(float4*)&v[4 * q];
    }
  }
  tc::tc_tile_end();
}

// ---------------------------------------------------------------- backward d[x,h]
// p: 0 dz-map (KA), 1 WT-map (KB; the KA map of the same buffer is the one before it),
//    5 lens, 6 dh_next(f32), 11 dx(f32), 12 dh(f32); s: 0 t, 2 dz slot
// 256-row tiles (sub bit 1) are 256 rows x kDxhN2 columns. The d[x,h] GEMM sits on the gradient
// loop's critical path (EW -> d[x,h] -> next step's EW); 128-column tiles (twice the tiles, half
// the latency each) were measured 41% less efficient per flop with no net gain.
constexpr int kDxhN2 = 256;
template <class Hook>
__device__ void tile_lstm_dxh_tc(const Inst& I, int tile, tc::TcShared& ts, uint32_t& cnt,
                                 uint32_t& cnt2, uint32_t& ntile, Hook hook) {
  const int B = (int)I.m, In = (int)I.k, H = (int)I.n, KT = In + H;
  const bool m2 = I.sub & 2;
  const int bn = m2 ? kDxhN2 : 256;
  const int tn = KT / bn;
  const int mt = tile / tn, nt = tile % tn;
  const int m0 = mt * (m2 ? 2 * tc::BM : tc::BM);
  const CUtensorMap* mz = (const CUtensorMap*)I.p[0];
  const CUtensorMap* mwt = (const CUtensorMap*)I.p[1] - (bn == 128 ? 1 : 0);   // box rows = bn
  const int sz = (int)I.s[2];
  auto plan_a = [&](int kb, tc::Box* b) {
    b[0] = {mz, kb * 64, m0, sz, 0};
    if (m2) b[1] = {mz, kb * 64, m0 + 128, sz, tc::kStageA};
    return m2 ? 2 : 1;
  };
  const int keep_w = !(kDbgFlagsTC & 32);
  auto plan_b = [&](int kb, tc::Box* b) {
    b[0] = {mwt, kb * 64, nt * bn, 0, 0, keep_w};
    return 1;
  };
  if (I.sub & 1) {
    // finished rows have dz = 0 (the EW tile), so their dx is 0 and their dh is dh_next: a
    // tile with no live row skips the GEMM and writes exactly that
    const int64_t t = I.s[0];
    const int64_t* lens = (const int64_t*)I.p[5];
    const int rows = m2 ? 2 * tc::BM : tc::BM;
    bool any = false;
    for (int rr = threadIdx.x; rr < rows; rr += blockDim.x)
      any |= m0 + rr < B && t < lens[m0 + rr];
    if (__syncthreads_or(any) == 0) {
      const int n0 = nt * bn;
      const float* dhn = (const float*)I.p[6];
      float* dst = n0 < In ? (float*)I.p[11] + n0 : (float*)I.p[12] + (n0 - In);
      const int64_t ld = n0 < In ? In : H;
      const int nr = min(rows, B - m0), nq = bn / 4;
      for (int q = threadIdx.x; q < nr * nq; q += blockDim.x) {
        const int rr = q / nq, c = (q % nq) * 4;
        const int64_t r = m0 + rr;
        *(float4*)(dst + r * ld + c) = n0 < In ? make_float4(0.f, 0.f, 0.f, 0.f)
                                               : *(const float4*)(dhn + r * H + (n0 - In) + c);
      }
      return;
    }
  }
  const long long ph0 = phase_now();
  if (m2) tc::tc_tile2(ts, (4 * H) / 64, 0, 0, cnt2, ntile, plan_a, plan_b, bn, 0, hook);
  else tc::tc_tile(ts, (4 * H) / 64, 256, 0, 0, cnt, ntile, plan_a, plan_b, hook);
  phase_add(1, ph0, ph0);
  const long long ph2 = ph0 ? clock64() : 0;
  if (m2 && bn == 256 && !(kDbgFlagsTC & (1 << 21))) {
    // four passes of 128 rows x 128 columns through two stage buffers; the copy engine writes
    // each 512-byte row (cp.async.bulk) while the next pass is staged (debug flag bit 21: the
    // legacy thread stores, A/B)
    constexpr int kRow = 512 + 16;
    static_assert(2 * 128 * kRow <= tc::kStages * (tc::kStageA + tc::kStageBmax), "d[x,h] staging fits");
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int rl = 32 * (warp % 4) + lane;
    const bool masked = I.sub & 1;
    const int64_t t = I.s[0];
    const int64_t* lens = (const int64_t*)I.p[5];
    const float* dhn = (const float*)I.p[6];
    const int n0 = nt * 256;   // the tile is all dx or all dh columns (In % 256 == 0)
    float* dst0 = n0 < In ? (float*)I.p[11] + n0 : (float*)I.p[12] + (n0 - In);
    const int64_t ld = n0 < In ? In : H;
    for (int pass = 0; pass < 4; ++pass) {
      const int half = pass >> 1, cb = (pass & 1) * 128;
      uint8_t* stg = ts.a[0] + (pass & 1) * 128 * kRow;
      if (pass >= 2) {
        if (threadIdx.x < 128) tc::bulk_wait_read1();
        __syncthreads();
      }
      const int r = m0 + 128 * half + rl;
      const bool dead_row = r < B && masked && !(t < lens[r]);
      const int c0 = (warp / 4) * 64;   // this warp's 64 columns of the pass: four loads, one wait
      uint32_t v[4][16];
      const uint32_t ta = *ts.tmem_slot + ((uint32_t)(32 * (warp % 4)) << 16) + (uint32_t)(256 * half + cb + c0);
#pragma unroll
      for (int j = 0; j < 4; ++j) tc::tmem_ld16_nowait(ta + 16 * j, v[j]);
      tc::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (n0 >= In && dead_row) {   // finished row: dh passes dh_next through (reading R10)
          const int64_t o = (int64_t)r * H + (n0 - In) + cb + c0 + 16 * j;
#pragma unroll
          for (int q = 0; q < 4; ++q) *(float4*)&v[j][4 * q] = ((const float4*)(dhn + o))[q];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *(uint4*)(stg + rl * kRow + (c0 + 16 * j + 4 * q) * 4) = *(uint4*)&v[j][4 * q];
      }
      tc::fence_proxy_async_smem();
      __syncthreads();
      const int rr = m0 + 128 * half + (int)threadIdx.x;
      if (threadIdx.x < 128 && rr < B) {
        tc::bulk_s2g(dst0 + (int64_t)rr * ld + cb, stg + threadIdx.x * kRow, 512);
        tc::bulk_commit();
      }
    }
    if (threadIdx.x < 128) {
      tc::bulk_wait_all();   // dx / dh written before the tile completes
      tc::fence_proxy_async_global();
    }
    tc::tc_tile_end();
    phase_epi(1, ph2);
    return;
  }
  // epilogue: per 128-row half, the accumulator goes through the (idle) stage buffers and out
  // as whole 1 KB rows (debug flag bit 21: direct per-row stores, A/B)
  const bool staged = !(kDbgFlagsTC & (1 << 21)) && bn == 256;
  uint8_t* stg = ts.a[0];
  constexpr int kRow = 1024 + 16;   // 256 fp32 + pad (conflict-free 16-byte stores)
  for (int half = 0; half < (m2 ? 2 : 1); ++half) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int r = m0 + 128 * half + 32 * (warp % 4) + lane;
  const int tcol = 256 * half;
  const bool masked = I.sub & 1;
  const int64_t t = I.s[0];
  const int64_t* lens = (const int64_t*)I.p[5];
  const float* dhn = (const float*)I.p[6];
  float* dx = (float*)I.p[11];
  float* dh = (float*)I.p[12];
  const bool dead_row = r < B && masked && !(t < lens[r]);
  const int cw = bn / 2;   // columns per warp group
  const int rl = 32 * (warp % 4) + lane;
  for (int c = (warp / 4) * cw; c < (warp / 4) * cw + cw; c += 16) {
    float v[16];
    tc::tc_acc16(ts, tcol + c, v);
    if (r >= B) continue;
    const int n = nt * bn + c;
    if (n >= In && dead_row) {
      const int64_t o = (int64_t)r * H + (n - In);
#pragma unroll
      for (int q = 0; q < 4; ++q) *(float4*)&v[4 * q] = ((const float4*)(dhn + o))[q];
    }
    if (staged) {
#pragma unroll
      for (int q = 0; q < 4; ++q) *(float4*)(stg + rl * kRow + (c + 4 * q) * 4) = *(float4*)&v[4 * q];
      continue;
    }
    if (n < In) {
      float* d = dx + (int64_t)r * In + n;
#pragma unroll
      for (int q = 0; q < 4; ++q) ((float4*)d)[q] = *(float4*)&v[4 * q];
    } else {
      const int64_t o = (int64_t)r * H + (n - In);
#pragma unroll
      for (int q = 0; q < 4; ++q) ((float4*)(dh + o))[q] = *(float4*)&v[4 * q];
    }
  }
  if (staged) {
    __syncthreads();
    const int n0 = nt * bn;
    float* dst = n0 < In ? dx + n0 : dh + (n0 - In);
    const int64_t ld = n0 < In ? In : H;
    const int nrows = min(128, B - (m0 + 128 * half));
    for (int q = threadIdx.x; q < nrows * 64; q += 256) {   // 64 x 16 B per row
      const int rr = q >> 6, ch = q & 63;
      *(uint4*)((uint8_t*)(dst + (int64_t)(m0 + 128 * half + rr) * ld) + ch * 16) =
          *(const uint4*)(stg + rr * kRow + ch * 16);
    }
    __syncthreads();
  }
  }
  if (staged) tc::fence_proxy_async_smem();   // the next tile's TMA overwrites the stage buffers
  tc::tc_tile_end();
  phase_epi(1, ph2);
}

// ---------------------------------------------------------------- backward dW / db
// Chunked over up to 8 gradient-loop steps (K = steps x B): the fp32 read-modify-write of the
// accumulator is paid once per chunk. p: 0 dz-map (MN), 3 dW(f32), 4 db(f32), 6 step records
// (6 x i64 per step: dz slot, x-map, x slot, h-map, h slot, db-partials ptr);
// s: 6 flags (bit0 accumulate dW, bit1 accumulate db), 7 number of steps
template <class Hook>
__device__ void tile_lstm_dw_tc(const Inst& I, int tile, tc::TcShared& ts, uint32_t& cnt,
                                uint32_t& cnt2, uint32_t& ntile, Hook hook) {
  const int B = (int)I.m, In = (int)I.k, H = (int)I.n, KT = In + H, G = 4 * H;
  const int tn = KT / 256;
  const int n_dw = (G / (2 * tc::BM)) * tn;   // 256 gate rows per tile
  const int flags = (int)I.s[6];
  const int ns = (int)I.s[7];
  const int64_t* ax = (const int64_t*)I.p[6];
  if (tile >= n_dw) {
    // db tile: 256 gate columns; fixed-order sum over steps and row-tile partials
    const int c = (tile - n_dw) * 256 + threadIdx.x;
    float* db = (float*)I.p[4];
    if (c < G) {
      float s = 0.f;
      for (int q = 0; q < ns; ++q) {
        const float* partial = (const float*)ax[q * 6 + 5];
        for (int rt = 0; rt < (B + 127) / 128; ++rt) s += partial[(int64_t)rt * G + c];
      }
      db[c] = (flags & 2) ? db[c] + s : s;
    }
    return;
  }
  const int mt = tile / tn, nt = tile % tn;
  const int m0 = mt * 2 * tc::BM;
  const CUtensorMap* mz = (const CUtensorMap*)I.p[0];
  const bool xpart = nt * 256 < In;
  const int col0 = xpart ? nt * 256 : nt * 256 - In;
  const int nkb = (B + 63) / 64;
  auto plan_a = [&](int kb, tc::Box* b) {
    const int q = kb / nkb, r = kb % nkb;
    const int sz = (int)ax[q * 6 + 0];
    for (int j = 0; j < 4; ++j) b[j] = {mz, m0 + 64 * j, r * 64, sz, j * 8192};
    return 4;
  };
  auto plan_b = [&](int kb, tc::Box* b) {
    const int q = kb / nkb, r = kb % nkb;
    const CUtensorMap* mb = (const CUtensorMap*)ax[q * 6 + (xpart ? 1 : 3)];
    const int sb = (int)ax[q * 6 + (xpart ? 2 : 4)];
    for (int j = 0; j < 4; ++j) b[j] = {mb, col0 + 64 * j, r * 64, sb, j * 8192};
    return 4;
  };
  const long long ph0 = phase_now();
  tc::tc_tile2(ts, ns * nkb, 1, 1, cnt2, ntile, plan_a, plan_b, 256, 0, hook);
  phase_add(2, ph0, ph0);
  const long long ph2 = ph0 ? clock64() : 0;
  const bool acc = flags & 1;
  if (!(kDbgFlagsTC & (1 << 21))) {
    // four passes of 128 rows x 128 columns: the accumulator goes to the (idle) stage buffers
    // as 512-byte rows and the copy engine adds them into dW in L2 (cp.reduce.async.bulk
    // .add.f32; a plain bulk copy for the chunk that starts the accumulation). The SM never
    // reads the old dW, and each pass is staged while the previous one drains (two buffers)
    constexpr int kRow = 512 + 16;   // padded rows: conflict-free 16-byte stores
    static_assert(2 * 128 * kRow <= tc::kStages * (tc::kStageA + tc::kStageBmax), "dW staging fits");
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int rl = 32 * (warp % 4) + lane;
    for (int pass = 0; pass < 4; ++pass) {
      const int half = pass >> 1, cb = (pass & 1) * 128;   // accumulator, first column
      uint8_t* stg = ts.a[0] + (pass & 1) * 128 * kRow;
      if (pass >= 2) {   // this buffer's previous pass has been read by the copy engine
        if (threadIdx.x < 128) tc::bulk_wait_read1();
        __syncthreads();
      }
      const int c0 = (warp / 4) * 64;   // this warp's 64 columns of the pass: four loads, one wait
      uint32_t v[4][16];
      const uint32_t ta = *ts.tmem_slot + ((uint32_t)(32 * (warp % 4)) << 16) + (uint32_t)(256 * half + cb + c0);
#pragma unroll
      for (int j = 0; j < 4; ++j) tc::tmem_ld16_nowait(ta + 16 * j, v[j]);
      tc::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *(uint4*)(stg + rl * kRow + (c0 + 16 * j + 4 * q) * 4) = *(uint4*)&v[j][4 * q];
      tc::fence_proxy_async_smem();   // generic-proxy stores -> the bulk copy's async reads
      __syncthreads();
      if (threadIdx.x < 128) {
        float* dst = (float*)I.p[3] + (int64_t)(m0 + 128 * half + threadIdx.x) * KT + nt * 256 + cb;
        if (acc) tc::bulk_s2g_add_f32(dst, stg + threadIdx.x * kRow, 512);
        else tc::bulk_s2g(dst, stg + threadIdx.x * kRow, 512);
        tc::bulk_commit();
      }
    }
    if (threadIdx.x < 128) {
      tc::bulk_wait_all();                // dW written before the tile completes
      tc::fence_proxy_async_global();
    }
    tc::tc_tile_end();                    // (its barrier also keeps the stage buffers until read)
    phase_epi(2, ph2);
    return;
  }
  for (int half = 0; half < 2; ++half) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int m = m0 + 128 * half + 32 * (warp % 4) + lane;
  float* dW = (float*)I.p[3] + (int64_t)m * KT + nt * 256;
  for (int c = (warp / 4) * 128; c < (warp / 4) * 128 + 128; c += 32) {
    float v[32];
    tc::tc_acc16(ts, 256 * half + c, v);
    tc::tc_acc16(ts, 256 * half + c + 16, v + 16);
    float4* d = (float4*)(dW + c);
    if (acc) {
      float4 old[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) old[q] = d[q];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        v[4 * q] += old[q].x;
        v[4 * q + 1] += old[q].y;
        v[4 * q + 2] += old[q].z;
        v[4 * q + 3] += old[q].w;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) d[q] = *(float4*)&v[4 * q];
  }
  }
  tc::tc_tile_end();
  phase_epi(2, ph2);
}

}  // namespace cfdev
