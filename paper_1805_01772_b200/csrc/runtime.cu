// libcf device runtime: ONE persistent kernel per cf_run.
//
//   block 0, thread 0  -- the device-resident loop driver: the paper's local executor
//                          moved onto the GPU. It evaluates every control
//                         node (Switch/Merge/Enter/Exit/NextIteration, the loop predicate,
//                         TensorArray and Stack bookkeeping) with the evaluation rules of
//                         PAPER.md:712-735, skips dead work, admits
//                         iteration i only when i - oldest_incomplete < K
//                         and turns every live float op into a tiled "heavy instance" whose
//                         dependencies it tracks. No host round trip per iteration.
//   blocks 1..G-1      -- workers: claim tiles from the job queue in publication order,
//                         execute them, report instance completion.
//
// The driver publishes an instance only when all its producers completed, so workers never
// wait on data; ordering is release (worker) -> acquire (driver) -> release (driver) ->
// acquire (worker), with __threadfence() (which also invalidates L1) on both sides.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <new>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "compiler.h"
#include "ir.h"
#include "program.h"
#include "tiles_tc.cuh"
#include "tmap.h"

using namespace cfdev;

namespace cf {
void set_error(const std::string& m);
}
const cf::Graph& cf_graph_ir(const cf_graph* g);

#define CUDA_OK(x)                                                                       \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      throw cf::CfError(CF_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));     \
  } while (0)

namespace {

constexpr int kThreads = 256;
constexpr int kEwTile = 4096;
#ifdef CF_PROFILE
constexpr bool kProfBuild = true;    // libcf_prof.so: driver region/instance profiler compiled in
#else
constexpr bool kProfBuild = false;   // libcf.so: no profiler code on the driver's path
#endif
constexpr int kEwBig = 16384;   // elementwise (HK_EW) tile
// forward / d[x,h] GEMMs use 256-row tiles from this batch size on (dW always does)
constexpr int kM2Default = 512;   // measured on cfg3 (B = 512): 2% faster than 1024
__device__ int kM2MinRows = kM2Default;
// test/profiling knob (cf_debug_set_flags): bit 0 = workers skip the tile bodies (isolates the
// driver's own cost; results are garbage)
__device__ int kDbgFlags = 0;
// worker roles (cf_debug_set_worker_roles): low 16 bits = workers that take low-priority (dW)
// work first, bit 16 = the other workers never take it
__device__ int kLowWorkers = 0;

// ----------------------------------------------------------------------------- helpers
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  return *(volatile const unsigned long long*)p;
}
__device__ __forceinline__ int ld_volatile_i32(const int* p) { return *(volatile const int*)p; }
__device__ __forceinline__ int ld_acquire_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// system scope: channel words written by / read from the peer GPU over NVLink
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void backoff(int& n) {
  if (n < 8) {
    ++n;
    return;
  }
  __nanosleep(n < 64 ? 32 : 256);
  if (n < 64) ++n;
}

__device__ __forceinline__ float sigm(float x) { return 1.0f / (1.0f + __expf(-x)); }
__device__ __forceinline__ float tanh_f(float x) { return tanhf(x); }

// ----------------------------------------------------------------------------- worker tiles
template <class LA, class LB, class EP>
__device__ void gemm_tile64(float* sm, int m0, int n0, int M, int N, int K, LA la, LB lb, EP ep) {
  float* As = sm;            // [16][64]
  float* Bs = sm + 16 * 64;  // [16][64]
  const int tid = threadIdx.x;
  const int ty = tid / 16, tx = tid % 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int idx = tid + i * 256;
      int kk = idx / 64, mm = idx % 64;
      int m = m0 + mm, k = k0 + kk;
      As[kk * 64 + mm] = (m < M && k < K) ? la(m, k) : 0.0f;
      int n = n0 + mm;
      Bs[kk * 64 + mm] = (n < N && k < K) ? lb(k, n) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        a[j] = As[kk * 64 + ty * 4 + j];
        b[j] = Bs[kk * 64 + tx * 4 + j];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < M && n < N) ep(m, n, acc[i][j]);
    }
}

// elementwise tile: kEwBig elements; 8 loads per input in flight per thread (memory-latency
// bound otherwise), dtype / broadcast decisions are warp-uniform
__device__ void tile_ew(const Inst& I, int tile) {
  const int64_t n = I.n;
  const int64_t b0 = (int64_t)tile * kEwBig;
  const int64_t e1 = min(n, b0 + kEwBig);
  const int op = I.sub;
  const int flags = (int)I.s[1];
  // fast path: fp32 binary add/sub/mul/addn2 without broadcast, 16 B vectors, 4 in flight
  const bool vec = flags == 0 && (I.dts & 0xF000000FFLL) == ((int64_t)D_F32 << 32 | D_F32 << 4 | D_F32) &&
                   (op == EW_ADD || op == EW_SUB || op == EW_MUL || (op == EW_ADDN && I.s[0] == 2)) &&
                   ((I.p[0] | I.p[1] | I.p[13]) & 15) == 0 && ((e1 - b0) & 4095) == 0;
  if (vec) {
    for (int64_t c0 = b0; c0 < e1; c0 += 4096) {
      const float4* a = (const float4*)I.p[0] + c0 / 4;
      const float4* b = (const float4*)I.p[1] + c0 / 4;
      float4* o = (float4*)I.p[13] + c0 / 4;
      float4 x[4], y[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        x[j] = a[threadIdx.x + j * kThreads];
        y[j] = b[threadIdx.x + j * kThreads];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float4 r;
        if (op == EW_MUL) r = make_float4(x[j].x * y[j].x, x[j].y * y[j].y, x[j].z * y[j].z, x[j].w * y[j].w);
        else if (op == EW_SUB) r = make_float4(x[j].x - y[j].x, x[j].y - y[j].y, x[j].z - y[j].z, x[j].w - y[j].w);
        else r = make_float4(x[j].x + y[j].x, x[j].y + y[j].y, x[j].z + y[j].z, x[j].w + y[j].w);
        o[threadIdx.x + j * kThreads] = r;
      }
    }
    return;
  }
  void* out = (void*)I.p[13];
  const int odt = (int)((I.dts >> 32) & 15);
  // 4-wide path for mixed fp32 / bf16 operands and broadcast scalars (16 / 8-byte accesses)
  const int dt0 = (int)(I.dts & 15), dt1 = (int)((I.dts >> 4) & 15);
  const bool ok_dt = (dt0 == D_F32 || dt0 == D_BF16) && (dt1 == D_F32 || dt1 == D_BF16) &&
                     (odt == D_F32 || odt == D_BF16);
  if (ok_dt && (op == EW_ADD || op == EW_SUB || op == EW_MUL || (op == EW_ADDN && I.s[0] == 2)) &&
      ((I.p[0] | I.p[1] | I.p[13]) & 7) == 0 && (b0 & 3) == 0) {
    const int64_t e4 = b0 + ((e1 - b0) & ~(int64_t)3);
    const bool bc0 = flags & 1, bc1 = flags & 2;
    const float s0 = bc0 ? ldf((const void*)I.p[0], dt0, 0) : 0.f, s1 = bc1 ? ldf((const void*)I.p[1], dt1, 0) : 0.f;
    auto ld4 = [&](int j, int dt, bool bc, float sv, int64_t e) -> float4 {
      if (bc) return make_float4(sv, sv, sv, sv);
      if (dt == D_F32) return *(const float4*)((const float*)I.p[j] + e);
      const uint2 u = *(const uint2*)((const __nv_bfloat16*)I.p[j] + e);
      const float2 a = __bfloat1622float2(*(const __nv_bfloat162*)&u.x);
      const float2 b = __bfloat1622float2(*(const __nv_bfloat162*)&u.y);
      return make_float4(a.x, a.y, b.x, b.y);
    };
    constexpr int V = 4;
    for (int64_t base = b0 + 4 * threadIdx.x; base < e4; base += (int64_t)4 * V * kThreads) {
      float4 x[V], y[V];
#pragma unroll
      for (int k = 0; k < V; ++k) {
        int64_t e = base + (int64_t)4 * k * kThreads;
        if (e > e4 - 4) e = e4 - 4;
        x[k] = ld4(0, dt0, bc0, s0, e);
        y[k] = ld4(1, dt1, bc1, s1, e);
      }
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const int64_t e = base + (int64_t)4 * k * kThreads;
        if (e >= e4) break;
        float4 r;
        if (op == EW_MUL) r = make_float4(x[k].x * y[k].x, x[k].y * y[k].y, x[k].z * y[k].z, x[k].w * y[k].w);
        else if (op == EW_SUB) r = make_float4(x[k].x - y[k].x, x[k].y - y[k].y, x[k].z - y[k].z, x[k].w - y[k].w);
        else r = make_float4(x[k].x + y[k].x, x[k].y + y[k].y, x[k].z + y[k].z, x[k].w + y[k].w);
        if (odt == D_F32) {
          *(float4*)((float*)out + e) = r;
        } else {
          __nv_bfloat162 lo = __floats2bfloat162_rn(r.x, r.y), hi = __floats2bfloat162_rn(r.z, r.w);
          uint2 u;
          u.x = *(unsigned*)&lo;
          u.y = *(unsigned*)&hi;
          *(uint2*)((__nv_bfloat16*)out + e) = u;
        }
      }
    }
    for (int64_t e = e4 + threadIdx.x; e < e1; e += kThreads) {   // ragged tail
      const float a = bc0 ? s0 : ldf((const void*)I.p[0], dt0, e), b = bc1 ? s1 : ldf((const void*)I.p[1], dt1, e);
      stf(out, odt, e, op == EW_MUL ? a * b : op == EW_SUB ? a - b : a + b);
    }
    return;
  }
  auto in = [&](int j, int64_t e) -> float {
    return ldf((const void*)I.p[j], (int)((I.dts >> (4 * j)) & 15), (flags >> j & 1) ? 0 : e);
  };
  const int nin = op == EW_ADDN ? (int)I.s[0] : (op == EW_SELECT ? 3 : (op == EW_NEG || op == EW_SIGMOID ||
                  op == EW_TANH || op == EW_RELU || op == EW_ZEROS) ? 1 : 2);
  constexpr int U = 8;
  for (int64_t base = b0 + threadIdx.x; base < e1; base += (int64_t)U * kThreads) {
    float v0[U], v1[U], v2[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t e = min(base + (int64_t)k * kThreads, e1 - 1);
      v0[k] = op == EW_ZEROS || op == EW_SELECT || op == EW_ADDN ? 0.0f : in(0, e);
      v1[k] = nin > 1 && op != EW_BIASADD && op != EW_SELECT && op != EW_ADDN ? in(1, e) : 0.0f;
      v2[k] = 0.0f;
      if (op == EW_ADDN)
        for (int j = 0; j < nin; ++j) v2[k] += in(j, e);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t e = base + (int64_t)k * kThreads;
      if (e >= e1) break;
      float r = 0.0f;
      switch (op) {
        case EW_ADD: r = v0[k] + v1[k]; break;
        case EW_SUB: r = v0[k] - v1[k]; break;
        case EW_MUL: r = v0[k] * v1[k]; break;
        case EW_NEG: r = -v0[k]; break;
        case EW_SIGMOID: r = 1.0f / (1.0f + expf(-v0[k])); break;
        case EW_TANH: r = tanhf(v0[k]); break;
        case EW_RELU: r = fmaxf(v0[k], 0.0f); break;
        case EW_RELUGRAD: r = v1[k] > 0.0f ? v0[k] : 0.0f; break;
        case EW_BIASADD: r = v0[k] + ldf((const void*)I.p[1], (int)((I.dts >> 4) & 15), e % I.m); break;
        case EW_SELECT: {
          const uint8_t* c = (const uint8_t*)I.p[0];
          bool cv = I.s[2] ? c[0] != 0 : (I.m > 0 ? c[e / I.m] != 0 : c[e] != 0);
          r = cv ? in(1, e) : in(2, e);
          break;
        }
        case EW_ADDN: r = v2[k]; break;
        case EW_ZEROS: r = 0.0f; break;
      }
      stf(out, odt, e, r);
    }
  }
}

__device__ void tile_fill(const Inst& I, int tile) {
  float v = I.p[0] ? ldf((const void*)I.p[0], (int)(I.dts & 15), 0) : __int_as_float((int)I.s[0]);
  const int odt = (int)((I.dts >> 32) & 15);
  int64_t b0 = (int64_t)tile * kEwBig, e1 = min(I.n, b0 + kEwBig);
  if (odt == D_F32 && (I.p[13] & 15) == 0 && ((e1 - b0) & 3) == 0) {
    float4* o = (float4*)((float*)I.p[13] + b0);
    for (int64_t e = threadIdx.x; e < (e1 - b0) / 4; e += kThreads) o[e] = make_float4(v, v, v, v);
    return;
  }
  for (int64_t e = b0 + threadIdx.x; e < e1; e += kThreads) stf((void*)I.p[13], odt, e, v);
}

__device__ void tile_copy(const Inst& I, int tile) {
  // I.n bytes; 64 KiB per tile
  const int64_t chunk = 65536;
  int64_t b0 = (int64_t)tile * chunk, e1 = min(I.n, b0 + chunk);
  const uint8_t* src = (const uint8_t*)I.p[0];
  uint8_t* dst = (uint8_t*)I.p[13];
  bool aligned = ((I.p[0] | I.p[13]) & 15) == 0;
  if (aligned && I.sub == 1) {
    // channel slot written by the peer GPU: bypass L1 (a stale line of an earlier message
    // in the same slot could otherwise be returned)
    int64_t v0 = b0 / 16, v1 = e1 / 16;
    for (int64_t e = v0 + threadIdx.x; e < v1; e += kThreads) ((int4*)dst)[e] = __ldcv((const int4*)src + e);
    for (int64_t e = v1 * 16 + threadIdx.x; e < e1; e += kThreads) dst[e] = src[e];
  } else if (aligned) {
    int64_t v0 = b0 / 16, v1 = e1 / 16;
    int64_t e = v0 + threadIdx.x;
    for (; e + 3 * kThreads < v1; e += 4 * kThreads) {
      int4 r[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) r[j] = ((const int4*)src)[e + j * kThreads];
#pragma unroll
      for (int j = 0; j < 4; ++j) ((int4*)dst)[e + j * kThreads] = r[j];
    }
    for (; e < v1; e += kThreads) ((int4*)dst)[e] = ((const int4*)src)[e];
    for (int64_t e = v1 * 16 + threadIdx.x; e < e1; e += kThreads) dst[e] = src[e];
  } else {
    for (int64_t e = b0 + threadIdx.x; e < e1; e += kThreads) dst[e] = src[e];
  }
}

__device__ void tile_acc(const Inst& I, int tile) {
  const int sdt = (int)(I.dts & 15), odt = (int)((I.dts >> 32) & 15);
  int64_t b0 = (int64_t)tile * kEwTile, e1 = min(I.n, b0 + kEwTile);
  for (int64_t e = b0 + threadIdx.x; e < e1; e += kThreads)
    stf((void*)I.p[13], odt, e, ldf((void*)I.p[13], odt, e) + ldf((const void*)I.p[0], sdt, e));
}

__device__ float block_sum(float v, float* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float s = 0.0f;
  if (threadIdx.x == 0)
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
  __syncthreads();
  return s;
}

// deterministic: tile t sums a fixed contiguous chunk; the last tile sums partials in order
__device__ void tile_reduce_sum(const Inst& I, int tile, float* sm) {
  const void* x = (const void*)I.p[0];
  const int xdt = (int)(I.dts & 15);
  float* out = (float*)I.p[13];
  float* partial = out + 1024;   // placement reserves 1024 partial floats at +4 KiB
  int64_t chunk = (I.n + I.ntiles - 1) / I.ntiles;
  int64_t b0 = (int64_t)tile * chunk, e1 = min(I.n, b0 + chunk);
  float s = 0.0f;
  for (int64_t e = b0 + threadIdx.x; e < e1; e += kThreads) s += ldf(x, xdt, e);
  s = block_sum(s, sm);
  if (threadIdx.x == 0) partial[tile] = s;
}
__device__ void finalize_reduce_sum(const Inst& I, float* sm) {
  float* out = (float*)I.p[13];
  const volatile float* partial = out + 1024;
  if (threadIdx.x == 0) {
    float s = 0.0f;
    for (int t = 0; t < I.ntiles; ++t) s += partial[t];
    out[0] = s;
  }
  (void)sm;
}

__device__ void tile_reduce_sum0(const Inst& I, int tile) {
  const void* x = (const void*)I.p[0];
  const int xdt = (int)(I.dts & 15), odt = (int)((I.dts >> 32) & 15);
  int64_t M = I.m, N = I.n;
  int64_t c = (int64_t)tile * kThreads + threadIdx.x;
  if (c >= N) return;
  float s = 0.0f;
  for (int64_t r = 0; r < M; ++r) s += ldf(x, xdt, r * N + c);
  stf((void*)I.p[13], odt, c, s);
}

__device__ void tile_matmul(const Inst& I, int tile, float* sm) {
  int M = (int)I.m, N = (int)I.n, K = (int)I.k;
  bool ta = I.sub & 1, tb = I.sub & 2;
  int64_t lda = I.s[0], ldb = I.s[1];
  const void* A = (const void*)I.p[0];
  const void* B = (const void*)I.p[1];
  const int adt = (int)(I.dts & 15), bdt = (int)((I.dts >> 4) & 15), odt = (int)((I.dts >> 32) & 15);
  int tn = (N + 63) / 64;
  int m0 = (tile / tn) * 64, n0 = (tile % tn) * 64;
  gemm_tile64(
      sm, m0, n0, M, N, K,
      [&](int m, int k) { return ldf(A, adt, ta ? (int64_t)k * lda + m : (int64_t)m * lda + k); },
      [&](int k, int n) { return ldf(B, bdt, tb ? (int64_t)n * ldb + k : (int64_t)k * ldb + n); },
      [&](int m, int n, float v) { stf((void*)I.p[13], odt, (int64_t)m * N + n, v); });
}

// Fused LSTM cell forward (reading R9): tile = 32 batch rows x 32 hidden units; each thread
// owns 4 rows x 1 unit x all 4 gates, so the sigma/tanh/state epilogue is thread-local.
__device__ void tile_lstm_fwd(const Inst& I, int tile, float* sm) {
  const int B = (int)I.m, In = (int)I.k, H = (int)I.n;
  const int KT = In + H;
  const float* x = (const float*)I.p[0];
  const float* h = (const float*)I.p[1];
  const float* c = (const float*)I.p[2];
  const float* W = (const float*)I.p[3];
  const float* bias = (const float*)I.p[4];
  const int64_t* lens = (const int64_t*)I.p[5];
  float* h_next = (float*)I.p[8];
  float* c_next = (float*)I.p[9];
  float* out = (float*)I.p[10];
  float* gates = (float*)I.p[11];
  const bool masked = I.sub & 1;
  const int64_t t = I.s[0];
  const float fbias = __int_as_float((int)I.s[1]);
  const int n_ut = (H + 31) / 32;
  const int r0 = (tile / n_ut) * 32, u0 = (tile % n_ut) * 32;
  float* Xs = sm;               // [32 k][33]
  float* Ws = sm + 32 * 33;     // [32 k][129]
  const int tid = threadIdx.x, ty = tid / 32, tx = tid % 32;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < KT; k0 += 32) {
    for (int idx = tid; idx < 32 * 32; idx += kThreads) {
      int rr = idx / 32, kk = idx % 32;
      int r = r0 + rr, k = k0 + kk;
      float v = 0.0f;
      if (r < B && k < KT) v = k < In ? x[(int64_t)r * In + k] : h[(int64_t)r * H + (k - In)];
      Xs[kk * 33 + rr] = v;
    }
    for (int idx = tid; idx < 128 * 32; idx += kThreads) {
      int col = idx / 32, kk = idx % 32;
      int g = col / 32, u = u0 + col % 32, k = k0 + kk;
      Ws[kk * 129 + col] = (u < H && k < KT) ? W[(int64_t)(g * H + u) * KT + k] : 0.0f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      float a[4], w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) a[j] = Xs[kk * 33 + ty * 4 + j];
#pragma unroll
      for (int g = 0; g < 4; ++g) w[g] = Ws[kk * 129 + g * 32 + tx];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int g = 0; g < 4; ++g) acc[j][g] = fmaf(a[j], w[g], acc[j][g]);
    }
    __syncthreads();
  }
  const int u = u0 + tx;
  if (u >= H) return;
  const float bi = bias[u], bf = bias[H + u], bg = bias[2 * H + u], bo = bias[3 * H + u];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int r = r0 + ty * 4 + j;
    if (r >= B) continue;
    const int64_t o = (int64_t)r * H + u;
    float ig = 1.0f / (1.0f + expf(-(acc[j][0] + bi)));
    float fg = 1.0f / (1.0f + expf(-(acc[j][1] + bf + fbias)));
    float gg = tanhf(acc[j][2] + bg);
    float og = 1.0f / (1.0f + expf(-(acc[j][3] + bo)));
    float cp = c[o];
    float cn = fg * cp + ig * gg;
    float hn = og * tanhf(cn);
    bool live = !masked || t < lens[r];
    h_next[o] = live ? hn : h[o];
    c_next[o] = live ? cn : cp;
    out[o] = live ? hn : 0.0f;
    float* gr = gates + (int64_t)r * 4 * H;
    gr[u] = ig;
    gr[H + u] = fg;
    gr[2 * H + u] = gg;
    gr[3 * H + u] = og;
  }
}

// LSTM cell backward, elementwise part: dz (pre-activation grads) and dc_prev.
__device__ void tile_lstm_bwd_ew(const Inst& I, int tile) {
  const int B = (int)I.m, H = (int)I.n;
  const float* c = (const float*)I.p[2];
  const float* gates = (const float*)I.p[4];
  const int64_t* lens = (const int64_t*)I.p[5];
  const float* dhn = (const float*)I.p[6];
  const float* dcn = (const float*)I.p[7];
  const float* dout = (const float*)I.p[8];
  float* dc = (float*)I.p[9];
  float* dz = (float*)I.p[10];
  const bool masked = I.sub & 1;
  const int64_t t = I.s[0];
  int64_t b0 = (int64_t)tile * kEwTile, e1 = min((int64_t)B * H, b0 + kEwTile);
  for (int64_t e = b0 + threadIdx.x; e < e1; e += kThreads) {
    int64_t r = e / H, u = e % H;
    const float* gr = gates + r * 4 * H;
    float ig = gr[u], fg = gr[H + u], gg = gr[2 * H + u], og = gr[3 * H + u];
    float cp = c[e];
    float cn = fg * cp + ig * gg;
    float tc = tanhf(cn);
    float dh = dhn[e] + dout[e];
    if (I.p[14]) dh += ((const float*)I.p[14])[e];   // folded AddN terms (compiler fuse_dout_sums)
    if (I.p[15]) dh += ((const float*)I.p[15])[e];
    float dcs = dh * og * (1.0f - tc * tc) + dcn[e];
    float dzi = dcs * gg * ig * (1.0f - ig);
    float dzf = dcs * cp * fg * (1.0f - fg);
    float dzg = dcs * ig * (1.0f - gg * gg);
    float dzo = dh * tc * og * (1.0f - og);
    float dcp = dcs * fg;
    if (masked && !(t < lens[r])) {
      dzi = dzf = dzg = dzo = 0.0f;
      dcp = dcn[e];
    }
    float* zr = dz + r * 4 * H;
    zr[u] = dzi;
    zr[H + u] = dzf;
    zr[2 * H + u] = dzg;
    zr[3 * H + u] = dzo;
    dc[e] = dcp;
  }
}

// LSTM cell backward, contractions: d[x,h] = dz W ; dW = dz^T [x,h] ; db = colsum(dz).
__device__ void tile_lstm_bwd_mm(const Inst& I, int tile, float* sm) {
  const int B = (int)I.m, In = (int)I.k, H = (int)I.n, KT = In + H, G = 4 * H;
  const float* x = (const float*)I.p[0];
  const float* h = (const float*)I.p[1];
  const float* W = (const float*)I.p[3];
  const int64_t* lens = (const int64_t*)I.p[5];
  const float* dhn = (const float*)I.p[6];
  const float* dz = (const float*)I.p[10];
  float* dx = (float*)I.p[11];
  float* dh = (float*)I.p[12];
  float* dW = (float*)I.p[13];
  float* db = (float*)I.s[3];
  const bool masked = I.sub & 1;
  const int64_t t = I.s[0];
  const int tA = ((B + 63) / 64) * ((KT + 63) / 64);
  const int tB = ((G + 63) / 64) * ((KT + 63) / 64);
  if (tile < tA) {
    int tn = (KT + 63) / 64;
    int m0 = (tile / tn) * 64, n0 = (tile % tn) * 64;
    gemm_tile64(
        sm, m0, n0, B, KT, G, [&](int m, int k) { return dz[(int64_t)m * G + k]; },
        [&](int k, int n) { return W[(int64_t)k * KT + n]; },
        [&](int m, int n, float v) {
          if (n < In) {
            dx[(int64_t)m * In + n] = v;
          } else {
            int64_t o = (int64_t)m * H + (n - In);
            dh[o] = (masked && !(t < lens[m])) ? dhn[o] : v;
          }
        });
  } else if (tile < tA + tB) {
    int tt = tile - tA;
    int tn = (KT + 63) / 64;
    int m0 = (tt / tn) * 64, n0 = (tt % tn) * 64;
    gemm_tile64(
        sm, m0, n0, G, KT, B, [&](int m, int k) { return dz[(int64_t)k * G + m]; },
        [&](int k, int n) { return n < In ? x[(int64_t)k * In + n] : h[(int64_t)k * H + (n - In)]; },
        [&](int m, int n, float v) {
          float* d = dW + (int64_t)m * KT + n;
          *d = (I.s[6] & 1) ? *d + v : v;
        });
  } else {
    int tt = tile - tA - tB;
    int col = tt * kThreads + threadIdx.x;
    if (col < G) {
      float s = 0.0f;
      for (int r = 0; r < B; ++r) s += dz[(int64_t)r * G + col];
      db[col] = (I.s[6] & 2) ? db[col] + s : s;
    }
  }
}

// ----------------------------------------------------------------------------- driver
enum EvalResult { EV_OK = 0, EV_BLOCKED = 1, EV_ERROR = 2 };

// ---- routing / stack nodes without the general evaluator (PAPER.md:712-735 rules on 16-byte
// tokens; token word w = dead (bits 0-7) | kind (8-15) | dt (16-23)). Shared by the driver
// thread and the helper warps that evaluate a wave of independent nodes in parallel.
struct FastEnv {
  int4* tk;
  const int32_t* iv;
  int it, bb;
  int git;                   // iteration index over all instances of a nested frame
  uint8_t* bbits;
  const int8_t* lval;        // liveness of structured cond contexts (this iteration)
  const DStack* stacks;
  int32_t* depth;
  int4* pool;
  // accumulators and TensorArray bookkeeping (ACC / TA_READ / TA_WRITE fast paths)
  const DAcc* accs;
  const int32_t* accw;
  const DTA* tas;
  const int64_t* tab;
  const int32_t* tso;
  int32_t* ta_writer;
  uint8_t* ta_written;
};
struct FastCount {
  int push, pop, maxd, err;
  long long err_info;
};
// 1 = evaluated, 0 = needs the general evaluator (nothing written), -1 = error (in c.err)
__device__ __forceinline__ int fast_node(const DNode* d, const FastEnv& e, FastCount& c) {
  const int op = d->op;
  int4* tk = e.tk;
  const int32_t* iv = e.iv;
  if (op == OP_SWITCH) {
    if (d->n_ctrl) return 0;
    const int4 dv = tk[iv[d->in_off]];
    const int4 pt = tk[iv[d->in_off + 1]];
    const int dead = (dv.w | pt.w) & 0xff;
    if (((pt.w >> 8) & 0xff) != TK_IMM && !dead) return 0;
    int4 o0 = dv, o1 = dv;
    if (dead) {
      o0.w |= 1;
      o1.w |= 1;
    } else {
      const bool p = (pt.x | pt.y) != 0;
      o0.w = (o0.w & ~0xff) | (p ? 1 : 0);   // false port dead iff p
      o1.w = (o1.w & ~0xff) | (p ? 0 : 1);
      if (d->aux[0] >= 0 && e.git < e.bb) e.bbits[d->aux[0] * e.bb + e.git] = p ? 2 : 1;
    }
    tk[d->out_vid] = o0;
    tk[d->out_vid + 1] = o1;
    tk[d->ctrl_vid] = make_int4(0, 0, -1, (TK_FLOW << 8) | dead);
    return 1;
  }
  if (op == OP_MERGE) {
    const int4 a = tk[iv[d->in_off]];
    const int4 b = tk[iv[d->in_off + 1]];
    int4 o = (a.w & 0xff) ? b : a;   // "if is_dead(d1) then d2 else d1"
    if (d->aux[5]) {   // structured: the live branch's input (the other one was not evaluated)
      const int l1 = e.lval[d->aux[6]], l0 = e.lval[d->aux[5]];
      o = l1 ? b : a;
      if (!l1 && !l0) o.w |= 1;
    }
    tk[d->out_vid] = o;
    tk[d->ctrl_vid] = make_int4(0, 0, -1, (TK_FLOW << 8) | (o.w & 0xff));
    return 1;
  }
  if (op == OP_MERGE_LOOP || (op == OP_NEXTITER && !d->n_ctrl)) {
    const int4 o = tk[iv[d->in_off + (op == OP_MERGE_LOOP && e.it != 0 ? 1 : 0)]];
    tk[d->out_vid] = o;
    tk[d->ctrl_vid] = make_int4(0, 0, -1, (TK_FLOW << 8) | (o.w & 0xff));
    return 1;
  }
  if ((op >= OP_CONST && op <= OP_TA_GRAD) || op == OP_ACC) {
    // value-free ops: dead if any data or control input is dead
    int dead = 0;
    for (int j = 0; j < d->n_in; ++j) dead |= tk[iv[d->in_off + j]].w & 0xff;
    for (int j = 0; j < d->n_ctrl; ++j) dead |= tk[iv[d->ctrl_off + j]].w & 0xff;
    dead = dead ? 1 : 0;
    const int4 ctrl = make_int4(0, 0, -1, (TK_FLOW << 8) | dead);
    switch (op) {
      case OP_CONST: {
        const long long v = d->imm[0];
        tk[d->out_vid] = make_int4((int)(v & 0xffffffffLL), (int)(v >> 32), -1,
                                   dead | ((d->aux[0] == 1 ? TK_IMM : TK_PTR) << 8) | ((d->aux[1] & 0xff) << 16));
        break;
      }
      case OP_PASS:
      case OP_FLOW: {
        int4 t = op == OP_PASS && d->n_in ? tk[iv[d->in_off]] : make_int4(0, 0, 0, 0);
        if (op == OP_FLOW) t = make_int4(0, 0, -1, TK_FLOW << 8);
        t.w = (t.w & ~0xff) | dead;
        for (int p = 0; p < d->n_out; ++p) tk[d->out_vid + p] = t;
        break;
      }
      case OP_SCALAR: {
        if (dead) {
          for (int p = 0; p < d->n_out; ++p) tk[d->out_vid + p] = make_int4(0, 0, -1, 1);
          break;
        }
        long long ab[2] = {0, 0};
        for (int j = 0; j < d->n_in && j < 2; ++j) {
          const int4 t = tk[iv[d->in_off + j]];
          const int kind = (t.w >> 8) & 0xff;
          if (kind == TK_PTR) return 0;   // device value: the general evaluator waits for it
          if (kind == TK_IMM) ab[j] = (long long)(((unsigned long long)(unsigned)t.y << 32) | (unsigned)t.x);
        }
        const long long a = ab[0], b = ab[1];
        long long r = 0;
        switch (d->aux[0]) {
          case SC_ADD: r = a + b; break;
          case SC_SUB: r = a - b; break;
          case SC_MUL: r = a * b; break;
          case SC_LESS: r = a < b; break;
          case SC_LEQ: r = a <= b; break;
          case SC_GREATER: r = a > b; break;
          case SC_EQ: r = a == b; break;
          case SC_AND: r = (a != 0) && (b != 0); break;
          case SC_NOT: r = a == 0; break;
          case SC_CAST: r = d->aux[1] == D_BOOL ? (a != 0) : a; break;
        }
        tk[d->out_vid] = make_int4((int)(r & 0xffffffffLL), (int)(r >> 32), -1,
                                   (TK_IMM << 8) | ((d->aux[1] & 0xff) << 16));
        break;
      }
      case OP_ACC: {   // fused accumulator: producers added in place
        const long long v = e.accs[d->aux[0]].base;
        tk[d->out_vid] = make_int4((int)(v & 0xffffffffLL), (int)(v >> 32), e.accw[d->aux[0]],
                                   dead | (TK_PTR << 8) | (D_F32 << 16));
        break;
      }
      case OP_TA_GRAD: {
        tk[d->out_vid] = make_int4(d->aux[0], 0, -1, dead | (TK_HANDLE << 8));
        tk[d->out_vid + 1] = make_int4(0, 0, -1, dead | (TK_FLOW << 8));
        break;
      }
      case OP_TA_READ:
      case OP_TA_WRITE: {
        if (dead) {
          if (op == OP_TA_READ) tk[d->out_vid] = make_int4(0, 0, -1, 1);
          else tk[d->out_vid] = make_int4(0, 0, -1, 1 | (TK_FLOW << 8));
          break;
        }
        const int4 ht = tk[iv[d->in_off]], it = tk[iv[d->in_off + 1]];
        if (((it.w >> 8) & 0xff) != TK_IMM) return 0;
        const int ta = ht.x;
        const long long ix = (long long)(((unsigned long long)(unsigned)it.y << 32) | (unsigned)it.x);
        const DTA& T = e.tas[ta];
        if (ix < 0 || ix >= T.size) return 0;   // the general evaluator reports it
        const int so = e.tso[ta] + (int)ix;
        const long long addr = e.tab[ta] + ix * T.elem_bytes;
        if (op == OP_TA_READ) {
          if (!T.is_grad && !e.ta_written[so]) return 0;
          tk[d->out_vid] = make_int4((int)(addr & 0xffffffffLL), (int)(addr >> 32), e.ta_writer[so],
                                     (TK_PTR << 8) | ((T.dt & 0xff) << 16));
        } else {
          // zero-copy write only (the producer was placed in the slot); first write
          const int4 v = tk[iv[d->in_off + 2]];
          const long long vp = (long long)(((unsigned long long)(unsigned)v.y << 32) | (unsigned)v.x);
          if (vp != addr || e.ta_written[so]) return 0;
          e.ta_writer[so] = v.z;
          e.ta_written[so] = 1;
          tk[d->out_vid] = make_int4(0, 0, -1, TK_FLOW << 8);
        }
        break;
      }
      default:
        return 0;
    }
    tk[d->ctrl_vid] = ctrl;
    return 1;
  }
  if (op == OP_STACK_PUSH || op == OP_STACK_POP) {
    const int4 h = tk[iv[d->in_off]];
    const int4 v = op == OP_STACK_PUSH ? tk[iv[d->in_off + 1]] : h;
    int dead = (h.w | v.w) & 0xff;
    for (int j = 0; j < d->n_ctrl; ++j) dead |= tk[iv[d->ctrl_off + j]].w & 0xff;
    if (dead) {   // dead push: nothing stored; dead pop: dead output
      if (op == OP_STACK_POP) {
        int4 t = make_int4(0, 0, -1, 1);
        tk[d->out_vid] = t;
      }
      tk[d->ctrl_vid] = make_int4(0, 0, -1, (TK_FLOW << 8) | 1);
      return 1;
    }
    // TK_HANDLE: v = stack id | instance << 20 (x = low 32 bits, y = high)
    const long long hv = (long long)(((unsigned long long)(unsigned)h.y << 32) | (unsigned)h.x);
    const int sid = (int)(hv & 0xFFFFF), inst = (int)(hv >> 20);
    const DStack& S = e.stacks[sid];
    const int di = S.depth_off + inst;
    const int dp = e.depth[di];
    int4* pool = e.pool + S.entry_off + (long long)inst * S.capacity;
    if (op == OP_STACK_PUSH) {
      if (dp >= S.capacity) {
        c.err = CF_E_STACK_BUDGET;
        c.err_info = dp;
        return -1;
      }
      pool[dp] = v;
      e.depth[di] = dp + 1;
      c.push++;
      c.maxd = max(c.maxd, dp + 1);
    } else {
      if (dp <= 0) {
        c.err = CF_E_POP_EMPTY;
        c.err_info = sid | ((long long)inst << 20);
        return -1;
      }
      int4 t = pool[dp - 1];
      t.w &= ~0xff;
      e.depth[di] = dp - 1;
      tk[d->out_vid] = t;
      c.pop++;
    }
    tk[d->ctrl_vid] = make_int4(0, 0, -1, TK_FLOW << 8);
    return 1;
  }
  return 0;
}

// helper warps serving waves: warps 1-3 and 5-7 (warp 4 shares the driver warp's scheduler)
constexpr int kWaveWarps = 6;
__device__ __forceinline__ int wave_lane(int tid) {
  const int w = tid >> 5;
  return w < 4 ? tid - 32 : tid - 64;   // 0..191 for warps 1-3, 5-7
}
__device__ __forceinline__ int wave_lane5(int tid) {
  const int w = tid >> 5;
  return w < 4 ? tid - 64 : tid - 96;   // 0..159 for warps 2-3, 5-7 (warp 1 busy with a batch)
}

// a wave request from the driver thread to the helper warps (shared memory)
struct Wave {
  int seq, done;          // request number / helper warps finished
  int start, n;           // body program range
  int nslow;
  FastCount cnt;
  const DNode* bn;
  FastEnv env;
  int env_frame;          // frame whose FastEnv is in env (-2: none); env.it is per wave
  // job 1: preparation of a tensor-core LSTM node (Driver::heavy_prep_lane): dead check,
  // output placements, operand-registry lookups, computed by the helper lanes in parallel
  int job;
  const DNode* hd;
  int chain;              // routing wave followed by the preparation of node hd (same job)
  int nlev, lev_stop;     // fused levels; levels completed (set by the helpers)
  int lev_start[16], lev_n[16];
  unsigned long long lev_ctx[16];   // cond contexts each level reads (evaluated by a helper lane
                                    // before the level when the driver did not know them yet)
  unsigned long long lev_ctx_hi[16];   // contexts 64..127
  int cstop;              // level the helpers could not start (a context's predicate was not
                          // available yet), or -1
  int hdead, hfail;
  int64_t houtp[8];
  int64_t hmap[5], hslot[5];
  int slow[256];          // wave positions left for the general evaluator
  // job 2: a heavy batch (Driver::run_batch): helper warp 1 builds the members' instances,
  // lane m = member m; ids reserved by the driver thread (-1: none / member not live)
  int bpc, bcount, bfail;
  int bid[32][4];         // per member: main (fwd) / EW (bwd), DXH (bwd), dW flush, weight prep
  int bnid[32];           // per member: graph node id
  // profiling build: batch phase clocks (issue by the driver, lane 0's start / phase A end,
  // the slowest lane's end)
  long long bt_issue, bt_start, bt_a, bt_chk, bt_res, bt_built;
  unsigned long long bt_end;
  // job 3 (the whole batch on the lanes): id base, the frame's body offset, and what the
  // lanes hand back (ids used, tiles, dead members, queue tails touched, last dW chunk)
  int bbase, bfoff;
  int bids, btiles, bdead, bdirty, blast;
  // job 3 runs on its own request counter (bseq, warp 1 only) with its own signals: placements
  // and tokens done (bphase), everything done (bdone). Meanwhile the driver may dispatch the
  // next wave job to the other five helper warps (nw = 5, skip1): the lanes' records, edges
  // and submissions overlap the routing after the batch
  int bseq, bphase, bdone;
  int bgo;                // the driver stopped processing completions: the lanes may add edges
  int nw, skip1;          // warps in the current wave / prep job, warp 1 excluded
};

__device__ void wave_work(Wave& w, int start, int n, int h, int nh) {
  FastCount c{0, 0, 0, 0, 0};
  for (int j = h; j < n; j += nh) {
    const DNode* d = w.bn + start + j;
    if (d->ctx && !w.env.lval[d->ctx]) continue;   // node of a dead cond branch
    const int r = fast_node(d, w.env, c);
    if (r == 0) w.slow[atomicAdd(&w.nslow, 1)] = j;
    if (r < 0) {
      w.cnt.err = c.err;
      w.cnt.err_info = c.err_info;
    }
  }
  if (c.push) atomicAdd(&w.cnt.push, c.push);
  if (c.pop) atomicAdd(&w.cnt.pop, c.pop);
  if (c.maxd) atomicMax(&w.cnt.maxd, c.maxd);
}

struct Driver {
  const RunArgs& A;
  const Prog& P;
  RunState* st;
  int32_t ninst = 0, nedge = 0;
  unsigned long long q_tail = 0;
  unsigned long long cq_head_ = 0;
  int64_t outstanding = 0;     // created - completed
  int32_t root_pc = 0, cur_frame = -1, iter = 0, body_pc = 0;
  bool iter_started = false, fetched = false;
  int32_t oldest = 0;
  // nested frames: the enclosing frames' evaluation state, and the
  // iteration index base of the current frame instance (indices run on over the instances
  // of a nested frame: arena slots, stack instances and branch bits use them)
  struct FrameSave {
    const DNode* bn;
    const int32_t* iv;
    int32_t frame, iter, oldest, body_pc, gbase, started;
  };
  static constexpr int kMaxNest = 4;
  FrameSave fstack_[kMaxNest];
  int fdepth_ = 0;
  int32_t gbase_ = 0;
  int32_t gnext_[16] = {};
  __forceinline__ __device__ int git() const { return cur_frame >= 0 ? gbase_ + iter : 0; }
  unsigned long long last_progress = 0;
  int64_t pend_mz = 0;
  int32_t last_dw = -1;
  unsigned long long lq_tail = 0;
  // pending channel waits (HK_WAIT instances), polled by drain()
  static constexpr int kMaxWaits = 64;   // f3's exchange at 4 GPUs needs 2 x 8 layers x 3 peers = 48
  struct ChanWait {
    unsigned long long* flag;
    unsigned long long want;
    unsigned long long* ack;
    unsigned long long ackv;
    int32_t id, pad;
  };
  ChanWait waits_[kMaxWaits];
  int n_waits_ = 0;
  // waits published while the table is full (many Recvs in flight: K iterations x peers)
  static constexpr int kWaitOvf = 4096;
  int ovf_head_ = 0, ovf_tail_ = 0;
  __device__ void add_wait(int32_t id) {
    const Inst& I = A.insts[id];
    ChanWait& w = waits_[n_waits_++];
    w.flag = (unsigned long long*)I.p[0];
    w.want = (unsigned long long)I.s[0];
    w.ack = (unsigned long long*)I.p[1];
    w.ackv = (unsigned long long)I.s[1];
    w.id = id;
  }
  // swap I/O (a8)
  unsigned long long io_tail = 0, io_head = 0;
  int io_out = 0;   // swap requests not yet completed
  long long n_swap_out = 0, n_swap_in = 0, b_d2h = 0, b_h2d = 0;
  unsigned long long q_done_seen = 0;

  // driver-private state; shared memory when it fits (see cf_driver_kernel), else global
  const PlaceDesc* places_;
  const DReg* reg_;
  int32_t* stack_depth_;
  int32_t* prep_inst_;
  int32_t* dw_count_;
  int32_t* acc_writer_;
  int32_t* iter_out_;
  const DStack* stacks_;
  // TensorArray metadata (shared memory when it fits, else the global tables)
  const DTA* tas_;
  int64_t* tab_;
  const int32_t* tso_;
  long long n_push = 0, n_pop = 0, n_dead = 0, n_inst = 0, n_tiles = 0, n_sent = 0, n_recv = 0;
  long long op_cnt[64] = {}, op_cyc[64] = {};   // [0, 32) opcodes, [32, 64) regions
  int32_t max_depth = 0, n_exitf = 0;
  // structured cond contexts (reading R20): liveness per context, valid for generation lgen_
  // (one generation per started iteration)
  static constexpr int kMaxCtx = 128;
  uint32_t lgen_ = 1;
  uint32_t lstamp_[kMaxCtx];
  int8_t lval_[kMaxCtx];
  const DCtx* ctxs_ = nullptr;   // the program's table (global memory)
  Tok* toks_;            // token table: driver-CTA shared memory when it fits, else global
  const int32_t* iv_;    // input-id table of the nodes being evaluated
  const DNode* bn_;      // current frame's body program (smem copy or global)
  DNode* sm_nodes_;      // smem staging area (nullptr: no room)
  int32_t* sm_iv_;
  volatile int* req_;    // helper-warp copy protocol (block 0 warps 1..7)

  __device__ Driver(const RunArgs& a, Tok* t, DNode* smn, int32_t* smi, volatile int* req)
      : A(a), P(a.prog), st(a.st), places_(a.prog.places), reg_(a.prog.reg),
        stack_depth_(a.stack_depth), prep_inst_(a.prep_inst), dw_count_(a.dw_count),
        acc_writer_(a.acc_writer), iter_out_(a.iter_outstanding), stacks_(a.prog.stacks),
        tas_(a.prog.tas), tab_(a.ta_base), tso_(a.ta_slot_off),
        toks_(t), iv_(a.prog.in_vids), bn_(nullptr), sm_nodes_(smn), sm_iv_(smi), req_(req) {}
  Wave* wave_ = nullptr;

  __device__ FastEnv fast_env() {
    FastEnv e;
    e.tk = (int4*)toks_;
    e.iv = iv_;
    e.it = cur_frame >= 0 ? iter : 0;   // the frame instance's own iteration (loop Merges)
    e.git = git();                       // over a nested frame's instances (branch bits)
    e.bb = P.branch_bound;
    e.bbits = A.branch_bits;
    e.lval = lval_;
    e.stacks = stacks_;
    e.depth = stack_depth_;
    e.pool = (int4*)A.stack_pool;
    e.accs = P.accs;
    e.accw = acc_writer_;
    e.tas = tas_;
    e.tab = tab_;
    e.tso = tso_;
    e.ta_writer = A.ta_writer;
    e.ta_written = A.ta_written;
    return e;
  }

  // OP_WAVE at body position pc: liveness of the contexts its nodes need, then the helper
  // warps evaluate the n nodes in parallel; leftovers go through the general evaluator.
  // Returns the number of body positions consumed (n + 1), or 1 to run the nodes serially.
  // OP_WAVE at body position pc, fused with the directly following waves (up to kMaxLev
  // levels, one helper job; the helpers separate the levels with a named barrier). A level
  // joins only if the cond contexts it reads are already known for this iteration. Returns
  // the number of body positions consumed, or 1 to run the first wave's nodes serially.
  static constexpr int kMaxLev = 16;
  // a wave job started early (by the forward LSTM node before it, overlapping the driver's
  // instance construction) and not yet finished: body position and frame iteration
  int pend_wave_pc_ = -1;
  long long pend_wave_key_ = -1;
  int cur_pc_ = 0;
  const DFrame* cur_F_ = nullptr;
  __forceinline__ __device__ long long iter_key() const {
    return ((long long)(cur_frame + 1) << 32) | (unsigned)iter;
  }
  __noinline__ __device__ int run_wave(const DFrame& F, int pc, int n) {
    if (pend_wave_pc_ >= 0) {
      const bool mine = pend_wave_pc_ == pc && pend_wave_key_ == iter_key();
      pend_wave_pc_ = -1;
      if (mine) return wave_finish(F, pc);
      wave_wait();   // (not expected) never leave a job in flight
    }
    if (!wave_start(F, pc)) return 1;
    return wave_finish(F, pc);
  }
  // forward LSTM node: its output tokens are set, so the wave job after it (skipping dead
  // twins in the other cond branch) can start while the driver builds the instance
  __device__ void start_next_wave() {
    if ((dbg_ & (1 << 27)) || !cur_F_ || pend_wave_pc_ >= 0) return;   // bit 27: off (A/B)
    const DFrame& F = *cur_F_;
    int q = cur_pc_ + 1;
    while (q < F.n_body && bn_[q].op == OP_HEAVY && bn_[q].ctx && lstamp_[bn_[q].ctx] == lgen_ &&
           lval_[bn_[q].ctx] == 0)
      ++q;
    if (q < F.n_body && bn_[q].op == OP_WAVE && wave_start(F, q)) {
      pend_wave_pc_ = q;
      pend_wave_key_ = iter_key();
    }
  }
  __device__ void wave_wait() {
    while (*(volatile int*)&wave_->done < wave_->nw) {
    }
    __threadfence_block();
  }
  // dispatch the wave job at body position pc (fused with the following waves); false: the
  // first wave's cond contexts are not known yet (run its nodes serially)
  __noinline__ __device__ bool wave_start(const DFrame& F, int pc) {
    Region rg(this, 32 + 13);
    chain_ok_ = false;
    // contexts whose liveness the wave's nodes read (bit mask from the compiler, marker imm0)
    for (int hw = 0; hw < 2; ++hw)
      for (unsigned long long m = (unsigned long long)bn_[pc].imm[hw]; m; m &= m - 1)
        if (ctx_live(64 * hw + __ffsll((long long)m) - 1) < 0) return false;
    Wave& w = *wave_;
    int nlev = 0, q = pc;
    // consecutive waves fuse into one job; a level reading cond contexts not known yet has them
    // evaluated by a helper lane after the previous level (their predicates are computed by
    // earlier levels of the same job); bit 25: no fusion, bit 31: stop at unknown contexts (A/B)
    while (true) {
      w.lev_start[nlev] = q + 1;
      w.lev_n[nlev] = bn_[q].aux[0];
      w.lev_ctx[nlev] = (unsigned long long)bn_[q].imm[0];
      w.lev_ctx_hi[nlev] = (unsigned long long)bn_[q].imm[1];
      ++nlev;
      q += bn_[q].aux[0] + 1;
      if (nlev == kMaxLev || q >= F.n_body || bn_[q].op != OP_WAVE || (dbg_ & (1 << 25))) break;
      if (dbg_ & (1 << 31)) {
        bool known = true;
        for (int hw = 0; hw < 2; ++hw)
          for (unsigned long long m = (unsigned long long)bn_[q].imm[hw]; m && known; m &= m - 1) {
            const int c = 64 * hw + __ffsll((long long)m) - 1;
            for (int x = c; x; x = ctxs_[x].parent)
              if (lstamp_[x] != lgen_) known = false;
          }
        if (!known) break;
      }
    }
    w.nlev = nlev;
    w.lev_stop = nlev;
    w.cstop = -1;
    w.nslow = 0;
    // chain the preparation of the node after the last level when it is a tensor-core LSTM
    // node whose cond context is already known to be live (saves one helper round trip)
    w.chain = 0;
    if (q < F.n_body && !(dbg_ & (1 << 24))) {   // bit 24: no chaining (A/B)
      const DNode& nx = bn_[q];
      if (nx.op == OP_HEAVY && prep_ok(nx) &&
          (nx.ctx == 0 || (lstamp_[nx.ctx] == lgen_ && lval_[nx.ctx] == 1))) {
        w.chain = 1;
        w.hd = &nx;
        w.hdead = 0;
        w.hfail = 0;
      }
    }
    w.cnt = FastCount{0, 0, 0, 0, 0};
    w.bn = bn_;
    if (w.env_frame != cur_frame) {   // the environment changes with the frame only
      w.env = fast_env();
      w.env_frame = cur_frame;
    }
    w.env.it = cur_frame >= 0 ? iter : 0;
    w.env.git = git();
    w.done = 0;
    w.skip1 = pend_batch_ ? 1 : 0;   // warp 1 still runs the batch job
    w.nw = pend_batch_ ? kWaveWarps - 1 : kWaveWarps;
    __threadfence_block();
    *(volatile int*)&w.seq = (((w.seq >> 1) + 1) << 1) | w.skip1;   // bit 0: warp 1 not in the job
    flush_publish();
    return true;
  }
  // wait for the wave job of position pc, evaluate its leftovers; positions consumed
  __noinline__ __device__ int wave_finish(const DFrame& F, int pc) {
    Wave& w = *wave_;
    const int nlev = w.nlev;
    long long wq0 = (kProfBuild && A.prof) ? clock64() : 0, wdr = 0;
    while (*(volatile int*)&w.done < w.nw) {
      long long d0 = (kProfBuild && A.prof) ? clock64() : 0;
      maybe_drain();   // the helper warps touch tokens and stacks only, never instance state
      if (kProfBuild && A.prof) wdr += clock64() - d0;
    }
    if (kProfBuild && A.prof) {   // W_WAIT: signal -> done seen; W_WAIT_DRAIN: drains inside
      op_cyc[32 + 20] += clock64() - wq0;
      op_cnt[32 + 20]++;
      op_cyc[32 + 21] += wdr;
      op_cnt[32 + 21] += w.nslow;   // count = leftover nodes
    }
    __threadfence_block();
    const int stop = w.lev_stop;   // levels completed (a level with leftovers ends the job)
    const int last = stop < nlev ? stop : nlev - 1;
    // a level the helpers could not start (context not known): resume at its marker
    const int end = w.cstop > 0 ? w.lev_start[w.cstop] - 1 : w.lev_start[last] + w.lev_n[last];
    if (w.chain && w.nslow == 0 && stop == nlev) {   // wave_->hd prepared for this iteration
      chain_ok_ = true;
      chain_key_ = ((long long)(cur_frame + 1) << 32) | (unsigned)iter;
    }
    n_push += w.cnt.push;
    n_pop += w.cnt.pop;
    if (w.cnt.maxd > max_depth) max_depth = w.cnt.maxd;
    if (w.cnt.err) {
      fail(w.cnt.err, w.cnt.err_info);
      return end - pc;
    }
    // leftovers of the last level run (e.g. a Switch whose predicate is a device value)
    for (int a = 0; a < w.nslow; ++a)
      for (int b = a + 1; b < w.nslow; ++b)
        if (w.slow[b] < w.slow[a]) {
          int t = w.slow[a];
          w.slow[a] = w.slow[b];
          w.slow[b] = t;
        }
    for (int a = 0; a < w.nslow; ++a) {
      const int q2 = w.lev_start[last] + w.slow[a];
      while (true) {
        const int r = eval(bn_[q2], P.order[F.body_off + q2]);
        if (r == EV_OK) break;
        if (r == EV_ERROR || st->error) return end - pc;
        drain();   // the predicate's producer has to finish first
      }
    }
    return end - pc;
  }

  // ---- heavy-node preparation on the helper lanes (job 1). Everything here is read-only
  // for driver bookkeeping (tokens, placements, registry, TensorArray bases; hint slots in
  // the node copy): the driver thread waits for the job and then builds the instances.
  bool chain_ok_ = false;
  long long chain_key_ = -1;
  __device__ bool prep_ok(const DNode& d) const {
    return P.precision == D_BF16 && !P.n_swaps && !(dbg_ & 128) &&
           (d.aux[0] == HK_LSTM_FWD || d.aux[0] == HK_LSTM_BWD_EW) && d.n_in <= 32 &&
           d.n_ctrl <= 32 && prep_nplace(d) <= 8;
  }
  __device__ int prep_nplace(const DNode& d) const {
    // backward: dz scratch + W^T prep; forward: W prep (+ the x-projection scratch)
    return d.n_out + (d.aux[0] == HK_LSTM_BWD_EW ? 2 : (d.aux[1] & 4) ? 2 : 1);
  }
  __device__ void heavy_prep_lane(Wave& w, int h) {
    const DNode& d = *w.hd;
    if (h < d.n_in) {
      if (in_tok(d, h).dead) atomicOr(&w.hdead, 1);
    } else if (h >= 32 && h < 32 + d.n_ctrl) {
      if (toks_[iv_[d.ctrl_off + h - 32]].dead) atomicOr(&w.hdead, 1);
    } else if (h >= 64 && h < 64 + prep_nplace(d)) {
      int64_t v = 0;
      if (!place_core(d, h - 64, &v)) atomicOr(&w.hfail, 1);
      else w.houtp[h - 64] = v;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(32 * w.nw) : "memory");
    if (w.hdead || w.hfail || h >= 5) return;
    const int64_t B = d.imm[0], In = d.imm[1], H = d.imm[2], KT = In + H;
    int16_t* hint = (int16_t*)const_cast<DNode&>(d).pad;
    int64_t p = 0;
    int rows = 0, cols = 0, kind = 0;
    if (d.aux[0] == HK_LSTM_FWD) {
      if (h == 0) { p = in_tok(d, 0).v; rows = (int)B; cols = (int)In; kind = 0; }
      else if (h == 1) { p = in_tok(d, 1).v; rows = (int)B; cols = (int)H; kind = 0; }
      else if (h == 2) { p = w.houtp[4]; rows = (int)(4 * H); cols = (int)KT; kind = 1; }
      else return;
    } else {
      if (h == 0) { p = w.houtp[5]; rows = (int)B; cols = (int)(4 * H); kind = 0; }
      else if (h == 1) { p = w.houtp[6]; rows = (int)KT; cols = (int)(4 * H); kind = 1; }
      else if (h == 2) { p = w.houtp[5]; rows = (int)B; cols = (int)(4 * H); kind = 2; }
      else if (h == 3) { p = in_tok(d, 0).v; rows = (int)B; cols = (int)In; kind = 2; }
      else { p = in_tok(d, 1).v; rows = (int)B; cols = (int)H; kind = 2; }
    }
    if (!resolve_core(p, rows, cols, kind, &w.hmap[h], &w.hslot[h], hint + h)) atomicOr(&w.hfail, 2);
  }
  // dispatch job 1 for node d and wait; the results are in *wave_
  __noinline__ __device__ void run_heavy_prep(const DNode& d) {
    Wave& w = *wave_;
    if (pend_wave_pc_ >= 0) {   // a started wave job must be finished by run_wave first
      fail(CF_E_UNSUPPORTED, -500);
      wave_wait();
      return;
    }
    w.job = 1;
    w.chain = 0;
    w.hd = &d;
    w.hdead = 0;
    w.hfail = 0;
    w.done = 0;
    w.skip1 = pend_batch_ ? 1 : 0;
    w.nw = pend_batch_ ? kWaveWarps - 1 : kWaveWarps;
    __threadfence_block();
    *(volatile int*)&w.seq = (((w.seq >> 1) + 1) << 1) | w.skip1;   // bit 0: warp 1 not in the job
    flush_publish();
    while (*(volatile int*)&w.done < w.nw) {
      maybe_drain();
    }
    __threadfence_block();
    w.job = 0;
  }

  // ask the helper warps to copy [src, src+bytes) -> dst (16 B aligned), wait for them
  __device__ void helper_copy(void* dst0, const void* src0, int64_t b0, void* dst1, const void* src1,
                              int64_t b1) {
    int64_t* q = (int64_t*)(req_ + 4);
    q[0] = (int64_t)dst0; q[1] = (int64_t)src0; q[2] = b0;
    q[3] = (int64_t)dst1; q[4] = (int64_t)src1; q[5] = b1;
    __threadfence_block();
    int seq = req_[0] + 1;
    req_[1] = 0;
    __threadfence_block();
    req_[0] = seq;
    while (req_[1] < 7) {
    }
    __threadfence_block();
  }

  __device__ void fail(int code, int64_t info) {
    if (st->error == 0) {
      st->error = code;
      st->error_info = info;
    }
  }

  __device__ Tok& tok(int vid) { return toks_[vid]; }
  __device__ const DNode& node(int id) { return P.nodes[id]; }
  __device__ int in_vid(const DNode& d, int j) { return iv_[d.in_off + j]; }
  __device__ Tok& in_tok(const DNode& d, int j) { return toks_[in_vid(d, j)]; }
  // frame-level nodes (Enter / Exit) always index the global input-id table
  __device__ Tok& in_tok_g(const DNode& d, int j) { return toks_[P.in_vids[d.in_off + j]]; }

  __device__ bool writer_done(int32_t w) { return done(w); }

  // scalar value of a token; false if its bytes are not produced yet
  __device__ bool scalar(const Tok& t, int64_t* out) {
    if (t.kind == TK_IMM) {
      *out = t.v;
      return true;
    }
    if (t.kind != TK_PTR) {
      *out = 0;
      return true;
    }
    if (!writer_done(t.writer)) return false;
    __threadfence();
    switch (t.dt) {
      case D_BOOL: *out = *(const volatile uint8_t*)t.v; break;
      case D_I32: *out = *(const volatile int32_t*)t.v; break;
      case D_I64: *out = *(const volatile int64_t*)t.v; break;
      case D_F32: {
        float f = *(const volatile float*)t.v;
        *out = (int64_t)f;
        break;
      }
      default: *out = 0;
    }
    return true;
  }

  __device__ void set_out(const DNode& d, int port, const Tok& t) { toks_[d.out_vid + port] = t; }
  __device__ void set_dead_all(const DNode& d) {
    for (int p = 0; p < d.n_out; ++p) {
      Tok t{};
      t.dead = 1;
      t.writer = -1;
      toks_[d.out_vid + p] = t;
    }
  }

  // ---------------------------------------------------------------- instances
  // ---- in-flight instance bookkeeping: a shared-memory ring indexed by id & kRingMask.
  // A slot is reused only after its previous occupant completed, so `done(w)` is simply
  // "the slot no longer holds w". Successor edges stay in global memory (written here, read
  // once at completion).
  static constexpr int kRing = 1024, kRingMask = kRing - 1;
  int32_t* r_id;     // occupant id (-1 free)
  int32_t* r_pend;   // producers outstanding
  int32_t* r_succ;   // successor edge list head
  int32_t* r_last;   // last successor added (dedupe)
  int32_t* r_nt;     // tiles
  int32_t* r_kfi;    // kind (8) | frame + 1 (8) | iter (16)

  __device__ bool done(int32_t w) const { return w < 0 || r_id[w & kRingMask] != w; }
  // per-frame iteration-counter offsets, cached (a global load on every submit/complete)
  static constexpr int kIbCache = 16;
  int32_t ib_[kIbCache];
  __device__ __forceinline__ int frame_ib(int f) const { return f < kIbCache ? ib_[f] : P.frames[f].iter_base; }
  // successors of an in-flight instance: up to kInlineSucc in shared memory (r_sn count,
  // r_sv ids), the rest in the global edge list (r_succ head)
  static constexpr int kInlineSucc = 4;
  int32_t* r_sn;
  int32_t* r_sv;
  // region profiler (profiling runs only): cycles + count into op_cyc/op_cnt[slot]
  struct Region {
    Driver* d; int slot; long long c0;
#ifdef __CUDA_ARCH__
    __device__ Region(Driver* dd, int s) : d(dd), slot(s), c0((kProfBuild && dd->A.prof) ? clock64() : 0) {}
    __device__ ~Region() {
      if (kProfBuild && d->A.prof) { d->op_cyc[slot] += clock64() - c0; d->op_cnt[slot]++; }
    }
#else
    __device__ Region(Driver* dd, int s) : d(dd), slot(s), c0(0) {}
#endif
  };

  __noinline__ __device__ int32_t new_inst(int kind, int sub, int ntiles) {
    const int32_t id = reserve_inst(kind, ntiles);
    if (id >= 0) inst_header(id, kind, sub, ntiles);
    return id;
  }
  // an instance id and its in-flight ring slot (driver-private shared-memory bookkeeping)
  __noinline__ __device__ int32_t reserve_inst(int kind, int ntiles) {
    finish_batch();
    if (ninst >= A.inst_cap) {
      fail(CF_E_STACK_BUDGET, -1);
      return -1;
    }
    int32_t id = ninst++;
    const int sl = id & kRingMask;
    if (r_id[sl] != -1) {   // ring full: wait for the oldest in-flight instance
      const long long rf0 = (kProfBuild && A.prof) ? clock64() : 0;
      while (r_id[sl] != -1) {
        const unsigned long long now = globaltimer();
        if (drain()) last_progress = now;
        else if ((long long)(now - last_progress) > A.watchdog_ns) fail(CF_E_DEADLOCK, -700);
        if (st->error) return -1;
      }
      if (kProfBuild && A.prof) { op_cyc[27] += clock64() - rf0; op_cnt[27]++; }   // RING_FULL
    }
    ntiles = max(ntiles, 1);
    r_id[sl] = id;
    r_pend[sl] = 0;
    r_succ[sl] = -1;
    r_last[sl] = -1;
    r_sn[sl] = 0;
    r_nt[sl] = ntiles;
    // iteration in the top 16 bits; 0xFFFF = read the full iteration from the record (loops
    // longer than 65534 iterations)
    // bit 7 of the kind byte: low-priority queue (root work no frame depends on)
    r_kfi[sl] = (int)((unsigned)(kind & 127) | (low_root_ ? 128u : 0u) |
                      ((unsigned)((cur_frame + 1) & 255) << 8) |
                      ((unsigned)min(cur_frame >= 0 ? iter : 0, 0xFFFF) << 16));
    return id;
  }
  // the instance record's header (global memory; also written by the helper lanes of a batch)
  __device__ void inst_header(int32_t id, int kind, int sub, int ntiles) {
    ntiles = max(ntiles, 1);
    Inst& I = A.insts[id];
    I.kind = kind;
    I.sub = sub;
    I.ntiles = ntiles;
    I.frame = cur_frame;
    I.iter = cur_frame >= 0 ? iter : 0;
    for (int j = 0; j < 14; ++j) I.p[j] = 0;
    for (int j = 0; j < 4; ++j) I.s[j] = 0;
    I.n = I.m = I.k = 0;
    I.signal = nullptr;
    if (kProfBuild && A.prof) {
      unsigned long long* pr = A.prof + 6 * (int64_t)id;
      pr[0] = globaltimer();
      pr[1] = 0;
      pr[2] = ~0ULL;
      pr[3] = 0;
      pr[4] = 0;
      pr[5] = ((unsigned long long)kind << 32) | (unsigned)ntiles;
    }
  }
  // add_dep for the helper lanes of a batch (several lanes, and the driver's own add_dep while
  // the batch is pending, register successors concurrently; no completion runs until the
  // batch is settled): shared-memory atomics, no dedupe across lanes (a repeated producer
  // just counts twice, consistently)
  __device__ void add_dep_atomic(int32_t id, int32_t w) {
    if (done(w)) return;
    const int ws = w & kRingMask;
    const int ns = atomicAdd(&r_sn[ws], 1);
    if (ns < kInlineSucc) {
      r_sv[ws * kInlineSucc + ns] = id;
    } else {
      const int32_t e = atomicAdd(&nedge, 1);
      if (e >= A.edge_cap) {
        fail(CF_E_STACK_BUDGET, -2);
        return;
      }
      A.edge_to[e] = id;
      A.edge_next[e] = atomicExch(&r_succ[ws], e);
    }
    atomicAdd(&r_pend[id & kRingMask], 1);
  }
  __forceinline__ __device__ void add_dep(int32_t id, int32_t w) {
    if (done(w)) return;
    const int ws = w & kRingMask;
    if (r_last[ws] == id) return;   // dedupe repeated inputs from the same producer
    if (pend_batch_) {   // a batch's lanes may be adding edges to the same producer right now
      r_last[ws] = id;
      add_dep_atomic(id, w);
      return;
    }
    const int ns = r_sn[ws];
    if (ns < kInlineSucc) {
      r_sv[ws * kInlineSucc + ns] = id;
      r_sn[ws] = ns + 1;
      r_last[ws] = id;
      r_pend[id & kRingMask]++;
      return;
    }
    if (nedge >= A.edge_cap) {
      fail(CF_E_STACK_BUDGET, -2);
      return;
    }
    int32_t e = nedge++;
    A.edge_to[e] = id;
    A.edge_next[e] = r_succ[ws];
    r_succ[ws] = e;
    r_sn[ws] = ns + 1;   // every successor counted (the atomic path above counts them too)
    r_last[ws] = id;
    r_pend[id & kRingMask]++;
  }
  // two rings: critical-path work (high) and filler work (low: dW chunks) so that the
  // recurrence never queues behind throughput work
  __noinline__ __device__ void publish(int32_t id) {
    const int sl = id & kRingMask;
    if ((r_kfi[sl] & 255) == HK_WAIT) {   // polled by drain() until the flag arrives
      if (n_waits_ == kMaxWaits) {   // table full: queued in order, moved in as waits complete
        if (ovf_tail_ - ovf_head_ >= kWaitOvf) {
          fail(CF_E_UNSUPPORTED, -400);
          return;
        }
        A.wait_ovf[ovf_tail_++ & (kWaitOvf - 1)] = id;
        return;
      }
      add_wait(id);
      return;
    }
    if ((r_kfi[sl] & 255) == HK_SWAP) {   // to the host I/O thread's copy streams
      const Inst& I = A.insts[id];
      unsigned long long* e = A.io_req + 4 * (io_tail & (unsigned long long)(A.io_cap - 1));
      e[0] = (unsigned long long)I.p[0];
      e[1] = (unsigned long long)I.p[13];
      e[2] = (unsigned long long)I.n;
      e[3] = (unsigned long long)(unsigned)id | ((unsigned long long)I.sub << 32);
      io_tail++;
      io_out++;
      st_release_sys_u64(A.io_req_tail, io_tail);
      return;
    }
    const bool low = (r_kfi[sl] & 255) == HK_LSTM_DW_TC || (r_kfi[sl] & 128);
    // one entry per instance; workers claim its tiles through tile_next[id]. At most kRing
    // instances are in flight, so the 2^22-entry rings never wrap onto live entries.
    if (kProfBuild && A.prof) A.prof[6 * (int64_t)id + 1] = globaltimer();
    unsigned long long* ring = low ? A.lq : A.queue;
    unsigned long long& tail = low ? lq_tail : q_tail;
    ring[tail & (A.q_cap - 1)] = (unsigned long long)id;
    tail += 1;
    // the tail is released by flush_publish() at the end of the current driver step (drain,
    // heavy node, wave): one release fence covers every instance published in the step, and
    // the record stores have mostly completed by then
    dirty_ |= low ? 2 : 1;
    if (dbg_ & 16) flush_publish();   // A/B knob: release after every publication
  }
  int dirty_ = 0;
  __forceinline__ __device__ void flush_publish() {
    if (!dirty_) return;
    // release: instance records + queue entries visible before the new tails
    if (dirty_ & 1) st_release_u64(&st->q_tail, q_tail);
    if (dirty_ & 2) st_release_u64(&st->lq_tail, lq_tail);
    dirty_ = 0;
  }
  __device__ void submit(int32_t id, bool = false) {
    if (id < 0) return;
    const int sl = id & kRingMask;
    outstanding++;
    n_inst++;
    n_tiles += r_nt[sl];
    if (cur_frame >= 0) iter_out_[frame_ib(cur_frame) + iter]++;
    if (r_pend[sl] == 0) publish(id);
  }
  __noinline__ __device__ void complete(int32_t id) {
    const int sl = id & kRingMask;
    outstanding--;
    const unsigned kfi = (unsigned)r_kfi[sl];
    const int fr = (int)((kfi >> 8) & 255) - 1;
    if (fr >= 0) {
      int it = (int)(kfi >> 16);
      if (it == 0xFFFF) it = A.insts[id].iter;
      iter_out_[frame_ib(fr) + it]--;
    }
    int32_t e = r_succ[sl];
    const int ns = min(r_sn[sl], kInlineSucc);   // helper lanes count past the inline slots
    r_id[sl] = -1;   // done
    for (int k = 0; k < ns; ++k) {
      const int32_t s2 = r_sv[sl * kInlineSucc + k];
      if (--r_pend[s2 & kRingMask] == 0) publish(s2);
    }
    while (e >= 0) {
      const int32_t s2 = A.edge_to[e];
      const int32_t nx = A.edge_next[e];
      if (--r_pend[s2 & kRingMask] == 0) publish(s2);
      e = nx;
    }
  }
  // completions of swap copies: written by the copy streams into io_cq (id + 1), possibly out
  // of order between the D2H and H2D streams; consumed slots are marked -1
  __noinline__ __device__ bool drain_io() {
    Region rg(this, 32 + 11);
    bool any = false;
    const unsigned long long m = (unsigned long long)(A.io_cap - 1);
    for (unsigned long long j = io_head; j < io_tail; ++j) {
      volatile int* p = (volatile int*)&A.io_cq[j & m];
      const int v = *p;
      if (v > 0) {
        __threadfence();
        *p = -1;
        io_out--;
        complete(v - 1);
        any = true;
      }
    }
    while (io_head < io_tail && ((volatile int*)A.io_cq)[io_head & m] == -1) {
      ((volatile int*)A.io_cq)[io_head & m] = 0;
      io_head++;
    }
    return any;
  }
  // the completion poll is an L2 round trip: on the body path it is issued at most every
  // kDrainCycles (bounds the completion latency without polling after every node)
  // measured on cfg3: 3000 cycles 84.0 ms, 6000 83.6, 12000 82.5, 24000 82.5 ms per step
  static constexpr long long kDrainCycles = 12000;
  long long drain_cycles_ = kDrainCycles;   // A/B knob: debug flags bits 8-15 (x 1000 cycles)

  long long last_drain_ = 0;
  int dbg_ = 0;
  bool low_root_ = false;   // the root step being evaluated is low priority (kRootLow)
  // dW chunk length in steps (K = chunk * B per dW tile): the compiler's P.dw_chunk, which
  // sized the dz and swap-in rings
  __device__ __forceinline__ int dw_chunk() const { return P.dw_chunk; }
  __forceinline__ __device__ void maybe_drain() {
    if ((dbg_ & 4) || clock64() - last_drain_ > drain_cycles_) drain();
  }
  __noinline__ __device__ bool drain() {
    Region rg(this, 32 + 4);
    finish_batch();   // completions must not run while a batch's lanes add edges
    last_drain_ = clock64();
    bool any = false;
    if (io_out > 0) any = drain_io();
    for (int k = 0; k < n_waits_;) {   // channel messages (Recv): flag = want, or the dead twin
      ChanWait& w = waits_[k];
      const unsigned long long f = ld_relaxed_sys_u64(w.flag);   // poll without acquire cost
      if ((f | 1) != (w.want | 1)) {
        ++k;
        continue;
      }
      __threadfence_system();   // acquire: the payload is visible before the copy is released
      if (f != w.want) {   // replicated control disagrees with the sender (reading R18)
        fail(CF_E_INVALID_GRAPH, -401);
        return true;
      }
      if (w.ack) st_release_sys_u64(w.ack, w.ackv);
      const int32_t id = w.id;
      waits_[k] = waits_[--n_waits_];
      complete(id);
      any = true;
    }
    while (n_waits_ < kMaxWaits && ovf_head_ < ovf_tail_) add_wait(A.wait_ovf[ovf_head_++ & (kWaitOvf - 1)]);
    // relaxed poll (an acquire load would invalidate L1 at every poll); the release store
    // that publishes successors orders this observation before them (fence.acq_rel).
    // (A helper warp mirroring this queue into shared memory measured 5% slower.)
    // four slots per round trip (the loads are independent): a drain that finds one
    // completion costs one L2 latency, not two
    for (int round = 0; round < 64; ++round) {
      const unsigned long long m = (unsigned long long)(A.cq_cap - 1);
      int v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = ld_volatile_i32(&A.cq[(cq_head_ + q) & m]);
      int k = 0;
      for (; k < 4 && v[k] != 0; ++k) {
        *(volatile int*)&A.cq[(cq_head_ + k) & m] = 0;
        complete(v[k] - 1);
      }
      cq_head_ += k;
      if (k) any = true;
      if (k < 4) break;
    }
    flush_publish();
    return any;
  }

  // ---------------------------------------------------------------- placement
  // code size matters on the driver's path (the I-cache is 32 KB): the placement and the
  // operand-registry lookups are out of line, returning their results in registers
  __forceinline__ __device__ bool place(const DNode& d, int port, int64_t* ptr) {
    const int64_t v = place_(d, port);
    *ptr = v;
    return v != -1;
  }
  __noinline__ __device__ int64_t place_(const DNode& d, int port) {
    int64_t r = -1;
    return place_core(d, port, &r) ? r : -1;
  }
  __forceinline__ __device__ bool place_core(const DNode& d, int port, int64_t* ptr) {
    const PlaceDesc& pl = places_[d.place_off + port];
    const int it = git();   // iteration index over all instances of a nested frame
    switch (pl.kind) {
      case PL_ROOT: *ptr = pl.base; return true;
      case PL_RING: *ptr = pl.base + (int64_t)(it % pl.slots) * pl.elem_bytes; return true;
      case PL_ARENA:
        if (it >= pl.slots) {
          fail(CF_E_STACK_BUDGET, it);
          return false;
        }
        *ptr = pl.base + (int64_t)it * pl.elem_bytes;
        return true;
      case PL_ACC: *ptr = P.accs[pl.slots].base; return true;
      case PL_SWAP: {
        // the slot now holds a new value: no stack entry is resident in it until pushed
        const int r = it % pl.slots;
        A.swap_owner[P.swaps[pl.ta].owner_off + r] = -2;
        *ptr = pl.base + (int64_t)r * pl.elem_bytes;
        return true;
      }
      case PL_TA: {
        int64_t ix;
        if (!scalar(toks_[pl.index_vid], &ix)) return false;
        const DTA& ta = tas_[pl.ta];
        if (ix < 0 || ix >= ta.size) {
          fail(CF_E_SHAPE, ix);
          return false;
        }
        *ptr = tab_[pl.ta] + ix * pl.elem_bytes;
        return true;
      }
    }
    return false;
  }
  __device__ Tok ptr_tok(int64_t p, int32_t writer, int dt) {
    Tok t{};
    t.v = p;
    t.writer = writer;
    t.kind = TK_PTR;
    t.dt = (uint8_t)dt;
    return t;
  }

  // ---------------------------------------------------------------- heavy ops
  // ---------------------------------------------------------------- operand registry
  // pointer -> (tensor map, slot) for a bf16 [rows][cols] GEMM operand; kind 0 = K-major A
  // (box 64x128), 1 = K-major B (box 64x256), 2 = MN-major (box 64x64)
  // registry entry i as the answer for (p, rows, cols)? -> slot, map
  __device__ __forceinline__ bool reg_match(int i, int64_t p, int rows, int cols, int kind, int64_t* map,
                                            int64_t* slot) {
    const DReg& r = reg_[i];
    if (r.rows != rows || r.cols != cols) return false;
    if (p < r.base || p >= r.base + (int64_t)r.slots * r.slot_bytes) return false;
    const int64_t off = p - r.base;
    int64_t q = (int64_t)((double)off * r.inv_slot);
    int64_t rem = off - q * r.slot_bytes;
    if (rem < 0) { --q; rem += r.slot_bytes; }
    else if (rem >= r.slot_bytes) { ++q; rem -= r.slot_bytes; }
    if (rem) return false;
    *slot = q;
    *map = (int64_t)((const uint8_t*)P.maps + (int64_t)(r.map0 + kind) * 128);
    return true;
  }
  // with a per-(node, operand) hint: the entry found last time is tried first (an operand of a
  // given node nearly always lives in the same ring / arena / TensorArray)
  struct MapSlot {
    int64_t map, slot;
  };
  __forceinline__ __device__ bool resolve(int64_t p, int rows, int cols, int kind, int64_t* map, int64_t* slot,
                                          int16_t* hint) {
    const MapSlot r = resolve_(p, rows, cols, kind, hint);
    *map = r.map;
    *slot = r.slot;
    return r.map != 0;
  }
  __noinline__ __device__ MapSlot resolve_(int64_t p, int rows, int cols, int kind, int16_t* hint) {
    MapSlot r{0, 0};
    if (!resolve_core(p, rows, cols, kind, &r.map, &r.slot, hint)) r.map = 0;
    return r;
  }
  // registry lookup that may miss (the generic GEMM then takes the SIMT tile)
  __noinline__ __device__ bool resolve_try(int64_t p, int rows, int cols, int kind, int64_t* map, int64_t* slot,
                                           int16_t* hint) {
    int lo = 0, hi = P.n_reg - 1, at = -1;
    while (lo <= hi) {
      const int mid = (lo + hi) >> 1;
      if (reg_[mid].base <= p) { at = mid; lo = mid + 1; } else hi = mid - 1;
    }
    for (int i = at; i >= 0 && reg_[i].base == reg_[at].base; --i)
      if (reg_match(i, p, rows, cols, kind, map, slot)) {
        *hint = (int16_t)i;
        return true;
      }
    return false;
  }
  __forceinline__ __device__ bool resolve_core(int64_t p, int rows, int cols, int kind, int64_t* map, int64_t* slot,
                                               int16_t* hint) {
    const int h = *hint;
    if (h >= 0 && h < P.n_reg && reg_match(h, p, rows, cols, kind, map, slot)) return true;
    // entries are sorted by base (host): binary search for the last base <= p, then the
    // entries sharing that base (one buffer registered under several shapes)
    int lo = 0, hi = P.n_reg - 1, at = -1;
    while (lo <= hi) {
      const int mid = (lo + hi) >> 1;
      if (reg_[mid].base <= p) { at = mid; lo = mid + 1; } else hi = mid - 1;
    }
    for (int i = at; i >= 0 && reg_[i].base == reg_[at].base; --i) {
      if (!reg_match(i, p, rows, cols, kind, map, slot)) continue;
      *hint = (int16_t)i;
      return true;
    }
    fail(CF_E_UNSUPPORTED, -100 - rows);
    return false;
  }

  __device__ int64_t pack_dts(const DNode& d, int out_dt) {
    int64_t w = 0;
    for (int j = 0; j < d.n_in && j < 8; ++j) w |= (int64_t)(in_tok(d, j).dt & 15) << (4 * j);
    w |= (int64_t)(out_dt & 15) << 32;
    return w;
  }

  // per-run weight preparation (bf16 permuted W / W^T), created on first use of the node
  // the W^T preparation of tensor-core LSTMCellGrad node nid from its root weight (value id
  // imm[3] - 1), issued as soon as the weight is available, at low priority: it runs under
  // the forward loop; the node's first gradient step finds it in prep_inst_
  // the node whose W^T preparation a gradient LSTM node shares (compiler: one per root weight)
  __device__ __forceinline__ int prep_slot(const DNode& d, int nid) const {
    return (d.imm[3] >> 32) > 0 ? (int)(d.imm[3] >> 32) - 1 : nid;
  }
  __noinline__ __device__ bool prep_early(int nid) {
    finish_batch();
    const DNode& d = node(nid);
    if (prep_inst_[nid] >= 0 || (d.imm[3] & 0xffffffffLL) <= 0) return true;
    const Tok& w = toks_[(d.imm[3] & 0xffffffffLL) - 1];
    const bool fwd = d.aux[0] == HK_LSTM_FWD;   // packed W (needed first) or W^T (low priority)
    const PlaceDesc& pl = places_[d.place_off + (fwd ? 4 : 6)];
    if (w.kind != TK_PTR || pl.kind != PL_ROOT) return true;   // the node prepares it itself
    const int64_t In = d.imm[1], H = d.imm[2], KT = In + H;
    low_root_ = !fwd;
    const int32_t id = fwd ? new_inst(HK_PREP_WP, 0, (int)((4 * H + 15) / 16))
                           : new_inst(HK_PREP_WT, 0, (int)((KT / 64) * (4 * H / 128)));
    low_root_ = false;
    if (id < 0) return false;
    Inst& I = A.insts[id];
    I.n = H;
    I.k = KT;
    I.p[0] = w.v;
    I.p[13] = pl.base;   // the node's W^T place
    add_dep(id, w.writer);
    submit(id);
    prep_inst_[nid] = id;
    return true;
  }

  __noinline__ __device__ int32_t prep(const DNode& d, int nid, int kind, int64_t dst) {
    if (prep_inst_[nid] >= 0) return prep_inst_[nid];
    const int64_t In = d.imm[1], H = d.imm[2], KT = In + H;
    int ntiles = kind == HK_PREP_WP ? (int)((4 * H + 15) / 16) : (int)((KT / 64) * (4 * H / 128));
    int32_t id = new_inst(kind, 0, ntiles);
    if (id < 0) return -1;
    Inst& I = A.insts[id];
    I.n = H;
    I.k = KT;
    I.p[0] = in_tok(d, 3).v;
    I.p[13] = dst;
    add_dep(id, in_tok(d, 3).writer);
    submit(id);
    prep_inst_[nid] = id;
    return id;
  }

  // pm / ps: operand-registry lookups already made by the helper lanes (nullptr: here)
  __noinline__ __device__ int eval_lstm_tc(const DNode& d, int nid, const int64_t* outp,
                                           const int64_t* pm = nullptr, const int64_t* ps = nullptr) {
    finish_batch();   // reads the dW / accumulator writers a pending batch may still set
    // operand-registry hints live in the (driver-private) body-program copy of the node
    int16_t* hint = (int16_t*)const_cast<DNode&>(d).pad;
    Region rg(this, 32 + 9);
    const int kind = d.aux[0];
    const bool masked = d.aux[1] & 1;
    int64_t t = 0;
    if (masked && !scalar(in_tok(d, 5), &t)) return EV_BLOCKED;
    const int64_t B = d.imm[0], In = d.imm[1], H = d.imm[2], KT = In + H;
    auto ip = [&](int j) { return in_tok(d, j).v; };
    if (kind == HK_LSTM_FWD) {
      long long q0 = (kProfBuild && A.prof) ? clock64() : 0;
      // outp / pm / ps may live in the Wave (helper results): copy them before the next wave
      // job is started below
      int64_t op_[6];
      for (int k = 0; k < 6; ++k) op_[k] = outp[k];
      int32_t pw = prep(d, prep_slot(d, nid), HK_PREP_WP, op_[4]);
      int64_t mx, sx, mh, sh, mw, sw;
      if (pm) {
        mx = pm[0]; sx = ps[0]; mh = pm[1]; sh = ps[1]; mw = pm[2]; sw = ps[2];
      } else if (!resolve(ip(0), (int)B, (int)In, 0, &mx, &sx, hint + 0) ||
                 !resolve(ip(1), (int)B, (int)H, 0, &mh, &sh, hint + 1) ||
                 !resolve(op_[4], (int)(4 * H), (int)KT, 1, &mw, &sw, hint + 2)) {
        return EV_ERROR;
      }
      long long q1 = (kProfBuild && A.prof) ? clock64() : 0;
      if (kProfBuild && A.prof) { op_cyc[32 + 14] += q1 - q0; op_cnt[32 + 14]++; }
      // 256-row tiles (tc_tile2) trade tile count for operand bytes: only for large batches;
      // the recurrence wants many short tiles (measured on cfg3)
      const bool m2 = B >= kM2MinRows;
      const bool split = d.aux[1] & 4;   // x-projection ahead of the recurrence
      const int ntiles = (int)((m2 ? (B + 255) / 256 : (B + 127) / 128) * (H / 64));
      int32_t xp = -1;
      if (split) {
        xp = new_inst(HK_LSTM_XPROJ_TC, m2 ? 2 : 0, ntiles);
        if (xp < 0) return EV_ERROR;
        Inst& X = A.insts[xp];
        X.m = B; X.k = In; X.n = H;
        X.p[0] = mx; X.p[3] = mw; X.p[7] = outp[5];
        X.s[2] = sx;
        add_dep(xp, in_tok(d, 0).writer);
        add_dep(xp, pw);
        submit(xp);
      }
      int32_t id = new_inst(HK_LSTM_FWD_TC, masked | (m2 ? 2 : 0) | (split ? 4 : 0), ntiles);
      long long q2 = (kProfBuild && A.prof) ? clock64() : 0;
      if (kProfBuild && A.prof) { op_cyc[32 + 15] += q2 - q1; op_cnt[32 + 15]++; }
      if (id < 0) return EV_ERROR;
      // tokens first: the next wave job then overlaps this instance's construction
      set_out(d, 0, ptr_tok(op_[0], id, D_BF16));
      set_out(d, 1, ptr_tok(op_[1], id, D_F32));
      set_out(d, 2, ptr_tok(op_[2], id, D_BF16));
      set_out(d, 3, ptr_tok(op_[3], id, D_BF16));
      toks_[d.ctrl_vid] = Tok{0, -1, 0, TK_FLOW, 0, 0};
      start_next_wave();
      Inst& I = A.insts[id];
      I.m = B; I.k = In; I.n = H;
      I.p[0] = mx; I.p[1] = mh; I.p[2] = ip(2); I.p[3] = mw; I.p[4] = ip(4);
      I.p[5] = masked ? ip(6) : 0;
      I.p[6] = ip(1);
      for (int p = 0; p < 4; ++p) I.p[8 + p] = op_[p];
      I.s[0] = t; I.s[1] = d.aux[2]; I.s[2] = sx; I.s[3] = sh;
      if (split) I.p[7] = op_[5];
      long long q3 = (kProfBuild && A.prof) ? clock64() : 0;
      if (kProfBuild && A.prof) { op_cyc[32 + 16] += q3 - q2; op_cnt[32 + 16]++; }
      for (int j = 0; j < d.n_in; ++j)
        if (!(split && j == 0)) add_dep(id, in_tok(d, j).writer);   // x: through the projection
      add_dep(id, pw);
      add_dep(id, xp);
      long long q4 = (kProfBuild && A.prof) ? clock64() : 0;
      if (kProfBuild && A.prof) { op_cyc[32 + 17] += q4 - q3; op_cnt[32 + 17]++; }
      submit(id);
      if (kProfBuild && A.prof) { op_cyc[32 + 18] += clock64() - q4; op_cnt[32 + 18]++; }
      return EV_OK;
    }
    // ---- backward: EW (dz, dc, db partials) -> DXH (dx, dh) and DW (dW, db). On steps that
    // do not close a dW chunk (7 of 8 when the gradients accumulate in place) the ids and
    // tokens come first and the next wave job overlaps the records and dependency edges.
    int64_t op_[7];
    for (int k = 0; k < 7; ++k) op_[k] = outp[k];   // may live in the Wave (helper results)
    outp = op_;
    const int acc_w = d.aux[3], acc_b = d.aux[4];
    const int cnt0 = dw_count_[nid];
    const bool early = !(dbg_ & (1 << 29)) && acc_w >= 0 && acc_b >= 0 && cnt0 + 1 < dw_chunk();   // bit 29: off
    const int o = masked ? 7 : 5;
    const int64_t dz_ptr = outp[5];
    const int64_t dz_bytes = ((B * 4 * H * 2 + 1023) / 1024) * 1024;
    int32_t pw = prep(d, prep_slot(d, nid), HK_PREP_WT, outp[6]);
    int64_t mz, sz, mwt, swt, mzn, szn, mxn, sxn, mhn, shn;
    if (pm) {
      mz = pm[0]; sz = ps[0]; mwt = pm[1]; swt = ps[1]; mzn = pm[2]; szn = ps[2];
      mxn = pm[3]; sxn = ps[3]; mhn = pm[4]; shn = ps[4];
    } else if (!resolve(dz_ptr, (int)B, (int)(4 * H), 0, &mz, &sz, hint + 0) ||
               !resolve(outp[6], (int)KT, (int)(4 * H), 1, &mwt, &swt, hint + 1) ||
               !resolve(dz_ptr, (int)B, (int)(4 * H), 2, &mzn, &szn, hint + 2) ||
               !resolve(ip(0), (int)B, (int)In, 2, &mxn, &sxn, hint + 3) ||
               !resolve(ip(1), (int)B, (int)H, 2, &mhn, &shn, hint + 4)) {
      return EV_ERROR;
    }
    int32_t e = new_inst(HK_LSTM_BWD_EW_BF, masked, (int)(((B + 127) / 128) * ((H + kEwUnits - 1) / kEwUnits)));
    if (e < 0) return EV_ERROR;
    const bool m2 = B >= kM2MinRows;
    int32_t x = new_inst(HK_LSTM_DXH_TC, masked | (m2 ? 2 : 0),
                         (int)((m2 ? (B + 255) / 256 : (B + 127) / 128) * (m2 ? KT / kDxhN2 : KT / 256)));
    if (x < 0) return EV_ERROR;
    if (early) {
      set_out(d, 0, ptr_tok(outp[0], x, D_F32));
      set_out(d, 1, ptr_tok(outp[1], x, D_F32));
      set_out(d, 2, ptr_tok(outp[2], e, D_F32));
      set_out(d, 3, ptr_tok(outp[3], acc_writer_[acc_w], D_F32));
      set_out(d, 4, ptr_tok(outp[4], acc_writer_[acc_b], D_F32));
      toks_[d.ctrl_vid] = Tok{0, -1, 0, TK_FLOW, 0, 0};
      start_next_wave();
    }
    {
      Inst& I = A.insts[e];
      I.m = B; I.k = In; I.n = H;
      I.p[2] = ip(2); I.p[4] = ip(4); I.p[5] = masked ? ip(6) : 0;
      I.p[6] = ip(o); I.p[7] = ip(o + 1); I.p[8] = ip(o + 2);
      {   // folded AddN terms of dout (appended inputs)
        const int nx = d.aux[5], base = d.n_in - nx;
        I.p[14] = nx > 0 ? ip(base) : 0;
        I.p[15] = nx > 1 ? ip(base + 1) : 0;
      }
      I.p[9] = outp[2]; I.p[10] = dz_ptr;
      I.s[0] = t; I.s[4] = in_tok(d, o + 2).dt; I.s[5] = dz_bytes;
      for (int j = 0; j < d.n_in; ++j) add_dep(e, in_tok(d, j).writer);
    }
    {
      Inst& I = A.insts[x];
      I.m = B; I.k = In; I.n = H;
      I.p[0] = mz; I.p[1] = mwt; I.p[5] = masked ? ip(6) : 0; I.p[6] = ip(o);
      I.p[11] = outp[0]; I.p[12] = outp[1];
      I.s[0] = t; I.s[2] = sz;
      add_dep(x, e);
      add_dep(x, pw);
      add_dep(x, in_tok(d, o).writer);
    }
    // dW / db: steps are queued and multiplied in chunks of up to P.dw_chunk (K = 8 B) when both
    // gradients accumulate in place; otherwise one step per instance
    {
      int cnt = dw_count_[nid];
      int64_t* rec = A.dw_pend + ((int64_t)nid * kDwMax + cnt) * 10;
      rec[0] = szn; rec[1] = mxn; rec[2] = sxn; rec[3] = mhn; rec[4] = shn;
      rec[5] = dz_ptr + dz_bytes;
      rec[6] = e; rec[7] = in_tok(d, 0).writer; rec[8] = in_tok(d, 1).writer;
      A.dw_pend[(int64_t)nid * kDwMax * 10 + 9] = mzn;   // dz map (same for all steps of the node)
      dw_count_[nid] = cnt + 1;
      pend_mz = mzn;
      if (!(acc_w >= 0 && acc_b >= 0) || cnt + 1 >= dw_chunk()) {
        if (flush_dw(d, nid, mzn, outp[3], outp[4]) < 0) return EV_ERROR;
      }
    }
    if (!early) {
      set_out(d, 0, ptr_tok(outp[0], x, D_F32));
      set_out(d, 1, ptr_tok(outp[1], x, D_F32));
      set_out(d, 2, ptr_tok(outp[2], e, D_F32));
      set_out(d, 3, ptr_tok(outp[3], acc_w >= 0 ? acc_writer_[acc_w] : last_dw, D_F32));
      set_out(d, 4, ptr_tok(outp[4], acc_b >= 0 ? acc_writer_[acc_b] : last_dw, D_F32));
    }
    submit(e);
    submit(x);
    return EV_OK;
  }

  // ---------------------------------------------------------------- heavy batches
  // OP_HEAVY_BATCH at body position pc: the next n nodes are tensor-core LSTM nodes of one
  // phase (compiler.cpp form_waves): every input is ready before the marker or an output of an
  // earlier member. The driver thread checks liveness and reserves the instance ids; helper
  // warp 1 builds all members at once (lane m = member m: placements and output tokens, then
  // operand-registry lookups, records and dependency edges); the driver then submits. Returns
  // the body positions consumed: n + 1, or 1 when the members must go through the general
  // path one by one (a context or a scalar not known yet, a dead member, a pending wave job).
  // settle the batch job in flight (job 3): wait for its lanes, then account its instances
  bool pend_batch_ = false;
  __noinline__ __device__ void finish_batch() {
    if (!pend_batch_) return;
    Wave& w = *wave_;
    while (*(volatile int*)&w.bdone == 0) {
    }
    __threadfence_block();
    pend_batch_ = false;
    if (kProfBuild && A.prof) {   // lane-0 clocks: wake, checks, reserve, placements,
      const long long now = clock64();   // records + edges (slowest lane), settle
      op_cyc[28] += w.bt_start - w.bt_issue; op_cyc[29] += w.bt_chk - w.bt_start;
      op_cyc[30] += w.bt_res - w.bt_chk;
      op_cyc[32 + 25] += w.bt_a - w.bt_res;
      op_cyc[32 + 26] += (long long)w.bt_end - w.bt_a;
      op_cyc[32 + 27] += now - (long long)w.bt_end;
      op_cnt[28]++; op_cnt[29]++; op_cnt[30]++;
      op_cnt[32 + 25]++; op_cnt[32 + 26]++; op_cnt[32 + 27]++;
    }
    n_tiles += w.btiles;
    n_dead += w.bdead;
    if (w.blast >= 0) last_dw = w.blast;
    dirty_ |= w.bdirty;
    flush_publish();
    if (w.bfail && !st->error) fail(CF_E_UNSUPPORTED, -600);
  }

  __noinline__ __device__ int run_batch(const DFrame& F, int pc, int n) {
    Region rg(this, 32 + 23);
    const long long bt_enter = (kProfBuild && A.prof) ? clock64() : 0;
    finish_batch();
    if (pend_wave_pc_ >= 0 || P.precision != D_BF16 || P.n_swaps || (dbg_ & (1 << 30))) return 1;
    Wave& w = *wave_;
    if (!(dbg_ & (1 << 28)) && n <= 32) {
      // the whole batch on helper warp 1, lane m = member m (job 3, batch_lane_par): liveness,
      // id reservation, placements and tokens, records and edges, submission. The driver thread
      // only makes sure every member's cond context is known, waits, and adds the totals.
      // (Debug flag bit 28: the serial path below, A/B.)
      for (int m = 0; m < n; ++m) {
        const int c = bn_[pc + 1 + m].ctx;
        if (c && !(lstamp_[c] == lgen_ && lval_[c] >= 0) && ctx_live(c) < 0) return 1;
      }
      flush_publish();   // before the lanes start appending to the queues
      w.bpc = pc + 1;
      w.bcount = n;
      w.bfail = 0;
      w.bphase = 0;
      w.bdone = 0;
      w.bgo = 0;
      w.bbase = ninst;
      w.bfoff = F.body_off;
      w.bids = w.btiles = w.bdead = w.bdirty = 0;
      w.blast = -1;
      if (kProfBuild && A.prof) {
        w.bt_end = 0;
        w.bt_issue = clock64();
      }
      __threadfence_block();
      *(volatile int*)&w.bseq = w.bseq + 1;
      // the member tokens are set once phase A is done; the records, edges and submissions
      // finish while the driver goes on with the routing (finish_batch settles them before
      // anything reads or changes instance state). Until then the lanes only read tokens and
      // claim free ring slots, so completions may still be processed meanwhile
      while (*(volatile int*)&w.bphase == 0) {
        maybe_drain();
      }
      __threadfence_block();
      *(volatile int*)&w.bgo = 1;   // no completion runs from here until finish_batch
      if (w.bphase == 2) {   // a member needs the general path; nothing was changed
        while (*(volatile int*)&w.bdone == 0) {
        }
        __threadfence_block();
      } else {
        // the ids and the iteration's outstanding count now; tiles and queue state at settling
        ninst += w.bids;
        outstanding += w.bids;
        n_inst += w.bids;
        if (cur_frame >= 0) iter_out_[frame_ib(cur_frame) + iter] += w.bids;
        pend_batch_ = true;
        if (tc::kKnobs[1]) finish_batch();   // A/B knob 1: no overlap
        return n + 1;
      }
    }
    // liveness: contexts first (no state is changed before every member is known)
    unsigned live = 0;
    for (int m = 0; m < n; ++m) {
      const DNode& d = bn_[pc + 1 + m];
      int l = 1;
      if (d.ctx) {
        l = lstamp_[d.ctx] == lgen_ && lval_[d.ctx] >= 0 ? lval_[d.ctx] : ctx_live(d.ctx);
        if (l < 0) return 1;
      }
      if (!l) continue;
      // inputs that are not earlier members' outputs, and control inputs, must be live; the
      // masked cells' time step must be an immediate
      const unsigned inb = (unsigned)d.aux[6];
      for (int j = 0; j < d.n_in; ++j)
        if (!(inb >> j & 1) && in_tok(d, j).dead) return 1;
      for (int j = 0; j < d.n_ctrl; ++j)
        if (toks_[iv_[d.ctrl_off + j]].dead) return 1;
      if ((d.aux[1] & 1) && in_tok(d, 5).kind != TK_IMM) return 1;
      live |= 1u << m;
    }
    const long long bt_live = (kProfBuild && A.prof) ? clock64() : 0;
    // reserve the ids (ring slots: may drain completions, so before the helpers start)
    const bool m2rows = bn_[pc + 1].imm[0] >= kM2MinRows;
    int32_t last_flush = -1;
    for (int m = 0; m < n; ++m) {
      int* id = w.bid[m];
      id[0] = id[1] = id[2] = id[3] = -1;
      if (!(live >> m & 1)) {
        n_dead++;
        continue;
      }
      const DNode& d = bn_[pc + 1 + m];
      const int nid = ((const int16_t*)d.pad)[5] >= 0 ? ((const int16_t*)d.pad)[5] : P.order[F.body_off + pc + 1 + m];
      w.bnid[m] = nid;
      const int64_t B = d.imm[0], In = d.imm[1], H = d.imm[2], KT = In + H;
      const bool masked = d.aux[1] & 1;
      const bool m2 = B >= kM2MinRows;
      (void)m2rows;
      if (d.aux[0] == HK_LSTM_FWD) {
        const int ps = prep_slot(d, nid);   // shared with the other nodes of its weight
        if (prep_inst_[ps] < 0) {
          id[3] = reserve_inst(HK_PREP_WP, (int)((4 * H + 15) / 16));
          prep_inst_[ps] = id[3];
        }
        const int nt = (int)((m2 ? (B + 255) / 256 : (B + 127) / 128) * (H / 64));
        if (d.aux[1] & 4) id[1] = reserve_inst(HK_LSTM_XPROJ_TC, nt);   // x-projection first
        id[0] = reserve_inst(HK_LSTM_FWD_TC, nt);
      } else {
        const int ps = prep_slot(d, nid);   // shared with the other nodes of its weight
        if (prep_inst_[ps] < 0) {
          id[3] = reserve_inst(HK_PREP_WT, (int)((KT / 64) * (4 * H / 128)));
          prep_inst_[ps] = id[3];
        }
        const int acc_w = d.aux[3], acc_b = d.aux[4];
        if (!(acc_w >= 0 && acc_b >= 0) || dw_count_[nid] + 1 >= dw_chunk()) {
          id[2] = reserve_inst(HK_LSTM_DW_TC, (int)((4 * H / 256) * (KT / 256) + (4 * H + 255) / 256));
          last_flush = id[2];
        }
        id[0] = reserve_inst(HK_LSTM_BWD_EW_BF, (int)(((B + 127) / 128) * ((H + kEwUnits - 1) / kEwUnits)));
        id[1] = reserve_inst(HK_LSTM_DXH_TC, (int)((m2 ? (B + 255) / 256 : (B + 127) / 128) * (m2 ? KT / kDxhN2 : KT / 256)));
      }
      (void)masked;
      if (st->error) return n + 1;
    }
    w.job = 2;
    w.bpc = pc + 1;
    w.bcount = n;
    w.bfail = 0;
    w.chain = 0;
    w.done = 0;
    w.nw = kWaveWarps;
    w.skip1 = 0;
    if (kProfBuild && A.prof) {
      w.bt_end = 0;
      w.bt_issue = clock64();
    }
    __threadfence_block();
    *(volatile int*)&w.seq = (((w.seq >> 1) + 1) << 1) | w.skip1;   // bit 0: warp 1 not in the job
    flush_publish();
    while (*(volatile int*)&w.done < kWaveWarps) {
    }
    __threadfence_block();
    if (kProfBuild && A.prof) {   // B_PHASE_A, B_BUILD (slowest lane; wake-up + tail < 1 us)
      op_cyc[32 + 25] += w.bt_a - w.bt_issue;
      op_cyc[32 + 26] += (long long)w.bt_end - w.bt_a;
      op_cyc[32 + 24] += w.bt_issue - bt_live; op_cyc[32 + 27] += bt_live - bt_enter;
      for (int k = 24; k < 28; ++k) op_cnt[32 + k]++;
    }
    const long long bt_post = (kProfBuild && A.prof) ? clock64() : 0;
    w.job = 0;
    if (w.bfail && !st->error) fail(CF_E_UNSUPPORTED, -600);
    if (last_flush >= 0) last_dw = last_flush;
    // submit in creation order (weight prep, dW chunk, then the members' own instances)
    for (int m = 0; m < n; ++m) {
      const int* id = w.bid[m];
      const bool fwd = bn_[pc + 1 + m].aux[0] == HK_LSTM_FWD;
      if (id[3] >= 0) submit(id[3]);
      if (id[2] >= 0) submit(id[2], true);
      if (fwd && id[1] >= 0) submit(id[1]);   // the x-projection before its cell
      if (id[0] >= 0) submit(id[0]);
      if (!fwd && id[1] >= 0) submit(id[1]);
    }
    flush_publish();
    if (kProfBuild && A.prof) { op_cyc[32 + 28] += clock64() - bt_post; op_cnt[32 + 28]++; }
    return n + 1;
  }

  // helper lane m of warp 1: member m of the batch dispatched by run_batch
  __device__ void batch_lane(Wave& w, int m, bool signal_a = false) {
    if (kProfBuild && A.prof && m == 0 && w.job == 2) w.bt_start = clock64();
    const bool mine = m < w.bcount && w.bid[m][0] >= 0;
    const DNode* dp = mine ? &bn_[w.bpc + m] : nullptr;
    int64_t outp[8];
    bool ok = true;
    // phase A: placements and output tokens (later members read them in phase B)
    if (mine) {
      const DNode& d = *dp;
      const int np = prep_nplace(d);
      for (int q = 0; q < np; ++q)
        if (!place_core(d, q, &outp[q])) ok = false;
      const int* id = w.bid[m];
      if (ok) {
        if (d.aux[0] == HK_LSTM_FWD) {
          set_out(d, 0, ptr_tok(outp[0], id[0], D_BF16));
          set_out(d, 1, ptr_tok(outp[1], id[0], D_F32));
          set_out(d, 2, ptr_tok(outp[2], id[0], D_BF16));
          set_out(d, 3, ptr_tok(outp[3], id[0], D_BF16));
        } else {
          const int acc_w = d.aux[3], acc_b = d.aux[4];
          set_out(d, 0, ptr_tok(outp[0], id[1], D_F32));
          set_out(d, 1, ptr_tok(outp[1], id[1], D_F32));
          set_out(d, 2, ptr_tok(outp[2], id[0], D_F32));
          set_out(d, 3, ptr_tok(outp[3], id[2] >= 0 ? id[2] : acc_writer_[acc_w], D_F32));
          set_out(d, 4, ptr_tok(outp[4], id[2] >= 0 ? id[2] : acc_writer_[acc_b], D_F32));
        }
        toks_[d.ctrl_vid] = Tok{0, -1, 0, TK_FLOW, 0, 0};
      }
    }
    __syncwarp();
    if (kProfBuild && A.prof && m == 0) w.bt_a = clock64();
    if (signal_a) {   // the members' output tokens are set: the driver may go on
      __threadfence_block();
      if (m == 0) {
        *(volatile int*)&w.bphase = 1;
        // edges only once the driver has left its completion polling (it drains while it
        // waits for phase A; a completion walking a successor list must not meet a new edge)
        while (*(volatile int*)&w.bgo == 0) {
        }
      }
      __syncwarp();
      __threadfence_block();
    }
    // phase B: operand lookups, records, dependency edges
    if (mine && ok) ok = batch_build(*dp, w.bnid[m], w.bid[m], outp);
    if (mine && !ok) atomicOr(&w.bfail, 1);
    if (kProfBuild && A.prof) atomicMax(&w.bt_end, (unsigned long long)clock64());
    __syncwarp();
  }

  // job 3: lane m of helper warp 1 runs member m of the batch end to end. Nothing is changed
  // until every lane has checked its member (a dead input, a control token or a time step not
  // known yet, or an occupied ring slot hands the whole batch back to the driver: bfail = 2).
  // While the lanes run, the driver thread only waits: no completion is processed, so the
  // dependency edges (shared-memory atomics) and the submissions cannot race with one.
  __device__ void batch_lane_par(Wave& w, int m) {
    const unsigned full = 0xffffffffu;
    if (kProfBuild && A.prof && m == 0) w.bt_start = clock64();
    const int n = w.bcount;
    const bool in = m < n;
    const DNode* dp = in ? &bn_[w.bpc + m] : nullptr;
    // ---- checks (read only)
    int live = 0, bad = 0, nid = -1, cnt = 0;
    bool fwd = false, prep = false, xp = false, flush = false;
    if (in) {
      const DNode& d = *dp;
      live = d.ctx ? lval_[d.ctx] : 1;
      if (live) {
        const unsigned inb = (unsigned)d.aux[6];
        for (int j = 0; j < d.n_in; ++j)
          if (!(inb >> j & 1) && in_tok(d, j).dead) bad = 1;
        for (int j = 0; j < d.n_ctrl; ++j)
          if (toks_[iv_[d.ctrl_off + j]].dead) bad = 1;
        if ((d.aux[1] & 1) && in_tok(d, 5).kind != TK_IMM) bad = 1;
        nid = ((const int16_t*)d.pad)[5] >= 0 ? ((const int16_t*)d.pad)[5] : P.order[w.bfoff + w.bpc + m];
        fwd = d.aux[0] == HK_LSTM_FWD;
        prep = prep_inst_[prep_slot(d, nid)] < 0;
        if (fwd) {
          xp = d.aux[1] & 4;
        } else {
          const int acc_w = d.aux[3], acc_b = d.aux[4];
          flush = !(acc_w >= 0 && acc_b >= 0) || dw_count_[nid] + 1 >= dw_chunk();
        }
        cnt = 1 + (prep ? 1 : 0) + (fwd ? (xp ? 1 : 0) : 1 + (flush ? 1 : 0));
      }
    }
    // ids: consecutive per member, members in order (the serial path's numbering)
    int off = cnt;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      const int v = __shfl_up_sync(full, off, k);
      if (m >= k) off += v;
    }
    const int total = __shfl_sync(full, off, 31);
    if (kProfBuild && A.prof && m == 0) w.bt_chk = clock64();
    off -= cnt;
    int first = w.bbase + off;
    for (int k = 0; k < cnt; ++k)
      if (r_id[(first + k) & kRingMask] != -1 || first + k >= A.inst_cap) bad = 1;
    if (__any_sync(full, bad)) {   // handed back: nothing changed, the job is over
      if (m == 0) w.bfail = 2;
      __syncwarp();
      __threadfence_block();
      if (m == 0) {
        *(volatile int*)&w.bdone = 1;
        *(volatile int*)&w.bphase = 2;
      }
      return;
    }
    // ---- reserve (the serial path's order: weight prep, dW chunk / x-projection, main)
    int* id = in ? w.bid[m] : nullptr;
    int tiles = 0;
    if (in) {
      id[0] = id[1] = id[2] = id[3] = -1;
      if (!live) {
        atomicAdd(&w.bdead, 1);
      } else {
        const DNode& d = *dp;
        w.bnid[m] = nid;
        const int64_t B = d.imm[0], In = d.imm[1], H = d.imm[2], KT = In + H;
        const bool m2 = B >= kM2MinRows;
        auto take = [&](int kind, int nt) {
          const int32_t x = first++;
          const int sl = x & kRingMask;
          nt = max(nt, 1);
          r_id[sl] = x;
          r_pend[sl] = 0;
          r_succ[sl] = -1;
          r_last[sl] = -1;
          r_sn[sl] = 0;
          r_nt[sl] = nt;
          r_kfi[sl] = (int)((unsigned)(kind & 127) | ((unsigned)((cur_frame + 1) & 255) << 8) |
                            ((unsigned)min(cur_frame >= 0 ? iter : 0, 0xFFFF) << 16));
          tiles += nt;
          return x;
        };
        if (fwd) {
          if (prep) {
            id[3] = take(HK_PREP_WP, (int)((4 * H + 15) / 16));
            prep_inst_[prep_slot(d, nid)] = id[3];
          }
          const int nt = (int)((m2 ? (B + 255) / 256 : (B + 127) / 128) * (H / 64));
          if (xp) id[1] = take(HK_LSTM_XPROJ_TC, nt);
          id[0] = take(HK_LSTM_FWD_TC, nt);
        } else {
          if (prep) {
            id[3] = take(HK_PREP_WT, (int)((KT / 64) * (4 * H / 128)));
            prep_inst_[prep_slot(d, nid)] = id[3];
          }
          if (flush) {
            id[2] = take(HK_LSTM_DW_TC, (int)((4 * H / 256) * (KT / 256) + (4 * H + 255) / 256));
            atomicMax(&w.blast, id[2]);
          }
          id[0] = take(HK_LSTM_BWD_EW_BF, (int)(((B + 127) / 128) * ((H + kEwUnits - 1) / kEwUnits)));
          id[1] = take(HK_LSTM_DXH_TC, (int)((m2 ? (B + 255) / 256 : (B + 127) / 128) *
                                              (m2 ? KT / kDxhN2 : KT / 256)));
        }
      }
    }
    if (m == 0) {
      w.bids = total;
      w.bcount = n;
    }
    __syncwarp();
    if (kProfBuild && A.prof && m == 0) w.bt_res = clock64();
    // ---- placements, tokens, records, edges (the job-2 lanes' code; phase A done -> bphase)
    batch_lane(w, m, true);
    if (kProfBuild && A.prof && m == 0) w.bt_built = clock64();
    // ---- submit (every member's edges exist: each lane adds only its own instances' edges)
    if (in && live) {
      int dirty = 0;
      auto sub = [&](int x) {
        if (x < 0) return;
        if (r_pend[x & kRingMask] != 0) return;
        const int sl = x & kRingMask;
        const bool low = (r_kfi[sl] & 255) == HK_LSTM_DW_TC;
        if (kProfBuild && A.prof) A.prof[6 * (int64_t)x + 1] = globaltimer();
        const unsigned long long t = atomicAdd(low ? &lq_tail : &q_tail, 1ULL);
        (low ? A.lq : A.queue)[t & (A.q_cap - 1)] = (unsigned long long)x;
        dirty |= low ? 2 : 1;
      };
      sub(id[3]);
      sub(id[2]);
      if (fwd) sub(id[1]);
      sub(id[0]);
      if (!fwd) sub(id[1]);
      if (dirty) atomicOr(&w.bdirty, dirty);
      atomicAdd(&w.btiles, tiles);
    }
    __syncwarp();
    __threadfence_block();
    if (m == 0) *(volatile int*)&w.bdone = 1;
  }

  __device__ bool batch_build(const DNode& d, int nid, const int* id, const int64_t* outp) {
    int16_t* hint = (int16_t*)const_cast<DNode&>(d).pad;
    const bool masked = d.aux[1] & 1;
    const int64_t t = masked ? in_tok(d, 5).v : 0;
    const int64_t B = d.imm[0], In = d.imm[1], H = d.imm[2], KT = In + H;
    const bool m2 = B >= kM2MinRows;
    auto ip = [&](int j) { return in_tok(d, j).v; };
    // the same dependency added twice by one lane is counted once
    int32_t seen[12];
    int ns = 0;
    auto dep = [&](int32_t idd, int32_t wr) {
      if (wr < 0) return;
      for (int k = 0; k < ns; ++k)
        if (seen[k] == wr) return;
      if (ns < 12) seen[ns++] = wr;
      add_dep_atomic(idd, wr);
    };
    if (d.aux[0] == HK_LSTM_FWD) {
      int32_t pw = prep_inst_[prep_slot(d, nid)];
      if (id[3] >= 0) {   // per-run weight preparation (gate-interleaved bf16 W)
        inst_header(id[3], HK_PREP_WP, 0, (int)((4 * H + 15) / 16));
        Inst& Q = A.insts[id[3]];
        Q.n = H;
        Q.k = KT;
        Q.p[0] = in_tok(d, 3).v;
        Q.p[13] = outp[4];
        add_dep_atomic(id[3], in_tok(d, 3).writer);
      }
      const bool pl0 = kProfBuild && A.prof && (threadIdx.x & 31) == 0;
      long long c0 = pl0 ? clock64() : 0;
      int64_t mx, sx, mh, sh, mw, sw;
      if (!resolve_core(ip(0), (int)B, (int)In, 0, &mx, &sx, hint + 0) ||
          !resolve_core(ip(1), (int)B, (int)H, 0, &mh, &sh, hint + 1) ||
          !resolve_core(outp[4], (int)(4 * H), (int)KT, 1, &mw, &sw, hint + 2))
        return false;
      long long c1 = pl0 ? clock64() : 0;
      const int ntiles = (int)((m2 ? (B + 255) / 256 : (B + 127) / 128) * (H / 64));
      const bool split = id[1] >= 0;
      if (split) {   // x-projection ahead of the recurrence (HK_LSTM_XPROJ_TC)
        inst_header(id[1], HK_LSTM_XPROJ_TC, m2 ? 2 : 0, ntiles);
        Inst& X = A.insts[id[1]];
        X.m = B; X.k = In; X.n = H;
        X.p[0] = mx; X.p[3] = mw; X.p[7] = outp[5];
        X.s[2] = sx;
        add_dep_atomic(id[1], in_tok(d, 0).writer);
        add_dep_atomic(id[1], pw);
      }
      inst_header(id[0], HK_LSTM_FWD_TC, masked | (m2 ? 2 : 0) | (split ? 4 : 0), ntiles);
      Inst& I = A.insts[id[0]];
      I.m = B; I.k = In; I.n = H;
      I.p[0] = mx; I.p[1] = mh; I.p[2] = ip(2); I.p[3] = mw; I.p[4] = ip(4);
      I.p[5] = masked ? ip(6) : 0;
      I.p[6] = ip(1);
      I.p[7] = split ? outp[5] : 0;
      for (int q = 0; q < 4; ++q) I.p[8 + q] = outp[q];
      I.s[0] = t; I.s[1] = d.aux[2]; I.s[2] = sx; I.s[3] = sh;
      long long c2 = pl0 ? clock64() : 0;
      for (int j = 0; j < d.n_in; ++j)
        if (!(split && j == 0)) dep(id[0], in_tok(d, j).writer);   // x: through the projection
      dep(id[0], pw);
      if (split) dep(id[0], id[1]);
      if (pl0) {   // B_F_RECORD (lookups + record), B_F_DEPS (lane 0 of the batch)
        const long long c3 = clock64();
        op_cyc[32 + 29] += c2 - c0; op_cyc[63] += c3 - c2;
        op_cnt[32 + 29]++; op_cnt[63]++;
      }
      return true;
    }
    // backward: EW (dz, dc, db partials) -> DXH (dx, dh); dW / db chunked over 8 steps
    const int acc_w = d.aux[3], acc_b = d.aux[4];
    const int o = masked ? 7 : 5;
    const int64_t dz_ptr = outp[5];
    const int64_t dz_bytes = ((B * 4 * H * 2 + 1023) / 1024) * 1024;
    const int32_t pw = prep_inst_[prep_slot(d, nid)];
    if (id[3] >= 0) {   // per-run weight preparation (bf16 W^T)
      inst_header(id[3], HK_PREP_WT, 0, (int)((KT / 64) * (4 * H / 128)));
      Inst& Q = A.insts[id[3]];
      Q.n = H;
      Q.k = KT;
      Q.p[0] = in_tok(d, 3).v;
      Q.p[13] = outp[6];
      add_dep_atomic(id[3], in_tok(d, 3).writer);
    }
    int64_t mz, sz, mwt, swt, mzn, szn, mxn, sxn, mhn, shn;
    if (!resolve_core(dz_ptr, (int)B, (int)(4 * H), 0, &mz, &sz, hint + 0) ||
        !resolve_core(outp[6], (int)KT, (int)(4 * H), 1, &mwt, &swt, hint + 1) ||
        !resolve_core(dz_ptr, (int)B, (int)(4 * H), 2, &mzn, &szn, hint + 2) ||
        !resolve_core(ip(0), (int)B, (int)In, 2, &mxn, &sxn, hint + 3) ||
        !resolve_core(ip(1), (int)B, (int)H, 2, &mhn, &shn, hint + 4))
      return false;
    const int32_t e = id[0], x = id[1];
    inst_header(e, HK_LSTM_BWD_EW_BF, masked, (int)(((B + 127) / 128) * ((H + kEwUnits - 1) / kEwUnits)));
    inst_header(x, HK_LSTM_DXH_TC, masked | (m2 ? 2 : 0),
                (int)((m2 ? (B + 255) / 256 : (B + 127) / 128) * (m2 ? KT / kDxhN2 : KT / 256)));
    {
      Inst& I = A.insts[e];
      I.m = B; I.k = In; I.n = H;
      I.p[2] = ip(2); I.p[4] = ip(4); I.p[5] = masked ? ip(6) : 0;
      I.p[6] = ip(o); I.p[7] = ip(o + 1); I.p[8] = ip(o + 2);
      const int nx = d.aux[5], base = d.n_in - nx;   // folded AddN terms of dout
      I.p[14] = nx > 0 ? ip(base) : 0;
      I.p[15] = nx > 1 ? ip(base + 1) : 0;
      I.p[9] = outp[2]; I.p[10] = dz_ptr;
      I.s[0] = t; I.s[4] = in_tok(d, o + 2).dt; I.s[5] = dz_bytes;
      for (int j = 0; j < d.n_in; ++j) dep(e, in_tok(d, j).writer);
    }
    {
      ns = 0;
      Inst& I = A.insts[x];
      I.m = B; I.k = In; I.n = H;
      I.p[0] = mz; I.p[1] = mwt; I.p[5] = masked ? ip(6) : 0; I.p[6] = ip(o);
      I.p[11] = outp[0]; I.p[12] = outp[1];
      I.s[0] = t; I.s[2] = sz;
      dep(x, e);
      dep(x, pw);
      dep(x, in_tok(d, o).writer);
    }
    const int cnt = dw_count_[nid];
    int64_t* rec = A.dw_pend + ((int64_t)nid * kDwMax + cnt) * 10;
    rec[0] = szn; rec[1] = mxn; rec[2] = sxn; rec[3] = mhn; rec[4] = shn;
    rec[5] = dz_ptr + dz_bytes;
    rec[6] = e; rec[7] = in_tok(d, 0).writer; rec[8] = in_tok(d, 1).writer;
    A.dw_pend[(int64_t)nid * kDwMax * 10 + 9] = mzn;
    dw_count_[nid] = cnt + 1;
    if (id[2] >= 0) {   // close the dW chunk (the driver reserved its id)
      const int32_t wd = id[2];
      const int c2 = cnt + 1;
      inst_header(wd, HK_LSTM_DW_TC, d.aux[1] & 1, (int)((4 * H / 256) * (KT / 256) + (4 * H + 255) / 256));
      Inst& I = A.insts[wd];
      I.m = B; I.k = In; I.n = H;
      I.p[0] = mzn;
      I.p[3] = acc_w >= 0 ? P.accs[acc_w].base : outp[3];
      I.p[4] = acc_b >= 0 ? P.accs[acc_b].base : outp[4];
      int64_t* ax = A.inst_aux + (int64_t)wd * kDwMax * 6;
      I.p[6] = (int64_t)ax;
      I.s[6] = (acc_w >= 0 ? 1 : 0) | (acc_b >= 0 ? 2 : 0);
      I.s[7] = c2;
      ns = 0;
      for (int q = 0; q < c2; ++q) {
        const int64_t* rq = A.dw_pend + ((int64_t)nid * kDwMax + q) * 10;
        for (int k = 0; k < 6; ++k) ax[q * 6 + k] = rq[k];
        dep(wd, (int32_t)rq[6]);
        dep(wd, (int32_t)rq[7]);
        dep(wd, (int32_t)rq[8]);
      }
      if (acc_w >= 0) dep(wd, acc_writer_[acc_w]);
      if (acc_b >= 0) dep(wd, acc_writer_[acc_b]);
      if (acc_w >= 0) acc_writer_[acc_w] = wd;
      if (acc_b >= 0) acc_writer_[acc_b] = wd;
      dw_count_[nid] = 0;
    }
    return true;
  }

  // create the dW/db instance for the queued steps of LSTMCellGrad node nid
  __noinline__ __device__ int32_t flush_dw(const DNode& d, int nid, int64_t mzn, int64_t dw_ptr, int64_t db_ptr) {
    Region rg(this, 32 + 8);
    const int cnt = dw_count_[nid];
    if (cnt == 0) return 0;
    const int64_t B = d.imm[0], In = d.imm[1], H = d.imm[2], KT = In + H;
    const int acc_w = d.aux[3], acc_b = d.aux[4];
    int32_t w = new_inst(HK_LSTM_DW_TC, d.aux[1] & 1,
                         (int)((4 * H / 256) * (KT / 256) + (4 * H + 255) / 256));
    if (w < 0) return -1;
    Inst& I = A.insts[w];
    I.m = B; I.k = In; I.n = H;
    I.p[0] = mzn;
    I.p[3] = acc_w >= 0 ? P.accs[acc_w].base : dw_ptr;
    I.p[4] = acc_b >= 0 ? P.accs[acc_b].base : db_ptr;
    int64_t* ax = A.inst_aux + (int64_t)w * kDwMax * 6;
    I.p[6] = (int64_t)ax;
    I.s[6] = (acc_w >= 0 ? 1 : 0) | (acc_b >= 0 ? 2 : 0);
    I.s[7] = cnt;
    for (int q = 0; q < cnt; ++q) {
      const int64_t* rec = A.dw_pend + ((int64_t)nid * kDwMax + q) * 10;
      for (int k = 0; k < 6; ++k) ax[q * 6 + k] = rec[k];
      add_dep(w, (int32_t)rec[6]);
      add_dep(w, (int32_t)rec[7]);
      add_dep(w, (int32_t)rec[8]);
    }
    if (acc_w >= 0) add_dep(w, acc_writer_[acc_w]);
    if (acc_b >= 0) add_dep(w, acc_writer_[acc_b]);
    submit(w, true);
    if (acc_w >= 0) acc_writer_[acc_w] = w;
    if (acc_b >= 0) acc_writer_[acc_b] = w;
    dw_count_[nid] = 0;
    last_dw = w;
    return w;
  }

  // ---------------------------------------------------------------- heavy ops
  __forceinline__ __device__ int eval_heavy(const DNode& d, int nid) {
    Region rg(this, 32 + 10);
    const int kind = d.aux[0];
    int64_t outp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const bool tcm = P.precision == D_BF16;
    int nplace = d.n_out;
    if (kind == HK_LSTM_BWD_EW) nplace += tcm ? 2 : 1;
    if (kind == HK_LSTM_FWD && tcm) nplace += (d.aux[1] & 4) ? 2 : 1;
    long long q0 = (kProfBuild && A.prof) ? clock64() : 0;
    for (int p = 0; p < nplace; ++p)
      if (!place(d, p, &outp[p])) return st->error ? EV_ERROR : EV_BLOCKED;
    if (kProfBuild && A.prof) { op_cyc[32 + 19] += clock64() - q0; op_cnt[32 + 19]++; }
    if (tcm && (kind == HK_LSTM_FWD || kind == HK_LSTM_BWD_EW)) return eval_lstm_tc(d, nid, outp);
    auto ip = [&](int j) { return in_tok(d, j).v; };
    auto dep_all = [&](int32_t id) {
      for (int j = 0; j < d.n_in; ++j) add_dep(id, in_tok(d, j).writer);
    };
    const int odt = places_[d.place_off].dt;
    if (kind == HK_LSTM_FWD || kind == HK_LSTM_BWD_EW) {
      const bool masked = d.aux[1] & 1;
      int64_t t = 0;
      if (masked && !scalar(in_tok(d, 5), &t)) return EV_BLOCKED;
      const int64_t B = d.imm[0], In = d.imm[1], H = d.imm[2];
      if (kind == HK_LSTM_FWD) {
        int ntiles = (int)(((B + 31) / 32) * ((H + 31) / 32));
        int32_t id = new_inst(HK_LSTM_FWD, masked, ntiles);
        if (id < 0) return EV_ERROR;
        Inst& I = A.insts[id];
        I.m = B; I.k = In; I.n = H;
        for (int j = 0; j < 5; ++j) I.p[j] = ip(j);
        I.p[5] = masked ? ip(6) : 0;
        for (int p = 0; p < 4; ++p) I.p[8 + p] = outp[p];
        I.s[0] = t;
        I.s[1] = d.aux[2];
        dep_all(id);
        for (int p = 0; p < 4; ++p) set_out(d, p, ptr_tok(outp[p], id, D_F32));
        submit(id);
      } else {
        // inputs: x h c W gates [t len] dh_next dc_next dout
        int o = masked ? 7 : 5;
        int ntiles_ew = (int)((B * H + kEwTile - 1) / kEwTile);
        int32_t e = new_inst(HK_LSTM_BWD_EW, masked, ntiles_ew);
        if (e < 0) return EV_ERROR;
        {
          Inst& I = A.insts[e];
          I.m = B; I.k = In; I.n = H;
          I.p[2] = ip(2);
          I.p[4] = ip(4);
          I.p[5] = masked ? ip(6) : 0;
          I.p[6] = ip(o);
          I.p[7] = ip(o + 1);
          I.p[8] = ip(o + 2);
          {
            const int nx = d.aux[5], base = d.n_in - nx;
            I.p[14] = nx > 0 ? ip(base) : 0;
            I.p[15] = nx > 1 ? ip(base + 1) : 0;
          }
          I.p[9] = outp[2];
          I.p[10] = outp[5];
          I.s[0] = t;
          dep_all(e);
        }
        const int64_t KT = In + H, G = 4 * H;
        int tA = (int)(((B + 63) / 64) * ((KT + 63) / 64));
        int tB = (int)(((G + 63) / 64) * ((KT + 63) / 64));
        int tC = (int)((G + kThreads - 1) / kThreads);
        int32_t m = new_inst(HK_LSTM_BWD_MM, masked, tA + tB + tC);
        if (m < 0) return EV_ERROR;
        const int acc_w = d.aux[3], acc_b = d.aux[4];
        {
          Inst& I = A.insts[m];
          I.m = B; I.k = In; I.n = H;
          I.p[0] = ip(0);
          I.p[1] = ip(1);
          I.p[3] = ip(3);
          I.p[5] = masked ? ip(6) : 0;
          I.p[6] = ip(o);
          I.p[10] = outp[5];
          I.p[11] = outp[0];
          I.p[12] = outp[1];
          I.p[13] = outp[3];
          I.s[3] = outp[4];
          I.s[0] = t;
          I.s[6] = (acc_w >= 0 ? 1 : 0) | (acc_b >= 0 ? 2 : 0);
          dep_all(m);
          add_dep(m, e);
          if (acc_w >= 0) add_dep(m, acc_writer_[acc_w]);
          if (acc_b >= 0) add_dep(m, acc_writer_[acc_b]);
        }
        set_out(d, 0, ptr_tok(outp[0], m, D_F32));
        set_out(d, 1, ptr_tok(outp[1], m, D_F32));
        set_out(d, 2, ptr_tok(outp[2], e, D_F32));
        set_out(d, 3, ptr_tok(outp[3], m, D_F32));
        set_out(d, 4, ptr_tok(outp[4], m, D_F32));
        submit(e);
        submit(m);
        if (acc_w >= 0) acc_writer_[acc_w] = m;
        if (acc_b >= 0) acc_writer_[acc_b] = m;
      }
      return EV_OK;
    }
    int32_t id = -1;
    switch (kind) {
      case HK_EW: {
        int64_t n = d.imm[0];
        if (d.aux[1] == EW_ADDN && d.n_in > 8) return eval_addn_chain(d, outp[0], odt);
        id = new_inst(HK_EW, d.aux[1], (int)((n + kEwBig - 1) / kEwBig));
        if (id < 0) return EV_ERROR;
        Inst& I = A.insts[id];
        I.n = n;
        I.m = d.imm[1];
        for (int j = 0; j < d.n_in && j < 8; ++j) I.p[j] = ip(j);
        I.p[13] = outp[0];
        I.s[0] = d.n_in;
        I.s[1] = d.aux[2];
        I.s[2] = d.aux[3];
        I.dts = pack_dts(d, odt);
        break;
      }
      case HK_FILL: {
        int64_t n = d.imm[0];
        id = new_inst(HK_FILL, 0, (int)((n + kEwBig - 1) / kEwBig));
        if (id < 0) return EV_ERROR;
        Inst& I = A.insts[id];
        I.n = n;
        I.p[0] = ip(0);
        I.p[13] = outp[0];
        I.dts = pack_dts(d, odt);
        break;
      }
      case HK_REDUCE_SUM: {
        int64_t n = d.imm[0];
        int64_t nt0 = (n + kEwTile - 1) / kEwTile;
        int nt = (int)(nt0 < 1024 ? nt0 : 1024);
        id = new_inst(HK_REDUCE_SUM, 0, max(nt, 1));
        if (id < 0) return EV_ERROR;
        Inst& I = A.insts[id];
        I.n = n;
        I.p[0] = ip(0);
        I.p[13] = outp[0];
        I.dts = pack_dts(d, odt);
        break;
      }
      case HK_REDUCE_SUM0: {
        id = new_inst(HK_REDUCE_SUM0, 0, (int)((d.imm[1] + kThreads - 1) / kThreads));
        if (id < 0) return EV_ERROR;
        Inst& I = A.insts[id];
        I.m = d.imm[0];
        I.n = d.imm[1];
        I.p[0] = ip(0);
        I.p[13] = outp[0];
        I.dts = pack_dts(d, odt);
        break;
      }
      case HK_MATMUL: {
        int64_t M = d.imm[0], N = d.imm[1], K = d.imm[2];
        const bool ta = d.aux[1] & 1, tb = d.aux[1] & 2;
        int64_t ma, sa, mb, sb;
        int16_t hint_a = -1, hint_b = -1;
        // the tensor-core GEMM when both operands are registered bf16 buffers (TMA operands)
        if (tcm && N % 256 == 0 && K % 64 == 0 && !(kDbgFlags & (1 << 1)) &&
            in_tok(d, 0).dt == D_BF16 && in_tok(d, 1).dt == D_BF16 &&
            resolve_try(ip(0), (int)(ta ? K : M), (int)(ta ? M : K), ta ? 2 : 0, &ma, &sa, &hint_a) &&
            resolve_try(ip(1), (int)(tb ? N : K), (int)(tb ? K : N), tb ? 1 : 2, &mb, &sb, &hint_b)) {
          id = new_inst(HK_MATMUL_TC, d.aux[1], (int)(((M + 127) / 128) * (N / 256)));
          if (id < 0) return EV_ERROR;
          Inst& I = A.insts[id];
          I.m = M; I.n = N; I.k = K;
          I.p[0] = ma; I.p[1] = mb; I.p[13] = outp[0];
          I.s[0] = sa; I.s[1] = sb; I.s[2] = odt;
          break;
        }
        id = new_inst(HK_MATMUL, d.aux[1], (int)(((M + 63) / 64) * ((N + 63) / 64)));
        if (id < 0) return EV_ERROR;
        Inst& I = A.insts[id];
        I.m = M; I.n = N; I.k = K;
        I.p[0] = ip(0);
        I.p[1] = ip(1);
        I.p[13] = outp[0];
        I.s[0] = d.imm[3] & 0xffffffffLL;
        I.s[1] = d.imm[3] >> 32;
        I.dts = pack_dts(d, odt);
        break;
      }
      default:
        fail(CF_E_UNSUPPORTED, kind);
        return EV_ERROR;
    }
    dep_all(id);
    set_out(d, 0, ptr_tok(outp[0], id, odt));
    submit(id);
    return EV_OK;
  }

  // AddN of more than 8 terms (e.g. a weight gradient summed over a statically unrolled loop's
  // steps): a chain of 8-input sums, each adding up to 7 more terms to the running sum in the
  // output buffer (elementwise, in place)
  __noinline__ __device__ int eval_addn_chain(const DNode& d, int64_t out, int odt) {
    const int64_t n = d.imm[0];
    int32_t prev = -1;
    for (int j0 = 0; j0 < d.n_in;) {
      const int first = j0 == 0 ? 0 : 1;
      const int take = min(8 - first, d.n_in - j0);
      const int32_t id = new_inst(HK_EW, EW_ADDN, (int)((n + kEwBig - 1) / kEwBig));
      if (id < 0) return EV_ERROR;
      Inst& I = A.insts[id];
      I.n = n;
      I.m = d.imm[1];
      int k = 0;
      int64_t dts = (int64_t)(odt & 15) << 32;
      if (first) {
        dts |= (int64_t)(odt & 15) << (4 * k);
        I.p[k++] = out;
      }
      for (int q = 0; q < take; ++q) {
        const Tok& t = in_tok(d, j0 + q);
        dts |= (int64_t)(t.dt & 15) << (4 * k);
        I.p[k++] = t.v;
        add_dep(id, t.writer);
      }
      I.p[13] = out;
      I.s[0] = k;
      I.s[1] = 0;
      I.s[2] = d.aux[3];
      I.dts = dts;
      add_dep(id, prev);
      submit(id);
      prev = id;
      j0 += take;
    }
    set_out(d, 0, ptr_tok(out, prev, odt));
    return EV_OK;
  }

  __noinline__ __device__ int32_t copy_inst(int64_t dst, int64_t src, int64_t bytes, int32_t dep,
                                            unsigned long long* signal = nullptr,
                                            unsigned long long signal_value = 0, int sub = 0) {
    int32_t id = new_inst(HK_COPY, sub, (int)((bytes + 65535) / 65536));
    if (id < 0) return -1;
    Inst& I = A.insts[id];
    I.n = bytes;
    I.p[0] = src;
    I.p[13] = dst;
    I.signal = signal;
    I.signal_value = signal_value;
    add_dep(id, dep);
    submit(id);
    return id;
  }

  // ---------------------------------------------------------------- channels (a14)
  // Send / Recv of iteration `it` over channel slot it % slots: the
  // payload moves GPU -> GPU by a copy instance whose workers store straight into the peer's
  // slot over NVLink; the last tile publishes the flag (release, system scope). The dead
  // signal is a flag with the low bit set and no payload.
  // ---------------------------------------------------------------- stack swapping (a8)
  // "move tensors from GPU to CPU memory when they are pushed onto stacks,
  // and bring them back gradually before they are needed in backpropagation". A swapped value
  // lives in a (K + 1)-slot device ring; the parallel-iterations window guarantees that the
  // iteration which last used a ring slot has completed (including its copies) before the
  // slot is written again, in the forward and in the gradient loop (reading R19).
  __device__ int find_swap(int64_t p, int64_t* slot) const {
    for (int k = 0; k < P.n_swaps; ++k) {
      const DSwap& w = P.swaps[k];
      if (p >= w.dev_base && p < w.dev_base + (int64_t)w.ring * w.elem_bytes) {
        *slot = (p - w.dev_base) / w.elem_bytes;
        return k;
      }
    }
    return -1;
  }
  __noinline__ __device__ int swap_copy(int dir, int64_t dst, int64_t src, int64_t bytes, int32_t dep) {
    int32_t id = new_inst(HK_SWAP, dir, 1);
    if (id < 0) return -1;
    Inst& I = A.insts[id];
    I.n = bytes;
    I.p[0] = src;
    I.p[13] = dst;
    add_dep(id, dep);
    submit(id);
    return id;
  }
  __noinline__ __device__ int swap_out(const Tok& v, int32_t entry, int dp) {
    int64_t r;
    const int k = find_swap(v.v, &r);
    if (k < 0) return 0;
    const DSwap& w = P.swaps[k];
    if (dp >= w.capacity) {
      fail(CF_E_STACK_BUDGET, dp);
      return -1;
    }
    A.swap_owner[w.owner_off + r] = entry;
    if (swap_copy(0, w.host_base + (int64_t)dp * w.elem_bytes, v.v, w.elem_bytes, v.writer) < 0) return -1;
    n_swap_out++;
    b_d2h += w.elem_bytes;
    return 1;
  }
  __noinline__ __device__ int swap_in(Tok* t, int32_t entry, int dp) {
    int64_t r;
    const int k = find_swap(t->v, &r);
    if (k < 0) return 0;
    const DSwap& w = P.swaps[k];
    if (A.swap_owner[w.owner_off + r] == entry) return 0;   // still resident in its ring slot
    const int it = git();
    const int64_t dst = w.in_base + (int64_t)(it % w.in_ring) * w.elem_bytes;
    int32_t id = swap_copy(1, dst, w.host_base + (int64_t)dp * w.elem_bytes, w.elem_bytes, -1);
    if (id < 0) return -1;
    t->v = dst;
    t->writer = id;
    n_swap_in++;
    b_h2d += w.elem_bytes;
    return 1;
  }

  __noinline__ __device__ int eval_send(const DNode& d, bool dead) {
    const DChan& C = P.chans[d.aux[0]];
    const int it = cur_frame >= 0 ? iter : 0;
    const int slot = it % C.slots;
    const unsigned long long ep = A.epoch << 32;
    if (it >= C.slots) {   // slot still holds message it - slots until the receiver acks it
      const unsigned long long need = ep | (unsigned long long)(it - C.slots + 1);
      if (ld_acquire_sys_u64(&C.acks[slot]) < need) return EV_BLOCKED;
    }
    const int64_t stride = (C.elem_bytes + 255) / 256 * 256;
    n_sent++;
    if (dead) {
      st_release_sys_u64(&C.flags[slot], ep | (2ULL * (it + 1) + 1));
      return EV_OK;
    }
    const Tok& v = in_tok(d, 0);
    if (copy_inst((int64_t)(C.data + slot * stride), v.v, C.elem_bytes, v.writer, &C.flags[slot],
                  ep | (2ULL * (it + 1))) < 0)
      return EV_ERROR;
    return EV_OK;
  }
  // Recv never blocks the driver: a wait instance (HK_WAIT, completed by drain() when the
  // flag shows the message) gates the copy out of the slot; the copy's last tile acks the
  // slot. The message is expected live exactly when this Recv is live: both partitions
  // evaluate the same control (reading R18); a mismatch is an error.
  __noinline__ __device__ int eval_recv(const DNode& d, bool dead, bool* out_dead) {
    const DChan& C = P.chans[d.aux[0]];
    const int it = cur_frame >= 0 ? iter : 0;
    const int slot = it % C.slots;
    const unsigned long long ep = A.epoch << 32;
    const unsigned long long live = ep | (2ULL * (it + 1));
    const unsigned long long ackv = ep | (unsigned long long)(it + 1);
    n_recv++;
    int64_t out = 0;
    if (!dead && !place(d, 0, &out)) return st->error ? EV_ERROR : EV_BLOCKED;
    int32_t w = new_inst(HK_WAIT, dead ? 1 : 0, 1);
    if (w < 0) return EV_ERROR;
    {
      Inst& I = A.insts[w];
      I.p[0] = (int64_t)&C.flags[slot];
      I.s[0] = (int64_t)(dead ? (live | 1) : live);
      I.p[1] = dead ? (int64_t)&C.acks[slot] : 0;   // a dead message is acked on arrival
      I.s[1] = (int64_t)ackv;
    }
    submit(w);
    if (dead) {
      set_dead_all(d);
      *out_dead = true;
      return EV_OK;
    }
    const int64_t stride = (C.elem_bytes + 255) / 256 * 256;
    int32_t id = copy_inst(out, (int64_t)(C.data + slot * stride), C.elem_bytes, w, &C.acks[slot], ackv, 1);
    if (id < 0) return EV_ERROR;
    set_out(d, 0, ptr_tok(out, id, C.dt));
    return EV_OK;
  }

  // ---------------------------------------------------------------- node evaluation
  // Hot path: the routing primitives evaluated hundreds of times per iteration stay in a
  // small function (I-cache); everything else goes through eval_cold.
  __noinline__ __device__ int eval(const DNode& d, int nid) {
    const int op = d.op;
    if (op == OP_SWITCH || op == OP_MERGE || op == OP_MERGE_LOOP || op == OP_NEXTITER ||
        op == OP_PASS || (op == OP_CONST && d.aux[0] == 1)) {
      bool dead = false;
      if (op != OP_MERGE && op != OP_MERGE_LOOP) {
        for (int j = 0; j < d.n_in; ++j) dead |= toks_[iv_[d.in_off + j]].dead != 0;
        for (int j = 0; j < d.n_ctrl; ++j) dead |= toks_[iv_[d.ctrl_off + j]].dead != 0;
      }
      bool ctrl_dead = dead;
      if (op == OP_SWITCH) {
        Tok dv = toks_[iv_[d.in_off]];
        const Tok& pt = toks_[iv_[d.in_off + 1]];
        Tok o0 = dv, o1 = dv;
        if (dead) {
          o0.dead = o1.dead = 1;
        } else {
          int64_t pv;
          if (pt.kind == TK_IMM) pv = pt.v;
          else if (!scalar(pt, &pv)) return EV_BLOCKED;
          o0.dead = pv != 0;   // false port: dead iff p
          o1.dead = pv == 0;   // true port: dead iff !p
          if (d.aux[0] >= 0) {
            const int it = git();
            if (it < P.branch_bound) A.branch_bits[d.aux[0] * P.branch_bound + it] = pv ? 2 : 1;
          }
        }
        toks_[d.out_vid] = o0;
        toks_[d.out_vid + 1] = o1;
      } else if (op == OP_MERGE) {
        const Tok& a = toks_[iv_[d.in_off]];
        const Tok& b = toks_[iv_[d.in_off + 1]];
        Tok o = !a.dead ? a : b;   // "if is_dead(d1) then d2 else d1"
        toks_[d.out_vid] = o;
        ctrl_dead = o.dead;
      } else if (op == OP_MERGE_LOOP) {
        Tok o = toks_[iv_[d.in_off + (iter == 0 ? 0 : 1)]];
        toks_[d.out_vid] = o;
        ctrl_dead = o.dead;
      } else if (op == OP_NEXTITER) {
        toks_[d.out_vid] = toks_[iv_[d.in_off]];
      } else if (op == OP_PASS) {
        Tok t = toks_[iv_[d.in_off]];
        t.dead = dead;
        for (int p = 0; p < d.n_out; ++p) toks_[d.out_vid + p] = t;
      } else {
        Tok t{};
        t.writer = -1;
        t.dead = dead;
        t.kind = TK_IMM;
        t.v = d.imm[0];
        t.dt = (uint8_t)d.aux[1];
        toks_[d.out_vid] = t;
      }
      Tok c{};
      c.dead = ctrl_dead;
      c.writer = -1;
      c.kind = TK_FLOW;
      toks_[d.ctrl_vid] = c;
      return EV_OK;
    }
    return eval_cold(d, nid);
  }

  // heavy node straight from the body loop (one call level: eval_heavy / eval_lstm_tc inline)
  __noinline__ __device__ int eval_heavy_node(const DNode& d, int nid) {
    bool dead = false;
    const bool prepped = prep_ok(d);
    if (prepped) {   // dead check, placements and lookups on the helper lanes
      const long long key = ((long long)(cur_frame + 1) << 32) | (unsigned)iter;
      if (!(chain_ok_ && wave_->hd == &d && chain_key_ == key)) run_heavy_prep(d);   // else done
                                                                                     // by the last wave
      chain_ok_ = false;
      dead = wave_->hdead != 0;
    } else {
      for (int j = 0; j < d.n_in; ++j) dead |= in_tok(d, j).dead != 0;
      for (int j = 0; j < d.n_ctrl; ++j) dead |= toks_[iv_[d.ctrl_off + j]].dead != 0;
    }
    if (dead) {
      set_dead_all(d);
      n_dead++;
    } else {
      if (dbg_ & (1 << 26)) maybe_drain();   // bit 26: poll before each heavy node (A/B; the
                                              // wave waits poll often enough, measured ~1%)
      const bool use = prepped && !wave_->hfail;
      const int r = use ? eval_lstm_tc(d, nid, wave_->houtp, wave_->hmap, wave_->hslot)
                        : eval_heavy(d, nid);
      flush_publish();
      if (r != EV_OK) return r;
    }
    toks_[d.ctrl_vid] = Tok{0, -1, (uint8_t)dead, TK_FLOW, 0, 0};
    return EV_OK;
  }

  __noinline__ __device__ int eval_cold(const DNode& d, int nid) {
    const int op = d.op;
    bool dead = false;
    if (op != OP_MERGE && op != OP_MERGE_LOOP) {
      for (int j = 0; j < d.n_in; ++j) dead |= in_tok(d, j).dead != 0;
      for (int j = 0; j < d.n_ctrl; ++j) dead |= toks_[iv_[d.ctrl_off + j]].dead != 0;
    }
    int res = EV_OK;
    bool ctrl_dead = dead;
    switch (op) {
      case OP_NOP:
      case OP_PLACEHOLDER:
        break;
      case OP_CONST: {
        Tok t{};
        t.writer = -1;
        t.dead = dead;
        if (d.aux[0] == 1) {
          t.kind = TK_IMM;
          t.v = d.imm[0];
        } else {
          t.kind = TK_PTR;
          t.v = d.imm[0];
        }
        t.dt = (uint8_t)d.aux[1];
        set_out(d, 0, t);
        break;
      }
      case OP_PASS:
      case OP_FLOW: {
        Tok t = d.n_in ? in_tok(d, 0) : Tok{};
        if (op == OP_FLOW) {
          t = Tok{};
          t.kind = TK_FLOW;
          t.writer = -1;
        }
        t.dead = dead;
        for (int p = 0; p < d.n_out; ++p) set_out(d, p, t);
        break;
      }
      case OP_SWITCH: {
        Tok dv = in_tok(d, 0);
        const Tok& pt = in_tok(d, 1);
        Tok o0 = dv, o1 = dv;
        if (dv.dead || pt.dead || dead) {
          o0.dead = o1.dead = 1;
          ctrl_dead = true;
        } else {
          int64_t pv;
          if (!scalar(pt, &pv)) return EV_BLOCKED;
          o0.dead = pv != 0;   // false port: dead iff p
          o1.dead = pv == 0;   // true port: dead iff !p
          if (d.aux[0] >= 0 && d.aux[0] < P.n_conds) {
            const int it = git();
            if (it < P.branch_bound) A.branch_bits[d.aux[0] * P.branch_bound + it] = pv ? 2 : 1;
          }
        }
        set_out(d, 0, o0);
        set_out(d, 1, o1);
        break;
      }
      case OP_MERGE: {
        const Tok& a = in_tok(d, 0);
        const Tok& b = in_tok(d, 1);
        Tok o = !a.dead ? a : b;   // "if is_dead(d1) then d2 else d1"
        set_out(d, 0, o);
        ctrl_dead = o.dead;
        break;
      }
      case OP_MERGE_LOOP: {
        Tok o = iter == 0 ? in_tok(d, 0) : in_tok(d, 1);
        set_out(d, 0, o);
        ctrl_dead = o.dead;
        break;
      }
      case OP_NEXTITER:
        set_out(d, 0, in_tok(d, 0));
        break;
      case OP_ENTER:
      case OP_EXIT:
        set_out(d, 0, in_tok(d, 0));
        break;
      case OP_SCALAR: {
        if (dead) {
          set_dead_all(d);
          break;
        }
        int64_t a = 0, b = 0;
        if (!scalar(in_tok(d, 0), &a)) return EV_BLOCKED;
        if (d.n_in > 1 && !scalar(in_tok(d, 1), &b)) return EV_BLOCKED;
        int64_t r = 0;
        switch (d.aux[0]) {
          case SC_ADD: r = a + b; break;
          case SC_SUB: r = a - b; break;
          case SC_MUL: r = a * b; break;
          case SC_LESS: r = a < b; break;
          case SC_LEQ: r = a <= b; break;
          case SC_GREATER: r = a > b; break;
          case SC_EQ: r = a == b; break;
          case SC_AND: r = (a != 0) && (b != 0); break;
          case SC_NOT: r = a == 0; break;
          case SC_CAST: r = d.aux[1] == D_BOOL ? (a != 0) : a; break;
        }
        Tok t{};
        t.kind = TK_IMM;
        t.v = r;
        t.writer = -1;
        t.dt = (uint8_t)d.aux[1];
        set_out(d, 0, t);
        break;
      }
      case OP_REDUCE_I: {
        if (dead) {
          set_dead_all(d);
          break;
        }
        const Tok& v = in_tok(d, 0);
        if (!writer_done(v.writer)) return EV_BLOCKED;
        __threadfence();
        int n = d.aux[1];
        int64_t r = 0;
        if (d.aux[2] == D_I64) {
          const int64_t* p = (const int64_t*)v.v;
          r = p[0];
          for (int k = 1; k < n; ++k) r = d.aux[0] ? min(r, p[k]) : max(r, p[k]);
        } else {
          const int32_t* p = (const int32_t*)v.v;
          r = p[0];
          for (int k = 1; k < n; ++k) {
            int64_t q = p[k];
            r = d.aux[0] ? (q < r ? q : r) : (q > r ? q : r);
          }
        }
        Tok t{};
        t.kind = TK_IMM;
        t.v = r;
        t.writer = -1;
        t.dt = (uint8_t)d.aux[2];
        set_out(d, 0, t);
        break;
      }
      case OP_SLICE_I: {
        Tok t = in_tok(d, 0);
        t.v += d.imm[0];
        t.dead = dead;
        set_out(d, 0, t);
        break;
      }
      case OP_TA_CREATE: {
        Tok h{};
        h.kind = TK_HANDLE;
        h.v = d.aux[0];
        h.writer = -1;
        h.dead = dead;
        Tok f{};
        f.kind = TK_FLOW;
        f.writer = -1;
        f.dead = dead;
        set_out(d, 0, h);
        set_out(d, 1, f);
        break;
      }
      case OP_TA_GRAD: {
        Tok h{};
        h.kind = TK_HANDLE;
        h.v = d.aux[0];
        h.writer = -1;
        h.dead = dead;
        Tok f{};
        f.kind = TK_FLOW;
        f.writer = -1;
        f.dead = dead;
        set_out(d, 0, h);
        set_out(d, 1, f);
        break;
      }
      case OP_TA_READ: {
        if (dead) {
          set_dead_all(d);
          break;
        }
        int ta = (int)in_tok(d, 0).v;
        int64_t ix;
        if (!scalar(in_tok(d, 1), &ix)) return EV_BLOCKED;
        const DTA& T = tas_[ta];
        if (ix < 0 || ix >= T.size) {
          fail(CF_E_SHAPE, ix);
          return EV_ERROR;
        }
        int so = tso_[ta] + (int)ix;
        if (!T.is_grad && !A.ta_written[so]) {
          fail(CF_E_INVALID_GRAPH, ix);
          return EV_ERROR;
        }
        set_out(d, 0, ptr_tok(tab_[ta] + ix * T.elem_bytes, A.ta_writer[so], T.dt));
        break;
      }
      case OP_TA_WRITE: {
        Tok f{};
        f.kind = TK_FLOW;
        f.writer = -1;
        f.dead = dead;
        if (!dead) {
          int ta = (int)in_tok(d, 0).v;
          int64_t ix;
          if (!scalar(in_tok(d, 1), &ix)) return EV_BLOCKED;
          const DTA& T = tas_[ta];
          if (ix < 0 || ix >= T.size) {
            fail(CF_E_SHAPE, ix);
            return EV_ERROR;
          }
          int so = tso_[ta] + (int)ix;
          const Tok& v = in_tok(d, 2);
          int64_t dst = tab_[ta] + ix * T.elem_bytes;
          if (A.ta_written[so]) {
            if (!T.is_grad) {
              fail(CF_E_DOUBLE_WRITE, ix);
              return EV_ERROR;
            }
            // grad TensorArray: "holds the sum of the partial gradients"
            int32_t id = new_inst(HK_ACC, 0, (int)((T.elem_bytes / 4 + kEwTile - 1) / kEwTile));
            if (id < 0) return EV_ERROR;
            A.insts[id].n = T.elem_bytes / 4;
            A.insts[id].p[0] = v.v;
            A.insts[id].p[13] = dst;
            add_dep(id, v.writer);
            add_dep(id, A.ta_writer[so]);
            submit(id);
            A.ta_writer[so] = id;
          } else if (v.v == dst) {
            A.ta_writer[so] = v.writer;    // producer was placed in the slot: zero-copy
          } else {
            A.ta_writer[so] = copy_inst(dst, v.v, T.elem_bytes, v.writer);
          }
          A.ta_written[so] = 1;
        }
        set_out(d, 0, f);
        break;
      }
      case OP_TA_STACK: {
        if (dead) {
          set_dead_all(d);
          break;
        }
        int ta = (int)in_tok(d, 0).v;
        const DTA& T = tas_[ta];
        int32_t join = new_inst(HK_NOP, 0, 1);
        if (join < 0) return EV_ERROR;
        for (int i = 0; i < T.size; ++i) {
          int so = tso_[ta] + i;
          if (!T.is_grad && !A.ta_written[so]) {
            fail(CF_E_INVALID_GRAPH, i);
            return EV_ERROR;
          }
          add_dep(join, A.ta_writer[so]);
        }
        submit(join);
        set_out(d, 0, ptr_tok(tab_[ta], join, T.dt));
        break;
      }
      case OP_TA_UNSTACK: {
        Tok f{};
        f.kind = TK_FLOW;
        f.writer = -1;
        f.dead = dead;
        if (!dead) {
          int ta = (int)in_tok(d, 0).v;
          const DTA& T = tas_[ta];
          const Tok& v = in_tok(d, 1);
          bool any = false;
          for (int i = 0; i < T.size; ++i) any |= A.ta_written[tso_[ta] + i] != 0;
          if (!any) {
            tab_[ta] = v.v;   // alias the unstacked tensor (no copy)
            for (int i = 0; i < T.size; ++i) {
              A.ta_writer[tso_[ta] + i] = v.writer;
              A.ta_written[tso_[ta] + i] = 1;
            }
          } else {
            fail(CF_E_DOUBLE_WRITE, 0);
            return EV_ERROR;
          }
        }
        set_out(d, 0, f);
        break;
      }
      case OP_STACK_CREATE: {
        Tok h{};
        h.kind = TK_HANDLE;
        // handle = stack id | instance << 20: a stack created in a loop body (a nested loop's,
        // SURVEY.md §8(f) f2) has one instance per iteration index of that loop
        h.v = (int64_t)d.aux[0] | ((int64_t)git() << 20);
        h.writer = -1;
        h.dead = dead;
        if (!dead && git() >= stacks_[d.aux[0]].instances) {
          fail(CF_E_STACK_BUDGET, -900);
          return EV_ERROR;
        }
        set_out(d, 0, h);
        break;
      }
      case OP_STACK_PUSH: {
        if (!dead) {
          const int64_t hv = in_tok(d, 0).v;
          const int s = (int)(hv & 0xFFFFF), inst = (int)(hv >> 20);
          const DStack& S = stacks_[s];
          const int di = S.depth_off + inst;
          const int64_t e0 = S.entry_off + (int64_t)inst * S.capacity;
          int dp = stack_depth_[di];
          if (dp >= S.capacity) {
            fail(CF_E_STACK_BUDGET, dp);
            return EV_ERROR;
          }
          const Tok& pv = in_tok(d, 1);
          A.stack_pool[e0 + dp] = pv;
          stack_depth_[di] = dp + 1;
          n_push++;
          if (P.n_swaps && pv.kind == TK_PTR && swap_out(pv, (int32_t)(e0 + dp), dp) < 0) return EV_ERROR;
          if (dp + 1 > max_depth) max_depth = dp + 1;
        }
        break;
      }
      case OP_STACK_POP: {
        if (dead) {
          set_dead_all(d);
          break;
        }
        const int64_t hv = in_tok(d, 0).v;
        const int s = (int)(hv & 0xFFFFF), inst = (int)(hv >> 20);
        const DStack& S = stacks_[s];
        const int di = S.depth_off + inst;
        const int64_t e0 = S.entry_off + (int64_t)inst * S.capacity;
        int dp = stack_depth_[di];
        if (dp <= 0) {
          fail(CF_E_POP_EMPTY, s | ((int64_t)inst << 20));
          return EV_ERROR;
        }
        Tok t = A.stack_pool[e0 + dp - 1];
        stack_depth_[di] = dp - 1;
        t.dead = 0;
        if (P.n_swaps && t.kind == TK_PTR && swap_in(&t, (int32_t)(e0 + dp - 1), dp - 1) < 0) return EV_ERROR;
        set_out(d, 0, t);
        n_pop++;
        break;
      }
      case OP_ACC: {
        // fused accumulator: the producers already added in place
        const DAcc& a = P.accs[d.aux[0]];
        Tok t = ptr_tok(a.base, acc_writer_[d.aux[0]], D_F32);
        t.dead = dead;
        set_out(d, 0, t);
        break;
      }
      case OP_HEAVY: {
        if (dead) {
          set_dead_all(d);
          n_dead++;
          break;
        }
        res = eval_heavy(d, nid);
        break;
      }
      case OP_SEND:
        res = eval_send(d, dead);
        break;
      case OP_RECV: {
        bool md = false;
        res = eval_recv(d, dead, &md);
        ctrl_dead |= md;
        break;
      }
      default:
        fail(CF_E_UNSUPPORTED, op);
        return EV_ERROR;
    }
    if (res != EV_OK) return res;
    Tok c{};
    c.dead = ctrl_dead;
    c.writer = -1;
    c.kind = TK_FLOW;
    toks_[d.ctrl_vid] = c;
    return EV_OK;
  }

  // ---------------------------------------------------------------- frames
  // a frame nested in the current frame's body: one instance per iteration of the
  // enclosing frame. The instance starts after everything created so far has completed (the
  // previous instance's storage and the consumers of its Exits are then free); a dead
  // instance (the enclosing frame's exiting iteration) only fires its Exits, dead.
  __noinline__ __device__ void enter_nested(int f) {
    const DFrame& F = P.frames[f];
    bool dead = true;
    for (int k = 0; k < F.n_enter && dead; ++k) dead = in_tok_g(node(P.order[F.enter_off + k]), 0).dead != 0;
    if (dead || fdepth_ >= kMaxNest) {
      if (!dead) fail(CF_E_UNSUPPORTED, -800);
      for (int k = 0; k < F.n_exit; ++k) set_dead_all(node(P.order[F.exit_off + k]));
      n_exitf += F.n_exit;
      return;
    }
    while (outstanding > 0 && !st->error) {
      const unsigned long long now = globaltimer();
      if (drain()) last_progress = now;
      else if ((long long)(now - last_progress) > A.watchdog_ns) fail(CF_E_DEADLOCK, -801);
    }
    fstack_[fdepth_++] = FrameSave{bn_, iv_, cur_frame, iter, oldest, body_pc, gbase_, iter_started ? 1 : 0};
    start_frame(f);
    gbase_ = f < 16 ? gnext_[f] : 0;
  }
  // the nested frame instance has fired its Exits: back to the enclosing body
  __device__ void leave_nested() {
    const int f = cur_frame;
    if (f < 16) gnext_[f] = gbase_ + iter;
    const FrameSave& s = fstack_[--fdepth_];
    bn_ = s.bn;
    iv_ = s.iv;
    cur_frame = s.frame;
    iter = s.iter;
    oldest = s.oldest;
    body_pc = s.body_pc;
    gbase_ = s.gbase;
    iter_started = s.started != 0;
    cur_F_ = &P.frames[cur_frame];
  }
  __noinline__ __device__ void start_frame(int f) {
    const DFrame& F = P.frames[f];
    for (int k = 0; k < F.n_enter; ++k) {
      const DNode& e = node(P.order[F.enter_off + k]);
      set_out(e, 0, in_tok_g(e, 0));
      Tok c{};
      c.dead = in_tok_g(e, 0).dead;
      c.writer = -1;
      toks_[e.ctrl_vid] = c;
    }
    // the frame's control program: staged in shared memory when there is room (not with
    // nested frames: the enclosing body's program would be overwritten)
    if (sm_nodes_ && !P.nested) {
      helper_copy(sm_nodes_, P.body_nodes + F.bn_off, (int64_t)F.n_body * sizeof(DNode), sm_iv_,
                  P.body_ivids + F.bi_off, (int64_t)F.bi_count * 4);
      bn_ = sm_nodes_;
      iv_ = sm_iv_;
    } else {
      bn_ = P.body_nodes + F.bn_off;
      iv_ = P.body_ivids + F.bi_off;
    }
    cur_frame = f;
    iter = 0;
    oldest = 0;
    body_pc = 0;
    iter_started = false;
    gbase_ = 0;
    // fused accumulators start from the loop variable's initial value
    for (int k = 0; k < F.n_acc; ++k) {
      int a = P.order[F.acc_off + k];
      const DAcc& ac = P.accs[a];
      int32_t id;
      if (ac.init_zero) {
        id = new_inst(HK_FILL, 0, (int)((ac.bytes / 4 + kEwBig - 1) / kEwBig));
        if (id < 0) return;
        A.insts[id].n = ac.bytes / 4;
        A.insts[id].p[0] = 0;
        A.insts[id].s[0] = 0;
        A.insts[id].p[13] = ac.base;
        A.insts[id].dts = (int64_t)D_F32 << 32;
        submit(id);
      } else {
        const Tok& it0 = toks_[ac.init_vid];
        id = copy_inst(ac.base, it0.v, ac.bytes, it0.writer);
      }
      acc_writer_[a] = id;
    }
  }

  // liveness of structured cond context c in the current iteration: 1 live, 0 dead, -1 the
  // predicate is not available yet. Records the cond's branch bit like a live Switch would.
  __noinline__ __device__ int ctx_live(int c) {
    int chain[8];
    int n = 0;
    for (int x = c; x && lstamp_[x] != lgen_; x = ctxs_[x].parent) {
      if (n == 8) {
        fail(CF_E_UNSUPPORTED, -300);
        return -1;
      }
      chain[n++] = x;
    }
    for (int k = n - 1; k >= 0; --k) {
      const int x = chain[k];
      const DCtx& cx = ctxs_[x];
      int live = cx.parent ? lval_[cx.parent] : 1;
      if (live) {
        const Tok& pt = toks_[cx.pred_vid];
        if (pt.dead) {
          live = 0;
        } else {
          int64_t pv;
          if (pt.kind == TK_IMM) pv = pt.v;
          else if (!scalar(pt, &pv)) return -1;
          live = (pv != 0) == (cx.branch == 1);
          const int it = git();
          if (cx.cond_id >= 0 && cx.cond_id < P.n_conds && it < P.branch_bound)
            A.branch_bits[cx.cond_id * P.branch_bound + it] = pv ? 2 : 1;
        }
      }
      lval_[x] = (int8_t)live;
      lstamp_[x] = lgen_;
    }
    return lval_[c];
  }

  // contexts of mask m for a fused wave level, evaluated by a helper lane between levels (the
  // driver thread is waiting for the job): false when a predicate is not available yet
  __noinline__ __device__ bool helper_ctx(unsigned long long m0, unsigned long long m1) {
    for (int hw = 0; hw < 2; ++hw)
      for (unsigned long long m = hw ? m1 : m0; m; m &= m - 1) {
        const int c = 64 * hw + __ffsll((long long)m) - 1;
        if (lstamp_[c] == lgen_) continue;
        if (ctx_live(c) < 0) return false;
      }
    return true;
  }

  // The per-iteration control loop: kept small and out of line so that its instructions stay
  // resident in the SM's instruction cache (the routing primitives dominate the node count).
  // The per-iteration control loop. Routing primitives are ~90% of the evaluations, so they
  // get a tiny straight-line path (16-byte token moves, no calls) at the head of the loop;
  // everything else goes through the out-of-line eval().
  __noinline__ __device__ bool run_body(const DFrame& F) {
    Region rg(this, 32 + 0);
    bool progress = false;
    const bool prof = (kProfBuild && A.prof != nullptr);
    const int n_body = F.n_body;
    int pc = body_pc;
    const FastEnv env = fast_env();
    FastCount fc{0, 0, 0, 0, 0};
    int since_drain = 0;
    while (pc < n_body) {
      const DNode* d = bn_ + pc;
      const int op = d->op;
      // completions are picked up every few nodes and before every heavy node: the latency
      // from a producer's last tile to its consumers' publication is on the recurrence's
      // critical path
      if (++since_drain >= 16) {
        maybe_drain();
        since_drain = 0;
      }
      if (d->ctx) {   // node of a structured cond branch: skip it when the branch is dead
        const int l = lval_[d->ctx] >= 0 && lstamp_[d->ctx] == lgen_ ? lval_[d->ctx] : ctx_live(d->ctx);
        if (l < 0) break;
        if (!l) {
          if (op == OP_HEAVY) n_dead++;
          ++pc;
          progress = true;
          continue;
        }
      }
      if (op == OP_WAVE) {
        pc += run_wave(F, pc, d->aux[0]);
        progress = true;
        if (st->error) break;
        continue;
      }
      if (op == OP_FRAME) {   // a nested frame: run it to its Exits, then continue here
        body_pc = pc + 1;
        enter_nested(d->aux[0]);
        progress = true;
        n_push += fc.push;
        n_pop += fc.pop;
        if (fc.maxd > max_depth) max_depth = fc.maxd;
        return progress;
      }
      if (op == OP_HEAVY_BATCH) {   // 1: build the members one by one (the general path)
        pc += run_batch(F, pc, d->aux[0]);
        progress = true;
        if (st->error) break;
        continue;
      }
      if (op == OP_MERGE && d->aux[5] && (ctx_live(d->aux[6]) < 0 || ctx_live(d->aux[5]) < 0)) break;
      if (op <= OP_TA_GRAD || op == OP_ACC || op == OP_STACK_PUSH || op == OP_STACK_POP) {
        long long cs0 = prof ? clock64() : 0;
        const int r = P.n_swaps && (op == OP_STACK_PUSH || op == OP_STACK_POP) ? 0 : fast_node(d, env, fc);
        if (r < 0) {
          fail(fc.err, fc.err_info);
          break;
        }
        if (r > 0) {
          ++pc;
          progress = true;
          if (prof) { op_cyc[62] += clock64() - cs0; op_cnt[62]++; }
          continue;
        }
      }
      body_pc = pc;
      long long c0 = prof ? clock64() : 0;
      const int16_t hn = ((const int16_t*)d->pad)[5];   // node id (compiler; -1: look it up)
      const int nid = hn >= 0 ? hn : P.order[F.body_off + pc];
      const bool routing = op == OP_SWITCH || op == OP_MERGE || op == OP_MERGE_LOOP || op == OP_NEXTITER ||
                           op == OP_PASS || (op == OP_CONST && d->aux[0] == 1);
      // one call level: heavy nodes and the general ops skip the routing front end
      cur_pc_ = pc;
      cur_F_ = &F;
      int r = op == OP_HEAVY ? eval_heavy_node(*d, nid) : routing ? eval(*d, nid) : eval_cold(*d, nid);
      if (prof) {
        op_cyc[op & 31] += clock64() - c0;
        op_cnt[op & 31]++;
      }
      if (r != EV_OK) break;   // blocked / error: resume at this node (counters folded below)
      ++pc;
      progress = true;
    }
    body_pc = pc;
    n_push += fc.push;
    n_pop += fc.pop;
    if (fc.maxd > max_depth) max_depth = fc.maxd;
    return progress;
  }

  // one step of control evaluation; returns true on progress
  __device__ bool step() {
    if (cur_frame < 0) {
      if (root_pc >= P.n_root_steps) {
        if (!fetched) {
          issue_fetches();
          fetched = true;
          return true;
        }
        return false;
      }
      int s = P.root_steps[root_pc];
      if (s >= kRootPrep) {   // early W^T preparation of a tensor-core LSTMCellGrad node
        if (!prep_early(s & kRootNode)) return false;
        root_pc++;
        return true;
      }
      if (s >= 0) {
        const int nid = s & kRootNode;
        low_root_ = (s & kRootLow) != 0;   // instances of a node no frame waits for
        int r = eval(node(nid), nid);
        low_root_ = false;
        if (r != EV_OK) return false;
        root_pc++;
        return true;
      }
      start_frame(-s - 1);
      return true;
    }
    const DFrame& F = P.frames[cur_frame];
    if (!iter_started) {
      while (oldest < iter && iter_out_[F.iter_base + oldest] == 0) oldest++;
      if (iter - oldest >= F.K) return false;   // parallel_iterations window
      if (iter > F.bound) {
        fail(CF_E_STACK_BUDGET, iter);
        return false;
      }
      int infl = iter - oldest + 1;
      if (cur_frame < 16 && infl > st->max_inflight[cur_frame]) st->max_inflight[cur_frame] = infl;
      iter_started = true;
      lgen_++;
      body_pc = 0;
    }
    bool progress = run_body(F);
    if (body_pc < F.n_body) return progress;
    // the counter's Switch decides: true port dead => the predicate was false (or the frame
    // is dead) => Exit fires once with this iteration's values (reading R2)
    const DNode& cs = node(F.counter_switch);
    if (toks_[cs.out_vid + 1].dead) {
      finish_batch();   // the frame's last batch settles before the frame exits
      // flush partially filled dW chunks before the accumulators leave the frame
      for (int k = 0; k < F.n_body; ++k) {
        const int nid = P.order[F.body_off + k];
        const DNode& dn = node(nid);
        if (dn.op == OP_HEAVY && dn.aux[0] == HK_LSTM_BWD_EW && dw_count_[nid] > 0) {
          if (flush_dw(dn, nid, A.dw_pend[(int64_t)nid * kDwMax * 10 + 9], 0, 0) < 0) return false;
        }
      }
      iv_ = P.in_vids;
      bn_ = nullptr;
      for (int k = 0; k < F.n_exit; ++k) {
        const DNode& x = node(P.order[F.exit_off + k]);
        Tok xt = in_tok_g(x, 0);
        for (int a = 0; a < P.n_accs; ++a)
          if (xt.kind == TK_PTR && xt.v == P.accs[a].base) xt.writer = acc_writer_[a];
        set_out(x, 0, xt);
        Tok c{};
        c.dead = xt.dead;
        c.writer = -1;
        toks_[x.ctrl_vid] = c;
      }
      n_exitf += F.n_exit;
      if (cur_frame < 16) st->trip[cur_frame] += iter;   // summed over a nested frame's instances
      if (F.parent >= 0) {
        leave_nested();
        return true;
      }
      cur_frame = -1;
      root_pc++;
      return true;
    }
    iter++;
    iter_started = false;
    return true;
  }

  __noinline__ __device__ void issue_fetches() {
    for (int i = 0; i < P.n_fetch; ++i) {
      const Tok& t = toks_[P.fetch_vids[i]];
      if (t.dead) {
        A.fetch_dead[i] = 1;
        continue;
      }
      A.fetch_dead[i] = 0;
      int64_t bytes = A.fetch_bytes[i];
      if (t.kind == TK_IMM) {
        uint8_t* o = (uint8_t*)A.fetch_out[i];
        int64_t v = t.v;
        for (int b = 0; b < bytes && b < 8; ++b) o[b] = (uint8_t)(v >> (8 * b));
      } else if (t.kind == TK_PTR && bytes > 0) {
        copy_inst((int64_t)A.fetch_out[i], t.v, bytes, t.writer);
      }
    }
  }

  __device__ void run() {
    st->t_start = globaltimer();
    last_progress = st->t_start;
    // a sending half may reuse its peer's slots only after the receiver finished the
    // previous run (its `done` word carries that run's epoch)
    for (int c = 0; c < P.n_chans; ++c) {
      const DChan& C = P.chans[c];
      if (C.role != 1) continue;
      int spins = 0;
      while (ld_acquire_sys_u64(C.done) + 1 < A.epoch) {
        backoff(spins);
        if ((long long)(globaltimer() - last_progress) > A.watchdog_ns) {
          fail(CF_E_DEADLOCK, -1000 - c);
          break;
        }
      }
    }
    last_progress = globaltimer();
    while (!st->error) {
      long long ci = (kProfBuild && A.prof) ? clock64() : 0;
      bool p = drain();
      if (st->error) break;
      p |= step();
      flush_publish();
      (void)ci;
      if (st->error) break;
      if (fetched && cur_frame < 0 && root_pc >= P.n_root_steps && outstanding == 0) break;
      unsigned long long now = globaltimer();
      if (p) {
        last_progress = now;
      } else if ((long long)(now - last_progress) > A.watchdog_ns) {
        fail(CF_E_DEADLOCK, outstanding);
        break;
      }
    }
    // never leave a helper job in flight (an error can end the loop after start_next_wave()):
    // the helpers must see the quit request between jobs, not inside one
    if (pend_wave_pc_ >= 0) {
      wave_wait();
      pend_wave_pc_ = -1;
    }
    // receiving halves: every message of this run has been copied out of its slot
    if (!st->error)
      for (int c = 0; c < P.n_chans; ++c)
        if (P.chans[c].role == 0) st_release_sys_u64(P.chans[c].done, A.epoch);
    for (int k = 0; k < 64; ++k) {
      st->op_count[k] = op_cnt[k];
      st->op_cycles[k] = op_cyc[k];
    }
    st->op_count[31] = st->smem_mask;   // profiling: which driver arrays live in smem
    st->op_cycles[31] = st->smem_used;
    st->pushes = n_push;
    st->pops = n_pop;
    st->sends = n_sent;
    st->recvs = n_recv;
    st->swap_out = n_swap_out;
    st->swap_in = n_swap_in;
    st->bytes_d2h = b_d2h;
    st->bytes_h2d = b_h2d;
    st->dead_skipped = n_dead;
    st->instances = n_inst;
    st->tiles = n_tiles;
    st->max_depth = max_depth;
    st->exit_fires = n_exitf;
    st->t_end = globaltimer();
    __threadfence();
    *(volatile int*)&st->quit = 1;
  }
};

__device__ void worker_loop(const RunArgs& A) {
  __shared__ __align__(16) float sm[32 * 33 + 32 * 129 + 64];
  __shared__ unsigned long long s_entry;
  __shared__ int s_last, s_use_next;
  // the next tile, claimed by an epilogue thread while the current tensor-core tile's mainloop
  // runs (its record staged here): the claim / record round trips leave the critical path
  __shared__ unsigned long long s_next;
  __shared__ Inst s_inst_next;
  extern __shared__ __align__(1024) uint8_t dyn_smem[];
  RunState* st = A.st;
  const bool tcmode = A.prog.precision == D_BF16;
  tc::TcShared ts{};
  uint32_t tc_cnt = 0, tc_cnt2 = 0, tc_tiles = 0;
  if (tcmode) {
    ts = tc::tc_carve(dyn_smem);
    tc::tc_setup(ts);
  }
  if (threadIdx.x == 0) s_next = ~0ULL;
  __syncthreads();
  // queue entries are instance ids; a tile is claimed with one atomicAdd on the instance's tile
  // counter, and whoever takes (or overshoots) the last tile advances the head past the
  // instance. 1 = claimed (*e), 2 = overshot (retry), 0 = ring empty
  auto claim = [&](unsigned long long* headp, unsigned long long* tailp, const unsigned long long* ring,
                   unsigned long long* e) -> int {
    unsigned long long h = ld_volatile_u64(headp);
    if (h >= ld_volatile_u64(tailp)) return 0;
    __threadfence();
    const int32_t id = (int32_t)((volatile const unsigned long long*)ring)[h & (A.q_cap - 1)];
    const int nt = ((volatile const Inst*)(A.insts + id))->ntiles;
    const int t = atomicAdd(&A.tile_next[id], 1);
    if (t >= nt - 1) atomicCAS(headp, h, h + 1);
    if (t >= nt) return 2;
    *e = ((unsigned long long)id << 32) | (unsigned)t;
    return 1;
  };
  // one non-blocking attempt over both rings (high priority first)
  // SM roles for the low-priority ring (dW chunks, off the critical path): the first n_low
  // workers take low-priority work first; with `strict`, the others never take it (so a long
  // dW tile never holds an SM the recurrence's next tile is waiting for). kLowWorkers = 0:
  // every worker prefers high-priority work (cf_debug_set_worker_roles)
  const int n_low = kLowWorkers & 0xffff;
  const bool low_first = (int)blockIdx.x <= n_low;
  const bool no_low = n_low > 0 && !low_first && (kLowWorkers >> 16);
  // race check (cf_run_opts.sched_seed != 0): every claim attempt first sleeps a pseudo-random
  // 0-4 us and picks the ring order at random, so tiles run in other orders and at other times
  // than FIFO; results must not change (tests/test_gpu_sched.py)
  uint32_t sched_ctr = 0;
  auto try_claim = [&](unsigned long long* e) -> bool {
    bool lf = low_first;
    if (A.sched_seed) {
      uint32_t h = (uint32_t)A.sched_seed * 0x9E3779B9u ^ (blockIdx.x * 0x85EBCA6Bu) ^ (++sched_ctr * 0xC2B2AE35u);
      h ^= h >> 16;
      h *= 0x7FEB352Du;
      h ^= h >> 15;
      __nanosleep(h & 4095);
      lf = lf || (h >> 31);
    }
    for (int k = 0; k < 8; ++k) {
      int r = 0;
      if (lf) {
        r = claim(&st->lq_head, &st->lq_tail, A.lq, e);
        if (r == 1) return true;
        if (r == 2) continue;
      }
      r = claim(&st->q_head, &st->q_tail, A.queue, e);
      if (r == 1) return true;
      if (r == 2) continue;
      if (lf || no_low) return false;
      r = claim(&st->lq_head, &st->lq_tail, A.lq, e);
      if (r == 1) return true;
      if (r == 2) continue;
      return false;
    }
    return false;
  };
  const bool ahead = tcmode && !(kDbgFlags & 64);   // A/B: debug flag bit 6 = no claim-ahead
  auto claim_ahead = [&]() {
    if (!ahead || s_next != ~0ULL) return;
    unsigned long long e;
    if (!try_claim(&e)) return;
    const int32_t id = (int32_t)(e >> 32);
    // the record was published before the claim could see it: after the fence, plain L2 loads
    // (all in flight at once; one round trip instead of one per word)
    __threadfence();
    constexpr int kW = (int)(sizeof(Inst) / 8);
    long long w[kW];
    const long long* src = (const long long*)(A.insts + id);
#pragma unroll
    for (int k = 0; k < kW; ++k) w[k] = __ldcg(src + k);
#pragma unroll
    for (int k = 0; k < kW; ++k) ((long long*)&s_inst_next)[k] = w[k];
    s_next = e;
  };
  while (true) {
    if (threadIdx.x == 0) {
      unsigned long long e = ~0ULL;
      int use_next = 0;
      if (s_next != ~0ULL) {
        e = s_next;
        s_next = ~0ULL;
        use_next = 1;
      } else {
        int spins = 0;
        while (true) {
          if (try_claim(&e)) break;
          if (ld_volatile_i32(&st->quit)) break;
          backoff(spins);
        }
      }
      __threadfence();
      if (A.prog.precision == D_BF16) tc::fence_proxy_async_global();
      s_entry = e;
      s_use_next = use_next;
    }
    __syncthreads();
    unsigned long long e = s_entry;
    if (e == ~0ULL) break;
    const int32_t id = (int32_t)(e >> 32);
    const int tile = (int)(e & 0xffffffffULL);
    unsigned long long t_tile0 = (kProfBuild && A.prof) ? globaltimer() : 0;
    __shared__ Inst s_inst;
    if (threadIdx.x < (int)(sizeof(Inst) / 8))
      ((int64_t*)&s_inst)[threadIdx.x] = s_use_next ? ((const int64_t*)&s_inst_next)[threadIdx.x]
                                                    : ((volatile const int64_t*)(A.insts + id))[threadIdx.x];
    __syncthreads();
    const Inst I = s_inst;
    switch (kDbgFlags & 1 ? (int)HK_NOP : (int)I.kind) {
      case HK_NOP: break;
      case HK_EW: tile_ew(I, tile); break;
      case HK_FILL: tile_fill(I, tile); break;
      case HK_COPY: tile_copy(I, tile); break;
      case HK_ACC: tile_acc(I, tile); break;
      case HK_REDUCE_SUM: tile_reduce_sum(I, tile, sm); break;
      case HK_REDUCE_SUM0: tile_reduce_sum0(I, tile); break;
      case HK_MATMUL: tile_matmul(I, tile, sm); break;
      case HK_LSTM_FWD: tile_lstm_fwd(I, tile, sm); break;
      case HK_LSTM_BWD_EW: tile_lstm_bwd_ew(I, tile); break;
      case HK_LSTM_BWD_MM: tile_lstm_bwd_mm(I, tile, sm); break;
      case HK_PREP_WP: tile_prep_wp(I, tile); break;
      case HK_PREP_WT: tile_prep_wt(I, tile, (float*)dyn_smem); break;
      case HK_LSTM_FWD_TC: tile_lstm_fwd_tc(I, tile, ts, tc_cnt, tc_cnt2, tc_tiles, sm, claim_ahead); break;
      case HK_LSTM_XPROJ_TC: tile_lstm_xproj_tc(I, tile, ts, tc_cnt, tc_cnt2, tc_tiles, claim_ahead); break;
      case HK_LSTM_BWD_EW_BF: tile_lstm_bwd_ew_bf(I, tile, sm); break;
      case HK_LSTM_DXH_TC: tile_lstm_dxh_tc(I, tile, ts, tc_cnt, tc_cnt2, tc_tiles, claim_ahead); break;
      case HK_LSTM_DW_TC: tile_lstm_dw_tc(I, tile, ts, tc_cnt, tc_cnt2, tc_tiles, claim_ahead); break;
      case HK_MATMUL_TC: tile_matmul_tc(I, tile, ts, tc_cnt, tc_tiles, claim_ahead); break;
      default: break;
    }
    // epilogue stores (generic proxy) must be visible to later TMA (async proxy) reads, and a
    // tile's generic shared-memory accesses ordered before the next tile's bulk / TMA writes
    if (tcmode) tc::fence_proxy_async_all();
    __syncthreads();
    if (threadIdx.x == 0) {
      if (kProfBuild && A.prof) {
        unsigned long long t1 = globaltimer();
        unsigned long long* pr = A.prof + 6 * (int64_t)id;
        atomicMin(&pr[2], t_tile0);
        atomicMax(&pr[3], t1);
        atomicAdd(&pr[4], t1 - t_tile0);
      }
      if (I.signal) __threadfence_system();   // peer-visible stores before the count
      __threadfence();
      int old = atomicAdd(&A.inst_tiles_done[id], 1);
      s_last = (old == I.ntiles - 1);
      atomicAdd(&st->q_done, 1ULL);
    }
    __syncthreads();
    if (s_last) {
      if (I.signal && threadIdx.x == 0) {
        __threadfence_system();
        st_release_sys_u64(I.signal, I.signal_value);
      }
      if (I.kind == HK_REDUCE_SUM) {
        __threadfence();
        finalize_reduce_sum(I, sm);
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        __threadfence();
        unsigned long long slot = atomicAdd(&st->cq_tail, 1ULL);
        int* p = &A.cq[slot & (A.cq_cap - 1)];
        int spins = 0;
        while (ld_volatile_i32(p) != 0) {
          if (ld_volatile_i32(&st->quit)) break;
          backoff(spins);
        }
        __threadfence();
        *(volatile int*)p = id + 1;
      }
    }
  }
  if (tcmode) tc::tc_teardown(ts);
}

// per-run parameters (tensor maps, registry, TensorArray bases, feed tokens, fetch targets)
// copied from the pinned staging area by the SMs, not by a copy engine: a caller's large
// host->device copy in flight (the next step's inputs) would queue these small uploads behind
// it and delay the launch by the whole copy (tools/copy_interference.py)
struct StageJob {
  uint8_t* dst;
  const uint8_t* src;   // pinned host memory (UVA: device-accessible)
  unsigned long long bytes;
};
struct StageJobs {
  StageJob j[6];
  int n;
};
__global__ void __launch_bounds__(256) cf_stage_kernel(StageJobs J) {
  const size_t t0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
  for (int k = 0; k < J.n; ++k) {
    const StageJob& sj = J.j[k];
    const bool v16 = (((uintptr_t)sj.dst | (uintptr_t)sj.src) & 15) == 0;
    const size_t n16 = v16 ? sj.bytes / 16 : 0;
    for (size_t i = t0; i < n16; i += nt) ((uint4*)sj.dst)[i] = ((const uint4*)sj.src)[i];
    for (size_t i = n16 * 16 + t0; i < sj.bytes; i += nt) sj.dst[i] = sj.src[i];
  }
}

__global__ void __launch_bounds__(kThreads, 1) cf_driver_kernel(RunArgs A_param) {
  // kernel parameters are addressed through references below; keep them in shared memory
  // (a reference to the parameter block would force a local-memory copy)
  __shared__ __align__(16) RunArgs A;
  if (threadIdx.x == 0) A = A_param;
  __syncthreads();
  if (blockIdx.x == 0) {
    extern __shared__ __align__(1024) uint8_t drv_smem[];
    __shared__ int req[16];   // [0] seq (-1: quit), [1] helpers done, [4..15] copy args
    __shared__ Wave wave;     // routing waves evaluated by the helper warps
    // this run's placeholder tokens into the (zeroed) table before anything reads it
    for (int k = threadIdx.x; k < A.n_preset; k += blockDim.x) A.toks[A.preset[k].vid] = A.preset[k].t;
    __syncthreads();
    Tok* toks = A.toks;
    DNode* smn = nullptr;
    int32_t* smi = nullptr;
    // in-flight instance ring + completion mirror ring (always in smem)
    const int64_t ring_b = (7 + Driver::kInlineSucc) * 4 * 1024;   // in-flight ring (always in smem)
    uint8_t* base = drv_smem + ring_b;
    const int64_t avail = A.dyn_smem - ring_b;
    const int64_t tok_b = (int64_t)A.prog.n_vids * (int64_t)sizeof(Tok);
    const int64_t node_b = (int64_t)A.prog.max_body * (int64_t)sizeof(DNode);
    const int64_t iv_b = ((int64_t)A.prog.max_bi * 4 + 15) / 16 * 16;
    if (tok_b <= avail) {
      // stage the token table (placeholders preset by the host) in shared memory
      Tok* sm = (Tok*)base;
      for (int i = threadIdx.x; i < A.prog.n_vids; i += blockDim.x) sm[i] = A.toks[i];
      toks = sm;
      const int64_t tok_pad = (tok_b + 15) / 16 * 16;
      if (tok_pad + node_b + iv_b <= avail) {
        smn = (DNode*)(base + tok_pad);
        smi = (int32_t*)(base + tok_pad + node_b);
      }
    }
    // further driver-private arrays into the remaining shared memory
    int64_t used = ring_b;
    if (toks != A.toks) used += (tok_b + 15) / 16 * 16 + (smn ? node_b + iv_b : 0);
    auto carve = [&](int64_t bytes) -> uint8_t* {
      bytes = (bytes + 15) / 16 * 16;
      if (toks == A.toks || used + bytes > A.dyn_smem) return nullptr;
      uint8_t* p = drv_smem + used;
      used += bytes;
      return p;
    };
    const Prog& P = A.prog;
    DTA* s_tas = (DTA*)carve((int64_t)P.n_tas * sizeof(DTA));
    int64_t* s_tab = (int64_t*)carve(8 * (int64_t)P.n_tas);
    int32_t* s_tso = (int32_t*)carve(4 * (int64_t)P.n_tas);
    PlaceDesc* s_pl = (PlaceDesc*)carve((int64_t)P.n_places * sizeof(PlaceDesc));
    DReg* s_reg = (DReg*)carve((int64_t)P.n_reg * sizeof(DReg));
    int32_t* s_sd = (int32_t*)carve(4 * (int64_t)P.n_stack_depths);
    int32_t* s_prep = (int32_t*)carve(4 * (int64_t)P.n_nodes);
    int32_t* s_dwc = (int32_t*)carve(4 * (int64_t)P.n_nodes);
    int32_t* s_accw = (int32_t*)carve(4 * (int64_t)P.n_accs);
    int32_t* s_iter = (int32_t*)carve(4 * (int64_t)P.iter_counters);
    int32_t* s_ring = (int32_t*)drv_smem;
    DStack* s_stk = (DStack*)carve((int64_t)P.n_stacks * sizeof(DStack));
    if (threadIdx.x == 0) {
      A.st->smem_mask = (toks != A.toks) | (smn ? 2 : 0) | (s_pl ? 4 : 0) | (s_reg ? 8 : 0) |
                        (s_sd ? 16 : 0) | (s_prep ? 32 : 0) | (s_dwc ? 64 : 0) | (s_accw ? 128 : 0) |
                        (s_iter ? 256 : 0) | (s_stk ? 512 : 0);
      A.st->smem_used = (int32_t)used;
    }
    for (int i = threadIdx.x; s_tas && i < P.n_tas; i += blockDim.x) s_tas[i] = P.tas[i];
    for (int i = threadIdx.x; s_tab && i < P.n_tas; i += blockDim.x) s_tab[i] = A.ta_base[i];
    for (int i = threadIdx.x; s_tso && i < P.n_tas; i += blockDim.x) s_tso[i] = A.ta_slot_off[i];
    for (int i = threadIdx.x; s_pl && i < P.n_places; i += blockDim.x) s_pl[i] = P.places[i];
    for (int i = threadIdx.x; s_reg && i < P.n_reg; i += blockDim.x) s_reg[i] = P.reg[i];
    for (int i = threadIdx.x; s_sd && i < P.n_stack_depths; i += blockDim.x) s_sd[i] = 0;
    for (int i = threadIdx.x; s_prep && i < P.n_nodes; i += blockDim.x) s_prep[i] = -1;
    for (int i = threadIdx.x; s_dwc && i < P.n_nodes; i += blockDim.x) s_dwc[i] = 0;
    for (int i = threadIdx.x; s_accw && i < P.n_accs; i += blockDim.x) s_accw[i] = -1;
    for (int i = threadIdx.x; s_iter && i < P.iter_counters; i += blockDim.x) s_iter[i] = 0;
    for (int i = threadIdx.x; s_ring && i < 1024; i += blockDim.x) s_ring[i] = -1;
    for (int i = threadIdx.x; s_stk && i < P.n_stacks; i += blockDim.x) s_stk[i] = P.stacks[i];
    if (threadIdx.x == 0) {
      req[0] = 0;
      req[1] = 0;
      wave.seq = 0;
      wave.done = 0;
      wave.bseq = 0;
      wave.bphase = 0;
      wave.bdone = 0;
      wave.bgo = 0;
      wave.nw = kWaveWarps;
      wave.skip1 = 0;
      wave.env_frame = -2;
      wave.job = 0;
      wave.chain = 0;
    }
    __syncthreads();
    // the driver object itself lives in shared memory: its members are touched on every node
    // evaluation, and local memory would go to L2 (this SM has almost no L1 left)
    __shared__ __align__(16) unsigned char drv_obj[sizeof(Driver)];
    if (threadIdx.x == 0) {
      Driver& d = *new (drv_obj) Driver(A, toks, smn, smi, req);
      d.wave_ = &wave;
      d.dbg_ = kDbgFlags;
      if ((d.dbg_ >> 8) & 255) d.drain_cycles_ = 1000LL * ((d.dbg_ >> 8) & 255);

      if (s_pl) d.places_ = s_pl;
      if (s_reg) d.reg_ = s_reg;
      if (s_sd) d.stack_depth_ = s_sd;
      if (s_prep) d.prep_inst_ = s_prep;
      if (s_dwc) d.dw_count_ = s_dwc;
      if (s_accw) d.acc_writer_ = s_accw;
      if (s_iter) d.iter_out_ = s_iter;
      if (!s_ring) {
        d.fail(CF_E_UNSUPPORTED, -7);   // no room for the in-flight ring
      } else {
        d.r_id = s_ring;
        d.r_pend = s_ring + 1024;
        d.r_succ = s_ring + 2048;
        d.r_last = s_ring + 3072;
        d.r_nt = s_ring + 4096;
        d.r_kfi = s_ring + 5120;
        d.r_sn = s_ring + 6144;
        d.r_sv = s_ring + 7168;
      }
      if (s_stk) d.stacks_ = s_stk;
      if (s_tas && s_tab && s_tso) {
        d.tas_ = s_tas;
        d.tab_ = s_tab;
        d.tso_ = s_tso;
      }
      for (int f = 0; f < P.n_frames && f < Driver::kIbCache; ++f) d.ib_[f] = P.frames[f].iter_base;
      d.ctxs_ = P.ctxs;
      for (int c = 0; c < P.n_ctxs && c < Driver::kMaxCtx; ++c) {
        d.lstamp_[c] = 0;
        d.lval_[c] = 0;
      }
      d.run();
      d.finish_batch();   // (an error path may leave a batch job's lanes running)
      *(volatile int*)&req[0] = -1;
    } else if (threadIdx.x >= 32) {
      // helper warps: cooperative smem staging on request from the driver thread
      int seen = 0, wseen = 0, bseen = 0;
      const bool nosleep = kDbgFlags & 8;   // A/B knob: wave helpers spin without sleeping
      const int h = threadIdx.x - 32, nh = blockDim.x - 32;
      while (true) {
        int q = *(volatile int*)&req[0];
        if (q < 0) break;
        if ((threadIdx.x >> 5) == 1) {   // warp 1: batch jobs first (their own counter)
          const int bs = *(volatile int*)&wave.bseq;
          if (bs != bseen) {
            bseen = bs;
            __threadfence_block();
            ((Driver*)drv_obj)->batch_lane_par(wave, threadIdx.x & 31);
            continue;
          }
        }
        const int ws = (threadIdx.x >> 5) == 4 ? wseen : *(volatile int*)&wave.seq;
        if (ws != wseen) {
          wseen = ws;
          __threadfence_block();
          // whether warp 1 takes part comes with the request number itself (bit 0): warp 1 may
          // read the number of a job it sat out only after the next job's fields were written
          const bool no1 = ws & 1;
          if (no1 && (threadIdx.x >> 5) == 1) continue;
          const int nthr = no1 ? 32 * (kWaveWarps - 1) : 32 * kWaveWarps;
          const int hl = no1 ? wave_lane5(threadIdx.x) : wave_lane(threadIdx.x);
          if (wave.job == 1) {
            ((Driver*)drv_obj)->heavy_prep_lane(wave, hl);
          } else if (wave.job == 2) {
            if ((threadIdx.x >> 5) == 1) ((Driver*)drv_obj)->batch_lane(wave, threadIdx.x & 31);
          } else {
            // fused levels: each reads the previous one's tokens (named barrier between)
            int k = 0;
            for (; k < wave.nlev; ++k) {
              if (k > 0 && (wave.lev_ctx[k] | wave.lev_ctx_hi[k])) {   // this level's contexts
                if (hl == 0 && !((Driver*)drv_obj)->helper_ctx(wave.lev_ctx[k], wave.lev_ctx_hi[k]))
                  wave.cstop = k;
                __threadfence_block();
                asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
                if (wave.cstop >= 0) break;
              }
              wave_work(wave, wave.lev_start[k], wave.lev_n[k], hl, nthr);
              __threadfence_block();
              asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
              if (wave.nslow || wave.cnt.err) break;   // the driver evaluates the leftovers
            }
            if (hl == 0) wave.lev_stop = wave.cstop >= 0 ? wave.cstop : k < wave.nlev ? k : wave.nlev;
            if (k == wave.nlev && wave.chain)   // the next node's preparation
              ((Driver*)drv_obj)->heavy_prep_lane(wave, hl);
          }
          __threadfence_block();
          __syncwarp();
          if ((threadIdx.x & 31) == 0) atomicAdd(&wave.done, 1);
          continue;
        }
        if (q == seen) {
          if ((threadIdx.x >> 5) == 4) __nanosleep(500);
          else if (!nosleep) __nanosleep(20);
          continue;
        }
        seen = q;
        const int64_t* a = (const int64_t*)(req + 4);
        for (int part = 0; part < 2; ++part) {
          int4* dst = (int4*)a[3 * part];
          const int4* src = (const int4*)a[3 * part + 1];
          int64_t n = (a[3 * part + 2] + 15) / 16;
          for (int64_t i = h; i < n; i += nh) dst[i] = src[i];
        }
        __threadfence_block();
        __syncwarp();
        if ((threadIdx.x & 31) == 0) atomicAdd(&req[1], 1);
      }
    }
    return;
  }
  worker_loop(A);
}

}  // namespace

// ============================================================================= host side
struct cf_session {
  cf::HostProgram P;
  int device = 0;
  int precision = CF_F32;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int grid = 0;
  std::vector<void*> allocs;
  std::vector<void*> buf_ptr;
  RunArgs args{};
  // device copies of tables
  void* d_tables = nullptr;
  RunState* d_state = nullptr;
  void** d_fetch_out = nullptr;
  uint8_t* d_fetch_dead = nullptr;
  int64_t* d_fetch_bytes = nullptr;
  int64_t* d_ta_base_init = nullptr;
  std::vector<int64_t> ta_base_host;
  size_t state_bytes = 0;
  void* d_state_block = nullptr;   // zeroed at every run
  std::vector<std::pair<void*, size_t>> zero_each_run;
  std::vector<std::pair<void*, int>> fill_ff_each_run;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_in = nullptr;
  int64_t watchdog_ns = 60LL * 1000 * 1000 * 1000;
  int sched_seed = 0;
  int dyn_smem = 0;
  std::vector<DReg> reg_host;
  std::vector<CUtensorMap> maps_host;
  int n_reg_static = 0;
  std::vector<DReg> reg_sorted;   // per-run upload, sorted by base
  // per-run parameters (tensor maps of bf16 feeds, registry, TA bases, placeholder tokens,
  // fetch pointers) go through one pinned staging area: every upload is asynchronous, no
  // stream synchronisation before the launch
  uint8_t* stage_host = nullptr;
  size_t stage_cap = 0;
  PresetTok* d_preset = nullptr;
  int preset_cap = 0;
  // cross-GPU channels (a14): this session's halves live in one IPC-exported allocation
  void* chan_mem = nullptr;
  std::vector<DChan> chans;        // device view (remote pointers filled by cf_session_connect)
  DChan* d_chans = nullptr;
  bool chans_dirty = true;
  std::map<int, void*> peer_mem;   // imported peer channel memory, by peer rank
  unsigned long long epoch = 0;
  // stack swapping (a8): pinned host backing + the host I/O thread's request ring / streams
  std::vector<void*> host_allocs;
  unsigned long long* io_req_host = nullptr;    // mapped [io_cap][4]
  unsigned long long* io_tail_host = nullptr;   // mapped, written by the driver
  int32_t* io_ids_host = nullptr;               // pinned completion words (id + 1)
  // several copy streams per direction so that the per-copy setup of the 1-4 MB swap copies
  // overlaps the previous transfer (round robin)
  static constexpr int kIoStreams = 3;
  cudaStream_t io_d2h[kIoStreams] = {}, io_h2d[kIoStreams] = {};
  cudaStream_t user_d2h = nullptr, user_h2d = nullptr;   // caller's copy streams (cf_run_opts)
  void* (*dev_alloc)(size_t, void*) = nullptr;           // caller allocator (cf_run_opts)
  void (*dev_free)(void*, void*) = nullptr;
  void* alloc_user = nullptr;
};

namespace {

// bytes of a dense cf_buffer (rank 0..8, non-negative extents); -1 when malformed
int64_t buffer_bytes(const cf_buffer& b) {
  static const int sz[] = {1, 4, 8, 4, 8, 2};
  if (b.rank < 0 || b.rank > 8 || b.dtype < 0 || b.dtype > 5) return -1;
  int64_t n = sz[b.dtype];
  for (int k = 0; k < b.rank; ++k) {
    if (b.shape[k] < 0) return -1;
    n *= b.shape[k];
  }
  return n;
}

// every session-owned device buffer: the caller's allocator when one is given (cf_run_opts)
void* dalloc(cf_session* s, size_t bytes) {
  void* p = nullptr;
  bytes = std::max<size_t>(bytes, 16);
  if (s->dev_alloc) {
    p = s->dev_alloc(bytes, s->alloc_user);
    if (!p) throw cf::CfError(CF_E_CUDA, "caller allocator returned NULL for " + std::to_string(bytes) + " bytes");
    if ((uintptr_t)p % 256) {
      s->dev_free(p, s->alloc_user);
      throw cf::CfError(CF_E_CUDA, "caller allocator returned a pointer not 256-byte aligned");
    }
  } else {
    CUDA_OK(cudaMalloc(&p, bytes));
  }
  s->allocs.push_back(p);
  return p;
}

template <class T>
T* upload(cf_session* s, const std::vector<T>& v) {
  void* p = dalloc(s, v.size() * sizeof(T));
  if (!v.empty()) CUDA_OK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return (T*)p;
}

// Host I/O executor (one thread per run of a session with swapped stacks): takes the driver's
// swap requests from the mapped ring in order and issues them on the D2H / H2D copy streams,
// each followed by a 4-byte completion write into io_cq (stream-ordered after the data).
// stream-ordered 32-bit store (driver API cuStreamWriteValue32): the completion word needs no
// copy-engine transfer of its own
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_writeValue32 get_write_value32() {
  static PFN_writeValue32 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_writeValue32)p;
  }
  return fn;
}

void io_executor(cf_session* s, std::atomic<bool>* stop, std::atomic<int>* err) {
  cudaSetDevice(s->device);
  PFN_writeValue32 wv = get_write_value32();
  const unsigned long long m = (unsigned long long)(s->args.io_cap - 1);
  unsigned long long head = 0;
  int idle = 0;
  while (true) {
    const unsigned long long tail = *(volatile unsigned long long*)s->io_tail_host;
    if (head < tail) {
      std::atomic_thread_fence(std::memory_order_acquire);
      volatile unsigned long long* e = s->io_req_host + 4 * (head & m);
      const unsigned long long src = e[0], dst = e[1], bytes = e[2], w = e[3];
      const int id = (int)(w & 0xffffffffULL), dir = (int)(w >> 32);
      cudaStream_t st = dir == 0 ? s->io_d2h[head % cf_session::kIoStreams]
                                 : s->io_h2d[head % cf_session::kIoStreams];
      s->io_ids_host[head & m] = id + 1;
      cudaError_t r = cudaMemcpyAsync((void*)dst, (const void*)src, bytes,
                                      dir == 0 ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, st);
      if (r == cudaSuccess) {
        if (wv) {
          if (wv((CUstream)st, (CUdeviceptr)(s->args.io_cq + (head & m)), (cuuint32_t)(id + 1), 0) != CUDA_SUCCESS)
            r = cudaErrorUnknown;
        } else {
          r = cudaMemcpyAsync(s->args.io_cq + (head & m), s->io_ids_host + (head & m), 4,
                              cudaMemcpyHostToDevice, st);
        }
      }
      if (r != cudaSuccess) err->store(1);
      head++;
      idle = 0;
      continue;
    }
    if (stop->load()) break;
    if (++idle > 64) std::this_thread::yield();
  }
}

void build_session(cf_session* s, const cf::Graph& g, const cf_run_opts* o,
                   const std::vector<cf::TRef>& fetches) {
  cf::CompileOpts co;
  if (o) {
    co.precision = o->precision ? o->precision : CF_F32;
    co.parallel_iterations = o->parallel_iterations;
    co.max_iterations = o->max_iterations;
    co.stack_budget_bytes = o->stack_budget_bytes > 0 ? o->stack_budget_bytes : -1;
    co.swap_min_bytes = o->swap_min_bytes > 0 ? o->swap_min_bytes : 4096;
    co.swap_smallest_first = o->swap_smallest_first != 0;
    s->device = o->device;
    if (o->watchdog_ms > 0) s->watchdog_ns = o->watchdog_ms * 1000000LL;
    s->sched_seed = o->sched_seed;
    if ((o->dev_alloc != nullptr) != (o->dev_free != nullptr))
      throw cf::CfError(CF_E_UNSUPPORTED, "cf_run_opts: dev_alloc and dev_free go together");
    s->dev_alloc = o->dev_alloc;
    s->dev_free = o->dev_free;
    s->alloc_user = o->alloc_user;
    s->user_d2h = (cudaStream_t)o->d2h_stream;
    s->user_h2d = (cudaStream_t)o->h2d_stream;
  }
  if (co.precision != CF_F32 && co.precision != CF_BF16)
    throw cf::CfError(CF_E_DTYPE, "precision must be CF_F32 or CF_BF16");
  s->precision = co.precision;
  s->P = cf::compile(g, co, fetches);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw cf::CfError(CF_E_CUDA, "no CUDA device (libcf has no CPU fallback)");
  CUDA_OK(cudaSetDevice(s->device));
  if (o && o->stream) {
    s->stream = (cudaStream_t)o->stream;
  } else {
    CUDA_OK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    s->own_stream = true;
  }
  CUDA_OK(cudaEventCreate(&s->ev0));
  CUDA_OK(cudaEventCreate(&s->ev1));
  CUDA_OK(cudaEventCreateWithFlags(&s->ev_in, cudaEventDisableTiming));
  cf::HostProgram& P = s->P;
  // ---- buffers
  s->buf_ptr.resize(P.bufs.size());
  for (size_t b = 0; b < P.bufs.size(); ++b) {
    void* p = dalloc(s, P.bufs[b].bytes);
    s->buf_ptr[b] = p;
    if (!P.bufs[b].init.empty())
      CUDA_OK(cudaMemcpy(p, P.bufs[b].init.data(), P.bufs[b].init.size(), cudaMemcpyHostToDevice));
    if (P.bufs[b].zero) s->zero_each_run.push_back({p, P.bufs[b].bytes});
  }
  auto addr = [&](int64_t id) { return (int64_t)(uintptr_t)s->buf_ptr.at(id); };
  for (auto& pl : P.places)
    if (pl.kind != PL_TA && pl.kind != PL_ACC) pl.base = addr(pl.base);
  for (auto& n : P.nodes)
    if (n.op == OP_CONST && n.aux[0] == 0) n.imm[0] = addr(n.imm[0]);
  for (auto& n : P.body_nodes)
    if (n.op == OP_CONST && n.aux[0] == 0) n.imm[0] = addr(n.imm[0]);
  for (auto& t : P.tas) t.base = addr(t.base);
  for (auto& a : P.accs) a.base = addr(a.base);
  for (auto& r : P.reg) r.base = addr(r.base);
  s->ta_base_host.clear();
  for (auto& t : P.tas) s->ta_base_host.push_back(t.base);
  // ---- tables
  RunArgs& A = s->args;
  Prog& pg = A.prog;
  pg.n_nodes = (int)P.nodes.size();
  pg.n_vids = P.n_vids;
  pg.n_frames = (int)P.frames.size();
  pg.n_tas = (int)P.tas.size();
  pg.n_stacks = (int)P.stacks.size();
  pg.n_stack_depths = P.stack_depths;
  pg.nested = P.nested ? 1 : 0;
  pg.n_root_steps = (int)P.root_steps.size();
  pg.n_fetch = (int)P.fetches.size();
  pg.n_conds = P.n_conds;
  pg.branch_bound = P.branch_bound;
  pg.dw_chunk = P.dw_chunk;
  pg.nodes = upload(s, P.nodes);
  pg.in_vids = upload(s, P.in_vids);
  pg.places = upload(s, P.places);
  pg.frames = upload(s, P.frames);
  pg.order = upload(s, P.order);
  pg.root_steps = upload(s, P.root_steps);
  pg.tas = upload(s, P.tas);
  pg.stacks = upload(s, P.stacks);
  pg.fetch_vids = upload(s, P.fetch_vids);
  pg.body_nodes = upload(s, P.body_nodes);
  pg.body_ivids = upload(s, P.body_ivids);
  pg.max_body = P.max_body;
  pg.max_bi = P.max_bi;
  pg.n_places = (int)P.places.size();
  pg.iter_counters = P.iter_counters;
  pg.accs = upload(s, P.accs);
  pg.n_accs = (int)P.accs.size();
  pg.precision = s->precision == CF_BF16 ? D_BF16 : D_F32;
  // ---- TMA operand registry: 3 tensor maps per bf16 buffer (K-major A / B boxes, MN box);
  //      feeds are appended at every cf_run
  {
    int n_static = (int)P.reg.size();
    int cap = n_static + (int)P.feeds.size() + 1;
    std::vector<CUtensorMap> maps((size_t)3 * cap);
    for (int i = 0; i < n_static; ++i) {
      DReg& r = P.reg[i];
      r.map0 = 3 * i;
      maps[3 * i + 0] = cf::make_map_bf16_strided((void*)r.base, r.cols, r.rows, r.slots, r.slot_bytes, 64, 128);
      maps[3 * i + 1] = cf::make_map_bf16_strided((void*)r.base, r.cols, r.rows, r.slots, r.slot_bytes, 64, 256);
      maps[3 * i + 2] = cf::make_map_bf16_strided((void*)r.base, r.cols, r.rows, r.slots, r.slot_bytes, 64, 64);
    }
    s->reg_host = P.reg;
    s->reg_host.resize(cap);
    s->maps_host = maps;
    s->n_reg_static = n_static;
    pg.reg = (const DReg*)dalloc(s, sizeof(DReg) * cap);
    pg.maps = dalloc(s, sizeof(CUtensorMap) * 3 * cap);
    CUDA_OK(cudaMemcpy((void*)pg.reg, s->reg_host.data(), sizeof(DReg) * cap, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy((void*)pg.maps, maps.data(), sizeof(CUtensorMap) * 3 * cap, cudaMemcpyHostToDevice));
    pg.n_reg = n_static;
  }
  A.vdt = upload(s, P.vdt);
  // ---- channel halves (a14): zeroed once; epochs keep runs apart
  if (!P.chans.empty()) {
    CUDA_OK(cudaMalloc(&s->chan_mem, (size_t)P.chan_bytes));
    CUDA_OK(cudaMemset(s->chan_mem, 0, (size_t)P.chan_bytes));
    for (auto& c : P.chans) {
      DChan d{};
      d.channel = c.channel;
      d.role = c.role;
      d.peer = c.peer;
      d.slots = c.slots;
      d.elem_bytes = c.elem_bytes;
      d.dt = c.dt;
      d.frame = c.frame;
      uint8_t* base = (uint8_t*)s->chan_mem + c.offset;
      const int64_t fb = ((int64_t)c.slots * 8 + 255) / 256 * 256;
      if (c.role == 0) {
        d.flags = (unsigned long long*)base;
        d.data = base + fb;
      } else {
        d.acks = (unsigned long long*)base;
        d.done = (unsigned long long*)(base + fb);
      }
      s->chans.push_back(d);
    }
    s->d_chans = (DChan*)dalloc(s, sizeof(DChan) * s->chans.size());
  }
  A.prog.n_chans = (int32_t)s->chans.size();
  A.prog.chans = s->d_chans;
  A.prog.n_ctxs = (int32_t)P.ctxs.size();
  A.prog.ctxs = upload(s, P.ctxs);
  // ---- swapped stack arenas (a8)
  A.io_cap = 4096;
  if (!P.swaps.empty()) {
    std::vector<DSwap> sw;
    int owner_total = 0;
    for (auto& sp : P.swaps) {
      DSwap d{};
      d.dev_base = P.places[sp.place].base;
      d.in_base = (int64_t)(uintptr_t)s->buf_ptr.at(sp.in_buf);
      d.elem_bytes = sp.elem_bytes;
      d.ring = sp.ring;
      d.capacity = sp.capacity;
      d.in_ring = sp.in_ring;
      d.owner_off = owner_total;
      owner_total += sp.ring;
      void* h = nullptr;
      CUDA_OK(cudaHostAlloc(&h, (size_t)sp.capacity * sp.elem_bytes, cudaHostAllocPortable));
      s->host_allocs.push_back(h);
      d.host_base = (int64_t)(uintptr_t)h;
      sw.push_back(d);
    }
    A.prog.swaps = upload(s, sw);
    A.prog.n_swaps = (int32_t)sw.size();
    A.swap_owner = (int32_t*)dalloc(s, 4 * (size_t)owner_total);
    s->fill_ff_each_run.push_back({A.swap_owner, 4 * owner_total});
    CUDA_OK(cudaHostAlloc((void**)&s->io_req_host, 32 * (size_t)A.io_cap, cudaHostAllocMapped));
    CUDA_OK(cudaHostAlloc((void**)&s->io_tail_host, 64, cudaHostAllocMapped));
    CUDA_OK(cudaHostAlloc((void**)&s->io_ids_host, 4 * (size_t)A.io_cap, cudaHostAllocDefault));
    s->host_allocs.push_back(s->io_req_host);
    s->host_allocs.push_back(s->io_tail_host);
    s->host_allocs.push_back(s->io_ids_host);
    CUDA_OK(cudaHostGetDevicePointer((void**)&A.io_req, s->io_req_host, 0));
    CUDA_OK(cudaHostGetDevicePointer((void**)&A.io_req_tail, s->io_tail_host, 0));
    A.io_cq = (int32_t*)dalloc(s, 4 * (size_t)A.io_cap);
    s->zero_each_run.push_back({A.io_cq, 4 * (size_t)A.io_cap});
    for (int k = 0; k < cf_session::kIoStreams; ++k) {
      if (s->user_d2h) s->io_d2h[k] = s->user_d2h;   // the caller's streams: not destroyed
      else CUDA_OK(cudaStreamCreateWithFlags(&s->io_d2h[k], cudaStreamNonBlocking));
      if (s->user_h2d) s->io_h2d[k] = s->user_h2d;
      else CUDA_OK(cudaStreamCreateWithFlags(&s->io_h2d[k], cudaStreamNonBlocking));
    }
  }
  A.inst_aux = (int64_t*)dalloc(s, 8 * kDwMax * 6 * (size_t)P.inst_bound);
  A.dw_count = (int32_t*)dalloc(s, 4 * P.nodes.size());
  s->zero_each_run.push_back({A.dw_count, 4 * P.nodes.size()});
  A.dw_pend = (int64_t*)dalloc(s, 8 * kDwMax * 10 * P.nodes.size());
  A.prep_inst = (int32_t*)dalloc(s, 4 * P.nodes.size());
  s->fill_ff_each_run.push_back({A.prep_inst, (int)(4 * P.nodes.size())});
  A.acc_writer = (int32_t*)dalloc(s, 4 * std::max<size_t>(P.accs.size(), 1));
  s->fill_ff_each_run.push_back({A.acc_writer, (int)(4 * std::max<size_t>(P.accs.size(), 1))});
  // ---- runtime state
  A.st = (RunState*)dalloc(s, sizeof(RunState));
  s->zero_each_run.push_back({A.st, sizeof(RunState)});
  A.toks = (Tok*)dalloc(s, sizeof(Tok) * P.n_vids);
  A.wait_ovf = (int32_t*)dalloc(s, 4 * Driver::kWaitOvf);
  s->preset_cap = (int)std::max<size_t>(P.feeds.size(), 1);
  s->d_preset = (PresetTok*)dalloc(s, sizeof(PresetTok) * s->preset_cap);
  s->zero_each_run.push_back({A.toks, sizeof(Tok) * P.n_vids});
  A.stack_pool = (Tok*)dalloc(s, sizeof(Tok) * std::max(P.stack_pool, 1));
  A.stack_depth = (int32_t*)dalloc(s, 4 * std::max<size_t>(P.stack_depths, 1));
  s->zero_each_run.push_back({A.stack_depth, 4 * std::max<size_t>(P.stack_depths, 1)});
  A.ta_base = (int64_t*)dalloc(s, 8 * std::max<size_t>(P.tas.size(), 1));
  std::vector<int32_t> slot_off;
  int so = 0;
  for (auto& t : P.tas) {
    slot_off.push_back(so);
    so += t.size;
  }
  A.ta_slot_off = upload(s, slot_off);
  A.ta_writer = (int32_t*)dalloc(s, 4 * std::max(so, 1));
  s->fill_ff_each_run.push_back({A.ta_writer, 4 * std::max(so, 1)});
  A.ta_written = (uint8_t*)dalloc(s, std::max(so, 1));
  s->zero_each_run.push_back({A.ta_written, (size_t)std::max(so, 1)});
  int64_t cap = P.inst_bound;
  A.inst_cap = (int32_t)cap;
  A.insts = (Inst*)dalloc(s, sizeof(Inst) * cap);
  A.tile_next = (int32_t*)dalloc(s, 4 * cap);
  s->zero_each_run.push_back({A.tile_next, (size_t)(4 * cap)});
  A.inst_tiles_done = (int32_t*)dalloc(s, 4 * cap);
  s->zero_each_run.push_back({A.inst_tiles_done, (size_t)(4 * cap)});
  A.edge_cap = (int32_t)std::min<int64_t>(cap * 24, 1LL << 30);
  A.edge_next = (int32_t*)dalloc(s, 4 * (size_t)A.edge_cap);
  A.edge_to = (int32_t*)dalloc(s, 4 * (size_t)A.edge_cap);
  A.q_cap = 1ULL << 22;
  A.queue = (unsigned long long*)dalloc(s, 8 * A.q_cap);
  A.lq = (unsigned long long*)dalloc(s, 8 * A.q_cap);
  A.cq_cap = 1ULL << 16;
  A.cq = (int32_t*)dalloc(s, 4 * A.cq_cap);
  s->zero_each_run.push_back({A.cq, 4 * A.cq_cap});
  A.iter_outstanding = (int32_t*)dalloc(s, 4 * std::max(P.iter_counters, 1));
  s->zero_each_run.push_back({A.iter_outstanding, 4 * (size_t)std::max(P.iter_counters, 1)});
  size_t bb = (size_t)std::max(P.n_conds, 1) * P.branch_bound;
  A.branch_bits = (uint8_t*)dalloc(s, bb);
  s->zero_each_run.push_back({A.branch_bits, bb});
  std::vector<int64_t> fb;
  for (auto& f : P.fetches) fb.push_back(f.bytes);
  A.fetch_bytes = upload(s, fb);
  A.fetch_out = (void**)dalloc(s, 8 * std::max<size_t>(P.fetches.size(), 1));
  A.fetch_dead = (uint8_t*)dalloc(s, std::max<size_t>(P.fetches.size(), 1));
  A.watchdog_ns = s->watchdog_ns;
  A.prof = nullptr;
  if (o && o->reserved[0]) A.prof = (unsigned long long*)dalloc(s, 6 * 8 * (size_t)cap);
  A.sched_seed = s->sched_seed;
  // ---- grid: one CTA per SM, all co-resident (cooperative launch)
  int sms = 0, per_sm = 0;
  s->dyn_smem = s->precision == CF_BF16 ? tc::kSmemTC : 0;
  // driver CTA: ring + tokens + body program + private arrays; capped below the opt-in limit
  size_t need = (7 + 4) * 4 * 1024;   // in-flight ring incl. inline successors (kInlineSucc)
  need += (sizeof(Tok) * (size_t)P.n_vids + 15) / 16 * 16;
  need += sizeof(DNode) * (size_t)P.max_body + ((size_t)P.max_bi * 4 + 15) / 16 * 16;
  need += sizeof(PlaceDesc) * P.places.size() + sizeof(DReg) * (P.reg.size() + P.feeds.size() + 1);
  need += sizeof(DStack) * P.stacks.size() + 4 * (size_t)P.stack_depths + 8 * P.nodes.size() +
          4 * (P.accs.size() + P.iter_counters);
  need += (sizeof(DTA) + 12) * P.tas.size() + 48;
  need += 16 * 12;
  // dynamic shared memory: what the opt-in limit leaves next to the kernel's static smem
  cudaFuncAttributes fa{};
  CUDA_OK(cudaFuncGetAttributes(&fa, cf_driver_kernel));
  int optin = 0;
  CUDA_OK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, s->device));
  const size_t smem_cap = (size_t)optin - fa.sharedSizeBytes;
  if ((size_t)s->dyn_smem > smem_cap) throw cf::CfError(CF_E_CUDA, "tile engine does not fit in shared memory");
  if ((int)std::min(need, smem_cap) > s->dyn_smem) s->dyn_smem = (int)std::min(need, smem_cap);
  A.dyn_smem = s->dyn_smem;
  CUDA_OK(cudaFuncSetAttribute(cf_driver_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, s->dyn_smem));
  CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device));
  CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cf_driver_kernel, kThreads, s->dyn_smem));
  if (per_sm < 1) throw cf::CfError(CF_E_CUDA, "driver kernel cannot be resident");
  int workers = o && o->num_workers > 0 ? o->num_workers : sms - 1;
  s->grid = std::min(workers + 1, sms * per_sm);
  A.num_workers = s->grid - 1;
}

}  // namespace

extern "C" {

cf_status cf_session_create(const cf_graph* g, const cf_run_opts* opts, int32_t n_fetch,
                            const cf_tensor* fetches, cf_session** out) {
  cf_session* s = nullptr;
  try {
    if (!g || !out) throw cf::CfError(CF_E_INVALID_GRAPH, "null argument");
    const cf::Graph& ir = cf_graph_ir(g);
    std::vector<cf::TRef> fv;
    for (int i = 0; i < n_fetch; ++i) {
      if (fetches[i].node < 0 || fetches[i].node >= (int)ir.nodes.size())
        throw cf::CfError(CF_E_INVALID_GRAPH, "bad fetch tensor");
      fv.push_back(cf::TRef{fetches[i].node, fetches[i].port});
    }
    s = new cf_session();
    build_session(s, ir, opts, fv);
    *out = s;
    return CF_OK;
  } catch (const cf::CfError& e) {
    cf::set_error(e.what());
    if (s) cf_session_destroy(s);
    return e.code;
  } catch (const std::exception& e) {
    cf::set_error(std::string("internal: ") + e.what());
    if (s) cf_session_destroy(s);
    return CF_E_INVALID_GRAPH;
  }
}

cf_status cf_run(cf_session* s, int32_t n_feed, const char* const* feed_names,
                 const cf_buffer* feeds, cf_buffer* outs, uint8_t* out_dead, cf_trace* trace) {
  try {
    if (!s) throw cf::CfError(CF_E_INVALID_GRAPH, "null session");
    cf::HostProgram& P = s->P;
    RunArgs& A = s->args;
    CUDA_OK(cudaSetDevice(s->device));
    for (auto& [p, b] : s->zero_each_run) CUDA_OK(cudaMemsetAsync(p, 0, b, s->stream));
    for (auto& [p, b] : s->fill_ff_each_run) CUDA_OK(cudaMemsetAsync(p, 0xff, b, s->stream));
    // token presets: placeholders
    std::vector<Tok> preset;
    std::vector<int> preset_vid;
    std::map<std::string, int> seen;
    for (int i = 0; i < n_feed; ++i) seen[feed_names[i]] = i;
    for (auto& [name, fi] : P.feeds) {
      auto it = seen.find(name);
      if (it == seen.end()) throw cf::CfError(CF_E_MISSING_FEED, "no feed for placeholder " + name);
      const cf_buffer& b = feeds[it->second];
      if (!b.data && fi.bytes > 0) throw cf::CfError(CF_E_MISSING_FEED, "null feed " + name);
      if (b.dtype != fi.dev_dt)
        throw cf::CfError(CF_E_DTYPE, "feed " + name + " has dtype " + std::to_string(b.dtype) +
                                          ", session expects " + std::to_string(fi.dev_dt));
      if (buffer_bytes(b) != fi.bytes)
        throw cf::CfError(CF_E_SHAPE, "feed " + name + " holds " + std::to_string(buffer_bytes(b)) +
                                          " bytes, placeholder needs " + std::to_string(fi.bytes));
      Tok t{};
      t.kind = TK_PTR;
      t.v = (int64_t)(uintptr_t)b.data;
      t.writer = -1;
      t.dt = (uint8_t)fi.dev_dt;
      preset.push_back(t);
      preset_vid.push_back(fi.vid);
    }
    // bf16 feeds become TMA operands: registry entries + tensor maps for this run
    int nf_maps = 0;
    if (s->precision == CF_BF16) {
      int n = s->n_reg_static;
      for (int i = 0; i < n_feed; ++i) {
        auto it = P.feeds.find(feed_names[i]);
        if (it == P.feeds.end() || it->second.dev_dt != D_BF16) continue;
        const cf_buffer& b = feeds[i];
        int64_t rows, cols, slots;
        if (b.rank == 2) { slots = 1; rows = b.shape[0]; cols = b.shape[1]; }
        else if (b.rank == 3) { slots = b.shape[0]; rows = b.shape[1]; cols = b.shape[2]; }
        else continue;
        if (cols % 64 || n >= (int)s->reg_host.size()) continue;
        DReg r{};
        r.base = (int64_t)(uintptr_t)b.data;
        r.slots = (int32_t)slots; r.rows = (int32_t)rows; r.cols = (int32_t)cols;
        r.slot_bytes = rows * cols * 2;
        r.map0 = 3 * n;
        s->reg_host[n] = r;
        s->maps_host[3 * n + 0] = cf::make_map_bf16_strided(b.data, cols, rows, slots, r.slot_bytes, 64, 128);
        s->maps_host[3 * n + 1] = cf::make_map_bf16_strided(b.data, cols, rows, slots, r.slot_bytes, 64, 256);
        s->maps_host[3 * n + 2] = cf::make_map_bf16_strided(b.data, cols, rows, slots, r.slot_bytes, 64, 64);
        ++n;
      }
      nf_maps = n - s->n_reg_static;
      // the device looks entries up by binary search over base
      s->reg_sorted.assign(s->reg_host.begin(), s->reg_host.begin() + n);
      for (auto& r : s->reg_sorted) r.inv_slot = 1.0 / (double)r.slot_bytes;
      std::sort(s->reg_sorted.begin(), s->reg_sorted.end(),
                [](const DReg& a, const DReg& b) { return a.base < b.base; });
      A.prog.n_reg = n;
    }
    std::vector<void*> fo(P.fetches.size());
    for (size_t i = 0; i < P.fetches.size(); ++i) {
      fo[i] = outs ? outs[i].data : nullptr;
      if (outs && outs[i].dtype != P.fetches[i].dev_dt && P.fetches[i].bytes > 0)
        throw cf::CfError(CF_E_DTYPE, "fetch buffer " + std::to_string(i) + " dtype mismatch");
      if (outs && P.fetches[i].bytes > 0 && (!outs[i].data || buffer_bytes(outs[i]) != P.fetches[i].bytes))
        throw cf::CfError(CF_E_SHAPE, "fetch buffer " + std::to_string(i) + " holds " +
                                          std::to_string(buffer_bytes(outs[i])) + " bytes, fetch needs " +
                                          std::to_string(P.fetches[i].bytes));
    }
    if (!s->chans.empty())
      for (auto& c : s->chans)
        if (!(c.flags && c.data && c.acks && c.done))
          throw cf::CfError(CF_E_UNSUPPORTED, "channel " + std::to_string(c.channel) + " to rank " +
                                                  std::to_string(c.peer) +
                                                  " not connected (cf_session_connect)");
    // ---- one pinned staging area, then asynchronous uploads from it
    const bool up_chans = !s->chans.empty() && s->chans_dirty;
    auto al = [](size_t x) { return (x + 127) / 128 * 128; };
    const size_t b_maps = sizeof(CUtensorMap) * 3 * (size_t)nf_maps, b_reg = sizeof(DReg) * s->reg_sorted.size();
    const size_t b_ta = 8 * s->ta_base_host.size(), b_pre = sizeof(PresetTok) * preset.size();
    const size_t b_fo = 8 * fo.size(), b_ch = up_chans ? sizeof(DChan) * s->chans.size() : 0;
    const size_t o_maps = 0, o_reg = al(o_maps + b_maps), o_ta = al(o_reg + b_reg), o_pre = al(o_ta + b_ta);
    const size_t o_fo = al(o_pre + b_pre), o_ch = al(o_fo + b_fo), total = al(o_ch + b_ch);
    if (total > s->stage_cap) {
      if (s->stage_host) cudaFreeHost(s->stage_host);
      s->stage_host = nullptr;
      s->stage_cap = 0;
      CUDA_OK(cudaMallocHost((void**)&s->stage_host, total * 2));
      s->stage_cap = total * 2;
    }
    if ((int)preset.size() > s->preset_cap) {   // one token per placeholder (sized at creation)
      s->d_preset = (PresetTok*)dalloc(s, sizeof(PresetTok) * preset.size());
      s->preset_cap = (int)preset.size();
    }
    uint8_t* sh = s->stage_host;
    StageJobs jobs{};
    auto upload = [&](void* dst, size_t off, const void* src, size_t bytes) {
      if (!bytes) return;
      std::memcpy(sh + off, src, bytes);
      jobs.j[jobs.n++] = StageJob{(uint8_t*)dst, sh + off, (unsigned long long)bytes};
    };
    upload((uint8_t*)A.prog.maps + sizeof(CUtensorMap) * 3 * s->n_reg_static, o_maps,
           s->maps_host.data() + 3 * s->n_reg_static, b_maps);
    upload((void*)A.prog.reg, o_reg, s->reg_sorted.data(), b_reg);
    upload(A.ta_base, o_ta, s->ta_base_host.data(), b_ta);   // ta bases reset (unstack may alias)
    std::vector<PresetTok> pt(preset.size());
    for (size_t k = 0; k < preset.size(); ++k) pt[k] = PresetTok{preset_vid[k], preset[k]};
    upload(s->d_preset, o_pre, pt.data(), b_pre);
    A.preset = s->d_preset;
    A.n_preset = (int32_t)preset.size();
    upload(A.fetch_out, o_fo, fo.data(), b_fo);
    if (up_chans) {
      upload(s->d_chans, o_ch, s->chans.data(), b_ch);
      s->chans_dirty = false;
    }
    if (jobs.n) {
      const size_t tot = o_ch + b_ch;
      const int nb = (int)std::min<size_t>(32, std::max<size_t>(1, tot / 16384));
      cf_stage_kernel<<<nb, 256, 0, s->stream>>>(jobs);
      CUDA_OK(cudaGetLastError());
    }
    A.epoch = ++s->epoch;
    // (the staging area is rewritten only by the next cf_run, after this one's final sync)
    void* kargs[] = {(void*)&A};
    // host I/O executor for swapped stacks (separate streams for
    // GPU-to-CPU and CPU-to-GPU transfers next to the compute stream)
    std::atomic<bool> io_stop{false};
    std::atomic<int> io_err{0};
    std::thread io;
    if (s->own_stream) {
      // a library-owned stream is non-blocking: order the run after the caller's work on the
      // legacy default stream (e.g. the copies of this run's inputs)
      CUDA_OK(cudaEventRecord(s->ev_in, cudaStreamLegacy));
      CUDA_OK(cudaStreamWaitEvent(s->stream, s->ev_in, 0));
    }
    CUDA_OK(cudaEventRecord(s->ev0, s->stream));
    // started after the last call that can throw before the join below (a joinable
    // std::thread destroyed during unwinding would terminate the process)
    if (A.prog.n_swaps) {
      *(volatile unsigned long long*)s->io_tail_host = 0;
      io = std::thread([s, &io_stop, &io_err]() { io_executor(s, &io_stop, &io_err); });
    }
    cudaError_t lerr = cudaLaunchCooperativeKernel((void*)cf_driver_kernel, dim3(s->grid), dim3(kThreads),
                                                   kargs, s->dyn_smem, s->stream);
    if (lerr == cudaSuccess) lerr = cudaEventRecord(s->ev1, s->stream);
    if (lerr == cudaSuccess) lerr = cudaStreamSynchronize(s->stream);
    if (io.joinable()) {
      io_stop = true;
      io.join();
      for (int k = 0; k < cf_session::kIoStreams; ++k) {
        cudaStreamSynchronize(s->io_d2h[k]);
        cudaStreamSynchronize(s->io_h2d[k]);
      }
    }
    CUDA_OK(lerr);
    if (io_err.load()) throw cf::CfError(CF_E_CUDA, "swap I/O copy failed");
    RunState st;
    CUDA_OK(cudaMemcpy(&st, A.st, sizeof(RunState), cudaMemcpyDeviceToHost));
    if (st.error) {
      std::string tr;
      for (int f = 0; f < (int)P.frames.size() && f < 16; ++f) tr += (f ? "," : "") + std::to_string(st.trip[f]);
      throw cf::CfError(st.error, "device driver error " + std::to_string(st.error) + " (info " +
                                      std::to_string(st.error_info) + "; trips so far " + tr + ")");
    }
    std::vector<uint8_t> dead(std::max<size_t>(P.fetches.size(), 1));
    CUDA_OK(cudaMemcpy(dead.data(), A.fetch_dead, dead.size(), cudaMemcpyDeviceToHost));
    if (out_dead)
      for (size_t i = 0; i < P.fetches.size(); ++i) out_dead[i] = dead[i];
    if (trace) {
      float ms = 0;
      cudaEventElapsedTime(&ms, s->ev0, s->ev1);
      trace->wall_ms = ms;
      trace->n_frames = (int32_t)P.frames.size();
      for (int f = 0; f < 16; ++f) {
        trace->trip_count[f] = st.trip[f];
        trace->max_inflight[f] = st.max_inflight[f];
      }
      trace->pushes = st.pushes;
      trace->pops = st.pops;
      trace->max_depth = st.max_depth;
      trace->exit_fires = st.exit_fires;
      trace->instances = st.instances;
      trace->tiles = st.tiles;
      trace->dead_skipped = st.dead_skipped;
      trace->sends = st.sends;
      trace->recvs = st.recvs;
      trace->swap_out = st.swap_out;
      trace->swap_in = st.swap_in;
      trace->bytes_d2h = st.bytes_d2h;
      trace->bytes_h2d = st.bytes_h2d;
      int nb = P.n_conds * P.branch_bound;
      trace->n_branch_bits = nb;
      if (trace->branch_bits && trace->branch_bits_cap > 0)
        CUDA_OK(cudaMemcpy(trace->branch_bits, A.branch_bits,
                           std::min(nb, trace->branch_bits_cap), cudaMemcpyDeviceToHost));
    }
    return CF_OK;
  } catch (const cf::CfError& e) {
    cf::set_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    cf::set_error(std::string("internal: ") + e.what());
    return CF_E_CUDA;
  }
}

cf_status cf_session_feed_dtype(const cf_session* s, const char* name, int32_t* dtype) {
  if (!s || !name || !dtype) return CF_E_INVALID_GRAPH;
  auto it = s->P.feeds.find(name);
  if (it == s->P.feeds.end()) {
    cf::set_error(std::string("no placeholder ") + name);
    return CF_E_MISSING_FEED;
  }
  *dtype = it->second.dev_dt;
  return CF_OK;
}

cf_status cf_session_fetch_dtype(const cf_session* s, int32_t i, int32_t* dtype) {
  if (!s || !dtype || i < 0 || i >= (int)s->P.fetches.size()) return CF_E_INVALID_GRAPH;
  *dtype = s->P.fetches[i].dev_dt;
  return CF_OK;
}

cf_status cf_session_describe(const cf_session* s, char* buf, size_t cap) {
  if (!s || !buf || !cap) return CF_E_INVALID_GRAPH;
  std::string d = s->P.describe + "grid=" + std::to_string(s->grid) + "\n";
  std::strncpy(buf, d.c_str(), cap - 1);
  buf[cap - 1] = 0;
  return CF_OK;
}

// ---- cross-GPU channels (include/cf.h)
cf_status cf_session_channels(const cf_session* s, int32_t cap, int64_t* table, int32_t* n) {
  if (!s || !n) return CF_E_INVALID_GRAPH;
  const auto& cs = s->P.chans;
  *n = (int32_t)cs.size();
  for (int i = 0; i < (int)cs.size() && i < cap && table; ++i) {
    int64_t* r = table + 7 * i;
    r[0] = cs[i].channel;
    r[1] = cs[i].role;
    r[2] = cs[i].peer;
    r[3] = cs[i].slots;
    r[4] = cs[i].elem_bytes;
    r[5] = cs[i].dt;
    r[6] = cs[i].offset;
  }
  return CF_OK;
}

cf_status cf_session_ipc_handle(const cf_session* s, void* handle) {
  if (!s || !handle) return CF_E_INVALID_GRAPH;
  std::memset(handle, 0, CF_IPC_HANDLE_BYTES);
  if (!s->chan_mem) return CF_OK;
  cudaIpcMemHandle_t h;
  if (cudaSetDevice(s->device) != cudaSuccess || cudaIpcGetMemHandle(&h, s->chan_mem) != cudaSuccess) {
    cf::set_error("cudaIpcGetMemHandle failed");
    return CF_E_CUDA;
  }
  static_assert(sizeof(h) <= CF_IPC_HANDLE_BYTES, "ipc handle size");
  std::memcpy(handle, &h, sizeof(h));
  return CF_OK;
}

cf_status cf_session_connect(cf_session* s, int32_t peer, const void* handle, int32_t n,
                             const int64_t* table) {
  try {
    if (!s || !handle || (n > 0 && !table)) throw cf::CfError(CF_E_INVALID_GRAPH, "null argument");
    bool used = false;
    for (auto& c : s->chans) used |= c.peer == peer;
    if (!used) return CF_OK;
    CUDA_OK(cudaSetDevice(s->device));
    void* base = nullptr;
    auto it = s->peer_mem.find(peer);
    if (it != s->peer_mem.end()) {
      base = it->second;
    } else {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handle, sizeof(h));
      CUDA_OK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
      s->peer_mem[peer] = base;
    }
    for (auto& c : s->chans) {
      if (c.peer != peer) continue;
      const int64_t* row = nullptr;
      for (int i = 0; i < n; ++i)
        if (table[7 * i] == c.channel && table[7 * i + 1] == 1 - c.role) row = table + 7 * i;
      if (!row)
        throw cf::CfError(CF_E_UNSUPPORTED, "rank " + std::to_string(peer) + " has no " +
                                                (c.role ? "Recv" : "Send") + " for channel " +
                                                std::to_string(c.channel));
      if (row[3] != c.slots || row[4] != c.elem_bytes || row[5] != c.dt)
        throw cf::CfError(CF_E_UNSUPPORTED, "channel " + std::to_string(c.channel) +
                                                ": the two halves disagree on slots / payload bytes / "
                                                "dtype (same parallel_iterations and precision on "
                                                "both ranks?)");
      uint8_t* pb = (uint8_t*)base + row[6];
      const int64_t fb = ((int64_t)c.slots * 8 + 255) / 256 * 256;
      if (c.role == 1) {
        c.flags = (unsigned long long*)pb;
        c.data = pb + fb;
      } else {
        c.acks = (unsigned long long*)pb;
        c.done = (unsigned long long*)(pb + fb);
      }
    }
    s->chans_dirty = true;
    return CF_OK;
  } catch (const cf::CfError& e) {
    cf::set_error(e.what());
    return e.code;
  }
}

int32_t cf_debug_set_knob(int32_t which, int32_t value) {
  if (which < 0 || which >= 8) return CF_E_SHAPE;
  return cudaMemcpyToSymbol(tc::kKnobs, &value, sizeof(value), sizeof(int) * which) == cudaSuccess
             ? CF_OK : CF_E_CUDA;
}

int32_t cf_debug_tile_phases(uint64_t* out20, int32_t reset) {
  if (cudaMemcpyFromSymbol(out20, g_tile_phase, 20 * 8) != cudaSuccess) return CF_E_CUDA;
  if (reset) {
    const unsigned long long z[20] = {};
    if (cudaMemcpyToSymbol(g_tile_phase, z, sizeof(z)) != cudaSuccess) return CF_E_CUDA;
  }
  return CF_OK;
}

int32_t cf_debug_set_flags(int32_t flags) {
  if (cudaMemcpyToSymbol(kDbgFlagsTC, &flags, sizeof(flags)) != cudaSuccess) return CF_E_CUDA;
  return cudaMemcpyToSymbol(kDbgFlags, &flags, sizeof(flags)) == cudaSuccess ? CF_OK : CF_E_CUDA;
}
int32_t cf_debug_set_worker_roles(int32_t low_first, int32_t strict) {
  const int v = (low_first & 0xffff) | (strict ? 1 << 16 : 0);
  return cudaMemcpyToSymbol(kLowWorkers, &v, sizeof(v)) == cudaSuccess ? CF_OK : CF_E_CUDA;
}

int32_t cf_debug_set_m2_rows(int32_t rows) {
  if (rows <= 0) rows = kM2Default;
  return cudaMemcpyToSymbol(kM2MinRows, &rows, sizeof(rows)) == cudaSuccess ? CF_OK : CF_E_CUDA;
}

// profiling hook (include/cf_debug.h): per-instance timing of the last cf_run
int32_t cf_debug_session_profile(const cf_session* s, unsigned long long* out, int64_t cap,
                                 int64_t* n_inst, unsigned long long* t0) {
  if (!s) return CF_E_INVALID_GRAPH;
  RunState st;
  if (cudaMemcpy(&st, s->args.st, sizeof(RunState), cudaMemcpyDeviceToHost) != cudaSuccess) return CF_E_CUDA;
  // without the profiling build / profile=True only the driver counters (t0) are available
  int64_t n = s->args.prof ? std::min<int64_t>(st.instances + 64, s->args.inst_cap) : 0;
  if (n_inst) *n_inst = n;
  if (t0) {
    t0[0] = st.t_start;
    t0[1] = st.t_end;
    for (int k = 0; k < 64; ++k) {
      t0[2 + k] = (unsigned long long)st.op_count[k];
      t0[66 + k] = (unsigned long long)st.op_cycles[k];
    }
  }
  if (out && cap > 0 && n > 0) {
    int64_t k = std::min(cap, 6 * n);
    if (cudaMemcpy(out, s->args.prof, 8 * k, cudaMemcpyDeviceToHost) != cudaSuccess) return CF_E_CUDA;
  }
  return CF_OK;
}

void cf_session_destroy(cf_session* s) {
  if (!s) return;
  for (void* p : s->allocs) {
    if (s->dev_free) s->dev_free(p, s->alloc_user);
    else cudaFree(p);
  }
  for (auto& [r, p] : s->peer_mem) cudaIpcCloseMemHandle(p);
  for (void* h : s->host_allocs) cudaFreeHost(h);
  if (s->stage_host) cudaFreeHost(s->stage_host);
  for (int k = 0; k < cf_session::kIoStreams; ++k) {
    if (s->io_d2h[k] && s->io_d2h[k] != s->user_d2h) cudaStreamDestroy(s->io_d2h[k]);
    if (s->io_h2d[k] && s->io_h2d[k] != s->user_h2d) cudaStreamDestroy(s->io_h2d[k]);
  }
  if (s->chan_mem) cudaFree(s->chan_mem);
  if (s->ev0) cudaEventDestroy(s->ev0);
  if (s->ev_in) cudaEventDestroy(s->ev_in);
  if (s->ev1) cudaEventDestroy(s->ev1);
  if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
  delete s;
}

}  // extern "C"
