// Test hooks (include/cf_debug.h): exercise the tcgen05 tile engine in isolation.
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/cf_debug.h"
#include "tc_engine.cuh"
#include "tmap.h"

namespace cf {
void set_error(const std::string& m);
}

namespace {

// C[M][N] = sum_k A(m,k) B(n,k); A stored [M][K] (K-major) or [K][M] (MN-major); same for B.
__global__ void __launch_bounds__(256, 1)
    debug_gemm_kernel(const CUtensorMap* maps, int M, int N, int K, int bn, int a_mn, int b_mn,
                      float* C) {
  extern __shared__ uint8_t dyn[];
  tc::TcShared s = tc::tc_carve(dyn);
  tc::tc_setup(s);
  const CUtensorMap* ma = maps;
  const CUtensorMap* mb = maps + 1;
  if (threadIdx.x == 0) {
    tc::tma_prefetch(ma);
    tc::tma_prefetch(mb);
  }
  const int tn = (N + bn - 1) / bn;
  const int m0 = (blockIdx.x / tn) * tc::BM, n0 = (blockIdx.x % tn) * bn;
  uint32_t cnt = 0, tiles = 0;
  const int nk = (K + tc::BK - 1) / tc::BK;
  auto plan_a = [&](int kb, tc::Box* b) {
    if (!a_mn) {
      b[0] = {ma, kb * 64, m0, 0, 0};
      return 1;
    }
    for (int j = 0; j < tc::BM / 64; ++j) b[j] = {ma, m0 + 64 * j, kb * 64, 0, j * 8192};
    return tc::BM / 64;
  };
  auto plan_b = [&](int kb, tc::Box* b) {
    if (!b_mn) {
      b[0] = {mb, kb * 64, n0, 0, 0};
      return 1;
    }
    for (int j = 0; j < bn / 64; ++j) b[j] = {mb, n0 + 64 * j, kb * 64, 0, j * 8192};
    return bn / 64;
  };
  tc::tc_tile(s, nk, bn, a_mn, b_mn, cnt, tiles, plan_a, plan_b);
  // epilogue: 8 warps; warp w -> rows 32*(w%4).., column half (w/4)
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int row = m0 + 32 * (warp % 4) + lane;
  const int half = bn / 2;
  for (int c = (warp / 4) * half; c < (warp / 4 + 1) * half; c += 16) {
    float v[16];
    tc::tc_acc16(s, c, v);
    if (row < M)
      for (int i = 0; i < 16; ++i)
        if (n0 + c + i < N) C[(int64_t)row * N + n0 + c + i] = v[i];
  }
  tc::tc_tile_end();
  tc::tc_teardown(s);
}

}  // namespace

extern "C" int32_t cf_debug_tc_gemm(int32_t M, int32_t N, int32_t K, int32_t bn, int32_t a_mn,
                                    int32_t b_mn, const void* A, const void* B, float* C,
                                    void* stream) {
  try {
    if (bn != 128 && bn != 256) throw std::runtime_error("bn must be 128 or 256");
    CUtensorMap maps[2];
    maps[0] = a_mn ? cf::make_map_bf16(A, M, K, 1, 64, 64) : cf::make_map_bf16(A, K, M, 1, 64, 128);
    maps[1] = b_mn ? cf::make_map_bf16(B, N, K, 1, 64, 64) : cf::make_map_bf16(B, K, N, 1, 64, bn);
    CUtensorMap* d = nullptr;
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMalloc(&d, sizeof(maps)) != cudaSuccess) throw std::runtime_error("cudaMalloc");
    cudaMemcpyAsync(d, maps, sizeof(maps), cudaMemcpyHostToDevice, st);
    cudaFuncSetAttribute(debug_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::kSmemTC);
    int tiles = ((M + tc::BM - 1) / tc::BM) * ((N + bn - 1) / bn);
    debug_gemm_kernel<<<tiles, 256, tc::kSmemTC, st>>>(d, M, N, K, bn, a_mn, b_mn, C);
    cudaError_t e = cudaStreamSynchronize(st);
    cudaFree(d);
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    return 0;
  } catch (const std::exception& ex) {
    cf::set_error(ex.what());
    return 15;
  }
}

// ---- mainloop throughput probe: persistent CTAs (one per SM) run 256 x 256 tiles of
// C = A B^T with the worker's 256-row engine (tc_tile2), A [M][K] and B [N][K] K-major, the
// B operand chosen round-robin from `nb` weight copies (nb x N x K bf16: > L2 when large).
// The epilogue only reads the accumulator (no stores): the time is the mainloop's.
namespace {
__global__ void __launch_bounds__(256, 1)
    debug_pipe_kernel(const CUtensorMap* maps, int M, int N, int K, int nb, int reps, int pf,
                      unsigned long long* cycles) {
  extern __shared__ uint8_t dyn[];
  tc::TcShared s = tc::tc_carve(dyn);
  tc::tc_setup(s);
  const int tn = N / 256, nk = K / 64;
  uint32_t cnt2 = 0, tiles = 0, cnt = 0;
  const long long c0 = clock64();
  if (pf < 0) {   // 128-row tiles (tc_tile, one 128 x 256 accumulator)
    const int tm = M / 128;
    for (int w = blockIdx.x; w < tm * tn * nb * reps; w += gridDim.x) {
      const int b = (w / (tm * tn)) % nb, mt = (w % (tm * tn)) / tn, nt = w % tn;
      const CUtensorMap* ma = maps;
      const CUtensorMap* mb = maps + 1;
      auto plan_a = [&](int kb, tc::Box* bx) {
        bx[0] = {ma, kb * 64, mt * 128, 0, 0};
        return 1;
      };
      auto plan_b = [&](int kb, tc::Box* bx) {
        bx[0] = {mb, kb * 64, nt * 256, b, 0, 1};
        return 1;
      };
      tc::tc_tile(s, nk, 256, 0, 0, cnt, tiles, plan_a, plan_b);
      float v[16];
      tc::tc_acc16(s, 0, v);
      if (v[0] == 12345.f) cycles[1] = 1;
      tc::tc_tile_end();
    }
    if (threadIdx.x == 0) atomicAdd(cycles, (unsigned long long)(clock64() - c0));
    tc::tc_teardown(s);
    return;
  }
  const int tm = M / 256;
  for (int w = blockIdx.x; w < tm * tn * nb * reps; w += gridDim.x) {
    const int b = (w / (tm * tn)) % nb, mt = (w % (tm * tn)) / tn, nt = w % tn;
    const CUtensorMap* ma = maps;
    const CUtensorMap* mb = maps + 1;
    auto plan_a = [&](int kb, tc::Box* bx) {
      bx[0] = {ma, kb * 64, mt * 256, 0, 0};
      bx[1] = {ma, kb * 64, mt * 256 + 128, 0, tc::kStageA};
      return 2;
    };
    auto plan_b = [&](int kb, tc::Box* bx) {
      bx[0] = {mb, kb * 64, nt * 256, b, 0, 1};
      return 1;
    };
    tc::tc_tile2(s, nk, 0, 0, cnt2, tiles, plan_a, plan_b, 256, pf);
    float v[16];
    tc::tc_acc16(s, 0, v);
    if (v[0] == 12345.f) cycles[1] = 1;   // keep the load
    tc::tc_tile_end();
  }
  if (threadIdx.x == 0) atomicAdd(cycles, (unsigned long long)(clock64() - c0));
  tc::tc_teardown(s);
}
}  // namespace

// ms of the probe (all tiles of `reps` passes over nb weight copies); see debug_pipe_kernel
extern "C" int32_t cf_debug_tc_pipe(int32_t M, int32_t N, int32_t K, int32_t nb, int32_t reps,
                                    int32_t prefetch, const void* A, const void* B, float* ms_out) {
  try {
    CUtensorMap maps[2];
    maps[0] = cf::make_map_bf16(A, K, M, 1, 64, 128);
    maps[1] = cf::make_map_bf16(B, K, N, nb, 64, 256);
    CUtensorMap* d = nullptr;
    unsigned long long* cyc = nullptr;
    if (cudaMalloc(&d, sizeof(maps)) != cudaSuccess) throw std::runtime_error("cudaMalloc");
    cudaMalloc(&cyc, 16);
    cudaMemset(cyc, 0, 16);
    cudaMemcpy(d, maps, sizeof(maps), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(debug_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::kSmemTC);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    debug_pipe_kernel<<<sms, 256, tc::kSmemTC>>>(d, M, N, K, nb, 1, prefetch, cyc);   // warm-up
    cudaEventRecord(e0);
    debug_pipe_kernel<<<sms, 256, tc::kSmemTC>>>(d, M, N, K, nb, reps, prefetch, cyc);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    *ms_out = ms;
    cudaFree(d);
    cudaFree(cyc);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    return 0;
  } catch (const std::exception& ex) {
    cf::set_error(ex.what());
    return 15;
  }
}
