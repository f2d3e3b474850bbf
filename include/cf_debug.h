/*
 * cf_debug.h -- test hooks of libcf. NOT part of the product API: used by tests/ to check the
 * sm_100a tcgen05 tile engine in isolation against a plain matmul.
 */
#ifndef CF_DEBUG_H_
#define CF_DEBUG_H_
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* C[M][N] (fp32, row-major, device) = sum_k A(m,k) * B(n,k) with bf16 device inputs:
 *   A: a_mn = 0 -> stored [M][K] (K-major); a_mn = 1 -> stored [K][M] (MN-major)
 *   B: b_mn = 0 -> stored [N][K] (K-major); b_mn = 1 -> stored [K][N] (MN-major)
 * bn = 128 or 256 (tile N). M, N, K multiples of 64 (M, N: any; K: multiple of 64).
 * Synchronous on `stream`. Returns 0 or CF_E_CUDA (15; message in cf_last_error()). */
int32_t cf_debug_tc_gemm(int32_t M, int32_t N, int32_t K, int32_t bn, int32_t a_mn, int32_t b_mn,
                         const void* A, const void* B, float* C, void* stream);
/* Profiling hook: with cf_run_opts.reserved[0] = 1 at session creation, the driver records
 * per heavy instance 6 x u64 {create ns, publish ns, first tile start ns, last tile end ns,
 * summed tile busy ns, (kind << 32) | ntiles} (%globaltimer). Copies up to cap u64 of the
 * last run into out; *n_inst = records available; t0 (130 x u64) = {run start ns, run end ns,
 * 64 driver counts, 64 driver cycles: opcodes [0,32), profiled regions [32,64)}; count/cycle
 * slot 31 = the driver's shared-memory staging mask / bytes. Without profiling only t0 is
 * filled (*n_inst = 0). */
struct cf_session;
int32_t cf_debug_session_profile(const struct cf_session* s, unsigned long long* out, int64_t cap,
                                 int64_t* n_inst, unsigned long long* t0);
/* Batch size from which the forward and d[x,h] GEMMs use 256-row tiles (two TMEM accumulators
 * per CTA); product default 512 (rows <= 0 restores it). Lets tests exercise that tile shape
 * at small sizes. Returns 0 or CF_E_CUDA. */
int32_t cf_debug_set_m2_rows(int32_t rows);
/* Mainloop throughput probe of the 256-row tcgen05 engine: one CTA per SM runs every
 * 256 x 256 tile of C = A B^T (A [M][K], B nb copies of [N][K], bf16, K-major; B copy chosen
 * round-robin, `reps` passes; L2 prefetch `prefetch` k-blocks ahead, 0 = off) with an
 * accumulator-read-only epilogue. *ms_out = device time. Returns 0 or CF_E_CUDA. */
int32_t cf_debug_tc_pipe(int32_t M, int32_t N, int32_t K, int32_t nb, int32_t reps,
                         int32_t prefetch, const void* A, const void* B, float* ms_out);
/* Worker roles: the first `low_first` worker CTAs take low-priority work (dW chunks) before
 * the critical-path ring; with `strict` != 0 the other workers never take low-priority work.
 * (0, 0) = every worker prefers the critical-path ring (the default). Returns 0 or CF_E_CUDA. */
int32_t cf_debug_set_worker_roles(int32_t low_first, int32_t strict);
/* Profiling knobs: bit 0 = workers skip every tile body (the device driver's own cost in
 * isolation; results are garbage); A/B switches (results unchanged): bit 2 = poll
 * completions after every node, bit 3 = wave helpers spin without sleeping, bit 4 = release
 * the queue tail after every publication, bit 7 = tensor-core LSTM nodes prepared by the
 * driver thread instead of the helper lanes; bits 8-15 = completion-poll interval in 1000
 * cycles (0 = default); bit 24 = no chaining of a node's preparation onto the preceding
 * wave; bit 25 = no fusion of consecutive waves into one helper job;
 * bit 26 = poll completions before each heavy node; bit 27 = no overlap of the next wave job
 * with a forward LSTM node's instance construction, bit 29 = the same for a backward node
 * (steps that do not close a dW chunk). Returns 0 or CF_E_CUDA. */
int32_t cf_debug_set_flags(int32_t flags);
/* A/B knobs, read by the kernel as it runs (0 = default): knob 0 = how many k-blocks before
 * a tensor-core tile's last MMA issue the worker claims its next tile (default 8); knob 1 = 1:
 * no overlap of a heavy batch's records and submissions with the routing after it. Returns 0,
 * CF_E_SHAPE (which outside 0..7) or CF_E_CUDA. */
int32_t cf_debug_set_knob(int32_t which, int32_t value);
/* Tile phase clocks, collected while cf_debug_set_flags bit 22 is set: out20[4k + 0] tiles,
 * [4k + 1] SM cycles from tile entry to the mainloop's first issue, [4k + 2] mainloop cycles
 * (until the accumulator is complete; for the backward EW the whole tile), [4k + 3] epilogue
 * cycles; k = 0 forward, 1 d[x,h], 2 dW, 3 backward EW (thread 0 of each tile); [16] forward
 * epilogue TMEM + math + staging, [17] its barrier wait, [18] / [19] forward tiles' wall-clock
 * ns / SM cycles (their ratio is the SM clock under load). reset != 0 zeroes the counters after
 * the read. Returns 0 or CF_E_CUDA. */
int32_t cf_debug_tile_phases(uint64_t* out20, int32_t reset);
/* Compile a graph for the device program without a GPU and write its description and body
 * programs (one node per line, evaluation order) into buf; *needed = length + 1. The
 * environment variable CF_DEBUG_MAX_ITERATIONS plays cf_run_opts.max_iterations. */
struct cf_graph;
typedef struct { int32_t node, port; } cf_debug_tensor;
int32_t cf_debug_program_listing(const struct cf_graph* g, int32_t precision,
                                 int32_t parallel_iterations, int32_t n_fetch,
                                 const cf_debug_tensor* fetches, char* buf, size_t cap,
                                 size_t* needed);
#ifdef __cplusplus
}
#endif
#endif
