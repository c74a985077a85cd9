// common.cuh -- shared plumbing of libmoddit (plan struct, error handling, sm_100a PTX wrappers).
#pragma once
#include <cuda_runtime.h>
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "moddit.h"

// ------------------------------------------------------------------------------------------------
// error handling (thread-local message, see mod_last_error)
// ------------------------------------------------------------------------------------------------
void mod_set_error(const char* fmt, ...);
void mod_note_launches(int n);

#define MOD_REQUIRE(cond, status, ...)     \
  do {                                     \
    if (!(cond)) {                         \
      mod_set_error(__VA_ARGS__);          \
      return (status);                     \
    }                                      \
  } while (0)

#define MOD_CUDA(call)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      mod_set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(e_), __FILE__, __LINE__, \
                    cudaGetErrorString(e_));                                              \
      return MOD_ERR_CUDA;                                                                \
    }                                                                                     \
  } while (0)

// Checks for an earlier asynchronous fault before launching, and for a launch error after.
mod_status mod_check_sticky();
#define MOD_LAUNCH_CHECK() MOD_CUDA(cudaGetLastError())

// ------------------------------------------------------------------------------------------------
// plan
// ------------------------------------------------------------------------------------------------
struct mod_plan_s {
  mod_layout L;
  mod_config cfg;
  int device;
  int N, n, p, F, prefix_last;  // prefix_last = last prefix block or -1
  float scale;                  // softmax scale s
  std::vector<int> frame_ab;    // host [2F]
  int* d_frame_ab;              // device [2F]
  int* d_row_frames;            // device [2n]: frames containing block i are [lo, hi] (hi < lo: none)
  float* d_log_sizes;           // device [n]: ln |I_j|
  double* d_ginv;               // device [p rows x ginv_ld] deflated Gram inverse (symmetric)
  int ginv_ld;                  // leading dimension of d_ginv (p rounded up to 32: 256-byte rows)
  CUtensorMap tm_ginv;          // 2D TMA map over d_ginv: {ld, p} fp64, box {128 columns, 32 rows}
  size_t ws_bytes;
  // workspace carve (byte offsets)
  size_t ws_qbar, ws_kbar, ws_qs, ws_ks, ws_part, ws_r, ws_x, ws_nae, ws_sel, ws_cnt, ws_solve;
  int proj_tiles, proj_rows;    // row tiles of the projection kernel / map rows per tile (<= 32, in smem)
  int solve_segs, solve_seg_len; // split-K segments of the X = G'^-1 r stream (fit.cu)
  int sm_count;
  double min_pivot;             // smallest Gauss-Jordan pivot (magnitude) of the accepted inversion
  int null_dim;                 // dimension of the deflated null space (analytic + numerically found)
  double cond_est;              // condition estimate of the accepted inversion (max G_ii x max Ginv_ii)
  int solver;                   // mod_solver that produced d_ginv (App. B chain: Cholesky, LU, pinv)
  double create_ms;             // host wall time of mod_plan_create
};

mod_status mod_validate_plan(mod_plan plan);

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// NVTX range around every C-ABI entry point (host side: it brackets the enqueue of the call's launches),
// so that profiler timelines attribute the kernels to mod_* calls; free when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define MOD_NVTX(name) NvtxRange mod_nvtx_range_(name)

constexpr int kProjRows = 32;    // max rows per projection tile (fit / update)
constexpr int kProjSmemFloats = 28672;   // shared-memory map tile of the projection (112 KB)
constexpr int kMaxBlocks = 2048; // n limit (pattern pool 3n-1 sorted in shared memory)

// ------------------------------------------------------------------------------------------------
// device helpers
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ int4 ld_nc_v4(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
