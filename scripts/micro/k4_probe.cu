// k4_probe.cu -- calibration microbenchmarks for the K4 softmax chain (bring-up tool, not product).
//   mode A  softmax arithmetic of one 128-key row block per lane, registers only (no local memory),
//           WARPS warps per SM (one CTA per SM), EMU/8 of the exponentials on the FMA pipe
//   mode B  tcgen05.ld bandwidth: each warp reads its 32 TMEM lanes x 128 columns (16 KB) per iteration
//   mode C  mode A + the TMEM traffic of K4 (tcgen05.ld of the S row block, tcgen05.st of packed P)
// Prints cycles per iteration per warp (median over SMs of the max over warps).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include "../../paper_2601_11641_b200/csrc/sm100.cuh"
using namespace sm100;

__device__ __forceinline__ void keep(float& x) { asm volatile("" : "+f"(x)); }
__device__ __forceinline__ void keepu(uint32_t& x) { asm volatile("" : "+r"(x)); }

template <int EMU>
__device__ __forceinline__ void softmax_row(float (&s)[128], float& m_run, float& l_run, uint32_t (&pk)[64],
                                            float scale_log2) {
  float mx0 = fmax3f(s[0], s[1], s[2]), mx1 = fmax3f(s[3], s[4], s[5]);
#pragma unroll
  for (int c = 6; c < 126; c += 4) {
    mx0 = fmax3f(mx0, s[c], s[c + 1]);
    mx1 = fmax3f(mx1, s[c + 2], s[c + 3]);
  }
  const float mx = fmax3f(mx0, mx1, fmaxf(s[126], s[127]));
  const float m_new = fmaxf(m_run, mx * scale_log2);
  const bool rescale = (m_new - m_run) > 8.0f;
  const float m_use = rescale ? m_new : m_run;
  const float alpha = rescale ? ex2(m_run - m_new) : 1.0f;
  const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m_use, -m_use);
  float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int c = 0; c < 128; c += 2) {
    const float2 x = ffma2(make_float2(s[c], s[c + 1]), sc2, nm2);
    float2 p;
    if (((c / 2) & 7) < EMU) {
      p = ex2_poly2(x);
    } else {
      p.x = ex2(x.x);
      p.y = ex2(x.y);
    }
    acc2[(c / 2) & 1] = fadd2(acc2[(c / 2) & 1], p);
    pk[c / 2] = pack_bf16(p.x, p.y);
  }
  l_run = fmaf(l_run, alpha, (acc2[0].x + acc2[0].y) + (acc2[1].x + acc2[1].y));
  m_run = m_use;
}

template <int EMU, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) mode_a(float* out, int iters) {
  float s[128];
#pragma unroll
  for (int c = 0; c < 128; ++c) s[c] = (float)((c * 37 + threadIdx.x) % 101) * 0.05f;
  float m_run = -INFINITY, l_run = 0.f;
  uint32_t sink = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 128; ++c) keep(s[c]);   // the scores "change" every iteration (no hoisting)
    uint32_t pk[64];
    softmax_row<EMU>(s, m_run, l_run, pk, 0.127f);
#pragma unroll
    for (int c = 0; c < 64; ++c) keepu(pk[c]);
    sink ^= pk[it & 1 ? 3 : 5];
    m_run -= 1e-3f;
  }
  long long t1 = clock64();
  __shared__ float red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = (float)(t1 - t0) / iters;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) m = fmaxf(m, red[w]);
    out[blockIdx.x] = m;
  }
  if (sink == 0x12345678u && l_run == 1.f) out[4095] = 0;
}

// tcgen05.ld bandwidth: warp w reads TMEM lanes [32*(w%4), +32), columns [128*(w/4) % 512, +128)
template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1) mode_b(float* out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t t = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((128 * (warp / 4)) & 511);
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[4][32];
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_ld32(t + c * 32, r[c]);
    tmem_ld_wait();
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int e = 0; e < 32; e += 8) acc += r[c][e];
  }
  long long t1 = clock64();
  __shared__ float red[32];
  if ((threadIdx.x & 31) == 0) red[warp] = (float)(t1 - t0) / iters;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
  if (threadIdx.x == 0) {
    float m = 0;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) m = fmaxf(m, red[w]);
    out[blockIdx.x] = m;
  }
  if (acc == 0x12345678u) out[4095] = 1;
}

// mode C: per iteration each warp tcgen05.ld's its 128-column S row block, runs the softmax, and
// tcgen05.st's the 64 packed P columns over the first half of S (as K4 does)
template <int EMU, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) mode_c(float* out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t t = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((128 * (warp / 4)) & 511);
  {   // initialise S with finite values
    uint32_t r[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) r[e] = __float_as_uint((float)((e * 13 + threadIdx.x) % 29) * 0.1f);
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_st32(t + c * 32, r);
    tmem_st_wait();
  }
  float m_run = -INFINITY, l_run = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t sr[128];
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_ld32(t + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
    tmem_ld_wait();
    uint32_t pk[64];
    softmax_row<EMU>(*reinterpret_cast<float(*)[128]>(sr), m_run, l_run, pk, 0.127f);
    // restore S for the next iteration: write P into columns 64..127 (K4 aliases P over S; here we keep
    // the first half of S intact so that the scores stay finite)
#pragma unroll
    for (int c = 0; c < 2; ++c) tmem_st32(t + 64 + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[c * 32]));
    tmem_st_wait();
    m_run -= 1e-3f;
  }
  long long t1 = clock64();
  __shared__ float red[32];
  if ((threadIdx.x & 31) == 0) red[warp] = (float)(t1 - t0) / iters;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
  if (threadIdx.x == 0) {
    float m = 0;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) m = fmaxf(m, red[w]);
    out[blockIdx.x] = m;
  }
  if (l_run == 1.2345f) out[4095] = 2;
}

static float median148(float* d) {
  std::vector<float> h(148);
  cudaMemcpy(h.data(), d, 148 * 4, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  return h[74];
}

template <typename K>
static void run(const char* name, K kern, int warps, int iters, float* d, int elems_per_warp_iter) {
  kern<<<148, warps * 32>>>(d, 20);
  cudaDeviceSynchronize();
  kern<<<148, warps * 32>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  const float c = median148(d);
  printf("%-28s warps=%2d  %8.1f cycles/iter/warp   %6.2f elem/clk/SM  (%s)\n", name, warps, c,
         elems_per_warp_iter * warps / c, cudaGetErrorString(e));
}

int main() {
  float* d;
  cudaMalloc(&d, 4096 * 4);
  run("A softmax regs EMU=0", mode_a<0, 256>, 4, 400, d, 4096);
  run("A softmax regs EMU=0", mode_a<0, 256>, 8, 400, d, 4096);
  run("A softmax regs EMU=2", mode_a<2, 256>, 4, 400, d, 4096);
  run("A softmax regs EMU=2", mode_a<2, 256>, 8, 400, d, 4096);
  run("A softmax regs EMU=2", mode_a<2, 384>, 12, 400, d, 4096);
  run("A softmax regs EMU=3", mode_a<3, 256>, 4, 400, d, 4096);
  run("A softmax regs EMU=3", mode_a<3, 256>, 8, 400, d, 4096);
  run("A softmax regs EMU=3", mode_a<3, 384>, 12, 400, d, 4096);
  run("A softmax regs EMU=4", mode_a<4, 256>, 8, 400, d, 4096);
  run("B tmem ld 16KB/warp", mode_b<256>, 4, 400, d, 4096);
  run("B tmem ld 16KB/warp", mode_b<256>, 8, 400, d, 4096);
  run("B tmem ld 16KB/warp", mode_b<512>, 16, 400, d, 4096);
  run("C softmax+tmem EMU=2", mode_c<2, 256>, 4, 400, d, 4096);
  run("C softmax+tmem EMU=2", mode_c<2, 256>, 8, 400, d, 4096);
  run("C softmax+tmem EMU=2", mode_c<2, 384>, 12, 400, d, 4096);
  run("C softmax+tmem EMU=3", mode_c<3, 256>, 4, 400, d, 4096);
  run("C softmax+tmem EMU=3", mode_c<3, 256>, 8, 400, d, 4096);
  run("C softmax+tmem EMU=3", mode_c<3, 384>, 12, 400, d, 4096);
  return 0;
}
