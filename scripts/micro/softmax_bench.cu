// Cycles of one softmax row-block (128 scores -> 64 packed bf16 P) per thread, as in attn.cu's loop body,
// with WARPS warps per CTA (one CTA per SM), no TMEM / barriers.  Bring-up microbenchmark.
#include <cstdio>
#include <cstdint>
#include "../../paper_2601_11641_b200/csrc/sm100.cuh"
using namespace sm100;
template <int EMU>
__global__ void k(float* out, int iters, float scale_log2) {
  float s[128];
  for (int c = 0; c < 128; ++c) s[c] = (float)((c * 37 + threadIdx.x) % 101) * 0.05f;
  float m_run = -INFINITY, l_run = 0.f;
  uint32_t sink = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float mxv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) mxv[u] = s[u];
#pragma unroll
    for (int c = 8; c < 128; c += 8)
#pragma unroll
      for (int u = 0; u < 8; ++u) mxv[u] = fmaxf(mxv[u], s[c + u]);
    const float mx = fmaxf(fmaxf(fmaxf(mxv[0], mxv[1]), fmaxf(mxv[2], mxv[3])), fmaxf(fmaxf(mxv[4], mxv[5]), fmaxf(mxv[6], mxv[7])));
    const float m_new = fmaxf(m_run, mx * scale_log2);
    const bool rescale = (m_new - m_run) > 8.0f;
    const float m_use = rescale ? m_new : m_run;
    const float alpha = rescale ? ex2(m_run - m_new) : 1.0f;
    const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m_use, -m_use);
    float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    uint32_t pk[64];
    if (EMU >= 0) {
#pragma unroll
    for (int c = 0; c < 128; c += 2) {
      const float2 x = ffma2(make_float2(s[c], s[c + 1]), sc2, nm2);
      float2 p;
      if (((c / 2) & 7) < EMU) p = ex2_poly2(x);
      else { p.x = ex2(x.x); p.y = ex2(x.y); }
      acc2[(c / 2) & 1] = fadd2(acc2[(c / 2) & 1], p);
      pk[c / 2] = pack_bf16(p.x, p.y);
    }
    } else {
      // phased: all FFMA2, then all ex2 (in place), then pack + sums -- maximal ILP per phase
      float x[128];
#pragma unroll
      for (int c = 0; c < 128; c += 2) { const float2 t = ffma2(make_float2(s[c], s[c + 1]), sc2, nm2); x[c] = t.x; x[c + 1] = t.y; }
#pragma unroll
      for (int c = 0; c < 128; ++c) x[c] = ex2(x[c]);
#pragma unroll
      for (int c = 0; c < 128; c += 2) {
        acc2[(c / 2) & 1] = fadd2(acc2[(c / 2) & 1], make_float2(x[c], x[c + 1]));
        pk[c / 2] = pack_bf16(x[c], x[c + 1]);
      }
    }
    l_run = fmaf(l_run, alpha, (acc2[0].x + acc2[0].y) + (acc2[1].x + acc2[1].y));
    m_run = m_use - 0.001f * it;   // keep the loop live
#pragma unroll
    for (int c = 0; c < 64; ++c) sink ^= pk[c];
    s[it & 127] += 1e-3f;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (float)(t1 - t0) / iters;
  if (sink == 0x12345678u) out[1000] = l_run;
}
int main() {
  float* d; cudaMalloc(&d, 4096 * 4);
  float h[148];
  for (int warps : {4, 8}) {
    k<-1><<<148, warps * 32>>>(d, 1000, 0.127f); cudaMemcpy(h, d, 148 * 4, cudaMemcpyDeviceToHost);
    printf("warps/CTA=%2d phased MUFU-only: %.0f cycles per row-block per warp\n", warps, h[0]);
    k<0><<<148, warps * 32>>>(d, 200, 0.127f); cudaDeviceSynchronize();
    k<0><<<148, warps * 32>>>(d, 1000, 0.127f); cudaMemcpy(h, d, 148 * 4, cudaMemcpyDeviceToHost);
    printf("warps/CTA=%2d EMU=0/8: %.0f cycles per row-block per warp\n", warps, h[0]);
    k<2><<<148, warps * 32>>>(d, 1000, 0.127f); cudaMemcpy(h, d, 148 * 4, cudaMemcpyDeviceToHost);
    printf("warps/CTA=%2d EMU=2/8: %.0f cycles per row-block per warp\n", warps, h[0]);
    k<3><<<148, warps * 32>>>(d, 1000, 0.127f); cudaMemcpy(h, d, 148 * 4, cudaMemcpyDeviceToHost);
    printf("warps/CTA=%2d EMU=3/8: %.0f cycles per row-block per warp\n", warps, h[0]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
