// tcgen05.mma issue-rate calibration on sm_100a (bring-up microbenchmark, not part of libmoddit):
// one CTA per SM, one thread issues NITER back-to-back kind::f16 MMAs (bf16 in, fp32 accumulate).
#include <cstdio>
#include <cstdint>
#include "../../paper_2601_11641_b200/csrc/sm100.cuh"
using namespace sm100;
template <int N, bool TS, int MODE = 0>   // MODE 0: B K-major; 1: B MN-major (like V); 2: S(SS,K-major) + PV(TS,MN-major) alternating;
// 3: 8 MMAs + commit; 4: 8 MMAs + commit + wait on a completed barrier; 5: 8 MMAs + wait (no commit);
// 6: SS MMAs while warps 1-3 stream tcgen05.ld/st over other TMEM columns (softmax-like traffic); 7: same with TS MMAs
__global__ void __launch_bounds__(288, 1) k(long long* cyc, int niter) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar, bar_a, bar_b;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  fence_async_shared();
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar_a, 1); mbar_init(&bar_b, 1); fence_mbar_init(); mbar_arrive(&bar_b); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  __shared__ volatile int stop_flag;
  if (threadIdx.x == 0) stop_flag = 0;
  __syncthreads();
  if ((MODE == 8 || MODE == 9) && threadIdx.x >= 32) {
    // warps 1-3: stream 16-byte shared-memory stores over [96 KB, 160 KB) (TMA-write-like traffic)
    uint4* p = reinterpret_cast<uint4*>(smem + 96 * 1024);
    const uint4 val = make_uint4(threadIdx.x, 1, 2, 3);
    int i = threadIdx.x - 32;
    while (!stop_flag) {
#pragma unroll 8
      for (int u = 0; u < 64; ++u) {
        p[i] = val;
        i += 96;
        if (i >= 4096) i -= 4096;
      }
    }
  }
  if ((MODE == 10 || MODE == 11) && threadIdx.x >= 32) {
    // warps 1-3: back-to-back 4 x LDTM.x32 bursts (a softmax warp reading its 128-column S row)
    const int w = threadIdx.x / 32;
    const uint32_t base = tmem + ((uint32_t)(w * 32) << 16) + 256;
    uint32_t r[4][32];
    uint32_t acc = 0;
    while (!stop_flag) {
      tmem_ld32(base, r[0]);
      tmem_ld32(base + 32, r[1]);
      tmem_ld32(base + 64, r[2]);
      tmem_ld32(base + 96, r[3]);
      tmem_ld_wait();
      acc += r[0][0] + r[1][5] + r[2][9] + r[3][31];
    }
    if (acc == 0x12345678u) cyc[0] = acc;
  }
  if ((MODE == 16 || MODE == 17) && threadIdx.x >= 32) {
    // warps 1..8: softmax-like TMEM traffic on their lane quarter: ld 128 columns of S, st 64 of P
    const int w = threadIdx.x / 32;
    const uint32_t base = tmem + ((uint32_t)((w & 3) * 32) << 16) + ((w >> 2) & 1) * 128;
    uint32_t r[4][32];
    uint32_t acc = 0;
    while (!stop_flag) {
      tmem_ld32(base, r[0]);
      tmem_ld32(base + 32, r[1]);
      tmem_ld32(base + 64, r[2]);
      tmem_ld32(base + 96, r[3]);
      tmem_ld_wait();
      acc += r[0][0] + r[1][5] + r[2][9] + r[3][31];
      if (MODE == 17) {
        tmem_st32(base, r[0]);
        tmem_st32(base + 32, r[1]);
        tmem_st_wait();
      }
      for (int d = 0; d < 40; ++d) acc = acc * 1664525u + 1013904223u;   // some ALU work between bursts
    }
    if (acc == 0x12345678u) cyc[0] = acc;
  }
  if ((MODE == 6 || MODE == 7) && threadIdx.x >= 32) {
    // warps 1-3: lane quarters 1-3, columns [256, 384): ld 32 columns, st them back, repeat
    const int w = threadIdx.x / 32;
    const uint32_t base = tmem + ((uint32_t)(w * 32) << 16) + 256;
    uint32_t r[32];
    while (!stop_flag) {
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        tmem_ld32(base + c * 32, r);
        tmem_ld_wait();
        tmem_st32(base + c * 32, r);
      }
      tmem_st_wait();
    }
  }
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, N, false, MODE == 1);
    constexpr uint32_t idesc_mn = idesc_bf16_f32(128, N, false, true);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);  // B: up to 256 rows x 2 atoms = 64KB
    long long t0 = clock64();
    for (int it = 0; it < niter; ++it) {
      if (MODE >= 12) {  // 16/17: as 12 with softmax-like TMEM traffic from 8 warps
        // K4's tensor-pipe sequence per block pair (j even / odd share nothing but the pipe):
        //   PV_j: A = P_j (bf16, TMEM S[b]), D = O_b;  S_{j+2}: D = S[b] (overwrites what PV_j read).
        // 12: exactly that (WAR on S[b] right after PV_j);  13: S_{j+2} into a disjoint region (no WAR);
        // 14: 12 + commit/try_wait(completed)/fence::after before each group (K4's sync points);
        // 15: 12 + commit after each group, no waits
        for (int b = 0; b < 2; ++b) {
          const uint32_t s_b = tmem + b * 128, o_b = tmem + 256 + b * 128;
          if (MODE == 14) { mbar_wait(&bar_b, 0); tc_fence_after(); }
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t bd = smem_desc_sw128(sb + kk * 2048, 128 * 128, 1024);
            mma_ts(o_b, s_b + kk * 8, bd, idesc_mn, 1u);
          }
          if (MODE == 14 || MODE == 15) mma_commit(&bar_a);
          if (MODE == 14) { mbar_wait(&bar_b, 0); tc_fence_after(); }
          const uint32_t d_s = MODE == 13 ? tmem + 64 + b * 128 + 32 : s_b;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t ad = smem_desc_sw128(sa + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024);
            const uint64_t bd = smem_desc_sw128(sb + (kk / 4) * (128 * 128) + (kk % 4) * 32, 16, 1024);
            mma_ss(MODE == 13 ? (b ? tmem + 64 : tmem + 192 + 0) : d_s, ad, bd, idesc, kk > 0 ? 1u : 0u);
          }
          if (MODE == 14 || MODE == 15) mma_commit(&bar_a);
        }
        continue;
      }
      if (MODE == 2) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t ad = smem_desc_sw128(sa + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024);
          const uint64_t bd = smem_desc_sw128(sb + (kk / 4) * (N * 128) + (kk % 4) * 32, 16, 1024);
          mma_ss(tmem, ad, bd, idesc, 1u);
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bd = smem_desc_sw128(sb + kk * 2048, 128 * 128, 1024);
          mma_ts(tmem + 256, tmem + 128 + kk * 8, bd, idesc_mn, 1u);
        }
        continue;
      }
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t bd = MODE == 1 ? smem_desc_sw128(sb + kk * 2048, 128 * 128, 1024)
                                      : smem_desc_sw128(sb + (kk / 4) * (N * 128) + (kk % 4) * 32, 16, 1024);
        if (TS || MODE == 7 || MODE == 9 || MODE == 11) mma_ts(tmem, tmem + 384 + kk * 8, bd, idesc, 1u);
        else if (MODE >= 3) {
          const uint64_t ad = smem_desc_sw128(sa + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024);
          mma_ss(tmem, ad, bd, idesc, 1u);
          if (kk == 7) {
            if (MODE == 3 || MODE == 4) mma_commit(&bar_a);
            if (MODE == 4 || MODE == 5) mbar_wait(&bar_b, 0);
          }
        }
        else {
          const uint64_t ad = smem_desc_sw128(sa + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024);
          mma_ss(tmem, ad, bd, idesc, 1u);
        }
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
    stop_flag = 1;
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}
template <int N, bool TS, int MODE = 0> void run(const char* name) {
  long long* d = nullptr;
  cudaError_t e = cudaMalloc(&d, 148 * 8);
  printf("malloc %s\n", cudaGetErrorString(e)); fflush(stdout);
  auto kern = k<N, TS, MODE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024 + 1024);
  int niter = 2000;
  const int nthr = (MODE == 16 || MODE == 17) ? 288 : 128;
  kern<<<148, nthr, 160 * 1024 + 1024>>>(d, niter);
  printf("first launch %s\n", cudaGetErrorString(cudaDeviceSynchronize())); fflush(stdout);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); kern<<<148, nthr, 160 * 1024 + 1024>>>(d, niter); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[148]; cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  double flops = (MODE >= 12 ? 4 : MODE == 2 ? 2 : 1) * 148.0 * niter * 8 * 2.0 * 128 * N * 16;
  printf("%-14s %s cycles/MMA=%.1f  ideal=%d  TFLOPS=%.0f  (%.3f ms) err=%s\n", name, TS ? "TS" : "SS", avg / (niter * (MODE >= 12 ? 32.0 : MODE == 2 ? 16.0 : 8.0)),
         128 * N / 256, flops / ms / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<128, false>("M128 N128 K16");
  run<256, false>("M128 N256 K16");
  run<64, false>("M128 N64 K16");
  run<128, true>("M128 N128 K16");
  run<256, true>("M128 N256 K16");
  run<128, false, 1>("N128 B-MN");
  run<128, true, 1>("N128 B-MN");
  run<128, false, 2>("S+PV pair/2");
  run<128, false, 3>("8+commit");
  run<128, false, 4>("8+commit+wait");
  run<128, false, 5>("8+wait");
  run<128, false, 6>("SS + TMEM ld/st");
  run<128, false, 7>("TS + TMEM ld/st");
  run<128, false, 8>("SS + smem stores");
  run<128, false, 9>("TS + smem stores");
  run<128, false, 10>("SS + LDTM bursts");
  run<128, false, 11>("TS + LDTM bursts");
  run<128, false, 12>("K4seq WAR");
  run<128, false, 13>("K4seq noWAR");
  run<128, false, 14>("K4seq+sync");
  run<128, false, 15>("K4seq+commit");
  run<128, false, 16>("K4seq+8w ld");
  run<128, false, 17>("K4seq+8w ld/st");
  return 0;
}
