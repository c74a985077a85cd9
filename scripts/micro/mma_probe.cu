// mma_probe.cu -- what slows K4's tcgen05 MMAs in situ (bring-up tool, not product).
// One CTA per SM runs K4's tensor sequence per "block": S = Q K^T (8 x SS M128 N128 K16, Q / K 128B-swizzled
// K-major in shared memory) then PV (8 x TS M128 N128 K16, P from TMEM, V MN-major in shared memory), with one
// commit per MMA group and waits only on commits two groups back (so the pipe never drains), while optional
// side traffic runs:
//   bit 1  a producer warp streams bulk copies (cp.async.bulk, the TMA engine) of 64 KB per block into other
//          shared-memory slots (K4's K/V gathers)
//   bit 2  8 warps tcgen05.ld 32 columns + tcgen05.st 16 columns of other TMEM columns per ~block (softmax)
//   bit 4  A/B of the S MMA: A (Q) from TMEM instead of shared memory (TS form)
// Prints cycles per block (16 MMAs) per mode.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include "../../paper_2601_11641_b200/csrc/sm100.cuh"
using namespace sm100;

constexpr int BLOCKS = 256;
constexpr uint32_t IDESC_S = idesc_bf16_f32(128, 128, false, false);
constexpr uint32_t IDESC_O = idesc_bf16_f32(128, 128, false, true);
constexpr int TILE = 32768;   // one 128 x 128 bf16 tile

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void keepf(float& x) { asm volatile("" : "+f"(x)); }

template <int MODE>
__global__ void __launch_bounds__(MODE & 16 ? 576 : 320, 1) probe(const unsigned char* __restrict__ gsrc, float* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  // Q | K | V | side slots (3 x 32 KB) | barriers
  unsigned char* sq = smem;
  unsigned char* sk = smem + TILE;
  unsigned char* sv = smem + 2 * TILE;
  unsigned char* side = smem + 3 * TILE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * TILE);
  uint64_t* done = bars;          // [2] MMA group commits
  uint64_t* tma_bar = bars + 2;   // [1]
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 4);
  volatile int* stop = reinterpret_cast<volatile int*>(bars + 5);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&done[0], 1);
    mbar_init(&done[1], 1);
    mbar_init(tma_bar, 1);
    *stop = 0;
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if constexpr (MODE & 8) {   // random bf16 operands (N(0,1)-like magnitudes) instead of zeros
    uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x;
    auto rnd = [&]() {
      x ^= x << 13; x ^= x >> 17; x ^= x << 5;
      const float a = ((x & 0xffff) / 65536.f - 0.5f) * 3.f, b = ((x >> 16) / 65536.f - 0.5f) * 3.f;
      return pack_bf16(a, b);
    };
    uint32_t* w = reinterpret_cast<uint32_t*>(smem);
    for (int i = threadIdx.x; i < 3 * TILE / 4; i += blockDim.x) w[i] = rnd();
    fence_async_shared();
    if (warp >= 2 && warp < 6) {
      const uint32_t tq = tmem + ((uint32_t)((warp & 3) * 32) << 16);
      uint32_t r[32];
      for (int c = 0; c < 512; c += 32) {
#pragma unroll
        for (int e = 0; e < 32; ++e) r[e] = rnd();
        tmem_st32(tq + c, r);
      }
      tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (warp == 1 && lane == 0) {
    const uint64_t a_base = smem_desc_sw128(smem_u32(sq), 16, 1024);
    const uint64_t b_base = smem_desc_sw128(smem_u32(sk), 16, 1024);
    const uint64_t v_base = smem_desc_sw128(smem_u32(sv), 128 * 128, 1024);
    long long t0 = 0;
    for (int j = 0; j < BLOCKS; ++j) {
      if (j == 16) t0 = clock64();
      if (j >= 2) mbar_wait(&done[j & 1], ((j >> 1) - 1) & 1);   // group j-2 retired (never drains the pipe)
      tc_fence_after();
      const uint32_t s_t = tmem + (j & 1) * 128;   // S buffer
      if constexpr (MODE & 4) {
        static_for<8>([&](auto kc) {
          constexpr int kk = decltype(kc)::value;
          mma_ts_off<kk * 8, ((kk / 4) * 16384 + (kk % 4) * 32) / 16>(s_t, tmem + 384, b_base, IDESC_S, kk > 0);
        });
      } else {
        static_for<8>([&](auto kc) {
          constexpr int kk = decltype(kc)::value;
          mma_ss_off<((kk / 4) * 16384 + (kk % 4) * 32) / 16, ((kk / 4) * 16384 + (kk % 4) * 32) / 16>(
              s_t, a_base, b_base, IDESC_S, kk > 0);
        });
      }
      const uint32_t p_t = tmem + ((j + 1) & 1) * 128;   // P of the previous block
      static_for<8>([&](auto kc) {
        constexpr int kk = decltype(kc)::value;
        mma_ts_off<kk * 8, kk * 2048 / 16>(tmem + 256, p_t, v_base, IDESC_O, kk > 0 ? 1u : (j > 0));
      });
      mma_commit(&done[j & 1]);
    }
    mbar_wait(&done[(BLOCKS - 1) & 1], ((BLOCKS - 1) >> 1) & 1);
    const long long t1 = clock64();
    out[blockIdx.x] = (float)(t1 - t0) / (BLOCKS - 16);
    *stop = 1;
  } else if (warp == 0 && (MODE & 1)) {
    if (lane == 0) {
      uint32_t ph = 0;
      for (int it = 0; !*stop && it < 100000; ++it) {
        mbar_arrive_expect_tx(tma_bar, 2 * TILE);
        const unsigned char* src = gsrc + (size_t)((blockIdx.x * 7 + it) % 64) * 2 * TILE;
        for (int c = 0; c < 2; ++c)
          bulk_g2s(side + ((it + c) % 3) * TILE, src + c * TILE, TILE, tma_bar);
        mbar_wait(tma_bar, ph);
        ph ^= 1;
      }
    }
  } else if (warp >= 2 && (MODE & 16) && !((MODE & 128) && (warp & 3) == 1)) {
    // softmax-like arithmetic (FFMA2, MUFU ex2, FADD2, F2FP on 32 scores per thread), 4 warps per SMSP
    float s[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) s[c] = (float)((c * 37 + threadIdx.x) % 101) * 0.05f;
    float acc = 0.f;
    uint32_t sink = 0;
    for (int it = 0; !*stop && it < 1000000; ++it) {
#pragma unroll
      for (int c = 0; c < 32; ++c) keepf(s[c]);
      const float2 sc2 = make_float2(0.127f, 0.127f), nm2 = make_float2(-acc, -acc);
      float2 a2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        const float2 x = ffma2(make_float2(s[c], s[c + 1]), sc2, nm2);
        float2 p;
        if ((MODE & 32) || (!(MODE & 64) && ((c / 2) & 7) < 3)) p = ex2_poly2(x);
        else { p.x = ex2(x.x); p.y = ex2(x.y); }
        a2 = fadd2(a2, p);
        sink ^= pack_bf16(p.x, p.y);
      }
      acc = (a2.x + a2.y) * 1e-9f;
    }
    if (sink == 0x1234567u) out[4001] = acc;
  } else if (warp >= 2 && (MODE & 2)) {
    const int q = warp & 3, h = (warp - 2) >> 2;
    const uint32_t t = tmem + ((uint32_t)(q * 32) << 16) + 448 + h * 32;   // columns 448..511 (not the MMA's)
    uint32_t acc = 0;
    for (int it = 0; !*stop && it < 100000; ++it) {
      uint32_t r[32];
      tmem_ld32(t, r);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 32; ++e) acc += r[e];
      // about the arithmetic time of one block between two bursts
      for (int w = 0; w < 8; ++w) __nanosleep(100);
      tmem_st16(t, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
      tmem_st_wait();
    }
    if (acc == 0x1234567u) out[4000] = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int MODE>
void run(const char* name, const unsigned char* g, float* d) {
  const int smem = 6 * TILE + 64;
  cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int threads = MODE & 16 ? 576 : 320;
  probe<MODE><<<148, threads, smem>>>(g, d);
  probe<MODE><<<148, threads, smem>>>(g, d);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> h(148);
  cudaMemcpy(h.data(), d, 148 * 4, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  printf("%-44s %7.1f cycles/block (16 MMAs)  min %.1f max %.1f  (%s)\n", name, h[74], h[0], h[147],
         cudaGetErrorString(e));
}

int main() {
  unsigned char* g;
  float* d;
  cudaMalloc(&g, 64 * 2 * TILE);
  cudaMemset(g, 0, 64 * 2 * TILE);
  cudaMalloc(&d, 4096 * 4);
  run<0>("MMA only (S: SS, PV: TS)", g, d);
  run<1>("+ bulk copies 64 KB/block into smem", g, d);
  run<2>("+ 8 warps tcgen05.ld/st of other columns", g, d);
  run<3>("+ both", g, d);
  run<4>("S as TS (Q in TMEM)", g, d);
  run<5>("S as TS + bulk copies", g, d);
  run<7>("S as TS + both", g, d);
  run<8>("random operands: MMA only", g, d);
  run<11>("random operands: + both", g, d);
  run<12>("random operands: S as TS", g, d);
  run<16>("+ 16 arithmetic warps (4 per SMSP)", g, d);
  run<17>("+ 16 arithmetic warps + bulk copies", g, d);
  run<20>("S as TS + 16 arithmetic warps", g, d);
  run<16 + 32>("+ 16 warps, FMA-pipe exp only (no MUFU)", g, d);
  run<16 + 64>("+ 16 warps, MUFU exp only", g, d);
  run<16 + 128>("+ 12 warps, none on the MMA warp's SMSP", g, d);
  return 0;
}
