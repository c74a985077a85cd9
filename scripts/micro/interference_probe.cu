// interference_probe.cu -- does a warp that issues tcgen05 MMAs slow the arithmetic warps of its SM
// sub-partition?  (K4 traces show the softmax warps of the issuers' sub-partitions lagging.)
// One CTA per SM, 320 threads: warps 2..9 run a fixed softmax-like loop (FFMA2, MUFU ex2, FADD2, F2FP on 64
// scores per thread, 2 warps per sub-partition) and record their cycles; warp 1 runs the mode's activity
// until the workers are done.  Prints the mean worker cycles per sub-partition for each mode.
//   mode 0  issuer idle
//   mode 1  K4's MMA stream: 8 SS MMAs (128x128x16) + 8 TS MMAs + commit per group, waits 2 groups back
//   mode 2  the same MMAs, elect.sync + whole warp converged (K4's issue form)
//   mode 3  try_wait polling on a barrier that never completes (a waiting issuer)
//   mode 4  try_wait with a suspend-time hint on a barrier that never completes
//   mode 5  one MMA group every ~2000 cycles (light issue)
//   mode 6  one lane streaming bulk copies global -> shared (4 x 16 KB per round, waiting on each round)
//   mode 7  the same from a converged warp (elect one lane per copy)
#include <cstdio>
#include <cstdint>
#include "../../paper_2601_11641_b200/csrc/sm100.cuh"
using namespace sm100;

constexpr uint32_t IDESC_S = idesc_bf16_f32(128, 128, false, false);
constexpr uint32_t IDESC_O = idesc_bf16_f32(128, 128, false, true);
constexpr int TILE = 32768;

template <int MODE>
__global__ void __launch_bounds__(320, 1) probe(float* out, int iters, const unsigned char* __restrict__ gsrc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 3 * TILE);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 5);
  volatile int* stop = reinterpret_cast<volatile int*>(bars + 6);
  __shared__ long long cyc[8];
  __shared__ int ndone;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 3 * TILE / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  fence_async_shared();
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);   // never completes
    mbar_init(&bars[3], 1);   // bulk-copy rounds (modes 6, 7)
    *stop = 0;
    ndone = 0;
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp >= 2) {
    float s[64];
#pragma unroll
    for (int c = 0; c < 64; ++c) s[c] = (float)((c * 37 + threadIdx.x) % 101) * 0.05f;
    uint32_t sink = 0;
    float acc = 0.f;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int c = 0; c < 64; ++c) asm volatile("" : "+f"(s[c]));
      const float2 sc2 = make_float2(0.127f, 0.127f), nm2 = make_float2(-acc, -acc);
      float2 a2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < 64; c += 2) {
        const float2 x = ffma2(make_float2(s[c], s[c + 1]), sc2, nm2);
        float2 p;
        if (((c / 2) & 7) < 2) {
          p = ex2_poly2<true>(x);
        } else {
          p.x = ex2(x.x);
          p.y = ex2(x.y);
        }
        a2 = fadd2(a2, p);
        sink ^= pack_bf16(p.x, p.y);
      }
      acc = (a2.x + a2.y) * 1e-9f;
    }
    const long long t1 = clock64();
    if (lane == 0) {
      cyc[warp - 2] = t1 - t0;
      if (atomicAdd(&ndone, 1) == 7) *stop = 1;   // the last worker stops the issuer
    }
    if (sink == 0x12345678u) out[0] = acc;
  } else if (warp == 1) {
    const uint64_t a_base = smem_desc_sw128(smem_u32(smem), 16, 1024);
    const uint64_t b_base = smem_desc_sw128(smem_u32(smem + TILE), 16, 1024);
    const uint64_t v_base = smem_desc_sw128(smem_u32(smem + 2 * TILE), 128 * 128, 1024);
    if (MODE == 1 || MODE == 5) {
      if (lane == 0) {
        for (int j = 0; !*stop; ++j) {
          if (j >= 2) mbar_wait(&bars[j & 1], ((j >> 1) - 1) & 1);
          tc_fence_after();
          if (MODE == 5) {
            const long long t = clock64();
            while (clock64() - t < 2000) {
            }
          }
          const uint32_t s_t = tmem + (j & 1) * 128;
          static_for<8>([&](auto kc) {
            constexpr int kk = decltype(kc)::value;
            mma_ss_off<((kk / 4) * 16384 + (kk % 4) * 32) / 16, ((kk / 4) * 16384 + (kk % 4) * 32) / 16>(
                s_t, a_base, b_base, IDESC_S, kk > 0);
          });
          const uint32_t p_t = tmem + ((j + 1) & 1) * 128;
          static_for<8>([&](auto kc) {
            constexpr int kk = decltype(kc)::value;
            mma_ts_off<kk * 8, kk * 2048 / 16>(tmem + 256, p_t, v_base, IDESC_O, 1u);
          });
          mma_commit(&bars[j & 1]);
        }
      }
    } else if (MODE == 2) {
      for (int j = 0; !*stop; ++j) {
        if (j >= 2) mbar_wait_sleep(&bars[j & 1], ((j >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t s_t = tmem + (j & 1) * 128;
        static_for<8>([&](auto kc) {
          constexpr int kk = decltype(kc)::value;
          mma_ss_e<((kk / 4) * 16384 + (kk % 4) * 32) / 16, ((kk / 4) * 16384 + (kk % 4) * 32) / 16>(
              s_t, a_base, b_base, IDESC_S, kk > 0 ? 1u : 0u);
        });
        const uint32_t p_t = tmem + ((j + 1) & 1) * 128;
        static_for<8>([&](auto kc) {
          constexpr int kk = decltype(kc)::value;
          mma_ts_e<kk * 8, kk * 2048 / 16>(tmem + 256, p_t, v_base, IDESC_O, 1u);
        });
        mma_commit_e(&bars[j & 1]);
        __syncwarp();
      }
    } else if (MODE == 6 || MODE == 7) {
      uint32_t ph = 0;
      for (int it = 0; !*stop; ++it) {
        if (MODE == 6 && lane != 0) break;
        const unsigned char* src = gsrc + (size_t)((blockIdx.x * 7 + it) % 64) * 4 * 16384;
        if (lane == 0) mbar_arrive_expect_tx(&bars[3], 4 * 16384);
        if (MODE == 7) __syncwarp();
        for (int c = 0; c < 4; ++c) {
          const bool me = MODE == 6 ? true : elect_one();
          if (me)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(smem + 16384 * c)), "l"(src + 16384 * c), "r"(16384), "r"(smem_u32(&bars[3]))
                         : "memory");
        }
        mbar_wait_sleep(&bars[3], ph);
        ph ^= 1;
      }
    } else if (MODE == 3 || MODE == 4) {
      if (lane == 0) {
        while (!*stop) {
          uint32_t ok;
          if (MODE == 3)
            asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\nselp.u32 %0,1,0,P;\n}\n"
                         : "=r"(ok) : "r"(smem_u32(&bars[2])) : "memory");
          else
            asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0, %2;\nselp.u32 %0,1,0,P;\n}\n"
                         : "=r"(ok) : "r"(smem_u32(&bars[2])), "r"(0x100000u) : "memory");
          if (ok) break;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
  if (threadIdx.x == 0) {
    for (int w = 0; w < 8; ++w) atomicAdd(&out[1 + (w + 2) % 4], (float)cyc[w] * 0.5f);   // per sub-partition
  }
}

template <int MODE>
void run(const char* name, int sms) {
  static unsigned char* g = nullptr;
  if (!g) {
    cudaMalloc(&g, 64ull * 4 * 16384);
    cudaMemset(g, 0, 64ull * 4 * 16384);
  }
  float* d;
  cudaMalloc(&d, 5 * sizeof(float));
  cudaMemset(d, 0, 5 * sizeof(float));
  const int smem = 3 * TILE + 128;
  cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<MODE><<<sms, 320, smem>>>(d, 200, g);   // warm-up
  cudaMemset(d, 0, 5 * sizeof(float));
  probe<MODE><<<sms, 320, smem>>>(d, 2000, g);
  cudaError_t e = cudaDeviceSynchronize();
  float h[5];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("mode %d %-44s %s  cycles per worker iteration by sub-partition: %.0f %.0f %.0f %.0f\n", MODE, name,
         cudaGetErrorString(e), h[1] / sms / 2000, h[2] / sms / 2000, h[3] / sms / 2000, h[4] / sms / 2000);
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("issuer idle", sms);
  run<1>("single-lane MMA stream (waits 2 groups back)", sms);
  run<2>("converged elect.sync MMA stream (K4 form)", sms);
  run<3>("try_wait polling", sms);
  run<4>("try_wait with suspend hint", sms);
  run<5>("light MMA issue (1 group / 2000 cycles)", sms);
  run<6>("one lane streaming bulk copies", sms);
  run<7>("converged warp streaming bulk copies", sms);
  run<0>("issuer idle (again)", sms);
  return 0;
}
