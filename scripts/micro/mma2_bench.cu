// tcgen05.mma cta_group::2 calibration on sm_100a (bring-up microbenchmark for the round-2 K4 design,
// not part of libmoddit): clusters of 2 CTAs (one per SM of a TPC), TMEM allocated with
// cta_group::2, the leader CTA's single thread issues M=256 MMAs (128 rows in each CTA's TMEM, each
// CTA's shared memory holding its own 128 rows of A and half of B), commits multicast to both CTAs.
// Modes: 0 = SS M256 N128 K16 back to back; 1 = K4-like sequence per step: 8 SS MMAs into S[b],
// then 8 TS MMAs (A = P from TMEM) into O[b], alternating b; 2 = mode 1 + commit/wait per group.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
               "r"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar, uint16_t mask) {   // mask: CTAs of the pair to signal
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::
                   "r"(smem_u32(bar)), "h"(mask)
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::
                   "r"(smem_u32(bar)), "r"(parity)
               : "memory");
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(long long* cyc, int niter) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  const bool leader = cluster_rank() == 0;
  if (leader && threadIdx.x == 0) {
    // A: 128 rows x 64 cols bf16 atoms at [0, 32K) (2 atoms: K = 128); B (K-major, N/2 = 64 rows per CTA
    // for the S MMA): [32K, 48K); V (MN-major, 128 keys x 64 columns per CTA): [64K, 96K)
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768), sv = smem_u32(smem + 65536);
    constexpr uint32_t IS = idesc_bf16(256, 128, false), IO = idesc_bf16(256, 128, true);
    long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < niter; ++it) {
      if (MODE == 0) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma2_ss(tmem, desc_sw128(sa + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024),
                  desc_sw128(sb + (kk / 4) * 8192 + (kk % 4) * 32, 16, 1024), IS, 1u);
        continue;
      }
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const uint32_t s_b = tmem + b * 128, o_b = tmem + 256 + b * 128;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma2_ts(o_b, s_b + kk * 8, desc_sw128(sv + kk * 2048, 8192, 1024), IO, 1u);
        if (MODE == 2) { commit2(&bar, 1); mbar_wait(&bar, ph); ph ^= 1; asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma2_ss(s_b, desc_sw128(sa + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024),
                  desc_sw128(sb + (kk / 4) * 8192 + (kk % 4) * 32, 16, 1024), IS, kk > 0 ? 1u : 0u);
        if (MODE == 2) { commit2(&bar, 1); mbar_wait(&bar, ph); ph ^= 1; asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
      }
    }
    commit2(&bar, 3);   // the only commit that also reaches the peer CTA
    mbar_wait(&bar, ph);
    long long t1 = clock64();
    cyc[blockIdx.x / 2] = t1 - t0;
  } else if (!leader && threadIdx.x == 0) {
    // the peer's barrier receives only the final commit: the pair's MMAs are done when it completes
    mbar_wait(&bar, 0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

template <int MODE>
void run(const char* name, double mmas_per_iter) {
  long long* d = nullptr;
  cudaMalloc(&d, 74 * 8);
  auto kern = k<MODE>;
  const int smem = 128 * 1024 + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int niter = 1000;
  kern<<<148, 128, smem>>>(d, niter);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<148, 128, smem>>>(d, niter);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[74]; cudaMemcpy(h, d, 74 * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 74; ++i) avg += h[i]; avg /= 74;
  const double flops = 74.0 * niter * mmas_per_iter * 2.0 * 256 * 128 * 16;
  printf("%-22s cycles per M256 MMA = %.1f (64 = both SMs' tensor cores saturated)  TFLOPS=%.0f  err=%s\n", name,
         avg / (niter * mmas_per_iter), flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0>("SS M256 N128 K16", 8);
  run<1>("K4 seq (TS+SS)", 32);
  run<2>("K4 seq + commit/wait", 32);
  return 0;
}
