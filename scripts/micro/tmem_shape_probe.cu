// tmem_shape_probe.cu -- bring-up check of the tcgen05.ld/st .16x32bx2 thread <-> (lane, column) mapping
// that the K4 softmax uses to give each warp 16 full rows (two threads per row: column halves).
// One CTA of 4 warps: warp w fills its TMEM lane quarter with v(lane, col) = lane * 1000 + col through the
// .32x32b shape, then reads lanes [32w + 16h, +16) with .16x32bx2.x32 (second half at column + 64) and
// reports mismatches against the assumed mapping: thread t -> lane 32w + 16h + (t % 16),
// column c0 + (t / 16) * 64 + r for register r.  Then the reverse: store with .16x32bx2, load with .32x32b.
#include <cstdio>
#include <cstdint>
#include "../../paper_2601_11641_b200/csrc/sm100.cuh"
using namespace sm100;

__device__ __forceinline__ void ld16x2_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32], 64;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void st16x2_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x32bx2.x16.b32 [%0], 32, {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

__global__ void probe(int* bad) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t lo = (uint32_t)(warp * 32) << 16;
  for (int c = 0; c < 128; c += 32) {
    uint32_t v[32];
    for (int e = 0; e < 32; ++e) v[e] = (warp * 32 + lane) * 1000 + c + e;
    tmem_st32(tmem + lo + c, v);
  }
  tmem_st_wait();
  int nbad = 0;
  for (int h = 0; h < 2; ++h) {
    uint32_t r[32];
    ld16x2_x32(tmem + ((uint32_t)(warp * 32 + 16 * h) << 16) + 0, r);
    tmem_ld_wait();
    for (int e = 0; e < 32; ++e) {
      const uint32_t want = (warp * 32 + 16 * h + lane % 16) * 1000 + (lane / 16) * 64 + e;
      if (r[e] != want) {
        if (nbad < 4) printf("ld w%d h%d t%d r%d got %u want %u\n", warp, h, lane, e, r[e], want);
        ++nbad;
      }
    }
  }
  // store: row (32w + 16h + t%16), packed columns 256 + (t/16)*32 + e  (second half at +32)
  for (int h = 0; h < 2; ++h) {
    uint32_t v[16];
    for (int e = 0; e < 16; ++e) v[e] = 7000000 + (warp * 32 + 16 * h + lane % 16) * 1000 + (lane / 16) * 32 + e;
    st16x2_x16(tmem + ((uint32_t)(warp * 32 + 16 * h) << 16) + 256, v);
  }
  tmem_st_wait();
  uint32_t r[32];
  tmem_ld32(tmem + lo + 256, r);   // columns 256..287: halves at 256..271 and 288.. -> check 256..271 and 288..303
  uint32_t r2[16];
  tmem_ld16(tmem + lo + 288, r2);
  tmem_ld_wait();
  for (int e = 0; e < 16; ++e) {
    const uint32_t w0 = 7000000 + (warp * 32 + lane) * 1000 + e, w1 = 7000000 + (warp * 32 + lane) * 1000 + 32 + e;
    if (r[e] != w0 || r2[e] != w1) {
      if (nbad < 8) printf("st w%d t%d e%d got %u %u want %u %u\n", warp, lane, e, r[e], r2[e], w0, w1);
      ++nbad;
    }
  }
  atomicAdd(bad, nbad);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int main() {
  int* d;
  cudaMalloc(&d, 4);
  cudaMemset(d, 0, 4);
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  int h = -1;
  cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
  printf("tmem_shape_probe: %s, mismatches %d\n", cudaGetErrorString(e), h);
  return h != 0;
}
