// fp64_bench.cu -- DFMA (FP64 pipe) and DMMA (mma.sync m8n8k4 f64) throughput per SM on this GPU, to size
// the fp64 solve of the mixture fit (fit.cu).  Prints DFMA/clk/SM and fp64 TFLOP/s for both.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
  const double b = 1.0000001, c = 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double acc[4][2] = {};
  double a = threadIdx.x * 1e-9, b = 1.0000001;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int sms = prop.multiProcessorCount, iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    dfma_kernel<<<sms * 4, 256>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double dfma = (double)sms * 4 * 256 * iters * 8;
    printf("DFMA: %.3f ms, %.2f TFLOP/s fp64, %.1f DFMA/clk/SM at %d MHz nominal\n", ms, 2 * dfma / (ms * 1e-3) / 1e12,
           dfma / (ms * 1e-3) / sms / (clk_khz * 1e3), clk_khz / 1000);
    cudaEventRecord(e0);
    dmma_kernel<<<sms * 4, 256>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = (double)sms * 4 * 8 * iters * 4 * (2.0 * 8 * 8 * 4);   // per warp per mma: 2*m*n*k
    printf("DMMA m8n8k4: %.3f ms, %.2f TFLOP/s fp64\n", ms, fl / (ms * 1e-3) / 1e12);
  }
  return 0;
}
