// Throughput of exp2 variants on sm_100a (bring-up microbenchmark, not part of libmoddit).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ float ex2f(float x){float y;asm volatile("ex2.approx.ftz.f32 %0, %1;":"=f"(y):"f"(x));return y;}
__device__ __forceinline__ uint32_t ex2bf(uint32_t x){uint32_t y;asm volatile("ex2.approx.ftz.bf16x2 %0, %1;":"=r"(y):"r"(x));return y;}
__device__ __forceinline__ uint32_t ex2h(uint32_t x){uint32_t y;asm volatile("ex2.approx.f16x2 %0, %1;":"=r"(y):"r"(x));return y;}
__device__ __forceinline__ float ex2poly(float x){  // 2^x, x <= 0, degree-3 minimax on [0,1)
  x = fmaxf(x, -126.f);
  float fl = floorf(x); float f = x - fl;
  float p = fmaf(fmaf(fmaf(0.0555041086648216f, f, 0.2402264923172000f), f, 0.6931471805599453f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((int)fl << 23));
}
__device__ __forceinline__ float ex2poly2(float x){  // 2^x via round-to-nearest split, FMA pipe only
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.0f;            // 1.5*2^23: integer part lands in the low mantissa bits
  const float j = t - 12582912.0f;
  const float f = x - j;                       // [-0.5, 0.5]
  float p = fmaf(fmaf(fmaf(0.05550411f, f, 0.24022652f), f, 0.69314718f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
template<int MODE> __global__ void k(float* out, int iters){
  float a[8]; uint32_t b[8];
  for(int i=0;i<8;++i){a[i]=-(threadIdx.x%7)*0.01f-i*0.1f; b[i]=0xBF80BF80u+i;}
  for(int it=0;it<iters;++it){
#pragma unroll
    for(int i=0;i<8;++i){
      if(MODE==0) a[i]=ex2f(a[i])-1.0f;
      if(MODE==1) b[i]=ex2bf(b[i])^0x80008000u;
      if(MODE==2) b[i]=ex2h(b[i])^0x80008000u;
      if(MODE==3) a[i]=ex2poly(a[i])-1.0f;
      if(MODE==4) a[i]=ex2poly2(a[i])-1.0f;
      if(MODE==5) { a[i]=(i&1)? ex2poly2(a[i])-1.0f : ex2f(a[i])-1.0f; }
    }
  }
  float s=0; for(int i=0;i<8;++i) s+=a[i]+__uint_as_float(b[i]);
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  float* o; cudaMalloc(&o, 148*8*1024*4);
  int iters=4096; cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[6]={"ex2.f32","ex2.bf16x2","ex2.f16x2","poly(floor)","poly(magic)","half/half"};
  for(int m=0;m<6;++m){
    for(int rep=0;rep<2;++rep){
      cudaEventRecord(e0);
      if(m==0) k<0><<<148*4,256>>>(o,iters); if(m==1) k<1><<<148*4,256>>>(o,iters);
      if(m==2) k<2><<<148*4,256>>>(o,iters); if(m==3) k<3><<<148*4,256>>>(o,iters);
      if(m==4) k<4><<<148*4,256>>>(o,iters); if(m==5) k<5><<<148*4,256>>>(o,iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms,e0,e1);
      double ops=148.0*4*256*iters*8*(m==1||m==2?2:1);
      int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      if(rep) printf("%-12s %.3f ms  %.1f Gexp/s  = %.2f exp/clk/SM at %d MHz\n",names[m],ms,ops/ms/1e6, ops/(ms*1e-3)/(clk*1e3)/148, clk/1000);
    }
  }
  return 0;
}
