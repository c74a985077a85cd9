// quant.cu -- Sage-style quantization of Q, K, V for the quantized sparse attention.
//
// Reading Z30 (the paper's sparse stage is SageAttention, precision unstated):
//   Q, K : symmetric INT8 per (head, 128-token block): s = absmax / 127, code = rint(x * (127 / absmax))
//          in fp32 (round half to even), |code| <= 127; an all-zero block has s = 0, codes 0
//   V    : FP8 e4m3 per (head, channel): s_d = absmax_d / 448, code = RN_e4m3(v * (448 / absmax_d)),
//          satfinite; stored transposed [B,H,D,Np] so that the PV MMA reads it K-major
// Kernels (HBM-bound):
//   vmax_kernel        per-channel |V| maxima (uint atomicMax on the fp32 bit pattern of |v|: exact and
//                      order independent, hence deterministic)
//   qk_quant_kernel    one CTA per (tensor, head, block): block absmax (fixed tree), codes
//   v_quant_kernel     one CTA per (head, block): e4m3 codes, transposed through shared memory
#include <algorithm>

#include "common.cuh"

namespace {

constexpr int QD = 128;          // head dim of the quantized path
constexpr int QB = 128;          // block size of the quantized path

struct QuantLayout {
  size_t q8, k8, vt8, qs, ks, vs, vmax, bytes;
  int Np;
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

QuantLayout quant_layout(mod_plan P) {
  QuantLayout Lq{};
  const size_t BH = (size_t)P->L.batch * P->L.heads;
  Lq.Np = (P->N + 15) / 16 * 16;
  size_t off = 0;
  Lq.q8 = off;   off = align256(off + BH * P->N * QD);
  Lq.k8 = off;   off = align256(off + BH * P->N * QD);
  Lq.vt8 = off;  off = align256(off + BH * QD * (size_t)Lq.Np);
  Lq.qs = off;   off = align256(off + BH * P->n * sizeof(float));
  Lq.ks = off;   off = align256(off + BH * P->n * sizeof(float));
  Lq.vs = off;   off = align256(off + BH * QD * sizeof(float));
  Lq.vmax = off; off = align256(off + BH * QD * sizeof(uint32_t));
  Lq.bytes = off;
  return Lq;
}

mod_status check_quant_plan(mod_plan P) {
  MOD_REQUIRE(P->L.head_dim == QD && P->L.block == QB, MOD_ERR_UNSUPPORTED,
              "quantized attention supports head_dim=128, block=128 only (got head_dim=%d, block=%d)",
              P->L.head_dim, P->L.block);
  return MOD_OK;
}

// fp32 pair -> two e4m3 bytes in memory order (x0 at the lower address)
__device__ __forceinline__ uint16_t e4m3x2(float x0, float x1) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(x1), "f"(x0));
  return r;
}

__global__ void __launch_bounds__(256) vmax_kernel(const __nv_bfloat16* __restrict__ v, uint32_t* __restrict__ vmax,
                                                   int N, int rows_per_cta) {
  // 16 threads per token row (8 channels = 16 bytes each), 16 rows per step
  const size_t bh = blockIdx.y;
  const int t = threadIdx.x, c8 = (t % 16) * 8, r0 = t / 16;
  const int lo = blockIdx.x * rows_per_cta, hi = min(lo + rows_per_cta, N);
  const __nv_bfloat16* src = v + bh * (size_t)N * QD;
  float m[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) m[e] = 0.f;
  for (int r = lo + r0; r < hi; r += 64) {   // 4 independent 16-byte loads in flight per thread
    int4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = (r + 16 * u < hi) ? ld_nc_v4(src + (size_t)(r + 16 * u) * QD + c8) : make_int4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&x[u]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(h2[e]);
        m[2 * e] = fmaxf(m[2 * e], fabsf(f.x));
        m[2 * e + 1] = fmaxf(m[2 * e + 1], fabsf(f.y));
      }
    }
  }
  __shared__ float red[16][QD];
#pragma unroll
  for (int e = 0; e < 8; ++e) red[r0][c8 + e] = m[e];
  __syncthreads();
  if (t < QD) {
    float mx = 0.f;
    for (int r = 0; r < 16; ++r) mx = fmaxf(mx, red[r][t]);
    atomicMax(vmax + bh * QD + t, __float_as_uint(mx));   // |v| >= 0: uint order == float order
  }
}

// one CTA (256 threads) per (head, block, tensor): 128 rows x 128 channels, 64 values per thread
__global__ void __launch_bounds__(256) qk_quant_kernel(const __nv_bfloat16* __restrict__ q,
                                                       const __nv_bfloat16* __restrict__ k, int8_t* __restrict__ q8,
                                                       int8_t* __restrict__ k8, float* __restrict__ qs,
                                                       float* __restrict__ ks, int N, int n) {
  const int i = blockIdx.x;
  const size_t bh = blockIdx.y;
  const bool isk = blockIdx.z;
  const __nv_bfloat16* src = (isk ? k : q) + (bh * (size_t)N + (size_t)i * QB) * QD;
  int8_t* dst = (isk ? k8 : q8) + (bh * (size_t)N + (size_t)i * QB) * QD;
  const int rows = min(QB, N - i * QB);
  const int t = threadIdx.x;
  // element chunk e (8 bf16 = 16 bytes) for e = t + 256*u, u < 8: row e / 16, channels (e % 16) * 8
  int4 x[8];
  float amax = 0.f;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = t + 256 * u, r = e / 16;
    x[u] = r < rows ? ld_nc_v4(src + (size_t)e * 8) : make_int4(0, 0, 0, 0);
    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&x[u]);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float2 f = __bfloat1622float2(h2[w]);
      amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  __shared__ float red[8];
  if (t % 32 == 0) red[t / 32] = amax;
  __syncthreads();
  amax = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) amax = fmaxf(amax, red[w]);
  const float inv = amax > 0.f ? __fdiv_rn(127.0f, amax) : 0.f;
  if (t == 0) (isk ? ks : qs)[bh * n + i] = amax > 0.f ? __fdiv_rn(amax, 127.0f) : 0.f;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = t + 256 * u, r = e / 16;
    if (r >= rows) continue;
    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&x[u]);
    uint32_t packed[2] = {0u, 0u};
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float2 f = __bfloat1622float2(h2[w]);
      const int c0 = max(-127, min(127, __float2int_rn(__fmul_rn(f.x, inv))));
      const int c1 = max(-127, min(127, __float2int_rn(__fmul_rn(f.y, inv))));
      packed[w / 2] |= ((uint32_t)(c0 & 0xff) | ((uint32_t)(c1 & 0xff) << 8)) << (16 * (w % 2));
    }
    *reinterpret_cast<uint2*>(dst + (size_t)e * 8) = make_uint2(packed[0], packed[1]);
  }
}

// one CTA (256 threads) per (head, block): the bf16 block is staged in shared memory with coalesced
// 16-byte loads; thread (channel c, token half) then reads its channel column (a warp reads 32
// adjacent channels of one token: no bank conflicts), converts to e4m3 and stores 32 consecutive
// tokens of V^T row c as two 16-byte stores (one full 32-byte sector)
__global__ void __launch_bounds__(256) v_quant_kernel(const __nv_bfloat16* __restrict__ v,
                                                      const uint32_t* __restrict__ vmax, uint8_t* __restrict__ vt8,
                                                      float* __restrict__ vs, int N, int Np) {
  const int i = blockIdx.x;
  const size_t bh = blockIdx.y;
  const int t = threadIdx.x;
  const int tok0 = i * QB;
  const int rows = min(QB, N - tok0);
  __shared__ __align__(16) __nv_bfloat16 tile[QB][QD];   // [token][channel]
  const __nv_bfloat16* src = v + (bh * (size_t)N + tok0) * QD;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = t + 256 * u, r = e / 16;
    const int4 x = r < rows ? ld_nc_v4(src + (size_t)e * 8) : make_int4(0, 0, 0, 0);
    *reinterpret_cast<int4*>(&tile[0][0] + (size_t)e * 8) = x;
  }
  const int c = t % QD, half = t / QD;
  const float am = __uint_as_float(vmax[bh * QD + c]);
  const float inv = am > 0.f ? __fdiv_rn(448.0f, am) : 0.f;
  if (i == 0 && half == 0) vs[bh * QD + c] = am > 0.f ? __fdiv_rn(am, 448.0f) : 0.f;
  __syncthreads();
  uint8_t* dst = vt8 + (bh * (size_t)QD + c) * Np;
#pragma unroll
  for (int chunk = 0; chunk < 2; ++chunk) {
    const int r0 = half * 64 + chunk * 32;
    uint32_t w[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float x0 = __bfloat162float(tile[r0 + 4 * q][c]), x1 = __bfloat162float(tile[r0 + 4 * q + 1][c]);
      const float x2 = __bfloat162float(tile[r0 + 4 * q + 2][c]), x3 = __bfloat162float(tile[r0 + 4 * q + 3][c]);
      w[q] = (uint32_t)e4m3x2(__fmul_rn(x0, inv), __fmul_rn(x1, inv)) |
             ((uint32_t)e4m3x2(__fmul_rn(x2, inv), __fmul_rn(x3, inv)) << 16);
    }
    const int tok = tok0 + r0;
    if (tok < Np) *reinterpret_cast<uint4*>(dst + tok) = make_uint4(w[0], w[1], w[2], w[3]);
    if (tok + 16 < Np) *reinterpret_cast<uint4*>(dst + tok + 16) = make_uint4(w[4], w[5], w[6], w[7]);
  }
}

}  // namespace

extern "C" size_t mod_quant_buffer_bytes(mod_plan P) {
  if (mod_validate_plan(P) != MOD_OK || check_quant_plan(P) != MOD_OK) return 0;
  return quant_layout(P).bytes;
}

extern "C" mod_status mod_quant_buffer_layout(mod_plan P, size_t* offsets) {
  MOD_NVTX("mod_quant_buffer_layout");
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  if ((st = check_quant_plan(P)) != MOD_OK) return st;
  MOD_REQUIRE(offsets, MOD_ERR_USAGE, "mod_quant_buffer_layout: offsets must be non-NULL");
  const QuantLayout Lq = quant_layout(P);
  const size_t o[6] = {Lq.q8, Lq.k8, Lq.vt8, Lq.qs, Lq.ks, Lq.vs};
  std::copy(o, o + 6, offsets);
  return MOD_OK;
}

extern "C" mod_status mod_quantize_qkv(mod_plan P, const void* q, const void* k, const void* v, void* qbuf,
                                       void* stream) {
  MOD_NVTX("mod_quantize_qkv");
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  if ((st = check_quant_plan(P)) != MOD_OK) return st;
  MOD_REQUIRE(q && k && v && qbuf, MOD_ERR_USAGE, "mod_quantize_qkv: q, k, v, qbuf must be non-NULL");
  MOD_REQUIRE(((uintptr_t)q & 15) == 0 && ((uintptr_t)k & 15) == 0 && ((uintptr_t)v & 15) == 0 &&
                  ((uintptr_t)qbuf & 255) == 0,
              MOD_ERR_INPUT, "mod_quantize_qkv: q, k, v must be 16-byte and qbuf 256-byte aligned");
  cudaStream_t s = as_stream(stream);
  const QuantLayout Lq = quant_layout(P);
  char* base = static_cast<char*>(qbuf);
  const int BH = P->L.batch * P->L.heads, n = P->n, N = P->N;
  uint32_t* vmax = reinterpret_cast<uint32_t*>(base + Lq.vmax);
  MOD_CUDA(cudaMemsetAsync(vmax, 0, (size_t)BH * QD * sizeof(uint32_t), s));
  constexpr int kRows = 1024;
  vmax_kernel<<<dim3((N + kRows - 1) / kRows, BH), 256, 0, s>>>((const __nv_bfloat16*)v, vmax, N, kRows);
  MOD_LAUNCH_CHECK();
  qk_quant_kernel<<<dim3(n, BH, 2), 256, 0, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                                 reinterpret_cast<int8_t*>(base + Lq.q8),
                                                 reinterpret_cast<int8_t*>(base + Lq.k8),
                                                 reinterpret_cast<float*>(base + Lq.qs),
                                                 reinterpret_cast<float*>(base + Lq.ks), N, n);
  MOD_LAUNCH_CHECK();
  v_quant_kernel<<<dim3(n, BH), 256, 0, s>>>((const __nv_bfloat16*)v, vmax, reinterpret_cast<uint8_t*>(base + Lq.vt8),
                                             reinterpret_cast<float*>(base + Lq.vs), N, Lq.Np);
  MOD_LAUNCH_CHECK();
  mod_note_launches(3);
  return MOD_OK;
}
