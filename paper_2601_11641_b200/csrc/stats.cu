// stats.cu -- K1 mod_collect_block_stats: pooled block score + row-softmax block mass.
//
// BASELINE.json north_star (1): "a mean-pooled QK^T block-score plus row-softmax block-mass kernel
// (warp-shuffle reductions, vectorised 128-bit loads)".  The paper's own statistic is Eq. 2
// (P:204-206), which needs the full post-softmax map; the pooled surrogate is reading Z1:
//   qbar_i = (1/|I_i|) sum_{p in I_i} Q_p,  kbar_j likewise          (fp32 accumulation)
//   z_ij   = s * qbar_i . kbar_j                                      (s = 1/sqrt(D))
//   W_ij   = |I_j| e^{z_ij} / sum_j' |I_j'| e^{z_ij'}                 (block mass; ragged blocks Z16)
//
// Two kernels:
//   pool_kernel   -- HBM-bound: streams Q and K once (2*B*H*N*D*2 bytes) with 128-bit
//                    non-allocating loads; one CTA per (tensor, head, block); fixed-order
//                    reduction (deterministic).
//   score_kernel  -- z = qbar kbar^T (n x n x D per head, packed fp32 FFMA2, 4x4 register tiles over
//                    shared-memory tiles) fused with the log-size bias and the row softmax; one CTA
//                    owns 64 full rows so the softmax needs no inter-CTA communication.
#include "common.cuh"

namespace {

template <int D>
__global__ void __launch_bounds__(256) pool_kernel(const __nv_bfloat16* __restrict__ q,
                                                    const __nv_bfloat16* __restrict__ k, float* __restrict__ qbar,
                                                    float* __restrict__ kbar, int N, int n, int block) {
  constexpr int TPR = D / 8;          // threads per token row (8 bf16 = 16 bytes each)
  constexpr int RPI = 256 / TPR;      // rows per iteration
  const int i = blockIdx.x;           // block index
  const size_t bh = blockIdx.y;
  const bool isk = blockIdx.z;
  const __nv_bfloat16* src = (isk ? k : q) + bh * (size_t)N * D;
  float* dst = (isk ? kbar : qbar) + (bh * n + i) * D;
  const int lo = i * block;
  const int hi = min(lo + block, N);
  const int t = threadIdx.x;
  const int c8 = (t % TPR) * 8;
  const int r0 = t / TPR;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  // 4 independent 16-byte loads in flight per thread
  for (int r = lo + r0; r < hi; r += 4 * RPI) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int rr = r + u * RPI;
      v[u] = rr < hi ? ld_nc_v4(src + (size_t)rr * D + c8) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 f = __bfloat1622float2(h2[e]);
        acc[2 * e] += f.x;
        acc[2 * e + 1] += f.y;
      }
    }
  }
  __shared__ float red[RPI][D + 4];
#pragma unroll
  for (int e = 0; e < 8; ++e) red[r0][c8 + e] = acc[e];
  __syncthreads();
  const float inv = 1.0f / (float)(hi - lo);
  for (int c = t; c < D; c += 256) {
    float s = 0.f;
    for (int r = 0; r < RPI; ++r) s += red[r][c];  // fixed order
    dst[c] = s * inv;
  }
}

// z = s * qbar kbar^T for 64 rows x all n columns of one head per CTA (256 threads, 4 x 4 outputs
// each, packed FFMA2), fused with ln|I_j| and the row softmax.  The qbar tile is staged once
// (transposed, D x 64); kbar tiles of 64 columns are prefetched into registers while the previous
// tile is consumed.
constexpr int SR = 64, SC = 64;

__device__ __forceinline__ float2 ffma2s(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n mov.b64 rc, {%6,%7};\n"
      " fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

template <int D>
__global__ void __launch_bounds__(256) score_kernel(const float* __restrict__ qbar, const float* __restrict__ kbar,
                                                     const float* __restrict__ log_sizes, float* __restrict__ W,
                                                     int n, float scale) {
  extern __shared__ __align__(16) float sm[];
  float (*As)[SR + 4] = reinterpret_cast<float(*)[SR + 4]>(sm);                       // [D][SR+4]
  float (*Bs)[SC + 4] = reinterpret_cast<float(*)[SC + 4]>(sm + D * (SR + 4));        // [D][SC+4]
  __shared__ float rowmax_s[SR], rowsum_s[SR];
  const size_t bh = blockIdx.y;
  const int r0 = blockIdx.x * SR;
  const float* Q = qbar + bh * (size_t)n * D;
  const float* K = kbar + bh * (size_t)n * D;
  float* Wh = W + bh * (size_t)n * n;
  const int t = threadIdx.x;
  const int tr = (t / 16) * 4;       // rows tr..tr+3 of the tile
  const int tc = (t % 16) * 4;       // cols tc..tc+3 of the tile
  const float scale_l2 = scale * 1.4426950408889634f;
  constexpr int V4 = SR * D / 4 / 256;   // float4 loads per thread per tile
  // stage qbar (transposed)
#pragma unroll
  for (int u = 0; u < V4; ++u) {
    const int e = t + u * 256;            // float4 index: consecutive threads -> consecutive rows
    const int r = e % SR, d4 = (e / SR) * 4; // (transposed shared-memory stores stay conflict-free)
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r0 + r < n) v = *reinterpret_cast<const float4*>(Q + (size_t)(r0 + r) * D + d4);
    As[d4][r] = v.x; As[d4 + 1][r] = v.y; As[d4 + 2][r] = v.z; As[d4 + 3][r] = v.w;
  }
  float4 pre[V4];
  auto load_b = [&](int c0) {
#pragma unroll
    for (int u = 0; u < V4; ++u) {
      const int e = t + u * 256;
      const int c = e % SC, d4 = (e / SC) * 4;
      pre[u] = (c0 + c < n) ? *reinterpret_cast<const float4*>(K + (size_t)(c0 + c) * D + d4)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  float m_run[4], l_run[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    m_run[a] = -INFINITY;
    l_run[a] = 0.f;
  }
  load_b(0);
  for (int c0 = 0; c0 < n; c0 += SC) {
    __syncthreads();                      // previous tile consumed
#pragma unroll
    for (int u = 0; u < V4; ++u) {
      const int e = t + u * 256;
      const int c = e % SC, d4 = (e / SC) * 4;
      Bs[d4][c] = pre[u].x; Bs[d4 + 1][c] = pre[u].y; Bs[d4 + 2][c] = pre[u].z; Bs[d4 + 3][c] = pre[u].w;
    }
    __syncthreads();
    if (c0 + SC < n) load_b(c0 + SC);     // prefetch the next tile while computing this one
    float2 acc[4][2];
#pragma unroll
    for (int x = 0; x < 4; ++x) acc[x][0] = acc[x][1] = make_float2(0.f, 0.f);
    // software-pipelined: the shared-memory operands of step d+1 are loaded before step d's FFMA2s
    float4 an = *reinterpret_cast<const float4*>(&As[0][tr]);
    float4 bn = *reinterpret_cast<const float4*>(&Bs[0][tc]);
#pragma unroll 4
    for (int d = 0; d < D; ++d) {
      const float4 a = an, b = bn;
      if (d + 1 < D) {
        an = *reinterpret_cast<const float4*>(&As[d + 1][tr]);
        bn = *reinterpret_cast<const float4*>(&Bs[d + 1][tc]);
      }
      const float av[4] = {a.x, a.y, a.z, a.w};
      const float2 b01 = make_float2(b.x, b.y), b23 = make_float2(b.z, b.w);
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        acc[x][0] = ffma2s(make_float2(av[x], av[x]), b01, acc[x][0]);
        acc[x][1] = ffma2s(make_float2(av[x], av[x]), b23, acc[x][1]);
      }
    }
    // logits = s*z + ln|I_j|, written in place; online row max / sum
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int r = r0 + tr + x;
      const float zz[4] = {acc[x][0].x, acc[x][0].y, acc[x][1].x, acc[x][1].y};
      float v[4];
#pragma unroll
      for (int y = 0; y < 4; ++y) {   // log2-domain logits: (s z + ln|I_j|) * log2(e)
        const int c = c0 + tc + y;
        v[y] = (c < n) ? fmaf(zz[y], scale_l2, log_sizes[c] * 1.4426950408889634f) : -INFINITY;
        if (r < n && c < n) Wh[(size_t)r * n + c] = v[y];
      }
      const float mx = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
      const float mnew = fmaxf(m_run[x], mx);
      if (mnew > -INFINITY) {
        float sacc = l_run[x] * exp2f(m_run[x] - mnew);
#pragma unroll
        for (int y = 0; y < 4; ++y) sacc += exp2f(v[y] - mnew);
        l_run[x] = sacc;
        m_run[x] = mnew;
      }
    }
  }
  // combine the 16 column-threads of each row (16 consecutive lanes)
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    float m = m_run[x];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float l = (m_run[x] > -INFINITY) ? l_run[x] * exp2f(m_run[x] - m) : 0.f;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if ((t % 16) == 0) {
      rowmax_s[tr + x] = m;
      rowsum_s[tr + x] = l;
    }
  }
  __syncthreads();
  // W = exp(logit - m) / l, in place (this CTA owns rows r0..r0+63)
  for (int rr = t / 32; rr < SR; rr += 8) {
    const int r = r0 + rr;
    if (r >= n) break;
    const float m = rowmax_s[rr];
    const float invl = 1.0f / rowsum_s[rr];
    for (int c = t % 32; c < n; c += 32) {
      float* p = &Wh[(size_t)r * n + c];
      *p = exp2f(*p - m) * invl;
    }
  }
}

}  // namespace

extern "C" mod_status mod_collect_block_stats(mod_plan P, const void* q, const void* k, float* stats, void* ws,
                                              void* stream) {
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  MOD_REQUIRE(q && k && stats && ws, MOD_ERR_USAGE, "mod_collect_block_stats: q, k, stats, ws must be non-NULL");
  const int BH = P->L.batch * P->L.heads, n = P->n, D = P->L.head_dim;
  float* qbar = reinterpret_cast<float*>(static_cast<char*>(ws) + P->ws_qbar);
  float* kbar = reinterpret_cast<float*>(static_cast<char*>(ws) + P->ws_kbar);
  cudaStream_t s = as_stream(stream);
  const dim3 pg(n, BH, 2);
  if (D == 128)
    pool_kernel<128><<<pg, 256, 0, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k, qbar, kbar, P->N, n,
                                        P->L.block);
  else
    pool_kernel<64><<<pg, 256, 0, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k, qbar, kbar, P->N, n,
                                       P->L.block);
  MOD_LAUNCH_CHECK();
  const size_t ssm = (size_t)D * ((SR + 4) + (SC + 4)) * sizeof(float);
  if (D == 128) {
    MOD_CUDA(cudaFuncSetAttribute(score_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
    score_kernel<128><<<dim3((n + SR - 1) / SR, BH), 256, ssm, s>>>(qbar, kbar, P->d_log_sizes, stats, n, P->scale);
  } else {
    MOD_CUDA(cudaFuncSetAttribute(score_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
    score_kernel<64><<<dim3((n + SR - 1) / SR, BH), 256, ssm, s>>>(qbar, kbar, P->d_log_sizes, stats, n, P->scale);
  }
  MOD_LAUNCH_CHECK();
  mod_note_launches(2);
  return MOD_OK;
}
