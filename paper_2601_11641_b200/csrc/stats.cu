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
//   score_kernel  -- z = qbar kbar^T (n x n x D per head, fp32 FMA, 4x4 register tiles over
//                    shared-memory tiles) fused with the log-size bias and the row softmax; one CTA
//                    owns 32 full rows so the softmax needs no inter-CTA communication.
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

// z tile: 32 rows x 128 cols per step, 256 threads, each 4 rows x 4 cols.
constexpr int SR = 32, SC = 128, SK = 32;  // rows, cols, k-chunk

__global__ void __launch_bounds__(256) score_kernel(const float* __restrict__ qbar, const float* __restrict__ kbar,
                                                     const float* __restrict__ log_sizes, float* __restrict__ W,
                                                     int n, int D, float scale) {
  __shared__ __align__(16) float As[SK][SR + 4];  // qbar^T chunk: As[d][r] (padded)
  __shared__ __align__(16) float Bs[SK][SC + 4];  // kbar^T chunk: Bs[d][c] (padded)
  __shared__ float rowmax_s[SR][33], rowsum_s[SR][33];
  const size_t bh = blockIdx.y;
  const int r0 = blockIdx.x * SR;
  const float* Q = qbar + bh * (size_t)n * D;
  const float* K = kbar + bh * (size_t)n * D;
  float* Wh = W + bh * (size_t)n * n;
  const int t = threadIdx.x;
  const int tr = (t / 32) * 4;   // rows tr..tr+3  (warp w -> rows 4w..4w+3)
  const int tc = (t % 32) * 4;   // cols tc..tc+3
  float m_run[4], l_run[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    m_run[a] = -INFINITY;
    l_run[a] = 0.f;
  }
  for (int c0 = 0; c0 < n; c0 += SC) {
    float acc[4][4] = {};
    for (int d0 = 0; d0 < D; d0 += SK) {
      __syncthreads();
      for (int e = t; e < SR * SK; e += 256) {
        const int r = e / SK, d = e % SK;
        As[d][r] = (r0 + r < n) ? Q[(size_t)(r0 + r) * D + d0 + d] : 0.f;
      }
      for (int e = t; e < SC * SK; e += 256) {
        const int c = e / SK, d = e % SK;
        Bs[d][c] = (c0 + c < n) ? K[(size_t)(c0 + c) * D + d0 + d] : 0.f;
      }
      __syncthreads();
#pragma unroll 8
      for (int d = 0; d < SK; ++d) {
        const float4 a = *reinterpret_cast<const float4*>(&As[d][tr]);
        const float4 b = *reinterpret_cast<const float4*>(&Bs[d][tc]);
        const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(av[x], bv[y], acc[x][y]);
      }
    }
    // logits = s*z + ln|I_j|; write them and keep an online row max / sum
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int r = r0 + tr + x;
      float v[4];
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int c = c0 + tc + y;
        v[y] = (c < n) ? fmaf(acc[x][y], scale, log_sizes[c]) : -INFINITY;
      }
      if (r < n) {
#pragma unroll
        for (int y = 0; y < 4; ++y)
          if (c0 + tc + y < n) Wh[(size_t)r * n + c0 + tc + y] = v[y];
      }
      const float mx = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
      const float mnew = fmaxf(m_run[x], mx);
      if (mnew > -INFINITY) {
        float s = l_run[x] * expf(m_run[x] - mnew);
#pragma unroll
        for (int y = 0; y < 4; ++y) s += expf(v[y] - mnew);
        l_run[x] = s;
        m_run[x] = mnew;
      }
    }
  }
  // combine the 32 column-threads of each row (they are the 32 lanes of one warp)
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    float m = warp_max_f(m_run[x]);
    float l = (m_run[x] > -INFINITY) ? l_run[x] * expf(m_run[x] - m) : 0.f;
    l = warp_sum_f(l);
    rowmax_s[tr + x][t % 32] = m;
    rowsum_s[tr + x][t % 32] = l;
  }
  __syncthreads();
  // W = exp(logit - m) / l, in place (this CTA owns rows r0..r0+31)
  for (int rr = t / 32; rr < SR; rr += 8) {
    const int r = r0 + rr;
    if (r >= n) break;
    const float m = rowmax_s[rr][0];
    const float invl = 1.0f / rowsum_s[rr][0];
    for (int c = t % 32; c < n; c += 32) {
      float* p = &Wh[(size_t)r * n + c];
      *p = expf(*p - m) * invl;
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
  score_kernel<<<dim3((n + SR - 1) / SR, BH), 256, 0, s>>>(qbar, kbar, P->d_log_sizes, stats, n, D, P->scale);
  MOD_LAUNCH_CHECK();
  mod_note_launches(2);
  return MOD_OK;
}
