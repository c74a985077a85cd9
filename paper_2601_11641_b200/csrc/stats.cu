// stats.cu -- K1 mod_collect_block_stats: pooled block score + row-softmax block mass.
//
// BASELINE.json north_star (1): "a mean-pooled QK^T block-score plus row-softmax block-mass kernel
// (warp-shuffle reductions, vectorised 128-bit loads)".  The paper's own statistic is Eq. 2
// (P:204-206), which needs the full post-softmax map; the pooled surrogate is reading Z1:
//   qbar_i = (1/|I_i|) sum_{p in I_i} Q_p,  kbar_j likewise          (fp32 accumulation)
//   z_ij   = s * qbar_i . kbar_j                                      (s = 1/sqrt(D))
//   W_ij   = |I_j| e^{z_ij} / sum_j' |I_j'| e^{z_ij'}                 (block mass; ragged blocks Z16)
//
// Four kernels:
//   pool_kernel   -- HBM-bound: streams Q and K once (2*B*H*N*D*2 bytes) with 128-bit non-allocating
//                    loads; one CTA per (tensor, head, block); fixed-order reduction (deterministic);
//   split_kernel  -- the bf16 (hi, lo) split of the means into pre-swizzled 128-row operand tiles;
//   score_kernel<D, false> / <D, true> -- z = qbar kbar^T on tcgen05 (3 bf16 MMAs per K step from the
//                    split tiles), pass 0 the rows' (max, sum) partials per column chunk, pass 1 the
//                    normalised W written once (the MMA is recomputed instead of storing logits).
#include "common.cuh"
#include "sm100.cuh"

using namespace sm100;

namespace {

// Pre-split operand tiles of the score MMA, written by pool_kernel: for each 128-row tile t of the n
// block means of a head, [hi | lo][D/64 atoms][128 rows x 128 bytes] bf16 in exactly the 128B-swizzled
// K-major shared-memory layout (row r, 16-byte chunk c of an atom at r*128 + ((c ^ (r & 7)) << 4)), so a
// CTA of the score kernel fetches an operand tile with ONE contiguous bulk copy.  Rows >= n are zero.
template <int D>
struct SplitTile {
  static constexpr int NATOM = D / 64, ATOM = 128 * 128;
  static constexpr int HALF = NATOM * ATOM;        // bytes of hi (or lo) of one tile
  static constexpr int BYTES = 2 * HALF;           // hi + lo
  __device__ static size_t offset(int row, int c16) {   // byte offset inside a tile's hi half
    const int r = row & 127;
    return (size_t)(c16 >> 3) * ATOM + r * 128 + (((c16 & 7) ^ (r & 7)) << 4);
  }
};

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

// fp32 means [BH, n, D] -> the pre-split tiles (SplitTile): one thread per 16-byte chunk of a tile row,
// hi = bf16(x), lo = bf16(x - hi) (the dropped lo*lo product is < 2^-16 relative); rows >= n are zero.
template <int D>
__global__ void __launch_bounds__(256) split_kernel(const float* __restrict__ qbar, const float* __restrict__ kbar,
                                                     unsigned char* __restrict__ qs, unsigned char* __restrict__ ks,
                                                     int n, int T, int BH) {
  using ST = SplitTile<D>;
  constexpr int CPR = D / 8;
  const size_t per = (size_t)BH * T * 128 * CPR;
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 2 * per) return;
  const bool isk = e >= per;
  const size_t f = isk ? e - per : e;
  const int c16 = (int)(f % CPR);
  const size_t rr = f / CPR;                   // bh * T*128 + row
  const int row = (int)(rr % ((size_t)T * 128));
  const size_t bh = rr / ((size_t)T * 128);
  float x[8];
  if (row < n) {
    const float4* src = reinterpret_cast<const float4*>((isk ? kbar : qbar) + (bh * n + row) * D + 8 * c16);
    const float4 a = __ldg(src), b = __ldg(src + 1);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
  } else {
#pragma unroll
    for (int w = 0; w < 8; ++w) x[w] = 0.f;
  }
  uint32_t h[4], l[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const __nv_bfloat16 h0 = __float2bfloat16_rn(x[2 * w]), h1 = __float2bfloat16_rn(x[2 * w + 1]);
    const __nv_bfloat16 l0 = __float2bfloat16_rn(x[2 * w] - __bfloat162float(h0));
    const __nv_bfloat16 l1 = __float2bfloat16_rn(x[2 * w + 1] - __bfloat162float(h1));
    h[w] = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
    l[w] = (uint32_t)__bfloat16_as_ushort(l0) | ((uint32_t)__bfloat16_as_ushort(l1) << 16);
  }
  unsigned char* tile = (isk ? ks : qs) + (bh * T + (row >> 7)) * (size_t)ST::BYTES;
  const size_t off = ST::offset(row, c16);
  *reinterpret_cast<uint4*>(tile + off) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(tile + ST::HALF + off) = make_uint4(l[0], l[1], l[2], l[3]);
}

// z = s * qbar kbar^T on the tensor cores (north_star: "tensor cores are used ... in the QK^T of the
// pooled scores"), the log-size bias and the row softmax, in two passes that recompute the MMA instead
// of storing logits (the MMA is cheap; the n x n map is written to HBM exactly once):
//   pass 0 (score_kernel<D, false>): per (row tile, column chunk) the rows' online (max, sum 2^(v - max))
//          over the chunk's columns -> part[bh][row][chunk];
//   pass 1 (score_kernel<D, true>):  the row's chunk partials combined in a fixed order, the logits
//          recomputed and W = 2^(v - m) / l written through a swizzled shared-memory stage as coalesced
//          row segments.
// v = (s z + ln|I_j|) log2 e; z = A_hi B_hi^T + A_hi B_lo^T + A_lo B_hi^T from the pre-split tiles of
// pool_kernel (one bulk copy per operand tile), fp32 accumulation in TMEM.  One CTA per (row tile of 128
// blocks, chunk of up to 4 column tiles of 128, head); thread = row; the next column tile's MMA runs
// while the current one's epilogue reads TMEM (two accumulators), and its B tile streams in meanwhile.
template <int D>
struct Score2Cfg {
  using ST = SplitTile<D>;
  static constexpr int CHUNK = 4;                          // column tiles per CTA
  static constexpr int OP = ST::BYTES;                     // one operand tile (hi + lo)
  static constexpr int OFF_A = 0, OFF_B = OP;              // A, then the B ring (2 tiles)
  static constexpr int STAGE_BYTES = 128 * 128 * 4;        // W staging of one 128 x 128 tile
  static constexpr bool STAGE_IN_B = OP >= STAGE_BYTES;    // D = 128: reuse the consumed B tile
  static constexpr int OFF_ST = OFF_B + 2 * OP;            // D = 64: dedicated staging
  static constexpr int OFF_BAR = OFF_ST + (STAGE_IN_B ? 0 : STAGE_BYTES);   // one stage: written, synced, stored
  static constexpr int SMEM = OFF_BAR + 64 + 1024;         // + alignment slack
  static constexpr uint32_t IDESC = idesc_bf16_f32(128, 128, false, false);
};

template <int D, bool WRITE>
__global__ void __launch_bounds__(256, 1) score_kernel(const unsigned char* __restrict__ qs,
                                                       const unsigned char* __restrict__ ks,
                                                       const float* __restrict__ log_sizes, float* __restrict__ W,
                                                       float2* __restrict__ part, int n, int T, int NCH,
                                                       float scale) {
  using C = Score2Cfg<D>;
  using ST = SplitTile<D>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar_a = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* bar_b = bar_a + 1;      // [2]
  uint64_t* done = bar_a + 3;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_a + 5);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int rt = blockIdx.x, ch = blockIdx.y;
  const size_t bh = blockIdx.z;
  const int ct0 = ch * C::CHUNK, nt = min(C::CHUNK, T - ct0);
  const unsigned char* A = qs + (bh * T + rt) * (size_t)C::OP;
  const unsigned char* Bt = ks + bh * T * (size_t)C::OP;
  const float L2E = 1.4426950408889634f;
  const float sl2 = scale * L2E;
  const int row = (warp & 3) * 32 + lane;     // tile row = TMEM lane (warp w reads lane quarter w % 4)
  const int half = warp >> 2;                 // column half [64 half, +64) of each tile this thread handles
  const int grow = rt * 128 + row;
  __shared__ float ls2[C::CHUNK * 128];       // ln|I_j| log2 e of the chunk's columns (-inf past n)
  for (int e = threadIdx.x; e < C::CHUNK * 128; e += blockDim.x) {
    const int c = ct0 * 128 + e;
    ls2[e] = c < n ? log_sizes[c] * L2E : -INFINITY;
  }
  if (threadIdx.x == 0) {
    mbar_init(bar_a, 1);
    mbar_init(&bar_b[0], 1);
    mbar_init(&bar_b[1], 1);
    mbar_init(&done[0], 1);
    mbar_init(&done[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // final (m, l) of the row (pass 1): its chunk partials in chunk order
  float m_row = -INFINITY, l_row = 0.f;
  if (WRITE && grow < n) {
    const float2* pr = part + (bh * n + grow) * NCH;
    for (int c = 0; c < NCH; ++c) m_row = fmaxf(m_row, pr[c].x);
    for (int c = 0; c < NCH; ++c)
      if (pr[c].x > -INFINITY) l_row += pr[c].y * ex2(pr[c].x - m_row);
  }
  const float inv_l = 1.0f / l_row;
  auto load_b = [&](int i) {   // thread 0
    const int s = i & 1;
    mbar_arrive_expect_tx(&bar_b[s], C::OP);
    bulk_load(smem + C::OFF_B + s * C::OP, Bt + (size_t)(ct0 + i) * C::OP, C::OP, &bar_b[s]);
  };
  auto issue = [&](int i) {   // thread 0: z tile i into accumulator i & 1
    const int s = i & 1;
    mbar_wait(&bar_b[s], (i >> 1) & 1);
    tc_fence_after();
    const uint32_t ah = smem_u32(smem + C::OFF_A), al = ah + ST::HALF;
    const uint32_t bhs = smem_u32(smem + C::OFF_B + s * C::OP), bls = bhs + ST::HALF;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const uint32_t ko = (kk / 4) * ST::ATOM + (kk % 4) * 32;
      const uint64_t dah = smem_desc_sw128(ah + ko, 16, 1024), dal = smem_desc_sw128(al + ko, 16, 1024);
      const uint64_t dbh = smem_desc_sw128(bhs + ko, 16, 1024), dbl = smem_desc_sw128(bls + ko, 16, 1024);
      const uint32_t d = tmem + s * 128;
      mma_ss(d, dah, dbh, C::IDESC, kk > 0 ? 1u : 0u);
      mma_ss(d, dah, dbl, C::IDESC, 1u);
      mma_ss(d, dal, dbh, C::IDESC, 1u);
    }
    mma_commit(&done[s]);
  };
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar_a, C::OP);
    bulk_load(smem + C::OFF_A, A, C::OP, bar_a);
    load_b(0);
    if (nt > 1) load_b(1);
    mbar_wait(bar_a, 0);
    issue(0);
  }
  float m_part = -INFINITY, l_part = 0.f;     // pass 0: this row's online (max, sum) over the chunk
  for (int i = 0; i < nt; ++i) {
    const int s = i & 1, ct = ct0 + i;
    if (threadIdx.x == 0 && i + 1 < nt) issue(i + 1);   // next tile's MMA overlaps this epilogue
    mbar_wait(&done[s], (i >> 1) & 1);
    tc_fence_after();
    const int valid = min(128, n - ct * 128);
    float* stage = reinterpret_cast<float*>(smem + (C::STAGE_IN_B ? C::OFF_B + s * C::OP : C::OFF_ST));
#pragma unroll
    for (int k2 = 0; k2 < 2; ++k2) {
      const int k = half * 2 + k2;            // 32-column group of the tile
      uint32_t z[32];
      tmem_ld32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + s * 128 + k * 32, z);
      tmem_ld_wait();
      float v[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] = fmaf(__uint_as_float(z[e]), sl2, ls2[i * 128 + k * 32 + e]);
      if (!WRITE) {
        float mx = v[0];
#pragma unroll
        for (int e = 1; e < 32; ++e) mx = fmaxf(mx, v[e]);
        const float m_new = fmaxf(m_part, mx);
        float sum = 0.f;
#pragma unroll
        for (int e = 0; e < 32; ++e) sum += ex2(v[e] - m_new);
        l_part = (m_part > -INFINITY ? l_part * ex2(m_part - m_new) : 0.f) + sum;
        m_part = m_new;
      } else {
        // W row segment into the stage: float4 chunk cq of row r at chunk (cq ^ (r & 31)) (conflict-free
        // both for this thread-per-row store and the warp-per-row read below)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int cq = k * 8 + u;
          float4 w4;
          w4.x = ex2(v[4 * u] - m_row) * inv_l;
          w4.y = ex2(v[4 * u + 1] - m_row) * inv_l;
          w4.z = ex2(v[4 * u + 2] - m_row) * inv_l;
          w4.w = ex2(v[4 * u + 3] - m_row) * inv_l;
          reinterpret_cast<float4*>(stage)[row * 32 + (cq ^ (row & 31))] = w4;
        }
      }
    }
    tc_fence_before();
    __syncthreads();   // TMEM accumulator s read by everyone; stage s complete; B tile s consumed by MMA i
    if (WRITE) {
      // warp w writes rows w, w + 4, ...: 128 B per instruction along the row
      for (int r = warp; r < 128 && rt * 128 + r < n; r += 8) {
        float* dst = W + (bh * n + rt * 128 + r) * (size_t)n + ct * 128;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int c = k * 32 + lane;
          if (c < valid) dst[c] = stage[r * 128 + (((c >> 2) ^ (r & 31)) << 2) + (c & 3)];
        }
      }
      __syncthreads();   // stage s (the B tile s when STAGE_IN_B) free again
    }
    tc_fence_after();
    if (threadIdx.x == 0 && i + 2 < nt) load_b(i + 2);
  }
  if (!WRITE) {   // the two column halves of each row (warps w and w + 4), combined in a fixed order
    float2* xr = reinterpret_cast<float2*>(ls2);   // reuse: 128 rows x float2 of the upper half
    __syncthreads();
    if (half == 1) xr[row] = make_float2(m_part, l_part);
    __syncthreads();
    if (half == 0 && grow < n) {
      const float2 o = xr[row];
      const float m = fmaxf(m_part, o.x);
      const float l = (m_part > -INFINITY ? l_part * ex2(m_part - m) : 0.f) + (o.x > -INFINITY ? o.y * ex2(o.x - m) : 0.f);
      part[(bh * n + grow) * NCH + ch] = make_float2(m, l);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

}  // namespace

extern "C" mod_status mod_collect_block_stats(mod_plan P, const void* q, const void* k, float* stats, void* ws,
                                              void* stream) {
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  MOD_REQUIRE(q && k && stats && ws, MOD_ERR_USAGE, "mod_collect_block_stats: q, k, stats, ws must be non-NULL");
  const int BH = P->L.batch * P->L.heads, n = P->n, D = P->L.head_dim;
  const int T = (n + 127) / 128, NCH = (T + Score2Cfg<128>::CHUNK - 1) / Score2Cfg<128>::CHUNK;
  float* qbar = reinterpret_cast<float*>(static_cast<char*>(ws) + P->ws_qbar);   // fp32 means [BH, n, D]
  float* kbar = reinterpret_cast<float*>(static_cast<char*>(ws) + P->ws_kbar);
  unsigned char* qs = static_cast<unsigned char*>(ws) + P->ws_qs;                  // pre-split tiles [BH][T][hi|lo]
  unsigned char* ks = static_cast<unsigned char*>(ws) + P->ws_ks;
  cudaStream_t s = as_stream(stream);
  const dim3 pg(n, BH, 2);
  const dim3 sg(T, NCH, BH);
  float2* part = reinterpret_cast<float2*>(static_cast<char*>(ws) + P->ws_part);   // [BH, n, NCH] (free during K1)
  auto run = [&](auto dc) -> mod_status {
    constexpr int DD = decltype(dc)::value;
    using C = Score2Cfg<DD>;
    pool_kernel<DD><<<pg, 256, 0, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k, qbar, kbar, P->N, n, P->L.block);
    MOD_LAUNCH_CHECK();
    const size_t chunks = 2ull * BH * T * 128 * (DD / 8);
    split_kernel<DD><<<(unsigned)((chunks + 255) / 256), 256, 0, s>>>(qbar, kbar, qs, ks, n, T, BH);
    MOD_LAUNCH_CHECK();
    MOD_CUDA(cudaFuncSetAttribute(score_kernel<DD, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    MOD_CUDA(cudaFuncSetAttribute(score_kernel<DD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    score_kernel<DD, false><<<sg, 256, C::SMEM, s>>>(qs, ks, P->d_log_sizes, stats, part, n, T, NCH, P->scale);
    MOD_LAUNCH_CHECK();
    score_kernel<DD, true><<<sg, 256, C::SMEM, s>>>(qs, ks, P->d_log_sizes, stats, part, n, T, NCH, P->scale);
    MOD_LAUNCH_CHECK();
    return MOD_OK;
  };
  st = D == 128 ? run(std::integral_constant<int, 128>{}) : run(std::integral_constant<int, 64>{});
  if (st != MOD_OK) return st;
  mod_note_launches(4);
  return MOD_OK;
}
