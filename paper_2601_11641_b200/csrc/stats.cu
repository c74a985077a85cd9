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
// v = (s z + ln|I_j|) log2 e; z = A_hi B_hi^T + A_hi B_lo^T + A_lo B_hi^T from the pre-split tiles
// (fp32 accumulation in TMEM).  One CTA per (128-row tile, chunk of 512 columns, head), warp-specialised:
// warp 8 (one thread) streams the chunk's 64-column B sub-tiles by bulk copy through a 3-deep ring and
// issues the MMAs into two TMEM accumulators; warps 0-7 (thread = row, half of a sub-tile's columns) run
// the epilogue of sub-tile i while the MMA of i+1 and the copies of i+2.. proceed.
template <int D>
struct Score2Cfg {
  using ST = SplitTile<D>;
  static constexpr int TN = 64;                            // columns per sub-tile (MMA N)
  static constexpr int CHUNK_COLS = 512;                   // columns per CTA
  static constexpr int NB = 3;                             // B ring depth
  static constexpr int OPA = ST::BYTES;                    // A tile (128 rows, hi + lo)
  static constexpr int SUB = ST::NATOM * 64 * 128;         // one 64-row piece of hi (or lo)
  static constexpr int OPB = 2 * SUB;                      // B sub-tile (64 rows, hi + lo)
  static constexpr int STAGE_BYTES = 128 * TN * 4;
  static constexpr int OFF_A = 0, OFF_B = OPA, OFF_ST = OFF_B + NB * OPB;
  static constexpr int OFF_BAR = OFF_ST + 2 * STAGE_BYTES;
  static constexpr int OFF_LS = OFF_BAR + 128;             // ln|I_j| log2 e of the chunk's columns
  static constexpr int SMEM = OFF_LS + CHUNK_COLS * 4;     // 226 KB at D = 128
  static constexpr int THREADS = 288;
  static constexpr uint32_t IDESC = idesc_bf16_f32(128, TN, false, false);
};

template <int D, bool WRITE>
__global__ void __launch_bounds__(Score2Cfg<D>::THREADS, 1) score_kernel(
    const unsigned char* __restrict__ qs, const unsigned char* __restrict__ ks, const float* __restrict__ log_sizes,
    float* __restrict__ W, float2* __restrict__ part, int n, int T, int NCH, float scale) {
  using C = Score2Cfg<D>;
  using ST = SplitTile<D>;
  extern __shared__ __align__(1024) unsigned char smem[];
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023u) != 0) __trap();   // SWIZZLE_128B operands need 1024B alignment
  uint64_t* a_full = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* b_full = a_full + 1;          // [NB]
  uint64_t* b_empty = b_full + C::NB;     // [NB]  (MMA commit: the sub-tile's MMAs have read the buffer)
  uint64_t* acc_full = b_empty + C::NB;   // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2]   (8 epilogue warps have read the accumulator)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int rt = blockIdx.x, ch = blockIdx.y;
  const size_t bh = blockIdx.z;
  const int c0 = ch * C::CHUNK_COLS;
  const int nt = min(C::CHUNK_COLS / C::TN, (n - c0 + C::TN - 1) / C::TN);   // sub-tiles of this chunk
  const float L2E = 1.4426950408889634f;
  const float sl2 = scale * L2E;
  float* ls2 = reinterpret_cast<float*>(smem + C::OFF_LS);   // -inf past n
  for (int e = threadIdx.x; e < C::CHUNK_COLS; e += blockDim.x) {
    const int c = c0 + e;
    ls2[e] = c < n ? log_sizes[c] * L2E : -INFINITY;
  }
  if (threadIdx.x == 0) {
    mbar_init(a_full, 1);
    for (int i = 0; i < C::NB; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 8);
    }
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ------------------------------------------------------------ bulk copies + MMA issue (one thread)
    if (lane == 0) {
      const unsigned char* A = qs + (bh * T + rt) * (size_t)C::OPA;
      auto load_b = [&](int i) {
        const int sb = i % C::NB;
        const int col = c0 + i * C::TN;                       // first column: rows of k-bar tile col / 128
        const unsigned char* tile = ks + (bh * T + col / 128) * (size_t)ST::BYTES + (col % 128) * 128;
        unsigned char* dst = smem + C::OFF_B + sb * C::OPB;
        mbar_arrive_expect_tx(&b_full[sb], C::OPB);
#pragma unroll
        for (int hl = 0; hl < 2; ++hl)
#pragma unroll
          for (int a = 0; a < ST::NATOM; ++a)
            bulk_load(dst + hl * C::SUB + a * 64 * 128, tile + hl * ST::HALF + a * ST::ATOM, 64 * 128, &b_full[sb]);
      };
      mbar_arrive_expect_tx(a_full, C::OPA);
      bulk_load(smem + C::OFF_A, A, C::OPA, a_full);
      for (int i = 0; i < C::NB && i < nt; ++i) load_b(i);
      mbar_wait(a_full, 0);
      const uint32_t ah = smem_u32(smem + C::OFF_A), al = ah + ST::HALF;
      for (int i = 0; i < nt; ++i) {
        const int sb = i % C::NB, s = i & 1;
        mbar_wait(&b_full[sb], (i / C::NB) & 1);
        if (i >= 2) mbar_wait(&acc_empty[s], ((i >> 1) - 1) & 1);   // epilogue of sub-tile i-2 read acc s
        tc_fence_after();
        const uint32_t bhs = smem_u32(smem + C::OFF_B + sb * C::OPB), bls = bhs + C::SUB;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t ka = (kk / 4) * ST::ATOM + (kk % 4) * 32, kb = (kk / 4) * (64 * 128) + (kk % 4) * 32;
          const uint64_t dah = smem_desc_sw128(ah + ka, 16, 1024), dal = smem_desc_sw128(al + ka, 16, 1024);
          const uint64_t dbh = smem_desc_sw128(bhs + kb, 16, 1024), dbl = smem_desc_sw128(bls + kb, 16, 1024);
          const uint32_t d = tmem + s * C::TN;
          mma_ss(d, dah, dbh, C::IDESC, kk > 0 ? 1u : 0u);
          mma_ss(d, dah, dbl, C::IDESC, 1u);
          mma_ss(d, dal, dbh, C::IDESC, 1u);
        }
        mma_commit(&acc_full[s]);
        mma_commit(&b_empty[sb]);
        if (i >= 1 && i - 1 + C::NB < nt) {   // refill the buffer sub-tile i-1 used (its MMAs precede these)
          mbar_wait(&b_empty[(i - 1) % C::NB], ((i - 1) / C::NB) & 1);
          load_b(i - 1 + C::NB);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue: thread = (row, column half)
    const int row = (warp & 3) * 32 + lane;
    const int half = warp >> 2;             // columns [32 half, +32) of each 64-column sub-tile
    const int grow = rt * 128 + row;
    float m_row = -INFINITY, l_row = 0.f;
    if (WRITE && grow < n) {   // final (m, l) of the row: its chunk partials in chunk order
      const float2* pr = part + (bh * n + grow) * NCH;
      for (int c = 0; c < NCH; ++c) m_row = fmaxf(m_row, pr[c].x);
      for (int c = 0; c < NCH; ++c)
        if (pr[c].x > -INFINITY) l_row += pr[c].y * ex2(pr[c].x - m_row);
    }
    const float inv_l = 1.0f / l_row;
    float m_part = -INFINITY, l_part = 0.f;
    for (int i = 0; i < nt; ++i) {
      const int s = i & 1;
      mbar_wait(&acc_full[s], (i >> 1) & 1);
      tc_fence_after();
      uint32_t z[32];
      tmem_ld32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + s * C::TN + half * 32, z);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[s]);
      float v[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] = fmaf(__uint_as_float(z[e]), sl2, ls2[i * C::TN + half * 32 + e]);
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
        float* stage = reinterpret_cast<float*>(smem + C::OFF_ST + s * C::STAGE_BYTES);
        // float4 chunk cq (0..15) of row r at chunk (cq ^ (r & 15)): spread banks for both access orders
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int cq = half * 8 + u;
          float4 w4;
          w4.x = ex2(v[4 * u] - m_row) * inv_l;
          w4.y = ex2(v[4 * u + 1] - m_row) * inv_l;
          w4.z = ex2(v[4 * u + 2] - m_row) * inv_l;
          w4.w = ex2(v[4 * u + 3] - m_row) * inv_l;
          reinterpret_cast<float4*>(stage)[row * 16 + (cq ^ (row & 15))] = w4;
        }
        named_bar_sync(1, 256);
        const int cb = c0 + i * C::TN, valid = min(C::TN, n - cb);
        for (int r = warp; r < 128 && rt * 128 + r < n; r += 8) {
          float* dst = W + (bh * n + rt * 128 + r) * (size_t)n + cb;
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int c = k * 32 + lane;
            if (c < valid) dst[c] = stage[r * 64 + (((c >> 2) ^ (r & 15)) << 2) + (c & 3)];
          }
        }
      }
    }
    if (!WRITE) {   // the two column halves of each row (warps w and w + 4), combined in a fixed order
      float2* xr = reinterpret_cast<float2*>(smem + C::OFF_ST);
      if (half == 1) xr[row] = make_float2(m_part, l_part);
      named_bar_sync(1, 256);
      if (half == 0 && grow < n) {
        const float2 o = xr[row];
        const float m = fmaxf(m_part, o.x);
        const float l = (m_part > -INFINITY ? l_part * ex2(m_part - m) : 0.f) + (o.x > -INFINITY ? o.y * ex2(o.x - m) : 0.f);
        part[(bh * n + grow) * NCH + ch] = make_float2(m, l);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
}

}  // namespace

extern "C" mod_status mod_collect_block_stats(mod_plan P, const void* q, const void* k, float* stats, void* ws,
                                              void* stream) {
  MOD_NVTX("mod_collect_block_stats");
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  MOD_REQUIRE(q && k && stats && ws, MOD_ERR_USAGE, "mod_collect_block_stats: q, k, stats, ws must be non-NULL");
  const int BH = P->L.batch * P->L.heads, n = P->n, D = P->L.head_dim;
  const int T = (n + 127) / 128, NCH = (n + Score2Cfg<128>::CHUNK_COLS - 1) / Score2Cfg<128>::CHUNK_COLS;
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
    score_kernel<DD, false><<<sg, C::THREADS, C::SMEM, s>>>(qs, ks, P->d_log_sizes, stats, part, n, T, NCH, P->scale);
    MOD_LAUNCH_CHECK();
    score_kernel<DD, true><<<sg, C::THREADS, C::SMEM, s>>>(qs, ks, P->d_log_sizes, stats, part, n, T, NCH, P->scale);
    MOD_LAUNCH_CHECK();
    return MOD_OK;
  };
  st = D == 128 ? run(std::integral_constant<int, 128>{}) : run(std::integral_constant<int, 64>{});
  if (st != MOD_OK) return st;
  mod_note_launches(4);
  return MOD_OK;
}
