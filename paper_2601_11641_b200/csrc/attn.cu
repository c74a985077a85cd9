// attn.cu -- K4 mod_block_sparse_attn_fwd: block-sparse FlashAttention forward for sm_100a.
//
// What it computes (§3 Eq. 1 P:110-115 with the block mask of §5.3 upsampled to tokens,
// Alg. 1): for token p of query block i,
//     O_p = sum_{q in K(i)} softmax_q(s Q_p . K_q) V_q,   K(i) = U_{j in list(i)} I_j,
//     lse_p = ln sum_{q in K(i)} exp(s Q_p . K_q);  empty list -> O = 0, lse = -inf (reading Z15).
// The paper's sparse stage calls SageAttention; the index list replaces the token mask so
// that skipped blocks cost nothing (§5.4 P:460 "block-wise ... block size of 128").
//
// Design (one CTA per (b, h, query block); 320 threads, warp-specialised):
//   warp 0      TMA producer: Q tile once, then K_j / V_j tiles gathered BY INDEX from the CSR
//               list into a 2-stage shared-memory ring (128B-swizzled boxes, 3D tensor maps so
//               keys >= N are zero-filled per head).
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer:
//                  S_j = Q K_j^T       (SS: A = Q smem K-major, B = K_j smem K-major) -> TMEM S[j%2]
//                  O  += P_j V_j       (TS: A = P_j bf16 in TMEM over S[j%2], B = V_j smem MN-major)
//               issue order S_0, S_1, PV_0, S_2, PV_1, ... so S_{j+1} and PV_{j-1} overlap softmax j.
//   warps 2..9  softmax: two threads per query row (column halves); tcgen05.ld of the S row, online softmax in the
//               log2 domain (ex2.approx), bf16 P written back into TMEM (tcgen05.st), lazy O
//               rescale only when the running max grows by > 8 (exact: O and l share the
//               reference max), epilogue O / l -> bf16 and lse.
// TMEM: S[0] cols [0,BN), S[1] [BN,2BN), O [2BN,2BN+D), l [2BN+D, +16); 512 (or 256) columns.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

using namespace sm100;

namespace {

template <int D, int BN>
struct AttnCfg {
  static constexpr int BM = 128;                      // query rows per tile (tcgen05 M)
  static constexpr int STAGES = 3;                    // K ring
  static constexpr int VSTAGES = 2;                   // V ring
  static constexpr int Q_BOX = BM * 128;              // bytes of one 64-column box of Q
  static constexpr int KV_BOX = BN * 128;             // bytes of one 64-column box of K or V
  static constexpr int NATOM = D / 64;                // 128B swizzle atoms along D
  static constexpr int Q_BYTES = Q_BOX * NATOM;
  static constexpr int KV_BYTES = KV_BOX * NATOM;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + STAGES * KV_BYTES;
  static constexpr int OFF_ONES = OFF_V + VSTAGES * KV_BYTES;       // all-ones B operand (16 x BN bf16)
  static constexpr int ONES_BYTES = 16 * BN * 2;
  static constexpr int OFF_BAR = OFF_ONES + ONES_BYTES;
  static constexpr int NUM_BARS = 1 + 2 * STAGES + 2 * VSTAGES + 2 + 2 + 1;
  static constexpr int OFF_RED = OFF_BAR + NUM_BARS * 8 + 16;      // softmax max exchange [2][2][128] f32
  static constexpr int SMEM = OFF_RED + 2 * 2 * 128 * 4;
  // TMEM columns: S[0] | S[1] | O | l (row sums of the bf16 P, accumulated by the tensor core)
  static constexpr int TMEM_S0 = 0, TMEM_S1 = BN, TMEM_O = 2 * BN, TMEM_L = 2 * BN + D;
  static constexpr uint32_t TMEM_COLS = (2 * BN + D + 16) <= 256 ? 256 : 512;
  static constexpr uint32_t IDESC_S = idesc_bf16_f32(BM, BN, false, false);
  static constexpr uint32_t IDESC_O = idesc_bf16_f32(BM, D, false, true);
  static constexpr uint32_t IDESC_L = idesc_bf16_f32(BM, 16, false, false);
  static constexpr int THREADS = 320;
};

template <int D, int BN>
__global__ void __launch_bounds__(320, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const int* __restrict__ row_ptr,
                    const int* __restrict__ col_idx, __nv_bfloat16* __restrict__ out, float* __restrict__ lse,
                    int N, int n, int block, float scale_log2, int dbg) {
  using C = AttnCfg<D, BN>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw;   // 1024-aligned (no static shared memory; checked below)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + C::STAGES;
  uint64_t* v_full = k_empty + C::STAGES;
  uint64_t* v_empty = v_full + C::VSTAGES;
  uint64_t* s_full = v_empty + C::VSTAGES;
  uint64_t* p_full = s_full + 2;
  uint64_t* o_done = p_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023u) != 0) __trap();   // SWIZZLE_128B needs 1024B alignment
  const int item = blockIdx.x;
  const int bh = item / n, qi = item % n;
  const int beg = row_ptr[(size_t)bh * (n + 1) + qi];
  const int L = row_ptr[(size_t)bh * (n + 1) + qi + 1] - beg;
  const int* cols = col_idx + (size_t)bh * n * n + beg;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < C::VSTAGES; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 256);
    }
    mbar_init(o_done, 1);
    fence_mbar_init();
  }
  {  // constant all-ones B operand for the row-sum MMA (swizzle-invariant: every element is 1.0)
    uint32_t* ones = reinterpret_cast<uint32_t*>(smem + C::OFF_ONES);
    for (int e = threadIdx.x; e < C::ONES_BYTES / 4; e += blockDim.x) ones[e] = 0x3F803F80u;
    fence_async_shared();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && L > 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
      unsigned char* sq = smem + C::OFF_Q;
      mbar_arrive_expect_tx(q_full, C::Q_BYTES);
#pragma unroll
      for (int a = 0; a < C::NATOM; ++a) tma_load_3d(sq + a * C::Q_BOX, &tm_q, q_full, a * 64, qi * block, bh, pol_q);
      auto load_k = [&](int j) {
        const int s = j % C::STAGES;
        mbar_wait(&k_empty[s], ((j / C::STAGES) & 1) ^ 1);
        unsigned char* dst = smem + C::OFF_K + s * C::KV_BYTES;
        if (dbg == 2) { mbar_arrive(&k_full[s]); return; }
        mbar_arrive_expect_tx(&k_full[s], C::KV_BYTES);
        const int row = cols[j] * block;
#pragma unroll
        for (int a = 0; a < C::NATOM; ++a) tma_load_3d(dst + a * C::KV_BOX, &tm_k, &k_full[s], a * 64, row, bh, pol_kv);
      };
      auto load_v = [&](int j) {
        const int s = j % C::VSTAGES;
        mbar_wait(&v_empty[s], ((j / C::VSTAGES) & 1) ^ 1);
        unsigned char* dst = smem + C::OFF_V + s * C::KV_BYTES;
        if (dbg == 2) { mbar_arrive(&v_full[s]); return; }
        mbar_arrive_expect_tx(&v_full[s], C::KV_BYTES);
        const int row = cols[j] * block;
#pragma unroll
        for (int a = 0; a < C::NATOM; ++a) tma_load_3d(dst + a * C::KV_BOX, &tm_v, &v_full[s], a * 64, row, bh, pol_kv);
      };
      // demand order of the MMA warp: K0, K1, V0, K2, V1, ...
      load_k(0);
      for (int j = 0; j < L; ++j) {
        if (j + 1 < L) load_k(j + 1);
        load_v(j);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && L > 0) {
      const uint32_t sq = smem_u32(smem + C::OFF_Q);
      mbar_wait(q_full, 0);
      tc_fence_after();
      for (int j = 0; j <= L; ++j) {
        if (j < L) {
          const int s = j % C::STAGES;
          mbar_wait(&k_full[s], (j / C::STAGES) & 1);
          tc_fence_after();
          const uint32_t sk = smem_u32(smem + C::OFF_K + s * C::KV_BYTES);
          const uint32_t d_s = tmem + ((j & 1) ? C::TMEM_S1 : C::TMEM_S0);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk / 4) * 0 + (kk % 4) * 32;
            const uint64_t ad = smem_desc_sw128(sq + (kk / 4) * C::Q_BOX + off, 16, 1024);
            const uint64_t bd = smem_desc_sw128(sk + (kk / 4) * C::KV_BOX + off, 16, 1024);
            mma_ss(d_s, ad, bd, C::IDESC_S, kk > 0 ? 1u : 0u);
          }
          mma_commit(&k_empty[s]);
          mma_commit(&s_full[j & 1]);
        }
        if (j >= 1) {
          const int jj = j - 1;
          const int s = jj % C::VSTAGES;
          mbar_wait(&p_full[jj & 1], (jj >> 1) & 1);
          mbar_wait(&v_full[s], (jj / C::VSTAGES) & 1);
          tc_fence_after();
          const uint32_t sv = smem_u32(smem + C::OFF_V + s * C::KV_BYTES);
          const uint32_t p_t = tmem + ((jj & 1) ? C::TMEM_S1 : C::TMEM_S0);
#pragma unroll
          const uint32_t s_ones = smem_u32(smem + C::OFF_ONES);
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk) {
            // B = V_j: N = D (MN-major, 64-column atoms LBO = KV_BOX apart), K = 16 keys = 2048 bytes
            const uint64_t bd = smem_desc_sw128(sv + kk * 2048, C::KV_BOX, 1024);
            mma_ts(tmem + C::TMEM_O, p_t + kk * 8, bd, C::IDESC_O, (jj > 0 || kk > 0) ? 1u : 0u);
            // l += P_j 1  (N = 16 all-ones columns, K-major)
            const uint64_t ld = smem_desc_sw128(s_ones + (kk / 4) * 2048 + (kk % 4) * 32, 16, 1024);
            mma_ts(tmem + C::TMEM_L, p_t + kk * 8, ld, C::IDESC_L, (jj > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&v_empty[s]);
          mma_commit(o_done);
        }
      }
    }
  } else if (warp >= 2) {
    // ------------------------------------------------------------ softmax / epilogue (8 warps)
    // Two threads per query row: warps w and w+4 read the same TMEM lane quarter and split the BN
    // score columns (and, in the epilogue, the D output columns) in halves, so every SM
    // sub-partition runs two independent softmax warps (latency hiding).  Per element: one FFMA
    // (s*log2e/sqrt(d) - m) and half a MUFU: pairs are packed to bf16x2 and exponentiated with
    // ex2.approx.bf16x2, which yields P in the packed format the PV MMA consumes.  The row sum l is
    // not accumulated here: the tensor core computes l += P*1 next to O += P*V, so O and l see
    // exactly the same rounded P.
    constexpr int CPT = BN / 2;                // score columns per thread
    constexpr int OPT = D / 2;                 // output columns per thread (epilogue)
    auto red_max = reinterpret_cast<float(*)[2][128]>(smem + C::OFF_RED);   // [iter parity][half][row]
    const int half = (warp - 2) >> 2;
    const int quarter = warp & 3;              // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;       // query row within the tile
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const int q_row0 = qi * block;
    const int q_rows = min(block, N - q_row0);
    float m_run = -INFINITY;
    for (int j = 0; j < L; ++j) {
      const int b = j & 1;
      const uint32_t t_s = tmem + lane_off + (b ? C::TMEM_S1 : C::TMEM_S0);
      mbar_wait(&s_full[b], (j >> 1) & 1);
      tc_fence_after();
      uint32_t sr[CPT];
#pragma unroll
      for (int c = 0; c < CPT / 32; ++c)
        tmem_ld32(t_s + half * CPT + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
      tmem_ld_wait();
      float* s = reinterpret_cast<float*>(sr);
      const int kv_valid = N - cols[j] * block - half * CPT;  // valid keys among this thread's columns
      if (kv_valid < CPT) {
#pragma unroll
        for (int c = 0; c < CPT; ++c)
          if (c >= kv_valid) s[c] = -INFINITY;
      }
      float mxv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mxv[u] = s[u];
#pragma unroll
      for (int c = 8; c < CPT; c += 8)
#pragma unroll
        for (int u = 0; u < 8; ++u) mxv[u] = fmaxf(mxv[u], s[c + u]);
      float mx = fmaxf(fmaxf(fmaxf(mxv[0], mxv[1]), fmaxf(mxv[2], mxv[3])),
                       fmaxf(fmaxf(mxv[4], mxv[5]), fmaxf(mxv[6], mxv[7])));
      red_max[b][half][row] = mx;
      named_bar_sync(1 + quarter, 64);
      mx = fmaxf(mx, red_max[b][half ^ 1][row]);
      const float m_new = fmaxf(m_run, mx * scale_log2);
      const bool rescale = (m_new - m_run) > 8.0f;   // also true on the first block (m_run = -inf)
      const float m_use = rescale ? m_new : m_run;
      const float alpha = rescale ? ex2(m_run - m_new) : 1.0f;
      m_run = m_use;
      uint32_t pk[CPT / 2];
#pragma unroll
      for (int c = 0; c < CPT; c += 2)
        pk[c / 2] = ex2_bf16x2(pack_bf16(fmaf(s[c], scale_log2, -m_use), fmaf(s[c + 1], scale_log2, -m_use)));
      if constexpr (CPT / 2 == 32) tmem_st32(t_s + half * (CPT / 2), *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
      else tmem_st16(t_s + half * (CPT / 2), *reinterpret_cast<uint32_t(*)[16]>(&pk[0]));
      if (j >= 1) {
        mbar_wait(o_done, (j - 1) & 1);   // PV_{j-1} finished writing O and l
        tc_fence_after();
        if (__any_sync(0xffffffffu, rescale)) {
          const uint32_t t_o = tmem + lane_off + C::TMEM_O + half * OPT;
#pragma unroll
          for (int c = 0; c < OPT / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(t_o + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st32(t_o + c * 32, o);
          }
          if (half == 0) {
            uint32_t lv = tmem_ld1(tmem + lane_off + C::TMEM_L);
            tmem_ld_wait();
            tmem_st1(tmem + lane_off + C::TMEM_L, __float_as_uint(__uint_as_float(lv) * alpha));
          }
        }
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[b]);
    }
    // epilogue: O / l -> bf16 (each thread of the pair writes half of the row), lse
    const bool valid = row < q_rows;
    const size_t grow = (size_t)bh * N + q_row0 + row;
    if (L > 0) {
      mbar_wait(o_done, (L - 1) & 1);
      tc_fence_after();
      const float l = __uint_as_float(tmem_ld1(tmem + lane_off + C::TMEM_L));
      tmem_ld_wait();
      const float inv_l = 1.0f / l;
      const uint32_t t_o = tmem + lane_off + C::TMEM_O + half * OPT;
#pragma unroll
      for (int c = 0; c < OPT / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(t_o + c * 32, o);
        tmem_ld_wait();
        uint32_t pkd[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
          pkd[e] = pack_bf16(__uint_as_float(o[2 * e]) * inv_l, __uint_as_float(o[2 * e + 1]) * inv_l);
        if (valid) {
          int4* dst = reinterpret_cast<int4*>(out + grow * D + half * OPT + c * 32);
#pragma unroll
          for (int e = 0; e < 4; ++e) dst[e] = make_int4(pkd[4 * e], pkd[4 * e + 1], pkd[4 * e + 2], pkd[4 * e + 3]);
        }
      }
      if (valid && lse && half == 0) lse[grow] = (m_run + __log2f(l)) * 0.69314718055994531f;
    } else if (valid) {
      int4* dst = reinterpret_cast<int4*>(out + grow * D + half * OPT);
#pragma unroll
      for (int e = 0; e < OPT / 8; ++e) dst[e] = make_int4(0, 0, 0, 0);
      if (lse && half == 0) lse[grow] = -INFINITY;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3D map over [BH, N, D] bf16 (dims innermost first), box {64, rows, 1}, 128B swizzle.
mod_status make_map(CUtensorMap* m, const void* base, int BH, int N, int D, int rows) {
  auto enc = get_encode();
  MOD_REQUIRE(enc, MOD_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled driver entry point unavailable");
  MOD_REQUIRE(((uintptr_t)base & 127) == 0, MOD_ERR_INPUT, "Q/K/V pointers must be 128-byte aligned");
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)N, (cuuint64_t)BH};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)N * D * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MOD_REQUIRE(r == CUDA_SUCCESS, MOD_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return MOD_OK;
}

template <int D, int BN>
mod_status launch(mod_plan P, const void* q, const void* k, const void* v, const int* row_ptr, const int* col_idx,
                  void* o, float* lse, cudaStream_t s) {
  using C = AttnCfg<D, BN>;
  const int BH = P->L.batch * P->L.heads;
  CUtensorMap tq, tk, tv;
  mod_status st;
  if ((st = make_map(&tq, q, BH, P->N, D, C::BM)) != MOD_OK) return st;
  if ((st = make_map(&tk, k, BH, P->N, D, BN)) != MOD_OK) return st;
  if ((st = make_map(&tv, v, BH, P->N, D, BN)) != MOD_OK) return st;
  auto kern = attn_fwd_kernel<D, BN>;
  MOD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  const float scale_log2 = P->scale * 1.4426950408889634f;
  static const int dbg = getenv("MOD_ATTN_DEBUG") ? atoi(getenv("MOD_ATTN_DEBUG")) : 0;   // bring-up only
  kern<<<BH * P->n, C::THREADS, C::SMEM, s>>>(tq, tk, tv, row_ptr, col_idx, (__nv_bfloat16*)o, lse, P->N, P->n,
                                              P->L.block, scale_log2, dbg);
  MOD_LAUNCH_CHECK();
  return MOD_OK;
}

}  // namespace

extern "C" mod_status mod_block_sparse_attn_fwd(mod_plan P, const void* q, const void* k, const void* v,
                                                const int32_t* row_ptr, const int32_t* col_idx, void* o, float* lse,
                                                void* ws, void* stream) {
  (void)ws;
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  MOD_REQUIRE(q && k && v && row_ptr && col_idx && o, MOD_ERR_USAGE,
              "mod_block_sparse_attn_fwd: q, k, v, row_ptr, col_idx, o must be non-NULL");
  MOD_REQUIRE(((uintptr_t)o & 15) == 0, MOD_ERR_INPUT, "o must be 16-byte aligned");
  cudaStream_t s = as_stream(stream);
  const int D = P->L.head_dim, BN = P->L.block;
  if (D == 128 && BN == 128) st = launch<128, 128>(P, q, k, v, row_ptr, col_idx, o, lse, s);
  else if (D == 64 && BN == 128) st = launch<64, 128>(P, q, k, v, row_ptr, col_idx, o, lse, s);
  else if (D == 128 && BN == 64) st = launch<128, 64>(P, q, k, v, row_ptr, col_idx, o, lse, s);
  else st = launch<64, 64>(P, q, k, v, row_ptr, col_idx, o, lse, s);
  if (st == MOD_OK) mod_note_launches(1);
  return st;
}
