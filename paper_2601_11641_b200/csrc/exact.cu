// exact.cu -- mod_collect_exact_sparsity: the paper's own block statistic (§4.1 Eq. 2,
// P:204-206) on the GPU, in informativeness polarity U = -S (reading Z3:
// the paper's Top-K takes the patterns with the SMALLEST fitted S, i.e. the largest fitted -S):
//     S_ij = (1/|I_i||I_j|) #{(p,q) in I_i x I_j : P_pq < eta},   P_pq = exp(s Q_p.K_q - lse_p)
// for every block (i,j) of the CSR list.  lse_p is the log-sum-exp of the attention that produced
// the map: the dense warm-up attention (all-ones list, t = m-1, m; Alg. 1) or the sparse
// attention at a re-estimation step, whose lse is over the unmasked keys only -- exactly Eq. 5's
// A_masked renormalised over the selected blocks (reading Z12).  Both come out of
// mod_block_sparse_attn_fwd.  No exponential is needed:
//     P_pq < eta  <=>  Q_p.K_q < (lse_p + ln eta) / s          (strict, as Eq. 2's indicator)
//
// Design: one CTA per (b, h, query block); warp 0 = TMA (Q once, K_j by index, 2-slot ring),
// warp 1 = single-thread tcgen05.mma issuer of S_j = Q K_j^T into TMEM S[j%2] (fp32),
// warps 2..9 = two counting groups (blocks j = g mod 2): thread = query row, tcgen05.ld of its S row,
// compare-and-count against the row threshold, warp redux + a 4-warp named barrier for the block
// total.  The S buffer is released as soon as the row is in registers.
#include <cudaTypedefs.h>

#include <cmath>

#include "common.cuh"
#include "sm100.cuh"

using namespace sm100;

namespace {

template <int D, int BN>
struct ExCfg {
  static constexpr int BM = 128;
  static constexpr int Q_BOX = BM * 128;
  static constexpr int KV_BOX = BN * 128;
  static constexpr int NATOM = D / 64;
  static constexpr int Q_BYTES = Q_BOX * NATOM;
  static constexpr int KV_BYTES = KV_BOX * NATOM;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_BAR = OFF_K + 2 * KV_BYTES;
  static constexpr int NUM_BARS = 1 + 2 + 2 + 2;   // q_full, k_full[2], s_full[2], s_free[2]
  static constexpr int OFF_RED = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr int SMEM = OFF_RED + 2 * 2 * 4 * 4;   // int red[group][parity][warp]
  static constexpr int TMEM_S0 = 0, TMEM_S1 = BN;
  static constexpr uint32_t TMEM_COLS = 2 * BN <= 128 ? 128 : 256;
  static constexpr uint32_t IDESC_S = idesc_bf16_f32(BM, BN, false, false);
};

template <int D, int BN>
__global__ void __launch_bounds__(320, 1)
    exact_stat_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const float* __restrict__ lse, const int* __restrict__ row_ptr, const int* __restrict__ col_idx,
                      float* __restrict__ U, int N, int n, int block, float inv_scale, float ln_eta) {
  using C = ExCfg<D, BN>;
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* s_full = k_full + 2;
  uint64_t* s_free = s_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_free + 2);
  auto red = reinterpret_cast<int(*)[2][4]>(smem + C::OFF_RED);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023u) != 0) __trap();
  const int item = blockIdx.x;
  const int bh = item / n, qi = item % n;
  const int beg = row_ptr[(size_t)bh * (n + 1) + qi];
  const int L = row_ptr[(size_t)bh * (n + 1) + qi + 1] - beg;
  const int* cols = col_idx + (size_t)bh * n * n + beg;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&k_full[b], 1);
      mbar_init(&s_full[b], 1);
      mbar_init(&s_free[b], 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0 && L > 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      const uint64_t pol_q = policy_evict_first(), pol_k = policy_evict_last();
      mbar_arrive_expect_tx(q_full, C::Q_BYTES);
#pragma unroll
      for (int a = 0; a < C::NATOM; ++a)
        tma_load_3d(smem + C::OFF_Q + a * C::Q_BOX, &tm_q, q_full, a * 64, qi * block, bh, pol_q);
      for (int j = 0; j < L; ++j) {
        const int b = j & 1;
        if (j >= 2) mbar_wait(&s_full[b], ((j - 2) >> 1) & 1);   // S_{j-2} consumed K slot b
        unsigned char* dst = smem + C::OFF_K + b * C::KV_BYTES;
        mbar_arrive_expect_tx(&k_full[b], C::KV_BYTES);
        const int row = cols[j] * block;
#pragma unroll
        for (int a = 0; a < C::NATOM; ++a) tma_load_3d(dst + a * C::KV_BOX, &tm_k, &k_full[b], a * 64, row, bh, pol_k);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && L > 0) {
      const uint32_t sq = smem_u32(smem + C::OFF_Q);
      mbar_wait(q_full, 0);
      tc_fence_after();
      for (int j = 0; j < L; ++j) {
        const int b = j & 1;
        if (j >= 2) mbar_wait(&s_free[b], ((j - 2) >> 1) & 1);    // counters have S_{j-2} in registers
        mbar_wait(&k_full[b], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t sk = smem_u32(smem + C::OFF_K + b * C::KV_BYTES);
        const uint32_t d_s = tmem + (b ? C::TMEM_S1 : C::TMEM_S0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t ad = smem_desc_sw128(sq + (kk / 4) * C::Q_BOX + (kk % 4) * 32, 16, 1024);
          const uint64_t bd = smem_desc_sw128(sk + (kk / 4) * C::KV_BOX + (kk % 4) * 32, 16, 1024);
          mma_ss(d_s, ad, bd, C::IDESC_S, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[b]);
      }
    }
  } else {
    const int g = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t t_s = tmem + ((uint32_t)(quarter * 32) << 16) + (g ? C::TMEM_S1 : C::TMEM_S0);
    const int q_row0 = qi * block;
    const int q_rows = min(block, N - q_row0);
    const bool valid_row = row < q_rows;
    // raw-score threshold of this row: Q_p.K_q < (lse_p + ln eta) / s
    const float thr = valid_row ? (lse[(size_t)bh * N + q_row0 + row] + ln_eta) * inv_scale : -INFINITY;
    float* Urow = U + ((size_t)bh * n + qi) * n;
    int it = 0;
    for (int j = g; j < L; j += 2, ++it) {
      mbar_wait(&s_full[g], it & 1);
      tc_fence_after();
      uint32_t sr[BN];
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) tmem_ld32(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&s_free[g]);                  // S buffer free: the row is in registers
      const int jb = cols[j];
      const int kv_valid = min(BN, N - jb * block);
      int cnt = 0;
#pragma unroll
      for (int c = 0; c < BN; ++c) cnt += (__uint_as_float(sr[c]) < thr) && (c < kv_valid);
      cnt = __reduce_add_sync(0xffffffffu, cnt);
      if (lane == 0) red[g][it & 1][quarter] = cnt;
      named_bar_sync(1 + g, 128);
      if (quarter == 0 && lane == 0) {
        const int tot = red[g][it & 1][0] + red[g][it & 1][1] + red[g][it & 1][2] + red[g][it & 1][3];
        Urow[jb] = -((float)tot / (float)(q_rows * kv_valid));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_ex() {
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

mod_status make_map_ex(CUtensorMap* m, const void* base, int BH, int N, int D, int rows) {
  auto enc = get_encode_ex();
  MOD_REQUIRE(enc, MOD_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled driver entry point unavailable");
  MOD_REQUIRE(((uintptr_t)base & 127) == 0, MOD_ERR_INPUT, "Q/K pointers must be 128-byte aligned");
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
mod_status launch_ex(mod_plan P, const void* q, const void* k, const float* lse, const int* row_ptr,
                     const int* col_idx, float eta, float* U, cudaStream_t s) {
  using C = ExCfg<D, BN>;
  const int BH = P->L.batch * P->L.heads;
  CUtensorMap tq, tk;
  mod_status st;
  if ((st = make_map_ex(&tq, q, BH, P->N, D, C::BM)) != MOD_OK) return st;
  if ((st = make_map_ex(&tk, k, BH, P->N, D, BN)) != MOD_OK) return st;
  auto kern = exact_stat_kernel<D, BN>;
  MOD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  kern<<<BH * P->n, 320, C::SMEM, s>>>(tq, tk, lse, row_ptr, col_idx, U, P->N, P->n, P->L.block, 1.0f / P->scale,
                                       logf(eta));
  MOD_LAUNCH_CHECK();
  return MOD_OK;
}

}  // namespace

extern "C" mod_status mod_collect_exact_sparsity(mod_plan P, const void* q, const void* k, const float* lse,
                                                 const int32_t* row_ptr, const int32_t* col_idx, float eta,
                                                 float* stats, void* ws, void* stream) {
  MOD_NVTX("mod_collect_exact_sparsity");
  (void)ws;
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  MOD_REQUIRE(q && k && lse && row_ptr && col_idx && stats, MOD_ERR_USAGE,
              "mod_collect_exact_sparsity: q, k, lse, row_ptr, col_idx, stats must be non-NULL");
  MOD_REQUIRE(eta > 0.f && eta < 1.f, MOD_ERR_INPUT, "eta=%g must be in (0, 1)", eta);
  cudaStream_t s = as_stream(stream);
  const int D = P->L.head_dim, BN = P->L.block;
  if (D == 128 && BN == 128) st = launch_ex<128, 128>(P, q, k, lse, row_ptr, col_idx, eta, stats, s);
  else if (D == 64 && BN == 128) st = launch_ex<64, 128>(P, q, k, lse, row_ptr, col_idx, eta, stats, s);
  else if (D == 128 && BN == 64) st = launch_ex<128, 64>(P, q, k, lse, row_ptr, col_idx, eta, stats, s);
  else st = launch_ex<64, 64>(P, q, k, lse, row_ptr, col_idx, eta, stats, s);
  if (st == MOD_OK) mod_note_launches(1);
  return st;
}
