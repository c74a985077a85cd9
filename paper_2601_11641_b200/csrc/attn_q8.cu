// attn_q8.cu -- K4 on quantized operands: mod_block_sparse_attn_fwd_q8.
//
// Same computation and outputs as attn.cu (Eq. 1 P:110-115 over the CSR block lists, lse, empty
// list -> O = 0 / lse = -inf), on the Sage-style operands of quant.cu (reading Z30; the paper's
// sparse stage is SageAttention):
//   S_j = s_q[i] s_k[j] (Q8 K8_j^T)            tcgen05 kind::i8, int32 accumulate in TMEM
//   P_j = 2^(S_j log2e / sqrt(d) - m)           fp32 online softmax, rounded to e4m3 for the MMA
//   O  += P_j V8_j   then  O_d *= s_v[d] / l    tcgen05 kind::f8f6f4, fp32 accumulate
// The structure is attn.cu's (warp 0 TMA, warp 1 single-thread MMA issue, two split-KV softmax
// groups of 4 warps, merged epilogue); the operand tiles are half the bytes (Q 16 KB, K and V 16 KB
// per block), the S and PV MMAs have K = 32 per instruction (4 per block instead of 8).
// int32 scores become fp32 with the 1.5*2^23 trick (exact for |S| < 2^22; |S| <= 127*127*128).
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

using namespace sm100;

namespace {

constexpr int kEmuPairs = 2;       // of 8 pairs of exponentials evaluated on the FMA pipe

struct Q8Cfg {
  static constexpr int D = 128, BN = 128, BM = 128;
  static constexpr int TILE = 128 * 128;              // one 128 x 128-byte tile (Q, K_j or V_j^T)
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + TILE;          // K ring: slot j % 2
  static constexpr int OFF_V = OFF_K + 2 * TILE;      // V^T ring: slot j % 2
  static constexpr int OFF_BAR = OFF_V + 2 * TILE;
  static constexpr int NUM_BARS = 1 + 2 + 2 + 2 + 2 + 2;
  static constexpr int OFF_RED = OFF_BAR + NUM_BARS * 8 + 16;   // epilogue (m, l) exchange [2][2][128]
  static constexpr int SMEM = OFF_RED + 2 * 2 * 128 * 4;
  static constexpr int TMEM_S0 = 0, TMEM_S1 = BN, TMEM_O = 2 * BN;   // O_g at TMEM_O + g*D
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr uint32_t IDESC_S = idesc_s8_s32(BM, BN);
  static constexpr uint32_t IDESC_O = idesc_e4m3_f32(BM, D);
};

__device__ __forceinline__ uint16_t e4m3x2(float x0, float x1) {   // x0 -> lower byte
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(x1), "f"(x0));
  return r;
}

__global__ void __launch_bounds__(320, 1)
    attn_q8_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const float* __restrict__ q_scale,
                   const float* __restrict__ k_scale, const float* __restrict__ v_scale,
                   const int* __restrict__ row_ptr, const int* __restrict__ col_idx, __nv_bfloat16* __restrict__ out,
                   float* __restrict__ lse, int N, int n, float scale_log2) {
  using C = Q8Cfg;
  constexpr int D = C::D, BN = C::BN;
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* v_full = k_full + 2;
  uint64_t* s_full = v_full + 2;
  uint64_t* p_full = s_full + 2;
  uint64_t* o_done = p_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

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
      mbar_init(&v_full[b], 1);
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 128);
      mbar_init(&o_done[b], 1);
    }
    fence_mbar_init();
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
      mbar_arrive_expect_tx(q_full, C::TILE);
      tma_load_3d(smem + C::OFF_Q, &tm_q, q_full, 0, qi * BN, bh, pol_q);
      auto load_k = [&](int j) {
        const int s = j & 1;
        if (j >= 2) mbar_wait(&s_full[s], ((j - 2) >> 1) & 1);   // S_{j-2} consumed K slot s
        mbar_arrive_expect_tx(&k_full[s], C::TILE);
        tma_load_3d(smem + C::OFF_K + s * C::TILE, &tm_k, &k_full[s], 0, cols[j] * BN, bh, pol_kv);
      };
      auto load_v = [&](int j) {
        const int s = j & 1;
        if (j >= 2) mbar_wait(&o_done[s], ((j - 2) >> 1) & 1);   // PV_{j-2} consumed V slot s
        mbar_arrive_expect_tx(&v_full[s], C::TILE);
        // V^T [B*H, D, Np]: box {128 tokens, 128 channels}
        tma_load_3d(smem + C::OFF_V + s * C::TILE, &tm_v, &v_full[s], cols[j] * BN, 0, bh, pol_kv);
      };
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
      auto issue_s = [&](int j) {
        const int b = j & 1;
        mbar_wait(&k_full[b], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t sk = smem_u32(smem + C::OFF_K + b * C::TILE);
        const uint32_t d_s = tmem + (b ? C::TMEM_S1 : C::TMEM_S0);
#pragma unroll
        for (int kk = 0; kk < D / 32; ++kk) {   // K = 32 int8 per MMA = 32 bytes inside the 128B atom
          const uint64_t ad = smem_desc_sw128(sq + kk * 32, 16, 1024);
          const uint64_t bd = smem_desc_sw128(sk + kk * 32, 16, 1024);
          mma_ss_i8(d_s, ad, bd, C::IDESC_S, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[b]);
      };
      issue_s(0);
      if (L > 1) issue_s(1);
      for (int j = 0; j < L; ++j) {
        const int b = j & 1;
        mbar_wait(&v_full[b], (j >> 1) & 1);
        mbar_wait(&p_full[b], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t sv = smem_u32(smem + C::OFF_V + b * C::TILE);
        const uint32_t p_t = tmem + (b ? C::TMEM_S1 : C::TMEM_S0);
#pragma unroll
        for (int kk = 0; kk < BN / 32; ++kk) {
          // A = P_j (e4m3, 4 per TMEM column: 8 columns per 32 keys); B = V_j^T K-major (token bytes)
          const uint64_t bd = smem_desc_sw128(sv + kk * 32, 16, 1024);
          mma_ts_f8(tmem + C::TMEM_O + b * D, p_t + kk * 8, bd, C::IDESC_O, (j > 1 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&o_done[b]);
        if (j + 2 < L) issue_s(j + 2);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue (2 groups x 4 warps)
    const int g = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t t_s = tmem + lane_off + (g ? C::TMEM_S1 : C::TMEM_S0);
    const uint32_t t_og = tmem + lane_off + C::TMEM_O + g * D;
    const int q_row0 = qi * BN;
    const int q_rows = min(BN, N - q_row0);
    const float sq_l2 = q_scale[(size_t)bh * n + qi] * scale_log2;
    float m_run = -INFINITY, l_run = 0.f;
    int it = 0;
    for (int j = g; j < L; j += 2, ++it) {
      mbar_wait(&s_full[g], it & 1);
      tc_fence_after();
      uint32_t sr[BN];
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) tmem_ld32(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
      tmem_ld_wait();
      const int col = cols[j];
      const float sc = sq_l2 * k_scale[(size_t)bh * n + col];   // log2-domain scale of this block's int32 scores
      const int kv_valid = N - col * BN;
      int mi = -(1 << 22);
#pragma unroll
      for (int c = 0; c < BN; ++c)
        if (kv_valid >= BN || c < kv_valid) mi = max(mi, (int)sr[c]);
      const float m_new = fmaxf(m_run, (float)mi * sc);
      const bool rescale = (m_new - m_run) > 8.0f;
      const float m_use = rescale ? m_new : m_run;
      const float alpha = rescale ? ex2(m_run - m_new) : 1.0f;
      // x = S*sc - m = t*sc - (1.5*2^23*sc + m) with t = float(S + 1.5*2^23) taken from the bits
      const float off = -fmaf(12582912.0f, sc, m_use);
      const float2 sc2 = make_float2(sc, sc), of2 = make_float2(off, off);
      float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      uint32_t pk[BN / 4];
#pragma unroll
      for (int c = 0; c < BN; c += 4) {
        float p4[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cc = c + 2 * h;
          const float2 tt = make_float2(__int_as_float((int)sr[cc] + 0x4B400000),
                                        __int_as_float((int)sr[cc + 1] + 0x4B400000));
          float2 x = ffma2(tt, sc2, of2);
          if (kv_valid < BN) {
            if (cc >= kv_valid) x.x = -INFINITY;
            if (cc + 1 >= kv_valid) x.y = -INFINITY;
          }
          float2 p;
          if (((cc / 2) & 7) < kEmuPairs) {
            p = ex2_poly2(x);
          } else {
            p.x = ex2(x.x);
            p.y = ex2(x.y);
          }
          acc2[h] = fadd2(acc2[h], p);
          p4[2 * h] = p.x;
          p4[2 * h + 1] = p.y;
        }
        pk[c / 4] = (uint32_t)e4m3x2(p4[0], p4[1]) | ((uint32_t)e4m3x2(p4[2], p4[3]) << 16);
      }
      l_run = fmaf(l_run, alpha, (acc2[0].x + acc2[0].y) + (acc2[1].x + acc2[1].y));
      m_run = m_use;
      tmem_st32(t_s, pk);                        // P_j (e4m3) over the first 32 columns of S[g]
      if (it >= 1) {
        mbar_wait(&o_done[g], (it - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(t_og + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st32(t_og + c * 32, o);
          }
        }
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[g]);
    }
    // epilogue: merge the two split-KV partial results, O * s_v / l -> bf16, lse
    auto red = reinterpret_cast<float(*)[2][128]>(smem + C::OFF_RED);
    red[g][0][row] = m_run;
    red[g][1][row] = l_run;
    named_bar_sync(1, 256);
    const int n0 = (L + 1) / 2, n1 = L / 2;
    const float m0 = red[0][0][row], l0 = red[0][1][row], m1 = red[1][0][row], l1 = red[1][1][row];
    const bool valid = row < q_rows;
    const size_t grow = (size_t)bh * N + q_row0 + row;
    const float* vsc = v_scale + (size_t)bh * D;
    if (L > 0) {
      mbar_wait(&o_done[0], (n0 - 1) & 1);
      if (n1 > 0) mbar_wait(&o_done[1], (n1 - 1) & 1);
      tc_fence_after();
      const float m = fmaxf(m0, m1);
      const float f0 = ex2(m0 - m);
      const float f1 = n1 > 0 ? ex2(m1 - m) : 0.f;
      const float l = l0 * f0 + l1 * f1;
      const float a0 = f0 / l, a1 = f1 / l;
      const uint32_t t_o0 = tmem + lane_off + C::TMEM_O + g * (D / 2);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        uint32_t o0[32], o1[32];
        tmem_ld32(t_o0 + c * 32, o0);
        if (n1 > 0) tmem_ld32(t_o0 + D + c * 32, o1);
        tmem_ld_wait();
        uint32_t pkd[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int d0 = g * (D / 2) + c * 32 + 2 * e;
          float x0 = __uint_as_float(o0[2 * e]) * a0, x1 = __uint_as_float(o0[2 * e + 1]) * a0;
          if (n1 > 0) {
            x0 = fmaf(__uint_as_float(o1[2 * e]), a1, x0);
            x1 = fmaf(__uint_as_float(o1[2 * e + 1]), a1, x1);
          }
          pkd[e] = pack_bf16(x0 * __ldg(vsc + d0), x1 * __ldg(vsc + d0 + 1));
        }
        if (valid) {
          int4* dst = reinterpret_cast<int4*>(out + grow * D + g * (D / 2) + c * 32);
#pragma unroll
          for (int e = 0; e < 4; ++e) dst[e] = make_int4(pkd[4 * e], pkd[4 * e + 1], pkd[4 * e + 2], pkd[4 * e + 3]);
        }
      }
      if (valid && lse && g == 0) lse[grow] = (m + __log2f(l)) * 0.69314718055994531f;
    } else if (valid) {
      int4* dst = reinterpret_cast<int4*>(out + grow * D + g * (D / 2));
#pragma unroll
      for (int e = 0; e < D / 16; ++e) dst[e] = make_int4(0, 0, 0, 0);
      if (lse && g == 0) lse[grow] = -INFINITY;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_q8() {
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

// 3D byte map: dims {inner, rows, BH}, row pitch `pitch` bytes, box {128, 128, 1}, 128B swizzle
mod_status make_map_u8(CUtensorMap* m, const void* base, int inner, int rows, int pitch, int BH) {
  auto enc = get_encode_q8();
  MOD_REQUIRE(enc, MOD_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled driver entry point unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)BH};
  cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)pitch * rows};
  cuuint32_t box[3] = {128, 128, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MOD_REQUIRE(r == CUDA_SUCCESS, MOD_ERR_CUDA, "cuTensorMapEncodeTiled (u8) failed (%d)", (int)r);
  return MOD_OK;
}

}  // namespace

extern "C" mod_status mod_block_sparse_attn_fwd_q8(mod_plan P, const void* qbuf, const int32_t* row_ptr,
                                                   const int32_t* col_idx, void* o, float* lse, void* ws,
                                                   void* stream) {
  MOD_NVTX("mod_block_sparse_attn_fwd_q8");
  (void)ws;
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  size_t off[6];
  if ((st = mod_quant_buffer_layout(P, off)) != MOD_OK) return st;
  MOD_REQUIRE(qbuf && row_ptr && col_idx && o, MOD_ERR_USAGE,
              "mod_block_sparse_attn_fwd_q8: qbuf, row_ptr, col_idx, o must be non-NULL");
  MOD_REQUIRE(((uintptr_t)qbuf & 255) == 0 && ((uintptr_t)o & 15) == 0, MOD_ERR_INPUT,
              "mod_block_sparse_attn_fwd_q8: qbuf must be 256-byte and o 16-byte aligned");
  const char* base = static_cast<const char*>(qbuf);
  const int BH = P->L.batch * P->L.heads, N = P->N, Np = (N + 15) / 16 * 16;
  CUtensorMap tq, tk, tv;
  if ((st = make_map_u8(&tq, base + off[0], Q8Cfg::D, N, Q8Cfg::D, BH)) != MOD_OK) return st;
  if ((st = make_map_u8(&tk, base + off[1], Q8Cfg::D, N, Q8Cfg::D, BH)) != MOD_OK) return st;
  if ((st = make_map_u8(&tv, base + off[2], N, Q8Cfg::D, Np, BH)) != MOD_OK) return st;
  MOD_CUDA(cudaFuncSetAttribute(attn_q8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Q8Cfg::SMEM));
  const float scale_log2 = P->scale * 1.4426950408889634f;
  cudaStream_t s = as_stream(stream);
  attn_q8_kernel<<<BH * P->n, 320, Q8Cfg::SMEM, s>>>(
      tq, tk, tv, reinterpret_cast<const float*>(base + off[3]), reinterpret_cast<const float*>(base + off[4]),
      reinterpret_cast<const float*>(base + off[5]), row_ptr, col_idx, (__nv_bfloat16*)o, lse, N, P->n, scale_log2);
  MOD_LAUNCH_CHECK();
  mod_note_launches(1);
  return MOD_OK;
}
