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
//   warp 0      TMA producer: Q once, then K_j / V_j tiles gathered BY INDEX from the CSR list into
//               shared-memory rings (128B-swizzled boxes; 3D tensor maps zero-fill keys >= N per head).
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer, in the order
//                  S_0, S_1, PV_0, S_2, PV_1, S_3, ...   (one wait point per PV/S pair)
//               S_j = Q K_j^T  (SS, fp32 into TMEM S[j%2]);  O_{j%2} += P_j V_j (TS: A = bf16 P_j in TMEM).
//   warps 2..9  softmax in two independent groups of 4 warps: group g owns the KV blocks j = g mod 2
//               (split-KV inside the CTA) with its own S buffer, running max / sum and accumulator
//               O_g.  Each SM sub-partition therefore runs two unsynchronised softmax warps, so the
//               MUFU pipe (16 ex2/clk/SM -- exactly the tcgen05 rate of a 128x128 tile) stays busy
//               while the other group reads S or waits; 3/8 of the exponentials run as a
//               polynomial on the FMA pipe.  Thread = query row: tcgen05.ld of the S row, online
//               softmax in the log2 domain, bf16 P back into TMEM (tcgen05.st), lazy O rescale only
//               when the running max grows by > 8 (exact: O_g and l_g share the reference max).
//               Epilogue: split-KV merge of (m_g, l_g, O_g), O / l -> bf16, lse.
// TMEM: S[b] [b*BN,(b+1)*BN) for b < NS, O_0, O_1 after them: NS = 3 S buffers where they fit
// (D = 64 or 64-key blocks: the MMA then runs S two blocks ahead of the softmax), else NS = 2.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "sm100.cuh"

using namespace sm100;

namespace {

constexpr int kEmuPairsPer8 = 2;

template <int D, int BN>
struct SplitCfg {
  static constexpr int BM = 128;                      // query rows per tile (tcgen05 M)
  // S buffers in TMEM: 3 when they fit beside the two O accumulators (D = 64, or 64-key blocks), so the
  // MMA issues S_{j+2} before PV_j has consumed P_j and each softmax group finds its next S ready
  // (its MUFU-bound exponentials then run back to back); 2 at D = 128 with 128-key blocks
  static constexpr int NS = (3 * BN + 2 * D) <= 512 ? 3 : 2;
  static constexpr int STAGES = NS;                   // K ring slot = j % NS = S buffer (k_empty == s_full)
  __device__ static int sbuf(int j) { return NS == 2 ? (j & 1) : (int)((unsigned)j % (unsigned)NS); }
  __device__ static uint32_t sphase(int j) { return NS == 2 ? ((j >> 1) & 1) : (((unsigned)j / (unsigned)NS) & 1u); }
  static constexpr int VSTAGES = 2;                   // V ring slot = j % 2 = O_g (v_empty == o_done[g])
  static constexpr int Q_BOX = BM * 128;              // bytes of one 64-column box of Q
  static constexpr int KV_BOX = BN * 128;             // bytes of one 64-column box of K or V
  static constexpr int NATOM = D / 64;                // 128B swizzle atoms along D
  static constexpr int Q_BYTES = Q_BOX * NATOM;
  static constexpr int KV_BYTES = KV_BOX * NATOM;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + STAGES * KV_BYTES;
  static constexpr int OFF_BAR = OFF_V + VSTAGES * KV_BYTES;
  static constexpr int NUM_BARS = 1 + STAGES + VSTAGES + NS + 2 + 2;
  static constexpr int OFF_RED = OFF_BAR + NUM_BARS * 8 + 16;      // epilogue (m, l) exchange [2][2][128] f32
  static constexpr int SMEM = OFF_RED + 2 * 2 * 128 * 4;
  static constexpr int TMEM_O = NS * BN;                            // S[b] at b*BN; O_g at TMEM_O + g*D
  static constexpr uint32_t TMEM_COLS = (NS * BN + 2 * D) <= 256 ? 256 : 512;
  static constexpr uint32_t IDESC_S = idesc_bf16_f32(BM, BN, false, false);
  static constexpr uint32_t IDESC_O = idesc_bf16_f32(BM, D, false, true);
  static constexpr int THREADS = 320;
};

template <int D, int BN>
__global__ void __launch_bounds__(320, 1)
    attn_split_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const int* __restrict__ row_ptr,
                    const int* __restrict__ col_idx, __nv_bfloat16* __restrict__ out, float* __restrict__ lse,
                    int N, int n, int block, float scale_log2) {
  using C = SplitCfg<D, BN>;
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* v_full = k_full + C::STAGES;
  uint64_t* s_full = v_full + C::VSTAGES;   // [NS], per S buffer
  uint64_t* p_full = s_full + C::NS;
  uint64_t* o_done = p_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023u) != 0) __trap();   // SWIZZLE_128B needs 1024B alignment
  const int item = blockIdx.x;
  const int bh = item / n, qi = item % n;
  const int beg = row_ptr[(size_t)bh * (n + 1) + qi];
  const int L = row_ptr[(size_t)bh * (n + 1) + qi + 1] - beg;
  const int* cols = col_idx + (size_t)bh * n * n + beg;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < C::STAGES; ++s) mbar_init(&k_full[s], 1);
    for (int s = 0; s < C::VSTAGES; ++s) mbar_init(&v_full[s], 1);
    for (int b = 0; b < C::NS; ++b) mbar_init(&s_full[b], 1);
    for (int b = 0; b < 2; ++b) {
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
      mbar_arrive_expect_tx(q_full, C::Q_BYTES);
#pragma unroll
      for (int a = 0; a < C::NATOM; ++a)
        tma_load_3d(smem + C::OFF_Q + a * C::Q_BOX, &tm_q, q_full, a * 64, qi * block, bh, pol_q);
      auto load_k = [&](int j) {
        const int s = C::sbuf(j);
        if (j >= C::NS) mbar_wait(&s_full[s], C::NS == 2 ? (((j - 2) >> 1) & 1) : C::sphase(j) ^ 1u);   // S_{j-NS} consumed K slot s
        unsigned char* dst = smem + C::OFF_K + s * C::KV_BYTES;
        mbar_arrive_expect_tx(&k_full[s], C::KV_BYTES);
        const int row = cols[j] * block;
#pragma unroll
        for (int a = 0; a < C::NATOM; ++a) tma_load_3d(dst + a * C::KV_BOX, &tm_k, &k_full[s], a * 64, row, bh, pol_kv);
      };
      auto load_v = [&](int j) {
        const int s = j & 1;
        if (j >= 2) mbar_wait(&o_done[s], ((j - 2) >> 1) & 1);   // PV_{j-2} consumed V slot s
        unsigned char* dst = smem + C::OFF_V + s * C::KV_BYTES;
        mbar_arrive_expect_tx(&v_full[s], C::KV_BYTES);
        const int row = cols[j] * block;
#pragma unroll
        for (int a = 0; a < C::NATOM; ++a) tma_load_3d(dst + a * C::KV_BOX, &tm_v, &v_full[s], a * 64, row, bh, pol_kv);
      };
      // demand order of the MMA warp: K0 .. K_{NS-1}, V0, K_NS, V1, K_{NS+1}, ...
      for (int j = 0; j < C::NS - 1 && j < L; ++j) load_k(j);
      for (int j = 0; j < L; ++j) {
        if (j + C::NS - 1 < L) load_k(j + C::NS - 1);
        load_v(j);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // tcgen05.mma issue blocks while the pipe is busy (shallow queue): every wait of this thread
    // drains the pipe, so the loop has few wait points and one commit per MMA group:
    //   S_0, S_1, then per j:  [wait V_j, P_j] PV_j -> O_{j%2}   [wait K_{j+2}] S_{j+2} -> S[j%2]
    if (lane == 0 && L > 0) {
      const uint32_t sq = smem_u32(smem + C::OFF_Q);
      mbar_wait(q_full, 0);
      tc_fence_after();
      auto issue_s = [&](int j, int b) {   // b = C::sbuf(j) (a literal where the caller knows it)
        mbar_wait(&k_full[b], C::sphase(j));
        tc_fence_after();
        const uint64_t a_base = smem_desc_sw128(sq, 16, 1024);
        const uint64_t b_base = smem_desc_sw128(smem_u32(smem + C::OFF_K + b * C::KV_BYTES), 16, 1024);
        const uint32_t d_s = tmem + b * BN;
        // K-major SW128: 32 bytes per K step inside a 128B atom, atoms one box apart (offsets in 16 B)
        static_for<D / 16>([&](auto kc) {
          constexpr int kk = decltype(kc)::value;
          mma_ss_off<((kk / 4) * C::Q_BOX + (kk % 4) * 32) / 16, ((kk / 4) * C::KV_BOX + (kk % 4) * 32) / 16>(
              d_s, a_base, b_base, C::IDESC_S, kk > 0 ? 1u : 0u);
        });
        mma_commit(&s_full[b]);          // also releases K slot b to the producer
      };
      for (int j = 0; j < C::NS && j < L; ++j) issue_s(j, C::sbuf(j));
      // PV_j, then S_{j+NS} into the S buffer PV_j just read
      auto pv_then_s = [&](int j, int b, int sb) {
        mbar_wait(&v_full[b], (j >> 1) & 1);
        mbar_wait(&p_full[b], (j >> 1) & 1);
        tc_fence_after();
        const uint64_t v_base = smem_desc_sw128(smem_u32(smem + C::OFF_V + b * C::KV_BYTES), C::KV_BOX, 1024);
        const uint32_t p_t = tmem + sb * BN;
        const uint32_t acc0 = j > 1 ? 1u : 0u;
        // B = V_j: N = D (MN-major, 64-column atoms LBO = KV_BOX apart), K = 16 keys = 2048 bytes
        static_for<BN / 16>([&](auto kc) {
          constexpr int kk = decltype(kc)::value;
          mma_ts_off<kk * 8, kk * 2048 / 16>(tmem + C::TMEM_O + b * D, p_t, v_base, C::IDESC_O, kk > 0 ? 1u : acc0);
        });
        mma_commit(&o_done[b]);          // also releases V slot b to the producer
        if (j + C::NS < L) issue_s(j + C::NS, sb);   // S[sb] is free once PV_j (issued above, in order) read P_j
      };
      if constexpr (C::NS == 2) {
        // unrolled by two so that every slot index is a compile-time constant: the descriptors and
        // TMEM addresses of both halves are loop-invariant (uniform registers, no per-MMA R2UR)
        for (int j = 0; j < L; j += 2) {
          pv_then_s(j, 0, 0);
          if (j + 1 < L) pv_then_s(j + 1, 1, 1);
        }
      } else {
        for (int j = 0; j < L; ++j) pv_then_s(j, j & 1, C::sbuf(j));
      }
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue (2 groups x 4 warps)
    const int g = (warp - 2) >> 2;
    const int quarter = warp & 3;          // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;   // query row within the tile
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t t_og = tmem + lane_off + C::TMEM_O + g * D;
    const uint32_t t_sg = tmem + lane_off + (g ? BN : 0);   // this group's S buffer when NS == 2
    const int q_row0 = qi * block;
    const int q_rows = min(block, N - q_row0);
    float m_run = -INFINITY, l_run = 0.f;
    int it = 0;
    for (int j = g; j < L; j += 2, ++it) {
      const int sb = C::NS == 2 ? g : C::sbuf(j);                 // S_j, then P_j
      const uint32_t t_s = C::NS == 2 ? t_sg : tmem + lane_off + sb * BN;
      mbar_wait(&s_full[sb], C::NS == 2 ? (uint32_t)(it & 1) : C::sphase(j));
      tc_fence_after();
      uint32_t sr[BN];
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) tmem_ld32(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
      tmem_ld_wait();
      float* s = reinterpret_cast<float*>(sr);
      const int kv_valid = N - cols[j] * block;  // keys of this block inside the sequence
      if (kv_valid < BN) {
#pragma unroll
        for (int c = 0; c < BN; ++c)
          if (c >= kv_valid) s[c] = -INFINITY;
      }
      float mxv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mxv[u] = s[u];
#pragma unroll
      for (int c = 8; c < BN; c += 8)
#pragma unroll
        for (int u = 0; u < 8; ++u) mxv[u] = fmaxf(mxv[u], s[c + u]);
      const float mx = fmaxf(fmaxf(fmaxf(mxv[0], mxv[1]), fmaxf(mxv[2], mxv[3])),
                             fmaxf(fmaxf(mxv[4], mxv[5]), fmaxf(mxv[6], mxv[7])));
      const float m_new = fmaxf(m_run, mx * scale_log2);
      const bool rescale = (m_new - m_run) > 8.0f;   // also true on the first block (m_run = -inf)
      const float m_use = rescale ? m_new : m_run;
      const float alpha = rescale ? ex2(m_run - m_new) : 1.0f;
      // packed fp32x2 FMA-pipe ops (FFMA2 / FADD2): x = s*log2e/sqrt(d) - m per pair; a share of the
      // pairs is exponentiated by a polynomial on the FMA pipe, the rest by MUFU ex2 (16/clk/SM, the
      // tcgen05 rate of a 128x128 tile, so MUFU alone would pace the whole loop)
      const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m_use, -m_use);
      float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      uint32_t pk[BN / 2];
#pragma unroll
      for (int c = 0; c < BN; c += 2) {
        const float2 x = ffma2(make_float2(s[c], s[c + 1]), sc2, nm2);
        float2 p;
        if (((c / 2) & 7) < kEmuPairsPer8) {
          p = ex2_poly2(x);
        } else {
          p.x = ex2(x.x);
          p.y = ex2(x.y);
        }
        acc2[(c / 2) & 1] = fadd2(acc2[(c / 2) & 1], p);
        pk[c / 2] = pack_bf16(p.x, p.y);
      }
      l_run = fmaf(l_run, alpha, (acc2[0].x + acc2[0].y) + (acc2[1].x + acc2[1].y));
      m_run = m_use;
#pragma unroll
      for (int c = 0; c < BN / 64; ++c) tmem_st32(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[c * 32]));
      if (it >= 1) {
        mbar_wait(&o_done[g], (it - 1) & 1);   // this group's previous PV finished writing O_g
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
    // epilogue: merge the two split-KV partial results, O / l -> bf16, lse
    auto red = reinterpret_cast<float(*)[2][128]>(smem + C::OFF_RED);   // [group][m|l][row]
    red[g][0][row] = m_run;
    red[g][1][row] = l_run;
    named_bar_sync(1, 256);
    const int n0 = (L + 1) / 2, n1 = L / 2;   // blocks handled by group 0 / 1
    const float m0 = red[0][0][row], l0 = red[0][1][row], m1 = red[1][0][row], l1 = red[1][1][row];
    const bool valid = row < q_rows;
    const size_t grow = (size_t)bh * N + q_row0 + row;
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
          float x0 = __uint_as_float(o0[2 * e]) * a0, x1 = __uint_as_float(o0[2 * e + 1]) * a0;
          if (n1 > 0) {
            x0 = fmaf(__uint_as_float(o1[2 * e]), a1, x0);
            x1 = fmaf(__uint_as_float(o1[2 * e + 1]), a1, x1);
          }
          pkd[e] = pack_bf16(x0, x1);
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

// ================================================================================================
// Default K4 schedule (MOD_ATTN_DEFAULT): ONE softmax group of 8 warps, NS S buffers ahead of it.
//   warp 0      TMA producer (as above): Q once; K_j into ring slot j % NS, V_j into slot j % 2.
//   warp 1      TMEM allocator + tcgen05.mma issuer:  S_0 .. S_{NS-1}, then per j
//                  [wait P_j, V_j] PV_j -> O      [wait K_{j+NS}] S_{j+NS} -> S[j % NS]
//               so S_{j+1} .. S_{j+NS-1} and PV_{j-1} are queued while the softmax works on S_j: the
//               tensor pipe has 2(NS-1) MMA groups (2048 cycles at NS = 3) of work between S_j and PV_j.
//   warps 2..9  softmax, two INDEPENDENT warps per SM sub-partition: warp (quarter q, half h) owns the 16
//               full rows [32q + 16h, +16) of the tile.  Its TMEM accesses use the .16x32bx2 shape, so
//               thread t holds row 32q + 16h + t % 16 and the column half t / 16 of every S block (and of O):
//               the two halves of a row sit in lanes t and t ^ 16 of the SAME warp, and the two warps of a
//               sub-partition share nothing -- no named barrier per block, so they drift out of phase and
//               one's loads / stores / waits overlap the other's exponentials (MUFU-bound).
//               The running max is NOT recomputed per block: the scores are exponentiated against the
//               current reference max m and the half-row sum tells whether any score exceeded m by
//               more than 20 (log2 units: p <= sum <= 2^20 -- far from fp32 overflow, exact in the
//               bf16 P and fp32 l / O that follow).  Only then (first block, or a jump of the row
//               maximum) do the two lanes of a row exchange half-row maxima (shuffle), redo the block
//               against the new m and rescale l and this warp's 16 rows of O -- the online softmax with a
//               lazily updated reference, which is exact for any reference (same result up to
//               rounding).  P_j is packed bf16 over the first BN/2 columns of S_j's buffer (the TS operand
//               of PV_j); the warp's own S loads complete (tcgen05.wait::ld) before its P stores.
// TMEM: S[b] at [b BN, (b+1) BN) for b < NS, O after them (NS = 3 at D = BN = 128: 512 columns).
#ifndef K4_WAIT
#define K4_WAIT mbar_wait_sleep   // producer / MMA-issuer waits (the softmax warps poll)
#endif
#ifndef K4_SWAIT
#define K4_SWAIT mbar_wait        // the softmax warps' wait for S (try_wait loop)
#endif
// MMA issue form.  K4_LANE0_ISSUE = 1: one lane of the issuing warp runs the issue loop (the other lanes
// leave it).  0: the whole warp runs it converged and elect.sync picks the issuing lane per MMA.  Measured
// (scripts/micro/interference_probe.cu): a converged issuing warp slows the arithmetic warps of its SM
// sub-partition by 19 %, a single issuing lane by 2 %.
#ifndef K4_LANE0_ISSUE
#define K4_LANE0_ISSUE 1
#endif
// P packed in place over the score registers (exp_pack_inplace) in the default schedule's softmax
#ifndef K4_INPLACE_P
#define K4_INPLACE_P 1
#endif
#ifndef K4_EARLY_LOADS
#define K4_EARLY_LOADS 1
#endif
// Q of the query block one wave ahead (item + number of SMs: the CTA the block scheduler starts about when
// this one ends) is prefetched into L2 by the producer, so that CTA's first load -- the only HBM read on its
// critical path (K / V of the head are L2-resident) -- hits L2.
#ifndef K4_PREFETCH_Q
#define K4_PREFETCH_Q 1
#endif
// A tile of `rows` token rows x D bf16 of head bh into shared memory as NATOM 128B-swizzled 64-column
// atoms one `box` apart.  K4_TMA4D (D = 128): ONE 4D TMA box {64 columns, rows, 2 atoms, 1} over the
// [B*H, N, D] tensor viewed as {64, N, D/64, B*H} (make_map_tile), whose shared-memory image is exactly
// the two atoms back to back -- half the TMA instructions of the producer thread.
#ifndef K4_TMA4D
#define K4_TMA4D 1
#endif
template <int NATOM>
__device__ __forceinline__ void tma_load_tile(unsigned char* dst, int box, const CUtensorMap* m, uint64_t* bar, int row,
                                              int bh, uint64_t policy) {
  if constexpr (K4_TMA4D && NATOM == 2) {
    tma_load_4d(dst, m, bar, 0, row, 0, bh, policy);
  } else {
#pragma unroll
    for (int a = 0; a < NATOM; ++a) tma_load_3d(dst + a * box, m, bar, a * 64, row, bh, policy);
  }
}
template <int NATOM, bool TILE_MAP = false>   // TILE_MAP: tm_q was made by make_map_tile
__device__ __forceinline__ void prefetch_next_q(const CUtensorMap* tm_q, int item, int n, int block) {
  if constexpr (K4_PREFETCH_Q) {
    const int nx = item + (int)num_sms();
    if (nx < (int)gridDim.x) {
      // evict_last: the tile must survive ~one CTA lifetime of K / V streaming (themselves evict_last); a
      // normal-priority prefetch was evicted before use ~60 % of the time (+0.43 GB DRAM per launch)
      const uint64_t pol = policy_evict_last();
      if constexpr (TILE_MAP && K4_TMA4D && NATOM == 2) {
        tma_prefetch_l2_4d(tm_q, 0, (nx % n) * block, 0, nx / n, pol);
      } else {
#pragma unroll
        for (int a = 0; a < NATOM; ++a) tma_prefetch_l2_3d(tm_q, a * 64, (nx % n) * block, nx / n, pol);
      }
    }
  }
}

template <uint32_t A_OFF, uint32_t B_OFF>
__device__ __forceinline__ void k4_mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (K4_LANE0_ISSUE) mma_ss_off<A_OFF, B_OFF>(d, a, b, idesc, acc);
  else mma_ss_e<A_OFF, B_OFF>(d, a, b, idesc, acc);
}
template <uint32_t A_COL, uint32_t B_OFF>
__device__ __forceinline__ void k4_mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (K4_LANE0_ISSUE) mma_ts_off<A_COL, B_OFF>(d, a, b, idesc, acc);
  else mma_ts_e<A_COL, B_OFF>(d, a, b, idesc, acc);
}
__device__ __forceinline__ void k4_commit(uint64_t* bar) {
  if constexpr (K4_LANE0_ISSUE) mma_commit(bar);
  else mma_commit_e(bar);
}
template <int D, int BN>
struct Attn1Cfg {
  static constexpr int BM = 128;
  static constexpr int NS = (512 - D) / BN > 7 ? 7 : (512 - D) / BN;
  static constexpr int VSTAGES = 2;
  static constexpr int COLS = BN / 2;                 // score columns per thread (half a row)
  static constexpr int OCOLS = D / 2;                 // O columns per thread (rescale, epilogue)
  static constexpr int Q_BOX = BM * 128, KV_BOX = BN * 128, NATOM = D / 64;
  static constexpr int Q_BYTES = Q_BOX * NATOM, KV_BYTES = KV_BOX * NATOM;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + NS * KV_BYTES;
  static constexpr int OFF_BAR = OFF_V + VSTAGES * KV_BYTES;
  // q_full, k_full[NS], v_full[2], s_full[NS], p_full[NS], o_done[NS] (PV_j commits to o_done[j % NS])
  static constexpr int NUM_BARS = 1 + NS + VSTAGES + NS + NS + NS;
  static constexpr int SMEM = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr int TMEM_O = NS * BN;
  static constexpr uint32_t TMEM_COLS = (NS * BN + D) <= 256 ? 256 : 512;
  static constexpr int SOFTMAX_WARPS = 8;
  // MMA issue.  A tcgen05.mma that finds the (shallow) tensor queue full stalls its warp AND slows the
  // softmax warps of the same SM sub-partition (measured: that sub-partition's softmax falls behind and
  // paces the CTA), so the issue is spread over two warps on different sub-partitions: warp 0 loads (TMA),
  // warp 1 issues PV, warp 10 issues S.  (Measured and dropped: one issuer for both, 1580 vs 1444 cycles
  // per block; S on two alternating warps; pairs of MMAs paced by commits; four issuers over N-halves
  // with the left S half in the load warp: its waits delay the V loads, 2304 cycles per block.)
  static constexpr int S_WARP = 2 + SOFTMAX_WARPS;
  static constexpr int THREADS = 64 + 32 * SOFTMAX_WARPS + 32;
  static constexpr uint32_t IDESC_S = idesc_bf16_f32(BM, BN, false, false);
  static constexpr uint32_t IDESC_O = idesc_bf16_f32(BM, D, false, true);
#ifndef K4_EMU
#define K4_EMU 2
#endif
#ifndef K4_EMU1
#define K4_EMU1 2
#endif
#ifndef K4_EMU_D64
#define K4_EMU_D64 K4_EMU
#endif
  // pairs of every 8 exponentiated on the FMA pipe (the rest on MUFU); D = 64 has half the tensor work per
  // block, so its softmax can move more of the exponentials off MUFU
  static constexpr int EMU = D == 64 ? K4_EMU_D64 : K4_EMU;
  static constexpr int EMU1 = D == 64 ? K4_EMU_D64 : K4_EMU1;   // the same on the MMA issuers' sub-partitions
  static constexpr float OVF = 1048576.0f;            // 2^20: half-row sum bound of the lazy reference
};

// Bring-up instrumentation, compiled only into trace builds (-DMOD_K4_TRACE, scripts/k4_trace.py):
// clock64 stamps of the MMA thread and of one softmax warp for every 4096th CTA, and per-CTA
// clock64 / globaltimer spans of every CTA.  The shipped library contains none of it.
#ifdef MOD_K4_TRACE
constexpr int kTrCtas = 8, kTrBlocks = 512;
__device__ long long g_k4_ev[kTrCtas][18][kTrBlocks][6];
__device__ long long g_k4_span[1 << 16][4];
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define K4T(role, ev, j)                                                                      \
  do {                                                                                        \
    if ((blockIdx.x & 4095) == 1234 && (j) < kTrBlocks && (blockIdx.x >> 12) < kTrCtas)       \
      g_k4_ev[blockIdx.x >> 12][role][j][ev] = clock64();                                     \
  } while (0)
#else
#define K4T(role, ev, j) \
  do {                   \
  } while (0)
#endif


template <int EMU, int NC>
__device__ __forceinline__ float exp_pack(const float* s, float scale_log2, float m, uint32_t* pk) {
  const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m, -m);
  float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int c = 0; c < NC; c += 2) {
    const float2 x = ffma2(make_float2(s[c], s[c + 1]), sc2, nm2);
    float2 p;
    if (((c / 2) & 7) < EMU) {
      p = ex2_poly2<true>(x);
    } else {
      p.x = ex2(x.x);
      p.y = ex2(x.y);
    }
    acc2[(c / 2) & 1] = fadd2(acc2[(c / 2) & 1], p);
    pk[c / 2] = pack_bf16(p.x, p.y);
  }
  return (acc2[0].x + acc2[0].y) + (acc2[1].x + acc2[1].y);
}

// exp_pack with P packed IN PLACE: the scores r[0..NC) (fp32 bits) become P in r[0..NC/2) (bf16 pairs).  Pair
// c is read before word c/2 <= c is written, so the packed row lands in the registers the tcgen05.st of P
// takes without register moves (the score registers are dead after their pair is exponentiated).
template <int EMU, int NC>
__device__ __forceinline__ float exp_pack_inplace(uint32_t* r, float scale_log2, float m) {
  const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m, -m);
  float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int c = 0; c < NC; c += 2) {
    const float2 x = ffma2(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])), sc2, nm2);
    float2 p;
    if (((c / 2) & 7) < EMU) {
      p = ex2_poly2<true>(x);
    } else {
      p.x = ex2(x.x);
      p.y = ex2(x.y);
    }
    acc2[(c / 2) & 1] = fadd2(acc2[(c / 2) & 1], p);
    r[c / 2] = pack_bf16(p.x, p.y);
  }
  return (acc2[0].x + acc2[0].y) + (acc2[1].x + acc2[1].y);
}

template <int NC>
__device__ __forceinline__ float row_max(const float* s) {   // max of s[0..NC), two FMNMX3 chains
  static_assert(NC % 4 == 0, "row_max: NC must be a multiple of 4");
  float a = s[0], b = s[1];
#pragma unroll
  for (int c = 2; c < NC; c += 4) {
    a = fmax3f(a, s[c], s[c + 1]);
    if (c + 3 < NC) b = fmax3f(b, s[c + 2], s[c + 3]);
  }
  return fmaxf(a, b);
}

template <int D, int BN>
__global__ void __launch_bounds__(Attn1Cfg<D, BN>::THREADS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const int* __restrict__ row_ptr,
                    const int* __restrict__ col_idx, __nv_bfloat16* __restrict__ out, float* __restrict__ lse,
                    int N, int n, int block, float scale_log2) {
  using C = Attn1Cfg<D, BN>;
  constexpr int NS = C::NS;
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* v_full = k_full + NS;
  uint64_t* s_full = v_full + C::VSTAGES;
  uint64_t* p_full = s_full + NS;
  uint64_t* o_done = p_full + NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + NS);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023u) != 0) __trap();   // SWIZZLE_128B needs 1024B alignment
  const int item = blockIdx.x;
  const int bh = item / n, qi = item % n;
  const int beg = row_ptr[(size_t)bh * (n + 1) + qi];
  const int L = row_ptr[(size_t)bh * (n + 1) + qi + 1] - beg;
  const int* cols = col_idx + (size_t)bh * n * n + beg;

  const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
  auto load_k = [&](int j) {   // one thread
    const int s = j % NS;
    unsigned char* dst = smem + C::OFF_K + s * C::KV_BYTES;
    mbar_arrive_expect_tx(&k_full[s], C::KV_BYTES);
    tma_load_tile<C::NATOM>(dst, C::KV_BOX, &tm_k, &k_full[s], cols[j] * block, bh, pol_kv);
  };
  auto load_v = [&](int j) {   // one thread
    const int s = j & 1;
    unsigned char* dst = smem + C::OFF_V + s * C::KV_BYTES;
    mbar_arrive_expect_tx(&v_full[s], C::KV_BYTES);
    tma_load_tile<C::NATOM>(dst, C::KV_BOX, &tm_v, &v_full[s], cols[j] * block, bh, pol_kv);
  };
  auto load_first = [&]() {   // Q and K_0 .. K_{NS-1}: the producer's first loads (one thread)
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    mbar_arrive_expect_tx(q_full, C::Q_BYTES);
    tma_load_tile<C::NATOM>(smem + C::OFF_Q, C::Q_BOX, &tm_q, q_full, qi * block, bh, pol_q);
    for (int j = 0; j < NS && j < L; ++j) load_k(j);
  };
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], C::SOFTMAX_WARPS);   // one elected arrival per softmax warp
      mbar_init(&o_done[s], 1);
    }
    for (int s = 0; s < C::VSTAGES; ++s) mbar_init(&v_full[s], 1);
    fence_mbar_init();
    // K4_EARLY_LOADS: the first loads go out before the TMEM allocation and the CTA barrier (thread 0 is the
    // producer lane), so their latency overlaps the CTA's set-up
    if (K4_EARLY_LOADS && L > 0) load_first();
  }
#ifdef MOD_K4_TRACE
  const long long span_c0 = clock64(), span_t0 = gtimer();
#endif
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // ---------------------------------------------------------------- loads and MMA issue (warps 0, 1, 10, 11)
  // S_j = Q K_j^T into S buffer b = j % NS; whole warp, converged (elect.sync inside each MMA keeps the
  // descriptors in uniform registers)
  auto issue_s = [&](int j, auto bc) {
    constexpr int b = decltype(bc)::value;
    K4_WAIT(&k_full[b], (j / NS) & 1);
    tc_fence_after();
    const uint64_t a_base = smem_desc_sw128(smem_u32(smem + C::OFF_Q), 16, 1024);
    const uint64_t b_base = smem_desc_sw128(smem_u32(smem + C::OFF_K + b * C::KV_BYTES), 16, 1024);
    // K-major SW128: 32 bytes per K step inside a 128B atom, atoms one box apart (offsets in 16 B)
    static_for<D / 16>([&](auto kc) {
      constexpr int kk = decltype(kc)::value;
      k4_mma_ss<((kk / 4) * C::Q_BOX + (kk % 4) * 32) / 16, ((kk / 4) * C::KV_BOX + (kk % 4) * 32) / 16>(
          tmem + b * BN, a_base, b_base, C::IDESC_S, kk > 0 ? 1u : 0u);
    });
    k4_commit(&s_full[b]);          // also releases K slot b to the producer
  };
  // PV_j: O += P_j V_j with P_j from TMEM (TS form)
  auto issue_pv = [&](int j, auto bc, auto vc) {
    constexpr int b = decltype(bc)::value, vs = decltype(vc)::value;
    K4T(0, 0, j);
    K4_WAIT(&v_full[vs], (j >> 1) & 1);
    K4T(0, 1, j);
    K4_WAIT(&p_full[b], (j / NS) & 1);
    K4T(0, 2, j);
    tc_fence_after();
    // B = V_j: N = D (MN-major, 64-column atoms LBO = KV_BOX apart), K = 16 keys = 2048 bytes
    const uint64_t v_base = smem_desc_sw128(smem_u32(smem + C::OFF_V + vs * C::KV_BYTES), C::KV_BOX, 1024);
    const uint32_t acc0 = j > 0 ? 1u : 0u;
    static_for<BN / 16>([&](auto kc) {
      constexpr int kk = decltype(kc)::value;
      k4_mma_ts<kk * 8, kk * 2048 / 16>(tmem + C::TMEM_O, tmem + b * BN, v_base, C::IDESC_O, kk > 0 ? 1u : acc0);
    });
    k4_commit(&o_done[b]);          // also releases V slot vs to the producer
    K4T(0, 3, j);
  };
  constexpr int UPV = (NS % 2) ? 2 * NS : NS;   // PV loops unrolled over lcm(NS, 2): literal slots

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && L > 0) {
      // demand order of the MMA warps: Q, K_0 .. K_{NS-1}, then V_j, K_{j+NS} for j = 0, 1, ...
      if (!K4_EARLY_LOADS) load_first();
      prefetch_next_q<C::NATOM, true>(&tm_q, item, n, block);
      for (int j = 0; j < L; ++j) {
        if (j >= 2) K4_WAIT(&o_done[(j - 2) % NS], ((j - 2) / NS) & 1);   // PV_{j-2} has consumed V slot j % 2
        load_v(j);
        if (j + NS < L) {
          K4_WAIT(&s_full[j % NS], (j / NS) & 1);   // S_j has consumed K slot j % NS
          load_k(j + NS);
        }
      }
    }
  } else if (warp == 1 || warp == C::S_WARP) {
    // ------------------------------------------------------------ MMA issuers
    if (L > 0 && (!K4_LANE0_ISSUE || lane == 0)) {
      K4_WAIT(q_full, 0);
      tc_fence_after();
      if (warp == 1) {
        for (int j0 = 0; j0 < L; j0 += UPV) {
          static_for<UPV>([&](auto uc) {
            constexpr int u = decltype(uc)::value;
            if (j0 + u < L) issue_pv(j0 + u, std::integral_constant<int, u % NS>{}, std::integral_constant<int, u % 2>{});
          });
        }
      } else {
        // S_j into buffer j % NS once PV_{j-NS} has completed (it read P_{j-NS} from that buffer; MMAs of
        // different issuing threads are not ordered, so the wait is on the PV commit).  Each wait is on
        // the next phase of its barrier in order, so the parities are unambiguous.
        for (int j0 = 0; j0 < L; j0 += NS) {
          static_for<NS>([&](auto uc) {
            constexpr int u = decltype(uc)::value;
            const int j = j0 + u;
            if (j < L) {
              if (j >= NS) {
                K4_WAIT(&o_done[u], ((j - NS) / NS) & 1);
                tc_fence_after();
              }
              issue_s(j, uc);
            }
          });
        }
      }
    }
  } else if (warp < 2 + C::SOFTMAX_WARPS) {
    // ------------------------------------------------------------ softmax / epilogue (8 independent warps)
    constexpr int COLS = C::COLS, OCOLS = C::OCOLS, OCH = OCOLS < 32 ? OCOLS : 32;
    constexpr unsigned FULL = 0xffffffffu;
    const int quarter = warp & 3;           // TMEM lane quarter this warp may access
    const int h = (warp - 2) >> 2;          // which 16 rows of the quarter
    const int half = lane >> 4;             // which column half of the row this thread holds
    const int row = quarter * 32 + h * 16 + (lane & 15);   // query row within the tile
    const uint32_t lane_off = (uint32_t)(quarter * 32 + h * 16) << 16;
    const int q_row0 = qi * block;
    const int q_rows = min(block, N - q_row0);
    float m_run = -INFINITY, l_run = 0.f;   // reference max (log2 units, scaled) / this half-row's sum
    const bool tr = lane == 0;
    [[maybe_unused]] const int trole = warp - 1;   // trace role of this softmax warp (1..)
    int col_next = L > 0 ? cols[0] : 0;   // column index of the next block, loaded one block ahead
#pragma unroll 1
    for (int j = 0; j < L; ++j) {
      const int b = j % NS;
      const int col = col_next;
      if (j + 1 < L) col_next = cols[j + 1];
      if (tr) K4T(trole, 0, j);
      K4_SWAIT(&s_full[b], (j / NS) & 1);
      if (tr) K4T(trole, 1, j);
      tc_fence_after();
      uint32_t sr[COLS];
      tmem_ld_rows<COLS, BN / 2>(tmem + lane_off + b * BN, sr);   // columns half * BN/2 + [0, COLS)
      tmem_ld_wait();
      float* s = reinterpret_cast<float*>(sr);
      const int kv_valid = N - col * block - half * COLS;   // keys of this half inside the sequence
      if (kv_valid < COLS) {
#pragma unroll
        for (int c = 0; c < COLS; ++c)
          if (c >= kv_valid) s[c] = -INFINITY;
      }
      if (j == 0) {   // first block of the list: the exact row maximum (both halves)
        const float mx = row_max<COLS>(s) * scale_log2;
        m_run = fmaxf(mx, __shfl_xor_sync(FULL, mx, 16));   // finite: every listed block holds >= 1 key
      }
      if (tr) K4T(trole, 2, j);
#if K4_INPLACE_P
      uint32_t* pk = sr;   // P_j packed over the scores (exp_pack_inplace)
      float sum = exp_pack_inplace<C::EMU, COLS>(sr, scale_log2, m_run);
#else
      uint32_t pk[COLS / 2];
      float sum;
      if constexpr (C::EMU1 == C::EMU)   // one copy of the loop body (instruction-cache footprint)
        sum = exp_pack<C::EMU, COLS>(s, scale_log2, m_run, pk);
      else
        sum = (quarter == 1 || quarter == C::S_WARP % 4) ? exp_pack<C::EMU1, COLS>(s, scale_log2, m_run, pk)
                           : exp_pack<C::EMU, COLS>(s, scale_log2, m_run, pk);
#endif
      const bool need = !(sum <= C::OVF);
      if (tr) K4T(trole, 3, j);
      if (__any_sync(FULL, need)) {
        // rare: a row maximum moved up by > 20 (log2): exchange half-row maxima, redo against the new m
        const int need_peer = __shfl_xor_sync(FULL, (int)need, 16);   // every lane shuffles (no short-circuit)
        const bool need_row = need || need_peer != 0;
#if K4_INPLACE_P
        // the scores were overwritten by P: reload S_j (unchanged in TMEM until P_j is stored) and re-mask
        tmem_ld_rows<COLS, BN / 2>(tmem + lane_off + b * BN, sr);
        tmem_ld_wait();
        if (kv_valid < COLS) {
#pragma unroll
          for (int c = 0; c < COLS; ++c)
            if (c >= kv_valid) s[c] = -INFINITY;
        }
#endif
        float rmax = row_max<COLS>(s) * scale_log2;
        rmax = fmaxf(rmax, __shfl_xor_sync(FULL, rmax, 16));
        const float m_new = need_row ? fmaxf(m_run, rmax) : m_run;
        const float alpha = ex2(m_run - m_new);
#if K4_INPLACE_P
        sum = exp_pack_inplace<0, COLS>(sr, scale_log2, m_new);   // every lane: its P was overwritten by the reload
#else
        if (need_row) sum = exp_pack<0, COLS>(s, scale_log2, m_new, pk);
#endif
        l_run *= alpha;
        m_run = m_new;
        if (j > 0 && __any_sync(FULL, alpha < 1.f)) {
          // PV_{j-1} has written O: its slot's previous PV_{j-1-NS} is complete (S_j, committed after
          // PV_{j-NS}, has been seen) and PV_{j-1+NS} cannot start before this warp's P_{j-1+NS}: unambiguous
          mbar_wait(&o_done[(j - 1) % NS], ((j - 1) / NS) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < OCOLS / OCH; ++c) {
            uint32_t o[OCH];
            tmem_ld_rows<OCH, D / 2>(tmem + lane_off + C::TMEM_O + c * OCH, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < OCH; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st_rows<OCH, D / 2>(tmem + lane_off + C::TMEM_O + c * OCH, o);
          }
        }
      }
      if (tr) K4T(trole, 4, j);
      l_run += sum;
      tmem_st_rows<COLS / 2, BN / 4>(tmem + lane_off + b * BN, pk);   // packed P columns half * BN/4 + [0, COLS/2)
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[b]);
      if (tr) K4T(trole, 5, j);
    }
    // epilogue: l = sum of the two half-row sums (they share m), O / l -> bf16 (this thread's D half), lse
    const float l = l_run + __shfl_xor_sync(FULL, l_run, 16);
    const bool valid = row < q_rows;
    const size_t grow = (size_t)bh * N + q_row0 + row;
    if (L > 0) {
      mbar_wait(&o_done[(L - 1) % NS], ((L - 1) / NS) & 1);   // the last PV (its slot's previous PV is complete)
      tc_fence_after();
      const float inv = 1.0f / l;
#pragma unroll
      for (int c = 0; c < OCOLS / OCH; ++c) {
        uint32_t o[OCH];
        tmem_ld_rows<OCH, D / 2>(tmem + lane_off + C::TMEM_O + c * OCH, o);   // columns half * D/2 + c*OCH + [0, OCH)
        tmem_ld_wait();
        uint32_t pkd[OCH / 2];
#pragma unroll
        for (int e = 0; e < OCH / 2; ++e) pkd[e] = pack_bf16(__uint_as_float(o[2 * e]) * inv, __uint_as_float(o[2 * e + 1]) * inv);
        if (valid) {
          int4* dst = reinterpret_cast<int4*>(out + grow * D + half * OCOLS + c * OCH);
#pragma unroll
          for (int e = 0; e < OCH / 8; ++e) dst[e] = make_int4(pkd[4 * e], pkd[4 * e + 1], pkd[4 * e + 2], pkd[4 * e + 3]);
        }
      }
      if (valid && lse && half == 0) lse[grow] = (m_run + __log2f(l)) * 0.69314718055994531f;
    } else if (valid) {
      int4* dst = reinterpret_cast<int4*>(out + grow * D + half * OCOLS);
#pragma unroll
      for (int e = 0; e < OCOLS / 8; ++e) dst[e] = make_int4(0, 0, 0, 0);
      if (lse && half == 0) lse[grow] = -INFINITY;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem);
  }
#ifdef MOD_K4_TRACE
  if (threadIdx.x == 0 && blockIdx.x < (1 << 16)) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_k4_span[blockIdx.x][0] = clock64() - span_c0;
    g_k4_span[blockIdx.x][1] = gtimer() - span_t0;
    g_k4_span[blockIdx.x][2] = span_t0;
    g_k4_span[blockIdx.x][3] = ((long long)smid << 32) | (unsigned)L;
  }
#endif
}

// ================================================================================================
// Wide K4 schedule (MOD_ATTN_WIDE, 128-token blocks): FOUR softmax warps per SM sub-partition.
// ncu of the default schedule shows ~0.7 eligible warps per scheduler and 50 % issue utilisation: the
// softmax is latency-bound with two warps per sub-partition.  Here warp (quarter q, half h, key half c)
// owns the 16 rows [32q + 16h, +16) and the 64 keys [64c, +64) of every block (32 per thread, the two
// 32-key chunks of a row in lanes t and t ^ 16), i.e. a split-KV over the two key halves of each block:
// key half c has its own reference max, row sums and accumulator O_c, so no warp ever waits for another
// until the epilogue merges (m_c, l_c, O_c).  P of key half c is written over the first 32 columns of
// that half's own S columns (no cross-warp overlap); PV^c accumulates into O_c from those columns.
// TMEM: S[b] for b < NS, then O_0, O_1 (NS = 2 at D = 128, 3 at D = 64).  608 threads: producer,
// PV issuer, 16 softmax warps, S issuer.
template <int D, int BN>
struct WideCfg {
  static constexpr int BM = 128;
  static constexpr int NS = (512 - 2 * D) / BN > 7 ? 7 : (512 - 2 * D) / BN;
  static constexpr int VSTAGES = 2;
  static constexpr int KH = BN / 2;                   // keys per key half
  static constexpr int COLS = KH / 2;                 // score columns per thread
  static constexpr int Q_BOX = BM * 128, KV_BOX = BN * 128, NATOM = D / 64;
  static constexpr int Q_BYTES = Q_BOX * NATOM, KV_BYTES = KV_BOX * NATOM;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + NS * KV_BYTES;
  static constexpr int OFF_BAR = OFF_V + VSTAGES * KV_BYTES;
  // q_full, k_full[NS], v_full[2], s_full[NS], p_full[NS][2], o_done[NS]
  static constexpr int NUM_BARS = 1 + NS + VSTAGES + NS + 2 * NS + NS;
  static constexpr int OFF_XCH = (OFF_BAR + NUM_BARS * 8 + 16 + 15) / 16 * 16;
  static constexpr int SMEM = OFF_XCH + 2 * 2 * 128 * 4;   // epilogue (m, l) per key half per row
  static constexpr int TMEM_O = NS * BN;              // O_c at TMEM_O + c * D
  static constexpr uint32_t TMEM_COLS = (NS * BN + 2 * D) <= 256 ? 256 : 512;
  static constexpr uint32_t IDESC_S = idesc_bf16_f32(BM, BN, false, false);
  static constexpr uint32_t IDESC_O = idesc_bf16_f32(BM, D, false, true);
  static constexpr int SOFTMAX_WARPS = 16;
  static constexpr int S_WARP = 2 + SOFTMAX_WARPS;
  static constexpr int THREADS = 64 + 32 * SOFTMAX_WARPS + 32;
  static constexpr int EMU = K4_EMU;
  static constexpr float OVF = 1048576.0f;
};

template <int D, int BN>
__global__ void __launch_bounds__(WideCfg<D, BN>::THREADS, 1)
    attn_wide_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const int* __restrict__ row_ptr,
                     const int* __restrict__ col_idx, __nv_bfloat16* __restrict__ out, float* __restrict__ lse,
                     int N, int n, int block, float scale_log2) {
  using C = WideCfg<D, BN>;
  constexpr int NS = C::NS;
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* v_full = k_full + NS;
  uint64_t* s_full = v_full + C::VSTAGES;
  uint64_t* p_full = s_full + NS;        // [b * 2 + c]
  uint64_t* o_done = p_full + 2 * NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + NS);
  float* xch = reinterpret_cast<float*>(smem + C::OFF_XCH);   // [c][m|l][row]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023u) != 0) __trap();
  const int item = blockIdx.x;
  const int bh = item / n, qi = item % n;
  const int beg = row_ptr[(size_t)bh * (n + 1) + qi];
  const int L = row_ptr[(size_t)bh * (n + 1) + qi + 1] - beg;
  const int* cols = col_idx + (size_t)bh * n * n + beg;

  const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
  auto load_k = [&](int j) {
    const int s = j % NS;
    unsigned char* dst = smem + C::OFF_K + s * C::KV_BYTES;
    mbar_arrive_expect_tx(&k_full[s], C::KV_BYTES);
    const int row = cols[j] * block;
#pragma unroll
    for (int a = 0; a < C::NATOM; ++a) tma_load_3d(dst + a * C::KV_BOX, &tm_k, &k_full[s], a * 64, row, bh, pol_kv);
  };
  auto load_first = [&]() {   // Q and K_0 .. K_{NS-1} (one thread)
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    mbar_arrive_expect_tx(q_full, C::Q_BYTES);
#pragma unroll
    for (int a = 0; a < C::NATOM; ++a)
      tma_load_3d(smem + C::OFF_Q + a * C::Q_BOX, &tm_q, q_full, a * 64, qi * block, bh, pol_q);
    for (int j = 0; j < NS && j < L; ++j) load_k(j);
  };
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[2 * s], C::SOFTMAX_WARPS / 2);
      mbar_init(&p_full[2 * s + 1], C::SOFTMAX_WARPS / 2);
      mbar_init(&o_done[s], 1);
    }
    for (int s = 0; s < C::VSTAGES; ++s) mbar_init(&v_full[s], 1);
    fence_mbar_init();
    if (K4_EARLY_LOADS && L > 0) load_first();   // before the TMEM allocation and the CTA barrier
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto load_v = [&](int j) {
    const int s = j & 1;
    unsigned char* dst = smem + C::OFF_V + s * C::KV_BYTES;
    mbar_arrive_expect_tx(&v_full[s], C::KV_BYTES);
    const int row = cols[j] * block;
#pragma unroll
    for (int a = 0; a < C::NATOM; ++a) tma_load_3d(dst + a * C::KV_BOX, &tm_v, &v_full[s], a * 64, row, bh, pol_kv);
  };
  auto issue_s = [&](int j, auto bc) {
    constexpr int b = decltype(bc)::value;
    K4_WAIT(&k_full[b], (j / NS) & 1);
    tc_fence_after();
    const uint64_t a_base = smem_desc_sw128(smem_u32(smem + C::OFF_Q), 16, 1024);
    const uint64_t b_base = smem_desc_sw128(smem_u32(smem + C::OFF_K + b * C::KV_BYTES), 16, 1024);
    static_for<D / 16>([&](auto kc) {
      constexpr int kk = decltype(kc)::value;
      k4_mma_ss<((kk / 4) * C::Q_BOX + (kk % 4) * 32) / 16, ((kk / 4) * C::KV_BOX + (kk % 4) * 32) / 16>(
          tmem + b * BN, a_base, b_base, C::IDESC_S, kk > 0 ? 1u : 0u);
    });
    k4_commit(&s_full[b]);
  };
  // PV^c_j: O_c += P_j[:, keys of half c] V_j[keys of half c, :]; P^c packed in that half's first KH/2 columns
  auto issue_pv = [&](int j, auto bc, auto vc) {
    constexpr int b = decltype(bc)::value, vs = decltype(vc)::value;
    K4T(0, 0, j);
    K4_WAIT(&v_full[vs], (j >> 1) & 1);
    K4T(0, 1, j);
    const uint64_t v_base = smem_desc_sw128(smem_u32(smem + C::OFF_V + vs * C::KV_BYTES), C::KV_BOX, 1024);
    const uint32_t acc0 = j > 0 ? 1u : 0u;
    static_for<2>([&](auto cc) {
      constexpr int c = decltype(cc)::value;
      K4_WAIT(&p_full[2 * b + c], (j / NS) & 1);
      tc_fence_after();
      static_for<C::KH / 16>([&](auto kc) {
        constexpr int kk = decltype(kc)::value;
        k4_mma_ts<c * C::KH + kk * 8, (c * C::KH / 16 + kk) * 2048 / 16>(tmem + C::TMEM_O + c * D, tmem + b * BN,
                                                                        v_base, C::IDESC_O, kk > 0 ? 1u : acc0);
      });
    });
    k4_commit(&o_done[b]);
    K4T(0, 2, j);
    K4T(0, 3, j);
  };
  constexpr int UPV = (NS % 2) ? 2 * NS : NS;

  if (warp == 0) {
    if (lane == 0 && L > 0) {
      if (!K4_EARLY_LOADS) load_first();
      prefetch_next_q<C::NATOM>(&tm_q, item, n, block);
      for (int j = 0; j < L; ++j) {
        if (j >= 2) K4_WAIT(&o_done[(j - 2) % NS], ((j - 2) / NS) & 1);
        load_v(j);
        if (j + NS < L) {
          K4_WAIT(&s_full[j % NS], (j / NS) & 1);
          load_k(j + NS);
        }
      }
    }
  } else if (warp == 1 || warp == C::S_WARP) {
    if (L > 0 && (!K4_LANE0_ISSUE || lane == 0)) {
      K4_WAIT(q_full, 0);
      tc_fence_after();
      if (warp == 1) {
        for (int j0 = 0; j0 < L; j0 += UPV) {
          static_for<UPV>([&](auto uc) {
            constexpr int u = decltype(uc)::value;
            if (j0 + u < L) issue_pv(j0 + u, std::integral_constant<int, u % NS>{}, std::integral_constant<int, u % 2>{});
          });
        }
      } else {
        for (int j0 = 0; j0 < L; j0 += NS) {
          static_for<NS>([&](auto uc) {
            constexpr int u = decltype(uc)::value;
            const int j = j0 + u;
            if (j < L) {
              if (j >= NS) {
                K4_WAIT(&o_done[u], ((j - NS) / NS) & 1);
                tc_fence_after();
              }
              issue_s(j, uc);
            }
          });
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax: warp (quarter, row half, key half)
    constexpr int COLS = C::COLS, KH = C::KH;
    constexpr unsigned FULL = 0xffffffffu;
    const int quarter = warp & 3;
    const int g = (warp - 2) >> 2;
    const int h = g & 1, c = g >> 1;
    const int colq = lane >> 4;
    const int row = quarter * 32 + h * 16 + (lane & 15);
    const uint32_t lane_off = (uint32_t)(quarter * 32 + h * 16) << 16;
    const int q_row0 = qi * block;
    const int q_rows = min(block, N - q_row0);
    float m_run = -INFINITY, l_run = 0.f;   // this key half's reference max (log2, scaled) / this thread's sum
    int col_next = L > 0 ? cols[0] : 0;
#pragma unroll 1
    for (int j = 0; j < L; ++j) {
      const int b = j % NS;
      const int col = col_next;
      if (j + 1 < L) col_next = cols[j + 1];
      K4_SWAIT(&s_full[b], (j / NS) & 1);
      tc_fence_after();
      uint32_t sr[COLS];
      tmem_ld_rows<COLS, COLS>(tmem + lane_off + b * BN + c * KH, sr);   // keys c*KH + colq*COLS + [0, COLS)
      tmem_ld_wait();
      float* s = reinterpret_cast<float*>(sr);
      const int kv_valid = N - col * block - c * KH - colq * COLS;
      if (kv_valid < COLS) {
#pragma unroll
        for (int e = 0; e < COLS; ++e)
          if (e >= kv_valid) s[e] = -INFINITY;
      }
      if (__any_sync(FULL, m_run == -INFINITY)) {
        // no finite score of this key half seen yet (first block, or a fully masked ragged half): exact max
        const float mx = row_max<COLS>(s) * scale_log2;
        const float mxp = fmaxf(mx, __shfl_xor_sync(FULL, mx, 16));
        if (m_run == -INFINITY) m_run = mxp;
      }
      const float m_e = m_run == -INFINITY ? 0.f : m_run;   // all scores -inf so far: p = 0 for any finite m
      uint32_t pk[COLS / 2];
      float sum = exp_pack<C::EMU, COLS>(s, scale_log2, m_e, pk);
      const bool need = !(sum <= C::OVF);
      if (__any_sync(FULL, need)) {
        const int need_peer = __shfl_xor_sync(FULL, (int)need, 16);
        const bool need_row = need || need_peer != 0;
        float rmax = row_max<COLS>(s) * scale_log2;
        rmax = fmaxf(rmax, __shfl_xor_sync(FULL, rmax, 16));
        const float m_new = need_row ? fmaxf(m_e, rmax) : m_e;
        const float alpha = ex2(m_e - m_new);
        if (need_row) sum = exp_pack<0, COLS>(s, scale_log2, m_new, pk);
        l_run *= alpha;
        m_run = m_new;
        if (j > 0 && __any_sync(FULL, alpha < 1.f)) {
          mbar_wait(&o_done[(j - 1) % NS], ((j - 1) / NS) & 1);   // PV_{j-1} (both halves) has written O
          tc_fence_after();
          constexpr int OH = D / 2, OCH = OH < 32 ? OH : 32;
#pragma unroll
          for (int k = 0; k < OH / OCH; ++k) {
            uint32_t o[OCH];
            tmem_ld_rows<OCH, OH>(tmem + lane_off + C::TMEM_O + c * D + k * OCH, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < OCH; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st_rows<OCH, OH>(tmem + lane_off + C::TMEM_O + c * D + k * OCH, o);
          }
        }
      }
      l_run += sum;
      tmem_st_rows<COLS / 2, COLS / 2>(tmem + lane_off + b * BN + c * KH, pk);   // P^c over its half's columns
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[2 * b + c]);
    }
    // epilogue: merge the two key halves' (m_c, l_c, O_c); warp c writes O columns [c D/2, (c+1) D/2)
    const float l_c = l_run + __shfl_xor_sync(FULL, l_run, 16);
    auto red = reinterpret_cast<float(*)[2][128]>(xch);   // [c][m|l][row]
    if (lane < 16) {
      red[c][0][row] = m_run;
      red[c][1][row] = l_c;
    }
    named_bar_sync(1 + quarter * 2 + h, 64);   // the two key-half warps of these 16 rows
    const float m0 = red[0][0][row], l0 = red[0][1][row], m1 = red[1][0][row], l1 = red[1][1][row];
    const float m = fmaxf(m0, m1);
    const float f0 = m0 == -INFINITY ? 0.f : ex2(m0 - m), f1 = m1 == -INFINITY ? 0.f : ex2(m1 - m);
    const float l = l0 * f0 + l1 * f1;
    const bool valid = row < q_rows;
    const size_t grow = (size_t)bh * N + q_row0 + row;
    constexpr int OQ = D / 4;               // O columns per thread
    if (L > 0) {
      mbar_wait(&o_done[(L - 1) % NS], ((L - 1) / NS) & 1);
      tc_fence_after();
      const float a0 = f0 / l, a1 = f1 / l;
      uint32_t o0[OQ], o1[OQ];
      tmem_ld_rows<OQ, OQ>(tmem + lane_off + C::TMEM_O + c * (D / 2), o0);
      tmem_ld_rows<OQ, OQ>(tmem + lane_off + C::TMEM_O + D + c * (D / 2), o1);
      tmem_ld_wait();
      uint32_t pkd[OQ / 2];
#pragma unroll
      for (int e = 0; e < OQ / 2; ++e)
        pkd[e] = pack_bf16(fmaf(__uint_as_float(o1[2 * e]), a1, __uint_as_float(o0[2 * e]) * a0),
                           fmaf(__uint_as_float(o1[2 * e + 1]), a1, __uint_as_float(o0[2 * e + 1]) * a0));
      if (valid) {
        int4* dst = reinterpret_cast<int4*>(out + grow * D + c * (D / 2) + colq * OQ);
#pragma unroll
        for (int e = 0; e < OQ / 8; ++e) dst[e] = make_int4(pkd[4 * e], pkd[4 * e + 1], pkd[4 * e + 2], pkd[4 * e + 3]);
      }
      if (valid && lse && c == 0 && colq == 0) lse[grow] = (m + __log2f(l)) * 0.69314718055994531f;
    } else if (valid) {
      int4* dst = reinterpret_cast<int4*>(out + grow * D + c * (D / 2) + colq * OQ);
#pragma unroll
      for (int e = 0; e < OQ / 8; ++e) dst[e] = make_int4(0, 0, 0, 0);
      if (lse && c == 0 && colq == 0) lse[grow] = -INFINITY;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem);
  }
}

// ================================================================================================
// Paired query blocks: one CTA per (b, h, pair of query blocks 2p, 2p+1).
// Adjacent rows of the MOD-DiT mask share most of their index lists (vertical columns, frame
// squares, diagonals whose neighbour offset is also selected: 79 % at Hunyuan 720p, Family S), so the
// two query tiles A = block 2p and B = block 2p+1 walk the MERGED list ("stream") of their columns:
// each stream entry's K/V tile is fetched ONCE and feeds S and PV of every tile whose list holds it.
// FLOPs are exactly those of the selected blocks (a column in one list only is computed for that
// tile only), while L2->SMEM K/V traffic and TMA/barrier work per block drop by the shared fraction.
//   warp 0      producer: Q_A, Q_B once; then K(u), V(u) for stream entries u (K one entry ahead).
//   warp 1      single-thread tcgen05 issuer.  Per stream entry u, for each tile X holding u:
//                  [wait P_X(prev)] PV_X(prev) -> O_X ;  S_X(u) = Q_X K(u)^T -> S_X
//               (the FA4-style interleave when both tiles hold u; the single kernel's split-KV order
//               when the lists alternate).  A PV still pending two entries back is issued first, so
//               its V slot can be refilled (no deadlock however the lists interleave).
//   warps 2..5  softmax of tile A, warps 6..9 softmax of tile B (thread = query row), as in the
//               single kernel; P overwrites S_X in TMEM; each tile owns O_X, so no split-KV merge.
// TMEM: S_A [0,BN), S_B [BN,2BN), O_A [2BN,2BN+D), O_B [2BN+D,2BN+2D).
template <int D, int BN>
struct PairCfg {
  static constexpr int BM = 128;
  static constexpr int Q_BOX = BM * 128, KV_BOX = BN * 128, NATOM = D / 64;
  static constexpr int Q_BYTES = Q_BOX * NATOM, KV_BYTES = KV_BOX * NATOM;
  static constexpr int OFF_Q = 0;                          // Q_A, Q_B
  static constexpr int OFF_K = OFF_Q + 2 * Q_BYTES;       // 2 slots, slot = u & 1
  static constexpr int OFF_V = OFF_K + 2 * KV_BYTES;      // 2 slots, slot = u & 1
  static constexpr int OFF_BAR = OFF_V + 2 * KV_BYTES;
  // q_full, k_full[2], k_empty[2], v_full[2], v_empty[2], s_full[2], p_full[2], o_done[2], tmem slot
  static constexpr int NUM_BARS = 1 + 2 * 7;
  static constexpr int OFF_LIST = OFF_BAR + NUM_BARS * 8 + 16;   // uint16 columns of A then B
  static constexpr int MAX_LIST = (232448 - OFF_LIST) / 4;       // per tile
  static constexpr int SMEM_BASE = OFF_LIST;
  static constexpr int TMEM_S = 0, TMEM_O = 2 * BN;
  static constexpr uint32_t TMEM_COLS = (2 * BN + 2 * D) <= 256 ? 256 : 512;
  static constexpr uint32_t IDESC_S = idesc_bf16_f32(BM, BN, false, false);
  static constexpr uint32_t IDESC_O = idesc_bf16_f32(BM, D, false, true);
  static constexpr int THREADS = 320;
};

template <int D, int BN>
__global__ void __launch_bounds__(320, 1)
    attn_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const int* __restrict__ row_ptr,
                     const int* __restrict__ col_idx, __nv_bfloat16* __restrict__ out, float* __restrict__ lse,
                     int N, int n, float scale_log2) {
  using C = PairCfg<D, BN>;
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + 2;
  uint64_t* v_full = k_empty + 2;
  uint64_t* v_empty = v_full + 2;
  uint64_t* s_full = v_empty + 2;   // [tile]
  uint64_t* p_full = s_full + 2;    // [tile]
  uint64_t* o_done = p_full + 2;    // [tile]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);
  uint16_t* lists = reinterpret_cast<uint16_t*>(smem + C::OFF_LIST);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int npair = (n + 1) >> 1;
  const int bh = blockIdx.x / npair, qa = 2 * (blockIdx.x % npair), qb = qa + 1;
  const int* rp = row_ptr + (size_t)bh * (n + 1);
  const int begA = rp[qa], LA = rp[qa + 1] - begA;
  const int begB = qb < n ? rp[qb] : 0, LB = qb < n ? rp[qb + 1] - begB : 0;
  const int* colsA = col_idx + (size_t)bh * n * n + begA;
  const int* colsB = col_idx + (size_t)bh * n * n + begB;
  uint16_t* la = lists;
  uint16_t* lb = lists + LA;
  for (int t = threadIdx.x; t < LA + LB; t += blockDim.x) lists[t] = (uint16_t)(t < LA ? colsA[t] : colsB[t - LA]);
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 128);
      mbar_init(&o_done[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const bool any = LA + LB > 0;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (stream order)
    if (lane == 0 && any) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
      mbar_arrive_expect_tx(q_full, (LB > 0 ? 2 : 1) * C::Q_BYTES);
#pragma unroll
      for (int a = 0; a < C::NATOM; ++a)
        tma_load_3d(smem + C::OFF_Q + a * C::Q_BOX, &tm_q, q_full, a * 64, qa * BN, bh, pol_q);
      if (LB > 0) {
#pragma unroll
        for (int a = 0; a < C::NATOM; ++a)
          tma_load_3d(smem + C::OFF_Q + C::Q_BYTES + a * C::Q_BOX, &tm_q, q_full, a * 64, qb * BN, bh, pol_q);
      }
      auto load = [&](uint64_t* full, uint64_t* empty, int off, const CUtensorMap* tm, int u, int col) {
        const int s = u & 1;
        if (u >= 2) mbar_wait(&empty[s], ((u >> 1) - 1) & 1);   // entry u-2 released the slot
        unsigned char* dst = smem + off + s * C::KV_BYTES;
        mbar_arrive_expect_tx(&full[s], C::KV_BYTES);
#pragma unroll
        for (int a = 0; a < C::NATOM; ++a) tma_load_3d(dst + a * C::KV_BOX, tm, &full[s], a * 64, col * BN, bh, pol_kv);
      };
      // walk the merged stream; K runs one entry ahead of V (the issuer's demand order)
      int ia = 0, ib = 0, u = 0, vcol_prev = -1;
      while (ia < LA || ib < LB) {
        const int ca = ia < LA ? la[ia] : 0x7fffffff, cb = ib < LB ? lb[ib] : 0x7fffffff;
        const int c = min(ca, cb);
        ia += ca == c;
        ib += cb == c;
        load(k_full, k_empty, C::OFF_K, &tm_k, u, c);
        if (u >= 1) load(v_full, v_empty, C::OFF_V, &tm_v, u - 1, vcol_prev);
        vcol_prev = c;
        ++u;
      }
      load(v_full, v_empty, C::OFF_V, &tm_v, u - 1, vcol_prev);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && any) {
      const uint32_t sq = smem_u32(smem + C::OFF_Q);
      mbar_wait(q_full, 0);
      // scalar state (no dynamically indexed arrays: they would live in local memory)
      int pend0 = -1, pend1 = -1;      // stream entry of tile X's issued S whose PV is still due
      int npv0 = 0, npv1 = 0;          // PVs issued per tile (phase of p_full[X])
      int vrem0 = 0, vrem1 = 0;        // PVs still to read V slot 0 / 1
      auto emit_pv = [&](int X) {
        const int e = X ? pend1 : pend0, s = e & 1;
        const int np = X ? npv1 : npv0;
        mbar_wait(&v_full[s], (e >> 1) & 1);
        mbar_wait(&p_full[X], np & 1);
        tc_fence_after();
        const uint32_t sv = smem_u32(smem + C::OFF_V + s * C::KV_BYTES);
        const uint32_t p_t = tmem + C::TMEM_S + X * BN;
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          const uint64_t bd = smem_desc_sw128(sv + kk * 2048, C::KV_BOX, 1024);
          mma_ts(tmem + C::TMEM_O + X * D, p_t + kk * 8, bd, C::IDESC_O, (np > 0 || kk > 0) ? 1u : 0u);
        }
        if (np + 1 == (X ? LB : LA)) mma_commit(&o_done[X]);   // only the tile's last PV is waited (epilogue)
        const int left = s ? --vrem1 : --vrem0;
        if (left == 0) mma_commit(&v_empty[s]);
        if (X) { pend1 = -1; ++npv1; } else { pend0 = -1; ++npv0; }
      };
      bool kwait = false;              // K(u) already waited for by this entry's first S
      auto emit_s = [&](int X, int u) {
        if (!kwait) {
          mbar_wait(&k_full[u & 1], (u >> 1) & 1);
          kwait = true;
        }
        const uint32_t sk = smem_u32(smem + C::OFF_K + (u & 1) * C::KV_BYTES);
        const uint32_t qx = sq + X * C::Q_BYTES;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t ad = smem_desc_sw128(qx + (kk / 4) * C::Q_BOX + (kk % 4) * 32, 16, 1024);
          const uint64_t bd = smem_desc_sw128(sk + (kk / 4) * C::KV_BOX + (kk % 4) * 32, 16, 1024);
          mma_ss(tmem + C::TMEM_S + X * BN, ad, bd, C::IDESC_S, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[X]);
        if (X) pend1 = u; else pend0 = u;
      };
      // the older pending PV first (V slots drain in stream order); only those at or before `lim`
      auto drain = [&](int lim) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const bool x0 = pend0 >= 0 && (pend1 < 0 || pend0 <= pend1);
          const int e = x0 ? pend0 : pend1;
          if (e >= 0 && e <= lim) emit_pv(x0 ? 0 : 1);
        }
      };
      int ia = 0, ib = 0, u = 0;
      while (ia < LA || ib < LB) {
        const int ca = ia < LA ? la[ia] : 0x7fffffff, cb = ib < LB ? lb[ib] : 0x7fffffff;
        const int c = min(ca, cb);
        const bool fa = ca == c, fb = cb == c;
        ia += fa;
        ib += fb;
        // V slot (u & 1) is refilled with V(u) once entry u-2's PVs are done: issue any still pending
        drain(u - 2);
        if (u & 1) vrem1 = (int)fa + (int)fb; else vrem0 = (int)fa + (int)fb;
        kwait = false;
        // FA4-style interleave when both lists hold u: PV_A, S_A(u), PV_B, S_B(u)
        if (fa) {
          if (pend0 >= 0) emit_pv(0);
          emit_s(0, u);
        }
        if (fb) {
          if (pend1 >= 0) emit_pv(1);
          emit_s(1, u);
        }
        mma_commit(&k_empty[u & 1]);   // both S of entry u issued: K slot free once they complete
        ++u;
      }
      drain(0x7fffffff);
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue, tile X = (warp-2)/4
    const int X = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t t_s = tmem + lane_off + C::TMEM_S + X * BN;
    const uint32_t t_o = tmem + lane_off + C::TMEM_O + X * D;
    const int qx = X ? qb : qa;
    const int LX = X ? LB : LA;
    const uint16_t* lx = X ? lb : la;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < LX; ++j) {
      mbar_wait(&s_full[X], j & 1);
      tc_fence_after();
      uint32_t sr[BN];
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) tmem_ld32(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
      tmem_ld_wait();
      float* s = reinterpret_cast<float*>(sr);
      const int kv_valid = N - (int)lx[j] * BN;
      if (kv_valid < BN) {
#pragma unroll
        for (int c = 0; c < BN; ++c)
          if (c >= kv_valid) s[c] = -INFINITY;
      }
      float mxv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mxv[u] = s[u];
#pragma unroll
      for (int c = 8; c < BN; c += 8)
#pragma unroll
        for (int u = 0; u < 8; ++u) mxv[u] = fmaxf(mxv[u], s[c + u]);
      const float mx = fmaxf(fmaxf(fmaxf(mxv[0], mxv[1]), fmaxf(mxv[2], mxv[3])),
                             fmaxf(fmaxf(mxv[4], mxv[5]), fmaxf(mxv[6], mxv[7])));
      const float m_new = fmaxf(m_run, mx * scale_log2);
      const bool rescale = (m_new - m_run) > 8.0f;
      const float m_use = rescale ? m_new : m_run;
      const float alpha = rescale ? ex2(m_run - m_new) : 1.0f;
      const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m_use, -m_use);
      float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      uint32_t pk[BN / 2];
#pragma unroll
      for (int c = 0; c < BN; c += 2) {
        const float2 x = ffma2(make_float2(s[c], s[c + 1]), sc2, nm2);
        float2 p;
        if (((c / 2) & 7) < kEmuPairsPer8) {
          p = ex2_poly2(x);
        } else {
          p.x = ex2(x.x);
          p.y = ex2(x.y);
        }
        acc2[(c / 2) & 1] = fadd2(acc2[(c / 2) & 1], p);
        pk[c / 2] = pack_bf16(p.x, p.y);
      }
      l_run = fmaf(l_run, alpha, (acc2[0].x + acc2[0].y) + (acc2[1].x + acc2[1].y));
      m_run = m_use;
#pragma unroll
      for (int c = 0; c < BN / 64; ++c) tmem_st32(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[c * 32]));
      // S_X(j) was issued after PV_X(j-1), so s_full above already implies O_X holds PV_X(j-1)
      if (j >= 1 && __any_sync(0xffffffffu, rescale)) {
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t o[32];
          tmem_ld32(t_o + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
          tmem_st32(t_o + c * 32, o);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[X]);
    }
    // epilogue: O_X / l -> bf16, lse (no merge: each tile owns its accumulator)
    if (qx < n) {
      const int q_row0 = qx * BN;
      const bool valid = row < min(BN, N - q_row0);
      const size_t grow = (size_t)bh * N + q_row0 + row;
      if (LX > 0) {
        mbar_wait(&o_done[X], 0);   // committed once, after the tile's last PV
        tc_fence_after();
        const float inv = 1.0f / l_run;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t o[32];
          tmem_ld32(t_o + c * 32, o);
          tmem_ld_wait();
          uint32_t pkd[16];
#pragma unroll
          for (int e = 0; e < 16; ++e)
            pkd[e] = pack_bf16(__uint_as_float(o[2 * e]) * inv, __uint_as_float(o[2 * e + 1]) * inv);
          if (valid) {
            int4* dst = reinterpret_cast<int4*>(out + grow * D + c * 32);
#pragma unroll
            for (int e = 0; e < 4; ++e) dst[e] = make_int4(pkd[4 * e], pkd[4 * e + 1], pkd[4 * e + 2], pkd[4 * e + 3]);
          }
        }
        if (valid && lse) lse[grow] = (m_run + __log2f(l_run)) * 0.69314718055994531f;
      } else if (valid) {
        int4* dst = reinterpret_cast<int4*>(out + grow * D);
#pragma unroll
        for (int e = 0; e < D / 8; ++e) dst[e] = make_int4(0, 0, 0, 0);
        if (lse) lse[grow] = -INFINITY;
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

// The tensor map tma_load_tile expects: 3D {D, N, BH} with {64, rows, 1} boxes, or for D = 128 with K4_TMA4D
// the 4D view {64, N, 2, BH} (strides D*2, 128, N*D*2 bytes) with {64, rows, 2, 1} boxes.
mod_status make_map_tile(CUtensorMap* m, const void* base, int BH, int N, int D, int rows) {
  if (!(K4_TMA4D && D == 128)) return make_map(m, base, BH, N, D, rows);
  auto enc = get_encode();
  MOD_REQUIRE(enc, MOD_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled driver entry point unavailable");
  MOD_REQUIRE(((uintptr_t)base & 127) == 0, MOD_ERR_INPUT, "Q/K/V pointers must be 128-byte aligned");
  cuuint64_t dims[4] = {64, (cuuint64_t)N, 2, (cuuint64_t)BH};
  cuuint64_t strides[3] = {(cuuint64_t)D * 2, 128, (cuuint64_t)N * D * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)rows, 2, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MOD_REQUIRE(r == CUDA_SUCCESS, MOD_ERR_CUDA, "cuTensorMapEncodeTiled (4D tile view) failed (%d)", (int)r);
  return MOD_OK;
}

// One launcher for the single-query-block schedules (DEFAULT, SPLITKV): grid = (b, h, query block).
template <typename Cfg, typename Kern>
mod_status launch_rows(mod_plan P, Kern kern, int D, int BN, const void* q, const void* k, const void* v,
                       const int* row_ptr, const int* col_idx, void* o, float* lse, cudaStream_t s) {
  const int BH = P->L.batch * P->L.heads;
  CUtensorMap tq, tk, tv;
  mod_status st;
  if ((st = make_map(&tq, q, BH, P->N, D, Cfg::BM)) != MOD_OK) return st;
  if ((st = make_map(&tk, k, BH, P->N, D, BN)) != MOD_OK) return st;
  if ((st = make_map(&tv, v, BH, P->N, D, BN)) != MOD_OK) return st;
  MOD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const float scale_log2 = P->scale * 1.4426950408889634f;
  kern<<<BH * P->n, Cfg::THREADS, Cfg::SMEM, s>>>(tq, tk, tv, row_ptr, col_idx, (__nv_bfloat16*)o, lse, P->N, P->n,
                                                  P->L.block, scale_log2);
  MOD_LAUNCH_CHECK();
  return MOD_OK;
}

template <int D, int BN>
mod_status launch_default(mod_plan P, const void* q, const void* k, const void* v, const int* row_ptr,
                          const int* col_idx, void* o, float* lse, cudaStream_t s) {
  using Cfg = Attn1Cfg<D, BN>;
  const int BH = P->L.batch * P->L.heads;
  CUtensorMap tq, tk, tv;
  mod_status st;
  if ((st = make_map_tile(&tq, q, BH, P->N, D, Cfg::BM)) != MOD_OK) return st;
  if ((st = make_map_tile(&tk, k, BH, P->N, D, BN)) != MOD_OK) return st;
  if ((st = make_map_tile(&tv, v, BH, P->N, D, BN)) != MOD_OK) return st;
  auto kern = attn_fwd_kernel<D, BN>;
  MOD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const float scale_log2 = P->scale * 1.4426950408889634f;
  kern<<<BH * P->n, Cfg::THREADS, Cfg::SMEM, s>>>(tq, tk, tv, row_ptr, col_idx, (__nv_bfloat16*)o, lse, P->N, P->n,
                                                  P->L.block, scale_log2);
  MOD_LAUNCH_CHECK();
  return MOD_OK;
}

template <int D, int BN>
mod_status launch_wide(mod_plan P, const void* q, const void* k, const void* v, const int* row_ptr,
                       const int* col_idx, void* o, float* lse, cudaStream_t s) {
  return launch_rows<WideCfg<D, BN>>(P, attn_wide_kernel<D, BN>, D, BN, q, k, v, row_ptr, col_idx, o, lse, s);
}

template <int D, int BN>
mod_status launch_split(mod_plan P, const void* q, const void* k, const void* v, const int* row_ptr,
                        const int* col_idx, void* o, float* lse, cudaStream_t s) {
  return launch_rows<SplitCfg<D, BN>>(P, attn_split_kernel<D, BN>, D, BN, q, k, v, row_ptr, col_idx, o, lse, s);
}

template <int D>
mod_status launch_pair(mod_plan P, const void* q, const void* k, const void* v, const int* row_ptr, const int* col_idx,
                       void* o, float* lse, cudaStream_t s) {
  using C = PairCfg<D, 128>;
  const int BH = P->L.batch * P->L.heads;
  CUtensorMap tq, tk, tv;
  mod_status st;
  if ((st = make_map(&tq, q, BH, P->N, D, C::BM)) != MOD_OK) return st;
  if ((st = make_map(&tk, k, BH, P->N, D, 128)) != MOD_OK) return st;
  if ((st = make_map(&tv, v, BH, P->N, D, 128)) != MOD_OK) return st;
  // two index lists of at most n uint16 columns each follow the barriers
  const int smem = C::SMEM_BASE + 4 * P->n;
  auto kern = attn_pair_kernel<D, 128>;
  MOD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const float scale_log2 = P->scale * 1.4426950408889634f;
  const int npair = (P->n + 1) / 2;
  kern<<<BH * npair, C::THREADS, smem, s>>>(tq, tk, tv, row_ptr, col_idx, (__nv_bfloat16*)o, lse, P->N, P->n,
                                            scale_log2);
  MOD_LAUNCH_CHECK();
  return MOD_OK;
}

// The schedule a plan runs: its config's attn_kernel where that variant supports the layout (pair:
// 128-token blocks, both lists in shared memory), else the default.
int effective_kernel(mod_plan P) {
  const int want = P->cfg.attn_kernel;
  if (want == MOD_ATTN_PAIR) {
    const int cap = P->L.head_dim == 128 ? PairCfg<128, 128>::MAX_LIST : PairCfg<64, 128>::MAX_LIST;
    if (P->L.block == 128 && P->n <= cap && P->n <= 65535) return MOD_ATTN_PAIR;
    return MOD_ATTN_DEFAULT;
  }
  if (want == MOD_ATTN_WIDE) return P->L.block == 128 ? MOD_ATTN_WIDE : MOD_ATTN_DEFAULT;
  // the default schedule by shape: at D = 64 the tensor work per block halves and the softmax alone bounds
  // the kernel; the wide schedule's four softmax warps per sub-partition hide its latencies better there
  // (CogVideoX-5B: 598 vs 559 TFLOP/s), while at D = 128 the 8-warp schedule with three S buffers is faster
  // (1212 vs 1161 TFLOP/s at Hunyuan; profiles/r2/README.md)
  if (want == MOD_ATTN_DEFAULT && P->L.head_dim == 64 && P->L.block == 128) return MOD_ATTN_WIDE;
  return want;
}
}  // namespace

#ifdef MOD_K4_TRACE
// trace builds only: copy out the event stamps [kTrCtas][18][kTrBlocks][6] and the CTA spans [n][4]
extern "C" int mod_debug_k4_trace(long long* ev, long long* span, int n_span) {
  cudaMemcpyFromSymbol(ev, g_k4_ev, sizeof(g_k4_ev));
  cudaMemcpyFromSymbol(span, g_k4_span, sizeof(long long) * 4 * (size_t)n_span);
  return kTrBlocks;
}
#endif


extern "C" const char* mod_attn_kernel_name(mod_plan P) {
  if (mod_validate_plan(P) != MOD_OK) return "";
  const int D = P->L.head_dim, BN = P->L.block;
  switch (effective_kernel(P)) {
    case MOD_ATTN_SPLITKV:
      return D == 128 ? (BN == 128 ? "attn_split_kernel<128,128>" : "attn_split_kernel<128,64>")
                      : (BN == 128 ? "attn_split_kernel<64,128>" : "attn_split_kernel<64,64>");
    case MOD_ATTN_PAIR: return D == 128 ? "attn_pair_kernel<128,128>" : "attn_pair_kernel<64,128>";
    case MOD_ATTN_WIDE: return D == 128 ? "attn_wide_kernel<128,128>" : "attn_wide_kernel<64,128>";
    default:
      return D == 128 ? (BN == 128 ? "attn_fwd_kernel<128,128>" : "attn_fwd_kernel<128,64>")
                      : (BN == 128 ? "attn_fwd_kernel<64,128>" : "attn_fwd_kernel<64,64>");
  }
}

extern "C" mod_status mod_block_sparse_attn_fwd(mod_plan P, const void* q, const void* k, const void* v,
                                                const int32_t* row_ptr, const int32_t* col_idx, void* o, float* lse,
                                                void* ws, void* stream) {
  MOD_NVTX("mod_block_sparse_attn_fwd");
  (void)ws;
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  MOD_REQUIRE(q && k && v && row_ptr && col_idx && o, MOD_ERR_USAGE,
              "mod_block_sparse_attn_fwd: q, k, v, row_ptr, col_idx, o must be non-NULL");
  MOD_REQUIRE(((uintptr_t)o & 15) == 0, MOD_ERR_INPUT, "o must be 16-byte aligned");
  cudaStream_t s = as_stream(stream);
  const int D = P->L.head_dim, BN = P->L.block;
  switch (effective_kernel(P)) {
    case MOD_ATTN_PAIR:
      st = D == 128 ? launch_pair<128>(P, q, k, v, row_ptr, col_idx, o, lse, s)
                    : launch_pair<64>(P, q, k, v, row_ptr, col_idx, o, lse, s);
      break;
    case MOD_ATTN_WIDE:
      st = D == 128 ? launch_wide<128, 128>(P, q, k, v, row_ptr, col_idx, o, lse, s)
                    : launch_wide<64, 128>(P, q, k, v, row_ptr, col_idx, o, lse, s);
      break;
    case MOD_ATTN_SPLITKV:
      if (D == 128 && BN == 128) st = launch_split<128, 128>(P, q, k, v, row_ptr, col_idx, o, lse, s);
      else if (D == 64 && BN == 128) st = launch_split<64, 128>(P, q, k, v, row_ptr, col_idx, o, lse, s);
      else if (D == 128 && BN == 64) st = launch_split<128, 64>(P, q, k, v, row_ptr, col_idx, o, lse, s);
      else st = launch_split<64, 64>(P, q, k, v, row_ptr, col_idx, o, lse, s);
      break;
    default:
      if (D == 128 && BN == 128) st = launch_default<128, 128>(P, q, k, v, row_ptr, col_idx, o, lse, s);
      else if (D == 64 && BN == 128) st = launch_default<64, 128>(P, q, k, v, row_ptr, col_idx, o, lse, s);
      else if (D == 128 && BN == 64) st = launch_default<128, 64>(P, q, k, v, row_ptr, col_idx, o, lse, s);
      else st = launch_default<64, 64>(P, q, k, v, row_ptr, col_idx, o, lse, s);
  }
  if (st == MOD_OK) mod_note_launches(1);
  return st;
}
