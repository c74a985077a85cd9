// ulysses.cu -- relayout kernels around the Ulysses all-to-all (BASELINE config 5).
//
// When DiT activations arrive sequence-sharded over P ranks ([B, N/P, H, D] per rank), the hot path
// (per head: PAPER.md §4.1 P:202 "We process each attention head independently") needs head shards
// [B, H/P, N, D].  The exchange is an all-to-all (NCCL all_to_all_single on contiguous per-peer
// chunks); these kernels are the pack before it and the unpack after it, in both directions, so that
// no PyTorch permute runs on the data path.  Each is a permutation of D-element bf16 rows (HBM-bound:
// one read and one write of the tensor), enumerated in destination order with 16-byte vectors so that
// writes are fully coalesced and reads move whole 2*D-byte rows.
//
// Row maps (p = peer / chunk, b = batch, s = token within a chunk of Ns, h = head, hp = head within a
// group of Hp = H/P):
//   SEQ_PACK    x_seq [B,Ns,H,D]   -> send [P,B,Ns,Hp,D]   (p,b,s,hp) <- (b,s,p*Hp+hp)
//   SEQ_UNPACK  recv  [P,B,Ns,Hp,D] -> x_head [B,Hp,P*Ns,D] (b,hp,p*Ns+s) <- (p,b,s,hp)
//   HEAD_PACK   x_head [B,Hp,P*Ns,D] -> send [P,B,Ns,Hp,D] (p,b,s,hp) <- (b,hp,p*Ns+s)
//   HEAD_UNPACK recv  [P,B,Ns,Hp,D] -> x_seq [B,Ns,P*Hp,D] (b,s,p*Hp+hp) <- (p,b,s,hp)
// With P = 1 the pack/unpack pair collapses to the [B,N,H,D] <-> [B,H,N,D] transpose.
#include "common.cuh"

namespace {

enum { SEQ_PACK = 0, SEQ_UNPACK = 1, HEAD_PACK = 2, HEAD_UNPACK = 3 };

// 32-bit row arithmetic (the host checks rows < 2^31): 64-bit divisions would dominate the copy.
// Ht / h0: the x_seq side may hold more heads than the exchanged group -- SEQ_PACK reads heads
// [h0, h0 + P*Hp) of an [B, Ns, Ht] source and HEAD_UNPACK writes them into an [B, Ns, Ht] destination
// (the head chunks of the overlapped Ulysses pipeline, parallel.py); Ht = P*Hp, h0 = 0 is the whole tensor.
template <int MODE>
__device__ __forceinline__ uint32_t src_row(uint32_t r, uint32_t B, uint32_t Ns, uint32_t Hp, uint32_t P,
                                            uint32_t Ht, uint32_t h0) {
  if (MODE == SEQ_PACK || MODE == HEAD_PACK) {
    // destination [P, B, Ns, Hp]
    const uint32_t hp = r % Hp;
    uint32_t t = r / Hp;
    const uint32_t s = t % Ns;
    t /= Ns;
    const uint32_t b = t % B, p = t / B;
    if (MODE == SEQ_PACK) return (b * Ns + s) * Ht + h0 + p * Hp + hp;    // x_seq [B,Ns,Ht]
    return (b * Hp + hp) * (P * Ns) + p * Ns + s;                         // x_head [B,Hp,N]
  } else if (MODE == SEQ_UNPACK) {
    // destination [B, Hp, P*Ns]
    const uint32_t N = P * Ns;
    const uint32_t tok = r % N, t = r / N;
    const uint32_t hp = t % Hp, b = t / Hp;
    const uint32_t p = tok / Ns, s = tok % Ns;
    return ((p * B + b) * Ns + s) * Hp + hp;                              // recv [P,B,Ns,Hp]
  } else {
    // HEAD_UNPACK, destination [B, Ns, P*Hp]
    const uint32_t H = P * Hp;
    const uint32_t h = r % H, t = r / H;
    const uint32_t s = t % Ns, b = t / Ns;
    const uint32_t p = h / Hp, hp = h % Hp;
    return ((p * B + b) * Ns + s) * Hp + hp;                              // recv [P,B,Ns,Hp]
  }
}

// destination row index of enumerated row r: identity except for HEAD_UNPACK into a wider x_seq
template <int MODE>
__device__ __forceinline__ uint32_t dst_row(uint32_t r, uint32_t Hp, uint32_t P, uint32_t Ht, uint32_t h0) {
  if (MODE != HEAD_UNPACK) return r;
  const uint32_t H = P * Hp;
  return (r / H) * Ht + h0 + r % H;
}

template <int MODE, int VPR>   // VPR = 16-byte vectors per row (D / 8)
__global__ void __launch_bounds__(256) relayout_kernel(const int4* __restrict__ src, int4* __restrict__ dst,
                                                       uint32_t rows, uint32_t B, uint32_t Ns, uint32_t Hp,
                                                       uint32_t P, uint32_t Ht, uint32_t h0) {
  // one row per VPR consecutive threads; 4 rows in flight per thread for memory-level parallelism
  constexpr int UNROLL = 4;
  const uint32_t c = threadIdx.x % VPR;
  const uint32_t rows_per_block = blockDim.x / VPR;
  for (uint32_t r0 = blockIdx.x * rows_per_block * UNROLL + threadIdx.x / VPR; r0 < rows;
       r0 += gridDim.x * rows_per_block * UNROLL) {
    int4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint32_t r = r0 + u * rows_per_block;
      if (r < rows) v[u] = __ldcs(src + (size_t)src_row<MODE>(r, B, Ns, Hp, P, Ht, h0) * VPR + c);   // read once
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint32_t r = r0 + u * rows_per_block;
      if (r < rows) __stcs(dst + (size_t)dst_row<MODE>(r, Hp, P, Ht, h0) * VPR + c, v[u]);
    }
  }
}

template <int MODE>
mod_status launch(const void* src, void* dst, int B, int Ns, int Hp, int D, int P, void* stream, int Ht = -1,
                  int h0 = 0) {
  if (Ht < 0) Ht = P * Hp;
  MOD_REQUIRE(h0 >= 0 && h0 + P * Hp <= Ht, MOD_ERR_INPUT, "ulysses relayout: heads [%d, %d) outside the %d heads",
              h0, h0 + P * Hp, Ht);
  MOD_REQUIRE((size_t)B * Ns * Ht < (1ull << 31), MOD_ERR_INPUT, "ulysses relayout: x_seq rows exceed 2^31");
  MOD_REQUIRE(src && dst, MOD_ERR_USAGE, "ulysses relayout: src and dst must be non-NULL");
  MOD_REQUIRE(B >= 1 && Ns >= 1 && Hp >= 1 && P >= 1, MOD_ERR_INPUT,
              "ulysses relayout: B=%d Ns=%d Hp=%d P=%d must all be >= 1", B, Ns, Hp, P);
  MOD_REQUIRE(D == 64 || D == 128, MOD_ERR_INPUT, "ulysses relayout: head_dim=%d must be 64 or 128", D);
  MOD_REQUIRE(src != dst, MOD_ERR_INPUT, "ulysses relayout: src and dst must not alias");
  MOD_REQUIRE((((uintptr_t)src | (uintptr_t)dst) & 15) == 0, MOD_ERR_INPUT,
              "ulysses relayout: src and dst must be 16-byte aligned");
  mod_status st = mod_check_sticky();
  if (st != MOD_OK) return st;
  const size_t rows = (size_t)P * B * Ns * Hp;
  MOD_REQUIRE(rows < (1ull << 31), MOD_ERR_INPUT, "ulysses relayout: %zu rows exceed the 2^31 row limit", rows);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t rows_per_cta = (256 / (D / 8)) * 4;
  const int grid = (int)std::min<size_t>((rows + rows_per_cta - 1) / rows_per_cta, (size_t)sms * 8);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (D == 128)
    relayout_kernel<MODE, 16><<<grid, 256, 0, s>>>((const int4*)src, (int4*)dst, (uint32_t)rows, B, Ns, Hp, P, Ht, h0);
  else
    relayout_kernel<MODE, 8><<<grid, 256, 0, s>>>((const int4*)src, (int4*)dst, (uint32_t)rows, B, Ns, Hp, P, Ht, h0);
  MOD_LAUNCH_CHECK();
  mod_note_launches(1);
  return MOD_OK;
}

}  // namespace

extern "C" mod_status mod_ulysses_seq_pack(const void* x_seq, void* send, int32_t B, int32_t Ns, int32_t H,
                                           int32_t D, int32_t P, void* stream) {
  MOD_NVTX("mod_ulysses_seq_pack");
  MOD_REQUIRE(P >= 1 && H % P == 0, MOD_ERR_INPUT, "mod_ulysses_seq_pack: heads=%d not divisible by P=%d", H, P);
  return launch<SEQ_PACK>(x_seq, send, B, Ns, H / P, D, P, stream);
}

extern "C" mod_status mod_ulysses_seq_unpack(const void* recv, void* x_head, int32_t B, int32_t Ns, int32_t Hp,
                                             int32_t D, int32_t P, void* stream) {
  MOD_NVTX("mod_ulysses_seq_unpack");
  return launch<SEQ_UNPACK>(recv, x_head, B, Ns, Hp, D, P, stream);
}

extern "C" mod_status mod_ulysses_head_pack(const void* x_head, void* send, int32_t B, int32_t N, int32_t Hp,
                                            int32_t D, int32_t P, void* stream) {
  MOD_NVTX("mod_ulysses_head_pack");
  MOD_REQUIRE(P >= 1 && N % P == 0, MOD_ERR_INPUT, "mod_ulysses_head_pack: tokens=%d not divisible by P=%d", N, P);
  return launch<HEAD_PACK>(x_head, send, B, N / P, Hp, D, P, stream);
}

extern "C" mod_status mod_ulysses_head_unpack(const void* recv, void* x_seq, int32_t B, int32_t Ns, int32_t Hp,
                                              int32_t D, int32_t P, void* stream) {
  MOD_NVTX("mod_ulysses_head_unpack");
  return launch<HEAD_UNPACK>(recv, x_seq, B, Ns, Hp, D, P, stream);
}

// Head-chunk variants (the overlapped Ulysses pipeline): pack heads [h0, h0 + Hc) of an H-head x_seq, and
// unpack into heads [h0, h0 + P*Hp) of an H-head x_seq.
extern "C" mod_status mod_ulysses_seq_pack_heads(const void* x_seq, void* send, int32_t B, int32_t Ns, int32_t H,
                                                 int32_t h0, int32_t Hc, int32_t D, int32_t P, void* stream) {
  MOD_NVTX("mod_ulysses_seq_pack_heads");
  MOD_REQUIRE(P >= 1 && Hc >= 1 && Hc % P == 0, MOD_ERR_INPUT,
              "mod_ulysses_seq_pack_heads: chunk of %d heads not divisible by P=%d", Hc, P);
  return launch<SEQ_PACK>(x_seq, send, B, Ns, Hc / P, D, P, stream, H, h0);
}

extern "C" mod_status mod_ulysses_head_unpack_heads(const void* recv, void* x_seq, int32_t B, int32_t Ns, int32_t Hp,
                                                    int32_t D, int32_t P, int32_t H, int32_t h0, void* stream) {
  MOD_NVTX("mod_ulysses_head_unpack_heads");
  return launch<HEAD_UNPACK>(recv, x_seq, B, Ns, Hp, D, P, stream, H, h0);
}
