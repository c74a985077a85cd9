/*
 * moddit_step.c -- one re-estimation step of MOD-DiT's hot path (Algorithm 1)
 * driven from plain C through include/moddit.h: no Python, no PyTorch.  Demonstrates the boundary:
 * the caller owns every device buffer (cudaMalloc), passes raw pointers and a stream, and checks the
 * returned mod_status.
 *
 *   moddit_step <B> <H> <D> <prefix> <F> <Hh> <Ww> <block> <top_k> <in.bin> <out.bin>
 *
 * in.bin  : Q, K, V (bf16 [B,H,N,D] each, in that order) followed by Q', K' of the previous step
 *           (the statistic at t = m-1).
 * out.bin : O (bf16 [B,H,N,D]), lse (fp32 [B,H,N]), row_ptr (int32 [B,H,n+1]), then the refitted
 *           x_curr (fp64 [B,H,p]).
 * The step: W1 = stats(Q', K'), W2 = stats(Q, K); x_prev = fit(W1), x_curr = fit(W2);
 * keep = keep_frames(x_prev, x_curr); mask = predict(x_prev, x_curr, t_prev=11, t_curr=12, t=13);
 * O, lse = attention(Q, K, V, mask); update(stats(Q, K), mask, hist = W2, x_prev, x_curr).
 * Exit code: 0 on success, otherwise the failing mod_status (or 10 + errno-like codes for I/O).
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "moddit.h"

#define CHECK(call)                                                                        \
  do {                                                                                     \
    mod_status s_ = (call);                                                                \
    if (s_ != MOD_OK) {                                                                    \
      fprintf(stderr, "%s failed (%d): %s\n", #call, (int)s_, mod_last_error());           \
      return (int)s_;                                                                      \
    }                                                                                      \
  } while (0)
#define CUDA(call)                                                                         \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));                          \
      return 4;                                                                            \
    }                                                                                      \
  } while (0)

static void* dmalloc(size_t bytes) {
  void* p = NULL;
  if (cudaMalloc(&p, bytes < 256 ? 256 : bytes) != cudaSuccess) return NULL;
  return p;
}

int main(int argc, char** argv) {
  if (argc != 12) {
    fprintf(stderr, "usage: %s B H D prefix F Hh Ww block top_k in.bin out.bin\n", argv[0]);
    return 1;
  }
  mod_layout L;
  L.batch = atoi(argv[1]);
  L.heads = atoi(argv[2]);
  L.head_dim = atoi(argv[3]);
  L.prefix_tokens = atoi(argv[4]);
  L.frames = atoi(argv[5]);
  L.height = atoi(argv[6]);
  L.width = atoi(argv[7]);
  L.block = atoi(argv[8]);
  mod_config cfg = {1e-8, 0.0f, atoi(argv[9]), MOD_SELECT_TOPK, 0.0f, MOD_STAT_POOLED, 1, 1, 0.0f, MOD_ATTN_DEFAULT};

  mod_plan plan;
  CHECK(mod_plan_create(&L, &cfg, 0, &plan));
  const size_t BH = (size_t)L.batch * L.heads;
  const size_t N = (size_t)L.prefix_tokens + (size_t)L.frames * L.height * L.width;
  const size_t n = (size_t)mod_plan_num_blocks(plan), p = (size_t)mod_plan_num_patterns(plan);
  const size_t act = BH * N * L.head_dim * 2;   /* bytes of one bf16 activation */

  /* host input */
  FILE* f = fopen(argv[10], "rb");
  if (!f) return 11;
  unsigned char* h_in = (unsigned char*)malloc(5 * act);
  if (fread(h_in, 1, 5 * act, f) != 5 * act) return 12;
  fclose(f);

  /* device buffers (caller-owned) */
  void *q = dmalloc(act), *k = dmalloc(act), *v = dmalloc(act), *q1 = dmalloc(act), *k1 = dmalloc(act);
  void* o = dmalloc(act);
  float* lse = (float*)dmalloc(BH * N * 4);
  float *W1 = (float*)dmalloc(BH * n * n * 4), *W2 = (float*)dmalloc(BH * n * n * 4);
  float* Wf = (float*)dmalloc(BH * n * n * 4);
  double *x_prev = (double*)dmalloc(BH * p * 8), *x_curr = (double*)dmalloc(BH * p * 8);
  uint8_t* keep = (uint8_t*)dmalloc(BH * L.frames);
  int32_t* row_ptr = (int32_t*)dmalloc(BH * (n + 1) * 4);
  int32_t* col_idx = (int32_t*)dmalloc(BH * n * n * 4);
  void* ws = dmalloc(mod_plan_workspace_bytes(plan));
  if (!q || !k || !v || !q1 || !k1 || !o || !lse || !W1 || !W2 || !Wf || !x_prev || !x_curr || !keep || !row_ptr ||
      !col_idx || !ws)
    return 13;
  CUDA(cudaMemcpy(q, h_in, act, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(k, h_in + act, act, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(v, h_in + 2 * act, act, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(q1, h_in + 3 * act, act, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(k1, h_in + 4 * act, act, cudaMemcpyHostToDevice));

  cudaStream_t st;
  CUDA(cudaStreamCreate(&st));
  /* warm-up statistics and fits (Alg. 1), keep decision */
  CHECK(mod_collect_block_stats(plan, q1, k1, W1, ws, st));
  CHECK(mod_collect_block_stats(plan, q, k, W2, ws, st));
  CHECK(mod_fit_mixture(plan, W1, x_prev, NULL, ws, st));
  CHECK(mod_fit_mixture(plan, W2, x_curr, NULL, ws, st));
  CHECK(mod_keep_frames(plan, x_prev, x_curr, keep, st));
  /* sparse step t = 13: predicted mask (Eq. 6/7), block-sparse attention (Eq. 1) */
  CHECK(mod_predict_block_mask(plan, x_prev, x_curr, 11, 12, 13, keep, NULL, row_ptr, col_idx, ws, st));
  CHECK(mod_block_sparse_attn_fwd(plan, q, k, v, row_ptr, col_idx, o, lse, ws, st));
  /* online update (Eq. 5) with the fresh statistic; history starts as W2 */
  CHECK(mod_collect_block_stats(plan, q, k, Wf, ws, st));
  CHECK(mod_update_online_mask(plan, Wf, row_ptr, col_idx, W2, x_prev, x_curr, ws, st));
  CUDA(cudaStreamSynchronize(st));

  /* host output */
  unsigned char* h_out = (unsigned char*)malloc(act + BH * N * 4 + BH * (n + 1) * 4 + BH * p * 8);
  size_t off = 0;
  CUDA(cudaMemcpy(h_out + off, o, act, cudaMemcpyDeviceToHost));
  off += act;
  CUDA(cudaMemcpy(h_out + off, lse, BH * N * 4, cudaMemcpyDeviceToHost));
  off += BH * N * 4;
  CUDA(cudaMemcpy(h_out + off, row_ptr, BH * (n + 1) * 4, cudaMemcpyDeviceToHost));
  off += BH * (n + 1) * 4;
  CUDA(cudaMemcpy(h_out + off, x_curr, BH * p * 8, cudaMemcpyDeviceToHost));
  off += BH * p * 8;
  f = fopen(argv[11], "wb");
  if (!f || fwrite(h_out, 1, off, f) != off) return 14;
  fclose(f);

  long long nnz = 0;
  const int32_t* rp = (const int32_t*)(h_out + act + BH * N * 4);
  for (size_t bh = 0; bh < BH; ++bh) nnz += rp[bh * (n + 1) + n];
  printf("moddit_step ok: %s, N=%zu n=%zu p=%zu, selected blocks=%lld\n", mod_version(), N, n, p, nnz);

  cudaFree(q); cudaFree(k); cudaFree(v); cudaFree(q1); cudaFree(k1); cudaFree(o); cudaFree(lse);
  cudaFree(W1); cudaFree(W2); cudaFree(Wf); cudaFree(x_prev); cudaFree(x_curr); cudaFree(keep);
  cudaFree(row_ptr); cudaFree(col_idx); cudaFree(ws);
  cudaStreamDestroy(st);
  mod_plan_destroy(plan);
  free(h_in);
  free(h_out);
  return 0;
}
