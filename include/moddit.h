/*
 * moddit.h -- C ABI of the B200 (sm_100a) MOD-DiT hot path (arxiv 2601.11641).
 *
 * The five compute calls follow the paper's statement of the problem (Algorithm 1, PAPER.md
 * P:983-1033) and BASELINE.json north_star:
 *     mod_collect_block_stats   block statistic of Q, K            (north_star (1); Eq. 2 P:204-206 is
 *                                                                   the paper's statistic, Z1)
 *     mod_fit_mixture           least-squares mixture fit, Eq. 4   (App. B)
 *     mod_keep_frames           block-diagonal preservation        (§5.3; Alg. 1)
 *     mod_predict_block_mask    linear prediction + selection + CSR (Eq. 6/7 P:335-337, P:418-420;
 *                                                                   §5.3; Alg. 1)
 *     mod_update_online_mask    Eq. 5 reconstruction + refit + roll (Alg. 1)
 *     mod_block_sparse_attn_fwd block-sparse attention forward     (Eq. 1; §5.4)
 *
 * Conventions
 *  - Every pointer is a DEVICE pointer unless marked (host).  Tensors are dense, contiguous,
 *    row-major, 16-byte aligned (Q/K/V/O 128-byte aligned for TMA).
 *  - Q, K, V, O: bf16 [B, H, N, D].  Token order inside a head: [prefix | frame-major, y, x],
 *    N = prefix_tokens + frames*height*width.
 *  - n = ceil(N / block) blocks; block i holds tokens [i*block, min((i+1)*block, N)).
 *  - p = 3n - 1 + frames intensities per head, ordered C_0..C_{2n-2} (offset delta_k = k-(n-1)),
 *    D_0..D_{n-1} (column k), E_0..E_{F-1} (frame square r)  (reading Z4).
 *  - Block statistic / history maps: fp32 [B, H, n, n] row-major; intensities fp64 [B, H, p].
 *  - Block masks are per-head CSR index lists: row_ptr int32 [B, H, n+1] holding offsets local to
 *    the head (row_ptr[..,0] = 0, row_ptr[..,n] = nnz of that head), col_idx int32 [B, H, n*n]
 *    (capacity n*n per head; entries [row_ptr[i], row_ptr[i+1]) are the ascending passing columns).
 *  - Every compute call is asynchronous and stream-ordered on `stream` (a cudaStream_t; 0 =
 *    legacy default stream).  Only mod_plan_create synchronizes.
 *  - Ownership: the caller allocates every tensor and the workspace `ws` (size from
 *    mod_plan_workspace_bytes); the library allocates device memory only inside
 *    mod_plan_create (constant tables) and frees it in mod_plan_destroy.  Nothing is retained
 *    after a call returns.  A plan is immutable after creation and may be used concurrently from
 *    several host threads / streams provided each concurrent call has its own workspace.
 *  - Errors: host-side validation runs before any launch.  A failing call launches nothing,
 *    returns the status and sets a thread-local message (mod_last_error) naming the argument
 *    and the values.  Asynchronous device faults surface as MOD_ERR_CUDA on a later call.
 *    There is no CPU fallback: on a device other than sm_100 the plan fails with
 *    MOD_ERR_UNSUPPORTED.
 *  - Determinism: no floating-point atomics; two runs on the same inputs are bitwise identical.
 */
#ifndef MODDIT_H_
#define MODDIT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MOD_OK = 0,
  MOD_ERR_USAGE = 1,       /* null required pointer, bad enum, bad handle */
  MOD_ERR_INPUT = 2,       /* shape / layout / range violation */
  MOD_ERR_NUMERICAL = 3,   /* plan factorization failed (App. B P:1251-1270 chain exhausted) */
  MOD_ERR_CUDA = 4,        /* CUDA runtime / driver error (incl. earlier async faults) */
  MOD_ERR_UNSUPPORTED = 5  /* device is not sm_100 / missing driver entry point */
} mod_status;

/* Selection rule over the 3n-1 pool of predicted C/D intensities (§5.3, reading Z3/Z14):
 * keys are sorted descending ("informativeness" polarity), ties by ascending pattern id. */
typedef enum {
  MOD_SELECT_TOPK = 0,      /* the K largest keys (the paper's Top-K router) */
  MOD_SELECT_THRESHOLD = 1, /* keys > select_param (north_star "threshold selection") */
  MOD_SELECT_TOPMASS = 2    /* shortest sorted prefix whose sum of max(key,0)*|supp| reaches
                               select_param * total (north_star "top-mass selection") */
} mod_select_mode;

typedef enum {
  MOD_STAT_POOLED = 0       /* north_star (1): mean-pooled q.k block score + row softmax mass */
} mod_stat_mode;

/* K4 kernel schedule (all compute the same Eq. 1 result; parity-tested alike).  DEFAULT is the one
 * bench.py times; the others are kept for A/B measurement. */
typedef enum {
  MOD_ATTN_DEFAULT = 0,     /* D = 128 (or 64-token blocks): 8 free-running softmax warps of 16 rows, NS S
                               buffers ahead of them, MMA issue split over two warps; D = 64 with 128-token
                               blocks: the WIDE schedule (measured faster there) */
  MOD_ATTN_SPLITKV = 1,     /* two 4-warp softmax groups splitting the index list (round-1 kernel) */
  MOD_ATTN_PAIR = 2,        /* two query blocks per CTA walking their merged index list (f4) */
  MOD_ATTN_WIDE = 3         /* 16 softmax warps, split-KV over the two key halves of each block (128-token blocks) */
} mod_attn_kernel;

typedef struct {
  int32_t batch, heads, head_dim;  /* B, H, D; D in {64, 128} */
  int32_t prefix_tokens;           /* P0 >= 0 (226 for CogVideoX text tokens) */
  int32_t frames, height, width;   /* latent F, Hh, Ww; N = P0 + F*Hh*Ww */
  int32_t block;                   /* 128, or 64 */
} mod_layout;

typedef struct {
  double lambda;        /* Tikhonov parameter, 1e-8 (App. B) */
  float tau_e;          /* block-diagonal threshold; reading Z7 default 0 */
  int32_t top_k;        /* default K for MOD_SELECT_TOPK (App. C) */
  int32_t select_mode;  /* mod_select_mode default */
  float select_param;   /* default threshold / mass fraction */
  int32_t stat_mode;    /* mod_stat_mode */
  int32_t masked_renorm;/* 1: Eq. 5 uses the fresh map renormalised over the selected blocks (Z12) */
  int32_t diag_guard;   /* 1: every row keeps block (i,i) (reading Z15) */
  float softmax_scale;  /* 0 -> 1/sqrt(D) */
  int32_t attn_kernel;  /* mod_attn_kernel (K4 schedule); 0 = default */
} mod_config;

/* Which step of the App. B solver chain produced the plan's Gram inverse. */
typedef enum {
  MOD_SOLVER_CHOLESKY = 0,  /* SPD elimination without pivoting (the primary method) */
  MOD_SOLVER_LU = 1,        /* elimination with partial pivoting */
  MOD_SOLVER_PINV = 2       /* pseudo-inverse: eigenvalues below 1e-6 x max G_ii dropped */
} mod_solver;

/* Per-call selection override for mod_predict_block_mask (nullable: plan defaults). */
typedef struct {
  int32_t select_mode;
  int32_t top_k;
  float select_param;
} mod_selection;

typedef struct mod_plan_s* mod_plan;

/* Builds the per-layout constants on `device` and synchronizes:
 *   frame block ranges [a_r,b_r] = [floor((P0+r*HW)/block), floor((P0+(r+1)*HW-1)/block)] (Z5);
 *   the closed-form Gram G = M^T M + lambda*I (App. B, plus counted C^T E, D^T E,
 *   overlapping E^T E) and its inverse after deflating the analytically known null space of M
 *   (DESIGN.md "Fit numerics"): fp64, p rows of mod_plan_gram_inverse_ld doubles on the device.
 *   The inverse follows the App. B chain: Gauss-Jordan without pivoting (Cholesky class:
 *   accepted when every pivot is positive and the condition estimate max G_ii x max (G^-1)_ii <= 1e7);
 *   else with partial pivoting (LU class, same acceptance on finite pivots); else the pseudo-inverse
 *   step -- the eigenvectors whose eigenvalues fall below 1e-6 x max G_ii are found by inverse iteration
 *   and deflated like the analytic null space (a dependency the analytic list misses, e.g. degenerate
 *   tiny layouts).
 * Returns MOD_ERR_INPUT for a bad layout, MOD_ERR_NUMERICAL if the whole chain fails,
 * MOD_ERR_UNSUPPORTED if `device` is not sm_100. */
mod_status mod_plan_create(const mod_layout* layout /*host*/, const mod_config* cfg /*host*/, int device,
                           mod_plan* out /*host*/);
void mod_plan_destroy(mod_plan plan);
size_t mod_plan_workspace_bytes(mod_plan plan);
int32_t mod_plan_num_blocks(mod_plan plan);   /* n */
int32_t mod_plan_num_patterns(mod_plan plan); /* p = 3n - 1 + F */
/* Copies the frame block ranges: a_b (host) receives 2*F ints (a_0,b_0,a_1,b_1,...). */
mod_status mod_plan_frame_blocks(mod_plan plan, int32_t* a_b /*host*/);
/* Smallest pivot met while inverting the deflated Gram (host out) and the dimension of the deflated
 * analytic null space (host out).  A min pivot of order lambda flags a dependency the analytic list
 * missed (degenerate tiny layouts); X then carries the undeflated ~cond(G)*eps error. */
mod_status mod_plan_diagnostics(mod_plan plan, double* min_pivot, int32_t* null_dim);
/* Device pointer to the fp64 deflated Gram inverse (p rows, leading dimension mod_plan_gram_inverse_ld
 * doubles; symmetric), for diagnostics. */
const double* mod_plan_gram_inverse(mod_plan plan);
int32_t mod_plan_gram_inverse_ld(mod_plan plan);
/* mod_solver of the App. B chain step that produced the inverse. */
int32_t mod_plan_solver(mod_plan plan);
/* Host wall time of mod_plan_create (milliseconds). */
double mod_plan_create_ms(mod_plan plan);
const char* mod_last_error(void);
const char* mod_version(void);
/* Name of the K4 kernel instantiation mod_block_sparse_attn_fwd launches for this plan (static string,
 * e.g. "attn_fwd_kernel<128,128>"), so that measurements can name what they timed. */
const char* mod_attn_kernel_name(mod_plan plan);

/* K1: W[b,h,i,j] = |I_j| exp(z_ij) / sum_j' |I_j'| exp(z_ij'),  z_ij = s * qbar_i . kbar_j,
 * qbar_i = mean_{p in I_i} Q_p (fp32 accumulation), s = softmax_scale.
 * q, k: bf16 [B,H,N,D]; stats: out fp32 [B,H,n,n]. */
mod_status mod_collect_block_stats(mod_plan plan, const void* q, const void* k, float* stats, void* ws,
                                   void* stream);

/* K2a: X = G^-1 M^T vec(U) per head, U = stats (fp32 [B,H,n,n]); x: out fp64 [B,H,p];
 * nae: nullable out fp32 [B,H] = ||U - MX||_F / ||U||_F (§4.2). */
mod_status mod_fit_mixture(mod_plan plan, const float* stats, double* x, float* nae, void* ws, void* stream);

/* keep[b,h,r] = min(e_r(x_a), e_r(x_b)) > tau_e  (uint8 [B,H,F]). */
mod_status mod_keep_frames(mod_plan plan, const double* x_a, const double* x_b, uint8_t* keep, void* stream);

/* K2b: x_hat = x_curr + (x_curr - x_prev)/(t_curr - t_prev)*(t - t_curr) on the C,D parts (IEEE fp64,
 * no FMA contraction), selection over the 3n-1 pool, block mask = union of selected supports,
 * kept frame squares, the diagonal guard and the prefix rows/columns, emitted as CSR.
 * Requires t_prev != t_curr.  keep may be NULL (no frame squares). */
mod_status mod_predict_block_mask(mod_plan plan, const double* x_prev, const double* x_curr, int32_t t_prev,
                                  int32_t t_curr, int32_t t, const uint8_t* keep, const mod_selection* sel /*host,
                                  nullable*/, int32_t* row_ptr, int32_t* col_idx, void* ws, void* stream);

/* K3: for every selected (i,j) of the CSR mask: hist[i,j] = stats[i,j] / sum_{j' selected} stats[i,j']
 * (masked_renorm=1) or stats[i,j] (0); unselected entries keep their history bit-for-bit (Eq. 5).
 * Then X = fit(hist); x_prev <- x_curr; x_curr <- X. */
mod_status mod_update_online_mask(mod_plan plan, const float* stats_fresh, const int32_t* row_ptr,
                                  const int32_t* col_idx, float* stats_hist, double* x_prev, double* x_curr,
                                  void* ws, void* stream);

/* K4: for token p of query block i: O_p = sum_{q in K(i)} softmax(s Q_p.K_q) V_q over the keys of
 * the listed blocks (keys >= N masked), lse_p = ln sum exp(s Q_p.K_q); an empty list gives O = 0,
 * lse = -inf (Z15).  bf16 inputs, fp32 accumulation and softmax (tcgen05 + TMEM), bf16 output.
 * o: out bf16 [B,H,N,D]; lse: nullable out fp32 [B,H,N].  Column indices must be < n. */
mod_status mod_block_sparse_attn_fwd(mod_plan plan, const void* q, const void* k, const void* v,
                                     const int32_t* row_ptr, const int32_t* col_idx, void* o, float* lse,
                                     void* ws, void* stream);

/* EXACT statistic (Eq. 2) in informativeness polarity (reading Z3):
 * for every block (i,j) listed in the CSR, stats[b,h,i,j] = -S_ij with
 *   S_ij = #{(p,q) in I_i x I_j : exp(s Q_p.K_q - lse_p) < eta} / (|I_i||I_j|)   (strict <),
 * lse: fp32 [B,H,N] natural-log row normalisers -- from mod_block_sparse_attn_fwd on the dense list
 * (warm-up, full map) or on the sparse list (Eq. 5's A_masked renormalised over the kept blocks).
 * Unlisted entries of stats are left untouched.  eta in (0,1) (1e-4, App. A). */
mod_status mod_collect_exact_sparsity(mod_plan plan, const void* q, const void* k, const float* lse,
                                      const int32_t* row_ptr, const int32_t* col_idx, float eta, float* stats,
                                      void* ws, void* stream);

/* ---- quantized sparse attention ------------------------------------------------
 * The paper's sparse stage is SageAttention, whose precision PAPER.md does not state.
 * Reading Z30 fixes a Sage-style scheme: Q and K symmetric INT8 per (head, 128-token
 * block), s = absmax/127, code = rint(x * (127/absmax)) in fp32; V FP8 e4m3 per (head, channel),
 * s_d = absmax_d/448, code = RN_e4m3(v * (448/absmax_d)) in fp32 (saturating); the attention takes
 * S = s_q s_k (Q8 K8^T) on the INT8 tensor cores, P rounded to e4m3, O = (P V8) s_d on the FP8
 * tensor cores, fp32 softmax and accumulation.  Head dim 128 and block 128 only
 * (MOD_ERR_UNSUPPORTED otherwise).
 *
 * Quantized operand buffer (device, caller-allocated, mod_quant_buffer_bytes), byte offsets from
 * mod_quant_buffer_layout (6 entries, in this order):
 *   [0] q8   int8  [B,H,N,D]        [1] k8  int8  [B,H,N,D]
 *   [2] vt8  e4m3  [B,H,D,Np]  V transposed (token-contiguous), Np = N rounded up to 16; tokens in
 *                              [N, Np) are zero
 *   [3] q_scale fp32 [B,H,n]   [4] k_scale fp32 [B,H,n]   [5] v_scale fp32 [B,H,D]
 * (the buffer also holds a [B,H,D] uint32 scratch for the V channel maxima after [5]). */
size_t mod_quant_buffer_bytes(mod_plan plan);
mod_status mod_quant_buffer_layout(mod_plan plan, size_t* offsets /*host, 6 entries*/);

/* Quantize bf16 Q, K, V [B,H,N,D] into qbuf (3 launches + 1 memset: V channel maxima, Q/K blocks,
 * V transpose).  Deterministic. */
mod_status mod_quantize_qkv(mod_plan plan, const void* q, const void* k, const void* v, void* qbuf, void* stream);

/* K4 on the quantized operands: same index lists and outputs as mod_block_sparse_attn_fwd
 * (o bf16 [B,H,N,D], lse nullable fp32 [B,H,N]; empty list -> O = 0, lse = -inf). */
mod_status mod_block_sparse_attn_fwd_q8(mod_plan plan, const void* qbuf, const int32_t* row_ptr,
                                        const int32_t* col_idx, void* o, float* lse, void* ws, void* stream);

/* ---- analysis metrics (the paper's ablations on its own maps, App. A) ---------- */

/* Relative Frobenius distance per head:  out[b,h] = ||A_bh - B_bh||_F / ||B_bh||_F,  fp64 accumulation
 * in a fixed order (deterministic).  It is
 *   DER(t) = ||S^(t) - S^(12)|| / ||S^(12)||        (difference error ratio), and
 *   NRE(t) = ||S_hat^(t) - S_GT^(t)|| / ||S_GT^(t)||   (normalised reconstruction error),
 * with the matrix 2-norm read as Frobenius (reading Z20).  a, b: fp32 [B,H,n,n] (device); out: fp64
 * [B,H] (device).  ||B_bh|| = 0 gives out = 0 when A_bh = B_bh and +inf otherwise.  ws: the plan's
 * workspace (mod_plan_workspace_bytes). */
mod_status mod_map_rel_error(mod_plan plan, const float* a, const float* b, double* out, void* ws, void* stream);

/* Linearity NRE of the C/D intensity trajectories (App. A) over one prediction window:
 *   x_hat_k^(t) = x_curr_k + (x_curr_k - x_prev_k)/(t_curr - t_prev) * (t - t_curr)   (Eq. 6/7),
 *   out[b,h,k]  = sqrt( (1/S) sum_s (x_k^(t_s) - x_hat_k^(t_s))^2 ) / (max_s x_k^(t_s) - min_s x_k^(t_s))
 * for the 3n-1 C and D patterns k (frame intensities are not predicted).  x_prev, x_curr: fp64
 * [B,H,p] anchors at steps t_prev != t_curr; x_traj: fp64 [S,B,H,p] the fitted intensities at the steps
 * t_steps[0..S-1] (host array); out: fp64 [B,H,3n-1] (device).  A pattern whose S values are all
 * equal gets NaN (its range is 0).  S >= 1. */
mod_status mod_linearity_nre(mod_plan plan, const double* x_prev, const double* x_curr, int32_t t_prev,
                             int32_t t_curr, const double* x_traj, const int32_t* t_steps /*host*/, int32_t S,
                             double* out, void* stream);

/* Dense mask helper (the warm-up's full attention, Alg. 1): all-ones CSR. */
mod_status mod_fill_dense_mask(mod_plan plan, int32_t* row_ptr, int32_t* col_idx, void* stream);

/* ---- Ulysses relayout around the sequence<->head all-to-all (BASELINE config 5) ----
 * When activations arrive sequence-sharded over P ranks, the per-head hot path ("We process
 * each attention head independently") needs head shards; the exchange is an all-to-all of contiguous
 * per-peer chunks (NCCL all_to_all_single).  These four calls are the pack before it and the unpack
 * after it, both directions.  All tensors are DEVICE bf16, contiguous, 16-byte aligned; src and dst
 * must not alias; head_dim D in {64, 128}.  Stream-ordered, asynchronous.  Errors: NULL pointer ->
 * MOD_ERR_USAGE; non-divisible sizes, bad D, aliasing or misalignment -> MOD_ERR_INPUT.
 *   seq_pack:    x_seq [B,Ns,H,D]      -> send [P,B,Ns,H/P,D]     (chunk p = heads [p*H/P, (p+1)*H/P))
 *   seq_unpack:  recv [P,B,Ns,Hp,D]    -> x_head [B,Hp,P*Ns,D]    (chunk p = tokens [p*Ns, (p+1)*Ns))
 *   head_pack:   x_head [B,Hp,N,D]     -> send [P,B,N/P,Hp,D]     (chunk p = tokens [p*N/P, (p+1)*N/P))
 *   head_unpack: recv [P,B,Ns,Hp,D]    -> x_seq [B,Ns,P*Hp,D]     (chunk p = heads [p*Hp, (p+1)*Hp))
 * With P = 1 each pack/unpack is the [B,N,H,D] <-> [B,H,N,D] transpose. */
mod_status mod_ulysses_seq_pack(const void* x_seq, void* send, int32_t B, int32_t Ns, int32_t H, int32_t D,
                                int32_t P, void* stream);
mod_status mod_ulysses_seq_unpack(const void* recv, void* x_head, int32_t B, int32_t Ns, int32_t Hp, int32_t D,
                                  int32_t P, void* stream);
mod_status mod_ulysses_head_pack(const void* x_head, void* send, int32_t B, int32_t N, int32_t Hp, int32_t D,
                                 int32_t P, void* stream);
mod_status mod_ulysses_head_unpack(const void* recv, void* x_seq, int32_t B, int32_t Ns, int32_t Hp, int32_t D,
                                   int32_t P, void* stream);
/* Head-chunk variants for the overlapped (chunked) Ulysses exchange: seq_pack of heads [h0, h0+Hc) of an
 * H-head x_seq [B,Ns,H,D] -> send [P,B,Ns,Hc/P,D] (Hc % P == 0); head_unpack of recv [P,B,Ns,Hp,D] into
 * heads [h0, h0+P*Hp) of x_seq [B,Ns,H,D] (other heads untouched).  Same alignment / size rules. */
mod_status mod_ulysses_seq_pack_heads(const void* x_seq, void* send, int32_t B, int32_t Ns, int32_t H, int32_t h0,
                                      int32_t Hc, int32_t D, int32_t P, void* stream);
mod_status mod_ulysses_head_unpack_heads(const void* recv, void* x_seq, int32_t B, int32_t Ns, int32_t Hp, int32_t D,
                                         int32_t P, int32_t H, int32_t h0, void* stream);

/* Number of kernels the last successful compute call on this thread launched (for bench.py). */
int32_t mod_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* MODDIT_H_ */
