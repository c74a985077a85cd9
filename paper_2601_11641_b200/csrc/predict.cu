// predict.cu -- K2b mod_predict_block_mask (+ the dense all-ones mask helper).
//
// Per head:
//  1. linear prediction (§5.2 Eq. 6, Eq. 7) of the C and D
//     intensities, evaluated in IEEE fp64 without contraction so that the integer decisions below
//     match the oracle bit for bit:  d = x_c - x_p;  s = d / (t_c - t_p);  x_hat = x_c + s*(t - t_c);
//  2. selection over the 3n-1 pool (§5.3; reading Z3: keys descending, Z14: ties by id):
//     TOPK / TOPMASS sort the (key, id) pairs with an in-shared-memory bitonic network; THRESHOLD
//     compares directly.  TOPMASS accumulates max(key,0)*|supp| sequentially in sorted order;
//  3. block mask = selected diagonals (j - i = delta_k) | selected columns | kept frame squares
//     [a_r,b_r]^2 | diagonal guard | prefix rows/columns (Alg. 1; Z15, Z17),
//     emitted as a CSR index list.  Steps 1 (one CTA per head), 2 (row counts) and 3 (row
//     pointers + column lists) are separate launches so that the O(n^2) mask work spreads over
//     (row chunk, head) CTAs: a warp per row, ballot + popc for counts and write positions.
#include "common.cuh"

namespace {

__device__ __forceinline__ bool before(double ka, int ia, double kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}

struct PredictArgs {
  const double* x_prev;
  const double* x_curr;
  const uint8_t* keep;
  const int* frame_ab;
  const int* row_frames;
  int* row_ptr;
  int* col_idx;
  uint8_t* sel;    // workspace [BH, 3n-1]: selected C/D patterns
  int* cnt;        // workspace [BH, n]: passing blocks per row
  int n, F, p, prefix_last, diag_guard, mode, top_k;
  double param;
  double dt_hist;  // t_curr - t_prev
  double dt_pred;  // t - t_curr
  int P2;          // sort size (power of two >= 3n-1)
};

// 1. keys + selection, one CTA per head
__global__ void __launch_bounds__(1024) select_kernel(PredictArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.n, P = 3 * n - 1, P2 = a.P2;
  double* keys = reinterpret_cast<double*>(smem);
  int* ids = reinterpret_cast<int*>(keys + P2);
  __shared__ int sel_len;
  const int t = threadIdx.x;
  const size_t bh = blockIdx.x;
  const double* xp = a.x_prev + bh * a.p;
  const double* xc = a.x_curr + bh * a.p;
  uint8_t* sel = a.sel + bh * P;
  for (int e = t; e < P2; e += blockDim.x) {
    if (e < P) {
      const double c = xc[e];
      const double d = __dsub_rn(c, xp[e]);
      const double s = __ddiv_rn(d, a.dt_hist);
      keys[e] = __dadd_rn(c, __dmul_rn(s, a.dt_pred));
    } else {
      keys[e] = -INFINITY;
    }
    ids[e] = e;
  }
  __syncthreads();
  if (a.mode == MOD_SELECT_THRESHOLD) {
    for (int e = t; e < P; e += blockDim.x) sel[e] = keys[e] > a.param;
    return;
  }
  for (int k = 2; k <= P2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = t; i < P2; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const double ki = keys[i], kl = keys[l];
          const int ii = ids[i], il = ids[l];
          const bool up = (i & k) == 0;
          const bool sw = up ? before(kl, il, ki, ii) : before(ki, ii, kl, il);
          if (sw) {
            keys[i] = kl; keys[l] = ki;
            ids[i] = il; ids[l] = ii;
          }
        }
      }
      __syncthreads();
    }
  }
  if (t == 0) {
    int L = 0;
    if (a.mode == MOD_SELECT_TOPK) {
      L = min(a.top_k, P);
    } else {  // TOPMASS: sequential fp64 sum in sorted order (bit-identical to the oracle)
      double acc = 0.0;
      for (int e = 0; e < P; ++e) {
        const int id = ids[e];
        const double supp = id < 2 * n - 1 ? (double)(n - abs(id - (n - 1))) : (double)n;
        acc = __dadd_rn(acc, __dmul_rn(fmax(keys[e], 0.0), supp));
      }
      if (acc > 0.0) {
        const double target = __dmul_rn(a.param, acc);
        double c = 0.0;
        L = P;
        for (int e = 0; e < P; ++e) {
          const int id = ids[e];
          const double supp = id < 2 * n - 1 ? (double)(n - abs(id - (n - 1))) : (double)n;
          c = __dadd_rn(c, __dmul_rn(fmax(keys[e], 0.0), supp));
          if (c >= target) {
            L = e + 1;
            break;
          }
        }
      }
    }
    sel_len = L;
  }
  __syncthreads();
  for (int e = t; e < P; e += blockDim.x) sel[e] = 0;
  __syncthreads();
  for (int e = t; e < sel_len; e += blockDim.x) sel[ids[e]] = 1;
}

constexpr int kRowsPerCta = 32;   // 8 warps x 4 rows

struct RowCtx {
  const uint8_t* selC;   // smem [2n-1], index j - i + n - 1
  const uint8_t* selD;   // smem [n]
  const uint8_t* keep;   // global [F] or null
  const int* frame_ab;
  const int* row_frames;
  int n, prefix_last, diag_guard;
  __device__ __forceinline__ bool pass(int i, int j) const {
    if (selC[j - i + n - 1] || selD[j]) return true;
    if (diag_guard && i == j) return true;
    if (i <= prefix_last || j <= prefix_last) return true;
    if (keep) {
      const int rlo = row_frames[2 * i], rhi = row_frames[2 * i + 1];
      for (int r = rlo; r <= rhi; ++r)
        if (keep[r] && frame_ab[2 * r] <= j && j <= frame_ab[2 * r + 1]) return true;
    }
    return false;
  }
};

__device__ __forceinline__ RowCtx load_row_ctx(const PredictArgs& a, uint8_t* s_sel, size_t bh) {
  const int P = 3 * a.n - 1;
  const uint8_t* g = a.sel + bh * P;
  for (int e = threadIdx.x; e < P; e += blockDim.x) s_sel[e] = g[e];
  __syncthreads();
  RowCtx c;
  c.selC = s_sel;
  c.selD = s_sel + 2 * a.n - 1;
  c.keep = a.keep ? a.keep + bh * a.F : nullptr;
  c.frame_ab = a.frame_ab;
  c.row_frames = a.row_frames;
  c.n = a.n;
  c.prefix_last = a.prefix_last;
  c.diag_guard = a.diag_guard;
  return c;
}

// 2. passing blocks per row (warp per row, ballot + popc)
__global__ void __launch_bounds__(256) count_kernel(PredictArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const size_t bh = blockIdx.y;
  const RowCtx c = load_row_ctx(a, smem, bh);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, n = a.n;
  for (int r = 0; r < kRowsPerCta / 8; ++r) {
    const int i = blockIdx.x * kRowsPerCta + warp * (kRowsPerCta / 8) + r;
    if (i >= n) break;
    int cnt = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      cnt += __popc(__ballot_sync(0xffffffffu, j < n && c.pass(i, j)));
    }
    if (lane == 0) a.cnt[bh * n + i] = cnt;
  }
}

// 3. row pointers (prefix over the counts) and ascending column lists
__global__ void __launch_bounds__(256) write_kernel(PredictArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int red[8];
  __shared__ int rowoff[kRowsPerCta + 1];
  const size_t bh = blockIdx.y;
  const RowCtx c = load_row_ctx(a, smem, bh);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, n = a.n;
  const int i0 = blockIdx.x * kRowsPerCta;
  const int* cnt = a.cnt + bh * n;
  int partial = 0;   // rows before this chunk
  for (int i = threadIdx.x; i < i0; i += blockDim.x) partial += cnt[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) partial += __shfl_xor_sync(0xffffffffu, partial, o);
  if (lane == 0) red[warp] = partial;
  __syncthreads();
  if (threadIdx.x == 0) {
    int base = 0;
    for (int w = 0; w < 8; ++w) base += red[w];
    rowoff[0] = base;
    for (int r = 0; r < kRowsPerCta; ++r) rowoff[r + 1] = rowoff[r] + (i0 + r < n ? cnt[i0 + r] : 0);
  }
  __syncthreads();
  int* rp = a.row_ptr + bh * (n + 1);
  for (int r = threadIdx.x; r <= kRowsPerCta; r += blockDim.x) {
    const int i = i0 + r;
    if (i <= n && (r < kRowsPerCta || i == n)) rp[i] = rowoff[r];
  }
  int* ci = a.col_idx + bh * (size_t)n * n;
  for (int r = 0; r < kRowsPerCta / 8; ++r) {
    const int rr = warp * (kRowsPerCta / 8) + r;
    const int i = i0 + rr;
    if (i >= n) break;
    int pos = rowoff[rr];
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      const bool ps = j < n && c.pass(i, j);
      const unsigned m = __ballot_sync(0xffffffffu, ps);
      if (ps) ci[pos + __popc(m & ((1u << lane) - 1u))] = j;
      pos += __popc(m);
    }
  }
}

__global__ void dense_mask_kernel(int* __restrict__ row_ptr, int* __restrict__ col_idx, int n) {
  const size_t bh = blockIdx.y;
  const int i = blockIdx.x;
  if (threadIdx.x == 0) row_ptr[bh * (n + 1) + i] = i * n;
  if (i == 0 && threadIdx.x == 0) row_ptr[bh * (n + 1) + n] = n * n;
  int* ci = col_idx + bh * (size_t)n * n + (size_t)i * n;
  for (int j = threadIdx.x; j < n; j += blockDim.x) ci[j] = j;
}

}  // namespace

extern "C" mod_status mod_predict_block_mask(mod_plan P, const double* x_prev, const double* x_curr, int32_t t_prev,
                                             int32_t t_curr, int32_t t, const uint8_t* keep,
                                             const mod_selection* sel, int32_t* row_ptr, int32_t* col_idx,
                                             void* ws, void* stream) {
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  MOD_REQUIRE(x_prev && x_curr && row_ptr && col_idx && ws, MOD_ERR_USAGE,
              "mod_predict_block_mask: x_prev, x_curr, row_ptr, col_idx, ws must be non-NULL");
  MOD_REQUIRE(t_prev != t_curr, MOD_ERR_INPUT, "mod_predict_block_mask: t_prev == t_curr == %d (zero denominator)",
              t_curr);
  PredictArgs a;
  a.mode = sel ? sel->select_mode : P->cfg.select_mode;
  a.top_k = sel ? sel->top_k : P->cfg.top_k;
  a.param = (double)(sel ? sel->select_param : P->cfg.select_param);
  MOD_REQUIRE(a.mode >= 0 && a.mode <= 2, MOD_ERR_USAGE, "select_mode=%d invalid", a.mode);
  MOD_REQUIRE(a.mode != MOD_SELECT_TOPK || a.top_k >= 1, MOD_ERR_INPUT, "top_k=%d must be >= 1", a.top_k);
  a.x_prev = x_prev;
  a.x_curr = x_curr;
  a.keep = keep;
  a.frame_ab = P->d_frame_ab;
  a.row_frames = P->d_row_frames;
  a.row_ptr = row_ptr;
  a.col_idx = col_idx;
  a.n = P->n;
  a.F = P->F;
  a.p = P->p;
  a.prefix_last = P->prefix_last;
  a.diag_guard = P->cfg.diag_guard;
  a.dt_hist = (double)(t_curr - t_prev);
  a.dt_pred = (double)(t - t_curr);
  a.sel = reinterpret_cast<uint8_t*>(static_cast<char*>(ws) + P->ws_sel);
  a.cnt = reinterpret_cast<int*>(static_cast<char*>(ws) + P->ws_cnt);
  int P2 = 1;
  while (P2 < 3 * P->n - 1) P2 <<= 1;
  a.P2 = P2;
  const size_t smem = (size_t)P2 * (sizeof(double) + sizeof(int));
  MOD_CUDA(cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int BH = P->L.batch * P->L.heads;
  cudaStream_t s = as_stream(stream);
  select_kernel<<<BH, 1024, smem, s>>>(a);
  MOD_LAUNCH_CHECK();
  const dim3 rg((P->n + kRowsPerCta - 1) / kRowsPerCta, BH);
  const size_t rsm = (size_t)(3 * P->n + 16);
  count_kernel<<<rg, 256, rsm, s>>>(a);
  MOD_LAUNCH_CHECK();
  write_kernel<<<rg, 256, rsm, s>>>(a);
  MOD_LAUNCH_CHECK();
  mod_note_launches(3);
  return MOD_OK;
}

extern "C" mod_status mod_fill_dense_mask(mod_plan P, int32_t* row_ptr, int32_t* col_idx, void* stream) {
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  MOD_REQUIRE(row_ptr && col_idx, MOD_ERR_USAGE, "mod_fill_dense_mask: NULL argument");
  const int BH = P->L.batch * P->L.heads;
  dense_mask_kernel<<<dim3(P->n, BH), 256, 0, as_stream(stream)>>>(row_ptr, col_idx, P->n);
  MOD_LAUNCH_CHECK();
  mod_note_launches(1);
  return MOD_OK;
}
