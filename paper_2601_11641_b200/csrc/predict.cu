// predict.cu -- K2b mod_predict_block_mask (+ the dense all-ones mask helper).
//
// Per head (one CTA, 1024 threads):
//  1. linear prediction (§5.2 Eq. 6, Eq. 7) of the C and D
//     intensities, evaluated in IEEE fp64 without contraction so that the integer decisions below
//     match the oracle bit for bit:  d = x_c - x_p;  s = d / (t_c - t_p);  x_hat = x_c + s*(t - t_c);
//  2. selection over the 3n-1 pool (§5.3; reading Z3: keys descending, Z14: ties by id):
//     TOPK / TOPMASS sort the (key, id) pairs with an in-shared-memory bitonic network; THRESHOLD
//     compares directly.  TOPMASS accumulates max(key,0)*|supp| sequentially in sorted order;
//  3. block mask = selected diagonals (j - i = delta_k) | selected columns | kept frame squares
//     [a_r,b_r]^2 | diagonal guard | prefix rows/columns (Alg. 1; Z15, Z17),
//     emitted as a CSR index list: a warp per row, ballot + popc for the counts and the write
//     positions, one block-wide scan for the row pointers.
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
  int n, F, p, prefix_last, diag_guard, mode, top_k;
  double param;
  double dt_hist;  // t_curr - t_prev
  double dt_pred;  // t - t_curr
  int P2;          // sort size (power of two >= 3n-1)
};

__global__ void __launch_bounds__(1024) predict_kernel(PredictArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.n, P = 3 * n - 1, P2 = a.P2;
  double* keys = reinterpret_cast<double*>(smem);
  int* ids = reinterpret_cast<int*>(keys + P2);
  int* cnt = ids + P2;                                   // [n + 1]
  unsigned char* sel = reinterpret_cast<unsigned char*>(cnt + n + 1);   // [P]
  __shared__ int warp_tot[32];
  __shared__ int sel_len;
  const int t = threadIdx.x;
  const size_t bh = blockIdx.x;
  const double* xp = a.x_prev + bh * a.p;
  const double* xc = a.x_curr + bh * a.p;

  // 1. keys
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
  for (int e = t; e < P; e += blockDim.x) sel[e] = 0;
  __syncthreads();

  // 2. selection
  if (a.mode == MOD_SELECT_THRESHOLD) {
    for (int e = t; e < P; e += blockDim.x) sel[e] = keys[e] > a.param;
  } else {
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
      } else {  // TOPMASS
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
    for (int e = t; e < sel_len; e += blockDim.x) sel[ids[e]] = 1;
  }
  __syncthreads();

  // 3. mask rows -> counts
  const unsigned char* selC = sel;            // [2n-1], index j - i + n - 1
  const unsigned char* selD = sel + 2 * n - 1;
  const uint8_t* keep = a.keep ? a.keep + bh * a.F : nullptr;
  const int warp = t / 32, lane = t % 32, nwarps = blockDim.x / 32;
  auto pass = [&](int i, int j) -> bool {
    if (selC[j - i + n - 1] || selD[j]) return true;
    if (a.diag_guard && i == j) return true;
    if (i <= a.prefix_last || j <= a.prefix_last) return true;
    if (keep) {
      const int rlo = a.row_frames[2 * i], rhi = a.row_frames[2 * i + 1];
      for (int r = rlo; r <= rhi; ++r)
        if (keep[r] && a.frame_ab[2 * r] <= j && j <= a.frame_ab[2 * r + 1]) return true;
    }
    return false;
  };
  for (int i = warp; i < n; i += nwarps) {
    int c = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      const unsigned m = __ballot_sync(0xffffffffu, j < n && pass(i, j));
      c += __popc(m);
    }
    if (lane == 0) cnt[i] = c;
  }
  __syncthreads();
  // exclusive scan of cnt[0..n) -> row_ptr (block-wide: 2 rows per thread, n <= 2048)
  {
    const int i0 = 2 * t;
    const int v0 = i0 < n ? cnt[i0] : 0, v1 = i0 + 1 < n ? cnt[i0 + 1] : 0;
    int s = v0 + v1;
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int w = lane < nwarps ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_tot[lane] = w;  // inclusive
    }
    __syncthreads();
    const int base = (warp > 0 ? warp_tot[warp - 1] : 0) + incl - s;
    __syncthreads();
    if (i0 < n) cnt[i0] = base;
    if (i0 + 1 < n) cnt[i0 + 1] = base + v0;
    if (t == 0) cnt[n] = warp_tot[31];
  }
  __syncthreads();
  int* rp = a.row_ptr + bh * (n + 1);
  for (int i = t; i <= n; i += blockDim.x) rp[i] = cnt[i];
  int* ci = a.col_idx + bh * (size_t)n * n;
  for (int i = warp; i < n; i += nwarps) {
    int pos = cnt[i];
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      const bool ps = j < n && pass(i, j);
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
  (void)ws;
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  MOD_REQUIRE(x_prev && x_curr && row_ptr && col_idx, MOD_ERR_USAGE,
              "mod_predict_block_mask: x_prev, x_curr, row_ptr, col_idx must be non-NULL");
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
  int P2 = 1;
  while (P2 < 3 * P->n - 1) P2 <<= 1;
  a.P2 = P2;
  const size_t smem = (size_t)P2 * (sizeof(double) + sizeof(int)) + (P->n + 1) * sizeof(int) + 3 * P->n + 16;
  MOD_CUDA(cudaFuncSetAttribute(predict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int BH = P->L.batch * P->L.heads;
  predict_kernel<<<BH, 1024, smem, as_stream(stream)>>>(a);
  MOD_LAUNCH_CHECK();
  mod_note_launches(1);
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
