// fit.cu -- K2a mod_fit_mixture, mod_keep_frames, K3 mod_update_online_mask.
//
// Fit (Eq. 4; App. B normal equations, RHS P:1171-1186):
//   r = M^T vec U  = [diagonal sums over D_k | column sums | frame-square sums],
//   X = G'^{-1} r  with G'^{-1} the plan's deflated Tikhonov inverse (see plan.cu).
// The paper parallelises the RHS over heads (grid.y), pattern families and 256-thread tree
// reductions with atomics.  Here the map is read in 32-row tiles (coalesced: the
// diagonal sums of consecutive offsets touch consecutive columns), every tile writes fp64 partial
// sums for all p patterns, and a second kernel reduces the tiles in fixed order -- deterministic,
// no atomics.  The solve for all B*H heads is one fp64 GEMM against G'^{-1}, so the p x p inverse
// is streamed from HBM once per call rather than once per head.
//
// Update (Eq. 5, readings Z11/Z12): for every selected block (i,j) of the CSR mask,
//   hist[i,j] = W[i,j] / sum_{j' selected in row i} W[i,j']   (fp64 sum, rounded once to fp32),
// unselected entries untouched; then X = fit(hist), x_prev <- x_curr, x_curr <- X.
#include "common.cuh"

namespace {

__global__ void __launch_bounds__(256) project_kernel(const float* __restrict__ U, double* __restrict__ part,
                                                       const int* __restrict__ frame_ab, int n, int F, int p,
                                                       int tiles) {
  const size_t bh = blockIdx.y;
  const int tile = blockIdx.x;
  const int i0 = tile * kProjRows, i1 = min(i0 + kProjRows, n);
  const float* Uh = U + bh * (size_t)n * n;
  double* out = part + (bh * tiles + tile) * (size_t)p;
  const int t = threadIdx.x;
  // C part: diagonal offset d = k - (n-1); entries (i, i+d) of this tile
  for (int k = t; k < 2 * n - 1; k += blockDim.x) {
    const int d = k - (n - 1);
    double s = 0.0;
    for (int i = i0; i < i1; ++i) {
      const int j = i + d;
      if (j >= 0 && j < n) s += (double)Uh[(size_t)i * n + j];
    }
    out[k] = s;
  }
  // D part: column sums of this tile
  for (int j = t; j < n; j += blockDim.x) {
    double s = 0.0;
    for (int i = i0; i < i1; ++i) s += (double)Uh[(size_t)i * n + j];
    out[2 * n - 1 + j] = s;
  }
  // E part: frame squares intersecting this tile (one warp per frame)
  const int warp = t / 32, lane = t % 32;
  for (int r = warp; r < F; r += blockDim.x / 32) {
    const int a = frame_ab[2 * r], b = frame_ab[2 * r + 1];
    double s = 0.0;
    for (int i = max(a, i0); i <= min(b, i1 - 1); ++i)
      for (int j = a + lane; j <= b; j += 32) s += (double)Uh[(size_t)i * n + j];
    s = warp_sum_d(s);
    if (lane == 0) out[3 * n - 1 + r] = s;
  }
}

__global__ void reduce_rhs_kernel(const double* __restrict__ part, double* __restrict__ r, int p, int tiles,
                                  int BH) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)BH * p) return;
  const size_t bh = e / p, k = e % p;
  double s = 0.0;
  for (int t = 0; t < tiles; ++t) s += part[(bh * tiles + t) * p + k];
  r[e] = s;
}

// X[bh][k] = sum_l G'^-1[k][l] r[bh][l] as a split-K GEMM: CTA (32 rows k, 32 heads, one l segment),
// 64 threads with 4 x 4 register tiles over shared-memory chunks of 32 l; partial sums go to a
// [segments, BH, p] buffer that solve_reduce_kernel adds in fixed order (deterministic, no atomics).
constexpr int SK_SEG = 8, SK_T = 32, SK_L = 32;
__global__ void __launch_bounds__(64) solve_partial_kernel(const double* __restrict__ Ginv, const double* __restrict__ r,
                                                           double* __restrict__ part, int p, int BH, int seg_len) {
  __shared__ double Gs[SK_L][SK_T + 1];   // [l][k]
  __shared__ double Rs[SK_L][SK_T + 1];   // [l][bh]
  const int k0 = blockIdx.x * SK_T, b0 = blockIdx.y * SK_T, seg = blockIdx.z;
  const int lbeg = seg * seg_len, lend = min(p, lbeg + seg_len);
  const int t = threadIdx.x, tk = t / 8, tb = t % 8;      // rows k0+4tk.., heads b0+tb+8m
  double acc[4][4] = {};
  for (int l0 = lbeg; l0 < lend; l0 += SK_L) {
    __syncthreads();
    for (int e = t; e < SK_T * SK_L; e += 64) {
      const int a = e / SK_L, l = e % SK_L;               // coalesced along l
      Gs[l][a] = (k0 + a < p && l0 + l < lend) ? Ginv[(size_t)(k0 + a) * p + l0 + l] : 0.0;
      Rs[l][a] = (b0 + a < BH && l0 + l < lend) ? r[(size_t)(b0 + a) * p + l0 + l] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int l = 0; l < SK_L; ++l) {
      double g[4], rv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        g[i] = Gs[l][tk * 4 + i];
        rv[i] = Rs[l][tb + 8 * i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int m = 0; m < 4; ++m) acc[i][m] = fma(g[i], rv[m], acc[i][m]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int k = k0 + tk * 4 + i, b = b0 + tb + 8 * m;
      if (k < p && b < BH) part[((size_t)seg * BH + b) * p + k] = acc[i][m];
    }
}

__global__ void solve_reduce_kernel(const double* __restrict__ part, double* __restrict__ X, int p, int BH, int nseg) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)BH * p) return;
  double s = 0.0;
  for (int g = 0; g < nseg; ++g) s += part[(size_t)g * BH * p + e];
  X[e] = s;
}

// ||U - MX||^2 and ||U||^2 per (head, row tile)
__global__ void __launch_bounds__(256) nae_partial_kernel(const float* __restrict__ U, const double* __restrict__ X,
                                                           const int* __restrict__ frame_ab,
                                                           const int* __restrict__ row_frames,
                                                           double* __restrict__ out, int n, int p, int tiles) {
  const size_t bh = blockIdx.y;
  const int tile = blockIdx.x;
  const int i0 = tile * kProjRows, i1 = min(i0 + kProjRows, n);
  const float* Uh = U + bh * (size_t)n * n;
  const double* x = X + bh * (size_t)p;
  double res = 0.0, nrm = 0.0;
  for (int i = i0; i < i1; ++i) {
    const int rlo = row_frames[2 * i], rhi = row_frames[2 * i + 1];
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      double m = x[j - i + n - 1] + x[2 * n - 1 + j];
      for (int r = rlo; r <= rhi; ++r)
        if (frame_ab[2 * r] <= j && j <= frame_ab[2 * r + 1]) m += x[3 * n - 1 + r];
      const double u = (double)Uh[(size_t)i * n + j];
      res += (u - m) * (u - m);
      nrm += u * u;
    }
  }
  __shared__ double sr[8], sn[8];
  res = warp_sum_d(res);
  nrm = warp_sum_d(nrm);
  if (threadIdx.x % 32 == 0) {
    sr[threadIdx.x / 32] = res;
    sn[threadIdx.x / 32] = nrm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0;
    for (int w = 0; w < 8; ++w) {
      a += sr[w];
      b += sn[w];
    }
    out[(bh * tiles + tile) * 2] = a;
    out[(bh * tiles + tile) * 2 + 1] = b;
  }
}

__global__ void nae_final_kernel(const double* __restrict__ part, float* __restrict__ nae, int tiles, int BH) {
  const int bh = blockIdx.x * blockDim.x + threadIdx.x;
  if (bh >= BH) return;
  double a = 0, b = 0;
  for (int t = 0; t < tiles; ++t) {
    a += part[((size_t)bh * tiles + t) * 2];
    b += part[((size_t)bh * tiles + t) * 2 + 1];
  }
  nae[bh] = (float)(b > 0 ? sqrt(a / b) : 0.0);
}

__global__ void keep_kernel(const double* __restrict__ xa, const double* __restrict__ xb, uint8_t* __restrict__ keep,
                            int n, int F, int p, float tau, int BH) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= BH * F) return;
  const int bh = e / F, r = e % F;
  const double a = xa[(size_t)bh * p + 3 * n - 1 + r], b = xb[(size_t)bh * p + 3 * n - 1 + r];
  keep[e] = (fmin(a, b) > (double)tau) ? 1 : 0;
}

// Eq. 5 merge; one warp per row
__global__ void merge_kernel(const float* __restrict__ W, const int* __restrict__ row_ptr,
                             const int* __restrict__ col_idx, float* __restrict__ hist, int n, int renorm) {
  const size_t bh = blockIdx.y;
  const int i = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (i >= n) return;
  const int* rp = row_ptr + bh * (n + 1);
  const int* ci = col_idx + bh * (size_t)n * n;
  const float* Wr = W + (bh * n + i) * (size_t)n;
  float* Hr = hist + (bh * n + i) * (size_t)n;
  const int beg = rp[i], end = rp[i + 1];
  if (!renorm) {
    for (int e = beg + lane; e < end; e += 32) Hr[ci[e]] = Wr[ci[e]];
    return;
  }
  double s = 0.0;
  for (int e = beg + lane; e < end; e += 32) s += (double)Wr[ci[e]];
  s = warp_sum_d(s);
  for (int e = beg + lane; e < end; e += 32) {
    const int j = ci[e];
    Hr[j] = s > 0.0 ? (float)((double)Wr[j] / s) : 0.f;
  }
}

__global__ void roll_kernel(double* __restrict__ x_prev, double* __restrict__ x_curr, const double* __restrict__ X,
                            size_t total) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  x_prev[e] = x_curr[e];
  x_curr[e] = X[e];
}

// r = M^T vec U for every head, then X = G'^{-1} r.  4 launches.
mod_status fit_from_map(mod_plan P, const float* U, double* X, void* ws, cudaStream_t s) {
  const int BH = P->L.batch * P->L.heads, n = P->n, p = P->p, tiles = P->proj_tiles;
  double* part = reinterpret_cast<double*>(static_cast<char*>(ws) + P->ws_part);
  double* r = reinterpret_cast<double*>(static_cast<char*>(ws) + P->ws_r);
  project_kernel<<<dim3(tiles, BH), 256, 0, s>>>(U, part, P->d_frame_ab, n, P->F, p, tiles);
  MOD_LAUNCH_CHECK();
  const size_t tot = (size_t)BH * p;
  reduce_rhs_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(part, r, p, tiles, BH);
  MOD_LAUNCH_CHECK();
  const int seg_len = ((p + SK_SEG - 1) / SK_SEG + SK_L - 1) / SK_L * SK_L;
  double* spart = reinterpret_cast<double*>(static_cast<char*>(ws) + P->ws_solve);
  solve_partial_kernel<<<dim3((p + SK_T - 1) / SK_T, (BH + SK_T - 1) / SK_T, SK_SEG), 64, 0, s>>>(P->d_ginv, r, spart, p,
                                                                                             BH, seg_len);
  MOD_LAUNCH_CHECK();
  solve_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(spart, X, p, BH, SK_SEG);
  MOD_LAUNCH_CHECK();
  return MOD_OK;
}

}  // namespace

extern "C" mod_status mod_fit_mixture(mod_plan P, const float* stats, double* x, float* nae, void* ws, void* stream) {
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  MOD_REQUIRE(stats && x && ws, MOD_ERR_USAGE, "mod_fit_mixture: stats, x, ws must be non-NULL");
  cudaStream_t s = as_stream(stream);
  st = fit_from_map(P, stats, x, ws, s);
  if (st != MOD_OK) return st;
  int launches = 4;
  if (nae) {
    const int BH = P->L.batch * P->L.heads, tiles = P->proj_tiles;
    double* part = reinterpret_cast<double*>(static_cast<char*>(ws) + P->ws_nae);
    nae_partial_kernel<<<dim3(tiles, BH), 256, 0, s>>>(stats, x, P->d_frame_ab, P->d_row_frames, part, P->n, P->p,
                                                       tiles);
    MOD_LAUNCH_CHECK();
    nae_final_kernel<<<(BH + 127) / 128, 128, 0, s>>>(part, nae, tiles, BH);
    MOD_LAUNCH_CHECK();
    launches += 2;
  }
  mod_note_launches(launches);
  return MOD_OK;
}

extern "C" mod_status mod_keep_frames(mod_plan P, const double* x_a, const double* x_b, uint8_t* keep, void* stream) {
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  MOD_REQUIRE(x_a && x_b && keep, MOD_ERR_USAGE, "mod_keep_frames: x_a, x_b, keep must be non-NULL");
  const int BH = P->L.batch * P->L.heads;
  keep_kernel<<<(BH * P->F + 255) / 256, 256, 0, as_stream(stream)>>>(x_a, x_b, keep, P->n, P->F, P->p,
                                                                         P->cfg.tau_e, BH);
  MOD_LAUNCH_CHECK();
  mod_note_launches(1);
  return MOD_OK;
}

extern "C" mod_status mod_update_online_mask(mod_plan P, const float* stats_fresh, const int32_t* row_ptr,
                                             const int32_t* col_idx, float* stats_hist, double* x_prev,
                                             double* x_curr, void* ws, void* stream) {
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  MOD_REQUIRE(stats_fresh && row_ptr && col_idx && stats_hist && x_prev && x_curr && ws, MOD_ERR_USAGE,
              "mod_update_online_mask: all pointers must be non-NULL");
  cudaStream_t s = as_stream(stream);
  const int BH = P->L.batch * P->L.heads, n = P->n;
  merge_kernel<<<dim3((n + 3) / 4, BH), 128, 0, s>>>(stats_fresh, row_ptr, col_idx, stats_hist, n,
                                                     P->cfg.masked_renorm);
  MOD_LAUNCH_CHECK();
  double* X = reinterpret_cast<double*>(static_cast<char*>(ws) + P->ws_x);
  st = fit_from_map(P, stats_hist, X, ws, s);
  if (st != MOD_OK) return st;
  const size_t tot = (size_t)BH * P->p;
  roll_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(x_prev, x_curr, X, tot);
  MOD_LAUNCH_CHECK();
  mod_note_launches(6);
  return MOD_OK;
}
