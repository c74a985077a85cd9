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
#include <algorithm>

#include "common.cuh"
#include "sm100.cuh"

using namespace sm100;

namespace {

// One CTA per (head, tile of `rows` consecutive map rows).  The tile is a contiguous run of rows * n fp32
// values of U: its 16-byte-aligned interior is staged in shared memory by ONE bulk copy on the TMA engine
// (HBM-bound: every map byte is read once; two CTAs per SM overlap one's copy with the other's sums),
// then the C (diagonal), D (column) and E (frame-square) partial sums of the tile are formed from shared
// memory in fp64, each in a fixed order (deterministic).
__global__ void __launch_bounds__(256) project_kernel(const float* __restrict__ U, double* __restrict__ part,
                                                       const int* __restrict__ frame_ab, int n, int F, int p,
                                                       int tiles, int rows) {
  extern __shared__ __align__(128) float tile_raw[];
  __shared__ __align__(8) uint64_t bar;
  const size_t bh = blockIdx.y;
  const int tile = blockIdx.x;
  const int i0 = tile * rows, i1 = min(i0 + rows, n), R = i1 - i0;
  const size_t start = (bh * n + i0) * (size_t)n;     // first element of the tile (contiguous rows)
  const size_t count = (size_t)R * n;
  // so that 16-byte global chunks land 16-byte aligned (U itself may be a head slice: use the address)
  const int shift = (int)((reinterpret_cast<uintptr_t>(U + start) >> 2) & 3);
  float* t = tile_raw + 4 + shift;                    // t[i * n + j] = U[bh][i0 + i][j]; tile_raw[0..3] pad
  const float* src = U + start;
  const size_t head = min(count, (size_t)((4 - shift) & 3));    // scalars before the first aligned chunk
  const size_t nvec = (count - head) / 4;                       // aligned 16-byte chunks
  const uint32_t bytes = (uint32_t)(nvec * 16);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0 && bytes > 0) {
    mbar_arrive_expect_tx(&bar, bytes);
    bulk_load(t + head, src + head, bytes, &bar);
  }
  for (size_t e = threadIdx.x; e < head; e += blockDim.x) t[e] = src[e];
  for (size_t e = head + 4 * nvec + threadIdx.x; e < count; e += blockDim.x) t[e] = src[e];
  if (bytes > 0) mbar_wait(&bar, 0);
  __syncthreads();
  double* out = part + (bh * tiles + tile) * (size_t)p;
  const int tid = threadIdx.x;
  // C part: diagonal offset d = k - (n-1); entries (i, i+d) of this tile
  // (each sum is formed as four interleaved partial sums over i mod 4 added at the end: a fixed order,
  // with four independent shared-memory load -> add chains in flight)
  for (int k = tid; k < 2 * n - 1; k += blockDim.x) {
    const int d = k - (n - 1);
    const int ilo = max(0, -(i0 + d)), ihi = min(R, n - (i0 + d));   // rows of the tile with 0 <= i0+i+d < n
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    const float* q = t + i0 + d;   // q[i * (n + 1)] = t[i * n + i0 + i + d]
    int i = ilo;
    for (; i + 4 <= ihi; i += 4) {
      s0 += (double)q[i * (n + 1)];
      s1 += (double)q[(i + 1) * (n + 1)];
      s2 += (double)q[(i + 2) * (n + 1)];
      s3 += (double)q[(i + 3) * (n + 1)];
    }
    for (; i < ihi; ++i) s0 += (double)q[i * (n + 1)];
    out[k] = (s0 + s1) + (s2 + s3);
  }
  // D part: column sums of this tile
  for (int j = tid; j < n; j += blockDim.x) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int i = 0;
    for (; i + 4 <= R; i += 4) {
      s0 += (double)t[i * n + j];
      s1 += (double)t[(i + 1) * n + j];
      s2 += (double)t[(i + 2) * n + j];
      s3 += (double)t[(i + 3) * n + j];
    }
    for (; i < R; ++i) s0 += (double)t[i * n + j];
    out[2 * n - 1 + j] = (s0 + s1) + (s2 + s3);
  }
  // E part: frame squares intersecting this tile (one warp per frame)
  const int warp = tid / 32, lane = tid % 32;
  for (int r = warp; r < F; r += blockDim.x / 32) {
    const int a = frame_ab[2 * r], b = frame_ab[2 * r + 1];
    double s = 0.0;
    for (int i = max(a, i0); i <= min(b, i1 - 1); ++i)
      for (int j = a + lane; j <= b; j += 32) s += (double)t[(i - i0) * n + j];
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

// X[bh][k] = sum_l G'^-1[k][l] r[bh][l].  G'^-1 is symmetric (inverse of the SPD deflated Gram), so the
// sum runs over its ROWS l.  One CTA per (tile of 128 columns k, segment of rows l, chunk of HB heads),
// one wave over the SMs.  A producer thread streams the segment's 32-row x 128-column boxes of G'^-1
// (one 32 KB TMA load each, 2D tensor map) through a 3-stage shared-memory ring (~96 KB in flight per SM).  256 consumer threads are register-blocked: thread (column quad, head half, row group) forms
// 4 columns x HB/2 heads of X from 2 + HB/4 shared-memory vector loads per row (G values and r values,
// the segment's r staged in shared memory), so the loop is bound by the fp64 FMAs (~62 DFMA/clk/SM on
// B200, scripts/micro/fp64_bench.cu), about the time of the HBM stream at HB = 24.  The four row groups
// are added in fixed order through shared memory; split-K partials over segments are added by
// solve_reduce_kernel in fixed order (deterministic, no atomics).  G'^-1 is read once per call for up to
// HB heads.
constexpr int SV_K = 128;                  // columns k per CTA
constexpr int SV_G = 4;                    // row groups
constexpr int SV_ROWS = 32;                // rows per ring stage
constexpr int SV_STAGES = 3;
constexpr int SV_SMEM_G = SV_STAGES * SV_ROWS * SV_K * 8;   // 96 KB
constexpr int SV_CONS = (SV_K / 4) * 2 * SV_G;              // 256 consumer threads
constexpr int SV_THREADS = SV_CONS + 32;
template <int HB>
__global__ void __launch_bounds__(SV_THREADS, 1) solve_stream_kernel(const __grid_constant__ CUtensorMap tm, int ld,
                                                                     const double* __restrict__ r,
                                                                     double* __restrict__ part, int p, int BH,
                                                                     int seg_len) {
  constexpr int HT = HB / 2;               // heads per thread
  extern __shared__ __align__(128) unsigned char sv_smem[];
  double* gs = reinterpret_cast<double*>(sv_smem);                          // [STAGES][ROWS][SV_K]
  double* rs = reinterpret_cast<double*>(sv_smem + SV_SMEM_G);             // [seg_len][HB]
  const int rs_doubles = max(seg_len * HB, (SV_G - 1) * HB * SV_K);       // r, then the row-group partials
  uint64_t* full = reinterpret_cast<uint64_t*>(rs + rs_doubles);
  uint64_t* empty = full + SV_STAGES;
  const int k0 = blockIdx.x * SV_K;
  const int seg = blockIdx.y, h0 = blockIdx.z * HB;
  const int lbeg = seg * seg_len, lend = min(p, lbeg + seg_len);
  const int nl = lend - lbeg;
  const int nchunks = (nl + SV_ROWS - 1) / SV_ROWS;
  const int kw = min(SV_K, ld - k0);       // columns of this tile inside the padded row (multiple of 32)
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int CW = SV_CONS / 32;         // consumer warps
  if (threadIdx.x == 0) {
    for (int s = 0; s < SV_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_mbar_init();
  }
  {   // stage r[h0 .. h0+HB)[lbeg .. lend) (L2-resident) with 8 independent loads in flight per thread
    const int total = HB * seg_len;
    for (int e0 = 0; e0 < total; e0 += 8 * (int)blockDim.x) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * (int)blockDim.x + (int)threadIdx.x;
        const int h = e / seg_len, l = e % seg_len;   // coalesced along l
        v[u] = (e < total && h0 + h < BH && l < nl) ? __ldg(r + (size_t)(h0 + h) * p + lbeg + l) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * (int)blockDim.x + (int)threadIdx.x;
        if (e < total) rs[(e % seg_len) * HB + e / seg_len] = v[u];
      }
    }
  }
  __syncthreads();
  const int kq = threadIdx.x % 32;         // column quad: columns 4 kq .. 4 kq + 3
  const int hh = (threadIdx.x / 32) % 2;   // head half: heads hh HT .. + HT
  const int g = (threadIdx.x / 64);        // row group (consumers: 0..3)
  double acc[4][HT];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int h = 0; h < HT; ++h) acc[c][h] = 0.0;
  if (warp == CW) {
    // ---------------------------------------------------------------- producer: lane = row of the stage
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % SV_STAGES;
      if (c >= SV_STAGES) mbar_wait(&empty[s], ((c / SV_STAGES) - 1) & 1);
      const int rows = min(SV_ROWS, nl - c * SV_ROWS);
      (void)rows;
      if (lane == 0) {
        // one 32 x 128 box (32 KB); rows / columns outside the {ld, p} map are zero-filled by the TMA
        // engine and still count towards the transaction bytes.  Rows past this segment's end belong to
        // the next segment; the consumers skip them.
        mbar_arrive_expect_tx(&full[s], (uint32_t)(SV_ROWS * SV_K * 8));
        tma_load_2d(gs + (size_t)s * SV_ROWS * SV_K, &tm, &full[s], k0, lbeg + c * SV_ROWS);
      }
    }
  } else {
    // ---------------------------------------------------------------- consumers
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % SV_STAGES;
      mbar_wait(&full[s], (c / SV_STAGES) & 1);
      const int rows = min(SV_ROWS, nl - c * SV_ROWS);
      const double* gr = gs + (size_t)s * SV_ROWS * SV_K + 4 * kq;
      const double* rr = rs + (size_t)c * SV_ROWS * HB + hh * HT;
      if (4 * kq < kw) {
#pragma unroll 2
        for (int i = g; i < rows; i += SV_G) {
          const double2 ga = *reinterpret_cast<const double2*>(gr + i * SV_K);
          const double2 gb = *reinterpret_cast<const double2*>(gr + i * SV_K + 2);
          const double gv[4] = {ga.x, ga.y, gb.x, gb.y};
          const double2* r2 = reinterpret_cast<const double2*>(rr + i * HB);
#pragma unroll
          for (int h = 0; h < HT / 2; ++h) {
            const double2 x = r2[h];
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
              acc[cc][2 * h] = fma(gv[cc], x.x, acc[cc][2 * h]);
              acc[cc][2 * h + 1] = fma(gv[cc], x.y, acc[cc][2 * h + 1]);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();   // rs is dead: reuse it for the row-group partials [g-1][head][k]
  double* red = rs;
  if (warp < CW && g > 0) {
#pragma unroll
    for (int cc = 0; cc < 4; ++cc)
#pragma unroll
      for (int h = 0; h < HT; ++h) red[((g - 1) * HB + hh * HT + h) * SV_K + 4 * kq + cc] = acc[cc][h];
  }
  __syncthreads();
  if (warp < CW && g == 0) {
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const int k = k0 + 4 * kq + cc;
      if (k >= p) continue;
#pragma unroll
      for (int h = 0; h < HT; ++h) {
        double v = acc[cc][h];
        for (int gg = 1; gg < SV_G; ++gg) v += red[((gg - 1) * HB + hh * HT + h) * SV_K + 4 * kq + cc];
        if (h0 + hh * HT + h < BH) part[((size_t)seg * BH + h0 + hh * HT + h) * p + k] = v;
      }
    }
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
                                                           double* __restrict__ out, int n, int p, int tiles,
                                                           int rows) {
  const size_t bh = blockIdx.y;
  const int tile = blockIdx.x;
  const int i0 = tile * rows, i1 = min(i0 + rows, n);
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
  const int smem = (P->proj_rows * n + 8) * (int)sizeof(float);
  MOD_CUDA(cudaFuncSetAttribute(project_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  project_kernel<<<dim3(tiles, BH), 256, smem, s>>>(U, part, P->d_frame_ab, n, P->F, p, tiles, P->proj_rows);
  MOD_LAUNCH_CHECK();
  const size_t tot = (size_t)BH * p;
  reduce_rhs_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(part, r, p, tiles, BH);
  MOD_LAUNCH_CHECK();
  double* spart = reinterpret_cast<double*>(static_cast<char*>(ws) + P->ws_solve);
  const dim3 sg((p + SV_K - 1) / SV_K, P->solve_segs, BH <= 8 ? 1 : (BH + 23) / 24);
  const int hb = BH <= 8 ? 8 : 24;
  const int ssmem = SV_SMEM_G + std::max(P->solve_seg_len * hb, (SV_G - 1) * hb * SV_K) * 8 + 2 * SV_STAGES * 8;
  if (BH <= 8) {
    MOD_CUDA(cudaFuncSetAttribute(solve_stream_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssmem));
    solve_stream_kernel<8><<<sg, SV_THREADS, ssmem, s>>>(P->tm_ginv, P->ginv_ld, r, spart, p, BH, P->solve_seg_len);
  } else {
    MOD_CUDA(cudaFuncSetAttribute(solve_stream_kernel<24>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssmem));
    solve_stream_kernel<24><<<sg, SV_THREADS, ssmem, s>>>(P->tm_ginv, P->ginv_ld, r, spart, p, BH, P->solve_seg_len);
  }
  MOD_LAUNCH_CHECK();
  solve_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(spart, X, p, BH, P->solve_segs);
  MOD_LAUNCH_CHECK();
  return MOD_OK;
}

}  // namespace

extern "C" mod_status mod_fit_mixture(mod_plan P, const float* stats, double* x, float* nae, void* ws, void* stream) {
  MOD_NVTX("mod_fit_mixture");
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
                                                       tiles, P->proj_rows);
    MOD_LAUNCH_CHECK();
    nae_final_kernel<<<(BH + 127) / 128, 128, 0, s>>>(part, nae, tiles, BH);
    MOD_LAUNCH_CHECK();
    launches += 2;
  }
  mod_note_launches(launches);
  return MOD_OK;
}

extern "C" mod_status mod_keep_frames(mod_plan P, const double* x_a, const double* x_b, uint8_t* keep, void* stream) {
  MOD_NVTX("mod_keep_frames");
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
  MOD_NVTX("mod_update_online_mask");
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
