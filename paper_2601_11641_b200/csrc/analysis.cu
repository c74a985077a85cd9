// analysis.cu -- analysis metrics of the paper's ablations, on the GPU.
//
//   mod_map_rel_error   ||A - B||_F / ||B||_F per head: DER(t) (App. A) and the
//                       normalised reconstruction error NRE(t) of Eq. 5 (App. A).
//   mod_linearity_nre   RMS residual of the Eq. 6/7 linear prediction of the C/D intensities over a
//                       window, divided by the trajectory's range (App. A).
// Both are HBM- or latency-bound; fp64 accumulation in a fixed order so results are deterministic.
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace {

constexpr int kRelThreads = 256;
constexpr int kMaxSteps = 64;

// partial (||A-B||^2, ||B||^2) of one chunk of one head's n*n map.  The chunk count per head is
// chosen so that all CTAs are resident at once (kRelCtas = 148 SMs x 8 CTAs, a constant so the
// partition -- and hence the fp64 summation order -- does not depend on the device); each thread
// streams its share in rounds of 8 independent coalesced loads per array and reduces once.
constexpr int kRelPer = 8;
constexpr int kRelRound = kRelThreads * kRelPer;
constexpr int kRelCtas = 148 * 8;

__global__ void __launch_bounds__(kRelThreads) rel_partial_kernel(const float* __restrict__ A,
                                                                   const float* __restrict__ B,
                                                                   double* __restrict__ part, int n, int chunks,
                                                                   size_t chunk_len) {
  const size_t bh = blockIdx.y;
  const size_t nn = (size_t)n * n;
  const size_t c0 = (size_t)blockIdx.x * chunk_len, c1 = min(c0 + chunk_len, nn);
  const float* a = A + bh * nn;
  const float* b = B + bh * nn;
  double d2 = 0.0, b2 = 0.0;
  for (size_t r = c0; r < c1; r += kRelRound) {
    float x[kRelPer], y[kRelPer];
#pragma unroll
    for (int u = 0; u < kRelPer; ++u) {
      const size_t e = r + (size_t)u * kRelThreads + threadIdx.x;
      x[u] = e < c1 ? __ldg(a + e) : 0.f;
      y[u] = e < c1 ? __ldg(b + e) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kRelPer; ++u) {
      const double dx = (double)x[u] - (double)y[u];
      d2 += dx * dx;
      b2 += (double)y[u] * (double)y[u];
    }
  }
  __shared__ double sd[kRelThreads / 32], sb[kRelThreads / 32];
  d2 = warp_sum_d(d2);
  b2 = warp_sum_d(b2);
  if (threadIdx.x % 32 == 0) {
    sd[threadIdx.x / 32] = d2;
    sb[threadIdx.x / 32] = b2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int w = 0; w < kRelThreads / 32; ++w) {
      s0 += sd[w];
      s1 += sb[w];
    }
    part[(bh * chunks + blockIdx.x) * 2] = s0;
    part[(bh * chunks + blockIdx.x) * 2 + 1] = s1;
  }
}

__global__ void rel_final_kernel(const double* __restrict__ part, double* __restrict__ out, int tiles, int BH) {
  const int bh = blockIdx.x * blockDim.x + threadIdx.x;
  if (bh >= BH) return;
  double d2 = 0.0, b2 = 0.0;
  for (int t = 0; t < tiles; ++t) {
    d2 += part[((size_t)bh * tiles + t) * 2];
    b2 += part[((size_t)bh * tiles + t) * 2 + 1];
  }
  out[bh] = b2 > 0.0 ? sqrt(d2 / b2) : (d2 > 0.0 ? INFINITY : 0.0);
}

struct Steps {
  int t[kMaxSteps];
};

// one thread per (head, C/D pattern k)
__global__ void linearity_kernel(const double* __restrict__ xp, const double* __restrict__ xc, int t_prev, int t_curr,
                                 const double* __restrict__ traj, Steps steps, int S, double* __restrict__ out,
                                 int n, int p, int BH) {
  const int npool = 3 * n - 1;
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)BH * npool) return;
  const size_t bh = e / npool;
  const int k = (int)(e % npool);
  const double a = xp[bh * p + k], c = xc[bh * p + k];
  // Eq. 6 in the predict kernel's operation order, IEEE fp64 without contraction
  const double slope = __ddiv_rn(__dsub_rn(c, a), (double)(t_curr - t_prev));
  double ss = 0.0, lo = INFINITY, hi = -INFINITY;
  for (int s = 0; s < S; ++s) {
    const double x = traj[((size_t)s * BH + bh) * p + k];
    const double xh = __dadd_rn(c, __dmul_rn(slope, (double)(steps.t[s] - t_curr)));
    const double r = __dsub_rn(x, xh);
    ss = __dadd_rn(ss, __dmul_rn(r, r));
    lo = fmin(lo, x);
    hi = fmax(hi, x);
  }
  const double range = __dsub_rn(hi, lo);
  out[e] = range > 0.0 ? __ddiv_rn(sqrt(__ddiv_rn(ss, (double)S)), range) : NAN;
}

}  // namespace

extern "C" mod_status mod_map_rel_error(mod_plan P, const float* a, const float* b, double* out, void* ws,
                                        void* stream) {
  MOD_NVTX("mod_map_rel_error");
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  MOD_REQUIRE(a && b && out && ws, MOD_ERR_USAGE, "mod_map_rel_error: a, b, out, ws must be non-NULL");
  cudaStream_t s = as_stream(stream);
  const int BH = P->L.batch * P->L.heads;
  // chunks per head: fill kRelCtas resident CTAs; at most n (the ws_nae partial buffer holds 2*BH*n)
  const size_t nn = (size_t)P->n * P->n;
  int chunks = std::max(1, std::min(P->n, kRelCtas / BH));
  const size_t chunk_len = ((nn + chunks - 1) / chunks + kRelRound - 1) / kRelRound * kRelRound;
  chunks = (int)((nn + chunk_len - 1) / chunk_len);
  double* part = reinterpret_cast<double*>(static_cast<char*>(ws) + P->ws_nae);   // 2*BH*chunks doubles
  rel_partial_kernel<<<dim3(chunks, BH), kRelThreads, 0, s>>>(a, b, part, P->n, chunks, chunk_len);
  MOD_LAUNCH_CHECK();
  rel_final_kernel<<<(BH + 127) / 128, 128, 0, s>>>(part, out, chunks, BH);
  MOD_LAUNCH_CHECK();
  mod_note_launches(2);
  return MOD_OK;
}

extern "C" mod_status mod_linearity_nre(mod_plan P, const double* x_prev, const double* x_curr, int32_t t_prev,
                                        int32_t t_curr, const double* x_traj, const int32_t* t_steps, int32_t S,
                                        double* out, void* stream) {
  MOD_NVTX("mod_linearity_nre");
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  MOD_REQUIRE(x_prev && x_curr && x_traj && t_steps && out, MOD_ERR_USAGE,
              "mod_linearity_nre: x_prev, x_curr, x_traj, t_steps, out must be non-NULL");
  MOD_REQUIRE(t_prev != t_curr, MOD_ERR_INPUT, "mod_linearity_nre: t_prev == t_curr (%d)", t_prev);
  MOD_REQUIRE(S >= 1 && S <= kMaxSteps, MOD_ERR_INPUT, "mod_linearity_nre: S = %d outside [1, %d]", S, kMaxSteps);
  Steps steps{};
  for (int i = 0; i < S; ++i) steps.t[i] = t_steps[i];
  const int BH = P->L.batch * P->L.heads;
  const size_t tot = (size_t)BH * (3 * P->n - 1);
  linearity_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, as_stream(stream)>>>(x_prev, x_curr, t_prev, t_curr,
                                                                                  x_traj, steps, S, out, P->n, P->p,
                                                                                  BH);
  MOD_LAUNCH_CHECK();
  mod_note_launches(1);
  return MOD_OK;
}
