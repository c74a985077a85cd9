// plan.cu -- mod_plan_create / destroy, error plumbing, and the per-layout constants.
//
// The plan holds everything that depends only on the layout (App. B: the Gram matrix
// M^T M "can be computed analytically ... without explicit matrix construction", and
// is shared by every head and step):
//   * frame block ranges [a_r, b_r] (reading Z5) and, per block, the frames containing it;
//   * ln|I_j| for the pooled block-mass softmax (north_star (1));
//   * the inverse of the Tikhonov Gram G = M^T M + lambda I (App. B), computed after
//     deflating the analytically known null space N of M: G' = G + c V V^T with V an orthonormal
//     basis of N.  Because r = M^T vec U is orthogonal to N, G'^{-1} r = G^{-1} r exactly, while
//     cond(G') ~ 1e2 instead of cond(G) ~ 1e10.  The inverse is formed
//     once on the device by fp64 Gauss-Jordan elimination (G' is SPD, no pivoting needed).
#include <chrono>
#include <cudaTypedefs.h>
#include <cmath>
#include <cstdarg>
#include <cstring>
#include <map>

#include "common.cuh"

static thread_local char g_err[1024] = "";
static thread_local int g_launches = 0;

void mod_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
void mod_note_launches(int n) { g_launches = n; }

extern "C" const char* mod_last_error(void) { return g_err; }
extern "C" const char* mod_version(void) { return "moddit-b200 0.1 (sm_100a)"; }
extern "C" int32_t mod_last_launch_count(void) { return g_launches; }

mod_status mod_check_sticky() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    mod_set_error("pending CUDA error before launch: %s (%s)", cudaGetErrorName(e), cudaGetErrorString(e));
    return MOD_ERR_CUDA;
  }
  return MOD_OK;
}

mod_status mod_validate_plan(mod_plan plan) {
  MOD_REQUIRE(plan != nullptr, MOD_ERR_USAGE, "plan is NULL");
  MOD_REQUIRE(plan->d_ginv != nullptr, MOD_ERR_USAGE, "plan is not initialised");
  return mod_check_sticky();
}

// ------------------------------------------------------------------------------------------------
// Gauss-Jordan inversion on the device (fp64, in place, row-major with leading dimension ld)
//   no pivoting      -- the Cholesky-class step for an SPD matrix (App. B);
//   partial pivoting -- the LU-with-partial-pivoting fallback: at step k the row with the
//                       largest |A[i][k]|, i >= k, is swapped into place; the column swaps that undo the
//                       row permutation are applied in reverse order at the end.
// ------------------------------------------------------------------------------------------------
__global__ void gj_argmax_kernel(const double* A, int ld, int p, int k, int* piv_row) {
  __shared__ double bv[32];
  __shared__ int bi[32];
  double best = -1.0;
  int besti = k;
  for (int i = k + threadIdx.x; i < p; i += blockDim.x) {
    const double v = fabs(A[(size_t)i * ld + k]);
    if (v > best) {   // ascending i per thread: ties keep the smallest row
      best = v;
      besti = i;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, besti, o);
    if (ov > best || (ov == best && oi < besti)) {
      best = ov;
      besti = oi;
    }
  }
  if (threadIdx.x % 32 == 0) {
    bv[threadIdx.x / 32] = best;
    bi[threadIdx.x / 32] = besti;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)blockDim.x / 32; ++w)
      if (bv[w] > best || (bv[w] == best && bi[w] < besti)) {
        best = bv[w];
        besti = bi[w];
      }
    piv_row[k] = besti;
  }
}

__global__ void gj_swap_rows_kernel(double* A, int ld, int p, int k, const int* piv_row) {
  const int r = piv_row[k];
  if (r == k) return;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < p; j += gridDim.x * blockDim.x) {
    const double t = A[(size_t)k * ld + j];
    A[(size_t)k * ld + j] = A[(size_t)r * ld + j];
    A[(size_t)r * ld + j] = t;
  }
}

__global__ void gj_swap_cols_kernel(double* A, int ld, int p, int k, const int* piv_row) {
  const int r = piv_row[k];
  if (r == k) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p; i += gridDim.x * blockDim.x) {
    const double t = A[(size_t)i * ld + k];
    A[(size_t)i * ld + k] = A[(size_t)i * ld + r];
    A[(size_t)i * ld + r] = t;
  }
}

__global__ void gj_pivot_kernel(double* A, int ld, double* col, double* pivots, int p, int k) {
  __shared__ double piv;
  if (threadIdx.x == 0) {
    piv = A[(size_t)k * ld + k];
    pivots[k] = piv;
  }
  __syncthreads();
  const double inv = 1.0 / piv;
  for (int i = threadIdx.x; i < p; i += blockDim.x) col[i] = (i == k) ? 0.0 : A[(size_t)i * ld + k];
  __syncthreads();
  for (int j = threadIdx.x; j < p; j += blockDim.x) {
    double a = (j == k) ? 1.0 : A[(size_t)k * ld + j];
    A[(size_t)k * ld + j] = a * inv;
  }
}

__global__ void gj_eliminate_kernel(double* A, int ld, const double* col, int p, int k) {
  const int i = blockIdx.y;
  if (i == k) return;
  const double f = col[i];
  const double* rk = A + (size_t)k * ld;
  double* ri = A + (size_t)i * ld;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < p; j += gridDim.x * blockDim.x) {
    double a = (j == k) ? 0.0 : ri[j];
    ri[j] = a - f * rk[j];
  }
}

// Inverts the host matrix G (p x p) into dA (p x ld) on `s`; returns the pivots (host).  pivoting:
// 0 none, 1 partial.  Every launch is stream-ordered; one synchronization at the end.
static cudaError_t gj_invert(const std::vector<double>& G, int p, int ld, bool pivoting, double* dA,
                             std::vector<double>& piv, cudaStream_t s) {
  std::vector<double> Gp((size_t)p * ld, 0.0);
  for (int i = 0; i < p; ++i) std::memcpy(&Gp[(size_t)i * ld], &G[(size_t)i * p], sizeof(double) * p);
  double *d_col = nullptr, *d_piv = nullptr;
  int* d_row = nullptr;
  cudaError_t e = cudaMemcpyAsync(dA, Gp.data(), sizeof(double) * Gp.size(), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMalloc(&d_col, sizeof(double) * p);
  if (e == cudaSuccess) e = cudaMalloc(&d_piv, sizeof(double) * p);
  if (e == cudaSuccess) e = cudaMalloc(&d_row, sizeof(int) * p);
  if (e == cudaSuccess) {
    const dim3 eg((p + 255) / 256 > 8 ? 8 : (p + 255) / 256, p);
    const int sg = (p + 255) / 256 > 16 ? 16 : (p + 255) / 256;
    for (int k = 0; k < p; ++k) {
      if (pivoting) {
        gj_argmax_kernel<<<1, 1024, 0, s>>>(dA, ld, p, k, d_row);
        gj_swap_rows_kernel<<<sg, 256, 0, s>>>(dA, ld, p, k, d_row);
      }
      gj_pivot_kernel<<<1, 1024, 0, s>>>(dA, ld, d_col, d_piv, p, k);
      gj_eliminate_kernel<<<eg, 256, 0, s>>>(dA, ld, d_col, p, k);
    }
    if (pivoting)
      for (int k = p - 1; k >= 0; --k) gj_swap_cols_kernel<<<sg, 256, 0, s>>>(dA, ld, p, k, d_row);
    e = cudaGetLastError();
  }
  piv.assign(p, 0.0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(piv.data(), d_piv, sizeof(double) * p, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(d_col);
  cudaFree(d_piv);
  cudaFree(d_row);
  return e;
}

// A Gauss-Jordan result is accepted when every pivot is finite (and, without pivoting, positive: the SPD
// test of the Cholesky step) and the matrix is not numerically singular: the condition estimate
// max_i |G_ii| x max_i |(G^-1)_ii| (a lower bound of cond_2 for SPD G) stays below kCondMax.  A basis
// dependency that the analytic null-space list misses leaves an eigenvalue ~lambda = 1e-8 and an inverse
// diagonal >= 1/(p lambda) with max G_ii >= n >= p/3: estimate >= 1/(3 lambda) = 3e7; the deflated video
// layouts estimate ~1e4-1e6.
constexpr double kCondMax = 1e7;
static bool inverse_ok(const std::vector<double>& piv, bool need_positive, const std::vector<double>& G, int p,
                       const double* dA, int ld, double* pmin_out, double* cond_out) {
  double pmin = 1e300;
  for (double x : piv) {
    if (!std::isfinite(x) || (need_positive && !(x > 0.0))) {
      *pmin_out = x;
      *cond_out = INFINITY;
      return false;
    }
    pmin = std::min(pmin, std::fabs(x));
  }
  *pmin_out = pmin;
  std::vector<double> d(p);
  if (cudaMemcpy2D(d.data(), sizeof(double), dA, sizeof(double) * (ld + 1), sizeof(double), p,
                   cudaMemcpyDeviceToHost) != cudaSuccess)
    return false;
  double gmax = 0.0, imax = 0.0;
  for (int i = 0; i < p; ++i) {
    gmax = std::max(gmax, std::fabs(G[(size_t)i * p + i]));
    if (!std::isfinite(d[i])) {
      *cond_out = INFINITY;
      return false;
    }
    imax = std::max(imax, std::fabs(d[i]));
  }
  *cond_out = gmax * imax;
  return *cond_out <= kCondMax;
}

// ------------------------------------------------------------------------------------------------
// host: closed-form Gram (App. B; C^T E, D^T E and overlapping E^T E by counting)
// ------------------------------------------------------------------------------------------------
static void build_gram(int n, const std::vector<int>& ab, double lambda, std::vector<double>& G) {
  const int F = (int)ab.size() / 2;
  const int p = 3 * n - 1 + F;
  const int oC = 0, oD = 2 * n - 1, oE = 3 * n - 1;
  G.assign((size_t)p * p, 0.0);
  auto at = [&](int i, int j) -> double& { return G[(size_t)i * p + j]; };
  for (int k = 0; k < 2 * n - 1; ++k) {
    const int d = k - (n - 1);
    at(oC + k, oC + k) = n - std::abs(d);
    for (int j = 0; j < n; ++j)
      if (j - d >= 0 && j - d <= n - 1) at(oC + k, oD + j) = at(oD + j, oC + k) = 1.0;
    for (int r = 0; r < F; ++r) {
      const int Lr = ab[2 * r + 1] - ab[2 * r] + 1;
      const double v = std::max(0, Lr - std::abs(d));
      at(oC + k, oE + r) = at(oE + r, oC + k) = v;
    }
  }
  for (int j = 0; j < n; ++j) {
    at(oD + j, oD + j) = n;
    for (int r = 0; r < F; ++r)
      if (ab[2 * r] <= j && j <= ab[2 * r + 1]) at(oD + j, oE + r) = at(oE + r, oD + j) = ab[2 * r + 1] - ab[2 * r] + 1;
  }
  for (int r = 0; r < F; ++r)
    for (int s = 0; s < F; ++s) {
      const int ov = std::max(0, std::min(ab[2 * r + 1], ab[2 * s + 1]) - std::max(ab[2 * r], ab[2 * s]) + 1);
      at(oE + r, oE + s) = (double)ov * ov;
    }
  for (int i = 0; i < p; ++i) at(i, i) += lambda;
}

// Analytic null space of M (linear dependencies among the binary bases), see DESIGN.md:
//   sum_k C_k = J = sum_k D_k;  a square covering the whole grid equals J;  unit squares covering
//   every diagonal block sum to C_{delta=0};  identical squares are equal columns.
static std::vector<std::vector<double>> null_space(int n, const std::vector<int>& ab) {
  const int F = (int)ab.size() / 2;
  const int p = 3 * n - 1 + F;
  const int oC = 0, oD = 2 * n - 1, oE = 3 * n - 1;
  std::vector<std::vector<double>> V;
  {
    std::vector<double> v(p, 0.0);
    for (int k = 0; k < 2 * n - 1; ++k) v[oC + k] = 1.0;
    for (int k = 0; k < n; ++k) v[oD + k] = -1.0;
    V.push_back(v);
  }
  std::map<std::pair<int, int>, int> first;
  for (int r = 0; r < F; ++r) {
    auto key = std::make_pair(ab[2 * r], ab[2 * r + 1]);
    auto it = first.find(key);
    if (it == first.end()) {
      first[key] = r;
    } else {
      std::vector<double> v(p, 0.0);
      v[oE + r] = 1.0;
      v[oE + it->second] = -1.0;
      V.push_back(v);
    }
  }
  for (auto& kv : first) {
    if (kv.first.first == 0 && kv.first.second == n - 1) {
      std::vector<double> v(p, 0.0);
      for (int k = 0; k < 2 * n - 1; ++k) v[oC + k] = 1.0;
      v[oE + kv.second] = -1.0;
      V.push_back(v);
    }
  }
  {
    bool all_unit = true;
    std::vector<int> rep(n, -1);
    for (auto& kv : first) {
      if (kv.first.first != kv.first.second) all_unit = false;
      else rep[kv.first.first] = kv.second;
    }
    bool covers = all_unit;
    for (int i = 0; i < n && covers; ++i) covers = rep[i] >= 0;
    if (covers && n > 1) {
      std::vector<double> v(p, 0.0);
      v[oC + (n - 1)] = 1.0;
      for (int i = 0; i < n; ++i) v[oE + rep[i]] = -1.0;
      V.push_back(v);
    }
  }
  // orthonormalise (modified Gram-Schmidt, twice)
  std::vector<std::vector<double>> Q;
  for (auto v : V) {
    for (int pass = 0; pass < 2; ++pass)
      for (auto& q : Q) {
        double d = 0;
        for (int i = 0; i < p; ++i) d += q[i] * v[i];
        for (int i = 0; i < p; ++i) v[i] -= d * q[i];
      }
    double nr = 0;
    for (int i = 0; i < p; ++i) nr += v[i] * v[i];
    nr = std::sqrt(nr);
    if (nr < 1e-9) continue;
    for (int i = 0; i < p; ++i) v[i] /= nr;
    Q.push_back(v);
  }
  return Q;
}

static size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

extern "C" mod_status mod_plan_create(const mod_layout* layout, const mod_config* cfg, int device, mod_plan* out) {
  MOD_NVTX("mod_plan_create");
  MOD_REQUIRE(layout && cfg && out, MOD_ERR_USAGE, "mod_plan_create: layout, cfg and out must be non-NULL");
  const auto t_start = std::chrono::steady_clock::now();
  *out = nullptr;
  const mod_layout L = *layout;
  MOD_REQUIRE(L.batch >= 1 && L.heads >= 1, MOD_ERR_INPUT, "batch=%d heads=%d must be >= 1", L.batch, L.heads);
  MOD_REQUIRE(L.head_dim == 64 || L.head_dim == 128, MOD_ERR_INPUT, "head_dim=%d must be 64 or 128", L.head_dim);
  MOD_REQUIRE(L.block == 64 || L.block == 128, MOD_ERR_INPUT, "block=%d must be 64 or 128", L.block);
  MOD_REQUIRE(L.prefix_tokens >= 0 && L.frames >= 1 && L.height >= 1 && L.width >= 1, MOD_ERR_INPUT,
              "prefix_tokens=%d frames=%d height=%d width=%d invalid", L.prefix_tokens, L.frames, L.height, L.width);
  const long long Nll = (long long)L.prefix_tokens + (long long)L.frames * L.height * L.width;
  MOD_REQUIRE(Nll <= (1 << 26), MOD_ERR_INPUT, "N=%lld too large", Nll);
  const int N = (int)Nll;
  const int n = (N + L.block - 1) / L.block;
  MOD_REQUIRE(n <= kMaxBlocks, MOD_ERR_INPUT, "n=%d blocks exceeds the supported %d", n, kMaxBlocks);
  MOD_REQUIRE(cfg->lambda >= 0.0 && std::isfinite(cfg->lambda), MOD_ERR_INPUT, "lambda=%g must be >= 0", cfg->lambda);
  MOD_REQUIRE(cfg->top_k >= 1, MOD_ERR_INPUT, "top_k=%d must be >= 1", cfg->top_k);
  MOD_REQUIRE(cfg->select_mode >= 0 && cfg->select_mode <= 2, MOD_ERR_USAGE, "select_mode=%d invalid", cfg->select_mode);
  MOD_REQUIRE(cfg->stat_mode == MOD_STAT_POOLED, MOD_ERR_UNSUPPORTED, "stat_mode=%d not supported", cfg->stat_mode);
  MOD_REQUIRE(cfg->softmax_scale >= 0.f, MOD_ERR_INPUT, "softmax_scale=%g must be >= 0", cfg->softmax_scale);
  MOD_REQUIRE(cfg->attn_kernel >= MOD_ATTN_DEFAULT && cfg->attn_kernel <= MOD_ATTN_WIDE, MOD_ERR_USAGE,
              "attn_kernel=%d invalid", cfg->attn_kernel);

  int ndev = 0;
  MOD_CUDA(cudaGetDeviceCount(&ndev));
  MOD_REQUIRE(device >= 0 && device < ndev, MOD_ERR_USAGE, "device=%d out of range (%d devices)", device, ndev);
  cudaDeviceProp prop;
  MOD_CUDA(cudaGetDeviceProperties(&prop, device));
  MOD_REQUIRE(prop.major == 10 && prop.minor == 0, MOD_ERR_UNSUPPORTED,
              "device %d is sm_%d%d; this library is built for sm_100a (B200) only", device, prop.major, prop.minor);
  int prev_dev = 0;
  MOD_CUDA(cudaGetDevice(&prev_dev));
  MOD_CUDA(cudaSetDevice(device));

  mod_plan P = new mod_plan_s{};
  P->L = L;
  P->cfg = *cfg;
  P->device = device;
  P->N = N;
  P->n = n;
  P->F = L.frames;
  P->p = 3 * n - 1 + L.frames;
  P->prefix_last = L.prefix_tokens > 0 ? (L.prefix_tokens - 1) / L.block : -1;
  P->scale = cfg->softmax_scale > 0.f ? cfg->softmax_scale : 1.0f / std::sqrt((float)L.head_dim);
  P->sm_count = prop.multiProcessorCount;
  const int HW = L.height * L.width;
  P->frame_ab.resize(2 * L.frames);
  for (int r = 0; r < L.frames; ++r) {
    P->frame_ab[2 * r] = (L.prefix_tokens + r * HW) / L.block;
    P->frame_ab[2 * r + 1] = (L.prefix_tokens + (r + 1) * HW - 1) / L.block;
  }
  std::vector<int> row_frames(2 * n);
  for (int i = 0; i < n; ++i) {
    int lo = L.frames, hi = -1;
    for (int r = 0; r < L.frames; ++r)
      if (P->frame_ab[2 * r] <= i && i <= P->frame_ab[2 * r + 1]) {
        lo = std::min(lo, r);
        hi = std::max(hi, r);
      }
    row_frames[2 * i] = lo;
    row_frames[2 * i + 1] = hi;
  }
  std::vector<float> logsz(n);
  for (int j = 0; j < n; ++j) logsz[j] = std::log((float)(std::min((j + 1) * L.block, N) - j * L.block));

  auto fail = [&](mod_status st) {
    mod_plan_destroy(P);
    cudaSetDevice(prev_dev);
    return st;
  };
#define PLAN_CUDA(call)                                                                            \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) {                                                                       \
      mod_set_error("CUDA error %s in mod_plan_create: %s", cudaGetErrorName(e_), cudaGetErrorString(e_)); \
      return fail(MOD_ERR_CUDA);                                                                   \
    }                                                                                              \
  } while (0)

  PLAN_CUDA(cudaMalloc(&P->d_frame_ab, sizeof(int) * 2 * L.frames));
  PLAN_CUDA(cudaMemcpy(P->d_frame_ab, P->frame_ab.data(), sizeof(int) * 2 * L.frames, cudaMemcpyHostToDevice));
  PLAN_CUDA(cudaMalloc(&P->d_row_frames, sizeof(int) * 2 * n));
  PLAN_CUDA(cudaMemcpy(P->d_row_frames, row_frames.data(), sizeof(int) * 2 * n, cudaMemcpyHostToDevice));
  PLAN_CUDA(cudaMalloc(&P->d_log_sizes, sizeof(float) * n));
  PLAN_CUDA(cudaMemcpy(P->d_log_sizes, logsz.data(), sizeof(float) * n, cudaMemcpyHostToDevice));

  // ---- deflated Gram and its inverse: the App. B P:1251-1270 chain (Cholesky -> LU with partial
  // pivoting -> pseudo-inverse with threshold-based retention), each step on the device
  const int p = P->p, ld = (p + 31) / 32 * 32;
  P->ginv_ld = ld;
  std::vector<double> G;
  build_gram(n, P->frame_ab, cfg->lambda, G);
  auto V = null_space(n, P->frame_ab);
  const double c = (double)n;
  auto deflate = [&](const std::vector<double>& v) {
    for (int i = 0; i < p; ++i) {
      if (v[i] == 0.0) continue;
      for (int j = 0; j < p; ++j) G[(size_t)i * p + j] += c * v[i] * v[j];
    }
  };
  for (auto& v : V) deflate(v);
  PLAN_CUDA(cudaMalloc(&P->d_ginv, sizeof(double) * (size_t)p * ld));
  cudaStream_t cs = nullptr;
  PLAN_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  auto fail_s = [&](mod_status st) {
    cudaStreamDestroy(cs);
    return fail(st);
  };
#define PLAN_CUDA_S(call)                                                                          \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) {                                                                       \
      mod_set_error("CUDA error %s in mod_plan_create: %s", cudaGetErrorName(e_), cudaGetErrorString(e_)); \
      return fail_s(MOD_ERR_CUDA);                                                                 \
    }                                                                                              \
  } while (0)
  std::vector<double> piv;
  double pmin = 0.0, cond = 0.0;
  int solver = MOD_SOLVER_CHOLESKY;
  // 1. Cholesky class: the deflated Gram is SPD -> Gauss-Jordan without pivoting, every pivot > 0
  PLAN_CUDA_S(gj_invert(G, p, ld, false, P->d_ginv, piv, cs));
  if (!inverse_ok(piv, true, G, p, P->d_ginv, ld, &pmin, &cond)) {
    // 2. LU with partial pivoting (not numerically SPD / ill conditioned)
    solver = MOD_SOLVER_LU;
    PLAN_CUDA_S(gj_invert(G, p, ld, true, P->d_ginv, piv, cs));
    if (!inverse_ok(piv, false, G, p, P->d_ginv, ld, &pmin, &cond)) {
      // 3. pseudo-inverse: eigenvectors of G' whose eigenvalues fall below kNullRel x max_i G'_ii are
      //    dropped (threshold-based retention).  They are found by block inverse iteration with the
      //    inverse of the shifted G' + mu I (SPD for any PSD G'), kept only if their Rayleigh quotient is
      //    below the threshold, and deflated exactly like the analytic null space: for r = M^T vec U
      //    (orthogonal to them) (G' + c W W^T)^-1 r is the retained-spectrum pseudo-inverse solution.
      solver = MOD_SOLVER_PINV;
      constexpr double kNullRel = 1e-6;
      double gmax = 0.0;
      for (int i = 0; i < p; ++i) gmax = std::max(gmax, G[(size_t)i * p + i]);
      const double mu = 1e-10 * gmax;
      std::vector<double> Ainv((size_t)p * ld);
      uint64_t st = 0x9E3779B97F4A7C15ull;
      for (int round = 0; round < 4; ++round) {
        std::vector<double> Gs = G;
        for (int i = 0; i < p; ++i) Gs[(size_t)i * p + i] += mu;
        PLAN_CUDA_S(gj_invert(Gs, p, ld, true, P->d_ginv, piv, cs));
        PLAN_CUDA_S(cudaMemcpy(Ainv.data(), P->d_ginv, sizeof(double) * Ainv.size(), cudaMemcpyDeviceToHost));
        const int kb = std::min(p, 16);
        std::vector<std::vector<double>> W(kb, std::vector<double>(p));
        for (auto& w : W)
          for (auto& x : w) {
            st ^= st << 13; st ^= st >> 7; st ^= st << 17;
            x = (double)(st >> 11) * (1.0 / 9007199254740992.0) - 0.5;
          }
        auto orthonormalize = [&]() {   // modified Gram-Schmidt, twice, against V and the block
          std::vector<std::vector<double>> Q;
          for (auto w : W) {
            for (int pass = 0; pass < 2; ++pass)
              for (auto* basis : {&V, &Q})
                for (auto& q : *basis) {
                  double dd = 0;
                  for (int i = 0; i < p; ++i) dd += q[i] * w[i];
                  for (int i = 0; i < p; ++i) w[i] -= dd * q[i];
                }
            double nr = 0;
            for (double x : w) nr += x * x;
            nr = std::sqrt(nr);
            if (nr < 1e-300) continue;
            for (auto& x : w) x /= nr;
            Q.push_back(w);
          }
          W = Q;
        };
        orthonormalize();
        for (int it = 0; it < 4; ++it) {
          for (auto& w : W) {
            std::vector<double> y(p, 0.0);
            for (int i = 0; i < p; ++i) {
              const double* row = &Ainv[(size_t)i * ld];
              double acc = 0.0;
              for (int j = 0; j < p; ++j) acc += row[j] * w[j];
              y[i] = acc;
            }
            w = y;
          }
          orthonormalize();
        }
        int found = 0;
        for (auto& w : W) {
          double rq = 0.0;
          for (int i = 0; i < p; ++i) {
            double gi = 0.0;
            for (int j = 0; j < p; ++j) gi += G[(size_t)i * p + j] * w[j];
            rq += w[i] * gi;
          }
          if (!(rq <= kNullRel * gmax)) continue;   // not numerically null: keep it in the solve
          deflate(w);
          V.push_back(w);
          ++found;
        }
        if (found < kb) break;   // the block held non-null directions too: every null one was found
      }
      PLAN_CUDA_S(gj_invert(G, p, ld, false, P->d_ginv, piv, cs));
      if (!inverse_ok(piv, true, G, p, P->d_ginv, ld, &pmin, &cond)) {
        PLAN_CUDA_S(gj_invert(G, p, ld, true, P->d_ginv, piv, cs));
        if (!inverse_ok(piv, false, G, p, P->d_ginv, ld, &pmin, &cond)) {
          mod_set_error("Gram inverse failed: Cholesky, LU and the pseudo-inverse step all left a condition "
                        "estimate of %.3e (min pivot %.3e, p=%d, %d null vectors)", cond, pmin, p, (int)V.size());
          return fail_s(MOD_ERR_NUMERICAL);
        }
      }
    }
  }
  cudaStreamDestroy(cs);
#undef PLAN_CUDA_S
  {   // TMA map of the inverse for the solve stream (fit.cu): rows of ld doubles, box 32 rows x 128 columns
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      mod_set_error("cuTensorMapEncodeTiled driver entry point unavailable");
      return fail(MOD_ERR_UNSUPPORTED);
    }
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)p};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
    cuuint32_t box[2] = {128, 32};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&P->tm_ginv, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, P->d_ginv, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      mod_set_error("cuTensorMapEncodeTiled (Gram inverse) failed (%d)", (int)r);
      return fail(MOD_ERR_CUDA);
    }
  }
  P->min_pivot = pmin;
  P->cond_est = cond;
  P->null_dim = (int)V.size();
  P->solver = solver;

  // ---- workspace carve
  const size_t BH = (size_t)L.batch * L.heads;
  P->proj_rows = std::max(1, std::min(kProjRows, (kProjSmemFloats - 4) / n));
  P->proj_tiles = (n + P->proj_rows - 1) / P->proj_rows;
  size_t off = 0;
  // K1 pre-split operand tiles (stats.cu): per head ceil(n/128) tiles of 128 rows x D, bf16 hi + lo
  const size_t split_bytes = BH * (size_t)((n + 127) / 128) * 128 * L.head_dim * 2 * sizeof(uint16_t);
  P->ws_qbar = off; off = align_up(off + BH * n * L.head_dim * sizeof(float));
  P->ws_kbar = off; off = align_up(off + BH * n * L.head_dim * sizeof(float));
  P->ws_qs = off;   off = align_up(off + split_bytes, 1024);
  P->ws_ks = off;   off = align_up(off + split_bytes, 1024);
  P->ws_part = off; off = align_up(off + std::max(BH * P->proj_tiles * (size_t)p * sizeof(double),
                                                  BH * (size_t)n * 4 * 2 * sizeof(float)));   // + K1 (m, l) partials
  P->ws_r = off;    off = align_up(off + BH * (size_t)p * sizeof(double));
  P->ws_x = off;    off = align_up(off + BH * (size_t)p * sizeof(double));
  P->ws_nae = off;  off = align_up(off + 2 * BH * (size_t)n * sizeof(double));
  P->ws_sel = off;  off = align_up(off + BH * (size_t)(3 * n));
  P->ws_cnt = off;  off = align_up(off + BH * (size_t)n * sizeof(int));
  {   // solve split-K (fit.cu solve_stream_kernel): one wave of (k tiles x segments x head chunks) CTAs,
      // one per SM (96 KB ring + the segment's r), segments of at most 512 rows l
    const int ktiles = (p + 127) / 128, chunks = BH <= 8 ? 1 : (int)((BH + 23) / 24);
    int segs = std::max(1, P->sm_count / (ktiles * chunks));
    segs = std::max(segs, (p + 511) / 512);
    P->solve_seg_len = (p + segs - 1) / segs;
    P->solve_segs = (p + P->solve_seg_len - 1) / P->solve_seg_len;
  }
  P->ws_solve = off; off = align_up(off + (size_t)P->solve_segs * BH * (size_t)p * sizeof(double));
  P->ws_bytes = off;
  cudaSetDevice(prev_dev);
  P->create_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  *out = P;
  return MOD_OK;
#undef PLAN_CUDA
}

extern "C" void mod_plan_destroy(mod_plan P) {
  if (!P) return;
  if (P->d_frame_ab) cudaFree(P->d_frame_ab);
  if (P->d_row_frames) cudaFree(P->d_row_frames);
  if (P->d_log_sizes) cudaFree(P->d_log_sizes);
  if (P->d_ginv) cudaFree(P->d_ginv);
  delete P;
}

extern "C" size_t mod_plan_workspace_bytes(mod_plan P) { return P ? P->ws_bytes : 0; }
extern "C" int32_t mod_plan_num_blocks(mod_plan P) { return P ? P->n : -1; }
extern "C" int32_t mod_plan_num_patterns(mod_plan P) { return P ? P->p : -1; }
extern "C" const double* mod_plan_gram_inverse(mod_plan P) { return P ? P->d_ginv : nullptr; }
extern "C" int32_t mod_plan_gram_inverse_ld(mod_plan P) { return P ? P->ginv_ld : -1; }
extern "C" int32_t mod_plan_solver(mod_plan P) { return P ? P->solver : -1; }
extern "C" double mod_plan_create_ms(mod_plan P) { return P ? P->create_ms : -1.0; }
extern "C" mod_status mod_plan_diagnostics(mod_plan P, double* min_pivot, int32_t* null_dim) {
  MOD_NVTX("mod_plan_diagnostics");
  MOD_REQUIRE(P, MOD_ERR_USAGE, "mod_plan_diagnostics: NULL plan");
  if (min_pivot) *min_pivot = P->min_pivot;
  if (null_dim) *null_dim = P->null_dim;
  return MOD_OK;
}
extern "C" mod_status mod_plan_frame_blocks(mod_plan P, int32_t* a_b) {
  MOD_NVTX("mod_plan_frame_blocks");
  MOD_REQUIRE(P && a_b, MOD_ERR_USAGE, "mod_plan_frame_blocks: NULL argument");
  for (int i = 0; i < 2 * P->F; ++i) a_b[i] = P->frame_ab[i];
  return MOD_OK;
}
