// predict.cu -- K2b mod_predict_block_mask (+ the dense all-ones mask helper).
//
// Per head:
//  1. linear prediction (§5.2 Eq. 6, Eq. 7) of the C and D
//     intensities, evaluated in IEEE fp64 without contraction so that the integer decisions below
//     match the oracle bit for bit:  d = x_c - x_p;  s = d / (t_c - t_p);  x_hat = x_c + s*(t - t_c);
//  2. selection over the 3n-1 pool (§5.3; reading Z3: keys descending, Z14: ties by id):
//     TOPK takes the K-th largest key by a radix select (no sort); TOPMASS sorts the (key, id)
//     pairs with an in-shared-memory bitonic network; THRESHOLD compares directly.  TOPMASS accumulates max(key,0)*|supp| sequentially in sorted order;
//  3. block mask = selected diagonals (j - i = delta_k) | selected columns | kept frame squares
//     [a_r,b_r]^2 | diagonal guard | prefix rows/columns (Alg. 1; Z15, Z17),
//     emitted as a CSR index list.  Steps 1 (one CTA per head), 2 (row counts) and 3 (row
//     pointers + column lists) are separate launches so that the mask work spreads over
//     (row chunk, head) CTAs: a warp per row, 32 columns per lane-word built from bit strings.
#include "common.cuh"

namespace {

__device__ __forceinline__ bool before(double ka, int ia, double kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}


// Order-preserving map of a double to uint64 (larger key -> larger code; -0 folded onto +0 so that
// equal keys compare equal, as in the oracle's numeric comparison).
__device__ __forceinline__ unsigned long long key_code(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x == 0.0 ? 0.0 : x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Radix select, one CTA: the k-th largest (k >= 1) of the values code(e) over the elements e < P for
// which pred(e) holds, BITS wide, 8 bits per pass from the top.  Returns the value; `hist` is a
// 256-int shared buffer.  All threads must call it.
template <int BITS, typename Code, typename Pred>
__device__ unsigned long long radix_kth_largest(int P, int k, Code code, Pred pred, int* hist) {
  __shared__ unsigned long long s_prefix;
  __shared__ int s_k;
  const int t = threadIdx.x;
  unsigned long long prefix = 0, mask = 0;
  for (int shift = BITS - 8; shift >= 0; shift -= 8) {
    for (int b = t; b < 256; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (int e = t; e < P; e += blockDim.x) {
      if (!pred(e)) continue;
      const unsigned long long c = code(e);
      if ((c & mask) == prefix) atomicAdd(&hist[(c >> shift) & 255], 1);
    }
    __syncthreads();
    if (t < 32) {
      // lane l owns bins [255 - 8l - 7, 255 - 8l] (from the top); warp scan of the lane sums
      int own = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) own += hist[255 - 8 * t - u];
      int incl = own;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (t >= o) incl += y;
      }
      const int excl = incl - own;
      const unsigned hit = __ballot_sync(0xffffffffu, incl >= k && excl < k);
      const int lane = __ffs(hit) - 1;
      if (t == lane) {
        int cum = excl;
        for (int u = 0; u < 8; ++u) {
          const int bin = 255 - 8 * t - u;
          if (cum + hist[bin] >= k) {
            s_prefix = prefix | ((unsigned long long)bin << shift);
            s_k = k - cum;
            break;
          }
          cum += hist[bin];
        }
      }
    }
    __syncthreads();
    prefix = s_prefix;
    k = s_k;
    mask |= 255ull << shift;
    __syncthreads();
  }
  return prefix;
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
  if (a.mode == MOD_SELECT_TOPK && P <= 0xffff) {
    // Top-K by radix select instead of a full sort: T = the K-th largest key code; every key above T
    // is in, and of the keys equal to T the lowest ids fill the remaining places (reading Z14: key
    // descending, ties by ascending pattern id) -- the same set the sorted order gives.
    __shared__ int hist[256];
    __shared__ int n_above;
    const int K = min(a.top_k, P);
    if (K >= P) {
      for (int e = t; e < P; e += blockDim.x) sel[e] = 1;
      return;
    }
    const unsigned long long T = radix_kth_largest<64>(
        P, K, [&](int e) { return key_code(keys[e]); }, [](int) { return true; }, hist);
    if (t == 0) n_above = 0;
    __syncthreads();
    int mine = 0;
    for (int e = t; e < P; e += blockDim.x) mine += key_code(keys[e]) > T;
    mine = __reduce_add_sync(0xffffffffu, mine);
    if ((t & 31) == 0) atomicAdd(&n_above, mine);
    __syncthreads();
    const int m = K - n_above;   // >= 1 places for keys equal to T, lowest ids first
    const unsigned long long id_code = radix_kth_largest<16>(
        P, m, [&](int e) { return (unsigned long long)(0xffff - e); },
        [&](int e) { return key_code(keys[e]) == T; }, hist);
    const int max_id = 0xffff - (int)id_code;
    for (int e = t; e < P; e += blockDim.x) {
      const unsigned long long c = key_code(keys[e]);
      sel[e] = c > T || (c == T && e <= max_id);
    }
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

// The passing set of row i is a union of shifted / fixed bit strings: the selected
// diagonals are the C selection bits read through a window that slides with i, the selected columns
// the D selection bits, kept frame squares and the prefix contiguous ranges, the guard one bit.
// Rows are therefore built 32 columns per lane-word (funnel shift + range masks) instead of testing
// the n columns one by one.
struct RowBits {
  const uint32_t* cbits;   // smem: bit k = C_k selected (k in [0, 2n-1)), zero padded
  const uint32_t* dbits;   // smem: bit j = D_j selected
  const uint8_t* keep;     // global [F] or null
  const int* frame_ab;
  const int* row_frames;
  int n, prefix_last, diag_guard;
};

__device__ __forceinline__ uint32_t range_bits(int a, int b, int j0) {   // bits of [a, b] in word [j0, j0+32)
  const int lo = max(a, j0), hi = min(b, j0 + 31);
  if (lo > hi) return 0u;
  return (0xffffffffu >> (31 - (hi - lo))) << (lo - j0);
}

__device__ __forceinline__ uint32_t row_word(const RowBits& c, int i, int w) {
  const int n = c.n, j0 = 32 * w;
  if (j0 >= n) return 0u;
  uint32_t m = c.dbits[w];
  const int o = n - 1 - i + j0;                 // C bit of column j0: delta = j0 - i
  m |= __funnelshift_r(c.cbits[o >> 5], c.cbits[(o >> 5) + 1], o & 31);
  if (c.diag_guard && (i >> 5) == w) m |= 1u << (i & 31);
  if (c.prefix_last >= 0) m |= (i <= c.prefix_last) ? 0xffffffffu : range_bits(0, c.prefix_last, j0);
  if (c.keep) {
    const int rlo = c.row_frames[2 * i], rhi = c.row_frames[2 * i + 1];
    for (int r = rlo; r <= rhi; ++r)
      if (c.keep[r]) m |= range_bits(c.frame_ab[2 * r], c.frame_ab[2 * r + 1], j0);
  }
  if (j0 + 32 > n) m &= (1u << (n - j0)) - 1u;
  return m;
}

// selection bytes of head bh -> bit strings in shared memory (warp per word, ballot)
__device__ __forceinline__ RowBits load_row_bits(const PredictArgs& a, uint32_t* s_bits, size_t bh) {
  const int n = a.n, P = 3 * n - 1;
  const int wc = (2 * n + 63) / 32 + 1, wd = (n + 31) / 32;
  const uint8_t* g = a.sel + bh * P;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int w = warp; w < wc + wd; w += nw) {
    bool bit;
    if (w < wc) {
      const int k = 32 * w + lane;
      bit = k < 2 * n - 1 && g[k];
    } else {
      const int j = 32 * (w - wc) + lane;
      bit = j < n && g[2 * n - 1 + j];
    }
    const uint32_t m = __ballot_sync(0xffffffffu, bit);
    if (lane == 0) s_bits[w] = m;
  }
  __syncthreads();
  RowBits c;
  c.cbits = s_bits;
  c.dbits = s_bits + wc;
  c.keep = a.keep ? a.keep + bh * a.F : nullptr;
  c.frame_ab = a.frame_ab;
  c.row_frames = a.row_frames;
  c.n = n;
  c.prefix_last = a.prefix_last;
  c.diag_guard = a.diag_guard;
  return c;
}

// 2. passing blocks per row: warp per row, lane-words of 32 columns (n <= 2048: <= 2 words per lane)
__global__ void __launch_bounds__(256) count_kernel(PredictArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const size_t bh = blockIdx.y;
  const RowBits c = load_row_bits(a, reinterpret_cast<uint32_t*>(smem), bh);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, n = a.n;
  for (int r = 0; r < kRowsPerCta / 8; ++r) {
    const int i = blockIdx.x * kRowsPerCta + warp * (kRowsPerCta / 8) + r;
    if (i >= n) break;
    int cnt = __popc(row_word(c, i, lane)) + __popc(row_word(c, i, lane + 32));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) a.cnt[bh * n + i] = cnt;
  }
}

// 3. row pointers (prefix over the counts) and ascending column lists
__global__ void __launch_bounds__(256) write_kernel(PredictArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int red[8];
  __shared__ int rowoff[kRowsPerCta + 1];
  const size_t bh = blockIdx.y;
  const RowBits c = load_row_bits(a, reinterpret_cast<uint32_t*>(smem), bh);
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
#pragma unroll
    for (int h = 0; h < 2; ++h) {   // words 0..31, then 32..63: ascending columns
      uint32_t m = row_word(c, i, lane + 32 * h);
      const int pc = __popc(m);
      int incl = pc;                 // inclusive warp scan of the lane counts
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int q = pos + incl - pc;
      const int j0 = 32 * (lane + 32 * h);
      while (m) {
        const int b = __ffs(m) - 1;
        ci[q++] = j0 + b;
        m &= m - 1u;
      }
      pos += __shfl_sync(0xffffffffu, incl, 31);
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
  MOD_NVTX("mod_predict_block_mask");
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
  const size_t rsm = (size_t)((2 * P->n + 63) / 32 + 1 + (P->n + 31) / 32) * sizeof(uint32_t);
  count_kernel<<<rg, 256, rsm, s>>>(a);
  MOD_LAUNCH_CHECK();
  write_kernel<<<rg, 256, rsm, s>>>(a);
  MOD_LAUNCH_CHECK();
  mod_note_launches(3);
  return MOD_OK;
}

extern "C" mod_status mod_fill_dense_mask(mod_plan P, int32_t* row_ptr, int32_t* col_idx, void* stream) {
  MOD_NVTX("mod_fill_dense_mask");
  mod_status st = mod_validate_plan(P);
  if (st != MOD_OK) return st;
  MOD_REQUIRE(row_ptr && col_idx, MOD_ERR_USAGE, "mod_fill_dense_mask: NULL argument");
  const int BH = P->L.batch * P->L.heads;
  dense_mask_kernel<<<dim3(P->n, BH), 256, 0, as_stream(stream)>>>(row_ptr, col_idx, P->n);
  MOD_LAUNCH_CHECK();
  mod_note_launches(1);
  return MOD_OK;
}
