// Device generators for the BASELINE stencil matrices, written straight into
// HBM as CSR (int64 row_ptr, int32 col_idx, f64 values) for a row range
// [row_begin, row_end) — one rank's slab or the whole matrix.
//
// Bitwise equal to the host generators (paper_2604_13433_b200/stencil.py,
// itself equal to reference stencil.py:10-52) followed by the reference
// scalings sym_diag_scale (matrix.py:305-316) or row_sum_scale (294-302):
// the same IEEE f64 sqrt / mul / div, and the row sum accumulated left to
// right from 0 as np.add.at does.
#include "psell_internal.cuh"

namespace psell {

struct Grid {
  long long d0, d1, d2;  // slowest .. fastest
  int box;
  double diag;
  int scale;  // 0 none, 1 sym_diag_scale, 2 row_sum_scale
};

// neighbour k of the stencil in ascending column order; returns false past the end
__device__ __forceinline__ bool nb_offset(const Grid& g, int k, int& a, int& b, int& c) {
  if (g.box) {
    if (k >= 27) return false;
    a = k / 9 - 1;
    b = (k / 3) % 3 - 1;
    c = k % 3 - 1;
    return true;
  }
  // (-1,0,0) (0,-1,0) (0,0,-1) (0,0,0) (0,0,1) (0,1,0) (1,0,0)
  const int t[7][3] = {{-1, 0, 0}, {0, -1, 0}, {0, 0, -1}, {0, 0, 0}, {0, 0, 1}, {0, 1, 0}, {1, 0, 0}};
  if (k >= 7) return false;
  a = t[k][0];
  b = t[k][1];
  c = t[k][2];
  return true;
}

template <bool FILL>
__global__ void gen_kernel(Grid g, long long r0, long long r1, long long* __restrict__ counts,
                           const int64_t* __restrict__ row_ptr, int32_t* __restrict__ col,
                           double* __restrict__ val) {
  const long long i = r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r1) return;
  const long long x2 = i % g.d2, x1 = (i / g.d2) % g.d1, x0 = i / (g.d1 * g.d2);
  const long long s0 = g.d1 * g.d2, s1 = g.d2;
  int a, b, c;
  long long cnt = 0;
  double rsum = 0.0;
  long long t = FILL ? row_ptr[i - r0] : 0;
  for (int k = 0; nb_offset(g, k, a, b, c); ++k) {
    const long long y0 = x0 + a, y1 = x1 + b, y2 = x2 + c;
    if (y0 < 0 || y0 >= g.d0 || y1 < 0 || y1 >= g.d1 || y2 < 0 || y2 >= g.d2) continue;
    const double v = (a == 0 && b == 0 && c == 0) ? g.diag : -1.0;
    if (FILL) {
      col[t] = (int32_t)(y0 * s0 + y1 * s1 + y2);
      val[t] = v;
      ++t;
    }
    rsum = __dadd_rn(rsum, fabs(v));
    ++cnt;
  }
  if (!FILL) {
    counts[i - r0] = cnt;
    return;
  }
  if (g.scale == 1) {
    const double gg = sqrt(fabs(g.diag));
    const double den = __dmul_rn(gg, gg);
    for (long long j = row_ptr[i - r0]; j < t; ++j) val[j] = __ddiv_rn(val[j], den);
  } else if (g.scale == 2) {
    for (long long j = row_ptr[i - r0]; j < t; ++j) val[j] = __ddiv_rn(val[j], rsum);
  }
}

// ---------------------------------------------------------------- power-law (config 4)
// Counter-based: every random number is splitmix64(seed, row, stream, j), so a
// row can be generated independently (GPU slab, CPU sample) and the host
// mirror (stencil.powerlaw_rows) reproduces it bit for bit.
// Only integer hashing and correctly rounded IEEE ops (sqrt, div, mul, add) are
// used, so numpy reproduces every draw exactly:
//   u     = (h >> 11) * 2^-53
//   L_i   = max{k <= 8192 : u <= T_k},  T_k = (4/k)^1.5 from a host table
//           (= min(8192, floor(4 u^(-2/3))): Pareto alpha 1.5 tail, mean ~12)
//   G_i   = max(1, 8192 / L_i); start = max(0, i - 4096)
//   col_{j+1} = col_j + 1 + h1 % (2 G_i)            (a band of ~16K columns around i)
//             + (h2 % 5 == 0 ? h5 % max(1, n / (8 L_i)) : 0)   (far jumps, bounded total drift)
//   the walk stops at n (the row is truncated); value = (0.01 + 0.99 u4) * (h3 & 1 ? -1 : 1)
__host__ __device__ __forceinline__ uint64_t smix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t hrow(uint64_t seed, long long row) {
  return smix(seed ^ ((uint64_t)row * 0xD1B54A32D192ED03ull));
}
__device__ __forceinline__ uint64_t hdraw(uint64_t hr, int stream, long long j) {
  return smix(hr ^ ((uint64_t)stream << 56) ^ (uint64_t)j);
}
__device__ __forceinline__ double u53(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

struct PlParams {
  long long n;
  uint64_t seed;
  const double* thr;  // T_1..T_8192 at thr[0..8191], non-increasing
};

template <bool FILL>
__global__ void powerlaw_kernel(PlParams P, long long r0, long long r1, long long* __restrict__ counts,
                                const int64_t* __restrict__ row_ptr, int32_t* __restrict__ col,
                                double* __restrict__ val) {
  const long long i = r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r1) return;
  const uint64_t hr = hrow(P.seed, i);
  const double u = u53(hdraw(hr, 0, 0));
  // L = number of leading thresholds >= u (binary search on the non-increasing table)
  int lo = 0, hi = 8192;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (P.thr[mid] >= u) lo = mid + 1;
    else hi = mid;
  }
  const long long L = lo < 1 ? 1 : lo;
  const uint64_t G2 = 2ull * (uint64_t)(8192 / L > 1 ? 8192 / L : 1);
  const long long fj = P.n / (8 * L);
  const uint64_t far = (uint64_t)(fj > 0 ? fj : 1);
  long long c = i - 4096;
  if (c < 0) c = 0;
  long long t = FILL ? row_ptr[i - r0] : 0;
  long long cnt = 0;
  for (long long j = 0; j < L && c < P.n; ++j) {
    if (FILL) {
      col[t] = (int32_t)c;
      const double m = __dadd_rn(0.01, __dmul_rn(0.99, u53(hdraw(hr, 4, j))));
      val[t] = (hdraw(hr, 3, j) & 1ull) ? -m : m;
      ++t;
    }
    ++cnt;
    c += 1 + (long long)(hdraw(hr, 1, j) % G2);
    if (hdraw(hr, 2, j) % 5ull == 0ull) c += (long long)(hdraw(hr, 5, j) % far);
  }
  if (!FILL) counts[i - r0] = cnt;
}

// ---------------------------------------------------------------- far-column power-law (config 4b)
// SURVEY §8d's proposal: the same Pareto row lengths, but ~20 % of a row's entries
// uniform over [0, n) instead of near the diagonal, so the lower bandwidth k_left
// is ~n, every base offset d_i is 0 and the first gap of a row is its first column
// (the dummy-heavy far-gap regime).  Counter-based like config 4:
//   L_i    as config 4 (stream 0)
//   far_j  = h(2, j) % 5 == 0 for j < L_i; m_f = #far, m_n = L_i - m_f
//   near   : c = max(0, i - 4096) + h(6, 0) % 1024, then c += 1 + h(1, k) % G2,
//            G2 = 2 max(1, 8192 / max(m_n, 1))            (a band of ~16 K columns)
//   far    : S = max(1, n / (m_f + 1)), c = h(5, 0) % S, then c += 1 + h(7, k) % (2 S)
//   row    = sorted union of the two increasing walks below n (a column both walks
//            reach is stored once); value(col) = (0.01 + 0.99 u53(h(4, col))) * (h(3, col) & 1 ? -1 : 1)
__device__ __forceinline__ double far_value(uint64_t hr, long long c) {
  const double m = __dadd_rn(0.01, __dmul_rn(0.99, u53(hdraw(hr, 4, c))));
  return (hdraw(hr, 3, c) & 1ull) ? -m : m;
}

template <bool FILL>
__global__ void powerlaw_far_kernel(PlParams P, long long r0, long long r1, long long* __restrict__ counts,
                                    const int64_t* __restrict__ row_ptr, int32_t* __restrict__ col,
                                    double* __restrict__ val) {
  const long long i = r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r1) return;
  const uint64_t hr = hrow(P.seed, i);
  const double u = u53(hdraw(hr, 0, 0));
  int lo = 0, hi = 8192;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (P.thr[mid] >= u) lo = mid + 1;
    else hi = mid;
  }
  const long long L = lo < 1 ? 1 : lo;
  long long mf = 0;
  for (long long j = 0; j < L; ++j) mf += hdraw(hr, 2, j) % 5ull == 0ull;
  const long long mn = L - mf;
  const uint64_t G2 = 2ull * (uint64_t)(8192 / (mn > 1 ? mn : 1) > 1 ? 8192 / (mn > 1 ? mn : 1) : 1);
  const long long Sl = P.n / (mf + 1);
  const uint64_t S = (uint64_t)(Sl > 1 ? Sl : 1);
  long long cn = (i - 4096 > 0 ? i - 4096 : 0) + (long long)(hdraw(hr, 6, 0) % 1024ull);
  long long cf = (long long)(hdraw(hr, 5, 0) % S);
  long long kn = 0, kf = 0;
  long long t = FILL ? row_ptr[i - r0] : 0;
  long long cnt = 0;
  const long long BIG = 1ll << 62;
  for (;;) {
    const long long a = (kn < mn && cn < P.n) ? cn : BIG;
    const long long b = (kf < mf && cf < P.n) ? cf : BIG;
    const long long c = a < b ? a : b;
    if (c == BIG) break;
    if (FILL) {
      col[t] = (int32_t)c;
      val[t] = far_value(hr, c);
      ++t;
    }
    ++cnt;
    if (a == c) {
      cn += 1 + (long long)(hdraw(hr, 1, kn) % G2);
      ++kn;
    }
    if (b == c) {
      cf += 1 + (long long)(hdraw(hr, 7, kf) % (2ull * S));
      ++kf;
    }
  }
  if (!FILL) counts[i - r0] = cnt;
}

}  // namespace psell

using namespace psell;

extern "C" PSELL_API int psell_gen_powerlaw_plan(int64_t n, uint64_t seed, const double* thresholds, int64_t row_begin, int64_t row_end,
                                                 void* ws, size_t ws_bytes, int64_t* row_ptr,
                                                 int64_t* nnz_host, void* stream, psell_error* err) {
  const long long m = row_end - row_begin;
  if (m < 0 || row_end > n) return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, "bad row range");
  if (!ws || ws_bytes < psell_gen_workspace_bytes(m)) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "workspace too small");
  cudaStream_t st = as_stream(stream);
  long long* counts = static_cast<long long*>(ws);
  long long* tmp = reinterpret_cast<long long*>(static_cast<char*>(ws) + align_up(8 * (size_t)(m > 0 ? m : 1)));
  PlParams P{n, seed, thresholds};
  if (m > 0) powerlaw_kernel<false><<<(unsigned)ceil_div(m, kBlock), kBlock, 0, st>>>(P, row_begin, row_end, counts, nullptr, nullptr, nullptr);
  PSELL_CHECK_LAUNCH(err, "powerlaw_count");
  if (int rc = scan_i64(counts, m, tmp, reinterpret_cast<long long*>(row_ptr), st, err)) return rc;
  long long nnz = 0;
  PSELL_CUDA(cudaMemcpyAsync(&nnz, row_ptr + m, 8, cudaMemcpyDeviceToHost, st), err);
  PSELL_CUDA(cudaStreamSynchronize(st), err);
  *nnz_host = nnz;
  return ok(err);
}

extern "C" PSELL_API int psell_gen_powerlaw_fill(int64_t n, uint64_t seed, const double* thresholds, int64_t row_begin, int64_t row_end,
                                                 const int64_t* row_ptr, int32_t* col_idx, double* values,
                                                 void* stream, psell_error* err) {
  const long long m = row_end - row_begin;
  if (m <= 0) return ok(err);
  PlParams P{n, seed, thresholds};
  powerlaw_kernel<true><<<(unsigned)ceil_div(m, kBlock), kBlock, 0, as_stream(stream)>>>(P, row_begin, row_end, nullptr, row_ptr, col_idx, values);
  PSELL_CHECK_LAUNCH(err, "powerlaw_fill");
  return ok(err);
}

extern "C" PSELL_API int psell_gen_powerlaw_far_plan(int64_t n, uint64_t seed, const double* thresholds,
                                                     int64_t row_begin, int64_t row_end, void* ws, size_t ws_bytes,
                                                     int64_t* row_ptr, int64_t* nnz_host, void* stream,
                                                     psell_error* err) {
  const long long m = row_end - row_begin;
  if (m < 0 || row_end > n) return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, "bad row range");
  if (!ws || ws_bytes < psell_gen_workspace_bytes(m)) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "workspace too small");
  cudaStream_t st = as_stream(stream);
  long long* counts = static_cast<long long*>(ws);
  long long* tmp = reinterpret_cast<long long*>(static_cast<char*>(ws) + align_up(8 * (size_t)(m > 0 ? m : 1)));
  PlParams P{n, seed, thresholds};
  if (m > 0) powerlaw_far_kernel<false><<<(unsigned)ceil_div(m, kBlock), kBlock, 0, st>>>(P, row_begin, row_end, counts, nullptr, nullptr, nullptr);
  PSELL_CHECK_LAUNCH(err, "powerlaw_far_count");
  if (int rc = scan_i64(counts, m, tmp, reinterpret_cast<long long*>(row_ptr), st, err)) return rc;
  long long nnz = 0;
  PSELL_CUDA(cudaMemcpyAsync(&nnz, row_ptr + m, 8, cudaMemcpyDeviceToHost, st), err);
  PSELL_CUDA(cudaStreamSynchronize(st), err);
  *nnz_host = nnz;
  return ok(err);
}

extern "C" PSELL_API int psell_gen_powerlaw_far_fill(int64_t n, uint64_t seed, const double* thresholds,
                                                     int64_t row_begin, int64_t row_end, const int64_t* row_ptr,
                                                     int32_t* col_idx, double* values, void* stream, psell_error* err) {
  const long long m = row_end - row_begin;
  if (m <= 0) return ok(err);
  PlParams P{n, seed, thresholds};
  powerlaw_far_kernel<true><<<(unsigned)ceil_div(m, kBlock), kBlock, 0, as_stream(stream)>>>(P, row_begin, row_end, nullptr, row_ptr, col_idx, values);
  PSELL_CHECK_LAUNCH(err, "powerlaw_far_fill");
  return ok(err);
}

extern "C" {

PSELL_API size_t psell_gen_workspace_bytes(int64_t n_rows) {
  const long long n = n_rows > 0 ? n_rows : 1;
  return align_up(8 * (size_t)n) + align_up(8 * (size_t)(ceil_div(n, 4096) + 4096 + 1));
}

PSELL_API int psell_gen_stencil_plan(int64_t d0, int64_t d1, int64_t d2, int32_t box, double diag,
                                     int64_t row_begin, int64_t row_end, void* ws, size_t ws_bytes,
                                     int64_t* row_ptr, int64_t* nnz_host, void* stream,
                                     psell_error* err) {
  const long long n = row_end - row_begin;
  if (n < 0 || d0 < 1 || d1 < 1 || d2 < 1 || row_end > d0 * d1 * d2)
    return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, "bad grid or row range");
  if (!ws || ws_bytes < psell_gen_workspace_bytes(n)) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "workspace too small");
  cudaStream_t st = as_stream(stream);
  long long* counts = static_cast<long long*>(ws);
  long long* tmp = reinterpret_cast<long long*>(static_cast<char*>(ws) + align_up(8 * (size_t)(n > 0 ? n : 1)));
  Grid g{d0, d1, d2, box, diag, 0};
  if (n > 0) gen_kernel<false><<<(unsigned)ceil_div(n, kBlock), kBlock, 0, st>>>(g, row_begin, row_end, counts, nullptr, nullptr, nullptr);
  PSELL_CHECK_LAUNCH(err, "gen_count");
  if (int rc = scan_i64(counts, n, tmp, reinterpret_cast<long long*>(row_ptr), st, err)) return rc;
  long long nnz = 0;
  PSELL_CUDA(cudaMemcpyAsync(&nnz, row_ptr + n, 8, cudaMemcpyDeviceToHost, st), err);
  PSELL_CUDA(cudaStreamSynchronize(st), err);
  *nnz_host = nnz;
  return ok(err);
}

PSELL_API int psell_gen_stencil_fill(int64_t d0, int64_t d1, int64_t d2, int32_t box, double diag,
                                     int32_t scale, int64_t row_begin, int64_t row_end,
                                     const int64_t* row_ptr, int32_t* col_idx, double* values,
                                     void* stream, psell_error* err) {
  const long long n = row_end - row_begin;
  if (n <= 0) return ok(err);
  Grid g{d0, d1, d2, box, diag, scale};
  gen_kernel<true><<<(unsigned)ceil_div(n, kBlock), kBlock, 0, as_stream(stream)>>>(g, row_begin, row_end, nullptr, row_ptr, col_idx, values);
  PSELL_CHECK_LAUNCH(err, "gen_fill");
  return ok(err);
}

}  // extern "C"
