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

}  // namespace psell

using namespace psell;

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
