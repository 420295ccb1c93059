// K6 — backward error of an SpMV output, one pass over the CSR (sm_100a).
//
// Replaces the numpy body of backward_error / inf_norm_matrix (reference
// metrics.py:43-66):  || y - A x ||_inf / (||A||_inf ||x||_inf)  in float64
// against the unquantised A.  Thread i owns row i and, in the same pass,
// entry i of x:
//   resid_i = y_i - (A x)_i   with (A x)_i accumulated left to right, one
//                              rounding per product and per sum, from the first
//                              product (csr_spmv, matrix.py:272-291, same as K4)
//   rowsum_i = sum_j |a_ij|   left to right (np.add.at order, metrics.py:46-49)
// and the three maxima (|resid|, rowsum, |x|) reduce through a warp/CTA max
// and one atomicMax per CTA on the IEEE bit pattern: for non-negative doubles
// the unsigned order is the numeric order and a NaN (0x7FF8...) beats +inf, so
// NaN propagates like numpy's max.  The result is order independent, hence
// bit-identical to the reference.  HBM-bound: 8(n+1) + 12 nnz + 8 n_rows (y,
// f64) + 8 n_cols (x) bytes (+ the x gathers, L2 resident).
#include "psell_internal.cuh"

namespace psell {

template <typename T> __device__ __forceinline__ double wide(T v);
template <> __device__ __forceinline__ double wide<double>(double v) { return v; }
template <> __device__ __forceinline__ double wide<float>(float v) { return (double)v; }
template <> __device__ __forceinline__ double wide<__half>(__half v) { return (double)__half2float(v); }

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, v, o);
    v = t > v ? t : v;
  }
  return v;
}

template <typename XT, typename YT>
__global__ void __launch_bounds__(kBlock) backward_error_kernel(
    long long n_rows, long long n_cols, const int64_t* __restrict__ row_ptr,
    const int32_t* __restrict__ col_idx, const double* __restrict__ values, const XT* __restrict__ x,
    const YT* __restrict__ y, unsigned long long* __restrict__ out /* [3]: |r|, rowsum, |x| */) {
  __shared__ unsigned long long sh[3][kBlock / 32];
  const long long n = n_rows > n_cols ? n_rows : n_cols;
  unsigned long long mr = 0, ms = 0, mx = 0;
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long long)gridDim.x * kBlock) {
    if (i < n_rows) {
      const long long beg = row_ptr[i], end = row_ptr[i + 1];
      double acc = 0.0, rs = 0.0;
      if (end > beg) {
        const double v0 = values[beg];
        acc = __dmul_rn(v0, wide<XT>(x[col_idx[beg]]));
        rs = fabs(v0);
        for (long long j = beg + 1; j < end; ++j) {
          const double v = values[j];
          acc = __dadd_rn(acc, __dmul_rn(v, wide<XT>(x[col_idx[j]])));
          rs = __dadd_rn(rs, fabs(v));
        }
      }
      const unsigned long long r = (unsigned long long)__double_as_longlong(fabs(__dsub_rn(wide<YT>(y[i]), acc)));
      const unsigned long long s = (unsigned long long)__double_as_longlong(rs);
      mr = r > mr ? r : mr;
      ms = s > ms ? s : ms;
    }
    if (i < n_cols) {
      const unsigned long long a = (unsigned long long)__double_as_longlong(fabs(wide<XT>(x[i])));
      mx = a > mx ? a : mx;
    }
  }
  mr = warp_max_u64(mr);
  ms = warp_max_u64(ms);
  mx = warp_max_u64(mx);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sh[0][warp] = mr;
    sh[1][warp] = ms;
    sh[2][warp] = mx;
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      unsigned long long v = lane < kBlock / 32 ? sh[q][lane] : 0ull;
      v = warp_max_u64(v);
      if (lane == 0 && v) atomicMax(out + q, v);
    }
  }
}

template <typename XT>
static int launch_be(long long n_rows, long long n_cols, const int64_t* rp, const int32_t* ci, const double* v,
                     const void* x, const void* y, int32_t y_dtype, unsigned long long* out, unsigned grid,
                     cudaStream_t st) {
  const XT* xp = static_cast<const XT*>(x);
  switch (y_dtype) {
    case PSELL_DT_F64:
      backward_error_kernel<XT, double><<<grid, kBlock, 0, st>>>(n_rows, n_cols, rp, ci, v, xp,
                                                                 static_cast<const double*>(y), out);
      return 0;
    case PSELL_DT_F32:
      backward_error_kernel<XT, float><<<grid, kBlock, 0, st>>>(n_rows, n_cols, rp, ci, v, xp,
                                                                static_cast<const float*>(y), out);
      return 0;
    case PSELL_DT_F16:
      backward_error_kernel<XT, __half><<<grid, kBlock, 0, st>>>(n_rows, n_cols, rp, ci, v, xp,
                                                                 static_cast<const __half*>(y), out);
      return 0;
  }
  return 1;
}

}  // namespace psell

using namespace psell;

extern "C" int psell_backward_error(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                                    const int32_t* col_idx, const double* values, const void* x,
                                    int32_t x_dtype, const void* y, int32_t y_dtype, double* out,
                                    void* stream, psell_error* err) {
  if (!out) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "null output");
  cudaStream_t st = as_stream(stream);
  PSELL_CUDA(cudaMemsetAsync(out, 0, 3 * sizeof(double), st), err);
  const long long n = n_rows > n_cols ? n_rows : n_cols;
  if (n <= 0) return ok(err);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long full = ceil_div(n, kBlock);
  const unsigned grid = (unsigned)(full < 8LL * sms ? full : 8LL * sms);  // persistent: 8 CTAs per SM
  auto* o = reinterpret_cast<unsigned long long*>(out);
  int bad = 1;
  switch (x_dtype) {
    case PSELL_DT_F64: bad = launch_be<double>(n_rows, n_cols, row_ptr, col_idx, values, x, y, y_dtype, o, grid, st); break;
    case PSELL_DT_F32: bad = launch_be<float>(n_rows, n_cols, row_ptr, col_idx, values, x, y, y_dtype, o, grid, st); break;
    case PSELL_DT_F16: bad = launch_be<__half>(n_rows, n_cols, row_ptr, col_idx, values, x, y, y_dtype, o, grid, st); break;
  }
  if (bad) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "unsupported x / y dtype");
  PSELL_CHECK_LAUNCH(err, "psell_backward_error");
  return ok(err);
}
