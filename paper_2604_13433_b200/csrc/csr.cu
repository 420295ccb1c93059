// K4 — CSR SpMV in the reference's row-sequential rounding order.
//
// Replaces csr_spmv (reference matrix.py:272-291): values (f64) and x are
// converted to the working dtype, each row accumulates left to right with one
// rounding per product and per sum, starting from the first product (no +0).
// It is the FP64 operator of the outer FCG / FP64 PCG (solvers.py:121-122,
// 162, 258) and the true-residual audit (solvers.py:162).  One thread per row
// (the 7-point rows of the PCG configs are 7 words); rows are contiguous, so a
// warp's col/value reads cover one contiguous span served by L1.
#include "psell_internal.cuh"

namespace psell {

template <typename XT> struct CsrOps;
template <> struct CsrOps<double> {
  __device__ static double cv(double v) { return v; }
  __device__ static double mul(double a, double b) { return __dmul_rn(a, b); }
  __device__ static double add(double a, double b) { return __dadd_rn(a, b); }
  __device__ static double zero() { return 0.0; }
};
template <> struct CsrOps<float> {
  __device__ static float cv(double v) { return __double2float_rn(v); }
  __device__ static float mul(float a, float b) { return __fmul_rn(a, b); }
  __device__ static float add(float a, float b) { return __fadd_rn(a, b); }
  __device__ static float zero() { return 0.f; }
};
template <> struct CsrOps<__half> {
  __device__ static __half cv(double v) { return __double2half(v); }
  __device__ static __half mul(__half a, __half b) { return __hmul_rn(a, b); }
  __device__ static __half add(__half a, __half b) { return __hadd_rn(a, b); }
  __device__ static __half zero() { return __ushort_as_half(0); }
};

template <typename XT>
__global__ void __launch_bounds__(kBlock) csr_spmv_kernel(long long n, const int64_t* __restrict__ row_ptr,
                                                          const int32_t* __restrict__ col_idx,
                                                          const double* __restrict__ values,
                                                          const XT* __restrict__ x,
                                                          XT* __restrict__ y) {
  using O = CsrOps<XT>;
  const long long i = (long long)blockIdx.x * kBlock + threadIdx.x;
  if (i >= n) return;
  const long long beg = row_ptr[i], end = row_ptr[i + 1];
  XT acc = O::zero();
  if (end > beg) {
    acc = O::mul(O::cv(values[beg]), x[col_idx[beg]]);
    for (long long j = beg + 1; j < end; ++j) acc = O::add(acc, O::mul(O::cv(values[j]), x[col_idx[j]]));
  }
  y[i] = acc;
}

}  // namespace psell

using namespace psell;

extern "C" int psell_csr_spmv(int64_t n_rows, const int64_t* row_ptr, const int32_t* col_idx,
                              const double* values, const void* x, int32_t x_dtype, void* y,
                              void* stream, psell_error* err) {
  if (n_rows <= 0) return ok(err);
  const unsigned grid = (unsigned)ceil_div(n_rows, kBlock);
  cudaStream_t st = as_stream(stream);
  switch (x_dtype) {
    case PSELL_DT_F64:
      csr_spmv_kernel<double><<<grid, kBlock, 0, st>>>(n_rows, row_ptr, col_idx, values,
                                                       static_cast<const double*>(x), static_cast<double*>(y));
      break;
    case PSELL_DT_F32:
      csr_spmv_kernel<float><<<grid, kBlock, 0, st>>>(n_rows, row_ptr, col_idx, values,
                                                      static_cast<const float*>(x), static_cast<float*>(y));
      break;
    case PSELL_DT_F16:
      csr_spmv_kernel<__half><<<grid, kBlock, 0, st>>>(n_rows, row_ptr, col_idx, values,
                                                       static_cast<const __half*>(x), static_cast<__half*>(y));
      break;
    default:
      return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "unsupported x dtype");
  }
  PSELL_CHECK_LAUNCH(err, "psell_csr_spmv");
  return ok(err);
}
