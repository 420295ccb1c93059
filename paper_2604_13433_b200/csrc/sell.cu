// SELL-C-sigma comparator format on sm_100a: the FP64 / FP32 /
// FP16 sliced-ELL baseline of the reference (sell.py:49-204), used by
// make_backend("sell64" | "sell32" | "sell16") and the FP32 IO-CG comparator.
//
// The layout plan (widths from row lengths, stable descending sigma-block
// sort, int64 offsets, perm) is the PackSELL plan with a format that can never
// emit a dummy word (W = 64, D = 31), so it is shared with K1.  The fill writes
// values converted to the value dtype (direct RNE) and int32 columns; padding
// carries value 0 and the row's last column (0 for empty rows) (sell.py:161-172).
// The SpMV reproduces sell_spmv's numpy rounding: values cast to x's dtype,
// accumulator from 0, one rounding per product and per sum (sell.py:181-204).
#include "psell_internal.cuh"

#include <cstdlib>
#include <cstring>

namespace psell {

template <typename V> __device__ __forceinline__ V from_f64(double v);
template <> __device__ __forceinline__ double from_f64<double>(double v) { return v; }
template <> __device__ __forceinline__ float from_f64<float>(double v) { return __double2float_rn(v); }
template <> __device__ __forceinline__ __half from_f64<__half>(double v) { return __double2half(v); }

template <typename V>
__global__ void __launch_bounds__(kBlock) sell_fill_kernel(const int64_t* __restrict__ row_ptr,
                                                           const int32_t* __restrict__ col_idx,
                                                           const double* __restrict__ values,
                                                           const int32_t* __restrict__ order,
                                                           const int64_t* __restrict__ offset, long long n,
                                                           long long n_slices, int c, V* __restrict__ val,
                                                           int32_t* __restrict__ col) {
  const long long s = (long long)blockIdx.x * kBlock + threadIdx.x;
  if (s >= n_slices * c) return;
  const long long k = s / c, lane = s - k * c;
  const long long o = offset[k];
  const long long width = (offset[k + 1] - o) / c;
  long long q = 0;
  int32_t last = 0;
  if (s < n) {
    const long long r = order ? (long long)order[s] : s;
    const long long beg = row_ptr[r], end = row_ptr[r + 1];
    for (long long j = beg; j < end; ++j, ++q) {
      const long long pos = o + lane + q * c;
      val[pos] = from_f64<V>(values[j]);
      col[pos] = col_idx[j];
    }
    if (end > beg) last = col_idx[end - 1];
  }
  for (; q < width; ++q) {
    const long long pos = o + lane + q * c;
    val[pos] = from_f64<V>(0.0);
    col[pos] = last;
  }
}

// value (stored dtype VT) -> x dtype XT, numpy astype semantics (RNE)
template <typename VT, typename XT> __device__ __forceinline__ XT vcast(VT v);
template <> __device__ __forceinline__ double vcast<double, double>(double v) { return v; }
template <> __device__ __forceinline__ float vcast<double, float>(double v) { return __double2float_rn(v); }
template <> __device__ __forceinline__ __half vcast<double, __half>(double v) { return __double2half(v); }
template <> __device__ __forceinline__ double vcast<float, double>(float v) { return (double)v; }
template <> __device__ __forceinline__ float vcast<float, float>(float v) { return v; }
template <> __device__ __forceinline__ __half vcast<float, __half>(float v) { return __float2half_rn(v); }
template <> __device__ __forceinline__ double vcast<__half, double>(__half v) { return (double)__half2float(v); }
template <> __device__ __forceinline__ float vcast<__half, float>(__half v) { return __half2float(v); }
template <> __device__ __forceinline__ __half vcast<__half, __half>(__half v) { return v; }

template <typename T> struct RefOps;
template <> struct RefOps<double> {
  __device__ static double step(double a, double v, double x) { return __dadd_rn(a, __dmul_rn(v, x)); }
  __device__ static double zero() { return 0.0; }
};
template <> struct RefOps<float> {
  __device__ static float step(float a, float v, float x) { return __fadd_rn(a, __fmul_rn(v, x)); }
  __device__ static float zero() { return 0.f; }
};
template <> struct RefOps<__half> {
  __device__ static __half step(__half a, __half v, __half x) { return __hadd_rn(a, __hmul_rn(v, x)); }
  __device__ static __half zero() { return __ushort_as_half(0); }
};

template <typename VT, typename XT>
__global__ void __launch_bounds__(kBlock) sell_spmv_kernel(const VT* __restrict__ val,
                                                           const int32_t* __restrict__ col,
                                                           const int64_t* __restrict__ offset,
                                                           const void* perm, int perm_bytes, int implicit,
                                                           int sigma, long long n_rows, int c,
                                                           const XT* __restrict__ x, XT* __restrict__ y) {
  const long long s = (long long)blockIdx.x * kBlock + threadIdx.x;
  if (s >= n_rows) return;
  const long long k = s / c, lane = s - k * c;
  const long long o = offset[k];
  const long long width = (offset[k + 1] - o) / c;
  XT acc = RefOps<XT>::zero();
  for (long long q = 0; q < width; ++q) {
    const long long pos = o + lane + q * c;
    acc = RefOps<XT>::step(acc, vcast<VT, XT>(val[pos]), x[col[pos]]);
  }
  long long out = s;
  if (implicit) {
    const long long p = perm_bytes == 1 ? (long long)static_cast<const uint8_t*>(perm)[s]
                                        : (long long)static_cast<const uint16_t*>(perm)[s];
    out = (s / sigma) * sigma + p;
  }
  y[out] = acc;
}

// C == 32 fast path: a warp per slice (lane = row), 8-step chunks whose value
// and column loads (coalesced 128-B lines, evict-first) are all issued before
// the 8 gathers, which are issued before the first dependent add; 32-bit index
// math.  Same per-row operation order as sell_spmv_kernel (bitwise equal).
// PSELL_SELL=generic forces the one-thread-per-row kernel (A/B)
static bool sell_generic() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PSELL_SELL");
    v = e && strcmp(e, "generic") == 0;
  }
  return v != 0;
}

template <typename VT, typename XT>
__global__ void __launch_bounds__(kBlock, 6) sell_spmv_c32_kernel(const VT* __restrict__ val,
                                                                  const int32_t* __restrict__ col,
                                                                  const int64_t* __restrict__ offset,
                                                                  const void* perm, int perm_bytes, int implicit,
                                                                  unsigned sigma, long long n_rows,
                                                                  long long n_slices, const XT* __restrict__ x,
                                                                  XT* __restrict__ y) {
  constexpr int U = 8;
  const long long k = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= n_slices) return;
  const long long o = offset[k];
  const int width = (int)((offset[k + 1] - o) >> 5);
  const VT* pv = val + o + lane;
  const int32_t* pc = col + o + lane;
  XT acc = RefOps<XT>::zero();
  for (int q = 0; q < width; q += U) {
    VT v[U];
    int32_t c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool in = q + u < width;
      v[u] = in ? __ldcs(pv + (q + u) * 32) : VT(0);
      c[u] = in ? __ldcs(pc + (q + u) * 32) : 0;
    }
    XT xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = x[c[u]];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (q + u < width) acc = RefOps<XT>::step(acc, vcast<VT, XT>(v[u]), xv[u]);
  }
  const unsigned s = (unsigned)(k * 32) + lane;
  if ((long long)s >= n_rows) return;
  unsigned out = s;
  if (implicit) {
    const unsigned pp = perm_bytes == 1 ? (unsigned)static_cast<const uint8_t*>(perm)[s]
                                        : (unsigned)static_cast<const uint16_t*>(perm)[s];
    out = (s / sigma) * sigma + pp;
  }
  y[out] = acc;
}

// The FP32 IO-CG comparator's inner operator fused like the PackSELL one (psell_spmv_dot_alpha):
// sell_spmv_c32_kernel's SpMV (same per-row order: bitwise y) plus this thread's rows of
// p_own . y in FP64, the CTA sums as partials and, in the last CTA, the fixed-order total and
// the alpha step -- one launch instead of SpMV, dot and alpha.
template <typename VT, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) sell_spmv_dot_alpha_kernel(const VT* __restrict__ val,
                                                                        const int32_t* __restrict__ col,
                                                                        const int64_t* __restrict__ offset,
                                                                        const void* perm, int perm_bytes, int implicit,
                                                                        unsigned sigma, long long n_rows,
                                                                        long long n_slices, const float* __restrict__ x,
                                                                        float* __restrict__ y,
                                                                        const float* __restrict__ p_own,
                                                                        double* __restrict__ parts, double* scal,
                                                                        int32_t* iflags, unsigned* ticket) {
  constexpr int U = 8;
  if (*iflags) return;  // breakdown / closed gate: the whole inner solve is a no-op
  __shared__ double sh[kBlock / 32];
  // persistent: short CTAs would each pay the fence + ticket of the epilogue, so every warp walks
  // slices with a grid stride and the CTA reduces once
  const int lane = threadIdx.x & 31;
  const long long n_warps = (long long)gridDim.x * (kBlock / 32);
  double dotv = 0.0;
  for (long long k = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5; k < n_slices; k += n_warps) {
    const long long o = offset[k];
    const int width = (int)((offset[k + 1] - o) >> 5);
    const VT* pv = val + o + lane;
    const int32_t* pc = col + o + lane;
    float acc = RefOps<float>::zero();
    for (int q = 0; q < width; q += U) {
      VT v[U];
      int32_t c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool in = q + u < width;
        v[u] = in ? __ldcs(pv + (q + u) * 32) : VT(0);
        c[u] = in ? __ldcs(pc + (q + u) * 32) : 0;
      }
      float xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = x[c[u]];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q + u < width) acc = RefOps<float>::step(acc, vcast<VT, float>(v[u]), xv[u]);
    }
    const unsigned s = (unsigned)(k * 32) + lane;
    if ((long long)s < n_rows) {
      unsigned out = s;
      if (implicit) {
        const unsigned pp = perm_bytes == 1 ? (unsigned)static_cast<const uint8_t*>(perm)[s]
                                            : (unsigned)static_cast<const uint16_t*>(perm)[s];
        out = (s / sigma) * sigma + pp;
      }
      y[out] = acc;
      dotv += (double)p_own[out] * (double)acc;
    }
  }
  const double t = block_sum<kBlock>(dotv, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = t;
  double pq;
  if (last_cta_sum<kBlock>(parts, ticket, pq, sh) && threadIdx.x == 0) ipcg_alpha_step(pq, scal, iflags);
}

// persistent grid of the fused kernel: its resident CTAs per SM (launch bounds), never more
// CTAs than slices need
// resident CTAs per SM of the fused kernel: 6 (40 registers, 24 B of spills) beats 4 (no spills,
// 0.539 vs 0.455 s per comparator solve, profiles/r02/sell_dot_minb_ab.txt); PSELL_SELL_DOT_MINB=4|8 A/B
static int sell_dot_minb() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PSELL_SELL_DOT_MINB");
    const int m = e ? atoi(e) : 6;
    v = (m == 4 || m == 8) ? m : 6;
  }
  return v;
}

static long long sell_dot_grid(long long n_slices) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const long long need = ceil_div(n_slices * 32, (long long)kBlock), cap = (long long)sell_dot_minb() * sms;
  return need < 1 ? 1 : (need < cap ? need : cap);
}

template <typename VT, typename XT>
static void launch_sell(const psell_desc* d, const void* val, const int32_t* col, const int64_t* offset,
                        const void* perm, const void* x, void* y, cudaStream_t st) {
  // (f16 values: ptxas defers the 2-byte value loads behind the gathers in the
  // chunked kernel, 1033 vs 735 us on the 27-point matrix; they keep the row kernel)
  if (d->c == 32 && sizeof(VT) >= 4 && d->n_rows < (1LL << 31) && !sell_generic()) {
    const long long ns = ceil_div(d->n_rows, 32);
    sell_spmv_c32_kernel<VT, XT><<<(unsigned)ceil_div(ns * 32, kBlock), kBlock, 0, st>>>(
        static_cast<const VT*>(val), col, offset, perm, d->sigma <= 256 ? 1 : 2, d->mode == PSELL_MODE_IMPLICIT,
        (unsigned)d->sigma, d->n_rows, ns, static_cast<const XT*>(x), static_cast<XT*>(y));
    return;
  }
  const unsigned grid = (unsigned)ceil_div(d->n_rows, kBlock);
  sell_spmv_kernel<VT, XT><<<grid, kBlock, 0, st>>>(
      static_cast<const VT*>(val), col, offset, perm, d->sigma <= 256 ? 1 : 2, d->mode == PSELL_MODE_IMPLICIT,
      d->sigma, d->n_rows, d->c, static_cast<const XT*>(x), static_cast<XT*>(y));
}

template <typename VT>
static int dispatch_sell_x(const psell_desc* d, const void* val, const int32_t* col, const int64_t* offset,
                           const void* perm, const void* x, int32_t xdt, void* y, cudaStream_t st) {
  switch (xdt) {
    case PSELL_DT_F64: launch_sell<VT, double>(d, val, col, offset, perm, x, y, st); return 0;
    case PSELL_DT_F32: launch_sell<VT, float>(d, val, col, offset, perm, x, y, st); return 0;
    case PSELL_DT_F16: launch_sell<VT, __half>(d, val, col, offset, perm, x, y, st); return 0;
  }
  return 1;
}

}  // namespace psell

using namespace psell;

extern "C" {

PSELL_API int psell_sell_fill(const psell_desc* d, const int64_t* row_ptr, const int32_t* col_idx,
                              const double* values, const void* workspace, const int64_t* offset,
                              int32_t val_dtype, void* val, int32_t* col, void* stream, psell_error* err) {
  if (!d || d->c < 1) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "bad descriptor");
  const long long n = d->n_rows;
  const long long ns = ceil_div(n, d->c);
  if (ns == 0) return ok(err);
  const int32_t* order = d->mode == PSELL_MODE_NONE ? nullptr : build_ws_order(d, workspace);
  const unsigned grid = (unsigned)ceil_div(ns * d->c, kBlock);
  cudaStream_t st = as_stream(stream);
  switch (val_dtype) {
    case PSELL_DT_F64:
      sell_fill_kernel<double><<<grid, kBlock, 0, st>>>(row_ptr, col_idx, values, order, offset, n, ns, d->c,
                                                        static_cast<double*>(val), col);
      break;
    case PSELL_DT_F32:
      sell_fill_kernel<float><<<grid, kBlock, 0, st>>>(row_ptr, col_idx, values, order, offset, n, ns, d->c,
                                                       static_cast<float*>(val), col);
      break;
    case PSELL_DT_F16:
      sell_fill_kernel<__half><<<grid, kBlock, 0, st>>>(row_ptr, col_idx, values, order, offset, n, ns, d->c,
                                                        static_cast<__half*>(val), col);
      break;
    default:
      return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "bad value dtype");
  }
  PSELL_CHECK_LAUNCH(err, "psell_sell_fill");
  return ok(err);
}

PSELL_API int psell_sell_spmv(const psell_desc* d, const void* val, int32_t val_dtype, const int32_t* col,
                              const int64_t* offset, const void* perm, const void* x, int32_t x_dtype,
                              void* y, void* stream, psell_error* err) {
  if (!d || d->c < 1) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "bad descriptor");
  if (d->n_rows <= 0) return ok(err);
  cudaStream_t st = as_stream(stream);
  int bad = 1;
  switch (val_dtype) {
    case PSELL_DT_F64: bad = dispatch_sell_x<double>(d, val, col, offset, perm, x, x_dtype, y, st); break;
    case PSELL_DT_F32: bad = dispatch_sell_x<float>(d, val, col, offset, perm, x, x_dtype, y, st); break;
    case PSELL_DT_F16: bad = dispatch_sell_x<__half>(d, val, col, offset, perm, x, x_dtype, y, st); break;
  }
  if (bad) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "bad dtype");
  PSELL_CHECK_LAUNCH(err, "psell_sell_spmv");
  return ok(err);
}

PSELL_API int64_t psell_sell_spmv_dot_partials(const psell_desc* d) {
  if (!d || d->n_rows <= 0) return 1;
  return sell_dot_grid(ceil_div(d->n_rows, 32));
}

PSELL_API int psell_sell_spmv_dot_alpha(const psell_desc* d, const void* val, int32_t val_dtype, const int32_t* col,
                                        const int64_t* offset, const void* perm, const float* x, float* y,
                                        const float* p_own, double* partials, double* scal, int32_t* iflags,
                                        unsigned* ticket, void* stream, psell_error* err) {
  if (!d || d->c != 32 || d->n_rows <= 0 || d->n_rows >= (1LL << 31) || val_dtype != PSELL_DT_F32 || !ticket ||
      !scal || !iflags || !partials)
    return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0,
                   "psell_sell_spmv_dot_alpha: C = 32 f32 SELL, f32 x, scalar state");
  const long long ns = ceil_div(d->n_rows, 32);
  const int mb = sell_dot_minb();
  auto kern = mb == 6 ? sell_spmv_dot_alpha_kernel<float, 6>
                      : mb == 8 ? sell_spmv_dot_alpha_kernel<float, 8> : sell_spmv_dot_alpha_kernel<float, 4>;
  kern<<<(unsigned)sell_dot_grid(ns), kBlock, 0, as_stream(stream)>>>(
      static_cast<const float*>(val), col, offset, perm, d->sigma <= 256 ? 1 : 2, d->mode == PSELL_MODE_IMPLICIT,
      (unsigned)d->sigma, d->n_rows, ns, x, y, p_own, partials, scal, iflags, ticket);
  PSELL_CHECK_LAUNCH(err, "psell_sell_spmv_dot_alpha");
  return ok(err);
}

}  // extern "C"
