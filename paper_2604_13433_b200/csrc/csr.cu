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

#include <cstdlib>
#include <cstring>

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

// Tiled variant (default): a CTA owns 256 consecutive rows, whose entries are one
// contiguous span of col_idx / values.  The span is staged through shared memory
// in tiles of kTile entries with fully coalesced loads; each thread then walks
// the part of its row inside the tile, left to right, so every row keeps the
// reference's sequential rounding order (bitwise equal to the thread-per-row
// kernel) while HBM sees unit-stride streams instead of 256 interleaved rows.
constexpr int kTile = 2048;  // 2048 x (4 + 8) B = 24 KB of shared memory
#ifndef PSELL_CSR_MINB
#define PSELL_CSR_MINB 4
#endif

template <typename XT>
__global__ void __launch_bounds__(kBlock, PSELL_CSR_MINB) csr_spmv_tiled_kernel(long long n, const int64_t* __restrict__ row_ptr,
                                                                const int32_t* __restrict__ col_idx,
                                                                const double* __restrict__ values,
                                                                const XT* __restrict__ x, XT* __restrict__ y) {
  using O = CsrOps<XT>;
  __shared__ int32_t sc[kTile];
  __shared__ double sv[kTile];
  const long long r0 = (long long)blockIdx.x * kBlock;
  const long long r1 = r0 + kBlock < n ? r0 + kBlock : n;
  const long long i = r0 + threadIdx.x;
  const long long span0 = row_ptr[r0], span1 = row_ptr[r1];
  long long beg = 0, end = 0;
  if (i < n) {
    beg = row_ptr[i];
    end = row_ptr[i + 1];
  }
  XT acc = O::zero();
  bool started = false;
  for (long long t0 = span0; t0 < span1; t0 += kTile) {
    const int m = (int)(span1 - t0 < kTile ? span1 - t0 : kTile);
    __syncthreads();
    for (int k = threadIdx.x; k < m; k += kBlock) {
      sc[k] = __ldcs(col_idx + t0 + k);
      sv[k] = __ldcs(values + t0 + k);
    }
    __syncthreads();
    const int a = (int)((beg > t0 ? beg : t0) - t0);
    const int b = (int)((end < t0 + m ? end : t0 + m) - t0);
    // 8 entries per round: all 8 gathers issue before the first dependent add
    for (int j = a; j < b; j += 8) {
      XT xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) xv[u] = (j + u < b) ? x[sc[j + u]] : O::zero();
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (j + u < b) {
          const XT prod = O::mul(O::cv(sv[j + u]), xv[u]);
          acc = started ? O::add(acc, prod) : prod;
          started = true;
        }
      }
    }
  }
  if (i < n) y[i] = acc;
}

// Pipelined variant (default): persistent CTAs (4 per SM) walk 256-row blocks
// grid-stride; block k+1's col/value span is copied into the second half of a
// double-buffered shared-memory stage with cp.async (no registers held) while
// block k is computed, and block k+2's row_ptr bounds are loaded a block ahead.
// Blocks whose span exceeds one stage fall back to the synchronous tile loop
// in their own (idle) stage.  Same per-row order as the kernels above.
constexpr int kPTile = 2040;  // entries per stage; 2 stages x 2040 x 12 B (+ the epilogue ticket flag) <= 48 KB

__device__ __forceinline__ void cp_async4(void* smem, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(g));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(g));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

struct CsrBounds {
  long long s0, s1, rb, re;
};

template <typename XT, bool DOT = false>
__global__ void __launch_bounds__(kBlock, 4) csr_spmv_pipe_kernel(long long n, long long nb,
                                                               const int64_t* __restrict__ row_ptr,
                                                               const int32_t* __restrict__ col_idx,
                                                               const double* __restrict__ values,
                                                               const XT* __restrict__ x, XT* __restrict__ y,
                                                               const double* __restrict__ p_own = nullptr,
                                                               double* __restrict__ parts = nullptr,
                                                               double* __restrict__ scal = nullptr,
                                                               int32_t* __restrict__ gate = nullptr,
                                                               unsigned* __restrict__ ticket = nullptr) {
  using O = CsrOps<XT>;
  // FP64 PCG fused epilogue (ticket != NULL): a closed gate (the solve has stopped) makes
  // the whole kernel a no-op, and the last CTA turns the p.q partials into alpha
  if (ticket && *gate) return;
  double dotv = 0.0;  // DOT: this thread's rows of p_own . y, in row order
  __shared__ int32_t sc[2][kPTile];
  __shared__ double sv[2][kPTile];
  const int t = threadIdx.x;
  auto bounds = [&](long long blk) {
    CsrBounds b;
    const long long r0 = blk * kBlock;
    const long long r1 = r0 + kBlock < n ? r0 + kBlock : n;
    b.s0 = row_ptr[r0];
    b.s1 = row_ptr[r1];
    b.rb = b.re = 0;
    if (r0 + t < n) {
      b.rb = row_ptr[r0 + t];
      b.re = row_ptr[r0 + t + 1];
    }
    return b;
  };
  auto issue = [&](int buf, const CsrBounds& b) {
    const int m = (int)(b.s1 - b.s0);
    if (m <= kPTile) {
      for (int k = t; k < m; k += kBlock) {
        cp_async4(&sc[buf][k], col_idx + b.s0 + k);
        cp_async8(&sv[buf][k], values + b.s0 + k);
      }
    }
    cp_async_commit();
  };
  // the row's entries [a, e) of a tile, left to right, 8 gathers in flight
  auto walk = [&](const int32_t* tc, const double* tv, int a, int e, XT& acc, bool& started) {
    for (int j = a; j < e; j += 8) {
      XT xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) xv[u] = (j + u < e) ? x[tc[j + u]] : O::zero();
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (j + u < e) {
          const XT prod = O::mul(O::cv(tv[j + u]), xv[u]);
          acc = started ? O::add(acc, prod) : prod;
          started = true;
        }
      }
    }
  };
  long long blk = blockIdx.x;
  if (blk >= nb) return;  // (grid <= nb: every CTA has a block)
  CsrBounds cur = bounds(blk);
  issue(0, cur);
  CsrBounds nxt = cur;
  if (blk + gridDim.x < nb) nxt = bounds(blk + gridDim.x);
  int buf = 0;
  for (;;) {
    const long long bn = blk + gridDim.x;
    if (bn < nb) issue(buf ^ 1, nxt);
    else cp_async_commit();
    CsrBounds nn = nxt;
    if (bn + gridDim.x < nb) nn = bounds(bn + gridDim.x);
    cp_async_wait1();
    __syncthreads();
    XT acc = O::zero();
    bool started = false;
    const int m = (int)(cur.s1 - cur.s0);
    if (m <= kPTile) {
      walk(sc[buf], sv[buf], (int)(cur.rb - cur.s0), (int)(cur.re - cur.s0), acc, started);
    } else {  // long rows: synchronous tiles through this block's (unused) stage
      for (long long t0 = cur.s0; t0 < cur.s1; t0 += kPTile) {
        const int mt = (int)(cur.s1 - t0 < kPTile ? cur.s1 - t0 : kPTile);
        __syncthreads();
        for (int k = t; k < mt; k += kBlock) {
          sc[buf][k] = __ldcs(col_idx + t0 + k);
          sv[buf][k] = __ldcs(values + t0 + k);
        }
        __syncthreads();
        const int a = (int)((cur.rb > t0 ? cur.rb : t0) - t0);
        const int e = (int)((cur.re < t0 + mt ? cur.re : t0 + mt) - t0);
        walk(sc[buf], sv[buf], a, e, acc, started);
      }
    }
    if (blk * kBlock + t < n) {
      y[blk * kBlock + t] = acc;
      if constexpr (DOT) dotv += __dmul_rn(p_own[blk * kBlock + t], (double)acc);
    }
    __syncthreads();  // this stage is refilled by the next iteration's issue
    if (bn >= nb) break;
    blk = bn;
    cur = nxt;
    nxt = nn;
    buf ^= 1;
  }
  if constexpr (DOT) {  // the stages are idle now (last iteration ended on a barrier)
    const double tsum = block_sum<kBlock>(dotv, sv[0]);
    if (t == 0) parts[blockIdx.x] = tsum;
    double pq;
    if (ticket && last_cta_sum<kBlock>(parts, ticket, pq, sv[0]) && t == 0) pcg_alpha_step(pq, scal, gate);
  }
}

// Bulk-staged variant (default): the pipelined kernel with each 256-row block's col / value
// span fetched by two cp.async.bulk copies (one elected thread, mbarrier completion) instead
// of one 4- or 8-byte cp.async per entry per thread (14 LSU ops per thread per 7-point block).
// A bulk copy needs 16-byte aligned ends, so the copy covers [s0 & ~3, s1 & ~3) and the
// <= 3 tail entries [s1 & ~3, s1) travel in registers of threads 0..2, loaded one block
// ahead with the bounds.  Same per-row order and arithmetic: bitwise the pipelined kernel.
constexpr int kBT = 2048;  // entries per stage
constexpr size_t kBulkSmem = 2 * kBT * (4 + 8) + 2 * 8;

template <typename XT, bool DOT = false>
__global__ void __launch_bounds__(kBlock, 4) csr_spmv_bulk_kernel(long long n, long long nb,
                                                               const int64_t* __restrict__ row_ptr,
                                                               const int32_t* __restrict__ col_idx,
                                                               const double* __restrict__ values,
                                                               const XT* __restrict__ x, XT* __restrict__ y,
                                                               const double* __restrict__ p_own = nullptr,
                                                               double* __restrict__ parts = nullptr,
                                                               double* __restrict__ scal = nullptr,
                                                               int32_t* __restrict__ gate = nullptr,
                                                               unsigned* __restrict__ ticket = nullptr) {
  using O = CsrOps<XT>;
  if (ticket && *gate) return;
  extern __shared__ __align__(128) unsigned char cb_smem[];
  int32_t* sc = reinterpret_cast<int32_t*>(cb_smem);                   // [2][kBT]
  double* sv = reinterpret_cast<double*>(cb_smem + 2 * kBT * 4);        // [2][kBT]
  uint64_t* bar = reinterpret_cast<uint64_t*>(cb_smem + 2 * kBT * 12);  // [2]
  const int t = threadIdx.x;
  double dotv = 0.0;
  long long blk = blockIdx.x;
  if (blk >= nb) return;  // (grid <= nb: every CTA has a block)
  if (t == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto bounds = [&](long long b) {
    CsrBounds c;
    const long long r0 = b * kBlock;
    const long long r1 = r0 + kBlock < n ? r0 + kBlock : n;
    c.s0 = row_ptr[r0];
    c.s1 = row_ptr[r1];
    c.rb = c.re = 0;
    if (r0 + t < n) {
      c.rb = row_ptr[r0 + t];
      c.re = row_ptr[r0 + t + 1];
    }
    return c;
  };
  auto fits = [&](const CsrBounds& c) { return c.s1 - (c.s0 & ~3LL) <= kBT; };
  // thread 0: the aligned body of block c's span into stage buf (a plain arrive when there
  // is none, or the span does not fit and the block takes the synchronous path)
  auto issue = [&](int buf, const CsrBounds& c) {
    const long long a0 = c.s0 & ~3LL, e0 = c.s1 & ~3LL;
    if (fits(c) && e0 > a0) {
      const uint32_t m = (uint32_t)(e0 - a0);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar + buf, m * 12u);
      const uint64_t pol = policy_evict_first();
      bulk_g2s(sc + buf * kBT, col_idx + a0, m * 4u, bar + buf, pol);
      bulk_g2s(sv + buf * kBT, values + a0, m * 8u, bar + buf, pol);
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar + buf)) : "memory");
    }
  };
  // threads 0..2: block c's tail entries into registers
  auto tail = [&](const CsrBounds& c, int32_t& tc, double& tv) {
    const long long e = (c.s1 & ~3LL) + t;
    if (t < 3 && e < c.s1 && fits(c)) {
      tc = __ldcs(col_idx + e);
      tv = __ldcs(values + e);
    }
  };
  auto walk = [&](const int32_t* tcol, const double* tval, int a, int e, XT& acc, bool& started) {
    for (int j = a; j < e; j += 8) {
      XT xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) xv[u] = (j + u < e) ? x[tcol[j + u]] : O::zero();
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (j + u < e) {
          const XT prod = O::mul(O::cv(tval[j + u]), xv[u]);
          acc = started ? O::add(acc, prod) : prod;
          started = true;
        }
      }
    }
  };
  CsrBounds cur = bounds(blk);
  if (t == 0) issue(0, cur);
  int32_t tc = 0;
  double tv = 0.0;
  tail(cur, tc, tv);
  CsrBounds nxt = cur;
  if (blk + gridDim.x < nb) nxt = bounds(blk + gridDim.x);
  int buf = 0;
  uint32_t phase = 0u;  // bit b: parity of stage b's next completion
  for (;;) {
    const long long bn = blk + gridDim.x;
    if (bn < nb && t == 0) issue(buf ^ 1, nxt);
    int32_t ntc = 0;
    double ntv = 0.0;
    if (bn < nb) tail(nxt, ntc, ntv);
    CsrBounds nn = nxt;
    if (bn + gridDim.x < nb) nn = bounds(bn + gridDim.x);
    const long long a0 = cur.s0 & ~3LL, e0 = cur.s1 & ~3LL;
    const bool fit = fits(cur);
    if (fit && t < 3 && e0 + t < cur.s1) {
      sc[buf * kBT + (int)(e0 + t - a0)] = tc;
      sv[buf * kBT + (int)(e0 + t - a0)] = tv;
    }
    mbar_wait(bar + buf, (phase >> buf) & 1u);
    phase ^= 1u << buf;
    __syncthreads();
    XT acc = O::zero();
    bool started = false;
    if (fit) {
      walk(sc + buf * kBT, sv + buf * kBT, (int)(cur.rb - a0), (int)(cur.re - a0), acc, started);
    } else {  // long rows: synchronous tiles through this block's stage
      for (long long t0 = cur.s0; t0 < cur.s1; t0 += kBT) {
        const int mt = (int)(cur.s1 - t0 < kBT ? cur.s1 - t0 : kBT);
        __syncthreads();
        for (int k = t; k < mt; k += kBlock) {
          sc[buf * kBT + k] = __ldcs(col_idx + t0 + k);
          sv[buf * kBT + k] = __ldcs(values + t0 + k);
        }
        __syncthreads();
        const int a = (int)((cur.rb > t0 ? cur.rb : t0) - t0);
        const int e = (int)((cur.re < t0 + mt ? cur.re : t0 + mt) - t0);
        walk(sc + buf * kBT, sv + buf * kBT, a, e, acc, started);
      }
    }
    if (blk * kBlock + t < n) {
      y[blk * kBlock + t] = acc;
      if constexpr (DOT) dotv += __dmul_rn(p_own[blk * kBlock + t], (double)acc);
    }
    __syncthreads();  // this stage is refilled by the next iteration's issue
    if (bn >= nb) break;
    blk = bn;
    cur = nxt;
    nxt = nn;
    tc = ntc;
    tv = ntv;
    buf ^= 1;
  }
  if constexpr (DOT) {  // the stages are idle now (last iteration ended on a barrier)
    const double tsum = block_sum<kBlock>(dotv, sv);
    if (t == 0) parts[blockIdx.x] = tsum;
    double pq;
    if (ticket && last_cta_sum<kBlock>(parts, ticket, pq, sv) && t == 0) pcg_alpha_step(pq, scal, gate);
  }
}

__global__ void __launch_bounds__(1024) csr_dot_finalize_kernel(const double* __restrict__ parts, int np,
                                                                double* __restrict__ out) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < np; i += 1024) v += parts[i];
  const double tsum = block_sum<1024>(v, sh);
  if (threadIdx.x == 0) out[0] = tsum;
}

}  // namespace psell

using namespace psell;

static unsigned csr_pipe_grid(long long nb) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return (unsigned)(nb < 4LL * sms ? nb : 4LL * sms);
}

// K4 variant (read once per process): PSELL_CSR=pipe (per-entry cp.async stages) or
// tiled (no pipelining) instead of the bulk-staged default (A/B; all bitwise equal)
static int csr_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PSELL_CSR");
    v = !e ? 0 : strcmp(e, "pipe") == 0 ? 1 : strcmp(e, "tiled") == 0 ? 2 : 0;
  }
  return v;
}

template <typename XT, bool DOT>
static void launch_csr(long long n, const int64_t* row_ptr, const int32_t* col_idx, const double* values,
                       const XT* x, XT* y, const double* p_own, double* parts, double* scal, int32_t* gate,
                       unsigned* ticket, cudaStream_t st, unsigned* grid_out = nullptr) {
  const long long nb = ceil_div(n, kBlock);
  const unsigned pg = csr_pipe_grid(nb);
  if (grid_out) *grid_out = pg;
  if (csr_variant() == 1) {
    csr_spmv_pipe_kernel<XT, DOT><<<pg, kBlock, 0, st>>>(n, nb, row_ptr, col_idx, values, x, y, p_own, parts, scal,
                                                         gate, ticket);
    return;
  }
  static bool attr = false;  // idempotent attribute, benign race
  if (!attr) {
    cudaFuncSetAttribute(csr_spmv_bulk_kernel<XT, DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBulkSmem);
    attr = true;
  }
  csr_spmv_bulk_kernel<XT, DOT><<<pg, kBlock, kBulkSmem, st>>>(n, nb, row_ptr, col_idx, values, x, y, p_own, parts,
                                                               scal, gate, ticket);
}

extern "C" int psell_csr_spmv_dot(int64_t n_rows, const int64_t* row_ptr, const int32_t* col_idx,
                                  const double* values, const double* x, double* y, const double* p_own,
                                  double* partials, double* out1, void* stream, psell_error* err) {
  cudaStream_t st = as_stream(stream);
  if (n_rows <= 0) {
    cudaMemsetAsync(out1, 0, sizeof(double), st);
    return ok(err);
  }
  unsigned pg = 0;
  launch_csr<double, true>(n_rows, row_ptr, col_idx, values, x, y, p_own, partials, nullptr, nullptr, nullptr, st, &pg);
  csr_dot_finalize_kernel<<<1, 1024, 0, st>>>(partials, (int)pg, out1);
  PSELL_CHECK_LAUNCH(err, "psell_csr_spmv_dot");
  return ok(err);
}

// FP64 PCG iteration head: q = A p, pq = p.q, alpha = rz / pq (solvers.py:196-200), one launch
extern "C" int psell_csr_spmv_dot_alpha(int64_t n_rows, const int64_t* row_ptr, const int32_t* col_idx,
                                        const double* values, const double* x, double* y, const double* p_own,
                                        double* partials, double* scal, int32_t* gate, unsigned* ticket,
                                        void* stream, psell_error* err) {
  if (n_rows <= 0 || !ticket || !gate || !scal)
    return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "psell_csr_spmv_dot_alpha: empty operator or missing scalars");
  launch_csr<double, true>(n_rows, row_ptr, col_idx, values, x, y, p_own, partials, scal, gate, ticket,
                           as_stream(stream));
  PSELL_CHECK_LAUNCH(err, "psell_csr_spmv_dot_alpha");
  return ok(err);
}

extern "C" int psell_csr_spmv(int64_t n_rows, const int64_t* row_ptr, const int32_t* col_idx,
                              const double* values, const void* x, int32_t x_dtype, void* y,
                              void* stream, psell_error* err) {
  if (n_rows <= 0) return ok(err);
  const unsigned grid = (unsigned)ceil_div(n_rows, kBlock);
  cudaStream_t st = as_stream(stream);
  if (csr_variant() != 2) {
    switch (x_dtype) {
      case PSELL_DT_F64:
        launch_csr<double, false>(n_rows, row_ptr, col_idx, values, static_cast<const double*>(x),
                                  static_cast<double*>(y), nullptr, nullptr, nullptr, nullptr, nullptr, st);
        break;
      case PSELL_DT_F32:
        launch_csr<float, false>(n_rows, row_ptr, col_idx, values, static_cast<const float*>(x),
                                 static_cast<float*>(y), nullptr, nullptr, nullptr, nullptr, nullptr, st);
        break;
      case PSELL_DT_F16:
        launch_csr<__half, false>(n_rows, row_ptr, col_idx, values, static_cast<const __half*>(x),
                                  static_cast<__half*>(y), nullptr, nullptr, nullptr, nullptr, nullptr, st);
        break;
      default:
        return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "unsupported x dtype");
    }
    PSELL_CHECK_LAUNCH(err, "psell_csr_spmv");
    return ok(err);
  }
  switch (x_dtype) {
    case PSELL_DT_F64:
      csr_spmv_tiled_kernel<double><<<grid, kBlock, 0, st>>>(n_rows, row_ptr, col_idx, values,
                                                       static_cast<const double*>(x), static_cast<double*>(y));
      break;
    case PSELL_DT_F32:
      csr_spmv_tiled_kernel<float><<<grid, kBlock, 0, st>>>(n_rows, row_ptr, col_idx, values,
                                                      static_cast<const float*>(x), static_cast<float*>(y));
      break;
    case PSELL_DT_F16:
      csr_spmv_tiled_kernel<__half><<<grid, kBlock, 0, st>>>(n_rows, row_ptr, col_idx, values,
                                                       static_cast<const __half*>(x), static_cast<__half*>(y));
      break;
    default:
      return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "unsupported x dtype");
  }
  PSELL_CHECK_LAUNCH(err, "psell_csr_spmv");
  return ok(err);
}
