// K3 — solver vector kernels with deterministic FP64 reductions.
//
// Replaces the numpy vector algebra of pcg / fcg / _inner_pcg (reference
// solvers.py:171-308) and _dot/_norm (87-93).  All reductions go through
// fixed-grid partials (one per CTA, grid-stride over a fixed grid of
// PSELL_RED_BLOCKS CTAs) summed by one CTA in a fixed tree, so results are
// bit-reproducible run to run (SPEC determinism, test_acceptance c09).  Across
// ranks each rank's local sum is gathered and summed in rank order by the
// scalar kernels (n_parts > 1).  Scalars (alpha, beta, rz, the breakdown flag,
// the done counter) never leave the device: the inner loop is launch-only and
// CUDA-graph capturable.  Vector updates reproduce numpy's rounding: the
// Python-float coefficient is rounded to the vector dtype, then a separately
// rounded product and sum (no FMA contraction).
#include "psell_internal.cuh"

namespace psell {

constexpr int kRB = PSELL_RED_BLOCKS;

// grid-stride loops of the f64 vector kernels: 4 trips unrolled so each thread
// has 4 independent loads per vector in flight (the per-thread summation order,
// hence every result bit, is unchanged)
#ifndef PSELL_GS_UNROLL
#define PSELL_GS_UNROLL _Pragma("unroll 4")
#endif

__global__ void __launch_bounds__(1024) sum_partials_kernel(const double* __restrict__ parts,
                                                            long long np, int n_out,
                                                            double* __restrict__ out,
                                                            const int32_t* skip) {
  if (skip && *skip) return;
  __shared__ double sh[32];
  for (int k = 0; k < n_out; ++k) {
    double v = 0.0;
    for (long long i = threadIdx.x; i < np; i += 1024) v += parts[k * np + i];
    const double t = block_sum<1024>(v, sh);
    if (threadIdx.x == 0) out[k] = t;
  }
}

static int finalize(const double* parts, long long np, int n_out, double* out, const int32_t* skip,
                    cudaStream_t st) {
  sum_partials_kernel<<<1, 1024, 0, st>>>(parts, np, n_out, out, skip);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

template <typename T>
__global__ void __launch_bounds__(kBlock) dot_kernel(const T* __restrict__ a, const T* __restrict__ b,
                                                     long long n, double* __restrict__ parts) {
  __shared__ double sh[kBlock / 32];
  double v = 0.0;
  PSELL_GS_UNROLL
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long long)kRB * kBlock)
    v += (double)a[i] * (double)b[i];
  v = block_sum<kBlock>(v, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = v;
}

// ---------------------------------------------------------------- inner PCG (f32)
// solvers.py:286-291: b = r.astype(f32); x = 0; r = b; z = P(r); p = z; rz = r.z
__global__ void __launch_bounds__(kBlock) ipcg_begin_kernel(long long n, const double* __restrict__ r64,
                                                            float* __restrict__ x, float* r, float* z,
                                                            float* __restrict__ p,
                                                            const float* __restrict__ inv,
                                                            double* __restrict__ parts) {
  __shared__ double sh[kBlock / 32];
  double v = 0.0;
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long long)kRB * kBlock) {
    const float rf = __double2float_rn(r64[i]);
    x[i] = 0.f;
    r[i] = rf;
    float zf = rf;
    if (inv) {
      zf = __fmul_rn(rf, inv[i]);
      z[i] = zf;
    }
    p[i] = zf;
    v += (double)rf * (double)zf;
  }
  v = block_sum<kBlock>(v, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = v;
}

// scal: [0]=rz [1]=pq [2]=alpha [3]=beta [4]=rz_new ; iflags: [0]=breakdown [1]=done
// gate (optional): an outer loop's convergence gate (psell_pcg_status); when it is
// closed the inner solve starts "broken down", so every kernel of the (captured)
// inner loop returns at once -- the outer loop queues its next iteration before
// reading the current one's status
__global__ void ipcg_set_rz_kernel(const double* parts, int np, int stride, double* scal, int32_t* iflags,
                                   const int32_t* gate) {
  double s = 0.0;
  for (int i = 0; i < np; ++i) s += parts[(long long)i * stride];
  scal[0] = s;
  iflags[0] = (gate && gate[0]) ? 1 : 0;
  iflags[1] = 0;
}

// solvers.py:295-299
__global__ void ipcg_alpha_kernel(const double* parts, int np, int stride, double* scal, int32_t* iflags) {
  if (iflags[0]) return;
  double pq = 0.0;
  for (int i = 0; i < np; ++i) pq += parts[(long long)i * stride];
  scal[1] = pq;
  if (pq <= 0.0 || !isfinite(pq) || scal[0] == 0.0) {
    iflags[0] = 1;
    return;
  }
  scal[2] = scal[0] / pq;
}

// solvers.py:300-304: x += a p; r -= a q; z = P(r); rz_new partials.
// VEC: 16-byte vectors (4 rows per thread per trip) for memory-level parallelism;
// each row is still updated with the reference's separately rounded ops.
__device__ __forceinline__ void upd1(float a, float& xv, float& rv, float& zv, float pv, float qv,
                                     const float* inv, long long i) {
  xv = __fadd_rn(xv, __fmul_rn(a, pv));
  rv = __fsub_rn(rv, __fmul_rn(a, qv));
  zv = inv ? __fmul_rn(rv, inv[i]) : rv;
}

// r -= a q; z = P(r) only (the x += a p half moves into the direction kernel)
__device__ __forceinline__ void upd1_r(float a, float& rv, float& zv, float qv, const float* inv, long long i) {
  rv = __fsub_rn(rv, __fmul_rn(a, qv));
  zv = inv ? __fmul_rn(rv, inv[i]) : rv;
}

// Fused tail of one inner iteration, x half of the update deferred here:
// x += alpha p_old; p = z + beta p_old (solvers.py:301, 307).  Same separately
// rounded f32 ops as ipcg_update + ipcg_direction, one pass over p instead of two.
__global__ void __launch_bounds__(kBlock) ipcg_direction_x_kernel(long long n, float* __restrict__ p,
                                                                  const float* __restrict__ z,
                                                                  float* __restrict__ x,
                                                                  const double* __restrict__ scal,
                                                                  const int32_t* __restrict__ iflags,
                                                                  bool rev = false) {
  if (iflags[0]) return;
  const float al = __double2float_rn(scal[2]);
  const float b = __double2float_rn(scal[3]);
  const long long gt = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long gs = (long long)gridDim.x * kBlock;
  long long done = 0;
  const bool vec = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(z) |
                     reinterpret_cast<uintptr_t>(x)) & 15) == 0;
  if (vec) {
    const long long n4 = n >> 2;
    for (long long k4 = gt; k4 < n4; k4 += gs) {
      const long long i4 = rev ? n4 - 1 - k4 : k4;  // rev: descending rows (see ipcg_update_kernel)
      float4 pv = reinterpret_cast<float4*>(p)[i4];
      float4 xv = reinterpret_cast<float4*>(x)[i4];
      const float4 zv = reinterpret_cast<const float4*>(z)[i4];
      xv.x = __fadd_rn(xv.x, __fmul_rn(al, pv.x));
      xv.y = __fadd_rn(xv.y, __fmul_rn(al, pv.y));
      xv.z = __fadd_rn(xv.z, __fmul_rn(al, pv.z));
      xv.w = __fadd_rn(xv.w, __fmul_rn(al, pv.w));
      pv.x = __fadd_rn(zv.x, __fmul_rn(b, pv.x));
      pv.y = __fadd_rn(zv.y, __fmul_rn(b, pv.y));
      pv.z = __fadd_rn(zv.z, __fmul_rn(b, pv.z));
      pv.w = __fadd_rn(zv.w, __fmul_rn(b, pv.w));
      reinterpret_cast<float4*>(x)[i4] = xv;
      reinterpret_cast<float4*>(p)[i4] = pv;
    }
    done = n4 * 4;
  }
  for (long long i = done + gt; i < n; i += gs) {
    const float pv = p[i];
    x[i] = __fadd_rn(x[i], __fmul_rn(al, pv));
    p[i] = __fadd_rn(z[i], __fmul_rn(b, pv));
  }
}

// The distributed direction pass with the halo push fused in (peer transport): the same
// x += alpha p_old; p = z + beta p_old as ipcg_direction_x_kernel, and every row a peer's
// slab reads (up to kHaloRanges contiguous local ranges, each owed to one peer) is stored
// straight into that peer's full vector in its arena as soon as it is computed; the last
// CTA then runs the K8 signal / wait (system-scope fence, epoch released into every peer's
// flag, acquire-wait for every peer), so when this kernel ends every peer's halo of the
// next SpMV has arrived -- the halo exchange costs no kernel of its own.
constexpr int kHaloRanges = 2;
struct HaloRanges {
  long long lo[kHaloRanges], hi[kHaloRanges];
  int dst[kHaloRanges];
  int n;
};

__global__ void __launch_bounds__(kBlock) ipcg_direction_x_push_kernel(long long n, float* __restrict__ p,
                                                                       const float* __restrict__ z,
                                                                       float* __restrict__ x,
                                                                       const double* __restrict__ scal,
                                                                       const int32_t* __restrict__ iflags, bool rev,
                                                                       const unsigned long long* __restrict__ peers,
                                                                       int G, int rank, long long row0,
                                                                       long long vec_off, HaloRanges hr,
                                                                       long long timeout_ns) {
  if (iflags[0]) return;  // breakdown / closed gate: every rank skips alike (global scalars)
  const float al = __double2float_rn(scal[2]);
  const float b = __double2float_rn(scal[3]);
  const long long gt = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long gs = (long long)gridDim.x * kBlock;
  auto owed = [&](long long i0, long long i1) {  // does [i0, i1) meet a halo range?
    bool m = false;
#pragma unroll
    for (int k = 0; k < kHaloRanges; ++k) m |= k < hr.n && i0 < hr.hi[k] && i1 > hr.lo[k];
    return m;
  };
  auto push = [&](long long i, float v) {
#pragma unroll
    for (int k = 0; k < kHaloRanges; ++k)
      if (k < hr.n && i >= hr.lo[k] && i < hr.hi[k])
        reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(peers[hr.dst[k]]) + vec_off)[row0 + i] = v;
  };
  long long done = 0;
  const bool vec = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(z) |
                     reinterpret_cast<uintptr_t>(x)) & 15) == 0;
  if (vec) {
    const long long n4 = n >> 2;
    for (long long k4 = gt; k4 < n4; k4 += gs) {
      const long long i4 = rev ? n4 - 1 - k4 : k4;
      float4 pv = reinterpret_cast<float4*>(p)[i4];
      float4 xv = reinterpret_cast<float4*>(x)[i4];
      const float4 zv = reinterpret_cast<const float4*>(z)[i4];
      xv.x = __fadd_rn(xv.x, __fmul_rn(al, pv.x));
      xv.y = __fadd_rn(xv.y, __fmul_rn(al, pv.y));
      xv.z = __fadd_rn(xv.z, __fmul_rn(al, pv.z));
      xv.w = __fadd_rn(xv.w, __fmul_rn(al, pv.w));
      pv.x = __fadd_rn(zv.x, __fmul_rn(b, pv.x));
      pv.y = __fadd_rn(zv.y, __fmul_rn(b, pv.y));
      pv.z = __fadd_rn(zv.z, __fmul_rn(b, pv.z));
      pv.w = __fadd_rn(zv.w, __fmul_rn(b, pv.w));
      reinterpret_cast<float4*>(x)[i4] = xv;
      reinterpret_cast<float4*>(p)[i4] = pv;
      if (owed(4 * i4, 4 * i4 + 4)) {
        push(4 * i4, pv.x);
        push(4 * i4 + 1, pv.y);
        push(4 * i4 + 2, pv.z);
        push(4 * i4 + 3, pv.w);
      }
    }
    done = n4 * 4;
  }
  for (long long i = done + gt; i < n; i += gs) {
    const float pv = p[i];
    x[i] = __fadd_rn(x[i], __fmul_rn(al, pv));
    const float pn = __fadd_rn(z[i], __fmul_rn(b, pv));
    p[i] = pn;
    push(i, pn);
  }
  // signal / wait: this rank's halo pushes are complete toward every peer
  __threadfence_system();
  __syncthreads();
  __shared__ bool last;
  unsigned char* self = reinterpret_cast<unsigned char*>(peers[rank]);
  uint32_t* ticket = reinterpret_cast<uint32_t*>(self + kTicketOff);
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence_system();
  *ticket = 0u;
  uint32_t* flags = reinterpret_cast<uint32_t*>(self + kFlagOff);
  uint32_t* epoch_p = reinterpret_cast<uint32_t*>(self + kEpochOff);
  const uint32_t e = *reinterpret_cast<volatile uint32_t*>(epoch_p) + 1u;
  for (int q = 0; q < G; ++q)
    st_release_sys(reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(peers[q]) + kFlagOff) + rank, e);
  const unsigned long long t0 = globaltimer();
  for (int q = 0; q < G; ++q) {
    unsigned spins = 0;
    while ((int)(ld_acquire_sys(flags + q) - e) < 0) {
      if ((++spins & 1023u) == 0 && (long long)(globaltimer() - t0) > timeout_ns) {
        atomicExch(reinterpret_cast<int*>(self + kErrOff), 1);
        break;
      }
    }
  }
  *epoch_p = e;
}

template <bool VEC>
__global__ void __launch_bounds__(kBlock) ipcg_update_kernel(long long n, float* __restrict__ x, float* r,
                                                             float* z, const float* __restrict__ p,
                                                             const float* __restrict__ q,
                                                             const float* __restrict__ inv,
                                                             double* scal, int32_t* iflags,
                                                             double* __restrict__ parts, unsigned* ticket,
                                                             bool rev = false,
                                                             const unsigned long long* peers = nullptr,
                                                             int peer_G = 1, int peer_rank = 0,
                                                             long long peer_timeout = 0) {
  if (iflags[0]) return;
  __shared__ double sh[kBlock / 32];
  const float a = __double2float_rn(scal[2]);
  double v = 0.0;
  const long long gt = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long gs = (long long)kRB * kBlock;
  long long done = 0;
  if (VEC) {
    const long long n4 = n >> 2;
    // rev: rows in descending order (the SpMV before this pass wrote q ascending, so the
    // most recently written -- still L2-resident -- part of q is read first)
    auto at = [&](long long i4) { return rev ? n4 - 1 - i4 : i4; };
    auto step = [&](long long i4, float4 rv, const float4 qv) {
      float4 zv;
      i4 = at(i4);
      const long long i = i4 * 4;
      if (x) {
        float4 xv = reinterpret_cast<float4*>(x)[i4];
        const float4 pv = reinterpret_cast<const float4*>(p)[i4];
        upd1(a, xv.x, rv.x, zv.x, pv.x, qv.x, inv, i);
        upd1(a, xv.y, rv.y, zv.y, pv.y, qv.y, inv, i + 1);
        upd1(a, xv.z, rv.z, zv.z, pv.z, qv.z, inv, i + 2);
        upd1(a, xv.w, rv.w, zv.w, pv.w, qv.w, inv, i + 3);
        reinterpret_cast<float4*>(x)[i4] = xv;
      } else {
        upd1_r(a, rv.x, zv.x, qv.x, inv, i);
        upd1_r(a, rv.y, zv.y, qv.y, inv, i + 1);
        upd1_r(a, rv.z, zv.z, qv.z, inv, i + 2);
        upd1_r(a, rv.w, zv.w, qv.w, inv, i + 3);
      }
      reinterpret_cast<float4*>(r)[i4] = rv;
      if (inv) reinterpret_cast<float4*>(z)[i4] = zv;
      v += (double)rv.x * (double)zv.x;
      v += (double)rv.y * (double)zv.y;
      v += (double)rv.z * (double)zv.z;
      v += (double)rv.w * (double)zv.w;
    };
    long long i4 = gt;
    // two grid-stride elements per trip, all four loads issued first (same
    // per-thread order of the dot sum as one element per trip)
#ifndef PSELL_UPD_U1
    for (; i4 + gs < n4; i4 += 2 * gs) {
      const float4 r0 = reinterpret_cast<float4*>(r)[at(i4)];
      const float4 q0 = reinterpret_cast<const float4*>(q)[at(i4)];
      const float4 r1 = reinterpret_cast<float4*>(r)[at(i4 + gs)];
      const float4 q1 = reinterpret_cast<const float4*>(q)[at(i4 + gs)];
      step(i4, r0, q0);
      step(i4 + gs, r1, q1);
    }
#endif
    for (; i4 < n4; i4 += gs) step(i4, reinterpret_cast<float4*>(r)[at(i4)], reinterpret_cast<const float4*>(q)[at(i4)]);
    done = n4 * 4;
  }
  for (long long i = done + gt; i < n; i += gs) {
    float rv = r[i], zv;
    if (x) {
      float xv = x[i];
      upd1(a, xv, rv, zv, p[i], q[i], inv, i);
      x[i] = xv;
    } else {
      upd1_r(a, rv, zv, q[i], inv, i);
    }
    r[i] = rv;
    if (inv) z[i] = zv;
    v += (double)rv * (double)zv;
  }
  v = block_sum<kBlock>(v, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = v;
  double rz_new;  // fused beta (psell_ipcg_update_beta): the last CTA finishes the iteration's scalars
  if (ticket && last_cta_sum<kBlock>(parts, ticket, rz_new, sh) && threadIdx.x == 0) {
    if (peer_G > 1) rz_new = peer_allreduce1(peer_G, peer_rank, peers, peer_timeout, rz_new);
    ipcg_beta_step(rz_new, scal, iflags);
  }
}

// solvers.py:304-306
__global__ void ipcg_beta_kernel(const double* parts, int np, int stride, double* scal, int32_t* iflags) {
  if (iflags[0]) return;
  double s = 0.0;
  for (int i = 0; i < np; ++i) s += parts[(long long)i * stride];
  scal[4] = s;
  scal[3] = s / scal[0];
  scal[0] = s;
  iflags[1] += 1;
}

// solvers.py:307: p = z + beta p
__global__ void __launch_bounds__(kBlock) ipcg_direction_kernel(long long n, float* __restrict__ p,
                                                                const float* __restrict__ z,
                                                                const double* __restrict__ scal,
                                                                const int32_t* __restrict__ iflags) {
  if (iflags[0]) return;
  const float b = __double2float_rn(scal[3]);
  const long long gt = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long gs = (long long)gridDim.x * kBlock;
  long long done = 0;
  const bool vec = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(z)) & 15) == 0;
  if (vec) {
    const long long n4 = n >> 2;
    for (long long i4 = gt; i4 < n4; i4 += gs) {
      float4 pv = reinterpret_cast<float4*>(p)[i4];
      const float4 zv = reinterpret_cast<const float4*>(z)[i4];
      pv.x = __fadd_rn(zv.x, __fmul_rn(b, pv.x));
      pv.y = __fadd_rn(zv.y, __fmul_rn(b, pv.y));
      pv.z = __fadd_rn(zv.z, __fmul_rn(b, pv.z));
      pv.w = __fadd_rn(zv.w, __fmul_rn(b, pv.w));
      reinterpret_cast<float4*>(p)[i4] = pv;
    }
    done = n4 * 4;
  }
  for (long long i = done + gt; i < n; i += gs) p[i] = __fadd_rn(z[i], __fmul_rn(b, p[i]));
}

__global__ void __launch_bounds__(kBlock) ipcg_end_kernel(long long n, const float* __restrict__ x,
                                                          double* __restrict__ z64) {
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long long)gridDim.x * kBlock)
    z64[i] = (double)x[i];
}

// ---------------------------------------------------------------- outer f64
// solvers.py:254,256: {z.(r - r_prev), z.r}
__global__ void __launch_bounds__(kBlock) fcg_zr_kernel(long long n, const double* __restrict__ z,
                                                        const double* __restrict__ r,
                                                        const double* __restrict__ rp,
                                                        double* __restrict__ parts) {
  __shared__ double sh[kBlock / 32];
  double v0 = 0.0, v1 = 0.0;
  PSELL_GS_UNROLL
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long long)kRB * kBlock) {
    const double zi = z[i], ri = r[i];
    if (rp) v0 += __dmul_rn(zi, __dsub_rn(ri, rp[i]));
    v1 += __dmul_rn(zi, ri);
  }
  v0 = block_sum<kBlock>(v0, sh);
  v1 = block_sum<kBlock>(v1, sh);
  if (threadIdx.x == 0) {
    parts[blockIdx.x] = v0;
    parts[kRB + blockIdx.x] = v1;
  }
}

// solvers.py:259,263: {p.q, p.r}
__global__ void __launch_bounds__(kBlock) pq_pr_kernel(long long n, const double* __restrict__ p,
                                                       const double* __restrict__ q,
                                                       const double* __restrict__ r,
                                                       double* __restrict__ parts) {
  __shared__ double sh[kBlock / 32];
  double v0 = 0.0, v1 = 0.0;
  PSELL_GS_UNROLL
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long long)kRB * kBlock) {
    const double pi = p[i];
    v0 += __dmul_rn(pi, q[i]);
    if (r) v1 += __dmul_rn(pi, r[i]);
  }
  v0 = block_sum<kBlock>(v0, sh);
  v1 = block_sum<kBlock>(v1, sh);
  if (threadIdx.x == 0) {
    parts[blockIdx.x] = v0;
    parts[kRB + blockIdx.x] = v1;
  }
}

// solvers.py:201-204 / 264-267: x += a p; r -= a q; {r.r}
__global__ void __launch_bounds__(kBlock) axpy2_kernel(long long n, double* __restrict__ x,
                                                       double* __restrict__ r,
                                                       const double* __restrict__ p,
                                                       const double* __restrict__ q,
                                                       const double* __restrict__ coef,
                                                       const int32_t* skip,
                                                       double* __restrict__ parts) {
  if (skip && *skip) return;
  __shared__ double sh[kBlock / 32];
  const double a = coef[0];
  double v = 0.0;
  const long long gs = (long long)kRB * kBlock;
  long long i = (long long)blockIdx.x * kBlock + threadIdx.x;
  // 4 trips per pass with every load issued before the first store (the
  // compiler would otherwise re-order nothing across the x / r stores)
  for (; i + 3 * gs < n; i += 4 * gs) {
    double xv[4], rv[4], pv[4], qv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      xv[u] = x[i + u * gs];
      rv[u] = r[i + u * gs];
      pv[u] = p[i + u * gs];
      qv[u] = q[i + u * gs];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x[i + u * gs] = __dadd_rn(xv[u], __dmul_rn(a, pv[u]));
      const double rn = __dsub_rn(rv[u], __dmul_rn(a, qv[u]));
      r[i + u * gs] = rn;
      v += __dmul_rn(rn, rn);
    }
  }
  for (; i < n; i += gs) {
    x[i] = __dadd_rn(x[i], __dmul_rn(a, p[i]));
    const double rn = __dsub_rn(r[i], __dmul_rn(a, q[i]));
    r[i] = rn;
    v += __dmul_rn(rn, rn);
  }
  v = block_sum<kBlock>(v, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = v;
}

// FP64 PCG iteration tail, identity preconditioner (solvers.py:201-209), one launch after
// psell_csr_spmv_dot_alpha: x += alpha p; r -= alpha q (axpy2's ops); rr = r.r in a fixed
// order (the last CTA); the status {breakdown, pq, sqrt(rr) / bnorm} the host appends to
// the history (psell_pcg_status's semantics, gate closed at convergence); beta = rr / rz;
// rz = rr.  With the gate already closed only the status is written.
__global__ void __launch_bounds__(kBlock) pcg_update_status_kernel(long long n, double* __restrict__ x,
                                                                   double* __restrict__ r,
                                                                   const double* __restrict__ p,
                                                                   const double* __restrict__ q,
                                                                   double* scal, int32_t* gate, double bnorm,
                                                                   double tol, double* out,
                                                                   double* __restrict__ parts, unsigned* ticket) {
  __shared__ double sh[kBlock / 32];
  const int g0 = gate[0];  // changed only by this kernel's last CTA, after every CTA read it
  if (g0 != 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (g0 == 2 || gate[1]) {
        out[0] = -1.0;
      } else {  // breakdown found by this iteration's alpha step: report it once
        out[0] = 1.0;
        out[1] = scal[10];
        out[2] = __ddiv_rn(__dsqrt_rn(scal[12]), bnorm);
        gate[1] = 1;
      }
    }
    return;
  }
  const double a = scal[0];
  double v = 0.0;
  const long long gs = (long long)gridDim.x * kBlock;
  long long i = (long long)blockIdx.x * kBlock + threadIdx.x;
  for (; i + 3 * gs < n; i += 4 * gs) {
    double xv[4], rv[4], pv[4], qv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      xv[u] = x[i + u * gs];
      rv[u] = r[i + u * gs];
      pv[u] = p[i + u * gs];
      qv[u] = q[i + u * gs];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x[i + u * gs] = __dadd_rn(xv[u], __dmul_rn(a, pv[u]));
      const double rn = __dsub_rn(rv[u], __dmul_rn(a, qv[u]));
      r[i + u * gs] = rn;
      v += __dmul_rn(rn, rn);
    }
  }
  for (; i < n; i += gs) {
    x[i] = __dadd_rn(x[i], __dmul_rn(a, p[i]));
    const double rn = __dsub_rn(r[i], __dmul_rn(a, q[i]));
    r[i] = rn;
    v += __dmul_rn(rn, rn);
  }
  v = block_sum<kBlock>(v, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = v;
  double rr;
  if (last_cta_sum<kBlock>(parts, ticket, rr, sh) && threadIdx.x == 0) {
    scal[12] = rr;
    const double rel = __ddiv_rn(__dsqrt_rn(rr), bnorm);
    out[0] = 0.0;
    out[1] = scal[10];
    out[2] = rel;
    if (rel < tol) gate[0] = 2;
    scal[2] = rr / scal[4];  // beta
    scal[4] = rr;            // rz
  }
}

// p = z + b p  (solvers.py:209,255); coef == NULL -> p = z (252)
__global__ void __launch_bounds__(kBlock) xpby_kernel(long long n, double* __restrict__ p,
                                                      const double* __restrict__ z,
                                                      const double* __restrict__ coef) {
  const bool first = coef == nullptr;
  const double b = first ? 0.0 : coef[0];
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long long)gridDim.x * kBlock)
    p[i] = first ? z[i] : __dadd_rn(z[i], __dmul_rn(b, p[i]));
}

// solvers.py:162-163: {(b - Ax).(b - Ax)}
__global__ void __launch_bounds__(kBlock) resid_kernel(long long n, const double* __restrict__ b,
                                                       const double* __restrict__ ax,
                                                       double* __restrict__ parts) {
  __shared__ double sh[kBlock / 32];
  double v = 0.0;
  PSELL_GS_UNROLL
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long long)kRB * kBlock) {
    const double d = __dsub_rn(b[i], ax[i]);
    v += __dmul_rn(d, d);
  }
  v = block_sum<kBlock>(v, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = v;
}

// Jacobi z = r * inv (solvers.py:148-149), {r.z}
__global__ void __launch_bounds__(kBlock) precond_dot_kernel(long long n, double* __restrict__ z,
                                                             const double* __restrict__ r,
                                                             const double* __restrict__ inv,
                                                             double* __restrict__ parts) {
  __shared__ double sh[kBlock / 32];
  double v = 0.0;
  PSELL_GS_UNROLL
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long long)kRB * kBlock) {
    const double ri = r[i];
    const double zi = inv ? __dmul_rn(ri, inv[i]) : ri;
    if (inv) z[i] = zi;
    v += __dmul_rn(ri, zi);
  }
  v = block_sum<kBlock>(v, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = v;
}

__global__ void scalar_div_kernel(const double* num, const double* den, int np, int stride,
                                  double* dst, int32_t* flag, int check) {
  if (flag && *flag) return;
  double a = 0.0, b = 0.0;
  for (int i = 0; i < np; ++i) {
    a += num[(long long)i * stride];
    b += den[(long long)i * stride];
  }
  dst[1] = b;
  if (check && (b <= 0.0 || !isfinite(b))) {
    if (flag) *flag = 1;
    return;
  }
  dst[0] = a / b;
}

// FP64 PCG convergence gate (solvers.py:183-207 loop head): gate[0] = 0 running,
// 1 breakdown (written by scalar_div's curvature check), 2 converged; gate[1] =
// breakdown already reported.  Writes this iteration's status {breakdown, p.q,
// sqrt(r.r) / bnorm} (or {-1} when the solve had stopped before it) and closes
// the gate when the recurred residual is below tol, so iterations the host
// enqueued ahead of reading the status change nothing.  sqrt and / are IEEE
// round-to-nearest, the host's float(np.sqrt(rr)) / bnorm bit for bit.
__global__ void pcg_status_kernel(const double* pq, const double* rr, int32_t* gate, double bnorm, double tol,
                                  double* out) {
  const int g = gate[0];
  if (g == 2 || (g == 1 && gate[1])) {
    out[0] = -1.0;
    return;
  }
  const double rel = __ddiv_rn(__dsqrt_rn(rr[0]), bnorm);
  out[0] = g == 1 ? 1.0 : 0.0;
  out[1] = pq[0];
  out[2] = rel;
  if (g == 1) gate[1] = 1;
  else if (rel < tol) gate[0] = 2;
}

// out[j] = sum_{i < n_parts} parts[i * stride + j], j < n_out: rank-ordered global sums
__global__ void sum_strided_kernel(const double* parts, int np, int stride, int n_out, double* out) {
  const int j = threadIdx.x;
  if (j >= n_out) return;
  double s = 0.0;
  for (int i = 0; i < np; ++i) s += parts[(long long)i * stride + j];
  out[j] = s;
}

// traversal order of the inner PCG's vector passes (A/B knobs, read once per process):
// PSELL_UPD_REV / PSELL_DIR_REV = 1 walk the update / direction pass in descending rows
static bool env_flag(const char* name, int dflt) {
  const char* e = getenv(name);
  return (e ? atoi(e) : dflt) != 0;
}
static bool upd_rev() {
  static const bool v = env_flag("PSELL_UPD_REV", 0);
  return v;
}
static bool dir_rev() {
  static const bool v = env_flag("PSELL_DIR_REV", 1);
  return v;
}

static unsigned vgrid(long long n) {
  long long g = ceil_div(n, kBlock);
  if (g > kRB) g = kRB;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace psell

using namespace psell;

#define LAUNCH_OK() (cudaGetLastError() == cudaSuccess ? PSELL_OK : PSELL_ECUDA)

extern "C" {

int psell_sum_partials(const double* partials, int64_t n_partials, int32_t n_out, double* out,
                       const int32_t* skip_flag, void* stream) {
  sum_partials_kernel<<<1, 1024, 0, as_stream(stream)>>>(partials, n_partials, n_out, out, skip_flag);
  return LAUNCH_OK();
}

int psell_sum_strided(const double* parts, int32_t n_parts, int32_t stride, int32_t n_out, double* out,
                      void* stream) {
  sum_strided_kernel<<<1, 32, 0, as_stream(stream)>>>(parts, n_parts, stride, n_out, out);
  return LAUNCH_OK();
}

int psell_dot(const void* a, const void* b, int32_t dtype, int64_t n, double* partials, double* out,
              void* stream) {
  cudaStream_t st = as_stream(stream);
  if (dtype == PSELL_DT_F64)
    dot_kernel<double><<<kRB, kBlock, 0, st>>>(static_cast<const double*>(a), static_cast<const double*>(b), n, partials);
  else if (dtype == PSELL_DT_F32)
    dot_kernel<float><<<kRB, kBlock, 0, st>>>(static_cast<const float*>(a), static_cast<const float*>(b), n, partials);
  else
    return PSELL_EARG;
  finalize(partials, kRB, 1, out, nullptr, st);
  return LAUNCH_OK();
}

int psell_ipcg_begin(int64_t n, const double* r64, float* x, float* r, float* z, float* p,
                     const float* inv_diag, double* partials, double* local_out, void* stream) {
  cudaStream_t st = as_stream(stream);
  ipcg_begin_kernel<<<kRB, kBlock, 0, st>>>(n, r64, x, r, z, p, inv_diag, partials);
  finalize(partials, kRB, 1, local_out, nullptr, st);
  return LAUNCH_OK();
}

int psell_ipcg_set_rz(const double* parts, int32_t n_parts, int32_t stride, double* scal, int32_t* iflags, void* stream) {
  ipcg_set_rz_kernel<<<1, 1, 0, as_stream(stream)>>>(parts, n_parts, stride, scal, iflags, nullptr);
  return LAUNCH_OK();
}

int psell_ipcg_set_rz_gated(const double* parts, int32_t n_parts, int32_t stride, double* scal, int32_t* iflags,
                            const int32_t* gate, void* stream) {
  ipcg_set_rz_kernel<<<1, 1, 0, as_stream(stream)>>>(parts, n_parts, stride, scal, iflags, gate);
  return LAUNCH_OK();
}

int psell_ipcg_alpha(const double* parts, int32_t n_parts, int32_t stride, double* scal, int32_t* iflags, void* stream) {
  ipcg_alpha_kernel<<<1, 1, 0, as_stream(stream)>>>(parts, n_parts, stride, scal, iflags);
  return LAUNCH_OK();
}

int psell_ipcg_update(int64_t n, float* x, float* r, float* z, const float* p, const float* q,
                      const float* inv_diag, const double* scal, const int32_t* iflags,
                      double* partials, double* local_out, void* stream) {
  cudaStream_t st = as_stream(stream);
  const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(r) | reinterpret_cast<uintptr_t>(z) |
                     reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(inv_diag)) & 15) == 0;
  double* sc = const_cast<double*>(scal);
  int32_t* fl = const_cast<int32_t*>(iflags);
  if (vec) ipcg_update_kernel<true><<<kRB, kBlock, 0, st>>>(n, x, r, z, p, q, inv_diag, sc, fl, partials, nullptr, upd_rev());
  else ipcg_update_kernel<false><<<kRB, kBlock, 0, st>>>(n, x, r, z, p, q, inv_diag, sc, fl, partials, nullptr);
  finalize(partials, kRB, 1, local_out, iflags, st);
  return LAUNCH_OK();
}

int psell_ipcg_update_beta(int64_t n, float* x, float* r, float* z, const float* p, const float* q,
                           const float* inv_diag, double* scal, int32_t* iflags, double* partials,
                           unsigned* ticket, void* stream) {
  if (!ticket) return 1;
  cudaStream_t st = as_stream(stream);
  const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(r) | reinterpret_cast<uintptr_t>(z) |
                     reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(inv_diag)) & 15) == 0;
  if (vec) ipcg_update_kernel<true><<<kRB, kBlock, 0, st>>>(n, x, r, z, p, q, inv_diag, scal, iflags, partials, ticket, upd_rev());
  else ipcg_update_kernel<false><<<kRB, kBlock, 0, st>>>(n, x, r, z, p, q, inv_diag, scal, iflags, partials, ticket);
  return LAUNCH_OK();
}

// psell_ipcg_update_beta across G ranks: the last CTA all-reduces r.z over the peer arenas
// (K8 protocol, one value) before the beta step (reference solvers.py:300-306 on a slab)
int psell_ipcg_update_beta_peer(int64_t n, float* x, float* r, float* z, const float* p, const float* q,
                                const float* inv_diag, double* scal, int32_t* iflags, double* partials,
                                unsigned* ticket, int32_t G, int32_t rank, const uint64_t* peers, int64_t timeout_ns,
                                void* stream) {
  if (!ticket || G < 1 || G > kPeerMax || rank < 0 || rank >= G || (G > 1 && !peers)) return PSELL_EARG;
  cudaStream_t st = as_stream(stream);
  const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(r) | reinterpret_cast<uintptr_t>(z) |
                     reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(inv_diag)) & 15) == 0;
  const unsigned long long* pp = reinterpret_cast<const unsigned long long*>(peers);
  if (vec)
    ipcg_update_kernel<true><<<kRB, kBlock, 0, st>>>(n, x, r, z, p, q, inv_diag, scal, iflags, partials, ticket,
                                                     upd_rev(), pp, G, rank, timeout_ns);
  else
    ipcg_update_kernel<false><<<kRB, kBlock, 0, st>>>(n, x, r, z, p, q, inv_diag, scal, iflags, partials, ticket,
                                                      false, pp, G, rank, timeout_ns);
  return LAUNCH_OK();
}

int psell_ipcg_beta(const double* parts, int32_t n_parts, int32_t stride, double* scal, int32_t* iflags, void* stream) {
  ipcg_beta_kernel<<<1, 1, 0, as_stream(stream)>>>(parts, n_parts, stride, scal, iflags);
  return LAUNCH_OK();
}

int psell_ipcg_direction(int64_t n, float* p, const float* z, const double* scal,
                         const int32_t* iflags, void* stream) {
  ipcg_direction_kernel<<<vgrid(n) * 2, kBlock, 0, as_stream(stream)>>>(n, p, z, scal, iflags);
  return LAUNCH_OK();
}

int psell_ipcg_direction_x(int64_t n, float* p, const float* z, float* x, const double* scal,
                           const int32_t* iflags, void* stream) {
  ipcg_direction_x_kernel<<<vgrid(n) * 2, kBlock, 0, as_stream(stream)>>>(n, p, z, x, scal, iflags, dir_rev());
  return LAUNCH_OK();
}

int psell_ipcg_direction_x_push(int64_t n, float* p, const float* z, float* x, const double* scal,
                                const int32_t* iflags, int32_t G, int32_t rank, const uint64_t* peers, int64_t row0,
                                int64_t vec_off, int32_t n_ranges, const int64_t* lo, const int64_t* hi,
                                const int32_t* dst, int64_t timeout_ns, void* stream) {
  if (G < 2 || G > kPeerMax || rank < 0 || rank >= G || !peers || n_ranges < 0 || n_ranges > kHaloRanges ||
      (n_ranges > 0 && (!lo || !hi || !dst)))
    return PSELL_EARG;
  HaloRanges hr;
  hr.n = n_ranges;
  for (int k = 0; k < kHaloRanges; ++k) {
    hr.lo[k] = k < n_ranges ? lo[k] : 0;
    hr.hi[k] = k < n_ranges ? hi[k] : 0;
    hr.dst[k] = k < n_ranges ? dst[k] : 0;
    if (k < n_ranges && (dst[k] < 0 || dst[k] >= G || dst[k] == rank)) return PSELL_EARG;
  }
  ipcg_direction_x_push_kernel<<<vgrid(n) * 2, kBlock, 0, as_stream(stream)>>>(
      n, p, z, x, scal, iflags, dir_rev(), reinterpret_cast<const unsigned long long*>(peers), G, rank, row0, vec_off,
      hr, timeout_ns);
  return LAUNCH_OK();
}

int psell_ipcg_end(int64_t n, const float* x, double* z64, void* stream) {
  ipcg_end_kernel<<<vgrid(n) * 2, kBlock, 0, as_stream(stream)>>>(n, x, z64);
  return LAUNCH_OK();
}

int psell_fcg_zr(int64_t n, const double* z, const double* r, const double* r_prev,
                 double* partials, double* out2, void* stream) {
  cudaStream_t st = as_stream(stream);
  fcg_zr_kernel<<<kRB, kBlock, 0, st>>>(n, z, r, r_prev, partials);
  finalize(partials, kRB, 2, out2, nullptr, st);
  return LAUNCH_OK();
}

int psell_pq_pr(int64_t n, const double* p, const double* q, const double* r, double* partials,
                double* out2, void* stream) {
  cudaStream_t st = as_stream(stream);
  pq_pr_kernel<<<kRB, kBlock, 0, st>>>(n, p, q, r, partials);
  finalize(partials, kRB, 2, out2, nullptr, st);
  return LAUNCH_OK();
}

int psell_axpy2(int64_t n, double* x, double* r, const double* p, const double* q,
                const double* coef, const int32_t* skip_flag, double* partials, double* out1,
                void* stream) {
  cudaStream_t st = as_stream(stream);
  axpy2_kernel<<<kRB, kBlock, 0, st>>>(n, x, r, p, q, coef, skip_flag, partials);
  finalize(partials, kRB, 1, out1, skip_flag, st);
  return LAUNCH_OK();
}

int psell_pcg_update_status(int64_t n, double* x, double* r, const double* p, const double* q, double* scal,
                            int32_t* gate, double bnorm, double tol, double* out, double* partials,
                            unsigned* ticket, void* stream) {
  if (!ticket || !gate || !scal || !out) return PSELL_EARG;
  pcg_update_status_kernel<<<kRB, kBlock, 0, as_stream(stream)>>>(n, x, r, p, q, scal, gate, bnorm, tol, out,
                                                                   partials, ticket);
  return LAUNCH_OK();
}

int psell_xpby(int64_t n, double* p, const double* z, const double* coef, void* stream) {
  xpby_kernel<<<vgrid(n) * 2, kBlock, 0, as_stream(stream)>>>(n, p, z, coef);
  return LAUNCH_OK();
}

// p = z + b p unless the inner-PCG breakdown flag is set (f64 inner, solvers.py:307)
__global__ void __launch_bounds__(kBlock) xpby_checked_kernel(long long n, double* __restrict__ p,
                                                              const double* __restrict__ z,
                                                              const double* __restrict__ coef,
                                                              const int32_t* __restrict__ iflags) {
  if (iflags[0]) return;
  const double b = coef[0];
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long long)gridDim.x * kBlock)
    p[i] = __dadd_rn(z[i], __dmul_rn(b, p[i]));
}

int psell_xpby_checked(int64_t n, double* p, const double* z, const double* coef, const int32_t* iflags,
                       void* stream) {
  xpby_checked_kernel<<<vgrid(n) * 2, kBlock, 0, as_stream(stream)>>>(n, p, z, coef, iflags);
  return LAUNCH_OK();
}

int psell_resid(int64_t n, const double* b, const double* ax, double* partials, double* out1,
                void* stream) {
  cudaStream_t st = as_stream(stream);
  resid_kernel<<<kRB, kBlock, 0, st>>>(n, b, ax, partials);
  finalize(partials, kRB, 1, out1, nullptr, st);
  return LAUNCH_OK();
}

int psell_precond_dot(int64_t n, double* z, const double* r, const double* inv, double* partials,
                      double* out1, void* stream) {
  cudaStream_t st = as_stream(stream);
  precond_dot_kernel<<<kRB, kBlock, 0, st>>>(n, z, r, inv, partials);
  finalize(partials, kRB, 1, out1, nullptr, st);
  return LAUNCH_OK();
}

int psell_scalar_div(const double* num_parts, const double* den_parts, int32_t n_parts,
                     int32_t stride, double* dst, int32_t* flag, int32_t check_curvature,
                     void* stream) {
  scalar_div_kernel<<<1, 1, 0, as_stream(stream)>>>(num_parts, den_parts, n_parts, stride, dst,
                                                    flag, check_curvature);
  return LAUNCH_OK();
}

int psell_pcg_status(const double* pq, const double* rr, int32_t* gate, double bnorm, double tol, double* out,
                     void* stream) {
  pcg_status_kernel<<<1, 1, 0, as_stream(stream)>>>(pq, rr, gate, bnorm, tol, out);
  return LAUNCH_OK();
}

}  // extern "C"
