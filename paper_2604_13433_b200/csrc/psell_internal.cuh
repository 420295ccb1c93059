// Internal helpers shared by the libpsell translation units (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/psell.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libpsell is built for sm_100a only"
#endif

namespace psell {

constexpr int kBlock = 256;

// ---------------------------------------------------------------- errors
inline int set_err(psell_error* e, int code, int kind, int64_t index, int64_t aux, double value,
                   const char* msg) {
  if (e) {
    e->code = code;
    e->kind = kind;
    e->index = index;
    e->aux = aux;
    e->value = value;
    snprintf(e->msg, sizeof(e->msg), "%s", msg ? msg : "");
  }
  return code;
}

inline int ok(psell_error* e) { return set_err(e, PSELL_OK, PSELL_KIND_NONE, -1, 0, 0.0, ""); }

inline int cuda_err(psell_error* e, cudaError_t st, const char* where) {
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", where, cudaGetErrorString(st));
  return set_err(e, PSELL_ECUDA, PSELL_KIND_CUDA, -1, 0, 0.0, buf);
}

#define PSELL_CHECK_LAUNCH(err, where)                         \
  do {                                                         \
    cudaError_t _st = cudaGetLastError();                      \
    if (_st != cudaSuccess) return ::psell::cuda_err(err, _st, where); \
  } while (0)

#define PSELL_CUDA(call, err)                                  \
  do {                                                         \
    cudaError_t _st = (call);                                  \
    if (_st != cudaSuccess) return ::psell::cuda_err(err, _st, #call); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// ---------------------------------------------------------------- format
struct Fmt {
  int w, d, codec;
  __host__ __device__ int v() const { return w - d - 1; }
};

inline Fmt fmt_of(const psell_desc* d) { return Fmt{d->w, d->d, d->codec}; }

// codec.py:45-62 (host-side re-validation at the ABI boundary)
inline bool fmt_valid(const Fmt& f) {
  if (f.w != 32 && f.w != 64) return false;
  if (f.d < 1 || f.d > f.w - 2) return false;
  int v = f.w - f.d - 1;
  if (f.codec == PSELL_FP16) return v == 16;
  if (f.codec == PSELL_E8MY) return f.w == 32 && v - 9 >= 1;
  if (f.codec == PSELL_FP32EMBED) return f.w == 64 && v >= 32;
  return false;
}

// The device build / SpMV / decode read fp16 words as 32-bit words (D = 15).
// PackFormat(64, 47, "fp16") passes codec.py:45-62, but its reference decode
// takes the value from bits 16..31 of the 64-bit word (codec.py:242), i.e. from
// delta bits: it is rejected here instead of being reproduced.
inline bool fmt_device_ok(const Fmt& f) { return fmt_valid(f) && !(f.codec == PSELL_FP16 && f.w != 32); }
#define PSELL_FP16_W64_MSG "fp16 values need 32-bit words on the device (PackFormat(64, 47, 'fp16') is not supported)"

// ---------------------------------------------------------------- encode
// Error codes of the per-value encoders.
enum { ENC_OK = 0, ENC_NONFINITE = 1, ENC_OVERFLOW = 2 };

// f64 -> IEEE half, direct round-to-nearest-even (codec.py:130-138).
// __double2half lowers to cvt.rn.f16.f64 on sm_100a (no f32 double rounding).
__device__ __forceinline__ uint32_t enc_fp16(double v, int& st) {
  if (!isfinite(v)) { st = ENC_NONFINITE; return 0u; }
  unsigned short b = __half_as_ushort(__double2half(v));
  if ((b & 0x7FFFu) == 0x7C00u) st = ENC_OVERFLOW;
  return (uint32_t)b;
}

// e8my: f64 -> f32 RNE, subnormal flush to signed zero, then round half away
// from zero at mantissa bit D on the integer form, inf => overflow
// (codec.py:141-160; integer form verified in SURVEY.md App. A.2).
__device__ __forceinline__ uint32_t enc_e8my(double v, int d, int& st) {
  if (!isfinite(v)) { st = ENC_NONFINITE; return 0u; }
  uint32_t b = __float_as_uint(__double2float_rn(v));
  uint32_t sign = b & 0x80000000u;
  uint32_t mag = b & 0x7FFFFFFFu;
  uint32_t r = 0u;
  if (mag >= 0x00800000u) {
    r = (mag + (1u << d)) & ~((2u << d) - 1u);
    if (r >= 0x7F800000u) st = ENC_OVERFLOW;
  }
  return (sign | r) >> (d + 1);
}

// fp32embed: f32 bits << (V - 32) (codec.py:163-170).
__device__ __forceinline__ uint64_t enc_fp32(double v, int vbits, int& st) {
  if (!isfinite(v)) { st = ENC_NONFINITE; return 0ull; }
  float f = __double2float_rn(v);
  if (isinf(f)) st = ENC_OVERFLOW;
  return ((uint64_t)__float_as_uint(f)) << (vbits - 32);
}

__device__ __forceinline__ uint64_t encode_value(const Fmt& f, double v, int& st) {
  if (f.codec == PSELL_FP16) return enc_fp16(v, st);
  if (f.codec == PSELL_E8MY) return enc_e8my(v, f.d, st);
  return enc_fp32(v, f.v(), st);
}

// ---------------------------------------------------------------- decode
// Branch-free unpack (codec.py:227-250).  Flag in bit 0, delta above it.
template <typename W>
__device__ __forceinline__ W unpack_delta(W w, int d) {
  const W flag = w & W(1);
  const W mask = flag ? ((W(1) << d) - W(1)) : ~W(0);
  return (w >> 1) & mask;
}

// value bits of an e8my word as f32 (0 for flag == 0)
__device__ __forceinline__ float e8my_value(uint32_t w, int d) {
  uint32_t keep = (w & 1u) ? ~((2u << d) - 1u) : 0u;
  return __uint_as_float(w & keep);
}

__device__ __forceinline__ __half fp16_value(uint32_t w) {
  return __ushort_as_half((unsigned short)((w & 1u) ? (w >> 16) : 0u));
}

__device__ __forceinline__ float fp32e_value(uint64_t w) {
  return __uint_as_float((w & 1ull) ? (uint32_t)(w >> 32) : 0u);
}

// ---------------------------------------------------------------- loads
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// streaming (read-once) 32/64-bit loads: no L1 allocation, L2 evict-first
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t ld_stream(const uint64_t* p, uint64_t pol) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], %2;"
               : "=l"(v) : "l"(p), "l"(pol));
  return v;
}

// gathered (reused) loads of x: read-only path, L2 evict-last
__device__ __forceinline__ unsigned short ld_keep_u16(const unsigned short* p, uint64_t pol) {
  unsigned short v;
  asm("ld.global.nc.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_keep(const float* p, uint64_t pol) {
  float v;
  asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_keep(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ __half ld_keep(const __half* p, uint64_t pol) {
  return __ushort_as_half(ld_keep_u16(reinterpret_cast<const unsigned short*>(p), pol));
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ long long warp_max_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic CTA sum (fixed tree); result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh /* NT/32 */) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = (lane < NT / 32) ? sh[lane] : 0.0;
    t = warp_sum(t);
  }
  __syncthreads();
  return t;
}

// Fixed-order grid reduction epilogue ("last CTA reduces"), two levels so no
// thread ever walks a long chain of dependent loads.  Thread 0 of every CTA
// has stored parts[blockIdx.x].  CTAs form groups of NT; the last CTA of a
// group to arrive (ticket tickets[1 + g]) sums the group's partials (one load
// per thread, fixed CTA tree) into parts[gridDim.x + g]; the last group to
// finish (ticket tickets[0]) sums the group partials the same way.  Every sum
// has a fixed association, so the total is deterministic run to run.  Returns
// true in that final CTA (total valid in thread 0) and re-arms its tickets.
// Needs parts[gridDim.x + ceil(gridDim.x / NT)] and tickets[1 + ceil(gridDim.x / NT)],
// all tickets zero before the first launch.
template <int NT>
__device__ __forceinline__ bool last_cta_sum(double* parts, unsigned* tickets, double& total,
                                             double* sh /* NT/32 */) {
  __shared__ unsigned s_last;
  const unsigned n_grp = (gridDim.x + NT - 1) / NT;
  const unsigned g = blockIdx.x / NT;
  const unsigned g_size = min((unsigned)NT, gridDim.x - g * NT);
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(tickets + 1 + g, 1u) == g_size - 1;
  }
  __syncthreads();
  if (!s_last) return false;
  double v = threadIdx.x < g_size ? __ldcg(parts + g * NT + threadIdx.x) : 0.0;
  v = block_sum<NT>(v, sh);
  if (threadIdx.x == 0) {
    parts[gridDim.x + g] = v;
    tickets[1 + g] = 0u;
    __threadfence();
    s_last = atomicAdd(tickets, 1u) == n_grp - 1;
  }
  __syncthreads();
  if (!s_last) return false;
  double w = 0.0;
  for (unsigned i = threadIdx.x; i < n_grp; i += NT) w += __ldcg(parts + gridDim.x + i);
  total = block_sum<NT>(w, sh);
  if (threadIdx.x == 0) tickets[0] = 0u;
  return true;
}

// inner-PCG scalar steps shared by the fused epilogues (solvers.py:295-299, 304-306)
// scal: [0]=rz [1]=pq [2]=alpha [3]=beta [4]=rz_new ; iflags: [0]=breakdown [1]=done
__device__ __forceinline__ void ipcg_alpha_step(double pq, double* scal, int32_t* iflags) {
  scal[1] = pq;
  if (pq <= 0.0 || !isfinite(pq) || scal[0] == 0.0) {
    iflags[0] = 1;
    return;
  }
  scal[2] = scal[0] / pq;
}

// shared-memory mbarrier + bulk-copy (TMA 1-D) helpers of the staged kernels
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// ---- peer-memory arena protocol (K8, csrc/peer.cu; layout in include/psell.h)
constexpr int kPeerMax = 64;
constexpr int kFlagOff = 0;
constexpr int kEpochOff = 256;
constexpr int kTicketOff = 260;
constexpr int kErrOff = 264;
constexpr int kGlobOff = 4096;

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_relaxed_sys(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// The dot all-reduce of the fused distributed inner PCG, run by ONE thread (thread 0 of the
// last CTA of the kernel that produced this rank's sum): one exchange of the K8 protocol
// with a single value -- store `local` into every peer's glob[parity][rank][0], fence at
// system scope, release this rank's epoch into every peer's flag, acquire-wait for every
// peer's flag, and return the rank-ordered sum (the order the scalar kernels use), so a
// fused kernel's epilogue replaces the separate partial-sum, exchange and scalar kernels.
// A wait past timeout_ns sets the arena's error word and returns the partial sum (the
// host raises on it after the solve).
__device__ __forceinline__ double peer_allreduce1(int G, int rank, const unsigned long long* peers,
                                                  long long timeout_ns, double local) {
  unsigned char* self = reinterpret_cast<unsigned char*>(peers[rank]);
  uint32_t* flags = reinterpret_cast<uint32_t*>(self + kFlagOff);
  uint32_t* epoch_p = reinterpret_cast<uint32_t*>(self + kEpochOff);
  const uint32_t e = *reinterpret_cast<volatile uint32_t*>(epoch_p) + 1u;
  const int par = e & 1;
  for (int p = 0; p < G; ++p) {
    double* g = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(peers[p]) + kGlobOff);
    g[(par * kPeerMax + rank) * 8] = local;
  }
  __threadfence_system();
  for (int p = 0; p < G; ++p)
    st_release_sys(reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(peers[p]) + kFlagOff) + rank, e);
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
  const double* g = reinterpret_cast<const double*>(self + kGlobOff);
  double s = 0.0;
  for (int q = 0; q < G; ++q) s += ld_relaxed_sys(g + (par * kPeerMax + q) * 8);
  *epoch_p = e;
  return s;
}

// FP64 PCG scalar steps of the fused iteration (solvers.py:196-207), identity preconditioner.
// scal: [0]=alpha [1]=pq [2]=beta [4]=rz [10]=pq [12]=rr; gate: see psell_pcg_status
__device__ __forceinline__ void pcg_alpha_step(double pq, double* scal, int32_t* gate) {
  scal[1] = pq;
  scal[10] = pq;
  if (pq <= 0.0 || !isfinite(pq)) {
    gate[0] = 1;
    return;
  }
  scal[0] = scal[4] / pq;
}

__device__ __forceinline__ void ipcg_beta_step(double rz_new, double* scal, int32_t* iflags) {
  scal[4] = rz_new;
  scal[3] = rz_new / scal[0];
  scal[0] = rz_new;
  iflags[1] += 1;
}

}  // namespace psell

namespace psell {
// out[0] = 0, out[i+1] = in[0] + ... + in[i]   (build.cu); tmp >= ceil(n/4096)+1 longs
int scan_i64(const long long* in, long long n, long long* tmp, long long* out, cudaStream_t st,
             psell_error* err);
// storage-row -> original-row order stored in a psell_build_plan workspace (build.cu)
const int32_t* build_ws_order(const psell_desc* d, const void* ws);
}  // namespace psell
