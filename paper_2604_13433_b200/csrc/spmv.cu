// K2 — PackSELL SpMV and K5 — PackSELL -> CSR decode, sm_100a.
//
// Replaces packsell_spmv (reference packed.py:242-271), unpack_words
// (codec.py:227-250) and packsell_to_csr (packed.py:274-303).
//
// Mapping (one thread per row): thread <-> storage row.
// For C = 32 a warp owns one slice, so step q of all 32 lanes is one
// contiguous 128 B line of `pack` (column-major slices, packed.py:224).  The
// fast kernel streams those lines with L1::no_allocate + L2 evict_first
// loads, U steps per batch, double buffered in registers so 2U lines per warp
// are in flight; it decodes branch-free (flag/delta/value with SEL+LOP), runs
// the column cursor as a 32-bit register prefix, gathers x through the
// read-only path with an L2 evict_last policy (x stays L2 resident while the
// 2 GB pack streams past it) and accumulates with FP32 FMA.  REF_ORDER
// switches to numpy's rounding (value cast to x dtype, separately rounded
// product and sum) for bitwise parity.  Generic C uses the same thread/row
// mapping without the warp-uniform fast path.
#include "psell_internal.cuh"

#include <atomic>

namespace psell {

struct SpmvArgs {
  const void* pack;
  const int64_t* offset;
  const void* perm;
  const void* x;
  void* y;
  const float* p_own;
  double* partials;
  const int32_t* skip;
  // fused alpha epilogue (psell_spmv_dot_alpha): last CTA sums the partials
  unsigned* ticket;
  double* scal;
  int32_t* iflags;
  // ... and, across ranks (psell_spmv_dot_alpha_peer), all-reduces the sum over the
  // peer-memory arenas before the alpha step (peer_G > 1)
  const unsigned long long* peers;
  int peer_G, peer_rank;
  long long peer_timeout;
  long long n_rows, n_cols, n_slices, row0, k_left;
  int c, se, sigma, mode, d, perm_bytes;
  int variant;  // 0: register-pipelined kernels (default), 2: persistent TMA stream
  int narrow;   // mean slice width <= 12 steps (PSELL_SPMV_NARROW)
  int narrow12; // every slice <= 12 steps (PSELL_SPMV_NARROW12): the slot kernel applies
  int w32;      // every slice <= 32 steps (PSELL_SPMV_W32): the wide TMA kernel applies
  int codec;
  // long-slice segmentation (0 = off): slices wider than seg_len steps run as
  // segments (see spmv_seg_kernel)
  int seg_len;
  // bulk L2 prefetch of each slice pair's words at warp start (dual kernel,
  // non-persistent pair kernel: 27-point 359 -> 325 us).  PSELL_L2PF=0 disables
  // (A/B).  Prefetching the next pair in the persistent pair kernel was measured
  // slower (7-point 166 -> 180-187 us) and is not implemented.
  int l2pf;
  int sched_static;  // sched holds the static pair ranges behind the counters (PSELL_DSTATIC)
  const int32_t* seg_slice;   // [n_seg] slice of each segment
  const int32_t* seg_q0;      // [n_seg] first step of each segment
  uint32_t* seg_c2;           // [n_seg][32] cursor checkpoints (2 * column)
  float* seg_partial;         // [n_seg][32] partial sums
  const int32_t* long_slice;  // [n_long] slices run as segments
  const int32_t* long_seg0;   // [n_long + 1] first segment of each long slice
  // n / se and n / sigma for n < 2^31 as (umulhi(n, m) + n) >> l (Granlund-Montgomery)
  uint32_t se_m, se_l, sig_m, sig_l;
  // SM-affine persistent scheduling of the dual kernel (irregular matrices):
  // claim counters, one per chunk, + exit count; zero between launches
  uint32_t* sched;
  int aff_chunks;
};

// (m, l) with n / d == (umulhi(n, m) + n) >> l for every n < 2^31 (d >= 1)
static inline void magic_div(uint32_t d, uint32_t& m, uint32_t& l) {
  l = 0;
  while ((1ull << l) < d) ++l;
  m = (uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1);
}

__device__ __forceinline__ uint32_t fast_div(uint32_t n, uint32_t m, uint32_t l) {
  return (__umulhi(n, m) + n) >> l;
}

// One TMA-engine L2 prefetch of a contiguous byte range (16-B aligned, multiple
// of 16 B): the slice pair's whole word stream is requested from HBM up front,
// without holding registers, so the chunked register loads that follow hit L2.
__device__ __forceinline__ void l2_prefetch_bulk(const void* p, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p), "r"(bytes), "l"(pol)
               : "memory");
}

template <int CODEC> struct WordOf { using T = uint32_t; };
template <> struct WordOf<PSELL_FP32EMBED> { using T = uint64_t; };

// ---- value decode: returns the value as f32 (exact for every codec) and,
//      for REF mode with half x, the value rounded to half.
template <int CODEC, typename W>
__device__ __forceinline__ float word_value(W w, int d) {
  if constexpr (CODEC == PSELL_FP16) return __half2float(fp16_value((uint32_t)w));
  else if constexpr (CODEC == PSELL_E8MY) return e8my_value((uint32_t)w, d);
  else return fp32e_value((uint64_t)w);
}

template <int CODEC, typename W>
__device__ __forceinline__ __half word_value_h(W w, int d) {
  if constexpr (CODEC == PSELL_FP16) return fp16_value((uint32_t)w);
  else return __float2half_rn(word_value<CODEC, W>(w, d));
}

template <int CODEC>
__device__ __forceinline__ int word_dbits(int d) {
  if constexpr (CODEC == PSELL_FP16) return 15;
  else return d;
}

// Accumulator policy.  REF: numpy order in the x dtype.  Fast: FP32 FMA (FP64 for f64 x).
template <typename XT, bool REF> struct Acc;
template <> struct Acc<__half, true> {
  using T = __half;
  __device__ static T zero() { return __ushort_as_half(0); }
  template <int CODEC, typename W>
  __device__ static T step(T acc, W w, int d, __half xv) {
    return __hadd_rn(acc, __hmul_rn(word_value_h<CODEC, W>(w, d), xv));
  }
  __device__ static __half out(T a) { return a; }
  __device__ static float as_f(T a) { return __half2float(a); }
};
template <> struct Acc<__half, false> {
  using T = float;
  __device__ static T zero() { return 0.f; }
  template <int CODEC, typename W>
  __device__ static T step(T acc, W w, int d, __half xv) {
    return fmaf(word_value<CODEC, W>(w, d), __half2float(xv), acc);
  }
  __device__ static __half out(T a) { return __float2half_rn(a); }
};
template <> struct Acc<float, true> {
  using T = float;
  __device__ static T zero() { return 0.f; }
  template <int CODEC, typename W>
  __device__ static T step(T acc, W w, int d, float xv) {
    return __fadd_rn(acc, __fmul_rn(word_value<CODEC, W>(w, d), xv));
  }
  __device__ static float out(T a) { return a; }
};
template <> struct Acc<float, false> {
  using T = float;
  __device__ static T zero() { return 0.f; }
  template <int CODEC, typename W>
  __device__ static T step(T acc, W w, int d, float xv) {
    return fmaf(word_value<CODEC, W>(w, d), xv, acc);
  }
  __device__ static float out(T a) { return a; }
};
template <> struct Acc<double, true> {
  using T = double;
  __device__ static T zero() { return 0.0; }
  template <int CODEC, typename W>
  __device__ static T step(T acc, W w, int d, double xv) {
    return __dadd_rn(acc, __dmul_rn((double)word_value<CODEC, W>(w, d), xv));
  }
  __device__ static double out(T a) { return a; }
};
template <> struct Acc<double, false> {
  using T = double;
  __device__ static T zero() { return 0.0; }
  template <int CODEC, typename W>
  __device__ static T step(T acc, W w, int d, double xv) {
    return fma((double)word_value<CODEC, W>(w, d), xv, acc);
  }
  __device__ static double out(T a) { return a; }
};

template <typename XT> __device__ __forceinline__ float to_f(XT v);
template <> __device__ __forceinline__ float to_f<__half>(__half v) { return __half2float(v); }
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<double>(double v) { return (float)v; }

__device__ __forceinline__ long long storage_base(long long s_global, int se, long long k_left,
                                                  long long n_cols) {
  const long long blk = (s_global / se) * se;
  long long d = blk > k_left ? blk - k_left : 0;
  const long long cmax = n_cols > 0 ? n_cols - 1 : 0;
  return d < cmax ? d : cmax;
}

__device__ __forceinline__ long long out_row(const SpmvArgs& a, long long s) {
  if (a.mode != PSELL_MODE_IMPLICIT) return s;
  const long long blk = (s / a.sigma) * a.sigma;
  const int p = a.perm_bytes == 1 ? (int)static_cast<const uint8_t*>(a.perm)[s]
                                  : (int)static_cast<const uint16_t*>(a.perm)[s];
  return blk + p;
}

template <bool DOT, int NT = kBlock>
__device__ __forceinline__ void finish_dot(const SpmvArgs& a, double v) {
  if constexpr (DOT) {
    __shared__ double sh[NT / 32];
    const double t = block_sum<NT>(v, sh);
    if (threadIdx.x == 0) a.partials[blockIdx.x] = t;
    double pq;
    if (a.ticket && last_cta_sum<NT>(a.partials, a.ticket, pq, sh) && threadIdx.x == 0) {
      if (a.peer_G > 1) pq = peer_allreduce1(a.peer_G, a.peer_rank, a.peers, a.peer_timeout, pq);
      ipcg_alpha_step(pq, a.scal, a.iflags);
    }
  }
}

constexpr int kWarpsPerCta = kBlock / 32;
#ifndef PSELL_PAIR_U
#define PSELL_PAIR_U 12  // tail steps of the persistent pair kernel
#endif
// split point of the pair kernel's tail: steps [0, K) always decoded, [K, U) only when reached
template <int U> struct PairK {
#ifdef PSELL_PAIR_K
  static constexpr int K = PSELL_PAIR_K < U ? PSELL_PAIR_K : U;
#else
  static constexpr int K = 3 * U / 4;
#endif
};
#ifndef PSELL_PAIR_MINB
#define PSELL_PAIR_MINB 6  // resident 256-thread pair-kernel CTAs per SM the register budget is sized for (40 regs)
#endif

// A/B knobs: getenv once per call site, re-read after psell_reload_env() (the
// launch path of a small SpMV is host-bound; a getenv scans the environment)
static std::atomic<unsigned> g_env_gen{1};
struct EnvCache {
  unsigned gen = 0;
  bool set = false;
  int val = 0;
};
static inline bool env_int(EnvCache& c, const char* name, int& v) {
  const unsigned g = g_env_gen.load(std::memory_order_relaxed);
  if (c.gen != g) {
    const char* e = getenv(name);
    c.set = e != nullptr;
    c.val = e ? atoi(e) : 0;
    c.gen = g;
  }
  v = c.val;
  return c.set;
}

// dual-slice kernel switch (PSELL_DUAL=1 forces it on, =0 off; A/B)
static bool dual_slices(long long n_slices) {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_DUAL", v)) return v != 0;
  return n_slices >= 2;  // measured faster than one slice per warp on configs 2, 3, 5
}

// steps per chunk of the dual-slice kernel (PSELL_DUAL_U overrides: 8 | 12)
static int dual_chunk(bool narrow) {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_DUAL_U", v) && (v == 8 || v == 12)) return v;
  return narrow ? 12 : 8;  // 12 covers a whole 7-point slice in one chunk (sweep: +14 %)
}

// exact-tail pair kernel instead of the chunk-rounded dual kernel (PSELL_PAIR=0: dual, A/B)
static bool pair_kernel() {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_PAIR", v)) return v != 0;
  return true;
}

// CTA size of the narrow pair kernel (PSELL_PAIR_NT = 64 | 128 | 256, A/B).  128
// measured ~2.5 % faster than 256 on 7-point slices (smaller CTAs retire sooner);
// the fused-dot variant keeps 256 so its partial count (one per CTA) stays small.
static int pair_nt(bool dot) {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_PAIR_NT", v) && (v == 64 || v == 128 || v == 256)) return v;
  return dot ? 256 : 128;
}

// persistent grid-stride pair kernel: one resident wave of 6 CTAs per SM walks the
// slice pairs (PSELL_PAIR_PERSIST = CTAs per SM, 0 = one CTA per 8 pairs; A/B).
// 7-point 256^3: 164 vs 170 us plain, 169 vs 183 us with the fused dot, whose
// partials (and fixed-order last-CTA sum) shrink to one per resident CTA.
// Returns its grid (0 = not used).
static int sm_count();
static unsigned pair_persist_grid(long long n_slices, bool dot) {
  int per_sm = PSELL_PAIR_MINB;
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_PAIR_PERSIST", v)) per_sm = v;
  (void)dot;
  if (per_sm <= 0) return 0;
  if (per_sm > PSELL_PAIR_MINB) per_sm = PSELL_PAIR_MINB;
  const long long full = ceil_div(ceil_div(n_slices, 2), kWarpsPerCta);
  const long long cap = (long long)sm_count() * per_sm;
  return (unsigned)(full < cap ? full : cap);
}

// narrow kernel for slices of <= 12 steps (PSELL_NARROW=0: the persistent pair kernel, A/B)
// and its resident CTAs per SM (PSELL_NARROW_MINB = 4 | 5: 64 / 48 registers)
static bool narrow_on() {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_NARROW", v)) return v != 0;
  return true;
}
static int narrow_minb() {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_NARROW_MINB", v) && (v == 4 || v == 5)) return v;
  return 4;
}
static bool narrow_tma();
static unsigned narrow_grid(long long n_slices) {
  const long long full = ceil_div(ceil_div(n_slices, 2), kWarpsPerCta);
  const long long cap = (long long)sm_count() * (narrow_tma() ? 4 : narrow_minb());
  return (unsigned)(full < cap ? full : cap);
}

// pair kernel for wide slices too (PSELL_PAIR_WIDE=1, A/B; default: dual kernel)
static bool pair_wide() {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_PAIR_WIDE", v)) return v != 0;
  return false;
}

// threads per CTA of the one-warp-per-slice kernel (PSELL_NT overrides, A/B)
static int fast_nt() {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_NT", v) && (v == 64 || v == 128 || v == 256)) return v;
  return 256;
}

// ---- fast path: C == 32, warp == slice
template <int CODEC, typename XT, bool REF, bool DOT, int U>
__global__ void __launch_bounds__(kBlock) spmv_c32_kernel(const SpmvArgs a) {
  using W = typename WordOf<CODEC>::T;
  using A = Acc<XT, REF>;
  if constexpr (DOT) {
    if (a.skip && *a.skip) return;
  }
  const long long s = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long k = s >> 5;
  const int lane = threadIdx.x & 31;
  double dotv = 0.0;
  if (k < a.n_slices) {
    const long long o0 = a.offset[k];
    const int width = (int)((a.offset[k + 1] - o0) >> 5);
    const W* p = static_cast<const W*>(a.pack) + o0 + lane;
    const XT* __restrict__ x = static_cast<const XT*>(a.x);
    const uint64_t pol_s = policy_evict_first();
    const uint64_t pol_x = policy_evict_last();
    const int dbits = word_dbits<CODEC>(a.d);
    int cursor = (int)storage_base(a.row0 + s, a.se, a.k_left, a.n_cols);
    typename A::T acc = A::zero();
    W cur[U], nxt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = (u < width) ? ld_stream(p + u * 32, pol_s) : W(0);
    for (int q = 0; q < width; q += U) {
      const W* pn = p + (q + U) * 32;
#pragma unroll
      for (int u = 0; u < U; ++u) nxt[u] = (q + U + u < width) ? ld_stream(pn + u * 32, pol_s) : W(0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        cursor += (int)unpack_delta<W>(cur[u], dbits);
        const XT xv = ld_keep(x + cursor, pol_x);
        acc = A::template step<CODEC, W>(acc, cur[u], a.d, xv);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) cur[u] = nxt[u];
    }
    if (s < a.n_rows) {
      const long long o = out_row(a, s);
      const XT yv = A::out(acc);
      static_cast<XT*>(a.y)[o] = yv;
      if constexpr (DOT) dotv = (double)a.p_own[o] * (double)to_f<XT>(yv);
    }
  }
  finish_dot<DOT>(a, dotv);
}

// ---- fast production path (C == 32, FMA accumulation)
//
// Per word: flag predicate, cursor2 += w & mask (cursor2 = 2 * column, so for
// f16 x it is already the byte offset), one gather, one predicated FMA.  The
// fp16 codec with f16 x uses the sm_100 mixed-precision FMA (FHFMA: f16 x f16
// + f32), so neither the value nor x is converted.  Dummy and padding words
// only move the cursor (FMA predicated off).
template <typename XT>
__device__ __forceinline__ const char* xbyte(const XT* x, uint32_t c2) {
  return reinterpret_cast<const char*>(x) + (size_t)c2 * (sizeof(XT) / 2);
}

// Gathers predicated on the flag (GR = true): dummy and padding words issue no
// x load, they only move the cursor.  Used for irregular (segmented power-law)
// matrices, whose dummy gathers land on scattered L2 sectors: config 4
// 397 -> 367 us.  The stencils keep GR = false (their dummy gathers fall where
// the next real gather goes anyway, and the predicated asm loads schedule worse
// there: -10-15 %).
template <bool GR>
__device__ __forceinline__ unsigned short gather_u16(const void* p, uint32_t f) {
  unsigned short v;
  if (GR)
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %1, 0;\n mov.b16 %0, 0;\n @p ld.global.nc.u16 %0, [%2];\n}"
                 : "=h"(v) : "r"(f), "l"(p));
  else
    v = __ldg(reinterpret_cast<const unsigned short*>(p));
  return v;
}
template <bool GR>
__device__ __forceinline__ float gather_f32(const void* p, uint32_t f) {
  float v;
  if (GR)
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %1, 0;\n mov.b32 %0, 0;\n @p ld.global.nc.f32 %0, [%2];\n}"
                 : "=f"(v) : "r"(f), "l"(p));
  else
    v = __ldg(reinterpret_cast<const float*>(p));
  return v;
}

template <int CODEC, typename XT, bool GR = false> struct FastStep;

template <bool GR> struct FastStep<PSELL_FP16, __half, GR> {
  using Acc = float;
  __device__ static void run(uint32_t w, uint32_t& c2, const __half* x, float& acc, uint32_t, uint32_t) {
    const uint32_t f = w & 1u;
    c2 += w & (f ? 0xFFFEu : 0xFFFFFFFEu);
    const unsigned short xb = gather_u16<GR>(xbyte(x, c2), f);
    asm("{\n .reg .pred p;\n .reg .b16 lo, hi;\n setp.ne.b32 p, %1, 0;\n mov.b32 {lo, hi}, %2;\n"
        " @p fma.rn.f32.f16 %0, hi, %3, %0;\n}" : "+f"(acc) : "r"(f), "r"(w), "h"(xb));
  }
};
template <bool GR> struct FastStep<PSELL_FP16, float, GR> {
  using Acc = float;
  __device__ static void run(uint32_t w, uint32_t& c2, const float* x, float& acc, uint32_t, uint32_t) {
    const uint32_t f = w & 1u;
    c2 += w & (f ? 0xFFFEu : 0xFFFFFFFEu);
    const float xv = gather_f32<GR>(xbyte(x, c2), f);
    asm("{\n .reg .pred p;\n .reg .b16 lo, hi;\n .reg .f32 v;\n setp.ne.b32 p, %1, 0;\n mov.b32 {lo, hi}, %2;\n"
        " cvt.f32.f16 v, hi;\n @p fma.rn.f32 %0, v, %3, %0;\n}" : "+f"(acc) : "r"(f), "r"(w), "f"(xv));
  }
};
template <bool GR> struct FastStep<PSELL_E8MY, float, GR> {
  using Acc = float;
  // m_real = 2^(D+1) - 2 (delta field << 1), vmask = ~(2^(D+1) - 1) (value bits)
  __device__ static void run(uint32_t w, uint32_t& c2, const float* x, float& acc, uint32_t m_real,
                             uint32_t vmask) {
    const uint32_t f = w & 1u;
    c2 += w & (f ? m_real : 0xFFFFFFFEu);
#ifdef PSELL_DEBUG_NOGATHER  // measurement-only build: the word stream without the x gathers
    const float xv = __uint_as_float(c2 & 0x3F800000u);
#else
    const float xv = gather_f32<GR>(xbyte(x, c2), f);
#endif
    const float v = __uint_as_float(w & vmask);
    asm("{\n .reg .pred p;\n setp.ne.b32 p, %1, 0;\n @p fma.rn.f32 %0, %2, %3, %0;\n}"
        : "+f"(acc) : "r"(f), "f"(v), "f"(xv));
  }
};
template <bool GR> struct FastStep<PSELL_E8MY, __half, GR> {
  using Acc = float;
  __device__ static void run(uint32_t w, uint32_t& c2, const __half* x, float& acc, uint32_t m_real,
                             uint32_t vmask) {
    const uint32_t f = w & 1u;
    c2 += w & (f ? m_real : 0xFFFFFFFEu);
    const float xv = __half2float(__ushort_as_half(gather_u16<GR>(xbyte(x, c2), f)));
    const float v = __uint_as_float(w & vmask);
    asm("{\n .reg .pred p;\n setp.ne.b32 p, %1, 0;\n @p fma.rn.f32 %0, %2, %3, %0;\n}"
        : "+f"(acc) : "r"(f), "f"(v), "f"(xv));
  }
};

template <int CODEC, typename XT> struct FastPolicy {
  static constexpr bool kHave = false;
};
template <> struct FastPolicy<PSELL_FP16, __half> { static constexpr bool kHave = true; };
template <> struct FastPolicy<PSELL_FP16, float> { static constexpr bool kHave = true; };
template <> struct FastPolicy<PSELL_E8MY, float> { static constexpr bool kHave = true; };
template <> struct FastPolicy<PSELL_E8MY, __half> { static constexpr bool kHave = true; };

template <int CODEC, typename XT, bool DOT, int U, int NT = kBlock>
__global__ void __launch_bounds__(NT, 6 * kBlock / NT) spmv_fast_kernel(const SpmvArgs a) {
  using S = FastStep<CODEC, XT>;
  if constexpr (DOT) {
    if (a.skip && *a.skip) return;
  }
  const long long s = (long long)blockIdx.x * NT + threadIdx.x;
  const long long k = s >> 5;
  const int lane = threadIdx.x & 31;
  double dotv = 0.0;
  if (k < a.n_slices) {
    // (Hoisting the perm / p_own side loads to the kernel start was measured
    // slower: 404 vs 383 us on config 2 — the held registers cost more than
    // the hidden latency.)
    const long long o0 = a.offset[k];
    const int width = (int)((a.offset[k + 1] - o0) >> 5);
    if (a.seg_len > 0 && width > a.seg_len) goto done;  // long slice: segment kernels own it
    {
    const uint32_t* p = static_cast<const uint32_t*>(a.pack) + o0 + lane;
    const XT* __restrict__ x = static_cast<const XT*>(a.x);
    const uint32_t m_real = CODEC == PSELL_FP16 ? 0xFFFEu : ((2u << a.d) - 2u);
    const uint32_t vmask = CODEC == PSELL_FP16 ? 0u : ~((2u << a.d) - 1u);
    // 32-bit index math (rows and columns < 2^31 are checked at the ABI)
    const uint32_t sg = (uint32_t)(a.row0 + s);
    const uint32_t se = (uint32_t)a.se;
    const uint32_t blk = (sg / se) * se;
    const uint32_t kl = (uint32_t)a.k_left;
    const uint32_t cmax = a.n_cols > 0 ? (uint32_t)(a.n_cols - 1) : 0u;
    const uint32_t d0 = blk > kl ? blk - kl : 0u;
    uint32_t c2 = 2u * (d0 < cmax ? d0 : cmax);
    float acc = 0.f;
    uint32_t cur[U], nxt[U];
    int q = 0;
    if (width >= U) {
#pragma unroll
      for (int u = 0; u < U; ++u) cur[u] = __ldcs(p + u * 32);
      // full chunks with the next full chunk in flight
      for (; q + 2 * U <= width; q += U) {
#pragma unroll
        for (int u = 0; u < U; ++u) nxt[u] = __ldcs(p + (q + U + u) * 32);
#pragma unroll
        for (int u = 0; u < U; ++u) S::run(cur[u], c2, x, acc, m_real, vmask);
#pragma unroll
        for (int u = 0; u < U; ++u) cur[u] = nxt[u];
      }
      // last full chunk, with the (partial) tail chunk in flight
      const int rem = width - (q + U);
#pragma unroll
      for (int u = 0; u < U; ++u) nxt[u] = (u < rem) ? __ldcs(p + (q + U + u) * 32) : 0u;
#pragma unroll
      for (int u = 0; u < U; ++u) S::run(cur[u], c2, x, acc, m_real, vmask);
      q += U;
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) nxt[u] = (u < width) ? __ldcs(p + u * 32) : 0u;
    }
    if (q < width) {
      // tail of r < U steps, processed in groups of 4 / 2 / 1 (U == 8)
      int r = width - q;
      static_assert(U == 8, "tail decomposition assumes U == 8");
      if (r >= 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) S::run(nxt[u], c2, x, acc, m_real, vmask);
#pragma unroll
        for (int u = 0; u < 4; ++u) nxt[u] = nxt[u + 4];
        r -= 4;
      }
      if (r >= 2) {
        S::run(nxt[0], c2, x, acc, m_real, vmask);
        S::run(nxt[1], c2, x, acc, m_real, vmask);
        nxt[0] = nxt[2];
        r -= 2;
      }
      if (r >= 1) S::run(nxt[0], c2, x, acc, m_real, vmask);
    }
    if (s < a.n_rows) {
      uint32_t o = (uint32_t)s;
      if (a.mode == PSELL_MODE_IMPLICIT) {
        const uint32_t sig = (uint32_t)a.sigma;
        const uint32_t p8 = a.perm_bytes == 1 ? (uint32_t)static_cast<const uint8_t*>(a.perm)[s]
                                              : (uint32_t)static_cast<const uint16_t*>(a.perm)[s];
        o = ((uint32_t)s / sig) * sig + p8;
      }
      XT yv;
      if constexpr (sizeof(XT) == 2) yv = __float2half_rn(acc);
      else yv = acc;
      static_cast<XT*>(a.y)[o] = yv;
      if constexpr (DOT) dotv = (double)a.p_own[o] * (double)to_f<XT>(yv);
    }
    }
  }
done:
  finish_dot<DOT, NT>(a, dotv);
}

// ---- dual-slice kernel (C == 32): a warp runs slices 2w and 2w+1 in lockstep
// chunks, so the two per-slice latency chains (offset -> words -> x -> y)
// overlap inside one warp.  Aimed at narrow slices (7-point rows: ~9 steps),
// where one slice per warp leaves the chain exposed.
// SM-affine persistent scheduling (AFF, irregular matrices): the slice pairs are
// cut into one contiguous chunk per SM; the warps resident on SM j claim pairs
// of chunk j (per-chunk atomic counter), then steal from the following chunks.
// Consecutive slices are neighbouring rows of the same sigma-block, so the x
// columns one SM gathers stay within a narrow window and hit its L1 instead of
// each gather crossing to L2 (block-linear CTA order puts slices 2368 apart on
// one SM).  sched[0..nchunk) claim counters, sched[nchunk] exit count; the last
// warp to leave resets them for the next launch (no memset node).
__device__ __forceinline__ uint32_t smid_u32() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

struct AffSched {
  uint32_t owner, tried;
};

// next slice pair for this warp, or ~0u when every chunk is exhausted (warp-uniform)
__device__ __forceinline__ uint32_t aff_next(const SpmvArgs& a, AffSched& st, uint32_t npairs) {
  const uint32_t nc = (uint32_t)a.aff_chunks;
  uint32_t pair = ~0u;
  if ((threadIdx.x & 31) == 0) {
    while (st.tried < nc) {
      const uint32_t o = st.owner;
      const uint32_t lo = (uint32_t)(((unsigned long long)npairs * o) / nc);
      const uint32_t hi = (uint32_t)(((unsigned long long)npairs * (o + 1)) / nc);
      // cheap read first: exhausted chunks cost no atomic once seen
      if (*reinterpret_cast<volatile uint32_t*>(a.sched + o) < hi - lo) {
        const uint32_t t = atomicAdd(a.sched + o, 1u);
        if (t < hi - lo) {
          pair = lo + t;
          break;
        }
      }
      st.owner = st.owner + 1 == nc ? 0 : st.owner + 1;
      ++st.tried;
    }
  }
  return __shfl_sync(0xffffffffu, pair, 0);
}

__device__ __forceinline__ void aff_exit(const SpmvArgs& a) {
  if ((threadIdx.x & 31) == 0) {
    const uint32_t nw = gridDim.x * (blockDim.x >> 5);
    const uint32_t nc = (uint32_t)a.aff_chunks;
    if (atomicAdd(a.sched + nc, 1u) == nw - 1) {
      for (uint32_t i = 0; i <= nc; ++i) a.sched[i] = 0u;
      __threadfence();
    }
  }
}

// the dual kernel's body for CTA `bid` of its grid (spmv_dual_seg_kernel runs it from a
// merged grid whose first CTAs take the long-slice segments)
template <int CODEC, typename XT, bool DOT, int U, bool GR = false, bool AFF = false, bool STATIC = false,
          int NT = kBlock>
__device__ __forceinline__ void dual_body(const SpmvArgs& a, unsigned bid) {
  using S = FastStep<CODEC, XT, GR>;
  if constexpr (DOT) {
    if (a.skip && *a.skip) return;
  }
  const int lane = threadIdx.x & 31;
  double dotv = 0.0;
  const uint32_t npairs = (uint32_t)((a.n_slices + 1) >> 1);
  AffSched sched{AFF ? smid_u32() % (uint32_t)a.aff_chunks : 0u, 0u};
  // STATIC: this CTA walks the contiguous, word-balanced pair range [pb, pe) of the ranges
  // table behind the SM-affine counters (sched[aff_chunks + 1 ...]), its warps interleaved
  long long st_pe = 0;
  long long wg;
  if constexpr (STATIC) {
    // the table holds 2 x aff_chunks word-balanced chunks: a 1024-thread CTA (one per SM) takes
    // chunks 2b, 2b+1; with 768-thread CTAs (two per SM, CTA b and b + G sharing an SM when
    // the grid is dispatched round robin) CTA b < G takes chunk 2b and CTA b + G chunk 2b + 1
    const uint32_t* rg = a.sched + a.aff_chunks + 1;
    const unsigned G = (unsigned)a.aff_chunks;
    const unsigned c0 = NT == 1024 ? 2u * bid : (bid < G ? 2u * bid : 2u * (bid - G) + 1u);
    const unsigned c1 = NT == 1024 ? c0 + 2u : c0 + 1u;
    st_pe = rg[c1];
    wg = (long long)rg[c0] + (threadIdx.x >> 5);
  } else {
    wg = AFF ? (long long)aff_next(a, sched, npairs) : ((long long)bid * NT + threadIdx.x) >> 5;
  }
  for (; STATIC ? wg < st_pe : (!AFF || wg != (long long)~0u);
       wg = STATIC ? wg + NT / 32 : AFF ? (long long)aff_next(a, sched, npairs) : (long long)~0u) {
  const long long kA = 2 * wg, kB = kA + 1;
  if (kA < a.n_slices) {
    const bool hasB = kB < a.n_slices;
    const long long oA = a.offset[kA], oB = a.offset[kA + 1];
    const long long oE = hasB ? a.offset[kB + 1] : oB;
    // long slices (power-law rows) belong to the segment kernels when segmentation is on
    const bool skipA = a.seg_len > 0 && (int)((oB - oA) >> 5) > a.seg_len;
    const bool skipB = a.seg_len > 0 && (int)((oE - oB) >> 5) > a.seg_len;
    const int wA = skipA ? 0 : (int)((oB - oA) >> 5), wB = skipB ? 0 : (int)((oE - oB) >> 5);
    const uint32_t* pA = static_cast<const uint32_t*>(a.pack) + oA + lane;
    const uint32_t* pB = static_cast<const uint32_t*>(a.pack) + oB + lane;
    if (a.l2pf && lane == 0 && oE > oA) {
      const uint64_t bytes = (uint64_t)(oE - oA) * 4u;
      l2_prefetch_bulk(static_cast<const uint32_t*>(a.pack) + oA, (uint32_t)(bytes < (1u << 20) ? bytes : (1u << 20)),
                       policy_evict_first());
    }
    const XT* __restrict__ x = static_cast<const XT*>(a.x);
    const uint32_t m_real = CODEC == PSELL_FP16 ? 0xFFFEu : ((2u << a.d) - 2u);
    const uint32_t vmask = CODEC == PSELL_FP16 ? 0u : ~((2u << a.d) - 1u);
    const uint32_t se = (uint32_t)a.se, kl = (uint32_t)a.k_left;
    const uint32_t cmax = a.n_cols > 0 ? (uint32_t)(a.n_cols - 1) : 0u;
    // The fp16 x f16 instantiation (config 2) measured slower with each of the
    // e8mY tunings below (multiply-high base division 324 -> 326 us, last-chunk
    // split 324 -> 328 us, unpredicated full chunks 324 -> 328 us) and keeps the
    // plain forms; e8mY / f32 x (config 3) takes all three (364 -> 351 us).
    constexpr bool kTuned = !(CODEC == PSELL_FP16 && sizeof(XT) == 2);
    auto base2 = [&](long long k) -> uint32_t {
      const uint32_t g = (uint32_t)a.row0 + (uint32_t)(k * 32) + lane;
      const uint32_t blk = !kTuned ? (g / se) * se : se == 1 ? g : fast_div(g, a.se_m, a.se_l) * se;
      const uint32_t d = blk > kl ? blk - kl : 0u;
      return 2u * (d < cmax ? d : cmax);
    };
    uint32_t cA = base2(kA), cB = base2(kB);
    float accA = 0.f, accB = 0.f;
    const int wmax = wA > wB ? wA : wB;
    // kTuned: all chunks but the last in the loop; the last one (<= U steps) after
    // it, decoding its last quarter only when some slice reaches it
    constexpr bool kTail2 = kTuned;
    const int qlast = wmax > 0 ? ((wmax - 1) / U) * U : 0;
    for (int q = 0; q < (kTail2 ? qlast : wmax); q += U) {
      uint32_t a8[U], b8[U];
#ifndef PSELL_DUAL_NOFULL
      // kTuned: full chunk of both slices with no per-word predicates
      if (kTuned && q + U <= wA && q + U <= wB) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          a8[u] = __ldcs(pA + (q + u) * 32);
          b8[u] = __ldcs(pB + (q + u) * 32);
        }
      } else
#endif
      {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          a8[u] = (q + u < wA) ? __ldcs(pA + (q + u) * 32) : 0u;
          b8[u] = (q + u < wB) ? __ldcs(pB + (q + u) * 32) : 0u;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        S::run(a8[u], cA, x, accA, m_real, vmask);
        S::run(b8[u], cB, x, accB, m_real, vmask);
      }
    }
    if (kTail2 && wmax > 0) {
      const int q = qlast;
      uint32_t a8[U], b8[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a8[u] = (q + u < wA) ? __ldcs(pA + (q + u) * 32) : 0u;
        b8[u] = (q + u < wB) ? __ldcs(pB + (q + u) * 32) : 0u;
      }
      constexpr int K = 3 * U / 4;
#pragma unroll
      for (int u = 0; u < K; ++u) {
        S::run(a8[u], cA, x, accA, m_real, vmask);
        S::run(b8[u], cB, x, accB, m_real, vmask);
      }
      if (q + K < wmax) {
#pragma unroll
        for (int u = K; u < U; ++u) {
          S::run(a8[u], cA, x, accA, m_real, vmask);
          S::run(b8[u], cB, x, accB, m_real, vmask);
        }
      }
    }
    const uint32_t sig = (uint32_t)a.sigma;
    // output rows: branch-free clamped perm loads, multiply-high division
    const uint32_t nr = (uint32_t)a.n_rows;
    auto out_row = [&](long long k) -> uint32_t {
      const uint32_t s = (uint32_t)(k * 32) + lane;
      if (a.mode != PSELL_MODE_IMPLICIT) return s;
      const uint32_t sc = s < nr ? s : nr - 1u;
      const uint32_t pp = a.perm_bytes == 1 ? (uint32_t)__ldg(static_cast<const uint8_t*>(a.perm) + sc)
                                            : (uint32_t)__ldg(static_cast<const uint16_t*>(a.perm) + sc);
      return fast_div((uint32_t)(k * 32), a.sig_m, a.sig_l) * sig + pp;
    };
    auto flush = [&](long long k, float acc) {
      const uint32_t s = (uint32_t)(k * 32) + lane;
      const uint32_t o = out_row(k);
      if ((long long)s < a.n_rows) {
        XT yv;
        if constexpr (sizeof(XT) == 2) yv = __float2half_rn(acc);
        else yv = acc;
        static_cast<XT*>(a.y)[o] = yv;
        if constexpr (DOT) dotv += (double)a.p_own[o] * (double)to_f<XT>(yv);
      }
    };
    if (!skipA) flush(kA, accA);
    if (hasB && !skipB) flush(kB, accB);
  }
  if (!AFF && !STATIC) break;
  }
  if constexpr (AFF) aff_exit(a);
  finish_dot<DOT, NT>(a, dotv);
}

// Static SM-affine kernel (segmented matrices, the default): one 1024-thread CTA per SM, each
// running its share of the long slices' segments and then one contiguous, word-balanced range
// of short-slice pairs -- about a sigma window of rows per SM, whose x gathers then hit the
// SM's L1 (the SM-affine claim scheduler, PSELL_AFF=1, got the locality but paid per-pair
// atomics) -- so one launch covers segments and short slices, then the combine
template <int CODEC, typename XT, int U>
__device__ __forceinline__ void seg_one(const SpmvArgs& a, long long sg);

template <int CODEC, typename XT, int U, int NT = 1024>
__global__ void __launch_bounds__(NT, NT == 1024 ? 1 : 2) spmv_dual_static_kernel(const SpmvArgs a, long long n_seg) {
  // this CTA's share of the long slices' segments first (the same per-warp code as
  // spmv_seg_kernel), then its contiguous range of short-slice pairs
  const long long s0 = n_seg * blockIdx.x / gridDim.x, s1 = n_seg * (blockIdx.x + 1) / gridDim.x;
  for (long long sg = s0 + (threadIdx.x >> 5); sg < s1; sg += NT / 32) seg_one<CODEC, XT, U>(a, sg);
  dual_body<CODEC, XT, false, U, true, false, true, NT>(a, blockIdx.x);
}

// PSELL_DSTATIC_NT=768: two 768-thread CTAs per SM (A/B; config 4b 323 vs 257 us -- the two
// CTAs an SM receives do not get adjacent chunks, so each SM holds two x windows)
static int dual_static_nt() {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_DSTATIC_NT", v) && v == 768) return 768;
  return 1024;
}

template <int CODEC, typename XT, bool DOT, int U, bool GR = false, bool AFF = false>
#ifndef PSELL_DUAL_MINB
#define PSELL_DUAL_MINB 6
#endif
__global__ void __launch_bounds__(kBlock, PSELL_DUAL_MINB) spmv_dual_kernel(const SpmvArgs a) {
  dual_body<CODEC, XT, DOT, U, GR, AFF>(a, blockIdx.x);
}

// ---- pair kernel (C == 32): a warp runs slices 2w and 2w+1.  Full U-step
// chunks run in lockstep with unpredicated loads; the tails (< U steps) load
// with one predicate per word from a fixed base (immediate offsets).  Base offsets and output rows use multiply-high
// division by sigma; the perm bytes are loaded before the word stream so
// their latency hides under it.
template <int CODEC, typename XT, bool DOT, int U, bool HOIST, int NT = kBlock, bool PERSIST = false>
__global__ void __launch_bounds__(NT, PSELL_PAIR_MINB * kBlock / NT) spmv_pair_kernel(const SpmvArgs a) {
    using S = FastStep<CODEC, XT>;
  if constexpr (DOT) {
    if (a.skip && *a.skip) return;
  }
  const uint32_t wg0 = (uint32_t)((blockIdx.x * (unsigned)NT + threadIdx.x) >> 5);
  const uint32_t wstride = gridDim.x * (unsigned)(NT / 32);  // PERSIST: grid-stride over slice pairs
  const int lane = threadIdx.x & 31;
  const uint32_t ns = (uint32_t)a.n_slices;
  double dotv = 0.0;
  for (uint32_t wg = wg0; 2u * wg < ns; wg += wstride) {
    const uint32_t kA = 2u * wg, kB = kA + 1u;
    const bool hasB = kB < ns;
    const uint32_t n_rows = (uint32_t)a.n_rows;
    const uint32_t sA = kA * 32u + lane, sB = sA + 32u;
    // output rows; with HOIST (narrow slices) the perm bytes load before the
    // word stream so their latency hides under it (wide slices: at the end,
    // where the registers are free)
    const bool impl = a.mode == PSELL_MODE_IMPLICIT;
    auto out_of = [&](uint32_t k, uint32_t s) -> uint32_t {
      if (!impl) return s;
      const uint32_t blk = fast_div(k * 32u, a.sig_m, a.sig_l) * (uint32_t)a.sigma;
      // rows past n_rows (last slice) read the last valid perm entry and are never
      // stored: no divergent branch around the load (7-point 152.7 -> 145.6 us)
      const uint32_t sc = s < n_rows ? s : n_rows - 1u;
      const uint32_t pp = a.perm_bytes == 1 ? (uint32_t)__ldg(static_cast<const uint8_t*>(a.perm) + sc)
                                            : (uint32_t)__ldg(static_cast<const uint16_t*>(a.perm) + sc);
      return blk + pp;
    };
    uint32_t oA = sA, oB = sB;
#ifndef PSELL_PAIR_PERM_EARLY
    // HOIST: the perm bytes are issued here but added into the output rows only at the
    // flush (the add right after the load stalled the warp for the load's full latency
    // before its word stream: the hottest stall of this kernel in ncu)
    uint32_t ppA = 0u, ppB = 0u;
    if constexpr (HOIST) {
      if (impl) {
        const uint32_t scA = sA < n_rows ? sA : n_rows - 1u, scB = sB < n_rows ? sB : n_rows - 1u;
        ppA = a.perm_bytes == 1 ? (uint32_t)__ldg(static_cast<const uint8_t*>(a.perm) + scA)
                                : (uint32_t)__ldg(static_cast<const uint16_t*>(a.perm) + scA);
        ppB = a.perm_bytes == 1 ? (uint32_t)__ldg(static_cast<const uint8_t*>(a.perm) + scB)
                                : (uint32_t)__ldg(static_cast<const uint16_t*>(a.perm) + scB);
      }
    }
#else
    if constexpr (HOIST) {
      oA = out_of(kA, sA);
      oB = out_of(kB, sB);
    }
#endif
    const long long o0 = a.offset[kA], o1 = a.offset[kA + 1];
    const long long o2 = hasB ? a.offset[kA + 2] : o1;
    const bool skipA = a.seg_len > 0 && (int)((o1 - o0) >> 5) > a.seg_len;  // segment kernels own it
    const bool skipB = a.seg_len > 0 && (int)((o2 - o1) >> 5) > a.seg_len;
    const int wA = skipA ? 0 : (int)((o1 - o0) >> 5), wB = skipB ? 0 : (int)((o2 - o1) >> 5);
    const uint32_t* pA = static_cast<const uint32_t*>(a.pack) + o0 + lane;
    const uint32_t* pB = static_cast<const uint32_t*>(a.pack) + o1 + lane;
    if (!PERSIST && a.l2pf && lane == 0 && o2 > o0) {  // this pair's words, one TMA request
      const uint64_t bytes = (uint64_t)(o2 - o0) * 4u;
      l2_prefetch_bulk(static_cast<const uint32_t*>(a.pack) + o0, (uint32_t)(bytes < (1u << 20) ? bytes : (1u << 20)),
                       policy_evict_first());
    }
    const XT* __restrict__ x = static_cast<const XT*>(a.x);
    const uint32_t m_real = CODEC == PSELL_FP16 ? 0xFFFEu : ((2u << a.d) - 2u);
    const uint32_t vmask = CODEC == PSELL_FP16 ? 0u : ~((2u << a.d) - 1u);
    const uint32_t kl = (uint32_t)a.k_left;
    const uint32_t cmax = a.n_cols > 0 ? (uint32_t)(a.n_cols - 1) : 0u;
    auto base2 = [&](uint32_t k) -> uint32_t {
      const uint32_t g = (uint32_t)a.row0 + k * 32u + lane;
      const uint32_t blk = a.se == 1 ? g : fast_div(g, a.se_m, a.se_l) * (uint32_t)a.se;
      const uint32_t d = blk > kl ? blk - kl : 0u;
      return 2u * (d < cmax ? d : cmax);
    };
    uint32_t cA = base2(kA), cB = base2(kB);
    float accA = 0.f, accB = 0.f;
    uint32_t wa[U], wb[U];
    const int both = (wA < wB ? wA : wB) / U;
    int q = 0;
    for (int c = 0; c < both; ++c, q += U) {  // lockstep full chunks
#pragma unroll
      for (int u = 0; u < U; ++u) {
        wa[u] = __ldcs(pA + (q + u) * 32);
        wb[u] = __ldcs(pB + (q + u) * 32);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        S::run(wa[u], cA, x, accA, m_real, vmask);
        S::run(wb[u], cB, x, accB, m_real, vmask);
      }
    }
    int qa = q, qb = q;
    for (; qa + U <= wA; qa += U) {  // the longer slice's remaining full chunks
#pragma unroll
      for (int u = 0; u < U; ++u) wa[u] = __ldcs(pA + (qa + u) * 32);
#pragma unroll
      for (int u = 0; u < U; ++u) S::run(wa[u], cA, x, accA, m_real, vmask);
    }
    for (; qb + U <= wB; qb += U) {
#pragma unroll
      for (int u = 0; u < U; ++u) wb[u] = __ldcs(pB + (qb + u) * 32);
#pragma unroll
      for (int u = 0; u < U; ++u) S::run(wb[u], cB, x, accB, m_real, vmask);
    }
    // tails (< U steps): predicated loads from a fixed base, branch-free decode
    // (zero words past the width only move nothing: delta 0, FMA predicated off),
    // A and B interleaved so all gathers issue before the first FMA waits
    const int ra = wA - qa, rb = wB - qb;
    if (ra > 0 || rb > 0) {
      const uint32_t* tA = pA + qa * 32;
      const uint32_t* tB = pB + qb * 32;
#ifndef PSELL_PAIR_NOFULLK
      if (ra >= PairK<U>::K && rb >= PairK<U>::K) {  // both reach 3U/4 steps: those loads unpredicated (fused dot 162 -> 160 us)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          wa[u] = (u < PairK<U>::K || u < ra) ? __ldcs(tA + u * 32) : 0u;
          wb[u] = (u < PairK<U>::K || u < rb) ? __ldcs(tB + u * 32) : 0u;
        }
      } else
#endif
      {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          wa[u] = u < ra ? __ldcs(tA + u * 32) : 0u;
          wb[u] = u < rb ? __ldcs(tB + u * 32) : 0u;
        }
      }
#ifndef PSELL_PAIR_NOTAILSPLIT
      // decode the first 3U/4 steps unconditionally and the rest only when a
      // slice reaches them (7-point slices: 9 of 12 steps; 161 -> 153 us)
      constexpr int K = PairK<U>::K;
#pragma unroll
      for (int u = 0; u < K; ++u) {
        S::run(wa[u], cA, x, accA, m_real, vmask);
        S::run(wb[u], cB, x, accB, m_real, vmask);
      }
      if (ra > K || rb > K) {
#pragma unroll
        for (int u = K; u < U; ++u) {
          S::run(wa[u], cA, x, accA, m_real, vmask);
          S::run(wb[u], cB, x, accB, m_real, vmask);
        }
      }
#else
#pragma unroll
      for (int u = 0; u < U; ++u) {
        S::run(wa[u], cA, x, accA, m_real, vmask);
        S::run(wb[u], cB, x, accB, m_real, vmask);
      }
#endif
    }
    auto flush = [&](uint32_t s, uint32_t o, float acc) {
      if (s < n_rows) {
        XT yv;
        if constexpr (sizeof(XT) == 2) yv = __float2half_rn(acc);
        else yv = acc;
        static_cast<XT*>(a.y)[o] = yv;
        if constexpr (DOT) dotv += (double)a.p_own[o] * (double)to_f<XT>(yv);
      }
    };
    if constexpr (!HOIST) {
      oA = out_of(kA, sA);
      oB = out_of(kB, sB);
    }
#ifndef PSELL_PAIR_PERM_EARLY
    if constexpr (HOIST) {
      if (impl) {
        oA = fast_div(kA * 32u, a.sig_m, a.sig_l) * (uint32_t)a.sigma + ppA;
        oB = fast_div(kB * 32u, a.sig_m, a.sig_l) * (uint32_t)a.sigma + ppB;
      }
    }
#endif
    if (!skipA) flush(sA, oA, accA);
    if (hasB && !skipB) flush(sB, oB, accB);
    if (!PERSIST) break;
  }
  finish_dot<DOT, NT>(a, dotv);
}

// ---- narrow kernel (C == 32, every slice <= 12 steps, no segmentation: 7-point rows,
// the PCG inner operator).  The pair kernel's slice pairing and FMA order (outputs are
// bitwise equal to it), with the per-pair bookkeeping cut to what such slices need
// (71.7 M instead of 94.6 M warp instructions on 7-point 256^3 e8m14, ncu) and the
// memory round trips of a pair taken off its critical path:
//  * the next pair's offsets and perm bytes load while this pair runs (software
//    pipelined, no select on a loaded value: a select on the prefetched offset stalled
//    on it and made the prefetch synchronous -- 12 % of the stall samples, 145.5 -> 137.3 us);
//  * decode runs in two passes (cursor prefix and gathers, then the FMAs), so ptxas
//    issues the gathers of a pair in ~3 batches instead of one per few words;
//  * the p_own load of the fused dot issues between the gather and FMA passes;
//  * perm width, mode and the tail split are compile-time; offsets in 32-bit arithmetic.
// Steps [0, K) are decoded for every pair, [K, 12) only when a slice reaches them.
// 4 CTAs x 8 warps per SM (64 registers, no spills; PSELL_NARROW_MINB=5: 48 registers).
// Measured and dropped (profiles/r02/narrow_ab*.txt): the next pair's words in registers
// (3 CTAs/SM, 140.2 us, fused dot 159.7 us), a bulk L2 prefetch of the next pair
// (147.9 us), a __syncwarp fence forcing every gather before the first FMA (ptxas then
// parks the flag predicates in a register: 144.2 us), a 64-bit byte-pointer cursor
// (ptxas splits the mad.wide into LEA + LEA.HI.X: 168.8 us), 6 CTAs/SM (spills).
#ifndef PSELL_NARROW_K
#define PSELL_NARROW_K 9
#endif

// cursor step (c2 = 2 * column), the flag test fused into the AND (LOP3 with a predicate
// output): the C form of this loses the fusion once the flag is tested again in the FMA pass
__device__ __forceinline__ void narrow_cursor(uint32_t w, uint32_t& c2, uint32_t m_real) {
  asm("{\n .reg .pred p;\n .reg .b32 t, m;\n and.b32 t, %1, 1;\n setp.ne.b32 p, t, 0;\n"
      " selp.b32 m, %2, 0xFFFFFFFE, p;\n and.b32 t, %1, m;\n add.u32 %0, %0, t;\n}"
      : "+r"(c2) : "r"(w), "r"(m_real));
}
template <int CODEC, typename XT> struct NarrowStep;
template <> struct NarrowStep<PSELL_E8MY, float> {
  __device__ static uint32_t gather(uint32_t w, uint32_t& c2, const float* x, uint32_t m_real) {
    narrow_cursor(w, c2, m_real);
    return __float_as_uint(__ldg(reinterpret_cast<const float*>(xbyte(x, c2))));
  }
  __device__ static void fma(uint32_t w, uint32_t xr, float& acc, uint32_t vmask) {
    asm("{\n .reg .pred p;\n setp.ne.b32 p, %1, 0;\n @p fma.rn.f32 %0, %2, %3, %0;\n}"
        : "+f"(acc) : "r"(w & 1u), "f"(__uint_as_float(w & vmask)), "f"(__uint_as_float(xr)));
  }
};
template <> struct NarrowStep<PSELL_E8MY, __half> {
  __device__ static uint32_t gather(uint32_t w, uint32_t& c2, const __half* x, uint32_t m_real) {
    narrow_cursor(w, c2, m_real);
    return (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(xbyte(x, c2)));
  }
  __device__ static void fma(uint32_t w, uint32_t xr, float& acc, uint32_t vmask) {
    const float xv = __half2float(__ushort_as_half((unsigned short)xr));
    asm("{\n .reg .pred p;\n setp.ne.b32 p, %1, 0;\n @p fma.rn.f32 %0, %2, %3, %0;\n}"
        : "+f"(acc) : "r"(w & 1u), "f"(__uint_as_float(w & vmask)), "f"(xv));
  }
};
template <> struct NarrowStep<PSELL_FP16, __half> {
  __device__ static uint32_t gather(uint32_t w, uint32_t& c2, const __half* x, uint32_t) {
    narrow_cursor(w, c2, 0xFFFEu);
    return (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(xbyte(x, c2)));
  }
  __device__ static void fma(uint32_t w, uint32_t xr, float& acc, uint32_t) {
    asm("{\n .reg .pred p;\n .reg .b16 lo, hi;\n setp.ne.b32 p, %1, 0;\n mov.b32 {lo, hi}, %2;\n"
        " @p fma.rn.f32.f16 %0, hi, %3, %0;\n}" : "+f"(acc) : "r"(w & 1u), "r"(w), "h"((unsigned short)xr));
  }
};
template <> struct NarrowStep<PSELL_FP16, float> {
  __device__ static uint32_t gather(uint32_t w, uint32_t& c2, const float* x, uint32_t) {
    narrow_cursor(w, c2, 0xFFFEu);
    return __float_as_uint(__ldg(reinterpret_cast<const float*>(xbyte(x, c2))));
  }
  __device__ static void fma(uint32_t w, uint32_t xr, float& acc, uint32_t) {
    asm("{\n .reg .pred p;\n .reg .b16 lo, hi;\n .reg .f32 v;\n setp.ne.b32 p, %1, 0;\n mov.b32 {lo, hi}, %2;\n"
        " cvt.f32.f16 v, hi;\n @p fma.rn.f32 %0, v, %3, %0;\n}"
        : "+f"(acc) : "r"(w & 1u), "r"(w), "f"(__uint_as_float(xr)));
  }
};

template <int CODEC, typename XT, bool DOT, int PB, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) spmv_narrow_kernel(const SpmvArgs a) {
  using S = NarrowStep<CODEC, XT>;
  constexpr int U = 12, K = PSELL_NARROW_K;
  if constexpr (DOT) {
    if (a.skip && *a.skip) return;
  }
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t ns = (uint32_t)a.n_slices, np = (ns + 1u) >> 1;
  const uint32_t n_rows = (uint32_t)a.n_rows;
  const uint32_t wstride = gridDim.x * (unsigned)kWarpsPerCta;
  const XT* __restrict__ x = static_cast<const XT*>(a.x);
  const uint32_t* __restrict__ pack = static_cast<const uint32_t*>(a.pack);
  const int64_t* __restrict__ off = a.offset;
  const uint32_t m_real = CODEC == PSELL_FP16 ? 0xFFFEu : ((2u << a.d) - 2u);
  const uint32_t vmask = CODEC == PSELL_FP16 ? 0u : ~((2u << a.d) - 1u);
  const uint32_t kl = (uint32_t)a.k_left, row0 = (uint32_t)a.row0, se = (uint32_t)a.se;
  const uint32_t cmax = a.n_cols > 0 ? (uint32_t)(a.n_cols - 1) : 0u;
  auto perm_of = [&](uint32_t s) -> uint32_t {
    const uint32_t sc = s < n_rows ? s : n_rows - 1u;  // rows past n_rows are never stored
    if constexpr (PB == 1) return (uint32_t)__ldg(static_cast<const uint8_t*>(a.perm) + sc);
    else return (uint32_t)__ldg(static_cast<const uint16_t*>(a.perm) + sc);
  };
  double dotv = 0.0;
  uint32_t wg = (blockIdx.x * (unsigned)kBlock + threadIdx.x) >> 5;
  // pipelined per-pair metadata: offsets (o0 64-bit, o1 / o2 low words) and perm bytes
  long long n_o0 = 0;
  uint32_t n_o1 = 0u, n_o2 = 0u, n_ppA = 0u, n_ppB = 0u;
  auto fetch = [&](uint32_t g) {
    if (g < np) {
      const uint32_t k = 2u * g;
      // no select on a loaded value: a lone last slice reads off[ns] == off[k + 1]
      // (the select waited for the load, which made this prefetch synchronous)
      n_o0 = __ldg(off + k);
      n_o1 = (uint32_t)__ldg(off + k + 1);
      n_o2 = (uint32_t)__ldg(off + (k + 2u < ns ? k + 2u : ns));
      if constexpr (PB != 0) {
        n_ppA = perm_of(k * 32u + lane);
        n_ppB = perm_of(k * 32u + 32u + lane);
      }
    }
  };
  fetch(wg);
  for (; wg < np; wg += wstride) {
    const uint32_t kA = 2u * wg;
    const bool hasB = kA + 1u < ns;
    const long long o0 = n_o0;
    const uint32_t wA = (n_o1 - (uint32_t)o0) >> 5, wB = (n_o2 - n_o1) >> 5;
    const uint32_t ppA = n_ppA, ppB = n_ppB;
    fetch(wg + wstride);
    const uint32_t* pA = pack + o0 + lane;
    const uint32_t* pB = pA + wA * 32u;
    auto base2 = [&](uint32_t k) -> uint32_t {
      const uint32_t g = row0 + k * 32u + lane;
      const uint32_t blk = se == 1u ? g : fast_div(g, a.se_m, a.se_l) * se;
      const uint32_t d = blk > kl ? blk - kl : 0u;
      return 2u * (d < cmax ? d : cmax);
    };
    uint32_t cA = base2(kA), cB = base2(kA + 1u);
    uint32_t wa[U], wb[U], xa[U], xb[U];
    if (wA >= (uint32_t)K && wB >= (uint32_t)K) {
#pragma unroll
      for (int u = 0; u < K; ++u) {
        wa[u] = __ldcs(pA + u * 32);
        wb[u] = __ldcs(pB + u * 32);
      }
    } else {
#pragma unroll
      for (int u = 0; u < K; ++u) {
        wa[u] = (uint32_t)u < wA ? __ldcs(pA + u * 32) : 0u;
        wb[u] = (uint32_t)u < wB ? __ldcs(pB + u * 32) : 0u;
      }
    }
#pragma unroll
    for (int u = 0; u < K; ++u) {
      xa[u] = S::gather(wa[u], cA, x, m_real);
      xb[u] = S::gather(wb[u], cB, x, m_real);
    }
    const uint32_t sA = kA * 32u + lane, sB = sA + 32u;
    uint32_t oA = sA, oB = sB;
    if constexpr (PB != 0) {
      oA = fast_div(kA * 32u, a.sig_m, a.sig_l) * (uint32_t)a.sigma + ppA;
      oB = fast_div(kA * 32u + 32u, a.sig_m, a.sig_l) * (uint32_t)a.sigma + ppB;
    }
    const bool stA = sA < n_rows, stB = hasB && sB < n_rows;
    float pvA = 0.f, pvB = 0.f;
    if constexpr (DOT) {  // in flight under the FMA pass
      if (stA) pvA = __ldg(a.p_own + oA);
      if (stB) pvB = __ldg(a.p_own + oB);
    }
    float accA = 0.f, accB = 0.f;
#pragma unroll
    for (int u = 0; u < K; ++u) {
      S::fma(wa[u], xa[u], accA, vmask);
      S::fma(wb[u], xb[u], accB, vmask);
    }
    // steps [K, 12): rare (boundary slices), after the main pass so they hold no
    // registers across it
    if (wA > (uint32_t)K || wB > (uint32_t)K) {
#pragma unroll
      for (int u = K; u < U; ++u) {
        wa[u] = (uint32_t)u < wA ? __ldcs(pA + u * 32) : 0u;
        wb[u] = (uint32_t)u < wB ? __ldcs(pB + u * 32) : 0u;
      }
#pragma unroll
      for (int u = K; u < U; ++u) {
        xa[u] = S::gather(wa[u], cA, x, m_real);
        xb[u] = S::gather(wb[u], cB, x, m_real);
      }
#pragma unroll
      for (int u = K; u < U; ++u) {
        S::fma(wa[u], xa[u], accA, vmask);
        S::fma(wb[u], xb[u], accB, vmask);
      }
    }
    auto flush = [&](bool st, uint32_t o, float acc, float pv) {
      if (st) {
        XT yv;
        if constexpr (sizeof(XT) == 2) yv = __float2half_rn(acc);
        else yv = acc;
        static_cast<XT*>(a.y)[o] = yv;
        if constexpr (DOT) dotv += (double)pv * (double)to_f<XT>(yv);
      }
    };
    flush(stA, oA, accA, pvA);
    flush(stB, oB, accB, pvB);
  }
  finish_dot<DOT>(a, dotv);
}

// ---- long slices (power-law rows): segments of seg_len steps per warp.
// The column cursor of a delta chain cannot start mid-row, so each segment
// carries a checkpoint: 2 * column of every lane before its first step
// (psell_spmv_seg_checkpoints, computed once per matrix).  Segment partial
// sums land in `partial` and a combine pass adds them in segment order
// (deterministic) and writes y through the permutation.
__device__ __forceinline__ uint32_t word_c2(uint32_t w, uint32_t m_real) {
  return w & ((w & 1u) ? m_real : 0xFFFFFFFEu);
}

// checkpoint pass 1: per segment and lane, sum of 2*delta over the segment's steps
__global__ void __launch_bounds__(kBlock) seg_dsum_kernel(const SpmvArgs a, long long n_seg) {
  const long long sg = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (sg >= n_seg) return;
  const int k = a.seg_slice[sg];
  const int q0 = a.seg_q0[sg];
  const long long o0 = a.offset[k];
  const int width = (int)((a.offset[k + 1] - o0) >> 5);
  const int q1 = min(q0 + a.seg_len, width);
  const uint32_t* p = static_cast<const uint32_t*>(a.pack) + o0 + lane;
  const uint32_t m_real = a.codec == PSELL_FP16 ? 0xFFFEu : ((2u << a.d) - 2u);
  uint32_t s = 0;
  for (int q = q0; q < q1; ++q) s += word_c2(__ldg(p + (long long)q * 32), m_real);
  a.seg_c2[sg * 32 + lane] = s;
}

// checkpoint pass 2: per long slice, exclusive prefix of the segment sums + base
__global__ void __launch_bounds__(kBlock) seg_prefix_kernel(const SpmvArgs a, long long n_long) {
  const long long l = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (l >= n_long) return;
  const int k = a.long_slice[l];
  const uint32_t g = (uint32_t)a.row0 + (uint32_t)k * 32u + lane;
  const uint32_t se = (uint32_t)a.se, kl = (uint32_t)a.k_left;
  const uint32_t cmax = a.n_cols > 0 ? (uint32_t)(a.n_cols - 1) : 0u;
  const uint32_t blk = (g / se) * se;
  const uint32_t d0 = blk > kl ? blk - kl : 0u;
  uint32_t run = 2u * (d0 < cmax ? d0 : cmax);
  for (int sgi = a.long_seg0[l]; sgi < a.long_seg0[l + 1]; ++sgi) {
    const uint32_t t = a.seg_c2[(long long)sgi * 32 + lane];
    a.seg_c2[(long long)sgi * 32 + lane] = run;
    run += t;
  }
}

// one 256-step segment of a long slice, by one warp (sg warp-uniform)
template <int CODEC, typename XT, int U>
__device__ __forceinline__ void seg_one(const SpmvArgs& a, long long sg) {
  using S = FastStep<CODEC, XT, true>;  // irregular rows: flag-predicated gathers
  const int lane = threadIdx.x & 31;
  const int k = a.seg_slice[sg];
  const int q0 = a.seg_q0[sg];
  const long long o0 = a.offset[k];
  const int width = (int)((a.offset[k + 1] - o0) >> 5);
  const int nst = min(a.seg_len, width - q0);
  const uint32_t* p = static_cast<const uint32_t*>(a.pack) + o0 + (long long)q0 * 32 + lane;
  const XT* __restrict__ x = static_cast<const XT*>(a.x);
  const uint32_t m_real = CODEC == PSELL_FP16 ? 0xFFFEu : ((2u << a.d) - 2u);
  const uint32_t vmask = CODEC == PSELL_FP16 ? 0u : ~((2u << a.d) - 1u);
  uint32_t c2 = a.seg_c2[sg * 32 + lane];
  float acc = 0.f;
  uint32_t cur[U], nxt[U];
#pragma unroll
  for (int u = 0; u < U; ++u) cur[u] = (u < nst) ? __ldcs(p + u * 32) : 0u;
  for (int q = 0; q < nst; q += U) {
    const int qn = q + U;
    if (qn + U <= nst) {
#pragma unroll
      for (int u = 0; u < U; ++u) nxt[u] = __ldcs(p + (qn + u) * 32);
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) nxt[u] = (qn + u < nst) ? __ldcs(p + (qn + u) * 32) : 0u;
    }
    // words past the segment end were loaded as 0: delta 0, FMA predicated off
#pragma unroll
    for (int u = 0; u < U; ++u) S::run(cur[u], c2, x, acc, m_real, vmask);
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = nxt[u];
  }
  a.seg_partial[sg * 32 + lane] = acc;
}

template <int CODEC, typename XT, int U>
__device__ __forceinline__ void seg_body(const SpmvArgs& a, long long n_seg, unsigned bid) {
  const long long sg = ((long long)bid * kBlock + threadIdx.x) >> 5;
  if (sg < n_seg) seg_one<CODEC, XT, U>(a, sg);
}

template <int CODEC, typename XT, int U>
__global__ void __launch_bounds__(kBlock, 6) spmv_seg_kernel(const SpmvArgs a, long long n_seg) {
  seg_body<CODEC, XT, U>(a, n_seg, blockIdx.x);
}

// Segments and short slices in ONE grid (the default for segmented matrices): the first
// seg_ctas CTAs run the long slices' segments, the rest the dual kernel over the short
// slices.  CTAs dispatch in index order, so the segments start first and the dual CTAs
// fill the GPU around them: the segment launch (551 CTAs on config 4, 62 % of one wave at
// 6 CTAs/SM) no longer runs alone after the dual kernel.  Same code per warp: bitwise.
template <int CODEC, typename XT, int U>
__global__ void __launch_bounds__(kBlock, 6) spmv_dual_seg_kernel(const SpmvArgs a, long long n_seg,
                                                                 unsigned seg_ctas) {
  if (blockIdx.x < seg_ctas) seg_body<CODEC, XT, U>(a, n_seg, blockIdx.x);
  else dual_body<CODEC, XT, false, 8, true, false>(a, blockIdx.x - seg_ctas);
}

template <typename XT>
__global__ void __launch_bounds__(kBlock) seg_combine_kernel(const SpmvArgs a, long long n_long) {
  const long long l = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (l >= n_long) return;
  const int k = a.long_slice[l];
  float acc = 0.f;
  for (int sgi = a.long_seg0[l]; sgi < a.long_seg0[l + 1]; ++sgi) acc += a.seg_partial[(long long)sgi * 32 + lane];
  const uint32_t s = (uint32_t)k * 32u + lane;
  if ((long long)s < a.n_rows) {
    uint32_t o = s;
    if (a.mode == PSELL_MODE_IMPLICIT) {
      const uint32_t sig = (uint32_t)a.sigma;
      const uint32_t p8 = a.perm_bytes == 1 ? (uint32_t)static_cast<const uint8_t*>(a.perm)[s]
                                            : (uint32_t)static_cast<const uint16_t*>(a.perm)[s];
      o = (s / sig) * sig + p8;
    }
    if constexpr (sizeof(XT) == 2) static_cast<XT*>(a.y)[o] = __float2half_rn(acc);
    else static_cast<XT*>(a.y)[o] = acc;
  }
}

// ---- TMA-staged production path (C == 32): per-warp cp.async.bulk ring
//
// Each warp owns one slice.  Its words stream global -> shared memory through
// a ring of kStages chunks of kChunk steps (kChunk * 128 B, contiguous in
// `pack` because slices are column major), issued by lane 0 with
// cp.async.bulk + mbarrier complete_tx and an L2 evict_first hint, so up to
// kStages KB per warp (the whole slice for config 2) are in flight without
// holding registers.  Lanes read step q as one conflict-free 128 B LDS wave.
// The decode / gather / FMA per word is FastStep (above).
constexpr int kChunk = 8;
constexpr int kStages = 4;
constexpr int kWarps = kBlock / 32;

constexpr int kTmaCtasPerSm = 6;

// ---- TMA stream path (C == 32), the production kernel.
//
// Persistent; warp w owns the contiguous slice range [kb, ke) whose words are
// the w-th 1/nwarps of `pack` (lower_bound on the int64 slice offsets), so
// work is balanced by stored words, not rows (power-law matrices included).
// Slices are contiguous in `pack`, so the warp's input is ONE contiguous byte
// range: lane 0 streams it through the ring in kChunk-step (1 KB) bulk copies,
// refilling each stage as soon as the warp has read it.  Lanes consume
// chunk-major and detect slice boundaries on the fly (flush y, reset cursor).
__device__ __forceinline__ long long lower_bound_off(const int64_t* off, long long n, long long target) {
  long long lo = 0, hi = n;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (off[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <int CODEC, typename XT, bool DOT>
__global__ void __launch_bounds__(kBlock, kTmaCtasPerSm) spmv_stream_kernel(const SpmvArgs a) {
  using S = FastStep<CODEC, XT>;
  __shared__ alignas(128) uint32_t ring[kWarps][kStages][kChunk * 32];
  __shared__ alignas(8) uint64_t bars[kWarps][kStages];
  if constexpr (DOT) {
    if (a.skip && *a.skip) return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * kWarps;
  const long long wid = (long long)blockIdx.x * kWarps + warp;
  const int64_t* off = a.offset;
  const long long total = off[a.n_slices];
  const long long kb = lower_bound_off(off, a.n_slices, total * wid / nw);
  const long long ke = (wid == nw - 1) ? a.n_slices : lower_bound_off(off, a.n_slices, total * (wid + 1) / nw);
  uint64_t* bar = bars[warp];
  uint32_t(*buf)[kChunk * 32] = ring[warp];
  double dotv = 0.0;
  if (kb < ke) {
    const long long T0 = off[kb] >> 5;
    const long long nsteps = (off[ke] >> 5) - T0;
    const long long nchunks = (nsteps + kChunk - 1) / kChunk;
    const uint32_t* src = static_cast<const uint32_t*>(a.pack) + T0 * 32;
    uint64_t pol = 0;
    if (lane == 0) {
      pol = policy_evict_first();
#pragma unroll
      for (int st = 0; st < kStages; ++st) mbar_init(&bar[st], 1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (long long i = 0; i < kStages && i < nchunks; ++i) {
        const uint32_t bytes = (uint32_t)min((long long)kChunk, nsteps - i * kChunk) * 128u;
        mbar_expect_tx(&bar[i], bytes);
        bulk_g2s(buf[i], src + i * (kChunk * 32), bytes, &bar[i], pol);
      }
    }
    __syncwarp();
    const XT* __restrict__ x = static_cast<const XT*>(a.x);
    const uint32_t m_real = CODEC == PSELL_FP16 ? 0xFFFEu : ((2u << a.d) - 2u);
    const uint32_t vmask = CODEC == PSELL_FP16 ? 0u : ~((2u << a.d) - 1u);
    const uint32_t se = (uint32_t)a.se, sig = (uint32_t)a.sigma;
    const uint32_t cmax = a.n_cols > 0 ? (uint32_t)(a.n_cols - 1) : 0u;
    const uint32_t row0 = (uint32_t)a.row0, kl = (uint32_t)a.k_left;
    auto base2 = [&](long long k) -> uint32_t {  // 2 * min(d_s, n_cols - 1), 32-bit (n < 2^31)
      const uint32_t g = row0 + (uint32_t)(k * 32 + lane);
      const uint32_t blk = (g / se) * se;
      const uint32_t d = blk > kl ? blk - kl : 0u;
      return 2u * (d < cmax ? d : cmax);
    };
    auto flush = [&](long long k, float acc) {
      const uint32_t s = (uint32_t)(k * 32 + lane);
      if ((long long)s < a.n_rows) {
        uint32_t o = s;
        if (a.mode == PSELL_MODE_IMPLICIT) {
          const uint32_t p = a.perm_bytes == 1 ? (uint32_t)static_cast<const uint8_t*>(a.perm)[s]
                                               : (uint32_t)static_cast<const uint16_t*>(a.perm)[s];
          o = (s / sig) * sig + p;
        }
        XT yv;
        if constexpr (sizeof(XT) == 2) yv = __float2half_rn(acc);
        else yv = acc;
        static_cast<XT*>(a.y)[o] = yv;
        if constexpr (DOT) dotv += (double)a.p_own[o] * (double)to_f<XT>(yv);
      }
    };
    // current slice: k, its end step (relative to T0), cursor, accumulator
    long long k = kb;
    long long bnd = (off[k + 1] >> 5) - T0;
    while (bnd == 0 && k + 1 < ke) {  // leading zero-width slices
      flush(k, 0.f);
      ++k;
      bnd = (off[k + 1] >> 5) - T0;
    }
    uint32_t c2 = base2(k);
    float acc = 0.f;
    auto advance = [&](long long g) {  // slice k ended at step g: flush it and the empty ones after it
      flush(k, acc);
      ++k;
      bnd = (off[k + 1] >> 5) - T0;
      while (bnd == g && k + 1 < ke) {
        flush(k, 0.f);
        ++k;
        bnd = (off[k + 1] >> 5) - T0;
      }
      c2 = base2(k);
      acc = 0.f;
    };
    for (long long i = 0; i < nchunks; ++i) {
      const int st = (int)(i % kStages);
      mbar_wait(&bar[st], (uint32_t)(i / kStages) & 1u);
      uint32_t w[kChunk];
#pragma unroll
      for (int u = 0; u < kChunk; ++u) w[u] = buf[st][u * 32 + lane];
      __syncwarp();
      if (lane == 0 && i + kStages < nchunks) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const long long cn = i + kStages;
        const uint32_t bytes = (uint32_t)min((long long)kChunk, nsteps - cn * kChunk) * 128u;
        mbar_expect_tx(&bar[st], bytes);
        bulk_g2s(buf[st], src + cn * (kChunk * 32), bytes, &bar[st], pol);
      }
      const long long g0 = i * kChunk;
      if (g0 + kChunk <= nsteps) {
#pragma unroll
        for (int u = 0; u < kChunk; ++u) {
          if (g0 + u == bnd) advance(g0 + u);
          S::run(w[u], c2, x, acc, m_real, vmask);
        }
      } else {
        for (int u = 0; g0 + u < nsteps; ++u) {
          if (g0 + u == bnd) advance(g0 + u);
          S::run(w[u], c2, x, acc, m_real, vmask);
        }
      }
    }
    flush(k, acc);  // last non-empty slice (or the only, empty, one)
    for (++k; k < ke; ++k) flush(k, 0.f);  // trailing zero-width slices
  }
  finish_dot<DOT>(a, dotv);
}

// ---- tile-TMA kernel (C == 32, narrow slices): producer/consumer over a smem ring
//
// A persistent CTA = 8 consumer warps + 1 producer warp.  Tiles of 16
// consecutive slices are dealt round-robin over the CTAs (so the tiles in
// flight across the chip form one dense window of `pack`, keeping DRAM pages
// open).  The producer's elected lane streams each tile's words — one
// contiguous byte range, since slices are stored back to back — into a 4-stage
// shared-memory ring with ONE cp.async.bulk per tile (mbarrier complete_tx),
// up to 4 tiles ahead; consumer warps take two slices each, read the words
// with conflict-free LDS (step q of a slice is 32 consecutive words), and run
// the usual decode / gather / FMA.  HBM latency is off the consumers' critical
// path; they only wait on the L2-resident x gathers.  A tile wider than a
// stage (12 steps per slice on average) is flagged and read straight from HBM.
constexpr int kTileSlices = 16;
constexpr int kTileStages = 4;
constexpr int kTileStageWords = kTileSlices * 12 * 32;  // 24 KB
constexpr int kTileConsumers = 8;
constexpr int kTileThreads = (kTileConsumers + 1) * 32;
constexpr int kTileCtasPerSm = 2;
constexpr size_t kTileSmemBytes = (size_t)kTileStages * kTileStageWords * 4;

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// both slices of a warp interleaved step by step (24 gathers in flight per 12-step chunk)
template <int CODEC, typename XT, bool SMEM>
__device__ __forceinline__ void tile_pair(const uint32_t* pA, int wA, const uint32_t* pB, int wB, uint32_t cA,
                                          uint32_t cB, const XT* x, uint32_t m_real, uint32_t vmask, float& accA,
                                          float& accB) {
  using S = FastStep<CODEC, XT>;
  constexpr int U = 12;
  accA = 0.f;
  accB = 0.f;
  const int wm = wA > wB ? wA : wB;
  for (int q = 0; q < wm; q += U) {
    uint32_t ua[U], ub[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (SMEM) {
        ua[u] = (q + u < wA) ? pA[(q + u) * 32] : 0u;
        ub[u] = (q + u < wB) ? pB[(q + u) * 32] : 0u;
      } else {
        ua[u] = (q + u < wA) ? __ldcs(pA + (q + u) * 32) : 0u;
        ub[u] = (q + u < wB) ? __ldcs(pB + (q + u) * 32) : 0u;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      S::run(ua[u], cA, x, accA, m_real, vmask);
      S::run(ub[u], cB, x, accB, m_real, vmask);
    }
  }
}

template <int CODEC, typename XT, bool DOT>
__global__ void __launch_bounds__(kTileThreads, kTileCtasPerSm) spmv_tile_kernel(const SpmvArgs a) {
  extern __shared__ __align__(128) uint32_t tsm[];  // [kTileStages][kTileStageWords]
  __shared__ __align__(8) uint64_t full[kTileStages];
  __shared__ __align__(8) uint64_t empty[kTileStages];
  __shared__ long long tbase[kTileStages];
  __shared__ int tdirect[kTileStages];
  if constexpr (DOT) {
    if (a.skip && *a.skip) return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ns = (uint32_t)a.n_slices;
  const uint32_t n_tiles = (ns + kTileSlices - 1) / kTileSlices;
  const uint32_t* pack = static_cast<const uint32_t*>(a.pack);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int st = 0; st < kTileStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kTileConsumers);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  double dotv = 0.0;
  if (warp == kTileConsumers) {  // producer warp
    // the word ranges of the CTA's next 32 tiles are loaded warp-wide at once
    // (lane j: tile j of the batch), so the issuing lane never waits on an
    // offset load between two bulk copies
    const uint64_t pol = policy_evict_first();
    int i = 0;
    for (uint32_t tb = blockIdx.x; tb < n_tiles; tb += 32u * gridDim.x) {
      const uint32_t tj = tb + (uint32_t)lane * gridDim.x;
      long long bj = 0, ej = 0;
      if (tj < n_tiles) {
        bj = a.offset[tj * kTileSlices];
        ej = a.offset[min((tj + 1) * (uint32_t)kTileSlices, ns)];
      }
      const int nb = (int)min(32u, (n_tiles - tb + gridDim.x - 1) / gridDim.x);
      for (int j = 0; j < nb; ++j, ++i) {
        const long long w0 = __shfl_sync(0xffffffffu, bj, j);
        const long long words = __shfl_sync(0xffffffffu, ej, j) - w0;
        if (lane == 0) {
          const int st = i % kTileStages;
          if (i >= kTileStages) mbar_wait(&empty[st], (uint32_t)((i / kTileStages) - 1) & 1u);
          tbase[st] = w0;
          if (words <= kTileStageWords) {
            tdirect[st] = 0;
            const uint32_t bytes = (uint32_t)words * 4u;
            mbar_expect_tx(&full[st], bytes);
            if (bytes) bulk_g2s(tsm + st * kTileStageWords, pack + w0, bytes, &full[st], pol);
          } else {
            tdirect[st] = 1;
            mbar_arrive(&full[st]);
          }
        }
        __syncwarp();
      }
    }
  } else {  // consumers: slices 2w, 2w+1 of each tile
    const XT* __restrict__ x = static_cast<const XT*>(a.x);
    const uint32_t m_real = CODEC == PSELL_FP16 ? 0xFFFEu : ((2u << a.d) - 2u);
    const uint32_t vmask = CODEC == PSELL_FP16 ? 0u : ~((2u << a.d) - 1u);
    const uint32_t kl = (uint32_t)a.k_left, n_rows = (uint32_t)a.n_rows;
    const uint32_t cmax = a.n_cols > 0 ? (uint32_t)(a.n_cols - 1) : 0u;
    const bool impl = a.mode == PSELL_MODE_IMPLICIT;
    int i = 0;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
      const int st = i % kTileStages;
      const uint32_t kA = t * kTileSlices + 2u * warp, kB = kA + 1u;
      const bool hasA = kA < ns, hasB = kB < ns;
      // independent of the stage: offsets, perm bytes, base offsets (latency overlaps the wait)
      long long o0 = 0, o1 = 0, o2 = 0;
      uint32_t oA = 0, oB = 0;
      if (hasA) {
        o0 = a.offset[kA];
        o1 = a.offset[kA + 1];
        o2 = hasB ? a.offset[kA + 2] : o1;
        const uint32_t sA = kA * 32u + lane, sB = sA + 32u;
        oA = sA;
        oB = sB;
        if (impl) {
          const uint32_t blkA = fast_div(kA * 32u, a.sig_m, a.sig_l) * (uint32_t)a.sigma;
          const uint32_t blkB = fast_div(kB * 32u, a.sig_m, a.sig_l) * (uint32_t)a.sigma;
          if (a.perm_bytes == 1) {
            const uint8_t* pm = static_cast<const uint8_t*>(a.perm);
            oA = blkA + (sA < n_rows ? (uint32_t)__ldg(pm + sA) : 0u);
            oB = blkB + (sB < n_rows ? (uint32_t)__ldg(pm + sB) : 0u);
          } else {
            const uint16_t* pm = static_cast<const uint16_t*>(a.perm);
            oA = blkA + (sA < n_rows ? (uint32_t)__ldg(pm + sA) : 0u);
            oB = blkB + (sB < n_rows ? (uint32_t)__ldg(pm + sB) : 0u);
          }
        }
      }
      auto base2 = [&](uint32_t k) -> uint32_t {
        const uint32_t g = (uint32_t)a.row0 + k * 32u + lane;
        const uint32_t blk = a.se == 1 ? g : fast_div(g, a.se_m, a.se_l) * (uint32_t)a.se;
        const uint32_t d = blk > kl ? blk - kl : 0u;
        return 2u * (d < cmax ? d : cmax);
      };
      mbar_wait(&full[st], (uint32_t)(i / kTileStages) & 1u);
      if (hasA) {
        const int wA = (int)((o1 - o0) >> 5), wB = (int)((o2 - o1) >> 5);
        float accA, accB;
        if (!tdirect[st]) {
          const uint32_t* sp = tsm + st * kTileStageWords + (uint32_t)(o0 - tbase[st]) + lane;
          tile_pair<CODEC, XT, true>(sp, wA, sp + (uint32_t)(o1 - o0), wB, base2(kA), base2(kB), x, m_real, vmask,
                                     accA, accB);
        } else {
          tile_pair<CODEC, XT, false>(pack + o0 + lane, wA, pack + o1 + lane, wB, base2(kA), base2(kB), x, m_real,
                                      vmask, accA, accB);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);  // words consumed: the producer may refill
        auto flush = [&](uint32_t s, uint32_t o, float acc) {
          if (s < n_rows) {
            XT yv;
            if constexpr (sizeof(XT) == 2) yv = __float2half_rn(acc);
            else yv = acc;
            static_cast<XT*>(a.y)[o] = yv;
            if constexpr (DOT) dotv += (double)a.p_own[o] * (double)to_f<XT>(yv);
          }
        };
        flush(kA * 32u + lane, oA, accA);
        if (hasB) flush(kB * 32u + lane, oB, accB);
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
    }
  }
  finish_dot<DOT, kTileThreads>(a, dotv);
}

// ---- slot kernel (narrow slices, C == 32): the persistent pair kernel with the next
// pair's words in flight during the current pair's gathers.
// Each warp owns one shared-memory slot (a pair of slices <= 12 steps each: 3 KB)
// and an mbarrier.  Iteration k: wait for pair k in the slot, copy it into
// registers, and immediately refill the slot with pair k+1 (ONE cp.async.bulk by
// lane 0, L2 evict-first), so pair k+1's HBM latency overlaps pair k's x gathers
// and FMAs instead of following them.  No per-lane global word loads and no word
// pointers in registers; lane 0 keeps the look-ahead offsets in shared memory and
// every lane reads the current widths from there.  The same FMAs in the same order
// as the pair kernel (bitwise equal).  Launched only when every slice is <= 12 steps
// wide (PSELL_SPMV_NARROW12: 7-point rows are 9).
constexpr int kSlotWords = 768;
#ifndef PSELL_SLOT_MINB
#define PSELL_SLOT_MINB 6  // resident CTAs per SM the slot kernel's register budget is sized for
#endif
constexpr int kSlotCtasPerSm = PSELL_SLOT_MINB;
// per warp: the word slot, its mbarrier, two look-ahead offset triples (cp.async'd
// 8-byte LDGSTS, so lane 0 never waits on an offset load) and the current widths
struct SlotMeta {
  long long off[2][4];
  uint32_t cur;
  uint32_t pad[3];
};
constexpr size_t kSlotSmemBytes = kWarpsPerCta * (kSlotWords * 4 + 8 + sizeof(SlotMeta));

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem_dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_group1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <int CODEC, typename XT, bool DOT>
__global__ void __launch_bounds__(kBlock, kSlotCtasPerSm) spmv_slot_kernel(const SpmvArgs a) {
  using S = FastStep<CODEC, XT>;
  if constexpr (DOT) {
    if (a.skip && *a.skip) return;
  }
  extern __shared__ __align__(128) unsigned char slot_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* slot = reinterpret_cast<uint32_t*>(slot_smem) + warp * kSlotWords;
  uint64_t* bar = reinterpret_cast<uint64_t*>(slot_smem + kWarpsPerCta * kSlotWords * 4) + warp;
  SlotMeta* meta = reinterpret_cast<SlotMeta*>(slot_smem + kWarpsPerCta * (kSlotWords * 4 + 8)) + warp;
  const uint32_t ns = (uint32_t)a.n_slices;
  const uint32_t npairs = (ns + 1u) >> 1;
  const uint32_t wstride = gridDim.x * (unsigned)kWarpsPerCta;
  uint32_t pk = blockIdx.x * (unsigned)kWarpsPerCta + warp;
  // lanes 0..2: request the offset triple of pair p into look-ahead slot r (async)
  auto request_offsets = [&](uint32_t p, int r) {
    if (lane < 3 && p < npairs) {
      const uint32_t kk = 2u * p + (uint32_t)lane;
      cp_async8(&meta->off[r][lane], a.offset + (kk <= ns ? kk : ns));
    }
    cp_async_commit();
  };
  // lane 0: the bulk copy of a pair whose offsets sit in look-ahead slot r; records its widths
  auto issue_words = [&](int r) {
    const long long o0 = meta->off[r][0], o1 = meta->off[r][1], o2 = meta->off[r][2];
    const uint32_t wA = (uint32_t)((o1 - o0) >> 5), wB = (uint32_t)((o2 - o1) >> 5);
    meta->cur = wA | (wB << 16);
    const uint32_t bytes = (wA + wB) * 128u;
    if (bytes == 0) return;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar, bytes);
    bulk_g2s(slot, static_cast<const uint32_t*>(a.pack) + o0, bytes, bar, policy_evict_first());
  };
  if (lane == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // prologue: offsets of the first two pairs, words of the first
  request_offsets(pk, 0);
  request_offsets(pk + wstride, 1);
  cp_async_wait_all();
  __syncwarp();
  if (lane == 0 && pk < npairs) issue_words(0);
  __syncwarp();
  int rnext = 1;  // look-ahead slot holding the offsets of the next pair
  uint32_t phase = 0;
  const XT* __restrict__ x = static_cast<const XT*>(a.x);
  const uint32_t m_real = CODEC == PSELL_FP16 ? 0xFFFEu : ((2u << a.d) - 2u);
  const uint32_t vmask = CODEC == PSELL_FP16 ? 0u : ~((2u << a.d) - 1u);
  double dotv = 0.0;
  constexpr int U = 12, K = PairK<12>::K;
  for (; pk < npairs; pk += wstride) {
    const uint32_t kA = 2u * pk, kB = kA + 1u;
    const uint32_t n_rows = (uint32_t)a.n_rows;
    const uint32_t sA = kA * 32u + lane, sB = sA + 32u;
    // perm bytes issued first, consumed only at the flush: adding them into the output
    // row right away put a full-latency stall in front of the word decode (ncu: the
    // hottest stall of the pair kernel)
    const bool impl = a.mode == PSELL_MODE_IMPLICIT;
    auto perm_of = [&](uint32_t s) -> uint32_t {
      if (!impl) return 0u;
      const uint32_t sc = s < n_rows ? s : n_rows - 1u;
      return a.perm_bytes == 1 ? (uint32_t)__ldg(static_cast<const uint8_t*>(a.perm) + sc)
                               : (uint32_t)__ldg(static_cast<const uint16_t*>(a.perm) + sc);
    };
    const uint32_t ppA = perm_of(sA), ppB = perm_of(sB);
    auto base2 = [&](uint32_t k) -> uint32_t {
      const uint32_t kl = (uint32_t)a.k_left;
      const uint32_t cmax = a.n_cols > 0 ? (uint32_t)(a.n_cols - 1) : 0u;
      const uint32_t g = (uint32_t)a.row0 + k * 32u + lane;
      const uint32_t blk = a.se == 1 ? g : fast_div(g, a.se_m, a.se_l) * (uint32_t)a.se;
      const uint32_t d = blk > kl ? blk - kl : 0u;
      return 2u * (d < cmax ? d : cmax);
    };
    uint32_t cA = base2(kA), cB = base2(kB);
    mbar_wait(bar, phase);
    phase ^= 1u;
    const uint32_t wab = meta->cur;
    const int wA = (int)(wab & 0xFFFFu), wB = (int)(wab >> 16);
    uint32_t wa[U], wb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      wa[u] = u < wA ? slot[u * 32 + lane] : 0u;
      wb[u] = u < wB ? slot[(wA + u) * 32 + lane] : 0u;
    }
    // the next pair's offsets were requested an iteration ago: refill the slot with its
    // words now, and request the offsets of the pair after it into the freed slot
    cp_async_wait_all();
    __syncwarp();
    if (lane == 0 && pk + wstride < npairs) issue_words(rnext);
    __syncwarp();
    request_offsets(pk + 2u * wstride, rnext ^ 1);
    rnext ^= 1;
    float accA = 0.f, accB = 0.f;
#pragma unroll
    for (int u = 0; u < K; ++u) {
      S::run(wa[u], cA, x, accA, m_real, vmask);
      S::run(wb[u], cB, x, accB, m_real, vmask);
    }
    if (wA > K || wB > K) {
#pragma unroll
      for (int u = K; u < U; ++u) {
        S::run(wa[u], cA, x, accA, m_real, vmask);
        S::run(wb[u], cB, x, accB, m_real, vmask);
      }
    }
    auto flush = [&](uint32_t k, uint32_t s, uint32_t pp, float acc) {
      if (s < n_rows) {
        const uint32_t o = impl ? fast_div(k * 32u, a.sig_m, a.sig_l) * (uint32_t)a.sigma + pp : s;
        XT yv;
        if constexpr (sizeof(XT) == 2) yv = __float2half_rn(acc);
        else yv = acc;
        static_cast<XT*>(a.y)[o] = yv;
        if constexpr (DOT) dotv += (double)a.p_own[o] * (double)to_f<XT>(yv);
      }
    };
    flush(kA, sA, ppA, accA);
    if (kB < ns) flush(kB, sB, ppB, accB);
  }
  finish_dot<DOT>(a, dotv);
}

// ---- narrow TMA kernel (PSELL_NARROW_TMA=1): the narrow kernel with each warp's
// slice-pair words staged through two shared-memory slots by cp.async.bulk (one bulk copy
// per pair, issued by lane 0 about one pair ahead), so a pair's words are resident when the
// warp reaches it instead of costing an HBM round trip per pair (29 % of the narrow
// kernel's stall samples wait on its first word).  The offsets of the pairs ahead travel
// through a 4-entry shared ring by cp.async (a register rotation of prefetched offsets
// waits on the loads).  Same decode, FMAs and order as the narrow kernel.  (Per-lane
// 16-byte cp.async.cg staging instead of the bulk copy: 130.5 us, fused dot 162 us.)
constexpr int kNtSlotWords = 24 * 32;  // a pair of slices of <= 12 steps
struct NtMeta {
  long long off[4][4];  // ring of {o0, o1, o2, pad} for the pairs ahead
};
constexpr size_t kNtSmemBytes = kWarpsPerCta * (2 * kNtSlotWords * 4 + 2 * 8 + sizeof(NtMeta));
template <int CODEC, typename XT, bool DOT, int PB, bool P2>
__global__ void __launch_bounds__(kBlock, 4) spmv_narrow_tma_kernel(const SpmvArgs a) {
  using S = NarrowStep<CODEC, XT>;
  constexpr int U = 12, K = PSELL_NARROW_K;
  if constexpr (DOT) {
    if (a.skip && *a.skip) return;
  }
  extern __shared__ __align__(128) unsigned char nt_smem[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  uint32_t* slots = reinterpret_cast<uint32_t*>(nt_smem) + warp * 2 * kNtSlotWords;
  uint64_t* bars = reinterpret_cast<uint64_t*>(nt_smem + kWarpsPerCta * 2 * kNtSlotWords * 4) + warp * 2;
  NtMeta* meta = reinterpret_cast<NtMeta*>(nt_smem + kWarpsPerCta * (2 * kNtSlotWords * 4 + 16)) + warp;
  const uint32_t ns = (uint32_t)a.n_slices, np = (ns + 1u) >> 1;
  const uint32_t n_rows = (uint32_t)a.n_rows;
  const uint32_t ws = gridDim.x * (unsigned)kWarpsPerCta;
  const XT* __restrict__ x = static_cast<const XT*>(a.x);
  const uint32_t* __restrict__ pack = static_cast<const uint32_t*>(a.pack);
  const uint32_t m_real = CODEC == PSELL_FP16 ? 0xFFFEu : ((2u << a.d) - 2u);
  const uint32_t vmask = CODEC == PSELL_FP16 ? 0u : ~((2u << a.d) - 1u);
  const uint32_t kl = (uint32_t)a.k_left, row0 = (uint32_t)a.row0, se = (uint32_t)a.se;
  const uint32_t cmax = a.n_cols > 0 ? (uint32_t)(a.n_cols - 1) : 0u;
  auto perm_of = [&](uint32_t s) -> uint32_t {
    const uint32_t sc = s < n_rows ? s : n_rows - 1u;
    if constexpr (PB == 1) return (uint32_t)__ldg(static_cast<const uint8_t*>(a.perm) + sc);
    else return (uint32_t)__ldg(static_cast<const uint16_t*>(a.perm) + sc);
  };
  // lanes 0..2: the offset triple of pair g into ring entry r (async; one commit group per call)
  auto request = [&](uint32_t g, uint32_t r) {
    if (lane < 3u && g < np) {
      const uint32_t k = 2u * g + lane;
      cp_async8(&meta->off[r][lane], a.offset + (k <= ns ? k : ns));
    }
    cp_async_commit();
  };
  // the whole warp: the bulk copy of the pair in ring entry r into slot sl, issued by one
  // elected lane (operands warp-uniform: no divergent lane-0 path for ptxas to serialise);
  // an empty pair just arrives on the barrier
  auto issue = [&](uint32_t sl, uint32_t r) {
    const long long o0 = meta->off[r][0], o2 = meta->off[r][2];
    const uint32_t bytes = (uint32_t)(o2 - o0) * 4u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile(
        "{\n .reg .pred e, z;\n elect.sync _|e, 0xffffffff;\n setp.eq.u32 z, %2, 0;\n"
        " @e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %2;\n"
        " @!z and.pred e, e, !z;\n"
        " @e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%3], %2, [%1], %4;\n}"
        ::"r"(smem_u32(slots + sl * kNtSlotWords)), "r"(smem_u32(bars + sl)), "r"(bytes), "l"(pack + o0),
        "l"(policy_evict_first())
        : "memory");
  };
  uint32_t wg = blockIdx.x * (unsigned)kWarpsPerCta + warp;
  if (lane == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  request(wg, 0);
  request(wg + ws, 1);
  request(wg + 2u * ws, 2);
  cp_async_wait_all();
  __syncwarp();
  if (wg < np) issue(0, 0);
  if (wg + ws < np) issue(1, 1);
  uint32_t n_ppA = 0u, n_ppB = 0u;
  if constexpr (PB != 0) {
    n_ppA = perm_of(2u * wg * 32u + lane);
    n_ppB = perm_of(2u * wg * 32u + 32u + lane);
  }
  double dotv = 0.0;
  for (uint32_t it = 0; wg < np; wg += ws, ++it) {
    const uint32_t sl = it & 1u, r = it & 3u;
    request(wg + 3u * ws, (it + 3u) & 3u);
    const uint32_t* slot = slots + sl * kNtSlotWords;
    const uint32_t kA = 2u * wg;
    const bool hasB = kA + 1u < ns;
    const uint32_t q0 = (uint32_t)meta->off[r][0], q1 = (uint32_t)meta->off[r][1], q2 = (uint32_t)meta->off[r][2];
    const uint32_t wA = (q1 - q0) >> 5, wB = (q2 - q1) >> 5;
    const uint32_t ppA = n_ppA, ppB = n_ppB;
    if constexpr (PB != 0) {
      if (wg + ws < np) {
        n_ppA = perm_of(2u * (wg + ws) * 32u + lane);
        n_ppB = perm_of(2u * (wg + ws) * 32u + 32u + lane);
      }
    }
    auto base2 = [&](uint32_t k) -> uint32_t {
      const uint32_t g = row0 + k * 32u + lane;
      const uint32_t blk = P2 ? g & ~(se - 1u) : se == 1u ? g : fast_div(g, a.se_m, a.se_l) * se;
      const uint32_t d = blk > kl ? blk - kl : 0u;
      return 2u * (d < cmax ? d : cmax);
    };
    uint32_t cA = base2(kA), cB = base2(kA + 1u);
    mbar_wait(bars + sl, (it >> 1) & 1u);
    const uint32_t* sA = slot + lane;
    const uint32_t* sB = sA + wA * 32u;
    uint32_t wa[U], wb[U], xa[U], xb[U];
    if (wA >= (uint32_t)K && wB >= (uint32_t)K) {
#pragma unroll
      for (int u = 0; u < K; ++u) {
        wa[u] = sA[u * 32];
        wb[u] = sB[u * 32];
      }
    } else {
#pragma unroll
      for (int u = 0; u < K; ++u) {
        wa[u] = (uint32_t)u < wA ? sA[u * 32] : 0u;
        wb[u] = (uint32_t)u < wB ? sB[u * 32] : 0u;
      }
    }
#pragma unroll
    for (int u = 0; u < K; ++u) {
      xa[u] = S::gather(wa[u], cA, x, m_real);
      xb[u] = S::gather(wb[u], cB, x, m_real);
    }
    const uint32_t rA = kA * 32u + lane, rB = rA + 32u;
    uint32_t oA = rA, oB = rB;
    if constexpr (PB != 0) {
      if constexpr (P2) {  // power-of-two sigma: block starts by mask
        const uint32_t sm = ~((uint32_t)a.sigma - 1u);
        oA = ((kA * 32u) & sm) + ppA;
        oB = ((kA * 32u + 32u) & sm) + ppB;
      } else {
        oA = fast_div(kA * 32u, a.sig_m, a.sig_l) * (uint32_t)a.sigma + ppA;
        oB = fast_div(kA * 32u + 32u, a.sig_m, a.sig_l) * (uint32_t)a.sigma + ppB;
      }
    }
    const bool stA = rA < n_rows, stB = hasB && rB < n_rows;
    float pvA = 0.f, pvB = 0.f;
    if constexpr (DOT) {  // unpredicated: rows past n_rows read a valid row, their product is dropped
      pvA = __ldg(a.p_own + (oA < n_rows ? oA : n_rows - 1u));
      pvB = __ldg(a.p_own + (oB < n_rows ? oB : n_rows - 1u));
    }
    float accA = 0.f, accB = 0.f;
#pragma unroll
    for (int u = 0; u < K; ++u) {
      S::fma(wa[u], xa[u], accA, vmask);
      S::fma(wb[u], xb[u], accB, vmask);
    }
    if (wA > (uint32_t)K || wB > (uint32_t)K) {
#pragma unroll
      for (int u = K; u < U; ++u) {
        wa[u] = (uint32_t)u < wA ? sA[u * 32] : 0u;
        wb[u] = (uint32_t)u < wB ? sB[u * 32] : 0u;
      }
#pragma unroll
      for (int u = K; u < U; ++u) {
        xa[u] = S::gather(wa[u], cA, x, m_real);
        xb[u] = S::gather(wb[u], cB, x, m_real);
      }
#pragma unroll
      for (int u = K; u < U; ++u) {
        S::fma(wa[u], xa[u], accA, vmask);
        S::fma(wb[u], xb[u], accB, vmask);
      }
    }
    // every lane has read the slot and the offsets of pair +2 (requested two pairs ago)
    // have landed: refill the slot with that pair
    cp_async_wait_group1();
    __syncwarp();
    if (wg + 2u * ws < np) issue(sl, (it + 2u) & 3u);
    auto flush = [&](bool st, uint32_t o, float acc, float pv) {
      if (st) {
        XT yv;
        if constexpr (sizeof(XT) == 2) yv = __float2half_rn(acc);
        else yv = acc;
        static_cast<XT*>(a.y)[o] = yv;
        if constexpr (DOT) dotv += (double)pv * (double)to_f<XT>(yv);
      }
    };
    flush(stA, oA, accA, pvA);
    flush(stB, oB, accB, pvB);
  }
  cp_async_wait_all();
  finish_dot<DOT>(a, dotv);
}

// ---- wide TMA kernel (slices of <= 32 steps: 27-point rows, config 2 / 3).  A read-only
// stream reaches ~7.2 TB/s on this GPU against the 6.6 TB/s copy rate (scripts/probe/
// stream_read.py), so the dual kernel's 6.2 TB/s leaves room: it has bytes in flight only
// between a chunk's load and its decode.  Here each warp keeps the NEXT slice's words
// (<= 4 KB) in flight while it decodes the current one: one slice per iteration, its words
// staged by one cp.async.bulk (elected lane, mbarrier completion, evict-first) into one of
// two per-warp shared-memory slots, the offsets of the slices ahead through a 4-entry
// cp.async ring (as the narrow TMA kernel).  Decode in 8-step two-pass chunks (cursor
// prefix + gathers, then FMAs).  Per row the same steps in the same order with the same
// FMA as the dual kernel: bitwise equal to it.
constexpr int kWtSteps = 32;
constexpr int kWtSlotWords = kWtSteps * 32;
struct WtMeta {
  long long off[4][2];  // ring of {o0, o1} for the slices ahead
};
constexpr size_t kWtSmemBytes = kWarpsPerCta * (2 * kWtSlotWords * 4 + 2 * 8 + sizeof(WtMeta));
#ifndef PSELL_WIDE_CTAS
#define PSELL_WIDE_CTAS 3
#endif
#ifndef PSELL_WIDE_K
#define PSELL_WIDE_K 16
#endif
template <int CODEC, typename XT, bool DOT, int PB, bool P2>
__global__ void __launch_bounds__(kBlock, PSELL_WIDE_CTAS) spmv_wide_tma_kernel(const SpmvArgs a) {
  using S = NarrowStep<CODEC, XT>;
  constexpr int K = PSELL_WIDE_K;
  if constexpr (DOT) {
    if (a.skip && *a.skip) return;
  }
  extern __shared__ __align__(128) unsigned char wt_smem[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  uint32_t* slots = reinterpret_cast<uint32_t*>(wt_smem) + warp * 2 * kWtSlotWords;
  uint64_t* bars = reinterpret_cast<uint64_t*>(wt_smem + kWarpsPerCta * 2 * kWtSlotWords * 4) + warp * 2;
  WtMeta* meta = reinterpret_cast<WtMeta*>(wt_smem + kWarpsPerCta * (2 * kWtSlotWords * 4 + 16)) + warp;
  const uint32_t ns = (uint32_t)a.n_slices;
  const uint32_t n_rows = (uint32_t)a.n_rows;
  const uint32_t ws = gridDim.x * (unsigned)kWarpsPerCta;
  const XT* __restrict__ x = static_cast<const XT*>(a.x);
  const uint32_t* __restrict__ pack = static_cast<const uint32_t*>(a.pack);
  const uint32_t m_real = CODEC == PSELL_FP16 ? 0xFFFEu : ((2u << a.d) - 2u);
  const uint32_t vmask = CODEC == PSELL_FP16 ? 0u : ~((2u << a.d) - 1u);
  const uint32_t kl = (uint32_t)a.k_left, row0 = (uint32_t)a.row0, se = (uint32_t)a.se;
  const uint32_t cmax = a.n_cols > 0 ? (uint32_t)(a.n_cols - 1) : 0u;
  auto perm_of = [&](uint32_t s) -> uint32_t {
    const uint32_t sc = s < n_rows ? s : n_rows - 1u;
    if constexpr (PB == 1) return (uint32_t)__ldg(static_cast<const uint8_t*>(a.perm) + sc);
    else return (uint32_t)__ldg(static_cast<const uint16_t*>(a.perm) + sc);
  };
  // lanes 0..1: offsets k, k + 1 into ring entry r (async; one commit group per call)
  auto request = [&](uint32_t k, uint32_t r) {
    if (lane < 2u && k < ns) cp_async8(&meta->off[r][lane], a.offset + k + lane);
    cp_async_commit();
  };
  // the whole warp: the bulk copy of the slice in ring entry r into slot sl (elected lane);
  // an empty slice just arrives on the barrier
  auto issue = [&](uint32_t sl, uint32_t r) {
    const long long o0 = meta->off[r][0], o1 = meta->off[r][1];
    const uint32_t b = (uint32_t)(o1 - o0) * 4u;
    const uint32_t bytes = b < kWtSlotWords * 4u ? b : kWtSlotWords * 4u;  // never past the slot
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile(
        "{\n .reg .pred e, z;\n elect.sync _|e, 0xffffffff;\n setp.eq.u32 z, %2, 0;\n"
        " @e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %2;\n"
        " @!z and.pred e, e, !z;\n"
        " @e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%3], %2, [%1], %4;\n}"
        ::"r"(smem_u32(slots + sl * kWtSlotWords)), "r"(smem_u32(bars + sl)), "r"(bytes), "l"(pack + o0),
        "l"(policy_evict_first())
        : "memory");
  };
  uint32_t k = blockIdx.x * (unsigned)kWarpsPerCta + warp;
  if (lane == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  request(k, 0);
  request(k + ws, 1);
  request(k + 2u * ws, 2);
  cp_async_wait_all();
  __syncwarp();
  if (k < ns) issue(0, 0);
  if (k + ws < ns) issue(1, 1);
  uint32_t n_pp = 0u;
  if constexpr (PB != 0) n_pp = perm_of(k * 32u + lane);
  double dotv = 0.0;
  for (uint32_t it = 0; k < ns; k += ws, ++it) {
    const uint32_t sl = it & 1u, r = it & 3u;
    request(k + 3u * ws, (it + 3u) & 3u);
    const uint32_t q0 = (uint32_t)meta->off[r][0], q1 = (uint32_t)meta->off[r][1];
    const uint32_t wf = (q1 - q0) >> 5, w = wf < (uint32_t)kWtSteps ? wf : (uint32_t)kWtSteps;
    const uint32_t pp = n_pp;
    if constexpr (PB != 0) {
      if (k + ws < ns) n_pp = perm_of((k + ws) * 32u + lane);
    }
    uint32_t c2;
    {
      const uint32_t g = row0 + k * 32u + lane;
      const uint32_t blk = P2 ? g & ~(se - 1u) : se == 1u ? g : fast_div(g, a.se_m, a.se_l) * se;
      const uint32_t d = blk > kl ? blk - kl : 0u;
      c2 = 2u * (d < cmax ? d : cmax);
    }
    const uint32_t rs = k * 32u + lane;
    uint32_t o = rs;
    if constexpr (PB != 0) {
      if constexpr (P2) o = ((k * 32u) & ~((uint32_t)a.sigma - 1u)) + pp;
      else o = fast_div(k * 32u, a.sig_m, a.sig_l) * (uint32_t)a.sigma + pp;
    }
    float pv = 0.f;
    if constexpr (DOT) pv = __ldg(a.p_own + (o < n_rows ? o : n_rows - 1u));
    mbar_wait(bars + sl, (it >> 1) & 1u);
    const uint32_t* sp = slots + sl * kWtSlotWords + lane;
    float acc = 0.f;
#if PSELL_WIDE_K >= 32
    // every gather of the slice in flight at once (one L2 round trip per slice); the FMA
    // pass reads the words from the slot again instead of holding them in registers
    uint32_t xv[kWtSteps];
#pragma unroll
    for (int u = 0; u < kWtSteps; ++u)
      if ((uint32_t)u < w) xv[u] = S::gather(sp[u * 32], c2, x, m_real);
#pragma unroll
    for (int u = 0; u < kWtSteps; ++u)
      if ((uint32_t)u < w) S::fma(sp[u * 32], xv[u], acc, vmask);
#else
    for (uint32_t q = 0; q < w; q += K) {
      uint32_t wv[K], xv[K];
      if (q + K <= w) {
#pragma unroll
        for (int u = 0; u < K; ++u) wv[u] = sp[(q + u) * 32u];
      } else {
#pragma unroll
        for (int u = 0; u < K; ++u) wv[u] = q + u < w ? sp[(q + u) * 32u] : 0u;
      }
#pragma unroll
      for (int u = 0; u < K; ++u) xv[u] = S::gather(wv[u], c2, x, m_real);
#pragma unroll
      for (int u = 0; u < K; ++u) S::fma(wv[u], xv[u], acc, vmask);
    }
#endif
    // every lane has read the slot and the offsets of slice +2 (requested an iteration
    // ago) have landed: refill the slot with that slice
    cp_async_wait_group1();
    __syncwarp();
    if (k + 2u * ws < ns) issue(sl, (it + 2u) & 3u);
    if (rs < n_rows) {
      XT yv;
      if constexpr (sizeof(XT) == 2) yv = __float2half_rn(acc);
      else yv = acc;
      static_cast<XT*>(a.y)[o] = yv;
      if constexpr (DOT) dotv += (double)pv * (double)to_f<XT>(yv);
    }
  }
  cp_async_wait_all();
  finish_dot<DOT>(a, dotv);
}

// the wide TMA kernel for slices of <= 32 steps instead of the dual kernel (PSELL_WIDE=1, A/B;
// off by default).  27-point 256^3 fp16 / f16 x (profiles/r02/wide_ab*.txt): 8-step chunks
// 374 us, 16-step 357 us, all 32 gathers in flight with the words re-read from the slot
// 433 us, against the dual kernel's 324-342 us; bitwise equal.  ncu (8-step): 78 % L1 hits
// on the gathers (dual 41 %) but 24 resident warps instead of 48 -- the FMAs wait on the
// gathers (55 % of stall samples), and the staging's shared memory is what caps the warps.
static bool wide_tma() {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_WIDE", v)) return v != 0;
  return false;
}

static unsigned wide_grid(long long n_slices) {  // persistent: one warp per slice at most
  const long long need = ceil_div(n_slices, kWarpsPerCta);
  const long long cap = (long long)sm_count() * PSELL_WIDE_CTAS;
  return (unsigned)(need < cap ? need : cap);
}

template <int CODEC, typename XT, bool DOT, int PB>
static void launch_wide_pb(const SpmvArgs& a, cudaStream_t st) {
  static bool attr = false;  // idempotent attributes, benign race
  if (!attr) {
    cudaFuncSetAttribute(spmv_wide_tma_kernel<CODEC, XT, DOT, PB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kWtSmemBytes);
    cudaFuncSetAttribute(spmv_wide_tma_kernel<CODEC, XT, DOT, PB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kWtSmemBytes);
    attr = true;
  }
  const unsigned g = wide_grid(a.n_slices);
  const bool p2 = (a.se & (a.se - 1)) == 0 && (a.sigma & (a.sigma - 1)) == 0;  // power-of-two blocks
  if (p2) spmv_wide_tma_kernel<CODEC, XT, DOT, PB, true><<<g, kBlock, kWtSmemBytes, st>>>(a);
  else spmv_wide_tma_kernel<CODEC, XT, DOT, PB, false><<<g, kBlock, kWtSmemBytes, st>>>(a);
}

template <int CODEC, typename XT, bool DOT>
static void launch_wide(const SpmvArgs& a, cudaStream_t st) {
  if (a.mode != PSELL_MODE_IMPLICIT) launch_wide_pb<CODEC, XT, DOT, 0>(a, st);
  else if (a.perm_bytes == 1) launch_wide_pb<CODEC, XT, DOT, 1>(a, st);
  else launch_wide_pb<CODEC, XT, DOT, 2>(a, st);
}

// ---- staged dual kernel (PSELL_DSTAGE=1, A/B): the dual kernel's pair of slices per warp
// and its grid, with each 8-step chunk of both slices brought into a per-warp shared-memory
// stage by two cp.async.bulk copies (1 KB each, elected lane, mbarrier) TWO chunks ahead of
// its decode, so a chunk costs one L2 round trip (the x gathers) instead of two (the word
// loads, then the gathers), at the dual kernel's full residency (2 x 2 KB of stages per
// warp: 6 CTAs x 8 warps per SM).  Same FMAs in the same order: bitwise the dual kernel.
constexpr int kDsU = 8;
constexpr int kDsChunkWords = kDsU * 32;  // one slice's chunk, 1 KB
constexpr size_t kDsSmemBytes = kWarpsPerCta * (2 * 2 * kDsChunkWords * 4 + 2 * 8);
template <int CODEC, typename XT, bool DOT, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) spmv_dual_stage_kernel(const SpmvArgs a) {
  using S = NarrowStep<CODEC, XT>;
  if constexpr (DOT) {
    if (a.skip && *a.skip) return;
  }
  extern __shared__ __align__(128) unsigned char ds_smem[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  uint32_t* stages = reinterpret_cast<uint32_t*>(ds_smem) + warp * 4 * kDsChunkWords;  // [2][A, B][256]
  uint64_t* bars = reinterpret_cast<uint64_t*>(ds_smem + kWarpsPerCta * 4 * kDsChunkWords * 4) + warp * 2;
  double dotv = 0.0;
  const long long wg = (long long)blockIdx.x * kWarpsPerCta + warp;
  const long long kA = 2 * wg, kB = kA + 1;
  if (kA < a.n_slices) {
    const bool hasB = kB < a.n_slices;
    const long long oA = a.offset[kA], oB = a.offset[kA + 1];
    const long long oE = hasB ? a.offset[kB + 1] : oB;
    const int wA = (int)((oB - oA) >> 5), wB = (int)((oE - oB) >> 5);
    const uint32_t* __restrict__ pack = static_cast<const uint32_t*>(a.pack);
    const XT* __restrict__ x = static_cast<const XT*>(a.x);
    const uint32_t m_real = CODEC == PSELL_FP16 ? 0xFFFEu : ((2u << a.d) - 2u);
    const uint32_t vmask = CODEC == PSELL_FP16 ? 0u : ~((2u << a.d) - 1u);
    const uint32_t se = (uint32_t)a.se, kl = (uint32_t)a.k_left;
    const uint32_t cmax = a.n_cols > 0 ? (uint32_t)(a.n_cols - 1) : 0u;
    if (lane == 0) {
      mbar_init(bars, 1);
      mbar_init(bars + 1, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // shared-window addresses computed once (not per chunk)
    const uint32_t stage_u32 = smem_u32(stages), bar_u32 = smem_u32(bars);
    // chunk c of both slices into stage st (warp-uniform operands, one elected lane)
    auto issue = [&](uint32_t st, int c) {
      const int rA = wA - c * kDsU, rB = wB - c * kDsU;
      const uint32_t nA = rA <= 0 ? 0u : rA >= kDsU ? (uint32_t)kDsU : (uint32_t)rA;
      const uint32_t nB = rB <= 0 ? 0u : rB >= kDsU ? (uint32_t)kDsU : (uint32_t)rB;
      const uint32_t bA = nA * 128u, bB = nB * 128u;
      uint32_t* sA = stages + st * 2 * kDsChunkWords;
      // steps past a slice's end read as 0 words (no-ops: no cursor move, FMA predicated off),
      // so every chunk decodes unpredicated; each lane zeroes its own column, the only one it reads
#pragma unroll
      for (int u = 0; u < kDsU; ++u) {
        if ((uint32_t)u >= nA) sA[u * 32 + lane] = 0u;
        if ((uint32_t)u >= nB) sA[kDsChunkWords + u * 32 + lane] = 0u;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile(
          "{\n .reg .pred e, pa, pb;\n elect.sync _|e, 0xffffffff;\n"
          " setp.ne.and.u32 pa, %2, 0, e;\n setp.ne.and.u32 pb, %3, 0, e;\n"
          " @e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%4], %5;\n"
          " @pa cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%6], %2, [%4], %8;\n"
          " @pb cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%1], [%7], %3, [%4], %8;\n}"
          ::"r"(stage_u32 + st * (2 * kDsChunkWords * 4)), "r"(stage_u32 + st * (2 * kDsChunkWords * 4) + kDsChunkWords * 4),
            "r"(bA), "r"(bB), "r"(bar_u32 + st * 8u),
          "r"(bA + bB), "l"(pack + oA + c * kDsChunkWords), "l"(pack + oB + c * kDsChunkWords),
          "l"(policy_evict_first())
          : "memory");
    };
    const int wmax = wA > wB ? wA : wB;
    const int nch = (wmax + kDsU - 1) / kDsU;
    if (nch > 0) issue(0, 0);
    if (nch > 1) issue(1, 1);
    auto base2 = [&](long long k) -> uint32_t {
      const uint32_t g = (uint32_t)a.row0 + (uint32_t)(k * 32) + lane;
      const uint32_t blk = se == 1u ? g : fast_div(g, a.se_m, a.se_l) * se;
      const uint32_t d = blk > kl ? blk - kl : 0u;
      return 2u * (d < cmax ? d : cmax);
    };
    uint32_t cA = base2(kA), cB = base2(kB);
    float accA = 0.f, accB = 0.f;
    for (int c = 0; c < nch; ++c) {
      const uint32_t st = (uint32_t)c & 1u;
      asm volatile(
          "{\n .reg .pred p;\n WAIT_%=:\n"
          " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          " @!p bra WAIT_%=;\n}" ::"r"(bar_u32 + st * 8u), "r"(((uint32_t)c >> 1) & 1u)
          : "memory");
      const uint32_t* sa = stages + st * 2 * kDsChunkWords + lane;
      const uint32_t* sb = sa + kDsChunkWords;
      uint32_t xa[kDsU], xb[kDsU];
      {  // the stage is zero-padded past each slice's end: no predicates
        uint32_t wa[kDsU], wb[kDsU];
#pragma unroll
        for (int u = 0; u < kDsU; ++u) {
          wa[u] = sa[u * 32];
          wb[u] = sb[u * 32];
        }
#pragma unroll
        for (int u = 0; u < kDsU; ++u) {
          xa[u] = S::gather(wa[u], cA, x, m_real);
          xb[u] = S::gather(wb[u], cB, x, m_real);
        }
#pragma unroll
        for (int u = 0; u < kDsU; ++u) {
          S::fma(wa[u], xa[u], accA, vmask);
          S::fma(wb[u], xb[u], accB, vmask);
        }
      }
      __syncwarp();  // every lane has read stage st: refill it two chunks on
      if (c + 2 < nch) issue(st, c + 2);
    }
    const uint32_t sig = (uint32_t)a.sigma;
    const uint32_t nr = (uint32_t)a.n_rows;
    auto out_row = [&](long long k) -> uint32_t {
      const uint32_t s = (uint32_t)(k * 32) + lane;
      if (a.mode != PSELL_MODE_IMPLICIT) return s;
      const uint32_t sc = s < nr ? s : nr - 1u;
      const uint32_t pp = a.perm_bytes == 1 ? (uint32_t)__ldg(static_cast<const uint8_t*>(a.perm) + sc)
                                            : (uint32_t)__ldg(static_cast<const uint16_t*>(a.perm) + sc);
      return fast_div((uint32_t)(k * 32), a.sig_m, a.sig_l) * sig + pp;
    };
    auto flush = [&](long long k, float acc) {
      const uint32_t s = (uint32_t)(k * 32) + lane;
      const uint32_t o = out_row(k);
      if ((long long)s < a.n_rows) {
        XT yv;
        if constexpr (sizeof(XT) == 2) yv = __float2half_rn(acc);
        else yv = acc;
        static_cast<XT*>(a.y)[o] = yv;
        if constexpr (DOT) dotv += (double)a.p_own[o] * (double)to_f<XT>(yv);
      }
    };
    flush(kA, accA);
    if (hasB) flush(kB, accB);
  }
  finish_dot<DOT>(a, dotv);
}

static bool dual_stage() {  // PSELL_DSTAGE=1: the staged dual kernel (A/B)
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_DSTAGE", v)) return v != 0;
  return false;
}

static int dual_stage_minb() {  // PSELL_DSTAGE=1: 6 CTAs/SM (40 registers), 2: 5 (48 registers)
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_DSTAGE", v)) return v == 2 ? 5 : 6;
  return 6;
}

template <int CODEC, typename XT, bool DOT>
static void launch_dual_stage(const SpmvArgs& a, cudaStream_t st, unsigned grid) {
  static bool attr = false;  // idempotent attributes, benign race
  if (!attr) {
    cudaFuncSetAttribute(spmv_dual_stage_kernel<CODEC, XT, DOT, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kDsSmemBytes);
    cudaFuncSetAttribute(spmv_dual_stage_kernel<CODEC, XT, DOT, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kDsSmemBytes);
    attr = true;
  }
  if (dual_stage_minb() == 5) spmv_dual_stage_kernel<CODEC, XT, DOT, 5><<<grid, kBlock, kDsSmemBytes, st>>>(a);
  else spmv_dual_stage_kernel<CODEC, XT, DOT, 6><<<grid, kBlock, kDsSmemBytes, st>>>(a);
}

// word staging of the narrow kernel (PSELL_NARROW_TMA=0: words loaded per lane from global
// memory, A/B).  7-point 256^3 e8m14 / f32 x: 124.9 vs 137.3 us; fp16 / f16 x 116.1 vs
// 128.9 us; fused p.q 134.5 vs 139.5 us (profiles/r02/narrow_tma_ab.txt)
static bool narrow_tma() {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_NARROW_TMA", v)) return v != 0;
  return true;
}

// slot kernel for narrow slices instead of the persistent pair kernel (PSELL_SLOT=1: on, A/B).
// Off by default: 7-point 256^3 e8m14 / f32 x 156-160 us at 6 CTAs/SM (40 registers,
// 52-92 B of spills; ncu: long-scoreboard stalls per issue 13.4 -> 9.7, eligible warps
// 1.5 -> 2.0, but 21 % more instructions) and 147 us at 5 CTAs/SM (48 registers, no
// spills in the plain kernel) against the pair kernel's 146 us (scripts/slot_ab.py).
template <int CODEC, typename XT, bool DOT, int PB>
static void launch_narrow_tma(const SpmvArgs& a, cudaStream_t st, unsigned g) {
  static bool attr = false;  // idempotent attributes, benign race
  if (!attr) {
    cudaFuncSetAttribute(spmv_narrow_tma_kernel<CODEC, XT, DOT, PB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kNtSmemBytes);
    cudaFuncSetAttribute(spmv_narrow_tma_kernel<CODEC, XT, DOT, PB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kNtSmemBytes);
    attr = true;
  }
  const bool p2 = (a.se & (a.se - 1)) == 0 && (a.sigma & (a.sigma - 1)) == 0;  // power-of-two blocks
  if (p2) spmv_narrow_tma_kernel<CODEC, XT, DOT, PB, true><<<g, kBlock, kNtSmemBytes, st>>>(a);
  else spmv_narrow_tma_kernel<CODEC, XT, DOT, PB, false><<<g, kBlock, kNtSmemBytes, st>>>(a);
}

static bool slot_kernel() {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_SLOT", v)) return v != 0;
  return false;
}

template <int CODEC, typename XT, bool DOT>
static void launch_slot(const SpmvArgs& a, cudaStream_t st, unsigned grid) {
  static bool attr = false;  // idempotent attribute, benign race
  if (!attr) {
    cudaFuncSetAttribute(spmv_slot_kernel<CODEC, XT, DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSlotSmemBytes);
    attr = true;
  }
  spmv_slot_kernel<CODEC, XT, DOT><<<grid, kBlock, kSlotSmemBytes, st>>>(a);
}

static int sm_count();

template <int CODEC, typename XT, bool DOT>
static void launch_tile(const SpmvArgs& a, cudaStream_t st) {
  static bool attr = false;  // idempotent attribute, benign race
  if (!attr) {
    cudaFuncSetAttribute(spmv_tile_kernel<CODEC, XT, DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kTileSmemBytes);
    attr = true;
  }
  const long long n_tiles = ceil_div(a.n_slices, kTileSlices);
  const long long cap = (long long)sm_count() * kTileCtasPerSm;
  const unsigned g = (unsigned)(n_tiles < cap ? n_tiles : cap);
  spmv_tile_kernel<CODEC, XT, DOT><<<g, kTileThreads, kTileSmemBytes, st>>>(a);
}

// tile-TMA kernel for narrow slices instead of the persistent pair kernel (PSELL_TILE=1, A/B)
static bool tile_kernel() {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_TILE", v)) return v != 0;
  return false;
}

static int sm_count() {  // per device, queried once
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

// grid of the C = 32 launch: persistent for the TMA ring, one warp per slice otherwise
static long long spmv_grid(long long n_slices, int c, bool tma) {
  if (c != 32) return 0;
  const long long full = ceil_div(n_slices, kWarps);
  if (!tma) return full;
  const long long cap = (long long)sm_count() * kTmaCtasPerSm;
  return full < cap ? full : cap;
}

// ---- generic C: thread per storage row, slice k = s / C
template <int CODEC, typename XT, bool REF, bool DOT>
__global__ void __launch_bounds__(kBlock) spmv_generic_kernel(const SpmvArgs a) {
  using W = typename WordOf<CODEC>::T;
  using A = Acc<XT, REF>;
  if constexpr (DOT) {
    if (a.skip && *a.skip) return;
  }
  const long long s = (long long)blockIdx.x * kBlock + threadIdx.x;
  double dotv = 0.0;
  if (s < a.n_rows) {
    const long long k = s / a.c;
    const long long lane = s - k * a.c;
    const long long o0 = a.offset[k];
    const long long width = (a.offset[k + 1] - o0) / a.c;
    const W* p = static_cast<const W*>(a.pack) + o0 + lane;
    const XT* __restrict__ x = static_cast<const XT*>(a.x);
    const uint64_t pol_x = policy_evict_last();
    const int dbits = word_dbits<CODEC>(a.d);
    long long cursor = storage_base(a.row0 + s, a.se, a.k_left, a.n_cols);
    typename A::T acc = A::zero();
    for (long long q = 0; q < width; ++q) {
      const W w = p[q * a.c];
      cursor += (long long)unpack_delta<W>(w, dbits);
      const XT xv = ld_keep(x + cursor, pol_x);
      acc = A::template step<CODEC, W>(acc, w, a.d, xv);
    }
    const long long o = out_row(a, s);
    const XT yv = A::out(acc);
    static_cast<XT*>(a.y)[o] = yv;
    if constexpr (DOT) dotv = (double)a.p_own[o] * (double)to_f<XT>(yv);
  }
  finish_dot<DOT>(a, dotv);
}

template <int CODEC, typename XT, bool DOT, int PB>
static void launch_narrow_tma(const SpmvArgs& a, cudaStream_t st, unsigned g);
template <int CODEC, typename XT, bool DOT, int PB>
static void launch_narrow_pb(const SpmvArgs& a, cudaStream_t st) {
  const unsigned g = narrow_grid(a.n_slices);
  if (narrow_tma()) {
    launch_narrow_tma<CODEC, XT, DOT, PB>(a, st, g);
    return;
  }
  switch (narrow_minb()) {
    case 5: spmv_narrow_kernel<CODEC, XT, DOT, PB, 5><<<g, kBlock, 0, st>>>(a); break;
    default: spmv_narrow_kernel<CODEC, XT, DOT, PB, 4><<<g, kBlock, 0, st>>>(a); break;
  }
}
template <int CODEC, typename XT, bool DOT>
static void launch_narrow(const SpmvArgs& a, cudaStream_t st) {
  if constexpr (CODEC == PSELL_FP32EMBED) return;
  else if (a.mode != PSELL_MODE_IMPLICIT) launch_narrow_pb<CODEC, XT, DOT, 0>(a, st);
  else if (a.perm_bytes == 1) launch_narrow_pb<CODEC, XT, DOT, 1>(a, st);
  else launch_narrow_pb<CODEC, XT, DOT, 2>(a, st);
}

template <int CODEC, typename XT, bool REF, bool DOT, bool GR = false>
static void launch_spmv(const SpmvArgs& a, cudaStream_t st) {
  if (a.c == 32) {
    const long long rows = a.n_slices * 32;
    const unsigned grid = (unsigned)ceil_div(rows, kBlock);
    constexpr int U = sizeof(typename WordOf<CODEC>::T) == 4 ? 8 : 4;
    if constexpr (!REF && FastPolicy<CODEC, XT>::kHave) {
      if (a.variant != 2) {
        {
          const int nt = fast_nt();
          const unsigned gnt = (unsigned)ceil_div(rows, nt);
          const unsigned gd = (unsigned)ceil_div(ceil_div(a.n_slices, 2), kWarpsPerCta);
          const int du = dual_chunk(a.narrow);
          if (a.narrow && tile_kernel()) {
            launch_tile<CODEC, XT, DOT>(a, st);
          } else if (a.narrow12 && a.seg_len == 0 && narrow_on()) {
            launch_narrow<CODEC, XT, DOT>(a, st);
          } else if (a.w32 && !a.narrow && a.seg_len == 0 && wide_tma()) {
            launch_wide<CODEC, XT, DOT>(a, st);
          } else if (dual_slices(a.n_slices) && a.narrow && pair_kernel()) {
            const int pn = pair_nt(DOT);
            const unsigned gp = (unsigned)ceil_div(ceil_div(a.n_slices, 2), pn / 32);
            const unsigned gpp = pair_persist_grid(a.n_slices, DOT);
            if (gpp && slot_kernel() && a.narrow12 && a.seg_len == 0) launch_slot<CODEC, XT, DOT>(a, st, gpp);
            else if (gpp) spmv_pair_kernel<CODEC, XT, DOT, PSELL_PAIR_U, true, kBlock, true><<<gpp, kBlock, 0, st>>>(a);
            else if (pn == 64) spmv_pair_kernel<CODEC, XT, DOT, 12, true, 64><<<gp, 64, 0, st>>>(a);
            else if (pn == 128) spmv_pair_kernel<CODEC, XT, DOT, 12, true, 128><<<gp, 128, 0, st>>>(a);
            else spmv_pair_kernel<CODEC, XT, DOT, 12, true><<<gd, kBlock, 0, st>>>(a);
          } else if (dual_slices(a.n_slices) && pair_wide()) {
            spmv_pair_kernel<CODEC, XT, DOT, 8, false><<<gd, kBlock, 0, st>>>(a);
          } else if (dual_slices(a.n_slices) && !a.narrow && a.seg_len == 0 && dual_stage()) {
            launch_dual_stage<CODEC, XT, DOT>(a, st, gd);
          } else if (dual_slices(a.n_slices) && du == 12)
            spmv_dual_kernel<CODEC, XT, DOT, 12><<<gd, kBlock, 0, st>>>(a);
          else if (dual_slices(a.n_slices))
            spmv_dual_kernel<CODEC, XT, DOT, 8, GR><<<gd, kBlock, 0, st>>>(a);
          else if (nt == 64) spmv_fast_kernel<CODEC, XT, DOT, 8, 64><<<gnt, 64, 0, st>>>(a);
          else if (nt == 128) spmv_fast_kernel<CODEC, XT, DOT, 8, 128><<<gnt, 128, 0, st>>>(a);
          else spmv_fast_kernel<CODEC, XT, DOT, 8, 256><<<gnt, 256, 0, st>>>(a);
        }
      } else {
        static bool carveout = false;  // idempotent attribute, benign race
        if (!carveout) {
          cudaFuncSetAttribute(spmv_stream_kernel<CODEC, XT, DOT>,
                               cudaFuncAttributePreferredSharedMemoryCarveout, 100);
          carveout = true;
        }
        const unsigned g = (unsigned)spmv_grid(a.n_slices, 32, true);
        spmv_stream_kernel<CODEC, XT, DOT><<<g, kBlock, 0, st>>>(a);
      }
    } else
      spmv_c32_kernel<CODEC, XT, REF, DOT, U><<<grid, kBlock, 0, st>>>(a);
  } else {
    const unsigned grid = (unsigned)ceil_div(a.n_rows, kBlock);
    spmv_generic_kernel<CODEC, XT, REF, DOT><<<grid, kBlock, 0, st>>>(a);
  }
}

template <int CODEC, typename XT>
static void dispatch_ref(const SpmvArgs& a, bool ref, cudaStream_t st) {
  if (ref) launch_spmv<CODEC, XT, true, false>(a, st);
  else launch_spmv<CODEC, XT, false, false>(a, st);
}

template <int CODEC>
static int dispatch_x(const SpmvArgs& a, int xdt, bool ref, cudaStream_t st) {
  switch (xdt) {
    case PSELL_DT_F16: dispatch_ref<CODEC, __half>(a, ref, st); return 0;
    case PSELL_DT_F32: dispatch_ref<CODEC, float>(a, ref, st); return 0;
    case PSELL_DT_F64: dispatch_ref<CODEC, double>(a, ref, st); return 0;
  }
  return 1;
}

static int make_args(const psell_desc* d, const void* pack, const int64_t* offset,
                     const void* perm, SpmvArgs& a, psell_error* err, bool need_perm = true) {
  if (!d) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "null descriptor");
  if (!fmt_valid(fmt_of(d))) return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, "invalid PackFormat");
  if (!fmt_device_ok(fmt_of(d))) return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, PSELL_FP16_W64_MSG);
  if (d->c < 1) return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, "invalid C");
  if (need_perm && d->mode == PSELL_MODE_IMPLICIT && d->n_rows > 0 && (!perm || d->sigma < 1))
    return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "implicit mode needs perm");
  if (d->n_cols >= (1ll << 31) || d->n_rows >= (1ll << 31))
    return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "dimensions exceed 32-bit indexing");
  a.pack = pack;
  a.offset = offset;
  a.perm = perm;
  a.x = nullptr;
  a.y = nullptr;
  a.p_own = nullptr;
  a.partials = nullptr;
  a.skip = nullptr;
  a.ticket = nullptr;
  a.scal = nullptr;
  a.iflags = nullptr;
  a.peers = nullptr;
  a.peer_G = 1;
  a.peer_rank = 0;
  a.peer_timeout = 0;
  a.sched = nullptr;
  a.aff_chunks = 0;
  a.n_rows = d->n_rows;
  a.n_cols = d->n_cols;
  a.n_slices = ceil_div(d->n_rows, d->c);
  a.row0 = d->row0;
  a.k_left = d->k_left < 0 ? 0 : d->k_left;
  a.c = d->c;
  a.se = d->mode == PSELL_MODE_NONE ? 1 : d->sigma;
  a.sigma = d->sigma;
  a.mode = d->mode;
  a.d = d->d;
  a.perm_bytes = d->sigma <= 256 ? 1 : 2;
  a.variant = 0;
  a.narrow = 0;
  a.narrow12 = 0;
  a.w32 = 0;
  a.codec = d->codec;
  a.seg_len = 0;
  a.seg_slice = a.seg_q0 = a.long_slice = a.long_seg0 = nullptr;
  a.seg_c2 = nullptr;
  a.seg_partial = nullptr;
  magic_div((uint32_t)(a.se > 0 ? a.se : 1), a.se_m, a.se_l);
  magic_div((uint32_t)(a.sigma > 0 ? a.sigma : 1), a.sig_m, a.sig_l);
  a.l2pf = 1;
  a.sched_static = 0;
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_L2PF", v)) a.l2pf = v;
  return PSELL_OK;
}

// ---------------------------------------------------------------- K5 decode
__device__ __forceinline__ long long raw_base(long long s_global, int se, long long k_left) {
  const long long blk = (s_global / se) * se;
  return blk > k_left ? blk - k_left : 0;
}

template <typename W>
__global__ void to_csr_count_kernel(const SpmvArgs a, long long* __restrict__ counts) {
  const long long s = (long long)blockIdx.x * kBlock + threadIdx.x;
  if (s >= a.n_rows) return;
  const long long k = s / a.c, lane = s - k * a.c;
  const long long o0 = a.offset[k];
  const long long width = (a.offset[k + 1] - o0) / a.c;
  const W* p = static_cast<const W*>(a.pack) + o0 + lane;
  long long cnt = 0;
  for (long long q = 0; q < width; ++q) cnt += (long long)(p[q * a.c] & W(1));
  counts[out_row(a, s)] = cnt;
}

template <int CODEC>
__global__ void to_csr_fill_kernel(const SpmvArgs a, const int64_t* __restrict__ row_ptr,
                                   int32_t* __restrict__ col_idx, double* __restrict__ values) {
  using W = typename WordOf<CODEC>::T;
  const long long s = (long long)blockIdx.x * kBlock + threadIdx.x;
  if (s >= a.n_rows) return;
  const long long k = s / a.c, lane = s - k * a.c;
  const long long o0 = a.offset[k];
  const long long width = (a.offset[k + 1] - o0) / a.c;
  const W* p = static_cast<const W*>(a.pack) + o0 + lane;
  const int dbits = word_dbits<CODEC>(a.d);
  long long cursor = raw_base(a.row0 + s, a.se, a.k_left);  // unclamped (packed.py:285-288)
  long long t = row_ptr[out_row(a, s)];
  for (long long q = 0; q < width; ++q) {
    const W w = p[q * a.c];
    cursor += (long long)unpack_delta<W>(w, dbits);
    if (w & W(1)) {
      col_idx[t] = (int32_t)cursor;
      values[t] = (double)word_value<CODEC, W>(w, a.d);
      ++t;
    }
  }
}

// Largest column a real word of the stream addresses, over every storage row the
// SpMV walks (padding rows of the last slice included), starting from the SpMV's
// clamped cursor (packed.py:257).  A container whose deltas run past n_cols would
// make the SpMV gather out of bounds: read_psell rejects it with this value.
template <int CODEC>
__global__ void max_column_kernel(const SpmvArgs a, long long n_storage, unsigned long long* __restrict__ out) {
  using W = typename WordOf<CODEC>::T;
  const long long s = (long long)blockIdx.x * kBlock + threadIdx.x;
  long long m = -1;
  if (s < n_storage) {
    const long long k = s / a.c, lane = s - k * a.c;
    const long long o0 = a.offset[k];
    const long long width = (a.offset[k + 1] - o0) / a.c;
    const W* p = static_cast<const W*>(a.pack) + o0 + lane;
    const int dbits = word_dbits<CODEC>(a.d);
    long long cursor = raw_base(a.row0 + s, a.se, a.k_left);
    cursor = a.n_cols > 0 ? (cursor < a.n_cols - 1 ? cursor : a.n_cols - 1) : 0;
    for (long long q = 0; q < width; ++q) {
      const W w = p[q * a.c];
      const unsigned long long dl = (unsigned long long)unpack_delta<W>(w, dbits);
      // saturate instead of wrapping on absurd deltas
      cursor = dl > (unsigned long long)(LLONG_MAX / 2) || cursor > LLONG_MAX / 2 ? LLONG_MAX / 2
                                                                                  : cursor + (long long)dl;
      if ((w & W(1)) && cursor > m) m = cursor;
    }
  }
  m = warp_max_ll(m);
  if ((threadIdx.x & 31) == 0 && m >= 0) atomicMax(out, (unsigned long long)m);
}

}  // namespace psell

using namespace psell;

extern "C" {

int psell_max_column(const psell_desc* d, const void* pack, const int64_t* offset, const void* perm,
                     int64_t* out_host, void* ws8, void* stream, psell_error* err) {
  SpmvArgs a;
  if (int rc = make_args(d, pack, offset, perm, a, err)) return rc;
  if (!ws8 || !out_host) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "missing workspace");
  cudaStream_t st = as_stream(stream);
  unsigned long long* dm = static_cast<unsigned long long*>(ws8);
  PSELL_CUDA(cudaMemsetAsync(dm, 0, 8, st), err);
  const long long n_storage = a.n_slices * a.c;
  unsigned long long any = 0;
  if (n_storage > 0) {
    const unsigned grid = (unsigned)ceil_div(n_storage, kBlock);
    switch (d->codec) {
      case PSELL_FP16: max_column_kernel<PSELL_FP16><<<grid, kBlock, 0, st>>>(a, n_storage, dm); break;
      case PSELL_E8MY: max_column_kernel<PSELL_E8MY><<<grid, kBlock, 0, st>>>(a, n_storage, dm); break;
      default: max_column_kernel<PSELL_FP32EMBED><<<grid, kBlock, 0, st>>>(a, n_storage, dm); break;
    }
    PSELL_CHECK_LAUNCH(err, "max_column");
  }
  // 0 is both "no real word" and "column 0": one more pass would tell them apart, but
  // column 0 is in range whenever n_cols > 0, which is all the caller checks
  PSELL_CUDA(cudaMemcpyAsync(&any, dm, 8, cudaMemcpyDeviceToHost, st), err);
  PSELL_CUDA(cudaStreamSynchronize(st), err);
  *out_host = (int64_t)any;
  return ok(err);
}


int psell_spmv(const psell_desc* d, const void* pack, const int64_t* offset, const void* perm,
               const void* x, int32_t x_dtype, void* y, int32_t flags, void* stream,
               psell_error* err) {
  SpmvArgs a;
  if (int rc = make_args(d, pack, offset, perm, a, err)) return rc;
  a.x = x;
  a.y = y;
  if (a.n_rows == 0) return ok(err);
  cudaStream_t st = as_stream(stream);
  const bool ref = (flags & PSELL_SPMV_REF_ORDER) != 0;
  a.variant = (flags & PSELL_SPMV_TMA_STREAM) ? 2 : 0;
  a.narrow = (flags & PSELL_SPMV_NARROW) != 0;
  a.narrow12 = a.narrow && (flags & PSELL_SPMV_NARROW12) != 0;
  a.w32 = (flags & PSELL_SPMV_W32) != 0;
  int bad = 1;
  switch (d->codec) {
    case PSELL_FP16: bad = dispatch_x<PSELL_FP16>(a, x_dtype, ref, st); break;
    case PSELL_E8MY: bad = dispatch_x<PSELL_E8MY>(a, x_dtype, ref, st); break;
    case PSELL_FP32EMBED: bad = dispatch_x<PSELL_FP32EMBED>(a, x_dtype, ref, st); break;
  }
  if (bad) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "unsupported x dtype");
  PSELL_CHECK_LAUNCH(err, "psell_spmv");
  return ok(err);
}

const char* psell_spmv_kernel_name(const psell_desc* d, int32_t x_dtype, int32_t flags) {
  if (!d || d->n_rows <= 0) return "none";
  const bool ref = (flags & PSELL_SPMV_REF_ORDER) != 0;
  const bool fast = !ref && d->codec != PSELL_FP32EMBED && x_dtype != PSELL_DT_F64;
  if (d->c != 32) return "spmv_generic_kernel";
  if (!fast) return "spmv_c32_kernel";
  if (flags & PSELL_SPMV_TMA_STREAM) return "spmv_stream_kernel";
  const long long ns = ceil_div(d->n_rows, d->c);
  if ((flags & PSELL_SPMV_NARROW) && tile_kernel()) return "spmv_tile_kernel (TMA ring)";
  if (!(flags & PSELL_SPMV_NARROW) && (flags & PSELL_SPMV_W32) && wide_tma())
    return "spmv_wide_tma_kernel (next slice's words staged by cp.async.bulk, two-pass decode, persistent)";
  if ((flags & PSELL_SPMV_NARROW) && (flags & PSELL_SPMV_NARROW12) && narrow_on())
    return narrow_tma() ? "spmv_narrow_tma_kernel (pair words staged by cp.async.bulk, two-pass decode, persistent)"
                        : "spmv_narrow_kernel (pipelined pair metadata, two-pass decode, persistent)";
  if (dual_slices(ns) && (flags & PSELL_SPMV_NARROW) && pair_kernel())
    return pair_persist_grid(ns, false) ? (slot_kernel() && (flags & PSELL_SPMV_NARROW12)
                                               ? "spmv_slot_kernel (TMA slot per warp, persistent)"
                                                         : "spmv_pair_kernel<U=12, persistent>")
                                        : "spmv_pair_kernel<U=12>";
  if (dual_slices(ns) && pair_wide()) return "spmv_pair_kernel<U=8>";
  if (dual_slices(ns) && !(flags & PSELL_SPMV_NARROW) && dual_stage())
    return "spmv_dual_stage_kernel (8-step chunks of both slices staged 2 ahead by cp.async.bulk)";
  if (dual_slices(ns)) {
    const int du = dual_chunk((flags & PSELL_SPMV_NARROW) != 0);
    return du == 12 ? "spmv_dual_kernel<U=12>" : "spmv_dual_kernel<U=8>";
  }
  return "spmv_fast_kernel";
}

int psell_spmv_seg_checkpoints(const psell_desc* d, const void* pack, const int64_t* offset,
                               int32_t seg_len, int64_t n_seg, const int32_t* seg_slice,
                               const int32_t* seg_q0, int64_t n_long, const int32_t* long_slice,
                               const int32_t* long_seg0, uint32_t* seg_c2, void* stream,
                               psell_error* err) {
  SpmvArgs a;
  if (int rc = make_args(d, pack, offset, nullptr, a, err, /*need_perm=*/false)) return rc;
  if (d->c != 32 || d->w != 32 || seg_len < 1)
    return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "segmentation needs C = 32, W = 32");
  a.seg_len = seg_len;
  a.seg_slice = seg_slice;
  a.seg_q0 = seg_q0;
  a.seg_c2 = seg_c2;
  a.long_slice = long_slice;
  a.long_seg0 = long_seg0;
  cudaStream_t st = as_stream(stream);
  if (n_seg > 0) seg_dsum_kernel<<<(unsigned)ceil_div(n_seg * 32, kBlock), kBlock, 0, st>>>(a, n_seg);
  if (n_long > 0) seg_prefix_kernel<<<(unsigned)ceil_div(n_long * 32, kBlock), kBlock, 0, st>>>(a, n_long);
  PSELL_CHECK_LAUNCH(err, "psell_spmv_seg_checkpoints");
  return ok(err);
}

}  // extern "C"

namespace psell {
// SM-affine dual kernel for the short slices of an irregular matrix (PSELL_AFF=1: on, A/B;
// PSELL_AFF_CTAS = resident CTAs per SM, default 6).  Off by default: on config 4 it
// raised the L1 hit rate of the x gathers from 26 % to 39 % and cut L2 sectors by 10 %,
// but ran 480-540 us against 366 us (twice the instructions; the claim atomics and the
// end-of-work chunk scan are serial L2 round trips), scripts/c4_aff.py.
static bool aff_on() {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_AFF", v)) return v != 0;
  return false;
}
static int aff_ctas() {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_AFF_CTAS", v) && v >= 1 && v <= 6) return v;
  return 6;
}

// one merged grid for segments + short slices (PSELL_SEGMERGE=0: two launches, A/B)
static bool seg_merge() {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_SEGMERGE", v)) return v != 0;
  return true;
}

// the static SM-affine grid for segmented matrices (default; PSELL_DSTATIC=0: the merged
// segment + dual grid).  Config 4 327.8 -> 275.8 us, 4b 309.2 -> 257.1 us, bitwise
// (profiles/r02/static_ab*.txt): a sigma window's rows per SM keep the x gathers in its L1.
static bool dual_static() {
  static EnvCache c;
  int v;
  if (env_int(c, "PSELL_DSTATIC", v)) return v != 0;
  return true;
}

template <int CODEC, typename XT>
static void launch_segmented(const SpmvArgs& a, long long n_seg, long long n_long, cudaStream_t st) {
  if (a.sched && a.aff_chunks > 0 && dual_static() && !aff_on() && a.n_slices >= 2 && a.sched_static) {
    if (dual_static_nt() == 768)
      spmv_dual_static_kernel<CODEC, XT, 8, 768><<<2u * (unsigned)a.aff_chunks, 768, 0, st>>>(a, n_seg);
    else
      spmv_dual_static_kernel<CODEC, XT, 8, 1024><<<(unsigned)a.aff_chunks, 1024, 0, st>>>(a, n_seg);
    if (n_long > 0)
      seg_combine_kernel<XT><<<(unsigned)ceil_div(n_long * 32, kBlock), kBlock, 0, st>>>(a, n_long);
    return;
  }
  const bool aff = a.sched && a.aff_chunks > 0 && aff_on() && a.n_slices >= 2;
  if (!aff && n_seg > 0 && seg_merge() && dual_slices(a.n_slices) && !a.narrow && dual_chunk(false) == 8 &&
      !pair_wide()) {
    const unsigned seg_ctas = (unsigned)ceil_div(n_seg * 32, kBlock);
    const unsigned gd = (unsigned)ceil_div(ceil_div(a.n_slices, 2), kWarpsPerCta);
    spmv_dual_seg_kernel<CODEC, XT, 8><<<seg_ctas + gd, kBlock, 0, st>>>(a, n_seg, seg_ctas);
    if (n_long > 0)
      seg_combine_kernel<XT><<<(unsigned)ceil_div(n_long * 32, kBlock), kBlock, 0, st>>>(a, n_long);
    return;
  }
  if (aff) {
    const unsigned g = (unsigned)(sm_count() * aff_ctas());
    spmv_dual_kernel<CODEC, XT, false, 8, true, true><<<g, kBlock, 0, st>>>(a);
  } else
    launch_spmv<CODEC, XT, false, false, true>(a, st);  // short slices (long ones are skipped); flag-predicated gathers
  if (n_seg > 0)
    spmv_seg_kernel<CODEC, XT, 8><<<(unsigned)ceil_div(n_seg * 32, kBlock), kBlock, 0, st>>>(a, n_seg);
  if (n_long > 0)
    seg_combine_kernel<XT><<<(unsigned)ceil_div(n_long * 32, kBlock), kBlock, 0, st>>>(a, n_long);
}
}  // namespace psell

extern "C" {

int psell_spmv_segmented(const psell_desc* d, const void* pack, const int64_t* offset, const void* perm,
                         const void* x, int32_t x_dtype, void* y, int32_t seg_len, int64_t n_seg,
                         const int32_t* seg_slice, const int32_t* seg_q0, const uint32_t* seg_c2,
                         float* seg_partial, int64_t n_long, const int32_t* long_slice,
                         const int32_t* long_seg0, uint32_t* sched, int32_t sched_chunks, void* stream,
                         psell_error* err) {
  SpmvArgs a;
  if (int rc = make_args(d, pack, offset, perm, a, err)) return rc;
  a.sched = sched;
  // sched_chunks < 0: sched also carries the static grid's 2 |sched_chunks| + 1 chunk bounds
  a.aff_chunks = sched ? (sched_chunks < 0 ? -sched_chunks : sched_chunks) : 0;
  a.sched_static = sched && sched_chunks < 0 ? 1 : 0;
  if (d->c != 32 || d->codec == PSELL_FP32EMBED || (x_dtype != PSELL_DT_F16 && x_dtype != PSELL_DT_F32))
    return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0,
                   "segmented SpMV: C = 32, fp16/e8my codec, f16/f32 x only");
  a.x = x;
  a.y = y;
  a.seg_len = seg_len;
  a.seg_slice = seg_slice;
  a.seg_q0 = seg_q0;
  a.seg_c2 = const_cast<uint32_t*>(seg_c2);
  a.seg_partial = seg_partial;
  a.long_slice = long_slice;
  a.long_seg0 = long_seg0;
  if (a.n_rows == 0) return ok(err);
  cudaStream_t st = as_stream(stream);
  if (d->codec == PSELL_FP16) {
    if (x_dtype == PSELL_DT_F16) launch_segmented<PSELL_FP16, __half>(a, n_seg, n_long, st);
    else launch_segmented<PSELL_FP16, float>(a, n_seg, n_long, st);
  } else {
    if (x_dtype == PSELL_DT_F16) launch_segmented<PSELL_E8MY, __half>(a, n_seg, n_long, st);
    else launch_segmented<PSELL_E8MY, float>(a, n_seg, n_long, st);
  }
  PSELL_CHECK_LAUNCH(err, "psell_spmv_segmented");
  return ok(err);
}

int64_t psell_spmv_dot_partials(const psell_desc* d, int32_t flags) {
  if (!d || d->n_rows <= 0 || d->c < 1) return 1;
  const long long ns = ceil_div(d->n_rows, d->c);
  if (d->c == 32) {
    // must match launch_spmv<.., DOT=true>: fp16/e8my take the (persistent) pair kernel for
    // narrow slices, the dual kernel otherwise; fp32embed one warp per slice (REF-style kernel)
    if (d->codec != PSELL_FP32EMBED && tile_kernel() && (flags & PSELL_SPMV_NARROW)) {
      const long long n_tiles = ceil_div(ns, kTileSlices);
      const long long cap = (long long)sm_count() * kTileCtasPerSm;
      return n_tiles < cap ? n_tiles : cap;
    }
    if (d->codec != PSELL_FP32EMBED && (flags & PSELL_SPMV_NARROW) && (flags & PSELL_SPMV_NARROW12) && narrow_on())
      return narrow_grid(ns);
    if (d->codec != PSELL_FP32EMBED && !(flags & PSELL_SPMV_NARROW) && (flags & PSELL_SPMV_W32) && wide_tma())
      return wide_grid(ns);
    if (d->codec != PSELL_FP32EMBED && dual_slices(ns) && pair_kernel() && (flags & PSELL_SPMV_NARROW)) {
      if (const unsigned g = pair_persist_grid(ns, true)) return g;
      return ceil_div(ceil_div(ns, 2), pair_nt(true) / 32);
    }
    if (d->codec != PSELL_FP32EMBED && dual_slices(ns)) return ceil_div(ceil_div(ns, 2), kWarpsPerCta);
    if (d->codec != PSELL_FP32EMBED) return ceil_div(ns * 32, fast_nt());
    return ceil_div(ns * 32, kBlock);
  }
  return ceil_div(d->n_rows, kBlock);
}

int psell_spmv_dot(const psell_desc* d, const void* pack, const int64_t* offset, const void* perm,
                   const float* x, float* y, const float* p_own, double* partials,
                   const int32_t* skip_flag, int32_t flags, void* stream, psell_error* err) {
  SpmvArgs a;
  if (int rc = make_args(d, pack, offset, perm, a, err)) return rc;
  a.narrow = (flags & PSELL_SPMV_NARROW) != 0;
  a.narrow12 = a.narrow && (flags & PSELL_SPMV_NARROW12) != 0;
  a.w32 = (flags & PSELL_SPMV_W32) != 0;
  a.x = x;
  a.y = y;
  a.p_own = p_own;
  a.partials = partials;
  a.skip = skip_flag;
  cudaStream_t st = as_stream(stream);
  if (a.n_rows == 0) {
    PSELL_CUDA(cudaMemsetAsync(partials, 0, sizeof(double), st), err);
    return ok(err);
  }
  switch (d->codec) {
    case PSELL_FP16: launch_spmv<PSELL_FP16, float, false, true>(a, st); break;
    case PSELL_E8MY: launch_spmv<PSELL_E8MY, float, false, true>(a, st); break;
    case PSELL_FP32EMBED: launch_spmv<PSELL_FP32EMBED, float, false, true>(a, st); break;
  }
  PSELL_CHECK_LAUNCH(err, "psell_spmv_dot");
  return ok(err);
}

int psell_spmv_dot_alpha(const psell_desc* d, const void* pack, const int64_t* offset, const void* perm,
                         const float* x, float* y, const float* p_own, double* partials, double* scal,
                         int32_t* iflags, unsigned* ticket, int32_t flags, void* stream, psell_error* err) {
  SpmvArgs a;
  if (int rc = make_args(d, pack, offset, perm, a, err)) return rc;
  if (!ticket || !scal || !iflags) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "null scalar state");
  a.narrow = (flags & PSELL_SPMV_NARROW) != 0;
  a.narrow12 = a.narrow && (flags & PSELL_SPMV_NARROW12) != 0;
  a.w32 = (flags & PSELL_SPMV_W32) != 0;
  a.x = x;
  a.y = y;
  a.p_own = p_own;
  a.partials = partials;
  a.skip = iflags;
  a.ticket = ticket;
  a.scal = scal;
  a.iflags = iflags;
  cudaStream_t st = as_stream(stream);
  if (a.n_rows == 0) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "empty operator");
  switch (d->codec) {
    case PSELL_FP16: launch_spmv<PSELL_FP16, float, false, true>(a, st); break;
    case PSELL_E8MY: launch_spmv<PSELL_E8MY, float, false, true>(a, st); break;
    case PSELL_FP32EMBED: launch_spmv<PSELL_FP32EMBED, float, false, true>(a, st); break;
  }
  PSELL_CHECK_LAUNCH(err, "psell_spmv_dot_alpha");
  return ok(err);
}

// psell_spmv_dot_alpha across G ranks: the last CTA all-reduces p.q over the peer arenas
// (K8 protocol, one value) before the alpha step (reference solvers.py:293-299 on a slab)
int psell_spmv_dot_alpha_peer(const psell_desc* d, const void* pack, const int64_t* offset, const void* perm,
                              const float* x, float* y, const float* p_own, double* partials, double* scal,
                              int32_t* iflags, unsigned* ticket, int32_t flags, int32_t G, int32_t rank,
                              const uint64_t* peers, int64_t timeout_ns, void* stream, psell_error* err) {
  SpmvArgs a;
  if (int rc = make_args(d, pack, offset, perm, a, err)) return rc;
  if (!ticket || !scal || !iflags) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "null scalar state");
  a.narrow = (flags & PSELL_SPMV_NARROW) != 0;
  a.narrow12 = a.narrow && (flags & PSELL_SPMV_NARROW12) != 0;
  a.w32 = (flags & PSELL_SPMV_W32) != 0;
  a.x = x;
  a.y = y;
  a.p_own = p_own;
  a.partials = partials;
  a.skip = iflags;
  a.ticket = ticket;
  a.scal = scal;
  a.iflags = iflags;
  if (G < 1 || G > kPeerMax || rank < 0 || rank >= G || (G > 1 && !peers))
    return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "invalid peer group");
  a.peers = reinterpret_cast<const unsigned long long*>(peers);
  a.peer_G = G;
  a.peer_rank = rank;
  a.peer_timeout = timeout_ns;
  cudaStream_t st = as_stream(stream);
  if (a.n_rows == 0) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "empty operator");
  switch (d->codec) {
    case PSELL_FP16: launch_spmv<PSELL_FP16, float, false, true>(a, st); break;
    case PSELL_E8MY: launch_spmv<PSELL_E8MY, float, false, true>(a, st); break;
    case PSELL_FP32EMBED: launch_spmv<PSELL_FP32EMBED, float, false, true>(a, st); break;
  }
  PSELL_CHECK_LAUNCH(err, "psell_spmv_dot_alpha_peer");
  return ok(err);
}

size_t psell_to_csr_workspace_bytes(const psell_desc* d) {
  if (!d) return 0;
  const long long n = d->n_rows > 0 ? d->n_rows : 0;
  return align_up(8 * (size_t)n) + align_up(8 * (size_t)(ceil_div(n, 4096) + 4096 + 1));
}

int psell_to_csr_plan(const psell_desc* d, const void* pack, const int64_t* offset,
                      const void* perm, void* ws, size_t ws_bytes, int64_t* row_ptr,
                      int64_t* nnz_host, void* stream, psell_error* err) {
  SpmvArgs a;
  if (int rc = make_args(d, pack, offset, perm, a, err)) return rc;
  if (ws_bytes < psell_to_csr_workspace_bytes(d) || !ws)
    return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "workspace too small");
  cudaStream_t st = as_stream(stream);
  long long* counts = static_cast<long long*>(ws);
  long long* tmp = reinterpret_cast<long long*>(static_cast<char*>(ws) + align_up(8 * (size_t)a.n_rows));
  if (a.n_rows > 0) {
    const unsigned grid = (unsigned)ceil_div(a.n_rows, kBlock);
    if (d->w == 32) to_csr_count_kernel<uint32_t><<<grid, kBlock, 0, st>>>(a, counts);
    else to_csr_count_kernel<uint64_t><<<grid, kBlock, 0, st>>>(a, counts);
    PSELL_CHECK_LAUNCH(err, "to_csr_count");
  }
  if (int rc = scan_i64(counts, a.n_rows, tmp, reinterpret_cast<long long*>(row_ptr), st, err)) return rc;
  long long nnz = 0;
  PSELL_CUDA(cudaMemcpyAsync(&nnz, row_ptr + a.n_rows, 8, cudaMemcpyDeviceToHost, st), err);
  PSELL_CUDA(cudaStreamSynchronize(st), err);
  *nnz_host = nnz;
  return ok(err);
}

int psell_to_csr_fill(const psell_desc* d, const void* pack, const int64_t* offset,
                      const void* perm, const int64_t* row_ptr, int32_t* col_idx, double* values,
                      void* stream, psell_error* err) {
  SpmvArgs a;
  if (int rc = make_args(d, pack, offset, perm, a, err)) return rc;
  if (a.n_rows == 0) return ok(err);
  cudaStream_t st = as_stream(stream);
  const unsigned grid = (unsigned)ceil_div(a.n_rows, kBlock);
  switch (d->codec) {
    case PSELL_FP16: to_csr_fill_kernel<PSELL_FP16><<<grid, kBlock, 0, st>>>(a, row_ptr, col_idx, values); break;
    case PSELL_E8MY: to_csr_fill_kernel<PSELL_E8MY><<<grid, kBlock, 0, st>>>(a, row_ptr, col_idx, values); break;
    default: to_csr_fill_kernel<PSELL_FP32EMBED><<<grid, kBlock, 0, st>>>(a, row_ptr, col_idx, values); break;
  }
  PSELL_CHECK_LAUNCH(err, "to_csr_fill");
  return ok(err);
}

}  // extern "C"

extern "C" PSELL_API int32_t psell_reload_env(void) {
  g_env_gen.fetch_add(1, std::memory_order_relaxed);
  return 0;
}
