// K1 — CSR -> PackSELL builder on sm_100a.
//
// Replaces build_packsell (reference packed.py:176-239) and the helpers it
// calls: compute_stats().lower_bandwidth (matrix.py:319-349), _leftmost_offsets
// (packed.py:50-52), _stream_layout (packed.py:145-173), row_sort_order
// (sell.py:22-30) and the codec (codec.py:124-224).  Output is byte-identical
// to the reference: pack (every word written, padding = 0), int64 offset,
// u8/u16 perm, k_left, counts.
//
// Pipeline (all device, stream ordered):
//   lower_bandwidth  thread/row, CTA max -> atomicMax          (skipped with k_left override)
//   row_stats        thread/row: stored count = len + #(gap >= 2^D), n_dummy,
//                    min first gap, max gap                   -> layout errors (sync #1)
//   sort_blocks      CTA/sigma-block stable LSD radix sort on (max - count), 4-bit digits,
//                    warp match_any ranks; keys in smem (sigma <= 2048) or L2-resident scratch
//   slice_width      thread/slice: width*C
//   scan_i64         3-kernel reduce-then-scan -> offset                  (sync #2: n_stored)
//   fill             thread/storage row, warp == slice for C = 32: walks its CSR row,
//                    encodes values, emits dummy + real words and zero padding
//                    with coalesced 128 B stores per step; codec errors (sync #3)
#include "psell_internal.cuh"

namespace psell {

struct BuildStats {
  long long k_left;
  long long min_first_gap;
  long long first_gap_row;
  long long max_gap;
  long long n_dummy;
  long long nonfinite_pos;
  long long overflow_pos;
  long long n_long;  // rows listed for the warp-per-row kernels (row_stats, then fill)
};

constexpr int kSortSmemMaxSigma = 2048;
constexpr long long kI64Max = 0x7FFFFFFFFFFFFFFFll;
constexpr long long kI64Min = (-0x7FFFFFFFFFFFFFFFll - 1);

struct BuildWs {
  BuildStats* stats;
  uint32_t* counts;     // n   stored words per original row
  int32_t* order;       // n   storage row -> local original row
  uint32_t* scount;     // n   stored words per storage row
  long long* wwords;    // n_slices  width*C
  long long* scan_tmp;  // scan block sums
  uint32_t* sort_tmp;   // 4n  (only sigma > kSortSmemMaxSigma)
  int32_t* long_rows;   // n   rows longer than kLongRow, walked one warp per row
  size_t bytes;
};

constexpr int kScanTile = 4096;  // 1024 threads x 4

static BuildWs carve(const psell_desc* d, void* base) {
  const int64_t n = d->n_rows;
  const int64_t ns = ceil_div(n, d->c);
  const int64_t nb = ceil_div(ns, kScanTile) + 1;
  BuildWs w{};
  size_t off = 0;
  char* b = static_cast<char*>(base);
  auto take = [&](size_t bytes) {
    char* p = b ? b + off : nullptr;
    off += align_up(bytes);
    return p;
  };
  w.stats = reinterpret_cast<BuildStats*>(take(sizeof(BuildStats)));
  w.counts = reinterpret_cast<uint32_t*>(take(4 * (size_t)n));
  w.order = reinterpret_cast<int32_t*>(take(4 * (size_t)n));
  w.scount = reinterpret_cast<uint32_t*>(take(4 * (size_t)n));
  w.wwords = reinterpret_cast<long long*>(take(8 * (size_t)ns));
  w.scan_tmp = reinterpret_cast<long long*>(take(8 * (size_t)(nb + kScanTile)));
  const bool big = d->mode != PSELL_MODE_NONE && d->sigma > kSortSmemMaxSigma;
  w.sort_tmp = reinterpret_cast<uint32_t*>(take(big ? 16 * (size_t)n : 0));
  w.long_rows = reinterpret_cast<int32_t*>(take(4 * (size_t)n));
  w.bytes = off;
  return w;
}

// storage-row -> original-row order the plan leaves in the workspace (SELL fill reuses it)
const int32_t* build_ws_order(const psell_desc* d, const void* ws) {
  return carve(d, const_cast<void*>(ws)).order;
}

// Eq. 4 base offset of global row g (packed.py:40-52).
constexpr long long kLongRow = 64;  // rows longer than this are walked by a whole warp

// grid of the warp-per-long-row kernels: a resident wave (8 CTAs of 8 warps per SM)
// PSELL_FOLD_KLEFT=0: the separate lower_bandwidth pass before row_stats (A/B)
static bool fold_k_left() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PSELL_FOLD_KLEFT");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static unsigned long_grid() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return (unsigned)(8 * sms);
}

__device__ __forceinline__ long long base_of(long long g, long long se, long long k_left) {
  const long long blk = (g / se) * se;
  return blk > k_left ? blk - k_left : 0;
}

__global__ void init_stats_kernel(BuildStats* s, long long k_left) {
  s->k_left = k_left < 0 ? 0 : k_left;
  s->min_first_gap = kI64Max;
  s->first_gap_row = kI64Max;
  s->max_gap = kI64Min;
  s->n_dummy = 0;
  s->nonfinite_pos = kI64Max;
  s->overflow_pos = kI64Max;
  s->n_long = 0;
}

template <typename T, typename Op>
__device__ __forceinline__ T warp_reduce(T v, Op op) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

struct MaxOp { __device__ long long operator()(long long a, long long b) const { return a > b ? a : b; } };
struct MinOp { __device__ long long operator()(long long a, long long b) const { return a < b ? a : b; } };
struct AddOp { __device__ long long operator()(long long a, long long b) const { return a + b; } };

// CTA reduce then one atomic per CTA (integer => order independent).
template <typename Op>
__device__ __forceinline__ long long cta_reduce(long long v, Op op, long long ident, long long* sh) {
  v = warp_reduce(v, op);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  long long t = ident;
  if (warp == 0) {
    t = lane < (int)(blockDim.x >> 5) ? sh[lane] : ident;
    t = warp_reduce(t, op);
  }
  __syncthreads();
  return t;
}

// matrix.py:334-339 — max over non-empty rows of (i - first column), floor 0.
__global__ void lower_bandwidth_kernel(const int64_t* __restrict__ row_ptr,
                                       const int32_t* __restrict__ col_idx, long long n,
                                       long long row0, BuildStats* st) {
  __shared__ long long sh[32];
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long v = 0;
  if (i < n) {
    const long long b = row_ptr[i];
    if (row_ptr[i + 1] > b) v = (row0 + i) - (long long)col_idx[b];
  }
  v = cta_reduce(v, MaxOp{}, 0ll, sh);
  if (threadIdx.x == 0 && v > 0) atomicMax(&st->k_left, v);
}

// packed.py:145-173 — stored word count per row and the layout error inputs.
// FOLD (k_left not given): the lower bandwidth is reduced in this same pass (matrix.py:334-339:
// max over non-empty rows of i - first column, floor 0) instead of a pass of its own over the
// rows' scattered first columns; only each row's FIRST gap depends on k_left, so this pass
// counts the inner gaps, records the first column in fcol[], and first_gap_fold_kernel adds
// the first gaps once k_left is known.  Same counts, sums, minima and maxima.
template <bool FOLD>
__global__ void row_stats_kernel(const int64_t* __restrict__ row_ptr,
                                 const int32_t* __restrict__ col_idx, long long n, long long row0,
                                 long long se, int d_bits, BuildStats* st,
                                 uint32_t* __restrict__ counts, int32_t* __restrict__ long_rows,
                                 int32_t* __restrict__ fcol) {
  __shared__ long long sh[32];
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long dum = 0, fg = kI64Max, gmax = kI64Min, kl = 0;
  const long long k_left = FOLD ? 0 : st->k_left;
  const long long thr = 1ll << d_bits;
  long long beg = 0, end = 0, first = 0;
  if (i < n) {
    beg = row_ptr[i];
    end = row_ptr[i + 1];
    if (end > beg) {
      first = col_idx[beg];
      if (FOLD) {
        kl = (row0 + i) - first;
        fcol[i] = (int32_t)first;
      } else {
        fg = first - base_of(row0 + i, se, k_left);
      }
    }
  }
  // rows longer than kLongRow entries go to row_stats_long_kernel, one warp each
  // (power-law rows: one thread per row left the kernel waiting on its longest row)
  const bool lng = i < n && end - beg > kLongRow;
  if (i < n && !lng) {
    long long prev = FOLD ? first : base_of(row0 + i, se, k_left);
    for (long long j = FOLD ? beg + 1 : beg; j < end; ++j) {
      const long long col = col_idx[j];
      const long long gap = col - prev;
      prev = col;
      dum += gap >= thr;
      gmax = gap > gmax ? gap : gmax;
    }
    counts[i] = (uint32_t)((end - beg) + dum);
  }
  if (lng) long_rows[atomicAdd(reinterpret_cast<unsigned long long*>(&st->n_long), 1ull)] = (int32_t)i;
  const long long sd = cta_reduce(dum, AddOp{}, 0ll, sh);
  const long long sf = FOLD ? kI64Max : cta_reduce(fg, MinOp{}, kI64Max, sh);
  const long long sg = cta_reduce(gmax, MaxOp{}, kI64Min, sh);
  const long long sk = FOLD ? cta_reduce(kl, MaxOp{}, 0ll, sh) : 0;
  if (threadIdx.x == 0) {
    if (sd) atomicAdd(reinterpret_cast<unsigned long long*>(&st->n_dummy), (unsigned long long)sd);
    if (sf != kI64Max) atomicMin(&st->min_first_gap, sf);
    if (sg != kI64Min) atomicMax(&st->max_gap, sg);
    if (sk > 0) atomicMax(&st->k_left, sk);
  }
}

// FOLD: every non-empty row's first gap (first column - Eq. 4 base with the reduced k_left):
// its dummy added to the row's count and the sum, the minimum first gap, the maximum gap
__global__ void __launch_bounds__(kBlock) first_gap_fold_kernel(const int64_t* __restrict__ row_ptr,
                                                                const int32_t* __restrict__ fcol, long long n,
                                                                long long row0, long long se, int d_bits,
                                                                BuildStats* st, uint32_t* __restrict__ counts) {
  // a resident grid-stride grid, 4 rows per trip with their loads issued together: one set of
  // CTA reductions per CTA (one per 256 rows cost more than the row work)
  constexpr int R = 4;
  __shared__ long long sh[32];
  const long long k_left = st->k_left, thr = 1ll << d_bits;
  const long long gs = (long long)gridDim.x * blockDim.x;
  long long dum = 0, fg = kI64Max, gmax = kI64Min;
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += R * gs) {
    long long b[R], e[R];
    int32_t f[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const long long i = i0 + u * gs;
      b[u] = i < n ? row_ptr[i] : 0;
      e[u] = i < n ? row_ptr[i + 1] : 0;
      f[u] = i < n ? fcol[i] : 0;
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const long long i = i0 + u * gs;
      if (e[u] > b[u]) {
        const long long g = (long long)f[u] - base_of(row0 + i, se, k_left);
        fg = g < fg ? g : fg;
        gmax = g > gmax ? g : gmax;
        if (g >= thr) {
          ++dum;
          counts[i] += 1u;
        }
      }
    }
  }
  const long long sd = cta_reduce(dum, AddOp{}, 0ll, sh);
  const long long sf = cta_reduce(fg, MinOp{}, kI64Max, sh);
  const long long sg = cta_reduce(gmax, MaxOp{}, kI64Min, sh);
  if (threadIdx.x == 0) {
    if (sd) atomicAdd(reinterpret_cast<unsigned long long*>(&st->n_dummy), (unsigned long long)sd);
    if (sf != kI64Max) atomicMin(&st->min_first_gap, sf);
    if (sg != kI64Min) atomicMax(&st->max_gap, sg);
  }
}

template <bool FOLD>
__global__ void __launch_bounds__(kBlock) row_stats_long_kernel(const int64_t* __restrict__ row_ptr,
                                                                const int32_t* __restrict__ col_idx,
                                                                long long row0, long long se, int d_bits,
                                                                BuildStats* st, uint32_t* __restrict__ counts,
                                                                const int32_t* __restrict__ long_rows) {
  __shared__ long long sh[32];
  const long long nl = st->n_long;
  const long long k_left = FOLD ? 0 : st->k_left;
  const long long thr = 1ll << d_bits;
  const int lane = threadIdx.x & 31;
  long long dum = 0, gmax = kI64Min;
  for (long long w = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5; w < nl;
       w += (long long)gridDim.x * (kBlock / 32)) {
    const long long ri = long_rows[w];
    const long long rb = row_ptr[ri], re = row_ptr[ri + 1];
    const long long d0 = FOLD ? 0 : base_of(row0 + ri, se, k_left);
    long long cnt = 0;
    for (long long j = rb + lane + (FOLD ? 1 : 0); j < re; j += 32) {  // FOLD: first gap in first_gap_fold
      const long long col = col_idx[j];
      const long long gap = col - (j == rb ? d0 : (long long)col_idx[j - 1]);
      cnt += gap >= thr;
      gmax = gap > gmax ? gap : gmax;
    }
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    dum += lane == 0 ? cnt : 0;
    if (lane == 0) counts[ri] = (uint32_t)((re - rb) + cnt);
  }
  const long long sd = cta_reduce(dum, AddOp{}, 0ll, sh);
  const long long sg = cta_reduce(gmax, MaxOp{}, kI64Min, sh);
  if (threadIdx.x == 0) {
    if (sd) atomicAdd(reinterpret_cast<unsigned long long*>(&st->n_dummy), (unsigned long long)sd);
    if (sg != kI64Min) atomicMax(&st->max_gap, sg);
  }
}

// packed.py:162 — the reported row is the first one attaining the minimum first gap.
__global__ void first_gap_row_kernel(const int64_t* __restrict__ row_ptr,
                                     const int32_t* __restrict__ col_idx, long long n,
                                     long long row0, long long se, BuildStats* st) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long beg = row_ptr[i];
  if (row_ptr[i + 1] <= beg) return;
  const long long fg = (long long)col_idx[beg] - base_of(row0 + i, se, st->k_left);
  if (fg == st->min_first_gap) atomicMin(&st->first_gap_row, i);
}

// sell.py:22-30 — stable descending sort of stored counts inside each sigma
// block (the last partial block alone).  LSD radix on key = max - count.
// RB-bit digits: 8 for the 256-thread kernel (sigma <= 256: the stencils' counts need <= 8 bits,
// one pass), 4 for the 1024-thread one (a 256-bucket warp table would be 32 KB there)
template <int NT, int RB = (NT == 256 ? 8 : 4)>
__global__ void __launch_bounds__(NT) sort_blocks_kernel(const uint32_t* __restrict__ counts,
                                                         long long n, int sigma,
                                                         int32_t* __restrict__ order,
                                                         uint32_t* __restrict__ scount,
                                                         void* perm, int perm_bytes,
                                                         uint32_t* gscratch) {
  constexpr int NB = 1 << RB;
  static_assert(NB <= 16 || (NB % 32 == 0 && NB <= NT), "wide digits scan one bucket per thread");
  extern __shared__ uint32_t dyn[];
  __shared__ int hist[NB];
  __shared__ int wcnt[NT / 32][NB];
  __shared__ uint32_t s_red[NT / 32];
  __shared__ int s_wtot[NT / 32];
  const long long b0 = (long long)blockIdx.x * sigma;
  const int len = (int)min((long long)sigma, n - b0);
  uint32_t *ka, *ia, *kb, *ib;
  if (gscratch) {
    ka = gscratch + b0;
    ia = gscratch + n + b0;
    kb = gscratch + 2 * n + b0;
    ib = gscratch + 3 * n + b0;
  } else {
    ka = dyn;
    ia = dyn + sigma;
    kb = dyn + 2 * sigma;
    ib = dyn + 3 * sigma;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t mx = 0;
  for (int i = tid; i < len; i += NT) {
    const uint32_t c = counts[b0 + i];
    ka[i] = c;
    ia[i] = (uint32_t)i;
    mx = c > mx ? c : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint32_t t = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = t > mx ? t : mx;
  }
  if (lane == 0) s_red[warp] = mx;
  __syncthreads();
  uint32_t smax = 0;
  for (int w = 0; w < NT / 32; ++w) smax = s_red[w] > smax ? s_red[w] : smax;
  for (int i = tid; i < len; i += NT) ka[i] = smax - ka[i];
  const int bits = smax ? 32 - __clz(smax) : 0;
  const unsigned lt = (1u << lane) - 1u;
  __syncthreads();
  for (int sh = 0; sh < bits; sh += RB) {
    if (tid < NB) hist[tid] = 0;
    __syncthreads();
    for (int i = tid; i < len; i += NT) atomicAdd(&hist[(ka[i] >> sh) & (NB - 1)], 1);
    __syncthreads();
    if constexpr (NB <= 16) {
      if (tid == 0) {
        int run = 0;
        for (int dg = 0; dg < NB; ++dg) {
          const int t = hist[dg];
          hist[dg] = run;
          run += t;
        }
      }
    } else {  // exclusive scan of the NB buckets, one per thread of the first NB / 32 warps
      int h = 0, inc = 0;
      if (tid < NB) {  // whole warps (NB is a multiple of 32)
        h = hist[tid];
        inc = h;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += t;
        }
        if (lane == 31) s_wtot[warp] = inc;
      }
      __syncthreads();
      if (tid < NB) {
        int before = 0;
        for (int w2 = 0; w2 < warp; ++w2) before += s_wtot[w2];
        hist[tid] = before + inc - h;
      }
    }
    __syncthreads();
    for (int t0 = 0; t0 < len; t0 += NT) {
      const int i = t0 + tid;
      const bool valid = i < len;
      const uint32_t key = valid ? ka[i] : 0u;
      const int dg = valid ? (int)((key >> sh) & (NB - 1)) : NB;
      const unsigned m = __match_any_sync(0xffffffffu, dg);
      const int rank = __popc(m & lt);
      for (int e = tid; e < (NT / 32) * NB; e += NT) (&wcnt[0][0])[e] = 0;
      __syncthreads();
      if (valid && rank == 0) wcnt[warp][dg] = __popc(m);
      __syncthreads();
      if (tid < NB) {
        int run = hist[tid];
        for (int w = 0; w < NT / 32; ++w) {
          const int t = wcnt[w][tid];
          wcnt[w][tid] = run;
          run += t;
        }
        hist[tid] = run;
      }
      __syncthreads();
      if (valid) {
        const int pos = wcnt[warp][dg] + rank;
        kb[pos] = key;
        ib[pos] = ia[i];
      }
      __syncthreads();
    }
    uint32_t* t1 = ka; ka = kb; kb = t1;
    uint32_t* t2 = ia; ia = ib; ib = t2;
    __syncthreads();
  }
  for (int i = tid; i < len; i += NT) {
    const uint32_t src = ia[i];
    order[b0 + i] = (int32_t)(b0 + src);
    scount[b0 + i] = smax - ka[i];
    if (perm_bytes == 1) static_cast<uint8_t*>(perm)[b0 + i] = (uint8_t)src;
    else if (perm_bytes == 2) static_cast<uint16_t*>(perm)[b0 + i] = (uint16_t)src;
  }
}

// packed.py:208-212 — width of slice k = max stored count of its C storage rows.
__global__ void slice_width_kernel(const uint32_t* __restrict__ scount, long long n, int c,
                                   long long n_slices, long long* __restrict__ wwords) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_slices) return;
  uint32_t m = 0;
  const long long r0 = k * c;
  const long long r1 = min(r0 + c, n);
  for (long long r = r0; r < r1; ++r) m = scount[r] > m ? scount[r] : m;
  wwords[k] = (long long)m * c;
}

// ---------------------------------------------------------------- int64 scan
__device__ __forceinline__ long long block_incl_scan_1024(long long v, long long* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    long long w = sh[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    sh[lane] = w;
  }
  __syncthreads();
  if (warp > 0) v += sh[warp - 1];
  __syncthreads();
  return v;
}

__global__ void __launch_bounds__(1024) scan_reduce_kernel(const long long* __restrict__ in,
                                                           long long n, long long* bsum) {
  __shared__ long long sh[32];
  const long long t0 = (long long)blockIdx.x * kScanTile;
  long long s = 0;
  for (int e = 0; e < 4; ++e) {
    const long long i = t0 + (long long)e * 1024 + threadIdx.x;
    if (i < n) s += in[i];
  }
  s = cta_reduce(s, AddOp{}, 0ll, sh);
  if (threadIdx.x == 0) bsum[blockIdx.x] = s;
}

// exclusive scan of the block sums in place (single CTA, sequential over chunks)
__global__ void __launch_bounds__(1024) scan_bsum_kernel(long long* bsum, long long nb) {
  __shared__ long long sh[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (long long c0 = 0; c0 < nb; c0 += 1024) {
    const long long i = c0 + threadIdx.x;
    const long long v = i < nb ? bsum[i] : 0;
    const long long inc = block_incl_scan_1024(v, sh);
    const long long base = carry;
    if (i < nb) bsum[i] = base + inc - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry = base + inc;
    __syncthreads();
  }
}

// out[0] = 0, out[i+1] = sum_{j<=i} in[j]
__global__ void __launch_bounds__(1024) scan_apply_kernel(const long long* __restrict__ in,
                                                          long long n,
                                                          const long long* __restrict__ bsum,
                                                          long long* __restrict__ out) {
  __shared__ long long sh[32];
  const long long t0 = (long long)blockIdx.x * kScanTile;
  long long v[4];
  long long local = 0;
  const long long i0 = t0 + (long long)threadIdx.x * 4;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    v[e] = (i0 + e < n) ? in[i0 + e] : 0;
    local += v[e];
  }
  const long long inc = block_incl_scan_1024(local, sh);
  long long run = bsum[blockIdx.x] + inc - local;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    run += v[e];
    if (i0 + e < n) out[i0 + e + 1] = run;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = 0;
}

int scan_i64(const long long* in, long long n, long long* tmp, long long* out, cudaStream_t st,
             psell_error* err) {
  if (n == 0) {
    PSELL_CUDA(cudaMemsetAsync(out, 0, sizeof(long long), st), err);
    return PSELL_OK;
  }
  const long long nb = ceil_div(n, kScanTile);
  scan_reduce_kernel<<<(unsigned)nb, 1024, 0, st>>>(in, n, tmp);
  scan_bsum_kernel<<<1, 1024, 0, st>>>(tmp, nb);
  scan_apply_kernel<<<(unsigned)nb, 1024, 0, st>>>(in, n, tmp, out);
  PSELL_CHECK_LAUNCH(err, "scan_i64");
  return PSELL_OK;
}

// ---------------------------------------------------------------- fill
struct FillArgs {
  const int64_t* row_ptr;
  const int32_t* col_idx;
  const double* values;
  const int32_t* order;  // null for mode none
  const int64_t* offset;
  void* pack;
  BuildStats* st;
  int32_t* long_rows;  // storage rows longer than kLongRow (fill_long_kernel)
  long long n, n_slices, row0, se, k_left;
  int c;
  Fmt f;
};

// packed.py:216-231: word q of storage row s lives at offset[s//C] + s%C + q*C.
// A dummy (flag 0, full gap) precedes a real word whose gap >= 2^D; that real
// word then stores delta 0.  Everything past the stored count is padding 0.
#ifndef PSELL_FILL_U
#define PSELL_FILL_U 4
#endif
#ifndef PSELL_FILL_MINB
#define PSELL_FILL_MINB 1
#endif
constexpr int kFillU = PSELL_FILL_U;

template <typename W>
__global__ void __launch_bounds__(kBlock, PSELL_FILL_MINB) fill_kernel(FillArgs a) {
  __shared__ long long sh[32];
  const long long s = (long long)blockIdx.x * kBlock + threadIdx.x;
  long long bad_nf = kI64Max, bad_of = kI64Max;
  const long long thr = 1ll << a.f.d;
  const int sh_v = a.f.d + 1;
  const long long stride = a.c;
  // rows longer than kLongRow entries are listed for fill_long_kernel (one warp each)
  bool lng = false;
  if (s < a.n_slices * a.c) {
    // 32-bit divisions when the sizes allow (the 64-bit ones cost ~2x a row's encode work)
    const bool n32 = a.n_slices * a.c < (1ll << 31);
    const long long k = n32 ? (long long)((uint32_t)s / (uint32_t)a.c) : s / a.c;
    const int lane = (int)(s - k * a.c);
    const long long o = a.offset[k];
    const long long width = (a.offset[k + 1] - o) / a.c;
    W* out = static_cast<W*>(a.pack) + o + lane;
    long long q = 0;
    if (s < a.n) {
      const long long r = a.order ? (long long)a.order[s] : s;
      const long long beg = a.row_ptr[r], end = a.row_ptr[r + 1];
      long long prev = [&] {
        const long long g = a.row0 + r;
        const long long blk = (g < (1ll << 32) && a.se < (1ll << 32))
                                  ? (long long)((uint32_t)g / (uint32_t)a.se) * a.se : (g / a.se) * a.se;
        return blk > a.k_left ? blk - a.k_left : 0ll;
      }();
      lng = end - beg > kLongRow;
      const long long jend = lng ? beg : end;
      // entries in groups of kFillU: the group's column / value loads issue together (the
      // walk itself is sequential: the gap and the word index carry from entry to entry)
      for (long long j0 = beg; j0 < jend; j0 += kFillU) {
        int32_t cv[kFillU];
        double vv[kFillU];
#pragma unroll
        for (int u = 0; u < kFillU; ++u) {
          const bool in = j0 + u < jend;
          cv[u] = in ? a.col_idx[j0 + u] : 0;
          vv[u] = in ? a.values[j0 + u] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kFillU; ++u) {
          const long long j = j0 + u;
          if (j >= jend) break;
          const long long col = cv[u];
          long long gap = col - prev;
          prev = col;
          int stc = ENC_OK;
          const W pat = (W)encode_value(a.f, vv[u], stc);
          if (stc == ENC_NONFINITE) bad_nf = j < bad_nf ? j : bad_nf;
          else if (stc == ENC_OVERFLOW) bad_of = j < bad_of ? j : bad_of;
          if (gap >= thr) {
            out[q * stride] = ((W)gap) << 1;
            ++q;
            gap = 0;
          }
          out[q * stride] = (pat << sh_v) | (((W)gap) << 1) | W(1);
          ++q;
        }
      }
    }
    if (!lng)
      for (; q < width; ++q) out[q * stride] = W(0);
  }
  if (lng) a.long_rows[atomicAdd(reinterpret_cast<unsigned long long*>(&a.st->n_long), 1ull)] = (int32_t)s;
  // the error reductions only in a CTA that saw a non-finite or overflowing value
  if (!__syncthreads_or(bad_nf != kI64Max || bad_of != kI64Max)) return;
  const long long m1 = cta_reduce(bad_nf, MinOp{}, kI64Max, sh);
  const long long m2 = cta_reduce(bad_of, MinOp{}, kI64Max, sh);
  if (threadIdx.x == 0) {
    if (m1 != kI64Max) atomicMin(&a.st->nonfinite_pos, m1);
    if (m2 != kI64Max) atomicMin(&a.st->overflow_pos, m2);
  }
}

// fill of the listed long storage rows: one warp per row, 32 entries per trip, the
// word positions from a warp prefix sum of (1 + dummy) -- the same words at the
// same places as the sequential walk of fill_kernel
template <typename W>
__global__ void __launch_bounds__(kBlock) fill_long_kernel(FillArgs a) {
  __shared__ long long sh[32];
  long long bad_nf = kI64Max, bad_of = kI64Max;
  const long long thr = 1ll << a.f.d;
  const int sh_v = a.f.d + 1;
  const long long stride = a.c;
  const long long nl = a.st->n_long;
  const int wl = threadIdx.x & 31;
  for (long long w = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5; w < nl;
       w += (long long)gridDim.x * (kBlock / 32)) {
    const long long s = a.long_rows[w];
    const long long k = s / a.c;
    const long long o = a.offset[k];
    const long long width = (a.offset[k + 1] - o) / a.c;
    W* out = static_cast<W*>(a.pack) + o + (s - k * a.c);
    const long long r = a.order ? (long long)a.order[s] : s;
    const long long rb = a.row_ptr[r], re = a.row_ptr[r + 1];
    const long long d0 = [&] {
      const long long g = a.row0 + r;
      const long long blk = (g / a.se) * a.se;
      return blk > a.k_left ? blk - a.k_left : 0ll;
    }();
    long long q0 = 0;  // words stored before this trip
    for (long long j0 = rb; j0 < re; j0 += 32) {
      const long long j = j0 + wl;
      const bool in = j < re;
      long long gap = 0;
      W pat = 0;
      if (in) {
        const long long col = a.col_idx[j];
        gap = col - (j == rb ? d0 : (long long)a.col_idx[j - 1]);
        int stc = ENC_OK;
        pat = (W)encode_value(a.f, a.values[j], stc);
        if (stc == ENC_NONFINITE) bad_nf = j < bad_nf ? j : bad_nf;
        else if (stc == ENC_OVERFLOW) bad_of = j < bad_of ? j : bad_of;
      }
      const int dm = in && gap >= thr;
      int inc = in ? 1 + dm : 0;  // inclusive scan of words per entry
      for (int sft = 1; sft < 32; sft <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, sft);
        if (wl >= sft) inc += t;
      }
      if (in) {
        const long long qr = q0 + inc - 1;  // this entry's real word
        if (dm) {
          out[(qr - 1) * stride] = ((W)gap) << 1;
          gap = 0;
        }
        out[qr * stride] = (pat << sh_v) | (((W)gap) << 1) | W(1);
      }
      q0 += __shfl_sync(0xffffffffu, inc, 31);
    }
    for (long long q = q0 + wl; q < width; q += 32) out[q * stride] = W(0);
  }
  const long long m1 = cta_reduce(bad_nf, MinOp{}, kI64Max, sh);
  const long long m2 = cta_reduce(bad_of, MinOp{}, kI64Max, sh);
  if (threadIdx.x == 0) {
    if (m1 != kI64Max) atomicMin(&a.st->nonfinite_pos, m1);
    if (m2 != kI64Max) atomicMin(&a.st->overflow_pos, m2);
  }
}

static int check_desc(const psell_desc* d, psell_error* err) {
  if (!d) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "null descriptor");
  if (!fmt_valid(fmt_of(d)))
    return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, "invalid PackFormat");
  if (!fmt_device_ok(fmt_of(d))) return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, PSELL_FP16_W64_MSG);
  if (d->mode < PSELL_MODE_NONE || d->mode > PSELL_MODE_IMPLICIT)
    return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, "invalid mode");
  if (d->c < 1) return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, "slice size must be >= 1");
  if (d->mode != PSELL_MODE_NONE) {
    if (d->sigma < 1 || d->sigma % d->c != 0)
      return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, "sigma must be a positive multiple of C");
    if (d->sigma > 65536)
      return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, "sigma above 65536");
  }
  if (d->n_rows < 0 || d->n_cols < 0 || d->n_rows >= (1ll << 31) || d->n_cols > (1ll << 31))
    return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "matrix dimensions out of range");
  const long long se = d->mode == PSELL_MODE_NONE ? 1 : d->sigma;
  const long long align = d->mode == PSELL_MODE_NONE ? d->c : d->sigma;
  if (d->row0 < 0 || d->row0 % align != 0)
    return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "row0 must be sigma (C) aligned");
  (void)se;
  return PSELL_OK;
}

}  // namespace psell

using namespace psell;

extern "C" {

const char* psell_version(void) { return "psell 0.1.0 (sm_100a, abi 1)"; }
int32_t psell_abi_version(void) { return PSELL_ABI_VERSION; }

size_t psell_build_workspace_bytes(const psell_desc* desc) {
  if (!desc) return 0;
  return carve(desc, nullptr).bytes;
}

int psell_lower_bandwidth(const psell_desc* d, const int64_t* row_ptr, const int32_t* col_idx,
                          void* ws, size_t ws_bytes, int64_t* k_left_host, void* stream,
                          psell_error* err) {
  if (int rc = check_desc(d, err)) return rc;
  BuildWs w = carve(d, ws);
  if (!ws || ws_bytes < w.bytes) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "workspace too small");
  cudaStream_t st = as_stream(stream);
  init_stats_kernel<<<1, 1, 0, st>>>(w.stats, 0);
  const long long n = d->n_rows;
  if (n > 0)
    lower_bandwidth_kernel<<<(unsigned)ceil_div(n, kBlock), kBlock, 0, st>>>(row_ptr, col_idx, n,
                                                                            d->row0, w.stats);
  PSELL_CHECK_LAUNCH(err, "lower_bandwidth");
  BuildStats hs;
  PSELL_CUDA(cudaMemcpyAsync(&hs, w.stats, sizeof(hs), cudaMemcpyDeviceToHost, st), err);
  PSELL_CUDA(cudaStreamSynchronize(st), err);
  *k_left_host = hs.k_left;
  return ok(err);
}

int psell_build_plan(const psell_desc* d, const int64_t* row_ptr, const int32_t* col_idx,
                     void* ws, size_t ws_bytes, int64_t* offset, void* perm, int64_t* out_host,
                     void* stream, psell_error* err) {
  if (int rc = check_desc(d, err)) return rc;
  BuildWs w = carve(d, ws);
  if (!ws || ws_bytes < w.bytes) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "workspace too small");
  cudaStream_t st = as_stream(stream);
  const long long n = d->n_rows;
  const long long ns = ceil_div(n, d->c);
  const long long se = d->mode == PSELL_MODE_NONE ? 1 : d->sigma;
  const unsigned grid_rows = (unsigned)ceil_div(n > 0 ? n : 1, kBlock);

  init_stats_kernel<<<1, 1, 0, st>>>(w.stats, d->k_left);
  if (n > 0) {
    if (d->k_left < 0 && fold_k_left()) {
      // w.scount is free until the sort (which writes every entry): the rows' first columns
      int32_t* fcol = reinterpret_cast<int32_t*>(w.scount);
      row_stats_kernel<true><<<grid_rows, kBlock, 0, st>>>(row_ptr, col_idx, n, d->row0, se, d->d, w.stats,
                                                           w.counts, w.long_rows, fcol);
      row_stats_long_kernel<true><<<long_grid(), kBlock, 0, st>>>(row_ptr, col_idx, d->row0, se, d->d, w.stats,
                                                                  w.counts, w.long_rows);
      first_gap_fold_kernel<<<grid_rows < long_grid() ? grid_rows : long_grid(), kBlock, 0, st>>>(
          row_ptr, fcol, n, d->row0, se, d->d, w.stats, w.counts);
    } else {
      if (d->k_left < 0)
        lower_bandwidth_kernel<<<grid_rows, kBlock, 0, st>>>(row_ptr, col_idx, n, d->row0, w.stats);
      row_stats_kernel<false><<<grid_rows, kBlock, 0, st>>>(row_ptr, col_idx, n, d->row0, se, d->d, w.stats,
                                                            w.counts, w.long_rows, nullptr);
      row_stats_long_kernel<false><<<long_grid(), kBlock, 0, st>>>(row_ptr, col_idx, d->row0, se, d->d,
                                                                   w.stats, w.counts, w.long_rows);
    }
  }
  PSELL_CHECK_LAUNCH(err, "row_stats");
  BuildStats hs;
  PSELL_CUDA(cudaMemcpyAsync(&hs, w.stats, sizeof(hs), cudaMemcpyDeviceToHost, st), err);
  PSELL_CUDA(cudaStreamSynchronize(st), err);
  if (hs.min_first_gap < 0) {
    first_gap_row_kernel<<<grid_rows, kBlock, 0, st>>>(row_ptr, col_idx, n, d->row0, se, w.stats);
    PSELL_CHECK_LAUNCH(err, "first_gap_row");
    PSELL_CUDA(cudaMemcpyAsync(&hs, w.stats, sizeof(hs), cudaMemcpyDeviceToHost, st), err);
    long long rp = 0;
    int32_t col = 0;
    PSELL_CUDA(cudaMemcpyAsync(&rp, row_ptr + hs.first_gap_row, 8, cudaMemcpyDeviceToHost, st), err);
    PSELL_CUDA(cudaStreamSynchronize(st), err);
    PSELL_CUDA(cudaMemcpyAsync(&col, col_idx + rp, 4, cudaMemcpyDeviceToHost, st), err);
    PSELL_CUDA(cudaStreamSynchronize(st), err);
    return set_err(err, PSELL_EVALUE, PSELL_KIND_FIRST_GAP, d->row0 + hs.first_gap_row, col, 0,
                   "first column is left of its base offset");
  }
  const long long max_dummy = d->w == 32 ? 0x7FFFFFFFll : kI64Max;
  if (hs.max_gap != kI64Min && hs.max_gap > max_dummy)
    return set_err(err, PSELL_EVALUE, PSELL_KIND_GAP_RANGE, -1, 0, 0, "gap exceeds the dummy range");

  const uint32_t* scount = w.counts;
  if (d->mode != PSELL_MODE_NONE && n > 0) {
    const unsigned nblk = (unsigned)ceil_div(n, d->sigma);
    const int perm_bytes = (d->mode == PSELL_MODE_IMPLICIT && perm) ? (d->sigma <= 256 ? 1 : 2) : 0;
    if (d->sigma <= kSortSmemMaxSigma) {
      const size_t smem = 16 * (size_t)d->sigma;
      if (d->sigma <= 256)
        sort_blocks_kernel<256><<<nblk, 256, smem, st>>>(w.counts, n, d->sigma, w.order, w.scount,
                                                         perm, perm_bytes, nullptr);
      else
        sort_blocks_kernel<1024><<<nblk, 1024, smem, st>>>(w.counts, n, d->sigma, w.order, w.scount,
                                                           perm, perm_bytes, nullptr);
    } else {
      // keys in global scratch: the 8-bit digit table fits beside them (fewer passes)
      sort_blocks_kernel<1024, 8><<<nblk, 1024, 0, st>>>(w.counts, n, d->sigma, w.order, w.scount,
                                                         perm, perm_bytes, w.sort_tmp);
    }
    PSELL_CHECK_LAUNCH(err, "sort_blocks");
    scount = w.scount;
  }
  if (ns > 0) {
    slice_width_kernel<<<(unsigned)ceil_div(ns, kBlock), kBlock, 0, st>>>(scount, n, d->c, ns, w.wwords);
    PSELL_CHECK_LAUNCH(err, "slice_width");
  }
  if (int rc = scan_i64(w.wwords, ns, w.scan_tmp, reinterpret_cast<long long*>(offset), st, err)) return rc;
  long long n_stored = 0;
  PSELL_CUDA(cudaMemcpyAsync(&n_stored, offset + ns, 8, cudaMemcpyDeviceToHost, st), err);
  PSELL_CUDA(cudaStreamSynchronize(st), err);
  out_host[0] = hs.k_left;
  out_host[1] = n_stored;
  out_host[2] = hs.n_dummy;
  return ok(err);
}

int psell_build_fill(const psell_desc* d, const int64_t* row_ptr, const int32_t* col_idx,
                     const double* values, const void* ws, size_t ws_bytes, const int64_t* offset,
                     void* pack, void* stream, psell_error* err) {
  if (int rc = check_desc(d, err)) return rc;
  BuildWs w = carve(d, const_cast<void*>(ws));
  if (!ws || ws_bytes < w.bytes) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "workspace too small");
  if (d->k_left < 0) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "fill needs the planned k_left");
  cudaStream_t st = as_stream(stream);
  const long long n = d->n_rows;
  const long long ns = ceil_div(n, d->c);
  FillArgs a;
  a.row_ptr = row_ptr;
  a.col_idx = col_idx;
  a.values = values;
  a.order = d->mode == PSELL_MODE_NONE ? nullptr : w.order;
  a.offset = offset;
  a.pack = pack;
  a.st = w.stats;
  a.long_rows = w.long_rows;
  a.n = n;
  a.n_slices = ns;
  a.row0 = d->row0;
  a.se = d->mode == PSELL_MODE_NONE ? 1 : d->sigma;
  a.k_left = d->k_left;
  a.c = d->c;
  a.f = fmt_of(d);
  init_stats_kernel<<<1, 1, 0, st>>>(w.stats, d->k_left);
  const long long rows = ns * d->c;
  if (rows > 0) {
    const unsigned grid = (unsigned)ceil_div(rows, kBlock);
    PSELL_CUDA(cudaMemsetAsync(&w.stats->n_long, 0, sizeof(long long), st), err);
    if (d->w == 32) {
      fill_kernel<uint32_t><<<grid, kBlock, 0, st>>>(a);
      fill_long_kernel<uint32_t><<<long_grid(), kBlock, 0, st>>>(a);
    } else {
      fill_kernel<uint64_t><<<grid, kBlock, 0, st>>>(a);
      fill_long_kernel<uint64_t><<<long_grid(), kBlock, 0, st>>>(a);
    }
    PSELL_CHECK_LAUNCH(err, "fill");
  }
  BuildStats hs;
  PSELL_CUDA(cudaMemcpyAsync(&hs, w.stats, sizeof(hs), cudaMemcpyDeviceToHost, st), err);
  PSELL_CUDA(cudaStreamSynchronize(st), err);
  if (hs.nonfinite_pos != kI64Max || hs.overflow_pos != kI64Max) {
    const bool nf = hs.nonfinite_pos != kI64Max;
    const long long pos = nf ? hs.nonfinite_pos : hs.overflow_pos;
    double v = 0;
    PSELL_CUDA(cudaMemcpyAsync(&v, values + pos, 8, cudaMemcpyDeviceToHost, st), err);
    PSELL_CUDA(cudaStreamSynchronize(st), err);
    return set_err(err, PSELL_ECODEC, nf ? PSELL_KIND_NONFINITE : PSELL_KIND_OVERFLOW, pos, 0, v,
                   nf ? "non-finite value" : "value overflows the codec");
  }
  return ok(err);
}

size_t psell_sort_workspace_bytes(int64_t n, int32_t sigma) {
  return align_up(4 * (size_t)(n > 0 ? n : 1)) + (sigma > kSortSmemMaxSigma ? 16 * (size_t)(n > 0 ? n : 1) : 0);
}

int psell_sort_order(const uint32_t* counts, int64_t n, int32_t sigma, int32_t* order, void* ws,
                     size_t ws_bytes, void* stream, psell_error* err) {
  if (sigma < 1 || sigma > 65536) return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, "invalid sigma");
  if (ws_bytes < psell_sort_workspace_bytes(n, sigma) || !ws)
    return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "workspace too small");
  if (n <= 0) return ok(err);
  cudaStream_t st = as_stream(stream);
  uint32_t* scount = static_cast<uint32_t*>(ws);
  uint32_t* tmp = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + align_up(4 * (size_t)n));
  const unsigned nblk = (unsigned)ceil_div(n, sigma);
  if (sigma <= 256)
    sort_blocks_kernel<256><<<nblk, 256, 16 * (size_t)sigma, st>>>(counts, n, sigma, order, scount, nullptr, 0, nullptr);
  else if (sigma <= kSortSmemMaxSigma)
    sort_blocks_kernel<1024><<<nblk, 1024, 16 * (size_t)sigma, st>>>(counts, n, sigma, order, scount, nullptr, 0, nullptr);
  else
    sort_blocks_kernel<1024, 8><<<nblk, 1024, 0, st>>>(counts, n, sigma, order, scount, nullptr, 0, tmp);
  PSELL_CHECK_LAUNCH(err, "psell_sort_order");
  return ok(err);
}

}  // extern "C"
