/*
 * psell.h — C ABI of the B200-native PackSELL path (libpsell.so, sm_100a).
 *
 * This is the drop-in boundary for the reference package `packsell` 0.1.0
 * (pure Python/numpy, /root/reference/pkg/src/packsell).  The reference has
 * no FFI of its own; each entry point below replaces the numpy body of the
 * reference function named beside it, and the Python mirror
 * (the modules of paper_2604_13433_b200/) binds them with ctypes exactly where the
 * reference calls numpy.  See INTEGRATION.md for the bindings.
 *
 * Conventions
 *  - All array arguments are DEVICE pointers (cudaMalloc / torch CUDA
 *    storage) unless the name ends in `_host`.  `stream` is a cudaStream_t
 *    passed as void* (NULL = legacy default stream).
 *  - Calls are stream ordered.  The library keeps no global mutable state
 *    and allocates nothing persistent; scratch comes from a caller-owned
 *    workspace sized by the matching *_workspace_bytes() call.
 *  - Every call returns a psell_status; on failure *err is filled with the
 *    reference's error payload (kind, first offending index, value) so the
 *    host can raise the same exception class and message as the reference.
 *  - Calls that must report data-dependent errors or sizes synchronise the
 *    stream (build plan/fill, to_csr plan, encode); SpMV and the solver
 *    kernels never synchronise and are CUDA-graph capturable.
 */
#ifndef PSELL_H
#define PSELL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSELL_ABI_VERSION 1

#if defined(__GNUC__)
#define PSELL_API __attribute__((visibility("default")))
#else
#define PSELL_API
#endif

typedef enum psell_status {
  PSELL_OK = 0,
  PSELL_EVALUE = 1, /* -> ValueError (layout / parameter), packed.py:159-170, sell.py:33-42 */
  PSELL_ECODEC = 2, /* -> CodecError(ValueError), codec.py:33-34,124-170 */
  PSELL_ECUDA = 3,  /* CUDA runtime failure (message in err->msg) */
  PSELL_EARG = 4    /* bad argument to the ABI itself (null pointer, small workspace) */
} psell_status;

typedef enum psell_err_kind {
  PSELL_KIND_NONE = 0,
  PSELL_KIND_FIRST_GAP = 1, /* row index, aux = its first column (packed.py:159-164) */
  PSELL_KIND_GAP_RANGE = 2, /* any gap > 2^(W-1)-1 (packed.py:166-170) */
  PSELL_KIND_NONFINITE = 3, /* value index, value (codec.py:124-127) */
  PSELL_KIND_OVERFLOW = 4,  /* value index, value (codec.py:133-137,154-156,166-169) */
  PSELL_KIND_PARAM = 5,
  PSELL_KIND_CUDA = 6
} psell_err_kind;

typedef enum psell_codec { PSELL_FP16 = 0, PSELL_E8MY = 1, PSELL_FP32EMBED = 2 } psell_codec;
typedef enum psell_mode { PSELL_MODE_NONE = 0, PSELL_MODE_EXPLICIT = 1, PSELL_MODE_IMPLICIT = 2 } psell_mode;
typedef enum psell_dtype { PSELL_DT_F16 = 0, PSELL_DT_F32 = 1, PSELL_DT_F64 = 2 } psell_dtype;

/* psell_spmv flags */
#define PSELL_SPMV_REF_ORDER 1 /* numpy rounding order: value cast to x dtype, product and sum rounded separately */
#define PSELL_SPMV_TMA_STREAM 2 /* C=32 fast path: persistent TMA bulk-copy stream instead of the default
                                  register-pipelined dual-slice kernel (A/B experiments) */
#define PSELL_SPMV_NARROW 4     /* mean slice width <= 12 steps (e.g. 7-point rows): 12-step chunks */
#define PSELL_SPMV_NARROW12 8   /* with NARROW: every slice <= 12 steps, the TMA slot kernel may run */
#define PSELL_SPMV_W32 16       /* every slice <= 32 steps: the wide TMA kernel may run.  Like NARROW12
                                  it must be true of the matrix (PackSellMatrix.spmv_flags derives it from
                                  the offsets); a wider slice under it is cut to its first 32 steps (the
                                  staging never overruns its slot) and its rows come out wrong */

typedef struct psell_error {
  int32_t code;  /* psell_status */
  int32_t kind;  /* psell_err_kind */
  int64_t index; /* first offending row / value position (reference semantics) */
  int64_t aux;   /* e.g. the offending first column */
  double value;  /* offending value for codec errors */
  char msg[256];
} psell_error;

/*
 * One descriptor serves build and SpMV.  Mirrors PackFormat (codec.py:37-44)
 * plus the layout arguments of build_packsell (packed.py:176-178) and the
 * scalar fields of PackSellMatrix (packed.py:83-100).
 *
 * Multi-GPU slabs: a rank owns global rows [row0, row0 + n_rows); row0 must be
 * sigma-aligned (C-aligned in mode none).  Base offsets use the global row
 * index and the global k_left, so the concatenation of slab packs over ranks
 * is byte-identical to the single-GPU pack.
 */
typedef struct psell_desc {
  int32_t w, d, codec;    /* word bits (32|64), delta bits, psell_codec */
  int32_t c, sigma, mode; /* slice height C, sorting window sigma, psell_mode */
  int64_t n_rows;         /* rows of this slab */
  int64_t n_cols;         /* global number of columns */
  int64_t row0;           /* global index of local row 0 */
  int64_t k_left;         /* build: < 0 => compute (matrix.py:319-349); spmv: the matrix's k_left */
  int64_t nnz;            /* build: CSR nnz of the slab */
} psell_desc;

PSELL_API const char* psell_version(void);
PSELL_API int32_t psell_abi_version(void);

/* Re-read the PSELL_* A/B environment knobs of the SpMV launchers (cached per
 * call site otherwise: a getenv per launch is measurable on small matrices). */
PSELL_API int32_t psell_reload_env(void);

/* ---- K1: CSR -> PackSELL builder (replaces build_packsell, packed.py:176-239) ---- */

PSELL_API size_t psell_build_workspace_bytes(const psell_desc* desc);

/* Local lower bandwidth max(0, max_i(row0+i - first_col_i)) (matrix.py:334-339);
 * ranks all-reduce MAX of this to get the global k_left.  Synchronises. */
PSELL_API int psell_lower_bandwidth(const psell_desc* desc, const int64_t* row_ptr, const int32_t* col_idx,
                          void* workspace, size_t ws_bytes, int64_t* k_left_host, void* stream,
                          psell_error* err);

/* Plan: k_left (unless desc->k_left >= 0), per-row stored counts with dummy
 * words (packed.py:145-173), stable descending sigma-block sort (sell.py:22-30),
 * slice widths and the int64 slice offsets (packed.py:208-215), perm
 * (packed.py:233-235).  offset has n_slices+1 entries (n_slices = ceil(n_rows/C)),
 * perm has n_rows entries of 1 byte (sigma<=256) or 2 bytes, NULL unless mode
 * implicit.  out_host receives {k_left, n_stored, n_dummy}.  Synchronises. */
PSELL_API int psell_build_plan(const psell_desc* desc, const int64_t* row_ptr, const int32_t* col_idx,
                     void* workspace, size_t ws_bytes, int64_t* offset, void* perm,
                     int64_t* out_host, void* stream, psell_error* err);

/* Fill: writes every word of pack (offset[n_slices] words of W bits: real,
 * dummy and all-zero padding) (packed.py:218-231) and validates the codec
 * (non-finite first, then overflow; minimum position).  desc->k_left must be
 * the value the plan returned.  Synchronises. */
PSELL_API int psell_build_fill(const psell_desc* desc, const int64_t* row_ptr, const int32_t* col_idx,
                     const double* values, const void* workspace, size_t ws_bytes,
                     const int64_t* offset, void* pack, void* stream, psell_error* err);

/* Stable descending order of counts inside sigma blocks (sell.py:22-30):
 * order[i] = global (0-based) row stored at position i.  counts are uint32. */
PSELL_API size_t psell_sort_workspace_bytes(int64_t n, int32_t sigma);
PSELL_API int psell_sort_order(const uint32_t* counts, int64_t n, int32_t sigma, int32_t* order,
                               void* workspace, size_t ws_bytes, void* stream, psell_error* err);

/* ---- K2: PackSELL SpMV (replaces packsell_spmv, packed.py:242-271) ----
 * y[out(s)] = sum_q value(q) * x[cursor(q)] for every storage row s < n_rows,
 * cursor starting at min(d_s, n_cols-1).  y has x's dtype.  Default: FP32 FMA
 * accumulation (FP64 for f64 x); PSELL_SPMV_REF_ORDER reproduces numpy's
 * rounding bit for bit.  x is the GLOBAL vector (n_cols entries). */
PSELL_API int psell_spmv(const psell_desc* desc, const void* pack, const int64_t* offset, const void* perm,
               const void* x, int32_t x_dtype, void* y, int32_t flags, void* stream,
               psell_error* err);

/* Name of the kernel psell_spmv launches for this descriptor, x dtype and flags
 * (the same dispatch, no launch): lets a benchmark report the kernel it timed. */
PSELL_API const char* psell_spmv_kernel_name(const psell_desc* desc, int32_t x_dtype, int32_t flags);

/* Long-slice segmentation for irregular (power-law) matrices.  Slices wider than
 * seg_len steps are cut into segments (seg_slice/seg_q0: the slice and first
 * step of each; long_slice/long_seg0: the long slices and their first segment,
 * n_long + 1 entries).  psell_spmv_seg_checkpoints fills seg_c2[n_seg][32] with
 * each lane's cursor (2 * column) before the segment, once per matrix;
 * psell_spmv_segmented then runs short slices one warp each and every segment
 * on its own warp, combining the segment partials of a row in segment order.
 * C = 32, W = 32 (fp16 / e8my), f16 / f32 x.  FMA accumulation. */
PSELL_API int psell_spmv_seg_checkpoints(const psell_desc* desc, const void* pack, const int64_t* offset,
                                         int32_t seg_len, int64_t n_seg, const int32_t* seg_slice,
                                         const int32_t* seg_q0, int64_t n_long, const int32_t* long_slice,
                                         const int32_t* long_seg0, uint32_t* seg_c2, void* stream,
                                         psell_error* err);
PSELL_API int psell_spmv_segmented(const psell_desc* desc, const void* pack, const int64_t* offset,
                                   const void* perm, const void* x, int32_t x_dtype, void* y,
                                   int32_t seg_len, int64_t n_seg, const int32_t* seg_slice,
                                   const int32_t* seg_q0, const uint32_t* seg_c2, float* seg_partial,
                                   int64_t n_long, const int32_t* long_slice, const int32_t* long_seg0,
                                   uint32_t* sched, int32_t sched_chunks, void* stream, psell_error* err);
/* sched (nullable): G + 1 zeroed uint32 of device scratch kept with the matrix, G =
 * |sched_chunks| = the SM count; with PSELL_AFF=1 the short slices then run on an
 * SM-affine claim grid (one chunk of consecutive slice pairs per SM, work stealing) and
 * the kernel leaves the counters zeroed.  sched_chunks < 0: the G + 1 counters are
 * followed by 2 G + 1 slice-pair bounds (2 G chunks balanced by the short slices' words),
 * and the default static SM-affine grid runs: one 1024-thread CTA per SM takes chunks
 * 2b, 2b + 1 after its share of the segments, no atomics (PackSellMatrix builds both). */

/* Number of double partials psell_spmv_dot writes (one per CTA) for these flags. */
PSELL_API int64_t psell_spmv_dot_partials(const psell_desc* desc, int32_t flags);

/* SpMV fused with the PCG curvature dot: also writes partials[b] =
 * sum over the CTA's rows of (double)p_own[i] * (double)y[i] (solvers.py:294-295),
 * p_own = the slab's own rows of the direction vector.  f32 x/y only.  If
 * skip_flag != NULL and *skip_flag != 0 the kernel does nothing (breakdown). */
PSELL_API int psell_spmv_dot(const psell_desc* desc, const void* pack, const int64_t* offset,
                   const void* perm, const float* x, float* y, const float* p_own,
                   double* partials, const int32_t* skip_flag, int32_t flags, void* stream,
                   psell_error* err);

/* ---- K5: PackSELL -> CSR decode (replaces packsell_to_csr, packed.py:274-303) ---- */
PSELL_API size_t psell_to_csr_workspace_bytes(const psell_desc* desc);
/* Writes row_ptr (n_rows+1, logical row order) and returns nnz in *nnz_host. Synchronises. */
PSELL_API int psell_to_csr_plan(const psell_desc* desc, const void* pack, const int64_t* offset,
                      const void* perm, void* workspace, size_t ws_bytes, int64_t* row_ptr,
                      int64_t* nnz_host, void* stream, psell_error* err);
/* Largest column a real (flag = 1) word addresses, walking every storage row from the
 * SpMV's clamped start (packed.py:257); 0 when there is none.  ws8: 8 bytes of device
 * scratch.  Synchronises.  read_psell rejects containers whose streams reach n_cols. */
PSELL_API int psell_max_column(const psell_desc* desc, const void* pack, const int64_t* offset, const void* perm,
                               int64_t* out_host, void* ws8, void* stream, psell_error* err);
PSELL_API int psell_to_csr_fill(const psell_desc* desc, const void* pack, const int64_t* offset,
                      const void* perm, const int64_t* row_ptr, int32_t* col_idx, double* values,
                      void* stream, psell_error* err);

/* ---- value codecs on device (replace codec.py:173-250) ---- */
/* patterns: uint32 (W=32) or uint64 (W=64).  Synchronises (error check). */
PSELL_API int psell_encode(const psell_desc* fmt, const double* values, int64_t n, void* patterns,
                 void* workspace16, void* stream, psell_error* err);
/* values out: float16 (fp16 codec) or float32 */
PSELL_API int psell_decode(const psell_desc* fmt, const void* patterns, int64_t n, void* values,
                 void* stream, psell_error* err);
PSELL_API int psell_pack_words(const psell_desc* fmt, const void* patterns, const int64_t* deltas,
                     const uint8_t* flags, int64_t n, void* words, void* stream, psell_error* err);
/* deltas out as uint64; values out float16 (fp16) or float32 */
PSELL_API int psell_unpack_words(const psell_desc* fmt, const void* words, int64_t n, void* values,
                       uint64_t* deltas, uint8_t* flags, void* stream, psell_error* err);

/* ---- K4: CSR SpMV in the reference's row-sequential order (matrix.py:272-291) ----
 * values are f64; converted to x's dtype per element, every product and sum
 * rounded in that dtype.  Rows [0, n_rows) of the slab, x global. */
PSELL_API int psell_csr_spmv(int64_t n_rows, const int64_t* row_ptr, const int32_t* col_idx,
                   const double* values, const void* x, int32_t x_dtype, void* y, void* stream,
                   psell_error* err);

/* psell_csr_spmv in f64 fused with the PCG's p.q (solvers.py:197-198):
 * y = A x (bitwise as psell_csr_spmv) and out1[0] = sum_i p_own[i] * y[i] over
 * the slab's rows (p_own = this rank's slab of x), summed per CTA of the
 * persistent grid in row order, then over CTAs in a fixed tree (deterministic).
 * partials: >= 4 * SM count doubles. */
PSELL_API int psell_csr_spmv_dot(int64_t n_rows, const int64_t* row_ptr, const int32_t* col_idx,
                       const double* values, const double* x, double* y, const double* p_own,
                       double* partials, double* out1, void* stream, psell_error* err);

/* ---- K3: solver vector kernels (solvers.py:87-93,171-308) ----
 * Reductions are deterministic: fixed-grid partials summed in a fixed tree.
 * Device scalar blocks (double* scal, int32_t* iflags) are described in
 * paper_2604_13433_b200/solvers.py. */
#define PSELL_RED_BLOCKS 1184 /* 8 x 148 SMs */

/* out[k] = sum_b partials[k * n_partials + b] for k < n_out (fixed order) */
PSELL_API int psell_sum_partials(const double* partials, int64_t n_partials, int32_t n_out, double* out,
                       const int32_t* skip_flag, void* stream);

/* Multi-rank reductions: out[j] = sum_{i<n_parts} parts[i*stride + j] in rank order (j < n_out <= 32). */
PSELL_API int psell_sum_strided(const double* parts, int32_t n_parts, int32_t stride, int32_t n_out,
                                double* out, void* stream);

/* Generic f64 dots: out = {a.b}; a, b of dtype (f32|f64); PSELL_RED_BLOCKS partials. */
PSELL_API int psell_dot(const void* a, const void* b, int32_t dtype, int64_t n, double* partials,
              double* out, void* stream);

/* Inner reduced-precision PCG (solvers.py:278-308), f32 vectors.
 * scal[0]=rz scal[1]=pq scal[2]=alpha scal[3]=beta scal[4]=rz_new  scal[8..] local sums
 * iflags[0]=breakdown iflags[1]=done */
PSELL_API int psell_ipcg_begin(int64_t n, const double* r64, float* x, float* r, float* z, float* p,
                     const float* inv_diag, double* partials, double* local_out, void* stream);
PSELL_API int psell_ipcg_set_rz(const double* parts, int32_t n_parts, int32_t stride, double* scal, int32_t* iflags,
                      void* stream);
/* psell_ipcg_set_rz with an outer loop's gate (psell_pcg_status): gate[0] != 0
 * sets the inner breakdown flag, so the whole inner solve is a no-op. */
PSELL_API int psell_ipcg_set_rz_gated(const double* parts, int32_t n_parts, int32_t stride, double* scal,
                            int32_t* iflags, const int32_t* gate, void* stream);
PSELL_API int psell_ipcg_alpha(const double* parts, int32_t n_parts, int32_t stride, double* scal, int32_t* iflags,
                     void* stream);
PSELL_API int psell_ipcg_update(int64_t n, float* x, float* r, float* z, const float* p, const float* q,
                      const float* inv_diag, const double* scal, const int32_t* iflags,
                      double* partials, double* local_out, void* stream);
/* Single-GPU fused variants of the inner-PCG step (one launch each instead of
 * kernel + partial sum + scalar kernel).  `ticket` is a device array of
 * 1 + ceil(P / 256) unsigned ints (P = partials of the launch: psell_spmv_dot_partials
 * or PSELL_RED_BLOCKS), zero before the first call and left zero by every call;
 * `partials` holds P + ceil(P / 256) doubles.  The last CTAs of the launch sum the
 * partials in a fixed two-level order (deterministic) and perform the scalar step.  psell_spmv_dot_alpha = psell_spmv_dot + psell_sum_partials +
 * psell_ipcg_alpha (solvers.py:294-299); psell_ipcg_update_beta =
 * psell_ipcg_update + psell_ipcg_beta (solvers.py:300-306). */
PSELL_API int psell_spmv_dot_alpha(const psell_desc* desc, const void* pack, const int64_t* offset,
                                   const void* perm, const float* x, float* y, const float* p_own,
                                   double* partials, double* scal, int32_t* iflags, unsigned* ticket,
                                   int32_t flags, void* stream, psell_error* err);
PSELL_API int psell_ipcg_update_beta(int64_t n, float* x, float* r, float* z, const float* p, const float* q,
                                     const float* inv_diag, double* scal, int32_t* iflags, double* partials,
                                     unsigned* ticket, void* stream);
/* With x == NULL, psell_ipcg_update(_beta) only does r -= alpha q, z = P(r), r.z;
 * psell_ipcg_direction_x then applies x += alpha p_old and p = z + beta p_old in
 * one pass (same f32 ops, 4 fewer bytes per row per iteration). */
PSELL_API int psell_ipcg_direction_x(int64_t n, float* p, const float* z, float* x, const double* scal,
                                     const int32_t* iflags, void* stream);
/* f64 inner PCG direction (real64 inner precision): p = z + coef[0] p, skipped after a breakdown. */
PSELL_API int psell_xpby_checked(int64_t n, double* p, const double* z, const double* coef, const int32_t* iflags,
                                 void* stream);
PSELL_API int psell_ipcg_beta(const double* parts, int32_t n_parts, int32_t stride, double* scal, int32_t* iflags,
                    void* stream);
PSELL_API int psell_ipcg_direction(int64_t n, float* p, const float* z, const double* scal,
                         const int32_t* iflags, void* stream);
PSELL_API int psell_ipcg_end(int64_t n, const float* x, double* z64, void* stream);

/* Outer FCG / PCG f64 helpers (solvers.py:171-275).
 * fcg_zr:  out2 = {z.(r - r_prev), z.r}  (r_prev may be NULL: first iteration)
 * pq_pr:   out2 = {p.q, p.r}
 * axpy2:   x += a*p; r -= a*q with a = coef[0] (numpy rounding), out1 = {r.r}
 * xpby:    p = z + b*p with b = coef[0]; if coef == NULL: p = z
 * resid:   out1 = {(b - ax).(b - ax)} */
PSELL_API int psell_fcg_zr(int64_t n, const double* z, const double* r, const double* r_prev,
                 double* partials, double* out2, void* stream);
PSELL_API int psell_pq_pr(int64_t n, const double* p, const double* q, const double* r, double* partials,
                double* out2, void* stream);
PSELL_API int psell_axpy2(int64_t n, double* x, double* r, const double* p, const double* q,
                const double* coef, const int32_t* skip_flag, double* partials, double* out1,
                void* stream);
PSELL_API int psell_xpby(int64_t n, double* p, const double* z, const double* coef, void* stream);
PSELL_API int psell_resid(int64_t n, const double* b, const double* ax, double* partials, double* out1,
                void* stream);
/* z = r * inv (f64 Jacobi) and rz partial: out1 = {r.z} */
PSELL_API int psell_precond_dot(int64_t n, double* z, const double* r, const double* inv, double* partials,
                      double* out1, void* stream);
/* scalar programs on device: alpha = num/den with breakdown test, beta = num/den */
PSELL_API int psell_scalar_div(const double* num_parts, const double* den_parts, int32_t n_parts,
                     int32_t stride, double* dst, int32_t* flag, int32_t check_curvature,
                     void* stream);

/* Fused FP64 PCG iteration (identity preconditioner, one GPU; reference solvers.py:183-209,
 * the loop body of pcg): three launches per iteration instead of eleven.
 *   psell_csr_spmv_dot_alpha: q = A p (bitwise psell_csr_spmv), pq = p.q, and in the last CTA
 *     scal[1] = scal[10] = pq, gate[0] = 1 on non-positive / non-finite curvature, else
 *     scal[0] = alpha = scal[4] / pq.  A no-op when gate[0] != 0.
 *   psell_pcg_update_status: x += alpha p; r -= alpha q; scal[12] = rr = r.r (fixed order);
 *     out[3] = psell_pcg_status's {breakdown, pq, sqrt(rr) / bnorm} (gate[0] = 2 below tol);
 *     scal[2] = beta = rr / scal[4]; scal[4] = rr.
 *   then psell_xpby_checked(n, p, r, scal + 2, gate): p = r + beta p.
 * partials >= 2 * PSELL_RED_BLOCKS doubles; ticket: two zeroed regions of
 * 1 + PSELL_RED_BLOCKS / 32 counters (one per kernel), left zero. */
PSELL_API int psell_csr_spmv_dot_alpha(int64_t n_rows, const int64_t* row_ptr, const int32_t* col_idx,
                                       const double* values, const double* x, double* y, const double* p_own,
                                       double* partials, double* scal, int32_t* gate, unsigned* ticket,
                                       void* stream, psell_error* err);
PSELL_API int psell_pcg_update_status(int64_t n, double* x, double* r, const double* p, const double* q,
                                      double* scal, int32_t* gate, double bnorm, double tol, double* out,
                                      double* partials, unsigned* ticket, void* stream);

/* Fused distributed inner PCG (G ranks joined by the K8 peer arenas, reference
 * solvers.py:293-306 on a row slab): psell_spmv_dot_alpha / psell_ipcg_update_beta whose
 * last CTA all-reduces its local FP64 sum over the arenas (push into every peer's dot slot,
 * system-scope release of the epoch, acquire-wait for every peer, rank-ordered sum) before
 * the alpha / beta step -- one kernel instead of sum + exchange + scalar kernels.  peers =
 * device array of the G arena base addresses (rank order); a wait past timeout_ns sets the
 * arena's error word (psell_peer_error).  With G = 1 they are the single-GPU entry points. */
PSELL_API int psell_spmv_dot_alpha_peer(const psell_desc* d, const void* pack, const int64_t* offset,
                                        const void* perm, const float* x, float* y, const float* p_own,
                                        double* partials, double* scal, int32_t* iflags, unsigned* ticket,
                                        int32_t flags, int32_t G, int32_t rank, const uint64_t* peers,
                                        int64_t timeout_ns, void* stream, psell_error* err);
PSELL_API int psell_ipcg_update_beta_peer(int64_t n, float* x, float* r, float* z, const float* p, const float* q,
                                          const float* inv_diag, double* scal, int32_t* iflags, double* partials,
                                          unsigned* ticket, int32_t G, int32_t rank, const uint64_t* peers,
                                          int64_t timeout_ns, void* stream);

/* psell_ipcg_direction_x across G ranks with the halo push fused in: the rows listed as up
 * to 2 contiguous local ranges [lo[k], hi[k]) owed to rank dst[k] are stored into that
 * peer's arena vector (vec_off, global position row0 + row) as they are computed, and the
 * last CTA runs the K8 signal / wait -- the next SpMV's halo has arrived when it returns. */
PSELL_API int psell_ipcg_direction_x_push(int64_t n, float* p, const float* z, float* x, const double* scal,
                                          const int32_t* iflags, int32_t G, int32_t rank, const uint64_t* peers,
                                          int64_t row0, int64_t vec_off, int32_t n_ranges, const int64_t* lo,
                                          const int64_t* hi, const int32_t* dst, int64_t timeout_ns, void* stream);

/* FP64 PCG convergence gate (solvers.py:183-207): gate[2] int32 (0 running,
 * 1 breakdown -- pass gate as psell_scalar_div's flag and psell_axpy2's skip
 * flag -- 2 converged; gate[1] = breakdown reported).  out[3] = {breakdown,
 * pq, sqrt(rr) / bnorm}, out[0] = -1 when the solve had already stopped; sets
 * gate[0] = 2 once sqrt(rr) / bnorm < tol, so iterations enqueued ahead of the
 * host's status read are no-ops on x and r. */
PSELL_API int psell_pcg_status(const double* pq, const double* rr, int32_t* gate, double bnorm, double tol,
                     double* out, void* stream);

/* ---- synthetic stencil generators (device) for the BASELINE configs ----
 * Grid d0 x d1 x d2 (d0 slowest), rows [row_begin, row_end) of the matrix.
 * box = 1: 27-point (HPCG, diag = 26), box = 0: star (2*ndim+1 point, diag 2*ndim).
 * scale: 0 none, 1 sym_diag_scale (matrix.py:305-316), 2 row_sum_scale (294-302).
 * Bitwise equal to reference stencil.py:10-52 + the scaling on the host. */
PSELL_API size_t psell_gen_workspace_bytes(int64_t n_rows);
PSELL_API int psell_gen_stencil_plan(int64_t d0, int64_t d1, int64_t d2, int32_t box, double diag,
                                     int64_t row_begin, int64_t row_end, void* workspace,
                                     size_t ws_bytes, int64_t* row_ptr, int64_t* nnz_host,
                                     void* stream, psell_error* err);
PSELL_API int psell_gen_stencil_fill(int64_t d0, int64_t d1, int64_t d2, int32_t box, double diag,
                                     int32_t scale, int64_t row_begin, int64_t row_end,
                                     const int64_t* row_ptr, int32_t* col_idx, double* values,
                                     void* stream, psell_error* err);

/* ---- SELL-C-sigma comparator (reference sell.py:49-204) ----
 * Layout from psell_build_plan with a no-dummy format (w=64, d=31, fp32embed),
 * then psell_sell_fill writes values (val_dtype f64/f32/f16, direct RNE) and
 * int32 columns (padding: value 0, the row's last column).  psell_sell_spmv is
 * bitwise sell_spmv (values cast to x dtype, numpy rounding order). */
PSELL_API int psell_sell_fill(const psell_desc* desc, const int64_t* row_ptr, const int32_t* col_idx,
                              const double* values, const void* plan_workspace, const int64_t* offset,
                              int32_t val_dtype, void* val, int32_t* col, void* stream, psell_error* err);
/* The FP32 IO-CG comparator's inner operator (SELL-C-sigma f32, C = 32, f32 x): the SpMV
 * (bitwise psell_sell_spmv) fused with p_own . y and, in the last CTA, the alpha step
 * (psell_spmv_dot_alpha's contract; partials >= psell_sell_spmv_dot_partials + groups). */
PSELL_API int64_t psell_sell_spmv_dot_partials(const psell_desc* desc);
PSELL_API int psell_sell_spmv_dot_alpha(const psell_desc* desc, const void* val, int32_t val_dtype,
                                        const int32_t* col, const int64_t* offset, const void* perm, const float* x,
                                        float* y, const float* p_own, double* partials, double* scal,
                                        int32_t* iflags, unsigned* ticket, void* stream, psell_error* err);
PSELL_API int psell_sell_spmv(const psell_desc* desc, const void* val, int32_t val_dtype, const int32_t* col,
                              const int64_t* offset, const void* perm, const void* x, int32_t x_dtype,
                              void* y, void* stream, psell_error* err);

/* Config-4 power-law matrix (counter-based splitmix64 law in csrc/gen.cu), rows
 * [row_begin, row_end) of an n x n matrix; reproduced bit for bit on the host by
 * paper_2604_13433_b200.stencil.powerlaw_rows. */
PSELL_API int psell_gen_powerlaw_plan(int64_t n, uint64_t seed, const double* thresholds, int64_t row_begin, int64_t row_end,
                                      void* workspace, size_t ws_bytes, int64_t* row_ptr,
                                      int64_t* nnz_host, void* stream, psell_error* err);
PSELL_API int psell_gen_powerlaw_fill(int64_t n, uint64_t seed, const double* thresholds, int64_t row_begin, int64_t row_end,
                                      const int64_t* row_ptr, int32_t* col_idx, double* values,
                                      void* stream, psell_error* err);
/* Config 4b (SURVEY §8d's proposal): same row lengths, ~20 % of each row's entries uniform
 * over [0, n) (k_left ~ n, every d_i = 0: the dummy-heavy far-gap regime).  Law in csrc/gen.cu;
 * host mirror stencil.powerlaw_far_rows. */
PSELL_API int psell_gen_powerlaw_far_plan(int64_t n, uint64_t seed, const double* thresholds, int64_t row_begin,
                                          int64_t row_end, void* workspace, size_t ws_bytes, int64_t* row_ptr,
                                          int64_t* nnz_host, void* stream, psell_error* err);
PSELL_API int psell_gen_powerlaw_far_fill(int64_t n, uint64_t seed, const double* thresholds, int64_t row_begin,
                                          int64_t row_end, const int64_t* row_ptr, int32_t* col_idx, double* values,
                                          void* stream, psell_error* err);

/* ---- K6 metrics: backward error (replaces metrics.py:43-66 backward_error /
 * inf_norm_matrix).  One pass over the f64 CSR A (unquantised source), x and
 * y (any psell_dtype each, widened to f64).  Writes out[0] = max_i |y_i - (Ax)_i|
 * ((Ax)_i row-sequential as csr_spmv, matrix.py:272-291), out[1] = ||A||_inf
 * (max absolute row sum), out[2] = ||x||_inf; the host forms out[0] / (out[1] *
 * out[2]) and raises the reference's ValueError when the denominator is 0.
 * Order-independent maxima: bit-identical to the reference.  out is a device
 * pointer to 3 doubles. */
PSELL_API int psell_backward_error(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                                   const int32_t* col_idx, const double* values, const void* x,
                                   int32_t x_dtype, const void* y, int32_t y_dtype, double* out,
                                   void* stream, psell_error* err);

/* ---- K7 halo exchange: dst[i] = src[idx[i]] (pack the entries
 * a peer rank needs from the local slab) and dst[idx[i]] = src[i] (scatter
 * received entries to their global positions); elem_bytes 4 or 8.  Index
 * lists come from dist.Halo (built once per operator). */
PSELL_API int psell_halo_pack(int64_t n, const void* src, const int32_t* idx, void* dst, int32_t elem_bytes,
                              void* stream);
PSELL_API int psell_halo_unpack(int64_t n, const void* src, const int64_t* idx, void* dst, int32_t elem_bytes,
                                void* stream);

/* ---- K8 peer-memory exchange: the distributed PCG's halo
 * exchange and FP64 dot all-gather as ONE kernel over NVLink peer memory, so the
 * distributed inner iteration is CUDA-graph capturable (csrc/peer.cu).  The
 * reference is single-process (solvers.py:278-308 runs on one vector); this
 * replaces the NCCL all-gather / all-reduce north_star names for those steps.
 * Every rank allocates one arena (psell_peer_alloc), exports its IPC handle,
 * maps the others' (psell_peer_open) and passes the G arena bases as a device
 * array `peers` (peers[rank] = its own).  Arena layout: see csrc/peer.cu. */
#define PSELL_PEER_HDR_BYTES 12288
#define PSELL_PEER_HANDLE_BYTES 64
PSELL_API size_t psell_peer_arena_bytes(int64_t n_cols);
/* byte offset of the full-length f32 (elem_bytes 4) or f64 (8) vector inside an arena */
PSELL_API int64_t psell_peer_vec_offset(int64_t n_cols, int32_t elem_bytes);
PSELL_API int psell_peer_alloc(size_t bytes, void** out_ptr, void* out_handle /* 64 B */);
PSELL_API int psell_peer_open(const void* handle, void** out_ptr);
PSELL_API int psell_peer_close(void* ptr);
PSELL_API int psell_peer_free(void* ptr);
/* Push local[send_local[i]] to peer send_dst[i]'s vector at global row0 + send_local[i]
 * (elem_bytes 4 | 8, vector at vec_off in every arena), push loc[0..n_loc) (n_loc <= 8)
 * to every rank, signal, wait for every rank (timeout_ns), then
 * out[q*8 + k] = rank q's loc[k] (rank order).  Stream ordered, no host sync. */
PSELL_API int psell_peer_exchange(int32_t G, int32_t rank, const uint64_t* peers, int64_t n_send,
                                  const int32_t* send_dst, const int32_t* send_local, int64_t row0,
                                  const void* local, int32_t elem_bytes, int64_t vec_off, const double* loc,
                                  int32_t n_loc, double* out, int64_t timeout_ns, void* stream);
/* *out_host <- the arena's error word (nonzero: a wait timed out). Synchronous. */
PSELL_API int psell_peer_error(const void* arena, int32_t* out_host);

#ifdef __cplusplus
}
#endif
#endif /* PSELL_H */
