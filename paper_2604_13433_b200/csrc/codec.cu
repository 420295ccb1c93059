// Value codecs and word (un)packing on device: replaces encode_values,
// decode_patterns, pack_words and unpack_words (reference codec.py:173-250).
// These back the module-level codec API of the drop-in; the builder and the
// SpMV inline the same device functions (psell_internal.cuh).
#include "psell_internal.cuh"

namespace psell {

constexpr long long kMax = 0x7FFFFFFFFFFFFFFFll;

__global__ void encode_kernel(Fmt f, const double* __restrict__ v, long long n, void* out,
                              long long* bad /* [nonfinite, overflow] */) {
  long long nf = kMax, of = kMax;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int st = ENC_OK;
    const uint64_t p = encode_value(f, v[i], st);
    if (f.w == 32) static_cast<uint32_t*>(out)[i] = (uint32_t)p;
    else static_cast<uint64_t*>(out)[i] = p;
    if (st == ENC_NONFINITE) nf = i < nf ? i : nf;
    else if (st == ENC_OVERFLOW) of = i < of ? i : of;
  }
  if (nf != kMax) atomicMin(&bad[0], nf);
  if (of != kMax) atomicMin(&bad[1], of);
}

__global__ void init_bad_kernel(long long* bad) { bad[0] = kMax; bad[1] = kMax; }

// decode_patterns (codec.py:184-192): fp16 -> half bits, e8my -> f32 bits << (D+1),
// fp32embed -> (p >> (V-32)) as f32
__global__ void decode_kernel(Fmt f, const void* __restrict__ pat, long long n, void* out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (f.codec == PSELL_FP16) {
      static_cast<uint16_t*>(out)[i] = (uint16_t)static_cast<const uint32_t*>(pat)[i];
    } else if (f.codec == PSELL_E8MY) {
      static_cast<uint32_t*>(out)[i] = static_cast<const uint32_t*>(pat)[i] << (f.d + 1);
    } else {
      static_cast<uint32_t*>(out)[i] =
          (uint32_t)(static_cast<const uint64_t*>(pat)[i] >> (f.v() - 32));
    }
  }
}

// pack_words (codec.py:210-224); deltas reduce modulo 2^W like numpy's astype
template <typename W>
__global__ void pack_words_kernel(Fmt f, const W* __restrict__ pat, const int64_t* __restrict__ dl,
                                  const uint8_t* __restrict__ fl, long long n, W* out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const W d = (W)dl[i];
    out[i] = fl[i] ? (W)((pat[i] << (f.d + 1)) | (d << 1) | W(1)) : (W)(d << 1);
  }
}

// unpack_words (codec.py:227-250)
template <typename W>
__global__ void unpack_words_kernel(Fmt f, const W* __restrict__ words, long long n, void* vals,
                                    uint64_t* deltas, uint8_t* flags) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const W w = words[i];
    deltas[i] = (uint64_t)unpack_delta<W>(w, f.d);
    flags[i] = (uint8_t)(w & W(1));
    if (f.codec == PSELL_FP16) static_cast<__half*>(vals)[i] = fp16_value((uint32_t)w);
    else if (f.codec == PSELL_E8MY) static_cast<float*>(vals)[i] = e8my_value((uint32_t)w, f.d);
    else static_cast<float*>(vals)[i] = fp32e_value((uint64_t)w);
  }
}

static unsigned grid_for(long long n) {
  long long g = ceil_div(n, kBlock);
  if (g > 148 * 16) g = 148 * 16;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace psell

using namespace psell;

extern "C" {

int psell_encode(const psell_desc* d, const double* values, int64_t n, void* patterns,
                 void* ws16, void* stream, psell_error* err) {
  if (!d || !fmt_valid(fmt_of(d))) return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, "invalid PackFormat");
  if (!ws16) return set_err(err, PSELL_EARG, PSELL_KIND_PARAM, -1, 0, 0, "missing 16-byte workspace");
  cudaStream_t st = as_stream(stream);
  long long* bad = static_cast<long long*>(ws16);
  init_bad_kernel<<<1, 1, 0, st>>>(bad);
  if (n > 0) encode_kernel<<<grid_for(n), kBlock, 0, st>>>(fmt_of(d), values, n, patterns, bad);
  PSELL_CHECK_LAUNCH(err, "psell_encode");
  long long hb[2];
  PSELL_CUDA(cudaMemcpyAsync(hb, bad, 16, cudaMemcpyDeviceToHost, st), err);
  PSELL_CUDA(cudaStreamSynchronize(st), err);
  if (hb[0] != kMax || hb[1] != kMax) {
    const bool nf = hb[0] != kMax;
    const long long pos = nf ? hb[0] : hb[1];
    double v = 0;
    PSELL_CUDA(cudaMemcpyAsync(&v, values + pos, 8, cudaMemcpyDeviceToHost, st), err);
    PSELL_CUDA(cudaStreamSynchronize(st), err);
    return set_err(err, PSELL_ECODEC, nf ? PSELL_KIND_NONFINITE : PSELL_KIND_OVERFLOW, pos, 0, v,
                   nf ? "non-finite value" : "value overflows the codec");
  }
  return ok(err);
}

int psell_decode(const psell_desc* d, const void* patterns, int64_t n, void* values, void* stream,
                 psell_error* err) {
  if (!d || !fmt_valid(fmt_of(d))) return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, "invalid PackFormat");
  if (n > 0) decode_kernel<<<grid_for(n), kBlock, 0, as_stream(stream)>>>(fmt_of(d), patterns, n, values);
  PSELL_CHECK_LAUNCH(err, "psell_decode");
  return ok(err);
}

int psell_pack_words(const psell_desc* d, const void* patterns, const int64_t* deltas,
                     const uint8_t* flags, int64_t n, void* words, void* stream, psell_error* err) {
  if (!d || !fmt_valid(fmt_of(d))) return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, "invalid PackFormat");
  if (n > 0) {
    if (d->w == 32)
      pack_words_kernel<uint32_t><<<grid_for(n), kBlock, 0, as_stream(stream)>>>(
          fmt_of(d), static_cast<const uint32_t*>(patterns), deltas, flags, n, static_cast<uint32_t*>(words));
    else
      pack_words_kernel<uint64_t><<<grid_for(n), kBlock, 0, as_stream(stream)>>>(
          fmt_of(d), static_cast<const uint64_t*>(patterns), deltas, flags, n, static_cast<uint64_t*>(words));
  }
  PSELL_CHECK_LAUNCH(err, "psell_pack_words");
  return ok(err);
}

int psell_unpack_words(const psell_desc* d, const void* words, int64_t n, void* values,
                       uint64_t* deltas, uint8_t* flags, void* stream, psell_error* err) {
  if (!d || !fmt_valid(fmt_of(d))) return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, "invalid PackFormat");
  if (!fmt_device_ok(fmt_of(d))) return set_err(err, PSELL_EVALUE, PSELL_KIND_PARAM, -1, 0, 0, PSELL_FP16_W64_MSG);
  if (n > 0) {
    if (d->w == 32)
      unpack_words_kernel<uint32_t><<<grid_for(n), kBlock, 0, as_stream(stream)>>>(
          fmt_of(d), static_cast<const uint32_t*>(words), n, values, deltas, flags);
    else
      unpack_words_kernel<uint64_t><<<grid_for(n), kBlock, 0, as_stream(stream)>>>(
          fmt_of(d), static_cast<const uint64_t*>(words), n, values, deltas, flags);
  }
  PSELL_CHECK_LAUNCH(err, "psell_unpack_words");
  return ok(err);
}

}  // extern "C"
