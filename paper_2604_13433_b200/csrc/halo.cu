// K7 — halo exchange pack / unpack for the row-partitioned PCG.
//
// A rank's PackSELL / CSR slab reads x only at the columns its rows touch; for
// banded matrices that is its own slab plus a thin halo from the neighbouring
// ranks (7-point 256^3 over 8 GPUs: 2 planes = 128 K entries instead of the
// 14.7 M-entry all-gather).  pack gathers the entries a peer needs from the
// local slab into a contiguous send buffer; unpack scatters the received
// entries into their global positions of the rank's full-length vector.  Both
// are unit-stride on the buffer side; the index lists are built once per
// operator (dist.Halo).  4- and 8-byte elements (the f32 inner and f64 outer
// vectors) move as raw words.
#include "psell_internal.cuh"

namespace psell {

template <typename T>
__global__ void __launch_bounds__(kBlock) halo_pack_kernel(long long n, const T* __restrict__ src,
                                                           const int32_t* __restrict__ idx, T* __restrict__ dst) {
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long long)gridDim.x * kBlock)
    dst[i] = src[idx[i]];
}

template <typename T>
__global__ void __launch_bounds__(kBlock) halo_unpack_kernel(long long n, const T* __restrict__ src,
                                                             const int64_t* __restrict__ idx, T* __restrict__ dst) {
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long long)gridDim.x * kBlock)
    dst[idx[i]] = src[i];
}

static unsigned halo_grid(long long n) {
  const long long g = ceil_div(n, kBlock);
  return (unsigned)(g < 4096 ? (g > 0 ? g : 1) : 4096);
}

}  // namespace psell

using namespace psell;

extern "C" int psell_halo_pack(int64_t n, const void* src, const int32_t* idx, void* dst, int32_t elem_bytes,
                               void* stream) {
  if (n <= 0) return 0;
  cudaStream_t st = as_stream(stream);
  if (elem_bytes == 4)
    halo_pack_kernel<uint32_t><<<halo_grid(n), kBlock, 0, st>>>(n, static_cast<const uint32_t*>(src), idx,
                                                                static_cast<uint32_t*>(dst));
  else if (elem_bytes == 8)
    halo_pack_kernel<uint64_t><<<halo_grid(n), kBlock, 0, st>>>(n, static_cast<const uint64_t*>(src), idx,
                                                                static_cast<uint64_t*>(dst));
  else
    return 1;
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

extern "C" int psell_halo_unpack(int64_t n, const void* src, const int64_t* idx, void* dst, int32_t elem_bytes,
                                 void* stream) {
  if (n <= 0) return 0;
  cudaStream_t st = as_stream(stream);
  if (elem_bytes == 4)
    halo_unpack_kernel<uint32_t><<<halo_grid(n), kBlock, 0, st>>>(n, static_cast<const uint32_t*>(src), idx,
                                                                  static_cast<uint32_t*>(dst));
  else if (elem_bytes == 8)
    halo_unpack_kernel<uint64_t><<<halo_grid(n), kBlock, 0, st>>>(n, static_cast<const uint64_t*>(src), idx,
                                                                  static_cast<uint64_t*>(dst));
  else
    return 1;
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
