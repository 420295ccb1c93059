// K8 — peer-memory exchange for the row-partitioned PCG over NVLink / NVSwitch
// (SURVEY.md §8e, §8f f4).
//
// One process per GPU.  Every rank owns an "arena": one cudaMalloc'd block,
// exported with a CUDA IPC handle and mapped by every other rank of the node
// (cudaIpcOpenMemHandle, lazy peer access).  Layout (include/psell.h):
//
//   [0, 256)        uint32 flags[64]   flags[src] = last epoch src completed toward this rank
//   [256, 272)      uint32 epoch, ticket; int32 err, pad
//   [4096, 12288)   double glob[2][64][8]  per-rank FP64 dot contributions, by epoch parity
//   [12288, ...)    the full-length f32 and f64 vectors peers push halo entries into
//
// psell_peer_exchange is one kernel that does the whole collective step of the
// distributed inner / outer PCG iteration, so that iteration is a chain of
// kernels only and is captured in one CUDA graph:
//   1. push: every CTA stores this rank's halo entries (the slab rows a peer's
//      PackSELL / CSR slab reads) straight into the peers' full vectors at their
//      global positions (remote st.global over NVLink), and CTA 0 stores the up
//      to 8 local FP64 dot sums into every peer's glob[parity][rank];
//   2. signal: the last CTA to finish (ticket) fences at system scope and
//      release-stores the new epoch into flags[rank] of every peer;
//   3. wait: it then acquire-spins on its own flags[q] >= epoch for every q, and
//      copies glob[parity][q][*] into the caller's private rank-ordered buffer,
//      which the scalar kernels (psell_ipcg_alpha / _beta, psell_sum_strided)
//      sum in rank order — the same fixed order as the NCCL all-gather path, so
//      results do not depend on the transport.
// Safety of buffer reuse: a rank can run at most one exchange ahead of any
// peer (it cannot pass exchange k+1 before every peer has pushed k+1, which
// each does only after finishing exchange k), so two glob parities suffice;
// halo entries for iteration i+1 are pushed only after the dot exchanges of
// iteration i, which every peer enters after its SpMV of iteration i has read
// the halo of iteration i.
// A wait that exceeds `timeout_ns` (a dead or diverged peer) sets err and
// returns instead of hanging the GPU; the host checks it after each solve.
#include "psell_internal.cuh"

namespace psell {

template <typename T>
__global__ void __launch_bounds__(kBlock) peer_exchange_kernel(
    int G, int rank, const unsigned long long* __restrict__ peers, long long n_send,
    const int32_t* __restrict__ send_dst, const int32_t* __restrict__ send_local, long long row0,
    const T* __restrict__ local, long long vec_off, const double* __restrict__ loc, int n_loc,
    double* __restrict__ out, long long timeout_ns) {
  unsigned char* self = reinterpret_cast<unsigned char*>(peers[rank]);
  uint32_t* flags = reinterpret_cast<uint32_t*>(self + kFlagOff);
  uint32_t* epoch_p = reinterpret_cast<uint32_t*>(self + kEpochOff);
  uint32_t* ticket = reinterpret_cast<uint32_t*>(self + kTicketOff);
  int* err = reinterpret_cast<int*>(self + kErrOff);
  // the epoch only changes in the last CTA of the previous exchange (stream ordered)
  const uint32_t e = *reinterpret_cast<volatile uint32_t*>(epoch_p) + 1u;
  const int par = e & 1;

  // 1. push halo entries to their owners' peers at global positions
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < n_send; i += (long long)gridDim.x * kBlock) {
    const int32_t li = send_local[i];
    T* dst = reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(peers[send_dst[i]]) + vec_off);
    dst[row0 + li] = local[li];
  }
  //    and the local dot sums into every rank's glob[par][rank][*]
  if (blockIdx.x == 0 && threadIdx.x < G * n_loc) {
    const int p = threadIdx.x / n_loc, k = threadIdx.x % n_loc;
    double* g = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(peers[p]) + kGlobOff);
    g[(par * kPeerMax + rank) * 8 + k] = loc[k];
  }
  __threadfence_system();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;

  // 2. signal: this rank's epoch e is complete toward every peer
  if (threadIdx.x == 0) {
    __threadfence_system();
    *ticket = 0u;
    for (int p = 0; p < G; ++p)
      st_release_sys(reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(peers[p]) + kFlagOff) + rank, e);
  }
  // 3. wait for every peer's epoch e
  if (threadIdx.x < G) {
    const unsigned long long t0 = globaltimer();
    unsigned spins = 0;
    while ((int)(ld_acquire_sys(flags + threadIdx.x) - e) < 0) {
      if ((++spins & 1023u) == 0 && (long long)(globaltimer() - t0) > timeout_ns) {
        atomicExch(err, 1);
        break;
      }
    }
  }
  __syncthreads();
  if (out != nullptr && threadIdx.x < G * n_loc) {
    const int q = threadIdx.x / n_loc, k = threadIdx.x % n_loc;
    const double* g = reinterpret_cast<const double*>(self + kGlobOff);
    out[q * 8 + k] = ld_relaxed_sys(g + (par * kPeerMax + q) * 8 + k);
  }
  if (threadIdx.x == 0) *epoch_p = e;
}

}  // namespace psell

using namespace psell;

extern "C" size_t psell_peer_arena_bytes(int64_t n_cols) {
  const size_t f32 = ((size_t)n_cols * 4 + 255) & ~(size_t)255;
  return (size_t)PSELL_PEER_HDR_BYTES + f32 + (size_t)n_cols * 8;
}

extern "C" int64_t psell_peer_vec_offset(int64_t n_cols, int32_t elem_bytes) {
  if (elem_bytes == 4) return PSELL_PEER_HDR_BYTES;
  return PSELL_PEER_HDR_BYTES + ((n_cols * 4 + 255) & ~(int64_t)255);
}

extern "C" int psell_peer_alloc(size_t bytes, void** out_ptr, void* out_handle) {
  if (!out_ptr || !out_handle || bytes < PSELL_PEER_HDR_BYTES) return PSELL_EARG;
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return PSELL_ECUDA;
  if (cudaMemset(p, 0, bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(p);
    return PSELL_ECUDA;
  }
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
    cudaFree(p);
    return PSELL_ECUDA;
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == PSELL_PEER_HANDLE_BYTES, "IPC handle size");
  memcpy(out_handle, &h, sizeof(h));
  *out_ptr = p;
  return PSELL_OK;
}

extern "C" int psell_peer_open(const void* handle, void** out_ptr) {
  if (!handle || !out_ptr) return PSELL_EARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return cudaIpcOpenMemHandle(out_ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? PSELL_OK : PSELL_ECUDA;
}

extern "C" int psell_peer_close(void* ptr) {
  return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? PSELL_OK : PSELL_ECUDA;
}

extern "C" int psell_peer_free(void* ptr) { return cudaFree(ptr) == cudaSuccess ? PSELL_OK : PSELL_ECUDA; }

extern "C" int psell_peer_exchange(int32_t G, int32_t rank, const uint64_t* peers, int64_t n_send,
                                   const int32_t* send_dst, const int32_t* send_local, int64_t row0,
                                   const void* local, int32_t elem_bytes, int64_t vec_off, const double* loc,
                                   int32_t n_loc, double* out, int64_t timeout_ns, void* stream) {
  if (G < 1 || G > kPeerMax || rank < 0 || rank >= G || n_loc < 0 || n_loc > 8 || G * n_loc > kBlock ||
      !peers || (n_send > 0 && (!send_dst || !send_local || !local)) || (n_loc > 0 && !loc))
    return PSELL_EARG;
  cudaStream_t st = as_stream(stream);
  long long g = n_send > 0 ? ceil_div((long long)n_send, (long long)kBlock) : 1;
  if (g > 4 * 148) g = 4 * 148;
  const unsigned long long* pp = reinterpret_cast<const unsigned long long*>(peers);
  if (elem_bytes == 8)
    peer_exchange_kernel<uint64_t><<<(unsigned)g, kBlock, 0, st>>>(
        G, rank, pp, n_send, send_dst, send_local, row0, static_cast<const uint64_t*>(local), vec_off, loc, n_loc,
        out, timeout_ns);
  else if (elem_bytes == 4)
    peer_exchange_kernel<uint32_t><<<(unsigned)g, kBlock, 0, st>>>(
        G, rank, pp, n_send, send_dst, send_local, row0, static_cast<const uint32_t*>(local), vec_off, loc, n_loc,
        out, timeout_ns);
  else
    return PSELL_EARG;
  return cudaGetLastError() == cudaSuccess ? PSELL_OK : PSELL_ECUDA;
}

extern "C" int psell_peer_error(const void* arena, int32_t* out_host) {
  if (!arena || !out_host) return PSELL_EARG;
  return cudaMemcpy(out_host, static_cast<const unsigned char*>(arena) + kErrOff, 4, cudaMemcpyDeviceToHost) ==
                 cudaSuccess
             ? PSELL_OK
             : PSELL_ECUDA;
}
