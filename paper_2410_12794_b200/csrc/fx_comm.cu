// fx_comm: the SURVEY §8(b) communicator / all-to-allv of the C-ABI, over
// CUDA-IPC-mapped peer memory of one NVLink/NVSwitch node (no NCCL).
//
// The reference's fan-out (ranker.py:263-347, post_subrequest ->
// _server_handler -> _on_response over the transport) moves sub-requests to
// the owners and pooled partials back. On one B200 node the two exchange
// legs are one-sided peer stores: every rank owns a receive window of
// `world` slots of `slot_bytes` and a flag / count area; the sender writes
// its slice for rank d straight into slot [rank] of d's window (16-byte
// stores over NVLink when aligned), records the byte count next to it, then
// the ranks meet in a release/acquire peer barrier (as in fx_p2p.cu). The
// whole exchange is one kernel + one barrier kernel on the caller's stream,
// with device-resident counts (no host sync). Windows are double-buffered
// by exchange parity: exchange k+1 writes the other half than exchange k,
// which its owner consumes on its stream before it enqueues exchange k+1,
// and exchange k+2 (k's half again) cannot start before every rank passed
// the barrier of exchange k+1.
#include <cstring>
#include <vector>

#include "fx_common.cuh"

namespace fx {

__device__ __forceinline__ void st_release_sys64(int64_t *p, int64_t v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_acquire_sys64(const int64_t *p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// window layout (one allocation, exported once): [2 halves x world x
// slot_bytes data][2 halves x world int64 counts][world int64 barrier flags]
struct CommPeers {
  unsigned char *win[32];   // this exchange's half of each rank's data area
  int64_t *counts[32];      // this exchange's half of each rank's count area
  int64_t *flags[32];
};

// grid (C, world): blockIdx.y = destination; the C blocks copy disjoint
// 16-byte pieces of the slice (bytes when unaligned), block 0 writes the count
__global__ void __launch_bounds__(256) k_alltoallv(const unsigned char *__restrict__ send,
                                                   const int64_t *__restrict__ counts,
                                                   const int64_t *__restrict__ displs, CommPeers peers, int rank,
                                                   int64_t slot_bytes, int32_t *overflow) {
  const int d = blockIdx.y;
  int64_t n = counts[d];
  if (n > slot_bytes) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(overflow, 1);
    n = slot_bytes;
  }
  const unsigned char *src = send + displs[d];
  unsigned char *dst = peers.win[d] + static_cast<int64_t>(rank) * slot_bytes;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    const int64_t n16 = n >> 4;
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
    uint4 *d4 = reinterpret_cast<uint4 *>(dst);
    int64_t i = tid;
    for (; i + 3 * T < n16; i += 4 * T) {  // four 16-byte stores in flight per thread
      const uint4 a = __ldg(s4 + i), b = __ldg(s4 + i + T), c = __ldg(s4 + i + 2 * T), e = __ldg(s4 + i + 3 * T);
      d4[i] = a;
      d4[i + T] = b;
      d4[i + 2 * T] = c;
      d4[i + 3 * T] = e;
    }
    for (; i < n16; i += T) d4[i] = __ldg(s4 + i);
    for (int64_t i = (n16 << 4) + tid; i < n; i += T) dst[i] = src[i];
  } else {
    for (int64_t i = tid; i < n; i += T) dst[i] = src[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) peers.counts[d][rank] = n;
}

__global__ void k_comm_barrier(CommPeers peers, int64_t *my_flags, int rank, int world, int64_t epoch,
                               int32_t *timed_out) {
  __threadfence_system();  // every peer store of this stream before the signal
  for (int r = threadIdx.x; r < world; r += blockDim.x) st_release_sys64(peers.flags[r] + rank, epoch);
  for (int r = threadIdx.x; r < world; r += blockDim.x) {
    long long spins = 0;
    while (ld_acquire_sys64(my_flags + r) < epoch) {
      __nanosleep(200);
      if (++spins > (1ll << 25)) {  // ~10 s: never hang the GPU on a dead peer
        atomicExch(timed_out, 1);
        break;
      }
    }
  }
  __syncwarp();
  __threadfence_system();
}

}  // namespace fx

struct fx_comm {
  int32_t rank = 0, world = 1;
  int64_t slot_bytes = 0;
  unsigned char *base = nullptr;  // my window allocation
  size_t bytes = 0;
  unsigned char *pbase[32] = {nullptr};  // every rank's window base (mine included)
  std::vector<void *> opened;     // IPC mappings of the peers' windows
  int32_t *status = nullptr;      // [0] overflow, [1] barrier timeout
  int64_t epoch = 0;
};

using namespace fx;

extern "C" {

int fx_comm_init(fx_comm **out, int32_t rank, int32_t world, int64_t slot_bytes) {
  if (!out || world < 1 || world > 32 || rank < 0 || rank >= world || slot_bytes < 0) {
    set_error("fx_comm_init: bad rank / world / slot size");
    return FX_E_CONFIG;
  }
  fx_comm *c = new fx_comm();
  c->rank = rank;
  c->world = world;
  c->slot_bytes = (slot_bytes + 15) / 16 * 16;
  c->bytes = 2 * static_cast<size_t>(world) * c->slot_bytes + 3 * static_cast<size_t>(world) * 8;
  int rc = cuda_check(cudaMalloc(&c->base, c->bytes), "fx_comm_init: window");
  rc = rc ? rc : cuda_check(cudaMemset(c->base, 0, c->bytes), "fx_comm_init: window");
  rc = rc ? rc : cuda_check(cudaMalloc(&c->status, 2 * sizeof(int32_t)), "fx_comm_init: status");
  rc = rc ? rc : cuda_check(cudaMemset(c->status, 0, 2 * sizeof(int32_t)), "fx_comm_init: status");
  if (rc) {
    if (c->base) cudaFree(c->base);
    if (c->status) cudaFree(c->status);
    delete c;
    return rc;
  }
  *out = c;
  return FX_OK;
}

int fx_comm_handle(fx_comm *c, unsigned char handle_out[64]) {
  cudaIpcMemHandle_t h;
  int rc = cuda_check(cudaIpcGetMemHandle(&h, c->base), "fx_comm_handle");
  if (rc == FX_OK) std::memcpy(handle_out, &h, 64);
  return rc;
}

namespace {
int64_t half_bytes(const fx_comm *c) { return static_cast<int64_t>(c->world) * c->slot_bytes; }
unsigned char *data_half(const fx_comm *c, unsigned char *base, int64_t epoch) {
  return base + (epoch & 1) * half_bytes(c);
}
int64_t *count_half(const fx_comm *c, unsigned char *base, int64_t epoch) {
  return reinterpret_cast<int64_t *>(base + 2 * half_bytes(c)) + (epoch & 1) * c->world;
}
int64_t *flag_area(const fx_comm *c, unsigned char *base) {
  return reinterpret_cast<int64_t *>(base + 2 * half_bytes(c)) + 2 * c->world;
}
}  // namespace

int fx_comm_connect(fx_comm *c, const unsigned char *handles) {
  for (int r = 0; r < c->world; ++r) {
    unsigned char *p = nullptr;
    if (r == c->rank) {
      p = c->base;
    } else {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + 64 * r, 64);
      void *q = nullptr;
      int rc = cuda_check(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess), "fx_comm_connect");
      if (rc) return rc;
      c->opened.push_back(q);
      p = static_cast<unsigned char *>(q);
    }
    c->pbase[r] = p;
  }
  return FX_OK;
}

// the receive half of the last exchange: slot s (bytes [s*slot, s*slot + count[s]))
// holds what rank s sent to this rank
void *fx_comm_recv_buffer(fx_comm *c) { return c ? data_half(c, c->base, c->epoch) : nullptr; }

const int64_t *fx_comm_recv_counts(fx_comm *c) { return c ? count_half(c, c->base, c->epoch) : nullptr; }

int fx_alltoallv(fx_comm *c, const void *send, const int64_t *send_counts, const int64_t *send_displs,
                 void *stream) {
  if (!c || !send_counts || !send_displs || (!send && c->slot_bytes > 0)) {
    set_error("fx_alltoallv: bad arguments");
    return FX_E_CONFIG;
  }
  if (c->pbase[c->world > 1 ? (c->rank + 1) % c->world : 0] == nullptr) {
    set_error("fx_alltoallv: fx_comm_connect has not run");
    return FX_E_CONFIG;
  }
  cudaStream_t st = as_stream(stream);
  c->epoch += 1;
  CommPeers peers;
  for (int r = 0; r < c->world; ++r) {
    peers.win[r] = data_half(c, c->pbase[r], c->epoch);
    peers.counts[r] = count_half(c, c->pbase[r], c->epoch);
    peers.flags[r] = flag_area(c, c->pbase[r]);
  }
  const int C = 4 * num_sms() / c->world > 1 ? 4 * num_sms() / c->world : 1;
  k_alltoallv<<<dim3(C, c->world), 256, 0, st>>>(static_cast<const unsigned char *>(send), send_counts, send_displs,
                                                 peers, c->rank, c->slot_bytes, c->status);
  k_comm_barrier<<<1, 32, 0, st>>>(peers, flag_area(c, c->base), c->rank, c->world, c->epoch, c->status + 1);
  FX_LAUNCH_CHECK("fx_alltoallv");
  return FX_OK;
}

int fx_comm_status(fx_comm *c, int32_t *overflow, int32_t *timed_out) {
  int32_t h[2] = {0, 0};
  int rc = cuda_check(cudaMemcpy(h, c->status, sizeof(h), cudaMemcpyDeviceToHost), "fx_comm_status");
  if (overflow) *overflow = h[0];
  if (timed_out) *timed_out = h[1];
  return rc;
}

int fx_comm_destroy(fx_comm *c) {
  if (!c) return FX_OK;
  for (void *p : c->opened) cudaIpcCloseMemHandle(p);
  if (c->base) cudaFree(c->base);
  if (c->status) cudaFree(c->status);
  delete c;
  return FX_OK;
}

}  // extern "C"
