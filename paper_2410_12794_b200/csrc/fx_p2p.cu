// Peer memory over NVLink (CUDA IPC) and a bounded cross-GPU flag barrier.
//
// The fused sharded exchange (sharded.P2PShardedLookup): every rank exports
// its staging buffers (CSR batch in, pooled rows out, barrier flags) once;
// owners' K4 launches then read the requesters' indices and store pooled
// rows into the requesters' output buffers directly through the mapped
// pointers, and two barriers per step order "inputs staged" and "outputs
// landed" across the GPUs. This replaces the reference's fan-out/response
// messages (ranker.py:298-347) and the NCCL all-to-all of the baseline path.
#include <cub/device/device_scan.cuh>

#include <cstring>

#include "fx_common.cuh"

namespace fx {

__device__ __forceinline__ void st_release_sys(int64_t *p, int64_t v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t *p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// One warp: lane r signals rank r, then lane r waits for rank r's signal.
__global__ void k_peer_barrier(int64_t *my_flags, int64_t *const *peer_flags, int rank, int world, int64_t epoch,
                               int32_t *timed_out) {
  __threadfence_system();  // order every prior write of this stream (incl. peer stores) before the signal
  for (int r = threadIdx.x; r < world; r += blockDim.x) st_release_sys(peer_flags[r] + rank, epoch);
  for (int r = threadIdx.x; r < world; r += blockDim.x) {
    long long spins = 0;
    while (ld_acquire_sys(my_flags + r) < epoch) {
      __nanosleep(200);
      if (++spins > (1ll << 25)) {  // ~10 s: never hang the GPU on a dead peer
        if (timed_out) atomicExch(timed_out, 1);
        break;
      }
    }
  }
  __syncwarp();
  __threadfence_system();
}

// Push a requester's table-wise CSR batch to the owners' staging buffers.
// grid (C, F): blockIdx.y = feature f (owned by rank feat_owner[f], its
// feat_pos[f]-th owned feature); the C blocks of a feature copy disjoint
// slices of its index range and of its B+1 rebased offsets.
template <typename IdxT>
__global__ void __launch_bounds__(256) k_push_csr(const IdxT *__restrict__ indices, const int64_t *__restrict__ offsets,
                                                  int B, int F, const int32_t *__restrict__ feat_owner,
                                                  const int32_t *__restrict__ feat_pos, int32_t *const *dst_idx,
                                                  int64_t *const *dst_offs, const int64_t *__restrict__ feat_nrows,
                                                  int64_t *err, int32_t *err_code, bool sysfence) {
  const int f = blockIdx.y;
  const int d = feat_owner[f];
  __shared__ long long s_base;
  if (threadIdx.x == 0) {
    long long base = 0;  // indices of the owner's earlier features in this requester's slot
    for (int g = 0; g < f; ++g)
      if (feat_owner[g] == d) base += offsets[(int64_t)(g + 1) * B] - offsets[(int64_t)g * B];
    s_base = base;
  }
  __syncthreads();
  const long long base = s_base;
  const int64_t b0 = offsets[(int64_t)f * B], b1 = offsets[(int64_t)(f + 1) * B];
  int32_t *di = dst_idx[d] + base;
  const int64_t n = b1 - b0;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = min(n, lo + per);
  // ingress validation fused into the copy (same check and error position as
  // K1 k_route's validate pass): idx in [0, num_rows of the feature's table)
  const int64_t nr = feat_nrows ? feat_nrows[f] : LLONG_MAX;
  // 4 independent loads in flight per thread before the peer stores
  int64_t i = lo + threadIdx.x;
  for (; i + 3 * blockDim.x < hi; i += 4 * blockDim.x) {
    IdxT v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = indices[b0 + i + u * blockDim.x];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (static_cast<int64_t>(v[u]) < 0 || static_cast<int64_t>(v[u]) >= nr)
        record_bad(err, err_code, b0 + i + u * blockDim.x, FX_E_LOOKUP_VALIDATION);
      di[i + u * blockDim.x] = static_cast<int32_t>(v[u]);
    }
  }
  for (; i < hi; i += blockDim.x) {
    const IdxT v = indices[b0 + i];
    if (static_cast<int64_t>(v) < 0 || static_cast<int64_t>(v) >= nr)
      record_bad(err, err_code, b0 + i, FX_E_LOOKUP_VALIDATION);
    di[i] = static_cast<int32_t>(v);
  }
  int64_t *dof = dst_offs[d] + (int64_t)feat_pos[f] * B;
  const int64_t pb = (B + 1 + gridDim.x - 1) / gridDim.x;
  const int64_t olo = blockIdx.x * pb, ohi = min((int64_t)B + 1, olo + pb);
  for (int64_t s = olo + threadIdx.x; s < ohi; s += blockDim.x) dof[s] = offsets[(int64_t)f * B + s] - b0 + base;
  if (sysfence) __threadfence_system();
}


// ---- row-wise push (routing.py:117-148 group_by_server, per destination rank)
__device__ __forceinline__ int route_dest(const int64_t *route_off, const int64_t *starts, const int32_t *owners,
                                          int t, int64_t idx) {
  int64_t lo = route_off[t], hi = route_off[t + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (starts[mid] <= idx) lo = mid + 1; else hi = mid;
  }
  // out-of-range indices (flagged by the requester's ingress validation) go to
  // shard 0's owner, which records a routing violation instead of reading them
  return owners[lo > route_off[t] ? lo - 1 : route_off[t]];
}

// one warp per bag: counts[d * n_bags + b] = #indices of bag b owned by rank d
template <typename IdxT, int WM>
__global__ void __launch_bounds__(256) k_rw_count(const int64_t *route_off, const int64_t *starts,
                                                  const int32_t *owners, const int32_t *bag_table,
                                                  const IdxT *indices, const int64_t *offsets, int64_t n_bags,
                                                  int W, int32_t *counts, const int32_t *hit_slot = nullptr,
                                                  int32_t *hit_cnt = nullptr) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = warp; b < n_bags; b += nw) {
    const int t = bag_table[b];
    const int64_t beg = offsets[b], end = offsets[b + 1];
    int cnt[WM];  // per-destination counts (warp-uniform, register-resident after unrolling)
#pragma unroll
    for (int d = 0; d < WM; ++d) cnt[d] = 0;
    int hits = 0;
    for (int64_t c0 = beg; c0 < end; c0 += 32) {
      const bool on = c0 + lane < end;
      const bool hit = on && hit_slot && hit_slot[c0 + lane] >= 0;  // served by the requester's cache
      const int my_d = (on && !hit)
                           ? route_dest(route_off, starts, owners, t, static_cast<int64_t>(indices[c0 + lane]))
                           : -1;
      hits += __popc(__ballot_sync(0xffffffffu, hit));
#pragma unroll
      for (int d = 0; d < WM; ++d)
        if (d < W) cnt[d] += __popc(__ballot_sync(0xffffffffu, my_d == d));
    }
#pragma unroll
    for (int d = 0; d < WM; ++d)
      if (d < W && lane == 0) counts[(int64_t)d * n_bags + b] = cnt[d];
    if (hit_cnt && lane == 0) hit_cnt[b] = hits;
  }
}

// one warp per bag: stable per-destination scatter of the bag's indices into
// rank d's staging slot (IPC pointer dst_idx[d]) at scan[d*n_bags+b] - scan[d*n_bags] + rank
template <typename IdxT, int WM>
__global__ void __launch_bounds__(256) k_rw_push(const int64_t *route_off, const int64_t *starts,
                                                 const int32_t *owners, const int32_t *bag_table,
                                                 const IdxT *indices, const int64_t *offsets, int64_t n_bags, int W,
                                                 const int64_t *scan, int32_t *const *dst_idx, bool sysfence) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int32_t *dst[WM];
  int64_t base[WM];
#pragma unroll
  for (int d = 0; d < WM; ++d) {
    dst[d] = d < W ? dst_idx[d] : nullptr;
    base[d] = d < W ? scan[(int64_t)d * n_bags] : 0;
  }
  for (int64_t b = warp; b < n_bags; b += nw) {
    const int t = bag_table[b];
    const int64_t beg = offsets[b], end = offsets[b + 1];
    int run[WM];
#pragma unroll
    for (int d = 0; d < WM; ++d) run[d] = d < W ? static_cast<int>(scan[(int64_t)d * n_bags + b] - base[d]) : 0;
    for (int64_t c0 = beg; c0 < end; c0 += 32) {
      const bool on = c0 + lane < end;
      int64_t idx = 0;
      int my_d = -1;
      if (on) {
        idx = static_cast<int64_t>(indices[c0 + lane]);
        my_d = route_dest(route_off, starts, owners, t, idx);
      }
#pragma unroll
      for (int d = 0; d < WM; ++d) {
        if (d < W) {
          const unsigned m = __ballot_sync(0xffffffffu, my_d == d);
          if (my_d == d) dst[d][run[d] + __popc(m & lt)] = static_cast<int32_t>(idx);
          run[d] += __popc(m);
        }
      }
    }
  }
  if (sysfence) __threadfence_system();
}

// per-destination bag offsets into rank d's slot: dst_offs[d][b] = scan[d*n+b] - scan[d*n], b in [0, n]
__global__ void k_rw_push_offsets(const int64_t *scan, int64_t n_bags, int W, int64_t *const *dst_offs,
                                  bool sysfence) {
  const int64_t total = (int64_t)W * (n_bags + 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = i / (n_bags + 1), b = i % (n_bags + 1);
    dst_offs[d][b] = scan[d * n_bags + b] - scan[d * n_bags];
  }
  if (sysfence) __threadfence_system();
}

// ---- planned row-wise push (pooling.py:88-100 plan_hierarchical per (bag, rank))
// thread per bag: a group of >= threshold indices is pushed down (kept in
// counts), a smaller one is raw-fetched (its count is zeroed so the push and
// the K5 partial lookup skip it); raw_cnt[b] = raw rows of bag b; counters
// [3][n_bags] = (pushdown_groups, pushdown_rows, raw_rows) (ranker.py:281-293).
__global__ void k_rw_plan(int32_t *counts, int64_t n_bags, int W, int32_t threshold, int32_t *raw_cnt,
                          int32_t *counters, const int32_t *hit_cnt) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n_bags; b += (int64_t)gridDim.x * blockDim.x) {
    int pg = 0, pr = 0, rr = 0;
    for (int d = 0; d < W; ++d) {
      const int64_t i = (int64_t)d * n_bags + b;
      const int c = counts[i];
      if (c <= 0) continue;
      if (c >= threshold) {
        ++pg;
        pr += c;
      } else {
        rr += c;
        counts[i] = 0;
      }
    }
    raw_cnt[b] = rr + (hit_cnt ? hit_cnt[b] : 0);  // cache hits join the raw vectors (ranker.py:409-411)
    if (counters) {
      counters[b] = pg;
      counters[n_bags + b] = pr;
      counters[2 * n_bags + b] = rr;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) raw_cnt[n_bags] = 0;
}

__device__ __forceinline__ int route_shard(const int64_t *route_off, const int64_t *starts, int t, int64_t idx) {
  int64_t lo = route_off[t], hi = route_off[t + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (starts[mid] <= idx) lo = mid + 1; else hi = mid;
  }
  return static_cast<int>(lo > route_off[t] ? lo - 1 : route_off[t]);
}

// one warp per bag, indices in position order: raw-fetched ones (their
// (bag, rank) group was zeroed by k_rw_plan) get the address of their row in
// the owning shard — a peer (IPC-mapped) pointer for other ranks' shards, read
// later by K5 over NVLink (the PlanMode.RAW_FETCH / RDMA-read analogue).
template <typename IdxT>
__global__ void __launch_bounds__(256) k_rw_raw(const int64_t *route_off, const int64_t *starts,
                                                const int32_t *owners, const int64_t *nrows,
                                                const int32_t *bag_table, const IdxT *indices,
                                                const int64_t *offsets, int64_t n_bags, const int32_t *counts,
                                                const int64_t *raw_off, const float *const *shard_base, int64_t ld,
                                                const float **raw_ptr, const int32_t *hit_slot,
                                                const float *cache_rows, int64_t cache_ld) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = warp; b < n_bags; b += nw) {
    const int64_t r0 = raw_off[b];
    if (raw_off[b + 1] == r0) continue;
    const int t = bag_table[b];
    const int64_t beg = offsets[b], end = offsets[b + 1];
    int64_t run = r0;
    for (int64_t c0 = beg; c0 < end; c0 += 32) {
      bool raw = false;
      const float *ptr = nullptr;
      const int32_t hs = (c0 + lane < end && hit_slot) ? hit_slot[c0 + lane] : -1;
      if (hs >= 0) {
        raw = true;
        ptr = cache_rows + static_cast<int64_t>(hs) * cache_ld;
      } else if (c0 + lane < end) {
        int64_t idx = static_cast<int64_t>(indices[c0 + lane]);
        const int sid = route_shard(route_off, starts, t, idx);
        const int d = owners[sid];
        raw = counts[(int64_t)d * n_bags + b] == 0;
        // invalid indices (flagged by ingress validation) are clamped into the shard
        const int64_t lo = starts[sid];
        const int64_t hi = sid + 1 < route_off[t + 1] ? starts[sid + 1] : nrows[t];
        idx = idx < lo ? lo : (idx >= hi ? hi - 1 : idx);
        ptr = shard_base[sid] + (idx - lo) * ld;
      }
      const unsigned m = __ballot_sync(0xffffffffu, raw);
      if (raw) raw_ptr[run + __popc(m & lt)] = ptr;
      run += __popc(m);
    }
  }
}

// k_rw_push restricted to pushed-down groups (counts[d][b] > 0 after the plan)
template <typename IdxT, int WM>
__global__ void __launch_bounds__(256) k_rw_push_planned(const int64_t *route_off, const int64_t *starts,
                                                         const int32_t *owners, const int32_t *bag_table,
                                                         const IdxT *indices, const int64_t *offsets, int64_t n_bags,
                                                         int W, const int32_t *counts, const int64_t *scan,
                                                         int32_t *const *dst_idx, const int32_t *hit_slot) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int32_t *dst[WM];
  int64_t base[WM];
#pragma unroll
  for (int d = 0; d < WM; ++d) {
    dst[d] = d < W ? dst_idx[d] : nullptr;
    base[d] = d < W ? scan[(int64_t)d * n_bags] : 0;
  }
  for (int64_t b = warp; b < n_bags; b += nw) {
    const int t = bag_table[b];
    const int64_t beg = offsets[b], end = offsets[b + 1];
    int run[WM];
    unsigned pushed = 0;
#pragma unroll
    for (int d = 0; d < WM; ++d) {
      run[d] = d < W ? static_cast<int>(scan[(int64_t)d * n_bags + b] - base[d]) : 0;
      if (d < W && counts[(int64_t)d * n_bags + b] > 0) pushed |= 1u << d;
    }
    if (!pushed) continue;
    for (int64_t c0 = beg; c0 < end; c0 += 32) {
      const bool on = c0 + lane < end;
      int64_t idx = 0;
      int my_d = -1;
      if (on && !(hit_slot && hit_slot[c0 + lane] >= 0)) {
        idx = static_cast<int64_t>(indices[c0 + lane]);
        my_d = route_dest(route_off, starts, owners, t, idx);
        if (!((pushed >> my_d) & 1u)) my_d = -1;
      }
#pragma unroll
      for (int d = 0; d < WM; ++d) {
        if (d < W && ((pushed >> d) & 1u)) {
          const unsigned m = __ballot_sync(0xffffffffu, my_d == d);
          if (my_d == d) dst[d][run[d] + __popc(m & lt)] = static_cast<int32_t>(idx);
          run[d] += __popc(m);
        }
      }
    }
  }
  __threadfence_system();
}

static inline int wm_for(int W) { return W <= 2 ? 2 : W <= 4 ? 4 : W <= 8 ? 8 : W <= 16 ? 16 : 32; }

#define FX_WM_SWITCH(W, CALL) \
  switch (wm_for(W)) {        \
    case 2: CALL(2); break;   \
    case 4: CALL(4); break;   \
    case 8: CALL(8); break;   \
    case 16: CALL(16); break; \
    default: CALL(32); break; \
  }

}  // namespace fx

using namespace fx;

extern "C" {

int fx_dev_alloc(size_t bytes, void **out) {
  *out = nullptr;
  return cuda_check(cudaMalloc(out, bytes ? bytes : 1), "fx_dev_alloc");
}

int fx_dev_free(void *ptr) { return ptr ? cuda_check(cudaFree(ptr), "fx_dev_free") : FX_OK; }

int fx_ipc_export(void *ptr, unsigned char handle_out[64]) {
  cudaIpcMemHandle_t h;
  int rc = cuda_check(cudaIpcGetMemHandle(&h, ptr), "fx_ipc_export");
  if (rc) return rc;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle_out, &h, 64);
  return FX_OK;
}

int fx_ipc_open(const unsigned char handle[64], void **out) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  *out = nullptr;
  return cuda_check(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess), "fx_ipc_open");
}

int fx_ipc_close(void *ptr) { return cuda_check(cudaIpcCloseMemHandle(ptr), "fx_ipc_close"); }

int fx_can_access_peer(int device, int peer_device) {
  int ok = 0;
  if (cudaDeviceCanAccessPeer(&ok, device, peer_device) != cudaSuccess) return -1;
  return ok;
}

int fx_memcpy_async(void *dst, const void *src, size_t bytes, void *stream) {
  if (bytes == 0) return FX_OK;
  return cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, as_stream(stream)), "fx_memcpy_async");
}

int fx_push_csr(const void *indices, int32_t idx_type, const int64_t *offsets, int32_t B, int32_t F,
                const int32_t *feat_owner, const int32_t *feat_pos, int32_t *const *dst_idx, int64_t *const *dst_offs,
                const int64_t *feat_nrows, int64_t *err, int32_t *err_code, int32_t sysfence, void *stream) {
  if (B < 1 || F < 1) {
    set_error("fx_push_csr: bad shape");
    return FX_E_CONFIG;
  }
  // blocks per SM of the push grid, split evenly across features: the push
  // runs concurrently with the previous step's gather, and one block per SM
  // steals the fewest gather slots (N=2 cfg2, same box: 1,213 vs 1,188 M
  // bags/s at 8; scripts/run_stage_ab.sh). FX_PUSH_BPS overrides.
  static const int bps = [] {
    const char *e = getenv("FX_PUSH_BPS");
    const int v = e ? atoi(e) : 1;
    return v > 0 ? v : 1;
  }();
  int per_f = (num_sms() * bps + F - 1) / F;
  if (per_f < 1) per_f = 1;
  if (per_f > 64) per_f = 64;
  dim3 grid(per_f, F);
  if (idx_type == FX_IDX_I32)
    k_push_csr<int32_t><<<grid, 256, 0, as_stream(stream)>>>(static_cast<const int32_t *>(indices), offsets, B, F,
                                                             feat_owner, feat_pos, dst_idx, dst_offs, feat_nrows, err,
                                                             err_code, sysfence != 0);
  else
    k_push_csr<int64_t><<<grid, 256, 0, as_stream(stream)>>>(static_cast<const int64_t *>(indices), offsets, B, F,
                                                             feat_owner, feat_pos, dst_idx, dst_offs, feat_nrows, err,
                                                             err_code, sysfence != 0);
  FX_LAUNCH_CHECK("fx_push_csr");
  return FX_OK;
}

int fx_rw_push(const int64_t *route_off, const int64_t *starts, const int32_t *owners, const int32_t *bag_table,
               const void *indices, int32_t idx_type, const int64_t *offsets, int64_t n_bags, int32_t W,
               int32_t *counts, int64_t *scan, int32_t *const *dst_idx, int64_t *const *dst_offs, void *ws,
               size_t *ws_bytes, void *stream) {
  if (W < 1 || W > 32 || n_bags < 0) {
    set_error("fx_rw_push: bad arguments");
    return FX_E_CONFIG;
  }
  const int64_t n = static_cast<int64_t>(W) * n_bags + 1;
  size_t need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, (const int32_t *)nullptr, (int64_t *)nullptr, static_cast<int>(n));
  if (ws == nullptr) {
    *ws_bytes = need;
    return FX_OK;
  }
  cudaStream_t st = as_stream(stream);
  cudaMemsetAsync(counts, 0, n * sizeof(int32_t), st);
  const int grid = grid_for(n_bags * 32, 256);
#define FX_COUNT(WM)                                                                                          \
  if (idx_type == FX_IDX_I32)                                                                                 \
    k_rw_count<int32_t, WM><<<grid, 256, 0, st>>>(route_off, starts, owners, bag_table,                       \
                                                  static_cast<const int32_t *>(indices), offsets, n_bags, W, counts); \
  else                                                                                                        \
    k_rw_count<int64_t, WM><<<grid, 256, 0, st>>>(route_off, starts, owners, bag_table,                       \
                                                  static_cast<const int64_t *>(indices), offsets, n_bags, W, counts);
  FX_WM_SWITCH(W, FX_COUNT)
#undef FX_COUNT
  cub::DeviceScan::ExclusiveSum(ws, need, counts, scan, static_cast<int>(n), st);
#define FX_PUSH(WM)                                                                                            \
  if (idx_type == FX_IDX_I32)                                                                                  \
    k_rw_push<int32_t, WM><<<grid, 256, 0, st>>>(route_off, starts, owners, bag_table,                         \
                                                 static_cast<const int32_t *>(indices), offsets, n_bags, W, scan,   \
                                                 dst_idx, true);                                               \
  else                                                                                                         \
    k_rw_push<int64_t, WM><<<grid, 256, 0, st>>>(route_off, starts, owners, bag_table,                         \
                                                 static_cast<const int64_t *>(indices), offsets, n_bags, W, scan,   \
                                                 dst_idx, true);
  FX_WM_SWITCH(W, FX_PUSH)
#undef FX_PUSH
  k_rw_push_offsets<<<grid_for((int64_t)W * (n_bags + 1), 256), 256, 0, st>>>(scan, n_bags, W, dst_offs, true);
  FX_LAUNCH_CHECK("fx_rw_push");
  return FX_OK;
}

int fx_rw_push_planned(const int64_t *route_off, const int64_t *starts, const int32_t *owners, const int64_t *nrows,
                       const int32_t *bag_table, const void *indices, int32_t idx_type, const int64_t *offsets,
                       int64_t n_bags, int32_t W, int32_t threshold, int32_t *counts, int64_t *scan,
                       int32_t *const *dst_idx, int64_t *const *dst_offs, const float *const *shard_base, int64_t ld,
                       int64_t *raw_off, const float **raw_ptr, int32_t *counters, const int32_t *hit_slot,
                       const float *cache_rows, int64_t cache_ld, void *ws, size_t *ws_bytes, void *stream) {
  if (W < 1 || W > 32 || n_bags < 0 || threshold < 2) {
    set_error("fx_rw_push_planned: bad arguments (threshold must be >= 2)");
    return FX_E_CONFIG;
  }
  const int64_t n = static_cast<int64_t>(W) * n_bags + 1;
  size_t c1 = 0, c2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, c1, (const int32_t *)nullptr, (int64_t *)nullptr, static_cast<int>(n));
  cub::DeviceScan::ExclusiveSum(nullptr, c2, (const int32_t *)nullptr, (int64_t *)nullptr,
                                static_cast<int>(n_bags + 1));
  const size_t cub_bytes = ((c1 > c2 ? c1 : c2) + 255) & ~size_t(255);
  const size_t need = cub_bytes + static_cast<size_t>(n_bags + 1) * 4 * 2;
  if (ws == nullptr) {
    *ws_bytes = need;
    return FX_OK;
  }
  if (*ws_bytes < need) {
    set_error("fx_rw_push_planned: workspace too small");
    return FX_E_CONFIG;
  }
  int32_t *raw_cnt = reinterpret_cast<int32_t *>(static_cast<char *>(ws) + cub_bytes);
  int32_t *hit_cnt = hit_slot ? raw_cnt + (n_bags + 1) : nullptr;
  size_t cb = cub_bytes;
  cudaStream_t st = as_stream(stream);
  cudaMemsetAsync(counts, 0, n * sizeof(int32_t), st);
  const int grid = grid_for(n_bags * 32, 256);
#define FX_COUNT(WM)                                                                                        \
  if (idx_type == FX_IDX_I32)                                                                               \
    k_rw_count<int32_t, WM><<<grid, 256, 0, st>>>(route_off, starts, owners, bag_table,                     \
                                                  static_cast<const int32_t *>(indices), offsets, n_bags, W, \
                                                  counts, hit_slot, hit_cnt);                               \
  else                                                                                                      \
    k_rw_count<int64_t, WM><<<grid, 256, 0, st>>>(route_off, starts, owners, bag_table,                     \
                                                  static_cast<const int64_t *>(indices), offsets, n_bags, W, \
                                                  counts, hit_slot, hit_cnt);
  FX_WM_SWITCH(W, FX_COUNT)
#undef FX_COUNT
  k_rw_plan<<<grid_for(n_bags + 1, 256), 256, 0, st>>>(counts, n_bags, W, threshold, raw_cnt, counters, hit_cnt);
  cub::DeviceScan::ExclusiveSum(ws, cb, raw_cnt, raw_off, static_cast<int>(n_bags + 1), st);
  cb = cub_bytes;
  cub::DeviceScan::ExclusiveSum(ws, cb, counts, scan, static_cast<int>(n), st);
  if (idx_type == FX_IDX_I32) {
    k_rw_raw<int32_t><<<grid, 256, 0, st>>>(route_off, starts, owners, nrows, bag_table,
                                            static_cast<const int32_t *>(indices), offsets, n_bags, counts, raw_off,
                                            shard_base, ld, raw_ptr, hit_slot, cache_rows, cache_ld);
#define FX_PP(WM)                                                                                             \
  k_rw_push_planned<int32_t, WM><<<grid, 256, 0, st>>>(route_off, starts, owners, bag_table,                   \
                                                       static_cast<const int32_t *>(indices), offsets, n_bags, W, \
                                                       counts, scan, dst_idx, hit_slot);
    FX_WM_SWITCH(W, FX_PP)
#undef FX_PP
  } else {
    k_rw_raw<int64_t><<<grid, 256, 0, st>>>(route_off, starts, owners, nrows, bag_table,
                                            static_cast<const int64_t *>(indices), offsets, n_bags, counts, raw_off,
                                            shard_base, ld, raw_ptr, hit_slot, cache_rows, cache_ld);
#define FX_PP(WM)                                                                                             \
  k_rw_push_planned<int64_t, WM><<<grid, 256, 0, st>>>(route_off, starts, owners, bag_table,                   \
                                                       static_cast<const int64_t *>(indices), offsets, n_bags, W, \
                                                       counts, scan, dst_idx, hit_slot);
    FX_WM_SWITCH(W, FX_PP)
#undef FX_PP
  }
  k_rw_push_offsets<<<grid_for((int64_t)W * (n_bags + 1), 256), 256, 0, st>>>(scan, n_bags, W, dst_offs, true);
  FX_LAUNCH_CHECK("fx_rw_push_planned");
  return FX_OK;
}

int fx_peer_barrier(int64_t *my_flags, int64_t *const *peer_flags, int32_t rank, int32_t world, int64_t epoch,
                    int32_t *timed_out, void *stream) {
  if (world < 1 || world > 32 || rank < 0 || rank >= world) {
    set_error("fx_peer_barrier: bad rank/world");
    return FX_E_CONFIG;
  }
  k_peer_barrier<<<1, 32, 0, as_stream(stream)>>>(my_flags, peer_flags, rank, world, epoch, timed_out);
  FX_LAUNCH_CHECK("fx_peer_barrier");
  return FX_OK;
}

}  // extern "C"
