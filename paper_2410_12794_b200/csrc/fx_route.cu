// K1 range routing + stable per-destination bucketing, K2 per-batch dedup.
//
// Reference semantics (paths under /root/reference/pkg/src/embserve):
//   RoutingTable.resolve_many   routing.py:87-97  (searchsorted 'right' - 1)
//   group_by_server             routing.py:117-148 (order-preserving groups)
//   dedup                       no counterpart; parity is
//                               np.unique(keys, return_inverse, return_counts)
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "fx_common.cuh"

namespace fx {

constexpr uint64_t kEmptyKey = ~0ull;
constexpr int kRowBits = 40;

// Group of 8 lanes per bag; lanes stride the bag's positions.
template <typename IdxT>
__global__ void __launch_bounds__(256) k_route(const int64_t *__restrict__ route_off,
                                               const int64_t *__restrict__ starts,
                                               const int32_t *__restrict__ servers,
                                               const int64_t *__restrict__ num_rows,
                                               const int32_t *__restrict__ bag_table, const IdxT *__restrict__ indices,
                                               const int64_t *__restrict__ offsets, int64_t n_bags,
                                               int32_t *__restrict__ dest, int64_t *err, int32_t *err_code) {
  constexpr int G = 8;
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int64_t ngrp = (gridDim.x * (int64_t)blockDim.x) / G;
  for (int64_t b = grp; b < n_bags; b += ngrp) {
    const int t = bag_table[b];
    const int64_t lo0 = route_off[t], hi0 = route_off[t + 1], nr = num_rows[t];
    const int64_t beg = offsets[b], end = offsets[b + 1];
    for (int64_t i = beg + gl; i < end; i += G) {
      const int64_t idx = load_index(indices + i);
      if (idx < 0 || idx >= nr) {
        record_bad(err, err_code, i, FX_E_LOOKUP_VALIDATION);
        if (dest) dest[i] = -1;
        continue;
      }
      if (!dest) continue;
      int64_t lo = lo0, hi = hi0;  // rightmost start <= idx (routing.py:80-85)
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(&starts[mid]) <= idx) lo = mid + 1; else hi = mid;
      }
      dest[i] = __ldg(&servers[lo - 1]);
    }
  }
}

__global__ void k_iota(int64_t *p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = i;
}

// per-(dest, bag) and per-dest counts; one group of 8 lanes per bag
__global__ void __launch_bounds__(256) k_bucket_counts(const int32_t *__restrict__ dest,
                                                       const int64_t *__restrict__ offsets, int64_t n_bags,
                                                       int n_dest, int64_t *dest_count, int32_t *bag_count) {
  extern __shared__ unsigned long long sh_cnt[];
  for (int d = threadIdx.x; d < n_dest; d += blockDim.x) sh_cnt[d] = 0;
  __syncthreads();
  constexpr int G = 8;
  const int gl = threadIdx.x % G;
  const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int64_t ngrp = (gridDim.x * (int64_t)blockDim.x) / G;
  for (int64_t b = grp; b < n_bags; b += ngrp) {
    for (int64_t i = offsets[b] + gl; i < offsets[b + 1]; i += G) {
      const int d = dest[i];
      if (d < 0 || d >= n_dest) continue;
      atomicAdd(&bag_count[static_cast<int64_t>(d) * n_bags + b], 1);
      atomicAdd(&sh_cnt[d], 1ull);
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < n_dest; d += blockDim.x)
    if (sh_cnt[d]) atomicAdd(reinterpret_cast<unsigned long long *>(&dest_count[d]), sh_cnt[d]);
}

// ----------------------------------------------------------------- K2 dedup
// Open-addressing hash table (linear probing, CAS on the 64-bit key).
struct DedupWS {
  uint64_t *keys;
  long long *first_ord;
  long long *last_ord;
  int32_t *count;
  int32_t *slot_of;     // per occurrence (CSR order)
  int32_t *first_flag;  // per ordinal
  int32_t *uid_scan;    // per ordinal
  int32_t *uid_of_slot;
  int64_t cap;
};

template <typename IdxT>
__global__ void __launch_bounds__(256) k_dedup_insert(DedupWS ws, const int32_t *__restrict__ bag_table,
                                                      const IdxT *__restrict__ indices,
                                                      const int64_t *__restrict__ offsets,
                                                      const int64_t *__restrict__ sm_start, int64_t n_bags) {
  constexpr int G = 8;
  const int gl = threadIdx.x % G;
  const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int64_t ngrp = (gridDim.x * (int64_t)blockDim.x) / G;
  const uint64_t mask = static_cast<uint64_t>(ws.cap - 1);
  for (int64_t b = grp; b < n_bags; b += ngrp) {
    const uint64_t thi = static_cast<uint64_t>(bag_table[b]) << kRowBits;
    const int64_t beg = offsets[b], end = offsets[b + 1], o0 = sm_start[b];
    for (int64_t i = beg + gl; i < end; i += G) {
      const uint64_t key = thi | static_cast<uint64_t>(load_index(indices + i));
      const long long ord = o0 + (i - beg);
      uint64_t h = hash_key(key) & mask;
      while (true) {
        const uint64_t prev = atomicCAS(reinterpret_cast<unsigned long long *>(&ws.keys[h]),
                                        static_cast<unsigned long long>(kEmptyKey),
                                        static_cast<unsigned long long>(key));
        if (prev == kEmptyKey || prev == key) break;
        h = (h + 1) & mask;
      }
      atomicMin(&ws.first_ord[h], ord);
      atomicMax(&ws.last_ord[h], ord);
      atomicAdd(&ws.count[h], 1);
      ws.slot_of[i] = static_cast<int32_t>(h);
    }
  }
}

template <typename IdxT>
__global__ void __launch_bounds__(256) k_dedup_flag(DedupWS ws, const int64_t *__restrict__ offsets,
                                                    const int64_t *__restrict__ sm_start, int64_t n_bags) {
  constexpr int G = 8;
  const int gl = threadIdx.x % G;
  const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int64_t ngrp = (gridDim.x * (int64_t)blockDim.x) / G;
  for (int64_t b = grp; b < n_bags; b += ngrp) {
    const int64_t beg = offsets[b], end = offsets[b + 1], o0 = sm_start[b];
    for (int64_t i = beg + gl; i < end; i += G) {
      const long long ord = o0 + (i - beg);
      ws.first_flag[ord] = (ws.first_ord[ws.slot_of[i]] == ord) ? 1 : 0;
    }
  }
}

// For each first occurrence (ordinal order) assign its unique id.
__global__ void __launch_bounds__(256) k_dedup_assign(DedupWS ws, const int64_t *__restrict__ offsets,
                                                      const int64_t *__restrict__ sm_start, int64_t n_bags,
                                                      int64_t nnz, uint64_t *uniq, int32_t *mult,
                                                      int64_t *first_ord, int64_t *last_ord, int64_t *n_uniq) {
  constexpr int G = 8;
  const int gl = threadIdx.x % G;
  const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int64_t ngrp = (gridDim.x * (int64_t)blockDim.x) / G;
  for (int64_t b = grp; b < n_bags; b += ngrp) {
    const int64_t beg = offsets[b], end = offsets[b + 1], o0 = sm_start[b];
    for (int64_t i = beg + gl; i < end; i += G) {
      const long long ord = o0 + (i - beg);
      if (!ws.first_flag[ord]) continue;
      const int32_t h = ws.slot_of[i];
      const int32_t u = ws.uid_scan[ord];
      ws.uid_of_slot[h] = u;
      uniq[u] = ws.keys[h];
      mult[u] = ws.count[h];
      first_ord[u] = ws.first_ord[h];
      last_ord[u] = ws.last_ord[h];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && nnz > 0)
    *n_uniq = static_cast<int64_t>(ws.uid_scan[nnz - 1]) + ws.first_flag[nnz - 1];
}

__global__ void k_dedup_inverse(DedupWS ws, int64_t nnz, int32_t *inverse) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
    inverse[i] = ws.uid_of_slot[ws.slot_of[i]];
}

__global__ void k_dedup_clear(DedupWS ws) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ws.cap; i += (int64_t)gridDim.x * blockDim.x) {
    ws.keys[i] = kEmptyKey;
    ws.first_ord[i] = LLONG_MAX;
    ws.last_ord[i] = -1;
    ws.count[i] = 0;
  }
}

static inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace fx

using namespace fx;

extern "C" {

int fx_route(const int64_t *route_off, const int64_t *starts, const int32_t *servers, const int64_t *num_rows,
             const int32_t *bag_table, const void *indices, int32_t idx_type, const int64_t *offsets,
             int64_t n_bags, int32_t *dest, int64_t *err, int32_t *err_code, void *stream) {
  if (n_bags < 0) {
    set_error("fx_route: bad arguments");
    return FX_E_CONFIG;
  }
  if (n_bags == 0) return FX_OK;
  cudaStream_t st = as_stream(stream);
  const int grid = grid_for(n_bags * 8, 256);
  if (idx_type == FX_IDX_I32)
    k_route<int32_t><<<grid, 256, 0, st>>>(route_off, starts, servers, num_rows, bag_table,
                                           static_cast<const int32_t *>(indices), offsets, n_bags, dest, err,
                                           err_code);
  else
    k_route<int64_t><<<grid, 256, 0, st>>>(route_off, starts, servers, num_rows, bag_table,
                                           static_cast<const int64_t *>(indices), offsets, n_bags, dest, err,
                                           err_code);
  FX_LAUNCH_CHECK("fx_route");
  return FX_OK;
}

int fx_bucket(const int32_t *dest, int64_t nnz, const int64_t *offsets, int64_t n_bags, int32_t n_dest,
              int64_t *perm, int64_t *dest_count, int32_t *bag_count, void *ws, size_t *ws_bytes, void *stream) {
  if (n_dest < 1 || n_dest > 256 || nnz < 0 || nnz > INT32_MAX) {
    set_error("fx_bucket: bad arguments");
    return FX_E_CONFIG;
  }
  int bits = 1;
  while ((1 << bits) < n_dest) ++bits;
  // layout: [sorted keys int32 nnz][iota int64 nnz][cub temp]
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (const int32_t *)nullptr, (int32_t *)nullptr,
                                  (const int64_t *)nullptr, (int64_t *)nullptr, static_cast<int>(nnz), 0, bits);
  const size_t need = align_up(nnz * sizeof(int32_t)) + align_up(nnz * sizeof(int64_t)) + align_up(cub_bytes);
  if (ws == nullptr) {
    *ws_bytes = need;
    return FX_OK;
  }
  if (*ws_bytes < need) {
    set_error("fx_bucket: workspace too small");
    return FX_E_CONFIG;
  }
  cudaStream_t st = as_stream(stream);
  char *p = static_cast<char *>(ws);
  int32_t *keys_out = reinterpret_cast<int32_t *>(p);
  p += align_up(nnz * sizeof(int32_t));
  int64_t *iota = reinterpret_cast<int64_t *>(p);
  p += align_up(nnz * sizeof(int64_t));
  cudaMemsetAsync(dest_count, 0, n_dest * sizeof(int64_t), st);
  cudaMemsetAsync(bag_count, 0, static_cast<size_t>(n_dest) * n_bags * sizeof(int32_t), st);
  if (nnz == 0) return FX_OK;
  k_iota<<<grid_for(nnz, 256), 256, 0, st>>>(iota, nnz);
  cub::DeviceRadixSort::SortPairs(p, cub_bytes, dest, keys_out, iota, perm, static_cast<int>(nnz), 0, bits, st);
  k_bucket_counts<<<grid_for(n_bags * 8, 256), 256, n_dest * sizeof(unsigned long long), st>>>(
      dest, offsets, n_bags, n_dest, dest_count, bag_count);
  FX_LAUNCH_CHECK("fx_bucket");
  return FX_OK;
}

int fx_dedup(const int32_t *bag_table, const void *indices, int32_t idx_type, const int64_t *offsets,
             const int64_t *sm_start, int64_t n_bags, int64_t nnz, uint64_t *uniq, int32_t *mult,
             int64_t *first_ord, int64_t *last_ord, int32_t *inverse, int64_t *n_uniq_dev, void *ws,
             size_t *ws_bytes, void *stream) {
  if (nnz < 0 || nnz > (INT32_MAX / 2)) {
    set_error("fx_dedup: nnz out of range");
    return FX_E_CONFIG;
  }
  int64_t cap = 1024;
  while (cap < 2 * nnz) cap <<= 1;
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const int32_t *)nullptr, (int32_t *)nullptr,
                                static_cast<int>(nnz > 0 ? nnz : 1));
  const size_t need = align_up(cap * 8) * 3 + align_up(cap * 4) * 2 + align_up(nnz * 4) * 3 + align_up(scan_bytes);
  if (ws == nullptr) {
    *ws_bytes = need;
    return FX_OK;
  }
  if (*ws_bytes < need) {
    set_error("fx_dedup: workspace too small");
    return FX_E_CONFIG;
  }
  cudaStream_t st = as_stream(stream);
  char *p = static_cast<char *>(ws);
  DedupWS w;
  w.cap = cap;
  w.keys = reinterpret_cast<uint64_t *>(p); p += align_up(cap * 8);
  w.first_ord = reinterpret_cast<long long *>(p); p += align_up(cap * 8);
  w.last_ord = reinterpret_cast<long long *>(p); p += align_up(cap * 8);
  w.count = reinterpret_cast<int32_t *>(p); p += align_up(cap * 4);
  w.uid_of_slot = reinterpret_cast<int32_t *>(p); p += align_up(cap * 4);
  w.slot_of = reinterpret_cast<int32_t *>(p); p += align_up(nnz * 4);
  w.first_flag = reinterpret_cast<int32_t *>(p); p += align_up(nnz * 4);
  w.uid_scan = reinterpret_cast<int32_t *>(p); p += align_up(nnz * 4);
  if (nnz == 0) {
    cudaMemsetAsync(n_uniq_dev, 0, sizeof(int64_t), st);
    return FX_OK;
  }
  k_dedup_clear<<<grid_for(cap, 256), 256, 0, st>>>(w);
  const int grid = grid_for(n_bags * 8, 256);
  if (idx_type == FX_IDX_I32) {
    k_dedup_insert<int32_t><<<grid, 256, 0, st>>>(w, bag_table, static_cast<const int32_t *>(indices), offsets,
                                                  sm_start, n_bags);
    k_dedup_flag<int32_t><<<grid, 256, 0, st>>>(w, offsets, sm_start, n_bags);
  } else {
    k_dedup_insert<int64_t><<<grid, 256, 0, st>>>(w, bag_table, static_cast<const int64_t *>(indices), offsets,
                                                  sm_start, n_bags);
    k_dedup_flag<int64_t><<<grid, 256, 0, st>>>(w, offsets, sm_start, n_bags);
  }
  cub::DeviceScan::ExclusiveSum(p, scan_bytes, w.first_flag, w.uid_scan, static_cast<int>(nnz), st);
  k_dedup_assign<<<grid, 256, 0, st>>>(w, offsets, sm_start, n_bags, nnz, uniq, mult, first_ord, last_ord,
                                       n_uniq_dev);
  k_dedup_inverse<<<grid_for(nnz, 256), 256, 0, st>>>(w, nnz, inverse);
  FX_LAUNCH_CHECK("fx_dedup");
  return FX_OK;
}

}  // extern "C"
