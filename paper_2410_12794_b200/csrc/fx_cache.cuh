// Shared definitions of the GPU hot-row cache (fx_cache.cu) and the fused
// per-batch cache step (fx_step.cu): device scalars, the cache view, the
// open-addressing hash helpers and the host handle.
#pragma once

#include <climits>
#include <vector>

#include "fx_ckptr.cuh"
#include "fx_common.cuh"

namespace fx {

constexpr uint64_t kEmpty = ~0ull;
constexpr uint64_t kTomb = ~0ull - 1;
constexpr long long kFree = LLONG_MAX;
constexpr int kRowBitsC = 40;
constexpr uint64_t kRowMask = (1ull << kRowBitsC) - 1;

struct Scalars {
  long long budget, used, tick, hits, misses, entries;
  long long free_top, sketch_live, sketch_tomb, hash_tomb, pending;
  long long n_evlog, n_acc, n_ev, n_cand, staged;
  long long err;   // 1: eviction queue exhausted (the reference's popitem on an empty
                   //    OrderedDict), 2: pooled-key fingerprint collision
  long long n_ov;  // in-place pooled re-puts recorded by the last put call
  long long n_par_puts;  // put calls resolved by the parallel closed form (cumulative)
  long long tiles_bulk, tiles_chain;  // k_offer_par sketch tiles resolved as one run / by peeling (cumulative)
};

struct CacheView {
  Scalars *sc;
  CkPtr<uint64_t> hkeys;
  CkPtr<int32_t> hslot;
  int64_t hcap;
  CkPtr<uint64_t> skey;
  CkPtr<uint64_t> skey2;  // second fingerprint of pooled-result keys (0 for row keys)
  CkPtr<long long> stick;
  CkPtr<int32_t> ssize;
  CkPtr<int32_t> shits;
  CkPtr<float> rows;
  int64_t scap;
  int32_t row_ld;
  CkPtr<int32_t> free_stack;
  CkPtr<uint64_t> kkeys;
  CkPtr<double> kval;
  CkPtr<uint8_t> kflag;
  int64_t kcap;
  CkPtr<uint64_t> pend;
  int64_t pend_cap;
  CkPtr<uint64_t> evlog;
  int64_t evlog_cap;
  const fx_table_dir *dir;
  int32_t n_dir;
  const int32_t *tbytes;
  int32_t n_tbytes;
  int32_t admission;
  double decay, prune;
};

// ---------------------------------------------------------------- hashing
__device__ __forceinline__ int32_t h_find(const CacheView &c, uint64_t key) {
  const uint64_t m = static_cast<uint64_t>(c.hcap - 1);
  uint64_t h = hash_key(key) & m;
  for (int64_t probe = 0; probe < c.hcap; ++probe) {
    const uint64_t k = c.hkeys[h];
    if (k == key) return c.hslot[h];
    if (k == kEmpty) return -1;
    h = (h + 1) & m;
  }
  return -1;
}

__device__ __forceinline__ void h_insert(const CacheView &c, uint64_t key, int32_t slot) {
  const uint64_t m = static_cast<uint64_t>(c.hcap - 1);
  uint64_t h = hash_key(key) & m;
  while (true) {
    const unsigned long long prev =
        atomicCAS(reinterpret_cast<unsigned long long *>(&c.hkeys[h]), (unsigned long long)kEmpty,
                  (unsigned long long)key);
    if (prev == kEmpty || prev == key) {
      c.hslot[h] = slot;
      return;
    }
    h = (h + 1) & m;
  }
}

__device__ __forceinline__ bool h_erase(const CacheView &c, uint64_t key) {
  const uint64_t m = static_cast<uint64_t>(c.hcap - 1);
  uint64_t h = hash_key(key) & m;
  for (int64_t probe = 0; probe < c.hcap; ++probe) {
    const uint64_t k = c.hkeys[h];
    if (k == key) {
      c.hkeys[h] = kTomb;
      return true;
    }
    if (k == kEmpty) return false;
    h = (h + 1) & m;
  }
  return false;
}

__device__ __forceinline__ int64_t k_find(const CacheView &c, uint64_t key) {
  const uint64_t m = static_cast<uint64_t>(c.kcap - 1);
  uint64_t h = hash_key(key) & m;
  for (int64_t probe = 0; probe < c.kcap; ++probe) {
    const uint64_t k = c.kkeys[h];
    if (k == key) return static_cast<int64_t>(h);
    if (k == kEmpty) return -1;
    h = (h + 1) & m;
  }
  return -1;
}

__device__ __forceinline__ double k_est(const CacheView &c, uint64_t key) {
  const int64_t i = k_find(c, key);
  return i >= 0 ? c.kval[i] : 0.0;
}

// insert-or-add (returns true when the key was new)
__device__ __forceinline__ bool k_add(const CacheView &c, uint64_t key, double w) {
  const uint64_t m = static_cast<uint64_t>(c.kcap - 1);
  uint64_t h = hash_key(key) & m;
  while (true) {
    const unsigned long long prev =
        atomicCAS(reinterpret_cast<unsigned long long *>(&c.kkeys[h]), (unsigned long long)kEmpty,
                  (unsigned long long)key);
    if (prev == kEmpty || prev == key) {
      atomicAdd(&c.kval[h], w);
      return prev == kEmpty;
    }
    h = (h + 1) & m;
  }
}

__device__ __forceinline__ int32_t table_bytes_of(const CacheView &c, uint64_t key) {
  const int64_t t = static_cast<int64_t>(key >> kRowBitsC);
  return (t >= 0 && t < c.n_tbytes) ? c.tbytes[t] : -1;
}

__device__ __forceinline__ const float *dir_row(const CacheView &c, uint64_t key, int32_t *dim) {
  const int32_t t = static_cast<int32_t>(key >> kRowBitsC);
  const int64_t r = static_cast<int64_t>(key & kRowMask);
  for (int i = 0; i < c.n_dir; ++i) {
    const fx_table_dir &d = c.dir[i];
    if (d.table == t && r >= d.row_begin && r < d.row_end) {
      *dim = d.dim;
      return d.base + (r - d.row_begin) * d.ld;
    }
  }
  *dim = 0;
  return nullptr;
}

}  // namespace fx

struct fx_cache {
  using CacheView = fx::CacheView;
  CacheView v;
  int32_t record;
  std::vector<fx_table_dir> dir_host;
  std::vector<int32_t> tbytes_host;
  fx_table_dir *dir_dev = nullptr;
  int32_t *tbytes_dev = nullptr;
  void *ws = nullptr;
  size_t ws_bytes = 0;
  int32_t uniform = 0;             // common row size of every table (0 unset, -1 mixed)
  int parallel_offers = 1;         // use k_offer_par when sizes are uniform
  uint64_t *last_ev = nullptr;     // keys evicted by the last offer/apply/resize
  int64_t last_ev_cap = 0;
  const float *const *pending_rows = nullptr;  // optional per-pending-key row pointers
  int32_t *lru_hist = nullptr;     // 65536 bins + counter for the partial LRU order
  // LRU queue kept by the fused batch step (fx_step.cu): q[0, entries) = the
  // occupied slots in ascending last_tick order, -1 beyond. Any other entry
  // point that moves entries (probe, offer, resize, apply, pooled ops,
  // reserve_slots) clears queue_valid; the next step rebuilds it by a sort.
  int32_t *q = nullptr;
  int64_t q_cap = 0;
  int32_t queue_valid = 0;
  // the fused step maintains a dense slot index instead of the hash below;
  // hash_valid = 0 makes the next staged-pipeline entry point rebuild it
  int32_t hash_valid = 1;
};
