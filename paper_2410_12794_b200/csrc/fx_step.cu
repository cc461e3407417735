// Fused per-batch cache step: the whole locality layer of one Ranker batch
// (embserve ranker.py:218-442 with cache.py:189-352) as one stream of device
// kernels with NO host synchronisation, so a batch can be captured in a CUDA
// graph and overlapped with the gather+pool kernel (K4) on another stream.
//
// Domain (checked by the host before it chooses this path): row keys only
// (no pooled-result keyspace), one entry size S for every table, one shard
// per table on this GPU. Order and semantics are the canonical order of
// SURVEY §8(c), bit-exact with the reference's AdaptiveCache:
//
//   1. apply_pending_admissions: staged keys inserted in order, always-admit
//      _insert (cache.py:344-352, 256-268) — one warp;
//   2. ingress validation + per-batch dedup (K2): u64 key table<<40|row,
//      multiplicity, first / last (lookup, feature, position) ordinal. A bad
//      index sets an error word and every later kernel of the batch is a
//      no-op, so a rejected batch leaves the cache untouched
//      (ranker.py:184-193 validates before any probe);
//   3. probe (K3) once per unique key: a key cached at batch start hits on
//      every occurrence, last_tick = tick0 + last ordinal + 1, hits += mult;
//      a missing key bumps the exact sketch by its multiplicity
//      (cache.py:189-202);
//   4. plan + per-bag counters: a bag is one (lookup, feature, server) group;
//      misses >= threshold push down, else they are raw-fetched
//      (pooling.py:88-100; threshold None = every miss raw);
//   5. offers of the raw-fetched misses in first raw-occurrence order
//      (ranker.py:338-340, 417-423; cache.py:237-268);
//   6. stage_hot_admissions(limit) (cache.py:311-342) and sketch age
//      (cache.py:128-136) — fx_step_maintain.
//
// The offers (5) are the order-dependent part. With one entry size, after
// the F free units are used every accept evicts exactly one entry, so the
// eviction queue is V = [entries in LRU order] and accept r evicts V[r - F].
// Candidate j (j >= F) is accepted iff est(c_j) >= est(V[a_j]), a_j = number
// of phase-2 accepts before j. Every candidate was bumped this batch, so
// est(c_j) >= minC >= 1 and a victim with est <= minC accepts whoever comes:
// only "hard" victims (est > minC; ~0.1% of V on cfg3) can reject. One warp
// walks the hard victims: it jumps over the easy stretch between two hard
// victims (each easy victim takes the next candidate), and for a hard victim
// of estimate e finds the next candidate with est >= e (a shared-memory
// table of per-block maxima plus one coalesced 256-candidate probe). The
// rejected intervals it emits fully determine the decisions; ticks, slots,
// evictions, hash updates and row copies are then applied in parallel over
// accept ranks. Batches outside that domain (more accepts than entries, a
// cache above budget) run an exact single-thread loop instead
// (ks_seq_offer), chosen on the device.
//
// The LRU order is kept as an explicit queue (fx_cache.q): each step
// compacts it to [entries not hit this batch, old order] ++ [hit entries by
// last ordinal] — the reference's OrderedDict after the probes — and appends
// the accepts, so no tick sort is needed.

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <climits>
#include <cstring>
#include <string>
#include <vector>

#include "fx_cache.cuh"

namespace fx {
namespace stp {

constexpr int kFine = 256;          // candidates per fine probe of the offer chain
constexpr int kTopkBins = 1 << 16;  // radix-select digit histogram (16-bit digits)

enum { MODE_NONE = 0, MODE_PAR = 1, MODE_SEQ = 2 };

// Device-resident per-step state (all per-batch control lives here so the
// captured graph needs no host input).
struct StepScalars {
  long long err;           // 0 ok, 1 bad index (batch rejected), 2 sketch capacity, 3 invariant
  unsigned long long err_at;  // min over bad occurrences of (sample-major ordinal << 32 | CSR position)
  long long epoch;         // batch counter (slot hit marks)
  long long n_uniq, n_cand, n_hitu, n_nonhit, n_hard, n_rej, n_off;
  long long e0, F, mode, n_acc, n_ev, ftop0, log0;
  long long tick0, tick_base;
  long long minc_bits;     // min candidate estimate (bits of a positive double)
  long long b_hits, b_misses, b_groups;   // this batch
  long long b_applied;     // pending admissions installed at batch start
  long long b_pd_groups, b_pd_rows, b_raw_rows;     // per-batch sums of the per-bag counters
  long long rebuild_index, rehash_sketch, rehash_n;
  long long stage_on, topk_live, topk_krem, topk_n;  // stage(limit) radix select
  unsigned long long topk_hi, topk_lo;               // selected prefix of (vinv, key)
  long long topk_digit;
  long long qlen_new;
  long long n_levels, codes_on;  // distinct hard-victim estimates (<= 255 -> byte codes)
  long long chain_cycles;        // clock64 cycles of the decision chain (diagnostics)
  long long dyn;                 // a candidate was cached at offer time (several batches in flight)
  long long claim_tag, claim_clear;  // dense dedup: this batch's tag; clear the claim words first
  long long dedup_merge;   // (global block) merge a warp's equal keys in the next dedup
  long long stage_thr;     // (global block) bits of a lower bound on the limit-th hottest count, 0 = none
  long long topk_fast;     // this stage selects from the entries at or above stage_thr
};

struct DEnt {       // per dedup-hash slot (one 16-byte line for the atomics); all-zero = empty
  int32_t mult;      // occurrences
  int32_t first;     // INT_MAX - first sample-major ordinal (atomicMax)
  int32_t last;      // last ordinal + 1 (atomicMax)
  int32_t hit;       // cache slot at probe time, -1 = miss
};
__device__ __forceinline__ int32_t d_first(const DEnt &e) { return INT_MAX - e.first; }
__device__ __forceinline__ int32_t d_last(const DEnt &e) { return e.last - 1; }

// Per table row (dense): this batch's dedup claim word and the row's cache
// slot, in one 8-byte record so the dedup claimer reads the slot from the
// sector it just claimed (the probe then needs no slot-index access).
struct __align__(8) DRow {
  unsigned int claim;  // batch tag << rep_bits | first claimer's CSR position
  int32_t slot;        // cache slot or -1
};

struct StepView {
  StepScalars *ss;   // this batch's slot
  StepScalars *gs;   // global (epoch counter)
  // dedup hash
  CkPtr<uint64_t> dkey;
  CkPtr<DEnt> dent;
  CkPtr<int32_t> dfraw;    // first raw-occurrence ordinal (threshold mode)
  int64_t dcap;
  CkPtr<DRow> drow;        // dense per-row claim word + cache slot (one record per table row)
  int32_t rep_bits;  // bits of the claimer position in a claim word
  CkPtr<int32_t> uniq;     // claimed dedup slots
  CkPtr<int32_t> claim;    // [max_nnz] per occurrence: the dedup slot it claimed, else -1
  CkPtr<double> dC;        // [dcap] sketch estimate after this batch's bump (misses)
  CkPtr<int32_t> inv;      // per occurrence (CSR position) -> dedup slot
  CkPtr<uint8_t> umiss;    // [max_nnz] per unique id: 1 = missed the cache (the plan's dense lookup)
  CkPtr<int32_t> cand_by_first;  // [max_nnz] scatter by ordinal
  CkPtr<int32_t> hit_by_last;    // [max_nnz]
  CkPtr<int32_t> cand;     // compacted candidates (dedup slots) in first raw-occurrence order
  CkPtr<uint64_t> ckey;    // [max_nnz] this slot's candidate keys (kept from start to offer)
  CkPtr<double> cest;      // [max_nnz] this slot's candidate estimates at probe time
  CkPtr<double> estv;      // [max_nnz] candidate estimates at offer time
  CkPtr<int32_t> pres;     // [max_nnz] 1 = candidate absent at offer time
  CkPtr<int32_t> cidx;     // [max_nnz] absent candidates (positions into ckey)
  CkPtr<uint64_t> okey;    // [max_nnz] absent candidate keys in offer order
  CkPtr<int32_t> hits_ord; // compacted hit cache slots in last-ordinal order
  CkPtr<double> cC;        // candidate estimates in offer order
  CkPtr<double> bmax;      // per kFine-block max of cC
  CkPtr<int32_t> q;        // the cache's LRU queue (fx_cache.q)
  const int64_t *kbase;  // per table: first dense position
  CkPtr<int32_t> qnew;     // [scap] V = compacted queue
  CkPtr<uint32_t> hitbits; // [scap / 32] slots hit by this batch's probes (cleared per batch;
                           // 0.8 MB for 6.4 M slots: stays in L2 for the queue compaction)
  CkPtr<double> E;         // [scap] victim estimates
  CkPtr<int32_t> hardf;    // [scap] scratch (queue rebuild sort values)
  CkPtr<uint32_t> hardbits;  // [scap / 32] hard-victim flags, one bit per victim position
  CkPtr<int32_t> hard;     // [scap] compacted hard positions
  CkPtr<int32_t> rj_beg; CkPtr<int32_t> rj_end;  // reject intervals
  CkPtr<uint8_t> code;     // [max_nnz] per candidate: number of distinct hard levels <= its estimate
  CkPtr<uint8_t> bsum;     // [max_nnz / 32 + 1] max code per 32 candidates
  CkPtr<uint8_t> hrank;    // [scap] per hard victim: 1 + index of its level (accept iff code >= hrank)
  CkPtr<double> levels;    // [256] distinct hard-victim estimates, ascending
  CkPtr<int32_t> acc;      // [max_nnz] accept flags, then ranks
  CkPtr<int32_t> rank;
  CkPtr<int32_t> aslot;    // [max_nnz] slot taken by accept r
  CkPtr<uint64_t> akey;    // [max_nnz] key of accept r
  CkPtr<int32_t> accj;     // [max_nnz] candidate index of accept r (sequential mode)
  int64_t max_nnz;
  // per-table row source and validation bounds (dense by table id)
  const float *const *tbase;
  const int64_t *tld;
  const int64_t *trows;
  int32_t n_tables;
  int32_t S;         // entry size in bytes
  int32_t dim;       // floats per row
  // rehash / top-k temporaries
  CkPtr<uint64_t> tk_key;
  CkPtr<uint64_t> tk_vinv;
  CkPtr<double> tk_val;
  CkPtr<uint8_t> tk_flag;
  int64_t tk_cap;
  CkPtr<int32_t> tk_hist;
  CkPtr<int32_t> tk_sel;   // selected top-k list positions
};

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ bool aborted(const StepView &v) { return v.ss->err != 0; }

__device__ __forceinline__ long long warp_sum(long long x) {
  for (int o = 16; o; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
  return x;
}

// block-aggregated atomicAdd (every thread of the block calls it): one global
// atomic per block instead of one per warp — same-address atomics serialise
__device__ __forceinline__ void block_add(unsigned long long *ctr, long long x) {
  __shared__ long long red[32];
  x = warp_sum(x);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = x;
  __syncthreads();
  if (w == 0) {
    long long y = lane < static_cast<int>(blockDim.x >> 5) ? red[lane] : 0;
    y = warp_sum(y);
    if (lane == 0 && y) atomicAdd(ctr, static_cast<unsigned long long>(y));
  }
}

// block-aggregated append (every thread calls it): position of this thread's
// item when `want`, one global atomic per block
__device__ __forceinline__ long long block_append(unsigned long long *ctr, int want) {
  __shared__ int wcnt[32];
  __shared__ unsigned long long base;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(0xffffffffu, want);
  __syncthreads();
  if (lane == 0) wcnt[w] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) {
      const int c = wcnt[i];
      wcnt[i] = tot;
      tot += c;
    }
    base = tot ? atomicAdd(ctr, static_cast<unsigned long long>(tot)) : 0ull;
  }
  __syncthreads();
  return static_cast<long long>(base) + wcnt[w] + __popc(m & ((1u << lane) - 1u));
}

// warp-aggregated atomicAdd of a per-lane count; returns this lane's base
__device__ __forceinline__ long long warp_append(unsigned long long *ctr, int want) {
  const unsigned m = __ballot_sync(0xffffffffu, want);
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (m) {
    const int leader = __ffs(m) - 1;
    if (lane == leader) base = atomicAdd(ctr, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
  }
  return (long long)base + __popc(m & ((1u << lane) - 1u));
}

// Dense slot index: HBM is plentiful (4 bytes per table row, 1.28 GB for
// cfg3's 320 M rows, 0.8 % of the tables), so the fast path maps (table, row)
// to its cache slot directly — one 4-byte access instead of a hash probe
// chain, and inserts / evictions are plain stores (no tombstones, no
// rebuilds). The open-addressing hash of fx_cache.cu is rebuilt lazily from
// the slots when a staged-pipeline entry point needs it.
__device__ __forceinline__ int64_t dpos(const StepView &v, uint64_t key) {
  return v.kbase[key >> kRowBitsC] + static_cast<int64_t>(key & kRowMask);
}
__device__ __forceinline__ int32_t d_find(const StepView &v, uint64_t key) { return v.drow[dpos(v, key)].slot; }

__device__ __forceinline__ const float *row_src(const StepView &v, uint64_t key) {
  const int64_t t = static_cast<int64_t>(key >> kRowBitsC);
  const int64_t r = static_cast<int64_t>(key & kRowMask);
  return v.tbase[t] + r * v.tld[t];
}

// copy one row (dim floats) with the calling warp
__device__ __forceinline__ void warp_copy_row(float *dst, const float *src, int dim, int lane) {
  if ((dim & 3) == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    const float4 *s4 = reinterpret_cast<const float4 *>(src);
    float4 *d4 = reinterpret_cast<float4 *>(dst);
    for (int i = lane; i < dim / 4; i += 32) d4[i] = __ldg(&s4[i]);
  } else {
    for (int i = lane; i < dim; i += 32) dst[i] = __ldg(&src[i]);
  }
}

// bump(key, w) for a key probed once per batch (a unique key of the batch):
// no other thread touches this key's entry in the kernel, so a found entry is
// updated with a plain load/store; only a new key claims an empty slot by CAS
// (slots only go empty -> key during the kernel, and an empty slot's value is
// 0, so the new value is 0.0 + w exactly as in the reference's dict).
__device__ __forceinline__ double sketch_add_val(const CacheView &c, uint64_t key, double w, bool *born) {
  const uint64_t m = static_cast<uint64_t>(c.kcap - 1);
  uint64_t h = hash_key(key) & m;
  while (true) {
    uint64_t k = __ldcg(reinterpret_cast<const unsigned long long *>(&c.kkeys[h]));
    if (k == kEmpty) {
      k = atomicCAS(reinterpret_cast<unsigned long long *>(&c.kkeys[h]), (unsigned long long)kEmpty,
                    (unsigned long long)key);
      if (k == kEmpty) {
        const double nv = 0.0 + w;
        c.kval[h] = nv;
        *born = true;
        return nv;
      }
    }
    if (k == key) {
      const double nv = c.kval[h] + w;
      c.kval[h] = nv;
      *born = false;
      return nv;
    }
    h = (h + 1) & m;
  }
}

// ---------------------------------------------------------------- 0. start
__global__ void ks_begin(CacheView c, StepView v, int64_t max_nnz) {
  StepScalars *s = v.ss;
  s->err = 0;
  s->err_at = ~0ull;
  v.gs->epoch += 1;  // global batch counter (slot hit marks)
  s->epoch = v.gs->epoch;
  {  // dense-dedup tag in [1, 2^(32-rep_bits) - 1]; a new cycle clears the claim words
    const long long ntag = (1ll << (32 - v.rep_bits)) - 1;
    s->claim_tag = ((s->epoch - 1) % ntag) + 1;
    s->claim_clear = (s->claim_tag == 1 && s->epoch > 1) ? 1 : 0;
  }
  s->n_uniq = s->n_cand = s->n_hitu = s->n_nonhit = s->n_hard = s->n_rej = s->n_off = 0;
  s->dyn = 0;
  s->n_acc = s->n_ev = 0;
  s->mode = MODE_NONE;
  s->minc_bits = LLONG_MAX;
  s->b_hits = s->b_misses = s->b_groups = 0;
  s->b_applied = 0;
  s->b_pd_groups = s->b_pd_rows = s->b_raw_rows = 0;
  // sketch room for this batch's new keys (bounded by the batch's nnz)
  const Scalars *sc = c.sc;
  const long long live = sc->sketch_live, tomb = sc->sketch_tomb;
  s->rehash_sketch = ((live + tomb + max_nnz) * 10 > c.kcap * 7) ? 1 : 0;
  s->rehash_n = 0;
  if ((live + max_nnz) * 10 > c.kcap * 7) s->err = 2;  // sketch_capacity too small for this batch
}

__global__ void ks_claim_clear(StepView v, int64_t n_dense) {
  if (!v.ss->claim_clear) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_dense; i += (int64_t)gridDim.x * blockDim.x)
    v.drow[i].claim = 0u;
}

// in-place sketch rehash (drops tombstones): collect -> clear -> reinsert
__global__ void ks_sketch_collect(CacheView c, StepView v) {
  if (!v.ss->rehash_sketch) return;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < c.kcap; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const uint64_t k = i < c.kcap ? c.kkeys[i] : kEmpty;
    const bool live = k != kEmpty && k != kTomb;
    const long long p = block_append(reinterpret_cast<unsigned long long *>(&v.ss->rehash_n), live);
    if (live) {
      v.tk_key[p] = k;
      v.tk_val[p] = c.kval[i];
      v.tk_flag[p] = c.kflag[i];
    }
  }
}

__global__ void ks_sketch_clear(CacheView c, StepView v) {
  if (!v.ss->rehash_sketch) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.kcap; i += (int64_t)gridDim.x * blockDim.x) {
    c.kkeys[i] = kEmpty;
    c.kval[i] = 0.0;
    c.kflag[i] = 0;
  }
}

__global__ void ks_sketch_reinsert(CacheView c, StepView v) {
  if (!v.ss->rehash_sketch) return;
  const long long n = v.ss->rehash_n;
  const uint64_t m = static_cast<uint64_t>(c.kcap - 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = v.tk_key[i];
    uint64_t h = hash_key(k) & m;
    while (atomicCAS(reinterpret_cast<unsigned long long *>(&c.kkeys[h]), (unsigned long long)kEmpty,
                     (unsigned long long)k) != kEmpty)
      h = (h + 1) & m;
    c.kval[h] = v.tk_val[i];
    c.kflag[h] = v.tk_flag[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) c.sc->sketch_tomb = 0;
}

// a key claimed by this batch's dedup has its probe-time slot in its entry:
// apply_pending (which runs between dedup and probe) keeps it current
__device__ __forceinline__ void patch_hit(const StepView &v, uint64_t key, int32_t slot) {
  const unsigned int w = v.drow[dpos(v, key)].claim;
  if ((w >> v.rep_bits) == static_cast<unsigned int>(v.ss->claim_tag))
    v.dent[w & ((1u << v.rep_bits) - 1u)].hit = slot;
}

// ---------------------------------------------------------------- 1. apply pending
// cache.py:344-352: install the keys staged by the last maintenance, in
// order, always-admit (_insert evicts the LRU head until the entry fits).
// One warp: lane 0 decides, the warp copies each installed row.
__global__ void ks_apply_pending(CacheView c, StepView v) {
  const int lane = threadIdx.x & 31;
  if (blockIdx.x != 0 || threadIdx.x >= 32 || aborted(v)) return;
  Scalars *sc = c.sc;
  const long long n = sc->pending;
  if (n <= 0) return;
  const long long S = v.S;
  long long e = sc->entries, head = 0, ftop = sc->free_top, tick = sc->tick, nlog = sc->n_evlog;
  long long applied = 0;
  long long qlen = e;
  for (long long i = 0; i < n; ++i) {
    const uint64_t key = c.pend[i];
    int32_t slot = -1;
    if (lane == 0) {
      const int64_t kp = k_find(c, key);
      if (kp >= 0) c.kflag[kp] = 0;
      const bool present = d_find(v, key) >= 0;
      if (!present && S <= sc->budget) {
        while ((e + 1) * S > sc->budget && e > 0) {  // evict the LRU head
          const int32_t vs = v.q[head];
          v.q[head] = -1;
          ++head;
          const uint64_t ok = c.skey[vs];
          if (c.evlog_cap > 0 && nlog < c.evlog_cap) c.evlog[nlog] = ok;
          if (c.evlog_cap > 0) ++nlog;
          v.drow[dpos(v, ok)].slot = -1;
          patch_hit(v, ok, -1);
          c.stick[vs] = kFree;
          c.skey[vs] = kEmpty;
          c.free_stack[ftop++] = vs;
          --e;
        }
        slot = c.free_stack[--ftop];
        ++tick;
        c.skey[slot] = key;
        c.skey2[slot] = 0;
        c.stick[slot] = tick;
        c.ssize[slot] = static_cast<int32_t>(S);
        c.shits[slot] = 0;
        v.drow[dpos(v, key)].slot = slot;
        patch_hit(v, key, slot);
        v.q[qlen++] = slot;
        ++e;
        ++applied;
      }
    }
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if (slot >= 0) warp_copy_row(c.rows + static_cast<int64_t>(slot) * c.row_ld, row_src(v, key), v.dim, lane);
  }
  if (lane == 0) {
    sc->entries = e;
    sc->used = e * S;
    sc->free_top = ftop;
    sc->tick = tick;
    sc->n_evlog = nlog;
    sc->pending = 0;
    v.ss->b_applied = applied;
  }
}

// ---------------------------------------------------------------- 2. validate + dedup
// A block takes 256 consecutive bags (32 per warp; a warp's lanes walk its
// bags' occurrences 32 at a time, each lane locating its bag with a shuffle
// search over the warp's 33 bag offsets). Occurrences are first merged per
// block in a shared-memory table (key -> multiplicity, first / last ordinal,
// first CSR position), so a hot key costs one global claim and three global
// atomics per block instead of per occurrence (Zipf: the hottest row of a
// cfg3 table occurs ~5,000 times per batch). The global step then claims the
// key's dense claim word — (batch tag << rep_bits) | the CSR position of its
// first claimer, which becomes the key's unique id (per-unique data lives in
// nnz-sized arrays) — and folds the block's counts in.
constexpr int kDBags = 256;     // bags per block chunk (8 warps x 32)
constexpr int kDHash = 4096;    // shared-memory table entries per block
constexpr size_t kDSmem = kDHash * (8 + 4 * 5);

// Claim a row's record for this batch with one 64-bit CAS over (claim, slot):
// the claimer learns the row's cache slot from the same access. Returns the
// key's unique id (the first claimer's CSR position); *slot_out is set when
// this call claimed.
__device__ __forceinline__ int32_t claim_row(const StepView &v, int64_t pos, unsigned int tag, unsigned int rmask,
                                             int32_t rep, bool *claimed, int32_t *slot_out) {
  unsigned long long *cw = reinterpret_cast<unsigned long long *>(&v.drow[pos]);
  const unsigned long long mine = (tag << v.rep_bits) | static_cast<unsigned int>(rep);
  unsigned long long w = *cw;
  while (true) {
    const unsigned int cl = static_cast<unsigned int>(w);
    if ((cl >> v.rep_bits) == tag) {
      *claimed = false;
      return static_cast<int32_t>(cl & rmask);
    }
    const unsigned long long prev = atomicCAS(cw, w, (w & 0xffffffff00000000ull) | mine);
    if (prev == w) {
      *claimed = true;
      *slot_out = static_cast<int32_t>(w >> 32);
      return rep;
    }
    w = prev;
  }
}

__device__ __forceinline__ int32_t dedup_global(const StepView &v, uint64_t key, int t, int64_t r, int rep,
                                                unsigned int tag, unsigned int rmask, bool *claimed) {
  int32_t slot = -1;
  const int32_t u = claim_row(v, v.kbase[t] + r, tag, rmask, rep, claimed, &slot);
  if (*claimed) v.dent[rep].hit = slot;  // the key's cache slot at dedup time
  return u;
}

template <typename IdxT>
__global__ void __launch_bounds__(256) ks_dedup(StepView v, const int32_t *__restrict__ bag_table,
                                                const IdxT *__restrict__ idx, const int64_t *__restrict__ offsets,
                                                const int64_t *__restrict__ sm_start, int64_t n_bags) {
  extern __shared__ __align__(16) unsigned char dsm[];
  unsigned long long *hkey = reinterpret_cast<unsigned long long *>(dsm);
  int *hmult = reinterpret_cast<int *>(hkey + kDHash);
  int *hfirst = hmult + kDHash;
  int *hlast = hfirst + kDHash;
  int *hrep = hlast + kDHash;
  int *hu = hrep + kDHash;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const unsigned int tag = static_cast<unsigned int>(v.ss->claim_tag);
  const unsigned int rmask = (1u << v.rep_bits) - 1u;
  for (int i = threadIdx.x; i < kDHash; i += blockDim.x) {
    hkey[i] = kEmpty;
    hmult[i] = 0;
    hfirst[i] = INT_MAX;
    hlast[i] = -1;
    hrep[i] = INT_MAX;
  }
  __syncthreads();
  for (int64_t c0 = blockIdx.x * (int64_t)kDBags; c0 < n_bags; c0 += (int64_t)gridDim.x * kDBags) {
    // ---- phase 1: occurrences -> block table
    const int64_t b0 = c0 + wib * 32;
    if (b0 < n_bags) {
      const int64_t nb = n_bags - b0 < 32 ? n_bags - b0 : 32;
      const int64_t my = b0 + (lane < nb ? lane : nb - 1);
      const int64_t off = lane < nb ? __ldg(&offsets[b0 + lane]) : __ldg(&offsets[b0 + nb]);
      const int64_t end = __ldg(&offsets[b0 + nb]);
      const int32_t tab = __ldg(&bag_table[my]);
      const int64_t sms = __ldg(&sm_start[my]);
      const int64_t start = __shfl_sync(0xffffffffu, off, 0);
      for (int64_t p0 = start; p0 < end; p0 += 32) {
        const int64_t p = p0 + lane;
        int lo = 0, hi = static_cast<int>(nb);  // bag j: last lane with off_j <= p
#pragma unroll
        for (int it = 0; it < 6; ++it) {
          const int mid = (lo + hi) >> 1;
          const int64_t om = __shfl_sync(0xffffffffu, off, mid & 31);
          if (hi - lo > 1) {
            if (om <= p) lo = mid; else hi = mid;
          }
        }
        const int j = lo;
        const int64_t bo = __shfl_sync(0xffffffffu, off, j);
        const int32_t t = __shfl_sync(0xffffffffu, tab, j);
        const int64_t sm = __shfl_sync(0xffffffffu, sms, j);
        if (p >= end) continue;
        v.claim[p] = -1;
        const int64_t r = static_cast<int64_t>(idx[p]);
        const int ord = static_cast<int>(sm + (p - bo));
        if (t < 0 || t >= v.n_tables || r < 0 || r >= v.trows[t]) {
          atomicMin(reinterpret_cast<unsigned long long *>(&v.ss->err_at),
                    (static_cast<unsigned long long>(ord) << 32) | static_cast<unsigned long long>(p & 0xffffffff));
          v.ss->err = 1;
          v.inv[p] = -1;
          continue;
        }
        const uint64_t key = (static_cast<uint64_t>(t) << kRowBitsC) | static_cast<uint64_t>(r);
        int h = static_cast<int>(hash_key(key) & (kDHash - 1)), probe = 0;
        for (; probe < 64; ++probe) {
          const unsigned long long prev = atomicCAS(&hkey[h], (unsigned long long)kEmpty, (unsigned long long)key);
          if (prev == kEmpty || prev == key) break;
          h = (h + 1) & (kDHash - 1);
        }
        if (probe < 64) {
          atomicAdd(&hmult[h], 1);
          atomicMin(&hfirst[h], ord);
          atomicMax(&hlast[h], ord);
          atomicMin(&hrep[h], static_cast<int>(p));
          v.inv[p] = -2 - h;  // resolved in phase 3
        } else {              // block table crowded: straight to the global path
          bool claimed = false;
          const int32_t u = dedup_global(v, key, t, r, static_cast<int>(p), tag, rmask, &claimed);
          if (claimed) {
            v.dkey[u] = key;
            v.claim[p] = u;
          }
          DEnt *e = &v.dent[u];
          atomicAdd(&e->mult, 1);
          atomicMax(&e->first, INT_MAX - ord);  // zero-initialised encodings (memset reset)
          atomicMax(&e->last, ord + 1);
          v.inv[p] = u;
        }
      }
    }
    __syncthreads();
    // ---- phase 2: one global claim + fold per distinct key of the chunk
    for (int i = threadIdx.x; i < kDHash; i += blockDim.x) {
      const uint64_t key = hkey[i];
      if (key == kEmpty) continue;
      const int t = static_cast<int>(key >> kRowBitsC);
      const int64_t r = static_cast<int64_t>(key & kRowMask);
      bool claimed = false;
      const int32_t u = dedup_global(v, key, t, r, hrep[i], tag, rmask, &claimed);
      if (claimed) {
        v.dkey[u] = key;
        v.claim[u] = u;
      }
      DEnt *e = &v.dent[u];
      atomicAdd(&e->mult, hmult[i]);
      atomicMax(&e->first, INT_MAX - hfirst[i]);
      atomicMax(&e->last, hlast[i] + 1);
      hu[i] = u;
    }
    __syncthreads();
    // ---- phase 3: occurrences learn their unique id; the table is reset
    const int64_t pe = __ldg(&offsets[c0 + kDBags < n_bags ? c0 + kDBags : n_bags]);
    for (int64_t p = __ldg(&offsets[c0]) + threadIdx.x; p < pe; p += blockDim.x) {
      const int32_t w = v.inv[p];
      if (w <= -2) v.inv[p] = hu[-2 - w];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kDHash; i += blockDim.x) {
      if (hkey[i] == kEmpty) continue;
      hkey[i] = kEmpty;
      hmult[i] = 0;
      hfirst[i] = INT_MAX;
      hlast[i] = -1;
      hrep[i] = INT_MAX;
    }
    __syncthreads();
  }
}

// Default dedup (ks_dedup_occ): one lane per occurrence does the dense claim
// and the entry atomics; on skewed batches lanes of a warp holding the same
// key merge first. ncu, cfg3 2 %, alpha 0.6 / 1.0 / 1.2: per-occurrence
// 135 / 132 / 208 us, warp-merged 183 / 162 / 125 us, block-merge variant
// above (FX_DEDUP=blk) 375 / 223 / 127 us — hence the switch on the previous
// batch's unique fraction (0.97 / 0.48 / 0.17 at those alphas).
// A warp takes `bw` (<= 32) consecutive bags; its lanes walk the bags'
// occurrences 32 at a time, each lane locating its bag with a shuffle search
// over the bw + 1 bag offsets the warp holds. Each round of 32 occurrences is
// a chain of dependent random accesses (claim word in HBM, entry atomics), so
// fewer bags per warp = more warps in flight.
template <typename IdxT>
__global__ void __launch_bounds__(256) ks_dedup_occ(StepView v, const int32_t *__restrict__ bag_table,
                                                const IdxT *__restrict__ idx, const int64_t *__restrict__ offsets,
                                                const int64_t *__restrict__ sm_start, int64_t n_bags, int bw) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned int tag = static_cast<unsigned int>(v.ss->claim_tag);
  const unsigned int rmask = (1u << v.rep_bits) - 1u;
  const bool merge = v.gs->dedup_merge != 0;
  for (int64_t b0 = warp * bw; b0 < n_bags; b0 += nw * bw) {
    const int64_t nb = n_bags - b0 < bw ? n_bags - b0 : bw;
    const int64_t my = b0 + (lane < nb ? lane : nb - 1);
    const int64_t off = lane < nb ? __ldg(&offsets[b0 + lane]) : __ldg(&offsets[b0 + nb]);
    const int64_t end = __ldg(&offsets[b0 + nb]);
    const int32_t tab = __ldg(&bag_table[my]);
    const int64_t sms = __ldg(&sm_start[my]);
    const int64_t start = __shfl_sync(0xffffffffu, off, 0);
    for (int64_t p0 = start; p0 < end; p0 += 32) {
      const int64_t p = p0 + lane;
      // bag j: last lane with off_j <= p
      int lo = 0, hi = static_cast<int>(nb);
#pragma unroll
      for (int it = 0; it < 6; ++it) {
        const int mid = (lo + hi) >> 1;
        const int64_t om = __shfl_sync(0xffffffffu, off, mid & 31);
        if (hi - lo > 1) {
          if (om <= p) lo = mid; else hi = mid;
        }
      }
      const int j = lo;
      const int64_t bo = __shfl_sync(0xffffffffu, off, j);
      const int32_t t = __shfl_sync(0xffffffffu, tab, j);
      const int64_t sm = __shfl_sync(0xffffffffu, sms, j);
      const bool act = p < end;
      bool claimed = false;
      int32_t u = -1;
      int ord = 0;
      uint64_t key = ~0ull - 2;  // lanes without a valid occurrence get a key no occurrence has
      int64_t r = 0;
      if (act) {
        r = static_cast<int64_t>(idx[p]);
        ord = static_cast<int>(sm + (p - bo));
        const bool okt = t >= 0 && t < v.n_tables;
        if (!okt || r < 0 || r >= v.trows[t]) {
          atomicMin(reinterpret_cast<unsigned long long *>(&v.ss->err_at),
                    (static_cast<unsigned long long>(ord) << 32) | static_cast<unsigned long long>(p & 0xffffffff));
          v.ss->err = 1;
        } else {
          key = (static_cast<uint64_t>(t) << kRowBitsC) | static_cast<uint64_t>(r);
        }
      }
      // skewed batches (unique fraction < 0.35 in the previous batch): lanes
      // of the warp holding the same key merge first, then the group's lowest
      // lane — also its first CSR position — does the global work; otherwise
      // every lane is its own group (the warp match costs more than it saves)
      unsigned peers = 1u << lane;
      int gmin = ord, gmax = ord;
      if (merge) {
        peers = __match_any_sync(0xffffffffu, key);
        gmin = __reduce_min_sync(peers, static_cast<unsigned>(ord));
        gmax = __reduce_max_sync(peers, static_cast<unsigned>(ord));
      }
      const int leader = __ffs(peers) - 1;
      const bool valid = key < (~0ull - 2);
      if (valid && lane == leader) {
        int32_t slot = -1;
        u = claim_row(v, v.kbase[t] + r, tag, rmask, static_cast<int32_t>(p), &claimed, &slot);
        if (claimed) {
          v.dkey[u] = key;
          v.dent[u].hit = slot;  // the key's cache slot at dedup time
        }
        DEnt *e = &v.dent[u];
        atomicAdd(&e->mult, __popc(peers));
        atomicMax(&e->first, INT_MAX - gmin);  // zero-initialised encodings (memset reset)
        atomicMax(&e->last, gmax + 1);
      }
      u = __shfl_sync(peers, u, leader);
      if (act) {
        if (valid) v.inv[p] = u;
        v.claim[p] = claimed ? u : -1;
      }
    }
  }
}

// ---------------------------------------------------------------- 3. probe
// One thread per CSR position: the claimer of a key (claim[p] == p, the
// key's unique id) probes it, so no compaction of the claim words is needed;
// the unique count is block-aggregated here. Two positions per thread and
// iteration, their loads issued together (the probe is a chain of dependent
// random accesses: claim word -> entry -> dense slot index -> sketch).
template <int KP>
__global__ void __launch_bounds__(256) ks_probe(CacheView c, StepView v, int32_t threshold_on, int64_t nnz) {
  if (aborted(v)) return;
  const long long tick0 = c.sc->tick;
  long long hits = 0, misses = 0, born = 0, nu = 0;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < nnz; i0 += KP * T) {
    int32_t u[KP];
#pragma unroll
    for (int k = 0; k < KP; ++k) u[k] = i0 + k * T < nnz ? v.claim[i0 + k * T] : -1;
    uint64_t key[KP];
    DEnt e[KP];
#pragma unroll
    for (int k = 0; k < KP; ++k)
      if (u[k] >= 0) {
        key[k] = v.dkey[u[k]];
        e[k] = v.dent[u[k]];
      }
    int32_t sl[KP];  // the slot dedup recorded (kept current by apply_pending)
#pragma unroll
    for (int k = 0; k < KP; ++k) sl[k] = u[k] >= 0 ? e[k].hit : -1;
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      if (u[k] < 0) continue;
      ++nu;
      const int32_t s = sl[k];
      v.umiss[u[k]] = s < 0 ? 1 : 0;
      if (s >= 0) {
        c.stick[s] = tick0 + d_last(e[k]) + 1;
        c.shits[s] += e[k].mult;
        atomicOr(&v.hitbits[s >> 5], 1u << (s & 31));
        v.hit_by_last[d_last(e[k])] = s;
        hits += e[k].mult;
      } else {
        bool b = false;
        v.dC[u[k]] = sketch_add_val(c, key[k], static_cast<double>(e[k].mult), &b);
        born += b ? 1 : 0;
        misses += e[k].mult;
        if (!threshold_on) v.cand_by_first[d_first(e[k])] = u[k];
      }
    }
  }
  block_add(reinterpret_cast<unsigned long long *>(&c.sc->hits), hits);
  block_add(reinterpret_cast<unsigned long long *>(&c.sc->misses), misses);
  block_add(reinterpret_cast<unsigned long long *>(&c.sc->sketch_live), born);
  block_add(reinterpret_cast<unsigned long long *>(&v.ss->b_hits), hits);
  block_add(reinterpret_cast<unsigned long long *>(&v.ss->b_misses), misses);
  block_add(reinterpret_cast<unsigned long long *>(&v.ss->n_uniq), nu);
}

__global__ void ks_after_probe(CacheView c, StepView v, int64_t nnz) {
  if (aborted(v)) return;
  v.ss->tick0 = c.sc->tick;
  c.sc->tick += nnz;  // one tick per probed occurrence (cache.py:193)
  // few distinct keys -> hot keys repeat inside a warp's 32 occurrences and
  // their same-address atomics serialise: the next dedup merges them first
  v.gs->dedup_merge = (v.ss->n_uniq * 20 < nnz * 7) ? 1 : 0;
}

// ---------------------------------------------------------------- 4. plan + counters
// warp per bag: misses m; threshold t > 0 and m >= t -> one pushdown group,
// else the misses are raw rows (and raw occurrences feed the offers)
__global__ void __launch_bounds__(256) ks_bag_plan(StepView v, const int64_t *__restrict__ offsets,
                                                   const int64_t *__restrict__ sm_start, int64_t n_bags,
                                                   int32_t threshold, int32_t *hits_bag, int32_t *pd_groups,
                                                   int32_t *pd_rows, int32_t *raw_rows) {
  if (aborted(v)) return;  // uniform: the whole grid returns
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  long long groups = 0, pdg = 0, pdr = 0, raw = 0;
  for (int64_t b = warp; b < n_bags; b += nw) {
    const int64_t beg = __ldg(&offsets[b]), end = __ldg(&offsets[b + 1]);
    int m = 0;
    for (int64_t p = beg + lane; p < end; p += 32) m += v.umiss[v.inv[p]];
    for (int o = 16; o; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
    const int L = static_cast<int>(end - beg);
    const bool push = threshold > 0 && m >= threshold;
    if (lane == 0) {
      if (hits_bag) hits_bag[b] = L - m;
      if (pd_groups) pd_groups[b] = (push && m > 0) ? 1 : 0;
      if (pd_rows) pd_rows[b] = push ? m : 0;
      if (raw_rows) raw_rows[b] = push ? 0 : m;
      groups += m > 0 ? 1 : 0;
      pdg += (push && m > 0) ? 1 : 0;
      pdr += push ? m : 0;
      raw += push ? 0 : m;
    }
    if (threshold > 0 && !push && m > 0) {
      const int64_t sm = __ldg(&sm_start[b]);
      for (int64_t p = beg + lane; p < end; p += 32) {
        const int32_t u = v.inv[p];
        if (v.umiss[u]) atomicMax(&v.dfraw[u], INT_MAX - static_cast<int32_t>(sm + (p - beg)));
      }
    }
  }
  block_add(reinterpret_cast<unsigned long long *>(&v.ss->b_groups), groups);
  block_add(reinterpret_cast<unsigned long long *>(&v.ss->b_pd_groups), pdg);
  block_add(reinterpret_cast<unsigned long long *>(&v.ss->b_pd_rows), pdr);
  block_add(reinterpret_cast<unsigned long long *>(&v.ss->b_raw_rows), raw);
}

__global__ void ks_cand_scatter_raw(StepView v, int64_t nnz) {
  if (aborted(v)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = v.claim[i];
    if (u < 0) continue;
    const int32_t f = v.dfraw[u];
    if (f != 0) v.cand_by_first[INT_MAX - f] = u;
  }
}

// ---------------------------------------------------------------- 5. offers
struct NonNeg {
  __host__ __device__ __forceinline__ bool operator()(const int32_t &x) const { return x >= 0; }
};

struct QueueKeep {
  const uint32_t *hitbits;
  __device__ __forceinline__ bool operator()(const int32_t &s) const {
    return s >= 0 && ((__ldg(&hitbits[s >> 5]) >> (s & 31)) & 1u) == 0;
  }
};

__global__ void ks_cand_keys(StepView v) {
  if (aborted(v)) return;
  const long long n = v.ss->n_cand;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = v.cand[j];
    v.ckey[j] = v.dkey[u];
    v.cest[j] = v.dC[u];  // the sketch value right after this batch's bump
  }
}

// offer time: a candidate installed since the probes (apply_pending of a
// later batch when several are in flight) is present -> offer() returns True
// with no side effect (cache.py:245-246); the rest keep their order
// `fresh`: no other batch ran between this batch's probes and its offers
// (pipeline_depth 1), so every candidate is still absent and its estimate is
// the probe-time value
__global__ void ks_offer_prep(CacheView c, StepView v, int64_t max_nnz, int32_t fresh) {
  const bool on = !aborted(v);
  const long long n = on ? v.ss->n_cand : 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < max_nnz; j += (int64_t)gridDim.x * blockDim.x) {
    int32_t f = 0;
    if (j < n) {
      const uint64_t key = v.ckey[j];
      if (fresh) {
        f = 1;
        v.estv[j] = v.cest[j];
      } else {
        f = d_find(v, key) < 0 ? 1 : 0;
        v.estv[j] = k_est(c, key);
        if (!f) v.ss->dyn = 1;
      }
    }
    if (!fresh) v.pres[j] = f;
  }
}

// `fresh` offers (one batch in flight): every candidate is still absent, so
// the offer list is the candidate list itself (no flag compaction)
__global__ void ks_cidx_identity(StepView v) {
  const long long n = aborted(v) ? 0 : v.ss->n_cand;
  if (blockIdx.x == 0 && threadIdx.x == 0) v.ss->n_off = n;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    v.cidx[j] = static_cast<int32_t>(j);
}

// a candidate cached at offer time can be evicted by an earlier offer of the
// same call and then be offered for real: such calls keep every candidate
// and take the sequential path, which checks presence as it goes
__global__ void ks_offer_flags(StepView v, int64_t max_nnz) {
  if (aborted(v) || !v.ss->dyn) return;
  const long long n = v.ss->n_cand;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < max_nnz; j += (int64_t)gridDim.x * blockDim.x)
    v.pres[j] = j < n ? 1 : 0;
}

// candidate estimates in offer order, their minimum and per-block maxima
__global__ void __launch_bounds__(kFine) ks_cand_est(StepView v) {
  if (aborted(v)) return;
  const long long n = v.ss->n_off;
  __shared__ double red[kFine / 32];
  for (int64_t b = blockIdx.x; b * kFine < n; b += gridDim.x) {
    const int64_t j = b * kFine + threadIdx.x;
    double x = 0.0, mn = 1e300;
    if (j < n) {
      const int32_t i = v.cidx[j];
      x = v.estv[i];
      v.cC[j] = x;
      v.okey[j] = v.ckey[i];
      mn = x;
    }
    double mx = x;
    for (int o = 16; o; o >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if ((threadIdx.x & 31) == 0 && mn < 1e300)
      atomicMin(reinterpret_cast<long long *>(&v.ss->minc_bits), __double_as_longlong(mn));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m2 = red[0];
      for (int w = 1; w < kFine / 32; ++w) m2 = fmax(m2, red[w]);
      v.bmax[b] = m2;
    }
    __syncthreads();
  }
}

__global__ void ks_queue_append_hits(StepView v) {
  if (aborted(v)) return;
  const long long nh = v.ss->n_hitu, base = v.ss->n_nonhit;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nh; i += (int64_t)gridDim.x * blockDim.x)
    v.qnew[base + i] = v.hits_ord[i];
}

// decisions' domain: F free units, parallel (accepts <= entries) or sequential
__global__ void ks_offer_plan(CacheView c, StepView v) {
  if (aborted(v)) return;
  StepScalars *s = v.ss;
  const Scalars *sc = c.sc;
  const long long e0 = sc->entries;  // q[0, e0) = the entries in LRU order
  s->e0 = e0;
  const long long n = s->n_off, S = v.S, budget = sc->budget;
  s->ftop0 = sc->free_top;
  s->log0 = sc->n_evlog;
  s->tick_base = sc->tick;  // each insert takes the next tick (cache.py:262)
  if (n == 0) { s->mode = MODE_NONE; return; }
  if (S > budget) { s->mode = MODE_NONE; s->F = 0; return; }  // size > budget: every offer -> False
  const long long cap = budget / S;
  const long long F = cap > e0 ? (cap - e0 < n ? cap - e0 : n) : 0;
  s->F = F;
  s->mode = (e0 <= cap && n - F <= e0 && !s->dyn) ? MODE_PAR : MODE_SEQ;
}

// victim estimates for V[0, n - F) and hard flags (est > minC)
__global__ void ks_victim_est(CacheView c, StepView v, int64_t scap) {
  if (aborted(v)) return;
  const StepScalars *s = v.ss;
  const bool on = s->mode == MODE_PAR && c.admission == 0;
  const long long need = on ? s->n_off - s->F : 0;
  const double minc = __longlong_as_double(s->minc_bits);
  // a warp covers 32 consecutive positions (the grid is a multiple of 32
  // threads): one ballot word per warp and iteration
  const int lane = threadIdx.x & 31;
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h - lane < scap;
       h += (int64_t)gridDim.x * blockDim.x) {
    bool f = false;
    if (h < need) {
      const double e = k_est(c, c.skey[v.q[h]]);
      v.E[h] = e;
      f = e > minc;
    }
    const unsigned b = __ballot_sync(0xffffffffu, f);
    if (lane == 0) v.hardbits[(h - lane) >> 5] = b;
  }
}

// selection predicate over victim positions: the hard-victim bit
struct HardBit {
  const uint32_t *bits;
  __device__ __forceinline__ bool operator()(const int32_t &h) const {
    return ((__ldg(&bits[h >> 5]) >> (h & 31)) & 1u) != 0;
  }
};

// first j in [x, n) with cC[j] >= e (n if none); whole warp, uniform result
__device__ __forceinline__ long long next_ge(const StepView &v, const double *sbm, long long nblk, long long n,
                                             long long x, double e, int lane) {
  // fine probe of [x, x + kFine): 8 coalesced loads per lane, issued first
  double f[kFine / 32];
#pragma unroll
  for (int i = 0; i < kFine / 32; ++i) {
    const long long j = x + i * 32 + lane;
    f[i] = j < n ? v.cC[j] : -1.0;
  }
  // meanwhile: first block at or after blk(x + kFine) whose max reaches e
  long long B = nblk;
  for (long long b0 = (x + kFine) / kFine; b0 < nblk; b0 += 32) {
    const long long b = b0 + lane;
    const unsigned m = __ballot_sync(0xffffffffu, b < nblk && sbm[b] >= e);
    if (m) { B = b0 + __ffs(m) - 1; break; }
  }
#pragma unroll
  for (int i = 0; i < kFine / 32; ++i) {
    const unsigned m = __ballot_sync(0xffffffffu, f[i] >= e);
    if (m) return x + i * 32 + __ffs(m) - 1;
  }
  if (B >= nblk) return n;
  const long long lo = B * kFine > x + kFine ? B * kFine : x + kFine;
#pragma unroll
  for (int i = 0; i < kFine / 32; ++i) {
    const long long j = lo + i * 32 + lane;
    f[i] = (j < n && j < (B + 1) * kFine) ? v.cC[j] : -1.0;
  }
#pragma unroll
  for (int i = 0; i < kFine / 32; ++i) {
    const unsigned m = __ballot_sync(0xffffffffu, f[i] >= e);
    if (m) return lo + i * 32 + __ffs(m) - 1;
  }
  return n;  // not reached: bmax[B] >= e
}

// The decision chain over hard victims (one block; warp 0 walks, the block
// first stages the per-block maxima in shared memory).
__global__ void __launch_bounds__(1024) ks_chain(StepView v) {
  extern __shared__ double sbm[];
  if (aborted(v) || v.ss->mode != MODE_PAR || v.ss->codes_on) return;
  const long long n = v.ss->n_off, F = v.ss->F, nh = v.ss->n_hard;
  const long long nblk = (n + kFine - 1) / kFine;
  for (long long b = threadIdx.x; b < nblk; b += blockDim.x) sbm[b] = v.bmax[b];
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  long long x = F, h = 0, nrej = 0;
  for (long long k0 = 0; k0 < nh; k0 += 32) {
    const long long kk = k0 + lane;
    const int32_t hp = kk < nh ? v.hard[kk] : 0;
    const double he = kk < nh ? v.E[hp] : 0.0;
    const int cnt = nh - k0 < 32 ? static_cast<int>(nh - k0) : 32;
    bool stop = false;
    for (int t = 0; t < cnt; ++t) {
      const long long b = __shfl_sync(0xffffffffu, hp, t);
      const double e = __shfl_sync(0xffffffffu, he, t);
      const long long gap = b - h;
      if (x + gap >= n) { x = n; stop = true; break; }  // candidates run out in an easy stretch
      x += gap;
      h = b;
      const long long j = next_ge(v, sbm, nblk, n, x, e, lane);
      if (j > x) {
        if (lane == 0) {
          v.rj_beg[nrej] = static_cast<int32_t>(x);
          v.rj_end[nrej] = static_cast<int32_t>(j);
        }
        ++nrej;
      }
      if (j >= n) { x = n; stop = true; break; }
      x = j + 1;
      h = b + 1;
    }
    if (stop) break;
  }
  if (lane == 0) v.ss->n_rej = nrej;
}

// Distinct hard-victim estimates (sorted) and each hard victim's rank; one
// block. More than 255 distinct levels -> codes off (f64 chain instead).
__global__ void __launch_bounds__(1024) ks_levels(StepView v, int32_t stream_ok) {
  __shared__ unsigned long long set[4096];
  __shared__ double lv[256];
  __shared__ int nset, overflow;
  if (aborted(v) || v.ss->mode != MODE_PAR) return;
  const long long nh = v.ss->n_hard;
  if (threadIdx.x == 0) {
    nset = 0;
    overflow = 0;
    v.ss->codes_on = 0;
    v.ss->n_levels = 0;
  }
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) set[i] = 0ull;
  __syncthreads();
  if (nh == 0) return;
  for (long long k = threadIdx.x; k < nh && !overflow; k += blockDim.x) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v.E[v.hard[k]]));
    unsigned h = static_cast<unsigned>(hash_key(b)) & 4095u;
    for (int probe = 0; probe < 4096; ++probe) {
      const unsigned long long prev = atomicCAS(&set[h], 0ull, b);
      if (prev == 0ull) {
        if (atomicAdd(&nset, 1) >= 255) overflow = 1;
        break;
      }
      if (prev == b) break;
      h = (h + 1) & 4095u;
    }
  }
  __syncthreads();
  if (overflow) return;
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < 4096; i += blockDim.x)
    if (set[i]) lv[atomicAdd(&cnt, 1)] = __longlong_as_double(static_cast<long long>(set[i]));
  __syncthreads();
  const int K = cnt;
  if (threadIdx.x < K) {  // rank by counting (distinct values)
    const double x = lv[threadIdx.x];
    int r = 0;
    for (int j = 0; j < K; ++j) r += lv[j] < x ? 1 : 0;
    v.levels[r] = x;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < K; i += blockDim.x) lv[i] = v.levels[i];
  __syncthreads();
  for (long long k = threadIdx.x; k < nh; k += blockDim.x) {
    const double e = v.E[v.hard[k]];
    int lo = 0, hi = K;  // first index with lv >= e (== e: e is a level)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (lv[mid] < e) lo = mid + 1; else hi = mid;
    }
    v.hrank[k] = static_cast<uint8_t>(lo + 1);
  }
  if (threadIdx.x == 0) {
    v.ss->n_levels = K;
    v.ss->codes_on = stream_ok ? 2 : 1;
  }
}

// code per candidate (number of levels <= its estimate) and per-32 maxima
__global__ void __launch_bounds__(256) ks_cand_codes(StepView v) {
  __shared__ double lv[256];
  if (aborted(v) || v.ss->mode != MODE_PAR || !v.ss->codes_on) return;
  const int K = static_cast<int>(v.ss->n_levels);
  for (int i = threadIdx.x; i < K; i += blockDim.x) lv[i] = v.levels[i];
  __syncthreads();
  const long long n = v.ss->n_off;
  for (int64_t j0 = blockIdx.x * (int64_t)blockDim.x; j0 < n; j0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = j0 + threadIdx.x;
    int code = 0;
    if (j < n) {
      const double x = v.cC[j];
      int lo = 0, hi = K;  // number of levels <= x
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (lv[mid] <= x) lo = mid + 1; else hi = mid;
      }
      code = lo;
      v.code[j] = static_cast<uint8_t>(code);
    }
    int m = code;
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && j < n) v.bsum[j >> 5] = static_cast<uint8_t>(m);
  }  // the streamed chain reads whole 16-byte words: codes past n are zero
  if (blockIdx.x == 0 && threadIdx.x < 32) v.code[n + threadIdx.x] = 0;
}

// The decision chain on byte codes: per hard victim one 32-byte probe of the
// arrival's block and one of the first block (shared-memory per-32 maxima)
// that can satisfy it, both in flight together.
__global__ void __launch_bounds__(1024) ks_chain_codes(StepView v) {
  extern __shared__ uint8_t sb[];
  if (aborted(v) || v.ss->mode != MODE_PAR || v.ss->codes_on != 1) return;
  const long long n = v.ss->n_off, F = v.ss->F, nh = v.ss->n_hard;
  const long long nblk = (n + 31) >> 5;
  for (long long b = threadIdx.x; b < nblk; b += blockDim.x) sb[b] = v.bsum[b];
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const uint8_t *code = v.code;
  const long long t_start = clock64();
  long long x = F, h = 0, nrej = 0;
  for (long long k0 = 0; k0 < nh; k0 += 32) {
    const long long kk = k0 + lane;
    const int32_t hp = kk < nh ? v.hard[kk] : 0;
    const int hr = kk < nh ? v.hrank[kk] : 0;
    const int cnt = nh - k0 < 32 ? static_cast<int>(nh - k0) : 32;
    bool stop = false;
    for (int t = 0; t < cnt; ++t) {
      const long long b = __shfl_sync(0xffffffffu, hp, t);
      const int r = __shfl_sync(0xffffffffu, hr, t);
      const long long gap = b - h;
      if (x + gap >= n) { x = n; stop = true; break; }
      x += gap;
      h = b;
      // next candidate j >= x with code[j] >= r
      const long long base = x & ~31ll;
      const long long p1 = base + lane;
      const int c1 = p1 < n ? code[p1] : 0;
      long long B = nblk;
      for (long long b0 = (x >> 5) + 1; b0 < nblk; b0 += 32) {
        const long long bb = b0 + lane;
        const unsigned m = __ballot_sync(0xffffffffu, bb < nblk && sb[bb] >= r);
        if (m) { B = b0 + __ffs(m) - 1; break; }
      }
      const long long p2 = B * 32 + lane;
      const int c2 = (B < nblk && p2 < n) ? code[p2] : 0;
      long long j = n;
      const unsigned m1 = __ballot_sync(0xffffffffu, p1 >= x && p1 < n && c1 >= r);
      if (m1) {
        j = base + __ffs(m1) - 1;
      } else if (B < nblk) {
        const unsigned m2 = __ballot_sync(0xffffffffu, p2 < n && c2 >= r);
        if (m2) j = B * 32 + __ffs(m2) - 1;
      }
      if (j > x) {
        if (lane == 0) {
          v.rj_beg[nrej] = static_cast<int32_t>(x);
          v.rj_end[nrej] = static_cast<int32_t>(j);
        }
        ++nrej;
      }
      if (j >= n) { x = n; stop = true; break; }
      x = j + 1;
      h = b + 1;
    }
    if (stop) break;
  }
  if (lane == 0) {
    v.ss->n_rej = nrej;
    v.ss->chain_cycles = clock64() - t_start;
  }
}

// The same chain with the codes streamed through a shared-memory ring: the
// chain's candidate position only moves forward, so producer warps copy the
// code array ahead of it (16-byte loads, several in flight per thread) while
// warp 0 walks the hard victims entirely from shared memory — the per-32
// maxima to skip, the ring to find the exact candidate. Warp 0 publishes the
// lowest position it can still need; producers restart there when it jumps.
constexpr int kRing = 1 << 16;        // ring bytes (power of two)
constexpr int kProdWarps = 16;        // producer warps (1..16)
constexpr int kProdUnroll = 2;        // 16-byte loads in flight per producer thread
constexpr int kChunk = kProdWarps * 32 * 16 * kProdUnroll;  // bytes per producer round
constexpr int kSumPad = 64;           // zero per-32 maxima past the last block

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }
__device__ __forceinline__ long long ld_acquire_cta(const volatile long long *p) {
  long long v;
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(const_cast<const long long *>(p)));
  asm volatile("ld.acquire.cta.shared::cta.b64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(volatile long long *p, long long v) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(const_cast<const long long *>(p)));
  asm volatile("st.release.cta.shared::cta.b64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}

__global__ void __launch_bounds__(1024) ks_chain_stream(StepView v) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ volatile long long filled, consumed, ppos;
  __shared__ volatile int done;
  __shared__ long long pstart;
  if (aborted(v) || v.ss->mode != MODE_PAR || v.ss->codes_on != 2) return;
  const long long n = v.ss->n_off, F = v.ss->F, nh = v.ss->n_hard;
  const long long nblk = (n + 31) >> 5;
  uint8_t *sum = smem;
  uint8_t *ring = smem + ((nblk + kSumPad + 15) & ~15ll);  // sum[] zero-padded past nblk
  for (long long b = threadIdx.x; b < nblk / 16; b += blockDim.x)
    reinterpret_cast<int4 *>(sum)[b] = __ldg(reinterpret_cast<const int4 *>(raw(v.bsum)) + b);
  for (long long b = nblk / 16 * 16 + threadIdx.x; b < nblk + kSumPad; b += blockDim.x)
    sum[b] = b < nblk ? v.bsum[b] : 0;
  if (threadIdx.x == 0) {
    filled = F & ~15ll;
    consumed = F & ~15ll;
    ppos = F & ~15ll;
    done = 0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= 1 && warp <= kProdWarps) {
    // ---- producers
    const int pt = threadIdx.x - 32;
    while (true) {
      if (pt == 0) {
        long long st;
        while (true) {
          const long long c = consumed;
          st = ppos > (c & ~15ll) ? ppos : (c & ~15ll);
          if (done || st >= n + 256 || st + kChunk <= c + kRing) break;
        }
        pstart = (done || st >= n + 256) ? -1 : st;  // the ring runs 256 zero codes past n
      }
      named_bar(1, kProdWarps * 32);
      const long long st = pstart;
      if (st < 0) break;
      int4 tmp[kProdUnroll];
#pragma unroll
      for (int u = 0; u < kProdUnroll; ++u) {
        const long long p = st + (static_cast<long long>(u) * kProdWarps * 32 + pt) * 16;
        tmp[u] = p < n ? __ldg(reinterpret_cast<const int4 *>(v.code + p)) : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < kProdUnroll; ++u) {
        const long long p = st + (static_cast<long long>(u) * kProdWarps * 32 + pt) * 16;
        *reinterpret_cast<int4 *>(ring + (p & (kRing - 1))) = tmp[u];
      }
      named_bar(1, kProdWarps * 32);  // orders every producer's ring stores before pt 0's release
      if (pt == 0) {
        ppos = st + kChunk;
        st_release_cta(&filled, st + kChunk);
      }
    }
    return;
  }
  if (warp != 0) return;
  // ---- the chain: 32-bit positions (n <= max_nnz < 2^31), every probe from
  // shared memory. A step reads a 256-candidate window at x (8 codes per
  // lane, byte-wise compares) and, in the same round, the per-32 maxima of
  // the 32 blocks after it; only a longer reject run scans further. The next
  // hard victim's (position, rank) is fetched a step ahead; codes past n are
  // zero (and ranks >= 1), so no probe needs an upper bound check.
  const long long t_start = clock64();
  const int n32 = static_cast<int>(n), nb32 = static_cast<int>(nblk);
  const int nh32 = static_cast<int>(nh);
  int x = static_cast<int>(F), h = 0, nrej = 0;
  int pub = x & ~31;  // last published `consumed`
  int fl = 0;         // last seen `filled`
  int thr = -1;       // a window at w > thr must refresh `filled` or publish progress
  const int lane8 = 8 * lane;
  int hp = lane < nh32 ? v.hard[lane] : 0, hpn = 32 + lane < nh32 ? v.hard[32 + lane] : 0;
  unsigned hr = lane < nh32 ? v.hrank[lane] * 0x01010101u : 0u;  // rank in every byte
  unsigned hrn = 32 + lane < nh32 ? v.hrank[32 + lane] * 0x01010101u : 0u;
  int b_nx = __shfl_sync(0xffffffffu, hp, 0);
  unsigned rr_nx = __shfl_sync(0xffffffffu, hr, 0);
  for (int k = 0; k < nh32; ++k) {
    const int b = b_nx;
    const unsigned rr = rr_nx;
    const int r = static_cast<int>(rr & 0xffu);
    const int t = (k + 1) & 31;
    if (t == 0) {
      hp = hpn;
      hr = hrn;
      const int kk = k + 33 + lane;
      hpn = kk < nh32 ? v.hard[kk] : 0;
      hrn = kk < nh32 ? v.hrank[kk] * 0x01010101u : 0u;
    }
    b_nx = __shfl_sync(0xffffffffu, hp, t);
    rr_nx = __shfl_sync(0xffffffffu, hr, t);
    x += b - h;  // easy victims between take one candidate each
    if (x >= n32) break;
    h = b + 1;
    const int w = x & ~31;
    if (w > thr) {  // rare: publish progress / wait for the window's codes
      pub = w;
      if (lane == 0) consumed = pub;
      while ((fl = static_cast<int>(ld_acquire_cta(&filled))) < w + 256) {
      }
      thr = min(fl - 256, pub + 16384);
    }
    const uint2 q = *reinterpret_cast<const uint2 *>(ring + ((w + lane8) & (kRing - 1)));
    const int sm = sum[(w >> 5) + 8 + lane];
    unsigned long long M = (static_cast<unsigned long long>(__vcmpgeu4(q.y, rr)) << 32) | __vcmpgeu4(q.x, rr);
    const int o = x & 31;  // lanes below o/8 hold codes below x; lane o/8 drops o%8
    M &= ~0ull << (lane == (o >> 3) ? (o & 7) * 8 : 0);
    const int byte = (__ffsll(static_cast<long long>(M)) - 1) >> 3;
    const unsigned mw = __ballot_sync(0xffffffffu, M != 0ull) & (0xffffffffu << (o >> 3));
    int j;
    if (mw) {
      const int L = __ffs(mw) - 1;
      j = w + 8 * L + __shfl_sync(0xffffffffu, byte, L);
    } else {
      int B = nb32;
      const unsigned mb = __ballot_sync(0xffffffffu, sm >= r);
      if (mb) {
        B = (w >> 5) + 8 + __ffs(mb) - 1;
      } else {
        for (int b0 = (w >> 5) + 40; b0 < nb32; b0 += 32) {
          const int bb = b0 + lane;
          const unsigned m3 = __ballot_sync(0xffffffffu, sum[bb] >= r);  // zero-padded past nblk
          if (m3) { B = b0 + __ffs(m3) - 1; break; }
        }
      }
      if (B >= nb32) {
        j = n32;
      } else {
        if (B * 32 + 32 > fl) {
          pub = B * 32;
          if (lane == 0) consumed = pub;
          while ((fl = static_cast<int>(ld_acquire_cta(&filled))) < B * 32 + 32) {
          }
          thr = min(fl - 256, pub + 16384);
        }
        const int c2 = ring[(B * 32 + lane) & (kRing - 1)];
        const unsigned m2 = __ballot_sync(0xffffffffu, c2 >= r);
        j = B * 32 + __ffs(m2) - 1;  // m2 != 0: the block's maximum reaches r
      }
    }
    if (j > x) {
      if (lane == 0) {
        v.rj_beg[nrej] = x;
        v.rj_end[nrej] = j;
      }
      ++nrej;
    }
    if (j >= n32) break;
    x = j + 1;
  }
  if (lane == 0) {
    v.ss->n_rej = nrej;
    v.ss->chain_cycles = clock64() - t_start;
    done = 1;
  }
}

// accept flag per candidate (0 inside a reject interval)
__global__ void ks_accept_flags(StepView v, int64_t max_nnz) {
  if (aborted(v)) return;
  const long long n = v.ss->n_off, nr = v.ss->n_rej, mode = v.ss->mode;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < max_nnz; j += (int64_t)gridDim.x * blockDim.x) {
    int32_t a = 0;
    if (j < n && mode == MODE_PAR) {
      // last interval with beg <= j
      long long lo = 0, hi = nr;
      while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (v.rj_beg[mid] <= j) lo = mid + 1; else hi = mid;
      }
      a = (lo > 0 && j < v.rj_end[lo - 1]) ? 0 : 1;
    }
    v.acc[j] = a;
  }
}

// side effects of the accepts, thread per candidate: accept rank r takes a
// free slot (r < F) or evicts V[r - F] and takes its slot; tick
// tick_base + r + 1. Rows are copied by ks_copy_rows.
__global__ void __launch_bounds__(256) ks_apply(CacheView c, StepView v) {
  if (aborted(v) || v.ss->mode != MODE_PAR) return;
  const long long n = v.ss->n_off, F = v.ss->F, e0 = v.ss->e0, ftop0 = v.ss->ftop0, log0 = v.ss->log0;
  const long long tick_base = v.ss->tick_base;
  const long long n_acc = n > 0 ? v.rank[n - 1] + v.acc[n - 1] : 0;
  const long long n_ev = n_acc > F ? n_acc - F : 0;
  for (int64_t j0 = blockIdx.x * (int64_t)blockDim.x; j0 < n; j0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = j0 + threadIdx.x;
    if (j < n && v.acc[j]) {
      const long long r = v.rank[j];
      const uint64_t key = v.okey[j];
      int32_t slot;
      if (r < F) {
        slot = c.free_stack[ftop0 - 1 - r];
        c.ssize[slot] = v.S;
      } else {
        const long long q = r - F;
        slot = v.q[q];
        const uint64_t ok = c.skey[slot];
        if (c.evlog_cap > 0 && log0 + q < c.evlog_cap) c.evlog[log0 + q] = ok;
        v.drow[dpos(v, ok)].slot = -1;
      }
      c.skey[slot] = key;
      c.stick[slot] = tick_base + r + 1;
      c.shits[slot] = 0;
      v.drow[dpos(v, key)].slot = slot;
      v.qnew[e0 - n_ev + r] = slot;
      v.aslot[r] = slot;
      v.akey[r] = key;
    }
  }

}

// row copies of the accepts (both decision modes): thread per 16 bytes
__global__ void __launch_bounds__(256) ks_copy_rows(CacheView c, StepView v) {
  if (aborted(v) || v.ss->mode == MODE_NONE) return;
  const long long na = v.ss->n_acc;
  const bool seq = v.ss->mode == MODE_SEQ;
  const int dim = v.dim;
  const bool vec = (dim & 3) == 0 && (c.row_ld & 3) == 0;
  const int per = vec ? dim / 4 : dim;
  const long long total = na * per;
  // (a four-pieces-per-thread variant measured slower: 187 vs 150 us at cfg3
  // alpha 1.0 / 2 %)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const long long r = i / per;
    const int k = static_cast<int>(i - r * per);
    const int32_t slot = v.aslot[r];
    const uint64_t key = v.akey[r];
    if (seq && (c.skey[slot] != key || c.stick[slot] == kFree)) continue;  // evicted again in the same call
    const float *src = row_src(v, key);
    float *dst = c.rows + static_cast<int64_t>(slot) * c.row_ld;
    if (vec) reinterpret_cast<float4 *>(dst)[k] = __ldg(reinterpret_cast<const float4 *>(src) + k);
    else dst[k] = __ldg(src + k);
  }
}

// surviving victims move to the queue front: qnew[i] = q[n_ev + i]
__global__ void ks_queue_survivors(CacheView c, StepView v) {
  if (aborted(v)) return;
  const StepScalars *s = v.ss;
  if (s->mode == MODE_SEQ) return;  // ks_seq_offer wrote qnew
  long long n_ev = 0;
  if (s->mode == MODE_PAR) {
    const long long n = s->n_off;
    const long long n_acc = n > 0 ? v.rank[n - 1] + v.acc[n - 1] : 0;
    n_ev = n_acc > s->F ? n_acc - s->F : 0;
  }
  const long long keep = s->e0 - n_ev;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < keep; i += (int64_t)gridDim.x * blockDim.x)
    v.qnew[i] = v.q[n_ev + i];
}

// the destination queue of the offers starts as all -1 (no-op for a rejected
// batch, whose queue stays where it is)
__global__ void ks_queue_clear(StepView v, int64_t scap) {
  if (aborted(v)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < scap; i += (int64_t)gridDim.x * blockDim.x)
    v.qnew[i] = -1;
}

__global__ void ks_queue_commit(StepView v, int64_t scap) {
  if (aborted(v)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < scap; i += (int64_t)gridDim.x * blockDim.x)
    v.q[i] = v.qnew[i];
}

__global__ void ks_offer_finish(CacheView c, StepView v) {
  if (aborted(v)) return;
  StepScalars *s = v.ss;
  Scalars *sc = c.sc;
  if (s->mode == MODE_PAR) {
    const long long n = s->n_off;
    const long long n_acc = n > 0 ? v.rank[n - 1] + v.acc[n - 1] : 0;
    const long long n_ev = n_acc > s->F ? n_acc - s->F : 0;
    const long long fr = n_acc < s->F ? n_acc : s->F;
    s->n_acc = n_acc;
    s->n_ev = n_ev;
    sc->entries = s->e0 + fr;
    sc->used = sc->entries * v.S;
    sc->tick = s->tick_base + n_acc;
    sc->free_top = s->ftop0 - fr;
    if (c.evlog_cap > 0) sc->n_evlog = s->log0 + n_ev;
    sc->n_acc = n_acc;
    sc->n_ev = n_ev;
    s->qlen_new = sc->entries;
  } else if (s->mode == MODE_NONE) {
    s->qlen_new = s->e0;
  }
  s->rebuild_index = 0;
}

// Exact sequential offers for batches outside the parallel domain
// (cache.py:237-268; V grows by this call's own accepts, or the cache is
// above budget). Single thread; rows are copied by ks_copy_rows.
__global__ void ks_seq_offer(CacheView c, StepView v) {
  if (aborted(v) || v.ss->mode != MODE_SEQ || threadIdx.x != 0 || blockIdx.x != 0) return;
  StepScalars *s = v.ss;
  Scalars *sc = c.sc;
  const long long n = s->n_off, e0 = s->e0, S = v.S, budget = sc->budget;
  long long e = e0, h = 0, n_acc = 0, ftop = sc->free_top, tick = s->tick_base, nlog = sc->n_evlog;
  const bool sketch = c.admission == 0;
  auto vslot = [&](long long q) -> int32_t { return q < e0 ? v.q[q] : v.aslot[q - e0]; };
  for (long long j = 0; j < n; ++j) {
    const double cj = v.cC[j];
    if (s->dyn && d_find(v, v.okey[j]) >= 0) continue;  // still cached: offer -> True, no side effect
    if ((e + 1) * S > budget) {
      if (sketch && e > 0) {
        const int32_t vs = vslot(h);
        const double ve = h < e0 ? k_est(c, c.skey[vs]) : v.cC[v.accj[h - e0]];
        if (cj < ve) continue;
      }
      while ((e + 1) * S > budget && e > 0) {
        const int32_t vs = vslot(h);
        ++h;
        const uint64_t ok = c.skey[vs];
        if (c.evlog_cap > 0 && nlog < c.evlog_cap) c.evlog[nlog] = ok;
        if (c.evlog_cap > 0) ++nlog;
        v.drow[dpos(v, ok)].slot = -1;
        c.stick[vs] = kFree;
        c.skey[vs] = kEmpty;
        c.free_stack[ftop++] = vs;
        --e;
      }
      if ((e + 1) * S > budget) continue;  // cannot fit (budget < S handled by the plan)
    }
    const uint64_t key = v.okey[j];
    const int32_t slot = c.free_stack[--ftop];
    ++tick;
    c.skey[slot] = key;
    c.skey2[slot] = 0;
    c.stick[slot] = tick;
    c.ssize[slot] = static_cast<int32_t>(S);
    c.shits[slot] = 0;
    v.drow[dpos(v, key)].slot = slot;
    v.aslot[n_acc] = slot;
    v.akey[n_acc] = key;
    v.accj[n_acc] = static_cast<int32_t>(j);
    ++n_acc;
    ++e;
  }
  // queue: V[h, e0 + n_acc) still resident, in order
  long long w = 0;
  for (long long q = h; q < e0 + n_acc; ++q) v.qnew[w++] = vslot(q);
  sc->entries = e;
  sc->used = e * S;
  sc->tick = tick;
  sc->free_top = ftop;
  sc->n_evlog = nlog;
  sc->n_acc = n_acc;
  s->n_acc = n_acc;
  s->n_ev = h;
  s->qlen_new = e;
}

__global__ void ks_index_clear(CacheView c, StepView v) {
  if (!v.ss->rebuild_index) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.hcap; i += (int64_t)gridDim.x * blockDim.x)
    c.hkeys[i] = kEmpty;
}

__global__ void ks_index_fill(CacheView c, StepView v) {
  if (!v.ss->rebuild_index) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.scap; i += (int64_t)gridDim.x * blockDim.x)
    if (c.stick[i] != kFree) h_insert(c, c.skey[i], static_cast<int32_t>(i));
  if (blockIdx.x == 0 && threadIdx.x == 0) c.sc->hash_tomb = 0;
}

// ---------------------------------------------------------------- 6. stage(limit)
// stage_hot_admissions(limit) (cache.py:311-342): hottest(limit) ranks every
// sketch key by (-count, key) and takes the top `limit`; cached / pending
// keys and keys larger than the spare room are skipped. Exact top-k by a
// radix select over the 128-bit key (~bits(count), key) with 16-bit digits;
// every kernel is a no-op unless room > 0.
__device__ __forceinline__ uint64_t vinv_of(double x) {
  return static_cast<uint64_t>(~__double_as_longlong(x) & LLONG_MAX);  // ascending = descending count
}

__global__ void ks_stage_begin(CacheView c, StepView v, int64_t limit) {
  StepScalars *s = v.ss;
  const Scalars *sc = c.sc;
  // every row here is S bytes: with room < S each of the hottest keys is
  // skipped as too big (cache.py:329-330), so the selection is skipped too
  s->stage_on = (s->err == 0 && limit > 0 && sc->budget - sc->used >= v.S && sc->sketch_live > 0) ? 1 : 0;
  s->topk_live = 0;
  s->topk_krem = limit;
  s->topk_hi = s->topk_lo = 0;
  s->topk_digit = 0;
  s->topk_n = 0;
  s->topk_fast = (s->stage_on && v.gs->stage_thr != 0) ? 1 : 0;
}

// Fast stage: the last selection's limit-th count, decayed by every age since
// (ks_age), bounds this batch's limit-th count from below unless those keys
// were pruned — counts only grow between ages. One pass collects the entries
// at or above it; if at least `limit` of them exist they hold the whole top
// `limit` and the radix select runs on that list alone (else: full path).
__global__ void __launch_bounds__(256) ks_topk_fast_collect(CacheView c, StepView v) {
  if (!v.ss->stage_on || !v.ss->topk_fast) return;
  const uint64_t thr = vinv_of(__longlong_as_double(v.gs->stage_thr));
  // four entries per thread (32-byte key and value loads); few entries pass,
  // so a warp appends with one atomic per ballot that has any
  const int64_t n4 = c.kcap >> 2;
  const ulonglong2 *k2 = reinterpret_cast<const ulonglong2 *>(raw(c.kkeys));
  const double2 *v2 = reinterpret_cast<const double2 *>(raw(c.kval));
  const int lane = threadIdx.x & 31;
  for (int64_t q0 = blockIdx.x * (int64_t)blockDim.x; q0 < n4; q0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = q0 + threadIdx.x;
    uint64_t kk[4] = {kEmpty, kEmpty, kEmpty, kEmpty};
    double vv[4] = {0.0, 0.0, 0.0, 0.0};
    if (q < n4) {
      const ulonglong2 a = k2[2 * q], b = k2[2 * q + 1];
      const double2 x = v2[2 * q], y = v2[2 * q + 1];
      kk[0] = a.x; kk[1] = a.y; kk[2] = b.x; kk[3] = b.y;
      vv[0] = x.x; vv[1] = x.y; vv[2] = y.x; vv[3] = y.y;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t vi = vinv_of(vv[u]);
      const bool in = kk[u] != kEmpty && kk[u] != kTomb && vi <= thr;
      const unsigned m = __ballot_sync(0xffffffffu, in);
      if (m) {
        const int leader = __ffs(m) - 1;
        unsigned long long base = 0;
        if (lane == leader)
          base = atomicAdd(reinterpret_cast<unsigned long long *>(&v.ss->topk_live),
                           static_cast<unsigned long long>(__popc(m)));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (in) {
          const long long p = static_cast<long long>(base) + __popc(m & ((1u << lane) - 1u));
          v.tk_key[p] = kk[u];
          v.tk_vinv[p] = vi;
        }
      }
    }
  }
}

__global__ void ks_topk_fast_check(StepView v) {
  StepScalars *s = v.ss;
  if (s->stage_on && s->topk_fast && s->topk_live < s->topk_krem) {
    s->topk_fast = 0;  // the bound missed (pruned keys): full path
    s->topk_live = 0;
  }
}

// pass 0 over the whole sketch: histogram of the top 16 bits of vinv. Decayed
// counts take few distinct values, so lanes are merged per warp (match_any)
// and bins per block in a shared-memory table before one global atomic per
// (block, bin): plain global atomics on a handful of hot bins serialise.
__global__ void __launch_bounds__(256) ks_topk_hist0(CacheView c, StepView v) {
  constexpr int kSlots = 1024;
  __shared__ int sbin[kSlots];
  __shared__ int scnt[kSlots];
  if (!v.ss->stage_on || v.ss->topk_fast) return;
  for (int i = threadIdx.x; i < kSlots; i += blockDim.x) {
    sbin[i] = -1;
    scnt[i] = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); i0 < c.kcap;
       i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + lane;
    int bin = -1;
    if (i < c.kcap) {
      const uint64_t k = c.kkeys[i];
      if (k != kEmpty && k != kTomb) bin = static_cast<int>(vinv_of(c.kval[i]) >> 48);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, bin);
    if (bin >= 0 && lane == __ffs(peers) - 1) {
      int h = (bin * 40503) & (kSlots - 1), probe = 0;
      for (; probe < kSlots; ++probe) {
        const int prev = atomicCAS(&sbin[h], -1, bin);
        if (prev == -1 || prev == bin) break;
        h = (h + 1) & (kSlots - 1);
      }
      if (probe < kSlots) atomicAdd(&scnt[h], __popc(peers));
      else atomicAdd(&v.tk_hist[bin], __popc(peers));  // table full: straight to global
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kSlots; i += blockDim.x)
    if (scnt[i]) atomicAdd(&v.tk_hist[sbin[i]], scnt[i]);
}

// live entries whose top digit is <= the selected one: every key that can be
// in the top `limit` (keys below the digit are in for sure)
__global__ void __launch_bounds__(256) ks_topk_collect(CacheView c, StepView v) {
  if (!v.ss->stage_on || v.ss->topk_fast) return;
  const uint64_t g0 = v.ss->topk_hi >> 48;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < c.kcap; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const uint64_t k = i < c.kcap ? c.kkeys[i] : kEmpty;
    uint64_t vi = 0;
    bool in = k != kEmpty && k != kTomb;
    if (in) {
      vi = vinv_of(c.kval[i]);
      in = (vi >> 48) <= g0;
    }
    const long long p = block_append(reinterpret_cast<unsigned long long *>(&v.ss->topk_live), in);
    if (in) {
      v.tk_key[p] = k;
      v.tk_vinv[p] = vi;
    }
  }
}

// A short list (the usual fast stage: about `limit` entries) is ranked in one
// block by counting — keys are distinct — instead of eight radix passes.
constexpr int kTopkSmall = 1024;
__global__ void __launch_bounds__(1024) ks_topk_small(StepView v) {
  __shared__ uint64_t sh[kTopkSmall], sl[kTopkSmall];
  __shared__ int cnt;
  StepScalars *s = v.ss;
  if (!s->stage_on || !s->topk_fast || s->topk_live > kTopkSmall) return;
  const int n = static_cast<int>(s->topk_live);
  const long long k = s->topk_krem;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sh[i] = v.tk_vinv[i];
    sl[i] = v.tk_key[i];
  }
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t hi = sh[i], lo = sl[i];
    int r = 0;
    for (int j = 0; j < n; ++j) r += (sh[j] < hi || (sh[j] == hi && sl[j] < lo)) ? 1 : 0;
    if (r < k) v.tk_sel[atomicAdd(&cnt, 1)] = i;  // ks_stage_finish orders them
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    s->topk_n = cnt;
    s->topk_digit = 8;  // the radix passes and the gather stand down
    s->topk_fast = 2;
  }
}

// digit d (0..7): d < 4 from vinv (most significant first), then from key
__device__ __forceinline__ uint32_t digit_of(uint64_t hi, uint64_t lo, int d) {
  return d < 4 ? static_cast<uint32_t>((hi >> (48 - 16 * d)) & 0xffff)
               : static_cast<uint32_t>((lo >> (48 - 16 * (d - 4))) & 0xffff);
}

__device__ __forceinline__ bool prefix_match(uint64_t hi, uint64_t lo, uint64_t phi, uint64_t plo, int d) {
  // digits [0, d) equal
  if (d == 0) return true;
  if (d <= 4) {
    const int sh = 64 - 16 * d;
    return (hi >> sh) == (phi >> sh);
  }
  if (hi != phi) return false;
  const int sh = 64 - 16 * (d - 4);
  return sh >= 64 ? true : (lo >> sh) == (plo >> sh);
}

// passes d >= 1 over the collected list
__global__ void __launch_bounds__(256) ks_topk_hist(StepView v, int d) {
  if (!v.ss->stage_on || v.ss->topk_digit == 8 || (d == 0 && !v.ss->topk_fast)) return;
  const long long n = v.ss->topk_live;
  const uint64_t phi = v.ss->topk_hi, plo = v.ss->topk_lo;
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); i0 < n;
       i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + lane;
    int bin = -1;
    if (i < n) {
      const uint64_t hi = v.tk_vinv[i], lo = v.tk_key[i];
      if (prefix_match(hi, lo, phi, plo, d)) bin = static_cast<int>(digit_of(hi, lo, d));
    }
    const unsigned peers = __match_any_sync(0xffffffffu, bin);
    if (bin >= 0 && lane == __ffs(peers) - 1) atomicAdd(&v.tk_hist[bin], __popc(peers));
  }
}

// one block: the digit holding the k-th remaining key (parallel prefix over
// the 65536 bins); a digit whose bucket is taken whole ends the search
__global__ void __launch_bounds__(1024) ks_topk_select(StepView v, int d) {
  __shared__ long long wsum[32];
  if (!v.ss->stage_on || v.ss->topk_digit == 8) return;
  constexpr int per = kTopkBins / 1024;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  long long sum = 0;
  for (int i = 0; i < per; ++i) sum += v.tk_hist[t * per + i];
  // inclusive block scan of the per-thread sums
  long long x = sum;
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    long long y = wsum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const long long z = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += z;
    }
    wsum[lane] = y;
  }
  __syncthreads();
  const long long incl = x + (w ? wsum[w - 1] : 0);
  const long long k = v.ss->topk_krem;
  const long long excl = incl - sum;
  if (t == 1023 && incl < k) {  // fewer than k keys in total: take every candidate
    v.ss->topk_hi = ~0ull;
    v.ss->topk_lo = ~0ull;
    v.ss->topk_digit = 8;
  }
  if (excl < k && k <= incl) {
    long long cum = excl;
    for (int i = 0; i < per; ++i) {
      const long long hc = v.tk_hist[t * per + i];
      if (cum + hc >= k) {
        const uint64_t g = static_cast<uint64_t>(t * per + i);
        const long long kr = k - cum;
        uint64_t hi = v.ss->topk_hi, lo = v.ss->topk_lo;
        if (d < 4) hi |= g << (48 - 16 * d);
        else lo |= g << (48 - 16 * (d - 4));
        if (hc == kr) {  // the whole bucket is in: close every lower digit
          if (d < 4) {
            hi |= (48 - 16 * d) ? ((1ull << (48 - 16 * d)) - 1) : 0ull;
            lo = ~0ull;
          } else {
            const int sh = 48 - 16 * (d - 4);
            lo |= sh ? ((1ull << sh) - 1) : 0ull;
          }
          v.ss->topk_digit = 8;
        }
        v.ss->topk_hi = hi;
        v.ss->topk_lo = lo;
        v.ss->topk_krem = kr;
        break;
      }
      cum += hc;
    }
  }
  __syncthreads();
  for (int i = t; i < kTopkBins; i += blockDim.x) v.tk_hist[i] = 0;
}

// the (vinv, key) <= threshold entries: exactly min(limit, live) of them
__global__ void __launch_bounds__(256) ks_topk_gather(StepView v) {
  if (!v.ss->stage_on || v.ss->topk_fast == 2) return;
  const long long n = v.ss->topk_live;
  const uint64_t thi = v.ss->topk_hi, tlo = v.ss->topk_lo;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    bool in = false;
    if (i < n) {
      const uint64_t hi = v.tk_vinv[i], lo = v.tk_key[i];
      in = hi < thi || (hi == thi && lo <= tlo);
    }
    const long long p = block_append(reinterpret_cast<unsigned long long *>(&v.ss->topk_n), in);
    if (in) v.tk_sel[p] = static_cast<int32_t>(i);
  }
}

// rank the <= limit selected keys; look their pending / cached state up in
// parallel; then the ordered staging loop over those flags (one block)
__global__ void __launch_bounds__(1024) ks_stage_finish(CacheView c, StepView v, int64_t limit) {
  if (!v.ss->stage_on) return;
  extern __shared__ unsigned char smem_raw[];
  const long long m = v.ss->topk_n < limit ? v.ss->topk_n : limit;
  uint64_t *hi = reinterpret_cast<uint64_t *>(smem_raw);
  uint64_t *lo = hi + limit;
  int32_t *ord = reinterpret_cast<int32_t *>(lo + limit);
  int32_t *kpos = ord + limit;
  for (long long i = threadIdx.x; i < m; i += blockDim.x) {
    const int32_t p = v.tk_sel[i];
    hi[i] = v.tk_vinv[p];
    lo[i] = v.tk_key[p];
  }
  __syncthreads();
  for (long long i = threadIdx.x; i < m; i += blockDim.x) {  // rank by counting (keys are distinct)
    long long r = 0;
    for (long long j = 0; j < m; ++j) r += (hi[j] < hi[i] || (hi[j] == hi[i] && lo[j] < lo[i])) ? 1 : 0;
    ord[r] = static_cast<int32_t>(i);
  }
  __syncthreads();
  for (long long r = threadIdx.x; r < m; r += blockDim.x) {  // -1: pending or cached (skipped)
    const uint64_t key = lo[ord[r]];
    const int64_t kp = k_find(c, key);
    kpos[r] = (kp < 0 || c.kflag[kp] || d_find(v, key) >= 0) ? -1 : static_cast<int32_t>(kp);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  // the next stage's bound: this selection's limit-th count (ks_age decays it)
  v.gs->stage_thr = m >= limit && m > 0
                        ? static_cast<long long>(~hi[ord[m - 1]] & static_cast<uint64_t>(LLONG_MAX))
                        : 0;
  Scalars *sc = c.sc;
  long long room = sc->budget - sc->used;
  long long staged = 0, pend = sc->pending;
  for (long long r = 0; r < m; ++r) {
    if (kpos[r] < 0) continue;
    const long long size = v.S;
    if (size > room) continue;
    if (pend >= c.pend_cap) break;
    c.pend[pend++] = lo[ord[r]];
    c.kflag[kpos[r]] = 1;
    room -= size;
    ++staged;
    if (staged >= limit) break;
  }
  sc->pending = pend;
  sc->staged = staged;
}

// sketch age (cache.py:128-136): halve, prune below prune_below
__global__ void __launch_bounds__(256) ks_age(CacheView c, StepView v) {
  if (v.ss->err) return;
  long long dead = 0;
  // four table entries per thread and iteration: two 16-byte key loads, the
  // value loads only for live entries, all issued before any is used
  const int64_t n4 = c.kcap >> 2;
  const ulonglong2 *k2 = reinterpret_cast<const ulonglong2 *>(raw(c.kkeys));
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n4; q += (int64_t)gridDim.x * blockDim.x) {
    const ulonglong2 a = k2[2 * q], b = k2[2 * q + 1];
    const uint64_t kk[4] = {a.x, a.y, b.x, b.y};
    double val[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) val[u] = (kk[u] != kEmpty && kk[u] != kTomb) ? c.kval[4 * q + u] : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (kk[u] == kEmpty || kk[u] == kTomb) continue;
      const int64_t i = 4 * q + u;
      const double x = val[u] * c.decay;
      if (x < c.prune) {
        c.kkeys[i] = kTomb;
        c.kval[i] = 0.0;
        c.kflag[i] = 0;
        ++dead;
      } else {
        c.kval[i] = x;
      }
    }
  }
  block_add(reinterpret_cast<unsigned long long *>(&c.sc->sketch_live), -dead);
  block_add(reinterpret_cast<unsigned long long *>(&c.sc->sketch_tomb), dead);
  if (blockIdx.x == 0 && threadIdx.x == 0 && v.gs->stage_thr != 0)
    v.gs->stage_thr = __double_as_longlong(__longlong_as_double(v.gs->stage_thr) * c.decay);
}

}  // namespace stp
}  // namespace fx

using namespace fx;
using namespace fx::stp;

struct fx_step {
  fx_cache *cache = nullptr;
  StepView v{};
  StepScalars *ss_base = nullptr;  // [slots + 1]: per in-flight batch, then the global block
  uint64_t *ckey_base = nullptr;   // [slots * max_nnz]
  double *cest_base = nullptr;     // [slots * max_nnz]
  int32_t slots = 1;
  int64_t max_nnz = 0, max_bags = 0;
  int64_t scap = 0;
  void *cub_tmp = nullptr;
  size_t cub_bytes = 0;
  std::vector<void *> allocs;
  int chain_smem = 0;
  int code_smem = 0;
  int stream_smem = 0;
  int stage_smem = 0;
  int64_t stage_limit_cap = 0;
  int64_t launches = 0;  // kernels this handle launched (CUB sweeps count 2)
  int64_t n_dense = 0;   // dense slot index length (sum of table rows)
  // The accepts' row copies (bandwidth-bound, nothing else in the batch reads
  // the cache rows) run on a side stream, forked after the decisions and
  // joined at the end of fx_step_maintain (or the next start / offer), so
  // they overlap the queue commit and the maintenance (FX_COPY_SIDE=0: inline)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool copy_pending = false;
  // one batch in flight (slots == 1): the post-probe LRU queue stays in qnew
  // after fx_step_start and fx_step_offer writes the final queue back into
  // fx_cache.q (the roles of the two buffers swap), so neither phase copies
  // the whole queue; true between such a start and its offer
  bool queue_in_qnew = false;
};

namespace {

template <typename T>
int salloc(fx_step *s, T **p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void **>(p), n * sizeof(T));
  if (e != cudaSuccess) return cuda_check(e, "fx_step: cudaMalloc");
  s->allocs.push_back(*p);
  return FX_OK;
}
#ifdef FX_BOUNDS
template <typename T>
int salloc(fx_step *s, CkPtr<T> *p, size_t n) {
  T *q = nullptr;
  const int rc = salloc(s, &q, n);
  *p = q;
  ck_size(*p, static_cast<long long>(n));
  return rc;
}
#endif

// side-stream work of the step (FX_COPY_SIDE=0: everything inline)
bool side_on() {
  static const bool on = !(getenv("FX_COPY_SIDE") && atoi(getenv("FX_COPY_SIDE")) == 0);
  return on;
}

// resident 256-thread blocks per SM for the side-stream row copies
// (FX_SIDE_BLOCKS; default 0 = a full grid). cfg3 ms per batch, alpha 1.0 /
// 1.2 / 0.6: full grid 1.224 / 0.772 / 2.84, 4 blocks 1.233 / 0.760 / 2.91,
// 2 blocks 1.360 / 0.798 / 3.23, inline 1.262 / 0.784 / 2.94
// (profiles/r2_summary.md)
int side_blocks() {
  static const int b = (getenv("FX_SIDE_BLOCKS") && atoi(getenv("FX_SIDE_BLOCKS")) > 0) ? atoi(getenv("FX_SIDE_BLOCKS"))
                                                                                         : 0;
  return b;
}

int side_fork(fx_step *s, cudaStream_t st) {
  if (!s->side) {
    if (cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming) != cudaSuccess)
      return cuda_check(cudaGetLastError(), "fx_step: side stream");
  }
  cudaEventRecord(s->ev_fork, st);
  cudaStreamWaitEvent(s->side, s->ev_fork, 0);
  return FX_OK;
}

// after launching on s->side: the next join waits for everything on it so far
void side_close(fx_step *s) {
  cudaEventRecord(s->ev_join, s->side);
  s->copy_pending = true;
}

// rejoin the side-stream work (plan counters of a start, row copies of an offer)
void join_copies(fx_step *s, cudaStream_t st) {
  if (s->copy_pending) {
    cudaStreamWaitEvent(st, s->ev_join, 0);
    s->copy_pending = false;
  }
}

int64_t pow2_ge(int64_t x) {
  int64_t p = 1024;
  while (p < x) p <<= 1;
  return p;
}

__global__ void k_lru_sortkeys(CacheView c, long long *keys, int32_t *vals, long long free_key) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.scap; i += (int64_t)gridDim.x * blockDim.x) {
    const long long t = c.stick[i];
    keys[i] = t == kFree ? free_key : t;
    vals[i] = static_cast<int32_t>(i);
  }
}

// dense slot index from the slots (after any entry point that moved entries)
__global__ void k_didx_clear(StepView v, int64_t n_dense) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_dense; i += (int64_t)gridDim.x * blockDim.x)
    v.drow[i].slot = -1;
}

__global__ void k_didx_fill(CacheView c, StepView v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.scap; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = c.skey[i];
    if (c.stick[i] == kFree || (k >> 63)) continue;  // free slot / pooled-result key
    const int64_t t = static_cast<int64_t>(k >> kRowBitsC);
    if (t < v.n_tables) v.drow[dpos(v, k)].slot = static_cast<int32_t>(i);
  }
}

__global__ void k_queue_from_sorted(CacheView c, const int32_t *sorted, int32_t *q, int64_t scap) {
  const long long e = c.sc->entries;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < scap; i += (int64_t)gridDim.x * blockDim.x)
    q[i] = i < e ? sorted[i] : -1;
}

int ensure_queue(fx_step *s, cudaStream_t st) {
  fx_cache *c = s->cache;
  const int64_t scap = c->v.scap;
  if (scap != s->scap) {
    set_error("fx_step: the cache's slot capacity changed; recreate the step");
    return FX_E_CONFIG;
  }
  if (c->q_cap < scap) {
    if (c->q) cudaFree(c->q);
    c->q = nullptr;
    int rc = cuda_check(cudaMalloc(&c->q, scap * sizeof(int32_t)), "fx_step: queue");
    if (rc) return rc;
    c->q_cap = scap;
    c->queue_valid = 0;
  }
  s->v.q = c->q;
  ck_size(s->v.q, scap);
  if (c->queue_valid) return FX_OK;
  // rebuild: occupied slots by ascending tick (free slots sort last)
  long long *k0 = reinterpret_cast<long long *>(raw(s->v.E));  // scratch: scap doubles
  long long *k1 = reinterpret_cast<long long *>(raw(s->v.tk_vinv));
  int32_t *v0 = s->v.hardf, *v1 = s->v.hard;
  k_lru_sortkeys<<<grid_for(scap, 256), 256, 0, st>>>(c->v, k0, v0, LLONG_MAX);
  size_t need = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, need, k0, k1, v0, v1, static_cast<int>(scap), 0, 64, st);
  void *tmp = nullptr;
  int rc = cuda_check(cudaMallocAsync(&tmp, need, st), "fx_step: sort tmp");
  if (rc) return rc;
  cub::DeviceRadixSort::SortPairs(tmp, need, k0, k1, v0, v1, static_cast<int>(scap), 0, 64, st);
  k_queue_from_sorted<<<grid_for(scap, 256), 256, 0, st>>>(c->v, v1, c->q, scap);
  cudaFreeAsync(tmp, st);
  k_didx_clear<<<grid_for(s->n_dense, 256), 256, 0, st>>>(s->v, s->n_dense);
  k_didx_fill<<<grid_for(scap, 256), 256, 0, st>>>(c->v, s->v);
  FX_LAUNCH_CHECK("fx_step: queue rebuild");
  c->queue_valid = 1;
  return FX_OK;
}

int select_slot(fx_step *s, int32_t slot, StepView *v) {
  if (slot < 0 || slot >= s->slots) {
    set_error("fx_step: slot out of range");
    return FX_E_CONFIG;
  }
  *v = s->v;
  v->ss = s->ss_base + slot;
  v->gs = s->ss_base + s->slots;
  v->ckey = s->ckey_base + static_cast<int64_t>(slot) * s->max_nnz;
  v->cest = s->cest_base + static_cast<int64_t>(slot) * s->max_nnz;
  ck_size(v->ckey, s->max_nnz);
  ck_size(v->cest, s->max_nnz);
  v->q = s->cache->q;
  ck_size(v->q, s->cache->q_cap);
  return FX_OK;
}

}  // namespace

extern "C" {

int fx_step_create(fx_step **out, fx_cache *cache, int64_t max_nnz, int64_t max_bags, const float *const *table_base,
                   const int64_t *table_ld, const int64_t *table_rows, int32_t n_tables, int32_t dim,
                   int64_t stage_limit_cap, int32_t slots) {
  if (!out || !cache || max_nnz < 0 || max_bags < 0 || n_tables < 1 || dim < 1 || dim > cache->v.row_ld ||
      slots < 1 || slots > 64) {
    set_error("fx_step_create: bad arguments");
    return FX_E_CONFIG;
  }
  if (max_nnz >= (1ll << 31) - 1) {
    set_error("fx_step_create: max_nnz must be < 2^31 (int32 ordinals)");
    return FX_E_CONFIG;
  }
  fx_step *s = new fx_step();
  s->cache = cache;
  s->slots = slots;
  s->max_nnz = max_nnz > 0 ? max_nnz : 1;
  s->max_bags = max_bags > 0 ? max_bags : 1;
  s->scap = cache->v.scap;
  StepView &v = s->v;
  const int64_t N = s->max_nnz, SC = s->scap;
  v.max_nnz = N;
  v.dcap = pow2_ge(2 * N);
  v.n_tables = n_tables;
  v.dim = dim;
  v.S = dim * 4;
  v.tk_cap = cache->v.kcap > SC ? cache->v.kcap : SC;
  int rc = FX_OK;
  rc = rc ? rc : salloc(s, &s->ss_base, slots + 1);
  rc = rc ? rc : salloc(s, &s->ckey_base, static_cast<size_t>(slots) * N);
  rc = rc ? rc : salloc(s, &v.dkey, N);
  rc = rc ? rc : salloc(s, &v.dent, N);
  rc = rc ? rc : salloc(s, &v.dfraw, N);
  rc = rc ? rc : salloc(s, &v.uniq, N);
  rc = rc ? rc : salloc(s, &v.inv, N);
  rc = rc ? rc : salloc(s, &v.umiss, N);
  rc = rc ? rc : salloc(s, &v.cand_by_first, N);
  rc = rc ? rc : salloc(s, &v.hit_by_last, N);
  rc = rc ? rc : salloc(s, &v.cand, N);
  rc = rc ? rc : salloc(s, &v.hits_ord, N);
  rc = rc ? rc : salloc(s, &v.estv, N);
  rc = rc ? rc : salloc(s, &v.pres, N);
  rc = rc ? rc : salloc(s, &v.cidx, N);
  rc = rc ? rc : salloc(s, &v.okey, N);
  rc = rc ? rc : salloc(s, &v.cC, N);
  rc = rc ? rc : salloc(s, &v.bmax, (N + kFine - 1) / kFine + 1);
  rc = rc ? rc : salloc(s, &v.qnew, SC);
  rc = rc ? rc : salloc(s, &v.hitbits, (SC + 31) / 32);
  rc = rc ? rc : salloc(s, &v.E, SC);
  rc = rc ? rc : salloc(s, &v.hardf, SC);
  rc = rc ? rc : salloc(s, &v.hardbits, (SC + 31) / 32);
  rc = rc ? rc : salloc(s, &v.hard, SC);
  rc = rc ? rc : salloc(s, &v.rj_beg, SC + 1);
  rc = rc ? rc : salloc(s, &v.rj_end, SC + 1);
  rc = rc ? rc : salloc(s, &v.acc, N);
  rc = rc ? rc : salloc(s, &v.rank, N);
  rc = rc ? rc : salloc(s, &v.code, N + kChunk);
  rc = rc ? rc : salloc(s, &v.bsum, N / 32 + 2);
  rc = rc ? rc : salloc(s, &v.hrank, SC);
  rc = rc ? rc : salloc(s, &v.levels, 256);
  rc = rc ? rc : salloc(s, &v.aslot, N);
  rc = rc ? rc : salloc(s, &v.akey, N);
  rc = rc ? rc : salloc(s, &v.claim, N);
  rc = rc ? rc : salloc(s, &v.dC, N);
  rc = rc ? rc : salloc(s, &s->cest_base, static_cast<size_t>(slots) * N);
  rc = rc ? rc : salloc(s, &v.accj, N);
  rc = rc ? rc : salloc(s, &v.tk_key, v.tk_cap);
  rc = rc ? rc : salloc(s, &v.tk_vinv, v.tk_cap);
  rc = rc ? rc : salloc(s, &v.tk_val, v.tk_cap);
  rc = rc ? rc : salloc(s, &v.tk_flag, v.tk_cap);
  rc = rc ? rc : salloc(s, &v.tk_hist, kTopkBins);
  rc = rc ? rc : salloc(s, &v.tk_sel, v.tk_cap);
  float **tb = nullptr;
  int64_t *tl = nullptr, *tr = nullptr;
  rc = rc ? rc : salloc(s, &tb, n_tables);
  rc = rc ? rc : salloc(s, &tl, n_tables);
  rc = rc ? rc : salloc(s, &tr, n_tables);
  if (rc) {
    fx_step_destroy(s);
    return rc;
  }
  cudaMemcpy(tb, table_base, n_tables * sizeof(float *), cudaMemcpyHostToDevice);
  cudaMemcpy(tl, table_ld, n_tables * sizeof(int64_t), cudaMemcpyHostToDevice);
  cudaMemcpy(tr, table_rows, n_tables * sizeof(int64_t), cudaMemcpyHostToDevice);
  v.tbase = tb;
  v.tld = tl;
  v.trows = tr;
  {
    std::vector<int64_t> kb(n_tables);
    int64_t tot = 0;
    for (int32_t t = 0; t < n_tables; ++t) {
      kb[t] = tot;
      tot += table_rows[t] > 0 ? table_rows[t] : 0;
    }
    s->n_dense = tot > 0 ? tot : 1;
    int64_t *kbd = nullptr;
    rc = salloc(s, &kbd, n_tables);
    rc = rc ? rc : salloc(s, &v.drow, static_cast<size_t>(s->n_dense));
    if (rc) {
      fx_step_destroy(s);
      return rc;
    }
    cudaMemcpy(kbd, kb.data(), n_tables * sizeof(int64_t), cudaMemcpyHostToDevice);
    v.kbase = kbd;
    cudaMemset(raw(v.drow), 0, static_cast<size_t>(s->n_dense) * sizeof(DRow));
    int rb = 1;
    while ((1ll << rb) < N) ++rb;
    if (rb > 26) {
      set_error("fx_step_create: max_nnz above 2^26 (dense dedup claim words)");
      fx_step_destroy(s);
      return FX_E_CONFIG;
    }
    v.rep_bits = rb;
    cache->queue_valid = 0;  // the dense index is built with the queue
  }
  const int big = static_cast<int>(N > SC ? N : SC);
  size_t b1 = 0, b2 = 0, b3 = 0, b4 = 0;
  cub::DeviceSelect::If(nullptr, b1, (const int32_t *)nullptr, (int32_t *)nullptr, (int64_t *)nullptr, big, NonNeg());
  cub::DeviceSelect::Flagged(nullptr, b2, cub::CountingInputIterator<int32_t>(0), (const int32_t *)nullptr,
                             (int32_t *)nullptr, (int64_t *)nullptr, big);
  cub::DeviceScan::ExclusiveSum(nullptr, b3, (const int32_t *)nullptr, (int32_t *)nullptr, static_cast<int>(N));
  QueueKeep qk{nullptr};
  cub::DeviceSelect::If(nullptr, b4, (const int32_t *)nullptr, (int32_t *)nullptr, (int64_t *)nullptr,
                        static_cast<int>(SC), qk);
  size_t b5 = 0;
  cub::DeviceSelect::If(nullptr, b5, cub::CountingInputIterator<int32_t>(0), (int32_t *)nullptr, (int64_t *)nullptr,
                        static_cast<int>(SC), HardBit{nullptr});
  s->cub_bytes = b1 > b2 ? b1 : b2;
  if (b3 > s->cub_bytes) s->cub_bytes = b3;
  if (b4 > s->cub_bytes) s->cub_bytes = b4;
  if (b5 > s->cub_bytes) s->cub_bytes = b5;
  rc = cuda_check(cudaMalloc(&s->cub_tmp, s->cub_bytes + 256), "fx_step: cub tmp");
  if (rc) {
    fx_step_destroy(s);
    return rc;
  }
  s->allocs.push_back(s->cub_tmp);
  cudaMemset(s->ss_base, 0, (slots + 1) * sizeof(StepScalars));
  cudaMemset(raw(v.hitbits), 0, (SC + 31) / 32 * 4);
  cudaMemset(v.tk_hist, 0, kTopkBins * 4);
  const int64_t nblk = (N + kFine - 1) / kFine;
  s->chain_smem = static_cast<int>(nblk * sizeof(double));
  if (s->chain_smem > 227 * 1024) {
    set_error("fx_step_create: max_nnz too large for the chain's shared-memory block maxima");
    fx_step_destroy(s);
    return FX_E_CONFIG;
  }
  cudaFuncSetAttribute(ks_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, s->chain_smem > 0 ? s->chain_smem : 8);
  s->code_smem = static_cast<int>(N / 32 + 2);
  if (s->code_smem > 227 * 1024) {
    set_error("fx_step_create: max_nnz too large for the chain's shared-memory block maxima");
    fx_step_destroy(s);
    return FX_E_CONFIG;
  }
  cudaFuncSetAttribute(ks_chain_codes, cudaFuncAttributeMaxDynamicSharedMemorySize, s->code_smem);
  cudaFuncSetAttribute(ks_dedup<int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kDSmem));
  cudaFuncSetAttribute(ks_dedup<int64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kDSmem));
  {
    const int64_t need = ((N / 32 + 2 + kSumPad + 15) & ~15ll) + kRing;
    s->stream_smem = need + 1024 <= 227 * 1024 ? static_cast<int>(need) : 0;  // else the global-memory chain
    if (s->stream_smem)
      cudaFuncSetAttribute(ks_chain_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, s->stream_smem);
  }
  s->stage_limit_cap = stage_limit_cap > 0 ? stage_limit_cap : 64;
  s->stage_smem = static_cast<int>(s->stage_limit_cap * (8 + 8 + 4 + 4));
  cudaFuncSetAttribute(ks_stage_finish, cudaFuncAttributeMaxDynamicSharedMemorySize, s->stage_smem);
  rc = cuda_check(cudaDeviceSynchronize(), "fx_step_create");
  if (rc) {
    fx_step_destroy(s);
    return rc;
  }
  *out = s;
  return FX_OK;
}

int fx_step_destroy(fx_step *s) {
  if (!s) return FX_OK;
  if (s->side) cudaStreamDestroy(s->side);
  if (s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s->ev_join) cudaEventDestroy(s->ev_join);
  for (void *p : s->allocs) cudaFree(p);
  delete s;
  return FX_OK;
}

int fx_step_prepare(fx_step *s, void *stream) { return ensure_queue(s, as_stream(stream)); }

int fx_step_start(fx_step *s, int32_t slot, const int32_t *bag_table, const void *indices, int32_t idx_type,
                  const int64_t *offsets, const int64_t *sm_start, int64_t n_bags, int64_t nnz, int32_t threshold,
                  int32_t *hits_bag, int32_t *pd_groups, int32_t *pd_rows, int32_t *raw_rows, void *stream) {
  cudaStream_t st = as_stream(stream);
  if (nnz > s->max_nnz || n_bags > s->max_bags || nnz < 0 || n_bags < 0) {
    set_error("fx_step_start: batch larger than the step's capacity");
    return FX_E_CAPACITY;
  }
  join_copies(s, st);
  if (s->queue_in_qnew) {  // the previous start's offers never ran: rebuild the queue from the ticks
    s->cache->queue_valid = 0;
    s->queue_in_qnew = false;
  }
  int rc = ensure_queue(s, st);
  if (rc) return rc;
  StepView v;
  rc = select_slot(s, slot, &v);
  if (rc) return rc;
  fx_cache *cc = s->cache;
  CacheView &c = cc->v;
  const int64_t SC = s->scap;
  if (c.kcap > v.tk_cap) {
    set_error("fx_step_start: sketch grew beyond the step's temporaries; recreate the step");
    return FX_E_CONFIG;
  }
  ks_begin<<<1, 1, 0, st>>>(c, v, nnz);
  s->launches += 1;
  // dedup table reset: a memset beats clearing the claimed slots one by one
  cudaMemsetAsync(v.dent, 0, static_cast<size_t>(nnz > 0 ? nnz : 1) * sizeof(DEnt), st);
  if (threshold > 0) cudaMemsetAsync(v.dfraw, 0, static_cast<size_t>(nnz > 0 ? nnz : 1) * sizeof(int32_t), st);
  ks_claim_clear<<<grid_for(s->n_dense, 256), 256, 0, st>>>(v, s->n_dense);
  s->launches += 1;
  ks_sketch_collect<<<grid_for(c.kcap, 256), 256, 0, st>>>(c, v);
  s->launches += 1;
  ks_sketch_clear<<<grid_for(c.kcap, 256), 256, 0, st>>>(c, v);
  s->launches += 1;
  ks_sketch_reinsert<<<grid_for(c.kcap, 256), 256, 0, st>>>(c, v);
  s->launches += 1;
  // validation + dedup first: a bad index aborts the batch before any state change
  if (n_bags > 0) {
    int g = static_cast<int>((n_bags + kDBags - 1) / kDBags);
    const int gmax = num_sms() * 2;
    if (g > gmax) g = gmax;
    static const bool occ = !(getenv("FX_DEDUP") && std::string(getenv("FX_DEDUP")) == "blk");
    if (occ) {
      // bags per warp (FX_DEDUP_BW, default 32). cfg3 2 % / 1 % cache, ms per
      // batch at 32 / 16 / 8 / 4 bags per warp: alpha 1.0 1.238 / 1.258 /
      // 1.284 / 1.301, alpha 1.2 0.790 / 0.798 / 0.810 / 0.837, alpha 0.6
      // 2.865 / 2.866 / 2.854 / 2.846 (profiles/r2_summary.md)
      static const int bw = (getenv("FX_DEDUP_BW") && atoi(getenv("FX_DEDUP_BW")) >= 1 &&
                             atoi(getenv("FX_DEDUP_BW")) <= 32) ? atoi(getenv("FX_DEDUP_BW")) : 32;
      const int go = grid_for((n_bags + bw - 1) / bw * 32, 256);
      if (idx_type == FX_IDX_I32)
        ks_dedup_occ<int32_t><<<go, 256, 0, st>>>(v, bag_table, static_cast<const int32_t *>(indices), offsets,
                                                  sm_start, n_bags, bw);
      else
        ks_dedup_occ<int64_t><<<go, 256, 0, st>>>(v, bag_table, static_cast<const int64_t *>(indices), offsets,
                                                  sm_start, n_bags, bw);
    } else if (idx_type == FX_IDX_I32) {
      ks_dedup<int32_t><<<g, 256, kDSmem, st>>>(v, bag_table, static_cast<const int32_t *>(indices), offsets,
                                                sm_start, n_bags);
    } else {
      ks_dedup<int64_t><<<g, 256, kDSmem, st>>>(v, bag_table, static_cast<const int64_t *>(indices), offsets,
                                                sm_start, n_bags);
    }
    s->launches += 1;
  }
  const int nn = static_cast<int>(nnz > 0 ? nnz : 1);
  size_t cb = s->cub_bytes;
  // ranker.py:218-222 order: validate, apply_pending, (admission check: host), probes
  ks_apply_pending<<<1, 32, 0, st>>>(c, v);
  s->launches += 1;
  cudaMemsetAsync(v.cand_by_first, 0xff, static_cast<size_t>(nn) * 4, st);
  cudaMemsetAsync(raw(v.hitbits), 0, static_cast<size_t>((SC + 31) / 32) * 4, st);
  cudaMemsetAsync(v.hit_by_last, 0xff, static_cast<size_t>(nn) * 4, st);
  {  // keys in flight per thread (FX_PROBE_ILP: 2 default, 4 measured 2.5 % slower)
    static const int ilp = (getenv("FX_PROBE_ILP") && atoi(getenv("FX_PROBE_ILP")) == 4) ? 4 : 2;
    if (ilp == 4)
      ks_probe<4><<<grid_for(nn, 256), 256, 0, st>>>(c, v, threshold > 0 ? 1 : 0, nnz);
    else
      ks_probe<2><<<grid_for(nn, 256), 256, 0, st>>>(c, v, threshold > 0 ? 1 : 0, nnz);
  }
  s->launches += 1;
  ks_after_probe<<<1, 1, 0, st>>>(c, v, nnz);
  s->launches += 1;
  // (on a side stream beside the compactions the plan measured slower: the
  // compactions and the plan both want every SM)
  ks_bag_plan<<<grid_for(n_bags > 0 ? n_bags * 32 : 32, 256), 256, 0, st>>>(v, offsets, sm_start, n_bags, threshold,
                                                                            hits_bag, pd_groups, pd_rows, raw_rows);
  s->launches += 1;
  if (threshold > 0) {
    ks_cand_scatter_raw<<<grid_for(nn, 256), 256, 0, st>>>(v, nnz);
    s->launches += 1;
  }
  // candidates in first raw-occurrence order; hit slots in last-ordinal order
  cub::DeviceSelect::If(s->cub_tmp, cb, raw(v.cand_by_first), raw(v.cand), reinterpret_cast<int64_t *>(&v.ss->n_cand), nn,
                        NonNeg(), st);
  s->launches += 2;
  ks_cand_keys<<<grid_for(nn, 256), 256, 0, st>>>(v);
  s->launches += 1;
  cub::DeviceSelect::If(s->cub_tmp, cb, raw(v.hit_by_last), raw(v.hits_ord), reinterpret_cast<int64_t *>(&v.ss->n_hitu), nn,
                        NonNeg(), st);
  s->launches += 2;
  // LRU order after the probes: [entries not hit, old order] ++ [hit entries by last ordinal]
  // with one batch in flight only qnew[0, entries) is read before the offers
  // rewrite fx_cache.q; otherwise qnew is copied back whole (-1 beyond)
  if (s->slots > 1) cudaMemsetAsync(v.qnew, 0xff, SC * 4, st);
  QueueKeep qk{raw(v.hitbits)};
  cub::DeviceSelect::If(s->cub_tmp, cb, cc->q, raw(v.qnew), reinterpret_cast<int64_t *>(&v.ss->n_nonhit),
                        static_cast<int>(SC), qk, st);
  s->launches += 2;
  ks_queue_append_hits<<<grid_for(nn, 256), 256, 0, st>>>(v);
  s->launches += 1;
  if (s->slots == 1) {
    s->queue_in_qnew = true;  // the offers read it from qnew (no copy back)
  } else {
    cudaMemcpyAsync(cc->q, raw(v.qnew), SC * 4, cudaMemcpyDeviceToDevice, st);
  }
  cc->hash_valid = 0;  // the fast path keeps the dense index; the hash is rebuilt on demand
  FX_LAUNCH_CHECK("fx_step_start");
  return FX_OK;
}

int fx_step_offer(fx_step *s, int32_t slot, void *stream) {
  cudaStream_t st = as_stream(stream);
  join_copies(s, st);
  const bool swapped = s->queue_in_qnew && s->cache->queue_valid;
  s->queue_in_qnew = false;  // either consumed below, or invalidated meanwhile and rebuilt from the ticks
  int rc = ensure_queue(s, st);
  if (rc) return rc;
  StepView v;
  rc = select_slot(s, slot, &v);
  if (rc) return rc;
  if (swapped) {  // current queue = qnew; the offers write the final queue into fx_cache.q
    CkPtr<int32_t> t = v.q;
    v.q = v.qnew;
    v.qnew = t;
  }
  fx_cache *cc = s->cache;
  CacheView &c = cc->v;
  const int64_t SC = s->scap;
  const int nn = static_cast<int>(s->max_nnz);
  size_t cb = s->cub_bytes;
  ks_offer_prep<<<grid_for(nn, 256), 256, 0, st>>>(c, v, nn, s->slots == 1 ? 1 : 0);
  s->launches += 1;
  if (s->slots == 1) {
    ks_cidx_identity<<<grid_for(nn, 256), 256, 0, st>>>(v);
    s->launches += 1;
  } else {
    ks_offer_flags<<<grid_for(nn, 256), 256, 0, st>>>(v, nn);
    s->launches += 1;
    cub::DeviceSelect::Flagged(s->cub_tmp, cb, cub::CountingInputIterator<int32_t>(0), raw(v.pres), raw(v.cidx),
                               reinterpret_cast<int64_t *>(&v.ss->n_off), nn, st);
    s->launches += 2;
  }
  ks_cand_est<<<grid_for(nn, kFine), kFine, 0, st>>>(v);
  s->launches += 1;
  ks_offer_plan<<<1, 1, 0, st>>>(c, v);
  s->launches += 1;
  ks_victim_est<<<grid_for(SC, 256), 256, 0, st>>>(c, v, SC);
  s->launches += 1;
  cub::DeviceSelect::If(s->cub_tmp, cb, cub::CountingInputIterator<int32_t>(0), raw(v.hard),
                        reinterpret_cast<int64_t *>(&v.ss->n_hard), static_cast<int>(SC), HardBit{raw(v.hardbits)}, st);
  s->launches += 2;
  ks_levels<<<1, 1024, 0, st>>>(v, s->stream_smem > 0 ? 1 : 0);
  s->launches += 1;
  ks_cand_codes<<<grid_for(nn, 256), 256, 0, st>>>(v);
  s->launches += 1;
  if (s->stream_smem > 0) ks_chain_stream<<<1, 1024, s->stream_smem, st>>>(v);
  s->launches += 1;
  ks_chain_codes<<<1, 1024, s->code_smem, st>>>(v);
  s->launches += 1;
  ks_chain<<<1, 1024, s->chain_smem, st>>>(v);
  s->launches += 1;
  ks_accept_flags<<<grid_for(nn, 256), 256, 0, st>>>(v, nn);
  s->launches += 1;
  cub::DeviceScan::ExclusiveSum(s->cub_tmp, cb, raw(v.acc), raw(v.rank), nn, st);
  s->launches += 2;
  ks_queue_clear<<<grid_for(SC, 256), 256, 0, st>>>(v, SC);
  s->launches += 1;
  ks_apply<<<grid_for(nn, 256), 256, 0, st>>>(c, v);
  s->launches += 1;
  ks_queue_survivors<<<grid_for(SC, 256), 256, 0, st>>>(c, v);
  s->launches += 1;
  ks_seq_offer<<<1, 1, 0, st>>>(c, v);
  s->launches += 1;
  ks_offer_finish<<<1, 1, 0, st>>>(c, v);
  s->launches += 1;
  if (side_on()) {
    rc = side_fork(s, st);
    if (rc) return rc;
    ks_copy_rows<<<side_blocks() > 0 ? num_sms() * side_blocks()
                                      : grid_for(static_cast<int64_t>(nn) * (v.dim / 4 + 1), 256),
                   256, 0, s->side>>>(c, v);
    side_close(s);
  } else {
    ks_copy_rows<<<grid_for(static_cast<int64_t>(nn) * (v.dim / 4 + 1), 256), 256, 0, st>>>(c, v);
  }
  s->launches += 1;
  if (!swapped) {
    ks_queue_commit<<<grid_for(SC, 256), 256, 0, st>>>(v, SC);
    s->launches += 1;
  }
  FX_LAUNCH_CHECK("fx_step_offer");
  return FX_OK;
}

int fx_step_maintain(fx_step *s, int32_t slot, int64_t stage_limit, int32_t do_age, void *stream) {
  cudaStream_t st = as_stream(stream);
  StepView v;
  int rc = select_slot(s, slot, &v);
  if (rc) return rc;
  CacheView &c = s->cache->v;
  if (stage_limit > s->stage_limit_cap) {
    set_error("fx_step_maintain: stage limit above the step's cap");
    return FX_E_CONFIG;
  }
  ks_stage_begin<<<1, 1, 0, st>>>(c, v, stage_limit);
  s->launches += 1;
  if (stage_limit > 0) {
    ks_topk_fast_collect<<<grid_for(c.kcap / 4, 256), 256, 0, st>>>(c, v);
    ks_topk_fast_check<<<1, 1, 0, st>>>(v);
    ks_topk_small<<<1, 1024, 0, st>>>(v);
    s->launches += 1;
    ks_topk_hist<<<grid_for(4 * 65536, 256), 256, 0, st>>>(v, 0);  // fast: digit 0 over the list
    ks_topk_hist0<<<grid_for(c.kcap, 256), 256, 0, st>>>(c, v);     // else: over the whole sketch
    s->launches += 4;
    ks_topk_select<<<1, 1024, 0, st>>>(v, 0);
    s->launches += 1;
    ks_topk_collect<<<grid_for(c.kcap, 256), 256, 0, st>>>(c, v);
    s->launches += 1;
    for (int d = 1; d < 8; ++d) {
      ks_topk_hist<<<grid_for(4 * 65536, 256), 256, 0, st>>>(v, d);
      s->launches += 1;
      ks_topk_select<<<1, 1024, 0, st>>>(v, d);
      s->launches += 1;
    }
    ks_topk_gather<<<grid_for(c.kcap, 256), 256, 0, st>>>(v);
    s->launches += 1;
    ks_stage_finish<<<1, 1024, s->stage_smem, st>>>(c, v, stage_limit);
    s->launches += 1;
  }
  if (do_age) {
    ks_age<<<grid_for(c.kcap / 4, 256), 256, 0, st>>>(c, v);
    s->launches += 1;
  }
  join_copies(s, st);
  FX_LAUNCH_CHECK("fx_step_maintain");
  return FX_OK;
}

int fx_step_join(fx_step *s, void *stream) {
  if (!s) return FX_OK;
  join_copies(s, as_stream(stream));
  return cuda_check(cudaGetLastError(), "fx_step_join");
}

int fx_step_scalars(fx_step *s, int32_t slot, int64_t *out, int64_t n, void *stream) {
  cudaStream_t st = as_stream(stream);
  if (slot < 0 || slot > s->slots) {
    set_error("fx_step_scalars: slot out of range");
    return FX_E_CONFIG;
  }
  const int64_t cnt = static_cast<int64_t>(sizeof(StepScalars) / 8);
  int rc = cuda_check(cudaMemcpyAsync(out, s->ss_base + slot, (n < cnt ? n : cnt) * 8, cudaMemcpyDeviceToHost, st),
                      "fx_step_scalars");
  if (rc) return rc;
  return cuda_check(cudaStreamSynchronize(st), "fx_step_scalars sync");
}

int64_t fx_step_launches(fx_step *s) { return s->launches; }

const void *fx_step_scalars_device(fx_step *s, int32_t slot) {
  return (slot >= 0 && slot <= s->slots) ? static_cast<const void *>(s->ss_base + slot) : nullptr;
}

}  // extern "C"
