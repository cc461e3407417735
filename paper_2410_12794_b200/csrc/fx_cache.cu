// K3 cache probe + K6 admission / eviction / staging / aging: the GPU-resident
// hot-row cache (mirror of embserve cache.py:114-352 AdaptiveCache +
// FrequencySketch).
//
// Semantics kept bit-exact with the reference under the canonical order
// (SURVEY §8(c)):
//  * LRU order == ascending last_tick; every probe advances the tick, a hit's
//    last_tick = tick0 + (ordinal of its LAST occurrence in the batch) + 1
//    (cache.py:189-202);
//  * a miss bumps the exact decayed-frequency sketch by 1.0 per occurrence
//    (cache.py:194-197), i.e. by the key's miss multiplicity;
//  * offers are processed strictly in order: sketch admission compares the
//    candidate against the CURRENT LRU victim, inserts evict LRU until the
//    byte budget fits and take a fresh tick (cache.py:237-280);
//  * stage_hot_admissions ranks ALL sketch keys by (-count, key), takes the
//    top `limit`, skips cached/pending keys and keys that do not fit the spare
//    room (cache.py:311-342); apply_pending inserts them in order;
//  * age halves every count and drops counts < prune (cache.py:128-136).
// The order-dependent steps run as one sequential device thread over
// precomputed, parallel-gathered inputs (sketch estimates, LRU order); the
// hash-index and row-copy side effects are applied afterwards in parallel.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fx_cache.cuh"

namespace fx {

// ---------------------------------------------------------------- init
__global__ void k_cache_init(CacheView c) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t i = i0; i < c.hcap; i += stride) c.hkeys[i] = kEmpty;
  for (int64_t i = i0; i < c.kcap; i += stride) {
    c.kkeys[i] = kEmpty;
    c.kval[i] = 0.0;
    c.kflag[i] = 0;
  }
  for (int64_t i = i0; i < c.scap; i += stride) {
    c.stick[i] = kFree;
    c.skey[i] = kEmpty;
    c.skey2[i] = 0;
    c.free_stack[i] = static_cast<int32_t>(c.scap - 1 - i);  // pops give 0, 1, 2, ...
  }
}

// ---------------------------------------------------------------- K3 probe
__global__ void __launch_bounds__(256) k_probe(CacheView c, const uint64_t *__restrict__ uniq,
                                               const int32_t *__restrict__ mult,
                                               const int64_t *__restrict__ last_ord, const int64_t *n_ptr,
                                               int64_t n_host, int32_t *slot_out) {
  const int64_t n = n_ptr ? *n_ptr : n_host;
  const long long tick0 = c.sc->tick;
  long long hits = 0, misses = 0, born = 0;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = uniq[u];
    const int32_t m = mult[u];
    const int32_t s = h_find(c, key);
    if (s >= 0) {
      c.stick[s] = tick0 + last_ord[u] + 1;
      c.shits[s] += m;
      hits += m;
    } else {
      born += k_add(c, key, static_cast<double>(m)) ? 1 : 0;
      misses += m;
    }
    if (slot_out) slot_out[u] = s;
  }
  // warp-aggregate the counters
  for (int o = 16; o; o >>= 1) {
    hits += __shfl_down_sync(0xffffffffu, hits, o);
    misses += __shfl_down_sync(0xffffffffu, misses, o);
    born += __shfl_down_sync(0xffffffffu, born, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (hits) atomicAdd(reinterpret_cast<unsigned long long *>(&c.sc->hits), (unsigned long long)hits);
    if (misses) atomicAdd(reinterpret_cast<unsigned long long *>(&c.sc->misses), (unsigned long long)misses);
    if (born) atomicAdd(reinterpret_cast<unsigned long long *>(&c.sc->sketch_live), (unsigned long long)born);
  }
}

__global__ void k_advance_tick(Scalars *sc, long long nnz) { sc->tick += nnz; }

// ---------------------------------------------------------------- offers
struct OfferWS {
  double *est_cand;
  int32_t *size_cand;
  uint8_t *present;
  int32_t *lru_slot;   // sorted occupied slots (ascending tick)
  double *est_vic;
  int32_t *acc_slot;
  int32_t *acc_j;
  uint64_t *ev_keys;
  long long *sort_keys_in;
  long long *sort_keys_out;
  int32_t *iota;
  int32_t *par_flag;
  int32_t *par_iota;
  int32_t *par_cand;
  int64_t *par_m;
  double *est_cc;      // est_cand in compacted candidate order (contiguous tile loads)
  long long *pstate;   // decide -> apply hand-off (see k_offer_par)
  long long lru_valid; // lru_slot[0, lru_valid) holds the LRU-ordered prefix
};

__global__ void k_offer_prep(CacheView c, const uint64_t *keys, int64_t n, const int32_t *sizes, OfferWS w) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = keys[j];
    w.est_cand[j] = k_est(c, key);
    w.size_cand[j] = sizes ? sizes[j] : table_bytes_of(c, key);
    w.present[j] = h_find(c, key) >= 0 ? 1 : 0;
  }
}

// LRU sort keys: ticks, free slots mapped to free_key (> every live tick) so
// the radix sort only needs the low lru_bits(tick) bits.
__global__ void k_lru_keys(CacheView c, OfferWS w, long long free_key) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.scap; i += (int64_t)gridDim.x * blockDim.x) {
    const long long t = c.stick[i];
    w.sort_keys_in[i] = t == kFree ? free_key : t;
    w.iota[i] = static_cast<int32_t>(i);
  }
}

// partial LRU order: histogram of the live ticks' top bits, then only the
// slots in the oldest bins (a superset of the `need` oldest) are sorted
__global__ void k_lru_hist(CacheView c, int shift, int32_t *hist) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); i0 < c.scap; i0 += stride) {
    const int64_t i = i0 + lane;
    int bin = -1;
    if (i < c.scap) {
      const long long t = c.stick[i];
      if (t != kFree) bin = static_cast<int>(t >> shift);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, bin);
    if (bin >= 0 && lane == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
  }
}

__global__ void k_lru_collect(CacheView c, int shift, int32_t max_bin, OfferWS w, unsigned long long *count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.scap; i += (int64_t)gridDim.x * blockDim.x) {
    const long long t = c.stick[i];
    if (t == kFree || (t >> shift) > max_bin) continue;
    const unsigned long long p = atomicAdd(count, 1ull);
    w.sort_keys_in[p] = t;
    w.iota[p] = static_cast<int32_t>(i);
  }
}

__global__ void k_vic_prep(CacheView c, OfferWS w, int64_t k) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
    w.est_vic[i] = k_est(c, c.skey[w.lru_slot[i]]);
}

// mode 0: offer (admission policy); mode 1: apply pending (always admit,
// skip present keys); n == 0 with used > budget: evict to budget (shrink).
__global__ void k_offer_seq(CacheView c, const uint64_t *keys, int64_t n, int32_t mode, OfferWS w, int64_t k_vic,
                            uint8_t *accepted, int32_t record) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Scalars *sc = c.sc;
  long long used = sc->used, budget = sc->budget, tick = sc->tick, entries = sc->entries, ftop = sc->free_top;
  const long long e0 = entries;
  long long h = 0, n_acc = 0, n_ev = 0, n_log = sc->n_evlog;
  auto head_slot = [&](long long q) -> int32_t { return q < e0 ? w.lru_slot[q] : w.acc_slot[q - e0]; };
  auto evict_head = [&]() {
    const int32_t s = head_slot(h);
    ++h;
    used -= c.ssize[s];
    const uint64_t k = c.skey[s];
    w.ev_keys[n_ev++] = k;
    if (record && n_log < c.evlog_cap) c.evlog[n_log] = k;
    if (record) ++n_log;
    c.stick[s] = kFree;
    c.skey[s] = kEmpty;
    c.free_stack[ftop++] = s;
    --entries;
  };
  long long err = 0;
  while (used > budget && entries > 0) evict_head();  // resize shrink (cache.py:270-274)
  if (used > budget) err = 1;  // only leaked pooled bytes left: the reference's popitem raises
  for (int64_t j = 0; j < n; ++j) {
    const uint64_t key = keys[j];
    const int32_t size = w.size_cand[j];
    if (w.present[j]) {  // already cached: offer -> True; apply -> skip
      if (accepted) accepted[j] = mode == 0 ? 1 : 0;
      continue;
    }
    if (size < 0 || size > budget) {
      if (accepted) accepted[j] = 0;
      continue;
    }
    if (mode == 0 && c.admission == 0 && used + size > budget && entries > 0) {
      const double ve = h < k_vic ? w.est_vic[h] : (h < e0 ? k_est(c, c.skey[w.lru_slot[h]])
                                                            : w.est_cand[w.acc_j[h - e0]]);
      if (w.est_cand[j] < ve) {
        if (accepted) accepted[j] = 0;
        continue;
      }
    }
    while (used + size > budget && entries > 0) evict_head();
    if (used + size > budget) {  // queue exhausted (leaked pooled bytes): reference KeyError
      err = 1;
      if (accepted) accepted[j] = 0;
      break;
    }
    ++tick;
    const int32_t s = c.free_stack[--ftop];
    c.skey[s] = key;
    c.stick[s] = tick;
    c.ssize[s] = size;
    c.shits[s] = 0;
    w.acc_slot[n_acc] = s;
    w.acc_j[n_acc] = static_cast<int32_t>(j);
    ++n_acc;
    used += size;
    ++entries;
    if (accepted) accepted[j] = 1;
  }
  sc->used = used;
  sc->tick = tick;
  sc->entries = entries;
  sc->free_top = ftop;
  sc->n_acc = n_acc;
  sc->n_ev = n_ev;
  sc->n_evlog = n_log;
  if (err) sc->err = err;
}


// ---------------------------------------------------------------- parallel ordered offers
// Exact parallel form of k_offer_seq when every candidate and every cached
// entry has the same size S (uniform dims). With cap = budget / S slots:
//  * the first (cap - entries) non-present candidates are inserted without
//    eviction (used + S <= budget, cache.py:250 is not reached);
//  * afterwards every accept evicts exactly one LRU entry. The LRU queue is
//    V = [existing entries by tick] ++ [accepted candidates in order]; with
//    head h, candidate j is accepted iff est(c_j) >= est(V[h]) (sketch) or
//    always ("always" admission / apply-pending).
// Decisions come in runs. Accept-run from (j, h): c_{j+t} is accepted iff
// est(c_{j+t}) >= est(V[h+t]) for all earlier t; reject-run from (j, h):
// c_{j+t} is rejected iff est(c_{j+t}) < est(V[h]). A tile of at most
// min(OFFER_TILE, cap) candidates (so V[h+t] never refers to a candidate
// accepted inside the same tile) is applied at once when it is a single run,
// otherwise warp 0 peels it run by run 32 candidates at a time. Ticks, slots
// and evictions are then assigned in parallel (k_offer_apply_*) exactly as
// the sequential loop would.
struct ParWS {
  const int32_t *cand;   // compacted non-present candidate positions (ascending)
  int64_t m;             // number of compacted candidates
  const int64_t *m_dev;  // optional device count (overrides m)
};

__device__ __forceinline__ double est_v(const CacheView &c, const OfferWS &w, long long k, long long e0,
                                        long long k_vic) {
  if (k < e0) {
    if (k < k_vic) return w.est_vic[k];
    return k < w.lru_valid ? k_est(c, c.skey[w.lru_slot[k]]) : 0.0;  // beyond: padding, never a victim
  }
  return w.est_cand[w.acc_j[k - e0]];
}

__global__ void k_est_compact(const OfferWS w, ParWS pw) {
  const long long m = pw.m_dev ? *pw.m_dev : pw.m;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
    w.est_cc[t] = w.est_cand[pw.cand[t]];
}

constexpr int OFFER_TILE = 4096;  // candidates per resolver tile (dynamic shared memory)
constexpr size_t OFFER_SMEM = (2 * OFFER_TILE + 32) * sizeof(double) + 2 * OFFER_TILE * sizeof(int);

// pstate layout (written by k_offer_par, read by k_offer_apply)
enum { PS_E0 = 0, PS_H0, PS_NF, PS_N2, PS_TICK0, PS_LOG0, PS_EV0, PS_VALID };

// Decisions only: phases 0/1 and the phase-2 accept/reject sequence. The
// evictions and installs of phase-2 accepts are applied afterwards by
// k_offer_apply, in parallel over the accept ranks, so each tile costs one
// contiguous load of candidate / victim estimates plus the shared-memory
// resolution.
__global__ void __launch_bounds__(1024) k_offer_par(CacheView c, const uint64_t *keys, int32_t mode, OfferWS w,
                                                    ParWS pw, int64_t k_vic, int32_t S, uint8_t *accepted,
                                                    int32_t record) {
  __shared__ long long st[8];  // j, h, n_acc, n_ev, tick, ftop, n_log, entries
  const int tid = threadIdx.x;
  Scalars *sc = c.sc;
  const long long m = pw.m_dev ? *pw.m_dev : pw.m;
  const long long e0 = sc->entries;
  // bytes leaked by in-place pooled re-puts (cache.py:256-263 adds the size
  // again without a new entry) occupy budget units that no eviction frees
  const long long ph = sc->used / S > e0 ? sc->used / S - e0 : 0;
  long long cap = sc->budget / S - ph;
  if (cap < 0) {
    cap = 0;
    if (tid == 0) sc->err = 1;
  }
  if (tid == 0) {
    st[0] = 0; st[1] = 0; st[2] = 0; st[3] = 0;
    st[4] = sc->tick; st[5] = sc->free_top; st[6] = sc->n_evlog; st[7] = e0;
    w.pstate[PS_VALID] = 0;
  }
  __syncthreads();
  // phase 0: entries beyond cap (budget shrank): evict LRU heads
  {
    const long long over = e0 > cap ? e0 - cap : 0;
    for (long long k = tid; k < over; k += blockDim.x) {
      const int32_t vs = w.lru_slot[k];
      const uint64_t key = c.skey[vs];
      w.ev_keys[k] = key;
      if (record && st[6] + k < c.evlog_cap) c.evlog[st[6] + k] = key;
      c.stick[vs] = kFree;
      c.skey[vs] = kEmpty;
      c.free_stack[st[5] + k] = vs;
    }
    __syncthreads();
    if (tid == 0 && over) {
      st[1] = over; st[3] = over; st[5] += over; st[6] += record ? over : 0; st[7] = cap;
    }
    __syncthreads();
  }
  if (S > sc->budget) {  // every candidate is larger than the whole budget
    for (long long t = tid; t < m; t += blockDim.x) if (accepted) accepted[pw.cand[t]] = 0;
    __syncthreads();
    if (tid == 0) {
      sc->entries = st[7]; sc->used = (st[7] + ph) * S; sc->free_top = st[5];
      sc->n_acc = 0; sc->n_ev = st[3]; sc->n_evlog = st[6];
    }
    return;
  }
  // phase 1: free slots, no eviction
  {
    const long long fr = cap - st[7];
    const long long nf = fr < m ? (fr > 0 ? fr : 0) : m;
    for (long long t = tid; t < nf; t += blockDim.x) {
      const int32_t j = pw.cand[t];
      const int32_t s = c.free_stack[st[5] - 1 - t];
      c.skey[s] = keys[j];
      c.stick[s] = st[4] + t + 1;
      c.ssize[s] = S;
      c.shits[s] = 0;
      w.acc_slot[t] = s;
      w.acc_j[t] = j;
      if (accepted) accepted[j] = 1;
    }
    __syncthreads();
    if (tid == 0) {
      st[0] = nf; st[2] = nf; st[4] += nf; st[5] -= nf; st[7] += nf;
    }
    __syncthreads();
  }
  if (cap == 0 && st[0] < m && tid == 0) sc->err = 1;  // nothing left to evict: reference KeyError
  // phase 2 (full cache): every accept evicts the queue head V[h]. Only the
  // decisions are taken here; acc_j[n_acc + r] = candidate of accept rank r.
  const long long j0 = st[0], h0 = st[1], nacc0 = st[2];
  const bool always = (mode != 0) || (c.admission != 0);
  if (always) {
    for (long long t = j0 + tid; t < m; t += blockDim.x) {
      const int32_t jj = pw.cand[t];
      w.acc_j[nacc0 + (t - j0)] = jj;
      if (accepted) accepted[jj] = 1;
    }
    __syncthreads();
    if (tid == 0 && cap > 0) { st[2] += m - j0; st[0] = m; }
    __syncthreads();
  } else {
    // sketch admission: tiles of T <= min(OFFER_TILE, cap) candidates; a tile
    // that is one accept- or reject-run is applied at once, otherwise warp 0
    // peels it run by run, 32 candidates at a time (see below).
    extern __shared__ __align__(16) unsigned char offer_smem[];
    double *s_ec = reinterpret_cast<double *>(offer_smem);
    double *s_ev = s_ec + OFFER_TILE;
    int *s_acc = reinterpret_cast<int *>(s_ev + OFFER_TILE + 32);
    int *s_rank = s_acc + OFFER_TILE;
    __shared__ int s_chunk_a;
    __shared__ int s_ffa, s_ffr;
    const long long tmax = cap < OFFER_TILE ? cap : OFFER_TILE;
    while (tmax > 0 && st[0] < m) {
      const long long j = st[0], h = st[1], nacc = st[2];
      const int T = static_cast<int>((m - j) < tmax ? (m - j) : tmax);
      for (int t = tid; t < T; t += blockDim.x) s_ec[t] = w.est_cc[j + t];
      for (int t = tid; t < T + 32; t += blockDim.x) s_ev[t] = t < cap ? est_v(c, w, h + t, e0, k_vic) : 0.0;
      if (tid == 0) { s_ffa = T; s_ffr = T; }
      __syncthreads();
      // run detection: accept-run (c_t >= V[h+t]) or reject-run (c_t < V[h])
      for (int t = tid; t < T; t += blockDim.x) {
        if (!(s_ec[t] >= s_ev[t])) atomicMin(&s_ffa, t);
        if (!(s_ec[t] < s_ev[0])) atomicMin(&s_ffr, t);
      }
      __syncthreads();
      const int ffa = s_ffa, ffr = s_ffr;
      const bool bulk = ffa == T || ffr == T;  // whole tile one run; otherwise peel every chunk
      if (tid == 0) {
        if (bulk) sc->tiles_bulk += 1; else sc->tiles_chain += 1;
      }
      if (bulk) {
        // long run: decisions are the prefix run, no chain needed
        const bool acc_run = ffa >= ffr;
        const int run = acc_run ? ffa : ffr;
        for (int t = tid; t < T; t += blockDim.x) {
          s_acc[t] = (t < run && acc_run) ? 1 : 0;
          s_rank[t] = t;
        }
        if (tid == 0) {
          s_chunk_a = acc_run ? run : 0;
          s_ffr = run;  // decisions resolved in this tile
        }
      } else if (tid < 32) {
        // Run peeling per 32-candidate chunk: from the first unresolved
        // candidate u0 (queue offset a0), an accept-run lasts while
        // c_{u0+t} >= V[h + a0 + t] and a reject-run while c_{u0+t} < V[h + a0];
        // the candidate at u0 always starts one of them, so every step
        // resolves >= 1 decision with two ballots (no per-decision chain).
        int a0 = 0;  // accepts so far in this tile
        for (int c0 = 0; c0 < T; c0 += 32) {
          const int q = c0 + tid;
          const int nq = (T - c0) < 32 ? (T - c0) : 32;
          const double ec = q < T ? s_ec[q] : 0.0;
          int u0 = 0;
          while (u0 < nq) {
            const bool mine = tid >= u0 && tid < nq;
            const unsigned fa = __ballot_sync(0xffffffffu, mine && !(ec >= s_ev[a0 + (tid - u0)]));
            const int end_a = fa ? __ffs(fa) - 1 : nq;  // accept-run [u0, end_a)
            if (end_a > u0) {
              if (mine && tid < end_a) {
                s_acc[q] = 1;
                s_rank[q] = a0 + (tid - u0);
              }
              a0 += end_a - u0;
              u0 = end_a;
              continue;
            }
            const unsigned fr = __ballot_sync(0xffffffffu, mine && !(ec < s_ev[a0]));
            const int end_r = fr ? __ffs(fr) - 1 : nq;  // reject-run [u0, end_r)
            if (mine && tid < end_r) {
              s_acc[q] = 0;
              s_rank[q] = a0;
            }
            u0 = end_r;
          }
        }
        __syncwarp();
        if (tid == 0) {
          s_chunk_a = a0;
          s_ffr = T;
        }
      }
      __syncthreads();
      const int na = s_chunk_a;
      const int R = s_ffr;  // decisions resolved in this tile (bulk run or the whole tile)
      for (int t = tid; t < R; t += blockDim.x) {
        const int32_t jj = pw.cand[j + t];
        if (s_acc[t]) w.acc_j[nacc + s_rank[t]] = jj;
        if (accepted) accepted[jj] = s_acc[t] ? 1 : 0;
      }
      __syncthreads();  // acc_j of this tile visible to the next tile's victim estimates
      if (tid == 0) {
        st[0] += R; st[1] += na; st[2] += na;
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    const long long n2 = st[2] - nacc0;  // phase-2 accepts, each evicting one queue head
    w.pstate[PS_E0] = e0;
    w.pstate[PS_H0] = h0;
    w.pstate[PS_NF] = nacc0;
    w.pstate[PS_N2] = n2;
    w.pstate[PS_TICK0] = st[4];  // tick after phase 1
    w.pstate[PS_LOG0] = st[6];
    w.pstate[PS_EV0] = st[3];
    w.pstate[PS_VALID] = 1;
    sc->tick = st[4] + n2;
    sc->free_top = st[5];
    sc->entries = st[7];
    sc->used = (st[7] + ph) * S;
    sc->n_acc = st[2];
    sc->n_ev = st[3] + n2;
    sc->n_evlog = st[6] + (record ? n2 : 0);
  }
}

// Side effects of the phase-2 accepts, in parallel over accept ranks r:
// accept r evicts queue position k = h0 + r of V = [existing entries by LRU]
// ++ [accepted candidates in order] and takes its slot with tick tick0+r+1.
// Victims at k >= e0 are candidates accepted earlier in the same call; their
// slot is followed back to the entry (or free slot) they took. Only the
// final occupant of a slot writes it (an accept evicted again later in the
// call leaves its slot to the accept that evicted it).
__device__ __forceinline__ int32_t apply_slot(const OfferWS &w, long long k, long long e0, long long h0,
                                              long long nf) {
  // slot that queue position k occupies
  while (k >= e0) {
    const long long i = k - e0;  // index in the accepted list
    if (i < nf) return w.acc_slot[i];
    k = h0 + (i - nf);           // phase-2 accept: the slot of its own victim
  }
  return w.lru_slot[k];
}

__global__ void k_offer_apply_keys(CacheView c, const uint64_t *keys, OfferWS w, int32_t record) {
  if (!w.pstate[PS_VALID]) return;
  const long long e0 = w.pstate[PS_E0], h0 = w.pstate[PS_H0], nf = w.pstate[PS_NF], n2 = w.pstate[PS_N2];
  const long long log0 = w.pstate[PS_LOG0], ev0 = w.pstate[PS_EV0];
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n2;
       r += (long long)gridDim.x * blockDim.x) {
    const long long k = h0 + r;
    const uint64_t key = k < e0 ? c.skey[w.lru_slot[k]] : keys[w.acc_j[k - e0]];
    w.ev_keys[ev0 + r] = key;
    if (record && log0 + r < c.evlog_cap) c.evlog[log0 + r] = key;
    w.acc_slot[nf + r] = apply_slot(w, k, e0, h0, nf);
  }
}

__global__ void k_offer_apply_slots(CacheView c, const uint64_t *keys, OfferWS w, int32_t S) {
  if (!w.pstate[PS_VALID]) return;
  const long long e0 = w.pstate[PS_E0], h0 = w.pstate[PS_H0], nf = w.pstate[PS_NF], n2 = w.pstate[PS_N2];
  const long long tick0 = w.pstate[PS_TICK0];
  const long long hend = h0 + n2;  // final queue head
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n2;
       r += (long long)gridDim.x * blockDim.x) {
    if (e0 + nf + r < hend) continue;  // evicted again within this call
    const int32_t s = w.acc_slot[nf + r];
    c.skey[s] = keys[w.acc_j[nf + r]];
    c.stick[s] = tick0 + r + 1;
    c.ssize[s] = S;
    c.shits[s] = 0;
  }
  // phase-1 entries evicted within the call: their slot now belongs to a phase-2 accept
}

__global__ void k_mark_absent(const uint8_t *present, int64_t n, int32_t *flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = present[i] ? 0 : 1;
}

__global__ void k_present_accept(const uint8_t *present, int64_t n, int32_t mode, uint8_t *accepted) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (present[i] && accepted) accepted[i] = mode == 0 ? 1 : 0;
}

__global__ void k_iota32(int32_t *p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = static_cast<int32_t>(i);
}

__global__ void k_hash_erase(CacheView c, OfferWS w) {
  const long long n = c.sc->n_ev;
  long long t = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    t += h_erase(c, w.ev_keys[i]) ? 1 : 0;
  if (t) atomicAdd(reinterpret_cast<unsigned long long *>(&c.sc->hash_tomb), (unsigned long long)t);
}

// one warp per accepted entry: index it and copy its row into the slot
__global__ void __launch_bounds__(256) k_install(CacheView c, OfferWS w, const uint64_t *keys,
                                                 const float *const *src_rows) {
  const long long n = c.sc->n_acc;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t a = warp; a < n; a += nw) {
    const int32_t s = w.acc_slot[a];
    const int32_t j = w.acc_j[a];
    const uint64_t key = keys[j];
    if (c.skey[s] != key || c.stick[s] == kFree) continue;  // evicted again later in the same call
    if (lane == 0) h_insert(c, key, s);
    int32_t dim = c.ssize[s] / 4;
    const float *src = src_rows ? src_rows[j] : nullptr;
    if (!src) src = dir_row(c, key, &dim);
    float *dst = c.rows + static_cast<int64_t>(s) * c.row_ld;
    if (src)
      for (int i = lane; i < dim; i += 32) dst[i] = src[i];
  }
}

// ---------------------------------------------------------------- pooled-result keyspace
// (cache.py:204-223, ranker.py:243-249,412-414). Keys are the bag
// fingerprints of fx_bag_fingerprint: A (top bit set) indexes the shared
// hash/LRU/budget, B is verified per slot.

__global__ void k_pooled_find(CacheView c, const uint64_t *key_a, const uint64_t *key_b, int64_t n,
                              int32_t *slot_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t s = h_find(c, key_a[i]);
    if (s >= 0 && c.skey2[s] != key_b[i]) {  // same A, different multiset
      atomicExch(reinterpret_cast<unsigned long long *>(&c.sc->err), 2ull);
      s = -1;
    }
    slot_out[i] = s;
  }
}

// pooled_get hits: last_tick = tick0 + pos + 1 (latest probe of the entry in
// this batch), entry.hits += 1 per probe; the tick itself advances with the
// batch's row probes (fx_cache_probe / fx_cache_advance_tick).
__global__ void k_pooled_touch(CacheView c, const int32_t *slot, const int64_t *pos, int64_t n) {
  const long long tick0 = c.sc->tick;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = slot[i];
    if (s < 0) continue;
    atomicMax(&c.stick[s], tick0 + pos[i] + 1);
    atomicAdd(&c.shits[s], 1);
  }
}

// one warp per item: copy the row of slot[i] (if >= 0) into out[i]
__global__ void k_read_slots(CacheView c, const int32_t *slot, int64_t n, float *out, int32_t out_ld,
                             int32_t *size_out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    const int32_t s = slot[i];
    if (size_out && lane == 0) size_out[i] = s < 0 ? 0 : c.ssize[s];
    if (s < 0) continue;
    const int32_t dim = c.ssize[s] / 4;
    const float *src = c.rows + static_cast<int64_t>(s) * c.row_ld;
    for (int k = lane; k < dim && k < out_ld; k += 32) out[i * out_ld + k] = src[k];
  }
}

struct PutWS {
  int32_t *present_slot;  // slot of key j at call start (-1 absent)
  int32_t *prev;          // previous put of the same key in this call (-1 none)
  int32_t *slot_of;       // slot holding key j right after put j (-1 skipped)
  int32_t *iota;
  int32_t *perm;
  uint64_t *keys_sorted;
  int32_t *ov_slot;       // in-place re-puts (slot, j)
  int32_t *ov_j;
  int32_t *writer;        // [slots] last put that wrote the slot (valid for recorded slots)
  // parallel path (uniform sizes)
  int32_t *run_in;        // sorted position if it starts a key run, else 0
  int32_t *run_start;     // inclusive max-scan of run_in
  int32_t *first;         // first put of j's key in this call
  int32_t *lastj;         // [first put] last put of that key (its vector wins)
  int32_t *fresh;         // 1 for the first put of a key
  int32_t *rank;          // exclusive prefix of fresh
  int32_t *fail;          // device flag: parallel preconditions violated -> sequential loop
};

__global__ void k_put_prep(CacheView c, const uint64_t *key_a, const uint64_t *key_b, int64_t n,
                           const int32_t *sizes, int32_t uniform_size, OfferWS w, PutWS pw) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    int32_t s = h_find(c, key_a[j]);
    if (s >= 0 && c.skey2[s] != key_b[j]) {
      atomicExch(reinterpret_cast<unsigned long long *>(&c.sc->err), 2ull);
      s = -1;
    }
    pw.present_slot[j] = s;
    w.size_cand[j] = sizes ? sizes[j] : uniform_size;
    pw.iota[j] = static_cast<int32_t>(j);
  }
}

// after a stable sort of (key_a, j): prev[j] = the previous put of the same key
__global__ void k_put_prev(const uint64_t *keys_sorted, const int32_t *perm, int64_t n, const uint64_t *key_b,
                           PutWS pw, Scalars *sc) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = perm[p];
    int32_t pv = -1;
    if (p > 0 && keys_sorted[p - 1] == keys_sorted[p]) {
      pv = perm[p - 1];
      if (key_b[pv] != key_b[j]) atomicExch(reinterpret_cast<unsigned long long *>(&sc->err), 2ull);
    }
    pw.prev[j] = pv;
  }
}

__global__ void k_put_heads(const uint64_t *keys_sorted, int64_t n, PutWS pw) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    pw.run_in[p] = (p == 0 || keys_sorted[p - 1] != keys_sorted[p]) ? static_cast<int32_t>(p) : 0;
}

__global__ void k_put_links(const uint64_t *keys_sorted, int64_t n, PutWS pw) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = pw.perm[p];
    const int32_t f = pw.perm[pw.run_start[p]];
    pw.first[j] = f;
    pw.fresh[j] = (f == j) ? 1 : 0;
    if (p == n - 1 || keys_sorted[p + 1] != keys_sorted[p]) pw.lastj[f] = j;
  }
}

// Parallel form of k_put_seq for one entry size S (uniform dims). With
// units0 = used / S (entries + leaked units), cap = budget / S and e0 live
// entries, put i (0-based) leaves ev(i) = max(0, units0 + i + 1 - cap)
// evictions behind it, taken from the queue V = [entries by LRU] ++ [first
// puts of each key, in order]. If every re-put finds its key still resident
// (queue position e0 + rank(first) >= ev(i)), no key was resident at call
// start and the queue never runs dry, the loop's outcome is closed-form:
// V[0, E) evicted (E = ev(n-1)), surviving first puts installed with tick
// tick0 + i + 1 and the vector of their key's last put, used = (units0 + n -
// E) * S. Otherwise `fail` is raised and k_put_seq runs instead.
__global__ void k_putp_verify(CacheView c, int64_t n, int32_t S, PutWS pw) {
  const Scalars *sc = c.sc;
  const long long units0 = sc->used / S, cap = sc->budget / S, e0 = sc->entries;
  bool bad = (sc->used % S) != 0 || S > sc->budget;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n && !bad;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (pw.present_slot[i] >= 0) bad = true;
    const long long ev = units0 + i + 1 - cap > 0 ? units0 + i + 1 - cap : 0;
    if (ev > e0 + pw.rank[i]) bad = true;
    if (!pw.fresh[i] && e0 + pw.rank[pw.first[i]] < ev) bad = true;
  }
  if (bad) atomicExch(pw.fail, 1);
}

__global__ void k_putp_evict(CacheView c, int64_t n, int32_t S, OfferWS w, PutWS pw, int32_t record) {
  if (*pw.fail) return;
  const Scalars *sc = c.sc;
  const long long units0 = sc->used / S, cap = sc->budget / S, e0 = sc->entries;
  const long long E = units0 + n - cap > 0 ? units0 + n - cap : 0;
  const long long ee = E < e0 ? E : e0;
  const long long ftop = sc->free_top, log0 = sc->n_evlog;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ee; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = w.lru_slot[k];
    const uint64_t key = c.skey[s];
    w.ev_keys[k] = key;
    if (record && log0 + k < c.evlog_cap) c.evlog[log0 + k] = key;
    c.stick[s] = kFree;
    c.skey[s] = kEmpty;
    c.free_stack[ftop + k] = s;
  }
}

__global__ void k_putp_insert(CacheView c, const uint64_t *key_a, const uint64_t *key_b, int64_t n, int32_t S,
                              OfferWS w, PutWS pw, int32_t record) {
  if (*pw.fail) return;
  const Scalars *sc = c.sc;
  const long long units0 = sc->used / S, cap = sc->budget / S, e0 = sc->entries;
  const long long E = units0 + n - cap > 0 ? units0 + n - cap : 0;
  const long long ee = E < e0 ? E : e0, fe = E - ee;  // evicted entries / evicted first puts
  const long long ftop = sc->free_top + ee, log0 = sc->n_evlog, tick0 = sc->tick;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    if (!pw.fresh[j]) continue;
    const long long r = pw.rank[j];
    if (r < fe) {  // inserted and evicted again within the call
      w.ev_keys[e0 + r] = key_a[j];
      if (record && log0 + e0 + r < c.evlog_cap) c.evlog[log0 + e0 + r] = key_a[j];
      continue;
    }
    const long long u = r - fe;
    const int32_t s = c.free_stack[ftop - 1 - u];
    const int32_t lj = pw.lastj[j];
    c.skey[s] = key_a[j];
    c.skey2[s] = key_b[j];
    c.stick[s] = tick0 + j + 1;
    c.ssize[s] = S;
    c.shits[s] = 0;
    pw.writer[s] = lj;
    w.acc_slot[u] = s;
    w.acc_j[u] = lj;
  }
}

__global__ void k_putp_finish(CacheView c, int64_t n, int32_t S, PutWS pw, int32_t record) {
  if (*pw.fail) return;
  Scalars *sc = c.sc;
  const long long units0 = sc->used / S, cap = sc->budget / S, e0 = sc->entries;
  const long long E = units0 + n - cap > 0 ? units0 + n - cap : 0;
  const long long ee = E < e0 ? E : e0, fe = E - ee;
  const long long F = pw.rank[n - 1] + pw.fresh[n - 1];
  const long long inst = F - fe;
  sc->used = (units0 + n - E) * S;
  sc->tick += n;
  sc->entries = e0 - ee + inst;
  sc->free_top = sc->free_top + ee - inst;
  sc->n_acc = inst;
  sc->n_ov = 0;
  sc->n_ev = E;
  if (record) sc->n_evlog += E;
  sc->n_par_puts += 1;
}

// Ordered pooled_put loop (cache.py:219-223 -> _insert, cache.py:256-268):
// no admission test; evict LRU until the size fits, take a tick, insert at
// MRU. A key that is still resident (put twice in one batch, or re-put
// through the API) is replaced IN PLACE by the reference's OrderedDict
// assignment: its LRU position is kept, hits restart at 0 and used_bytes
// grows by the size again without a new entry (the bytes are never freed).
__global__ void k_put_seq(CacheView c, const uint64_t *key_a, const uint64_t *key_b, int64_t n, OfferWS w,
                          PutWS pw, int32_t record, int32_t only_on_fail) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (only_on_fail && *pw.fail == 0) return;
  Scalars *sc = c.sc;
  long long used = sc->used, budget = sc->budget, tick = sc->tick, entries = sc->entries, ftop = sc->free_top;
  const long long e0 = entries;
  long long h = 0, n_acc = 0, n_ov = 0, n_ev = 0, n_log = sc->n_evlog, err = 0;
  auto head_slot = [&](long long q) -> int32_t { return q < e0 ? w.lru_slot[q] : w.acc_slot[q - e0]; };
  for (int64_t j = 0; j < n; ++j) {
    const uint64_t key = key_a[j];
    const int32_t size = w.size_cand[j];
    if (size < 0 || size > budget) {  // _insert: size > budget -> False, no tick
      pw.slot_of[j] = -1;
      continue;
    }
    const int32_t pv = pw.prev[j];
    const int32_t live = pv >= 0 ? pw.slot_of[pv] : pw.present_slot[j];
    while (used + size > budget && h < e0 + n_acc) {
      const int32_t s = head_slot(h);
      ++h;
      used -= c.ssize[s];
      const uint64_t k = c.skey[s];
      w.ev_keys[n_ev++] = k;
      if (record && n_log < c.evlog_cap) c.evlog[n_log] = k;
      if (record) ++n_log;
      c.stick[s] = kFree;
      c.skey[s] = kEmpty;
      c.free_stack[ftop++] = s;
      --entries;
    }
    if (used + size > budget) {  // queue exhausted: the reference's popitem raises KeyError
      err = 1;
      break;
    }
    ++tick;
    if (live >= 0 && c.skey[live] == key) {  // still resident: replace in place
      c.shits[live] = 0;
      c.ssize[live] = size;
      pw.writer[live] = static_cast<int32_t>(j);
      pw.ov_slot[n_ov] = live;
      pw.ov_j[n_ov] = static_cast<int32_t>(j);
      ++n_ov;
      used += size;
      pw.slot_of[j] = live;
      continue;
    }
    const int32_t s = c.free_stack[--ftop];
    c.skey[s] = key;
    c.skey2[s] = key_b[j];
    c.stick[s] = tick;
    c.ssize[s] = size;
    c.shits[s] = 0;
    pw.writer[s] = static_cast<int32_t>(j);
    w.acc_slot[n_acc] = s;
    w.acc_j[n_acc] = static_cast<int32_t>(j);
    ++n_acc;
    used += size;
    ++entries;
    pw.slot_of[j] = s;
  }
  sc->used = used;
  sc->tick = tick;
  sc->entries = entries;
  sc->free_top = ftop;
  sc->n_acc = n_acc;
  sc->n_ov = n_ov;
  sc->n_ev = n_ev;
  sc->n_evlog = n_log;
  if (err) sc->err = err;
}

// one warp per recorded put (fresh inserts, then in-place re-puts): index it
// and copy its vector, unless evicted again or overwritten by a later put
__global__ void __launch_bounds__(256) k_install_put(CacheView c, OfferWS w, PutWS pw, const uint64_t *key_a,
                                                     const uint64_t *key_b, const float *const *src_rows) {
  const long long na = c.sc->n_acc, no = c.sc->n_ov;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t a = warp; a < na + no; a += nw) {
    const int32_t s = a < na ? w.acc_slot[a] : pw.ov_slot[a - na];
    const int32_t j = a < na ? w.acc_j[a] : pw.ov_j[a - na];
    const uint64_t key = key_a[j];
    if (c.skey[s] != key || c.stick[s] == kFree || pw.writer[s] != j) continue;
    if (lane == 0) {
      h_insert(c, key, s);
      c.skey2[s] = key_b[j];
    }
    const int32_t dim = c.ssize[s] / 4;
    const float *src = src_rows[j];
    float *dst = c.rows + static_cast<int64_t>(s) * c.row_ld;
    if (src)
      for (int i = lane; i < dim; i += 32) dst[i] = src[i];
  }
}

// ---------------------------------------------------------------- staging
__global__ void k_sketch_collect(CacheView c, uint64_t *out_keys, long long *out_vbits, int32_t *out_pos,
                                 long long *count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.kcap; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = c.kkeys[i];
    if (k == kEmpty || k == kTomb) continue;
    const long long p = atomicAdd(reinterpret_cast<unsigned long long *>(count), 1ull);
    out_keys[p] = k;
    out_vbits[p] = ~__double_as_longlong(c.kval[i]) & LLONG_MAX;  // ascending = descending count
    out_pos[p] = static_cast<int32_t>(i);
  }
}

// top-k preselection for stage(limit): histogram of the top 16 bits of the
// (descending-count) sort key over live sketch keys
__global__ void k_sketch_hist(CacheView c, int32_t *hist) {
  // decayed counts take few distinct values: lanes hitting the same bin are
  // merged (one atomic per distinct bin per warp instead of one per key)
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); i0 < c.kcap; i0 += stride) {
    const int64_t i = i0 + lane;
    int bin = -1;
    if (i < c.kcap) {
      const uint64_t k = c.kkeys[i];
      if (k != kEmpty && k != kTomb) bin = static_cast<int>((~__double_as_longlong(c.kval[i]) & LLONG_MAX) >> 47);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, bin);
    if (bin >= 0 && lane == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
  }
}

// live keys whose bin <= max_bin (every key that can be among the top k)
__global__ void k_sketch_collect_upto(CacheView c, int32_t max_bin, uint64_t *out_keys, int32_t *out_pos,
                                      long long *count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.kcap; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = c.kkeys[i];
    if (k == kEmpty || k == kTomb) continue;
    const long long vb = ~__double_as_longlong(c.kval[i]) & LLONG_MAX;
    if ((vb >> 47) > max_bin) continue;
    const long long p = atomicAdd(reinterpret_cast<unsigned long long *>(count), 1ull);
    out_keys[p] = k;
    out_pos[p] = static_cast<int32_t>(i);
  }
}

// ranked keys -> pending (sequential room accounting, cache.py:323-342)
__global__ void k_stage_seq(CacheView c, const int32_t *ranked_pos, int64_t m, int64_t limit) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Scalars *sc = c.sc;
  long long room = sc->budget - sc->used;
  long long staged = 0, pend = sc->pending;
  if (room > 0 && sc->sketch_live > 0) {
    for (int64_t i = 0; i < m; ++i) {
      const int32_t p = ranked_pos[i];
      const uint64_t key = c.kkeys[p];
      if (c.kflag[p] || h_find(c, key) >= 0) continue;
      const int32_t size = table_bytes_of(c, key);
      if (size < 0 || size > room) continue;
      if (pend >= c.pend_cap) break;
      c.pend[pend++] = key;
      c.kflag[p] = 1;
      room -= size;
      ++staged;
      if (limit >= 0 && staged >= limit) break;
    }
  }
  sc->pending = pend;
  sc->staged = staged;
}

__global__ void k_clear_pending_flags(CacheView c) {
  const long long n = c.sc->pending;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = k_find(c, c.pend[i]);
    if (p >= 0) c.kflag[p] = 0;
  }
}

__global__ void k_pending_done(Scalars *sc) { sc->pending = 0; }

// ---------------------------------------------------------------- aging
__global__ void k_age(CacheView c) {
  long long dead = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.kcap; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = c.kkeys[i];
    if (k == kEmpty || k == kTomb) continue;
    const double v = c.kval[i] * c.decay;
    if (v < c.prune) {
      c.kkeys[i] = kTomb;
      c.kval[i] = 0.0;
      c.kflag[i] = 0;
      ++dead;
    } else {
      c.kval[i] = v;
    }
  }
  for (int o = 16; o; o >>= 1) dead += __shfl_down_sync(0xffffffffu, dead, o);
  if ((threadIdx.x & 31) == 0 && dead) {
    atomicAdd(reinterpret_cast<unsigned long long *>(&c.sc->sketch_live), (unsigned long long)(-dead));
    atomicAdd(reinterpret_cast<unsigned long long *>(&c.sc->sketch_tomb), (unsigned long long)dead);
  }
}

// ---------------------------------------------------------------- rehash
__global__ void k_sketch_rehash(CacheView dst, const uint64_t *okeys, const double *oval, const uint8_t *oflag,
                                int64_t ocap) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ocap; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = okeys[i];
    if (k == kEmpty || k == kTomb) continue;
    const uint64_t m = static_cast<uint64_t>(dst.kcap - 1);
    uint64_t h = hash_key(k) & m;
    while (atomicCAS(reinterpret_cast<unsigned long long *>(&dst.kkeys[h]), (unsigned long long)kEmpty,
                     (unsigned long long)k) != kEmpty)
      h = (h + 1) & m;
    dst.kval[h] = oval[i];
    dst.kflag[h] = oflag[i];
  }
}

__global__ void k_index_rebuild(CacheView c) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.scap; i += (int64_t)gridDim.x * blockDim.x)
    if (c.stick[i] != kFree) h_insert(c, c.skey[i], static_cast<int32_t>(i));
}

__global__ void k_fill_u64(uint64_t *p, int64_t n, uint64_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// ---------------------------------------------------------------- queries
__global__ void k_lookup_rows(CacheView c, const uint64_t *keys, int64_t n, float *out, int32_t out_ld,
                              int32_t *found) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    const int32_t s = h_find(c, keys[i]);
    if (lane == 0) found[i] = s;
    if (s < 0) continue;
    const int32_t dim = c.ssize[s] / 4;
    for (int k = lane; k < dim && k < out_ld; k += 32) out[i * out_ld + k] = c.rows[(int64_t)s * c.row_ld + k];
  }
}

__global__ void k_sketch_lookup(CacheView c, const uint64_t *keys, int64_t n, double *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = k_est(c, keys[i]);
}

__global__ void k_sketch_bump(CacheView c, const uint64_t *keys, const double *w, int64_t n) {
  long long born = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    born += k_add(c, keys[i], w[i]) ? 1 : 0;
  if (born) atomicAdd(reinterpret_cast<unsigned long long *>(&c.sc->sketch_live), (unsigned long long)born);
}

__global__ void k_gather_vbits(CacheView c, const int32_t *pos, int64_t n, long long *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = ~__double_as_longlong(c.kval[pos[i]]) & LLONG_MAX;
}

__global__ void k_dump_lru(CacheView c, const int32_t *lru_slot, int64_t n, uint64_t *keys, long long *ticks,
                           int32_t *hits) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = lru_slot[i];
    keys[i] = c.skey[s];
    if (ticks) ticks[i] = c.stick[s];
    if (hits) hits[i] = c.shits[s];
  }
}

__global__ void k_dump_sketch(CacheView c, const int32_t *pos, int64_t n, uint64_t *keys, double *vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = c.kkeys[pos[i]];
    vals[i] = c.kval[pos[i]];
  }
}

static inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

// bits needed for LRU sort keys when every live tick is <= tick (free slots
// sort last as (1 << bits) - 1)
static inline int lru_bits(long long tick) {
  int b = 1;
  while (b < 63 && (1ll << b) - 1 <= tick) ++b;
  return b;
}

}  // namespace fx

using namespace fx;


namespace {

template <typename T>
int dmalloc(T **p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void **>(p), n * sizeof(T));
  return cuda_check(e, "fx_cache: cudaMalloc");
}
#ifdef FX_BOUNDS
template <typename T>
int dmalloc(CkPtr<T> *p, size_t n) {
  T *q = nullptr;
  const int rc = dmalloc(&q, n);
  *p = q;
  ck_size(*p, static_cast<long long>(n));
  return rc;
}
#endif

int ensure_ws(fx_cache *c, size_t need) {
  if (c->ws_bytes >= need) return FX_OK;
  if (c->ws) cudaFree(c->ws);
  c->ws = nullptr;
  c->ws_bytes = 0;
  int rc = cuda_check(cudaMalloc(&c->ws, need), "fx_cache: workspace");
  if (rc == FX_OK) c->ws_bytes = need;
  return rc;
}

int64_t pow2_at_least(int64_t x) {
  int64_t p = 1024;
  while (p < x) p <<= 1;
  return p;
}

int read_scalars(fx_cache *c, Scalars *h, cudaStream_t st) {
  int rc = cuda_check(cudaMemcpyAsync(h, c->v.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, st), "scalars");
  if (rc) return rc;
  return cuda_check(cudaStreamSynchronize(st), "scalars sync");
}

// rebuild the open-addressing index from the slots after fused steps (which
// keep a dense index instead)
int ensure_hash(fx_cache *c, cudaStream_t st) {
  if (c->hash_valid) return FX_OK;
  k_fill_u64<<<grid_for(c->v.hcap, 256), 256, 0, st>>>(c->v.hkeys, c->v.hcap, kEmpty);
  k_index_rebuild<<<grid_for(c->v.scap, 256), 256, 0, st>>>(c->v);
  cudaMemsetAsync(&c->v.sc->hash_tomb, 0, sizeof(long long), st);
  FX_LAUNCH_CHECK("fx_cache: hash rebuild");
  c->hash_valid = 1;
  return FX_OK;
}

// LRU order of the live slots into w.lru_slot: the full order, or — when only
// the `need` oldest entries can be touched (uniform entry size: every accept
// evicts one entry) and need is small — just a sorted prefix covering them.
int sort_lru(fx_cache *c, cudaStream_t st, OfferWS &w, void *cub_tmp, size_t cb, const Scalars &h, int64_t need) {
  const int64_t S = c->v.scap;
  const int bits = lru_bits(h.tick);
  w.lru_valid = h.entries;
  if (h.entries <= 0) return FX_OK;
  if (c->uniform <= 0 || need * 4 >= h.entries || bits <= 16) {
    k_lru_keys<<<grid_for(S, 256), 256, 0, st>>>(c->v, w, (1ll << bits) - 1);
    cub::DeviceRadixSort::SortPairs(cub_tmp, cb, w.sort_keys_in, w.sort_keys_out, w.iota, w.lru_slot,
                                    static_cast<int>(S), 0, bits, st);
    return cuda_check(cudaGetLastError(), "sort_lru");
  }
  constexpr int kBins = 1 << 16;
  const int shift = bits - 16;
  if (!c->lru_hist) {
    int rc = dmalloc(&c->lru_hist, kBins + 4);
    if (rc) return rc;
  }
  cudaMemsetAsync(c->lru_hist, 0, (kBins + 4) * 4, st);
  k_lru_hist<<<grid_for(S, 256), 256, 0, st>>>(c->v, shift, c->lru_hist);
  std::vector<int32_t> hh(kBins);
  int rc = cuda_check(cudaMemcpyAsync(hh.data(), c->lru_hist, kBins * 4, cudaMemcpyDeviceToHost, st), "lru hist");
  if (rc) return rc;
  rc = cuda_check(cudaStreamSynchronize(st), "lru hist sync");
  if (rc) return rc;
  int64_t cum = 0;
  int b = kBins - 1;
  for (int i = 0; i < kBins; ++i) {
    cum += hh[i];
    if (cum >= need) {
      b = i;
      break;
    }
  }
  unsigned long long *cnt = reinterpret_cast<unsigned long long *>(c->lru_hist + kBins);
  cudaMemsetAsync(cnt, 0, 8, st);
  k_lru_collect<<<grid_for(S, 256), 256, 0, st>>>(c->v, shift, b, w, cnt);
  cub::DeviceRadixSort::SortPairs(cub_tmp, cb, w.sort_keys_in, w.sort_keys_out, w.iota, w.lru_slot,
                                  static_cast<int>(cum), 0, bits, st);
  w.lru_valid = cum;
  return cuda_check(cudaGetLastError(), "sort_lru partial");
}

// Layout one offer workspace for n candidates over the cache's slot capacity.
size_t offer_ws_bytes(fx_cache *c, int64_t n, size_t *cub_bytes) {
  const int64_t S = c->v.scap;
  size_t cb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cb, (const long long *)nullptr, (long long *)nullptr,
                                  (const int32_t *)nullptr, (int32_t *)nullptr, static_cast<int>(S));
  *cub_bytes = cb;
  const int64_t nn = n > 0 ? n : 1;
  size_t cs = 0;
  cub::DeviceSelect::Flagged(nullptr, cs, (const int32_t *)nullptr, (const int32_t *)nullptr, (int32_t *)nullptr,
                             (int64_t *)nullptr, static_cast<int>(nn));
  if (cs > cb) cb = cs;
  *cub_bytes = cb;
  return al(nn * 8) + al(nn * 4) + al(nn) + al(S * 4) + al(S * 8) + al(S * 4 + nn * 4) + al(nn * 4) +
         al(S * 8 + nn * 8) + al(S * 8) * 2 + al(S * 4) + al(nn * 4) * 3 + al(8) + al(nn * 8) + al(64) + al(cb);
}

OfferWS carve_offer_ws(fx_cache *c, int64_t n, void **cub_tmp) {
  const int64_t S = c->v.scap;
  const int64_t nn = n > 0 ? n : 1;
  char *p = static_cast<char *>(c->ws);
  OfferWS w;
  w.est_cand = reinterpret_cast<double *>(p); p += al(nn * 8);
  w.size_cand = reinterpret_cast<int32_t *>(p); p += al(nn * 4);
  w.present = reinterpret_cast<uint8_t *>(p); p += al(nn);
  w.lru_slot = reinterpret_cast<int32_t *>(p); p += al(S * 4);
  w.est_vic = reinterpret_cast<double *>(p); p += al(S * 8);
  w.acc_slot = reinterpret_cast<int32_t *>(p); p += al(S * 4 + nn * 4);
  w.acc_j = reinterpret_cast<int32_t *>(p); p += al(nn * 4);
  w.ev_keys = reinterpret_cast<uint64_t *>(p); p += al(S * 8 + nn * 8);
  w.sort_keys_in = reinterpret_cast<long long *>(p); p += al(S * 8);
  w.sort_keys_out = reinterpret_cast<long long *>(p); p += al(S * 8);
  w.iota = reinterpret_cast<int32_t *>(p); p += al(S * 4);
  w.par_flag = reinterpret_cast<int32_t *>(p); p += al(nn * 4);
  w.par_iota = reinterpret_cast<int32_t *>(p); p += al(nn * 4);
  w.par_cand = reinterpret_cast<int32_t *>(p); p += al(nn * 4);
  w.par_m = reinterpret_cast<int64_t *>(p); p += al(8);
  w.est_cc = reinterpret_cast<double *>(p); p += al(nn * 8);
  w.pstate = reinterpret_cast<long long *>(p); p += al(64);
  *cub_tmp = p;
  return w;
}

// Shared offer/apply/shrink pipeline (see k_offer_seq).
int run_offer(fx_cache *c, const uint64_t *keys, int64_t n, int32_t mode, const int32_t *sizes,
              const float *const *src_rows, uint8_t *accepted, cudaStream_t st) {
  size_t cb = 0;
  const size_t need = offer_ws_bytes(c, n, &cb);
  int rc = ensure_ws(c, need);
  if (rc) return rc;
  void *cub_tmp = nullptr;
  OfferWS w = carve_offer_ws(c, n, &cub_tmp);
  Scalars h;
  rc = read_scalars(c, &h, st);
  if (rc) return rc;
  if (c->last_ev_cap < h.entries + n + 1) {
    if (c->last_ev) cudaFree(c->last_ev);
    c->last_ev_cap = 2 * (h.entries + n + 1);
    rc = dmalloc(&c->last_ev, c->last_ev_cap);
    if (rc) return rc;
  }
  w.ev_keys = c->last_ev;
  // room check: capacity for the worst case (every candidate inserted)
  if (h.entries + n > c->v.scap) {
    // slots can run out only if the byte budget admits more rows than the
    // reserved slot capacity; the host reserves slots for the budget.
    long long min_bytes = LLONG_MAX;
    for (int32_t b : c->tbytes_host)
      if (b > 0 && b < min_bytes) min_bytes = b;
    if (min_bytes == LLONG_MAX || h.budget / min_bytes > c->v.scap) {
      set_error("fx_cache: slot capacity below the budget's row count; call fx_cache_reserve_slots");
      return FX_E_CAPACITY;
    }
  }
  static const bool prof = getenv("FX_CACHE_PROFILE") != nullptr;
  cudaEvent_t pe[5];
  if (prof) {
    for (auto &e : pe) cudaEventCreate(&e);
    cudaEventRecord(pe[0], st);
  }
  if (n > 0) k_offer_prep<<<grid_for(n, 256), 256, 0, st>>>(c->v, keys, n, sizes, w);
  int64_t k_vic = 0;
  w.lru_valid = 0;
  if (h.entries > 0) {
    // entries that can be evicted: the over-budget excess plus one per candidate
    int64_t over = 0;
    if (c->uniform > 0) {
      const long long S1 = c->uniform;
      const long long ph = h.used / S1 > h.entries ? h.used / S1 - h.entries : 0;
      const long long capn = h.budget / S1 - ph;
      over = h.entries > capn ? h.entries - (capn > 0 ? capn : 0) : 0;
    }
    rc = sort_lru(c, st, w, cub_tmp, cb, h, over + n + 1);
    if (rc) return rc;
    k_vic = h.entries < n ? h.entries : n;
    if (mode == 0 && c->v.admission == 0 && k_vic > 0)
      k_vic_prep<<<grid_for(k_vic, 256), 256, 0, st>>>(c->v, w, k_vic);
    else
      k_vic = 0;
  }
  if (prof) cudaEventRecord(pe[1], st);
  static bool offer_smem_set[64] = {false};  // per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!offer_smem_set[dev & 63]) {
    cudaFuncSetAttribute(k_offer_par, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(OFFER_SMEM));
    offer_smem_set[dev & 63] = true;
  }
  const bool par = c->parallel_offers && c->uniform > 0 && sizes == nullptr && n > 0;
  if (par) {
    // compact the non-present candidates, then resolve decisions run by run
    k_mark_absent<<<grid_for(n, 256), 256, 0, st>>>(w.present, n, w.par_flag);
    k_iota32<<<grid_for(n, 256), 256, 0, st>>>(w.par_iota, n);
    cub::DeviceSelect::Flagged(cub_tmp, cb, w.par_iota, w.par_flag, w.par_cand, w.par_m, static_cast<int>(n), st);
    k_present_accept<<<grid_for(n, 256), 256, 0, st>>>(w.present, n, mode, accepted);
    ParWS pw{w.par_cand, n, w.par_m};
    k_est_compact<<<grid_for(n, 256), 256, 0, st>>>(w, pw);
    k_offer_par<<<1, 1024, OFFER_SMEM, st>>>(c->v, keys, mode, w, pw, k_vic, c->uniform, accepted, c->record);
    k_offer_apply_keys<<<grid_for(n, 256), 256, 0, st>>>(c->v, keys, w, c->record);
    k_offer_apply_slots<<<grid_for(n, 256), 256, 0, st>>>(c->v, keys, w, c->uniform);
  } else if (c->uniform > 0 && n == 0 && h.used > h.budget) {
    ParWS pw{w.par_cand, 0, nullptr};
    k_offer_par<<<1, 1024, OFFER_SMEM, st>>>(c->v, keys, mode, w, pw, k_vic, c->uniform, accepted, c->record);
  } else {
    k_offer_seq<<<1, 32, 0, st>>>(c->v, keys, n, mode, w, k_vic, accepted, c->record);
  }
  if (prof) cudaEventRecord(pe[2], st);
  k_hash_erase<<<grid_for(h.entries + n + 1, 256), 256, 0, st>>>(c->v, w);
  if (n > 0) k_install<<<grid_for(n * 32, 256), 256, 0, st>>>(c->v, w, keys, src_rows);
  FX_LAUNCH_CHECK("fx_cache offer");
  if (prof) {
    cudaEventRecord(pe[3], st);
    cudaEventSynchronize(pe[3]);
    float a = 0, b = 0, cc = 0;
    cudaEventElapsedTime(&a, pe[0], pe[1]);
    cudaEventElapsedTime(&b, pe[1], pe[2]);
    cudaEventElapsedTime(&cc, pe[2], pe[3]);
    fprintf(stderr, "[fx_cache offer] n=%lld entries=%lld prep+sort %.3f ms, decide %.3f ms, index+rows %.3f ms\n",
            (long long)n, (long long)h.entries, a, b, cc);
    for (auto &e : pe) cudaEventDestroy(e);
  }
  // keep the index below half tombstones
  rc = read_scalars(c, &h, st);
  if (rc) return rc;
  if ((h.hash_tomb + h.entries) * 2 > c->v.hcap) {
    k_fill_u64<<<grid_for(c->v.hcap, 256), 256, 0, st>>>(c->v.hkeys, c->v.hcap, kEmpty);
    k_index_rebuild<<<grid_for(c->v.scap, 256), 256, 0, st>>>(c->v);
    cudaMemsetAsync(&c->v.sc->hash_tomb, 0, sizeof(long long), st);
    FX_LAUNCH_CHECK("fx_cache index rebuild");
  }
  return FX_OK;
}

int upload_dir(fx_cache *c) {
  if (c->dir_dev) cudaFree(c->dir_dev);
  if (c->tbytes_dev) cudaFree(c->tbytes_dev);
  c->dir_dev = nullptr;
  c->tbytes_dev = nullptr;
  int rc = dmalloc(&c->dir_dev, c->dir_host.size());
  if (rc) return rc;
  rc = dmalloc(&c->tbytes_dev, c->tbytes_host.size());
  if (rc) return rc;
  if (!c->dir_host.empty())
    cudaMemcpy(c->dir_dev, c->dir_host.data(), c->dir_host.size() * sizeof(fx_table_dir), cudaMemcpyHostToDevice);
  if (!c->tbytes_host.empty())
    cudaMemcpy(c->tbytes_dev, c->tbytes_host.data(), c->tbytes_host.size() * 4, cudaMemcpyHostToDevice);
  c->v.dir = c->dir_dev;
  c->v.n_dir = static_cast<int32_t>(c->dir_host.size());
  c->v.tbytes = c->tbytes_dev;
  c->v.n_tbytes = static_cast<int32_t>(c->tbytes_host.size());
  return cuda_check(cudaGetLastError(), "fx_cache: upload dir");
}

}  // namespace

extern "C" {

int fx_cache_create(fx_cache **out, int64_t slot_capacity, int32_t max_dim, int32_t admission, double decay,
                    double prune_below, int64_t budget_bytes, int64_t sketch_capacity, int32_t record_evictions) {
  if (!out || slot_capacity < 0 || max_dim < 1 || (admission != 0 && admission != 1) || budget_bytes < 0) {
    set_error("fx_cache_create: bad arguments");
    return FX_E_CONFIG;
  }
  fx_cache *c = new fx_cache();
  CacheView &v = c->v;
  v.scap = slot_capacity > 0 ? slot_capacity : 1;
  v.row_ld = (max_dim + 3) & ~3;
  v.hcap = pow2_at_least(4 * v.scap);
  v.kcap = pow2_at_least(sketch_capacity > 0 ? 2 * sketch_capacity : 4096);
  v.pend_cap = v.scap + 1024;
  v.evlog_cap = record_evictions ? (8 * v.scap > (1 << 20) ? 8 * v.scap : (1 << 20)) : 0;
  v.admission = admission;
  v.decay = decay;
  v.prune = prune_below;
  c->record = record_evictions;
  int rc = FX_OK;
  rc = rc ? rc : dmalloc(&v.sc, 1);
  rc = rc ? rc : dmalloc(&v.hkeys, v.hcap);
  rc = rc ? rc : dmalloc(&v.hslot, v.hcap);
  rc = rc ? rc : dmalloc(&v.skey, v.scap);
  rc = rc ? rc : dmalloc(&v.skey2, v.scap);
  rc = rc ? rc : dmalloc(&v.stick, v.scap);
  rc = rc ? rc : dmalloc(&v.ssize, v.scap);
  rc = rc ? rc : dmalloc(&v.shits, v.scap);
  rc = rc ? rc : dmalloc(&v.rows, static_cast<size_t>(v.scap) * v.row_ld);
  rc = rc ? rc : dmalloc(&v.free_stack, v.scap);
  rc = rc ? rc : dmalloc(&v.kkeys, v.kcap);
  rc = rc ? rc : dmalloc(&v.kval, v.kcap);
  rc = rc ? rc : dmalloc(&v.kflag, v.kcap);
  rc = rc ? rc : dmalloc(&v.pend, v.pend_cap);
  rc = rc ? rc : dmalloc(&v.evlog, v.evlog_cap);
  if (rc) {
    delete c;
    return rc;
  }
  Scalars h{};
  h.budget = budget_bytes;
  h.free_top = v.scap;
  cudaMemcpy(v.sc, &h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemset(v.ssize, 0, v.scap * 4);
  cudaMemset(v.shits, 0, v.scap * 4);
  upload_dir(c);
  k_cache_init<<<grid_for(v.hcap > v.kcap ? v.hcap : v.kcap, 256), 256>>>(v);
  rc = cuda_check(cudaDeviceSynchronize(), "fx_cache_create");
  if (rc) {
    delete c;
    return rc;
  }
  *out = c;
  return FX_OK;
}

int fx_cache_destroy(fx_cache *c) {
  if (!c) return FX_OK;
  CacheView &v = c->v;
  void *ps[] = {v.sc, v.hkeys, v.hslot, v.skey, v.skey2, v.stick, v.ssize, v.shits, v.rows, v.free_stack, v.kkeys,
                v.kval, v.kflag, v.pend, v.evlog, c->dir_dev, c->tbytes_dev, c->ws, c->last_ev, c->lru_hist, c->q};
  for (void *p : ps)
    if (p) cudaFree(p);
  delete c;
  return FX_OK;
}

int fx_cache_set_tables(fx_cache *c, const fx_table_dir *dir, int32_t n_dir, const int32_t *table_bytes,
                        int32_t n_tables) {
  c->dir_host.assign(dir, dir + n_dir);
  c->tbytes_host.assign(table_bytes, table_bytes + n_tables);
  for (int32_t b : c->tbytes_host) {  // sticky: once two sizes are seen, stay on the general path
    if (b <= 0 || c->uniform < 0) continue;
    if (c->uniform == 0) c->uniform = b;
    else if (c->uniform != b) c->uniform = -1;
  }
  int max_dim = 0;
  for (auto &d : c->dir_host) max_dim = d.dim > max_dim ? d.dim : max_dim;
  for (int32_t b : c->tbytes_host) max_dim = b / 4 > max_dim ? b / 4 : max_dim;
  if (max_dim > c->v.row_ld) {
    set_error("fx_cache_set_tables: table dim exceeds the cache row width");
    return FX_E_CONFIG;
  }
  return upload_dir(c);
}

int fx_cache_scalars(fx_cache *c, int64_t *out, void *stream) {
  Scalars h;
  int rc = read_scalars(c, &h, as_stream(stream));
  if (rc) return rc;
  const long long *p = reinterpret_cast<const long long *>(&h);
  for (size_t i = 0; i < sizeof(Scalars) / 8; ++i) out[i] = p[i];
  return FX_OK;
}

const void *fx_cache_scalars_device(fx_cache *c) { return c->v.sc; }

int fx_cache_queue_valid(fx_cache *c) { return c->queue_valid; }

int fx_cache_capacity(fx_cache *c, int64_t *out3) {
  out3[0] = c->v.scap;
  out3[1] = c->v.hcap;
  out3[2] = c->v.kcap;
  return FX_OK;
}

int fx_cache_set_budget(fx_cache *c, int64_t budget, void *stream) {
  { int hrc = ensure_hash(c, as_stream(stream)); if (hrc) return hrc; }
  c->queue_valid = 0;
  cudaStream_t st = as_stream(stream);
  cudaMemcpyAsync(&c->v.sc->budget, &budget, 8, cudaMemcpyHostToDevice, st);
  // shrink: evict LRU until used <= budget (cache.py:270-274)
  return run_offer(c, nullptr, 0, 1, nullptr, nullptr, nullptr, st);
}

int fx_cache_reserve_sketch(fx_cache *c, int64_t new_keys, void *stream) {
  cudaStream_t st = as_stream(stream);
  Scalars h;
  int rc = read_scalars(c, &h, st);
  if (rc) return rc;
  const int64_t need = 2 * (h.sketch_live + new_keys) + 1024;
  if (need <= c->v.kcap && (h.sketch_live + h.sketch_tomb + new_keys) * 2 <= c->v.kcap) return FX_OK;
  CacheView nv = c->v;
  nv.kcap = pow2_at_least(need > c->v.kcap ? 2 * need : c->v.kcap);
  rc = dmalloc(&nv.kkeys, nv.kcap);
  rc = rc ? rc : dmalloc(&nv.kval, nv.kcap);
  rc = rc ? rc : dmalloc(&nv.kflag, nv.kcap);
  if (rc) return rc;
  k_fill_u64<<<grid_for(nv.kcap, 256), 256, 0, st>>>(nv.kkeys, nv.kcap, kEmpty);
  cudaMemsetAsync(nv.kval, 0, nv.kcap * 8, st);
  cudaMemsetAsync(nv.kflag, 0, nv.kcap, st);
  k_sketch_rehash<<<grid_for(c->v.kcap, 256), 256, 0, st>>>(nv, c->v.kkeys, c->v.kval, c->v.kflag, c->v.kcap);
  cudaMemsetAsync(&c->v.sc->sketch_tomb, 0, 8, st);
  rc = cuda_check(cudaStreamSynchronize(st), "fx_cache_reserve_sketch");
  cudaFree(c->v.kkeys);
  cudaFree(c->v.kval);
  cudaFree(c->v.kflag);
  c->v = nv;
  return rc;
}

int fx_cache_reserve_slots(fx_cache *c, int64_t slots, void *stream) {
  c->queue_valid = 0;
  cudaStream_t st = as_stream(stream);
  if (slots <= c->v.scap) return FX_OK;
  int rc = cuda_check(cudaStreamSynchronize(st), "fx_cache_reserve_slots");
  if (rc) return rc;
  CacheView nv = c->v;
  nv.scap = slots;
  nv.hcap = pow2_at_least(4 * slots);
  nv.pend_cap = slots + 1024;
  rc = dmalloc(&nv.skey, nv.scap);
  rc = rc ? rc : dmalloc(&nv.skey2, nv.scap);
  rc = rc ? rc : dmalloc(&nv.stick, nv.scap);
  rc = rc ? rc : dmalloc(&nv.ssize, nv.scap);
  rc = rc ? rc : dmalloc(&nv.shits, nv.scap);
  rc = rc ? rc : dmalloc(&nv.rows, static_cast<size_t>(nv.scap) * nv.row_ld);
  rc = rc ? rc : dmalloc(&nv.free_stack, nv.scap);
  rc = rc ? rc : dmalloc(&nv.hkeys, nv.hcap);
  rc = rc ? rc : dmalloc(&nv.hslot, nv.hcap);
  rc = rc ? rc : dmalloc(&nv.pend, nv.pend_cap);
  if (rc) return rc;
  const int64_t S0 = c->v.scap;
  // old slots keep their ids; new slots are appended to the free stack
  k_fill_u64<<<grid_for(nv.scap, 256), 256, 0, st>>>(nv.skey, nv.scap, kEmpty);
  std::vector<long long> freeticks(1, kFree);
  cudaMemcpyAsync(nv.skey, c->v.skey, S0 * 8, cudaMemcpyDeviceToDevice, st);
  cudaMemsetAsync(nv.skey2, 0, nv.scap * 8, st);
  cudaMemcpyAsync(nv.skey2, c->v.skey2, S0 * 8, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(nv.ssize, c->v.ssize, S0 * 4, cudaMemcpyDeviceToDevice, st);
  cudaMemsetAsync(nv.ssize + S0, 0, (nv.scap - S0) * 4, st);
  cudaMemcpyAsync(nv.shits, c->v.shits, S0 * 4, cudaMemcpyDeviceToDevice, st);
  cudaMemsetAsync(nv.shits + S0, 0, (nv.scap - S0) * 4, st);
  cudaMemcpyAsync(nv.rows, c->v.rows, static_cast<size_t>(S0) * c->v.row_ld * 4, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(nv.pend, c->v.pend, c->v.pend_cap * 8, cudaMemcpyDeviceToDevice, st);
  // ticks: copy then mark the new slots free
  cudaMemcpyAsync(nv.stick, c->v.stick, S0 * 8, cudaMemcpyDeviceToDevice, st);
  k_fill_u64<<<grid_for(nv.scap - S0, 256), 256, 0, st>>>(reinterpret_cast<uint64_t *>(nv.stick + S0),
                                                           nv.scap - S0, static_cast<uint64_t>(kFree));
  // free stack: existing free entries first (top of stack = old order), new ids below them
  Scalars h;
  rc = read_scalars(c, &h, st);
  if (rc) return rc;
  std::vector<int32_t> fs(nv.scap);
  int64_t k = 0;
  for (int64_t s = nv.scap - 1; s >= S0; --s) fs[k++] = static_cast<int32_t>(s);
  std::vector<int32_t> oldfs(h.free_top > 0 ? h.free_top : 1);
  if (h.free_top > 0) cudaMemcpy(oldfs.data(), c->v.free_stack, h.free_top * 4, cudaMemcpyDeviceToHost);
  for (long long i = 0; i < h.free_top; ++i) fs[k++] = oldfs[i];
  cudaMemcpy(nv.free_stack, fs.data(), k * 4, cudaMemcpyHostToDevice);
  h.free_top = k;
  h.hash_tomb = 0;
  cudaMemcpy(c->v.sc, &h, sizeof(h), cudaMemcpyHostToDevice);
  k_fill_u64<<<grid_for(nv.hcap, 256), 256, 0, st>>>(nv.hkeys, nv.hcap, kEmpty);
  k_index_rebuild<<<grid_for(nv.scap, 256), 256, 0, st>>>(nv);
  rc = cuda_check(cudaStreamSynchronize(st), "fx_cache_reserve_slots");
  c->hash_valid = 1;  // rebuilt from the slots above
  void *old[] = {c->v.skey, c->v.skey2, c->v.stick, c->v.ssize, c->v.shits, c->v.rows, c->v.free_stack, c->v.hkeys,
                 c->v.hslot, c->v.pend};
  for (void *p : old) cudaFree(p);
  c->v = nv;
  return rc;
}

int fx_cache_probe(fx_cache *c, const uint64_t *uniq, const int32_t *mult, const int64_t *last_ord,
                   const int64_t *n_uniq_dev, int64_t n_uniq_host, int64_t nnz, int32_t *slot_out, void *stream) {
  { int hrc = ensure_hash(c, as_stream(stream)); if (hrc) return hrc; }
  c->queue_valid = 0;
  cudaStream_t st = as_stream(stream);
  const int64_t work = n_uniq_dev ? nnz : n_uniq_host;
  k_probe<<<grid_for(work > 0 ? work : 1, 256), 256, 0, st>>>(c->v, uniq, mult, last_ord, n_uniq_dev, n_uniq_host,
                                                              slot_out);
  k_advance_tick<<<1, 1, 0, st>>>(c->v.sc, nnz);
  FX_LAUNCH_CHECK("fx_cache_probe");
  return FX_OK;
}

int fx_cache_offer(fx_cache *c, const uint64_t *keys, int64_t n, const int32_t *sizes, const float *const *src_rows,
                   uint8_t *accepted, void *stream) {
  { int hrc = ensure_hash(c, as_stream(stream)); if (hrc) return hrc; }
  c->queue_valid = 0;
  return run_offer(c, keys, n, 0, sizes, src_rows, accepted, as_stream(stream));
}

int fx_cache_apply_pending(fx_cache *c, int64_t *applied, void *stream) {
  { int hrc = ensure_hash(c, as_stream(stream)); if (hrc) return hrc; }
  c->queue_valid = 0;
  cudaStream_t st = as_stream(stream);
  Scalars h;
  int rc = read_scalars(c, &h, st);
  if (rc) return rc;
  const int64_t n = h.pending;
  long long e0 = h.entries;
  if (n > 0) {
    // clear the pending flags first (keys stay in c->v.pend until the insert ran)
    k_clear_pending_flags<<<grid_for(n, 256), 256, 0, st>>>(c->v);
    rc = run_offer(c, c->v.pend, n, 1, nullptr, c->pending_rows, nullptr, st);
    c->pending_rows = nullptr;
    if (rc) return rc;
    k_pending_done<<<1, 1, 0, st>>>(c->v.sc);
    rc = read_scalars(c, &h, st);
    if (rc) return rc;
  }
  if (applied) *applied = n > 0 ? h.n_acc : 0;
  (void)e0;
  return FX_OK;
}

// Rank all live sketch keys by (-count, key) into ranked positions (device
// workspace); returns the live count. Used by stage + hottest queries.
static int rank_sketch(fx_cache *c, cudaStream_t st, int64_t *n_live, int32_t **ranked, void **tail) {
  Scalars h;
  int rc = read_scalars(c, &h, st);
  if (rc) return rc;
  const int64_t L = h.sketch_live;
  *n_live = L;
  if (L <= 0) return FX_OK;
  size_t cb1 = 0, cb2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cb1, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                  (const int32_t *)nullptr, (int32_t *)nullptr, static_cast<int>(L));
  cub::DeviceRadixSort::SortPairs(nullptr, cb2, (const long long *)nullptr, (long long *)nullptr,
                                  (const int32_t *)nullptr, (int32_t *)nullptr, static_cast<int>(L));
  size_t cb = cb1 > cb2 ? cb1 : cb2;
  const size_t need = al(L * 8) * 4 + al(L * 4) * 3 + al(8) + al(cb) + al(L * 16);
  rc = ensure_ws(c, need);
  if (rc) return rc;
  char *p = static_cast<char *>(c->ws);
  uint64_t *keys = reinterpret_cast<uint64_t *>(p); p += al(L * 8);
  uint64_t *keys2 = reinterpret_cast<uint64_t *>(p); p += al(L * 8);
  long long *vb = reinterpret_cast<long long *>(p); p += al(L * 8);
  long long *vb2 = reinterpret_cast<long long *>(p); p += al(L * 8);
  int32_t *pos = reinterpret_cast<int32_t *>(p); p += al(L * 4);
  int32_t *pos2 = reinterpret_cast<int32_t *>(p); p += al(L * 4);
  int32_t *pos3 = reinterpret_cast<int32_t *>(p); p += al(L * 4);
  long long *cnt = reinterpret_cast<long long *>(p); p += al(8);
  void *tmp = p; p += al(cb);
  cudaMemsetAsync(cnt, 0, 8, st);
  k_sketch_collect<<<grid_for(c->v.kcap, 256), 256, 0, st>>>(c->v, keys, vb, pos, cnt);
  // LSD: stable sort by key, then stable sort by inverted count bits
  cub::DeviceRadixSort::SortPairs(tmp, cb, keys, keys2, pos, pos2, static_cast<int>(L), 0, 64, st);
  k_gather_vbits<<<grid_for(L, 256), 256, 0, st>>>(c->v, pos2, L, vb);
  cub::DeviceRadixSort::SortPairs(tmp, cb, vb, vb2, pos2, pos3, static_cast<int>(L), 0, 64, st);
  FX_LAUNCH_CHECK("fx_cache rank sketch");
  *ranked = pos3;
  *tail = p;
  return FX_OK;
}

// Exact top-k of the sketch by (-count, key) without sorting every key: a
// 65536-bin histogram of the sort key's top bits finds the bin holding the
// k-th key; only keys in that bin or hotter are collected and fully ranked.
static int rank_sketch_topk(fx_cache *c, cudaStream_t st, int64_t k, int64_t *n_cand, int32_t **ranked) {
  constexpr int kBins = 1 << 16;
  int rc = ensure_ws(c, al(kBins * 4));
  if (rc) return rc;
  int32_t *hist = static_cast<int32_t *>(c->ws);
  cudaMemsetAsync(hist, 0, kBins * 4, st);
  k_sketch_hist<<<grid_for(c->v.kcap, 256), 256, 0, st>>>(c->v, hist);
  std::vector<int32_t> h(kBins);
  rc = cuda_check(cudaMemcpyAsync(h.data(), hist, kBins * 4, cudaMemcpyDeviceToHost, st), "sketch hist");
  if (rc) return rc;
  rc = cuda_check(cudaStreamSynchronize(st), "sketch hist sync");
  if (rc) return rc;
  int64_t cum = 0;
  int bin = kBins - 1;
  for (int b = 0; b < kBins; ++b) {
    cum += h[b];
    if (cum >= k) {
      bin = b;
      break;
    }
  }
  const int64_t C = cum;  // keys in bins <= bin
  *n_cand = C;
  if (C <= 0) return FX_OK;
  size_t cb1 = 0, cb2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cb1, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                  (const int32_t *)nullptr, (int32_t *)nullptr, static_cast<int>(C));
  cub::DeviceRadixSort::SortPairs(nullptr, cb2, (const long long *)nullptr, (long long *)nullptr,
                                  (const int32_t *)nullptr, (int32_t *)nullptr, static_cast<int>(C));
  size_t cb = cb1 > cb2 ? cb1 : cb2;
  const size_t need = al(C * 8) * 4 + al(C * 4) * 3 + al(8) + al(cb);
  rc = ensure_ws(c, need);
  if (rc) return rc;
  char *p = static_cast<char *>(c->ws);
  uint64_t *keys = reinterpret_cast<uint64_t *>(p); p += al(C * 8);
  uint64_t *keys2 = reinterpret_cast<uint64_t *>(p); p += al(C * 8);
  long long *vb = reinterpret_cast<long long *>(p); p += al(C * 8);
  long long *vb2 = reinterpret_cast<long long *>(p); p += al(C * 8);
  int32_t *pos = reinterpret_cast<int32_t *>(p); p += al(C * 4);
  int32_t *pos2 = reinterpret_cast<int32_t *>(p); p += al(C * 4);
  int32_t *pos3 = reinterpret_cast<int32_t *>(p); p += al(C * 4);
  long long *cnt = reinterpret_cast<long long *>(p); p += al(8);
  void *tmp = p;
  cudaMemsetAsync(cnt, 0, 8, st);
  k_sketch_collect_upto<<<grid_for(c->v.kcap, 256), 256, 0, st>>>(c->v, bin, keys, pos, cnt);
  cub::DeviceRadixSort::SortPairs(tmp, cb, keys, keys2, pos, pos2, static_cast<int>(C), 0, 64, st);
  k_gather_vbits<<<grid_for(C, 256), 256, 0, st>>>(c->v, pos2, C, vb);
  cub::DeviceRadixSort::SortPairs(tmp, cb, vb, vb2, pos2, pos3, static_cast<int>(C), 0, 64, st);
  FX_LAUNCH_CHECK("fx_cache rank sketch top-k");
  *ranked = pos3;
  return FX_OK;
}

int fx_cache_stage(fx_cache *c, int64_t limit, int64_t *staged, void *stream) {
  { int hrc = ensure_hash(c, as_stream(stream)); if (hrc) return hrc; }
  cudaStream_t st = as_stream(stream);
  Scalars h;
  int rc = read_scalars(c, &h, st);
  if (rc) return rc;
  if (staged) *staged = 0;
  if (h.budget - h.used <= 0 || h.sketch_live <= 0) return FX_OK;  // cache.py:319-320
  int64_t L = 0;
  int32_t *ranked = nullptr;
  void *tail = nullptr;
  if (limit >= 0 && limit * 16 < h.sketch_live) {
    rc = rank_sketch_topk(c, st, limit, &L, &ranked);  // L = candidates, a superset of the top `limit`
  } else {
    rc = rank_sketch(c, st, &L, &ranked, &tail);
  }
  if (rc || L <= 0) return rc;
  // hottest(n=limit) considers the top `limit` keys overall (cache.py:323-324)
  const int64_t m = limit >= 0 ? (limit < L ? limit : L) : L;
  k_stage_seq<<<1, 32, 0, st>>>(c->v, ranked, m, limit);
  FX_LAUNCH_CHECK("fx_cache_stage");
  rc = read_scalars(c, &h, st);
  if (rc) return rc;
  if (staged) *staged = h.staged;
  return FX_OK;
}

int fx_cache_age(fx_cache *c, void *stream) {
  cudaStream_t st = as_stream(stream);
  k_age<<<grid_for(c->v.kcap, 256), 256, 0, st>>>(c->v);
  FX_LAUNCH_CHECK("fx_cache_age");
  return FX_OK;
}

int fx_cache_lookup(fx_cache *c, const uint64_t *keys, int64_t n, float *rows_out, int32_t out_ld, int32_t *slot_out,
                    void *stream) {
  { int hrc = ensure_hash(c, as_stream(stream)); if (hrc) return hrc; }
  if (n <= 0) return FX_OK;
  k_lookup_rows<<<grid_for(n * 32, 256), 256, 0, as_stream(stream)>>>(c->v, keys, n, rows_out, out_ld, slot_out);
  FX_LAUNCH_CHECK("fx_cache_lookup");
  return FX_OK;
}

int fx_cache_sketch_estimate(fx_cache *c, const uint64_t *keys, int64_t n, double *out, void *stream) {
  if (n <= 0) return FX_OK;
  k_sketch_lookup<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(c->v, keys, n, out);
  FX_LAUNCH_CHECK("fx_cache_sketch_estimate");
  return FX_OK;
}

int fx_cache_sketch_bump(fx_cache *c, const uint64_t *keys, const double *weights, int64_t n, void *stream) {
  if (n <= 0) return FX_OK;
  k_sketch_bump<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(c->v, keys, weights, n);
  FX_LAUNCH_CHECK("fx_cache_sketch_bump");
  return FX_OK;
}

int fx_cache_sketch_ranked(fx_cache *c, uint64_t *keys_out, double *vals_out, int64_t cap, int64_t *n_out,
                           void *stream) {
  cudaStream_t st = as_stream(stream);
  int64_t L = 0;
  int32_t *ranked = nullptr;
  void *tail = nullptr;
  int rc = rank_sketch(c, st, &L, &ranked, &tail);
  if (rc) return rc;
  const int64_t n = L < cap ? L : cap;
  if (n > 0) k_dump_sketch<<<grid_for(n, 256), 256, 0, st>>>(c->v, ranked, n, keys_out, vals_out);
  *n_out = n;
  FX_LAUNCH_CHECK("fx_cache_sketch_ranked");
  return cuda_check(cudaStreamSynchronize(st), "fx_cache_sketch_ranked");
}

int fx_cache_lru(fx_cache *c, uint64_t *keys_out, int64_t *ticks_out, int32_t *hits_out, int64_t cap,
                 int64_t *n_out, void *stream) {
  cudaStream_t st = as_stream(stream);
  Scalars h;
  int rc = read_scalars(c, &h, st);
  if (rc) return rc;
  size_t cb = 0;
  const size_t need = offer_ws_bytes(c, 0, &cb);
  rc = ensure_ws(c, need);
  if (rc) return rc;
  void *cub_tmp = nullptr;
  OfferWS w = carve_offer_ws(c, 0, &cub_tmp);
  const int64_t S = c->v.scap;
  k_lru_keys<<<grid_for(S, 256), 256, 0, st>>>(c->v, w, (1ll << lru_bits(h.tick)) - 1);
  cub::DeviceRadixSort::SortPairs(cub_tmp, cb, w.sort_keys_in, w.sort_keys_out, w.iota, w.lru_slot,
                                  static_cast<int>(S), 0, lru_bits(h.tick), st);
  const int64_t n = h.entries < cap ? h.entries : cap;
  if (n > 0)
    k_dump_lru<<<grid_for(n, 256), 256, 0, st>>>(c->v, w.lru_slot, n, keys_out,
                                                  reinterpret_cast<long long *>(ticks_out), hits_out);
  *n_out = n;
  FX_LAUNCH_CHECK("fx_cache_lru");
  return cuda_check(cudaStreamSynchronize(st), "fx_cache_lru");
}

int fx_cache_eviction_log(fx_cache *c, uint64_t *out, int64_t cap, int64_t *n_out, void *stream) {
  cudaStream_t st = as_stream(stream);
  Scalars h;
  int rc = read_scalars(c, &h, st);
  if (rc) return rc;
  int64_t n = h.n_evlog < c->v.evlog_cap ? h.n_evlog : c->v.evlog_cap;
  if (n > cap) n = cap;
  if (n > 0) cudaMemcpyAsync(out, c->v.evlog, n * 8, cudaMemcpyDeviceToDevice, st);
  *n_out = h.n_evlog;
  return cuda_check(cudaStreamSynchronize(st), "fx_cache_eviction_log");
}

int fx_cache_pending(fx_cache *c, uint64_t *out, int64_t cap, int64_t *n_out, void *stream) {
  cudaStream_t st = as_stream(stream);
  Scalars h;
  int rc = read_scalars(c, &h, st);
  if (rc) return rc;
  const int64_t n = h.pending < cap ? h.pending : cap;
  if (n > 0) cudaMemcpyAsync(out, c->v.pend, n * 8, cudaMemcpyDeviceToDevice, st);
  *n_out = h.pending;
  return cuda_check(cudaStreamSynchronize(st), "fx_cache_pending");
}

int fx_cache_rows(fx_cache *c, const float **rows, int64_t *ld) {
  *rows = c->v.rows;
  *ld = c->v.row_ld;
  return FX_OK;
}

int fx_cache_advance_tick(fx_cache *c, int64_t n, void *stream) {
  c->queue_valid = 0;
  k_advance_tick<<<1, 1, 0, as_stream(stream)>>>(c->v.sc, n);
  FX_LAUNCH_CHECK("fx_cache_advance_tick");
  return FX_OK;
}

int fx_cache_pooled_find(fx_cache *c, const uint64_t *key_a, const uint64_t *key_b, int64_t n, int32_t *slot_out,
                         void *stream) {
  { int hrc = ensure_hash(c, as_stream(stream)); if (hrc) return hrc; }
  if (n <= 0) return FX_OK;
  k_pooled_find<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(c->v, key_a, key_b, n, slot_out);
  FX_LAUNCH_CHECK("fx_cache_pooled_find");
  return FX_OK;
}

int fx_cache_pooled_touch(fx_cache *c, const int32_t *slot, const int64_t *pos, int64_t n, void *stream) {
  { int hrc = ensure_hash(c, as_stream(stream)); if (hrc) return hrc; }
  c->queue_valid = 0;
  if (n <= 0) return FX_OK;
  k_pooled_touch<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(c->v, slot, pos, n);
  FX_LAUNCH_CHECK("fx_cache_pooled_touch");
  return FX_OK;
}

int fx_cache_read_slots(fx_cache *c, const int32_t *slot, int64_t n, float *out, int32_t out_ld, int32_t *size_out,
                        void *stream) {
  if (n <= 0) return FX_OK;
  k_read_slots<<<grid_for(n * 32, 256), 256, 0, as_stream(stream)>>>(c->v, slot, n, out, out_ld, size_out);
  FX_LAUNCH_CHECK("fx_cache_read_slots");
  return FX_OK;
}

int fx_cache_pooled_put(fx_cache *c, const uint64_t *key_a, const uint64_t *key_b, int64_t n, const int32_t *sizes,
                        int32_t uniform_size, const float *const *src_rows, void *stream) {
  { int hrc = ensure_hash(c, as_stream(stream)); if (hrc) return hrc; }
  c->queue_valid = 0;
  cudaStream_t st = as_stream(stream);
  if (n <= 0) return FX_OK;
  if (!key_a || !key_b || !src_rows || (!sizes && uniform_size <= 0)) {
    set_error("fx_cache_pooled_put: bad arguments");
    return FX_E_CONFIG;
  }
  if (sizes) c->uniform = -1;
  else if (c->uniform == 0) c->uniform = uniform_size;
  else if (c->uniform > 0 && c->uniform != uniform_size) c->uniform = -1;
  size_t cb = 0;
  const size_t base = offer_ws_bytes(c, n, &cb);
  size_t cb2 = 0, cb3 = 0, cb4 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cb2, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                  (const int32_t *)nullptr, (int32_t *)nullptr, static_cast<int>(n));
  cub::DeviceScan::InclusiveScan(nullptr, cb3, (const int32_t *)nullptr, (int32_t *)nullptr, cub::Max(),
                                 static_cast<int>(n));
  cub::DeviceScan::ExclusiveSum(nullptr, cb4, (const int32_t *)nullptr, (int32_t *)nullptr, static_cast<int>(n));
  if (cb3 > cb2) cb2 = cb3;
  if (cb4 > cb2) cb2 = cb4;
  const int64_t S = c->v.scap;
  const size_t extra = al(n * 4) * 13 + al(n * 8) + al(S * 4) + al(8) + al(cb2);
  int rc = ensure_ws(c, base + extra);
  if (rc) return rc;
  void *cub_tmp = nullptr;
  OfferWS w = carve_offer_ws(c, n, &cub_tmp);
  char *p = static_cast<char *>(c->ws) + base;
  PutWS pw;
  pw.present_slot = reinterpret_cast<int32_t *>(p); p += al(n * 4);
  pw.prev = reinterpret_cast<int32_t *>(p); p += al(n * 4);
  pw.slot_of = reinterpret_cast<int32_t *>(p); p += al(n * 4);
  pw.iota = reinterpret_cast<int32_t *>(p); p += al(n * 4);
  pw.perm = reinterpret_cast<int32_t *>(p); p += al(n * 4);
  pw.ov_slot = reinterpret_cast<int32_t *>(p); p += al(n * 4);
  pw.ov_j = reinterpret_cast<int32_t *>(p); p += al(n * 4);
  pw.keys_sorted = reinterpret_cast<uint64_t *>(p); p += al(n * 8);
  pw.writer = reinterpret_cast<int32_t *>(p); p += al(S * 4);
  pw.run_in = reinterpret_cast<int32_t *>(p); p += al(n * 4);
  pw.run_start = reinterpret_cast<int32_t *>(p); p += al(n * 4);
  pw.first = reinterpret_cast<int32_t *>(p); p += al(n * 4);
  pw.lastj = reinterpret_cast<int32_t *>(p); p += al(n * 4);
  pw.fresh = reinterpret_cast<int32_t *>(p); p += al(n * 4);
  pw.rank = reinterpret_cast<int32_t *>(p); p += al(n * 4);
  pw.fail = reinterpret_cast<int32_t *>(p); p += al(8);
  void *cub2 = p;
  Scalars h;
  rc = read_scalars(c, &h, st);
  if (rc) return rc;
  if (c->last_ev_cap < h.entries + n + 1) {
    if (c->last_ev) cudaFree(c->last_ev);
    c->last_ev_cap = 2 * (h.entries + n + 1);
    rc = dmalloc(&c->last_ev, c->last_ev_cap);
    if (rc) return rc;
  }
  w.ev_keys = c->last_ev;
  // entries never exceed budget / size (every insert first evicts to fit)
  if (h.entries + n > S && (sizes || h.budget / uniform_size > S)) {
    set_error("fx_cache_pooled_put: slot capacity below the budget's entry count; call fx_cache_reserve_slots");
    return FX_E_CAPACITY;
  }
  k_put_prep<<<grid_for(n, 256), 256, 0, st>>>(c->v, key_a, key_b, n, sizes, uniform_size, w, pw);
  cub::DeviceRadixSort::SortPairs(cub2, cb2, key_a, pw.keys_sorted, pw.iota, pw.perm, static_cast<int>(n), 0, 64,
                                  st);
  k_put_prev<<<grid_for(n, 256), 256, 0, st>>>(pw.keys_sorted, pw.perm, n, key_b, pw, c->v.sc);
  w.lru_valid = 0;
  if (h.entries > 0) {
    const long long S1 = uniform_size > 0 ? uniform_size : 1;
    const long long ph = h.used / S1 > h.entries ? h.used / S1 - h.entries : 0;
    const long long capn = h.budget / S1 - ph;
    const int64_t over = h.entries > capn ? h.entries - (capn > 0 ? capn : 0) : 0;
    rc = sort_lru(c, st, w, cub_tmp, cb, h, sizes ? h.entries : over + n + 1);
    if (rc) return rc;
  }
  const bool par = c->parallel_offers && !sizes && c->uniform > 0 && c->uniform == uniform_size;
  if (par) {
    cudaMemsetAsync(pw.fail, 0, 4, st);
    k_put_heads<<<grid_for(n, 256), 256, 0, st>>>(pw.keys_sorted, n, pw);
    cub::DeviceScan::InclusiveScan(cub2, cb2, pw.run_in, pw.run_start, cub::Max(), static_cast<int>(n), st);
    k_put_links<<<grid_for(n, 256), 256, 0, st>>>(pw.keys_sorted, n, pw);
    cub::DeviceScan::ExclusiveSum(cub2, cb2, pw.fresh, pw.rank, static_cast<int>(n), st);
    k_putp_verify<<<grid_for(n, 256), 256, 0, st>>>(c->v, n, uniform_size, pw);
    k_putp_evict<<<grid_for(h.entries + 1, 256), 256, 0, st>>>(c->v, n, uniform_size, w, pw, c->record);
    k_putp_insert<<<grid_for(n, 256), 256, 0, st>>>(c->v, key_a, key_b, n, uniform_size, w, pw, c->record);
    k_putp_finish<<<1, 1, 0, st>>>(c->v, n, uniform_size, pw, c->record);
  }
  k_put_seq<<<1, 32, 0, st>>>(c->v, key_a, key_b, n, w, pw, c->record, par ? 1 : 0);
  k_hash_erase<<<grid_for(h.entries + n + 1, 256), 256, 0, st>>>(c->v, w);
  k_install_put<<<grid_for(n * 32, 256), 256, 0, st>>>(c->v, w, pw, key_a, key_b, src_rows);
  FX_LAUNCH_CHECK("fx_cache_pooled_put");
  rc = read_scalars(c, &h, st);
  if (rc) return rc;
  if ((h.hash_tomb + h.entries) * 2 > c->v.hcap) {
    k_fill_u64<<<grid_for(c->v.hcap, 256), 256, 0, st>>>(c->v.hkeys, c->v.hcap, kEmpty);
    k_index_rebuild<<<grid_for(c->v.scap, 256), 256, 0, st>>>(c->v);
    cudaMemsetAsync(&c->v.sc->hash_tomb, 0, sizeof(long long), st);
    FX_LAUNCH_CHECK("fx_cache index rebuild");
  }
  return FX_OK;
}

int fx_cache_set_parallel(fx_cache *c, int32_t on) {
  c->parallel_offers = on ? 1 : 0;
  return FX_OK;
}

int fx_cache_last_evicted(fx_cache *c, uint64_t *out, int64_t cap, int64_t *n_out, void *stream) {
  cudaStream_t st = as_stream(stream);
  Scalars h;
  int rc = read_scalars(c, &h, st);
  if (rc) return rc;
  const int64_t n = h.n_ev < cap ? h.n_ev : cap;
  if (n > 0 && c->last_ev) cudaMemcpyAsync(out, c->last_ev, n * 8, cudaMemcpyDeviceToDevice, st);
  *n_out = n;
  return cuda_check(cudaStreamSynchronize(st), "fx_cache_last_evicted");
}

int fx_cache_set_pending_rows(fx_cache *c, const float *const *rows, int64_t n) {
  (void)n;
  c->pending_rows = rows;
  return FX_OK;
}

}  // extern "C"
