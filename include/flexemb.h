/*
 * flexemb.h — C-ABI of the B200-native embedding-lookup path (libflexemb.so).
 *
 * Drop-in boundary for the hot path of the reference `embserve` package
 * (FlexEMR, arXiv 2410.12794; paths below are relative to
 * /root/reference/pkg/src/embserve). The reference has no FFI: its seams are
 * Python module APIs. Each entry point below names the reference function
 * whose semantics it replaces; the Python mirror package
 * (paper_2410_12794_b200) binds these through ctypes.
 *
 * Conventions
 *  - plain C types only; every device buffer is caller-owned device memory
 *    (e.g. a torch CUDA tensor's data_ptr()); no allocation on the hot path
 *    except where a `workspace` is documented;
 *  - every call is asynchronous on the given stream (a cudaStream_t passed
 *    as void*; NULL = legacy default stream) unless marked [sync];
 *  - return codes map 1:1 onto embserve/errors.py:4-41 (see FX_E_*);
 *    fx_last_error() returns a thread-local message for the last failure;
 *  - handles are thread-compatible, not thread-safe (one host thread drives
 *    one handle and stream), like the reference's single-writer cache
 *    (SPEC.md:306).
 */
#ifndef FLEXEMB_H
#define FLEXEMB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes (errors.py:4-41) ------------------------------------ */
#define FX_OK 0
#define FX_E_CONFIG 1             /* ConfigError            errors.py:8   */
#define FX_E_LOOKUP_VALIDATION 2  /* LookupValidationError  errors.py:13  */
#define FX_E_ROUTING_VIOLATION 3  /* RoutingViolationError  errors.py:18  */
#define FX_E_CAPACITY 4           /* CapacityError          errors.py:23  */
#define FX_E_INVARIANT 5          /* InvariantError         errors.py:40  */
#define FX_E_EMPTY 6              /* EmbServeError (empty pool/combine)   */
#define FX_E_CUDA 7               /* EmbServeError (device failure)       */

/* ---- enums -------------------------------------------------------------- */
#define FX_OP_SUM 0               /* PoolingOp.SUM   pooling.py:25-27 */
#define FX_OP_MEAN 1              /* PoolingOp.MEAN */

#define FX_IDX_I32 0              /* index element type */
#define FX_IDX_I64 1

#define FX_OUT_F32 0              /* final pooled f32 (Mean divided once)        */
#define FX_OUT_F64_PARTIAL 1      /* f64 partial sum (Mean deferred), see counts */
#define FX_OUT_F32_PARTIAL 2      /* f64-accumulated partial sum rounded to f32 (Mean deferred):
                                     PartialResult.vector semantics, pooling.py:35-47 */
#define FX_OUT_SYSFENCE 16        /* OR-flag: system-scope fence after the epilogue stores
                                     (outputs written to peer GPUs over NVLink)        */
#define FX_OUT_SCALAR 32          /* OR-flag: scalar kernel (a segment's table / output pointer, ld or
                                     out_stride is not 16-byte aligned) */
#define FX_OUT_SHARE 64           /* OR-flag: the launch shares the GPU with a concurrent stream (the
                                     one-wave gather kernels keep at most 2 resident blocks per SM) */
/* In both partial modes an EMPTY bag's output row is not written (its count
 * is 0: the partial is absent and K5 never reads it). */

const char *fx_last_error(void);
int fx_version(void);
int fx_num_sms(int device);
/* Bounds-checked builds (FX_BOUNDS, libflexemb_chk.so; compute-sanitizer
 * stand-in): out4 = {violations, array base, first bad index, array length}
 * on the current device; returns 1, 0 for a normal build (out4 untouched),
 * -1 on a CUDA error. No reference counterpart (test infrastructure). */
int fx_bounds_report(int64_t *out4);
/* FX_BOUNDS builds: launch a kernel that reads a checked 4-element array at
 * index 5 and verify the record caught it (then clear it): 1 = the checks are
 * live, 0 = normal build, -1 = not caught. */
int fx_bounds_selftest(void);

/* ---- K0: table materialisation (store.py:62-89 table_block/_table_base) --
 * out[r*ld + c] = f32(((mix64(base_t + (row_start+r)*dim + c) >> 11) * 2^-53)
 *                 * 2 - 1),  base_t = mix64(table_id ^ mix64(seed)).
 * Bit-exact with the reference PRF. */
int fx_table_init(float *out, int64_t ld, uint64_t seed, int64_t table_id,
                  int32_t dim, int64_t row_start, int64_t n_rows, void *stream);
uint64_t fx_table_base(uint64_t seed, int64_t table_id); /* host helper */

/* ---- bag segments ---------------------------------------------------------
 * A batch is CSR bags (offsets[n_bags+1], indices[nnz]) grouped into
 * segments: contiguous bag ranges that read one shard of one table with one
 * pooling op. Row r of the shard lives at table + (r - row_begin)*ld. */
typedef struct fx_segment {
  const float *table;   /* device shard base                                  */
  int64_t row_begin;    /* first hosted row (global row id)                   */
  int64_t row_end;      /* one past the last hosted row                       */
  int64_t bag_begin;    /* first bag of this segment                          */
  int64_t bag_end;      /* one past the last bag                              */
  void *out;            /* output base (float* or double*, see out mode)      */
  int64_t out_stride;   /* elements between consecutive bags' outputs         */
  int64_t ld;           /* elements between consecutive shard rows (>= dim)   */
  int32_t dim;          /* embedding dimension                                */
  int32_t op;           /* FX_OP_*                                            */
  const void *idx;      /* optional: indices base for this segment's bags (may be a peer/IPC
                           pointer); NULL -> the launch's `indices`                          */
  const int64_t *offs;  /* optional: offsets of this segment's bags, offs[b - bag_begin] ..
                           offs[b - bag_begin + 1] index into `idx`; NULL -> launch offsets  */
} fx_segment;

/* ---- K4: fused gather + pool (store.py:184-193 partial_pool,
 *      pooling.py:60-85 sum_rows_f64/pool_flat, ranker.py:458-465) --------
 * For every bag: f64 accumulation of its rows in index order (each lane owns
 * columns, so the per-element summation order is exactly the reference's
 * sequential order), then
 *   FX_OUT_F32:         emit f32 (Mean divides the f64 sum by the bag length
 *                       once, pooling.py:82-84); empty bag -> zeros;
 *   FX_OUT_F64_PARTIAL: emit the f64 sum; counts[bag] = bag length
 *                       (PartialResult(sum, count), pooling.py:35-47).
 * Indices outside [row_begin,row_end) are never dereferenced: the first bad
 * occurrence's CSR position is atomically min-recorded in err[0] (init it to
 * INT64_MAX) and err_code (if non-NULL) is set to `bad_code`
 * (FX_E_LOOKUP_VALIDATION at ingress, FX_E_ROUTING_VIOLATION on a shard).
 * `segs` is a DEVICE array; all segments must share one dim (host groups by
 * dim). `counts` may be NULL. */
int fx_gather_pool(const fx_segment *segs, int32_t n_segs, int32_t dim,
                   const void *indices, int32_t idx_type, const int64_t *offsets,
                   int64_t n_bags, int32_t out_mode, int32_t *counts,
                   int64_t *err, int32_t bad_code, int32_t *err_code, void *stream);

/* ---- raw row gather (store.py:151-182 lookup_rows) ---------------------
 * out[i*dim + c] = shard[indices[i] - row_begin][c], input order,
 * duplicates per occurrence; unhosted index -> err/err_code as above. */
int fx_gather_rows(const float *table, int64_t ld, int64_t row_begin, int64_t row_end,
                   int32_t dim, const void *indices, int32_t idx_type, int64_t n,
                   float *out, int64_t *err, int32_t *err_code, void *stream);

/* ---- K5: combine (pooling.py:103-123 combine_partials) ------------------
 * out[b] = f32( sum_{s=0..n_src-1} partials[s][b] (f64, ascending s)
 *               + sum_{k} raw rows of bag b in position order (f64) )
 * Mean divides by (sum_s counts[s][b] + raw count) once.
 * partials: device array of n_src pointers to [n_bags, dim] f64 (f32 when
 * partial_is_f32: each partial already rounded once, as PartialResult) (row stride
 * p_stride); counts: n_src pointers to int32[n_bags] (NULL -> partial absent
 * for every bag). raw_offsets/raw_rows: optional CSR of f32 raw vectors
 * (raw_rows row stride = dim), may be NULL. When dim % 4 == 0 the kernel
 * reads and writes 16-byte vectors: partial rows, raw rows and out rows must
 * then start on 16-byte boundaries. ops: int32[n_bags] or NULL (all
 * `op`). out row stride = out_stride. Bags with nothing to combine get
 * zeros and set *err_code = FX_E_EMPTY if err_code != NULL. */
int fx_combine(const void *const *partials, int32_t partial_is_f32, const int32_t *const *counts, int32_t n_src,
               int64_t p_stride, const int64_t *raw_offsets, const float *raw_rows,
               int64_t n_bags, int32_t dim, int32_t op, const int32_t *ops,
               float *out, int64_t out_stride, int32_t *err_code, void *stream);
/* fx_combine with raw vectors given as row pointers (raw_ptrs[r], e.g. rows
 * in a peer GPU's shard read over NVLink; NULL = none) instead of a packed
 * raw_rows array. sample_major_B > 0: bags are table-major (b = f*B + s) and
 * bag b is written to out + s * out_stride + f * dim, i.e. straight into a
 * sample-major [B, F*dim] batch output; 0: out + b * out_stride. */
int fx_combine_ptr(const void *const *partials, int32_t partial_is_f32, const int32_t *const *counts, int32_t n_src,
                   int64_t p_stride, const int64_t *raw_offsets, const float *const *raw_ptrs, int64_t n_bags,
                   int32_t dim, int32_t op, const int32_t *ops, float *out, int64_t out_stride, int32_t *err_code,
                   int64_t sample_major_B, void *stream);

/* ---- K1: range routing (routing.py:87-97 resolve_many, 117-148) ---------
 * For occurrence i of a bag of table t:
 *   shard = upper_bound(starts[route_off[t]..route_off[t+1]), idx) - 1
 *   dest[i] = servers[route_off[t] + shard]
 * bag_table[n_bags] gives the table per bag; num_rows[t] bounds validation
 * (bad -> err/err_code FX_E_LOOKUP_VALIDATION). dest may be NULL (validate only). */
int fx_route(const int64_t *route_off, const int64_t *starts, const int32_t *servers,
             const int64_t *num_rows, const int32_t *bag_table, const void *indices,
             int32_t idx_type, const int64_t *offsets, int64_t n_bags, int32_t *dest,
             int64_t *err, int32_t *err_code, void *stream);

/* Stable per-destination bucketing (routing.py:117-148 group_by_server,
 * GroupItem.positions): given dest[nnz] in CSR (bag, position) order, produce
 *   perm[nnz]        CSR positions ordered by (dest, bag, position)
 *   dest_count[n_dest]  occurrences per destination
 *   bag_count[n_dest*n_bags] occurrences of bag b routed to dest d.
 * Requires n_dest <= 256. workspace: query with ws == NULL (*ws_bytes set). */
int fx_bucket(const int32_t *dest, int64_t nnz, const int64_t *offsets, int64_t n_bags,
              int32_t n_dest, int64_t *perm, int64_t *dest_count, int32_t *bag_count,
              void *ws, size_t *ws_bytes, void *stream);

/* ---- K2: per-batch dedup (no reference counterpart) ---
 * keys[i] = bag_table[bag(i)] << 40 | row(i) for every occurrence in CSR
 * order; ordinal[i] = the occurrence's (lookup, feature, position) ordinal
 * (sm_start[bag] + position). Produces, deterministically, the unique keys
 * in FIRST-OCCURRENCE (ordinal) order:
 *   uniq[n_uniq], mult[n_uniq] (multiplicity), first_ord / last_ord[n_uniq],
 *   inverse[nnz] (unique id per occurrence), *n_uniq_dev (device int64).
 * Sorting uniq reproduces np.unique exactly. workspace: query with ws==NULL. */
int fx_dedup(const int32_t *bag_table, const void *indices, int32_t idx_type,
             const int64_t *offsets, const int64_t *sm_start, int64_t n_bags, int64_t nnz,
             uint64_t *uniq, int32_t *mult, int64_t *first_ord, int64_t *last_ord,
             int32_t *inverse, int64_t *n_uniq_dev, void *ws, size_t *ws_bytes, void *stream);


/* ---- K3/K6: GPU hot-row cache (cache.py:114-352 AdaptiveCache +
 *      FrequencySketch) ------------------------------------------------------
 * Keys are u64 (table << 40 | row). The handle owns its device memory
 * (cudaMalloc at create / reserve; documented exception to "no allocation").
 * Scalars (fx_cache_scalars order, 21 x int64): budget, used, tick, hits,
 * misses, entries, free_top, sketch_live, sketch_tomb, hash_tomb, pending,
 * n_evlog, n_acc, n_ev, n_cand, staged, err, n_ov, n_par_puts, tiles_bulk,
 * tiles_chain (offer-resolution statistics). err: 1 = an insert or
 * shrink found nothing left to evict (the reference raises KeyError from
 * OrderedDict.popitem there), 2 = pooled-key fingerprint collision.
 * Calls marked [sync] read scalars back to the host. */
typedef struct fx_cache fx_cache;
typedef struct fx_table_dir {   /* where rows of `table` in [row_begin,row_end) live */
  const float *base;
  int64_t row_begin;
  int64_t row_end;
  int64_t ld;
  int32_t table;
  int32_t dim;
} fx_table_dir;

/* admission 0 = "sketch", 1 = "always" (cache.py:164-186) */
int fx_cache_create(fx_cache **out, int64_t slot_capacity, int32_t max_dim, int32_t admission, double decay,
                    double prune_below, int64_t budget_bytes, int64_t sketch_capacity, int32_t record_evictions);
int fx_cache_destroy(fx_cache *c);
int fx_cache_set_tables(fx_cache *c, const fx_table_dir *dir, int32_t n_dir, const int32_t *table_bytes,
                        int32_t n_tables);                                     /* host arrays */
int fx_cache_scalars(fx_cache *c, int64_t *out21, void *stream);               /* [sync] */
const void *fx_cache_scalars_device(fx_cache *c);  /* the 21 scalars in device memory (async snapshots) */
int fx_cache_capacity(fx_cache *c, int64_t *out3);  /* slot, index and sketch table capacities */
int fx_cache_queue_valid(fx_cache *c);  /* 1 while the fused step's LRU queue / dense index are current */
int fx_cache_reserve_sketch(fx_cache *c, int64_t new_keys, void *stream);      /* [sync] */
int fx_cache_reserve_slots(fx_cache *c, int64_t slots, void *stream);          /* [sync] */
/* get() per unique key (cache.py:189-202): hit -> last_tick = tick0 +
 * last_ord + 1, hits += mult; miss -> sketch += mult, misses += mult;
 * tick += nnz. n_uniq from device (n_uniq_dev) or host. slot_out: slot|-1 */
int fx_cache_probe(fx_cache *c, const uint64_t *uniq, const int32_t *mult, const int64_t *last_ord,
                   const int64_t *n_uniq_dev, int64_t n_uniq_host, int64_t nnz, int32_t *slot_out, void *stream);
/* ordered offers (cache.py:237-268); rows from src_rows[j] or the table dir  [sync] */
int fx_cache_offer(fx_cache *c, const uint64_t *keys, int64_t n, const int32_t *sizes,
                   const float *const *src_rows, uint8_t *accepted, void *stream);
/* resize: new budget; shrink evicts LRU to fit (cache.py:290-309)        [sync] */
int fx_cache_set_budget(fx_cache *c, int64_t budget, void *stream);
/* stage_hot_admissions(limit; -1 = None) (cache.py:311-342)                [sync] */
int fx_cache_stage(fx_cache *c, int64_t limit, int64_t *staged, void *stream);
/* apply_pending_admissions (cache.py:344-352)                             [sync] */
int fx_cache_apply_pending(fx_cache *c, int64_t *applied, void *stream);
/* FrequencySketch.age (cache.py:128-136) */
int fx_cache_age(fx_cache *c, void *stream);
int fx_cache_lookup(fx_cache *c, const uint64_t *keys, int64_t n, float *rows_out, int32_t out_ld,
                    int32_t *slot_out, void *stream);
int fx_cache_sketch_estimate(fx_cache *c, const uint64_t *keys, int64_t n, double *out, void *stream);
int fx_cache_sketch_bump(fx_cache *c, const uint64_t *keys, const double *weights, int64_t n, void *stream);
/* FrequencySketch.hottest order (-count, key), device outputs            [sync] */
int fx_cache_sketch_ranked(fx_cache *c, uint64_t *keys_out, double *vals_out, int64_t cap, int64_t *n_out,
                           void *stream);
/* entries in LRU order (ascending last_tick), device outputs            [sync] */
int fx_cache_lru(fx_cache *c, uint64_t *keys_out, int64_t *ticks_out, int32_t *hits_out, int64_t cap,
                 int64_t *n_out, void *stream);
int fx_cache_eviction_log(fx_cache *c, uint64_t *out, int64_t cap, int64_t *n_out, void *stream); /* [sync] */
int fx_cache_pending(fx_cache *c, uint64_t *out, int64_t cap, int64_t *n_out, void *stream);      /* [sync] */
/* 1 (default): resolve ordered offers with the exact run-parallel kernel when
 * every row has one size; 0: always use the sequential reference loop */
int fx_cache_set_parallel(fx_cache *c, int32_t on);
/* keys evicted by the last offer / apply / set_budget call                 [sync] */
int fx_cache_last_evicted(fx_cache *c, uint64_t *out, int64_t cap, int64_t *n_out, void *stream);
/* device array of row pointers for the pending keys (NULL entry -> table dir),
 * consumed by the next fx_cache_apply_pending (host-fetched admissions) */
int fx_cache_set_pending_rows(fx_cache *c, const float *const *rows, int64_t n);
/* device base of the cache's row storage and its row stride in floats
 * (valid until the next fx_cache_reserve_slots) */
int fx_cache_rows(fx_cache *c, const float **rows, int64_t *ld);
/* tick += n (the batch's probes when no row probe call advances it) */
int fx_cache_advance_tick(fx_cache *c, int64_t n, void *stream);

/* ---- pooled-result keyspace (cache.py:204-223; ranker.py:243-249,412-414) ----
 * Key of a bag = ("pooled", table, op, sorted(indices)), represented by two
 * 64-bit multiset fingerprints (fx_bag_fingerprint):
 *   sA = sum mix64(x ^ 0xA0761D6478BD642F), sB = sum mix64(x ^ 0xE7037ED1A0B428DB)  (mod 2^64)
 *   A = mix64(sA ^ mix64(mix64(table ^ SALT_A) + op) ^ (L * SALT_B)) | 2^63
 *   B = mix64(sB ^ mix64(mix64(table ^ SALT_B) + op) ^ (L * SALT_A))
 * A indexes the shared LRU / budget (disjoint from row keys), B is verified on
 * every match (mismatch -> scalars.err = 2). */
int fx_bag_fingerprint(const int32_t *bag_table, const int32_t *bag_op, const void *indices, int32_t idx_type,
                       const int64_t *offsets, int64_t n_bags, uint64_t *key_a, uint64_t *key_b, void *stream);
/* slot of each pooled key (-1 absent); no state change */
int fx_cache_pooled_find(fx_cache *c, const uint64_t *key_a, const uint64_t *key_b, int64_t n, int32_t *slot_out,
                         void *stream);
/* pooled_get hits: last_tick = tick + pos[i] + 1 (max per slot), hits += 1;
 * the tick is advanced by the caller (fx_cache_probe nnz / advance_tick) */
int fx_cache_pooled_touch(fx_cache *c, const int32_t *slot, const int64_t *pos, int64_t n, void *stream);
/* out[i] = cached row of slot[i] (rows with slot -1 untouched); optional
 * size_out[i] = the entry's bytes (0 for slot -1) */
int fx_cache_read_slots(fx_cache *c, const int32_t *slot, int64_t n, float *out, int32_t out_ld, int32_t *size_out,
                        void *stream);
/* ordered pooled_put of n vectors src_rows[j] (device array of device
 * pointers), sizes[j] bytes (or uniform_size when sizes == NULL): evict LRU to
 * fit, fresh tick, insert at MRU; a resident key is replaced in place
 * (position kept, used += size again: the reference's _insert quirk).  [sync] */
int fx_cache_pooled_put(fx_cache *c, const uint64_t *key_a, const uint64_t *key_b, int64_t n, const int32_t *sizes,
                        int32_t uniform_size, const float *const *src_rows, void *stream);

/* ---- peer memory (NVLink P2P over CUDA IPC) and the cross-GPU barrier ----
 * The fused exchange: an owner's K4 reads a requester's CSR batch through an
 * IPC-mapped pointer and stores pooled rows straight into the requester's
 * output buffer, so the pooled "all-to-all" rides on the gather's own stores
 * (replaces ranker.py:298-347 post_subrequest/_on_response). */
int fx_dev_alloc(size_t bytes, void **out);                       /* cudaMalloc (IPC-exportable) */
int fx_dev_free(void *ptr);
int fx_ipc_export(void *ptr, unsigned char handle_out[64]);      /* cudaIpcGetMemHandle */
int fx_ipc_open(const unsigned char handle[64], void **out);     /* cudaIpcOpenMemHandle */
int fx_ipc_close(void *ptr);
int fx_can_access_peer(int device, int peer_device);
int fx_memcpy_async(void *dst, const void *src, size_t bytes, void *stream);
/* table-wise push: the requester copies, for every feature f, its bag range
 * (indices as int32 + offsets rebased to the owner's slot) into the staging
 * of feature f's owner (dst_idx[d] / dst_offs[d]: DEVICE arrays of IPC-mapped
 * pointers to THIS requester's slot in rank d's staging). feat_pos[f] = rank
 * of f among its owner's features (ascending f). With feat_nrows (device,
 * [F]: rows of feature f's table) the copy also performs the ingress
 * validation of fx_route (routing.py:87-101): an index outside
 * [0, feat_nrows[f]) records its position in *err (atomic min) and
 * FX_E_LOOKUP_VALIDATION in *err_code. */
int fx_push_csr(const void *indices, int32_t idx_type, const int64_t *offsets, int32_t B, int32_t F,
                const int32_t *feat_owner, const int32_t *feat_pos, int32_t *const *dst_idx, int64_t *const *dst_offs,
                const int64_t *feat_nrows, int64_t *err, int32_t *err_code, int32_t sysfence, void *stream);
/* row-wise push: counts[d*n_bags+b] (int32, W*n_bags+1 entries) = indices of
 * bag b routed to rank d (K1 range routing); scan = exclusive prefix over
 * (d, b); then every index is scattered, stable per destination, into rank
 * d's staging slot dst_idx[d] (int32) and rank d's per-bag offsets
 * dst_offs[d][0..n_bags] are written (IPC-mapped pointers, DEVICE arrays).
 * workspace: query with ws == NULL. */
int fx_rw_push(const int64_t *route_off, const int64_t *starts, const int32_t *owners, const int32_t *bag_table,
               const void *indices, int32_t idx_type, const int64_t *offsets, int64_t n_bags, int32_t W,
               int32_t *counts, int64_t *scan, int32_t *const *dst_idx, int64_t *const *dst_offs, void *ws,
               size_t *ws_bytes, void *stream);
/* planned row-wise push (pooling.py:88-100 plan_hierarchical per (bag,
 * rank), ranker.py:263-301): counts as fx_rw_push; a (bag, rank) group of
 * >= threshold indices is pushed to the owner (pushdown, its counts entry
 * kept for K5), a smaller group is RAW-FETCHED: its count is zeroed and each
 * of its indices gets raw_ptr[raw_off[b] + k] (position order within the bag)
 * = the row's address in the owning shard, shard_base[sid] + (idx -
 * starts[sid]) * ld — an IPC-mapped peer pointer for other ranks' shards,
 * read by fx_combine_ptr over NVLink. raw_off: int64[n_bags+1]; raw_ptr:
 * capacity nnz; counters (optional): int32[3][n_bags] = pushdown_groups,
 * pushdown_rows, raw_rows per bag. hit_slot (optional, int32 per
 * occurrence): occurrences with a cache slot >= 0 are served by the
 * requester's cache — excluded from the groups, and joined to the raw list at
 * their position as cache_rows + slot * cache_ld (cache hits combine as raw
 * vectors, ranker.py:409-411). workspace: query with ws == NULL. */
int fx_rw_push_planned(const int64_t *route_off, const int64_t *starts, const int32_t *owners, const int64_t *nrows,
                       const int32_t *bag_table, const void *indices, int32_t idx_type, const int64_t *offsets,
                       int64_t n_bags, int32_t W, int32_t threshold, int32_t *counts, int64_t *scan,
                       int32_t *const *dst_idx, int64_t *const *dst_offs, const float *const *shard_base, int64_t ld,
                       int64_t *raw_off, const float **raw_ptr, int32_t *counters, const int32_t *hit_slot,
                       const float *cache_rows, int64_t cache_ld, void *ws, size_t *ws_bytes, void *stream);
/* one-block barrier: release-store `epoch` into peer_flags[r][rank] for every
 * rank r (system scope, after a system fence), then acquire-spin until
 * my_flags[r] >= epoch for every r. peer_flags is a DEVICE array of `world`
 * pointers (IPC-mapped flag arrays; own entry = my_flags). Spins are bounded
 * (~10 s); on timeout *timed_out (device int32, may be NULL) is set to 1. */
int fx_peer_barrier(int64_t *my_flags, int64_t *const *peer_flags, int32_t rank, int32_t world, int64_t epoch,
                    int32_t *timed_out, void *stream);


/* ---- fused per-batch cache step (fx_step.cu) ------------------------------
 * One Ranker batch's locality layer with no host synchronisation
 * (ranker.py:218-442 + cache.py:189-352 in the canonical order of SURVEY
 * §8(c)): apply_pending_admissions -> validation + dedup -> probe -> plan
 * (pushdown threshold, 0 = None) -> offers of raw-fetched misses; then
 * fx_step_maintain: stage_hot_admissions(limit) -> sketch age. Domain: row
 * keys of one entry size (dim*4 bytes) for every table, one shard per table
 * on this GPU, no pooled-result keyspace. Errors raised on the device (bad
 * index -> LookupValidationError, sketch capacity -> CapacityError) are read
 * back with fx_step_scalars; a rejected batch leaves the cache untouched.
 * Capturable in a CUDA graph once fx_step_prepare has run. */
typedef struct fx_step fx_step;
/* `slots` batches may be in flight (RankerParams.pipeline_depth): start(k)
 * runs apply_pending + validation + probes of batch k, offer(k) its offers,
 * maintain(k) stage + age; the reference interleaves them as S0 S1 F0 S2 F1
 * ... (ranker.py:161-182), each phase reading the cache as it is then. */
int fx_step_create(fx_step **out, fx_cache *cache, int64_t max_nnz, int64_t max_bags, const float *const *table_base,
                   const int64_t *table_ld, const int64_t *table_rows, int32_t n_tables, int32_t dim,
                   int64_t stage_limit_cap, int32_t slots);                     /* [sync] */
int fx_step_destroy(fx_step *s);
int fx_step_prepare(fx_step *s, void *stream);  /* LRU queue (re)build when another call moved entries */
int fx_step_start(fx_step *s, int32_t slot, const int32_t *bag_table, const void *indices, int32_t idx_type,
                  const int64_t *offsets, const int64_t *sm_start, int64_t n_bags, int64_t nnz, int32_t threshold,
                  int32_t *hits_bag, int32_t *pd_groups, int32_t *pd_rows, int32_t *raw_rows, void *stream);
int fx_step_offer(fx_step *s, int32_t slot, void *stream);
int fx_step_maintain(fx_step *s, int32_t slot, int64_t stage_limit, int32_t do_age, void *stream);
int fx_step_scalars(fx_step *s, int32_t slot, int64_t *out, int64_t n, void *stream);   /* [sync] */
const void *fx_step_scalars_device(fx_step *s, int32_t slot);
int64_t fx_step_launches(fx_step *s);  /* kernels launched by this handle so far (CUB sweeps count 2) */
/* Make `stream` wait for the step's side-stream work (the accepts' row
 * copies, forked by fx_step_offer and otherwise joined at the end of
 * fx_step_maintain / the next start or offer). Call it before touching the
 * cache through any other entry point, or at the end of a captured batch
 * that has no maintenance. No reference counterpart (stream plumbing). */
int fx_step_join(fx_step *s, void *stream);


/* ---- store (fx_store_create / fx_store_shard_view) ------------
 * The shards a placement assigns to `my_rank`, allocated on `device` (row-major
 * [end-start, dim] f32, ld = dim rounded up to 4) and materialised by K0 with
 * the reference PRF (store.py:62-89, 228-251); the placement is validated
 * like validate_placement (store.py:92-119: overlap / gap / end -> FX_E_CONFIG). */
typedef struct fx_store fx_store;
typedef struct fx_shard_desc { int32_t table; int32_t owner; int64_t start; int64_t end; } fx_shard_desc;
int fx_store_create(fx_store **out, int32_t device, int32_t n_tables, const int64_t *rows, const int32_t *dims,
                    int32_t n_shards, const fx_shard_desc *shards, int32_t my_rank, uint64_t seed, void *stream);
int fx_store_destroy(fx_store *s);
/* zero-copy view of the local shard holding (table, row); FX_E_ROUTING_VIOLATION when not hosted here */
int fx_store_shard_view(fx_store *s, int32_t table, int64_t row, const float **base, int64_t *start, int64_t *end,
                        int64_t *ld, int32_t *dim);
/* [sync] read a kernel's device status pair (first bad position, FX_E_* code) */
int fx_poll_error(const int32_t *err_code, const int64_t *err_pos, int32_t *code, int64_t *pos, void *stream);
/* ---- communicator (fx_comm_init / fx_alltoallv) -------------
 * The fan-out / response seam (ranker.py:263-347: post_subrequest ->
 * _server_handler -> _on_response) as a byte all-to-allv over CUDA-IPC-mapped
 * peer memory of one node, no NCCL: every rank owns a double-buffered window of
 * `world` slots of `slot_bytes`; fx_alltoallv stores rank r's slice for d
 * (send + send_displs[d], send_counts[d] bytes; device arrays) into slot r of
 * d's window and its count next to it, then the ranks meet in a
 * release/acquire peer barrier. Setup: fx_comm_init on every rank,
 * fx_comm_handle -> exchange the 64-byte handles out of band (e.g. a
 * torch.distributed all_gather) -> fx_comm_connect(world x 64 bytes). After
 * an exchange, fx_comm_recv_buffer / fx_comm_recv_counts give this rank's
 * received slots (valid until the next-but-one exchange; consume them on the
 * same stream). The exchange epoch is host-side: not for CUDA-graph capture.
 * sharded.P2PShardedLookup fuses the same one-sided stores into the push and
 * gather kernels instead (fx_push_csr / fx_rw_push* / K4 epilogue). */
typedef struct fx_comm fx_comm;
int fx_comm_init(fx_comm **out, int32_t rank, int32_t world, int64_t slot_bytes);
int fx_comm_handle(fx_comm *c, unsigned char handle_out[64]);
int fx_comm_connect(fx_comm *c, const unsigned char *handles);
int fx_alltoallv(fx_comm *c, const void *send, const int64_t *send_counts, const int64_t *send_displs, void *stream);
void *fx_comm_recv_buffer(fx_comm *c);
const int64_t *fx_comm_recv_counts(fx_comm *c);
int fx_comm_status(fx_comm *c, int32_t *overflow, int32_t *timed_out);  /* [sync] slot overflow / barrier timeout */
int fx_comm_destroy(fx_comm *c);

#ifdef __cplusplus
}
#endif
#endif /* FLEXEMB_H */
