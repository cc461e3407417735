// K0 table materialisation, K4 fused gather+pool, raw gather, K5 combine.
//
// Reference semantics (paths under /root/reference/pkg/src/embserve):
//   table_block / _table_base / _mix64      store.py:62-89
//   ServerStore.lookup_rows                 store.py:151-182
//   ServerStore.partial_pool, sum_rows_f64  store.py:184-193, pooling.py:60-71
//   pool_flat                               pooling.py:74-85
//   combine_partials                        pooling.py:103-123
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>
#include <cstdlib>
#include <mutex>

#include "fx_common.cuh"
#include "fx_pool_async.cuh"

namespace fx {

// ----------------------------------------------------------------- K0
// One warp per row, lanes stride the columns: coalesced stores, integer
// SplitMix64 + exact f64 scaling + one RN rounding to f32 (bit-exact).
__global__ void __launch_bounds__(256) k_table_init(float *__restrict__ out, int64_t ld, uint64_t base,
                                                    int32_t dim, int64_t row_start, int64_t n_rows) {
  const int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t r = w; r < n_rows; r += nw) {
    const uint64_t ctr0 = static_cast<uint64_t>(row_start + r) * static_cast<uint64_t>(dim) + base;
    float *dst = out + r * ld;
    for (int c = lane; c < dim; c += 32) {
      const uint64_t bits = mix64(ctr0 + static_cast<uint64_t>(c));
      const double unit = static_cast<double>(bits >> 11) * 0x1p-53;
      dst[c] = __double2float_rn(unit * 2.0 - 1.0);  // both ops exact; one rounding
    }
  }
}

// ----------------------------------------------------------------- K4
// Vectorised path: rows are 16-B aligned (dim % 4 == 0, ld % 4 == 0).
// A group of G lanes owns one bag; lane gl owns columns (k*G + gl)*4 .. +3 for
// k < NCH, so every output element is accumulated over the bag's rows in
// index order (the reference's sequential order) in f64. Indices are staged
// G at a time (one coalesced load), broadcast by shuffle, and U row loads
// are issued before any accumulation to keep U*16 B per lane in flight.
template <int G, int NCH, int U, typename IdxT, int MODE>
__global__ void __launch_bounds__(256) k_gather_pool_v4(
    const fx_segment *__restrict__ segs, int n_segs, int dim, const IdxT *__restrict__ indices_g,
    const int64_t *__restrict__ offsets, int64_t n_bags, int32_t *__restrict__ counts,
    int64_t *err, int32_t bad_code, int32_t *err_code, bool sysfence) {
  constexpr int GPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const int gw = lane / G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gw * G));
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;

  for (int64_t bag = warp * GPW + gw; bag < n_bags; bag += nwarps * GPW) {
    const int s = find_segment(segs, n_segs, bag);
    const float *__restrict__ tab = segs[s].table;
    const int64_t rb = segs[s].row_begin, re = segs[s].row_end, ld = segs[s].ld;
    int64_t beg, end;
    bag_bounds(segs, s, bag, offsets, beg, end);
    const IdxT *indices = seg_indices(segs, s, indices_g);

    double acc[NCH][4];
#pragma unroll
    for (int k = 0; k < NCH; ++k) acc[k][0] = acc[k][1] = acc[k][2] = acc[k][3] = 0.0;

    for (int64_t c0 = beg; c0 < end; c0 += G) {
      const int n = static_cast<int>((end - c0 < G ? end - c0 : (int64_t)G));
      int64_t my_off = 0;
      if (gl < n) {
        const int64_t idx = load_index(indices + c0 + gl);
        if (idx < rb || idx >= re) {
          record_bad(err, err_code, c0 + gl, bad_code);
        } else {
          my_off = (idx - rb) * ld;
        }
      }
      for (int r = 0; r < n; r += U) {
        float4 v[U][NCH];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t off = __shfl_sync(gmask, my_off, (r + u) & (G - 1), G);
          if (r + u < n) {
#pragma unroll
            for (int k = 0; k < NCH; ++k) {
              const int col = (k * G + gl) * 4;
              if (NCH == 1 || col < dim) v[u][k] = ldg_f4(tab + off + col);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (r + u < n) {
#pragma unroll
            for (int k = 0; k < NCH; ++k) {
              acc[k][0] += static_cast<double>(v[u][k].x);
              acc[k][1] += static_cast<double>(v[u][k].y);
              acc[k][2] += static_cast<double>(v[u][k].z);
              acc[k][3] += static_cast<double>(v[u][k].w);
            }
          }
        }
      }
    }

    const int64_t cnt = end - beg;
    const int64_t orow = bag - segs[s].bag_begin;
    if (MODE == FX_OUT_F32) {
      float *o = static_cast<float *>(segs[s].out) + orow * segs[s].out_stride;
      const bool mean = segs[s].op == FX_OP_MEAN && cnt > 0;
      const double dn = static_cast<double>(cnt);
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        const int col = (k * G + gl) * 4;
        if (NCH == 1 || col < dim) {
          float4 q;
          if (mean) {
            q = make_float4(__double2float_rn(acc[k][0] / dn), __double2float_rn(acc[k][1] / dn),
                            __double2float_rn(acc[k][2] / dn), __double2float_rn(acc[k][3] / dn));
          } else {
            q = make_float4(__double2float_rn(acc[k][0]), __double2float_rn(acc[k][1]),
                            __double2float_rn(acc[k][2]), __double2float_rn(acc[k][3]));
          }
          *reinterpret_cast<float4 *>(o + col) = q;
        }
      }
    } else if (MODE == FX_OUT_F32_PARTIAL) {
      float *o = static_cast<float *>(segs[s].out) + orow * segs[s].out_stride;
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        const int col = (k * G + gl) * 4;
        if (NCH == 1 || col < dim)
          *reinterpret_cast<float4 *>(o + col) =
              make_float4(__double2float_rn(acc[k][0]), __double2float_rn(acc[k][1]),
                          __double2float_rn(acc[k][2]), __double2float_rn(acc[k][3]));
      }
      if (counts && gl == 0) counts[bag] = static_cast<int32_t>(cnt);
    } else {
      double *o = static_cast<double *>(segs[s].out) + orow * segs[s].out_stride;
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        const int col = (k * G + gl) * 4;
        if (NCH == 1 || col < dim) {
          *reinterpret_cast<double2 *>(o + col) = make_double2(acc[k][0], acc[k][1]);
          *reinterpret_cast<double2 *>(o + col + 2) = make_double2(acc[k][2], acc[k][3]);
        }
      }
      if (counts && gl == 0) counts[bag] = static_cast<int32_t>(cnt);
    }
  }
}


// Generic path (any dim / alignment): one warp per (bag, 128-column tile),
// scalar coalesced loads, same per-element sequential f64 order.
template <typename IdxT, int MODE>
__global__ void __launch_bounds__(256) k_gather_pool_generic(
    const fx_segment *__restrict__ segs, int n_segs, int dim, const IdxT *__restrict__ indices_g,
    const int64_t *__restrict__ offsets, int64_t n_bags, int32_t *__restrict__ counts,
    int64_t *err, int32_t bad_code, int32_t *err_code, bool sysfence) {
  constexpr int TILE = 128, U = 4;
  const int lane = threadIdx.x & 31;
  const int tiles = (dim + TILE - 1) / TILE;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t work = warp; work < n_bags * tiles; work += nwarps) {
    const int64_t bag = work / tiles;
    const int tile = static_cast<int>(work % tiles);
    const int s = find_segment(segs, n_segs, bag);
    const float *__restrict__ tab = segs[s].table;
    const int64_t rb = segs[s].row_begin, re = segs[s].row_end, ld = segs[s].ld;
    int64_t beg, end;
    bag_bounds(segs, s, bag, offsets, beg, end);
    const IdxT *indices = seg_indices(segs, s, indices_g);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t c0 = beg; c0 < end; c0 += 32) {
      const int n = static_cast<int>((end - c0 < 32 ? end - c0 : (int64_t)32));
      int64_t my_off = 0;
      if (lane < n) {
        const int64_t idx = load_index(indices + c0 + lane);
        if (idx < rb || idx >= re) {
          if (tile == 0) record_bad(err, err_code, c0 + lane, bad_code);
        } else {
          my_off = (idx - rb) * ld;
        }
      }
      for (int r = 0; r < n; r += U) {
        float v[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t off = __shfl_sync(0xffffffffu, my_off, (r + u) & 31);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int col = tile * TILE + k * 32 + lane;
            v[u][k] = (r + u < n && col < dim) ? __ldg(tab + off + col) : 0.0f;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (r + u < n) {
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[k] += static_cast<double>(v[u][k]);
          }
      }
    }
    const int64_t cnt = end - beg;
    const int64_t orow = bag - segs[s].bag_begin;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int col = tile * TILE + k * 32 + lane;
      if (col >= dim || (MODE != FX_OUT_F32 && cnt == 0)) continue;  // empty partial: absent, not stored
      if (MODE == FX_OUT_F32) {
        float *o = static_cast<float *>(segs[s].out) + orow * segs[s].out_stride;
        const double v = (segs[s].op == FX_OP_MEAN && cnt > 0) ? acc[k] / static_cast<double>(cnt) : acc[k];
        o[col] = __double2float_rn(v);
      } else if (MODE == FX_OUT_F32_PARTIAL) {
        float *o = static_cast<float *>(segs[s].out) + orow * segs[s].out_stride;
        o[col] = __double2float_rn(acc[k]);
      } else {
        double *o = static_cast<double *>(segs[s].out) + orow * segs[s].out_stride;
        o[col] = acc[k];
      }
    }
    if (MODE != FX_OUT_F32 && counts && tile == 0 && lane == 0) counts[bag] = static_cast<int32_t>(cnt);
  }
  if (sysfence) __threadfence_system();
}

template <typename IdxT>
__global__ void __launch_bounds__(256) k_gather_rows(const float *__restrict__ tab, int64_t ld, int64_t rb,
                                                     int64_t re, int dim, const IdxT *__restrict__ indices,
                                                     int64_t n, float *__restrict__ out, int64_t *err,
                                                     int32_t *err_code) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    const int64_t idx = load_index(indices + i);
    if (idx < rb || idx >= re) {
      if (lane == 0) record_bad(err, err_code, i, FX_E_ROUTING_VIOLATION);
      continue;
    }
    const float *src = tab + (idx - rb) * ld;
    for (int c = lane; c < dim; c += 32) out[i * dim + c] = __ldg(src + c);
  }
}

// ----------------------------------------------------------------- K5
// One warp per bag, lanes over columns (stride 32): fold partial sums in
// ascending source order, then raw rows in position order, in f64; round once.
__global__ void __launch_bounds__(256) k_combine(const void *const *__restrict__ partials, int p_f32,
                                                 const int32_t *const *__restrict__ counts, int n_src,
                                                 int64_t p_stride, const int64_t *__restrict__ raw_offsets,
                                                 const float *__restrict__ raw_rows,
                                                 const float *const *__restrict__ raw_ptrs, int64_t n_bags, int dim,
                                                 int op, const int32_t *__restrict__ ops, float *__restrict__ out,
                                                 int64_t out_stride, int32_t *err_code, int64_t sm_B) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t b = warp; b < n_bags; b += nwarps) {
    int64_t total = 0;
    int present = 0;
    for (int s = 0; s < n_src; ++s) {
      const int32_t c = counts && counts[s] ? counts[s][b] : 1;
      if (c > 0) { total += c; ++present; }
    }
    int64_t r0 = 0, r1 = 0;
    if (raw_offsets) { r0 = raw_offsets[b]; r1 = raw_offsets[b + 1]; }
    total += r1 - r0;
    if (present == 0 && r1 == r0 && err_code && lane == 0) atomicExch(err_code, FX_E_EMPTY);
    const int bop = ops ? ops[b] : op;
    for (int c = lane; c < dim; c += 32) {
      double acc = 0.0;
      for (int s = 0; s < n_src; ++s) {
        const int32_t cs = counts && counts[s] ? counts[s][b] : 1;
        if (cs > 0)
          acc += p_f32 ? static_cast<double>(static_cast<const float *>(partials[s])[b * p_stride + c])
                       : static_cast<const double *>(partials[s])[b * p_stride + c];
      }
      if (raw_ptrs)
        for (int64_t r = r0; r < r1; ++r) acc += static_cast<double>(raw_ptrs[r][c]);
      else
        for (int64_t r = r0; r < r1; ++r) acc += static_cast<double>(raw_rows[r * dim + c]);
      if (bop == FX_OP_MEAN && total > 0) acc /= static_cast<double>(total);
      float *orow = sm_B > 0 ? out + (b % sm_B) * out_stride + (b / sm_B) * dim : out + b * out_stride;
      orow[c] = __double2float_rn(acc);
    }
  }
}

// K5 with 16-byte accesses (dim % 4 == 0, 16-B aligned rows): each lane owns
// 4 consecutive columns; per column the same order as k_combine (partials by
// ascending source, then raw rows in order, f64, one rounding).
__global__ void __launch_bounds__(256) k_combine_v4(const void *const *__restrict__ partials, int p_f32,
                                                    const int32_t *const *__restrict__ counts, int n_src,
                                                    int64_t p_stride, const int64_t *__restrict__ raw_offsets,
                                                    const float *__restrict__ raw_rows,
                                                    const float *const *__restrict__ raw_ptrs, int64_t n_bags,
                                                    int dim, int op, const int32_t *__restrict__ ops,
                                                    float *__restrict__ out, int64_t out_stride, int32_t *err_code,
                                                    int64_t sm_B) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t b = warp; b < n_bags; b += nwarps) {
    int64_t total = 0;
    unsigned present = 0;  // n_src <= 32
    for (int s = 0; s < n_src; ++s) {
      const int32_t c = counts && counts[s] ? counts[s][b] : 1;
      if (c > 0) {
        total += c;
        present |= 1u << s;
      }
    }
    int64_t r0 = 0, r1 = 0;
    if (raw_offsets) {
      r0 = raw_offsets[b];
      r1 = raw_offsets[b + 1];
    }
    total += r1 - r0;
    if (present == 0 && r1 == r0 && err_code && lane == 0) atomicExch(err_code, FX_E_EMPTY);
    const int bop = ops ? ops[b] : op;
    for (int c = lane * 4; c < dim; c += 128) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      for (int s = 0; s < n_src; ++s) {
        if (!((present >> s) & 1u)) continue;
        if (p_f32) {
          const float4 v = *reinterpret_cast<const float4 *>(static_cast<const float *>(partials[s]) + b * p_stride + c);
          a0 += static_cast<double>(v.x); a1 += static_cast<double>(v.y);
          a2 += static_cast<double>(v.z); a3 += static_cast<double>(v.w);
        } else {
          const double *pp = static_cast<const double *>(partials[s]) + b * p_stride + c;
          const double2 u = *reinterpret_cast<const double2 *>(pp);
          const double2 w = *reinterpret_cast<const double2 *>(pp + 2);
          a0 += u.x; a1 += u.y; a2 += w.x; a3 += w.y;
        }
      }
      for (int64_t r = r0; r < r1; ++r) {
        const float *row = raw_ptrs ? raw_ptrs[r] : raw_rows + r * dim;
        const float4 v = *reinterpret_cast<const float4 *>(row + c);
        a0 += static_cast<double>(v.x); a1 += static_cast<double>(v.y);
        a2 += static_cast<double>(v.z); a3 += static_cast<double>(v.w);
      }
      if (bop == FX_OP_MEAN && total > 0) {
        const double dn = static_cast<double>(total);
        a0 /= dn; a1 /= dn; a2 /= dn; a3 /= dn;
      }
      float *orow = sm_B > 0 ? out + (b % sm_B) * out_stride + (b / sm_B) * dim : out + b * out_stride;
      *reinterpret_cast<float4 *>(orow + c) =
          make_float4(__double2float_rn(a0), __double2float_rn(a1), __double2float_rn(a2), __double2float_rn(a3));
    }
  }
}

}  // namespace fx

using namespace fx;

// 16-byte path when every row start is 16-B aligned
static bool combine_vec4_ok(const void *const *partials, int32_t n_src, int64_t p_stride, int64_t dim,
                            int64_t out_stride, const float *out) {
  (void)partials;
  return n_src <= 32 && dim % 4 == 0 && p_stride % 4 == 0 && out_stride % 4 == 0 &&
         (reinterpret_cast<uintptr_t>(out) & 15) == 0;
}

static int pool_variant() {
  static int v = -1;
  if (v < 0) {
    // 2 (default): TMA bulk-copy staging for D = 128 (512-B rows), cp.async otherwise;
    // 1: cp.async staging everywhere; 0: register-staged v4
    const char *e = getenv("FX_POOL_VARIANT");
    v = e ? atoi(e) : 2;
  }
  return v;
}

// FX_OUT_SHARE: this call's cap on resident blocks per SM for the persistent
// (one-wave) kernels, so a concurrent stream keeps room on every SM. Measured
// on the Ranker step (cfg3, K4 beside the cache step): 7 (all) / 3 / 2 / 1
// blocks per SM -> 1.27 / 1.19 / 1.18 / 1.34 ms per batch.
static thread_local int tl_share = 0;
static int share_blocks() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("FX_SHARE_MAXB");
    v = (e && atoi(e) > 0) ? atoi(e) : 2;
  }
  return v;
}

template <int G, int NCH, int CR, typename IdxT, int MODE>
static void launch_async_cr(const fx_segment *segs, int n_segs, int dim, const IdxT *ix, const int64_t *offsets,
                            int64_t n_bags, int32_t *counts, int64_t *err, int32_t bad_code, int32_t *err_code,
                            cudaStream_t st, bool sf) {
  constexpr int WARPS = 4;
  // per group: CR rows x (G lanes * 16 B * NCH); 32/G groups per warp
  const size_t smem = static_cast<size_t>(WARPS) * (32 / G) * CR * G * 16 * NCH;
  // function attributes and occupancy are per device: cache them per device
  static int per_sm_dev[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int &per_sm = per_sm_dev[dev & 63];
  if (per_sm <= 0) {
    cudaFuncSetAttribute(k_pool_async<G, NCH, CR, IdxT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pool_async<G, NCH, CR, IdxT, MODE>, WARPS * 32, smem);
    // FX_POOL_MAXB caps resident blocks per SM (leaves room for a concurrent
    // push kernel in the pipelined sharded mode)
    const char *e = getenv("FX_POOL_MAXB");
    if (e && atoi(e) > 0 && per_sm > atoi(e)) per_sm = atoi(e);
    if (per_sm < 1) per_sm = 1;
  }
  int64_t blocks = static_cast<int64_t>(num_sms()) * (tl_share > 0 && per_sm > tl_share ? tl_share : per_sm);
  const int64_t need = (n_bags + WARPS * (32 / G) - 1) / (WARPS * (32 / G));
  if (blocks > need) blocks = need;
  k_pool_async<G, NCH, CR, IdxT, MODE><<<static_cast<int>(blocks), WARPS * 32, smem, st>>>(
      segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code, sf);
}

template <int G, int NCH, int CR, typename IdxT, int MODE, int MINB = FX_POOL_MINB>
static void launch_bulk_cr(const fx_segment *segs, int n_segs, int dim, const IdxT *ix, const int64_t *offsets,
                           int64_t n_bags, int32_t *counts, int64_t *err, int32_t bad_code, int32_t *err_code,
                           cudaStream_t st, bool sf) {
  constexpr int WARPS = 4;
  const size_t smem = static_cast<size_t>(WARPS) * (32 / G) * (CR * G * 16 * NCH + 8);
  static int per_sm_dev[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int &per_sm = per_sm_dev[dev & 63];
  if (per_sm <= 0) {
    cudaFuncSetAttribute(k_pool_bulk<G, NCH, CR, IdxT, MODE, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pool_bulk<G, NCH, CR, IdxT, MODE, MINB>, WARPS * 32,
                                                  smem);
    if (per_sm < 1) per_sm = 1;
  }
  int64_t blocks = static_cast<int64_t>(num_sms()) * (tl_share > 0 && per_sm > tl_share ? tl_share : per_sm);
  const int64_t need = (n_bags + WARPS * (32 / G) - 1) / (WARPS * (32 / G));
  if (blocks > need) blocks = need;
  k_pool_bulk<G, NCH, CR, IdxT, MODE, MINB><<<static_cast<int>(blocks), WARPS * 32, smem, st>>>(
      segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code, sf);
}

static int pool_chunk_rows() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("FX_POOL_CR");
    v = e ? atoi(e) : 0;  // 0: per-width default below
  }
  return v;
}

// ---- FX_POOL_VARIANT=3: TMA tile::gather4 (D = 128). One 2-D tensor map per
// segment ([INT32_MAX rows, 128] f32, box {128, 1}; indices are validated in
// the kernel before any copy is issued), built on the launch stream from a
// host-encoded template by patching the global address and row stride with
// tensormap.replace. Maps come from a per-device ring (kTmapRing launches of
// up to kTmapSegs segments may be in flight at once).
constexpr int kTmapSegs = 256;
constexpr int kTmapRing = 64;

__global__ void k_tmap_build(const fx_segment *__restrict__ segs, int n_segs, const __grid_constant__ CUtensorMap tmpl,
                             unsigned char *__restrict__ maps) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_segs) return;
  unsigned char *m = maps + static_cast<size_t>(i) * 128;
  const uint4 *src = reinterpret_cast<const uint4 *>(&tmpl);
  uint4 *dst = reinterpret_cast<uint4 *>(m);
#pragma unroll
  for (int k = 0; k < 8; ++k) dst[k] = src[k];
  const uint64_t addr = reinterpret_cast<uint64_t>(segs[i].table);
  const uint64_t stride = static_cast<uint64_t>(segs[i].ld) * 4ull;
  asm volatile("tensormap.replace.tile.global_address.global.b1024.b64 [%0], %1;" ::"l"(m), "l"(addr) : "memory");
  asm volatile("tensormap.replace.tile.global_stride.global.b1024.b64 [%0], 0, %1;" ::"l"(m), "l"(stride)
               : "memory");
  asm volatile("fence.proxy.tensormap::generic.release.gpu;" ::: "memory");
}

struct TmapState {
  bool ok = false;
  CUtensorMap tmpl;
  unsigned char *ring = nullptr;
  int next = 0;
};

static TmapState *tmap_state() {
  static std::mutex mu;
  static TmapState st[64];
  int dev = 0;
  cudaGetDevice(&dev);
  TmapState &t = st[dev & 63];
  std::lock_guard<std::mutex> g(mu);
  if (!t.ring) {
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", reinterpret_cast<void **>(&enc), 12000,
                                         cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !enc)
      return nullptr;
    if (cudaMalloc(&t.ring, static_cast<size_t>(kTmapRing) * kTmapSegs * 128) != cudaSuccess) {
      t.ring = nullptr;
      return nullptr;
    }
    // template: a dummy 16-B aligned address (replaced per segment)
    cuuint64_t gdim[2] = {128, 0x7fffffffull};
    cuuint64_t gstride[1] = {512};
    cuuint32_t box[2] = {128, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&t.tmpl, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, t.ring, gdim, gstride, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    t.ok = r == CUDA_SUCCESS;
  }
  return t.ok ? &t : nullptr;
}

template <int CR, typename IdxT, int MODE, int MINB>
static bool launch_g4(const fx_segment *segs, int n_segs, int dim, const IdxT *ix, const int64_t *offsets,
                      int64_t n_bags, int32_t *counts, int64_t *err, int32_t bad_code, int32_t *err_code,
                      cudaStream_t st, bool sf) {
  if (n_segs > kTmapSegs) return false;
  TmapState *t = tmap_state();
  if (!t) return false;
  unsigned char *maps;
  {
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    maps = t->ring + static_cast<size_t>(t->next) * kTmapSegs * 128;
    t->next = (t->next + 1) % kTmapRing;
  }
  k_tmap_build<<<(n_segs + 127) / 128, 128, 0, st>>>(segs, n_segs, t->tmpl, maps);
  constexpr int WARPS = 4;
  const size_t smem = static_cast<size_t>(WARPS) * (CR * 512 + 8);
  static int per_sm_dev[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int &per_sm = per_sm_dev[dev & 63];
  if (per_sm <= 0) {
    cudaFuncSetAttribute(k_pool_g4<CR, IdxT, MODE, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pool_g4<CR, IdxT, MODE, MINB>, WARPS * 32, smem);
    if (per_sm < 1) per_sm = 1;
  }
  int64_t blocks = static_cast<int64_t>(num_sms()) * (tl_share > 0 && per_sm > tl_share ? tl_share : per_sm);
  const int64_t need = (n_bags + WARPS - 1) / WARPS;
  if (blocks > need) blocks = need;
  k_pool_g4<CR, IdxT, MODE, MINB><<<static_cast<int>(blocks), WARPS * 32, smem, st>>>(
      segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code, sf, maps);
  return true;
}

template <int G, int NCH, typename IdxT, int MODE>
static void launch_async(const fx_segment *segs, int n_segs, int dim, const IdxT *ix, const int64_t *offsets,
                         int64_t n_bags, int32_t *counts, int64_t *err, int32_t bad_code, int32_t *err_code,
                         cudaStream_t st, bool sf) {
  // default chunk: 12 rows for 256-B rows (D=64: cfg1 graph 691 vs 669 M bags/s at 16), else 16
  const int cr = pool_chunk_rows() > 0 ? pool_chunk_rows() : (G == 16 ? 12 : 16);
  if (G == 32 && cr == 24)
    launch_async_cr<G, NCH, (G >= 24 ? 24 : G), IdxT, MODE>(segs, n_segs, dim, ix, offsets, n_bags, counts, err,
                                                          bad_code, err_code, st, sf);
  else if (G >= 8 && cr == 8)
    launch_async_cr<G, NCH, 8, IdxT, MODE>(segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code,
                                           st, sf);
  else if (G >= 12 && cr == 12)
    launch_async_cr<G, NCH, (G >= 12 ? 12 : G), IdxT, MODE>(segs, n_segs, dim, ix, offsets, n_bags, counts, err,
                                                          bad_code, err_code, st, sf);
  else if (G >= 16 && cr == 16)
    launch_async_cr<G, NCH, (G >= 16 ? 16 : G), IdxT, MODE>(segs, n_segs, dim, ix, offsets, n_bags, counts, err,
                                                          bad_code, err_code, st, sf);
  else
    launch_async_cr<G, NCH, G, IdxT, MODE>(segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code,
                                           st, sf);
}

template <typename IdxT, int MODE>
static int launch_pool(const fx_segment *segs, int n_segs, int dim, const void *indices, const int64_t *offsets,
                       int64_t n_bags, int32_t *counts, int64_t *err, int32_t bad_code, int32_t *err_code,
                       cudaStream_t st, bool vec4, bool sf) {
  const IdxT *ix = static_cast<const IdxT *>(indices);
  const int var = vec4 ? pool_variant() : 0;
  if (var == 3 && dim == 128 &&
      launch_g4<12, IdxT, MODE, 7>(segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code, st, sf)) {
    // TMA gather4 A/B (falls through to the bulk copies when maps are unavailable)
  } else if (var >= 2 && dim == 128) {
    // 12-row chunks, <= 72 registers: 7 blocks (28 warps) per SM; tuned on B200
    // against 16-row / 6-block and 8..14-row / 7..10-block configurations
    launch_bulk_cr<32, 1, 12, IdxT, MODE, 7>(segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code,
                                             st, sf);
  } else if (var >= 1 && dim == 256) {
    launch_async<32, 2, IdxT, MODE>(segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code, st, sf);
  } else if (var >= 1 && dim == 64) {
    launch_async<16, 1, IdxT, MODE>(segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code, st, sf);
  } else if (var >= 1 && dim == 32) {
    launch_async<8, 1, IdxT, MODE>(segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code, st, sf);
  } else if (var >= 1 && dim == 512) {
    launch_async<32, 4, IdxT, MODE>(segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code, st, sf);
  } else if (vec4 && dim == 128) {
    k_gather_pool_v4<32, 1, 8, IdxT, MODE><<<grid_for(n_bags * 32, 256), 256, 0, st>>>(
        segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code, sf);
  } else if (vec4 && dim == 64) {
    k_gather_pool_v4<16, 1, 8, IdxT, MODE><<<grid_for(n_bags * 16, 256), 256, 0, st>>>(
        segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code, sf);
  } else if (vec4 && dim == 32) {
    k_gather_pool_v4<8, 1, 8, IdxT, MODE><<<grid_for(n_bags * 8, 256), 256, 0, st>>>(
        segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code, sf);
  } else if (vec4 && dim <= 256) {
    k_gather_pool_v4<32, 2, 4, IdxT, MODE><<<grid_for(n_bags * 32, 256), 256, 0, st>>>(
        segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code, sf);
  } else if (vec4 && dim <= 512) {
    k_gather_pool_v4<32, 4, 2, IdxT, MODE><<<grid_for(n_bags * 32, 256), 256, 0, st>>>(
        segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code, sf);
  } else {
    const int tiles = (dim + 127) / 128;
    k_gather_pool_generic<IdxT, MODE><<<grid_for(n_bags * tiles * 32, 256), 256, 0, st>>>(
        segs, n_segs, dim, ix, offsets, n_bags, counts, err, bad_code, err_code, sf);
  }
  FX_LAUNCH_CHECK("fx_gather_pool");
  return FX_OK;
}


extern "C" {

uint64_t fx_table_base(uint64_t seed, int64_t table_id) {
  return mix64(static_cast<uint64_t>(table_id) ^ mix64(seed));
}

int fx_table_init(float *out, int64_t ld, uint64_t seed, int64_t table_id, int32_t dim, int64_t row_start,
                  int64_t n_rows, void *stream) {
  if (dim < 1 || n_rows < 0 || ld < dim) {
    set_error("fx_table_init: bad shape");
    return FX_E_CONFIG;
  }
  if (n_rows == 0) return FX_OK;
  const uint64_t base = fx_table_base(seed, table_id);
  k_table_init<<<grid_for(n_rows * 32, 256, 16), 256, 0, as_stream(stream)>>>(out, ld, base, dim, row_start,
                                                                               n_rows);
  FX_LAUNCH_CHECK("fx_table_init");
  return FX_OK;
}

int fx_gather_pool(const fx_segment *segs, int32_t n_segs, int32_t dim, const void *indices, int32_t idx_type,
                   const int64_t *offsets, int64_t n_bags, int32_t out_mode, int32_t *counts, int64_t *err,
                   int32_t bad_code, int32_t *err_code, void *stream) {
  const bool sf = (out_mode & FX_OUT_SYSFENCE) != 0;
  const bool scalar = (out_mode & FX_OUT_SCALAR) != 0;
  tl_share = (out_mode & FX_OUT_SHARE) ? share_blocks() : 0;
  out_mode &= ~(FX_OUT_SYSFENCE | FX_OUT_SCALAR | FX_OUT_SHARE);
  if (n_segs < 1 || dim < 1 || (idx_type != FX_IDX_I32 && idx_type != FX_IDX_I64) ||
      (out_mode != FX_OUT_F32 && out_mode != FX_OUT_F64_PARTIAL && out_mode != FX_OUT_F32_PARTIAL)) {
    set_error("fx_gather_pool: bad arguments");
    return FX_E_CONFIG;
  }
  if (n_bags == 0) return FX_OK;
  // The vector / bulk-copy kernels move 16-byte pieces: they need every
  // segment's table base, output pointer (column offset included), ld and
  // out_stride 16-B aligned. The segments live in device memory, so the caller
  // states it: FX_OUT_SCALAR selects the scalar kernel (the Python bindings
  // check the alignment of the descriptors they build and set it otherwise).
  const bool vec4 = (dim % 4) == 0 && !scalar;
  cudaStream_t st = as_stream(stream);
  if (out_mode == FX_OUT_F32_PARTIAL) {
    return idx_type == FX_IDX_I32
               ? launch_pool<int32_t, FX_OUT_F32_PARTIAL>(segs, n_segs, dim, indices, offsets, n_bags, counts, err,
                                                          bad_code, err_code, st, vec4, sf)
               : launch_pool<int64_t, FX_OUT_F32_PARTIAL>(segs, n_segs, dim, indices, offsets, n_bags, counts, err,
                                                          bad_code, err_code, st, vec4, sf);
  }
  if (idx_type == FX_IDX_I32) {
    return out_mode == FX_OUT_F32
               ? launch_pool<int32_t, FX_OUT_F32>(segs, n_segs, dim, indices, offsets, n_bags, counts, err, bad_code,
                                                  err_code, st, vec4, sf)
               : launch_pool<int32_t, FX_OUT_F64_PARTIAL>(segs, n_segs, dim, indices, offsets, n_bags, counts, err,
                                                          bad_code, err_code, st, vec4, sf);
  }
  return out_mode == FX_OUT_F32
             ? launch_pool<int64_t, FX_OUT_F32>(segs, n_segs, dim, indices, offsets, n_bags, counts, err, bad_code,
                                                err_code, st, vec4, sf)
             : launch_pool<int64_t, FX_OUT_F64_PARTIAL>(segs, n_segs, dim, indices, offsets, n_bags, counts, err,
                                                        bad_code, err_code, st, vec4, sf);
}

int fx_gather_rows(const float *table, int64_t ld, int64_t row_begin, int64_t row_end, int32_t dim,
                   const void *indices, int32_t idx_type, int64_t n, float *out, int64_t *err, int32_t *err_code,
                   void *stream) {
  if (dim < 1 || n < 0) {
    set_error("fx_gather_rows: bad arguments");
    return FX_E_CONFIG;
  }
  if (n == 0) return FX_OK;
  cudaStream_t st = as_stream(stream);
  const int grid = grid_for(n * 32, 256);
  if (idx_type == FX_IDX_I32)
    k_gather_rows<int32_t><<<grid, 256, 0, st>>>(table, ld, row_begin, row_end, dim,
                                                 static_cast<const int32_t *>(indices), n, out, err, err_code);
  else
    k_gather_rows<int64_t><<<grid, 256, 0, st>>>(table, ld, row_begin, row_end, dim,
                                                 static_cast<const int64_t *>(indices), n, out, err, err_code);
  FX_LAUNCH_CHECK("fx_gather_rows");
  return FX_OK;
}

int fx_combine(const void *const *partials, int32_t partial_is_f32, const int32_t *const *counts, int32_t n_src,
               int64_t p_stride,
               const int64_t *raw_offsets, const float *raw_rows, int64_t n_bags, int32_t dim, int32_t op,
               const int32_t *ops, float *out, int64_t out_stride, int32_t *err_code, void *stream) {
  if (dim < 1 || n_src < 0 || n_bags < 0) {
    set_error("fx_combine: bad arguments");
    return FX_E_CONFIG;
  }
  if (n_bags == 0) return FX_OK;
  if (combine_vec4_ok(partials, n_src, p_stride, dim, out_stride, out) && (reinterpret_cast<uintptr_t>(raw_rows) & 15) == 0)
    k_combine_v4<<<grid_for(n_bags * 32, 256), 256, 0, as_stream(stream)>>>(
        partials, partial_is_f32, counts, n_src, p_stride, raw_offsets, raw_rows, nullptr, n_bags, dim, op, ops, out,
        out_stride, err_code, 0);
  else
    k_combine<<<grid_for(n_bags * 32, 256), 256, 0, as_stream(stream)>>>(
        partials, partial_is_f32, counts, n_src, p_stride, raw_offsets, raw_rows, nullptr, n_bags, dim, op, ops,
        out, out_stride, err_code, 0);
  FX_LAUNCH_CHECK("fx_combine");
  return FX_OK;
}

int fx_combine_ptr(const void *const *partials, int32_t partial_is_f32, const int32_t *const *counts, int32_t n_src,
                   int64_t p_stride, const int64_t *raw_offsets, const float *const *raw_ptrs, int64_t n_bags,
                   int32_t dim, int32_t op, const int32_t *ops, float *out, int64_t out_stride, int32_t *err_code,
                   int64_t sample_major_B, void *stream) {
  if (dim < 1 || n_src < 0 || n_bags < 0) {
    set_error("fx_combine_ptr: bad arguments");
    return FX_E_CONFIG;
  }
  if (n_bags == 0) return FX_OK;
  if (combine_vec4_ok(partials, n_src, p_stride, dim, out_stride, out))
    k_combine_v4<<<grid_for(n_bags * 32, 256), 256, 0, as_stream(stream)>>>(
        partials, partial_is_f32, counts, n_src, p_stride, raw_offsets, nullptr, raw_ptrs, n_bags, dim, op, ops, out,
        out_stride, err_code, sample_major_B);
  else
    k_combine<<<grid_for(n_bags * 32, 256), 256, 0, as_stream(stream)>>>(
        partials, partial_is_f32, counts, n_src, p_stride, raw_offsets, nullptr, raw_ptrs, n_bags, dim, op, ops,
        out, out_stride, err_code, sample_major_B);
  FX_LAUNCH_CHECK("fx_combine_ptr");
  return FX_OK;
}

}  // extern "C"
