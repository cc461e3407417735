// K4 latency-tolerant variants of the fused gather+pool (included by fx_pool.cu).
//
// Both keep the reference's per-element sequential f64 order (each lane owns
// columns and adds the bag's rows in index order), cf. store.py:184-193 and
// pooling.py:60-71.
#pragma once

#include "fx_common.cuh"

namespace fx {

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ---- TMA bulk-copy staging (cp.async.bulk + mbarrier transaction counts)
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(mbar),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int NCH, int MODE>
__device__ __forceinline__ void emit_bag(const fx_segment &sg, int64_t bag, int64_t cnt, double (&acc)[NCH][4],
                                         int lane, int G, int32_t *counts) {
  const int64_t orow = bag - sg.bag_begin;
  if (MODE == FX_OUT_F32) {
    float *o = static_cast<float *>(sg.out) + orow * sg.out_stride;
    const bool mean = sg.op == FX_OP_MEAN && cnt > 0;
    const double dn = static_cast<double>(cnt);
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const int col = (k * G + lane) * 4;
      float4 q;
      if (mean)
        q = make_float4(__double2float_rn(acc[k][0] / dn), __double2float_rn(acc[k][1] / dn),
                        __double2float_rn(acc[k][2] / dn), __double2float_rn(acc[k][3] / dn));
      else
        q = make_float4(__double2float_rn(acc[k][0]), __double2float_rn(acc[k][1]), __double2float_rn(acc[k][2]),
                        __double2float_rn(acc[k][3]));
      *reinterpret_cast<float4 *>(o + col) = q;
    }
  } else if (MODE == FX_OUT_F32_PARTIAL) {
    // an empty partial is absent (count 0, never read by K5): skip the store,
    // which for row-wise shards is mostly a remote NVLink write
    if (counts && lane == 0) counts[bag] = static_cast<int32_t>(cnt);
    if (cnt == 0) return;
    float *o = static_cast<float *>(sg.out) + orow * sg.out_stride;
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const int col = (k * G + lane) * 4;
      *reinterpret_cast<float4 *>(o + col) =
          make_float4(__double2float_rn(acc[k][0]), __double2float_rn(acc[k][1]), __double2float_rn(acc[k][2]),
                      __double2float_rn(acc[k][3]));
    }
  } else {
    if (counts && lane == 0) counts[bag] = static_cast<int32_t>(cnt);
    if (cnt == 0) return;
    double *o = static_cast<double *>(sg.out) + orow * sg.out_stride;
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const int col = (k * G + lane) * 4;
      *reinterpret_cast<double2 *>(o + col) = make_double2(acc[k][0], acc[k][1]);
      *reinterpret_cast<double2 *>(o + col + 2) = make_double2(acc[k][2], acc[k][3]);
    }
  }
}

// Async-staged variant (dim == 4*G*NCH): persistent warps, a group of G lanes
// owns one bag at a time (32/G bags per warp). All rows of a G-index chunk
// are copied global->shared with cp.async (16 B per lane per row, no
// register staging), so the whole bag is in flight at once; while the copies
// land the group prefetches the NEXT bag's offsets and first index chunk.
// Rows are then summed from shared memory in index order.
#ifndef FX_POOL_MINB
#define FX_POOL_MINB 6
#endif
template <int G, int NCH, int CR, typename IdxT, int MODE>
__global__ void __launch_bounds__(128, FX_POOL_MINB) k_pool_async(const fx_segment *__restrict__ segs, int n_segs, int dim,
                                                    const IdxT *__restrict__ indices_g,
                                                    const int64_t *__restrict__ offsets, int64_t n_bags,
                                                    int32_t *__restrict__ counts, int64_t *err, int32_t bad_code,
                                                    int32_t *err_code, bool sysfence) {
  // CR = rows staged per chunk (<= G): smaller chunks -> less shared memory
  // per warp -> more resident warps.
  static_assert(CR <= G, "chunk rows <= lanes per group");
  constexpr int ROWB = G * 16 * NCH;  // bytes per row
  constexpr int GPW = 32 / G;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const int gw = lane / G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gw * G));
  const int wib = threadIdx.x >> 5;
  unsigned char *buf = smem + (static_cast<size_t>(wib) * GPW + gw) * CR * ROWB;
  const uint32_t sbuf = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t step = nwarps * GPW;

  int64_t bag = warp * GPW + gw;
  if (bag >= n_bags) {
    if (sysfence) __threadfence_system();
    return;
  }
  int s = find_segment(segs, n_segs, bag);
  int64_t beg, end;
  bag_bounds(segs, s, bag, offsets, beg, end);
  const IdxT *indices = seg_indices(segs, s, indices_g);
  IdxT pidx = (gl < CR && beg + gl < end) ? indices[beg + gl] : IdxT(0);

  while (bag < n_bags) {
    const float *__restrict__ tab = segs[s].table;
    const int64_t rb = segs[s].row_begin, re = segs[s].row_end, ld = segs[s].ld;
    double acc[NCH][4];
#pragma unroll
    for (int k = 0; k < NCH; ++k) acc[k][0] = acc[k][1] = acc[k][2] = acc[k][3] = 0.0;
    const int64_t nbag = bag + step;
    const int ns = nbag < n_bags ? find_segment(segs, n_segs, nbag) : s;
    const IdxT *nindices = seg_indices(segs, ns, indices_g);
    int64_t nbeg = 0, nend = 0;
    IdxT nidx = IdxT(0);
    bool have_next = false;
    for (int64_t c0 = beg; c0 < end; c0 += CR) {
      const int n = static_cast<int>((end - c0) < CR ? (end - c0) : (int64_t)CR);
      const int64_t idx = static_cast<int64_t>(pidx);
      int64_t my_off = 0;
      if (gl < n) {
        if (idx < rb || idx >= re) record_bad(err, err_code, c0 + gl, bad_code);
        else my_off = (idx - rb) * ld;
      }
      // issue: 4 rows per step so the shuffles / address math overlap
      int r = 0;
      for (; r + 4 <= n; r += 4) {
        const float *src[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) src[u] = tab + __shfl_sync(gmask, my_off, r + u, G);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int k = 0; k < NCH; ++k)
            cp_async16(sbuf + (r + u) * ROWB + (k * G + gl) * 16, src[u] + (k * G + gl) * 4);
      }
      for (; r < n; ++r) {
        const float *src = tab + __shfl_sync(gmask, my_off, r, G);
#pragma unroll
        for (int k = 0; k < NCH; ++k) cp_async16(sbuf + r * ROWB + (k * G + gl) * 16, src + (k * G + gl) * 4);
      }
      cp_async_commit();
      // overlap the copies with the next chunk's / next bag's index loads
      if (c0 + CR < end) {
        pidx = (gl < CR && c0 + CR + gl < end) ? indices[c0 + CR + gl] : IdxT(0);
      } else if (nbag < n_bags) {
        bag_bounds(segs, ns, nbag, offsets, nbeg, nend);
        nidx = (gl < CR && nbeg + gl < nend) ? nindices[nbeg + gl] : IdxT(0);
        have_next = true;
      }
      cp_async_wait_all();
      __syncwarp(gmask);
      // accumulate in row order; 4 rows' shared loads in flight at a time
      r = 0;
      for (; r + 4 <= n; r += 4) {
        float4 v[4][NCH];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int k = 0; k < NCH; ++k)
            v[u][k] = *reinterpret_cast<const float4 *>(buf + (r + u) * ROWB + (k * G + gl) * 16);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int k = 0; k < NCH; ++k) {
            acc[k][0] += f2d(v[u][k].x);
            acc[k][1] += f2d(v[u][k].y);
            acc[k][2] += f2d(v[u][k].z);
            acc[k][3] += f2d(v[u][k].w);
          }
      }
      for (; r < n; ++r) {
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
          const float4 v = *reinterpret_cast<const float4 *>(buf + r * ROWB + (k * G + gl) * 16);
          acc[k][0] += f2d(v.x);
          acc[k][1] += f2d(v.y);
          acc[k][2] += f2d(v.z);
          acc[k][3] += f2d(v.w);
        }
      }
      __syncwarp(gmask);
    }
    if (!have_next && nbag < n_bags) {
      bag_bounds(segs, ns, nbag, offsets, nbeg, nend);
      nidx = (gl < CR && nbeg + gl < nend) ? nindices[nbeg + gl] : IdxT(0);
    }
    emit_bag<NCH, MODE>(segs[s], bag, end - beg, acc, gl, G, counts);
    bag = nbag;
    s = ns;
    indices = nindices;
    beg = nbeg;
    end = nend;
    pidx = nidx;
  }
  if (sysfence) __threadfence_system();
}

}  // namespace fx


namespace fx {

// Bulk-copy variant of k_pool_async (FX_POOL_VARIANT=2): each row of a chunk
// is ONE cp.async.bulk (TMA engine, G*16*NCH bytes) issued by one lane and
// completing on the group's mbarrier, instead of G 16-byte cp.async per row.
// Same order of accumulation (index order, f64 per column).
template <int G, int NCH, int CR, typename IdxT, int MODE, int MINB = FX_POOL_MINB>
__global__ void __launch_bounds__(128, MINB) k_pool_bulk(const fx_segment *__restrict__ segs, int n_segs,
                                                                int dim, const IdxT *__restrict__ indices_g,
                                                                const int64_t *__restrict__ offsets, int64_t n_bags,
                                                                int32_t *__restrict__ counts, int64_t *err,
                                                                int32_t bad_code, int32_t *err_code, bool sysfence) {
  static_assert(CR <= G, "chunk rows <= lanes per group");
  constexpr int ROWB = G * 16 * NCH;
  constexpr int GPW = 32 / G;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const int gw = lane / G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gw * G));
  const int wib = threadIdx.x >> 5;
  const int grp = wib * GPW + gw;
  unsigned char *buf = smem + static_cast<size_t>(grp) * CR * ROWB;
  const uint32_t sbuf = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
  const uint32_t mbar = static_cast<uint32_t>(__cvta_generic_to_shared(
      smem + static_cast<size_t>(blockDim.x / 32) * GPW * CR * ROWB + grp * 8));
  if (gl == 0) mbar_init(mbar, 1);
  fence_proxy_async_smem();
  __syncwarp();
  uint32_t phase = 0;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t step = nwarps * GPW;

  int64_t bag = warp * GPW + gw;
  if (bag >= n_bags) {
    if (sysfence) __threadfence_system();
    return;
  }
  int s = find_segment(segs, n_segs, bag);
  int64_t beg, end;
  bag_bounds(segs, s, bag, offsets, beg, end);
  const IdxT *indices = seg_indices(segs, s, indices_g);
  IdxT pidx = (gl < CR && beg + gl < end) ? indices[beg + gl] : IdxT(0);

  while (bag < n_bags) {
    const float *__restrict__ tab = segs[s].table;
    const int64_t rb = segs[s].row_begin, re = segs[s].row_end, ld = segs[s].ld;
    double acc[NCH][4];
#pragma unroll
    for (int k = 0; k < NCH; ++k) acc[k][0] = acc[k][1] = acc[k][2] = acc[k][3] = 0.0;
    const int64_t nbag = bag + step;
    const int ns = nbag < n_bags ? find_segment(segs, n_segs, nbag) : s;
    const IdxT *nindices = seg_indices(segs, ns, indices_g);
    int64_t nbeg = 0, nend = 0;
    IdxT nidx = IdxT(0);
    bool have_next = false;
    for (int64_t c0 = beg; c0 < end; c0 += CR) {
      const int n = static_cast<int>((end - c0) < CR ? (end - c0) : (int64_t)CR);
      const int64_t idx = static_cast<int64_t>(pidx);
      int64_t my_off = 0;
      if (gl < n) {
        if (idx < rb || idx >= re) record_bad(err, err_code, c0 + gl, bad_code);
        else my_off = (idx - rb) * ld;
      }
      if (gl == 0) mbar_expect_tx(mbar, static_cast<uint32_t>(n) * ROWB);
      __syncwarp(gmask);
      if (gl < n) bulk_g2s(sbuf + gl * ROWB, tab + my_off, ROWB, mbar);
      // overlap the copies with the next chunk's / next bag's index loads
      if (c0 + CR < end) {
        pidx = (gl < CR && c0 + CR + gl < end) ? indices[c0 + CR + gl] : IdxT(0);
      } else if (nbag < n_bags) {
        bag_bounds(segs, ns, nbag, offsets, nbeg, nend);
        nidx = (gl < CR && nbeg + gl < nend) ? nindices[nbeg + gl] : IdxT(0);
        have_next = true;
      }
      mbar_wait(mbar, phase);
      phase ^= 1u;
      int r = 0;
      for (; r + 4 <= n; r += 4) {
        float4 v[4][NCH];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int k = 0; k < NCH; ++k)
            v[u][k] = *reinterpret_cast<const float4 *>(buf + (r + u) * ROWB + (k * G + gl) * 16);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int k = 0; k < NCH; ++k) {
            acc[k][0] += f2d(v[u][k].x);
            acc[k][1] += f2d(v[u][k].y);
            acc[k][2] += f2d(v[u][k].z);
            acc[k][3] += f2d(v[u][k].w);
          }
      }
      for (; r < n; ++r) {
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
          const float4 v = *reinterpret_cast<const float4 *>(buf + r * ROWB + (k * G + gl) * 16);
          acc[k][0] += f2d(v.x);
          acc[k][1] += f2d(v.y);
          acc[k][2] += f2d(v.z);
          acc[k][3] += f2d(v.w);
        }
      }
      fence_proxy_async_smem();  // generic reads of buf before the next bulk writes into it
      __syncwarp(gmask);
    }
    if (!have_next && nbag < n_bags) {
      bag_bounds(segs, ns, nbag, offsets, nbeg, nend);
      nidx = (gl < CR && nbeg + gl < nend) ? nindices[nbeg + gl] : IdxT(0);
    }
    emit_bag<NCH, MODE>(segs[s], bag, end - beg, acc, gl, G, counts);
    bag = nbag;
    s = ns;
    indices = nindices;
    beg = nbeg;
    end = nend;
    pidx = nidx;
  }
  if (sysfence) __threadfence_system();
}

}  // namespace fx

// ---- TMA tensor gather (FX_POOL_VARIANT=3, D = 128): the A/B SURVEY §2.3
// asks for against the 1-D bulk copies above. One lane per 4 rows issues
// cp.async.bulk.tensor.2d...tile::gather4 (SASS UTMALDG.2D.GATHER4) through
// the segment's 2-D tensor map ([rows, 128] f32, box {128, 1}; row
// coordinates are shard-relative and validated before issue), so a 12-row
// chunk is 3 TMA requests instead of 12. A chunk whose row count is not a
// multiple of 4 repeats its last row in the padding slots (loaded, never
// summed). Tensor maps live in global memory (one 128-B CUtensorMap per
// segment, written by k_tmap_build on the same stream).
namespace fx {

__device__ __forceinline__ void tma_gather4(uint32_t dst, const void *tmap, int32_t col, int32_t r0, int32_t r1,
                                            int32_t r2, int32_t r3, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(tmap), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void tmap_acquire(const void *tmap) {
  asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(tmap) : "memory");
}

template <int CR, typename IdxT, int MODE, int MINB = FX_POOL_MINB>
__global__ void __launch_bounds__(128, MINB) k_pool_g4(const fx_segment *__restrict__ segs, int n_segs, int dim,
                                                       const IdxT *__restrict__ indices_g,
                                                       const int64_t *__restrict__ offsets, int64_t n_bags,
                                                       int32_t *__restrict__ counts, int64_t *err, int32_t bad_code,
                                                       int32_t *err_code, bool sysfence,
                                                       const unsigned char *__restrict__ tmaps) {
  static_assert(CR % 4 == 0 && CR <= 32, "whole gather4 groups");
  constexpr int G = 32, NCH = 1, ROWB = 512;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char *buf = smem + static_cast<size_t>(wib) * CR * ROWB;
  const uint32_t sbuf = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
  const uint32_t mbar = static_cast<uint32_t>(
      __cvta_generic_to_shared(smem + static_cast<size_t>(blockDim.x / 32) * CR * ROWB + wib * 8));
  if (lane == 0) mbar_init(mbar, 1);
  fence_proxy_async_smem();
  __syncwarp();
  uint32_t phase = 0;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t step = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t bag = warp;
  if (bag >= n_bags) {
    if (sysfence) __threadfence_system();
    return;
  }
  int s = find_segment(segs, n_segs, bag);
  int acq = -1;  // segment whose tensor map this warp has acquired
  int64_t beg, end;
  bag_bounds(segs, s, bag, offsets, beg, end);
  const IdxT *indices = seg_indices(segs, s, indices_g);
  IdxT pidx = (lane < CR && beg + lane < end) ? indices[beg + lane] : IdxT(0);
  while (bag < n_bags) {
    const int64_t rb = segs[s].row_begin, re = segs[s].row_end;
    const unsigned char *tm = tmaps + static_cast<size_t>(s) * 128;
    if (acq != s) {
      tmap_acquire(tm);
      acq = s;
    }
    double acc[NCH][4];
    acc[0][0] = acc[0][1] = acc[0][2] = acc[0][3] = 0.0;
    const int64_t nbag = bag + step;
    const int ns = nbag < n_bags ? find_segment(segs, n_segs, nbag) : s;
    const IdxT *nindices = seg_indices(segs, ns, indices_g);
    int64_t nbeg = 0, nend = 0;
    IdxT nidx = IdxT(0);
    bool have_next = false;
    for (int64_t c0 = beg; c0 < end; c0 += CR) {
      const int n = static_cast<int>((end - c0) < CR ? (end - c0) : (int64_t)CR);
      const int ng = (n + 3) >> 2;
      const int64_t idx = static_cast<int64_t>(pidx);
      int32_t rel = 0;
      if (lane < n) {
        if (idx < rb || idx >= re) record_bad(err, err_code, c0 + lane, bad_code);
        else rel = static_cast<int32_t>(idx - rb);
      }
      // padding slots repeat the chunk's last row
      const int32_t last = __shfl_sync(0xffffffffu, rel, n - 1);
      if (lane >= n) rel = last;
      const int q = (lane & 7) << 2;  // lanes 0..ng-1 gather rows 4*lane .. 4*lane+3
      const int32_t g0 = __shfl_sync(0xffffffffu, rel, q);
      const int32_t g1 = __shfl_sync(0xffffffffu, rel, q + 1);
      const int32_t g2 = __shfl_sync(0xffffffffu, rel, q + 2);
      const int32_t g3 = __shfl_sync(0xffffffffu, rel, q + 3);
      if (lane == 0) mbar_expect_tx(mbar, static_cast<uint32_t>(ng) * 4 * ROWB);
      __syncwarp();
      if (lane < ng) tma_gather4(sbuf + lane * 4 * ROWB, tm, 0, g0, g1, g2, g3, mbar);
      if (c0 + CR < end) {
        pidx = (lane < CR && c0 + CR + lane < end) ? indices[c0 + CR + lane] : IdxT(0);
      } else if (nbag < n_bags) {
        bag_bounds(segs, ns, nbag, offsets, nbeg, nend);
        nidx = (lane < CR && nbeg + lane < nend) ? nindices[nbeg + lane] : IdxT(0);
        have_next = true;
      }
      mbar_wait(mbar, phase);
      phase ^= 1u;
      int r = 0;
      for (; r + 4 <= n; r += 4) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = *reinterpret_cast<const float4 *>(buf + (r + u) * ROWB + lane * 16);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc[0][0] += f2d(v[u].x);
          acc[0][1] += f2d(v[u].y);
          acc[0][2] += f2d(v[u].z);
          acc[0][3] += f2d(v[u].w);
        }
      }
      for (; r < n; ++r) {
        const float4 v = *reinterpret_cast<const float4 *>(buf + r * ROWB + lane * 16);
        acc[0][0] += f2d(v.x);
        acc[0][1] += f2d(v.y);
        acc[0][2] += f2d(v.z);
        acc[0][3] += f2d(v.w);
      }
      fence_proxy_async_smem();
      __syncwarp();
    }
    if (!have_next && nbag < n_bags) {
      bag_bounds(segs, ns, nbag, offsets, nbeg, nend);
      nidx = (lane < CR && nbeg + lane < nend) ? nindices[nbeg + lane] : IdxT(0);
    }
    emit_bag<NCH, MODE>(segs[s], bag, end - beg, acc, lane, G, counts);
    bag = nbag;
    s = ns;
    indices = nindices;
    beg = nbeg;
    end = nend;
    pidx = nidx;
  }
  if (sysfence) __threadfence_system();
}

}  // namespace fx
