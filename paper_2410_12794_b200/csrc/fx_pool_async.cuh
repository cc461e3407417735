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
    float *o = static_cast<float *>(sg.out) + orow * sg.out_stride;
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const int col = (k * G + lane) * 4;
      *reinterpret_cast<float4 *>(o + col) =
          make_float4(__double2float_rn(acc[k][0]), __double2float_rn(acc[k][1]), __double2float_rn(acc[k][2]),
                      __double2float_rn(acc[k][3]));
    }
    if (counts && lane == 0) counts[bag] = static_cast<int32_t>(cnt);
  } else {
    double *o = static_cast<double *>(sg.out) + orow * sg.out_stride;
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const int col = (k * G + lane) * 4;
      *reinterpret_cast<double2 *>(o + col) = make_double2(acc[k][0], acc[k][1]);
      *reinterpret_cast<double2 *>(o + col + 2) = make_double2(acc[k][2], acc[k][3]);
    }
    if (counts && lane == 0) counts[bag] = static_cast<int32_t>(cnt);
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
            acc[k][0] += static_cast<double>(v[u][k].x);
            acc[k][1] += static_cast<double>(v[u][k].y);
            acc[k][2] += static_cast<double>(v[u][k].z);
            acc[k][3] += static_cast<double>(v[u][k].w);
          }
      }
      for (; r < n; ++r) {
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
          const float4 v = *reinterpret_cast<const float4 *>(buf + r * ROWB + (k * G + gl) * 16);
          acc[k][0] += static_cast<double>(v.x);
          acc[k][1] += static_cast<double>(v.y);
          acc[k][2] += static_cast<double>(v.z);
          acc[k][3] += static_cast<double>(v.w);
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

__device__ __forceinline__ void cp_async_wait_n(int n) {
  switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
  }
}

// One chunk = up to 32 consecutive indices of one bag.
template <typename IdxT>
struct PoolChunk {
  int64_t bag;   // -1 when past the warp's last bag
  int64_t c0;    // first CSR position of the chunk
  int64_t end;   // bag end (CSR)
  int64_t cnt;   // bag length
  int s;         // segment
  int n;         // rows in the chunk
  int first;     // chunk opens the bag
  int last;      // chunk closes the bag
  IdxT idx;      // this lane's index (position c0 + lane), prefetched
};

// Ring-staged variant (dim == 128*NCH): persistent warps; each warp owns a
// shared-memory ring of RING rows and keeps up to 4 chunks (cp.async groups)
// in flight, issuing the next chunks while it sums the oldest one, so the
// accumulate/emit work overlaps the row fetches. Chunks of one bag are summed
// in order (per-element sequential f64, as the reference).
template <int NCH, int RING, typename IdxT, int MODE>
__global__ void __launch_bounds__(128) k_pool_ring(const fx_segment *__restrict__ segs, int n_segs, int dim,
                                                   const IdxT *__restrict__ indices_g,
                                                   const int64_t *__restrict__ offsets, int64_t n_bags,
                                                   int32_t *__restrict__ counts, int64_t *err, int32_t bad_code,
                                                   int32_t *err_code, bool sysfence) {
  constexpr int ROWB = 32 * 16 * NCH;
  constexpr int MAXF = 4;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char *ring = smem + static_cast<size_t>(wib) * RING * ROWB;
  const uint32_t sring = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;

  auto open_bag = [&](int64_t bag) {
    PoolChunk<IdxT> c;
    c.bag = bag;
    if (bag >= n_bags) {
      c.bag = -1;
      return c;
    }
    c.s = find_segment(segs, n_segs, bag);
    int64_t beg, end;
    bag_bounds(segs, c.s, bag, offsets, beg, end);
    const IdxT *ix = seg_indices(segs, c.s, indices_g);
    c.c0 = beg;
    c.end = end;
    c.cnt = end - beg;
    c.n = static_cast<int>(end - beg < 32 ? end - beg : 32);
    c.first = 1;
    c.last = (beg + 32 >= end) ? 1 : 0;
    c.idx = (beg + lane < end) ? ix[beg + lane] : IdxT(0);
    return c;
  };
  auto advance = [&](const PoolChunk<IdxT> &x) {
    if (x.last) return open_bag(x.bag + nwarps);
    PoolChunk<IdxT> c = x;
    c.c0 = x.c0 + 32;
    c.n = static_cast<int>(x.end - c.c0 < 32 ? x.end - c.c0 : 32);
    c.first = 0;
    c.last = (c.c0 + 32 >= x.end) ? 1 : 0;
    const IdxT *ix = seg_indices(segs, c.s, indices_g);
    c.idx = (c.c0 + lane < x.end) ? ix[c.c0 + lane] : IdxT(0);
    return c;
  };

  PoolChunk<IdxT> q[MAXF];   // in-flight chunks (oldest first)
  int qhead[MAXF];           // ring row where each chunk starts
  int nq = 0, head = 0, used = 0;
  PoolChunk<IdxT> nxt = open_bag(warp);
  double acc[NCH][4];
#pragma unroll
  for (int k = 0; k < NCH; ++k) acc[k][0] = acc[k][1] = acc[k][2] = acc[k][3] = 0.0;

  while (true) {
    // issue as many chunks as fit
    while (nxt.bag >= 0 && nq < MAXF && used + nxt.n <= RING) {
      const fx_segment &sg = segs[nxt.s];
      const float *__restrict__ tab = sg.table;
      const int64_t idx = static_cast<int64_t>(nxt.idx);
      int64_t my_off = 0;
      if (lane < nxt.n) {
        if (idx < sg.row_begin || idx >= sg.row_end) record_bad(err, err_code, nxt.c0 + lane, bad_code);
        else my_off = (idx - sg.row_begin) * sg.ld;
      }
      const int start = (head + used) % RING;
      for (int r = 0; r < nxt.n; ++r) {
        const float *src = tab + __shfl_sync(0xffffffffu, my_off, r);
        const int row = (start + r) % RING;
#pragma unroll
        for (int k = 0; k < NCH; ++k)
          cp_async16(sring + row * ROWB + (k * 32 + lane) * 16, src + (k * 32 + lane) * 4);
      }
      cp_async_commit();
      // shift the queue entry in (small fixed-size queue, register-resident after unrolling)
#pragma unroll
      for (int i = 0; i < MAXF; ++i)
        if (i == nq) {
          q[i] = nxt;
          qhead[i] = start;
        }
      ++nq;
      used += nxt.n;
      nxt = advance(nxt);  // prefetch the following chunk's indices
    }
    if (nq == 0) break;
    cp_async_wait_n(nq - 1);  // the oldest chunk has landed
    __syncwarp();
    const PoolChunk<IdxT> x = q[0];
    const int xs = qhead[0];
    for (int r = 0; r < x.n; ++r) {
      const int row = (xs + r) % RING;
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        const float4 v = *reinterpret_cast<const float4 *>(ring + row * ROWB + (k * 32 + lane) * 16);
        acc[k][0] += static_cast<double>(v.x);
        acc[k][1] += static_cast<double>(v.y);
        acc[k][2] += static_cast<double>(v.z);
        acc[k][3] += static_cast<double>(v.w);
      }
    }
    __syncwarp();
    if (x.last) {
      emit_bag<NCH, MODE>(segs[x.s], x.bag, x.cnt, acc, lane, 32, counts);
#pragma unroll
      for (int k = 0; k < NCH; ++k) acc[k][0] = acc[k][1] = acc[k][2] = acc[k][3] = 0.0;
    }
    head = (head + x.n) % RING;
    used -= x.n;
#pragma unroll
    for (int i = 0; i < MAXF - 1; ++i) {
      q[i] = q[i + 1];
      qhead[i] = qhead[i + 1];
    }
    --nq;
  }
  if (sysfence) __threadfence_system();
}

// Bag-per-group register variant with next-bag software prefetch: the next
// chunk's indices (or the next bag's offsets + first chunk) are loaded right
// after the first round of row loads is issued.
template <int G, int NCH, int U, typename IdxT, int MODE>
__global__ void __launch_bounds__(256) k_pool_prefetch(const fx_segment *__restrict__ segs, int n_segs, int dim,
                                                       const IdxT *__restrict__ indices_g,
                                                       const int64_t *__restrict__ offsets, int64_t n_bags,
                                                       int32_t *__restrict__ counts, int64_t *err, int32_t bad_code,
                                                       int32_t *err_code, bool sysfence) {
  constexpr int GPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const int gw = lane / G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gw * G));
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
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
  IdxT pidx = (beg + gl < end) ? indices[beg + gl] : IdxT(0);
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
    for (int64_t c0 = beg; c0 < end; c0 += G) {
      const int n = static_cast<int>((end - c0) < G ? (end - c0) : (int64_t)G);
      const int64_t idx = static_cast<int64_t>(pidx);
      int64_t my_off = 0;
      if (gl < n) {
        if (idx < rb || idx >= re) record_bad(err, err_code, c0 + gl, bad_code);
        else my_off = (idx - rb) * ld;
      }
      for (int r = 0; r < n; r += U) {
        float4 v[U][NCH];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t off = __shfl_sync(gmask, my_off, (r + u) & (G - 1), G);
          if (r + u < n) {
#pragma unroll
            for (int k = 0; k < NCH; ++k) v[u][k] = ldg_f4(tab + off + (k * G + gl) * 4);
          }
        }
        if (r == 0) {
          if (c0 + G < end) {
            pidx = (c0 + G + gl < end) ? indices[c0 + G + gl] : IdxT(0);
          } else if (nbag < n_bags) {
            bag_bounds(segs, ns, nbag, offsets, nbeg, nend);
            nidx = (nbeg + gl < nend) ? nindices[nbeg + gl] : IdxT(0);
            have_next = true;
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
    if (!have_next && nbag < n_bags) {
      bag_bounds(segs, ns, nbag, offsets, nbeg, nend);
      nidx = (nbeg + gl < nend) ? nindices[nbeg + gl] : IdxT(0);
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
