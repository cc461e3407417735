// Shared device/host helpers for libflexemb (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/flexemb.h"

namespace fx {

// thread-local last error message (fx_last_error)
void set_error(const std::string &msg);

inline int cuda_check(cudaError_t e, const char *what) {
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return FX_E_CUDA;
  }
  return FX_OK;
}

#define FX_LAUNCH_CHECK(what)                                  \
  do {                                                         \
    cudaError_t _e = cudaGetLastError();                       \
    if (_e != cudaSuccess) return ::fx::cuda_check(_e, what); \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

int num_sms();

// SplitMix64 finaliser (embserve store.py:62-67), u64 wraparound.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// 64-bit hash for the dedup / cache hash tables (not the content PRF).
__device__ __forceinline__ uint64_t hash_key(uint64_t k) { return mix64(k ^ 0x5851F42D4C957F2Dull); }

template <typename IdxT>
__device__ __forceinline__ int64_t load_index(const IdxT *p) {
  return static_cast<int64_t>(__ldg(p));
}

// Exact f32 -> f64 widening. The default (FX_F2D_ALU undefined) is the
// hardware conversion (F2F.F64.F32, XU pipe, quarter rate); FX_F2D_ALU builds
// the double with integer ops on the ALU pipe (rebias the exponent, shift
// the mantissa) and leaves only zero / denormal / inf / nan to F2F — an A/B
// for K4's XU-pipe pressure (profiles/r2_summary.md).
__device__ __forceinline__ double f2d(float x) {
#ifdef FX_F2D_ALU
  const uint32_t u = __float_as_uint(x);
  const uint32_t e = (u >> 23) & 0xffu;
  if (e == 0u || e == 0xffu) return static_cast<double>(x);
  const uint32_t hi = (u & 0x80000000u) | ((e + 896u) << 20) | ((u >> 3) & 0xfffffu);
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(u << 29));
#else
  return static_cast<double>(x);
#endif
}

// 128-bit streaming load of 4 floats; rows are read-only for the kernel's life.
__device__ __forceinline__ float4 ldg_f4(const float *p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void record_bad(int64_t *err, int32_t *err_code, int64_t pos, int32_t code) {
  if (err) atomicMin(reinterpret_cast<long long *>(err), static_cast<long long>(pos));
  if (err_code) atomicExch(err_code, code);
}

// Last segment whose bag_begin <= bag (segments sorted by bag_begin).
__device__ __forceinline__ int find_segment(const fx_segment *segs, int n, int64_t bag) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (__ldg(&segs[mid].bag_begin) <= bag) lo = mid; else hi = mid;
  }
  return lo;
}

// Bag bounds / index base honouring the optional per-segment sources
// (fx_segment.offs / .idx, e.g. a requester's batch mapped over NVLink).
__device__ __forceinline__ void bag_bounds(const fx_segment *segs, int s, int64_t bag, const int64_t *offsets,
                                           int64_t &beg, int64_t &end) {
  const int64_t *o = segs[s].offs;
  if (o) {
    const int64_t j = bag - segs[s].bag_begin;
    beg = o[j];
    end = o[j + 1];
  } else {
    beg = __ldg(&offsets[bag]);
    end = __ldg(&offsets[bag + 1]);
  }
}

template <typename IdxT>
__device__ __forceinline__ const IdxT *seg_indices(const fx_segment *segs, int s, const IdxT *indices) {
  const void *p = segs[s].idx;
  return p ? static_cast<const IdxT *>(p) : indices;
}

// Last bag b with offsets[b] <= pos (for per-occurrence kernels).
__device__ __forceinline__ int64_t find_bag(const int64_t *offsets, int64_t n_bags, int64_t pos) {
  int64_t lo = 0, hi = n_bags;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(&offsets[mid]) <= pos) lo = mid; else hi = mid;
  }
  return lo;
}

inline int grid_for(int64_t work_items, int per_block, int max_blocks_per_sm = 8) {
  int64_t b = (work_items + per_block - 1) / per_block;
  int64_t cap = static_cast<int64_t>(num_sms()) * max_blocks_per_sm;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return static_cast<int>(b);
}

}  // namespace fx
