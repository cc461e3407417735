// Pooled-result cache keys (cache.py:204-223): the reference keys a pooled
// vector by ("pooled", table, op, tuple(sorted(indices))). On the GPU a bag's
// key is a pair of 64-bit multiset fingerprints (order-independent, so no
// per-bag sort is needed):
//   sA = sum_i mix64(x_i ^ SALT_A),  sB = sum_i mix64(x_i ^ SALT_B)   (mod 2^64)
//   A  = mix64(sA ^ mix64(mix64(table ^ SALT_A) + op) ^ (L * SALT_B)) | 2^63
//   B  = mix64(sB ^ mix64(mix64(table ^ SALT_B) + op) ^ (L * SALT_A))
// A (top bit set, disjoint from row keys table << 40 | row) indexes the
// cache; B is stored per slot and verified on every match, so two different
// multisets are confused only if both 64-bit fingerprints collide; an A-only
// collision is reported as FX_E_INVARIANT instead of returning a wrong vector.
#include "fx_common.cuh"

namespace fx {

constexpr uint64_t kSaltA = 0xA0761D6478BD642Full;
constexpr uint64_t kSaltB = 0xE7037ED1A0B428DBull;

template <typename IdxT>
__global__ void __launch_bounds__(256) k_bag_fingerprint(const int32_t *__restrict__ bag_table,
                                                         const int32_t *__restrict__ bag_op,
                                                         const IdxT *__restrict__ indices,
                                                         const int64_t *__restrict__ offsets, int64_t n_bags,
                                                         uint64_t *__restrict__ key_a, uint64_t *__restrict__ key_b) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = warp; b < n_bags; b += nw) {
    const int64_t beg = __ldg(&offsets[b]), end = __ldg(&offsets[b + 1]);
    uint64_t sa = 0, sb = 0;
    for (int64_t i = beg + lane; i < end; i += 32) {
      const uint64_t x = static_cast<uint64_t>(static_cast<int64_t>(__ldg(&indices[i])));
      sa += mix64(x ^ kSaltA);
      sb += mix64(x ^ kSaltB);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
      sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    if (lane == 0) {
      const uint64_t t = static_cast<uint64_t>(static_cast<uint32_t>(bag_table[b]));
      const uint64_t op = static_cast<uint64_t>(static_cast<uint32_t>(bag_op[b]));
      const uint64_t L = static_cast<uint64_t>(end - beg);
      key_a[b] = mix64(sa ^ mix64(mix64(t ^ kSaltA) + op) ^ (L * kSaltB)) | (1ull << 63);
      key_b[b] = mix64(sb ^ mix64(mix64(t ^ kSaltB) + op) ^ (L * kSaltA));
    }
  }
}

}  // namespace fx

using namespace fx;

extern "C" int fx_bag_fingerprint(const int32_t *bag_table, const int32_t *bag_op, const void *indices,
                                  int32_t idx_type, const int64_t *offsets, int64_t n_bags, uint64_t *key_a,
                                  uint64_t *key_b, void *stream) {
  if (n_bags <= 0) return FX_OK;
  if (!bag_table || !bag_op || !offsets || !key_a || !key_b || (idx_type != FX_IDX_I32 && idx_type != FX_IDX_I64)) {
    set_error("fx_bag_fingerprint: bad arguments");
    return FX_E_CONFIG;
  }
  const int grid = grid_for(n_bags * 32, 256);
  cudaStream_t st = as_stream(stream);
  if (idx_type == FX_IDX_I32)
    k_bag_fingerprint<int32_t><<<grid, 256, 0, st>>>(bag_table, bag_op, static_cast<const int32_t *>(indices),
                                                     offsets, n_bags, key_a, key_b);
  else
    k_bag_fingerprint<int64_t><<<grid, 256, 0, st>>>(bag_table, bag_op, static_cast<const int64_t *>(indices),
                                                     offsets, n_bags, key_a, key_b);
  FX_LAUNCH_CHECK("fx_bag_fingerprint");
  return FX_OK;
}
