// The store side of the C-ABI (SURVEY §8(b) contract): a placement's shards
// owned by one rank, allocated in HBM and materialised with K0 — the
// reference's init_store / Deployment (store.py:92-119, 215-251) for a
// caller that does not go through the Python mirror — plus a zero-copy view
// of a shard and a reader for the kernels' device-side status words.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "fx_common.cuh"

struct fx_store {
  int device = 0;
  std::vector<fx_shard_desc> shards;  // the rank's own shards
  std::vector<float *> data;
  std::vector<int64_t> ld;
  std::vector<int32_t> dims;
};

extern "C" {

int fx_store_create(fx_store **out, int32_t device, int32_t n_tables, const int64_t *rows, const int32_t *dims,
                    int32_t n_shards, const fx_shard_desc *shards, int32_t my_rank, uint64_t seed, void *stream) {
  if (!out || n_tables < 1 || n_shards < 0 || !rows || !dims || (n_shards > 0 && !shards)) {
    fx::set_error("fx_store_create: bad arguments");
    return FX_E_CONFIG;
  }
  // placement validation (store.py:92-119): per table, shards disjoint and covering [0, rows)
  for (int32_t t = 0; t < n_tables; ++t) {
    std::vector<std::pair<int64_t, int64_t>> iv;
    for (int32_t i = 0; i < n_shards; ++i)
      if (shards[i].table == t) iv.emplace_back(shards[i].start, shards[i].end);
    std::sort(iv.begin(), iv.end());
    int64_t cur = 0;
    for (auto &p : iv) {
      if (p.first < cur) {
        fx::set_error("fx_store_create: table " + std::to_string(t) + " overlap at row " + std::to_string(p.first));
        return FX_E_CONFIG;
      }
      if (p.first > cur) {
        fx::set_error("fx_store_create: table " + std::to_string(t) + " gap [" + std::to_string(cur) + "," +
                      std::to_string(p.first) + ")");
        return FX_E_CONFIG;
      }
      cur = p.second;
    }
    if (cur != rows[t]) {
      fx::set_error("fx_store_create: table " + std::to_string(t) + " shards end at " + std::to_string(cur) +
                    ", not at its " + std::to_string(rows[t]) + " rows");
      return FX_E_CONFIG;
    }
  }
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) {
    fx::set_error("fx_store_create: bad device");
    return FX_E_CONFIG;
  }
  fx_store *s = new fx_store();
  s->device = device;
  int rc = FX_OK;
  for (int32_t i = 0; i < n_shards && rc == FX_OK; ++i) {
    const fx_shard_desc &d = shards[i];
    if (d.owner != my_rank) continue;
    if (d.table < 0 || d.table >= n_tables) {
      fx::set_error("fx_store_create: shard of an unknown table");
      rc = FX_E_CONFIG;
      break;
    }
    const int32_t dim = dims[d.table];
    const int64_t ld = (dim + 3) & ~3;  // 16-byte aligned rows
    const int64_t n = d.end - d.start;
    float *p = nullptr;
    rc = fx::cuda_check(cudaMalloc(&p, static_cast<size_t>(n > 0 ? n : 1) * ld * sizeof(float)), "fx_store_create");
    if (rc) break;
    s->shards.push_back(d);
    s->data.push_back(p);
    s->ld.push_back(ld);
    s->dims.push_back(dim);
    rc = fx_table_init(p, ld, seed, d.table, dim, d.start, n, stream);
  }
  cudaSetDevice(prev);
  if (rc) {
    fx_store_destroy(s);
    return rc;
  }
  *out = s;
  return FX_OK;
}

int fx_store_destroy(fx_store *s) {
  if (!s) return FX_OK;
  for (float *p : s->data) cudaFree(p);
  delete s;
  return FX_OK;
}

int fx_store_shard_view(fx_store *s, int32_t table, int64_t row, const float **base, int64_t *start, int64_t *end,
                        int64_t *ld, int32_t *dim) {
  for (size_t i = 0; i < s->shards.size(); ++i) {
    const fx_shard_desc &d = s->shards[i];
    if (d.table == table && row >= d.start && row < d.end) {
      if (base) *base = s->data[i];
      if (start) *start = d.start;
      if (end) *end = d.end;
      if (ld) *ld = s->ld[i];
      if (dim) *dim = s->dims[i];
      return FX_OK;
    }
  }
  fx::set_error("fx_store_shard_view: row " + std::to_string(row) + " of table " + std::to_string(table) +
                " is not hosted by this store");
  return FX_E_ROUTING_VIOLATION;
}

int fx_poll_error(const int32_t *err_code, const int64_t *err_pos, int32_t *code, int64_t *pos, void *stream) {
  cudaStream_t st = fx::as_stream(stream);
  int32_t c = 0;
  int64_t p = -1;
  int rc = FX_OK;
  if (err_code) rc = fx::cuda_check(cudaMemcpyAsync(&c, err_code, 4, cudaMemcpyDeviceToHost, st), "fx_poll_error");
  if (!rc && err_pos) rc = fx::cuda_check(cudaMemcpyAsync(&p, err_pos, 8, cudaMemcpyDeviceToHost, st), "fx_poll_error");
  if (!rc) rc = fx::cuda_check(cudaStreamSynchronize(st), "fx_poll_error");
  if (code) *code = c;
  if (pos) *pos = p;
  return rc;
}

}  // extern "C"
