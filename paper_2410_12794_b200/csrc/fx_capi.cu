// C-ABI housekeeping: error strings, version, device queries.
#include <string>

#include "fx_ckptr.cuh"
#include "fx_common.cuh"

namespace fx {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int num_sms() {
  static thread_local int cached_dev = -1;
  static thread_local int cached_sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cached_sms;
  if (dev != cached_dev) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
      cached_sms = sms;
    cached_dev = dev;
  }
  return cached_sms;
}

OobRecord *oob_record() {
#ifdef FX_BOUNDS
  static OobRecord *rec[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  OobRecord *&r = rec[dev & 63];
  if (!r) {
    if (cudaMalloc(&r, sizeof(OobRecord)) != cudaSuccess) return r = nullptr;
    cudaMemset(r, 0, sizeof(OobRecord));
  }
  return r;
#else
  return nullptr;
#endif
}

#ifdef FX_BOUNDS
__global__ void k_bounds_selftest(CkPtr<int32_t> a, int32_t i, int32_t *out) { *out = a[i]; }
#endif

}  // namespace fx

extern "C" {

int fx_bounds_selftest(void) {
#ifdef FX_BOUNDS
  // a checked 4-element array read at index 5 must be caught and recorded;
  // the record is cleared afterwards
  fx::OobRecord *r = fx::oob_record();
  int32_t *buf = nullptr;
  if (!r || cudaMalloc(&buf, 8 * sizeof(int32_t)) != cudaSuccess) return -1;
  fx::CkPtr<int32_t> a(buf, 4, r);
  fx::OobRecord before{}, after{};
  cudaMemcpy(&before, r, sizeof(before), cudaMemcpyDeviceToHost);
  fx::k_bounds_selftest<<<1, 1>>>(a, 5, buf + 4);
  cudaMemcpy(&after, r, sizeof(after), cudaMemcpyDeviceToHost);
  cudaFree(buf);
  const bool ok = after.count == before.count + 1 && (before.count > 0 || (after.index == 5 && after.length == 4));
  if (before.count == 0) cudaMemset(r, 0, sizeof(fx::OobRecord));
  return ok ? 1 : -1;
#else
  return 0;
#endif
}

int fx_bounds_report(int64_t *out4) {
#ifdef FX_BOUNDS
  fx::OobRecord *r = fx::oob_record();
  if (!r) return -1;
  fx::OobRecord h{};
  if (cudaMemcpy(&h, r, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  out4[0] = static_cast<int64_t>(h.count);
  out4[1] = static_cast<int64_t>(h.base);
  out4[2] = h.index;
  out4[3] = h.length;
  return 1;
#else
  (void)out4;
  return 0;
#endif
}

const char *fx_last_error(void) { return fx::g_last_error.c_str(); }

int fx_version(void) { return 1; }

int fx_num_sms(int device) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return sms;
}

}  // extern "C"
