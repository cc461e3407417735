// C-ABI housekeeping: error strings, version, device queries.
#include <string>

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

}  // namespace fx

extern "C" {

const char *fx_last_error(void) { return fx::g_last_error.c_str(); }

int fx_version(void) { return 1; }

int fx_num_sms(int device) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return sms;
}

}  // extern "C"
