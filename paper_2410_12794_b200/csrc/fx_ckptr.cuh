// Bounds-checked device arrays for the FX_BOUNDS build (compute-sanitizer is
// not available on the GPU pool, so the library checks its own indexing).
//
// Normal builds: CkPtr<T> is T* — zero cost, identical code.
// FX_BOUNDS builds (FX_EXTRA_NVCC=-DFX_BOUNDS FX_BUILD_TAG=chk python build.py
// -> libflexemb_chk.so): the arrays of the cache view (fx_cache.cuh) and of the
// fused step (fx_step.cu) carry their allocated length; every subscript is
// checked on the device. An out-of-range subscript is redirected to element 0
// and recorded (first violation: array base, index, length; plus a count) in
// one device record per process, read by fx_bounds_report(). The Python side
// (tests/conftest.py) fails the test session when the record is non-empty.
#pragma once

#include <stdint.h>

namespace fx {

struct OobRecord {
  unsigned long long count;
  unsigned long long base;
  long long index;
  long long length;
};

// device record of this process (allocated on first use; nullptr in normal builds)
OobRecord *oob_record();

#ifdef FX_BOUNDS

template <class T>
struct CkPtr {
  T *p = nullptr;
  long long n = -1;  // -1: length unknown (unchecked)
  OobRecord *rep = nullptr;
  __host__ __device__ CkPtr() {}
  __host__ __device__ CkPtr(T *q) : p(q) {}
  __host__ __device__ CkPtr(T *q, long long len, OobRecord *r) : p(q), n(len), rep(r) {}
  __host__ __device__ operator T *() const { return p; }
  __host__ __device__ CkPtr &operator=(T *q) {
    p = q;
    n = -1;
    return *this;
  }
  __device__ T &operator[](long long i) const {
    if (n >= 0 && (i < 0 || i >= n)) {
      if (rep) {
        if (atomicAdd(&rep->count, 1ull) == 0ull) {
          rep->base = reinterpret_cast<unsigned long long>(p);
          rep->index = i;
          rep->length = n;
        }
      }
      return p[0];
    }
    return p[i];
  }
};

template <class T>
__host__ __device__ inline T *raw(const CkPtr<T> &q) {
  return q.p;
}
template <class T>
__host__ __device__ inline T *raw(T *q) {
  return q;
}
template <class T>
inline void ck_size(CkPtr<T> &q, long long n) {
  q.n = n;
  q.rep = oob_record();
}
template <class T>
inline void ck_size(T *&, long long) {}

#else

template <class T>
using CkPtr = T *;
template <class T>
__host__ __device__ inline T *raw(T *q) {
  return q;
}
template <class T>
inline void ck_size(T *&, long long) {}

#endif

}  // namespace fx
