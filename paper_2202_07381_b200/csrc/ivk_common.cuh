// Shared helpers for libivk (sm_100a).  Error plumbing, launch accounting,
// cache-hinted loads.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <atomic>
#include <string>

#include "../../include/ivk.h"

namespace ivk {

void set_error(const char* fmt, ...);
int check_launch(const char* what);
extern std::atomic<long long> g_launches;

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kSMs = 148;  // B200

// Streaming (evict-first, no L1 allocate) load for data read exactly once per
// sweep -- the patch-inverse stream must not evict the L2-resident vectors.
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.L1::no_allocate.L2::evict_first.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_stream2(const double2* p) {
  double2 v;
  asm volatile("ld.global.L1::no_allocate.L2::evict_first.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
// L2-resident (evict-last) read-only loads for vectors that are gathered.
__device__ __forceinline__ double ld_keep(const double* p) {
  double v;
  asm volatile("ld.global.nc.L2::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

}  // namespace ivk

#define IVK_REQUIRE(cond, ...)            \
  do {                                    \
    if (!(cond)) {                        \
      ::ivk::set_error(__VA_ARGS__);      \
      return IVK_EINVAL;                  \
    }                                     \
  } while (0)
