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
// (the L2::evict_first qualifier needs a 256-bit vector on sm_100a; 128-bit
// streams use the cache-streaming .cs hint instead)
__device__ __forceinline__ double2 ld_stream2(const double2* p) { return __ldcs(p); }

// ---- TMA bulk copies (cp.async.bulk global -> shared, mbarrier completion) --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  // the slot was last read through the generic proxy (before a CTA barrier)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

}  // namespace ivk

#define IVK_REQUIRE(cond, ...)            \
  do {                                    \
    if (!(cond)) {                        \
      ::ivk::set_error(__VA_ARGS__);      \
      return IVK_EINVAL;                  \
    }                                     \
  } while (0)
