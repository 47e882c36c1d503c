// Shared helpers for the pc_b200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/pc_b200.h"

namespace pc {

void set_error(const std::string& msg);

// Status helpers -----------------------------------------------------------
#define PC_REQUIRE(cond, code, ...)                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      char _b[512];                                                   \
      snprintf(_b, sizeof(_b), __VA_ARGS__);                          \
      ::pc::set_error(_b);                                            \
      return (code);                                                  \
    }                                                                 \
  } while (0)

void count_launches(int n);

// Programmatic dependent launch: a bandwidth kernel lets the next tensor-core
// GEMM (launched with programmatic stream serialization) start its prologue
// (barrier init, TMEM allocation, descriptor prefetch) while this kernel's last
// blocks run; the GEMM waits (griddepcontrol.wait) before touching global memory.
#define PC_PDL_TRIGGER() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")

// Every kernel launch site is followed by this check; it also feeds the
// launch counter behind pc_launch_count() (one launch per check unless the
// site calls count_launches() for the extra ones).
#define PC_CUDA_CHECK_LAUNCH(what)                                                   \
  do {                                                                               \
    ::pc::count_launches(1);                                                         \
    cudaError_t _e = cudaGetLastError();                                             \
    if (_e != cudaSuccess) {                                                         \
      ::pc::set_error(std::string(what) + ": " + cudaGetErrorString(_e));            \
      return PC_ECUDA;                                                               \
    }                                                                                \
  } while (0)

inline cudaStream_t S(pc_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Element access in either storage precision --------------------------------
template <typename T> __device__ __forceinline__ float ld(const T* p);
template <> __device__ __forceinline__ float ld<float>(const float* p) { return __ldg(p); }
template <> __device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}
template <typename T> __device__ __forceinline__ T cvt(float v);
template <> __device__ __forceinline__ float cvt<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// Channel-blocked addressing (see pc_b200.h).
struct Blocked {
  long long ld, cb, bstride;
  __host__ __device__ __forceinline__ long long at(long long r, long long c) const {
    long long blk = c / cb;
    return blk * bstride + r * ld + (c - blk * cb);
  }
};

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// Division by a runtime-invariant divisor d (Granlund-Montgomery round-up method):
// q = (umulhi(n, m) + n) >> l for n < 2^31 — three instructions instead of the
// ~20-instruction reciprocal sequence of a runtime integer division.
struct FastDiv {
  uint32_t d, m, l;
  FastDiv() = default;
  explicit FastDiv(uint32_t div) : d(div), m(0), l(0) {
    while ((1ull << l) < div) ++l;
    m = (uint32_t)(((1ull << 32) * ((1ull << l) - div)) / div + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> l; }
};

}  // namespace pc
