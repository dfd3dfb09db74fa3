// Shared device helpers for the sdb200 kernels (sm_100a).
//
// Log-space conventions follow the reference's numerics (structdist
// numerics.py:32-46): max-shifted log-sum-exp, an all -inf slice reduces to
// -inf (never NaN), an empty reduction is -inf.  Transcendentals run on the
// MUFU pipe (ex2/lg2.approx) on SMALL-magnitude arguments only: every kernel
// keeps large log values either normalised per step (float) or in double, and
// exponentiates differences.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include <map>
#include <atomic>
#include <mutex>
#include <utility>

#include "../../include/sdb200.h"

#define SDB_LOG2E 1.4426950408889634f
#define SDB_LN2 0.6931471805599453f

__device__ __forceinline__ float ninf() { return __int_as_float(0xff800000); }
__device__ __forceinline__ double ninfd() { return __longlong_as_double(0xfff0000000000000ULL); }

// MUFU exp2 / log2 (ftz). ex2(-inf) = +0, lg2(0) = -inf.
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// natural exp/log through MUFU
__device__ __forceinline__ float fexp(float x) { return ex2(x * SDB_LOG2E); }
__device__ __forceinline__ float flog(float x) { return lg2(x) * SDB_LN2; }

__device__ __forceinline__ bool is_ninf(float x) { return x == ninf(); }
__device__ __forceinline__ bool is_ninfd(double x) { return x == ninfd(); }

// Input validity (numerics.py:22-29): NaN and +inf are rejected, -inf allowed.
// NaN or +inf (one unordered compare: !(x < +inf))
__device__ __forceinline__ bool bad_input(float x) { return !(x < __int_as_float(0x7f800000)); }
// NaN or +inf for either precision (the exact-mode kernels read float64 potentials)
__device__ __forceinline__ bool bad_value(float x) { return bad_input(x); }
__device__ __forceinline__ bool bad_value(double x) { return !(x < __longlong_as_double(0x7ff0000000000000LL)); }

// (max, sum exp(x - max)) accumulator for a log-sum-exp reduction.
struct Lse {
  float m, s;
  __device__ __forceinline__ Lse() : m(ninf()), s(0.f) {}
  __device__ __forceinline__ void add(float x) {
    if (x > m) {
      s = s * fexp(m - x) + 1.f;  // m=-inf -> s*0 + 1
      m = x;
    } else if (x != ninf()) {
      s += fexp(x - m);
    }
  }
  __device__ __forceinline__ void merge(float om, float os) {
    if (om > m) {
      s = s * fexp(m - om) + os;
      m = om;
    } else if (om != ninf()) {
      s += os * fexp(om - m);
    }
  }
  __device__ __forceinline__ float result() const { return m == ninf() ? ninf() : m + flog(s); }
};

// Same accumulator with a double max (for large-magnitude log values).
struct LseD {
  double m;
  float s;
  __device__ __forceinline__ LseD() : m(ninfd()), s(0.f) {}
  __device__ __forceinline__ void add(double x) {
    if (x > m) {
      s = s * fexp((float)(m - x)) + 1.f;
      m = x;
    } else if (x != ninfd()) {
      s += fexp((float)(x - m));
    }
  }
  __device__ __forceinline__ void merge(double om, float os) {
    if (om > m) {
      s = s * fexp((float)(m - om)) + os;
      m = om;
    } else if (om != ninfd()) {
      s += os * fexp((float)(om - m));
    }
  }
  __device__ __forceinline__ double result() const { return m == ninfd() ? ninfd() : m + (double)flog(s); }
};

// Full-warp float max as ONE redux.sync.max.u32 on order-preserving keys
// (sign-magnitude -> unsigned order; NaN maps to key 0, so like fmaxf it only
// wins when every lane is NaN) instead of five dependent shuffle+max rounds.
__device__ __forceinline__ float warp_max(float v) {
  const uint32_t u = __float_as_uint(v);
  uint32_t key = u ^ ((uint32_t)((int32_t)u >> 31) | 0x80000000u);
  key = (v != v) ? 0u : key;
  const uint32_t mk = __reduce_max_sync(0xffffffffu, key);
  return __uint_as_float(mk ^ (((mk >> 31) - 1u) | 0x80000000u));
}
// Full-warp max of doubles truncated to their high words (sign, exponent, 20
// mantissa bits): one REDUX on the same order-preserving keys as warp_max.  The
// result is within 2^-20 relative of the true maximum and, inside the fp32
// exponent range, exactly representable as a float.
__device__ __forceinline__ double warp_max_hi(double v) {
  const uint32_t u = (uint32_t)__double2hiint(v);
  const uint32_t key = u ^ ((uint32_t)((int32_t)u >> 31) | 0x80000000u);
  const uint32_t mk = __reduce_max_sync(0xffffffffu, key);
  return __hiloint2double((int)(mk ^ (((mk >> 31) - 1u) | 0x80000000u)), 0);
}
__device__ __forceinline__ float warp_max_shfl(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_maxd(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_or(int v) {
  return __any_sync(0xffffffffu, v) ? 1 : 0;
}

// warp log-sum-exp of one value per lane
__device__ __forceinline__ float warp_lse(float v) {
  float mx = warp_max(v);
  float e = (mx == ninf()) ? 0.f : fexp(v - mx);
  float s = warp_sum(e);
  return mx == ninf() ? ninf() : mx + flog(s);
}

// Workspace carving helper: 256-byte aligned sub-allocations.
struct Carve {
  char* p;
  size_t used;
  __host__ Carve(void* base) : p((char*)base), used(0) {}
  template <class T>
  __host__ T* take(size_t count) {
    size_t off = (used + 255) & ~(size_t)255;
    used = off + count * sizeof(T);
    return p ? (T*)(p + off) : nullptr;
  }
};

// last CUDA runtime error seen by an entry point (sdb_last_cuda_error)
inline std::atomic<int>& sdb_last_cuda() {
  static std::atomic<int> e{0};
  return e;
}
inline cudaError_t sdb_note(cudaError_t e) {
  if (e != cudaSuccess) sdb_last_cuda().store((int)e);
  return e;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel):
// the runtime call costs microseconds of host time on every launch otherwise
inline cudaError_t sdb_set_smem(const void* kern, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{dev, kern}];
  if (have >= smem) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) have = smem;
  return sdb_note(e);
}

#define SDB_CHECK_LAUNCH()                       \
  do {                                           \
    cudaError_t _e = cudaGetLastError();         \
    if (_e != cudaSuccess) {                     \
      sdb_note(_e);                              \
      return SDB_ERR_CUDA;                       \
    }                                            \
  } while (0)
