// common.cuh -- shared device helpers for libgscan (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/gscan.h"

namespace gs {

// ---------------------------------------------------------------------------
// error plumbing: thread-local message, no exceptions across the C-ABI
void set_error(const std::string& msg);
std::string cuda_msg(cudaError_t e, const char* what, const char* file, int line);

#define GS_CUDA(call)                                                          \
  do {                                                                         \
    cudaError_t _e = (call);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::gs::set_error(::gs::cuda_msg(_e, #call, __FILE__, __LINE__));          \
      return _e == cudaErrorMemoryAllocation ? GS_ENOMEM : GS_ECUDA;           \
    }                                                                          \
  } while (0)

#define GS_TRY(call)                                                           \
  do {                                                                         \
    int _r = (call);                                                           \
    if (_r != GS_OK) return _r;                                                \
  } while (0)

// ---------------------------------------------------------------------------
// per-edge similarity status (scan.py:38-40) and role codes (scan.py:43-52)
// SIM_PENDING: identify stage 1 could not decide the edge; stage 2 decides it
// (or resets it to SIM_UNKNOWN when pruning skips it), so it never outlives identify
enum : uint8_t { SIM_UNKNOWN = 0, SIM_SIMILAR = 1, SIM_DISSIMILAR = 2, SIM_PENDING = 3 };
enum : uint8_t {
  ROLE_UNKNOWN = 0,
  ROLE_CORE = 1,
  ROLE_NONCORE = 2,
  ROLE_MEMBER = 3,
  ROLE_HUB = 5,
  ROLE_OUTLIER = 6
};

// ---------------------------------------------------------------------------
// Exact threshold (scan.py:232-233):  (c+2)^2 * q >= p * (da+1)(db+1).
// x = (c+2)^2 < 2^64, d = (da+1)(db+1) < 2^64, p,q < 2^128 -> 192-bit compare.
struct Eps2 {
  uint64_t p_lo, p_hi, q_lo, q_hi;
  double ratio;  // p/q as a double, only used to seed c_min (then verified)
};

__host__ __device__ __forceinline__ void mul64x128(uint64_t x, uint64_t lo, uint64_t hi,
                                                   uint64_t& r0, uint64_t& r1,
                                                   uint64_t& r2) {
#ifdef __CUDA_ARCH__
  r0 = x * lo;
  uint64_t c0 = __umul64hi(x, lo);
  uint64_t m1 = x * hi;
  uint64_t m2 = __umul64hi(x, hi);
  r1 = m1 + c0;
  r2 = m2 + (r1 < m1 ? 1u : 0u);
#else
  unsigned __int128 a = (unsigned __int128)x * lo;
  unsigned __int128 b = (unsigned __int128)x * hi + (uint64_t)(a >> 64);
  r0 = (uint64_t)a;
  r1 = (uint64_t)b;
  r2 = (uint64_t)(b >> 64);
#endif
}

__host__ __device__ __forceinline__ bool pred_ge(uint64_t x, uint64_t d, const Eps2& e) {
  uint64_t a0, a1, a2, b0, b1, b2;
  mul64x128(x, e.q_lo, e.q_hi, a0, a1, a2);
  mul64x128(d, e.p_lo, e.p_hi, b0, b1, b2);
  if (a2 != b2) return a2 > b2;
  if (a1 != b1) return a1 > b1;
  return a0 >= b0;
}

__host__ __device__ __forceinline__ bool is_similar(int64_t c, int64_t da, int64_t db,
                                                    const Eps2& e) {
  uint64_t s = (uint64_t)(c + 2);
  return pred_ge(s * s, (uint64_t)(da + 1) * (uint64_t)(db + 1), e);
}

// Smallest c >= 0 with is_similar(c, da, db); returns a value > cmax when
// even cmax common neighbours are not enough.  Seeded by a double estimate,
// then corrected with the exact predicate so the result is exact.
__device__ __forceinline__ int64_t c_min_exact(int64_t da, int64_t db, int64_t cmax,
                                               const Eps2& e) {
  double dd = (double)(da + 1) * (double)(db + 1);
  double est = sqrt(e.ratio * dd) - 2.0;
  int64_t c = est <= 0.0 ? 0 : (int64_t)ceil(est);
  if (c > cmax + 1) c = cmax + 1;
  while (c > 0 && is_similar(c - 1, da, db, e)) --c;
  while (c <= cmax && !is_similar(c, da, db, e)) ++c;
  return c;
}

// ---------------------------------------------------------------------------
// warp helpers
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

// multiplicative hash to [0, T) without a power-of-two table
__device__ __forceinline__ uint32_t hslot(uint32_t key, uint32_t T) {
  return __umulhi(key * 0x9E3779B1u, T);
}

}  // namespace gs
