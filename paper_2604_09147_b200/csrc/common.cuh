// common.cuh — shared device/host utilities of libhh (CUDA path only; never used by oracle/).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/hh.h"

namespace hh {

// ------------------------------------------------------------------ error plumbing
struct Error : std::runtime_error {
  hh_status st;
  Error(hh_status s, const std::string &m) : std::runtime_error(m), st(s) {}
};

#define HH_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t e__ = (call);                                                              \
    if (e__ != cudaSuccess)                                                                \
      throw ::hh::Error(e__ == cudaErrorMemoryAllocation ? HH_ENOMEM : HH_ECUDA,           \
                        std::string(#call) + ": " + cudaGetErrorString(e__) + " @" +       \
                            __FILE__ + ":" + std::to_string(__LINE__));                    \
  } while (0)

#define HH_REQUIRE(cond, status, msg)                                                      \
  do {                                                                                     \
    if (!(cond)) throw ::hh::Error(status, msg);                                           \
  } while (0)

void count_launch(int n = 1);  // launch accounting (api.cpp)

#define HH_LAUNCHED()                                                                      \
  do {                                                                                     \
    ::hh::count_launch();                                                                  \
    cudaError_t e__ = cudaGetLastError();                                                  \
    if (e__ != cudaSuccess)                                                                \
      throw ::hh::Error(HH_ECUDA, std::string("launch: ") + cudaGetErrorString(e__) +      \
                                      " @" + __FILE__ + ":" + std::to_string(__LINE__));   \
  } while (0)

// ------------------------------------------------------------------ constants
constexpr int TAG_FP64 = 0, TAG_FP32 = 1, TAG_FP16 = 2, TAG_BF16 = 3, TAG_Q43 = 4, TAG_BF24 = 5, TAG_FP48 = 6;
constexpr int NTAG = 7;
constexpr int KIND_FAR = 0, KIND_NBR = 1, KIND_SIB = 2, KIND_LNBR = 3, KIND_DIAG = 4;
constexpr int STORE_LR = 0, STORE_DENSE = 1;
constexpr int64_t ALIGN = 16;
__host__ __device__ inline int tag_bytes(int t) {
  return t == TAG_FP64 ? 8 : t == TAG_FP32 ? 4 : t == TAG_Q43 ? 1 : t == TAG_BF24 ? 3 : t == TAG_FP48 ? 6 : 2;
}
inline int64_t align_up(int64_t x, int64_t a = ALIGN) { return (x + a - 1) / a * a; }

// ------------------------------------------------------------------ kernel functions
// f(r) of Eq. 5.1.  Distance computed as sqrt(sum (x_k - y_k)^2).
struct KernelFn {
  int kind;
  double scale;     // GAUSS: -1/(2 s^2) stored in c; EXP: -1/s in c
  double c;
};

__device__ __forceinline__ double kernel_eval(const KernelFn &K, double r2) {
  // r2 = squared distance, > 0 for distinct points; singular kernels at r2 == 0 -> 0 (G18)
  switch (K.kind) {
    case HH_K_LOG:
      return r2 > 0.0 ? 0.5 * log(r2) : 0.0;
    case HH_K_INV_R:
      return r2 > 0.0 ? 1.0 / sqrt(r2) : 0.0;
    case HH_K_INV_R2:
      return r2 > 0.0 ? 1.0 / r2 : 0.0;
    case HH_K_GAUSS:
      return exp(r2 * K.c);
    default:  // HH_K_EXP
      return exp(sqrt(r2) * K.c);
  }
}

// ------------------------------------------------------------------ storage rounding
// Single round-to-nearest-even from float64 to an (M mantissa bits, EMIN, EMAX) format,
// subnormals kept, overflow -> inf (reading G16).  Returns the bit pattern of the target.
template <int M, int EMIN, int EMAX>
__host__ __device__ inline uint32_t rne_bits(double x) {
  uint64_t b;
  memcpy(&b, &x, 8);
  const uint32_t sign = (uint32_t)(b >> 63);
  const uint64_t a = b & 0x7FFFFFFFFFFFFFFFull;
  constexpr int EBITS = (EMAX == 15) ? 5 : (EMAX == 7) ? 4 : 8;
  constexpr uint32_t INF = ((1u << EBITS) - 1u) << M;
  const uint32_t sbit = sign << (M + EBITS);
  if (a >= 0x7FF0000000000000ull) {  // inf / nan
    return sbit | INF | (a > 0x7FF0000000000000ull ? (1u << (M - 1)) : 0u);
  }
  if (a == 0) return sbit;
  int e = (int)(a >> 52);
  uint64_t mant = a & 0xFFFFFFFFFFFFFull;
  if (e == 0) {  // fp64 subnormal: far below every target's range
    return sbit;
  }
  mant |= 1ull << 52;
  int E = e - 1023;
  if (E > EMAX) return sbit | INF;
  int shift = 52 - M;             // bits dropped for a normal result
  int biased;
  if (E >= EMIN) {
    biased = E - EMIN + 1;        // target biased exponent (>= 1)
  } else {
    shift += EMIN - E;            // subnormal: drop more bits
    biased = 0;
    if (shift > 63) return sbit;  // rounds to zero (below half the smallest subnormal)
  }
  uint64_t keep = mant >> shift;
  uint64_t rem = mant & ((1ull << shift) - 1ull);
  uint64_t half = 1ull << (shift - 1);
  if (rem > half || (rem == half && (keep & 1ull))) keep += 1;
  // assemble: for normals keep includes the hidden bit; adding handles binade carry
  uint64_t r;
  if (biased > 0) {
    r = ((uint64_t)biased << M) + (keep - (1ull << M));
  } else {
    r = keep;  // subnormal, may carry into the smallest normal
  }
  if (r >= INF) return sbit | INF;
  return sbit | (uint32_t)r;
}

__host__ __device__ inline uint16_t to_fp16_bits(double x) { return (uint16_t)rne_bits<10, -14, 15>(x); }
__host__ __device__ inline uint16_t to_bf16_bits(double x) { return (uint16_t)rne_bits<7, -126, 127>(x); }
__host__ __device__ inline uint32_t to_fp32_bits(double x) { return rne_bits<23, -126, 127>(x); }
// q43 (Table 1: 1-4-3, e_min -6, e_max 7): exponent field 15 = inf, x_max = 240
__host__ __device__ inline uint8_t to_q43_bits(double x) { return (uint8_t)rne_bits<3, -6, 7>(x); }
// accessor formats: bf24 = 1-8-15 (fp32's range, the top 24 bits of an fp32)
__host__ __device__ inline uint32_t to_bf24_bits(double x) { return rne_bits<15, -126, 127>(x); }
// fp48 = 1-11-36 (fp64's range, the top 48 bits of an fp64): RNE at bit 16 of the fp64 pattern
// (normals and subnormals alike: a 1-11-36 subnormal has spacing 2^(-1022-36) = 2^16 fp64
// subnormal ulps); a carry into the exponent field is the correct rounding, inf stays inf
__host__ __device__ inline uint64_t to_fp48_bits(double x) {
  uint64_t b;
  memcpy(&b, &x, 8);
  const uint64_t mag = b & 0x7FFFFFFFFFFFFFFFull;
  if (mag >= 0x7FF0000000000000ull) return b >> 16;  // inf / nan
  const uint64_t r = mag + 0x7FFFull + ((mag >> 16) & 1ull);
  return ((b & 0x8000000000000000ull) | (r & 0xFFFFFFFFFFFF0000ull)) >> 16;
}

}  // namespace hh
