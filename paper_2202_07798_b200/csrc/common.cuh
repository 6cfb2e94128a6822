// common.cuh — shared device helpers: precision-generic math, status,
// error plumbing.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/bbml.h"
#include "f64math.cuh"

namespace bbml {

// Accurate (non-approx) transcendentals.  tanh.approx.f32 is NOT used: the
// survey measured it at 4.4e-4 relative on predicted counts.
__device__ __forceinline__ float f_tanh(float x) { return tanhf(x); }
__device__ __forceinline__ double f_tanh(double x) { return tanh(x); }
__device__ __forceinline__ float f_exp(float x) { return expf(x); }
__device__ __forceinline__ double f_exp(double x) { return exp(x); }
__device__ __forceinline__ float f_log(float x) { return logf(x); }
__device__ __forceinline__ double f_log(double x) { return log(x); }
__device__ __forceinline__ float f_log1p(float x) { return log1pf(x); }
__device__ __forceinline__ double f_log1p(double x) { return log1p(x); }
__device__ __forceinline__ float f_sqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ double f_sqrt(double x) { return sqrt(x); }
__device__ __forceinline__ bool f_finite(float x) { return isfinite(x); }
__device__ __forceinline__ bool f_finite(double x) { return isfinite(x); }

// numpy.logaddexp(0, z) (npy_math logaddexp): z < 0 -> log1p(exp(z)),
// z > 0 -> z + log1p(exp(-z)), z == 0 -> ln 2 (= log1p(exp(0))), NaN -> NaN.
// Written branch-free (max(z,0) + log1p(exp(-|z|))) so a warp never runs both
// sides; the value is the same expression numpy evaluates on either side.
template <typename T>
__device__ __forceinline__ T softplus(T z) {
  const T m = z > T(0) ? z : T(0);
  return m + f_log1p(f_exp(-fabs(z)));
}

// FP32 tanh in ~12 instructions (vs ~31 for tanhf): odd Taylor polynomial for
// |x| < 0.125 (truncation < 2e-10 relative), else (1 - e)/(1 + e) with
// e = 2^(-2|x| log2 e) from MUFU.EX2 (~1e-6 relative).  NOT tanh.approx.f32
// (5e-4 relative).
__device__ __forceinline__ float tanh_fast(float x) {
  const float ax = fabsf(x);
  const float x2 = x * x;
  const float poly = x * (1.0f + x2 * (-0.333333343f + x2 * (0.133333340f + x2 * -0.0539682540f)));
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-2.8853900817779268f * ax));
  const float big = __fdividef(1.0f - e, 1.0f + e);
  return ax < 0.125f ? poly : copysignf(big, x);
}

// brbpnn.tansig (brbpnn.py:33-38): 2/(1+exp(-2x)) - 1, saturating, with the
// branch-free (bit-identical) division of f64math.cuh, so the per-sample
// loops of the LM kernels overlap more of consecutive samples' tansig chains.
// BBML_TANSIG_EXP_BF also swaps exp for the branch-free one (within 1 ulp of
// libdevice: LM call 455 -> 428 ms on suite16, but the near-chaotic BR fits
// then move by more than the artifact test's tolerance -- not the default).
__device__ __forceinline__ double tansig(double x) {
#ifdef BBML_TANSIG_EXP_BF
  const double t = __dsub_rn(div_rn_bf(2.0, __dadd_rn(1.0, exp_any_bf(-2.0 * x))), 1.0);
  return x != x ? x : t;
#else
  // exp from libdevice (bit-identical results to r01), division branch-free
  const double e = exp(-2.0 * x);
  const double t = __dsub_rn(div_rn_bf(2.0, __dadd_rn(1.0, e)), 1.0);
  return e == INFINITY ? -1.0 : t;  // 2 / inf = 0 exactly in IEEE; div_rn_bf(2, inf) is not
#endif
}

__device__ __forceinline__ double shfl_xor(double v, int m, unsigned mask = 0xffffffffu,
                                           int width = 32) {
  return __shfl_xor_sync(mask, v, m, width);
}
__device__ __forceinline__ float shfl_xor(float v, int m, unsigned mask = 0xffffffffu,
                                          int width = 32) {
  return __shfl_xor_sync(mask, v, m, width);
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// thread-local last-error string
void set_error(const char* fmt, ...);
bbml_status cuda_status(cudaError_t e, const char* what);

}  // namespace bbml
