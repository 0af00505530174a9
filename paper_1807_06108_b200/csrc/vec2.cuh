// vec2.cuh -- two samples per thread in one register pair (sm_100 packed FP32).
//
// F2 holds the same scalar of two independent samples; its arithmetic maps
// one-to-one onto the packed f32x2 instructions FFMA2 / FMUL2 / FADD2 (one
// issue slot for both samples, the same IEEE round-to-nearest as the scalar
// FFMA / FMUL / FADD on each half), with a plain float operand issued as a
// broadcast (`R.F32` / `UR.F32` source), so a loop-invariant parameter costs
// one register, not two.  The per-lane results are bit-identical to the
// scalar code that performs the same operations in the same order -- which is
// why systems.cuh writes every multiply-add as an explicit fma: the scalar
// compile must not contract differently from the packed one.
//
// Scalar<V>::type is the parameter type of an arithmetic type V (float for
// F2, V itself otherwise); the device plugins (systems.cuh) take their
// constants as Scalar<V> and their state as V.
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

namespace jm {

using ::fma;  // the scalar fma(float|double, ...) stays visible next to the F2 overloads

struct F2 {
  float2 v;
  F2() = default;
  __device__ __forceinline__ explicit F2(float s) : v(make_float2(s, s)) {}  // broadcast
  __device__ __forceinline__ F2(float a, float b) : v(make_float2(a, b)) {}
  __device__ __forceinline__ explicit F2(float2 p) : v(p) {}
  __device__ __forceinline__ float lo() const { return v.x; }
  __device__ __forceinline__ float hi() const { return v.y; }
};

template <typename V>
struct Scalar {
  using type = V;
};
template <>
struct Scalar<F2> {
  using type = float;
};
template <typename V>
using scalar_t = typename Scalar<V>::type;

__device__ __forceinline__ float2 f2b(float s) { return make_float2(s, s); }

__device__ __forceinline__ F2 fma(F2 a, F2 b, F2 c) { return F2(__ffma2_rn(a.v, b.v, c.v)); }
__device__ __forceinline__ F2 fma(F2 a, float b, F2 c) { return F2(__ffma2_rn(a.v, f2b(b), c.v)); }
__device__ __forceinline__ F2 fma(float a, F2 b, F2 c) { return F2(__ffma2_rn(f2b(a), b.v, c.v)); }
__device__ __forceinline__ F2 fma(F2 a, F2 b, float c) { return F2(__ffma2_rn(a.v, b.v, f2b(c))); }
__device__ __forceinline__ F2 fma(F2 a, float b, float c) { return F2(__ffma2_rn(a.v, f2b(b), f2b(c))); }
__device__ __forceinline__ F2 fma(float a, F2 b, float c) { return F2(__ffma2_rn(f2b(a), b.v, f2b(c))); }

__device__ __forceinline__ F2 operator*(F2 a, F2 b) { return F2(__fmul2_rn(a.v, b.v)); }
__device__ __forceinline__ F2 operator*(F2 a, float b) { return F2(__fmul2_rn(a.v, f2b(b))); }
__device__ __forceinline__ F2 operator*(float a, F2 b) { return F2(__fmul2_rn(f2b(a), b.v)); }
__device__ __forceinline__ F2 operator+(F2 a, F2 b) { return F2(__fadd2_rn(a.v, b.v)); }
__device__ __forceinline__ F2 operator+(F2 a, float b) { return F2(__fadd2_rn(a.v, f2b(b))); }
__device__ __forceinline__ F2 operator+(float a, F2 b) { return F2(__fadd2_rn(f2b(a), b.v)); }
__device__ __forceinline__ F2 operator-(F2 a) { return F2(make_float2(-a.v.x, -a.v.y)); }
__device__ __forceinline__ F2 operator-(F2 a, F2 b) { return a + (-b); }
__device__ __forceinline__ F2 operator-(F2 a, float b) { return a + (-b); }
__device__ __forceinline__ F2 operator-(float a, F2 b) { return a + (-b); }
__device__ __forceinline__ F2& operator+=(F2& a, F2 b) { return a = a + b; }
__device__ __forceinline__ F2& operator-=(F2& a, F2 b) { return a = a - b; }
__device__ __forceinline__ F2& operator*=(F2& a, F2 b) { return a = a * b; }

// per-half helpers (no packed form exists: MUFU, compares, integer ops)
__device__ __forceinline__ F2 rcp_r(F2 x) {
  float a, b;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(x.v.x));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(x.v.y));
  return F2(a, b);
}
__device__ __forceinline__ bool both_finite(F2 x) { return isfinite(x.v.x) && isfinite(x.v.y); }

// lane access of the generic per-sample code: half h of V (h = 0 for scalars)
__device__ __forceinline__ float half_of(F2 x, int h) { return h ? x.v.y : x.v.x; }
__device__ __forceinline__ float half_of(float x, int) { return x; }
__device__ __forceinline__ double half_of(double x, int) { return x; }

}  // namespace jm
