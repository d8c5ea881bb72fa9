// Packed fp32 pair arithmetic (sm_100a FADD2 / FMUL2 / FFMA2).
//
// Each lane of add.rn.f32x2 / mul.rn.f32x2 is one correctly rounded IEEE
// operation, so pairs of reference operations can be issued as one
// instruction.  Caveat measured on nvcc 12.9: ptxas contracts
// mul.rn.f32x2 -> add.rn.f32x2 chains into FFMA2 even with -fmad=false, so
// EXACT-mode code forms products with scalar __fmul_rn (never contracted)
// and only sums/differences with the packed forms -- or packed products as
// FFMA2 with an opaque -0 addend (xmul2 below).
#pragma once

#include <cstdint>

namespace stb {

typedef unsigned long long f2;

__device__ __forceinline__ f2 pk(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk(f2 v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
// Exact packed product: fma.rn(a, b, -0) is bitwise a*b (a*b = +0 gives
// +0 + -0 = +0).  nz must be -0 held in a register whose value ptxas cannot
// see (a kernel parameter): with a literal -0 it folds the FFMA2 into a
// following FADD2 exactly as it contracts mul.rn.f32x2; with an opaque
// addend it cannot, so the product and the sum stay separately rounded.
__device__ __forceinline__ f2 xmul2(f2 a, f2 b, f2 nz) { return fma2(a, b, nz); }
// scalar-coefficient product formed with two uncontractable scalar muls
__device__ __forceinline__ f2 smul2(f2 a, float c) {
  float lo, hi;
  upk(a, lo, hi);
  return pk(__fmul_rn(lo, c), __fmul_rn(hi, c));
}
__device__ __forceinline__ f2 bcast(float c) { return pk(c, c); }

}  // namespace stb
