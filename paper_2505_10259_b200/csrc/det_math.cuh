// Deterministic fp32 arithmetic for the sampling-mode accept/reject kernel.
//
// "Bit-exact given identical logits and uniforms" (BASELINE.json north star)
// needs every float operation on the decision path to be a correctly rounded
// IEEE op with a fixed evaluation order.  CUDA's expf and glibc's expf differ
// in the last ulp, and nvcc contracts a*b+c into FMA by default, so this file
// spells out:
//   * det_exp: Cody–Waite range reduction + degree-6 minimax polynomial, all
//     with explicit __fmaf_rn/__fmul_rn/__fadd_rn (no contraction);
//   * the canonical summation order over a vocabulary row: NCHUNK contiguous
//     chunks, each summed left-to-right, chunk sums then summed left-to-right.
// oracle/csrc/accept_oracle.c restates the same definition independently for
// the CPU (DESIGN.md §K7 is the normative text).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define SO_NCHUNK 256  // threads per vocabulary row == canonical chunk count

__device__ __forceinline__ float d_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float d_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float d_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float d_fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ float d_div(float a, float b) { return __fdiv_rn(a, b); }

__device__ __forceinline__ float det_exp(float x) {
  if (!(x > -87.0f)) return 0.0f;  // also maps NaN / -inf to 0
  if (x > 88.0f) return __int_as_float(0x7f800000);
  const float n = rintf(d_mul(x, 1.44269504088896341f));
  float r = d_fma(-n, 0.693359375f, x);
  r = d_fma(-n, -2.12194440e-4f, r);
  const float z = d_mul(r, r);
  float p = 1.9875691500e-4f;
  p = d_fma(p, r, 1.3981999507e-3f);
  p = d_fma(p, r, 8.3334519073e-3f);
  p = d_fma(p, r, 4.1665795894e-2f);
  p = d_fma(p, r, 1.6666665459e-1f);
  p = d_fma(p, r, 5.0000001201e-1f);
  p = d_fma(p, z, r);
  p = d_add(p, 1.0f);
  // scale by 2^n in two exact halves so that neither factor over/underflows
  const int ni = (int)n;
  const int n1 = ni / 2;
  const int n2 = ni - n1;
  const float s1 = __int_as_float((n1 + 127) << 23);
  const float s2 = __int_as_float((n2 + 127) << 23);
  return d_mul(d_mul(p, s1), s2);
}

// Chunk bounds of the canonical order: chunk c of a row of length V.
__device__ __forceinline__ void det_chunk(int V, int c, int& lo, int& hi) {
  const int C = (V + SO_NCHUNK - 1) / SO_NCHUNK;
  lo = c * C;
  hi = lo + C;
  if (lo > V) lo = V;
  if (hi > V) hi = V;
}
