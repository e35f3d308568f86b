/*
 * ORACLE — test infrastructure only.  det_exp: the deterministic fp32 exp of
 * the canonical arithmetic — Cody–Waite range reduction and a
 * degree-6 minimax polynomial, every step one IEEE op (fmaf / * / +), scaled
 * by 2^n in two exact halves.  Restates the definition that
 * paper_2505_10259_b200/csrc/det_math.cuh implements for the GPU.
 */
#ifndef ORACLE_DET_EXP_H
#define ORACLE_DET_EXP_H
#include <math.h>
#include <stdint.h>
#include <string.h>

static float o_det_exp(float x) {
  if (!(x > -87.0f)) return 0.0f;
  if (x > 88.0f) return INFINITY;
  float n = rintf(x * 1.44269504088896341f);
  float r = fmaf(-n, 0.693359375f, x);
  r = fmaf(-n, -2.12194440e-4f, r);
  float z = r * r;
  float p = 1.9875691500e-4f;
  p = fmaf(p, r, 1.3981999507e-3f);
  p = fmaf(p, r, 8.3334519073e-3f);
  p = fmaf(p, r, 4.1665795894e-2f);
  p = fmaf(p, r, 1.6666665459e-1f);
  p = fmaf(p, r, 5.0000001201e-1f);
  p = fmaf(p, z, r);
  p = p + 1.0f;
  int ni = (int)n;
  int n1 = ni / 2, n2 = ni - n1;
  uint32_t b1 = (uint32_t)(n1 + 127) << 23, b2 = (uint32_t)(n2 + 127) << 23;
  float s1, s2;
  memcpy(&s1, &b1, 4);
  memcpy(&s2, &b2, 4);
  return (p * s1) * s2;
}

#endif
