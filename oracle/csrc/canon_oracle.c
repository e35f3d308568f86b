/*
 * ORACLE — test infrastructure only.  CPU restatement of the canonical-order
 * model arithmetic (the parity mode of the B200 path), used by tests/ and
 * __graft_entry__.smoke() as the checker; never linked into the product.
 *
 * What it computes: the per-layer ops of the Mixtral / Mistral blocks the
 * verify and draft passes run (attention → FFN dataflow of PAPER.md:157 and
 * simulator.py:168-192; block arithmetic of transformers modeling_mixtral.py
 * / modeling_mistral.py, third-party, pinned in fp32 by
 * tests/golden/hf_tiny.npz), each with one definition of its float evaluation
 * order:
 *   dot(a, b)   acc = 0; for k in order: acc = fmaf(a_k, b_k, acc)
 *   gemm        C = epi(dot): bf16 | fp32 | bf16(bf16(acc) + r) | bf16(acc · w_r)
 *   swiglu      bf16(silu(dot(a, g)) · dot(a, u)), silu(g) = g / (1 + det_exp(-g))
 *   rmsnorm     ss = Σ fmaf(x, x, ss); r = 1 / sqrtf(ss / H + eps);
 *               y = bf16(bf16(x · r) · w)
 *   rope        y0 = x0·c − x1·s, y1 = x1·c + x0·s with c, s from a caller table
 *   attention   scores s_t = dot(q, k_t) · scale; m = max_t s_t;
 *               p_t = det_exp(s_t − m), Z = Σ p_t, o = Σ p_t · v_t (in key
 *               order), out = bf16(o / Z)
 *   router      l_e = dot(x, w_e); top-2 by strict > in expert order;
 *               w1 = 1 / (1 + det_exp(l0 − l1)), w0 = 1 − w1
 * Every float op is a single correctly rounded IEEE op (-ffp-contract=off,
 * fmaf = C99 fused multiply-add).  Written independently of
 * paper_2505_10259_b200/csrc/canon.cu; equality is what the tests check.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "det_exp.h"

enum { EPI_BF16 = 0, EPI_F32 = 1, EPI_BF16_RESID = 2, EPI_BF16_ROWSCALE = 4 };

static float b2f(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static uint16_t f2b(float f) { /* round to nearest even (finite inputs) */
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return (uint16_t)((u >> 16) | ((u & 0xffffu) ? 0x40u : 0u));
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

static float bfr(float f) { return b2f(f2b(f)); }

static float dot(const uint16_t* a, const uint16_t* b, int K) {
  float acc = 0.0f;
  for (int k = 0; k < K; ++k) acc = fmaf(b2f(a[k]), b2f(b[k]), acc);
  return acc;
}

static float silu(float g) { return g / (1.0f + o_det_exp(-g)); }

/* C[r, c] = epi(dot(A[r], B[c])), A [M, K], B [N, K] (bf16 bit patterns). */
void canon_gemm(const uint16_t* A, const uint16_t* B, int M, int N, int K, void* C, int ldc, int epi,
                const void* aux) {
  for (int r = 0; r < M; ++r) {
    for (int c = 0; c < N; ++c) {
      const float acc = dot(A + (size_t)r * K, B + (size_t)c * K, K);
      if (epi == EPI_F32) {
        ((float*)C)[(size_t)r * ldc + c] = acc;
        continue;
      }
      float v = acc;
      if (epi == EPI_BF16_RESID) v = bfr(acc) + b2f(((const uint16_t*)aux)[(size_t)r * ldc + c]);
      else if (epi == EPI_BF16_ROWSCALE) v = acc * ((const float*)aux)[r];
      ((uint16_t*)C)[(size_t)r * ldc + c] = f2b(v);
    }
  }
}

/* out[r, c] = bf16(silu(dot(A[r], G[c])) · dot(A[r], U[c])), G/U [N, K]. */
void canon_swiglu(const uint16_t* A, const uint16_t* G, const uint16_t* U, int M, int N, int K, uint16_t* out) {
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < N; ++c) {
      const float g = dot(A + (size_t)r * K, G + (size_t)c * K, K);
      const float u = dot(A + (size_t)r * K, U + (size_t)c * K, K);
      out[(size_t)r * N + c] = f2b(silu(g) * u);
    }
}

void canon_rmsnorm(const uint16_t* x, const uint16_t* w, int T, int H, float eps, uint16_t* out) {
  for (int t = 0; t < T; ++t) {
    const uint16_t* xr = x + (size_t)t * H;
    float ss = 0.0f;
    for (int i = 0; i < H; ++i) {
      const float v = b2f(xr[i]);
      ss = fmaf(v, v, ss);
    }
    const float r = 1.0f / sqrtf(ss / (float)H + eps);
    for (int i = 0; i < H; ++i) out[(size_t)t * H + i] = f2b(bfr(b2f(xr[i]) * r) * b2f(w[i]));
  }
}

/* x, out [T, heads, dh]; table [rows, dh] = cos | sin per position. */
void canon_rope(const uint16_t* x, int T, int heads, int dh, const int32_t* pos, const float* table,
                uint16_t* out) {
  const int half = dh / 2;
  for (int t = 0; t < T; ++t)
    for (int h = 0; h < heads; ++h) {
      const uint16_t* xr = x + ((size_t)t * heads + h) * dh;
      uint16_t* o = out + ((size_t)t * heads + h) * dh;
      const float* row = table + (size_t)pos[t] * dh;
      for (int i = 0; i < half; ++i) {
        const float c = row[i], s = row[half + i];
        const float x0 = b2f(xr[i]), x1 = b2f(xr[half + i]);
        o[i] = f2b(x0 * c - x1 * s);
        o[half + i] = f2b(x1 * c + x0 * s);
      }
    }
}

/* q [n_q, hq, dh]; keys/values [n_keys, hkv, dh] of one sequence; query row j
 * attends keys [0, p0 + j]; out [n_q, hq, dh]. */
void canon_attn(const uint16_t* q, const uint16_t* k, const uint16_t* v, int n_q, int p0, int hq, int hkv, int dh,
                float scale, uint16_t* out) {
  const int G = hq / hkv;
  float o[512];
  for (int j = 0; j < n_q; ++j)
    for (int h = 0; h < hq; ++h) {
      const uint16_t* qr = q + ((size_t)j * hq + h) * dh;
      const int g = h / G, n_keys = p0 + j + 1;
      float m = -INFINITY;
      for (int t = 0; t < n_keys; ++t) {
        const float s = dot(qr, k + ((size_t)t * hkv + g) * dh, dh) * scale;
        m = fmaxf(m, s);
      }
      for (int d = 0; d < dh; ++d) o[d] = 0.0f;
      float Z = 0.0f;
      for (int t = 0; t < n_keys; ++t) {
        const float p = o_det_exp(dot(qr, k + ((size_t)t * hkv + g) * dh, dh) * scale - m);
        Z = Z + p;
        const uint16_t* vr = v + ((size_t)t * hkv + g) * dh;
        for (int d = 0; d < dh; ++d) o[d] = fmaf(p, b2f(vr[d]), o[d]);
      }
      uint16_t* orow = out + ((size_t)j * hq + h) * dh;
      for (int d = 0; d < dh; ++d) orow[d] = f2b(o[d] / Z);
    }
}

void canon_route(const uint16_t* x, const uint16_t* wg, int T, int H, int E, int32_t* idx, float* w) {
  for (int t = 0; t < T; ++t) {
    float l0 = -INFINITY, l1 = -INFINITY;
    int i0 = 0, i1 = 1;
    for (int e = 0; e < E; ++e) {
      const float v = dot(x + (size_t)t * H, wg + (size_t)e * H, H);
      if (v > l0) {
        l1 = l0;
        i1 = i0;
        l0 = v;
        i0 = e;
      } else if (v > l1) {
        l1 = v;
        i1 = e;
      }
    }
    const float w1 = 1.0f / (1.0f + o_det_exp(l0 - l1));
    idx[2 * t] = i0;
    idx[2 * t + 1] = i1;
    w[2 * t] = 1.0f - w1;
    w[2 * t + 1] = w1;
  }
}
