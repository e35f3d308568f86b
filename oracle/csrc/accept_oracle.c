/*
 * ORACLE — test infrastructure only.  CPU restatement of the speculative
 * accept/reject step, used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the checker; never linked into the product.
 *
 * Semantics (reference + paper):
 *   - committed tokens per round = longest correct draft prefix + 1 bonus,
 *     on {1..n_cand+1}: pkg/src/specpipe/acceptance.py:1-6;
 *   - clamp to the remaining budget: pkg/src/specpipe/simulator.py:213-214,
 *     SPEC.md:265;
 *   - sampling verification = Leviathan et al. Alg. 1 (
 *     third-party call site transformers generation/utils.py
 *     `_speculative_sampling`).
 * Arithmetic: the canonical deterministic order of DESIGN.md §K7 — every float
 * op is a single correctly-rounded IEEE op (compiled with -ffp-contract=off),
 * exp is the Cody–Waite/minimax det_exp, sums run over 256 contiguous chunks
 * left to right.  This file is written independently of the CUDA kernel
 * (paper_2505_10259_b200/csrc/accept.cu); agreement is what the tests check.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define NCHUNK 256

#include "det_exp.h"
#define o_exp o_det_exp

float oracle_det_exp(float x) { return o_exp(x); }

static void chunk_bounds(int V, int c, int* lo, int* hi) {
  int C = (V + NCHUNK - 1) / NCHUNK;
  *lo = c * C;
  *hi = *lo + C;
  if (*lo > V) *lo = V;
  if (*hi > V) *hi = V;
}

/* weights of a row: kind 0 = exp(inv_t (l - max)); kind 1 = max(w/Z - q, 0) */
typedef struct {
  const float* l;
  const float* q;
  float mx, inv_t, Z;
  int kind;
} Row;

static float row_w(const Row* R, int v) {
  float w = o_exp((R->l[v] - R->mx) * R->inv_t);
  if (R->kind == 0) return w;
  float p = w / R->Z;
  float d = p - R->q[v];
  return d > 0.0f ? d : 0.0f;
}

static float row_max(const float* l, int V) {
  float m = -INFINITY;
  for (int v = 0; v < V; ++v) m = fmaxf(m, l[v]);
  return m;
}

static float row_total(const Row* R, int V, float* chunk) {
  for (int c = 0; c < NCHUNK; ++c) {
    int lo, hi;
    chunk_bounds(V, c, &lo, &hi);
    float a = 0.0f;
    for (int v = lo; v < hi; ++v) a = a + row_w(R, v);
    chunk[c] = a;
  }
  float t = 0.0f;
  for (int c = 0; c < NCHUNK; ++c) t = t + chunk[c];
  return t;
}

static int row_pick(const Row* R, int V, const float* chunk, float target) {
  float acc = 0.0f, base = 0.0f;
  int cstar = -1;
  for (int c = 0; c < NCHUNK; ++c) {
    float nxt = acc + chunk[c];
    if (nxt > target) {
      cstar = c;
      base = acc;
      break;
    }
    acc = nxt;
  }
  if (cstar >= 0) {
    int lo, hi, last = -1;
    chunk_bounds(V, cstar, &lo, &hi);
    float a = base;
    for (int v = lo; v < hi; ++v) {
      float w = row_w(R, v);
      if (w > 0.0f) last = v;
      a = a + w;
      if (a > target) return v;
    }
    if (last >= 0) return last;
  }
  for (int v = V - 1; v >= 0; --v)
    if (row_w(R, v) > 0.0f) return v;
  return 0;
}

static int argmax_low(const float* l, int V) {
  int bi = 0;
  float bv = -INFINITY;
  int found = 0;
  for (int v = 0; v < V; ++v) {
    if (l[v] > bv) {
      bv = l[v];
      bi = v;
      found = 1;
    }
  }
  return found ? bi : 0;
}

static void emit(int n_cand, int n_acc, int final_tok, const int32_t* draft, int rem, int32_t* out_tok,
                 int32_t* out_cnt) {
  int count = n_acc + 1;
  if (count > rem) count = rem < 0 ? 0 : rem;
  for (int j = 0; j <= n_cand; ++j) {
    int tok = j < n_acc ? draft[j] : (j == n_acc ? final_tok : -1);
    out_tok[j] = j < count ? tok : -1;
  }
  *out_cnt = count;
}

void oracle_accept_greedy(const int32_t* draft, const float* logits, const int32_t* remaining,
                          const int32_t* forced, int bs, int n_cand, int V, int32_t* out_tokens,
                          int32_t* out_counts) {
  for (int s = 0; s < bs; ++s) {
    const float* L = logits + (size_t)s * (n_cand + 1) * V;
    const int32_t* d = draft + (size_t)s * n_cand;
    int n_acc = 0;
    while (n_acc < n_cand && d[n_acc] == argmax_low(L + (size_t)n_acc * V, V)) ++n_acc;
    if (forced) {
      int f = forced[s] - 1;
      n_acc = f < 0 ? 0 : (f > n_cand ? n_cand : f);
    }
    int final_tok = argmax_low(L + (size_t)n_acc * V, V);
    emit(n_cand, n_acc, final_tok, d, remaining[s], out_tokens + (size_t)s * (n_cand + 1), out_counts + s);
  }
}

void oracle_accept_sample(const int32_t* draft, const float* logits, const float* qprobs, const float* u_acc,
                          const float* u_res, const int32_t* remaining, float inv_t, int bs, int n_cand, int V,
                          int32_t* out_tokens, int32_t* out_counts) {
  float chunk[NCHUNK];
  for (int s = 0; s < bs; ++s) {
    const float* L = logits + (size_t)s * (n_cand + 1) * V;
    const float* Q = qprobs + (size_t)s * n_cand * V;
    const int32_t* d = draft + (size_t)s * n_cand;
    int n_acc = n_cand, final_tok = 0;
    for (int i = 0; i <= n_cand; ++i) {
      Row W = {L + (size_t)i * V, Q + (size_t)i * V, 0.0f, inv_t, 0.0f, 0};
      W.mx = row_max(W.l, V);
      float Z = row_total(&W, V, chunk);
      W.Z = Z;
      if (i == n_cand) {
        final_tok = row_pick(&W, V, chunk, u_res[s] * Z);
        n_acc = n_cand;
        break;
      }
      float p = row_w(&W, d[i]) / Z;
      float q = Q[(size_t)i * V + d[i]];
      if (u_acc[(size_t)s * n_cand + i] * q <= p) continue;
      Row R = W;
      R.kind = 1;
      float Rt = row_total(&R, V, chunk);
      if (Rt > 0.0f) {
        final_tok = row_pick(&R, V, chunk, u_res[s] * Rt);
      } else {
        float Z2 = row_total(&W, V, chunk);
        final_tok = row_pick(&W, V, chunk, u_res[s] * Z2);
      }
      n_acc = i;
      break;
    }
    emit(n_cand, n_acc, final_tok, d, remaining[s], out_tokens + (size_t)s * (n_cand + 1), out_counts + s);
  }
}

void oracle_sample_tokens(const float* logits, const float* uniforms, float inv_t, int rows, int V,
                          int32_t* out_tokens, float* out_probs) {
  float chunk[NCHUNK];
  for (int r = 0; r < rows; ++r) {
    const float* l = logits + (size_t)r * V;
    if (!uniforms && !out_probs) {
      out_tokens[r] = argmax_low(l, V);
      continue;
    }
    Row W = {l, 0, row_max(l, V), inv_t, 0.0f, 0};
    float Z = row_total(&W, V, chunk);
    W.Z = Z;
    if (out_probs)
      for (int v = 0; v < V; ++v) out_probs[(size_t)r * V + v] = row_w(&W, v) / Z;
    out_tokens[r] = uniforms ? row_pick(&W, V, chunk, uniforms[r] * Z) : argmax_low(l, V);
  }
}
