// K7 — speculative accept / reject on the target's verification logits.
//
// Reference semantics: acceptance.py:1-6 (longest correct prefix + one bonus
// token, committed count on {1..n_cand+1}); clamp to the remaining budget
// simulator.py:213-214 / SPEC.md:265.  The reference only *samples* the count
// (acceptance.py:55-72); here the count is decided on real logits.
//
// One CTA (256 threads) per sequence.  Greedy mode reads each of the n_cand+1
// logit rows once with 16-B loads, block-reduces the argmax (lowest index on
// ties, like torch.argmax), and finds the first mismatch with one warp ballot:
// lane i holds (draft[i] == argmax[i]); the accepted prefix length is the
// count of trailing ones of the ballot — a warp-scan prefix acceptance.
#include "common.cuh"
#include "det_math.cuh"

namespace {

constexpr int kThreads = SO_NCHUNK;  // 256
constexpr int kMaxCand = 31;         // ballot holds n_cand+1 <= 32 positions

struct ArgMax {
  float v;
  int i;
};

__device__ __forceinline__ ArgMax better(ArgMax a, ArgMax b) {
  // larger value wins; equal values keep the lower index; NaN never wins
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

__device__ ArgMax block_argmax(const float* __restrict__ row, int V, ArgMax* red) {
  ArgMax best{-__int_as_float(0x7f800000), 0x7fffffff};
  const int tid = threadIdx.x;
  if ((V & 3) == 0 && ((reinterpret_cast<uintptr_t>(row) & 15) == 0)) {
    const float4* r4 = reinterpret_cast<const float4*>(row);
    for (int j = tid; j < V / 4; j += kThreads) {
      float4 x = __ldg(r4 + j);
      int base = 4 * j;
      if (x.x > best.v) best = {x.x, base};
      if (x.y > best.v) best = {x.y, base + 1};
      if (x.z > best.v) best = {x.z, base + 2};
      if (x.w > best.v) best = {x.w, base + 3};
    }
  } else {
    for (int j = tid; j < V; j += kThreads) {
      float x = __ldg(row + j);
      if (x > best.v) best = {x, j};
    }
  }
  // per-thread candidates are visited in increasing index order with a
  // strict '>' so each holds its lowest-index maximum; combine with ties→low
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax other{__shfl_xor_sync(0xffffffffu, best.v, o), __shfl_xor_sync(0xffffffffu, best.i, o)};
    best = better(best, other);
  }
  const int warp = tid >> 5, lane = tid & 31;
  __syncthreads();
  if (lane == 0) red[warp] = best;
  __syncthreads();
  ArgMax r = red[0];
  for (int w = 1; w < kThreads / 32; ++w) r = better(r, red[w]);
  if (r.i == 0x7fffffff) r.i = 0;  // all-NaN row
  return r;
}

__global__ void __launch_bounds__(kThreads) accept_greedy_kernel(
    const int32_t* __restrict__ draft, const float* __restrict__ logits,
    const int32_t* __restrict__ remaining, const int32_t* __restrict__ forced, int n_cand,
    int V, int32_t* __restrict__ out_tokens, int32_t* __restrict__ out_counts) {
  __shared__ ArgMax red[kThreads / 32];
  __shared__ int amax[kMaxCand + 1];
  const int s = blockIdx.x;
  const int npos = n_cand + 1;
  const float* base = logits + (size_t)s * npos * V;
  for (int i = 0; i < npos; ++i) {
    ArgMax a = block_argmax(base + (size_t)i * V, V, red);
    if (threadIdx.x == 0) amax[i] = a.i;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const bool match = lane < n_cand && draft[(size_t)s * n_cand + lane] == amax[lane];
    const unsigned ballot = __ballot_sync(0xffffffffu, match);
    int n_acc = __ffs(~ballot) - 1;  // trailing ones = accepted prefix
    if (n_acc < 0 || n_acc > n_cand) n_acc = n_cand;
    if (forced != nullptr) {
      int f = forced[s] - 1;
      n_acc = f < 0 ? 0 : (f > n_cand ? n_cand : f);
    }
    int rem = remaining[s];
    int count = n_acc + 1;
    if (count > rem) count = rem < 0 ? 0 : rem;
    if (lane < npos) {
      int tok = lane < n_acc ? draft[(size_t)s * n_cand + lane] : (lane == n_acc ? amax[n_acc] : -1);
      out_tokens[(size_t)s * npos + lane] = lane < count ? tok : -1;
    }
    if (lane == 0) out_counts[s] = count;
  }
}

// ---- deterministic softmax pieces (canonical order, see det_math.cuh) -------

__device__ float block_max(const float* __restrict__ row, int V, float* red) {
  float m = -__int_as_float(0x7f800000);
  for (int j = threadIdx.x; j < V; j += kThreads) m = fmaxf(m, row[j]);
  m = warp_max(m);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  float r = red[0];
  for (int w = 1; w < kThreads / 32; ++w) r = fmaxf(r, red[w]);
  __syncthreads();
  return r;
}

// Weight of element v in a row: kind 0 = exp(inv_t·(l−max)); kind 1 =
// residual max(w/Z − q, 0).
struct RowWeights {
  const float* logits;
  const float* q;  // residual only
  float mx, inv_t, Z;
  int kind;
  __device__ __forceinline__ float operator()(int v) const {
    float w = det_exp(d_mul(d_sub(logits[v], mx), inv_t));
    if (kind == 0) return w;
    float p = d_div(w, Z);
    return fmaxf(d_sub(p, q[v]), 0.0f);
  }
};

// Chunk sums in canonical order; returns the row total (left-to-right over
// chunks).  chunk_sums lives in shared memory.
__device__ float canonical_total(const RowWeights& W, int V, float* chunk_sums) {
  int lo, hi;
  det_chunk(V, threadIdx.x, lo, hi);
  float acc = 0.0f;
  for (int v = lo; v < hi; ++v) acc = d_add(acc, W(v));
  chunk_sums[threadIdx.x] = acc;
  __syncthreads();
  __shared__ float total;
  if (threadIdx.x == 0) {
    float t = 0.0f;
    for (int c = 0; c < kThreads; ++c) t = d_add(t, chunk_sums[c]);
    total = t;
  }
  __syncthreads();
  return total;
}

// Inverse-CDF pick with threshold `target` over the canonical prefix sums;
// thread 0 only.  Falls back to the last positive element when rounding
// leaves the threshold uncrossed.
__device__ int canonical_pick(const RowWeights& W, int V, const float* chunk_sums, float target) {
  float acc = 0.0f;
  int cstar = -1;
  float base = 0.0f;
  for (int c = 0; c < kThreads; ++c) {
    float nxt = d_add(acc, chunk_sums[c]);
    if (nxt > target) {
      cstar = c;
      base = acc;
      break;
    }
    acc = nxt;
  }
  int last_pos = -1;
  if (cstar >= 0) {
    int lo, hi;
    det_chunk(V, cstar, lo, hi);
    float a = base;
    for (int v = lo; v < hi; ++v) {
      float w = W(v);
      if (w > 0.0f) last_pos = v;
      a = d_add(a, w);
      if (a > target) return v;
    }
    if (last_pos >= 0) return last_pos;
  }
  for (int v = V - 1; v >= 0; --v)
    if (W(v) > 0.0f) return v;
  return 0;
}

__global__ void __launch_bounds__(kThreads) accept_sample_kernel(
    const int32_t* __restrict__ draft, const float* __restrict__ logits,
    const float* __restrict__ qprobs, const float* __restrict__ u_acc,
    const float* __restrict__ u_res, const int32_t* __restrict__ remaining, float inv_t,
    int n_cand, int V, int32_t* __restrict__ out_tokens, int32_t* __restrict__ out_counts) {
  __shared__ float red[kThreads / 32];
  __shared__ float chunk_sums[kThreads];
  __shared__ int s_result[2];  // [n_acc, final token]
  const int s = blockIdx.x;
  const int npos = n_cand + 1;
  const float* L = logits + (size_t)s * npos * V;
  const float* Q = qprobs + (size_t)s * n_cand * V;
  if (threadIdx.x == 0) s_result[0] = -1;
  __syncthreads();
  int n_acc = n_cand;
  int final_tok = 0;
  for (int i = 0; i <= n_cand; ++i) {
    const float* row = L + (size_t)i * V;
    float mx = block_max(row, V, red);
    RowWeights W{row, Q + (size_t)i * V, mx, inv_t, 0.0f, 0};
    float Z = canonical_total(W, V, chunk_sums);
    W.Z = Z;
    if (i == n_cand) {  // every draft token accepted: bonus from p_n
      if (threadIdx.x == 0) s_result[1] = canonical_pick(W, V, chunk_sums, d_mul(u_res[s], Z));
      __syncthreads();
      final_tok = s_result[1];
      n_acc = n_cand;
      break;
    }
    const int d = draft[(size_t)s * n_cand + i];
    // p(d) recomputed by every thread identically
    float p = d_div(W(d), Z);
    float q = Q[(size_t)i * V + d];
    bool accept = d_mul(u_acc[(size_t)s * n_cand + i], q) <= p;
    if (accept) continue;
    // first rejection at i: sample norm(max(p − q, 0))
    __syncthreads();
    RowWeights R = W;
    R.kind = 1;
    float Rt = canonical_total(R, V, chunk_sums);
    if (Rt > 0.0f) {
      if (threadIdx.x == 0) s_result[1] = canonical_pick(R, V, chunk_sums, d_mul(u_res[s], Rt));
    } else {
      __syncthreads();
      float Z2 = canonical_total(W, V, chunk_sums);
      if (threadIdx.x == 0) s_result[1] = canonical_pick(W, V, chunk_sums, d_mul(u_res[s], Z2));
    }
    __syncthreads();
    final_tok = s_result[1];
    n_acc = i;
    break;
  }
  if (threadIdx.x == 0) {
    int rem = remaining[s];
    int count = n_acc + 1;
    if (count > rem) count = rem < 0 ? 0 : rem;
    for (int j = 0; j < npos; ++j) {
      int tok = j < n_acc ? draft[(size_t)s * n_cand + j] : (j == n_acc ? final_tok : -1);
      out_tokens[(size_t)s * npos + j] = j < count ? tok : -1;
    }
    out_counts[s] = count;
  }
}

__global__ void __launch_bounds__(kThreads) sample_rows_kernel(
    const float* __restrict__ logits, int64_t row_stride, const float* __restrict__ uniforms,
    float inv_t, int V, int32_t* __restrict__ out_tokens, int64_t token_stride,
    float* __restrict__ out_probs, int64_t probs_stride) {
  __shared__ float red[kThreads / 32];
  __shared__ float chunk_sums[kThreads];
  __shared__ ArgMax ared[kThreads / 32];
  __shared__ int s_tok;
  const int r = blockIdx.x;
  const float* row = logits + (size_t)r * row_stride;
  if (uniforms == nullptr && out_probs == nullptr) {
    ArgMax a = block_argmax(row, V, ared);
    if (threadIdx.x == 0) out_tokens[(size_t)r * token_stride] = a.i;
    return;
  }
  float mx = block_max(row, V, red);
  RowWeights W{row, nullptr, mx, inv_t, 0.0f, 0};
  float Z = canonical_total(W, V, chunk_sums);
  W.Z = Z;
  if (out_probs != nullptr) {
    float* P = out_probs + (size_t)r * probs_stride;
    for (int v = threadIdx.x; v < V; v += kThreads) P[v] = d_div(W(v), Z);
  }
  if (uniforms == nullptr) {
    ArgMax a = block_argmax(row, V, ared);
    if (threadIdx.x == 0) out_tokens[(size_t)r * token_stride] = a.i;
    return;
  }
  if (threadIdx.x == 0) s_tok = canonical_pick(W, V, chunk_sums, d_mul(uniforms[r], Z));
  __syncthreads();
  if (threadIdx.x == 0) out_tokens[(size_t)r * token_stride] = s_tok;
}

}  // namespace

extern "C" int so_accept_greedy(const int32_t* draft_tokens, const float* target_logits,
                                const int32_t* remaining, const int32_t* forced_accept, int bs,
                                int n_cand, int vocab, int32_t* out_tokens, int32_t* out_counts,
                                void* stream) {
  SO_REQUIRE(draft_tokens && target_logits && remaining && out_tokens && out_counts, SO_E_NULLPTR);
  SO_REQUIRE(bs >= 0 && n_cand >= 1 && n_cand <= kMaxCand && vocab >= 1, SO_E_SHAPE);
  if (bs == 0) return SO_OK;
  accept_greedy_kernel<<<bs, kThreads, 0, as_stream(stream)>>>(
      draft_tokens, target_logits, remaining, forced_accept, n_cand, vocab, out_tokens, out_counts);
  SO_CHECK_LAUNCH();
  return SO_OK;
}

extern "C" int so_accept_sample(const int32_t* draft_tokens, const float* target_logits,
                                const float* draft_probs, const float* u_accept,
                                const float* u_resample, const int32_t* remaining,
                                float inv_temperature, int bs, int n_cand, int vocab,
                                int32_t* out_tokens, int32_t* out_counts, void* stream) {
  SO_REQUIRE(draft_tokens && target_logits && draft_probs && u_accept && u_resample && remaining &&
                 out_tokens && out_counts,
             SO_E_NULLPTR);
  SO_REQUIRE(bs >= 0 && n_cand >= 1 && n_cand <= kMaxCand && vocab >= 1, SO_E_SHAPE);
  SO_REQUIRE(inv_temperature > 0.0f, SO_E_SHAPE);
  if (bs == 0) return SO_OK;
  accept_sample_kernel<<<bs, kThreads, 0, as_stream(stream)>>>(
      draft_tokens, target_logits, draft_probs, u_accept, u_resample, remaining, inv_temperature,
      n_cand, vocab, out_tokens, out_counts);
  SO_CHECK_LAUNCH();
  return SO_OK;
}

extern "C" int so_sample_tokens(const float* logits, int64_t row_stride, const float* uniforms,
                                float inv_temperature, int rows, int vocab, int32_t* out_tokens,
                                int64_t token_stride, float* out_probs, int64_t probs_row_stride,
                                void* stream) {
  SO_REQUIRE(logits && out_tokens, SO_E_NULLPTR);
  SO_REQUIRE(rows >= 0 && vocab >= 1 && row_stride >= vocab, SO_E_SHAPE);
  SO_REQUIRE(inv_temperature > 0.0f, SO_E_SHAPE);
  if (rows == 0) return SO_OK;
  sample_rows_kernel<<<rows, kThreads, 0, as_stream(stream)>>>(
      logits, row_stride, uniforms, inv_temperature, vocab, out_tokens, token_stride, out_probs,
      probs_row_stride);
  SO_CHECK_LAUNCH();
  return SO_OK;
}
