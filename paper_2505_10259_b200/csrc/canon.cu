// Canonical-order arithmetic: the parity mode of the model ops.
//
// The tcgen05 / mma.sync kernels accumulate in an order the tensor pipe
// chooses, so their logits match a CPU restatement only to a tolerance and a
// greedy token can flip on a near-tie.  North star: "bit-exact
// accepted tokens versus the reference on the tiny config".  These kernels
// compute the SAME ops at the SAME bf16 rounding points as the product
// kernels (so_gemm_bf16 epilogues, so_rmsnorm, so_rope_kv_append,
// so_attn_paged, so_router_top2), but every float op is one correctly rounded
// IEEE op in a fixed, documented order:
//   * dot products: acc = 0; for k = 0..K-1: acc = fma(a_k, b_k, acc);
//   * exp: det_exp (det_math.cuh), SiLU g / (1 + det_exp(-g));
//   * rsqrt: 1 / sqrt(mean + eps) with IEEE sqrt and division;
//   * RoPE: cos/sin from a caller table (host-computed, fp32), two products and
//     one add/sub per output;
//   * attention: two passes per (query row, head) — max of the scaled scores,
//     then Z = Σ det_exp(s − max) and o = Σ p·v left to right, out = o / Z.
// oracle/csrc/canon_oracle.c restates the same definitions for the CPU; the
// tiny-config tests assert token (and logit) equality, not a tolerance.
// One thread per output element: these run at tiny shapes only.
#include "common.cuh"
#include "det_math.cuh"

namespace {

__device__ __forceinline__ float bfr(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }

__device__ __forceinline__ float canon_silu(float g) { return d_div(g, d_add(1.0f, det_exp(-g))); }

__device__ __forceinline__ float canon_dot(const __nv_bfloat16* __restrict__ a, const __nv_bfloat16* __restrict__ b,
                                           int K) {
  float acc = 0.0f;
  for (int k = 0; k < K; ++k) acc = d_fma(bf2f(a[k]), bf2f(b[k]), acc);
  return acc;
}

// Row r of A uses expert e's weights when offs != nullptr (offs[e] ≤ r < offs[e+1]).
__device__ __forceinline__ int canon_expert(const int32_t* __restrict__ offs, int E, int r) {
  int e = 0;
  while (e < E && r >= offs[e + 1]) ++e;
  return e;
}

__global__ void canon_gemm_kernel(const __nv_bfloat16* __restrict__ A, const __nv_bfloat16* __restrict__ B,
                                  const int32_t* __restrict__ offs, int E, int M, int N, int K, void* __restrict__ C,
                                  int ldc, int epi, const void* __restrict__ aux) {
  const int out_cols = epi == SO_EPI_SWIGLU ? N / 2 : N;
  const long long total = (long long)M * out_cols;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / out_cols), c = (int)(i % out_cols);
    const __nv_bfloat16* Bw = B;
    if (offs != nullptr) {
      if (r >= offs[E]) continue;
      Bw = B + (size_t)canon_expert(offs, E, r) * N * K;
    }
    const __nv_bfloat16* a = A + (size_t)r * K;
    if (epi == SO_EPI_SWIGLU) {
      // gate/up rows interleaved in 64-row blocks (the window layout, weights.py)
      const int p = c / 64, j = c % 64;
      const float g = canon_dot(a, Bw + (size_t)(p * 128 + j) * K, K);
      const float u = canon_dot(a, Bw + (size_t)(p * 128 + 64 + j) * K, K);
      reinterpret_cast<__nv_bfloat16*>(C)[(size_t)r * ldc + c] = __float2bfloat16_rn(d_mul(canon_silu(g), u));
      continue;
    }
    const float acc = canon_dot(a, Bw + (size_t)c * K, K);
    if (epi == SO_EPI_F32) {
      reinterpret_cast<float*>(C)[(size_t)r * ldc + c] = acc;
    } else {
      float v = acc;
      if (epi == SO_EPI_BF16_RESID) {
        v = d_add(bfr(acc), bf2f(reinterpret_cast<const __nv_bfloat16*>(aux)[(size_t)r * ldc + c]));
      } else if (epi == SO_EPI_BF16_ROWSCALE) {
        v = d_mul(acc, reinterpret_cast<const float*>(aux)[r]);
      }
      reinterpret_cast<__nv_bfloat16*>(C)[(size_t)r * ldc + c] = __float2bfloat16_rn(v);
    }
  }
}

__global__ void canon_rmsnorm_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w, int T,
                                     int H, float eps, __nv_bfloat16* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const __nv_bfloat16* xr = x + (size_t)t * H;
  float ss = 0.0f;
  for (int i = 0; i < H; ++i) {
    const float v = bf2f(xr[i]);
    ss = d_fma(v, v, ss);
  }
  const float r = d_div(1.0f, __fsqrt_rn(d_add(d_div(ss, (float)H), eps)));
  for (int i = 0; i < H; ++i)
    out[(size_t)t * H + i] = __float2bfloat16_rn(d_mul(bfr(d_mul(bf2f(xr[i]), r)), bf2f(w[i])));
}

// One thread per (token, head, frequency pair i < dh/2) for q and k heads, and
// per (token, kv head, element) for the V copy.
__global__ void canon_rope_kernel(const __nv_bfloat16* __restrict__ qkv, const int32_t* __restrict__ pos,
                                  const int32_t* __restrict__ slots, int T, int hq, int hkv, int dh,
                                  const float* __restrict__ table, int table_rows, int page_size,
                                  __nv_bfloat16* __restrict__ q_out, __nv_bfloat16* __restrict__ k_cache,
                                  __nv_bfloat16* __restrict__ v_cache) {
  const int half = dh / 2;
  const int width = (hq + 2 * hkv) * dh;
  const int per_tok = (hq + hkv) * half + hkv * dh;
  const long long total = (long long)T * per_tok;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(idx / per_tok), o = (int)(idx % per_tok);
    const int p = pos[t];
    if (p < 0 || p >= table_rows) __trap();  // the caller's table must cover every position
    const int slot = slots[t];
    const int page = slot / page_size, off = slot % page_size;
    const __nv_bfloat16* row = qkv + (size_t)t * width;
    if (o < (hq + hkv) * half) {
      const int h = o / half, i = o % half;
      const float c = table[(size_t)p * dh + i], s = table[(size_t)p * dh + half + i];
      const float x0 = bf2f(row[h * dh + i]), x1 = bf2f(row[h * dh + half + i]);
      const float y0 = d_sub(d_mul(x0, c), d_mul(x1, s));
      const float y1 = d_add(d_mul(x1, c), d_mul(x0, s));
      __nv_bfloat16* dst = h < hq ? q_out + ((size_t)t * hq + h) * dh
                                  : k_cache + (((size_t)page * hkv + (h - hq)) * page_size + off) * dh;
      dst[i] = __float2bfloat16_rn(y0);
      dst[half + i] = __float2bfloat16_rn(y1);
    } else {
      const int v = o - (hq + hkv) * half;
      const int kh = v / dh, d = v % dh;
      v_cache[(((size_t)page * hkv + kh) * page_size + off) * dh + d] = row[(hq + hkv) * dh + kh * dh + d];
    }
  }
}

constexpr int kCanonMaxDh = 128;

__device__ __forceinline__ float canon_score(const __nv_bfloat16* __restrict__ q,
                                             const __nv_bfloat16* __restrict__ k, int dh, float scale) {
  return d_mul(canon_dot(q, k, dh), scale);
}

__global__ void canon_attn_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k_cache,
                                  const __nv_bfloat16* __restrict__ v_cache, const int32_t* __restrict__ block_table,
                                  int max_pages, const int32_t* __restrict__ q_start,
                                  const int32_t* __restrict__ kv_before, int bs, int max_q, int hq, int hkv, int dh,
                                  int page_size, float scale, __nv_bfloat16* __restrict__ out) {
  const long long total = (long long)bs * max_q * hq;
  const int G = hq / hkv;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(idx / ((long long)max_q * hq));
    const int j = (int)((idx / hq) % max_q);
    const int h = (int)(idx % hq);
    const int q0 = q_start[s], q1 = q_start[s + 1];
    if (j >= q1 - q0) continue;
    const int row = q0 + j;
    const int n_keys = kv_before[s] + j + 1;
    const int g = h / G;
    const __nv_bfloat16* qr = q + ((size_t)row * hq + h) * dh;
    const int32_t* bt = block_table + (size_t)s * max_pages;
    float m = -__int_as_float(0x7f800000);
    for (int t = 0; t < n_keys; ++t) {
      const int page = bt[t / page_size], off = t % page_size;
      const float sc = canon_score(qr, k_cache + (((size_t)page * hkv + g) * page_size + off) * dh, dh, scale);
      m = fmaxf(m, sc);
    }
    float o[kCanonMaxDh];
    for (int d = 0; d < dh; ++d) o[d] = 0.0f;
    float Z = 0.0f;
    for (int t = 0; t < n_keys; ++t) {
      const int page = bt[t / page_size], off = t % page_size;
      const size_t base = (((size_t)page * hkv + g) * page_size + off) * dh;
      const float p = det_exp(d_sub(canon_score(qr, k_cache + base, dh, scale), m));
      Z = d_add(Z, p);
      for (int d = 0; d < dh; ++d) o[d] = d_fma(p, bf2f(v_cache[base + d]), o[d]);
    }
    __nv_bfloat16* orow = out + ((size_t)row * hq + h) * dh;
    for (int d = 0; d < dh; ++d) orow[d] = __float2bfloat16_rn(d_div(o[d], Z));
  }
}

// Router: one thread per token — E sequential dot products, top-2 with strict
// comparisons in expert order (ties → lower index), pair weights
// w1 = 1 / (1 + det_exp(l0 − l1)), w0 = 1 − w1.
__global__ void canon_route_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg, int T,
                                   int H, int E, int32_t* __restrict__ idx, float* __restrict__ w) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  float l0 = -__int_as_float(0x7f800000), l1 = l0;
  int i0 = 0, i1 = 1;
  for (int e = 0; e < E; ++e) {
    const float v = canon_dot(x + (size_t)t * H, wg + (size_t)e * H, H);
    if (v > l0) {
      l1 = l0; i1 = i0;
      l0 = v; i0 = e;
    } else if (v > l1) {
      l1 = v; i1 = e;
    }
  }
  const float w1 = d_div(1.0f, d_add(1.0f, det_exp(d_sub(l0, l1))));
  idx[2 * t] = i0;
  idx[2 * t + 1] = i1;
  w[2 * t] = d_sub(1.0f, w1);
  w[2 * t + 1] = w1;
}

// Stable expert-major permutation (row order = token order inside an expert),
// the same layout so_router_top2 produces.  One thread: tiny T only.
__global__ void canon_permute_kernel(const int32_t* __restrict__ idx, const float* __restrict__ w, int T, int E,
                                     int32_t* __restrict__ fill, int32_t* __restrict__ offs,
                                     int32_t* __restrict__ perm_token, float* __restrict__ row_weight,
                                     int32_t* __restrict__ token_rows) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (int e = 0; e < E; ++e) fill[e] = 0;
  for (int p = 0; p < 2 * T; ++p) ++fill[idx[p]];
  int a = 0;
  for (int e = 0; e < E; ++e) {
    offs[e] = a;
    a += fill[e];
    fill[e] = 0;
  }
  offs[E] = a;
  for (int p = 0; p < 2 * T; ++p) {
    const int e = idx[p];
    const int row = offs[e] + fill[e]++;
    perm_token[row] = p >> 1;
    row_weight[row] = w[p];
    token_rows[p] = row;
  }
}

__global__ void canon_gather_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ perm_token,
                                    int rows, int H, __nv_bfloat16* __restrict__ x_perm) {
  const long long total = (long long)rows * H;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / H), c = (int)(i % H);
    x_perm[i] = x[(size_t)perm_token[r] * H + c];
  }
}

int canon_grid(long long work) {
  long long g = (work + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  return g < 1 ? 1 : (int)g;
}

}  // namespace

extern "C" int so_canon_gemm(const void* A, const void* B, const int32_t* expert_offsets, int E, int M, int N, int K,
                             void* C, int ldc, int epilogue, const void* aux, void* stream) {
  SO_REQUIRE(A && B && C, SO_E_NULLPTR);
  SO_REQUIRE(M >= 0 && N > 0 && K > 0 && (expert_offsets == nullptr || E >= 1), SO_E_SHAPE);
  SO_REQUIRE(epilogue >= SO_EPI_BF16 && epilogue <= SO_EPI_BF16_ROWSCALE, SO_E_UNSUPPORTED);
  if (epilogue == SO_EPI_SWIGLU) SO_REQUIRE(N % 128 == 0 && ldc >= N / 2, SO_E_SHAPE);
  else SO_REQUIRE(ldc >= N, SO_E_SHAPE);
  if (epilogue == SO_EPI_BF16_RESID || epilogue == SO_EPI_BF16_ROWSCALE) SO_REQUIRE(aux != nullptr, SO_E_NULLPTR);
  if (M == 0) return SO_OK;
  const long long outs = (long long)M * (epilogue == SO_EPI_SWIGLU ? N / 2 : N);
  canon_gemm_kernel<<<canon_grid(outs), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(A), reinterpret_cast<const __nv_bfloat16*>(B), expert_offsets, E, M, N,
      K, C, ldc, epilogue, aux);
  SO_CHECK_LAUNCH();
  return SO_OK;
}

extern "C" int so_canon_rmsnorm(const void* x, const void* w, int T, int H, float eps, void* out, void* stream) {
  SO_REQUIRE(x && w && out, SO_E_NULLPTR);
  SO_REQUIRE(T >= 0 && H > 0, SO_E_SHAPE);
  if (T == 0) return SO_OK;
  canon_rmsnorm_kernel<<<(T + 127) / 128, 128, 0, as_stream(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(x), reinterpret_cast<const __nv_bfloat16*>(w), T, H, eps,
      reinterpret_cast<__nv_bfloat16*>(out));
  SO_CHECK_LAUNCH();
  return SO_OK;
}

extern "C" int so_canon_rope_kv_append(const void* qkv, const int32_t* positions, const int32_t* slot_mapping, int T,
                                       int hq, int hkv, int dh, const float* rope_table, int table_rows,
                                       int page_size, void* q_out, void* k_cache, void* v_cache, void* stream) {
  SO_REQUIRE(qkv && positions && slot_mapping && rope_table && q_out && k_cache && v_cache, SO_E_NULLPTR);
  SO_REQUIRE(T >= 0 && hq > 0 && hkv > 0 && hq % hkv == 0 && dh > 0 && dh % 2 == 0 && page_size > 0 &&
                 table_rows > 0, SO_E_SHAPE);
  if (T == 0) return SO_OK;
  const long long work = (long long)T * ((hq + hkv) * (dh / 2) + hkv * dh);
  canon_rope_kernel<<<canon_grid(work), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(qkv), positions, slot_mapping, T, hq, hkv, dh, rope_table, table_rows,
      page_size, reinterpret_cast<__nv_bfloat16*>(q_out), reinterpret_cast<__nv_bfloat16*>(k_cache),
      reinterpret_cast<__nv_bfloat16*>(v_cache));
  SO_CHECK_LAUNCH();
  return SO_OK;
}

extern "C" int so_canon_attn_paged(const void* q, const void* k_cache, const void* v_cache,
                                   const int32_t* block_table, int max_pages, const int32_t* q_start,
                                   const int32_t* kv_before, int bs, int max_q, int hq, int hkv, int dh,
                                   int page_size, float scale, void* out, void* stream) {
  SO_REQUIRE(q && k_cache && v_cache && block_table && q_start && kv_before && out, SO_E_NULLPTR);
  SO_REQUIRE(bs >= 0 && max_q >= 1 && hq > 0 && hkv > 0 && hq % hkv == 0 && max_pages > 0 && page_size >= 1 &&
                 dh > 0 && dh <= kCanonMaxDh, SO_E_SHAPE);
  if (bs == 0) return SO_OK;
  canon_attn_kernel<<<canon_grid((long long)bs * max_q * hq), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(k_cache),
      reinterpret_cast<const __nv_bfloat16*>(v_cache), block_table, max_pages, q_start, kv_before, bs, max_q, hq, hkv,
      dh, page_size, scale, reinterpret_cast<__nv_bfloat16*>(out));
  SO_CHECK_LAUNCH();
  return SO_OK;
}

extern "C" int so_canon_router_top2(const void* x, const void* w_gate, int T, int H, int E, int32_t* topk_idx,
                                    float* topk_w, int32_t* expert_offsets, int32_t* perm_token, float* row_weight,
                                    int32_t* token_rows, void* x_perm, void* workspace, void* stream) {
  SO_REQUIRE(x && w_gate && expert_offsets && perm_token && row_weight && token_rows && x_perm && workspace,
             SO_E_NULLPTR);
  SO_REQUIRE(T >= 0 && H > 0 && E >= 2 && E <= 64, SO_E_SHAPE);
  cudaStream_t st = as_stream(stream);
  // workspace layout of so_router_workspace_bytes: [per-expert counters | topk idx | topk w]
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  int32_t* fill = reinterpret_cast<int32_t*>(ws);
  int32_t* idx = topk_idx ? topk_idx : reinterpret_cast<int32_t*>(ws + 256);
  float* w = topk_w ? topk_w : reinterpret_cast<float*>(ws + 256 + (size_t)T * 2 * sizeof(int32_t));
  if (T > 0) {
    canon_route_kernel<<<(T + 127) / 128, 128, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(x),
                                                        reinterpret_cast<const __nv_bfloat16*>(w_gate), T, H, E,
                                                        idx, w);
    SO_CHECK_LAUNCH();
  }
  canon_permute_kernel<<<1, 1, 0, st>>>(idx, w, T, E, fill, expert_offsets, perm_token, row_weight, token_rows);
  SO_CHECK_LAUNCH();
  if (T > 0) {
    canon_gather_kernel<<<canon_grid((long long)2 * T * H), 256, 0, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(x), perm_token, 2 * T, H, reinterpret_cast<__nv_bfloat16*>(x_perm));
    SO_CHECK_LAUNCH();
  }
  return SO_OK;
}
