// K8 — auxiliary per-token kernels on the verify / draft forward:
// embedding gather, RMSNorm, RoPE + paged KV append.
//
// These are the non-GEMM pieces of the per-layer dataflow the reference models
// as a single `attn_cpu` + `ffn_gpu` pair (simulator.py:168-191); numerics follow
// the Mistral/Mixtral blocks (fp32 statistics, bf16 storage).
#include "common.cuh"

namespace {

__global__ void embed_kernel(const int32_t* __restrict__ tok, const __nv_bfloat16* __restrict__ table, int T, int H,
                             __nv_bfloat16* __restrict__ out) {
  const int vec = H / 8;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < (size_t)T * vec;
       i += (size_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / vec), c = (int)(i % vec);
    const int id = tok[t];
    reinterpret_cast<int4*>(out + (size_t)t * H)[c] = __ldg(reinterpret_cast<const int4*>(table + (size_t)id * H) + c);
  }
}

// One CTA per row; the row is read once into registers (≤ 8 int4 per thread
// at H = 8192 with 128 threads), sum of squares in fp32, then
// out = bf16( bf16(x · rsqrt(mean(x²)+eps)) · w ).
constexpr int kNormThreads = 128;
constexpr int kNormMaxVec = 8;

__global__ void __launch_bounds__(kNormThreads) rmsnorm_kernel(const __nv_bfloat16* __restrict__ x,
                                                               const __nv_bfloat16* __restrict__ w, int H,
                                                               float eps, __nv_bfloat16* __restrict__ out) {
  __shared__ float red[kNormThreads / 32];
  const int t = blockIdx.x;
  const int vec = H / 8;
  const int4* xr = reinterpret_cast<const int4*>(x + (size_t)t * H);
  int4 buf[kNormMaxVec];
  float ss = 0.0f;
#pragma unroll
  for (int k = 0; k < kNormMaxVec; ++k) {
    const int c = threadIdx.x + k * kNormThreads;
    if (c < vec) {
      buf[k] = __ldg(xr + c);
      float f[8];
      unpack8(buf[k], f);
#pragma unroll
      for (int j = 0; j < 8; ++j) ss = fmaf(f[j], f[j], ss);
    }
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.0f;
#pragma unroll
  for (int i = 0; i < kNormThreads / 32; ++i) tot += red[i];
  const float r = rsqrtf(tot / (float)H + eps);
  int4* orow = reinterpret_cast<int4*>(out + (size_t)t * H);
  const int4* wr = reinterpret_cast<const int4*>(w);
#pragma unroll
  for (int k = 0; k < kNormMaxVec; ++k) {
    const int c = threadIdx.x + k * kNormThreads;
    if (c < vec) {
      float f[8], g[8];
      unpack8(buf[k], f);
      unpack8(__ldg(wr + c), g);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] = __bfloat162float(__float2bfloat16_rn(f[j] * r)) * g[j];
      orow[c] = pack8(f);
    }
  }
}

// One CTA per token.  Rotate-half RoPE (HF Mistral convention): for i < dh/2,
//   y[i]        = x[i]·cos(p·f_i) − x[i+dh/2]·sin(p·f_i)
//   y[i+dh/2]   = x[i+dh/2]·cos(p·f_i) + x[i]·sin(p·f_i),   f_i = θ^(−2i/dh)
// computed in fp32 and rounded once.  K and V go to the paged caches laid out
// [page][kv_head][page_slot][dh].
__global__ void rope_append_kernel(const __nv_bfloat16* __restrict__ qkv, const int32_t* __restrict__ pos,
                                   const int32_t* __restrict__ slots, int hq, int hkv, int dh, float theta,
                                   int page_size, __nv_bfloat16* __restrict__ q_out,
                                   __nv_bfloat16* __restrict__ k_cache, __nv_bfloat16* __restrict__ v_cache) {
  const int t = blockIdx.x;
  const int half = dh / 2;
  const int width = (hq + 2 * hkv) * dh;
  const __nv_bfloat16* row = qkv + (size_t)t * width;
  const float p = (float)pos[t];
  const int slot = slots[t];
  const int page = slot / page_size, off = slot % page_size;
  // rotated heads: hq query heads then hkv key heads
  for (int idx = threadIdx.x; idx < (hq + hkv) * half; idx += blockDim.x) {
    const int h = idx / half, i = idx % half;
    const float inv_freq = 1.0f / powf(theta, (float)(2 * i) / (float)dh);
    float sn, cs;
    sincosf(p * inv_freq, &sn, &cs);
    const float x0 = __bfloat162float(row[h * dh + i]);
    const float x1 = __bfloat162float(row[h * dh + i + half]);
    const __nv_bfloat16 y0 = __float2bfloat16_rn(x0 * cs - x1 * sn);
    const __nv_bfloat16 y1 = __float2bfloat16_rn(x1 * cs + x0 * sn);
    if (h < hq) {
      __nv_bfloat16* qo = q_out + ((size_t)t * hq + h) * dh;
      qo[i] = y0;
      qo[i + half] = y1;
    } else {
      const int kh = h - hq;
      __nv_bfloat16* ko = k_cache + (((size_t)page * hkv + kh) * page_size + off) * dh;
      ko[i] = y0;
      ko[i + half] = y1;
    }
  }
  for (int idx = threadIdx.x; idx < hkv * dh; idx += blockDim.x) {
    const int kh = idx / dh, d = idx % dh;
    v_cache[(((size_t)page * hkv + kh) * page_size + off) * dh + d] = row[(hq + hkv) * dh + idx];
  }
}

__global__ void build_verify_tokens_kernel(const int32_t* __restrict__ t_last, const int32_t* __restrict__ drafts,
                                           int ld, int bs, int n, int32_t* __restrict__ tokens,
                                           int32_t* __restrict__ rows) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= bs * (n + 1)) return;
  const int s = i / (n + 1), j = i % (n + 1);
  if (j == 0) {
    tokens[i] = t_last[s];
  } else {
    const int d = drafts[(size_t)(j - 1) * ld + s];
    tokens[i] = d;
    rows[(size_t)s * n + j - 1] = d;
  }
}

__global__ void gather_i32_kernel(const int32_t* __restrict__ src, const int64_t* __restrict__ idx, int n,
                                  int32_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = src[idx[i]];
}

__global__ void scatter_i32_kernel(int32_t* __restrict__ dst, const int64_t* __restrict__ idx,
                                   const int32_t* __restrict__ val, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[idx[i]] = val[i];
}

int grid_for(size_t work, int threads) {
  size_t g = (work + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

extern "C" int so_embed(const int32_t* tokens, const void* table, int T, int H, void* out, void* stream) {
  SO_REQUIRE(tokens && table && out, SO_E_NULLPTR);
  SO_REQUIRE(T >= 0 && H > 0 && H % 8 == 0, SO_E_SHAPE);
  SO_REQUIRE(aligned16(table) && aligned16(out), SO_E_ALIGN);
  if (T == 0) return SO_OK;
  embed_kernel<<<grid_for((size_t)T * (H / 8), 256), 256, 0, as_stream(stream)>>>(
      tokens, reinterpret_cast<const __nv_bfloat16*>(table), T, H, reinterpret_cast<__nv_bfloat16*>(out));
  SO_CHECK_LAUNCH();
  return SO_OK;
}

extern "C" int so_build_verify_tokens(const int32_t* t_last, const int32_t* drafts, int ld, int bs, int n_cand,
                                      int32_t* tokens, int32_t* draft_rows, void* stream) {
  SO_REQUIRE(t_last && drafts && tokens && draft_rows, SO_E_NULLPTR);
  SO_REQUIRE(bs >= 0 && n_cand >= 1 && ld >= bs, SO_E_SHAPE);
  if (bs == 0) return SO_OK;
  const int total = bs * (n_cand + 1);
  build_verify_tokens_kernel<<<(total + 255) / 256, 256, 0, as_stream(stream)>>>(t_last, drafts, ld, bs, n_cand,
                                                                                  tokens, draft_rows);
  SO_CHECK_LAUNCH();
  return SO_OK;
}

extern "C" int so_gather_i32(const int32_t* src, const int64_t* idx, int n, int32_t* out, void* stream) {
  SO_REQUIRE(src && idx && out, SO_E_NULLPTR);
  if (n <= 0) return SO_OK;
  gather_i32_kernel<<<grid_for((size_t)n, 256), 256, 0, as_stream(stream)>>>(src, idx, n, out);
  SO_CHECK_LAUNCH();
  return SO_OK;
}

extern "C" int so_scatter_i32(int32_t* dst, const int64_t* idx, const int32_t* val, int n, void* stream) {
  SO_REQUIRE(dst && idx && val, SO_E_NULLPTR);
  if (n <= 0) return SO_OK;
  scatter_i32_kernel<<<grid_for((size_t)n, 256), 256, 0, as_stream(stream)>>>(dst, idx, val, n);
  SO_CHECK_LAUNCH();
  return SO_OK;
}

extern "C" int so_rmsnorm(const void* x, const void* w, int T, int H, float eps, void* out, void* stream) {
  SO_REQUIRE(x && w && out, SO_E_NULLPTR);
  SO_REQUIRE(T >= 0 && H > 0 && H % 8 == 0 && H <= 8 * kNormThreads * kNormMaxVec, SO_E_SHAPE);
  SO_REQUIRE(aligned16(x) && aligned16(w) && aligned16(out), SO_E_ALIGN);
  if (T == 0) return SO_OK;
  rmsnorm_kernel<<<T, kNormThreads, 0, as_stream(stream)>>>(reinterpret_cast<const __nv_bfloat16*>(x),
                                                            reinterpret_cast<const __nv_bfloat16*>(w), H, eps,
                                                            reinterpret_cast<__nv_bfloat16*>(out));
  SO_CHECK_LAUNCH();
  return SO_OK;
}

extern "C" int so_rope_kv_append(const void* qkv, const int32_t* positions, const int32_t* slot_mapping, int T,
                                 int hq, int hkv, int dh, float rope_theta, int page_size, void* q_out,
                                 void* k_cache, void* v_cache, void* stream) {
  SO_REQUIRE(qkv && positions && slot_mapping && q_out && k_cache && v_cache, SO_E_NULLPTR);
  SO_REQUIRE(T >= 0 && hq > 0 && hkv > 0 && hq % hkv == 0 && dh > 0 && dh % 2 == 0 && page_size > 0, SO_E_SHAPE);
  if (T == 0) return SO_OK;
  rope_append_kernel<<<T, 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(qkv), positions, slot_mapping, hq, hkv, dh, rope_theta, page_size,
      reinterpret_cast<__nv_bfloat16*>(q_out), reinterpret_cast<__nv_bfloat16*>(k_cache),
      reinterpret_cast<__nv_bfloat16*>(v_cache));
  SO_CHECK_LAUNCH();
  return SO_OK;
}
