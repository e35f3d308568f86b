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
  // a programmatically launched successor (K5c) may be scheduled now: it prefetches its weights and
  // waits (griddepcontrol.wait) for this grid to finish before reading the normalised rows.  Only
  // short kernels release early — a successor's CTAs spin on SMs the concurrent stream could use
  // (the persistent GEMM releasing early cost the verify stream 13 %: profiles/kernels_r2.md)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
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

// One warp per token (grid-stride).  Rotate-half RoPE (HF Mistral convention):
// for i < dh/2,
//   y[i]        = x[i]·cos(p·f_i) − x[i+dh/2]·sin(p·f_i)
//   y[i+dh/2]   = x[i+dh/2]·cos(p·f_i) + x[i]·sin(p·f_i),   f_i = θ^(−2i/dh)
// computed in fp32 and rounded once.  Lane l owns frequencies i = 2l, 2l+1:
// its two f_i come from powf once per warp, its two sincosf once per token,
// and every rotated head is one 4-B (bf16×2) load/store per lane per half —
// a contiguous 128-B run per warp.  K and V go to the paged caches laid out
// [page][kv_head][page_slot][dh]; V rows move as 16-B vectors.
constexpr int kRopeWarps = 4;

__global__ void __launch_bounds__(32 * kRopeWarps) rope_append_kernel(
    const __nv_bfloat16* __restrict__ qkv, const int32_t* __restrict__ pos, const int32_t* __restrict__ slots, int T,
    int hq, int hkv, int dh, float theta, int page_size, __nv_bfloat16* __restrict__ q_out,
    __nv_bfloat16* __restrict__ k_cache, __nv_bfloat16* __restrict__ v_cache) {
  const int lane = threadIdx.x & 31;
  const int half = dh / 2;
  const int width = (hq + 2 * hkv) * dh;
  const bool own = 2 * lane < half;  // dh ≤ 128: at most one frequency pair per lane
  const int i0 = 2 * lane;
  const float f0 = own ? 1.0f / powf(theta, (float)(2 * i0) / (float)dh) : 0.0f;
  const float f1 = own ? 1.0f / powf(theta, (float)(2 * (i0 + 1)) / (float)dh) : 0.0f;
  for (int t = blockIdx.x * kRopeWarps + (threadIdx.x >> 5); t < T; t += gridDim.x * kRopeWarps) {
    const __nv_bfloat16* row = qkv + (size_t)t * width;
    const float p = (float)pos[t];
    const int slot = slots[t];
    const int page = slot / page_size, off = slot % page_size;
    float s0 = 0.0f, c0 = 0.0f, s1 = 0.0f, c1 = 0.0f;
    if (own) {
      sincosf(p * f0, &s0, &c0);
      sincosf(p * f1, &s1, &c1);
    }
    if (own) {
      for (int h = 0; h < hq + hkv; ++h) {
        const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(row + h * dh + i0);
        const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(row + h * dh + half + i0);
        const float2 x0 = __bfloat1622float2(a), x1 = __bfloat1622float2(b);
        const __nv_bfloat162 y0 = __floats2bfloat162_rn(x0.x * c0 - x1.x * s0, x0.y * c1 - x1.y * s1);
        const __nv_bfloat162 y1 = __floats2bfloat162_rn(x1.x * c0 + x0.x * s0, x1.y * c1 + x0.y * s1);
        __nv_bfloat16* o = h < hq ? q_out + ((size_t)t * hq + h) * dh
                                  : k_cache + (((size_t)page * hkv + (h - hq)) * page_size + off) * dh;
        *reinterpret_cast<__nv_bfloat162*>(o + i0) = y0;
        *reinterpret_cast<__nv_bfloat162*>(o + half + i0) = y1;
      }
    }
    const int vec = dh / 8;  // 16-B vectors per V head row
    for (int idx = lane; idx < hkv * vec; idx += 32) {
      const int kh = idx / vec, c = idx % vec;
      *reinterpret_cast<int4*>(v_cache + (((size_t)page * hkv + kh) * page_size + off) * dh + c * 8) =
          *reinterpret_cast<const int4*>(row + (hq + hkv) * dh + kh * dh + c * 8);
    }
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
  SO_REQUIRE(T >= 0 && hq > 0 && hkv > 0 && hq % hkv == 0 && dh > 0 && dh % 8 == 0 && dh <= 128 && page_size > 0,
             SO_E_SHAPE);
  SO_REQUIRE(aligned16(qkv) && aligned16(q_out) && aligned16(k_cache) && aligned16(v_cache), SO_E_ALIGN);
  if (T == 0) return SO_OK;
  const int ctas = 16 * device_sm_count();  // 64 warps per SM, grid-stride over the tokens
  const int need = (T + kRopeWarps - 1) / kRopeWarps;
  rope_append_kernel<<<need < ctas ? need : ctas, 32 * kRopeWarps, 0, as_stream(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(qkv), positions, slot_mapping, T, hq, hkv, dh, rope_theta, page_size,
      reinterpret_cast<__nv_bfloat16*>(q_out), reinterpret_cast<__nv_bfloat16*>(k_cache),
      reinterpret_cast<__nv_bfloat16*>(v_cache));
  SO_CHECK_LAUNCH();
  return SO_OK;
}
