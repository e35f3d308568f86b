// K2 — fused Mixtral top-2 router + stable expert-major token permutation, and
// the deterministic two-slot combine that closes the MoE block.
//
// The reference charges the whole MoE block as one `ffn_gpu` event per layer
// (simulator.py:185-191); its routing semantics are the third-party Mixtral
// block (transformers modeling_mixtral.py: fp32 softmax → top-2 → renormalise),
// cited in SURVEY.md §8c.  Three launches, no host synchronisation:
//   1. route:   one warp per token — E dot products (fp32), top-2 (ties → lower
//               expert index), pair-renormalised weights, per-expert histogram;
//   2. scan:    one CTA — exclusive scan of the histogram into expert offsets,
//               then a stable rank of every (token, slot) inside its expert using
//               __match_any_sync + popc (order = token index, so the permutation
//               is deterministic);
//   3. gather:  x_perm[row] = x[perm_token[row]] with 16-B vector copies.
#include "common.cuh"

namespace {

constexpr int kMaxE = 16;  // Mixtral uses 8; accumulators stay in registers

__global__ void route_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg, int T,
                             int H, int E, int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
                             int32_t* __restrict__ counts) {
  const int warps = blockDim.x >> 5;
  const int t = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  float acc[kMaxE];
#pragma unroll
  for (int e = 0; e < kMaxE; ++e) acc[e] = 0.0f;
  const int4* xr = reinterpret_cast<const int4*>(x + (size_t)t * H);
  for (int c = lane; c < H / 8; c += 32) {
    float xf[8];
    unpack8(__ldg(xr + c), xf);
#pragma unroll
    for (int e = 0; e < kMaxE; ++e) {
      if (e >= E) break;
      float wf[8];
      unpack8(__ldg(reinterpret_cast<const int4*>(wg + (size_t)e * H) + c), wf);
      float s = 0.0f;
#pragma unroll
      for (int j = 0; j < 8; ++j) s = fmaf(xf[j], wf[j], s);
      acc[e] += s;
    }
  }
  float l0 = -3.4e38f, l1 = -3.4e38f;
  int i0 = 0, i1 = 1;
#pragma unroll
  for (int e = 0; e < kMaxE; ++e) {
    if (e >= E) break;
    float v = warp_sum(acc[e]);
    if (v > l0) {
      l1 = l0; i1 = i0;
      l0 = v; i0 = e;
    } else if (v > l1) {
      l1 = v; i1 = e;
    }
  }
  if (lane == 0) {
    // softmax over all E then renormalising the top pair == softmax over the pair
    const float w1 = 1.0f / (1.0f + expf(l0 - l1));
    const float w0 = 1.0f - w1;
    topk_idx[2 * t] = i0;
    topk_idx[2 * t + 1] = i1;
    topk_w[2 * t] = w0;
    topk_w[2 * t + 1] = w1;
    atomicAdd(&counts[i0], 1);
    atomicAdd(&counts[i1], 1);
  }
}

constexpr int kScanThreads = 1024;

__global__ void __launch_bounds__(kScanThreads) scan_kernel(const int32_t* __restrict__ topk_idx,
                                                            const float* __restrict__ topk_w,
                                                            const int32_t* __restrict__ counts, int T, int E,
                                                            int32_t* __restrict__ offs, int32_t* __restrict__ perm_token,
                                                            float* __restrict__ row_weight,
                                                            int32_t* __restrict__ token_rows) {
  __shared__ int s_offs[kMaxE + 1];
  __shared__ int s_base[kMaxE];
  __shared__ int s_warp_cnt[kScanThreads / 32][kMaxE];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    int a = 0;
    for (int e = 0; e < E; ++e) {
      s_offs[e] = a;
      s_base[e] = 0;
      a += counts[e];
    }
    s_offs[E] = a;
  }
  __syncthreads();
  if (tid <= E) offs[tid] = s_offs[tid];
  const int pairs = 2 * T;
  for (int tile = 0; tile < pairs; tile += kScanThreads) {
    const int p = tile + tid;
    const bool live = p < pairs;
    const int e = live ? topk_idx[p] : -1;
    for (int i = tid; i < (kScanThreads / 32) * kMaxE; i += kScanThreads) (&s_warp_cnt[0][0])[i] = 0;
    __syncthreads();
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int rank_in_warp = __popc(peers & ((1u << lane) - 1u));
    if (live && rank_in_warp == 0) s_warp_cnt[warp][e] = __popc(peers);
    __syncthreads();
    if (live) {
      int before = 0;
      for (int w = 0; w < warp; ++w) before += s_warp_cnt[w][e];
      const int row = s_offs[e] + s_base[e] + before + rank_in_warp;
      const int t = p >> 1;
      perm_token[row] = t;
      row_weight[row] = topk_w[p];
      token_rows[p] = row;
    }
    __syncthreads();
    if (tid < E) {
      int tot = 0;
      for (int w = 0; w < kScanThreads / 32; ++w) tot += s_warp_cnt[w][tid];
      s_base[tid] += tot;
    }
    __syncthreads();
  }
}

__global__ void gather_rows_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ perm_token,
                                   int rows, int H, __nv_bfloat16* __restrict__ x_perm) {
  const int vec = H / 8;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < (size_t)rows * vec;
       i += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / vec), c = (int)(i % vec);
    const int t = perm_token[r];
    reinterpret_cast<int4*>(x_perm + (size_t)r * H)[c] = __ldg(reinterpret_cast<const int4*>(x + (size_t)t * H) + c);
  }
}

__global__ void combine_kernel(const __nv_bfloat16* __restrict__ y, const int32_t* __restrict__ token_rows,
                               const __nv_bfloat16* __restrict__ resid, int T, int H,
                               __nv_bfloat16* __restrict__ out) {
  const int vec = H / 8;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < (size_t)T * vec;
       i += (size_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / vec), c = (int)(i % vec);
    const int r0 = token_rows[2 * t], r1 = token_rows[2 * t + 1];
    float a[8], b[8], r[8];
    unpack8(__ldg(reinterpret_cast<const int4*>(y + (size_t)r0 * H) + c), a);
    unpack8(__ldg(reinterpret_cast<const int4*>(y + (size_t)r1 * H) + c), b);
    unpack8(__ldg(reinterpret_cast<const int4*>(resid + (size_t)t * H) + c), r);
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      // moe = bf16(y0 + y1); out = bf16(resid + moe)
      const float moe = __bfloat162float(__float2bfloat16_rn(a[j] + b[j]));
      o[j] = r[j] + moe;
    }
    reinterpret_cast<int4*>(out + (size_t)t * H)[c] = pack8(o);
  }
}

int grid_for(size_t work, int threads) {
  size_t g = (work + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

extern "C" size_t so_router_workspace_bytes(int T, int E) {
  // counts[E] + topk scratch when the caller passes NULL for topk outputs
  return 256 + (size_t)T * 2 * (sizeof(int32_t) + sizeof(float)) + (size_t)E * sizeof(int32_t);
}

extern "C" int so_router_top2(const void* x, const void* w_gate, int T, int H, int E, int32_t* topk_idx,
                              float* topk_w, int32_t* expert_offsets, int32_t* perm_token, float* row_weight,
                              int32_t* token_rows, void* x_perm, void* workspace, void* stream) {
  SO_REQUIRE(x && w_gate && expert_offsets && perm_token && row_weight && token_rows && x_perm && workspace,
             SO_E_NULLPTR);
  SO_REQUIRE(T >= 0 && H > 0 && H % 8 == 0 && E >= 2 && E <= kMaxE, SO_E_SHAPE);
  SO_REQUIRE(aligned16(x) && aligned16(w_gate) && aligned16(x_perm), SO_E_ALIGN);
  cudaStream_t st = as_stream(stream);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  int32_t* counts = reinterpret_cast<int32_t*>(ws);
  int32_t* idx = topk_idx ? topk_idx : reinterpret_cast<int32_t*>(ws + 256);
  float* w = topk_w ? topk_w : reinterpret_cast<float*>(ws + 256 + (size_t)T * 2 * sizeof(int32_t));
  cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(int32_t) * E, st);
  if (e != cudaSuccess) return (int)e;
  if (T > 0) {
    const int warps = 8;
    route_kernel<<<(T + warps - 1) / warps, warps * 32, 0, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(x), reinterpret_cast<const __nv_bfloat16*>(w_gate), T, H, E, idx,
        w, counts);
    SO_CHECK_LAUNCH();
  }
  scan_kernel<<<1, kScanThreads, 0, st>>>(idx, w, counts, T, E, expert_offsets, perm_token, row_weight,
                                          token_rows);
  SO_CHECK_LAUNCH();
  if (T > 0) {
    gather_rows_kernel<<<grid_for((size_t)2 * T * (H / 8), 256), 256, 0, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(x), perm_token, 2 * T, H, reinterpret_cast<__nv_bfloat16*>(x_perm));
    SO_CHECK_LAUNCH();
  }
  return SO_OK;
}

extern "C" int so_moe_combine(const void* y_perm, const int32_t* token_rows, const void* resid, int T, int H,
                              void* out, void* stream) {
  SO_REQUIRE(y_perm && token_rows && resid && out, SO_E_NULLPTR);
  SO_REQUIRE(T >= 0 && H > 0 && H % 8 == 0, SO_E_SHAPE);
  SO_REQUIRE(aligned16(y_perm) && aligned16(resid) && aligned16(out), SO_E_ALIGN);
  if (T == 0) return SO_OK;
  combine_kernel<<<grid_for((size_t)T * (H / 8), 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(y_perm), token_rows, reinterpret_cast<const __nv_bfloat16*>(resid), T,
      H, reinterpret_cast<__nv_bfloat16*>(out));
  SO_CHECK_LAUNCH();
  return SO_OK;
}
