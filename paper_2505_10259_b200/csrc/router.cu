// K2 — fused Mixtral top-2 router + stable expert-major token permutation, and
// the deterministic two-slot combine that closes the MoE block.
//
// The reference charges the whole MoE block as one `ffn_gpu` event per layer
// (simulator.py:185-191); its routing semantics are the third-party Mixtral
// block (transformers modeling_mixtral.py: fp32 softmax → top-2 → renormalise),
// cited in SURVEY.md §8c.  ONE cooperative launch, no host synchronisation.
// CTA c owns the contiguous token range [T·c/G, T·(c+1)/G):
//   A. route:   one warp per token — E dot products (fp32), top-2 (ties → lower
//               expert index), pair-renormalised weights; a per-CTA expert
//               histogram in shared memory, published to the workspace;
//   —  grid barrier (all CTAs are co-resident: cooperative launch, ≤ one wave);
//   B. place:   every CTA sums the published histograms — expert offsets
//               (exclusive scan over experts) plus its own base inside each
//               expert (the counts of lower CTAs) — then ranks its (token, slot)
//               pairs stably in token order with __match_any_sync + popc, so
//               the permutation is the same as one global stable sort;
//   C. gather:  x_perm[row] = x[token] for its own tokens, 16-B vectors (the x
//               rows were read in A a few µs earlier: L2 hits).
#include <map>
#include <mutex>

#include "common.cuh"

namespace {

constexpr int kMaxE = 16;  // Mixtral uses 8; accumulators stay in registers

constexpr int kRThreads = 512;
constexpr size_t kRouterSmemMax = 160 * 1024;  // the gate weights E·H bf16 staged in shared memory up to this
constexpr int kRWarps = kRThreads / 32;
constexpr int kMaxRouterCtas = 1024;

__device__ __forceinline__ void route_token(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* wg,
                                            int t, int H, int E, int lane, int& i0, int& i1, float& w0, float& w1) {
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
      unpack8(reinterpret_cast<const int4*>(wg + (size_t)e * H)[c], wf);
      float s = 0.0f;
#pragma unroll
      for (int j = 0; j < 8; ++j) s = fmaf(xf[j], wf[j], s);
      acc[e] += s;
    }
  }
  float l0 = -3.4e38f, l1 = -3.4e38f;
  i0 = 0;
  i1 = 1;
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
  // softmax over all E then renormalising the top pair == softmax over the pair
  w1 = 1.0f / (1.0f + expf(l0 - l1));
  w0 = 1.0f - w1;
}

__global__ void __launch_bounds__(kRThreads) router_fused_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg, int T, int H, int E,
    int32_t* __restrict__ topk_idx, float* __restrict__ topk_w, int32_t* __restrict__ cta_counts,
    unsigned int* __restrict__ barrier, int32_t* __restrict__ offs, int32_t* __restrict__ perm_token,
    float* __restrict__ row_weight, int32_t* __restrict__ token_rows, __nv_bfloat16* __restrict__ x_perm,
    int stage_w) {
  __shared__ int s_cnt[kMaxE];
  __shared__ int s_cursor[kMaxE];
  __shared__ int s_warp_cnt[kRWarps][kMaxE];
  const int G = gridDim.x, c = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t0 = (int)((long)T * c / G), t1 = (int)((long)T * (c + 1) / G);
  if (tid < kMaxE) s_cnt[tid] = 0;
  // the gate weights (Mixtral-8x22B: 8 × 6144 bf16 = 96 KB) read once per CTA into shared memory:
  // every token's E dot products then read them at shared-memory speed instead of through L1/L2
  extern __shared__ int4 s_wg[];
  const __nv_bfloat16* wsrc = wg;
  if (stage_w) {
    const int n16 = E * H / 8;
    for (int i = tid; i < n16; i += kRThreads) s_wg[i] = __ldg(reinterpret_cast<const int4*>(wg) + i);
    wsrc = reinterpret_cast<const __nv_bfloat16*>(s_wg);
  }
  __syncthreads();

  // ---- A. route this CTA's tokens ----
  for (int t = t0 + warp; t < t1; t += kRWarps) {
    int i0, i1;
    float w0, w1;
    route_token(x, wsrc, t, H, E, lane, i0, i1, w0, w1);
    if (lane == 0) {
      topk_idx[2 * t] = i0;
      topk_idx[2 * t + 1] = i1;
      topk_w[2 * t] = w0;
      topk_w[2 * t + 1] = w1;
      atomicAdd(&s_cnt[i0], 1);
      atomicAdd(&s_cnt[i1], 1);
    }
  }
  __syncthreads();
  if (tid < E) cta_counts[c * kMaxE + tid] = s_cnt[tid];

  // ---- grid barrier: every CTA's histogram published (bounded spin: an error, never a hung GPU) ----
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    atomicAdd(barrier, 1u);
    unsigned int polls = 0;
    while (atomicAdd(barrier, 0u) < (unsigned int)G) {
      if (++polls > (1u << 28)) __trap();
      __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();

  // ---- B. offsets and this CTA's base inside each expert ----
  if (tid < E) {
    int below = 0, total = 0;
    for (int k = 0; k < G; ++k) {
      const int v = __ldcg(&cta_counts[k * kMaxE + tid]);
      total += v;
      if (k < c) below += v;
    }
    s_cnt[tid] = total;
    s_cursor[tid] = below;
  }
  __syncthreads();
  if (tid == 0) {
    int a = 0;
    for (int e = 0; e < E; ++e) {
      s_cursor[e] += a;  // offs[e] + rows of expert e owned by lower CTAs
      if (c == 0) offs[e] = a;
      a += s_cnt[e];
    }
    if (c == 0) offs[E] = a;
  }
  __syncthreads();
  // stable rank of every (token, slot) pair of [2·t0, 2·t1) inside its expert, token order
  for (int tile = 2 * t0; tile < 2 * t1; tile += kRThreads) {
    const int p = tile + tid;
    const bool live = p < 2 * t1;
    const int e = live ? topk_idx[p] : -1;
    for (int i = tid; i < kRWarps * kMaxE; i += kRThreads) (&s_warp_cnt[0][0])[i] = 0;
    __syncthreads();
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int rank_in_warp = __popc(peers & ((1u << lane) - 1u));
    if (live && rank_in_warp == 0) s_warp_cnt[warp][e] = __popc(peers);
    __syncthreads();
    if (live) {
      int before = 0;
      for (int w = 0; w < warp; ++w) before += s_warp_cnt[w][e];
      const int row = s_cursor[e] + before + rank_in_warp;
      perm_token[row] = p >> 1;
      row_weight[row] = topk_w[p];
      token_rows[p] = row;
    }
    __syncthreads();
    if (tid < E) {
      int tot = 0;
      for (int w = 0; w < kRWarps; ++w) tot += s_warp_cnt[w][tid];
      s_cursor[tid] += tot;
    }
    __syncthreads();
  }

  // ---- C. gather this CTA's tokens into their two expert rows ----
  const int vec = H / 8;
  for (int p = 2 * t0 + warp; p < 2 * t1; p += kRWarps) {
    const int row = token_rows[p];
    const int4* src = reinterpret_cast<const int4*>(x + (size_t)(p >> 1) * H);
    int4* dst = reinterpret_cast<int4*>(x_perm + (size_t)row * H);
    for (int v = lane; v < vec; v += 32) dst[v] = __ldg(src + v);
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


int router_grid(int T, size_t smem) {
  // co-resident CTAs of the cooperative launch at this shared-memory size (per process; fixed for a device model)
  static std::mutex mu;
  static std::map<size_t, int> per_size;
  int max_ctas;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = per_size.find(smem);
    if (it == per_size.end()) {
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, router_fused_kernel, kRThreads, smem) != cudaSuccess)
        per_sm = 1;
      it = per_size.emplace(smem, per_sm * device_sm_count()).first;
    }
    max_ctas = it->second;
  }
  int g = (T + kRWarps - 1) / kRWarps;  // ≥ one token per warp
  const int cap = device_sm_count() < max_ctas ? device_sm_count() : max_ctas;  // one wave: ≤ one CTA per SM
  if (g > cap) g = cap;
  if (g > kMaxRouterCtas) g = kMaxRouterCtas;
  return g < 1 ? 1 : g;
}

constexpr size_t kRouterHdr = 256 + (size_t)kMaxRouterCtas * kMaxE * sizeof(int32_t);

}  // namespace

extern "C" size_t so_router_workspace_bytes(int T, int E) {
  // barrier word + per-CTA histograms, then topk scratch for callers passing NULL topk outputs
  (void)E;
  return kRouterHdr + (size_t)T * 2 * (sizeof(int32_t) + sizeof(float));
}

extern "C" int so_router_top2(const void* x, const void* w_gate, int T, int H, int E, int32_t* topk_idx,
                              float* topk_w, int32_t* expert_offsets, int32_t* perm_token, float* row_weight,
                              int32_t* token_rows, void* x_perm, void* workspace, void* stream) {
  SO_REQUIRE(x && w_gate && expert_offsets && perm_token && row_weight && token_rows && x_perm && workspace,
             SO_E_NULLPTR);
  SO_REQUIRE(T >= 0 && H > 0 && H % 8 == 0 && E >= 2 && E <= kMaxE, SO_E_SHAPE);
  SO_REQUIRE(aligned16(x) && aligned16(w_gate) && aligned16(x_perm) && aligned16(workspace), SO_E_ALIGN);
  cudaStream_t st = as_stream(stream);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  unsigned int* barrier = reinterpret_cast<unsigned int*>(ws);
  int32_t* cta_counts = reinterpret_cast<int32_t*>(ws + 256);
  int32_t* idx = topk_idx ? topk_idx : reinterpret_cast<int32_t*>(ws + kRouterHdr);
  float* w = topk_w ? topk_w : reinterpret_cast<float*>(ws + kRouterHdr + (size_t)T * 2 * sizeof(int32_t));
  cudaError_t e = cudaMemsetAsync(barrier, 0, sizeof(unsigned int), st);
  if (e != cudaSuccess) return (int)e;
  const size_t wbytes = (size_t)E * H * sizeof(__nv_bfloat16);
  int stage_w = wbytes <= kRouterSmemMax ? 1 : 0;
  const size_t smem = stage_w ? wbytes : 0;
  if (stage_w) {
    if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(router_fused_kernel), smem)) return rc;
  }
  const int grid = router_grid(T, smem);
  const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(x);
  const __nv_bfloat16* wb = reinterpret_cast<const __nv_bfloat16*>(w_gate);
  __nv_bfloat16* xp = reinterpret_cast<__nv_bfloat16*>(x_perm);
  void* args[] = {&xb, &wb, &T, &H, &E, &idx, &w, &cta_counts, &barrier, &expert_offsets, &perm_token, &row_weight,
                  &token_rows, &xp, &stage_w};
  // cooperative: the runtime guarantees every CTA is resident at once (the grid barrier needs it)
  e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(router_fused_kernel), dim3(grid), dim3(kRThreads),
                                  args, smem, st);
  if (e != cudaSuccess) return (int)e;
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
