// K5b — weight-streaming GEMM for decode steps: M ≤ 128 activation rows.
//
//   C[m, n] = EPI( Σ_k X[m, k] · W[n, k] )      X [M, K] bf16, W [N, K] bf16
//
// A draft decode step (costmodel.py:53-57 `t_draft_decode_gpu`; SURVEY.md §8
// a17) multiplies 16–128 token rows by every weight of the layer once: the
// work is the weight bytes, so the kernel must stream W from HBM at the
// memory roofline on all 148 SMs.  Three choices follow from that:
//
// * swap A/B: the tcgen05 MMA's M = 128 side is a tile of 128 WEIGHT rows and
//   its N side the NT ≤ 128 token rows (rounded up to 16), so no operand is
//   padded to 128 rows — a k-block moves 16 KB of weights + NT·128 B of
//   activations through shared memory instead of 2 × 16 KB;
// * stream-K: the (n-tile, k-block) space is cut into equal contiguous ranges,
//   one per persistent CTA, so every SM streams the same weight bytes — no
//   wave tail for 32- or 48-tile projections;
// * in-kernel fixup: a tile split across CTAs leaves fp32 partials in the
//   workspace; the CTA that finishes the tile's LAST contribution (a per-tile
//   arrival counter) sums them in contributor order — deterministic — and
//   applies the epilogue.  No second kernel.
//
// Warp roles (192 threads, one CTA per SM): warp 0 TMA producer, warp 1 TMEM
// allocator + single-thread MMA issuer, warps 2–5 epilogue (TMEM lane window
// = weight row, 32 token columns per tcgen05.ld).  Two TMEM accumulators let
// the MMA of the next segment overlap the previous segment's epilogue.
#include "tc_common.cuh"

namespace {

constexpr int kGThreads = 192;
constexpr int kGMaxStages = 12;
constexpr int kWRows = 128;                   // weight rows per tile (MMA M)
constexpr int kWBytes = kWRows * kTmaBoxK * 2;  // 16 KB per k-block
constexpr size_t kGSmemBudget = 200 * 1024;
constexpr size_t kArrivalBytes = 64 * 1024;   // per-tile arrival counters: ≤ 16384 weight tiles (N ≤ 2 Mi)

// contiguous range [lo, hi) of the flattened (tile, k-block) space owned by CTA g of G
__device__ __forceinline__ void cta_range(long total, int g, int G, long& lo, long& hi) {
  lo = total * g / G;
  hi = total * (g + 1) / G;
}

// first CTA whose range contains flattened index x
__device__ __forceinline__ int owner(long x, long total, int G) {
  int g = (int)((x * G) / total);
  while (g > 0 && total * g / G > x) --g;
  while (g + 1 < G && total * (g + 1) / G <= x) ++g;
  return g;
}

template <int EPI>
__device__ __forceinline__ void store_row(int row, int n, int M, int NT, const float* acc, void* __restrict__ C, int ldc,
                                          const void* __restrict__ aux, float* swap) {
  // acc[m] for m < NT: this thread's weight row n, every token column m
  if constexpr (EPI == SO_EPI_SWIGLU) {
    // rows [0,64) of the tile are gate rows, [64,128) the matching up rows
    // (64-row interleave of the packed FFN): the up threads publish, the gate
    // threads combine and write output column (n0/2) + row
    const int j = row & 63;
    if (row >= 64)
      for (int m = 0; m < NT; ++m) swap[m * 64 + j] = acc[m];
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (row < 64) {
      const int col = (n - row) / 2 + j;
      __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(C);
      for (int m = 0; m < M; ++m) out[(size_t)m * ldc + col] = f2bf(silu(acc[m]) * swap[m * 64 + j]);
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
  } else if constexpr (EPI == SO_EPI_F32) {
    float* out = reinterpret_cast<float*>(C);
    for (int m = 0; m < M; ++m) out[(size_t)m * ldc + n] = acc[m];
  } else if constexpr (EPI == SO_EPI_BF16_RESID) {
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(C);
    const __nv_bfloat16* res = reinterpret_cast<const __nv_bfloat16*>(aux);
    for (int m = 0; m < M; ++m)
      out[(size_t)m * ldc + n] = f2bf(bf2f(f2bf(acc[m])) + bf2f(res[(size_t)m * ldc + n]));
  } else {
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(C);
    for (int m = 0; m < M; ++m) out[(size_t)m * ldc + n] = f2bf(acc[m]);
  }
}

template <int EPI>
__global__ void __launch_bounds__(kGThreads, 1)
    gemv_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, int M, int N,
                   int K, int NT, int stages, void* __restrict__ C, int ldc, const void* __restrict__ aux,
                   float* __restrict__ partials, int* __restrict__ arrivals, int max_contrib) {
  const int num_kb = K / kTmaBoxK;
  const int n_tiles = N / kWRows;
  const long total = (long)n_tiles * num_kb;
  const int G = gridDim.x, g = blockIdx.x;
  long lo, hi;
  cta_range(total, g, G, lo, hi);
  const uint32_t xbytes = (uint32_t)NT * kTmaBoxK * 2;
  const uint32_t stage_bytes = kWBytes + xbytes;
  // two accumulators, each a power of two ≥ 32 columns (tcgen05.ld reads 32 at a time)
  const uint32_t acc_cols = NT <= 32 ? 64 : (NT <= 64 ? 128 : 256);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sX = smem + (size_t)stages * kWBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * stage_bytes);
  uint64_t* empty = full + kGMaxStages;
  uint64_t* tmem_full = empty + kGMaxStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_holder + 1);
  float* swap = reinterpret_cast<float*>(smem + (size_t)stages * stage_bytes + 1024);  // SwiGLU exchange [NT][64]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(acc_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer: this CTA's k-blocks, tile by tile =====
      uint32_t it = 0;
      for (long x = lo; x < hi;) {
        const int tile = (int)(x / num_kb);
        const int kb1 = (int)min((long)num_kb, hi - (long)tile * num_kb);
        for (int kb = (int)(x - (long)tile * num_kb); kb < kb1; ++kb, ++it) {
          const int s = it % stages;
          const uint32_t ph = (it / stages) & 1;
          mbar_wait_guard(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], stage_bytes);
          tma_load_2d(sW + (size_t)s * kWBytes, &tmW, &full[s], kb * kTmaBoxK, tile * kWRows);
          tma_load_2d(sX + (size_t)s * xbytes, &tmX, &full[s], kb * kTmaBoxK, 0);
        }
        x = (long)(tile + 1) * num_kb;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer: D[128 weight rows, NT tokens] += W_tile · X_tileᵀ =====
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NT >> 3) << 17) |
                             ((uint32_t)(kWRows >> 4) << 24);
      uint32_t it = 0, acc = 0;
      for (long x = lo; x < hi; ++acc) {
        const int tile = (int)(x / num_kb);
        const int kb0 = (int)(x - (long)tile * num_kb);
        const int kb1 = (int)min((long)num_kb, hi - (long)tile * num_kb);
        const uint32_t buf = acc & 1, aph = (acc >> 1) & 1;
        mbar_wait_guard(&tmem_empty[buf], aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem_base + buf * (acc_cols / 2);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % stages;
          const uint32_t ph = (it / stages) & 1;
          mbar_wait_guard(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a0 = smem_u32(sW + (size_t)s * kWBytes);
          const uint32_t b0 = smem_u32(sX + (size_t)s * xbytes);
#pragma unroll
          for (int kk = 0; kk < kTmaBoxK / 16; ++kk)
            umma_bf16(d, umma_desc_sw128(a0 + kk * 32), umma_desc_sw128(b0 + kk * 32), idesc,
                      (kb != kb0) | (kk != 0));
          umma_commit(&empty[s]);
        }
        umma_commit(&tmem_full[buf]);
        x = (long)(tile + 1) * num_kb;
      }
    }
  } else {
    // ===== epilogue warps: one weight row per thread =====
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    uint32_t acc_i = 0;
    float accv[128];
    for (long x = lo; x < hi; ++acc_i) {
      const int tile = (int)(x / num_kb);
      const long t0 = (long)tile * num_kb, t1 = t0 + num_kb;
      const uint32_t buf = acc_i & 1, aph = (acc_i >> 1) & 1;
      mbar_wait_guard(&tmem_full[buf], aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tbase = tmem_base + buf * (acc_cols / 2) + ((uint32_t)(quarter * 32) << 16);
      for (int c = 0; c < NT; c += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) accv[c + j] = __uint_as_float(r[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tmem_empty[buf])) : "memory");
      const int n = tile * kWRows + row;
      const int first = owner(t0, total, G), last = owner(t1 - 1, total, G);
      if (first == last) {  // the whole tile is this CTA's: epilogue straight from the accumulator
        store_row<EPI>(row, n, M, NT, accv, C, ldc, aux, swap);
      } else {
        // publish this contribution, token-major [NT][128] (coalesced across the rows)
        float* slot = partials + ((size_t)tile * max_contrib + (g - first)) * (size_t)NT * kWRows;
        for (int m = 0; m < NT; ++m) slot[(size_t)m * kWRows + row] = accv[m];
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) {
          const int prev = atomicAdd(&arrivals[tile], 1);
          *last_flag = prev == last - first;
          if (prev == last - first) arrivals[tile] = 0;  // every contributor arrived: reset for the next launch
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (*last_flag) {
          __threadfence();
          // fixed contributor order 0..last-first: the sum does not depend on arrival order
          const float* base = partials + (size_t)tile * max_contrib * NT * kWRows;
          // 16 token columns per step, every contributor's loads issued before the adds (L2 latency overlapped)
          for (int m0 = 0; m0 < NT; m0 += 16) {
            float s16[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) s16[i] = 0.f;
            for (int j = 0; j <= last - first; ++j) {
              const float* src = base + ((size_t)j * NT + m0) * kWRows + row;
              float v16[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) v16[i] = __ldcg(src + (size_t)i * kWRows);
#pragma unroll
              for (int i = 0; i < 16; ++i) s16[i] += v16[i];
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) accv[m0 + i] = s16[i];
          }
          store_row<EPI>(row, n, M, NT, accv, C, ldc, aux, swap);
        }
      }
      x = t1;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(acc_cols));
  }
}

struct GemvPlan {
  int NT, stages, G, n_tiles, max_contrib;
  size_t arrivals_bytes, partial_bytes;
};

GemvPlan plan_gemv(int M, int N, int K) {
  GemvPlan p{};
  p.NT = ((M + 15) / 16) * 16;
  if (p.NT < 16) p.NT = 16;
  const int stage = kWBytes + p.NT * kTmaBoxK * 2;
  p.stages = (int)((kGSmemBudget - (size_t)p.NT * 64 * 4 - 2048) / stage);
  if (p.stages > kGMaxStages) p.stages = kGMaxStages;
  p.n_tiles = N / kWRows;
  const long total = (long)p.n_tiles * (K / kTmaBoxK);
  int G = device_sm_count();
  if (total < (long)G * 2) G = (int)((total + 1) / 2);  // ≥ 2 k-blocks per CTA
  if (G < 1) G = 1;
  p.G = G;
  // contributors of one tile: ≤ ceil(num_kb / per_cta) + 1
  const long per = total / G;
  p.max_contrib = (int)((K / kTmaBoxK + per - 1) / (per > 0 ? per : 1)) + 2;
  // a FIXED counter region for every shape: a workspace serves many shapes in
  // turn, and a shape with fewer tiles must not lay its partials over counters
  // a wider shape relies on being zero
  p.arrivals_bytes = kArrivalBytes;
  p.partial_bytes = (size_t)p.n_tiles * p.max_contrib * p.NT * kWRows * 4;
  return p;
}

size_t smem_bytes(const GemvPlan& p) {
  return 1024 + (size_t)p.stages * (kWBytes + p.NT * kTmaBoxK * 2) + 1024 + (size_t)p.NT * 64 * 4;
}

template <int EPI>
int launch_gemv(const GemvPlan& p, const CUtensorMap& mw, const CUtensorMap& mx, int M, int N, int K, void* C,
                int ldc, const void* aux, uint8_t* ws, cudaStream_t st) {
  auto kern = gemv_tc_kernel<EPI>;
  const size_t smem = smem_bytes(p);
  if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem)) return rc;
  kern<<<p.G, kGThreads, smem, st>>>(mw, mx, M, N, K, p.NT, p.stages, C, ldc, aux,
                                     reinterpret_cast<float*>(ws + p.arrivals_bytes), reinterpret_cast<int*>(ws),
                                     p.max_contrib);
  SO_CHECK_LAUNCH();
  return SO_OK;
}

}  // namespace

extern "C" size_t so_gemv_workspace_bytes(int M, int N, int K) {
  if (M <= 0 || M > 128 || N <= 0 || K <= 0 || N % kWRows || K % kTmaBoxK) return 0;
  if ((size_t)(N / kWRows) * sizeof(int) > kArrivalBytes) return 0;
  const GemvPlan p = plan_gemv(M, N, K);
  return p.arrivals_bytes + p.partial_bytes;
}

extern "C" int so_gemv_bf16(const void* X, const void* W, int M, int N, int K, void* C, int ldc, int epilogue,
                            const void* aux, void* workspace, size_t ws_bytes, void* stream) {
  SO_REQUIRE(X && W && C && workspace, SO_E_NULLPTR);
  SO_REQUIRE(M >= 0 && M <= 128 && N > 0 && K > 0 && N % kWRows == 0 && K % kTmaBoxK == 0, SO_E_SHAPE);
  SO_REQUIRE((size_t)(N / kWRows) * sizeof(int) <= kArrivalBytes, SO_E_SHAPE);
  SO_REQUIRE(aligned16(X) && aligned16(W) && aligned16(workspace), SO_E_ALIGN);
  if (epilogue == SO_EPI_SWIGLU) SO_REQUIRE(ldc >= N / 2, SO_E_SHAPE);
  else SO_REQUIRE(ldc >= N, SO_E_SHAPE);
  if (epilogue == SO_EPI_BF16_RESID) SO_REQUIRE(aux != nullptr, SO_E_NULLPTR);
  if (M == 0) return SO_OK;
  const GemvPlan p = plan_gemv(M, N, K);
  SO_REQUIRE(ws_bytes >= p.arrivals_bytes + p.partial_bytes, SO_E_SHAPE);
  CUtensorMap mw, mx;
  int rc = make_map_2d(&mw, W, (uint64_t)N, (uint64_t)K, kWRows);
  if (rc) return rc;
  rc = make_map_2d(&mx, X, (uint64_t)M, (uint64_t)K, (uint32_t)p.NT);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  switch (epilogue) {
    case SO_EPI_BF16: return launch_gemv<SO_EPI_BF16>(p, mw, mx, M, N, K, C, ldc, aux, ws, st);
    case SO_EPI_F32: return launch_gemv<SO_EPI_F32>(p, mw, mx, M, N, K, C, ldc, aux, ws, st);
    case SO_EPI_BF16_RESID: return launch_gemv<SO_EPI_BF16_RESID>(p, mw, mx, M, N, K, C, ldc, aux, ws, st);
    case SO_EPI_SWIGLU: return launch_gemv<SO_EPI_SWIGLU>(p, mw, mx, M, N, K, C, ldc, aux, ws, st);
    default: return SO_E_UNSUPPORTED;
  }
}
