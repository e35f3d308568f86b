// K5c — weight-streaming GEMM for decode steps: M ≤ 128 activation rows.
//
//   C[m, n] = EPI( Σ_k X[m, k] · W[n, k] )      X [M, K] bf16, W [N, K] bf16
//
// A draft decode step (costmodel.py:53-57 `t_draft_decode_gpu`; SURVEY.md §8
// a17) multiplies 16–128 token rows by every weight of the layer once: the
// work is the weight bytes, so the kernel must stream W from HBM at the
// memory roofline on (nearly) all 148 SMs.  Three choices follow from that:
//
// * swap A/B: the tcgen05 MMA's M = 128 side is a tile of 128 WEIGHT rows and
//   its N side the NT ≤ 128 token rows (rounded up to 16), so no operand is
//   padded to 128 rows — a k-block moves 16 KB of weights + NT·128 B of
//   activations through shared memory instead of 2 × 16 KB;
// * split-K inside a thread-block CLUSTER: a projection has only N/128 = 32–48
//   weight tiles, so each tile's K range is cut over the C ≤ 8 CTAs of one
//   cluster (C·tiles ≤ SMs) and every SM streams an equal share of the weights;
// * the split is reduced through DISTRIBUTED SHARED MEMORY: each CTA leaves its
//   fp32 partial tile in its own shared memory, signals its peers through
//   their mbarriers (release.cluster), and then sums 1/C of the tile's rows
//   over all C partials in fixed CTA order (deterministic) and applies the
//   epilogue — no global partials, no atomics, no second kernel, and the
//   reduction is spread over the whole cluster instead of one last CTA.
//
// Warp roles (192 threads, one CTA per SM): warp 0 TMA producer, warp 1 TMEM
// allocator + single-thread MMA issuer, warps 2–5 epilogue (TMEM lane window
// = weight row, 32 token columns per tcgen05.ld).  Two TMEM accumulators let
// the next tile's MMA overlap the previous tile's reduction when a cluster
// owns more than one tile.
#include <map>
#include <mutex>

#include "tc_common.cuh"

namespace {

constexpr int kGThreads = 192;
constexpr int kGMaxStages = 12;
constexpr int kWRows = 128;                   // weight rows per tile (MMA M)
constexpr int kWBytes = kWRows * kTmaBoxK * 2;  // 16 KB per k-block
constexpr size_t kGSmemBudget = 200 * 1024;
constexpr int kMaxCluster = 8;

__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t n;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
  return n;
}

__device__ __forceinline__ uint32_t map_peer(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}

__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// wait with cluster-scope acquire: the peers' shared-memory writes before their release-arrive are visible
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0, spins = 0;
  const uint32_t a = smem_u32(bar);
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (++spins > (1u << 26)) __trap();
  } while (!done);
}

__device__ __forceinline__ float ld_dsmem(uint32_t cluster_addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(cluster_addr) : "memory");
  return v;
}

#ifdef SO_GEMV_TRACE
// debug build only (make EXTRA=-DSO_GEMV_TRACE): per-CTA phase timestamps, read by so_gemv_trace_copy
__device__ unsigned long long g_gemv_trace[1024][8];
__device__ __forceinline__ void gtrace(int slot) {
  if (blockIdx.x < 1024) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_gemv_trace[blockIdx.x][slot] = t;
  }
}
#else
__device__ __forceinline__ void gtrace(int) {}
#endif

template <int EPI>
__device__ __forceinline__ void store_out(int m, int n, float v, float up, void* __restrict__ C, int ldc,
                                          const void* __restrict__ aux) {
  if constexpr (EPI == SO_EPI_SWIGLU) {
    reinterpret_cast<__nv_bfloat16*>(C)[(size_t)m * ldc + n] = f2bf(silu(v) * up);
  } else if constexpr (EPI == SO_EPI_F32) {
    reinterpret_cast<float*>(C)[(size_t)m * ldc + n] = v;
  } else if constexpr (EPI == SO_EPI_BF16_RESID) {
    const __nv_bfloat16* res = reinterpret_cast<const __nv_bfloat16*>(aux);
    reinterpret_cast<__nv_bfloat16*>(C)[(size_t)m * ldc + n] = f2bf(bf2f(f2bf(v)) + bf2f(res[(size_t)m * ldc + n]));
  } else {
    reinterpret_cast<__nv_bfloat16*>(C)[(size_t)m * ldc + n] = f2bf(v);
  }
}

template <int EPI>
__global__ void __launch_bounds__(kGThreads, 1)
    gemv_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, int M, int N,
                   int K, int NT, int stages, void* __restrict__ C, int ldc, const void* __restrict__ aux) {
  if (threadIdx.x == 0) gtrace(0);
  const int num_kb = K / kTmaBoxK;
  const int n_tiles = N / kWRows;
  const uint32_t CS = cluster_size();
  const uint32_t rank = CS > 1 ? cluster_rank() : 0;
  const int cluster = blockIdx.x / CS, n_clusters = gridDim.x / CS;
  const int kb_lo = (int)((long)num_kb * rank / CS), kb_hi = (int)((long)num_kb * (rank + 1) / CS);
  const uint32_t xbytes = (uint32_t)NT * kTmaBoxK * 2;
  const uint32_t stage_bytes = kWBytes + xbytes;
  // two accumulators, each a power of two ≥ 32 columns (tcgen05.ld reads 32 at a time)
  const uint32_t acc_cols = NT <= 32 ? 64 : (NT <= 64 ? 128 : 256);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sX = smem + (size_t)stages * kWBytes;
  float* red = reinterpret_cast<float*>(smem + (size_t)stages * stage_bytes);  // partial tile [NT][128] fp32
  uint64_t* full = reinterpret_cast<uint64_t*>(red + (size_t)NT * kWRows);
  uint64_t* empty = full + kGMaxStages;
  uint64_t* tmem_full = empty + kGMaxStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint64_t* ready = tmem_empty + 2;     // every CTA's partial of the tile is in its shared memory
  uint64_t* consumed = ready + 1;       // every CTA has read this CTA's partial
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(consumed + 1);

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
    mbar_init(ready, 4 * CS);
    mbar_init(consumed, 4 * CS);
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
  if (CS > 1) cluster_sync();  // every CTA's barriers initialised before any remote arrive
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_holder;
  if (threadIdx.x == 0) gtrace(1);

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer: this CTA's k-blocks of each of the cluster's tiles =====
      uint32_t it = 0;
      for (int tile = cluster; tile < n_tiles; tile += n_clusters) {
        for (int kb = kb_lo; kb < kb_hi; ++kb, ++it) {
          const int s = it % stages;
          const uint32_t ph = (it / stages) & 1;
          mbar_wait_guard(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], stage_bytes);
          if (it == 0) gtrace(2);
          tma_load_2d(sW + (size_t)s * kWBytes, &tmW, &full[s], kb * kTmaBoxK, tile * kWRows);
          tma_load_2d(sX + (size_t)s * xbytes, &tmX, &full[s], kb * kTmaBoxK, 0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer: D[128 weight rows, NT tokens] += W_tile · X_tileᵀ =====
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NT >> 3) << 17) |
                             ((uint32_t)(kWRows >> 4) << 24);
      uint32_t it = 0, acc = 0;
      for (int tile = cluster; tile < n_tiles; tile += n_clusters, ++acc) {
        const uint32_t buf = acc & 1, aph = (acc >> 1) & 1;
        mbar_wait_guard(&tmem_empty[buf], aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem_base + buf * (acc_cols / 2);
        for (int kb = kb_lo; kb < kb_hi; ++kb, ++it) {
          const int s = it % stages;
          const uint32_t ph = (it / stages) & 1;
          mbar_wait_guard(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a0 = smem_u32(sW + (size_t)s * kWBytes);
          const uint32_t b0 = smem_u32(sX + (size_t)s * xbytes);
#pragma unroll
          for (int kk = 0; kk < kTmaBoxK / 16; ++kk)
            umma_bf16(d, umma_desc_sw128(a0 + kk * 32), umma_desc_sw128(b0 + kk * 32), idesc,
                      (kb != kb_lo) | (kk != 0));
          umma_commit(&empty[s]);
        }
        umma_commit(&tmem_full[buf]);
      }
      gtrace(3);
    }
  } else {
    // ===== epilogue warps: TMEM partial → shared memory → cluster reduction of 1/CS of the rows =====
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int tid = threadIdx.x - 64;  // 0..127
    const uint32_t red_s = smem_u32(red);
    uint32_t red_peer[kMaxCluster];  // every peer's partial tile (own rank included), cluster addresses
#pragma unroll
    for (int p = 0; p < kMaxCluster; ++p) red_peer[p] = CS > 1 && p < (int)CS ? map_peer(red_s, p) : red_s;
    const bool swiglu = EPI == SO_EPI_SWIGLU;
    // this CTA's share of the reduction: rows [r_lo, r_hi) of the tile (SwiGLU: gate rows of the lower
    // half, each with its up row + 64)
    const int R = swiglu ? kWRows / 2 : kWRows;
    const int r_lo = (int)((long)R * rank / CS), r_hi = (int)((long)R * (rank + 1) / CS);
    const int nr = r_hi - r_lo;
    uint32_t acc_i = 0;
    for (int tile = cluster; tile < n_tiles; tile += n_clusters, ++acc_i) {
      const uint32_t buf = acc_i & 1, aph = (acc_i >> 1) & 1;
      if (acc_i > 0) mbar_wait_cluster(consumed, (acc_i - 1) & 1);  // peers are done with my previous partial
      mbar_wait_guard(&tmem_full[buf], aph);
      if (tid == 0) gtrace(4);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tbase = tmem_base + buf * (acc_cols / 2) + ((uint32_t)(quarter * 32) << 16);
      for (int c = 0; c < NT; c += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c + j < NT) red[(size_t)(c + j) * kWRows + row] = __uint_as_float(r[j]);  // token-major: conflict-free
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tmem_empty[buf])) : "memory");
        for (uint32_t p = 0; p < CS; ++p)  // release: my partial is readable by every peer
          arrive_remote(CS > 1 ? map_peer(smem_u32(ready), p) : smem_u32(ready));
      }
      mbar_wait_cluster(ready, acc_i & 1);
      if (tid == 0) gtrace(5);
      const int n0 = tile * kWRows;
      // fixed peer order 0..CS-1: the sum does not depend on arrival order; 4 outputs per
      // thread per step, every peer's DSMEM load of them issued before the adds
      const int total = nr * M;
      for (int base = tid; base < total; base += 4 * 128) {
        float v[4][kMaxCluster], u[4][kMaxCluster];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int idx = base + q * 128;
          if (idx < total) {
            const uint32_t off = (uint32_t)(((idx / nr) * kWRows + r_lo + idx % nr) * 4);
#pragma unroll
            for (int p = 0; p < kMaxCluster; ++p)
              if (p < (int)CS) {
                v[q][p] = ld_dsmem(red_peer[p] + off);
                if (swiglu) u[q][p] = ld_dsmem(red_peer[p] + off + 64 * 4);
              }
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int idx = base + q * 128;
          if (idx < total) {
            float sv = 0.f, su = 0.f;
#pragma unroll
            for (int p = 0; p < kMaxCluster; ++p)
              if (p < (int)CS) {
                sv += v[q][p];
                if (swiglu) su += u[q][p];
              }
            const int rl = r_lo + idx % nr;
            // SwiGLU: gate row rl ↔ output column n0/2 + rl (64-row interleave of the packed FFN)
            store_out<EPI>(idx / nr, swiglu ? n0 / 2 + rl : n0 + rl, sv, su, C, ldc, aux);
          }
        }
      }
      __syncwarp();
      if (tid == 0) gtrace(6);
      if (lane == 0)  // I am done reading every peer's partial
        for (uint32_t p = 0; p < CS; ++p) arrive_remote(CS > 1 ? map_peer(smem_u32(consumed), p) : smem_u32(consumed));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CS > 1) cluster_sync();  // no CTA leaves while a peer may still read its shared memory
  else __syncthreads();
  if (threadIdx.x == 0) gtrace(7);
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(acc_cols));
  }
}

struct GemvPlan {
  int NT, stages, CS, clusters, n_tiles;
};

size_t smem_bytes(int NT, int stages) {
  return 1024 + (size_t)stages * (kWBytes + NT * kTmaBoxK * 2) + (size_t)NT * kWRows * 4 + 512;
}

// how many clusters of `cs` CTAs (this kernel, this shared-memory size) the GPU holds at once: clusters
// must fit inside one GPC, so fewer than SMs / cs may be co-resident (cached, thread-safe)
template <int EPI>
int max_active_clusters(int cs, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, size_t>, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({cs, smem});
  if (it != cache.end()) return it->second;
  auto kern = gemv_tc_kernel<EPI>;
  int n = 0;
  if (ensure_smem_attr(reinterpret_cast<const void*>(kern), smem) == 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(kGThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
  }
  if (n <= 0) n = device_sm_count() / cs;  // no answer: the arithmetic bound
  cache[{cs, smem}] = n;
  return n;
}

template <int EPI>
GemvPlan plan_gemv(int M, int N, int K) {
  GemvPlan p{};
  p.NT = ((M + 15) / 16) * 16;
  if (p.NT < 16) p.NT = 16;
  const int stage = kWBytes + p.NT * kTmaBoxK * 2;
  p.stages = (int)((kGSmemBudget - (size_t)p.NT * kWRows * 4 - 2048) / stage);
  if (p.stages > kGMaxStages) p.stages = kGMaxStages;
  p.n_tiles = N / kWRows;
  const int num_kb = K / kTmaBoxK;
  const size_t smem = smem_bytes(p.NT, p.stages);
  // the widest split whose clusters ALL fit at once (one wave: every tile streamed concurrently)
  p.CS = 1;
  p.clusters = p.n_tiles;
  for (int cs = kMaxCluster; cs >= 1; --cs) {
    if (cs > 1 && (cs * p.n_tiles > device_sm_count() || num_kb < 2 * cs)) continue;
    const int fit = max_active_clusters<EPI>(cs, smem);
    if (p.n_tiles <= fit || cs == 1) {
      p.CS = cs;
      p.clusters = p.n_tiles < fit ? p.n_tiles : fit;
      break;
    }
  }
  if (p.clusters < 1) p.clusters = 1;
  return p;
}

template <int EPI>
int launch_gemv(const GemvPlan& p, const CUtensorMap& mw, const CUtensorMap& mx, int M, int N, int K, void* C,
                int ldc, const void* aux, cudaStream_t st) {
  auto kern = gemv_tc_kernel<EPI>;
  const size_t smem = smem_bytes(p.NT, p.stages);
  if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem)) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.clusters * p.CS);
  cfg.blockDim = dim3(kGThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, mw, mx, M, N, K, p.NT, p.stages, C, ldc, aux);
  if (e != cudaSuccess) return (int)e;
  SO_CHECK_LAUNCH();
  return SO_OK;
}

template <int EPI>
int run_gemv(const CUtensorMap& mw, const void* X, int M, int N, int K, void* C, int ldc, const void* aux,
             cudaStream_t st) {
  const GemvPlan p = plan_gemv<EPI>(M, N, K);
  CUtensorMap mx;
  if (int rc = make_map_2d(&mx, X, (uint64_t)M, (uint64_t)K, (uint32_t)p.NT)) return rc;
  return launch_gemv<EPI>(p, mw, mx, M, N, K, C, ldc, aux, st);
}

bool gemv_eligible(int M, int N, int K) {
  // below one tile per SM; from there on the weight tiles alone fill the SMs and the
  // persistent GEMM streams them as well
  return M > 0 && M <= 128 && N > 0 && K > 0 && N % kWRows == 0 && K % (2 * kTmaBoxK) == 0 &&
         N / kWRows < device_sm_count();
}

}  // namespace

extern "C" size_t so_gemv_workspace_bytes(int M, int N, int K) {
  // K5c reduces in distributed shared memory and needs no scratch: a token size marks eligibility (0 = not)
  return gemv_eligible(M, N, K) ? 256 : 0;
}

extern "C" int so_gemv_bf16(const void* X, const void* W, int M, int N, int K, void* C, int ldc, int epilogue,
                            const void* aux, void* workspace, size_t ws_bytes, void* stream) {
  (void)workspace;
  (void)ws_bytes;
  SO_REQUIRE(X && W && C, SO_E_NULLPTR);
  SO_REQUIRE(M >= 0 && M <= 128 && N > 0 && K > 0 && N % kWRows == 0 && K % (2 * kTmaBoxK) == 0, SO_E_SHAPE);
  SO_REQUIRE(aligned16(X) && aligned16(W), SO_E_ALIGN);
  if (epilogue == SO_EPI_SWIGLU) SO_REQUIRE(ldc >= N / 2, SO_E_SHAPE);
  else SO_REQUIRE(ldc >= N, SO_E_SHAPE);
  if (epilogue == SO_EPI_BF16_RESID) SO_REQUIRE(aux != nullptr, SO_E_NULLPTR);
  if (M == 0) return SO_OK;
  CUtensorMap mw;
  int rc = make_map_2d(&mw, W, (uint64_t)N, (uint64_t)K, kWRows);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  switch (epilogue) {
    case SO_EPI_BF16: return run_gemv<SO_EPI_BF16>(mw, X, M, N, K, C, ldc, aux, st);
    case SO_EPI_F32: return run_gemv<SO_EPI_F32>(mw, X, M, N, K, C, ldc, aux, st);
    case SO_EPI_BF16_RESID: return run_gemv<SO_EPI_BF16_RESID>(mw, X, M, N, K, C, ldc, aux, st);
    case SO_EPI_SWIGLU: return run_gemv<SO_EPI_SWIGLU>(mw, X, M, N, K, C, ldc, aux, st);
    default: return SO_E_UNSUPPORTED;
  }
}

#ifdef SO_GEMV_TRACE
extern "C" int so_gemv_trace_copy(void* host, size_t bytes) {
  if (bytes > sizeof(g_gemv_trace)) bytes = sizeof(g_gemv_trace);
  return (int)cudaMemcpyFromSymbol(host, g_gemv_trace, bytes);
}
#endif
