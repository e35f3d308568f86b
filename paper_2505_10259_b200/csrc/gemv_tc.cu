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

// 16-B asynchronous store into (possibly another CTA's) shared memory; completion is counted in bytes on
// the destination CTA's mbarrier (complete_tx), so the receiver needs no round trip to the sender
__device__ __forceinline__ void st_async4(uint32_t cluster_addr, const uint32_t* v, uint32_t cluster_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   cluster_addr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(cluster_bar)
               : "memory");
}

// wait with cluster-scope acquire: the data the peers' asynchronous stores delivered is visible
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

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
  uint8_t* sW = smem;
  uint8_t* sX = smem + (size_t)stages * kWBytes;
  // receive buffer of the rows this CTA reduces: [CS senders][its rows][NT + 4] fp32 (a row's tokens
  // contiguous for 16-B loads; the 4-float pad spreads the rows over the banks)
  const int ldr = NT + 4;
  float* red = reinterpret_cast<float*>(smem + (size_t)stages * stage_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(red + (size_t)(kWRows + kMaxCluster) * ldr);
  uint64_t* empty = full + kGMaxStages;
  uint64_t* tmem_full = empty + kGMaxStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint64_t* ready = tmem_empty + 2;     // every sender's slice of the rows I reduce has landed (tx bytes)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(ready + 2);

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
    mbar_init(ready, 1);
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
      // The weights never depend on the previous kernel: the first `stages` weight tiles are
      // requested before griddep_wait(), so under programmatic dependent launch they stream
      // while the kernel that produces X (and the residual) finishes; X loads follow the wait.
      const uint32_t pre = (uint32_t)stages;
      {
        uint32_t it = 0;
        for (int tile = cluster; tile < n_tiles && it < pre; tile += n_clusters)
          for (int kb = kb_lo; kb < kb_hi && it < pre; ++kb, ++it) {
            mbar_expect_tx(&full[it], stage_bytes);  // weights + tokens land on the same barrier
            tma_load_2d(sW + (size_t)it * kWBytes, &tmW, &full[it], kb * kTmaBoxK, tile * kWRows);
          }
      }
      griddep_wait();
      uint32_t it = 0;
      for (int tile = cluster; tile < n_tiles; tile += n_clusters) {
        for (int kb = kb_lo; kb < kb_hi; ++kb, ++it) {
          const int s = it % stages;
          if (it >= pre) {
            const uint32_t ph = (it / stages) & 1;
            mbar_wait_guard(&empty[s], ph ^ 1);
            mbar_expect_tx(&full[s], stage_bytes);
            tma_load_2d(sW + (size_t)s * kWBytes, &tmW, &full[s], kb * kTmaBoxK, tile * kWRows);
          }
          if (it == 0) gtrace(2);
          tma_load_2d(sX + (size_t)s * xbytes, &tmX, &full[s], kb * kTmaBoxK, 0);
        }
      }
    } else {
      griddep_wait();
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
    // ===== epilogue warps: TMEM partial → pushed to the row's owner CTA → owner reduces its rows =====
    griddep_wait();  // the residual (aux) and C's previous readers belong to earlier kernels
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int tid = threadIdx.x - 64;  // 0..127
    const bool swiglu = EPI == SO_EPI_SWIGLU;
    // row ownership: CTA r reduces rows [r_lo, r_hi) of the tile (SwiGLU: gate rows of the lower
    // half, each with its up row + 64)
    const int R = swiglu ? kWRows / 2 : kWRows;
    const int r_lo = (int)((long)R * rank / CS), r_hi = (int)((long)R * (rank + 1) / CS);
    const int nr = r_hi - r_lo;
    // where MY row goes: owner CTA, its local row index in each sender's block, the block's row count
    const int key = swiglu ? (row & 63) : row;
    int owner = (int)(((long)key * CS) / R);
    while (owner > 0 && (int)((long)R * owner / CS) > key) --owner;
    while (owner + 1 < (int)CS && (int)((long)R * (owner + 1) / CS) <= key) ++owner;
    const int o_lo = (int)((long)R * owner / CS), o_nr = (int)((long)R * (owner + 1) / CS) - o_lo;
    const int blk_rows = swiglu ? 2 * o_nr : o_nr;
    const int li = key - o_lo + ((swiglu && row >= 64) ? o_nr : 0);
    // receive buffer [CS senders][blk_rows][ldr] on the owner; my slice starts at sender block `rank`
    const uint32_t dst = (CS > 1 ? map_peer(smem_u32(red), owner) : smem_u32(red)) +
                         (uint32_t)(((int)rank * blk_rows + li) * ldr * 4);
    const uint32_t dst_bar = CS > 1 ? map_peer(smem_u32(ready), owner) : smem_u32(ready);
    const int my_blk = swiglu ? 2 * nr : nr;                  // rows per sender block that I receive
    const int quads = (M + 3) / 4;                            // 16-B token quads per row
    const uint32_t tx = (uint32_t)(CS * my_blk * quads * 16);  // bytes all senders push to me, per tile
    uint32_t acc_i = 0;
    for (int tile = cluster; tile < n_tiles; tile += n_clusters, ++acc_i) {
      const uint32_t buf = acc_i & 1, aph = (acc_i >> 1) & 1;
      if (acc_i > 0) asm volatile("bar.sync 2, 128;" ::: "memory");  // CS == 1: my previous tile's reads done
      if (tid == 0) mbar_expect_tx(ready, tx);                       // arm before or after the pushes land
      mbar_wait_guard(&tmem_full[buf], aph);
      if (tid == 0) gtrace(4);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tbase = tmem_base + buf * (acc_cols / 2) + ((uint32_t)(quarter * 32) << 16);
      for (int c = 0; c < M; c += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if ((c >> 2) + j < quads)  // 16-B asynchronous stores into the owner's shared memory, counted on its barrier
            st_async4(dst + (uint32_t)((c + 4 * j) * 4), r + 4 * j, dst_bar);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tmem_empty[buf])) : "memory");
      mbar_wait_cluster(ready, acc_i & 1);  // every sender's slice of my rows has landed
      if (tid == 0) gtrace(5);
      const int n0 = tile * kWRows;
      // fixed sender order 0..CS-1 (deterministic); thread → (row, 4 tokens), consecutive threads on
      // consecutive rows (coalesced output stores); local 16-B loads
      for (int w = tid; w < nr * quads; w += 128) {
        const int rl = w % nr, q = w / nr;
        float4 sv = make_float4(0.f, 0.f, 0.f, 0.f), su = sv;
        for (int p = 0; p < (int)CS; ++p) {
          const float* src = red + (size_t)(p * my_blk + rl) * ldr + 4 * q;
          const float4 v = *reinterpret_cast<const float4*>(src);
          sv.x += v.x; sv.y += v.y; sv.z += v.z; sv.w += v.w;
          if (swiglu) {
            const float4 u = *reinterpret_cast<const float4*>(src + (size_t)nr * ldr);
            su.x += u.x; su.y += u.y; su.z += u.z; su.w += u.w;
          }
        }
        // SwiGLU: gate row ↔ output column n0/2 + row (64-row interleave of the packed FFN)
        const int n = swiglu ? n0 / 2 + r_lo + rl : n0 + r_lo + rl;
        const int m = 4 * q;
        store_out<EPI>(m, n, sv.x, su.x, C, ldc, aux);
        if (m + 1 < M) store_out<EPI>(m + 1, n, sv.y, su.y, C, ldc, aux);
        if (m + 2 < M) store_out<EPI>(m + 2, n, sv.z, su.z, C, ldc, aux);
        if (m + 3 < M) store_out<EPI>(m + 3, n, sv.w, su.w, C, ldc, aux);
      }
      if (tid == 0) gtrace(6);
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

// SO_NO_PDL=1 launches K5c with plain stream serialization (A/B measurement); read once
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("SO_NO_PDL");
    return !(v && v[0] && v[0] != '0');
  }();
  return on;
}

struct GemvPlan {
  int NT, stages, CS, clusters, n_tiles;
};

size_t smem_bytes(int NT, int stages) {
  return 1024 + (size_t)stages * (kWBytes + NT * kTmaBoxK * 2) + (size_t)(NT + 4) * (kWRows + kMaxCluster) * 4 + 512;
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
  p.stages = (int)((kGSmemBudget - (size_t)(p.NT + 4) * (kWRows + kMaxCluster) * 4 - 2048) / stage);
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
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // programmatic dependent launch: the kernel may start while its predecessor finishes; it prefetches
  // weights, then griddepcontrol.wait()s before touching anything the predecessor wrote
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
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
