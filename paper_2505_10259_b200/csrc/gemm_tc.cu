// K3/K4/K5 — bf16 GEMMs on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
//   C[M,N] = A[M,K] · B[N,K]ᵀ            (dense: QKV / O / LM head / draft MLP)
//   C[r,:] = A[r,:] · B_e[N,K]ᵀ, r ∈ [offs[e], offs[e+1])   (grouped: MoE experts)
//
// Where the reference models this work: the per-layer `ffn_gpu` event
// (simulator.py:185-191, cost bs·t_ffn_gpu at costmodel.py:75) and the draft
// granules (costmodel.py:53-57).  Shapes: SURVEY.md §2c K3–K5.
//
// Kernel structure (one CTA = one 128×BN output tile, 6 warps):
//   warp 0      TMA producer: A/B k-slices (64 bf16 = 128 B rows, SWIZZLE_128B)
//               into an S-stage smem ring, completion on `full[s]` mbarriers;
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (M=128, N=BN, K=16 per instruction, fp32 accumulator in TMEM),
//               tcgen05.commit frees each smem stage on `empty[s]`;
//   warps 2..5  epilogue: tcgen05.ld 32 lanes × 32 columns per warp quarter,
//               fused op (bf16 / fp32 / +residual / SwiGLU / row scale), store.
// The grouped variant derives its M-tile → (expert, row0) map on device from
// the router's expert offsets, so no host synchronisation is needed between
// routing and the expert GEMMs.
#include "tc_common.cuh"

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one SWIZZLE_128B row
constexpr int kThreads = 192;
constexpr int kEpiWarp0 = 2;

template <int BN>
__device__ __forceinline__ constexpr uint32_t instr_desc_bf16() {
  // D=f32 (bits 4-5 = 1), A=bf16 (7-9 = 1), B=bf16 (10-12 = 1), both K-major,
  // N>>3 at 17-22, M>>4 at 24-28.
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}


template <int BN>
struct Cfg {
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = BN;  // fp32 accumulator: one column per N
  static constexpr size_t kSmem = 1024 /*align slack*/ + (size_t)kStages * kStageBytes + 256;
};


// Grouped raster of a 1-D tile index: bands of G m-tiles sweep every n-tile
// before the next band starts, so a band's A rows stay L2-resident across the
// n sweep (a 33k-row re-prefill activation would otherwise be re-read from HBM
// once per n-tile) while each B tile is shared by the band's G m-tiles.
__device__ __forceinline__ void raster_tile(int lin, int m_tiles, int n_tiles, int& mt, int& nt) {
  constexpr int G = 16;
  const int group = lin / (G * n_tiles);
  const int first = group * G;
  const int gm = min(G, m_tiles - first);
  const int r = lin - group * G * n_tiles;
  mt = first + r % gm;
  nt = r / gm;
}

// TMEM → registers → global for one thread's accumulator row (32 columns per
// tcgen05.ld), with the fused epilogue op.  `tbase` addresses lane window
// (warp % 4)·32 of the CTA's accumulator.
template <int BN, int EPI>
__device__ __forceinline__ void epilogue_tile(uint32_t tbase, bool valid, int grow, int n0, int N,
                                              void* __restrict__ C, int ldc, const void* __restrict__ aux) {
  if constexpr (EPI == SO_EPI_SWIGLU) {
    // accumulator columns [128p, 128p+64) = gate, [128p+64, 128p+128) = up
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(C);
#pragma unroll 1
    for (int p = 0; p < BN / 128; ++p) {
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        uint32_t g[32], u[32];
        tmem_ld32(tbase + p * 128 + h * 32, g);
        tmem_ld32(tbase + p * 128 + 64 + h * 32, u);
        tmem_ld_wait();
        const int col = (n0 + p * 128) / 2 + h * 32;
        if (valid && n0 + p * 128 < N) {
          float f[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] = silu(__uint_as_float(g[j])) * __uint_as_float(u[j]);
          int4* dst = reinterpret_cast<int4*>(out + (size_t)grow * ldc + col);
#pragma unroll
          for (int v = 0; v < 4; ++v) dst[v] = pack8(f + 8 * v);
        }
      }
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      tmem_ld32(tbase + c, r);
      tmem_ld_wait();
      const int col = n0 + c;
      if (!valid || col >= N) continue;
      float f[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(r[j]);
      if constexpr (EPI == SO_EPI_F32) {
        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(C) + (size_t)grow * ldc + col);
#pragma unroll
        for (int v = 0; v < 8; ++v) dst[v] = make_float4(f[4 * v], f[4 * v + 1], f[4 * v + 2], f[4 * v + 3]);
      } else {
        if constexpr (EPI == SO_EPI_BF16_RESID) {
          const int4* res =
              reinterpret_cast<const int4*>(reinterpret_cast<const __nv_bfloat16*>(aux) + (size_t)grow * ldc + col);
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            float rr[8];
            unpack8(res[v], rr);
            // round the GEMM result to bf16 first, then add (the bf16
            // `residual + o_proj(x)` of the reference models)
#pragma unroll
            for (int j = 0; j < 8; ++j) f[8 * v + j] = __bfloat162float(__float2bfloat16_rn(f[8 * v + j])) + rr[j];
          }
        } else if constexpr (EPI == SO_EPI_BF16_ROWSCALE) {
          const float w = reinterpret_cast<const float*>(aux)[grow];
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] *= w;
        }
        int4* dst = reinterpret_cast<int4*>(reinterpret_cast<__nv_bfloat16*>(C) + (size_t)grow * ldc + col);
#pragma unroll
        for (int v = 0; v < 4; ++v) dst[v] = pack8(f + 8 * v);
      }
    }
  }
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const int32_t* __restrict__ offs, int E, int M, int N, int K, void* __restrict__ C,
                   int ldc, const void* __restrict__ aux, int m_tiles, int n_tiles) {
  using CF = Cfg<BN>;
  // ---- tile → (expert, row range) -------------------------------------------
  int mt, nt;
  raster_tile(blockIdx.x, m_tiles, n_tiles, mt, nt);
  int expert = 0, row0 = mt * BM, row_end = M;
  if (offs != nullptr) {
    int before = 0;
    expert = -1;
    for (int e = 0; e < E; ++e) {
      const int lo = offs[e], hi = offs[e + 1];
      const int nt_e = (hi - lo + BM - 1) / BM;
      if (mt < before + nt_e) {
        expert = e;
        row0 = lo + (mt - before) * BM;
        row_end = hi;
        break;
      }
      before += nt_e;
    }
    if (expert < 0) return;  // tile beyond the routed rows (uniform across the CTA)
  } else if (row0 >= M) {
    return;
  }
  const int n0 = nt * BN;
  const int num_kb = K / BK;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + CF::kStages * CF::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CF::kStages * CF::kStageBytes);
  uint64_t* empty = full + CF::kStages;
  uint64_t* tmem_full = empty + CF::kStages;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < CF::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(CF::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % CF::kStages;
        const uint32_t ph = (kb / CF::kStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], CF::kStageBytes);
        tma_load_2d(sA + s * CF::kABytes, &tmA, &full[s], kb * BK, row0);
        tma_load_3d(sB + s * CF::kBBytes, &tmB, &full[s], kb * BK, n0, expert);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer (single thread) =====
      constexpr uint32_t idesc = instr_desc_bf16<BN>();
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % CF::kStages;
        const uint32_t ph = (kb / CF::kStages) & 1;
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a0 = smem_u32(sA + s * CF::kABytes);
        const uint32_t b0 = smem_u32(sB + s * CF::kBBytes);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
          // advance 16 bf16 = 32 B along K inside the 128-B swizzle atom
          umma_bf16(tmem_base, umma_desc_sw128(a0 + kk * 32), umma_desc_sw128(b0 + kk * 32), idesc,
                    (kb | kk) != 0);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(tmem_full);
    }
  } else {
    // ===== epilogue: TMEM → registers → global =====
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int quarter = warp & 3;  // tcgen05.ld lane window of this warp
    const int row = quarter * 32 + lane;
    const int grow = row0 + row;
    const bool valid = grow < row_end && grow < M;
    const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16);
    epilogue_tile<BN, EPI>(tbase, valid, grow, n0, N, C, ldc, aux);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(CF::kTmemCols));
  }
}

// ---- 2-CTA variant: one 256×256 tile per CTA pair (cta_group::2) --------------
//
// The pair shares the operands of one M=256 × N=256 UMMA: CTA r of the pair
// loads A rows [m0+128r, +128) and B rows [n0+128r, +128) into its own smem,
// the leader (rank 0) issues tcgen05.mma.cta_group::2 that reads both CTAs'
// halves, and each CTA's TMEM receives its 128 accumulator rows × 256 columns.
// Per SM per k-block that is 32 KB of operand traffic instead of the 48 KB of
// the 1-CTA 128×256 tile (whose L2 operand stream, not the tensor pipe, caps
// it near 1 PFLOP/s).  Barrier protocol (as CUTLASS's PipelineTmaUmmaAsync):
//   full[s]   leader's barrier only; armed once per phase by the leader with
//             both halves' bytes; both CTAs' TMAs complete_tx on it (peer bit
//             of the barrier address cleared);
//   empty[s]  per CTA; the leader's tcgen05.commit multicasts to both;
//   tmem_full per CTA; multicast commit after the last k-block.


__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0, int c1,
                                                 int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(leader_bar)
      : "memory");
}

__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

struct Cfg2 {
  static constexpr int kStages = 6;
  static constexpr int kABytes = 128 * BK * 2;  // this CTA's half of A
  static constexpr int kBBytes = 128 * BK * 2;  // this CTA's half of B (N = 256 per pair)
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 256;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * kStageBytes + 256;
};

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const int32_t* __restrict__ offs, int E, int M, int N, int K, void* __restrict__ C, int ldc,
                    const void* __restrict__ aux, int m_tiles, int n_tiles) {
  using CF = Cfg2;
  constexpr int BN = 256;
  const uint32_t rank = cluster_rank();
  int pt, nt;  // 256-row pair tile, n tile (both CTAs of the cluster decode the same pair)
  raster_tile(blockIdx.x >> 1, m_tiles, n_tiles, pt, nt);
  int expert = 0, prow0 = pt * 256, row_end = M;
  if (offs != nullptr) {
    int before = 0;
    expert = -1;
    for (int e = 0; e < E; ++e) {
      const int lo = offs[e], hi = offs[e + 1];
      const int nt_e = (hi - lo + 255) / 256;
      if (pt < before + nt_e) {
        expert = e;
        prow0 = lo + (pt - before) * 256;
        row_end = hi;
        break;
      }
      before += nt_e;
    }
    if (expert < 0) return;  // both CTAs of the pair see the same offsets → exit together
  } else if (prow0 >= M) {
    return;
  }
  const int row0 = prow0 + (int)rank * 128;
  const int n0 = nt * BN;
  const int num_kb = K / BK;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + CF::kStages * CF::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CF::kStages * CF::kStageBytes);
  uint64_t* empty = full + CF::kStages;
  uint64_t* tmem_full = empty + CF::kStages;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < CF::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(CF::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated in both
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs: each loads its halves) =====
      const uint32_t leader_full0 = smem_u32(&full[0]) & 0xFEFFFFFFu;
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % CF::kStages;
        const uint32_t ph = (kb / CF::kStages) & 1;
        mbar_wait_guard(&empty[s], ph ^ 1);
        if (rank == 0) mbar_expect_tx(&full[s], 2 * CF::kStageBytes);
        const uint32_t bar = leader_full0 + s * 8;
        tma_load_2d_pair(sA + s * CF::kABytes, &tmA, bar, kb * BK, row0);
        tma_load_3d_pair(sB + s * CF::kBBytes, &tmB, bar, kb * BK, n0 + (int)rank * 128, expert);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ===== MMA issuer (leader CTA only) =====
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                 ((uint32_t)(256 >> 4) << 24);
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % CF::kStages;
        const uint32_t ph = (kb / CF::kStages) & 1;
        mbar_wait_guard(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a0 = smem_u32(sA + s * CF::kABytes);
        const uint32_t b0 = smem_u32(sB + s * CF::kBBytes);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)
          umma_bf16_pair(tmem_base, umma_desc_sw128(a0 + kk * 32), umma_desc_sw128(b0 + kk * 32), idesc,
                         (kb | kk) != 0);
        umma_commit_pair(&empty[s]);
      }
      umma_commit_pair(tmem_full);
    }
  } else {
    // ===== epilogue (both CTAs, own 128 rows) =====
    mbar_wait_guard(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int grow = row0 + row;
    const bool valid = grow < row_end && grow < M;
    const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16);
    epilogue_tile<BN, EPI>(tbase, valid, grow, n0, N, C, ldc, aux);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  cluster_sync();  // the peer's TMEM is done with before the pair frees it
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(CF::kTmemCols));
  }
}

// ---- persistent variants: double-buffered TMEM accumulator --------------------
//
// One CTA (cta_group::1) or CTA pair (cta_group::2) per SM (pair), looping over
// a static round-robin tile schedule.  The accumulator is double-buffered in
// TMEM (2 × BN columns), so the epilogue of tile i (TMEM → registers → global)
// runs while the tensor pipe accumulates tile i+1, and the prologue (barrier
// init, TMEM alloc, descriptor prefetch, pipeline fill) is paid once per CTA
// instead of once per tile.  Pipelines:
//   smem ring   full[s] / empty[s]        TMA producer  ↔ MMA issuer
//   accumulator tmem_full[b] / tmem_empty[b]  MMA issuer ↔ epilogue warps
// In pair mode tmem_empty lives in the leader and counts the epilogue warps
// of both CTAs (the peer arrives remotely through its cluster address).

template <int CG, int BN>
struct CfgP {
  static constexpr int kABytes = 128 * BK * 2;                          // this CTA's A rows per stage
  static constexpr int kBBytes = (CG == 2 ? BN / 2 : BN) * BK * 2;      // this CTA's B rows per stage
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (196 * 1024) / kStageBytes;            // 6 × 32 KB or 4 × 48 KB
  static constexpr int kTmemCols = 2 * BN;                              // two fp32 accumulators
  static constexpr size_t kSmem = 1024 + (size_t)kStages * kStageBytes + 256;
};

struct TileInfo {
  int expert, row0, row_end, n0;
  int ks, kb0, kb1;  // split-K slice of this tile (k-blocks [kb0, kb1))
  bool valid;
};

// tile t → rows/expert/columns (tileM = output rows of one tile: 128, or 256 for a
// pair); with k_split > 1, consecutive tiles are the K slices of one output tile
__device__ __forceinline__ TileInfo tile_info(int t, const int32_t* __restrict__ offs, int E, int M, int m_tiles,
                                              int n_tiles, int tileM, int BNc, int k_split = 1, int num_kb = 0) {
  int mt, nt;
  TileInfo ti;
  ti.ks = t % k_split;
  t /= k_split;
  const int kbs = (num_kb + k_split - 1) / k_split;
  ti.kb0 = ti.ks * kbs;
  ti.kb1 = min(num_kb, ti.kb0 + kbs);
  ti.expert = 0;
  ti.row_end = M;
  if (offs == nullptr) {
    raster_tile(t, m_tiles, n_tiles, mt, nt);
    ti.row0 = mt * tileM;
    ti.n0 = nt * BNc;
    ti.valid = ti.row0 < M;
    return ti;
  }
  // grouped: the raster runs expert by expert (bands of ≤ 16 of the expert's own
  // m-tiles), so an expert's weight tiles are read once by every m-tile that needs
  // them instead of once per band the expert straddles (a global band raster read
  // 2.07× the weight bytes at bs 472: profiles/ncu_gemm_persistent_r1.md)
  ti.valid = false;
  ti.row0 = M;
  ti.n0 = 0;
  int base = 0;
  for (int e = 0; e < E; ++e) {
    const int lo = offs[e], hi = offs[e + 1];
    const int nt_e = (hi - lo + tileM - 1) / tileM;
    const int span = nt_e * n_tiles;
    if (t < base + span) {
      raster_tile(t - base, nt_e, n_tiles, mt, nt);
      ti.expert = e;
      ti.row0 = lo + mt * tileM;
      ti.row_end = hi;
      ti.n0 = nt * BNc;
      ti.valid = true;
      break;
    }
    base += span;
  }
  return ti;
}

// EPI == SO_EPI_PARTIAL: split-K slice — the fp32 accumulator goes to
// partial[ks][row][col]; splitk_reduce_kernel sums the slices and applies the
// real epilogue.  Used for skinny GEMMs (draft decode steps, M ≤ 128) whose
// few output tiles would otherwise stream the weights through a few SMs.
constexpr int SO_EPI_PARTIAL = 100;

template <int CG, int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tcp_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const int32_t* __restrict__ offs, int E, int M, int N, int K, void* __restrict__ C, int ldc,
                    const void* __restrict__ aux, int m_tiles, int n_tiles, int k_split) {
  using CF = CfgP<CG, BN>;
  constexpr int kTileM = 128 * CG;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  const int unit = CG == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int units = CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int total = m_tiles * n_tiles * k_split;
  const int num_kb = K / BK;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + CF::kStages * CF::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CF::kStages * CF::kStageBytes);
  uint64_t* empty = full + CF::kStages;
  uint64_t* tmem_full = empty + CF::kStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < CF::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 4 * CG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "r"(CF::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "r"(CF::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (CG == 2) cluster_sync();
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      const uint32_t leader_full0 = smem_u32(&full[0]) & 0xFEFFFFFFu;
      uint32_t it = 0;
      for (int t = unit; t < total; t += units) {
        const TileInfo ti = tile_info(t, offs, E, M, m_tiles, n_tiles, kTileM, BN, k_split, num_kb);
        if (!ti.valid) continue;
        const int rowA = ti.row0 + (int)rank * 128;
        const int rowB = ti.n0 + (CG == 2 ? (int)rank * (BN / 2) : 0);
        for (int kb = ti.kb0; kb < ti.kb1; ++kb, ++it) {
          const int s = it % CF::kStages;
          const uint32_t ph = (it / CF::kStages) & 1;
          mbar_wait_guard(&empty[s], ph ^ 1);
          if constexpr (CG == 2) {
            if (rank == 0) mbar_expect_tx(&full[s], 2 * CF::kStageBytes);
            const uint32_t bar = leader_full0 + s * 8;
            tma_load_2d_pair(sA + s * CF::kABytes, &tmA, bar, kb * BK, rowA);
            tma_load_3d_pair(sB + s * CF::kBBytes, &tmB, bar, kb * BK, rowB, ti.expert);
          } else {
            mbar_expect_tx(&full[s], CF::kStageBytes);
            tma_load_2d(sA + s * CF::kABytes, &tmA, &full[s], kb * BK, rowA);
            tma_load_3d(sB + s * CF::kBBytes, &tmB, &full[s], kb * BK, rowB, ti.expert);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ===== MMA issuer (single thread; the leader CTA in pair mode) =====
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                 ((uint32_t)(kTileM >> 4) << 24);
      uint32_t it = 0, acc = 0;
      for (int t = unit; t < total; t += units) {
        const TileInfo ti = tile_info(t, offs, E, M, m_tiles, n_tiles, kTileM, BN, k_split, num_kb);
        if (!ti.valid) continue;
        const uint32_t buf = acc & 1, aph = (acc >> 1) & 1;
        mbar_wait_guard(&tmem_empty[buf], aph ^ 1);  // the epilogue drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem_base + buf * BN;
        for (int kb = ti.kb0; kb < ti.kb1; ++kb, ++it) {
          const int s = it % CF::kStages;
          const uint32_t ph = (it / CF::kStages) & 1;
          mbar_wait_guard(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a0 = smem_u32(sA + s * CF::kABytes);
          const uint32_t b0 = smem_u32(sB + s * CF::kBBytes);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint32_t accum = (kb != ti.kb0) | (kk != 0);
            if constexpr (CG == 2)
              umma_bf16_pair(d, umma_desc_sw128(a0 + kk * 32), umma_desc_sw128(b0 + kk * 32), idesc, accum);
            else
              umma_bf16(d, umma_desc_sw128(a0 + kk * 32), umma_desc_sw128(b0 + kk * 32), idesc, accum);
          }
          if constexpr (CG == 2) umma_commit_pair(&empty[s]);
          else umma_commit(&empty[s]);
        }
        if constexpr (CG == 2) umma_commit_pair(&tmem_full[buf]);
        else umma_commit(&tmem_full[buf]);
        ++acc;
      }
    }
  } else {
    // ===== epilogue warps: TMEM → registers → global, then release the accumulator =====
    const int quarter = warp & 3;  // tcgen05.ld lane window of this warp
    const int row = quarter * 32 + lane;
    uint32_t acc = 0;
    uint32_t empty0 = smem_u32(&tmem_empty[0]), empty1 = smem_u32(&tmem_empty[1]);
    if constexpr (CG == 2) {  // the leader's barriers
      asm volatile("mapa.shared::cluster.u32 %0, %0, 0;" : "+r"(empty0));
      asm volatile("mapa.shared::cluster.u32 %0, %0, 0;" : "+r"(empty1));
    }
    for (int t = unit; t < total; t += units) {
      const TileInfo ti = tile_info(t, offs, E, M, m_tiles, n_tiles, kTileM, BN, k_split, num_kb);
      if (!ti.valid) continue;
      const uint32_t buf = acc & 1, aph = (acc >> 1) & 1;
      mbar_wait_guard(&tmem_full[buf], aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int grow = ti.row0 + (int)rank * 128 + row;
      const bool valid = grow < ti.row_end && grow < M;
      const uint32_t tbase = tmem_base + buf * BN + ((uint32_t)(quarter * 32) << 16);
      if constexpr (EPI == SO_EPI_PARTIAL)
        epilogue_tile<BN, SO_EPI_F32>(tbase, valid, grow, ti.n0, N,
                                      reinterpret_cast<float*>(C) + (size_t)ti.ks * M * N, N, nullptr);
      else
        epilogue_tile<BN, EPI>(tbase, valid, grow, ti.n0, N, C, ldc, aux);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(buf ? empty1 : empty0)
                       : "memory");
        else
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(buf ? empty1 : empty0) : "memory");
      }
      ++acc;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (CG == 2) cluster_sync();  // the peer's TMEM is done with before the pair frees it
  else __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(CF::kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(CF::kTmemCols));
  }
}

// Split-K finish: out = EPI(Σ_ks partial[ks]) with the same arithmetic as the
// fused epilogues (bf16 rounding before the residual add, SwiGLU on the 64-row
// interleaved gate/up column blocks).  One thread per 8 output columns.
template <int EPI>
__global__ void splitk_reduce_kernel(const float* __restrict__ partial, int k_split, int M, int N, void* __restrict__ C,
                                     int ldc, const void* __restrict__ aux) {
  const int out_cols = EPI == SO_EPI_SWIGLU ? N / 2 : N;
  const int groups = out_cols / 8;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= M * groups) return;
  const int row = idx / groups, c0 = (idx % groups) * 8;
  float f[8];
  if constexpr (EPI == SO_EPI_SWIGLU) {
    // output column c ↔ gate column 128·(c/64) + c%64, up column +64
    const int gcol = 128 * (c0 / 64) + c0 % 64;
    float g[8], u[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) g[j] = u[j] = 0.0f;
    for (int ks = 0; ks < k_split; ++ks) {
      const float* pr = partial + ((size_t)ks * M + row) * N;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        g[j] += pr[gcol + j];
        u[j] += pr[gcol + 64 + j];
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = silu(g[j]) * u[j];
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = 0.0f;
    for (int ks = 0; ks < k_split; ++ks) {
      const float4* pr = reinterpret_cast<const float4*>(partial + ((size_t)ks * M + row) * N + c0);
      const float4 a = pr[0], b = pr[1];
      f[0] += a.x, f[1] += a.y, f[2] += a.z, f[3] += a.w, f[4] += b.x, f[5] += b.y, f[6] += b.z, f[7] += b.w;
    }
  }
  if constexpr (EPI == SO_EPI_F32) {
    float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(C) + (size_t)row * ldc + c0);
    dst[0] = make_float4(f[0], f[1], f[2], f[3]);
    dst[1] = make_float4(f[4], f[5], f[6], f[7]);
    return;
  }
  if constexpr (EPI == SO_EPI_BF16_RESID) {
    float rr[8];
    unpack8(*reinterpret_cast<const int4*>(reinterpret_cast<const __nv_bfloat16*>(aux) + (size_t)row * ldc + c0), rr);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = __bfloat162float(__float2bfloat16_rn(f[j])) + rr[j];
  } else if constexpr (EPI == SO_EPI_BF16_ROWSCALE) {
    const float w = reinterpret_cast<const float*>(aux)[row];
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] *= w;
  }
  *reinterpret_cast<int4*>(reinterpret_cast<__nv_bfloat16*>(C) + (size_t)row * ldc + c0) = pack8(f);
}

// ---- host side ---------------------------------------------------------------


int sm_count() { return device_sm_count(); }

template <int BN, int EPI>
int launch_bn(const CUtensorMap& ma, const CUtensorMap& mb, const int32_t* offs, int E, int m_tiles, int M,
              int N, int K, void* C, int ldc, const void* aux, cudaStream_t st) {
  using CF = Cfg<BN>;
  auto kern = gemm_tc_kernel<BN, EPI>;
  if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), CF::kSmem)) return rc;
  const int n_tiles = (N + BN - 1) / BN;
  kern<<<m_tiles * n_tiles, kThreads, CF::kSmem, st>>>(ma, mb, offs, E, M, N, K, C, ldc, aux, m_tiles, n_tiles);
  SO_CHECK_LAUNCH();
  return SO_OK;
}

// Tile variant, an explicit argument of every launch (no process state):
// 0 = auto, 1 = 1-CTA tiles only, 2 = CTA-pair tiles where legal, 3 = one tile per CTA

// persistent launch: one CTA (pair) per SM (pair), never more than the tiles
template <int CG, int BN, int EPI>
int launch_persistent(const CUtensorMap& ma, const CUtensorMap& mb, const int32_t* offs, int E, int m_tiles,
                      int M, int N, int K, void* C, int ldc, const void* aux, cudaStream_t st, int k_split = 1) {
  using CF = CfgP<CG, BN>;
  auto kern = gemm_tcp_kernel<CG, BN, EPI>;
  if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), CF::kSmem)) return rc;
  const int n_tiles = (N + BN - 1) / BN;
  const int tiles = m_tiles * n_tiles * k_split;
  int units = sm_count() / CG;
  if (units > tiles) units = tiles;
  if (units < 1) units = 1;
  if constexpr (CG == 2) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * units);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = CF::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, offs, E, M, N, K, C, ldc, aux, m_tiles, n_tiles, k_split);
    if (e != cudaSuccess) return (int)e;
  } else {
    kern<<<units, kThreads, CF::kSmem, st>>>(ma, mb, offs, E, M, N, K, C, ldc, aux, m_tiles, n_tiles, k_split);
  }
  SO_CHECK_LAUNCH();
  return SO_OK;
}

template <int EPI>
int launch_pair(const void* A, const void* B, const int32_t* offs, int E, int M, int N, int K, void* C, int ldc,
                const void* aux, int variant, cudaStream_t st) {
  CUtensorMap ma, mb;
  int rc = make_map_2d(&ma, A, (uint64_t)M, (uint64_t)K, 128);
  if (rc) return rc;
  rc = make_map_3d(&mb, B, (uint64_t)E, (uint64_t)N, (uint64_t)K, 128);
  if (rc) return rc;
  const int pair_tiles = offs ? (M + 255) / 256 + E : (M + 255) / 256;
  if (variant != 3) return launch_persistent<2, 256, EPI>(ma, mb, offs, E, pair_tiles, M, N, K, C, ldc, aux, st);
  auto kern = gemm_tc2_kernel<EPI>;
  if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), Cfg2::kSmem)) return rc;
  const int n_tiles = N / 256;
  kern<<<2 * pair_tiles * n_tiles, kThreads, Cfg2::kSmem, st>>>(ma, mb, offs, E, M, N, K, C, ldc, aux, pair_tiles,
                                                                 n_tiles);
  SO_CHECK_LAUNCH();
  return SO_OK;
}

template <int EPI>
int launch_epi(const void* A, const void* B, const int32_t* offs, int E, int M, int N, int K, void* C, int ldc,
               const void* aux, int variant, cudaStream_t st) {
  // CTA-pair 256×256 tiles cut the per-SM operand stream by a third; 1-CTA
  // 128-row tiles pad less when M is small or split into experts (~560 rows
  // each at bs 248: measured 0.58 vs 0.51 of peak, profiles/gemm_bench_r1.json).
  const bool pair_ok = (N % 256) == 0;
  if (pair_ok && (variant == 2 || ((variant == 0 || variant == 3) && offs == nullptr && M >= 1024)))
    return launch_pair<EPI>(A, B, offs, E, M, N, K, C, ldc, aux, variant, st);
  const int m_tiles = offs ? (M + BM - 1) / BM + E : (M + BM - 1) / BM;
  // prefer the wide tile unless it leaves most SMs idle
  bool wide = (long)m_tiles * ((N + 255) / 256) >= sm_count() || EPI == SO_EPI_SWIGLU && (N % 256) == 0;
  if (EPI == SO_EPI_SWIGLU && (N % 256) != 0) wide = false;
  CUtensorMap ma, mb;
  int rc = make_map_2d(&ma, A, (uint64_t)M, (uint64_t)K, BM);
  if (rc) return rc;
  if (wide) {
    rc = make_map_3d(&mb, B, (uint64_t)E, (uint64_t)N, (uint64_t)K, 256);
    if (rc) return rc;
    if (variant != 3) return launch_persistent<1, 256, EPI>(ma, mb, offs, E, m_tiles, M, N, K, C, ldc, aux, st);
    return launch_bn<256, EPI>(ma, mb, offs, E, m_tiles, M, N, K, C, ldc, aux, st);
  }
  rc = make_map_3d(&mb, B, (uint64_t)E, (uint64_t)N, (uint64_t)K, 128);
  if (rc) return rc;
  if (variant != 3) return launch_persistent<1, 128, EPI>(ma, mb, offs, E, m_tiles, M, N, K, C, ldc, aux, st);
  return launch_bn<128, EPI>(ma, mb, offs, E, m_tiles, M, N, K, C, ldc, aux, st);
}

int gemm_dispatch(const void* A, const void* B, const int32_t* offs, int E, int M, int N, int K, void* C,
                  int ldc, int epi, const void* aux, int variant, cudaStream_t st) {
  SO_REQUIRE(A && B && C, SO_E_NULLPTR);
  SO_REQUIRE(M >= 0 && N > 0 && K > 0 && E >= 1, SO_E_SHAPE);
  SO_REQUIRE(K % BK == 0 && N % 32 == 0, SO_E_SHAPE);
  SO_REQUIRE(aligned16(A) && aligned16(B) && aligned16(C), SO_E_ALIGN);
  if (epi == SO_EPI_SWIGLU) SO_REQUIRE(N % 128 == 0 && ldc % 8 == 0 && ldc >= N / 2, SO_E_SHAPE);
  else if (epi == SO_EPI_F32) SO_REQUIRE(ldc % 4 == 0 && ldc >= N, SO_E_SHAPE);
  else SO_REQUIRE(ldc % 8 == 0 && ldc >= N, SO_E_SHAPE);
  if (epi == SO_EPI_BF16_RESID || epi == SO_EPI_BF16_ROWSCALE) SO_REQUIRE(aux != nullptr, SO_E_NULLPTR);
  SO_REQUIRE(variant >= 0 && variant <= 3, SO_E_SHAPE);
  if (M == 0) return SO_OK;
  switch (epi) {
    case SO_EPI_BF16: return launch_epi<SO_EPI_BF16>(A, B, offs, E, M, N, K, C, ldc, aux, variant, st);
    case SO_EPI_F32: return launch_epi<SO_EPI_F32>(A, B, offs, E, M, N, K, C, ldc, aux, variant, st);
    case SO_EPI_BF16_RESID: return launch_epi<SO_EPI_BF16_RESID>(A, B, offs, E, M, N, K, C, ldc, aux, variant, st);
    case SO_EPI_SWIGLU: return launch_epi<SO_EPI_SWIGLU>(A, B, offs, E, M, N, K, C, ldc, aux, variant, st);
    case SO_EPI_BF16_ROWSCALE:
      return launch_epi<SO_EPI_BF16_ROWSCALE>(A, B, offs, E, M, N, K, C, ldc, aux, variant, st);
    default: return SO_E_UNSUPPORTED;
  }
}

// Split-K choice for a dense GEMM with few output tiles (0 = not worth it)
int splitk_factor(int M, int N, int K, int variant = 0) {
  if (M > 256 || variant == 3) return 0;
  const int tiles = ((M + BM - 1) / BM) * ((N + 127) / 128);
  const int sms = sm_count();
  if (2 * tiles >= sms) return 0;
  const int num_kb = K / BK;
  int ks = (sms + tiles - 1) / tiles;
  if (ks > num_kb / 4) ks = num_kb / 4;  // ≥ 4 k-blocks per slice
  if (ks > 16) ks = 16;
  while (ks > 1) {  // no empty slice
    const int kbs = (num_kb + ks - 1) / ks;
    if ((ks - 1) * kbs < num_kb) break;
    --ks;
  }
  return ks >= 2 ? ks : 0;
}

template <int EPI>
int launch_splitk(const void* A, const void* B, int M, int N, int K, void* C, int ldc, const void* aux, int ks,
                  float* ws, cudaStream_t st) {
  CUtensorMap ma, mb;
  int rc = make_map_2d(&ma, A, (uint64_t)M, (uint64_t)K, BM);
  if (rc) return rc;
  rc = make_map_3d(&mb, B, 1, (uint64_t)N, (uint64_t)K, 128);
  if (rc) return rc;
  rc = launch_persistent<1, 128, SO_EPI_PARTIAL>(ma, mb, nullptr, 1, (M + BM - 1) / BM, M, N, K, ws, N, nullptr, st,
                                                ks);
  if (rc) return rc;
  const int out_cols = EPI == SO_EPI_SWIGLU ? N / 2 : N;
  const int threads = M * (out_cols / 8);
  splitk_reduce_kernel<EPI><<<(threads + 255) / 256, 256, 0, st>>>(ws, ks, M, N, C, ldc, aux);
  SO_CHECK_LAUNCH();
  return SO_OK;
}

}  // namespace

extern "C" size_t so_gemm_workspace_bytes(int M, int N, int K) {
  // split-K scratch; decode steps K5c serves (gemv_tc.cu) need none
  const int ks = (M > 0 && N > 0 && K >= BK) ? splitk_factor(M, N, K, 0) : 0;
  return ks ? (size_t)ks * M * N * sizeof(float) : 0;
}

extern "C" int so_gemm_bf16_v(const void* A, const void* B, const int32_t* expert_offsets, int E, int M, int N,
                              int K, void* C, int ldc, int epilogue, const void* aux, void* workspace, size_t ws_bytes,
                              int variant, void* stream) {
  cudaStream_t st = as_stream(stream);
  if (expert_offsets != nullptr) return gemm_dispatch(A, B, expert_offsets, E, M, N, K, C, ldc, epilogue, aux, variant, st);
  // decode steps (M ≤ 128 rows, fewer weight tiles than SMs): the K5c cluster split-K kernel
  // (no scratch), unless a tile variant is forced
  if ((variant == 0 || variant == 4) && epilogue != SO_EPI_BF16_ROWSCALE && so_gemv_workspace_bytes(M, N, K) > 0)
    return so_gemv_bf16(A, B, M, N, K, C, ldc, epilogue, aux, nullptr, 0, stream);
  if (variant == 4) variant = 0;  // not eligible: the automatic choice
  const int ks = (M > 0 && N > 0 && K >= BK && K % BK == 0 && N % 128 == 0) ? splitk_factor(M, N, K, variant) : 0;
  if (ks == 0 || workspace == nullptr || ws_bytes < (size_t)ks * M * N * sizeof(float))
    return gemm_dispatch(A, B, nullptr, 1, M, N, K, C, ldc, epilogue, aux, variant, st);
  SO_REQUIRE(A && B && C, SO_E_NULLPTR);
  SO_REQUIRE(aligned16(A) && aligned16(B) && aligned16(C) && aligned16(workspace), SO_E_ALIGN);
  if (epilogue == SO_EPI_SWIGLU) SO_REQUIRE(ldc % 8 == 0 && ldc >= N / 2, SO_E_SHAPE);
  else if (epilogue == SO_EPI_F32) SO_REQUIRE(ldc % 4 == 0 && ldc >= N, SO_E_SHAPE);
  else SO_REQUIRE(ldc % 8 == 0 && ldc >= N, SO_E_SHAPE);
  if (epilogue == SO_EPI_BF16_RESID || epilogue == SO_EPI_BF16_ROWSCALE) SO_REQUIRE(aux != nullptr, SO_E_NULLPTR);
  float* ws = reinterpret_cast<float*>(workspace);
  switch (epilogue) {
    case SO_EPI_BF16: return launch_splitk<SO_EPI_BF16>(A, B, M, N, K, C, ldc, aux, ks, ws, st);
    case SO_EPI_F32: return launch_splitk<SO_EPI_F32>(A, B, M, N, K, C, ldc, aux, ks, ws, st);
    case SO_EPI_BF16_RESID: return launch_splitk<SO_EPI_BF16_RESID>(A, B, M, N, K, C, ldc, aux, ks, ws, st);
    case SO_EPI_SWIGLU: return launch_splitk<SO_EPI_SWIGLU>(A, B, M, N, K, C, ldc, aux, ks, ws, st);
    case SO_EPI_BF16_ROWSCALE: return launch_splitk<SO_EPI_BF16_ROWSCALE>(A, B, M, N, K, C, ldc, aux, ks, ws, st);
    default: return SO_E_UNSUPPORTED;
  }
}

extern "C" int so_gemm_bf16_ex(const void* A, const void* B, int M, int N, int K, void* C, int ldc, int epilogue,
                               const void* aux, void* workspace, size_t ws_bytes, void* stream) {
  return so_gemm_bf16_v(A, B, nullptr, 1, M, N, K, C, ldc, epilogue, aux, workspace, ws_bytes, 0, stream);
}

extern "C" int so_gemm_bf16(const void* A, const void* B, int M, int N, int K, void* C, int ldc, int epilogue,
                            const void* aux, void* stream) {
  return gemm_dispatch(A, B, nullptr, 1, M, N, K, C, ldc, epilogue, aux, 0, as_stream(stream));
}

extern "C" int so_gemm_grouped_bf16(const void* A, const void* B, const int32_t* expert_offsets, int E,
                                    int max_rows, int N, int K, void* C, int ldc, int epilogue,
                                    const void* aux, void* stream) {
  SO_REQUIRE(expert_offsets != nullptr, SO_E_NULLPTR);
  return gemm_dispatch(A, B, expert_offsets, E, max_rows, N, K, C, ldc, epilogue, aux, 0, as_stream(stream));
}

extern "C" int so_device_sm_count(void) { return sm_count(); }

