// K6 — multi-token verification attention over the paged KV cache.
//
// In the paper this is the CPU attention the reference charges as
// `n_cand · bs · t_attn_cpu` per layer (costmodel.py:73, simulator.py:169-171,
// PAPER.md:157).  On B200 the target KV lives in HBM and the
// verify pass attends n_cand+1 new query positions per sequence over
// ctx + n_cand + 1 keys, causally inside the new block.  The same kernel serves
// prefill (q_len = prompt length).
//
// Work unit: one CTA (4 warps) per (sequence, kv-head, 64-row query tile).  The
// rows of a (sequence, kv-head) pair are all q_len positions × the G = hq/hkv
// query heads sharing that KV head (GQA), so each K/V tile read from HBM feeds
// every query head of the group.  K/V tiles of 32 keys are staged with 16-B
// cp.async into an XOR-swizzled, 4-stage smem ring (one page = one
// contiguous [page_size, dh] block per kv-head, so a tile is one coalesced
// 8–16 KB run); S = QKᵀ and O += PV run on bf16 mma.sync with fp32 accumulate;
// the softmax is the online (flash) form with quad-shuffle row reductions.
#include <cuda.h>

#include <cstring>
#include <mutex>

#include "common.cuh"

namespace {

constexpr int kRows = 64;   // query rows per CTA (4 warps × 16)
constexpr int kTcPrefillRows = 64;  // auto: calls with at least this many query positions per sequence go to K6c
constexpr int kKeys = 32;   // keys per smem tile
#ifndef SO_ATTN_STAGES
#define SO_ATTN_STAGES 4
#endif
constexpr int kStages = SO_ATTN_STAGES;  // cp.async ring depth (16 KB of K+V per stage at dh = 128)
constexpr int kThreads = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// src_bytes = 0 → the 16 smem bytes are zero-filled (rows past the valid keys)
__device__ __forceinline__ void cp_async16_zfill(void* dst, const void* src, bool valid) {
  const uint32_t n = valid ? 16u : 0u;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void mma_bf16(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Two ways to stage a K/V tile (the compute that follows is shared):
//   TMA = false  every thread issues 16-B cp.async copies (any page size),
//                tile rows XOR-swizzled in 256-B rows;
//   TMA = true   one thread issues 2-D TMA boxes of [min(page,32) rows × 64
//                columns] per page and half-row (SWIZZLE_128B), completion on
//                a per-stage mbarrier — the other 127 threads spend no issue
//                slots on address generation, which ncu showed as a third of
//                the instruction stream of this latency-bound kernel.
template <int DH, bool TMA>
struct Tile {
  static constexpr int kChunks = DH / 8;                 // 16-B chunks per key row
  static constexpr int kBytes = kKeys * DH * 2;          // one K or V tile
  // swizzled byte offset of (key row, chunk)
  __device__ __forceinline__ static uint32_t off(int row, int chunk) {
    if constexpr (TMA)  // [half][row][128 B], SWIZZLE_128B: chunk ^ (row mod 8) inside each 128-B row
      return (uint32_t)((chunk >> 3) * (kKeys * 128) + row * 128 + (((chunk & 7) ^ (row & 7)) << 4));
    else
      return (uint32_t)(row * DH * 2 + ((chunk ^ (row & 7)) << 4));
  }
};

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// bounded wait: a protocol bug traps (a reported kernel error) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0, spins = 0;
  const uint32_t a = smem_u32(bar);
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (++spins > (1u << 28)) __trap();
  } while (!done);
}

__device__ __forceinline__ void tma_box(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

#ifndef SO_ATTN_MINB
#define SO_ATTN_MINB 3  // CTAs per SM the register budget must allow (3 × 128 threads ≤ 170 regs)
#endif

template <int DH, bool TMA>
__global__ void __launch_bounds__(kThreads, SO_ATTN_MINB) attn_paged_kernel(
    const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ kc, const __nv_bfloat16* __restrict__ vc,
    const int32_t* __restrict__ block_table, int max_pages, const int32_t* __restrict__ q_start,
    const int32_t* __restrict__ kv_before, int hq, int hkv, int page_size, float scale_log2,
    __nv_bfloat16* __restrict__ out) {
  using TL = Tile<DH, TMA>;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // SWIZZLE_128B boxes land on 1024-B aligned stage buffers
  uint8_t* smem = TMA ? reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023))
                      : smem_raw;
  const int tile = blockIdx.x, g_kv = blockIdx.y, s = blockIdx.z;
  const int G = hq / hkv;
  const int qs = q_start[s];
  const int q_len = q_start[s + 1] - qs;
  const int rows_total = q_len * G;
  const int r0 = tile * kRows;
  if (r0 >= rows_total) return;
  const int kvb = kv_before[s];
  const int j_last = min(q_len - 1, (r0 + kRows - 1) / G);
  const int n_keys = kvb + j_last + 1;
  const int n_tiles = (n_keys + kKeys - 1) / kKeys;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;

  // ---- Q fragments (A operand, row-major [16 rows × DH]) ----
  // decode steps (≤ 16 query rows per CTA, cp.async staging): only warp 0 would hold live rows, so
  // every warp takes those rows and a different share of the KEY tiles ("warp split"), and the
  // warps' (m, l, O) merge through shared memory at the end
  const bool wsplit = !TMA && rows_total - r0 <= 16;
  const int rA = r0 + (wsplit ? 0 : warp * 16) + g, rB = rA + 8;
  const bool vA = rA < rows_total, vB = rB < rows_total;
  const int jA = vA ? rA / G : 0, jB = vB ? rB / G : 0;
  const int hA = g_kv * G + (vA ? rA % G : 0), hB = g_kv * G + (vB ? rB % G : 0);
  const __nv_bfloat16* qA = q + ((size_t)(qs + jA) * hq + hA) * DH;
  const __nv_bfloat16* qB = q + ((size_t)(qs + jB) * hq + hB) * DH;
  const bool warp_live = wsplit || (r0 + warp * 16) < rows_total;
  uint32_t qf[DH / 16][4];
#pragma unroll
  for (int ks = 0; ks < DH / 16; ++ks) {
    const int d0 = ks * 16 + 2 * c;
    qf[ks][0] = vA ? *reinterpret_cast<const uint32_t*>(qA + d0) : 0u;
    qf[ks][1] = vB ? *reinterpret_cast<const uint32_t*>(qB + d0) : 0u;
    qf[ks][2] = vA ? *reinterpret_cast<const uint32_t*>(qA + d0 + 8) : 0u;
    qf[ks][3] = vB ? *reinterpret_cast<const uint32_t*>(qB + d0 + 8) : 0u;
  }
  const int limA = vA ? kvb + jA : -1;  // last key this row may see
  const int limB = vB ? kvb + jB : -1;

  float o[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.0f;
  float mA = -INFINITY, mB = -INFINITY, lA = 0.0f, lB = 0.0f;

  // The sequence's page list is staged in smem once: every K/V row resolves its
  // page from it, so issuing a tile's copies never waits on a dependent
  // global load (which had cost one memory latency per tile step).
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * 2 * TL::kBytes);  // TMA stage barriers
  uint64_t* empty = full + kStages;  // TMA: every warp arrives once it has consumed the stage
  int32_t* bt = reinterpret_cast<int32_t*>(empty + kStages);
  const int used = min(max_pages, (n_keys + page_size - 1) / page_size);
  {
    const int32_t* gbt = block_table + (size_t)s * max_pages;
    for (int i = threadIdx.x; i < used; i += kThreads) bt[i] = gbt[i];
    if (TMA && threadIdx.x == 0) {
      for (int i = 0; i < kStages; ++i) {
        mbar_init(&full[i], 1);
        mbar_init(&empty[i], kThreads / 32);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmK)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmV)) : "memory");
    }
    __syncthreads();
  }
  // TMA: one thread puts tile kt's K and V boxes in flight on full[stage]
  const int box_rows = page_size < kKeys ? page_size : kKeys;
  auto issue_tile = [&](int kt, int buf) {
    const int key0 = kt * kKeys;
    uint8_t* sk = smem + buf * 2 * TL::kBytes;
    uint8_t* sv = sk + TL::kBytes;
    mbar_expect_tx(&full[buf], 2 * TL::kBytes);
    for (int r = 0; r < kKeys; r += box_rows) {
      const int key = key0 + r;
      const int pi = key / page_size;
      const int page = pi < used ? bt[pi] : bt[0];  // past the sequence: any valid page (masked / zeroed below)
      const int row = (page * hkv + g_kv) * page_size + key % page_size;
#pragma unroll
      for (int h = 0; h < DH / 64; ++h) {
        tma_box(sk + h * (kKeys * 128) + r * 128, &tmK, &full[buf], h * 64, row);
        tma_box(sv + h * (kKeys * 128) + r * 128, &tmV, &full[buf], h * 64, row);
      }
    }
  };
  // Each key row resolves its own page, so any page size works (a tile may
  // span several pages); rows at or past n_keys are zero-filled, keeping
  // 0·V finite for masked keys whatever the unwritten cache holds.
  auto load_tile = [&](int kt, int buf) {
    const int key0 = kt * kKeys;
    uint8_t* sk = smem + buf * 2 * TL::kBytes;
    uint8_t* sv = sk + TL::kBytes;
#pragma unroll
    for (int i = threadIdx.x; i < kKeys * TL::kChunks; i += kThreads) {
      const int row = i / TL::kChunks, ch = i % TL::kChunks;
      const int key = key0 + row;
      const bool valid = key < n_keys;
      const int kk = valid ? key : 0;
      const int page = bt[kk / page_size];
      const size_t src = (((size_t)page * hkv + g_kv) * page_size + (kk % page_size)) * DH + ch * 8;
      cp_async16_zfill(sk + TL::off(row, ch), kc + src, valid);
      cp_async16_zfill(sv + TL::off(row, ch), vc + src, valid);
    }
  };

  // one key tile from ring stage `stage`: S = Q·Kᵀ, masked online softmax, O += P·V (this warp's rows)
  auto compute_tile = [&](int kt, int stage) {
      const uint32_t sk = smem_u32(smem + stage * 2 * TL::kBytes);
      const uint32_t sv = sk + TL::kBytes;
      // ---- S = Q Kᵀ  (16 rows × kKeys keys per warp) ----
      float sfr[kKeys / 8][4];
#pragma unroll
      for (int nt = 0; nt < kKeys / 8; ++nt) sfr[nt][0] = sfr[nt][1] = sfr[nt][2] = sfr[nt][3] = 0.0f;
      const int mat = lane >> 3, mi = lane & 7;
#pragma unroll
      for (int ks = 0; ks < DH / 16; ++ks) {
#pragma unroll
        for (int nt = 0; nt < kKeys / 8; nt += 2) {
          const int key = (nt + (mat >> 1)) * 8 + mi;
          const int ch = ks * 2 + (mat & 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(sk + TL::off(key, ch), b0, b1, b2, b3);
          mma_bf16(sfr[nt], qf[ks], b0, b1);
          mma_bf16(sfr[nt + 1], qf[ks], b2, b3);
        }
      }
      // ---- mask + online softmax ----
      const int key0 = kt * kKeys;
      float tmA = -INFINITY, tmB = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < kKeys / 8; ++nt) {
        const int k0 = key0 + nt * 8 + 2 * c;
        sfr[nt][0] = k0 <= limA ? sfr[nt][0] * scale_log2 : -INFINITY;
        sfr[nt][1] = k0 + 1 <= limA ? sfr[nt][1] * scale_log2 : -INFINITY;
        sfr[nt][2] = k0 <= limB ? sfr[nt][2] * scale_log2 : -INFINITY;
        sfr[nt][3] = k0 + 1 <= limB ? sfr[nt][3] * scale_log2 : -INFINITY;
        tmA = fmaxf(tmA, fmaxf(sfr[nt][0], sfr[nt][1]));
        tmB = fmaxf(tmB, fmaxf(sfr[nt][2], sfr[nt][3]));
      }
      tmA = fmaxf(tmA, __shfl_xor_sync(0xffffffffu, tmA, 1));
      tmA = fmaxf(tmA, __shfl_xor_sync(0xffffffffu, tmA, 2));
      tmB = fmaxf(tmB, __shfl_xor_sync(0xffffffffu, tmB, 1));
      tmB = fmaxf(tmB, __shfl_xor_sync(0xffffffffu, tmB, 2));
      const float nmA = fmaxf(mA, tmA), nmB = fmaxf(mB, tmB);
      const float baseA = nmA == -INFINITY ? 0.0f : nmA;
      const float baseB = nmB == -INFINITY ? 0.0f : nmB;
      const float corrA = exp2f(mA - baseA), corrB = exp2f(mB - baseB);
      mA = nmA;
      mB = nmB;
      float rsA = 0.0f, rsB = 0.0f;
      uint32_t pf[kKeys / 16][4];
#pragma unroll
      for (int nt = 0; nt < kKeys / 8; ++nt) {
        const float p0 = exp2f(sfr[nt][0] - baseA), p1 = exp2f(sfr[nt][1] - baseA);
        const float p2 = exp2f(sfr[nt][2] - baseB), p3 = exp2f(sfr[nt][3] - baseB);
        rsA += p0 + p1;
        rsB += p2 + p3;
        // C-fragment → A-fragment of the PV product (k = keys)
        const int kk = nt >> 1;
        if ((nt & 1) == 0) {
          pf[kk][0] = pack_bf16(p0, p1);
          pf[kk][1] = pack_bf16(p2, p3);
        } else {
          pf[kk][2] = pack_bf16(p0, p1);
          pf[kk][3] = pack_bf16(p2, p3);
        }
      }
      lA = lA * corrA + rsA;
      lB = lB * corrB + rsB;
#pragma unroll
      for (int dn = 0; dn < DH / 8; ++dn) {
        o[dn][0] *= corrA;
        o[dn][1] *= corrA;
        o[dn][2] *= corrB;
        o[dn][3] *= corrB;
      }
      // ---- O += P V ----
#pragma unroll
      for (int kk = 0; kk < kKeys / 16; ++kk) {
#pragma unroll
        for (int dn = 0; dn < DH / 8; dn += 2) {
          const int key = kk * 16 + (mat & 1) * 8 + mi;
          const int ch = dn + (mat >> 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(sv + TL::off(key, ch), b0, b1, b2, b3);
          mma_bf16(o[dn], pf[kk], b0, b1);
          mma_bf16(o[dn + 1], pf[kk], b2, b3);
        }
      }
      };
  if (wsplit) {
    // rounds of kStages tiles, one per warp (kStages == warps): all loads of a round in flight together
    static_assert(kStages == kThreads / 32, "warp split: one ring stage per warp");
    for (int kt0 = 0; kt0 < n_tiles; kt0 += kStages) {
#pragma unroll
      for (int w = 0; w < kStages; ++w)
        if (kt0 + w < n_tiles) load_tile(kt0 + w, w);
      cp_commit();
      cp_wait<0>();
      __syncthreads();
      if (kt0 + warp < n_tiles) compute_tile(kt0 + warp, warp);
      __syncthreads();
    }
    // merge: every warp's rows g, g+8 (row sums reduced over the quad first) through shared memory
    lA += __shfl_xor_sync(0xffffffffu, lA, 1);
    lA += __shfl_xor_sync(0xffffffffu, lA, 2);
    lB += __shfl_xor_sync(0xffffffffu, lB, 1);
    lB += __shfl_xor_sync(0xffffffffu, lB, 2);
    float* sm = reinterpret_cast<float*>(smem);                // [warp][16] row maxima
    float* sl = sm + kStages * 16;                             // [warp][16] row sums
    float* so = sl + kStages * 16;                             // [warp][16][DH] unnormalised O
    if (c == 0) {
      sm[warp * 16 + g] = mA;
      sm[warp * 16 + g + 8] = mB;
      sl[warp * 16 + g] = lA;
      sl[warp * 16 + g + 8] = lB;
    }
#pragma unroll
    for (int dn = 0; dn < DH / 8; ++dn) {
      const int d = dn * 8 + 2 * c;
      so[(warp * 16 + g) * DH + d] = o[dn][0];
      so[(warp * 16 + g) * DH + d + 1] = o[dn][1];
      so[(warp * 16 + g + 8) * DH + d] = o[dn][2];
      so[(warp * 16 + g + 8) * DH + d + 1] = o[dn][3];
    }
    __syncthreads();
    const int rows = rows_total - r0;
    for (int i = threadIdx.x; i < rows * DH; i += kThreads) {
      const int r = i / DH, d = i % DH;
      float M = -INFINITY;
      for (int w = 0; w < kStages; ++w) M = fmaxf(M, sm[w * 16 + r]);
      float L = 0.f, O = 0.f;
      for (int w = 0; w < kStages; ++w) {
        if (sm[w * 16 + r] == -INFINITY) continue;  // a warp that saw no key of this row
        const float f = exp2f(sm[w * 16 + r] - M);
        L += sl[w * 16 + r] * f;
        O += so[(w * 16 + r) * DH + d] * f;
      }
      const int row = r0 + r, j = row / G, hh = g_kv * G + row % G;
      out[((size_t)(qs + j) * hq + hh) * DH + d] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
    }
    return;
  }
  // kStages-deep ring: kStages−1 tiles stream from HBM while one is consumed
  // (cp.async: one commit group per tile, empty groups past the end keep the
  // wait_group arithmetic uniform; TMA: one mbarrier phase per tile and stage)
  if constexpr (TMA) {
    if (threadIdx.x == 0)
      for (int p = 0; p < kStages - 1 && p < n_tiles; ++p) issue_tile(p, p);
  } else {
#pragma unroll
    for (int p = 0; p < kStages - 1; ++p) {
      if (p < n_tiles) load_tile(p, p);
      cp_commit();
    }
  }
  for (int kt = 0; kt < n_tiles; ++kt) {
    const int nxt = kt + kStages - 1;
    if constexpr (TMA) {
      // the stage of tile nxt held tile kt−1: refill it once every warp is done
      // with that tile — warps otherwise run up to kStages−1 tiles apart, no
      // CTA-wide barrier per tile
      if (threadIdx.x == 0 && nxt < n_tiles) {
        if (kt >= 1) mbar_wait(&empty[(kt - 1) % kStages], ((kt - 1) / kStages) & 1);
        issue_tile(nxt, nxt % kStages);
      }
      mbar_wait(&full[kt % kStages], (kt / kStages) & 1);
      const int valid = n_keys - kt * kKeys;
      if (valid < kKeys) {  // last tile: V rows past the keys hold stale data (0·NaN must not reach O)
        uint8_t* sv = smem + (kt % kStages) * 2 * TL::kBytes + TL::kBytes;
        for (int i = threadIdx.x; i < (kKeys - valid) * (DH / 64) * 8; i += kThreads) {
          const int row = valid + i / ((DH / 64) * 8), rest = i % ((DH / 64) * 8);
          *reinterpret_cast<int4*>(sv + (rest >> 3) * (kKeys * 128) + row * 128 + ((rest & 7) << 4)) =
              make_int4(0, 0, 0, 0);
        }
        __syncthreads();
      }
    } else {
      if (nxt < n_tiles) load_tile(nxt, nxt % kStages);
      cp_commit();
      cp_wait<kStages - 1>();
      __syncthreads();
    }
    if (warp_live) compute_tile(kt, kt % kStages);
    if constexpr (TMA) {
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[kt % kStages])) : "memory");
    } else {
      __syncthreads();
    }
  }
  if constexpr (!TMA) cp_wait<0>();
  if (!warp_live) return;
  // ---- normalise and store ----
  lA += __shfl_xor_sync(0xffffffffu, lA, 1);
  lA += __shfl_xor_sync(0xffffffffu, lA, 2);
  lB += __shfl_xor_sync(0xffffffffu, lB, 1);
  lB += __shfl_xor_sync(0xffffffffu, lB, 2);
  const float invA = lA > 0.0f ? 1.0f / lA : 0.0f;
  const float invB = lB > 0.0f ? 1.0f / lB : 0.0f;
  __nv_bfloat16* oA = out + ((size_t)(qs + jA) * hq + hA) * DH;
  __nv_bfloat16* oB = out + ((size_t)(qs + jB) * hq + hB) * DH;
#pragma unroll
  for (int dn = 0; dn < DH / 8; ++dn) {
    const int d = dn * 8 + 2 * c;
    if (vA) *reinterpret_cast<uint32_t*>(oA + d) = pack_bf16(o[dn][0] * invA, o[dn][1] * invA);
    if (vB) *reinterpret_cast<uint32_t*>(oB + d) = pack_bf16(o[dn][2] * invB, o[dn][3] * invB);
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn lookup_encode() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult qr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
      qr == cudaDriverEntryPointSuccess)
    return reinterpret_cast<EncodeTiledFn>(p);
  return nullptr;
}

// thread-safe one-time lookup (the verify and draft streams are fed from two host threads)
EncodeTiledFn get_encode() {
  static const EncodeTiledFn fn = lookup_encode();
  return fn;
}

// The cache of one layer as a 2-D tensor [rows = page·hkv·page_size + slot, dh]; every coordinate the kernel
// issues names a page of the block table, so the row extent only bounds the map.
int cache_map(CUtensorMap* m, const void* base, int dh, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return SO_E_DRIVER;
  cuuint64_t dims[2] = {(cuuint64_t)dh, (cuuint64_t)1 << 31};
  cuuint64_t strides[1] = {(cuuint64_t)dh * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? SO_OK : SO_E_DRIVER;
}

template <int DH, bool TMA>
int launch(const void* q, const void* k, const void* v, const int32_t* bt, int max_pages, const int32_t* q_start,
           const int32_t* kv_before, int bs, int max_q, int hq, int hkv, int page_size, float scale, void* out,
           cudaStream_t st) {
  const int G = hq / hkv;
  const int tiles = (max_q * G + kRows - 1) / kRows;
  const size_t smem = (TMA ? 1024 : 0) + (size_t)kStages * 2 * Tile<DH, TMA>::kBytes + 2 * kStages * sizeof(uint64_t) +
                      (size_t)max_pages * sizeof(int32_t);
  auto kern = attn_paged_kernel<DH, TMA>;
  // raised when a longer block table needs more smem (per kernel and device, under a lock:
  // the verify and the draft streams launch from two host threads); carveout 100 = all of
  // L1/smem as shared memory, 3 × 64 KB tiles per SM
  if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem, 100)) return rc;
  CUtensorMap mk, mv;
  memset(&mk, 0, sizeof(mk));
  memset(&mv, 0, sizeof(mv));
  if (TMA) {
    const int box_rows = page_size < kKeys ? page_size : kKeys;
    int rc = cache_map(&mk, k, DH, box_rows);
    if (rc) return rc;
    rc = cache_map(&mv, v, DH, box_rows);
    if (rc) return rc;
  }
  dim3 grid(tiles, hkv, bs);
  kern<<<grid, kThreads, smem, st>>>(mk, mv, reinterpret_cast<const __nv_bfloat16*>(q),
                                     reinterpret_cast<const __nv_bfloat16*>(k),
                                     reinterpret_cast<const __nv_bfloat16*>(v), bt, max_pages, q_start, kv_before, hq,
                                     hkv, page_size, scale * 1.4426950408889634f,
                                     reinterpret_cast<__nv_bfloat16*>(out));
  SO_CHECK_LAUNCH();
  return SO_OK;
}

// K6d — decode-step attention (one query position per sequence: the draft's n_cand decode steps,
// costmodel.py:53-57).  The G query heads of a kv head share one pass over its keys; the work is
// the K/V bytes, so the kernel is a streaming reduction on the CUDA cores rather than a tensor-core
// tile with G of 64 rows live:
//   CTA = (sequence, kv head), 8 warps; warp w takes 32-key chunks w, w+8, …;
//   scores: lane = key — the lane's 256-B K row in 16-B loads, G dot products against the queries
//           in shared memory (broadcast reads), online softmax per head with warp reductions;
//   P·V:    the chunk's V rows are staged into the warp's shared memory by cp.async (lane = key,
//           issued before the score loads, so K and V of a chunk are in flight together), then
//           lane = 4 of the 128 dims reads them key by key, p of the key broadcast by shuffle;
//   the 8 warps' (m, l, O) merge through shared memory at the end.
constexpr int kDecWarps = 8;
constexpr int kDecGMax = 8;

template <int DH>
__global__ void __launch_bounds__(32 * kDecWarps, 2) attn_decode_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k_cache,
    const __nv_bfloat16* __restrict__ v_cache, const int32_t* __restrict__ block_table, int max_pages,
    const int32_t* __restrict__ q_start, const int32_t* __restrict__ kv_before, int hq, int hkv, int page_size,
    float scale_log2, __nv_bfloat16* __restrict__ out) {
  constexpr int kDPL = DH / 32;  // dims per lane in P·V
  const int s = blockIdx.x / hkv, h = blockIdx.x % hkv;
  const int qs = q_start[s];
  if (q_start[s + 1] == qs) return;  // no query row for this sequence
  const int G = hq / hkv;
  const int n_keys = kv_before[s] + 1;  // the row at position kv_before[s] sees keys [0, kv_before[s]]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ __align__(16) __nv_bfloat16 sq[kDecGMax][DH];
  __shared__ float sm[kDecWarps][kDecGMax], sl[kDecWarps][kDecGMax];
  extern __shared__ __align__(16) uint8_t dec_smem[];
  __nv_bfloat16* sv = reinterpret_cast<__nv_bfloat16*>(dec_smem) + (size_t)warp * 32 * DH;  // this warp's V rows
  float (*so)[kDecGMax][DH] = reinterpret_cast<float (*)[kDecGMax][DH]>(dec_smem);      // merge (after the loop)
  for (int i = threadIdx.x; i < G * DH / 8; i += blockDim.x)
    reinterpret_cast<int4*>(&sq[0][0])[i] = reinterpret_cast<const int4*>(q + ((size_t)qs * hq + (size_t)h * G) * DH)[i];
  __syncthreads();
  const int32_t* bt = block_table + (size_t)s * max_pages;
  float m[kDecGMax], l[kDecGMax], o[kDecGMax][kDPL];
#pragma unroll
  for (int g = 0; g < kDecGMax; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int d = 0; d < kDPL; ++d) o[g][d] = 0.f;
  }
  for (int c0 = warp * 32; c0 < n_keys; c0 += kDecWarps * 32) {
    // ---- scores: lane = key ----
    const int key = c0 + lane;
    const bool valid = key < n_keys;
    const size_t krow = valid ? (((size_t)bt[key / page_size] * hkv + h) * page_size + key % page_size) * DH : 0;
    if (valid) {  // this key's V row → the warp's staging rows, in flight while the scores are computed
#pragma unroll
      for (int c = 0; c < DH / 8; ++c) cp_async16(sv + (size_t)lane * DH + 8 * c, v_cache + krow + 8 * c);
    }
    cp_commit();
    float sc[kDecGMax];
#pragma unroll
    for (int g = 0; g < kDecGMax; ++g) sc[g] = 0.f;
    if (valid) {
      const int4* kr = reinterpret_cast<const int4*>(k_cache + krow);
      // the row in two halves of ≤ 8 16-B loads (all of a half in flight before its FMAs)
#pragma unroll
      for (int c0 = 0; c0 < DH / 8; c0 += 8) {
        int4 kv[8];
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c0 + c < DH / 8) kv[c] = __ldg(kr + c0 + c);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c0 + c >= DH / 8) break;
          float kf[8];
          unpack8(kv[c], kf);
#pragma unroll
          for (int g = 0; g < kDecGMax; ++g) {
            if (g >= G) break;
            float qf[8];
            unpack8(reinterpret_cast<const int4*>(&sq[g][0])[c0 + c], qf);
#pragma unroll
            for (int j = 0; j < 8; ++j) sc[g] = fmaf(qf[j], kf[j], sc[g]);
          }
        }
      }
    }
    // ---- online softmax per head over the chunk ----
    float p[kDecGMax];
#pragma unroll
    for (int g = 0; g < kDecGMax; ++g) {
      if (g >= G) break;
      const float v = valid ? sc[g] * scale_log2 : -INFINITY;
      float mx = v;
#pragma unroll
      for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float mn = fmaxf(m[g], mx);  // finite: key c0 < n_keys is valid
      const float alpha = exp2f(m[g] - mn);
      p[g] = valid ? exp2f(v - mn) : 0.f;
      float sum = p[g];
#pragma unroll
      for (int off = 16; off; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
      l[g] = l[g] * alpha + sum;
      m[g] = mn;
#pragma unroll
      for (int d = 0; d < kDPL; ++d) o[g][d] *= alpha;
    }
    // ---- P·V from the staged rows: lane = dims [kDPL·lane, +kDPL) ----
    cp_wait<0>();
    __syncwarp();
    const int nk = min(32, n_keys - c0);
#pragma unroll 4
    for (int k = 0; k < nk; ++k) {
      const __nv_bfloat16* vr = sv + (size_t)k * DH + kDPL * lane;
      float vf[kDPL];
      if constexpr (kDPL == 4) {
        const uint2 raw = *reinterpret_cast<const uint2*>(vr);
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.x));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.y));
        vf[0] = a.x; vf[1] = a.y; vf[2] = b.x; vf[3] = b.y;
      } else {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vr));
        vf[0] = a.x; vf[1] = a.y;
      }
#pragma unroll
      for (int g = 0; g < kDecGMax; ++g) {
        if (g >= G) break;
        const float pk = __shfl_sync(0xffffffffu, p[g], k);
#pragma unroll
        for (int d = 0; d < kDPL; ++d) o[g][d] = fmaf(pk, vf[d], o[g][d]);
      }
    }
    __syncwarp();  // the staged rows are read before the next chunk's copies land
  }
  __syncthreads();  // the merge buffer aliases every warp's staging rows
  // ---- merge the warps ----
#pragma unroll
  for (int g = 0; g < kDecGMax; ++g) {
    if (g >= G) break;
    if (lane == 0) {
      sm[warp][g] = m[g];
      sl[warp][g] = l[g];
    }
#pragma unroll
    for (int d = 0; d < kDPL; ++d) so[warp][g][kDPL * lane + d] = o[g][d];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * DH; i += blockDim.x) {
    const int g = i / DH, d = i % DH;
    float M = -INFINITY;
    for (int w = 0; w < kDecWarps; ++w) M = fmaxf(M, sm[w][g]);
    float L = 0.f, O = 0.f;
    for (int w = 0; w < kDecWarps; ++w) {
      if (sm[w][g] == -INFINITY) continue;  // a warp that saw no key
      const float f = exp2f(sm[w][g] - M);
      L += sl[w][g] * f;
      O += so[w][g][d] * f;
    }
    out[((size_t)qs * hq + (size_t)h * G + g) * DH + d] = __float2bfloat16_rn(O / L);
  }
}

template <int DH>
int launch_decode(const void* q, const void* k, const void* v, const int32_t* bt, int max_pages,
                  const int32_t* q_start, const int32_t* kv_before, int bs, int hq, int hkv, int page_size, float scale,
                  void* out, cudaStream_t st) {
  // dynamic shared memory: 32 V rows per warp, reused for the warps' (m, l, O) merge
  constexpr size_t smem = (size_t)kDecWarps * 32 * DH * 2 > (size_t)kDecWarps * kDecGMax * DH * 4
                              ? (size_t)kDecWarps * 32 * DH * 2
                              : (size_t)kDecWarps * kDecGMax * DH * 4;
  if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(attn_decode_kernel<DH>), smem)) return rc;
  attn_decode_kernel<DH><<<bs * hkv, 32 * kDecWarps, smem, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(k),
      reinterpret_cast<const __nv_bfloat16*>(v), bt, max_pages, q_start, kv_before, hq, hkv, page_size,
      scale * 1.4426950408889634f, reinterpret_cast<__nv_bfloat16*>(out));
  SO_CHECK_LAUNCH();
  return SO_OK;
}

template <int DH>
int launch_dh(const void* q, const void* k, const void* v, const int32_t* bt, int max_pages, const int32_t* q_start,
              const int32_t* kv_before, int bs, int max_q, int hq, int hkv, int page_size, float scale, void* out,
              int variant, cudaStream_t st) {
  // TMA boxes cover whole pages (≤ 32 rows) or 32-row halves of larger pages
  const bool tma_ok = (page_size <= kKeys ? kKeys % page_size == 0 : page_size % kKeys == 0) &&
                      (reinterpret_cast<uintptr_t>(k) & 15) == 0 && (reinterpret_cast<uintptr_t>(v) & 15) == 0;
  // K6d on request only: measured slower than the tiled kernel at the draft's decode shape
  // (bs 64, ctx 520: 88 vs 53 µs, profiles/attn_r2.md) — kept as a tested alternative
  if (variant == 3 && max_q == 1 && hq / hkv <= kDecGMax && (DH == 128 || DH == 64))
    return launch_decode<DH>(q, k, v, bt, max_pages, q_start, kv_before, bs, hq, hkv, page_size, scale, out, st);
  if (variant == 3) variant = 0;
  // decode steps (one query row per sequence): cp.async staging measured faster than the TMA boxes
  // (bs 64, ctx 520: 52.9 vs 57.5 µs, profiles/kernels_r2.md)
  if (variant == 0 && tma_ok && max_q > 1)
    return launch<DH, true>(q, k, v, bt, max_pages, q_start, kv_before, bs, max_q, hq, hkv, page_size, scale, out, st);
  return launch<DH, false>(q, k, v, bt, max_pages, q_start, kv_before, bs, max_q, hq, hkv, page_size, scale, out, st);
}

}  // namespace

extern "C" int so_attn_paged_v(const void* q, const void* k_cache, const void* v_cache, const int32_t* block_table,
                               int max_pages, const int32_t* q_start, const int32_t* kv_before, int bs, int max_q,
                               int hq, int hkv, int dh, int page_size, float scale, void* out, int variant,
                               void* stream) {
  SO_REQUIRE(q && k_cache && v_cache && block_table && q_start && kv_before && out, SO_E_NULLPTR);
  SO_REQUIRE(bs >= 0 && max_q >= 1 && hq > 0 && hkv > 0 && hq % hkv == 0 && max_pages > 0, SO_E_SHAPE);
  SO_REQUIRE(page_size >= 1 && variant >= 0 && variant <= 3, SO_E_SHAPE);
  // prefill-shaped calls (the draft's context re-prefill, prompt prefill): K6c, the tcgen05 kernel —
  // FLOP-bound there, 221 vs 187 TF/s at 32-token pages (profiles/kernels_r2.md); verify and decode
  // steps stay on the tiled kernel, faster at a few query rows
  const bool tc_ok = dh == 128 && hq / hkv <= 128 && page_size >= 8 &&
                     (page_size <= 64 ? 64 % page_size == 0 : page_size % 64 == 0) && aligned16(q) &&
                     aligned16(k_cache) && aligned16(v_cache) && aligned16(out);
  if (variant == 2 || (variant == 0 && max_q >= kTcPrefillRows && tc_ok))
    return so_attn_paged_tc(q, k_cache, v_cache, block_table, max_pages, q_start, kv_before, bs, max_q, hq, hkv, dh,
                            page_size, scale, out, stream);
  SO_REQUIRE(aligned16(k_cache) && aligned16(v_cache), SO_E_ALIGN);
  if (bs == 0) return SO_OK;
  cudaStream_t st = as_stream(stream);
  if (dh == 128)
    return launch_dh<128>(q, k_cache, v_cache, block_table, max_pages, q_start, kv_before, bs, max_q, hq, hkv,
                          page_size, scale, out, variant, st);
  if (dh == 64)
    return launch_dh<64>(q, k_cache, v_cache, block_table, max_pages, q_start, kv_before, bs, max_q, hq, hkv,
                         page_size, scale, out, variant, st);
  return SO_E_UNSUPPORTED;
}

extern "C" int so_attn_paged(const void* q, const void* k_cache, const void* v_cache, const int32_t* block_table,
                             int max_pages, const int32_t* q_start, const int32_t* kv_before, int bs, int max_q,
                             int hq, int hkv, int dh, int page_size, float scale, void* out, void* stream) {
  return so_attn_paged_v(q, k_cache, v_cache, block_table, max_pages, q_start, kv_before, bs, max_q, hq, hkv, dh,
                         page_size, scale, out, 0, stream);
}
