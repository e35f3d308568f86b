// K6b — paged attention on the 5th-generation tensor cores (tcgen05, S and O in TMEM).
//
// Same contract as K6 (attention.cu, so_attn_paged): queries of each sequence
// attend causally over kv_before[s] cached keys plus their own block, through
// the block table; GQA rows = (position, query head of the kv-head group).
// The reference charges this work as CPU attention (costmodel.py:73,
// simulator.py:169-171); here it serves the verify pass (n_cand + 1 rows per
// sequence), the draft's context re-prefill and prefill inside a verify pass.
//
// Work unit = (sequence, kv head, tile of 128 query rows).  Persistent CTAs
// (one per SM: the unit's TMEM takes all 512 columns) walk the units
// round-robin; the K/V ring, the S / O TMEM buffers and every barrier phase
// run on across units, so the next unit's keys stream in while the previous
// one finishes.  Per 64-key tile:
//   warp 0      TMA producer: K and V page boxes (≤ 64 rows × 64 columns,
//               SWIZZLE_128B) of the tile into a 4-stage ring;
//   warp 1      TMEM allocator + single-thread MMA issuer:
//                 S  = Q · Kᵀ   M = 128 rows, N = 64 keys, K = dh (K-major both)
//                 O  = P · V    M = 128 rows, N = dh, K = 64 keys (V MN-major)
//               S of tile t+1 is issued before O of tile t, so the tensor
//               pipe works while the softmax runs;
//   warps 2–5   one query row per thread (the TMEM lane): load the unit's Q
//               row into shared memory, then per tile the online softmax on
//               the S row (no shuffles: a thread owns its row), P as bf16
//               into shared memory, and O_t (a fresh accumulator per tile)
//               folded into the register accumulator with the running
//               rescale; finally O / l to global.
// Keys past the causal limit are masked by select, and V rows past the
// sequence's keys in the last tile are zeroed so 0 · V stays finite whatever
// the unwritten cache holds.
#include "tc_common.cuh"

namespace {

constexpr int kDH = 128;
constexpr int kQRows = 128;
constexpr int kTKeys = 64;                   // keys per tile
constexpr int kTStages = 4;
constexpr int kAThreads = 192;
constexpr int kHalf = kTKeys * 128;          // one 64-column half of a K or V tile: 8 KB
constexpr int kKVBytes = 4 * kHalf;          // K (2 halves) + V (2 halves): 32 KB per stage
constexpr int kQBytes = 2 * kQRows * 128;    // 32 KB
constexpr int kPBytes = kQRows * 128;        // [128 rows × 64 keys] bf16: 16 KB
constexpr uint32_t kTmemCols = 512;          // S: 2 × 64 columns at 0, O: 2 × 128 at 256
constexpr uint32_t kOCol = 256;

struct Unit {
  int seq, kvh, p0, np, kvb, qs, n_keys, n_kt;
  bool live;
};

__device__ __forceinline__ Unit unit_info(int u, int hkv, int row_tiles, int P, const int32_t* __restrict__ q_start,
                                          const int32_t* __restrict__ kv_before) {
  Unit x;
  x.seq = u / (hkv * row_tiles);
  const int rem = u % (hkv * row_tiles);
  x.kvh = rem / row_tiles;
  const int t = rem % row_tiles;
  x.qs = q_start[x.seq];
  const int q_len = q_start[x.seq + 1] - x.qs;
  x.p0 = t * P;
  x.np = min(P, q_len - x.p0);
  x.live = x.np > 0;
  x.kvb = kv_before[x.seq];
  x.n_keys = x.live ? x.kvb + x.p0 + x.np : 0;  // the last row sees keys [0, kvb + p0 + np)
  x.n_kt = (x.n_keys + kTKeys - 1) / kTKeys;
  return x;
}

// MN-major SWIZZLE_128B operand descriptor: 64-element rows along N (128 B),
// 8-row groups along K at `sbo` bytes, the next 64 N-elements at `lbo` bytes
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(kAThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                   const __nv_bfloat16* __restrict__ q, const int32_t* __restrict__ block_table, int max_pages,
                   const int32_t* __restrict__ q_start, const int32_t* __restrict__ kv_before, int n_units,
                   int row_tiles, int hq, int hkv, int page_size, float scale_log2, __nv_bfloat16* __restrict__ out) {
  const int G = hq / hkv;
  const int P = kQRows / G;  // positions per unit
  const int box_rows = page_size < kTKeys ? page_size : kTKeys;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + kQBytes;
  uint8_t* sP = sKV + kTStages * kKVBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + kPBytes);
  uint64_t* kv_full = bars;                      // [kTStages]
  uint64_t* kv_empty = kv_full + kTStages;       // [kTStages]
  uint64_t* s_full = kv_empty + kTStages;        // [2]
  uint64_t* s_empty = s_full + 2;                // [2]
  uint64_t* o_full = s_empty + 2;                // [2]
  uint64_t* o_empty = o_full + 2;                // [2]
  uint64_t* q_full = o_empty + 2;
  uint64_t* q_empty = q_full + 1;
  uint64_t* p_full = q_empty + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(p_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kTStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], 4);
      mbar_init(&o_full[b], 1);
      mbar_init(&o_empty[b], 4);
    }
    mbar_init(q_full, 4);
    mbar_init(q_empty, 1);
    mbar_init(p_full, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmK)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmV)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      uint32_t it = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const Unit x = unit_info(u, hkv, row_tiles, P, q_start, kv_before);
        if (!x.live) continue;
        const int32_t* bt = block_table + (size_t)x.seq * max_pages;
        const int used = (x.n_keys + page_size - 1) / page_size;
        for (int kt = 0; kt < x.n_kt; ++kt, ++it) {
          const int s = it % kTStages;
          mbar_wait_guard(&kv_empty[s], ((it / kTStages) & 1) ^ 1);
          mbar_expect_tx(&kv_full[s], kKVBytes);
          uint8_t* sk = sKV + s * kKVBytes;
          uint8_t* sv = sk + 2 * kHalf;
          for (int r = 0; r < kTKeys; r += box_rows) {
            const int key = kt * kTKeys + r;
            const int pi = key / page_size;
            const int page = pi < used ? bt[pi] : bt[0];  // past the keys: any valid page (masked, V zeroed)
            const int row = (page * hkv + x.kvh) * page_size + key % page_size;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              tma_load_2d(sk + h * kHalf + r * 128, &tmK, &kv_full[s], h * 64, row);
              tma_load_2d(sv + h * kHalf + r * 128, &tmV, &kv_full[s], h * 64, row);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      constexpr uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTKeys >> 3) << 17) |
                                   ((uint32_t)(kQRows >> 4) << 24);
      constexpr uint32_t idesc_o = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) /* B = V, MN-major */ |
                                   ((uint32_t)(kDH >> 3) << 17) | ((uint32_t)(kQRows >> 4) << 24);
      uint32_t it = 0, uq = 0;  // global tile counter (ring stage, S/O buffer), unit counter (Q phase)
      const uint32_t q0 = smem_u32(sQ), p0 = smem_u32(sP);
      auto issue_s = [&](uint32_t t) {
        const int s = t % kTStages;
        mbar_wait_guard(&kv_full[s], (t / kTStages) & 1);
        mbar_wait_guard(&s_empty[t & 1], ((t >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t k0 = smem_u32(sKV + s * kKVBytes);
#pragma unroll
        for (int kk = 0; kk < kDH / 16; ++kk)
          umma_bf16(tmem_base + (t & 1) * kTKeys, umma_desc_sw128(q0 + (kk >> 2) * (kQRows * 128) + (kk & 3) * 32),
                    umma_desc_sw128(k0 + (kk >> 2) * kHalf + (kk & 3) * 32), idesc_s, kk != 0);
        umma_commit(&s_full[t & 1]);
      };
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const Unit x = unit_info(u, hkv, row_tiles, P, q_start, kv_before);
        if (!x.live) continue;
        mbar_wait_guard(q_full, uq & 1);
        const uint32_t t0 = it;
        issue_s(t0);
        for (int kt = 0; kt < x.n_kt; ++kt, ++it) {
          if (kt + 1 < x.n_kt) issue_s(it + 1);
          else umma_commit(q_empty);  // the unit's last S MMA: Q may be replaced once it completes
          mbar_wait_guard(p_full, it & 1);
          mbar_wait_guard(&o_empty[it & 1], ((it >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t v0 = smem_u32(sKV + (it % kTStages) * kKVBytes + 2 * kHalf);
#pragma unroll
          for (int kk = 0; kk < kTKeys / 16; ++kk)
            umma_bf16(tmem_base + kOCol + (it & 1) * kDH, umma_desc_sw128(p0 + kk * 32),
                      umma_desc_sw128_mn(v0 + kk * 2048, kHalf, 1024), idesc_o, kk != 0);
          umma_commit(&o_full[it & 1]);
          umma_commit(&kv_empty[it % kTStages]);
        }
        ++uq;
      }
    }
  } else {
    // ===== softmax / epilogue: one query row per thread =====
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    uint32_t it = 0, uq = 0;
    float o[kDH];
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const Unit x = unit_info(u, hkv, row_tiles, P, q_start, kv_before);
      if (!x.live) continue;
      const int j = row / G, hi = row % G;
      const bool valid = row < x.np * G;
      const int lim = valid ? x.kvb + x.p0 + j : -1;  // last key this row may see
      const size_t qrow = ((size_t)(x.qs + x.p0 + j) * hq + x.kvh * G + hi) * kDH;
      // ---- Q row → shared memory (K-major SWIZZLE_128B, two 64-column halves) ----
      mbar_wait_guard(q_empty, (uq & 1) ^ 1);
      {
        const int4* src = reinterpret_cast<const int4*>(q + qrow);
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const int4 v = valid ? src[c] : make_int4(0, 0, 0, 0);
          *reinterpret_cast<int4*>(sQ + (c >> 3) * (kQRows * 128) + row * 128 + (((c & 7) ^ (row & 7)) << 4)) = v;
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_full);
      float m = -INFINITY, l = 0.f;
#pragma unroll
      for (int d = 0; d < kDH; ++d) o[d] = 0.f;
      for (int kt = 0; kt < x.n_kt; ++kt, ++it) {
        // ---- S row of this tile ----
        mbar_wait_guard(&s_full[it & 1], (it >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        float sv[kTKeys];
#pragma unroll
        for (int c = 0; c < kTKeys; c += 32) {
          uint32_t r[32];
          tmem_ld32(tmem_base + (it & 1) * kTKeys + c + lane_off, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) sv[c + i] = __uint_as_float(r[i]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[it & 1]);
        const int key0 = kt * kTKeys;
        float mx = m;
#pragma unroll
        for (int c = 0; c < kTKeys; ++c) {
          sv[c] = key0 + c <= lim ? sv[c] * scale_log2 : -INFINITY;
          mx = fmaxf(mx, sv[c]);
        }
        const float mref = mx == -INFINITY ? 0.f : mx;  // fully masked row (padding): keep exp2 finite
        const float alpha = exp2f(m - mref);
        float sum = 0.f;
#pragma unroll
        for (int c = 0; c < kTKeys; ++c) {
          sv[c] = exp2f(sv[c] - mref);
          sum += sv[c];
        }
        l = l * alpha + sum;
        m = mx;
        // ---- fold the previous tile's P·V into the register accumulator ----
        if (kt > 0) {
          const uint32_t pt = it - 1;
          mbar_wait_guard(&o_full[pt & 1], (pt >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int c = 0; c < kDH; c += 32) {
            uint32_t r[32];
            tmem_ld32(tmem_base + kOCol + (pt & 1) * kDH + c + lane_off, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[c + i] += __uint_as_float(r[i]);
          }
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&o_empty[pt & 1]);
        }
#pragma unroll
        for (int d = 0; d < kDH; ++d) o[d] *= alpha;
        // ---- last tile: zero V rows past the keys (0 · V must stay finite) ----
        if (kt == x.n_kt - 1) {
          const int keep = x.n_keys - key0;
          const int vr = row & (kTKeys - 1);
          if (keep < kTKeys && vr >= keep) {
            uint8_t* sv_row = sKV + (it % kTStages) * kKVBytes + 2 * kHalf + (row >> 6) * kHalf + vr * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c) reinterpret_cast<int4*>(sv_row)[c] = make_int4(0, 0, 0, 0);
          }
        }
        // ---- P row (bf16) → shared memory (K-major SWIZZLE_128B, keys along K) ----
#pragma unroll
        for (int c = 0; c < kTKeys / 8; ++c)
          *reinterpret_cast<int4*>(sP + row * 128 + ((c ^ (row & 7)) << 4)) = pack8(sv + 8 * c);
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
      }
      // ---- the unit's last P·V, then O / l → global ----
      {
        const uint32_t pt = it - 1;
        mbar_wait_guard(&o_full[pt & 1], (pt >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int c = 0; c < kDH; c += 32) {
          uint32_t r[32];
          tmem_ld32(tmem_base + kOCol + (pt & 1) * kDH + c + lane_off, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[c + i] += __uint_as_float(r[i]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_empty[pt & 1]);
      }
      if (valid) {
        const float inv = 1.f / l;
        int4* dst = reinterpret_cast<int4*>(out + qrow);
#pragma unroll
        for (int c = 0; c < kDH / 8; ++c) {
          float f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = o[8 * c + i] * inv;
          dst[c] = pack8(f);
        }
      }
      ++uq;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

// the cache of one layer as a 2-D tensor [page·hkv·page_size + slot rows, dh]
int kv_map(CUtensorMap* m, const void* base, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return SO_E_DRIVER;
  cuuint64_t dims[2] = {(cuuint64_t)kDH, (cuuint64_t)1 << 31};
  cuuint64_t strides[1] = {(cuuint64_t)kDH * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? SO_OK : SO_E_DRIVER;
}

constexpr size_t kASmem = 1024 + kQBytes + (size_t)kTStages * kKVBytes + kPBytes + 256;

}  // namespace

extern "C" int so_attn_paged_tc(const void* q, const void* k_cache, const void* v_cache, const int32_t* block_table,
                                int max_pages, const int32_t* q_start, const int32_t* kv_before, int bs, int max_q,
                                int hq, int hkv, int dh, int page_size, float scale, void* out, void* stream) {
  SO_REQUIRE(q && k_cache && v_cache && block_table && q_start && kv_before && out, SO_E_NULLPTR);
  SO_REQUIRE(bs >= 0 && max_q >= 1 && hq > 0 && hkv > 0 && hq % hkv == 0 && max_pages > 0, SO_E_SHAPE);
  SO_REQUIRE(dh == kDH && hq / hkv <= kQRows, SO_E_UNSUPPORTED);
  SO_REQUIRE(page_size >= 8 && (page_size <= kTKeys ? kTKeys % page_size == 0 : page_size % kTKeys == 0),
             SO_E_UNSUPPORTED);
  SO_REQUIRE(aligned16(q) && aligned16(k_cache) && aligned16(v_cache) && aligned16(out), SO_E_ALIGN);
  if (bs == 0) return SO_OK;
  const int G = hq / hkv;
  const int P = kQRows / G;
  const int row_tiles = (max_q + P - 1) / P;
  const long n_units = (long)bs * hkv * row_tiles;
  SO_REQUIRE(n_units < (1L << 31), SO_E_SHAPE);
  int grid = device_sm_count();
  if (grid > n_units) grid = (int)n_units;
  CUtensorMap mk, mv;
  const int box_rows = page_size < kTKeys ? page_size : kTKeys;
  int rc = kv_map(&mk, k_cache, box_rows);
  if (rc) return rc;
  rc = kv_map(&mv, v_cache, box_rows);
  if (rc) return rc;
  if (int e = ensure_smem_attr(reinterpret_cast<const void*>(attn_tc_kernel), kASmem)) return e;
  attn_tc_kernel<<<grid, kAThreads, kASmem, as_stream(stream)>>>(
      mk, mv, reinterpret_cast<const __nv_bfloat16*>(q), block_table, max_pages, q_start, kv_before, (int)n_units,
      row_tiles, hq, hkv, page_size, scale * 1.4426950408889634f, reinterpret_cast<__nv_bfloat16*>(out));
  SO_CHECK_LAUNCH();
  return SO_OK;
}
