// K6c — paged attention on the 5th-generation tensor cores (tcgen05; S and O in TMEM).
//
// Same contract as K6 (attention.cu, so_attn_paged): queries of each sequence
// attend causally over kv_before[s] cached keys plus their own block, through
// the block table; GQA rows = (position, query head of the kv-head group).
// The reference charges this work as CPU attention (costmodel.py:73,
// simulator.py:169-171); here it serves the verify pass (n_cand + 1 rows per
// sequence), the draft's context re-prefill and prefill inside a verify pass.
//
// Work unit = (sequence, kv head, tile of ⌊128 / G⌋ positions × G heads).
// Persistent CTAs (one per SM) walk the units round-robin; every ring, TMEM
// buffer and barrier phase runs on across units, so the next unit's Q and
// keys stream in while the current one finishes.  Per 64-key tile:
//
//   warp 0      TMA producer: the unit's Q rows (one box of G heads × 64
//               columns per position, double-buffered across units) and the
//               K / V page boxes of each tile into SEPARATE rings (K runs a
//               tile ahead of V, and a K stage is recycled as soon as its S
//               MMA completes, so more of the shared memory is bytes in flight);
//   warp 1      TMEM allocator + single-thread MMA issuer:
//                 S  = Q · Kᵀ          M = 128 rows, N = 64 keys, K = dh
//                 O += P · V           M = 128 rows, N = dh, K = 64 keys (V MN-major)
//               S of tile t+1 is issued before P·V of tile t (two S buffers);
//               O ACCUMULATES IN TMEM over the unit's tiles (two O buffers, so
//               unit u's epilogue overlaps unit u+1);
//   warps 2–9   softmax, two threads per query row (the row's TMEM lane; each
//               thread 32 of the tile's 64 keys, partner maxima exchanged
//               through shared memory): masked row max, P = exp2(s − m_ref)
//               as bf16 into one of two P buffers, running row sum.  m_ref is
//               LAZY: it moves only when the tile max exceeds it by more than
//               2^8 (P ≤ 256 stays exact in bf16 and fp32), and only then is the
//               row of O rescaled in TMEM (after the previous P·V completes) —
//               with the max settling in the first tiles, the steady state
//               never touches O until the unit's epilogue O / l.
//
// Keys past the causal limit are masked by select; V rows past the unit's keys
// in its last tile are zeroed so 0 · V stays finite whatever the cache holds.
#include "tc_common.cuh"

namespace {

constexpr int kDH = 128;
constexpr int kQRows = 128;
constexpr int kTKeys = 64;                   // keys per tile
constexpr int kKStages = 4;                  // K ring: a stage frees once S = Q·Kᵀ has consumed it
constexpr int kVStages = 3;                  // V ring: a stage frees once P·V has consumed it
constexpr int kSoftWarps = 8;
constexpr int kAThreads = 64 + 32 * kSoftWarps;  // producer, MMA, 8 softmax warps
constexpr int kHalf = kTKeys * 128;          // one 64-column half of a K or V tile: 8 KB
constexpr int kKBytes = 2 * kHalf;           // one K (or V) tile: 2 halves, 16 KB
constexpr int kQHalf = kQRows * 128;         // one 64-column half of the Q tile: 16 KB
constexpr int kQBytes = 2 * kQHalf;          // 32 KB
constexpr int kPBytes = kQRows * 128;        // [128 rows × 64 keys] bf16: 16 KB
constexpr uint32_t kTmemCols = 512;          // S: 2 × 64 columns at 0; O: 2 × 128 at 128
constexpr uint32_t kOCol = 128;
constexpr float kRescaleLog2 = 8.0f;         // lazy max: rescale only past a 2^8 growth

#ifdef SO_ATTN_TRACE
// debug build only (make EXTRA=-DSO_ATTN_TRACE): per CTA, cycles each role spent in each wait
// (slot = wait site) plus the role's total cycles; read with so_attn_trace_copy
__device__ unsigned long long g_attn_trace[1024][16];
#define AW(slot, call)                                                         \
  do {                                                                         \
    const long long t0_ = clock64();                                           \
    call;                                                                      \
    if (blockIdx.x < 1024 && (threadIdx.x == 0 || threadIdx.x == 32 || threadIdx.x == 64)) \
      g_attn_trace[blockIdx.x][slot] += clock64() - t0_;                      \
  } while (0)
#else
#define AW(slot, call) call
#endif

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

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void softmax_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kSoftWarps) : "memory"); }

__global__ void __launch_bounds__(kAThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                   const __grid_constant__ CUtensorMap tmQ, const int32_t* __restrict__ block_table, int max_pages,
                   const int32_t* __restrict__ q_start, const int32_t* __restrict__ kv_before, int n_units,
                   int row_tiles, int hq, int hkv, int page_size, float scale_log2, __nv_bfloat16* __restrict__ out) {
  const int G = hq / hkv;
  const int P = kQRows / G;  // positions per unit
  const int box_rows = page_size < kTKeys ? page_size : kTKeys;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
  uint8_t* sQ = smem;                          // [2 units][2 halves][128 rows × 128 B]
  uint8_t* sK = sQ + 2 * kQBytes;              // [kKStages][half 0, half 1]
  uint8_t* sV = sK + kKStages * kKBytes;       // [kVStages][half 0, half 1]
  uint8_t* sP = sV + kVStages * kKBytes;       // [2][128 rows × 128 B]
  float* xmax = reinterpret_cast<float*>(sP + 2 * kPBytes);  // [2 tiles][2 halves][128 rows]
  float* xsum = xmax + 2 * 2 * kQRows;                        // [2 halves][128 rows]
  uint64_t* bars = reinterpret_cast<uint64_t*>(xsum + 2 * kQRows);
  uint64_t* k_full = bars;                     // [kKStages]
  uint64_t* k_empty = k_full + kKStages;       // [kKStages]
  uint64_t* v_full = k_empty + kKStages;       // [kVStages]
  uint64_t* v_empty = v_full + kVStages;       // [kVStages]
  uint64_t* s_full = v_empty + kVStages;       // [2]
  uint64_t* s_empty = s_full + 2;              // [2]
  uint64_t* p_full = s_empty + 2;              // [2]
  uint64_t* p_empty = p_full + 2;              // [2]  (P buffer free = its P·V completed)
  uint64_t* o_full = p_empty + 2;              // [2]
  uint64_t* o_empty = o_full + 2;              // [2]
  uint64_t* q_full = o_empty + 2;              // [2]
  uint64_t* q_empty = q_full + 2;              // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(q_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kKStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kVStages; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], kSoftWarps);
      mbar_init(&p_full[b], kSoftWarps);
      mbar_init(&p_empty[b], 1);
      mbar_init(&o_full[b], 1);
      mbar_init(&o_empty[b], kSoftWarps);
      mbar_init(&q_full[b], 1);
      mbar_init(&q_empty[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmK)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmV)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmQ)) : "memory");
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
#ifdef SO_ATTN_TRACE
  const long long t_start = clock64();
#endif

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer: per unit its Q rows, then its K / V tiles =====
      uint32_t it = 0, uq = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const Unit x = unit_info(u, hkv, row_tiles, P, q_start, kv_before);
        if (!x.live) continue;
        const uint32_t qb = uq & 1;
        AW(0, mbar_wait_guard(&q_empty[qb], ((uq >> 1) & 1) ^ 1));
        mbar_expect_tx(&q_full[qb], (uint32_t)(x.np * G * 256));
        uint8_t* q_dst = sQ + qb * kQBytes;
        for (int j = 0; j < x.np; ++j) {
          const int qrow = (x.qs + x.p0 + j) * hq + x.kvh * G;  // the G heads of position j are contiguous rows
#pragma unroll
          for (int h = 0; h < 2; ++h) tma_load_2d(q_dst + h * kQHalf + j * G * 128, &tmQ, &q_full[qb], h * 64, qrow);
        }
        ++uq;
        const int32_t* bt = block_table + (size_t)x.seq * max_pages;
        const int used = (x.n_keys + page_size - 1) / page_size;
        // one tile's page boxes (≤ 64 rows × 64 columns each, both halves) of the K or V cache
        auto load_tile = [&](const CUtensorMap* map, uint8_t* dst, uint64_t* bar, int kt) {
          for (int r = 0; r < kTKeys; r += box_rows) {
            const int key = kt * kTKeys + r;
            const int pi = key / page_size;
            const int page = pi < used ? bt[pi] : bt[0];  // past the keys: any valid page (masked, V zeroed)
            const int row = (page * hkv + x.kvh) * page_size + key % page_size;
#pragma unroll
            for (int h = 0; h < 2; ++h) tma_load_2d(dst + h * kHalf + r * 128, map, bar, h * 64, row);
          }
        };
        // K runs one tile ahead of V: S(t+1) needs K(t+1) while P·V(t) still holds V(t)
        for (int kt = 0; kt <= x.n_kt; ++kt) {
          if (kt < x.n_kt) {
            const uint32_t t = it + kt;
            const int s = t % kKStages;
            AW(1, mbar_wait_guard(&k_empty[s], ((t / kKStages) & 1) ^ 1));
            mbar_expect_tx(&k_full[s], kKBytes);
            load_tile(&tmK, sK + s * kKBytes, &k_full[s], kt);
          }
          if (kt > 0) {
            const uint32_t t = it + kt - 1;
            const int s = t % kVStages;
            AW(2, mbar_wait_guard(&v_empty[s], ((t / kVStages) & 1) ^ 1));
            mbar_expect_tx(&v_full[s], kKBytes);
            load_tile(&tmV, sV + s * kKBytes, &v_full[s], kt - 1);
          }
        }
        it += x.n_kt;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      constexpr uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTKeys >> 3) << 17) |
                                   ((uint32_t)(kQRows >> 4) << 24);
      constexpr uint32_t idesc_o = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) /* B = V, MN-major */ |
                                   ((uint32_t)(kDH >> 3) << 17) | ((uint32_t)(kQRows >> 4) << 24);
      uint32_t it = 0, uq = 0;  // global tile counter (ring stage, S/P buffer), unit counter (Q/O buffer)
      auto issue_s = [&](uint32_t t, uint32_t q0) {
        const int s = t % kKStages;
        AW(3, mbar_wait_guard(&k_full[s], (t / kKStages) & 1));
        AW(4, mbar_wait_guard(&s_empty[t & 1], ((t >> 1) & 1) ^ 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t k0 = smem_u32(sK + s * kKBytes);
#pragma unroll
        for (int kk = 0; kk < kDH / 16; ++kk)
          umma_bf16(tmem_base + (t & 1) * kTKeys, umma_desc_sw128(q0 + (kk >> 2) * kQHalf + (kk & 3) * 32),
                    umma_desc_sw128(k0 + (kk >> 2) * kHalf + (kk & 3) * 32), idesc_s, kk != 0);
        umma_commit(&s_full[t & 1]);
        umma_commit(&k_empty[s]);  // the K stage is free once this S completes
      };
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const Unit x = unit_info(u, hkv, row_tiles, P, q_start, kv_before);
        if (!x.live) continue;
        const uint32_t qb = uq & 1, ob = uq & 1;
        const uint32_t q0 = smem_u32(sQ + qb * kQBytes);
        const uint32_t o_tm = tmem_base + kOCol + ob * kDH;
        AW(5, mbar_wait_guard(&q_full[qb], (uq >> 1) & 1));
        issue_s(it, q0);
        AW(6, mbar_wait_guard(&o_empty[ob], ((uq >> 1) & 1) ^ 1));  // unit uq−2's epilogue has read this O buffer
        for (int kt = 0; kt < x.n_kt; ++kt, ++it) {
          if (kt + 1 < x.n_kt) issue_s(it + 1, q0);
          else umma_commit(&q_empty[qb]);  // the unit's last S MMA: Q may be replaced once it completes
          AW(7, mbar_wait_guard(&v_full[it % kVStages], (it / kVStages) & 1));
          AW(8, mbar_wait_guard(&p_full[it & 1], (it >> 1) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t v0 = smem_u32(sV + (it % kVStages) * kKBytes);
          const uint32_t p0 = smem_u32(sP + (it & 1) * kPBytes);
#pragma unroll
          for (int kk = 0; kk < kTKeys / 16; ++kk)
            umma_bf16(o_tm, umma_desc_sw128(p0 + kk * 32), umma_desc_sw128_mn(v0 + kk * 2048, kHalf, 1024), idesc_o,
                      (kt > 0) | (kk != 0));
          umma_commit(&v_empty[it % kVStages]);
          umma_commit(&p_empty[it & 1]);
        }
        umma_commit(&o_full[ob]);
        ++uq;
      }
    }
  } else {
    // ===== softmax / epilogue: two threads per query row =====
    const int sw = warp - 2;
    const int half = sw >> 2;                 // keys [32·half, 32·half + 32) of each tile, O columns [64·half, +64)
    const int quarter = warp & 3;             // TMEM lane window of this warp
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    uint32_t it = 0, uq = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const Unit x = unit_info(u, hkv, row_tiles, P, q_start, kv_before);
      if (!x.live) continue;
      const uint32_t ob = uq & 1;
      const uint32_t o_tm = tmem_base + kOCol + ob * kDH + half * 64 + lane_off;
      const int j = row / G, hi = row % G;
      const bool valid = row < x.np * G;
      const int lim = valid ? x.kvb + x.p0 + j : -1;  // last key this row may see
      float m_ref = -INFINITY, l = 0.f;
      for (int kt = 0; kt < x.n_kt; ++kt, ++it) {
        // ---- this thread's 32 S values of the tile ----
        AW(9, mbar_wait_guard(&s_full[it & 1], (it >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        float sv[32];
        {
          uint32_t r[32];
          tmem_ld32(tmem_base + (it & 1) * kTKeys + half * 32 + lane_off, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) sv[i] = __uint_as_float(r[i]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[it & 1]);
        const int key0 = kt * kTKeys + half * 32;
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          sv[c] = key0 + c <= lim ? sv[c] * scale_log2 : -INFINITY;
          mx = fmaxf(mx, sv[c]);
        }
        // ---- row max across the two halves ----
        float* xm = xmax + (it & 1) * 2 * kQRows;
        xm[half * kQRows + row] = mx;
        softmax_sync();
        mx = fmaxf(mx, xm[(half ^ 1) * kQRows + row]);
        // lazy max: move the reference only past a 2^8 growth (always on a valid row's first tile)
        const bool move = mx > m_ref + kRescaleLog2;
        const float alpha = move ? exp2f(m_ref - mx) : 1.f;  // 0 on the first tile
        if (kt > 0 && __any_sync(0xffffffffu, move)) {
          // rescale the warp's rows of O (its 64-column half) in TMEM once the previous tile's P·V has
          // landed — warp-wide (tcgen05.ld/st are .sync.aligned); rows that keep their max scale by 1
          const uint32_t pt = it - 1;
          AW(10, mbar_wait_guard(&p_empty[pt & 1], (pt >> 1) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int c = 0; c < 64; c += 32) {
            uint32_t r[32];
            tmem_ld32(o_tm + c, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            tmem_st32(o_tm + c, r);
          }
          tmem_st_wait();
        }
        if (move) {
          l *= alpha;
          m_ref = mx;
        }
        const float mr = m_ref == -INFINITY ? 0.f : m_ref;  // fully masked row (padding): P = 0
        float sum = 0.f;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          sv[c] = sv[c] == -INFINITY ? 0.f : exp2f(sv[c] - mr);
          sum += sv[c];
        }
        l += sum;
        // ---- last tile: zero V rows past the keys (0 · V must stay finite) ----
        if (kt == x.n_kt - 1) {
          const int keep = x.n_keys - kt * kTKeys;
          const int vr = row & (kTKeys - 1);
          if (keep < kTKeys && vr >= keep) {
            // V(t) lands after S(t) is read (the producer runs K ahead): wait for it
            AW(11, mbar_wait_guard(&v_full[it % kVStages], (it / kVStages) & 1));
            uint8_t* v_row = sV + (it % kVStages) * kKBytes + (row >> 6) * kHalf + vr * 128;
#pragma unroll
            for (int c = 0; c < 4; ++c) reinterpret_cast<int4*>(v_row)[half * 4 + c] = make_int4(0, 0, 0, 0);
          }
        }
        // ---- P (bf16) → shared memory once the buffer's previous P·V is done (K-major SWIZZLE_128B) ----
        AW(12, mbar_wait_guard(&p_empty[it & 1], ((it >> 1) & 1) ^ 1));
        uint8_t* pb = sP + (it & 1) * kPBytes + row * 128;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int chunk = half * 4 + c;
          *reinterpret_cast<int4*>(pb + ((chunk ^ (row & 7)) << 4)) = pack8(sv + 8 * c);
        }
        fence_async_smem();
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[it & 1]);
      }
      // ---- epilogue: O / l of this thread's 64 columns ----
      xsum[half * kQRows + row] = l;
      softmax_sync();
      l += xsum[(half ^ 1) * kQRows + row];
      AW(13, mbar_wait_guard(&o_full[ob], (uq >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float o[64];
#pragma unroll
      for (int c = 0; c < 64; c += 32) {
        uint32_t r[32];
        tmem_ld32(o_tm + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) o[c + i] = __uint_as_float(r[i]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[ob]);
      if (valid) {
        const float inv = 1.f / l;
        const size_t qrow = ((size_t)(x.qs + x.p0 + j) * hq + x.kvh * G + hi) * kDH + half * 64;
        int4* dst = reinterpret_cast<int4*>(out + qrow);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = o[8 * c + i] * inv;
          dst[c] = pack8(f);
        }
      }
      softmax_sync();  // xsum / xmax reuse by the next unit
      ++uq;
    }
  }
#ifdef SO_ATTN_TRACE
  if (threadIdx.x == 64 && blockIdx.x < 1024) g_attn_trace[blockIdx.x][14] += clock64() - t_start;
  if (threadIdx.x == 32 && blockIdx.x < 1024) g_attn_trace[blockIdx.x][15] += clock64() - t_start;
#endif
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

// a [rows, dh] view with 64-column × box_rows boxes (SWIZZLE_128B); rows unbounded (the kernel
// only addresses rows it was given)
int rows_map(CUtensorMap* m, const void* base, int box_rows) {
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

constexpr size_t kASmem = 1024 + 2 * (size_t)kQBytes + (size_t)(kKStages + kVStages) * kKBytes + 2 * (size_t)kPBytes +
                          (2 * 2 * kQRows + 2 * kQRows) * sizeof(float) + 256;

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
  CUtensorMap mk, mv, mq;
  const int box_rows = page_size < kTKeys ? page_size : kTKeys;
  int rc = rows_map(&mk, k_cache, box_rows);
  if (rc) return rc;
  rc = rows_map(&mv, v_cache, box_rows);
  if (rc) return rc;
  rc = rows_map(&mq, q, G);  // q [T, hq, dh] as rows (t, head): one box = the G heads of one position
  if (rc) return rc;
  if (int e = ensure_smem_attr(reinterpret_cast<const void*>(attn_tc_kernel), kASmem)) return e;
  attn_tc_kernel<<<grid, kAThreads, kASmem, as_stream(stream)>>>(
      mk, mv, mq, block_table, max_pages, q_start, kv_before, (int)n_units, row_tiles, hq, hkv, page_size,
      scale * 1.4426950408889634f, reinterpret_cast<__nv_bfloat16*>(out));
  SO_CHECK_LAUNCH();
  return SO_OK;
}

#ifdef SO_ATTN_TRACE
extern "C" int so_attn_trace_copy(void* host, size_t bytes, int reset) {
  if (bytes > sizeof(g_attn_trace)) bytes = sizeof(g_attn_trace);
  int rc = (int)cudaMemcpyFromSymbol(host, g_attn_trace, bytes);
  if (reset) {
    static unsigned long long zero[1024][16];
    cudaMemcpyToSymbol(g_attn_trace, zero, sizeof(zero));
  }
  return rc;
}
#endif
