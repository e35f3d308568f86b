/*
 * specoffload_b200.h — C ABI of the B200-native offloaded speculative-decoding
 * hot path (SpecOffload, arXiv 2505.10259).
 *
 * The reference (`specpipe`, /root/reference/pkg) is a Python performance model
 * with no FFI; the path it models is entered through
 *   simulate_decoding(policy, workload, hw, target, draft, plan, seed)
 *       pkg/src/specpipe/simulator.py:108-116
 * whose per-round, per-layer body (simulator.py:155-215) is
 *   attention ‖ FFN C2G load  →  FFN compute  →  barrier → sample_accepted
 * Each entry point below is one of the physical operations that loop models;
 * the comment on each names the reference line it replaces.  The Python host
 * layer (paper_2505_10259_b200/native.py) binds these with ctypes.
 *
 * Conventions:
 *  - every call is asynchronous on the caller's cudaStream_t (passed as void*);
 *  - all pointers are device pointers unless named *_host / pinned;
 *  - the caller owns every buffer; the library never allocates or frees
 *    caller-visible memory and keeps no per-call state;
 *  - return 0 on success, a negative SO_E_* code for argument errors, or a
 *    positive cudaError_t for launch failures.  Nothing throws or aborts.
 *  - bf16 tensors are passed as `const void*` (uint16 bit patterns).
 */
#ifndef SPECOFFLOAD_B200_H
#define SPECOFFLOAD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SO_OK 0
#define SO_E_NULLPTR (-1)
#define SO_E_SHAPE (-2)
#define SO_E_ALIGN (-3)
#define SO_E_UNSUPPORTED (-4)
#define SO_E_DRIVER (-5)

/* GEMM epilogues (so_gemm_bf16 / grouped GEMMs). */
#define SO_EPI_BF16 0          /* C = A·Bᵀ                         (bf16 out) */
#define SO_EPI_F32 1           /* C = A·Bᵀ                         (fp32 out) */
#define SO_EPI_BF16_RESID 2    /* C = A·Bᵀ + R                     (bf16 out) */
#define SO_EPI_SWIGLU 3        /* C = silu(A·Bgᵀ) ⊙ (A·Buᵀ), B rows interleaved in 64-row gate/up blocks */
#define SO_EPI_BF16_ROWSCALE 4 /* C[r,:] = w[r] · (A·Bᵀ)[r,:]      (bf16 out) */

int so_abi_version(void);
const char* so_status_string(int status);
int so_device_sm_count(void);
/* Make `device` current for the calling host thread (each enqueuing thread —
 * the verify and the draft streams are fed from two — calls this once). */
int so_set_device(int device);

/* Stream plumbing for the per-layer loops (events, async copies).  They wrap
 * the CUDA runtime so a host binding never blocks on a full launch queue
 * while holding its own interpreter lock. */
int so_event_create(int timing, void** out_event);
int so_event_destroy(void* event);
int so_event_record(void* event, void* stream);
int so_stream_wait_event(void* stream, void* event);
int so_event_synchronize(void* event);
int so_event_elapsed_ms(void* start, void* end, float* ms);
int so_memcpy_async(void* dst, const void* src, size_t bytes, void* stream);
int so_stream_synchronize(void* stream);
/* Non-blocking probes (0 = complete, 600 = cudaErrorNotReady) for stall
 * diagnostics (tools/stall_probe.py). */
int so_stream_query(void* stream);
int so_event_query(void* event);
/* Small transfer (KBs) between pinned host memory and HBM done by SMs over
 * UVA, so per-round metadata never queues behind layer copies on the copy
 * engine. */
int so_copy_sm(void* dst, const void* src, size_t bytes, void* stream);

/* Verify-batch assembly: tokens[s] = [t_last[s], drafts[0..n-1][s]] and
 * draft_rows[s] = drafts[..][s] from the step-major draft buffer [n, ld]. */
int so_build_verify_tokens(const int32_t* t_last, const int32_t* drafts, int ld, int bs, int n_cand,
                           int32_t* tokens, int32_t* draft_rows, void* stream);
/* out[i] = src[idx[i]] (int32 gather, e.g. the token history of a re-prefill). */
int so_gather_i32(const int32_t* src, const int64_t* idx, int n, int32_t* out, void* stream);
/* dst[idx[i]] = val[i] (int32 scatter into the token history). */
int so_scatter_i32(int32_t* dst, const int64_t* idx, const int32_t* val, int n, void* stream);

/* ---- K7: speculative accept / reject ------------------------------------
 * Replaces the statistical draw `sample_accepted` (acceptance.py:55-72,
 * called at simulator.py:213) and the clamp `remaining - accepted`
 * (simulator.py:214) with the real decision on target logits.
 * Greedy: n = leading count of draft[i] == argmax(logits[i]) (lowest index on
 * ties); emit draft[0:n] ++ [argmax(logits[n])]; count = min(n+1, remaining).
 * forced_accept (optional, may be NULL) replaces n by min(forced-1, n_cand)
 * (forced-acceptance benchmark mode).
 * out_tokens [bs, n_cand+1] (entries past count are -1), out_counts [bs]. */
int so_accept_greedy(const int32_t* draft_tokens, const float* target_logits,
                     const int32_t* remaining, const int32_t* forced_accept,
                     int bs, int n_cand, int vocab,
                     int32_t* out_tokens, int32_t* out_counts, void* stream);

/* Sampling verification (Leviathan et al. Alg. 1): accept draft token i iff
 * u_accept[i]·q_i(d_i) ≤ p_i(d_i), p = softmax(inv_temp·logits) in the
 * canonical deterministic order; on the first rejection
 * sample norm(max(p_i−q_i,0)) with u_resample, else the bonus from p_n. */
int so_accept_sample(const int32_t* draft_tokens, const float* target_logits,
                     const float* draft_probs, const float* u_accept,
                     const float* u_resample, const int32_t* remaining,
                     float inv_temperature, int bs, int n_cand, int vocab,
                     int32_t* out_tokens, int32_t* out_counts, void* stream);

/* Draft-side token choice: greedy argmax (uniforms == NULL) or inverse-CDF
 * sampling from softmax(inv_temp·logits); optionally writes the normalised
 * probabilities (needed by so_accept_sample).  logits may be strided rows. */
int so_sample_tokens(const float* logits, int64_t row_stride, const float* uniforms,
                     float inv_temperature, int rows, int vocab,
                     int32_t* out_tokens, int64_t token_stride,
                     float* out_probs, int64_t probs_row_stride, void* stream);

/* ---- K2: fused top-2 router + token permutation --------------------------
 * Mixtral routing: logits = x·Wgᵀ (fp32 accumulate), fp32 softmax, top-2
 * (ties → lower expert), renormalise by the pair sum.  Produces a stable
 * (token-ordered) expert-major permutation so the grouped GEMMs see one
 * contiguous row block per expert.
 * outputs: expert_offsets [E+1]; perm_token [2T] (row → token);
 * row_weight [2T] (routing weight of the row); token_rows [T,2] (token →
 * its two rows); x_perm [2T,H] (gathered activations);
 * topk_idx [T,2] / topk_w [T,2] (for inspection, may be NULL).
 * workspace: so_router_workspace_bytes(T, E) bytes of device scratch. */
size_t so_router_workspace_bytes(int T, int E);
int so_router_top2(const void* x, const void* w_gate, int T, int H, int E,
                   int32_t* topk_idx, float* topk_w, int32_t* expert_offsets,
                   int32_t* perm_token, float* row_weight, int32_t* token_rows,
                   void* x_perm, void* workspace, void* stream);

/* out[t] = resid[t] + y[token_rows[t,0]] + y[token_rows[t,1]] (fixed order) */
int so_moe_combine(const void* y_perm, const int32_t* token_rows, const void* resid,
                   int T, int H, void* out, void* stream);

/* ---- K3/K4/K5: tcgen05 GEMMs (bf16 in, fp32 accumulate in TMEM) ---------
 * C[M,N] = A[M,K] · B[N,K]ᵀ, both K-major, K % 64 == 0, 16-B aligned rows.
 * epilogue SO_EPI_*; aux = residual (bf16 [M,ldc]) or row scale (fp32 [M]).
 * For SO_EPI_SWIGLU, N counts the interleaved gate+up rows and C has N/2
 * columns. */
int so_gemm_bf16(const void* A, const void* B, int M, int N, int K,
                 void* C, int ldc, int epilogue, const void* aux, void* stream);
/* Same contract with caller-owned scratch: skinny GEMMs (M ≤ 256 with fewer
 * output tiles than half the SMs — the draft's decode steps) split K across
 * the SMs into fp32 partials in `workspace`, then one reduce kernel applies
 * the epilogue.  so_gemm_workspace_bytes(M, N, K) is the scratch that choice
 * needs (0 = no split); a smaller workspace falls back to so_gemm_bf16. */
size_t so_gemm_workspace_bytes(int M, int N, int K);
int so_gemm_bf16_ex(const void* A, const void* B, int M, int N, int K, void* C, int ldc, int epilogue,
                    const void* aux, void* workspace, size_t ws_bytes, void* stream);

/* Grouped (MoE) GEMM: rows [offs[e], offs[e+1]) of A use expert e's weight
 * B + e·N·K.  max_rows bounds offs[E] (no host sync: the tile schedule is
 * derived on device from offs). */
/* K5c — decode-step GEMM, M ≤ 128 activation rows (the draft's n_cand decode
 * steps, costmodel.py:53-57 t_draft_decode_gpu): the weights W [N,K] stream
 * once from HBM over (nearly) every SM — swap-AB tcgen05 tiles of 128 weight
 * rows; each tile's K range split over the C ≤ 8 CTAs of a thread-block
 * cluster; the fp32 partials reduced through distributed shared memory in
 * fixed CTA order (deterministic) with the epilogue fused.  N % 128 == 0,
 * K % 128 == 0; epilogues SO_EPI_BF16 / F32 / BF16_RESID / SWIGLU.
 * so_gemv_workspace_bytes returns 256 for shapes K5c serves (fewer weight
 * tiles than SMs) and 0 otherwise; the kernel itself needs no scratch (the
 * workspace arguments are accepted and ignored).  so_gemm_bf16_v (variant 0
 * or 4) routes eligible shapes here.  Launched with programmatic stream
 * serialization (PDL): it may start while the previous kernel on the stream
 * finishes, prefetching weight tiles, and reads X / aux only after
 * griddepcontrol.wait — stream semantics are unchanged for callers
 * (environment SO_NO_PDL=1 launches it plainly). */
size_t so_gemv_workspace_bytes(int M, int N, int K);
int so_gemv_bf16(const void* X, const void* W, int M, int N, int K, void* C, int ldc, int epilogue,
                 const void* aux, void* workspace, size_t ws_bytes, void* stream);
int so_gemm_grouped_bf16(const void* A, const void* B, const int32_t* expert_offsets,
                         int E, int max_rows, int N, int K, void* C, int ldc,
                         int epilogue, const void* aux, void* stream);
/* The general GEMM entry the three above specialise: dense (expert_offsets ==
 * NULL, optional split-K workspace) or grouped (M = max_rows), with the tile
 * variant an explicit argument — 0 = auto (persistent kernels with
 * double-buffered TMEM accumulators: CTA-pair 256×256 cta_group::2 tiles for
 * dense M ≥ 1024 with N % 256 == 0, else 1-CTA 128×{128,256}), 1 = persistent
 * 1-CTA only, 2 = persistent CTA-pair wherever legal, 3 = the auto choice with
 * one tile per CTA (non-persistent, no split-K), 4 = the K5c decode-step
 * kernel (so_gemv_bf16) where eligible, else auto.  Auto (0) takes K5c for
 * dense M ≤ 128 with fewer weight tiles than SMs.  No process-wide state. */
int so_gemm_bf16_v(const void* A, const void* B, const int32_t* expert_offsets, int E, int M, int N, int K,
                   void* C, int ldc, int epilogue, const void* aux, void* workspace, size_t ws_bytes,
                   int variant, void* stream);

/* ---- K8: auxiliary ------------------------------------------------------- */
int so_embed(const int32_t* tokens, const void* table, int T, int H, void* out, void* stream);
int so_rmsnorm(const void* x, const void* w, int T, int H, float eps, void* out, void* stream);
/* qkv [T, (hq+2hkv)·dh] (dh % 8 == 0, dh ≤ 128, 16-B aligned) → RoPE(q) into q_out [T,hq,dh]; RoPE(k), v appended
 * to the paged caches at slot_mapping[t] (page·page_size + offset).
 * cache layout: [num_pages, hkv, page_size, dh]. */
int so_rope_kv_append(const void* qkv, const int32_t* positions, const int32_t* slot_mapping,
                      int T, int hq, int hkv, int dh, float rope_theta, int page_size,
                      void* q_out, void* k_cache, void* v_cache, void* stream);

/* ---- K6: multi-token verification attention over the paged KV cache ------
 * Sequence s owns query rows [q_start[s], q_start[s+1]); query row j of s
 * sits at position kv_before[s] + j and attends keys [0, kv_before[s]+j]
 * (causal inside the new tokens).  GQA: q head h reads kv head h/(hq/hkv).
 * out [rows, hq·dh] bf16. */
int so_attn_paged(const void* q, const void* k_cache, const void* v_cache,
                  const int32_t* block_table, int max_pages,
                  const int32_t* q_start, const int32_t* kv_before,
                  int bs, int max_q, int hq, int hkv, int dh, int page_size,
                  float scale, void* out, void* stream);
/* Same with the kernel an explicit argument: 0 = auto (so_attn_paged's
 * choice): prefill-shaped calls (max_q ≥ 64, dh 128, K6c page sizes) go to
 * K6c; otherwise TMA boxes issued by one thread where the page size allows
 * (pages of ≤ 32 slots dividing 32, or multiples of 32) and more than one
 * query row, else cp.async; 1 = cp.async by
 * every thread; 2 = K6c, the tcgen05 kernel (so_attn_paged_tc); 3 = K6d, a
 * CUDA-core streaming kernel for decode steps (max_q == 1, hq/hkv ≤ 8: CTA per
 * sequence × kv head, lane-per-key scores, cp.async-staged V, warps merged in
 * shared memory) where eligible, else auto. */
int so_attn_paged_v(const void* q, const void* k_cache, const void* v_cache,
                    const int32_t* block_table, int max_pages,
                    const int32_t* q_start, const int32_t* kv_before,
                    int bs, int max_q, int hq, int hkv, int dh, int page_size,
                    float scale, void* out, int variant, void* stream);
/* K6c — the same attention on the tcgen05 tensor cores: persistent CTAs over
 * (sequence, kv head, 128 query rows) units, S = Q·Kᵀ in TMEM, O accumulated
 * in TMEM (lazy rescale), TMA-staged Q and K/V tiles of 64 keys, two softmax
 * threads per query row.
 * dh = 128, hq/hkv ≤ 128, page_size ≥ 8 dividing 64 or a multiple of 64. */
int so_attn_paged_tc(const void* q, const void* k_cache, const void* v_cache,
                     const int32_t* block_table, int max_pages,
                     const int32_t* q_start, const int32_t* kv_before,
                     int bs, int max_q, int hq, int hkv, int dh, int page_size,
                     float scale, void* out, void* stream);

/* ---- Canonical-order arithmetic (parity mode, tiny shapes) ----------------
 * The same ops, operands, epilogues and bf16 rounding points as the product
 * kernels above (so_gemm_bf16 / so_gemm_grouped_bf16, so_rmsnorm,
 * so_rope_kv_append, so_attn_paged, so_router_top2), computed by CUDA cores
 * with every float op a single correctly rounded IEEE op in a fixed order
 * (sequential fma dot products, det_exp, IEEE sqrt/div; csrc/canon.cu header).
 * oracle/csrc/canon_oracle.c restates them, so a model run through these
 * entry points reproduces the CPU oracle's logits and tokens bit for bit —
 * the "bit-exact accepted tokens on the tiny config" target (
 * the verify pass it serves is modeled at costmodel.py:60-76).  One thread per
 * output element: for parity tests, not throughput.
 * so_canon_gemm: expert_offsets == NULL → dense C = epi(A·Bᵀ); else grouped as
 * so_gemm_grouped_bf16 with M = max_rows.
 * so_canon_rope_kv_append: rope_table [table_rows, dh] fp32 holds cos(p·f_i)
 * in columns [0, dh/2) and sin(p·f_i) in [dh/2, dh) for position p (every
 * position must be < table_rows; the kernel traps otherwise). */
int so_canon_gemm(const void* A, const void* B, const int32_t* expert_offsets, int E, int M, int N, int K,
                  void* C, int ldc, int epilogue, const void* aux, void* stream);
int so_canon_rmsnorm(const void* x, const void* w, int T, int H, float eps, void* out, void* stream);
int so_canon_rope_kv_append(const void* qkv, const int32_t* positions, const int32_t* slot_mapping, int T,
                            int hq, int hkv, int dh, const float* rope_table, int table_rows, int page_size,
                            void* q_out, void* k_cache, void* v_cache, void* stream);
int so_canon_attn_paged(const void* q, const void* k_cache, const void* v_cache, const int32_t* block_table,
                        int max_pages, const int32_t* q_start, const int32_t* kv_before, int bs, int max_q,
                        int hq, int hkv, int dh, int page_size, float scale, void* out, void* stream);
int so_canon_router_top2(const void* x, const void* w_gate, int T, int H, int E, int32_t* topk_idx,
                         float* topk_w, int32_t* expert_offsets, int32_t* perm_token, float* row_weight,
                         int32_t* token_rows, void* x_perm, void* workspace, void* stream);

/* ---- K1: layer streamer -------------------------------------------------
 * Pinned host → HBM window slot, `chunk`-byte cudaMemcpyAsync pieces on the
 * caller's copy stream, then records `done_event` (may be NULL).
 * Replaces the modeled `ffn_load` event (simulator.py:172-176). */
int so_stream_layer(void* slot, const void* pinned_src, size_t bytes, size_t chunk,
                    void* stream, void* done_event);

/* ---- K9: XC4 lossless exponent-coded weight units ------------------------
 * Same streamed bytes' *meaning* as so_stream_layer (the modeled `ffn_load`,
 * simulator.py:172-176; ffn_bytes / c2g_bandwidth, costmodel.py:74), fewer
 * bytes on the link: sign+mantissa byte + a 3- or 4-bit exponent code per
 * bf16 weight, escapes in a side stream (format: csrc/wcodec.cu).  Decoding
 * is bit-exact.  A unit = this header | u64 frame_off[n_frames+1] | frames. */
typedef struct so_xc4_header {
  uint32_t magic;          /* "XC41" */
  uint32_t version;        /* 1: 4-bit codes (15 exponents + escape); 2: 3-bit codes (7 + escape) */
  uint64_t n_elems;        /* bf16 weights in the unit (multiple of 16) */
  uint32_t frame_elems;    /* elements per frame (multiple of 4096) */
  uint32_t n_frames;
  uint8_t exp_of_code[16]; /* code → exponent byte; code 15 = escape */
  uint64_t total_bytes;    /* encoded unit size */
  uint64_t n_escapes;
  uint8_t reserved[8];
} so_xc4_header;

/* Device scratch for so_xc4_encode, and an upper bound of the encoded size. */
size_t so_xc4_scratch_bytes(uint64_t n_elems, uint32_t frame_elems);
size_t so_xc4_bound(uint64_t n_elems, uint32_t frame_elems);
/* Encode `n_elems` bf16 weights (device) into `dst` (device, 16-B aligned).
 * code_bits: 0 = the smaller of 3- and 4-bit codes for this unit, 3 or 4 =
 * forced (3 needs n_elems % 32 == 0).  dst == NULL → size query: *out_bytes =
 * encoded size.  Synchronises `stream` (setup-time call, not a hot-path one). */
int so_xc4_encode(const void* src, uint64_t n_elems, uint32_t frame_elems, int code_bits, void* dst,
                  size_t dst_cap, void* scratch, uint64_t* out_bytes, so_xc4_header* out_header, void* stream);
/* Decode frames [frame_begin, frame_end) of a unit whose bytes sit at
 * unit_dev (device) into dst (the unit's full bf16 output; frame f lands at
 * element f·frame_elems).  unit_host = a host copy of at least the header and
 * frame table (the streamed unit in pinned memory). */
int so_xc4_decode(const void* unit_host, const void* unit_dev, uint32_t frame_begin, uint32_t frame_end,
                  void* dst, void* stream);
/* K1 over XC4: per frame, H2D copy of the encoded frame (pinned → ring slot,
 * copy stream) then its decode into `slot` (decode stream).  ring_events =
 * 2·ring_slots caller-created events (copied, consumed) per ring slot;
 * *ring_cursor counts frames across calls.  The decode stream waits on
 * slot_free_event (may be NULL) before writing the slot and records
 * done_event after the last frame. */
int so_xc4_stream(void* slot, const void* pinned_unit, uint32_t frame_begin, uint32_t frame_end,
                  void* ring, size_t ring_slot_bytes, int ring_slots, void* const* ring_events,
                  uint64_t* ring_cursor, void* copy_stream, void* decode_stream, void* slot_free_event,
                  void* done_event);

#ifdef __cplusplus
}
#endif
#endif /* SPECOFFLOAD_B200_H */
