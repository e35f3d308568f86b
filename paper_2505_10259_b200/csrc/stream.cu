// K1 — layer streamer: pinned host DRAM → HBM window slot on a copy stream.
//
// Replaces the modeled `ffn_load` C2G event (simulator.py:172-176; duration
// ffn_bytes / c2g_bandwidth, costmodel.py:74) with the copy itself.  The copy
// engine moves the bytes; no SMs are used, so the target's and the draft's
// kernels keep the whole GPU while the PCIe link streams.  Chunking keeps each
// DMA descriptor moderate (64–256 MiB) so a waiting stream can interleave and
// the completion event lands promptly.
#include "common.cuh"

extern "C" int so_stream_layer(void* slot, const void* pinned_src, size_t bytes, size_t chunk, void* stream,
                               void* done_event) {
  SO_REQUIRE(slot && pinned_src, SO_E_NULLPTR);
  if (chunk == 0) chunk = bytes;
  cudaStream_t st = as_stream(stream);
  const uint8_t* src = reinterpret_cast<const uint8_t*>(pinned_src);
  uint8_t* dst = reinterpret_cast<uint8_t*>(slot);
  for (size_t off = 0; off < bytes; off += chunk) {
    const size_t n = bytes - off < chunk ? bytes - off : chunk;
    cudaError_t e = cudaMemcpyAsync(dst + off, src + off, n, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return (int)e;
  }
  if (done_event != nullptr) {
    cudaError_t e = cudaEventRecord(reinterpret_cast<cudaEvent_t>(done_event), st);
    if (e != cudaSuccess) return (int)e;
  }
  return SO_OK;
}

extern "C" int so_abi_version(void) { return 1; }

extern "C" int so_set_device(int device) { return (int)cudaSetDevice(device); }

// ---- stream plumbing used inside the per-layer loops ---------------------
// These exist so the host layer never makes a potentially blocking stream
// call while holding the Python GIL: a full launch queue blocks the caller,
// and the verify and draft streams are fed from two host threads.

extern "C" int so_event_create(int timing, void** out_event) {
  SO_REQUIRE(out_event, SO_E_NULLPTR);
  cudaEvent_t e;
  cudaError_t r = cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming);
  *out_event = r == cudaSuccess ? reinterpret_cast<void*>(e) : nullptr;
  return (int)r;
}

extern "C" int so_event_destroy(void* event) {
  return event ? (int)cudaEventDestroy(reinterpret_cast<cudaEvent_t>(event)) : SO_OK;
}

extern "C" int so_event_record(void* event, void* stream) {
  SO_REQUIRE(event, SO_E_NULLPTR);
  return (int)cudaEventRecord(reinterpret_cast<cudaEvent_t>(event), as_stream(stream));
}

extern "C" int so_stream_wait_event(void* stream, void* event) {
  SO_REQUIRE(event, SO_E_NULLPTR);
  return (int)cudaStreamWaitEvent(as_stream(stream), reinterpret_cast<cudaEvent_t>(event), 0);
}

extern "C" int so_event_synchronize(void* event) {
  SO_REQUIRE(event, SO_E_NULLPTR);
  return (int)cudaEventSynchronize(reinterpret_cast<cudaEvent_t>(event));
}

extern "C" int so_event_elapsed_ms(void* start, void* end, float* ms) {
  SO_REQUIRE(start && end && ms, SO_E_NULLPTR);
  return (int)cudaEventElapsedTime(ms, reinterpret_cast<cudaEvent_t>(start), reinterpret_cast<cudaEvent_t>(end));
}

extern "C" int so_memcpy_async(void* dst, const void* src, size_t bytes, void* stream) {
  SO_REQUIRE(dst && src, SO_E_NULLPTR);
  if (bytes == 0) return SO_OK;
  return (int)cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, as_stream(stream));
}

extern "C" int so_stream_synchronize(void* stream) { return (int)cudaStreamSynchronize(as_stream(stream)); }

// Non-blocking status probes (0 = all work done, 600 = cudaErrorNotReady):
// diagnostics of a stalled pipeline read which stream / event is pending.
extern "C" int so_stream_query(void* stream) { return (int)cudaStreamQuery(as_stream(stream)); }

extern "C" int so_event_query(void* event) {
  SO_REQUIRE(event, SO_E_NULLPTR);
  return (int)cudaEventQuery(reinterpret_cast<cudaEvent_t>(event));
}

// Small host↔device transfers executed by SMs over UVA (zero-copy) instead of
// the copy engine.  The H2D copy engine is busy streaming 4.8 GB layers whose
// copies are gated on the verify's slot releases; a metadata copy queued
// behind them on the same engine would stall the draft stream for a whole
// layer.  Pinned host memory is device-addressable under UVA, so a kernel
// moves the few KB directly.
namespace {
__global__ void copy_sm_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, size_t bytes) {
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  size_t done = 0;
  if (vec) {
    const size_t n16 = bytes / 16;
    for (size_t i = tid; i < n16; i += stride)
      reinterpret_cast<int4*>(dst)[i] = reinterpret_cast<const int4*>(src)[i];
    done = n16 * 16;
  }
  for (size_t i = done + tid; i < bytes; i += stride) dst[i] = src[i];
}
}  // namespace

extern "C" int so_copy_sm(void* dst, const void* src, size_t bytes, void* stream) {
  SO_REQUIRE(dst && src, SO_E_NULLPTR);
  if (bytes == 0) return SO_OK;
  size_t blocks = (bytes / 16 + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 64) blocks = 64;
  copy_sm_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(reinterpret_cast<uint8_t*>(dst),
                                                                   reinterpret_cast<const uint8_t*>(src), bytes);
  SO_CHECK_LAUNCH();
  return SO_OK;
}

extern "C" const char* so_status_string(int status) {
  switch (status) {
    case SO_OK: return "ok";
    case SO_E_NULLPTR: return "null pointer argument";
    case SO_E_SHAPE: return "invalid shape or size argument";
    case SO_E_ALIGN: return "pointer not 16-byte aligned";
    case SO_E_UNSUPPORTED: return "unsupported configuration";
    case SO_E_DRIVER: return "CUDA driver entry point unavailable";
    default: break;
  }
  if (status > 0) return cudaGetErrorString(static_cast<cudaError_t>(status));
  return "unknown status";
}
