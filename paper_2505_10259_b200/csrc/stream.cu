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
