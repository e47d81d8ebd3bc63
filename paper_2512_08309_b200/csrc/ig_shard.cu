// Halo exchange plumbing for the sharded world plane:
// packing a rank's outgoing boundary windows into its exported buffer with
// one launch, and cross-process CUDA events so a consumer's blend is ordered
// after the producer's pack on the DEVICE (no host synchronisation per step).
#include <cstring>

#include "ig_common.cuh"

namespace ig {

// Copies n windows of `words` 16-byte words each from arbitrary device
// addresses (src[k]) into consecutive slots of dst.  grid.y walks windows,
// grid.x strides over one window's words.
__global__ void __launch_bounds__(256) pack_windows_kernel(const int64_t* __restrict__ src,
                                                           int n, int64_t words,
                                                           int4* __restrict__ dst) {
  for (int k = blockIdx.y; k < n; k += gridDim.y) {
    const int4* s = reinterpret_cast<const int4*>(src[k]);
    int4* d = dst + (int64_t)k * words;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < words;
         i += (int64_t)gridDim.x * blockDim.x)
      d[i] = __ldg(s + i);
  }
}

}  // namespace ig

using namespace ig;

extern "C" {

int ig_pack_windows(const int64_t* src_ptrs, int32_t n, int64_t window_bytes, void* dst,
                    void* cuda_stream) {
  IG_REQUIRE(n >= 0 && window_bytes > 0 && window_bytes % 16 == 0,
             "pack_windows: window size %lld must be a positive multiple of 16 bytes",
             (long long)window_bytes);
  if (n == 0) return IG_OK;
  const int64_t words = window_bytes / 16;
  const int bx = (int)((words + 255) / 256 < 64 ? (words + 255) / 256 : 64);
  const dim3 grid((unsigned)bx, (unsigned)(n < 65535 ? n : 65535));
  pack_windows_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(cuda_stream)>>>(
      src_ptrs, n, words, reinterpret_cast<int4*>(dst));
  note_launch();
  return cuda_check("ig_pack_windows");
}

static int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return IG_OK;
  set_error("%s: %s", what, cudaGetErrorString(e));
  return IG_ERR_CUDA;
}

int ig_ipc_event_create(uint8_t* handle64, void** event_out) {
  IG_REQUIRE(handle64 != nullptr && event_out != nullptr, "ipc_event_create: null argument");
  cudaEvent_t ev;
  int rc = cuda_status(
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming | cudaEventInterprocess),
      "ipc_event_create: cudaEventCreateWithFlags");
  if (rc != IG_OK) return rc;
  cudaIpcEventHandle_t h;
  rc = cuda_status(cudaIpcGetEventHandle(&h, ev), "ipc_event_create: cudaIpcGetEventHandle");
  if (rc != IG_OK) {
    cudaEventDestroy(ev);
    return rc;
  }
  static_assert(sizeof(h) == 64, "cudaIpcEventHandle_t is 64 bytes");
  memcpy(handle64, &h, 64);
  *event_out = ev;
  return IG_OK;
}

int ig_ipc_event_open(const uint8_t* handle64, void** event_out) {
  IG_REQUIRE(handle64 != nullptr && event_out != nullptr, "ipc_event_open: null argument");
  cudaIpcEventHandle_t h;
  memcpy(&h, handle64, 64);
  cudaEvent_t ev;
  const int rc = cuda_status(cudaIpcOpenEventHandle(&ev, h), "ipc_event_open");
  if (rc == IG_OK) *event_out = ev;
  return rc;
}

int ig_event_record(void* event, void* cuda_stream) {
  return cuda_status(cudaEventRecord(reinterpret_cast<cudaEvent_t>(event),
                                     reinterpret_cast<cudaStream_t>(cuda_stream)),
                     "event_record");
}

int ig_stream_wait_event(void* cuda_stream, void* event) {
  return cuda_status(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(cuda_stream),
                                         reinterpret_cast<cudaEvent_t>(event), 0),
                     "stream_wait_event");
}

int ig_event_destroy(void* event) {
  return cuda_status(cudaEventDestroy(reinterpret_cast<cudaEvent_t>(event)), "event_destroy");
}

}  // extern "C"
