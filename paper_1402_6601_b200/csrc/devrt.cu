// Device plumbing of the online (XKaapi-style) executor behind the C-ABI:
// slot allocation, per-worker streams, events (completion polling and kernel
// timing), async H2D / peer copies and status words.  online.py drives the
// reference's event loop (sim.py:140-203) and binds these through ctypes, so
// its data path is this library, not torch.
//
// Handles are opaque pointers (cudaStream_t / cudaEvent_t / device pointers);
// every call selects its device first, so the host loop may interleave GPUs.
#include <cuda_runtime.h>

#include "hetgpu.h"
#include "tiles.h"

using hg::set_error;

#define HG_RT(call)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      set_error("%s failed: %s", #call, cudaGetErrorString(e_));                           \
      cudaGetLastError();                                                                  \
      return HG_ECUDA;                                                                     \
    }                                                                                      \
  } while (0)

static int check_device(int32_t device) {
  int n = 0;
  HG_RT(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) {
    set_error("device id %d out of range (%d devices)", device, n);
    return HG_EINVAL;
  }
  HG_RT(cudaSetDevice(device));
  return HG_OK;
}

extern "C" {

int hg_dev_alloc(int32_t device, size_t bytes, void** out) {
  if (!out) {
    set_error("hg_dev_alloc: null out");
    return HG_EINVAL;
  }
  *out = nullptr;
  if (int rc = check_device(device)) return rc;
  HG_RT(cudaMalloc(out, bytes ? bytes : 1));
  return HG_OK;
}

int hg_dev_free(int32_t device, void* ptr) {
  if (!ptr) return HG_OK;
  if (int rc = check_device(device)) return rc;
  HG_RT(cudaFree(ptr));
  return HG_OK;
}

int hg_dev_memset(int32_t device, void* ptr, int32_t value, size_t bytes, void* stream) {
  if (int rc = check_device(device)) return rc;
  HG_RT(cudaMemsetAsync(ptr, value, bytes, (cudaStream_t)stream));
  return HG_OK;
}

int hg_dev_enable_peer(int32_t device, int32_t peer) {
  if (device == peer) return HG_OK;
  if (int rc = check_device(device)) return rc;
  int can = 0;
  HG_RT(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can) {
    set_error("GPU %d cannot access GPU %d's memory (no peer route)", device, peer);
    return HG_EPEER;
  }
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return HG_OK;
  }
  HG_RT(e);
  return HG_OK;
}

int hg_stream_create(int32_t device, void** out) {
  if (!out) {
    set_error("hg_stream_create: null out");
    return HG_EINVAL;
  }
  if (int rc = check_device(device)) return rc;
  cudaStream_t s;
  HG_RT(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *out = s;
  return HG_OK;
}

int hg_stream_destroy(int32_t device, void* stream) {
  if (!stream) return HG_OK;
  if (int rc = check_device(device)) return rc;
  HG_RT(cudaStreamDestroy((cudaStream_t)stream));
  return HG_OK;
}

int hg_stream_wait_event(void* stream, void* event) {
  HG_RT(cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)event, 0));
  return HG_OK;
}

int hg_event_create(int32_t device, int32_t timing, void** out) {
  if (!out) {
    set_error("hg_event_create: null out");
    return HG_EINVAL;
  }
  if (int rc = check_device(device)) return rc;
  cudaEvent_t e;
  HG_RT(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  *out = e;
  return HG_OK;
}

int hg_event_destroy(int32_t device, void* event) {
  if (!event) return HG_OK;
  if (int rc = check_device(device)) return rc;
  HG_RT(cudaEventDestroy((cudaEvent_t)event));
  return HG_OK;
}

int hg_event_record(void* event, void* stream) {
  HG_RT(cudaEventRecord((cudaEvent_t)event, (cudaStream_t)stream));
  return HG_OK;
}

/* 1: every work captured by the event is done; 0: not yet */
int hg_event_query(void* event) {
  cudaError_t e = cudaEventQuery((cudaEvent_t)event);
  if (e == cudaSuccess) return 1;
  if (e == cudaErrorNotReady) {
    cudaGetLastError();
    return 0;
  }
  set_error("cudaEventQuery: %s", cudaGetErrorString(e));
  cudaGetLastError();
  return HG_ECUDA;
}

int hg_event_elapsed_ms(void* start, void* end, float* ms) {
  HG_RT(cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)end));
  return HG_OK;
}

/* dst <- src (bytes) on `stream` of `device`; host <-> device or device <-> device
 * (UVA: a peer source needs hg_dev_enable_peer(device, peer) first).  Async with
 * respect to the host when the host side is page-locked (hg_matrix_register). */
int hg_copy_async(int32_t device, void* dst, const void* src, size_t bytes, void* stream) {
  if (!dst || !src) {
    set_error("hg_copy_async: null pointer");
    return HG_EINVAL;
  }
  if (int rc = check_device(device)) return rc;
  HG_RT(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream));
  return HG_OK;
}

int hg_dev_sync(int32_t device) {
  if (int rc = check_device(device)) return rc;
  HG_RT(cudaDeviceSynchronize());
  return HG_OK;
}

}  // extern "C"
