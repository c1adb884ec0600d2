// FP64 peak probe (roofline denominator): DMMA and DFMA issue-bound kernels.
#include <cuda_runtime.h>
#include "../../include/hetgpu.h"
#include "hg_common.cuh"

namespace hg {
void set_error(const char* fmt, ...);

__global__ void __launch_bounds__(256) k_dmma_peak(double* out, int iters) {
  double c[16][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i][0] = c[i][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) dmma_8x8x4(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters) {
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = threadIdx.x;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 1234.5) out[0] = s;
}
}  // namespace hg

extern "C" int hg_fp64_peak(int32_t device, double* dmma_tflops, double* dfma_tflops) {
  using namespace hg;
  if (cudaSetDevice(device) != cudaSuccess) {
    set_error("hg_fp64_peak: cudaSetDevice(%d) failed", device);
    return HG_ECUDA;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  cudaEvent_t e0, e1;
  if (cudaMalloc(&out, 8) != cudaSuccess || cudaEventCreate(&e0) != cudaSuccess ||
      cudaEventCreate(&e1) != cudaSuccess) {
    set_error("hg_fp64_peak: allocation failed");
    return HG_ECUDA;
  }
  const int blocks = sms * 4, threads = 256, iters = 4096;
  float ms = 0.f;
  double best_dmma = 0, best_dfma = 0;
  k_dmma_peak<<<blocks, threads>>>(out, 64);
  k_dfma_peak<<<blocks, threads>>>(out, 64);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k_dmma_peak<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double f = double(blocks) * (threads / 32) * iters * 16 * 512.0;
    best_dmma = fmax(best_dmma, f / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0);
    k_dfma_peak<<<blocks, threads>>>(out, iters / 4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    f = double(blocks) * threads * (iters / 4) * 16 * 2.0;
    best_dfma = fmax(best_dfma, f / (ms * 1e-3) / 1e12);
  }
  cudaError_t err = cudaGetLastError();
  cudaFree(out);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (err != cudaSuccess) {
    set_error("hg_fp64_peak: %s", cudaGetErrorString(err));
    return HG_ECUDA;
  }
  if (dmma_tflops) *dmma_tflops = best_dmma;
  if (dfma_tflops) *dfma_tflops = best_dfma;
  return HG_OK;
}
