// FP64 peak + DMMA tile-GEMM microbenchmark (run under gpurun).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I paper_1402_6601_b200/csrc tools/microbench.cu -o tools/microbench
// Prints one JSON object per measurement.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "dgemm_dmma.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void dmma_peak(double* out, int iters) {
  double c[16][2];
  for (int i = 0; i < 16; ++i) c[i][0] = c[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) hg::dmma_8x8x4(c[i][0], c[i][1], a, b);
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_peak(double* out, int iters) {
  double c[16];
  for (int i = 0; i < 16; ++i) c[i] = threadIdx.x;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

template <class Cfg, int MINB = 1>
__global__ void __launch_bounds__(Cfg::THREADS, MINB) gemm_nt_bench_nd(const double* A, const double* B, double* C, int nb) {
  extern __shared__ double smem[];
  size_t off = size_t(blockIdx.z) * nb * nb;
  const double* a = A + off; const double* b = B + off; double* c = C + off;
  int m0 = blockIdx.x * Cfg::BM, n0 = blockIdx.y * Cfg::BN;
  double acc[Cfg::FM][Cfg::FN][2];
  hg::zero_acc<Cfg>(acc);
  hg::TileLoader<Cfg, hg::M_MAJOR, Cfg::BM> la{a, nb, m0};
  hg::TileLoader<Cfg, hg::M_MAJOR, Cfg::BN> lb{b, nb, n0};
  hg::gemm_mainloop_nd<Cfg>(acc, smem, la, lb, 0, nb);
  hg::sub_store<Cfg>(acc, c, nb, m0, n0);
}

template <class Cfg, int MINB = 1>
__global__ void __launch_bounds__(Cfg::THREADS, MINB) gemm_nt_bench_mb(const double* A, const double* B, double* C, int nb) {
  extern __shared__ double smem[];
  size_t off = size_t(blockIdx.z) * nb * nb;
  const double* a = A + off; const double* b = B + off; double* c = C + off;
  int m0 = blockIdx.x * Cfg::BM, n0 = blockIdx.y * Cfg::BN;
  double acc[Cfg::FM][Cfg::FN][2];
  hg::zero_acc<Cfg>(acc);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + hg::GemmSmem<Cfg, hg::M_MAJOR, hg::M_MAJOR>::DOUBLES);
  hg::gemm_mainloop_mb<Cfg>(acc, smem, bars, a, nb, m0, b, nb, n0, 0, nb);
  hg::sub_store<Cfg>(acc, c, nb, m0, n0);
}

template <class Cfg, int MINB = 1>
__global__ void __launch_bounds__(Cfg::THREADS, MINB) gemm_nt_bench(const double* A, const double* B, double* C, int nb) {
  extern __shared__ double smem[];
  size_t off = size_t(blockIdx.z) * nb * nb;
  const double* a = A + off; const double* b = B + off; double* c = C + off;
  int m0 = blockIdx.x * Cfg::BM, n0 = blockIdx.y * Cfg::BN;
  double acc[Cfg::FM][Cfg::FN][2];
  hg::zero_acc<Cfg>(acc);
  hg::TileLoader<Cfg, hg::M_MAJOR, Cfg::BM> la{a, nb, m0};
  hg::TileLoader<Cfg, hg::M_MAJOR, Cfg::BN> lb{b, nb, n0};
  hg::gemm_mainloop<Cfg>(acc, smem, la, lb, 0, nb);
  hg::sub_store<Cfg>(acc, c, nb, m0, n0);
}

__global__ void gemm_nt_ref(const double* A, const double* B, double* C, int nb) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i >= nb) return;
  double s = 0;
  for (int k = 0; k < nb; ++k) s += A[size_t(k) * nb + i] * B[size_t(k) * nb + j];
  C[size_t(j) * nb + i] -= s;
}

__global__ void fill(double* p, size_t n, unsigned seed) {
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  if (i < n) {
    unsigned x = (unsigned)(i * 2654435761u) ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = (x & 0xffffff) / double(0x1000000) - 0.5;
  }
}

template <class Cfg, int MINB = 1, int ND = 0>
void bench_cfg(const char* name, int nb, int batch) {
  auto kern = ND == 2 ? gemm_nt_bench_mb<Cfg, MINB> : (ND ? gemm_nt_bench_nd<Cfg, MINB> : gemm_nt_bench<Cfg, MINB>);
  size_t n = size_t(nb) * nb * batch;
  double *A, *B, *C, *R;
  CK(cudaMalloc(&A, n * 8)); CK(cudaMalloc(&B, n * 8)); CK(cudaMalloc(&C, n * 8)); CK(cudaMalloc(&R, n * 8));
  fill<<<(n + 255) / 256, 256>>>(A, n, 1); fill<<<(n + 255) / 256, 256>>>(B, n, 2);
  fill<<<(n + 255) / 256, 256>>>(C, n, 3); CK(cudaMemcpy(R, C, n * 8, cudaMemcpyDeviceToDevice));
  size_t smem = hg::GemmSmem<Cfg, hg::M_MAJOR, hg::M_MAJOR>::BYTES + (ND == 2 ? 2 * Cfg::STAGES * 8 : 0);
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(nb / Cfg::BM, nb / Cfg::BN, batch);
  kern<<<grid, Cfg::THREADS, smem>>>(A, B, C, nb);
  CK(cudaGetLastError());
  // correctness on batch 0 only
  gemm_nt_ref<<<dim3((nb + 127) / 128, nb), 128>>>(A, B, R, nb);
  CK(cudaDeviceSynchronize());
  std::vector<double> hc(size_t(nb) * nb), hr(size_t(nb) * nb);
  CK(cudaMemcpy(hc.data(), C, hc.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hr.data(), R, hr.size() * 8, cudaMemcpyDeviceToHost));
  double md = 0, mx = 0;
  for (size_t i = 0; i < hc.size(); ++i) { md = fmax(md, fabs(hc[i] - hr[i])); mx = fmax(mx, fabs(hr[i])); }
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (int w = 0; w < 3; ++w) kern<<<grid, Cfg::THREADS, smem>>>(A, B, C, nb);
  int reps = 10;
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) kern<<<grid, Cfg::THREADS, smem>>>(A, B, C, nb);
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  double flops = 2.0 * nb * double(nb) * nb * batch * reps;
  printf("{\"bench\":\"gemm_nt\",\"cfg\":\"%s\",\"nb\":%d,\"batch\":%d,\"smem\":%zu,\"us_per_launch\":%.2f,\"tflops\":%.3f,\"max_abs_err\":%.3e,\"max_ref\":%.3e}\n",
         name, nb, batch, smem, ms * 1e3 / reps, flops / (ms * 1e-3) / 1e12, md, mx);
  CK(cudaFree(A)); CK(cudaFree(B)); CK(cudaFree(C)); CK(cudaFree(R));
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("{\"device\":\"%s\",\"sms\":%d,\"cc\":\"%d.%d\"}\n", p.name, p.multiProcessorCount, p.major, p.minor);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (int blocksPerSm : {1, 2, 4}) {
    int iters = 4096, threads = 256, blocks = p.multiProcessorCount * blocksPerSm;
    dmma_peak<<<blocks, threads>>>(out, 16);
    CK(cudaEventRecord(e0)); dmma_peak<<<blocks, threads>>>(out, iters); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1)); float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = double(blocks) * (threads / 32) * iters * 16 * 512.0;
    printf("{\"bench\":\"dmma_peak\",\"blocks_per_sm\":%d,\"tflops\":%.3f,\"ms\":%.3f}\n", blocksPerSm, flops / (ms * 1e-3) / 1e12, ms);
    dfma_peak<<<blocks, threads>>>(out, 16);
    CK(cudaEventRecord(e0)); dfma_peak<<<blocks, threads>>>(out, iters); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    flops = double(blocks) * threads * iters * 16 * 2.0;
    printf("{\"bench\":\"dfma_peak\",\"blocks_per_sm\":%d,\"tflops\":%.3f,\"ms\":%.3f}\n", blocksPerSm, flops / (ms * 1e-3) / 1e12, ms);
  }
  using C64 = hg::GemmCfg<64, 64, 16, 32, 32, 3>;
  using C64s4 = hg::GemmCfg<64, 64, 16, 32, 32, 4>;
  using C64k8s4 = hg::GemmCfg<64, 64, 8, 32, 32, 4>;
  using C64k8s3 = hg::GemmCfg<64, 64, 8, 32, 32, 3>;
  using C64k32s3 = hg::GemmCfg<64, 64, 32, 32, 32, 3>;
  for (int batch : {32}) {
    bench_cfg<C64, 4, 1>("ND_64x64x16_w32x32_s3_minb4", 1024, batch);
    bench_cfg<C64s4, 3, 1>("ND_64x64x16_w32x32_s4_minb3", 1024, batch);
    bench_cfg<C64, 4, 2>("MB_64x64x16_w32x32_s3_minb4", 1024, batch);
    bench_cfg<C64s4, 3, 2>("MB_64x64x16_w32x32_s4_minb3", 1024, batch);
    bench_cfg<C64k8s4, 4, 2>("MB_64x64x8_w32x32_s4_minb4", 1024, batch);
    bench_cfg<C64k32s3, 2, 2>("MB_64x64x32_w32x32_s3_minb2", 1024, batch);
  }
  return 0;
}
