// Micro-timing of the POTRF building blocks (clock64 inside one CTA / one cluster).
//   nvcc ... -I paper_1402_6601_b200/csrc tools/potrf_micro.cu -o tools/potrf_micro
#include <cstdio>
#include <vector>
#include "../paper_1402_6601_b200/csrc/tiles_chol.cu"

namespace hg {
void set_error(const char*, ...) {}
}
using namespace hg;

__global__ void __launch_bounds__(128) k_time_diag(double* A, int ld, long long* out, int reps, int* st) {
  extern __shared__ double sm[];
  auto s = reinterpret_cast<double(*)[kR + 1]>(sm);
  auto iv = reinterpret_cast<double(*)[kR + 1]>(sm + kR * (kR + 1));
  auto tm = reinterpret_cast<double(*)[33]>(sm + 2 * kR * (kR + 1));
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) diag64_blocked(A, ld, 0, st, &s[0][0]);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / reps;
}

__global__ void __launch_bounds__(128) k_time_leaf(double* A, int ld, long long* out, int reps, int* st) {
  extern __shared__ double sm[];
  auto s = reinterpret_cast<double(*)[kR + 1]>(sm);
  auto iv = reinterpret_cast<double(*)[kR + 1]>(sm + kR * (kR + 1));
  for (int e = threadIdx.x; e < kR * kR; e += 128) s[e / kR][e % kR] = A[(e / kR) * ld + e % kR];
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x < 32) leaf32(&s[0][0], kR + 1, 0, &iv[0][0], kR + 1, st);
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[1] = (t1 - t0) / reps;
}

__global__ void __launch_bounds__(128) k_time_leaf16(double* A, int ld, long long* out, int reps, int* st) {
  extern __shared__ double sm[];
  for (int e = threadIdx.x; e < kR * kBL; e += 128) sm[e] = (e % kBL == e / kBL) ? 64.0 : 0.001;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x < 32) leaf16(sm, 0, sm + 2 * kR * kBL);
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[5] = (t1 - t0) / reps;
}

__global__ void __launch_bounds__(128) k_time_update(double* A, int ld, long long* out, int reps) {
  extern __shared__ double sm[];
  TileLoader<CfgG, M_MAJOR, kR> la{A, ld, 64};
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) block_update(A + 2 * 64 * ld + 128, ld, la, la, false, false, sm);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[2] = (t1 - t0) / reps;
}

__global__ void __launch_bounds__(128) k_time_apply(double* A, int ld, long long* out, int reps) {
  extern __shared__ double sm[];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) apply_inv_right(A + 128, ld, A, sm);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[3] = (t1 - t0) / reps;
}

__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(128) k_time_cluster(long long* out, int reps) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    __threadfence();
    cl.sync();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[4] = (t1 - t0) / reps;
}

int main() {
  const int nb = 1024;
  std::vector<double> h(size_t(nb) * nb);
  for (int j = 0; j < nb; ++j)
    for (int i = 0; i < nb; ++i) h[size_t(j) * nb + i] = (i == j ? nb : 0.0) + 0.001 * ((i * 7 + j * 13) % 17) / 17.0;
  double* A;
  long long* out;
  int* st;
  cudaMalloc(&A, h.size() * 8);
  cudaMalloc(&out, 8 * 8);
  cudaMalloc(&st, 4);
  cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  const int smem = (2 * kR * kBL + 16 * 17) * 8;
  cudaFuncSetAttribute(k_time_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_time_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_time_update, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k_time_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k_time_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  k_time_diag<<<1, 128, smem>>>(A, nb, out, 20, st);
  k_time_leaf<<<1, 128, smem>>>(A, nb, out, 20, st);
  cudaFuncSetAttribute(k_time_leaf16, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_time_leaf16<<<1, 128, smem>>>(A, nb, out, 20, st);
  k_time_update<<<1, 128, 100000>>>(A, nb, out, 50);
  k_time_apply<<<1, 128, 100000>>>(A, nb, out, 50);
  k_time_cluster<<<16, 128>>>(out, 200);
  cudaError_t e = cudaDeviceSynchronize();
  long long r[8];
  cudaMemcpy(r, out, sizeof(r), cudaMemcpyDeviceToHost);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double mhz = clk / 1000.0;
  printf("{\"err\":\"%s\",\"mhz\":%.0f,\"diag64_cycles\":%lld,\"leaf32_cycles\":%lld,\"block_update_cycles\":%lld,"
         "\"apply_inv_cycles\":%lld,\"cluster_sync_cycles\":%lld,\"leaf16_cycles\":%lld}\n",
         cudaGetErrorString(e), mhz, r[0], r[1], r[2], r[3], r[4], r[5]);
  printf("{\"diag64_us\":%.2f,\"leaf32_us\":%.2f,\"block_update_us\":%.2f,\"apply_inv_us\":%.2f,\"cluster_sync_us\":%.3f}\n",
         r[0] / mhz, r[1] / mhz, r[2] / mhz, r[3] / mhz, r[4] / mhz);
  return 0;
}
