// Shared device helpers for the hetgpu tile kernels (sm_100a).
//
// FP64 tensor math on sm_100a is warp-level DMMA only: `tcgen05.mma` has no
// f64 kind (ptxas rejects it), while `mma.sync.aligned.m8n8k4.row.col.f64`
// lowers to SASS `DMMA.8x8x4`.  Every dense trailing update in this library
// (GEMM, SYRK, SSSSM, TSMQR and the blocked parts of TRSM/GESSM/UNMQR) is
// built on the 8x8x4 fragment below, fed from shared memory staged by
// cp.async (LDGSTS).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define HG_DEVICE __device__ __forceinline__

namespace hg {

// Fragment ownership of mma.m8n8k4.f64 (g = lane>>2, t = lane&3):
//   A (8x4, row):  a = A[g][t]
//   B (4x8, col):  b = B[t][g]
//   C (8x8):       c0 = C[g][2t], c1 = C[g][2t+1]
// (not volatile: a pure function of its operands, so the compiler may hoist the
// next k-step's fragment loads above it)
HG_DEVICE void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 "
      "{%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

HG_DEVICE void cp_async16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
HG_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
HG_DEVICE void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// C += v as a fire-and-forget reduction performed at L2 (no load round trip to
// the SM).  fl(c + (-a)) == fl(c - a), so "red(-acc)" is bit-identical to the
// read-modify-write "c = c - acc" when one thread owns the element.
HG_DEVICE void red_add_f64(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;\n" ::"l"(p), "d"(v) : "memory");
}

HG_DEVICE double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace hg
