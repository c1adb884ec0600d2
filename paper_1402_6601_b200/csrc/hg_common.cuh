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
#ifdef HG_EXP_RED_AS_STORE  // tools/ssssm_ab.cu timing experiment only (wrong results)
  asm volatile("st.global.cg.f64 [%0], %1;\n" ::"l"(p), "d"(v) : "memory");
#else
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;\n" ::"l"(p), "d"(v) : "memory");
#endif
}

// ---- mbarrier + bulk-copy (TMA engine, no tensor map) helpers --------------
HG_DEVICE unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
HG_DEVICE void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
HG_DEVICE void mbar_arrive(uint64_t* b) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(b)) : "memory");
}
HG_DEVICE void mbar_arrive_tx(uint64_t* b, unsigned bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
HG_DEVICE void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy on the TMA engine, completion counted on mbarrier b
// (16-byte aligned addresses, bytes % 16 == 0)
HG_DEVICE void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}

// 2-D tensor-map TMA load (cp.async.bulk.tensor, SASS UTMALDG) of the box at coordinates
// (c0 = inner / row, c1 = outer / column) into dense shared memory; `tmap` is the generic
// address of a CUtensorMap in parameter (__grid_constant__) or global memory.
HG_DEVICE void tma_load_2d(void* dst, const void* tmap, int c0, int c1, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem_u32(b))
      : "memory");
}
// generic-proxy accesses of shared memory before this are ordered before later async-proxy ones (TMA writes)
HG_DEVICE void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// ---- cluster push messages: remote shared-memory stores that complete on the
// receiver's mbarrier (no cluster barrier, no release fence over global memory) ----
// shared::cluster address of `p` (this CTA's smem) in CTA `rank` of the cluster
HG_DEVICE unsigned cluster_addr(const void* p, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// 8-byte store into another CTA's smem, counted (8 bytes) on that CTA's mbarrier
HG_DEVICE void st_async_f64(unsigned remote_addr, double v, unsigned remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(remote_addr),
               "d"(v), "r"(remote_bar)
               : "memory");
}
HG_DEVICE void st_async_v2f64(unsigned remote_addr, double a, double b, unsigned remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(
                   remote_addr),
               "d"(a), "d"(b), "r"(remote_bar)
               : "memory");
}
// wait for phase `parity` of a local mbarrier whose bytes arrive from other CTAs
HG_DEVICE void mbar_wait_cluster(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
HG_DEVICE void fence_mbar_init_cluster() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

// Phase timestamps of the panel kernels for tools/panel_stamps.cu (built with -DHG_PANEL_STAMPS;
// the product build compiles them out): g_panel_stamps[cta][k] = %globaltimer of thread 0 of CTA q.
#ifdef HG_PANEL_STAMPS
__device__ unsigned long long g_panel_stamps[16][512];
#define HG_STAMP(k)                                                  \
  do {                                                               \
    if (threadIdx.x == 0 && (q) >= 0) {                              \
      unsigned long long t_;                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));         \
      ::hg::g_panel_stamps[q][(k)] = t_;                             \
    }                                                                \
  } while (0)
#else
#define HG_STAMP(k) \
  do {              \
  } while (0)
#endif

HG_DEVICE double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace hg
