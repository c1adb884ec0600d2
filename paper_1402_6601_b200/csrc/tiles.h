// Tile-kernel launch descriptors shared by the per-kind entry points
// (hg_tile_run) and the CUDA-graph executor (runtime.cu).
//
// A task of the DAG maps to a short sequence of kernel launches ("steps").
// Every kernel takes ONE by-value parameter struct, so a launch is fully
// described by (function, grid, block, dynamic smem, parameter bytes) and can
// be either launched on a stream or added to a cudaGraph as a kernel node.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <vector>

namespace hg {

constexpr int kParamBytes = 512;

// Producer-push fusion: at most this many (consumer GPU, output block) pairs receive a
// task's output straight from the producing kernel (peer stores), see PushList / runtime.cu.
constexpr int kMaxPush = 8;

// Destinations of a pushed output: the same block's slot on up to kMaxPush other GPUs
// (peer / IPC-mapped pointers; same layout as the local slot).  The runtime fills dst and op
// (index of the written operand in TaskOperands::t); the kind's launch builder resolves src
// (the local slot of that operand) and len (doubles per slot: the tile, plus the side area for
// the LU / QR panel kinds, whose consumers read the dL / IPIV / T factors from it).
struct PushList {
  double* dst[kMaxPush];
  const double* src[kMaxPush];
  unsigned char op[kMaxPush];
  int n;
  int len;
};

struct LaunchDesc {
  const void* func = nullptr;
  dim3 grid, block;
  unsigned smem = 0;
  alignas(64) unsigned char params[kParamBytes];
  template <class P>
  void set(const void* f, dim3 g, dim3 b, unsigned sm, const P& p) {
    static_assert(sizeof(P) <= kParamBytes, "param struct too large");
    func = f; grid = g; block = b; smem = sm;
    memset(params, 0, sizeof(params));
    memcpy(params, &p, sizeof(P));
  }
};

// Operands of one tile task: tile pointers in the order of the task's
// accesses (kernels.py access lists), each tile nb x nb column-major with
// ld = nb, followed (LU/QR only) by its side area (T / dL panel + IPIV).
struct TaskOperands {
  double* t[4] = {nullptr, nullptr, nullptr, nullptr};
  int n_t = 0;
  int nb = 0;
  int ib = 0;
  int* status = nullptr;  // device word; kernels OR error bits into it
  int* scratch = nullptr; // per-task device ints (task_scratch_ints), zero-initialised once;
                          // kernels keep them self-consistent across runs
  PushList push{};        // producer-push: where the written tile also goes (kinds with push support)
  int side = 0;           // doubles of a tile's side area (LU / QR), the slot is nb*nb + side
};

// Kinds whose kernels can push their output tiles to consumer GPUs in the epilogue: the
// Cholesky kinds (the store epilogue), the LU / QR trailing updates (each strip CTA pushes its
// columns once its last L2 reduction landed) and the LU / QR panels (the task's last panel
// kernel pushes the whole slots after its final cluster barrier).  LU only on the ib = 128
// kernels (the sub-panel cluster and the strip apply).
inline bool kind_can_push(int kind, int nb, int ib) {
  if (kind >= 0 && kind <= 3) return true;                          // POTRF, TRSM, SYRK, GEMM
  if (kind >= 4 && kind <= 7) return ib == 128 && nb % 128 == 0;    // GETRF_INC, GESSM, TSTRF, SSSSM
  return kind >= 8 && kind <= 11;                                   // GEQRT, UNMQR, TSQRT, TSMQR
}

// The task's push list with src / len resolved: whole slots (tile + side) or tiles only.
inline PushList resolve_push(const TaskOperands& o, bool whole_slots) {
  PushList pl = o.push;
  for (int q = 0; q < pl.n; ++q) pl.src[q] = o.t[pl.op[q]];
  pl.len = o.nb * o.nb + (whole_slots ? o.side : 0);
  return pl;
}

// Device ints of per-task scratch a kind needs (0 for most kinds).
int task_scratch_ints(int kind, int nb, int ib);

// Kind ids == index in kernels.ALL_KINDS == HG_KIND_* in include/hetgpu.h
enum Kind {
  K_POTRF = 0, K_TRSM, K_SYRK, K_GEMM,
  K_GETRF_INC, K_GESSM, K_TSTRF, K_SSSSM,
  K_GEQRT, K_UNMQR, K_TSQRT, K_TSMQR,
  K_COUNT
};

// Appends the launches of one task. Returns false on unsupported kind /
// geometry (message via set_error).
bool build_task_launches(int kind, const TaskOperands& ops, std::vector<LaunchDesc>& out);

// Runs once per process: raises dynamic-smem limits of the kernels.
bool init_kernel_attributes();

void set_error(const char* fmt, ...);

}  // namespace hg
