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

constexpr int kParamBytes = 160;

// Producer-push fusion: at most this many consumer GPUs receive a task's output tile
// straight from the producing kernel (peer stores), see PushList / runtime.cu.
constexpr int kMaxPush = 7;

// Destinations of a pushed output tile: the same block's slot on up to kMaxPush other GPUs
// (peer / IPC-mapped pointers; same nb x nb column-major layout as the local tile).
struct PushList {
  double* dst[kMaxPush];
  int n;
};

struct LaunchDesc {
  const void* func = nullptr;
  dim3 grid, block;
  unsigned smem = 0;
  alignas(16) unsigned char params[kParamBytes];
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
};

// Kinds whose kernels can push their output tile to consumer GPUs in the epilogue.
inline bool kind_can_push(int kind) { return kind >= 0 && kind <= 3; }  // POTRF, TRSM, SYRK, GEMM

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
