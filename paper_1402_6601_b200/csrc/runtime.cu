// Executor of a planned tile DAG on B200s (replaces the simulated execution
// of /root/reference/pkg/src/hetsim/sim.py:237-385).
//
// The whole plan becomes ONE CUDA graph:
//   * every transfer job of the plan (sim.py:242-267) is a copy node moving
//     the job's block version from its source node to its destination GPU
//     (H2D from the host image, or peer D2D over NVLink/NVSwitch);
//   * every task is a short chain of sm_100a tile-kernel nodes
//     (tiles_chol.cu, tiles_lu.cu, tiles_qr.cu) reading/writing the task's
//     tiles in the destination GPU's slot pool;
//   * edges: job <- the task that wrote the version (or the job that brought
//     it to the source node); task <- its jobs and all its DAG predecessors.
//     Waiting on every predecessor also orders the WAR / WAW hazards on a
//     GPU's single slot per block (a writer depends on all readers of the
//     previous version, and each reader started only after its own copy).
// Independent branches run concurrently (several tile kernels per GPU at
// once), which fills 148 SMs with 64-CTA tile kernels without changing the
// plan's task->GPU map or its transfer list.
#include <cuda_runtime.h>
#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <unordered_map>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hetgpu.h"
#include "tiles.h"

namespace hg {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

bool init_chol_attributes();
bool build_chol_launches(int kind, const TaskOperands& o, std::vector<LaunchDesc>& out);
bool init_lu_attributes();
bool build_lu_launches(int kind, const TaskOperands& o, std::vector<LaunchDesc>& out);
bool init_qr_attributes();
bool build_qr_launches(int kind, const TaskOperands& o, std::vector<LaunchDesc>& out);

int chol_scratch_ints(int kind, int nb);

int task_scratch_ints(int kind, int nb, int ib) {
  (void)ib;
  if (kind >= K_POTRF && kind <= K_GEMM) return chol_scratch_ints(kind, nb);
  return 0;
}

bool init_kernel_attributes() {
  return init_chol_attributes() && init_lu_attributes() && init_qr_attributes();
}

bool build_task_launches(int kind, const TaskOperands& ops, std::vector<LaunchDesc>& out) {
  if (kind >= K_POTRF && kind <= K_GEMM) return build_chol_launches(kind, ops, out);
  if (kind >= K_GETRF_INC && kind <= K_SSSSM) return build_lu_launches(kind, ops, out);
  if (kind >= K_GEQRT && kind <= K_TSMQR) return build_qr_launches(kind, ops, out);
  set_error("unknown kernel kind %d", kind);
  return false;
}

}  // namespace hg

using namespace hg;

#define HG_CUDA(call)                                                               \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return HG_ECUDA;                                                              \
    }                                                                               \
  } while (0)

static std::once_flag g_attr_once[64];
static bool g_attr_ok[64];
static std::string g_attr_msg[64];

static int ensure_attributes(int dev) {
  if (dev < 0 || dev >= 64) {
    set_error("device id %d out of range", dev);
    return HG_EINVAL;
  }
  std::call_once(g_attr_once[dev], [dev] {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
    g_attr_ok[dev] = init_kernel_attributes();
    if (!g_attr_ok[dev]) g_attr_msg[dev] = g_err;
    cudaSetDevice(prev);
  });
  if (!g_attr_ok[dev]) {
    set_error("kernel attribute setup failed on device %d: %s", dev, g_attr_msg[dev].c_str());
    return HG_ECUDA;
  }
  return HG_OK;
}

extern "C" {

const char* hg_last_error(void) { return g_err.c_str(); }
int hg_abi_version(void) { return HG_ABI_VERSION; }

int hg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int hg_tile_run(int32_t kind, int32_t device, void* stream, double* const* t, int32_t n_t, int32_t nb,
                int32_t ib, int32_t* status_dev) {
  if (n_t < 1 || n_t > 4 || t == nullptr) {
    set_error("hg_tile_run: need 1..4 tile pointers");
    return HG_EINVAL;
  }
  HG_CUDA(cudaSetDevice(device));
  int rc = ensure_attributes(device);
  if (rc) return rc;
  TaskOperands ops;
  for (int i = 0; i < n_t; ++i) ops.t[i] = t[i];
  ops.n_t = n_t;
  ops.nb = nb;
  ops.ib = ib;
  ops.status = status_dev;
  // per-device scratch for hg_tile_run (flags are self-advancing; calls on one
  // device must not overlap in time)
  static int* scratch[64] = {nullptr};
  static std::mutex scratch_mu;
  const int need = task_scratch_ints(kind, nb, ib);
  if (need > 0) {
    std::lock_guard<std::mutex> lk(scratch_mu);
    if (!scratch[device]) {
      HG_CUDA(cudaMalloc(&scratch[device], size_t(1 << 16) * sizeof(int)));
      HG_CUDA(cudaMemset(scratch[device], 0, size_t(1 << 16) * sizeof(int)));
    }
    if (need > (1 << 16)) {
      set_error("hg_tile_run: scratch too small");
      return HG_EINVAL;
    }
    ops.scratch = scratch[device];
  }
  std::vector<LaunchDesc> launches;
  if (!build_task_launches(kind, ops, launches)) return HG_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (auto& d : launches) {
    void* args[1] = {d.params};
    HG_CUDA(cudaLaunchKernel(d.func, d.grid, d.block, args, d.smem, s));
  }
  return HG_OK;
}

// Same as hg_tile_run with caller-owned per-task scratch (hg_task_scratch_ints
// ints, zeroed once, self-consistent across runs), so independent tasks may run
// concurrently on different streams (the online executor).
int hg_tile_run_scratch(int32_t kind, int32_t device, void* stream, double* const* t, int32_t n_t, int32_t nb,
                        int32_t ib, int32_t* status_dev, int32_t* scratch_dev) {
  if (n_t < 1 || n_t > 4 || t == nullptr) {
    set_error("hg_tile_run_scratch: need 1..4 tile pointers");
    return HG_EINVAL;
  }
  HG_CUDA(cudaSetDevice(device));
  int rc = ensure_attributes(device);
  if (rc) return rc;
  TaskOperands ops;
  for (int i = 0; i < n_t; ++i) ops.t[i] = t[i];
  ops.n_t = n_t;
  ops.nb = nb;
  ops.ib = ib;
  ops.status = status_dev;
  if (task_scratch_ints(kind, nb, ib) > 0) {
    if (!scratch_dev) {
      set_error("hg_tile_run_scratch: kind %d needs %d scratch ints", kind, task_scratch_ints(kind, nb, ib));
      return HG_EINVAL;
    }
    ops.scratch = scratch_dev;
  }
  std::vector<LaunchDesc> launches;
  if (!build_task_launches(kind, ops, launches)) return HG_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (auto& d : launches) {
    void* args[1] = {d.params};
    HG_CUDA(cudaLaunchKernel(d.func, d.grid, d.block, args, d.smem, s));
  }
  return HG_OK;
}

int hg_task_scratch_ints(int32_t kind, int32_t nb, int32_t ib) { return task_scratch_ints(kind, nb, ib); }

}  // extern "C"

// ---------------------------------------------------------------------------
// Executor.  Two modes share one graph builder:
//  * single process (opts.rank_node == 0): every GPU node is local; one CUDA
//    graph spans all devices and cross-device ordering is plain graph edges;
//  * one process per GPU (opts.rank_node == r+1): the process builds only its
//    node's tasks and inbound copy jobs.  Peer slot pools are mapped with CUDA
//    IPC (hg_exec_ipc_handle / hg_exec_ipc_open), and every dependency that
//    crosses processes becomes a device flag in the producer's pool header:
//    the producer's graph ends the task/job with a release store of the run's
//    epoch, the consumer's graph waits for it with an acquire spin before the
//    copy / kernel that needs it.
// Pool layout per node: [flag header: int task_flag[n_tasks], job_flag[n_jobs],
// epoch; 256-byte aligned] [slots of every block the plan ever places there].

namespace hg {

__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// status bit of a cross-rank wait that gave up (-> HG_EDEADLOCK / DeadlockError)
constexpr int kStatusWaitTimeout = 4;

struct FlagParams {
  int* flag;
  const int* epoch;
  int* status;                    // this rank's status word (waits only)
  unsigned long long timeout_ns;  // waits only: give up after this long
};

// Bounded spin: a dead peer rank or a plan/partition mismatch would otherwise
// hang the device (the reference raises DeadlockError when no event is left,
// sim.py:24-29, 164-166).  On timeout the wait records kStatusWaitTimeout and
// returns; the run completes with garbage and hg_exec_wait reports HG_EDEADLOCK.
__global__ void k_wait_flag(FlagParams p) {
  if (threadIdx.x == 0) {
    const int e = *reinterpret_cast<volatile const int*>(p.epoch);
    const unsigned long long t0 = global_ns();
    while (ld_acquire_sys(p.flag) < e) {
      // once one wait of this run gave up, the others stop spinning too
      if ((*reinterpret_cast<volatile int*>(p.status) & kStatusWaitTimeout) || global_ns() - t0 > p.timeout_ns) {
        atomicOr(p.status, kStatusWaitTimeout);
        break;
      }
      __nanosleep(256);
    }
  }
}

__global__ void k_signal_flag(FlagParams p) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(p.flag, *reinterpret_cast<volatile const int*>(p.epoch));
  }
}

// Step fence between launches (one process per GPU): before run e starts, every
// peer must have finished run e-1 -- a peer's last pulls from THIS rank's slots
// (consumer-pull copies) may still be pending when this rank's own graph is done,
// and run e's first touches would overwrite those slots.
struct StepFence {
  const int* peer_done[16];
  int n;
  int need;
  int* status;
  unsigned long long timeout_ns;
};
__global__ void k_wait_peers_done(StepFence f) {
  if (threadIdx.x < f.n) {
    const unsigned long long t0 = global_ns();
    while (ld_acquire_sys(f.peer_done[threadIdx.x]) < f.need) {
      if ((*reinterpret_cast<volatile int*>(f.status) & kStatusWaitTimeout) || global_ns() - t0 > f.timeout_ns) {
        atomicOr(f.status, kStatusWaitTimeout);
        break;
      }
      __nanosleep(256);
    }
  }
}

__global__ void k_mark_done(int* done, int v) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(done, v);
  }
}

__global__ void k_set_epoch(int* epoch, int v) {
  if (threadIdx.x == 0) *epoch = v;
}

// trace mode: device time (ns) at which a task / copy job starts and ends (hg_exec_read_stamps)
__global__ void k_stamp(unsigned long long* p) {
  if (threadIdx.x == 0) *p = global_ns();
}

}  // namespace hg

struct hg_exec {
  // plan (owned copy)
  int k = 0, nb = 0, ib = 0, side = 0, n_blocks = 0, n_tasks = 0, n_jobs = 0;
  std::vector<int32_t> task_kind, task_node, acc_block, pred, dispatch, wait_job;
  std::vector<int8_t> acc_mode;
  std::vector<int64_t> acc_ptr, pred_ptr, wait_ptr, block_bytes;
  std::vector<int32_t> job_block, job_src, job_dst, job_version, job_src_job, job_requester, final_writer;
  std::vector<int32_t> job_stage_job;
  int p2p = 1;
  int push = 0;                          // producer-push fusion requested (hg_exec_plan.push)
  std::vector<char> job_push;            // job delivered by its version's producer kernel (no copy node)
  std::vector<std::vector<std::pair<int, int>>> push_to;  // per task: (destination node, block) its kernels push
  double* host_stage = nullptr;          // p2p = 0: pinned staging image, slot-sized regions
  std::vector<int64_t> stage_off;
  // options
  int rank_node = 0;
  const double* host_in = nullptr;
  double* host_out = nullptr;
  double* host_side_out = nullptr;
  int device_input = 0;
  std::vector<double> task_weight;     // predicted seconds per task (node priorities)
  int priority_levels = 0;
  // memory
  std::vector<int> dev;                 // node g+1 -> device
  std::vector<double*> base;            // per node: pool base (local allocation or IPC mapping)
  std::vector<char> ipc;                // per node: base came from cudaIpcOpenMemHandle
  std::vector<double*> replica;         // per local node: device copy of host_in
  std::vector<int*> status, scratch;    // per local node
  std::vector<unsigned long long*> stamps;  // per local node, trace mode: [2 * (n_tasks + n_jobs)]
  int trace = 0;
  std::vector<std::vector<int64_t>> slot;  // [node-1][block] -> doubles offset, -1 = none
  std::vector<int64_t> pool_doubles;    // per node
  int64_t header_doubles = 0;
  std::vector<int64_t> host_off, blk_doubles, slot_doubles;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // single process, several devices: each non-first device's status word is reset on its own
  // stream, ordered after the previous run (ev_prev on `stream`) and before this one (ev_reset)
  std::vector<cudaStream_t> aux_stream;
  std::vector<cudaEvent_t> ev_reset;
  cudaEvent_t ev_prev = nullptr;
  unsigned long long wait_timeout_ns = 60ull * 1000000000ull;  // cross-rank waits (hg_exec_set_wait_timeout)
  hg_exec_stats stats{};
  cudaStream_t last_stream = nullptr;
  bool launched = false;
  int epoch = 0;
  bool built = false;

  bool is_local(int node) const { return node >= 1 && node <= k && (rank_node == 0 || node == rank_node); }
  int* flags(int node) const { return reinterpret_cast<int*>(base[node - 1]); }
  int* task_flag(int node, int t) const { return flags(node) + t; }
  int* job_flag(int node, int j) const { return flags(node) + n_tasks + j; }
  int* epoch_ptr(int node) const { return flags(node) + n_tasks + n_jobs; }
  int* done_ptr(int node) const { return flags(node) + n_tasks + n_jobs + 1; }  // last finished epoch
  double* slot_ptr(int node, int b) const {
    int64_t off = slot[node - 1][b];
    return off < 0 ? nullptr : base[node - 1] + off;
  }
};

static void release(hg_exec* ex) {
  if (!ex) return;
  if (ex->exec) cudaGraphExecDestroy(ex->exec);
  if (ex->graph) cudaGraphDestroy(ex->graph);
  for (int g = 0; g < ex->k; ++g) {
    if (g >= (int)ex->base.size()) break;
    cudaSetDevice(ex->dev[g]);
    if (ex->base[g]) {
      if (ex->ipc[g]) cudaIpcCloseMemHandle(ex->base[g]);
      else cudaFree(ex->base[g]);
    }
    if (ex->replica[g]) cudaFree(ex->replica[g]);
    if (ex->status[g]) cudaFree(ex->status[g]);
    if (g < (int)ex->stamps.size() && ex->stamps[g]) cudaFree(ex->stamps[g]);
    if (ex->scratch[g]) cudaFree(ex->scratch[g]);
  }
  for (size_t g = 0; g < ex->aux_stream.size(); ++g) {
    if (ex->aux_stream[g]) {
      cudaSetDevice(ex->dev[g]);
      cudaStreamDestroy(ex->aux_stream[g]);
    }
    if (ex->ev_reset[g]) cudaEventDestroy(ex->ev_reset[g]);
  }
  if (ex->ev_prev) cudaEventDestroy(ex->ev_prev);
  if (ex->ev0) cudaEventDestroy(ex->ev0);
  if (ex->ev1) cudaEventDestroy(ex->ev1);
  if (ex->stream) cudaStreamDestroy(ex->stream);
  delete ex;
}

// Deterministic per-node layout (every process computes every node's).
static void plan_layout(hg_exec* ex) {
  const int64_t tile_d = int64_t(ex->nb) * ex->nb;
  ex->host_off.resize(ex->n_blocks);
  ex->blk_doubles.resize(ex->n_blocks);
  ex->slot_doubles.resize(ex->n_blocks);
  int64_t host_total = 0;
  for (int b = 0; b < ex->n_blocks; ++b) {
    ex->blk_doubles[b] = ex->block_bytes[b] / 8;
    ex->slot_doubles[b] = ex->blk_doubles[b] + (ex->blk_doubles[b] == tile_d ? ex->side : 0);
    ex->host_off[b] = host_total;
    host_total += ex->blk_doubles[b];
  }
  ex->stage_off.resize(ex->n_blocks);
  int64_t so = 0;
  for (int b = 0; b < ex->n_blocks; ++b) {
    ex->stage_off[b] = so;
    so += ex->slot_doubles[b];
  }
  const int64_t flag_ints = int64_t(ex->n_tasks) + ex->n_jobs + 2;
  ex->header_doubles = ((flag_ints * 4 + 255) / 256) * 32;
  ex->slot.assign(ex->k, std::vector<int64_t>(ex->n_blocks, -1));
  ex->pool_doubles.assign(ex->k, ex->header_doubles);
  auto need = [&](int node, int b) {
    if (node < 1 || node > ex->k) return;
    int64_t& s = ex->slot[node - 1][b];
    if (s < 0) {
      s = ex->pool_doubles[node - 1];
      ex->pool_doubles[node - 1] += (ex->slot_doubles[b] + 31) / 32 * 32;  // 256-byte aligned slots
    }
  };
  for (int t = 0; t < ex->n_tasks; ++t)
    for (int64_t a = ex->acc_ptr[t]; a < ex->acc_ptr[t + 1]; ++a) need(ex->task_node[t], ex->acc_block[a]);
  for (int j = 0; j < ex->n_jobs; ++j) need(ex->job_dst[j], ex->job_block[j]);
}

// Producer-push fusion: a peer job that moves version v of block b (written
// by task v) to GPU node D is delivered by task v's own kernels -- their epilogue stores the final
// tile to D's slot of b as well (peer / IPC pointers) -- when v's kind supports it (tiles.h
// kind_can_push: the Cholesky kinds, the LU / QR trailing updates and panels) and b is a tile
// (materialised T blocks travel by copy node).  At most kMaxPush (D, b) pairs per task are
// pushed; further jobs keep their copy nodes.  Bytes per (version, destination) equal the
// plan's; the copy node disappears and the consumer depends on task v itself.  WAR-safe: every
// reader of any older version of the block precedes v in the DAG (graph.py:58-84), and the
// step fence orders runs across ranks.  Deterministic from the plan, so every rank agrees.
static void plan_push(hg_exec* ex) {
  ex->job_push.assign(ex->n_jobs, 0);
  ex->push_to.assign(ex->n_tasks, {});
  if (!ex->push || !ex->p2p || ex->k < 2) return;
  const int64_t tile_d = int64_t(ex->nb) * ex->nb;
  for (int j = 0; j < ex->n_jobs; ++j) {
    const int v = ex->job_version[j], dst = ex->job_dst[j], b = ex->job_block[j];
    if (v < 0 || dst < 1 || ex->job_src[j] < 1 || !kind_can_push(ex->task_kind[v], ex->nb, ex->ib)) continue;
    if (ex->blk_doubles[b] != tile_d) continue;
    auto& d = ex->push_to[v];
    const std::pair<int, int> e{dst, b};
    if ((int)d.size() < kMaxPush && std::find(d.begin(), d.end(), e) == d.end()) d.push_back(e);
  }
  for (int j = 0; j < ex->n_jobs; ++j) {
    const int v = ex->job_version[j];
    if (v < 0) continue;
    const auto& d = ex->push_to[v];
    ex->job_push[j] = std::find(d.begin(), d.end(), std::make_pair(ex->job_dst[j], ex->job_block[j])) != d.end();
  }
}

// Which producers must signal (consumer on another, non-local node) and which
// consumers must wait (producer on another, non-local node).
struct Partition {
  std::vector<char> sig_task, sig_job, waited;  // waited: [n_tasks + n_jobs] flags this rank spins on
  int n_local_tasks = 0, n_local_jobs = 0, n_waits = 0, n_signals = 0;
};

static Partition partition(const hg_exec* ex) {
  Partition P;
  P.sig_task.assign(ex->n_tasks, 0);
  P.sig_job.assign(ex->n_jobs, 0);
  auto cross = [&](int prod_node, int cons_node) {
    return prod_node != cons_node && !(ex->is_local(prod_node) && ex->is_local(cons_node));
  };
  std::vector<char> wt(ex->n_tasks + ex->n_jobs, 0);  // remote flags this rank waits on
  for (int t = 0; t < ex->n_tasks; ++t) {
    const int cn = ex->task_node[t];
    if (ex->is_local(cn)) P.n_local_tasks++;
    for (int64_t q = ex->pred_ptr[t]; q < ex->pred_ptr[t + 1]; ++q) {
      const int u = ex->pred[q];
      if (cross(ex->task_node[u], cn)) {
        P.sig_task[u] = 1;
        if (ex->is_local(cn)) wt[u] = 1;
      }
    }
  }
  for (int j = 0; j < ex->n_jobs; ++j) {
    const int cn = ex->job_dst[j];
    if (ex->is_local(cn)) P.n_local_jobs++;
    if (!ex->job_push.empty() && ex->job_push[j]) {  // delivered by the producer task itself
      const int v = ex->job_version[j];
      if (cross(ex->task_node[v], cn)) {
        P.sig_task[v] = 1;
        if (ex->is_local(cn)) wt[v] = 1;
      }
    } else if (ex->job_src_job[j] >= 0) {
      const int sj = ex->job_src_job[j];
      if (cross(ex->job_dst[sj], cn)) {
        P.sig_job[sj] = 1;
        if (ex->is_local(cn)) wt[ex->n_tasks + sj] = 1;
      }
    } else if (ex->job_version[j] >= 0) {
      const int v = ex->job_version[j];
      if (cross(ex->task_node[v], cn)) {
        P.sig_task[v] = 1;
        if (ex->is_local(cn)) wt[v] = 1;
      }
    }
  }
  for (char w : wt) P.n_waits += w;
  P.waited = wt;
  for (int t = 0; t < ex->n_tasks; ++t) P.n_signals += P.sig_task[t] && ex->is_local(ex->task_node[t]);
  for (int j = 0; j < ex->n_jobs; ++j)
    P.n_signals += P.sig_job[j] && ex->is_local(ex->job_dst[j]) && !(ex->job_push.size() && ex->job_push[j]);
  return P;
}

static int add_flag_kernel(cudaGraph_t g, cudaGraphNode_t* out, const cudaGraphNode_t* deps, size_t nd,
                           const void* fn, hg::FlagParams fp) {
  cudaKernelNodeParams kp{};
  void* args[1] = {&fp};
  kp.func = const_cast<void*>(fn);
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(32);
  kp.sharedMemBytes = 0;
  kp.kernelParams = args;
  HG_CUDA(cudaGraphAddKernelNode(out, g, deps, nd, &kp));
  return HG_OK;
}

// CUDA priority of each task's kernel nodes from its slack: the longest path
// through the task (top level + bottom level, weights = predicted durations)
// against the DAG's critical path.  Zero-slack tasks (the POTRF / panel chain
// and what feeds it) get the device's greatest priority; ready work with slack
// fills the SMs behind them.  Task ids are a topological order (every DAG edge
// goes from a lower to a higher id, graph.py:58-84).
static std::vector<int> task_priorities(const hg_exec* ex, int dev) {
  const int n = ex->n_tasks;
  std::vector<int> prio(n, 0);
  if (ex->priority_levels <= 0 || (int)ex->task_weight.size() != n) return prio;
  int least = 0, greatest = 0;
  if (cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) {
    cudaGetLastError();
    return prio;
  }
  const int range = least - greatest + 1;  // greatest is numerically smallest
  const int levels = std::min(ex->priority_levels, range);
  if (levels <= 1) return prio;
  (void)dev;
  std::vector<double> top(n, 0.0), bot(n, 0.0);
  for (int t = 0; t < n; ++t)
    for (int64_t q = ex->pred_ptr[t]; q < ex->pred_ptr[t + 1]; ++q) {
      const int u = ex->pred[q];
      top[t] = std::max(top[t], top[u] + ex->task_weight[u]);
    }
  for (int t = n - 1; t >= 0; --t) {
    bot[t] += ex->task_weight[t];
    for (int64_t q = ex->pred_ptr[t]; q < ex->pred_ptr[t + 1]; ++q) {
      const int u = ex->pred[q];
      bot[u] = std::max(bot[u], bot[t]);
    }
  }
  double cp = 0.0;
  for (int t = 0; t < n; ++t) cp = std::max(cp, top[t] + bot[t]);
  if (!(cp > 0.0)) return prio;
  // level 0 (most urgent) for slack < cp / (2 levels), then bands of the same width
  const double band = cp / (2.0 * levels);
  for (int t = 0; t < n; ++t) {
    const double slack = std::max(0.0, cp - top[t] - bot[t]);
    const int lvl = std::min(levels - 1, int(slack / band));
    prio[t] = greatest + lvl;
  }
  return prio;
}

static int build_graph(hg_exec* ex) {
  const int n = ex->n_tasks;
  plan_push(ex);
  const Partition part = partition(ex);
  HG_CUDA(cudaGraphCreate(&ex->graph, 0));
  std::vector<cudaGraphNode_t> task_last(n, nullptr);
  std::vector<cudaGraphNode_t> job_node(ex->n_jobs, nullptr);
  std::vector<cudaGraphNode_t> d2h_node(ex->n_jobs, nullptr);  // GPU->host leg of host-staged moves
  std::vector<cudaGraphNode_t> wait_node(size_t(n) + ex->n_jobs, nullptr);
  std::vector<std::vector<int>> jobs_of(n);
  for (int j = 0; j < ex->n_jobs; ++j) jobs_of[ex->job_requester[j]].push_back(j);
  std::vector<LaunchDesc> launches;
  std::vector<cudaGraphNode_t> deps;
  int64_t side_bytes = 0;
  std::vector<int64_t> scratch_used(ex->k, 0);
  hg_exec_stats& st = ex->stats;
  {
    const int first = ex->rank_node ? ex->rank_node : 1;
    HG_CUDA(cudaSetDevice(ex->dev[first - 1]));
  }
  const std::vector<int> prio = task_priorities(ex, 0);
  const bool use_prio = ex->priority_levels > 0 && !ex->task_weight.empty();
  int prio_greatest = 0;
  {
    int least = 0;
    if (cudaDeviceGetStreamPriorityRange(&least, &prio_greatest) != cudaSuccess) cudaGetLastError();
  }

  // Delivery of a block version to a node: a task must wait for the copy job
  // that brought the version it reads to its node, even when that job was
  // requested by ANOTHER task (sim.py:242-253 dedups (data, node) in flight
  // and skips blocks already valid on the node, so the plan's wait list of
  // this task does not name it, and the DAG does not order it either).
  // Version read by access a = last writer of the block before the task in
  // program order (the DAG's sequential consistency, graph.py:58-84).
  std::vector<int32_t> acc_version(ex->acc_block.size(), -1);
  {
    std::vector<int32_t> cur(ex->n_blocks, -1);
    for (int t = 0; t < n; ++t) {
      for (int64_t a = ex->acc_ptr[t]; a < ex->acc_ptr[t + 1]; ++a) acc_version[a] = cur[ex->acc_block[a]];
      for (int64_t a = ex->acc_ptr[t]; a < ex->acc_ptr[t + 1]; ++a)
        if (ex->acc_mode.empty() || (ex->acc_mode[a] & HG_ACCESS_W)) cur[ex->acc_block[a]] = t;
    }
  }
  auto dkey = [&](int b, int v, int node) {
    return (uint64_t(uint32_t(b)) << 40) ^ (uint64_t(uint32_t(v + 1)) << 8) ^ uint64_t(node);
  };
  std::unordered_map<uint64_t, int> delivery;  // (block, version, dst node) -> job
  for (int j = 0; j < ex->n_jobs; ++j) {
    // the version a job moves: the writer task, or (H2D of an untouched block) -1
    const int v = ex->job_version[j];
    if (ex->job_dst[j] >= 1) delivery.emplace(dkey(ex->job_block[j], v, ex->job_dst[j]), j);
  }

  constexpr int h2d_chains = 1;
  std::vector<cudaGraphNode_t> h2d_tail(size_t(ex->k) * h2d_chains, nullptr);
  std::vector<int> h2d_count(ex->k, 0);

  // Cross-rank waits (one process per GPU).  Each spinning wait holds a CTA slot, so waits are
  // (1) gated: a wait only starts once the task that needs it is otherwise ready (its local
  //     predecessors are done) -- the planner likewise issues a copy only when its requester is
  //     dispatched (sim.py:237-267);
  // (2) chained: wait nodes join kWaitChains chains round-robin in creation (= dispatch) order,
  //     so at most kWaitChains spinners are resident per device however many remote edges the
  //     plan has.  Deadlock-free by induction over the plan's dispatch order: the producer of a
  //     flag completed (in the plan) before the waiting task was dispatched, so it never depends
  //     on a task dispatched later, i.e. on anything queued behind the wait in its chain.
  constexpr int kWaitChains = 8;
  std::vector<cudaGraphNode_t> chain_tail(kWaitChains, nullptr);
  int chain_next = 0;
  std::vector<cudaGraphNode_t> gate;  // local predecessors of the task being dispatched
  auto add_wait = [&](cudaGraphNode_t* w, const std::vector<cudaGraphNode_t>& gate_deps, int* flag,
                      int cons_node) -> int {
    std::vector<cudaGraphNode_t> wd = gate_deps;
    cudaGraphNode_t& tail = chain_tail[chain_next];
    chain_next = (chain_next + 1) % kWaitChains;
    if (tail) wd.push_back(tail);
    std::sort(wd.begin(), wd.end());
    wd.erase(std::unique(wd.begin(), wd.end()), wd.end());
    HG_CUDA(cudaSetDevice(ex->dev[cons_node - 1]));
    int rc = add_flag_kernel(ex->graph, w, wd.data(), wd.size(), (const void*)hg::k_wait_flag,
                             hg::FlagParams{flag, ex->epoch_ptr(cons_node), ex->status[cons_node - 1],
                                            ex->wait_timeout_ns});
    if (rc) return rc;
    tail = *w;
    return HG_OK;
  };
  // dependency on the producer of a task output / job delivery for a consumer on cons_node
  auto dep_task = [&](int u, int cons_node) -> int {
    const int pn = ex->task_node[u];
    if (ex->is_local(pn) && (ex->is_local(cons_node))) {
      deps.push_back(task_last[u]);
      return HG_OK;
    }
    cudaGraphNode_t& w = wait_node[u];
    if (!w) {
      int rc = add_wait(&w, gate, ex->task_flag(pn, u), cons_node);
      if (rc) return rc;
    }
    deps.push_back(w);
    return HG_OK;
  };
  auto dep_job = [&](int sj, int cons_node) -> int {
    const int pn = ex->job_dst[sj];
    if (ex->is_local(pn) && ex->is_local(cons_node)) {
      deps.push_back(job_node[sj]);
      return HG_OK;
    }
    cudaGraphNode_t& w = wait_node[size_t(n) + sj];
    if (!w) {
      int rc = add_wait(&w, gate, ex->job_flag(pn, sj), cons_node);
      if (rc) return rc;
    }
    deps.push_back(w);
    return HG_OK;
  };

  // trace mode: a 1-thread stamp node before and after each task's kernel chain / each copy job
  auto add_stamp = [&](cudaGraphNode_t* out, const cudaGraphNode_t* d, size_t nd, int node, int64_t slot,
                       int prio) -> int {
    unsigned long long* p = ex->stamps[node - 1] + slot;
    cudaKernelNodeParams kp{};
    void* args[1] = {&p};
    kp.func = (void*)hg::k_stamp;
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(32);
    kp.kernelParams = args;
    HG_CUDA(cudaSetDevice(ex->dev[node - 1]));
    HG_CUDA(cudaGraphAddKernelNode(out, ex->graph, d, nd, &kp));
    if (use_prio) {
      cudaKernelNodeAttrValue v{};
      v.priority = prio;
      HG_CUDA(cudaGraphKernelNodeSetAttribute(*out, cudaKernelNodeAttributePriority, &v));
    }
    return HG_OK;
  };

  for (int di = 0; di < n; ++di) {
    const int t = ex->dispatch[di];
    gate.clear();
    if (ex->rank_node)
      for (int64_t q = ex->pred_ptr[t]; q < ex->pred_ptr[t + 1]; ++q) {
        const int u = ex->pred[q];
        if (ex->is_local(ex->task_node[u]) && task_last[u]) gate.push_back(task_last[u]);
      }
    // 1) inbound copy jobs created by this dispatch
    for (int j : jobs_of[t]) {
      const int dst = ex->job_dst[j];
      if (!ex->is_local(dst)) continue;
      const int b = ex->job_block[j], src = ex->job_src[j];
      deps.clear();
      int rc = HG_OK;
      if (ex->job_push[j]) {
        // delivered by the producer's epilogue: "arrival" is the producer task's completion
        rc = dep_task(ex->job_version[j], dst);
        if (rc) return rc;
        job_node[j] = deps[0];
        st.bytes_d2d += size_t(ex->blk_doubles[b]) * 8;
        st.n_push_jobs++;
        {  // the LU / QR panel kinds push whole slots: the side area rides along as with a copy node
          const int pk = ex->task_kind[ex->job_version[j]];
          if (pk == K_GETRF_INC || pk == K_TSTRF || pk == K_GEQRT || pk == K_TSQRT)
            side_bytes += int64_t(ex->slot_doubles[b] - ex->blk_doubles[b]) * 8;
        }
        continue;
      }
      const bool staged_in = src == 0 && (ex->job_version[j] >= 0 || ex->job_src_job[j] >= 0 ||
                                          ex->job_stage_job[j] >= 0);
      const bool staged_move = src >= 1 && dst >= 1 && !ex->p2p;
      if (staged_in) {
        // a version staged in host memory by an earlier GPU->host leg (sim.py:255-261, 322-337)
        const int sj = ex->job_stage_job[j] >= 0 ? ex->job_stage_job[j] : ex->job_src_job[j];
        if (sj < 0 || !d2h_node[sj]) {
          set_error("job %d: staged version of block %d without its host leg", j, b);
          return HG_EINVAL;
        }
        deps.push_back(d2h_node[sj]);
      } else if (ex->job_src_job[j] >= 0) {
        rc = dep_job(ex->job_src_job[j], dst);
      } else if (ex->job_version[j] >= 0) {
        rc = dep_task(ex->job_version[j], dst);
      }
      if (rc) return rc;
      // host -> device first touches are serialised into one chain per GPU in dispatch order, so the
      // copy engine delivers tiles in the order tasks need them instead of all at once in arbitrary
      // order (C2 e2e: 427 -> 372 ms, i.e. PCIe fully hidden behind compute)
      const bool from_host = src == 0 && !ex->device_input && !staged_in;
      if (from_host && h2d_chains > 0) {
        cudaGraphNode_t& prev = h2d_tail[size_t(dst - 1) * h2d_chains + (h2d_count[dst - 1]++ % h2d_chains)];
        if (prev) deps.push_back(prev);
      }
      const int64_t jslot = 2 * (int64_t(n) + j);
      if (ex->trace) {
        cudaGraphNode_t s0;
        int rc2 = add_stamp(&s0, deps.data(), deps.size(), dst, jslot, prio_greatest);
        if (rc2) return rc2;
        deps.assign(1, s0);
      }
      double* dptr = ex->slot_ptr(dst, b);
      const void* sptr;
      size_t bytes;
      if (staged_move) {
        // GPU -> host -> GPU (platform.py:117): two copy nodes through the staging image
        const size_t sb = size_t(ex->slot_doubles[b]) * 8;
        double* stage = ex->host_stage + ex->stage_off[b];
        HG_CUDA(cudaSetDevice(ex->dev[src - 1]));
        HG_CUDA(cudaGraphAddMemcpyNode1D(&d2h_node[j], ex->graph, deps.data(), deps.size(), stage,
                                         ex->slot_ptr(src, b), sb, cudaMemcpyDefault));
        st.bytes_d2h += size_t(ex->blk_doubles[b]) * 8;
        st.n_copy_nodes++;
        deps.assign(1, d2h_node[j]);
        bytes = sb;
        sptr = stage;
        st.bytes_h2d += size_t(ex->blk_doubles[b]) * 8;
        side_bytes += 2 * (sb - size_t(ex->blk_doubles[b]) * 8);
      } else if (staged_in) {
        bytes = size_t(ex->slot_doubles[b]) * 8;
        sptr = ex->host_stage + ex->stage_off[b];
        st.bytes_h2d += size_t(ex->blk_doubles[b]) * 8;
        side_bytes += bytes - size_t(ex->blk_doubles[b]) * 8;
      } else if (src == 0) {
        bytes = size_t(ex->blk_doubles[b]) * 8;
        sptr = ex->device_input ? (const void*)(ex->replica[dst - 1] + ex->host_off[b])
                                : (const void*)(ex->host_in + ex->host_off[b]);
        st.bytes_h2d += bytes;
      } else if (dst == 0) {
        set_error("job %d: device->host jobs are not executable on a GPU-only platform", j);
        return HG_EINVAL;
      } else {
        bytes = size_t(ex->slot_doubles[b]) * 8;
        sptr = ex->slot_ptr(src, b);
        st.bytes_d2d += size_t(ex->blk_doubles[b]) * 8;
        side_bytes += bytes - size_t(ex->blk_doubles[b]) * 8;
      }
      if (!dptr || !sptr) {
        set_error("job %d: missing slot (block %d, %d -> %d)", j, b, src, dst);
        return HG_EINVAL;
      }
      HG_CUDA(cudaSetDevice(ex->dev[dst - 1]));
      HG_CUDA(cudaGraphAddMemcpyNode1D(&job_node[j], ex->graph, deps.data(), deps.size(), dptr, sptr, bytes,
                                       cudaMemcpyDefault));
      if (ex->trace) {
        cudaGraphNode_t s1;
        int rc2 = add_stamp(&s1, &job_node[j], 1, dst, jslot + 1, prio_greatest);
        if (rc2) return rc2;
        job_node[j] = s1;
      }
      if (from_host && h2d_chains > 0)
        h2d_tail[size_t(dst - 1) * h2d_chains + ((h2d_count[dst - 1] - 1) % h2d_chains)] = job_node[j];
      st.n_copy_nodes++;
      if (part.sig_job[j]) {
        cudaGraphNode_t sn;
        int rc2 = add_flag_kernel(ex->graph, &sn, &job_node[j], 1, (const void*)hg::k_signal_flag,
                                  hg::FlagParams{ex->job_flag(dst, j), ex->epoch_ptr(dst), nullptr, 0});
        if (rc2) return rc2;
      }
    }
    // 2) the task's kernel chain
    const int node = ex->task_node[t];
    if (!ex->is_local(node)) continue;
    TaskOperands ops;
    ops.nb = ex->nb;
    ops.ib = ex->ib;
    ops.status = ex->status[node - 1];
    const int sc = task_scratch_ints(ex->task_kind[t], ex->nb, ex->ib);
    if (sc > 0) {
      ops.scratch = ex->scratch[node - 1] + scratch_used[node - 1];
      scratch_used[node - 1] += sc;
    }
    const int64_t a0 = ex->acc_ptr[t], a1 = ex->acc_ptr[t + 1];
    if (a1 - a0 > 4) {
      set_error("task %d has %lld accesses (max 4)", t, (long long)(a1 - a0));
      return HG_EINVAL;
    }
    for (int64_t a = a0; a < a1; ++a) ops.t[ops.n_t++] = ex->slot_ptr(node, ex->acc_block[a]);
    ops.side = ex->side;
    for (const auto& e : ex->push_to[t]) {
      const int d = e.first, b = e.second;
      int op = -1;  // the written operand holding block b
      for (int64_t a = a0; a < a1; ++a)
        if (ex->acc_block[a] == b && (ex->acc_mode.empty() || (ex->acc_mode[a] & HG_ACCESS_W))) op = int(a - a0);
      double* q = ex->slot_ptr(d, b);
      if (op < 0 || !q) {
        set_error("task %d: block %d is not an output with a slot on push destination node %d", t, b, d);
        return HG_EINVAL;
      }
      ops.push.dst[ops.push.n] = q;
      ops.push.op[ops.push.n++] = (unsigned char)op;
    }
    launches.clear();
    if (!build_task_launches(ex->task_kind[t], ops, launches)) return HG_EINVAL;
    deps.clear();
    for (int64_t w = ex->wait_ptr[t]; w < ex->wait_ptr[t + 1]; ++w) deps.push_back(job_node[ex->wait_job[w]]);
    for (int64_t a = a0; a < a1; ++a) {
      if (!ex->acc_mode.empty() && !(ex->acc_mode[a] & HG_ACCESS_R)) continue;
      auto it = delivery.find(dkey(ex->acc_block[a], acc_version[a], node));
      if (it == delivery.end()) continue;
      const int j = it->second;
      if (!job_node[j]) {
        set_error("task %d reads block %d on node %d before its delivery job %d exists", t, ex->acc_block[a], node, j);
        return HG_EINVAL;
      }
      deps.push_back(job_node[j]);
    }
    // local predecessors first; a predecessor on another rank becomes a flag-wait
    // node of THIS task that itself waits for the task's local dependencies, so it
    // only spins once the task is otherwise ready (a root wait node per remote edge
    // would keep thousands of 1-warp CTAs spinning from the start of the graph)
    int n_remote = 0;
    for (int64_t q = ex->pred_ptr[t]; q < ex->pred_ptr[t + 1]; ++q) {
      const int u = ex->pred[q];
      if (ex->is_local(ex->task_node[u])) {
        int rc = dep_task(u, node);
        if (rc) return rc;
      } else {
        ++n_remote;
      }
    }
    if (n_remote) {
      std::sort(deps.begin(), deps.end());
      deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
      const std::vector<cudaGraphNode_t> local = deps;
      for (int64_t q = ex->pred_ptr[t]; q < ex->pred_ptr[t + 1]; ++q) {
        const int u = ex->pred[q];
        const int pn = ex->task_node[u];
        if (ex->is_local(pn)) continue;
        cudaGraphNode_t w;
        int rc = add_wait(&w, local, ex->task_flag(pn, u), node);
        if (rc) return rc;
        deps.push_back(w);
      }
    }
    std::sort(deps.begin(), deps.end());  // a delivery job may also be in the wait list
    deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
    if (ex->trace) {
      cudaGraphNode_t s0;
      int rc = add_stamp(&s0, deps.data(), deps.size(), node, 2 * int64_t(t), use_prio ? prio[t] : 0);
      if (rc) return rc;
      deps.assign(1, s0);
    }
    HG_CUDA(cudaSetDevice(ex->dev[node - 1]));
    cudaGraphNode_t prev = nullptr;
    for (size_t li = 0; li < launches.size(); ++li) {
      cudaKernelNodeParams kp{};
      void* args[1] = {launches[li].params};
      kp.func = const_cast<void*>(launches[li].func);
      kp.gridDim = launches[li].grid;
      kp.blockDim = launches[li].block;
      kp.sharedMemBytes = launches[li].smem;
      kp.kernelParams = args;
      cudaGraphNode_t nd;
      if (li == 0) HG_CUDA(cudaGraphAddKernelNode(&nd, ex->graph, deps.data(), deps.size(), &kp));
      else HG_CUDA(cudaGraphAddKernelNode(&nd, ex->graph, &prev, 1, &kp));
      if (use_prio) {
        cudaKernelNodeAttrValue v{};
        v.priority = prio[t];
        HG_CUDA(cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributePriority, &v));
      }
      prev = nd;
      st.n_kernel_nodes++;
    }
    if (ex->trace) {
      cudaGraphNode_t s1;
      int rc = add_stamp(&s1, &prev, 1, node, 2 * int64_t(t) + 1, use_prio ? prio[t] : 0);
      if (rc) return rc;
      prev = s1;
    }
    task_last[t] = prev;
    if (part.sig_task[t]) {
      cudaGraphNode_t sn;
      int rc = add_flag_kernel(ex->graph, &sn, &task_last[t], 1, (const void*)hg::k_signal_flag,
                               hg::FlagParams{ex->task_flag(node, t), ex->epoch_ptr(node), nullptr, 0});
      if (rc) return rc;
    }
  }
  // 3) write-back of final versions produced on local nodes
  if (ex->host_out) {
    for (int b = 0; b < ex->n_blocks; ++b) {
      const int w = ex->final_writer[b];
      if (w < 0) continue;
      const int node = ex->task_node[w];
      if (!ex->is_local(node)) continue;
      size_t bytes = size_t(ex->blk_doubles[b]) * 8;
      cudaGraphNode_t nd;
      HG_CUDA(cudaSetDevice(ex->dev[node - 1]));
      HG_CUDA(cudaGraphAddMemcpyNode1D(&nd, ex->graph, &task_last[w], 1, ex->host_out + ex->host_off[b],
                                       ex->slot_ptr(node, b), bytes, cudaMemcpyDefault));
      st.bytes_d2h += bytes;
      st.n_copy_nodes++;
      if (ex->host_side_out && ex->side > 0 && ex->slot_doubles[b] > ex->blk_doubles[b]) {
        HG_CUDA(cudaGraphAddMemcpyNode1D(&nd, ex->graph, &task_last[w], 1,
                                         ex->host_side_out + int64_t(b) * ex->side,
                                         ex->slot_ptr(node, b) + ex->blk_doubles[b], size_t(ex->side) * 8,
                                         cudaMemcpyDefault));
        st.n_copy_nodes++;
      }
    }
  }
  st.bytes_side = side_bytes;
  int first = ex->rank_node ? ex->rank_node : 1;
  HG_CUDA(cudaSetDevice(ex->dev[first - 1]));
  HG_CUDA(cudaGraphInstantiate(&ex->exec, ex->graph, use_prio ? cudaGraphInstantiateFlagUseNodePriority : 0));
  ex->built = true;
  return HG_OK;
}

template <class T>
static std::vector<T> vcopy(const T* p, int64_t n) {
  return n > 0 && p ? std::vector<T>(p, p + n) : std::vector<T>();
}

extern "C" int hg_exec_create(const hg_exec_plan* P, const hg_exec_opts* O, hg_exec** out) {
  if (!P || !O || !out || P->k < 1 || !O->devices) {
    set_error("hg_exec_create: bad arguments");
    return HG_EINVAL;
  }
  if (!O->host_in) {
    set_error("hg_exec_create: host_in is required (initial residency is the host, sim.py:47-48)");
    return HG_EINVAL;
  }
  if (O->rank_node < 0 || O->rank_node > P->k) {
    set_error("hg_exec_create: rank_node %d out of range", O->rank_node);
    return HG_EINVAL;
  }
  hg_exec* ex = new hg_exec();
  ex->k = P->k;
  ex->nb = P->nb;
  ex->ib = P->ib;
  ex->side = P->side_doubles;
  ex->n_blocks = P->n_blocks;
  ex->n_tasks = P->n_tasks;
  ex->n_jobs = P->n_jobs;
  const int n = P->n_tasks, nj = P->n_jobs;
  ex->task_kind = vcopy(P->task_kind, n);
  ex->task_node = vcopy(P->task_node, n);
  ex->acc_ptr = vcopy(P->acc_ptr, n + 1);
  ex->acc_block = vcopy(P->acc_block, P->acc_ptr[n]);
  ex->acc_mode = vcopy(P->acc_mode, P->acc_ptr[n]);
  ex->job_stage_job = vcopy(P->job_stage_job, P->n_jobs);
  ex->p2p = P->p2p;
  ex->push = P->push;
  ex->host_stage = O->host_stage;
  if (!ex->p2p && P->k > 1) {
    if (!O->host_stage) {
      set_error("hg_exec_create: a p2p=0 plan needs opts.host_stage (pinned, slot-sized regions)");
      delete ex;
      return HG_EINVAL;
    }
    if (O->rank_node != 0) {
      set_error("hg_exec_create: host-staged routes need the single-process executor (rank_node 0)");
      delete ex;
      return HG_EINVAL;
    }
  }
  ex->pred_ptr = vcopy(P->pred_ptr, n + 1);
  ex->pred = vcopy(P->pred, P->pred_ptr[n]);
  ex->dispatch = vcopy(P->dispatch, n);
  ex->wait_ptr = vcopy(P->wait_ptr, n + 1);
  ex->wait_job = vcopy(P->wait_job, P->wait_ptr[n]);
  ex->job_block = vcopy(P->job_block, nj);
  ex->job_src = vcopy(P->job_src, nj);
  ex->job_dst = vcopy(P->job_dst, nj);
  ex->job_version = vcopy(P->job_version, nj);
  ex->job_src_job = vcopy(P->job_src_job, nj);
  ex->job_requester = vcopy(P->job_requester, nj);
  ex->block_bytes = vcopy(P->block_bytes, P->n_blocks);
  ex->final_writer = vcopy(P->final_writer, P->n_blocks);
  ex->rank_node = O->rank_node;
  ex->host_in = O->host_in;
  ex->host_out = O->host_out;
  ex->host_side_out = O->host_side_out;
  ex->device_input = O->device_input;
  ex->task_weight = vcopy(O->task_weight, n);
  ex->priority_levels = O->task_weight ? O->priority_levels : 0;
  ex->dev.assign(O->devices, O->devices + P->k);
  ex->base.assign(P->k, nullptr);
  ex->ipc.assign(P->k, 0);
  ex->replica.assign(P->k, nullptr);
  ex->status.assign(P->k, nullptr);
  ex->scratch.assign(P->k, nullptr);
  ex->stamps.assign(P->k, nullptr);
  ex->trace = O->trace;
  plan_layout(ex);
  int64_t host_total = 0;
  for (int b = 0; b < ex->n_blocks; ++b) host_total += ex->blk_doubles[b];
  int rc = HG_OK;
  for (int g = 0; g < P->k && rc == HG_OK; ++g) {
    const int node = g + 1;
    if (!ex->is_local(node)) continue;
    if (cudaSetDevice(ex->dev[g]) != cudaSuccess) {
      set_error("cudaSetDevice(%d) failed", ex->dev[g]);
      rc = HG_ECUDA;
      break;
    }
    if ((rc = ensure_attributes(ex->dev[g]))) break;
    for (int h = 0; h < P->k && ex->rank_node == 0; ++h) {
      if (h == g || ex->dev[h] == ex->dev[g]) continue;
      // a p2p plan moves tiles GPU->GPU directly (platform.py:117); without peer access the copy
      // engine would silently stage through host memory, which is a different machine model
      int can = 0;
      cudaDeviceCanAccessPeer(&can, ex->dev[g], ex->dev[h]);
      if (!can && ex->p2p) {
        set_error("devices %d and %d have no peer access: a p2p=True plan needs NVLink/P2P between "
                  "every pair of its GPUs (plan with p2p=False for host-staged routes)", ex->dev[g], ex->dev[h]);
        rc = HG_EPEER;
        break;
      }
      if (can) {
        cudaError_t e = cudaDeviceEnablePeerAccess(ex->dev[h], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          set_error("peer access %d->%d: %s", ex->dev[g], ex->dev[h], cudaGetErrorString(e));
          rc = HG_ECUDA;
        }
        cudaGetLastError();
      }
    }
    if (rc) break;
    if (cudaMalloc(&ex->base[g], size_t(ex->pool_doubles[g]) * 8) != cudaSuccess ||
        cudaMalloc(&ex->status[g], sizeof(int)) != cudaSuccess) {
      set_error("cudaMalloc of the tile pool failed on device %d (%lld bytes)", ex->dev[g],
                (long long)ex->pool_doubles[g] * 8);
      rc = HG_ECUDA;
      break;
    }
    if (ex->trace) {
      const size_t sb = size_t(2) * (size_t(P->n_tasks) + P->n_jobs) * sizeof(unsigned long long);
      if (cudaMalloc(&ex->stamps[g], sb) != cudaSuccess || cudaMemset(ex->stamps[g], 0, sb) != cudaSuccess) {
        set_error("trace stamp buffer allocation failed on device %d", ex->dev[g]);
        rc = HG_ECUDA;
        break;
      }
    }
    cudaMemset(ex->base[g], 0, size_t(ex->header_doubles) * 8);  // flags + epoch
    cudaMemset(ex->status[g], 0, sizeof(int));
    int64_t sc = 0;
    for (int t = 0; t < P->n_tasks; ++t)
      if (ex->task_node[t] == node) sc += task_scratch_ints(ex->task_kind[t], P->nb, P->ib);
    if (sc > 0 && (cudaMalloc(&ex->scratch[g], size_t(sc) * sizeof(int)) != cudaSuccess ||
                   cudaMemset(ex->scratch[g], 0, size_t(sc) * sizeof(int)) != cudaSuccess)) {
      set_error("scratch allocation failed on device %d", ex->dev[g]);
      rc = HG_ECUDA;
      break;
    }
    if (O->device_input) {
      if (cudaMalloc(&ex->replica[g], size_t(host_total) * 8) != cudaSuccess ||
          cudaMemcpy(ex->replica[g], O->host_in, size_t(host_total) * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
        set_error("device replica of the input failed on device %d", ex->dev[g]);
        rc = HG_ECUDA;
        break;
      }
    }
  }
  if (rc == HG_OK) {
    const int first = ex->rank_node ? ex->rank_node : 1;
    ex->aux_stream.assign(P->k, nullptr);
    ex->ev_reset.assign(P->k, nullptr);
    for (int g = 0; g < P->k && rc == HG_OK && ex->rank_node == 0; ++g) {
      if (g + 1 == first) continue;
      cudaSetDevice(ex->dev[g]);
      if (cudaStreamCreateWithFlags(&ex->aux_stream[g], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&ex->ev_reset[g], cudaEventDisableTiming) != cudaSuccess) {
        set_error("stream/event creation failed on device %d", ex->dev[g]);
        rc = HG_ECUDA;
      }
    }
    cudaSetDevice(ex->dev[first - 1]);
    if (rc == HG_OK &&
        (cudaStreamCreateWithFlags(&ex->stream, cudaStreamNonBlocking) != cudaSuccess ||
         cudaEventCreate(&ex->ev0) != cudaSuccess || cudaEventCreate(&ex->ev1) != cudaSuccess ||
         cudaEventCreateWithFlags(&ex->ev_prev, cudaEventDisableTiming) != cudaSuccess)) {
      set_error("stream/event creation failed");
      rc = HG_ECUDA;
    }
  }
  if (rc == HG_OK && ex->rank_node == 0) rc = build_graph(ex);
  if (rc != HG_OK) {
    release(ex);
    return rc;
  }
  *out = ex;
  return HG_OK;
}

extern "C" int hg_exec_ipc_handle(hg_exec* ex, void* handle64) {
  if (!ex || !handle64 || ex->rank_node == 0) {
    set_error("hg_exec_ipc_handle: needs a per-rank executor");
    return HG_EINVAL;
  }
  cudaIpcMemHandle_t h;
  HG_CUDA(cudaSetDevice(ex->dev[ex->rank_node - 1]));
  HG_CUDA(cudaIpcGetMemHandle(&h, ex->base[ex->rank_node - 1]));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
  memcpy(handle64, &h, 64);
  return HG_OK;
}

extern "C" int hg_exec_ipc_open(hg_exec* ex, int32_t node, const void* handle64) {
  if (!ex || !handle64 || ex->rank_node == 0 || node < 1 || node > ex->k || node == ex->rank_node) {
    set_error("hg_exec_ipc_open: bad arguments");
    return HG_EINVAL;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  void* p = nullptr;
  HG_CUDA(cudaSetDevice(ex->dev[ex->rank_node - 1]));
  HG_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  ex->base[node - 1] = static_cast<double*>(p);
  ex->ipc[node - 1] = 1;
  return HG_OK;
}

extern "C" int hg_exec_build(hg_exec* ex) {
  if (!ex || ex->built) {
    set_error("hg_exec_build: bad handle or already built");
    return HG_EINVAL;
  }
  for (int g = 0; g < ex->k; ++g)
    if (!ex->base[g]) {
      set_error("hg_exec_build: pool of node %d is not mapped (hg_exec_ipc_open)", g + 1);
      return HG_EINVAL;
    }
  return build_graph(ex);
}

extern "C" int hg_exec_partition(const hg_exec_plan* P, int32_t rank_node, int32_t* counts4, int32_t* waits,
                                 int32_t* signals) {
  if (!P || !counts4) {
    set_error("hg_exec_partition: bad arguments");
    return HG_EINVAL;
  }
  hg_exec ex;
  ex.k = P->k;
  ex.n_tasks = P->n_tasks;
  ex.n_jobs = P->n_jobs;
  ex.rank_node = rank_node;
  const int n = P->n_tasks, nj = P->n_jobs;
  ex.task_node = vcopy(P->task_node, n);
  ex.pred_ptr = vcopy(P->pred_ptr, n + 1);
  ex.pred = vcopy(P->pred, P->pred_ptr[n]);
  ex.job_dst = vcopy(P->job_dst, nj);
  ex.job_version = vcopy(P->job_version, nj);
  ex.job_src_job = vcopy(P->job_src_job, nj);
  ex.job_src = vcopy(P->job_src, nj);
  ex.task_kind = vcopy(P->task_kind, n);
  ex.job_block = vcopy(P->job_block, nj);
  ex.nb = P->nb;
  ex.ib = P->ib;
  ex.n_blocks = P->n_blocks;
  ex.blk_doubles.resize(P->n_blocks);
  for (int b = 0; b < P->n_blocks; ++b) ex.blk_doubles[b] = P->block_bytes[b] / 8;
  ex.p2p = P->p2p;
  ex.push = P->push;
  plan_push(&ex);
  Partition part = partition(&ex);
  counts4[0] = part.n_local_tasks;
  counts4[1] = part.n_local_jobs;
  counts4[2] = part.n_waits;
  counts4[3] = part.n_signals;
  // flag ids: task t -> t, job j -> n_tasks + j
  int nw = 0, ns = 0;
  for (int f = 0; f < n + nj; ++f) {
    if (waits && part.waited[f]) waits[nw++] = f;
    const bool sig = f < n ? (part.sig_task[f] && ex.is_local(ex.task_node[f]))
                           : (part.sig_job[f - n] && ex.is_local(ex.job_dst[f - n]));
    if (signals && sig) signals[ns++] = f;
  }
  return HG_OK;
}

static int all_status(hg_exec* ex, int* bad) {
  *bad = 0;
  for (int g = 0; g < ex->k; ++g) {
    if (!ex->is_local(g + 1)) continue;
    int st = 0;
    HG_CUDA(cudaSetDevice(ex->dev[g]));
    HG_CUDA(cudaMemcpy(&st, ex->status[g], sizeof(int), cudaMemcpyDeviceToHost));
    *bad |= st;
  }
  return HG_OK;
}

static int status_error(const hg_exec* ex, int bad) {
  if (bad & hg::kStatusWaitTimeout) {
    set_error("a cross-rank wait timed out after %.1f s: a peer rank died or ranks executed different "
              "plans/partitions (hg_exec_set_wait_timeout)", double(ex->wait_timeout_ns) * 1e-9);
    return HG_EDEADLOCK;
  }
  if (bad & 1) {
    set_error("POTRF: matrix is not positive definite (non-positive pivot)");
    return HG_ENOTSPD;
  }
  if (bad & 2) {
    set_error("LU: exactly zero pivot encountered");
    return HG_ESINGULAR;
  }
  return HG_OK;
}

// Asynchronous launch on exactly the caller's stream (NULL = the legacy
// default stream); pair with hg_exec_wait.  Lets a caller bracket K
// back-to-back runs with its own CUDA events on that stream.
extern "C" int hg_exec_launch(hg_exec* ex, void* stream) {
  if (!ex || !ex->built) {
    set_error("hg_exec_launch: null handle or graph not built");
    return HG_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ex->epoch++;
  const int first = ex->rank_node ? ex->rank_node : 1;
  // status resets: the first device's on the launch stream; every other device's (single-process
  // mode) on its own stream, after everything enqueued on `s` so far (the previous run) and before
  // this run's graph -- fully asynchronous, no host synchronisation
  HG_CUDA(cudaSetDevice(ex->dev[first - 1]));
  HG_CUDA(cudaMemsetAsync(ex->status[first - 1], 0, sizeof(int), s));
  if (ex->rank_node) {  // flags are only used across processes
    hg::k_set_epoch<<<1, 32, 0, s>>>(ex->epoch_ptr(first), ex->epoch);
    HG_CUDA(cudaGetLastError());
  } else if (ex->k > 1) {
    HG_CUDA(cudaEventRecord(ex->ev_prev, s));
    for (int g = 0; g < ex->k; ++g) {
      if (g + 1 == first) continue;
      HG_CUDA(cudaSetDevice(ex->dev[g]));
      HG_CUDA(cudaStreamWaitEvent(ex->aux_stream[g], ex->ev_prev, 0));
      HG_CUDA(cudaMemsetAsync(ex->status[g], 0, sizeof(int), ex->aux_stream[g]));
      HG_CUDA(cudaEventRecord(ex->ev_reset[g], ex->aux_stream[g]));
    }
    HG_CUDA(cudaSetDevice(ex->dev[first - 1]));
    for (int g = 0; g < ex->k; ++g)
      if (g + 1 != first) HG_CUDA(cudaStreamWaitEvent(s, ex->ev_reset[g], 0));
  }
  if (ex->rank_node) {
    hg::StepFence f{};
    for (int g = 0; g < ex->k && f.n < 16; ++g)
      if (g + 1 != ex->rank_node) f.peer_done[f.n++] = ex->done_ptr(g + 1);
    f.need = ex->epoch - 1;
    f.status = ex->status[first - 1];
    f.timeout_ns = ex->wait_timeout_ns;
    if (ex->k > 17) {
      set_error("hg_exec_launch: step fence supports up to 17 ranks");
      return HG_EINVAL;
    }
    hg::k_wait_peers_done<<<1, 32, 0, s>>>(f);
    HG_CUDA(cudaGetLastError());
  }
  HG_CUDA(cudaGraphLaunch(ex->exec, s));
  if (ex->rank_node) {
    hg::k_mark_done<<<1, 32, 0, s>>>(ex->done_ptr(ex->rank_node), ex->epoch);
    HG_CUDA(cudaGetLastError());
  }
  ex->last_stream = s;
  ex->launched = true;
  return HG_OK;
}

extern "C" int hg_exec_wait(hg_exec* ex) {
  if (!ex) {
    set_error("hg_exec_wait: null handle");
    return HG_EINVAL;
  }
  const int first = ex->rank_node ? ex->rank_node : 1;
  HG_CUDA(cudaSetDevice(ex->dev[first - 1]));
  HG_CUDA(cudaStreamSynchronize(ex->launched ? ex->last_stream : ex->stream));
  ex->launched = false;
  int bad = 0;
  int rc = all_status(ex, &bad);
  if (rc) return rc;
  HG_CUDA(cudaSetDevice(ex->dev[first - 1]));
  return status_error(ex, bad);
}

extern "C" int hg_exec_run(hg_exec* ex, hg_exec_stats* stats) {
  if (!ex || !ex->built) {
    set_error("hg_exec_run: null handle or graph not built");
    return HG_EINVAL;
  }
  const int first = ex->rank_node ? ex->rank_node : 1;
  HG_CUDA(cudaSetDevice(ex->dev[first - 1]));
  HG_CUDA(cudaEventRecord(ex->ev0, ex->stream));
  int rc = hg_exec_launch(ex, ex->stream);
  if (rc) return rc;
  HG_CUDA(cudaSetDevice(ex->dev[first - 1]));
  HG_CUDA(cudaEventRecord(ex->ev1, ex->stream));
  rc = hg_exec_wait(ex);
  float ms = 0.f;
  HG_CUDA(cudaEventElapsedTime(&ms, ex->ev0, ex->ev1));
  ex->stats.elapsed_ms = ms;
  if (stats) *stats = ex->stats;
  return rc;
}

extern "C" int hg_exec_info(hg_exec* ex, hg_exec_stats* stats) {
  if (!ex || !stats) {
    set_error("hg_exec_info: bad arguments");
    return HG_EINVAL;
  }
  *stats = ex->stats;
  return HG_OK;
}

extern "C" int hg_exec_read_block(hg_exec* ex, int32_t block, int32_t node, double* host, int64_t doubles) {
  if (!ex || block < 0 || block >= ex->n_blocks || node < 1 || node > ex->k || !ex->base[node - 1]) {
    set_error("hg_exec_read_block: bad arguments");
    return HG_EINVAL;
  }
  int64_t off = ex->slot[node - 1][block];
  if (off < 0) {
    set_error("block %d never resident on node %d", block, node);
    return HG_EINVAL;
  }
  if (doubles > ex->slot_doubles[block]) doubles = ex->slot_doubles[block];
  const int first = ex->rank_node ? ex->rank_node : node;
  HG_CUDA(cudaSetDevice(ex->dev[first - 1]));
  HG_CUDA(cudaMemcpy(host, ex->base[node - 1] + off, size_t(doubles) * 8, cudaMemcpyDefault));
  return HG_OK;
}

extern "C" int hg_exec_destroy(hg_exec* ex) {
  release(ex);
  return HG_OK;
}

extern "C" int hg_exec_read_stamps(hg_exec* ex, uint64_t* out) {
  if (!ex || !out || !ex->trace) {
    set_error("hg_exec_read_stamps: bad handle or executor created without opts.trace");
    return HG_EINVAL;
  }
  const int64_t n = ex->n_tasks, nj = ex->n_jobs;
  std::fill(out, out + 2 * (n + nj), uint64_t(0));
  std::vector<unsigned long long> buf(size_t(2) * (n + nj));
  for (int g = 0; g < ex->k; ++g) {
    if (!ex->is_local(g + 1) || !ex->stamps[g]) continue;
    HG_CUDA(cudaSetDevice(ex->dev[g]));
    HG_CUDA(cudaMemcpy(buf.data(), ex->stamps[g], buf.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    for (int64_t t = 0; t < n; ++t)
      if (ex->task_node[t] == g + 1) out[2 * t] = buf[2 * t], out[2 * t + 1] = buf[2 * t + 1];
    for (int64_t j = 0; j < nj; ++j)
      if (ex->job_dst[j] == g + 1)
        out[2 * (n + j)] = buf[2 * (n + j)], out[2 * (n + j) + 1] = buf[2 * (n + j) + 1];
  }
  return HG_OK;
}

extern "C" int hg_exec_set_wait_timeout(hg_exec* ex, double seconds) {
  if (!ex || !(seconds > 0.0) || ex->built) {
    set_error("hg_exec_set_wait_timeout: bad handle, non-positive timeout, or graph already built");
    return HG_EINVAL;
  }
  ex->wait_timeout_ns = (unsigned long long)(seconds * 1e9);
  return HG_OK;
}

// Teardown of the one-process-per-GPU mode: unmap every peer pool (cudaIpcCloseMemHandle) while
// this rank's own pool stays allocated.  The Python side runs: wait -> barrier -> hg_exec_ipc_close
// -> barrier -> hg_exec_destroy, so no rank frees an exported pool a peer still reads or maps.
extern "C" int hg_exec_ipc_close(hg_exec* ex) {
  if (!ex || ex->rank_node == 0) {
    set_error("hg_exec_ipc_close: needs a per-rank executor");
    return HG_EINVAL;
  }
  HG_CUDA(cudaSetDevice(ex->dev[ex->rank_node - 1]));
  for (int g = 0; g < ex->k; ++g) {
    if (ex->ipc[g] && ex->base[g]) {
      HG_CUDA(cudaIpcCloseMemHandle(ex->base[g]));
      ex->base[g] = nullptr;
      ex->ipc[g] = 0;
    }
  }
  return HG_OK;
}

// Page-lock caller-owned host memory (the tile-major input / output images) so the plan's H2D
// jobs and the write-back run as async DMA instead of staged pageable copies.  The caller keeps
// ownership; hg_matrix_unregister before freeing it.
extern "C" int hg_matrix_register(void* host, size_t bytes) {
  if (!host || bytes == 0) {
    set_error("hg_matrix_register: null pointer or empty range");
    return HG_EINVAL;
  }
  cudaError_t e = cudaHostRegister(host, bytes, cudaHostRegisterPortable);
  if (e == cudaErrorHostMemoryAlreadyRegistered) {
    cudaGetLastError();
    return HG_OK;
  }
  if (e != cudaSuccess) {
    set_error("cudaHostRegister(%p, %zu): %s", host, bytes, cudaGetErrorString(e));
    cudaGetLastError();
    return HG_ECUDA;
  }
  return HG_OK;
}

extern "C" int hg_matrix_unregister(void* host) {
  if (!host) {
    set_error("hg_matrix_unregister: null pointer");
    return HG_EINVAL;
  }
  cudaError_t e = cudaHostUnregister(host);
  if (e != cudaSuccess && e != cudaErrorHostMemoryNotRegistered) {
    set_error("cudaHostUnregister(%p): %s", host, cudaGetErrorString(e));
    cudaGetLastError();
    return HG_ECUDA;
  }
  cudaGetLastError();
  return HG_OK;
}
