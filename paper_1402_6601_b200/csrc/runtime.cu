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

}  // extern "C"

// ---------------------------------------------------------------------------
struct hg_exec {
  int k = 0, nb = 0, ib = 0, side = 0;
  int n_blocks = 0;
  std::vector<int> dev;                 // node g+1 -> device
  std::vector<double*> pool;            // per GPU node
  std::vector<double*> replica;         // per GPU node: device copy of host_in (device_input)
  std::vector<int*> status;             // per GPU node
  std::vector<int*> scratch;            // per GPU node: per-task scratch ints
  std::vector<std::vector<int64_t>> slot;  // [node-1][block] -> offset in doubles, -1 = none
  std::vector<int64_t> host_off;        // doubles offset of each block in the host image
  std::vector<int64_t> blk_doubles;     // host-image doubles per block
  std::vector<int64_t> slot_doubles;    // device slot doubles per block
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  hg_exec_stats stats{};
  cudaStream_t last_stream = nullptr;
  bool launched = false;
};

static void release(hg_exec* ex) {
  if (!ex) return;
  if (ex->exec) cudaGraphExecDestroy(ex->exec);
  if (ex->graph) cudaGraphDestroy(ex->graph);
  for (int g = 0; g < ex->k; ++g) {
    cudaSetDevice(ex->dev[g]);
    if (g < (int)ex->pool.size() && ex->pool[g]) cudaFree(ex->pool[g]);
    if (g < (int)ex->replica.size() && ex->replica[g]) cudaFree(ex->replica[g]);
    if (g < (int)ex->status.size() && ex->status[g]) cudaFree(ex->status[g]);
    if (g < (int)ex->scratch.size() && ex->scratch[g]) cudaFree(ex->scratch[g]);
  }
  if (ex->ev0) cudaEventDestroy(ex->ev0);
  if (ex->ev1) cudaEventDestroy(ex->ev1);
  if (ex->stream) cudaStreamDestroy(ex->stream);
  delete ex;
}

static int build_graph(hg_exec* ex, const hg_exec_plan* P, const hg_exec_opts* O) {
  const int n = P->n_tasks;
  HG_CUDA(cudaGraphCreate(&ex->graph, 0));
  std::vector<cudaGraphNode_t> task_last(n, nullptr), task_first(n, nullptr);
  std::vector<cudaGraphNode_t> job_node(P->n_jobs, nullptr);
  // jobs grouped by requester, in job order
  std::vector<std::vector<int>> jobs_of(n);
  for (int j = 0; j < P->n_jobs; ++j) jobs_of[P->job_requester[j]].push_back(j);
  std::vector<LaunchDesc> launches;
  std::vector<cudaGraphNode_t> deps;
  int64_t side_bytes = 0;
  std::vector<int64_t> scratch_used(ex->k, 0);

  auto slot_ptr = [&](int node, int block) -> double* {
    int64_t off = ex->slot[node - 1][block];
    return off < 0 ? nullptr : ex->pool[node - 1] + off;
  };

  for (int di = 0; di < n; ++di) {
    const int t = P->dispatch[di];
    // 1) the copy jobs this dispatch created
    for (int j : jobs_of[t]) {
      const int b = P->job_block[j], src = P->job_src[j], dst = P->job_dst[j];
      deps.clear();
      if (P->job_src_job[j] >= 0) deps.push_back(job_node[P->job_src_job[j]]);
      else if (P->job_version[j] >= 0) deps.push_back(task_last[P->job_version[j]]);
      double* dptr = slot_ptr(dst, b);
      const void* sptr;
      size_t bytes;
      if (src == 0) {
        bytes = size_t(ex->blk_doubles[b]) * 8;
        if (P->job_version[j] >= 0 || P->job_src_job[j] >= 0) {
          set_error("job %d: host-staged versions (p2p=False) are not executable", j);
          return HG_EINVAL;
        }
        sptr = O->device_input ? (const void*)(ex->replica[dst - 1] + ex->host_off[b])
                               : (const void*)(O->host_in + ex->host_off[b]);
        if (O->device_input) ex->stats.bytes_d2d += 0;  // served from HBM, still an H2D job of the plan
        ex->stats.bytes_h2d += bytes;
      } else if (dst == 0) {
        set_error("job %d: device->host jobs are not executable on a GPU-only platform", j);
        return HG_EINVAL;
      } else {
        bytes = size_t(ex->slot_doubles[b]) * 8;
        sptr = slot_ptr(src, b);
        ex->stats.bytes_d2d += size_t(ex->blk_doubles[b]) * 8;
        side_bytes += bytes - size_t(ex->blk_doubles[b]) * 8;
      }
      if (!dptr || !sptr) {
        set_error("job %d: missing slot (block %d, %d -> %d)", j, b, src, dst);
        return HG_EINVAL;
      }
      HG_CUDA(cudaSetDevice(ex->dev[dst - 1]));
      HG_CUDA(cudaGraphAddMemcpyNode1D(&job_node[j], ex->graph, deps.data(), deps.size(), dptr, sptr,
                                       bytes, cudaMemcpyDefault));
      ex->stats.n_copy_nodes++;
    }
    // 2) the task's kernel chain
    const int node = P->task_node[t];
    TaskOperands ops;
    ops.nb = ex->nb;
    ops.ib = ex->ib;
    ops.status = ex->status[node - 1];
    const int sc = task_scratch_ints(P->task_kind[t], ex->nb, ex->ib);
    if (sc > 0) {
      ops.scratch = ex->scratch[node - 1] + scratch_used[node - 1];
      scratch_used[node - 1] += sc;
    }
    const int64_t a0 = P->acc_ptr[t], a1 = P->acc_ptr[t + 1];
    if (a1 - a0 > 4) {
      set_error("task %d has %lld accesses (max 4)", t, (long long)(a1 - a0));
      return HG_EINVAL;
    }
    for (int64_t a = a0; a < a1; ++a) ops.t[ops.n_t++] = slot_ptr(node, P->acc_block[a]);
    launches.clear();
    if (!build_task_launches(P->task_kind[t], ops, launches)) return HG_EINVAL;
    deps.clear();
    for (int64_t w = P->wait_ptr[t]; w < P->wait_ptr[t + 1]; ++w) deps.push_back(job_node[P->wait_job[w]]);
    for (int64_t q = P->pred_ptr[t]; q < P->pred_ptr[t + 1]; ++q) deps.push_back(task_last[P->pred[q]]);
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
      kp.extra = nullptr;
      cudaGraphNode_t nd;
      if (li == 0) {
        HG_CUDA(cudaGraphAddKernelNode(&nd, ex->graph, deps.data(), deps.size(), &kp));
        task_first[t] = nd;
      } else {
        HG_CUDA(cudaGraphAddKernelNode(&nd, ex->graph, &prev, 1, &kp));
      }
      prev = nd;
      ex->stats.n_kernel_nodes++;
    }
    task_last[t] = prev;
  }
  // 3) write-back of final versions
  if (O->host_out) {
    for (int b = 0; b < ex->n_blocks; ++b) {
      const int w = P->final_writer[b];
      if (w < 0) continue;
      const int node = P->task_node[w];
      size_t bytes = size_t(ex->blk_doubles[b]) * 8;
      cudaGraphNode_t nd;
      HG_CUDA(cudaSetDevice(ex->dev[node - 1]));
      HG_CUDA(cudaGraphAddMemcpyNode1D(&nd, ex->graph, &task_last[w], 1, O->host_out + ex->host_off[b],
                                       slot_ptr(node, b), bytes, cudaMemcpyDefault));
      ex->stats.bytes_d2h += bytes;
      ex->stats.n_copy_nodes++;
      if (O->host_side_out && ex->side > 0 && ex->slot_doubles[b] > ex->blk_doubles[b]) {
        HG_CUDA(cudaGraphAddMemcpyNode1D(&nd, ex->graph, &task_last[w], 1,
                                         O->host_side_out + int64_t(b) * ex->side,
                                         slot_ptr(node, b) + ex->blk_doubles[b], size_t(ex->side) * 8,
                                         cudaMemcpyDefault));
        ex->stats.n_copy_nodes++;
      }
    }
  }
  ex->stats.bytes_side = side_bytes;
  HG_CUDA(cudaSetDevice(ex->dev[0]));
  HG_CUDA(cudaGraphInstantiate(&ex->exec, ex->graph, 0));
  return HG_OK;
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
  hg_exec* ex = new hg_exec();
  ex->k = P->k;
  ex->nb = P->nb;
  ex->ib = P->ib;
  ex->side = P->side_doubles;
  ex->n_blocks = P->n_blocks;
  ex->dev.assign(O->devices, O->devices + P->k);
  ex->pool.assign(P->k, nullptr);
  ex->replica.assign(P->k, nullptr);
  ex->status.assign(P->k, nullptr);
  ex->scratch.assign(P->k, nullptr);
  const int64_t tile_d = int64_t(P->nb) * P->nb;
  ex->host_off.resize(P->n_blocks);
  ex->blk_doubles.resize(P->n_blocks);
  ex->slot_doubles.resize(P->n_blocks);
  int64_t host_total = 0;
  for (int b = 0; b < P->n_blocks; ++b) {
    ex->blk_doubles[b] = P->block_bytes[b] / 8;
    ex->slot_doubles[b] = ex->blk_doubles[b] + (ex->blk_doubles[b] == tile_d ? P->side_doubles : 0);
    ex->host_off[b] = host_total;
    host_total += ex->blk_doubles[b];
  }
  // slots: (block, node) pairs the plan ever touches
  ex->slot.assign(P->k, std::vector<int64_t>(P->n_blocks, -1));
  std::vector<int64_t> used(P->k, 0);
  auto need = [&](int node, int b) {
    if (node < 1 || node > P->k) return;
    int64_t& s = ex->slot[node - 1][b];
    if (s < 0) {
      s = used[node - 1];
      used[node - 1] += (ex->slot_doubles[b] + 31) / 32 * 32;  // 256-byte aligned slots
    }
  };
  for (int t = 0; t < P->n_tasks; ++t)
    for (int64_t a = P->acc_ptr[t]; a < P->acc_ptr[t + 1]; ++a) need(P->task_node[t], P->acc_block[a]);
  for (int j = 0; j < P->n_jobs; ++j) need(P->job_dst[j], P->job_block[j]);
  int rc = HG_OK;
  for (int g = 0; g < P->k && rc == HG_OK; ++g) {
    if (cudaSetDevice(ex->dev[g]) != cudaSuccess) {
      set_error("cudaSetDevice(%d) failed", ex->dev[g]);
      rc = HG_ECUDA;
      break;
    }
    if ((rc = ensure_attributes(ex->dev[g]))) break;
    for (int h = 0; h < P->k; ++h) {
      if (h == g || ex->dev[h] == ex->dev[g]) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, ex->dev[g], ex->dev[h]);
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
    if (cudaMalloc(&ex->pool[g], size_t(std::max<int64_t>(used[g], 32)) * 8) != cudaSuccess ||
        cudaMalloc(&ex->status[g], sizeof(int)) != cudaSuccess) {
      set_error("cudaMalloc of the tile pool failed on device %d (%lld bytes)", ex->dev[g],
                (long long)used[g] * 8);
      rc = HG_ECUDA;
      break;
    }
    cudaMemset(ex->status[g], 0, sizeof(int));
    int64_t sc = 0;
    for (int t = 0; t < P->n_tasks; ++t)
      if (P->task_node[t] == g + 1) sc += task_scratch_ints(P->task_kind[t], P->nb, P->ib);
    if (sc > 0) {
      if (cudaMalloc(&ex->scratch[g], size_t(sc) * sizeof(int)) != cudaSuccess ||
          cudaMemset(ex->scratch[g], 0, size_t(sc) * sizeof(int)) != cudaSuccess) {
        set_error("scratch allocation failed on device %d", ex->dev[g]);
        rc = HG_ECUDA;
        break;
      }
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
    cudaSetDevice(ex->dev[0]);
    if (cudaStreamCreateWithFlags(&ex->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&ex->ev0) != cudaSuccess || cudaEventCreate(&ex->ev1) != cudaSuccess) {
      set_error("stream/event creation failed");
      rc = HG_ECUDA;
    }
  }
  if (rc == HG_OK) rc = build_graph(ex, P, O);
  if (rc != HG_OK) {
    release(ex);
    return rc;
  }
  *out = ex;
  return HG_OK;
}

extern "C" int hg_exec_run(hg_exec* ex, hg_exec_stats* stats) {
  if (!ex) {
    set_error("hg_exec_run: null handle");
    return HG_EINVAL;
  }
  for (int g = 0; g < ex->k; ++g) {
    HG_CUDA(cudaSetDevice(ex->dev[g]));
    HG_CUDA(cudaMemset(ex->status[g], 0, sizeof(int)));
  }
  HG_CUDA(cudaSetDevice(ex->dev[0]));
  HG_CUDA(cudaEventRecord(ex->ev0, ex->stream));
  HG_CUDA(cudaGraphLaunch(ex->exec, ex->stream));
  HG_CUDA(cudaEventRecord(ex->ev1, ex->stream));
  HG_CUDA(cudaEventSynchronize(ex->ev1));
  float ms = 0.f;
  HG_CUDA(cudaEventElapsedTime(&ms, ex->ev0, ex->ev1));
  int bad = 0;
  for (int g = 0; g < ex->k; ++g) {
    int st = 0;
    HG_CUDA(cudaSetDevice(ex->dev[g]));
    HG_CUDA(cudaMemcpy(&st, ex->status[g], sizeof(int), cudaMemcpyDeviceToHost));
    bad |= st;
  }
  HG_CUDA(cudaSetDevice(ex->dev[0]));
  ex->stats.elapsed_ms = ms;
  if (stats) *stats = ex->stats;
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
  if (!ex) {
    set_error("hg_exec_launch: null handle");
    return HG_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int g = 0; g < ex->k; ++g) {
    HG_CUDA(cudaSetDevice(ex->dev[g]));
    HG_CUDA(cudaMemsetAsync(ex->status[g], 0, sizeof(int), g == 0 ? s : nullptr));
  }
  HG_CUDA(cudaSetDevice(ex->dev[0]));
  HG_CUDA(cudaGraphLaunch(ex->exec, s));
  ex->last_stream = s;
  ex->launched = true;
  return HG_OK;
}

extern "C" int hg_exec_wait(hg_exec* ex) {
  if (!ex) {
    set_error("hg_exec_wait: null handle");
    return HG_EINVAL;
  }
  HG_CUDA(cudaSetDevice(ex->dev[0]));
  HG_CUDA(cudaStreamSynchronize(ex->launched ? ex->last_stream : ex->stream));
  ex->launched = false;
  int bad = 0;
  for (int g = 0; g < ex->k; ++g) {
    int st = 0;
    HG_CUDA(cudaSetDevice(ex->dev[g]));
    HG_CUDA(cudaMemcpy(&st, ex->status[g], sizeof(int), cudaMemcpyDeviceToHost));
    bad |= st;
  }
  HG_CUDA(cudaSetDevice(ex->dev[0]));
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

extern "C" int hg_exec_info(hg_exec* ex, hg_exec_stats* stats) {
  if (!ex || !stats) {
    set_error("hg_exec_info: bad arguments");
    return HG_EINVAL;
  }
  *stats = ex->stats;
  return HG_OK;
}

extern "C" int hg_exec_read_block(hg_exec* ex, int32_t block, int32_t node, double* host, int64_t doubles) {
  if (!ex || block < 0 || block >= ex->n_blocks || node < 1 || node > ex->k) {
    set_error("hg_exec_read_block: bad arguments");
    return HG_EINVAL;
  }
  int64_t off = ex->slot[node - 1][block];
  if (off < 0) {
    set_error("block %d never resident on node %d", block, node);
    return HG_EINVAL;
  }
  if (doubles > ex->slot_doubles[block]) doubles = ex->slot_doubles[block];
  HG_CUDA(cudaSetDevice(ex->dev[node - 1]));
  HG_CUDA(cudaMemcpy(host, ex->pool[node - 1] + off, size_t(doubles) * 8, cudaMemcpyDeviceToHost));
  return HG_OK;
}

extern "C" int hg_exec_destroy(hg_exec* ex) {
  release(ex);
  return HG_OK;
}
