/*
 * hetgpu.h -- C-ABI of libhetgpu.so, the B200-native execution path for the
 * data-flow tiled FP64 factorizations of arXiv 1402.6601.
 *
 * The reference (`hetsim`, pure Python) has no FFI; its execution layer is
 * the simulator `run(graph, platform, scheduler, model, ...)`
 * (/root/reference/pkg/src/hetsim/sim.py:388-390) whose task execution call
 * site is `Simulation._start_exec` (sim.py:353-360, `true_exec`) and whose
 * planning decisions come from `scheduler.activate` (sim.py:201 ->
 * sched.py:353-412).  This library replaces:
 *
 *   hg_plan_build  <- sim.py:97-385 event loop + sched.py:229-412 (HEFT,
 *                     DADA) replayed bit-exactly in virtual time
 *   hg_exec_*      <- sim.py:237-385 transfers + `_start_exec`: the planned
 *                     DAG executed on B200s (one CUDA graph; cudaMemcpy
 *                     peer/H2D nodes for transfer jobs, sm_100a tile kernels
 *                     for tasks)
 *   hg_tile_run    <- one tile kernel of kernels.py:23-38 (unit-test /
 *                     calibration entry)
 *
 * Conventions: every function returns 0 on success and a negative HG_E*
 * code otherwise; hg_last_error() returns a thread-local message.  Plain
 * pointers and sizes only; no torch types.  Not re-entrant per handle.
 */
#ifndef HETGPU_H
#define HETGPU_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HG_ABI_VERSION 3

/* error codes */
#define HG_OK 0
#define HG_EINVAL (-1)     /* bad argument / unsupported shape        -> ValueError   */
#define HG_ECUDA (-2)      /* CUDA runtime error                      -> SimulationError */
#define HG_ENOTSPD (-3)    /* POTRF met a non-positive pivot          -> SimulationError */
#define HG_EDEADLOCK (-4)  /* planner: tasks left with no events      -> DeadlockError */
#define HG_EMODEL (-5)     /* planner: missing timing                 -> PerfModelError */
#define HG_ESINGULAR (-6)  /* LU met an exactly zero pivot            -> SimulationError */
#define HG_EPEER (-7)      /* two GPUs of a p2p plan lack peer access -> PlatformError */
/* HG_EDEADLOCK is also returned by hg_exec_wait/run when a cross-rank wait timed out
 * (hg_exec_set_wait_timeout): a dead peer rank or ranks running different plans. */

/* kernel kinds: index in kernels.ALL_KINDS (kernels.py:39-42) */
enum {
  HG_KIND_POTRF = 0, HG_KIND_TRSM, HG_KIND_SYRK, HG_KIND_GEMM,
  HG_KIND_GETRF_INC, HG_KIND_GESSM, HG_KIND_TSTRF, HG_KIND_SSSSM,
  HG_KIND_GEQRT, HG_KIND_UNMQR, HG_KIND_TSQRT, HG_KIND_TSMQR,
  HG_KIND_COUNT
};

/* access modes (graph.py:20-33) */
#define HG_ACCESS_R 1
#define HG_ACCESS_W 2
#define HG_ACCESS_RW 3

const char* hg_last_error(void);
int hg_abi_version(void);
/* number of CUDA devices visible (0 on a CPU-only host; never fails) */
int hg_device_count(void);

/* ------------------------------------------------------------------------
 * Planner (sim.py:97-385 + sched.py:229-412, noise = 0)
 * ---------------------------------------------------------------------- */
typedef struct hg_graph_desc {
  int32_t n_tasks;
  int32_t n_blocks;
  const int32_t* task_kind;   /* index into the model's kind table */
  const double* task_flops;
  const int64_t* acc_ptr;     /* CSR [n_tasks + 1] */
  const int32_t* acc_block;
  const int8_t* acc_mode;     /* HG_ACCESS_* */
  const int64_t* succ_ptr;    /* CSR [n_tasks + 1], ascending */
  const int32_t* succ;
  const int64_t* block_bytes; /* [n_blocks] */
} hg_graph_desc;

typedef struct hg_platform_desc {
  int32_t m, k, n_switches;
  double link_bandwidth;      /* B/s, every link (build_platform) */
  double link_latency;        /* s */
  int32_t switch_slots;       /* Platform.switch_slots, -1 = unlimited */
  int32_t p2p;
} hg_platform_desc;

typedef struct hg_model_desc {
  int32_t n_kinds;
  const double* fallback_cpu; /* [n_kinds], NaN = missing */
  const double* fallback_gpu;
  const int64_t* count_cpu;   /* PerfModel.samples[(kind, cls)][0], -1 if absent */
  const int64_t* count_gpu;
  const double* mean_cpu;     /* PerfModel.samples[(kind, cls)][1] */
  const double* mean_gpu;
  int64_t sample_threshold;
} hg_model_desc;

typedef struct hg_sched_desc {
  int32_t type;               /* 0 = HEFT, 1 = DADA */
  int32_t with_cp;
  double alpha, epsilon, rho;
} hg_sched_desc;

typedef struct hg_plan_out {
  /* per task [n_tasks] */
  int32_t* worker;
  double* start;
  double* end;
  int32_t* dispatch;          /* task ids in global dispatch order */
  int64_t* wait_ptr;          /* [n_tasks + 1] */
  int32_t* wait_job;
  /* per transfer job [n_jobs] */
  int32_t n_jobs;
  int32_t* job_block;
  int32_t* job_src;
  int32_t* job_dst;
  int32_t* job_version;
  int32_t* job_src_job;
  int32_t* job_stage_job;
  int32_t* job_requester;
  int64_t* job_bytes;
  /* totals */
  int64_t bytes_h2d, bytes_d2h, bytes_d2d;
  double makespan;
  double gflops;
  double* busy;               /* [n_workers] */
  int32_t n_workers;
  int32_t n_activations;
  int32_t n_fallbacks;        /* DADA batches that fell back to HEFT */
  double plan_seconds;        /* wall time of the planner itself */
} hg_plan_out;

int hg_plan_build(const hg_graph_desc* g, const hg_platform_desc* p, const hg_model_desc* m,
                  const hg_sched_desc* s, hg_plan_out* out);
void hg_plan_free(hg_plan_out* out);
/* CPython 3.12 builtin sum() over doubles (Neumaier), exposed for parity tests */
double hg_pysum(const double* x, int64_t n);

/* ------------------------------------------------------------------------
 * Executor: one CUDA graph per plan (tile kernels + transfer copies)
 * ---------------------------------------------------------------------- */
typedef struct hg_exec_plan {
  int32_t n_tasks, n_blocks, n_jobs, k;
  int32_t nb, ib;
  int32_t side_doubles;       /* per-tile side area (IPIV / dL / T), 0 for Cholesky */
  const int32_t* task_kind;   /* HG_KIND_* */
  const int32_t* task_node;   /* memory node 1..k */
  const int64_t* acc_ptr;
  const int32_t* acc_block;
  const int64_t* pred_ptr;    /* CSR predecessors */
  const int32_t* pred;
  const int32_t* dispatch;
  const int64_t* wait_ptr;
  const int32_t* wait_job;
  const int32_t* job_block;
  const int32_t* job_src;
  const int32_t* job_dst;
  const int32_t* job_version;
  const int32_t* job_src_job;
  const int32_t* job_requester;
  const int64_t* block_bytes; /* host image bytes per block (tile or T factor) */
  const int32_t* final_writer;/* last writer task per block, -1 = never written */
  const int8_t* acc_mode;     /* HG_ACCESS_* per access (CSR like acc_block) */
  const int32_t* job_stage_job; /* host-staged route: the job whose first leg stages the block, or -1 */
  int32_t p2p;                /* 0: every GPU->GPU job is host-staged (GPU->host->GPU, platform.py:117) */
  int32_t push;               /* 1: producer-push fusion -- a peer job moving a tile version is done by
                                 the producing task's own kernels (stores into the consumer GPU's slot:
                                 store epilogues of POTRF / TRSM / SYRK / GEMM, each column strip of the
                                 LU / QR trailing updates, the last panel kernel of the LU / QR panels
                                 with the side area), not a copy node; at most 8 (GPU, block) pairs per
                                 task; bytes per (version, destination) stay the plan's */
} hg_exec_plan;

typedef struct hg_exec_opts {
  const int32_t* devices;     /* CUDA device of GPU node g+1, [k] */
  const double* host_in;      /* tile-major image, blocks in id order (pinned for async H2D) */
  double* host_out;           /* final versions written back here; NULL = no write-back */
  double* host_side_out;      /* optional: side areas of final tiles, n_blocks*side_doubles */
  int32_t device_input;       /* 1: keep a replica of host_in in each GPU's HBM and serve
                                 the plan's H2D jobs from it (inputs resident in HBM) */
  int32_t rank_node;          /* 0: this process drives every GPU node (one CUDA graph over all
                                 devices).  r+1: one process per GPU -- this process executes
                                 node r+1 only; exchange pools with hg_exec_ipc_handle /
                                 hg_exec_ipc_open, then hg_exec_build */
  const double* task_weight;  /* optional [n_tasks] predicted seconds per task (the plan's
                                 end - start); NULL = no node priorities */
  double* host_stage;         /* p2p = 0 plans: pinned staging image (same layout as host_in) for the
                                 GPU->host legs of host-staged moves; NULL otherwise */
  int32_t priority_levels;    /* >0: kernel nodes get CUDA priorities from the task's slack
                                 (longest path through it vs the DAG's critical path, weights
                                 task_weight) quantised to min(levels, device range) levels;
                                 0 = every node at default priority.  Never changes the plan,
                                 only the order in which ready kernels get SMs. */
  int32_t trace;              /* 1: stamp %globaltimer before/after every task's kernel chain and
                                 every copy job (one 1-thread node each); read with
                                 hg_exec_read_stamps -> the executed schedule (sim.py:66-80 TaskRun,
                                 TraceEvent).  0 = no extra nodes. */
} hg_exec_opts;

typedef struct hg_exec hg_exec;

typedef struct hg_exec_stats {
  double elapsed_ms;          /* device time of the whole graph (CUDA events) */
  int64_t bytes_h2d;          /* bytes moved by the graph's copy nodes, by direction */
  int64_t bytes_d2d;
  int64_t bytes_d2h;          /* incl. final write-back */
  int64_t bytes_side;         /* side-area bytes that rode along with peer copies */
  int32_t n_kernel_nodes;
  int32_t n_copy_nodes;
  int32_t n_push_jobs;        /* plan jobs delivered by producer-push (no copy node) */
} hg_exec_stats;

int hg_exec_create(const hg_exec_plan* plan, const hg_exec_opts* opts, hg_exec** out);
/* one-process-per-GPU mode: export this rank's pool (64-byte cudaIpcMemHandle),
 * map a peer node's pool, then build the rank-local graph.  Cross-rank
 * dependencies are device flags (release/acquire, system scope) carrying the
 * run's epoch. */
int hg_exec_ipc_handle(hg_exec* ex, void* handle64);
int hg_exec_ipc_open(hg_exec* ex, int32_t node, const void* handle64);
int hg_exec_build(hg_exec* ex);
/* CPU-only dry run of the per-rank partition: counts4 = {local tasks, local
 * copy jobs, remote flags waited on, flags signalled}; optional id lists
 * (capacity n_tasks + n_jobs; flag id = task id, or n_tasks + job id) */
int hg_exec_partition(const hg_exec_plan* plan, int32_t rank_node, int32_t* counts4, int32_t* waits,
                      int32_t* signals);
int hg_exec_run(hg_exec* ex, hg_exec_stats* stats);
/* asynchronous variant: launch on exactly `stream` (NULL = legacy default stream), then wait */
int hg_exec_launch(hg_exec* ex, void* stream);
int hg_exec_wait(hg_exec* ex);
int hg_exec_info(hg_exec* ex, hg_exec_stats* stats);
int hg_exec_read_block(hg_exec* ex, int32_t block, int32_t node, double* host, int64_t doubles);
int hg_exec_destroy(hg_exec* ex);
/* one-process-per-GPU mode: bound on every cross-rank spin (flag waits, the step fence);
 * default 60 s; set before hg_exec_build.  A wait that gives up makes hg_exec_wait return
 * HG_EDEADLOCK instead of hanging the device (reference: DeadlockError, sim.py:24-29). */
int hg_exec_set_wait_timeout(hg_exec* ex, double seconds);
/* trace mode (opts.trace = 1), after a run: out[2t], out[2t+1] = device ns at which task t started /
 * ended; out[2(n_tasks+j)], out[2(n_tasks+j)+1] = the same for copy job j (0 for work of other
 * ranks).  Capacity 2 * (n_tasks + n_jobs). */
int hg_exec_read_stamps(hg_exec* ex, uint64_t* out);
/* one-process-per-GPU teardown: unmap the peers' pools (run after a barrier; then barrier
 * again before hg_exec_destroy frees this rank's exported pool) */
int hg_exec_ipc_close(hg_exec* ex);

/* Page-lock caller-owned host images (input / output) for async H2D / D2H DMA
 * (cudaHostRegister, portable).  The caller keeps ownership and unregisters before
 * freeing.  Registering an already registered range is not an error. */
int hg_matrix_register(void* host, size_t bytes);
int hg_matrix_unregister(void* host);

/* ------------------------------------------------------------------------
 * One tile kernel on a stream (tests / calibration).  t[] are device
 * pointers to the task's tiles in access order (kernels.py access lists);
 * each tile is nb*nb doubles followed by side_doubles of side area.
 * ---------------------------------------------------------------------- */
int hg_tile_run(int32_t kind, int32_t device, void* stream, double* const* t, int32_t n_t,
                int32_t nb, int32_t ib, int32_t* status_dev);
/* the same with caller-owned scratch (hg_task_scratch_ints(kind, nb, ib) ints on the device,
 * zeroed once): independent tasks may then run concurrently on different streams
 * (the online executor, paper_1402_6601_b200/online.py).  No kernel of this build
 * needs scratch any more (the TRSM strip barrier is a cluster barrier); the size
 * query stays so callers remain valid if a kind needs it again. */
int hg_tile_run_scratch(int32_t kind, int32_t device, void* stream, double* const* t, int32_t n_t,
                        int32_t nb, int32_t ib, int32_t* status_dev, int32_t* scratch_dev);
int hg_task_scratch_ints(int32_t kind, int32_t nb, int32_t ib);

/* ------------------------------------------------------------------------
 * Device plumbing of the online executor (paper_1402_6601_b200/online.py):
 * it plays sim.py's event loop (sim.py:140-203) on the host and issues one
 * hg_tile_run_scratch per dispatched task; slots, streams, events and the
 * H2D / peer copies of non-resident inputs (sim.py:237-267's transfers,
 * executed) go through these calls.  Handles are opaque (cudaStream_t,
 * cudaEvent_t, device pointers).  Replaces nothing in the reference (its
 * execution is simulated); the call sites it serves are sim.py:353-371
 * (_start_exec / _task_end: run a kernel, record its measured duration).
 * ---------------------------------------------------------------------- */
int hg_dev_alloc(int32_t device, size_t bytes, void** out);
int hg_dev_free(int32_t device, void* ptr);
int hg_dev_memset(int32_t device, void* ptr, int32_t value, size_t bytes, void* stream);
/* peer access device -> peer (HG_EPEER when the pair has no peer route) */
int hg_dev_enable_peer(int32_t device, int32_t peer);
int hg_dev_sync(int32_t device);
int hg_stream_create(int32_t device, void** out);      /* non-blocking stream */
int hg_stream_destroy(int32_t device, void* stream);
int hg_stream_wait_event(void* stream, void* event);
int hg_event_create(int32_t device, int32_t timing, void** out);
int hg_event_destroy(int32_t device, void* event);
int hg_event_record(void* event, void* stream);
int hg_event_query(void* event);                       /* 1 done, 0 pending, <0 error */
int hg_event_elapsed_ms(void* start, void* end, float* ms);
/* dst <- src on `stream` (cudaMemcpyDefault: H2D, D2H, D2D or peer over NVLink) */
int hg_copy_async(int32_t device, void* dst, const void* src, size_t bytes, void* stream);

/* FP64 roofline denominator: DMMA (mma.sync m8n8k4 f64) throughput of a
 * register-only kernel filling every SM, in TFLOP/s (MEASURED_PEAKS.json has
 * no FP64 entry).  Runs ~10 ms on `device`. */
int hg_fp64_peak(int32_t device, double* dmma_tflops, double* dfma_tflops);

#ifdef __cplusplus
}
#endif
#endif /* HETGPU_H */
