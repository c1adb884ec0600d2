"""ctypes binding of ``libhetgpu.so`` (declarations in ``include/hetgpu.h``).

The library is the product path: the native planner (``hg_plan_build``), the
CUDA-graph executor (``hg_exec_*``) and the per-kind tile entry
(``hg_tile_run``).  There is no fallback -- if the library is missing the
import-time loader raises with the build command to run.
"""

from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhetgpu.so")

HG_OK, HG_EINVAL, HG_ECUDA, HG_ENOTSPD, HG_EDEADLOCK, HG_EMODEL, HG_ESINGULAR, HG_EPEER = 0, -1, -2, -3, -4, -5, -6, -7

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_i8p = C.POINTER(C.c_int8)


class GraphDesc(C.Structure):
    _fields_ = [("n_tasks", C.c_int32), ("n_blocks", C.c_int32), ("task_kind", _i32p),
                ("task_flops", _f64p), ("acc_ptr", _i64p), ("acc_block", _i32p), ("acc_mode", _i8p),
                ("succ_ptr", _i64p), ("succ", _i32p), ("block_bytes", _i64p)]


class PlatformDesc(C.Structure):
    _fields_ = [("m", C.c_int32), ("k", C.c_int32), ("n_switches", C.c_int32),
                ("link_bandwidth", C.c_double), ("link_latency", C.c_double),
                ("switch_slots", C.c_int32), ("p2p", C.c_int32)]


class ModelDesc(C.Structure):
    _fields_ = [("n_kinds", C.c_int32), ("fallback_cpu", _f64p), ("fallback_gpu", _f64p),
                ("count_cpu", _i64p), ("count_gpu", _i64p), ("mean_cpu", _f64p), ("mean_gpu", _f64p),
                ("sample_threshold", C.c_int64)]


class SchedDesc(C.Structure):
    _fields_ = [("type", C.c_int32), ("with_cp", C.c_int32), ("alpha", C.c_double),
                ("epsilon", C.c_double), ("rho", C.c_double)]


class PlanOut(C.Structure):
    _fields_ = [("worker", _i32p), ("start", _f64p), ("end", _f64p), ("dispatch", _i32p),
                ("wait_ptr", _i64p), ("wait_job", _i32p), ("n_jobs", C.c_int32),
                ("job_block", _i32p), ("job_src", _i32p), ("job_dst", _i32p), ("job_version", _i32p),
                ("job_src_job", _i32p), ("job_stage_job", _i32p), ("job_requester", _i32p),
                ("job_bytes", _i64p), ("bytes_h2d", C.c_int64), ("bytes_d2h", C.c_int64),
                ("bytes_d2d", C.c_int64), ("makespan", C.c_double), ("gflops", C.c_double),
                ("busy", _f64p), ("n_workers", C.c_int32), ("n_activations", C.c_int32),
                ("n_fallbacks", C.c_int32), ("plan_seconds", C.c_double)]


class ExecPlan(C.Structure):
    _fields_ = [("n_tasks", C.c_int32), ("n_blocks", C.c_int32), ("n_jobs", C.c_int32), ("k", C.c_int32),
                ("nb", C.c_int32), ("ib", C.c_int32), ("side_doubles", C.c_int32),
                ("task_kind", _i32p), ("task_node", _i32p), ("acc_ptr", _i64p), ("acc_block", _i32p),
                ("pred_ptr", _i64p), ("pred", _i32p), ("dispatch", _i32p), ("wait_ptr", _i64p),
                ("wait_job", _i32p), ("job_block", _i32p), ("job_src", _i32p), ("job_dst", _i32p),
                ("job_version", _i32p), ("job_src_job", _i32p), ("job_requester", _i32p),
                ("block_bytes", _i64p), ("final_writer", _i32p), ("acc_mode", _i8p),
                ("job_stage_job", _i32p), ("p2p", C.c_int32), ("push", C.c_int32)]


class ExecOpts(C.Structure):
    _fields_ = [("devices", _i32p), ("host_in", _f64p), ("host_out", _f64p), ("host_side_out", _f64p),
                ("device_input", C.c_int32), ("rank_node", C.c_int32),
                ("task_weight", _f64p), ("host_stage", _f64p), ("priority_levels", C.c_int32),
                ("trace", C.c_int32)]


class ExecStats(C.Structure):
    _fields_ = [("elapsed_ms", C.c_double), ("bytes_h2d", C.c_int64), ("bytes_d2d", C.c_int64),
                ("bytes_d2h", C.c_int64), ("bytes_side", C.c_int64), ("n_kernel_nodes", C.c_int32),
                ("n_copy_nodes", C.c_int32), ("n_push_jobs", C.c_int32)]


EXPORTS = ("hg_last_error", "hg_abi_version", "hg_device_count", "hg_plan_build", "hg_plan_free",
           "hg_pysum", "hg_exec_create", "hg_exec_run", "hg_exec_read_block", "hg_exec_destroy",
           "hg_tile_run", "hg_exec_launch", "hg_exec_wait", "hg_exec_info", "hg_fp64_peak",
           "hg_exec_ipc_handle", "hg_exec_ipc_open", "hg_exec_build", "hg_exec_partition",
           "hg_tile_run_scratch", "hg_task_scratch_ints", "hg_exec_set_wait_timeout", "hg_exec_ipc_close", "hg_exec_read_stamps",
           "hg_matrix_register", "hg_matrix_unregister",
           "hg_dev_alloc", "hg_dev_free", "hg_dev_memset", "hg_dev_enable_peer", "hg_dev_sync",
           "hg_stream_create", "hg_stream_destroy", "hg_stream_wait_event", "hg_event_create",
           "hg_event_destroy", "hg_event_record", "hg_event_query", "hg_event_elapsed_ms", "hg_copy_async")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    """Load ``libhetgpu.so`` (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1402_6601_b200.build` "
                          "(there is no CPU fallback for the execution path)")
    L = C.CDLL(LIB_PATH)
    L.hg_last_error.restype = C.c_char_p
    L.hg_abi_version.restype = C.c_int
    L.hg_device_count.restype = C.c_int
    L.hg_plan_build.argtypes = [C.POINTER(GraphDesc), C.POINTER(PlatformDesc), C.POINTER(ModelDesc),
                                C.POINTER(SchedDesc), C.POINTER(PlanOut)]
    L.hg_plan_free.argtypes = [C.POINTER(PlanOut)]
    L.hg_pysum.argtypes = [_f64p, C.c_int64]
    L.hg_pysum.restype = C.c_double
    L.hg_exec_create.argtypes = [C.POINTER(ExecPlan), C.POINTER(ExecOpts), C.POINTER(C.c_void_p)]
    L.hg_exec_run.argtypes = [C.c_void_p, C.POINTER(ExecStats)]
    L.hg_exec_read_block.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _f64p, C.c_int64]
    L.hg_exec_destroy.argtypes = [C.c_void_p]
    L.hg_tile_run.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.POINTER(C.c_void_p), C.c_int32,
                              C.c_int32, C.c_int32, C.c_void_p]
    L.hg_tile_run_scratch.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.POINTER(C.c_void_p), C.c_int32,
                                      C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]
    L.hg_task_scratch_ints.argtypes = [C.c_int32, C.c_int32, C.c_int32]
    L.hg_exec_launch.argtypes = [C.c_void_p, C.c_void_p]
    L.hg_exec_wait.argtypes = [C.c_void_p]
    L.hg_exec_info.argtypes = [C.c_void_p, C.POINTER(ExecStats)]
    L.hg_fp64_peak.argtypes = [C.c_int32, _f64p, _f64p]
    L.hg_exec_ipc_handle.argtypes = [C.c_void_p, C.c_void_p]
    L.hg_exec_ipc_open.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
    L.hg_exec_build.argtypes = [C.c_void_p]
    L.hg_exec_partition.argtypes = [C.POINTER(ExecPlan), C.c_int32, _i32p, _i32p, _i32p]
    L.hg_exec_set_wait_timeout.argtypes = [C.c_void_p, C.c_double]
    L.hg_exec_ipc_close.argtypes = [C.c_void_p]
    L.hg_exec_read_stamps.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
    L.hg_matrix_register.argtypes = [C.c_void_p, C.c_size_t]
    L.hg_matrix_unregister.argtypes = [C.c_void_p]
    # device plumbing of the online executor (streams, events, slots, async copies)
    vp, i32, sz = C.c_void_p, C.c_int32, C.c_size_t
    L.hg_dev_alloc.argtypes = [i32, sz, C.POINTER(vp)]
    L.hg_dev_free.argtypes = [i32, vp]
    L.hg_dev_memset.argtypes = [i32, vp, i32, sz, vp]
    L.hg_dev_enable_peer.argtypes = [i32, i32]
    L.hg_dev_sync.argtypes = [i32]
    L.hg_stream_create.argtypes = [i32, C.POINTER(vp)]
    L.hg_stream_destroy.argtypes = [i32, vp]
    L.hg_stream_wait_event.argtypes = [vp, vp]
    L.hg_event_create.argtypes = [i32, i32, C.POINTER(vp)]
    L.hg_event_destroy.argtypes = [i32, vp]
    L.hg_event_record.argtypes = [vp, vp]
    L.hg_event_query.argtypes = [vp]
    L.hg_event_elapsed_ms.argtypes = [vp, vp, C.POINTER(C.c_float)]
    L.hg_copy_async.argtypes = [i32, vp, vp, sz, vp]
    _lib = L
    return L


def fp64_peak(device: int = 0):
    """(DMMA, DFMA) FP64 TFLOP/s measured on ``device`` (roofline denominator)."""
    a, b = C.c_double(), C.c_double()
    check(lib().hg_fp64_peak(device, C.byref(a), C.byref(b)), "hg_fp64_peak")
    return a.value, b.value


def last_error() -> str:
    return lib().hg_last_error().decode(errors="replace")


def check(rc: int, what: str):
    if rc == HG_OK:
        return
    msg = f"{what}: {last_error()} (code {rc})"
    from .perfmodel import PerfModelError
    from .platform import PlatformError
    from .sim import DeadlockError, SimulationError

    if rc == HG_EINVAL:
        raise ValueError(msg)
    if rc == HG_EMODEL:
        raise PerfModelError(msg)
    if rc == HG_EPEER:
        raise PlatformError(msg)
    if rc == HG_EDEADLOCK:
        err = DeadlockError([])
        err.args = (msg,)
        raise err
    raise SimulationError(msg)


def ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def pysum(values) -> float:
    a = np.ascontiguousarray(values, dtype=np.float64)
    return lib().hg_pysum(ptr(a, C.c_double), a.shape[0])


# -- planner ----------------------------------------------------------------

def _model_arrays(model, kinds):
    from .platform import ResourceClass

    n = len(kinds)
    fb = {c: np.full(n, math.nan) for c in ResourceClass}
    cnt = {c: np.full(n, -1, np.int64) for c in ResourceClass}
    mean = {c: np.zeros(n) for c in ResourceClass}
    for i, kind in enumerate(kinds):
        for c in ResourceClass:
            v = model.fallback.get((kind, c))
            if v is not None:
                fb[c][i] = v
            s = model.samples.get((kind, c))
            if s is not None:
                cnt[c][i] = int(s[0])
                mean[c][i] = float(s[1])
    return fb, cnt, mean


def plan_build(graph, platform, scheduler, model):
    """Run ``hg_plan_build`` and return a :class:`sim.Plan`."""
    from .platform import ResourceClass
    from .sched import DadaScheduler
    from .sim import Plan

    if not platform.is_uniform():
        raise ValueError("native planner needs build_platform-style uniform links")
    if platform.k > 62:
        raise ValueError("native planner supports up to 62 GPUs")
    L = lib()
    fl = graph.flat()
    gd = GraphDesc(len(graph), len(graph.data), ptr(fl["kind_id"], C.c_int32), ptr(fl["flops"], C.c_double),
                   ptr(fl["acc_ptr"], C.c_int64), ptr(fl["acc_block"], C.c_int32),
                   ptr(fl["acc_mode"], C.c_int8), ptr(fl["succ_ptr"], C.c_int64), ptr(fl["succ"], C.c_int32),
                   ptr(fl["sizes"], C.c_int64))
    pp = platform.native_params()
    pd = PlatformDesc(pp["m"], pp["k"], pp["n_switches"], pp["bw"], pp["lat"], pp["slots"], int(pp["p2p"]))
    fb, cnt, mean = _model_arrays(model, fl["kinds"])
    CPU, GPU = ResourceClass.CPU, ResourceClass.GPU
    md = ModelDesc(len(fl["kinds"]), ptr(fb[CPU], C.c_double), ptr(fb[GPU], C.c_double),
                   ptr(cnt[CPU], C.c_int64), ptr(cnt[GPU], C.c_int64), ptr(mean[CPU], C.c_double),
                   ptr(mean[GPU], C.c_double), int(model.sample_threshold))
    if isinstance(scheduler, DadaScheduler):
        cfg = scheduler.cfg
        sd = SchedDesc(1, int(bool(cfg.with_cp)), float(cfg.alpha), float(cfg.epsilon), float(cfg.rho))
    else:
        sd = SchedDesc(0, 0, 0.0, 1e-4, 2.0)
    out = PlanOut()
    rc = L.hg_plan_build(C.byref(gd), C.byref(pd), C.byref(md), C.byref(sd), C.byref(out))
    check(rc, "hg_plan_build")
    try:
        n = len(graph)
        nj = out.n_jobs

        def arr(p, count, dt):
            if count == 0:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(p, shape=(count,)).astype(dt, copy=True)

        plan = Plan(
            n_tasks=n,
            worker=arr(out.worker, n, np.int32),
            start=arr(out.start, n, np.float64),
            end=arr(out.end, n, np.float64),
            dispatch=arr(out.dispatch, n, np.int32),
            job_block=arr(out.job_block, nj, np.int32),
            job_src=arr(out.job_src, nj, np.int32),
            job_dst=arr(out.job_dst, nj, np.int32),
            job_version=arr(out.job_version, nj, np.int32),
            job_src_job=arr(out.job_src_job, nj, np.int32),
            job_stage_job=arr(out.job_stage_job, nj, np.int32),
            job_requester=arr(out.job_requester, nj, np.int32),
            job_bytes=arr(out.job_bytes, nj, np.int64),
            wait_ptr=arr(out.wait_ptr, n + 1, np.int64),
            wait_job=None,
            bytes_h2d=int(out.bytes_h2d),
            bytes_d2h=int(out.bytes_d2h),
            bytes_d2d=int(out.bytes_d2d),
            busy=tuple(float(x) for x in arr(out.busy, out.n_workers, np.float64)),
            makespan=float(out.makespan),
            gflops=float(out.gflops),
            n_activations=int(out.n_activations),
            n_fallbacks=int(out.n_fallbacks),
        )
        plan.wait_job = arr(out.wait_job, int(plan.wait_ptr[-1]) if n else 0, np.int32)
        plan.plan_seconds = float(out.plan_seconds)
        return plan
    finally:
        L.hg_plan_free(C.byref(out))
