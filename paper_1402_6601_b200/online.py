"""Online (XKaapi-style) execution: scheduling decisions on REAL completion
events with the wall clock, and the history cost model fed by measured
kernel durations (the paper's runtime).

The planned path (:mod:`runtime`) replays the reference simulator in virtual
time and executes the resulting plan as one CUDA graph; this module instead
plays the role of ``sim.py``'s event loop (``sim.py:151-385``) against the
GPUs themselves:

* ``scheduler.activate`` (HEFT / DADA / any plugin, ``sched.py:415-452``) is
  called on every batch of tasks made ready by a *measured* completion, with
  ``now`` = seconds since the start and the same resync / idle rules
  (``sim.py:192-203``);
* a GPU worker runs up to ``depth`` tasks at once on its own CUDA streams
  (a B200 worker is not one-task-at-a-time); a task is dispatched from its
  worker's FIFO when a stream is free;
* the non-resident inputs of a dispatched task are copied in (H2D from the
  page-locked host image, or a peer copy from the lowest-numbered valid GPU,
  ``sim.py:242-266``) on the GPU's copy stream; the task's stream waits for
  those copies, then runs the sm_100a tile kernels (``hg_tile_run_scratch``);
* on completion the written blocks become valid only on that GPU
  (``sim.py:369-370``), ``model.record_sample`` receives the kernel's measured
  duration (CUDA events, ``sim.py:371``) and successors are activated.

By construction this is not bit-exact with the reference (decisions depend
on real timings); byte counts are reported the reference's way (a tile move
charges nb^2 * 8 bytes, side areas ride along).  Hazards: a task becomes
ready only after all its DAG predecessors completed, so the WAR/WAW reasoning
of the graph executor carries over (a copy of a newer version into a GPU's
slot exists only after its writer, which waited for every reader of the old
version, completed).
"""

from __future__ import annotations

import ctypes as C
import random
import time
from collections import deque
from dataclasses import dataclass

import numpy as np

from . import _native
from .kernels import ALL_KINDS
from .perfmodel import LoadTimestamps
from .platform import HOST, PlatformError, ResourceClass
from .sched import ActivationBatch, SchedContext
from .sim import ResidencyMap, SimulationError


@dataclass
class OnlineReport:
    makespan: float            # wall seconds from the first activation to the last completion
    gflops: float
    bytes_h2d: int
    bytes_d2d: int
    n_activations: int
    sched_seconds: float       # host time spent inside scheduler.activate
    worker: np.ndarray         # task -> worker
    kernel_seconds: dict       # kind -> list of measured durations
    steals_ok: int = 0
    steals_failed: int = 0


class _Plumb:
    """ctypes handles over libhetgpu's device plumbing (hg_dev_* / hg_stream_* /
    hg_event_* / hg_copy_async): the online executor's data path is this library."""

    def __init__(self, L):
        self.L = L

    def _out(self, fn, *args):
        h = C.c_void_p()
        _native.check(fn(*args, C.byref(h)), fn.__name__)
        return h.value

    def alloc(self, dev, nbytes):
        return self._out(self.L.hg_dev_alloc, dev, nbytes)

    def stream(self, dev):
        return self._out(self.L.hg_stream_create, dev)

    def event(self, dev, timing=False):
        return self._out(self.L.hg_event_create, dev, 1 if timing else 0)

    def record(self, ev, stream):
        _native.check(self.L.hg_event_record(C.c_void_p(ev), C.c_void_p(stream)), "hg_event_record")

    def wait(self, stream, ev):
        _native.check(self.L.hg_stream_wait_event(C.c_void_p(stream), C.c_void_p(ev)), "hg_stream_wait_event")

    def done(self, ev) -> bool:
        rc = self.L.hg_event_query(C.c_void_p(ev))
        if rc < 0:
            _native.check(rc, "hg_event_query")
        return rc == 1

    def elapsed_ms(self, e0, e1) -> float:
        ms = C.c_float()
        _native.check(self.L.hg_event_elapsed_ms(C.c_void_p(e0), C.c_void_p(e1), C.byref(ms)), "hg_event_elapsed_ms")
        return float(ms.value)

    def copy(self, dev, dst, src, nbytes, stream):
        _native.check(self.L.hg_copy_async(dev, C.c_void_p(dst), C.c_void_p(src), nbytes, C.c_void_p(stream)),
                      "hg_copy_async")

    def sync(self, dev):
        _native.check(self.L.hg_dev_sync(dev), "hg_dev_sync")


class OnlineExecutor:
    """Runs ``graph`` on the GPUs of ``platform`` (GPU-only, p2p) with online decisions."""

    def __init__(self, graph, platform, scheduler, model, host_in: np.ndarray, devices=None, depth: int = 8,
                 seed: int = 0):
        if platform.n_cpu_workers:
            raise PlatformError("the online executor runs GPU-only platforms (no CPU fallback)")
        if platform.k > 1 and not platform.p2p:
            raise PlatformError("the online executor needs the NVLink peer route (p2p=True)")
        self.g, self.plat, self.sched = graph, platform, scheduler
        self.model = model.copy()  # as sim.py:105: calibration never leaks to the caller
        lay = graph.layout
        self.nb, self.ib = lay.b, lay.ib
        self.k = platform.k
        self.L = _native.lib()
        self.rt = rt = _Plumb(self.L)
        ndev = self.L.hg_device_count()
        if ndev <= 0:
            raise PlatformError("the online executor needs a CUDA device (there is no CPU fallback)")
        self.devices = list(devices) if devices is not None else [g % ndev for g in range(self.k)]
        self.depth = depth
        self.seed = seed
        self.sizes = [s // 8 for s in graph.sizes]
        self.offs = np.cumsum([0] + self.sizes)
        side = lay.side_doubles
        tile = self.nb * self.nb
        self.slot_doubles = [s + (side if s == tile else 0) for s in self.sizes]
        # the host image, page-locked in place (async H2D DMA; unregistered by close())
        self.host = np.ascontiguousarray(host_in, np.float64)
        self._registered = self.host.nbytes > 0 and self.L.hg_matrix_register(
            C.c_void_p(self.host.ctypes.data), self.host.nbytes) == 0
        uniq = sorted(set(self.devices))
        for a in uniq:
            for b in uniq:
                if a != b:
                    _native.check(self.L.hg_dev_enable_peer(a, b), f"peer access GPU {a} -> GPU {b}")
        self.slots = [dict() for _ in range(self.k)]  # node-1 -> block -> device pointer
        self.streams = [[rt.stream(d) for _ in range(depth)] for d in self.devices]
        self.copy_streams = [rt.stream(d) for d in self.devices]
        self.status = [rt.alloc(d, 4) for d in self.devices]
        kinds = [ALL_KINDS.index(t.kind) for t in graph.tasks]
        self.kind_id = kinds
        need = max(self.L.hg_task_scratch_ints(kd, self.nb, self.ib) for kd in range(len(ALL_KINDS)))
        self.scratch = [[rt.alloc(d, 4 * max(need, 1)) for _ in range(depth)] for d in self.devices]
        for d, st in zip(self.devices, self.status):
            _native.check(self.L.hg_dev_memset(d, C.c_void_p(st), 0, 4, None), "hg_dev_memset")
        for d, scr in zip(self.devices, self.scratch):
            for p in scr:
                _native.check(self.L.hg_dev_memset(d, C.c_void_p(p), 0, 4 * max(need, 1), None), "hg_dev_memset")
        self._events = []  # (device, event) to destroy at close
        self._closed = False

    def _slot(self, node: int, block: int) -> int:
        s = self.slots[node - 1].get(block)
        if s is None:
            s = self.rt.alloc(self.devices[node - 1], self.slot_doubles[block] * 8)
            self.slots[node - 1][block] = s
        return s

    def _event(self, dev, timing=False):
        ev = self.rt.event(dev, timing)
        self._events.append((dev, ev))
        return ev

    def close(self):
        """Free slots, streams, events and the host registration (idempotent)."""
        if self._closed:
            return
        self._closed = True
        L = self.L
        for d in sorted(set(self.devices)):
            L.hg_dev_sync(d)
        for dev, ev in self._events:
            L.hg_event_destroy(dev, C.c_void_p(ev))
        for node, slots in enumerate(self.slots):
            for p in slots.values():
                L.hg_dev_free(self.devices[node], C.c_void_p(p))
        for d, ss in zip(self.devices, self.streams):
            for s_ in ss:
                L.hg_stream_destroy(d, C.c_void_p(s_))
        for d, s_ in zip(self.devices, self.copy_streams):
            L.hg_stream_destroy(d, C.c_void_p(s_))
        for d, p in zip(self.devices, self.status):
            L.hg_dev_free(d, C.c_void_p(p))
        for d, scr in zip(self.devices, self.scratch):
            for p in scr:
                L.hg_dev_free(d, C.c_void_p(p))
        if self._registered:
            L.hg_matrix_unregister(C.c_void_p(self.host.ctypes.data))
            self._registered = False

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self) -> OnlineReport:
        g, plat, rt = self.g, self.plat, self.rt
        n = len(g)
        nw = plat.n_workers
        worker_node = [plat.workers[w].memory for w in range(nw)]
        residency = ResidencyMap(len(g.data))
        stamps = LoadTimestamps(nw)
        ctx = SchedContext(g, plat, self.model, stamps, residency)
        queues = [deque() for _ in range(nw)]
        free_streams = [list(range(self.depth)) for _ in range(nw)]
        running = {}                   # task -> (worker, stream idx, ev_start, ev_end)
        copy_ev = {}                   # block -> {node: event of the copy that delivered the current version}
        preds_left = g.in_degrees()
        placed = np.full(n, -1, np.int32)
        bytes_h2d = bytes_d2d = 0
        measured = {}
        n_act = 0
        sched_time = 0.0
        t0 = time.perf_counter()

        def now():
            return time.perf_counter() - t0

        def activate(ready, completing):
            nonlocal n_act, sched_time
            idle = [len(free_streams[w]) == self.depth and not queues[w] for w in range(nw)]
            stamps.resync(now(), idle)
            a = time.perf_counter()
            asg = self.sched.activate(ActivationBatch(sorted(ready), now()), ctx, completing)
            sched_time += time.perf_counter() - a
            n_act += 1
            for w in sorted(asg.order):
                queues[w].extend(asg.order[w])

        def dispatch(w, tid):
            nonlocal bytes_h2d, bytes_d2d
            node = worker_node[w]
            dev = self.devices[node - 1]
            task = g.tasks[tid]
            si = free_streams[w].pop()
            stream = self.streams[node - 1][si]
            cs = self.copy_streams[node - 1]
            waits = []
            for d, mode in task.accesses:
                if not mode.reads:
                    self._slot(node, d)
                    continue
                if node in residency[d]:
                    ev = copy_ev.get(d, {}).get(node)
                    if ev is not None:
                        waits.append(ev)
                    continue
                dst = self._slot(node, d)
                holders = residency[d]
                if HOST in holders:
                    rt.copy(dev, dst, self.host.ctypes.data + int(self.offs[d]) * 8, self.sizes[d] * 8, cs)
                    bytes_h2d += self.sizes[d] * 8
                else:
                    src_node = min(holders)
                    src_ev = copy_ev.get(d, {}).get(src_node)  # the source may itself be in flight
                    if src_ev is not None:
                        rt.wait(cs, src_ev)
                    rt.copy(dev, dst, self._slot(src_node, d), self.slot_doubles[d] * 8, cs)
                    bytes_d2d += self.sizes[d] * 8
                ev = self._event(dev)
                rt.record(ev, cs)
                copy_ev.setdefault(d, {})[node] = ev
                residency.add(d, node)
                waits.append(ev)
            for ev in waits:
                rt.wait(stream, ev)
            ptrs = (C.c_void_p * len(task.accesses))(*[self._slot(node, d) for d, _ in task.accesses])
            e0, e1 = self._event(dev, True), self._event(dev, True)
            rt.record(e0, stream)
            _native.check(self.L.hg_tile_run_scratch(self.kind_id[tid], dev, C.c_void_p(stream), ptrs,
                                                     len(task.accesses), self.nb, self.ib,
                                                     C.c_void_p(self.status[node - 1]),
                                                     C.c_void_p(self.scratch[node - 1][si])),
                          f"online task {tid}")
            rt.record(e1, stream)
            running[tid] = (w, si, e0, e1)
            placed[tid] = w

        rng = random.Random(self.seed)
        steals = [0, 0]  # ok, failed

        def steal(thief):
            # a worker with free streams and an empty queue takes the newest task of a
            # random victim's queue (sim.py:219-233; the ws baseline, sched.py:434-452)
            pool = [v for v in range(nw) if v != thief]
            while pool:
                victim = pool.pop(rng.randrange(len(pool)))
                if queues[victim]:
                    steals[0] += 1
                    dispatch(thief, queues[victim].pop())
                    return True
                steals[1] += 1
            return False

        def dispatch_round():
            moved = True
            while moved:
                moved = False
                for w in range(nw):
                    if free_streams[w] and queues[w]:
                        dispatch(w, queues[w].popleft())
                        moved = True
                if self.sched.steals:
                    for w in range(nw):
                        if free_streams[w] and not queues[w] and steal(w):
                            moved = True

        activate([t for t in range(n) if preds_left[t] == 0], None)
        dispatch_round()
        done = 0
        while done < n:
            finished = [t for t, r in running.items() if rt.done(r[3])]
            if not finished:
                if not running:
                    raise SimulationError(f"online executor stalled with {n - done} tasks left")
                time.sleep(20e-6)
                continue
            for tid in sorted(finished):
                w, si, e0, e1 = running.pop(tid)
                task = g.tasks[tid]
                node = worker_node[w]
                dur = rt.elapsed_ms(e0, e1) * 1e-3
                measured.setdefault(task.kind, []).append(dur)
                for d in task.write_ids():
                    residency.set_only(d, node)
                    copy_ev.pop(d, None)  # the new version was produced in place
                self.model.record_sample(task.kind, ResourceClass.GPU, dur)
                stamps.on_complete(w, now())
                free_streams[w].append(si)
                done += 1
                ready = []
                for s in g.successors(tid):
                    preds_left[s] -= 1
                    if preds_left[s] == 0:
                        ready.append(s)
                if ready:
                    activate(ready, w)
            dispatch_round()
        for d_ in sorted(set(self.devices)):
            rt.sync(d_)
        span = now()
        for d_, st in zip(self.devices, self.status):
            word = np.zeros(1, np.int32)
            rt.copy(d_, word.ctypes.data, st, 4, None)
            rt.sync(d_)
            if int(word[0]) != 0:
                raise SimulationError(f"tile kernel status {int(word[0])} (non-SPD / singular pivot)")
        self._residency = residency
        from .sim import flops_of

        fl = flops_of(g.layout.family, g.layout.n)
        return OnlineReport(span, fl / span / 1e9, bytes_h2d, bytes_d2d, n_act, sched_time, placed, measured,
                            steals[0], steals[1])

    def result_image(self) -> np.ndarray:
        """Final version of every block (from the GPU that holds it), tile-major like host_in."""
        out = np.zeros(int(self.offs[-1]))
        for d in range(len(self.sizes)):
            nodes = [x for x in self._residency[d] if x != HOST]
            if not nodes:
                out[self.offs[d]:self.offs[d + 1]] = self.host[self.offs[d]:self.offs[d + 1]]
                continue
            node = min(nodes)
            self.rt.copy(self.devices[node - 1], out.ctypes.data + int(self.offs[d]) * 8, self._slot(node, d),
                         self.sizes[d] * 8, None)
        for d_ in sorted(set(self.devices)):
            self.rt.sync(d_)
        return out
