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
  pinned host image, or a peer copy from the lowest-numbered valid GPU,
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


class OnlineExecutor:
    """Runs ``graph`` on the GPUs of ``platform`` (GPU-only, p2p) with online decisions."""

    def __init__(self, graph, platform, scheduler, model, host_in: np.ndarray, devices=None, depth: int = 8,
                 seed: int = 0):
        import torch

        if platform.n_cpu_workers:
            raise PlatformError("the online executor runs GPU-only platforms (no CPU fallback)")
        if platform.k > 1 and not platform.p2p:
            raise PlatformError("the online executor needs the NVLink peer route (p2p=True)")
        self.torch = torch
        self.g, self.plat, self.sched = graph, platform, scheduler
        self.model = model.copy()  # as sim.py:105: calibration never leaks to the caller
        lay = graph.layout
        self.nb, self.ib = lay.b, lay.ib
        self.k = platform.k
        ndev = torch.cuda.device_count()
        self.devices = list(devices) if devices is not None else [g % max(1, ndev) for g in range(self.k)]
        self.depth = depth
        self.seed = seed
        self.L = _native.lib()
        self.sizes = [s // 8 for s in graph.sizes]
        self.offs = np.cumsum([0] + self.sizes)
        side = lay.side_doubles
        tile = self.nb * self.nb
        self.slot_doubles = [s + (side if s == tile else 0) for s in self.sizes]
        self.host = torch.from_numpy(np.ascontiguousarray(host_in, np.float64))
        if not self.host.is_pinned():
            self.host = self.host.pin_memory()
        self.slots = [dict() for _ in range(self.k)]  # node-1 -> block -> device tensor
        self.streams = [[torch.cuda.Stream(device=d) for _ in range(depth)] for d in self.devices]
        self.copy_streams = [torch.cuda.Stream(device=d) for d in self.devices]
        self.status = [torch.zeros(1, dtype=torch.int32, device=d) for d in self.devices]
        kinds = [ALL_KINDS.index(t.kind) for t in graph.tasks]
        self.kind_id = kinds
        need = max(self.L.hg_task_scratch_ints(kd, self.nb, self.ib) for kd in range(len(ALL_KINDS)))
        self.scratch = [[torch.zeros(max(need, 1), dtype=torch.int32, device=d) for _ in range(depth)]
                        for d in self.devices]

    def _slot(self, node: int, block: int):
        s = self.slots[node - 1].get(block)
        if s is None:
            s = self.torch.empty(self.slot_doubles[block], dtype=self.torch.float64,
                                 device=self.devices[node - 1])
            self.slots[node - 1][block] = s
        return s

    def run(self) -> OnlineReport:
        torch, g, plat = self.torch, self.g, self.plat
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
                with torch.cuda.stream(cs):
                    if HOST in holders:
                        dst[: self.sizes[d]].copy_(self.host[self.offs[d]:self.offs[d + 1]], non_blocking=True)
                        bytes_h2d += self.sizes[d] * 8
                    else:
                        src_node = min(holders)
                        src_ev = copy_ev.get(d, {}).get(src_node)  # the source may itself be in flight
                        if src_ev is not None:
                            cs.wait_event(src_ev)
                        dst.copy_(self._slot(src_node, d), non_blocking=True)
                        bytes_d2d += self.sizes[d] * 8
                    ev = torch.cuda.Event()
                    ev.record(cs)
                copy_ev.setdefault(d, {})[node] = ev
                residency.add(d, node)
                waits.append(ev)
            for ev in waits:
                stream.wait_event(ev)
            ptrs = (C.c_void_p * len(task.accesses))(*[self._slot(node, d).data_ptr() for d, _ in task.accesses])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _native.check(self.L.hg_tile_run_scratch(self.kind_id[tid], dev, C.c_void_p(stream.cuda_stream), ptrs,
                                                     len(task.accesses), self.nb, self.ib,
                                                     C.c_void_p(self.status[node - 1].data_ptr()),
                                                     C.c_void_p(self.scratch[node - 1][si].data_ptr())),
                          f"online task {tid}")
            e1.record(stream)
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
            finished = [t for t, r in running.items() if r[3].query()]
            if not finished:
                if not running:
                    raise SimulationError(f"online executor stalled with {n - done} tasks left")
                time.sleep(20e-6)
                continue
            for tid in sorted(finished):
                w, si, e0, e1 = running.pop(tid)
                task = g.tasks[tid]
                node = worker_node[w]
                dur = e0.elapsed_time(e1) * 1e-3
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
        for d_ in self.devices:
            torch.cuda.synchronize(d_)
        span = now()
        for st in self.status:
            if int(st.item()) != 0:
                raise SimulationError(f"tile kernel status {int(st.item())} (non-SPD / singular pivot)")
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
                out[self.offs[d]:self.offs[d + 1]] = self.host[self.offs[d]:self.offs[d + 1]].numpy()
                continue
            out[self.offs[d]:self.offs[d + 1]] = self._slot(min(nodes), d)[: self.sizes[d]].cpu().numpy()
        return out
