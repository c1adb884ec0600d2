"""Experiment harness with the reference's command line.

Same subcommands, flags, INI sections and CSV schema as ``hetsim``'s harness
(``/root/reference/pkg/src/hetsim/cli.py:25-29, 165-295``), so scripts and
sweeps written for the reference run unchanged:

    python -m paper_1402_6601_b200 run   --kernel cholesky --nt 32 --tile 1024 --cpus 1 --gpus 1 ...
    python -m paper_1402_6601_b200 sweep --gpus 1..8 --alpha 0,0.25,0.5,0.75,1 --scheduler heft,dada
    python -m paper_1402_6601_b200 export-dot | validate

Rows come from the bit-exact planner (the reference's simulated makespan and
bytes).  ``--execute`` (``run`` only, GPU-only platforms) also executes every
repetition's plan on the B200s and appends measured columns (EXEC_COLUMNS):
device time, GFLOP/s, the copy bytes the CUDA graph moved and, for
Cholesky, a randomized residual of the factor.
"""

from __future__ import annotations

import argparse
import configparser
import csv
import sys
from dataclasses import dataclass, fields, replace

from .graph import GraphError
from .kernels import default_timing_table, gen_family
from .perfmodel import PerfModel, PerfModelError, load_timing_table
from .platform import PlatformError, build_platform
from .sched import SchedulerError, make_scheduler
from .sim import SimulationError, flops_of, run

CSV_COLUMNS = [
    "scheduler", "alpha", "cp", "ncpu", "ngpu", "kernel", "n", "tile", "seed", "rep",
    "makespan_s", "gflops", "bytes_h2d", "bytes_d2h", "bytes_d2d", "bytes_total",
    "steals_ok", "steals_failed",
]
EXEC_COLUMNS = CSV_COLUMNS + ["measured_s", "measured_gflops", "exec_bytes_h2d", "exec_bytes_d2d", "residual"]

_USER_ERRORS = (GraphError, PlatformError, PerfModelError, SchedulerError, SimulationError, ValueError, OSError)


@dataclass
class Settings:
    """One experiment point (defaults = the reference harness's)."""

    kernel: str = "cholesky"
    nt: int = 16
    tile: int = 512
    ib: int = 128
    cpus: int = 12
    gpus: int = 8
    switches: int = 4
    bandwidth: float = 6e9
    latency: float = 1e-5
    switch_cap: float | None = None
    p2p: bool = False  # B200 extension: NVLink peer route (platform.py:93-117); required by --execute
    scheduler: str = "heft"
    alpha: float = 0.5
    epsilon: float = 1e-4
    cp: bool = False
    seed: int = 0
    noise: float = 0.0
    reps: int = 1
    timings: str | None = None

    def __post_init__(self):
        for name in ("reps", "nt"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be at least 1, got {getattr(self, name)}")


# INI layout: section -> {key in the file: (Settings field, parser)}
def _as_bool(v) -> bool:
    return v if isinstance(v, bool) else str(v).strip().lower() in ("1", "true", "yes", "on")


_INI = {
    "platform": {"cpus": ("cpus", int), "gpus": ("gpus", int), "switches": ("switches", int),
                 "bandwidth": ("bandwidth", float), "latency": ("latency", float),
                 "switch_cap": ("switch_cap", float), "p2p": ("p2p", _as_bool)},
    "kernel": {"family": ("kernel", str), "nt": ("nt", int), "tile": ("tile", int), "ib": ("ib", int)},
    "sched": {"name": ("scheduler", str), "alpha": ("alpha", float), "epsilon": ("epsilon", float),
              "cp": ("cp", _as_bool)},
    "run": {"seed": ("seed", int), "noise": ("noise", float), "reps": ("reps", int), "timings": ("timings", str)},
}


def settings_from_ini(path: str) -> Settings:
    ini = configparser.ConfigParser()
    if not ini.read(path):
        raise OSError(f"cannot read config file {path!r}")
    values = {}
    for section, keys in _INI.items():
        if not ini.has_section(section):
            continue
        for key, (field_name, conv) in keys.items():
            if key in ini[section]:
                values[field_name] = conv(ini[section][key])
    return Settings(**values)


def settings_from_args(args) -> Settings:
    """Config file first, then every flag that was given (flags win)."""
    base = settings_from_ini(args.config) if args.config else Settings()
    given = {f.name: getattr(args, f.name) for f in fields(Settings) if getattr(args, f.name, None) is not None}
    for flag in ("cp", "p2p"):
        if flag in given:
            given[flag] = bool(given[flag])
    return replace(base, **given)


def _model(s: Settings) -> PerfModel:
    table = default_timing_table(s.tile, s.ib)
    if s.timings:
        table.update(load_timing_table(s.timings))
    return PerfModel(table)


def _platform(s: Settings):
    return build_platform(s.cpus, s.gpus, s.switches, s.bandwidth, s.latency, s.switch_cap, p2p=s.p2p)


def _fmt_row(s: Settings, n: int, seed: int, rep: int, report, total_flops: float) -> list:
    gflops = total_flops / report.makespan / 1e9 if report.makespan > 0 else 0.0
    return [s.scheduler, repr(s.alpha), int(s.cp), s.cpus, s.gpus, s.kernel, n, s.tile, seed, rep,
            repr(report.makespan), repr(gflops), report.bytes_h2d, report.bytes_d2h, report.bytes_d2d,
            report.bytes_total, report.steals_ok, report.steals_failed]


def point_rows(s: Settings, trace_path: str | None = None, execute: bool = False):
    """Yield one CSV row per repetition (seeds seed, seed+1, ...)."""
    graph = gen_family(s.kernel, s.nt, s.tile, s.ib)
    plat = _platform(s)
    model = _model(s)
    sched = make_scheduler(s.scheduler, alpha=s.alpha, epsilon=s.epsilon, cp=s.cp)
    n = s.nt * s.tile
    total = flops_of(s.kernel, n)
    for rep in range(s.reps):
        seed = s.seed + rep
        trace = trace_path is not None and rep == 0
        report = run(graph, plat, sched, model, seed=seed, noise=s.noise, trace=trace)
        if trace:
            _write_trace(trace_path, report.events)
        row = _fmt_row(s, n, seed, rep, report, total)
        if execute:
            row += _execute(graph, plat, sched, model, seed, n, total,
                            trace_path=(trace_path + ".executed") if trace else None)
        yield row


def _write_trace(path: str, events) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("# time kind worker task data bytes\n")
        for ev in events:
            fh.write(f"{ev.time!r} {ev.kind} {ev.worker} {ev.task} {ev.data} {ev.nbytes}\n")


def _execute(graph, plat, sched, model, seed: int, n: int, total_flops: float, trace_path=None) -> list:
    """Execute the plan on the B200s (one process, one CUDA graph over every GPU).  With
    ``trace_path`` the timed run is stamped (runtime.Executor(trace=True)) and its measured
    TraceEvents go to that file in the simulated trace's format."""
    import numpy as np
    import torch

    from . import runtime
    from .sim import make_plan

    if plat.n_cpu_workers or (plat.k > 1 and not plat.p2p):
        raise PlatformError("--execute needs a GPU-only platform (cpus == gpus) with --p2p 1: no CPU fallback")
    plan = make_plan(graph, plat, sched, model, seed=seed)
    rng = np.random.default_rng(seed)
    R = rng.uniform(-0.5, 0.5, (n, n))
    A = (R + R.T) / 2 + n * np.eye(n) if graph.layout.family == "cholesky" else R
    img = torch.from_numpy(runtime.to_tile_major(A, graph)).pin_memory()
    out = torch.empty_like(img).pin_memory()
    ndev = torch.cuda.device_count()
    devices = [g % max(1, ndev) for g in range(plat.k)]
    ex = runtime.Executor(graph, plat, plan, img.numpy(), out.numpy(), devices=devices,
                          trace=trace_path is not None)
    ex.run()  # warm-up (graph upload, first-touch page faults)
    st = ex.run()
    if trace_path is not None:
        _write_trace(trace_path, ex.report(st, events=True).events)
    ex.close()
    residual = ""
    if graph.layout.family == "cholesky":
        L = np.tril(runtime.from_tile_major(out.numpy(), graph))
        x = rng.standard_normal(n)
        residual = repr(float(np.linalg.norm(A @ x - L @ (L.T @ x)) / np.linalg.norm(A @ x)))
    secs = st.elapsed_ms * 1e-3
    return [repr(secs), repr(total_flops / secs / 1e9), st.bytes_h2d, st.bytes_d2d, residual]


def _parse_ints(text: str) -> list:
    if ".." in text:
        lo, hi = text.split("..", 1)
        return list(range(int(lo), int(hi) + 1))
    return [int(x) for x in text.split(",") if x]


def _parse_floats(text: str) -> list:
    return [float(x) for x in text.split(",") if x]


class _Output:
    def __init__(self, path):
        self.path = path
        self.fh = None

    def __enter__(self):
        self.fh = sys.stdout if self.path in (None, "-") else open(self.path, "w", newline="", encoding="utf-8")
        return csv.writer(self.fh, lineterminator="\n")

    def __exit__(self, *exc):
        if self.fh is not sys.stdout:
            self.fh.close()


def cmd_run(args) -> int:
    s = settings_from_args(args)
    with _Output(args.out) as w:
        w.writerow(EXEC_COLUMNS if args.execute else CSV_COLUMNS)
        for row in point_rows(s, trace_path=args.trace, execute=args.execute):
            w.writerow(row)
    return 0


def cmd_sweep(args) -> int:
    s = settings_from_args(args)  # axis flags are strings here; the scalar fields come from the config
    gpus = _parse_ints(args.gpus) if args.gpus else [s.gpus]
    alphas = _parse_floats(args.alpha) if args.alpha else [s.alpha]
    scheds = [x.strip() for x in args.scheduler.split(",")] if args.scheduler else [s.scheduler]
    with _Output(args.out) as w:
        w.writerow(CSV_COLUMNS)
        # deterministic order: scheduler, then alpha, then GPU count, then repetition
        for name in scheds:
            for a in alphas:
                for k in gpus:
                    for row in point_rows(replace(s, scheduler=name, alpha=a, gpus=k)):
                        w.writerow(row)
    return 0


def cmd_export_dot(args) -> int:
    s = settings_from_args(args)
    text = gen_family(s.kernel, s.nt, s.tile, s.ib).export_dot()
    if args.out and args.out != "-":
        with open(args.out, "w", encoding="utf-8") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    return 0


def cmd_validate(args) -> int:
    s = settings_from_args(args)
    graph = gen_family(s.kernel, s.nt, s.tile, s.ib)
    plat = _platform(s)
    _model(s)
    make_scheduler(s.scheduler, alpha=s.alpha, epsilon=s.epsilon, cp=s.cp)
    print(f"ok: {s.kernel} nt={s.nt} -> {len(graph)} tasks, {plat.n_cpu_workers} CPU + {plat.k} GPU workers, "
          f"scheduler {s.scheduler}, reps {s.reps}")
    return 0


# flag name -> (argparse kwargs); the sweep variants of gpus / alpha / scheduler take lists
_FLAGS = {
    "config": dict(help="INI config file; flags override it"),
    "kernel": dict(help="kernel family: cholesky, lu or qr"),
    "nt": dict(type=int, help="tiles per matrix dimension"),
    "tile": dict(type=int, help="tile order b"),
    "ib": dict(type=int, help="inner block size"),
    "cpus": dict(type=int, help="CPU cores m (one per GPU is consumed)"),
    "switches": dict(type=int, help="number of PCIe switches"),
    "bandwidth": dict(type=float, help="link bandwidth in bytes/s"),
    "latency": dict(type=float, help="link latency in seconds"),
    "switch-cap": dict(dest="switch_cap", type=float, help="per-switch aggregate bandwidth in bytes/s"),
    "epsilon": dict(type=float, help="dual-approximation search precision"),
    "cp": dict(type=int, choices=(0, 1), help="communication prediction for dada"),
    "p2p": dict(type=int, choices=(0, 1), help="GPU-to-GPU peer route (NVLink) instead of host staging"),
    "seed": dict(type=int, help="base RNG seed"),
    "noise": dict(type=float, help="execution-time noise amplitude in [0,1)"),
    "reps": dict(type=int, help="repetitions per point (seeds seed, seed+1, ...)"),
    "timings": dict(help="timing table file with 'kind,class,seconds' lines"),
    "out": dict(help="output file (default stdout)"),
}
_POINT_AXES = {
    "gpus": dict(type=int, help="GPU count k (requires m >= k)"),
    "alpha": dict(type=float, help="dada affinity budget in [0,1]"),
    "scheduler": dict(help="heft, dada or ws"),
}
_SWEEP_AXES = {
    "gpus": dict(help="GPU counts, e.g. '0,2,4,8' or '0..8'"),
    "alpha": dict(help="comma-separated alpha values"),
    "scheduler": dict(help="comma-separated scheduler names"),
}


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_1402_6601_b200", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="command", required=True)
    specs = [("run", "plan (and optionally execute) one configuration", cmd_run, _POINT_AXES),
             ("sweep", "sweep GPU count, alpha and scheduler axes", cmd_sweep, _SWEEP_AXES),
             ("export-dot", "print the generated task graph as DOT", cmd_export_dot, _POINT_AXES),
             ("validate", "check a configuration without running", cmd_validate, _POINT_AXES)]
    for name, help_text, func, axes in specs:
        p = sub.add_parser(name, help=help_text)
        for flag, kw in {**_FLAGS, **axes}.items():
            p.add_argument("--" + flag, **kw)
        if name == "run":
            p.add_argument("--trace", help="write the first repetition's event trace to this file")
            p.add_argument("--execute", action="store_true",
                           help="also execute each plan on the B200s and append measured columns")
        p.set_defaults(func=func)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except _USER_ERRORS as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    raise SystemExit(main())
