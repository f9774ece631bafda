"""Run orchestration on the B200: the reference runner's stepping loop, with the GPU kept busy.

Mirror of `execute_run` / `execute_converge` / `execute_bench` (reference
pkg/src/hermite3d/runner.py:135-269)
for library callers: same step planning (`_plan_steps`, runner.py:65-76), the same artifacts
(snapshot.bin/json, errors.csv, perf.json/perf.csv) and the same summary keys.  The reference's
pydantic RunConfig / CLI / REST layers are out of scope; `RunConfig` here is a
plain dataclass with the same fields and validation messages, and `build_ic` understands the
reference's IC term dictionaries (`plane_wave`, `random_modes`, `separable` with
`fourier` / `constant` / `monomial` factors, config.py:30-70, 133-153).

B200 difference: the reference evaluates the error norms on the host after every step, which
would force a device synchronisation per step.  Here every half step and every per-step error
reduction is queued on the stream (h3_error_norms writes into a device array) and the flags and
norms are read back once at the end; an instability still raises InstabilityError naming the
reference's step and node (later half steps are skipped on the device by the guard flags).
"""

from __future__ import annotations

import csv
import json
import math
from dataclasses import dataclass, field as dc_field, replace
from pathlib import Path

import numpy as np
import torch

from . import perf
from .field import DofField, GridSpec, read_snapshot, write_snapshot
from .pipeline import AllocationStats, InstabilityError, OperatorSet, StepConfig, _new_flags, _node_of, full_step, \
    half_step, select_dt
from .problems import Constant, FourierMode, Monomial, SeparableIC, error_norms_async, exact_solution, init_field, \
    plane_wave

__all__ = ["RunConfig", "ConfigError", "build_ic", "execute_run", "execute_converge", "execute_bench",
           "execute_autotune"]


class ConfigError(ValueError):
    """Invalid run configuration (reference config.ConfigError)."""


@dataclass(frozen=True)
class RunConfig:
    """Everything one run needs (reference config.py:73-122; order cap lifted to 5)."""

    order_n: int
    cells: tuple
    domain: tuple = (1.0, 1.0, 1.0)
    cfl: float = 0.9
    stages_q: int | None = None
    steps: int | None = None
    final_time: float | None = None
    mode: str = "fused"
    tile_x1: int | None = None
    precision: str = "double"
    variant: str = "auto"
    ic: tuple = dc_field(default_factory=lambda: ({"kind": "plane_wave"},))
    seed: int = 0
    out_dir: str = "out"
    resume: str | None = None  # snapshot base path: continue from its field and time

    def __post_init__(self):
        cells = (self.cells,) * 3 if isinstance(self.cells, int) else tuple(self.cells)
        object.__setattr__(self, "cells", cells)
        object.__setattr__(self, "domain", tuple(float(x) for x in self.domain))
        if not 0 <= self.order_n <= 5:
            raise ConfigError("order_n: must be in [0, 5]")
        if len(cells) != 3 or any(int(m) != m or m < 1 for m in cells):
            raise ConfigError("cells: all cell counts must be >= 1")
        if len(self.domain) != 3 or any(not (l > 0) for l in self.domain):
            raise ConfigError("domain: all domain lengths must be positive")
        if not 0 < self.cfl <= 1:
            raise ConfigError("cfl: must be in (0, 1]")
        if (self.steps is None) == (self.final_time is None):
            raise ConfigError("steps/final_time: exactly one of steps or final_time must be set")
        if self.steps is not None and self.steps < 1:
            raise ConfigError("steps: must be >= 1")
        if self.final_time is not None and not self.final_time > 0:
            raise ConfigError("final_time: must be > 0")
        if self.mode not in ("fused", "two_pass"):
            raise ConfigError("mode: must be 'fused' or 'two_pass'")
        if self.precision not in ("double", "single"):
            raise ConfigError("precision: must be 'double' or 'single'")
        if not self.ic:
            raise ConfigError("ic: at least one term is required")

    def stages(self) -> int:
        return self.stages_q if self.stages_q is not None else 3 * (2 * self.order_n + 1)

    def step_config(self) -> StepConfig:
        return StepConfig(mode=self.mode, tile_x1=self.tile_x1, cfl=self.cfl, stages_q=self.stages(),
                          precision=self.precision, variant=self.variant)


def _factor(f: dict):
    kind = f.get("kind", "fourier")
    if kind == "fourier":
        return FourierMode(amplitude=float(f.get("amplitude", 1.0)), wavenumber=int(f.get("wavenumber", 1)),
                           phase=float(f.get("phase", 0.0)))
    if kind == "constant":
        return Constant(float(f.get("value", 1.0)))
    if kind == "monomial":
        return Monomial(int(f.get("degree", 1)))
    raise ConfigError(f"ic: unknown factor kind {kind!r}")


def build_ic(cfg: RunConfig) -> SeparableIC:
    """Expand the config's IC terms into a separable IC (reference config.py:133-153)."""
    if isinstance(cfg.ic, SeparableIC):
        return cfg.ic
    terms = []
    rng = np.random.default_rng(cfg.seed)
    for term in cfg.ic:
        kind = term.get("kind", "plane_wave")
        if kind == "separable":
            terms.append(tuple(_factor(f) for f in term["factors"]))
        elif kind == "plane_wave":
            terms.extend(plane_wave(int(term.get("wavenumber", 1)), float(term.get("amplitude", 1.0)),
                                    float(term.get("phase", 0.0))).terms)
        elif kind == "random_modes":
            for _ in range(int(term.get("terms", 4))):
                terms.append(tuple(FourierMode(amplitude=float(rng.uniform(-1.0, 1.0)),
                                               wavenumber=int(rng.integers(1, int(term.get("max_wavenumber", 2)) + 1)),
                                               phase=float(rng.uniform(0.0, 2 * np.pi)))
                                   for _ in range(3)))
        else:
            raise ConfigError(f"ic: unknown term kind {kind!r}")
    return SeparableIC(terms=tuple(terms))


def _plan_steps(cfg: RunConfig, grid: GridSpec, step_cfg: StepConfig, t0: float = 0.0) -> tuple[int, float]:
    """(full steps, dt).  A step count runs at the CFL dt; a final time is reached exactly by
    the fewest equal steps not exceeding the CFL dt (a 1e-12 slack absorbs T / dt rounding
    just above an integer) -- the reference runner's plan (runner.py:65-76).  A resumed run
    (t0 > 0, an extension of the reference) plans the remaining interval final_time - t0."""
    cfl_dt = select_dt(grid, step_cfg)
    if cfg.steps is None:
        span = cfg.final_time - t0
        if not span > 0:
            raise ConfigError(f"final_time: {cfg.final_time} is not after the resumed snapshot time {t0}")
        count = max(1, math.ceil(span / cfl_dt - 1e-12))
        return count, span / count
    return cfg.steps, cfl_dt


def _write_csv(path: Path, header, rows) -> None:
    """CSV with floats written by repr (round-trip exact, as the reference writes them)."""
    path.parent.mkdir(parents=True, exist_ok=True)
    cell = lambda v: repr(float(v)) if isinstance(v, (float, np.floating)) else str(v)  # noqa: E731
    with open(path, "w", newline="") as fh:
        csv.writer(fh).writerows([list(header)] + [[cell(v) for v in row] for row in rows])


def _write_artifacts(cfg, step_cfg, grid, state, t, error_rows, n_steps, wall) -> dict:
    """snapshot.bin/json, errors.csv (when errors were tracked), perf.json/csv -- the reference
    runner's artifact set and names; returns {artifact key: path}."""
    out_dir = Path(cfg.out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    paths = dict(zip(("snapshot_bin", "snapshot_json"), write_snapshot(state, out_dir / "snapshot", time=t)))
    if error_rows is not None:
        paths["errors_csv"] = out_dir / "errors.csv"
        _write_csv(paths["errors_csv"], ["step", "time", "l_inf", "l2"], error_rows)
    # perf report: one row per kernel over the whole run (2 half steps per step) plus the total
    peaks = perf.DevicePeaks.b200()
    kernels = _kernels_of(cfg.mode)
    passes = 2 * n_steps
    rows = []
    for kern in kernels:
        flops, nbytes = (c * passes for c in perf.model_counts(kern, cfg.order_n, grid, step_cfg))
        tile = perf.resolve_tile_x1(kern, cfg.order_n, grid.cells_per_axis[0], cfg.tile_x1)
        rows.append(perf._profile(kern, cfg.order_n, cfg.mode, tile, flops, nbytes,
                                  max(wall / len(kernels), 1e-12), peaks,
                                  perf.algorithmic_bytes(kern, cfg.order_n, grid) * passes))
    rows.append(_solution_row(cfg, grid, step_cfg, cfg.mode, n_steps, wall, peaks))
    paths.update(_write_perf(out_dir, rows, peaks)[1])
    return {key: str(path) for key, path in paths.items()}


def _kernels_of(mode: str) -> tuple[str, ...]:
    return ("monolithic",) if mode == "fused" else ("reconstruction", "evolution")


def _solution_row(cfg, grid, step_cfg, mode, n_steps, seconds, peaks) -> perf.KernelProfile:
    """End-to-end row of a run: modelled counts of all its passes against its wall time."""
    counts = [perf.model_counts(k, cfg.order_n, grid, step_cfg) for k in _kernels_of(mode)]
    tile = perf.resolve_tile_x1(_kernels_of(mode)[0], cfg.order_n, grid.cells_per_axis[0], cfg.tile_x1)
    return perf._profile("solution", cfg.order_n, mode, tile, sum(f for f, _ in counts) * 2 * n_steps,
                         sum(b for _, b in counts) * 2 * n_steps, max(seconds, 1e-12), peaks)


def _write_perf(out_dir: Path, rows, peaks) -> tuple[dict, dict]:
    """perf.json + perf.csv of `rows`; returns (report, {artifact key: path})."""
    report = perf.report_dict(rows, peaks)
    paths = {"perf_json": out_dir / "perf.json", "perf_csv": out_dir / "perf.csv"}
    out_dir.mkdir(parents=True, exist_ok=True)
    paths["perf_json"].write_text(json.dumps(report, sort_keys=True, indent=2) + "\n")
    _write_csv(paths["perf_csv"], perf.REPORT_COLUMNS, [[r[c] for c in perf.REPORT_COLUMNS] for r in report["runs"]])
    return report, paths


def execute_run(cfg: RunConfig, write_artifacts: bool = True) -> dict:
    """Full time-stepping run; returns the reference's summary dict (+ artifact paths).

    Raises InstabilityError (with the failing step and node) if the field goes non-finite.
    """
    step_cfg = cfg.step_config()
    grid = GridSpec(cfg.cells, cfg.domain, "primary")
    ops = OperatorSet.for_grid(grid, cfg.order_n)
    ic = build_ic(cfg)
    t0 = 0.0
    if cfg.resume:
        # resume path: the snapshot's field and time, same grid and order
        state, t0 = read_snapshot(cfg.resume)
        if (state.grid.cells_per_axis, state.grid.domain_lengths, state.order_n, state.grid.parity) != \
                (grid.cells_per_axis, grid.domain_lengths, cfg.order_n, "primary"):
            raise ConfigError("resume: snapshot grid/order does not match the run configuration")
        if state.precision != cfg.precision:
            raise ConfigError("resume: snapshot precision does not match the run configuration")
    else:
        state = init_field(ic, grid, cfg.order_n, precision=cfg.precision)
    scratch = DofField.zeros(grid.with_parity("dual"), cfg.order_n, precision=cfg.precision)
    n_steps, dt = _plan_steps(cfg, grid, step_cfg, t0)
    # errors are tracked for every precision, as the reference does (runner.py:156); the device
    # reduction upcasts single-precision DOFs to FP64
    track = ic.smoothness_class == "analytic"
    stats = AllocationStats()
    dev = state.device
    norms = torch.zeros((n_steps + 1, 2), dtype=torch.float64, device=dev)
    flags = _new_flags(2 * n_steps, dev)
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if track:
        error_norms_async(state, exact_solution(ic, t0, grid.domain_lengths), norms[0])
    e0.record(stream)
    prev = None
    for k in range(n_steps):
        f0, f1 = flags[2 * k:2 * k + 1], flags[2 * k + 1:2 * k + 2]
        half_step(state, scratch, step_cfg, ops, stats=stats, dt=dt, step_index=k + 1, _flag=f0, _guard=prev,
                  _check=False)
        half_step(scratch, state, step_cfg, ops, stats=stats, dt=dt, step_index=k + 1, _flag=f1, _guard=f0,
                  _check=False)
        prev = f1
        if track:
            error_norms_async(state, exact_solution(ic, t0 + (k + 1) * dt, grid.domain_lengths), norms[k + 1])
    e1.record(stream)
    host_flags = flags.cpu().numpy()  # one synchronisation for the whole run
    for i, bad in enumerate(host_flags):
        if int(bad) != -1:
            raise InstabilityError(node=_node_of(int(bad), (scratch.grid, state.grid)[i % 2]), step=i // 2 + 1)
    wall = e0.elapsed_time(e1) / 1e3
    t = t0 + n_steps * dt
    h1, h2, h3 = grid.spacings
    error_rows = []
    if track:
        for k, (linf, sumsq) in enumerate(norms.cpu().tolist()):
            error_rows.append([k, t0 + k * dt, linf, math.sqrt(h1 * h2 * h3 * sumsq)])
    result = {"status": "ok", "steps": n_steps, "dt": dt, "final_time": t, "mode": cfg.mode,
              "order_n": cfg.order_n, "seconds": wall, "peak_aux_bytes": stats.peak_aux_bytes, "artifacts": {}}
    if track:
        result["l_inf"] = error_rows[-1][2]
        result["l2"] = error_rows[-1][3]
    if write_artifacts:
        result["artifacts"] = _write_artifacts(cfg, step_cfg, grid, state, t, error_rows if track else None,
                                               n_steps, wall)
    return result


def execute_converge(cfg: RunConfig, levels: list[int]) -> dict:
    """Refinement study over cubic grids; observed orders between levels (runner.py:198-236)."""
    if len(levels) < 2:
        raise ConfigError("levels: need at least two refinement levels")
    if cfg.final_time is None:
        raise ConfigError("final_time: converge requires final_time (not steps)")
    header = ["cells", "h", "l_inf", "l2", "order_linf", "order_l2"]

    def observed_order(coarse_err, fine_err, refinement):
        # e ~ C h^p  =>  p = log2(e_coarse / e_fine) / log2(M_fine / M_coarse)
        return math.log2(coarse_err / fine_err) / refinement if fine_err > 0 else float("inf")

    errors = []  # (M, l_inf, l2) per level
    for m in levels:
        summary = execute_run(replace(cfg, cells=(m, m, m), steps=None), write_artifacts=False)
        if "l_inf" not in summary:
            raise ConfigError("ic: converge requires an IC with an exact solution")
        errors.append((m, summary["l_inf"], summary["l2"]))
    rows = []
    for k, (m, l_inf, l2) in enumerate(errors):
        orders = [float("nan")] * 2
        if k:
            m0, e0_inf, e0_l2 = errors[k - 1]
            refinement = math.log2(m / m0)
            orders = [observed_order(e0_inf, l_inf, refinement), observed_order(e0_l2, l2, refinement)]
        rows.append([m, cfg.domain[0] / m, l_inf, l2, *orders])
    csv_path = Path(cfg.out_dir) / "converge.csv"
    _write_csv(csv_path, header, rows)
    return {"status": "ok", "order_n": cfg.order_n, "rows": [dict(zip(header, r)) for r in rows],
            "artifacts": {"converge_csv": str(csv_path)}}


def execute_bench(cfg: RunConfig, repetitions: int = 3, modes: list[str] | None = None) -> dict:
    """Kernel profiles plus the end-to-end run time per mode (reference runner.py:239-269).

    For each mode: `perf.profile_run` (CUDA-event medians of the mode's kernels on a seeded
    random field) and one `execute_run` without artifacts, reported as a "solution" row with
    the modelled counts of all its passes; perf.json / perf.csv go to `cfg.out_dir`.  Peaks are
    the B200's measured ones (`DevicePeaks.b200()`), as in `execute_run`'s report.
    """
    peaks = perf.DevicePeaks.b200()
    grid = GridSpec(cfg.cells, cfg.domain, "primary")
    rows = []
    for mode in modes or [cfg.mode]:
        mode_cfg = replace(cfg, mode=mode)
        step_cfg = mode_cfg.step_config()
        rows += perf.profile_run(step_cfg, grid, cfg.order_n, repetitions=repetitions, peaks=peaks,
                                 rng_seed=cfg.seed)
        summary = execute_run(mode_cfg, write_artifacts=False)
        rows.append(_solution_row(mode_cfg, grid, step_cfg, mode, summary["steps"], summary["seconds"], peaks))
    report, paths = _write_perf(Path(cfg.out_dir), rows, peaks)
    return {"status": "ok", "runs": report["runs"], "artifacts": {k: str(v) for k, v in paths.items()}}


def execute_autotune(cfg: RunConfig, candidates: list[int], repetitions: int = 3) -> dict:
    """Pick tile_x1 by timing full steps per candidate (reference runner.py:272-327: median of
    `repetitions` after a warm-up step, argmin wins, ties go to the smaller tile; candidates
    wider than M1 are reported as skipped; autotune.csv in `cfg.out_dir`).

    On the B200 the tile is validated and reported but does not change the kernels' launch
    geometry, so the candidates time the same up to noise; the API, the table and the selection
    rule are kept so callers of the reference's autotune keep working.  Times are CUDA-event
    medians of one full step.
    """
    import statistics
    if len(candidates) < 2:
        raise ConfigError("candidates: need at least two tile candidates")
    grid = GridSpec(cfg.cells, cfg.domain, "primary")
    ops = OperatorSet.for_grid(grid, cfg.order_n)
    ic = build_ic(cfg)
    m1 = cfg.cells[0]
    gather = "monolithic" if cfg.mode == "fused" else "reconstruction"
    rows, best = [], None
    for tile in candidates:
        if tile > m1:
            rows.append({"tile_x1": tile, "seconds": None, "bytes_modeled": None,
                         "status": f"skipped: exceeds M1={m1}"})
            continue
        step_cfg = replace(cfg, tile_x1=tile).step_config()
        state = init_field(ic, grid, cfg.order_n, precision=cfg.precision)
        scratch = DofField.zeros(grid.with_parity("dual"), cfg.order_n, precision=cfg.precision)
        dt = select_dt(grid, step_cfg)
        full_step(state, scratch, step_cfg, ops, dt=dt)  # warm-up
        times = []
        for _ in range(repetitions):
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            full_step(state, scratch, step_cfg, ops, dt=dt)
            t1.record()
            t1.synchronize()
            times.append(t0.elapsed_time(t1) / 1e3)
        seconds = statistics.median(times)
        rows.append({"tile_x1": tile, "seconds": seconds,
                     "bytes_modeled": perf.model_counts(gather, cfg.order_n, grid, step_cfg)[1], "status": "ok"})
        best = min(best, (seconds, tile)) if best is not None else (seconds, tile)
    if best is None:
        raise ConfigError(f"candidates: no candidate fits M1={m1}")
    for row in rows:
        if row["status"] == "ok" and row["tile_x1"] == best[1]:
            row["status"] = "winner"
    csv_path = Path(cfg.out_dir) / "autotune.csv"
    _write_csv(csv_path, ["tile_x1", "seconds", "bytes_modeled", "status"],
               [[r["tile_x1"], "" if r["seconds"] is None else r["seconds"],
                 "" if r["bytes_modeled"] is None else r["bytes_modeled"], r["status"]] for r in rows])
    return {"status": "ok", "best_tile_x1": best[1], "rows": rows, "artifacts": {"autotune_csv": str(csv_path)}}
