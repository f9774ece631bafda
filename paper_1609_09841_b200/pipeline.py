"""Grid time stepping on the B200: fused and two-pass half steps.

Drop-in mirror of the reference's time-stepping API
(pkg/src/hermite3d/pipeline.py): same names, signatures, argument meaning
and errors (`StepConfig`, `OperatorSet`, `AllocationStats`,
`InstabilityError`, `select_dt`, `half_step`, `full_step`, ...).  Underneath,
every half step is one call into libh3b200.so (include/h3b200.h), issued on
the caller's current torch CUDA stream; there is no CPU fallback.

Differences that matter to callers:

* `DofField` data lives on the GPU; `.data` is a host copy.
* The finiteness check (pipeline.py:210-215) is fused into the kernels as a
  device flag; `full_step` reads both half steps' flags back once, and the
  second half step is skipped on the device when the first one failed, so
  the observable state matches the reference's raise-after-first-half-step.
* `StepConfig.variant` selects the kernel family: "separable" (exact
  node-factorised evolution, HBM-bound; requires q >= 3(2N+1)), "literal"
  (bit-identical to the reference), or "auto" (separable when exact,
  literal otherwise; always literal for precision="single").
* two_pass mode materialises the (2N+2)^3 coefficient field in slab chunks
  along x3 when the whole field would not fit in free HBM; AllocationStats
  records the buffer actually allocated.
* `timings` accumulates CUDA-event seconds per kernel
  ("monolithic" / "reconstruction" / "evolution").
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .field import DofField, GridSpec
from .operators import DerivOperator, InterpOperator, build_deriv_operator, build_interp_operator

__all__ = [
    "StepConfig", "CoeffField", "OperatorSet", "AllocationStats", "InstabilityError",
    "select_dt", "tile_schedule", "half_step", "full_step", "run_steps", "resolve_tile_x1",
    "set_worker_threads", "default_stages", "DEFAULT_TILE_X1", "MODES", "VARIANTS",
]

MODES = ("two_pass", "fused")
VARIANTS = ("auto", "literal", "separable")
ADVECTION_SPEED = 1.0  # u_t = c (u_x1 + u_x2 + u_x3) with c = 1

# Nominal x1 tile lengths per kernel and N (the reference's defaults, pipeline.py:52-56; other N
# fall back to 4).  On the GPU a tile is only validated and reported -- the launch geometry is
# the kernels' own and results never depend on it.
DEFAULT_TILE_X1 = {
    "reconstruction": {1: 16, 2: 10, 3: 4},
    "evolution": {1: 16, 2: 10, 3: 2},
    "monolithic": {1: 12, 2: 10, 3: 2},
}


def default_stages(order_n: int, dims: int = 3) -> int:
    """Taylor stages after which the local evolution is exact: the cell polynomial has degree
    2N+1 per axis, so dims (2N+1) applications of the nilpotent operator exhaust it."""
    return dims * (2 * order_n + 1)


class InstabilityError(RuntimeError):
    """A half step produced a non-finite DOF.  `node` = (m1, m2, m3) of the first one in the
    field's C order, `step` = the step index passed by the caller (or None)."""

    def __init__(self, node, step: int | None = None):
        self.node = tuple(int(v) for v in node)
        self.step = step
        where = "" if step is None else f" at step {step}"
        super().__init__(f"non-finite values detected{where}, first offending node {self.node}")


def _in(choices):
    return lambda v: v in choices


# (field, accepts, requirement) -- checked in this order by StepConfig
_STEP_CONFIG_RULES = (
    ("mode", _in(MODES), f"one of {MODES}"),
    ("tile_x1", lambda v: v is None or v >= 1, ">= 1"),
    ("cfl", lambda v: 0 < v <= 1, "in (0, 1]"),
    ("stages_q", lambda v: v is None or v >= 1, ">= 1"),
    ("precision", _in(("single", "double")), "'single' or 'double'"),
    ("variant", _in(VARIANTS), f"one of {VARIANTS}"),
)


@dataclass(frozen=True)
class StepConfig:
    """How a half / full step runs: the reference's knobs (mode, tile_x1, cfl, stages_q,
    precision) plus `variant` (kernel family) and `coeff_budget_bytes` (two-pass chunking)."""

    mode: str = "fused"
    tile_x1: int | None = None
    cfl: float = 0.9
    stages_q: int | None = None
    precision: str = "double"
    variant: str = "auto"
    coeff_budget_bytes: int | None = None

    def __post_init__(self):
        for name, ok, requirement in _STEP_CONFIG_RULES:
            value = getattr(self, name)
            if not ok(value):
                raise ValueError(f"{name} must be {requirement}, got {value!r}")

    def stages(self, order_n: int) -> int:
        return default_stages(order_n) if self.stages_q is None else self.stages_q


@dataclass
class CoeffField:
    """Two-pass intermediate: the (2N+2)^3 coefficients of cells [z_begin, z_end) (the whole
    grid, or one x3 chunk when it would not fit in HBM)."""

    parity: str
    data: torch.Tensor
    z_begin: int = 0
    z_end: int = 0


@dataclass(frozen=True)
class OperatorSet:
    """Read-only operators of one (N, grid): the shared H and one derivative per axis."""

    order_n: int
    interp: InterpOperator
    derivs: tuple[DerivOperator, DerivOperator, DerivOperator]

    @classmethod
    def for_grid(cls, grid: GridSpec, order_n: int) -> "OperatorSet":
        derivs = tuple(build_deriv_operator(order_n, h) for h in grid.spacings)
        return cls(order_n, build_interp_operator(order_n), derivs)

    @property
    def interp_triple(self):
        return (self.interp,) * 3

    @property
    def side(self) -> int:
        return self.interp.side


class AllocationStats:
    """Book-keeping of the grid-sized scratch the pipeline allocates (the two-pass coefficient
    buffer): `events` in order, bytes `live_bytes` now, `peak_aux_bytes` high-water mark."""

    def __init__(self):
        self.events: list[tuple[str, int]] = []
        self._sizes: dict[str, int] = {}
        self.peak_aux_bytes = 0

    @property
    def live_bytes(self) -> int:
        return sum(self._sizes.values())

    def allocate(self, name: str, nbytes: int) -> None:
        self.events.append((name, nbytes))
        self._sizes[name] = nbytes
        self.peak_aux_bytes = max(self.peak_aux_bytes, self.live_bytes)

    def release(self, name: str) -> None:
        self._sizes.pop(name, None)


def select_dt(grid: GridSpec, cfg: StepConfig) -> float:
    """Largest stable step the CFL number allows: cfl * min_k h_k / c."""
    if not 0 < cfg.cfl <= 1:
        raise ValueError(f"cfl must be in (0, 1], got {cfg.cfl}")
    return cfg.cfl * min(grid.spacings) / ADVECTION_SPEED


def resolve_tile_x1(kernel: str, order_n: int, m1: int, override: int | None = None) -> int:
    """The x1 tile length a pass reports: a validated override, else the kernel's nominal
    default for N, clipped to the grid."""
    if override is None:
        nominal = DEFAULT_TILE_X1.get(kernel, DEFAULT_TILE_X1["monolithic"]).get(order_n, 4)
        return min(max(nominal, 1), max(m1, 1)) if m1 >= 1 else 1
    if override < 1 or override > m1:
        raise ValueError(f"tile_x1 must be in [1, {m1}], got {override}")
    return override


def tile_schedule(grid: GridSpec, tile_x1: int) -> np.ndarray:
    """The reference's tile table, rows [c3, c2, x1_start, x1_len] in its traversal order
    (kept for API compatibility; the kernels cover the same cells with their own geometry)."""
    m1, m2, m3 = grid.cells_per_axis
    if not 1 <= tile_x1 <= m1:
        raise ValueError(f"tile_x1 must be in [1, {m1}], got {tile_x1}")
    starts = np.arange(0, m1, tile_x1, dtype=np.int64)
    lens = np.minimum(tile_x1, m1 - starts)
    c3, c2, k = np.meshgrid(np.arange(m3), np.arange(m2), np.arange(len(starts)), indexing="ij")
    return np.stack([c3.ravel(), c2.ravel(), starts[k.ravel()], lens[k.ravel()]], axis=1).astype(np.int64)


def set_worker_threads(n: int | None) -> int:
    """The reference sizes a CPU worker pool here; on the GPU the parallelism is the device's:
    returns its SM count (the argument is accepted and ignored)."""
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def _factor_arrays(ops: OperatorSet, dtype, delta: float, q: int):
    """(H, fac1, fac2, fac3, cfac) in the field dtype, the kernels' scale factors:
    fac_k[i] = (i+1) * (1/h_k) for i < s-1 and 0 last -- multiplied by the reciprocal, as the
    reference does, so the factors round identically -- and cfac[k-1] = delta / k."""
    s = ops.side
    inv_h = np.array([1.0 / d.spacing for d in ops.derivs])
    facs = np.zeros((3, s))
    facs[:, :-1] = np.arange(1, s)[None, :] * inv_h[:, None]
    facs = facs.astype(dtype)
    cfac = (delta / np.arange(1, q + 1, dtype=np.float64)).astype(dtype)
    h_mat = np.ascontiguousarray(ops.interp.matrix.astype(dtype))
    return h_mat, facs[0].copy(), facs[1].copy(), facs[2].copy(), cfac


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _new_flags(count: int, device) -> torch.Tensor:
    return torch.full((count,), -1, dtype=torch.int64, device=device)  # == H3_NO_BAD_NODE


def _node_of(lin: int, grid: GridSpec) -> tuple[int, int, int]:
    m1, m2, _ = grid.cells_per_axis
    lin = int(lin) & 0xFFFFFFFFFFFFFFFF
    return (lin % m1, (lin // m1) % m2, lin // (m1 * m2))


def _variant_code(cfg: StepConfig, precision: str) -> int:
    if precision == "single" and cfg.variant == "separable":
        raise ValueError("the separable variant is FP64-only; use variant='literal' or 'auto'")
    return _native.VARIANTS[cfg.variant]


_CHUNK_CACHE: dict = {}


def _coeff_chunk_planes(grid: GridSpec, order_n: int, itemsize: int, budget: int | None,
                        refresh: bool = False) -> int:
    """x3 planes of the two-pass coefficient field that fit the budget (default: 85 % of the free
    HBM minus 1 GiB).  The free-memory query (~65 us) is cached per grid; `refresh` re-queries."""
    m1, m2, m3 = grid.cells_per_axis
    s = 2 * order_n + 2
    per_plane = m1 * m2 * s ** 3 * itemsize
    if budget is None:
        key = (grid.cells_per_axis, order_n, itemsize, torch.cuda.current_device())
        if refresh or key not in _CHUNK_CACHE:
            free, _total = torch.cuda.mem_get_info()
            _CHUNK_CACHE[key] = max(per_plane, int(0.85 * free) - (1 << 30))
        budget = _CHUNK_CACHE[key]
    return max(1, min(m3, budget // per_plane))


def _check_pair(src: DofField, dst: DofField) -> None:
    """A half step maps a field onto a distinct field of the other parity, same shape/dtype."""
    problems = [
        (src.grid.parity == dst.grid.parity,
         f"src and dst must have opposite parity, both are {src.grid.parity!r}"),
        (src.tensor.data_ptr() == dst.tensor.data_ptr(), "src and dst must be disjoint fields"),
        (src.grid.cells_per_axis != dst.grid.cells_per_axis or src.order_n != dst.order_n,
         "src and dst must share grid dimensions and order"),
        (src.tensor.dtype != dst.tensor.dtype or src.device != dst.device,
         "src and dst must share dtype and device"),
    ]
    for bad, message in problems:
        if bad:
            raise ValueError(message)


def half_step(
    src: DofField,
    dst: DofField,
    cfg: StepConfig,
    ops: OperatorSet,
    stats: AllocationStats | None = None,
    dt: float | None = None,
    step_index: int | None = None,
    timings: dict | None = None,
    *,
    _flag: torch.Tensor | None = None,
    _guard: torch.Tensor | None = None,
    _check: bool = True,
) -> None:
    """Advance src's DOFs by dt/2 onto the opposite-parity field dst (reference
    pipeline.py:218-274: same arguments, same ValueErrors for mismatched fields, same
    InstabilityError after the pass), as one (fused) or two (two-pass) kernel launches on the
    current CUDA stream."""
    _check_pair(src, dst)
    if dt is None:
        dt = select_dt(src.grid, cfg)
    order_n = ops.order_n
    q = cfg.stages(order_n)
    delta = dt / 2
    # the gather offset: primary cell c reads nodes c, c+1; dual cell c reads c-1, c
    off = -1 if src.grid.parity == "dual" else 0
    kernel = "monolithic" if cfg.mode == "fused" else "reconstruction"
    resolve_tile_x1(kernel, order_n, src.grid.cells_per_axis[0], cfg.tile_x1)
    precision = src.precision
    dtype = np.float64 if precision == "double" else np.float32
    h_mat, fac1, fac2, fac3, cfac = _factor_arrays(ops, dtype, delta, q)
    variant = _variant_code(cfg, precision)

    lib = _native.lib()
    m1, m2, m3 = src.grid.cells_per_axis
    device = src.device
    with torch.cuda.device(device):
        stream = torch.cuda.current_stream(device)
        sh = ctypes.c_void_p(stream.cuda_stream)
        flag = _flag if _flag is not None else _new_flags(1, device)
        fptr = ctypes.c_void_p(flag.data_ptr())
        gptr = ctypes.c_void_p(_guard.data_ptr()) if _guard is not None else None
        events = []

        def mark():
            if timings is not None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(stream)
                events.append(ev)

        if cfg.mode == "fused":
            fn = lib.h3_fused_pass if precision == "double" else lib.h3_fused_pass_f32
            mark()
            rc = fn(ctypes.c_void_p(src.tensor.data_ptr()), ctypes.c_void_p(dst.tensor.data_ptr()),
                    m1, m2, m3, order_n, _ptr(h_mat), _ptr(fac1), _ptr(fac2), _ptr(fac3), _ptr(cfac),
                    q, off, 0, m3, 1, variant, sh, fptr, gptr)
            _native.check(rc, "h3_fused_pass")
            mark()
            if timings is not None:
                events[1].synchronize()
                timings["monolithic"] = timings.get("monolithic", 0.0) + events[0].elapsed_time(events[1]) / 1e3
        else:
            s = ops.side
            chunk = _coeff_chunk_planes(src.grid, order_n, src.tensor.element_size(), cfg.coeff_budget_bytes)
            try:
                coeff = torch.empty((chunk, m2, m1, s, s, s), dtype=src.tensor.dtype, device=device)
            except torch.OutOfMemoryError:  # free memory shrank since the cached query
                chunk = _coeff_chunk_planes(src.grid, order_n, src.tensor.element_size(), cfg.coeff_budget_bytes,
                                            refresh=True)
                coeff = torch.empty((chunk, m2, m1, s, s, s), dtype=src.tensor.dtype, device=device)
            if stats is not None:
                stats.allocate("coeff_field", coeff.numel() * coeff.element_size())
            try:
                recon = lib.h3_recon_pass if precision == "double" else lib.h3_recon_pass_f32
                evolve = lib.h3_evolve_pass if precision == "double" else lib.h3_evolve_pass_f32
                cptr = ctypes.c_void_p(coeff.data_ptr())
                t_rec = t_evo = 0.0
                for z0 in range(0, m3, chunk):
                    z1 = min(m3, z0 + chunk)
                    events.clear()
                    mark()
                    rc = recon(ctypes.c_void_p(src.tensor.data_ptr()), cptr, m1, m2, m3, order_n,
                               _ptr(h_mat), off, z0, z1, 1, variant, sh, gptr)
                    _native.check(rc, "h3_recon_pass")
                    mark()
                    rc = evolve(cptr, ctypes.c_void_p(dst.tensor.data_ptr()), m1, m2, m3, order_n,
                                _ptr(fac1), _ptr(fac2), _ptr(fac3), _ptr(cfac), q, z0, z1, variant,
                                sh, fptr, gptr)
                    _native.check(rc, "h3_evolve_pass")
                    mark()
                    if timings is not None:
                        events[2].synchronize()
                        t_rec += events[0].elapsed_time(events[1]) / 1e3
                        t_evo += events[1].elapsed_time(events[2]) / 1e3
                if timings is not None:
                    timings["reconstruction"] = timings.get("reconstruction", 0.0) + t_rec
                    timings["evolution"] = timings.get("evolution", 0.0) + t_evo
            finally:
                if stats is not None:
                    stats.release("coeff_field")
                # the caching allocator reuses the block only after queued kernels finish
                coeff.record_stream(stream)
                del coeff
        if _check:
            bad = int(flag[0].item())
            if bad != -1:
                raise InstabilityError(node=_node_of(bad, dst.grid), step=step_index)


def full_step(
    state: DofField,
    scratch: DofField,
    cfg: StepConfig,
    ops: OperatorSet,
    stats: AllocationStats | None = None,
    dt: float | None = None,
    step_index: int | None = None,
    timings: dict | None = None,
) -> None:
    """One full dt: primary -> dual -> primary, state updated in place (pipeline.py:277-293)."""
    if state.grid.parity != "primary" or scratch.grid.parity != "dual":
        raise ValueError("full_step expects state on the primary grid and scratch on the dual grid")
    if dt is None:
        dt = select_dt(state.grid, cfg)
    flags = _new_flags(2, state.device)
    half_step(state, scratch, cfg, ops, stats=stats, dt=dt, step_index=step_index, timings=timings,
              _flag=flags[0:1], _check=False)
    half_step(scratch, state, cfg, ops, stats=stats, dt=dt, step_index=step_index, timings=timings,
              _flag=flags[1:2], _guard=flags[0:1], _check=False)
    _raise_first_bad(flags.cpu().numpy(), (scratch.grid, state.grid), [step_index, step_index])


def _raise_first_bad(host_flags, grids, steps) -> None:
    for k, bad in enumerate(host_flags):
        if int(bad) != -1:
            raise InstabilityError(node=_node_of(int(bad), grids[k % 2]), step=steps[k])


def run_steps(
    state: DofField,
    scratch: DofField,
    cfg: StepConfig,
    ops: OperatorSet,
    steps: int,
    dt: float | None = None,
    first_step: int = 0,
    stats: AllocationStats | None = None,
    graph: bool | None = None,
) -> None:
    """`steps` full steps with ONE host synchronisation at the end.

    Every half step is guarded on the device by its predecessor's flag, so
    after an instability nothing further is computed, and the error raised
    names the same half step and node the per-step loop of the reference
    (runner.py:160-168) would have reported.

    graph: replay the steps from a captured CUDA graph (fused mode; removes the per-launch
    host cost that dominates small grids).  None = automatic: fused grids up to 64^3 cells.
    """
    if state.grid.parity != "primary" or scratch.grid.parity != "dual":
        raise ValueError("run_steps expects state on the primary grid and scratch on the dual grid")
    if steps <= 0:
        return
    if dt is None:
        dt = select_dt(state.grid, cfg)
    if graph is None:
        graph = cfg.mode == "fused" and state.grid.num_cells <= 64 ** 3 and steps >= 8
    if graph:
        if cfg.mode != "fused":
            raise ValueError("graph replay is available for the fused mode")
        _run_steps_graph(state, scratch, cfg, ops, steps, dt, first_step)
        return
    flags = _new_flags(2 * steps, state.device)
    prev = None
    for k in range(steps):
        f0, f1 = flags[2 * k:2 * k + 1], flags[2 * k + 1:2 * k + 2]
        half_step(state, scratch, cfg, ops, stats=stats, dt=dt, step_index=first_step + k,
                  _flag=f0, _guard=prev, _check=False)
        half_step(scratch, state, cfg, ops, stats=stats, dt=dt, step_index=first_step + k,
                  _flag=f1, _guard=f0, _check=False)
        prev = f1
    host = flags.cpu().numpy()
    _raise_first_bad(host, (scratch.grid, state.grid),
                     [first_step + k // 2 for k in range(2 * steps)])


# captured step blocks, keyed by (field addresses, shapes and dtype, config, dt, block length and
# the bytes of every operator the kernels receive): a graph replays its kernels with the field
# pointers and the launch parameters (H, the 1/h_k factors, the stage factors) baked in, so it is
# valid for whatever tensors occupy those addresses with that shape and dtype AND the same
# operators -- two grids with equal cells but different domain lengths (same dt) must not share
# it.  Small LRU (the graphs hold no field references).
_GRAPHS: "OrderedDict" = None
_GRAPH_CACHE_SIZE = 16


def _operator_key(ops: OperatorSet, dtype, dt: float, cfg: StepConfig) -> bytes:
    """The exact launch parameters of a half step with these operators (their bytes)."""
    np_dtype = np.float64 if dtype == torch.float64 else np.float32
    arrays = _factor_arrays(ops, np_dtype, dt / 2, cfg.stages(ops.order_n))
    return b"".join(np.ascontiguousarray(a).tobytes() for a in arrays)


def _run_steps_graph(state, scratch, cfg, ops, steps, dt, first_step, block: int = 32) -> None:
    """Replay blocks of `block` full steps from a CUDA graph; the flags are read back once per
    replay (the guard chain inside a block skips everything after an instability)."""
    dev = state.device
    cur = torch.cuda.current_stream(dev)
    done = 0
    while done < steps:
        nb = min(block, steps - done)
        key = (state.tensor.data_ptr(), scratch.tensor.data_ptr(), tuple(state.tensor.shape), state.tensor.dtype,
               cfg, ops.order_n, float(dt), nb, dev.index, _operator_key(ops, state.tensor.dtype, dt, cfg))
        global _GRAPHS
        if _GRAPHS is None:
            _GRAPHS = OrderedDict()
        entry = _GRAPHS.get(key)
        if entry is not None:
            _GRAPHS.move_to_end(key)
        else:
            flags = _new_flags(2 * nb, dev)
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(dev)
            side.wait_stream(cur)
            with torch.cuda.graph(g, stream=side):
                flags.fill_(-1)
                prev = None
                for k in range(nb):
                    f0, f1 = flags[2 * k:2 * k + 1], flags[2 * k + 1:2 * k + 2]
                    half_step(state, scratch, cfg, ops, dt=dt, _flag=f0, _guard=prev, _check=False)
                    half_step(scratch, state, cfg, ops, dt=dt, _flag=f1, _guard=f0, _check=False)
                    prev = f1
            cur.wait_stream(side)
            entry = _GRAPHS[key] = (g, flags)
            while len(_GRAPHS) > _GRAPH_CACHE_SIZE:
                _GRAPHS.popitem(last=False)
        g, flags = entry[0], entry[1]
        g.replay()
        host = flags.cpu().numpy()
        _raise_first_bad(host, (scratch.grid, state.grid),
                         [first_step + done + k // 2 for k in range(2 * nb)])
        done += nb
