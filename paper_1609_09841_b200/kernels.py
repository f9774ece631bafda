"""Per-cell API of the reference (pkg/src/hermite3d/kernels.py:73-191), computed on the GPU.

Same names, arguments, return types and errors as the reference's per-cell functions --
`TaylorParams`, `reconstruct_cell`, `advect_time_derivative`, `taylor_evolve_horner`,
`space_time_tensor`, `taylor_evolve_recursion`, `verify_space_time_identity`,
`default_stages` -- which are the semantic spec of the grid kernels (gather -> reconstruct ->
evolve -> scatter of one cell).  Inputs and outputs are host ndarrays / `CellCoeffs`, as in
the reference; the arithmetic runs in libh3b200.so's per-cell kernels (h3_cell.cu, declared
in include/h3b200.h) in the input's precision with the reference's operation order, so the
results are bit-identical to the reference's numpy evaluation (tests/test_gpu_cell_api.py).
Like every entry point of the package there is no CPU fallback: without a CUDA device these
raise.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .field import CellCoeffs
from .operators import DerivOperator, InterpOperator
from .pipeline import default_stages

__all__ = ["TaylorParams", "reconstruct_cell", "advect_time_derivative", "taylor_evolve_horner",
           "space_time_tensor", "taylor_evolve_recursion", "verify_space_time_identity", "default_stages"]


@dataclass(frozen=True)
class TaylorParams:
    """Temporal expansion of one step: q stages over a full step dt (reference kernels.py:55-70)."""

    stages_q: int
    dt: float

    def __post_init__(self):
        if self.stages_q < 1:
            raise ValueError(f"stages_q must be >= 1, got {self.stages_q}")
        if not self.dt > 0:
            raise ValueError(f"dt must be positive, got {self.dt}")

    @property
    def half_dt(self) -> float:
        return self.dt / 2


# ---- device plumbing ------------------------------------------------------------------------

def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1609_09841_b200 needs a CUDA device (B200); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def _as_float(a) -> np.ndarray:
    a = np.asarray(a)
    return a if a.dtype in (np.float32, np.float64) else a.astype(np.float64)


def _up(a: np.ndarray, dev) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def _vp(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())


def _stream(dev):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _cell_shape(a: np.ndarray):
    if a.ndim < 3:
        raise ValueError(f"a cell tensor needs three axes [n3][n2][n1], got shape {a.shape}")
    n3, n2, n1 = a.shape[-3:]
    return int(np.prod(a.shape[:-3], dtype=np.int64)), (n3, n2, n1)


def _axis_factors(d_ops, shape, dtype, dev):
    """fac_k[i] = (i+1) * (1/h_k), rounded to the precision (kernels.py:90-96 forms the same
    products in float64 and casts), padded to the axis length; axis k = 1 is the last index."""
    out = []
    for k, d in enumerate(d_ops, start=1):
        n = shape[-k]
        fac = np.zeros(n, dtype=dtype)
        fac[:-1] = (np.arange(1, n) * (1.0 / d.spacing)).astype(dtype)
        out.append(_up(fac, dev))
    return out


def _scalars(values, dtype, dev) -> torch.Tensor:
    """Python-float scalars rounded to the precision, as numpy rounds a Python float operand."""
    return _up(np.array([np.asarray(v, dtype=dtype) for v in values], dtype=dtype).reshape(-1), dev)


def _single(dtype) -> int:
    return 1 if np.dtype(dtype) == np.float32 else 0


# ---- the per-cell API -----------------------------------------------------------------------

def reconstruct_cell(h_ops: tuple[InterpOperator, InterpOperator, InterpOperator], u_loc) -> CellCoeffs:
    """Midpoint coefficients of the cell polynomial from its 8-vertex DOF tensor: H sweeps along
    x1, x2, x3 in that order (reference kernels.py:73-87)."""
    u = _as_float(u_loc)
    batch, shape = _cell_shape(u)
    dev = _device()
    cur = _up(u, dev)
    lib = _native.lib()
    for axis, op in zip((1, 2, 3), h_ops):
        mat = np.asarray(getattr(op, "matrix", op))
        if mat.shape != (shape[-axis],) * 2:
            raise ValueError(f"tensor axis {axis} has length {shape[-axis]}, operator needs {mat.shape[0]}")
        nxt = torch.empty_like(cur)
        rc = lib.h3_cell_apply_axis(_vp(cur), _vp(nxt), batch, *shape, _vp(_up(mat.astype(u.dtype), dev)), axis,
                                    _single(u.dtype), _stream(dev))
        _native.check(rc, "h3_cell_apply_axis")
        cur = nxt
    return CellCoeffs(order_n=h_ops[0].order_n, data=cur.cpu().numpy())


def advect_time_derivative(d_ops: tuple[DerivOperator, DerivOperator, DerivOperator], w) -> np.ndarray:
    """Coefficients of u_x1 + u_x2 + u_x3, accumulated in axis order (reference kernels.py:99-108)."""
    w = _as_float(w)
    batch, shape = _cell_shape(w)
    dev = _device()
    src = _up(w, dev)
    out = torch.empty_like(src)
    f1, f2, f3 = _axis_factors(d_ops, w.shape, w.dtype, dev)
    rc = _native.lib().h3_cell_advect(_vp(src), _vp(out), batch, *shape, _vp(f1), _vp(f2), _vp(f3),
                                      _single(w.dtype), _stream(dev))
    _native.check(rc, "h3_cell_advect")
    return out.cpu().numpy()


def taylor_evolve_horner(coeffs: CellCoeffs, d_ops, params: TaylorParams, step: float) -> CellCoeffs:
    """Advance a cell's coefficients by `step` (dt/2 in the grid pipeline): the q-stage nested
    recurrence w <- b + (step/k) L w, k = q..1, two-phase (reference kernels.py:111-128)."""
    if not step > 0:
        raise ValueError(f"step must be positive, got {step}")
    b = _as_float(coeffs.data)
    batch, shape = _cell_shape(b)
    dev = _device()
    src = _up(b, dev)
    out, tmp = torch.empty_like(src), torch.empty_like(src)
    f1, f2, f3 = _axis_factors(d_ops, b.shape, b.dtype, dev)
    q = params.stages_q
    cst = _scalars([step / k for k in range(1, q + 1)], b.dtype, dev)
    rc = _native.lib().h3_cell_horner(_vp(src), _vp(out), _vp(tmp), batch, *shape, _vp(f1), _vp(f2), _vp(f3),
                                      _vp(cst), q, _single(b.dtype), _stream(dev))
    _native.check(rc, "h3_cell_horner")
    return CellCoeffs(order_n=coeffs.order_n, data=out.cpu().numpy())


def _space_time_device(coeffs: CellCoeffs, d_ops, params: TaylorParams):
    b = _as_float(coeffs.data)
    batch, shape = _cell_shape(b)
    dev = _device()
    q = params.stages_q
    src = _up(b, dev)
    st = torch.empty((batch, q + 1, *shape), dtype=src.dtype, device=dev)
    facs = _axis_factors(d_ops, b.shape, b.dtype, dev)
    cst = _scalars([params.dt / (j + 1) for j in range(q)], b.dtype, dev)
    rc = _native.lib().h3_cell_space_time(_vp(src), _vp(st), batch, *shape, *map(_vp, facs), _vp(cst), q,
                                          _single(b.dtype), _stream(dev))
    _native.check(rc, "h3_cell_space_time")
    return b, batch, shape, dev, st, facs


def space_time_tensor(coeffs: CellCoeffs, d_ops, params: TaylorParams) -> np.ndarray:
    """Space-time coefficients b[j][n3][n2][n1], j = 0..q: b[j+1] = dt/(j+1) L b[j]
    (reference kernels.py:131-142)."""
    b, _batch, _shape, _dev, st, _ = _space_time_device(coeffs, d_ops, params)
    # device layout [cell][j][...] -> the reference's [j][cell...][...]
    return np.ascontiguousarray(np.moveaxis(st.cpu().numpy(), 1, 0)).reshape((params.stages_q + 1,) + b.shape)


def taylor_evolve_recursion(coeffs: CellCoeffs, d_ops, params: TaylorParams, tau: float) -> CellCoeffs:
    """The space-time expansion evaluated at fraction tau of the step, summed in ascending
    powers (reference kernels.py:144-164; the independent cross-check of the Horner form)."""
    if not 0 < tau <= 1:
        raise ValueError(f"tau must be in (0, 1], got {tau}")
    b, batch, shape, dev, st, _ = _space_time_device(coeffs, d_ops, params)
    powers, p = [], 1.0
    for _ in range(params.stages_q):
        p *= tau
        powers.append(p)
    tpow = _scalars(powers, b.dtype, dev)
    out = torch.empty(b.shape, dtype=st.dtype, device=dev)
    rc = _native.lib().h3_cell_time_sum(_vp(st), _vp(out), batch, int(np.prod(shape)), _vp(tpow),
                                        params.stages_q, _single(b.dtype), _stream(dev))
    _native.check(rc, "h3_cell_time_sum")
    return CellCoeffs(order_n=coeffs.order_n, data=out.cpu().numpy())


def verify_space_time_identity(coeffs: CellCoeffs, d_ops, params: TaylorParams) -> float:
    """Max |d/dt - sum_k d/dx_k| of the space-time expansion, coefficient-wise (reference
    kernels.py:167-191): (j+1)/dt b[j+1] - L b[j] for j < q and L b[q] at the top."""
    b, batch, shape, dev, st, facs = _space_time_device(coeffs, d_ops, params)
    inv_dt = 1.0 / params.dt
    coef = _scalars([(j + 1) * inv_dt for j in range(params.stages_q)] or [0.0], b.dtype, dev)
    worst = torch.zeros(1, dtype=torch.int64, device=dev)
    rc = _native.lib().h3_cell_identity_residual(_vp(st), batch, *shape, *map(_vp, facs), _vp(coef),
                                                 params.stages_q, _vp(worst), _single(b.dtype), _stream(dev))
    _native.check(rc, "h3_cell_identity_residual")
    return float(worst.cpu().view(torch.float64).item())
