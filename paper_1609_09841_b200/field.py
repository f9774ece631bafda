"""Grid description and device-resident DOF fields.

Mirrors the reference's data layer (pkg/src/hermite3d/field.py):

* `GridSpec` -- periodic tensor grid, h_k = L_k / M_k, primary nodes at m*h and
  dual nodes at (m + 1/2) h (field.py:34-77).
* `DofField` -- scaled-derivative DOFs h^|n|/n! D^n u of one parity in the
  reference's rank-6 C-order layout [m3][m2][m1][n3][n2][n1] (field.py:80-117).

B200 difference: the DOFs live in HBM as a torch tensor (`.tensor`) in exactly
that layout, so the CUDA kernels read and write it in place and host
readback is a plain device->host copy.  `.data` returns a host numpy copy
(assigning to `.data` uploads), `.values` the node values [m3][m2][m1].
Snapshots (field.py:175-217) read/write the reference's byte format.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

__all__ = ["GridSpec", "DofField", "write_snapshot", "read_snapshot", "PRECISION_DTYPES"]

PARITIES = ("primary", "dual")
PRECISION_DTYPES = {"single": np.float32, "double": np.float64}
_TORCH_DTYPES = {"single": torch.float32, "double": torch.float64}


@dataclass(frozen=True)
class GridSpec:
    """Periodic tensor grid: M_k cells and domain length L_k per axis (field.py:34-77)."""

    cells_per_axis: tuple[int, int, int]
    domain_lengths: tuple[float, float, float] = (1.0, 1.0, 1.0)
    parity: str = "primary"

    def __post_init__(self):
        cells = tuple(self.cells_per_axis)
        lengths = tuple(self.domain_lengths)
        if len(cells) != 3 or any(int(m) != m or m < 1 for m in cells):
            raise ValueError(f"cells_per_axis must be three positive ints, got {self.cells_per_axis}")
        if len(lengths) != 3 or any(not (l > 0) for l in lengths):
            raise ValueError(f"domain_lengths must be three positive reals, got {self.domain_lengths}")
        if self.parity not in PARITIES:
            raise ValueError(f"parity must be one of {PARITIES}, got {self.parity!r}")
        object.__setattr__(self, "cells_per_axis", tuple(int(m) for m in cells))
        object.__setattr__(self, "domain_lengths", lengths)

    @property
    def spacings(self) -> tuple[float, float, float]:
        return tuple(l / m for l, m in zip(self.domain_lengths, self.cells_per_axis))

    @property
    def num_cells(self) -> int:
        m1, m2, m3 = self.cells_per_axis
        return m1 * m2 * m3

    def wrap(self, axis: int, m: int) -> int:
        return m % self.cells_per_axis[axis - 1]

    def node_coord(self, axis: int, m: int) -> float:
        h = self.spacings[axis - 1]
        return (self.wrap(axis, m) + (0.5 if self.parity == "dual" else 0.0)) * h

    def axis_coords(self, axis: int) -> np.ndarray:
        m = self.cells_per_axis[axis - 1]
        h = self.spacings[axis - 1]
        return (np.arange(m) + (0.5 if self.parity == "dual" else 0.0)) * h

    def with_parity(self, parity: str) -> "GridSpec":
        return GridSpec(self.cells_per_axis, self.domain_lengths, parity)


def _default_device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1609_09841_b200 needs a CUDA device (B200); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


class DofField:
    """Scaled-derivative DOFs of one parity, resident on the GPU (field.py:80-117).

    `data` may be a numpy array (uploaded) or a CUDA torch tensor (adopted
    without a copy) of shape (M3, M2, M1, N+1, N+1, N+1).
    """

    def __init__(self, grid: GridSpec, order_n: int, data, device=None):
        self.grid = grid
        self.order_n = int(order_n)
        m1, m2, m3 = grid.cells_per_axis
        npts = self.order_n + 1
        expected = (m3, m2, m1, npts, npts, npts)
        if tuple(data.shape) != expected:
            raise ValueError(f"data shape {tuple(data.shape)} does not match grid/order {expected}")
        if isinstance(data, torch.Tensor):
            if not data.is_cuda:
                data = data.to(device or _default_device())
            if data.dtype not in (torch.float32, torch.float64):
                raise ValueError(f"unsupported dtype {data.dtype}")
            self.tensor = data.contiguous()
        else:
            arr = np.ascontiguousarray(data)
            if arr.dtype not in (np.float32, np.float64):
                raise ValueError(f"unsupported dtype {arr.dtype}")
            self.tensor = torch.from_numpy(arr).to(device or _default_device())

    @classmethod
    def zeros(cls, grid: GridSpec, order_n: int, precision: str = "double", device=None) -> "DofField":
        if precision not in PRECISION_DTYPES:
            raise ValueError(f"precision must be one of {tuple(PRECISION_DTYPES)}, got {precision!r}")
        m1, m2, m3 = grid.cells_per_axis
        npts = order_n + 1
        t = torch.zeros((m3, m2, m1, npts, npts, npts), dtype=_TORCH_DTYPES[precision],
                        device=device or _default_device())
        return cls(grid, order_n, t)

    @classmethod
    def empty(cls, grid: GridSpec, order_n: int, precision: str = "double", device=None) -> "DofField":
        """Uninitialised device field (every node is overwritten by a half step)."""
        m1, m2, m3 = grid.cells_per_axis
        npts = order_n + 1
        t = torch.empty((m3, m2, m1, npts, npts, npts), dtype=_TORCH_DTYPES[precision],
                        device=device or _default_device())
        return cls(grid, order_n, t)

    # ---- readback ---------------------------------------------------------------------
    @property
    def data(self) -> np.ndarray:
        """Host copy of the rank-6 DOF tensor (reference layout)."""
        return self.tensor.detach().cpu().numpy()

    @data.setter
    def data(self, value) -> None:
        value = torch.as_tensor(np.ascontiguousarray(value) if not isinstance(value, torch.Tensor) else value)
        if tuple(value.shape) != tuple(self.tensor.shape):
            raise ValueError(f"shape {tuple(value.shape)} does not match {tuple(self.tensor.shape)}")
        self.tensor.copy_(value.to(self.tensor.dtype))

    @property
    def values(self) -> np.ndarray:
        """Node values (the n = (0,0,0) DOF), indexed [m3][m2][m1]."""
        return self.tensor[..., 0, 0, 0].cpu().numpy()

    @property
    def precision(self) -> str:
        return "single" if self.tensor.dtype == torch.float32 else "double"

    @property
    def device(self):
        return self.tensor.device

    @property
    def nbytes(self) -> int:
        return self.tensor.numel() * self.tensor.element_size()

    def copy(self) -> "DofField":
        return DofField(self.grid, self.order_n, self.tensor.clone())

    def all_finite(self) -> bool:
        return bool(torch.isfinite(self.tensor).all().item())


def write_snapshot(field: DofField, base_path, time: float = 0.0) -> tuple[Path, Path]:
    """<base>.bin (flat little-endian, rank-6 layout) + <base>.json sidecar (field.py:175-201)."""
    base = Path(base_path)
    bin_path, json_path = base.with_suffix(".bin"), base.with_suffix(".json")
    bin_path.parent.mkdir(parents=True, exist_ok=True)
    host = field.data
    bin_path.write_bytes(host.astype(host.dtype.newbyteorder("<"), copy=False).tobytes())
    meta = {
        "cells_per_axis": list(field.grid.cells_per_axis),
        "domain_lengths": list(field.grid.domain_lengths),
        "order_n": field.order_n,
        "parity": field.grid.parity,
        "precision": field.precision,
        "time": time,
        "layout": "m3,m2,m1,n3,n2,n1",
        "dtype": "<f4" if field.precision == "single" else "<f8",
    }
    json_path.write_text(json.dumps(meta, sort_keys=True, indent=2) + "\n")
    return bin_path, json_path


def read_snapshot(base_path, device=None) -> tuple[DofField, float]:
    """Load a snapshot written by write_snapshot (field.py:204-217) onto the GPU."""
    base = Path(base_path)
    meta = json.loads(base.with_suffix(".json").read_text())
    grid = GridSpec(tuple(meta["cells_per_axis"]), tuple(meta["domain_lengths"]), meta["parity"])
    order_n = int(meta["order_n"])
    npts = order_n + 1
    m1, m2, m3 = grid.cells_per_axis
    raw = np.frombuffer(base.with_suffix(".bin").read_bytes(), dtype=np.dtype(meta["dtype"]))
    data = raw.reshape(m3, m2, m1, npts, npts, npts).astype(PRECISION_DTYPES[meta["precision"]])
    return DofField(grid, order_n, data, device=device), float(meta["time"])
