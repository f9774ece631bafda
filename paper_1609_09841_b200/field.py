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
_SNAPSHOT_LAYOUT = "m3,m2,m1,n3,n2,n1"


@dataclass(frozen=True)
class GridSpec:
    """Periodic tensor-product grid: `cells_per_axis` (M1, M2, M3) over `domain_lengths`
    (L1, L2, L3); primary nodes sit at m h, dual nodes at (m + 1/2) h (reference field.py:34-77)."""

    cells_per_axis: tuple[int, int, int]
    domain_lengths: tuple[float, float, float] = (1.0, 1.0, 1.0)
    parity: str = "primary"

    def __post_init__(self):
        cells, lengths = tuple(self.cells_per_axis), tuple(self.domain_lengths)
        cells_ok = len(cells) == 3 and all(int(m) == m and m >= 1 for m in cells)
        lengths_ok = len(lengths) == 3 and all(l > 0 for l in lengths)  # NaN fails too
        if not cells_ok:
            raise ValueError(f"cells_per_axis must be three positive ints, got {self.cells_per_axis}")
        if not lengths_ok:
            raise ValueError(f"domain_lengths must be three positive reals, got {self.domain_lengths}")
        if self.parity not in PARITIES:
            raise ValueError(f"parity must be one of {PARITIES}, got {self.parity!r}")
        object.__setattr__(self, "cells_per_axis", tuple(int(m) for m in cells))
        object.__setattr__(self, "domain_lengths", lengths)

    @property
    def _shift(self) -> float:
        return 0.5 if self.parity == "dual" else 0.0

    @property
    def spacings(self) -> tuple[float, float, float]:
        """h_k = L_k / M_k."""
        return tuple(length / cells for length, cells in zip(self.domain_lengths, self.cells_per_axis))

    @property
    def num_cells(self) -> int:
        return int(np.prod(self.cells_per_axis, dtype=np.int64))

    def wrap(self, axis: int, m: int) -> int:
        """Periodic index along `axis` (1-based, as the reference numbers axes)."""
        return m % self.cells_per_axis[axis - 1]

    def node_coord(self, axis: int, m: int) -> float:
        return (self.wrap(axis, m) + self._shift) * self.spacings[axis - 1]

    def axis_coords(self, axis: int) -> np.ndarray:
        """Coordinates of this parity's nodes along `axis`, index order."""
        return (np.arange(self.cells_per_axis[axis - 1]) + self._shift) * self.spacings[axis - 1]

    def with_parity(self, parity: str) -> "GridSpec":
        return GridSpec(self.cells_per_axis, self.domain_lengths, parity)


def _default_device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1609_09841_b200 needs a CUDA device (B200); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def _dof_shape(grid: GridSpec, order_n: int) -> tuple[int, ...]:
    m1, m2, m3 = grid.cells_per_axis
    return (m3, m2, m1) + (order_n + 1,) * 3


class DofField:
    """Scaled-derivative DOFs h^|n|/n! D^n u of one parity, resident in HBM as `.tensor`
    with the reference's rank-6 layout [m3][m2][m1][n3][n2][n1] (reference field.py:80-117).

    `data` is a numpy array (uploaded) or a torch tensor (a CUDA tensor is adopted without a
    copy) of shape (M3, M2, M1, N+1, N+1, N+1), float32 or float64.
    """

    def __init__(self, grid: GridSpec, order_n: int, data, device=None):
        self.grid = grid
        self.order_n = int(order_n)
        want = _dof_shape(grid, self.order_n)
        if tuple(data.shape) != want:
            raise ValueError(f"data shape {tuple(data.shape)} does not match grid/order {want}")
        if not isinstance(data, torch.Tensor):
            data = torch.from_numpy(np.ascontiguousarray(data))
        if data.dtype not in (torch.float32, torch.float64):
            raise ValueError(f"unsupported dtype {data.dtype}")
        self.tensor = (data if data.is_cuda else data.to(device or _default_device())).contiguous()

    @classmethod
    def _allocate(cls, fill, grid, order_n, precision, device):
        if precision not in _TORCH_DTYPES:
            raise ValueError(f"precision must be one of {tuple(_TORCH_DTYPES)}, got {precision!r}")
        t = fill(_dof_shape(grid, order_n), dtype=_TORCH_DTYPES[precision], device=device or _default_device())
        return cls(grid, order_n, t)

    @classmethod
    def zeros(cls, grid: GridSpec, order_n: int, precision: str = "double", device=None) -> "DofField":
        return cls._allocate(torch.zeros, grid, order_n, precision, device)

    @classmethod
    def empty(cls, grid: GridSpec, order_n: int, precision: str = "double", device=None) -> "DofField":
        """Uninitialised device field (a half step overwrites every node)."""
        return cls._allocate(torch.empty, grid, order_n, precision, device)

    # ---- host readback / upload -------------------------------------------------------------
    @property
    def data(self) -> np.ndarray:
        """Host copy of the DOF tensor in the reference layout."""
        return self.tensor.detach().cpu().numpy()

    @data.setter
    def data(self, value) -> None:
        src = value if isinstance(value, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(value))
        if tuple(src.shape) != tuple(self.tensor.shape):
            raise ValueError(f"shape {tuple(src.shape)} does not match {tuple(self.tensor.shape)}")
        self.tensor.copy_(src.to(self.tensor.dtype))

    @property
    def values(self) -> np.ndarray:
        """Point values u at the nodes (DOF index (0, 0, 0)), [m3][m2][m1] on the host."""
        return self.tensor[..., 0, 0, 0].cpu().numpy()

    @property
    def precision(self) -> str:
        return "double" if self.tensor.dtype == torch.float64 else "single"

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


def _snapshot_paths(base_path) -> tuple[Path, Path]:
    base = Path(base_path)
    return base.with_suffix(".bin"), base.with_suffix(".json")


def write_snapshot(field: DofField, base_path, time: float = 0.0) -> tuple[Path, Path]:
    """The reference's snapshot format (field.py:175-201): `<base>.bin` holds the DOFs as flat
    little-endian floats in the rank-6 layout, `<base>.json` the grid, order, parity,
    precision, time, layout and dtype."""
    bin_path, json_path = _snapshot_paths(base_path)
    bin_path.parent.mkdir(parents=True, exist_ok=True)
    dtype = "<f8" if field.precision == "double" else "<f4"
    bin_path.write_bytes(np.ascontiguousarray(field.data, dtype=np.dtype(dtype)).tobytes())
    grid = field.grid
    meta = dict(cells_per_axis=list(grid.cells_per_axis), domain_lengths=list(grid.domain_lengths),
                order_n=field.order_n, parity=grid.parity, precision=field.precision, time=time,
                layout=_SNAPSHOT_LAYOUT, dtype=dtype)
    json_path.write_text(json.dumps(meta, sort_keys=True, indent=2) + "\n")
    return bin_path, json_path


def read_snapshot(base_path, device=None) -> tuple[DofField, float]:
    """Load a snapshot (reference field.py:204-217) straight into HBM; returns (field, time)."""
    bin_path, json_path = _snapshot_paths(base_path)
    meta = json.loads(json_path.read_text())
    grid = GridSpec(tuple(meta["cells_per_axis"]), tuple(meta["domain_lengths"]), meta["parity"])
    order_n = int(meta["order_n"])
    flat = np.frombuffer(bin_path.read_bytes(), dtype=np.dtype(meta["dtype"]))
    host = flat.reshape(_dof_shape(grid, order_n)).astype(PRECISION_DTYPES[meta["precision"]])
    return DofField(grid, order_n, host, device=device), float(meta["time"])
