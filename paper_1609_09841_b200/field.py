"""Grid description and device-resident DOF fields.

Mirrors the reference's data layer (pkg/src/hermite3d/field.py):

* `GridSpec` -- periodic tensor grid, h_k = L_k / M_k, primary nodes at m*h and
  dual nodes at (m + 1/2) h (field.py:34-77).
* `DofField` -- scaled-derivative DOFs h^|n|/n! D^n u of one parity in the
  reference's rank-6 C-order layout [m3][m2][m1][n3][n2][n1] (field.py:80-117).

* `CellCoeffs`, `gather_cell`, `scatter_dofs` -- the per-cell data helpers
  (field.py:120-172).

B200 difference: the DOFs live in HBM as a torch tensor (`.tensor`) in exactly
that layout, so the CUDA kernels read and write it in place.  `.data` is a
coherent host mirror (the ndarray the reference exposes: reads and in-place
writes behave as in the reference, see `DofField`), `.values` a view of its
node values [m3][m2][m1].  Snapshots (field.py:175-217) read/write the
reference's byte format.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

__all__ = ["GridSpec", "DofField", "CellCoeffs", "gather_cell", "scatter_dofs", "write_snapshot", "read_snapshot",
           "PRECISION_DTYPES"]

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


_FLOAT_DTYPES = (np.dtype(np.float32), np.dtype(np.float64))


class DofField:
    """Scaled-derivative DOFs h^|n|/n! D^n u of one parity in the reference's rank-6 layout
    [m3][m2][m1][n3][n2][n1] (reference field.py:80-117), resident in HBM for the kernels.

    Storage is a coherent pair: the device tensor `.tensor` (what every kernel reads and
    writes) and a host mirror `.data`, the ndarray the reference exposes.  Exactly one side
    is current at a time:

    * `.data` returns the host mirror ndarray, first copying the device contents into it if
      the device side is current.  Reads, and writes through it or through any view of it
      (`field.data[idx] = v`, `field.data.ravel()[k] = v`, `field.values[...] = v`), act on
      the field, as in the reference.
    * The next device use (`.tensor`: any half step, error norm, ...) uploads the mirror
      first, so those writes reach the kernels.  After a device operation, re-read `.data`
      (the same ndarray object is refreshed in place); a mirror obtained before a step is not
      updated by the step until then.

    A field stepped without touching `.data` never transfers anything.  `data` given to the
    constructor is adopted without a copy: a CUDA tensor becomes the device side, a numpy
    array (or CPU tensor) the host mirror (uploaded on first device use).  Without a CUDA
    device a field is a host container only; any kernel raises.
    """

    def __init__(self, grid: GridSpec, order_n: int, data, device=None):
        self.grid = grid
        self.order_n = int(order_n)
        want = _dof_shape(grid, self.order_n)
        if tuple(data.shape) != want:
            raise ValueError(f"data shape {tuple(data.shape)} does not match grid/order {want}")
        self._device_hint = torch.device(device) if device is not None else None
        self._dev: torch.Tensor | None = None
        self._host: np.ndarray | None = None
        if isinstance(data, torch.Tensor):
            if data.dtype not in (torch.float32, torch.float64):
                raise ValueError(f"unsupported dtype {data.dtype}")
            if data.is_cuda:
                self._dev, self._on_device = data.contiguous(), True
                return
            data = data.detach().numpy()
        arr = np.asarray(data)
        if arr.dtype not in _FLOAT_DTYPES:
            raise ValueError(f"unsupported dtype {arr.dtype}")
        self._host, self._on_device = np.ascontiguousarray(arr), False

    @classmethod
    def _allocate(cls, fill, grid, order_n, precision, device):
        if precision not in _TORCH_DTYPES:
            raise ValueError(f"precision must be one of {tuple(_TORCH_DTYPES)}, got {precision!r}")
        shape = _dof_shape(grid, order_n)
        if device is None and not torch.cuda.is_available():  # host container (no kernels)
            host = np.zeros if fill is torch.zeros else np.empty
            return cls(grid, order_n, host(shape, dtype=PRECISION_DTYPES[precision]))
        t = fill(shape, dtype=_TORCH_DTYPES[precision], device=device or _default_device())
        return cls(grid, order_n, t)

    @classmethod
    def zeros(cls, grid: GridSpec, order_n: int, precision: str = "double", device=None) -> "DofField":
        return cls._allocate(torch.zeros, grid, order_n, precision, device)

    @classmethod
    def empty(cls, grid: GridSpec, order_n: int, precision: str = "double", device=None) -> "DofField":
        """Uninitialised device field (a half step overwrites every node)."""
        return cls._allocate(torch.empty, grid, order_n, precision, device)

    # ---- the two sides ------------------------------------------------------------------------
    @property
    def tensor(self) -> torch.Tensor:
        """The device tensor the kernels use (uploads the host mirror first if it is current)."""
        if not self._on_device:
            src = torch.from_numpy(self._host)
            if self._dev is None or self._dev.dtype != src.dtype:
                self._dev = torch.empty(src.shape, dtype=src.dtype, device=self._device_hint or _default_device())
            self._dev.copy_(src)
            self._on_device = True
        return self._dev

    @tensor.setter
    def tensor(self, value: torch.Tensor | None) -> None:
        """Adopt a device tensor of the field's shape (None drops all storage: `release`)."""
        if value is None:
            self.release()
            return
        if tuple(value.shape) != _dof_shape(self.grid, self.order_n) or not value.is_cuda:
            raise ValueError("tensor must be a CUDA tensor of the field's shape")
        self._dev, self._on_device = value, True

    def release(self) -> None:
        """Free both storages (the field is unusable afterwards)."""
        self._dev = self._host = None
        self._on_device = True

    @property
    def data(self) -> np.ndarray:
        """The host mirror ndarray in the reference layout (see the class docstring)."""
        if self._on_device:
            if self._dev is None:
                raise RuntimeError("the field's storage was released")
            if self._host is None or self._host.dtype != _NP_OF[self._dev.dtype]:
                self._host = np.empty(tuple(self._dev.shape), dtype=_NP_OF[self._dev.dtype])
            torch.from_numpy(self._host).copy_(self._dev)
            self._on_device = False
        return self._host

    @data.setter
    def data(self, value) -> None:
        arr = value.detach().cpu().numpy() if isinstance(value, torch.Tensor) else np.asarray(value)
        if tuple(arr.shape) != _dof_shape(self.grid, self.order_n):
            raise ValueError(f"shape {tuple(arr.shape)} does not match {_dof_shape(self.grid, self.order_n)}")
        if arr.dtype not in _FLOAT_DTYPES:
            raise ValueError(f"unsupported dtype {arr.dtype}")
        self._host, self._on_device = np.ascontiguousarray(arr), False

    @property
    def values(self) -> np.ndarray:
        """Point values u at the nodes (DOF index (0, 0, 0)), [m3][m2][m1]: a view of `.data`."""
        return self.data[..., 0, 0, 0]

    def host_copy(self) -> np.ndarray:
        """The current contents on the host without changing which side is current (a copy
        when the device side is current, the mirror itself otherwise -- read it, don't write)."""
        if self._on_device:
            return self._dev.detach().cpu().numpy()
        return self._host

    def _read_nodes(self, index) -> np.ndarray:
        """Host copy of `field[index]` (node blocks) from whichever side is current."""
        if self._on_device:
            if isinstance(index, tuple):
                index = tuple(torch.as_tensor(i, device=self._dev.device) if isinstance(i, np.ndarray) else i
                              for i in index)
            return self._dev[index].cpu().numpy()
        return np.array(self._host[index])

    def _write_nodes(self, index, value) -> None:
        """`field[index] = value` on whichever side is current (no whole-field transfer)."""
        if self._on_device:
            self._dev[index] = torch.as_tensor(np.asarray(value), dtype=self._dev.dtype)
        else:
            self._host[index] = value

    @property
    def precision(self) -> str:
        dtype = self._dev.dtype if self._on_device else self._host.dtype
        return "double" if dtype in (torch.float64, np.float64) else "single"

    @property
    def device(self):
        if self._dev is not None:
            return self._dev.device
        return self._device_hint or _default_device()

    @property
    def nbytes(self) -> int:
        return int(np.prod(_dof_shape(self.grid, self.order_n))) * (8 if self.precision == "double" else 4)

    def copy(self) -> "DofField":
        if self._on_device:
            return DofField(self.grid, self.order_n, self._dev.clone())
        return DofField(self.grid, self.order_n, self._host.copy(), device=self._device_hint)

    def all_finite(self) -> bool:
        if self._on_device:
            return bool(torch.isfinite(self._dev).all().item())
        return bool(np.isfinite(self._host).all())


_NP_OF = {torch.float64: np.dtype(np.float64), torch.float32: np.dtype(np.float32)}


@dataclass
class CellCoeffs:
    """Coefficients of one cell's midpoint-centred tensor polynomial, data[n3][n2][n1] with
    side 2N+2 (reference field.py:120-139): a host ndarray, the per-cell API's currency."""

    order_n: int
    data: np.ndarray

    def __post_init__(self):
        side = 2 * self.order_n + 2
        if tuple(np.shape(self.data)) != (side, side, side):
            raise ValueError(f"coeff tensor must have side {side}, got shape {np.shape(self.data)}")

    @classmethod
    def zeros(cls, order_n: int, dtype=np.float64) -> "CellCoeffs":
        side = 2 * order_n + 2
        return cls(order_n=order_n, data=np.zeros((side, side, side), dtype=dtype))


def _wrapped_node(field: DofField, node) -> tuple[int, int, int]:
    c1, c2, c3 = node
    return field.grid.wrap(3, c3), field.grid.wrap(2, c2), field.grid.wrap(1, c1)


def gather_cell(field: DofField, cell: tuple[int, int, int]) -> np.ndarray:
    """The 8-vertex DOF tensor of the cell with low corner `cell` = (c1, c2, c3), wrapped
    periodically (reference field.py:142-162): side 2N+2, indices 0..N along an axis hold the
    low vertex's derivatives, N+1..2N+1 the high vertex's.  Reads only those 8 node blocks
    (from whichever side of the field is current)."""
    n = field.order_n + 1
    c1, c2, c3 = cell
    z = [field.grid.wrap(3, c3 + a) for a in (0, 1)]
    y = [field.grid.wrap(2, c2 + a) for a in (0, 1)]
    x = [field.grid.wrap(1, c1 + a) for a in (0, 1)]
    blocks = field._read_nodes((np.array(z)[:, None, None], np.array(y)[None, :, None], np.array(x)[None, None, :]))
    # blocks[a3, a2, a1, j3, j2, j1] -> out[a3 n + j3, a2 n + j2, a1 n + j1]
    return np.ascontiguousarray(blocks.transpose(0, 3, 1, 4, 2, 5).reshape(2 * n, 2 * n, 2 * n))


def scatter_dofs(coeffs: CellCoeffs, field: DofField, node: tuple[int, int, int]) -> None:
    """Write a cell's low coefficients (indices <= N per axis) as the DOFs of `node`
    = (m1, m2, m3), wrapped; the higher coefficients are dropped (reference field.py:165-172)."""
    n = field.order_n + 1
    field._write_nodes(_wrapped_node(field, node), np.asarray(coeffs.data)[:n, :n, :n])


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
    bin_path.write_bytes(np.ascontiguousarray(field.host_copy(), dtype=np.dtype(dtype)).tobytes())
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
