"""ctypes binding of libh3b200.so (the C ABI declared in include/h3b200.h).

The product path has no CPU fallback: if the shared library is missing or
fails to load, every entry point raises `NativeLibraryError`.
"""

from __future__ import annotations

import ctypes
import subprocess
from functools import lru_cache
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libh3b200.so"
CSRC = _PKG / "csrc"

NO_BAD_NODE = 0xFFFFFFFFFFFFFFFF
VARIANTS = {"auto": 0, "literal": 1, "separable": 2}

# exported symbol -> (restype, argtypes); must mirror include/h3b200.h
_i64, _i32, _vp, _u64p = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p
SIGNATURES = {
    "h3_fused_pass": (_i32, [_vp, _vp, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _i32, _i32,
                             _i64, _i64, _i32, _i32, _vp, _u64p, _u64p]),
    "h3_fused_pass_f32": (_i32, [_vp, _vp, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _i32,
                                 _i32, _i64, _i64, _i32, _i32, _vp, _u64p, _u64p]),
    "h3_recon_pass": (_i32, [_vp, _vp, _i64, _i64, _i64, _i32, _vp, _i32, _i64, _i64, _i32, _i32,
                             _vp, _u64p]),
    "h3_recon_pass_f32": (_i32, [_vp, _vp, _i64, _i64, _i64, _i32, _vp, _i32, _i64, _i64, _i32,
                                 _i32, _vp, _u64p]),
    "h3_evolve_pass": (_i32, [_vp, _vp, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _i32, _i64,
                              _i64, _i32, _vp, _u64p, _u64p]),
    "h3_evolve_pass_f32": (_i32, [_vp, _vp, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _i32, _i64,
                                  _i64, _i32, _vp, _u64p, _u64p]),
    "h3_separable_operators": (_i32, [_i32, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp]),
    "h3_init_separable": (_i32, [_vp, _i64, _i64, _i64, _i32, _i32, _vp, _vp, _vp, _vp]),
    "h3_error_norms": (_i32, [_vp, _i64, _i64, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _i64, _vp,
                              _vp]),
    "h3_check_finite": (_i32, [_vp, _i64, _i64, _i64, _i32, _u64p, _vp]),
    "h3_fused_pass_halo": (_i32, [_vp, _vp, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _i32, _i32,
                                  _i64, _i64, _vp, _vp, _i32, _vp, _u64p, _u64p]),
    "h3_ipc_export": (_i32, [_vp, _vp, _vp]),
    "h3_ipc_open": (_i32, [_vp, _vp]),
    "h3_ipc_close": (_i32, [_vp]),
    "h3_cell_apply_axis": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _i32, _i32, _vp]),
    "h3_cell_advect": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _i32, _vp]),
    "h3_cell_horner": (_i32, [_vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _i32, _i32, _vp]),
    "h3_cell_space_time": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _i32, _i32, _vp]),
    "h3_cell_time_sum": (_i32, [_vp, _vp, _i64, _i64, _vp, _i32, _i32, _vp]),
    "h3_cell_identity_residual": (_i32, [_vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _i32, _u64p, _i32,
                                         _vp]),
    "h3_version": (ctypes.c_char_p, []),
    "h3_error_string": (ctypes.c_char_p, [_i32]),
    "h3_max_order": (_i32, []),
    "h3_max_stages": (_i32, []),
}


class NativeLibraryError(RuntimeError):
    """libh3b200.so is missing, failed to load, or a call returned an error."""


def build(verbose: bool = False) -> Path:
    """Compile libh3b200.so in-tree for sm_100a (nvcc; no GPU needed)."""
    cmd = ["make", "-C", str(CSRC), "-j4"]
    res = subprocess.run(cmd, capture_output=not verbose, text=True)
    if res.returncode != 0:
        raise NativeLibraryError(f"building libh3b200.so failed:\n{res.stdout}\n{res.stderr}")
    return LIB_PATH


_LIB_OVERRIDE: Path | None = None


def use_library(path) -> None:
    """Bind a different build of the same C ABI before first use -- for the measurement tools,
    which load build/libh3b200_measure.so (`make -C csrc measure`: the same kernels plus
    measurement-only variants).  The product never calls this."""
    global _LIB_OVERRIDE
    if lib.cache_info().currsize:
        raise NativeLibraryError("use_library() must be called before the library is first used")
    _LIB_OVERRIDE = Path(path)


@lru_cache(maxsize=None)
def lib() -> ctypes.CDLL:
    path = _LIB_OVERRIDE or LIB_PATH
    if not path.exists():
        raise NativeLibraryError(
            f"{path} not found; build it with `make -C {CSRC}` or __graft_entry__.build()")
    try:
        so = ctypes.CDLL(str(path))
    except OSError as exc:
        raise NativeLibraryError(f"failed to load {path}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(so, name)
        fn.restype = res
        fn.argtypes = args
    return so


def error_string(status: int) -> str:
    return lib().h3_error_string(int(status)).decode()


def check(status: int, what: str) -> None:
    if status != 0:
        raise NativeLibraryError(f"{what} failed with status {status}: {error_string(status)}")


def version() -> str:
    return lib().h3_version().decode()
