"""Measurement tools bind the library named by H3_LIB (tools/ab.sh sets it to the measurement
build or another copy of libh3b200.so); the product package itself never reads it."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def select_library() -> None:
    from paper_1609_09841_b200 import _native
    path = os.environ.get("H3_LIB")
    if path:
        _native.use_library(path if os.path.isabs(path) else ROOT / path)
