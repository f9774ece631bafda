"""INTEGRATION.md's ctypes binding, executed as written, through the reference's call sites.

The code block under "ctypes binding a maintainer would add" is read from INTEGRATION.md and
executed (only the library path is made absolute).  Its fused_pass / recon_pass / evolve_pass
take the reference's exact signatures (gridkernels.py:121,142,163) and are called the way
pipeline.half_step calls them (pipeline.py:247-273): host numpy fields, factor arrays from
_factor_arrays, the tile table.  Every golden single pass of the reference is reproduced bit
for bit (literal variant), fused and two-pass.
"""

import hashlib
import re

import numpy as np
import pytest

from oracle import refmodel as rm
from conftest import GOLDEN, ROOT
import paper_1609_09841_b200 as hb
from paper_1609_09841_b200 import _native

pytestmark = pytest.mark.gpu


def _stub_namespace():
    text = (ROOT / "INTEGRATION.md").read_text()
    block = re.search(r"### ctypes binding.*?```python\n(.*?)```", text, re.S).group(1)
    code = block.replace('ctypes.CDLL("libh3b200.so")', f'ctypes.CDLL("{_native.LIB_PATH}")')
    ns: dict = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    return ns


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("mode", ["fused", "two_pass"])
@pytest.mark.parametrize("row", GOLDEN["passes"], ids=lambda r: f"N{r['order_n']}-{r['cells']}-off{r['off']}")
def test_integration_stub_reproduces_reference_passes(row, mode):
    stub = _stub_namespace()
    n = row["order_n"]
    m1, m2, m3 = row["cells"]
    src = np.random.default_rng(row["seed"]).uniform(-1, 1, (m3, m2, m1, n + 1, n + 1, n + 1))
    dst = np.empty_like(src)
    q = row["q"]
    h_mat, f1, f2, f3, cf = rm.factor_arrays(n, (m1, m2, m3), (1.0, 1.0, 1.0), row["dt"] / 2, q)
    tiles = hb.tile_schedule(hb.GridSpec((m1, m2, m3)), min(2, m1))
    if mode == "fused":
        stub["fused_pass"](src, dst, h_mat, f1, f2, f3, cf, tiles, row["off"])
    else:
        s = 2 * n + 2
        coeff = np.empty((m3, m2, m1, s, s, s))
        stub["recon_pass"](src, coeff, h_mat, tiles, row["off"])
        assert sha(coeff) == row["coeff_sha"]
        stub["evolve_pass"](coeff, dst, f1, f2, f3, cf, tiles)
    assert sha(dst) == row["dst_sha"]
