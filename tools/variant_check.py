"""Correctness of a measurement-build kernel variant (tools/ab.sh settings): one fused half step
of each parity on a smooth random field, separable (the variant selected by the H3_* knobs) vs
the literal kernel of the same library (the reference's arithmetic).

usage: H3_LIB=build/libh3b200_measure.so H3_DMMA5_CFG=9 python tools/variant_check.py 5 40 36 20 [MODE]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import _lib  # noqa: E402
_lib.select_library()
import paper_1609_09841_b200 as hb  # noqa: E402

n = int(sys.argv[1])
cells = tuple(int(v) for v in sys.argv[2:5])
mode = sys.argv[5] if len(sys.argv) > 5 else "fused"
grid = hb.GridSpec(cells)
rng = np.random.default_rng(5)
ic = hb.SeparableIC(tuple(tuple(hb.FourierMode(float(rng.uniform(-1, 1)), int(rng.integers(1, 4)),
                                               float(rng.uniform(0, 6.28))) for _ in range(3)) for _ in range(4)))
worst = 0.0
for parity in ("primary", "dual"):
    g = grid.with_parity(parity)
    other = g.with_parity("dual" if parity == "primary" else "primary")
    src = hb.init_field(ic, grid, n)
    src = hb.DofField(g, n, src.tensor)
    outs = {}
    for variant in ("literal", "separable"):
        dst = hb.DofField.zeros(other, n)
        hb.half_step(src, dst, hb.StepConfig(variant=variant, mode=mode), hb.OperatorSet.for_grid(grid, n))
        outs[variant] = dst.tensor
    err = float((outs["separable"] - outs["literal"]).abs().max() / outs["literal"].abs().max())
    worst = max(worst, err)
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("H3_") and k != "H3_LIB")
print(f"variant_check N={n} cells={cells} {mode} [{env}] separable vs literal (one half step, both parities): "
      f"{worst:.3e} {'OK' if worst <= (5e-9 if n >= 5 else 1e-12) else 'FAIL'}", flush=True)
torch.cuda.synchronize()
