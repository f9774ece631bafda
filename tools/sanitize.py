"""Small ragged-grid runs of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck): fused and two-pass, N = 1..5, separable and literal, both offsets, a slab range."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_09841_b200 as hb  # noqa: E402

cells = (19, 13, 11)
for n in (1, 2, 3, 4, 5):
    grid = hb.GridSpec(cells)
    ops = hb.OperatorSet.for_grid(grid, n)
    for mode in ("fused", "two_pass"):
        for variant in ("separable", "literal"):
            cfg = hb.StepConfig(mode=mode, variant=variant)
            st = hb.init_field(hb.plane_wave(), grid, n)
            sc = hb.DofField.zeros(grid.with_parity("dual"), n)
            hb.full_step(st, sc, cfg, ops)
    torch.cuda.synchronize()
    print("N", n, "ok", flush=True)
