"""compute-sanitizer target for the warp-specialised N=5 kernels alone: one full step of each mode
(fused: h3_dmma5ws.cu; two-pass: the reconstruction of h3_recon5ws.cu + the evolve kernel) on a
ragged grid (tiles cut at both x1/x2 edges, several z chunks).

usage: compute-sanitizer --tool racecheck python tools/sanitize_ws.py [M1 M2 M3]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_09841_b200 as hb  # noqa: E402

cells = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (7, 13, 5)
grid = hb.GridSpec(cells)
ops = hb.OperatorSet.for_grid(grid, 5)
for mode in ("fused", "two_pass"):
    st = hb.init_field(hb.plane_wave(), grid, 5)
    sc = hb.DofField.zeros(grid.with_parity("dual"), 5)
    hb.full_step(st, sc, hb.StepConfig(variant="separable", mode=mode), ops)
    torch.cuda.synchronize()
    print(f"ws {mode} ok", flush=True)
