"""Host overhead per step on small grids (launch-bound regime): eager vs CUDA-graph run_steps."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_09841_b200 as hb  # noqa: E402

case = sys.argv[1:] or ["3", "16", "fused"]
n, m, mode = int(case[0]), int(case[1]), case[2]
grid = hb.GridSpec((m, m, m))
cfg = hb.StepConfig(mode=mode)
ops = hb.OperatorSet.for_grid(grid, n)
st = hb.init_field(hb.plane_wave(), grid, n)
sc = hb.DofField.zeros(grid.with_parity("dual"), n)
k = 256
for graph in ((False, True) if mode == "fused" else (False,)):
    hb.run_steps(st, sc, cfg, ops, k, graph=graph)  # warm (captures the graphs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hb.run_steps(st, sc, cfg, ops, k, graph=graph)
    torch.cuda.synchronize()
    dt_ = (time.perf_counter() - t0) / k
    print(f"N={n} {m}^3 {mode} graph={graph}: {1e6 * dt_:.1f} us/step", flush=True)
