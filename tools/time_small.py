"""Host overhead per half step on small grids (launch-bound regime)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_09841_b200 as hb  # noqa: E402

for n, m, mode in ((3, 16, "fused"), (3, 16, "two_pass"), (1, 16, "fused"), (5, 8, "fused")):
    grid = hb.GridSpec((m, m, m))
    cfg = hb.StepConfig(mode=mode)
    ops = hb.OperatorSet.for_grid(grid, n)
    st = hb.init_field(hb.plane_wave(), grid, n)
    sc = hb.DofField.zeros(grid.with_parity("dual"), n)
    hb.run_steps(st, sc, cfg, ops, 5)
    torch.cuda.synchronize()
    k = 200
    t0 = time.perf_counter()
    hb.run_steps(st, sc, cfg, ops, k)
    t1 = time.perf_counter()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        hb.full_step(st, sc, cfg, ops)
    t2 = time.perf_counter()
    for _ in range(50):
        hb.full_step(st, sc, cfg, ops)
    t3 = time.perf_counter()
    print(f"N={n} {m}^3 {mode}: run_steps {1e6 * (t1 - t0) / k:.1f} us/step, full_step {1e6 * (t3 - t2) / 50:.1f} us/step",
          flush=True)
