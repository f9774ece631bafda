"""Time the fused (or two-pass) half step at one size: ms per half step and algorithmic GB/s.

usage: python tools/time_fused.py ORDER CELLS [MODE] [STEPS]   (env H3_* knobs select kernel variants)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import _lib  # noqa: E402
_lib.select_library()
import paper_1609_09841_b200 as hb  # noqa: E402

n = int(sys.argv[1])
m = int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "fused"
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 8
grid = hb.GridSpec((m, m, m))
cfg = hb.StepConfig(mode=mode, variant="separable")
ops = hb.OperatorSet.for_grid(grid, n)
st = hb.init_field(hb.plane_wave(), grid, n)
sc = hb.DofField.empty(grid.with_parity("dual"), n)
hb.run_steps(st, sc, cfg, ops, 2)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
hb.run_steps(st, sc, cfg, ops, steps)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / (2 * steps)
per = 16 * (n + 1) ** 3 if mode == "fused" else 16 * ((n + 1) ** 3 + (2 * n + 2) ** 3)
gbs = per * m ** 3 / (ms / 1e3) / 1e9
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("H3_"))
print(f"N={n} M={m} {mode} [{env}] {ms:.3f} ms/half-step  {gbs:.0f} GB/s  "
      f"{m**3 * (n + 1)**3 / (2 * ms / 1e3):.3e} DOF-updates/s", flush=True)
