"""Kernel-side cost of the multi-GPU halo paths on ONE GPU (no interconnect involved):
full steps of the periodic single field vs SlabSolver with world = 1 in p2p mode (one launch
per half step, ghost planes read through the halo pointers) and nccl mode (ghost copy +
interior launch + boundary-plane launch).  The difference is what a rank pays for the halo
machinery itself; the interconnect adds one 1-element all-reduce (p2p) or one plane transfer
(nccl) per half step on top.

usage: python tools/time_slab.py [CELLS] [STEPS]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_09841_b200 as hb  # noqa: E402
from paper_1609_09841_b200.distributed import SlabSolver  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 512
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = hb.StepConfig(variant="separable")


def timed(fn, k):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


grid = hb.GridSpec((m, m, m))
ops = hb.OperatorSet.for_grid(grid, 3)
st = hb.init_field(hb.plane_wave(), grid, 3)
sc = hb.DofField.empty(grid.with_parity("dual"), 3)
dt = hb.select_dt(grid, cfg)
base = timed(lambda: hb.full_step(st, sc, cfg, ops, dt=dt), steps)
del st, sc
torch.cuda.empty_cache()
print(f"periodic single field      {base:8.3f} ms/step")
for halo in ("p2p", "nccl"):
    s = SlabSolver((m, m, m), 3, cfg, halo=halo)
    s.init(hb.plane_wave())
    t = timed(s.step, steps)
    s.check()
    print(f"SlabSolver world=1 {halo:5s}   {t:8.3f} ms/step  ({100 * (t / base - 1):+.2f} %)")
    s.close()
    del s
    torch.cuda.empty_cache()
