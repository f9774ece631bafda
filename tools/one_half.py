"""One separable half step at (ORDER, CELLS, MODE) after a warm-up, for ncu captures."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import _lib  # noqa: E402
_lib.select_library()
import paper_1609_09841_b200 as hb  # noqa: E402

n, m = int(sys.argv[1]), int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "fused"
g = hb.GridSpec((m, m, m))
ops = hb.OperatorSet.for_grid(g, n)
cfg = hb.StepConfig(mode=mode, variant="separable")
st = hb.init_field(hb.plane_wave(), g, n)
sc = hb.DofField.empty(g.with_parity("dual"), n)
hb.half_step(st, sc, cfg, ops)
hb.half_step(sc, st, cfg, ops)
torch.cuda.synchronize()
