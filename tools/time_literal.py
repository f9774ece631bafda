"""Throughput of the bit-exact literal variant (the reference's arithmetic, no FMA) vs the fast
separable one: ms per half step and DOF-updates/s.   usage: python tools/time_literal.py ORDER CELLS"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import _lib  # noqa: E402
_lib.select_library()
import paper_1609_09841_b200 as hb  # noqa: E402

n, m = int(sys.argv[1]), int(sys.argv[2])
grid = hb.GridSpec((m, m, m))
ops = hb.OperatorSet.for_grid(grid, n)
for variant in ("literal", "separable"):
    for mode in ("fused", "two_pass"):
        cfg = hb.StepConfig(mode=mode, variant=variant)
        st = hb.init_field(hb.plane_wave(), grid, n)
        sc = hb.DofField.empty(grid.with_parity("dual"), n)
        hb.run_steps(st, sc, cfg, ops, 1)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        hb.run_steps(st, sc, cfg, ops, 2)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 4
        print(f"N={n} M={m} {variant:9s} {mode:8s} {ms:9.3f} ms/half-step  "
              f"{m ** 3 * (n + 1) ** 3 / (2 * ms / 1e3):.3e} DOF-updates/s", flush=True)
        del st, sc
        torch.cuda.empty_cache()
