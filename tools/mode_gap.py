"""SPEC acceptance 2 measured: fused vs two-pass max relative field difference,
N = 1..5, M = 12^3, 10 full steps, random multi-mode IC, for each kernel variant.

usage: python tools/mode_gap.py            (prints one line per (variant, N))
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_09841_b200 as hb  # noqa: E402


def random_ic(seed=3):
    rng = np.random.default_rng(seed)
    return hb.SeparableIC(tuple(tuple(hb.FourierMode(float(rng.uniform(-1, 1)), int(rng.integers(1, 3)),
                                                     float(rng.uniform(0, 6.28))) for _ in range(3))
                                for _ in range(4)))


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


grid = hb.GridSpec((12, 12, 12))
for variant in ("separable", "literal"):
    for n in range(1, 6):
        outs = {}
        for mode in ("fused", "two_pass"):
            st = hb.init_field(random_ic(), grid, n)
            sc = hb.DofField.zeros(grid.with_parity("dual"), n)
            hb.run_steps(st, sc, hb.StepConfig(mode=mode, variant=variant), hb.OperatorSet.for_grid(grid, n), 10,
                         graph=False)
            outs[mode] = st.data.copy()
        print(f"mode_gap variant={variant} N={n}: fused vs two_pass rel {rel(outs['two_pass'], outs['fused']):.3e}",
              flush=True)
