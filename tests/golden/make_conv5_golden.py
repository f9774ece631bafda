"""configs[3] convergence anchor from the reference (run in the build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_conv5_golden.py

The advection problem is scale invariant: (wavenumber k, M cells, final time T) and
(k/8, M/8, 8T) have identical scaled DOFs, dt/h and step counts, so their node errors agree up
to rounding.  The reference (numba, CPU) computes the 16^3 -> 32^3 m=5 study at k=5, T=0.8;
tests/test_gpu_configs.py runs configs[3]'s 128^3 -> 256^3 at k=40, T=0.1 on the GPU and
compares errors and observed order with these numbers.
"""
import json
import math
from pathlib import Path

import numba

import hermite3d as h3

numba.set_num_threads(numba.config.NUMBA_NUM_THREADS)
N, K, T = 5, 5, 0.8
rows = []
for m in (16, 32):
    grid = h3.GridSpec((m, m, m))
    ops = h3.OperatorSet.for_grid(grid, N)
    cfg = h3.StepConfig(mode="fused")
    ic = h3.plane_wave(K)
    state = h3.init_field(ic, grid, N)
    scratch = h3.DofField.zeros(grid.with_parity("dual"), N)
    steps = max(1, math.ceil(T / h3.select_dt(grid, cfg) - 1e-12))
    for _ in range(steps):
        h3.full_step(state, scratch, cfg, ops, dt=T / steps)
    err = h3.compute_error(state, h3.exact_solution(ic, T))
    rows.append({"cells": m, "steps": steps, "l_inf": err.l_inf, "l2": err.l2})
order = math.log2(rows[0]["l_inf"] / rows[1]["l_inf"])
out = {"order_n": N, "wavenumber": K, "final_time": T, "rows": rows, "order_linf": order,
       "scaled_to": {"wavenumber": 8 * K, "final_time": T / 8, "cells": [8 * r["cells"] for r in rows]}}
Path(__file__).with_name("conv5.json").write_text(json.dumps(out, indent=1))
print(json.dumps(out))
