"""Generate tests/golden/golden.json by running the REAL reference in this container.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

The reference (hermite3d, pure Python + numba) cannot travel to the GPU box,
so its outputs are frozen here as sha256 digests, scalars and exact
operator matrices.  tests/test_oracle_golden.py pins the CPU oracle
(oracle/) to these values; the GPU parity tests then compare the CUDA path
with the pinned oracle.  All inputs are reproducible from seeds / analytic
initial data, so only digests need to be stored.

Reference entry points exercised (pkg/src/hermite3d/):
  pipeline.full_step / half_step (pipeline.py:218-293), both modes
  gridkernels.fused_pass / recon_pass / evolve_pass (gridkernels.py:121-182)
  problems.init_field / plane_wave / compute_error (problems.py:131-213)
  operators.build_interp_operator (operators.py:62-110)
"""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

import hermite3d as h3
from hermite3d import gridkernels, pipeline

OUT = Path(__file__).resolve().parent / "golden.json"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_ic(seed, n_terms=3, kmax=2):
    rng = np.random.default_rng(seed)
    terms = []
    for _ in range(n_terms):
        terms.append(tuple(
            h3.FourierMode(amplitude=float(rng.uniform(-1, 1)),
                           wavenumber=int(rng.integers(1, kmax + 1)),
                           phase=float(rng.uniform(0, 2 * np.pi)))
            for _ in range(3)))
    return h3.SeparableIC(terms=tuple(terms))


def ic_terms(ic):
    return [[[f.amplitude, f.wavenumber, f.phase] for f in term] for term in ic.terms]


def run_steps(cells, lengths, order_n, steps, ic, mode, precision="double", stages_q=None):
    grid = h3.GridSpec(cells, lengths)
    ops = h3.OperatorSet.for_grid(grid, order_n)
    cfg = h3.StepConfig(mode=mode, precision=precision, stages_q=stages_q)
    state = h3.init_field(ic, grid, order_n, precision)
    init_sha = sha(state.data)
    scratch = h3.DofField.zeros(grid.with_parity("dual"), order_n, precision)
    dt = h3.select_dt(grid, cfg)
    for k in range(steps):
        h3.full_step(state, scratch, cfg, ops, dt=dt, step_index=k)
    err = h3.compute_error(state, h3.exact_solution(ic, steps * dt, lengths))
    return dict(init_sha=init_sha, final_sha=sha(state.data), scratch_sha=sha(scratch.data),
                dt=dt, l_inf=err.l_inf, l2=err.l2)


def main():
    out = {"generator": "tests/golden/make_golden.py", "reference_version": h3.__version__}

    # Exact interpolation matrices (operators.py:62-74), bit patterns as hex floats.
    out["interp_matrix_hex"] = {
        str(n): [[float(v).hex() for v in row] for row in h3.build_interp_operator(n).matrix]
        for n in range(0, 7)}

    # Multi-step runs (SURVEY Appendix A rows + extra coverage).
    runs = []
    plane = h3.plane_wave()
    for (n, m, steps) in [(1, 16, 10), (3, 12, 10), (3, 16, 4), (5, 8, 5), (0, 8, 6),
                          (2, 10, 6), (4, 6, 3)]:
        row = dict(order_n=n, cells=[m, m, m], lengths=[1.0, 1.0, 1.0], steps=steps,
                   ic="plane_wave", ic_terms=ic_terms(plane), precision="double")
        fused = run_steps((m, m, m), (1.0, 1.0, 1.0), n, steps, plane, "fused")
        two = run_steps((m, m, m), (1.0, 1.0, 1.0), n, steps, plane, "two_pass")
        assert fused["final_sha"] == two["final_sha"], "reference modes disagree"
        row.update(fused)
        runs.append(row)
    # anisotropic, non-cubic, random multi-mode IC, both precisions
    for precision in ("double", "single"):
        ic = random_ic(7)
        cells, lengths = (7, 5, 6), (1.0, 2.0, 3.0)
        row = dict(order_n=2, cells=list(cells), lengths=list(lengths), steps=3,
                   ic="random_ic(7)", ic_terms=ic_terms(ic), precision=precision)
        row.update(run_steps(cells, lengths, 2, 3, ic, "fused", precision))
        two = run_steps(cells, lengths, 2, 3, ic, "two_pass", precision)
        assert row["final_sha"] == two["final_sha"]
        runs.append(row)
    # reduced stage count q = 2N+1 (not exact; literal path only)
    ic = random_ic(11)
    row = dict(order_n=3, cells=[9, 8, 7], lengths=[1.0, 1.0, 1.0], steps=2, ic="random_ic(11)",
               ic_terms=ic_terms(ic), precision="double", stages_q=7)
    row.update(run_steps((9, 8, 7), (1.0, 1.0, 1.0), 3, 2, ic, "fused", stages_q=7))
    runs.append(row)
    out["runs"] = runs

    # Single passes on seeded uniform input (perf.py:189-191 input recipe), both offsets.
    passes = []
    for (n, cells) in [(1, (16, 16, 16)), (3, (16, 16, 16)), (5, (8, 8, 8)), (2, (5, 1, 3)),
                       (3, (1, 1, 1)), (1, (33, 7, 2))]:
        m1, m2, m3 = cells
        npts = n + 1
        grid = h3.GridSpec(cells)
        ops = h3.OperatorSet.for_grid(grid, n)
        cfg = h3.StepConfig()
        dt = h3.select_dt(grid, cfg)
        q = cfg.stages(n)
        src = np.random.default_rng(0).uniform(-1.0, 1.0, (m3, m2, m1, npts, npts, npts))
        for off in (0, -1):
            h_mat, f1, f2, f3, cf = pipeline._factor_arrays(ops, np.float64, dt / 2, q)
            tiles = gridkernels.make_tiles(cells, 3)
            dst = np.zeros_like(src)
            gridkernels.fused_pass(src, dst, h_mat, f1, f2, f3, cf, tiles, off)
            s = 2 * npts
            coeff = np.empty((m3, m2, m1, s, s, s))
            gridkernels.recon_pass(src, coeff, h_mat, tiles, off)
            dst2 = np.zeros_like(src)
            gridkernels.evolve_pass(coeff, dst2, f1, f2, f3, cf, tiles)
            assert sha(dst2) == sha(dst)
            passes.append(dict(order_n=n, cells=list(cells), off=off, seed=0, dt=dt, q=q,
                               dst_sha=sha(dst), coeff_sha=sha(coeff),
                               dst0=float(dst.flat[0]), max_abs=float(np.abs(dst).max())))
    out["passes"] = passes

    # Instability: a NaN planted in a primary node is reported as the first bad dual node.
    grid = h3.GridSpec((6, 5, 4))
    ops = h3.OperatorSet.for_grid(grid, 1)
    state = h3.init_field(plane, grid, 1)
    state.data[2, 3, 4, 0, 1, 0] = np.nan
    scratch = h3.DofField.zeros(grid.with_parity("dual"), 1)
    try:
        h3.full_step(state, scratch, h3.StepConfig(), ops, step_index=5)
        raise AssertionError("expected InstabilityError")
    except h3.InstabilityError as exc:
        out["instability"] = dict(cells=[6, 5, 4], order_n=1, nan_at=[2, 3, 4, 0, 1, 0],
                                  node=list(exc.node), step=exc.step)

    OUT.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
