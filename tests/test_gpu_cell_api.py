"""The per-cell API (reference kernels.py:73-191, field.py:120-172) on the GPU.

1. Bit-identity with the reference: every function's output on seeded inputs has the sha256
   the reference produced (tests/golden/cell.json, tests/golden/make_cell_golden.py), for
   N = 0, 1, 2, 3, 5 in both precisions.
2. The reference's own per-cell tests (pkg/tests/test_kernels.py), restated against this
   package: exactness of the reconstruction, nilpotency (extra stages are no-ops), exact
   linear shifts, Horner/recursion agreement within 8 ulp, exact local evolution against the
   shifted polynomial, linearity, and the space-time identity.
3. The coherent host mirror of a device-resident DofField: reference-style in-place writes
   through `.data` / `.values` reach the kernels, gather/scatter act on the device field.
"""

import hashlib
import json
import math
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_1609_09841_b200 as hb
from paper_1609_09841_b200.kernels import space_time_tensor

pytestmark = pytest.mark.gpu

CELL = json.loads((Path(__file__).parent / "golden" / "cell.json").read_text())


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def case_inputs(order_n, precision, seed):
    """Inputs of one golden case (as tests/golden/make_cell_golden.py draws them)."""
    dtype = np.float64 if precision == "double" else np.float32
    side = 2 * order_n + 2
    rng = np.random.default_rng(seed)
    u_loc = rng.uniform(-1, 1, (side, side, side)).astype(dtype)
    coeffs = rng.uniform(-1, 1, (side, side, side)).astype(dtype)
    batch = rng.uniform(-1, 1, (3, side, side, side)).astype(dtype)
    return u_loc, coeffs, batch


@pytest.mark.parametrize("row", CELL["cases"], ids=lambda r: f"N{r['order_n']}-{r['precision']}")
def test_per_cell_api_bit_identical_to_reference(row):
    n = row["order_n"]
    u_loc, coeffs, batch = case_inputs(n, row["precision"], row["seed"])
    interp = hb.build_interp_operator(n)
    d_ops = tuple(hb.build_deriv_operator(n, h) for h in row["spacings"])
    q, dt = hb.default_stages(n), row["dt"]
    cc = hb.CellCoeffs(n, coeffs)
    got = {
        "reconstruct": hb.reconstruct_cell((interp,) * 3, u_loc).data,
        "advect": hb.advect_time_derivative(d_ops, coeffs),
        "advect_batch": hb.advect_time_derivative(d_ops, batch),
        "horner": hb.taylor_evolve_horner(cc, d_ops, hb.TaylorParams(q, dt), step=dt / 2).data,
        "horner_q5": hb.taylor_evolve_horner(cc, d_ops, hb.TaylorParams(5, dt), step=0.3 * dt).data,
        "space_time": space_time_tensor(cc, d_ops, hb.TaylorParams(q, dt)),
        "recursion_half": hb.taylor_evolve_recursion(cc, d_ops, hb.TaylorParams(q, dt), 0.5).data,
        "recursion_03": hb.taylor_evolve_recursion(cc, d_ops, hb.TaylorParams(q + 2, dt), 0.3).data,
    }
    for key, value in got.items():
        assert value.dtype == u_loc.dtype, key
        assert sha(value) == row[key], key
    assert hb.verify_space_time_identity(cc, d_ops, hb.TaylorParams(q, dt)) == row["identity"]
    assert hb.verify_space_time_identity(cc, d_ops, hb.TaylorParams(3, dt)) == row["identity_short"]


# ---- the reference's per-cell tests (pkg/tests/test_kernels.py), restated -------------------

def _ops(order_n, spacings=(1.0, 1.0, 1.0)):
    interp = hb.build_interp_operator(order_n)
    return (interp,) * 3, tuple(hb.build_deriv_operator(order_n, h) for h in spacings)


def _endpoint_dofs(order_n):
    """E[(e, k)][j]: the k-th scaled derivative (Taylor coefficient) of z^j at z_e = -/+ 1/2,
    in exact rationals (independent of the package's H)."""
    from fractions import Fraction
    side = 2 * order_n + 2
    e = np.zeros((side, side), dtype=object)
    for ei, z in enumerate((Fraction(-1, 2), Fraction(1, 2))):
        for k in range(order_n + 1):
            for j in range(k, side):
                e[ei * (order_n + 1) + k, j] = math.comb(j, k) * z ** (j - k)
    return e


def _vertex_dofs(coeffs, order_n):
    """8-vertex DOF tensor of a coefficient tensor, contracted in long double, rounded once."""
    e = _endpoint_dofs(order_n).astype(np.longdouble)
    return np.einsum("ai,bj,ck,ijk->abc", e, e, e, coeffs.astype(np.longdouble)).astype(np.float64)


def _shifted(coeffs, shifts):
    """Coefficients of p(z1 + a1, z2 + a2, z3 + a3) (binomial expansion in long double)."""
    side = coeffs.shape[0]
    mats = []
    for a in shifts:
        s = np.zeros((side, side), dtype=np.longdouble)
        for j in range(side):
            for m in range(j + 1):
                s[m, j] = math.comb(j, m) * np.longdouble(a) ** (j - m)
        mats.append(s)
    return np.einsum("ai,bj,ck,ijk->abc", mats[2], mats[1], mats[0], coeffs.astype(np.longdouble)).astype(np.float64)


def _ulps(a, b):
    scale = max(np.abs(a).max(), np.abs(b).max())
    return 0.0 if scale == 0 else float(np.abs(a - b).max() / np.spacing(scale))


def _rel(got, want):
    scale = np.abs(want).max()
    return float(np.abs(got - want).max() / (scale if scale > 0 else 1.0))


def _unit(order_n, index, value=1.0):
    side = 2 * order_n + 2
    d = np.zeros((side,) * 3)
    d[index] = value
    return hb.CellCoeffs(order_n, d)


def test_taylor_params_and_validation():
    with pytest.raises(ValueError):
        hb.TaylorParams(stages_q=0, dt=0.1)
    with pytest.raises(ValueError):
        hb.TaylorParams(stages_q=3, dt=0.0)
    assert hb.TaylorParams(4, 0.5).half_dt == 0.25
    _, d_ops = _ops(1)
    with pytest.raises(ValueError):
        hb.taylor_evolve_horner(_unit(1, (0, 0, 0)), d_ops, hb.TaylorParams(9, 0.5), step=0.0)
    for bad in (0.0, -0.5, 1.5):
        with pytest.raises(ValueError):
            hb.taylor_evolve_recursion(_unit(1, (0, 0, 0)), d_ops, hb.TaylorParams(9, 0.5), tau=bad)
    with pytest.raises(ValueError):
        hb.CellCoeffs(1, np.zeros((3, 3, 3)))


def test_reconstruct_constant_and_two_value_cells():
    h_ops, _ = _ops(1)
    u = np.zeros((4, 4, 4))
    u[::2, ::2, ::2] = 7.5  # the value DOF of all 8 vertices
    want = np.zeros((4, 4, 4))
    want[0, 0, 0] = 7.5
    assert np.allclose(hb.reconstruct_cell(h_ops, u).data, want, rtol=0, atol=1e-14)
    h0, _ = _ops(0)
    u = np.empty((2, 2, 2))
    u[..., 0], u[..., 1] = 1.25, -0.75
    out = hb.reconstruct_cell(h0, u).data
    assert out[0, 0, 0] == 0.25 and out[0, 0, 1] == -2.0 and np.count_nonzero(out) == 2


@pytest.mark.parametrize("order_n", [1, 2, 3, 5])
def test_reconstruction_recovers_random_polynomials(order_n):
    h_ops, _ = _ops(order_n)
    side = 2 * order_n + 2
    rng = np.random.default_rng(order_n)
    for _ in range(10):
        coeffs = rng.uniform(-1, 1, (side,) * 3)
        u = _vertex_dofs(coeffs, order_n)
        out = hb.reconstruct_cell(h_ops, u).data
        tol = 1e-11 if order_n <= 3 else 1e-8  # H's condition number grows with N
        assert np.abs(out - coeffs).max() / max(np.abs(coeffs).max(), np.abs(u).max()) <= tol


def test_advect_constant_and_linear_terms():
    _, d_ops = _ops(1)
    assert np.array_equal(hb.advect_time_derivative(d_ops, _unit(1, (0, 0, 0)).data), np.zeros((4, 4, 4)))
    assert np.array_equal(hb.advect_time_derivative(d_ops, _unit(1, (0, 0, 1)).data), _unit(1, (0, 0, 0)).data)
    w = _unit(1, (0, 0, 1)).data + _unit(1, (0, 1, 0)).data + _unit(1, (1, 0, 0)).data
    assert np.array_equal(hb.advect_time_derivative(d_ops, w), 3.0 * _unit(1, (0, 0, 0)).data)


def test_horner_constant_and_linear_shift_exact():
    _, d2 = _ops(2)
    c = _unit(2, (0, 0, 0), 4.2)
    assert np.array_equal(hb.taylor_evolve_horner(c, d2, hb.TaylorParams(15, 0.8), step=0.4).data, c.data)
    _, d1 = _ops(1)
    lin = _unit(1, (0, 0, 1))
    out = hb.taylor_evolve_horner(lin, d1, hb.TaylorParams(9, 0.6), step=0.3)
    assert np.array_equal(out.data, lin.data + 0.3 * _unit(1, (0, 0, 0)).data)


@pytest.mark.parametrize("order_n", [1, 2, 3, 5])
def test_horner_extra_stages_are_noops(order_n):
    side = 2 * order_n + 2
    q = hb.default_stages(order_n)
    _, d_ops = _ops(order_n, (0.1, 0.1, 0.1))
    c = hb.CellCoeffs(order_n, np.random.default_rng(3).uniform(-1, 1, (side,) * 3))
    a = hb.taylor_evolve_horner(c, d_ops, hb.TaylorParams(q, 0.09), step=0.045)
    b = hb.taylor_evolve_horner(c, d_ops, hb.TaylorParams(q + 3, 0.09), step=0.045)
    assert np.array_equal(a.data, b.data)


def test_recursion_constant_and_linear():
    _, d_ops = _ops(1)
    c = _unit(1, (0, 0, 0), -2.0)
    for tau in (0.25, 0.5, 1.0):
        assert np.array_equal(hb.taylor_evolve_recursion(c, d_ops, hb.TaylorParams(9, 0.5), tau).data, c.data)
    lin = _unit(1, (0, 0, 1))
    out = hb.taylor_evolve_recursion(lin, d_ops, hb.TaylorParams(9, 0.6), tau=0.5)
    assert np.array_equal(out.data, lin.data + 0.3 * _unit(1, (0, 0, 0)).data)


@pytest.mark.parametrize("order_n", [1, 2, 3])
def test_horner_and_recursion_agree_within_8_ulp(order_n):
    """SPEC acceptance 5 (pkg/tests/test_kernels.py horner/recursion agreement)."""
    side = 2 * order_n + 2
    spacings = (0.1, 0.125, 0.1)
    _, d_ops = _ops(order_n, spacings)
    dt = 0.9 * min(spacings)
    params = hb.TaylorParams(hb.default_stages(order_n), dt)
    rng = np.random.default_rng(2024)
    worst = 0.0
    for _ in range(100):
        c = hb.CellCoeffs(order_n, rng.uniform(-1, 1, (side,) * 3))
        a = hb.taylor_evolve_horner(c, d_ops, params, step=dt / 2).data
        b = hb.taylor_evolve_recursion(c, d_ops, params, tau=0.5).data
        worst = max(worst, _ulps(a, b))
    assert worst <= 8


@pytest.mark.parametrize("order_n", [1, 2, 3])
def test_exact_local_evolution_matches_the_shifted_polynomial(order_n):
    """q = 3(2N+1) makes the local evolution exact (the identity the separable fast path uses,
    pkg/tests/test_kernels.py:184-199)."""
    side = 2 * order_n + 2
    spacings = (0.2, 0.25, 0.5)
    _, d_ops = _ops(order_n, spacings)
    dt = 0.9 * min(spacings)
    params = hb.TaylorParams(hb.default_stages(order_n), dt)
    rng = np.random.default_rng(11)
    for _ in range(10):
        data = rng.uniform(-1, 1, (side,) * 3)
        out = hb.taylor_evolve_horner(hb.CellCoeffs(order_n, data), d_ops, params, step=dt / 2)
        assert _rel(out.data, _shifted(data, tuple(dt / 2 / h for h in spacings))) <= 1e-12


def test_evolution_linearity():
    _, d_ops = _ops(2, (0.1, 0.1, 0.1))
    params = hb.TaylorParams(15, 0.09)
    rng = np.random.default_rng(5)
    u, v = rng.uniform(-1, 1, (2, 6, 6, 6))
    combo = hb.taylor_evolve_horner(hb.CellCoeffs(2, 0.7 * u - 1.3 * v), d_ops, params, 0.045).data
    sep = 0.7 * hb.taylor_evolve_horner(hb.CellCoeffs(2, u), d_ops, params, 0.045).data \
        - 1.3 * hb.taylor_evolve_horner(hb.CellCoeffs(2, v), d_ops, params, 0.045).data
    assert _rel(combo, sep) <= 1e-13


@pytest.mark.parametrize("order_n", [1, 2, 3])
def test_space_time_identity(order_n):
    """SPEC acceptance 4: the space-time tensor satisfies the advection equation
    as a polynomial identity to 1e-12 of the data scale; exactly 0 for zero / linear data."""
    _, d_ops = _ops(order_n)
    q = hb.default_stages(order_n)
    assert hb.verify_space_time_identity(hb.CellCoeffs.zeros(order_n), d_ops, hb.TaylorParams(q, 0.5)) == 0.0
    assert hb.verify_space_time_identity(_unit(order_n, (0, 0, 1)), d_ops, hb.TaylorParams(q, 0.5)) == 0.0
    side = 2 * order_n + 2
    rng = np.random.default_rng(order_n + 40)
    for _ in range(20):
        c = hb.CellCoeffs(order_n, rng.uniform(-1, 1, (side,) * 3))
        assert hb.verify_space_time_identity(c, d_ops, hb.TaylorParams(q, 0.2)) <= 1e-12 * np.abs(c.data).max()


def test_space_time_top_slab_closes():
    _, d_ops = _ops(1, (0.25, 0.25, 0.25))
    c = hb.CellCoeffs(1, np.random.default_rng(7).uniform(-1, 1, (4, 4, 4)))
    st = space_time_tensor(c, d_ops, hb.TaylorParams(hb.default_stages(1) + 1, 0.2))
    assert st.shape == (11, 4, 4, 4) and np.array_equal(st[-1], np.zeros_like(st[-1]))


# ---- DofField's coherent host mirror on a device-resident field ------------------------------

def test_reference_style_writes_through_data_reach_the_kernels():
    """pkg/tests/test_field.py writes `field.data[idx] = v` and reads `field.data` again; the same
    pattern on a device field must reach the next half step (the round-1 `.data` was a copy)."""
    grid = hb.GridSpec((6, 5, 4))
    n = 2
    cfg = hb.StepConfig(variant="literal")
    ops = hb.OperatorSet.for_grid(grid, n)
    a = hb.DofField.zeros(grid, n)
    a.data[2, 1, 3, 0, 0, 0] = 7.0            # write through the mirror ...
    a.values[0, 4, 1] = -2.5                  # ... and through a view of it
    a.data.ravel()[5] = 1.5
    host = np.zeros(a.data.shape)
    host[2, 1, 3, 0, 0, 0], host[0, 4, 1, 0, 0, 0] = 7.0, -2.5
    host.ravel()[5] = 1.5
    assert np.array_equal(a.data, host)
    b = hb.DofField(grid, n, host.copy())      # adopted ndarray, uploaded on first use
    out_a = hb.DofField.zeros(grid.with_parity("dual"), n)
    out_b = hb.DofField.zeros(grid.with_parity("dual"), n)
    hb.half_step(a, out_a, cfg, ops)
    hb.half_step(b, out_b, cfg, ops)
    assert torch.equal(out_a.tensor, out_b.tensor) and np.count_nonzero(out_a.data) > 0
    mirror = out_a.data
    hb.half_step(out_a, a, cfg, ops)           # device write; re-reading .data refreshes in place
    assert a.data is a.data and np.array_equal(a.data, a.tensor.cpu().numpy())
    assert mirror is out_a.data


def test_gather_and_scatter_on_a_device_field():
    grid = hb.GridSpec((3, 4, 2))
    f = hb.DofField.zeros(grid, 1)
    f.tensor.copy_(torch.arange(f.tensor.numel(), dtype=torch.float64, device="cuda").view_as(f.tensor))
    host = f.tensor.cpu().numpy()
    out = hb.gather_cell(f, (2, 3, 1))         # wraps along x1, x2 and x3
    for a3 in (0, 1):
        for a2 in (0, 1):
            for a1 in (0, 1):
                blk = host[(1 + a3) % 2, (3 + a2) % 4, (2 + a1) % 3]
                assert np.array_equal(out[2 * a3:2 * a3 + 2, 2 * a2:2 * a2 + 2, 2 * a1:2 * a1 + 2], blk)
    c = hb.CellCoeffs.zeros(1)
    c.data[:] = 9.0
    hb.scatter_dofs(c, f, (4, -1, 3))          # node (1, 3, 1) after the wrap; only n^3 entries land
    want = host.copy()
    want[1, 3, 1] = 9.0
    assert np.array_equal(f.tensor.cpu().numpy(), want)
