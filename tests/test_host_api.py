"""CPU tests of the host-side mirror of the reference API and of the C ABI surface.

None of these launch a kernel: they cover argument validation, operator
precompute, the drop-in names, and that libh3b200.so loads and exports every
symbol include/h3b200.h declares.
"""

import ctypes
import math
import re
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

import paper_1609_09841_b200 as hb
from paper_1609_09841_b200 import _native, pipeline
from oracle import refmodel as rm
from conftest import GOLDEN, ROOT


def test_gridspec_spacings_coords_and_validation():
    g = hb.GridSpec((4, 5, 8), (1.0, 2.0, 4.0))
    assert g.spacings == (0.25, 0.4, 0.5)
    assert np.allclose(g.axis_coords(1), [0, 0.25, 0.5, 0.75])
    assert np.allclose(g.with_parity("dual").axis_coords(2), (np.arange(5) + 0.5) * 0.4)
    assert g.wrap(3, -1) == 7 and g.num_cells == 160
    for bad in [dict(cells_per_axis=(0, 1, 1)), dict(cells_per_axis=(1, 1)),
                dict(cells_per_axis=(1, 1, 1), domain_lengths=(1, 0, 1)),
                dict(cells_per_axis=(1, 1, 1), parity="odd")]:
        with pytest.raises(ValueError):
            hb.GridSpec(**bad)


def test_stepconfig_validation_and_stages():
    assert hb.StepConfig().stages(3) == 21 and hb.StepConfig(stages_q=5).stages(3) == 5
    for bad in [dict(mode="x"), dict(tile_x1=0), dict(cfl=0), dict(cfl=1.5), dict(stages_q=0),
                dict(precision="half"), dict(variant="fast")]:
        with pytest.raises(ValueError):
            hb.StepConfig(**bad)


def test_select_dt_and_factor_arrays_match_oracle():
    grid = hb.GridSpec((7, 5, 6), (1.0, 2.0, 3.0))
    cfg = hb.StepConfig()
    dt = hb.select_dt(grid, cfg)
    assert dt == rm.select_dt((7, 5, 6), (1.0, 2.0, 3.0))
    ops = hb.OperatorSet.for_grid(grid, 2)
    ours = pipeline._factor_arrays(ops, np.float64, dt / 2, 15)
    theirs = rm.factor_arrays(2, (7, 5, 6), (1.0, 2.0, 3.0), dt / 2, 15)
    for a, b in zip(ours, theirs):
        assert a.dtype == b.dtype and np.array_equal(a, b)


@pytest.mark.parametrize("order_n", range(9))
def test_interp_matrix_inverts_the_endpoint_vandermonde_exactly(order_n):
    """H (built from closed-form Hermite cardinal polynomials) is the exact inverse of the
    reference's defining matrix V[(e,k)][j] = C(j,k) z_e^(j-k), z_e = -/+ 1/2."""
    import math
    from fractions import Fraction
    from paper_1609_09841_b200.operators import interp_matrix_rational
    side, n = 2 * order_n + 2, order_n + 1
    V = [[Fraction(0)] * side for _ in range(side)]
    for e, z in enumerate((Fraction(-1, 2), Fraction(1, 2))):
        for k in range(n):
            for j in range(k, side):
                V[e * n + k][j] = math.comb(j, k) * z ** (j - k)
    H = interp_matrix_rational(order_n)
    for r in range(side):
        for c in range(side):
            assert sum(V[r][j] * H[j][c] for j in range(side)) == (1 if r == c else 0)


@pytest.mark.parametrize("order_n", range(7))
def test_interp_matrix_bit_identical_to_reference(order_n):
    expected = np.array([[float.fromhex(v) for v in row] for row in GOLDEN["interp_matrix_hex"][str(order_n)]])
    m = hb.build_interp_operator(order_n).matrix
    assert np.array_equal(m, expected) and not m.flags.writeable


def test_deriv_operator_entries_and_validation():
    d = hb.build_deriv_operator(1, 0.25)
    expected = np.zeros((4, 4))
    expected[0, 1], expected[1, 2], expected[2, 3] = 4.0, 8.0, 12.0
    assert np.array_equal(d.matrix, expected)
    with pytest.raises(ValueError):
        hb.build_deriv_operator(1, 0.0)
    with pytest.raises(ValueError):
        hb.build_interp_operator(-1)


def test_tile_schedule_matches_reference_traversal():
    grid = hb.GridSpec((7, 3, 2))
    rows = []
    for c3 in range(2):
        for c2 in range(3):
            start = 0
            while start < 7:
                rows.append((c3, c2, start, min(3, 7 - start)))
                start += 3
    assert np.array_equal(hb.tile_schedule(grid, 3), np.array(rows))
    with pytest.raises(ValueError):
        hb.tile_schedule(grid, 8)
    with pytest.raises(ValueError):
        pipeline.resolve_tile_x1("monolithic", 1, 7, 9)


def test_allocation_stats_and_instability_error():
    s = hb.AllocationStats()
    s.allocate("a", 10)
    s.allocate("b", 5)
    s.release("a")
    s.allocate("c", 1)
    assert s.peak_aux_bytes == 15 and s.live_bytes == 6
    e = hb.InstabilityError((1, 2, 3), step=4)
    assert e.node == (1, 2, 3) and "step 4" in str(e)
    assert pipeline._node_of((2 * 5 + 3) * 6 + 4, hb.GridSpec((6, 5, 4))) == (4, 3, 2)


# ----------------------------------------------------------------------------- C ABI

def _header_symbols():
    text = (ROOT / "include" / "h3b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(h3_\w+)\s*\(", text, re.M)))


def test_library_loads_and_exports_every_header_symbol():
    so = _native.lib()
    syms = _header_symbols()
    assert len(syms) >= 14
    for name in syms:
        assert hasattr(so, name), name
        assert name in _native.SIGNATURES, name
    assert _native.version().startswith("h3b200")
    assert so.h3_max_order() == 5 and so.h3_max_stages() >= 33


def test_abi_argument_validation_without_gpu():
    so = _native.lib()
    dummy = ctypes.c_void_p(16)
    arr = np.zeros(64)
    p = arr.ctypes.data_as(ctypes.c_void_p)
    base = [dummy, dummy, 4, 4, 4, 1, p, p, p, p, p, 9, 0, 0, 4, 1, 0, None, None, None]

    def call(**over):
        args = list(base)
        keys = ["src", "dst", "M1", "M2", "M3", "N", "h", "f1", "f2", "f3", "cf", "q", "off",
                "zb", "ze", "per", "var", "st", "fb", "g"]
        for k, v in over.items():
            args[keys.index(k)] = v
        return so.h3_fused_pass(*args)

    assert call(N=6) == -2 and call(N=-1) == -2
    # the stage cap is the literal kernels' (their stage factors live in a fixed parameter block);
    # the separable path only reads cfac[0], so any q >= 3(2N+1) is accepted there
    assert call(q=0) == -3 and call(q=1000, var=1) == -3
    assert call(var=2, q=8) == -3  # separable needs q >= 3(2N+1) = 9
    assert call(var=7) == -4
    assert call(off=1) == -1 and call(src=None) == -1 and call(M1=0) == -1
    assert call(zb=3, ze=2) == -1 and call(ze=5) == -1
    assert so.h3_recon_pass_f32(dummy, dummy, 4, 4, 4, 1, p, 0, 0, 4, 1, 2, None, None) == -4
    assert _native.error_string(-2).startswith("order_n")


def test_halo_abi_argument_validation_without_gpu():
    """h3_fused_pass_halo (the multi-GPU slab entry) rejects bad arguments before touching the
    device: orders without a ghost-pointer kernel, the literal variant, a missing ghost plane
    the slab needs, bad offsets and inexact stage counts; IPC helpers reject null arguments."""
    so = _native.lib()
    dummy = ctypes.c_void_p(16)
    arr = np.zeros(256)
    p = arr.ctypes.data_as(ctypes.c_void_p)
    keys = ["src", "dst", "M1", "M2", "M3", "N", "h", "f1", "f2", "f3", "cf", "q", "off", "zb", "ze",
            "glo", "ghi", "var", "st", "fb", "g"]
    base = dict(src=dummy, dst=dummy, M1=4, M2=4, M3=4, N=3, h=p, f1=p, f2=p, f3=p, cf=p, q=21, off=0,
                zb=0, ze=4, glo=dummy, ghi=dummy, var=2, st=None, fb=None, g=None)

    def call(**over):
        args = dict(base, **over)
        return so.h3_fused_pass_halo(*[args[k] for k in keys])

    assert call(N=2, q=15) == -4 and call(var=1) == -4      # no ghost-pointer kernel / literal
    assert call(ghi=None) == -1                               # off = 0 needs plane M3 of the slab
    assert call(off=-1, glo=None) == -1                       # off = -1 needs plane -1
    assert call(off=1) == -1 and call(src=None) == -1
    assert call(q=20) == -3                                   # separable needs q >= 3(2N+1) = 21
    assert call(zb=3, ze=2) == -1
    h = (ctypes.c_ubyte * 64)()
    off = ctypes.c_int64()
    assert so.h3_ipc_export(None, h, ctypes.byref(off)) == -1
    assert so.h3_ipc_open(None, ctypes.byref(ctypes.c_void_p())) == -1
    assert so.h3_ipc_close(None) == -1


@pytest.mark.parametrize("order_n", [0, 1, 3, 5])
def test_separable_operators_exact(order_n):
    """h3_separable_operators (host math of the fast path) against exact rationals."""
    cells, lengths = (12, 10, 8), (1.0, 1.0, 2.0)
    grid = hb.GridSpec(cells, lengths)
    dt = hb.select_dt(grid, hb.StepConfig())
    q = 3 * (2 * order_n + 1)
    h_mat, f1, f2, f3, cf = pipeline._factor_arrays(hb.OperatorSet.for_grid(grid, order_n), np.float64, dt / 2, q)
    n, s = order_n + 1, 2 * order_n + 2
    A = np.zeros((3, n, s))
    S = np.zeros((3, n, s))
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    assert _native.lib().h3_separable_operators(order_n, ptr(h_mat), ptr(f1), ptr(f2), ptr(f3), ptr(cf), q,
                                                ptr(A), ptr(S)) == 0
    H = rm.interp_matrix_exact(order_n)
    for k, fac in enumerate((f1, f2, f3)):
        r = Fraction(cf[0]) * Fraction(fac[0])
        for m in range(n):
            for c in range(s):
                sx = Fraction(math.comb(c, m)) * r ** (c - m) if c >= m else Fraction(0)
                assert abs(S[k, m, c] - float(sx)) <= 2 ** -52 * abs(float(sx))
                ax = sum(Fraction(math.comb(j, m)) * r ** (j - m) * Fraction(float(H[j][c]))
                         for j in range(m, s))
                scale = max(1.0, max(abs(float(v)) for v in H[c]))
                assert abs(A[k, m, c] - float(ax)) <= 4e-16 * scale * 2 ** order_n


def test_no_oracle_imports_in_product():
    """The product package never imports or links the oracle (test infrastructure)."""
    pkg = ROOT / "paper_1609_09841_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")) + list(pkg.rglob("Makefile")):
        assert "oracle" not in f.read_text().replace("# oracle", ""), f


def test_streaming_chunk_plan_covers_the_grid():
    from paper_1609_09841_b200.streaming import chunk_plan
    for m3 in range(2, 40):
        for chunk in range(1, 45):
            plan = chunk_plan(m3, chunk)
            assert plan[0][0] == 0 and plan[-1][1] == m3
            assert all(a[1] == b[0] for a, b in zip(plan, plan[1:]))
            assert all(z1 - z0 >= 2 for z0, z1 in plan)
    with pytest.raises(ValueError):
        chunk_plan(1, 4)


def test_product_library_has_no_measurement_variants_or_environment_reads():
    """The measurement-only kernel variants (ablations that skip stores or DMMAs, alternative
    tiles, the DFMA A/B kernels) and every H3_* environment switch exist only in the tools build
    (-DH3_MEASURE, build/libh3b200_measure.so): the product objects reference no getenv and the
    product library holds one instantiation of the N=3 monolithic kernel, with no ablation bits."""
    import subprocess
    objs = sorted((ROOT / "build" / "obj").glob("*.o"))
    assert objs
    for o in objs:
        syms = subprocess.run(["nm", str(o)], capture_output=True, text=True).stdout
        assert " U getenv" not in syms, o
    dump = subprocess.run(["cuobjdump", "-symbols", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    fused3 = set(re.findall(r"sep_fused_dmma3_kernelINS_6Dm3CfgI(\w+?)EEEEEv", dump))
    assert len(fused3) == 1, fused3
    # template arguments <TY, WARPS, STAGES, VALIAS, MINB, ABL, ...>: ABL (the 6th) must be 0
    assert re.match(r"Li7ELi16ELi3ELb0ELi1ELi0E", next(iter(fused3))), fused3
