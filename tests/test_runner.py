"""runner mirror: IC expansion and run summaries against golden vectors from the reference's
own runner (tests/golden/make_runner_golden.py), artifacts, and validation."""

import csv
import json
import math
from pathlib import Path

import pytest

import paper_1609_09841_b200 as hb
from paper_1609_09841_b200 import runner

GOLD = json.loads((Path(__file__).parent / "golden" / "runner.json").read_text())
ICS = {
    "plane_wave": [{"kind": "plane_wave", "wavenumber": 2, "amplitude": 0.5, "phase": 0.25}],
    "random_modes": [{"kind": "random_modes", "terms": 3, "max_wavenumber": 3}],
    "separable": [{"kind": "separable", "factors": [{"kind": "fourier", "wavenumber": 1},
                                                    {"kind": "constant", "value": 2.0},
                                                    {"kind": "fourier", "phase": 0.5}]}],
}


@pytest.mark.parametrize("name", sorted(ICS))
def test_build_ic_matches_reference(name):
    ic = runner.build_ic(runner.RunConfig(order_n=3, cells=(8, 8, 8), steps=1, ic=tuple(ICS[name]), seed=7))
    want = GOLD["ics"][name]
    assert len(ic.terms) == len(want)
    for term, wterm in zip(ic.terms, want):
        for f, (cls, attrs) in zip(term, wterm):
            assert type(f).__name__ == cls
            for k, v in attrs.items():
                assert getattr(f, k) == v, (name, k)


def test_run_config_validation():
    with pytest.raises(runner.ConfigError, match="steps/final_time"):
        runner.RunConfig(order_n=3, cells=8)
    with pytest.raises(runner.ConfigError, match="order_n"):
        runner.RunConfig(order_n=6, cells=8, steps=1)
    with pytest.raises(runner.ConfigError, match="cells"):
        runner.RunConfig(order_n=1, cells=(8, 0, 8), steps=1)
    with pytest.raises(runner.ConfigError, match="mode"):
        runner.RunConfig(order_n=1, cells=8, steps=1, mode="bogus")
    with pytest.raises(runner.ConfigError, match="levels"):
        runner.execute_converge(runner.RunConfig(order_n=1, cells=8, final_time=0.1), [8])
    assert runner.RunConfig(order_n=2, cells=5, steps=1).cells == (5, 5, 5)


@pytest.mark.gpu
@pytest.mark.parametrize("row", GOLD["runs"], ids=lambda r: str(r["config"]))
def test_execute_run_matches_reference(row, tmp_path):
    kw = dict(row["config"])
    if "ic" in kw:
        kw["ic"] = tuple(kw["ic"])
    s = runner.execute_run(runner.RunConfig(out_dir=str(tmp_path), variant="literal", **kw))
    want = row["summary"]
    assert (s["steps"], s["dt"], s["final_time"]) == (want["steps"], want["dt"], want["final_time"])
    assert s["l_inf"] == pytest.approx(want["l_inf"], rel=1e-9)
    assert s["l2"] == pytest.approx(want["l2"], rel=1e-9)
    art = s["artifacts"]
    with open(art["errors_csv"]) as fh:
        rows = list(csv.reader(fh))
    assert rows[0] == ["step", "time", "l_inf", "l2"] and len(rows) == s["steps"] + 2
    assert float(rows[-1][2]) == s["l_inf"]
    rep = json.loads(Path(art["perf_json"]).read_text())
    assert [r["kernel"] for r in rep["runs"]][-1] == "solution"
    field, t = hb.read_snapshot(Path(art["snapshot_bin"]).with_suffix(""))
    assert t == s["final_time"] and field.grid.cells_per_axis == runner.RunConfig(steps=1, **{
        k: v for k, v in kw.items() if k not in ("steps", "final_time")}).cells


@pytest.mark.gpu
def test_execute_converge_matches_reference(tmp_path):
    g = GOLD["converge"]
    c = runner.execute_converge(runner.RunConfig(order_n=g["order_n"], cells=8, final_time=g["final_time"],
                                                 out_dir=str(tmp_path), variant="literal"), g["levels"])
    for got, want in zip(c["rows"], g["rows"]):
        assert got["cells"] == want["cells"] and got["h"] == want["h"]
        assert got["l_inf"] == pytest.approx(want["l_inf"], rel=1e-9)
        if not math.isnan(want["order_linf"]):
            assert got["order_linf"] == pytest.approx(want["order_linf"], abs=1e-6)
    assert Path(c["artifacts"]["converge_csv"]).exists()


@pytest.mark.gpu
def test_execute_run_separable_default_close_to_reference(tmp_path):
    row = GOLD["runs"][0]
    s = runner.execute_run(runner.RunConfig(out_dir=str(tmp_path), **row["config"]), write_artifacts=False)
    assert s["l_inf"] == pytest.approx(row["summary"]["l_inf"], rel=1e-2)


@pytest.mark.gpu
def test_resume_from_snapshot_continues_the_run(tmp_path):
    """10 steps == 4 steps, snapshot, resume for 6 more (bit-identical field, same errors)."""
    base = dict(order_n=3, cells=(12, 10, 8), variant="literal")
    full = runner.execute_run(runner.RunConfig(steps=10, out_dir=str(tmp_path / "full"), **base))
    first = runner.execute_run(runner.RunConfig(steps=4, out_dir=str(tmp_path / "a"), **base))
    snap = str(Path(first["artifacts"]["snapshot_bin"]).with_suffix(""))
    second = runner.execute_run(runner.RunConfig(steps=6, out_dir=str(tmp_path / "b"), resume=snap, **base))
    assert second["final_time"] == pytest.approx(full["final_time"], rel=1e-15)
    assert second["l_inf"] == pytest.approx(full["l_inf"], rel=1e-12)
    a = Path(full["artifacts"]["snapshot_bin"]).read_bytes()
    b = Path(second["artifacts"]["snapshot_bin"]).read_bytes()
    assert a == b
    with pytest.raises(runner.ConfigError, match="resume"):
        runner.execute_run(runner.RunConfig(steps=1, out_dir=str(tmp_path / "c"), resume=snap,
                                            order_n=3, cells=(12, 10, 9)))


@pytest.mark.gpu
@pytest.mark.filterwarnings("ignore:.*launch latency:RuntimeWarning")  # deliberately tiny grid
def test_execute_bench_profiles_and_solution_rows(tmp_path):
    """execute_bench (reference runner.py:239-269): per mode the kernel profiles then one
    end-to-end "solution" row; perf.json / perf.csv written; counts from the reference model."""
    cfg = runner.RunConfig(order_n=3, cells=(24, 20, 16), steps=3, out_dir=str(tmp_path), variant="separable")
    out = runner.execute_bench(cfg, repetitions=3, modes=["fused", "two_pass"])
    kernels = [r["kernel"] for r in out["runs"]]
    assert kernels == ["monolithic", "solution", "reconstruction", "evolution", "solution"]
    assert all(r["seconds"] > 0 for r in out["runs"])
    grid = hb.GridSpec((24, 20, 16))
    f, b = hb.perf.model_counts("monolithic", 3, grid, cfg.step_config())
    assert out["runs"][1]["flops"] == f * 2 * 3 and out["runs"][1]["bytes"] == b * 2 * 3
    assert (tmp_path / "perf.json").exists() and (tmp_path / "perf.csv").exists()


def test_execute_autotune_validates_candidates(tmp_path):
    cfg = runner.RunConfig(order_n=1, cells=(8, 8, 8), steps=1, out_dir=str(tmp_path))
    with pytest.raises(runner.ConfigError, match="candidates"):
        runner.execute_autotune(cfg, [2])


@pytest.mark.gpu
def test_execute_autotune_table_and_selection(tmp_path):
    """Reference runner.py:272-327 semantics: skipped rows for tiles wider than M1, one winner
    (argmin of the median time, ties to the smaller tile), autotune.csv written."""
    cfg = runner.RunConfig(order_n=3, cells=(12, 10, 8), steps=1, out_dir=str(tmp_path), variant="separable")
    out = runner.execute_autotune(cfg, [2, 4, 64], repetitions=3)
    status = {r["tile_x1"]: r["status"] for r in out["rows"]}
    assert status[64].startswith("skipped") and list(status.values()).count("winner") == 1
    assert status[out["best_tile_x1"]] == "winner" and out["best_tile_x1"] in (2, 4)
    assert (tmp_path / "autotune.csv").read_text().splitlines()[0] == "tile_x1,seconds,bytes_modeled,status"
    with pytest.raises(runner.ConfigError, match="no candidate"):
        runner.execute_autotune(cfg, [64, 128])
