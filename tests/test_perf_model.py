"""perf module: the reference's analytic model reproduced exactly (golden vectors from the
reference, tests/golden/make_perf_golden.py), report schema, B200 peaks; GPU profiling."""

import json
from pathlib import Path

import pytest

import paper_1609_09841_b200 as hb
from paper_1609_09841_b200 import perf

GOLD = json.loads((Path(__file__).parent / "golden" / "perf_model.json").read_text())


def test_model_counts_match_reference_golden():
    for row in GOLD["model_counts"]:
        cfg = hb.StepConfig(mode=row["mode"], tile_x1=row["tile_x1"], precision=row["precision"])
        got = perf.model_counts(row["kernel"], row["order_n"], hb.GridSpec(tuple(row["cells"])), cfg)
        assert got == (row["flops"], row["bytes"]), row


def test_roofline_ceiling_and_default_peaks_match_reference():
    peaks = perf.DevicePeaks()
    assert [peaks.peak_bandwidth, peaks.peak_gflops] == GOLD["default_peaks"]
    for i, c in GOLD["ceilings_default_peaks"]:
        assert perf.roofline_ceiling(i, peaks) == c
    with pytest.raises(ValueError):
        perf.roofline_ceiling(-1.0, peaks)
    with pytest.raises(ValueError):
        perf.DevicePeaks(0.0, 1.0)


def test_b200_peaks_and_algorithmic_bytes(tmp_path):
    f = tmp_path / "MEASURED_PEAKS.json"
    f.write_text(json.dumps({"hbm_gbs": 6551.4}))
    p = perf.DevicePeaks.b200(f)
    assert p.peak_bandwidth == 6551.4 and p.peak_gflops == perf.B200_FP64_GFLOPS
    assert perf.DevicePeaks.b200(tmp_path / "missing.json").peak_bandwidth == perf.B200_FALLBACK_BANDWIDTH
    g = hb.GridSpec((512, 512, 512))
    assert perf.algorithmic_bytes("monolithic", 3, g) == 16 * 64 * 512 ** 3  # 137.4 GB
    assert perf.algorithmic_bytes("reconstruction", 3, g) + perf.algorithmic_bytes("evolution", 3, g) \
        == 16 * (64 + 512) * 512 ** 3
    with pytest.raises(ValueError):
        perf.algorithmic_bytes("bogus", 3, g)


def test_report_dict_schema():
    prof = perf._profile("monolithic", 3, "fused", 2, 10 ** 12, 10 ** 9, 0.5, perf.DevicePeaks.b200(), 10 ** 9)
    rep = perf.report_dict([prof], perf.DevicePeaks.b200())
    assert set(perf.REPORT_COLUMNS) <= set(rep["runs"][0])
    assert rep["device"]["bw"] > 0 and "warnings" not in rep


@pytest.mark.gpu
@pytest.mark.parametrize("mode,order_n", [("fused", 3), ("two_pass", 3), ("fused", 5), ("two_pass", 1)])
def test_profile_run_on_gpu(mode, order_n):
    cfg = hb.StepConfig(mode=mode, variant="separable")
    profs = perf.profile_run(cfg, hb.GridSpec((48, 40, 32)), order_n)
    assert [p.kernel for p in profs] == (["monolithic"] if mode == "fused" else ["reconstruction", "evolution"])
    for p in profs:
        assert p.wall_time > 0 and 0 < p.hbm_fraction < 1.5
    rep = perf.report_dict(profs, perf.DevicePeaks.b200())
    assert len(rep["runs"]) == len(profs)
    with pytest.raises(ValueError):
        perf.profile_run(cfg, hb.GridSpec((8, 8, 8)), order_n, repetitions=2)
