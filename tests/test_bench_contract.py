"""bench.py's driver contract, end to end (the driver runs it at N = 1 and under torchrun at
N = 2, 4, 8).  GPU tests run small grids; two ranks share the one GPU over gloo, the
configuration the driver's first multi-GPU run would exercise with NCCL."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _json_lines(out: str):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def _torchrun(n, *args, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", str(ROOT / "bench.py"), "--gpus", str(n),
           *args]
    env = dict(os.environ, NCCL_DEBUG="INFO")
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)


def test_reference_arm_under_torchrun_prints_one_line():
    """--impl reference: rank 0 alone times the CPU restatement and prints one line; the other
    rank exits 0 without work."""
    out = _torchrun(2, "--impl", "reference", "--steps", "1", "--warmup", "1", "--cpu-seconds", "1", timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = _json_lines(out.stdout)
    assert len(lines) == 1
    line = lines[0]
    assert line["impl"] == "reference" and line["value"] > 0 and line["n_gpus"] == 2
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_bench_single_gpu_line_has_every_contract_key():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--cells", "64", "--steps", "3", "--warmup", "3",
                          "--no-extras", "--cpu-seconds", "1"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    (line,) = _json_lines(out.stdout)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["finite"]
    assert line["roofline"]["frac"] > 0 and line["e2e"]["value"] and line["e2e"]["h2d_bytes_per_step"] > 0
    assert line["gpu_launches"] == 2 * 3


@pytest.mark.gpu
@pytest.mark.parametrize("halo,mode", [("p2p", "fused"), ("nccl", "fused"), ("auto", "two_pass")])
def test_bench_two_ranks_under_torchrun(halo, mode):
    """The N > 1 path the driver's scaling run takes (slab decomposition, halo exchange,
    max-over-ranks timing, per-rank e2e streaming with halo planes), on one GPU over gloo."""
    out = _torchrun(2, "--backend", "gloo", "--cells", "64", "--steps", "2", "--warmup", "3", "--no-extras",
                    "--halo", halo, "--mode", mode)
    assert out.returncode == 0, out.stderr[-3000:]
    (line,) = _json_lines(out.stdout)
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["finite"] and line["scaling"] == "weak"
    assert line["config"]["global_cells"] == [64, 64, 128]
    assert line["config"]["halo"].startswith("p2p" if halo == "p2p" else "nccl")
    assert line["roofline"]["frac"] > 0
    assert "e2e" in line and (line["e2e"]["value"] or line["e2e"].get("error"))


@pytest.mark.gpu
def test_bench_strong_scaling_under_torchrun():
    """`--strong M` (configs[4]'s 1024^3 split over the ranks): one global grid divided into x3
    slabs, reported as strong scaling with the global cell count; exercised small on one GPU."""
    out = _torchrun(2, "--backend", "gloo", "--strong", "48", "--steps", "2", "--warmup", "3", "--no-extras",
                    "--no-e2e", "--halo", "auto")
    assert out.returncode == 0, out.stderr[-3000:]
    (line,) = _json_lines(out.stdout)
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["finite"] and line["scaling"] == "strong"
    assert line["config"]["global_cells"] == [48, 48, 48]
