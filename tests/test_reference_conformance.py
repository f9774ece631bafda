"""The reference's own test files run against this package through an import alias.

`hermite3d` (and its submodules field / kernels / operators / pipeline / problems) is aliased
to `paper_1609_09841_b200` by a shim package on PYTHONPATH, and pytest collects the
reference's unmodified pkg/tests/*.py (with its own conftest.py) in a subprocess.

* test_field.py and test_operators.py exercise only host-side containers and operators, so
  they run here on CPU (DofField is a host container without a CUDA device) -- every test must
  pass.
* test_kernels.py exercises the per-cell kernels, which run on the GPU; it runs when a GPU and
  the reference tree are both present (the GPU box has no /root/reference: there the same
  assertions run as tests/test_gpu_cell_api.py, pinned by golden digests).

Skipped when /root/reference is absent.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

REF_TESTS = Path("/root/reference/pkg/tests")
ROOT = Path(__file__).resolve().parent.parent

SHIM = '''import sys
import paper_1609_09841_b200 as _pkg
from paper_1609_09841_b200 import field, kernels, operators, pipeline, problems
sys.modules["hermite3d"] = _pkg
for _name, _mod in (("field", field), ("kernels", kernels), ("operators", operators),
                    ("pipeline", pipeline), ("problems", problems)):
    sys.modules["hermite3d." + _name] = _mod
'''


def _run_reference_tests(tmp_path, files):
    shim = tmp_path / "shim" / "hermite3d"
    shim.mkdir(parents=True)
    (shim / "__init__.py").write_text(SHIM)
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1",
               PYTHONPATH=os.pathsep.join([str(shim.parent), str(ROOT)]))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", str(tmp_path),
           *[str(REF_TESTS / f) for f in files]]
    return subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=tmp_path, timeout=900)


@pytest.mark.skipif(not REF_TESTS.exists(), reason="reference tree not present (GPU box)")
def test_reference_field_and_operator_tests_pass(tmp_path):
    out = _run_reference_tests(tmp_path, ["test_field.py", "test_operators.py"])
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert " passed" in out.stdout and "failed" not in out.stdout


@pytest.mark.gpu
@pytest.mark.skipif(not REF_TESTS.exists(), reason="reference tree not present (GPU box)")
def test_reference_kernel_tests_pass(tmp_path):
    assert torch.cuda.is_available()
    out = _run_reference_tests(tmp_path, ["test_kernels.py"])
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
