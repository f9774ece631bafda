#!/bin/bash
# One GPU session (gpurun): build check, gpu tests, smoke, mode-gap table, bench at N = 1.
# usage: tools/gpu_session.sh [TAG]   (outputs under gpurun_out/TAG_*)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
tag=${1:-s}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/${tag}_nvsmi.txt 2>&1
free -g >> gpurun_out/${tag}_nvsmi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rP --durations=30 > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 600 python tools/mode_gap.py > gpurun_out/${tag}_mode_gap.txt 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "rc=$?" >> gpurun_out/${tag}_bench.err
echo done
