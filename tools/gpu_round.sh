#!/bin/bash
# One GPU session: gpu tests, smoke, bench (N=1, extras on), ncu launch list + full captures
# of the fused (512^3 m=3, the headline launch) and the two-kernel / m=5 kernels.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extras > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sep_fused -s 2 -c 1 -o gpurun_out/prof_fused -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extras > gpurun_out/prof.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"recon_dmma3|sep_evolve" -s 4 -c 2 -o gpurun_out/prof_two3 -f python tools/time_fused.py 3 256 two_pass 1 >> gpurun_out/prof.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dmma_cp|sep_evolve" -s 6 -c 3 -o gpurun_out/prof_m5 -f python tools/time_fused.py 5 128 two_pass 1 >> gpurun_out/prof.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dmma_cp" -s 2 -c 1 -o gpurun_out/prof_m5f -f python tools/time_fused.py 5 128 fused 1 >> gpurun_out/prof.log 2>&1
echo done
