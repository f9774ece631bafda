#!/bin/bash
# ncu --set full (with SASS source) of the m=3 fused kernels at 256^3: the lock-step product kernel
# and a measurement-build variant.   usage: tools/gpu_prof_m3.sh TAG "CFG..."
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
tag=${1:-pm3}; cfgs=${2:-""}
mkdir -p gpurun_out
make -C paper_1609_09841_b200/csrc measure -j16 > gpurun_out/${tag}_make.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sep_fused -s 2 -c 1 -o gpurun_out/${tag}_base -f python tools/time_fused.py 3 256 fused 1 > gpurun_out/${tag}_prof.log 2>&1
for c in $cfgs; do
  H3_LIB=build/libh3b200_measure.so H3_DMMA_CFG=$c timeout 600 ncu --set full --clock-control none --import-source on -k regex:sep_fused -s 2 -c 1 -o gpurun_out/${tag}_v$c -f python tools/time_fused.py 3 256 fused 1 >> gpurun_out/${tag}_prof.log 2>&1
done
echo done
