#!/bin/bash
# m=3 warp-specialised fused kernel (h3_dmma3ws.cu): correctness of each variant on ragged grids,
# then interleaved timing against the lock-step kernel at 512^3.   usage: tools/gpu_ws3.sh TAG "VARIANTS"
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
tag=${1:-ws3}; variants=${2:-"101 102 103 104 105 106 107 108"}
mkdir -p gpurun_out
make -C paper_1609_09841_b200/csrc measure -j16 > gpurun_out/${tag}_make.txt 2>&1
for c in $variants; do
  for shape in "40 36 20" "16 14 9" "24 28 12"; do
    H3_LIB=build/libh3b200_measure.so H3_DMMA_CFG=$c timeout 120 python tools/variant_check.py 3 $shape
  done
done > gpurun_out/${tag}_check.txt 2>&1
args=("base:")
for c in $variants; do args+=("v$c:H3_DMMA_CFG=$c"); done
tools/ab.sh 2 "${args[@]}" -- tools/time_fused.py 3 512 fused 4 > gpurun_out/${tag}_ab.txt 2>&1
echo done
