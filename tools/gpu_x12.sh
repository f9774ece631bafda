#!/bin/bash
# m=3 x12-chained fused kernel variants (h3_dmma3x.cu): correctness, timing vs the product kernel,
# one ncu capture.   usage: tools/gpu_x12.sh TAG "VARIANTS" PROFILE_CFG
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
tag=$1; variants=$2; prof=$3
mkdir -p gpurun_out
make -C paper_1609_09841_b200/csrc measure -j16 > gpurun_out/${tag}_make.txt 2>&1
for c in $variants; do
  for shape in "40 36 20" "16 14 9"; do
    H3_LIB=build/libh3b200_measure.so H3_DMMA_CFG=$c timeout 120 python tools/variant_check.py 3 $shape
  done
done > gpurun_out/${tag}_check.txt 2>&1
args=("base:")
for c in $variants; do args+=("v$c:H3_DMMA_CFG=$c"); done
tools/ab.sh 2 "${args[@]}" -- tools/time_fused.py 3 512 fused 4 > gpurun_out/${tag}_ab.txt 2>&1
if [ -n "$prof" ]; then
  H3_LIB=build/libh3b200_measure.so H3_DMMA_CFG=$prof timeout 600 ncu --set full --clock-control none --import-source on -k regex:sep_fused -s 2 -c 1 -o gpurun_out/${tag}_v$prof -f python tools/time_fused.py 3 256 fused 1 > gpurun_out/${tag}_prof.log 2>&1
fi
echo done
