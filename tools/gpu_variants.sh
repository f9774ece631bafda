#!/bin/bash
# A/B session for measurement-build kernel variants (one gpurun call):
#   correctness of each variant vs the literal kernel (tools/variant_check.py, ragged grids),
#   interleaved timing vs the product library (tools/ab.sh), optional ncu --set full capture.
#
# usage: tools/gpu_variants.sh FAMILY TAG "VARIANTS" [PROFILE_VARIANT]
#   a variant is a number k (sets the family's variable to k) or any H3_* assignment (H3_DMMA_BAND=8)
#   FAMILY m3: m=3 fused kernels        (H3_DMMA_CFG:  10x warp-specialised, 20x x1->x2 chained)
#          m5: m=5 fused kernels        (H3_DMMA5_CFG: lock-step shapes, 20+k warp-specialised)
#          r5: m=5 reconstruction       (H3_RECON5_WS: warp-specialised variants)
#          r3: m=3 two-kernel step      (H3_BAND: tile rasterisation of the reconstruction)
# outputs: gpurun_out/TAG_{make,check,ab,prof}.txt, gpurun_out/TAG_vK.ncu-rep
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
family=$1; tag=$2; variants=$3; prof=$4
case $family in
  m3) var=H3_DMMA_CFG;  order=3; mode=fused;    tsize=512; tsteps=4; psize=256; kre=sep_fused ;;
  m5) var=H3_DMMA5_CFG; order=5; mode=fused;    tsize=256; tsteps=4; psize=128; kre=sep_fused ;;
  r5) var=H3_RECON5_WS; order=5; mode=two_pass; tsize=256; tsteps=2; psize=128; kre=recon ;;
  r3) var=H3_BAND;      order=3; mode=two_pass; tsize=256; tsteps=4; psize=128; kre=recon ;;
  *) echo "unknown family $family"; exit 2 ;;
esac
mkdir -p gpurun_out
make -C paper_1609_09841_b200/csrc measure -j16 > gpurun_out/${tag}_make.txt 2>&1
setting() { if [[ $1 == *=* ]]; then echo "$1"; else echo "$var=$1"; fi; }
for c in $variants; do
  for shape in "40 36 20" "16 14 9" "9 7 5"; do
    env H3_LIB=build/libh3b200_measure.so $(setting $c) timeout 120 python tools/variant_check.py $order $shape $mode
  done
done > gpurun_out/${tag}_check.txt 2>&1
args=("base:")
for c in $variants; do args+=("v$c:$(setting $c)"); done
tools/ab.sh 2 "${args[@]}" -- tools/time_fused.py $order $tsize $mode $tsteps > gpurun_out/${tag}_ab.txt 2>&1
if [ -n "$prof" ]; then
  env H3_LIB=build/libh3b200_measure.so $(setting $prof) timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:$kre -s 2 -c 1 -o gpurun_out/${tag}_v${prof//=/_} -f python tools/time_fused.py $order $psize $mode 1 \
    > gpurun_out/${tag}_prof.txt 2>&1
fi
echo done
