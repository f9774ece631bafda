#!/bin/bash
# Round-end evidence session (one gpurun call): ncu launch list of the bench, ncu --set full captures
# of every product hot kernel, the DFMA N=3 fused A/B capture (DMMA vs DFMA evidence), SASS of the
# built library.  usage: tools/gpu_final.sh TAG      (outputs gpurun_out/TAG_*)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
tag=${1:-r02}
mkdir -p gpurun_out
make -C paper_1609_09841_b200/csrc measure -j16 > gpurun_out/${tag}_make.txt 2>&1
full="ncu --set full --clock-control none --import-source on"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extras > gpurun_out/${tag}_launches.log 2>&1
timeout 900 $full -k regex:sep_fused -s 2 -c 1 -o gpurun_out/${tag}_fused3_512 -f \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extras > gpurun_out/${tag}_prof.log 2>&1
timeout 600 $full -k regex:sep_fused -s 2 -c 1 -o gpurun_out/${tag}_fused3_256 -f python tools/time_fused.py 3 256 fused 1 >> gpurun_out/${tag}_prof.log 2>&1
H3_LIB=build/libh3b200_measure.so H3_FUSED_IMPL=dfma timeout 600 $full -k regex:sep_fused -s 2 -c 1 -o gpurun_out/${tag}_fused3_256_dfma -f \
  python tools/time_fused.py 3 256 fused 1 >> gpurun_out/${tag}_prof.log 2>&1
timeout 600 $full -k regex:"recon_dmma3|sep_evolve" -s 4 -c 2 -o gpurun_out/${tag}_two3_256 -f python tools/time_fused.py 3 256 two_pass 1 >> gpurun_out/${tag}_prof.log 2>&1
timeout 600 $full -k regex:sep_fused -s 2 -c 1 -o gpurun_out/${tag}_fused5_256 -f python tools/time_fused.py 5 256 fused 1 >> gpurun_out/${tag}_prof.log 2>&1
timeout 900 $full -k regex:"recon_dmma|sep_evolve" -s 4 -c 2 -o gpurun_out/${tag}_two5_128 -f python tools/time_fused.py 5 128 two_pass 1 >> gpurun_out/${tag}_prof.log 2>&1
tools/ab.sh 2 "dmma:" "dfma:H3_FUSED_IMPL=dfma" -- tools/time_fused.py 3 512 fused 4 > gpurun_out/${tag}_dfma_ab.txt 2>&1
echo done
