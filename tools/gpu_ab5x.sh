# three-way A/B of m=5 fused K orders: old (x1 only) vs x1+x3 vs x1+x2
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=paper_1609_09841_b200/libh3b200.so
{
for r in 1 2; do
  for v in old x13 x12; do
    if [ $v = old ]; then cp paper_1609_09841_b200/libh3b200_old.so $L; else cp paper_1609_09841_b200/libh3b200_$v.so $L; fi
    echo -n "$v "; timeout 200 python tools/time_fused.py 5 256 fused 4
  done
done
} > gpurun_out/ab5x.txt 2>&1
