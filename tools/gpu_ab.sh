cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp paper_1609_09841_b200/libh3b200.so /tmp/new.so
{
for v in old new old new; do
  if [ $v = old ]; then cp paper_1609_09841_b200/libh3b200_old.so paper_1609_09841_b200/libh3b200.so; else cp /tmp/new.so paper_1609_09841_b200/libh3b200.so; fi
  echo $v; timeout 200 python tools/time_fused.py 5 256 fused 4; timeout 200 python tools/time_fused.py 5 128 fused 8
done
} > gpurun_out/ab.txt 2>&1
