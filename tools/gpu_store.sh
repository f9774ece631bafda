# output-store cache policy of the N=3 fused kernel: .cs (default) vs write-back vs L1::no_allocate
# (needs paper_1609_09841_b200/libh3b200_v1.so / _v2.so built with -DH3_OUT_STORE=1 / 2 of the
#  out_store() helper used for this measurement; the shipped kernel keeps st.global.cs)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=paper_1609_09841_b200/libh3b200.so
cp $L /tmp/v0.so
{
for r in 1 2; do
  for v in 0 1 2; do
    if [ $v = 0 ]; then cp /tmp/v0.so $L; else cp paper_1609_09841_b200/libh3b200_v$v.so $L; fi
    echo -n "store$v "; timeout 200 python tools/time_fused.py 3 512 fused 10
  done
done
cp /tmp/v0.so $L
for v in 1 2; do cp paper_1609_09841_b200/libh3b200_v$v.so $L
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:sep_fused -s 2 -c 1 python tools/time_fused.py 3 512 fused 1 2>&1 | grep -E "dram__|gpu__time"
done
cp /tmp/v0.so $L
} > gpurun_out/store.txt 2>&1
