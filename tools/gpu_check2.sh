cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp paper_2501_14336_b200/librtk_b200.so /tmp/lib_cur.so
for v in A B C A B C; do
  cp paper_2501_14336_b200/build/var/lib_$v.so paper_2501_14336_b200/librtk_b200.so
  echo "== $v"; KS=1048576 timeout 300 python tools/c2_ab.py ""
done > gpurun_out/var.log 2>&1
cp /tmp/lib_cur.so paper_2501_14336_b200/librtk_b200.so
cat gpurun_out/var.log
