cd $GRAFT_REPO_ROOT
cp paper_2501_14336_b200/librtk_b200.so /tmp/lib_cur.so
for v in ${VARS:-A B C D}; do
  cp paper_2501_14336_b200/build/var/lib_$v.so paper_2501_14336_b200/librtk_b200.so
  echo "== $v k=50"; BS=148,256 K=50 bash tools/gpu_c3rows.sh | grep -E "^B"
  echo "== $v k=4096"; BS=148,256 K=4096 bash tools/gpu_c3rows.sh | grep -E "^B"
done
cp /tmp/lib_cur.so paper_2501_14336_b200/librtk_b200.so
