cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log | grep -v '^\s*$' | tail -2
cp paper_2501_14336_b200/librtk_b200.so /tmp/lib_cur.so
for v in old new old new; do
  cp paper_2501_14336_b200/build/var/lib_$v.so paper_2501_14336_b200/librtk_b200.so
  echo "== $v"; KS=50 DT=f32,bf16 timeout 300 python tools/c3_ab.py ""
done > gpurun_out/var.log 2>&1
cp /tmp/lib_cur.so paper_2501_14336_b200/librtk_b200.so
cat gpurun_out/var.log
