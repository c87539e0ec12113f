# A/B of two builds on one box: LIBS="old new" (paper_2501_14336_b200/build/var/lib_<x>.so)
cd $GRAFT_REPO_ROOT
cp paper_2501_14336_b200/librtk_b200.so /tmp/lib_cur.so
for rep in 1 2; do
for v in ${LIBS:-old new}; do
  cp paper_2501_14336_b200/build/var/lib_$v.so paper_2501_14336_b200/librtk_b200.so
  timeout 300 python bench.py --no-cpu-baseline --steps 30 --e2e-steps 1 --c4 ${C4:-0} --batch-ks ${BKS:-50} > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['ms_per_step'],4), {k:round(v['ms_per_step'],4) for k,v in d['k_sweep'].items()}, {k:(round(v['ms_per_batch'],4)) for k,v in d['batch_llm']['results'].items()}, {k:round(v['ms'],4) for k,v in d.get('adversarial_c4',{}).get('results',{}).items()})" || tail -3 gpurun_out/ab.err
done
done
cp /tmp/lib_cur.so paper_2501_14336_b200/librtk_b200.so
