# A/B of env knobs on the C2 bench (device value + k sweep). usage: VARS="A=1 B=2;A=2" bash tools/gpu_ab2.sh
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARS}"
for v in "${VS[@]}"; do
  env $v timeout 300 python bench.py --no-cpu-baseline --steps 30 --e2e-steps 1 --c4 0 --batch-ks ${BKS:-50} > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['ms_per_step'],4), {k:round(v['ms_per_step'],4) for k,v in d['k_sweep'].items()}, {k:(round(v['ms_per_batch'],4)) for k,v in d['batch_llm']['results'].items()})" || tail -3 gpurun_out/ab.err
done
