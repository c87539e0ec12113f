for v in "A=1" "A=2"; do
  env $v timeout 300 python bench.py --no-cpu-baseline --steps 30 --e2e-steps 1 --batch-ks "" > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['ms_per_step'],4), {k:round(v['ms_per_step'],4) for k,v in d['k_sweep'].items()}, {k:round(v['ms'],4) for k,v in d['adversarial_c4']['results'].items()})" || tail -3 gpurun_out/ab.err
done
