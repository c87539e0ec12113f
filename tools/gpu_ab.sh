# A/B: prefetch budget with events off in graphs
for v in "RTK_PREFETCH_MB=0" "RTK_PREFETCH_MB=24" "RTK_PREFETCH_MB=48" "RTK_PREFETCH_MB=96"; do
  env $v RTK_GRAPH_EVENTS=0 timeout 300 python bench.py --no-cpu-baseline --steps 30 --e2e-steps 1 --batch-ks "" --c4 0 > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['ms_per_step'],4), {k:round(v['ms_per_step'],4) for k,v in d['k_sweep'].items()})"
done
