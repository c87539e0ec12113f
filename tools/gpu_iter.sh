# iteration: parity tests, per-stage marks for C2/C3, short bench (1 GPU)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -8
timeout 300 bash tools/gpu_prof_marks.sh > /dev/null 2>&1; bash tools/gpu_c4.sh
grep -E "^k |^batch|profile" gpurun_out/marks.log | awk 'NR%4==0 || /^k|^batch/' | cut -c1-330
timeout 600 python bench.py --no-cpu-baseline --steps 20 --e2e-steps 1 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench.json'))
print('value',round(d['value']),'ms',d['ms_per_step'],'roof',d['roofline']['frac'])
print('sweep',{k:(round(v['ms_per_step'],4),round(v['GBps'])) for k,v in d['k_sweep'].items()}); print("c4", {k:(round(v["ms"],4), round(v["GBps"])) for k,v in d["adversarial_c4"]["results"].items()}); print('batch',{k:(round(v['ms_per_batch'],4),round(v['queries_per_s'])) for k,v in d['batch_llm']['results'].items()}); print('bf16',{k:(round(v['ms_per_batch'],4),round(v['queries_per_s'])) for k,v in d['batch_llm_bf16']['results'].items()})
PY
