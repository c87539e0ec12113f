cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python tools/c3_ab.py "" "B=1" "DT=bf16" > gpurun_out/c3ab.log 2>&1
cat gpurun_out/c3ab.log
timeout 600 python bench.py --c4 0 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench.json'))
print('value',d['value'],'ms',d['ms_per_step'],'pyloop',d.get('python_loop_ms'),'roof',d['roofline']['frac'],d['roofline']['kernel_share_of_step'])
print('sweep',d['k_sweep']); print('batch',json.dumps(d['batch_llm']['results']))
PY
