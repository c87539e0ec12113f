timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -4
bash tools/gpu_run17.sh
timeout 300 python bench.py --no-cpu-baseline --steps 10 --sweep "" --e2e-steps 1 > gpurun_out/bench18.json 2> gpurun_out/bench18.err
python -c "
import json;d=json.load(open('gpurun_out/bench18.json'));print(d['value'],d['ms_per_step']); print(json.dumps(d['batch_llm']['results']))"; tail -3 gpurun_out/bench18.err
