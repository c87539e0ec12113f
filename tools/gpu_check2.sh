cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log | grep -v '^\s*$' | tail -3
timeout 600 python bench.py --batch-ks "" --no-cpu-baseline > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c4.json')); print(d['ms_per_step'], {k:v['ms_per_step'] for k,v in d['k_sweep'].items()}, json.dumps({k:v['ms'] for k,v in d['adversarial_c4']['results'].items()}))"
bash tools/gpu_marks_c4.sh | tail -4
