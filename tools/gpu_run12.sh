timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -15
RTK_PROFILE=1 timeout 300 python tools/prof_topk.py 28 1048576 3 2>&1 | tail -2
RTK_PROFILE=1 timeout 300 python tools/prof_topk.py 28 256 3 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench12.json 2> gpurun_out/bench12.err
python -c "
import json;d=json.load(open('gpurun_out/bench12.json'));print(d['value'],d['ms_per_step'],d['roofline']['kernel_ms'],d['k_sweep'])"; tail -3 gpurun_out/bench12.err
