timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -25
timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench5.json 2> gpurun_out/bench5.err
python -c "
import json;d=json.load(open('gpurun_out/bench5.json'));print(d['value'],d['ms_per_step'],d['roofline']['kernel_ms'],d['k_sweep'])"; tail -3 gpurun_out/bench5.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches5.csv python tools/prof_topk.py 28 1048576 1 > /dev/null 2>&1
