timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench4.json 2> gpurun_out/bench4.err
python -c "
import json;d=json.load(open('gpurun_out/bench4.json'));print(d['value'],d['ms_per_step'],d['roofline'],d['k_sweep'])"; tail -3 gpurun_out/bench4.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_compact -c 1 -o gpurun_out/compact4 python tools/prof_topk.py 28 1048576 1 > gpurun_out/ncu4.log 2>&1
tail -1 gpurun_out/ncu4.log
