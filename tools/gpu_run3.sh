timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -5 > gpurun_out/pytest3.txt
cat gpurun_out/pytest3.txt
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err
python -c "
import json;d=json.load(open('gpurun_out/bench3.json'));d.pop('step_ms_all');print(json.dumps(d)[:3000])"; tail -3 gpurun_out/bench3.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv python tools/prof_topk.py 28 1048576 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_compact -c 1 -o gpurun_out/compact3 python tools/prof_topk.py 28 1048576 1 > gpurun_out/ncu3.log 2>&1
tail -1 gpurun_out/ncu3.log
