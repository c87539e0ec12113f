set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest2.txt
cat gpurun_out/pytest2.txt
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err
tail -c 2500 gpurun_out/bench2.json; tail -5 gpurun_out/bench2.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2.csv python tools/prof_topk.py 28 1048576 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_compact -c 1 -o gpurun_out/compact2 python tools/prof_topk.py 28 1048576 1 > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu2.log
