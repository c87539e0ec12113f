set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch;p=torch.cuda.get_device_properties(0);print(p, p.L2_cache_size if hasattr(p,'L2_cache_size') else '')"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -40 > gpurun_out/pytest1.txt
cat gpurun_out/pytest1.txt
timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench1.json 2> gpurun_out/bench1.err
tail -c 3000 gpurun_out/bench1.json; tail -20 gpurun_out/bench1.err
