timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -x -q -k "lsd or vocab or 128256 or c3 or 16bit or batch" --timeout=600 2>&1 | tail -3
bash tools/gpu_lsd_trace.sh
