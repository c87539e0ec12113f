timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15
RTK_PROFILE=1 timeout 120 python -c "
import torch, paper_2501_14336_b200 as rtk
x=torch.randn(256,128256,device='cuda')
for kb in [50,4096]:
    for _ in range(3): r=rtk.batch_topk_dense(x, kb)
    print(kb, rtk.last_stats())
" 2>&1 | grep -v "^\[rtk sample" | tail -6
timeout 300 python bench.py --no-cpu-baseline --steps 20 --sweep "" > gpurun_out/bench16.json 2> gpurun_out/bench16.err
python -c "
import json;d=json.load(open('gpurun_out/bench16.json'));print(d['value'],d['ms_per_step']); print(json.dumps(d['batch_llm']))"; tail -3 gpurun_out/bench16.err
