timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench14.json 2> gpurun_out/bench14.err
python -c "
import json;d=json.load(open('gpurun_out/bench14.json'));print(d['value'],d['ms_per_step'],d['roofline']['kernel_ms'],d['k_sweep']); print(json.dumps(d['batch_llm']))"; tail -3 gpurun_out/bench14.err
RTK_PROFILE=1 timeout 120 python -c "
import torch, paper_2501_14336_b200 as rtk
V=128256; B=256
x=torch.randn(B*V, device='cuda')
for kb in [50,4096,128256]:
    bi=rtk.BatchInput(x,[i*V for i in range(B)],[V]*B,[kb]*B)
    for _ in range(2): rtk.batch_topk(bi)
    print(kb, rtk.last_stats())
" 2>&1 | grep -v "^\[rtk sample" | tail -8
