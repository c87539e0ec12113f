for v in "RTK_NO_FUSED=0" "RTK_NO_FUSED=1 RTK_SPARSE_MAX=96" "RTK_NO_FUSED=1 RTK_SPARSE_MAX=16" "RTK_SPARSE_MAX=16"; do
  env $v timeout 300 python bench.py --no-cpu-baseline --steps 20 --e2e-steps 1 --c4 0 --batch-ks 50,4096 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['ms_per_step'],4), {k:round(v['ms_per_step'],4) for k,v in d['k_sweep'].items()}, {k:(round(v['ms_per_batch'],4), round(v['queries_per_s'])) for k,v in d['batch_llm']['results'].items()})" || tail -3 gpurun_out/ab.err
done
RTK_NO_FUSED=1 RTK_SPARSE_MAX=16 RTK_PROFILE=1 python - <<'PY' 2>&1 | grep -E "profile" | tail -2
import torch, paper_2501_14336_b200 as rtk
L = torch.randn(256, 128256, device="cuda")
for k in (50, 4096):
    for _ in range(2): rtk.batch_topk_dense(L, k)
    torch.cuda.synchronize()
PY
