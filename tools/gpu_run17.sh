RTK_PROFILE=1 timeout 120 python -c "
import torch, paper_2501_14336_b200 as rtk
x=torch.randn(256,128256,device='cuda')
for kb in [50,4096]:
    for _ in range(2): r=rtk.batch_topk_dense(x, kb)
" 2>&1 | tail -8
