cd $GRAFT_REPO_ROOT
cat > /tmp/z.py <<'PY'
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch, oracle as O, paper_2501_14336_b200 as rtk
n = (1 << 20) + 3
x = O.ref_generate(2, n, 10000 + n * 7 + 2 * 3 + 0, dtype=np.uint32, b=1.0)
t = torch.from_numpy(x.view(np.int32)).cuda().view(torch.uint32)
for k in [n // 2]:
    for rep in range(2):
        r = rtk.topk(t, k)
        wv, wi, wp = O.ref_topk(x, k, 0, grid=4)
        gi = r.indices.cpu().numpy().astype(np.uint64)
        bad = np.nonzero(gi != wi)[0]
        print("k", k, "rep", rep, "bad", bad.size, bad[:3], bad[-3:] if bad.size else "", rtk.last_stats(), flush=True)
PY
RTK_CHECK_GROUPS=1 RTK_PROFILE=1 python /tmp/z.py 2>&1 | grep -E "^k |ctl|groups|gap|slot"
python /tmp/z.py 2>&1 | grep -E "^k "
