cd $GRAFT_REPO_ROOT
cat > /tmp/seq.py <<'PY'
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch, oracle as O, paper_2501_14336_b200 as rtk
n = (1 << 20) + 3
x = O.ref_generate(1, n, 10000 + n * 7 + 3, dtype=np.float32, b=1.0)
t = torch.from_numpy(x).cuda()
for k in [n // 2, n]:
    r = rtk.topk(t, k)
    wv, wi, wp = O.ref_topk(x, k, 0, grid=4)
    gi = r.indices.cpu().numpy().astype(np.uint64)
    bad = np.nonzero(gi != wi)[0]
    print("k", k, "bad", bad.size, bad[:3], rtk.last_stats())
PY
for v in "A=1" "RTK_FORCE_INIT=1" "RTK_SELFCLEAN=0"; do echo "== $v"; env $v python /tmp/seq.py 2>&1 | grep -E "^k |ctl|Error|error" | head; done
