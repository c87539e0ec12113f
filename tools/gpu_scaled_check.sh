cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -k "scaled or nan or adaptive or c4 or special or sanitizer" --timeout=600 2>&1 | tail -3
for m in 0 1 2; do python tools/ab_env.py c4 65536 $m; done
