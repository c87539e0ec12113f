cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in "" ab/rowsold; do for a in "c3 50" "c3 4096" "c3b 50" "c3b 4096"; do echo -n "${v:-tree} "; RTK_PKG_ROOT=$GRAFT_REPO_ROOT/$v python tools/ab_env.py $a; done; done; done
timeout 900 python -m pytest tests -m gpu -q -k "batch or vocab or c3_headline or 16bit or sample or ties or rows" --timeout=600 2>&1 | tail -2
