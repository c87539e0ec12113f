cd $GRAFT_REPO_ROOT
for a in "c1 256" "c3 50" "c3 4096" "c3b 50"; do
  python tools/ab_env.py $a; RTK_NO_FUSED=1 python tools/ab_env.py $a
done
python tools/ab_env.py c2 256; python tools/ab_env.py c2 1048576
