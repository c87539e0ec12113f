cd $GRAFT_REPO_ROOT
for k in 1048576 256; do
python tools/ab_env.py c2 $k
RTK_PDL_COMPACT=1 python tools/ab_env.py c2 $k
RTK_PREFETCH_MB=64 python tools/ab_env.py c2 $k
RTK_PDL_COMPACT=1 RTK_PREFETCH_MB=64 python tools/ab_env.py c2 $k
RTK_SAMPLE_R=256 python tools/ab_env.py c2 $k
RTK_SAMPLE_R=1024 python tools/ab_env.py c2 $k
RTK_DYN=0 python tools/ab_env.py c2 $k
RTK_DYN=24 python tools/ab_env.py c2 $k
done
RTK_MSD_Q=8 python tools/ab_env.py c2 1048576
RTK_MSD_Q=16 python tools/ab_env.py c2 1048576
RTK_MSD_BITS=13 python tools/ab_env.py c2 1048576
python tools/ab_env.py c2 16384
