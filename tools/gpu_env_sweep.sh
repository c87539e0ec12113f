#!/bin/bash
# C2 k=2^20 under engine knobs (one process per setting)
for e in "RTK_NONE=1" "RTK_MSD_BITS=13" "RTK_MSD_BITS=12" "RTK_SAMPLE_R=256" "RTK_SAMPLE_R=1024" "RTK_MSD_Q=8" "RTK_MSD_Q=12" "RTK_DYN=6" "RTK_DYN=24" "RTK_SPARSE_MAX=0"; do
  env $e timeout 120 python tools/ab_env.py c2 1048576
done
