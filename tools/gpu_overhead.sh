#!/bin/bash
# fixed per-call cost: graph replay vs plain launches
for g in 1 0; do
  for w in "tiny 1" "c1 256" "c3 50" "c4 65536 0"; do RTK_GRAPHS=$g timeout 120 python tools/ab_env.py $w; done
done
