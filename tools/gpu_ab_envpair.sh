#!/bin/bash
# same-box A/B of one engine knob: tools/gpu_ab_envpair.sh "ENV=a" "ENV=b" -- workloads...
A=$1; B=$2; shift 3
for rep in 1 2; do for w in "$@"; do
  env $A timeout 120 python tools/ab_env.py $w; env $B timeout 120 python tools/ab_env.py $w
done; done
