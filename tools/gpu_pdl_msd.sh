#!/bin/bash
for v in "RTK_GRAPH_EVENTS=1" "RTK_GRAPH_EVENTS=0" "RTK_GRAPH_EVENTS=0 RTK_PDL_MSD=1" "RTK_GRAPH_EVENTS=1 RTK_PDL_MSD=1"; do
  for w in "c2 1048576" "c2 256" "c4 65536 0" "c3 20000"; do env $v timeout 120 python tools/ab_env.py $w; done
done
RTK_GRAPH_EVENTS=0 RTK_PDL_MSD=1 timeout 600 python -m pytest tests/test_gpu_headline.py -x -q -k "c2 or c4" --timeout=300 2>&1 | tail -2
