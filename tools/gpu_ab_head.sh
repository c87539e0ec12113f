#!/bin/bash
# same-box A/B of the working tree against the build in ab/head (tools/ab_env.py workloads given as args)
for rep in 1 2; do
for w in "$@"; do
  RTK_PKG_ROOT=ab/head timeout 120 python tools/ab_env.py $w | sed 's/^/HEAD /'
  timeout 120 python tools/ab_env.py $w | sed 's/^/NEW  /'
done; done
