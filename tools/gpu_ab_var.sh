#!/bin/bash
# same-box A/B: ab/<variant> builds (tools/build_variant.sh) and the working tree; args: variants -- workloads
vars=(); while [ "$1" != "--" ]; do vars+=("$1"); shift; done; shift
for rep in 1 2; do
for w in "$@"; do
  for v in "${vars[@]}"; do RTK_PKG_ROOT=ab/$v timeout 120 python tools/ab_env.py $w | sed "s/^/$v /"; done
  timeout 120 python tools/ab_env.py $w | sed 's/^/NEW  /'
done; done
