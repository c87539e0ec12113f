#!/bin/bash
cd $GRAFT_REPO_ROOT
for k in 1 256 512; do RTK_ROWS_TRACE=1 RTK_PROFILE=1 python tools/prof_marks.py c1 $k 2>&1 | grep -E "rows trace|mark|us" | tail -12; done
