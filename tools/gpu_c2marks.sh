#!/bin/bash
for k in 256 1048576; do RTK_PROFILE=1 python tools/prof_marks.py c2 $k 2>&1 | grep -E "rtk profile|rtk dbg" | tail -3; done
MODE=0 RTK_PROFILE=1 python tools/prof_marks.py c4 2>&1 | grep -E "rtk profile|rtk dbg" | tail -3
