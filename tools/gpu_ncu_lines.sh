# per-CUDA-line instruction/stall profile of one kernel: tools/gpu_ncu_lines.sh NAME REGEX ARGS...
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out /tmp/ncu
N=$1; RX=$2; shift 2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 1 -c 1 -o /tmp/ncu/$N -f "$@" > /tmp/ncu/$N.log 2>&1; echo "cap rc=$?"
python tools/ncu_lines.py /tmp/ncu/$N.ncu-rep 45 > gpurun_out/lines_$N.txt 2>&1
python tools/ncu_summary.py /tmp/ncu/$N.ncu-rep 5 >> gpurun_out/lines_$N.txt 2>&1
