# Round-2 evidence (1 GPU): GPU suite + smoke + bench line + reference arm, ncu launch lists of the
# bench configs and full-capture summaries of the top kernels. Run under gpurun; outputs (text and
# JSON only: gpurun returns at most 64 MiB) in gpurun_out/r2/.
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2; mkdir -p $O /tmp/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader > $O/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> $O/gpu.txt
if [ -z "$SKIP_TESTS" ]; then
timeout 1700 python -m pytest tests -m gpu -q --timeout=600 --timeout-method=thread > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
fi
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_arm.json 2> $O/bench_ref.err; echo "ref rc=$?"
NCCL_DEBUG=INFO NCCL_DEBUG_FILE=/dev/stderr timeout 600 python bench.py --sharded-1gpu --steps 10 --warmup 3 > $O/bench_sharded_1gpu.json 2> $O/bench_sharded.err; echo "sharded rc=$?"
grep -E "NCCL INFO (comm|nranks|Init)" $O/bench_sharded.err | head -5 > $O/nccl_info.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
launches() { local name=$1; shift; timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_$name.csv "$@" > /dev/null 2>&1; echo "launches $name rc=$?"; }
launches c2_k2p20 env RTK_MSD_Q=1 python tools/prof_marks.py c2 1048576
launches c2_k256 python tools/prof_marks.py c2 256
launches c1 python tools/prof_marks.py c1 256
launches c3_k50 python tools/prof_marks.py c3 50
launches c3_k4096 python tools/prof_marks.py c3 4096
launches c3_vocab python tools/prof_marks.py c3 128256
launches c3_bf16_vocab env BF16=1 python tools/prof_marks.py c3 128256
launches c4_off env MODE=0 RTK_MSD_Q=1 python tools/prof_marks.py c4
launches c4_adaptive env MODE=2 RTK_MSD_Q=1 python tools/prof_marks.py c4
cap() {  # name, kernel regex, skip, count, [env...] python args...
  local name=$1 rx=$2 s=$3 c=$4; shift 4
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $s -c $c \
    -o /tmp/ncu/$name -f "$@" > /tmp/ncu/$name.log 2>&1; echo "cap $name rc=$?"
  python tools/ncu_summary.py /tmp/ncu/$name.ncu-rep 25 > $O/ncu_$name.txt 2>&1
}
cap compact "k_compact" 1 1 python tools/prof_marks.py c2 1048576
cap sample_c2 "k_sample_select" 1 1 python tools/prof_marks.py c2 1048576
cap sort_c2 "k_sort_groups" 1 1 python tools/prof_marks.py c2 1048576
cap rows50 "k_rows_fused" 1 1 python tools/prof_marks.py c3 50
cap rows4096 "k_rows_fused" 1 1 python tools/prof_marks.py c3 4096
cap lsd "k_lsd_pass" 1 1 python tools/prof_marks.py c3 128256
cap compact_c4a "k_compact" 1 1 env MODE=2 python tools/prof_marks.py c4
cap row_cluster "k_row_cluster" 1 1 python tools/prof_marks.py c1 256
cap radix_exact "k_radix_pass" 1 1 env RTK_FORCE_EXACT=1 python tools/prof_marks.py c1 256
cap sample_rows "k_sample_rows" 1 1 python tools/prof_marks.py samp 50
# the shipped multi-cluster level-0 MSD (cooperative launch, grid barrier): application replay,
# no graph capture (every call launches it directly)
timeout 900 ncu --set full --replay-mode application --clock-control none --import-source on -k regex:"k_msd_cluster" -s 1 -c 1 \
  -o /tmp/ncu/msd_q16 -f env RTK_GRAPHS=0 python tools/prof_marks.py c2 1048576 > /tmp/ncu/msd_q16.log 2>&1; echo "cap msd_q16 rc=$?"
python tools/ncu_summary.py /tmp/ncu/msd_q16.ncu-rep 25 > $O/ncu_msd_q16.txt 2>&1
tail -3 /tmp/ncu/msd_q16.log >> $O/ncu_msd_q16.txt
