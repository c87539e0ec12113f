cd $GRAFT_REPO_ROOT
python -m pytest tests -q -x -m gpu 2>&1 | tail -2
RTK_MSD_Q=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof_launches.csv python tools/prof_topk.py 28 1048576 3 > /dev/null 2>&1; echo "launches rc=$?"
RTK_MSD_Q=1 ncu --set full --clock-control none --import-source on -k regex:"k_msd_cluster|k_sort_groups|k_sample_select" -s 3 -c 3 \
    -o gpurun_out/prof_finish -f python tools/prof_topk.py 28 1048576 3 > gpurun_out/prof_finish.log 2>&1; echo "finish rc=$?"
timeout 600 python bench.py --no-cpu-baseline --steps 20 --e2e-steps 1 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench.json'))
print('value',round(d['value']),'ms',d['ms_per_step'])
print('batch',{k:(round(v['ms_per_batch'],4),round(v['queries_per_s'])) for k,v in d['batch_llm']['results'].items()}); print('bf16',{k:(round(v['ms_per_batch'],4),round(v['queries_per_s'])) for k,v in d['batch_llm_bf16']['results'].items()})
PY
