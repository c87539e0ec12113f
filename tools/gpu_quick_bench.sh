cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python bench.py --legs "" --no-cpu-baseline --steps 30 > gpurun_out/qb.json 2> gpurun_out/qb.err; echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/qb.json')); print('C2 k=2^20', round(d['ms_per_step']*1e3,1), 'us', round(d['fraction_of_hbm_peak'],4), 'compact', round(d['roofline']['kernel_ms']*1e3,1), {k: round(v['ms']*1e3,1) for k,v in d['k_sweep'].items()})"
