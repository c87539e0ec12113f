python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -4
timeout 600 python bench.py > gpurun_out/bench15.json 2> gpurun_out/bench15.err
python -c "
import json;d=json.load(open('gpurun_out/bench15.json'));d.pop('step_ms_all');print(json.dumps(d))"; tail -3 gpurun_out/bench15.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench15_ref.json 2>&1; tail -1 gpurun_out/bench15_ref.json
bash tools/profile_round.sh > gpurun_out/profile15.log 2>&1; tail -2 gpurun_out/profile15.log
nproc; lscpu | grep "Model name"
