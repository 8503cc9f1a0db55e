cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "cfg3 or upwind_vs_oracle" 2>&1 | tail -3
timeout 900 python bench.py --steps 2 --warmup 3 --extra-3d 0 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
tail -3 gpurun_out/bench_cfg3.err
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg3.json')); c=d['config_3']; c.pop('t_krylov_ms',None); print(json.dumps(c)); print(d['value'], d['ms_per_step'])"
