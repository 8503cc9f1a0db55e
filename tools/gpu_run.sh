cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 1500 python bench.py --extra-3d 0 --extra-cfg3 0 --no-cpu-baseline > gpurun_out/b.json 2> gpurun_out/b.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/b.json')); print(d['value'], d['ms_per_step'], d['e2e'])"
