cd $GRAFT_REPO_ROOT
python tools/prof_solve.py --ce --n 1025 2>&1 | tail -3
P=29711
run() { P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $P tools/dist_check.py "${@:2}" 2>&1 | grep -v "^\s*File\|^\s*\^\|OMP_NUM\|^\*\*\*" | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); [d.pop(k) for k in ('history','history_single')]; print(json.dumps(d))
    else: print(l.rstrip()[:300])
"; }
run 1 --case cfg4:257 --backend nccl
run 1 --case cfg4:513 --backend nccl
