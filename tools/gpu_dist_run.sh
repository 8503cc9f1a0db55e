cd $GRAFT_REPO_ROOT
P=29611
run() { P=$((P+1)); timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $P tools/dist_check.py "${@:2}" 2>&1 | grep -v "^\s*File\|^\s*\^\|OMP_NUM\|^\*\*\*" | cut -c1-700 | head -30; }
run 2 --case cfg4:33 --backend host --levels 3
run 1 --case cfg1:65 --backend nccl
run 2 --case cfg4:65 --backend host --levels 2 --c64 1
run 4 --case cfg4:65 --backend host --min-planes 4
run 2 --case cfg1:129 --backend host --min-planes 8
