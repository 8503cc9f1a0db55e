# A/B timing of the committed build (tools/old/libhadr.so) against the working tree's,
# both in one gpurun call (box-to-box variation is ~20%).
set -x
for w in "cfg2 1025" "cfg4 513"; do
  set -- $w
  for rep in 1 2; do
    for lib in tools/old/libhadr.so paper_1712_06091_b200/libhadr.so; do
      echo "$1 $lib"; HADR_WORKLOAD=$1 HADR_LIB_PATH=$lib python tools/prof_solve.py --n $2 --its 1000 --warm 1
    done
  done
done
